"""Integration-order harness on the B200 path.

The reference's `run_pipeline` (proj/src/harness.cpp:59-179, harness.hpp:14-101)
runs one of six integration orders of quantization and QUOTA pruning over a set
of eval samples and reports the mean L2 divergence of the final-position logits
from the full-precision forward, the prune traces, the final visual count and
the prefill GFLOPs of the executed schedule.  Here every forward runs on the
device through an `Engine`:

* full-precision forwards (fp_baseline, prune_only, and the FP reference of
  every mode) -> `Engine.prefill_fp` (fp64 on the device, k_fp.cu + DGEMM);
* quantized forwards -> `Engine.prefill` (the W4A4 hot path), batched;
* scale fits / inline recipe generation -> `Engine.fit_act_scales` /
  `Engine.run_quota_calibration`.

The host logic (mode table, sample synthesis, digests, cost model, report
JSON) is restated from the reference and pinned against it in
tests/test_harness_cpu.py.  Two deliberate differences, both from the device
path's weight layout: the engine quantizes weights per OUTPUT
channel, and the model is whatever the engine has loaded (the reference builds
it with init_model(config.model), model.cpp:113-135).
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field

import numpy as np

from . import lib

TOOL_VERSION = "0.1.0"  # version.hpp:5
RECIPE_SCHEMA_VERSION = 1  # recipe.hpp:36
FNV_SEED = 0xCBF29CE484222325  # digest.hpp:12

# harness.cpp:17-27, in enum order (harness.hpp:28-35)
MODES = ("fp_baseline", "quant_only", "prune_only", "quant_then_prune", "prune_then_quant", "collaborative")


def mode_name(mode: str) -> str:
    if mode not in MODES:
        return "unknown"
    return mode


def parse_mode(name: str):
    """parse_mode (harness.cpp:29-36): the mode, or None for an unknown name."""
    return name if name in MODES else None


def mode_prunes(mode):  # harness.cpp:46-49
    return mode in ("prune_only", "quant_then_prune", "prune_then_quant", "collaborative")


def mode_quantizes(mode):  # harness.cpp:51-54
    return mode in ("quant_only", "quant_then_prune", "prune_then_quant", "collaborative")


# ---------------------------------------------------------------- digests
def fnv1a64(data: bytes | np.ndarray, seed: int = FNV_SEED) -> int:
    """fnv1a64 (digest.hpp:12-20), computed by the native library."""
    b = np.ascontiguousarray(data).view(np.uint8) if isinstance(data, np.ndarray) else np.frombuffer(data, np.uint8)
    L = lib()
    L.qt_fnv1a64.restype = C.c_uint64
    L.qt_fnv1a64.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64]
    return int(L.qt_fnv1a64(b.ctypes.data if b.size else None, b.size, seed))


def to_hex(h: int) -> str:  # digest.hpp:27-35
    return f"{h & 0xFFFFFFFFFFFFFFFF:016x}"


def hex_digest(x) -> str:
    """hex_digest (digest.hpp:37-43) of fp64 values or of a string."""
    if isinstance(x, str):
        return to_hex(fnv1a64(x.encode()))
    return to_hex(fnv1a64(np.ascontiguousarray(x, dtype=np.float64)))


# ---------------------------------------------------------------- samples
_GAMMA = np.uint64(0x9E3779B97F4A7C15)


def _splitmix_block(state: int, n: int):
    """The next n outputs of SplitMix64 (rng.hpp:15-20) from `state`, vectorised: the
    generator is a counter, output i = mix(state + (i + 1) * gamma)."""
    with np.errstate(over="ignore"):
        z = np.uint64(state) + (np.arange(1, n + 1, dtype=np.uint64) * _GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z, (state + n * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF


def mix_seed(seed: int, index: int) -> int:  # rng.hpp:41-45
    s = (seed ^ ((0x632BE59BD9B4E019 + index * 0xFF51AFD7ED558CCD) & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF
    z, _ = _splitmix_block(s, 1)
    return int(z[0])


@dataclass
class Sample:
    """CalibSample (calibrator.hpp): embeddings [visual + text x d_model] fp64, prefix layout."""
    embeddings: np.ndarray
    visual: int
    text: int

    def as_tuple(self):
        return (self.embeddings, self.visual, self.text)


def make_calibration_samples(seed, count, v0, d_model, text_min, text_max):
    """make_calibration_samples (calibrator.cpp:12-29): per sample a SplitMix64 stream seeded
    mix_seed(seed, i); text count next_int(text_min, text_max), then U[-1, 1) embeddings."""
    if count < 1:
        raise ValueError("need at least one sample")
    if v0 < 1 or d_model < 1:
        raise ValueError("invalid sample dims")
    if text_min < 1 or text_max < text_min:
        raise ValueError("invalid text range")
    out = []
    for i in range(count):
        st = mix_seed(seed, i)
        z, st = _splitmix_block(st, 1)
        span = text_max - text_min + 1
        t = text_min + int(int(z[0]) % span)  # next_int, rng.hpp:34-37
        n = (v0 + t) * d_model
        z, st = _splitmix_block(st, n)
        u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)  # next_double, rng.hpp:23-25
        emb = (-1.0 + 2.0 * u).reshape(v0 + t, d_model)  # next_uniform(-1, 1), rng.hpp:28-30
        out.append(Sample(emb, v0, t))
    return out


def sample_set_digest(samples) -> str:
    """sample_set_digest (calibrator.cpp:31-40): FNV-1a over embeddings, positions, counts."""
    h = FNV_SEED
    for s in samples:
        e, v, t = s.as_tuple() if isinstance(s, Sample) else s
        h = fnv1a64(np.ascontiguousarray(e, dtype=np.float64), h)
        h = fnv1a64(np.arange(v + t, dtype=np.int32), h)
        h = fnv1a64(np.array([v, t], dtype=np.int32), h)
    return to_hex(h)


# ---------------------------------------------------------------- recipe
@dataclass
class MetricWeights:
    """MetricWeights (recipe.hpp:12-23)."""
    mag: float = 0.25
    inter: float = 0.45
    intra: float = 0.10
    quant: float = 0.20

    def sum(self):
        return self.mag + self.inter + self.intra + self.quant

    def without_quant(self):  # recipe.cpp:16-19
        share = self.quant / 3.0
        return MetricWeights(self.mag + share, self.inter + share, self.intra + share, 0.0)

    def as_tuple(self):
        return (self.mag, self.inter, self.intra, self.quant)


@dataclass
class PruningRecipe:
    """PruningRecipe (recipe.hpp:25-54)."""
    candidate_layers: list
    keep_ratios: list
    weights: MetricWeights = field(default_factory=MetricWeights)
    v0: int = 64
    quant_digest: str = ""
    schema_version: int = RECIPE_SCHEMA_VERSION

    def validate(self):  # recipe.cpp:21-46
        if self.schema_version != RECIPE_SCHEMA_VERSION:
            raise ValueError("unsupported recipe schema_version")
        if not self.candidate_layers or len(self.candidate_layers) != len(self.keep_ratios):
            raise ValueError("candidate_layers and keep_ratios must align and be nonempty")
        for i, (l, r) in enumerate(zip(self.candidate_layers, self.keep_ratios)):
            if l < 0:
                raise ValueError("negative candidate layer")
            if i > 0 and l <= self.candidate_layers[i - 1]:
                raise ValueError("candidate layers must be strictly increasing")
            if not (0.0 < r <= 1.0):
                raise ValueError("keep ratio outside (0,1]")
            if i > 0 and r > self.keep_ratios[i - 1] + 1e-12:
                raise ValueError("keep ratios must be non-increasing")
        w = self.weights
        if w.mag < 0 or w.inter < 0 or w.intra < 0 or w.quant < 0:
            raise ValueError("negative metric weight")
        if abs(w.sum() - 1.0) > 1e-9:
            raise ValueError("metric weights must sum to 1")
        if self.v0 < 1:
            raise ValueError("v0 must be >= 1")

    def serialize(self) -> str:
        """serialize_recipe (recipe.cpp:48-61): the JSON document, keys sorted, indent 2."""
        self.validate()
        j = {
            "schema_version": self.schema_version,
            "candidate_layers": [int(x) for x in self.candidate_layers],
            "keep_ratios": [float(x) for x in self.keep_ratios],
            "metric_weights": {"mag": self.weights.mag, "inter": self.weights.inter, "intra": self.weights.intra,
                               "quant": self.weights.quant},
            "v0": int(self.v0),
            "quant_digest": self.quant_digest,
        }
        return _dump2(j) + "\n"

    def digest(self) -> str:  # recipe.cpp:132-134
        return hex_digest(self.serialize())


def _num(x):
    if isinstance(x, bool):
        return "true" if x else "false"
    if isinstance(x, int):
        return str(x)
    if isinstance(x, float):
        if math.isfinite(x) and x == int(x) and abs(x) < 1e16:
            return f"{x:.1f}"  # nlohmann prints integral doubles as "1.0"
        return repr(x)  # shortest round-trip, like nlohmann's dtoa
    return json.dumps(x)


def _dump2(v, ind=0) -> str:
    """nlohmann::json::dump(2) as the reference's JSON library (nlohmann 3.11.3, the copy the
    oracle builds against; the reference's vendor/ tree is not shipped) prints it: objects with
    keys sorted, one member per line; float arrays one element per line, integer arrays
    inline; empty containers as {} / [].  Pinned in tests/test_harness_cpu.py."""
    pad, pad1 = " " * ind, " " * (ind + 2)
    if isinstance(v, dict):
        if not v:
            return "{}"
        items = [f'{pad1}{json.dumps(k)}: {_dump2(v[k], ind + 2)}' for k in sorted(v)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(v, (list, tuple)):
        if not v:
            return "[]"
        if all(isinstance(x, int) and not isinstance(x, bool) for x in v):
            return "[" + ",".join(str(x) for x in v) + "]"  # integer arrays stay on one line
        return "[\n" + ",\n".join(pad1 + _dump2(x, ind + 2) for x in v) + "\n" + pad + "]"
    return _num(v)


def quant_digest(weight_bits=4, act_bits=4, kv_bits=4):  # quant.cpp:121-124
    return f"w{weight_bits}a{act_bits}kv{kv_bits}-sym-rne"


# ---------------------------------------------------------------- cost model
@dataclass
class CostModel:
    """CostModel (gflops.hpp:22-31)."""
    f_vt: float = 0.0
    f_pj: float = 0.0
    d_model: int = 32
    d_ff: int = 128
    n_heads: int = 4
    text_len: int = 16

    def validate(self):  # gflops.cpp:9-14
        if self.f_vt < 0 or self.f_pj < 0:
            raise ValueError("negative constant cost")
        if self.d_model < 1 or self.d_ff < 1 or self.n_heads < 1:
            raise ValueError("invalid dims")
        if self.d_model % self.n_heads != 0:
            raise ValueError("d_model must divide by n_heads")
        if self.text_len < 0:
            raise ValueError("negative text length")


def layer_cost(seq_len, cm: CostModel) -> float:
    """layer_cost (gflops.cpp:16-22): 8 S d^2 + 4 S^2 d + 4 S d f."""
    if seq_len < 1:
        raise ValueError("sequence length must be >= 1")
    s, d, f = float(seq_len), float(cm.d_model), float(cm.d_ff)
    return 8.0 * s * d * d + 4.0 * s * s * d + 4.0 * s * d * f


def pipeline_flops(v_hat, v0, cm: CostModel) -> dict:
    """pipeline_flops (gflops.cpp:24-51) -> GflopsReport as a dict."""
    cm.validate()
    if len(v_hat) == 0:
        raise ValueError("empty schedule")
    if v0 < 1:
        raise ValueError("v0 must be >= 1")
    for l, v in enumerate(v_hat):
        if v < 1 or v > v0:
            raise ValueError("executed visual length outside [1, v0]")
        if l > 0 and v > v_hat[l - 1]:
            raise ValueError("executed visual lengths must be non-increasing")
    layers, sp, sb = [], 0.0, 0.0
    for l, v in enumerate(v_hat):
        c = layer_cost(cm.text_len + int(v), cm)
        layers.append({"layer": l, "v_hat": int(v), "cost": c})
        sp += c
        sb += layer_cost(cm.text_len + v0, cm)
    f_vlm = cm.f_vt + cm.f_pj + sp
    f_base = cm.f_vt + cm.f_pj + sb
    return {"layers": layers, "f_vlm": f_vlm, "f_base": f_base, "ratio_pct": f_vlm / f_base * 100.0}


def executed_visual_lengths(recipe: PruningRecipe, n_layers) -> list:
    """executed_visual_lengths (gflops.cpp:53-72)."""
    recipe.validate()
    if n_layers < 1:
        raise ValueError("n_layers must be >= 1")
    if recipe.candidate_layers and recipe.candidate_layers[-1] >= n_layers:
        raise ValueError("recipe candidate layer beyond model depth")
    out, cur, nxt = [], recipe.v0, 0
    for l in range(n_layers):
        out.append(cur)
        if nxt < len(recipe.candidate_layers) and recipe.candidate_layers[nxt] == l:
            cur = min(cur, int(math.ceil(recipe.keep_ratios[nxt] * recipe.v0)))
            nxt += 1
    return out


# ---------------------------------------------------------------- harness
@dataclass
class CalibrationConfig:
    """CalibrationConfig (calibrator.hpp:94-104)."""
    seed: int = 1001
    samples: int = 16
    v0: int = 64
    eta: float = 1e-6
    window: int = 5
    p_min: float = 0.30
    tau: float = 0.25
    text_min: int = 8
    text_max: int = 32


@dataclass
class HarnessConfig:
    """HarnessConfig (harness.hpp:38-48) minus the model, which is the engine's."""
    calib: CalibrationConfig = field(default_factory=CalibrationConfig)
    weights: MetricWeights = field(default_factory=MetricWeights)
    weight_bits: int = 4
    act_bits: int = 4
    kv_bits: int = 4
    eval_seed: int = 2002
    eval_samples: int = 8
    gflops_text_len: int = 16
    f_vt: float = 0.0
    f_pj: float = 0.0
    model_seed: int = 0


@dataclass
class RunReport:
    """RunReport (harness.hpp:50-61)."""
    mode: str
    model_seed: int = 0
    recipe_digest: str = ""
    eval_digest: str = ""
    eval_count: int = 0
    sample_logits_digests: list = field(default_factory=list)
    divergence_mean: float = 0.0
    traces: list = field(default_factory=list)  # per sample: [(layer, budget, retained positions)]
    final_visual_count: int = 0
    gflops: dict = field(default_factory=dict)
    recipe: PruningRecipe | None = None
    last_logits: list = field(default_factory=list)  # per sample: the final-position logits (fp64)


def make_eval_samples(cfg: HarnessConfig, d_model: int):
    """make_eval_samples (harness.cpp:38-42)."""
    c = cfg.calib
    return make_calibration_samples(cfg.eval_seed, cfg.eval_samples, c.v0, d_model, c.text_min, c.text_max)


def _tuples(samples):
    return [s.as_tuple() if isinstance(s, Sample) else s for s in samples]


def _quantized_logits(engine, samples):
    """Quantized forward_prefill of every sample (batched up to the engine's capacity):
    logits (fp32 rows widened), traces, final visual counts."""
    L = lib()
    d = engine.cfg.d_model
    last, traces, finals = [], [], []
    i = 0
    while i < len(samples):
        chunk, tok = [], 0
        while i < len(samples) and len(chunk) < engine.max_batch:
            e, v, t = samples[i]
            if chunk and tok + v + t > engine.max_tokens:
                break
            chunk.append((e, v, t))
            tok += v + t
            i += 1
        emb = np.ascontiguousarray(np.concatenate([np.asarray(e, np.float64).reshape(-1, d) for e, _, _ in chunk]))
        vis = np.array([v for _, v, _ in chunk], dtype=np.int32)
        txt = np.array([t for _, _, t in chunk], dtype=np.int32)
        out = np.empty((tok, d), dtype=np.float32)
        ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))
        L.qt_engine_prefill_f64.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        from . import check
        check(L.qt_engine_prefill_f64(engine.h, len(chunk), emb.ctypes.data, 0, ip(vis), ip(txt), None, None,
                                      out.ctypes.data, 0))
        o = 0
        for b in range(len(chunk)):
            fv, ft, _ = engine.layout(b)
            last.append(out[o:o + fv + ft].astype(np.float64))
            traces.append(engine.trace(b))
            finals.append(fv)
            o += fv + ft
    return last, traces, finals


def run_pipeline(engine, cfg: HarnessConfig, mode: str, eval_samples, recipe_override: PruningRecipe | None = None,
                 calib_samples=None) -> RunReport:
    """run_pipeline (harness.cpp:59-179) on the device.  engine: a loaded Engine created
    with keep_fp_weights (the FP forwards) and act_mode 0 for the reference's static scales.
    calib_samples default to make_calibration_samples(cfg.calib ...)."""
    if not eval_samples:
        raise ValueError("no eval samples")
    if parse_mode(mode) is None:
        raise ValueError(f"unknown mode '{mode}'")
    ev = _tuples(eval_samples)
    d, n_layers = engine.cfg.d_model, engine.cfg.n_layers
    prunes, quantized = mode_prunes(mode), mode_quantizes(mode)
    c = cfg.calib
    calib = None

    def ensure_calib():
        nonlocal calib
        if calib is None:
            calib = _tuples(calib_samples) if calib_samples is not None else _tuples(
                make_calibration_samples(c.seed, c.samples, c.v0, d, c.text_min, c.text_max))
        return calib

    recipe, calib_out = None, None
    if prunes:
        if recipe_override is not None:
            recipe_override.validate()
            recipe = recipe_override
        else:  # run_quota_calibration (calibrator.cpp:251-268) on the device
            calib_out = engine.run_quota_calibration(ensure_calib(), window=c.window, p_min=c.p_min, tau=c.tau,
                                                     eta=c.eta)
            recipe = PruningRecipe([int(x) for x in calib_out["layers"]], [float(x) for x in calib_out["keeps"]],
                                   cfg.weights, c.v0, quant_digest(cfg.weight_bits, cfg.act_bits, cfg.kv_bits))
            recipe.validate()
        if recipe.candidate_layers[-1] >= n_layers:
            raise RuntimeError("recipe candidate layers do not fit the model")

    stage_wise = mode in ("prune_only", "quant_then_prune", "prune_then_quant")
    scoring = (recipe.weights.without_quant() if stage_wise else recipe.weights) if prunes else None

    if quantized:
        if mode == "prune_then_quant":  # scales fit on the recipe-pruned FP graph
            engine.set_recipe(recipe.candidate_layers, recipe.keep_ratios, scoring.as_tuple(), recipe.v0, -1)
            scales = engine.fit_act_scales(ensure_calib(), apply=False, hooked=True)
        elif calib_out is not None:
            scales = calib_out["act_scales"]
        else:
            scales = engine.fit_act_scales(ensure_calib(), apply=False)
        engine.set_act_scales(scales)

    if prunes:
        engine.set_recipe(recipe.candidate_layers, recipe.keep_ratios, scoring.as_tuple(), recipe.v0,
                          cfg.act_bits if quantized else -1)
    else:
        engine.clear_recipe()

    rep = RunReport(mode=mode, model_seed=cfg.model_seed, recipe_digest=recipe.digest() if recipe else "",
                    eval_digest=sample_set_digest(ev), eval_count=len(ev), recipe=recipe)
    # full-precision reference forwards (harness.cpp:135-136), sequence by sequence
    fp_last = []
    bsz = max(1, engine.max_batch)
    for i in range(0, len(ev), bsz):
        for lg in engine.prefill_fp(ev[i:i + bsz], hook=False):
            fp_last.append(lg[-1])
    if quantized:
        run_logits, traces, finals = _quantized_logits(engine, ev)
    else:
        run_logits, traces, finals = [], [], []
        for i in range(0, len(ev), bsz):
            lgs = engine.prefill_fp(ev[i:i + bsz], hook=prunes)
            for b, lg in enumerate(lgs):
                run_logits.append(lg)
                traces.append(engine.trace(b))
                finals.append(engine.layout(b)[0])
    # divergence of the final-position logits (harness.cpp:148-155)
    div = 0.0
    for a, b in zip(run_logits, fp_last):
        div += math.sqrt(float(np.sum((a[-1] - b) ** 2)))
    rep.divergence_mean = div / len(ev)
    rep.last_logits = [np.asarray(x[-1], np.float64) for x in run_logits]
    # harness.cpp:144; quantized rows are the device's fp32 logits widened to fp64
    rep.sample_logits_digests = [hex_digest(x) for x in run_logits]
    rep.traces = [[(int(l), int(bu), [int(p) for p in ps]) for l, bu, ps in tr] for tr in traces]
    if len(set(finals)) > 1:
        raise RuntimeError("inconsistent final visual count across samples")  # harness.cpp:157-160
    rep.final_visual_count = finals[0]
    # cost (harness.cpp:165-177)
    cm = CostModel(cfg.f_vt, cfg.f_pj, d, engine.cfg.d_ff, engine.cfg.n_heads, cfg.gflops_text_len)
    v_hat = executed_visual_lengths(recipe, n_layers) if prunes else [c.v0] * n_layers
    rep.gflops = pipeline_flops(v_hat, recipe.v0 if prunes else c.v0, cm)
    return rep


def compare_reports(reports):
    """compare_reports (harness.cpp:180-196): rows (mode, divergence_mean, final_visual_count,
    gflops ratio_pct) sorted by mode name; every report must cover the same eval set."""
    if len(reports) < 2:
        raise ValueError("need at least two reports to compare")
    for r in reports:
        if r.eval_digest != reports[0].eval_digest or r.eval_count != reports[0].eval_count:
            raise RuntimeError("reports cover different eval sample sets")
    rows = [{"mode": r.mode, "divergence_mean": r.divergence_mean, "final_visual_count": r.final_visual_count,
             "gflops_ratio_pct": r.gflops["ratio_pct"]} for r in reports]
    return sorted(rows, key=lambda x: x["mode"])


def report_to_json(r: RunReport) -> dict:
    """report_to_json (harness.cpp:224-247)."""
    return {
        "meta": {"tool_version": TOOL_VERSION, "seed": r.model_seed, "recipe_digest": r.recipe_digest},
        "mode": r.mode,
        "eval": {"digest": r.eval_digest, "count": r.eval_count},
        "divergence_mean": r.divergence_mean,
        "final_visual_count": r.final_visual_count,
        "sample_logits_digests": r.sample_logits_digests,
        "traces": [[{"layer": l, "budget": b, "retained_indices": p} for l, b, p in tr] for tr in r.traces],
        "gflops": r.gflops,
    }


def render_comparison_text(rows) -> str:
    """render_comparison_text (harness.cpp:285-306): JSON scalar cells, columns padded to the
    widest cell + 2 spaces, one line per row."""
    cells = [["mode", "divergence_mean", "final_visual_count", "gflops_ratio_pct"]]
    for r in rows:
        cells.append([r["mode"], _num(float(r["divergence_mean"])), _num(int(r["final_visual_count"])),
                      _num(float(r["gflops_ratio_pct"]))])
    width = [max(len(row[c]) for row in cells) for c in range(4)]
    out = []
    for row in cells:
        out.append("".join(row[c] + (" " * (width[c] - len(row[c]) + 2) if c + 1 < 4 else "") for c in range(4)))
    return "".join(line + "\n" for line in out)
