"""oracle -- CPU checkers for the QUOTA hot path (TEST INFRASTRUCTURE ONLY).

Two checkers, both plain fp64 C++ behind ctypes:

* ``Ref``    -- oracle/_ref/libquota_ref.so: the UNMODIFIED reference library
  (/root/reference/proj/src/*.cpp compiled where it lies by oracle/Makefile)
  plus the marshalling shim oracle/ref_capi.cpp.  This is R0.
* ``Port``   -- oracle/_build/libquota_oracle.so: the restatement
  oracle/quota_oracle.cpp (R1) with the north_star switches (per-token
  activation scales, per-output-channel weights, SwiGLU, GQA).  Pinned to R0
  bit-for-bit by tests/test_oracle_cpu.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package.  The product
(paper_2604_17320_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libquota_ref.so")
PORT_SO = os.path.join(HERE, "_build", "libquota_oracle.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i8p = C.POINTER(C.c_int8)


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def _b(a):
    return a.ctypes.data_as(_i8p)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    pass


_ref_lib = None
_port_lib = None


def ref_lib():
    global _ref_lib
    if _ref_lib is None:
        if not os.path.exists(REF_SO):
            raise OracleError(f"{REF_SO} missing: run `make -C oracle ref`")
        lib = C.CDLL(REF_SO)
        lib.qref_last_error.restype = C.c_char_p
        lib.qref_round_half_even.restype = C.c_double
        lib.qref_round_half_even.argtypes = [C.c_double]
        lib.qref_silu.restype = C.c_double
        lib.qref_model_create.restype = C.c_void_p
        lib.qref_model_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64]
        lib.qref_model_free.argtypes = [C.c_void_p]
        lib.qref_model_weight_checksum.restype = C.c_uint64
        lib.qref_model_weight_checksum.argtypes = [C.c_void_p]
        lib.qref_model_get_weight.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_int64]
        lib.qref_model_set_weight.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_int64]
        lib.qref_model_prepare_quant.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        lib.qref_model_weight_codes.argtypes = [C.c_void_p, C.c_int, C.c_int, _i8p, _dp]
        lib.qref_fit_act_scales.argtypes = [C.c_void_p, C.c_int, C.POINTER(_dp), _ip, _ip, C.c_int, _dp]
        lib.qref_fit_act_scales_hooked.argtypes = [C.c_void_p, C.c_int, C.POINTER(_dp), _ip, _ip, C.c_int,
                                                   C.c_char_p, _dp, _dp]
        lib.qref_make_samples.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _ip, _dp,
                                          C.c_int64, C.c_char_p]
        lib.qref_pipeline_flops.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_double, C.c_double, _dp, _dp]
        lib.qref_prefill.restype = C.c_void_p
        lib.qref_prefill.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int, C.c_int, _ip, C.c_char_p, _dp, C.c_int]
        for n in ("qref_run_free", "qref_run_logits_rows", "qref_run_n_prunes"):
            getattr(lib, n).argtypes = [C.c_void_p]
        lib.qref_run_logits.argtypes = [C.c_void_p, _dp]
        lib.qref_run_layout.argtypes = [C.c_void_p, _ip, _ip, _ip, C.c_int]
        lib.qref_run_prune.argtypes = [C.c_void_p, C.c_int, _ip, _ip, _ip, C.c_int, _ip]
        lib.qref_run_block_output.argtypes = [C.c_void_p, C.c_int, _dp, _ip]
        lib.qref_run_kv.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _i8p, _dp, _ip, _ip]
        lib.qref_decode.argtypes = [C.c_void_p, _dp, _dp]
        lib.qref_fnv1a64.restype = C.c_uint64
        lib.qref_fnv1a64.argtypes = [_dp, C.c_int64]
        lib.qref_layer_cost.restype = C.c_double
        lib.qref_layer_cost.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
        lib.qref_percentile.argtypes = [_dp, C.c_int, C.c_double, _dp]
        lib.qref_prefill_threads.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64, _dp]
        lib.qref_quantize_fit.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _i8p]
        lib.qref_quantize_with.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp, C.c_int, _i8p, _dp]
        lib.qref_fake_quant_per_row.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp]
        lib.qref_kv_quantize.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _i8p, _dp]
        lib.qref_quantized_linear.argtypes = [_dp, C.c_int, C.c_int, _i8p, _dp, C.c_int, C.c_int, C.c_int, _dp]
        lib.qref_matmul.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, _dp]
        lib.qref_rms_norm_rows.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp]
        lib.qref_rope.argtypes = [_dp, C.c_int, C.c_int]
        lib.qref_silu.argtypes = [C.c_double]
        lib.qref_compute_budget.argtypes = [C.c_double, C.c_int, _ip]
        lib.qref_robust_normalize.argtypes = [_dp, C.c_int, _dp]
        lib.qref_select_top_k.argtypes = [_dp, C.c_int, C.c_int, _ip, _ip]
        lib.qref_score_tokens.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, C.c_int, _dp,
                                          _dp, _dp]
        lib.qref_parse_recipe.argtypes = [C.c_char_p, C.c_int, _ip, _ip, _dp, _dp, _ip, C.c_char_p, C.c_int]
        lib.qref_serialize_recipe.argtypes = [C.c_int, _ip, _dp, _dp, C.c_int, C.c_char_p, C.c_char_p, C.c_int,
                                              C.c_char_p]
        lib.qref_executed_visual_lengths.argtypes = [C.c_char_p, C.c_int, _ip]
        lib.qref_run_calibration.argtypes = [C.c_void_p, C.c_int, C.POINTER(_dp), _ip, _ip, C.c_int, C.c_double,
                                             C.c_double, C.c_double, _dp, _ip, _dp, _dp, _dp, _dp, _dp]
        lib.qref_profile_sensitivity.argtypes = [C.c_void_p, C.c_int, C.POINTER(_dp), _ip, _ip, C.c_int, _ip,
                                                 C.c_double, _dp, _dp]
        lib.qref_compute_metrics.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, C.c_int, _dp, _dp, C.c_int, _dp]
        _ref_lib = lib
    return _ref_lib


# ---------------------------------------------------------------- R0 primitives (kernel-level checkers)


def ref_make_samples(seed, count, v0, d_model, text_min, text_max):
    """make_calibration_samples + sample_set_digest (calibrator.cpp:12-40) of the reference:
    ([(emb fp64, v0, text)], digest)."""
    lib = ref_lib()
    txt = np.empty(count, dtype=np.int32)
    cap = count * (v0 + text_max) * d_model
    emb = np.empty(cap, dtype=np.float64)
    dg = C.create_string_buffer(17)
    _check(lib.qref_make_samples(seed, count, v0, d_model, text_min, text_max, _i(txt), _d(emb), cap, dg), lib,
           "qref")
    out, o = [], 0
    for t in txt:
        n = (v0 + int(t)) * d_model
        out.append((emb[o:o + n].reshape(v0 + int(t), d_model).copy(), v0, int(t)))
        o += n
    return out, dg.value.decode()


def ref_pipeline_flops(recipe_json, n_layers, v0, d_model, d_ff, n_heads, text_len, f_vt=0.0, f_pj=0.0):
    """pipeline_flops (gflops.cpp:24-51) of the recipe's executed lengths (None: all at v0)."""
    lib = ref_lib()
    costs, o3 = np.empty(n_layers), np.empty(3)
    rj = recipe_json.encode() if recipe_json is not None else None
    _check(lib.qref_pipeline_flops(rj, n_layers, v0, d_model, d_ff, n_heads, text_len, f_vt, f_pj, _d(costs),
                                   _d(o3)), lib, "qref")
    return costs, float(o3[0]), float(o3[1]), float(o3[2])


def ref_compute_budget(keep_ratio, v0):
    """compute_budget (selector.cpp:11-17)."""
    lib = ref_lib()
    out = C.c_int()
    _check(lib.qref_compute_budget(keep_ratio, v0, C.byref(out)), lib, "qref")
    return out.value


def ref_percentile(v, p):
    """percentile (numeric.cpp:84-96)."""
    lib = ref_lib()
    a = f64(v)
    out = C.c_double()
    _check(lib.qref_percentile(_d(a), a.size, p, C.byref(out)), lib, "qref")
    return out.value


def ref_robust_normalize(v):
    """robust_normalize (selector.cpp:70-84)."""
    lib = ref_lib()
    a = f64(v)
    out = np.empty_like(a)
    _check(lib.qref_robust_normalize(_d(a), a.size, _d(out)), lib, "qref")
    return out


def ref_select_top_k(scores, k):
    """select_top_k (selector.cpp:117-136): ascending retained slots."""
    lib = ref_lib()
    a = f64(scores)
    out = np.empty(max(1, min(k, a.size)), dtype=np.int32)
    n = C.c_int()
    _check(lib.qref_select_top_k(_d(a), a.size, k, _i(out), C.byref(n)), lib, "qref")
    return out[:n.value].copy()


def ref_score_tokens(visual, inter, intra, weights=(0.25, 0.45, 0.10, 0.20), res_bits=4):
    """compute_metrics + score_tokens (selector.cpp:19-115).  visual [n x d], inter [H x T x n],
    intra [H x n x n].  Returns (metrics [4 x n], normalised [4 x n], fused [n])."""
    lib = ref_lib()
    vis, it, ia, w = f64(visual), f64(inter), f64(intra), f64(weights)
    n, d = vis.shape
    H, T = it.shape[0], it.shape[1]
    m = np.empty((4, n))
    nn = np.empty((4, n))
    f = np.empty(n)
    _check(lib.qref_score_tokens(_d(vis), n, d, H, T, _d(it), _d(ia), _d(w), res_bits, _d(m), _d(nn), _d(f)),
           lib, "qref")
    return m, nn, f


def ref_parse_recipe(text, max_layers=256):
    """parse_recipe (recipe.cpp:91-116) -> dict; raises OracleError with the reference message."""
    lib = ref_lib()
    n = C.c_int()
    lay = np.empty(max_layers, dtype=np.int32)
    kp = np.empty(max_layers)
    w = np.empty(4)
    v0 = C.c_int()
    dg = C.create_string_buffer(256)
    _check(lib.qref_parse_recipe(text.encode() if isinstance(text, str) else text, max_layers, C.byref(n), _i(lay),
                                 _d(kp), _d(w), C.byref(v0), dg, 256), lib, "qref")
    k = n.value
    return dict(candidate_layers=lay[:k].tolist(), keep_ratios=kp[:k].tolist(), weights=tuple(w.tolist()),
                v0=v0.value, quant_digest=dg.value.decode())


def ref_quantize_fit(x, axis, bits=4):
    """fit_params + quantize (quant.cpp:47-91); axis 0/1/2 = PerTensor/PerRow/PerColumn."""
    lib = ref_lib()
    a = f64(x)
    rows, cols = a.shape
    sc = np.empty({0: 1, 1: rows, 2: cols}[axis])
    codes = np.empty(a.size, dtype=np.int8)
    _check(lib.qref_quantize_fit(_d(a), rows, cols, bits, axis, _d(sc), _b(codes)), lib, "qref")
    return codes.reshape(a.shape), sc


def ref_kv_quantize(x, bits=4):
    """kv_quantize (quant.cpp:117-119): per-row symmetric codes + scales."""
    lib = ref_lib()
    a = f64(x)
    rows, cols = a.shape
    codes = np.empty(a.size, dtype=np.int8)
    sc = np.empty(rows)
    _check(lib.qref_kv_quantize(_d(a), rows, cols, bits, _b(codes), _d(sc)), lib, "qref")
    return codes.reshape(a.shape), sc


def ref_rope(v, position):
    """rope_in_place (model.cpp:156-168) of one head vector (fp64), returned as a copy."""
    lib = ref_lib()
    a = f64(v).copy()
    _check(lib.qref_rope(_d(a), a.size, int(position)), lib, "qref")
    return a


def ref_fake_quant_per_row(x, bits=4):
    lib = ref_lib()
    a = f64(x)
    out = np.empty_like(a)
    _check(lib.qref_fake_quant_per_row(_d(a), a.shape[0], a.shape[1], bits, _d(out)), lib, "qref")
    return out


def ref_compute_metrics(visual_states, text_states, inter_blocks, intra_blocks, res_bits=4):
    """compute_metrics (selector.cpp:19-68) of the unmodified reference on a
    LayerActivationRecord: inter_blocks [H x T x N], intra_blocks [H x N x N] post-softmax
    probabilities.  res_bits None = nullopt.  Returns [4 x N] (mag, inter, intra, res)."""
    lib = ref_lib()
    vs, ts = f64(visual_states), f64(text_states)
    ib, ab = f64(inter_blocks), f64(intra_blocks)
    n, d = vs.shape
    out = np.empty((4, n))
    _check(lib.qref_compute_metrics(_d(vs), n, d, _d(ts), ts.shape[0], ib.shape[0], _d(ib), _d(ab),
                                    -1 if res_bits is None else int(res_bits), _d(out)), lib, "qref")
    return out


def port_masked_attention(q, k_codes, k_scales, v_codes, v_scales, pos, visual, H, Hkv, dh, want_probs=False):
    """The restatement's masked prefill attention (model.cpp:272-292,366-391) on given int4
    K/V rows: q fp64 [S x H*dh] post-RoPE, codes int8 [S x Hkv*dh], scales [S x Hkv].
    Returns out [S x H*dh] (and probs [H x S x S])."""
    lib = port_lib()
    qa = f64(q)
    S = qa.shape[0]
    kc, vc = (np.ascontiguousarray(a, dtype=np.int8) for a in (k_codes, v_codes))
    ks, vs = f64(k_scales), f64(v_scales)
    p = np.ascontiguousarray(pos, dtype=np.int32)
    out = np.empty((S, H * dh))
    probs = np.empty((H, S, S)) if want_probs else None
    _check(lib.qo_masked_attention(_d(qa), _b(kc), _d(ks), _b(vc), _d(vs), _i(p), S, visual, H, Hkv, dh, _d(out),
                                   _d(probs) if want_probs else None), lib, "qo")
    return (out, probs) if want_probs else out


def port_decode_attention(q, k_codes, k_scales, v_codes, v_scales, H, Hkv, dh):
    """The restatement's decode attention (model.cpp:515-535): q fp64 [H*dh]; codes int8
    [rows x Hkv*dh]; scales [rows x Hkv] -> out [H*dh]."""
    lib = port_lib()
    qa = f64(q).ravel()
    kc, vc = (np.ascontiguousarray(a, dtype=np.int8) for a in (k_codes, v_codes))
    ks, vs = f64(k_scales), f64(v_scales)
    out = np.empty(H * dh)
    _check(lib.qo_decode_attention(_d(qa), _b(kc), _d(ks), _b(vc), _d(vs), kc.shape[0], H, Hkv, dh, _d(out)), lib,
           "qo")
    return out


def port_lib():
    global _port_lib
    if _port_lib is None:
        if not os.path.exists(PORT_SO):
            raise OracleError(f"{PORT_SO} missing: run `make -C oracle port`")
        lib = C.CDLL(PORT_SO)
        lib.qo_last_error.restype = C.c_char_p
        lib.qo_model_create.restype = C.c_void_p
        lib.qo_model_create.argtypes = [_ip]
        lib.qo_model_free.argtypes = [C.c_void_p]
        lib.qo_model_set_weight.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_int64]
        lib.qo_model_prepare.argtypes = [C.c_void_p, _dp]
        lib.qo_model_weight_codes.argtypes = [C.c_void_p, C.c_int, C.c_int, _i8p, _dp]
        lib.qo_prefill.restype = C.c_void_p
        lib.qo_prefill.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int, C.c_int, _ip, C.c_int, _ip, _dp, _dp,
                                   C.c_int, C.c_int]
        for n in ("qo_run_free", "qo_run_logits_rows", "qo_run_n_prunes"):
            getattr(lib, n).argtypes = [C.c_void_p]
        lib.qo_run_logits.argtypes = [C.c_void_p, _dp]
        lib.qo_run_layout.argtypes = [C.c_void_p, _ip, _ip, _ip]
        lib.qo_run_prune.argtypes = [C.c_void_p, C.c_int, _ip, _ip, _ip, _ip]
        lib.qo_run_last_scores.argtypes = [C.c_void_p, _dp, _dp, _ip]
        lib.qo_run_block_output.argtypes = [C.c_void_p, C.c_int, _dp, _ip]
        lib.qo_run_kv.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _i8p, _dp, _ip, _ip]
        lib.qo_decode.argtypes = [C.c_void_p, _dp, _dp]
        lib.qo_run_tie_margin.restype = C.c_double
        lib.qo_run_tie_margin.argtypes = [C.c_void_p, C.c_int]
        lib.qo_run_batch.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(_dp), _ip, _ip, C.c_int, _ip, _dp,
                                     _dp, _ip, C.c_int, C.c_int, C.POINTER(_dp), C.c_int, _dp]
        lib.qo_masked_attention.argtypes = [_dp, _i8p, _dp, _i8p, _dp, _ip, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_int, _dp, _dp]
        lib.qo_decode_attention.argtypes = [_dp, _i8p, _dp, _i8p, _dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        lib.qo_set_threads.argtypes = [C.c_int]
        lib.qo_set_threads.restype = None
        u64p = C.POINTER(C.c_uint64)
        lib.qo_prefill_ex.restype = C.c_void_p
        lib.qo_prefill_ex.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int, C.c_int, _ip, C.c_int, _ip, _dp, _dp,
                                      C.c_int, C.c_int, C.c_int, C.c_int, u64p, _i8p]
        lib.qo_run_n_recs.argtypes = [C.c_void_p]
        lib.qo_run_rec.argtypes = [C.c_void_p, C.c_int, _ip, _i8p, _dp]
        lib.qo_run_clear_recs.argtypes = [C.c_void_p]
        lib.qo_run_clear_recs.restype = None
        lib.qo_run_n_applied.argtypes = [C.c_void_p]
        lib.qo_run_applied.argtypes = [C.c_void_p, u64p, _i8p, _dp]
        lib.qo_run_n_ties.argtypes = [C.c_void_p]
        lib.qo_run_ties.argtypes = [C.c_void_p, u64p, _i8p, _dp]
        _port_lib = lib
    return _port_lib


def _check(rc, lib, prefix):
    if rc != 0:
        msg = getattr(lib, prefix + "_last_error")().decode()
        raise OracleError(msg)


# ---------------------------------------------------------------- configs


@dataclass
class ModelCfg:
    """Shape + semantic switches.  Defaults = reference R0."""

    n_layers: int = 4
    d_model: int = 256
    n_heads: int = 4
    n_kv_heads: int = 4
    d_head: int = 64
    d_ff: int = 1024
    mlp: int = 0          # 0 SiLU (reference), 1 SwiGLU
    act_mode: int = 0     # 0 static per-tensor (reference), 1 dynamic per-token
    weight_axis: int = 2  # 1 PerRow (reference prepare_quant_env), 2 PerColumn
    act_bits: int = 4
    weight_bits: int = 4
    kv_bits: int = 4

    def as_array(self):
        return np.array([self.n_layers, self.d_model, self.n_heads, self.n_kv_heads, self.d_head, self.d_ff,
                         self.mlp, self.act_mode, self.weight_axis, self.act_bits, self.weight_bits,
                         self.kv_bits], dtype=np.int32)

    def is_reference_expressible(self):
        return (self.mlp == 0 and self.n_kv_heads == self.n_heads and self.d_ff == 4 * self.d_model
                and self.act_mode == 0)


@dataclass
class Recipe:
    candidate_layers: list
    keep_ratios: list
    weights: tuple = (0.25, 0.45, 0.10, 0.20)  # recipe.hpp:10-14
    v0: int = 144
    quant_digest: str = "w4a4kv4-sym-rne"

    def to_json(self):
        import json
        return json.dumps({"schema_version": 1, "candidate_layers": list(self.candidate_layers),
                           "keep_ratios": list(self.keep_ratios),
                           "metric_weights": {"mag": self.weights[0], "inter": self.weights[1],
                                              "intra": self.weights[2], "quant": self.weights[3]},
                           "v0": self.v0, "quant_digest": self.quant_digest})


@dataclass
class Weights:
    """fp64 weights, reference orientation W[d_in x d_out] (y = x W)."""

    layers: list = field(default_factory=list)  # dict(wq, wk, wv, wo, w1, w2, w3?, g1, g2)
    head: np.ndarray = None
    gf: np.ndarray = None


@dataclass
class RunResult:
    logits: np.ndarray
    visual: int
    text: int
    positions: np.ndarray
    trace: list  # [(layer, budget, positions ndarray)]


# ---------------------------------------------------------------- R0 (reference)


class Ref:
    """The unmodified reference (R0) through oracle/_ref/libquota_ref.so."""

    def __init__(self, cfg: ModelCfg, seed: int = 1):
        assert cfg.mlp == 0 and cfg.n_kv_heads == cfg.n_heads and cfg.d_ff == 4 * cfg.d_model
        self.lib = ref_lib()
        self.cfg = cfg
        self.h = self.lib.qref_model_create(cfg.n_layers, cfg.n_heads, cfg.d_model, cfg.d_head, seed)
        if not self.h:
            raise OracleError(self.lib.qref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.qref_model_free(self.h)
            self.h = None

    def get(self, layer, which, shape):
        out = np.empty(int(np.prod(shape)), dtype=np.float64)
        _check(self.lib.qref_model_get_weight(self.h, layer, which, _d(out), out.size), self.lib, "qref")
        return out.reshape(shape)

    def weights(self) -> Weights:
        c = self.cfg
        d, f = c.d_model, c.d_ff
        w = Weights()
        for l in range(c.n_layers):
            w.layers.append(dict(wq=self.get(l, 0, (d, d)), wk=self.get(l, 1, (d, d)), wv=self.get(l, 2, (d, d)),
                                 wo=self.get(l, 3, (d, d)), w1=self.get(l, 4, (d, f)), w2=self.get(l, 5, (f, d)),
                                 g1=self.get(l, 6, (d,)), g2=self.get(l, 7, (d,))))
        w.head = self.get(-1, 0, (d, d))
        w.gf = self.get(-1, 6, (d,))
        return w

    def set_weights(self, w: Weights):
        names = ["wq", "wk", "wv", "wo", "w1", "w2", "g1", "g2"]
        for l, lw in enumerate(w.layers):
            for i, n in enumerate(names):
                a = f64(lw[n]).ravel()
                _check(self.lib.qref_model_set_weight(self.h, l, i, _d(a), a.size), self.lib, "qref")
        a = f64(w.head).ravel()
        _check(self.lib.qref_model_set_weight(self.h, -1, 0, _d(a), a.size), self.lib, "qref")
        a = f64(w.gf).ravel()
        _check(self.lib.qref_model_set_weight(self.h, -1, 6, _d(a), a.size), self.lib, "qref")

    def checksum(self):
        return self.lib.qref_model_weight_checksum(self.h)

    def fit_act_scales(self, samples, recipe: "Recipe | None" = None, weights=None):
        """fit_act_scales (calibrator.cpp:237-249); samples = [(emb, visual, text)].  With a
        recipe: under make_recipe_hook(recipe, weights or recipe.weights, nullopt)."""
        embs = [f64(e) for e, _, _ in samples]
        arr = (_dp * len(embs))(*[_d(e) for e in embs])
        vis = np.array([v for _, v, _ in samples], dtype=np.int32)
        txt = np.array([t for _, _, t in samples], dtype=np.int32)
        out = np.empty(4 * self.cfg.n_layers + 1, dtype=np.float64)
        if recipe is None:
            _check(self.lib.qref_fit_act_scales(self.h, len(embs), arr, _i(vis), _i(txt), self.cfg.act_bits,
                                                _d(out)), self.lib, "qref")
        else:
            w = None if weights is None else f64(weights)
            _check(self.lib.qref_fit_act_scales_hooked(self.h, len(embs), arr, _i(vis), _i(txt), self.cfg.act_bits,
                                                       recipe.to_json().encode(), _d(w) if w is not None else None,
                                                       _d(out)), self.lib, "qref")
        return out

    def profile_sensitivity(self, samples, layers, eta=1e-6):
        """profile_sensitivity (calibrator.cpp:42-82) with the prepared env -> (raw, normalized)."""
        embs = [f64(e) for e, _, _ in samples]
        arr = (_dp * len(embs))(*[_d(e) for e in embs])
        vis = np.array([v for _, v, _ in samples], dtype=np.int32)
        txt = np.array([t for _, _, t in samples], dtype=np.int32)
        lay = np.array(layers, dtype=np.int32)
        raw = np.empty(len(lay))
        nrm = np.empty(len(lay))
        _check(self.lib.qref_profile_sensitivity(self.h, len(embs), arr, _i(vis), _i(txt), len(lay), _i(lay), eta,
                                                 _d(raw), _d(nrm)), self.lib, "qref")
        return raw, nrm

    def run_calibration(self, samples, window=5, p_min=0.3, tau=0.25, eta=1e-6):
        """run_quota_calibration (calibrator.cpp:251-268) on explicit samples with the per-column env."""
        embs = [f64(e) for e, _, _ in samples]
        arr = (_dp * len(embs))(*[_d(e) for e in embs])
        vis = np.array([v for _, v, _ in samples], dtype=np.int32)
        txt = np.array([t for _, _, t in samples], dtype=np.int32)
        L = self.cfg.n_layers
        acts, lay, kp = np.empty(4 * L + 1), np.empty(window, dtype=np.int32), np.empty(window)
        raw, nrm, cm, rm = np.empty(window), np.empty(window), np.empty(L), np.empty(L)
        _check(self.lib.qref_run_calibration(self.h, len(embs), arr, _i(vis), _i(txt), window, p_min, tau, eta,
                                             _d(acts), _i(lay), _d(kp), _d(raw), _d(nrm), _d(cm), _d(rm)),
               self.lib, "qref")
        return dict(act_scales=acts, layers=lay, keeps=kp, raw=raw, normalized=nrm, conc=cm, red=rm)

    def prepare(self, act_scales, weight_axis=None):
        c = self.cfg
        a = f64(act_scales)
        ax = c.weight_axis if weight_axis is None else weight_axis
        _check(self.lib.qref_model_prepare_quant(self.h, c.weight_bits, c.act_bits, c.kv_bits, ax, _d(a)),
               self.lib, "qref")

    def weight_codes(self, layer, which, shape, n_scales):
        codes = np.empty(int(np.prod(shape)), dtype=np.int8)
        scales = np.empty(n_scales, dtype=np.float64)
        _check(self.lib.qref_model_weight_codes(self.h, layer, which, _b(codes), _d(scales)), self.lib, "qref")
        return codes.reshape(shape), scales

    def prefill_threads(self, n_threads, visual, text, seed=1):
        """Reference forward_prefill on n_threads independent synthetic sequences, one per
        std::thread; returns wall seconds (CPU baseline)."""
        sec = np.zeros(1)
        _check(self.lib.qref_prefill_threads(self.h, n_threads, visual, text, seed, _d(sec)), self.lib, "qref")
        return float(sec[0])

    def prefill(self, emb, visual, text, recipe: Recipe | None = None, quantized=True, res_bits=4, pos=None,
                weights=None):
        """forward_prefill; weights (4 fp64, optional): the hook's MetricWeights instead of the recipe's."""
        e = f64(emb)
        p = None if pos is None else np.ascontiguousarray(pos, dtype=np.int32)
        rj = recipe.to_json().encode() if recipe is not None else None
        w = None if weights is None else f64(weights)
        r = self.lib.qref_prefill(self.h, int(quantized), _d(e), visual, text, _i(p) if p is not None else None,
                                  rj, _d(w) if w is not None else None, res_bits)
        if not r:
            raise OracleError(self.lib.qref_last_error().decode())
        return RefRun(self, r)


class RefRun:
    def __init__(self, owner, handle):
        self.o = owner
        self.lib = owner.lib
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.qref_run_free(self.h)
            self.h = None

    def result(self) -> RunResult:
        rows = self.lib.qref_run_logits_rows(self.h)
        lg = np.empty((rows, self.o.cfg.d_model), dtype=np.float64)
        self.lib.qref_run_logits(self.h, _d(lg))
        v, t = C.c_int(), C.c_int()
        pos = np.empty(rows + 4096, dtype=np.int32)
        _check(self.lib.qref_run_layout(self.h, C.byref(v), C.byref(t), _i(pos), pos.size), self.lib, "qref")
        trace = []
        for i in range(self.lib.qref_run_n_prunes(self.h)):
            lay, bud, cnt = C.c_int(), C.c_int(), C.c_int()
            ps = np.empty(1 << 16, dtype=np.int32)
            _check(self.lib.qref_run_prune(self.h, i, C.byref(lay), C.byref(bud), _i(ps), ps.size, C.byref(cnt)),
                   self.lib, "qref")
            trace.append((lay.value, bud.value, ps[:cnt.value].copy()))
        return RunResult(lg, v.value, t.value, pos[:v.value + t.value].copy(), trace)

    def kv(self, layer, head, which):
        rows = C.c_int()
        _check(self.lib.qref_run_kv(self.h, layer, head, which, None, None, None, C.byref(rows)), self.lib, "qref")
        dh = self.o.cfg.d_head
        codes = np.empty((rows.value, dh), dtype=np.int8)
        scales = np.empty(rows.value, dtype=np.float64)
        pos = np.empty(rows.value, dtype=np.int32)
        _check(self.lib.qref_run_kv(self.h, layer, head, which, _b(codes), _d(scales), _i(pos), C.byref(rows)),
               self.lib, "qref")
        return codes, scales, pos

    def block_output(self, layer):
        rows = C.c_int()
        _check(self.lib.qref_run_block_output(self.h, layer, None, C.byref(rows)), self.lib, "qref")
        out = np.empty((rows.value, self.o.cfg.d_model), dtype=np.float64)
        _check(self.lib.qref_run_block_output(self.h, layer, _d(out), C.byref(rows)), self.lib, "qref")
        return out

    def decode(self, emb):
        e = f64(emb)
        out = np.empty(self.o.cfg.d_model, dtype=np.float64)
        _check(self.lib.qref_decode(self.h, _d(e), _d(out)), self.lib, "qref")
        return out


# ---------------------------------------------------------------- R1 (restatement)


class Port:
    """The restatement (R1) through oracle/_build/libquota_oracle.so."""

    def __init__(self, cfg: ModelCfg):
        self.lib = port_lib()
        self.cfg = cfg
        a = cfg.as_array()
        self.h = self.lib.qo_model_create(_i(a))
        if not self.h:
            raise OracleError(self.lib.qo_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.qo_model_free(self.h)
            self.h = None

    def set_weights(self, w: Weights):
        names = {"wq": 0, "wk": 1, "wv": 2, "wo": 3, "w1": 4, "w2": 5, "g1": 6, "g2": 7, "w3": 8}
        for l, lw in enumerate(w.layers):
            for n, i in names.items():
                if n not in lw:
                    continue
                a = f64(lw[n]).ravel()
                _check(self.lib.qo_model_set_weight(self.h, l, i, _d(a), a.size), self.lib, "qo")
        a = f64(w.head).ravel()
        _check(self.lib.qo_model_set_weight(self.h, -1, 0, _d(a), a.size), self.lib, "qo")
        a = f64(w.gf).ravel()
        _check(self.lib.qo_model_set_weight(self.h, -1, 6, _d(a), a.size), self.lib, "qo")

    def prepare(self, act_scales=None):
        a = None if act_scales is None else f64(act_scales)
        _check(self.lib.qo_model_prepare(self.h, _d(a) if a is not None else None), self.lib, "qo")

    def weight_codes(self, layer, which, shape, n_scales):
        codes = np.empty(int(np.prod(shape)), dtype=np.int8)
        scales = np.empty(n_scales, dtype=np.float64)
        _check(self.lib.qo_model_weight_codes(self.h, layer, which, _b(codes), _d(scales)), self.lib, "qo")
        return codes.reshape(shape), scales

    @staticmethod
    def set_threads(n):
        """Worker threads of the row-parallel matmul / attention loops (results are
        bit-identical for any count)."""
        port_lib().qo_set_threads(int(n))

    def prefill(self, emb, visual, text, recipe: Recipe | None = None, quantized=True, res_bits=4, pos=None,
                v0=None, record=False, overrides=None):
        """record: keep every quantizer site's codes (PortRun.records); overrides: {decision
        key: code} the run follows instead of its own rounding (forced replay, tests/replay.py)."""
        e = f64(emb)
        p = None if pos is None else np.ascontiguousarray(pos, dtype=np.int32)
        ok = np.zeros(0, dtype=np.uint64) if not overrides else np.fromiter(overrides.keys(), dtype=np.uint64)
        oc = np.zeros(0, dtype=np.int8) if not overrides else np.fromiter(overrides.values(), dtype=np.int8)
        okp = ok.ctypes.data_as(C.POINTER(C.c_uint64))
        if recipe is not None:
            lay = np.array(recipe.candidate_layers, dtype=np.int32)
            kp = f64(recipe.keep_ratios)
            wt = f64(recipe.weights)
            n = len(lay)
            r = self.lib.qo_prefill_ex(self.h, int(quantized), _d(e), visual, text,
                                       _i(p) if p is not None else None, n, _i(lay), _d(kp), _d(wt),
                                       recipe.v0 if v0 is None else v0, res_bits, int(record), ok.size, okp, _b(oc))
        else:
            r = self.lib.qo_prefill_ex(self.h, int(quantized), _d(e), visual, text,
                                       _i(p) if p is not None else None, 0, None, None, None, 0, res_bits,
                                       int(record), ok.size, okp, _b(oc))
        if not r:
            raise OracleError(self.lib.qo_last_error().decode())
        return PortRun(self, r)

    def run_batch(self, embs, visual, text, recipe: Recipe, v0s, n_decode, dec_embs, n_threads, quantized=True,
                  res_bits=4):
        """prefill + n_decode steps per sequence, one sequence per thread; returns last logits."""
        n = len(embs)
        e = [f64(x) for x in embs]
        de = [f64(x) for x in dec_embs]
        ea = (_dp * n)(*[_d(x) for x in e])
        da = (_dp * n)(*[_d(x) for x in de])
        vis = np.array(visual, dtype=np.int32)
        txt = np.array(text, dtype=np.int32)
        lay = np.array(recipe.candidate_layers, dtype=np.int32)
        kp = f64(recipe.keep_ratios)
        wt = f64(recipe.weights)
        v0 = np.array(v0s, dtype=np.int32)
        out = np.empty((n, self.cfg.d_model), dtype=np.float64)
        _check(self.lib.qo_run_batch(self.h, int(quantized), n, ea, _i(vis), _i(txt), len(lay), _i(lay), _d(kp),
                                     _d(wt), _i(v0), res_bits, n_decode, da, n_threads, _d(out)), self.lib, "qo")
        return out


class PortRun:
    def __init__(self, owner, handle):
        self.o = owner
        self.lib = owner.lib
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.qo_run_free(self.h)
            self.h = None

    def result(self) -> RunResult:
        rows = self.lib.qo_run_logits_rows(self.h)
        lg = np.empty((rows, self.o.cfg.d_model), dtype=np.float64)
        self.lib.qo_run_logits(self.h, _d(lg))
        v, t = C.c_int(), C.c_int()
        pos = np.empty(rows + 4096, dtype=np.int32)
        self.lib.qo_run_layout(self.h, C.byref(v), C.byref(t), _i(pos))
        trace = []
        for i in range(self.lib.qo_run_n_prunes(self.h)):
            lay, bud, cnt = C.c_int(), C.c_int(), C.c_int()
            ps = np.empty(1 << 16, dtype=np.int32)
            self.lib.qo_run_prune(self.h, i, C.byref(lay), C.byref(bud), _i(ps), C.byref(cnt))
            trace.append((lay.value, bud.value, ps[:cnt.value].copy()))
        return RunResult(lg, v.value, t.value, pos[:v.value + t.value].copy(), trace)

    def last_scores(self):
        n = C.c_int()
        if self.lib.qo_run_last_scores(self.h, None, None, C.byref(n)) != 0:
            return None
        m = np.empty((4, n.value), dtype=np.float64)
        f = np.empty(n.value, dtype=np.float64)
        self.lib.qo_run_last_scores(self.h, _d(m), _d(f), C.byref(n))
        return m, f

    def kv(self, layer, head, which):
        rows = C.c_int()
        _check(self.lib.qo_run_kv(self.h, layer, head, which, None, None, None, C.byref(rows)), self.lib, "qo")
        dh = self.o.cfg.d_head
        codes = np.empty((rows.value, dh), dtype=np.int8)
        scales = np.empty(rows.value, dtype=np.float64)
        pos = np.empty(rows.value, dtype=np.int32)
        _check(self.lib.qo_run_kv(self.h, layer, head, which, _b(codes), _d(scales), _i(pos), C.byref(rows)),
               self.lib, "qo")
        return codes, scales, pos

    def block_output(self, layer):
        rows = C.c_int()
        _check(self.lib.qo_run_block_output(self.h, layer, None, C.byref(rows)), self.lib, "qo")
        out = np.empty((rows.value, self.o.cfg.d_model), dtype=np.float64)
        _check(self.lib.qo_run_block_output(self.h, layer, _d(out), C.byref(rows)), self.lib, "qo")
        return out

    def decode(self, emb):
        e = f64(emb)
        out = np.empty(self.o.cfg.d_model, dtype=np.float64)
        _check(self.lib.qo_decode(self.h, _d(e), _d(out)), self.lib, "qo")
        return out

    def records(self):
        """Recorded quantizer sites: list of dicts (phase, layer, site, codes [rows x cols],
        scales [rows x groups]); see tests/replay.py for the site numbering."""
        out = []
        for i in range(self.lib.qo_run_n_recs(self.h)):
            meta = np.empty(6, dtype=np.int32)
            _check(self.lib.qo_run_rec(self.h, i, _i(meta), None, None), self.lib, "qo")
            ph, ly, st, rows, cols, grp = (int(v) for v in meta)
            codes = np.empty((rows, cols), dtype=np.int8)
            scales = np.empty((rows, grp), dtype=np.float64)
            _check(self.lib.qo_run_rec(self.h, i, _i(meta), _b(codes), _d(scales)), self.lib, "qo")
            out.append(dict(phase=ph, layer=ly, site=st, codes=codes, scales=scales))
        return out

    def ties(self):
        """Decisions within the GPU's error budget of a rounding tie: (keys u64, codes, ratios)."""
        n = self.lib.qo_run_n_ties(self.h)
        k = np.empty(n, dtype=np.uint64)
        c = np.empty(n, dtype=np.int8)
        r = np.empty(n, dtype=np.float64)
        if n:
            self.lib.qo_run_ties(self.h, k.ctypes.data_as(C.POINTER(C.c_uint64)), _b(c), _d(r))
        return k, c, r

    def applied(self):
        """Overrides that changed one of this run's decisions: (keys, the restatement's own
        codes, their tie ratios)."""
        n = self.lib.qo_run_n_applied(self.h)
        k = np.empty(n, dtype=np.uint64)
        c = np.empty(n, dtype=np.int8)
        r = np.empty(n, dtype=np.float64)
        if n:
            self.lib.qo_run_applied(self.h, k.ctypes.data_as(C.POINTER(C.c_uint64)), _b(c), _d(r))
        return k, c, r

    def clear_records(self):
        self.lib.qo_run_clear_recs(self.h)

    def tie_margin(self, which):
        """Smallest |frac(x/s) - 0.5| over activation/KV quantizations of the last
        prefill (which=0) or decode step (which=1)."""
        return self.lib.qo_run_tie_margin(self.h, which)


# ---------------------------------------------------------------- synthetic inputs


def synth_weights(cfg: ModelCfg, seed: int, std: float = 0.02) -> Weights:
    """N(0, std) weights rounded to fp32 (so GPU and CPU see identical values)."""
    rng = np.random.default_rng(seed)
    d, f = cfg.d_model, cfg.d_ff
    kvd = cfg.n_kv_heads * cfg.d_head

    def g(*shape):
        return rng.normal(0.0, std, size=shape).astype(np.float32).astype(np.float64)

    w = Weights()
    for _ in range(cfg.n_layers):
        lw = dict(wq=g(d, d), wk=g(d, kvd), wv=g(d, kvd), wo=g(d, d), w1=g(d, f), w2=g(f, d),
                  g1=np.ones(d), g2=np.ones(d))
        if cfg.mlp == 1:
            lw["w3"] = g(d, f)
        w.layers.append(lw)
    w.head = g(d, d)
    w.gf = np.ones(d)
    return w


def synth_embeddings(n_tokens: int, d: int, seed: int, outlier_frac: float = 0.02, outlier_mult: float = 20.0):
    """N(0,1) hidden states with a seeded set of outlier channels x outlier_mult (BASELINE.json configs)."""
    rng = np.random.default_rng(seed)
    x = rng.normal(0.0, 1.0, size=(n_tokens, d))
    n_out = max(1, int(round(outlier_frac * d)))
    ch = rng.choice(d, size=n_out, replace=False)
    x[:, ch] *= outlier_mult
    return x.astype(np.float32).astype(np.float64)
