#!/usr/bin/env python3
"""bench.py -- QUOTA hot path on B200: W4A4 prefill with recipe-driven
visual-token pruning, then decode over the int4 paged KV cache.

One *step* = one request batch of the workload (BASELINE.json configs[1],
LLaVA-1.5-7B shape): B sequences of 576 visual + 64 text tokens prefilled
through 32 W4A4 layers with the QUOTA recipe (30 % visual retention from layer
2: 576 -> 173), then 128 teacher-forced decode steps over the int4 cache,
then the (N>1) gather of the final logits to rank 0.

  value  = whole-job tokens/s = N * (prefill tokens + B * D) / step time, inputs resident in HBM
  e2e    = the same through the public API with pinned HOST buffers
           (embeddings H2D and logits D2H inside the timed region, every step)

Synthetic data: seeded N(0, 0.02) weights generated on the device, N(0, 1)
hidden states with 1 % of the channels x20 (the configs' outlier model).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: one rank per GPU (NCCL).  Under torchrun WORLD_SIZE must equal --gpus; without
it bench.py starts the N ranks itself through torch.distributed.run.  The global
request batch is N x the per-GPU batch, sharded with shard.shard_range (sequences are
independent): each rank runs its own sequences (weak scaling) and NCCL only
gathers the final logits (inside the timed region, both legs) and the max-over-ranks
step time.  `--impl stub` runs the same rank plumbing on CPU (gloo) with a stand-in
engine, for the multi-process test (tests/test_bench_cpu.py).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "W4A4+QUOTA prefill ms & decode tok/s, 7B-shape, 1/2/4/8 B200, % roofline"
UNIT = "tokens/s"

CONFIGS = {
    # BASELINE.json configs[1]
    "c2": dict(workload="LLaVA-1.5-7B-shaped W4A4 + QUOTA 30% visual retention from layer 2 (configs[1])",
               n_layers=32, d_model=4096, n_heads=32, n_kv_heads=32, d_head=128, d_ff=11008, mlp=1, act_mode=1,
               batch=8, visual=576, text=64, decode=128, layers=[2], keeps=[0.3], v0=576, outlier=0.01),
    # BASELINE.json configs[2]: high-resolution prefix, multi-layer keep schedule
    "c3": dict(workload="LLaVA-7B shape, 2880 visual (5 tiles x 576) + 128 text, keep [1, 1, 0.25, 0.2 from L8] "
                        "(configs[2])",
               n_layers=32, d_model=4096, n_heads=32, n_kv_heads=32, d_head=128, d_ff=11008, mlp=1, act_mode=1,
               batch=4, visual=2880, text=128, decode=128, layers=[0, 1, 2, 8], keeps=[1.0, 1.0, 0.25, 0.2], v0=2880,
               outlier=0.01),
    # BASELINE.json configs[3]: Qwen2-VL shape, GQA, ragged visual lengths U[256, 1280] per sequence
    "c4": dict(workload="Qwen2-VL-7B shape (28 L, 3584, 28q/4kv GQA, SwiGLU 18944), ragged V~U[256,1280] + 64, "
                        "30% retention (configs[3])",
               n_layers=28, d_model=3584, n_heads=28, n_kv_heads=4, d_head=128, d_ff=18944, mlp=1, act_mode=1,
               batch=16, visual=(256, 1280), text=64, decode=256, layers=[2], keeps=[0.3], v0=None, outlier=0.01),
    # BASELINE.json configs[4]: decode-bound sweep point (already-pruned prefix 173 + 64); --batch/--decode override
    "c5": dict(workload="7B shape decode sweep point: pruned prefix 173 + 64, int4 group-128 KV (configs[4])",
               n_layers=32, d_model=4096, n_heads=32, n_kv_heads=32, d_head=128, d_ff=11008, mlp=1, act_mode=1,
               batch=64, visual=173, text=64, decode=512, layers=[], keeps=[], v0=173, outlier=0.01),
    # BASELINE.json configs[0] (tiny; parity case, also handy for a quick smoke bench)
    "c1": dict(workload="tiny VLM decoder (configs[0])", n_layers=4, d_model=256, n_heads=4, n_kv_heads=4,
               d_head=64, d_ff=688, mlp=1, act_mode=1, batch=1, visual=152, text=32, decode=16,
               layers=[0, 1, 2, 3], keeps=[1.0, 0.5, 0.3, 0.3], v0=152, outlier=0.02),
}


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi sampling of SM clocks + throttle reasons during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower() == "active"})
        under = [v for v in sm if v > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": float(np.median(under)) if under else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def load_traffic():
    """profiles/ncu_traffic.json (tools/ncu_traffic.py): DRAM bytes of single ncu-captured launches,
    with the algorithmic bytes of the same launch for the ratio."""
    try:
        rows = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        return {}
    out = {}
    for r in rows:
        k = r["kernel"]
        if "k_gemv_reg<1, 0" in k:  # decode QKV GEMV (any variant), B = 8: N 12288 x K 4096
            M, N, K = 8, 12288, 4096
            r["algorithmic_bytes"] = N * K / 2 + 8 * N + M * K / 2 + 8 * M + 4 * M * N
            out["gemv"] = r
        elif "k_attn_dec" in k:  # decode attention (k_attn_dec_w; earlier: k_attn_dec, k_attn_decode_pp2)
            out["attn_decode"] = dict(r, algorithmic_bytes=r["dram_bytes"])
    return out


def measure_int8_peak(torch, dev):
    """Dense int8 tensor-core throughput on this GPU through cuBLASLt (torch._int_mm),
    8192^3, best of 5 -- the roofline denominator for the int8 GEMMs (MEASURED_PEAKS.json
    has no int8 figure)."""
    try:
        a = torch.randint(-8, 8, (8192, 8192), dtype=torch.int8, device=dev)
        b = torch.randint(-8, 8, (8192, 8192), dtype=torch.int8, device=dev)
        torch._int_mm(a, b)
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        return 2.0 * 8192 ** 3 / (best / 1e3) / 1e12
    except Exception:
        return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def spawn_ranks(argv, n):
    """--gpus N > 1 without a torchrun environment: start N ranks of this script (one per
    GPU) through torch.distributed.run on 127.0.0.1; their rank 0 prints the line."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd)


def local_sequences(cfg, ws, rank):
    """This rank's share of the global request batch (ws x batch_per_gpu sequences):
    global sequence indices [first, first + count) (shard.shard_range)."""
    from paper_2604_17320_b200.shard import shard_range
    first, count = shard_range(ws * cfg["batch"], ws, rank)
    return list(range(first, first + count))


# --------------------------------------------------------------------------- reference arm


def reference_sample(threads, d_model, n_heads, d_head):
    """The UNMODIFIED reference (oracle/_ref) at 7B width: 4 layers (ModelConfig minimum),
    d_ff = 4 d SiLU MLP (the reference's fixed MLP; same FLOPs as SwiGLU 11008 within 1 %),
    static act scales, quantized mode.  Returns (model, setup seconds)."""
    import oracle as O
    t0 = time.time()
    cfg = O.ModelCfg(n_layers=4, d_model=d_model, n_heads=n_heads, n_kv_heads=n_heads, d_head=d_head,
                     d_ff=4 * d_model, weight_axis=1)
    ref = O.Ref(cfg, seed=1)
    ref.prepare(np.ones(4 * 4 + 1), weight_axis=1)
    return ref, time.time() - t0


def reference_tokens_per_s(ref, threads, n_layers_full, tokens_per_seq=1):
    """One bounded sample: `threads` sequences of `tokens_per_seq` tokens, one per host thread,
    through the 4-layer reference; scaled to the full depth (x 4 / n_layers_full)."""
    sec = ref.prefill_threads(threads, tokens_per_seq, 0, seed=int(time.time()) & 0xFFFF)
    return threads * tokens_per_seq / sec * (4.0 / n_layers_full), sec


def run_reference(args, cfg):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    ref, setup_s = reference_sample(threads, cfg["d_model"], cfg["n_heads"], cfg["d_head"])
    vals, secs = [], []
    for i in range(args.warmup + args.steps):
        v, sec = reference_tokens_per_s(ref, threads, cfg["n_layers"])
        if i >= args.warmup:
            vals.append(v)
            secs.append(sec * cfg["n_layers"] / 4.0)
    value = float(np.mean(vals))
    sample = (f"{threads} threads x 1-token sequence through the unmodified reference forward_prefill, 4 layers "
              f"at 7B width (d 4096, 32x128 heads, d_ff 16384 SiLU, static scales), quantized mode; "
              f"tokens/s extrapolated to {cfg['n_layers']} layers (x4/{cfg['n_layers']}); setup {setup_s:.1f}s")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            # one step = the extrapolated 32-layer sample
            "ms_per_step": float(np.mean(secs)) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "batch_per_gpu": cfg["batch"],
                       "visual": cfg["visual"], "text": cfg["text"], "decode_steps": cfg["decode"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- our arm


def build_engine(cfg, torch, Q, vis, seed=1234):
    c = Q.Config(n_layers=cfg["n_layers"], d_model=cfg["d_model"], n_heads=cfg["n_heads"],
                 n_kv_heads=cfg["n_kv_heads"], d_head=cfg["d_head"], d_ff=cfg["d_ff"], mlp=cfg["mlp"],
                 act_mode=cfg["act_mode"])
    B, D = cfg["batch"], cfg["decode"]
    S = max(vis) + cfg["text"]
    eng = Q.Engine(c, max_batch=B, max_tokens=sum(vis) + B * cfg["text"], max_seq=S, max_decode=D + 2)
    g = torch.Generator(device="cuda").manual_seed(seed)
    d, kvd, f = cfg["d_model"], cfg["n_kv_heads"] * cfg["d_head"], cfg["d_ff"]

    def rnd(*shape):
        return torch.randn(*shape, device="cuda", generator=g) * 0.02

    for l in range(cfg["n_layers"]):
        eng.load_layer(l, rnd(d, d), rnd(d, kvd), rnd(d, kvd), rnd(d, d), rnd(d, f), rnd(f, d),
                       rnd(d, f) if cfg["mlp"] == 1 else None)
    eng.load_head(rnd(d, d))
    if cfg["layers"]:
        eng.set_recipe(cfg["layers"], cfg["keeps"], v0=cfg["v0"] or 1, res_bits=4)
    else:
        eng.clear_recipe()
    torch.cuda.synchronize()
    return eng


def visual_lengths(cfg, seqs=None, seed=2024):
    """Per-sequence visual counts of the given global sequences (default: the first batch):
    fixed, or seeded U[lo, hi] draws for ragged batches (configs[3])."""
    v = cfg["visual"]
    seqs = list(range(cfg["batch"])) if seqs is None else seqs
    if isinstance(v, tuple):
        return [int(np.random.default_rng(seed + i).integers(v[0], v[1] + 1)) for i in seqs]
    return [v] * len(seqs)


def synth_inputs(cfg, torch, seqs, vis):
    """Hidden states N(0,1) with a seeded 1 % of channels x20 (BASELINE.json configs), seeded
    per GLOBAL sequence index so a sequence's inputs do not depend on the sharding."""
    D, d = cfg["decode"], cfg["d_model"]
    ch = torch.randperm(d, generator=torch.Generator(device="cpu").manual_seed(77))[
        :max(1, int(round(cfg["outlier"] * d)))]
    embs, decs = [], []
    for i, v in zip(seqs, vis):
        g = torch.Generator(device="cpu").manual_seed(1000 + i)
        e = torch.randn(v + cfg["text"], d, generator=g)
        dd = torch.randn(D, d, generator=g)
        e[:, ch] *= 20.0
        dd[:, ch] *= 20.0
        embs.append(e)
        decs.append(dd)
    return torch.cat(embs).contiguous(), torch.stack(decs, dim=1).contiguous()


def run_ours(args, cfg):
    import torch

    import paper_2604_17320_b200 as Q

    from paper_2604_17320_b200.shard import gather_equal_rows, max_over_ranks

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    B, T, D, d = cfg["batch"], cfg["text"], cfg["decode"], cfg["d_model"]
    seqs = local_sequences(cfg, ws, rank)  # this rank's global sequence indices
    assert len(seqs) == B
    vis = visual_lengths(cfg, seqs)
    V = max(vis)
    rows = sum(vis) + B * T  # prefill tokens of the batch
    v0s = vis if cfg["v0"] is None else None  # ragged: each sequence's own v0
    eng = build_engine(cfg, torch, Q, vis)
    if args.eager_decode:  # per-kernel tools (ncu launch lists): no graph replays
        eng.set_graphs(False)
    stream = torch.cuda.Stream(device=dev)
    eng.set_stream(stream)
    emb_h, dec_h = synth_inputs(cfg, torch, seqs, vis)
    emb_d, dec_d = emb_h.to(dev), dec_h.to(dev)
    logits_d = torch.empty(rows, d, device=dev)
    dlog_d = torch.empty(B, d, device=dev)
    greedy = not args.teacher_forced
    if greedy:  # the configs' "greedy steps": argmax token -> a seeded token-embedding table [d x d]
        gt = torch.Generator(device="cpu").manual_seed(55)
        table = torch.randn(d, d, generator=gt)
        table[:, torch.randperm(d, generator=gt)[:max(1, int(round(cfg["outlier"] * d)))]] *= 20.0
        eng.set_token_table(table.to(dev))
    tok_d = torch.zeros(D, B, dtype=torch.int32, device=dev)

    def decode_step(t, logits_out, tokens_out=None):
        if greedy:
            eng.decode_greedy(logits_out=logits_out, tokens_out=tokens_out if tokens_out is not None else tok_d[t])
        else:
            eng.decode(dec_d[t] if logits_out.is_cuda else dec_p[t], logits_out=logits_out)
    txt = [T] * B
    gathered = torch.empty(ws * B, d, device=dev) if ws > 1 else None

    def gather_outputs():  # the only collective: every sequence's final logits to rank 0's view
        if dist is not None:
            with torch.cuda.stream(stream):
                gather_equal_rows(dlog_d, gathered)

    def step_device():
        eng.prefill(emb_d, vis, txt, v0=v0s, logits_out=logits_d)
        for t in range(D):
            decode_step(t, dlog_d)
        gather_outputs()

    # e2e: pinned host buffers through the public API, copies inside the timed region
    emb_p, dec_p = emb_h.pin_memory(), dec_h.pin_memory()
    logits_p = torch.empty(rows, d).pin_memory()
    dlog_p = torch.empty(D, B, d).pin_memory()
    tok_p = torch.zeros(D, B, dtype=torch.int32).pin_memory()
    gathered_p = torch.empty(ws * B, d).pin_memory() if ws > 1 else None

    def step_e2e():
        # the prefill logits come back on the engine's copy stream while the decode steps run;
        # join_copies() puts their completion back on the timed stream before the step ends
        eng.prefill(emb_p, vis, txt, v0=v0s, logits_out=logits_p, logits_async=True)
        for t in range(D):
            if greedy:  # each step's tokens to the host; the logits stay on the device but the last
                decode_step(t, dlog_d, tok_p[t])
            else:
                decode_step(t, dlog_p[t] if t < D - 1 else dlog_d)
        with torch.cuda.stream(stream):
            dlog_p[D - 1].copy_(dlog_d, non_blocking=True)
            if dist is not None:  # the gathered final logits land in rank 0's host memory
                gather_equal_rows(dlog_d, gathered)
                if rank == 0:
                    gathered_p.copy_(gathered, non_blocking=True)
        eng.join_copies()

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def timed(fn, steps, sample_clocks=False):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sampler = ClockSampler(local) if sample_clocks else None
        if sampler:
            sampler.__enter__()
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        stream.synchronize()
        if sampler:
            sampler.__exit__()
        barrier()
        ms = e0.elapsed_time(e1) / steps
        if dist is not None:  # the job's step time is the slowest rank's
            ms = max_over_ranks(ms, device=dev)
        return ms, (sampler.summary() if sampler else None)

    for _ in range(args.warmup):
        step_device()
    ms_step, clocks = timed(step_device, args.steps, sample_clocks=True)

    # phase split (prefill ms, decode ms/step) on the device-resident path
    barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record(stream)
    eng.prefill(emb_d, vis, txt, v0=v0s, logits_out=logits_d)
    ev[1].record(stream)
    for t in range(D):
        decode_step(t, dlog_d)
    ev[2].record(stream)
    stream.synchronize()
    prefill_ms = ev[0].elapsed_time(ev[1])
    decode_ms = ev[1].elapsed_time(ev[2]) / D

    for _ in range(max(1, args.warmup // 2)):
        step_e2e()
    ms_e2e, _ = timed(step_e2e, args.steps)

    # per-kernel-class CUDA-event profile (one prefill + one eager decode step)
    eng.profile_next()
    eng.prefill(emb_d, vis, txt, v0=v0s, logits_out=logits_d)
    prof_pre = eng.profile_read()
    eng.profile_next()
    decode_step(0, dlog_d)
    prof_dec = eng.profile_read()
    # per-class decode time inside the CUDA graph (PDL overlap, real launch overheads): the
    # step replayed with only one kernel class left in (per-launch events break both)
    chain_ms = {"full": eng.profile_chain(0), "gemm": eng.profile_chain(2 | 4 | 8),
                "attention": eng.profile_chain(1 | 4 | 8), "quant": eng.profile_chain(1 | 2 | 8),
                "kv": eng.profile_chain(1 | 2 | 4), "none": eng.profile_chain(15)}
    info = eng.info()

    tokens = ws * (rows + B * D)
    value = tokens / (ms_step / 1e3)
    e2e_val = tokens / (ms_e2e / 1e3)
    final_rows = info["final_rows"]

    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs")
    peak_src = "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)" if hbm else "B200_PROFILING.md fallback"
    hbm = hbm or 6650.0
    int8_peak = measure_int8_peak(torch, dev) if rank == 0 else None
    traffic_db = load_traffic()
    # dominant kernel class over the whole step
    per_step = {}
    for c in prof_pre:
        per_step[("prefill", c)] = prof_pre[c]["ms"]
        # decode classes: graph-replayed chain time (the no-class floor -- head GEMV, final
        # norm, bump -- removed); the event profile of an eager step overstates every class
        per_step[("decode", c)] = (max(0.0, chain_ms[c] - chain_ms["none"]) if c in chain_ms
                                   else prof_dec[c]["ms"]) * D
    dom = max(per_step, key=per_step.get)
    phase, cls = dom
    src = prof_pre[cls] if phase == "prefill" else prof_dec[cls]
    avg_ms = src["ms"] / max(1, src["launches"])
    if phase == "decode" and cls in chain_ms:
        avg_ms = chain_ms[cls] / max(1, src["launches"])  # includes the head GEMV of the step
    if phase == "decode" and cls in ("gemm", "attention", "quant", "kv"):
        alg = src["bytes"] / max(1, src["launches"])
        achieved = alg / (avg_ms / 1e3) / 1e9
        traffic, tsrc = None, None
        ref = traffic_db.get("gemv" if cls == "gemm" else "attn_decode")
        if cls == "gemm" and B > 32:  # the capture is of the GEMV, not the int8 tcgen05 decode GEMM
            ref = None
        if ref:  # ncu --set full capture of one launch: DRAM bytes / algorithmic bytes of that launch
            ratio = ref["dram_bytes"] / ref["algorithmic_bytes"]
            traffic, tsrc = alg * ratio, f"{ref['source']}: dram/algorithmic = {ratio:.3f} on {ref['kernel']}"
        gname = "W4A4 GEMV, k_gemv_reg" if B <= 32 else "int8-operand tcgen05 GEMM, k_gemm_tc05_i8"
        roofline = {"bound": "hbm", "kernel": f"{phase} {cls} ({gname})" if cls == "gemm"
                    else f"{phase} {cls}", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "traffic": traffic, "traffic_source": tsrc, "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": alg, "avg_launch_ms": avg_ms,
                    "launch_time_method": "one decode step with only this kernel class, captured as a CUDA graph "
                                          "and replayed 20x (qt_engine_profile_chain), CUDA events on the engine "
                                          "stream; ms / launches",
                    "share_of_step": per_step[dom] / ms_step}
    else:
        tops = src["flops"] / max(1, src["launches"]) / (avg_ms / 1e3) / 1e12
        pk = int8_peak or 4500.0
        roofline = {"bound": "tensor", "kernel": f"{phase} {cls}", "achieved": tops, "peak": pk,
                    "unit": "TOP/s (int8)", "frac": tops / pk, "traffic": None,
                    "peak_source": "measured int8 cuBLASLt (torch._int_mm 8192^3)" if int8_peak
                    else "B200 dense int8 datasheet (no int8 figure in MEASURED_PEAKS.json)",
                    "avg_launch_ms": avg_ms, "share_of_step": per_step[dom] / ms_step}
    gemm_pre = prof_pre["gemm"]
    prefill_gemm_tops = gemm_pre["flops"] / (gemm_pre["ms"] / 1e3) / 1e12 if gemm_pre["ms"] else None
    gemv = prof_dec["gemm"]
    decode_gemv_gbs = gemv["bytes"] / (chain_ms["gemm"] / 1e3) / 1e9 if chain_ms["gemm"] else None
    attn = prof_dec["attention"]
    decode_attn_gbs = attn["bytes"] / (chain_ms["attention"] / 1e3) / 1e9 if chain_ms["attention"] else None

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            ref, setup_s = reference_sample(threads, d, cfg["n_heads"], cfg["d_head"])
            v, sec = reference_tokens_per_s(ref, threads, cfg["n_layers"])
            cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"{threads} threads x 1-token sequence, unmodified reference forward_prefill, 4 layers "
                             f"at 7B width (d_ff 16384 SiLU), {sec:.1f}s; extrapolated to {cfg['n_layers']} layers"}
            del ref
        except Exception as ex:  # the baseline is reported, never the product
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "reference", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int4xint4->int32 (W4A4), fp64 residual, int4 KV", "data": "synthetic",
            "config": {"workload": cfg["workload"], "batch_per_gpu": B, "global_batch": ws * B,
                       "visual": V if len(set(vis)) == 1 else {"ragged": list(cfg["visual"]), "mean": float(np.mean(vis))},
                       "text": T,
                       "decode_steps": D,
                       "decode": "teacher-forced (seeded step embeddings)" if not greedy else
                       "greedy: argmax over the d_model-wide logits -> row of a seeded token-embedding table "
                       "[d x d] (SURVEY.md 0.1; the argmax + embedding kernel is in the step's CUDA graph)",
                       "recipe": {"candidate_layers": cfg["layers"], "keep_ratios": cfg["keeps"],
                                                     "v0": cfg["v0"]},
                       "layers": cfg["n_layers"], "d_model": d, "heads": cfg["n_heads"], "d_ff": cfg["d_ff"],
                       "parallelism": f"dp{ws} (batch sharded, NCCL gather of outputs only)",
                       "l2": "working set > L2: 3.25 GB int4 weights streamed every decode step and prefill layer"},
            "prefill_ms": prefill_ms, "prefill_tokens_per_s": ws * rows / (prefill_ms / 1e3),
            "decode_ms_per_step": decode_ms, "decode_tokens_per_s": ws * B / (decode_ms / 1e3),
            "prefill_gemm_tops": prefill_gemm_tops, "int8_peak_tops_measured": int8_peak, "decode_gemv_gbs": decode_gemv_gbs,
            "decode_attn_gbs": decode_attn_gbs, "final_rows": final_rows,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": UNIT, "ms_per_step": ms_e2e,
                    "h2d_bytes_per_step": int(emb_p.numel() * 4 + (0 if greedy else dec_p.numel() * 4)),
                    "d2h_bytes_per_step": int(final_rows * d * 4 + (D * B * 4 + B * d * 4 if greedy else D * B * d * 4)
                                              + (ws * B * d * 4 if ws > 1 else 0)),
                    "per_rank": True, "gather": "final decode logits of all ws x B sequences to rank 0 host"
                    if ws > 1 else None},
            "gpu_launches": int(sum(v["launches"] for v in prof_pre.values())
                                + D * sum(v["launches"] for v in prof_dec.values())),
            "clocks": clocks,
            "profile": {"prefill": prof_pre, "decode_step": prof_dec, "decode_chain_ms": chain_ms},
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if dist is not None:
        dist.destroy_process_group()


def run_stub(args, cfg):
    """The multi-rank plumbing of run_ours on CPU (gloo) with a stand-in for the engine:
    shard the global batch, run each rank's sequences, gather every sequence's final row to
    rank 0, time steps as the max over ranks.  For tests/test_bench_cpu.py only."""
    import torch
    import torch.distributed as dist

    from paper_2604_17320_b200.shard import gather_equal_rows, max_over_ranks

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    B, d = cfg["batch"], 64
    seqs = local_sequences(cfg, ws, rank)
    w = torch.randn(d, d, generator=torch.Generator().manual_seed(5))

    def step():
        x = torch.stack([torch.full((d,), float(i)) for i in seqs])  # sequence i's "state"
        for _ in range(cfg["decode"]):
            x = torch.tanh(x @ w) + torch.tensor(seqs, dtype=torch.float32)[:, None]
        x[:, -1] = torch.tensor(seqs, dtype=torch.float32)  # tag each row with its global sequence
        out = torch.empty(ws * B, d)
        if ws > 1:
            gather_equal_rows(x, out)
        else:
            out.copy_(x)
        return out

    for _ in range(args.warmup):
        step()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out = step()
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    ms_max = max_over_ranks(ms) if ws > 1 else ms
    if rank == 0:
        print(json.dumps({"impl": "stub", "metric": METRIC, "n_gpus": ws, "steps": args.steps,
                          "ms_per_step": ms_max, "value": ws * B * cfg["decode"] / (ms_max / 1e3),
                          "config": {"batch_per_gpu": B, "global_batch": ws * B},
                          "gathered_last_col": out[:, -1].tolist(), "local_sequences": seqs}), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference", "stub"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--teacher-forced", action="store_true",
                    help="decode with seeded step embeddings instead of greedy argmax tokens")
    ap.add_argument("--batch", type=int, default=None, help="override the config's per-GPU batch (c5 sweep)")
    ap.add_argument("--decode", type=int, default=None, help="override the config's decode steps (c5 sweep)")
    ap.add_argument("--eager-decode", action="store_true",
                    help="decode steps as eager launches, not CUDA graph replays (for ncu launch lists)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.batch:
        cfg["batch"] = args.batch
    if args.decode:
        cfg["decode"] = args.decode
    ws = int(os.environ.get("WORLD_SIZE", "0"))
    if ws == 0 and args.gpus > 1:  # start the N ranks (one per GPU) ourselves
        sys.exit(spawn_ranks(sys.argv[1:], args.gpus))
    if ws and ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} does not match WORLD_SIZE {ws}")
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.impl == "stub":
        run_stub(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
