"""paper_2604_17320_b200 -- B200-native QUOTA hot path (W4A4 prefill with
recipe-driven visual-token pruning, decode over an int4 paged KV cache).

The product is the C-ABI library ``_build/libquota_b200.so`` (CUDA kernels for
sm_100a + the C++ host engine, declared in ``include/quota_b200.h``).  This
module is a thin ctypes binding used by tests and bench.py; it never computes
anything itself and there is no CPU fallback: if the library or a GPU is
missing every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QT_LIB_PATH") or os.path.join(HERE, "_build", "libquota_b200.so")  # override: A/B builds
ROOT = os.path.dirname(HERE)
HEADER = os.path.join(ROOT, "include", "quota_b200.h")

QT_EINVAL, QT_ERUNTIME, QT_ERANGE, QT_ECUDA = -1, -2, -3, -4
EPI_STORE, EPI_RESADD, EPI_SILU, EPI_SWIGLU = 0, 1, 2, 3


class QuotaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class QuotaInvalidArgument(QuotaError, ValueError):
    """std::invalid_argument in the reference."""


class QuotaRuntimeError(QuotaError):
    """std::runtime_error in the reference."""


class QuotaOutOfRange(QuotaError, IndexError):
    """std::out_of_range in the reference."""


_lib = None


class _Config(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("n_layers", "d_model", "n_heads", "n_kv_heads", "d_head", "d_ff", "mlp",
                                        "act_mode", "weight_bits", "act_bits", "kv_bits")]


def lib():
    """Load the CUDA library (fails loudly when it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        vp, ip, dp, fp = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_float)
        L.qt_last_error.restype = C.c_char_p
        L.qt_engine_create.argtypes = [C.POINTER(_Config), C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
        L.qt_engine_destroy.argtypes = [vp]
        L.qt_engine_destroy.restype = None
        L.qt_engine_set_stream.argtypes = [vp, vp]
        L.qt_engine_synchronize.argtypes = [vp]
        L.qt_engine_load_layer.argtypes = [vp, C.c_int] + [vp] * 9 + [C.c_int]
        L.qt_engine_load_head.argtypes = [vp, vp, vp, C.c_int]
        L.qt_engine_set_act_scales.argtypes = [vp, dp]
        L.qt_engine_set_recipe.argtypes = [vp, C.c_int, ip, dp, dp, C.c_int, C.c_int]
        L.qt_recipe_parse.argtypes = [C.c_char_p, C.c_int, ip, ip, dp, dp, ip, C.c_char_p, C.c_int]
        L.qt_engine_prefill.argtypes = [vp, C.c_int, vp, C.c_int, ip, ip, ip, ip, vp, C.c_int]
        L.qt_engine_prefill_rows.argtypes = [vp]
        L.qt_engine_decode.argtypes = [vp, vp, C.c_int, vp, C.c_int]
        L.qt_engine_layout.argtypes = [vp, C.c_int, ip, ip, ip, C.c_int]
        L.qt_engine_n_prunes.argtypes = [vp, C.c_int]
        L.qt_engine_prune.argtypes = [vp, C.c_int, C.c_int, ip, ip, ip, C.c_int, ip]
        L.qt_engine_kv.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, fp, ip, C.c_int]
        L.qt_engine_info.argtypes = [vp, C.POINTER(C.c_int64)]
        L.qt_engine_profile_next.argtypes = [vp]
        L.qt_engine_profile_read.argtypes = [vp, C.POINTER(C.c_double)]
        L.qt_rmsnorm_quant_i4.argtypes = [vp, C.c_int, C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                          vp, C.c_int, vp, vp, vp]
        L.qt_w4a4_gemm.argtypes = [C.c_int, vp, C.c_int, vp, vp, C.c_int, vp, C.c_int, C.c_int, C.c_int, vp, C.c_int,
                                   vp, C.c_int, vp]
        L.qt_quant_weight_i4.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, vp, vp, vp]
        L.qt_kv_quant_append_i4.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp,
                                            C.c_int, vp, C.c_int64, vp, vp]
        L.qt_rope_table.argtypes = [C.c_int, C.c_int, dp]
        L.qt_engine_keep_fp_weights.argtypes = [vp, C.c_int]
        L.qt_engine_fit_act_scales.argtypes = [vp, C.c_int, C.POINTER(dp), ip, ip, dp, C.c_int]
        L.qt_engine_fit_act_scales_hooked.argtypes = [vp, C.c_int, C.POINTER(dp), ip, ip, dp, C.c_int]
        L.qt_engine_profile_chain.argtypes = [vp, C.c_int, C.c_int, dp]
        L.qt_engine_join_copies.argtypes = [vp]
        L.qt_engine_prefill_fp.argtypes = [vp, C.c_int, C.POINTER(dp), ip, ip, C.c_int, dp, C.c_int64]
        L.qt_engine_profile_sensitivity.argtypes = [vp, C.c_int, C.POINTER(dp), ip, ip, C.c_int, ip, C.c_double,
                                                    dp, dp]
        L.qt_engine_profile_diagnostics.argtypes = [vp, C.c_int, C.POINTER(dp), ip, ip, dp, dp, dp]
        L.qt_engine_run_quota_calibration.argtypes = [vp, C.c_int, C.POINTER(dp), ip, ip, C.c_int, C.c_double,
                                                      C.c_double, C.c_double, dp, ip, dp, dp, dp, dp, dp]
        L.qt_engine_save.argtypes = [vp, C.c_char_p]
        L.qt_engine_load.argtypes = [vp, C.c_char_p]
        L.qt_engine_scores.argtypes = [vp, C.c_int, C.c_int, dp, dp, C.c_int, ip]
        L.qt_quota_topk.argtypes = [vp, C.c_int, C.c_int, vp, vp, dp, vp, vp, vp, vp]
        L.qt_w4a4_gemm_i8.argtypes = [C.c_int, vp, C.c_int, vp, vp, C.c_int, C.c_int, vp, C.c_int, C.c_int,
                                      C.c_int, vp, C.c_int, vp, vp, C.c_int, vp]
        L.qt_w4a4_gemm_i8_workspace.restype = C.c_int64
        L.qt_w4a4_gemm_i8_workspace.argtypes = [C.c_int, C.c_int, C.c_int]
        L.qt_engine_set_token_table.argtypes = [vp, vp, C.c_int, C.c_int]
        L.qt_engine_set_graphs.argtypes = [vp, C.c_int]
        L.qt_engine_decode_greedy.argtypes = [vp, vp, vp, C.c_int]
        L.qt_engine_capture.argtypes = [vp, C.c_int]
        L.qt_engine_capture_count.argtypes = [vp]
        L.qt_engine_capture_get.argtypes = [vp, C.c_int, ip, vp, dp]
        L.qt_unpack_codes.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, vp]
        ci = C.c_int
        L.qt_attn_prefill_i4kv.argtypes = [vp, ci, ci, ci, ci, ci, vp, vp, vp, ci, vp, C.c_int64, vp, ci, vp, ci, vp,
                                           vp]
        L.qt_attn_decode_workspace.restype = C.c_int64
        L.qt_attn_decode_workspace.argtypes = [ci, ci, ci, ci]
        L.qt_attn_decode_i4kv.argtypes = [vp, ci, ci, ci, ci, ci, vp, ci, vp, C.c_int64, vp, ci, vp, ci, vp, vp]
        L.qt_quota_score_workspace.restype = C.c_int64
        L.qt_quota_score_workspace.argtypes = [ci, ci, ci]
        L.qt_quota_score.argtypes = [vp, ci, vp, ci, ci, ci, ci, ci, vp, vp, vp, ci, vp, C.c_int64, vp, ci, vp, ci,
                                     vp, ci, vp, vp]
        L.qt_topk_compact.argtypes = [vp, ci, ci, vp, vp, vp, dp, vp, vp, vp, vp, ci, vp, ci, vp, vp, vp, C.c_int64,
                                      vp, ci, ci, ci, vp, vp, vp, vp]
        _lib = L
    return _lib


def _raise(rc):
    msg = lib().qt_last_error().decode()
    cls = {QT_EINVAL: QuotaInvalidArgument, QT_ERUNTIME: QuotaRuntimeError, QT_ERANGE: QuotaOutOfRange}.get(
        rc, QuotaError)
    raise cls(rc, msg)


def check(rc):
    if rc != 0:
        _raise(rc)
    return rc


def _ptr(t):
    """Device or host pointer of a torch tensor / numpy array (None passes through)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(C.c_void_p)
    return C.c_void_p(t.data_ptr())


def _on_device(t):
    """1 for a CUDA torch tensor, 0 for numpy / CPU (e.g. pinned) torch tensors."""
    return 0 if isinstance(t, np.ndarray) else int(bool(getattr(t, "is_cuda", False)))


def _i32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int32)


def _ip(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int))


@dataclass
class Config:
    """Shape + semantic switches (include/quota_b200.h qt_config)."""

    n_layers: int = 4
    d_model: int = 256
    n_heads: int = 4
    n_kv_heads: int = 4
    d_head: int = 64
    d_ff: int = 1024
    mlp: int = 0
    act_mode: int = 0
    weight_bits: int = 4
    act_bits: int = 4
    kv_bits: int = 4

    def c(self):
        return _Config(*[getattr(self, f) for f, _ in _Config._fields_])


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class Engine:
    """Owner of one device engine (weights, KV pool, buffers) on the current GPU."""

    def __init__(self, cfg: Config, max_batch=8, max_tokens=8192, max_seq=4096, max_decode=128):
        self.cfg = cfg
        self.max_batch, self.max_tokens, self.max_seq, self.max_decode = max_batch, max_tokens, max_seq, max_decode
        self.h = C.c_void_p()
        check(lib().qt_engine_create(C.byref(cfg.c()), max_batch, max_tokens, max_seq, max_decode, C.byref(self.h)))

    def close(self):
        if self.h:
            lib().qt_engine_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream):
        check(lib().qt_engine_set_stream(self.h, _stream_ptr(stream)))

    def synchronize(self):
        check(lib().qt_engine_synchronize(self.h))

    def load_layer(self, layer, wq, wk, wv, wo, w1, w2, w3=None, g1=None, g2=None):
        """Weights in reference orientation [d_in x d_out]: numpy fp32 (host) or torch fp32 cuda tensors."""
        arrs = [wq, wk, wv, wo, w1, w2, w3, g1, g2]
        on_dev = int(any(a is not None and not isinstance(a, np.ndarray) for a in arrs))
        keep = [None if a is None else (np.ascontiguousarray(a, dtype=np.float32) if isinstance(a, np.ndarray)
                                        else a.contiguous()) for a in arrs]
        check(lib().qt_engine_load_layer(self.h, layer, *[_ptr(a) for a in keep], on_dev))

    def load_head(self, w_head, gf=None):
        arrs = [w_head, gf]
        on_dev = int(any(a is not None and not isinstance(a, np.ndarray) for a in arrs))
        keep = [None if a is None else (np.ascontiguousarray(a, dtype=np.float32) if isinstance(a, np.ndarray)
                                        else a.contiguous()) for a in arrs]
        check(lib().qt_engine_load_head(self.h, _ptr(keep[0]), _ptr(keep[1]), on_dev))

    def load_weights(self, w):
        """w: oracle.Weights-like object (fp64 numpy, reference orientation)."""
        for l, lw in enumerate(w.layers):
            self.load_layer(l, lw["wq"], lw["wk"], lw["wv"], lw["wo"], lw["w1"], lw["w2"], lw.get("w3"),
                            lw.get("g1"), lw.get("g2"))
        self.load_head(w.head, w.gf)

    def keep_fp_weights(self, on=True):
        """Keep fp64 copies of the full-precision weights (call before load_*) for calibration."""
        check(lib().qt_engine_keep_fp_weights(self.h, int(on)))

    def fit_act_scales(self, samples, apply=True, hooked=False):
        """fit_act_scales (calibrator.cpp:237-249) on the device: samples = [(emb fp64 [S x d],
        visual, text)] -> 4 * n_layers + 1 static scales (installed when apply).  hooked: the
        forwards run under the engine's recipe (the prune_then_quant fit, harness.cpp:103-106)."""
        embs = [np.ascontiguousarray(e, dtype=np.float64) for e, _, _ in samples]
        arr = (C.POINTER(C.c_double) * len(embs))(*[e.ctypes.data_as(C.POINTER(C.c_double)) for e in embs])
        vis = _i32([v for _, v, _ in samples])
        txt = _i32([t for _, _, t in samples])
        out = np.empty(4 * self.cfg.n_layers + 1, dtype=np.float64)
        fn = lib().qt_engine_fit_act_scales_hooked if hooked else lib().qt_engine_fit_act_scales
        check(fn(self.h, len(embs), arr, _ip(vis), _ip(txt), out.ctypes.data_as(C.POINTER(C.c_double)), int(apply)))
        return out

    def prefill_fp(self, samples, hook=False):
        """forward_prefill in ExecMode::Fp (model.cpp:315-453), fp64 on the device, of each
        sample (emb fp64 [S x d], visual, text); hook: under the engine's recipe.  Returns the
        per-sample fp64 logits of the final layouts; trace() / layout() read the rest."""
        embs = [np.ascontiguousarray(e, dtype=np.float64) for e, _, _ in samples]
        arr = (C.POINTER(C.c_double) * len(embs))(*[e.ctypes.data_as(C.POINTER(C.c_double)) for e in embs])
        vis = _i32([v for _, v, _ in samples])
        txt = _i32([t for _, _, t in samples])
        cap = int(np.sum(vis + txt))
        out = np.empty((cap, self.cfg.d_model), dtype=np.float64)
        check(lib().qt_engine_prefill_fp(self.h, len(embs), arr, _ip(vis), _ip(txt), int(hook),
                                         out.ctypes.data_as(C.POINTER(C.c_double)), cap))
        res, o = [], 0
        for b in range(len(embs)):
            v, t, _ = self.layout(b)
            res.append(out[o:o + v + t])
            o += v + t
        return res

    def profile_sensitivity(self, samples, layers, eta=1e-6):
        """QUOTA Eq. 1 sensitivities (calibrator.cpp:42-82) -> (raw, normalized)."""
        embs = [np.ascontiguousarray(e, dtype=np.float64) for e, _, _ in samples]
        arr = (C.POINTER(C.c_double) * len(embs))(*[e.ctypes.data_as(C.POINTER(C.c_double)) for e in embs])
        vis, txt = _i32([v for _, v, _ in samples]), _i32([t for _, _, t in samples])
        lay = _i32(layers)
        raw, nrm = np.empty(len(lay)), np.empty(len(lay))
        check(lib().qt_engine_profile_sensitivity(self.h, len(embs), arr, _ip(vis), _ip(txt), len(lay), _ip(lay),
                                                  eta, raw.ctypes.data_as(C.POINTER(C.c_double)),
                                                  nrm.ctypes.data_as(C.POINTER(C.c_double))))
        return raw, nrm

    def run_quota_calibration(self, samples, window=5, p_min=0.3, tau=0.25, eta=1e-6):
        """run_quota_calibration (calibrator.cpp:251-268) on the device -> dict with the
        act scales (installed), recipe layers / keep ratios, sensitivities and diagnostics."""
        embs = [np.ascontiguousarray(e, dtype=np.float64) for e, _, _ in samples]
        arr = (C.POINTER(C.c_double) * len(embs))(*[e.ctypes.data_as(C.POINTER(C.c_double)) for e in embs])
        vis, txt = _i32([v for _, v, _ in samples]), _i32([t for _, _, t in samples])
        L = self.cfg.n_layers
        acts, lay, kp = np.empty(4 * L + 1), np.empty(window, dtype=np.int32), np.empty(window)
        raw, nrm, cm, rm = np.empty(window), np.empty(window), np.empty(L), np.empty(L)
        dp_ = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
        check(lib().qt_engine_run_quota_calibration(self.h, len(embs), arr, _ip(vis), _ip(txt), window, p_min, tau,
                                                    eta, dp_(acts), _ip(lay), dp_(kp), dp_(raw), dp_(nrm), dp_(cm),
                                                    dp_(rm)))
        return dict(act_scales=acts, layers=lay, keeps=kp, raw=raw, normalized=nrm, conc=cm, red=rm)

    def save(self, path):
        """Write the packed-int4 weight file (device layout, include/quota_b200.h)."""
        check(lib().qt_engine_save(self.h, os.fsencode(path)))

    def load(self, path):
        """Load a packed-int4 weight file written by save() for the same configuration."""
        check(lib().qt_engine_load(self.h, os.fsencode(path)))

    def set_act_scales(self, scales):
        a = np.ascontiguousarray(scales, dtype=np.float64)
        check(lib().qt_engine_set_act_scales(self.h, a.ctypes.data_as(C.POINTER(C.c_double))))

    def set_recipe(self, layers, keeps, weights=(0.25, 0.45, 0.10, 0.20), v0=64, res_bits=4):
        la = _i32(layers)
        ka = np.ascontiguousarray(keeps, dtype=np.float64)
        wa = np.ascontiguousarray(weights, dtype=np.float64)
        check(lib().qt_engine_set_recipe(self.h, len(la), _ip(la), ka.ctypes.data_as(C.POINTER(C.c_double)),
                                         wa.ctypes.data_as(C.POINTER(C.c_double)), v0, res_bits))

    def clear_recipe(self):
        check(lib().qt_engine_set_recipe(self.h, 0, None, None, None, 1, 4))

    def join_copies(self):
        """Order the engine stream after a pending asynchronous logits readback."""
        check(lib().qt_engine_join_copies(self.h))

    def prefill(self, emb, visual, text, v0=None, positions=None, logits_out=None, logits_async=False):
        """emb: packed [sum(S) x d] fp32 -- numpy / CPU (pinned) torch on the host, or a
        CUDA torch tensor.  Returns the logits rows (numpy, or a view of logits_out).
        logits_async=True (host logits_out): the rows are copied back on the engine's copy
        stream while later calls run and are valid only after synchronize()."""
        visual, text = _i32(visual), _i32(text)
        on_dev = _on_device(emb)
        if isinstance(emb, np.ndarray):
            emb = np.ascontiguousarray(emb, dtype=np.float32)
        v0a, pa = _i32(v0), _i32(positions)
        if logits_out is None:
            out = np.empty((int(np.sum(visual + text)), self.cfg.d_model), dtype=np.float32)
        else:
            out = logits_out
        odev = _on_device(out)
        if logits_async and not odev:
            odev = 2  # host readback on the engine's copy stream; valid after synchronize()
        check(lib().qt_engine_prefill(self.h, len(visual), _ptr(emb), on_dev, _ip(visual), _ip(text), _ip(v0a),
                                      _ip(pa), _ptr(out), odev))
        rows = lib().qt_engine_prefill_rows(self.h)
        return out[:rows]

    def decode(self, emb, logits_out=None):
        on_dev = _on_device(emb)
        if isinstance(emb, np.ndarray):
            emb = np.ascontiguousarray(emb, dtype=np.float32)
        out = np.empty((emb.shape[0], self.cfg.d_model), dtype=np.float32) if logits_out is None else logits_out
        check(lib().qt_engine_decode(self.h, _ptr(emb), on_dev, _ptr(out), _on_device(out)))
        return out

    def set_graphs(self, on):
        """Decode steps as CUDA graph replays (True, default) or eager launches (False)."""
        check(lib().qt_engine_set_graphs(self.h, int(bool(on))))

    def set_token_table(self, table):
        """Token-embedding table [vocab x d_model] fp32 (numpy or CUDA torch) for decode_greedy."""
        on_dev = _on_device(table)
        t = np.ascontiguousarray(table, dtype=np.float32) if isinstance(table, np.ndarray) else table.contiguous()
        check(lib().qt_engine_set_token_table(self.h, _ptr(t), t.shape[0], on_dev))

    def decode_greedy(self, logits_out=None, tokens_out=None):
        """One greedy step for every sequence: returns (tokens [B] int32 numpy, logits)."""
        B = self.info()["batch"]
        out = np.empty((B, self.cfg.d_model), dtype=np.float32) if logits_out is None else logits_out
        tok = np.empty(B, dtype=np.int32) if tokens_out is None else tokens_out
        check(lib().qt_engine_decode_greedy(self.h, _ptr(tok), _ptr(out), _on_device(out)))
        return tok, out

    def layout(self, seq):
        v, t = C.c_int(), C.c_int()
        pos = np.empty(1 << 16, dtype=np.int32)
        check(lib().qt_engine_layout(self.h, seq, C.byref(v), C.byref(t), _ip(pos), pos.size))
        return v.value, t.value, pos[:v.value + t.value].copy()

    def trace(self, seq):
        n = lib().qt_engine_n_prunes(self.h, seq)
        out = []
        for i in range(n):
            lay, bud, cnt = C.c_int(), C.c_int(), C.c_int()
            ps = np.empty(1 << 16, dtype=np.int32)
            check(lib().qt_engine_prune(self.h, seq, i, C.byref(lay), C.byref(bud), _ip(ps), ps.size, C.byref(cnt)))
            out.append((lay.value, bud.value, ps[:cnt.value].copy()))
        return out

    def kv(self, layer, seq, head, which):
        rows = C.c_int()
        check(lib().qt_engine_kv(self.h, layer, seq, head, which, None, None, C.byref(rows), 0))
        n = rows.value
        codes = np.empty((n, self.cfg.d_head), dtype=np.int8)
        scales = np.empty(n, dtype=np.float32)
        check(lib().qt_engine_kv(self.h, layer, seq, head, which, codes.ctypes.data_as(C.c_void_p),
                                 scales.ctypes.data_as(C.POINTER(C.c_float)), C.byref(rows), n))
        return codes, scales

    def scores(self, layer, seq):
        """(fused [n], normalised metrics [4 x n]) of the selection at `layer` in the last prefill."""
        n = C.c_int()
        check(lib().qt_engine_scores(self.h, layer, seq, None, None, 0, C.byref(n)))
        f = np.empty(n.value)
        m = np.empty((4, n.value))
        check(lib().qt_engine_scores(self.h, layer, seq, f.ctypes.data_as(C.POINTER(C.c_double)),
                                     m.ctypes.data_as(C.POINTER(C.c_double)), n.value, C.byref(n)))
        return f, m

    def capture(self, on=True):
        """Record every quantizer site's codes of the following prefill / decode calls
        (parity tests; decode steps then run eagerly).  Clears earlier records."""
        check(lib().qt_engine_capture(self.h, int(on)))

    def captured(self):
        """The records of capture(): list of dicts (phase, layer, site, codes [rows x cols]
        int8, scales [rows x groups] fp64), rows packed by sequence."""
        out = []
        for i in range(lib().qt_engine_capture_count(self.h)):
            meta = np.empty(6, dtype=np.int32)
            check(lib().qt_engine_capture_get(self.h, i, _ip(meta), None, None))
            ph, ly, st, rows, cols, grp = (int(v) for v in meta)
            codes = np.empty((rows, cols), dtype=np.int8)
            scales = np.empty((rows, grp), dtype=np.float64)
            check(lib().qt_engine_capture_get(self.h, i, _ip(meta), codes.ctypes.data_as(C.c_void_p),
                                              scales.ctypes.data_as(C.POINTER(C.c_double))))
            out.append(dict(phase=ph, layer=ly, site=st, codes=codes, scales=scales))
        return out

    PROFILE_CLASSES = ("gemm", "attention", "quant", "kv", "select", "other")

    def profile_chain(self, skip_mask, reps=20):
        """ms per decode step with the kernel classes in skip_mask left out (1 GEMM, 2 attention,
        4 quantizers, 8 KV append), graph-replayed; the cache state is restored."""
        ms = C.c_double()
        check(lib().qt_engine_profile_chain(self.h, int(skip_mask), int(reps), C.byref(ms)))
        return ms.value

    def profile_next(self):
        """Time every kernel of the next prefill/decode call with CUDA events."""
        check(lib().qt_engine_profile_next(self.h))

    def profile_read(self):
        o = (C.c_double * 24)()
        lib().qt_engine_profile_read(self.h, o)
        return {c: dict(ms=o[4 * i], launches=int(o[4 * i + 1]), bytes=o[4 * i + 2], flops=o[4 * i + 3])
                for i, c in enumerate(self.PROFILE_CLASSES)}

    def info(self):
        o = (C.c_int64 * 16)()
        lib().qt_engine_info(self.h, o)
        keys = ["stream", "n_pages", "page_bytes", "dec_splits", "dec_pps", "final_rows", "batch", "decode_steps",
                "decode_weight_bytes", "kv_rows", "pool", "n_qkv", "kd_pad", "kff_pad", "n_gu", "_"]
        return dict(zip(keys, list(o)))


def parse_recipe(text, max_layers=256):
    """parse_recipe (recipe.cpp:91-116) through qt_recipe_parse (host-side, strict keys,
    schema_version 1, PruningRecipe::validate); raises QuotaInvalidArgument like the
    reference's std::invalid_argument."""
    n = C.c_int()
    lay = np.empty(max_layers, dtype=np.int32)
    kp = np.empty(max_layers, dtype=np.float64)
    w = np.empty(4, dtype=np.float64)
    v0 = C.c_int()
    dg = C.create_string_buffer(256)
    check(lib().qt_recipe_parse(text.encode() if isinstance(text, str) else text, max_layers, C.byref(n), _ip(lay),
                                kp.ctypes.data_as(C.POINTER(C.c_double)), w.ctypes.data_as(C.POINTER(C.c_double)),
                                C.byref(v0), dg, 256))
    k = n.value
    return dict(candidate_layers=lay[:k].tolist(), keep_ratios=kp[:k].tolist(), weights=tuple(w.tolist()),
                v0=v0.value, quant_digest=dg.value.decode())


# ---------------------------------------------------------------- kernel-level ABI (torch tensors)


def rmsnorm_quant(x, gain, d_pad, act_mode, static_scale=0.0, codes=None, scales=None, normed=None, stream=0):
    """K1 on a torch fp32/fp64 cuda tensor x [M x D]; returns (packed codes, fp64 scales)."""
    import torch
    M, D = x.shape
    if codes is None:  # tiled layout: rows padded to 16
        codes = torch.zeros(((M + 15) // 16 * 16, d_pad // 2), dtype=torch.uint8, device=x.device)
    if scales is None:
        scales = torch.zeros(M, dtype=torch.float64, device=x.device)
    is64 = int(x.dtype == torch.float64)
    check(lib().qt_rmsnorm_quant_i4(_ptr(x), is64, x.stride(0), _ptr(gain), M, D, d_pad, act_mode,
                                    float(static_scale), _ptr(codes), codes.shape[0], _ptr(scales), _ptr(normed),
                                    C.c_void_p(stream)))
    return codes, scales


def w4a4_gemm(epi, a_codes, a_scales, w_codes, w_scales, M, N, K, out, acc_out=None, impl=0, stream=0):
    check(lib().qt_w4a4_gemm(epi, _ptr(a_codes), a_codes.shape[0], _ptr(a_scales), _ptr(w_codes), w_codes.shape[0],
                             _ptr(w_scales), M, N, K, _ptr(out), out.stride(0), _ptr(acc_out), impl,
                             C.c_void_p(stream)))
    return out


def w4a4_gemm_i8(epi, a8, sa, w8, sw, M, N, K, out, acc_out=None, workspace=None, single=False, stream=0, ksplit=0):
    """qt_w4a4_gemm_i8 on int8 operand tensors (16 x code, row-major)."""
    check(lib().qt_w4a4_gemm_i8(epi, _ptr(a8), a8.shape[1], _ptr(sa), _ptr(w8), w8.shape[0], w8.shape[1], _ptr(sw),
                                M, N, K, _ptr(out), out.stride(0), _ptr(acc_out), _ptr(workspace),
                                int(single) | (int(ksplit) << 8), C.c_void_p(stream)))
    return out


def quant_weight(w, k_pad, n_pad, row_mul=1, row_add=0, codes=None, scales=None, stream=0):
    import torch
    K, N = w.shape
    if codes is None:
        codes = torch.zeros((n_pad, k_pad // 2), dtype=torch.uint8, device=w.device)
    if scales is None:
        scales = torch.zeros(n_pad, dtype=torch.float64, device=w.device)
    scratch = torch.zeros(max(N, 64), dtype=torch.float64, device=w.device)
    check(lib().qt_quant_weight_i4(_ptr(w), K, N, row_mul, row_add, _ptr(codes), codes.shape[0], _ptr(scales),
                                   _ptr(scratch), C.c_void_p(stream)))
    return codes, scales


def quota_topk(metrics, visual, budget, weights=None, stream=0):
    """K3c+K4 on device metrics [B x 4 x vstride] (fp64 cuda tensor): returns
    (slots list per sequence, fused [B x vstride], normalised [B x 4 x vstride]).
    weights=None: metrics[:, 0] already is the fused score (select_top_k alone)."""
    import torch
    B, _, vs = metrics.shape
    dev = metrics.device
    vis = torch.tensor(visual, dtype=torch.int32, device=dev)
    bud = torch.tensor(budget, dtype=torch.int32, device=dev)
    slots = torch.full((B, vs), -1, dtype=torch.int32, device=dev)
    fused = torch.zeros((B, vs), dtype=torch.float64, device=dev)
    norm = torch.zeros((B, 4, vs), dtype=torch.float64, device=dev)
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    check(lib().qt_quota_topk(_ptr(metrics.contiguous()), B, vs, _ptr(vis), _ptr(bud),
                              None if w is None else w.ctypes.data_as(C.POINTER(C.c_double)), _ptr(slots),
                              _ptr(fused), _ptr(norm), C.c_void_p(stream)))
    torch.cuda.current_stream(dev).synchronize() if stream == 0 else None
    s = slots.cpu().numpy()
    return [s[b, :min(budget[b], visual[b])].copy() for b in range(B)], fused, norm


def unpack_codes(tiled, rows, K, stream=0):
    """qt_unpack_codes: tiled int4 codes (torch uint8 cuda [rows_pad x K/2]) -> int8 [rows x K]."""
    import torch
    out = torch.empty((rows, K), dtype=torch.int8, device=tiled.device)
    check(lib().qt_unpack_codes(_ptr(tiled), tiled.shape[0], rows, K, _ptr(out), C.c_void_p(stream)))
    return out


def _dev_i32(a, device):
    import torch
    return torch.tensor(np.asarray(a, dtype=np.int32), dtype=torch.int32, device=device)


def attn_prefill(q, ldq, H, Hkv, d_head, seq_off, visual, seq_len, pool, page_bytes, page_table, max_pages, out,
                 row_stats=None, stream=0):
    """qt_attn_prefill_i4kv; int arrays given as device int32 tensors (or lists)."""
    dev = q.device
    so, vi, sl = (a if not isinstance(a, (list, tuple, np.ndarray)) else _dev_i32(a, dev)
                  for a in (seq_off, visual, seq_len))
    B = vi.numel()
    smax = int(sl.max().item())
    check(lib().qt_attn_prefill_i4kv(_ptr(q), ldq, B, H, Hkv, d_head, _ptr(so), _ptr(vi), _ptr(sl), smax, _ptr(pool),
                                     int(page_bytes), _ptr(page_table), max_pages, _ptr(out), out.stride(0),
                                     _ptr(row_stats), C.c_void_p(stream)))
    return out


def attn_decode(q, ldq, H, Hkv, d_head, kv_len, pool, page_bytes, page_table, max_pages, out, stream=0):
    """qt_attn_decode_i4kv over kv_len (list / device int32) cached rows per sequence."""
    import torch
    dev = q.device
    kl = kv_len if not isinstance(kv_len, (list, tuple, np.ndarray)) else _dev_i32(kv_len, dev)
    B = kl.numel()
    max_len = int(kl.max().item())
    ws = torch.empty(int(lib().qt_attn_decode_workspace(B, H, d_head, max_len)), dtype=torch.uint8, device=dev)
    check(lib().qt_attn_decode_i4kv(_ptr(q), ldq, B, H, Hkv, d_head, _ptr(kl), max_len, _ptr(pool), int(page_bytes),
                                    _ptr(page_table), max_pages, _ptr(out), out.stride(0), _ptr(ws),
                                    C.c_void_p(stream)))
    return out


def quota_score(x, q, ldq, H, Hkv, d_head, seq_off, visual, seq_len, pool, page_bytes, page_table, max_pages,
                row_stats, res_bits=4, vstride=None, stream=0):
    """qt_quota_score -> fp64 metrics [B x 4 x vstride] (mag, inter, intra, res)."""
    import torch
    dev = x.device
    so, vi, sl = (a if not isinstance(a, (list, tuple, np.ndarray)) else _dev_i32(a, dev)
                  for a in (seq_off, visual, seq_len))
    B = vi.numel()
    vmax = int(vi.max().item())
    vs = vstride or max(64, (vmax + 63) // 64 * 64)
    met = torch.zeros((B, 4, vs), dtype=torch.float64, device=dev)
    ws = torch.empty(int(lib().qt_quota_score_workspace(B, H, vs)), dtype=torch.uint8, device=dev)
    check(lib().qt_quota_score(_ptr(x), x.shape[1], _ptr(q), ldq, B, H, Hkv, d_head, _ptr(so), _ptr(vi), _ptr(sl),
                               vmax, _ptr(pool), int(page_bytes), _ptr(page_table), max_pages, _ptr(row_stats),
                               res_bits, _ptr(met), vs, _ptr(ws), C.c_void_p(stream)))
    return met


def topk_compact(metrics, visual, text, budget, weights, seq_off, x, pos, pool=None, page_bytes=0, page_table=None,
                 max_pages=0, Hkv=1, d_head=64, stream=0):
    """qt_topk_compact: returns (x_out, pos_out, kept slots per sequence, new_off)."""
    import torch
    dev = metrics.device
    B, _, vs = metrics.shape
    vis, txt, bud = (np.asarray(a, dtype=np.int32) for a in (visual, text, budget))
    nv = np.minimum(bud, vis)
    nlen = nv + txt
    noff = np.concatenate([[0], np.cumsum(nlen)]).astype(np.int32)
    rows = int(noff[-1])
    x_out = torch.zeros((max(rows, 1), x.shape[1]), dtype=torch.float64, device=dev)
    pos_out = torch.zeros(max(rows, 1), dtype=torch.int32, device=dev)
    kl = torch.zeros((B, vs), dtype=torch.int32, device=dev)
    ks = torch.zeros(max(rows, 1), dtype=torch.int32, device=dev)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    d = [_dev_i32(a, dev) for a in (vis, txt, bud, noff, nlen)]
    so = seq_off if not isinstance(seq_off, (list, tuple, np.ndarray)) else _dev_i32(seq_off, dev)
    check(lib().qt_topk_compact(_ptr(metrics.contiguous()), B, vs, _ptr(d[0]), _ptr(d[1]), _ptr(d[2]),
                                w.ctypes.data_as(C.POINTER(C.c_double)), _ptr(so), _ptr(d[3]), _ptr(d[4]), _ptr(x),
                                x.shape[1], _ptr(pos), rows, _ptr(x_out), _ptr(pos_out), _ptr(pool), int(page_bytes),
                                _ptr(page_table), max_pages, Hkv, d_head, _ptr(kl), _ptr(ks), None,
                                C.c_void_p(stream)))
    torch.cuda.synchronize(dev)
    k = kl.cpu().numpy()
    return x_out[:rows], pos_out[:rows], [k[b, :nv[b]].copy() for b in range(B)], noff


def rope_table(max_pos, d_head):
    out = np.empty((max_pos, d_head // 2, 2), dtype=np.float64)
    lib().qt_rope_table(max_pos, d_head, out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def unpack_i4(codes_u8, n):
    """Host helper for tests: packed int4 (low nibble first) -> int8 [.., n]."""
    c = np.asarray(codes_u8, dtype=np.uint8)
    lo = (c & 0xF).astype(np.int16)
    hi = (c >> 4).astype(np.int16)
    out = np.empty(c.shape[:-1] + (c.shape[-1] * 2,), dtype=np.int16)
    out[..., 0::2] = lo
    out[..., 1::2] = hi
    out = np.where(out >= 8, out - 16, out).astype(np.int8)
    return out[..., :n]


def exported_symbols():
    """Function names declared in include/quota_b200.h."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+char\*|int|int64_t|uint64_t|void)\s+(qt_\w+)\s*\(", txt,
                                 flags=re.M)))


def tile_w4(rows_u8):
    """Row-major packed int4 [rows_pad x K_pad/2] -> the engine's tiled layout (same shape):
    1 KB tiles of 16 rows x 64 bytes, k-block-major: tile (rt, kt) at (kt * rows_pad/16 + rt) * 1024."""
    a = np.ascontiguousarray(rows_u8, dtype=np.uint8)
    n, rb = a.shape
    assert n % 16 == 0 and rb % 64 == 0
    return a.reshape(n // 16, 16, rb // 64, 64).transpose(2, 0, 1, 3).reshape(n, rb).copy()


def untile_w4(tiled_u8, n, row_bytes):
    a = np.ascontiguousarray(tiled_u8, dtype=np.uint8).reshape(row_bytes // 64, n // 16, 16, 64)
    return a.transpose(1, 2, 0, 3).reshape(n, row_bytes).copy()
