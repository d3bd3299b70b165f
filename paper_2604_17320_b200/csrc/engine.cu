// engine.cu -- C++ host runtime of the QUOTA hot path + the C ABI
// (include/quota_b200.h).
//
// Restates the control flow of forward_prefill / decode_step
// (/root/reference/proj/src/model.cpp:315-562) and make_recipe_hook /
// apply_pruning (selector.cpp:138-228) for a batch of independent sequences
// packed back to back; every operator is a device kernel (k_*.cu), the host
// only schedules, allocates and tracks shapes.  All shapes after pruning are
// known on the host (budget = ceil(r * v0), selector.cpp:11-17), so a prefill
// never synchronises on device results; a decode step is captured once into a
// CUDA graph and replayed (its lengths and positions live in device memory).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>
#include <mutex>

#include "../../include/quota_b200.h"
#include "qt_common.cuh"
#include "qt_kernels.h"
#include <cublas_v2.h>

namespace {

thread_local std::string g_err;

struct QtError : std::runtime_error {
    int code;
    QtError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& msg) { throw QtError(code, msg); }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(QT_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
bool g_capturing = false;

void ckl(int rc, const char* what) {
    if (rc != 0) {
        cudaError_t e = cudaGetLastError();
        fail(rc > 0 ? QT_ECUDA : QT_EINVAL,
             std::string(what) + (rc > 0 ? std::string(": ") + cudaGetErrorString((cudaError_t)rc)
                                          : std::string(": unsupported shape")) +
                 (e != cudaSuccess ? std::string(" / ") + cudaGetErrorString(e) : std::string()));
    }
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return QT_OK;
    } catch (const QtError& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return QT_EINVAL;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return QT_ERANGE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return QT_ERUNTIME;
    }
}

int round_up(int x, int m) { return (x + m - 1) / m * m; }

template <class T>
T* dalloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    ck(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
    // cudaMemset runs on the legacy stream, which the engine's non-blocking stream does
    // not order against: finish it here, or a late zero-fill could land on data the
    // engine stream already wrote (e.g. a regrown weight-staging buffer)
    ck(cudaMemset(p, 0, n * sizeof(T)), "cudaMemset");
    ck(cudaDeviceSynchronize(), "cudaMemset");
    return static_cast<T*>(p);
}

struct LayerW {
    uint8_t* qkv = nullptr;
    double* s_qkv = nullptr;
    uint8_t* o = nullptr;
    double* s_o = nullptr;
    uint8_t* gu = nullptr;
    double* s_gu = nullptr;
    uint8_t* down = nullptr;
    double* s_down = nullptr;
    float* g1 = nullptr;
    float* g2 = nullptr;
    bool loaded = false;
    // int8 copies (16 x code, row-major, k natural) for the int8-operand prefill GEMM, made lazily
    int8_t *qkv8 = nullptr, *o8 = nullptr, *gu8 = nullptr, *down8 = nullptr;
    bool w8_ok = false;
};

// fp64 copies of the full-precision weights (reference orientation [d_in x d_out]),
// kept only when calibration is enabled (qt_engine_keep_fp_weights)
struct FpLayer {
    double* w[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // q k v o w1 w2 w3
};

struct Recipe {
    std::vector<int> layers;
    std::vector<double> keeps;
    double w[4] = {0.25, 0.45, 0.10, 0.20};
    int v0 = 64;
    int res_bits = 4;
};

struct PruneEv {
    int layer, budget;
    std::vector<int> positions;
};

// Per-launch CUDA-event profiler (bench.py roofline): kernel classes
enum ProfClass { P_GEMM = 0, P_ATTN = 1, P_QUANT = 2, P_KV = 3, P_SELECT = 4, P_OTHER = 5, P_NCLASS = 6 };

struct Profiler {
    struct Rec {
        int cls;
        cudaEvent_t a, b;
        double bytes, flops;
    };
    std::vector<Rec> recs;
    cudaStream_t st = nullptr;
    int open_cls = -1;
    cudaEvent_t open_ev = nullptr;
    void begin(int cls) {
        cudaEventCreate(&open_ev);
        cudaEventRecord(open_ev, st);
        open_cls = cls;
    }
    void end(double bytes, double flops) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        recs.push_back({open_cls, open_ev, e, bytes, flops});
        open_cls = -1;
    }
    // out[c*4 + {0,1,2,3}] = {ms, launches, bytes, flops}
    void read(double* out) {
        cudaStreamSynchronize(st);
        for (int i = 0; i < P_NCLASS * 4; ++i) out[i] = 0;
        for (auto& r : recs) {
            float ms = 0;
            cudaEventElapsedTime(&ms, r.a, r.b);
            out[r.cls * 4 + 0] += ms;
            out[r.cls * 4 + 1] += 1;
            out[r.cls * 4 + 2] += r.bytes;
            out[r.cls * 4 + 3] += r.flops;
        }
    }
    ~Profiler() {
        for (auto& r : recs) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
    }
};

}  // namespace

struct qt_engine {
    qt_config cfg{};
    int L = 0, d = 0, H = 0, Hkv = 0, dh = 0, dff = 0;
    int n_qkv = 0, n_qkv_pad = 0, kd_pad = 0, kff_pad = 0, n_gu = 0, n_gu_pad = 0, nd_pad = 0;
    int max_batch = 0, max_tokens = 0, max_seq = 0, max_decode = 0, max_pos = 0;
    cudaStream_t own_stream = nullptr, st = nullptr;
    // asynchronous host readback of prefill logits (qt_engine_prefill out_on_device = 2)
    cudaStream_t cst = nullptr;
    cudaEvent_t ev_lg = nullptr, ev_cp = nullptr;
    bool copy_pending = false;
    void join_copies() {  // order the engine stream after the pending readback
        if (!copy_pending) return;
        ck(cudaStreamWaitEvent(st, ev_cp, 0), "event wait");
        copy_pending = false;
        qt::g_pdl_block = true;
    }

    std::vector<LayerW> lw;
    uint8_t* head = nullptr;
    double* s_head = nullptr;
    float* gf = nullptr;
    bool head_loaded = false;
    std::vector<double> act;  // 4L + 1
    bool act_set = false;
    Recipe recipe;
    bool have_recipe = false;

    // activations (prefill capacity)
    double* x[2] = {nullptr, nullptr};  // fp64 residual stream
    int* pos[2] = {nullptr, nullptr};
    float* qkv = nullptr;
    float* attn = nullptr;
    float* mid = nullptr;
    uint8_t* codes = nullptr;
    int codes_rows = 0;  // padded rows of the tiled activation-code buffer
    double* ascale = nullptr;
    float* logits = nullptr;
    float* ml = nullptr;
    int* tok_seq = nullptr;
    int* tok_row = nullptr;
    int* seq_off = nullptr;  // [max_batch + 1]
    int* seq_vis = nullptr;
    int* seq_txt = nullptr;
    int* seq_len = nullptr;
    // scoring
    int vstride = 0;
    double* mag = nullptr;
    double* res = nullptr;
    float* inter = nullptr;
    float* intra = nullptr;
    double* w4 = nullptr;
    int* budget = nullptr;
    int* new_off = nullptr;
    int* new_len = nullptr;
    int* keep_src = nullptr;
    int* keep_local = nullptr;
    int* kept_pos = nullptr;
    double* sc_fused = nullptr;  // [L][mb][vstride] fused scores per prune event (parity readback)
    double* sc_norm = nullptr;   // [L][mb][4][vstride] robust-normalised metrics
    std::vector<int> ev_layers;               // candidate layers that ran selection, in order
    std::vector<std::vector<int>> ev_vis;     // visual count entering each event, per seq
    double* rope = nullptr;
    double* wscratch = nullptr;
    float* wstage = nullptr;
    size_t wstage_elems = 0;

    // KV cache
    uint8_t* pool = nullptr;
    long long page_bytes = 0;
    int n_pages_cap = 0;
    int max_pages = 0;       // per (layer, seq)
    int* pt = nullptr;       // [L][max_batch][max_pages]
    int* kv_len = nullptr;   // [L][max_batch]
    int* next_pos = nullptr; // [max_batch]
    int* dec_seq = nullptr;  // [max_batch] = 0..B-1

    // decode
    double* xd = nullptr;      // [max_batch x d] fp64 residual
    float* xd_in = nullptr;    // [max_batch x d] fp32 input staging
    float* dlogits = nullptr;  // [max_batch x d]
    float* part_ml = nullptr;
    float* part_o = nullptr;
    int dec_splits = 1, dec_pps = 1;   // the largest split plan over the layers (info)
    std::vector<int> dec_pages;        // cache pages per (layer, sequence) over the decode horizon
    std::vector<int> dec_lpps, dec_lsplit;  // decode-attention plan per layer (qt_attn_decode_plan)
    int n_sms = 148;
    cudaGraphExec_t graph = nullptr;
    bool graph_ok = false;
    // greedy decoding (qt_engine_decode_greedy): token-embedding table [vocab x d] fp32, the step's
    // tokens [max_batch], the prefill's last row per sequence; its own graph (argmax + embed first)
    float* tok_table = nullptr;
    int vocab = 0;
    int* dec_tok = nullptr;
    int* last_rows = nullptr;
    cudaGraphExec_t graph_g = nullptr;
    bool graph_g_ok = false;
    int decode_steps = 0;

    // host staging (pinned)
    char* pin = nullptr;
    size_t pin_cap = 0, pin_used = 0;

    // state of the last prefill
    int B = 0;
    int final_rows = 0;
    std::vector<int> h_vis, h_txt, h_off;
    std::vector<std::vector<int>> h_pos;  // final layout positions per seq
    std::vector<std::vector<PruneEv>> trace;
    std::vector<int> h_kvlen;             // [L][B]
    bool prefilled = false;
    static constexpr bool use_tc05 = true;  // tcgen05 GEMM for token-rich launches (M > 64)
    std::unique_ptr<Profiler> prof;      // active while profiling one call
    bool prof_next = false;
    double prof_out[P_NCLASS * 4] = {0};
    void pb(int cls) {
        if (prof) prof->begin(cls);
    }
    void pe(double bytes, double flops = 0) {
        if (prof) prof->end(bytes, flops);
    }
    std::vector<int> h_next;

    // full-precision calibration forward (k_fp.cu)
    bool keep_fp = false;
    std::vector<std::vector<double>>* rec_blocks = nullptr;  // block outputs of the next prefill (B = 1)
    // ForwardResult::records / block_outputs (model.cpp:382-402,439) and arbitrary host prune
    // hooks (model.cpp:404-405) for reference-API callers: B = 1, synchronous read-backs
    int rec_mode = 0;  // bit 1: block outputs, bit 2: layer records
    qt_prune_hook_fn host_hook = nullptr;
    void* host_user = nullptr;
    struct LayerRec {
        int layer, V, T;
        std::vector<int> pos;
        std::vector<double> states;  // [(V + T) x d]
        std::vector<float> probs;    // [H x (V + T) x V]
    };
    std::vector<LayerRec> lrecs;
    std::vector<std::vector<double>> blocks;
    float* probs_d = nullptr;
    size_t probs_cap = 0;
    // QUOTA diagnostics of the next prefill (B = 1, calibration only): per layer the text
    // queries' top-10 visual attention mass [H x T] and the visual-state cosine Gram [V x V]
    struct DiagRec {
        std::vector<std::vector<double>> top10, gram;
    };
    DiagRec* rec_diag = nullptr;
    std::vector<FpLayer> fpw;
    double* fp_head = nullptr;
    cublasHandle_t blas = nullptr;
    // int8-operand prefill GEMM (k_gemm_tc05_i8): activation codes as int8 next to the packed ones
    int8_t* codes8 = nullptr;
    int ld8 = 0;
    int8_t* head8 = nullptr;
    bool head8_ok = false;
    void ensure_w8() {
        auto conv = [&](const uint8_t* w, int rows, int K, int8_t*& dst) {
            if (!dst) dst = dalloc<int8_t>((size_t)rows * K);
            ckl(qt_launch_w4t_to_i8(w, rows, K, dst, st), "int8 weight copy");
        };
        for (auto& l : lw) {
            if (l.w8_ok) continue;
            conv(l.qkv, n_qkv_pad, kd_pad, l.qkv8);
            conv(l.o, nd_pad, kd_pad, l.o8);
            conv(l.gu, n_gu_pad, kd_pad, l.gu8);
            conv(l.down, nd_pad, kff_pad, l.down8);
            l.w8_ok = true;
        }
        if (!head8_ok) {
            conv(head, nd_pad, kd_pad, head8);
            head8_ok = true;
        }
        qt::g_pdl_block = true;
    }
    // per-row partial max |x| of the mlp_mid site left by the gate|up GEMM epilogue (act_mode 1)
    static constexpr int kPmaxLd = 512;
    static constexpr int kGemvMaxRows = 32;  // decode batches up to this many tokens: the int4 GEMV
    float* pmax = nullptr;
    int pm_parts = 0;
    float* pm_ptr = nullptr;  // where the last producer left them, row stride pm_ld
    int pm_ld = kPmaxLd;
    // decode: one atomically reduced max per (layer, token) from the gate|up GEMV (zeroed at the
    // end of every step) instead of one partial per GEMV CTA
    float* gmax = nullptr;
    int* splitk_ws = nullptr;     // int32 split-K partials of the tcgen05 GEMM at small M

    ~qt_engine() {
        if (cst) cudaStreamSynchronize(cst);  // a pending async logits readback still reads `logits`
        cudaStreamSynchronize(st ? st : 0);
        if (graph) cudaGraphExecDestroy(graph);
        if (graph_g) cudaGraphExecDestroy(graph_g);
        auto f = [](void* p) {
            if (p) cudaFree(p);
        };
        for (auto& l : lw) {
            f(l.qkv); f(l.s_qkv); f(l.o); f(l.s_o); f(l.gu); f(l.s_gu); f(l.down); f(l.s_down); f(l.g1); f(l.g2);
            f(l.qkv8); f(l.o8); f(l.gu8); f(l.down8);
        }
        f(head); f(s_head); f(gf);
        f(x[0]); f(x[1]); f(pos[0]); f(pos[1]); f(qkv); f(attn); f(mid); f(codes); f(ascale); f(logits); f(ml);
        f(tok_seq); f(tok_row); f(seq_off); f(seq_vis); f(seq_txt); f(seq_len);
        f(mag); f(res); f(inter); f(intra); f(w4); f(budget); f(new_off); f(new_len); f(keep_src); f(keep_local);
        f(kept_pos); f(sc_fused); f(sc_norm); f(rope); f(wscratch); f(wstage); f(pool); f(pt); f(kv_len); f(next_pos); f(dec_seq);
        f(xd); f(xd_in); f(dlogits); f(part_ml); f(part_o);
        for (auto& fl : fpw)
            for (double* p : fl.w) f(p);
        f(fp_head);
        if (blas) cublasDestroy(blas);
        f(splitk_ws); f(codes8); f(head8); f(pmax); f(gmax); f(probs_d);
        f(tok_table); f(dec_tok); f(last_rows);
        if (pin) cudaFreeHost(pin);
        if (cst) {
            cudaStreamSynchronize(cst);
            cudaStreamDestroy(cst);
            cudaEventDestroy(ev_lg);
            cudaEventDestroy(ev_cp);
        }
        if (own_stream) cudaStreamDestroy(own_stream);
    }

    // Host -> device copy ordered on the ENGINE stream and completed before returning.
    // (A plain cudaMemcpy/cudaMemset runs on the legacy stream, which the engine's
    // non-blocking stream does not wait for: a pageable cudaMemcpy may return before
    // its DMA lands, and a later kernel on `st` could read the old bytes.)
    void h2d(void* dst, const void* src, size_t bytes, const char* what) {
        ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st), what);
        ck(cudaStreamSynchronize(st), what);
    }

    // ------------------------------------------------------------ staging
    template <class T>
    T* stage(const T* src, size_t n) {
        size_t bytes = (n * sizeof(T) + 255) / 256 * 256;
        if (pin_used + bytes > pin_cap) fail(QT_EINVAL, "host staging buffer exhausted");
        T* p = reinterpret_cast<T*>(pin + pin_used);
        pin_used += bytes;
        std::memcpy(p, src, n * sizeof(T));
        return p;
    }
    template <class T>
    void upload(T* dst, const std::vector<T>& v) {
        if (v.empty()) return;
        T* p = stage(v.data(), v.size());
        ck(cudaMemcpyAsync(dst, p, v.size() * sizeof(T), cudaMemcpyHostToDevice, st), "upload");
        qt::g_pdl_block = true;
    }
    void reset_staging() {
        ck(cudaStreamSynchronize(st), "stream sync");
        pin_used = 0;
    }

    // ------------------------------------------------------------ setup
    void init(const qt_config& c, int mb, int mt, int ms, int md) {
        cfg = c;
        L = c.n_layers; d = c.d_model; H = c.n_heads; Hkv = c.n_kv_heads; dh = c.d_head; dff = c.d_ff;
        if (L < 1 || d < 8 || H < 1 || dh < 2) fail(QT_EINVAL, "invalid model config");
        if (dh % 2 != 0) fail(QT_EINVAL, "d_head must be even and >= 2");            // model.cpp:50-52
        if (d != H * dh) fail(QT_EINVAL, "d_model must equal n_heads * d_head");     // model.cpp:53-55
        if (dh != 64 && dh != 128) fail(QT_EINVAL, "d_head must be 64 or 128 on the B200 path");
        if (Hkv < 1 || H % Hkv != 0) fail(QT_EINVAL, "n_heads must be a multiple of n_kv_heads");
        if (c.weight_bits != 4 || c.act_bits != 4 || c.kv_bits != 4)
            fail(QT_EINVAL, "the B200 path implements W4A4KV4 only");
        if (c.mlp != 0 && c.mlp != 1) fail(QT_EINVAL, "mlp must be 0 (SiLU) or 1 (SwiGLU)");
        if (c.act_mode != 0 && c.act_mode != 1) fail(QT_EINVAL, "act_mode must be 0 (static) or 1 (dynamic)");
        if (d % 8 != 0 || dff % 8 != 0) fail(QT_EINVAL, "d_model and d_ff must be multiples of 8");
        max_batch = mb; max_tokens = mt; max_seq = ms; max_decode = md;
        if (mb < 1 || mt < 1 || ms < 1 || md < 0) fail(QT_EINVAL, "invalid capacity");
        n_qkv = (H + 2 * Hkv) * dh;
        n_qkv_pad = round_up(n_qkv, 128);
        kd_pad = round_up(d, 128);
        kff_pad = round_up(dff, 128);
        n_gu = c.mlp == 1 ? 2 * dff : dff;
        n_gu_pad = round_up(n_gu, 128);
        nd_pad = round_up(d, 128);
        max_pos = ms + md + 1;

        ck(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking), "stream");
        st = own_stream;
        lw.resize(L);
        for (auto& l : lw) {
            l.qkv = dalloc<uint8_t>((size_t)n_qkv_pad * kd_pad / 2);
            l.s_qkv = dalloc<double>(n_qkv_pad);
            l.o = dalloc<uint8_t>((size_t)nd_pad * kd_pad / 2);
            l.s_o = dalloc<double>(nd_pad);
            l.gu = dalloc<uint8_t>((size_t)n_gu_pad * kd_pad / 2);
            l.s_gu = dalloc<double>(n_gu_pad);
            l.down = dalloc<uint8_t>((size_t)nd_pad * kff_pad / 2);
            l.s_down = dalloc<double>(nd_pad);
            l.g1 = dalloc<float>(d);
            l.g2 = dalloc<float>(d);
        }
        head = dalloc<uint8_t>((size_t)nd_pad * kd_pad / 2);
        s_head = dalloc<double>(nd_pad);
        gf = dalloc<float>(d);

        const size_t T = mt;
        x[0] = dalloc<double>(T * d);
        x[1] = dalloc<double>(T * d);
        pos[0] = dalloc<int>(T);
        pos[1] = dalloc<int>(T);
        qkv = dalloc<float>(T * n_qkv);
        attn = dalloc<float>(T * d);
        mid = dalloc<float>(T * dff);
        codes_rows = round_up(std::max((int)T, mb), 16);
        codes = dalloc<uint8_t>((size_t)codes_rows * std::max(kd_pad, kff_pad) / 2);  // tiled rows
        if (std::max((int)T, mb) > kGemvMaxRows) {  // int8 activation copy for the tcgen05 GEMM
            ld8 = std::max(kd_pad, kff_pad);
            codes8 = dalloc<int8_t>((size_t)codes_rows * ld8);
        }
        ascale = dalloc<double>(T);
        logits = dalloc<float>(T * d);
        ml = dalloc<float>(T * H * 2);
        tok_seq = dalloc<int>(T);
        tok_row = dalloc<int>(T);
        seq_off = dalloc<int>(mb + 1);
        seq_vis = dalloc<int>(mb);
        seq_txt = dalloc<int>(mb);
        seq_len = dalloc<int>(mb);
        vstride = round_up(std::min(ms, mt), 64);
        mag = dalloc<double>((size_t)mb * vstride);
        res = dalloc<double>((size_t)mb * vstride);
        inter = dalloc<float>((size_t)mb * H * vstride);
        intra = dalloc<float>((size_t)mb * H * vstride);
        w4 = dalloc<double>(4);
        budget = dalloc<int>(mb);
        new_off = dalloc<int>(mb + 1);
        new_len = dalloc<int>(mb);
        keep_src = dalloc<int>(T);
        keep_local = dalloc<int>((size_t)mb * vstride);
        kept_pos = dalloc<int>((size_t)L * mb * vstride);
        sc_fused = dalloc<double>((size_t)L * mb * vstride);
        sc_norm = dalloc<double>((size_t)L * mb * 4 * vstride);
        wscratch = dalloc<double>(std::max({n_qkv_pad, n_gu_pad, nd_pad, kff_pad}) + 64);

        // RoPE table with the reference's own libm (model.cpp:156-168)
        std::vector<double> tab((size_t)max_pos * dh);
        qt_rope_table(max_pos, dh, tab.data());
        rope = dalloc<double>(tab.size());
        h2d(rope, tab.data(), tab.size() * sizeof(double), "rope upload");

        page_bytes = (long long)2 * Hkv * qt::kPage * (dh / 2 + 4);
        max_pages = (ms + md + qt::kPage - 1) / qt::kPage;
        pt = dalloc<int>((size_t)L * mb * max_pages);
        kv_len = dalloc<int>((size_t)L * mb);
        next_pos = dalloc<int>(mb);
        dec_seq = dalloc<int>(mb);
        xd = dalloc<double>((size_t)mb * d);
        xd_in = dalloc<float>((size_t)mb * d);
        dlogits = dalloc<float>((size_t)mb * d);
        dec_pps = 1;
        dec_splits = max_pages;  // splits never exceed the pages
        part_ml = dalloc<float>((size_t)mb * H * dec_splits * 2);
        part_o = dalloc<float>((size_t)mb * H * dec_splits * dh);
        {
            int dev = 0;
            ck(cudaGetDevice(&dev), "device");
            ck(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
        }
        {  // split-K workspace: the largest ksplit * M * N over the GEMM shapes that split
            const int shapes[5][2] = {{n_qkv, kd_pad}, {d, kd_pad}, {n_gu, kd_pad}, {d, kff_pad}, {d, kd_pad}};
            size_t need = 0;
            for (auto& sh : shapes)
                for (int m = 1; m <= std::min(mt, 128 * 148); m = (m < 1024 ? m + 1 : m + 128)) {
                    const int mm = std::min(m, mt);
                    const int ks = std::max(qt_tc05_splitk(mm, sh[0], sh[1]), qt_tc05_i8_splitk(mm, sh[0], sh[1]));
                    if (ks > 1) need = std::max(need, (size_t)ks * mm * sh[0]);
                }
            if (need) splitk_ws = dalloc<int>(need);
        }
        if (cfg.act_mode == 1) {
            pmax = dalloc<float>((size_t)std::max(mt, mb) * kPmaxLd);
            gmax = dalloc<float>((size_t)L * mb);
        }
        pin_cap = (size_t)64 << 20;
        pin_cap += (size_t)mt * (sizeof(int) * 8);
        ck(cudaMallocHost(&pin, pin_cap), "cudaMallocHost");
        ck(cudaDeviceSynchronize(), "init");  // every zero-fill of dalloc (legacy stream) has landed
    }

    // ------------------------------------------------------------ calibration (fp64 forward)
    // y[M x N] (+)= x[M x K] . W[K x N], all row-major fp64 (DGEMM on the transposed views)
    void dgemm(const double* x, int M, int K, const double* W, int N, double* y, int ldy, double beta) {
        const double one = 1.0;
        if (cublasDgemm(blas, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &one, W, N, x, K, &beta, y, ldy) !=
            CUBLAS_STATUS_SUCCESS)
            fail(QT_ECUDA, "cublasDgemm failed");
    }

    // Scratch of the fp64 forward (sized for the longest sample of one call).
    struct FpScratch {
        double *x = nullptr, *x2 = nullptr, *n = nullptr, *q = nullptr, *a = nullptr, *g = nullptr, *u = nullptr,
               *m = nullptr, *probs = nullptr, *met = nullptr;
        int *pos = nullptr, *pos2 = nullptr, *pid = nullptr;
        unsigned long long* obs = nullptr;
        void release() {
            for (void* p : {(void*)x, (void*)x2, (void*)n, (void*)q, (void*)a, (void*)g, (void*)u, (void*)m,
                            (void*)probs, (void*)met, (void*)pos, (void*)pos2, (void*)pid, (void*)obs})
                if (p) cudaFree(p);
            *this = FpScratch{};
        }
    };

    // hook_vmax > 0: the recipe hook runs, on visual prefixes up to hook_vmax tokens
    void fp_setup(FpScratch& fs, int smax, int hook_vmax = 0) {
        if (!keep_fp || fpw.empty() || !fp_head) fail(QT_EINVAL, "calibration needs the full-precision weights "
                                                                 "(qt_engine_keep_fp_weights before loading)");
        if (!blas && cublasCreate(&blas) != CUBLAS_STATUS_SUCCESS) fail(QT_ECUDA, "cublasCreate failed");
        cublasSetStream(blas, st);
        if (smax > max_pos - max_decode - 1) fail(QT_EINVAL, "sample longer than the engine's RoPE table");
        if (hook_vmax > vstride) fail(QT_EINVAL, "visual prefix exceeds engine capacity");
        const size_t S = smax;
        fs.x = dalloc<double>(S * d);
        fs.n = dalloc<double>(S * d);
        fs.q = dalloc<double>(S * n_qkv);
        fs.a = dalloc<double>(S * d);
        fs.g = dalloc<double>(S * dff);
        fs.u = cfg.mlp == 1 ? dalloc<double>(S * dff) : nullptr;
        fs.m = dalloc<double>(S * dff);
        fs.pos = dalloc<int>(S);
        fs.pid = dalloc<int>(S);
        fs.obs = dalloc<unsigned long long>(4 * L + 1);
        if (hook_vmax > 0) {
            fs.x2 = dalloc<double>(S * d);
            fs.pos2 = dalloc<int>(S);
            fs.probs = dalloc<double>((size_t)H * S * hook_vmax);
            fs.met = dalloc<double>((size_t)4 * vstride);
        }
        std::vector<int> hp(S);
        for (size_t i = 0; i < S; ++i) hp[i] = (int)i;
        h2d(fs.pid, hp.data(), S * sizeof(int), "positions");
    }

    // what a hooked / logits-producing fp64 forward reports (forward_prefill in ExecMode::Fp)
    struct FpOut {
        bool hook = false;                     // options.hook = make_recipe_hook(recipe, ...)
        std::vector<PruneEv>* trace = nullptr;  // ForwardResult::prune_trace
        std::vector<int>* positions = nullptr;  // final_layout.position_ids
        int* visual = nullptr;                  // final_layout.visual_count
        std::vector<double>* logits = nullptr;  // ForwardResult::logits
    };

    // forward_prefill in ExecMode::Fp (model.cpp:315-453) for one sample, fp64; max|x| per
    // site into fs.obs (ActStats, model.cpp:348,393,430,434,443); blocks (optional) gets the
    // post-block hidden states (ForwardResult::block_outputs, model.cpp:439).  With o->hook the
    // engine's recipe prunes at its candidate layers exactly as make_recipe_hook does
    // (selector.cpp:211-228): compute_metrics on the fp64 record (model.cpp:382-402), the
    // device robust-normalise + top-k, and the row compaction of apply_pruning (model.cpp:404-427).
    void fp_forward(FpScratch& fs, const double* emb, int V, int T, std::vector<std::vector<double>>* blocks,
                    const FpOut* o = nullptr) {
        const int kvd = Hkv * dh, ldq = n_qkv;
        const bool hook = o && o->hook;
        reset_staging();
        double *xc = fs.x, *xo = fs.x2;
        int *pc = fs.pos, *po = fs.pos2;
        h2d(xc, emb, (size_t)(V + T) * d * sizeof(double), "calibration sample");
        ck(cudaMemcpyAsync(pc, fs.pid, (size_t)(V + T) * sizeof(int), cudaMemcpyDeviceToDevice, st), "positions");
        if (blocks) blocks->assign(L, {});
        if (o && o->trace) o->trace->clear();
        std::vector<int> hpos(V + T);
        for (int i = 0; i < V + T; ++i) hpos[i] = i;
        int v = V;
        for (int l = 0; l < L; ++l) {
            const FpLayer& fl = fpw[l];
            const int Sq = v + T;
            int K = -1;  // budget when l is a candidate layer of the hook's recipe
            if (hook)
                for (size_t i = 0; i < recipe.layers.size(); ++i)
                    if (recipe.layers[i] == l) K = (int)std::ceil(recipe.keeps[i] * (double)recipe.v0);
            if (K >= 0 && v == 0) fail(QT_EINVAL, "empty sample");  // robust_normalize, selector.cpp:70-71
            const bool prune = K >= 0 && K < v;
            ckl(qt_launch_fp_rmsnorm(xc, lw[l].g1, Sq, d, fs.n, fs.obs + 4 * l + 0, st), "fp rmsnorm");
            dgemm(fs.n, Sq, d, fl.w[0], d, fs.q, ldq, 0.0);
            dgemm(fs.n, Sq, d, fl.w[1], kvd, fs.q + d, ldq, 0.0);
            dgemm(fs.n, Sq, d, fl.w[2], kvd, fs.q + d + kvd, ldq, 0.0);
            ckl(qt_launch_fp_rope(fs.q, ldq, Sq, H + Hkv, dh, pc, rope, st), "fp rope");
            ckl(qt_launch_fp_attention(fs.q, ldq, H, Hkv, dh, Sq, v, fs.a, d, fs.obs + 4 * l + 1,
                                       prune ? fs.probs : nullptr, st),
                "fp attention");
            dgemm(fs.a, Sq, d, fl.w[3], d, xc, d, 1.0);  // x += attn . Wo
            int S2 = Sq;
            if (prune) {
                double* met = fs.met;
                const std::vector<int> zero{0}, vv{v}, tt{T}, kk{K};
                upload(seq_off, zero);
                upload(new_off, zero);
                upload(seq_vis, vv);
                upload(seq_txt, tt);
                upload(budget, kk);
                ckl(qt_launch_token_metrics(xc, d, seq_off, seq_vis, v, 1, vstride, recipe.res_bits, met,
                                            met + 3 * vstride, st),
                    "fp token metrics");
                ckl(qt_launch_fp_colsum(fs.probs, H, Sq, v, met + vstride, met + 2 * vstride, st),
                    "fp attention metrics");
                ckl(qt_launch_select_topk(nullptr, nullptr, nullptr, nullptr, H, vstride, seq_vis, seq_txt, budget,
                                          seq_off, new_off, 1, v, recipe.w, keep_src, keep_local, vstride, pc,
                                          kept_pos, nullptr, nullptr, met, 0, st),
                    "quota top-k");
                S2 = K + T;
                ckl(qt_launch_gather_rows(xc, xo, d, pc, po, keep_src, S2, st), "compaction gather");
                std::swap(xc, xo);
                std::swap(pc, po);
                PruneEv e{l, K, std::vector<int>(K)};
                ck(cudaMemcpyAsync(e.positions.data(), kept_pos, K * sizeof(int), cudaMemcpyDeviceToHost, st),
                   "trace");
                ck(cudaStreamSynchronize(st), "trace");
                std::vector<int> np(e.positions);
                np.insert(np.end(), hpos.begin() + v, hpos.end());
                hpos = np;
                if (o->trace) o->trace->push_back(std::move(e));
                v = K;
            }
            ckl(qt_launch_fp_rmsnorm(xc, lw[l].g2, S2, d, fs.n, fs.obs + 4 * l + 2, st), "fp rmsnorm");
            dgemm(fs.n, S2, d, fl.w[4], dff, fs.g, dff, 0.0);
            if (fs.u) dgemm(fs.n, S2, d, fl.w[6], dff, fs.u, dff, 0.0);
            ckl(qt_launch_fp_mlp_act(fs.g, fs.u, (long long)S2 * dff, fs.m, fs.obs + 4 * l + 3, st), "fp mlp");
            dgemm(fs.m, S2, dff, fl.w[5], d, xc, d, 1.0);  // x += mid . W2
            if (blocks) {
                (*blocks)[l].resize((size_t)S2 * d);
                ck(cudaMemcpyAsync((*blocks)[l].data(), xc, (size_t)S2 * d * sizeof(double), cudaMemcpyDeviceToHost,
                                   st),
                   "block output");
            }
        }
        const int Sf = v + T;
        ckl(qt_launch_fp_rmsnorm(xc, gf, Sf, d, fs.n, fs.obs + 4 * L, st), "fp final norm");
        if (o && o->logits) {  // logits = final_norm . W_head (model.cpp:442-445)
            dgemm(fs.n, Sf, d, fp_head, d, fs.a, d, 0.0);
            o->logits->resize((size_t)Sf * d);
            ck(cudaMemcpyAsync(o->logits->data(), fs.a, (size_t)Sf * d * sizeof(double), cudaMemcpyDeviceToHost, st),
               "fp logits");
        }
        if (o && o->positions) *o->positions = hpos;
        if (o && o->visual) *o->visual = v;
        ck(cudaStreamSynchronize(st), "fp forward");
    }

    // fit_act_scales (calibrator.cpp:237-249): full-precision forwards of the samples with
    // an ActStats collector; returns max|x| / qmax per site (0 -> 1.0, model.cpp:198-210).
    // hook: the forwards run under the engine's recipe (the prune_then_quant calibration,
    // harness.cpp:103-106).
    void fit_act_scales(int n, const double* const* embs, const int* vis, const int* txt, double* out,
                        bool hook = false) {
        if (n < 1) fail(QT_EINVAL, "no calibration samples");  // calibrator.cpp:239
        if (hook && !have_recipe) fail(QT_EINVAL, "no recipe set");
        int smax = 0, vmax = 0;
        for (int i = 0; i < n; ++i) {
            if (vis[i] < 0 || txt[i] < 0 || vis[i] + txt[i] < 1) fail(QT_EINVAL, "invalid sample layout");
            smax = std::max(smax, vis[i] + txt[i]);
            vmax = std::max(vmax, vis[i]);
        }
        FpScratch fs;
        try {
            fp_setup(fs, smax, hook ? std::max(vmax, 1) : 0);
            FpOut fo;
            fo.hook = hook;
            for (int i = 0; i < n; ++i) fp_forward(fs, embs[i], vis[i], txt[i], nullptr, &fo);
            std::vector<unsigned long long> hm(4 * L + 1);
            ck(cudaMemcpyAsync(hm.data(), fs.obs, hm.size() * 8, cudaMemcpyDeviceToHost, st), "stats");
            ck(cudaStreamSynchronize(st), "stats");
            for (size_t i = 0; i < hm.size(); ++i) {
                double mxv;
                std::memcpy(&mxv, &hm[i], 8);
                out[i] = mxv == 0.0 ? 1.0 : mxv / 7.0;  // qmax at 4 act bits
            }
        } catch (...) {
            fs.release();
            throw;
        }
        fs.release();
    }

    // forward_prefill in ExecMode::Fp (model.cpp:315-453) of n independent samples, fp64 on the
    // device; hook: under the engine's recipe (make_recipe_hook, selector.cpp:211-228).  The
    // logits of each sample's final layout are concatenated into logits_out (cap_rows rows of
    // d); trace and final layout are readable with qt_engine_n_prunes / prune / layout.  The
    // fp64 forward keeps no device KV cache: qt_engine_decode after it fails.
    void prefill_fp(int n, const double* const* embs, const int* vis, const int* txt, bool hook, double* logits_out,
                    long long cap_rows) {
        for (auto& l : lw)
            if (!l.loaded) fail(QT_EINVAL, "model weights not loaded");
        if (!head_loaded) fail(QT_EINVAL, "model head not loaded");
        if (n < 1 || n > max_batch) fail(QT_EINVAL, "batch size outside engine capacity");
        if (hook && !have_recipe) fail(QT_EINVAL, "no recipe set");
        int smax = 0, vmax = 0;
        for (int i = 0; i < n; ++i) {
            if (vis[i] < 0 || txt[i] < 0) fail(QT_EINVAL, "negative token count");
            if (vis[i] + txt[i] < 1) fail(QT_EINVAL, "empty sequence");
            smax = std::max(smax, vis[i] + txt[i]);
            vmax = std::max(vmax, vis[i]);
        }
        graph_ok = false;
        prefilled = false;
        ev_layers.clear();
        ev_vis.clear();
        FpScratch fs;
        try {
            fp_setup(fs, smax, hook ? std::max(vmax, 1) : 0);
            B = n;
            h_txt.assign(txt, txt + n);
            h_vis.assign(n, 0);
            h_pos.assign(n, {});
            trace.assign(n, {});
            long long rows = 0;
            std::vector<double> lg;
            for (int i = 0; i < n; ++i) {
                FpOut fo;
                fo.hook = hook;
                fo.trace = &trace[i];
                fo.positions = &h_pos[i];
                fo.visual = &h_vis[i];
                fo.logits = &lg;
                fp_forward(fs, embs[i], vis[i], txt[i], nullptr, &fo);
                const long long r = (long long)lg.size() / d;
                if (logits_out) {
                    if (rows + r > cap_rows) fail(QT_EINVAL, "buffer too small");
                    std::memcpy(logits_out + rows * d, lg.data(), lg.size() * sizeof(double));
                }
                rows += r;
            }
            final_rows = (int)rows;
        } catch (...) {
            fs.release();
            throw;
        }
        fs.release();
    }

    // percentile (numeric.cpp:84-96) on a copy
    static double pctl(std::vector<double> v, double p) {
        if (v.empty()) fail(QT_EINVAL, "empty sample");
        std::sort(v.begin(), v.end());
        if (v.size() == 1) return v[0];
        const double hh = p / 100.0 * (double)(v.size() - 1);
        const size_t lo = (size_t)std::floor(hh), hi = std::min(lo + 1, v.size() - 1);
        return v[lo] + (hh - (double)lo) * (v[hi] - v[lo]);
    }

    // profile_sensitivity (calibrator.cpp:42-82): per listed layer, the median over samples of
    // ||x_q - x|| / (||x|| + eta) between the quantized (this engine) and fp64 block outputs,
    // then normalize_sensitivities (calibrator.cpp:84-98)
    void profile_sensitivity(int n, const double* const* embs, const int* vis, const int* txt, int nl,
                             const int* layers, double eta, double* raw, double* normd) {
        if (n < 1) fail(QT_EINVAL, "no calibration samples");
        if (nl < 1) fail(QT_EINVAL, "no layers to profile");
        for (int i = 0; i < nl; ++i)
            if (layers[i] < 0 || layers[i] >= L) fail(QT_EINVAL, "layer out of range");
        if (cfg.act_mode == 0 && !act_set) fail(QT_EINVAL, "quantized mode requires a QuantEnv");
        int smax = 0;
        for (int i = 0; i < n; ++i) {
            if (vis[i] < 0 || txt[i] < 0 || vis[i] + txt[i] < 1) fail(QT_EINVAL, "invalid sample layout");
            smax = std::max(smax, vis[i] + txt[i]);
        }
        std::vector<std::vector<double>> dev(nl);
        FpScratch fs;
        const bool had_recipe = have_recipe;
        have_recipe = false;  // no hook: the block outputs of unpruned forwards
        try {
            fp_setup(fs, smax);
            std::vector<std::vector<double>> fb, qb;
            std::vector<float> emb32;
            for (int i = 0; i < n; ++i) {
                const int Sq = vis[i] + txt[i];
                fp_forward(fs, embs[i], vis[i], txt[i], &fb);
                rec_blocks = &qb;
                prefill(1, embs[i], 0, 1, &vis[i], &txt[i], nullptr, nullptr, nullptr, 0);
                rec_blocks = nullptr;
                for (int k = 0; k < nl; ++k) {
                    const std::vector<double>& x = fb[layers[k]];
                    const std::vector<double>& xq = qb[layers[k]];
                    if (xq.size() != (size_t)Sq * d) fail(QT_ERUNTIME, "block output shape mismatch");
                    double acc = 0.0, nn = 0.0;
                    for (size_t j = 0; j < x.size(); ++j) {
                        const double df = xq[j] - x[j];
                        acc += df * df;  // l2_distance, numeric.cpp:61-71
                        nn += x[j] * x[j];  // frobenius_norm
                    }
                    dev[k].push_back(std::sqrt(acc) / (std::sqrt(nn) + eta));
                }
            }
        } catch (...) {
            rec_blocks = nullptr;
            have_recipe = had_recipe;
            fs.release();
            throw;
        }
        have_recipe = had_recipe;
        fs.release();
        std::vector<double> r(nl);
        for (int k = 0; k < nl; ++k) r[k] = raw[k] = pctl(dev[k], 50.0);  // median
        const double p10 = pctl(r, 10.0), p90 = pctl(r, 90.0);
        for (int k = 0; k < nl; ++k)
            normd[k] = p90 - p10 < 1e-12 ? 0.5 : std::clamp((r[k] - p10) * (1.0 / (p90 - p10)), 0.1, 0.9);
    }

    // one layer's diagnostics record (LayerActivationRecord, model.cpp:382-402) for B = 1
    void diag_layer(int l, const int* ptl, int V, int T, const double* x) {
        if (l == 0) {
            rec_diag->top10.assign(L, {});
            rec_diag->gram.assign(L, {});
        }
        const int S = V + T;
        if (T > 0 && V > 0) {
            double* dt = dalloc<double>((size_t)H * T);
            ckl(qt_launch_diag_top10(qkv, n_qkv, H, Hkv, dh, V, S, pool, page_bytes, ptl, dt, st), "diag top-10");
            rec_diag->top10[l].resize((size_t)H * T);
            ck(cudaMemcpyAsync(rec_diag->top10[l].data(), dt, (size_t)H * T * 8, cudaMemcpyDeviceToHost, st), "diag");
            ck(cudaStreamSynchronize(st), "diag");
            cudaFree(dt);
        }
        if (V >= 2) {  // Gram of the visual rows of the post-attention residual (fp64 DGEMM)
            if (!blas && cublasCreate(&blas) != CUBLAS_STATUS_SUCCESS) fail(QT_ECUDA, "cublasCreate failed");
            cublasSetStream(blas, st);
            double* g = dalloc<double>((size_t)V * V);
            const double one = 1.0, zero = 0.0;
            if (cublasDgemm(blas, CUBLAS_OP_T, CUBLAS_OP_N, V, V, d, &one, x, d, x, d, &zero, g, V) !=
                CUBLAS_STATUS_SUCCESS)
                fail(QT_ECUDA, "cublasDgemm failed");
            rec_diag->gram[l].resize((size_t)V * V);
            ck(cudaMemcpyAsync(rec_diag->gram[l].data(), g, (size_t)V * V * 8, cudaMemcpyDeviceToHost, st), "diag");
            ck(cudaStreamSynchronize(st), "diag");
            cudaFree(g);
        }
    }

    // profile_diagnostics (calibrator.cpp:147-195) with this engine's quantized forward:
    // per layer, over samples, the median / IQR of the text queries' top-10 visual mass
    // (averaged over heads and text rows) and the median of the visual rows' median
    // pairwise cosine (numeric.cpp:117-127)
    void profile_diagnostics(int n, const double* const* embs, const int* vis, const int* txt, double* conc_med,
                             double* conc_iqr, double* red_med) {
        if (n < 1) fail(QT_EINVAL, "no calibration samples");
        if (cfg.act_mode == 0 && !act_set) fail(QT_EINVAL, "quantized mode requires a QuantEnv");
        std::vector<std::vector<double>> conc(L), red(L);
        const bool had_recipe = have_recipe;
        have_recipe = false;
        DiagRec dr;
        try {
            for (int i = 0; i < n; ++i) {
                if (vis[i] < 2) fail(QT_EINVAL, "need at least two token rows");  // numeric.cpp:118
                rec_diag = &dr;
                prefill(1, embs[i], 0, 1, &vis[i], &txt[i], nullptr, nullptr, nullptr, 0);
                rec_diag = nullptr;
                const int V = vis[i], T = txt[i];
                for (int l = 0; l < L; ++l) {
                    double total = 0.0;
                    for (double v : dr.top10[l]) total += v;  // heads, then text rows
                    conc[l].push_back(T == 0 ? 0.0 : total / (double)(H * T));
                    const std::vector<double>& g = dr.gram[l];
                    std::vector<double> sims;
                    sims.reserve((size_t)V * (V - 1) / 2);
                    for (int a = 0; a < V; ++a) {
                        const double na = std::sqrt(g[(size_t)a * V + a]);
                        for (int b = a + 1; b < V; ++b) {
                            const double nb = std::sqrt(g[(size_t)b * V + b]);
                            if (na == 0.0 || nb == 0.0) fail(QT_EINVAL, "degenerate token");  // numeric.cpp:80
                            sims.push_back(g[(size_t)a * V + b] / (na * nb));
                        }
                    }
                    red[l].push_back(pctl(sims, 50.0));
                }
            }
        } catch (...) {
            rec_diag = nullptr;
            have_recipe = had_recipe;
            throw;
        }
        have_recipe = had_recipe;
        for (int l = 0; l < L; ++l) {
            conc_med[l] = pctl(conc[l], 50.0);
            conc_iqr[l] = pctl(conc[l], 75.0) - pctl(conc[l], 25.0);
            red_med[l] = pctl(red[l], 50.0);
        }
    }

    void ensure_pool(int pages) {
        if (pages <= n_pages_cap) return;
        ck(cudaStreamSynchronize(st), "sync");
        if (pool) cudaFree(pool);
        pool = nullptr;
        n_pages_cap = 0;
        void* p = nullptr;
        ck(cudaMalloc(&p, (size_t)pages * page_bytes), "KV pool cudaMalloc");
        ck(cudaMemsetAsync(p, 0, (size_t)pages * page_bytes, st), "KV pool memset");  // ordered on the engine stream
        qt::g_pdl_block = true;
        pool = static_cast<uint8_t*>(p);
        n_pages_cap = pages;
    }

    const float* to_device_f32(const float* src, size_t n, int on_device, float* slot_hint) {
        if (on_device) return src;
        (void)slot_hint;
        if (n > wstage_elems) {
            if (wstage) cudaFree(wstage);
            wstage = dalloc<float>(n);
            wstage_elems = n;
        }
        ck(cudaMemcpyAsync(wstage, src, n * sizeof(float), cudaMemcpyHostToDevice, st), "weight upload");
        return wstage;
    }

    void quant_into(const float* w, int K, int N, int on_device, int row_mul, int row_add, uint8_t* codes_dst,
                    int rows_pad, double* scales_dst) {
        const float* dw = to_device_f32(w, (size_t)K * N, on_device, nullptr);
        ckl(qt_launch_weight_quant(dw, K, N, 4, row_mul, row_add, codes_dst, rows_pad, scales_dst, wscratch, st),
            "weight quantize");
        ck(cudaStreamSynchronize(st), "weight quantize");
    }

    // fp64 copy of a full-precision weight for the calibration forward
    void keep64(double*& dst, const float* w, size_t n, int on_device) {
        if (!keep_fp || !w) return;
        const float* dw = to_device_f32(w, n, on_device, nullptr);
        if (!dst) dst = dalloc<double>(n);
        ckl(qt_launch_f32_to_f64(dw, dst, (long long)n, st), "fp64 weight copy");
        ck(cudaStreamSynchronize(st), "fp64 weight copy");
    }

    // pre-quantized codes (host int8 [K x N], reference orientation) + fp64 per-column scales
    void codes_into(const int8_t* c, const double* sc, int K, int N, int row_mul, int row_add, uint8_t* codes_dst,
                    int rows_pad, double* scales_dst) {
        if (!c || !sc) fail(QT_EINVAL, "null weight codes");
        const size_t n = (size_t)K * N;
        if ((n + 3) / 4 > wstage_elems) {
            if (wstage) cudaFree(wstage);
            wstage = dalloc<float>((n + 3) / 4);
            wstage_elems = (n + 3) / 4;
        }
        for (size_t i = 0; i < n; ++i)
            if (c[i] < -7 || c[i] > 7) fail(QT_EINVAL, "weight code outside the int4 range");
        for (int i = 0; i < N; ++i)
            if (!(sc[i] > 0.0) || !std::isfinite(sc[i])) fail(QT_EINVAL, "weight scales must be positive");
        ck(cudaMemcpyAsync(wstage, c, n, cudaMemcpyHostToDevice, st), "codes upload");
        ck(cudaMemcpyAsync(wscratch, sc, (size_t)N * sizeof(double), cudaMemcpyHostToDevice, st), "scales upload");
        ckl(qt_launch_codes_pack(reinterpret_cast<const int8_t*>(wstage), K, N, wscratch, row_mul, row_add,
                                 codes_dst, rows_pad, scales_dst, st),
            "codes pack");
        ck(cudaStreamSynchronize(st), "codes pack");
    }
    void load_gain64(float* dst, const double* g) {
        std::vector<float> v(d, 1.0f);
        if (g)
            for (int i = 0; i < d; ++i) v[i] = (float)g[i];
        h2d(dst, v.data(), d * sizeof(float), "gain");
    }

    void load_gain(float* dst, const float* g, int on_device) {
        if (!g) {
            std::vector<float> ones(d, 1.0f);
            h2d(dst, ones.data(), d * sizeof(float), "gain");
            return;
        }
        ck(cudaMemcpyAsync(dst, g, d * sizeof(float), on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st),
           "gain");
        ck(cudaStreamSynchronize(st), "gain");
    }

    // ------------------------------------------------------------ decision capture
    // Debug / parity mode (qt_engine_capture): after every quantizer site of a prefill or
    // decode step, the int4 codes and scales are read back (synchronously; decode runs
    // eagerly, not from the graph).  Sites: 0 attn_in, 1 attn_out, 2 mlp_in, 3 mlp_mid,
    // 4 head_in (layer = n_layers), 5 K and 6 V cache rows (groups = kv heads); phase 0 =
    // prefill, 1 + t = decode step t.  The parity tests compare them with the restatement's
    // decisions (oracle/quota_oracle.cpp dec_key) -- the product path never enables it.
    struct CapRec {
        int phase, layer, site, rows, cols, groups;
        std::vector<int8_t> codes;   // rows x cols
        std::vector<double> scales;  // rows x groups
    };
    bool capture = false;
    std::vector<CapRec> caps;
    int cap_phase() const { return prefilled ? 1 + decode_steps : 0; }
    void cap_site(int layer, int site, int M, int D, int dpad) {
        if (!capture) return;
        ck(cudaStreamSynchronize(st), "capture");
        std::vector<uint8_t> t((size_t)codes_rows * dpad / 2);
        ck(cudaMemcpy(t.data(), codes, t.size(), cudaMemcpyDeviceToHost), "capture codes");
        CapRec r{cap_phase(), layer, site, M, D, 1, std::vector<int8_t>((size_t)M * D), std::vector<double>(M)};
        ck(cudaMemcpy(r.scales.data(), ascale, (size_t)M * sizeof(double), cudaMemcpyDeviceToHost), "capture scales");
        for (int m = 0; m < M; ++m)
            for (int k = 0; k < D; ++k) {
                const int nibv = (t[qt::w4t_offset(m, k / 2, codes_rows)] >> (4 * (k & 1))) & 0xF;
                r.codes[(size_t)m * D + k] = (int8_t)(nibv >= 8 ? nibv - 16 : nibv);
            }
        caps.push_back(std::move(r));
    }
    // K / V rows [row0[b], row0[b] + n[b]) of every sequence at `layer`, packed by sequence
    void cap_kv(int layer, const std::vector<int>& row0, const std::vector<int>& n) {
        if (!capture) return;
        ck(cudaStreamSynchronize(st), "capture");
        int M = 0;
        for (int v : n) M += v;
        const int cols = Hkv * dh;
        const size_t cb = (size_t)Hkv * qt::kPage * (dh / 2);
        std::vector<int> hpt(max_pages);
        std::vector<uint8_t> page(page_bytes);
        for (int which = 0; which < 2; ++which) {
            CapRec r{cap_phase(), layer, 5 + which, M, cols, Hkv, std::vector<int8_t>((size_t)M * cols),
                     std::vector<double>((size_t)M * Hkv)};
            int o = 0;
            for (int b = 0; b < B; ++b) {
                ck(cudaMemcpy(hpt.data(), pt + ((size_t)layer * max_batch + b) * max_pages, max_pages * sizeof(int),
                              cudaMemcpyDeviceToHost),
                   "capture page table");
                int cur = -1;
                for (int i = 0; i < n[b]; ++i, ++o) {
                    const int row = row0[b] + i;
                    if (row / qt::kPage != cur) {
                        cur = row / qt::kPage;
                        ck(cudaMemcpy(page.data(), pool + (long long)hpt[cur] * page_bytes, page_bytes,
                                      cudaMemcpyDeviceToHost),
                           "capture page");
                    }
                    const int slot = row % qt::kPage;
                    const float* sc = reinterpret_cast<const float*>(page.data() + 2 * cb);
                    for (int h = 0; h < Hkv; ++h) {
                        const uint8_t* src = page.data() + (which ? cb : 0) + ((size_t)h * qt::kPage + slot) * (dh / 2);
                        for (int c = 0; c < dh; ++c) {
                            const int nibv = (src[c / 2] >> (4 * (c & 1))) & 0xF;
                            r.codes[(size_t)o * cols + h * dh + c] = (int8_t)(nibv >= 8 ? nibv - 16 : nibv);
                        }
                        r.scales[(size_t)o * Hkv + h] = sc[(which ? Hkv * qt::kPage : 0) + h * qt::kPage + slot];
                    }
                }
            }
            caps.push_back(std::move(r));
        }
    }

    // ------------------------------------------------------------ kernels
    // from_pmax: the site input is the fp32 output of the last gemm(), whose epilogue left the
    // per-row partial maxima in pmax (pm_parts > 0): quantize without a row reduction
    void norm_quant(const void* xin, int is_f64, int ldx, const float* gain, int M, int D, int dpad, int site_idx,
                    bool from_pmax = false) {
        const int mode = cfg.act_mode;
        const double s = mode == 0 ? act[site_idx] : 0.0;
        pb(P_QUANT);
        int8_t* c8 = i8_rows(M) ? codes8 : nullptr;  // the next GEMM runs on int8 operands
        if (from_pmax && pm_parts > 0 && !is_f64 && !gain && mode == 1)
            ckl(qt_launch_quant_pmax(static_cast<const float*>(xin), ldx, pm_ptr, pm_parts, pm_ld, M, D, dpad, 7, mode,
                                     s, codes, codes_rows, ascale, c8, ld8, st),
                "quant (producer row max)");
        else
            ckl(qt_launch_norm_quant(xin, is_f64, ldx, gain, M, D, dpad, 4, mode, s, codes, codes_rows, ascale,
                                     nullptr, c8, ld8, st),
                "rmsnorm+quant");
        pe((double)M * D * (is_f64 ? 8 : 4) + (double)M * dpad / 2 + 8.0 * M);
    }
    // the int8-operand tcgen05 GEMM serves this many token rows (activation codes8 written)
    bool i8_rows(int M) const { return use_tc05 && codes8 && M > kGemvMaxRows; }
    // w: tiled int4 weights with wrows padded rows; activation codes: tiled with codes_rows rows
    // want_pm: also leave the per-row partial max |out| in pmax (pm_parts slots; 0 = not produced)
    void gemm(int epi, const uint8_t* w, int wrows, const double* sw, int M, int N, int K, void* out, int ldo,
              bool want_pm = false, const int8_t* w8 = nullptr, float* pm_atomic = nullptr) {
        pb(P_GEMM);
        const bool i8 = i8_rows(M) && w8;
        const bool atomic_pm = want_pm && pm_atomic && !i8 && M <= 64;  // GEMV: one reduced max per row
        float* pm = want_pm ? (atomic_pm ? pm_atomic : pmax) : nullptr;
        const int pld = atomic_pm ? 0 : kPmaxLd;
        pm_parts = 0;
        pm_ptr = atomic_pm ? pm_atomic : pmax;
        pm_ld = atomic_pm ? 1 : kPmaxLd;
        // > 32 tokens: the int8-operand tcgen05 GEMM (TMA), with k slices for the decode batches'
        // narrow projections (qt_tc05_i8_single_splitk); up to 32 tokens the weight-streaming GEMV
        // on the int4 tiles (half the int8 copy's bytes).  Measured per shape at 32..256 tokens
        // against the GEMV and the packed-int4 tcgen05 kernel: tools/bench_decode_gemm.py
        int rc = i8 ? qt_launch_w4a4_tc05_i8(epi, codes8, ld8, ascale, w8, wrows, K, sw, M, N, K, out, ldo, nullptr, pm,
                                             kPmaxLd, &pm_parts, splitk_ws, st)
                 : (use_tc05 && M > 64)
                     ? qt_launch_w4a4_tc05_ex(epi, codes, codes_rows, ascale, w, wrows, sw, M, N, K, out, ldo, nullptr,
                                              splitk_ws, pm, kPmaxLd, &pm_parts, st)
                     : qt_launch_w4a4_mma_ex(epi, codes, codes_rows, ascale, w, wrows, sw, M, N, K, out, ldo, nullptr,
                                             pm, pld, &pm_parts, st);
        ckl(rc, "w4a4 gemm");
        const double out_bytes = epi == QT_EPI_RESADD ? 16.0 * M * N : (epi == QT_EPI_SWIGLU ? 2.0 * M * N : 4.0 * M * N);
        pe((double)N * K / 2 + 8.0 * N + (double)M * K / 2 + 8.0 * M + out_bytes, 2.0 * M * N * K);
    }

    // ------------------------------------------------------------ prefill
    struct SeqPlan {
        int V, T, v0;
        std::vector<int> vis_at;  // visual count entering each layer
    };

    void prefill(int nseq, const void* emb, int emb_dev, int emb_f64, const int* vis, const int* txt, const int* v0s,
                 const int* positions, float* logits_out, int out_dev) {
        for (auto& l : lw)
            if (!l.loaded) fail(QT_EINVAL, "model weights not loaded");
        if (!head_loaded) fail(QT_EINVAL, "model head not loaded");
        if (cfg.act_mode == 0 && !act_set) fail(QT_EINVAL, "quantized mode requires a QuantEnv");  // model.cpp:323-325
        if (nseq < 1 || nseq > max_batch) fail(QT_EINVAL, "batch size outside engine capacity");
        reset_staging();
        join_copies();  // the previous prefill's async logits readback still reads `logits`
        if (codes8) ensure_w8();
        graph_ok = false;
        prefilled = false;
        if (prof_next) {
            prof = std::make_unique<Profiler>();
            prof->st = st;
        }
        B = nseq;
        h_vis.assign(vis, vis + B);
        h_txt.assign(txt, txt + B);
        std::vector<int> v0v(B);
        int total = 0;
        for (int b = 0; b < B; ++b) {
            if (h_vis[b] < 0 || h_txt[b] < 0) fail(QT_EINVAL, "negative token count");  // model.cpp:59
            const int S = h_vis[b] + h_txt[b];
            if (S < 1) fail(QT_EINVAL, "empty sequence");
            if (S > max_seq) fail(QT_EINVAL, "sequence longer than engine capacity");
            total += S;
            v0v[b] = v0s ? v0s[b] : recipe.v0;
            if (have_recipe && v0v[b] < 1) fail(QT_EINVAL, "v0 must be >= 1");
        }
        if (total > max_tokens) fail(QT_EINVAL, "batch tokens exceed engine capacity");
        const bool want_rec = (rec_mode & 2) || host_hook;
        if ((want_rec || (rec_mode & 1)) && B != 1)
            fail(QT_EINVAL, "layer records, block outputs and host prune hooks need a batch of one sequence");
        if (host_hook && have_recipe) fail(QT_EINVAL, "a host prune hook and a device recipe are exclusive");
        lrecs.clear();
        blocks.clear();
        // positions: strictly increasing per sequence (model.cpp:64-68)
        std::vector<int> hpos(total);
        {
            int o = 0;
            for (int b = 0; b < B; ++b) {
                const int S = h_vis[b] + h_txt[b];
                for (int i = 0; i < S; ++i) hpos[o + i] = positions ? positions[o + i] : i;
                for (int i = 0; i + 1 < S; ++i)
                    if (hpos[o + i] >= hpos[o + i + 1]) fail(QT_EINVAL, "position_ids must be strictly increasing");
                if (hpos[o + S - 1] + 1 + max_decode >= max_pos || hpos[o] < 0)
                    fail(QT_EINVAL, "position ids outside the engine's RoPE table");
                o += S;
            }
        }
        // per-layer visual counts (host-side shape plan; selector.cpp:11-17, gflops.cpp:53-72)
        std::vector<std::vector<int>> vis_at(B, std::vector<int>(L + 1));
        std::vector<std::vector<int>> kbud(B, std::vector<int>(L, -1));  // budget at candidate layers
        for (int b = 0; b < B; ++b) {
            int v = h_vis[b];
            for (int l = 0; l < L; ++l) {
                vis_at[b][l] = v;
                if (have_recipe) {
                    for (size_t i = 0; i < recipe.layers.size(); ++i) {
                        if (recipe.layers[i] != l) continue;
                        const int K = (int)std::ceil(recipe.keeps[i] * (double)v0v[b]);
                        kbud[b][l] = K;
                        if (K < v) v = K;
                    }
                }
            }
            vis_at[b][L] = v;
            // the reference hook scores every candidate layer it reaches; an empty visual
            // range makes robust_normalize throw (selector.cpp:70-71) -- checked before any launch
            for (int l = 0; l < L; ++l)
                if (kbud[b][l] >= 0 && vis_at[b][l] == 0) fail(QT_EINVAL, "empty sample");
        }
        // KV pages: capacity per (layer, seq) = tokens entering the layer + decode steps
        std::vector<int> hpt((size_t)L * max_batch * max_pages, 0);
        int npages = 0;
        for (int l = 0; l < L; ++l)
            for (int b = 0; b < B; ++b) {
                const int cap = vis_at[b][l] + h_txt[b] + max_decode;
                const int np = (cap + qt::kPage - 1) / qt::kPage;
                for (int p = 0; p < np; ++p) hpt[((size_t)l * max_batch + b) * max_pages + p] = npages++;
            }
        ensure_pool(npages);
        upload(pt, hpt);

        // inputs
        double* xc = x[0];
        int* pc = pos[0];
        if (emb_f64) {  // fp64 embeddings go straight into the residual stream
            ck(cudaMemcpyAsync(xc, emb, (size_t)total * d * sizeof(double),
                               emb_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st),
               "emb");
            qt::g_pdl_block = true;
        } else {
            const float* emb_d = static_cast<const float*>(emb);
            if (!emb_dev) {  // stage through the fp32 attention buffer, widen on device
                ck(cudaMemcpyAsync(attn, emb, (size_t)total * d * sizeof(float), cudaMemcpyHostToDevice, st), "emb");
                emb_d = attn;
                qt::g_pdl_block = true;
            }
            ckl(qt_launch_f32_to_f64(emb_d, xc, (long long)total * d, st), "embedding widen");
        }
        upload(pc, hpos);
        std::vector<int> cur_v(h_vis);
        auto upload_layout = [&]() {
            std::vector<int> off(B + 1), ts, tr, ln(B);
            off[0] = 0;
            for (int b = 0; b < B; ++b) {
                const int S = cur_v[b] + h_txt[b];
                off[b + 1] = off[b] + S;
                ln[b] = S;
                for (int i = 0; i < S; ++i) {
                    ts.push_back(b);
                    tr.push_back(i);
                }
            }
            upload(seq_off, off);
            upload(seq_vis, cur_v);
            upload(seq_txt, h_txt);
            upload(seq_len, ln);
            upload(tok_seq, ts);
            upload(tok_row, tr);
            return off;
        };
        std::vector<int> off = upload_layout();
        int M = off[B];
        std::vector<double> hw4(recipe.w, recipe.w + 4);
        upload(w4, hw4);
        trace.assign(B, {});
        std::vector<int> trace_layers;  // candidate layers that pruned something, in order
        std::vector<std::vector<int>> ev_prev_v, ev_new_v;
        h_kvlen.assign((size_t)L * B, 0);
        std::vector<std::vector<int>> pos_host(B);
        {
            int o = 0;
            for (int b = 0; b < B; ++b) {
                const int S = h_vis[b] + h_txt[b];
                pos_host[b].assign(hpos.begin() + o, hpos.begin() + o + S);
                o += S;
            }
        }
        std::vector<int> cur_pos0 = pos_host[0];  // sequence 0's current layout (records / host hooks)

        for (int l = 0; l < L; ++l) {
            const LayerW& w = lw[l];
            int* ptl = pt + (size_t)l * max_batch * max_pages;
            // attention block (model.cpp:347-396)
            norm_quant(xc, 1, d, w.g1, M, d, kd_pad, 4 * l + 0);
            cap_site(l, 0, M, d, kd_pad);
            gemm(QT_EPI_STORE, w.qkv, n_qkv_pad, w.s_qkv, M, n_qkv, kd_pad, qkv, n_qkv, false, w.qkv8);
            pb(P_KV);
            ckl(qt_launch_rope_kv_append(qkv, n_qkv, M, H, Hkv, dh, pc, tok_seq, tok_row, rope, ptl, max_pages, pool,
                                         page_bytes, 4, nullptr, st),
                "rope+kv append");
            pe((double)M * n_qkv * 8 + (double)M * Hkv * 2 * (dh / 2 + 4));
            if (capture) {
                std::vector<int> r0(B, 0), nr(B);
                for (int b = 0; b < B; ++b) nr[b] = cur_v[b] + h_txt[b];
                cap_kv(l, r0, nr);
            }
            int smax = 0, vmax = 0;
            bool prune_any = false;
            for (int b = 0; b < B; ++b) {
                smax = std::max(smax, cur_v[b] + h_txt[b]);
                vmax = std::max(vmax, cur_v[b]);
                if (kbud[b][l] >= 0 && kbud[b][l] < cur_v[b]) prune_any = true;
            }
            const bool cand = have_recipe && std::any_of(kbud.begin(), kbud.end(), [l](const std::vector<int>& k) { return k[l] >= 0; });

            pb(P_ATTN);
            ckl(qt_launch_attn_prefill(qkv, n_qkv, H, Hkv, dh, seq_off, seq_vis, seq_len, B, smax, pool, page_bytes,
                                       ptl, max_pages, attn, d, (prune_any || want_rec) ? ml : nullptr, pmax, kPmaxLd,
                                       st),
                "prefill attention");
            {  // mask-allowed (query, key) pairs x 4 dh flops per head
                double pairs = 0;
                for (int b = 0; b < B; ++b) {
                    const double V = cur_v[b], T = h_txt[b];
                    pairs += V * V + T * V + T * (T + 1) / 2;
                }
                pe((double)M * (n_qkv * 4.0 + d * 4.0), 4.0 * pairs * dh * H);
            }
            pm_parts = pmax ? H : 0;  // the attention epilogue left max |out| per (row, head)
            pm_ptr = pmax;
            pm_ld = kPmaxLd;
            norm_quant(attn, 0, d, nullptr, M, d, kd_pad, 4 * l + 1, true);
            cap_site(l, 1, M, d, kd_pad);
            gemm(QT_EPI_RESADD, w.o, nd_pad, w.s_o, M, d, kd_pad, xc, d, false, w.o8);
            if (rec_diag) diag_layer(l, ptl, cur_v[0], h_txt[0], xc);
            // LayerActivationRecord (model.cpp:382-402) + a host prune hook (model.cpp:404-427)
            std::vector<int> host_slots;
            bool host_prune = false;
            int host_budget = 0;
            if (want_rec) {
                const int V = cur_v[0], T = h_txt[0], S = V + T;
                LayerRec r{l, V, T, cur_pos0, std::vector<double>((size_t)S * d),
                           std::vector<float>((size_t)H * S * V)};
                if (V > 0) {
                    if (r.probs.size() > probs_cap) {
                        ck(cudaStreamSynchronize(st), "sync");
                        if (probs_d) cudaFree(probs_d);
                        probs_d = dalloc<float>(r.probs.size());
                        probs_cap = r.probs.size();
                    }
                    ckl(qt_launch_attn_colsum(qkv, n_qkv, H, Hkv, dh, seq_off, seq_vis, seq_len, 1, V, pool, page_bytes,
                                              ptl, max_pages, ml, vstride, inter, intra, probs_d, S, V, st),
                        "record attention probabilities");
                    ck(cudaMemcpyAsync(r.probs.data(), probs_d, r.probs.size() * sizeof(float),
                                       cudaMemcpyDeviceToHost, st),
                       "record probabilities");
                }
                ck(cudaMemcpyAsync(r.states.data(), xc, r.states.size() * sizeof(double), cudaMemcpyDeviceToHost, st),
                   "record states");
                ck(cudaStreamSynchronize(st), "record");
                if (host_hook) {
                    qt_layer_record rec{l, V, T, d, H, r.pos.data(), r.states.data(), r.states.data() + (size_t)V * d,
                                        r.probs.data()};
                    std::vector<int> slots(std::max(V, 1));
                    int n = 0;
                    const int rc = host_hook(host_user, &rec, slots.data(), &n, &host_budget);
                    if (rc < 0) fail(QT_ERUNTIME, "prune hook failed");
                    if (rc == 1) {  // apply_pruning's validation (selector.cpp:140-148)
                        if (n < 1) fail(QT_ERUNTIME, "pruning would remove every visual token");
                        if (n > V) fail(QT_ERUNTIME, "pruning text or out-of-range token");
                        int prev = -1;
                        for (int i = 0; i < n; ++i) {
                            if (slots[i] <= prev) fail(QT_ERUNTIME, "retained slots must be ascending and unique");
                            if (slots[i] < 0 || slots[i] >= V) fail(QT_ERUNTIME, "pruning text or out-of-range token");
                            prev = slots[i];
                        }
                        if (n < V) {  // retain-all is a strict no-op (selector.cpp:153-154)
                            host_prune = true;
                            host_slots.assign(slots.begin(), slots.begin() + n);
                        }
                    }
                }
                if (rec_mode & 2) lrecs.push_back(std::move(r));
            }
            for (int b = 0; b < B; ++b) h_kvlen[(size_t)l * B + b] = cur_v[b] + h_txt[b];

            if (host_prune) {  // the host hook's retained set: the device gather + KV filter
                const int V = cur_v[0], T = h_txt[0], nv = (int)host_slots.size();
                std::vector<int> ksrc, kloc((size_t)max_batch * vstride, 0), kp((size_t)max_batch * vstride, 0);
                for (int j = 0; j < nv; ++j) {
                    ksrc.push_back(host_slots[j]);
                    kloc[j] = host_slots[j];
                    kp[j] = cur_pos0[host_slots[j]];
                }
                for (int t = 0; t < T; ++t) {
                    ksrc.push_back(V + t);
                    kloc[nv + t] = V + t;
                }
                const size_t evi = trace_layers.size();
                upload(keep_src, ksrc);
                upload(keep_local, kloc);
                ck(cudaMemcpyAsync(kept_pos + evi * max_batch * vstride, stage(kp.data(), kp.size()),
                                   kp.size() * sizeof(int), cudaMemcpyHostToDevice, st),
                   "kept positions");
                std::vector<int> nlen{nv + T};
                upload(new_len, nlen);
                double* xn = x[xc == x[0] ? 1 : 0];
                int* pn = pos[pc == pos[0] ? 1 : 0];
                ckl(qt_launch_gather_rows(xc, xn, d, pc, pn, keep_src, nv + T, st), "compaction gather");
                ckl(qt_launch_kv_compact(pool, page_bytes, ptl, max_pages, Hkv, dh, keep_local, vstride, new_len, 1, st),
                    "kv compaction");
                kbud[0][l] = host_budget;
                trace_layers.push_back(l);
                ev_prev_v.push_back(cur_v);
                ev_new_v.push_back({nv});
                h_kvlen[(size_t)l * B] = nv + T;
                std::vector<int> npos;
                for (int j = 0; j < nv; ++j) npos.push_back(cur_pos0[host_slots[j]]);
                npos.insert(npos.end(), cur_pos0.begin() + V, cur_pos0.end());
                cur_pos0 = std::move(npos);
                cur_v[0] = nv;
                xc = xn;
                pc = pn;
                off = upload_layout();
                M = off[B];
            }
            // recipe hook at candidate layers (selector.cpp:214-227, model.cpp:404-427)
            if (cand && prune_any) {
                if (vmax > vstride) fail(QT_EINVAL, "visual prefix exceeds engine capacity");
                pb(P_SELECT);
                ckl(qt_launch_attn_colsum(qkv, n_qkv, H, Hkv, dh, seq_off, seq_vis, seq_len, B, vmax, pool, page_bytes,
                                          ptl, max_pages, ml, vstride, inter, intra, nullptr, 0, 0, st),
                    "quota attention metrics");
                ckl(qt_launch_token_metrics(xc, d, seq_off, seq_vis, vmax, B, vstride, recipe.res_bits, mag, res, st),
                    "quota token metrics");
                std::vector<int> bud(B), noff(B + 1), nlen(B), nv(B);
                noff[0] = 0;
                for (int b = 0; b < B; ++b) {
                    const int K = kbud[b][l] >= 0 ? kbud[b][l] : cur_v[b];
                    nv[b] = std::min(K, cur_v[b]);
                    bud[b] = std::max(1, nv[b]);
                    nlen[b] = nv[b] + h_txt[b];
                    noff[b + 1] = noff[b] + nlen[b];
                }
                upload(budget, bud);
                upload(new_off, noff);
                upload(new_len, nlen);
                int* kp_ev = kept_pos + (size_t)trace_layers.size() * max_batch * vstride;
                const size_t evi = trace_layers.size();
                ckl(qt_launch_select_topk(mag, res, inter, intra, H, vstride, seq_vis, seq_txt, budget, seq_off, new_off,
                                          B, vmax, hw4.data(), keep_src, keep_local, vstride, pc, kp_ev,
                                          sc_fused + evi * max_batch * vstride,
                                          sc_norm + evi * max_batch * 4 * vstride, nullptr, 0, st),
                    "quota top-k");
                double* xn = x[xc == x[0] ? 1 : 0];
                int* pn = pos[pc == pos[0] ? 1 : 0];
                ckl(qt_launch_gather_rows(xc, xn, d, pc, pn, keep_src, noff[B], st), "compaction gather");
                ckl(qt_launch_kv_compact(pool, page_bytes, ptl, max_pages, Hkv, dh, keep_local, vstride, new_len, B, st),
                    "kv compaction");
                pe((double)M * d * 8 * 2);
                if (want_rec) {  // sequence 0's new layout, for the next layers' records
                    std::vector<int> kp0(nv[0]);
                    ck(cudaMemcpyAsync(kp0.data(), kp_ev, nv[0] * sizeof(int), cudaMemcpyDeviceToHost, st), "kept");
                    ck(cudaStreamSynchronize(st), "kept");
                    kp0.insert(kp0.end(), cur_pos0.begin() + cur_v[0], cur_pos0.end());
                    cur_pos0 = std::move(kp0);
                }
                // trace: kept visual positions, read back once after the prefill
                trace_layers.push_back(l);
                ev_prev_v.push_back(cur_v);
                ev_new_v.push_back(nv);
                for (int b = 0; b < B; ++b) {
                    h_kvlen[(size_t)l * B + b] = nlen[b];
                    cur_v[b] = nv[b];
                }
                xc = xn;
                pc = pn;
                off = upload_layout();
                M = off[B];
            }
            // MLP block (model.cpp:429-437)
            norm_quant(xc, 1, d, w.g2, M, d, kd_pad, 4 * l + 2);
            cap_site(l, 2, M, d, kd_pad);
            if (cfg.mlp == 1) gemm(QT_EPI_SWIGLU, w.gu, n_gu_pad, w.s_gu, M, n_gu, kd_pad, mid, dff, true, w.gu8);
            else gemm(QT_EPI_SILU, w.gu, n_gu_pad, w.s_gu, M, n_gu, kd_pad, mid, dff, true, w.gu8);
            norm_quant(mid, 0, dff, nullptr, M, dff, kff_pad, 4 * l + 3, true);
            cap_site(l, 3, M, dff, kff_pad);
            gemm(QT_EPI_RESADD, w.down, nd_pad, w.s_down, M, d, kff_pad, xc, d, false, w.down8);
            if (rec_mode & 1) {  // ForwardResult::block_outputs (model.cpp:439)
                blocks.resize(L);
                blocks[l].resize((size_t)M * d);
                ck(cudaMemcpyAsync(blocks[l].data(), xc, (size_t)M * d * sizeof(double), cudaMemcpyDeviceToHost, st),
                   "block output");
            }
            if (rec_blocks) {  // ForwardResult::block_outputs (model.cpp:439), calibration only
                if (l == 0) rec_blocks->assign(L, {});
                (*rec_blocks)[l].resize((size_t)M * d);
                ck(cudaMemcpyAsync((*rec_blocks)[l].data(), xc, (size_t)M * d * sizeof(double), cudaMemcpyDeviceToHost,
                                   st),
                   "block output");
            }
        }
        // final norm + head (model.cpp:442-445)
        norm_quant(xc, 1, d, gf, M, d, kd_pad, 4 * L);
        cap_site(L, 4, M, d, kd_pad);
        gemm(QT_EPI_STORE, head, nd_pad, s_head, M, d, kd_pad, logits, d, false, head8);
        final_rows = M;
        ev_layers = trace_layers;
        ev_vis = ev_prev_v;
        if (logits_out && out_dev == 2) {
            // asynchronous host readback on a copy stream: overlaps the decode steps that follow;
            // complete after qt_engine_synchronize / qt_engine_join_copies
            if (!cst) {
                ck(cudaStreamCreateWithFlags(&cst, cudaStreamNonBlocking), "copy stream");
                ck(cudaEventCreateWithFlags(&ev_lg, cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&ev_cp, cudaEventDisableTiming), "event");
            }
            ck(cudaEventRecord(ev_lg, st), "event");
            ck(cudaStreamWaitEvent(cst, ev_lg, 0), "event wait");
            ck(cudaMemcpyAsync(logits_out, logits, (size_t)M * d * sizeof(float), cudaMemcpyDeviceToHost, cst),
               "logits readback");
            ck(cudaEventRecord(ev_cp, cst), "event");
            copy_pending = true;
        } else if (logits_out) {
            ck(cudaMemcpyAsync(logits_out, logits, (size_t)M * d * sizeof(float),
                               out_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st),
               "logits readback");
        }

        // prune trace (PruneEvent, model.cpp:408-418) and final layout positions
        if (!trace_layers.empty()) {
            std::vector<int> kp(trace_layers.size() * (size_t)max_batch * vstride);
            ck(cudaMemcpyAsync(kp.data(), kept_pos, kp.size() * sizeof(int), cudaMemcpyDeviceToHost, st), "trace");
            ck(cudaStreamSynchronize(st), "trace");
            for (size_t ev = 0; ev < trace_layers.size(); ++ev) {
                const int l = trace_layers[ev];
                for (int b = 0; b < B; ++b) {
                    const int pv = ev_prev_v[ev][b], nvb = ev_new_v[ev][b];
                    if (nvb >= pv) continue;
                    PruneEv e{l, kbud[b][l], {}};
                    const int* kpv = kp.data() + (ev * max_batch + b) * (size_t)vstride;
                    e.positions.assign(kpv, kpv + nvb);
                    trace[b].push_back(e);
                    std::vector<int> npos(e.positions);
                    npos.insert(npos.end(), pos_host[b].begin() + pv, pos_host[b].end());
                    pos_host[b] = npos;
                }
            }
        }
        // decode state: cache lengths, next positions (model.cpp:447-451)
        {  // device layout is [L][max_batch]
            std::vector<int> kl((size_t)L * max_batch, 0);
            for (int l = 0; l < L; ++l)
                for (int b = 0; b < B; ++b) kl[(size_t)l * max_batch + b] = h_kvlen[(size_t)l * B + b];
            upload(kv_len, kl);
        }
        std::vector<int> np(B), ds(B);
        for (int b = 0; b < B; ++b) {
            np[b] = pos_host[b].back() + 1;
            ds[b] = b;
        }
        // next_position = last ORIGINAL position + 1 of the input layout
        {
            int o = 0;
            for (int b = 0; b < B; ++b) {
                const int S = h_vis[b] + h_txt[b];
                np[b] = hpos[o + S - 1] + 1;
                o += S;
            }
        }
        upload(next_pos, np);
        upload(dec_seq, ds);
        h_next = np;
        h_off = off;
        h_vis = cur_v;
        h_pos = pos_host;
        // decode attention split plan: per layer, the pages its longest sequence can reach over
        // the decode horizon (pruned layers need fewer page CTAs than the unpruned ones)
        int maxp = 1;
        dec_pages.assign(L, 1);
        for (int l = 0; l < L; ++l)
            for (int b = 0; b < B; ++b) {
                const int cap = h_kvlen[(size_t)l * B + b] + max_decode;
                dec_pages[l] = std::max(dec_pages[l], (cap + qt::kPage - 1) / qt::kPage);
                maxp = std::max(maxp, dec_pages[l]);
            }
        dec_lpps.assign(L, 1);
        dec_lsplit.assign(L, 1);
        dec_pps = dec_splits = 1;
        for (int l = 0; l < L; ++l) {
            if (qt_attn_decode_plan(B, H, Hkv, dec_pages[l], n_sms, &dec_lpps[l], &dec_lsplit[l]))
                fail(QT_EINVAL, "decode attention plan");
            dec_pps = std::max(dec_pps, dec_lpps[l]);
            dec_splits = std::max(dec_splits, dec_lsplit[l]);
        }
        (void)maxp;
        if (tok_table) {  // the greedy decoding's first argmax reads the prefill's last row per sequence
            std::vector<int> lr(B);
            for (int b = 0; b < B; ++b) lr[b] = off[b + 1] - 1;
            upload(last_rows, lr);
            ckl(qt_launch_copy_rows_f32(logits, last_rows, d, dlogits, B, st), "last logits rows");
        }
        ck(cudaStreamSynchronize(st), "prefill");
        decode_steps = 0;
        prefilled = true;
        graph_ok = graph_g_ok = false;
        finish_profile();
    }

    // ------------------------------------------------------------ decode
    bool use_graphs = true;  // qt_engine_set_graphs: decode steps as CUDA graph replays (else eager)
    int skip_mask = 0;  // kernel classes left out of decode_body (profile_chain: 1 GEMM, 2 attention, 4 quant, 8 kv)
    void decode_body() {
        double* xcur = xd;  // the step's input was written (widened) into xd before the graph
        for (int l = 0; l < L; ++l) {
            const LayerW& w = lw[l];
            int* ptl = pt + (size_t)l * max_batch * max_pages;
            int* lenl = kv_len + (size_t)l * max_batch;
            if (!(skip_mask & 4)) norm_quant(xcur, 1, d, w.g1, B, d, kd_pad, 4 * l + 0);
            cap_site(l, 0, B, d, kd_pad);
            if (!(skip_mask & 1))
                gemm(QT_EPI_STORE, w.qkv, n_qkv_pad, w.s_qkv, B, n_qkv, kd_pad, qkv, n_qkv, false, w.qkv8);
            pb(P_ATTN);
            // decode attention over the int4 pages with the new token's RoPE + K/V quantize +
            // append fused in, then the split merge fused with the attn_out quantizer
            if (!(skip_mask & 2))
                ckl(qt_launch_attn_decode(qkv, n_qkv, H, Hkv, dh, lenl, B, pool, page_bytes, ptl, max_pages,
                                          dec_lpps[l], dec_lsplit[l], rope, next_pos, part_ml, part_o, nullptr, d,
                                          codes, codes_rows, ascale, cfg.act_mode,
                                          cfg.act_mode == 0 ? act[4 * l + 1] : 0.0, kd_pad, 4,
                                          i8_rows(B) ? codes8 : nullptr, ld8, st),
                    "decode attention");
            {  // decode attention streams every cached K/V row of this layer once
                double rows = 0;
                for (int b = 0; b < B; ++b) rows += h_kvlen[(size_t)l * B + b] + 1;
                pe(rows * Hkv * 2 * (dh / 2 + 4) + (double)B * (H + 2 * Hkv) * dh * 4);
            }
            if (capture) {
                std::vector<int> r0(B), nr(B, 1);
                for (int b = 0; b < B; ++b) r0[b] = h_kvlen[(size_t)l * B + b];
                cap_kv(l, r0, nr);
            }
            cap_site(l, 1, B, d, kd_pad);
            if (!(skip_mask & 1)) gemm(QT_EPI_RESADD, w.o, nd_pad, w.s_o, B, d, kd_pad, xcur, d, false, w.o8);
            if (!(skip_mask & 4)) norm_quant(xcur, 1, d, w.g2, B, d, kd_pad, 4 * l + 2);
            cap_site(l, 2, B, d, kd_pad);
            float* gml = gmax ? gmax + (size_t)l * max_batch : nullptr;
            if (!(skip_mask & 1))
                gemm(cfg.mlp == 1 ? QT_EPI_SWIGLU : QT_EPI_SILU, w.gu, n_gu_pad, w.s_gu, B, n_gu, kd_pad, mid, dff, true,
                     w.gu8, gml);
            if (!(skip_mask & 4)) norm_quant(mid, 0, dff, nullptr, B, dff, kff_pad, 4 * l + 3, true);
            cap_site(l, 3, B, dff, kff_pad);
            if (!(skip_mask & 1))
                gemm(QT_EPI_RESADD, w.down, nd_pad, w.s_down, B, d, kff_pad, xcur, d, false, w.down8);
        }
        norm_quant(xcur, 1, d, gf, B, d, kd_pad, 4 * L);
        cap_site(L, 4, B, d, kd_pad);
        gemm(QT_EPI_STORE, head, nd_pad, s_head, B, d, kd_pad, dlogits, d, false, head8);
        ckl(qt_launch_kv_len_bump(kv_len, L * max_batch, next_pos, B, st), "kv length / position bump");
        if (gmax) ck(cudaMemsetAsync(gmax, 0, (size_t)L * max_batch * sizeof(float), st), "row-max reset");
    }

    void finish_profile() {
        if (!prof) return;
        prof->read(prof_out);
        prof.reset();
        prof_next = false;
    }

    // Device time of one decode step restricted to some kernel classes (skip: the classes to
    // leave out), as a CUDA graph replayed reps times back to back on the engine stream --
    // the per-class cost inside a graph with PDL, which per-launch events cannot see.  The
    // cache lengths and positions the step bumps are restored afterwards.
    double profile_chain(int skip, int reps) {
        if (!prefilled) fail(QT_ERUNTIME, "cache and execution mode mismatch");
        if (reps < 1) fail(QT_EINVAL, "reps must be >= 1");
        const size_t nkv = (size_t)L * max_batch;
        int* save = dalloc<int>(nkv + max_batch);
        ck(cudaMemcpyAsync(save, kv_len, nkv * sizeof(int), cudaMemcpyDeviceToDevice, st), "save");
        ck(cudaMemcpyAsync(save + nkv, next_pos, max_batch * sizeof(int), cudaMemcpyDeviceToDevice, st), "save");
        qt::g_pdl_block = true;
        const int old = skip_mask;
        skip_mask = skip;
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        float ms = 0.f;
        auto cleanup = [&]() {
            skip_mask = old;
            if (ge) cudaGraphExecDestroy(ge);
            if (g) cudaGraphDestroy(g);
            if (e0) cudaEventDestroy(e0);
            if (e1) cudaEventDestroy(e1);
        };
        try {
            ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "graph capture");
            g_capturing = true;
            try {
                decode_body();
            } catch (...) {
                g_capturing = false;
                cudaStreamEndCapture(st, &g);
                throw;
            }
            g_capturing = false;
            ck(cudaStreamEndCapture(st, &g), "graph capture end");
            ck(cudaGraphInstantiate(&ge, g, 0), "graph instantiate");
            ck(cudaEventCreate(&e0), "event");
            ck(cudaEventCreate(&e1), "event");
            ck(cudaGraphLaunch(ge, st), "graph launch");  // warm
            ck(cudaEventRecord(e0, st), "event");
            for (int r = 0; r < reps; ++r) ck(cudaGraphLaunch(ge, st), "graph launch");
            ck(cudaEventRecord(e1, st), "event");
            ck(cudaEventSynchronize(e1), "event");
            ck(cudaEventElapsedTime(&ms, e0, e1), "event");
            ck(cudaMemcpyAsync(kv_len, save, nkv * sizeof(int), cudaMemcpyDeviceToDevice, st), "restore");
            ck(cudaMemcpyAsync(next_pos, save + nkv, max_batch * sizeof(int), cudaMemcpyDeviceToDevice, st),
               "restore");
            ck(cudaStreamSynchronize(st), "restore");
        } catch (...) {
            cleanup();
            cudaFree(save);
            throw;
        }
        cleanup();
        cudaFree(save);
        qt::g_pdl_block = true;
        return (double)ms / reps;
    }

    // emb == nullptr: a greedy step (the input is the embedding of the argmax of the previous logits)
    void decode(const void* emb, int emb_dev, int emb_f64, float* out, int out_dev, int* tokens_out = nullptr) {
        if (!prefilled) fail(QT_ERUNTIME, "cache and execution mode mismatch");
        if (decode_steps >= max_decode) fail(QT_EINVAL, "decode steps exceed engine capacity");
        const bool greedy = emb == nullptr;
        if (greedy && !tok_table) fail(QT_EINVAL, "greedy decoding needs a token-embedding table");
        const bool profiling = prof_next;
        if (profiling) {
            prof = std::make_unique<Profiler>();
            prof->st = st;
        }
        auto greedy_in = [&]() {
            pb(P_OTHER);
            ckl(qt_launch_greedy_next(dlogits, d, vocab, tok_table, d, xd, dec_tok, B, st), "greedy argmax + embed");
            pe((double)B * d * 4 * 2 + (double)B * d * 8);
        };
        if (greedy) {
            // the argmax + embedding kernel is the first node of the greedy graph
        } else if (emb_f64) {
            ck(cudaMemcpyAsync(xd, emb, (size_t)B * d * sizeof(double),
                               emb_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st),
               "decode emb");
            qt::g_pdl_block = true;
        } else {
            ck(cudaMemcpyAsync(xd_in, emb, (size_t)B * d * sizeof(float),
                               emb_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st),
               "decode emb");
            qt::g_pdl_block = true;
            pb(P_OTHER);
            ckl(qt_launch_f32_to_f64(xd_in, xd, (long long)B * d, st), "embedding widen");
            pe((double)B * d * 12);
        }
        cudaGraphExec_t& gx = greedy ? graph_g : graph;
        bool& gx_ok = greedy ? graph_g_ok : graph_ok;
        if (profiling || capture || !use_graphs) {
            if (greedy) greedy_in();
            decode_body();  // eager launches so every kernel gets its own events / capture reads
        } else if (!gx_ok) {
            if (gx) cudaGraphExecDestroy(gx);
            gx = nullptr;
            cudaGraph_t g = nullptr;
            ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "graph capture");
            g_capturing = true;
            try {
                if (greedy) greedy_in();
                decode_body();
            } catch (...) {
                g_capturing = false;
                cudaStreamEndCapture(st, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            g_capturing = false;
            ck(cudaStreamEndCapture(st, &g), "graph capture end");
            ck(cudaGraphInstantiate(&gx, g, 0), "graph instantiate");
            cudaGraphDestroy(g);
            gx_ok = true;
        }
        if (!profiling && !capture && use_graphs) ck(cudaGraphLaunch(gx, st), "graph launch");
        if (greedy && tokens_out)
            ck(cudaMemcpyAsync(tokens_out, dec_tok, (size_t)B * sizeof(int), cudaMemcpyDefault, st), "tokens");
        if (out)
            ck(cudaMemcpyAsync(out, dlogits, (size_t)B * d * sizeof(float),
                               out_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st),
               "decode logits");
        ++decode_steps;
        finish_profile();
        for (int b = 0; b < B; ++b) {  // model.cpp:553-556
            h_txt[b] += 1;
            h_pos[b].push_back(h_next[b]++);
        }
        for (auto& v : h_kvlen) v += 1;
    }
};

// kv length / position bump after a decode step (device-resident so the
// captured graph replays unchanged)
namespace qt {
__global__ void k_bump(int* kv_len, int n, int* next_pos, int B) {
    pdl_launch_dependents();
    pdl_wait();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) kv_len[i] += 1;
    if (i < B) next_pos[i] += 1;  // model.cpp:556
}
}  // namespace qt

// ---- packed-weight file: the device layout, byte for byte -----
// header: magic "QTW4B200", u32 version, qt_config, the padded geometry, a flag for
// static activation scales (+ 4L+1 doubles), then per layer the tiled int4 codes
// and fp64 scales of qkv / o / gate|up / down and the fp32 gains, then the head.
namespace {
struct WFileHdr {
    char magic[8];
    uint32_t version;
    qt_config cfg;
    int32_t geom[6];  // n_qkv_pad, kd_pad, nd_pad, n_gu_pad, kff_pad, L
    int32_t has_act;
};

template <class F>
void for_each_blob(qt_engine* e, F&& f) {
    for (int l = 0; l < e->L; ++l) {
        LayerW& w = e->lw[l];
        f(w.qkv, (size_t)e->n_qkv_pad * e->kd_pad / 2);
        f(w.s_qkv, (size_t)e->n_qkv_pad * 8);
        f(w.o, (size_t)e->nd_pad * e->kd_pad / 2);
        f(w.s_o, (size_t)e->nd_pad * 8);
        f(w.gu, (size_t)e->n_gu_pad * e->kd_pad / 2);
        f(w.s_gu, (size_t)e->n_gu_pad * 8);
        f(w.down, (size_t)e->nd_pad * e->kff_pad / 2);
        f(w.s_down, (size_t)e->nd_pad * 8);
        f(w.g1, (size_t)e->d * 4);
        f(w.g2, (size_t)e->d * 4);
    }
    f(e->head, (size_t)e->nd_pad * e->kd_pad / 2);
    f(e->s_head, (size_t)e->nd_pad * 8);
    f(e->gf, (size_t)e->d * 4);
}

WFileHdr make_hdr(qt_engine* e) {
    WFileHdr h{};
    std::memcpy(h.magic, "QTW4B200", 8);
    h.version = 1;
    h.cfg = e->cfg;
    const int g[6] = {e->n_qkv_pad, e->kd_pad, e->nd_pad, e->n_gu_pad, e->kff_pad, e->L};
    std::memcpy(h.geom, g, sizeof(g));
    h.has_act = e->act_set ? 1 : 0;
    return h;
}
}  // namespace

extern "C" {

int qt_launch_kv_len_bump(int* kv_len, int n, int* next_pos, int B, cudaStream_t st) {
    return qt::launch_pdl(qt::k_bump, dim3((std::max(n, B) + 255) / 256), dim3(256), 0, st, kv_len, n, next_pos, B);
}

const char* qt_last_error(void) { return g_err.c_str(); }

void qt_set_last_error(const char* msg) { g_err = msg ? msg : ""; }

uint64_t qt_fnv1a64(const void* data, size_t len, uint64_t seed) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    uint64_t h = seed;
    for (size_t i = 0; i < len; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

int qt_rope_table(int max_pos, int d_head, double* out) {
    // cos/sin of pos * 10000^(-2i/d_head), exactly as rope_in_place (model.cpp:156-168)
    for (int p = 0; p < max_pos; ++p)
        for (int i = 0; i < d_head / 2; ++i) {
            double freq = std::pow(10000.0, -2.0 * static_cast<double>(i) / static_cast<double>(d_head));
            double ang = static_cast<double>(p) * freq;
            out[((size_t)p * (d_head / 2) + i) * 2] = std::cos(ang);
            out[((size_t)p * (d_head / 2) + i) * 2 + 1] = std::sin(ang);
        }
    return 0;
}

int qt_engine_create(const qt_config* cfg, int max_batch, int max_tokens, int max_seq, int max_decode,
                     qt_engine** out) {
    return guard([&] {
        if (!cfg || !out) fail(QT_EINVAL, "null argument");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            fail(QT_ECUDA, "no CUDA device: the B200 path has no CPU fallback");
        auto e = std::make_unique<qt_engine>();
        e->init(*cfg, max_batch, max_tokens, max_seq, max_decode);
        *out = e.release();
    });
}

void qt_engine_destroy(qt_engine* e) { delete e; }

int qt_engine_set_stream(qt_engine* e, void* stream) {
    return guard([&] {
        e->st = stream ? static_cast<cudaStream_t>(stream) : e->own_stream;
        e->graph_ok = false;
    });
}

int qt_engine_synchronize(qt_engine* e) {
    return guard([&] {
        e->join_copies();
        ck(cudaStreamSynchronize(e->st), "synchronize");
    });
}

int qt_engine_join_copies(qt_engine* e) {
    return guard([&] { e->join_copies(); });
}

int qt_engine_load_layer(qt_engine* e, int layer, const float* wq, const float* wk, const float* wv,
                         const float* wo, const float* w1, const float* w2, const float* w3, const float* g1,
                         const float* g2, int on_device) {
    return guard([&] {
        if (layer < 0 || layer >= e->L) fail(QT_ERANGE, "layer out of range");
        if (!wq || !wk || !wv || !wo || !w1 || !w2) fail(QT_EINVAL, "null weight");
        if (e->cfg.mlp == 1 && !w3) fail(QT_EINVAL, "SwiGLU needs w3 (up projection)");
        LayerW& l = e->lw[layer];
        const int d = e->d, kvd = e->Hkv * e->dh, f = e->dff;
        // device weights may come from another stream (e.g. torch's): let them land first
        if (on_device) ck(cudaDeviceSynchronize(), "weights ready");
        e->quant_into(wq, d, d, on_device, 1, 0, l.qkv, e->n_qkv_pad, l.s_qkv);
        e->quant_into(wk, d, kvd, on_device, 1, d, l.qkv, e->n_qkv_pad, l.s_qkv);
        e->quant_into(wv, d, kvd, on_device, 1, d + kvd, l.qkv, e->n_qkv_pad, l.s_qkv);
        e->quant_into(wo, d, d, on_device, 1, 0, l.o, e->nd_pad, l.s_o);
        if (e->cfg.mlp == 1) {
            e->quant_into(w1, d, f, on_device, 2, 0, l.gu, e->n_gu_pad, l.s_gu);
            e->quant_into(w3, d, f, on_device, 2, 1, l.gu, e->n_gu_pad, l.s_gu);
        } else {
            e->quant_into(w1, d, f, on_device, 1, 0, l.gu, e->n_gu_pad, l.s_gu);
        }
        e->quant_into(w2, f, d, on_device, 1, 0, l.down, e->nd_pad, l.s_down);
        if (e->keep_fp) {
            FpLayer& fl = e->fpw[layer];
            const float* ws[7] = {wq, wk, wv, wo, w1, w2, w3};
            const size_t ns[7] = {(size_t)d * d, (size_t)d * kvd, (size_t)d * kvd, (size_t)d * d, (size_t)d * f,
                                  (size_t)f * d, (size_t)d * f};
            for (int i = 0; i < 7; ++i) e->keep64(fl.w[i], ws[i], ns[i], on_device);
        }
        e->load_gain(l.g1, g1, on_device);
        e->load_gain(l.g2, g2, on_device);
        l.loaded = true;
        l.w8_ok = false;
        e->graph_ok = false;
    });
}

int qt_engine_load_layer_codes(qt_engine* e, int layer, const int8_t* const* codes, const double* const* scales,
                               const double* g1, const double* g2) {
    return guard([&] {
        if (layer < 0 || layer >= e->L) fail(QT_ERANGE, "layer out of range");
        if (!codes || !scales) fail(QT_EINVAL, "null weight codes");
        LayerW& l = e->lw[layer];
        const int d = e->d, kvd = e->Hkv * e->dh, f = e->dff;
        if (e->cfg.mlp == 1 && (!codes[6] || !scales[6])) fail(QT_EINVAL, "SwiGLU needs w3 (up projection)");
        e->codes_into(codes[0], scales[0], d, d, 1, 0, l.qkv, e->n_qkv_pad, l.s_qkv);
        e->codes_into(codes[1], scales[1], d, kvd, 1, d, l.qkv, e->n_qkv_pad, l.s_qkv);
        e->codes_into(codes[2], scales[2], d, kvd, 1, d + kvd, l.qkv, e->n_qkv_pad, l.s_qkv);
        e->codes_into(codes[3], scales[3], d, d, 1, 0, l.o, e->nd_pad, l.s_o);
        if (e->cfg.mlp == 1) {
            e->codes_into(codes[4], scales[4], d, f, 2, 0, l.gu, e->n_gu_pad, l.s_gu);
            e->codes_into(codes[6], scales[6], d, f, 2, 1, l.gu, e->n_gu_pad, l.s_gu);
        } else {
            e->codes_into(codes[4], scales[4], d, f, 1, 0, l.gu, e->n_gu_pad, l.s_gu);
        }
        e->codes_into(codes[5], scales[5], f, d, 1, 0, l.down, e->nd_pad, l.s_down);
        e->load_gain64(l.g1, g1);
        e->load_gain64(l.g2, g2);
        l.loaded = true;
        l.w8_ok = false;
        e->graph_ok = false;
    });
}

int qt_engine_load_head_codes(qt_engine* e, const int8_t* codes, const double* scales, const double* final_gain) {
    return guard([&] {
        e->codes_into(codes, scales, e->d, e->d, 1, 0, e->head, e->nd_pad, e->s_head);
        e->load_gain64(e->gf, final_gain);
        e->head_loaded = true;
        e->head8_ok = false;
        e->graph_ok = false;
    });
}

int qt_engine_keep_fp_weights(qt_engine* e, int on) {
    return guard([&] {
        e->keep_fp = on != 0;
        if (e->keep_fp && e->fpw.empty()) e->fpw.resize(e->L);
    });
}

int qt_engine_fit_act_scales(qt_engine* e, int n_samples, const double* const* embs, const int* visual,
                             const int* text, double* scales_out, int apply) {
    return guard([&] {
        if (!embs || !visual || !text || !scales_out) fail(QT_EINVAL, "null argument");
        e->fit_act_scales(n_samples, embs, visual, text, scales_out);
        if (apply && qt_engine_set_act_scales(e, scales_out) != 0) fail(QT_EINVAL, qt_last_error());
    });
}

int qt_engine_fit_act_scales_hooked(qt_engine* e, int n_samples, const double* const* embs, const int* visual,
                                    const int* text, double* scales_out, int apply) {
    return guard([&] {
        if (!embs || !visual || !text || !scales_out) fail(QT_EINVAL, "null argument");
        e->fit_act_scales(n_samples, embs, visual, text, scales_out, true);
        if (apply && qt_engine_set_act_scales(e, scales_out) != 0) fail(QT_EINVAL, qt_last_error());
    });
}

int qt_engine_prefill_fp(qt_engine* e, int n_seq, const double* const* embs, const int* visual, const int* text,
                         int hook, double* logits_out, long long cap_rows) {
    return guard([&] {
        if (!embs || !visual || !text) fail(QT_EINVAL, "null argument");
        e->prefill_fp(n_seq, embs, visual, text, hook != 0, logits_out, cap_rows);
    });
}

int qt_engine_profile_sensitivity(qt_engine* e, int n_samples, const double* const* embs, const int* visual,
                                  const int* text, int n_layers, const int* layers, double eta, double* raw,
                                  double* normalized) {
    return guard([&] {
        if (!embs || !visual || !text || !layers || !raw || !normalized) fail(QT_EINVAL, "null argument");
        e->profile_sensitivity(n_samples, embs, visual, text, n_layers, layers, eta, raw, normalized);
    });
}

int qt_engine_profile_diagnostics(qt_engine* e, int n_samples, const double* const* embs, const int* visual,
                                  const int* text, double* conc_median, double* conc_iqr, double* red_median) {
    return guard([&] {
        if (!embs || !visual || !text || !conc_median || !conc_iqr || !red_median) fail(QT_EINVAL, "null argument");
        e->profile_diagnostics(n_samples, embs, visual, text, conc_median, conc_iqr, red_median);
    });
}

// select_candidate_layers (calibrator.cpp:197-223): the window maximising mean(concentration)
// - mean(redundancy), excluding the first front_exclude and last tail_exclude layers
static std::vector<int> quota_select_window(const double* conc, const double* red, int n, int window,
                                            int front_exclude, int tail_exclude) {
    if (window < 1) fail(QT_EINVAL, "window must be >= 1");
    if (tail_exclude < 0) tail_exclude = n / 4;
    const int first = front_exclude, last = n - tail_exclude;
    if (last - first < window) fail(QT_EINVAL, "infeasible candidate window");
    int best = first;
    double best_score = -1e300;
    for (int st0 = first; st0 + window <= last; ++st0) {
        double c = 0.0, r = 0.0;
        for (int l = st0; l < st0 + window; ++l) {
            c += conc[l];
            r += red[l];
        }
        const double score = (c - r) / (double)window;
        if (score > best_score) {  // strict: ties keep the earliest window
            best_score = score;
            best = st0;
        }
    }
    std::vector<int> out(window);
    for (int i = 0; i < window; ++i) out[i] = best + i;
    return out;
}

// make_budget_schedule (calibrator.cpp:100-141): Eq. 3 drop shares softmax((1 - s)/tau),
// Eq. 4 cumulative keep ratios floored at p_min, the last one exactly p_min
static std::vector<double> quota_keep_schedule(const std::vector<double>& normalized, double tau, double p_min) {
    if (tau <= 0.0) fail(QT_EINVAL, "invalid temperature");
    if (!(p_min > 0.0 && p_min <= 1.0)) fail(QT_EINVAL, "p_min outside (0,1]");
    const size_t n = normalized.size();
    std::vector<double> logits(n), share(n);
    double mx = 1.0 - normalized[0];
    for (size_t i = 0; i < n; ++i) {
        logits[i] = 1.0 - normalized[i];
        mx = std::max(mx, logits[i]);
    }
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) {
        share[i] = std::exp((logits[i] - mx) / tau);
        sum += share[i];
    }
    for (double& v : share) v /= sum;
    const double budget = 1.0 - p_min;
    std::vector<double> keep(n);
    double dropped = 0.0;
    for (size_t i = 0; i < n; ++i) {
        dropped += budget * share[i];
        keep[i] = std::max(p_min, 1.0 - dropped);
    }
    keep.back() = p_min;
    return keep;
}

int qt_engine_run_quota_calibration(qt_engine* e, int n_samples, const double* const* embs, const int* visual,
                                    const int* text, int window, double p_min, double tau, double eta,
                                    double* act_scales, int* layers, double* keep_ratios, double* raw,
                                    double* normalized, double* conc_median, double* red_median) {
    return guard([&] {
        if (!embs || !visual || !text || !act_scales || !layers || !keep_ratios) fail(QT_EINVAL, "null argument");
        // run_quota_calibration (calibrator.cpp:251-268) on explicit samples
        e->fit_act_scales(n_samples, embs, visual, text, act_scales);
        if (qt_engine_set_act_scales(e, act_scales) != 0) fail(QT_EINVAL, qt_last_error());
        std::vector<double> cm(e->L), ci(e->L), rm(e->L);
        e->profile_diagnostics(n_samples, embs, visual, text, cm.data(), ci.data(), rm.data());
        const std::vector<int> cand = quota_select_window(cm.data(), rm.data(), e->L, window, 2, -1);
        std::vector<double> rw(cand.size()), nm(cand.size());
        e->profile_sensitivity(n_samples, embs, visual, text, (int)cand.size(), cand.data(), eta, rw.data(), nm.data());
        const std::vector<double> keep = quota_keep_schedule(nm, tau, p_min);
        std::copy(cand.begin(), cand.end(), layers);
        std::copy(keep.begin(), keep.end(), keep_ratios);
        if (raw) std::copy(rw.begin(), rw.end(), raw);
        if (normalized) std::copy(nm.begin(), nm.end(), normalized);
        if (conc_median) std::copy(cm.begin(), cm.end(), conc_median);
        if (red_median) std::copy(rm.begin(), rm.end(), red_median);
    });
}

int qt_engine_save(qt_engine* e, const char* path) {
    return guard([&] {
        for (auto& l : e->lw)
            if (!l.loaded) fail(QT_EINVAL, "model weights not loaded");
        if (!e->head_loaded) fail(QT_EINVAL, "model head not loaded");
        FILE* f = std::fopen(path, "wb");
        if (!f) fail(QT_ERUNTIME, std::string("cannot open ") + path);
        std::unique_ptr<FILE, int (*)(FILE*)> guard_f(f, std::fclose);
        WFileHdr h = make_hdr(e);
        if (std::fwrite(&h, sizeof(h), 1, f) != 1) fail(QT_ERUNTIME, "write failed");
        if (h.has_act && std::fwrite(e->act.data(), sizeof(double), e->act.size(), f) != e->act.size())
            fail(QT_ERUNTIME, "write failed");
        ck(cudaStreamSynchronize(e->st), "sync");
        std::vector<char> buf;
        for_each_blob(e, [&](void* dev, size_t bytes) {
            buf.resize(bytes);
            ck(cudaMemcpy(buf.data(), dev, bytes, cudaMemcpyDeviceToHost), "weights readback");
            if (std::fwrite(buf.data(), 1, bytes, f) != bytes) fail(QT_ERUNTIME, "write failed");
        });
    });
}

int qt_engine_load(qt_engine* e, const char* path) {
    return guard([&] {
        FILE* f = std::fopen(path, "rb");
        if (!f) fail(QT_EINVAL, std::string("cannot open ") + path);
        std::unique_ptr<FILE, int (*)(FILE*)> guard_f(f, std::fclose);
        WFileHdr h{}, mine = make_hdr(e);
        if (std::fread(&h, sizeof(h), 1, f) != 1 || std::memcmp(h.magic, "QTW4B200", 8) != 0 || h.version != 1)
            fail(QT_EINVAL, "not a quota_b200 weight file");
        if (std::memcmp(&h.cfg, &mine.cfg, sizeof(qt_config)) != 0 || std::memcmp(h.geom, mine.geom, sizeof(h.geom)))
            fail(QT_EINVAL, "weight file does not match the engine configuration");
        if (h.has_act) {
            std::vector<double> act(4 * e->L + 1);
            if (std::fread(act.data(), sizeof(double), act.size(), f) != act.size()) fail(QT_EINVAL, "truncated file");
            ck(cudaStreamSynchronize(e->st), "sync");
            if (qt_engine_set_act_scales(e, act.data()) != 0) fail(QT_EINVAL, qt_last_error());
        }
        // stream through the pinned staging buffer
        const size_t chunk = std::min<size_t>(e->pin_cap, (size_t)32 << 20);
        ck(cudaStreamSynchronize(e->st), "sync");
        for_each_blob(e, [&](void* dev, size_t bytes) {
            for (size_t o = 0; o < bytes; o += chunk) {
                const size_t n = std::min(chunk, bytes - o);
                if (std::fread(e->pin, 1, n, f) != n) fail(QT_EINVAL, "truncated file");
                ck(cudaMemcpy(static_cast<char*>(dev) + o, e->pin, n, cudaMemcpyHostToDevice), "weights upload");
            }
        });
        for (auto& l : e->lw) {
            l.loaded = true;
            l.w8_ok = false;
        }
        e->head_loaded = true;
        e->head8_ok = false;
        e->graph_ok = false;
    });
}

int qt_engine_load_head(qt_engine* e, const float* w_head, const float* final_gain, int on_device) {
    return guard([&] {
        if (!w_head) fail(QT_EINVAL, "null weight");
        if (on_device) ck(cudaDeviceSynchronize(), "weights ready");
        e->quant_into(w_head, e->d, e->d, on_device, 1, 0, e->head, e->nd_pad, e->s_head);
        e->keep64(e->fp_head, w_head, (size_t)e->d * e->d, on_device);
        e->load_gain(e->gf, final_gain, on_device);
        e->head_loaded = true;
        e->head8_ok = false;
        e->graph_ok = false;
    });
}

int qt_engine_set_act_scales(qt_engine* e, const double* scales) {
    return guard([&] {
        if (!scales) fail(QT_EINVAL, "activation scales do not cover all layers");
        e->act.assign(scales, scales + 4 * e->L + 1);
        for (double s : e->act)
            if (!(s > 0.0) || !std::isfinite(s)) fail(QT_EINVAL, "activation scales must be positive");
        e->act_set = true;
        e->graph_ok = false;
    });
}

int qt_engine_set_recipe(qt_engine* e, int n, const int* layers, const double* keeps, const double* w4, int v0,
                         int res_bits) {
    return guard([&] {
        if (n == 0) {
            e->have_recipe = false;
            return;
        }
        // PruningRecipe::validate (recipe.cpp:21-46)
        if (n < 0 || !layers || !keeps) fail(QT_EINVAL, "candidate_layers and keep_ratios must align and be nonempty");
        for (int i = 0; i < n; ++i) {
            if (layers[i] < 0) fail(QT_EINVAL, "negative candidate layer");
            if (i > 0 && layers[i] <= layers[i - 1]) fail(QT_EINVAL, "candidate layers must be strictly increasing");
            const double r = keeps[i];
            if (!(r > 0.0 && r <= 1.0)) fail(QT_EINVAL, "keep ratio outside (0,1]");
            if (i > 0 && r > keeps[i - 1] + 1e-12) fail(QT_EINVAL, "keep ratios must be non-increasing");
        }
        const double w[4] = {w4 ? w4[0] : 0.25, w4 ? w4[1] : 0.45, w4 ? w4[2] : 0.10, w4 ? w4[3] : 0.20};
        for (double x : w)
            if (x < 0) fail(QT_EINVAL, "negative metric weight");
        if (std::fabs(w[0] + w[1] + w[2] + w[3] - 1.0) > 1e-6) fail(QT_EINVAL, "metric weights must sum to 1");  // selector.cpp:91-93
        if (v0 < 1) fail(QT_EINVAL, "v0 must be >= 1");
        // candidate layers >= n_layers are never reached, as with the reference hook
        // (model.cpp:404-405 calls it for l < n_layers only); the harness-level check
        // (harness.cpp:86-88) is the caller's
        if (res_bits == 0 || res_bits == 1 || res_bits > 8) fail(QT_EINVAL, "bits out of range [2,8]");
        e->recipe.layers.assign(layers, layers + n);
        e->recipe.keeps.assign(keeps, keeps + n);
        std::copy(w, w + 4, e->recipe.w);
        e->recipe.v0 = v0;
        e->recipe.res_bits = res_bits < 0 ? 0 : res_bits;
        e->have_recipe = true;
    });
}

int qt_engine_prefill(qt_engine* e, int n_seq, const float* emb, int emb_on_device, const int* visual,
                      const int* text, const int* v0, const int* positions, float* logits_out, int out_on_device) {
    return guard([&] {
        if (!emb || !visual || !text) fail(QT_EINVAL, "null argument");
        e->prefill(n_seq, emb, emb_on_device, 0, visual, text, v0, positions, logits_out, out_on_device);
    });
}

int qt_engine_prefill_f64(qt_engine* e, int n_seq, const double* emb, int emb_on_device, const int* visual,
                          const int* text, const int* v0, const int* positions, float* logits_out, int out_on_device) {
    return guard([&] {
        if (!emb || !visual || !text) fail(QT_EINVAL, "null argument");
        e->prefill(n_seq, emb, emb_on_device, 1, visual, text, v0, positions, logits_out, out_on_device);
    });
}

int qt_engine_prefill_rows(qt_engine* e) { return e->final_rows; }

int qt_engine_decode(qt_engine* e, const float* emb, int emb_on_device, float* logits_out, int out_on_device) {
    return guard([&] {
        if (!emb) fail(QT_EINVAL, "embedding width mismatch");
        e->decode(emb, emb_on_device, 0, logits_out, out_on_device);
    });
}

int qt_engine_set_graphs(qt_engine* e, int on) {
    return guard([&] { e->use_graphs = on != 0; });
}

int qt_engine_set_token_table(qt_engine* e, const float* table, int vocab, int on_device) {
    return guard([&] {
        if (vocab < 1 || vocab > e->d) fail(QT_EINVAL, "vocab must be in [1, d_model] (the logits' width)");
        if (!table) fail(QT_EINVAL, "null token table");
        ck(cudaStreamSynchronize(e->st), "sync");
        if (e->tok_table) cudaFree(e->tok_table);
        e->tok_table = dalloc<float>((size_t)vocab * e->d);
        if (!e->dec_tok) e->dec_tok = dalloc<int>(e->max_batch);
        if (!e->last_rows) e->last_rows = dalloc<int>(e->max_batch);
        ck(cudaMemcpyAsync(e->tok_table, table, (size_t)vocab * e->d * sizeof(float),
                           on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, e->st),
           "token table");
        ck(cudaStreamSynchronize(e->st), "token table");
        e->vocab = vocab;
        e->graph_g_ok = false;
    });
}

int qt_engine_decode_greedy(qt_engine* e, int* tokens_out, float* logits_out, int out_on_device) {
    return guard([&] { e->decode(nullptr, 0, 0, logits_out, out_on_device, tokens_out); });
}

int qt_engine_decode_f64(qt_engine* e, const double* emb, int emb_on_device, float* logits_out, int out_on_device) {
    return guard([&] {
        if (!emb) fail(QT_EINVAL, "embedding width mismatch");
        e->decode(emb, emb_on_device, 1, logits_out, out_on_device);
    });
}

int qt_engine_layout(qt_engine* e, int seq, int* visual, int* text, int* positions, int cap) {
    return guard([&] {
        if (seq < 0 || seq >= e->B) fail(QT_ERANGE, "sequence out of range");
        *visual = e->h_vis[seq];
        *text = e->h_txt[seq];
        const auto& p = e->h_pos[seq];
        if ((int)p.size() > cap) fail(QT_EINVAL, "buffer too small");
        if (positions) std::copy(p.begin(), p.end(), positions);
    });
}

int qt_engine_scores(qt_engine* e, int layer, int seq, double* fused, double* norm4, int cap, int* n) {
    return guard([&] {
        if (seq < 0 || seq >= e->B) fail(QT_ERANGE, "sequence out of range");
        size_t ev = e->ev_layers.size();
        for (size_t i = 0; i < e->ev_layers.size(); ++i)
            if (e->ev_layers[i] == layer) ev = i;
        if (ev == e->ev_layers.size()) fail(QT_ERANGE, "no selection ran at this layer");
        const int V = e->ev_vis[ev][seq];
        *n = V;
        if (!fused && !norm4) return;
        if (V > cap) fail(QT_EINVAL, "buffer too small");
        ck(cudaStreamSynchronize(e->st), "sync");
        const size_t vs = e->vstride;
        if (fused)
            ck(cudaMemcpy(fused, e->sc_fused + (ev * e->max_batch + seq) * vs, V * sizeof(double),
                          cudaMemcpyDeviceToHost),
               "scores");
        if (norm4)
            for (int m = 0; m < 4; ++m)
                ck(cudaMemcpy(norm4 + (size_t)m * V, e->sc_norm + ((ev * e->max_batch + seq) * 4 + m) * vs,
                              V * sizeof(double), cudaMemcpyDeviceToHost),
                   "scores");
    });
}

int qt_engine_n_prunes(qt_engine* e, int seq) {
    if (seq < 0 || seq >= e->B) return -1;
    return (int)e->trace[seq].size();
}

int qt_engine_prune(qt_engine* e, int seq, int i, int* layer, int* budget, int* positions, int cap, int* count) {
    return guard([&] {
        const PruneEv& ev = e->trace.at(seq).at(i);
        *layer = ev.layer;
        *budget = ev.budget;
        if ((int)ev.positions.size() > cap) fail(QT_EINVAL, "buffer too small");
        std::copy(ev.positions.begin(), ev.positions.end(), positions);
        *count = (int)ev.positions.size();
    });
}

int qt_engine_kv(qt_engine* e, int layer, int seq, int kv_head, int which, int8_t* codes, float* scales, int* rows,
                 int cap_rows) {
    return guard([&] {
        if (layer < 0 || layer >= e->L || seq < 0 || seq >= e->B || kv_head < 0 || kv_head >= e->Hkv)
            fail(QT_ERANGE, "kv index out of range");
        ck(cudaStreamSynchronize(e->st), "sync");
        const int n = e->h_kvlen[(size_t)layer * e->B + seq];
        *rows = n;
        if (!codes) return;
        if (n > cap_rows) fail(QT_EINVAL, "buffer too small");
        std::vector<int> hpt(e->max_pages);
        ck(cudaMemcpy(hpt.data(), e->pt + ((size_t)layer * e->max_batch + seq) * e->max_pages,
                      e->max_pages * sizeof(int), cudaMemcpyDeviceToHost),
           "page table");
        const int dh = e->dh;
        const size_t cb = (size_t)e->Hkv * qt::kPage * (dh / 2);
        std::vector<uint8_t> page(e->page_bytes);
        for (int r0 = 0; r0 < n; r0 += qt::kPage) {
            ck(cudaMemcpy(page.data(), e->pool + (long long)hpt[r0 / qt::kPage] * e->page_bytes, e->page_bytes,
                          cudaMemcpyDeviceToHost),
               "page");
            for (int r = r0; r < std::min(n, r0 + qt::kPage); ++r) {
                const int slot = r % qt::kPage;
                const uint8_t* src = page.data() + (which ? cb : 0) + ((size_t)kv_head * qt::kPage + slot) * (dh / 2);
                for (int c = 0; c < dh; ++c) {
                    int nibv = (src[c / 2] >> (4 * (c & 1))) & 0xF;
                    codes[(size_t)r * dh + c] = (int8_t)(nibv >= 8 ? nibv - 16 : nibv);
                }
                const float* sc = reinterpret_cast<const float*>(page.data() + 2 * cb);
                scales[r] = sc[(which ? e->Hkv * qt::kPage : 0) + kv_head * qt::kPage + slot];
            }
        }
    });
}

int qt_engine_profile_chain(qt_engine* e, int skip_mask, int reps, double* ms_per_step) {
    return guard([&] {
        if (!ms_per_step) fail(QT_EINVAL, "null argument");
        *ms_per_step = e->profile_chain(skip_mask, reps);
    });
}

int qt_engine_set_records(qt_engine* e, int mode) {
    return guard([&] {
        if (mode < 0 || mode > 3) fail(QT_EINVAL, "record mode must be 0..3");
        e->rec_mode = mode;
    });
}

int qt_engine_set_prune_hook(qt_engine* e, qt_prune_hook_fn hook, void* user) {
    return guard([&] {
        e->host_hook = hook;
        e->host_user = user;
    });
}

int qt_engine_record_count(qt_engine* e) { return (int)e->lrecs.size(); }

int qt_engine_record_get(qt_engine* e, int i, int* meta, int* positions, double* states, float* probs) {
    return guard([&] {
        if (i < 0 || i >= (int)e->lrecs.size()) fail(QT_ERANGE, "record out of range");
        const auto& r = e->lrecs[i];
        if (meta) {
            meta[0] = r.layer;
            meta[1] = r.V;
            meta[2] = r.T;
            meta[3] = e->H;
        }
        if (positions) std::copy(r.pos.begin(), r.pos.end(), positions);
        if (states) std::copy(r.states.begin(), r.states.end(), states);
        if (probs) std::copy(r.probs.begin(), r.probs.end(), probs);
    });
}

int qt_engine_block_output(qt_engine* e, int layer, double* out, long long cap, int* rows) {
    return guard([&] {
        if (layer < 0 || layer >= (int)e->blocks.size()) fail(QT_ERANGE, "no block output for this layer");
        const auto& b = e->blocks[layer];
        *rows = (int)(b.size() / e->d);
        if (!out) return;
        if ((long long)b.size() > cap) fail(QT_EINVAL, "buffer too small");
        std::copy(b.begin(), b.end(), out);
    });
}

int qt_engine_capture(qt_engine* e, int on) {
    return guard([&] {
        e->capture = on != 0;
        e->caps.clear();
        e->caps.shrink_to_fit();
    });
}

int qt_engine_capture_count(qt_engine* e) { return (int)e->caps.size(); }

int qt_engine_capture_get(qt_engine* e, int i, int* meta, int8_t* codes, double* scales) {
    return guard([&] {
        if (i < 0 || i >= (int)e->caps.size()) fail(QT_ERANGE, "capture record out of range");
        const auto& r = e->caps[i];
        const int m[6] = {r.phase, r.layer, r.site, r.rows, r.cols, r.groups};
        std::copy(m, m + 6, meta);
        if (codes) std::memcpy(codes, r.codes.data(), r.codes.size());
        if (scales) std::copy(r.scales.begin(), r.scales.end(), scales);
    });
}

int qt_engine_profile_next(qt_engine* e) {
    e->prof_next = true;
    return 0;
}

int qt_engine_profile_read(qt_engine* e, double* out) {
    std::copy(e->prof_out, e->prof_out + P_NCLASS * 4, out);
    return P_NCLASS;
}

int qt_engine_info(qt_engine* e, int64_t* o) {
    o[0] = (int64_t)(uintptr_t)e->st;
    o[1] = e->n_pages_cap;
    o[2] = e->page_bytes;
    o[3] = e->dec_splits;
    o[4] = e->dec_pps;
    o[5] = e->final_rows;
    o[6] = e->B;
    o[7] = e->decode_steps;
    // weight bytes (codes + scales) streamed per decode step
    int64_t wb = 0;
    wb += (int64_t)e->L * ((int64_t)e->n_qkv * e->kd_pad / 2 + (int64_t)e->d * e->kd_pad / 2 +
                           (int64_t)e->n_gu * e->kd_pad / 2 + (int64_t)e->d * e->kff_pad / 2);
    wb += (int64_t)e->d * e->kd_pad / 2;
    wb += (int64_t)4 * (e->L * (e->n_qkv + e->d + e->n_gu + e->d) + e->d);
    o[8] = wb;
    int64_t kvb = 0;
    for (int v : e->h_kvlen) kvb += (int64_t)v;
    o[9] = kvb;  // cached rows summed over (layer, seq)
    o[10] = (int64_t)(uintptr_t)e->pool;
    o[11] = e->n_qkv;
    o[12] = e->kd_pad;
    o[13] = e->kff_pad;
    o[14] = e->n_gu;
    o[15] = 0;
    return 0;
}

// ---- per-kernel ABI -------------------------------------------------------

int qt_rmsnorm_quant_i4(const void* x, int x_is_f64, int ld_x, const float* gain, int M, int D, int d_pad,
                        int act_mode, double static_scale, uint8_t* codes, int ld_codes, double* scales,
                        float* normed, void* stream) {
    return guard([&] {
        ckl(qt_launch_norm_quant(x, x_is_f64, ld_x, gain, M, D, d_pad, 4, act_mode, static_scale, codes, ld_codes,
                                 scales, normed, nullptr, 0, (cudaStream_t)stream),
            "rmsnorm+quant");
    });
}

int qt_w4a4_gemm(int epi, const uint8_t* a, int lda, const double* sa, const uint8_t* w, int ldw, const double* sw,
                 int M, int N, int K, void* out, int ldo, int32_t* acc_out, int impl, void* stream) {
    return guard([&] {
        const cudaStream_t cs = (cudaStream_t)stream;
        if (impl == 3 || impl == 4) {  // int8-operand tcgen05 GEMM: operands widened to int8 first (test / ABI
                                       // path); impl 4 with the 2-SM kernel's split-K workspace
            int8_t *a8 = nullptr, *w8 = nullptr;
            int* ws = nullptr;
            ck(cudaMalloc(&a8, (size_t)lda * K), "int8 activations");
            ck(cudaMalloc(&w8, (size_t)ldw * K), "int8 weights");
            if (impl == 4)
                ck(cudaMalloc(&ws, (size_t)std::max(1, qt_tc05_i8_splitk(M, N, K)) * M * N * sizeof(int)), "split-K ws");
            int rc = qt_launch_w4t_to_i8(a, lda, K, a8, cs);
            if (!rc) rc = qt_launch_w4t_to_i8(w, ldw, K, w8, cs);
            if (!rc)
                rc = qt_launch_w4a4_tc05_i8(epi, a8, K, sa, w8, ldw, K, sw, M, N, K, out, ldo, acc_out, nullptr, 0,
                                            nullptr, ws, cs);
            cudaStreamSynchronize(cs);
            cudaFree(a8);
            cudaFree(w8);
            if (ws) cudaFree(ws);
            ckl(rc, "w4a4 gemm (int8 operands)");
            return;
        }
        int* ws = nullptr;  // impl 2: tcgen05 with split-K (a grow-only ABI-level workspace, so a
                            // timing loop over one shape allocates once)
        if (impl == 2) {
            static std::mutex mu;
            static int* g_ws = nullptr;
            static size_t g_bytes = 0;
            std::lock_guard<std::mutex> lk(mu);
            const size_t need = (size_t)std::max(qt_tc05_splitk(M, N, K), 1) * M * N * sizeof(int);
            if (need > g_bytes) {
                cudaStreamSynchronize(cs);
                if (g_ws) cudaFree(g_ws);
                g_ws = nullptr;
                g_bytes = 0;
                ck(cudaMalloc(&g_ws, need), "split-K workspace");
                g_bytes = need;
            }
            ws = g_ws;
            ckl(impl >= 1 ? qt_launch_w4a4_tc05(epi, a, lda, sa, w, ldw, sw, M, N, K, out, ldo, acc_out, ws, cs) : 0,
                "w4a4 gemm");
            return;
        }
        int rc = impl >= 1 ? qt_launch_w4a4_tc05(epi, a, lda, sa, w, ldw, sw, M, N, K, out, ldo, acc_out, ws, cs)
                           : qt_launch_w4a4_mma(epi, a, lda, sa, w, ldw, sw, M, N, K, out, ldo, acc_out, cs);
        ckl(rc, "w4a4 gemm");
    });
}

int qt_w4a4_gemm_i8(int epi, const int8_t* a8, int lda8, const double* sa, const int8_t* w8, int w_rows, int ldw8,
                    const double* sw, int M, int N, int K, void* out, int ldo, int32_t* acc_out, int* workspace,
                    int flags, void* stream) {
    return guard([&] {
        ckl(qt_launch_w4a4_tc05_i8_ex(epi, a8, lda8, sa, w8, w_rows, ldw8, sw, M, N, K, out, ldo, acc_out, nullptr, 0,
                                      nullptr, workspace, flags, (cudaStream_t)stream),
            "w4a4 gemm (int8 operands)");
    });
}

int64_t qt_w4a4_gemm_i8_workspace(int M, int N, int K) {
    const int ks = qt_tc05_i8_splitk(M, N, K);
    return ks > 1 ? (int64_t)ks * M * N * (int64_t)sizeof(int) : 0;
}


int qt_quant_weight_i4(const float* w, int K, int N, int row_mul, int row_add, uint8_t* codes, int ldc,
                       double* scales, double* scratch, void* stream) {
    return guard([&] {
        ckl(qt_launch_weight_quant(w, K, N, 4, row_mul, row_add, codes, ldc, scales, scratch, (cudaStream_t)stream),
            "weight quantize");
    });
}

int qt_kv_quant_append_i4(float* qkv, int ld_qkv, int M, int H, int Hkv, int d_head, const int* positions,
                          const int* tok_seq, const int* tok_row, const double* rope_table, const int* page_table,
                          int max_pages, uint8_t* pool, int64_t page_bytes, float* k_out, void* stream) {
    return guard([&] {
        ckl(qt_launch_rope_kv_append(qkv, ld_qkv, M, H, Hkv, d_head, positions, tok_seq, tok_row, rope_table,
                                     page_table, max_pages, pool, page_bytes, 4, k_out, (cudaStream_t)stream),
            "kv quant append");
    });
}

int qt_unpack_codes(const uint8_t* tiled, int rows_pad, int rows, int K, int8_t* out, void* stream) {
    return guard([&] {
        if (rows < 0 || rows > rows_pad || rows_pad % 16 || K % 2) fail(QT_EINVAL, "invalid code matrix shape");
        ckl(qt_launch_unpack_codes(tiled, rows_pad, rows, K, out, (cudaStream_t)stream), "unpack codes");
    });
}

int qt_attn_prefill_i4kv(const float* q, int ldq, int B, int H, int Hkv, int d_head, const int* seq_off,
                         const int* visual, const int* seq_len, int smax, const uint8_t* pool, int64_t page_bytes,
                         const int* page_table, int max_pages, float* out, int ldo, float* row_stats, void* stream) {
    return guard([&] {
        if (B < 0 || H < 1 || Hkv < 1 || H % Hkv) fail(QT_EINVAL, "invalid attention heads");
        if (d_head != 64 && d_head != 128) fail(QT_EINVAL, "d_head must be 64 or 128 on the B200 path");
        ckl(qt_launch_attn_prefill(q, ldq, H, Hkv, d_head, seq_off, visual, seq_len, B, smax, pool, page_bytes,
                                   page_table, max_pages, out, ldo, row_stats, nullptr, 0, (cudaStream_t)stream),
            "prefill attention");
    });
}

int64_t qt_attn_decode_workspace(int B, int H, int d_head, int max_len) {
    const int pages = (max_len + qt::kPage - 1) / qt::kPage;
    return (int64_t)B * H * pages * (d_head + 2) * (int64_t)sizeof(float);
}

int qt_attn_decode_i4kv(const float* q, int ldq, int B, int H, int Hkv, int d_head, const int* kv_len, int max_len,
                        const uint8_t* pool, int64_t page_bytes, const int* page_table, int max_pages, float* out,
                        int ldo, void* workspace, void* stream) {
    return guard([&] {
        if (B < 0 || H < 1 || Hkv < 1 || H % Hkv) fail(QT_EINVAL, "invalid attention heads");
        if (d_head != 64 && d_head != 128) fail(QT_EINVAL, "d_head must be 64 or 128 on the B200 path");
        if (max_len < 1 || (max_len + qt::kPage - 1) / qt::kPage > max_pages) fail(QT_EINVAL, "max_len exceeds the page table");
        if (!workspace) fail(QT_EINVAL, "null workspace");
        const int pages = (max_len + qt::kPage - 1) / qt::kPage;
        float* part_ml = static_cast<float*>(workspace);
        float* part_o = part_ml + (size_t)B * H * pages * 2;
        int dev = 0, sms = 148, pps = 1, nsplit = 1;
        ck(cudaGetDevice(&dev), "device");
        ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
        if (qt_attn_decode_plan(B, H, Hkv, pages, sms, &pps, &nsplit)) fail(QT_EINVAL, "decode attention plan");
        ckl(qt_launch_attn_decode(q, ldq, H, Hkv, d_head, kv_len, B, const_cast<uint8_t*>(pool), page_bytes,
                                  page_table, max_pages, pps, nsplit, nullptr, nullptr, part_ml, part_o, out, ldo,
                                  nullptr, 0, nullptr, 1, 0.0, 0, 4, nullptr, 0, (cudaStream_t)stream),
            "decode attention");
    });
}

int qt_quota_score(const double* x, int d_model, const float* q, int ldq, int B, int H, int Hkv, int d_head,
                   const int* seq_off, const int* visual, const int* seq_len, int vmax, const uint8_t* pool,
                   int64_t page_bytes, const int* page_table, int max_pages, const float* row_stats, int res_bits,
                   double* metrics, int vstride, void* workspace, void* stream) {
    return guard([&] {
        if (B < 0 || H < 1 || Hkv < 1 || H % Hkv) fail(QT_EINVAL, "invalid attention heads");
        if (vmax > vstride) fail(QT_EINVAL, "visual prefix exceeds vstride");
        if (res_bits == 0 || res_bits == 1 || res_bits > 8) fail(QT_EINVAL, "bits out of range [2,8]");
        if (!workspace || !row_stats) fail(QT_EINVAL, "null workspace / row statistics");
        const cudaStream_t cs = (cudaStream_t)stream;
        float* inter = static_cast<float*>(workspace);
        float* intra = inter + (size_t)B * H * vstride;
        double* mag = reinterpret_cast<double*>(intra + (size_t)B * H * vstride);
        double* res = mag + (size_t)B * vstride;
        ckl(qt_launch_attn_colsum(q, ldq, H, Hkv, d_head, seq_off, visual, seq_len, B, vmax, pool, page_bytes,
                                  page_table, max_pages, row_stats, vstride, inter, intra, nullptr, 0, 0, cs),
            "quota attention metrics");
        ckl(qt_launch_token_metrics(x, d_model, seq_off, visual, vmax, B, vstride, res_bits < 0 ? 0 : res_bits, mag,
                                    res, cs),
            "quota token metrics");
        ckl(qt_launch_metrics_pack(mag, res, inter, intra, H, vstride, visual, B, metrics, cs), "metrics pack");
    });
}

int64_t qt_quota_score_workspace(int B, int H, int vstride) {
    return (int64_t)2 * B * H * vstride * (int64_t)sizeof(float) + (int64_t)2 * B * vstride * (int64_t)sizeof(double);
}

int qt_topk_compact(const double* metrics, int B, int vstride, const int* visual, const int* text, const int* budget,
                    const double* weights4, const int* seq_off, const int* new_off, const int* new_len,
                    const double* x, int d_model, const int* pos, int new_rows, double* x_out, int* pos_out,
                    uint8_t* pool, int64_t page_bytes, const int* page_table, int max_pages, int Hkv, int d_head,
                    int* keep_local, int* keep_src, int* kept_pos, void* stream) {
    return guard([&] {
        if (B < 0 || vstride < 1) fail(QT_EINVAL, "invalid top-k shape");
        if (!weights4) fail(QT_EINVAL, "null metric weights");
        const cudaStream_t cs = (cudaStream_t)stream;
        ckl(qt_launch_select_topk(nullptr, nullptr, nullptr, nullptr, 1, vstride, visual, text, budget, seq_off,
                                  new_off, B, vstride, weights4, keep_src, keep_local, vstride, pos, kept_pos,
                                  nullptr, nullptr, metrics, 0, cs),
            "quota top-k");
        ckl(qt_launch_gather_rows(x, x_out, d_model, pos, pos_out, keep_src, new_rows, cs), "compaction gather");
        if (pool)
            ckl(qt_launch_kv_compact(pool, page_bytes, page_table, max_pages, Hkv, d_head, keep_local, vstride,
                                     new_len, B, cs),
                "kv compaction");
    });
}

int qt_quota_topk(const double* metrics, int B, int vstride, const int* visual, const int* budget,
                  const double* weights4, int* slots, double* fused_out, double* norm_out, void* stream) {
    return guard([&] {
        if (B < 0 || vstride < 1) fail(QT_EINVAL, "invalid top-k shape");
        ckl(qt_launch_select_topk(nullptr, nullptr, nullptr, nullptr, 1, vstride, visual, nullptr, budget, nullptr,
                                  nullptr, B, vstride, weights4, nullptr, slots, vstride, nullptr, nullptr, fused_out,
                                  norm_out, metrics, weights4 ? 0 : 1, (cudaStream_t)stream),
            "quota top-k");
    });
}

}  // extern "C"
