// oracle/ref_capi.cpp -- C-ABI shim over the UNMODIFIED reference library (R0).
//
// TEST INFRASTRUCTURE ONLY.  This file is compiled together with the
// reference sources where they lie (/root/reference/proj/src/*.cpp) into
// oracle/_ref/libquota_ref.so by oracle/Makefile.  It adds no arithmetic of
// its own: every entry point marshals plain arrays into the reference's
// public C++ types (proj/include/quota/*.hpp) and calls the reference
// function named in its comment.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load it.
//
// Error convention: 0 = OK, -1 = std::invalid_argument, -2 = runtime_error,
// -3 = out_of_range, -4 = other; qref_last_error() returns the message.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "quota/calibrator.hpp"
#include "quota/digest.hpp"
#include "quota/gflops.hpp"
#include "quota/model.hpp"
#include "quota/numeric.hpp"
#include "quota/quant.hpp"
#include "quota/recipe.hpp"
#include "quota/rng.hpp"
#include "quota/selector.hpp"

using namespace quota;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return -3;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return -2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -4;
    }
}

Matrix mat(const double* p, int rows, int cols) {
    return Matrix(rows, cols, std::vector<double>(p, p + static_cast<size_t>(rows) * cols));
}

struct RefModel {
    Model model;
    std::unique_ptr<QuantEnv> env;
};

struct RefRun {
    RefModel* owner = nullptr;
    ForwardResult result;
    bool quantized = false;
};

}  // namespace

extern "C" {

const char* qref_last_error() { return g_err.c_str(); }

// ---- quantizer (quant.cpp) -------------------------------------------------

// round_half_even (quant.cpp:39-45)
double qref_round_half_even(double x) { return round_half_even(x); }

// fit_params + quantize (quant.cpp:47-91); axis 0/1/2 = PerTensor/PerRow/PerColumn
int qref_quantize_fit(const double* x, int rows, int cols, int bits, int axis, double* scales_out,
                      int8_t* codes_out) {
    return guard([&] {
        Matrix m = mat(x, rows, cols);
        QuantParams p = fit_params(m, bits, static_cast<GroupAxis>(axis));
        QuantizedTensor t = quantize(m, p);
        std::copy(p.scales.begin(), p.scales.end(), scales_out);
        std::memcpy(codes_out, t.codes.data(), t.codes.size());
    });
}

// quantize with caller-provided scales (quant.cpp:71-91), then dequantize (93-102)
int qref_quantize_with(const double* x, int rows, int cols, int bits, int axis, const double* scales,
                       int n_scales, int8_t* codes_out, double* deq_out) {
    return guard([&] {
        Matrix m = mat(x, rows, cols);
        QuantParams p;
        p.bits = bits;
        p.axis = static_cast<GroupAxis>(axis);
        p.scales.assign(scales, scales + n_scales);
        QuantizedTensor t = quantize(m, p);
        if (codes_out) std::memcpy(codes_out, t.codes.data(), t.codes.size());
        if (deq_out) {
            Matrix d = dequantize(t);
            std::copy(d.data.begin(), d.data.end(), deq_out);
        }
    });
}

// fake_quant_per_row (quant.cpp:108-110)
int qref_fake_quant_per_row(const double* x, int rows, int cols, int bits, double* out) {
    return guard([&] {
        Matrix d = fake_quant_per_row(mat(x, rows, cols), bits);
        std::copy(d.data.begin(), d.data.end(), out);
    });
}

// kv_quantize (quant.cpp:117-119)
int qref_kv_quantize(const double* x, int rows, int cols, int bits, int8_t* codes_out,
                     double* scales_out) {
    return guard([&] {
        QuantizedTensor t = kv_quantize(mat(x, rows, cols), bits);
        std::memcpy(codes_out, t.codes.data(), t.codes.size());
        std::copy(t.params.scales.begin(), t.params.scales.end(), scales_out);
    });
}

// quantized_linear (quant.cpp:112-115); w quantized PerRow as in the reference test
int qref_quantized_linear(const double* x, int m, int k, const int8_t* w_codes, const double* w_scales,
                          int w_axis, int n, int act_bits, double* out) {
    return guard([&] {
        QuantizedTensor w;
        w.rows = k;
        w.cols = n;
        w.codes.assign(w_codes, w_codes + static_cast<size_t>(k) * n);
        w.params.bits = 4;
        w.params.axis = static_cast<GroupAxis>(w_axis);
        int groups = w_axis == 0 ? 1 : (w_axis == 1 ? k : n);
        w.params.scales.assign(w_scales, w_scales + groups);
        Matrix y = quantized_linear(mat(x, m, k), w, act_bits);
        std::copy(y.data.begin(), y.data.end(), out);
    });
}

// ---- numeric core (numeric.cpp) ----------------------------------------------

int qref_matmul(const double* a, int m, int k, const double* b, int n, double* out) {
    return guard([&] {
        Matrix c = matmul(mat(a, m, k), mat(b, k, n));
        std::copy(c.data.begin(), c.data.end(), out);
    });
}

int qref_percentile(const double* v, int n, double p, double* out) {
    return guard([&] { *out = percentile(std::span<const double>(v, static_cast<size_t>(n)), p); });
}

int qref_rms_norm_rows(const double* x, int rows, int cols, const double* gain, double* out) {
    return guard([&] {
        Matrix r = rms_norm_rows(mat(x, rows, cols), std::span<const double>(gain, cols));
        std::copy(r.data.begin(), r.data.end(), out);
    });
}

int qref_rope(double* v, int n, int position) {
    return guard([&] { rope_in_place(std::span<double>(v, n), position); });
}

double qref_silu(double x) { return silu(x); }

// ---- selector (selector.cpp) --------------------------------------------------

// compute_metrics (selector.cpp:19-68) on a LayerActivationRecord built from flat arrays:
// visual [n x d], text [t x d], inter [heads][t x n], intra [heads][n x n];
// res_bits < 0 = nullopt.  out: [4][n] = mag, inter, intra, res.
int qref_compute_metrics(const double* visual, int n, int d, const double* text, int t, int heads,
                         const double* inter, const double* intra, int res_bits, double* out) {
    return guard([&] {
        LayerActivationRecord rec;
        rec.visual_states = mat(visual, n, d);
        rec.text_states = mat(text, t, d);
        for (int h = 0; h < heads; ++h) {
            rec.attn_inter.push_back(mat(inter + static_cast<size_t>(h) * t * n, t, n));
            rec.attn_intra.push_back(mat(intra + static_cast<size_t>(h) * n * n, n, n));
        }
        TokenMetrics m = compute_metrics(rec, res_bits < 0 ? std::nullopt : std::optional<int>(res_bits));
        const Vector* v[4] = {&m.mag, &m.inter, &m.intra, &m.res};
        for (int i = 0; i < 4; ++i) std::copy(v[i]->begin(), v[i]->end(), out + static_cast<size_t>(i) * n);
    });
}

int qref_compute_budget(double keep_ratio, int v0, int* out) {
    return guard([&] { *out = compute_budget(keep_ratio, v0); });
}

int qref_robust_normalize(const double* v, int n, double* out) {
    return guard([&] {
        Vector r = robust_normalize(std::span<const double>(v, static_cast<size_t>(n)));
        std::copy(r.begin(), r.end(), out);
    });
}

// select_top_k (selector.cpp:117-136); slots_out needs room for min(k, n)
int qref_select_top_k(const double* scores, int n, int k, int* slots_out, int* count_out) {
    return guard([&] {
        RetainedSet rs = select_top_k(std::span<const double>(scores, static_cast<size_t>(n)), k);
        std::copy(rs.slots.begin(), rs.slots.end(), slots_out);
        *count_out = static_cast<int>(rs.slots.size());
    });
}

// compute_metrics + score_tokens (selector.cpp:19-115).
// visual [n x d]; inter [heads x t x n]; intra [heads x n x n]; weights4 =
// {mag, inter, intra, quant}; res_bits < 0 means nullopt.
// metrics_out / norm_out are [4 x n] in (mag, inter, intra, res) order.
int qref_score_tokens(const double* visual, int n, int d, int heads, int t, const double* inter,
                      const double* intra, const double* weights4, int res_bits, double* metrics_out,
                      double* norm_out, double* fused_out) {
    return guard([&] {
        LayerActivationRecord rec;
        rec.visual_states = mat(visual, n, d);
        for (int h = 0; h < heads; ++h) {
            rec.attn_inter.push_back(mat(inter + static_cast<size_t>(h) * t * n, t, n));
            rec.attn_intra.push_back(mat(intra + static_cast<size_t>(h) * n * n, n, n));
        }
        std::optional<int> rb = res_bits < 0 ? std::nullopt : std::optional<int>(res_bits);
        TokenMetrics m = compute_metrics(rec, rb);
        MetricWeights w{weights4[0], weights4[1], weights4[2], weights4[3]};
        ScoreVector s = score_tokens(m, w);
        const Vector* ms[4] = {&m.mag, &m.inter, &m.intra, &m.res};
        const Vector* ns[4] = {&s.mag_n, &s.inter_n, &s.intra_n, &s.res_n};
        for (int i = 0; i < 4; ++i) {
            if (metrics_out) std::copy(ms[i]->begin(), ms[i]->end(), metrics_out + static_cast<size_t>(i) * n);
            if (norm_out) std::copy(ns[i]->begin(), ns[i]->end(), norm_out + static_cast<size_t>(i) * n);
        }
        if (fused_out) std::copy(s.fused.begin(), s.fused.end(), fused_out);
    });
}

// ---- recipe (recipe.cpp) ------------------------------------------------------

// parse_recipe (recipe.cpp:91-116).  Arrays sized by the caller (max_layers).
int qref_parse_recipe(const char* text, int max_layers, int* n_layers, int* layers, double* keeps,
                      double* weights4, int* v0, char* digest_buf, int digest_cap) {
    return guard([&] {
        PruningRecipe r = parse_recipe(text);
        if (static_cast<int>(r.candidate_layers.size()) > max_layers) {
            throw std::invalid_argument("too many candidate layers for caller buffer");
        }
        *n_layers = static_cast<int>(r.candidate_layers.size());
        std::copy(r.candidate_layers.begin(), r.candidate_layers.end(), layers);
        std::copy(r.keep_ratios.begin(), r.keep_ratios.end(), keeps);
        weights4[0] = r.weights.mag;
        weights4[1] = r.weights.inter;
        weights4[2] = r.weights.intra;
        weights4[3] = r.weights.quant;
        *v0 = r.v0;
        std::snprintf(digest_buf, static_cast<size_t>(digest_cap), "%s", r.quant_digest.c_str());
    });
}

// serialize_recipe (recipe.cpp:48-61) + recipe_digest (132-134)
int qref_serialize_recipe(int n_layers, const int* layers, const double* keeps, const double* weights4,
                          int v0, const char* quant_digest, char* out, int cap, char* digest16) {
    return guard([&] {
        PruningRecipe r;
        r.candidate_layers.assign(layers, layers + n_layers);
        r.keep_ratios.assign(keeps, keeps + n_layers);
        r.weights = {weights4[0], weights4[1], weights4[2], weights4[3]};
        r.v0 = v0;
        r.quant_digest = quant_digest;
        std::string s = serialize_recipe(r);
        if (static_cast<int>(s.size()) + 1 > cap) throw std::invalid_argument("buffer too small");
        std::memcpy(out, s.c_str(), s.size() + 1);
        std::string dg = recipe_digest(r);
        std::memcpy(digest16, dg.c_str(), 17);
    });
}

// executed_visual_lengths (gflops.cpp:53-72)
int qref_executed_visual_lengths(const char* recipe_json, int n_layers, int* out) {
    return guard([&] {
        std::vector<int> v = executed_visual_lengths(parse_recipe(recipe_json), n_layers);
        std::copy(v.begin(), v.end(), out);
    });
}

// layer_cost (gflops.cpp:16-22)
double qref_layer_cost(int seq_len, int d_model, int d_ff, int n_heads) {
    CostModel cm;
    cm.d_model = d_model;
    cm.d_ff = d_ff;
    cm.n_heads = n_heads;
    return layer_cost(seq_len, cm);
}

// ---- model (model.cpp) --------------------------------------------------------

// init_model (model.cpp:113-135).  Weights can then be read back or overwritten.
void* qref_model_create(int n_layers, int n_heads, int d_model, int d_head, uint64_t seed) {
    RefModel* m = nullptr;
    int rc = guard([&] {
        ModelConfig c;
        c.n_layers = n_layers;
        c.n_heads = n_heads;
        c.d_model = d_model;
        c.d_head = d_head;
        c.seed = seed;
        m = new RefModel{init_model(c), nullptr};
    });
    return rc == 0 ? m : nullptr;
}

void qref_model_free(void* h) { delete static_cast<RefModel*>(h); }

uint64_t qref_model_weight_checksum(void* h) { return static_cast<RefModel*>(h)->model.weight_checksum(); }

// which: 0 wq, 1 wk, 2 wv, 3 wo, 4 w1, 5 w2, 6 norm1, 7 norm2; layer -1 with
// which 0 = w_head, 6 = final_norm_gain.  Row-major as stored (W is d_in x d_out).
static double* weight_ptr(RefModel* m, int layer, int which, size_t* count) {
    Model& md = m->model;
    if (layer < 0) {
        if (which == 0) {
            *count = md.w_head.data.size();
            return md.w_head.data.data();
        }
        *count = md.final_norm_gain.size();
        return md.final_norm_gain.data();
    }
    LayerWeights& l = md.layers.at(static_cast<size_t>(layer));
    Matrix* ms[6] = {&l.wq, &l.wk, &l.wv, &l.wo, &l.w1, &l.w2};
    if (which < 6) {
        *count = ms[which]->data.size();
        return ms[which]->data.data();
    }
    Vector& g = which == 6 ? l.norm1_gain : l.norm2_gain;
    *count = g.size();
    return g.data();
}

int qref_model_get_weight(void* h, int layer, int which, double* out, int64_t cap) {
    return guard([&] {
        size_t n = 0;
        double* p = weight_ptr(static_cast<RefModel*>(h), layer, which, &n);
        if (static_cast<int64_t>(n) > cap) throw std::invalid_argument("buffer too small");
        std::copy(p, p + n, out);
    });
}

int qref_model_set_weight(void* h, int layer, int which, const double* in, int64_t count) {
    return guard([&] {
        size_t n = 0;
        double* p = weight_ptr(static_cast<RefModel*>(h), layer, which, &n);
        if (static_cast<int64_t>(n) != count) throw std::invalid_argument("weight size mismatch");
        std::copy(in, in + n, p);
    });
}

// fit_act_scales (calibrator.cpp:237-249) over caller samples (all share d_model).
// out: n_layers*4 + 1 scales (attn_in, attn_out, mlp_in, mlp_mid per layer; head_in last).
static void fit_into(void* h, int n_samples, const double* const* embeddings, const int* visual, const int* text,
                     int act_bits, const PruneHook& hook, double* out) {
    RefModel* m = static_cast<RefModel*>(h);
    std::vector<CalibSample> samples;
    for (int i = 0; i < n_samples; ++i) {
        CalibSample s;
        s.layout = SequenceLayout::prefix(visual[i], text[i]);
        s.embeddings = mat(embeddings[i], s.layout.total(), m->model.config.d_model);
        samples.push_back(std::move(s));
    }
    ActScales a = fit_act_scales(m->model, samples, act_bits, hook);
    size_t k = 0;
    for (const auto& l : a.layers) {
        out[k++] = l.attn_in.scales[0];
        out[k++] = l.attn_out.scales[0];
        out[k++] = l.mlp_in.scales[0];
        out[k++] = l.mlp_mid.scales[0];
    }
    out[k] = a.head_in.scales[0];
}

int qref_fit_act_scales(void* h, int n_samples, const double* const* embeddings, const int* visual,
                        const int* text, int act_bits, double* out) {
    return guard([&] { fit_into(h, n_samples, embeddings, visual, text, act_bits, PruneHook{}, out); });
}

// fit_act_scales under make_recipe_hook(recipe, weights4, nullopt): the prune_then_quant
// scale fit of run_pipeline (harness.cpp:103-106).
int qref_fit_act_scales_hooked(void* h, int n_samples, const double* const* embeddings, const int* visual,
                               const int* text, int act_bits, const char* recipe_json, const double* weights4,
                               double* out) {
    return guard([&] {
        PruningRecipe r = parse_recipe(recipe_json);
        MetricWeights w = weights4 ? MetricWeights{weights4[0], weights4[1], weights4[2], weights4[3]} : r.weights;
        fit_into(h, n_samples, embeddings, visual, text, act_bits, make_recipe_hook(r, w, std::nullopt), out);
    });
}

// make_calibration_samples (calibrator.cpp:12-29) + sample_set_digest (31-40).
// text_out[count]; emb_out (may be null): the samples' embeddings concatenated,
// cap doubles at most; digest17: 16 hex chars + NUL.
int qref_make_samples(uint64_t seed, int count, int v0, int d_model, int text_min, int text_max, int* text_out,
                      double* emb_out, int64_t cap, char* digest17) {
    return guard([&] {
        std::vector<CalibSample> ss = make_calibration_samples(seed, count, v0, d_model, text_min, text_max);
        int64_t o = 0;
        for (int i = 0; i < count; ++i) {
            text_out[i] = ss[i].layout.text_count;
            const auto& e = ss[i].embeddings.data;
            if (emb_out) {
                if (o + static_cast<int64_t>(e.size()) > cap) throw std::invalid_argument("buffer too small");
                std::copy(e.begin(), e.end(), emb_out + o);
            }
            o += static_cast<int64_t>(e.size());
        }
        std::string dg = sample_set_digest(ss);
        std::memcpy(digest17, dg.c_str(), 17);
    });
}

// pipeline_flops (gflops.cpp:24-51) of a recipe's executed lengths (recipe_json null: every
// layer at v0, the non-pruning modes, harness.cpp:167-176).  out3 = f_vlm, f_base, ratio_pct.
int qref_pipeline_flops(const char* recipe_json, int n_layers, int v0, int d_model, int d_ff, int n_heads,
                        int text_len, double f_vt, double f_pj, double* layer_costs, double* out3) {
    return guard([&] {
        CostModel cm;
        cm.f_vt = f_vt;
        cm.f_pj = f_pj;
        cm.d_model = d_model;
        cm.d_ff = d_ff;
        cm.n_heads = n_heads;
        cm.text_len = text_len;
        std::vector<int> v_hat = recipe_json ? executed_visual_lengths(parse_recipe(recipe_json), n_layers)
                                             : std::vector<int>(n_layers, v0);
        GflopsReport g = pipeline_flops(v_hat, v0, cm);
        for (size_t l = 0; l < g.layers.size(); ++l) layer_costs[l] = g.layers[l].cost;
        out3[0] = g.f_vlm;
        out3[1] = g.f_base;
        out3[2] = g.ratio_pct;
    });
}

// profile_sensitivity (calibrator.cpp:42-82) against the prepared QuantEnv:
// per listed layer the median over samples of ||x_q - x|| / (||x|| + eta) of the
// block outputs (raw) and normalize_sensitivities of them (calibrator.cpp:84-98).
int qref_profile_sensitivity(void* h, int n_samples, const double* const* embeddings, const int* visual,
                             const int* text, int n_layers, const int* layers, double eta, double* raw,
                             double* normalized) {
    return guard([&] {
        RefModel* m = static_cast<RefModel*>(h);
        if (!m->env) throw std::invalid_argument("quantized mode requires a QuantEnv");
        std::vector<CalibSample> samples;
        for (int i = 0; i < n_samples; ++i) {
            CalibSample s;
            s.layout = SequenceLayout::prefix(visual[i], text[i]);
            s.embeddings = mat(embeddings[i], s.layout.total(), m->model.config.d_model);
            samples.push_back(std::move(s));
        }
        SensitivityProfile p = profile_sensitivity(m->model, samples, std::span<const int>(layers, n_layers), eta,
                                                   m->env.get());
        std::copy(p.raw.begin(), p.raw.end(), raw);
        std::copy(p.normalized.begin(), p.normalized.end(), normalized);
    });
}

// QuantEnv with the reference's prepare_quant_env (model.cpp:212-237) when
// weight_axis == 1 (PerRow, the reference default), or the same construction
// with GroupAxis::PerColumn (quant.hpp:22) when weight_axis == 2 -- the
// per-output-channel variant north_star names.  forward_prefill only reads
// QuantizedWeight::deq (model.cpp:25-28), so either env runs the UNMODIFIED
// forward.
int qref_model_prepare_quant(void* h, int weight_bits, int act_bits, int kv_bits, int weight_axis,
                             const double* act_scales) {
    return guard([&] {
        RefModel* m = static_cast<RefModel*>(h);
        QuantConfig qc{weight_bits, act_bits, kv_bits};
        ActScales a;
        auto mk = [act_bits](double s) {
            QuantParams p;
            p.bits = act_bits;
            p.axis = GroupAxis::PerTensor;
            p.scales = {s};
            return p;
        };
        const int L = m->model.config.n_layers;
        for (int l = 0; l < L; ++l) {
            a.layers.push_back({mk(act_scales[4 * l + 0]), mk(act_scales[4 * l + 1]),
                                mk(act_scales[4 * l + 2]), mk(act_scales[4 * l + 3])});
        }
        a.head_in = mk(act_scales[4 * L]);
        if (weight_axis == 1) {
            m->env = std::make_unique<QuantEnv>(prepare_quant_env(m->model, qc, a));
            return;
        }
        if (weight_axis != 2) throw std::invalid_argument("weight_axis must be 1 (PerRow) or 2 (PerColumn)");
        auto env = std::make_unique<QuantEnv>();
        env->config = qc;
        env->act = a;
        env->layers.resize(static_cast<size_t>(L));
        auto pack = [&qc](const Matrix& w) {
            QuantizedWeight qw;
            qw.codes = quantize(w, fit_params(w, qc.weight_bits, GroupAxis::PerColumn));
            qw.deq = dequantize(qw.codes);
            return qw;
        };
        for (int l = 0; l < L; ++l) {
            const LayerWeights& src = m->model.layers[static_cast<size_t>(l)];
            env->layers[static_cast<size_t>(l)] = {pack(src.wq), pack(src.wk), pack(src.wv),
                                                   pack(src.wo), pack(src.w1), pack(src.w2)};
        }
        env->w_head = pack(m->model.w_head);
        m->env = std::move(env);
    });
}

// Quantized weight codes + scales of the current env (for GPU weight parity).
int qref_model_weight_codes(void* h, int layer, int which, int8_t* codes, double* scales) {
    return guard([&] {
        RefModel* m = static_cast<RefModel*>(h);
        if (!m->env) throw std::invalid_argument("no QuantEnv prepared");
        const QuantizedWeight* qw = nullptr;
        if (layer < 0) {
            qw = &m->env->w_head;
        } else {
            const QuantizedLayerWeights& l = m->env->layers.at(static_cast<size_t>(layer));
            const QuantizedWeight* ws[6] = {&l.wq, &l.wk, &l.wv, &l.wo, &l.w1, &l.w2};
            qw = ws[which];
        }
        std::memcpy(codes, qw->codes.codes.data(), qw->codes.codes.size());
        std::copy(qw->codes.params.scales.begin(), qw->codes.params.scales.end(), scales);
    });
}

// forward_prefill (model.cpp:315-453) with make_recipe_hook (selector.cpp:211-228).
// recipe_json may be null (no hook).  weights4 null = recipe.weights.
// res_bits < 0 = nullopt.  Returns a run handle or null (see qref_last_error).
void* qref_prefill(void* h, int quantized, const double* emb, int visual, int text, const int* pos,
                   const char* recipe_json, const double* weights4, int res_bits) {
    RefRun* run = nullptr;
    int rc = guard([&] {
        RefModel* m = static_cast<RefModel*>(h);
        SequenceLayout layout = SequenceLayout::prefix(visual, text);
        if (pos) layout.position_ids.assign(pos, pos + visual + text);
        ForwardOptions opts;
        if (quantized) {
            opts.mode = ExecMode::Quantized;
            opts.quant = m->env.get();
        }
        if (recipe_json) {
            PruningRecipe r = parse_recipe(recipe_json);
            MetricWeights w = weights4 ? MetricWeights{weights4[0], weights4[1], weights4[2], weights4[3]}
                                       : r.weights;
            std::optional<int> rb = res_bits < 0 ? std::nullopt : std::optional<int>(res_bits);
            opts.hook = make_recipe_hook(r, w, rb);
        }
        auto out = std::make_unique<RefRun>();
        out->owner = m;
        out->quantized = quantized != 0;
        out->result = forward_prefill(m->model, mat(emb, visual + text, m->model.config.d_model), layout, opts);
        run = out.release();
    });
    return rc == 0 ? run : nullptr;
}

void qref_run_free(void* r) { delete static_cast<RefRun*>(r); }

int qref_run_logits_rows(void* r) { return static_cast<RefRun*>(r)->result.logits.rows; }

int qref_run_logits(void* r, double* out) {
    return guard([&] {
        const Matrix& l = static_cast<RefRun*>(r)->result.logits;
        std::copy(l.data.begin(), l.data.end(), out);
    });
}

// final layout: counts + position ids (cap >= total)
int qref_run_layout(void* r, int* visual, int* text, int* pos, int cap) {
    return guard([&] {
        const SequenceLayout& l = static_cast<RefRun*>(r)->result.cache.layout;
        *visual = l.visual_count;
        *text = l.text_count;
        if (l.total() > cap) throw std::invalid_argument("buffer too small");
        std::copy(l.position_ids.begin(), l.position_ids.end(), pos);
    });
}

int qref_run_n_prunes(void* r) { return static_cast<int>(static_cast<RefRun*>(r)->result.prune_trace.size()); }

int qref_run_prune(void* r, int i, int* layer, int* budget, int* positions, int cap, int* count) {
    return guard([&] {
        const PruneEvent& e = static_cast<RefRun*>(r)->result.prune_trace.at(static_cast<size_t>(i));
        *layer = e.layer;
        *budget = e.budget;
        if (static_cast<int>(e.retained_positions.size()) > cap) throw std::invalid_argument("buffer too small");
        std::copy(e.retained_positions.begin(), e.retained_positions.end(), positions);
        *count = static_cast<int>(e.retained_positions.size());
    });
}

// block_outputs[layer] (model.cpp:439) -- rows x d_model
int qref_run_block_output(void* r, int layer, double* out, int* rows) {
    return guard([&] {
        const Matrix& b = static_cast<RefRun*>(r)->result.block_outputs.at(static_cast<size_t>(layer));
        *rows = b.rows;
        if (out) std::copy(b.data.begin(), b.data.end(), out);
    });
}

// Quantized KV rows of one (layer, head): codes [rows x d_head], scales [rows], positions [rows]
int qref_run_kv(void* r, int layer, int head, int which, int8_t* codes, double* scales, int* pos,
                int* rows) {
    return guard([&] {
        const KVCacheState& c = static_cast<RefRun*>(r)->result.cache;
        const LayerKV& lk = c.layers.at(static_cast<size_t>(layer));
        const HeadKV& hk = lk.heads.at(static_cast<size_t>(head));
        const QuantizedTensor& t = which == 0 ? hk.k_q : hk.v_q;
        *rows = t.rows;
        if (codes) std::memcpy(codes, t.codes.data(), t.codes.size());
        if (scales) std::copy(t.params.scales.begin(), t.params.scales.end(), scales);
        if (pos) std::copy(lk.position_ids.begin(), lk.position_ids.end(), pos);
    });
}

// decode_step (model.cpp:455-562): appends one token, logits [d_model]
int qref_decode(void* r, const double* emb, double* logits_out) {
    return guard([&] {
        RefRun* run = static_cast<RefRun*>(r);
        const QuantEnv* env = run->quantized ? run->owner->env.get() : nullptr;
        Vector out = decode_step(run->owner->model, env, run->result.cache,
                                 std::span<const double>(emb, static_cast<size_t>(run->owner->model.config.d_model)));
        std::copy(out.begin(), out.end(), logits_out);
    });
}

// CPU baseline driver: n_threads independent sequences (visual + text tokens,
// U(-1,1) embeddings from SplitMix64), one per std::thread, each through the
// reference forward_prefill in quantized mode (thread-safe per sequence,
// SPEC.md:224).  Returns wall seconds of the parallel region in *seconds.
int qref_prefill_threads(void* h, int n_threads, int visual, int text, uint64_t seed, double* seconds) {
    return guard([&] {
        RefModel* m = static_cast<RefModel*>(h);
        if (!m->env) throw std::invalid_argument("quantized mode requires a QuantEnv");
        const int d = m->model.config.d_model, S = visual + text;
        std::vector<Matrix> embs;
        for (int t = 0; t < n_threads; ++t) {
            SplitMix64 rng(mix_seed(seed, static_cast<uint64_t>(t)));
            Matrix e(S, d);
            for (double& v : e.data) v = rng.next_uniform(-1.0, 1.0);
            embs.push_back(std::move(e));
        }
        SequenceLayout layout = SequenceLayout::prefix(visual, text);
        std::vector<std::string> errs(static_cast<size_t>(n_threads));
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < n_threads; ++t) {
            pool.emplace_back([&, t] {
                try {
                    ForwardOptions o;
                    o.mode = ExecMode::Quantized;
                    o.quant = m->env.get();
                    forward_prefill(m->model, embs[static_cast<size_t>(t)], layout, o);
                } catch (const std::exception& e) {
                    errs[static_cast<size_t>(t)] = e.what();
                }
            });
        }
        for (auto& th : pool) th.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
    });
}

// FNV-1a digest of a double array (digest.hpp:12-42), for determinism checks.
uint64_t qref_fnv1a64(const double* v, int64_t n) {
    return fnv1a64(std::span<const double>(v, static_cast<size_t>(n)));
}

// run_quota_calibration (calibrator.cpp:251-268) on explicit samples with the
// per-output-channel QuantEnv (the axis the B200 GEMM uses):
// fit_act_scales -> env -> profile_diagnostics -> select_candidate_layers ->
// profile_sensitivity -> make_budget_schedule, all reference functions.
int qref_run_calibration(void* h, int n_samples, const double* const* embeddings, const int* visual, const int* text,
                         int window, double p_min, double tau, double eta, double* act_scales, int* layers,
                         double* keeps, double* raw, double* normalized, double* conc_median, double* red_median) {
    return guard([&] {
        RefModel* m = static_cast<RefModel*>(h);
        std::vector<CalibSample> samples;
        for (int i = 0; i < n_samples; ++i) {
            CalibSample s;
            s.layout = SequenceLayout::prefix(visual[i], text[i]);
            s.embeddings = mat(embeddings[i], s.layout.total(), m->model.config.d_model);
            samples.push_back(std::move(s));
        }
        const int L = m->model.config.n_layers;
        ActScales a = fit_act_scales(m->model, samples, 4);
        size_t k = 0;
        for (const auto& l : a.layers) {
            act_scales[k++] = l.attn_in.scales[0];
            act_scales[k++] = l.attn_out.scales[0];
            act_scales[k++] = l.mlp_in.scales[0];
            act_scales[k++] = l.mlp_mid.scales[0];
        }
        act_scales[k] = a.head_in.scales[0];
        if (qref_model_prepare_quant(h, 4, 4, 4, 2, act_scales) != 0) throw std::runtime_error(g_err);
        LayerDiagnostics diag = profile_diagnostics(m->model, samples, m->env.get());
        std::vector<int> cand = select_candidate_layers(diag, window);
        SensitivityProfile prof = profile_sensitivity(m->model, samples, cand, eta, m->env.get());
        BudgetSchedule sched = make_budget_schedule(prof, tau, p_min);
        std::copy(cand.begin(), cand.end(), layers);
        std::copy(sched.keep_ratios.begin(), sched.keep_ratios.end(), keeps);
        std::copy(prof.raw.begin(), prof.raw.end(), raw);
        std::copy(prof.normalized.begin(), prof.normalized.end(), normalized);
        for (int l = 0; l < L; ++l) {
            conc_median[l] = diag.concentration_median[l];
            red_median[l] = diag.redundancy_median[l];
        }
    });
}

}  // extern "C"
