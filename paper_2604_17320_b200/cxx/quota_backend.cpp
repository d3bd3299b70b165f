// quota_backend.cpp -- the reference C++ API, served by the B200 engine.
//
// Drop-in for /root/reference/proj: compiled against the reference's OWN
// public headers (proj/include/quota/*.hpp, unmodified, on the include path),
// it defines the hot-path entry points with the reference's exact signatures
//
//   quota::forward_prefill   (model.hpp:174-175, model.cpp:315-453)
//   quota::decode_step       (model.hpp:179-180, model.cpp:455-562)
//   quota::make_recipe_hook  (selector.hpp:55-57, selector.cpp:211-228)
//
// and is linked (or LD_PRELOADed) ahead of the reference library, so every
// caller -- the reference harness (harness.cpp:134-142), calibrator, user code
// -- resolves to it.  Quantized-mode calls run on the device through the C ABI
// (include/quota_b200.h); there is no CPU path for them: without a GPU they
// throw.  Full-precision calls (calibration / baselines, not the deployed
// path) are forwarded to the next definition (the reference's) via
// dlsym(RTLD_NEXT).
//
// Semantics kept from the reference: validation order and exception types /
// messages, budget = ceil(r * v0) with the recipe's v0, pruning of the
// candidate layer's own KV rows, next_position = last original position + 1,
// decode appends one text token, ForwardResult::records and block_outputs
// filled for every layer, any PruneHook honoured.  Differences:
//   * weights are quantized per OUTPUT channel (GroupAxis::PerColumn): this
//     library also serves quota::prepare_quant_env (model.cpp:212-237) with that
//     axis, so stock callers (harness.cpp:113, calibrator.cpp:260) get an env the
//     device runs -- a per-input-channel scale cannot be applied after an int32
//     GEMM; a hand-built PerRow env is rejected;
//   * make_recipe_hook hooks run on the device (scoring, top-k and compaction
//     kernels); any other hook runs on the host once per layer on the
//     materialised record, its retained set applied on the device;
//   * record probabilities and KV scales come back from fp32 device values.
// Engines are cached per model / env CONTENT (a fingerprint of every weight
// code, scale, gain and activation scale), at most QUOTA_B200_MAX_ENGINES.
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <exception>
#include <list>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "quota/model.hpp"
#include "quota/quant.hpp"
#include "quota/recipe.hpp"
#include "quota/selector.hpp"
#include "quota_b200.h"
#include "quota_b200.hpp"

namespace {

using namespace quota;

void throw_status(int rc) {
    if (rc == QT_OK) return;
    std::string msg = qt_last_error();
    switch (rc) {
        case QT_EINVAL: throw std::invalid_argument(msg);
        case QT_ERANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

template <class F>
F next_symbol(const char* mangled) {
    void* p = dlsym(RTLD_NEXT, mangled);
    if (!p) throw std::runtime_error(std::string("quota_b200: reference symbol not found: ") + mangled);
    return reinterpret_cast<F>(p);
}

using PrefillFn = ForwardResult (*)(const Model&, const Matrix&, const SequenceLayout&, const ForwardOptions&);
using DecodeFn = Vector (*)(const Model&, const QuantEnv*, KVCacheState&, std::span<const double>);
using HookFn = PruneHook (*)(const PruningRecipe&, const MetricWeights&, std::optional<int>);

PrefillFn ref_prefill() {
    static PrefillFn f =
        next_symbol<PrefillFn>("_ZN5quota15forward_prefillERKNS_5ModelERKNS_6MatrixERKNS_14SequenceLayoutERKNS_14ForwardOptionsE");
    return f;
}
DecodeFn ref_decode() {
    static DecodeFn f = next_symbol<DecodeFn>(
        "_ZN5quota11decode_stepERKNS_5ModelEPKNS_8QuantEnvERNS_12KVCacheStateESt4spanIKdLm18446744073709551615EE");
    return f;
}
HookFn ref_hook() {
    static HookFn f =
        next_symbol<HookFn>("_ZN5quota16make_recipe_hookERKNS_13PruningRecipeERKNS_13MetricWeightsESt8optionalIiE");
    return f;
}

// The functor make_recipe_hook returns: recognisable through
// std::function::target<RecipeHook>(), and still a working reference hook
// when the full-precision forward calls it on the host.
struct RecipeHook {
    PruningRecipe recipe;
    MetricWeights weights;
    std::optional<int> res_bits;
    PruneHook host;  // the reference's own hook for the same arguments
    std::optional<RetainedSet> operator()(const LayerActivationRecord& r, const SequenceLayout& l) const {
        return host(r, l);
    }
};

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

// One device engine per (Model, QuantEnv) content; one live prefill session per
// engine (a new prefill invalidates the caches of earlier ones).
struct Device {
    qt_engine* e = nullptr;
    uint64_t fingerprint = 0;
    int max_tokens = 0, max_decode = 0;
    long long session = 0;  // id of the prefill whose KV the engine holds
    int steps = 0;
    ~Device() {
        if (e) qt_engine_destroy(e);
    }
};

struct SessionRef {
    Device* dev;
    long long session;
};

std::mutex g_mu;
std::list<std::unique_ptr<Device>> g_devices;  // most recently used first
std::map<const int*, SessionRef> g_sessions;  // keyed by cache.layout.position_ids.data()
long long g_next_session = 1;

void check_env(const Model& model, const QuantEnv& env) {
    const ModelConfig& c = model.config;
    if (env.layers.size() != static_cast<size_t>(c.n_layers))
        throw std::invalid_argument("activation scales do not cover all layers");
    if (env.act.layers.size() != static_cast<size_t>(c.n_layers))
        throw std::invalid_argument("activation scales do not cover all layers");
    if (env.config.weight_bits != 4 || env.config.act_bits != 4 || env.config.kv_bits != 4)
        throw std::invalid_argument("quota_b200: the device path implements W4A4KV4 only");
    auto chk = [&](const QuantizedWeight& w) {
        if (w.codes.params.axis != GroupAxis::PerColumn)
            throw std::invalid_argument(
                "quota_b200: weights must be quantized per output channel (GroupAxis::PerColumn), as this "
                "library's quota::prepare_quant_env does");
        if (w.codes.params.bits != 4) throw std::invalid_argument("quota_b200: weights must be 4-bit");
    };
    for (const auto& l : env.layers) {
        chk(l.wq); chk(l.wk); chk(l.wv); chk(l.wo); chk(l.w1); chk(l.w2);
    }
    chk(env.w_head);
}

// 64-bit content hash, 8 bytes per step (FNV-1a style multiply on words)
struct Fingerprint {
    uint64_t h = 0xcbf29ce484222325ULL;
    void bytes(const void* p, size_t n) {
        const unsigned char* c = static_cast<const unsigned char*>(p);
        size_t i = 0;
        for (; i + 8 <= n; i += 8) {
            uint64_t w;
            std::memcpy(&w, c + i, 8);
            h = (h ^ w) * 0x100000001b3ULL;
            h ^= h >> 29;
        }
        for (; i < n; ++i) h = (h ^ c[i]) * 0x100000001b3ULL;
        h ^= n;
    }
    template <class T>
    void vec(const std::vector<T>& v) { bytes(v.data(), v.size() * sizeof(T)); }
};

uint64_t fingerprint(const Model& model, const QuantEnv& env) {
    Fingerprint f;
    const ModelConfig& c = model.config;
    const int cfg[4] = {c.n_layers, c.d_model, c.n_heads, c.d_head};
    f.bytes(cfg, sizeof(cfg));
    const int qc[3] = {env.config.weight_bits, env.config.act_bits, env.config.kv_bits};
    f.bytes(qc, sizeof(qc));
    auto w = [&f](const QuantizedWeight& q) {
        f.vec(q.codes.codes);
        f.vec(q.codes.params.scales);
    };
    for (size_t l = 0; l < env.layers.size(); ++l) {
        const auto& q = env.layers[l];
        w(q.wq); w(q.wk); w(q.wv); w(q.wo); w(q.w1); w(q.w2);
    }
    w(env.w_head);
    for (const auto& lw : model.layers) {
        f.vec(lw.norm1_gain);
        f.vec(lw.norm2_gain);
    }
    f.vec(model.final_norm_gain);
    for (const auto& s : env.act.layers)
        for (const QuantParams* p : {&s.attn_in, &s.attn_out, &s.mlp_in, &s.mlp_mid}) f.vec(p->scales);
    f.vec(env.act.head_in.scales);
    return f.h;
}

void drop_sessions(const Device* dev) {
    for (auto it = g_sessions.begin(); it != g_sessions.end();)
        it = it->second.dev == dev ? g_sessions.erase(it) : std::next(it);
}

Device* device_for(const Model& model, const QuantEnv& env, int tokens) {
    check_env(model, env);
    const uint64_t fp = fingerprint(model, env);
    const int max_decode = env_int("QUOTA_B200_MAX_DECODE", 512);
    std::unique_ptr<Device>* slotp = nullptr;
    for (auto it = g_devices.begin(); it != g_devices.end(); ++it)
        if ((*it)->fingerprint == fp) {
            g_devices.splice(g_devices.begin(), g_devices, it);  // most recently used first
            slotp = &g_devices.front();
            break;
        }
    if (slotp && (*slotp)->max_tokens >= tokens && (*slotp)->max_decode >= max_decode) return slotp->get();
    if (!slotp) {
        g_devices.emplace_front();
        slotp = &g_devices.front();
        const size_t cap = (size_t)std::max(1, env_int("QUOTA_B200_MAX_ENGINES", 2));
        while (g_devices.size() > cap) {  // evict the least recently used engine (and its sessions)
            drop_sessions(g_devices.back().get());
            g_devices.pop_back();
        }
    }
    auto& slot = *slotp;
    const ModelConfig& c = model.config;
    auto dev = std::make_unique<Device>();
    dev->fingerprint = fp;
    qt_config qc{};
    qc.n_layers = c.n_layers;
    qc.d_model = c.d_model;
    qc.n_heads = c.n_heads;
    qc.n_kv_heads = c.n_heads;
    qc.d_head = c.d_head;
    qc.d_ff = c.d_ff();
    qc.mlp = 0;       // reference SiLU MLP
    qc.act_mode = 0;  // static per-tensor site scales (model.cpp:31-33)
    qc.weight_bits = qc.act_bits = qc.kv_bits = 4;
    const int cap = std::max(tokens, env_int("QUOTA_B200_MAX_TOKENS", 0));
    throw_status(qt_engine_create(&qc, 1, cap, cap, max_decode, &dev->e));
    dev->max_tokens = cap;
    dev->max_decode = max_decode;
    for (int l = 0; l < c.n_layers; ++l) {
        const QuantizedLayerWeights& q = env.layers[l];
        const int8_t* codes[7] = {q.wq.codes.codes.data(), q.wk.codes.codes.data(), q.wv.codes.codes.data(),
                                  q.wo.codes.codes.data(), q.w1.codes.codes.data(), q.w2.codes.codes.data(), nullptr};
        const double* scales[7] = {q.wq.codes.params.scales.data(), q.wk.codes.params.scales.data(),
                                   q.wv.codes.params.scales.data(), q.wo.codes.params.scales.data(),
                                   q.w1.codes.params.scales.data(), q.w2.codes.params.scales.data(), nullptr};
        throw_status(qt_engine_load_layer_codes(dev->e, l, codes, scales, model.layers[l].norm1_gain.data(),
                                                model.layers[l].norm2_gain.data()));
    }
    throw_status(qt_engine_load_head_codes(dev->e, env.w_head.codes.codes.data(), env.w_head.codes.params.scales.data(),
                                           model.final_norm_gain.data()));
    std::vector<double> act;
    for (const auto& s : env.act.layers)
        for (const QuantParams* p : {&s.attn_in, &s.attn_out, &s.mlp_in, &s.mlp_mid}) {
            if (p->scales.size() != 1) throw std::invalid_argument("quota_b200: activation scales must be per-tensor");
            act.push_back(p->scales[0]);
        }
    if (env.act.head_in.scales.size() != 1) throw std::invalid_argument("quota_b200: activation scales must be per-tensor");
    act.push_back(env.act.head_in.scales[0]);
    throw_status(qt_engine_set_act_scales(dev->e, act.data()));
    if (slot) drop_sessions(slot.get());  // the engine being replaced (grown capacity)
    slot = std::move(dev);
    return slot.get();
}

// host KV materialisation of one layer (KVCacheState::layers[l], model.hpp:96-112)
void read_layer_kv(Device* dev, const Model& model, int l, LayerKV& lk) {
    const int H = model.config.n_heads, dh = model.config.d_head;
    lk.heads.assign(H, HeadKV{});
    for (int h = 0; h < H; ++h)
        for (int which = 0; which < 2; ++which) {
            int rows = 0;
            throw_status(qt_engine_kv(dev->e, l, 0, h, which, nullptr, nullptr, &rows, 0));
            QuantizedTensor t;
            t.rows = rows;
            t.cols = dh;
            t.codes.resize(static_cast<size_t>(rows) * dh);
            std::vector<float> sc(rows);
            throw_status(qt_engine_kv(dev->e, l, 0, h, which, t.codes.data(), sc.data(), &rows, rows));
            t.params.bits = 4;
            t.params.axis = GroupAxis::PerRow;
            t.params.scales.assign(sc.begin(), sc.end());
            (which ? lk.heads[h].v_q : lk.heads[h].k_q) = std::move(t);
        }
}

// An arbitrary PruneHook, called by the engine once per layer on the materialised record
// (model.cpp:404-405); the retained set is validated as forward_prefill / apply_pruning
// do (model.cpp:408-416, selector.cpp:140-148, same messages) before the device applies it.
struct HostHook {
    const PruneHook* hook;
    std::exception_ptr err;
};

LayerActivationRecord to_record(const qt_layer_record& r) {
    LayerActivationRecord rec;
    rec.layer = r.layer;
    const int V = r.visual, T = r.text, S = V + T, d = r.d_model;
    rec.visual_states = Matrix(V, d);
    std::copy(r.visual_states, r.visual_states + (size_t)V * d, rec.visual_states.data.begin());
    rec.text_states = Matrix(T, d);
    std::copy(r.text_states, r.text_states + (size_t)T * d, rec.text_states.data.begin());
    for (int h = 0; h < r.n_heads; ++h) {
        const float* p = r.probs + (size_t)h * S * V;
        Matrix inter(T, V), intra(V, V);
        for (int q = 0; q < V; ++q)
            for (int k = 0; k < V; ++k) intra.at(q, k) = p[(size_t)q * V + k];
        for (int q = 0; q < T; ++q)
            for (int k = 0; k < V; ++k) inter.at(q, k) = p[(size_t)(V + q) * V + k];
        rec.attn_inter.push_back(std::move(inter));
        rec.attn_intra.push_back(std::move(intra));
    }
    return rec;
}

SequenceLayout layout_of(int V, int T, const int* pos) {
    SequenceLayout l;
    l.visual_count = V;
    l.text_count = T;
    l.position_ids.assign(pos, pos + V + T);
    l.modality.assign(V, Modality::Visual);
    l.modality.insert(l.modality.end(), T, Modality::Text);
    return l;
}

int host_hook_tramp(void* user, const qt_layer_record* r, int* slots, int* n_slots, int* budget) {
    HostHook* hh = static_cast<HostHook*>(user);
    try {
        const LayerActivationRecord rec = to_record(*r);
        const SequenceLayout cur = layout_of(r->visual, r->text, r->positions);
        std::optional<RetainedSet> rs = (*hh->hook)(rec, cur);
        if (!rs) return 0;
        const int V = r->visual;
        if (static_cast<int>(rs->slots.size()) < V)
            for (int s : rs->slots)
                if (s < 0 || s >= V) throw std::runtime_error("pruning text or out-of-range token");
        if (rs->slots.empty()) throw std::runtime_error("pruning would remove every visual token");
        int prev = -1;
        for (int s : rs->slots) {
            if (s <= prev) throw std::runtime_error("retained slots must be ascending and unique");
            if (s < 0 || s >= V) throw std::runtime_error("pruning text or out-of-range token");
            prev = s;
        }
        std::copy(rs->slots.begin(), rs->slots.end(), slots);
        *n_slots = static_cast<int>(rs->slots.size());
        *budget = rs->budget;
        return 1;
    } catch (...) {
        hh->err = std::current_exception();
        return -1;
    }
}

}  // namespace

namespace quota {

// prepare_quant_env (model.cpp:212-237) with per-OUTPUT-channel weights: the axis the
// device's int32-accumulator GEMMs can scale; same validation.
QuantEnv prepare_quant_env(const Model& model, const QuantConfig& config, const ActScales& act) {
    return quota_b200::prepare_quant_env_per_channel(model, config, act);
}

PruneHook make_recipe_hook(const PruningRecipe& recipe, const MetricWeights& weights, std::optional<int> res_bits) {
    PruneHook host = ref_hook()(recipe, weights, res_bits);  // validates like selector.cpp:213
    return RecipeHook{recipe, weights, res_bits, std::move(host)};
}

ForwardResult forward_prefill(const Model& model, const Matrix& embeddings, const SequenceLayout& layout,
                              const ForwardOptions& options) {
    if (options.mode != ExecMode::Quantized || options.act_stats) return ref_prefill()(model, embeddings, layout, options);
    // validation in the reference's order (model.cpp:317-325)
    model.config.validate();
    layout.validate();
    if (embeddings.rows != layout.total() || embeddings.cols != model.config.d_model)
        throw std::invalid_argument("embedding shape does not match layout");
    if (options.quant == nullptr) throw std::invalid_argument("quantized mode requires a QuantEnv");
    const RecipeHook* rh = options.hook ? options.hook.target<RecipeHook>() : nullptr;
    HostHook hh{options.hook ? &options.hook : nullptr, nullptr};
    const QuantEnv& env = *options.quant;
    const int L = model.config.n_layers, d = model.config.d_model;

    std::lock_guard<std::mutex> lock(g_mu);
    Device* dev = device_for(model, env, layout.total());
    if (rh) {
        const PruningRecipe& r = rh->recipe;
        const double w4[4] = {rh->weights.mag, rh->weights.inter, rh->weights.intra, rh->weights.quant};
        const int n = static_cast<int>(r.candidate_layers.size());
        throw_status(qt_engine_set_recipe(dev->e, n, r.candidate_layers.data(), r.keep_ratios.data(), w4, r.v0,
                                          rh->res_bits ? *rh->res_bits : -1));
        throw_status(qt_engine_set_prune_hook(dev->e, nullptr, nullptr));
    } else {
        throw_status(qt_engine_set_recipe(dev->e, 0, nullptr, nullptr, nullptr, 1, 4));
        throw_status(qt_engine_set_prune_hook(dev->e, hh.hook ? host_hook_tramp : nullptr, &hh));
    }
    // ForwardResult::records / block_outputs, as the reference always fills them
    // (QUOTA_B200_RECORDS=0 skips both: a serving caller that never reads them)
    const bool records = env_int("QUOTA_B200_RECORDS", 1) != 0;
    throw_status(qt_engine_set_records(dev->e, records ? 3 : 0));
    const int vis = layout.visual_count, txt = layout.text_count;
    std::vector<float> logits(static_cast<size_t>(layout.total()) * d);
    const int prc = qt_engine_prefill_f64(dev->e, 1, embeddings.data.data(), 0, &vis, &txt, nullptr,
                                          layout.position_ids.data(), logits.data(), 0);
    qt_engine_set_prune_hook(dev->e, nullptr, nullptr);
    if (hh.err) std::rethrow_exception(hh.err);  // the hook's own exception, as the reference propagates it
    throw_status(prc);
    const int rows = qt_engine_prefill_rows(dev->e);

    ForwardResult res;
    res.logits = Matrix(rows, d);
    for (size_t i = 0; i < res.logits.data.size(); ++i) res.logits.data[i] = logits[i];
    // final layout + prune trace (PruneEvent, model.cpp:408-418)
    int fv = 0, ft = 0;
    std::vector<int> pos(layout.total());
    throw_status(qt_engine_layout(dev->e, 0, &fv, &ft, pos.data(), static_cast<int>(pos.size())));
    SequenceLayout fl;
    fl.visual_count = fv;
    fl.text_count = ft;
    fl.position_ids.assign(pos.begin(), pos.begin() + fv + ft);
    fl.modality.assign(fv, Modality::Visual);
    fl.modality.insert(fl.modality.end(), ft, Modality::Text);
    const int np = qt_engine_n_prunes(dev->e, 0);
    std::vector<std::vector<int>> kept_after(L + 1);  // positions cached at layer l
    std::vector<int> cur = layout.position_ids;
    int cur_v = vis;
    int ev = 0;
    std::vector<PruneEvent> trace;
    for (int i = 0; i < np; ++i) {
        PruneEvent e;
        int cnt = 0;
        std::vector<int> buf(layout.total());
        throw_status(qt_engine_prune(dev->e, 0, i, &e.layer, &e.budget, buf.data(), static_cast<int>(buf.size()), &cnt));
        e.retained_positions.assign(buf.begin(), buf.begin() + cnt);
        trace.push_back(std::move(e));
    }
    res.prune_trace = trace;
    res.final_layout = fl;
    if (records) {
        const int nr = qt_engine_record_count(dev->e);
        for (int i = 0; i < nr; ++i) {
            int meta[4];
            throw_status(qt_engine_record_get(dev->e, i, meta, nullptr, nullptr, nullptr));
            const int V = meta[1], T = meta[2], H = meta[3];
            std::vector<int> pos(V + T);
            std::vector<double> states((size_t)(V + T) * d);
            std::vector<float> probs((size_t)H * (V + T) * V);
            throw_status(qt_engine_record_get(dev->e, i, meta, pos.data(), states.data(), probs.data()));
            qt_layer_record r{meta[0], V, T, d, H, pos.data(), states.data(), states.data() + (size_t)V * d,
                              probs.data()};
            res.records.push_back(to_record(r));
        }
        for (int l = 0; l < L; ++l) {
            int br = 0;
            throw_status(qt_engine_block_output(dev->e, l, nullptr, 0, &br));
            Matrix b(br, d);
            throw_status(qt_engine_block_output(dev->e, l, b.data.data(), (long long)b.data.size(), &br));
            res.block_outputs.push_back(std::move(b));
        }
    }
    // KV cache state (model.cpp:447-451); layer l caches the token set entering it,
    // filtered by a prune at l itself (selector.cpp:168-206)
    res.cache.mode = ExecMode::Quantized;
    res.cache.kv_bits = env.config.kv_bits;
    res.cache.layers.resize(L);
    for (int l = 0; l < L; ++l) {
        while (ev < np && trace[ev].layer == l) {
            std::vector<int> nxt(trace[ev].retained_positions);
            nxt.insert(nxt.end(), cur.begin() + cur_v, cur.end());
            cur_v = static_cast<int>(trace[ev].retained_positions.size());
            cur = std::move(nxt);
            ++ev;
        }
        res.cache.layers[l].position_ids = cur;
    }
    const bool host_kv = env_int("QUOTA_B200_HOST_KV", 1) != 0;
    if (host_kv)
        for (int l = 0; l < L; ++l) read_layer_kv(dev, model, l, res.cache.layers[l]);
    res.cache.layout = fl;
    res.cache.next_position = layout.position_ids.back() + 1;
    // bind the returned cache to the device session
    dev->session = g_next_session++;
    dev->steps = 0;
    for (auto it = g_sessions.begin(); it != g_sessions.end();)
        it = it->second.dev == dev ? g_sessions.erase(it) : std::next(it);
    g_sessions[res.cache.layout.position_ids.data()] = SessionRef{dev, dev->session};
    return res;
}

Vector decode_step(const Model& model, const QuantEnv* quant, KVCacheState& cache, std::span<const double> embedding) {
    const bool quantized = cache.mode == ExecMode::Quantized;
    if (quantized != (quant != nullptr)) throw std::runtime_error("cache and execution mode mismatch");
    if (!quantized) return ref_decode()(model, quant, cache, embedding);
    if (cache.layers.size() != static_cast<size_t>(model.config.n_layers))
        throw std::invalid_argument("cache does not match model depth");
    if (embedding.size() != static_cast<size_t>(model.config.d_model))
        throw std::invalid_argument("embedding width mismatch");
    std::lock_guard<std::mutex> lock(g_mu);
    auto it = g_sessions.find(cache.layout.position_ids.data());
    if (it == g_sessions.end() || it->second.dev->session != it->second.session)
        throw std::runtime_error("quota_b200: cache is not bound to a live device session "
                                 "(copied, or superseded by a later forward_prefill)");
    Device* dev = it->second.dev;
    const int d = model.config.d_model;
    std::vector<float> out(d);
    throw_status(qt_engine_decode_f64(dev->e, embedding.data(), 0, out.data(), 0));
    ++dev->steps;
    const SessionRef ref = it->second;
    g_sessions.erase(it);
    const int pos = cache.next_position;
    cache.layout.text_count += 1;  // model.cpp:553-556
    cache.layout.position_ids.push_back(pos);
    cache.layout.modality.push_back(Modality::Text);
    cache.next_position += 1;
    for (int l = 0; l < model.config.n_layers; ++l) {
        cache.layers[l].position_ids.push_back(pos);  // model.cpp:537
        if (!cache.layers[l].heads.empty()) read_layer_kv(dev, model, l, cache.layers[l]);
    }
    g_sessions[cache.layout.position_ids.data()] = ref;
    return Vector(out.begin(), out.end());
}

}  // namespace quota

namespace quota_b200 {

quota::QuantEnv prepare_quant_env_per_channel(const quota::Model& model, const quota::QuantConfig& config,
                                              const quota::ActScales& act) {
    using namespace quota;
    // prepare_quant_env (model.cpp:212-237) with GroupAxis::PerColumn weights
    if (act.layers.size() != static_cast<size_t>(model.config.n_layers))
        throw std::invalid_argument("activation scales do not cover all layers");
    QuantEnv env;
    env.config = config;
    env.act = act;
    env.layers.resize(model.layers.size());
    auto pack = [&config](const Matrix& w) {
        QuantizedWeight qw;
        qw.codes = quantize(w, fit_params(w, config.weight_bits, GroupAxis::PerColumn));
        qw.deq = dequantize(qw.codes);
        return qw;
    };
    for (size_t l = 0; l < model.layers.size(); ++l) {
        const auto& src = model.layers[l];
        env.layers[l].wq = pack(src.wq);
        env.layers[l].wk = pack(src.wk);
        env.layers[l].wv = pack(src.wv);
        env.layers[l].wo = pack(src.wo);
        env.layers[l].w1 = pack(src.w1);
        env.layers[l].w2 = pack(src.w2);
    }
    env.w_head = pack(model.w_head);
    return env;
}

void release_device_sessions() {
    std::lock_guard<std::mutex> lock(g_mu);
    g_sessions.clear();
    g_devices.clear();
}

}  // namespace quota_b200
