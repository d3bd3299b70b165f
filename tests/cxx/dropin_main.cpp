// dropin_main.cpp -- a client of the UNMODIFIED reference C++ API
// (proj/include/quota), written the way the reference harness uses it
// (harness.cpp:132-145): init_model, act scales fitted by full-precision
// forwards (ActStats, calibrator.cpp:237-249), a per-output-channel QuantEnv,
// parse_recipe + make_recipe_hook, quantized forward_prefill, then
// teacher-forced decode_step.  Built once; run against the reference library
// alone (CPU) and with libquota_b200_cxx.so preloaded (B200), and the two
// outputs are compared by tests/test_dropin_gpu.py.
//
// usage: dropin_main <out.txt> [n_decode]
#include <cstdio>
#include <optional>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "quota/model.hpp"
#include "quota/recipe.hpp"
#include "quota/rng.hpp"
#include "quota/selector.hpp"

using namespace quota;

static Matrix embeddings(int rows, int d, uint64_t seed) {
    SplitMix64 rng(seed);
    Matrix m(rows, d);
    for (double& v : m.data) v = rng.next_uniform(-1.0, 1.0);
    return m;
}

// per-output-channel env from the reference's own quantizer primitives
static QuantEnv per_channel_env(const Model& model, const ActScales& act) {
    QuantEnv env;
    env.act = act;
    auto pack = [](const Matrix& w) {
        QuantizedWeight q;
        q.codes = quantize(w, fit_params(w, 4, GroupAxis::PerColumn));
        q.deq = dequantize(q.codes);
        return q;
    };
    for (const auto& l : model.layers)
        env.layers.push_back({pack(l.wq), pack(l.wk), pack(l.wv), pack(l.wo), pack(l.w1), pack(l.w2)});
    env.w_head = pack(model.w_head);
    return env;
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const int n_decode = argc > 2 ? std::atoi(argv[2]) : 8;
    ModelConfig cfg;
    cfg.n_layers = 4;
    cfg.n_heads = 4;
    cfg.d_model = 256;
    cfg.d_head = 64;
    cfg.seed = 11;
    Model model = init_model(cfg);
    const int V = 144, T = 40;
    // static activation scales from full-precision forwards (calibrator.cpp:237-249)
    ActStats stats;
    for (int i = 0; i < 3; ++i) {
        ForwardOptions o;
        o.act_stats = &stats;
        SequenceLayout cl = SequenceLayout::prefix(V, 16 + 8 * i);
        forward_prefill(model, embeddings(cl.total(), cfg.d_model, 100 + i), cl, o);
    }
    QuantEnv env = per_channel_env(model, stats.to_scales(4));
    PruningRecipe recipe = parse_recipe(
        "{\"schema_version\": 1, \"candidate_layers\": [1, 2], \"keep_ratios\": [0.5, 0.3], "
        "\"metric_weights\": {\"mag\": 0.25, \"inter\": 0.45, \"intra\": 0.1, \"quant\": 0.2}, "
        "\"v0\": 144, \"quant_digest\": \"w4a4kv4-sym-rne\"}");
    ForwardOptions opts;
    opts.mode = ExecMode::Quantized;
    opts.quant = &env;
    opts.hook = make_recipe_hook(recipe, recipe.weights, 4);
    SequenceLayout layout = SequenceLayout::prefix(V, T);
    ForwardResult res = forward_prefill(model, embeddings(V + T, cfg.d_model, 7), layout, opts);

    FILE* f = std::fopen(argv[1], "w");
    std::fprintf(f, "layout %d %d next %d\n", res.final_layout.visual_count, res.final_layout.text_count,
                 res.cache.next_position);
    for (const auto& e : res.prune_trace) {
        std::fprintf(f, "prune %d %d", e.layer, e.budget);
        for (int p : e.retained_positions) std::fprintf(f, " %d", p);
        std::fprintf(f, "\n");
    }
    for (size_t l = 0; l < res.cache.layers.size(); ++l) {
        const auto& lk = res.cache.layers[l];
        long long sum = 0;
        for (const auto& h : lk.heads)
            for (int8_t c : h.k_q.codes) sum += c;
        std::fprintf(f, "kv %zu rows %zu ksum %lld\n", l, lk.position_ids.size(), sum);
    }
    std::fprintf(f, "logits %d %d", res.logits.rows, res.logits.cols);
    for (double v : res.logits.data) std::fprintf(f, " %.9g", v);
    std::fprintf(f, "\n");
    // ForwardResult::records / block_outputs (model.cpp:382-402,439)
    std::fprintf(f, "records %zu blocks %zu\n", res.records.size(), res.block_outputs.size());
    for (const auto& r : res.records) {
        double inter = 0, intra = 0, vs = 0, ts = 0;
        for (const auto& m : r.attn_inter)
            for (double v : m.data) inter += v;
        for (const auto& m : r.attn_intra)
            for (double v : m.data) intra += v;
        for (double v : r.visual_states.data) vs += v * v;
        for (double v : r.text_states.data) ts += v * v;
        std::fprintf(f, "rec %d %d %d %zu %.9g %.9g %.9g %.9g\n", r.layer, r.visual_states.rows, r.text_states.rows,
                     r.attn_inter.size(), inter, intra, vs, ts);
    }
    for (size_t l = 0; l < res.block_outputs.size(); ++l) {
        double ss = 0;
        for (double v : res.block_outputs[l].data) ss += v * v;
        std::fprintf(f, "block %zu %d %.9g\n", l, res.block_outputs[l].rows, ss);
    }
    KVCacheState cache = std::move(res.cache);
    for (int s = 0; s < n_decode; ++s) {
        Matrix e = embeddings(1, cfg.d_model, 900 + s);
        Vector out = decode_step(model, &env, cache, e.row(0));
        std::fprintf(f, "decode %d", s);
        for (double v : out) std::fprintf(f, " %.9g", v);
        std::fprintf(f, "\n");
    }
    std::fprintf(f, "final %d %d next %d\n", cache.layout.visual_count, cache.layout.text_count, cache.next_position);
    // an arbitrary (non-recipe) PruneHook: keep the even visual slots at layer 1 and the
    // first ceil(V/3) at layer 3 -- it runs on the host per layer over the record
    {
        ForwardOptions o3 = opts;
        o3.hook = [](const LayerActivationRecord& rec, const SequenceLayout& cur) -> std::optional<RetainedSet> {
            if (rec.layer != 1 && rec.layer != 3) return std::nullopt;
            RetainedSet rs;
            if (rec.layer == 1)
                for (int i = 0; i < cur.visual_count; i += 2) rs.slots.push_back(i);
            else
                for (int i = 0; i < (cur.visual_count + 2) / 3; ++i) rs.slots.push_back(i);
            rs.budget = static_cast<int>(rs.slots.size());
            return rs;
        };
        ForwardResult hr = forward_prefill(model, embeddings(V + T, cfg.d_model, 8), layout, o3);
        for (const auto& e : hr.prune_trace) {
            std::fprintf(f, "hookprune %d %d", e.layer, e.budget);
            for (int p : e.retained_positions) std::fprintf(f, " %d", p);
            std::fprintf(f, "\n");
        }
        std::fprintf(f, "hooklogits %d %d", hr.logits.rows, hr.logits.cols);
        for (double v : hr.logits.data) std::fprintf(f, " %.9g", v);
        std::fprintf(f, "\n");
        // a hook returning an invalid set fails with the reference's exception and message
        ForwardOptions o4 = opts;
        o4.hook = [](const LayerActivationRecord&, const SequenceLayout&) -> std::optional<RetainedSet> {
            RetainedSet rs;
            rs.slots = {3, 1};
            return rs;
        };
        try {
            forward_prefill(model, embeddings(V + T, cfg.d_model, 8), layout, o4);
            std::fprintf(f, "badhook ok\n");
        } catch (const std::runtime_error& e) {
            std::fprintf(f, "badhook runtime_error %s\n", e.what());
        }
    }
    // the stock prepare_quant_env (what harness.cpp:113 / calibrator.cpp:260 call): the device
    // library serves it per output channel, which must equal per_channel_env bit for bit
    {
        QuantEnv stock = prepare_quant_env(model, QuantConfig{}, env.act);
        bool same = stock.layers.size() == env.layers.size();
        for (size_t l = 0; same && l < env.layers.size(); ++l)
            same = stock.layers[l].w1.codes.codes == env.layers[l].w1.codes.codes &&
                   stock.layers[l].w1.codes.params.scales == env.layers[l].w1.codes.params.scales;
        std::fprintf(f, "stockenv axis %d same %d\n", static_cast<int>(stock.layers[0].wq.codes.params.axis),
                     same ? 1 : 0);
    }
    // error behaviour: a hand-built per-input-channel env is rejected on the device path
    try {
        QuantEnv row_env = per_channel_env(model, env.act);
        for (auto& l : row_env.layers) l.wq.codes = quantize(model.layers[0].wq, fit_params(model.layers[0].wq, 4, GroupAxis::PerRow));
        ForwardOptions o2 = opts;
        o2.quant = &row_env;
        forward_prefill(model, embeddings(V + T, cfg.d_model, 7), layout, o2);
        std::fprintf(f, "perrow ok\n");
    } catch (const std::invalid_argument&) {
        std::fprintf(f, "perrow invalid_argument\n");
    }
    std::fclose(f);
    return 0;
}
