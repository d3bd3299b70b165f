"""The six integration orders of run_pipeline (harness.cpp:59-179) on the
B200 -- fp64 device forwards for the full-precision graphs, the W4A4 path for the
quantized ones, device calibration for the scales and the inline recipe -- against the
same orchestration over the unmodified reference library (oracle/harness_ref.py) on
identical weights, samples and recipe.  Bit-exact: traces, final visual counts, cost
reports, digests of the eval set; within tolerance: the divergence (fp64 vs fp64 for the
full-precision modes, the device's fp32 logits for the quantized ones)."""
import numpy as np
import pytest

import oracle as O
from oracle.harness_ref import ref_run_pipeline
import paper_2604_17320_b200 as Q
from paper_2604_17320_b200 import harness as H

pytestmark = pytest.mark.gpu

L, D, NH, V0 = 8, 256, 4, 64


@pytest.fixture(scope="module")
def setup(torch_cuda):
    cfg = O.ModelCfg(n_layers=L, d_model=D, n_heads=NH, n_kv_heads=NH, d_head=D // NH, d_ff=4 * D, weight_axis=2)
    ref = O.Ref(cfg, seed=7)
    w = O.synth_weights(cfg, seed=3)
    ref.set_weights(w)
    e = Q.Engine(Q.Config(n_layers=L, d_model=D, n_heads=NH, n_kv_heads=NH, d_head=D // NH, d_ff=4 * D),
                 max_batch=4, max_tokens=2048, max_seq=512, max_decode=4)
    e.keep_fp_weights(True)
    e.load_weights(w)
    hc = H.HarnessConfig(calib=H.CalibrationConfig(samples=4, v0=V0, window=3, text_min=8, text_max=16),
                         eval_samples=3)
    ev = H.make_eval_samples(hc, D)
    calib = H.make_calibration_samples(hc.calib.seed, hc.calib.samples, V0, D, 8, 16)
    return ref, e, hc, ev, calib


RECIPE = ([2, 4, 5], [0.6, 0.4, 0.3])


def _compare(dev, exp, quantized):
    assert dev.final_visual_count == exp["final_visual_count"]
    assert dev.traces == exp["traces"]
    costs, f_vlm, f_base, ratio = exp["gflops"]
    assert [x["cost"] for x in dev.gflops["layers"]] == list(costs)
    assert (dev.gflops["f_vlm"], dev.gflops["f_base"], dev.gflops["ratio_pct"]) == (f_vlm, f_base, ratio)
    err = [np.abs(a - b[-1]).max() for a, b in zip(dev.last_logits, exp["logits"])]
    gap = np.mean([np.linalg.norm(a - b[-1]) for a, b in zip(dev.last_logits, exp["logits"])])
    print(dev.mode, "divergence device", dev.divergence_mean, "reference", exp["divergence_mean"],
          "max |logit err|", max(err))
    # |div_dev - div_ref| <= mean ||lg_dev - lg_ref|| (triangle inequality): the divergence
    # agrees as far as the final logits do
    assert abs(dev.divergence_mean - exp["divergence_mean"]) <= gap + 1e-12
    if quantized:  # fp32 device logits: the path's logits tolerance, 1e-2 abs
        assert max(err) <= 1e-2
    else:  # fp64 on both sides; DGEMM summation order only
        assert max(err) <= 1e-9
        assert abs(dev.divergence_mean - exp["divergence_mean"]) <= 1e-9 * max(1.0, exp["divergence_mean"])


@pytest.mark.parametrize("mode", H.MODES)
def test_mode_matches_reference(setup, mode):
    ref, e, hc, ev, calib = setup
    prunes = H.mode_prunes(mode)
    rec_dev = H.PruningRecipe(RECIPE[0], RECIPE[1], H.MetricWeights(), V0, H.quant_digest()) if prunes else None
    rec_ref = O.Recipe(RECIPE[0], RECIPE[1], v0=V0) if prunes else None
    dev = H.run_pipeline(e, hc, mode, ev, recipe_override=rec_dev, calib_samples=calib)
    exp = ref_run_pipeline(ref, mode, [s.as_tuple() for s in ev], [s.as_tuple() for s in calib], rec_ref, v0=V0)
    _compare(dev, exp, H.mode_quantizes(mode))
    assert dev.eval_digest == H.sample_set_digest(ev) and dev.eval_count == 3
    if mode == "fp_baseline":
        assert dev.divergence_mean == 0.0 and dev.final_visual_count == V0
    if mode == "quant_only":
        assert dev.final_visual_count == V0 and dev.gflops["ratio_pct"] == 100.0
    if prunes:
        assert dev.final_visual_count == int(np.ceil(0.3 * V0))
        assert dev.recipe_digest == rec_dev.digest()


def test_collaborative_inline_recipe_matches_reference(setup):
    """No recipe override: the recipe is generated inline from the calibration samples
    (run_quota_calibration, harness.cpp:77-85) on the device, then evaluated."""
    ref, e, hc, ev, calib = setup
    dev = H.run_pipeline(e, hc, "collaborative", ev, calib_samples=calib)
    exp = ref_run_pipeline(ref, "collaborative", [s.as_tuple() for s in ev], [s.as_tuple() for s in calib], None,
                           v0=V0, window=3)
    assert dev.recipe.candidate_layers == list(exp["recipe"].candidate_layers)
    np.testing.assert_allclose(dev.recipe.keep_ratios, exp["recipe"].keep_ratios, rtol=1e-6)
    _compare(dev, exp, True)


def test_compare_reports_over_modes(setup):
    ref, e, hc, ev, calib = setup
    rec = H.PruningRecipe(RECIPE[0], RECIPE[1], H.MetricWeights(), V0, H.quant_digest())
    reps = [H.run_pipeline(e, hc, m, ev, recipe_override=rec if H.mode_prunes(m) else None, calib_samples=calib)
            for m in ("fp_baseline", "quant_only", "collaborative")]
    rows = H.compare_reports(reps)
    assert [r["mode"] for r in rows] == ["collaborative", "fp_baseline", "quant_only"]
    assert rows[1]["divergence_mean"] == 0.0
    assert rows[0]["gflops_ratio_pct"] < 100.0
    print(H.render_comparison_text(rows))


def test_fp_prefill_hook_errors(setup):
    ref, e, hc, ev, calib = setup
    e.clear_recipe()
    with pytest.raises(Q.QuotaInvalidArgument, match="no recipe set"):
        e.prefill_fp([ev[0].as_tuple()], hook=True)
    # a candidate layer reached with an empty visual prefix: robust_normalize's "empty sample"
    e.set_recipe([1], [0.5], (0.25, 0.45, 0.10, 0.20), V0, -1)
    emb = ev[0].embeddings[V0:]
    with pytest.raises(Q.QuotaInvalidArgument, match="empty sample"):
        e.prefill_fp([(emb, 0, emb.shape[0])], hook=True)
    # decode needs the quantized prefill's device cache
    e.prefill_fp([ev[0].as_tuple()], hook=False)
    with pytest.raises(Q.QuotaError):
        e.decode(np.zeros((1, D), np.float32))
