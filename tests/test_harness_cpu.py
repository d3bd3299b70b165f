"""CPU tests of the harness host logic: the pieces of
run_pipeline that are not device work -- mode table, sample synthesis, digests,
recipe serialisation, cost model, report rendering -- pinned bit-for-bit against
the unmodified reference library (R0) where it is built, and by known answers
otherwise.  Reference: proj/src/harness.cpp:17-306, calibrator.cpp:12-40,
recipe.cpp:16-61,132-134, gflops.cpp:9-72, digest.hpp:12-43."""
import ctypes as C
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_2604_17320_b200 import harness as H

HAVE_REF = os.path.exists(O.REF_SO)
need_ref = pytest.mark.skipif(not HAVE_REF, reason="reference library not built (needs /root/reference)")


def test_modes():
    assert H.MODES == ("fp_baseline", "quant_only", "prune_only", "quant_then_prune", "prune_then_quant",
                       "collaborative")
    for m in H.MODES:
        assert H.parse_mode(H.mode_name(m)) == m
    assert H.parse_mode("quant-only") is None
    assert [H.mode_prunes(m) for m in H.MODES] == [False, False, True, True, True, True]
    assert [H.mode_quantizes(m) for m in H.MODES] == [False, True, False, True, True, True]


def test_fnv_known_answers():
    # FNV-1a 64 published vectors: "" -> offset basis, "a" -> af63dc4c8601ec8c
    assert H.to_hex(H.fnv1a64(b"")) == "cbf29ce484222325"
    assert H.to_hex(H.fnv1a64(b"a")) == "af63dc4c8601ec8c"
    assert H.to_hex(H.fnv1a64(b"foobar")) == "85944171f73967e8"


@need_ref
def test_fnv_matches_reference():
    rng = np.random.default_rng(3)
    for n in (0, 1, 7, 1000):
        v = rng.standard_normal(n)
        lib = O.ref_lib()
        ref = lib.qref_fnv1a64(O._d(v) if n else None, n)
        assert H.fnv1a64(v) == ref


@need_ref
@pytest.mark.parametrize("seed,count,v0,d,tmin,tmax", [(1001, 4, 16, 32, 8, 32), (2002, 8, 64, 48, 1, 1),
                                                       (7, 3, 1, 8, 3, 9), (2**63 + 5, 2, 5, 16, 2, 4)])
def test_samples_match_reference(seed, count, v0, d, tmin, tmax):
    ref, dg = O.ref_make_samples(seed, count, v0, d, tmin, tmax)
    mine = H.make_calibration_samples(seed, count, v0, d, tmin, tmax)
    assert len(mine) == count
    for (e, v, t), s in zip(ref, mine):
        assert (s.visual, s.text) == (v, t)
        assert np.array_equal(s.embeddings, e)  # bit-exact fp64
    assert H.sample_set_digest(mine) == dg


def test_samples_validation():
    with pytest.raises(ValueError, match="need at least one sample"):
        H.make_calibration_samples(1, 0, 4, 4, 1, 2)
    with pytest.raises(ValueError, match="invalid sample dims"):
        H.make_calibration_samples(1, 1, 0, 4, 1, 2)
    with pytest.raises(ValueError, match="invalid text range"):
        H.make_calibration_samples(1, 1, 4, 4, 3, 2)


RECIPES = [([2, 3], [0.5, 0.25], (0.25, 0.45, 0.10, 0.20), 64),
           ([5], [1.0], (0.3, 0.3, 0.3, 0.1), 576),
           ([1, 4, 9], [0.7, 0.7, 1e-3], (1 / 3, 1 / 3, 1 / 3, 0.0), 7),
           ([0, 11], [0.9, 0.30000000000000004], (0.25 + 0.2 / 3, 0.45 + 0.2 / 3, 0.1 + 0.2 / 3, 0.0), 144)]


@need_ref
@pytest.mark.parametrize("layers,keeps,w,v0", RECIPES)
def test_recipe_serialization_matches_reference(layers, keeps, w, v0):
    r = H.PruningRecipe(layers, keeps, H.MetricWeights(*w), v0, H.quant_digest())
    out, d17 = C.create_string_buffer(1 << 14), C.create_string_buffer(17)
    la, ka, wa = np.array(layers, np.int32), np.array(keeps, np.float64), np.array(w, np.float64)
    lib = O.ref_lib()
    assert lib.qref_serialize_recipe(len(layers), O._i(la), O._d(ka), O._d(wa), v0, b"w4a4kv4-sym-rne", out,
                                     out._length_, d17) == 0
    assert r.serialize() == out.value.decode()
    assert r.digest() == d17.value.decode()


def test_recipe_validation_and_weights():
    w = H.MetricWeights().without_quant()
    assert w.quant == 0.0 and abs(w.sum() - 1.0) < 1e-15
    assert w.mag == 0.25 + 0.2 / 3.0
    with pytest.raises(ValueError, match="strictly increasing"):
        H.PruningRecipe([3, 3], [0.5, 0.5]).validate()
    with pytest.raises(ValueError, match="non-increasing"):
        H.PruningRecipe([1, 3], [0.5, 0.6]).validate()
    with pytest.raises(ValueError, match="outside"):
        H.PruningRecipe([1], [0.0]).validate()
    with pytest.raises(ValueError, match="sum to 1"):
        H.PruningRecipe([1], [0.5], H.MetricWeights(0.5, 0.5, 0.5, 0.0)).validate()
    with pytest.raises(ValueError, match="nonempty"):
        H.PruningRecipe([], []).validate()
    assert H.quant_digest() == "w4a4kv4-sym-rne"


@need_ref
@pytest.mark.parametrize("layers,keeps,w,v0", RECIPES)
@pytest.mark.parametrize("n_layers,d,dff,heads,text_len,fvt,fpj", [(12, 32, 128, 4, 16, 0.0, 0.0),
                                                                   (32, 4096, 11008, 32, 64, 1e9, 2.5e8)])
def test_pipeline_flops_matches_reference(layers, keeps, w, v0, n_layers, d, dff, heads, text_len, fvt, fpj):
    r = H.PruningRecipe(layers, keeps, H.MetricWeights(*w), v0, H.quant_digest())
    cm = H.CostModel(fvt, fpj, d, dff, heads, text_len)
    g = H.pipeline_flops(H.executed_visual_lengths(r, n_layers), v0, cm)
    costs, f_vlm, f_base, ratio = O.ref_pipeline_flops(r.serialize(), n_layers, v0, d, dff, heads, text_len, fvt,
                                                       fpj)
    assert [x["cost"] for x in g["layers"]] == list(costs)
    assert (g["f_vlm"], g["f_base"], g["ratio_pct"]) == (f_vlm, f_base, ratio)
    # the non-pruning modes: every layer at v0 -> 100 %
    g0 = H.pipeline_flops([v0] * n_layers, v0, cm)
    _, a, b, r0 = O.ref_pipeline_flops(None, n_layers, v0, d, dff, heads, text_len, fvt, fpj)
    assert (g0["f_vlm"], g0["f_base"], g0["ratio_pct"]) == (a, b, r0) and r0 == 100.0


def test_cost_model_known_answers():
    cm = H.CostModel(0.0, 0.0, 32, 128, 4, 16)
    assert H.layer_cost(1, cm) == 8 * 32 * 32 + 4 * 32 + 4 * 32 * 128
    r = H.PruningRecipe([2, 4], [0.5, 0.25], v0=64)
    assert H.executed_visual_lengths(r, 6) == [64, 64, 64, 32, 32, 16]
    with pytest.raises(ValueError, match="non-increasing"):
        H.pipeline_flops([4, 5], 8, cm)
    with pytest.raises(ValueError, match="beyond model depth"):
        H.executed_visual_lengths(r, 4)


def test_compare_and_render():
    mk = lambda m, dv, fv, ratio, dg="e": H.RunReport(mode=m, eval_digest=dg, eval_count=2, divergence_mean=dv,
                                                       final_visual_count=fv, gflops={"ratio_pct": ratio})
    rows = H.compare_reports([mk("quant_only", 0.5, 64, 100.0), mk("collaborative", 0.25, 16, 42.5)])
    assert [r["mode"] for r in rows] == ["collaborative", "quant_only"]
    txt = H.render_comparison_text(rows)
    assert txt.splitlines() == ["mode           divergence_mean  final_visual_count  gflops_ratio_pct",
                                "collaborative  0.25             16                  42.5",
                                "quant_only     0.5              64                  100.0"]
    with pytest.raises(RuntimeError, match="different eval"):
        H.compare_reports([mk("a", 0, 1, 1.0), mk("b", 0, 1, 1.0, dg="f")])
    with pytest.raises(ValueError, match="at least two"):
        H.compare_reports([mk("a", 0, 1, 1.0)])
    j = H.report_to_json(H.RunReport(mode="prune_only", traces=[[(2, 3, [0, 5, 9])]], gflops={"ratio_pct": 1.0}))
    assert j["traces"] == [[{"layer": 2, "budget": 3, "retained_indices": [0, 5, 9]}]]
    assert j["meta"]["tool_version"] == "0.1.0"
    assert math.isclose(j["gflops"]["ratio_pct"], 1.0)
