"""Calibration on the B200: fit_act_scales (calibrator.cpp:237-249)
-- full-precision forwards with the ActStats collector (model.cpp:174-210) -- against
the unmodified reference on identical weights and samples, then the quantized
prefill with the device-fitted scales against the reference prefill with its own."""
import numpy as np
import pytest

import oracle as O
import paper_2604_17320_b200 as Q

pytestmark = pytest.mark.gpu


def _setup(L=4, d=256, H=4):
    cfg = O.ModelCfg(n_layers=L, d_model=d, n_heads=H, n_kv_heads=H, d_head=d // H, d_ff=4 * d, weight_axis=2)
    ref = O.Ref(cfg, seed=7)
    w = O.synth_weights(cfg, seed=3)
    ref.set_weights(w)
    calib = [(O.synth_embeddings(144 + 16 + 4 * i, d, seed=100 + i), 144, 16 + 4 * i) for i in range(4)]
    return cfg, ref, w, calib


def test_fit_act_scales_matches_reference(torch_cuda):
    cfg, ref, w, calib = _setup()
    exp = ref.fit_act_scales(calib)
    e = Q.Engine(Q.Config(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=1024),
                 max_batch=2, max_tokens=1024, max_seq=512, max_decode=16)
    e.keep_fp_weights(True)
    e.load_weights(w)
    got = e.fit_act_scales(calib)
    # fp64 on both sides; only reduction order (DGEMM, tree sums) differs
    np.testing.assert_allclose(got, exp, rtol=1e-10)
    # the quantized prefill with the device-fitted scales tracks the reference with its own
    ref.prepare(exp, weight_axis=2)
    rec = O.Recipe([0, 1, 2, 3], [1.0, 0.5, 0.3, 0.3], v0=144)
    emb = O.synth_embeddings(184, 256, seed=11)
    res = ref.prefill(emb, 144, 40, rec).result()
    e.set_recipe(rec.candidate_layers, rec.keep_ratios, rec.weights, rec.v0, 4)
    lg = e.prefill(emb.astype(np.float32), [144], [40])
    for (l1, b1, p1), (l2, b2, p2) in zip(e.trace(0), res.trace):
        assert (l1, b1) == (l2, b2) and np.array_equal(p1, p2)
    assert np.abs(lg - res.logits).max() <= 1e-2


def test_fit_act_scales_requires_fp_weights(torch_cuda):
    cfg, ref, w, calib = _setup()
    e = Q.Engine(Q.Config(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=1024),
                 max_batch=1, max_tokens=512, max_seq=512, max_decode=1)
    e.load_weights(w)
    with pytest.raises(Q.QuotaInvalidArgument, match="full-precision weights"):
        e.fit_act_scales(calib)


def test_profile_sensitivity_matches_reference(torch_cuda):
    """QUOTA Eq. 1 (calibrator.cpp:42-82): device quantized vs fp64 block outputs against the
    reference's own profile_sensitivity on identical weights, scales and samples."""
    cfg, ref, w, calib = _setup()
    acts = ref.fit_act_scales(calib)
    ref.prepare(acts, weight_axis=2)
    layers = [0, 1, 2, 3]
    raw_ref, nrm_ref = ref.profile_sensitivity(calib, layers)
    e = Q.Engine(Q.Config(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=1024),
                 max_batch=2, max_tokens=1024, max_seq=512, max_decode=16)
    e.keep_fp_weights(True)
    e.load_weights(w)
    e.set_act_scales(acts)
    raw, nrm = e.profile_sensitivity(calib, layers)
    print("raw ref", raw_ref, "gpu", raw)
    # the quantized side differs from the reference only by fp32 activation buffers (and the
    # rare rounding-tie code flip they cause); measured agreement is ~1e-8 relative
    np.testing.assert_allclose(raw, raw_ref, rtol=1e-4)
    np.testing.assert_allclose(nrm, nrm_ref, atol=1e-3)
    assert np.all((nrm >= 0.1) & (nrm <= 0.9))


def test_quota_calibration_recipe_matches_reference(torch_cuda):
    """The offline QUOTA pipeline on the device: act scales, layer diagnostics
    (top-10 text->visual attention mass, median pairwise cosine), the candidate window, Eq. 1
    sensitivities and the Eqs. 3-4 keep schedule -> the same recipe as the reference pipeline."""
    cfg = O.ModelCfg(n_layers=8, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=1024, weight_axis=2)
    ref = O.Ref(cfg, seed=7)
    w = O.synth_weights(cfg, seed=5)
    ref.set_weights(w)
    samples = [(O.synth_embeddings(64 + 8 + 4 * i, 256, seed=300 + i), 64, 8 + 4 * i) for i in range(6)]
    exp = ref.run_calibration(samples, window=3)
    e = Q.Engine(Q.Config(n_layers=8, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=1024),
                 max_batch=1, max_tokens=512, max_seq=512, max_decode=4)
    e.keep_fp_weights(True)
    e.load_weights(w)
    got = e.run_quota_calibration(samples, window=3)
    np.testing.assert_allclose(got["act_scales"], exp["act_scales"], rtol=1e-10)
    np.testing.assert_allclose(got["conc"], exp["conc"], rtol=1e-4)
    np.testing.assert_allclose(got["red"], exp["red"], rtol=1e-6, atol=1e-9)
    assert got["layers"].tolist() == exp["layers"].tolist()
    np.testing.assert_allclose(got["raw"], exp["raw"], rtol=1e-4)
    np.testing.assert_allclose(got["keeps"], exp["keeps"], rtol=1e-3)
    assert got["keeps"][-1] == 0.3 and np.all(np.diff(got["keeps"]) <= 1e-12)
