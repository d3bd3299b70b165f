"""TEST INFRASTRUCTURE ONLY -- the checker for paper_2604_17320_b200.harness.

run_pipeline (proj/src/harness.cpp:59-179) restated over the UNMODIFIED
reference library (R0, oracle/_ref/libquota_ref.so): every forward is the
reference's forward_prefill (model.cpp:315-453) with make_recipe_hook
(selector.cpp:211-228), every scale fit its fit_act_scales
(calibrator.cpp:237-249), the inline recipe its run_quota_calibration steps
(calibrator.cpp:251-268, on explicit samples), the cost its pipeline_flops
(gflops.cpp:24-72).  Only the orchestration is restated, line by line from
harness.cpp, so the model can be the one the device engine holds and the
QuantEnv per output channel (the device path's weight axis);
everything else is the reference's own code.
"""
from __future__ import annotations

import math

import numpy as np

from . import Recipe, Ref, ref_pipeline_flops

PRUNING = ("prune_only", "quant_then_prune", "prune_then_quant", "collaborative")  # harness.cpp:46-49
QUANTIZED = ("quant_only", "quant_then_prune", "prune_then_quant", "collaborative")  # harness.cpp:51-54
STAGE_WISE = ("prune_only", "quant_then_prune", "prune_then_quant")  # harness.cpp:92-94


def _without_quant(w):  # recipe.cpp:16-19
    share = w[3] / 3.0
    return (w[0] + share, w[1] + share, w[2] + share, 0.0)


def ref_run_pipeline(ref: Ref, mode, eval_samples, calib_samples, recipe: Recipe | None = None,
                     weights=(0.25, 0.45, 0.10, 0.20), v0=64, window=5, p_min=0.3, tau=0.25, eta=1e-6,
                     act_bits=4, text_len=16, f_vt=0.0, f_pj=0.0, weight_axis=2):
    """-> dict(divergence_mean, traces, final_visual_count, gflops=(costs, f_vlm, f_base, ratio),
    recipe, act_scales).  ref: a Ref holding the model; weight_axis: the QuantEnv weight axis
    (2 = PerColumn, the device path; 1 = PerRow, the reference harness)."""
    cfg = ref.cfg
    prunes, quantized = mode in PRUNING, mode in QUANTIZED
    calib_out = None
    if prunes:
        if recipe is None:
            calib_out = ref.run_calibration(calib_samples, window=window, p_min=p_min, tau=tau, eta=eta)
            recipe = Recipe([int(x) for x in calib_out["layers"]], [float(x) for x in calib_out["keeps"]],
                            tuple(weights), v0)
        if recipe.candidate_layers[-1] >= cfg.n_layers:
            raise RuntimeError("recipe candidate layers do not fit the model")
    scoring = None
    if prunes:
        scoring = _without_quant(recipe.weights) if mode in STAGE_WISE else tuple(recipe.weights)
    scales = None
    if quantized:
        if mode == "prune_then_quant":
            scales = ref.fit_act_scales(calib_samples, recipe=recipe, weights=np.array(scoring))
        elif calib_out is not None:
            scales = calib_out["act_scales"]
        else:
            scales = ref.fit_act_scales(calib_samples)
        ref.prepare(scales, weight_axis=weight_axis)
    res_bits = act_bits if quantized else -1
    div, traces, finals, logits = 0.0, [], [], []
    for emb, v, t in eval_samples:
        fp = ref.prefill(emb, v, t, recipe=None, quantized=False).result()
        run = ref.prefill(emb, v, t, recipe=recipe if prunes else None, quantized=quantized,
                          res_bits=res_bits, weights=np.array(scoring) if prunes else None).result()
        div += math.sqrt(float(np.sum((run.logits[-1] - fp.logits[-1]) ** 2)))
        traces.append([(int(l), int(b), [int(p) for p in ps]) for l, b, ps in run.trace])
        finals.append(int(run.visual))
        logits.append(run.logits)
    if len(set(finals)) > 1:
        raise RuntimeError("inconsistent final visual count across samples")
    fl = ref_pipeline_flops(recipe.to_json() if prunes else None, cfg.n_layers, recipe.v0 if prunes else v0,
                            cfg.d_model, cfg.d_ff, cfg.n_heads, text_len,
                            f_vt, f_pj)
    return dict(divergence_mean=div / len(eval_samples), traces=traces, final_visual_count=finals[0], gflops=fl,
                recipe=recipe, act_scales=scales, logits=logits)
