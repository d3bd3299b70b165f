"""C-ABI boundary checks that need no GPU: the sm_100a library loads, exports
every entry point include/quota_b200.h declares, the host-side recipe parser
behaves like the reference parse_recipe (recipe.cpp:21-46,65-116: same
accepted values, same exception class, same message), and compute entry points
fail loudly instead of falling back to the CPU when no device is present."""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_2604_17320_b200 as Q

KATS = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "kats.json")))


def test_library_exports_every_header_symbol():
    lib = Q.lib()
    syms = Q.exported_symbols()
    assert len(syms) >= 20
    nm = subprocess.run(["nm", "-D", "--defined-only", Q.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in nm.splitlines() if l.strip()}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        getattr(lib, s)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", Q.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out[:500]


def test_recipe_parse_matches_reference_on_valid_recipe():
    got = Q.parse_recipe(KATS["recipe_good"]["text"])
    exp = KATS["recipe_good"]["parsed"]
    assert got["candidate_layers"] == exp["candidate_layers"]
    assert got["keep_ratios"] == exp["keep_ratios"]
    assert tuple(got["weights"]) == tuple(exp["weights"])
    assert got["v0"] == exp["v0"] and got["quant_digest"] == exp["quant_digest"]


@pytest.mark.parametrize("name", sorted(KATS["recipe_bad"]))
def test_recipe_parse_errors_match_reference(name):
    case = KATS["recipe_bad"][name]
    with pytest.raises(Q.QuotaInvalidArgument) as ei:
        Q.parse_recipe(case["text"])
    if name == "syntax":  # the reference message comes from nlohmann's parser; ours names the byte offset
        assert "parse error" in str(ei.value)
    else:
        assert str(ei.value) == case["error"]


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(Q.QuotaError) as ei:
        Q.Engine(Q.Config(), max_batch=1, max_tokens=64, max_seq=64, max_decode=1)
    assert ei.value.code == Q.QT_ECUDA
