"""The reference C++ API as the drop-in surface (north_star).

tests/cxx/dropin_main.cpp is a client of the UNMODIFIED reference headers and
library: it fits static act scales with full-precision forwards, builds a
per-output-channel QuantEnv, parses a recipe, calls make_recipe_hook,
forward_prefill (quantized) and decode_step.  It runs twice: against the
reference library alone (CPU, fp64) and with libquota_b200_cxx.so preloaded,
which serves forward_prefill / decode_step / make_recipe_hook on the B200.
Retained positions, layouts and cache shapes must be identical; logits within
north_star's 1e-2 max-abs."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_main")
CXX_SO = os.path.join(ROOT, "paper_2604_17320_b200", "_build", "libquota_b200_cxx.so")


def _parse(path):
    out = {"prune": [], "kv": [], "decode": [], "hookprune": [], "rec": [], "block": []}
    for line in open(path):
        t = line.split()
        if t[0] in ("prune", "hookprune"):
            out[t[0]].append(list(map(int, t[1:])))
        elif t[0] == "rec":
            out["rec"].append(list(map(int, t[1:5])) + list(map(float, t[5:])))
        elif t[0] == "block":
            out["block"].append((int(t[1]), int(t[2]), float(t[3])))
        elif t[0] == "hooklogits":
            out["hooklogits"] = np.array(list(map(float, t[3:]))).reshape(int(t[1]), int(t[2]))
        elif t[0] == "kv":
            out["kv"].append((int(t[1]), int(t[3]), int(t[5])))
        elif t[0] == "logits":
            out["logits"] = np.array(list(map(float, t[3:]))).reshape(int(t[1]), int(t[2]))
        elif t[0] == "decode":
            out["decode"].append(np.array(list(map(float, t[2:]))))
        else:
            out[t[0]] = " ".join(t[1:])
    return out


def _run(tmp_path, name, preload):
    if not os.path.exists(EXE) or not os.path.exists(CXX_SO):
        pytest.skip("drop-in binaries not built (make -C oracle dropin; make -C paper_2604_17320_b200/csrc cxx)")
    env = dict(os.environ)
    if preload:
        env["LD_PRELOAD"] = CXX_SO
    out = tmp_path / name
    r = subprocess.run([EXE, str(out), "8"], env=env, capture_output=True, text=True, timeout=600)
    return r, out


@pytest.mark.gpu
def test_reference_api_client_runs_on_b200(tmp_path):
    r, cpu = _run(tmp_path, "cpu.txt", False)
    assert r.returncode == 0, r.stderr
    r, gpu = _run(tmp_path, "gpu.txt", True)
    assert r.returncode == 0, r.stderr
    a, b = _parse(cpu), _parse(gpu)
    assert a["layout"] == b["layout"]
    assert a["prune"] == b["prune"]  # retained original positions, bit-exact
    assert [(l, rows) for l, rows, _ in a["kv"]] == [(l, rows) for l, rows, _ in b["kv"]]
    assert a["logits"].shape == b["logits"].shape
    assert np.abs(a["logits"] - b["logits"]).max() <= 1e-2
    assert len(a["decode"]) == len(b["decode"]) == 8
    for x, y in zip(a["decode"], b["decode"]):
        assert np.abs(x - y).max() <= 1e-2
    assert a["final"] == b["final"]
    # records / block outputs: the same layers and shapes; probability and state sums agree
    assert a["records"] == b["records"] == "4 blocks 4"
    for ra, rb in zip(a["rec"], b["rec"]):
        assert ra[:4] == rb[:4]
        np.testing.assert_allclose(rb[4:], ra[4:], rtol=1e-3)
    for ba, bb in zip(a["block"], b["block"]):
        assert ba[:2] == bb[:2]
        np.testing.assert_allclose(bb[2], ba[2], rtol=1e-3)
    # an arbitrary PruneHook (host-side, per layer) prunes identically and keeps the logits
    assert a["hookprune"] == b["hookprune"] and len(a["hookprune"]) == 2
    assert np.abs(a["hooklogits"] - b["hooklogits"]).max() <= 1e-2
    assert a["badhook"] == b["badhook"] == "runtime_error retained slots must be ascending and unique"
    # the stock prepare_quant_env: per row on the reference, per output channel (== the
    # per-channel env, bitwise) under the device library
    assert a["stockenv"] == "axis 1 same 0" and b["stockenv"] == "axis 2 same 1"
    assert a["perrow"] == "ok" and b["perrow"] == "invalid_argument"


def test_backend_exports_reference_entry_points():
    if not os.path.exists(CXX_SO):
        pytest.skip("libquota_b200_cxx.so not built")
    nm = subprocess.run(["nm", "-DC", "--defined-only", CXX_SO], capture_output=True, text=True).stdout
    for sym in ("quota::forward_prefill(", "quota::decode_step(", "quota::make_recipe_hook(",
                "quota::prepare_quant_env(", "quota_b200::prepare_quant_env_per_channel("):
        assert sym in nm, sym


def test_backend_without_gpu_fails_loudly(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r, _ = _run(tmp_path, "x.txt", True)
    assert r.returncode != 0
    assert "no CPU fallback" in r.stderr


@pytest.mark.gpu
def test_reference_api_client_without_host_kv(tmp_path):
    """QUOTA_B200_HOST_KV=0: the returned KVCacheState carries layout and positions only (no
    host copy of the int4 cache); decode still runs on the device session."""
    r, cpu = _run(tmp_path, "cpu.txt", False)
    assert r.returncode == 0, r.stderr
    env = dict(os.environ, LD_PRELOAD=CXX_SO, QUOTA_B200_HOST_KV="0")
    out = tmp_path / "gpu_nokv.txt"
    r = subprocess.run([EXE, str(out), "8"], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    a, b = _parse(cpu), _parse(out)
    assert a["prune"] == b["prune"]
    assert all(ks == 0 for _, _, ks in b["kv"])  # no host codes materialised
    for x, y in zip(a["decode"], b["decode"]):
        assert np.abs(x - y).max() <= 1e-2
