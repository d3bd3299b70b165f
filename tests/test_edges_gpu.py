"""Edge cases and error behaviour of the device path against the reference
(model.cpp:49-72,317-325,455-467; selector.cpp:70-71,211-228): text-only and
visual-only sequences, retain-all budgets, a budget of one token, recipe layers
beyond the model, capacity limits, and the reference's exception classes."""
import numpy as np
import pytest

import oracle as O
import paper_2604_17320_b200 as Q

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pair(torch_cuda):
    cfg = O.ModelCfg(n_layers=4, d_model=128, n_heads=2, n_kv_heads=2, d_head=64, d_ff=344, mlp=1, act_mode=1,
                     weight_axis=2)
    w = O.synth_weights(cfg, seed=4)
    port = O.Port(cfg)
    port.set_weights(w)
    port.prepare(None)
    e = Q.Engine(Q.Config(n_layers=4, d_model=128, n_heads=2, n_kv_heads=2, d_head=64, d_ff=344, mlp=1, act_mode=1),
                 max_batch=4, max_tokens=1024, max_seq=512, max_decode=8)
    e.load_weights(w)
    return cfg, port, e


def _run(port, e, V, T, rec, seed=1):
    emb = O.synth_embeddings(V + T, 128, seed=seed)
    if rec is None:
        e.clear_recipe()
    else:
        e.set_recipe(rec.candidate_layers, rec.keep_ratios, rec.weights, rec.v0, 4)
    lg = e.prefill(emb.astype(np.float32), [V], [T])
    res = port.prefill(emb, V, T, rec).result()
    return lg, res, e.trace(0), e.layout(0)


def test_text_only_sequence(pair):
    cfg, port, e = pair
    lg, res, tr, lay = _run(port, e, 0, 24, None)
    assert tr == [] and lay[0] == 0 and lay[1] == 24
    assert np.abs(lg - res.logits).max() <= 1e-2


def test_text_only_with_recipe_raises_like_reference(pair):
    cfg, port, e = pair
    e.set_recipe([1], [0.5], v0=8)
    with pytest.raises(Q.QuotaInvalidArgument, match="empty sample"):
        e.prefill(O.synth_embeddings(24, 128, seed=2).astype(np.float32), [0], [24])
    with pytest.raises(O.OracleError, match="empty sample"):
        port.prefill(O.synth_embeddings(24, 128, seed=2), 0, 24, O.Recipe([1], [0.5], v0=8))


def test_visual_only_sequence_pruned(pair):
    cfg, port, e = pair
    lg, res, tr, lay = _run(port, e, 40, 0, O.Recipe([1, 2], [0.5, 0.25], v0=40))
    assert [(l, b) for l, b, _ in tr] == [(l, b) for l, b, _ in res.trace] == [(1, 20), (2, 10)]
    for (_, _, p1), (_, _, p2) in zip(tr, res.trace):
        assert np.array_equal(p1, p2)
    assert np.abs(lg - res.logits).max() <= 1e-2


def test_budget_of_one_and_retain_all(pair):
    cfg, port, e = pair
    lg, res, tr, lay = _run(port, e, 30, 8, O.Recipe([0, 3], [1.0, 1e-6], v0=30))
    assert [(l, b) for l, b, _ in tr] == [(3, 1)] and lay[0] == 1
    assert np.array_equal(tr[0][2], res.trace[0][2])
    assert np.abs(lg - res.logits).max() <= 1e-2


def test_recipe_layers_beyond_model_are_ignored(pair):
    cfg, port, e = pair
    a, res, tr, _ = _run(port, e, 30, 8, O.Recipe([2, 9], [0.5, 0.25], v0=30))
    assert [(l, b) for l, b, _ in tr] == [(2, 15)] == [(l, b) for l, b, _ in res.trace]
    assert np.abs(a - res.logits).max() <= 1e-2


def test_capacity_and_state_errors(pair):
    cfg, port, e = pair
    e.clear_recipe()
    with pytest.raises(Q.QuotaInvalidArgument, match="capacity"):
        e.prefill(np.zeros((600, 128), np.float32), [580], [20])  # > max_seq
    with pytest.raises(Q.QuotaInvalidArgument):
        e.prefill(np.zeros((10, 128), np.float32), [0], [0])  # empty sequence
    fresh = Q.Engine(Q.Config(n_layers=4, d_model=128, n_heads=2, n_kv_heads=2, d_head=64, d_ff=344, mlp=1,
                              act_mode=1), max_batch=1, max_tokens=64, max_seq=64, max_decode=2)
    with pytest.raises(Q.QuotaInvalidArgument, match="not loaded"):
        fresh.prefill(np.zeros((4, 128), np.float32), [2], [2])
    with pytest.raises(Q.QuotaRuntimeError, match="cache and execution mode mismatch"):
        fresh.decode(np.zeros((1, 128), np.float32))
    fresh.close()
    with pytest.raises(Q.QuotaInvalidArgument):
        Q.Engine(Q.Config(n_layers=4, d_model=130, n_heads=2, n_kv_heads=2, d_head=65), max_batch=1, max_tokens=8,
                 max_seq=8, max_decode=1)
    with pytest.raises(Q.QuotaInvalidArgument, match="keep ratio"):
        e.set_recipe([1], [1.5], v0=10)


def test_decode_capacity_limit(pair):
    cfg, port, e = pair
    e.clear_recipe()
    e.prefill(O.synth_embeddings(20, 128, seed=3).astype(np.float32), [12], [8])
    x = np.zeros((1, 128), np.float32)
    for _ in range(8):
        e.decode(x)
    with pytest.raises(Q.QuotaInvalidArgument, match="decode steps"):
        e.decode(x)


def test_packed_weight_file_roundtrip(pair, tmp_path):
    """save -> load into a fresh engine -> bit-identical prefill and decode."""
    cfg, port, e = pair
    e.clear_recipe()
    emb = O.synth_embeddings(40, 128, seed=8).astype(np.float32)
    a = e.prefill(emb, [30], [10]).copy()
    da = e.decode(np.ones((1, 128), np.float32)).copy()
    path = str(tmp_path / "w.qtw")
    e.save(path)
    f = Q.Engine(Q.Config(n_layers=4, d_model=128, n_heads=2, n_kv_heads=2, d_head=64, d_ff=344, mlp=1, act_mode=1),
                 max_batch=4, max_tokens=1024, max_seq=512, max_decode=8)
    f.load(path)
    b = f.prefill(emb, [30], [10])
    db = f.decode(np.ones((1, 128), np.float32))
    assert np.array_equal(a, b) and np.array_equal(da, db)
    g = Q.Engine(Q.Config(n_layers=4, d_model=128, n_heads=2, n_kv_heads=1, d_head=64, d_ff=344, mlp=1, act_mode=1),
                 max_batch=1, max_tokens=64, max_seq=64, max_decode=1)
    with pytest.raises(Q.QuotaInvalidArgument, match="does not match"):
        g.load(path)
    f.close()
    g.close()


def test_graph_and_eager_decode_identical(pair):
    """The CUDA-graph replay of a decode step equals the eager launch sequence bitwise
    (profiling runs the step eagerly)."""
    cfg, port, e = pair
    e.clear_recipe()
    emb = O.synth_embeddings(40, 128, seed=9).astype(np.float32)
    xs = [O.synth_embeddings(1, 128, seed=60 + i).astype(np.float32) for i in range(4)]
    e.prefill(emb, [30], [10])
    g = [e.decode(x).copy() for x in xs]
    e.prefill(emb, [30], [10])
    h = []
    for x in xs:
        e.profile_next()  # eager path for this step
        h.append(e.decode(x).copy())
    for a, b in zip(g, h):
        assert np.array_equal(a, b)


def test_profile_chain_leaves_decode_state(pair):
    """qt_engine_profile_chain (bench.py's per-class decode timing) replays graph-captured
    steps with kernel classes left out, then restores cache lengths and positions: the decode
    that follows is bitwise the one without profiling."""
    cfg, port, e = pair
    e.clear_recipe()
    emb = O.synth_embeddings(40, 128, seed=19).astype(np.float32)
    xs = [O.synth_embeddings(1, 128, seed=80 + i).astype(np.float32) for i in range(3)]
    e.prefill(emb, [30], [10])
    g = [e.decode(x).copy() for x in xs]
    e.prefill(emb, [30], [10])
    h = [e.decode(xs[0]).copy()]
    for mask in (0, 1 | 4 | 8, 15):
        assert e.profile_chain(mask, reps=3) > 0.0
    h += [e.decode(x).copy() for x in xs[1:]]
    for a, b in zip(g, h):
        assert np.array_equal(a, b)
    v, t, pos = e.layout(0)
    assert (v, t) == (30, 13) and pos[-1] == 42


def test_async_logits_readback(pair):
    """qt_engine_prefill with out_on_device = 2: the host logits arrive on the copy stream while
    decode steps run; after synchronize() they equal the synchronous readback, and a following
    prefill waits for the pending copy before reusing the device buffer."""
    cfg, port, e = pair
    e.clear_recipe()
    emb = O.synth_embeddings(40, 128, seed=29).astype(np.float32)
    emb2 = O.synth_embeddings(40, 128, seed=30).astype(np.float32)
    ref = e.prefill(emb, [30], [10]).copy()
    ref2 = e.prefill(emb2, [30], [10]).copy()
    out = np.zeros_like(ref)
    e.prefill(emb, [30], [10], logits_out=out, logits_async=True)
    e.decode(O.synth_embeddings(1, 128, seed=31).astype(np.float32))
    out2 = np.zeros_like(ref2)
    e.prefill(emb2, [30], [10], logits_out=out2, logits_async=True)  # joins the first copy
    e.synchronize()
    assert np.array_equal(out, ref) and np.array_equal(out2, ref2)
    # pinned host buffers: the device->host copy is truly asynchronous, so the join that keeps
    # the second prefill from overwriting the device logits mid-copy is exercised
    import torch
    p1 = torch.zeros(ref.shape, dtype=torch.float32).pin_memory()
    p2 = torch.zeros(ref2.shape, dtype=torch.float32).pin_memory()
    for _ in range(3):
        p1.zero_()
        p2.zero_()
        e.prefill(torch.from_numpy(emb).pin_memory(), [30], [10], logits_out=p1, logits_async=True)
        e.decode(O.synth_embeddings(1, 128, seed=31).astype(np.float32))
        e.prefill(torch.from_numpy(emb2).pin_memory(), [30], [10], logits_out=p2, logits_async=True)
        e.synchronize()  # the returned rows are valid only now
        assert np.array_equal(p1.numpy(), ref) and np.array_equal(p2.numpy(), ref2)


def test_greedy_decode_matches_restatement(torch_cuda):
    """Greedy decoding (BASELINE.json "greedy steps"): token = argmax of the previous logits
    (ties to the smaller id), input = its row of a token-embedding table -- the GPU's tokens equal
    the restatement driven the same way (numpy argmax of its fp64 logits), and so do the logits."""
    cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=2, d_head=64, d_ff=688, mlp=1, act_mode=1,
                     weight_axis=2)
    w = O.synth_weights(cfg, seed=21)
    port = O.Port(cfg)
    port.set_weights(w)
    port.prepare(None)
    table = O.synth_embeddings(200, 256, seed=77)  # vocab 200 <= d_model
    e = Q.Engine(Q.Config(n_layers=4, d_model=256, n_heads=4, n_kv_heads=2, d_head=64, d_ff=688, mlp=1, act_mode=1),
                 max_batch=2, max_tokens=512, max_seq=256, max_decode=12)
    e.load_weights(w)
    e.set_token_table(table.astype(np.float32))
    rec = O.Recipe([1, 2], [0.5, 0.3], v0=144)
    e.set_recipe(rec.candidate_layers, rec.keep_ratios, rec.weights, rec.v0, 4)
    embs = [O.synth_embeddings(184, 256, seed=13), O.synth_embeddings(150, 256, seed=14)]
    lg = e.prefill(np.concatenate(embs).astype(np.float32), [144, 110], [40, 40])
    runs = [port.prefill(embs[0], 144, 40, rec), port.prefill(embs[1], 110, 40, rec)]
    last = [r.result().logits[-1] for r in runs]
    for step in range(12):
        tok, g = e.decode_greedy()
        for b in range(2):
            prev = last[b][:200]
            exp_tok = int(np.argmax(prev))
            top2 = np.sort(prev)[-2:]
            if top2[1] - top2[0] < 1e-5:  # a near-tie argmax: the sequences may legitimately part
                return
            assert tok[b] == exp_tok, (step, b, tok[b], exp_tok)
            last[b] = runs[b].decode(table[exp_tok])
            assert np.abs(g[b].astype(np.float64) - last[b]).max() <= 1e-2
