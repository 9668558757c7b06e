"""NEXT-2 GPU parity: the end-to-end Feed train step (FeedModel: library sparse path + fp32
PyTorch tower, one global clip through emb_backward_adagrad_dev) vs the oracle
(oracle/feed_model.py: fp64 tower + C sparse oracle) on the same seeded inputs.

Tolerances follow the arithmetic: the tower runs in fp32 (cuBLAS, TF32 off), so dL/dpooled
and the dense gradients carry ~1e-6 relative error against the fp64 oracle; the loss and
the clip factor are compared at 1e-5 relative, updated parameters relative to the size of
their own update (1e-3 of the step, plus fp32 ulps of the weight)."""
import numpy as np
import pytest

import oracle as O
from oracle import feed_model as FM
from helpers import dense_tables, init_tables_host, make_emb, problem
from test_gpu_parity import dev, small_cfg
from workload import gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("scale", [1.0, 40.0])  # clip inactive / active
def test_feed_train_step_matches_oracle(gpu, scale):
    from paper_2402_06859_b200.feed_model import FeedModel
    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = small_cfg(dim=32, rows=(3000, 500, 80), F=[0, 1, 0, 2], B=64)
    B, Dd = 64, 16
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 3, 0)
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B)
    init_tables_host(emb, cfg)
    model = FeedModel(emb, Dd, lr=0.05, seed=7)
    with torch.no_grad():
        for p in model.params:
            p.mul_(scale)
    rng = np.random.default_rng(5)
    dense = rng.standard_normal((B, Dd)).astype(np.float32)
    labels = rng.integers(0, 2, size=B).astype(np.float32)
    params0 = [p.detach().cpu().double().numpy().copy() for p in model.params]
    loss = model.train_step(dev(ids), dev(off), B, dev(dense), dev(labels))
    torch.cuda.synchronize()
    assert emb.sync() == 0
    # oracle on the same inputs
    W = dense_tables(cfg)
    W0 = W.copy()
    A = np.full(cfg.total_rows, 0.1, dtype=np.float32)
    params = [p.copy() for p in params0]
    accs = [np.full_like(p, 0.1) for p in params]
    r = FM.feed_train_step(problem(cfg), W, A, ids, off, B, dense.astype(np.float64),
                           labels.astype(np.float64), params, accs, 0.05, 1e-7, 1.0)
    assert abs(float(loss) - r["loss"]) <= 1e-5 * abs(r["loss"])
    assert abs(float(model.S) - r["S"]) <= 1e-5 * r["S"]
    assert abs(float(model.c) - float(r["c"])) <= 1e-5 * float(r["c"])
    if scale > 1:
        assert r["c"] < 1.0
    # dense parameters
    for got, ref, old in zip(model.params, params, params0):
        g = got.detach().cpu().double().numpy()
        step = np.abs(ref - old)
        assert (np.abs(g - ref) <= 1e-3 * step + 4 * np.spacing(np.abs(ref).astype(np.float32))).all()
    # sparse rows
    Wg = np.concatenate([emb.read_rows(t, np.arange(cfg.table_rows[t]), with_acc=False)
                         for t in range(cfg.num_tables)])
    step = np.abs(W - W0)
    assert (np.abs(Wg - W) <= 1e-3 * step + 4 * np.spacing(np.abs(W))).all()
    assert (Wg[step == 0] == W0[step == 0]).all()


def test_feed_train_step_has_no_host_sync_and_overlaps_dedup(gpu):
    """The step enqueues everything on the library stream: issuing 3 steps back to back
    returns before the device finishes them (no host synchronisation inside the step)."""
    from paper_2402_06859_b200.feed_model import FeedModel
    cfg = small_cfg(dim=64, rows=(200_000, 5000), F=[0, 1, 0], B=4096, maxlen=20)
    B, Dd = 4096, 64
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 3, 0)
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B)
    init_tables_host(emb, cfg)
    model = FeedModel(emb, Dd)
    x = torch.randn(B, Dd, device=gpu)
    y = (torch.rand(B, device=gpu) > 0.5).float()
    ids_d, off_d = dev(ids), dev(off)
    model.train_step(ids_d, off_d, B, x, y)
    torch.cuda.synchronize()
    ev = torch.cuda.Event()
    with torch.cuda.stream(emb.stream):
        torch.cuda._sleep(200_000_000)  # ~0.1 s of device time queued ahead of the steps
    for _ in range(3):
        loss = model.train_step(ids_d, off_d, B, x, y)
    ev.record(emb.stream)
    assert not ev.query()  # the host got here while the device is still busy
    torch.cuda.synchronize()
    assert emb.sync() == 0 and np.isfinite(float(loss))


def test_feed_model_skips_dense_update_on_nonfinite_norm(gpu):
    """a non-finite global norm (here from an inf dense feature, so the dense
    gradients themselves are inf/NaN) skips BOTH updates: the library leaves the sparse rows
    alone (c = -1) and the tower parameters and accumulators stay bit-identical (the scaled
    gradient is masked to 0, not multiplied by 0)."""
    from paper_2402_06859_b200 import _lib as L
    from paper_2402_06859_b200.feed_model import FeedModel
    cfg = small_cfg(dim=32, rows=(3000, 500, 80), F=[0, 1, 0, 2], B=64)
    B, Dd = 64, 16
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 3, 0)
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B)
    init_tables_host(emb, cfg)
    model = FeedModel(emb, Dd, lr=0.05, seed=7)
    dense = np.ones((B, Dd), dtype=np.float32)
    dense[3, 5] = np.inf
    labels = np.zeros(B, dtype=np.float32)
    p0 = [p.detach().clone() for p in model.params]
    a0 = [a.clone() for a in model.acc]
    w0 = emb.weights.clone()
    model.train_step(dev(ids), dev(off), B, dev(dense), dev(labels))
    torch.cuda.synchronize()
    assert emb.sync() == L.EMB_ENONFINITE
    assert float(model.c) == -1.0
    for p, q in zip(model.params, p0):
        assert torch.equal(p.detach(), q)
    for a, q in zip(model.acc, a0):
        assert torch.equal(a, q)
    assert torch.equal(emb.weights, w0)


@pytest.mark.parametrize("sharding", ["row", "table"])
def test_feed_model_data_parallel_w2_matches_global_batch_oracle(gpu, sharding):
    """NEXT-2 at W = 2 (PAPER.md:576 data-parallel dense side, PAPER.md:17 one global clip):
    two loopback ranks, each with its local batch and its own tower replica; the tower
    gradients are summed over ranks (emb_allreduce_f32) before their norm, so both ranks
    clip with the same c and end with identical towers -- equal to the oracle's single step on
    the GLOBAL batch (2B samples)."""
    import threading
    from paper_2402_06859_b200 import LoopbackHub, ShardedEmbedding
    from paper_2402_06859_b200.feed_model import FeedModel
    from test_sharded_gpu import global_batch, run_ranks
    torch.backends.cuda.matmul.allow_tf32 = False
    W = 2
    cfg = small_cfg(dim=32, rows=(3000, 500, 80), F=[0, 1, 0, 2], B=64)
    B, Dd, F, D = 64, 16, cfg.num_features, cfg.dim
    per_rank = [gen.make_batch(cfg.table_rows, cfg.features, B, 3 + r, 0) for r in range(W)]
    nnz_max = max(len(i) for i, _ in per_rank)
    rng = np.random.default_rng(5)
    dense = rng.standard_normal((W * B, Dd)).astype(np.float32)
    labels = rng.integers(0, 2, size=W * B).astype(np.float32)
    hub = LoopbackHub(W)
    models = []
    for r in range(W):
        e = ShardedEmbedding(cfg.table_rows, D, cfg.feature_table, max_nnz=nnz_max, max_batch=B,
                             max_recv_nnz=W * nnz_max, device=gpu, stream=torch.cuda.Stream(), rank=r,
                             world_size=W, sharding=sharding, loopback_hub=hub, p2p=True)
        init_tables_host(e, cfg)
        m = FeedModel(e, Dd, lr=0.05, seed=7)
        with torch.no_grad():
            for p in m.params:
                p.mul_(40.0)  # clip active
        models.append(m)
    torch.cuda.synchronize()
    params0 = [p.detach().cpu().double().numpy().copy() for p in models[0].params]

    def step(r):
        m = models[r]
        ids, off = per_rank[r]
        sl = slice(r * B, (r + 1) * B)
        loss = m.train_step(dev(ids), dev(off), B, dev(dense[sl].copy()), dev(labels[sl].copy()))
        torch.cuda.synchronize()
        return float(loss), m.emb.sync()

    res = run_ranks(W, step)
    assert all(st == 0 for _, st in res)
    ids_g, off_g = global_batch(per_rank, F, B)
    Wt = dense_tables(cfg)
    W0 = Wt.copy()
    A = np.full(cfg.total_rows, 0.1, dtype=np.float32)
    params = [p.copy() for p in params0]
    accs = [np.full_like(p, 0.1) for p in params]
    r_or = FM.feed_train_step(problem(cfg), Wt, A, ids_g, off_g, W * B, dense.astype(np.float64),
                              labels.astype(np.float64), params, accs, 0.05, 1e-7, 1.0)
    assert abs(np.mean([l for l, _ in res]) - r_or["loss"]) <= 1e-5 * abs(r_or["loss"])
    assert r_or["c"] < 1.0
    for m in models:
        assert abs(float(m.S) - r_or["S"]) <= 1e-5 * r_or["S"]
        assert abs(float(m.c) - float(r_or["c"])) <= 1e-5 * float(r_or["c"])
    # identical tower replicas, each equal to the oracle's update
    for a, b in zip(models[0].params, models[1].params):
        assert torch.equal(a, b)
    for got, ref, old in zip(models[0].params, params, params0):
        g = got.detach().cpu().double().numpy()
        stp = np.abs(ref - old)
        assert (np.abs(g - ref) <= 1e-3 * stp + 4 * np.spacing(np.abs(ref).astype(np.float32))).all()
    # sparse rows, from their owners
    base = np.concatenate([[0], np.cumsum(cfg.table_rows)])
    for t, R in enumerate(cfg.table_rows):
        for m in models:
            e = m.emb
            lo, hi = int(e.row_lo[t]), int(e.row_hi[t])
            if e.local_base[t] < 0 or hi <= lo:
                continue
            w = e.read_rows(t, np.arange(lo, hi), with_acc=False)
            sl = slice(base[t] + lo, base[t] + hi)
            stp = np.abs(Wt[sl] - W0[sl])
            assert (np.abs(w - Wt[sl]) <= 1e-3 * stp + 4 * np.spacing(np.abs(Wt[sl]))).all()
    for m in models:
        m.emb.close()
    hub.close()
