"""Sharded path (a1/a3/a4) on one GPU through the loopback transport: W ranks
as W threads of this process, each with its own handle and stream, exchanging through the
same exchange code as NCCL (only the transport differs).  Results must equal the unsharded
oracle on the global batch: forward per rank (table-wise bit-exact: each bag is pooled by
one owner in bag order; row-wise within the pooled gate: partial sums from several owners),
dedup/update per owner within the update gates."""
import threading

import numpy as np
import pytest

import oracle as O
from helpers import S_close, cond_close, dense_tables, init_tables_host, w_close
from workload import configs, gen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def run_ranks(W, fn):
    out, err = [None] * W, []

    def body(r):
        try:
            out[r] = fn(r)
        except Exception as e:  # surface in the main thread
            err.append((r, e))

    ts = [threading.Thread(target=body, args=(r,)) for r in range(W)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if err:
        raise err[0][1]
    return out


def global_batch(per_rank, F, B):
    """Concatenate per-rank feature-major batches into one global batch (sample r*B + b)."""
    ids_g, lens = [], []
    for f in range(F):
        for (ids, off) in per_rank:
            o = off.astype(np.int64)
            ids_g.append(ids[o[f * B]:o[(f + 1) * B]])
            lens.append(np.diff(o[f * B:(f + 1) * B + 1]))
    off_g = np.zeros(F * B * len(per_rank) + 1, dtype=np.int64)
    off_g[1:] = np.cumsum(np.concatenate(lens))
    return np.concatenate(ids_g).astype(np.int32), off_g.astype(np.int32)


@pytest.mark.parametrize("p2p", [False, True])
@pytest.mark.parametrize("W", [2, 4, 3])
@pytest.mark.parametrize("sharding", ["table", "row"])
def test_sharded_train_step_matches_unsharded_oracle(gpu, W, sharding, p2p):
    from paper_2402_06859_b200 import LoopbackHub, ShardedEmbedding
    rows = [3000, 1200, 500, 77, 2000]
    ft = [0, 1, 2, 3, 4, 0, 1]  # features 5, 6 share tables 0, 1
    cfg = configs.Config("shard", rows, 32, [(t, ("range", 0, 12)) for t in ft], 64, seed=3)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    per_rank = [gen.make_batch(rows, cfg.features, B, cfg.seed + r, 0) for r in range(W)]
    ids_g, off_g = global_batch(per_rank, F, B)
    gshift = gen.grad_shift_for(len(ids_g), D)
    grad_g = gen.grad_values(cfg.seed, 0, W * B, F, D, gshift)
    hub = LoopbackHub(W)
    embs = []
    for r in range(W):
        s = torch.cuda.Stream()
        e = ShardedEmbedding(rows, D, ft, max_nnz=max(len(i) for i, _ in per_rank), max_batch=B,
                             max_recv_nnz=W * max(len(i) for i, _ in per_rank),
                             device=torch.device("cuda:0"), stream=s, rank=r, world_size=W,
                             sharding=sharding, loopback_hub=hub, p2p=p2p)
        init_tables_host(e, cfg)
        embs.append(e)
    torch.cuda.synchronize()

    def step(r):
        e = embs[r]
        ids, off = per_rank[r]
        with torch.cuda.stream(e.stream):
            out = e.forward(torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda(), B)
            g = torch.from_numpy(grad_g[r * B:(r + 1) * B].copy()).cuda()
            e.backward_adagrad(g, 0.05)
        st = e.sync()
        return out.cpu().numpy(), st

    res = run_ranks(W, step)
    assert all(st == 0 for _, st in res)
    pb = O.Problem(rows, D, ft)
    W0 = dense_tables(cfg)
    Wo = W0.copy()
    A = np.full(cfg.total_rows, 0.1, dtype=np.float32)
    r_or = O.train_step(pb, Wo, A, ids_g, off_g, W * B, grad_g, 0.05, 1e-7, 1.0)
    mag, _ = O.forward(pb, np.abs(W0), ids_g, off_g, W * B)
    for r in range(W):
        got = res[r][0]
        ref = r_or["out"][r * B:(r + 1) * B]
        assert cond_close(got, ref, mag[r * B:(r + 1) * B]).all()
        if sharding == "table":
            assert (got == ref).all()
    # global norm identical on every rank (rank partials summed in rank order)
    Ss = [e.last_stats()[0] for e in embs]
    assert all(S == Ss[0] for S in Ss)
    assert S_close(Ss[0], r_or["S"])
    assert sum(e.last_stats()[2] for e in embs) == r_or["U"]
    # every row from its owner
    base = np.concatenate([[0], np.cumsum(rows)])
    keys, segs, bags = O.dedup(pb, ids_g, off_g, W * B)
    G = O.segment_reduce(pb, off_g, W * B, segs, bags, grad_g)
    g = O.clip(G, r_or["c"])
    step = np.zeros_like(W0)
    step[keys] = np.abs(0.05 / (np.sqrt(np.full(len(keys), 0.1, np.float32) + 0.0) + 1e-7))[:, None] * np.abs(g)
    for t, R in enumerate(rows):
        for e in embs:
            lo, hi = int(e.row_lo[t]), int(e.row_hi[t])
            if e.local_base[t] < 0 or hi <= lo:
                continue
            w, a = e.read_rows(t, np.arange(lo, hi))
            sl = slice(base[t] + lo, base[t] + hi)
            assert (np.abs(a - A[sl]) <= 1e-6 * A[sl]).all()
            assert w_close(w, Wo[sl], W0[sl], np.maximum(step[sl], np.abs(Wo[sl] - W0[sl]))).all()
    for e in embs:
        e.close()
    hub.close()


@pytest.mark.parametrize("kind", ["inf", "nan"])
@pytest.mark.parametrize("sharding", ["table", "row"])
def test_sharded_nonfinite_grad_skips_update_on_every_rank(gpu, sharding, kind):
    """An Inf / NaN in one rank's upstream gradient: the owner's a6 (ALU widening) flags it and
    re-runs with the hardware conversions, so its norm partial is the oracle's class; the
    rank-ordered global S is then Inf (NaN) on EVERY rank, every rank reports EMB_ENONFINITE
    and no rank updates a row (P:17's clip has no finite factor)."""
    from paper_2402_06859_b200 import LoopbackHub, ShardedEmbedding
    from paper_2402_06859_b200._lib import EMB_ENONFINITE
    W = 2
    rows = [1500, 600, 90]
    ft = [0, 1, 2, 0]
    cfg = configs.Config("shnf", rows, 32, [(t, ("range", 1, 10)) for t in ft], 40, seed=12)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    per_rank = [gen.make_batch(rows, cfg.features, B, cfg.seed + r, 0) for r in range(W)]
    ids_g, off_g = global_batch(per_rank, F, B)
    grad_g = gen.grad_values(cfg.seed, 0, W * B, F, D, gen.grad_shift_for(len(ids_g), D))
    grad_g[B + 3, 1, 7] = np.inf if kind == "inf" else np.nan  # rank 1's sample 3
    hub = LoopbackHub(W)
    embs = []
    for r in range(W):
        e = ShardedEmbedding(rows, D, ft, max_nnz=max(len(i) for i, _ in per_rank), max_batch=B,
                             max_recv_nnz=W * max(len(i) for i, _ in per_rank),
                             device=torch.device("cuda:0"), stream=torch.cuda.Stream(), rank=r, world_size=W,
                             sharding=sharding, loopback_hub=hub)
        init_tables_host(e, cfg)
        embs.append(e)
    torch.cuda.synchronize()
    w0 = [e.weights.clone() for e in embs]

    def step(r):
        e = embs[r]
        ids, off = per_rank[r]
        with torch.cuda.stream(e.stream):
            e.forward(torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda(), B)
            e.backward_adagrad(torch.from_numpy(grad_g[r * B:(r + 1) * B].copy()).cuda(), 0.05)
        return e.sync()

    assert all(st == EMB_ENONFINITE for st in run_ranks(W, step))
    for e, w in zip(embs, w0):
        assert torch.equal(e.weights, w)
    pb = O.Problem(rows, D, ft)
    r_or = O.train_step(pb, dense_tables(cfg), np.full(cfg.total_rows, 0.1, dtype=np.float32), ids_g, off_g,
                        W * B, grad_g, 0.05, 1e-7, 1.0)
    for e in embs:
        S = e.last_stats()[0]
        assert (np.isnan(S) and np.isnan(r_or["S"])) if kind == "nan" else (S == np.inf and r_or["S"] == np.inf)
    for e in embs:
        e.close()
    hub.close()


@pytest.mark.parametrize("p2p", [False, True])
@pytest.mark.parametrize("sharding", ["table", "row"])
def test_sharded_q8_forward(gpu, sharding, p2p):
    from paper_2402_06859_b200 import LoopbackHub, ShardedEmbedding
    W = 2
    rows = [2000, 900, 300]
    ft = [0, 1, 2, 1]
    cfg = configs.Config("shq8", rows, 64, [(t, ("range", 1, 9)) for t in ft], 48, seed=8)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    per_rank = [gen.make_batch(rows, cfg.features, B, cfg.seed + r, 0) for r in range(W)]
    hub = LoopbackHub(W)
    embs = []
    for r in range(W):
        e = ShardedEmbedding(rows, D, ft, max_nnz=max(len(i) for i, _ in per_rank), max_batch=B,
                             max_recv_nnz=W * max(len(i) for i, _ in per_rank),
                             device=torch.device("cuda:0"), stream=torch.cuda.Stream(), rank=r,
                             world_size=W, sharding=sharding, q8=True, loopback_hub=hub, p2p=p2p)
        init_tables_host(e, cfg)
        e.quantize()
        embs.append(e)
    torch.cuda.synchronize()

    def fwd(r):
        e = embs[r]
        ids, off = per_rank[r]
        with torch.cuda.stream(e.stream):
            out = e.forward_q8(torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda(), B)
        assert e.sync() == 0
        return out.cpu().numpy()

    outs = run_ranks(W, fwd)

    def fwd_reuse(r):  # forward, then the q8 lookup of ITS batch (ids exchange skipped), twice
        e = embs[r]
        ids, off = per_rank[r]
        with torch.cuda.stream(e.stream):
            e.forward(torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda(), B)
            q1 = torch.empty((B, F, D), device="cuda")
            q2 = torch.empty((B, F, D), device="cuda")
            e.forward_q8(None, None, B, out=q1, nnz=len(ids))
            e.forward_q8(None, None, B, out=q2, nnz=len(ids))
        assert e.sync() == 0
        return q1.cpu().numpy(), q2.cpu().numpy()

    for r, (q1, q2) in enumerate(run_ranks(W, fwd_reuse)):
        assert (q1 == outs[r]).all() and (q2 == outs[r]).all()

    # alternate batches: each step's fp32 forward and its q8 reuse use the two destination sets of
    # the fused exchange in turn; every q8 output must equal the fresh lookup of its batch
    other = [gen.make_batch(rows, cfg.features, B, cfg.seed + 100 + r, 1) for r in range(W)]

    def alternate(r):
        e = embs[r]
        res = []
        for k in range(4):
            ids, off = (per_rank if k % 2 == 0 else other)[r]
            with torch.cuda.stream(e.stream):
                e.forward(torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda(), B)
                q = torch.empty((B, F, D), device="cuda")
                e.forward_q8(None, None, B, out=q, nnz=len(ids))
                fresh = e.forward_q8(torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda(), B)
            assert e.sync() == 0
            res.append((q.cpu().numpy(), fresh.cpu().numpy()))
        return res

    for r, res in enumerate(run_ranks(W, alternate)):
        for k, (q, fresh) in enumerate(res):
            assert (q == fresh).all(), (r, k)
    W0 = dense_tables(cfg)
    codes, mid, sc, _ = O.quantize(W0)
    pb = O.Problem(rows, D, ft)
    deq = np.abs(mid.astype(np.float64))[:, None] + np.abs(codes.astype(np.float64) * sc[:, None])
    for r in range(W):
        ref, _ = O.forward_q8(pb, codes, mid, sc, per_rank[r][0], per_rank[r][1], B)
        mag, _ = O.forward(pb, deq.astype(np.float32), per_rank[r][0], per_rank[r][1], B)
        assert cond_close(outs[r], ref, mag).all()
        if sharding == "table":
            assert (outs[r] == ref).all()
    hub.close()


@pytest.mark.parametrize("p2p", [False, True])
@pytest.mark.parametrize("sharding", ["table", "row"])
def test_nccl_transport_single_rank(gpu, sharding, p2p):
    """The NCCL transport (torch's libnccl, dlopen'ed) on a 1-rank communicator: the whole
    exchange path runs (send/recv to self, all-gather, reduce-scatter) and must reproduce
    the unsharded handle bit for bit (with one rank the owner sees occurrences in the
    unsharded order)."""
    from paper_2402_06859_b200 import ShardedEmbedding, nccl_unique_id
    rows = [3000, 700, 90]
    ft = [0, 1, 2, 0]
    cfg = configs.Config("nccl1", rows, 64, [(t, ("range", 0, 12)) for t in ft], 128, seed=5)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    ids, off = gen.make_batch(rows, cfg.features, B, cfg.seed, 0)
    grad = torch.from_numpy(gen.grad_values(cfg.seed, 0, B, F, D, gen.grad_shift_for(len(ids), D))).cuda()
    uid = nccl_unique_id()
    assert len(uid) == 128
    ex = ShardedEmbedding(rows, D, ft, max_nnz=len(ids), max_batch=B, device=torch.device("cuda:0"),
                          rank=0, world_size=1, sharding=sharding, nccl_unique_id=uid, force_exchange=True,
                          q8=True, p2p=p2p)
    ref = ShardedEmbedding(rows, D, ft, max_nnz=len(ids), max_batch=B, device=torch.device("cuda:0"), q8=True)
    for e in (ex, ref):
        init_tables_host(e, cfg)
    outs = []
    for e in (ex, ref):
        o = e.forward(torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda(), B)
        e.backward_adagrad(grad, 0.05)
        e.quantize()
        q = e.forward_q8(torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda(), B)
        assert e.sync() == 0
        outs.append((o.cpu().numpy(), q.cpu().numpy()))
    assert (outs[0][0] == outs[1][0]).all() and (outs[0][1] == outs[1][1]).all()
    assert torch.equal(ex.weights, ref.weights) and torch.equal(ex.accum_buf[:4 * sum(rows)], ref.accum_buf[:4 * sum(rows)])
    assert ex.last_stats()[0] == ref.last_stats()[0]
    ex.close()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("sharding", ["table", "row"])
def test_exchange_q8_forward_while_dedup_runs(gpu, sharding):
    """Regression: forward -> forward_q8 -> backward on the exchange path at a size where the
    a5 dedup (side stream) is still running when forward_q8's exchange scans start.  The
    scans have their own look-back words (they used to share the radix sort's and could
    wait forever on a word the sort overwrote)."""
    from paper_2402_06859_b200 import ShardedEmbedding, nccl_unique_id
    rows = [400_000, 20_000]
    ft = [0, 1, 0]
    cfg = configs.Config("ex_mid", rows, 64, [(t, ("range", 1, 60)) for t in ft], 8192, seed=21)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    ids, off = gen.make_batch(rows, cfg.features, B, cfg.seed, 0)
    grad = torch.from_numpy(gen.grad_values(cfg.seed, 0, B, F, D, gen.grad_shift_for(len(ids), D))).cuda()
    ex = ShardedEmbedding(rows, D, ft, max_nnz=len(ids), max_batch=B, device=torch.device("cuda:0"), rank=0,
                          world_size=1, sharding=sharding, nccl_unique_id=nccl_unique_id(), force_exchange=True,
                          q8=True, max_recv_nnz=len(ids))
    ref = ShardedEmbedding(rows, D, ft, max_nnz=len(ids), max_batch=B, device=torch.device("cuda:0"), q8=True)
    ids_d, off_d = torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda()
    res = []
    for e in (ex, ref):
        init_tables_host(e, cfg)
        e.quantize()
        for _ in range(3):
            o = e.forward(ids_d, off_d, B)
            q = e.forward_q8(ids_d, off_d, B)
            e.backward_adagrad(grad, 0.05)
        assert e.sync() == 0
        res.append((o.cpu().numpy(), q.cpu().numpy()))
    assert (res[0][0] == res[1][0]).all() and (res[0][1] == res[1][1]).all()
    assert torch.equal(ex.weights, ref.weights)


@pytest.mark.parametrize("W", [2, 3])
@pytest.mark.parametrize("sharding", ["table", "row"])
def test_p2p_exchange_matches_collective_exchange(gpu, W, sharding):
    """EMB_F_P2P (pooled rows stored straight into the destination rank's buffer, grad rows
    pushed into the owners' buffers, stream-ordered barriers) against the collective exchange
    on the same ranks: three back-to-back steps of forward -> forward_q8 -> backward (buffer
    reuse across steps) must agree bit for bit -- the row-wise slots are summed in rank order,
    as the reduce-scatter does."""
    from paper_2402_06859_b200 import LoopbackHub, ShardedEmbedding
    rows = [5000, 1500, 600, 64]
    ft = [0, 1, 2, 3, 0, 2]
    cfg = configs.Config("p2p", rows, 64, [(t, ("range", 0, 14)) for t in ft], 96, seed=31)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    nsteps = 3
    batches = [[gen.make_batch(rows, cfg.features, B, cfg.seed + 100 * k + r, 0) for r in range(W)]
               for k in range(nsteps)]
    nnz_max = max(len(i) for bk in batches for i, _ in bk)
    grads = [gen.grad_values(cfg.seed, k, W * B, F, D, gen.grad_shift_for(nnz_max * W, D)) for k in range(nsteps)]
    results = {}
    for p2p in (False, True):
        hub = LoopbackHub(W)
        embs = []
        for r in range(W):
            e = ShardedEmbedding(rows, D, ft, max_nnz=nnz_max, max_batch=B, max_recv_nnz=W * nnz_max,
                                 device=torch.device("cuda:0"), stream=torch.cuda.Stream(), rank=r,
                                 world_size=W, sharding=sharding, q8=True, requant=True, loopback_hub=hub,
                                 p2p=p2p)
            init_tables_host(e, cfg)
            e.quantize()
            embs.append(e)
        torch.cuda.synchronize()

        def run(r):
            e = embs[r]
            outs = []
            with torch.cuda.stream(e.stream):
                for k in range(nsteps):
                    ids, off = batches[k][r]
                    ids_d, off_d = torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda()
                    o = e.forward(ids_d, off_d, B)
                    q = e.forward_q8(ids_d, off_d, B)
                    e.backward_adagrad(torch.from_numpy(grads[k][r * B:(r + 1) * B].copy()).cuda(), 0.05)
                    outs.append((o.clone(), q.clone()))
            assert e.sync() == 0
            return [(o.cpu().numpy(), q.cpu().numpy()) for o, q in outs], e.weights.cpu().numpy().copy(), \
                e.last_stats()[0]

        results[p2p] = run_ranks(W, run)
        for e in embs:
            e.close()
        hub.close()
    for r in range(W):
        (o_c, w_c, s_c), (o_p, w_p, s_p) = results[False][r], results[True][r]
        for (a1, b1), (a2, b2) in zip(o_c, o_p):
            assert np.array_equal(a1, a2) and np.array_equal(b1, b2)
        assert np.array_equal(w_c, w_p)
        assert s_c == s_p
