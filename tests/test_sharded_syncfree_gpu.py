"""The sharded step without host synchronisation (PAPER.md:576 exchange; SURVEY.md §7
"variable-size all-to-all without a host sync"), through the loopback transport (W ranks as
W threads of this process on one GPU; no kernel ever waits on another rank's kernel):

1. a W = 2 step (forward -> q8 forward -> backward, fused and collective exchange, table-
   and row-wise) captured ONCE as a single CUDA graph spanning both ranks' streams replays
   bit-identically to eager execution -- the received id count never reaches the host;
2. a received-id overflow of the planned capacity is discarded on EVERY rank (zero outputs,
   no update) with sticky EMB_ENOMEM;
3. table-wise collective backward after a q8 forward of a DIFFERENT batch size scatters the
   gradient rows with the forward's B (the permute map is scaled by B on the device).
"""
import numpy as np
import pytest

import oracle as O
from helpers import cond_close, dense_tables, init_tables_host, w_close
from test_sharded_gpu import global_batch, run_ranks
from workload import configs, gen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _make(W, cfg, ft, nnz_max, sharding, p2p, B):
    from paper_2402_06859_b200 import LoopbackHub, ShardedEmbedding
    hub = LoopbackHub(W)
    embs = []
    for r in range(W):
        e = ShardedEmbedding(cfg.table_rows, cfg.dim, ft, max_nnz=nnz_max, max_batch=B,
                             max_recv_nnz=W * nnz_max, device=torch.device("cuda:0"), stream=torch.cuda.Stream(), rank=r, world_size=W,
                             sharding=sharding, loopback_hub=hub, p2p=p2p, q8=True, requant=True)
        init_tables_host(e, cfg)
        e.quantize()
        embs.append(e)
    torch.cuda.synchronize()
    return hub, embs


@pytest.mark.parametrize("p2p", [True, False])
@pytest.mark.parametrize("sharding", ["row", "table"])
def test_w2_step_graph_capture_replays_like_eager(gpu, sharding, p2p):
    W = 2
    rows = [6000, 1500, 300]
    ft = [0, 1, 2, 0, 1]
    cfg = configs.Config("g2", rows, 64, [(t, ("range", 0, 16)) for t in ft], 128, seed=41)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    nb = 3
    batches = [[gen.make_batch(rows, cfg.features, B, cfg.seed + 10 * k + r, 0) for r in range(W)]
               for k in range(nb)]
    nnz_max = max(len(i) for bk in batches for i, _ in bk)
    gshift = gen.grad_shift_for(W * nnz_max, D)
    dev_in = [[(torch.from_numpy(batches[k][r][0]).cuda(), torch.from_numpy(batches[k][r][1]).cuda(),
                torch.from_numpy(gen.grad_values(cfg.seed, k, W * B, F, D, gshift)[r * B:(r + 1) * B].copy()).cuda())
               for r in range(W)] for k in range(nb)]
    runs = {}
    for mode in ("eager", "graph"):
        hub, embs = _make(W, cfg, ft, nnz_max, sharding, p2p, B)
        # fixed input slots (a graph replays on fixed addresses): copy batch k in before a step
        slots = [(torch.zeros(nnz_max, dtype=torch.int32, device=gpu), torch.zeros(F * B + 1, dtype=torch.int32, device=gpu),
                  torch.zeros((B, F, D), device=gpu)) for _ in range(W)]
        outs = [(torch.zeros((B, F, D), device=gpu), torch.zeros((B, F, D), device=gpu)) for _ in range(W)]
        nnz_of = [[len(batches[k][r][0]) for r in range(W)] for k in range(nb)]

        def load(k):
            for r in range(W):
                i, o, g = dev_in[k][r]
                slots[r][0][: i.numel()].copy_(i)
                slots[r][1].copy_(o)
                slots[r][2].copy_(g)
            torch.cuda.synchronize()

        def step(r, k):
            e = embs[r]
            n = nnz_of[k][r]
            e.forward(slots[r][0][:n], slots[r][1], B, out=outs[r][0])
            e.forward_q8(slots[r][0][:n], slots[r][1], B, out=outs[r][1])
            e.backward_adagrad(slots[r][2], 0.05)

        # warm-up step on batch 0 (lazy module loading, peer mappings: host-side, not capturable)
        load(0)
        run_ranks(W, lambda r: step(r, 0))
        torch.cuda.synchronize()
        order = [1, 2, 1]
        res = []
        if mode == "eager":
            for k in order:
                load(k)
                run_ranks(W, lambda r: step(r, k))
                torch.cuda.synchronize()
                res.append([(o[0].cpu().clone(), o[1].cpu().clone()) for o in outs])
        else:
            # one graph per batch (a graph bakes in the per-rank id counts of its batch);
            # capturing executes nothing, so the tables stay in the warm-up state
            graphs = {}
            for k in (1, 2):
                load(k)
                g = torch.cuda.CUDAGraph()
                s0 = embs[0].stream
                with torch.cuda.graph(g, stream=s0, capture_error_mode="relaxed"):
                    fork = torch.cuda.Event()
                    fork.record(s0)
                    for e in embs[1:]:
                        e.stream.wait_event(fork)
                    run_ranks(W, lambda r: step(r, k))
                    for e in embs[1:]:
                        j = torch.cuda.Event()
                        j.record(e.stream)
                        s0.wait_event(j)
                graphs[k] = g
                torch.cuda.synchronize()
            for k in order:
                load(k)
                graphs[k].replay()
                torch.cuda.synchronize()
                res.append([(o[0].cpu().clone(), o[1].cpu().clone()) for o in outs])
        for e in embs:
            assert e.sync() == 0
        runs[mode] = (res, [e.weights.cpu().clone() for e in embs], [e.accum_buf.cpu().clone() for e in embs],
                      [e.codes_buf.cpu().clone() for e in embs], [e.last_stats()[0] for e in embs])
        for e in embs:
            e.close()
        hub.close()
    (re, we, ae, ce, se), (rg, wg, ag, cg, sg) = runs["eager"], runs["graph"]
    for a, b in zip(re, rg):
        for (x1, y1), (x2, y2) in zip(a, b):
            assert torch.equal(x1, x2) and torch.equal(y1, y2)
    for r in range(W):
        assert torch.equal(we[r], wg[r]) and torch.equal(ae[r], ag[r]) and torch.equal(ce[r], cg[r])
        assert se[r] == sg[r]


@pytest.mark.parametrize("p2p", [True, False])
@pytest.mark.parametrize("sharding", ["row", "table"])
def test_overflow_is_discarded_on_every_rank(gpu, sharding, p2p):
    from paper_2402_06859_b200 import _lib as L
    W = 2
    rows = [4000, 900]
    ft = [0, 1, 0]
    cfg = configs.Config("ovf", rows, 32, [(t, ("range", 2, 12)) for t in ft], 64, seed=43)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    per_rank = [gen.make_batch(rows, cfg.features, B, cfg.seed + r, 0) for r in range(W)]
    nnz_max = max(len(i) for i, _ in per_rank)
    # capacity: far below what one owner receives (each rank gets about half of all ids)
    from paper_2402_06859_b200 import LoopbackHub, ShardedEmbedding
    hub = LoopbackHub(W)
    embs = [ShardedEmbedding(rows, D, ft, max_nnz=nnz_max, max_batch=B, max_recv_nnz=nnz_max // 4,
                             device=gpu, stream=torch.cuda.Stream(), rank=r, world_size=W, sharding=sharding,
                             loopback_hub=hub, p2p=p2p) for r in range(W)]
    for e in embs:
        init_tables_host(e, cfg)
    torch.cuda.synchronize()
    w_before = [e.weights.cpu().clone() for e in embs]
    grad = gen.grad_values(cfg.seed, 0, W * B, F, D, gen.grad_shift_for(2 * nnz_max, D))

    def step(r):
        e = embs[r]
        ids, off = per_rank[r]
        with torch.cuda.stream(e.stream):
            out = torch.full((B, F, D), 7.0, device=gpu)
            e.forward(torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda(), B, out=out)
            e.backward_adagrad(torch.from_numpy(grad[r * B:(r + 1) * B].copy()).cuda(), 0.05)
        return out.cpu().numpy(), e.sync()

    res = run_ranks(W, step)
    for r in range(W):
        out, st = res[r]
        assert st == L.EMB_ENOMEM
        assert (out == 0).all()
        assert torch.equal(embs[r].weights.cpu(), w_before[r])  # no occurrence -> no update
    for e in embs:
        e.close()
    hub.close()


def test_table_wise_backward_uses_forward_batch_after_q8_of_other_batch(gpu):
    """the table-wise collective backward must place gradient rows by the batch
    of the forward it belongs to, even when a q8 forward of another batch size ran in
    between (the permute map is B-independent; k_permute scales it by B on the device)."""
    from paper_2402_06859_b200 import LoopbackHub, ShardedEmbedding
    W = 2
    rows = [3000, 1200, 500, 77]
    ft = [0, 1, 2, 3, 1]
    cfg = configs.Config("fmap", rows, 32, [(t, ("range", 0, 9)) for t in ft], 64, seed=47)
    B, B2, F, D = 64, 24, cfg.num_features, cfg.dim
    per_rank = [gen.make_batch(rows, cfg.features, B, cfg.seed + r, 0) for r in range(W)]
    small = [gen.make_batch(rows, cfg.features, B2, cfg.seed + 7 + r, 0) for r in range(W)]
    ids_g, off_g = global_batch(per_rank, F, B)
    grad_g = gen.grad_values(cfg.seed, 0, W * B, F, D, gen.grad_shift_for(len(ids_g), D))
    nnz_max = max(len(i) for i, _ in per_rank + small)
    hub = LoopbackHub(W)
    embs = [ShardedEmbedding(rows, D, ft, max_nnz=nnz_max, max_batch=B, max_recv_nnz=W * nnz_max, device=gpu,
                             stream=torch.cuda.Stream(), rank=r, world_size=W, sharding="table",
                             loopback_hub=hub, q8=True) for r in range(W)]
    for e in embs:
        init_tables_host(e, cfg)
        e.quantize()
    torch.cuda.synchronize()

    def step(r):
        e = embs[r]
        with torch.cuda.stream(e.stream):
            ids, off = per_rank[r]
            out = e.forward(torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda(), B)
            i2, o2 = small[r]
            e.forward_q8(torch.from_numpy(i2).cuda(), torch.from_numpy(o2).cuda(), B2)
            e.backward_adagrad(torch.from_numpy(grad_g[r * B:(r + 1) * B].copy()).cuda(), 0.05)
        return out.cpu().numpy(), e.sync()

    res = run_ranks(W, step)
    assert all(st == 0 for _, st in res)
    pb = O.Problem(rows, D, ft)
    W0 = dense_tables(cfg)
    Wo = W0.copy()
    A = np.full(cfg.total_rows, 0.1, dtype=np.float32)
    r_or = O.train_step(pb, Wo, A, ids_g, off_g, W * B, grad_g, 0.05, 1e-7, 1.0)
    for r in range(W):
        assert (res[r][0] == r_or["out"][r * B:(r + 1) * B]).all()
    base = np.concatenate([[0], np.cumsum(rows)])
    for t, R in enumerate(rows):
        for e in embs:
            if e.local_base[t] < 0:
                continue
            w, a = e.read_rows(t, np.arange(R))
            sl = slice(base[t], base[t] + R)
            assert (np.abs(a - A[sl]) <= 1e-6 * A[sl]).all()
            assert w_close(w, Wo[sl], W0[sl], np.abs(Wo[sl] - W0[sl])).all()
    for e in embs:
        e.close()
    hub.close()


@pytest.mark.parametrize("p2p", [True, False])
@pytest.mark.parametrize("sharding", ["row", "table"])
def test_sharded_empty_and_all_invalid_batches(gpu, sharding, p2p):
    """Degenerate sharded calls: a batch with no ids at all, and one whose ids are all out of
    range, on every rank -- zero outputs, no update, the id-range error only for the latter;
    then a normal step still matches the oracle (the device-resident count went to 0 and back)."""
    from paper_2402_06859_b200 import LoopbackHub, ShardedEmbedding
    from paper_2402_06859_b200._lib import EMB_EIDRANGE
    W = 2
    rows = [900, 300]
    ft = [0, 1, 0]
    cfg = configs.Config("deg", rows, 32, [(t, ("range", 0, 6)) for t in ft], 16, seed=71)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    per_rank = [gen.make_batch(rows, cfg.features, B, cfg.seed + r, 0) for r in range(W)]
    nnz_max = max(max(len(i) for i, _ in per_rank), 8)
    hub = LoopbackHub(W)
    embs = [ShardedEmbedding(rows, D, ft, max_nnz=nnz_max, max_batch=B, max_recv_nnz=W * nnz_max, device=gpu,
                             stream=torch.cuda.Stream(), rank=r, world_size=W, sharding=sharding,
                             loopback_hub=hub, p2p=p2p) for r in range(W)]
    for e in embs:
        init_tables_host(e, cfg)
    torch.cuda.synchronize()
    w0 = [e.weights.cpu().clone() for e in embs]
    empty_off = torch.zeros(F * B + 1, dtype=torch.int32, device=gpu)
    bad_ids = torch.full((8,), 10 ** 6, dtype=torch.int32, device=gpu)
    bad_off = torch.tensor([0] * (F * B) + [8], dtype=torch.int32, device=gpu)
    g = torch.ones((B, F, D), device=gpu)

    def step(r, ids, off):
        e = embs[r]
        with torch.cuda.stream(e.stream):
            out = torch.full((B, F, D), 3.0, device=gpu)
            e.forward(ids, off, B, out=out)
            e.backward_adagrad(g, 0.05)
        return out.cpu().numpy(), e.sync()

    res = run_ranks(W, lambda r: step(r, torch.zeros(0, dtype=torch.int32, device=gpu), empty_off))
    assert all(st == 0 and (o == 0).all() for o, st in res)
    res = run_ranks(W, lambda r: step(r, bad_ids, bad_off))
    assert all(st == EMB_EIDRANGE and (o == 0).all() for o, st in res)
    for e, w in zip(embs, w0):
        assert torch.equal(e.weights.cpu(), w)
    # a normal step afterwards
    ids_g, off_g = global_batch(per_rank, F, B)
    grad_g = gen.grad_values(cfg.seed, 0, W * B, F, D, gen.grad_shift_for(len(ids_g), D))
    res = run_ranks(W, lambda r: _normal(embs[r], per_rank[r], grad_g[r * B:(r + 1) * B], B))
    pb = O.Problem(rows, D, ft)
    Wo = dense_tables(cfg)
    A = np.full(cfg.total_rows, 0.1, dtype=np.float32)
    r_or = O.train_step(pb, Wo, A, ids_g, off_g, W * B, grad_g, 0.05, 1e-7, 1.0)
    mag, _ = O.forward(pb, np.abs(dense_tables(cfg)), ids_g, off_g, W * B)
    for r in range(W):
        out, st = res[r]
        assert st == 0
        assert cond_close(out, r_or["out"][r * B:(r + 1) * B], mag[r * B:(r + 1) * B]).all()
    for e in embs:
        e.close()
    hub.close()


def _normal(e, batch, grad, B):
    ids, off = batch
    with torch.cuda.stream(e.stream):
        out = e.forward(torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda(), B)
        e.backward_adagrad(torch.from_numpy(grad.copy()).cuda(), 0.05)
    return out.cpu().numpy(), e.sync()


def test_allreduce_f32_is_the_rank_ordered_sum(gpu):
    """emb_allreduce_f32 (NEXT-2's data-parallel dense side) over the loopback transport: every
    rank ends with the same fp32 vector, the sum over ranks in rank order."""
    from paper_2402_06859_b200 import LoopbackHub, ShardedEmbedding
    W = 3
    hub = LoopbackHub(W)
    embs = [ShardedEmbedding([100, 50], 8, [0, 1], max_nnz=16, max_batch=4, device=gpu, stream=torch.cuda.Stream(),
                             rank=r, world_size=W, sharding="row", loopback_hub=hub) for r in range(W)]
    rng = np.random.default_rng(9)
    vals = [rng.standard_normal(100_003).astype(np.float32) for _ in range(W)]

    def body(r):
        t = torch.from_numpy(vals[r]).to(gpu)
        with torch.cuda.stream(embs[r].stream):
            embs[r].allreduce_(t)
        embs[r].stream.synchronize()
        return t.cpu().numpy()

    res = run_ranks(W, body)
    ref = vals[0].copy()
    for r in range(1, W):
        ref = (ref + vals[r]).astype(np.float32)
    for r in range(W):
        assert np.array_equal(res[r], ref)
    for e in embs:
        e.close()
    hub.close()
