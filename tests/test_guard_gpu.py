"""Out-of-bounds writes, without compute-sanitizer (closed on this GPU pool): every buffer the
library is given -- tables, accumulators, q8 store, workspace (planned sizes) and the caller's
outputs -- is followed by a guard band, and the inputs (ids, offsets, upstream gradients) must
come back unchanged.  Runs every kernel of the path on small shapes with ragged tails: W = 1
training steps in each mode, the full-table quantize, the serving handle, and the sharded
exchange (loopback W = 2 and 3; collective and fused peer-store modes)."""
import threading

import numpy as np
import pytest

from helpers import init_tables_host
from workload import configs, gen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GUARD = 4096


def guarded(shape, dev):
    """A float32 tensor of `shape` inside a larger buffer whose margins hold a NaN pattern."""
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * 1024,), float("nan"), device=dev)
    return buf, buf[1024:1024 + n].view(*shape)


def margins_ok(buf):
    return bool(torch.isnan(buf[:1024]).all() and torch.isnan(buf[-1024:]).all())


def run_steps(e, batches, B, F, D, dev, q8=True):
    outs = []
    with torch.cuda.stream(e.stream):
        for k, (ids, off) in enumerate(batches):
            ids_d, off_d = torch.from_numpy(ids).to(dev), torch.from_numpy(off).to(dev)
            g = torch.from_numpy(gen.grad_values(7, k, B, F, D, gen.grad_shift_for(len(ids), D))).to(dev)
            ids_c, off_c, g_c = ids_d.clone(), off_d.clone(), g.clone()
            ob, o = guarded((B, F, D), dev)
            e.forward(ids_d, off_d, B, out=o)
            outs.append(ob)
            if q8:
                qb, q = guarded((B, F, D), dev)
                e.forward_q8(ids_d, off_d, B, out=q)
                outs.append(qb)
            e.backward_adagrad(g, 0.05)
            e.stream.synchronize()
            assert torch.equal(ids_d, ids_c) and torch.equal(off_d, off_c) and torch.equal(g, g_c)
    assert e.sync() == 0
    assert all(margins_ok(b) for b in outs)
    assert e.guards_intact()


@pytest.mark.parametrize("kw", [dict(q8=True, requant=True), dict(q8=True, requant=True, q8_mode="min_max"),
                                dict(pooling="mean", adagrad="elementwise", q8=True)])
@pytest.mark.parametrize("dim", [64, 30])
def test_guard_bands_single(gpu, kw, dim):
    from paper_2402_06859_b200 import ShardedEmbedding
    rows = [7001, 333, 5]
    ft = [0, 1, 2, 0]
    cfg = configs.Config("guard", rows, dim, [(t, ("range", 0, 23)) for t in ft], 301, seed=4)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    batches = [gen.make_batch(rows, cfg.features, B, cfg.seed, k) for k in range(2)]
    nnz = max(len(i) for i, _ in batches)
    e = ShardedEmbedding(rows, D, ft, max_nnz=nnz, max_batch=B, device=gpu, stream=torch.cuda.Stream(),
                         guard_bytes=GUARD, **kw)
    init_tables_host(e, cfg)
    e.quantize()
    run_steps(e, batches, B, F, D, gpu)
    e.close()


def test_guard_bands_serving(gpu):
    from paper_2402_06859_b200 import ShardedEmbedding
    rows = [5003, 77]
    ft = [0, 1, 0]
    cfg = configs.Config("guard_s", rows, 64, [(t, ("range", 0, 9)) for t in ft], 97, seed=5)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    ids, off = gen.make_batch(rows, cfg.features, B, cfg.seed, 0)
    e = ShardedEmbedding(rows, D, ft, max_nnz=len(ids), max_batch=B, device=gpu, q8_only=True, guard_bytes=GUARD)
    for t, R in enumerate(rows):
        e.quantize_block(t, 0, torch.from_numpy(gen.table_rows(cfg.seed, t, np.arange(R), D)).to(gpu))
    qb, q = guarded((B, F, D), gpu)
    e.forward_q8(torch.from_numpy(ids).to(gpu), torch.from_numpy(off).to(gpu), B, out=q)
    assert e.sync() == 0 and margins_ok(qb) and e.guards_intact()
    e.close()


@pytest.mark.parametrize("W", [2, 3])
@pytest.mark.parametrize("p2p", [False, True])
@pytest.mark.parametrize("sharding", ["table", "row"])
def test_guard_bands_sharded(gpu, W, p2p, sharding):
    from paper_2402_06859_b200 import LoopbackHub, ShardedEmbedding
    rows = [4001, 900, 31, 2500]
    ft = [0, 1, 2, 3, 0]
    cfg = configs.Config("guard_x", rows, 64, [(t, ("range", 0, 17)) for t in ft], 133, seed=6)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    per_rank = [[gen.make_batch(rows, cfg.features, B, cfg.seed + 10 * r, k) for k in range(2)] for r in range(W)]
    nnz = max(len(i) for bs in per_rank for i, _ in bs)
    hub = LoopbackHub(W)
    embs = [ShardedEmbedding(rows, D, ft, max_nnz=nnz, max_batch=B, max_recv_nnz=W * nnz, device=gpu,
                             stream=torch.cuda.Stream(), rank=r, world_size=W, sharding=sharding,
                             loopback_hub=hub, q8=True, requant=True, p2p=p2p, guard_bytes=GUARD)
            for r in range(W)]
    for e in embs:
        init_tables_host(e, cfg)
        e.quantize()
    torch.cuda.synchronize()
    err = []

    def body(r):
        try:
            run_steps(embs[r], per_rank[r], B, F, D, gpu)
        except Exception as ex:  # surfaced in the main thread
            err.append(ex)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(W)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not err, err
    for e in embs:
        e.close()
    hub.close()
