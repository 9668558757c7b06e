#!/usr/bin/env python
"""Every kernel of the library on the tiny config, for compute-sanitizer:

    compute-sanitizer --tool memcheck|racecheck|initcheck|synccheck python tools/sanitize_step.py

W = 1 training steps (a2, a10, a5-a8, a9 fused requant, MEAN pooling, element-wise AdaGrad),
the full-table quantize (middle-max and min-max), the FIM penalty + cold-weight init, the
MurmurHash / QR expansion, the serving handle, and the sharded exchange through the loopback
transport (W = 2, table- and row-wise, collective and fused peer-store modes).  Exits 0 when
every call returned EMB_OK and the sticky status is clean."""
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2402_06859_b200 import LoopbackHub, ShardedEmbedding, qr  # noqa: E402
from workload import configs, gen  # noqa: E402
from workload import gpu as G  # noqa: E402

dev = torch.device("cuda:0")
cfg = configs.CONFIGS["tiny"]()
rows, D, ft, B, F = cfg.table_rows, cfg.dim, cfg.feature_table, cfg.batch, cfg.num_features
batches = [gen.make_batch(rows, cfg.features, B, cfg.seed, k) for k in range(2)]
nnz = max(len(i) for i, _ in batches)
gshift = gen.grad_shift_for(nnz, D)


def fill(e):
    s = e.stream
    for t in range(len(rows)):
        v = e.table_view(t)
        if v.shape[0]:
            G.fill_table(v, v.shape[0], D, e.pitch, cfg.seed, t, row0=int(e.row_lo[t]), stream=s)


def steps(e, k0=0, q8=True):
    with torch.cuda.stream(e.stream):
        for k in range(2):
            ids, off = batches[(k0 + k) % 2]
            ids_d, off_d = torch.from_numpy(ids).to(dev), torch.from_numpy(off).to(dev)
            g = torch.empty((B, F, D), device=dev)
            G.fill_grad(g, B, F, D, cfg.seed, k, gshift, stream=e.stream)
            e.forward(ids_d, off_d, B)
            if q8:
                e.forward_q8(ids_d, off_d, B)
            e.backward_adagrad(g, 0.05)
    e.stream.synchronize()
    assert e.sync() == 0


# ---- W = 1 ---------------------------------------------------------------------------
for kw in (dict(q8=True, requant=True), dict(q8=True, requant=True, q8_mode="min_max"),
           dict(pooling="mean", adagrad="elementwise", q8=True)):
    e = ShardedEmbedding(rows, D, ft, max_nnz=nnz, max_batch=B, device=dev, stream=torch.cuda.Stream(), **kw)
    fill(e)
    e.quantize()
    steps(e)
    e.close()

# incremental training (FIM penalty, cold-weight init)
e = ShardedEmbedding(rows, D, ft, max_nnz=nnz, max_batch=B, device=dev, stream=torch.cuda.Stream())
fill(e)
n = e.local_rows * e.pitch
w0 = e.weights.reshape(-1).clone()
H = torch.full((n,), 0.5, device=dev)
e.set_incremental(w0, H, w0.clone(), H, 1e-3, 0.5)
steps(e, q8=False)
e.cold_weight_init(w0, w0.clone(), 0.25)
e.stream.synchronize()
e.close()

# serving handle
s = ShardedEmbedding(rows, D, ft, max_nnz=nnz, max_batch=B, device=dev, q8_only=True)
for t in range(len(rows)):
    blk = torch.from_numpy(gen.table_rows(cfg.seed, t, np.arange(rows[t]), D)).to(dev)
    s.quantize_block(t, 0, blk)
ids, off = batches[0]
s.forward_q8(torch.from_numpy(ids).to(dev), torch.from_numpy(off).to(dev), B)
torch.cuda.synchronize()
assert s.sync() == 0
s.close()

# MurmurHash3 + QR expansion
data, soff = qr.pack_strings([f"member:{i}" for i in range(1000)] + [""], dev)
h = qr.hash_ids(data, soff)
offs = torch.arange(0, 1002, 2, dtype=torch.int32, device=dev).clamp(max=1001)
qr.qr_expand(h, offs, 1000, (1 << 32) // 1000 + 1, True)
torch.cuda.synchronize()

# ---- sharded exchange, W = 2 loopback --------------------------------------------------
for sharding in ("table", "row"):
    for p2p in (False, True):
        hub = LoopbackHub(2)
        embs = [ShardedEmbedding(rows, D, ft, max_nnz=nnz, max_batch=B, max_recv_nnz=2 * nnz, device=dev,
                                 stream=torch.cuda.Stream(), rank=r, world_size=2, sharding=sharding,
                                 loopback_hub=hub, q8=True, requant=True, p2p=p2p) for r in range(2)]
        for e in embs:
            fill(e)
            e.quantize()
        torch.cuda.synchronize()
        err = []

        def run(r):
            try:
                steps(embs[r], k0=r)
            except Exception as ex:  # surfaced below
                err.append(ex)

        ts = [threading.Thread(target=run, args=(r,)) for r in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not err, err
        for e in embs:
            e.close()
        hub.close()
print("sanitize_step: ok")
