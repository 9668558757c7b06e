"""Serving handle (EMB_F_Q8_ONLY) and emb_quantize_block: the q8 store filled block by block
from fp32 rows and served by a10, vs the oracle (in-memory serving of the
quantized tables)."""
import numpy as np
import pytest

import oracle as O
from helpers import dense_tables, init_tables_host, make_emb, problem
from test_gpu_parity import dev, small_cfg
from workload import gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("mode", ["middle_max", "min_max"])
def test_serving_handle_block_fill_and_lookup(gpu, mode):
    cfg = small_cfg(dim=64, rows=(5000, 700), F=[0, 1, 0])
    B = 300
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 6, 0)
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B, q8_only=True, q8_mode=mode)
    assert emb.weights_buf is None and emb.accum_buf is None
    W = dense_tables(cfg)
    base = np.concatenate([[0], np.cumsum(cfg.table_rows)])
    for t in range(cfg.num_tables):
        r, chunk = 0, 1234
        while r < cfg.table_rows[t]:
            n = min(chunk, cfg.table_rows[t] - r)
            blk = np.zeros((n, 68), dtype=np.float32)  # ld = 68 > dim: the pad is ignored
            blk[:, :64] = W[base[t] + r: base[t] + r + n]
            blk[:, 64:] = 1e30
            emb.quantize_block(t, r, torch.from_numpy(blk).to(gpu))
            r += n
    out = emb.forward_q8(dev(ids), dev(off), B).cpu().numpy()
    assert emb.sync() == 0
    if mode == "middle_max":
        codes, base_, sc, _ = O.quantize(W)
        ref, _ = O.forward_q8(problem(cfg), codes, base_, sc, ids, off, B)
    else:
        codes, base_, sc, _ = O.quantize_minmax(W)
        ref, _ = O.forward_q8_minmax(problem(cfg), codes, base_, sc, ids, off, B)
    assert (out == ref).all()
    # training / fp32 calls are out of state on a serving handle
    from paper_2402_06859_b200 import EmbError
    with pytest.raises(EmbError):
        emb.forward(dev(ids), dev(off), B, out=torch.empty(B, 3, 64, device=gpu))
    with pytest.raises(EmbError):
        emb.quantize()
    # a block that is not (entirely) in the table is rejected
    with pytest.raises(EmbError):
        emb.quantize_block(1, 600, torch.zeros(200, 64, device=gpu))


def test_quantize_block_equals_full_quantize(gpu):
    cfg = small_cfg(dim=32, rows=(3000,), F=[0])
    a = make_emb(cfg, max_nnz=10, max_batch=4, q8=True)
    b = make_emb(cfg, max_nnz=10, max_batch=4, q8=True)
    for e in (a, b):
        init_tables_host(e, cfg)
    a.quantize()
    b.quantize_block(0, 0, b.table_view(0)[:1500])
    b.quantize_block(0, 1500, b.table_view(0)[1500:])
    assert a.sync() == 0 and b.sync() == 0
    ca, ma, sa = a.read_q8(0, np.arange(3000))
    cb, mb, sb = b.read_q8(0, np.arange(3000))
    assert (ca == cb).all() and (ma == mb).all() and (sa == sb).all()
