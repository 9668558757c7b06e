"""NEXT-4 GPU parity: min-max row-wise 8-bit quantization (EMB_F_Q8_MINMAX)
through the C ABI vs the CPU oracle -- codes, min and scale bit-exact; q8 lookup; fused
re-quantization of updated rows; and the error comparison with middle-max on the same rows."""
import numpy as np
import pytest

import oracle as O
from helpers import dense_tables, init_tables_host, make_emb, problem
from test_gpu_parity import dev, small_cfg, special_rows
from workload import gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("dim", [64, 32, 30, 128, 5])
def test_quantize_minmax_bit_exact(gpu, dim):
    cfg = small_cfg(dim=dim, rows=(3000, 41), F=[0, 1])
    emb = make_emb(cfg, max_nnz=100, max_batch=8, q8=True, q8_mode="min_max")
    init_tables_host(emb, cfg)
    sp = special_rows(dim)  # constant, ramp, large offset, exact ties (scale 1), one-hot
    emb.write_rows(0, np.arange(len(sp)), sp)
    bad = np.full((1, dim), 1.0, dtype=np.float32)
    bad[0, dim // 2] = np.inf
    emb.write_rows(1, [40], bad)
    emb.quantize()
    from paper_2402_06859_b200._lib import EMB_ENONFINITE
    assert emb.sync() == EMB_ENONFINITE
    W = dense_tables(cfg)
    W[:len(sp)] = sp
    W[3000 + 40] = bad
    codes, mn, sc, nbad = O.quantize_minmax(W)
    assert nbad == 1
    c0, m0, s0 = emb.read_q8(0, np.arange(3000))
    c1, m1, s1 = emb.read_q8(1, np.arange(41))
    assert c0.dtype == np.uint8
    assert (np.concatenate([c0, c1]) == codes).all()
    assert (np.concatenate([m0, m1]).view(np.uint32) == mn.view(np.uint32)).all()
    assert (np.concatenate([s0, s1]).view(np.uint32) == sc.view(np.uint32)).all()


@pytest.mark.parametrize("dim", [64, 30])
def test_forward_q8_minmax(gpu, dim):
    cfg = small_cfg(dim=dim, rows=(4000, 900), F=[0, 1, 0])
    B = 300
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 9, 0)
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B, q8=True, q8_mode="min_max")
    init_tables_host(emb, cfg)
    emb.quantize()
    out = emb.forward_q8(dev(ids), dev(off), B).cpu().numpy()
    assert emb.sync() == 0
    codes, mn, sc, _ = O.quantize_minmax(dense_tables(cfg))
    ref, bad = O.forward_q8_minmax(problem(cfg), codes, mn, sc, ids, off, B)
    assert bad == 0 and (out == ref).all()


def test_requant_minmax_tracks_updates(gpu):
    cfg = small_cfg(dim=64, rows=(3000,), F=[0, 0])
    B = 256
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 4, 0)
    grad = gen.grad_values(4, 0, B, 2, 64, gen.grad_shift_for(len(ids), 64))
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B, q8=True, requant=True, q8_mode="min_max")
    init_tables_host(emb, cfg)
    emb.quantize()
    emb.forward(dev(ids), dev(off), B)
    emb.backward_adagrad(dev(grad), 0.05)
    assert emb.sync() == 0
    w = emb.read_rows(0, np.arange(3000), with_acc=False)
    codes, mn, sc, _ = O.quantize_minmax(w)
    c, m, s = emb.read_q8(0, np.arange(3000))
    assert (c == codes).all() and (m == mn).all() and (s == sc).all()


def test_minmax_vs_middlemax_error_on_the_same_rows(gpu):
    """The two stores built on the GPU from the same table: their dequantization errors agree
    to fp32 rounding (same grid points) and stay within scale/2 (+ a few ulp)."""
    cfg = small_cfg(dim=64, rows=(20000,), F=[0])
    W = dense_tables(cfg)
    errs = {}
    for mode in ("middle_max", "min_max"):
        emb = make_emb(cfg, max_nnz=10, max_batch=4, q8=True, q8_mode=mode)
        init_tables_host(emb, cfg)
        emb.quantize()
        assert emb.sync() == 0
        c, base, sc = emb.read_q8(0, np.arange(20000))
        deq = c.astype(np.float64) * sc[:, None] + base[:, None]
        e = deq - W
        ulp = np.spacing(np.abs(W).max(axis=1).astype(np.float32)).astype(np.float64)[:, None]
        assert (np.abs(e) <= sc[:, None] * 0.5 + 4 * ulp).all()  # scale/2 + rounding of base, quotient
        errs[mode] = float(np.sqrt((e ** 2).mean()))
    assert abs(errs["min_max"] / errs["middle_max"] - 1) < 0.01, errs
