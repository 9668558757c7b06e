"""NEXT-3 GPU parity: incremental training through the C ABI vs the oracle --
cold-weight init bit-exact, and a training step with the diagonal-FIM penalty on the touched
rows (emb_set_incremental) within the a8 gates."""
import numpy as np
import pytest

import oracle as O
from helpers import S_close, dense_tables, init_tables_host, make_emb, problem, w_close
from test_gpu_parity import dev, small_cfg
from workload import gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def padded(emb, X):
    """[total_rows][dim] numpy -> device [local_rows][pitch] tensor with zero pads."""
    full = np.zeros((emb.local_rows, emb.pitch), dtype=np.float32)
    full[:, :X.shape[1]] = X
    return torch.from_numpy(full).cuda()


@pytest.mark.parametrize("dim", [32, 30])
def test_cold_weight_init_bit_exact(gpu, dim):
    cfg = small_cfg(dim=dim, rows=(2000, 300), F=[0, 1])
    emb = make_emb(cfg, max_nnz=10, max_batch=4)
    rng = np.random.default_rng(dim)
    w0 = rng.standard_normal((cfg.total_rows, dim)).astype(np.float32)
    w1 = rng.standard_normal((cfg.total_rows, dim)).astype(np.float32)
    for alpha in (0.0, 1.0, 0.3):
        emb.cold_weight_init(padded(emb, w0), padded(emb, w1), alpha)
        got = np.concatenate([emb.read_rows(t, np.arange(cfg.table_rows[t]), with_acc=False)
                              for t in range(cfg.num_tables)])
        assert (got == O.cold_weight_init(w0, w1, alpha)).all()


@pytest.mark.parametrize("mode", ["rowwise", "elementwise"])
@pytest.mark.parametrize("terms", ["both", "prior_only"])
def test_train_step_with_fim_penalty(gpu, mode, terms):
    cfg = small_cfg(dim=32, rows=(3000, 700), F=[0, 1, 0], B=256)
    B = 256
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 11, 0)
    grad = gen.grad_values(11, 0, B, 3, 32, gen.grad_shift_for(len(ids), 32))
    W0 = dense_tables(cfg)
    rng = np.random.default_rng(1)
    w0 = (W0 + rng.standard_normal(W0.shape) * 0.05).astype(np.float32)
    w1 = (W0 + rng.standard_normal(W0.shape) * 0.02).astype(np.float32)
    H0 = rng.uniform(0, 3, W0.shape).astype(np.float32)
    H1 = rng.uniform(0, 3, W0.shape).astype(np.float32)
    if terms == "prior_only":
        w0 = H0 = None
    lam, alpha = 0.5, 0.3
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B, adagrad=mode)
    init_tables_host(emb, cfg)
    dv = [None if x is None else padded(emb, x) for x in (w0, H0, w1, H1)]
    emb.set_incremental(*dv, lam, alpha)
    emb.forward(dev(ids), dev(off), B)
    emb.backward_adagrad(dev(grad), 0.05)
    assert emb.sync() == 0
    S_gpu, c_gpu, _ = emb.last_stats()
    W = W0.copy()
    A = np.full((cfg.total_rows,) if mode == "rowwise" else (cfg.total_rows, 32), 0.1, dtype=np.float32)
    r = O.train_step_fim(problem(cfg), W, A, ids, off, B, grad, 0.05, 1e-7, 1.0, w0, H0, w1, H1, lam, alpha,
                         mode=mode)
    assert S_close(S_gpu, r["S"])
    assert abs(float(c_gpu) - float(r["c"])) <= 2e-7 * float(r["c"])
    Wg = np.concatenate([emb.read_rows(t, np.arange(cfg.table_rows[t]), with_acc=False)
                         for t in range(cfg.num_tables)])
    keys, _, _ = O.dedup(problem(cfg), ids, off, B)
    step = np.abs(W - W0)
    assert w_close(Wg[keys], W[keys], W0[keys], step[keys]).all()
    untouched = np.setdiff1d(np.arange(cfg.total_rows), keys)
    assert (Wg[untouched] == W0[untouched]).all()
    assert (Wg[keys] == W[keys]).mean() > 0.99


def test_zero_lambda_is_the_plain_step(gpu):
    cfg = small_cfg(dim=32, rows=(3000,), F=[0, 0], B=128)
    B = 128
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 12, 0)
    grad = gen.grad_values(12, 0, B, 2, 32, gen.grad_shift_for(len(ids), 32))
    outs = []
    for lam in (None, 0.0):
        emb = make_emb(cfg, max_nnz=len(ids), max_batch=B)
        init_tables_host(emb, cfg)
        if lam is not None:
            z = torch.zeros(emb.local_rows, emb.pitch, device=gpu)
            emb.set_incremental(z, z + 1, None, None, lam, 1.0)
        emb.forward(dev(ids), dev(off), B)
        emb.backward_adagrad(dev(grad), 0.05)
        assert emb.sync() == 0
        outs.append(emb.read_rows(0, np.arange(3000), with_acc=False))
    assert (outs[0] == outs[1]).all()
