"""NEXT-3 pins (CPU): the incremental-training oracle (Eq. 2-3)
-- cold-weight init, the diagonal-FIM penalty and its gradient, and the regularized step."""
import numpy as np

import oracle as O


def test_cold_weight_init_examples():
    # alpha = 1 -> w0, alpha = 0 -> w_{t-1}, alpha = 0.25, [4], [0] -> [1]
    w0 = np.array([4.0, -2.5, 7.0], dtype=np.float32)
    w1 = np.array([0.0, 3.0, -1.0], dtype=np.float32)
    assert (O.cold_weight_init(w0, w1, 1.0) == w0).all()
    assert (O.cold_weight_init(w0, w1, 0.0) == w1).all()
    assert O.cold_weight_init(w0[:1], w1[:1], 0.25)[0] == 1.0


def test_penalty_hand_example_and_reductions():
    # H0 = H1 = I, alpha = 0.5, w0 = [0], w_{t-1} = [2] -> w = [1], penalty = lambda/2
    one = np.ones(1, dtype=np.float32)
    w = O.cold_weight_init(np.zeros(1, np.float32), np.full(1, 2.0, np.float32), 0.5)
    assert w[0] == 1.0
    lam = float(np.float32(0.3))  # the oracle takes lambda, alpha as fp32 scalars
    assert abs(O.fim_penalty(w, np.zeros(1), one, np.full(1, 2.0), one, lam, 0.5) - lam / 2) < 1e-12
    # lambda = 0 -> 0; alpha = 0 reduces Eq. (3) to Eq. (2) (only the w_{t-1} anchor)
    rng = np.random.default_rng(0)
    W, w0, w1 = (rng.standard_normal(50).astype(np.float32) for _ in range(3))
    H0, H1 = (rng.uniform(0, 2, 50).astype(np.float32) for _ in range(2))
    assert O.fim_penalty(W, w0, H0, w1, H1, 0.0, 0.4) == 0.0
    eq2 = float(np.float32(0.7)) / 2 * float(np.sum(H1.astype(np.float64) * (W.astype(np.float64) - w1) ** 2))
    assert abs(O.fim_penalty(W, w0, H0, w1, H1, 0.7, 0.0) - eq2) <= 1e-12 * eq2


def test_penalty_gradient_matches_finite_differences():
    """the penalty is quadratic, so central differences are exact up to rounding."""
    rng = np.random.default_rng(1)
    rows, D = 7, 5
    W, w0, w1 = (rng.standard_normal((rows, D)).astype(np.float32) for _ in range(3))
    H0, H1 = (rng.uniform(0, 2, (rows, D)).astype(np.float32) for _ in range(2))
    lam, alpha = float(np.float32(0.8)), float(np.float32(0.3))  # fp32 scalars, as the oracle's
    keys = np.array([1, 4, 6])
    g = O.fim_penalty_grad(W, keys, np.zeros((3, D), np.float32), w0, H0, w1, H1, lam, alpha)
    h = 1e-2
    for k, u in enumerate(keys):
        for d in range(D):
            Wp, Wm = W.astype(np.float64).copy(), W.astype(np.float64).copy()
            Wp[u, d] += h
            Wm[u, d] -= h
            pen = lambda X: (lam / 2) * (alpha * np.sum(H0 * (X - w0) ** 2) + (1 - alpha) * np.sum(H1 * (X - w1) ** 2))
            fd = (pen(Wp) - pen(Wm)) / (2 * h)
            assert abs(g[k, d] - fd) <= 1e-5 * max(1.0, abs(fd))
    # the oracle's fp64 penalty value agrees with the same finite-difference function
    assert abs(O.fim_penalty(W, w0, H0, w1, H1, lam, alpha) - pen(W.astype(np.float64))) < 1e-9


def test_regularized_step_reduces_to_plain_step_and_pulls_toward_anchor():
    rng = np.random.default_rng(2)
    rows, D, B = 40, 8, 16
    pb = O.Problem([rows], D, [0])
    W = (rng.standard_normal((rows, D)) * 0.1).astype(np.float32)
    lens = rng.integers(0, 4, size=B)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ids = rng.integers(0, rows, size=int(off[-1])).astype(np.int32)
    grad = (rng.standard_normal((B, 1, D)) * 0.01).astype(np.float32)
    w0 = np.zeros_like(W)
    H = np.ones_like(W)
    # lambda = 0 -> bit-exact the plain step
    Wa, Aa = W.copy(), np.full(rows, 0.1, np.float32)
    Wb, Ab = W.copy(), np.full(rows, 0.1, np.float32)
    O.train_step(pb, Wa, Aa, ids, off, B, grad, 0.05, 1e-7, 1.0, want_out=False)
    O.train_step_fim(pb, Wb, Ab, ids, off, B, grad, 0.05, 1e-7, 1.0, w0, H, None, None, 0.0, 1.0)
    assert (Wa == Wb).all() and (Aa == Ab).all()
    # zero loss gradient, strong pull toward w0 = 0: touched rows shrink, untouched rows do not move
    Wc, Ac = W.copy(), np.full(rows, 0.1, np.float32)
    O.train_step_fim(pb, Wc, Ac, ids, off, B, np.zeros_like(grad), 0.05, 1e-7, 1e9, w0, H, None, None, 1.0, 1.0)
    touched = np.unique(ids)
    untouched = np.setdiff1d(np.arange(rows), touched)
    assert (np.abs(Wc[touched]) <= np.abs(W[touched])).all() and (np.abs(Wc[touched]) < np.abs(W[touched])).any()
    assert (Wc[untouched] == W[untouched]).all()
