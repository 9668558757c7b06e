"""NEXT-2 pins (CPU): the end-to-end Feed train-step oracle (oracle/feed_model.py) against
finite differences, torch.optim.Adagrad, a closed-form loss and the unit-norm clip invariant
(PAPER.md:17, 538)."""
import math

import numpy as np
import pytest

import oracle as O
from oracle import feed_model as FM

torch = pytest.importorskip("torch")


def tiny(seed=0, F=2, D=4, Dd=3, B=6, rows=(50, 20)):
    rng = np.random.default_rng(seed)
    pb = O.Problem(list(rows), D, list(range(F)))
    W = (rng.standard_normal((sum(rows), D)) * 0.1).astype(np.float32)
    A = np.full(sum(rows), 0.1, dtype=np.float32)
    lens = rng.integers(0, 4, size=F * B)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ids = np.concatenate([rng.integers(0, rows[f], size=int(lens[f * B:(f + 1) * B].sum()))
                          for f in range(F)]).astype(np.int32)
    dense = rng.standard_normal((B, Dd))
    labels = rng.integers(0, 2, size=B).astype(np.float64)
    sizes = [F * D + Dd, 100, 100, 100, 100, 1]
    params = []
    for i in range(5):
        params += [rng.standard_normal((sizes[i + 1], sizes[i])) / math.sqrt(sizes[i]),
                   rng.standard_normal(sizes[i + 1]) * 0.1]
    return pb, W, A, ids, off, B, dense, labels, params


def test_tower_gradients_match_finite_differences():
    """The tower's analytic float64 gradients (inputs and every weight) vs central finite
    differences (torch.autograd.gradcheck), on an 8-wide copy of the 5-layer tower."""
    B = 6
    rng = np.random.default_rng(1)
    x = torch.tensor(rng.standard_normal((B, 11)), requires_grad=True)
    sizes = [11, 8, 8, 8, 8, 1]
    ws = []
    for i in range(5):
        ws += [torch.tensor(rng.standard_normal((sizes[i + 1], sizes[i])), requires_grad=True),
               torch.tensor(rng.standard_normal(sizes[i + 1]), requires_grad=True)]
    y = torch.tensor(rng.integers(0, 2, size=B).astype(np.float64))

    def f(x, *ws):
        return torch.nn.functional.binary_cross_entropy_with_logits(FM.tower_forward(x, list(ws)), y)
    assert torch.autograd.gradcheck(f, (x, *ws), eps=1e-6, atol=1e-6)


def test_zero_tower_closed_form_loss_and_dense_only_norm():
    """All weights 0 and the last bias b: logits = b, so loss = mean over samples of
    log(1 + e^-b) (y = 1) / log(1 + e^b) (y = 0), dL/dpooled = 0 (no sparse gradient), and
    S = |dL/db|^2 + |dL/dW_last|^2 with the last layer's input h = 0."""
    pb, W, A, ids, off, B, dense, labels, params = tiny(2)
    for p in params:
        p[...] = 0.0
    b = 0.7
    params[-1][...] = b
    W0, A0 = W.copy(), A.copy()
    accs = [np.full_like(p, 0.1) for p in params]
    r = FM.feed_train_step(pb, W, A, ids, off, B, dense, labels, params, accs, 0.05, 1e-7, 1.0)
    ref = np.mean([math.log1p(math.exp(-b)) if y == 1 else math.log1p(math.exp(b)) for y in labels])
    assert abs(r["loss"] - ref) < 1e-12
    assert (r["grad_pooled"] == 0).all() and (W == W0).all() and (A == A0).all()
    sig = 1 / (1 + math.exp(-b))
    dldb = np.mean([sig - y for y in labels])
    assert abs(r["dense_sq"] - dldb ** 2) < 1e-15 and abs(r["S"] - dldb ** 2) < 1e-15


def test_dense_adagrad_matches_torch_optim():
    """The dense update (with c = 1, clip inactive) equals torch.optim.Adagrad (eps outside
    the sqrt, initial accumulator 0.1, no lr decay) stepped on the same float64 gradients."""
    pb, W, A, ids, off, B, dense, labels, params = tiny(3)
    params = [p * 1e-3 for p in params]  # tiny weights -> tiny gradients -> c = 1
    pooled, _ = O.forward(pb, W, ids, off, B)  # pre-step pooled
    ws = [torch.tensor(p, requires_grad=True) for p in params]
    accs = [np.full_like(p, 0.1) for p in params]
    r = FM.feed_train_step(pb, W, A, ids, off, B, dense, labels, params, accs, 0.05, 1e-7, 1.0)
    assert r["c"] == 1.0
    x = torch.cat([torch.tensor(pooled, dtype=torch.float64).reshape(B, -1), torch.tensor(dense)], 1)
    loss = torch.nn.functional.binary_cross_entropy_with_logits(FM.tower_forward(x, ws), torch.tensor(labels))
    loss.backward()
    torch.optim.Adagrad(ws, lr=0.05, eps=1e-7, initial_accumulator_value=0.1).step()
    for got, t in zip(params, ws):
        assert np.allclose(got, t.detach().numpy(), rtol=1e-12, atol=1e-15)


def test_global_clip_covers_sparse_and_dense():
    """one global norm over the deduplicated sparse rows and every dense parameter;
    when it exceeds 1 the post-clip norm is exactly 1."""
    pb, W, A, ids, off, B, dense, labels, params = tiny(4)
    params = [p * 30.0 for p in params]  # large gradients -> clip active
    accs = [np.full_like(p, 0.1) for p in params]
    W0 = W.copy()
    r = FM.feed_train_step(pb, W, A, ids, off, B, dense, labels, params, accs, 0.05, 1e-7, 1.0)
    keys, segs, bags = O.dedup(pb, ids, off, B)
    G = O.segment_reduce(pb, off, B, segs, bags, r["grad_pooled"])
    sparse_sq = float(np.sum(G.astype(np.float64) ** 2))
    assert abs(r["S"] - (sparse_sq + r["dense_sq"])) <= 1e-12 * r["S"]
    assert r["S"] > 1.0 and abs(math.sqrt(r["S"]) * float(r["c"]) - 1.0) < 1e-6
    assert not (W == W0).all()
