"""GPU parity: the sm_100a path through the C ABI vs the CPU oracle on the same seeded inputs.

Gates (BASELINE.json north_star, SURVEY.md §8(c) comparison classes):
* dedup (unique rows, segment offsets, sorted bag list), int8 codes and q8 metadata:
  bit-exact;
* pooled fp32 outputs: |gpu - ora| <= 1e-5 * sum_j |term_j| (condition-aware 1e-5 rel.);
* updated accumulators: <= 1e-6 relative; updated rows: <= 1e-6 * max(|w'|, |w|, |step|).
"""
import numpy as np
import pytest

import oracle as O
from helpers import (Compact, S_close, cond_close, dense_tables, init_tables_gpu, init_tables_host, make_emb,
                     problem, sample_bags, w_close)
from workload import configs, gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def small_cfg(dim=32, rows=(10_000, 3000, 777, 10_000), F=None, B=256, maxlen=10, seed=1):
    ft = F if F is not None else list(range(len(rows)))
    return configs.Config(f"small{dim}", list(rows), dim, [(t, ("range", 0, maxlen)) for t in ft], B, seed=seed)


# ---------------------------------------------------------------------------
# generator pin (the GPU copy of workload/gen.py)
# ---------------------------------------------------------------------------

def test_gpu_generator_matches_numpy(gpu):
    from workload import gpu as G
    buf = torch.zeros(1000 * 68, device=gpu)
    G.fill_table(buf, 1000, 66, 68, 12345, 3, row0=999_000_000)
    torch.cuda.synchronize()
    got = buf.view(1000, 68).cpu().numpy()
    ref = gen.table_rows(12345, 3, np.arange(999_000_000, 999_001_000), 66)
    assert (got[:, :66] == ref).all() and (got[:, 66:] == 0).all()
    g = torch.zeros(7 * 3 * 16, device=gpu)
    G.fill_grad(g, 7, 3, 16, 99, 5, 30, sample0=11)
    torch.cuda.synchronize()
    assert (g.view(7, 3, 16).cpu().numpy() == gen.grad_values(99, 5, 7, 3, 16, 30, sample0=11)).all()


# ---------------------------------------------------------------------------
# a2 forward
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("dim", [32, 64, 128, 30, 8, 4, 1, 256, 1000])
@pytest.mark.parametrize("pooling", ["sum", "mean"])
def test_forward_small(gpu, dim, pooling):
    cfg = small_cfg(dim=dim, rows=(5000, 300, 7), F=[0, 1, 0, 2, 1])
    B = 200
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, cfg.seed, 0, alpha=1.05)
    emb = make_emb(cfg, max_nnz=len(ids) + 10, max_batch=B, pooling=pooling)
    init_tables_host(emb, cfg)
    out = emb.forward(dev(ids), dev(off), B)
    assert emb.sync() == 0
    pb = problem(cfg, 1 if pooling == "mean" else 0)
    W = dense_tables(cfg)
    ref, bad = O.forward(pb, W, ids, off, B)
    mag, _ = O.forward(pb, np.abs(W), ids, off, B)
    got = out.cpu().numpy()
    assert bad == 0
    assert cond_close(got, ref, mag).all()
    assert (got == ref).all()  # same add order -> bit-exact expected


def test_forward_invalid_ids_and_empty_bags(gpu):
    cfg = small_cfg(dim=64, rows=(100, 50))
    B = 64
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 3, 0)
    ids = ids.copy()
    ids[::7] = -3
    ids[1::11] = 10**6
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B)
    init_tables_host(emb, cfg)
    out = emb.forward(dev(ids), dev(off), B)
    from paper_2402_06859_b200._lib import EMB_EIDRANGE
    assert emb.sync() == EMB_EIDRANGE
    assert emb.sync() == 0  # cleared
    ref, bad = O.forward(problem(cfg), dense_tables(cfg), ids, off, B)
    assert bad > 0
    assert (out.cpu().numpy() == ref).all()
    assert (np.diff(off) == 0).any()


def test_forward_long_bag_and_duplicates(gpu):
    cfg = small_cfg(dim=64, rows=(1000,), F=[0])
    B = 3
    lens = [100_000, 0, 5]
    rng = np.random.default_rng(0)
    ids = rng.integers(0, 1000, sum(lens)).astype(np.int32)
    ids[-5:] = 7  # duplicates inside a bag count with multiplicity
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B)
    init_tables_host(emb, cfg)
    out = emb.forward(dev(ids), dev(off), B).cpu().numpy()
    ref, _ = O.forward(problem(cfg), dense_tables(cfg), ids, off, B)
    assert (out == ref).all()


def test_forward_host_pointers_equal_device(gpu):
    cfg = configs.tiny()
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, cfg.batch, cfg.seed, 1)
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=cfg.batch)
    init_tables_host(emb, cfg)
    a = emb.forward(dev(ids), dev(off), cfg.batch).cpu().numpy()
    hi = torch.from_numpy(ids).pin_memory()
    ho = torch.from_numpy(off).pin_memory()
    out_h = torch.empty((cfg.batch, cfg.num_features, cfg.dim), dtype=torch.float32).pin_memory()
    emb.forward(hi, ho, cfg.batch, out=out_h)
    assert emb.sync() == 0
    assert (out_h.numpy() == a).all()


def test_host_out_is_complete_when_the_call_returns(gpu):
    """a host `out` is filled and the call waits for it -- reading it right after
    the call (no emb_sync) sees the result, even with ~0.1 s of device work queued ahead."""
    cfg = configs.tiny()
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, cfg.batch, cfg.seed, 2)
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=cfg.batch, q8=True)
    init_tables_host(emb, cfg)
    emb.quantize()
    ref = emb.forward(dev(ids), dev(off), cfg.batch).cpu().numpy()
    ref_q8 = emb.forward_q8(dev(ids), dev(off), cfg.batch).cpu().numpy()
    for q8 in (False, True):
        out_h = torch.full((cfg.batch, cfg.num_features, cfg.dim), 7.0).pin_memory()
        with torch.cuda.stream(emb.stream):
            torch.cuda._sleep(200_000_000)
        (emb.forward_q8 if q8 else emb.forward)(dev(ids), dev(off), cfg.batch, out=out_h)
        assert (out_h.numpy() == (ref_q8 if q8 else ref)).all()
    assert emb.sync() == 0


def test_forward_q8_null_inputs_reuse_the_last_forward_batch(gpu):
    """emb_forward_q8(NULL, NULL): the batch of the last emb_forward -- host inputs are not
    staged again (its staged copy is used); batch / nnz must match; once its staging slot has
    been refilled by later host inputs, reuse is refused."""
    from paper_2402_06859_b200._lib import EmbError, EMB_EINVAL, EMB_ESTATE
    cfg = small_cfg(dim=64, rows=(4000, 900), F=[0, 1, 0])
    B = 200
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 11, 0)
    ids2, off2 = gen.make_batch(cfg.table_rows, cfg.features, B, 12, 0)
    emb = make_emb(cfg, max_nnz=max(len(ids), len(ids2)), max_batch=B, q8=True)
    init_tables_host(emb, cfg)
    emb.quantize()
    out = torch.empty((B, cfg.num_features, 64), device=gpu)
    with pytest.raises(EmbError) as e:  # no forward yet
        emb.forward_q8(None, None, B, out=out, nnz=len(ids))
    assert e.value.code == EMB_ESTATE
    ref = emb.forward_q8(dev(ids), dev(off), B).cpu().numpy()
    emb.forward(torch.from_numpy(ids).pin_memory(), torch.from_numpy(off).pin_memory(), B, out=out)
    q = torch.empty_like(out)
    emb.forward_q8(None, None, B, out=q, nnz=len(ids))
    assert emb.sync() == 0
    assert (q.cpu().numpy() == ref).all()
    with pytest.raises(EmbError) as e:
        emb.forward_q8(None, None, B, out=q, nnz=len(ids) + 1)
    assert e.value.code == EMB_EINVAL
    # host inputs are staged into two alternating slots: one q8 call with other host inputs
    # keeps the forward's staged batch; the second one overwrites it and reuse is refused
    h2 = (torch.from_numpy(ids2).pin_memory(), torch.from_numpy(off2).pin_memory())
    emb.forward_q8(*h2, B, out=q)
    q2 = torch.empty_like(out)
    emb.forward_q8(None, None, B, out=q2, nnz=len(ids))
    assert emb.sync() == 0
    assert (q2.cpu().numpy() == ref).all()
    emb.forward_q8(*h2, B, out=q)
    with pytest.raises(EmbError) as e:
        emb.forward_q8(None, None, B, out=q, nnz=len(ids))
    assert e.value.code == EMB_ESTATE
    assert emb.sync() == 0


# ---------------------------------------------------------------------------
# a5-a8 backward
# ---------------------------------------------------------------------------

def run_train_step(cfg, mode, pooling="sum", lr=0.05, gshift=None, ids=None, off=None, B=None,
                   init="host", extra=0.0, max_norm=1.0):
    B = cfg.batch if B is None else B
    if ids is None:
        ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, cfg.seed, 0, alpha=cfg.alpha)
    nnz = len(ids)
    gshift = gen.grad_shift_for(nnz, cfg.dim) if gshift is None else gshift
    grad = gen.grad_values(cfg.seed, 0, B, cfg.num_features, cfg.dim, gshift)
    emb = make_emb(cfg, max_nnz=max(nnz, 1), max_batch=B, adagrad=mode, pooling=pooling, max_norm=max_norm)
    (init_tables_host if init == "host" else init_tables_gpu)(emb, cfg)
    out = emb.forward(dev(ids), dev(off), B)
    S = emb.backward_adagrad(dev(grad), lr, extra_sq_norm=extra, want_norm=True)
    st = emb.sync()
    return emb, ids, off, B, grad, out, S, st


@pytest.mark.parametrize("mode", ["rowwise", "elementwise"])
@pytest.mark.parametrize("pooling", ["sum", "mean"])
@pytest.mark.parametrize("dim", [32, 64, 30])
def test_train_step_small_dense_oracle(gpu, mode, pooling, dim):
    cfg = small_cfg(dim=dim, rows=(2000, 500, 60), F=[0, 1, 0, 2], B=256)
    emb, ids, off, B, grad, out, S, st = run_train_step(cfg, mode, pooling)
    assert st == 0
    pb = problem(cfg, 1 if pooling == "mean" else 0)
    W0 = dense_tables(cfg)
    W = W0.copy()
    A = np.full((cfg.total_rows,) if mode == "rowwise" else (cfg.total_rows, dim), 0.1, dtype=np.float32)
    r = O.train_step(pb, W, A, ids, off, B, grad, 0.05, 1e-7, 1.0, mode=mode)
    # forward bit-exact
    assert (out.cpu().numpy() == r["out"]).all()
    # dedup bit-exact
    keys, segs, bags = O.dedup(pb, ids, off, B)
    u, s, bg = emb.last_dedup()
    assert (u == keys).all() and (s == segs).all() and (bg == bags).all()
    # norm / clip
    S_gpu, c_gpu, U = emb.last_stats()
    assert U == len(keys)
    assert S_close(S_gpu, r["S"])
    assert abs(float(c_gpu) - float(r["c"])) <= 2e-7 * float(r["c"])
    if pooling == "sum":
        assert r["c"] < 1.0  # clip active at the generated grad scale
    # updated rows (touched) and untouched rows
    base = np.concatenate([[0], np.cumsum(cfg.table_rows)])
    Wg, Ag = [], []
    for t in range(cfg.num_tables):
        w, a = emb.read_rows(t, np.arange(cfg.table_rows[t]))
        Wg.append(w)
        Ag.append(a)
    Wg, Ag = np.concatenate(Wg), np.concatenate(Ag)
    G = O.segment_reduce(pb, off, B, segs, bags, grad)
    g = O.clip(G, r["c"])
    if mode == "rowwise":
        den = np.sqrt(A[keys]) + np.float32(1e-7)
        step = np.abs(0.05 / den[:, None] * g)
        assert (np.abs(Ag - A) <= 1e-6 * np.abs(A)).all()
    else:
        den = np.sqrt(A[keys]) + np.float32(1e-7)
        step = np.abs(0.05 * g / den)
        assert (np.abs(Ag - A) <= 1e-6 * np.abs(A)).all()
    assert w_close(Wg[keys], W[keys], W0[keys], step).all()
    untouched = np.setdiff1d(np.arange(cfg.total_rows), keys)
    assert (Wg[untouched] == W0[untouched]).all()
    frac = (Wg[keys] == W[keys]).mean()
    assert frac > 0.99, frac  # bit-exact except rare 1-ulp fp64-order flips


def test_train_step_clip_inactive_and_extra_norm(gpu):
    cfg = small_cfg(dim=32)
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, 256, 5, 0)
    gshift = gen.grad_shift_for(len(ids), 32, target_norm=0.5)
    emb, ids, off, B, grad, out, S, st = run_train_step(cfg, "rowwise", ids=ids, off=off, B=256, gshift=gshift)
    S0, c, U = emb.last_stats()
    assert c == 1.0 and S0 < 1.0
    # extra_sq_norm folds a dense-tower norm into the clip ("global gradient")
    emb, *_ = run_train_step(cfg, "rowwise", ids=ids, off=off, B=256, gshift=gshift, extra=3.0)
    S1, c1, _ = emb.last_stats()
    assert abs(S1 - (S0 + 3.0)) < 1e-12 and abs(float(c1) - 1 / np.sqrt(S1)) < 1e-7


def test_grad_zeros_and_subnormals_widen_exactly(gpu):
    """Zeros, -0 and subnormals in the upstream gradient go through a6's fp64 sums like any
    value (reading 13): the update equals the oracle's as for ordinary grads."""
    cfg = small_cfg(dim=64, rows=(2000, 500, 60), F=[0, 1, 0, 2], B=256)
    B, F, D = 256, cfg.num_features, 64
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, cfg.seed, 0)
    grad = gen.grad_values(cfg.seed, 0, B, F, D, gen.grad_shift_for(len(ids), D))
    rng = np.random.default_rng(3)
    m = rng.random(grad.shape)
    grad[m < 0.05] = 0.0
    grad[(m >= 0.05) & (m < 0.07)] = -0.0
    grad[(m >= 0.07) & (m < 0.08)] = np.float32(3e-39) * np.sign(grad[(m >= 0.07) & (m < 0.08)] + 1e-30)
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B)
    init_tables_host(emb, cfg)
    emb.forward(dev(ids), dev(off), B)
    emb.backward_adagrad(dev(grad), 0.05)
    assert emb.sync() == 0
    pb = problem(cfg)
    W0 = dense_tables(cfg)
    W = W0.copy()
    A = np.full(cfg.total_rows, 0.1, dtype=np.float32)
    r = O.train_step(pb, W, A, ids, off, B, grad, 0.05, 1e-7, 1.0)
    S_gpu, c_gpu, U = emb.last_stats()
    assert S_close(S_gpu, r["S"])
    keys, segs, bags = O.dedup(pb, ids, off, B)
    Wg = np.concatenate([emb.read_rows(t, np.arange(cfg.table_rows[t]), with_acc=False)
                         for t in range(cfg.num_tables)])
    G = O.segment_reduce(pb, off, B, segs, bags, grad)
    g = O.clip(G, r["c"])
    step = np.abs(0.05 / (np.sqrt(A[keys]) + np.float32(1e-7))[:, None] * g)
    assert w_close(Wg[keys], W[keys], W0[keys], step).all()
    assert (Wg[keys] == W[keys]).mean() > 0.99


def test_nonfinite_grad_skips_update(gpu):
    cfg = small_cfg(dim=32)
    B = 64
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 7, 0)
    grad = gen.grad_values(7, 0, B, cfg.num_features, 32, 30)
    grad[3, 1, 5] = np.inf
    grad[9, 2, 7] = np.nan
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B)
    init_tables_host(emb, cfg)
    w0 = emb.weights.clone()
    emb.forward(dev(ids), dev(off), B)
    emb.backward_adagrad(dev(grad), 0.05)
    from paper_2402_06859_b200._lib import EMB_ENONFINITE
    assert emb.sync() == EMB_ENONFINITE
    assert torch.equal(emb.weights, w0)


@pytest.mark.parametrize("pooling", ["sum", "mean"])
def test_a6_widening_exact_over_the_fp32_range(gpu, pooling):
    """a6 widens fp32 -> fp64 on the ALU pipe (the fp32 bits placed in the fp64 fields, then a
    fused multiply-add by 2^896; MEAN: by (1/L) 2^896).  It must give the hardware conversion's
    sums bit for bit on every exponent class: gradient elements with random sign and mantissa and
    exponents from fp32 subnormals to 2^60, plus zeros and -0.  Element-wise AdaGrad with the
    clip inactive (c = 1) updates each element from its own G element only, so W and A must equal
    the oracle's exactly; every row occurs twice, so G is a real two-term sum."""
    rows, B, F, D = 600, 200, 2, 64
    cfg = small_cfg(dim=D, rows=(rows,), F=[0, 0], B=B)
    rng = np.random.default_rng(11)
    ids = rng.permutation(np.repeat(np.arange(rows), 2)).astype(np.int32)
    off = np.arange(0, 3 * F * B + 1, 3, dtype=np.int32)  # 400 bags of 3
    sign = rng.integers(0, 2, (B, F, D), dtype=np.uint32) << np.uint32(31)
    expo = rng.integers(0, 188, (B, F, D), dtype=np.uint32) << np.uint32(23)  # 2^-149 .. 2^60
    mant = rng.integers(0, 1 << 23, (B, F, D), dtype=np.uint32)
    grad = (sign | expo | mant).view(np.float32)
    m = rng.random(grad.shape)
    grad[m < 0.03] = 0.0
    grad[(m >= 0.03) & (m < 0.05)] = -0.0
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B, adagrad="elementwise", pooling=pooling, max_norm=1e30)
    init_tables_host(emb, cfg)
    emb.forward(dev(ids), dev(off), B)
    emb.backward_adagrad(dev(grad), 0.05)
    assert emb.sync() == 0
    pb = problem(cfg, 1 if pooling == "mean" else 0)
    W = dense_tables(cfg)
    A = np.full((rows, D), 0.1, dtype=np.float32)
    r = O.train_step(pb, W, A, ids, off, B, grad, 0.05, 1e-7, 1e30, mode="elementwise")
    assert float(r["c"]) == 1.0 and float(emb.last_stats()[1]) == 1.0
    w, a = emb.read_rows(0, np.arange(rows))
    assert (a == A).all()
    assert (w == W).all()


@pytest.mark.parametrize("kind,pooling", [("inf", "sum"), ("nan", "sum"), ("overflow", "sum"),
                                          ("inf", "mean"), ("nan", "mean")])
def test_nonfinite_S_matches_oracle(gpu, kind, pooling):
    """a6 widens on the ALU pipe and re-runs a batch with an Inf / NaN element (or a G that
    overflows fp32) with the hardware conversions: S is the oracle's (Inf stays Inf, NaN NaN)."""
    cfg = small_cfg(dim=64, rows=(300, 40), F=[0, 1, 0], B=128)
    B, F, D = 128, cfg.num_features, 64
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 5, 0)
    grad = gen.grad_values(5, 0, B, F, D, gen.grad_shift_for(len(ids), D))
    if kind == "inf":
        grad[7, 1, 3] = np.inf
    elif kind == "nan":
        grad[7, 1, 3] = np.nan
    else:  # two finite occurrences of one row whose fp64 sum rounds past FLT_MAX
        ids = ids.copy()
        b0, b1 = [b for b in range(B) if off[b + 1] > off[b]][:2]  # two non-empty feature-0 bags
        ids[off[b0]] = ids[off[b1]] = 17  # feature 0 (bags 0..B-1), table 0, row 17
        grad[b0, 0, 11] = grad[b1, 0, 11] = np.float32(3e38)
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B, pooling=pooling)
    init_tables_host(emb, cfg)
    w0 = emb.weights.clone()
    emb.forward(dev(ids), dev(off), B)
    emb.backward_adagrad(dev(grad), 0.05)
    from paper_2402_06859_b200._lib import EMB_ENONFINITE
    assert emb.sync() == EMB_ENONFINITE
    assert torch.equal(emb.weights, w0)
    pb = problem(cfg, 1 if pooling == "mean" else 0)
    W = dense_tables(cfg)
    A = np.full(cfg.total_rows, 0.1, dtype=np.float32)
    r = O.train_step(pb, W, A, ids, off, B, grad, 0.05, 1e-7, 1.0)
    S_gpu = emb.last_stats()[0]
    if kind == "nan":
        assert np.isnan(r["S"]) and np.isnan(S_gpu)
    else:
        assert r["S"] == np.inf and S_gpu == np.inf


def test_empty_batch_and_all_invalid(gpu):
    cfg = small_cfg(dim=32)
    emb = make_emb(cfg, max_nnz=100, max_batch=16)
    init_tables_host(emb, cfg)
    w0 = emb.weights.clone()
    ids = np.zeros(0, dtype=np.int32)
    off = np.zeros(4 * 16 + 1, dtype=np.int32)
    out = emb.forward(torch.zeros(0, dtype=torch.int32, device=gpu), dev(off), 16)
    emb.backward_adagrad(torch.ones(16, 4, 32, device=gpu), 0.1)
    assert emb.sync() == 0
    assert (out.cpu().numpy() == 0).all() and torch.equal(emb.weights, w0)
    S, c, U = emb.last_stats()
    assert U == 0 and S == 0 and c == 1.0
    ids = np.full(40, -1, dtype=np.int32)
    off = np.zeros(4 * 16 + 1, dtype=np.int32)
    off[1:] = 40
    emb.forward(dev(ids), dev(off), 16)
    emb.backward_adagrad(torch.ones(16, 4, 32, device=gpu), 0.1)
    emb.sync()
    assert torch.equal(emb.weights, w0)
    assert emb.last_stats()[2] == 0


def test_hot_row_spans_many_chunks(gpu):
    # one row with 300k occurrences: exercises the chunk partials and the long fix-up
    cfg = small_cfg(dim=64, rows=(5000,), F=[0, 0])
    B = 4096
    rng = np.random.default_rng(2)
    lens = rng.integers(1, 100, 2 * B)
    ids = rng.integers(0, 5000, lens.sum()).astype(np.int32)
    ids[rng.random(len(ids)) < 0.7] = 1234
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    emb, ids, off, B, grad, out, S, st = run_train_step(cfg, "rowwise", ids=ids, off=off, B=B)
    pb = problem(cfg)
    W0 = dense_tables(cfg)
    W = W0.copy()
    A = np.full(5000, 0.1, dtype=np.float32)
    r = O.train_step(pb, W, A, ids, off, B, grad, 0.05, 1e-7, 1.0)
    keys, segs, bags = O.dedup(pb, ids, off, B)
    u, s, bg = emb.last_dedup()
    assert (u == keys).all() and (s == segs).all() and (bg == bags).all()
    Sg, c, U = emb.last_stats()
    assert abs(Sg - r["S"]) <= 1e-9 * r["S"]
    w, a = emb.read_rows(0, keys)
    assert (np.abs(a - A[keys]) <= 1e-6 * A[keys]).all()
    G = O.segment_reduce(pb, off, B, segs, bags, grad)
    g = O.clip(G, r["c"])
    step = np.abs(0.05 / (np.sqrt(A[keys]) + 1e-7)[:, None] * g)
    assert w_close(w, W[keys], W0[keys], step).all()


def test_multi_step_and_determinism(gpu):
    cfg = small_cfg(dim=64, rows=(3000, 800), F=[0, 1, 1], B=512)
    pb = problem(cfg)
    W = dense_tables(cfg)
    A = np.full(cfg.total_rows, 0.1, dtype=np.float32)
    embs = [make_emb(cfg, max_nnz=20000, max_batch=512) for _ in range(2)]
    for e in embs:
        init_tables_host(e, cfg)
    for step in range(4):
        ids, off = gen.make_batch(cfg.table_rows, cfg.features, 512, 11, step)
        grad = gen.grad_values(11, step, 512, 3, 64, gen.grad_shift_for(len(ids), 64))
        outs = []
        for e in embs:
            outs.append(e.forward(dev(ids), dev(off), 512).cpu().numpy())
            e.backward_adagrad(dev(grad), 0.05)
            assert e.sync() == 0
        r = O.train_step(pb, W, A, ids, off, 512, grad, 0.05, 1e-7, 1.0)
        assert (outs[0] == outs[1]).all()
        assert cond_close(outs[0], r["out"], O.forward(pb, np.abs(W), ids, off, 512)[0] + 1e-3).all()
    assert torch.equal(embs[0].weights, embs[1].weights)  # run-to-run deterministic
    assert torch.equal(embs[0].accum_buf, embs[1].accum_buf)
    w = np.concatenate([embs[0].read_rows(t, np.arange(r), with_acc=False) for t, r in enumerate(cfg.table_rows)])
    rel = np.abs(w - W) / np.maximum(np.abs(W), 1e-3)
    assert rel.max() < 1e-5


# ---------------------------------------------------------------------------
# a9 / a10
# ---------------------------------------------------------------------------

def special_rows(dim):
    rows = [np.full(dim, 0.25), np.linspace(-1, 1, dim), np.full(dim, 1e6) + np.arange(dim) % 3 * 0.0625]
    tie = np.zeros(dim)
    tie[:5] = [0, 255, 0.5, 1.5, 2.5]
    tie[5:] = 128
    rows.append(tie)
    r = np.zeros(dim)
    r[0] = 1.0
    rows.append(r)
    return np.array(rows, dtype=np.float32)


@pytest.mark.parametrize("dim", [64, 32, 30, 128, 5])
def test_quantize_bit_exact(gpu, dim):
    cfg = small_cfg(dim=dim, rows=(3000, 41), F=[0, 1])
    emb = make_emb(cfg, max_nnz=100, max_batch=8, q8=True)
    init_tables_host(emb, cfg)
    sp = special_rows(dim)
    emb.write_rows(0, np.arange(len(sp)), sp)
    bad = np.full((1, dim), 1.0, dtype=np.float32)
    bad[0, dim // 2] = np.nan
    emb.write_rows(1, [40], bad)
    emb.quantize()
    from paper_2402_06859_b200._lib import EMB_ENONFINITE
    assert emb.sync() == EMB_ENONFINITE
    W = dense_tables(cfg)
    W[:len(sp)] = sp
    W[3000 + 40] = bad
    codes, mid, sc, nbad = O.quantize(W)
    assert nbad == 1
    c0, m0, s0 = emb.read_q8(0, np.arange(3000))
    c1, m1, s1 = emb.read_q8(1, np.arange(41))
    assert (np.concatenate([c0, c1]) == codes).all()
    assert (np.concatenate([m0, m1]).view(np.uint32) == mid.view(np.uint32)).all()
    assert (np.concatenate([s0, s1]).view(np.uint32) == sc.view(np.uint32)).all()


@pytest.mark.parametrize("dim", [64, 32, 30])
def test_forward_q8(gpu, dim):
    cfg = small_cfg(dim=dim, rows=(4000, 900), F=[0, 1, 0])
    B = 300
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 9, 0)
    ids = ids.copy()
    ids[5] = -1
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B, q8=True)
    init_tables_host(emb, cfg)
    emb.quantize()
    out = emb.forward_q8(dev(ids), dev(off), B).cpu().numpy()
    from paper_2402_06859_b200._lib import EMB_EIDRANGE
    assert emb.sync() == EMB_EIDRANGE
    W = dense_tables(cfg)
    codes, mid, sc, _ = O.quantize(W)
    pb = problem(cfg)
    ref, bad = O.forward_q8(pb, codes, mid, sc, ids, off, B)
    assert bad == 1
    assert (out == ref).all()


@pytest.mark.parametrize("mode,pooling,dim", [("rowwise", "sum", 64), ("elementwise", "sum", 64),
                                              ("rowwise", "mean", 30), ("elementwise", "mean", 128)])
def test_requant_tracks_updates(gpu, mode, pooling, dim):
    """The fused a8 + a9 re-quantization of the touched rows (both AdaGrad modes, both
    poolings, several geometries) equals the oracle's a9 of the updated table."""
    cfg = small_cfg(dim=dim, rows=(3000,), F=[0, 0])
    B = 256
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, 4, 0)
    grad = gen.grad_values(4, 0, B, 2, dim, gen.grad_shift_for(len(ids), dim))
    emb = make_emb(cfg, max_nnz=len(ids), max_batch=B, q8=True, requant=True, adagrad=mode, pooling=pooling)
    init_tables_host(emb, cfg)
    emb.quantize()
    emb.forward(dev(ids), dev(off), B)
    emb.backward_adagrad(dev(grad), 0.05)
    assert emb.sync() == 0
    w = emb.read_rows(0, np.arange(3000), with_acc=False)
    codes, mid, sc, _ = O.quantize(w)   # oracle quantize of the GPU's updated table
    c, m, s = emb.read_q8(0, np.arange(3000))
    assert (c == codes).all() and (m == mid).all() and (s == sc).all()


# ---------------------------------------------------------------------------
# full-size configs (the bench's launch configuration)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["jobs", "feed1", "feed1@alpha0", "ads", "feed1@elementwise", "feed1@minmax"])
def test_full_config_train_step(gpu, name):
    """The bench's launch configuration at full size (Feed-1 also with uniform ids, the
    alpha = 0 variant of SURVEY §8(d)'s gate: ~5x more unique rows, shorter segments; and
    Feed-1 with element-wise AdaGrad and with the NEXT-4 min-max q8 store)."""
    base, _, variant = name.partition("@")
    cfg = configs.get(base)
    if variant == "alpha0":
        cfg = cfg.with_(alpha=0.0)
    mode = "elementwise" if variant == "elementwise" else "rowwise"
    minmax = variant == "minmax"
    quant = O.quantize_minmax if minmax else O.quantize
    B = cfg.batch
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, cfg.seed, 0, alpha=cfg.alpha)
    nnz = len(ids)
    emb = make_emb(cfg, max_nnz=nnz, max_batch=B, q8=True, adagrad=mode,
                   q8_mode="min_max" if minmax else "middle_max")
    init_tables_gpu(emb, cfg)
    gshift = gen.grad_shift_for(nnz, cfg.dim)
    grad = torch.empty((B, cfg.num_features, cfg.dim), device=gpu)
    from workload import gpu as G
    G.fill_grad(grad, B, cfg.num_features, cfg.dim, cfg.seed, 0, gshift)
    out = emb.forward(dev(ids), dev(off), B)
    S = emb.backward_adagrad(grad, 0.05, want_norm=True)
    assert emb.sync() == 0
    comp = Compact(cfg, ids, off, B)
    # forward: sampled samples (all features) vs the oracle
    rng = np.random.default_rng(0)
    samples = np.sort(rng.choice(B, 64, replace=False))
    sids, soff = sample_bags(cfg, comp.cids, off, B, samples)
    ref, _ = O.forward(comp.pb, comp.W, sids, soff, len(samples))
    got = out.cpu().numpy()[samples]
    assert (got == ref).all()
    # whole backward on the compact problem
    W = comp.W.copy()
    A = np.full(len(comp.keys) if mode == "rowwise" else (len(comp.keys), cfg.dim), 0.1, dtype=np.float32)
    g_host = grad.cpu().numpy()
    assert (g_host[:3] == gen.grad_values(cfg.seed, 0, 3, cfg.num_features, cfg.dim, gshift)).all()
    r = O.train_step(comp.pb, W, A, comp.cids, off, B, g_host, 0.05, 1e-7, 1.0, want_out=False, mode=mode)
    u, s, bg = emb.last_dedup()
    keys, segs, bags = O.dedup(comp.pb, comp.cids, off, B)
    assert len(u) == len(comp.keys) == r["U"]
    assert (u.astype(np.int64) == comp.keys).all()  # W=1: local key = global key
    assert (s == segs).all() and (bg == bags).all()
    assert S_close(S, r["S"])
    # updated rows: a sample of touched rows, incl. the hottest
    counts = np.diff(segs)
    pick = np.unique(np.concatenate([np.argsort(counts)[-50:], rng.choice(len(keys), 2000, replace=False)]))
    for t in np.unique(comp.table_of_key[pick]):
        m = pick[comp.table_of_key[pick] == t]
        w, a = emb.read_rows(int(t), comp.row_of_key[m])
        assert (np.abs(a - A[m]) <= 1e-6 * A[m]).all()
        assert w_close(w, W[m], comp.W[m], np.abs(W[m] - comp.W[m])).all()
    # q8 of the updated table on a sample of rows
    emb.quantize()
    tq = int(np.argmax(cfg.table_rows))
    rows = rng.choice(cfg.table_rows[tq], min(5000, cfg.table_rows[tq]), replace=False)
    c, mm, ss = emb.read_q8(tq, rows)
    w = emb.read_rows(tq, rows, with_acc=False)
    codes, mid, sc, _ = quant(w)
    assert (c.view(np.uint8) == codes.view(np.uint8)).all() and (mm == mid).all() and (ss == sc).all()
    # a10 at full size: the q8 lookup of the same batch on the sampled samples, against the
    # oracle's lookup over the oracle's quantization of the (GPU-updated) compact rows
    q8 = emb.forward_q8(dev(ids), dev(off), B).cpu().numpy()[samples]
    assert emb.sync() == 0
    skeys = np.unique(sids[sids >= 0]) if len(sids) else np.zeros(0, np.int64)
    Wq = np.zeros_like(comp.W)
    for t in np.unique(comp.table_of_key[skeys]):
        m = skeys[comp.table_of_key[skeys] == t]
        Wq[m] = emb.read_rows(int(t), comp.row_of_key[m], with_acc=False)
    qc, qm, qs, _ = quant(Wq)
    ref_q8, _ = (O.forward_q8_minmax if minmax else O.forward_q8)(comp.pb, qc, qm, qs, sids, soff, len(samples))
    deq = np.abs(qm.astype(np.float64))[:, None] + np.abs(qc.astype(np.float64) * qs[:, None])
    mag, _ = O.forward(comp.pb, deq.astype(np.float32), sids, soff, len(samples))
    assert cond_close(q8, ref_q8, mag).all()


def test_q8_reuses_bag_order_of_a_different_batch(gpu):
    """emb_forward_q8 reuses the bag order the last emb_forward built when the offsets pointer
    and bag count match.  Any permutation of the bags is a correct visiting order (the kernels
    read the current lengths), so a q8 forward on DIFFERENT offsets written into the same
    buffer must still match the oracle exactly."""
    cfg = small_cfg(dim=64, rows=(4000, 900), F=[0, 1, 0])
    B = 300
    ids1, off1 = gen.make_batch(cfg.table_rows, cfg.features, B, 21, 0)
    ids2, off2 = gen.make_batch(cfg.table_rows, cfg.features, B, 22, 0)
    nmax = max(len(ids1), len(ids2))
    emb = make_emb(cfg, max_nnz=nmax, max_batch=B, q8=True)
    init_tables_host(emb, cfg)
    emb.quantize()
    off_buf = dev(off1)
    ids_buf = torch.zeros(nmax, dtype=torch.int32, device=gpu)
    ids_buf[:len(ids1)] = dev(ids1)
    emb.forward(ids_buf[:len(ids1)], off_buf, B)
    off_buf.copy_(dev(off2))           # same pointer, new content
    ids_buf[:len(ids2)] = dev(ids2)
    out = emb.forward_q8(ids_buf[:len(ids2)], off_buf, B).cpu().numpy()
    assert emb.sync() == 0
    codes, mid, sc, _ = O.quantize(dense_tables(cfg))
    ref, _ = O.forward_q8(problem(cfg), codes, mid, sc, ids2, off2, B)
    assert (out == ref).all()
