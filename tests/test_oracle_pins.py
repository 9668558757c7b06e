"""Pins of the CPU oracle to things other than itself (CPU only, -m "not gpu").

Each test names the passage that fixes the expected value: the paper's formula and its
stated properties, worked examples (SPEC.md, SURVEY.md hand computations), closed forms,
brute force on tiny inputs, and independent library routines (numpy / torch CPU).
"""
import ctypes
import math

import numpy as np
import pytest
import torch

import oracle as O
from workload import gen

f32 = np.float32


_libm = ctypes.CDLL("libm.so.6")
_libm.fmaf.restype = ctypes.c_float
_libm.fmaf.argtypes = [ctypes.c_float] * 3


def fmaf(a, b, c):
    """libm fmaf: one fp32 rounding of a*b+c (the dequant of reading 7)."""
    return np.float32(_libm.fmaf(float(a), float(b), float(c)))


def ulp(x):
    return np.spacing(np.abs(np.float32(x))).astype(np.float64)


# ---------------------------------------------------------------------------
# a9 quantization
# ---------------------------------------------------------------------------

def test_quantize_worked_example_0_1():
    # SPEC.md:321 / PAPER.md:340-342: row [0, 1], b=8 -> middle = 128/255, scale = 1/255,
    # x=0 -> -128, x=1 -> 127.  Closed forms rounded once to fp32.
    codes, mid, sc, bad = O.quantize(np.array([[0.0, 1.0]], dtype=f32))
    assert bad == 0
    assert mid[0] == f32(128.0 / 255.0)
    assert sc[0] == f32(1.0 / 255.0)
    assert codes.tolist() == [[-128, 127]]
    # dequant (fma form, SURVEY.md §8(c) reading 7) reproduces the endpoints exactly
    deq = [fmaf(float(c), float(sc[0]), float(mid[0])) for c in codes[0]]
    assert np.float32(deq[0]) == 0.0 and np.float32(deq[1]) == 1.0


def test_quantize_endpoint_closed_form():
    # Exact arithmetic: (min - middle)/scale = -128 and (max - middle)/scale = 127 for any
    # min < max (substitute PAPER.md:340-342).  Holds in fp32 for well-conditioned rows
    # (|mean| <~ range, SURVEY.md §8(c) "endpoint property").
    rng = np.random.default_rng(1)
    X = rng.uniform(-1, 1, size=(2000, 64)).astype(f32)
    codes, mid, sc, _ = O.quantize(X)
    amin, amax = X.argmin(1), X.argmax(1)
    r = np.arange(len(X))
    assert (codes[r, amin] == -128).all()
    assert (codes[r, amax] == 127).all()


def test_quantize_tie_row_half_away_from_zero():
    # SURVEY.md §8(c) reading 1: ties round half away from zero.
    # Row [0, 255, 0.5, 1.5, 2.5]: middle = 128, scale = 1 (exact), q = x - 128.
    codes, mid, sc, _ = O.quantize(np.array([[0, 255, 0.5, 1.5, 2.5]], dtype=f32))
    assert mid[0] == 128.0 and sc[0] == 1.0
    assert codes[0].tolist() == [-128, 127, -128, -127, -126]  # half-even would give -126 for 1.5


def test_quantize_survey_golden_row():
    # SURVEY.md §8(c) "Computed goldens": [-0.3, 0.1, 0.2, 0.5] -> middle 0.10156862,
    # scale 0.0031372549, codes [-128, 0, 31, 127].
    codes, mid, sc, _ = O.quantize(np.array([[-0.3, 0.1, 0.2, 0.5]], dtype=f32))
    assert abs(float(mid[0]) - 0.10156862) < 2e-8
    assert abs(float(sc[0]) - 0.0031372549) < 1e-10
    assert codes[0].tolist() == [-128, 0, 31, 127]


def test_quantize_constant_row():
    # SPEC.md:322 / reading 4: constant row -> middle = value, scale 0, codes 0 (exact).
    codes, mid, sc, _ = O.quantize(np.full((1, 3), 0.25, dtype=f32))
    assert (mid[0], sc[0]) == (0.25, 0.0) and codes.tolist() == [[0, 0, 0]]
    codes, mid, sc, _ = O.quantize(np.full((1, 64), 1e-3, dtype=f32))
    assert mid[0] == f32(1e-3) and sc[0] == 0.0


def test_quantize_saturates():
    # Reading 3: "int values fall within [-128,127]" holds in exact arithmetic
    # only; large offset + tiny range leaves it in fp32 -> saturate.
    row = np.array([[1e6, 1e6 + 0.1875, 1e6 + 0.0625]], dtype=f32)
    codes, mid, sc, _ = O.quantize(row)
    assert sc[0] > 0
    raw = (row.astype(np.float32) - mid[0]) / sc[0]
    assert (np.abs(raw) > 128).any()  # the raw quotient really leaves the range
    assert codes.min() >= -128 and codes.max() <= 127


def test_quantize_nonfinite_row():
    codes, mid, sc, bad = O.quantize(np.array([[1.0, np.nan, 2.0], [1, 2, 3]], dtype=f32))
    assert bad == 1
    assert codes[0].tolist() == [0, 0, 0] and mid[0] == 0 and sc[0] == 0
    assert codes[1].tolist() == [-128, 0, 127]


@pytest.mark.parametrize("dist", ["uniform", "normal", "offset", "ih4"])
def test_quantize_error_bound_and_range(dist):
    # |dequant - x| <= scale/2 (+ rounding slack: 2 ulp of max|row|,
    # SURVEY.md §8(c)); codes in [-128, 127].
    rng = np.random.default_rng(7)
    n, D = 3000, 64
    if dist == "uniform":
        X = rng.uniform(-1, 1, (n, D))
    elif dist == "normal":
        X = rng.normal(0, 0.036, (n, D))
    elif dist == "offset":
        X = rng.normal(3.0, 0.5, (n, D))
    else:
        X = gen.table_rows(5, 0, np.arange(n), D)
    X = X.astype(f32)
    codes, mid, sc, bad = O.quantize(X)
    assert bad == 0
    assert codes.min() >= -128 and codes.max() <= 127
    deq = np.array([[fmaf(float(c), float(s), float(m)) for c in row]
                    for row, s, m in zip(codes[:200], sc[:200], mid[:200])], dtype=np.float32)
    err = np.abs(deq.astype(np.float64) - X[:200].astype(np.float64))
    bound = sc[:200].astype(np.float64)[:, None] / 2 + 2 * ulp(np.abs(X[:200]).max(1))[:, None]
    assert (err <= bound).all()
    # vectorised check on all rows (fp64 dequant; same bound)
    deq64 = mid.astype(np.float64)[:, None] + codes.astype(np.float64) * sc.astype(np.float64)[:, None]
    bound = sc.astype(np.float64)[:, None] / 2 + 2 * ulp(np.abs(X).max(1))[:, None]
    assert (np.abs(deq64 - X) <= bound).all()


def test_quantize_matches_independent_numpy_float32():
    # An independent vectorised numpy-float32 transcription of PAPER.md:340-342 (each numpy
    # ufunc is one IEEE fp32 op), rounding half away from zero in fp64.
    rng = np.random.default_rng(3)
    X = np.concatenate([rng.normal(0, 0.036, (500, 64)), rng.uniform(-5, 5, (500, 64))]).astype(f32)
    mx, mn = X.max(1), X.min(1)
    mid = ((mx * f32(128)) + (mn * f32(127))) / f32(255)
    sc = (mx - mn) / f32(255)
    q = (X - mid[:, None]) / sc[:, None]
    q64 = q.astype(np.float64)
    r = np.sign(q64) * np.floor(np.abs(q64) + 0.5)
    ref = np.clip(r, -128, 127).astype(np.int8)
    codes, omid, osc, _ = O.quantize(X)
    assert (omid == mid).all() and (osc == sc).all() and (codes == ref).all()


def test_int8_roundtrip_and_size_claim():
    # codes in [-128,127] make the int8 cast reversible (all 256 values).
    v = np.arange(-128, 128)
    assert (v.astype(np.int8).astype(np.int32) == v).all()
    # 10M x 128 fp32 table, 8-bit row-wise -> "over 70%" smaller, with fp32
    # middle + fp32 scale per row (reading 6): 1 - (128 + 8) / 512 = 73.4%.
    rows, D = 10_000_000, 128
    red = 1 - (rows * D * 1 + rows * 8) / (rows * D * 4)
    assert red > 0.70 and abs(red - 0.734375) < 1e-12


# ---------------------------------------------------------------------------
# a2 forward
# ---------------------------------------------------------------------------

def hand_problem():
    # SURVEY.md §8(c) AdaGrad hand example: rows r0=[0.5,-0.25], r1=[1,2], r2=[-1,0.5];
    # one feature, B=2; ids [0,2,0,1], offsets [0,3,4].
    pb = O.Problem([3], 2, [0])
    W = np.array([[0.5, -0.25], [1, 2], [-1, 0.5]], dtype=f32)
    ids = np.array([0, 2, 0, 1], dtype=np.int32)
    off = np.array([0, 3, 4], dtype=np.int32)
    return pb, W, ids, off


def test_forward_hand_example():
    pb, W, ids, off = hand_problem()
    out, bad = O.forward(pb, W, ids, off, 2)
    assert bad == 0
    assert out.reshape(2, 2).tolist() == [[0.0, 0.0], [1.0, 2.0]]  # exact cancellation


def random_problem(seed=0, T=3, F=5, D=16, B=37, rows=(50, 7, 300), maxlen=9, pooling=0, bad_ids=False):
    rng = np.random.default_rng(seed)
    rows = list(rows)[:T]
    ft = rng.integers(0, T, size=F).astype(np.int32)
    pb = O.Problem(rows, D, ft, pooling)
    W = np.concatenate([gen.table_rows(seed, t, np.arange(r), D) for t, r in enumerate(rows)])
    lens = rng.integers(0, maxlen + 1, size=F * B)
    off = np.zeros(F * B + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    ids = np.empty(off[-1], dtype=np.int64)
    for f in range(F):
        a, b = off[f * B], off[(f + 1) * B]
        ids[a:b] = rng.integers(0, rows[ft[f]], size=b - a)
    if bad_ids and len(ids) > 4:
        ids[1] = -1
        ids[3] = rows[ft[0]] + 5 if rows[ft[0]] + 5 < 2**31 else -7
    return pb, W, ids.astype(np.int32), off.astype(np.int32), B


def brute_force_pool(pb, W, ids, off, B, fp64_table=None):
    """Dense incidence-count matrix (bags x rows) times the table, in fp64."""
    base = np.concatenate([[0], np.cumsum(pb.table_rows)])
    F = pb.F
    M = np.zeros((F * B, pb.total_rows))
    absM = np.zeros_like(M)
    for f in range(F):
        t = pb.feature_table[f]
        for b in range(B):
            bag = f * B + b
            for j in range(off[bag], off[bag + 1]):
                i = ids[j]
                if 0 <= i < pb.table_rows[t]:
                    M[bag, base[t] + i] += 1
    Wt = W.astype(np.float64) if fp64_table is None else fp64_table
    ref = M @ Wt
    mag = M @ np.abs(Wt)
    if pb.pooling == 1:
        L = np.diff(off.astype(np.int64)).astype(np.float64)
        L[L == 0] = 1
        ref /= L[:, None]
        mag /= L[:, None]
    # bags are feature-major; output is [B][F][D]
    ref = ref.reshape(F, B, -1).transpose(1, 0, 2)
    mag = mag.reshape(F, B, -1).transpose(1, 0, 2)
    return ref, mag


@pytest.mark.parametrize("pooling", [0, 1])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_forward_brute_force(seed, pooling):
    pb, W, ids, off, B = random_problem(seed, pooling=pooling, bad_ids=True)
    out, bad = O.forward(pb, W, ids, off, B)
    ref, mag = brute_force_pool(pb, W, ids, off, B)
    assert bad == 2
    assert (np.abs(out - ref) <= 1e-6 * mag + 1e-30).all()


@pytest.mark.parametrize("pooling", [0, 1])
def test_forward_matches_torch_embedding_bag(pooling):
    pb, W, ids, off, B = random_problem(11, T=2, F=4, D=32, B=64, rows=(1000, 200), pooling=pooling)
    out, _ = O.forward(pb, W, ids, off, B)
    base = np.concatenate([[0], np.cumsum(pb.table_rows)])
    Wt = torch.from_numpy(W)
    mode = "sum" if pooling == 0 else "mean"
    for f in range(pb.F):
        a, b = off[f * B], off[(f + 1) * B]
        t = pb.feature_table[f]
        ref = torch.nn.functional.embedding_bag(
            torch.from_numpy(ids[a:b].astype(np.int64) + base[t]),
            Wt, torch.from_numpy(off[f * B:(f + 1) * B].astype(np.int64) - a), mode=mode)
        # embedding_bag may add in another order: condition-aware tolerance
        mag = torch.nn.functional.embedding_bag(
            torch.from_numpy(ids[a:b].astype(np.int64) + base[t]),
            Wt.abs(), torch.from_numpy(off[f * B:(f + 1) * B].astype(np.int64) - a), mode=mode)
        assert (np.abs(out[:, f] - ref.numpy()) <= 1e-6 * mag.numpy() + 1e-30).all()


def test_forward_one_hot_is_index_select():
    pb = O.Problem([100, 50], 8, [0, 1, 0])
    W = gen.table_rows(3, 0, np.arange(150), 8)
    B = 20
    rng = np.random.default_rng(0)
    ids = np.concatenate([rng.integers(0, 100, B), rng.integers(0, 50, B), rng.integers(0, 100, B)]).astype(np.int32)
    off = np.arange(3 * B + 1, dtype=np.int32)
    out, _ = O.forward(pb, W, ids, off, B)
    base = [0, 100, 0]
    for f in range(3):
        assert (out[:, f] == W[ids[f * B:(f + 1) * B] + base[f]]).all()  # bit-exact


# ---------------------------------------------------------------------------
# a5 dedup / a6 segment-reduce
# ---------------------------------------------------------------------------

def test_dedup_hand_example():
    pb, W, ids, off = hand_problem()
    keys, segs, bags = O.dedup(pb, ids, off, 2)
    assert keys.tolist() == [0, 1, 2] and segs.tolist() == [0, 2, 3, 4]
    assert bags.tolist() == [0, 0, 1, 0]


@pytest.mark.parametrize("seed", [0, 4])
def test_dedup_matches_numpy_stable_argsort_and_torch_unique(seed):
    pb, W, ids, off, B = random_problem(seed, bad_ids=True)
    keys, segs, bags = O.dedup(pb, ids, off, B)
    base = np.concatenate([[0], np.cumsum(pb.table_rows)])
    F = pb.F
    bag_of = np.repeat(np.arange(F * B), np.diff(off))
    feat = bag_of // B
    t = pb.feature_table[feat]
    valid = (ids >= 0) & (ids < pb.table_rows[t])
    k = (base[t] + ids)[valid]
    order = np.argsort(k, kind="stable")
    u, cnt = torch.unique(torch.from_numpy(k), sorted=True, return_counts=True)
    assert (keys == u.numpy()).all()
    assert (np.diff(segs) == cnt.numpy()).all()
    assert (bags == bag_of[valid][order]).all()


def test_segment_reduce_hand_example():
    pb, W, ids, off = hand_problem()
    keys, segs, bags = O.dedup(pb, ids, off, 2)
    grad = np.array([[[1, 1]], [[0.5, -0.5]]], dtype=f32)  # [B=2][F=1][D=2]
    G = O.segment_reduce(pb, off, 2, segs, bags, grad)
    assert G.tolist() == [[2, 2], [0.5, -0.5], [1, 1]]
    assert O.sq_norm(G) == 10.5


@pytest.mark.parametrize("pooling", [0, 1])
def test_segment_reduce_matches_torch_index_add_fp64(pooling):
    pb, W, ids, off, B = random_problem(5, pooling=pooling, bad_ids=True)
    keys, segs, bags = O.dedup(pb, ids, off, B)
    grad = gen.grad_values(9, 0, B, pb.F, pb.dim, 20)
    G = O.segment_reduce(pb, off, B, segs, bags, grad)
    # torch: per valid occurrence, add grad[b][f] (x 1/L) into row index of its unique key
    base = np.concatenate([[0], np.cumsum(pb.table_rows)])
    bag_of = np.repeat(np.arange(pb.F * B), np.diff(off))
    t = pb.feature_table[bag_of // B]
    valid = (ids >= 0) & (ids < pb.table_rows[t])
    k = (base[t] + ids)[valid]
    bo = bag_of[valid]
    terms = torch.from_numpy(grad.astype(np.float64)[bo % B, bo // B])
    if pooling == 1:
        L = np.diff(off)[bo].astype(np.float64)
        terms = terms * torch.from_numpy(1.0 / L)[:, None]
    idx = torch.from_numpy(np.searchsorted(keys, k))
    acc = torch.zeros(len(keys), pb.dim, dtype=torch.float64).index_add_(0, idx, terms)
    mag = torch.zeros(len(keys), pb.dim, dtype=torch.float64).index_add_(0, idx, terms.abs())
    ref = acc.to(torch.float32).numpy()
    # both are fp64 sums rounded once; the fp32 results may differ by 1 ulp of |sum| terms
    assert (np.abs(G.astype(np.float64) - ref) <= 1e-7 * mag.numpy() + 1e-30).all()


# ---------------------------------------------------------------------------
# a7 clip
# ---------------------------------------------------------------------------

def test_clip_worked_example_3_4():
    # grad [3,4], clip 1 -> factor 0.2, grads [0.6, 0.8].
    G = np.array([[3.0, 4.0]], dtype=f32)
    S = O.sq_norm(G)
    assert S == 25.0
    c, nf = O.clip_factor(S, 1.0)
    assert not nf and c == f32(0.2)
    assert O.clip(G, c).tolist() == [[f32(3) * f32(0.2), f32(4) * f32(0.2)]]


def test_clip_inactive_and_zero():
    # norm <= 1 -> factor exactly 1; zero grads -> 1.
    assert O.clip_factor(0.25, 1.0) == (1.0, False)
    assert O.clip_factor(0.0, 1.0) == (1.0, False)
    assert O.clip_factor(1.0, 1.0) == (1.0, False)


def test_clip_nonfinite():
    # S:409 "non-finite gradient -> training-divergence error (aborts step)".
    assert O.clip_factor(float("inf"), 1.0)[1]
    assert O.clip_factor(float("nan"), 1.0)[1]


def test_clip_invariants_random():
    # post-clip global norm <= clip (+ fp32 slack) and direction preserved.
    rng = np.random.default_rng(2)
    for scale in (0.01, 1.0, 100.0):
        G = (rng.normal(size=(100, 16)) * scale).astype(f32)
        c, _ = O.clip_factor(O.sq_norm(G), 1.0)
        g = O.clip(G, c)
        n = math.sqrt(O.sq_norm(g))
        assert n <= 1.0 + 1e-6
        cos = float((g.astype(np.float64) * G).sum() / (np.linalg.norm(g.astype(np.float64)) * np.linalg.norm(G.astype(np.float64))))
        assert abs(cos - 1) < 1e-7
        if math.sqrt(O.sq_norm(G)) > 1:
            assert abs(n - 1) < 1e-6


# ---------------------------------------------------------------------------
# a8 AdaGrad
# ---------------------------------------------------------------------------

def test_adagrad_hand_example_elementwise_and_rowwise():
    # SURVEY.md §8(c) AdaGrad hand example: c = 1/sqrt(10.5), lr 0.1, eps 1e-7, A0 0.1.
    for mode, Aexp in (("elementwise", [[0.48095241] * 2, [0.12380952] * 2, [0.19523810] * 2]),
                       ("rowwise", [0.48095241, 0.12380953, 0.19523811])):
        pb, W, ids, off = hand_problem()
        A = np.full((3, 2) if mode == "elementwise" else (3,), 0.1, dtype=f32)
        grad = np.array([[[1, 1]], [[0.5, -0.5]]], dtype=f32)
        r = O.train_step(pb, W, A, ids, off, 2, grad, lr=0.1, eps=1e-7, max_norm=1.0, mode=mode)
        assert r["U"] == 3 and r["S"] == 10.5
        assert abs(float(r["c"]) - 0.3086067) < 1e-7
        assert r["out"].reshape(2, 2).tolist() == [[0, 0], [1, 2]]
        Wexp = [[0.41100118, -0.33899882], [0.95614713, 2.0438528], [-1.0698431, 0.43015698]]
        assert np.allclose(W, Wexp, rtol=2e-7, atol=0)
        assert np.allclose(A, Aexp, rtol=2e-7, atol=0)


def test_adagrad_second_hand_example():
    # w=[0.5,-0.25], g=[3,4] -> clip -> [0.6,0.8], A0=0.1, lr=0.1.
    for mode, Wexp, Aexp in (("elementwise", [0.41153485, -0.34299809], None),
                             ("rowwise", [0.42254034, -0.35327953], 0.6)):
        W = np.array([[0.5, -0.25]], dtype=f32)
        A = np.full((1, 2) if mode == "elementwise" else (1,), 0.1, dtype=f32)
        G = np.array([[3, 4]], dtype=f32)
        c, _ = O.clip_factor(O.sq_norm(G), 1.0)
        O.adagrad(W, A, [0], O.clip(G, c), 0.1, 1e-7, mode)
        assert np.allclose(W[0], Wexp, rtol=2e-7, atol=0)
        if Aexp is not None:
            assert abs(float(A[0]) - Aexp) < 1e-7


@pytest.mark.parametrize("mode", ["elementwise", "rowwise"])
def test_adagrad_epsilon_outside_the_root(mode):
    """Reading 9 (eps OUTSIDE the square root, Duchi et al. as the paper cites at P:12; TF,
    torch) pinned where the placement is decisive: A0 = 0 and g = 1e-7 give A' = g^2 = 1e-14,
    sqrt(A') = 1e-7 = eps, so w' = w - lr * g / (|g| + eps) = 0.5 - 0.1 / 2 = 0.45 exactly in
    the closed form -- eps inside the root would give w' = 0.5 - 0.1 * 1e-7 / sqrt(1e-14 +
    1e-7) ~ 0.49999997.  (The hand examples above have A' ~ 0.1-0.5, where the two forms differ
    by ~4e-8 relative, inside their 2e-7 tolerance.)"""
    W = np.array([[0.5, 0.5]], dtype=f32)
    A = np.zeros((1, 2) if mode == "elementwise" else (1,), dtype=f32)
    g = np.array([[1e-7, 1e-7]], dtype=f32)
    O.adagrad(W, A, [0], g, 0.1, 1e-7, mode)
    assert np.allclose(W[0], [0.45, 0.45], rtol=1e-6, atol=0)
    inside = 0.5 - 0.1 * 1e-7 / np.sqrt(1e-14 + 1e-7)
    assert abs(float(W[0, 0]) - inside) > 0.04


def test_adagrad_elementwise_matches_torch_optim():
    # torch.optim.Adagrad (dense, CPU): A += g^2; w -= lr * g / (sqrt(A) + eps).
    rng = np.random.default_rng(0)
    W0 = rng.normal(0, 0.05, (400, 32)).astype(f32)
    G = (rng.normal(0, 0.01, (400, 32))).astype(f32)
    for _ in range(3):
        W = W0.copy()
        A = np.full_like(W, 0.1)
        O.adagrad(W, A, np.arange(400), G, 0.05, 1e-7, "elementwise")
        p = torch.nn.Parameter(torch.from_numpy(W0.copy()))
        opt = torch.optim.Adagrad([p], lr=0.05, initial_accumulator_value=0.1, eps=1e-7)
        p.grad = torch.from_numpy(G.copy())
        opt.step()
        ref = p.detach().numpy()
        step = np.abs(0.05 * G / (np.sqrt(A) + 1e-7))
        tol = 1e-6 * np.maximum(np.maximum(np.abs(ref), np.abs(W0)), step) + 1e-12
        assert (np.abs(W - ref) <= tol).all()
        st = opt.state[p]["sum"].numpy()
        assert (np.abs(A - st) <= 1e-6 * np.abs(st)).all()


def test_adagrad_zero_grad_unchanged_and_sparse_equals_dense():
    # S:420 zero grad -> unchanged; so dense AdaGrad over all rows with G = 0 on untouched
    # rows equals sparse AdaGrad on the touched rows, bit-exactly.
    rng = np.random.default_rng(1)
    for mode in ("rowwise", "elementwise"):
        W = rng.normal(0, 0.05, (50, 8)).astype(f32)
        A = (np.full((50,), 0.1) if mode == "rowwise" else np.full((50, 8), 0.1)).astype(f32)
        touched = np.array([3, 7, 8, 20])
        g = rng.normal(0, 0.1, (4, 8)).astype(f32)
        Ws, As = W.copy(), A.copy()
        O.adagrad(Ws, As, touched, g, 0.05, 1e-7, mode)
        gd = np.zeros((50, 8), dtype=f32)
        gd[touched] = g
        Wd, Ad = W.copy(), A.copy()
        O.adagrad(Wd, Ad, np.arange(50), gd, 0.05, 1e-7, mode)
        assert (Ws == Wd).all() and (As == Ad).all()
        untouched = np.setdiff1d(np.arange(50), touched)
        assert (Ws[untouched] == W[untouched]).all()


@pytest.mark.parametrize("mode", ["rowwise", "elementwise"])
def test_adagrad_quadratic_convergence(mode):
    # f(w) = w^2, 200 AdaGrad steps from w=1, lr=0.5 -> |w| < 0.05.
    W = np.array([[1.0]], dtype=f32)
    A = np.zeros((1,) if mode == "rowwise" else (1, 1), dtype=f32)
    for _ in range(200):
        g = (2 * W).astype(f32)
        O.adagrad(W, A, [0], g, 0.5, 1e-7, mode)
    assert abs(float(W[0, 0])) < 0.05


# ---------------------------------------------------------------------------
# a10 q8 lookup
# ---------------------------------------------------------------------------

def test_forward_q8_brute_force():
    pb, W, ids, off, B = random_problem(8, D=64, bad_ids=True)
    codes, mid, sc, _ = O.quantize(W)
    out, bad = O.forward_q8(pb, codes, mid, sc, ids, off, B)
    assert bad == 2
    deq = mid.astype(np.float64)[:, None] + codes.astype(np.float64) * sc.astype(np.float64)[:, None]
    ref, mag = brute_force_pool(pb, W, ids, off, B, fp64_table=deq)
    assert (np.abs(out - ref) <= 1e-6 * mag + 1e-30).all()


def test_forward_q8_constant_table_exact():
    # constant rows dequantize exactly (reading 4), so one-hot q8 lookups return the value.
    pb = O.Problem([10], 4, [0])
    W = np.repeat(np.linspace(-1, 1, 10, dtype=f32)[:, None], 4, 1)
    codes, mid, sc, _ = O.quantize(W)
    ids = np.arange(10, dtype=np.int32)
    out, _ = O.forward_q8(pb, codes, mid, sc, ids, np.arange(11, dtype=np.int32), 10)
    assert (out[:, 0, :] == W).all()
