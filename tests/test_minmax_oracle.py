"""NEXT-4 pins (CPU): the oracle's min-max row-wise 8-bit quantization
against closed forms, the paper's algebra relating it to middle-max, and brute force."""
import numpy as np

import oracle as O


def test_unit_row_closed_form():
    # row spanning [0, 1]: X^min = 0, X^scale = 1/255, the endpoints map to 0 and 255
    x = np.array([[0.0, 1.0, 0.5, 0.25]], dtype=np.float32)
    codes, mn, sc, bad = O.quantize_minmax(x)
    assert bad == 0 and mn[0] == 0.0 and sc[0] == np.float32(1.0) / np.float32(255.0)
    assert codes[0, 0] == 0 and codes[0, 1] == 255
    # fl(1/255) = 0.0039215689 > 1/255, so fl(0.5 / scale) = 127.49999 (just below the tie) -> 127
    # and fl(0.25 / scale) = 63.749996 -> 64 (reading 2: fp32 operations in the written order)
    assert codes[0, 2] == 127 and codes[0, 3] == 64


def test_endpoints_on_random_rows():
    rng = np.random.default_rng(0)
    X = (rng.standard_normal((2000, 33)) * rng.uniform(1e-3, 1e3, size=(2000, 1))).astype(np.float32)
    codes, mn, sc, _ = O.quantize_minmax(X)
    assert (mn == X.min(axis=1)).all()
    am, ax = X.argmin(axis=1), X.argmax(axis=1)
    r = np.arange(len(X))
    assert (codes[r, am] == 0).all() and (codes[r, ax] == 255).all()


def test_ties_round_half_away_from_zero():
    # min 0, max 255 -> scale exactly 1: x = k + 0.5 must round up
    x = np.array([[0.0, 255.0, 2.5, 3.5, 100.5]], dtype=np.float32)
    codes, mn, sc, _ = O.quantize_minmax(x)
    assert sc[0] == 1.0 and codes[0].tolist() == [0, 255, 3, 4, 101]


def test_constant_and_nonfinite_rows():
    codes, mn, sc, bad = O.quantize_minmax(np.full((1, 8), -0.75, dtype=np.float32))
    assert bad == 0 and mn[0] == -0.75 and sc[0] == 0.0 and (codes == 0).all()
    x = np.ones((2, 4), dtype=np.float32)
    x[1, 2] = np.nan
    codes, mn, sc, bad = O.quantize_minmax(x)
    assert bad == 1 and mn[1] == 0.0 and sc[1] == 0.0 and (codes[1] == 0).all()


def test_same_grid_as_middle_max():
    """X^middle = (X^max 2^(b-1) + X^min (2^(b-1)-1)) / (2^b-1) = X^min + 128 X^scale,
    so (X - X^middle)/X^scale + 128 = (X - X^min)/X^scale: the middle-max code + 128 equals the
    min-max code (exactly, up to fp32 rounding of the stored middle near a rounding boundary).
    Catches an offset, sign or operand error in either oracle."""
    rng = np.random.default_rng(1)
    X = (rng.standard_normal((3000, 64)) * 0.036).astype(np.float32)
    c_mm, mid, sc_mm, _ = O.quantize(X)
    c_minmax, mn, sc, _ = O.quantize_minmax(X)
    assert (sc == sc_mm).all()
    d = c_minmax.astype(np.int32) - (c_mm.astype(np.int32) + 128)
    assert np.abs(d).max() <= 1 and (d == 0).mean() > 0.999


def test_dequant_error_bound_and_pooled_lookup_brute_force():
    rng = np.random.default_rng(2)
    rows, D = 500, 16
    X = (rng.standard_normal((rows, D)) * 0.05).astype(np.float32)
    codes, mn, sc, _ = O.quantize_minmax(X)
    deq = codes.astype(np.float64) * sc[:, None].astype(np.float64) + mn[:, None].astype(np.float64)
    assert (np.abs(deq - X) <= sc[:, None] / 2 * (1 + 1e-5) + 1e-7).all()
    # a10 over the min-max store vs an fp64 brute force over the dequantized table
    pb = O.Problem([rows], D, [0, 0])
    B = 40
    lens = rng.integers(0, 6, size=2 * B)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ids = rng.integers(0, rows, size=int(off[-1])).astype(np.int32)
    out, inv = O.forward_q8_minmax(pb, codes, mn, sc, ids, off, B)
    ref = np.zeros((B, 2, D))
    mag = np.zeros((B, 2, D))
    for f in range(2):
        for b in range(B):
            for j in ids[off[f * B + b]:off[f * B + b + 1]]:
                ref[b, f] += deq[j]
                mag[b, f] += np.abs(deq[j])
    assert inv == 0 and (np.abs(out - ref) <= 1e-6 * mag + 1e-30).all()


def test_error_comparison_with_middle_max():
    """NEXT-4: the dequantization error of min-max vs middle-max on the same normal rows
    ("embedding values typically follow a normal distribution").  The two grids are
    the same points (test_same_grid_as_middle_max), so the errors agree to fp32 rounding."""
    rng = np.random.default_rng(3)
    X = (rng.standard_normal((4000, 64)) * 0.036).astype(np.float32)
    c1, mid, s1, _ = O.quantize(X)
    c2, mn, s2, _ = O.quantize_minmax(X)
    e_mm = c1.astype(np.float64) * s1[:, None] + mid[:, None] - X
    e_minmax = c2.astype(np.float64) * s2[:, None] + mn[:, None] - X
    r = np.sqrt((e_minmax ** 2).mean()) / np.sqrt((e_mm ** 2).mean())
    assert 0.99 < r < 1.01
