"""NEXT-1 pins (CPU): the oracle's MurmurHash3 x64-128 id hashing and QR expansion
 against values fixed outside the oracle."""
import numpy as np
import pytest

import oracle as O



def test_murmur3_smhasher_verification_value():
    """SMHasher's published verification value for MurmurHash3_x64_128: hash keys
    {0}, {0,1}, ..., {0..254} (lengths 0..255) with seeds 256..1, concatenate the 256
    digests, hash that with seed 0; the first 4 bytes little-endian are 0x6384BA69.
    Covers every tail length 0..15, multi-block keys and non-zero seeds."""
    key = bytes(range(256))
    digests = bytearray()
    for i in range(256):
        h1, h2 = O.murmur3_x64_128(key[:i], 256 - i)
        digests += h1.to_bytes(8, "little") + h2.to_bytes(8, "little")
    f1, _ = O.murmur3_x64_128(bytes(digests), 0)
    assert int.from_bytes(f1.to_bytes(8, "little")[:4], "little") == 0x6384BA69


def test_murmur3_published_digests():
    # widely published digest of the pangram (seed 0), as the 16 output bytes
    h1, h2 = O.murmur3_x64_128(b"The quick brown fox jumps over the lazy dog", 0)
    assert (h1.to_bytes(8, "little") + h2.to_bytes(8, "little")).hex() == "6c1b07bc7bbc4be347939ac4a93c437a"
    # the empty string with seed 0 -> the all-zero digest (h1 = h2 = fmix64(0) = 0)
    assert O.murmur3_x64_128(b"", 0) == (0, 0)


def test_hash_id_is_h1_and_deterministic():
    ids = ["member:1234", "member:1235", "hashtag:#machinelearning", "", "é"]
    h = O.hash_ids(ids)
    for s, v in zip(ids, h):
        assert int(v) == O.murmur3_x64_128(s.encode("utf-8"), 0)[0]
    assert (O.hash_ids(ids) == h).all()


def test_no_collisions_over_a_million_sequential_member_ids():
    """10^6 sequential ids, zero 64-bit collisions expected (P:335
    "collision-resistant")."""
    h = O.hash_ids([f"member:{i}" for i in range(1_000_000)])
    assert len(np.unique(h)) == len(h)


def test_qr_paper_example():
    """a 4-billion vocabulary at 1000x compression -> ~4M quotient rows and ~1000
    remainder rows; R=1000, n=4_000_001 -> quotient 4000, remainder 1."""
    R = 1000
    Q = -(-(1 << 32) // R)  # ceil(2^32 / R): every 32-bit n has n / R < Q
    assert 4_000_000 < Q < 4_300_000
    ids, off = O.qr_expand(np.array([4_000_001], dtype=np.uint64), [0, 1], R, Q, dual=False)
    assert ids.tolist() == [4000, Q + 1] and off.tolist() == [0, 2]
    # the largest 32-bit n stays inside the quotient table without the mod
    ids, _ = O.qr_expand(np.array([(1 << 32) - 1], dtype=np.uint64), [0, 1], R, Q, dual=False)
    assert ids[0] == ((1 << 32) - 1) // R < Q and ids[1] == Q + ((1 << 32) - 1) % R
    assert O.qr_rows(R, Q, dual=False) == Q + R and O.qr_rows(R, Q, dual=True) == 2 * (Q + R)


def test_qr_dual_uses_both_int32_halves_with_independent_tables():
    """the int64 is bitcast to two int32-space numbers B and C that look up
    independent sets of QR tables.  Two hashes with the same low half and different high
    halves share the B rows and differ in the C rows; in single mode they collide
    completely."""
    R, Q = 7, 11
    lo = 123_456_789
    h = np.array([(5 << 32) | lo, (6 << 32) | lo], dtype=np.uint64)
    single, _ = O.qr_expand(h, [0, 2], R, Q, dual=False)
    assert single[0:2].tolist() == single[2:4].tolist()
    dual, off = O.qr_expand(h, [0, 2], R, Q, dual=True)
    assert off.tolist() == [0, 8]
    a, b = dual[0:4], dual[4:8]
    assert a[0:2].tolist() == b[0:2].tolist()      # B rows shared
    assert a[2:4].tolist() != b[2:4].tolist()      # C rows differ
    # each row lands in its own table of the concatenation [qB | rB | qC | rC]
    for r in (a, b):
        assert 0 <= r[0] < Q and Q <= r[1] < Q + R
        assert Q + R <= r[2] < 2 * Q + R and 2 * Q + R <= r[3] < 2 * (Q + R)
    # the quotient wraps modulo Q: n / R = 17636684 -> mod 11
    assert a[0] == (lo // R) % Q


def test_qr_sum_aggregation_is_pooling_over_the_expanded_bag():
    """P:335 "sum aggregation": the embedding of an id is quotient row + remainder row, so a
    SUM-pooled bag of L ids is the pooled sum over its 2L (4L) expanded rows; a single id
    gives exactly W[q] + W[r], and its gradient touches exactly 2 rows."""
    rng = np.random.default_rng(3)
    R, Q, D = 10, 50, 8
    rows = O.qr_rows(R, Q, dual=False)
    W = (rng.integers(-1000, 1000, size=(rows, D)) * 2.0 ** -10).astype(np.float32)
    h = np.array([987_654_321], dtype=np.uint64)
    ids, off = O.qr_expand(h, [0, 1], R, Q, dual=False)
    pb = O.Problem([rows], D, [0])
    out, _ = O.forward(pb, W, ids, off, 1)
    assert (out[0, 0] == W[ids[0]] + W[ids[1]]).all()
    # one training step: exactly the 2 expanded rows change; duplicates accumulate
    A = np.full(rows, 0.1, dtype=np.float32)
    W2 = W.copy()
    g = np.ones((1, 1, D), dtype=np.float32) * 0.25
    O.train_step(pb, W2, A, ids, off, 1, g, 0.05, 1e-7, 1e9)
    assert sorted(np.nonzero((W2 != W).any(axis=1))[0].tolist()) == sorted(ids.tolist())
    h2 = np.array([987_654_321, 987_654_321], dtype=np.uint64)
    ids2, off2 = O.qr_expand(h2, [0, 2], R, Q, dual=False)
    _, segs, _ = O.dedup(pb, ids2, off2, 1)
    assert np.diff(segs).tolist() == [2, 2]  # each of the 2 rows occurs twice
