"""Oracle vs the worked examples stored in tests/golden/*.json (each case cites the passage its
numbers come from: the paper, SPEC.md, SURVEY.md §8(c) or a published reference vector)."""
import json
import os

import numpy as np

import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_golden_quantize_middle_max():
    for c in load("quantize_middle_max.json")["cases"]:
        codes, mid, sc, bad = O.quantize(np.array([c["row"]], dtype=np.float32))
        assert bad == 0, c["cite"]
        assert abs(float(mid[0]) - c["middle"]) <= c["tol"] * max(1.0, abs(c["middle"])), c["cite"]
        assert abs(float(sc[0]) - c["scale"]) <= c["tol"], c["cite"]
        assert codes[0].tolist() == c["codes"], c["cite"]


def test_golden_clip_and_adagrad():
    g = load("clip_adagrad.json")
    for c in g["clip"]:
        G = np.array(c["grad"], dtype=np.float32)
        S = O.sq_norm(G)
        f, nf = O.clip_factor(S, 1.0)
        assert S == c["S"] and not nf and abs(float(f) - c["factor"]) < c["tol"], c["cite"]
        assert np.allclose(O.clip(G, f), c["clipped"], atol=c["tol"]), c["cite"]
    for c in g["adagrad_single_row"]:
        W = np.array([c["w"]], dtype=np.float32)
        A = np.full((1, 2) if c["mode"] == "elementwise" else (1,), 0.1, dtype=np.float32)
        G = np.array([c["g"]], dtype=np.float32)
        f, _ = O.clip_factor(O.sq_norm(G), 1.0)
        O.adagrad(W, A, [0], O.clip(G, f), 0.1, 1e-7, c["mode"])
        assert np.allclose(W[0], c["w_new"], rtol=c["tol_rel"], atol=0), c["cite"]
        if "A_new" in c:
            assert abs(float(A[0]) - c["A_new"]) < 1e-7, c["cite"]


def test_golden_murmur_and_qr():
    g = load("qr_murmur.json")
    for c in g["murmur3_x64_128"]:
        if "verification" in c:
            key = bytes(range(256))
            dig = bytearray()
            for i in range(256):
                h1, h2 = O.murmur3_x64_128(key[:i], 256 - i)
                dig += h1.to_bytes(8, "little") + h2.to_bytes(8, "little")
            f1, _ = O.murmur3_x64_128(bytes(dig), 0)
            assert int.from_bytes(f1.to_bytes(8, "little")[:4], "little") == c["verification"], c["cite"]
        else:
            h1, h2 = O.murmur3_x64_128(c["key"].encode("utf-8"), 0)
            assert (h1.to_bytes(8, "little") + h2.to_bytes(8, "little")).hex() == c["digest_hex"], c["cite"]
    for c in g["qr"]:
        Q = -(-(1 << 32) // c["R"])
        ids, _ = O.qr_expand(np.array([c["n"]], dtype=np.uint64), [0, 1], c["R"], Q, dual=False)
        assert ids.tolist() == [c["quotient"], Q + c["remainder"]], c["cite"]


def test_golden_incremental():
    g = load("incremental.json")
    for c in g["cold_init"]:
        for alpha, exp in c["cases"]:
            got = O.cold_weight_init(np.array(c["w0"], np.float32), np.array(c["w1"], np.float32), alpha)
            assert got.tolist() == exp, c["cite"]
    for c in g["penalty"]:
        w = O.cold_weight_init(np.array(c["w0"], np.float32), np.array(c["w1"], np.float32), c["alpha"])
        assert w.tolist() == c["w"], c["cite"]
        one = np.ones(1, np.float32)
        lam = 1.0
        p = O.fim_penalty(w, np.array(c["w0"], np.float32), one, np.array(c["w1"], np.float32), one, lam, c["alpha"])
        assert abs(p - c["penalty_over_lambda"] * lam) < 1e-12, c["cite"]
