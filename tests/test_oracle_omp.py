"""The OpenMP build of the oracle (liboracle_omp.so: the same oracle.c with -fopenmp, used to
time the oracle on all host cores) is bit-identical to the sequential build: its pragmas
only split independent iterations (bags, segments, rows, key-range sort buckets).  Sizes are
chosen so the parallel dedup takes its key-range bucket path (>= 65536 occurrences)."""
import numpy as np
import pytest

import oracle as O
from workload import configs, gen


@pytest.mark.parametrize("mode", ["rowwise", "elementwise"])
def test_omp_oracle_bit_identical_to_sequential(mode):
    rows = [60_000, 9000, 700]
    ft = [0, 1, 0, 2]
    cfg = configs.Config("omp", rows, 16, [(t, ("range", 0, 40)) for t in ft], 4096, seed=61)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    ids, off = gen.make_batch(rows, cfg.features, B, cfg.seed, 0, alpha=1.05)
    assert len(ids) >= 65536
    grad = gen.grad_values(cfg.seed, 0, B, F, D, gen.grad_shift_for(len(ids), D))
    pb = O.Problem(rows, D, ft)
    W0 = np.concatenate([gen.table_rows(cfg.seed, t, np.arange(r), D) for t, r in enumerate(rows)])
    res = {}
    for par in (False, True):
        n = O.set_parallel(par, threads=4)
        assert n == (4 if par else 1)
        W = W0.copy()
        A = np.full(len(W) if mode == "rowwise" else W.shape, 0.1, dtype=np.float32)
        r = O.train_step(pb, W, A, ids, off, B, grad, 0.05, 1e-7, 1.0, mode=mode)
        keys, segs, bags = O.dedup(pb, ids, off, B)
        codes, mid, sc, _ = O.quantize(W)
        q, _ = O.forward_q8(pb, codes, mid, sc, ids, off, B)
        cm, mn, scm, _ = O.quantize_minmax(W)
        qm, _ = O.forward_q8_minmax(pb, cm, mn, scm, ids, off, B)
        res[par] = (r["out"], W, A, r["S"], keys, segs, bags, codes, mid, sc, q, cm, mn, scm, qm)
    O.set_parallel(False)
    for a, b in zip(res[False], res[True]):
        if isinstance(a, float):
            assert a == b
        else:
            assert np.array_equal(np.asarray(a), np.asarray(b))
