"""The seeded input generator (workload/): determinism, exactness, distribution sanity."""
import numpy as np

from workload import configs, gen


def test_splitmix64_reference_vector():
    # SplitMix64 (Steele, Lea & Flood 2014) from state 0: the first outputs are the
    # published sequence 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F.
    outs = [int(gen.mix64(np.array([np.uint64(n) * gen.GAMMA], dtype=np.uint64))[0]) for n in (1, 2, 3)]
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_table_values_exact_and_deterministic():
    a = gen.table_rows(1, 3, np.array([0, 5, 999_999_999]), 64)
    b = gen.table_rows(1, 3, np.array([0, 5, 999_999_999]), 64)
    assert (a == b).all() and a.dtype == np.float32
    # each value is an integer in [-2^23, 2^23) times 2^-26: exact in fp32
    s = a.astype(np.float64) * 2.0 ** 26
    assert (s == np.round(s)).all() and (np.abs(s) <= 2 ** 23).all()
    # row-addressable: drawing rows one by one equals drawing them together
    c = np.concatenate([gen.table_rows(1, 3, np.array([r]), 64) for r in (0, 5, 999_999_999)])
    assert (a == c).all()
    # different table -> different values
    assert not (gen.table_rows(1, 4, np.array([0]), 64) == a[:1]).all()


def test_table_values_roughly_normal():
    v = gen.table_rows(0, 0, np.arange(20000), 64).ravel().astype(np.float64)
    sigma = 2.0 ** 22 / np.sqrt(3) * 2.0 ** -26
    assert abs(v.mean()) < 1e-3 and abs(v.std() / sigma - 1) < 0.01


def test_grad_values_slicing():
    g = gen.grad_values(7, 2, 8, 3, 16, 30)
    g2 = gen.grad_values(7, 2, 4, 3, 16, 30, sample0=4)
    assert (g[4:] == g2).all()


def test_zipf_frequencies():
    rng = np.random.default_rng(0)
    n, s, size = 1000, 1.05, 400_000
    r = gen._zipf_rejection_inversion(rng, n, s, size)
    assert r.min() >= 1 and r.max() <= n
    p = np.arange(1, n + 1, dtype=np.float64) ** -s
    p /= p.sum()
    emp = np.bincount(r, minlength=n + 1)[1:] / size
    assert np.abs(emp[:10] - p[:10]).max() < 3e-3
    # uniform when alpha = 0
    u = gen._zipf_rejection_inversion(rng, 10, 0.0, 100000)
    assert abs(np.bincount(u)[1:].std() / 10000) < 0.05


def test_zipf_rows_bijection():
    rows = 997
    ranks = np.arange(1, rows + 1)
    mapped = ((ranks - 1) * gen.ROW_MULT + 977 * 3) % rows
    assert len(np.unique(mapped)) == rows


def test_make_batch_layout():
    cfg = configs.tiny()
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, cfg.batch, cfg.seed, 0)
    assert off[0] == 0 and off[-1] == len(ids) and len(off) == cfg.num_features * cfg.batch + 1
    assert (np.diff(off) >= 0).all() and (np.diff(off) == 0).any()  # empty bags occur
    assert ids.min() >= 0 and ids.max() < 10_000
    ids2, off2 = gen.make_batch(cfg.table_rows, cfg.features, cfg.batch, cfg.seed, 0)
    assert (ids == ids2).all() and (off == off2).all()


def test_config_shapes():
    # SURVEY.md §8(d) nnz per step
    assert abs(configs.feed1().expected_nnz() - 13.24e6) / 13.24e6 < 0.01
    assert abs(configs.ads().expected_nnz() - 49.8e6) / 49.8e6 < 0.01
    assert abs(configs.jobs().expected_nnz() - 8.52e6) / 8.52e6 < 0.01
    assert abs(configs.ads().total_rows - 100e6) / 100e6 < 1e-3
