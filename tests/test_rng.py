"""The product's batch-sampling RNG (paper_2505_13215_b200/rng.py) against the
oracle's libstdc++ std::mt19937_64 / uniform_int_distribution<size_t> draws
(train.cpp:387-404): the training loop must draw the reference's (camera,
frame) schedule for the same seed."""
import numpy as np
import oracle as O
from paper_2505_13215_b200.rng import MT19937_64, uniform_index


def test_mt19937_64_raw_stream():
    for seed in (0, 1, 5489, 2**63 + 12345):
        ref, ours = O.Rng(seed), MT19937_64(seed)
        assert [ours() for _ in range(1000)] == [ref.raw() for _ in range(1000)]


def test_uniform_index_matches_libstdcxx():
    for seed, n in ((0, 1), (3, 2), (7, 18), (11, 300), (13, 5400), (17, 2**40 + 3), (19, 2**63 + 5)):
        ref, ours = O.Rng(seed), MT19937_64(seed)
        for _ in range(500):
            assert uniform_index(ours, 0, n - 1) == ref.index(0, n - 1)


def test_normal_distribution_matches_libstdcxx():
    """std::normal_distribution<double> (Marsaglia polar, cached second
    variate) drawn from one object, as the dynamics pool of densify does."""
    from paper_2505_13215_b200.rng import NormalDistribution

    for seed in (0, 7, 123456789):
        ref = O.Rng(seed).normal_seq(1001)
        g, nd = MT19937_64(seed), NormalDistribution()
        ours = [nd(g) for _ in range(1001)]
        assert ours == ref.tolist()


def test_fresh_distribution_per_call_matches_oracle_normal():
    """hgso_rng_normal draws from a fresh distribution each call (like
    sample_normal3's per-call object): the cached variate is discarded."""
    from paper_2505_13215_b200.rng import NormalDistribution

    ref, g = O.Rng(99), MT19937_64(99)
    for _ in range(200):
        assert NormalDistribution()(g) == ref.normal()


def test_native_stream_matches_python_and_oracle():
    """hgs_rng (libstdc++ in the product library) == rng.py == the oracle."""
    from paper_2505_13215_b200.api import Rng
    from paper_2505_13215_b200.rng import densify_normals

    a, b, c = Rng(2024), MT19937_64(2024), O.Rng(2024)
    for _ in range(50):
        assert a.raw() == b() == c.raw()
    for lo, hi in [(0, 9), (0, 1), (3, 3), (0, 2**40 + 7), (5, 2**64 - 1)]:
        assert a.index(lo, hi) == uniform_index(b, lo, hi) == c.index(lo, hi)
    picks = a.batch(5400, 8)
    assert picks == [uniform_index(b, 0, 5399) for _ in range(8)]
    for _ in range(8):
        c.index(0, 5399)
    rng = np.random.default_rng(0)
    k3 = rng.integers(1, 3, 37).astype(np.uint8)
    k4 = rng.integers(1, 3, 53).astype(np.uint8)
    n3a, n4a = a.densify_normals(k3, k4)
    n3b, n4b = densify_normals(b, k3.tolist(), k4.tolist())
    assert np.array_equal(n3a, n3b) and np.array_equal(n4a, n4b)
    assert a.raw() == b()  # the streams stay aligned after the draws


def test_sample_batches_is_the_reference_schedule():
    from paper_2505_13215_b200.train import sample_batches

    g = MT19937_64(7)
    want = [[uniform_index(g, 0, 99) for _ in range(3)] for _ in range(5)]
    assert sample_batches(100, 3, 5, 7) == want
