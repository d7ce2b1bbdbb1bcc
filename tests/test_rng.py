"""The product's batch-sampling RNG (paper_2505_13215_b200/rng.py) against the
oracle's libstdc++ std::mt19937_64 / uniform_int_distribution<size_t> draws
(train.cpp:387-404): the training loop must draw the reference's (camera,
frame) schedule for the same seed."""
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
