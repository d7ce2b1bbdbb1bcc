"""TrainConfig semantics (train.hpp:23-49, train.cpp:76-85, 456-458) -- host only."""
import pytest

from paper_2505_13215_b200.train import TrainConfig


def test_defaults_mirror_reference():
    c = TrainConfig()
    assert (c.iterations, c.batch_size, c.warmup_iters, c.densify_interval, c.densify_stop_iter) == (2000, 2, 500,
                                                                                                     100, 1500)
    assert (c.tau, c.ssim_lambda, c.sh_degree, c.weight_cutoff, c.probe_interval) == (0.5, 0.2, 1, 0.05, 100)


@pytest.mark.parametrize("kw", [dict(iterations=10, warmup_iters=11), dict(densify_interval=0),
                                dict(ssim_lambda=1.5), dict(batch_size=0), dict(tau=0.0)])
def test_validate_rejects(kw):
    with pytest.raises(ValueError):
        TrainConfig(**kw).validate()


def test_densify_window():
    assert TrainConfig().densifies()
    assert not TrainConfig(iterations=300, warmup_iters=100, densify_stop_iter=0).densifies()
    assert not TrainConfig(iterations=300, warmup_iters=100, densify_stop_iter=99).densifies()
    assert TrainConfig(iterations=300, warmup_iters=100, densify_stop_iter=100).densifies()
    assert not TrainConfig(iterations=150, warmup_iters=101, densify_interval=100, densify_stop_iter=1500).densifies()
