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


def test_config_file_parsing_and_validation(tmp_path):
    """test_train.cpp:235-272"""
    import pytest

    from paper_2505_13215_b200.dataset import FormatError
    from paper_2505_13215_b200.train import TrainConfig

    good = tmp_path / "good.txt"
    good.write_text("# training settings\niterations = 500\nbatch_size = 3\nwarmup_iters = 100\ntau = 0.25\n"
                    "lr_mean = 2e-4\nconversion_enabled = false\nseed = 18446744073709551615\n")
    cfg = TrainConfig.from_file(str(good))
    assert (cfg.iterations, cfg.batch_size, cfg.tau, cfg.lrs.mean) == (500, 3, 0.25, 2e-4)
    assert cfg.conversion_enabled is False and cfg.densify_interval == 100 and cfg.seed == 2**64 - 1
    for body in ("iterations = 10\nlr_typo = 1\n", "iterations = 10\niterations = 20\n",
                 "conversion_enabled = yes\n", "iterations = ten\n", "seed = -1\n"):
        p = tmp_path / "bad.txt"
        p.write_text(body)
        with pytest.raises(FormatError):
            TrainConfig.from_file(str(p))
    p = tmp_path / "invalid.txt"
    p.write_text("iterations = 10\nwarmup_iters = 50\n")
    with pytest.raises(ValueError):
        TrainConfig.from_file(str(p))


def test_train_log_csv(tmp_path):
    """TrainLog::write_csv (train.cpp:122-129): a parseable csv (test_train.cpp:309)"""
    import csv

    from paper_2505_13215_b200.train import TrainLogRow, write_train_log_csv

    rows = [TrainLogRow(iter=1, loss=0.25, probe_psnr=-1.0, n_static=10, n_dynamic=20, conversions=0,
                        wall_seconds=0.5),
            TrainLogRow(iter=2, loss=0.125, probe_psnr=21.5, n_static=12, n_dynamic=18, conversions=2,
                        wall_seconds=1.0)]
    p = str(tmp_path / "log.csv")
    write_train_log_csv(rows, p)
    got = list(csv.DictReader(open(p)))
    assert [int(r["iter"]) for r in got] == [1, 2] and float(got[1]["probe_psnr"]) == 21.5
    assert list(got[0]) == ["iter", "loss", "probe_psnr", "n_static", "n_dynamic", "conversions", "wall_seconds"]


def test_metric_report_aggregates_means():
    """test_metrics.cpp:180-190 (MetricReport::add, metrics.cpp:109-120)"""
    from paper_2505_13215_b200.train import MetricReport

    r = MetricReport()
    for p, s in ((20.0, 0.5), (30.0, 0.7), (25.0, 0.9)):
        r.add(p, s)
    assert r.frames == 3 and r.mean_psnr == 25.0 and abs(r.mean_ssim - 0.7) < 1e-15
    assert r.frame_psnr == [20.0, 30.0, 25.0]
