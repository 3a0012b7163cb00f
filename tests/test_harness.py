"""Experiment harness (§8(f) row 3): host logic on CPU with a fake
measurement (the reference's fault-injection pattern,
pkg/tests/test_config_cli.py:194-215), and one GPU sweep checked cell by
cell against the oracle's measure_dh."""

import csv
import math
from types import SimpleNamespace

import numpy as np
import pytest
from click.testing import CliRunner

from paper_1512_03812_b200 import harness as H


def read_csv(path):
    rows, comments = [], []
    with open(path) as fh:
        for line in fh:
            (comments if line.startswith("#") else rows).append(line.rstrip("\n"))
    return [r.split(",") for r in rows], comments


def test_loglog_slope_and_cost_interpolation():
    hs = [0.05, 0.1, 0.2]
    assert abs(H.loglog_slope([(h, 3 * h**2) for h in hs]) - 2.0) < 1e-12
    assert abs(H.loglog_slope([(h, h**4) for h in hs] + [(0.3, float("nan"))]) - 4.0) < 1e-12
    assert math.isnan(H.loglog_slope([(0.1, 1.0)]))
    pts = [(0.1, 1e-2, 100), (0.2, 1e-1, 50)]
    assert abs(H.cost_at_accuracy(pts, 1e-2) - 100) < 1e-9
    mid = H.cost_at_accuracy(pts, math.sqrt(1e-3))
    assert abs(mid - math.sqrt(100 * 50)) < 1e-9
    assert H.cost_at_accuracy(pts, 1e-4) is None


def test_bisect_step():
    fake = lambda h: SimpleNamespace(acceptance=1.0 - h)
    h, m = H.bisect_step(fake, 0.01, 0.4, 0.9)
    assert abs(m.acceptance - 0.9) <= 0.02 and abs(h - 0.1) <= 0.02
    h, ms = H.bisect_step(fake, 0.2, 0.4, 0.9)
    assert h is None and ms[0].acceptance == 0.8


@pytest.fixture
def experiment(tmp_path):
    from paper_1512_03812_b200.lattice import save_gauge_config
    rng = np.random.default_rng(1)
    gauge = tmp_path / "g.cfg"
    save_gauge_config(gauge, 0.3 * rng.standard_normal((2, 4, 4)), 1.0, 0.1, 7)
    exp = tmp_path / "exp.cfg"
    exp.write_text(f"L = 4\nT = 4\nbeta = 1.0\nm0 = 0.1\ntau = 0.5\ncg_tol = 1e-10\n"
                   f"n_samples = 4\nschemes = leapfrog, adapted-nested-fg\nh_grid = 0.125, 0.25\n"
                   f"micro_per_call = 2\ngauge_config = {gauge}\n")
    return tmp_path, exp


def fake_cell(q0, config, scheme, h, stream):
    from paper_1512_03812_b200.fermion import SolverError
    if scheme == "leapfrog" and h == 0.25:
        raise SolverError("injected failure", 0.5)
    mean = h**2 if scheme == "leapfrog" else h**4
    return SimpleNamespace(mean_abs=mean, stderr=0.1 * mean, acceptance=0.95, wall_per_traj=0.0,
                           inversions_per_traj=int(round(0.5 / h)) * H.INVERSIONS_PER_STEP[scheme])


def test_sweep_records_failures_and_continues(experiment, monkeypatch):
    tmp, exp = experiment
    monkeypatch.setattr(H, "measure_cell", fake_cell)
    out = tmp / "dh.csv"
    res = CliRunner().invoke(H.main, ["sweep-dh", "--config", str(exp), "--out", str(out)])
    assert res.exit_code == 0, res.output
    rows, comments = read_csv(out)
    assert rows[0] == H.CSV_HEADER and len(rows) == 1 + 4
    nan_rows = [r for r in rows[1:] if r[3] == "nan"]
    assert len(nan_rows) == 1 and nan_rows[0][0] == "leapfrog"
    assert any(c.startswith("# failed,leapfrog") for c in comments)
    assert any(c.startswith("# slope,adapted-nested-fg,4.000") for c in comments)
    m_col = {r[0]: r[2] for r in rows[1:]}
    assert m_col["leapfrog"] == "0" and m_col["adapted-nested-fg"] == "2"


def test_bench_cost_ranking_footer(experiment, monkeypatch):
    tmp, exp = experiment
    monkeypatch.setattr(H, "measure_cell", lambda *a: fake_cell(*a[:3], 0.125 if a[3] == 0.125 else 0.2, a[4]))
    out = tmp / "cost.csv"
    res = CliRunner().invoke(H.main, ["bench-cost", "--config", str(exp), "--out", str(out)])
    assert res.exit_code == 0, res.output
    rows, comments = read_csv(out)
    assert len(rows) == 5 and any(c.startswith("# rank at |dH|=") for c in comments)


def test_missing_gauge_and_bad_config(tmp_path):
    exp = tmp_path / "x.cfg"
    exp.write_text("L = 4\nT = 4\n")
    res = CliRunner().invoke(H.main, ["sweep-dh", "--config", str(exp)])
    assert res.exit_code != 0 and "gauge_config" in res.output
    bad = tmp_path / "bad.cfg"
    bad.write_text("turbo = on\n")
    assert CliRunner().invoke(H.main, ["sweep-dh", "--config", str(bad)]).exit_code != 0


@pytest.mark.gpu
def test_gpu_sweep_matches_oracle_cells(experiment):
    """Every cell of a GPU sweep equals the oracle's measure_dh on the same
    stream (idx*1000 + jdx)."""
    from oracle import schwinger_oracle as O
    tmp, exp = experiment
    out = tmp / "dh.csv"
    res = CliRunner().invoke(H.main, ["sweep-dh", "--config", str(exp), "--out", str(out)])
    assert res.exit_code == 0, res.output
    rows, _ = read_csv(out)
    q0, meta = O.load_gauge_config(tmp / "g.cfg")
    for r in rows[1:]:
        scheme, h = r[0], float(r[1])
        i = ("leapfrog", "adapted-nested-fg").index(scheme)
        j = (0.125, 0.25).index(h)
        cfg = O.Config(L=4, T=4, beta=1.0, m0=0.1, tau=0.5, h=h, scheme=scheme, micro_per_call=2,
                       cg_tol=1e-10, seed=20160905, n_samples=4)
        m = O.measure_dh(q0, cfg, O.make_rng(cfg.seed, i * 1000 + j))
        assert abs(float(r[3]) - m["mean_abs"]) <= 1e-8 + 1e-6 * m["mean_abs"]
        assert int(r[6]) == m["inversions_per_traj"]


def test_tune_acceptance_treats_cg_cap_as_rejection(experiment, monkeypatch):
    """A cell whose CG hits the cap (a wild trajectory at large h) counts as
    acceptance 0 in the bisection instead of aborting the tuning run."""
    from paper_1512_03812_b200.fermion import SolverError
    tmp, exp = experiment

    def cell(q0, config, scheme, h, stream):
        if h > 0.3:
            raise SolverError("injected cap", 1e-9)
        return SimpleNamespace(mean_abs=h**2, stderr=0.0, acceptance=1.0 - h, wall_per_traj=0.0,
                               inversions_per_traj=8)

    monkeypatch.setattr(H, "measure_cell", cell)
    text = exp.read_text() + "h_min = 0.01\nh_max = 0.5\n"
    exp.write_text(text)
    out = tmp / "tune.csv"
    res = CliRunner().invoke(H.main, ["tune-acceptance", "--config", str(exp), "--out", str(out)])
    assert res.exit_code == 0, res.output
    rows, _ = read_csv(out)
    assert len(rows) == 1 + 2
    for r in rows[1:]:
        assert abs(float(r[8]) - 0.9) <= 0.02


def test_load_setup_precedence(tmp_path):
    """cli.py:32-46: defaults shrink to desk scale unless --paper-scale; the
    experiment file replaces the defaults; --paper-scale, --seed and
    --micro-ratio override either."""
    from paper_1512_03812_b200.config import HmcConfig, desk_scale
    cfg, plan = H.load_setup(None, None, False, None)
    assert cfg == desk_scale(HmcConfig())
    cfg, _ = H.load_setup(None, 7, True, 12.5)
    assert (cfg.L, cfg.T, cfg.n_samples, cfg.seed, cfg.micro_ratio) == (32, 32, 200, 7, 12.5)
    exp = tmp_path / "e.cfg"
    exp.write_text("L = 8\nT = 8\nbeta = 1.5\nschemes = leapfrog\n")
    cfg, plan = H.load_setup(str(exp), None, False, None)
    assert (cfg.L, cfg.beta, plan.schemes) == (8, 1.5, ("leapfrog",))
    cfg, _ = H.load_setup(str(exp), 3, True, None)
    assert (cfg.L, cfg.beta, cfg.seed, cfg.n_samples) == (32, 1.5, 3, 200)
