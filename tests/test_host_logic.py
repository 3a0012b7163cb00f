"""Host-side logic of the mirror package that runs without a GPU: config
parsing, integrator specs and programs, inversion accounting tables."""

import numpy as np
import pytest

from paper_1512_03812_b200 import config as C
from paper_1512_03812_b200 import integrators as I


def test_spec_validation():
    with pytest.raises(ValueError):
        I.IntegratorSpec("newton", 0.1)
    with pytest.raises(ValueError):
        I.IntegratorSpec("leapfrog", -0.1)
    with pytest.raises(ValueError):
        I.IntegratorSpec("nested-fg", 0.1, micro_per_call=0)


def test_micro_step_resolution():
    # integrators.py:135-143 / test_integrators.py:50-55
    assert I.IntegratorSpec("nested-leapfrog", 0.1).micro_steps() == 10
    assert I.IntegratorSpec("nested-5stage", 0.1).micro_steps() == 5
    assert I.IntegratorSpec("adapted-nested-fg", 0.1, micro_ratio=20).micro_steps() == 10
    assert I.IntegratorSpec("nested-fg", 0.1, micro_per_call=7).micro_steps() == 7
    assert I.IntegratorSpec("leapfrog", 0.1).micro_steps() == 1


def test_eleven_stage_conditions():
    c1, c2 = I.fourth_order_defect(I.ELEVEN_SIGMA, I.ELEVEN_ETA, I.ELEVEN_LAM, I.ELEVEN_THETA)
    assert abs(c1) <= 1e-12 and abs(c2) <= 1e-12
    bad = I.fourth_order_defect(I.ELEVEN_SIGMA + 1e-3, I.ELEVEN_ETA, I.ELEVEN_LAM, I.ELEVEN_THETA)
    assert max(abs(bad[0]), abs(bad[1])) > 1e-6


def test_programs_are_palindromic_and_consistent():
    for name, prog in I.PROGRAMS.items():
        ops = [op for op, _ in prog]
        ws = [w(0.3) for _, w in prog]
        assert ops == ops[::-1], name
        assert np.allclose(ws, ws[::-1]), name
        kick_w = sum(w for op, w in zip(ops, ws) if op[0] in "KG")
        flow_w = sum(w for op, w in zip(ops, ws) if op[0] in "DI")
        assert np.isclose(kick_w, 0.3) and np.isclose(flow_w, 0.3), name


def test_inversion_table_matches_program_solves():
    # 2 inversions per chi/xi kick, +2 for the fermion FG piece, +4 for the
    # full FG kick (two Z pairs), +2 for the shifted force of fg-approx
    cost = {"K": 2, "Kf": 2, "Gfermion": 4, "Gfull": 6, "Gapprox": 4, "D": 0, "Ileapfrog": 0,
            "Ifg": 0}
    for name, prog in I.PROGRAMS.items():
        assert sum(cost[op] for op, _ in prog) == I.INVERSIONS_PER_STEP[name], name


def test_config_round_trip():
    cfg = C.HmcConfig(L=16, T=8, beta=2.0, m0=0.1, scheme="adapted-nested-fg", micro_per_call=2,
                      cg_tol=1e-10, fermion_bc="antiperiodic")
    again, plan = C.parse_experiment_file(C.format_config(cfg))
    assert again == cfg
    assert plan == C.SweepPlan()


def test_config_rejects_unknown_keys():
    with pytest.raises(ValueError):
        C.parse_experiment_file("L = 4\nbogus = 1\n")
    with pytest.raises(ValueError):
        C.parse_experiment_file("L = four\n")
    with pytest.raises(ValueError):
        C.HmcConfig(scheme="newton")
    with pytest.raises(ValueError):
        C.HmcConfig(fermion_bc="twisted")


def test_desk_scale():
    d = C.desk_scale(C.HmcConfig())
    assert (d.L, d.T, d.n_samples, d.n_thermalize) == (8, 8, 50, 200)


def test_captured_update_rejects_host_streams_before_touching_the_device():
    """EnsembleUpdateGraph needs the device-resident NumPy streams (checked
    before any CUDA work, so this runs without a GPU)."""
    import paper_1512_03812_b200 as sw
    cfg = sw.HmcConfig(L=8, T=8)
    with pytest.raises(TypeError):
        sw.EnsembleUpdateGraph(None, cfg, device_rng=object())


def test_dd_supports_every_reference_scheme():
    from paper_1512_03812_b200.dd_hmc import SUPPORTED
    from paper_1512_03812_b200.integrators import PROGRAMS, SCHEME_IDS
    assert set(SUPPORTED) == set(SCHEME_IDS)
    wired = {"D", "K", "Kf", "Gfermion", "Gfull", "Gapprox", "Ileapfrog", "Ifg"}
    for scheme in SCHEME_IDS:
        assert {name for name, _ in PROGRAMS[scheme]} <= wired, scheme


def test_bench_workload_labels_follow_the_workload():
    import importlib
    import sys
    sys.argv = ["bench.py", "--workload", "cfg4"]
    bench = importlib.import_module("bench")
    args = bench.parse()
    label = bench._phys_label(args.outer)
    assert label.startswith("64x64 chains") and "m0=0.02" in label and "8x4 steps" in label
    assert bench.CG_KERNELS["cfg4"]["kernel"].startswith("k_cg_cluster_tx")
    sys.argv = ["bench.py"]
    args = bench.parse()
    assert bench._phys_label(args.outer).startswith("16x16 chains")
