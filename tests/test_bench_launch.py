"""bench.py's multi-GPU launch contract: `python bench.py --gpus N` outside
torchrun starts N ranks itself (torch.distributed.run on 127.0.0.1), a
launcher whose WORLD_SIZE disagrees with --gpus is refused, and the
ensemble total is split across the ranks (strong scaling) unless --weak."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _run(args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=timeout)


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_gpus_2_spawns_two_ranks_reference_arm():
    """--impl reference under the self-launched world of 2: rank 0 runs the CPU
    reference path and prints the one line with n_gpus 2; rank 1 exits 0."""
    r = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
              "--outer", "2"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = _line(r.stdout)
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["cpu_baseline"]["kind"] == "port" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_world_size_mismatch_is_refused():
    r = _run(["--impl", "reference", "--gpus", "4", "--steps", "1", "--warmup", "0"],
             env_extra={"WORLD_SIZE": "2", "RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("weak", [False, True])
def test_gpus_2_ensemble_bench_splits_the_chains(weak):
    """The GPU arm at --gpus 2 (gloo for the control plane; both ranks share the
    pool's one GPU, their kernels never wait on each other): n_gpus 2 and the
    whole-ensemble chain count, strong by default, weak with --weak."""
    args = ["--gpus", "2", "--chains", "64", "--steps", "2", "--warmup", "3", "--no-cpu",
            "--no-stencil", "--no-e2e", "--no-compare"] + (["--weak"] if weak else [])
    r = _run(args, env_extra={"SCH_DIST_BACKEND": "gloo", "SCH_NO_CLOCKS": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    line = _line(r.stdout)
    assert line["n_gpus"] == 2
    assert line["scaling"] == ("weak" if weak else "strong")
    assert line["config"]["global_chains"] == (128 if weak else 64)
    assert line["config"]["chains_per_gpu"] == (64 if weak else 32)
    assert line["value"] > 0 and line["roofline"]["bound"] == "fp64"


@pytest.mark.gpu
def test_bench_line_contract():
    """The single-GPU bench line carries every key of the driver's contract
    (bench.py docstring / task contract): metric, value, unit, n_gpus,
    steps, warmup, ms_per_step, higher_is_better, scaling, vs_baseline,
    dtype, data, config.workload, roofline {bound, achieved, peak, unit,
    frac, traffic}, e2e {value, unit, h2d/d2h bytes}, gpu_launches, clocks."""
    r = _run(["--steps", "3", "--warmup", "3", "--no-cpu", "--no-stencil", "--no-compare"])
    assert r.returncode == 0, r.stderr[-3000:]
    line = _line(r.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "e2e", "gpu_launches", "clocks"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert "workload" in line["config"]
    roof = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in roof, k
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])
