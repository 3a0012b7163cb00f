#!/usr/bin/env python
"""Benchmark: HMC chain-trajectories/s of the Schwinger-model ensemble on B200.

Workload (BASELINE.json configs[2], "cfg3"): independent 16x16 chains,
beta=2.0, m0=0.1, tau=1, adapted nested force-gradient (the paper's scheme),
micro_per_call=2, CG tolerance 1e-10, complex128, hot start; 8192 chains in
the ensemble, split across the ranks (strong scaling, configs[2]; --weak keeps
--chains per GPU), no collective on the data path, one NCCL all-gather of
per-chain dH/accept at the end.  A "step" is one full HMC update of every
chain (heatbaths, H, trajectory, H, Metropolis).  `--gpus N` outside torchrun
starts the N ranks itself (torch.distributed.run, 127.0.0.1).

Also reported on the same line:
  roofline   : the dominant kernel (the resident per-chain CG) against the
               FP64 roofline (SMs x 128 flop/clk x max clock) on the SURVEY
               §8(d) algorithmic model (152 flop per site per CG iteration),
               with a live FP64 FMA probe beside it; its working set lives in
               registers/shared memory, so the 352 B/site/iteration streaming
               model's HBM rate is only a secondary "hbm_effective" field;
  stencil    : BASELINE configs[1] ("cfg2"): 4096 x 32^2, fused D^dag D GB/s at
               96 B/site and the streaming CG to 1e-10 at 352 B/site/iteration;
  cpu_baseline: the CPU oracle port (per-chain hmc_update) on the host cores;
  e2e        : the same metric through the public API with the links copied
               host->device and device->host every step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_PATH = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0

# The dominant kernel of each ensemble workload, and the DRAM bytes per
# lattice site of one of its launches measured by ncu --set full (U and b
# in, x out — the solve itself stays on chip):
#   cfg3: profiles/r02/ncu_full_k_cg_resblk_r02.txt, 134.322688 MB read +
#         36.037888 MB written for 8192 chains x 256 sites (x leaves partly
#         through L2 after the kernel ends); FP64 pipe 65.5 % active
#   cfg4: profiles/r02/ncu_cluster_tx.txt, 269.755648 MB read + 103.136512 MB
#         written for 1024 chains x 4096 sites (b is re-read by the
#         true-residual checks; part of it misses L2); FP64 pipe 37.4 % active
DRAM_CFG4 = (269.755648e6 + 103.136512e6) / (1024 * 4096)   # profiles/r02/ncu_cluster_tx.txt
CG_KERNELS = {
    "cfg3": dict(kernel="k_cg_resblk<16,16,2x2 sites/thread,t-faces by warp shuffle,"
                        "sigma1-diagonal spin basis> (per-chain CG, one 64-thread CTA per chain, "
                        "4 CTAs/SM)",
                 dram_per_site=(134.322688e6 + 36.037888e6) / (8192 * 256),
                 fp64_pipe_active=0.655,
                 source="profiles/r02/ncu_full_k_cg_resblk_r02.txt"),
    "cfg3_mega": dict(kernel="k_traj_anfg16 (trajectory megakernel: one 64-thread CTA per 16x16 "
                             "chain runs H(start), the 17 resident-CG solves, forces, FG terms, "
                             "inner leapfrogs and H(end) of the adapted-nested-fg trajectory)",
                      dram_per_site=None, fp64_pipe_active=None,
                      source="profiles/r01/ncu_full_k_traj_anfg16.txt"),
    "cfg4": dict(kernel="k_cg_cluster_tx<64,64,4 CTAs,2x2 sites/thread> (per-chain CG, one "
                        "4-CTA cluster per chain, faces and partial sums pushed with st.async "
                        "onto the receiver's mbarrier)",
                 dram_per_site=DRAM_CFG4,
                 fp64_pipe_active=0.374,
                 source="profiles/r02/ncu_cluster_tx.txt"),
}

CFG3 = dict(L=16, T=16, beta=2.0, m0=0.1, tau=1.0, scheme="adapted-nested-fg", micro_per_call=2,
            cg_tol=1e-10)

# BASELINE.json configs[2] (the bench line) and configs[3] (light fermions)
WORKLOADS = {
    "cfg3": dict(chains=8192, outer=4, phys=CFG3),
    "cfg4": dict(chains=1024, outer=8,
                 phys=dict(L=64, T=64, beta=4.0, m0=0.02, tau=1.0, scheme="adapted-nested-fg",
                           micro_per_call=4, cg_tol=1e-10)),
    "cfg5": dict(chains=1, outer=10,
                 phys=dict(L=2048, T=2048, beta=8.0, m0=0.05, tau=0.5, scheme="adapted-nested-fg",
                           micro_per_call=2, cg_tol=1e-10)),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg3",
                    help="cfg3 (default, the bench line) or cfg4 (64^2 light-fermion ensemble)")
    ap.add_argument("--chains", type=int, default=None,
                    help="the ensemble total, split across the ranks (strong scaling, the "
                         "default: BASELINE configs[2] reads '8192 chains sharded across "
                         "1/2/4/8 GPUs', configs[3] '1024 chains ... sharded across 8 GPUs'); "
                         "with --weak: chains per GPU")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: --chains per GPU, the ensemble grows with the ranks")
    ap.add_argument("--therm", type=int, default=0,
                    help="untimed updates before the warm-up (a thermalized start; cfg4's CG "
                         "iterations grow as its chains order)")
    ap.add_argument("--outer", type=int, default=None, help="outer (fermion) steps per trajectory")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-stencil", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-compare", action="store_true",
                    help="skip the cfg3 integrator comparison (five schemes at ~90%% acceptance)")
    ap.add_argument("--graph", choices=("auto", "on", "off"), default="auto",
                    help="replay each ensemble update as one captured CUDA graph (auto/on: "
                         "whenever one stream issues the ensemble and the megakernel is off; "
                         "off: eager issue, two updates queued ahead)")
    ap.add_argument("--streams", type=int, default=1,
                    help="sub-ensembles issued concurrently on separate streams (measured "
                         "slower than 1 on cfg3: 2 -> -6 %%, profiles/r01/README.md)")
    ap.add_argument("--strips", type=int, default=1, help="cfg5: strips on one GPU (local transport)")
    ap.add_argument("--cfg5-size", type=int, default=2048)
    ap.add_argument("--transport", choices=("local", "nccl", "p2p"), default=None,
                    help="cfg5 halo/sum transport (default: nccl under torchrun, else local)")
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    if args.chains is None:
        args.chains = w["chains"]
    if args.outer is None:
        args.outer = w["outer"]
    global CFG3
    CFG3 = dict(w["phys"])
    return args


def peaks():
    try:
        d = json.loads(PEAKS_PATH.read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


# ---------------------------------------------------------------------------
# CPU oracle leg (cpu_baseline and --impl reference): per-chain unbatched
# hmc_update of the CPU port, one process per host core.
# ---------------------------------------------------------------------------

def _cpu_cfg(outer):
    from oracle import schwinger_oracle as O
    return O.Config(h=1.0 / outer, **CFG3)


def _cpu_chain_worker(args):
    seed, stream, seconds, outer = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import schwinger_oracle as O
    cfg = _cpu_cfg(outer)
    rng = O.make_rng(seed, stream)
    q = O.hot_start(rng, cfg.L, cfg.T)
    n, t0 = 0, time.perf_counter()
    while True:
        q, _ = O.hmc_update(q, cfg, rng)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            return n, el


def _cpu_one_traj(args):
    seed, stream, outer = args
    from oracle import schwinger_oracle as O
    cfg = _cpu_cfg(outer)
    rng = O.make_rng(seed, stream)
    q = O.hot_start(rng, cfg.L, cfg.T)
    t0 = time.perf_counter()
    O.hmc_update(q, cfg, rng)
    return time.perf_counter() - t0


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _phys_label(outer):
    c = CFG3
    return (f"{c['L']}x{c['T']} chains, beta={c['beta']}, m0={c['m0']}, tau={c['tau']}, "
            f"{c['scheme']} {outer}x{c['micro_per_call']} steps, tol {c['cg_tol']:g}")


def _cpu_batched_worker(args):
    """Best-case CPU: the reference's batched measure_dh (fixed start, global
    CG stop, no Metropolis) on `n` samples per process, repeated for ~seconds."""
    seed, n, seconds, outer = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import schwinger_oracle as O
    cfg = _cpu_cfg(outer)
    q = O.hot_start(O.make_rng(seed, 0), cfg.L, cfg.T)
    done, t0, k = 0, time.perf_counter(), 0
    while True:
        O.measure_dh(q, cfg, O.make_rng(seed, 1 + k), n)
        done += n
        k += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            return done, el


def cpu_baseline(seconds, outer):
    cores = cpu_cores()
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        res = pool.map(_cpu_chain_worker, [(1234, c, seconds, outer) for c in range(cores)])
        best = pool.map(_cpu_batched_worker, [(4321 + c, 32, min(seconds, 10.0), outer)
                                              for c in range(cores)])
    n = sum(r[0] for r in res)
    rate = sum(r[0] / r[1] for r in res)
    batched = {"value": sum(r[0] / r[1] for r in best), "unit": "chain-trajectories/s",
               "sample": f"{sum(r[0] for r in best)} trajectories as batched measure_dh "
                         f"(32 samples per call, fixed start, global CG stop, no Metropolis), "
                         f"{cores} processes: the reference's best-case batched CPU path"}
    return {"value": rate, "unit": "chain-trajectories/s", "cores": cores, "kind": "port",
            "batched_best_case": batched,
            "sample": f"{n} unbatched hmc_update trajectories of independent hot-start "
                      f"{_phys_label(outer)}, {cores} processes x {seconds:.0f}s, "
                      "oracle/schwinger_oracle.py"}


def _cpu_cg_iter_worker(args):
    """Seconds per CG iteration of the CPU port on one L x L lattice (one
    core): repeated capped cg_normal calls for ~seconds."""
    L, m0, seconds, seed = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import schwinger_oracle as O
    rng = O.make_rng(seed, 0)
    U = O.fermion_links(O.hot_start(rng, L, L))
    psi = rng.standard_normal((L, L, 2)) + 1j * rng.standard_normal((L, L, 2))
    n, t0 = 0, time.perf_counter()
    while True:
        try:
            O.cg_normal(U, m0, psi, 1e-30, maxiter=10)
        except O.OracleSolverError:
            pass
        n += 10
        el = time.perf_counter() - t0
        if el >= seconds:
            return n, el


def cpu_cg_rate(L, m0, seconds):
    """SURVEY 8(d)(ii) for a workload whose CPU trajectory outlasts the
    bench's budget (cfg4: a 64^2 light-fermion trajectory is minutes on one
    core): every host core times the port's CG iteration; the trajectory
    rate is extrapolated with the GPU run's CG iterations per trajectory
    (finish_cpu_cg_rate).  The CG is >= 98 % of the CPU trajectory (SURVEY
    8(a) a7), so this slightly favours the CPU."""
    cores = cpu_cores()
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_cpu_cg_iter_worker, [(L, m0, seconds, 99 + c) for c in range(cores)])
    n = sum(r[0] for r in res)
    per_core_rate = sum(r[0] / r[1] for r in res) / cores
    return {"s_per_cg_iteration_per_core": 1.0 / per_core_rate, "cores": cores, "kind": "port",
            "cg_iterations_timed": n, "L": L}


def finish_cpu_cg_rate(rate, iters_per_chain_traj):
    if rate is None:
        return None
    per_traj = rate["s_per_cg_iteration_per_core"] * iters_per_chain_traj
    return {"value": rate["cores"] / per_traj, "unit": "chain-trajectories/s",
            "cores": rate["cores"], "kind": "port",
            "s_per_cg_iteration_per_core": rate["s_per_cg_iteration_per_core"],
            "sample": f"{rate['cg_iterations_timed']} CG iterations of the port "
                      f"(oracle/schwinger_oracle.py cg_normal) on hot-start {rate['L']}x"
                      f"{rate['L']} lattices, {rate['cores']} processes; chain-trajectories/s "
                      f"extrapolated = cores / (s per iteration x {iters_per_chain_traj:.0f} CG "
                      "iterations per chain-trajectory of this GPU run) — an extrapolation, "
                      "forces and kicks (< 2 % on CPU) not counted"}


# BASELINE.json configs[0] ("cfg1"): the reference's own CPU run, one chain
CFG1 = dict(L=16, T=16, beta=2.0, m0=0.1, tau=1.0, h=0.2, scheme="adapted-nested-fg",
            micro_per_call=2, cg_tol=1e-10)


def _cpu_cfg1_worker(n_traj):
    """cfg1 exactly as the reference runs it: hot_start(make_rng(0, 0)), then
    hmc_update on the same generator, one core."""
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import schwinger_oracle as O
    cfg = O.Config(**CFG1)
    rng = O.make_rng(0, 0)
    q = O.hot_start(rng, cfg.L, cfg.T)
    t0 = time.perf_counter()
    for _ in range(n_traj):
        q, _ = O.hmc_update(q, cfg, rng)
    return (time.perf_counter() - t0) / n_traj


def cpu_cfg1(n_traj=3):
    with mp.get_context("fork").Pool(1) as pool:
        sec = pool.apply(_cpu_cfg1_worker, (n_traj,))
    return {"s_per_trajectory": sec, "cores": 1, "kind": "port",
            "sample": f"first {n_traj} of cfg1's 20 trajectories (oracle/schwinger_oracle.py)"}


def _cpu_stencil_worker(args):
    """Oracle D^dag D on a slice of cfg2 (B_slice x 32^2) for ~seconds."""
    seed, nb, seconds = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import schwinger_oracle as O
    rng = np.random.default_rng(seed)
    q = rng.uniform(-np.pi, np.pi, size=(nb, 2, 32, 32))
    U = np.exp(1j * q)
    psi = rng.standard_normal((nb, 32, 32, 2)) + 1j * rng.standard_normal((nb, 32, 32, 2))
    n, t0 = 0, time.perf_counter()
    while True:
        O.normal_op(U, psi, 0.1)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            return n * nb * 32 * 32, el


def cpu_stencil_baseline(seconds):
    cores = cpu_cores()
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        res = pool.map(_cpu_stencil_worker, [(c, 16, seconds) for c in range(cores)])
    gbs = sum(96.0 * sites / el for sites, el in res) / 1e9
    return {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "port",
            "sample": f"oracle normal_op (NumPy, batched) on 16 x 32x32 lattices per process, "
                      f"{cores} processes x {seconds:.0f}s, 96 B/site"}


def run_reference(args):
    """--impl reference: the CPU port of the reference path on all host cores."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    cores = cpu_cores()
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(cores) as pool:
        for step in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(_cpu_one_traj, [(99, step * cores + c, args.outer) for c in range(cores)])
            if step >= args.warmup:
                times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    value = cores / t
    line = {
        "impl": "reference", "metric": "HMC trajectories/s", "value": value,
        "unit": "chain-trajectories/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64/c128", "data": "synthetic",
        "config": {"workload": f"{args.workload}: independent {_phys_label(args.outer)}, "
                               "hot start",
                   "chains_per_step": cores},
        "cpu_baseline": {"value": value, "unit": "chain-trajectories/s", "cores": cores,
                         "kind": "port",
                         "sample": f"each step: {cores} processes x 1 unbatched hmc_update "
                                   "trajectory (oracle/schwinger_oracle.py; the reference is "
                                   "pure Python, so the port is the runnable reference path)"},
        "e2e": {"value": value, "unit": "chain-trajectories/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.window = None

    def mark(self, t0, t1):
        """Wall-clock bounds of the timed region: only samples inside count."""
        self.window = (t0, t1)

    def start(self):
        if os.environ.get("SCH_NO_CLOCKS"):
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            if self.window is not None:
                try:   # e.g. "2026/10/20 10:42:16.123" (local time)
                    stamp, frac = parts[0].rsplit(".", 1)
                    ts = time.mktime(time.strptime(stamp, "%Y/%m/%d %H:%M:%S")) + float("0." + frac)
                    if not self.window[0] - 0.25 <= ts <= self.window[1] + 0.25:
                        continue
                except ValueError:
                    pass
            parts = parts[1:]
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nme, val in zip(names, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(nme)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def fp64_probe(torch, _lib):
    blocks, iters = 148 * 16, 4096
    scratch = torch.empty((blocks,), dtype=torch.float64, device="cuda")
    ctx = _lib.ctx()
    ctx.call("sch_probe_fp64", _lib.ptr(scratch), blocks, 64)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.call("sch_probe_fp64", _lib.ptr(scratch), blocks, iters)
        e1.record()
        torch.cuda.synchronize()
        flops = blocks * 256.0 * iters * 64
        best = max(best, flops / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def fp64_peak_theoretical(torch):
    """FP64 peak of the device: SMs x 64 FP64 FMA lanes x 2 flop x the max SM
    clock (MEASURED_PEAKS.json's sm_max_mhz; B200: 148 x 128 x 1.965 GHz =
    37.2 TFLOP/s).  FP64 is not in MEASURED_PEAKS.json, so this is the
    datasheet-class arithmetic peak; the live FMA probe is reported beside it."""
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    try:
        mhz = float(json.loads(PEAKS_PATH.read_text())["sm_max_mhz"])
        kind = "theoretical: SMs x 64 FP64 FMA/clk x 2 x sm_max_mhz (MEASURED_PEAKS.json)"
    except Exception:
        mhz = 1965.0
        kind = "theoretical: SMs x 64 FP64 FMA/clk x 2 x 1965 MHz (B200 max SM clock)"
    return sms * 128.0 * mhz * 1e6 / 1e12, kind


def stencil_bench(torch, sw, _lib, hbm_peak):
    """cfg2: 4096 x 32^2, fused D^dag D and the CG to 1e-10."""
    from paper_1512_03812_b200 import fermion as F
    B, L = 4096, 32
    V = L * L
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2)
    q = (torch.rand((B, 2, L, L), dtype=torch.float64, device="cuda", generator=gen) * 2 - 1) * math.pi
    psi = torch.randn((B, L, L, 2), dtype=torch.complex128, device="cuda", generator=gen)
    op = sw.WilsonDirac(q, 0.1)
    out = op.normal(psi)
    ctx = _lib.ctx()
    for _ in range(10):     # warm-up (inputs + U + output = 402 MB > L2: every rep streams HBM)
        ctx.call("sch_ddagd", _lib.ptr(op.U), _lib.ptr(psi), _lib.ptr(out), B, L, L, 0.1)
    torch.cuda.synchronize()
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):   # the C-ABI call itself, output preallocated
        ctx.call("sch_ddagd", _lib.ptr(op.U), _lib.ptr(psi), _lib.ptr(out), B, L, L, 0.1)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    sites = B * V
    ddd_gbs = 96.0 * sites / t / 1e9
    res = {"workload": "cfg2: 4096 x 32x32, m0=0.1, complex128",
           "ddagd": {"achieved": ddd_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": ddd_gbs / hbm_peak, "us_per_application": t * 1e6,
                     "bytes_model": "96 B/site (psi in + U + out)",
                     "kernel": "k_normal_tma<8,32,PLAIN,128 thr,2 stages,3 CTA/SM> "
                               "(persistent, cp.async.bulk + mbarrier pipeline)"}}
    # CG, both engines (an untimed short solve first loads every kernel)
    for mode, label in (("per_chain", "resident"), ("batch_global", "streaming")):
        F.cg_solve(op, psi, 1e-10, maxiter=60, stop=mode)
        torch.cuda.synchronize()
        F.CG_PROFILE = []
        x, info = F.cg_solve(op, psi, 1e-10, stop=mode)
        torch.cuda.synchronize()
        prof, F.CG_PROFILE = F.CG_PROFILE, None
        ev0, ev1, iters, vv = prof[0]
        ms = ev0.elapsed_time(ev1)
        tot_it = int(iters.sum().item()) if mode == "per_chain" else int(iters.max().item()) * B
        gbs = 352.0 * vv * tot_it / (ms * 1e-3) / 1e9
        res[f"cg_{label}"] = {"stop": mode, "ms": ms, "iterations_max": int(iters.max().item()),
                              "iterations_mean": float(iters.double().mean().item()),
                              "achieved": gbs, "unit": "GB/s", "frac": gbs / hbm_peak,
                              "bytes_model": "352 B/site/iteration",
                              "effective": label == "resident"}
        rel = float(info.relres_dev.max().item())
        res[f"cg_{label}"]["max_rel_residual"] = rel
    del q, psi, out, op, x
    torch.cuda.empty_cache()
    return res


def cfg1_bench(torch, sw, cpu=None, n_traj=20):
    """BASELINE configs[0] on the GPU: the single chain of the reference's CPU
    run (hot start from make_rng(0, 0), 20 trajectories, h = 0.2), each
    update one replay of a captured CUDA graph; beside the CPU port's
    seconds per trajectory on one core."""
    cfg = sw.HmcConfig(**CFG1)
    d = sw.NumpyDeviceRng(seed=0, n_chains=1, stream0=0)
    q = d.hot_start(sw.LatticeGeom(cfg.L, cfg.T))
    upd = sw.EnsembleUpdateGraph(q, cfg, d)
    upd.step()   # capture + first trajectory (untimed)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n_traj):
        upd.step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n_traj
    out = {"workload": "cfg1: one 16x16 chain, beta=2, m0=0.1, adapted-nested-fg 5x2 (h=0.2), "
                       "tol 1e-10, hot start make_rng(0, 0)",
           "gpu_ms_per_trajectory": ms, "trajectories": n_traj}
    if cpu is not None:
        out["cpu"] = cpu
        out["speedup_vs_1_core"] = cpu["s_per_trajectory"] * 1e3 / ms
    return out


def graph_bench(torch, sw, reps=10):
    """Small ensembles are launch-bound: one HMC update (cfg3 physics) per
    step eagerly vs replayed as one captured CUDA graph (EnsembleUpdateGraph)."""
    cfg = sw.HmcConfig(h=0.25, **{k: v for k, v in CFG3.items()})
    geom = sw.LatticeGeom(cfg.L, cfg.T)
    out = {"workload": f"cfg3 physics ({cfg.L}x{cfg.T}, adapted-nested-fg 4x2), one update per step"}
    if cfg.L * cfg.T > 1024:
        return None
    for B in (1, 64):
        d = sw.NumpyDeviceRng(seed=5, n_chains=B)
        q = d.hot_start(geom)
        for _ in range(2):
            q, _ = sw.hmc_update_ensemble(q, cfg, device_rng=d)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            q, p = sw.hmc_update_ensemble_async(q, cfg, d)
        e1.record()
        torch.cuda.synchronize()
        eager = e0.elapsed_time(e1) / reps
        upd = sw.EnsembleUpdateGraph(q, cfg, d)
        upd.step()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            upd.step()
        e1.record()
        torch.cuda.synchronize()
        graph = e0.elapsed_time(e1) / reps
        out[f"B{B}"] = {"eager_ms_per_update": eager, "graph_ms_per_update": graph,
                        "speedup": eager / graph}
    return out


# BASELINE.json configs[2]: the five schemes it names ("Omelyan 2MN" is the
# reference's 5stage, "force-gradient" its 5stage-fg) with the smallest outer
# step count reaching ~90 % acceptance; ladder starts from SURVEY 8(d)'s
# CPU estimates minus a margin.
COMPARE_SCHEMES = (("leapfrog", 6), ("5stage", 3), ("5stage-fg", 2), ("nested-fg", 2),
                   ("adapted-nested-fg", 2))
COMPARE_TARGET = 0.90


def force_evals_per_step(scheme):
    """Fermion-force evaluations per macro step as the reference executes the
    program (integrators.py:278-349, no merging of adjacent kicks): a kick
    is one force, an FG kick a force plus a force-gradient term (two)."""
    from paper_1512_03812_b200.integrators import PROGRAMS
    n = 0
    for name, _ in PROGRAMS[scheme]:
        if name in ("K", "Kf"):
            n += 1
        elif name.startswith("G"):
            n += 2
    return n


def integrator_comparison(torch, sw, F, q0, drng, reps=2, max_tries=8):
    """cfg3's integrator comparison on the bench ensemble: for every scheme,
    the smallest outer step count n (h = tau/n) whose acceptance over the
    whole ensemble from the common start q0 reaches COMPARE_TARGET, then
    `reps` timed updates at that n (CUDA events).  Reports chain-traj/s,
    reference-convention inversions, actual CG solves and CG iterations per
    chain-trajectory, and force evaluations per trajectory."""
    from paper_1512_03812_b200.integrators import INVERSIONS_PER_STEP
    chains = q0.shape[0]
    out = {"target_acceptance": COMPARE_TARGET, "chains": chains,
           "start_avg_plaquette": float(sw.avg_plaquette(q0).mean().item()),
           "micro_per_call": CFG3["micro_per_call"], "schemes": {}}
    for scheme, n0 in COMPARE_SCHEMES:
        ladder = []
        n = n0
        for _ in range(max_tries):
            cfg = sw.HmcConfig(h=1.0 / n, **{**CFG3, "scheme": scheme})
            _, pend = sw.hmc_update_ensemble_async(q0, cfg, drng)
            acc = float(pend.resolve().accepted.mean())
            ladder.append([n, acc])
            if acc >= COMPARE_TARGET:
                break
            n += 1
        cfg = sw.HmcConfig(h=1.0 / n, **{**CFG3, "scheme": scheme})
        torch.cuda.synchronize()
        F.CG_PROFILE = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q, pends = q0, []
        e0.record()
        for _ in range(reps):
            q, pend = sw.hmc_update_ensemble_async(q, cfg, drng)
            pends.append(pend)
        e1.record()
        torch.cuda.synchronize()
        sts = [p.resolve() for p in pends]
        prof, F.CG_PROFILE = F.CG_PROFILE, None
        ms = e0.elapsed_time(e1) / reps
        iters = sum(int(it.sum().item()) for _, _, it, _ in prof)
        out["schemes"][scheme] = {
            "n_steps": n, "h": 1.0 / n, "acceptance_ladder": ladder,
            "acceptance": float(np.mean([st.accepted.mean() for st in sts])),
            "chain_traj_per_s": chains / (ms * 1e-3), "ms_per_update": ms,
            "inversions_per_traj_reference_convention": INVERSIONS_PER_STEP[scheme] * n,
            "force_evals_per_traj": force_evals_per_step(scheme) * n,
            "cg_solves_per_traj": len(prof) / reps,
            "cg_iterations_per_chain_traj": iters / (chains * reps)}
    return out


def megakernel_leg(torch, sw, q0, drng, cfg, per_gpu_value, reps=3):
    """the same update through the opt-in trajectory
    megakernel (csrc/mega.cu, one launch for H, the trajectory and H),
    timed beside the kernel-per-map path of the bench line."""
    if not (cfg.scheme == "adapted-nested-fg" and cfg.L == 16 and cfg.T == 16):
        return None
    sw.hmc.USE_MEGA = True
    try:
        q, _ = sw.hmc_update_ensemble(q0, cfg, device_rng=drng)   # warm-up (workspace, attributes)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pends = []
        for _ in range(reps):
            q, p = sw.hmc_update_ensemble_async(q, cfg, drng)
            pends.append(p)
        e1.record()
        torch.cuda.synchronize()
        for p in pends:
            p.resolve()
    finally:
        sw.hmc.USE_MEGA = False
    v = q0.shape[0] / (e0.elapsed_time(e1) / reps * 1e-3)
    return {"kernel": "k_traj_anfg16", "chain_traj_per_s": v, "vs_kernel_per_map": v / per_gpu_value,
            "note": "opt-in (SCH_MEGA=1): equal results; its inlined solver loop compiles "
                    "~10 % longer than k_cg_resblk's (DESIGN.md)"}


def _device_for(local, torch):
    """One GPU per rank.  SCH_DIST_BACKEND=gloo (control-flow tests of the
    multi-rank bench on a 1-GPU box) maps ranks onto the visible devices."""
    if os.environ.get("SCH_DIST_BACKEND") == "gloo":
        return local % torch.cuda.device_count()
    return local


def _max_over_ranks(dist, torch, v):
    """Max of a host float over all ranks (device tensor on NCCL, host on gloo)."""
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _init_dist(dist, torch, local):
    backend = os.environ.get("SCH_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    hbm_peak, peak_kind = peaks()

    cpu = cpu_stencil = cpu1 = None
    cpu_rate = None
    if rank == 0 and world == 1 and not args.no_cpu and args.workload == "cfg4":
        ph = WORKLOADS["cfg4"]["phys"]
        cpu_rate = cpu_cg_rate(ph["L"], ph["m0"], args.cpu_seconds)   # before CUDA init
    elif rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.cpu_seconds, args.outer)   # before CUDA init (fork-safe)
        if not args.no_stencil:
            cpu_stencil = cpu_stencil_baseline(min(args.cpu_seconds, 5.0))
            if args.workload == "cfg3":
                cpu1 = cpu_cfg1()

    local = _device_for(local, torch)
    torch.cuda.set_device(local)
    if world > 1:
        _init_dist(dist, torch, local)
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200 import _lib
    from paper_1512_03812_b200 import fermion as F

    def barrier():
        if world > 1:
            dist.barrier()

    stencil = None
    if rank == 0 and not args.no_stencil:   # fresh allocator / caches
        stencil = stencil_bench(torch, sw, _lib, hbm_peak)
        if cpu_stencil is not None:
            stencil["ddagd"]["cpu_baseline"] = cpu_stencil

    from paper_1512_03812_b200.ensemble import gather_observables, shard_chains, summarize
    # strong scaling (default): the ensemble total fixed; --weak: chains per GPU fixed
    shard = shard_chains(args.chains * world if args.weak else args.chains, world, rank)
    chains = shard.count
    cfg = sw.HmcConfig(h=1.0 / args.outer, **CFG3)
    geom = sw.LatticeGeom(cfg.L, cfg.T)
    # chain c draws exactly the reference's make_rng(2024, c) stream, on device:
    # hot start first, then every trajectory's heatbaths and Metropolis draw
    # The shard can be issued as S contiguous sub-ensembles on S streams (each
    # with its own library context) so their kernels interleave on the GPU.
    # Chain c keeps stream c: results do not depend on S.  Default S=1: the
    # small kernels then squeeze resident-CG CTAs off the SMs and the step
    # gets slower (S=2: 164.5k -> 154.3k chain-traj/s).
    S = max(1, min(args.streams, chains))
    subs = [shard_chains(chains, S, i) for i in range(S)]
    main = torch.cuda.current_stream()
    streams = [torch.cuda.Stream() for _ in range(S)] if S > 1 else [main]
    drngs, qs = [], []
    for sub, stm in zip(subs, streams):
        stm.wait_stream(main)
        with torch.cuda.stream(stm):
            d = sw.NumpyDeviceRng(seed=2024, n_chains=sub.count, stream0=shard.start + sub.start)
            drngs.append(d)
            qs.append(d.hot_start(geom))

    def issue_step(qs):
        pend = []
        for i, stm in enumerate(streams):
            stm.wait_stream(main)
            with torch.cuda.stream(stm):
                qs[i], p = sw.hmc_update_ensemble_async(qs[i], cfg, drngs[i])
                pend.append(p)
        for stm in streams:
            main.wait_stream(stm)
        return pend

    def run_steps(n, on_stats=None, ahead=2):
        """n updates with `ahead` steps queued: step k+ahead is issued before
        step k's per-chain results are read back, so a host-side stall (the
        box shows occasional 10-120 ms ones, tools/step_jitter.py) is
        absorbed by the queued GPU work instead of idling the GPU."""
        queue, sts = [], None
        for _ in range(n):
            queue.append(issue_step(qs))
            if len(queue) > ahead:
                sts = [p.resolve() for p in queue.pop(0)]
                if on_stats:
                    on_stats(sts)
        while queue:
            sts = [p.resolve() for p in queue.pop(0)]
            if on_stats:
                on_stats(sts)
        return sts

    # The host only issues work; a Python garbage-collector pass in the middle
    # of a step stalls the issue thread for ~20 ms and starves the GPU
    # (tools/step_jitter.py), so collect once here and keep it off while timing.
    gc.collect()
    gc.disable()
    # an optional thermalization, then the warm-up in the timed region's own
    # pattern (steps queued ahead), so the caching allocator already holds the
    # buffers of every in-flight step
    sts = run_steps(args.therm + args.warmup)
    torch.cuda.synchronize()

    # One captured CUDA graph per update (EnsembleUpdateGraph) instead of
    # ~100 launches issued from Python: 1024 chains (the 8-GPU share) 141-142k
    # -> 152-154k chain-traj/s, 8192 chains 192.6-192.8k -> 194.0-194.2k, and
    # host stalls no longer reach the GPU (profiles/r02/README.md).  The CG
    # launches' events inside the graph are external event nodes, so the
    # roofline below reads the CG time and iterations of the last timed replay.
    mega_on = args.workload == "cfg3" and sw.hmc._mega_eligible(cfg, True)
    use_graph = S == 1 and not mega_on and args.graph in ("auto", "on")
    upd = graph_prof = None
    if use_graph:
        graph_prof = []
        upd = sw.EnsembleUpdateGraph(qs[0], cfg, drngs[0], cg_profile=graph_prof)
        upd.step()
        upd.stats()          # one untimed replay
        torch.cuda.synchronize()

    def run_graph_steps(n, on_stats=None, ahead=2):
        """run_steps for the graph: each replay's per-chain dH / accept copied
        out (the graph's buffers are rewritten by the next replay) and read
        back `ahead` replays later."""
        from types import SimpleNamespace
        queue, sts = [], None

        def resolve(item):
            dh, acc = item[0].cpu().numpy(), item[1].cpu().numpy()
            if int(item[2].item()):
                raise F.SolverError("a CG solve of the replayed update hit its cap", float("nan"))
            if (acc < 0).any():
                raise ValueError(f"non-finite energy change {dh[acc < 0][0]}")
            return [SimpleNamespace(dh=dh, accepted=acc == 1, inversions=upd.inversions)]
        for _ in range(n):
            dh, acc = upd.step()
            queue.append((dh.clone(), acc.clone(), upd.failed.clone()))
            if len(queue) > ahead:
                sts = resolve(queue.pop(0))
                if on_stats:
                    on_stats(sts)
        while queue:
            sts = resolve(queue.pop(0))
            if on_stats:
                on_stats(sts)
        return sts

    clocks = ClockSampler(local)
    # nvidia-smi's own start-up (NVML init) contends with this process's
    # launches: start it before the timed region and keep only its samples
    # from inside the region (ClockSampler.mark)
    clocks.start()
    time.sleep(0.75)
    barrier()
    torch.cuda.synchronize()
    t_wall0 = time.time()
    F.CG_PROFILE = []
    launches0 = _lib.launch_count()
    acc, dhs = [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    def record(sts):
        acc.append(np.concatenate([st.accepted for st in sts]))
        dhs.append(np.concatenate([st.dh for st in sts]))

    sts = run_graph_steps(args.steps, record) if use_graph else run_steps(args.steps, record)
    st = sts[0]
    e1.record()
    torch.cuda.synchronize()
    barrier()
    launches = _lib.launch_count() - launches0
    if use_graph:   # replays launch no kernels from the host: count the captured ones
        upd.stats()   # CG-cap / non-finite check of the last replay
        launches = upd.launches_per_replay * args.steps
        qs[0] = upd.q.clone()
    clocks.mark(t_wall0, time.time())
    clk = clocks.stop()
    prof, F.CG_PROFILE = F.CG_PROFILE, None
    prof_steps = 1 if use_graph else args.steps   # steps the CG events / iteration counts cover
    if use_graph:
        prof = graph_prof
    ms = e0.elapsed_time(e1)
    if world > 1:
        ms = _max_over_ranks(dist, torch, ms)
    ms_step = ms / args.steps
    value = shard.total / (ms_step * 1e-3)   # all ranks' chain-trajectories per step

    # dominant kernel: the resident CG (one launch per solve).  Its time is
    # the union of the CG launch intervals (they overlap across streams), so
    # achieved = CG bytes / time during which a CG kernel was running.
    spans = sorted((e0.elapsed_time(a), e0.elapsed_time(b)) for a, b, _, _ in prof)
    cg_ms, cur = 0.0, None
    for a0, b0 in spans:
        if cur is None or a0 > cur[1]:
            if cur is not None:
                cg_ms += cur[1] - cur[0]
            cur = [a0, b0]
        else:
            cur[1] = max(cur[1], b0)
    if cur is not None:
        cg_ms += cur[1] - cur[0]
    cg_iters = sum(int(it.sum().item()) for _, _, it, _ in prof)
    if prof_steps != args.steps:   # graph: the last replay stands for every timed step
        scale = args.steps / prof_steps
        cg_ms, cg_iters = cg_ms * scale, int(round(cg_iters * scale))
    V = cfg.L * cfg.T
    n_solves = len(prof) * (args.steps // prof_steps)   # CG launches in the timed region
    mega = args.workload == "cfg3" and sw.hmc._mega_eligible(cfg, True)
    kinfo = CG_KERNELS["cfg3_mega" if mega else args.workload]
    cg_bytes = 352.0 * V * cg_iters
    cg_flops = 152.0 * V * cg_iters
    achieved = cg_bytes / (cg_ms * 1e-3) / 1e9
    fp64_probe_peak = fp64_probe(torch, _lib)
    fp64_peak, fp64_kind = fp64_peak_theoretical(torch)
    fp64_achieved = cg_flops / (cg_ms * 1e-3) / 1e12
    # the megakernel runs every solve of a trajectory in one launch: 1 + 4n
    solves_per_traj = (1 + 4 * max(1, round(cfg.tau / cfg.h))) if mega else n_solves / args.steps

    # ensemble observables: one NCCL all-gather at the end (the only collective)
    obs = gather_observables({"dh": np.concatenate(dhs),
                              "accepted": np.concatenate(acc).astype(np.float64)},
                             shard_chains(shard.total * args.steps, world, rank))
    ens = summarize(obs)
    acc_rate = ens["acceptance"]

    # e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e and use_graph:
        # The same contract with the update as graph replays (public API:
        # EnsembleUpdateGraph): two captured graphs, one per in-flight step,
        # each with its own link buffer (they share the chains' RNG state).
        # Step k uploads the host links into graph k%2's buffer on a copy
        # stream, replays it, and downloads its new links and per-chain
        # dH / accept into pinned host memory; the host reads step k-1's
        # after issuing step k.
        q_host = qs[0].cpu().pin_memory()
        q_back = torch.empty_like(q_host).pin_memory()
        h2d = q_host.numel() * 8
        steps_e2e = max(4, args.steps)
        upds = [upd] + [sw.EnsembleUpdateGraph(qs[0], cfg, drngs[0])]
        dh_host = [torch.empty((chains,), dtype=torch.float64).pin_memory() for _ in range(2)]
        acc_host = [torch.empty((chains,), dtype=torch.int32).pin_memory() for _ in range(2)]
        fail_host = [torch.empty((), dtype=torch.int32).pin_memory() for _ in range(2)]
        cp = torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]   # slot's results downloaded
        ev_done = [torch.cuda.Event() for _ in range(2)]
        for slot in range(2):
            ev_out[slot].record(main)
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        cp.wait_stream(main)

        def upload(slot):
            with torch.cuda.stream(cp):
                cp.wait_event(ev_out[slot])   # the slot's previous step is downloaded
                upds[slot].q.copy_(q_host, non_blocking=True)
                ev_in[slot].record(cp)

        def read(k):
            slot = k % 2
            ev_out[slot].synchronize()
            if int(fail_host[slot].item()):
                raise F.SolverError("a CG solve of the replayed update hit its cap", float("nan"))
            if (acc_host[slot].numpy() < 0).any():
                raise ValueError("non-finite energy change")

        upload(0)
        for k in range(steps_e2e):
            slot = k % 2
            if k + 1 < steps_e2e:
                upload(1 - slot)
            main.wait_event(ev_in[slot])
            dh_dev, acc_dev = upds[slot].step()
            ev_done[slot].record(main)
            with torch.cuda.stream(cp):
                cp.wait_event(ev_done[slot])
                q_back.copy_(upds[slot].q, non_blocking=True)
                dh_host[slot].copy_(dh_dev, non_blocking=True)
                acc_host[slot].copy_(acc_dev, non_blocking=True)
                fail_host[slot].copy_(upds[slot].failed, non_blocking=True)
                ev_out[slot].record(cp)
            if k >= 1:   # step k-1's dH / accept (its slot is not rewritten before
                read(k - 1)   # step k+1 is issued), read while step k is queued
        read(steps_e2e - 1)
        main.wait_stream(cp)
        f1.record()
        torch.cuda.synchronize()
        barrier()
        ems = f0.elapsed_time(f1)
        if world > 1:
            ems = _max_over_ranks(dist, torch, ems)
        d2h = q_back.numel() * 8 + chains * (8 + 4)
        e2e = {"value": shard.total / (ems / steps_e2e * 1e-3), "unit": "chain-trajectories/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": ems / steps_e2e,
               "issue": "EnsembleUpdateGraph replays, host links in / out every step"}
    elif not args.no_e2e:
        # Every step is one public-API call on HOST links: H2D of the links,
        # the update, D2H of the new links and of the per-chain dH / accept.
        # Copies run on a copy stream, double-buffered, so step k+1's upload
        # and step k's download overlap the neighbouring step's compute (a
        # pipelined client; every byte still crosses PCIe inside the window).
        # The host reads step k-2's results after issuing step k (two steps
        # queued, as the device-timed leg), so a host stall does not idle the GPU.
        q_host = [qi.cpu().pin_memory() for qi in qs]
        q_back = [torch.empty_like(h).pin_memory() for h in q_host]
        h2d = sum(h.numel() for h in q_host) * 8
        steps_e2e = max(4, args.steps)
        copy = [torch.cuda.Stream() for _ in streams]
        din = [[torch.empty_like(qi) for _ in range(2)] for qi in qs]
        ev_in = [[torch.cuda.Event() for _ in range(2)] for _ in qs]
        ev_free = [[torch.cuda.Event() for _ in range(2)] for _ in qs]
        for i in range(S):
            for slot in range(2):
                ev_free[i][slot].record(main)

        def upload(i, slot):
            with torch.cuda.stream(copy[i]):
                copy[i].wait_event(ev_free[i][slot])
                din[i][slot].copy_(q_host[i], non_blocking=True)
                ev_in[i][slot].record(copy[i])

        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for i in range(S):
            copy[i].wait_stream(main)
            upload(i, 0)
        queued = []   # per step: the pendings of its chains' dH / accept
        for k in range(steps_e2e):
            slot = k % 2
            pend = []
            for i, stm in enumerate(streams):
                if k + 1 < steps_e2e:
                    upload(i, 1 - slot)
                with torch.cuda.stream(stm):
                    stm.wait_event(ev_in[i][slot])
                    out, p = sw.hmc_update_ensemble_async(din[i][slot], cfg, drngs[i])
                    ev_free[i][slot].record(stm)
                    done = torch.cuda.Event()
                    done.record(stm)
                with torch.cuda.stream(copy[i]):
                    copy[i].wait_event(done)
                    out.record_stream(copy[i])
                    q_back[i].copy_(out, non_blocking=True)
                pend.append(p)
            queued.append(pend)
            if len(queued) > 2:   # step k-2's dH / accept, read while k-1 and k are queued
                for p in queued.pop(0):
                    p.resolve()
        for pend in queued:
            for p in pend:
                p.resolve()
        for i, stm in enumerate(streams):
            main.wait_stream(stm)
            main.wait_stream(copy[i])
        f1.record()
        torch.cuda.synchronize()
        barrier()
        ems = f0.elapsed_time(f1)
        if world > 1:
            ems = _max_over_ranks(dist, torch, ems)
        d2h = sum(b.numel() for b in q_back) * 8 + chains * (8 + 4)
        e2e = {"value": shard.total / (ems / steps_e2e * 1e-3), "unit": "chain-trajectories/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": ems / steps_e2e}

    gc.enable()
    graphs = compare = single = None
    if rank == 0 and not args.no_stencil:
        graphs = graph_bench(torch, sw)
        if args.workload == "cfg3":
            single = cfg1_bench(torch, sw, cpu1)
    mega_leg = None
    if rank == 0 and not args.no_compare and S == 1:
        compare = integrator_comparison(torch, sw, F, qs[0], drngs[0])
        if args.workload == "cfg3" and not sw.hmc.USE_MEGA:
            mega_leg = megakernel_leg(torch, sw, qs[0], drngs[0], cfg, value / world)

    if cpu_rate is not None:
        cpu = finish_cpu_cg_rate(cpu_rate, cg_iters / (chains * args.steps))
    if rank == 0:
        line = {
            "metric": "HMC trajectories/s", "value": value, "unit": "chain-trajectories/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None,
            "dtype": "f64/c128",
            "data": "synthetic: hot start + heatbaths drawn on device from the reference's own "
                    "streams (chain c == make_rng(2024, c), value-identical NumPy Philox/ziggurat)",
            "config": {"workload": f"{args.workload}: independent {cfg.L}x{cfg.T} chains, "
                                   f"beta={cfg.beta}, m0={cfg.m0}, tau={cfg.tau}, adapted-nested-fg "
                                   f"{args.outer}x{cfg.micro_per_call} steps (h={1.0 / args.outer}), "
                                   "CG tol 1e-10 per-chain stop, complex128",
                       "chains_per_gpu": chains, "global_chains": shard.total,
                       "parallelism": f"chain-ensemble dp{world}",
                       "l2": "working set > L2 (126 MB); no flush needed",
                       "acceptance": acc_rate, "mean_abs_dh": ens["mean_abs_dh"],
                       "exp_minus_dh": ens["exp_minus_dh"],
                       "cg_solves_per_traj": solves_per_traj,
                       "inversions_per_traj_reference_convention": st.inversions,
                       "cg_iterations_per_chain_traj": cg_iters / (chains * args.steps),
                       "cg_iterations_per_solve": cg_iters / max(1, chains * n_solves),
                       "therm_updates_before_warmup": args.therm,
                       "update_issue": ("one CUDA-graph replay per update; the CG time and "
                                        "iterations are the last timed replay's (external "
                                        "event nodes) x steps") if use_graph else
                                       "eager, two updates queued ahead"},
            "roofline": {"bound": "fp64", "achieved": fp64_achieved, "peak": fp64_peak,
                         "unit": "TFLOP/s", "frac": fp64_achieved / fp64_peak,
                         "traffic": (None if kinfo["dram_per_site"] is None
                                     else kinfo["dram_per_site"] * V * chains),
                         "traffic_unit": "bytes per launch",
                         "traffic_source": "dram__bytes_read.sum+dram__bytes_write.sum of one "
                                           f"launch (ncu --set full, {kinfo['source']}), per "
                                           "site, x sites of one launch here",
                         "kernel": kinfo["kernel"],
                         "flops_model": "152 flop/site/CG-iteration (SURVEY 8(d): 112 D^dag D + "
                                        f"40 dots/axpys), {V} sites x {cg_iters} "
                                        "chain-iterations, / the union of the CG launch intervals "
                                        "(CUDA events on the launching stream)",
                         "algorithmic_flops_per_launch": cg_flops / max(1, n_solves),
                         "peak_kind": fp64_kind,
                         "fp64_peak_probe": fp64_probe_peak,
                         "frac_of_probe": fp64_achieved / fp64_probe_peak,
                         "fp64_pipe_active_ncu": kinfo["fp64_pipe_active"],
                         "note": "the solve's working set lives in registers and shared memory, "
                                 "so FP64 issue, not HBM, bounds it; the achieved rate counts the "
                                 "152-flop model, while the kernel issues ~96 FP64 instructions "
                                 "per site-iteration (sigma1-diagonal spin basis): ncu's FP64 "
                                 "pipe-active fraction is the issue-rate measure" + (
                                     "; the megakernel's time also holds its non-CG phases "
                                     "(forces, FG terms, inner leapfrogs, H)" if mega else ""),
                         "kernel_share_of_step": cg_ms / ms,
                         "hbm_effective": {"achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                                           "frac": achieved / hbm_peak, "peak_kind": peak_kind,
                                           "bytes_model": "352 B/site/CG-iteration (SURVEY 8(d) "
                                                          "streaming model)",
                                           "algorithmic_bytes_per_launch":
                                               cg_bytes / max(1, n_solves),
                                           "note": "a streaming-model rate, not a roofline "
                                                   "fraction: the solve does not stream HBM"}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "stencil": stencil,
            "graph_capture": graphs,
            "integrators": compare,
            "cfg1_single_chain": single,
            "megakernel": mega_leg,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _cpu_cfg5_worker(L):
    """one oracle D^dag D on the whole L x L lattice and five
    CG iterations (one core); the trajectory is extrapolated from them."""
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import schwinger_oracle as O
    rng = np.random.default_rng(5)
    U = O.fermion_links(rng.uniform(-np.pi, np.pi, (2, L, L)))
    psi = rng.standard_normal((L, L, 2)) + 1j * rng.standard_normal((L, L, 2))
    t0 = time.perf_counter()
    O.normal_op(U, psi, 0.05)
    t_op = time.perf_counter() - t0
    t0 = time.perf_counter()
    try:
        O.cg_normal(U, 0.05, psi, 1e-10, maxiter=5)
    except O.OracleSolverError:
        pass
    return t_op, (time.perf_counter() - t0) / 5


def run_cfg5(args):
    """BASELINE configs[4]: one 2048x2048 lattice (beta=8, m0=0.05, hot start),
    x-strip domain decomposition: one strip per rank over NCCL or peer-memory
    mailboxes (torchrun; --transport nccl|p2p), or --strips S strips on one
    GPU (local copy-kernel transport, or --transport p2p on local mailboxes).
    Reports the decomposed fused D^dag D (96 B/site), the CG to 1e-10
    (352 B/site/iteration) and one trajectory, with the CPU port's D^dag D and
    CG iteration on one core beside them (the CPU trajectory extrapolated)."""
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    hbm_peak, peak_kind = peaks()
    cpu5 = None
    if rank == 0 and world == 1 and not args.no_cpu:   # before CUDA init (fork-safe)
        with mp.get_context("fork").Pool(1) as pool:
            cpu5 = pool.apply(_cpu_cfg5_worker, (args.cfg5_size,))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1512_03812_b200.dd import DDWilsonDirac, StripLattice
    L = T = args.cfg5_size
    rng = np.random.default_rng(5)
    q = rng.uniform(-np.pi, np.pi, (2, L, T))
    psi = rng.standard_normal((L, T, 2)) + 1j * rng.standard_normal((L, T, 2))
    lat = StripLattice(L, T, strips=None if world > 1 else args.strips, transport=args.transport)
    op = DDWilsonDirac(lat, lat.scatter_links(q), 0.05)
    p_ext = lat.scatter_spinor(psi)
    del q, psi

    def sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # the D^dag D through the C-ABI on preallocated buffers (halo exchange +
    # stencil per call): op.normal's per-call tensor plumbing (allocation,
    # halo-row zeroing) costs more host time than the 2048^2 kernel takes
    from paper_1512_03812_b200 import _lib
    out_ext = op.normal(p_ext)
    lib_ctx = _lib.ctx()

    def ddagd():
        lib_ctx.call("sch_dd_ddagd", lat._handle, _lib.ptr(op.U), _lib.ptr(p_ext), _lib.ptr(out_ext),
                     0.05)

    for _ in range(args.warmup):
        ddagd()
    sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(20, args.steps)   # one application is ~0.1 ms: time a run of them
    e0.record()
    for _ in range(reps):
        ddagd()
    e1.record()
    sync()
    ms = e0.elapsed_time(e1) / reps
    from paper_1512_03812_b200.fermion import SolverError
    try:
        op.cg(p_ext, 1e-10, maxiter=40)   # untimed: loads every kernel
    except SolverError:
        pass
    sync()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    _, iters, rel = op.cg(p_ext, 1e-10)
    f1.record()
    sync()
    cg_ms = f0.elapsed_time(f1)
    if world > 1:
        t = torch.tensor([ms, cg_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, cg_ms = float(t[0]), float(t[1])
    # one full trajectory of the configs[4] schedule on the strips
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.dd_hmc import dd_hmc_update
    w = WORKLOADS["cfg5"]["phys"]
    cfg = sw.HmcConfig(L=L, T=T, beta=w["beta"], m0=w["m0"], tau=w["tau"], h=w["tau"] / args.outer,
                       scheme=w["scheme"], micro_per_call=w["micro_per_call"], cg_tol=w["cg_tol"])
    # the reference's make_rng(5, 0) stream walked on the device: hot start,
    # then the update's p / phi of the whole lattice (own rows kept) and the
    # Metropolis uniform
    drng = sw.NumpyDeviceRng(seed=5, n_chains=1, stream0=0)
    q_ext = lat.scatter_links(drng.hot_start(sw.LatticeGeom(L, T))[0])
    sync()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    q_ext, traj = dd_hmc_update(lat, q_ext, cfg, drng)
    g1.record()
    sync()
    traj_ms = g0.elapsed_time(g1)
    if world > 1:
        t = torch.tensor([traj_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        traj_ms = float(t[0])
    sites = L * T
    gbs = 96.0 * sites / (ms * 1e-3) / 1e9
    cg_gbs = 352.0 * sites * iters / (cg_ms * 1e-3) / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": "decomposed D^dag D GB/s (single lattice)", "value": gbs, "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic (hot start)",
            "config": {"workload": f"cfg5: one {L}x{T} lattice, m0=0.05, x-strips",
                       "ddagd_applications_timed": reps,
                       "strips": lat.G, "strip_rows": lat.Lloc,
                       "transport": lat.transport},
            "roofline": {"bound": "hbm", "achieved": gbs / max(world, 1), "peak": hbm_peak,
                         "unit": "GB/s per GPU", "frac": gbs / max(world, 1) / hbm_peak,
                         "peak_kind": peak_kind,
                         "kernel": "k_dd_march<PLAIN, 4-row register ring, 2 CTAs/SM> (warp-marching "
                                   "fused D^dag D, csrc/march.cuh) + the halo-row copy of each application",
                         "bytes_model": "96 B/site (psi in + U + out)"},
            "cg": {"iterations": iters, "ms": cg_ms, "ms_per_iteration": cg_ms / max(iters, 1),
                   "effective_GBs": cg_gbs, "effective_frac": cg_gbs / max(world, 1) / hbm_peak,
                   "bytes_model": "352 B/site/iteration (stencil pass 128 + update pass 224)",
                   "rel_residual": rel},
            "trajectory": {"scheme": cfg.scheme, "outer": args.outer,
                           "micro_per_call": cfg.micro_per_call, "tau": cfg.tau,
                           "ms": traj_ms, "trajectories_per_s": 1e3 / traj_ms, "dh": traj.dh,
                           "inversions": traj.inversions,
                           "includes": "heatbath draws of the full lattice on the device "
                                       "(the reference's Philox/ziggurat stream, csrc/nprng.cu), "
                                       "H at both ends, Metropolis"},
            "cpu_baseline": None if cpu5 is None else {
                "ddagd_GBs": 96.0 * sites / cpu5[0] / 1e9, "cg_s_per_iteration": cpu5[1],
                "trajectory_s_extrapolated": cpu5[1] * iters * traj.inversions / 2,
                "cores": 1, "kind": "port",
                "sample": "one oracle D^dag D and 5 CG iterations on the whole lattice; the "
                          "trajectory = CPU s/iteration x this run's CG iterations of one solve "
                          "x the trajectory's solves (inversions / 2) — an extrapolation"}}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(n):
    """`python bench.py --gpus N` outside torchrun: start the N ranks (one
    process per GPU) under torch.distributed.run on this node and return its
    exit code.  The ranks see WORLD_SIZE = N and run the same arguments."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        return launch_ranks(args.gpus)
    if world is not None and int(world) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
              "(torchrun --nproc-per-node N bench.py --gpus N) or drop the launcher",
              file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "cfg5":
        return run_cfg5(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
