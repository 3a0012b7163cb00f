"""Per-step host issue time vs GPU time of the cfg3 ensemble update (eager)."""
import gc
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_03812_b200 as sw  # noqa: E402


def main():
    B = 8192
    cfg = sw.HmcConfig(L=16, T=16, beta=2.0, m0=0.1, tau=1.0, h=0.25, scheme="adapted-nested-fg",
                       micro_per_call=2, cg_tol=1e-10)
    d = sw.NumpyDeviceRng(seed=2024, n_chains=B)
    q = d.hot_start(sw.LatticeGeom(16, 16))
    for _ in range(3):
        q, _ = sw.hmc_update_ensemble(q, cfg, device_rng=d)
    torch.cuda.synchronize()
    if os.environ.get("NOGC"):
        gc.collect()
        gc.disable()
    for k in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        q, p = sw.hmc_update_ensemble_async(q, cfg, d)
        e1.record()
        t1 = time.perf_counter()
        p.resolve()
        t2 = time.perf_counter()
        print(f"{'nogc' if os.environ.get('NOGC') else 'gc'} step {k}: issue {1e3 * (t1 - t0):7.2f} ms  wait {1e3 * (t2 - t1):7.2f} ms  "
              f"gpu {e0.elapsed_time(e1):7.2f} ms")


if __name__ == "__main__":
    main()
