"""Where one HMC trajectory of the decomposed lattice (cfg5) spends its GPU
time: kernel durations from CUPTI (torch.profiler), summed by kernel name,
beside the wall-clock of the update.

    python tools/dd_traj_breakdown.py [L] [strips] [transport]
"""
import sys
import time
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_03812_b200 as sw  # noqa: E402
from paper_1512_03812_b200.dd import StripLattice  # noqa: E402
from paper_1512_03812_b200.dd_hmc import dd_hmc_update  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
strips = int(sys.argv[2]) if len(sys.argv) > 2 else 1
transport = sys.argv[3] if len(sys.argv) > 3 else "local"
cfg = sw.HmcConfig(L=L, T=L, beta=8.0, m0=0.05, tau=0.5, h=0.05, scheme="adapted-nested-fg",
                   micro_per_call=2, cg_tol=1e-10)
lat = StripLattice(L, L, strips=strips, transport=transport)
drng = sw.NumpyDeviceRng(seed=5, n_chains=1, stream0=0)
q_ext = lat.scatter_links(drng.hot_start(sw.LatticeGeom(L, L))[0])
q_ext, _ = dd_hmc_update(lat, q_ext, cfg, drng)   # warm: loads every kernel
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    q_ext, s = dd_hmc_update(lat, q_ext, cfg, drng)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
tot = defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:70]
        tot[k][0] += 1
        tot[k][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
gpu = sum(v[1] for v in tot.values())
print(f"wall {wall * 1e3:.1f} ms, GPU kernels {gpu / 1e3:.1f} ms ({gpu / 1e3 / (wall * 1e3):.2f} of wall), "
      f"inversions {s.inversions}, dH {s.dh!r}")
for k, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{k:72s} n={n:6d}  {us / 1e3:9.2f} ms  {us / gpu:6.3f}")
