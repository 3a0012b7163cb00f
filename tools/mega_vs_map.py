"""Same ensemble update through the trajectory megakernel and through the
kernel-per-map path: device time of the whole update and CG iterations.

    python tools/mega_vs_map.py [chains] [reps]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_03812_b200 as sw  # noqa: E402
from paper_1512_03812_b200 import fermion as F  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = sw.HmcConfig(L=16, T=16, beta=2.0, m0=0.1, tau=1.0, h=0.25, scheme="adapted-nested-fg",
                   micro_per_call=2, cg_tol=1e-10)
d = sw.NumpyDeviceRng(seed=2024, n_chains=B)
q0 = d.hot_start(sw.LatticeGeom(16, 16))
for _ in range(2):   # move off the hot start
    q0, _ = sw.hmc_update_ensemble(q0, cfg, device_rng=d)
state0 = d.state.clone()
out = {}
for mega in (False, True, False, True):
    sw.hmc.USE_MEGA = mega
    d.state.copy_(state0)
    torch.cuda.synchronize()
    F.CG_PROFILE = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    q = q0
    for _ in range(reps):
        q, pend = sw.hmc_update_ensemble_async(q, cfg, d)
    e1.record()
    torch.cuda.synchronize()
    prof, F.CG_PROFILE = F.CG_PROFILE, None
    it = sum(int(x.sum().item()) for _, _, x, _ in prof)
    cg_ms = sum(a.elapsed_time(b) for a, b, _, _ in prof)
    ms = e0.elapsed_time(e1) / reps
    key = "mega" if mega else "map"
    out[key] = dict(ms_per_update=ms, cg_iterations_per_chain=it / (B * reps),
                    ns_per_chain_iteration=ms * 1e6 / (it / reps),
                    solver_kernel_ms=cg_ms / reps)
    print(key, out[key], flush=True)
