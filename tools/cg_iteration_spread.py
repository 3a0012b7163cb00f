import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1512_03812_b200 as sw
from paper_1512_03812_b200 import fermion as F
B = 1024
cfg = sw.HmcConfig(L=16, T=16, beta=2.0, m0=0.1, tau=1.0, h=0.25, scheme="adapted-nested-fg", micro_per_call=2, cg_tol=1e-10)
d = sw.NumpyDeviceRng(seed=2024, n_chains=B)
q = d.hot_start(sw.LatticeGeom(16, 16))
for _ in range(3):
    q, _ = sw.hmc_update_ensemble(q, cfg, device_rng=d)
F.CG_PROFILE = []
q, _ = sw.hmc_update_ensemble(q, cfg, device_rng=d)
prev = None
for a, b, it, V in F.CG_PROFILE:
    x = it.cpu().numpy().astype(float)
    corr = np.corrcoef(prev, x)[0, 1] if prev is not None else float('nan')
    print(f"min {x.min():.0f} mean {x.mean():.1f} max {x.max():.0f} std {x.std():.1f} corr_prev {corr:.2f} ms {a.elapsed_time(b):.3f}")
    prev = x
