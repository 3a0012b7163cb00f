"""ncu driver: a few iterations of the decomposed CG on cfg5's 2048^2 lattice.

    python tools/prof_dd.py [transport] [strips] [cg|normal]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1512_03812_b200.dd import DDWilsonDirac, StripLattice  # noqa: E402
from paper_1512_03812_b200.fermion import SolverError  # noqa: E402

transport = sys.argv[1] if len(sys.argv) > 1 else "local"
strips = int(sys.argv[2]) if len(sys.argv) > 2 else 1
L = 2048
rng = np.random.default_rng(5)
lat = StripLattice(L, L, strips=strips, transport=transport)
op = DDWilsonDirac(lat, lat.scatter_links(rng.uniform(-np.pi, np.pi, (2, L, L))), 0.05)
psi = lat.scatter_spinor(rng.standard_normal((L, L, 2)) + 1j * rng.standard_normal((L, L, 2)))
what = sys.argv[3] if len(sys.argv) > 3 else "cg"
if what == "normal":   # the D^dag D alone (halo exchange + the stencil pass)
    for _ in range(4):
        op.normal(psi)
for _ in range(0 if what == "normal" else 2):
    try:
        op.cg(psi, 1e-10, maxiter=12)
    except SolverError:
        pass
torch.cuda.synchronize()
print("done")
