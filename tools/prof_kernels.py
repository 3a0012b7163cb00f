"""Small driver for ncu captures of the hot kernels (one GPU).

    python tools/prof_kernels.py stencil   # cfg2 fused D^dag D, 4096 x 32^2
    python tools/prof_kernels.py cg        # cfg3-like resident CG, 8192 x 16^2
    python tools/prof_kernels.py stream    # streaming CG iterations, cfg2
    python tools/prof_kernels.py mega      # trajectory megakernel, 8192 x 16^2 (cfg3)
"""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_03812_b200 as sw  # noqa: E402
from paper_1512_03812_b200 import fermion as F  # noqa: E402


def field(B, L, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    q = (torch.rand((B, 2, L, L), dtype=torch.float64, device="cuda", generator=g) * 2 - 1) * math.pi
    psi = torch.randn((B, L, L, 2), dtype=torch.complex128, device="cuda", generator=g)
    return q, psi


def main(what):
    if what == "stencil":
        q, psi = field(4096, 32, 1)
        op = sw.WilsonDirac(q, 0.1)
        for _ in range(5):
            op.normal(psi)
    elif what == "cg":
        q, psi = field(8192, 16, 2)
        op = sw.WilsonDirac(q, 0.1)
        for _ in range(2):
            F.cg_solve(op, psi, 1e-10, stop="per_chain")
    elif what == "stream":
        q, psi = field(4096, 32, 3)
        op = sw.WilsonDirac(q, 0.1)
        F.cg_solve(op, psi, 1e-10, maxiter=12, stop="batch_global")
    elif what == "mega":
        cfg = sw.HmcConfig(L=16, T=16, beta=2.0, m0=0.1, tau=1.0, h=0.25,
                           scheme="adapted-nested-fg", micro_per_call=2, cg_tol=1e-10)
        d = sw.NumpyDeviceRng(seed=2024, n_chains=8192)
        q = d.hot_start(sw.LatticeGeom(16, 16))
        for _ in range(2):
            q, _ = sw.hmc_update_ensemble(q, cfg, device_rng=d)
    torch.cuda.synchronize()
    print("done", what)


if __name__ == "__main__":
    main(sys.argv[1])
