"""Dump one per-chain CG solve (solutions + iteration counts) of a B x L^2
batch under the current SCH_* kernel-variant environment, so that two
variants can be compared bit for bit:

    SCH_RESBLK_ROT=0 python tools/variant_dump.py 16 2048 out_ref_basis.npz
    python tools/variant_dump.py 16 2048 out_base.npz
    python tools/variant_dump.py --compare out_base.npz out_ref_basis.npz

(used in round 2 for the x-in-shared-memory, 8-CTA-cluster and mbarrier
variants, all bit-identical to the default, profiles/r02/README.md)
"""
import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def dump(L, B, path):
    import torch
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200 import fermion as F
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    q = (torch.rand((B, 2, L, L), dtype=torch.float64, device="cuda", generator=g) * 2 - 1) * math.pi
    b = torch.randn((B, L, L, 2), dtype=torch.complex128, device="cuda", generator=g)
    op = sw.WilsonDirac(q, 0.1)
    x, info = F.cg_solve(op, b, 1e-10, stop="per_chain")
    np.savez(path, x=x.cpu().numpy(), it=info.iters_dev.cpu().numpy(),
             rel=info.relres_dev.cpu().numpy())


def compare(a, b):
    A, Bz = np.load(a), np.load(b)
    same_it = np.array_equal(A["it"], Bz["it"])
    dx = np.max(np.abs(A["x"] - Bz["x"])) / np.max(np.abs(A["x"]))
    print(f"{a} vs {b}: iterations identical={same_it} (mean {A['it'].mean():.2f}), "
          f"max rel |dx|={dx:.3e}, bit-identical={np.array_equal(A['x'], Bz['x'])}")
    return same_it and dx < 1e-12


if __name__ == "__main__":
    if sys.argv[1] == "--compare":
        sys.exit(0 if compare(sys.argv[2], sys.argv[3]) else 1)
    dump(int(sys.argv[1]), int(sys.argv[2]), sys.argv[3])
