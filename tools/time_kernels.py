"""CUDA-event timings of the hot kernels in isolation (one GPU).

    python tools/time_kernels.py stencil      # cfg2 fused D^dag D, 4096 x 32^2
    python tools/time_kernels.py cg [L] [B]   # resident CG per chain, B x L^2
    python tools/time_kernels.py stream       # streaming CG, cfg2, batch_global
Set SCH_RESIDENT=NTxSPT to force a resident-CG instantiation.
"""
import json
import math
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_03812_b200 as sw  # noqa: E402
from paper_1512_03812_b200 import _lib  # noqa: E402
from paper_1512_03812_b200 import fermion as F  # noqa: E402


def field(B, L, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    q = (torch.rand((B, 2, L, L), dtype=torch.float64, device="cuda", generator=g) * 2 - 1) * math.pi
    psi = torch.randn((B, L, L, 2), dtype=torch.complex128, device="cuda", generator=g)
    return q, psi


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    what = sys.argv[1]
    out = {"what": what, "resident": os.environ.get("SCH_RESIDENT")}
    if what == "stencil":
        B, L = 4096, 32
        q, psi = field(B, L, 1)
        op = sw.WilsonDirac(q, 0.1)
        res = torch.empty_like(psi)
        ctx = _lib.ctx()

        def direct():
            ctx.call("sch_ddagd", _lib.ptr(op.U), _lib.ptr(psi), _lib.ptr(res), B, L, L, 0.1)

        out["api_ms"] = timed(lambda: op.normal(psi), 20)
        out["direct_ms"] = timed(direct, 20)
        out["dslash_ms"] = timed(lambda: op.apply(psi), 20)
        sites = B * L * L
        out["ddagd_GBs_direct"] = 96.0 * sites / (out["direct_ms"] * 1e-3) / 1e9
        out["ddagd_GBs_api"] = 96.0 * sites / (out["api_ms"] * 1e-3) / 1e9
        out["dslash_GBs"] = 96.0 * sites / (out["dslash_ms"] * 1e-3) / 1e9
    elif what == "cg":
        L = int(sys.argv[2]) if len(sys.argv) > 2 else 16
        B = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
        q, psi = field(B, L, 2)
        op = sw.WilsonDirac(q, 0.1)
        F.cg_solve(op, psi, 1e-10, stop="per_chain")
        torch.cuda.synchronize()
        F.CG_PROFILE = []
        for _ in range(3):
            F.cg_solve(op, psi, 1e-10, stop="per_chain")
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b, _, _ in F.CG_PROFILE)
        iters = sum(int(it.sum().item()) for _, _, it, _ in F.CG_PROFILE)
        V = L * L
        out.update(L=L, B=B, ms_per_solve=ms / 3, iters_mean=iters / (3 * B),
                   ns_per_chain_iter=ms * 1e6 / iters,
                   fp64_tflops=152.0 * V * iters / (ms * 1e-3) / 1e12,
                   eff_GBs=352.0 * V * iters / (ms * 1e-3) / 1e9)
        x, info = F.cg_solve(op, psi, 1e-10, stop="per_chain")
        out["max_relres"] = float(info.relres_dev.max().item())
        out["any_fail"] = int(info.status_dev.sum().item())
    elif what == "stream":
        B, L = 4096, 32
        q, psi = field(B, L, 3)
        op = sw.WilsonDirac(q, 0.1)
        F.cg_solve(op, psi, 1e-10, maxiter=60, stop="batch_global")   # load every kernel
        torch.cuda.synchronize()
        F.CG_PROFILE = []
        F.cg_solve(op, psi, 1e-10, stop="batch_global")
        torch.cuda.synchronize()
        a, b, it, V = F.CG_PROFILE[0]
        ms = a.elapsed_time(b)
        n = int(it.max().item())
        out.update(ms=ms, iters=n, ms_per_iter=ms / n,
                   eff_GBs=352.0 * V * B * n / (ms * 1e-3) / 1e9)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
