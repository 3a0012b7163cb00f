"""cfg3 ensemble update: eager async issue vs one CUDA-graph replay per step."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_03812_b200 as sw  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    cfg = sw.HmcConfig(L=16, T=16, beta=2.0, m0=0.1, tau=1.0, h=0.25, scheme="adapted-nested-fg",
                       micro_per_call=2, cg_tol=1e-10)
    geom = sw.LatticeGeom(16, 16)
    d = sw.NumpyDeviceRng(seed=2024, n_chains=B)
    q = d.hot_start(geom)
    for _ in range(3):
        q, _ = sw.hmc_update_ensemble(q, cfg, device_rng=d)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 5
    e0.record()
    for _ in range(n):
        q, p = sw.hmc_update_ensemble_async(q, cfg, d)
        p.resolve()
    e1.record()
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / n
    upd = sw.EnsembleUpdateGraph(q, cfg, d)
    upd.step()
    upd.stats()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        upd.step()
        upd.stats()
    e1.record()
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / n
    print({"B": B, "eager_ms": eager, "graph_ms": graph})


if __name__ == "__main__":
    main()
