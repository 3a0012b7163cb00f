"""measure_dh at the paper's benchmark point (HmcConfig defaults: 32x32,
beta 1, m0 -0.231367, tau 2, tol 1e-12) from a thermalized configuration,
on the GPU, for comparison with the reference run on the same inputs
(the reference's measure_dh with make_rng(seed, 7)).

    python tools/paper_point_check.py therm.cfg scheme h n [scheme h n ...]
"""
import sys
import time
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_03812_b200 as sw  # noqa: E402
from paper_1512_03812_b200.lattice import load_gauge_config  # noqa: E402

q, meta = load_gauge_config(sys.argv[1])
args = sys.argv[2:]
for i in range(0, len(args), 3):
    scheme, h, n = args[i], float(args[i + 1]), int(args[i + 2])
    cfg = replace(sw.HmcConfig(), scheme=scheme, h=h)
    t = time.time()
    try:
        m = sw.measure_dh(q, cfg, sw.make_rng(cfg.seed, 7), n_samples=n)
        print(scheme, h, n, "ok", repr(m.mean_abs), m.acceptance, m.inversions_per_traj,
              f"{time.time() - t:.1f}s", flush=True)
    except sw.SolverError as e:
        print(scheme, h, n, "SolverError", e, f"{time.time() - t:.1f}s", flush=True)
