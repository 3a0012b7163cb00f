"""Golden mean |dH| values of the reference's order-of-convergence test
(pkg/tests/test_acceptance.py:130-156) on the committed thermalized 8x8
fixture, made by running the REFERENCE itself (build container only; the
reference's own therm_8x8.cfg is missing, tests/fixtures/ holds one
regenerated with its thermalize).  One process per scheme.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_order_golden.py
"""

import math
import multiprocessing as mp
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
SECOND_ORDER = ("leapfrog", "5stage", "nested-leapfrog", "nested-5stage")
FOURTH_ORDER = ("5stage-fg", "fg-approx", "11stage", "nested-fg", "adapted-nested-fg")
GRID2 = (0.02, 0.025, 0.04, 0.0625)
GRID4 = (0.02, 0.025, 0.03125, 0.04)


def run(scheme):
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
    import schwinger as sw
    from schwinger.config import HmcConfig
    from schwinger.hmc import measure_dh
    from schwinger.lattice import load_gauge_config
    q, _ = load_gauge_config(str(HERE.parent / "fixtures" / "therm_8x8.cfg"))
    base = HmcConfig(L=8, T=8, beta=1.0, m0=-0.231367, tau=2.0, n_samples=50)
    grid = GRID2 if scheme in SECOND_ORDER else GRID4
    out = []
    for h in grid:
        micro = math.ceil(1.0 / h) if scheme in ("nested-fg", "adapted-nested-fg") else None
        m = measure_dh(q, replace(base, scheme=scheme, h=h, micro_per_call=micro),
                       sw.make_rng(400, 7), n_samples=50)
        out.append((m.mean_abs, m.inversions_per_traj))
    return scheme, np.array(grid), np.array(out)


if __name__ == "__main__":
    with mp.get_context("fork").Pool(8) as pool:
        res = pool.map(run, SECOND_ORDER + FOURTH_ORDER)
    arrays = {}
    for scheme, grid, out in res:
        arrays[f"{scheme}_h"] = grid
        arrays[f"{scheme}_mean"] = out[:, 0]
        arrays[f"{scheme}_inv"] = out[:, 1]
        slope = np.polyfit(np.log(grid), np.log(out[:, 0]), 1)[0]
        print(f"{scheme}: slope {slope:.4f}")
    np.savez(HERE / "order.npz", **arrays)
