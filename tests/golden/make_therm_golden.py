"""Golden thermalize run (hmc.py:133-155: cold start, leapfrog updates at
min(h, 0.1), the step annealed by 0.7 after any 20-update block under 80 %
acceptance), made by running the REFERENCE itself (build container only):
an 8x8 lattice at beta 1, m0 -0.231367 (the paper's mass), 60 updates —
the final links, the links after the first 5 updates and the plaquette
history.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_therm_golden.py
"""

import logging
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
    import schwinger as sw
    from schwinger.config import HmcConfig
    from schwinger.hmc import thermalize
    logging.basicConfig(level=logging.INFO)
    cfg = HmcConfig(L=8, T=8, beta=1.0, m0=-0.231367, tau=1.0, h=0.1, cg_tol=1e-10,
                    n_thermalize=60, seed=11)
    q, hist = thermalize(cfg, sw.make_rng(cfg.seed, 0))
    from dataclasses import replace
    q5, _ = thermalize(replace(cfg, n_thermalize=5), sw.make_rng(cfg.seed, 0))   # the first 5
    np.savez(HERE / "therm.npz", q=q, q5=q5, history=np.asarray(hist))
    print(np.asarray(hist)[::10])


if __name__ == "__main__":
    main()
