"""Golden quenched HMC updates (HmcConfig.quenched: eta = 0 and no
pseudofermion draw, hmc.py:79-80), made by running the REFERENCE itself
(build container only): a 12x12 hot start from make_rng(5, 0), then three
hmc_update calls on the same generator for two schemes — dH, accept,
inversions and the final links — plus a batched quenched measure_dh.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_quenched_golden.py
"""

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
SCHEMES = (("adapted-nested-fg", 0.25, 2), ("5stage", 0.2, None))


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
    import schwinger as sw
    from schwinger.config import HmcConfig
    from schwinger.hmc import hmc_update, measure_dh
    out = {}
    L = 12
    for scheme, h, micro in SCHEMES:
        cfg = HmcConfig(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=h, scheme=scheme,
                        micro_per_call=micro, cg_tol=1e-10, quenched=True)
        rng = sw.make_rng(5, 0)
        q = sw.hot_start(rng, sw.LatticeGeom(L, L))
        out[f"{scheme}_q0"] = q
        dh, acc, inv = [], [], []
        for _ in range(3):
            q, st = hmc_update(q, cfg, rng)
            dh.append(st.dh)
            acc.append(bool(st.accepted))
            inv.append(st.inversions)
        out[f"{scheme}_dh"] = np.array(dh)
        out[f"{scheme}_acc"] = np.array(acc)
        out[f"{scheme}_inv"] = np.array(inv)
        out[f"{scheme}_q"] = q
        m = measure_dh(out[f"{scheme}_q0"], cfg, sw.make_rng(6, 1), n_samples=8)
        out[f"{scheme}_mdh"] = np.asarray(m.dh)
        out[f"{scheme}_minv"] = np.array(m.inversions_per_traj)
    np.savez(HERE / "quenched.npz", **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
