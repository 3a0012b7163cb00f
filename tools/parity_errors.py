"""Print the measured relative error of every force / FG piece of the GPU path
against the reference goldens (tests/golden/forces.npz), so the tolerance in
tests/test_gpu_parity.py is a recorded measurement, not a guess.

Also prints the oracle's own error on the same inputs (the oracle is the
checker; its error against the reference is the floor of the comparison).
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def main():
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200 import fermion as F
    from oracle import schwinger_oracle as O
    g = dict(np.load(ROOT / "tests/golden/forces.npz"))
    for tag in ("u", "b"):
        q, eta = g[f"{tag}_q"], g[f"{tag}_eta"]
        op = sw.WilsonDirac(q, 0.1)
        U = O.fermion_links(q)
        chi, xi, _ = sw.chi_xi(op, eta, 1e-12)
        out = {"chi": chi, "xi": xi}
        z1, z2 = F.z_pair(op, g[f"{tag}_f"], g[f"{tag}_chi"], g[f"{tag}_xi"], 1e-12)
        out["z1"], out["z2"] = z1, z2
        out["fgff"] = F.fg_fermion_hessian_dot(op, g[f"{tag}_chi"], g[f"{tag}_xi"], g[f"{tag}_f"], 1e-12)
        out["fggf"] = F.fg_fermion_hessian_dot(op, g[f"{tag}_chi"], g[f"{tag}_xi"], g[f"{tag}_g"], 1e-12)
        oz1, oz2 = O.z_pair(U, 0.1, g[f"{tag}_f"], g[f"{tag}_chi"], g[f"{tag}_xi"], 1e-12)
        orc = {"z1": oz1, "z2": oz2,
               "fgff": O.fg_fermion_hessian_dot(U, 0.1, g[f"{tag}_chi"], g[f"{tag}_xi"], g[f"{tag}_f"], 1e-12),
               "fggf": O.fg_fermion_hessian_dot(U, 0.1, g[f"{tag}_chi"], g[f"{tag}_xi"], g[f"{tag}_g"], 1e-12)}
        for k, v in out.items():
            v = v.detach().cpu().numpy()
            line = f"{tag} {k:5s} gpu-vs-ref {rel(v, g[f'{tag}_{k}']):.3e}"
            if k in orc:
                line += f"  oracle-vs-ref {rel(orc[k], g[f'{tag}_{k}']):.3e}  gpu-vs-oracle {rel(v, orc[k]):.3e}"
            print(line)


if __name__ == "__main__":
    main()
