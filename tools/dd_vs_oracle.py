import numpy as np, sys
sys.path.insert(0, '.')
from paper_1512_03812_b200.dd import DDWilsonDirac, StripLattice
from oracle import schwinger_oracle as O
L, T, G = 32, 16, 4
rng = np.random.default_rng(3)
q = 0.3 * rng.standard_normal((2, L, T))
lat = StripLattice(L, T, strips=G)
op = DDWilsonDirac(lat, lat.scatter_links(q), -0.231367)
b = rng.standard_normal((L, T, 2)) + 1j * rng.standard_normal((L, T, 2))
x0 = 0.1 * (rng.standard_normal((L, T, 2)) + 1j * rng.standard_normal((L, T, 2)))
x, it, rel = op.cg(lat.scatter_spinor(b), 1e-12, x0_ext=lat.scatter_spinor(x0))
xo, ito, _ = O.cg_normal(O.fermion_links(q), -0.231367, b, 1e-12, x0=x0)
xg = lat.gather_spinor(x).cpu().numpy()
print("warm it", it, "oracle", ito, "relerr", np.max(np.abs(xg-xo))/np.max(np.abs(xo)))
for G in (1,2,4,8):
    lat = StripLattice(L, T, strips=G)
    op = DDWilsonDirac(lat, lat.scatter_links(q), -0.231367)
    x, it, rel = op.cg(lat.scatter_spinor(b), 1e-12)
    xo, ito, _ = O.cg_normal(O.fermion_links(q), -0.231367, b, 1e-12)
    xg = lat.gather_spinor(x).cpu().numpy()
    print("cold G", G, "it", it, "oracle", ito, "relerr", np.max(np.abs(xg-xo))/np.max(np.abs(xo)))
