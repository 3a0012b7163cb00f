import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_03812_b200 as sw
from paper_1512_03812_b200 import _lib
g = sw.NumpyDeviceRng(seed=20240401, n_chains=2, stream0=3)
print("state bytes", _lib.load().sch_np_rng_state_bytes(), g.state.numel(), hex(g.state.data_ptr()))
st0 = g.state.view(torch.int64).cpu().numpy()
print("state after init", st0.tolist())
out = g.standard_normal((8,))
print("out ptr", hex(out.data_ptr()))
st1 = g.state.view(torch.int64).cpu().numpy()
print("state after fill", st1.tolist())
got = out.cpu().numpy()
for c in range(2):
    print(c, got[c].tolist())
    print(c, sw.make_rng(20240401, 3 + c).standard_normal(8).tolist())
