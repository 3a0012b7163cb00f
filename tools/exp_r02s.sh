#!/bin/bash
# Record of a round-2 experiment (SCH_MARCH32 was removed afterwards: the marching pass on 32 x 32 lattices measured equal to the TMA tile kernel, 80-81 us).
# Round-2: warp-marching D^dag D on cfg2's batched 32 x 32 lattices vs the TMA tile kernel
set -u
O=gpurun_out/exp_r02s
mkdir -p $O
cat > /tmp/m32.py <<'PY'
import sys, math, torch
sys.path.insert(0, ".")
import paper_1512_03812_b200 as sw
g = torch.Generator(device="cuda"); g.manual_seed(1)
B, L = 4096, 32
q = (torch.rand((B, 2, L, L), dtype=torch.float64, device="cuda", generator=g) * 2 - 1) * math.pi
psi = torch.randn((B, L, L, 2), dtype=torch.complex128, device="cuda", generator=g)
op = sw.WilsonDirac(q, 0.1)
out = op.normal(psi)
torch.save(out.cpu(), sys.argv[1])
for _ in range(5): op.normal(psi)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): op.normal(psi)
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 50 * 1e3
print(f"{us:.2f} us per D^dag D, {B*L*L*96/us/1e3:.0f} GB/s")
PY
python /tmp/m32.py $O/ref.pt
for r in 32 16 8; do echo "R=$r"; SCH_MARCH32=$r python /tmp/m32.py $O/m$r.pt; done
python - <<PY
import torch
a = torch.load("$O/ref.pt")
for r in (32, 16, 8):
    b = torch.load(f"$O/m{r}.pt")
    print(r, float((a - b).abs().max() / a.abs().max()))
PY
rm -f $O/*.pt
for r in 32 16; do
SCH_MARCH32=$r ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_march32" -s 3 -c 2 --csv --log-file $O/m$r.csv python tools/prof_kernels.py stencil > /dev/null 2>&1
echo "ncu R=$r"; grep -E "gpu__time_duration|dram__bytes" $O/m$r.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | cut -c1-120
done
