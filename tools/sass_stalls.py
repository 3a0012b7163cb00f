"""Fixed stall counts the compiler encoded in the SASS control bits of a
kernel (Volta+ encoding: stall cycles = bits 105..108 of the 128-bit word),
summed per opcode class over an address range — a static view of how densely
a warp's instruction stream can issue (the 'wait' stall reason of ncu).

    cuobjdump -sass -fun <mangled> lib.o > k.sass
    python tools/sass_stalls.py k.sass [start_hex end_hex]
"""
import re
import sys
from collections import Counter, defaultdict

lines = open(sys.argv[1]).read().splitlines()
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 40
ins = []
i = 0
while i < len(lines):
    m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);\s*/\* 0x([0-9a-f]+) \*/", lines[i])
    if m and i + 1 < len(lines):
        m2 = re.match(r"\s*/\* 0x([0-9a-f]+) \*/", lines[i + 1])
        if m2:
            addr = int(m.group(1), 16)
            hiw = int(m2.group(1), 16)
            ctrl = (hiw >> 41) & 0x7FFFFF
            stall = ctrl & 0xF
            op = m.group(2).split()
            op = [o for o in op if not o.startswith("@")][0].split(".")[0]
            ins.append((addr, op, stall, m.group(2)))
            i += 2
            continue
    i += 1
sel = [x for x in ins if lo <= x[0] < hi]
tot = sum(s for _, _, s, _ in sel)
by = defaultdict(lambda: [0, 0])
for _, op, s, _ in sel:
    by[op][0] += 1
    by[op][1] += s
print(f"{len(sel)} instructions, {tot} encoded stall cycles")
for op, (n, s) in sorted(by.items(), key=lambda kv: -kv[1][1])[:20]:
    print(f"  {op:8s} n={n:5d} stall_cycles={s:6d} avg={s / n:.2f}")
hist = Counter(s for _, op, s, _ in sel if op in ("DFMA", "DADD", "DMUL"))
print("FP64 stall histogram:", sorted(hist.items()))
