"""Per-kernel times of one training step from an ncu launch list: the kernels
between the 2nd and 3rd xent launches (steady state)."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [r for r in rows if "Kernel Name" in r][0]
k, v, g = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
seq = [(r[k], float(r[v].replace(",", "")) / 1e3, r[g]) for r in rows if len(r) == len(hdr) and r is not hdr]
xs = [i for i, (n, _, _) in enumerate(seq) if "xent_kernel" in n or "head_fwd_kernel" in n]
a, b = xs[1], xs[2]
tot = 0.0
for n, t, grid in seq[a - 30 if a > 30 else 0:b + 1][:0] or seq[xs[1] + 1: xs[2] + 1]:
    m = re.search(r"tc_gemm_kernel<(\d+), (?:ce::)?(\w+)", n)
    name = f"{m.group(2)}_{m.group(1)}" if m else re.sub(r"^void |\(.*|<.*", "", n)
    print(f"{t:9.1f} us  {grid:14s} {name}")
    tot += t
print(f"step total {tot:.1f} us (backward of step i + forward of step i+1)")
