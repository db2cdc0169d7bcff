"""Per-launch DRAM bytes of the dense-backward class from an ncu CSV of the bench's
profiling pass (tools/gpu/r02_traffic.sh) -> profiles/traffic_r02.json, which
bench.py reports as roofline.traffic next to the class's algorithmic bytes."""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [r for r in rows if "Kernel Name" in r][0]
ki, mi, ui, vi, idi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0,
         "nsecond": 1e-3, "msecond": 1e3}
per = collections.defaultdict(dict)
for r in rows:
    if len(r) != len(hdr) or r is hdr or r[ui] not in scale:
        continue
    per[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * scale[r[ui]]
    per[r[idi]]["name"] = r[ki]
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in per.values():
    short = d["name"].split("(")[0].split("<")[0].replace("void ", "").strip()
    if "tc_gemm_kernel" in d["name"]:
        short = "tc_" + ("DenseDw" if "DenseDwLoader" in d["name"] else "DenseDx")
    t = tot[short]
    t[0] += 1
    t[1] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    t[2] += d.get("gpu__time_duration.sum", 0.0)
launches = int(sys.argv[2]) if len(sys.argv) > 2 else None  # dense_bwd class launches of the same pass
total_bytes = sum(v[1] for v in tot.values())
out = {"source": sys.argv[1], "kernels": {k: {"launches": v[0], "dram_bytes": v[1], "us": v[2]} for k, v in tot.items()},
       "classes": {"dense_bwd": {"dram_bytes_total": total_bytes,
                                 "dram_bytes_per_launch": total_bytes / launches if launches else None,
                                 "class_launches": launches}}}
print(json.dumps(out, indent=1))
