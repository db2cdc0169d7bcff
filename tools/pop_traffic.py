"""Per-kernel-class time share and DRAM traffic of a population run from one
single-pass ncu launch list:

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file launches.csv python tools/class_profile.py
    python tools/pop_traffic.py launches.csv class_profile.txt [profiles/traffic.json]

Kernels map to the library's profiling classes by template / kernel name (the
loader + epilogue of tc_gemm_kernel, the operand functors of simt_gemm).
class_profile.txt supplies the number of class launches (Prof scopes) of the
same population, so traffic.json holds DRAM bytes per class launch -- the
`traffic` field of bench.py's roofline (per launch, like `achieved`).
ncu serialises kernels and flushes caches, so shares (not absolute times) are
what compare with the bench.
"""
import collections
import csv
import json
import re
import sys


def klass(name):
    if "tc_gemm_kernel" in name:
        if "FwdTcEpi" in name:
            return "conv_fwd"
        if "Dgrad" in name:
            return "conv_dgrad"
        if "Wgrad" in name:
            return "conv_wgrad"
        if "DenseFwdEpi" in name:
            return "dense_fwd"
        return "dense_bwd"
    if "simt_gemm_kernel" in name:
        for key, cls in (("FwdA", "conv_fwd"), ("DgradA", "conv_dgrad"), ("WgradA", "conv_wgrad"),
                         ("DenseXA", "dense_fwd")):
            if key in name:
                return cls
        return "dense_bwd"
    rules = [("im2col_packed", "conv_fwd"), ("conv_sgd", "conv_sgd"), ("colsum8", "conv_sgd"),
             ("maxpool", "pool"), ("xent", "loss"), ("gather_u8", "gather"), ("head_fwd", "dense_fwd"),
             ("dense_reduce", "dense_fwd"), ("head_bwd", "dense_bwd"), ("dense_dw", "dense_bwd"),
             ("dense_dx", "dense_bwd"), ("bias_sgd", "dense_bwd"), ("colsum_partial", "dense_bwd"),
             ("f32_to_bf16_pad", "dense_bwd")]
    for key, cls in rules:
        if key in name:
            return cls
    return "other"


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = [r for r in rows if "Kernel Name" in r][0]
    ii, ki, mi, ui, vi = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = collections.defaultdict(dict)
    names = {}
    for r in rows:
        if len(r) != len(hdr) or r is hdr or r[ui] not in scale:
            continue
        per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * scale[r[ui]]
        names[r[ii]] = r[ki]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for kid, m in per.items():
        a = agg[klass(names[kid])]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    launches = {}
    if len(sys.argv) > 2:
        total = [ln for ln in open(sys.argv[2]) if ln.startswith("TOTAL")]
        if total:
            for k, n in re.findall(r"(\w+)=[\d.]+ms/(\d+)", total[0]):
                launches[k] = int(n)
    tot_us = sum(v[1] for v in agg.values())
    out = {}
    print(f"{'class':12s} {'kernels':>8s} {'share':>7s} {'GB':>8s} {'class launches':>15s} {'MB/launch':>10s}")
    for k, (n, us, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        nl = launches.get(k)
        per_launch = by / nl if nl else None
        if per_launch is not None:
            out[k] = per_launch
        print(f"{k:12s} {n:8d} {us / tot_us:7.1%} {by / 1e9:8.2f} {nl if nl else '-':>15} "
              f"{per_launch / 1e6 if per_launch else float('nan'):10.2f}")
    if len(sys.argv) > 3:
        json.dump({"_source": "tools/pop_traffic.py over an ncu dram__bytes launch list of tools/class_profile.py "
                              "(C2 population); DRAM bytes per class launch", **out}, open(sys.argv[3], "w"), indent=1)


if __name__ == "__main__":
    main()
