"""Table of the per-pass ncu captures of tools/gpu/r02_ncu_conv.sh
(gpurun_out/ncu_conv_<shape>_<pass>_raw.csv): duration, TF/s from the
algorithmic 2*M*N*K, % of the 1,646 TF/s measured burst peak, tensor-pipe and
L2 utilisation, DRAM MB and the SM clock ncu saw.

    python tools/ncu_conv_table.py gpurun_out > profiles/r02_ncu_conv_summary_final.txt
"""
import csv
import glob
import os
import re
import sys

PEAK = 1646.0
UNIT = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "us": 1.0, "usecond": 1.0, "ns": 1e-3,
        "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}


def metrics(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return None
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (u, v) for h, u, v in zip(hdr, units, vals)}


def num(m, key, unit_scale=False):
    u, v = m[key]
    x = float(v.replace(",", ""))
    return x * UNIT.get(u, 1.0) if unit_scale else x


def main():
    d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    print("ncu --set full --clock-control none of each conv pass (tools/gpu/r02_ncu_conv.sh; one launch each, cold L2,")
    print("serialised). TF/s = algorithmic 2*M*N*K / ncu duration; peak 1646 TF/s bf16 burst (MEASURED_PEAKS.json).")
    print("tensor% = sm__pipe_tensor_cycles_active (of elapsed); L2% = lts__t_sectors (of ncu's theoretical peak).")
    print(f"{'shape (n,c,h,co,k,s)':26s} {'pass':6s} {'us':>8s} {'TF/s':>7s} {'%peak':>6s} {'tensor%':>8s} {'L2%':>6s} "
          f"{'DRAM MB':>8s} {'SM GHz':>7s}  kernel")
    for path in sorted(glob.glob(os.path.join(d, "ncu_conv_*_raw.csv"))):
        mt = re.search(r"ncu_conv_(\d+)_(\d+)_(\d+)_(\d+)_(\d+)_(\d+)_(\w+)_raw", path)
        if not mt:
            continue
        n, c, h, co, k, s = (int(mt.group(i)) for i in range(1, 7))
        ps = mt.group(7)
        m = metrics(path)
        if not m:
            continue
        oh = (h - k) // s + 1
        flops = 2.0 * n * oh * oh * co * k * k * c
        us = num(m, "gpu__time_duration.sum", True)
        tf = flops / (us * 1e-6) / 1e12
        tensor = num(m, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
        l2 = num(m, "lts__t_sectors.avg.pct_of_peak_sustained_elapsed")
        dram = num(m, "dram__bytes_read.sum", True) + num(m, "dram__bytes_write.sum", True)
        ghz = num(m, "gpc__cycles_elapsed.max.per_second")
        kern = m.get("Kernel Name", ("", ""))[1]
        kern = re.sub(r"\(.*", "", kern).replace("void ", "").replace("ce::", "")
        print(f"{str((n, c, h, co, k, s)):26s} {ps:6s} {us:8.1f} {tf:7.1f} {100 * tf / PEAK:6.1f} {tensor:8.1f} "
              f"{l2:6.1f} {dram:8.1f} {ghz:7.2f}  {kern[:70]}")


if __name__ == "__main__":
    main()
