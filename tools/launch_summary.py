"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import re
import sys


def short_name(name):
    m = re.search(r"tc_gemm_kernel<(\d+), (?:ce::)?(\w+)", name)
    if m:
        return f"tc_{m.group(2).replace('TcLoader', '')}_BN{m.group(1)}"
    m = re.search(r"simt_gemm_kernel<(?:ce::)?(\w+)(?:<[^>]*>)?, (?:ce::)?(\w+)", name)
    if m:
        return f"simt_{m.group(1)}x{m.group(2)}"
    return re.sub(r"^void |\(.*|<.*", "", name).replace("ce::", "")


def summarise(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = [r for r in rows if "Kernel Name" in r][0]
    ki, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if len(r) != len(hdr) or r is hdr or r[ui] not in scale:
            continue
        a = agg[short_name(r[ki])]
        a[0] += 1
        a[1] += float(r[vi].replace(",", "")) * scale[r[ui]]
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':48s} {'launches':>8s} {'total_us':>12s} {'share':>6s} {'avg_us':>9s}"]
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        lines.append(f"{k:48s} {n:8d} {us:12.1f} {us / tot:6.3f} {us / n:9.1f}")
    lines.append(f"total {sum(v[0] for v in agg.values())} launches, {tot:.1f} us")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
