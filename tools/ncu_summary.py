"""Text summary of an .ncu-rep (speed-of-light, memory, occupancy, top stall
reasons, DRAM bytes per launch) for committing under profiles/."""
import csv
import io
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def summary(rep):
    out = [f"# ncu summary of {rep}"]
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    if rows:
        h = rows[0]
        last_kernel = None
        for r in rows[1:]:
            d = dict(zip(h, r))
            if d.get("Kernel Name") != last_kernel:
                last_kernel = d.get("Kernel Name")
                out.append(f"\n## kernel: {last_kernel[:160]}")
            if d.get("Section Name") in ("GPU Speed Of Light Throughput", "Memory Workload Analysis",
                                         "Compute Workload Analysis", "Occupancy", "Launch Statistics"):
                out.append(f"{d['Section Name'][:26]:26s} | {d['Metric Name']:40s} | {d['Metric Value']} {d['Metric Unit']}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    if len(raw) > 2:
        h = raw[0]
        for v in raw[2:]:
            m = dict(zip(h, v))
            out.append(f"\n## raw: {m.get('Kernel Name', '')[:120]}")
            for key in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                        "sm__cycles_active.min", "sm__cycles_active.max", "launch__grid_size",
                        "launch__registers_per_thread"):
                if key in m:
                    out.append(f"{key:75s} {m[key]}")
            stalls = sorted(((k, float(x.replace(",", ""))) for k, x in m.items()
                             if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                             and x.replace(",", "").replace(".", "").isdigit()), key=lambda t: -t[1])[:6]
            out += [f"stall {k[len('smsp__pcsamp_warps_issue_stalled_'):]:30s} {x:.0f}" for k, x in stalls]
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1]))
