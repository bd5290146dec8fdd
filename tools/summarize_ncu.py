"""Summarise ncu captures for profiles/: a launch list (--metrics gpu__time_duration.sum csv)
and/or a --set full report.  Also writes profiles/ncu_traffic.json (DRAM bytes per launch of
each captured kernel) that bench.py attaches to its roofline object.

  python tools/summarize_ncu.py --launches gpurun_out/launches.csv --out profiles/r01_launches.txt
  python tools/summarize_ncu.py --report gpurun_out/prof.ncu-rep --out profiles/r01_ncu_full.txt
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        agg.setdefault(name, [0, 0.0])
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) / 1e6  # ns -> ms
    tot = sum(v[1] for v in agg.values())
    out = ["# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised:",
           "# compare SHARES, not absolutes)", f"# total {tot:.3f} ms over {sum(v[0] for v in agg.values())} launches",
           f"{'ms':>10} {'share':>7} {'launches':>8}  kernel"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{t:10.3f} {100 * t / tot:6.1f}% {n:8d}  {k}")
    return "\n".join(out)


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, rows = r[0], r[2:]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
            "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
    ki = h.index("Kernel Name")
    out = ["# ncu --set full --clock-control none (one launch per row; units as reported by ncu)"]
    traffic = {}
    for x in rows:
        name = x[ki].split("(")[0]
        vals = {w: x[h.index(w)] for w in want if w in h}
        stalls = []
        for i, c in enumerate(h):
            if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("_not_issued"):
                try:
                    stalls.append((float(x[i].replace(",", "")), c.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(stalls, reverse=True)[:4])
        out.append(f"\n## {name}")
        for k, v in vals.items():
            out.append(f"  {k} = {v}")
        out.append(f"  top stall reasons: {top}")
        try:
            rd = float(vals["dram__bytes_read.sum"].replace(",", ""))
            wr = float(vals["dram__bytes_write.sum"].replace(",", ""))
            unit = h[h.index("dram__bytes_read.sum")]
            traffic.setdefault(name, []).append((rd + wr))
        except (KeyError, ValueError):
            pass
    units = {c: u for c, u in zip(h, r[1])}
    return "\n".join(out), traffic, units.get("dram__bytes_read.sum", "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    text = []
    if a.launches:
        text.append(launches(a.launches))
    if a.report:
        t, traffic, unit = report(a.report)
        text.append(t)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        tj = {k: {"dram_bytes_per_launch": sum(v) / len(v) * scale, "launches_captured": len(v),
                  "source": os.path.basename(a.report)} for k, v in traffic.items()}
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        merged = json.load(open(tp)) if os.path.exists(tp) else {}
        merged.update(tj)  # keep the other kernels' captures
        json.dump(merged, open(tp, "w"), indent=1)
    open(a.out, "w").write("\n\n".join(text) + "\n")
    print(open(a.out).read()[:3000])


if __name__ == "__main__":
    sys.exit(main())
