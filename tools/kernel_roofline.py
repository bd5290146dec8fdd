"""Per-kernel roofline table from an ncu CSV (--metrics ..., --csv --page raw): achieved DRAM
GB/s vs the measured HBM peak for the HBM-bound stages, FP32 / issue / shared-memory
utilisation for the compositing kernels (BASELINE.json north_star evidence)."""
import csv, io, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6546.9) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6546.9
rows = list(csv.reader(io.StringIO(open(sys.argv[1]).read())))
h = next(r for r in rows if "Kernel Name" in r)
i0 = rows.index(h)
units = rows[i0 + 1]
data = rows[i0 + 2:]
col = {n: h.index(n) for n in h}
def num(r, n):
    try:
        return float(r[col[n]].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")
agg = {}
for r in data:
    if len(r) < len(h):
        continue
    k = r[col["Kernel Name"]].split("(")[0]
    a = agg.setdefault(k, {"n": 0, "t": 0.0, "b": 0.0, "issue": [], "fma": [], "smem": [], "dram": []})
    t_unit = units[col["gpu__time_duration.sum"]]
    t = num(r, "gpu__time_duration.sum") * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}.get(t_unit, 1e-9)
    bunit = units[col["dram__bytes_read.sum"]]
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(bunit, 1)
    b = (num(r, "dram__bytes_read.sum") + num(r, "dram__bytes_write.sum") * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[col["dram__bytes_write.sum"]], 1) / sc) * sc
    a["n"] += 1; a["t"] += t; a["b"] += b
    a["issue"].append(num(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"))
    a["fma"].append(num(r, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"))
    a["smem"].append(num(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"))
    a["dram"].append(num(r, "dram__throughput.avg.pct_of_peak_sustained_elapsed"))
out = [f"# per-kernel roofline, one config-3 view (ncu --clock-control none, serialised launches)",
       f"# HBM peak {peak:.1f} GB/s (MEASURED_PEAKS.json); issue/FMA/shared % of peak, launch-averaged",
       f"{'kernel':46s} {'launches':>8s} {'ms':>8s} {'GB/s':>8s} {'%HBM':>6s} {'issue%':>7s} {'fma%':>6s} {'smem%':>6s}"]
avg = lambda v: sum(v) / len(v) if v else float("nan")
for k, a in sorted(agg.items(), key=lambda x: -x[1]["t"]):
    gbs = a["b"] / a["t"] / 1e9 if a["t"] > 0 else 0.0
    out.append(f"{k[:46]:46s} {a['n']:8d} {a['t'] * 1e3:8.3f} {gbs:8.0f} {100 * gbs / peak:6.1f} "
               f"{avg(a['issue']):7.1f} {avg(a['fma']):6.1f} {avg(a['smem']):6.1f}")
print("\n".join(out))
