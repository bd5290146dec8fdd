"""Per-kernel metrics of an `ncu --set full` report as JSON (profiles/r02_ncu_compositing.json,
read by bench.py's roofline object): duration, DRAM bytes, issue / FMA-pipe / warp occupancy,
instructions, registers, the occupancy limiters and the top stall reasons.

  python tools/ncu_json.py gpurun_out/x.ncu-rep profiles/r02_ncu_compositing.json [name-substring ...]
"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
want = sys.argv[3:]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
SCALE = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(d, key):
    v = float(d[key].replace(",", ""))
    return v * SCALE.get(units[hdr.index(key)], 1.0)

M = {"ms": "gpu__time_duration.sum", "inst": "smsp__inst_executed.sum",
     "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
     "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
     "threads_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
     "registers": "launch__registers_per_thread", "occ_limit_regs": "launch__occupancy_limit_registers",
     "occ_limit_smem": "launch__occupancy_limit_shared_mem",
     "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"}
res = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0]
    if want and not any(w in name for w in want):
        continue
    e = {k: val(d, v) for k, v in M.items() if d.get(v) not in (None, "", "n/a")}
    e["dram_bytes_per_launch"] = val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for k, v in d.items()
          if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued") and v not in ("", "n/a")}
    tot = sum(st.values()) or 1.0
    e["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:5]}
    e["source"] = rep.split("/")[-1]
    res.setdefault(name, e)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1)[:3000])
