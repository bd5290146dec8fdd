"""GPU timeline of one config-3 fit step (torch.profiler/CUPTI): busy time, largest idle
gaps and per-kernel totals.  Dev tool."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200.batch import FitStep, StepConfig

R, S, s, V = 128, 1024, 100.0, 8
g = ts.build_grid(R)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
cams = [ts.orbit_camera(i, V, width=S, height=S) for i in range(V)]
gen = torch.Generator(device="cuda").manual_seed(1)
dm = [ts.RenderMaps(torch.randn((S, S, 3), device="cuda", generator=gen), torch.randn((S, S), device="cuda", generator=gen),
                    torch.randn((S, S), device="cuda", generator=gen)) for _ in range(V)]
step = FitStep(g, f, cams, StepConfig())
for _ in range(3):
    step(s, range(V), lambda vi, m: dm[vi])
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step(s, range(V), lambda vi, m: dm[vi])
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type is not None and str(e.device_type).endswith("CUDA")]
ks = sorted([(e.time_range.start, e.time_range.end, e.name) for e in evs], key=lambda x: x[0])
t0, t1 = ks[0][0], max(k[1] for k in ks)
busy, cur_s, cur_e = 0.0, ks[0][0], ks[0][1]
gaps = []
for a, b, n in ks[1:]:
    if a > cur_e:
        busy += cur_e - cur_s
        gaps.append((a - cur_e, cur_e, n))
        cur_s, cur_e = a, b
    else:
        cur_e = max(cur_e, b)
busy += cur_e - cur_s
print(f"span {(t1 - t0)/1e3:.2f} ms, GPU busy {busy/1e3:.2f} ms, idle {(t1 - t0 - busy)/1e3:.2f} ms, kernels {len(ks)}")
gaps.sort(reverse=True)
for d, at, n in gaps[:15]:
    print(f"  gap {d/1e3:.3f} ms at {(at - t0)/1e3:.2f} ms before {n[:70]}")
tot = {}
for a, b, n in ks:
    k = n.split("(")[0][:60]
    tot[k] = tot.get(k, 0.0) + (b - a)
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:20]:
    print(f"  {v/1e3:8.3f} ms  {k}")

# concurrency sweep: time with 0 / 1 / 2+ kernels running, and per kernel the time it ran alone
pts = []
for a, b, n in ks:
    pts.append((a, 1, n))
    pts.append((b, -1, n))
pts.sort(key=lambda x: (x[0], x[1]))
active, last, lvl = {}, pts[0][0], {0: 0.0, 1: 0.0, 2: 0.0}
alone = {}
for tt, d, n in pts:
    c = sum(active.values())
    dt = tt - last
    lvl[min(c, 2)] += dt
    if c == 1:
        only = next(k for k, v in active.items() if v > 0)
        alone[only] = alone.get(only, 0.0) + dt
    k = n.split("(")[0][:60]
    active[k] = active.get(k, 0) + d
    last = tt
print(f"time with 0 / 1 / 2+ kernels: {lvl[0]/1e3:.2f} / {lvl[1]/1e3:.2f} / {lvl[2]/1e3:.2f} ms")
for k, v in sorted(alone.items(), key=lambda x: -x[1])[:12]:
    print(f"  alone {v/1e3:8.3f} ms  {k}")
