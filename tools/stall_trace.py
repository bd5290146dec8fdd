"""Profile several fit steps at R=256 / 2048^2 and list the longest CUDA runtime calls and GPU
idle gaps (stall hunting for multi-lane runs)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200.batch import FitStep, StepConfig
R = int(os.environ.get("R", 256)); S = int(os.environ.get("S", 2048)); V = 8
g = ts.build_grid(R)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
cams = [ts.orbit_camera(i, V, width=S, height=S) for i in range(V)]
gen = torch.Generator(device="cuda").manual_seed(1)
dm = [ts.RenderMaps(torch.randn((S, S, 3), device="cuda", generator=gen), torch.randn((S, S), device="cuda", generator=gen),
                    torch.randn((S, S), device="cuda", generator=gen)) for _ in range(V)]
step = FitStep(g, f, cams, StepConfig())
sdf0, def0 = f.sdf.clone(), f.deformation.clone()
for _ in range(2):
    step(100.0, range(V), lambda vi, m: dm[vi])
torch.cuda.synchronize()
times = []
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for k in range(int(os.environ.get("STEPS", 10))):
        f.sdf.copy_(sdf0); f.deformation.copy_(def0)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        step(100.0, range(V), lambda vi, m: dm[vi])
        torch.cuda.synchronize(); times.append((time.perf_counter() - t0) * 1e3)
print("ms/step:", " ".join(f"{t:.0f}" for t in times))
evs = prof.events()
cpu = [e for e in evs if e.device_type is not None and str(e.device_type).endswith("CPU") and e.name.startswith("cuda")]
cpu.sort(key=lambda e: -(e.time_range.end - e.time_range.start))
for e in cpu[:12]:
    print(f"  api {e.name:32s} {(e.time_range.end - e.time_range.start) / 1e3:9.2f} ms")
gpu = sorted([(e.time_range.start, e.time_range.end, e.name) for e in evs
              if e.device_type is not None and str(e.device_type).endswith("CUDA")])
gaps, cur = [], gpu[0][1]
for a, b, n in gpu[1:]:
    if a > cur:
        gaps.append((a - cur, n))
    cur = max(cur, b)
gaps.sort(reverse=True)
for d, n in gaps[:6]:
    print(f"  gpu idle {d / 1e3:8.2f} ms before {n[:60]}")
long = sorted(gpu, key=lambda x: -(x[1] - x[0]))[:6]
for a, b, n in long:
    print(f"  kernel {(b - a) / 1e3:8.2f} ms {n[:70]}")
