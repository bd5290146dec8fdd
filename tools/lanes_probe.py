"""Per-step times of the config-3 fit step for a given number of lanes (TS_INFLIGHT)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200.batch import FitStep, StepConfig
n = int(os.environ.get("TS_INFLIGHT", "2"))
R, S, s, V = 128, 1024, 100.0, 8
g = ts.build_grid(R)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
cams = [ts.orbit_camera(i, V, width=S, height=S) for i in range(V)]
gen = torch.Generator(device="cuda").manual_seed(1)
dm = [ts.RenderMaps(torch.randn((S, S, 3), device="cuda", generator=gen), torch.randn((S, S), device="cuda", generator=gen),
                    torch.randn((S, S), device="cuda", generator=gen)) for _ in range(V)]
step = FitStep(g, f, cams, StepConfig(inflight=n))
sdf0, def0 = f.sdf.clone(), f.deformation.clone()
ts_ = []
for k in range(25):
    f.sdf.copy_(sdf0); f.deformation.copy_(def0)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    step(s, range(V), lambda vi, m: dm[vi])
    torch.cuda.synchronize(); ts_.append((time.perf_counter() - t0) * 1e3)
print(n, "lanes, ms/step:", " ".join(f"{x:.1f}" for x in ts_), "| mem GB", torch.cuda.max_memory_allocated() / 1e9)
