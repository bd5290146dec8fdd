"""Per-step wall times of the fit step at a given resolution / image (R, S env) and lanes
(TS_INFLIGHT), with the slowest view-call durations of the slowest step (stall hunting)."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200 import view as view_mod
from paper_2406_01579_b200.batch import FitStep, StepConfig
R = int(os.environ.get("R", 256)); S = int(os.environ.get("S", 2048)); V = 8
n = int(os.environ["TS_INFLIGHT"]) if "TS_INFLIGHT" in os.environ else None
g = ts.build_grid(R)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
cams = [ts.orbit_camera(i, V, width=S, height=S) for i in range(V)]
gen = torch.Generator(device="cuda").manual_seed(1)
dm = [ts.RenderMaps(torch.randn((S, S, 3), device="cuda", generator=gen), torch.randn((S, S), device="cuda", generator=gen),
                    torch.randn((S, S), device="cuda", generator=gen)) for _ in range(V)]
log, lock = [], threading.Lock()
orig_fwd, orig_bwd = view_mod.ViewRenderer.forward, view_mod.ViewRenderer.backward
def fwd(self, *a, **k):
    t0 = time.perf_counter(); r = orig_fwd(self, *a, **k)
    with lock: log.append(("fwd", time.perf_counter() - t0))
    return r
def bwd(self, *a, **k):
    t0 = time.perf_counter(); r = orig_bwd(self, *a, **k)
    with lock: log.append(("bwd", time.perf_counter() - t0))
    return r
view_mod.ViewRenderer.forward, view_mod.ViewRenderer.backward = fwd, bwd
step = FitStep(g, f, cams, StepConfig(inflight=n))
sdf0, def0 = f.sdf.clone(), f.deformation.clone()
import gc
if os.environ.get("NOGC"):
    gc.collect(); gc.freeze(); gc.disable()
for k in range(int(os.environ.get("STEPS", 10))):
    f.sdf.copy_(sdf0); f.deformation.copy_(def0)
    torch.cuda.synchronize(); log.clear(); t0 = time.perf_counter()
    step(100.0, range(V), lambda vi, m: dm[vi])
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    worst = sorted(log, key=lambda x: -x[1])[:3]
    print(k, f"{t * 1e3:.1f} ms", " ".join(f"{a}:{b * 1e3:.1f}" for a, b in worst), flush=True)
