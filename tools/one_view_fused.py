"""One config-3 view through the fused view path bench.py times (ViewRenderer: prefilter,
scene, bins, window/pair counts, forward, backward + chain) plus the batch regularizers,
run `reps` times: the command profiled by ncu for profiles/r01_kernel_roofline_fused.txt."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200.view import ViewRenderer
R = int(os.environ.get("R", 128)); S = int(os.environ.get("S", 1024)); s = float(os.environ.get("SS", 100))
reps = int(os.environ.get("REPS", 2))
g = ts.build_grid(R)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
cam = ts.orbit_camera(0, 8, width=S, height=S)
gen = torch.Generator(device="cuda").manual_seed(1)
dm = ts.RenderMaps(torch.randn((S, S, 3), device="cuda", generator=gen), torch.randn((S, S), device="cuda", generator=gen),
                   torch.randn((S, S), device="cuda", generator=gen))
vr = ViewRenderer()
gb = ts.GradientBuffers.zeros(g.num_vertices)
for _ in range(reps):
    act = ts.prefilter(g, f, s)
    vr.forward(g, f, cam, s, act)
    vr.backward(f, dm, gb)
    ts.eikonal_loss(g, f, act, out=gb, scale=1000.0)
    ts.normal_consistency_loss(g, f, out=gb, scale=1000.0)
torch.cuda.synchronize()
print("ok", vr.counts[0], vr.counts[1])
