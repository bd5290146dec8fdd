"""One config-3 view (prefilter, scene, bins, forward, backward, regularizers), run `reps`
times: the command profiled by ncu (profiles/)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_01579_b200 as ts
R = int(os.environ.get("R", 128)); S = int(os.environ.get("S", 1024)); s = float(os.environ.get("SS", 100))
reps = int(os.environ.get("REPS", 2))
g = ts.build_grid(R)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
cam = ts.orbit_camera(0, 8, width=S, height=S)
gen = torch.Generator(device="cuda").manual_seed(1)
dm = ts.RenderMaps(torch.randn((S, S, 3), device="cuda", generator=gen), torch.randn((S, S), device="cuda", generator=gen),
                   torch.randn((S, S), device="cuda", generator=gen))
for _ in range(reps):
    act = ts.prefilter(g, f, s)
    sc = ts.build_scene(g, f, cam, s, active=act)
    b = ts.bin_and_sort(sc, cam)
    maps, sv = ts.render_forward(sc, b, cam, save_state=True)
    gb = ts.render_backward(sv, sc, g, f, cam, dm)
    ts.eikonal_loss(g, f, act, out=gb, scale=1000.0)
    ts.normal_consistency_loss(g, f, out=gb, scale=1000.0)
torch.cuda.synchronize()
print("ok", len(sc), b.num_pairs)
