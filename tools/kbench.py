"""Compositing-kernel timing harness: config-3 views through the fine-grained API, CUDA events
around the forward / backward launches (median of REPS), plus the fused view path per view."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200.view import ViewRenderer
R = int(os.environ.get("R", 128)); S = int(os.environ.get("S", 1024)); s = float(os.environ.get("SS", 100))
REPS = int(os.environ.get("REPS", 10))
views = [int(v) for v in os.environ.get("VIEWS", "0,3").split(",")]
g = ts.build_grid(R)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
gen = torch.Generator(device="cuda").manual_seed(1)
dm = ts.RenderMaps(torch.randn((S, S, 3), device="cuda", generator=gen), torch.randn((S, S), device="cuda", generator=gen),
                   torch.randn((S, S), device="cuda", generator=gen))
act = ts.prefilter(g, f, s)
from paper_2406_01579_b200 import _native
_native.check(_native.lib().ts_debug_set_flags(int(os.environ.get("FLAGS", "0"))))
tot_f = tot_b = tot_v = 0.0
for vi in views:
    cam = ts.orbit_camera(vi, 8, width=S, height=S)
    sc = ts.build_scene(g, f, cam, s, active=act)
    b = ts.bin_and_sort(sc, cam)
    tf, tb = [], []
    for _ in range(REPS):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        maps, sv = ts.render_forward(sc, b, cam, save_state=True, timing=(e[0], e[1]))
        gb = ts.render_backward(sv, sc, g, f, cam, dm, timing=(e[2], e[3]))
        torch.cuda.synchronize()
        tf.append(e[0].elapsed_time(e[1]))
        tb.append(e[2].elapsed_time(e[3]))
    vr = ViewRenderer()
    out = ts.GradientBuffers.zeros(g.num_vertices)
    tv = []
    for _ in range(REPS):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m2 = vr.forward(g, f, cam, s, act)
        vr.backward(f, dm, out)
        e1.record()
        torch.cuda.synchronize()
        tv.append(e0.elapsed_time(e1))
    mf, mb, mv = np.median(tf), np.median(tb), np.median(tv)
    tot_f += mf; tot_b += mb; tot_v += mv
    print(f"view {vi}: K={len(sc)} M={b.num_pairs} forward {mf:.3f} ms backward {mb:.3f} ms  fused view {mv:.3f} ms "
          f"(sum|maps| {float(maps.opacity.sum()):.4f} sum|grad| {float(gb.d_vert.abs().sum()):.4f})", flush=True)
n = len(views)
print(f"MEAN forward {tot_f / n:.3f} backward {tot_b / n:.3f} fused-view {tot_v / n:.3f} ms")
