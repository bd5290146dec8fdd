"""Experiment: forward/backward time with and without the exact FP64 re-decisions."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200 import _native
g = ts.build_grid(128); f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
cam = ts.orbit_camera(0, 8, width=1024, height=1024)
dm = ts.RenderMaps(torch.randn((1024, 1024, 3), device="cuda"), torch.randn((1024, 1024), device="cuda"), torch.randn((1024, 1024), device="cuda"))
act = ts.prefilter(g, f, 100.0); sc = ts.build_scene(g, f, cam, 100.0, active=act); b = ts.bin_and_sort(sc, cam)
for flags in (0, 1, 0, 1):
    _native.lib().ts_debug_set_flags(flags)
    for rep in range(3):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(); m, sv = ts.render_forward(sc, b, cam, save_state=True); e[1].record()
        ts.render_backward(sv, sc, g, f, cam, dm); e[2].record(); torch.cuda.synchronize()
    print(f"flags={flags} forward {e[0].elapsed_time(e[1]):.3f} ms backward {e[1].elapsed_time(e[2]):.3f} ms")
_native.lib().ts_debug_set_flags(0)
