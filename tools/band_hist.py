"""How far inside their error bounds the FP64 re-decided pairs of one config-3 view lie
(debug flag 64): histograms of |f_prev - f_next| / ftol (alpha) and |edge| / band (edges)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200 import _native
R = int(os.environ.get("R", 128)); S = int(os.environ.get("S", 1024)); s = float(os.environ.get("SS", 100))
g = ts.build_grid(R)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
L = _native.lib()
for vi in (0, 3):
    cam = ts.orbit_camera(vi, 8, width=S, height=S)
    act = ts.prefilter(g, f, s)
    sc = ts.build_scene(g, f, cam, s, active=act)
    b = ts.bin_and_sort(sc, cam)
    h = (ctypes.c_uint64 * 32)()
    L.ts_debug_hist(h, 1)
    _native.debug_counters(True)
    _native.check(L.ts_debug_set_flags(64))
    ts.render_forward(sc, b, cam, save_state=True)
    torch.cuda.synchronize()
    _native.check(L.ts_debug_set_flags(0))
    L.ts_debug_hist(h, 1)
    c = _native.debug_counters(True)
    print(f"view {vi}: edge re-decisions {c[0]}, alpha re-decisions {c[1]}")
    print("  alpha |dfl|/ftol in [2^-(b+1), 2^-b):", [int(h[i]) for i in range(16)])
    print("  edge  |e|/band   in [2^-(b+1), 2^-b):", [int(h[16 + i]) for i in range(16)])
