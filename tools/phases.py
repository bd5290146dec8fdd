"""Per-phase cycle split of k_forward / k_backward on one config-3 view (debug flag bit 2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200 import _native
R = int(os.environ.get("R", 128)); S = int(os.environ.get("S", 1024)); s = float(os.environ.get("SS", 100))
g = ts.build_grid(R)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
cam = ts.orbit_camera(0, 8, width=S, height=S)
gen = torch.Generator(device="cuda").manual_seed(1)
dm = ts.RenderMaps(torch.randn((S, S, 3), device="cuda", generator=gen), torch.randn((S, S), device="cuda", generator=gen),
                   torch.randn((S, S), device="cuda", generator=gen))
act = ts.prefilter(g, f, s)
sc = ts.build_scene(g, f, cam, s, active=act)
b = ts.bin_and_sort(sc, cam)
for flags in (0, 8, 4):
    _native.check(_native.lib().ts_debug_set_flags(flags | 16))
    _native.debug_phases(reset=True)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    maps, sv = ts.render_forward(sc, b, cam, save_state=True, timing=(e[0], e[1]))
    gb = ts.render_backward(sv, sc, g, f, cam, dm, timing=(e[2], e[3]))
    torch.cuda.synchronize()
    ph = _native.debug_phases(reset=True)
    print("counters (edge, alpha, evaluated, edge-from-uncertain-det):", _native.debug_counters(reset=True))
    print(f"flags={flags}: forward {e[0].elapsed_time(e[1]):.3f} ms  backward {e[2].elapsed_time(e[3]):.3f} ms")
fw, bw = ph[0:4], ph[8:13]
print(f"forward chunks {ph[4]}, with FP64 re-decisions {ph[5]}, re-decided pairs {ph[6]}, max per chunk {ph[7]}")
print("forward  stage/A/A'/B  :", " ".join(f"{100 * x / max(sum(fw), 1):.1f}%" for x in fw), f"(sum {sum(fw):.3e} cyc)")
print("backward stage/load/B/C/write:", " ".join(f"{100 * x / max(sum(bw), 1):.1f}%" for x in bw), f"(sum {sum(bw):.3e} cyc)")
_native.check(_native.lib().ts_debug_set_flags(0))
