"""Per-tile forward CTA durations (globaltimer, debug flag 2) vs list length at config 3: is the
kernel bound by its longest tiles?"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200 import _native
g = ts.build_grid(128); f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
cam = ts.orbit_camera(0, 8, width=1024, height=1024)
act = ts.prefilter(g, f, 100.0); sc = ts.build_scene(g, f, cam, 100.0, active=act); b = ts.bin_and_sort(sc, cam)
L = _native.lib()
for flags in (2,):
    L.ts_debug_set_flags(flags)
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); m, sv = ts.render_forward(sc, b, cam, save_state=True); e1.record(); torch.cuda.synchronize()
    T = b.num_tiles
    t2 = (ctypes.c_uint64 * (2 * T))(); smv = (ctypes.c_uint32 * T)()
    L.ts_debug_tile_times(t2, smv, T)
    t = np.array(t2, dtype=np.float64).reshape(T, 2); sm = np.array(smv)
    lens = np.diff(b.starts.cpu().numpy())
    busy = lens > 0
    t0 = t[:, 0].min()
    dur = (t[:, 1] - t[:, 0]) / 1e3
    print(f"flags={flags} kernel {e0.elapsed_time(e1):.3f} ms  span {(t[:,1].max()-t0)/1e6:.3f} ms; busy tiles {busy.sum()}")
    order = np.argsort(-dur)
    for i in order[:6]:
        print(f"  tile {i} L={lens[i]} dur {dur[i]:.1f} us start {(t[i,0]-t0)/1e3:.1f} us sm {sm[i]}")
    per_chunk = dur[busy] / np.maximum(1, lens[busy] / 32)
    print(f"  us per 32 entries: median {np.median(per_chunk):.2f} p90 {np.percentile(per_chunk, 90):.2f}; "
          f"sum(dur busy) {dur[busy].sum()/1e3:.1f} ms over {len(np.unique(sm))} SMs")
    # SM load: sum of CTA durations per SM
    load = np.zeros(sm.max() + 1)
    np.add.at(load, sm[busy], dur[busy])
    print(f"  per-SM busy sum: max {load.max()/1e3:.3f} ms mean {load.mean()/1e3:.3f} ms")
L.ts_debug_set_flags(0)
