"""Marching Tetrahedra at R^3 (default 256, sphere r=0.5): CUDA-event time of the API call
(mesh readback included), median of 3 after one warm-up — the command profiled for MT."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_01579_b200 as ts
R = int(os.environ.get("R", 256))
g = ts.build_grid(R)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
ms = []
for r in range(int(os.environ.get("REPS", 3)) + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    m = ts.marching_tetrahedra(g, f)
    e1.record()
    e1.synchronize()
    if r:
        ms.append(e0.elapsed_time(e1))
print(f"MT R={R}: {sorted(ms)[len(ms) // 2]:.3f} ms  V={m.vertices.shape[0]} F={m.triangles.shape[0]}")
