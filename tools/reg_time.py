"""Device time of the per-batch regularizers (eikonal over the active set, normal consistency)
at config 3 (128^3), CUDA events on the launching stream, mean of 20 after warm-up."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200.losses import eikonal_loss_async, normal_consistency_loss_async, nc_scratch_bytes
R = int(os.environ.get("R", 128))
g = ts.build_grid(R)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
act = ts.prefilter(g, f, 100.0)
gb = ts.GradientBuffers.zeros(g.num_vertices)
loss = torch.zeros(1, dtype=torch.float64, device="cuda")
scr = torch.empty(nc_scratch_bytes(g), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for name, fn in (("eikonal", lambda: eikonal_loss_async(g, f, act, gb, 1000.0, loss, st)),
                 ("normal_consistency", lambda: normal_consistency_loss_async(g, f, gb, 1000.0, loss, st, scr))):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 20:.3f} ms")
