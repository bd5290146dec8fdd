"""Stage timing probe at BASELINE config 3 (128^3, 1024^2, s=100, 8 views). Dev tool."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200.batch import FitStep, StepConfig, StepStats

R = int(os.environ.get("R", 128)); S = int(os.environ.get("S", 1024)); s = float(os.environ.get("SS", 100)); V = 8
g = ts.build_grid(R)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
cams = [ts.orbit_camera(i, V, width=S, height=S) for i in range(V)]
gen = torch.Generator(device="cuda").manual_seed(1)
dmaps = [ts.RenderMaps(torch.randn((S, S, 3), device="cuda", generator=gen), torch.randn((S, S), device="cuda", generator=gen),
                       torch.randn((S, S), device="cuda", generator=gen)) for _ in range(V)]
def ev(): return torch.cuda.Event(enable_timing=True)
# per-stage timing for view 0
for rep in range(3):
    e = [ev() for _ in range(8)]
    e[0].record(); act = ts.prefilter(g, f, s); e[1].record()
    sc = ts.build_scene(g, f, cams[0], s, active=act); e[2].record()
    b = ts.bin_and_sort(sc, cams[0]); e[3].record()
    from paper_2406_01579_b200 import _native
    _native.debug_counters(True)
    maps, sv = ts.render_forward(sc, b, cams[0], save_state=True); e[4].record()
    torch.cuda.synchronize(); print("fwd fallbacks (edge, alpha):", _native.debug_counters(True), "blends", int(sv.n_blend.sum()))
    gb = ts.render_backward(sv, sc, g, f, cams[0], dmaps[0]); e[5].record()
    le, ge = ts.eikonal_loss(g, f, act, out=gb, scale=1000.0); e[6].record()
    ln, gn = ts.normal_consistency_loss(g, f, out=gb, scale=1000.0); e[7].record()
    torch.cuda.synchronize()
    names = ["prefilter", "scene", "bin", "forward", "backward", "eikonal", "nc"]
    print("rep", rep, "K_a", act.numel(), "K_v", len(sc), "M", b.num_pairs, "maxL", b.max_len, "nonmono", int(b.nonmono.sum()),
          " | ".join(f"{n} {e[i].elapsed_time(e[i+1]):.3f}ms" for i, n in enumerate(names)))
step = FitStep(g, f, cams, StepConfig(optimizer=False))
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    a = ev(); bb = ev(); a.record()
    st = StepStats()
    step(s, range(V), lambda vi, m: dmaps[vi], st)
    bb.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(bb)
    print(f"step {rep}: {ms:.2f} ms  wall {1e3*(time.perf_counter()-t0):.2f} ms -> {V/ms*1e3:.1f} views/s; splats {st.splats[:2]} pairs {st.pairs[:2]}")
