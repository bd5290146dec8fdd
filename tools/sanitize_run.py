"""One small pass over every kernel of the library for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): config-1-sized inputs (R=12..16, 96-128 px), the fine-grained API
(plain, colour, reordering window), the fused view path (sizing and sync-free), the
warp-specialised forward, the regularizers, Adam, Marching Tetrahedra, the plugin's records /
backward_tiles, the mesh z-buffer.  Used by profiles/r02_sanitizer_*.log."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200 import _native
from paper_2406_01579_b200.view import ViewRenderer
from paper_2406_01579_b200.batch import FitStep, StepConfig
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import load_golden

_native.lib()
R, S, s = 12, 96, 100.0
g = ts.build_grid(R)
rng = np.random.default_rng(0)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
f.sdf += torch.as_tensor(0.05 * rng.normal(size=g.num_vertices), device="cuda")
f.deformation.copy_(torch.as_tensor(rng.uniform(-0.3, 0.3, size=(g.num_vertices, 3)) * f.deform_limit, device="cuda"))
cams = [ts.orbit_camera(i, 4, width=S, height=S) for i in range(4)]
gen = torch.Generator(device="cuda").manual_seed(1)
dm = ts.RenderMaps(torch.randn((S, S, 3), device="cuda", generator=gen), torch.randn((S, S), device="cuda", generator=gen),
                   torch.randn((S, S), device="cuda", generator=gen), torch.randn((S, S, 3), device="cuda", generator=gen))
colors = torch.rand((g.num_tets, 3), device="cuda", generator=gen)
act = ts.prefilter(g, f, s)
for flags in (0,):
    _native.check(_native.lib().ts_debug_set_flags(flags))
    for col in (None, colors):
        sc = ts.build_scene(g, f, cams[1], s, active=act, colors=col)
        b = ts.bin_and_sort(sc, cams[1])
        maps, sv = ts.render_forward(sc, b, cams[1], save_state=True)
        ts.render_backward(sv, sc, g, f, cams[1], dm if col is not None else ts.RenderMaps(dm.normal, dm.depth, dm.opacity))
        ts.render_reference(sc, cams[1])
_native.check(_native.lib().ts_debug_set_flags(0))
# reordering window
G = load_golden("window_noisy_r16_s100_cam3.npz")
g16 = ts.build_grid(16)
f16 = ts.FieldState.from_numpy(G["sdf"], G["deform"], ts.deform_limit_for(g16))
c16 = ts.orbit_camera(3, 8, width=128, height=128)
sc = ts.scene_from_arrays(G["tet_ids"], G["vert_ids"], G["proj"], G["depths"], G["f"], G["normals"], G["mean_depth"],
                          G["alpha_max"], G["bbox"], 100.0, c16)
b = ts.bin_and_sort(sc, c16)
for nw in (1, 5, 1 << 30):
    m, sv = ts.render_forward(sc, b, c16, n_w=nw, save_state=True)
    ts.render_backward(sv, sc, g16, f16, c16, ts.RenderMaps(*(torch.as_tensor(G[k]).cuda() for k in ("d_normal", "d_depth", "d_opacity"))))
# fused path, sizing and sync-free, Adam, regularizers
for sf in (False, True):
    fs2 = f.copy()
    step = FitStep(g, fs2, cams, StepConfig(sync_free=sf, inflight=2))
    for _ in range(2):
        step(s, range(4), lambda vi, mm: ts.RenderMaps(dm.normal, dm.depth, dm.opacity))
vr = ViewRenderer()
vr.forward(g, f, cams[2], s, act, colors=colors)
vr.backward(f, dm, ts.GradientBuffers.zeros(g.num_vertices, num_tets_color=g.num_tets))
ts.eikonal_loss(g, f, act)
ts.normal_consistency_loss(g, f)
# Marching Tetrahedra
ts.marching_tetrahedra(g, f)
# plugin records / backward_tiles
from oracle import ts_oracle as O
from paper_2406_01579_b200 import kernels
osc = O.SplatScene(*(t.detach().cpu().numpy() for t in (sc.tet_ids, sc.vert_ids, sc.proj, sc.depths, sc.f, sc.normals,
                                                         sc.mean_depth, sc.alpha_max, sc.bbox)), 100.0, None)
ob = O.bin_and_sort(osc, O.orbit_camera(3, 8, width=128, height=128))
real = O._load_ref()
O._REF = kernels
om, osv = O.render_forward(osc, ob, O.orbit_camera(3, 8, width=128, height=128), save_state=True, backend="ref")
O.splat_gradients(osv, osc, O.orbit_camera(3, 8, width=128, height=128), O.synthetic_dmaps(128, 128), backend="ref")
O._REF = real
# mesh z-buffer
mesh = ts.marching_tetrahedra(g, f)
ts.rasterize_mesh(mesh, cams[0])
torch.cuda.synchronize()
print("sanitize run ok")
