"""The sync-free per-view path (workspace.cu view_forward_dyn, batch.FitStep sync_free): no
host round trip per view, capacities from the sizes seen, device-side counts, overflow
detection and re-run.  Results must equal the sizing path's."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ts():
    import paper_2406_01579_b200 as ts
    from paper_2406_01579_b200 import _native
    _native.lib()
    return ts


def _problem(ts, R=32, S=256, V=4):
    from oracle import ts_oracle as O
    og = O.build_grid(R)
    of = O.noisy_field(og, noise=0.05, deform=0.3, seed=4)
    g = ts.build_grid(R)
    f = ts.FieldState.from_numpy(of.sdf, of.deformation, ts.deform_limit_for(g))
    cams = [ts.orbit_camera(i, V, width=S, height=S) for i in range(V)]
    gen = torch.Generator(device="cuda").manual_seed(9)
    dms = [ts.RenderMaps(torch.randn((S, S, 3), device="cuda", generator=gen),
                         torch.randn((S, S), device="cuda", generator=gen),
                         torch.randn((S, S), device="cuda", generator=gen)) for _ in range(V)]
    return g, f, cams, dms


def test_view_renderer_caps_equal_sizing_path(ts):
    from paper_2406_01579_b200.view import ViewRenderer
    g, f, cams, dms = _problem(ts)
    s = 100.0
    act = ts.prefilter(g, f, s)
    a, b = ViewRenderer(), ViewRenderer()
    ma = a.forward(g, f, cams[1], s, act)
    K, M, P = a.counts
    ga = a.backward(f, dms[1], ts.GradientBuffers.zeros(g.num_vertices))
    L = a.max_list
    out, out2 = torch.zeros(5, dtype=torch.int64, device="cuda"), torch.zeros(5, dtype=torch.int64, device="cuda")
    b.set_caps(M + 10, P + 10, L, out2)
    mb = b.forward(g, f, cams[1], s, act)
    assert b.counts == (-1, -1, -1)
    gb = b.backward(f, dms[1], ts.GradientBuffers.zeros(g.num_vertices))
    b.collect(out)
    assert out.tolist() == [K, M, P, L, 0] and out2.tolist() == [K, M, P, L, 0]
    for x, y in ((ma.normal, mb.normal), (ma.depth, mb.depth), (ma.opacity, mb.opacity)):
        assert torch.equal(x, y)
    assert torch.allclose(ga.d_vert, gb.d_vert, rtol=1e-6, atol=1e-6 * float(ga.d_vert.abs().max()))
    # a capacity one short of the need overflows: the flag is raised, the maps are not written
    b.set_caps(M - 1, P + 10)
    b.forward(g, f, cams[1], s, act)
    status = torch.zeros(4, device="cuda")
    b.collect(out, status)
    assert out.tolist()[4] == 1 and out.tolist()[1] == M and float(status[2]) == 1.0
    b.backward(f, dms[1], ts.GradientBuffers.zeros(g.num_vertices), status=status)  # flags it too
    assert float(status[2]) == 2.0
    b.set_caps(M + 10, P - 1)
    b.forward(g, f, cams[1], s, act)
    b.collect(out)
    assert out.tolist()[4] == 1 and out.tolist()[2] == P
    b.set_caps(M + 10, P + 10, L - 1)  # the longest list over its capacity
    b.forward(g, f, cams[1], s, act)
    b.collect(out)
    assert out.tolist()[4] == 1 and out.tolist()[3] == L


def test_fitstep_sync_free_equals_threaded(ts):
    """Three steps each (sizing step, then sync-free), Adam included; one step is forced to
    overflow (capacities shrunk) and must be re-run transparently."""
    from paper_2406_01579_b200.batch import FitStep, StepConfig, StepStats
    out = {}
    for mode in ("threaded", "sync_free"):
        g, f, cams, dms = _problem(ts)
        step = FitStep(g, f, cams, StepConfig(sync_free=mode == "sync_free"))
        grads = []
        for it in range(3):
            if mode == "sync_free" and it == 2:
                step._sizes = {vi: (m // 2, p // 2, l // 2) for vi, (m, p, l) in step._sizes.items()}
            st = StepStats()
            gr = step(100.0, range(4), lambda vi, m: dms[vi], st)
            torch.cuda.synchronize()
            step.check_status()
            grads.append(gr.d_vert.clone())
            assert st.views == 4 and all(k > 0 for k in st.splats)
            if it == 0:
                # the view sizes of the first step (same field in both modes: the FP32-atomic
                # gradients make the later fields differ in the last bits, which can move a
                # splat across a tile boundary)
                counts = dict(step.view_counts)
        out[mode] = (grads, f.sdf.clone(), step.opt.t, counts)
    (ga, sa, ta, ca), (gb, sb, tb, cb) = out["threaded"], out["sync_free"]
    assert ta == tb == 3
    assert ca == cb
    for x, y in zip(ga, gb):
        assert torch.allclose(x, y, rtol=1e-5, atol=1e-5 * float(x.abs().max()))
    assert float((sa - sb).abs().max()) < 1e-4


def test_sync_free_grows_capacities_when_the_workload_grows(ts):
    """Capacities learned at s = 100 overflow at s = 20 (more splats, pairs and longer lists):
    the step is re-run transparently with grown capacities and equals the sizing path."""
    from paper_2406_01579_b200.batch import FitStep, StepConfig
    res = {}
    for sf in (False, True):
        g, f, cams, dms = _problem(ts, R=48, S=384, V=4)
        step = FitStep(g, f, cams, StepConfig(sync_free=sf, optimizer=False))
        step(100.0, range(4), lambda vi, m: dms[vi])  # sizes learned at s = 100
        gr = step(20.0, range(4), lambda vi, m: dms[vi]).d_vert.clone()
        torch.cuda.synchronize()
        step.check_status()
        res[sf] = (gr, dict(step.view_counts))
    (ga, ca), (gb, cb) = res[False], res[True]
    assert ca == cb
    assert torch.allclose(ga, gb, rtol=1e-5, atol=1e-5 * float(ga.abs().max()))
