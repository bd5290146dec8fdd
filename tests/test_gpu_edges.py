"""GPU edge cases the reference handles without special-casing (raster.py:104-177,
206-250, splat.py:203-245): a field with no surface (prefilter keeps nothing), a camera
whose far plane culls every splat (K_v = 0, M = 0), and a camera that sees only part of
the grid.  Each runs through the same API the parity tests use and is checked against the
CPU oracle on identical inputs: empty sets / zero maps / zero gradients bit for bit, maps
and gradients at the usual bars otherwise.
"""
import numpy as np
import pytest
import torch

from conftest import rel_err

pytestmark = pytest.mark.gpu

S = 64
STEEP = 100.0


@pytest.fixture(scope="module")
def ts():
    import paper_2406_01579_b200 as ts
    from paper_2406_01579_b200 import _native
    _native.lib()
    return ts


def _pair(ts, R, sdf, far=10.0, fov=40.0):
    from oracle import ts_oracle as O
    sdf = np.ascontiguousarray(sdf, dtype=np.float64)
    g = ts.build_grid(R)
    og = O.build_grid(R)
    deform = np.zeros((len(sdf), 3))
    fs = ts.FieldState.from_numpy(sdf, deform, ts.deform_limit_for(g))
    ofs = O.FieldState(sdf, deform, O.DEFORM_FRACTION * og.cell_edge)
    cam = ts.orbit_camera(0, 8, width=S, height=S, far=far, fov_deg=fov)
    ocam = O.orbit_camera(0, 8, width=S, height=S, far=far, fov_deg=fov)
    return O, g, og, fs, ofs, cam, ocam


def _sphere_sdf(O, R, radius=0.5):
    return O.init_sphere_field(O.build_grid(R), radius).sdf


def test_field_without_surface(ts):
    R = 8
    from oracle import ts_oracle as O
    n = (R + 1) ** 3
    O, g, og, fs, ofs, cam, ocam = _pair(ts, R, np.full(n, 0.5))
    active = ts.prefilter(g, fs, STEEP)
    assert active.numel() == 0 and len(O.prefilter(og, ofs, STEEP)) == 0
    sc = ts.build_scene(g, fs, cam, STEEP, active=active)
    assert len(sc) == 0
    b = ts.bin_and_sort(sc, cam)
    assert b.num_pairs == 0 and int(b.starts[-1]) == 0
    maps, saved = ts.render_forward(sc, b, cam, save_state=True)
    assert float(maps.opacity.abs().max()) == 0.0 and float(maps.depth.abs().max()) == 0.0
    w = O.synthetic_dmaps(S, S)
    gb = ts.render_backward(saved, sc, g, fs, cam, ts.RenderMaps(w.normal, w.depth, w.opacity))
    assert float(gb.d_vert.abs().max()) == 0.0
    # the fit path's filter reports the reference's EmptySceneError (splat.py:101, fit.py:167)
    with pytest.raises(ts.EmptySceneError):
        ts.coarse_to_fine_filter(g, fs, STEEP)


def test_far_plane_culls_everything(ts):
    R = 12
    from oracle import ts_oracle as O
    O, g, og, fs, ofs, cam, ocam = _pair(ts, R, _sphere_sdf(O, R), far=0.5)
    active = ts.prefilter(g, fs, STEEP)
    oa = O.prefilter(og, ofs, STEEP)
    assert np.array_equal(active.cpu().numpy(), oa) and len(oa) > 0
    sc = ts.build_scene(g, fs, cam, STEEP, active=active)
    osc = O.build_scene(og, ofs, ocam, STEEP, active=oa)
    assert len(sc) == 0 and len(osc.tet_ids) == 0
    b = ts.bin_and_sort(sc, cam)
    assert b.num_pairs == 0
    maps, saved = ts.render_forward(sc, b, cam, save_state=True)
    assert float(maps.opacity.abs().max()) == 0.0
    w = O.synthetic_dmaps(S, S)
    gb = ts.render_backward(saved, sc, g, fs, cam, ts.RenderMaps(w.normal, w.depth, w.opacity))
    assert float(gb.d_vert.abs().max()) == 0.0
    # the fused single-call view path agrees on the empty view
    from paper_2406_01579_b200.view import ViewRenderer
    vr = ViewRenderer()
    m2 = vr.forward(g, fs, cam, STEEP, active)
    assert vr.counts[0] == 0 and vr.counts[1] == 0
    assert float(m2.opacity.abs().max()) == 0.0
    dmd = ts.RenderMaps(*(torch.as_tensor(x, dtype=torch.float32, device="cuda").contiguous()
                          for x in (w.normal, w.depth, w.opacity)))
    gb2 = vr.backward(fs, dmd, ts.GradientBuffers.zeros(g.num_vertices))
    assert float(gb2.d_vert.abs().max()) == 0.0


def test_partially_visible_grid(ts):
    """A narrow field of view leaves most splats outside the image: culling, tile clipping
    at the image border and ragged tile lists, against the oracle."""
    R = 16
    from oracle import ts_oracle as O
    O, g, og, fs, ofs, cam, ocam = _pair(ts, R, _sphere_sdf(O, R, 0.6), fov=12.0)
    active = ts.prefilter(g, fs, STEEP)
    oa = O.prefilter(og, ofs, STEEP)
    assert np.array_equal(active.cpu().numpy(), oa)
    osc = O.build_scene(og, ofs, ocam, STEEP, active=oa)
    ob = O.bin_and_sort(osc, ocam)
    om, osv = O.render_forward(osc, ob, ocam, save_state=True)
    # stage parity on the oracle's FP64 scene: bins bitwise
    sc0 = ts.scene_from_arrays(osc.tet_ids, osc.vert_ids, osc.proj, osc.depths, osc.f, osc.normals,
                               osc.mean_depth, osc.alpha_max, osc.bbox, STEEP, cam)
    b0 = ts.bin_and_sort(sc0, cam)
    assert np.array_equal(b0.starts.cpu().numpy(), ob.starts)
    assert np.array_equal(b0.items.cpu().numpy(), ob.items)
    assert 0 < len(osc.tet_ids) < len(oa)
    # end to end from the field
    sc = ts.build_scene(g, fs, cam, STEEP, active=active)
    b = ts.bin_and_sort(sc, cam)
    maps, saved = ts.render_forward(sc, b, cam, save_state=True)
    n, d, o, _ = maps.numpy()
    assert rel_err(n, om.normal) < 1e-4 and rel_err(d, om.depth) < 1e-4 and rel_err(o, om.opacity) < 1e-4
    w = O.synthetic_dmaps(S, S)
    gb = ts.render_backward(saved, sc, g, fs, cam, ts.RenderMaps(w.normal, w.depth, w.opacity))
    ogb = O.render_backward(osv, osc, og, ofs, ocam, w)
    assert rel_err(gb.d_sdf.cpu().numpy(), ogb.d_sdf) < 1e-3
    assert rel_err(gb.d_deform.cpu().numpy(), ogb.d_deform) < 1e-3


def test_fused_path_rejects_non_finite_map_gradients():
    """raster.py:209-211 on the fused path: a NaN in dL/dmaps is flagged on the device, the Adam
    update is skipped (the field stays intact, like the reference, which raises before
    opt.step), and check_status raises ValueError at the next sync."""
    import paper_2406_01579_b200 as ts
    from paper_2406_01579_b200.batch import FitStep, StepConfig
    g = ts.build_grid(16)
    f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
    cams = [ts.orbit_camera(i, 2, width=64, height=64) for i in range(2)]
    sdf0, def0 = f.sdf.clone(), f.deformation.clone()

    def dfn(vi, maps):
        d = ts.RenderMaps.zeros(64, 64)
        if vi == 1:
            d.depth[10, 20] = float("nan")
        return d

    step = FitStep(g, f, cams, StepConfig())
    step(100.0, [0, 1], dfn)
    torch.cuda.synchronize()
    with pytest.raises(ValueError):
        step.check_status()
    assert torch.equal(f.sdf, sdf0) and torch.equal(f.deformation, def0)
    # a clean step afterwards runs and updates
    step(100.0, [0, 1], lambda vi, m: ts.RenderMaps.zeros(64, 64))
    torch.cuda.synchronize()
    step.check_status()
    assert not torch.equal(f.sdf, sdf0)  # the regularizers move the field


def test_coarse_to_fine_filter_box_and_second_round():
    """splat.py:88-109 against the reference's fixture: the survivors' AABB and, with a
    positional field function, the second prefilter on the rescaled grid."""
    import numpy as np
    import paper_2406_01579_b200 as ts
    from conftest import load_golden
    G = load_golden("c2f_noisy_r12_s100.npz")
    g = ts.build_grid(int(G["R"]))
    fs = ts.FieldState.from_numpy(G["sdf"], G["deform"], ts.deform_limit_for(g))
    act, box = ts.coarse_to_fine_filter(g, fs, float(G["s"]))
    assert np.array_equal(act.cpu().numpy().astype(np.int64), G["active"])
    assert np.abs(box - G["box"]).max() <= 1e-12
    fn = lambda p: np.linalg.norm(p - np.array([0.05, -0.02, 0.01]), axis=1) - 0.4
    act2, box2 = ts.coarse_to_fine_filter(g, fs, float(G["s"]), field_fn=fn)
    assert np.array_equal(act2.cpu().numpy().astype(np.int64), G["active_fn"])
    assert np.abs(box2 - G["box_fn"]).max() <= 1e-12
