"""The reference-side binding (paper_2406_01579_b200.refbackend): the
reference's render_forward / render_backward called on reference-layout host objects (the
oracle's mirror types, same field names as tetsplat's) run on the B200 kernels and match the
CPU reference (maps <= 1e-4, vertex gradients <= 1e-3 relative, gradcheck.py:136-137)."""
import numpy as np
import pytest

from conftest import RENDER_CASES, load_golden, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rb():
    from paper_2406_01579_b200 import _native, refbackend
    _native.lib()
    return refbackend


@pytest.mark.parametrize("case", RENDER_CASES)
def test_reference_objects_in_and_out(rb, case):
    from oracle import ts_oracle as O
    G = load_golden(f"render_{case}.npz")
    R, S, s = int(G["R"]), int(G["S"]), float(G["s"])
    og = O.build_grid(R)
    of = O.FieldState(G["sdf"], G["deform"], O.DEFORM_FRACTION * og.cell_edge)
    cam = O.orbit_camera(int(G["cam_index"]), int(G["cam_count"]), width=S, height=S)
    sc = O.build_scene(og, of, cam, s, active=G["active"])
    bins = O.bin_and_sort(sc, cam)
    maps, saved = rb.render_forward(sc, bins, cam, save_state=True, maps_type=O.RenderMaps)
    assert isinstance(maps, O.RenderMaps)
    ref_maps, ref_saved = O.render_forward(sc, bins, cam, save_state=True)
    for a, b in ((maps.normal, ref_maps.normal), (maps.depth, ref_maps.depth), (maps.opacity, ref_maps.opacity)):
        assert rel_err(a, b) < 1e-4
    dm = O.synthetic_dmaps(S, S)
    gb = rb.render_backward(saved, sc, og, of, cam, dm, grads_type=O.GradientBuffers)
    ref = O.render_backward(ref_saved, sc, og, of, cam, dm)
    assert rel_err(gb.d_sdf, ref.d_sdf) < 1e-3
    assert rel_err(gb.d_deform, ref.d_deform) < 1e-3
    with pytest.raises(ValueError):
        rb.render_backward(None, sc, og, of, cam, dm)


@pytest.mark.parametrize("case", RENDER_CASES)
def test_reference_objects_prefilter_bins_regularizers(rb, case):
    from oracle import ts_oracle as O
    G = load_golden(f"render_{case}.npz")
    R, S, s = int(G["R"]), int(G["S"]), float(G["s"])
    og = O.build_grid(R)
    of = O.FieldState(G["sdf"], G["deform"], O.DEFORM_FRACTION * og.cell_edge)
    cam = O.orbit_camera(int(G["cam_index"]), int(G["cam_count"]), width=S, height=S)
    assert np.array_equal(rb.prefilter(og, of, s), G["active"])
    sc = O.build_scene(og, of, cam, s, active=G["active"])
    ts_, tx, ty, starts, items = rb.bin_and_sort_arrays(sc, cam)
    ob = O.bin_and_sort(sc, cam)
    assert (ts_, tx, ty) == (ob.tile_size, ob.tiles_x, ob.tiles_y)
    assert np.array_equal(starts, ob.starts) and np.array_equal(items, ob.items)
    le, ge = rb.eikonal_loss(og, of, G["active"], grads_type=O.GradientBuffers)
    ln, gn = rb.normal_consistency_loss(og, of, grads_type=O.GradientBuffers)
    assert abs(le - float(G["eik_loss"])) <= 1e-9 * max(1.0, abs(float(G["eik_loss"])))
    assert abs(ln - float(G["nc_loss"])) <= 1e-9 * max(1.0, abs(float(G["nc_loss"])))
    assert rel_err(ge.d_sdf, G["eik_d_sdf"]) < 1e-6 and rel_err(gn.d_deform, G["nc_d_deform"]) < 1e-6


def test_reference_objects_marching_tetrahedra(rb):
    from oracle import ts_oracle as O
    G = load_golden("mt.npz")
    og = O.build_grid(16)
    of = O.FieldState(G["r16_noisy_sdf"], G["r16_noisy_deform"], O.DEFORM_FRACTION * og.cell_edge)
    V, F = rb.marching_tetrahedra(og, of)
    assert np.array_equal(V, G["r16_noisy_V"]) and np.array_equal(F, G["r16_noisy_F"])
