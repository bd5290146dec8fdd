"""The CPU oracle pinned against the golden fixtures generated from the unmodified
reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import RENDER_CASES, load_golden, rel_err
from oracle import ts_oracle as O

BACKENDS = O.available_backends()


def _field(G):
    g = O.build_grid(int(G["R"]))
    return g, O.FieldState(G["sdf"], G["deform"], O.DEFORM_FRACTION * g.cell_edge)


def _cam(G):
    S = int(G["S"])
    return O.orbit_camera(int(G["cam_index"]), int(G["cam_count"]), width=S, height=S)


@pytest.mark.parametrize("R", [1, 2, 3])
def test_grid_matches_reference(R):
    G = load_golden(f"grid_R{R}.npz")
    g = O.build_grid(R)
    assert np.array_equal(g.rest_positions, G["rest"])
    assert np.array_equal(g.tets, G["tets"])
    assert np.array_equal(g.edges, G["edges"])
    h = O.build_grid(R, with_edges=False)  # the edge-free build used for the 256^3 MT check
    assert np.array_equal(h.rest_positions, G["rest"]) and np.array_equal(h.tets, G["tets"])
    assert h.edges.shape == (0, 2)


@pytest.mark.parametrize("case", RENDER_CASES)
def test_prefilter_scene_bins(case):
    G = load_golden(f"render_{case}.npz")
    g, fs = _field(G)
    cam = _cam(G)
    s = float(G["s"])
    active = O.prefilter(g, fs, s)
    assert np.array_equal(active, G["active"])
    sc = O.build_scene(g, fs, cam, s, active=active)
    assert np.array_equal(sc.tet_ids, G["tet_ids"])
    assert np.array_equal(sc.mean_depth, G["mean_depth"])
    b = O.bin_and_sort(sc, cam)
    assert np.array_equal(b.starts, G["starts"])
    assert np.array_equal(b.items, G["items"])


@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("case", [c for c in RENDER_CASES if "cfg1" not in c])
def test_render_and_gradients(case, backend):
    G = load_golden(f"render_{case}.npz")
    g, fs = _field(G)
    cam = _cam(G)
    sc = O.build_scene(g, fs, cam, float(G["s"]), active=G["active"])
    b = O.bin_and_sort(sc, cam)
    maps, saved = O.render_forward(sc, b, cam, save_state=True, backend=backend, want_counts=True)
    assert np.array_equal(saved.counts, G["counts"])
    assert rel_err(maps.normal, G["normal"]) < 1e-12
    assert rel_err(maps.depth, G["depth"]) < 1e-12
    assert rel_err(maps.opacity, G["opacity"]) < 1e-12
    dm = O.RenderMaps(G["d_normal"], G["d_depth"], G["d_opacity"])
    gb = O.render_backward(saved, sc, g, fs, cam, dm, backend=backend)
    assert rel_err(gb.d_sdf, G["d_sdf"]) < 1e-10
    assert rel_err(gb.d_deform, G["d_deform"]) < 1e-10
    ref = O.render_reference(sc, cam, backend=backend)
    assert rel_err(ref.opacity, G["ref_opacity"]) < 1e-12


@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("case", [c for c in RENDER_CASES if "cfg1" not in c])
def test_regularizers(case, backend):
    G = load_golden(f"render_{case}.npz")
    g, fs = _field(G)
    le, ge = O.eikonal_loss(g, fs, G["active"], backend=backend)
    ln, gn = O.normal_consistency_loss(g, fs, backend=backend)
    assert abs(le - float(G["eik_loss"])) <= 1e-12 * abs(float(G["eik_loss"]))
    assert abs(ln - float(G["nc_loss"])) <= 1e-12 * abs(float(G["nc_loss"]))
    assert rel_err(ge.d_sdf, G["eik_d_sdf"]) < 1e-12
    assert rel_err(gn.d_deform, G["nc_d_deform"]) < 1e-12


def test_marching_tetrahedra_matches_reference():
    G = load_golden("mt.npz")
    for tag in ("one_neg", "two_neg"):
        g = O.build_grid(1)
        fs = O.FieldState(G[f"{tag}_sdf"], np.zeros((g.num_vertices, 3)), 0.45 * g.cell_edge)
        V, F = O.marching_tetrahedra(g, fs)
        assert np.array_equal(V, G[f"{tag}_V"]) and np.array_equal(F, G[f"{tag}_F"])
    for tag, R in (("r16", 16), ("r16_noisy", 16), ("r24", 24)):
        g = O.build_grid(R)
        fs = O.FieldState(G[f"{tag}_sdf"], G[f"{tag}_deform"], 0.45 * g.cell_edge)
        V, F = O.marching_tetrahedra(g, fs)
        assert np.array_equal(V, G[f"{tag}_V"]) and np.array_equal(F, G[f"{tag}_F"])


def test_spec_known_answers():
    # SPEC.md:230-232 (exact value; SPEC's 0.01795 is a rounding slip)
    assert O.alpha_max(np.array([0.2, 0.5, 0.3, 0.4]), 20.0)[0] == 0.017941626604998095
    assert O.alpha_max(np.array([1.0, 1.0, 1.0, 1.0]), 7.0)[0] == 0.0
    # window identity on monotone mean depth: forward with n_w=1 and n_w=50 agree bitwise
    G = load_golden("render_sphere_r16_s100.npz")
    g, fs = _field(G)
    cam = _cam(G)
    sc = O.build_scene(g, fs, cam, float(G["s"]), active=G["active"])
    b = O.bin_and_sort(sc, cam)
    m1, _ = O.render_forward(sc, b, cam, n_w=1, backend=BACKENDS[0])
    m2, _ = O.render_forward(sc, b, cam, n_w=50, backend=BACKENDS[0])
    assert np.array_equal(m1.normal, m2.normal)


@pytest.mark.parametrize("backend", BACKENDS)
def test_color_path(backend):
    """Colour compositing and colour gradients (_core.pyx:202-205,219-222,410-413,433-436,
    raster.py:303-305) against the reference's fixture."""
    G = load_golden("color_noisy_r12_s100_cam5.npz")
    g, fs = _field(G)
    cam = _cam(G)
    sc = O.build_scene(g, fs, cam, float(G["s"]), active=G["active"], colors=G["colors"])
    assert np.array_equal(sc.tet_ids, G["tet_ids"])
    b = O.bin_and_sort(sc, cam)
    assert np.array_equal(b.items, G["items"])
    maps, saved = O.render_forward(sc, b, cam, save_state=True, backend=backend, want_counts=True)
    assert np.array_equal(saved.counts, G["counts"])
    for k in ("normal", "depth", "opacity", "color"):
        assert rel_err(getattr(maps, k), G[k]) < 1e-12, k
    dm = O.RenderMaps(G["d_normal"], G["d_depth"], G["d_opacity"], G["d_color"])
    gb = O.render_backward(saved, sc, g, fs, cam, dm, backend=backend)
    assert rel_err(gb.d_sdf, G["d_sdf"]) < 1e-10
    assert rel_err(gb.d_deform, G["d_deform"]) < 1e-10
    assert gb.d_color is not None and rel_err(gb.d_color, G["d_color_tet"]) < 1e-10


def window_scene(G):
    """The oracle SplatScene of the window fixture: the reference's FP64 arrays with the
    fixture's re-keyed mean depths (make_golden.window_depths)."""
    return O.SplatScene(G["tet_ids"], G["vert_ids"], G["proj"], G["depths"], G["f"], G["normals"],
                        G["mean_depth"], G["alpha_max"], G["bbox"], float(G["s"]), None)


@pytest.mark.parametrize("backend", BACKENDS)
def test_window_reorders(backend):
    """The N_w window on lists it actually reorders (_core.pyx:171-187): per-window maps,
    counts and gradients equal the reference's; the windows give different images."""
    G = load_golden("window_noisy_r16_s100_cam3.npz")
    g, fs = _field(G)
    cam = _cam(G)
    sc = window_scene(G)
    b = O.bin_and_sort(sc, cam)
    assert np.array_equal(b.starts, G["starts"]) and np.array_equal(b.items, G["items"])
    inv = sum(int((np.diff(G["mean_depth"][b.items[b.starts[t]:b.starts[t + 1]]]) < 0).sum()) for t in range(b.num_tiles))
    assert inv > 1000
    dm = O.RenderMaps(G["d_normal"], G["d_depth"], G["d_opacity"])
    for nw in G["windows"].tolist():
        maps, saved = O.render_forward(sc, b, cam, n_w=nw, save_state=True, backend=backend, want_counts=True)
        assert np.array_equal(saved.counts, G[f"counts_w{nw}"]), nw
        assert rel_err(maps.normal, G[f"normal_w{nw}"]) < 1e-12
        assert rel_err(maps.opacity, G[f"opacity_w{nw}"]) < 1e-12
        gb = O.render_backward(saved, sc, g, fs, cam, dm, backend=backend)
        assert rel_err(gb.d_sdf, G[f"d_sdf_w{nw}"]) < 1e-10
        assert rel_err(gb.d_deform, G[f"d_deform_w{nw}"]) < 1e-10
    assert np.abs(G["normal_w1"] - G["normal_w5"]).max() > 0.1
