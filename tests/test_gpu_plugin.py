"""The kernel plugin contract (paper_2406_01579_b200.kernels): the reference's own
orchestration — raster.py's chunked thread pools and ordered merges, restated in
oracle/ts_oracle.py — calling forward_tiles / backward_tiles / reference_render /
eikonal_kernel / normal_consistency_kernel exactly as tetsplat does through
kernels.get_backend() (kernels/__init__.py:35-36), with this backend swapped in for the
reference's Cython `_core`.  Results are compared with the reference's own `_core` (oracle/_ref)
on the same fixtures: maps <= 1e-4, gradients <= 1e-3, regularizers <= 1e-9 / 1e-6, and the
materialised SavedState.records equal the reference's records."""
import numpy as np
import pytest

from conftest import RENDER_CASES, load_golden, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    from oracle import ts_oracle as O
    from paper_2406_01579_b200 import _native, kernels
    _native.lib()
    real = O._load_ref()
    if real is None:
        pytest.skip("oracle/_ref (the reference's compiled kernels) is not built")
    return O, kernels, real


def _swap(O, mod):
    O._REF = mod


def _case(O, G, colors=None):
    R, S, s = int(G["R"]), int(G["S"]), float(G["s"])
    og = O.build_grid(R)
    of = O.FieldState(G["sdf"], G["deform"], O.DEFORM_FRACTION * og.cell_edge)
    cam = O.orbit_camera(int(G["cam_index"]), int(G["cam_count"]), width=S, height=S)
    sc = O.build_scene(og, of, cam, s, active=G["active"], colors=colors)
    return og, of, cam, sc, O.bin_and_sort(sc, cam)


def _compare_records(ours, ref):
    """Per tile: counts equal except on a few T_STOP-crossing pixels; idx equal and alpha
    within FP32 rounding (|d alpha| < 5e-5) wherever the counts agree."""
    assert [int(r[0]) for r in ours] == [int(r[0]) for r in ref]
    bad, worst = 0, 0.0
    for (t, c, i, a), (t2, c2, i2, a2) in zip(ours, ref):
        assert c.dtype == np.int32 and c.shape == (256,) and i.dtype == np.int64 and a.dtype == np.float64
        o1 = np.concatenate([[0], np.cumsum(c)])
        o2 = np.concatenate([[0], np.cumsum(c2)])
        for p in range(256):
            if c[p] != c2[p]:
                bad += 1
                assert abs(int(c[p]) - int(c2[p])) <= 2
                continue
            assert np.array_equal(i[o1[p]:o1[p + 1]], i2[o2[p]:o2[p + 1]])
            if c[p]:
                worst = max(worst, float(np.abs(a[o1[p]:o1[p + 1]] - a2[o2[p]:o2[p + 1]]).max()))
    assert bad <= 8
    # FP32 opacity (error-banded decisions are exact; values carry FP32 rounding, amplified by s)
    assert worst < 5e-5, worst


def _run(O, mod, og, of, cam, sc, b, dm, n_w=5):
    _swap(O, mod)
    maps, saved = O.render_forward(sc, b, cam, n_w=n_w, save_state=True, backend="ref")
    gb = O.render_backward(saved, sc, og, of, cam, dm, backend="ref")
    ref = O.render_reference(sc, cam, backend="ref")
    return maps, saved, gb, ref


def _check(O, kernels, real, og, of, cam, sc, b, dm, n_w=5):
    try:
        m1, s1, g1, r1 = _run(O, kernels, og, of, cam, sc, b, dm, n_w)
        m2, s2, g2, r2 = _run(O, real, og, of, cam, sc, b, dm, n_w)
    finally:
        _swap(O, real)
    for k in ("normal", "depth", "opacity", "color"):
        a, r = getattr(m1, k), getattr(m2, k)
        if r is None:
            assert a is None
            continue
        assert rel_err(a, r) < 1e-4, k
        assert rel_err(getattr(r1, k), getattr(r2, k)) < 1e-4, ("reference_render", k)
    _compare_records(s1.records, s2.records)
    assert rel_err(g1.d_sdf, g2.d_sdf) < 1e-3
    assert rel_err(g1.d_deform, g2.d_deform) < 1e-3
    if g2.d_color is not None:
        assert rel_err(g1.d_color, g2.d_color) < 1e-3


@pytest.mark.parametrize("case", RENDER_CASES)
def test_plugin_render_cases(env, case):
    O, kernels, real = env
    G = load_golden(f"render_{case}.npz")
    og, of, cam, sc, b = _case(O, G)
    S = int(G["S"])
    _check(O, kernels, real, og, of, cam, sc, b, O.synthetic_dmaps(S, S))


def test_plugin_colour(env):
    O, kernels, real = env
    G = load_golden("color_noisy_r12_s100_cam5.npz")
    og, of, cam, sc, b = _case(O, G, colors=G["colors"])
    dm = O.RenderMaps(G["d_normal"], G["d_depth"], G["d_opacity"], G["d_color"])
    _check(O, kernels, real, og, of, cam, sc, b, dm)


@pytest.mark.parametrize("n_w", [1, 5, 712])
def test_plugin_reordering_window(env, n_w):
    O, kernels, real = env
    G = load_golden("window_noisy_r16_s100_cam3.npz")
    R, S = int(G["R"]), int(G["S"])
    og = O.build_grid(R)
    of = O.FieldState(G["sdf"], G["deform"], O.DEFORM_FRACTION * og.cell_edge)
    cam = O.orbit_camera(int(G["cam_index"]), int(G["cam_count"]), width=S, height=S)
    sc = O.SplatScene(G["tet_ids"], G["vert_ids"], G["proj"], G["depths"], G["f"], G["normals"],
                      G["mean_depth"], G["alpha_max"], G["bbox"], float(G["s"]), None)
    b = O.bin_and_sort(sc, cam)
    dm = O.RenderMaps(G["d_normal"], G["d_depth"], G["d_opacity"])
    _check(O, kernels, real, og, of, cam, sc, b, dm, n_w=n_w)


@pytest.mark.parametrize("case", [c for c in RENDER_CASES if "cfg1" not in c])
def test_plugin_regularizers(env, case):
    O, kernels, real = env
    G = load_golden(f"render_{case}.npz")
    og = O.build_grid(int(G["R"]))
    of = O.FieldState(G["sdf"], G["deform"], O.DEFORM_FRACTION * og.cell_edge)
    try:
        _swap(O, kernels)
        le, ge = O.eikonal_loss(og, of, G["active"], backend="ref")
        ln, gn = O.normal_consistency_loss(og, of, backend="ref")
    finally:
        _swap(O, real)
    assert abs(le - float(G["eik_loss"])) <= 1e-9 * max(1.0, abs(float(G["eik_loss"])))
    assert abs(ln - float(G["nc_loss"])) <= 1e-9 * max(1.0, abs(float(G["nc_loss"])))
    assert rel_err(ge.d_sdf, G["eik_d_sdf"]) < 1e-6 and rel_err(ge.d_deform, G["eik_d_deform"]) < 1e-6
    assert rel_err(gn.d_sdf, G["nc_d_sdf"]) < 1e-6 and rel_err(gn.d_deform, G["nc_d_deform"]) < 1e-6


def test_plugin_argument_errors(env):
    """Cython's buffer acquisition raises ValueError on dtype / contiguity mismatches
    (SURVEY §8b); so do the B200 kernels, and on contract values they do not implement."""
    O, kernels, real = env
    G = load_golden("render_sphere_r16_s100.npz")
    og, of, cam, sc, b = _case(O, G)
    S = int(G["S"])
    maps = O.RenderMaps.zeros(S, S)
    args = [sc.proj, sc.depths, sc.f, sc.normals, sc.mean_depth, None, sc.bbox, b.starts, b.items,
            np.nonzero(np.diff(b.starts))[0], 16, b.tiles_x, S, S, 5, 100.0, 1e-4, 1 - 1e-4, maps.normal, maps.depth,
            maps.opacity, None, False]
    bad = list(args)
    bad[0] = sc.proj.astype(np.float32)
    with pytest.raises(ValueError):
        kernels.forward_tiles(*bad)
    bad = list(args)
    bad[7] = b.starts.astype(np.int32)
    with pytest.raises(ValueError):
        kernels.forward_tiles(*bad)
    bad = list(args)
    bad[10] = 8
    with pytest.raises(ValueError):
        kernels.forward_tiles(*bad)
    assert kernels.forward_tiles(*args) == []
    with pytest.raises(ValueError):  # records of another backend
        kernels.backward_tiles(sc.proj, sc.depths, sc.f, sc.normals, sc.mean_depth, None, sc.bbox,
                               [(0, np.zeros(256, np.int32), np.zeros(0, np.int64), np.zeros(0))], 16, b.tiles_x, S,
                               S, 100.0, 1 - 1e-4, maps.normal, maps.depth, maps.opacity, None,
                               np.zeros((len(sc), 4)), np.zeros((len(sc), 4, 2)), np.zeros((len(sc), 4)),
                               np.zeros((len(sc), 3)), np.zeros(len(sc)), None)
    assert kernels.get_backend() is kernels and kernels.get_backend_by_name("b200") is kernels
