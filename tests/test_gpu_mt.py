"""Marching Tetrahedra on the GPU against the reference fixtures (grid.py:136-239):
bit-exact vertex positions (welded, lexicographic) and triangle indices."""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ts():
    import paper_2406_01579_b200 as ts
    from paper_2406_01579_b200 import _native
    _native.lib()
    return ts


def _mt(ts, R, sdf, deform):
    g = ts.build_grid(R)
    fs = ts.FieldState.from_numpy(sdf, deform, ts.deform_limit_for(g))
    return ts.marching_tetrahedra(g, fs)


@pytest.mark.parametrize("tag", ["one_neg", "two_neg"])
def test_single_tet_examples(ts, tag):
    G = load_golden("mt.npz")
    sdf = G[f"{tag}_sdf"]
    m = _mt(ts, 1, sdf, np.zeros((len(sdf), 3)))
    assert np.array_equal(m.vertices, G[f"{tag}_V"])
    assert np.array_equal(m.triangles, G[f"{tag}_F"])


@pytest.mark.parametrize("tag,R", [("r16", 16), ("r16_noisy", 16), ("r24", 24)])
def test_grids_bitexact(ts, tag, R):
    G = load_golden("mt.npz")
    m = _mt(ts, R, G[f"{tag}_sdf"], G[f"{tag}_deform"])
    assert m.vertices.shape == G[f"{tag}_V"].shape
    assert np.array_equal(m.vertices, G[f"{tag}_V"])
    assert np.array_equal(m.triangles, G[f"{tag}_F"])


def test_sphere_watertight_and_empty(ts):
    g = ts.build_grid(32)
    f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.41,)))
    m = ts.marching_tetrahedra(g, f)
    assert m.euler_characteristic() == 2 and m.is_watertight()
    e = ts.FieldState.from_numpy(np.ones(g.num_vertices), np.zeros((g.num_vertices, 3)), ts.deform_limit_for(g))
    assert ts.marching_tetrahedra(g, e).is_empty


def test_two_phase_abi_matches_one_pass(ts):
    """ts_marching_tets_count + ts_marching_tets (caller-owned device outputs) == the one-pass
    run/fetch/release path behind marching_tetrahedra."""
    import ctypes
    import torch
    from paper_2406_01579_b200 import _native
    G = load_golden("mt.npz")
    R = 24
    g = ts.build_grid(R)
    fs = ts.FieldState.from_numpy(G["r24_sdf"], G["r24_deform"], ts.deform_limit_for(g))
    ref = ts.marching_tetrahedra(g, fs)
    L = _native.lib()
    nv, nt = _native.i64(), _native.i64()
    _native.check(L.ts_marching_tets_count(_native.ptr(fs.sdf), _native.ptr(fs.deformation), R, nv, nt, None))
    assert nv.value == ref.vertices.shape[0] and nt.value == ref.triangles.shape[0]
    V = torch.empty((nv.value, 3), dtype=torch.float64, device="cuda")
    F = torch.empty((nt.value, 3), dtype=torch.int64, device="cuda")
    counts = (ctypes.c_int64 * 2)()
    _native.check(L.ts_marching_tets(_native.ptr(fs.sdf), _native.ptr(fs.deformation), R, _native.ptr(V),
                                     _native.ptr(F), counts, None))
    assert counts[0] == nt.value and counts[1] == nv.value
    assert np.array_equal(V.cpu().numpy(), ref.vertices)
    assert np.array_equal(F.cpu().numpy(), ref.triangles)


@pytest.mark.parametrize("R", [20, 40])
def test_grids_match_oracle(ts, R):
    """R % 8 != 0 (per-cell corner bits) and R % 8 == 0 (z-fastest sign rows, eight cells per
    window) on a noisy, deformed field with exact zeros (f = 0 counts as outside; endpoint
    snaps), bit for bit against the oracle's restatement of grid.py:136-239."""
    from oracle import ts_oracle as O
    og = O.build_grid(R)
    of = O.noisy_field(og, noise=0.1, deform=0.4, seed=R)
    sdf = of.sdf.copy()
    sdf[::7] = 0.0
    V, F = O.marching_tetrahedra(og, O.FieldState(sdf, of.deformation, of.deform_limit))
    m = _mt(ts, R, sdf, of.deformation)
    assert len(F) > 0
    assert np.array_equal(m.vertices, V)
    assert np.array_equal(m.triangles, F)
