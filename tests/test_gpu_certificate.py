"""The never-blend certificate (records.cuh `never_blends`): splats whose SDF
increases along every camera ray through them get an empty pixel rectangle, so the
compositing kernels never evaluate their pairs.  The claim is that such a splat blends in
NO pixel of the reference (_core.pyx:189-196: alpha = 1 - exp(sp(x) - sp(y)) <= 0), for any
steepness and whatever the early stop.

Checked against the reference's own kernels with early stop disabled (t_stop = 0, every list
entry of every pixel evaluated): the certified set and the set of splats that blend anywhere
are disjoint, the certificate covers a large share of the splats (so the test has teeth), and
the rendered maps / per-pixel blend counts still match the reference at the usual bars.
"""
import numpy as np
import pytest
import torch

from conftest import rel_err

pytestmark = pytest.mark.gpu

CERT_BIT = 32  # SplatRec.flags bit 5


@pytest.fixture(scope="module")
def ts():
    import paper_2406_01579_b200 as ts
    from paper_2406_01579_b200 import _native
    _native.lib()
    return ts


def _certified(scene):
    rec = scene.records.cpu().numpy()
    flags = rec[:, 12:16].copy().view(np.uint32)[:, 0]
    rx = rec[:, 0:4].copy().view(np.int32)[:, 0]
    x0 = (rx & 0xFFFF).astype(np.int16).astype(np.int32)
    x1 = rx >> 16
    cert = (flags & CERT_BIT) != 0
    assert np.all(x1[cert] < x0[cert]), "a certified splat kept a non-empty rectangle"
    return cert


CASES = [  # (R, S, steepness, field, camera index, noise, deform)
    (32, 256, 100.0, "sphere", 0, 0.0, 0.0),
    (24, 192, 20.0, "noisy", 3, 0.08, 0.4),
    (24, 160, 1000.0, "noisy", 5, 0.05, 0.3),
    (16, 128, 5.0, "noisy", 1, 0.15, 0.4),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"R{c[0]}_S{c[1]}_s{c[2]:g}_{c[3]}_cam{c[4]}")
def test_certified_splats_never_blend(ts, case):
    from oracle import ts_oracle as O
    if "ref" not in O.available_backends():
        pytest.skip("the reference's compiled kernels (oracle/_ref) are not built")
    R, S, s, kind, ci, noise, deform = case
    og = O.build_grid(R)
    of = O.init_sphere_field(og) if kind == "sphere" else O.noisy_field(og, noise=noise, deform=deform, seed=7)
    ocam = O.orbit_camera(ci, 8, width=S, height=S)
    osc = O.build_scene(og, of, ocam, s)
    ob = O.bin_and_sort(osc, ocam)

    g = ts.build_grid(R)
    f = ts.FieldState.from_numpy(of.sdf, of.deformation, of.deform_limit)
    cam = ts.orbit_camera(ci, 8, width=S, height=S)
    sc = ts.build_scene(g, f, cam, s)
    assert np.array_equal(sc.tet_ids.cpu().numpy(), osc.tet_ids)
    cert = _certified(sc)
    assert cert.mean() > 0.25, f"certificate covers only {cert.mean():.3f} of the splats"

    # every list entry of every pixel evaluated: which splats blend anywhere in the reference
    _, sv = O.render_forward(osc, ob, ocam, t_stop=0.0, save_state=True, backend="ref")
    blended = np.zeros(len(osc), bool)
    for _tid, _cnt, idx, _al in sv.records:
        if len(idx):
            blended[np.asarray(idx, dtype=np.int64)] = True
    both = np.nonzero(cert & blended)[0]
    assert both.size == 0, f"{both.size} certified splats blend in the reference: {both[:10]}"

    # and the product path still matches the reference (with the normal early stop)
    om, osv = O.render_forward(osc, ob, ocam, want_counts=True, backend="ref")
    b = ts.bin_and_sort(sc, cam)
    maps, saved = ts.render_forward(sc, b, cam, save_state=True)
    torch.cuda.synchronize()
    n, d, o, _ = maps.numpy()
    assert max(rel_err(n, om.normal), rel_err(d, om.depth), rel_err(o, om.opacity)) < 1e-4
    counts = saved.n_blend.cpu().numpy().reshape(S, S)
    bad = np.argwhere(counts != osv.counts)
    for y, x in bad:  # only where FP32 transmittance crosses T_STOP on an opaque pixel
        assert om.opacity[y, x] >= 1.0 - 2e-4, (y, x, counts[y, x], osv.counts[y, x])
    assert len(bad) <= max(4, counts.size // 2000)
