"""Long-list split of the fused view path (composite.cu "Long-list split"): the longest tile
lists are composited by two CTAs — forward as a 2-CTA cluster that hands the per-pixel state
over at the half, backward as two CTAs the second of which starts from that state.  The split
must not change any result: maps and per-pixel blend counts bit-identical to one CTA per tile,
gradients equal to rounding (the second half's chunks start at h, so the per-run FP32 sums
that the fixed-point rows round are grouped differently).
Splitting EVERY tile (min_len 0) also covers lists that stop in the first half, empty halves
and one-entry lists; a capped split (max_tiles 3) mixes split and whole tiles in one launch."""
import numpy as np
import pytest
import torch

from conftest import load_golden, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ts():
    import paper_2406_01579_b200 as ts
    from paper_2406_01579_b200 import _native
    _native.lib()
    yield ts
    _native.check(_native.lib().ts_debug_set_split(-1, -1))


def _set_split(max_tiles, min_len):
    from paper_2406_01579_b200 import _native
    _native.check(_native.lib().ts_debug_set_split(max_tiles, min_len))


def _noisy(ts, R, S, V, seed, noise=0.08, deform=0.4):
    from oracle import ts_oracle as O
    og = O.build_grid(R)
    of = O.noisy_field(og, noise=noise, deform=deform, seed=seed)
    g = ts.build_grid(R)
    f = ts.FieldState.from_numpy(of.sdf, of.deformation, ts.deform_limit_for(g))
    cams = [ts.orbit_camera(i, V, width=S, height=S) for i in range(V)]
    return g, f, cams


def _dmaps(ts, S, seed, color=False):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    r = lambda *sh: torch.randn(sh, device="cuda", generator=gen)
    return ts.RenderMaps(r(S, S, 3), r(S, S), r(S, S), r(S, S, 3) if color else None)


def _run(ts, g, f, cam, s, active, dm, colors=None, n_w=None, caps=False):
    """maps, n_blend, fixed-point gradients, FP32 gradients of one fused view"""
    from paper_2406_01579_b200.view import ViewRenderer
    vr = ViewRenderer()
    kw = {} if n_w is None else {"n_w": n_w}
    if caps:  # the sync-free path: capacities from a sizing pass, device-side counts
        vr.forward(g, f, cam, s, active, colors=colors, **kw)
        K, M, P = vr.counts
        vr.set_caps(int(M * 1.2) + 64, int(P * 1.2) + 64, int(vr.max_list) + 64)
    maps = vr.forward(g, f, cam, s, active, colors=colors, **kw)
    out = tuple(torch.clone(t) for t in (maps.normal, maps.depth, maps.opacity)) + \
        ((torch.clone(maps.color),) if colors is not None else ())
    nb = vr.n_blend()
    fx = ts.FixedPointGradients.zeros(g.num_vertices, "cuda", num_tets_color=g.num_tets if colors is not None else None)
    vr.backward(f, dm, fx)
    gfx = fx.to_float()
    fp = ts.GradientBuffers.zeros(g.num_vertices, "cuda", num_tets_color=g.num_tets if colors is not None else None)
    vr.backward(f, dm, fp)
    torch.cuda.synchronize()
    return out, nb, gfx, fp


def _same(a, b):
    ma, na, ga, fa = a
    mb, nb, gb, fb = b
    for x, y in zip(ma, mb):
        assert torch.equal(x, y), "maps differ"
    assert torch.equal(na, nb), "n_blend differs"
    den = float(ga.d_vert.abs().max())
    assert den > 0
    assert float((ga.d_vert - gb.d_vert).abs().max()) <= 1e-5 * den
    if ga.d_color is not None:
        assert float((ga.d_color - gb.d_color).abs().max()) <= 1e-5 * float(ga.d_color.abs().max())
    den = float(fa.d_vert.abs().max())
    assert den > 0
    assert float((fa.d_vert - fb.d_vert).abs().max()) <= 1e-5 * den


@pytest.mark.parametrize("max_tiles,min_len", [(1 << 20, 0), (3, 0), (1 << 20, 64)])
def test_split_equals_whole_tiles_noisy(ts, max_tiles, min_len):
    g, f, cams = _noisy(ts, 32, 256, 4, seed=5)
    s = 100.0
    act = ts.prefilter(g, f, s)
    for i in (0, 2):
        dm = _dmaps(ts, 256, 10 + i)
        _set_split(0, 0)
        whole = _run(ts, g, f, cams[i], s, act, dm)
        _set_split(max_tiles, min_len)
        split = _run(ts, g, f, cams[i], s, act, dm)
        _same(whole, split)


def test_split_equals_whole_tiles_soft_long_lists(ts):
    """s = 20: wide, soft splats — long lists whose pixels never reach T_STOP"""
    g, f, cams = _noisy(ts, 48, 384, 2, seed=7, noise=0.05, deform=0.3)
    s = 20.0
    act = ts.prefilter(g, f, s)
    dm = _dmaps(ts, 384, 3)
    _set_split(0, 0)
    whole = _run(ts, g, f, cams[1], s, act, dm)
    _set_split(1 << 20, 256)
    split = _run(ts, g, f, cams[1], s, act, dm)
    _same(whole, split)
    _set_split(1 << 20, 0)
    _same(whole, _run(ts, g, f, cams[1], s, act, dm, caps=True))


def test_split_colour_and_window(ts):
    """colours (fixture of the reference) and a reordering window fixture, every tile split;
    the colour fixture is also checked against the reference's maps / gradients"""
    G = load_golden("color_noisy_r12_s100_cam5.npz")
    g = ts.build_grid(int(G["R"]))
    f = ts.FieldState.from_numpy(G["sdf"], G["deform"], ts.deform_limit_for(g))
    S = int(G["S"])
    cam = ts.orbit_camera(int(G["cam_index"]), int(G["cam_count"]), width=S, height=S)
    s = float(G["s"])
    act = ts.prefilter(g, f, s)
    colors = torch.as_tensor(G["colors"], dtype=torch.float32, device="cuda")
    f32 = lambda k: torch.as_tensor(G[k], dtype=torch.float32, device="cuda")
    dm = ts.RenderMaps(f32("d_normal"), f32("d_depth"), f32("d_opacity"), f32("d_color"))
    _set_split(0, 0)
    whole = _run(ts, g, f, cam, s, act, dm, colors=colors)
    _set_split(1 << 20, 0)
    split = _run(ts, g, f, cam, s, act, dm, colors=colors)
    _same(whole, split)
    m = split[0]
    assert rel_err(m[3].cpu().numpy(), G["color"]) < 1e-4
    assert rel_err(split[3].d_color.cpu().numpy(), G["d_color_tet"]) < 1e-3
    assert rel_err(split[3].d_sdf.cpu().numpy(), G["d_sdf"]) < 1e-3

    W = load_golden("window_noisy_r16_s100_cam3.npz")
    g = ts.build_grid(int(W["R"]))
    f = ts.FieldState.from_numpy(W["sdf"], W["deform"], ts.deform_limit_for(g))
    S = int(W["S"])
    cam = ts.orbit_camera(int(W["cam_index"]), int(W["cam_count"]), width=S, height=S)
    s = float(W["s"])
    act = ts.prefilter(g, f, s)
    dm = _dmaps(ts, S, 4)
    for n_w in (1, 5):
        _set_split(0, 0)
        whole = _run(ts, g, f, cam, s, act, dm, n_w=n_w)
        _set_split(1 << 20, 0)
        _same(whole, _run(ts, g, f, cam, s, act, dm, n_w=n_w))
