"""Deterministic (fixed-point) gradient mode: the reference merges per-chunk private buffers in
a fixed order (raster.py:217-247), so its gradients are bitwise reproducible; the FP32 atomics
of the default path are not.  With raster.FixedPointGradients / StepConfig(deterministic=True)
every contribution is an int64 round(v * 2^36) added by integer atomics:

* repeated runs give bitwise-identical gradients (fine-grained API, fused view path, colour
  gradients, the regularizers and the whole FitStep with four lanes in flight);
* the result equals the reference (same fixtures and bars as the FP32 path) and the FP32 path
  to rounding level;
* two ranks (gloo, all-reducing the int64 buffer) give exactly the single-process gradients
  and Adam update.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_golden, rel_err

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-3
R, S, V, STEEP = 32, 256, 4, 100.0


@pytest.fixture(scope="module")
def ts():
    import paper_2406_01579_b200 as ts
    from paper_2406_01579_b200 import _native
    _native.lib()
    return ts


def _setup(ts, G):
    g = ts.build_grid(int(G["R"]))
    fs = ts.FieldState.from_numpy(G["sdf"], G["deform"], ts.deform_limit_for(g))
    S_ = int(G["S"])
    cam = ts.orbit_camera(int(G["cam_index"]), int(G["cam_count"]), width=S_, height=S_)
    return g, fs, cam


def test_fine_grained_api_color_reproducible_and_matches_reference(ts):
    G = load_golden("color_noisy_r12_s100_cam5.npz")
    g, fs, cam = _setup(ts, G)
    s = float(G["s"])
    sc = ts.build_scene(g, fs, cam, s, active=torch.as_tensor(G["active"]).cuda(), colors=G["colors"])
    b = ts.bin_and_sort(sc, cam)
    maps, saved = ts.render_forward(sc, b, cam, save_state=True)
    dm = ts.RenderMaps(G["d_normal"], G["d_depth"], G["d_opacity"], G["d_color"])
    runs = [ts.render_backward(saved, sc, g, fs, cam, dm, deterministic=True) for _ in range(3)]
    for r in runs[1:]:
        assert torch.equal(r.d_vert, runs[0].d_vert) and torch.equal(r.d_color, runs[0].d_color)
    gb = runs[0]
    assert rel_err(gb.d_color.cpu().numpy(), G["d_color_tet"]) < GRAD_TOL
    assert rel_err(gb.d_sdf.cpu().numpy(), G["d_sdf"]) < GRAD_TOL
    assert rel_err(gb.d_deform.cpu().numpy(), G["d_deform"]) < GRAD_TOL
    # the FP32-atomic path agrees to rounding level
    fp = ts.render_backward(saved, sc, g, fs, cam, dm)
    den = float(fp.d_vert.abs().max())
    assert float((fp.d_vert - gb.d_vert).abs().max()) <= 1e-5 * den
    assert float((fp.d_color - gb.d_color).abs().max()) <= 1e-5 * float(fp.d_color.abs().max())
    # accumulating into a caller's FixedPointGradients: two backward passes add exactly
    acc = ts.FixedPointGradients.zeros(g.num_vertices, "cuda", num_tets_color=g.num_tets)
    ts.render_backward(saved, sc, g, fs, cam, dm, out=acc)
    one = acc.fx.clone()
    ts.render_backward(saved, sc, g, fs, cam, dm, out=acc)
    assert torch.equal(acc.fx[:-1], 2 * one[:-1]) and int(acc.dropped) == 0


def test_fused_view_path_reproducible(ts):
    from paper_2406_01579_b200.view import ViewRenderer
    G = load_golden("color_noisy_r12_s100_cam5.npz")
    g, fs, cam = _setup(ts, G)
    s = float(G["s"])
    active = ts.prefilter(g, fs, s)
    colors = torch.as_tensor(G["colors"], dtype=torch.float32, device="cuda")
    f32 = lambda k: torch.as_tensor(G[k], dtype=torch.float32, device="cuda")
    dm = ts.RenderMaps(f32("d_normal"), f32("d_depth"), f32("d_opacity"), f32("d_color"))
    outs = []
    for _ in range(2):
        vr = ViewRenderer()
        vr.forward(g, fs, cam, s, active, colors=colors)
        acc = ts.FixedPointGradients.zeros(g.num_vertices, "cuda", num_tets_color=g.num_tets)
        vr.backward(fs, dm, acc)
        outs.append(acc.to_float())
    assert torch.equal(outs[0].d_vert, outs[1].d_vert) and torch.equal(outs[0].d_color, outs[1].d_color)
    assert rel_err(outs[0].d_color.cpu().numpy(), G["d_color_tet"]) < GRAD_TOL
    assert rel_err(outs[0].d_sdf.cpu().numpy(), G["d_sdf"]) < GRAD_TOL
    assert rel_err(outs[0].d_deform.cpu().numpy(), G["d_deform"]) < GRAD_TOL


def test_regularizers_fixed_point(ts):
    from paper_2406_01579_b200.losses import eikonal_loss_async, normal_consistency_loss_async
    from oracle import ts_oracle as O
    og = O.build_grid(24)
    of = O.noisy_field(og, noise=0.08, deform=0.4, seed=3)
    g = ts.build_grid(24)
    f = ts.FieldState.from_numpy(of.sdf, of.deformation, ts.deform_limit_for(g))
    tets = torch.arange(g.num_tets, dtype=torch.int32, device="cuda")
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    res = []
    for fixed in (True, True, False):
        out = ts.FixedPointGradients.zeros(g.num_vertices) if fixed else ts.GradientBuffers.zeros(g.num_vertices)
        eikonal_loss_async(g, f, tets, out, 1000.0, loss)
        normal_consistency_loss_async(g, f, out, 1000.0, loss)
        res.append(out.to_float() if fixed else out)
    assert torch.equal(res[0].d_vert, res[1].d_vert)
    den = float(res[2].d_vert.abs().max())
    assert float((res[0].d_vert - res[2].d_vert).abs().max()) <= 1e-5 * den


def test_dropped_contributions_flag_the_step(ts):
    """Non-finite map gradients on the deterministic path: counted as dropped, surfaced in
    status[1] by the conversion (Adam skips) besides the status[0] map check."""
    from paper_2406_01579_b200.view import ViewRenderer
    G = load_golden("color_noisy_r12_s100_cam5.npz")
    g, fs, cam = _setup(ts, G)
    s = float(G["s"])
    active = ts.prefilter(g, fs, s)
    vr = ViewRenderer()
    vr.forward(g, fs, cam, s, active)
    f32 = lambda k: torch.as_tensor(G[k], dtype=torch.float32, device="cuda")
    dm = ts.RenderMaps(f32("d_normal"), f32("d_depth"), f32("d_opacity"))
    dm.depth[:] = float("nan")
    status = torch.zeros(4, device="cuda")
    acc = ts.FixedPointGradients.zeros(g.num_vertices)
    vr.backward(fs, dm, acc, status=status)
    acc.to_float(status=status)
    torch.cuda.synchronize()
    assert float(status[0]) > 0 and int(acc.dropped) > 0 and float(status[1]) == float(acc.dropped)


def _problem():
    import paper_2406_01579_b200 as ts
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
    return ts, g, f, cams, dms


def _run_step(views, deterministic=True, sync_free=None, inflight=None):
    from paper_2406_01579_b200.batch import FitStep, StepConfig
    ts, g, f, cams, dms = _problem()
    step = FitStep(g, f, cams, StepConfig(deterministic=deterministic, sync_free=sync_free, inflight=inflight))
    grads = step(STEEP, views, lambda vi, m: dms[vi])
    torch.cuda.synchronize()
    step.check_status()
    return grads.d_vert.cpu().numpy().copy(), f.sdf.cpu().numpy().copy(), f.deformation.cpu().numpy().copy()


def test_fitstep_bitwise_reproducible():
    a = _run_step(list(range(V)), inflight=4)
    b = _run_step(list(range(V)), inflight=2)
    c = _run_step(list(range(V)), sync_free=True, inflight=3)
    for x in (b, c):
        for u, v in zip(a, x):
            assert np.array_equal(u, v)
    # agrees with the FP32-atomic step to rounding level
    g_fp = _run_step(list(range(V)), deterministic=False)[0]
    assert np.abs(g_fp - a[0]).max() <= 1e-5 * np.abs(g_fp).max()


def _free_port():
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def _worker(rank, world, port, out):
    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_01579_b200.batch import shard_views
    out[rank] = _run_step(shard_views(V, rank, world))
    dist.destroy_process_group()


@pytest.mark.timeout(900)
def test_two_ranks_bitwise_equal_single_process():
    """The exact form of test_gpu_distributed: with int64 all-reduce the sharded step's
    gradients and Adam update equal the single-process ones bit for bit."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    ref = _run_step(list(range(V)))
    for r in range(world):
        for u, v in zip(out[r], ref):
            assert np.array_equal(u, v), r
