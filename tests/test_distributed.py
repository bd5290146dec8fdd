"""View-sharded multi-process path on CPU (gloo, world size 2): view partition, the one
gradient all-reduce of the batch (batch.allreduce_gradients) and the replicated Adam step.
Per-view gradients come from the CPU oracle here (no GPU in this container); the sum over
ranks must equal the single-process batch gradient."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_01579_b200.batch import Adam, allreduce_gradients, shard_views
from paper_2406_01579_b200.raster import GradientBuffers

R, S, S_STEEP, NV = 8, 48, 60.0, 5


def _view_grads(view):
    from oracle import ts_oracle as O
    g = O.build_grid(R)
    f = O.noisy_field(g, noise=0.04, deform=0.2, seed=11)
    cam = O.orbit_camera(view, NV, width=S, height=S)
    sc = O.build_scene(g, f, cam, S_STEEP)
    b = O.bin_and_sort(sc, cam)
    m, sv = O.render_forward(sc, b, cam, save_state=True, backend=O.default_backend())
    gr = O.render_backward(sv, sc, g, f, cam, O.synthetic_dmaps(S, S, seed=view), backend=O.default_backend())
    d = np.zeros((g.num_vertices, 4), dtype=np.float32)
    d[:, 0] = gr.d_sdf
    d[:, 1:] = gr.d_deform
    return d


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    views = shard_views(NV, rank, world)
    gb = GradientBuffers(torch.zeros(((R + 1) ** 3, 4), dtype=torch.float32))
    for v in views:
        gb.d_vert += torch.from_numpy(_view_grads(v))
    allreduce_gradients(gb)
    p = [torch.zeros((R + 1) ** 3, dtype=torch.float64), torch.zeros(((R + 1) ** 3, 3), dtype=torch.float64)]
    opt = Adam(p, [1e-2, 1e-3])
    opt.step(p, [gb.d_sdf, gb.d_deform])
    out[rank] = (gb.d_vert.numpy().copy(), p[0].numpy().copy(), views)
    dist.destroy_process_group()


def test_shard_views_partition():
    for n in (1, 5, 8, 64):
        for w in (1, 2, 3, 4, 8):
            parts = [shard_views(n, r, w) for r in range(w)]
            assert sorted(sum(parts, [])) == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


@pytest.mark.timeout(600)
def test_gloo_allreduce_matches_single_process():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    ref = sum(_view_grads(v) for v in range(NV))
    for r in range(world):
        d, sdf_after, views = out[r]
        assert np.allclose(d, ref, rtol=1e-5, atol=1e-5 * np.abs(ref).max())
    # every rank applies the identical optimizer update
    assert np.array_equal(out[0][1], out[1][1])
    assert sorted(out[0][2] + out[1][2]) == list(range(NV))


def test_default_inflight_respects_host_cpus(monkeypatch):
    import os
    from paper_2406_01579_b200 import batch
    monkeypatch.setattr(os, "sched_getaffinity", lambda pid: set(range(16)))
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "1")
    assert batch.default_inflight() == 4
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "8")
    assert batch.default_inflight() == 2  # never below two lanes (8 ranks on a 16-core host)
    monkeypatch.setattr(os, "sched_getaffinity", lambda pid: set(range(64)))
    assert batch.default_inflight() == 4
