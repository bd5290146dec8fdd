"""Multi-view fit step on the device, view-sharded across GPUs (fit.py:145-231 hot path).

One iteration = prefilter (K1) once, then per view: build_scene (K2) -> bin_and_sort
(K3-K5) -> render_forward (K6) -> render_backward (K7) accumulating into one FP32 [N,4]
gradient buffer; eikonal + normal consistency (K8) fused into the same buffer with their
lambda weights; then one NCCL all-reduce of that buffer across ranks (views are
partitioned, parameters replicated — SURVEY.md §8e) and an identical Adam step on every
rank (fit.py:70-90), followed by the deformation clamp (field.py:40-42).
"""
from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field as dc_field

import torch
import torch.distributed as dist

from .losses import eikonal_loss_async, nc_scratch_bytes, normal_consistency_loss_async
from .raster import FixedPointGradients, GradientBuffers
from .splat import EmptySceneError, prefilter
from .view import ViewRenderer


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """Contiguous partition of view indices over ranks (the first n % world ranks take one
    extra view); the union over ranks is range(n_views) exactly once."""
    base, extra = divmod(n_views, world)
    lo = rank * base + min(rank, extra)
    return list(range(lo, lo + base + (1 if rank < extra else 0)))


def allreduce_gradients(grads: GradientBuffers, group=None) -> None:
    """Sum the per-rank vertex gradients (the only data-path collective)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grads.d_vert, op=dist.ReduceOp.SUM, group=group)
        if grads.d_color is not None:
            dist.all_reduce(grads.d_color, op=dist.ReduceOp.SUM, group=group)


def host_cpus_per_rank() -> int:
    import os
    try:
        cpus = len(os.sched_getaffinity(0))
    except AttributeError:
        cpus = os.cpu_count() or 1
    return cpus // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))


def default_inflight() -> int:
    """Four views in flight (measured best at config 3: 2 / 3 / 4 / 8 lanes = 486 / 492 / 502 /
    502 views/s), fewer when the ranks of this node share few host CPUs (each lane has a host
    thread that waits on its stream)."""
    import os
    try:
        cpus = len(os.sched_getaffinity(0))
    except AttributeError:
        cpus = os.cpu_count() or 1
    per_rank = cpus // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
    # at least two lanes even when 8 ranks share 16 host CPUs: a lane's host thread spends
    # its time blocked on its stream's sizing syncs, so two fit on one core (1 -> 2 lanes
    # was +24% on one GPU)
    return max(2, min(4, per_rank - 1))


class Adam:
    """fit.py:70-90 on the device (FP64 moments, like the reference)."""

    def __init__(self, params, lrs, betas=(0.9, 0.99), eps=1e-8):
        self.lrs = list(lrs)
        self.b1, self.b2 = betas
        self.eps = eps
        self.t = 0
        self.m = [torch.zeros_like(p) for p in params]
        self.v = [torch.zeros_like(p) for p in params]

    @torch.no_grad()
    def step(self, params, grads):
        self.t += 1
        c1 = 1 - self.b1 ** self.t
        c2 = 1 - self.b2 ** self.t
        for p, g, m, v, lr in zip(params, grads, self.m, self.v, self.lrs):
            g = g.to(p.dtype)
            m.mul_(self.b1).add_(g, alpha=1 - self.b1)
            v.mul_(self.b2).addcmul_(g, g, value=1 - self.b2)
            p.addcdiv_(m / c1, (v / c2).sqrt_().add_(self.eps), value=-lr)

    @torch.no_grad()
    def step_field(self, field, grads: GradientBuffers, resolution: int, stream=None, status=None):
        """The same update for (sdf, deformation) in one fused kernel straight from the
        interleaved gradient buffer, deformation clamped to its limit (ts_adam_step).
        With `status` (device f32[2+], see FitStep) the update is skipped on the device when
        a map gradient or a gradient entry is non-finite."""
        from . import _native
        self.t += 1
        _native.check(_native.lib().ts_adam_step(
            int(resolution), _native.ptr(grads.d_vert), _native.ptr(field.sdf), _native.ptr(field.deformation),
            _native.ptr(self.m[0]), _native.ptr(self.v[0]), _native.ptr(self.m[1]), _native.ptr(self.v[1]),
            float(self.lrs[0]), float(self.lrs[1]), float(self.b1), float(self.b2), int(self.t), float(self.eps),
            float(field.deform_limit), _native.ptr(status), _native.stream_ptr(stream)))


@dataclass
class StepConfig:
    n_w: int = 5
    lambda_eik: float = 1000.0
    lambda_nc: float = 1000.0
    lr_sdf: float = 1e-2
    lr_deform: float = 1e-3
    betas: tuple = (0.9, 0.99)
    optimizer: bool = True
    inflight: int | None = None  # views in flight (renderer + workspace + stream + host thread
    #                              each); None = 4, fewer when the rank has < 5 host CPUs
    eik_all: bool = False  # eikonal over every tet (fit.py eikonal_scope="all") instead of the active set
    # one host thread, no per-view host round trip: each camera's first view sizes its buffers
    # (the sizing syncs), later views run with capacities from the largest sizes seen (x1.15);
    # an overflowing view is detected at the end of the step (one read) and the step re-run.
    # None = auto: sync-free when the rank has fewer than 6 host CPUs (8 ranks on a 16-48
    # core host), else one host thread per lane (measured 1.8% faster on one B200 with 16 CPUs)
    sync_free: bool | None = None
    # bitwise-reproducible gradients: every contribution (views, regularizers) is accumulated
    # as a 64-bit fixed-point integer (raster.FixedPointGradients) and the all-reduce sums
    # int64, so the step's gradients — and Adam's update — do not depend on atomic order,
    # lane scheduling or the number of ranks the views are split over
    deterministic: bool = False
    # the per-batch regularizers split over the ranks (eikonal tets / normal-consistency vertex
    # slabs) instead of all on rank 0
    shard_regularizers: bool = True


@dataclass
class StepStats:
    views: int = 0
    splats: list = dc_field(default_factory=list)
    pairs: list = dc_field(default_factory=list)
    active: int = 0


class FitStep:
    """Runs fwd+bwd for this rank's views; `d_maps_fn(view_index, maps)` returns dL/dmaps."""

    def __init__(self, grid, field, cameras, cfg: StepConfig | None = None, group=None):
        self.grid, self.field, self.cameras = grid, field, cameras
        self.cfg = cfg or StepConfig()
        self.group = group
        dev = field.sdf.device
        # one flat FP32 buffer: the [N,4] vertex gradients plus a 4-float status tail
        # ([0] non-finite map gradients, [1] non-finite gradient entries), so the single
        # all-reduce carries the failure flags too and every rank skips the same update
        N = grid.num_vertices
        self._flat = torch.zeros(4 * N + 4, dtype=torch.float32, device=dev)  # status: [2] overflowed views
        self.grads = GradientBuffers(self._flat[:4 * N].view(N, 4))
        self.status = self._flat[4 * N:]
        self._fx = FixedPointGradients.zeros(N, dev) if self.cfg.deterministic else None
        self._acc = self._fx if self._fx is not None else self.grads  # what the kernels add into
        self.eik_loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.nc_loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.opt = Adam([field.sdf, field.deformation], [self.cfg.lr_sdf, self.cfg.lr_deform], self.cfg.betas) \
            if self.cfg.optimizer else None
        # two views in flight: each renderer owns a workspace and a stream, so one view's
        # kernels run while the host waits on the other's sizing syncs (and kernel tails overlap)
        n = self.cfg.inflight if self.cfg.inflight is not None else default_inflight()
        n = max(1, int(n))
        self.renderers = [ViewRenderer(dev) for _ in range(n)]
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(n)]
        self.view = self.renderers[0]
        self.reg_stream = torch.cuda.Stream(device=dev)
        self._all_tets = None
        self._nc_scratch = None  # normal-consistency scratch, allocated once
        self.last_active = 0
        if self.cfg.sync_free is None:
            self.cfg.sync_free = host_cpus_per_rank() < 6
        self._pool = ThreadPoolExecutor(max_workers=n) if n > 1 and not self.cfg.sync_free else None
        self._sizes = {}   # camera index -> largest (M, P, longest list) seen (sync-free capacities)
        self._needs = None  # device int64[views, 5]: per view {K, M, P, longest list, overflow}
        self._retry = 0
        self.view_counts = {}  # view -> (K, M, P) of the last step

    def __call__(self, s: float, views, d_maps_fn, stats: StepStats | None = None, inputs_ready=None,
                 update: bool | None = None):
        """`inputs_ready`: optional CUDA event after which the deformation is valid (the SDF
        must be valid on the current stream); everything but the prefilter waits for it.
        `update`: run the Adam step at the end (default: when the config has an optimizer);
        `fit_field` passes False and calls `apply_update` after its host-side checks."""
        with torch.cuda.nvtx.range("FitStep"):  # (the ABI calls open their own ranges inside)
            return self._step(s, views, d_maps_fn, stats, inputs_ready, update)

    def _step(self, s, views, d_maps_fn, stats, inputs_ready, update):
        g, f, cfg = self.grid, self.field, self.cfg
        self._flat.zero_()
        if self._fx is not None:
            self._fx.zero_()
        active = prefilter(g, f, s)
        if active.numel() == 0:
            raise EmptySceneError("pre-filtering removed every tetrahedron")
        self.last_active = int(active.numel())
        if stats is not None:
            stats.active = self.last_active
        main = torch.cuda.current_stream()
        for st in self.streams + [self.reg_stream]:
            st.wait_stream(main)  # zeroed gradients, prefilter output
            if inputs_ready is not None:
                st.wait_event(inputs_ready)
            active.record_stream(st)
        # regularizers once per batch, sharded over the ranks (their gradient rides in the
        # all-reduce): rank r takes the r-th slice of the eikonal's tets and the r-th z-slab of
        # the normal-consistency vertices (SURVEY 8e "sharded by tet range"), so no rank carries
        # the whole per-batch term; eik_loss / nc_loss hold this rank's partial sums (fit_field
        # all-reduces them with the map losses).  They depend only on the field, so they run on
        # their own stream beside the views (every gradient kernel accumulates atomically).
        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1
        rank, world = (dist.get_rank(self.group), dist.get_world_size(self.group)) if multi else (0, 1)
        if not cfg.shard_regularizers and rank != 0:
            rank, world = -1, 1  # rank-0-only mode: nothing here
        if rank >= 0:
            with torch.cuda.stream(self.reg_stream):
                if cfg.lambda_eik > 0:
                    if cfg.eik_all and self._all_tets is None:
                        self._all_tets = torch.arange(g.num_tets, dtype=torch.int32, device=active.device)
                    tets = self._all_tets if cfg.eik_all else active
                    if world > 1:
                        tets = tets[rank * tets.numel() // world:(rank + 1) * tets.numel() // world]
                    eikonal_loss_async(g, f, tets, self._acc, cfg.lambda_eik, self.eik_loss, self.reg_stream)
                if cfg.lambda_nc > 0:
                    if self._nc_scratch is None:
                        self._nc_scratch = torch.empty(nc_scratch_bytes(g), dtype=torch.uint8, device=f.sdf.device)
                    n = g.resolution + 1
                    slab = (rank * n // world, (rank + 1) * n // world) if world > 1 else None
                    normal_consistency_loss_async(g, f, self._acc, cfg.lambda_nc, self.nc_loss, self.reg_stream,
                                                  self._nc_scratch, slab=slab)
        if cfg.sync_free:
            log = self._views_sync_free(s, list(views), d_maps_fn, active)
        else:
            log = [x for lane in self._views_threaded(s, views, d_maps_fn, active) for x in lane]
        for st in self.streams + [self.reg_stream]:
            main.wait_stream(st)
        if inputs_ready is not None:
            main.wait_event(inputs_ready)
        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1
        if self._fx is not None:
            # exact integer sums across ranks, then the same FP32 conversion on every rank
            if multi:
                dist.all_reduce(self._fx.fx, op=dist.ReduceOp.SUM, group=self.group)
                dist.all_reduce(self.status, op=dist.ReduceOp.SUM, group=self.group)
            self._fx.to_float(self.grads, status=self.status)
        elif multi:
            with torch.cuda.nvtx.range("gradient all-reduce"):
                dist.all_reduce(self._flat, op=dist.ReduceOp.SUM, group=self.group)
        if update is None:
            update = self.opt is not None
        if update:
            self.apply_update()
        pending = [k for k, x in enumerate(log) if x[1] is None]
        if pending:
            # one read per step: the sync-free views' sizes (the capacities of later steps) and
            # whether one overflowed — then Adam skipped the update on the device and the step
            # is re-run with the grown capacities
            vals = self._needs[:len(pending)].cpu().tolist()
            over = False
            for k, (K, M, P, L, ovf) in zip(pending, vals):
                vi = log[k][0]
                m0, p0, l0 = self._sizes.get(vi, (0, 0, 0))
                if ovf and M > m0:
                    # the tile pairs overflowed, so the pixel pairs were never counted: scale them
                    P = max(P, int(p0 * M / max(m0, 1)) + 1)
                self._sizes[vi] = (max(m0, M), max(p0, P), max(l0, L))
                log[k] = (vi, K, M, P)
                over |= bool(ovf)
            if over:
                if self._retry >= 3:
                    raise RuntimeError("a sync-free view still overflows after resizing")
                self._retry += 1
                if update:
                    self.opt.t -= 1  # the skipped update did not happen
                try:
                    return self(s, views, d_maps_fn, stats, inputs_ready, update)
                finally:
                    self._retry -= 1
        self.view_counts = {vi: (K, M, P) for vi, K, M, P in log}
        if stats is not None:
            for vi, K, M, P in log:
                if K:
                    stats.views += 1
                    stats.splats.append(K)
                    stats.pairs.append(M)
        return self.grads

    def _views_sync_free(self, s, views, d_maps_fn, active):
        """All views from this thread, round-robin over the renderers' streams; no host sync but a
        camera's first (sizing) view.  Returns [(view, K, M, P)] with K = None where the counts
        are still on the device (row i of self._needs for the i-th such view)."""
        g, f, cfg = self.grid, self.field, self.cfg
        lanes = len(self.renderers)
        if self._needs is None or self._needs.shape[0] < len(views):
            self._needs = torch.zeros((max(len(views), 8), 5), dtype=torch.int64, device=f.sdf.device)
        log, n_dyn = [], 0
        for i, vi in enumerate(views):
            r, st = self.renderers[i % lanes], self.streams[i % lanes]
            with torch.cuda.stream(st):
                size = self._sizes.get(vi)
                if size is None:  # first sight of this camera: the sizing path
                    r.set_caps(0, 0)
                    maps = r.forward(g, f, self.cameras[vi], s, active, n_w=cfg.n_w, stream=st)
                    K, M, P = r.counts
                    self._sizes[vi] = (M, P, r.max_list)
                    log.append((vi, K, M, P))
                    if K == 0:  # raster.py / fit.py skip a view without splats
                        continue
                else:
                    M, P, L = size
                    r.set_caps(int(M * 1.15) + 4096, int(P * 1.15) + 65536, int(L * 1.15) + 64, self._needs[n_dyn])
                    maps = r.forward(g, f, self.cameras[vi], s, active, n_w=cfg.n_w, stream=st)
                    n_dyn += 1
                    log.append((vi, None, None, None))
                r.backward(f, d_maps_fn(vi, maps), self._acc, stream=st, status=self.status)
        return log

    def _views_threaded(self, s, views, d_maps_fn, active):
        """views: one host thread per renderer/stream, so one view's sizing syncs never stall
        the other stream's launches (StepConfig.sync_free=False)"""
        g, f, cfg = self.grid, self.field, self.cfg
        lanes = len(self.renderers)
        work = [list(views)[j::lanes] for j in range(lanes)]

        def run_lane(j):
            r, st = self.renderers[j], self.streams[j]
            torch.cuda.set_device(st.device)  # worker threads start on device 0
            done = []
            with torch.cuda.stream(st):
                for vi in work[j]:
                    maps = r.forward(g, f, self.cameras[vi], s, active, n_w=cfg.n_w, stream=st)
                    K, M, P = r.counts
                    if K == 0:
                        done.append((vi, 0, M, P))
                        continue
                    r.backward(f, d_maps_fn(vi, maps), self._acc, stream=st, status=self.status)
                    done.append((vi, K, M, r.counts[2]))
            return done

        if lanes == 1:
            return [run_lane(0)]
        futs = [self._pool.submit(run_lane, j) for j in range(lanes)]
        return [fu.result() for fu in futs]

    def apply_update(self):
        """Adam + clamp on the device from the (all-reduced) gradient buffer; skipped on the
        device when the status flags a non-finite value (see check_status)."""
        if self.opt is None:
            raise RuntimeError("FitStep was built without an optimizer")
        self.opt.step_field(self.field, self.grads, self.grid.resolution, status=self.status)

    def check_status(self):
        """Host sync: raise like the reference when the last step saw non-finite values —
        ValueError for map gradients (raster.py:209-211), RuntimeError for gradients."""
        bad_maps, bad_grad = (float(v) for v in self.status[:2].tolist())
        if bad_maps:
            raise ValueError("non-finite incoming map gradients")
        if bad_grad:
            raise RuntimeError("non-finite parameter gradients")
