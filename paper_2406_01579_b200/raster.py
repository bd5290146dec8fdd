"""Tile-based forward rasterizer and analytic backward pass (mirrors raster.py).

All work runs in the sm_100a kernels of libtetsplat_b200.so (csrc/bin.cu, composite.cu);
this module owns the device buffers and keeps the reference's call signatures.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .splat import ALPHA_CLIP, T_STOP, SplatScene

TILE_SIZE = 16
DEFAULT_WINDOW = 5


@dataclass
class RenderMaps:
    """Opacity-premultiplied normal/depth/opacity (and optional color) images, FP32 on the
    device (raster.py:29-50)."""

    normal: torch.Tensor
    depth: torch.Tensor
    opacity: torch.Tensor
    color: torch.Tensor | None = None

    @classmethod
    def zeros(cls, height, width, with_color=False, device="cuda"):
        f = dict(dtype=torch.float32, device=device)
        return cls(torch.zeros((height, width, 3), **f), torch.zeros((height, width), **f),
                   torch.zeros((height, width), **f),
                   torch.zeros((height, width, 3), **f) if with_color else None)

    @classmethod
    def empty(cls, height, width, with_color=False, device="cuda"):
        f = dict(dtype=torch.float32, device=device)
        return cls(torch.empty((height, width, 3), **f), torch.empty((height, width), **f),
                   torch.empty((height, width), **f),
                   torch.empty((height, width, 3), **f) if with_color else None)

    def max_abs_difference(self, other: "RenderMaps") -> float:
        d = max(float((self.normal - other.normal).abs().max()), float((self.depth - other.depth).abs().max()),
                float((self.opacity - other.opacity).abs().max()))
        if self.color is not None and other.color is not None:
            d = max(d, float((self.color - other.color).abs().max()))
        return d

    def numpy(self):
        c = lambda t: None if t is None else t.detach().cpu().numpy().astype(np.float64)
        return c(self.normal), c(self.depth), c(self.opacity), c(self.color)


@dataclass
class TileBins:
    """Per-tile splat lists sorted by (tile id, quantized mean depth) (raster.py:53-71).

    starts/items equal the reference's bit for bit; pos_of, splat_off, nonmono and witems
    are the B200 extras (pair positions, resorting window)."""

    tile_size: int
    tiles_x: int
    tiles_y: int
    starts: torch.Tensor     # (T+1,) int64
    items: torch.Tensor      # (M,) int32
    splat_off: torch.Tensor  # (K+1,) int64
    pos_of: torch.Tensor     # (M,) int32
    nonmono: torch.Tensor    # (T,) uint8
    witems: torch.Tensor     # (M,) int32 — compositing lists (written by each forward)
    max_len: int = 0
    cpos: torch.Tensor | None = None  # (M,) int32 list position of each compositing entry
    clen: torch.Tensor | None = None  # (T,) int32 compositing-list length per tile

    @property
    def num_tiles(self) -> int:
        return self.tiles_x * self.tiles_y

    @property
    def num_pairs(self) -> int:
        return int(self.items.shape[0])

    def tile_list(self, tid: int) -> torch.Tensor:
        s = self.starts[tid:tid + 2].tolist()
        return self.items[s[0]:s[1]]

    def max_list_length(self) -> int:
        return self.max_len

    def abi(self) -> _native.ts_bins:
        b = _native.ts_bins()
        for n in ("starts", "splat_off", "items", "pos_of", "nonmono", "witems", "cpos", "clen"):
            t = getattr(self, n)
            setattr(b, n, t.data_ptr() if t is not None else None)
        return b


@dataclass
class GradientBuffers:
    """Loss derivatives per grid vertex (raster.py:74-91).  Stored interleaved as one FP32
    [N,4] buffer (d_sdf, d_deform xyz) — the all-reduce payload; d_sdf/d_deform are views."""

    d_vert: torch.Tensor
    d_color: torch.Tensor | None = None

    @classmethod
    def zeros(cls, num_vertices, device="cuda", num_tets_color: int | None = None):
        return cls(torch.zeros((num_vertices, 4), dtype=torch.float32, device=device),
                   None if num_tets_color is None else
                   torch.zeros((num_tets_color, 3), dtype=torch.float32, device=device))

    @property
    def d_sdf(self) -> torch.Tensor:
        return self.d_vert[:, 0]

    @property
    def d_deform(self) -> torch.Tensor:
        return self.d_vert[:, 1:]

    def __iadd__(self, other):
        self.d_vert += other.d_vert
        if self.d_color is not None and other.d_color is not None:
            self.d_color += other.d_color
        return self

    def scaled(self, w: float) -> "GradientBuffers":
        return GradientBuffers(self.d_vert * w, None if self.d_color is None else self.d_color * w)


FX_SCALE = 2.0 ** 36  # fixed-point gradients: value * 2^36 as int64 (include/tetsplat_b200.h)


@dataclass
class FixedPointGradients:
    """Deterministic accumulation target.  The reference merges per-chunk private buffers in a
    fixed order (raster.py:217-247), so its gradients are bitwise reproducible; here every
    contribution is added as the int64 round(v * 2^36) (integer addition is associative, so
    the sum does not depend on the order the atomics land in — across CTAs, streams and, all-
    reduced as int64, ranks).  fx: int64[4N + 1], the interleaved [N,4] layout of
    GradientBuffers.d_vert plus a count of dropped (non-finite or |v| >= 2^26) contributions;
    fx_color: int64[T,3] or None.  `to_float` converts (resolution 2^-36 ~ 1.5e-11)."""

    fx: torch.Tensor
    fx_color: torch.Tensor | None = None

    @classmethod
    def zeros(cls, num_vertices, device="cuda", num_tets_color: int | None = None):
        return cls(torch.zeros(4 * num_vertices + 1, dtype=torch.int64, device=device),
                   None if num_tets_color is None else
                   torch.zeros((num_tets_color, 3), dtype=torch.int64, device=device))

    @property
    def num_vertices(self) -> int:
        return (self.fx.numel() - 1) // 4

    @property
    def dropped(self) -> torch.Tensor:
        """device int64[1]: contributions dropped as non-finite or out of range"""
        return self.fx[-1:]

    def zero_(self):
        self.fx.zero_()
        if self.fx_color is not None:
            self.fx_color.zero_()
        return self

    def to_float(self, out: GradientBuffers | None = None, status: torch.Tensor | None = None,
                 stream=None) -> GradientBuffers:
        """FP32 gradients (overwriting `out`); status[1] += dropped count when `status` is given."""
        N = self.num_vertices
        dev = self.fx.device
        if out is None:
            out = GradientBuffers(torch.empty((N, 4), dtype=torch.float32, device=dev),
                                  None if self.fx_color is None else
                                  torch.empty(self.fx_color.shape, dtype=torch.float32, device=dev))
        L = _native.lib()
        _native.check(L.ts_fx_to_f32(_native.ptr(self.fx), 4 * N, _native.ptr(out.d_vert), _native.ptr(status),
                                     _native.stream_ptr(stream)))
        if self.fx_color is not None and out.d_color is not None:
            _native.check(L.ts_fx_to_f32(_native.ptr(self.fx_color), self.fx_color.numel(),
                                         _native.ptr(out.d_color), None, _native.stream_ptr(stream)))
        return out


@dataclass
class SavedState:
    """What the backward needs from the forward (raster.py:94-101).  Instead of per-pixel
    (idx, alpha) lists the B200 forward keeps the number of list entries each pixel
    consumed and its final composite (the forward maps)."""

    bins: TileBins
    n_w: int
    t_stop: float
    maps: RenderMaps
    n_proc: torch.Tensor   # (H,W) int32
    n_blend: torch.Tensor  # (H,W) int32 — the reference's per-pixel record counts
    item_off: torch.Tensor | None = None    # (M+1,) int64: first pair of each list position
    pair_bits: torch.Tensor | None = None   # (ceil(P/32)+1,) int32: blend bit per pair
    pair_rec: torch.Tensor | None = None    # (P,4) f32 (blending pairs): alpha, 1-alpha (negative:
    #   clipped), s*sigmoid(-s f_prev) | entry face, s*sigmoid(-s f_next) | exit face (low mantissa bits)


def bin_and_sort(scene: SplatScene, camera, tile_size: int = TILE_SIZE, stream=None) -> TileBins:
    """Replicate splats into overlapped tiles and sort by (tile id, depth) (raster.py:104-141)."""
    if tile_size != TILE_SIZE:
        raise ValueError("the B200 rasterizer uses 16x16 tiles (one 256-thread CTA per tile)")
    L = _native.lib()
    dev = scene.mean_depth.device
    tiles_x = (camera.width + tile_size - 1) // tile_size
    tiles_y = (camera.height + tile_size - 1) // tile_size
    T = tiles_x * tiles_y
    K = len(scene)
    starts = torch.zeros(T + 1, dtype=torch.int64, device=dev)
    splat_off = torch.zeros(K + 1, dtype=torch.int64, device=dev)
    nonmono = torch.zeros(T, dtype=torch.uint8, device=dev)
    if K == 0:
        e = torch.zeros(0, dtype=torch.int32, device=dev)
        return TileBins(tile_size, tiles_x, tiles_y, starts, e, splat_off, e, nonmono, e, 0)
    cam = camera.abi()
    sp = _native.stream_ptr(stream)
    M, maxL = _native.i64(), _native.i64()
    _native.check(L.ts_bin_count(_native.ptr(scene.bbox), _native.ptr(scene.mean_depth), K, cam, tile_size,
                                 _native.ptr(starts), _native.ptr(splat_off), M, maxL, sp))
    M = M.value
    buf = torch.empty(3 * max(M, 1), dtype=torch.int32, device=dev)
    bins = TileBins(tile_size, tiles_x, tiles_y, starts, buf[:M], splat_off, buf[M:2 * M], nonmono,
                    buf[2 * M:3 * M] if M else buf[:0], maxL.value)
    if M:
        _native.check(L.ts_bin_sort(_native.ptr(scene.bbox), _native.ptr(scene.mean_depth), K, cam, tile_size,
                                    bins.abi(), M, bins.max_len, sp))
    return bins


def render_forward(scene: SplatScene, bins: TileBins, camera, n_w: int = DEFAULT_WINDOW, t_stop: float = T_STOP,
                   save_state: bool = False, stream=None, timing=None):
    """Tile-based forward pass (raster.py:149-177).  Returns (RenderMaps, SavedState | None).
    `timing` = (start, end) CUDA events recorded around the compositing kernel launch."""
    if n_w < 1:
        raise ValueError("resorting window must be >= 1")
    L = _native.lib()
    dev = scene.mean_depth.device
    H, W = camera.height, camera.width
    with_color = scene.colors is not None
    maps = RenderMaps.empty(H, W, with_color, dev)
    n_proc = torch.empty((H, W), dtype=torch.int32, device=dev)
    n_blend = torch.empty((H, W), dtype=torch.int32, device=dev)
    K = len(scene)
    M = bins.num_pairs
    item_off = pair_bits = pair_rec = None
    if K == 0 or M == 0:
        for t in (maps.normal, maps.depth, maps.opacity, maps.color, n_proc, n_blend):
            if t is not None:
                t.zero_()
    else:
        sp = _native.stream_ptr(stream)
        # the compositing lists (window order, with their list positions) belong to this
        # forward: a later forward on the same bins with another n_w must not change the
        # order this SavedState's backward walks
        bins = dataclasses.replace(bins, witems=torch.empty(M, dtype=torch.int32, device=dev),
                                   cpos=torch.empty(M, dtype=torch.int32, device=dev),
                                   clen=torch.empty(bins.num_tiles, dtype=torch.int32, device=dev))
        sc_abi, b_abi, cam = scene.abi(), bins.abi(), camera.abi()
        item_off = torch.empty(M + 1, dtype=torch.int64, device=dev)
        npairs = _native.i64()
        _native.check(L.ts_forward_prepare(sc_abi, K, b_abi, M, cam, int(n_w), _native.ptr(item_off), npairs, sp))
        P = max(npairs.value, 1)
        pair_bits = torch.empty((P + 31) // 32 + 1, dtype=torch.int32, device=dev)
        pair_rec = torch.empty((P, 4), dtype=torch.float32, device=dev)
        if timing is not None:
            timing[0].record(stream if stream is not None else torch.cuda.current_stream())
        _native.check(L.ts_render_forward(sc_abi, K, _native.ptr(scene.colors), b_abi, M, cam,
                                          float(scene.steepness), float(t_stop), _native.ptr(item_off),
                                          npairs.value, _native.ptr(pair_bits), _native.ptr(pair_rec),
                                          _native.ptr(maps.normal), _native.ptr(maps.depth),
                                          _native.ptr(maps.opacity), _native.ptr(maps.color),
                                          _native.ptr(n_proc), _native.ptr(n_blend), sp))
        if timing is not None:
            timing[1].record(stream if stream is not None else torch.cuda.current_stream())
    saved = SavedState(bins, n_w, t_stop, maps, n_proc, n_blend, item_off, pair_bits,
                       pair_rec) if save_state else None
    return maps, saved


# A window at least as long as any list turns the N_w resorting into the exact mean-depth
# order (ties by splat index) — the order render_reference's global lexsort gives.
REFERENCE_WINDOW = 1 << 30


def render_reference(scene: SplatScene, camera, stream=None) -> RenderMaps:
    """Oracle renderer: exact per-pixel depth ordering, no early stop (raster.py:180-199,
    _core.reference_render _core.pyx:232-292).

    Every splat whose bbox holds a pixel is in that pixel's tile list, so the reference's
    per-pixel walk over the globally (mean depth, index)-sorted splats equals a walk over the
    tile list in that order: the tile lists sorted by (depth key, index) with an unbounded
    resorting window (which sorts each equal-key run by mean depth, ties by position) and
    compositing without early stop (t_stop = 0)."""
    bins = bin_and_sort(scene, camera, stream=stream)
    maps, _ = render_forward(scene, bins, camera, n_w=REFERENCE_WINDOW, t_stop=0.0, stream=stream)
    return maps


def _as_f32(t, dev):
    if t is None:
        return None
    return torch.as_tensor(t, device=dev).to(torch.float32).contiguous()


def render_backward(saved: SavedState, scene: SplatScene, grid, field, camera, d_maps: RenderMaps,
                    out: GradientBuffers | FixedPointGradients | None = None, stream=None, timing=None,
                    deterministic: bool = False) -> GradientBuffers | FixedPointGradients:
    """Exact reverse-mode pass: map gradients -> per-vertex SDF/deformation gradients
    (raster.py:206-306).  With `out`, gradients are accumulated into it (fused batch).
    `deterministic` (or a FixedPointGradients `out`): bitwise-reproducible fixed-point
    accumulation; without `out` the result is returned converted to FP32."""
    dev = scene.mean_depth.device
    dn, dd, do = _as_f32(d_maps.normal, dev), _as_f32(d_maps.depth, dev), _as_f32(d_maps.opacity, dev)
    for arr in (dn, dd, do):
        if not bool(torch.isfinite(arr).all()):
            raise ValueError("non-finite incoming map gradients")
    with_color = scene.colors is not None and d_maps.color is not None
    dc = _as_f32(d_maps.color, dev) if with_color else None
    convert = False
    if out is None and deterministic:
        out = FixedPointGradients.zeros(grid.num_vertices, dev, grid.num_tets if with_color else None)
        convert = True
    if out is None:
        out = GradientBuffers.zeros(grid.num_vertices, dev, grid.num_tets if with_color else None)
    fixed = isinstance(out, FixedPointGradients)
    K = len(scene)
    if K == 0 or saved.bins.num_pairs == 0:
        return out.to_float(stream=stream) if convert else out
    L = _native.lib()
    import ctypes
    maps = (ctypes.c_void_p * 4)(saved.maps.normal.data_ptr(), saved.maps.depth.data_ptr(),
                                 saved.maps.opacity.data_ptr(),
                                 saved.maps.color.data_ptr() if with_color else None)
    dmaps = (ctypes.c_void_p * 4)(dn.data_ptr(), dd.data_ptr(), do.data_ptr(), dc.data_ptr() if with_color else None)
    if timing is not None:
        timing[0].record(stream if stream is not None else torch.cuda.current_stream())
    fn = L.ts_render_backward_fx if fixed else L.ts_render_backward
    _native.check(fn(scene.abi(), K, _native.ptr(scene.colors), saved.bins.abi(),
                     saved.bins.num_pairs, camera.abi(), _native.ptr(saved.item_off),
                     _native.ptr(saved.pair_bits), _native.ptr(saved.pair_rec),
                     ctypes.cast(maps, ctypes.POINTER(ctypes.c_void_p)),
                     ctypes.cast(dmaps, ctypes.POINTER(ctypes.c_void_p)),
                     _native.ptr(saved.n_proc), _native.ptr(field.deformation), grid.resolution,
                     _native.ptr(out.fx if fixed else out.d_vert),
                     (_native.ptr(out.fx_color if fixed else out.d_color)) if with_color else None,
                     _native.stream_ptr(stream)))
    if timing is not None:
        timing[1].record(stream if stream is not None else torch.cuda.current_stream())
    return out.to_float(stream=stream) if convert else out
