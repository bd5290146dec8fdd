"""The reference's kernel plugin contract on the B200 kernels.

The reference selects its per-pixel kernels with ``tetsplat.kernels.get_backend()``
(kernels/__init__.py:35-36), a module exporting ``forward_tiles``, ``reference_render``,
``backward_tiles``, ``eikonal_kernel`` and ``normal_consistency_kernel`` with the signatures
of ``_core.pyx:98-107, 232-239, 344-355, 544-547, 571-575``.  This module exports the same
five functions (and ``get_backend`` / ``get_backend_by_name`` / ``BACKEND_NAME``), so the
reference's ``raster.py`` and ``losses.py`` run on the sm_100a kernels unchanged — the
backend selector only has to return this module.

Contract kept from the reference:

* host numpy arguments, C-contiguous float64 geometry and int64 indices (anything else raises
  ValueError, like Cython's buffer acquisition); the caller allocates the maps zero-filled and
  the gradient buffers, kernels write maps in place and ACCUMULATE (+=) gradients;
* ``forward_tiles`` renders and returns the records of exactly the tiles in ``tile_ids``, so
  raster.py's chunked thread pool (raster.py:164-175) works: the chunks of one render share
  one device forward (the first chunk runs it for every tile, the others copy their tiles);
* ``SavedState.records`` are the reference's ``(tid, counts int32[256], idx int64[m],
  alpha float64[m])`` tuples, materialised on the device from the pair records
  (``ts_saved_records``); each tuple also carries the device state ``backward_tiles`` needs
  (records that did not come from this module's ``forward_tiles`` are rejected);
* calls are serialised with a lock (the reference calls from several threads at once).

Differences: the arithmetic is the B200 path's (FP32 with exact FP64 decisions, see
DESIGN.md §3), so values match the reference within the north_star bars, not bit for bit;
``alpha_clip`` must be ALPHA_CLIP, ``tile_size`` 16 and ``eps_normal`` EPS_NORMAL, and the
regularizer kernels need the Kuhn grid's own ``tets`` / ``edges`` (the device grid is
implicit) — other values raise ValueError.
"""
from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict

import numpy as np
import torch

from . import _native
from .field import EPS_NORMAL
from .grid import TetrahedralGrid
from .raster import RenderMaps, TileBins
from .raster import render_forward as _render_forward
from .splat import ALPHA_CLIP, SplatScene, scene_from_arrays

BACKEND_NAME = "b200"
TILE_PX = 256

_lock = threading.RLock()
_cache: "OrderedDict[tuple, object]" = OrderedDict()
_CACHE_MAX = 2


def get_backend():
    """kernels/__init__.py:35-36: the module with the five kernels."""
    import sys
    return sys.modules[__name__]


def get_backend_by_name(name: str):
    """kernels/__init__.py:39-47."""
    if name in ("b200", BACKEND_NAME):
        return get_backend()
    raise ValueError(f"unknown backend {name!r}")


# --- argument checks (Cython buffer acquisition raises ValueError) -----------------------

def _f64(a, name, ndim=None, writable=False):
    if not isinstance(a, np.ndarray) or a.dtype != np.float64:
        raise ValueError(f"{name}: Buffer dtype mismatch, expected 'double'")
    if not a.flags.c_contiguous:
        raise ValueError(f"{name}: ndarray is not C-contiguous")
    if ndim is not None and a.ndim != ndim:
        raise ValueError(f"{name}: Buffer has wrong number of dimensions (expected {ndim}, got {a.ndim})")
    if writable and not a.flags.writeable:
        raise ValueError(f"{name}: buffer source array is read-only")
    return a


def _i64(a, name):
    if not isinstance(a, np.ndarray) or a.dtype != np.int64:
        raise ValueError(f"{name}: Buffer dtype mismatch, expected 'long long'")
    if not a.flags.c_contiguous:
        raise ValueError(f"{name}: ndarray is not C-contiguous")
    return a


def _check_common(tile_size, alpha_clip):
    if int(tile_size) != 16:
        raise ValueError("the B200 kernels composite 16x16 tiles (tile_size must be 16)")
    if float(alpha_clip) != ALPHA_CLIP:
        raise ValueError(f"the B200 kernels clip alpha at ALPHA_CLIP = {ALPHA_CLIP!r}")


class _Cam:
    """The few camera fields the compositing ABI reads: image size and a depth range for the
    32-bit window keys (any near < far keeps the key monotone in mean depth)."""

    def __init__(self, width, height, near, far):
        self.width, self.height, self.near, self.far = int(width), int(height), float(near), float(far)

    def abi(self):
        c = _native.ts_camera()
        c.R[0] = c.R[4] = c.R[8] = 1.0
        c.fx = c.fy = 1.0
        c.cx, c.cy = self.width / 2.0, self.height / 2.0
        c.near_, c.far_ = self.near, self.far
        c.width, c.height = self.width, self.height
        return c


def _depth_range(md):
    if md.size == 0:
        return 0.0, 1.0
    lo, hi = float(md.min()), float(md.max())
    return (lo, hi) if hi > lo else (lo, lo + 1.0)


def _upload_scene(proj, depths, f, normals, mean_depth, bbox, colors, s, cam) -> SplatScene:
    K = mean_depth.shape[0]
    z = np.zeros(K, np.int32)
    return scene_from_arrays(z, np.zeros((K, 4), np.int32), proj, depths, f, normals, mean_depth, np.zeros(K),
                             bbox, s, cam, colors=colors)


def _remember(key, value):
    _cache[key] = value
    _cache.move_to_end(key)
    while len(_cache) > _CACHE_MAX:
        _cache.popitem(last=False)


class Record(tuple):
    """A SavedState record (tid, counts, idx, alpha) that also knows its device forward."""

    def __new__(cls, tid, counts, idx, alpha, state):
        r = super().__new__(cls, (tid, counts, idx, alpha))
        r._state = state
        return r


class _Forward:
    """One device forward (all tiles) shared by the chunked forward_tiles calls of a render."""

    def __init__(self, keep, verify, scene, bins, cam, maps, saved, with_color):
        self.keep, self.verify = keep, verify  # strong refs: the keyed ids cannot be reused
        self.scene, self.bins, self.cam, self.maps, self.saved = scene, bins, cam, maps, saved
        self.with_color = with_color
        H, W = cam.height, cam.width
        self.host = [None if m is None else m.detach().double().cpu().numpy() for m in
                     (maps.normal, maps.depth, maps.opacity, maps.color)]
        self.n_blend = saved.n_blend.cpu().numpy() if saved is not None else np.zeros((H, W), np.int32)
        self.dmaps = None  # (key, device d_maps) of the last backward_tiles


def _tile_window(tid, tiles_x, W, H):
    x0, y0 = (tid % tiles_x) * 16, (tid // tiles_x) * 16
    return x0, y0, min(16, W - x0), min(16, H - y0)


def forward_tiles(proj, depths, f, normals, mean_depth, colors_obj, bbox, tile_starts, tile_items, tile_ids,
                  tile_size, tiles_x, width, height, n_w, s, t_stop, alpha_clip, normal_map, depth_map,
                  opacity_map, color_map_obj, save_state):
    """_core.pyx:98-229: composite the tiles `tile_ids`, write their pixels of the maps in
    place, return their records [(tid, counts, idx, alpha)] when save_state (else [])."""
    _check_common(tile_size, alpha_clip)
    proj, depths, f = _f64(proj, "proj", 3), _f64(depths, "depths", 2), _f64(f, "f", 2)
    normals, mean_depth, bbox = _f64(normals, "normals", 2), _f64(mean_depth, "mean_depth", 1), _f64(bbox, "bbox", 2)
    tile_starts, tile_items = _i64(tile_starts, "tile_starts"), _i64(tile_items, "tile_items")
    normal_map = _f64(normal_map, "normal_map", 3, True)
    depth_map, opacity_map = _f64(depth_map, "depth_map", 2, True), _f64(opacity_map, "opacity_map", 2, True)
    has_color = colors_obj is not None and color_map_obj is not None
    if has_color:
        colors_obj = _f64(colors_obj, "colors", 2)
        color_map_obj = _f64(color_map_obj, "color_map", 3, True)
    W, H, tiles_x = int(width), int(height), int(tiles_x)
    tiles_y = (H + 15) // 16
    if tile_starts.shape[0] != tiles_x * tiles_y + 1:
        raise ValueError("tile_starts must hold tiles_x * tiles_y + 1 offsets")
    tids = [int(t) for t in tile_ids]
    with _lock:
        key = ("fwd", id(normal_map), id(proj), id(tile_items), id(tile_starts), id(colors_obj), int(n_w), float(s),
               float(t_stop), W, H, tiles_x, has_color)
        verify = (mean_depth.shape[0], tile_items.shape[0], float(mean_depth.sum()), int(tile_items.sum()))
        st = _cache.get(key)
        if st is None or st.verify != verify:
            st = _run_forward(proj, depths, f, normals, mean_depth, bbox, tile_starts, tile_items,
                              colors_obj if has_color else None, W, H, tiles_x, tiles_y, int(n_w), float(s),
                              float(t_stop), verify, (normal_map, proj, tile_items, tile_starts, colors_obj))
            _remember(key, st)
        outs = (normal_map, depth_map, opacity_map, color_map_obj if has_color else None)
        for t in tids:
            x0, y0, w, h = _tile_window(t, tiles_x, W, H)
            if w <= 0 or h <= 0:
                continue
            for o, src in zip(outs, st.host):
                if o is not None:
                    o[y0:y0 + h, x0:x0 + w] = src[y0:y0 + h, x0:x0 + w]
        if not save_state:
            return []
        return _records(st, tids, tiles_x, W, H)


def _run_forward(proj, depths, f, normals, mean_depth, bbox, starts, items, colors, W, H, tiles_x, tiles_y, n_w, s,
                 t_stop, verify, keep):
    near, far = _depth_range(mean_depth)
    cam = _Cam(W, H, near, far)
    sc = _upload_scene(proj, depths, f, normals, mean_depth, bbox, colors, s, cam)
    dev = sc.mean_depth.device
    T = tiles_x * tiles_y
    M = int(items.shape[0])
    d_starts = torch.as_tensor(starts, device=dev)
    d_items = torch.as_tensor(items.astype(np.int32), device=dev)
    flags = torch.zeros(T, dtype=torch.uint8, device=dev)
    L = _native.lib()
    _native.check(L.ts_bins_from_lists(_native.ptr(d_starts), _native.ptr(d_items), T, _native.ptr(sc.mean_depth),
                                       near, far, _native.ptr(flags), _native.stream_ptr()))
    e = torch.zeros(0, dtype=torch.int32, device=dev)
    bins = TileBins(16, tiles_x, tiles_y, d_starts, d_items, torch.zeros(len(sc) + 1, dtype=torch.int64, device=dev),
                    e, flags, torch.empty(M, dtype=torch.int32, device=dev),
                    int(np.diff(starts).max(initial=0)))
    if n_w < 1:  # the reference's window never fills: nothing is composited
        maps = RenderMaps.zeros(H, W, colors is not None, dev)
        saved = None
    else:
        maps, saved = _render_forward(sc, bins, cam, n_w=n_w, t_stop=t_stop, save_state=True)
    torch.cuda.synchronize()
    return _Forward(keep, verify, sc, bins, cam, maps, saved, colors is not None)


def _records(st, tids, tiles_x, W, H):
    counts = np.zeros((len(tids), TILE_PX), np.int32)
    for i, t in enumerate(tids):
        x0, y0, w, h = _tile_window(t, tiles_x, W, H)
        if w > 0 and h > 0:
            counts[i].reshape(16, 16)[:h, :w] = st.n_blend[y0:y0 + h, x0:x0 + w]
    off = np.zeros(counts.size + 1, np.int64)
    np.cumsum(counts.ravel(), out=off[1:])
    total = int(off[-1])
    idx = np.empty(total, np.int64)
    alpha = np.empty(total, np.float64)
    if total and st.saved is not None:
        dev = st.scene.mean_depth.device
        d_tiles = torch.as_tensor(np.asarray(tids, np.int32), device=dev)
        d_off = torch.as_tensor(off, device=dev)
        d_idx = torch.empty(total, dtype=torch.int64, device=dev)
        d_alpha = torch.empty(total, dtype=torch.float64, device=dev)
        sv = st.saved
        _native.check(_native.lib().ts_saved_records(
            st.scene.abi(), sv.bins.abi(), st.cam.abi(), _native.ptr(sv.item_off), _native.ptr(sv.pair_bits),
            _native.ptr(sv.pair_rec), _native.ptr(sv.n_proc), _native.ptr(d_tiles), len(tids), _native.ptr(d_off),
            _native.ptr(d_idx), _native.ptr(d_alpha), _native.stream_ptr()))
        idx = d_idx.cpu().numpy()
        alpha = d_alpha.cpu().numpy()
    out = []
    for i, t in enumerate(tids):
        a, b = int(off[i * TILE_PX]), int(off[(i + 1) * TILE_PX])
        out.append(Record(t, counts[i].copy(), idx[a:b].copy(), alpha[a:b].copy(), st))
    return out


def backward_tiles(proj, depths, f, normals, mean_depth, colors_obj, bbox, saved, tile_size, tiles_x, width, height,
                   s, alpha_clip, d_normal_map, d_depth_map, d_opacity_map, d_color_map_obj, d_f, d_proj, d_depths,
                   d_normals, d_mean_depth, d_colors_obj):
    """_core.pyx:344-471: accumulate the per-splat gradients of the records' tiles into
    d_f[K,4], d_proj[K,4,2], d_depths[K,4], d_normals[K,3], d_mean_depth[K] (, d_colors[K,3])."""
    _check_common(tile_size, alpha_clip)
    mean_depth = _f64(mean_depth, "mean_depth", 1)
    dn, dd, do = (_f64(d_normal_map, "d_normal_map", 3), _f64(d_depth_map, "d_depth_map", 2),
                  _f64(d_opacity_map, "d_opacity_map", 2))
    outs = [_f64(d_f, "d_f", 2, True), _f64(d_proj, "d_proj", 3, True), _f64(d_depths, "d_depths", 2, True),
            _f64(d_normals, "d_normals", 2, True), _f64(d_mean_depth, "d_mean_depth", 1, True)]
    has_color = colors_obj is not None and d_color_map_obj is not None and d_colors_obj is not None
    dc = _f64(d_color_map_obj, "d_color_map", 3) if has_color else None
    d_colors = _f64(d_colors_obj, "d_colors", 2, True) if has_color else None
    groups = {}
    for r in saved:
        stt = getattr(r, "_state", None)
        if stt is None:
            raise ValueError("backward_tiles needs records produced by this backend's forward_tiles")
        groups.setdefault(id(stt), (stt, []))[1].append(int(r[0]))
    with _lock:
        for stt, tids in groups.values():
            if stt.saved is None or not tids:
                continue
            if stt.scene.mean_depth.shape[0] != mean_depth.shape[0]:
                raise ValueError("records belong to a different scene")
            if has_color and not stt.with_color:
                raise ValueError("colour gradients need a forward_tiles call with colours")
            rows = _backward_rows(stt, tids, dn, dd, do, dc if has_color else None)
            outs[0] += rows[:, 0:4]
            outs[2] += rows[:, 4:8]
            outs[1][:, :, 0] += rows[:, 8:12]
            outs[1][:, :, 1] += rows[:, 12:16]
            outs[3] += rows[:, 16:19]
            outs[4] += rows[:, 19]
            if has_color:
                d_colors += rows[:, 20:23]


def _backward_rows(st, tids, dn, dd, do, dc):
    dev = st.scene.mean_depth.device
    key = (id(dn), id(dd), id(do), id(dc))
    if st.dmaps is None or st.dmaps[0] != key:
        for a in (dn, dd, do) + ((dc,) if dc is not None else ()):
            if not np.all(np.isfinite(a)):
                raise ValueError("non-finite incoming map gradients")
        t = lambda a: torch.as_tensor(a, device=dev).to(torch.float32).contiguous()
        st.dmaps = (key, (t(dn), t(dd), t(do), None if dc is None else t(dc)), (dn, dd, do, dc))
    d4 = st.dmaps[1]
    color = dc is not None
    K = len(st.scene)
    AS = 24 if color else 20
    rows = torch.zeros((K, AS), dtype=torch.float32, device=dev)
    sv, m = st.saved, st.maps
    P = ctypes.c_void_p
    maps = (P * 4)(m.normal.data_ptr(), m.depth.data_ptr(), m.opacity.data_ptr(),
                   m.color.data_ptr() if color else None)
    dmaps = (P * 4)(d4[0].data_ptr(), d4[1].data_ptr(), d4[2].data_ptr(), d4[3].data_ptr() if color else None)
    d_tiles = torch.as_tensor(np.asarray(tids, np.int32), device=dev)
    _native.check(_native.lib().ts_backward_tiles(
        st.scene.abi(), K, _native.ptr(st.scene.colors) if color else None, sv.bins.abi(), sv.bins.num_pairs,
        st.cam.abi(), _native.ptr(sv.item_off), _native.ptr(sv.pair_bits), _native.ptr(sv.pair_rec),
        ctypes.cast(maps, ctypes.POINTER(P)), ctypes.cast(dmaps, ctypes.POINTER(P)), _native.ptr(sv.n_proc),
        _native.ptr(d_tiles), len(tids), _native.ptr(rows), _native.stream_ptr()))
    return rows.double().cpu().numpy()


def reference_render(proj, depths, f, normals, mean_depth, colors_obj, bbox, width, height, s, alpha_clip, row_lo,
                     row_hi, normal_map, depth_map, opacity_map, color_map_obj):
    """_core.pyx:232-292: exact mean-depth order (ties by index), no early stop, rows
    [row_lo, row_hi) written in place.  One device render per image, shared by the row bands."""
    from .raster import render_reference as _render_reference
    if float(alpha_clip) != ALPHA_CLIP:
        raise ValueError(f"the B200 kernels clip alpha at ALPHA_CLIP = {ALPHA_CLIP!r}")
    proj, depths, f = _f64(proj, "proj", 3), _f64(depths, "depths", 2), _f64(f, "f", 2)
    normals, mean_depth, bbox = _f64(normals, "normals", 2), _f64(mean_depth, "mean_depth", 1), _f64(bbox, "bbox", 2)
    normal_map = _f64(normal_map, "normal_map", 3, True)
    depth_map, opacity_map = _f64(depth_map, "depth_map", 2, True), _f64(opacity_map, "opacity_map", 2, True)
    has_color = colors_obj is not None and color_map_obj is not None
    if has_color:
        colors_obj = _f64(colors_obj, "colors", 2)
        color_map_obj = _f64(color_map_obj, "color_map", 3, True)
    W, H = int(width), int(height)
    with _lock:
        key = ("ref", id(normal_map), id(proj), id(colors_obj), float(s), W, H, has_color)
        verify = (mean_depth.shape[0], float(mean_depth.sum()))
        hit = _cache.get(key)
        if hit is None or hit[0] != verify:
            near, far = _depth_range(mean_depth)
            cam = _Cam(W, H, near, far)
            sc = _upload_scene(proj, depths, f, normals, mean_depth, bbox, colors_obj if has_color else None, s, cam)
            if len(sc) == 0:
                maps = [np.zeros_like(a) for a in (normal_map, depth_map, opacity_map)] + \
                    [np.zeros_like(color_map_obj) if has_color else None]
            else:
                m = _render_reference(sc, cam)
                maps = [None if t is None else t.double().cpu().numpy() for t in (m.normal, m.depth, m.opacity, m.color)]
            hit = (verify, maps, (normal_map, proj, colors_obj))
            _remember(key, hit)
        lo, hi = max(0, int(row_lo)), min(H, int(row_hi))
        for o, src in zip((normal_map, depth_map, opacity_map, color_map_obj if has_color else None), hit[1]):
            if o is not None and src is not None:
                o[lo:hi] = src[lo:hi]


# --- regularizers on the implicit grid --------------------------------------------------

_grid_ok: "OrderedDict[int, tuple]" = OrderedDict()


def _grid_of(positions, tets, edges=None) -> TetrahedralGrid:
    N = positions.shape[0]
    R = int(round(N ** (1.0 / 3.0))) - 1
    if R < 1 or (R + 1) ** 3 != N:
        raise ValueError("positions must hold the (R+1)^3 vertices of a Kuhn grid")
    g = TetrahedralGrid(R)
    key = id(tets)
    hit = _grid_ok.get(key)
    if hit is None or hit[0] is not tets:
        tets = _i64(tets, "tets")
        if tets.shape != (g.num_tets, 4) or not np.array_equal(tets, g.tets_numpy()):
            raise ValueError("the B200 regularizers run on the Kuhn grid of build_grid (implicit on the device)")
        _grid_ok[key] = (tets,)
        while len(_grid_ok) > 4:
            _grid_ok.popitem(last=False)
    if edges is not None:
        edges = _i64(edges, "edges")
        if edges.shape != (g.num_edges, 2) or (edges.shape[0] and not (edges[:, 0] < edges[:, 1]).all()):
            raise ValueError("edges must be the grid's sorted (a, b) edge list")
    return g


def _field_on_device(g, positions, sdf):
    """(sdf, deformation = positions - rest) on the device; the kernels re-form the positions
    as rest + deformation (FP64, ulp-level differences only)."""
    positions = _f64(positions, "positions", 2)
    sdf = _f64(sdf, "sdf", 1)
    dev = torch.device("cuda", torch.cuda.current_device())
    ax = g.axis()
    rest = np.stack(np.meshgrid(ax, ax, ax, indexing="ij")[::-1], axis=-1).reshape(-1, 3)  # x fastest
    return _RawField(torch.as_tensor(sdf, device=dev).contiguous(),
                     torch.as_tensor(positions - rest, device=dev).contiguous())


class _RawField:
    """sdf / deformation on the device without the deformation clamp (the kernel contract
    takes positions as given)."""

    def __init__(self, sdf, deformation):
        self.sdf, self.deformation = sdf, deformation


def _accumulate(d_vert, d_sdf, d_deform):
    d = d_vert.double().cpu().numpy()
    d_sdf += d[:, 0]
    d_deform += d[:, 1:]


def eikonal_kernel(positions, sdf, tets, tet_set, eps_normal, d_sdf, d_deform):
    """_core.pyx:544-568: sum over tet_set of (|g| - 1)^2, gradients accumulated."""
    from .losses import eikonal_loss
    from .raster import GradientBuffers
    if float(eps_normal) != EPS_NORMAL:
        raise ValueError(f"the B200 regularizers use eps_normal = {EPS_NORMAL!r}")
    g = _grid_of(positions, tets)
    d_sdf, d_deform = _f64(d_sdf, "d_sdf", 1, True), _f64(d_deform, "d_deform", 2, True)
    tet_set = _i64(tet_set, "tet_set")
    with _lock:
        fs = _field_on_device(g, positions, sdf)
        gb = GradientBuffers.zeros(g.num_vertices, fs.sdf.device)
        loss, gb = eikonal_loss(g, fs, tet_set, out=gb)
        _accumulate(gb.d_vert, d_sdf, d_deform)
    return float(loss)


def normal_consistency_kernel(positions, sdf, tets, edges, eps_normal, d_sdf, d_deform):
    """_core.pyx:571-668: sum over edges of (1 - n_a . n_b), gradients accumulated."""
    from .losses import normal_consistency_loss
    from .raster import GradientBuffers
    if float(eps_normal) != EPS_NORMAL:
        raise ValueError(f"the B200 regularizers use eps_normal = {EPS_NORMAL!r}")
    g = _grid_of(positions, tets, edges)
    d_sdf, d_deform = _f64(d_sdf, "d_sdf", 1, True), _f64(d_deform, "d_deform", 2, True)
    with _lock:
        fs = _field_on_device(g, positions, sdf)
        gb = GradientBuffers.zeros(g.num_vertices, fs.sdf.device)
        loss, gb = normal_consistency_loss(g, fs, out=gb)
        _accumulate(gb.d_vert, d_sdf, d_deform)
    return float(loss)
