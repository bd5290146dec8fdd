"""Prefilter + per-view splat setup on the device (mirrors splat.py of the reference)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native

T_FILTER = 1.0 / 255.0     # splat.py:13
ALPHA_CLIP = 1.0 - 1e-4    # splat.py:14
T_STOP = 1e-4              # splat.py:15
EPS_AREA = 1e-12           # splat.py:16
FACES = np.array([[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]], dtype=np.int64)
RECORD_BYTES = 96


class EmptySceneError(RuntimeError):
    """No tetrahedron survives pre-filtering (splat.py:22-23)."""


def prefilter(grid, field, s: float, threshold: float = T_FILTER, stream=None) -> torch.Tensor:
    """Ids (int32, increasing) of tets whose opacity upper bound reaches `threshold`
    (splat.py:66-69), via K1 on the implicit grid."""
    L = _native.lib()
    out = torch.empty(grid.num_tets, dtype=torch.int32, device=field.sdf.device)
    n = _native.i64()
    _native.check(L.ts_prefilter(_native.ptr(field.sdf), grid.resolution, float(s), float(threshold),
                                 _native.ptr(out), n, _native.stream_ptr(stream)))
    return out[:n.value]


def active_aabb(grid, field, active, margin: float = 0.1) -> np.ndarray:
    """splat.py:70-74: AABB of the active tets' deformed vertices, padded by margin x extent
    ((2,3) float64, computed on the device)."""
    from .grid import tet_vertex_ids
    act = torch.as_tensor(active, device=field.sdf.device)
    vid = tet_vertex_ids(grid, act).reshape(-1)
    pos = field.deformed_positions(grid)[vid]
    lo, hi = pos.min(dim=0).values, pos.max(dim=0).values
    pad = margin * (hi - lo)
    return torch.stack([lo - pad, hi + pad]).cpu().numpy()


def rescale_grid_to_box(grid, box) -> np.ndarray:
    """splat.py:77-83: the rest positions of the grid with the canonical cube mapped affinely
    onto `box` ((N,3) float64, same vertex order).  The device grid stays the canonical Kuhn
    grid (connectivity is identical); only positional field functions are sampled here."""
    lo, hi = (np.asarray(b, dtype=np.float64) for b in box)
    rest = grid.rest_positions("cpu").numpy()
    return (rest + 1.0) / 2.0 * (hi - lo) + lo


def coarse_to_fine_filter(grid, field, s: float, threshold: float = T_FILTER, margin: float = 0.1,
                          field_fn=None, stream=None):
    """splat.py:88-109: full-grid prefilter, AABB of the survivors (plus margin), and — when
    `field_fn` (a positional SDF callable) is given — a second prefilter of the field resampled
    on the grid rescaled to that box.  Returns (active ids, box)."""
    active = prefilter(grid, field, s, threshold, stream)
    if active.numel() == 0:
        raise EmptySceneError("pre-filtering removed every tetrahedron")
    box = active_aabb(grid, field, active, margin)
    if field_fn is not None:
        from .field import FieldState
        sdf = np.asarray(field_fn(rescale_grid_to_box(grid, box)), dtype=np.float64)
        fine = FieldState.from_numpy(sdf, np.zeros((grid.num_vertices, 3)), field.deform_limit,
                                     device=field.sdf.device)
        active = prefilter(grid, fine, s, threshold, stream)
    return active, box


@dataclass
class SplatScene:
    """Culled, pre-filtered splats of one view (splat.py:177-200), device resident.

    FP64 arrays mirror the reference; `records` is the compact FP32 compositing record.
    """

    tet_ids: torch.Tensor      # (K,) int32
    vert_ids: torch.Tensor     # (K,4) int32
    proj: torch.Tensor         # (K,4,2) f64
    depths: torch.Tensor       # (K,4) f64
    f: torch.Tensor            # (K,4) f64
    normals: torch.Tensor      # (K,3) f64
    mean_depth: torch.Tensor   # (K,) f64
    alpha_max: torch.Tensor    # (K,) f64
    bbox: torch.Tensor         # (K,4) f64
    records: torch.Tensor      # (K,96) uint8
    steepness: float = 1.0
    colors: torch.Tensor | None = None  # (K,3) f32

    def __len__(self):
        return int(self.tet_ids.shape[0])

    def abi(self) -> _native.ts_scene:
        s = _native.ts_scene()
        for name in ("tet_ids", "vert_ids", "proj", "depths", "f", "normals", "mean_depth", "alpha_max", "bbox",
                     "records"):
            setattr(s, name, getattr(self, name).data_ptr())
        return s


def _alloc_scene(K: int, device) -> dict:
    f64 = dict(dtype=torch.float64, device=device)
    return dict(tet_ids=torch.empty(K, dtype=torch.int32, device=device),
                vert_ids=torch.empty((K, 4), dtype=torch.int32, device=device),
                proj=torch.empty((K, 4, 2), **f64), depths=torch.empty((K, 4), **f64),
                f=torch.empty((K, 4), **f64), normals=torch.empty((K, 3), **f64),
                mean_depth=torch.empty(K, **f64), alpha_max=torch.empty(K, **f64),
                bbox=torch.empty((K, 4), **f64),
                records=torch.empty((K, RECORD_BYTES), dtype=torch.uint8, device=device))


def build_scene(grid, field, camera, s: float, active=None, colors=None, threshold: float = T_FILTER,
                stream=None) -> SplatScene:
    """Project the active tets into a SplatScene for one camera (splat.py:203-245) — K2."""
    L = _native.lib()
    dev = field.sdf.device
    if active is None:
        active = prefilter(grid, field, s, threshold, stream)
    active = torch.as_tensor(active, device=dev).to(torch.int32).contiguous()
    n_act = int(active.shape[0])
    arrs = _alloc_scene(max(n_act, 1), dev)
    tmp = SplatScene(**arrs, steepness=float(s))
    out = tmp.abi()
    k = _native.i64()
    cam = camera.abi()
    _native.check(L.ts_build_scene(_native.ptr(field.sdf), _native.ptr(field.deformation), grid.resolution,
                                   cam, float(s), _native.ptr(active), n_act, out, k, _native.stream_ptr(stream)))
    K = k.value
    sl = {n: v[:K] for n, v in arrs.items()}
    col = None
    if colors is not None:
        colors = torch.as_tensor(colors, device=dev)
        col = colors[sl["tet_ids"].long()].to(torch.float32).contiguous()
    return SplatScene(**sl, steepness=float(s), colors=col)


def scene_from_arrays(tet_ids, vert_ids, proj, depths, f, normals, mean_depth, alpha_max, bbox, steepness,
                      camera, colors=None, device="cuda", stream=None) -> SplatScene:
    """Upload a SplatScene given as reference-layout arrays (e.g. from the CPU reference)
    and derive its compositing records on the device."""
    L = _native.lib()
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), device=device).to(dt).contiguous()
    K = len(tet_ids)
    sc = SplatScene(tet_ids=t(tet_ids, torch.int32), vert_ids=t(vert_ids, torch.int32),
                    proj=t(proj, torch.float64), depths=t(depths, torch.float64), f=t(f, torch.float64),
                    normals=t(normals, torch.float64), mean_depth=t(mean_depth, torch.float64),
                    alpha_max=t(alpha_max, torch.float64), bbox=t(bbox, torch.float64),
                    records=torch.empty((max(K, 1), RECORD_BYTES), dtype=torch.uint8, device=device)[:K],
                    steepness=float(steepness),
                    colors=None if colors is None else t(colors, torch.float32))
    if K:
        _native.check(L.ts_prepare_records(sc.abi(), K, camera.width, camera.height, _native.stream_ptr(stream)))
    return sc
