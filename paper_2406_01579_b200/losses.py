"""Eikonal and normal-consistency regularizers + MSE map losses (mirrors losses.py)."""
from __future__ import annotations

import torch

from . import _native
from .raster import FixedPointGradients, GradientBuffers, RenderMaps


def eikonal_loss(grid, field, tet_set, out: GradientBuffers | None = None, scale: float = 1.0,
                 stream=None) -> tuple[float, GradientBuffers]:
    """sum_k (|g_k| - 1)^2 over `tet_set` (losses.py:25-36).  Gradients (times `scale`)
    are accumulated into `out` when given (the fit loop's lambda weighting fused)."""
    dev = field.sdf.device
    out = out if out is not None else GradientBuffers.zeros(grid.num_vertices, dev)
    tet_set = torch.as_tensor(tet_set, device=dev).to(torch.int32).contiguous()
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    if tet_set.numel() == 0:
        return 0.0, out
    _native.check(_native.lib().ts_eikonal(_native.ptr(field.sdf), _native.ptr(field.deformation), grid.resolution,
                                           _native.ptr(tet_set), int(tet_set.numel()), float(scale),
                                           _native.ptr(out.d_vert), _native.ptr(loss), _native.stream_ptr(stream)))
    return float(loss.item()), out


def eikonal_loss_async(grid, field, tet_set, out, scale, loss, stream=None):
    """Sync-free variant: loss (device f64[1]) is overwritten, gradients accumulated (into a
    FixedPointGradients: fixed point, order-independent)."""
    fixed = isinstance(out, FixedPointGradients)
    fn = _native.lib().ts_eikonal_fx if fixed else _native.lib().ts_eikonal
    _native.check(fn(_native.ptr(field.sdf), _native.ptr(field.deformation), grid.resolution,
                     _native.ptr(tet_set), int(tet_set.numel()), float(scale),
                     _native.ptr(out.fx if fixed else out.d_vert), _native.ptr(loss), _native.stream_ptr(stream)))


def normal_consistency_loss(grid, field, out: GradientBuffers | None = None, scale: float = 1.0,
                            stream=None) -> tuple[float, GradientBuffers]:
    """Cosine misalignment between vertex normals across grid edges (losses.py:39-52)."""
    dev = field.sdf.device
    out = out if out is not None else GradientBuffers.zeros(grid.num_vertices, dev)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    normal_consistency_loss_async(grid, field, out, scale, loss, stream)
    return float(loss.item()), out


def normal_consistency_loss_async(grid, field, out, scale, loss, stream=None, scratch=None, slab=None):
    """Sync-free variant; `scratch` (uint8 device tensor of nc_scratch_bytes(grid) bytes)
    avoids per-call stream-ordered allocations.  `slab=(z0, z1)`: only the vertex layers
    z0 <= z < z1 (their gradients and the penalty of the edges they start) — the regularizer
    sharded over ranks; the slabs of all ranks sum to the full loss and gradient."""
    L = _native.lib()
    if slab is not None:
        fixed = isinstance(out, FixedPointGradients)
        _native.check(L.ts_normal_consistency_slab(
            _native.ptr(field.sdf), _native.ptr(field.deformation), grid.resolution, float(scale),
            None if fixed else _native.ptr(out.d_vert), _native.ptr(out.fx) if fixed else None,
            _native.ptr(loss), _native.ptr(scratch), int(slab[0]), int(slab[1]), _native.stream_ptr(stream)))
        return
    if isinstance(out, FixedPointGradients):
        _native.check(L.ts_normal_consistency_fx(_native.ptr(field.sdf), _native.ptr(field.deformation),
                                                 grid.resolution, float(scale), _native.ptr(out.fx),
                                                 _native.ptr(loss), _native.ptr(scratch), _native.stream_ptr(stream)))
        return
    if scratch is not None:
        _native.check(L.ts_normal_consistency_ws(_native.ptr(field.sdf), _native.ptr(field.deformation),
                                                 grid.resolution, float(scale), _native.ptr(out.d_vert),
                                                 _native.ptr(loss), _native.ptr(scratch), _native.stream_ptr(stream)))
        return
    _native.check(L.ts_normal_consistency(_native.ptr(field.sdf), _native.ptr(field.deformation),
                                          grid.resolution, float(scale), _native.ptr(out.d_vert),
                                          _native.ptr(loss), _native.stream_ptr(stream)))


def nc_scratch_bytes(grid) -> int:
    return int(_native.lib().ts_normal_consistency_scratch_bytes(grid.resolution))


def map_mse_loss(rendered: RenderMaps, target: RenderMaps, weights: dict, sync: bool = True):
    """losses.py:55-81: weighted per-map MSE and the exact gradient images.

    sync=False keeps the loss and its components as FP64 device scalars (no host round trip
    per view; the fit loop reads them once per iteration)."""
    if rendered.opacity.shape != target.opacity.shape:
        raise ValueError("rendered/target map shapes differ")
    npix = rendered.opacity.numel()
    comps = {}
    total = torch.zeros((), dtype=torch.float64, device=rendered.opacity.device)
    g = {"color": None}
    pairs = [("normal", rendered.normal, target.normal), ("depth", rendered.depth, target.depth),
             ("opacity", rendered.opacity, target.opacity)]
    if rendered.color is not None and target.color is not None:
        pairs.append(("color", rendered.color, target.color))
    for name, r, t in pairs:
        diff = r - torch.as_tensor(t, device=r.device, dtype=r.dtype)
        mse = (diff * diff).sum(dtype=torch.float64) / npix
        comps[f"mse_{name}"] = mse
        w = float(weights.get(name, 1.0))
        total = total + w * mse
        g[name] = (2.0 / npix) * w * diff
    grads = RenderMaps(g["normal"], g["depth"], g["opacity"], g["color"])
    if sync:
        vals = torch.stack([total, *comps.values()]).tolist()
        return vals[0], dict(zip(comps.keys(), vals[1:])), grads
    return total, comps, grads
