"""Mesh-side helpers of the reference's mesh.py: the z-buffered mesh rasterizer (the
surface-limit reference the splatted maps are compared with, mesh.py:98-147) on the GPU, and
Wavefront OBJ I/O (mesh.py:48-76)."""
from __future__ import annotations

import numpy as np
import torch

from . import _native
from .grid import TriangleMesh


def rasterize_mesh(mesh: TriangleMesh, camera, device="cuda"):
    """(mask bool [H,W], depth f64 [H,W], normal f64 [H,W,3]) device tensors: coverage, camera
    depth of the nearest triangle (0 where uncovered) and its unit world-space face normal."""
    H, W = camera.height, camera.width
    mask = torch.zeros((H, W), dtype=torch.uint8, device=device)
    depth = torch.zeros((H, W), dtype=torch.float64, device=device)
    normal = torch.zeros((H, W, 3), dtype=torch.float64, device=device)
    if mesh.is_empty:
        return mask.bool(), depth, normal
    v = torch.as_tensor(np.ascontiguousarray(mesh.vertices, dtype=np.float64), device=device)
    t = torch.as_tensor(np.ascontiguousarray(mesh.triangles, dtype=np.int64), device=device)
    _native.check(_native.lib().ts_rasterize_mesh(_native.ptr(v), int(v.shape[0]), _native.ptr(t), int(t.shape[0]),
                                                  camera.abi(), _native.ptr(mask), _native.ptr(depth),
                                                  _native.ptr(normal), _native.stream_ptr(None)))
    return mask.bool(), depth, normal


def export_obj(mesh: TriangleMesh, path) -> None:
    """Write a Wavefront OBJ file (`v` records then `f` records, 1-based), mesh.py:48-58."""
    lines = ["v %.9g %.9g %.9g" % (v[0], v[1], v[2]) for v in mesh.vertices]
    lines += ["f %d %d %d" % (t[0] + 1, t[1] + 1, t[2] + 1) for t in mesh.triangles]
    with open(path, "w") as fh:
        fh.write("\n".join(lines))
        if lines:
            fh.write("\n")


def load_obj(path) -> TriangleMesh:
    """mesh.py:61-76."""
    verts, tris = [], []
    with open(path) as fh:
        for line in fh:
            parts = line.split()
            if not parts:
                continue
            if parts[0] == "v":
                verts.append([float(x) for x in parts[1:4]])
            elif parts[0] == "f":
                tris.append([int(p.split("/")[0]) - 1 for p in parts[1:4]])
    return TriangleMesh(np.asarray(verts, dtype=np.float64).reshape(-1, 3),
                        np.asarray(tris, dtype=np.int64).reshape(-1, 3))
