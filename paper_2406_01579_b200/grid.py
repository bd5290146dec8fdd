"""Implicit Kuhn tetrahedral grid and Marching Tetrahedra (mirrors grid.py of the reference).

The B200 framework never materialises connectivity: vertex id x + n*y + n^2*z and tet id
cell*6 + p are evaluated inside the kernels (csrc/common.cuh: tet_vertices).  Explicit
arrays are available on demand for interop/tests only.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native

# grid.py:18 — Kuhn subdivision axis permutations
AXIS_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


@dataclass(frozen=True)
class TetrahedralGrid:
    """Static connectivity of the deformable grid over [-1,1]^3 (grid.py:21-53)."""

    resolution: int

    def __post_init__(self):
        if self.resolution < 1:
            raise ValueError(f"resolution must be >= 1, got {self.resolution}")

    @property
    def num_vertices(self) -> int:
        return (self.resolution + 1) ** 3

    @property
    def num_tets(self) -> int:
        return 6 * self.resolution ** 3

    @property
    def num_edges(self) -> int:
        n = self.resolution + 1
        return 3 * n * n * (n - 1) + 3 * n * (n - 1) ** 2 + (n - 1) ** 3

    @property
    def cell_edge(self) -> float:
        return 2.0 / self.resolution

    def axis(self) -> np.ndarray:
        return np.linspace(-1.0, 1.0, self.resolution + 1)

    def rest_positions(self, device="cuda") -> torch.Tensor:
        """(N,3) float64, x fastest (grid.py:71-73)."""
        ax = torch.as_tensor(self.axis(), dtype=torch.float64, device=device)
        zz, yy, xx = torch.meshgrid(ax, ax, ax, indexing="ij")
        return torch.stack([xx.reshape(-1), yy.reshape(-1), zz.reshape(-1)], dim=1)

    def tets_numpy(self) -> np.ndarray:
        """Explicit (K,4) int64 connectivity, identical to the reference's build_grid."""
        R, n = self.resolution, self.resolution + 1
        ix, iy, iz = np.meshgrid(np.arange(R), np.arange(R), np.arange(R), indexing="ij")
        base = np.stack([ix.ravel(), iy.ravel(), iz.ravel()], axis=1)
        per = []
        for pi, p in enumerate(AXIS_PERMS):
            c = np.zeros((4, 3), dtype=np.int64)
            c[1, p[0]] = 1
            c[2] = c[1]
            c[2, p[1]] = 1
            c[3] = 1
            if pi in (1, 2, 5):  # odd permutations: negative volume, swap v2/v3 (grid.py:100-102)
                c[[2, 3]] = c[[3, 2]]
            ids = base[:, None, :] + c[None]
            per.append(ids[..., 0] + n * ids[..., 1] + n * n * ids[..., 2])
        return np.stack(per, axis=1).reshape(-1, 4)


def tet_vertex_ids(grid: TetrahedralGrid, tets: torch.Tensor) -> torch.Tensor:
    """(n,4) int64 vertex ids of the tets `tets` (device), the implicit formula of tets_numpy
    (grid.py:86-117) evaluated on the device."""
    R, n = grid.resolution, grid.resolution + 1
    t = tets.to(torch.int64)
    cell, p = t // 6, t % 6
    ix, iy, iz = cell // (R * R), (cell // R) % R, cell % R
    corners = torch.zeros((6, 4, 3), dtype=torch.int64, device=t.device)
    for pi, perm in enumerate(AXIS_PERMS):
        c = corners[pi]
        c[1, perm[0]] = 1
        c[2] = c[1]
        c[2, perm[1]] = 1
        c[3] = 1
        if pi in (1, 2, 5):
            c[[2, 3]] = c[[3, 2]].clone()
    off = corners[p]  # (n,4,3)
    x, y, z = ix[:, None] + off[..., 0], iy[:, None] + off[..., 1], iz[:, None] + off[..., 2]
    return x + n * y + n * n * z


def build_grid(resolution: int) -> TetrahedralGrid:
    """grid.py:64-117 (implicit: O(1) instead of the reference's 21-230 s at R=128-256)."""
    return TetrahedralGrid(int(resolution))


@dataclass
class TriangleMesh:
    """Indexed triangle soup (mesh.py:10-45): vertices (V,3) float64, triangles (F,3) int64."""

    vertices: np.ndarray
    triangles: np.ndarray

    @property
    def is_empty(self) -> bool:
        return len(self.triangles) == 0

    def edge_counts(self):
        if self.is_empty:
            return np.zeros((0, 2), dtype=np.int64), np.zeros(0, dtype=np.int64)
        e = np.concatenate([self.triangles[:, [0, 1]], self.triangles[:, [1, 2]], self.triangles[:, [2, 0]]])
        return np.unique(np.sort(e, axis=1), axis=0, return_counts=True)

    def euler_characteristic(self) -> int:
        if self.is_empty:
            return 0
        edges, _ = self.edge_counts()
        return int(len(np.unique(self.triangles)) - len(edges) + len(self.triangles))

    def is_watertight(self) -> bool:
        _, counts = self.edge_counts()
        return len(counts) > 0 and bool(np.all(counts == 2))


def marching_tetrahedra(grid: TetrahedralGrid, field, stream=None) -> TriangleMesh:
    """Zero level set as a welded triangle mesh (grid.py:136-239), computed on the GPU
    (csrc/mt.cu).  f < 0 inside, f = 0 counts as outside."""
    L = _native.lib()
    R = grid.resolution
    sp = _native.stream_ptr(stream)
    nv, nt = _native.i64(), _native.i64()
    h = ctypes.c_void_p()
    _native.check(L.ts_marching_tets_run(_native.ptr(field.sdf), _native.ptr(field.deformation), R,
                                         ctypes.byref(h), nv, nt, sp))
    try:
        # pinned host buffers (torch's caching host allocator): the D2H is a DMA copy, and the
        # returned numpy arrays share their memory
        V = torch.empty((nv.value, 3), dtype=torch.float64, pin_memory=True)
        F = torch.empty((nt.value, 3), dtype=torch.int64, pin_memory=True)
        if nv.value and nt.value:
            _native.check(L.ts_marching_tets_fetch(h, V.data_ptr(), F.data_ptr()))
    finally:
        _native.check(L.ts_marching_tets_release(h))
    if nv.value == 0 or nt.value == 0:
        return TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64))
    return TriangleMesh(V.numpy(), F.numpy())
