"""Optimisable field state on the device (mirrors field.py:22-177 of the reference).

sdf f64[N] and deformation f64[N,3] live in HBM; FP64 keeps the tile keys and exact
decisions bit-compatible with the reference (SURVEY.md §7 hard part 1).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

EPS_VOLUME = 1e-12
EPS_NORMAL = 1e-8
DEFORM_FRACTION = 0.45


@dataclass
class FieldState:
    sdf: torch.Tensor
    deformation: torch.Tensor
    deform_limit: float
    steepness: float | None = None

    def __post_init__(self):
        dev = self.sdf.device if isinstance(self.sdf, torch.Tensor) else "cuda"
        self.sdf = torch.as_tensor(self.sdf, dtype=torch.float64, device=dev).contiguous()
        self.deformation = torch.as_tensor(self.deformation, dtype=torch.float64, device=dev).contiguous()
        self.clamp_deformation()

    def clamp_deformation(self):
        self.deformation.clamp_(-self.deform_limit, self.deform_limit)

    def deformed_positions(self, grid) -> torch.Tensor:
        return grid.rest_positions(self.sdf.device) + self.deformation

    def copy(self) -> "FieldState":
        return FieldState(self.sdf.clone(), self.deformation.clone(), self.deform_limit, self.steepness)

    @classmethod
    def from_numpy(cls, sdf, deformation, deform_limit, steepness=None, device="cuda"):
        return cls(torch.as_tensor(np.asarray(sdf, dtype=np.float64), device=device),
                   torch.as_tensor(np.asarray(deformation, dtype=np.float64), device=device),
                   float(deform_limit), steepness)


def deform_limit_for(grid) -> float:
    return DEFORM_FRACTION * grid.cell_edge


@dataclass(frozen=True)
class AnalyticShape:
    """field.py:70-83: sphere (radius), torus (major, minor), box (half extents)."""

    kind: str
    params: tuple
    center: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        if self.kind not in ("sphere", "torus", "box"):
            raise ValueError(f"unknown shape kind {self.kind!r}")
        if any(p <= 0 for p in self.params):
            raise ValueError("shape parameters must be positive")


def analytic_sdf(shape: AnalyticShape, points: torch.Tensor) -> torch.Tensor:
    """field.py:86-104, evaluated on the device in FP64."""
    p = points.to(torch.float64) - torch.tensor(shape.center, dtype=torch.float64, device=points.device)
    if shape.kind == "sphere":
        return torch.linalg.norm(p, dim=-1) - shape.params[0]
    if shape.kind == "torus":
        major, minor = shape.params
        return torch.hypot(torch.hypot(p[..., 0], p[..., 1]) - major, p[..., 2]) - minor
    half = torch.tensor(shape.params, dtype=torch.float64, device=points.device)
    q = p.abs() - half
    return torch.linalg.norm(q.clamp_min(0.0), dim=-1) + q.max(dim=-1).values.clamp_max(0.0)


def init_sphere(grid, radius: float, device="cuda") -> FieldState:
    if not 0.0 < radius < 1.0:
        raise ValueError(f"sphere radius must be in (0, 1), got {radius}")
    pos = grid.rest_positions(device)
    return FieldState(torch.linalg.norm(pos, dim=1) - radius, torch.zeros_like(pos), deform_limit_for(grid))


def init_from_shape(grid, shape: AnalyticShape, device="cuda") -> FieldState:
    pos = grid.rest_positions(device)
    return FieldState(analytic_sdf(shape, pos), torch.zeros_like(pos), deform_limit_for(grid))
