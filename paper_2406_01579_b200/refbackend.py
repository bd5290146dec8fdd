"""Reference-side binding: the reference's raster entry points —
`render_forward` (raster.py:149) and `render_backward` (raster.py:206) — on the reference's
own host objects (numpy SplatScene / TileBins / Camera / TetrahedralGrid / FieldState /
RenderMaps), executed by the B200 kernels through the C ABI.

Objects are duck-typed on the reference's field names, so `tetsplat.raster` can route its two
calls here unchanged (tests/test_gpu_refbackend.py drives it with mirror types of the same layout).
The tile lists are rebuilt on the device from the scene — they equal the reference's
`bin_and_sort` output bit for bit (tests/test_gpu_parity.py::test_bins_bitexact) — and the
forward's saved state stays on the device until `render_backward`.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .camera import Camera
from .field import FieldState
from .grid import build_grid
from .raster import RenderMaps, bin_and_sort
from .raster import render_backward as _render_backward
from .raster import render_forward as _render_forward
from .splat import scene_from_arrays


def _camera(camera) -> Camera:
    return Camera(int(camera.width), int(camera.height), float(camera.fy), np.asarray(camera.rotation, np.float64),
                  np.asarray(camera.translation, np.float64), float(camera.near), float(camera.far))


@dataclass
class DeviceSaved:
    """What render_forward hands back for render_backward (the reference's SavedState slot)."""

    scene: object
    saved: object
    camera: Camera


def render_forward(scene, bins, camera, n_w: int = 5, t_stop: float = 1e-4, save_state: bool = False,
                   maps_type=None):
    """raster.py:149-177 on host objects: returns (maps, saved).  `maps` is built with
    `maps_type(normal, depth, opacity, color)` (the caller's RenderMaps class) when given, else
    a tuple of FP64 numpy arrays; `saved` is a DeviceSaved (None unless save_state)."""
    del bins  # rebuilt on the device from the same scene (bit-identical lists)
    cam = _camera(camera)
    sc = scene_from_arrays(scene.tet_ids, scene.vert_ids, scene.proj, scene.depths, scene.f, scene.normals,
                           scene.mean_depth, scene.alpha_max, scene.bbox, scene.steepness, cam,
                           colors=getattr(scene, "colors", None))
    b = bin_and_sort(sc, cam)
    maps, saved = _render_forward(sc, b, cam, n_w=n_w, t_stop=t_stop, save_state=save_state)
    arrays = maps.numpy()
    out = maps_type(*arrays) if maps_type is not None else arrays
    return out, (DeviceSaved(sc, saved, cam) if save_state else None)


def render_backward(saved: DeviceSaved, scene, grid, field, camera, d_maps, grads_type=None):
    """raster.py:206-306 on host objects: dL/dmaps (numpy) in, vertex gradients out — built
    with `grads_type(d_sdf, d_deform)` (the caller's GradientBuffers class) when given, else a
    (d_sdf, d_deform) tuple of FP64 numpy arrays (the device sums are FP32)."""
    if not isinstance(saved, DeviceSaved):
        raise ValueError("render_backward needs the state render_forward(save_state=True) returned")
    del scene, camera  # the device copies in `saved` are the same scene and camera
    g = build_grid(int(grid.resolution))
    fs = FieldState.from_numpy(field.sdf, field.deformation, float(field.deform_limit))
    dm = RenderMaps(d_maps.normal, d_maps.depth, d_maps.opacity, getattr(d_maps, "color", None))
    gb = _render_backward(saved.saved, saved.scene, g, fs, saved.camera, dm)
    d_sdf = gb.d_sdf.double().cpu().numpy()
    d_def = gb.d_deform.double().cpu().numpy()
    return grads_type(d_sdf, d_def) if grads_type is not None else (d_sdf, d_def)
