"""Reference-side binding: the reference's hot-path entry points —
`render_forward` (raster.py:149), `render_backward` (raster.py:206), `prefilter`
(splat.py:66), `bin_and_sort` (raster.py:104), `eikonal_loss` / `normal_consistency_loss`
(losses.py:25,39) and `marching_tetrahedra` (grid.py:136) — on the reference's own host
objects (numpy SplatScene / TileBins / Camera / TetrahedralGrid / FieldState / RenderMaps),
executed by the B200 kernels through the C ABI.

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
from .grid import marching_tetrahedra as _marching_tetrahedra
from .losses import eikonal_loss as _eikonal_loss
from .losses import normal_consistency_loss as _normal_consistency_loss
from .raster import RenderMaps, bin_and_sort
from .raster import render_backward as _render_backward
from .raster import render_forward as _render_forward
from .splat import prefilter as _prefilter
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
    with `grads_type(d_sdf, d_deform[, d_color])` (the caller's GradientBuffers class) when
    given, else a tuple of FP64 numpy arrays (the device sums are FP32)."""
    if not isinstance(saved, DeviceSaved):
        raise ValueError("render_backward needs the state render_forward(save_state=True) returned")
    del scene, camera  # the device copies in `saved` are the same scene and camera
    g = build_grid(int(grid.resolution))
    fs = _field(field)
    dm = RenderMaps(d_maps.normal, d_maps.depth, d_maps.opacity, getattr(d_maps, "color", None))
    gb = _render_backward(saved.saved, saved.scene, g, fs, saved.camera, dm)
    return _grads(gb, grads_type)


def _field(field) -> FieldState:
    return FieldState.from_numpy(field.sdf, field.deformation, float(field.deform_limit))


def _grads(gb, grads_type):
    """(d_sdf, d_deform[, d_color]) — d_color (num_tets, 3) when the scene had colours and
    the map gradients a colour image (raster.py:303-305), like the reference's GradientBuffers."""
    d_sdf = gb.d_sdf.double().cpu().numpy()
    d_def = gb.d_deform.double().cpu().numpy()
    if gb.d_color is None:
        return grads_type(d_sdf, d_def) if grads_type is not None else (d_sdf, d_def)
    d_col = gb.d_color.double().cpu().numpy()
    return grads_type(d_sdf, d_def, d_col) if grads_type is not None else (d_sdf, d_def, d_col)


def prefilter(grid, field, s, threshold=1.0 / 255.0):
    """splat.py:66-69: increasing int64 ids of the tets whose alpha_max reaches `threshold`."""
    return _prefilter(build_grid(int(grid.resolution)), _field(field), float(s), threshold).cpu().numpy().astype(
        np.int64)


def bin_and_sort_arrays(scene, camera, tile_size=16):
    """raster.py:104-141 on a host SplatScene: (tile_size, tiles_x, tiles_y, starts i64, items
    i64) — the fields of the reference's TileBins, bit for bit."""
    cam = _camera(camera)
    sc = scene_from_arrays(scene.tet_ids, scene.vert_ids, scene.proj, scene.depths, scene.f, scene.normals,
                           scene.mean_depth, scene.alpha_max, scene.bbox, scene.steepness, cam)
    b = bin_and_sort(sc, cam, tile_size)
    return (b.tile_size, b.tiles_x, b.tiles_y, b.starts.cpu().numpy(), b.items.cpu().numpy().astype(np.int64))


def eikonal_loss(grid, field, tet_set, grads_type=None):
    """losses.py:25-36: (loss, gradients)."""
    loss, gb = _eikonal_loss(build_grid(int(grid.resolution)), _field(field), np.asarray(tet_set))
    return loss, _grads(gb, grads_type)


def normal_consistency_loss(grid, field, grads_type=None):
    """losses.py:39-52: (loss, gradients)."""
    loss, gb = _normal_consistency_loss(build_grid(int(grid.resolution)), _field(field))
    return loss, _grads(gb, grads_type)


def marching_tetrahedra(grid, field, mesh_type=None):
    """grid.py:136-239: the welded mesh as `mesh_type(vertices, triangles)` (the caller's
    TriangleMesh class) or a (vertices f64[V,3], triangles i64[F,3]) tuple — bit for bit."""
    m = _marching_tetrahedra(build_grid(int(grid.resolution)), _field(field))
    return mesh_type(m.vertices, m.triangles) if mesh_type is not None else (m.vertices, m.triangles)
