"""paper_2406_01579_b200 — B200-native TeT-Splatting tetrahedron rasterizer.

Drop-in for the reference's render / backward / mesh-extraction path (tetsplat.splat,
tetsplat.raster, tetsplat.losses, tetsplat.grid) on sm_100a CUDA kernels.
"""
from .camera import Camera, orbit_camera, look_at, camera_from_json, camera_to_json
from .grid import TetrahedralGrid, TriangleMesh, build_grid, marching_tetrahedra, tet_vertex_ids
from .field import (FieldState, AnalyticShape, analytic_sdf, init_sphere, init_from_shape, deform_limit_for,
                    EPS_NORMAL)
from .splat import (T_FILTER, ALPHA_CLIP, T_STOP, EmptySceneError, SplatScene, prefilter, build_scene,
                    coarse_to_fine_filter, scene_from_arrays, active_aabb, rescale_grid_to_box)
from .raster import (TILE_SIZE, DEFAULT_WINDOW, RenderMaps, TileBins, GradientBuffers, FixedPointGradients,
                     SavedState, bin_and_sort, render_forward, render_reference, render_backward)
from .losses import eikonal_loss, normal_consistency_loss, map_mse_loss
from .mesh import rasterize_mesh, export_obj, load_obj
from .imgio import write_pfm, read_pfm, write_png, save_maps, save_checkpoint, load_checkpoint
from .fit import FitConfig, FitTrace, fit_field, make_targets, render_target, run_fit, s_schedule

BACKEND_NAME = "b200"
__version__ = "0.1.0"
