"""ts_oracle — TEST INFRASTRUCTURE ONLY: the CPU checker for the B200 rasterizer.

A numpy restatement of the TeT-Splatting reference's hot path
(/root/reference/pkg/src/tetsplat: grid.py, camera.py, field.py, splat.py,
raster.py, losses.py).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import it; the
product package never does.

Per-pixel loops run in one of two CPU kernel backends:
  * ``"ref"`` — the reference's own Cython kernels (kernels/_core.pyx) compiled
    from /root/reference by ``oracle/Makefile`` into ``oracle/_ref/`` (the real
    reference code, used whenever it was built);
  * ``"c"``   — ``oracle/liboracle.so``, a plain-C restatement of the same loops
    (ts_oracle_kernels.c), OpenMP-threaded.
Both are checked against each other and against the committed golden fixtures
(tests/golden/, generated from the unmodified reference package by
tests/golden/make_golden.py), which pins this oracle.

Arrays follow the reference's layouts and dtypes exactly: float64 geometry,
int64 indices.
"""

from __future__ import annotations

import ctypes
import glob
import math
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

# --- constants (splat.py:13-16, field.py:10-12, raster.py:16-17) ---------------
T_FILTER = 1.0 / 255.0
ALPHA_CLIP = 1.0 - 1e-4
T_STOP = 1e-4
EPS_NORMAL = 1e-8
DEFORM_FRACTION = 0.45
TILE_SIZE = 16
DEFAULT_WINDOW = 5
_GOLDEN = 0.6180339887498949  # camera.py:10
_AXIS_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]  # grid.py:18


class EmptySceneError(RuntimeError):
    pass


# --- kernel backends ---------------------------------------------------------------

_REF = None
_LIB = None


def _load_ref():
    global _REF
    if _REF is None:
        cands = glob.glob(os.path.join(HERE, "_ref", "_core*.so"))
        if not cands:
            return None
        import importlib.util
        spec = importlib.util.spec_from_file_location("_core", cands[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _REF = mod
    return _REF


def _load_c():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            return None
        lib = ctypes.CDLL(path)
        P = ctypes.c_void_p
        I, D, L = ctypes.c_int, ctypes.c_double, ctypes.c_int64
        lib.or_forward.argtypes = [P] * 9 + [I] * 6 + [D] * 3 + [P] * 5 + [I]
        lib.or_forward.restype = I
        lib.or_reference_render.argtypes = [P] * 7 + [L, P, I, I, D, D] + [P] * 4 + [I]
        lib.or_reference_render.restype = I
        lib.or_backward.argtypes = ([P] * 7 + [L, P, P] + [I] * 6 + [D] * 3 + [P] * 4
                                    + [P] * 6 + [I])
        lib.or_backward.restype = I
        lib.or_eikonal.argtypes = [P, P, P, P, L, D, P, P]
        lib.or_eikonal.restype = D
        lib.or_normal_consistency.argtypes = [P, P, L, P, L, P, L, D, P, P]
        lib.or_normal_consistency.restype = D
        _LIB = lib
    return _LIB


def available_backends():
    out = []
    if _load_ref() is not None:
        out.append("ref")
    if _load_c() is not None:
        out.append("c")
    return out


def default_backend():
    b = available_backends()
    if not b:
        raise RuntimeError("no oracle kernel backend built: run `make -C oracle` "
                           "(and `make -C oracle ref` where /root/reference exists)")
    return b[0]


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def n_threads():
    env = os.environ.get("TETSPLAT_THREADS")
    if env:
        return max(1, int(env))
    return os.cpu_count() or 1


# --- grid (grid.py:21-117) ---------------------------------------------------------

@dataclass(frozen=True)
class TetrahedralGrid:
    rest_positions: np.ndarray
    tets: np.ndarray
    edges: np.ndarray
    resolution: int

    @property
    def num_vertices(self):
        return len(self.rest_positions)

    @property
    def num_tets(self):
        return len(self.tets)

    @property
    def cell_edge(self):
        return 2.0 / self.resolution


def grid_axis(R):
    """np.linspace(-1, 1, R+1) (grid.py:71): i*(2/R) + (-1), last = 1."""
    return np.linspace(-1.0, 1.0, R + 1)


def build_grid(R: int, with_edges: bool = True) -> TetrahedralGrid:
    """Kuhn 6-tet grid (grid.py:64-117).  Vertex id x + n*y + n^2*z; tet id
    cell*6 + p with cell = ix*R^2 + iy*R + iz; negative-volume tets swap v2/v3.
    `with_edges=False` skips the sorted edge list (only normal consistency reads it; at
    R=256 its lexsort is most of the 130 s build)."""
    if R < 1:
        raise ValueError("resolution must be >= 1")
    n = R + 1
    ax = grid_axis(R)
    zz, yy, xx = np.meshgrid(ax, ax, ax, indexing="ij")
    pos = np.stack([xx.ravel(), yy.ravel(), zz.ravel()], axis=1)
    ix, iy, iz = np.meshgrid(np.arange(R), np.arange(R), np.arange(R), indexing="ij")
    base = np.stack([ix.ravel(), iy.ravel(), iz.ravel()], axis=1)
    per = []
    for p in _AXIS_PERMS:
        c = np.zeros((4, 3), dtype=np.int64)
        c[1, p[0]] = 1
        c[2] = c[1]
        c[2, p[1]] = 1
        c[3] = 1
        ids = base[:, None, :] + c[None]
        per.append(ids[..., 0] + n * ids[..., 1] + n * n * ids[..., 2])
    tets = np.stack(per, axis=1).reshape(-1, 4)
    a = pos[tets[:, 0]]
    vol = np.einsum("ij,ij->i", np.cross(pos[tets[:, 1]] - a, pos[tets[:, 2]] - a),
                    pos[tets[:, 3]] - a)
    flip = vol < 0
    tets[flip] = tets[flip][:, [0, 1, 3, 2]]
    if not with_edges:
        return TetrahedralGrid(pos, tets, np.zeros((0, 2), np.int64), R)
    g = np.arange(n)
    gx, gy, gz = np.meshgrid(g, g, g, indexing="ij")
    el = []
    for ox, oy, oz in [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (0, 1, 1), (1, 0, 1), (1, 1, 1)]:
        m = (gx + ox < n) & (gy + oy < n) & (gz + oz < n)
        el.append(np.stack([gx[m] + n * gy[m] + n * n * gz[m],
                            gx[m] + ox + n * (gy[m] + oy) + n * n * (gz[m] + oz)], axis=1))
    edges = np.concatenate(el)
    edges = edges[np.lexsort((edges[:, 1], edges[:, 0]))]
    return TetrahedralGrid(pos, tets, edges, R)


# --- field (field.py:22-177) -------------------------------------------------------

@dataclass
class FieldState:
    sdf: np.ndarray
    deformation: np.ndarray
    deform_limit: float
    steepness: float | None = None

    def __post_init__(self):
        self.sdf = np.asarray(self.sdf, dtype=np.float64)
        self.deformation = np.asarray(self.deformation, dtype=np.float64)
        np.clip(self.deformation, -self.deform_limit, self.deform_limit, out=self.deformation)

    def deformed_positions(self, grid):
        return grid.rest_positions + self.deformation


def init_sphere_field(grid, radius=0.5):
    """field.py:64-67 with AnalyticShape('sphere', (r,)): |p| - r, zero deformation."""
    sdf = np.linalg.norm(grid.rest_positions, axis=-1) - radius
    return FieldState(sdf, np.zeros_like(grid.rest_positions), DEFORM_FRACTION * grid.cell_edge)


def noisy_field(grid, radius=0.5, noise=0.08, deform=0.4, seed=0):
    """The gradcheck-style perturbed field (gradcheck.py:32-45): sdf + noise*N(0,1),
    deformation ~ U(+-deform*limit)."""
    rng = np.random.default_rng(seed)
    f = init_sphere_field(grid, radius)
    f.sdf = f.sdf + noise * rng.normal(size=f.sdf.shape)
    lim = f.deform_limit
    f.deformation = rng.uniform(-deform * lim, deform * lim, size=f.deformation.shape)
    return FieldState(f.sdf, f.deformation, lim)


def tet_sdf_gradients(positions, f):
    """field.py:140-150: solve [v 1] x = f per tet, gradient = x[:3]."""
    K = len(positions)
    B = np.concatenate([positions, np.ones((K, 4, 1))], axis=2)
    return np.linalg.solve(B, f[..., None])[..., 0][:, :3]


def tet_normals(g):
    """field.py:171-177."""
    nrm = np.linalg.norm(g, axis=1)
    ok = nrm >= EPS_NORMAL
    out = np.zeros_like(g)
    out[ok] = g[ok] / nrm[ok, None]
    return out, ok


# --- camera (camera.py:13-139) -----------------------------------------------------

@dataclass(frozen=True)
class Camera:
    width: int
    height: int
    fy: float
    rotation: np.ndarray
    translation: np.ndarray
    near: float
    far: float

    @property
    def fx(self):
        return self.fy

    @property
    def cx(self):
        return self.width / 2.0

    @property
    def cy(self):
        return self.height / 2.0

    def to_camera(self, pts):
        return np.atleast_2d(pts) @ self.rotation.T + self.translation

    def project_points(self, pts):
        """camera.py:59-67."""
        pc = self.to_camera(pts)
        z = pc[:, 2]
        zs = np.where(z > 1e-12, z, 1e-12)
        pix = np.stack([self.fx * pc[:, 0] / zs + self.cx, self.fy * pc[:, 1] / zs + self.cy], axis=1)
        return pix, z, z <= self.near


def look_at(position, target=(0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0)):
    """camera.py:105-117."""
    position = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - position
    fwd = fwd / np.linalg.norm(fwd)
    up = np.asarray(up, dtype=np.float64)
    if abs(np.dot(fwd, up)) > 1 - 1e-9:
        up = np.array([0.0, 1.0, 0.0])
    right = np.cross(fwd, up)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    return R, -R @ position


def orbit_camera(index, count, radius=3.0, elevation_range=(-30.0, 30.0), fov_deg=40.0,
                 width=256, height=256, near=0.1, far=10.0):
    """camera.py:120-139."""
    az = 2 * math.pi * (index % count) / count
    lo, hi = elevation_range
    el = math.radians(lo + ((index * _GOLDEN) % 1.0) * (hi - lo))
    pos = radius * np.array([math.cos(el) * math.cos(az), math.cos(el) * math.sin(az), math.sin(el)])
    R, t = look_at(pos)
    fy = 0.5 * height / math.tan(math.radians(fov_deg) / 2)
    return Camera(width, height, fy, R, t, near, far)


# --- splat (splat.py:26-245) -------------------------------------------------------

def _softplus(x):
    x = np.asarray(x, dtype=np.float64)
    return np.where(x > 30, x, np.log1p(np.exp(np.minimum(x, 30))))


def alpha_max(f, s):
    """splat.py:42-55."""
    f = np.atleast_2d(np.asarray(f, dtype=np.float64))
    a = s * f.max(axis=1)
    b = s * f.min(axis=1)
    return np.maximum(1.0 - np.exp(_softplus(-a) - _softplus(-b)), 0.0)


def prefilter(grid, field, s, threshold=T_FILTER):
    """splat.py:66-69."""
    return np.nonzero(alpha_max(field.sdf[grid.tets], s) >= threshold)[0]


@dataclass
class SplatScene:
    tet_ids: np.ndarray
    vert_ids: np.ndarray
    proj: np.ndarray
    depths: np.ndarray
    f: np.ndarray
    normals: np.ndarray
    mean_depth: np.ndarray
    alpha_max: np.ndarray
    bbox: np.ndarray
    steepness: float = 1.0
    colors: np.ndarray | None = None

    def __len__(self):
        return len(self.tet_ids)


def build_scene(grid, field, camera, s, active=None, colors=None, threshold=T_FILTER):
    """splat.py:203-245."""
    if active is None:
        active = prefilter(grid, field, s, threshold)
    active = np.asarray(active, dtype=np.int64)
    pos = field.deformed_positions(grid)
    pix, z, _ = camera.project_points(pos)
    tets = grid.tets[active]
    proj = pix[tets]
    depths = z[tets]
    dmin = depths.min(axis=1)
    keep = (dmin > camera.near) & (dmin <= camera.far)
    xmin, xmax = proj[..., 0].min(axis=1), proj[..., 0].max(axis=1)
    ymin, ymax = proj[..., 1].min(axis=1), proj[..., 1].max(axis=1)
    keep &= (xmax >= 0) & (xmin <= camera.width) & (ymax >= 0) & (ymin <= camera.height)
    active = active[keep]
    tets = tets[keep]
    proj = np.ascontiguousarray(proj[keep])
    depths = np.ascontiguousarray(depths[keep])
    f = np.ascontiguousarray(field.sdf[tets])
    g = tet_sdf_gradients(pos[tets], f) if len(tets) else np.zeros((0, 3))
    normals, _ = tet_normals(g)
    bbox = np.stack([xmin[keep], ymin[keep], xmax[keep], ymax[keep]], axis=1)
    return SplatScene(active, tets, proj, depths, f, normals, depths.mean(axis=1),
                      alpha_max(f, s) if len(tets) else np.zeros(0), np.ascontiguousarray(bbox),
                      float(s), None if colors is None else np.ascontiguousarray(colors[active]))


# --- raster (raster.py:53-306) -----------------------------------------------------

@dataclass
class TileBins:
    tile_size: int
    tiles_x: int
    tiles_y: int
    starts: np.ndarray
    items: np.ndarray

    @property
    def num_tiles(self):
        return self.tiles_x * self.tiles_y


@dataclass
class RenderMaps:
    normal: np.ndarray
    depth: np.ndarray
    opacity: np.ndarray
    color: np.ndarray | None = None

    @classmethod
    def zeros(cls, h, w, with_color=False):
        return cls(np.zeros((h, w, 3)), np.zeros((h, w)), np.zeros((h, w)),
                   np.zeros((h, w, 3)) if with_color else None)


@dataclass
class GradientBuffers:
    d_sdf: np.ndarray
    d_deform: np.ndarray
    d_color: np.ndarray | None = None


@dataclass
class SavedState:
    bins: TileBins
    n_w: int
    t_stop: float
    records: list | None = None  # "ref" backend only (raster.py:94-101)
    counts: np.ndarray | None = None  # per-pixel blended-record count


def tile_rects(bbox, tiles_x, tiles_y, tile_size=TILE_SIZE):
    """raster.py:118-121."""
    tx0 = np.clip(np.floor(bbox[:, 0] / tile_size), 0, tiles_x - 1).astype(np.int64)
    tx1 = np.clip(np.floor(bbox[:, 2] / tile_size), 0, tiles_x - 1).astype(np.int64)
    ty0 = np.clip(np.floor(bbox[:, 1] / tile_size), 0, tiles_y - 1).astype(np.int64)
    ty1 = np.clip(np.floor(bbox[:, 3] / tile_size), 0, tiles_y - 1).astype(np.int64)
    return tx0, tx1, ty0, ty1


def depth_keys(mean_depth, near, far):
    """raster.py:132-134: 32-bit fixed-point mean depth over [near, far]."""
    q = np.clip((mean_depth - near) / (far - near), 0.0, 1.0)
    return (q * (2 ** 32 - 1)).astype(np.uint64)


def bin_and_sort(scene, camera, tile_size=TILE_SIZE):
    """raster.py:104-141: duplicate splats into overlapped tiles, stable sort by
    (tile << 32 | q), searchsorted tile starts."""
    tiles_x = (camera.width + tile_size - 1) // tile_size
    tiles_y = (camera.height + tile_size - 1) // tile_size
    K = len(scene)
    if K == 0:
        return TileBins(tile_size, tiles_x, tiles_y, np.zeros(tiles_x * tiles_y + 1, np.int64),
                        np.zeros(0, np.int64))
    tx0, tx1, ty0, ty1 = tile_rects(scene.bbox, tiles_x, tiles_y, tile_size)
    nx = tx1 - tx0 + 1
    counts = nx * (ty1 - ty0 + 1)
    sid = np.repeat(np.arange(K, dtype=np.int64), counts)
    off = np.concatenate([[0], np.cumsum(counts)[:-1]])
    local = np.arange(counts.sum(), dtype=np.int64) - off[sid]
    tile = (ty0[sid] + local // nx[sid]) * tiles_x + tx0[sid] + local % nx[sid]
    q = depth_keys(scene.mean_depth, camera.near, camera.far)
    key = (tile.astype(np.uint64) << np.uint64(32)) | q[sid]
    order = np.argsort(key, kind="stable")
    starts = np.searchsorted(tile[order], np.arange(tiles_x * tiles_y + 1))
    return TileBins(tile_size, tiles_x, tiles_y, starts.astype(np.int64), sid[order])


def _scene_args(scene):
    c = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    return (c(scene.proj), c(scene.depths), c(scene.f), c(scene.normals), c(scene.mean_depth),
            None if scene.colors is None else c(scene.colors), c(scene.bbox))


def render_forward(scene, bins, camera, n_w=DEFAULT_WINDOW, t_stop=T_STOP, save_state=False,
                   backend=None, want_counts=False):
    """raster.py:149-177."""
    if n_w < 1:
        raise ValueError("resorting window must be >= 1")
    backend = backend or default_backend()
    H, W = camera.height, camera.width
    maps = RenderMaps.zeros(H, W, scene.colors is not None)
    args = _scene_args(scene)
    s = float(scene.steepness)
    records = None
    counts = None
    if backend == "ref":
        touched = np.nonzero(np.diff(bins.starts) > 0)[0]
        core = _load_ref()

        def run(tids):  # raster.py:164-175: chunked tiles over a thread pool (GIL released)
            return core.forward_tiles(
                *args, bins.starts, bins.items, tids, bins.tile_size, bins.tiles_x, W, H, n_w, s,
                t_stop, ALPHA_CLIP, maps.normal, maps.depth, maps.opacity, maps.color,
                bool(save_state or want_counts))

        nt = n_threads()
        if nt <= 1 or len(touched) < 2:
            records = run(touched)
        else:
            from concurrent.futures import ThreadPoolExecutor
            records = []
            with ThreadPoolExecutor(max_workers=nt) as pool:
                for part in pool.map(run, np.array_split(touched, min(nt * 4, len(touched)))):
                    records.extend(part)
        if want_counts:
            counts = np.zeros((H, W), np.int32)
            ts = bins.tile_size
            for tid, cnt, _, _ in records:
                x0, y0 = (tid % bins.tiles_x) * ts, (tid // bins.tiles_x) * ts
                c2 = cnt.reshape(ts, ts)
                h, w = min(ts, H - y0), min(ts, W - x0)
                counts[y0:y0 + h, x0:x0 + w] = c2[:h, :w]
    else:
        counts = np.zeros((H, W), np.int32) if want_counts else None
        rc = _load_c().or_forward(*[_ptr(a) for a in args], _ptr(bins.starts), _ptr(bins.items),
                                  bins.tile_size, bins.tiles_x, bins.tiles_y, W, H, n_w, s, t_stop,
                                  ALPHA_CLIP, _ptr(maps.normal), _ptr(maps.depth),
                                  _ptr(maps.opacity), _ptr(maps.color), _ptr(counts), n_threads())
        assert rc == 0
    saved = SavedState(bins, n_w, t_stop, records if save_state else None, counts) \
        if (save_state or want_counts) else None
    return maps, saved


def render_reference(scene, camera, backend=None):
    """raster.py:180-199 (exact mean-depth order, no tiles/window/early stop)."""
    backend = backend or default_backend()
    H, W = camera.height, camera.width
    maps = RenderMaps.zeros(H, W, scene.colors is not None)
    args = _scene_args(scene)
    if backend == "ref":
        _load_ref().reference_render(*args, W, H, float(scene.steepness), ALPHA_CLIP, 0, H,
                                     maps.normal, maps.depth, maps.opacity, maps.color)
    else:
        K = len(scene)
        order = np.lexsort((np.arange(K), scene.mean_depth)).astype(np.int64)
        _load_c().or_reference_render(*[_ptr(a) for a in args], K, _ptr(order), W, H,
                                      float(scene.steepness), ALPHA_CLIP, _ptr(maps.normal),
                                      _ptr(maps.depth), _ptr(maps.opacity), _ptr(maps.color),
                                      n_threads())
    return maps


def splat_gradients(saved, scene, camera, d_maps, backend=None):
    """backward_tiles + ordered merge (raster.py:206-247): per-splat gradients."""
    for arr in (d_maps.normal, d_maps.depth, d_maps.opacity):
        if not np.all(np.isfinite(arr)):
            raise ValueError("non-finite incoming map gradients")
    backend = backend or default_backend()
    K = len(scene)
    with_color = scene.colors is not None and d_maps.color is not None
    d = dict(d_f=np.zeros((K, 4)), d_proj=np.zeros((K, 4, 2)), d_depths=np.zeros((K, 4)),
             d_normals=np.zeros((K, 3)), d_mean_depth=np.zeros(K),
             d_colors=np.zeros((K, 3)) if with_color else None)
    args = _scene_args(scene)
    c = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)
    dm = (c(d_maps.normal), c(d_maps.depth), c(d_maps.opacity),
          c(d_maps.color) if with_color else None)
    H, W = camera.height, camera.width
    s = float(scene.steepness)
    b = saved.bins
    if backend == "ref":
        records = saved.records
        if records is None:
            raise ValueError("ref backend needs save_state=True records")
        core = _load_ref()

        def run(recs):  # raster.py:214-247: private per-chunk buffers, ordered merge
            p = {k: (None if v is None else np.zeros_like(v)) for k, v in d.items()}
            core.backward_tiles(*args, recs, b.tile_size, b.tiles_x, W, H, s, ALPHA_CLIP, *dm, p["d_f"],
                                p["d_proj"], p["d_depths"], p["d_normals"], p["d_mean_depth"], p["d_colors"])
            return p

        nt = n_threads()
        if nt <= 1 or len(records) < 2:
            parts = [run(records)]
        else:
            from concurrent.futures import ThreadPoolExecutor
            chunks = [c for c in np.array_split(np.arange(len(records)), nt) if len(c)]
            with ThreadPoolExecutor(max_workers=nt) as pool:
                parts = list(pool.map(lambda c: run([records[i] for i in c]), chunks))
        for k in d:
            if d[k] is not None:
                d[k] = sum(p[k] for p in parts)
    else:
        rc = _load_c().or_backward(*[_ptr(a) for a in args], K, _ptr(b.starts), _ptr(b.items),
                                   b.tile_size, b.tiles_x, b.tiles_y, W, H, saved.n_w, s,
                                   saved.t_stop, ALPHA_CLIP, *[_ptr(a) for a in dm],
                                   _ptr(d["d_f"]), _ptr(d["d_proj"]), _ptr(d["d_depths"]),
                                   _ptr(d["d_normals"]), _ptr(d["d_mean_depth"]),
                                   _ptr(d["d_colors"]), n_threads())
        assert rc == 0
    return d


def render_backward(saved, scene, grid, field, camera, d_maps, backend=None):
    """raster.py:206-250."""
    d = splat_gradients(saved, scene, camera, d_maps, backend)
    return splat_grads_to_vertices(scene, grid, field, camera, d["d_f"], d["d_proj"],
                                   d["d_depths"], d["d_normals"], d["d_mean_depth"], d["d_colors"])


def splat_grads_to_vertices(scene, grid, field, camera, d_f, d_proj, d_depths, d_normals,
                            d_mean_depth, d_colors=None):
    """raster.py:253-306: normal chain through the 4x4 solve, camera chain, scatter."""
    N = grid.num_vertices
    out = GradientBuffers(np.zeros(N), np.zeros((N, 3)))
    K = len(scene)
    if K == 0:
        return out
    pos = field.deformed_positions(grid)
    verts = scene.vert_ids
    d_f = d_f.copy()
    d_depths = d_depths + d_mean_depth[:, None] / 4.0
    d_pos = np.zeros((K, 4, 3))
    tp = pos[verts]
    g = tet_sdf_gradients(tp, scene.f)
    gn = np.linalg.norm(g, axis=1)
    ok = gn >= EPS_NORMAL
    if ok.any():
        n = np.zeros_like(g)
        n[ok] = g[ok] / gn[ok, None]
        d_g = np.zeros_like(g)
        dn = d_normals[ok]
        d_g[ok] = (dn - n[ok] * np.einsum("ij,ij->i", n[ok], dn)[:, None]) / gn[ok, None]
        B = np.concatenate([tp, np.ones((K, 4, 1))], axis=2)
        rhs = np.concatenate([d_g, np.zeros((K, 1))], axis=1)
        dfn = np.linalg.solve(np.transpose(B, (0, 2, 1)), rhs[..., None])[..., 0]
        d_f += dfn
        d_pos -= dfn[..., None] * g[:, None, :]
    pc = camera.to_camera(pos)[verts]
    X, Y, Z = pc[..., 0], pc[..., 1], pc[..., 2]
    dpx, dpy = d_proj[..., 0], d_proj[..., 1]
    d_pc = np.stack([dpx * camera.fx / Z, dpy * camera.fy / Z,
                     -dpx * camera.fx * X / Z ** 2 - dpy * camera.fy * Y / Z ** 2 + d_depths], axis=-1)
    d_pos += d_pc @ camera.rotation
    np.add.at(out.d_sdf, verts, d_f)
    np.add.at(out.d_deform, verts, d_pos)
    if d_colors is not None:
        out.d_color = np.zeros((grid.num_tets, 3))
        np.add.at(out.d_color, scene.tet_ids, d_colors)
    return out


# --- losses (losses.py:25-52) ------------------------------------------------------

def eikonal_loss(grid, field, tet_set, backend=None):
    backend = backend or default_backend()
    N = grid.num_vertices
    out = GradientBuffers(np.zeros(N), np.zeros((N, 3)))
    tet_set = np.ascontiguousarray(tet_set, dtype=np.int64)
    if len(tet_set) == 0:
        return 0.0, out
    pos = np.ascontiguousarray(field.deformed_positions(grid))
    sdf = np.ascontiguousarray(field.sdf)
    tets = np.ascontiguousarray(grid.tets, dtype=np.int64)
    if backend == "ref":
        loss = _load_ref().eikonal_kernel(pos, sdf, tets, tet_set, EPS_NORMAL, out.d_sdf, out.d_deform)
    else:
        loss = _load_c().or_eikonal(_ptr(pos), _ptr(sdf), _ptr(tets), _ptr(tet_set), len(tet_set),
                                    EPS_NORMAL, _ptr(out.d_sdf), _ptr(out.d_deform))
    return float(loss), out


def normal_consistency_loss(grid, field, backend=None):
    backend = backend or default_backend()
    N = grid.num_vertices
    out = GradientBuffers(np.zeros(N), np.zeros((N, 3)))
    pos = np.ascontiguousarray(field.deformed_positions(grid))
    sdf = np.ascontiguousarray(field.sdf)
    tets = np.ascontiguousarray(grid.tets, dtype=np.int64)
    edges = np.ascontiguousarray(grid.edges, dtype=np.int64)
    if backend == "ref":
        loss = _load_ref().normal_consistency_kernel(pos, sdf, tets, edges, EPS_NORMAL,
                                                     out.d_sdf, out.d_deform)
    else:
        loss = _load_c().or_normal_consistency(_ptr(pos), _ptr(sdf), N, _ptr(tets), len(tets),
                                               _ptr(edges), len(edges), EPS_NORMAL,
                                               _ptr(out.d_sdf), _ptr(out.d_deform))
    return float(loss), out


# --- marching tetrahedra (grid.py:120-239) -----------------------------------------

def _edge_crossings(pos, f, va, vb):
    fa = f[va][:, None]
    fb = f[vb][:, None]
    p = (fb * pos[va] - fa * pos[vb]) / (fb - fa)
    az, bz = (fa == 0)[:, 0], (fb == 0)[:, 0]
    p[az] = pos[va[az]]
    p[bz] = pos[vb[bz]]
    return p


def marching_tetrahedra(grid, field):
    """grid.py:136-239.  Returns (vertices (V,3) f64, triangles (F,3) i64)."""
    pos = field.deformed_positions(grid)
    f = np.asarray(field.sdf, dtype=np.float64)
    neg = f[grid.tets] < 0
    ncount = neg.sum(axis=1)
    cross, singles, quad, off = [], [], None, 0
    for count, lone_neg in ((1, True), (3, False)):
        sel = np.nonzero(ncount == count)[0]
        if len(sel) == 0:
            continue
        tt = grid.tets[sel]
        lone = neg[sel] if lone_neg else ~neg[sel]
        m = np.argmax(lone, axis=1)
        others = np.argsort(lone, axis=1, kind="stable")[:, :3]
        r = np.arange(len(sel))
        va = tt[r, m]
        for j in range(3):
            cross.append(np.sort(np.stack([va, tt[r, others[:, j]]], axis=1), axis=1))
        singles.append((off, len(sel), sel))
        off += 3 * len(sel)
    sel = np.nonzero(ncount == 2)[0]
    if len(sel):
        tt = grid.tets[sel]
        order = np.argsort(~neg[sel], axis=1, kind="stable")
        r = np.arange(len(sel))
        i_, j_, k_, l_ = (tt[r, order[:, c]] for c in range(4))
        for a, b in ((i_, k_), (i_, l_), (j_, l_), (j_, k_)):
            cross.append(np.sort(np.stack([a, b], axis=1), axis=1))
        quad = (off, len(sel), sel)
        off += 4 * len(sel)
    if off == 0:
        return np.zeros((0, 3)), np.zeros((0, 3), np.int64)
    cross = np.concatenate(cross)
    uniq, inv = np.unique(cross, axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    verts = _edge_crossings(pos, f, uniq[:, 0], uniq[:, 1])
    tris, tot = [], []
    for start, n1, st in singles:
        i = start + np.arange(n1)
        tris.append(np.stack([inv[i], inv[i + n1], inv[i + 2 * n1]], axis=1))
        tot.append(st)
    if quad is not None:
        start, nq, sq = quad
        i = start + np.arange(nq)
        ik, il, jl, jk = i, i + nq, i + 2 * nq, i + 3 * nq
        d1 = np.linalg.norm(verts[inv[ik]] - verts[inv[jl]], axis=1)
        d2 = np.linalg.norm(verts[inv[il]] - verts[inv[jk]], axis=1)
        k1 = np.minimum(cross[ik][:, 0], cross[jl][:, 0])
        k2 = np.minimum(cross[il][:, 0], cross[jk][:, 0])
        use1 = np.where(np.isclose(d1, d2), k1 <= k2, d1 < d2)
        t1 = np.where(use1[:, None], np.stack([inv[ik], inv[il], inv[jl]], axis=1),
                      np.stack([inv[ik], inv[il], inv[jk]], axis=1))
        t2 = np.where(use1[:, None], np.stack([inv[ik], inv[jl], inv[jk]], axis=1),
                      np.stack([inv[il], inv[jl], inv[jk]], axis=1))
        tris += [t1, t2]
        tot += [sq, sq]
    tris = np.concatenate(tris)
    tot = np.concatenate(tot)
    g = tet_sdf_gradients(pos[grid.tets[tot]], f[grid.tets[tot]])
    a = verts[tris[:, 0]]
    ntri = np.cross(verts[tris[:, 1]] - a, verts[tris[:, 2]] - a)
    flip = np.einsum("ij,ij->i", ntri, g) < 0
    tris[flip] = tris[flip][:, [0, 2, 1]]
    upos, remap = np.unique(verts, axis=0, return_inverse=True)
    tris = remap.reshape(-1)[tris]
    distinct = (tris[:, 0] != tris[:, 1]) & (tris[:, 1] != tris[:, 2]) & (tris[:, 0] != tris[:, 2])
    a = upos[tris[:, 0]]
    area2 = np.linalg.norm(np.cross(upos[tris[:, 1]] - a, upos[tris[:, 2]] - a), axis=1)
    return upos, tris[distinct & (area2 > 1e-14)].astype(np.int64)


# --- synthetic workload ----------------------------------------------

def synthetic_dmaps(H, W, seed=1, with_color=False):
    """dL/dmaps ~ N(0,1) with default_rng(seed), shapes (H,W,3),(H,W),(H,W) (gradcheck.py:88-93)."""
    rng = np.random.default_rng(seed)
    n = rng.normal(size=(H, W, 3))
    d = rng.normal(size=(H, W))
    o = rng.normal(size=(H, W))
    c = rng.normal(size=(H, W, 3)) if with_color else None
    return RenderMaps(n, d, o, c)
