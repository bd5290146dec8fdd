"""Golden fixtures for the fit-loop layer from the UNMODIFIED reference.

    python tests/golden/make_golden_fit.py /tmp/tsref/src      (see make_golden.py)

Writes fit.npz (sphere-traced target maps (fit.py:93-133) for two shapes / cameras, and the
trace of a 3-iteration fit_field run on a tiny configuration, fit.py:144-231) and
meshraster.npz (rasterize_mesh of a Marching-Tetrahedra torus, mesh.py:98-147) and
formats.npz (PFM / TSPF bytes written by the reference).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main(ref_src: str):
    sys.path.insert(0, ref_src)
    import tetsplat
    from tetsplat import camera, field, fit, grid
    assert tetsplat.BACKEND_NAME == "compiled", "build the reference's Cython kernels first"
    out = {}
    shapes = {"sphere": field.AnalyticShape("sphere", (0.6,)), "torus": field.AnalyticShape("torus", (0.45, 0.15))}
    for i, (name, shp) in enumerate(shapes.items()):
        cam = camera.orbit_camera(1 + i, 8, width=48, height=48)
        t = fit.render_target(shp, cam)
        out[f"target_{name}_normal"], out[f"target_{name}_depth"] = t.normal, t.depth
        out[f"target_{name}_opacity"] = t.opacity
    cfg = fit.FitConfig(resolution=8, image_size=32, n_views=4, batch_size=2, iterations=3, trace_every=1)
    g = grid.build_grid(cfg.resolution)
    f = field.init_from_shape(g, field.AnalyticShape("sphere", (0.5,)))
    cams, targets = fit.make_targets(field.AnalyticShape("sphere", (0.6,)), cfg)
    tr = fit.fit_field(g, f, cams, targets, cfg)
    out["fit_trace"] = np.array(json.dumps(tr.iterations))
    out["fit_final_sdf"] = f.sdf
    out["fit_final_deform"] = f.deformation
    np.savez_compressed(os.path.join(HERE, "fit.npz"), **out)

    # z-buffered mesh rasterization (mesh.py:98-147) of a Marching-Tetrahedra mesh
    from tetsplat import mesh as rmesh
    g = grid.build_grid(12)
    f = field.init_from_shape(g, field.AnalyticShape("torus", (0.45, 0.2)))
    m = grid.marching_tetrahedra(g, f)
    cam = camera.orbit_camera(2, 8, width=64, height=64)
    mask, depth, normal = rmesh.rasterize_mesh(m, cam)
    np.savez_compressed(os.path.join(HERE, "meshraster.npz"), vertices=m.vertices, triangles=m.triangles,
                        cam_index=2, cam_count=8, size=64, mask=mask, depth=depth, normal=normal)
    print("mesh", m.vertices.shape, m.triangles.shape, int(mask.sum()))

    # byte formats (imgio.py:18-48, field.py:180-203)
    import tempfile
    from tetsplat import imgio
    rng = np.random.default_rng(7)
    a1, a3 = rng.standard_normal((3, 5)), rng.standard_normal((3, 5, 3))
    st = field.FieldState(rng.standard_normal(6), 0.01 * rng.standard_normal((6, 3)), 0.05, 42.5)
    blobs = {}
    with tempfile.TemporaryDirectory() as d:
        for name, fn in (("pfm1", lambda p: imgio.write_pfm(p, a1)), ("pfm3", lambda p: imgio.write_pfm(p, a3)),
                         ("tspf", lambda p: field.save_checkpoint(st, p))):
            fn(os.path.join(d, name))
            blobs[name] = np.frombuffer(open(os.path.join(d, name), "rb").read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "formats.npz"), a1=a1, a3=a3, sdf=st.sdf, deform=st.deformation,
                        s=st.steepness, limit=0.05, **blobs)
    print(json.dumps(tr.iterations, indent=1)[:2000])


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "/tmp/tsref/src")
