"""Generate the golden fixtures from the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):
    cp -r /root/reference/pkg /tmp/tsref && (cd /tmp/tsref && python setup.py build_ext --inplace)
    python tests/golden/make_golden.py /tmp/tsref/src [--color-window]

It imports `tetsplat` (the reference) and writes small .npz fixtures next to this file.
These pin the CPU oracle (oracle/ts_oracle.py) and the GPU path; nothing at test time
reads /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main(ref_src: str):
    sys.path.insert(0, ref_src)
    import tetsplat
    from tetsplat import camera, field, grid, losses, raster, splat
    assert tetsplat.BACKEND_NAME == "compiled", "build the reference's Cython kernels first"

    # --- grid connectivity (grid.py:64-117) ------------------------------------------------
    for R in (1, 2, 3):
        g = grid.build_grid(R)
        np.savez_compressed(os.path.join(HERE, f"grid_R{R}.npz"), rest=g.rest_positions, tets=g.tets,
                            edges=g.edges)

    # --- render / backward / regularizers at small configs ---------------------------------
    cases = {
        # name: (R, image, s, camera index, count, perturbed field)
        "sphere_r16_s100": (16, 128, 100.0, 0, 8, False),
        "noisy_r16_s20": (16, 128, 20.0, 3, 8, True),
        "noisy_r12_s100_cam5": (12, 96, 100.0, 5, 8, True),
        "sphere_r32_s100_cfg1": (32, 256, 100.0, 0, 8, False),
    }
    for name, (R, S, s, ci, cc, noisy) in cases.items():
        g = grid.build_grid(R)
        if noisy:
            rng = np.random.default_rng(0)
            fs = field.init_sphere(g, 0.5)
            sdf = fs.sdf + 0.08 * rng.normal(size=fs.sdf.shape)
            lim = fs.deform_limit
            deform = rng.uniform(-0.4 * lim, 0.4 * lim, size=fs.deformation.shape)
            fs = field.FieldState(sdf, deform, lim)
        else:
            fs = field.init_from_shape(g, field.AnalyticShape("sphere", (0.5,)))
        cam = camera.orbit_camera(ci, cc, width=S, height=S)
        active = splat.prefilter(g, fs, s)
        sc = splat.build_scene(g, fs, cam, s, active=active)
        bins = raster.bin_and_sort(sc, cam)
        maps, saved = raster.render_forward(sc, bins, cam, n_w=5, save_state=True)
        counts = np.zeros((S, S), np.int32)
        for tid, cnt, _, _ in saved.records:
            x0, y0 = (tid % bins.tiles_x) * 16, (tid // bins.tiles_x) * 16
            c2 = cnt.reshape(16, 16)
            h, w = min(16, S - y0), min(16, S - x0)
            counts[y0:y0 + h, x0:x0 + w] = c2[:h, :w]
        ref_maps = raster.render_reference(sc, cam)
        rng = np.random.default_rng(1)
        dm = raster.RenderMaps(rng.normal(size=(S, S, 3)), rng.normal(size=(S, S)), rng.normal(size=(S, S)))
        gb = raster.render_backward(saved, sc, g, fs, cam, dm)
        le, ge = losses.eikonal_loss(g, fs, active)
        ln, gn = losses.normal_consistency_loss(g, fs)
        big = R >= 32
        fp = np.float32 if big else np.float64
        out = dict(R=R, S=S, s=s, cam_index=ci, cam_count=cc, noisy=noisy, sdf=fs.sdf, deform=fs.deformation,
                   active=active, tet_ids=sc.tet_ids, vert_ids=sc.vert_ids, proj=sc.proj, depths=sc.depths,
                   f=sc.f, normals=sc.normals, mean_depth=sc.mean_depth, alpha_max=sc.alpha_max, bbox=sc.bbox,
                   starts=bins.starts, items=bins.items, counts=counts,
                   normal=maps.normal.astype(fp), depth=maps.depth.astype(fp), opacity=maps.opacity.astype(fp),
                   ref_normal=ref_maps.normal.astype(fp), ref_depth=ref_maps.depth.astype(fp),
                   ref_opacity=ref_maps.opacity.astype(fp),
                   d_normal=dm.normal, d_depth=dm.depth, d_opacity=dm.opacity,
                   d_sdf=gb.d_sdf, d_deform=gb.d_deform, eik_loss=le, eik_d_sdf=ge.d_sdf, eik_d_deform=ge.d_deform,
                   nc_loss=ln, nc_d_sdf=gn.d_sdf, nc_d_deform=gn.d_deform)
        if big:  # keep the fixture small: drop what the tests recompute from the inputs
            for k in ("proj", "depths", "f", "normals", "alpha_max", "vert_ids", "d_normal", "d_depth",
                      "d_opacity", "ref_normal", "ref_depth", "ref_opacity"):
                out.pop(k)
        np.savez_compressed(os.path.join(HERE, f"render_{name}.npz"), **out)
        print(name, "K=", len(sc), "M=", len(bins.items), "blends=", int(counts.sum()))

    # --- marching tetrahedra (grid.py:136-239) ---------------------------------------------
    mt = {}
    g1 = grid.build_grid(1)
    for tag, fv in (("one_neg", (-1.0, 1.0, 1.0, 1.0)), ("two_neg", (-1.0, -1.0, 1.0, 1.0))):
        # SPEC.md:51-53 single-tet examples on tet 0 of a 1-cell grid
        sdf = np.ones(g1.num_vertices)
        sdf[g1.tets[0]] = fv
        fs = field.FieldState(sdf, np.zeros((g1.num_vertices, 3)), field.deform_limit_for(g1))
        m = grid.marching_tetrahedra(g1, fs)
        mt[f"{tag}_sdf"] = sdf
        mt[f"{tag}_V"] = m.vertices
        mt[f"{tag}_F"] = m.triangles
    for R, noisy in ((16, False), (16, True), (24, False)):
        g = grid.build_grid(R)
        fs = field.init_from_shape(g, field.AnalyticShape("sphere", (0.5,)))
        if noisy:
            rng = np.random.default_rng(2)
            fs = field.FieldState(fs.sdf + 0.03 * rng.normal(size=fs.sdf.shape),
                                  rng.uniform(-0.3, 0.3, size=fs.deformation.shape) * fs.deform_limit,
                                  fs.deform_limit)
        m = grid.marching_tetrahedra(g, fs)
        tag = f"r{R}{'_noisy' if noisy else ''}"
        mt[f"{tag}_sdf"] = fs.sdf
        mt[f"{tag}_deform"] = fs.deformation
        mt[f"{tag}_V"] = m.vertices
        mt[f"{tag}_F"] = m.triangles
        print("MT", tag, m.vertices.shape, m.triangles.shape, m.euler_characteristic())
    np.savez_compressed(os.path.join(HERE, "mt.npz"), **mt)


def window_depths(mean_depth, near, far, levels=6, seed=7):
    """Mean depths that make the N_w window reorder (on the stock fields every equal-key
    run is an exact tie, so the window never acts).  Splats are grouped into `levels` coarse depth
    layers; every splat of a layer gets the SAME 32-bit key q (raster.py:132-134) and a random
    mean depth inside that key's bucket, so the stable sort leaves each layer in splat-index
    order while the window (_core.pyx:171-187) sorts by mean depth: long runs, many inversions,
    overlapping splats in one run."""
    md = np.asarray(mean_depth, np.float64)
    lv = np.floor((md - md.min()) / (md.max() - md.min() + 1e-9) * levels)
    qbase = np.floor((md.min() - near) / (far - near) * 4294967295.0) + lv * 1000
    rng = np.random.default_rng(seed)
    md2 = near + (far - near) * (qbase + 0.1 + 0.8 * rng.uniform(size=md.shape)) / 4294967295.0
    q2 = (np.clip((md2 - near) / (far - near), 0, 1) * 4294967295.0).astype(np.uint64)
    assert np.array_equal(q2, qbase.astype(np.uint64))
    return md2


def _counts(saved, bins, S):
    counts = np.zeros((S, S), np.int32)
    for tid, cnt, _, _ in saved.records:
        x0, y0 = (tid % bins.tiles_x) * 16, (tid // bins.tiles_x) * 16
        c2 = cnt.reshape(16, 16)
        h, w = min(16, S - y0), min(16, S - x0)
        counts[y0:y0 + h, x0:x0 + w] = c2[:h, :w]
    return counts


def _noisy(field, g, seed=0):
    rng = np.random.default_rng(seed)
    fs = field.init_sphere(g, 0.5)
    sdf = fs.sdf + 0.08 * rng.normal(size=fs.sdf.shape)
    lim = fs.deform_limit
    deform = rng.uniform(-0.4 * lim, 0.4 * lim, size=fs.deformation.shape)
    return field.FieldState(sdf, deform, lim)


def main_color_window(ref_src: str):
    """Colour compositing / colour gradients and the reordering N_w window, from the reference."""
    sys.path.insert(0, ref_src)
    import tetsplat
    from tetsplat import camera, field, grid, raster, splat
    assert tetsplat.BACKEND_NAME == "compiled", "build the reference's Cython kernels first"

    # --- colour: build_scene(colors=) + colour map + d_color (_core.pyx:202-205,219-222,
    #     410-413,433-436; raster.py:303-305) ---------------------------------------------
    R, S, s, ci = 12, 96, 100.0, 5
    g = grid.build_grid(R)
    fs = _noisy(field, g)
    cam = camera.orbit_camera(ci, 8, width=S, height=S)
    colors = np.random.default_rng(5).uniform(size=(g.num_tets, 3))
    active = splat.prefilter(g, fs, s)
    sc = splat.build_scene(g, fs, cam, s, active=active, colors=colors)
    bins = raster.bin_and_sort(sc, cam)
    maps, saved = raster.render_forward(sc, bins, cam, n_w=5, save_state=True)
    rng = np.random.default_rng(1)
    dm = raster.RenderMaps(rng.normal(size=(S, S, 3)), rng.normal(size=(S, S)), rng.normal(size=(S, S)),
                           rng.normal(size=(S, S, 3)))
    gb = raster.render_backward(saved, sc, g, fs, cam, dm)
    np.savez_compressed(os.path.join(HERE, "color_noisy_r12_s100_cam5.npz"),
                        R=R, S=S, s=s, cam_index=ci, cam_count=8, sdf=fs.sdf, deform=fs.deformation,
                        colors=colors, active=active, tet_ids=sc.tet_ids, starts=bins.starts, items=bins.items,
                        counts=_counts(saved, bins, S), normal=maps.normal, depth=maps.depth, opacity=maps.opacity,
                        color=maps.color, d_normal=dm.normal, d_depth=dm.depth, d_opacity=dm.opacity,
                        d_color=dm.color, d_sdf=gb.d_sdf, d_deform=gb.d_deform, d_color_tet=gb.d_color)
    print("color K=", len(sc), "M=", len(bins.items), "|d_color|", np.abs(gb.d_color).max())

    # --- window: a scene whose tile lists the N_w window reorders ---------------------------
    R, S, s, ci = 16, 128, 100.0, 3
    g = grid.build_grid(R)
    fs = _noisy(field, g)
    cam = camera.orbit_camera(ci, 8, width=S, height=S)
    active = splat.prefilter(g, fs, s)
    sc = splat.build_scene(g, fs, cam, s, active=active)
    sc.mean_depth = window_depths(sc.mean_depth, cam.near, cam.far)
    bins = raster.bin_and_sort(sc, cam)
    rng = np.random.default_rng(1)
    dm = raster.RenderMaps(rng.normal(size=(S, S, 3)), rng.normal(size=(S, S)), rng.normal(size=(S, S)))
    out = dict(R=R, S=S, s=s, cam_index=ci, cam_count=8, sdf=fs.sdf, deform=fs.deformation, active=active,
               tet_ids=sc.tet_ids, vert_ids=sc.vert_ids, proj=sc.proj, depths=sc.depths, f=sc.f,
               normals=sc.normals, mean_depth=sc.mean_depth, alpha_max=sc.alpha_max, bbox=sc.bbox,
               starts=bins.starts, items=bins.items, d_normal=dm.normal, d_depth=dm.depth, d_opacity=dm.opacity)
    nws = (1, 2, 5, bins.max_list_length())
    out["windows"] = np.array(nws)
    for nw in nws:
        maps, saved = raster.render_forward(sc, bins, cam, n_w=nw, save_state=True)
        gb = raster.render_backward(saved, sc, g, fs, cam, dm)
        out.update({f"normal_w{nw}": maps.normal, f"depth_w{nw}": maps.depth, f"opacity_w{nw}": maps.opacity,
                    f"counts_w{nw}": _counts(saved, bins, S), f"d_sdf_w{nw}": gb.d_sdf,
                    f"d_deform_w{nw}": gb.d_deform})
    np.savez_compressed(os.path.join(HERE, "window_noisy_r16_s100_cam3.npz"), **out)
    print("window K=", len(sc), "M=", len(bins.items), "maxL", bins.max_list_length())


def main_c2f(ref_src: str):
    """coarse_to_fine_filter (splat.py:88-109): box of the survivors, and the second round with
    a positional field function on the rescaled grid."""
    sys.path.insert(0, ref_src)
    from tetsplat import field, grid, splat
    g = grid.build_grid(12)
    fs = _noisy(field, g)
    act, box = splat.coarse_to_fine_filter(g, fs, 100.0)
    fn = lambda p: np.linalg.norm(p - np.array([0.05, -0.02, 0.01]), axis=1) - 0.4
    act2, box2 = splat.coarse_to_fine_filter(g, fs, 100.0, field_fn=fn)
    np.savez_compressed(os.path.join(HERE, "c2f_noisy_r12_s100.npz"), sdf=fs.sdf, deform=fs.deformation, R=12,
                        s=100.0, active=act, box=box, active_fn=act2, box_fn=box2)
    print("c2f", len(act), len(act2), box)


if __name__ == "__main__":
    src = sys.argv[1] if len(sys.argv) > 1 else "/tmp/tsref/src"
    if "--color-window" in sys.argv:
        main_color_window(src)
    elif "--c2f" in sys.argv:
        main_c2f(src)
    else:
        main(src)
        main_color_window(src)
        main_c2f(src)
