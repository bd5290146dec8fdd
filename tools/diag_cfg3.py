"""Diagnose config-3 map differences per view: worst pixel, counts, per-pixel records (GPU
plugin vs the reference's _core) for the worst tile."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200 import kernels
from oracle import ts_oracle as O

R, S = 128, 1024
s = float(sys.argv[1]) if len(sys.argv) > 1 else 100.0
views = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else list(range(8))
og = O.build_grid(R)
of = O.init_sphere_field(og)
g = ts.build_grid(R)
f = ts.FieldState.from_numpy(of.sdf, of.deformation, ts.deform_limit_for(g))
active = O.prefilter(og, of, s)
real = O._load_ref()
for vi in views:
    cam = ts.orbit_camera(vi, 8, width=S, height=S)
    ocam = O.orbit_camera(vi, 8, width=S, height=S)
    osc = O.build_scene(og, of, ocam, s, active=active)
    ob = O.bin_and_sort(osc, ocam)
    om, osv = O.render_forward(osc, ob, ocam, save_state=True, want_counts=True)
    sc = ts.build_scene(g, f, cam, s, active=torch.as_tensor(active.astype(np.int32)).cuda())
    b = ts.bin_and_sort(sc, cam)
    maps, sv = ts.render_forward(sc, b, cam, save_state=True)
    n, d, o, _ = maps.numpy()
    cnt = sv.n_blend.cpu().numpy()
    for name, a, r in (("normal", n, om.normal), ("depth", d, om.depth), ("opacity", o, om.opacity)):
        err = np.abs(a - r)
        if err.ndim == 3:
            err = err.max(axis=2)
        y, x = np.unravel_index(np.argmax(err), err.shape)
        print(f"view {vi} {name}: rel {err.max() / np.abs(r).max():.3e} at ({y},{x}) cnt gpu {cnt[y, x]} ref "
              f"{osv.counts[y, x]} opac ref {om.opacity[y, x]:.9f} gpu {o[y, x]:.9f}", flush=True)
        if name == "normal" and err.max() / np.abs(r).max() > 5e-5:
            t = (y // 16) * ob.tiles_x + x // 16
            p = (y % 16) * 16 + x % 16
            # the GPU's own scene as the plugin's input, same for the reference kernels
            osc2 = O.SplatScene(*(a.detach().cpu().numpy() for a in (sc.tet_ids, sc.vert_ids, sc.proj, sc.depths, sc.f,
                                                                    sc.normals, sc.mean_depth, sc.alpha_max, sc.bbox)),
                                s, None)
            ob2 = O.bin_and_sort(osc2, ocam)
            out = {}
            for nm, mod in (("gpu", kernels), ("ref", real)):
                O._REF = mod
                mm, ss = O.render_forward(osc2, ob2, ocam, save_state=True, backend="ref")
                rec = [r for r in ss.records if int(r[0]) == t][0]
                off = np.concatenate([[0], np.cumsum(rec[1])])
                out[nm] = (rec[2][off[p]:off[p + 1]], rec[3][off[p]:off[p + 1]], mm.normal[y, x])
            O._REF = real
            for nm in out:
                idx, al, nn = out[nm]
                T = np.cumprod(np.concatenate([[1.0], 1 - al]))
                print(f"   {nm}: n={len(idx)} idx={idx.tolist()} alpha={np.array2string(al, precision=9)} T={np.array2string(T, precision=6)} normal={nn}")
