"""`tetsplat bench-sort` on the GPU (cli.py:194-225): the windowed tile renderer against the
exact-order render_reference, per resolution and window, with the time per frame.

    python -m paper_2406_01579_b200.bench_sort [--resolutions 16 32] [--windows 1 3 5 9]
                                               [--image-size 128] [--seed 0] [--s 100] [--out DIR]

Same field (sphere 0.55 + 0.05 N(0,1) from numpy's default_rng(seed)), camera (orbit 0 of 8)
and CSV columns as the reference; ms_per_frame is the compositing launch timed with CUDA
events (the reference's is wall time of its CPU render_forward).
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch


def bench_sort(resolutions=(16, 32), windows=(1, 3, 5, 9), image_size=128, seed=0, s=100.0) -> str:
    from . import (AnalyticShape, bin_and_sort, build_grid, build_scene, init_from_shape, orbit_camera,
                   render_forward, render_reference)
    rng = np.random.default_rng(int(seed))
    lines = ["resolution,window,max_abs,mean_abs,ms_per_frame"]
    for r in resolutions:
        grid = build_grid(int(r))
        field = init_from_shape(grid, AnalyticShape("sphere", (0.55,)))
        noise = torch.as_tensor(rng.standard_normal(grid.num_vertices), device=field.sdf.device)
        field.sdf.add_(0.05 * noise)
        camera = orbit_camera(0, 8, width=image_size, height=image_size)
        scene = build_scene(grid, field, camera, s)
        bins = bin_and_sort(scene, camera)
        ref = render_reference(scene, camera)
        for w in windows:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            maps, _ = render_forward(scene, bins, camera, n_w=int(w), timing=ev)
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1])
            diff = torch.cat([(maps.normal - ref.normal).abs().ravel(), (maps.depth - ref.depth).abs().ravel(),
                              (maps.opacity - ref.opacity).abs().ravel()])
            lines.append(f"{r},{w},{float(diff.max()):.6e},{float(diff.mean()):.6e},{ms:.2f}")
    return "\n".join(lines) + "\n"


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2406_01579_b200.bench_sort")
    ap.add_argument("--resolutions", type=int, nargs="+", default=[16, 32])
    ap.add_argument("--windows", type=int, nargs="+", default=[1, 3, 5, 9])
    ap.add_argument("--image-size", type=int, default=128)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--s", type=float, default=100.0)
    ap.add_argument("--out", default=None, help="directory for bench_sort.csv")
    a = ap.parse_args(argv)
    csv = bench_sort(a.resolutions, a.windows, a.image_size, a.seed, a.s)
    if a.out:
        os.makedirs(a.out, exist_ok=True)
        with open(os.path.join(a.out, "bench_sort.csv"), "w") as fh:
            fh.write(csv)
    print(csv, end="")
    return 0


if __name__ == "__main__":
    sys.exit(main())
