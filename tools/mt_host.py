"""Host-side split of one Marching Tetrahedra call: run (device pipeline, two syncs), fetch
(D2H into pageable numpy), release."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2406_01579_b200 as ts
from paper_2406_01579_b200 import _native
R = int(os.environ.get("R", 256))
g = ts.build_grid(R)
f = ts.init_from_shape(g, ts.AnalyticShape("sphere", (0.5,)))
L = _native.lib()
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h, nv, nt = ctypes.c_void_p(), _native.i64(), _native.i64()
    _native.check(L.ts_marching_tets_run(_native.ptr(f.sdf), _native.ptr(f.deformation), R, ctypes.byref(h), nv, nt, None))
    t1 = time.perf_counter()
    V = np.empty((nv.value, 3)); F = np.empty((nt.value, 3), np.int64)
    _native.check(L.ts_marching_tets_fetch(h, V.ctypes.data, F.ctypes.data))
    t2 = time.perf_counter()
    _native.check(L.ts_marching_tets_release(h))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"run {1e3*(t1-t0):.2f} ms  fetch {1e3*(t2-t1):.2f} ms  release {1e3*(t3-t2):.2f} ms")
