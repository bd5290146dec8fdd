"""ctypes binding of libtetsplat_b200.so (the C ABI in include/tetsplat_b200.h).

There is no CPU fallback: importing the kernels on a machine without the built library
or without a CUDA device raises immediately, so a silent non-GPU path can never run.
"""
from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TS_LIB_PATH") or os.path.join(HERE, "libtetsplat_b200.so")  # override: A/B timing only

TS_EINVAL = -1


class ts_camera(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3), ("fx", ctypes.c_double),
                ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("near_", ctypes.c_double), ("far_", ctypes.c_double), ("width", ctypes.c_int32),
                ("height", ctypes.c_int32), ("pad", ctypes.c_int32 * 2)]


class ts_scene(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("tet_ids", "vert_ids", "proj", "depths", "f", "normals",
                                               "mean_depth", "alpha_max", "bbox", "records")]


class ts_bins(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("starts", "splat_off", "items", "pos_of", "nonmono", "witems", "cpos",
                                                    "clen")]


_lib = None


def lib():
    """Load the library (once).  Raises when it is missing or no CUDA device exists."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built; run `python -m paper_2406_01579_b200.build`")
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 rasterizer needs a CUDA device; there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    PI64 = ctypes.POINTER(ctypes.c_int64)
    pc, ps, pb = ctypes.POINTER(ts_camera), ctypes.POINTER(ts_scene), ctypes.POINTER(ts_bins)
    sig = {
        "ts_last_error": ([], ctypes.c_char_p),
        "ts_version": ([], ctypes.c_int),
        "ts_prefilter": ([P, I32, D, D, P, PI64, P], ctypes.c_int),
        "ts_build_scene": ([P, P, I32, pc, D, P, I64, ps, PI64, P], ctypes.c_int),
        "ts_prepare_records": ([ps, I64, I32, I32, P], ctypes.c_int),
        "ts_bin_count": ([P, P, I64, pc, I32, P, P, PI64, PI64, P], ctypes.c_int),
        "ts_bin_sort": ([P, P, I64, pc, I32, pb, I64, I64, P], ctypes.c_int),
        "ts_forward_prepare": ([ps, I64, pb, I64, pc, I32, P, PI64, P], ctypes.c_int),
        "ts_render_forward": ([ps, I64, P, pb, I64, pc, D, D, P, I64, P, P, P, P, P, P, P, P, P], ctypes.c_int),
        "ts_render_backward": ([ps, I64, P, pb, I64, pc, P, P, P, ctypes.POINTER(P), ctypes.POINTER(P), P, P, I32,
                                P, P, P], ctypes.c_int),
        "ts_bins_from_lists": ([P, P, I32, P, D, D, P, P], ctypes.c_int),
        "ts_saved_records": ([ps, pb, pc, P, P, P, P, P, I32, P, P, P, P], ctypes.c_int),
        "ts_backward_tiles": ([ps, I64, P, pb, I64, pc, P, P, P, ctypes.POINTER(P), ctypes.POINTER(P), P, P, I32, P,
                               P], ctypes.c_int),
        "ts_eikonal": ([P, P, I32, P, I64, D, P, P, P], ctypes.c_int),
        "ts_normal_consistency": ([P, P, I32, D, P, P, P], ctypes.c_int),
        "ts_normal_consistency_scratch_bytes": ([I32], ctypes.c_int64),
        "ts_normal_consistency_ws": ([P, P, I32, D, P, P, P, P], ctypes.c_int),
        "ts_adam_step": ([I32, P, P, P, P, P, P, P, D, D, D, D, I64, D, D, P, P], ctypes.c_int),
        "ts_rasterize_mesh": ([P, I64, P, I64, pc, P, P, P, P], ctypes.c_int),
        "ts_marching_tets_count": ([P, P, I32, PI64, PI64, P], ctypes.c_int),
        "ts_marching_tets": ([P, P, I32, P, P, ctypes.POINTER(ctypes.c_int64), P], ctypes.c_int),
        "ts_marching_tets_run": ([P, P, I32, ctypes.POINTER(P), PI64, PI64, P], ctypes.c_int),
        "ts_marching_tets_fetch": ([P, P, P], ctypes.c_int),
        "ts_marching_tets_release": ([P], ctypes.c_int),
        "ts_debug_counters": ([ctypes.POINTER(ctypes.c_uint64), ctypes.c_int], ctypes.c_int),
        "ts_debug_set_flags": ([ctypes.c_int], ctypes.c_int),
        "ts_debug_hist": ([ctypes.POINTER(ctypes.c_uint64), ctypes.c_int], ctypes.c_int),
        "ts_debug_phases": ([ctypes.POINTER(ctypes.c_uint64), ctypes.c_int], ctypes.c_int),
        "ts_workspace_create": ([], P),
        "ts_workspace_destroy": ([P], None),
        "ts_view_forward": ([P, P, P, I32, pc, D, P, I64, I32, D, P, P, P, P, P, ctypes.POINTER(ctypes.c_int64), P],
                            ctypes.c_int),
        "ts_view_backward": ([P, P, ctypes.POINTER(P), ctypes.POINTER(P), P, P, P, P], ctypes.c_int),
        "ts_view_n_blend": ([P], P),
        "ts_view_backward_fx": ([P, P, ctypes.POINTER(P), ctypes.POINTER(P), P, P, P, P], ctypes.c_int),
        "ts_render_backward_fx": ([ps, I64, P, pb, I64, pc, P, P, P, ctypes.POINTER(P), ctypes.POINTER(P), P, P,
                                   I32, P, P, P], ctypes.c_int),
        "ts_eikonal_fx": ([P, P, I32, P, I64, D, P, P, P], ctypes.c_int),
        "ts_normal_consistency_fx": ([P, P, I32, D, P, P, P, P], ctypes.c_int),
        "ts_fx_to_f32": ([P, I64, P, P, P], ctypes.c_int),
        "ts_normal_consistency_slab": ([P, P, I32, D, P, P, P, P, I32, I32, P], ctypes.c_int),
        "ts_workspace_set_caps": ([P, I64, I64, I64, P], ctypes.c_int),
        "ts_view_collect": ([P, P, P, P], ctypes.c_int),
        "ts_view_status": ([P, PI64, P], ctypes.c_int),
        "ts_view_need": ([P], P),
        "ts_view_overflow": ([P], P),
        "ts_debug_tile_times": ([ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32), ctypes.c_int],
                                ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().ts_last_error().decode()
    if rc == TS_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def i64():
    return ctypes.c_int64(0)


def debug_counters(reset: bool = True):
    """(edge FP64 re-decisions, alpha FP64 re-decisions, forward rect-pass pairs, uncertain-det
    edge re-decisions, alpha re-decisions by reason [flag 8]: f band / tiny-or-clip, 0,
    softplus-chain re-decisions [flag 8]) since last reset."""
    out = (ctypes.c_uint64 * 8)()
    check(lib().ts_debug_counters(out, int(reset)))
    return tuple(int(v) for v in out)


def debug_phases(reset: bool = True):
    """Per-phase barrier-to-barrier cycles of the compositing kernels (flag bit 2; see the header)."""
    out = (ctypes.c_uint64 * 16)()
    check(lib().ts_debug_phases(out, int(reset)))
    return tuple(int(v) for v in out)
