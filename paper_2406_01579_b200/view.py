"""Fused per-view forward/backward over a persistent device workspace (csrc/workspace.cu).

`ViewRenderer.forward` runs build_scene -> bin_and_sort -> window -> render_forward in one C++
call (the host syncs that size the outputs happen inside C++), `ViewRenderer.backward` runs
render_backward + the vertex chain on the state the last forward left behind.  Same math
and kernels as the fine-grained API in splat.py / raster.py (which stays for reference-style
use); this is what the multi-view fit step uses.
"""
from __future__ import annotations

import ctypes

import torch

from . import _native
from .raster import DEFAULT_WINDOW, FixedPointGradients, GradientBuffers, RenderMaps
from .splat import T_STOP


class ViewRenderer:
    def __init__(self, device=None):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._L = _native.lib()
        self._ws = ctypes.c_void_p(self._L.ts_workspace_create())
        self._maps = {}
        self.counts = (0, 0, 0)

    def __del__(self):
        try:
            if self._ws and self._L is not None:
                self._L.ts_workspace_destroy(self._ws)
        except Exception:
            pass

    def _maps_for(self, H, W, color):
        key = (H, W, color)
        if key not in self._maps:
            self._maps[key] = RenderMaps.empty(H, W, color, self.device)
        return self._maps[key]

    def forward(self, grid, field, camera, s: float, active: torch.Tensor, n_w: int = DEFAULT_WINDOW,
                t_stop: float = T_STOP, colors: torch.Tensor | None = None, out: RenderMaps | None = None,
                stream=None) -> RenderMaps:
        """Render one view; `active` = int32 prefilter output.  Returns maps (reused buffers
        unless `out` is given).  With capacities set (set_caps) no host round trip happens and
        `counts` is (-1, -1, -1): the counts are on the device (collect)."""
        if n_w < 1:
            raise ValueError("resorting window must be >= 1")
        maps = out if out is not None else self._maps_for(camera.height, camera.width, colors is not None)
        counts = (ctypes.c_int64 * 4)()
        col = None if colors is None else colors.to(device=self.device, dtype=torch.float32).contiguous()
        _native.check(self._L.ts_view_forward(
            self._ws, _native.ptr(field.sdf), _native.ptr(field.deformation), grid.resolution, camera.abi(),
            float(s), _native.ptr(active), int(active.numel()), int(n_w), float(t_stop), _native.ptr(col),
            _native.ptr(maps.normal), _native.ptr(maps.depth), _native.ptr(maps.opacity), _native.ptr(maps.color),
            counts, _native.stream_ptr(stream)))
        self.counts = (counts[0], counts[1], counts[2])
        self.max_list = counts[3]
        self._last = maps
        return maps

    def n_blend(self) -> torch.Tensor:
        """(H, W) int32 blends per pixel of the last forward (a copy; stream-ordered on the
        current stream) — for parity checks."""
        H, W = self._last.depth.shape
        p = self._L.ts_view_n_blend(self._ws)

        class _Dev:  # the workspace buffer seen through __cuda_array_interface__
            __cuda_array_interface__ = {"shape": (H, W), "typestr": "<i4", "data": (int(p), False), "version": 2}
        return torch.as_tensor(_Dev(), device=self.device).clone()

    def set_caps(self, cap_pairs: int = 0, cap_pixel_pairs: int = 0, cap_list: int = 0,
                 need_out: torch.Tensor | None = None):
        """Capacities of the sync-free forward (tile pairs M, pixel pairs P, the longest tile
        list, 0 = unbounded); cap_pairs or cap_pixel_pairs 0 = the sizing path.  need_out
        (device int64[5]) receives {K, M, P, longest list, overflow} of each later forward."""
        self._need_out = need_out
        _native.check(self._L.ts_workspace_set_caps(self._ws, int(cap_pairs), int(cap_pixel_pairs), int(cap_list),
                                                    _native.ptr(need_out)))

    def collect(self, out5: torch.Tensor, status: torch.Tensor | None = None, stream=None):
        """Stream-ordered: out5 (device int64[5]) <- {K, M, P, longest list, overflow} of the last
        forward; status[2] += 1 when it overflowed its capacities."""
        _native.check(self._L.ts_view_collect(self._ws, _native.ptr(status), _native.ptr(out5),
                                              _native.stream_ptr(stream)))

    def backward(self, field, d_maps: RenderMaps, out: GradientBuffers | FixedPointGradients,
                 maps: RenderMaps | None = None,
                 stream=None, status: torch.Tensor | None = None) -> GradientBuffers:
        """Accumulate the last view's dL/d(sdf, deform) (and dL/dcolor) into `out` (a
        FixedPointGradients: bitwise-reproducible fixed-point accumulation).

        `status` (device f32, optional): incremented when a map gradient is non-finite — the
        fused path's form of raster.py:209-211, raised by the caller at its next sync
        (`batch.FitStep.check_status`)."""
        maps = maps if maps is not None else self._last
        P = ctypes.c_void_p
        m = (P * 4)(maps.normal.data_ptr(), maps.depth.data_ptr(), maps.opacity.data_ptr(),
                    maps.color.data_ptr() if maps.color is not None else None)
        d = (P * 4)(d_maps.normal.data_ptr(), d_maps.depth.data_ptr(), d_maps.opacity.data_ptr(),
                    d_maps.color.data_ptr() if d_maps.color is not None else None)
        fixed = isinstance(out, FixedPointGradients)  # deterministic (fixed-point) accumulation
        fn = self._L.ts_view_backward_fx if fixed else self._L.ts_view_backward
        _native.check(fn(self._ws, _native.ptr(field.deformation),
                         ctypes.cast(m, ctypes.POINTER(P)), ctypes.cast(d, ctypes.POINTER(P)),
                         _native.ptr(out.fx if fixed else out.d_vert),
                         _native.ptr(out.fx_color if fixed else out.d_color),
                         _native.ptr(status), _native.stream_ptr(stream)))
        return out
