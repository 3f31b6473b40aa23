"""The suffix side of trace_frame on the GPU: ordered film and
parent folds, the reverse pass, TrainSample emission and the Film buffers.

Mirrors the reference's `Film` (wavefront.hpp:78-123, wavefront.cpp:86-116) and the
tail of `trace_frame` (wavefront.cpp:483-550).  The f64 folds run in the reference's
order (one thread per pixel / parent run of the queue), so the film and every
vertex's suffix contribution are bit-identical to the CPU reference.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

from . import _capi
from .stage import GpuContext

# TrainSample (networks.hpp:20-32), 80 bytes
TRAIN_SAMPLE_DTYPE = np.dtype([("position", "<f4", 3), ("omega_o", "<f4", 2), ("roughness", "<f4"),
                               ("t_x", "<f4", 3), ("i_pixel", "<f4", 3), ("lo_sample", "<f4", 3),
                               ("q_norm", "<f4"), ("q_real", "<f4"), ("pixel", "<u4"), ("k_i", "<f4"),
                               ("depth", "<u2"), ("pad", "<u2")])
assert TRAIN_SAMPLE_DTYPE.itemsize == 80


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_contiguous():
        raise RuntimeError("suffix-side buffers must be contiguous")
    return t.data_ptr()


class SuffixStage:
    """Film folds, reverse pass and TrainSample emission on one GPU."""

    def __init__(self, device: int = 0, ctx: Optional[GpuContext] = None):
        self.ctx = ctx or GpuContext(device)
        self.device = torch.device("cuda", self.ctx.device)
        self._counts = torch.zeros(2, dtype=torch.int64, device=self.device)
        self._nonfinite = torch.zeros(1, dtype=torch.int64, device=self.device)

    @property
    def handle(self):
        return self.ctx.handle

    def fold_ordered(self, dst: torch.Tensor, keys: torch.Tensor, terms: torch.Tensor) -> None:
        """dst[keys[i]] += terms[i] in item order (f64 x3; keys int32, non-decreasing, -1 skipped):
        frame[pixel] += term (wavefront.cpp:299, :317, :355, :485), parent.s += term (:301, :319)."""
        self.ctx.bind_stream()
        n = int(keys.numel())
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_fold_ordered(self.handle, _ptr(dst), int(dst.numel() // 3),
                                                                    _ptr(keys), _ptr(terms), n))

    def reverse_pass(self, verts: List[Dict[str, torch.Tensor]]) -> None:
        """wavefront.cpp:505-507: for d = B..2, verts[d-1][parent].s += verts[d].s (verts[d] has
        'parent' int32 and 's' float64 [n, 3]; index 0 unused, as in the reference)."""
        for d in range(len(verts) - 1, 1, -1):
            if verts[d]["parent"].numel():
                self.fold_ordered(verts[d - 1]["s"], verts[d]["parent"], verts[d]["s"])

    def emit_train(self, verts: List[Dict[str, torch.Tensor]], i_acc: torch.Tensor, n_pixels: int,
                   out: torch.Tensor) -> Tuple[int, int]:
        """wavefront.cpp:510-543: TrainSamples for depths 1..B-1 in order, k_i per pixel.
        out: uint8 tensor [capacity, 80] (TRAIN_SAMPLE_DTYPE rows).  Returns (samples, nonfinite)."""
        self.ctx.bind_stream()
        capacity = int(out.shape[0])
        self._counts.zero_()
        self._nonfinite.zero_()
        cur = 0
        for d in range(1, len(verts)):
            v = verts[d]
            n = int(v["pixel"].numel())
            soa = _capi.VertexRecSoA(_ptr(v.get("p01")), _ptr(v.get("wo01")), _ptr(v.get("roughness")),
                                     _ptr(v.get("weight")), _ptr(v.get("pixel")), _ptr(v.get("q_norm")),
                                     _ptr(v.get("q_real")), _ptr(v.get("decided")), _ptr(v.get("s")))
            src, dst = self._counts[cur], self._counts[1 - cur]
            _capi.check(self.handle, self.ctx.lib.nrrs_gpu_emit_train(
                self.handle, d, C.byref(soa), n, _ptr(i_acc), _ptr(out), capacity, src.data_ptr(), dst.data_ptr(),
                self._nonfinite.data_ptr()))
            cur = 1 - cur
        end = self._counts[cur]
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_train_k_i(self.handle, _ptr(out), 0, end.data_ptr(), capacity,
                                                                 int(n_pixels)))
        return int(end.item()), int(self._nonfinite.item())

    def close(self) -> None:
        self.ctx.close()


class GpuFilm:
    """Film buffers on the device (wavefront.hpp:78-123): sum (f64), samples, i_cur, i_acc."""

    def __init__(self, width: int, height: int, suffix: SuffixStage):
        if width <= 0 or height <= 0:
            raise RuntimeError("Film: dimensions must be positive")
        self.width, self.height, self.sx = width, height, suffix
        n = width * height
        dev = suffix.device
        self.sum = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        self.samples = torch.zeros(n, dtype=torch.int32, device=dev)
        self.i_cur = torch.zeros((n, 3), dtype=torch.float32, device=dev)
        self.i_acc = torch.zeros((n, 3), dtype=torch.float32, device=dev)
        self.normal = torch.zeros((n, 3), dtype=torch.float32, device=dev)

    def pixel_count(self) -> int:
        return self.width * self.height

    def add_frame(self, frame: torch.Tensor) -> None:
        if frame.shape != self.sum.shape:
            raise RuntimeError("Film::add_frame: frame size mismatch")
        self.sx.ctx.bind_stream()
        _capi.check(self.sx.handle, self.sx.ctx.lib.nrrs_gpu_film_add_frame(
            self.sx.handle, _ptr(self.sum), _ptr(self.samples), _ptr(self.i_cur), _ptr(frame), self.pixel_count()))

    def roll_acc(self) -> None:
        self.sx.ctx.bind_stream()
        _capi.check(self.sx.handle, self.sx.ctx.lib.nrrs_gpu_film_roll_acc(
            self.sx.handle, _ptr(self.i_acc), _ptr(self.i_cur), self.pixel_count()))

    def reset_accumulation(self) -> None:
        self.sum.zero_()
        self.samples.zero_()
        self.i_cur.zero_()

    def mean_image(self) -> torch.Tensor:
        """(sum / samples).cast<float>() per pixel, 0 where samples == 0 (wavefront.hpp:92-96)."""
        s = self.samples.to(torch.float64).unsqueeze(1)
        return torch.where(s > 0, self.sum / s.clamp(min=1), torch.zeros_like(self.sum)).to(torch.float32)
