"""Host mirror of the reference's RRS core interface (proj/include/nrrs/rrs.hpp).

Same names, argument meaning and error behaviour as the C++ API; the array
operations (normalize_factors, realize_counts, plan_spawns) run on the GPU
through the C ABI -- there is no CPU path.
"""
from __future__ import annotations

import numpy as np

import ctypes as C
import dataclasses
import enum
import math
from typing import List

import torch

from . import _capi


class StrategyKind(enum.IntEnum):
    """rrs.hpp:72-79 (numbering shared with nrrs_strategy_kind)."""
    Fixed = 0
    Throughput = 1
    AdrrsTree = 2
    AdrrsNn = 3
    Nrrs = 4
    AidNrrs = 5


@dataclasses.dataclass
class Strategy:
    """rrs.hpp:81-92."""
    kind: StrategyKind = StrategyKind.Fixed
    fixed_value: float = 1.0

    def neural(self) -> bool:
        return self.kind in (StrategyKind.AdrrsNn, StrategyKind.Nrrs, StrategyKind.AidNrrs)

    def adaptive(self) -> bool:
        return self.kind != StrategyKind.Fixed

    def c(self) -> _capi.StrategyC:
        return _capi.StrategyC(int(self.kind), float(self.fixed_value))


def parse_strategy(name: str) -> Strategy:
    """rrs.cpp:47-90; raises RuntimeError like fail()."""
    if name.startswith("fixed"):
        value = 1.0
        if ":" in name:
            value = float(name.split(":", 1)[1])
        value = float(torch.tensor(value, dtype=torch.float32))  # std::stof
        if not value >= 0.0:
            raise RuntimeError("parse_strategy: fixed value must be >= 0")
        return Strategy(StrategyKind.Fixed, value)
    table = {"pt": Strategy(StrategyKind.Fixed, 1.0), "throughput": Strategy(StrategyKind.Throughput),
             "adrrs-tree": Strategy(StrategyKind.AdrrsTree), "adrrs-nn": Strategy(StrategyKind.AdrrsNn),
             "nrrs": Strategy(StrategyKind.Nrrs), "aid-nrrs": Strategy(StrategyKind.AidNrrs)}
    if name in table:
        return table[name]
    raise RuntimeError(f"parse_strategy: unknown strategy '{name}'")


def _fmt_float(v: float) -> str:
    # std::ostream << float: 6 significant digits, %g style
    return f"{v:g}"


def strategy_name(s: Strategy) -> str:
    """rrs.cpp:92-111."""
    names = {StrategyKind.Throughput: "throughput", StrategyKind.AdrrsTree: "adrrs-tree",
             StrategyKind.AdrrsNn: "adrrs-nn", StrategyKind.Nrrs: "nrrs", StrategyKind.AidNrrs: "aid-nrrs"}
    if s.kind == StrategyKind.Fixed:
        return "fixed:" + _fmt_float(s.fixed_value)
    return names[s.kind]


DepthAssignment = List[Strategy]


def uniform_assignment(s: Strategy, max_depth: int) -> DepthAssignment:
    return [dataclasses.replace(s) for _ in range(max_depth)]


def parse_assignment(spec: str, max_depth: int) -> DepthAssignment:
    """rrs.cpp:117-129: a single name is uniform; a list needs max_depth entries."""
    if "," not in spec:
        return uniform_assignment(parse_strategy(spec), max_depth)
    a = [parse_strategy(tok) for tok in spec.split(",")]
    if len(a) != max_depth:
        raise RuntimeError(f"parse_assignment: expected {max_depth} entries")
    return a


def assignment_name(a: DepthAssignment) -> str:
    return ",".join(strategy_name(s) for s in a)


def _f32(x: float) -> float:
    return float(torch.tensor(x, dtype=torch.float32))


@dataclasses.dataclass
class RateControl:
    """rrs.hpp:23-36 (float32 arithmetic, like the C++ struct)."""
    f_rate: float = 0.85
    alpha: float = 1.0
    eps: float = 0.01
    enabled: bool = True
    overflow_events: int = 0

    def gain(self) -> float:
        if not self.enabled:
            return 1.0
        return _f32(_f32(self.f_rate) * _f32(self.alpha))

    def note_overflow(self) -> None:
        self.overflow_events += 1
        self.alpha = _f32(_f32(self.alpha) * _f32(1.0 - _f32(self.eps)))


def bernstein_bound(f_rate: float, n_pixels: int) -> float:
    """rrs.cpp:26-33."""
    if f_rate >= 1.0:
        return 1.0
    gap = 1.0 - f_rate
    return math.exp(-(gap * gap * float(n_pixels) / (2.0 * f_rate + (2.0 / 3.0) * gap)))


def queue_capacity_for(n_pixels: int) -> int:
    """wavefront.cpp:82-84."""
    return int(_capi.lib().nrrs_queue_capacity_for(int(n_pixels)))


def throughput_rr_factor(weight) -> float:
    """rrs.hpp:49-51, float32."""
    w = torch.as_tensor(weight, dtype=torch.float32)
    lum = (torch.tensor(0.2126, dtype=torch.float32) * w[0] + torch.tensor(0.7152, dtype=torch.float32) * w[1]) \
        + torch.tensor(0.0722, dtype=torch.float32) * w[2]
    return float(torch.minimum(torch.tensor(1.0), lum))


# ---------------------------------------------------------------------------
# GPU array drop-ins (device tensors)
# ---------------------------------------------------------------------------
def _ctx(ctx=None):
    from .stage import default_context
    return ctx if ctx is not None else default_context()


def normalize_factors(q: torch.Tensor, n_pixels: int, ctx=None) -> float:
    """rrs.hpp:18 / rrs.cpp:8-24: scales q (float32 CUDA tensor) in place iff F < 1; returns F."""
    c = _ctx(ctx)
    _require_cuda(q, torch.float32)
    f = C.c_double(0.0)
    _capi.check(c.handle, _capi.lib().nrrs_gpu_normalize_factors(c.handle, q.data_ptr(), q.numel(),
                                                                 int(n_pixels), C.byref(f)))
    return f.value


def realize_counts(q: torch.Tensor, u: torch.Tensor, counts: torch.Tensor, ctx=None) -> int:
    """rrs.hpp:45-46 / rrs.cpp:35-45: stochastic rounding into int32 counts; returns S."""
    c = _ctx(ctx)
    if q.numel() != u.numel() or q.numel() != counts.numel():
        raise RuntimeError("realize_counts: size mismatch")
    _require_cuda(q, torch.float32)
    _require_cuda(u, torch.float32)
    _require_cuda(counts, torch.int32)
    total = C.c_uint64(0)
    _capi.check(c.handle, _capi.lib().nrrs_gpu_realize_counts(c.handle, q.data_ptr(), u.data_ptr(),
                                                              counts.data_ptr(), q.numel(), C.byref(total)))
    return total.value


@dataclasses.dataclass
class SpawnPlan:
    """wavefront.hpp:126-130."""
    offset: torch.Tensor
    spawned: int
    dropped: int


def plan_spawns(counts: torch.Tensor, capacity: int, ctx=None) -> SpawnPlan:
    """wavefront.hpp:132 / wavefront.cpp:141-154."""
    c = _ctx(ctx)
    _require_cuda(counts, torch.int32)
    offset = torch.empty(counts.numel(), dtype=torch.int32, device=counts.device)
    spawned, dropped = C.c_uint32(0), C.c_uint64(0)
    _capi.check(c.handle, _capi.lib().nrrs_gpu_plan_spawns(c.handle, counts.data_ptr(), counts.numel(),
                                                           int(capacity), offset.data_ptr(), C.byref(spawned),
                                                           C.byref(dropped)))
    return SpawnPlan(offset.view(torch.int32), spawned.value, dropped.value)


def _require_cuda(t: torch.Tensor, dtype) -> None:
    if not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise RuntimeError(f"expected a contiguous CUDA {dtype} tensor, got {t.dtype} on {t.device}")


ADRRS_EPS_SCALE = 1e-4  # TraceConfig::adrrs_eps_scale (wavefront.hpp:172)


def eps_div_from_luminance_sum(lum_sum: float, n_pixels: int, eps_scale: float = ADRRS_EPS_SCALE) -> float:
    """eps_div = adrrs_eps_scale * float(lum_acc / n_pixels), f32 product (wavefront.cpp:242-243)."""
    return float(np.float32(eps_scale) * np.float32(lum_sum / float(n_pixels)))
