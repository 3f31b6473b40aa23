"""The per-bounce RRS stage on the GPU -- the drop-in for trace_frame's RRS
decision block (wavefront.cpp:363-425, compaction :488-497).

`RrsStage` owns one nrrs_gpu_ctx (one CUDA device, the current torch stream)
and mirrors the reference's call sequence for one depth:

    strat = assignment[depth-1]                      # Mix-Depth gate (:366)
    q     = strategy_factor(...) per vertex          # (:368-389)
    F     = normalize_factors(q, n_pixels)           # (:390)
    gain  = rc.gain() if depth >= 2 and adaptive     # (:391)
    k     = realize_counts(q*gain, u)                # (:393-404)
    plan  = plan_spawns(k, capacity)                 # (:406)
    if plan.dropped: rc.note_overflow()              # (:407-411)
    slots = (parent j, child c) per queue slot       # (:421-425)

All arrays are torch CUDA tensors; the host only sequences launches.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Dict, Optional

import numpy as np
import torch

from . import _capi
from .networks import NeuralRrs
from .rrs import ADRRS_EPS_SCALE, RateControl, Strategy, StrategyKind, eps_div_from_luminance_sum, queue_capacity_for

VERTEX_FIELDS = ("p01", "wo01", "roughness", "weight", "i_pixel", "path_key")
FIELD_SHAPES = {"p01": 3, "wo01": 2, "roughness": 1, "weight": 3, "i_pixel": 3, "path_key": 1}


@dataclasses.dataclass
class StageResult:
    """Scalars of one stage call (SpawnPlan + FrameReport increments)."""
    f_norm: float
    sum_q: float
    total: int
    spawned: int
    dropped: int
    nonfinite: int
    box_cox_clamps: int
    overflow: bool

    @classmethod
    def from_c(cls, r: _capi.StageResultC) -> "StageResult":
        return cls(r.f_norm, r.sum_q, r.total, r.spawned, r.dropped, r.nonfinite, r.box_cox_clamps,
                   bool(r.overflow))


@dataclasses.dataclass
class StageOutputs:
    q_norm: torch.Tensor
    q_real: torch.Tensor
    slots: torch.Tensor          # [capacity, 2] int32 view of (parent, child) uint32
    k: Optional[torch.Tensor] = None
    offset: Optional[torch.Tensor] = None
    decided: Optional[torch.Tensor] = None
    q_orig: Optional[torch.Tensor] = None
    u: Optional[torch.Tensor] = None

    def c(self) -> _capi.StageOut:
        def p(t):
            return t.data_ptr() if t is not None else None
        return _capi.StageOut(p(self.q_norm), p(self.q_real), p(self.slots), p(self.k), p(self.offset),
                              p(self.decided), p(self.q_orig), p(self.u))


def vertex_soa(v: Dict[str, torch.Tensor]) -> _capi.VertexSoA:
    """nrrs_vertex_soa from a dict of contiguous CUDA tensors (float32; path_key int64/uint64)."""
    def p(name):
        t = v.get(name)
        if t is None:
            return None
        if not t.is_contiguous():
            raise RuntimeError(f"vertex field {name} must be contiguous")
        return t.data_ptr()
    return _capi.VertexSoA(p("p01"), p("wo01"), p("roughness"), p("weight"), p("i_pixel"), p("path_key"),
                           p("pixel"), p("i_acc"))


class GpuContext:
    """One nrrs_gpu_ctx bound to a CUDA device."""

    def __init__(self, device: int = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("nrrs: a CUDA (sm_100a) device is required; there is no CPU path")
        self.lib = _capi.lib()
        self.device = device
        h = C.c_void_p()
        rc = self.lib.nrrs_gpu_create(device, C.byref(h))
        if rc != 0:
            raise _capi.NrrsError(rc, f"nrrs_gpu_create(device={device}) failed (sm_100 device required)")
        self.handle = h

    def bind_stream(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        s = stream or torch.cuda.current_stream(self.device)
        _capi.check(self.handle, self.lib.nrrs_gpu_set_stream(self.handle, C.c_void_p(s.cuda_stream)))

    def launch_count(self) -> int:
        return int(self.lib.nrrs_gpu_launch_count(self.handle))

    def close(self) -> None:
        if self.handle:
            self.lib.nrrs_gpu_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_DEFAULT: Dict[int, GpuContext] = {}


def default_context(device: Optional[int] = None) -> GpuContext:
    dev = torch.cuda.current_device() if device is None else device
    if dev not in _DEFAULT:
        _DEFAULT[dev] = GpuContext(dev)
    ctx = _DEFAULT[dev]
    ctx.bind_stream()
    return ctx


class RrsStage:
    """Drop-in RRS decision stage for one film (n_pixels) on one GPU."""

    def __init__(self, n_pixels: int, nets: Optional[NeuralRrs] = None, capacity: int = 0, seed: int = 0,
                 device: int = 0):
        self.ctx = GpuContext(device)
        self.ctx.bind_stream()
        self.n_pixels = int(n_pixels)
        self.capacity = int(capacity) if capacity else queue_capacity_for(self.n_pixels)
        if self.capacity < self.n_pixels:
            raise RuntimeError("trace_frame: queue capacity below the pixel count")
        self.seed = int(seed)
        self.device = torch.device("cuda", device)
        self.nets = None
        if nets is not None:
            self.set_weights(nets)

    @property
    def handle(self):
        return self.ctx.handle

    def set_weights(self, nets: NeuralRrs) -> None:
        """Uploads the published snapshot (NeuralRrs::publish, networks.cpp:199-204)."""
        w = nets.weights_c()
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_set_weights(self.handle, C.byref(w)))
        self.nets = nets

    def set_weights_device(self, nets: NeuralRrs, blocks) -> None:
        """Uploads snapshot blocks that already live on this GPU (stat grid, stat MLP, rrs grid,
        rrs MLP as float32 CUDA tensors; `nets` gives the variant and grid spec): the table copies
        are built on the device (nrrs_gpu_set_weights_dev)."""
        c = nets.cfg
        blocks = [b.contiguous().float() for b in blocks]
        fp = C.POINTER(C.c_float)
        ptr = lambda t: C.cast(C.c_void_p(t.data_ptr()), fp) if t.numel() else None  # noqa: E731
        w = _capi.NetWeights(
            int(c.variant),
            _capi.GridSpec(c.grid.levels, c.grid.features, c.grid.base_resolution, c.grid.log2_table_size),
            ptr(blocks[0]), blocks[0].numel(), ptr(blocks[1]), blocks[1].numel(),
            ptr(blocks[2]), blocks[2].numel(), ptr(blocks[3]), blocks[3].numel())
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_set_weights_dev(self.handle, C.byref(w)))
        self.nets = nets

    def table_precision(self) -> tuple:
        """(AID grid stored in fp16?, error-budget probe max relative error of q; < 0 if not run)."""
        h, e = C.c_int32(0), C.c_double(0.0)
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_weights_info(self.handle, C.byref(h), C.byref(e)))
        return bool(h.value), float(e.value)

    def reserve(self, max_vertices: int) -> None:
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_reserve(self.handle, int(max_vertices), self.capacity))

    def alloc_outputs(self, n: int, full: bool = False) -> StageOutputs:
        dev = self.device
        o = StageOutputs(q_norm=torch.empty(n, dtype=torch.float32, device=dev),
                         q_real=torch.empty(n, dtype=torch.float32, device=dev),
                         slots=torch.empty((self.capacity, 2), dtype=torch.int32, device=dev))
        if full:
            o.k = torch.empty(n, dtype=torch.int32, device=dev)
            o.offset = torch.empty(n, dtype=torch.int32, device=dev)
            o.decided = torch.empty(n, dtype=torch.uint8, device=dev)
            o.q_orig = torch.empty(n, dtype=torch.float32, device=dev)
            o.u = torch.empty(n, dtype=torch.float32, device=dev)
        return o

    def params(self, depth: int, strategy: Strategy, gain: float, eps_div: float = 0.0,
               n_pixels: Optional[int] = None) -> _capi.StageParams:
        return _capi.StageParams(int(depth), int(n_pixels if n_pixels is not None else self.n_pixels),
                                 self.capacity, strategy.c(), float(gain), float(eps_div), self.seed)

    def run(self, vertices: Dict[str, torch.Tensor], depth: int, strategy: Strategy,
            rc: Optional[RateControl] = None, eps_div: float = 0.0, out: Optional[StageOutputs] = None,
            sync: bool = True, full: bool = False):
        """One depth of the decision block.  With sync=True returns (outputs, StageResult)
        and applies rc.note_overflow() on a dropped tail like wavefront.cpp:407-411."""
        self.ctx.bind_stream()
        n = int(vertices["p01"].shape[0]) if vertices["p01"].dim() == 2 else vertices["p01"].numel() // 3
        if out is None:
            out = self.alloc_outputs(n, full=full)
        gain = rc.gain() if rc is not None else 1.0
        p = self.params(depth, strategy, gain, eps_div)
        soa = vertex_soa(vertices)
        oc = out.c()
        if sync:
            r = _capi.StageResultC()
            _capi.check(self.handle, self.ctx.lib.nrrs_gpu_rrs_stage(self.handle, C.byref(soa), n, C.byref(p),
                                                                     C.byref(oc), C.byref(r)))
            res = StageResult.from_c(r)
            if rc is not None and res.dropped > 0:
                rc.note_overflow()
            return out, res
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_rrs_stage(self.handle, C.byref(soa), n, C.byref(p),
                                                                 C.byref(oc), None))
        return out, None

    def capture(self, vertices: Dict[str, torch.Tensor], depth: int, strategy: Strategy, out: StageOutputs,
                gain: float = 1.0, eps_div: float = 0.0, calls: int = 1) -> "torch.cuda.CUDAGraph":
        """Captures `calls` stage calls (K-A factors + K-B decide, no host sync) into a CUDA
        graph.  Every launch is replay-safe (device-side look-back epochs, self-resetting
        counters); gain and sizes are baked in, so re-capture when RateControl's gain
        changes.  One eager call first does any scratch allocation outside the capture.
        Read the scalars of the last replay with fetch_result()."""
        n = int(vertices["p01"].shape[0]) if vertices["p01"].dim() == 2 else vertices["p01"].numel() // 3
        p = self.params(depth, strategy, gain, eps_div)
        soa = vertex_soa(vertices)
        oc = out.c()
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            self.ctx.bind_stream()
            _capi.check(self.handle, self.ctx.lib.nrrs_gpu_rrs_stage(self.handle, C.byref(soa), n, C.byref(p),
                                                                     C.byref(oc), None))
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.ctx.bind_stream()
            for _ in range(int(calls)):
                _capi.check(self.handle, self.ctx.lib.nrrs_gpu_rrs_stage(self.handle, C.byref(soa), n, C.byref(p),
                                                                         C.byref(oc), None))
        self.ctx.bind_stream()
        return g

    def film_luminance_sum(self, i_acc: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Device f64 sum of luminance(i_acc[p]) over the film (wavefront.cpp:238-241), async."""
        self.ctx.bind_stream()
        n = i_acc.numel() // 3
        out = out if out is not None else torch.empty(1, dtype=torch.float64, device=self.device)
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_film_luminance_sum(self.handle, i_acc.data_ptr(), n,
                                                                          out.data_ptr()))
        return out

    def eps_div(self, i_acc: torch.Tensor, eps_scale: float = ADRRS_EPS_SCALE) -> float:
        """Per-frame ADRRS divisor guard (wavefront.cpp:238-243); syncs."""
        return eps_div_from_luminance_sum(float(self.film_luminance_sum(i_acc).item()), i_acc.numel() // 3,
                                          eps_scale)

    def fetch_result(self) -> StageResult:
        """Scalars of the most recent stage call (e.g. after a graph replay)."""
        self.ctx.bind_stream()
        r = _capi.StageResultC()
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_fetch_result(self.handle, C.byref(r)))
        return StageResult.from_c(r)

    def run_host(self, vertices: Dict[str, np.ndarray], depth: int, strategy: Strategy,
                 rc: Optional[RateControl] = None, eps_div: float = 0.0,
                 out: Optional[Dict[str, np.ndarray]] = None):
        """Reference-facing plugin path over HOST numpy buffers (H2D + stage + D2H)."""
        n = int(vertices["roughness"].shape[0]) if "roughness" in vertices else vertices["p01"].size // 3
        if out is None:
            out = {"q_norm": np.empty(n, np.float32), "q_real": np.empty(n, np.float32),
                   "slots": np.empty((self.capacity, 2), np.uint32)}
        gain = rc.gain() if rc is not None else 1.0
        p = self.params(depth, strategy, gain, eps_div)

        def hp(name, src):
            a = src.get(name)
            return a.ctypes.data if a is not None else None
        soa = _capi.VertexSoA(hp("p01", vertices), hp("wo01", vertices), hp("roughness", vertices),
                              hp("weight", vertices), hp("i_pixel", vertices), hp("path_key", vertices), None, None)
        oc = _capi.StageOut(hp("q_norm", out), hp("q_real", out), hp("slots", out), hp("k", out), hp("offset", out),
                            hp("decided", out), hp("q_orig", out), hp("u", out))
        r = _capi.StageResultC()
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_rrs_stage_host(self.handle, C.byref(soa), n, C.byref(p),
                                                                      C.byref(oc), C.byref(r)))
        res = StageResult.from_c(r)
        if rc is not None and res.dropped > 0:
            rc.note_overflow()
        return out, res

    def _host_args(self, vertices, out, n):
        def hp(name, src):
            a = src.get(name)
            return a.ctypes.data if a is not None else None
        soa = _capi.VertexSoA(hp("p01", vertices), hp("wo01", vertices), hp("roughness", vertices),
                              hp("weight", vertices), hp("i_pixel", vertices), hp("path_key", vertices), None, None)
        oc = _capi.StageOut(hp("q_norm", out), hp("q_real", out), hp("slots", out), hp("k", out), hp("offset", out),
                            hp("decided", out), hp("q_orig", out), hp("u", out))
        return soa, oc

    def submit_host(self, vertices: Dict[str, np.ndarray], depth: int, strategy: Strategy, gain: float = 1.0,
                    eps_div: float = 0.0, out: Optional[Dict[str, np.ndarray]] = None):
        """Asynchronous host-buffer stage (nrrs_gpu_rrs_stage_host_async) for a stream of independent
        batches: returns (ticket, out).  Two calls may be in flight; keep `vertices` and `out` alive
        (pinned) until wait_host(ticket).  out["slots"] receives all `capacity` records."""
        n = int(vertices["roughness"].shape[0]) if "roughness" in vertices else vertices["p01"].size // 3
        if out is None:
            out = {"q_norm": np.empty(n, np.float32), "q_real": np.empty(n, np.float32),
                   "slots": np.empty((self.capacity, 2), np.uint32)}
        p = self.params(depth, strategy, gain, eps_div)
        soa, oc = self._host_args(vertices, out, n)
        t = C.c_uint64(0)
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_rrs_stage_host_async(self.handle, C.byref(soa), n, C.byref(p),
                                                                            C.byref(oc), C.byref(t)))
        return int(t.value), out

    def wait_host(self, ticket: int) -> "StageResult":
        r = _capi.StageResultC()
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_stage_host_wait(self.handle, int(ticket), C.byref(r)))
        return StageResult.from_c(r)

    def compact(self, records: torch.Tensor, used: torch.Tensor, count: int, out: torch.Tensor,
                d_count: Optional[torch.Tensor] = None, sync: bool = True) -> Optional[int]:
        """Order-preserving compaction of filled slots (wavefront.cpp:488-497).
        records: [>=count, W] int32 (W = 2 slot records or 18 = 72-byte PathState)."""
        words = int(records.shape[1])
        hc = C.c_uint32(0)
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_compact(
            self.handle, records.data_ptr(), used.data_ptr(), int(count), words, out.data_ptr(),
            d_count.data_ptr() if d_count is not None else None, C.byref(hc) if sync else None))
        return hc.value if sync else None

    def strategy_factor(self, vertices: Dict[str, torch.Tensor], strategy: Strategy, eps_div: float = 0.0):
        """Batched strategy_factor (wavefront.cpp:186-215) without sanitize/normalize."""
        n = vertices["p01"].numel() // 3
        q = torch.empty(n, dtype=torch.float32, device=self.device)
        soa = vertex_soa(vertices)
        s = strategy.c()
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_strategy_factor(self.handle, C.byref(soa), n, C.byref(s),
                                                                       float(eps_div), q.data_ptr()))
        return q

    def predict_stats(self, vertices: Dict[str, torch.Tensor]) -> torch.Tensor:
        """Batched NeuralRrs::predict_stats (networks.cpp:252-264): [n, 6] = mean(3), m2(3)."""
        n = vertices["p01"].numel() // 3
        st = torch.empty((n, 6), dtype=torch.float32, device=self.device)
        soa = vertex_soa(vertices)
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_predict_stats(self.handle, C.byref(soa), n, st.data_ptr()))
        return st

    def encode_levels(self, p01: torch.Tensor) -> torch.Tensor:
        """Batched HashGrid::encode (hashgrid.cpp:38-82) of the AID RRSNet grid through K-A0:
        [levels, n, 2] level planes (fp16 tables staged in shared memory)."""
        n = p01.numel() // 3
        levels = self.nets.cfg.grid.levels if self.nets is not None else 0
        planes = torch.empty((levels, n, 2), dtype=torch.float32, device=self.device)
        _capi.check(self.handle, self.ctx.lib.nrrs_gpu_encode_levels(self.handle, p01.data_ptr(), n,
                                                                     planes.data_ptr(), n))
        return planes

    def close(self) -> None:
        self.ctx.close()


def strategy_for_depth(assignment, depth: int) -> Strategy:
    """Mix-Depth gate: entry d-1 governs depth d (wavefront.cpp:366)."""
    return assignment[depth - 1]


__all__ = ["RrsStage", "StageResult", "StageOutputs", "GpuContext", "default_context", "vertex_soa",
           "strategy_for_depth", "StrategyKind"]
