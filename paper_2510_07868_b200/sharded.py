"""Tile-sharded RRS stage across ranks.

Each rank owns a contiguous band of the image (rank order == pixel order), so
the global depth-d queue is the concatenation of the rank queues.  Per depth
the path has exactly two real exchange steps, both 8 bytes per rank:

  1. all-gather of the per-rank sum of sanitized factors (f64); every rank
     sums them in rank order, so F_norm = Npx_total / sum is identical on all
     ranks (normalization is global per depth, rrs.cpp:8-24; image-partition
     local normalization is a non-goal).
  2. all-gather of the per-rank realized totals (u64); the exclusive prefix in
     rank order is the rank's global slot base and the capacity clip of the
     global tail (wavefront.cpp:141-154) becomes a count truncation of the
     rank's records.  Overflow is a global event, so RateControl stays
     replicated.

The protocol functions take the phase callables as arguments so the host logic
is testable on CPU ranks (gloo); the product binds them to the C ABI.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

from . import _capi
from .rrs import ADRRS_EPS_SCALE, RateControl, Strategy, eps_div_from_luminance_sum
from .stage import RrsStage, StageOutputs, vertex_soa


@dataclasses.dataclass
class ShardOutcome:
    rank_sums: List[float]
    rank_totals: List[int]
    base: int           # global slot index of this rank's first record
    kept: int           # records this rank keeps after the global clip
    spawned: int        # global SpawnPlan::spawned
    dropped: int        # global SpawnPlan::dropped
    f_norm: float


def global_clip(totals: List[int], rank: int, capacity: int):
    """nrrs_gpu_sharded_clip: (base, kept, spawned_global, dropped_global)."""
    arr = (C.c_uint64 * len(totals))(*totals)
    base, kept, sp, dr = C.c_uint64(0), C.c_uint32(0), C.c_uint32(0), C.c_uint64(0)
    rc = _capi.lib().nrrs_gpu_sharded_clip(arr, len(totals), rank, capacity, C.byref(base), C.byref(kept),
                                           C.byref(sp), C.byref(dr))
    if rc:
        raise _capi.NrrsError(rc, "sharded_clip: invalid arguments")
    return base.value, kept.value, sp.value, dr.value


def f_norm_from_sums(rank_sums: List[float], n_pixels_total: int) -> float:
    s = 0.0
    for x in rank_sums:  # rank order
        s += x
    return 1.0 if s <= 0.0 else float(n_pixels_total) / s


# ---- exact rank sums (nrrs_gpu_stage_local_sum_exact): the stage's 128-bit fixed-point sum as two
# int64 words (lo, hi), value = hi * 2^24 + lo * 2^-40 (bit-exactness) ----
_U64 = (1 << 64) - 1


def fx_to_float(lo: int, hi: int) -> float:
    """The device's fx_to_double: float(hi) * 2^24 + float(lo) * 2^-40 (the same two roundings)."""
    return float(hi & _U64) * 16777216.0 + float(lo & _U64) * 9.094947017729282e-13


def exact_rank_floats(t: torch.Tensor) -> List[float]:
    w = [int(x) for x in t.reshape(-1).tolist()]
    return [fx_to_float(w[2 * r], w[2 * r + 1]) for r in range(len(w) // 2)]


def f_norm_from_exact(t: torch.Tensor, n_pixels_total: int) -> float:
    """F from the all-gathered exact rank sums, added exactly (decide3's rank_sums_fx path)."""
    w = [int(x) & _U64 for x in t.reshape(-1).tolist()]
    total = sum((w[2 * r + 1] << 64) | w[2 * r] for r in range(len(w) // 2)) & ((1 << 128) - 1)
    s = fx_to_float(total & _U64, total >> 64)
    return 1.0 if s <= 0.0 else float(n_pixels_total) / s


class _CudaWords:
    """__cuda_array_interface__ of a device address (zero-copy torch view)."""

    def __init__(self, addr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (addr, False), "version": 3}


def exact_sum_view(stage: RrsStage) -> torch.Tensor:
    """[2] int64 view of the context's exact sum of q (nrrs_gpu_stage_sum_exact_dev), current after
    every nrrs_gpu_stage_factors on that context's stream."""
    ptr = C.c_void_p()
    _capi.check(stage.handle, stage.ctx.lib.nrrs_gpu_stage_sum_exact_dev(stage.handle, C.byref(ptr)))
    return torch.as_tensor(_CudaWords(ptr.value, 2), device=stage.device)


def _outcome_sums(rank_sums_t: torch.Tensor, n_pixels_total: int):
    """(per-rank floats, F) for f64 rank sums or exact (int64 word pair) rank sums."""
    if rank_sums_t.dtype == torch.int64:
        return exact_rank_floats(rank_sums_t), f_norm_from_exact(rank_sums_t, n_pixels_total)
    sums_h = [float(x) for x in rank_sums_t.tolist()]
    return sums_h, f_norm_from_sums(sums_h, n_pixels_total)


def sharded_depth(local_sum: torch.Tensor, decide: Callable[[torch.Tensor], torch.Tensor], capacity: int,
                  n_pixels_total: int, group=None, rc: Optional[RateControl] = None,
                  after_exchange: Optional[Callable[[], None]] = None) -> ShardOutcome:
    """Runs the two exchanges of one depth.  local_sum: [1] float64, or the exact sum as [2] int64
    words (nrrs_gpu_stage_local_sum_exact), on the collective's device; decide(rank_sums) launches phase 2 and returns the
    rank's [1] int64 realized total.  after_exchange() (optional) is called once
    the second exchange is issued and before the host reads its result: device
    work that needs only this rank's queue (e.g. its compaction) is queued
    there, so the GPU does not idle through the host round trip."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    host = dist.get_backend(group) == "gloo" and local_sum.is_cuda  # gloo exchanges host copies
    src = local_sum.cpu() if host else local_sum
    sums = [torch.zeros_like(src) for _ in range(world)]
    dist.all_gather(sums, src, group=group)
    rank_sums_t = torch.cat(sums).to(local_sum.device)
    local_total = decide(rank_sums_t)
    src = local_total.cpu() if host else local_total
    totals = [torch.zeros_like(src) for _ in range(world)]
    dist.all_gather(totals, src, group=group)
    if after_exchange is not None:
        after_exchange()
    tot = [int(x) for x in torch.cat(totals).tolist()]  # the one host wait of the depth
    sums_h, f_norm = _outcome_sums(rank_sums_t, n_pixels_total)
    base, kept, spawned, dropped = global_clip(tot, rank, capacity)
    if rc is not None and dropped > 0:
        rc.note_overflow()
    return ShardOutcome(sums_h, tot, base, kept, spawned, dropped, f_norm)


@dataclasses.dataclass
class PendingDepth:
    """A depth of the sharded protocol whose scalars are still on the device."""
    rank_sums: torch.Tensor   # [world] f64, rank order
    rank_totals: torch.Tensor  # [world] i64, rank order
    clip: Optional[torch.Tensor]  # [4] i64: base, kept, spawned, dropped (None on the host-exchange path)
    n_pixels_total: int
    capacity: int
    rank: int
    check: Optional[Callable[[], None]] = None  # mailbox mode: raises if a peer wait timed out

    def resolve(self, rc: Optional[RateControl] = None) -> ShardOutcome:
        """Reads the depth's scalars (one host wait) and applies the overflow to RateControl."""
        if self.check is not None:
            self.check()
        tot = [int(x) for x in self.rank_totals.tolist()]
        sums_h, f_norm = _outcome_sums(self.rank_sums, self.n_pixels_total)
        if self.clip is not None:
            base, kept, spawned, dropped = (int(x) for x in self.clip.tolist())
        else:
            base, kept, spawned, dropped = global_clip(tot, self.rank, self.capacity)
        if rc is not None and dropped > 0:
            rc.note_overflow()
        return ShardOutcome(sums_h, tot, base, kept, spawned, dropped, f_norm)


def _all_gather_flat(x: torch.Tensor, host: bool, group=None) -> torch.Tensor:
    """[1] per rank -> [world] in rank order: one all_gather_into_tensor on NCCL (no list copies),
    the list form on gloo (host copies)."""
    world = dist.get_world_size(group)
    if not host and x.is_cuda and dist.get_backend(group) == "nccl":
        out = torch.empty(world * x.numel(), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(out, x.reshape(-1), group=group)
        return out
    src = x.cpu() if host else x
    parts = [torch.zeros_like(src) for _ in range(world)]
    dist.all_gather(parts, src, group=group)
    return torch.cat(parts)


def sharded_depth_async(local_sum: torch.Tensor, decide: Callable[[torch.Tensor], torch.Tensor], capacity: int,
                        n_pixels_total: int, stage: Optional[RrsStage] = None, group=None,
                        after_exchange: Optional[Callable[[torch.Tensor], None]] = None,
                        after_decide: Optional[Callable[[], None]] = None) -> PendingDepth:
    """sharded_depth without the host wait: the global clip runs on the device
    (nrrs_gpu_sharded_clip_dev on `stage`'s context stream) when the collective's tensors live on
    the GPU, so consecutive depths queue back to back.  after_exchange(clip) receives the [4]
    device tensor (kept = clip[1]) or None on the gloo host-exchange path.  The caller reads the
    scalars with PendingDepth.resolve(rc) when it needs them; RateControl sees the overflow then."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    host = dist.get_backend(group) == "gloo" and local_sum.is_cuda
    rank_sums_t = _all_gather_flat(local_sum, host, group).to(local_sum.device)
    local_total = decide(rank_sums_t)
    if after_decide is not None:  # work on this rank's queue only (its compaction) goes ahead of the exchange
        after_decide()
    totals_t = _all_gather_flat(local_total, host, group)
    clip = None
    if not host and stage is not None and totals_t.is_cuda:
        clip = torch.empty(4, dtype=torch.int64, device=totals_t.device)
        _capi.check(stage.handle, stage.ctx.lib.nrrs_gpu_sharded_clip_dev(stage.handle, totals_t.data_ptr(), world,
                                                                          rank, int(capacity), clip.data_ptr()))
    if after_exchange is not None:
        after_exchange(clip)
    return PendingDepth(rank_sums_t, totals_t, clip, n_pixels_total, capacity, rank)


# ---- mailbox mode: the two per-depth exchanges inside the kernels, over peer memory ----------
IPC_HANDLE_BYTES = 64  # NRRS_IPC_HANDLE_BYTES


def mailbox_init(stage: RrsStage, world: int, rank: int) -> Tuple[bytes, int]:
    """nrrs_gpu_mailbox_init: allocates the rank's mailbox; returns (CUDA IPC handle, device address)."""
    h = (C.c_uint8 * IPC_HANDLE_BYTES)()
    addr = C.c_uint64(0)
    _capi.check(stage.handle, stage.ctx.lib.nrrs_gpu_mailbox_init(stage.handle, world, rank, h, C.byref(addr)))
    return bytes(h), addr.value


def mailbox_connect(stage: RrsStage, handles: Sequence[bytes], same_process_addrs: Sequence[int]) -> None:
    """nrrs_gpu_mailbox_connect: maps every rank's mailbox (IPC handles in rank order; a nonzero
    same-process address is used directly)."""
    world = len(handles)
    buf = (C.c_uint8 * (IPC_HANDLE_BYTES * world)).from_buffer_copy(b"".join(handles))
    addrs = (C.c_uint64 * world)(*same_process_addrs)
    _capi.check(stage.handle, stage.ctx.lib.nrrs_gpu_mailbox_connect(stage.handle, buf, addrs))


def mailbox_check(stage: RrsStage) -> None:
    """Raises if a mailbox wait of this context gave up on a peer (nrrs_gpu_mailbox_status)."""
    t = C.c_int32(0)
    _capi.check(stage.handle, stage.ctx.lib.nrrs_gpu_mailbox_status(stage.handle, C.byref(t)))
    if t.value:
        raise RuntimeError("mailbox exchange timed out: a rank did not publish this depth (all ranks must run "
                           "the same sequence of depths)")


def connect_mailboxes_in_process(stages: Sequence[RrsStage]) -> None:
    """All ranks in ONE process (one RrsStage per rank, e.g. a functional check): mailboxes are
    connected through their device addresses, no IPC."""
    world = len(stages)
    infos = [mailbox_init(st, world, r) for r, st in enumerate(stages)]
    for st in stages:
        mailbox_connect(st, [h for h, _ in infos], [a for _, a in infos])


def mailbox_depth(stage: RrsStage, n: int, p, out: StageOutputs, local_total: torch.Tensor, world: int, rank: int,
                  capacity: int, n_pixels_total: int,
                  after_exchange: Optional[Callable[[torch.Tensor], None]] = None,
                  after_decide: Optional[Callable[[], None]] = None) -> PendingDepth:
    """Phase 2 of a depth in mailbox mode (phase 1, nrrs_gpu_stage_factors, already published the
    rank's sum): decide with the rank sums from the mailbox, then the global clip from the
    mailboxed totals, both on the device with no collective and no host wait.  after_decide()
    (optional) queues work that needs only this rank's queue (its compaction) right behind the
    decision kernel, ahead of the clip's wait for the other ranks."""
    lib = stage.ctx.lib
    oc = out.c()
    _capi.check(stage.handle, lib.nrrs_gpu_stage_decide_mbox(stage.handle, n, C.byref(p), C.byref(oc),
                                                             local_total.data_ptr()))
    if after_decide is not None:
        after_decide()
    dev = local_total.device
    clip = torch.empty(4, dtype=torch.int64, device=dev)
    sums = torch.empty(world, dtype=torch.float64, device=dev)
    tots = torch.empty(world, dtype=torch.int64, device=dev)
    _capi.check(stage.handle, lib.nrrs_gpu_sharded_clip_mbox(stage.handle, int(capacity), clip.data_ptr(),
                                                             sums.data_ptr(), tots.data_ptr()))
    if after_exchange is not None:
        after_exchange(clip)
    return PendingDepth(sums, tots, clip, n_pixels_total, capacity, rank, check=lambda: mailbox_check(stage))


def _gather_in_rank_order(local: torch.Tensor, group=None) -> torch.Tensor:
    host = dist.get_backend(group) == "gloo" and local.is_cuda  # gloo exchanges host copies
    src = local.cpu() if host else local
    parts = [torch.zeros_like(src) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, src, group=group)
    return torch.cat(parts)


def sharded_eps_div(local_lum_sum: torch.Tensor, n_pixels_total: int, eps_scale: float = ADRRS_EPS_SCALE,
                    group=None) -> float:
    """Per-frame exchange of SURVEY.md 8e: each rank's f64 sum of luminance(i_acc) over its
    band, gathered and summed in rank order (the reference sums the film in pixel order,
    wavefront.cpp:238-243), so every rank derives the same eps_div."""
    total = 0.0
    for x in _gather_in_rank_order(local_lum_sum.reshape(1).to(torch.float64), group).tolist():
        total += x
    return eps_div_from_luminance_sum(total, n_pixels_total, eps_scale)


def row_band(rank: int, world: int, height: int):
    """Contiguous pixel-row band [row0, row1) of `rank` (rank order == row order, as even as
    possible), the partition that keeps the global queue the concatenation of the rank queues."""
    return height * rank // world, height * (rank + 1) // world


def gather_film(band: torch.Tensor, dst: int = 0, group=None) -> Optional[torch.Tensor]:
    """Per-frame film exchange of SURVEY.md 8e: each rank's band of f64 film rows ([px_band, ...],
    pixel order) is gathered to rank `dst` in rank order, which is pixel order for row bands --
    a gather (one collective, only `dst` receives), not an all-gather.  Bands may differ in size:
    their lengths are exchanged first (8 bytes per rank) and each band is padded to the largest.
    Returns the full film on `dst`, None elsewhere."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    host = dist.get_backend(group) == "gloo" and band.is_cuda
    src = band.cpu() if host else band
    n_local = torch.tensor([src.shape[0]], dtype=torch.int64, device=src.device)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    sizes = [int(x.item()) for x in sizes]
    rows = max(sizes)
    pad = src
    if src.shape[0] != rows:
        pad = torch.zeros((rows,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
        pad[:src.shape[0]] = src
    parts = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad.contiguous(), gather_list=parts, dst=dst, group=group)
    if rank != dst:
        return None
    full = torch.cat([p[:k] for p, k in zip(parts, sizes)])
    return full.to(band.device)


def broadcast_weights(nets, src: int = 0, group=None, device=None):
    """Per publish() exchange of SURVEY.md 8e: rank `src`'s snapshot blocks (stat grid, stat MLP,
    rrs grid for AID, rrs MLP; networks.cpp:199-204) are broadcast to every rank.  On NCCL the
    blocks stay on the GPU (returns the four device tensors for ShardedRrsStage.set_weights ->
    nrrs_gpu_set_weights_dev, no host round trip); on gloo they are host tensors and `nets` is
    updated in place.  Returns the list of the four broadcast tensors."""
    nccl = dist.get_backend(group) == "nccl"
    out = []
    for name in ("stat_grid", "stat_mlp", "rrs_grid", "rrs_mlp"):
        a = getattr(nets, name)
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
        if nccl:
            t = t.to(device if device is not None else torch.device("cuda", torch.cuda.current_device()))
        if t.numel():
            dist.broadcast(t, src=src, group=group)
        if not nccl:
            setattr(nets, name, t.numpy().astype(np.float32, copy=False))
        out.append(t)
    return out


class ShardedRrsStage:
    """One rank of the tile-sharded stage (one GPU per process, NCCL over NVLink).

    exchange="collective" (default): the two per-depth exchanges are torch.distributed
    all-gathers.  exchange="mailbox": they run inside the stage kernels over peer memory
    (CUDA IPC mappings of every rank's mailbox, NVLink / NVSwitch); the handles are exchanged
    once here over the process group."""

    def __init__(self, n_pixels_total: int, nets=None, capacity: int = 0, seed: int = 0, device: int = 0,
                 group=None, exchange: str = "collective"):
        if exchange not in ("collective", "mailbox"):
            raise ValueError(f"exchange must be 'collective' or 'mailbox', got {exchange!r}")
        self.stage = RrsStage(n_pixels_total, nets, capacity=capacity, seed=seed, device=device)
        self.n_pixels_total = int(n_pixels_total)
        self.capacity = self.stage.capacity
        self.group = group
        self.device = self.stage.device
        self.exchange = exchange
        self._sum = torch.zeros(1, dtype=torch.float64, device=self.device)
        self._sum_fx = exact_sum_view(self.stage)  # the context's exact sum (lo, hi): exchanged without a copy
        self._total = torch.zeros(1, dtype=torch.int64, device=self.device)
        if exchange == "mailbox":
            world, rank = dist.get_world_size(group), dist.get_rank(group)
            h, addr = mailbox_init(self.stage, world, rank)
            infos = [None] * world
            dist.all_gather_object(infos, (h, addr, os.getpid()), group=group)
            mailbox_connect(self.stage, [i[0] for i in infos],
                            [i[1] if i[2] == os.getpid() else 0 for i in infos])

    def depth_async(self, n: int, depth: int, strategy: Strategy, out: StageOutputs, gain: float = 1.0,
                    eps_div: float = 0.0,
                    after_exchange: Optional[Callable[[torch.Tensor], None]] = None,
                    after_decide: Optional[Callable[[], None]] = None) -> PendingDepth:
        """Phase 2 of a depth after factors(): the exchanges (collective or mailbox), the decision
        and the device-side global clip, without a host wait."""
        if self.exchange == "mailbox":
            p = self.stage.params(depth, strategy, gain, eps_div, n_pixels=self.n_pixels_total)
            return mailbox_depth(self.stage, n, p, out, self._total, dist.get_world_size(self.group),
                                 dist.get_rank(self.group), self.capacity, self.n_pixels_total, after_exchange,
                                 after_decide)
        return sharded_depth_async(self._sum_fx, lambda rs: self.decide(n, depth, strategy, out, rs, gain, eps_div),
                                   self.capacity, self.n_pixels_total, self.stage, self.group, after_exchange,
                                   after_decide)

    def factors(self, vertices, depth: int, strategy: Strategy, out: StageOutputs, eps_div: float = 0.0,
                gain: float = 1.0) -> torch.Tensor:
        st = self.stage
        st.ctx.bind_stream()
        n = vertices["p01"].numel() // 3
        p = st.params(depth, strategy, gain, eps_div, n_pixels=self.n_pixels_total)
        soa = vertex_soa(vertices)
        oc = out.c()
        _capi.check(st.handle, st.ctx.lib.nrrs_gpu_stage_factors(st.handle, C.byref(soa), n, C.byref(p),
                                                                 C.byref(oc), self._sum.data_ptr()))
        # the exact 128-bit sum (a view of the context's words) is what the ranks exchange: F is then
        # the one-rank F bit for bit
        return self._sum_fx

    def decide(self, n: int, depth: int, strategy: Strategy, out: StageOutputs, rank_sums: torch.Tensor,
               gain: float = 1.0, eps_div: float = 0.0) -> torch.Tensor:
        st = self.stage
        p = st.params(depth, strategy, gain, eps_div, n_pixels=self.n_pixels_total)
        oc = out.c()
        rs = rank_sums.contiguous()
        if rs.dtype == torch.int64:  # exact rank sums (2 words per rank), added exactly
            _capi.check(st.handle, st.ctx.lib.nrrs_gpu_stage_decide_exact(st.handle, n, C.byref(p), rs.data_ptr(),
                                                                          rs.numel() // 2, C.byref(oc),
                                                                          self._total.data_ptr()))
        else:
            _capi.check(st.handle, st.ctx.lib.nrrs_gpu_stage_decide(st.handle, n, C.byref(p), rs.data_ptr(),
                                                                    rs.numel(), C.byref(oc), self._total.data_ptr()))
        return self._total

    def eps_div(self, i_acc_band: torch.Tensor, eps_scale: float = ADRRS_EPS_SCALE) -> float:
        """Global per-frame ADRRS divisor guard from this rank's band of the film."""
        return sharded_eps_div(self.stage.film_luminance_sum(i_acc_band), self.n_pixels_total, eps_scale,
                               self.group)

    def set_weights(self, nets, src: int = 0) -> None:
        """Per publish(): broadcast rank `src`'s snapshot and upload it on every rank (NCCL: the
        broadcast blocks never leave the GPU, nrrs_gpu_set_weights_dev)."""
        blocks = broadcast_weights(nets, src, self.group, device=self.device)
        if dist.get_backend(self.group) == "nccl":
            self.stage.set_weights_device(nets, blocks)
        else:
            self.stage.set_weights(nets)

    def run(self, vertices, depth: int, strategy: Strategy, rc: Optional[RateControl] = None,
            eps_div: float = 0.0, out: Optional[StageOutputs] = None):
        n = vertices["p01"].numel() // 3
        out = out or self.stage.alloc_outputs(n)
        gain = rc.gain() if rc is not None else 1.0
        if self.stage.capacity and out.q_orig is None:
            out.q_orig = torch.empty(n, dtype=torch.float32, device=self.device)
            out.u = torch.empty(n, dtype=torch.float32, device=self.device)
        local = self.factors(vertices, depth, strategy, out, eps_div, gain)
        if self.exchange == "mailbox":
            return out, self.depth_async(n, depth, strategy, out, gain, eps_div).resolve(rc)
        outcome = sharded_depth(local, lambda rs: self.decide(n, depth, strategy, out, rs, gain, eps_div),
                                self.capacity, self.n_pixels_total, self.group, rc)
        return out, outcome
