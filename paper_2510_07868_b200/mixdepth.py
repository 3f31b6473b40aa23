"""Mix-Depth strategy search: brute-force and segmented search over per-depth
strategy assignments, with the probe renders run as GPU trace_frame replicas.

Mirrors `mixdepth.hpp` / `mixdepth.cpp` (probe_score :75-77, search_segment :27-57, brute_force_search
:79-94, heuristic_search :96-118, the CSV log :59-68) and the probe of `run_search` (runner.cpp:396-461:
one frame at a fixed post-training frame index with a fresh film seeded by the trained pixel estimate,
scored by relmse against a reference image, metrics.cpp:5-20).

Multi-GPU: the probes of one segment are independent renders, so `search_segment` shards them across
ranks (probe i on rank i mod N) and all-gathers the outcomes; every rank then takes the same
lexicographic argmin, so the result and the log equal the sequential search's.  Segments stay
sequential because a segment's frozen prefix is the previous segment's winner.
"""
from __future__ import annotations

import enum
import math
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np
import torch

from .rrs import RateControl, Strategy, StrategyKind, assignment_name


class ScoreMode(enum.IntEnum):
    """mixdepth.hpp:16-19."""
    RelMseTime = 0
    RelMseOnly = 1


@dataclass
class ProbeOutcome:
    """mixdepth.hpp:22-26."""
    relmse: float = 0.0
    rays: int = 0
    seconds: float = 0.0


@dataclass
class SearchLogRow:
    assignment: List[Strategy]
    score: float
    rays: int
    seconds: float


@dataclass
class SearchOptions:
    """mixdepth.hpp:40-46 (same defaults)."""
    max_depth: int = 6
    segment_depth: int = 6
    brute_cap: int = 729
    score: ScoreMode = ScoreMode.RelMseTime
    log_path: str = ""


@dataclass
class SearchResult:
    best: List[Strategy] = field(default_factory=list)
    best_score: float = 0.0
    probes: int = 0
    log: List[SearchLogRow] = field(default_factory=list)


ProbeFn = Callable[[List[Strategy]], ProbeOutcome]


def probe_score(outcome: ProbeOutcome, mode: ScoreMode) -> float:
    """mixdepth.cpp:75-77."""
    return outcome.relmse * outcome.seconds if mode == ScoreMode.RelMseTime else outcome.relmse


def combination_count(n_strategies: int, width: int) -> int:
    """mixdepth.cpp:11-19 (saturates past 2^48)."""
    total = 1
    for _ in range(width):
        if total > (1 << 48):
            return (1 << 64) - 1
        total *= n_strategies
    return total


def _combos(n: int, width: int):
    """Odometer order with the last digit fastest (lexicographic ascending)."""
    idx = [0] * width
    while True:
        yield list(idx)
        k = width - 1
        while k >= 0:
            idx[k] += 1
            if idx[k] < n:
                break
            idx[k] = 0
            k -= 1
        if k < 0:
            return


def search_segment(strategies: Sequence[Strategy], probe: ProbeFn, mode: ScoreMode, assignment: List[Strategy],
                   begin: int, end: int, result: SearchResult, group=None) -> float:
    """mixdepth.cpp:27-57; with a torch.distributed group the probes are sharded across its ranks."""
    width = end - begin
    combos = list(_combos(len(strategies), width))
    assigns = []
    for idx in combos:
        a = list(assignment)
        for k in range(width):
            a[begin + k] = strategies[idx[k]]
        assigns.append(a)
    world, rank = 1, 0
    if group is not None or (torch.distributed.is_available() and torch.distributed.is_initialized()):
        world = torch.distributed.get_world_size(group)
        rank = torch.distributed.get_rank(group)
    outcomes: List[Optional[ProbeOutcome]] = [None] * len(assigns)
    local = np.zeros((len(assigns), 3), np.float64)
    for i in range(rank, len(assigns), world):
        o = probe(assigns[i])
        outcomes[i] = o
        local[i] = (o.relmse, float(o.rays), o.seconds)
    if world > 1:
        # each probe is owned by exactly one rank: a sum of the zero-padded tables gathers them
        t = torch.from_numpy(local)
        if torch.distributed.get_backend(group) == "nccl":
            t = t.cuda()
        torch.distributed.all_reduce(t, group=group)
        allv = t.cpu().numpy()
        for i in range(len(assigns)):
            if outcomes[i] is None:
                outcomes[i] = ProbeOutcome(float(allv[i, 0]), int(round(allv[i, 1])), float(allv[i, 2]))
    best, best_i = math.inf, -1
    for i, (a, o) in enumerate(zip(assigns, outcomes)):
        score = probe_score(o, mode)
        if not math.isfinite(score):
            raise RuntimeError("mix-depth search: probe returned a non-finite score for assignment "
                               + assignment_name(a))
        result.log.append(SearchLogRow(a, score, o.rays, o.seconds))
        result.probes += 1
        if best_i < 0 or score < best:  # ties keep the earliest (lexicographically smallest)
            best, best_i = score, i
    for k in range(width):
        assignment[begin + k] = assigns[best_i][begin + k]
    return best


def write_search_log(path: str, log: List[SearchLogRow]) -> None:
    """mixdepth.cpp:59-68: one quoted assignment per row; numbers like std::ostream (%g)."""
    try:
        with open(path, "w", newline="") as f:
            f.write("assignment,score,rays,seconds\n")
            for row in log:
                f.write(f'"{assignment_name(row.assignment)}",{row.score:g},{row.rays},{row.seconds:g}\n')
    except OSError as e:
        raise RuntimeError(f"mix-depth search: cannot write log: {path}") from e


def _check_inputs(strategies, probe, opt: SearchOptions) -> None:
    if not strategies:
        raise RuntimeError("mix-depth search: empty strategy candidate list")
    if opt.max_depth < 1:
        raise RuntimeError("mix-depth search: max_depth must be at least 1")
    if probe is None:
        raise RuntimeError("mix-depth search: missing probe function")


def brute_force_search(strategies: Sequence[Strategy], probe: ProbeFn, opt: SearchOptions,
                       group=None) -> SearchResult:
    """mixdepth.cpp:79-94."""
    _check_inputs(strategies, probe, opt)
    combos = combination_count(len(strategies), opt.max_depth)
    if combos > opt.brute_cap:
        raise RuntimeError(f"brute_force_search: {len(strategies)}^{opt.max_depth} combinations exceed the cap of "
                           f"{opt.brute_cap}; use heuristic_search")
    r = SearchResult(best=[strategies[0]] * opt.max_depth)
    r.best_score = search_segment(strategies, probe, opt.score, r.best, 0, opt.max_depth, r, group)
    if opt.log_path:
        write_search_log(opt.log_path, r.log)
    return r


def heuristic_search(strategies: Sequence[Strategy], probe: ProbeFn, opt: SearchOptions,
                     group=None) -> SearchResult:
    """mixdepth.cpp:96-118: fixed RR 1.0 everywhere, then segments of width T_d front to back."""
    _check_inputs(strategies, probe, opt)
    if opt.segment_depth < 1 or opt.segment_depth > opt.max_depth:
        raise RuntimeError("heuristic_search: segment_depth must satisfy 1 <= T_d <= max_depth")
    r = SearchResult(best=[Strategy(StrategyKind.Fixed, 1.0)] * opt.max_depth)
    score = math.inf
    for begin in range(0, opt.max_depth, opt.segment_depth):
        end = min(begin + opt.segment_depth, opt.max_depth)
        score = search_segment(strategies, probe, opt.score, r.best, begin, end, r, group)
    r.best_score = score
    if opt.log_path:
        write_search_log(opt.log_path, r.log)
    return r


def relmse(image: torch.Tensor, reference: torch.Tensor, eps: float = 0.01) -> float:
    """metrics.cpp:5-20 in f64: mean over pixels and channels of (I - R)^2 / (R^2 + eps)."""
    if image.numel() == 0:
        raise RuntimeError("relmse: empty image")
    if image.shape != reference.shape:
        raise RuntimeError(f"relmse: dimension mismatch: {image.shape[0]} vs {reference.shape[0]} pixels")
    r = reference.to(torch.float64)
    d = image.to(torch.float64) - r
    return float((d * d / (r * r + eps)).sum().item() / (3.0 * image.shape[0]))


class GpuProbe:
    """The probe of run_search (runner.cpp:414-434) on one GPU: one trace_frame with a fresh film
    whose i_acc / normal are the trained film's, RateControl(enabled, f_rate) fresh per probe, a
    fixed frame index, scored against `reference` ([W*H, 3] f32 on the device)."""

    def __init__(self, tracer, width: int, height: int, reference: torch.Tensor, i_acc: torch.Tensor,
                 normal: Optional[torch.Tensor] = None, frame_index: int = 0, seed: int = 0,
                 rate_control: bool = True, f_rate: float = 0.85, deterministic: bool = False,
                 adrrs_eps_scale: float = 1e-4):
        from .film import GpuFilm, SuffixStage
        self.tracer = tracer
        self.width, self.height = width, height
        self.reference = reference
        self.film = GpuFilm(width, height, SuffixStage(ctx=tracer.ctx))
        self.i_acc0 = i_acc.clone()
        self.normal0 = normal.clone() if normal is not None else None
        self.frame_index, self.seed = frame_index, seed
        self.rate_control, self.f_rate = rate_control, f_rate
        self.deterministic = deterministic
        self.adrrs_eps_scale = adrrs_eps_scale

    def __call__(self, assignment: List[Strategy]) -> ProbeOutcome:
        from .render import TraceConfig
        f = self.film
        f.sum.zero_()
        f.samples.zero_()
        f.i_cur.zero_()
        f.i_acc.copy_(self.i_acc0)
        if self.normal0 is not None:
            f.normal.copy_(self.normal0)
        rc = RateControl(f_rate=self.f_rate, enabled=self.rate_control)
        cfg = TraceConfig(max_depth=len(assignment), seed=self.seed, frame_index=self.frame_index,
                          adrrs_eps_scale=self.adrrs_eps_scale)
        torch.cuda.synchronize(self.film.sum.device)
        t0 = time.perf_counter()
        rep, _ = self.tracer.trace_frame(assignment, cfg, rc, f)
        torch.cuda.synchronize(self.film.sum.device)
        dt = time.perf_counter() - t0
        return ProbeOutcome(relmse(f.mean_image(), self.reference), rep.camera_rays + rep.scatter_rays +
                            rep.shadow_rays, 0.0 if self.deterministic else dt)


__all__ = ["ScoreMode", "ProbeOutcome", "SearchLogRow", "SearchOptions", "SearchResult", "assignment_name",
           "probe_score", "combination_count", "search_segment", "write_search_log", "brute_force_search",
           "heuristic_search", "relmse", "GpuProbe"]
