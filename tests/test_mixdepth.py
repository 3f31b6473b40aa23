"""Mix-Depth search on frozen-score probes, mirroring the reference's
test_mixdepth.cpp case by case, plus the rank-sharded segment search (gloo, world 2) against the
sequential search."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle as orc
from paper_2510_07868_b200.mixdepth import (ProbeOutcome, ScoreMode, SearchOptions, brute_force_search,
                                            heuristic_search, probe_score, relmse)
from paper_2510_07868_b200.rrs import Strategy, StrategyKind


def same(a: Strategy, b: Strategy) -> bool:
    return a.kind == b.kind and (a.kind != StrategyKind.Fixed or a.fixed_value == b.fixed_value)


def combo_index(a, sset) -> int:
    idx = 0
    for s in a:
        k = next(i for i, c in enumerate(sset) if same(c, s))
        idx = idx * len(sset) + k
    return idx


FIXED1 = Strategy(StrategyKind.Fixed, 1.0)
TP = Strategy(StrategyKind.Throughput)
NR = Strategy(StrategyKind.Nrrs)
SCORES8 = [0.82, 0.47, 0.93, 0.31, 0.55, 0.62, 0.44, 0.39]


def test_brute_force_exhaustive_minimum():
    """test_mixdepth.cpp:58-88."""
    sset = [FIXED1, TP]
    r = brute_force_search(sset, lambda a: ProbeOutcome(SCORES8[combo_index(a, sset)], 100 + combo_index(a, sset),
                                                        2.0), SearchOptions(max_depth=3, score=ScoreMode.RelMseOnly))
    assert r.probes == 8 and len(r.log) == 8
    assert r.best_score == pytest.approx(0.31)
    assert [s.kind for s in r.best] == [StrategyKind.Fixed, StrategyKind.Throughput, StrategyKind.Throughput]
    assert [combo_index(row.assignment, sset) for row in r.log] == list(range(8))


def test_score_mode_multiplies_time():
    """test_mixdepth.cpp:90-103."""
    sset = [FIXED1, TP]
    r = brute_force_search(sset, lambda a: ProbeOutcome(1.0, 10, 2.0 if a[0].kind == StrategyKind.Fixed else 0.5),
                           SearchOptions(max_depth=1, score=ScoreMode.RelMseTime))
    assert r.best[0].kind == StrategyKind.Throughput and r.best_score == pytest.approx(0.5)
    assert probe_score(ProbeOutcome(2.0, 1, 3.0), ScoreMode.RelMseTime) == 6.0
    assert probe_score(ProbeOutcome(2.0, 1, 3.0), ScoreMode.RelMseOnly) == 2.0


def test_combination_cap_points_to_heuristic():
    """test_mixdepth.cpp:105-119."""
    with pytest.raises(RuntimeError, match="heuristic_search"):
        brute_force_search([FIXED1, TP, NR], lambda a: ProbeOutcome(1.0, 1, 1.0), SearchOptions(max_depth=7))


def test_ties_break_lexicographically():
    """test_mixdepth.cpp:121-138."""
    sset = [TP, FIXED1]
    opt = SearchOptions(max_depth=2, score=ScoreMode.RelMseOnly)
    b = brute_force_search(sset, lambda a: ProbeOutcome(0.5, 1, 1.0), opt)
    assert b.probes == 4 and [s.kind for s in b.best] == [StrategyKind.Throughput] * 2
    opt.segment_depth = 1
    h = heuristic_search(sset, lambda a: ProbeOutcome(0.5, 1, 1.0), opt)
    assert h.probes == 4 and [s.kind for s in h.best] == [StrategyKind.Throughput] * 2


@pytest.mark.parametrize("sset,B,T,probes", [([FIXED1, TP, NR], 10, 6, 810), ([FIXED1, TP], 4, 2, 8),
                                              ([FIXED1, TP], 5, 2, 10)])
def test_heuristic_probe_counts(sset, B, T, probes):
    """test_mixdepth.cpp:140-182, including the frozen suffix / prefix rows of the 810 case."""
    r = heuristic_search(sset, lambda a: ProbeOutcome(1.0, 1, 1.0),
                         SearchOptions(max_depth=B, segment_depth=T, score=ScoreMode.RelMseOnly))
    assert r.probes == probes == len(r.log)
    if probes == 810:
        for row in r.log[:729]:
            assert all(s.kind == StrategyKind.Fixed and s.fixed_value == 1.0 for s in row.assignment[6:])
        for row in r.log[729:]:
            assert all(same(row.assignment[d], r.best[d]) for d in range(6))


def test_single_segment_heuristic_equals_brute():
    """test_mixdepth.cpp:184-201."""
    sset = [FIXED1, TP]
    probe = lambda a: ProbeOutcome(SCORES8[combo_index(a, sset)], 1, 1.0)
    opt = SearchOptions(max_depth=3, segment_depth=3, score=ScoreMode.RelMseOnly)
    b, h = brute_force_search(sset, probe, opt), heuristic_search(sset, probe, opt)
    assert h.probes == b.probes and h.best_score == b.best_score
    assert all(same(x, y) for x, y in zip(h.best, b.best))


def test_heuristic_between_minimum_and_fixed_baseline():
    """test_mixdepth.cpp:203-230 (scores from RngStream(99, i))."""
    L = orc.lib()
    sset = [FIXED1, NR]
    scores = []
    for i in range(16):
        r = (orc.C.c_uint64 * 2)()
        L.orc_rng_init(r, 99, i)
        scores.append(0.1 + L.orc_rng_next_float(r))
    h = heuristic_search(sset, lambda a: ProbeOutcome(scores[combo_index(a, sset)], 1, 1.0),
                         SearchOptions(max_depth=4, segment_depth=2, score=ScoreMode.RelMseOnly))
    assert min(scores) <= h.best_score <= scores[0]
    assert h.best_score == pytest.approx(scores[combo_index(h.best, sset)])


def test_non_finite_scores_rejected():
    """test_mixdepth.cpp:232-240."""
    with pytest.raises(RuntimeError, match="non-finite"):
        brute_force_search([FIXED1, TP], lambda a: ProbeOutcome(math.nan, 1, 1.0), SearchOptions(max_depth=1))


def test_search_log_csv(tmp_path):
    """test_mixdepth.cpp:242-268."""
    sset = [FIXED1, TP]
    path = str(tmp_path / "mixdepth_log_test.csv")
    r = brute_force_search(sset, lambda a: ProbeOutcome(1.0 + combo_index(a, sset), 7, 0.25),
                           SearchOptions(max_depth=2, score=ScoreMode.RelMseOnly, log_path=path))
    assert r.probes == 4
    lines = [l for l in open(path).read().splitlines() if l]
    assert lines[0] == "assignment,score,rays,seconds"
    assert len(lines) == 5 and all(l.startswith('"') and '",' in l for l in lines[1:])
    assert lines[1] == '"fixed:1,fixed:1",1,7,0.25'


def test_relmse_matches_metrics_cpp():
    g = np.random.default_rng(3)
    img = g.random((50, 3), dtype=np.float32)
    ref = g.random((50, 3), dtype=np.float32)
    s = 0.0
    for i in range(50):
        for c in range(3):
            r = float(ref[i, c])
            d = float(img[i, c]) - r
            s += d * d / (r * r + 0.01)
    assert relmse(torch.from_numpy(img), torch.from_numpy(ref)) == pytest.approx(s / 150, rel=1e-14)
    with pytest.raises(RuntimeError, match="dimension mismatch"):
        relmse(torch.zeros(3, 3), torch.zeros(4, 3))


# ---- rank-sharded segments (gloo, world 2) ----
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    sset = [FIXED1, TP, NR]
    calls = []

    def probe(a):
        calls.append(combo_index(a, sset))
        i = combo_index(a, sset)
        return ProbeOutcome(0.1 + ((i * 7919) % 97) / 97.0, 10 + i, 0.5)

    r = heuristic_search(sset, probe, SearchOptions(max_depth=5, segment_depth=3, score=ScoreMode.RelMseTime))
    q.put((rank, [combo_index(x.assignment, sset) for x in r.log], [x.score for x in r.log],
           combo_index(r.best, sset), r.best_score, r.probes, calls))
    torch.distributed.destroy_process_group()


def test_sharded_search_equals_sequential():
    sset = [FIXED1, TP, NR]

    def probe(a):
        i = combo_index(a, sset)
        return ProbeOutcome(0.1 + ((i * 7919) % 97) / 97.0, 10 + i, 0.5)

    seq = heuristic_search(sset, probe, SearchOptions(max_depth=5, segment_depth=3, score=ScoreMode.RelMseTime))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in ps:
        p.join(timeout=60)
    calls = []
    for rank, log_idx, log_scores, best, best_score, probes, c in res:
        assert log_idx == [combo_index(x.assignment, sset) for x in seq.log]
        assert log_scores == [x.score for x in seq.log]
        assert best == combo_index(seq.best, sset) and best_score == seq.best_score and probes == seq.probes
        calls += c
    assert len(calls) == seq.probes  # every probe rendered exactly once across the ranks
