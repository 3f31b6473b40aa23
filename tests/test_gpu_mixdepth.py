"""Mix-Depth search with real probes: every GPU probe render (trace_frame with a
fresh film seeded by i_acc, runner.cpp:414-434) scores like the oracle's probe of the same assignment,
and the brute-force / heuristic searches pick the same assignment."""
import numpy as np
import pytest
import torch

import oracle as orc

pytestmark = pytest.mark.gpu


def test_gpu_probes_match_oracle_probes_and_search():
    from paper_2510_07868_b200 import film as film_m, render, stage
    from paper_2510_07868_b200.mixdepth import (GpuProbe, ScoreMode, SearchOptions, brute_force_search,
                                                heuristic_search, relmse)
    from paper_2510_07868_b200.rrs import RateControl, Strategy, StrategyKind
    desc = render.make_cornell_scene()
    w, h, B = 32, 24, 3
    ctx = stage.GpuContext(0)
    scene = render.GpuScene(desc, ctx=ctx)
    tracer = render.Tracer(scene, w * h, B)
    # reference image: 8 path-traced frames on the GPU; i_acc from them (the "trained" film)
    film = film_m.GpuFilm(w, h, film_m.SuffixStage(ctx=ctx))
    for f in range(8):
        tracer.trace_frame([Strategy()] * B, render.TraceConfig(max_depth=B, seed=1, frame_index=f), RateControl(),
                           film)
        film.roll_acc()
    reference = film.mean_image()
    i_acc = film.i_acc.clone()
    probe = GpuProbe(tracer, w, h, reference, i_acc, frame_index=8, seed=2, deterministic=True)
    cands = [Strategy(StrategyKind.Fixed, 1.0), Strategy(StrategyKind.Throughput)]
    opt = SearchOptions(max_depth=B, score=ScoreMode.RelMseOnly)
    r = brute_force_search(cands, probe, opt)
    assert r.probes == 8

    ref_np = reference.cpu().numpy()
    i_acc_np = i_acc.cpu().numpy()

    def orc_probe(a):
        o = orc.trace_frame(desc, w, h, [(int(s.kind), s.fixed_value) for s in a], B, seed=2, frame_index=8,
                            i_acc=i_acc_np)
        img = o["frame"].astype(np.float32)  # mean of one sample, cast<float>
        return relmse(torch.from_numpy(img), torch.from_numpy(ref_np))

    for row in r.log:
        want = orc_probe(row.assignment)
        assert row.score == pytest.approx(want, rel=1e-5), row.assignment
    ro = [orc_probe(row.assignment) for row in r.log]
    assert int(np.argmin(ro)) == [i for i, row in enumerate(r.log) if row.score == r.best_score][0]
    h2 = heuristic_search(cands, probe, SearchOptions(max_depth=B, segment_depth=2, score=ScoreMode.RelMseOnly))
    assert h2.probes == 4 + 2
    assert h2.best_score >= r.best_score
