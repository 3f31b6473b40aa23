"""trace_frame on the GPU against the oracle's sequential restatement of
wavefront.cpp:217-551: per-depth queue sizes, the f64 film, depth-1 normals, FrameReport counters,
RateControl and the TrainSamples.  Heuristic strategies make every decision integer-exact, so the
frames agree bit for bit except where a direction sampled through cos / sin (double-evaluated on
the GPU, glibc cosf / sinf in the reference) lands on another rounding; that is allowed for a tiny
fraction of pixels and checked to stay small."""
import numpy as np
import pytest
import torch

import oracle as orc
from helpers import mirror_nets

pytestmark = pytest.mark.gpu


def _mods():
    from paper_2510_07868_b200 import film, render, rrs, stage
    return film, render, rrs, stage


def _gpu_trace(desc, w, h, assignment, B, seed=3, frames=1, capacity=0, collect=False, nets=None, roll=True,
               train_cap=0):
    film_m, render, rrs, stage = _mods()
    if nets is not None:
        st = stage.RrsStage(w * h, mirror_nets(nets))
        ctx = st.ctx
    else:
        ctx = stage.GpuContext(0)
    scene = render.GpuScene(desc, ctx=ctx)
    tracer = render.Tracer(scene, w * h, B, capacity)
    sx = film_m.SuffixStage(ctx=ctx)
    film = film_m.GpuFilm(w, h, sx)
    rc = rrs.RateControl()
    strat = [rrs.Strategy(rrs.StrategyKind(k), v) for k, v in assignment]
    cap = train_cap or (w * h * 8 if collect else 0)
    train = torch.zeros(max(cap, 1) * 80, dtype=torch.uint8, device=scene.device) if collect else None
    out = []
    for f in range(frames):
        cfg = render.TraceConfig(max_depth=B, queue_capacity=capacity, seed=seed, frame_index=f,
                                 collect_training=collect)
        before = film.sum.clone()
        rep, cnt = tracer.trace_frame(strat, cfg, rc, film, train=train, train_count=0)
        frame = (film.sum - before).cpu().numpy() if f else film.sum.cpu().numpy()
        tr = None
        if collect:
            tr = train[:cnt * 80].cpu().numpy().view(film_m.TRAIN_SAMPLE_DTYPE)
        out.append({"frame": frame, "sum": film.sum.cpu().numpy().copy(), "normals": film.normal.cpu().numpy(),
                    "report": rep, "train": tr, "i_acc": film.i_acc.cpu().numpy().copy(), "alpha": rc.alpha,
                    "overflow": rc.overflow_events})
        if roll:
            film.roll_acc()
    return out


def _orc_trace(desc, w, h, assignment, B, seed=3, frames=1, capacity=0, collect=False, nets=None, roll=True):
    rc = {"f_rate": 0.85, "alpha": 1.0, "eps": 0.01, "enabled": 1, "overflow_events": 0}
    i_acc = np.zeros((w * h, 3), np.float32)
    total = np.zeros((w * h, 3), np.float64)
    out = []
    for f in range(frames):
        r = orc.trace_frame(desc, w, h, assignment, B, seed=seed, frame_index=f, i_acc=i_acc, rc=rc, nets=nets,
                            capacity=capacity, collect_training=collect)
        total = total + r["frame"]
        r["sum"] = total.copy()
        r["i_acc"] = i_acc.copy()
        r["alpha"] = rc["alpha"]
        r["overflow"] = rc["overflow_events"]
        out.append(r)
        if roll:  # Film::add_frame's i_cur = float(frame), then roll_acc (wavefront.cpp:104-116)
            i_cur = r["frame"].astype(np.float32)
            i_acc = (np.float32(0.5) * i_acc + np.float32(0.5) * i_cur).astype(np.float32)
    return out


def _compare(g, r, exact_frac=0.97, rel=2e-3):
    rep = g["report"]
    assert rep.camera_rays == r["report"]["camera_rays"]
    dc_g, dc_r = np.array(rep.depth_counts, np.int64), np.array(r["report"]["depth_counts"], np.int64)
    assert dc_g[0] == dc_r[0]
    assert (np.abs(dc_g - dc_r) <= np.maximum(2, dc_r // 500)).all(), (dc_g, dc_r)
    fg, fr = g["frame"], r["frame"]
    same = (fg.view(np.uint64) == fr.view(np.uint64)).all(axis=1)
    assert same.mean() >= exact_frac, f"{(~same).sum()} of {same.size} pixels differ"
    # the rest differ by float rounding of sampled directions (measured <= 5e-7 relative)
    d = np.abs(fg - fr).max(1) / np.maximum(np.abs(fr).max(1), 1e-30)
    assert d.max() <= 1e-5, f"max relative pixel difference {d.max():.3e}"
    np.testing.assert_allclose(fg.sum(0), fr.sum(0), rtol=rel)
    ng, nr = g["normals"], r["normals"]
    nsame = (ng.view(np.uint32) == nr.view(np.uint32)).all(axis=1)
    assert nsame.mean() >= 0.999
    for k in ("shadow_rays", "scatter_rays"):
        a, b = getattr(rep, k), r["report"][k]
        assert abs(a - b) <= max(4, b // 500), (k, a, b)
    return same


CORNELL_PT = [(0, 1.0)] * 5


def test_cornell_path_tracing_matches_oracle():
    """pt (fixed 1) at every depth: the plain path tracer through the stage (wavefront.cpp:373-375 pin)."""
    _, render, _, _ = _mods()
    desc = render.make_cornell_scene()
    g = _gpu_trace(desc, 64, 48, CORNELL_PT, 5)[0]
    r = _orc_trace(desc, 64, 48, CORNELL_PT, 5)[0]
    _compare(g, r)
    assert g["report"].depth_counts[-1] > 0


@pytest.mark.parametrize("scene", ["cornell", "caustic", "furnace"])
def test_throughput_rr_with_training_matches_oracle(scene):
    """throughput RR + splitting budget, training collection and the reverse pass."""
    _, render, _, _ = _mods()
    desc = getattr(render, f"make_{scene}_scene")()
    B = 6
    assignment = [(0, 1.0)] + [(1, 1.0)] * (B - 1)
    g = _gpu_trace(desc, 48, 40, assignment, B, seed=11, collect=True)[0]
    r = _orc_trace(desc, 48, 40, assignment, B, seed=11, collect=True)[0]
    same = _compare(g, r)
    tg, tr = g["train"], r["train"]
    assert abs(len(tg) - len(tr)) <= max(2, len(tr) // 500)
    if len(tg) == len(tr) and same.all():
        for f in ("position", "omega_o", "roughness", "t_x", "i_pixel", "q_norm", "q_real", "pixel", "k_i", "depth"):
            np.testing.assert_array_equal(tg[f], tr[f], err_msg=f)
        np.testing.assert_array_equal(tg["lo_sample"].view(np.uint32), tr["lo_sample"].view(np.uint32))
    assert g["report"].train_samples == len(tg)


def test_env_emission_and_multi_frame_accumulation():
    """Escaped rays pick up env_emission (wavefront.cpp:295-303); three frames with roll_acc feed
    i_acc back into the strategies (ADRRS-free: throughput), Film sums accumulate."""
    _, render, _, _ = _mods()
    desc = render.make_cornell_scene()
    desc.env_emission = (0.2, 0.3, 0.4)
    B = 5
    assignment = [(0, 1.0)] + [(1, 1.0)] * (B - 1)
    gs = _gpu_trace(desc, 40, 32, assignment, B, seed=5, frames=3)
    rs = _orc_trace(desc, 40, 32, assignment, B, seed=5, frames=3)
    for g, r in zip(gs, rs):
        _compare(g, r)
        np.testing.assert_allclose(g["sum"].sum(0), r["sum"].sum(0), rtol=2e-3)
    assert gs[0]["frame"][:, 2].sum() > 0


def test_capacity_pressure_overflow_and_rate_control():
    """fixed:2 splitting against a queue capacity of exactly the pixel count: plan_spawns clips,
    RateControl::note_overflow decays alpha (wavefront.cpp:406-411)."""
    _, render, _, _ = _mods()
    desc = render.make_cornell_scene()
    w, h, B = 32, 32, 4
    assignment = [(0, 1.0), (0, 2.0), (1, 1.0), (1, 1.0)]
    g = _gpu_trace(desc, w, h, assignment, B, seed=9, capacity=w * h)[0]
    r = _orc_trace(desc, w, h, assignment, B, seed=9, capacity=w * h)[0]
    _compare(g, r)
    assert g["report"].overflow_events == r["report"]["overflow_events"] >= 1
    assert g["report"].bias_drop_events == r["report"]["bias_drop_events"]
    assert g["alpha"] == r["alpha"] < 1.0


@pytest.mark.parametrize("kind", [orc.NRRS, orc.AID_NRRS, orc.ADRRS_NN])
def test_neural_strategies_trace_statistically(kind):
    """Neural factors agree with the oracle to ~1e-3 (tcgen05 fp16 MLP), so single decisions can
    flip; the frame must agree statistically and the stage must run through trace_frame."""
    _, render, _, _ = _mods()
    desc = render.make_cornell_scene()
    on = orc.OracleNets(orc.VARIANT_AID if kind == orc.AID_NRRS else orc.VARIANT_NRRS, seed=1, randomize=True)
    B = 5
    assignment = [(0, 1.0)] + [(kind, 1.0)] * (B - 1)
    g = _gpu_trace(desc, 48, 40, assignment, B, seed=2, frames=2, nets=on)
    r = _orc_trace(desc, 48, 40, assignment, B, seed=2, frames=2, nets=on)
    for a, b in zip(g, r):
        assert a["report"].depth_counts[0] == b["report"]["depth_counts"][0]
        ca, cb = np.array(a["report"].depth_counts), np.array(b["report"]["depth_counts"])
        assert (np.abs(ca - cb) <= np.maximum(8, cb // 20)).all(), (ca, cb)
        np.testing.assert_allclose(a["frame"].sum(0), b["frame"].sum(0), rtol=0.05)


def test_trace_frame_errors():
    film_m, render, rrs, stage = _mods()
    from paper_2510_07868_b200 import _capi
    desc = render.make_cornell_scene()
    ctx = stage.GpuContext(0)
    scene = render.GpuScene(desc, ctx=ctx)
    tracer = render.Tracer(scene, 16 * 16, 4)
    film = film_m.GpuFilm(16, 16, film_m.SuffixStage(ctx=ctx))
    rc = rrs.RateControl()
    pt = [rrs.Strategy()] * 4
    with pytest.raises(_capi.NrrsError, match="needs networks"):
        tracer.trace_frame([rrs.Strategy()] + [rrs.Strategy(rrs.StrategyKind.Nrrs)] * 3,
                           render.TraceConfig(max_depth=4), rc, film)
    with pytest.raises(_capi.NrrsError, match="octree"):
        tracer.trace_frame([rrs.Strategy()] + [rrs.Strategy(rrs.StrategyKind.AdrrsTree)] * 3,
                           render.TraceConfig(max_depth=4), rc, film)
    with pytest.raises(_capi.NrrsError, match="capacity below"):
        tracer.trace_frame(pt, render.TraceConfig(max_depth=4, queue_capacity=100), rc, film)
    with pytest.raises(RuntimeError, match="one entry per depth"):
        tracer.trace_frame(pt[:3], render.TraceConfig(max_depth=4), rc, film)
    big = film_m.GpuFilm(32, 32, film_m.SuffixStage(ctx=ctx))
    with pytest.raises(_capi.NrrsError):
        tracer.trace_frame(pt, render.TraceConfig(max_depth=4), rc, big)


@pytest.mark.parametrize("kind,size", [(orc.AID_NRRS, (48, 40)), (orc.AID_NRRS, (512, 512)), (orc.NRRS, (96, 80))],
                         ids=["aid-fused-small", "aid-three-kernel", "nrrs"])
def test_neural_trace_is_bitwise_reproducible(kind, size):
    """The reference's renders are bit-identical across runs (test_engine.cpp:461-502); the GPU
    trace_frame with neural RRS (the fused small-batch AID stage, the three-kernel path at 512 x 512,
    NRRS) gives bit-identical films, normals and depth counts on two fresh contexts."""
    _, render, _, _ = _mods()
    desc = render.make_cornell_scene()
    on = orc.OracleNets(orc.VARIANT_AID if kind == orc.AID_NRRS else orc.VARIANT_NRRS, seed=1, randomize=True)
    B = 6
    assignment = [(0, 1.0)] + [(kind, 1.0)] * (B - 1)
    w, h = size
    a = _gpu_trace(desc, w, h, assignment, B, seed=7, frames=2, nets=on)
    b = _gpu_trace(desc, w, h, assignment, B, seed=7, frames=2, nets=on)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x["sum"], y["sum"])
        np.testing.assert_array_equal(x["normals"], y["normals"])
        assert list(x["report"].depth_counts) == list(y["report"].depth_counts)
