"""GPU: mailbox mode of the tile-sharded stage -- the two per-depth exchanges (rank sums of q,
rank totals; wavefront.cpp:141-154, rrs.cpp:8-24 across ranks) inside the kernels over peer
memory instead of host-issued all-gathers.

Only one GPU is reachable, so these checks keep every wait already satisfied when its kernel
starts: the ranks are RrsStage contexts in ONE process, their mailboxes connected by device
address, and every producer kernel (K-A publishing a sum, K-B publishing a total) is enqueued on
the same stream BEFORE the consumer that polls for it -- no kernel ever waits on a kernel that
has not run yet.  (Mailbox waits also give up after 10 s with a flag instead of hanging.)
Parity: the concatenated rank queues equal the single-rank stage on the whole batch, bit for bit,
exactly like the collective path (tests/test_gpu_sharded.py).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

import oracle as orc
from helpers import mirror_nets, to_dev
from paper_2510_07868_b200 import RateControl, RrsStage, Strategy, StrategyKind, _capi
from paper_2510_07868_b200.sharded import connect_mailboxes_in_process, mailbox_check, mailbox_depth

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy()


def _band(v, lo, hi):
    return {k: np.ascontiguousarray(a[lo:hi]) for k, a in v.items()}


def _factors(st, dv, n, p, out, local_sum):
    st.ctx.bind_stream()
    soa = __import__("paper_2510_07868_b200.stage", fromlist=["vertex_soa"]).vertex_soa(dv)
    oc = out.c()
    _capi.check(st.handle, st.ctx.lib.nrrs_gpu_stage_factors(st.handle, C.byref(soa), n, C.byref(p), C.byref(oc),
                                                             local_sum.data_ptr()))


@pytest.mark.parametrize("variant", [orc.VARIANT_NRRS, orc.VARIANT_AID], ids=["nrrs", "aid"])
def test_mailbox_two_ranks_match_single_rank(variant):
    n = npx = 40000
    cap = 40000  # slackless: the global tail clip fires at f_rate 1.2
    world = 2
    nets = orc.OracleNets(variant, seed=1, randomize=True)
    v = orc.gen_vertices(n, n_pixels=npx)
    kind = StrategyKind.AidNrrs if variant == orc.VARIANT_AID else StrategyKind.Nrrs
    rc = RateControl(f_rate=1.2)
    ref_st = RrsStage(npx, mirror_nets(nets), capacity=cap, seed=0)
    ref, r = ref_st.run(to_dev(v), 2, Strategy(kind), rc=RateControl(f_rate=1.2), full=True)
    torch.cuda.synchronize()
    assert r.dropped > 0

    stages = [RrsStage(npx, mirror_nets(nets), capacity=cap, seed=0) for _ in range(world)]
    connect_mailboxes_in_process(stages)
    bands = [(rk * n // world, (rk + 1) * n // world) for rk in range(world)]
    outs, sums, tots = [], [], []
    # phase 1 (both ranks publish their sums), then phase 2: every poll finds its data present
    for rk, st in enumerate(stages):
        lo, hi = bands[rk]
        out = st.alloc_outputs(hi - lo, full=True)
        sums.append(torch.zeros(1, dtype=torch.float64, device="cuda"))
        tots.append(torch.zeros(1, dtype=torch.int64, device="cuda"))
        p = st.params(2, Strategy(kind), rc.gain(), 0.0, n_pixels=npx)
        _factors(st, to_dev(_band(v, lo, hi)), hi - lo, p, out, sums[rk])
        outs.append(out)
    torch.cuda.synchronize()
    for rk, st in enumerate(stages):
        lo, hi = bands[rk]
        p = st.params(2, Strategy(kind), rc.gain(), 0.0, n_pixels=npx)
        _capi.check(st.handle, st.ctx.lib.nrrs_gpu_stage_decide_mbox(st.handle, hi - lo, C.byref(p),
                                                                     C.byref(outs[rk].c()), tots[rk].data_ptr()))
    torch.cuda.synchronize()
    clips, seen_s, seen_t = [], [], []
    for st in stages:
        clip = torch.zeros(4, dtype=torch.int64, device="cuda")
        s = torch.zeros(world, dtype=torch.float64, device="cuda")
        t = torch.zeros(world, dtype=torch.int64, device="cuda")
        _capi.check(st.handle, st.ctx.lib.nrrs_gpu_sharded_clip_mbox(st.handle, cap, clip.data_ptr(), s.data_ptr(),
                                                                     t.data_ptr()))
        clips.append(clip)
        seen_s.append(s)
        seen_t.append(t)
    torch.cuda.synchronize()
    for st in stages:
        mailbox_check(st)
    # both ranks saw the same sums and totals, in rank order, equal to what each published
    for rk in range(world):
        np.testing.assert_array_equal(_np(seen_s[rk]), np.array([float(x.item()) for x in sums]))
        np.testing.assert_array_equal(_np(seen_t[rk]), np.array([int(x.item()) for x in tots]))
    # the ranks exchanged their exact 128-bit sums: F equals the one-rank F bit for bit
    for st in stages:
        fr = _capi.StageResultC()
        _capi.check(st.handle, st.ctx.lib.nrrs_gpu_fetch_result(st.handle, C.byref(fr)))
        assert fr.f_norm == r.f_norm
    base0, kept0, sp0, dr0 = (int(x) for x in _np(clips[0]))
    base1, kept1, sp1, dr1 = (int(x) for x in _np(clips[1]))
    assert (sp0, dr0) == (sp1, dr1) == (r.spawned, r.dropped)
    assert base0 == 0 and base1 == int(tots[0].item())
    # bit-identical decisions, and the rank queues concatenate to the global queue
    np.testing.assert_array_equal(np.concatenate([_np(o.k) for o in outs]), _np(ref.k))
    np.testing.assert_array_equal(np.concatenate([_np(o.q_norm) for o in outs]), _np(ref.q_norm))
    slots = _np(ref.slots)[: r.spawned].view(np.uint32)
    r0 = _np(outs[0].slots)[:kept0].view(np.uint32)
    r1 = _np(outs[1].slots)[:kept1].view(np.uint32).copy()
    r1[:, 0] += bands[1][0]
    np.testing.assert_array_equal(np.concatenate([r0, r1]), slots)
    for st in stages + [ref_st]:
        st.close()


def test_mailbox_single_rank_depths_and_graph_replay():
    """world = 1 (the rank's own mailbox): consecutive depths advance the device generations, and
    a CUDA graph of depths replays with fresh generations; results equal the plain stage."""
    n = npx = 30000
    nets = orc.OracleNets(orc.VARIANT_NRRS, seed=1, randomize=True)
    v = orc.gen_vertices(n, n_pixels=npx)
    dv = to_dev(v)
    ref_st = RrsStage(npx, mirror_nets(nets), seed=0)
    ref, r = ref_st.run(dv, 2, Strategy(StrategyKind.Nrrs), rc=RateControl(), full=True)
    torch.cuda.synchronize()
    st = RrsStage(npx, mirror_nets(nets), seed=0)
    connect_mailboxes_in_process([st])
    out = st.alloc_outputs(n, full=True)
    local_sum = torch.zeros(1, dtype=torch.float64, device="cuda")
    total = torch.zeros(1, dtype=torch.int64, device="cuda")
    p = st.params(2, Strategy(StrategyKind.Nrrs), RateControl().gain(), 0.0, n_pixels=npx)

    def depth():
        _factors(st, dv, n, p, out, local_sum)
        return mailbox_depth(st, n, p, out, total, 1, 0, st.capacity, npx)

    for _ in range(3):
        pend = depth()
        o = pend.resolve()
        assert o.spawned == r.spawned and o.dropped == r.dropped and o.base == 0 and o.kept == r.spawned
        assert o.rank_totals == [r.total]
        np.testing.assert_array_equal(_np(out.k), _np(ref.k))
        np.testing.assert_array_equal(_np(out.slots)[: r.spawned], _np(ref.slots)[: r.spawned])
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        depth()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    pend = None
    with torch.cuda.graph(g):
        for _ in range(4):
            pend = depth()
    out.k.zero_()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    mailbox_check(st)  # a stale generation would have timed out
    o = pend.resolve()
    assert o.spawned == r.spawned and o.rank_totals == [r.total]
    np.testing.assert_array_equal(_np(out.k), _np(ref.k))
    st.close()
    ref_st.close()


def test_mailbox_empty_rank_still_exchanges():
    """A rank with no vertices this depth publishes a zero sum and a zero total (one-thread
    kernels), so the other rank's waits complete and its clip sees the right base."""
    n = npx = 20000
    nets = orc.OracleNets(orc.VARIANT_NRRS, seed=1, randomize=True)
    v = orc.gen_vertices(n, n_pixels=npx)
    stages = [RrsStage(npx, mirror_nets(nets), seed=0) for _ in range(2)]
    connect_mailboxes_in_process(stages)
    sums = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
    tots = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(2)]
    outs = [stages[0].alloc_outputs(1, full=True), stages[1].alloc_outputs(n, full=True)]
    bands = [(0, 0), (0, n)]  # rank 0 empty, rank 1 the whole film
    for rk, st in enumerate(stages):
        lo, hi = bands[rk]
        p = st.params(2, Strategy(StrategyKind.Nrrs), RateControl().gain(), 0.0, n_pixels=npx)
        _factors(st, to_dev(_band(v, lo, max(hi, lo))), hi - lo, p, outs[rk], sums[rk])
    torch.cuda.synchronize()
    for rk, st in enumerate(stages):
        lo, hi = bands[rk]
        p = st.params(2, Strategy(StrategyKind.Nrrs), RateControl().gain(), 0.0, n_pixels=npx)
        _capi.check(st.handle, st.ctx.lib.nrrs_gpu_stage_decide_mbox(st.handle, hi - lo, C.byref(p),
                                                                     C.byref(outs[rk].c()), tots[rk].data_ptr()))
    torch.cuda.synchronize()
    clips = []
    for st in stages:
        clip = torch.zeros(4, dtype=torch.int64, device="cuda")
        _capi.check(st.handle, st.ctx.lib.nrrs_gpu_sharded_clip_mbox(st.handle, st.capacity, clip.data_ptr(),
                                                                     None, None))
        clips.append(clip)
    torch.cuda.synchronize()
    for st in stages:
        mailbox_check(st)
    ref_st = RrsStage(npx, mirror_nets(nets), seed=0)
    ref, r = ref_st.run(to_dev(v), 2, Strategy(StrategyKind.Nrrs), rc=RateControl(), full=True)
    torch.cuda.synchronize()
    assert float(sums[0].item()) == 0.0 and int(tots[0].item()) == 0
    assert [int(x) for x in _np(clips[0])] == [0, 0, r.spawned, r.dropped]
    assert [int(x) for x in _np(clips[1])] == [0, r.spawned, r.spawned, r.dropped]
    np.testing.assert_array_equal(_np(outs[1].k), _np(ref.k))
    for st in stages + [ref_st]:
        st.close()
