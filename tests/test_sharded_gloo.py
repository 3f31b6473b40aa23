"""CPU, world_size 2 (gloo): the tile-sharded protocol of paper_2510_07868_b200.sharded.

Each rank owns a contiguous band of the vertex queue.  The per-rank phase
computations are done by the CPU oracle (test stand-in for the CUDA phases; the
product binds the same protocol to the C ABI), the exchanges run through
torch.distributed exactly as on NCCL.  Parity: the concatenation of the rank
decisions equals the single-rank oracle decision on the whole queue, including a
global capacity-clip case.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, port, n, npx, cap, fixed, gain, q_override, result_q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import oracle as orc
    from helpers import oracle_decide
    from paper_2510_07868_b200.rrs import RateControl
    from paper_2510_07868_b200.sharded import sharded_depth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    v = orc.gen_vertices(n, n_pixels=npx)
    lo, hi = rank * n // WORLD, (rank + 1) * n // WORLD
    band = {k: np.ascontiguousarray(a[lo:hi]) for k, a in v.items()}
    # phase 1 (stand-in for nrrs_gpu_stage_factors): sanitized factors + uniforms
    ref_local = orc.rrs_stage(band, 2, npx, cap, orc.FIXED, None, fixed_value=fixed, gain=gain, seed=9)
    q = ref_local["q_orig"] if q_override is None else np.ascontiguousarray(q_override[lo:hi])
    u = ref_local["u"]
    local_sum = torch.tensor([float(np.sum(q.astype(np.float64)))], dtype=torch.float64)
    state = {}

    def decide(rank_sums):
        # phase 2 (stand-in for nrrs_gpu_stage_decide): global F from the gathered sums
        s = float(sum(rank_sums.tolist()))
        f = npx / s if s > 0 else 1.0
        qn = q * np.float32(f) if f < 1.0 else q.copy()
        qn = qn.astype(np.float32)
        qr = (qn * np.float32(gain)).astype(np.float32)
        fl = np.floor(qr)
        k = fl.astype(np.int64) + (u < (qr - fl)).astype(np.int64)
        state.update(k=k, qn=qn)
        return torch.tensor([int(k.sum())], dtype=torch.int64)

    rc = RateControl()
    out = sharded_depth(local_sum, decide, cap, npx, None, rc)
    result_q.put((rank, out.base, out.kept, out.spawned, out.dropped, out.f_norm, state["k"].tolist(),
                  state["qn"].tolist(), rc.overflow_events))
    dist.barrier()
    dist.destroy_process_group()


def _run(n, npx, cap, fixed, gain, q_override=None):
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, n, npx, cap, fixed, gain, q_override, result_q))
             for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted([result_q.get(timeout=240) for _ in range(WORLD)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.timeout(300)
def test_sharded_protocol_matches_single_rank():
    import oracle as orc
    from helpers import oracle_decide
    n = npx = 4000
    cap = orc.lib().orc_queue_capacity_for(npx)
    q = orc.split_bound_factors(n)
    res = _run(n, npx, cap, 1.0, 0.85, q_override=q)
    v = orc.gen_vertices(n, n_pixels=npx)
    u = orc.rrs_stage(v, 2, npx, cap, orc.FIXED, None, seed=9)["u"]
    ref = oracle_decide(q, u, npx, cap, 0.85)
    k = np.concatenate([np.array(r[6]) for r in res])
    qn = np.concatenate([np.array(r[7], np.float32) for r in res])
    np.testing.assert_array_equal(k, ref["k"])
    np.testing.assert_array_equal(qn, ref["q_norm"])
    assert np.float32(res[0][5]) == np.float32(ref["f_norm"]) == np.float32(res[1][5])
    assert res[0][3] == res[1][3] == ref["spawned"] and res[0][4] == ref["dropped"]
    assert res[0][1] == 0 and res[1][1] == int(k[: n // 2].sum())
    assert res[0][2] + res[1][2] == ref["spawned"]


@pytest.mark.timeout(300)
def test_sharded_global_clip_on_overflow():
    import oracle as orc
    from helpers import oracle_decide
    # capacity below the realized total: the tail clip must land inside rank 1's band
    n, npx = 6000, 3000
    cap = 2000
    q = np.full(n, 1.0, np.float32)
    q[: n // 2] = 2.0  # rank 0 splits, rank 1 continues: the clip falls inside rank 1's band
    res = _run(n, npx, cap, 1.0, 1.0, q_override=q)
    v = orc.gen_vertices(n, n_pixels=npx)
    u = orc.rrs_stage(v, 2, npx, cap, orc.FIXED, None, seed=9)["u"]
    ref = oracle_decide(q, u, npx, cap, 1.0)
    assert res[0][3] == ref["spawned"] == cap
    assert res[0][4] == res[1][4] == ref["dropped"]
    assert ref["dropped"] > 0
    assert res[0][2] == min(int(np.sum(res[0][6])), cap) and res[0][2] + res[1][2] == cap
    assert res[0][8] == res[1][8] == 1  # overflow is a global, replicated event


def _lum_f32(c):
    """luminance (core.hpp:24-26), f32 left to right."""
    c = c.astype(np.float32)
    return (np.float32(0.2126) * c[:, 0] + np.float32(0.7152) * c[:, 1]) + np.float32(0.0722) * c[:, 2]


def _film(npx):
    g = np.random.default_rng(5)
    return (g.random((npx, 3), dtype=np.float32) * np.float32(3.0)).astype(np.float32)


def _worker_frame(rank, port, npx, result_q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    from paper_2510_07868_b200 import NeuralRrs, NeuralRrsConfig, RrsVariant
    from paper_2510_07868_b200.sharded import broadcast_weights, sharded_eps_div

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    film = _film(npx)
    lo, hi = rank * npx // WORLD, (rank + 1) * npx // WORLD
    local = 0.0
    for v in _lum_f32(film[lo:hi]):  # per-rank stand-in for nrrs_gpu_film_luminance_sum
        local += float(v)
    eps = sharded_eps_div(torch.tensor([local], dtype=torch.float64), npx)
    nets = NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Aid, seed=1))
    if rank == 0:
        nets.randomize_for_benchmark()
    broadcast_weights(nets, src=0)
    result_q.put((rank, eps, float(nets.rrs_mlp[-1]), float(np.sum(nets.rrs_grid, dtype=np.float64)),
                  float(np.sum(nets.stat_mlp, dtype=np.float64))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_eps_div_and_weight_broadcast():
    """Per-frame eps_div exchange and per-publish weight broadcast: every rank
    gets the single-film eps_div (wavefront.cpp:238-243) and rank 0's snapshot."""
    from paper_2510_07868_b200 import NeuralRrs, NeuralRrsConfig, RrsVariant
    from paper_2510_07868_b200.rrs import eps_div_from_luminance_sum
    npx = 5001
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_frame, args=(r, port, npx, result_q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted([result_q.get(timeout=240) for _ in range(WORLD)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lum_acc = 0.0
    for v in _lum_f32(_film(npx)):  # the reference's sequential film loop
        lum_acc += float(v)
    eps_ref = float(np.float32(1e-4) * np.float32(lum_acc / npx))
    assert eps_div_from_luminance_sum(lum_acc, npx) == eps_ref
    assert res[0][1] == res[1][1] == eps_ref
    ref = NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Aid, seed=1)).randomize_for_benchmark()
    for r in res:
        assert r[2] == float(ref.rrs_mlp[-1])
        assert r[3] == float(np.sum(ref.rrs_grid, dtype=np.float64))
        assert r[4] == float(np.sum(ref.stat_mlp, dtype=np.float64))


def _worker_film(rank, port, width, height, result_q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    from paper_2510_07868_b200.sharded import gather_film, row_band
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    r0, r1 = row_band(rank, WORLD, height)
    full = torch.arange(width * height * 3, dtype=torch.float64).reshape(width * height, 3) * 0.5
    band = full[r0 * width:r1 * width].clone()
    out = gather_film(band, dst=0)
    result_q.put((rank, None if out is None else out.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_film_gather_row_bands():
    """Per-frame film gather of SURVEY.md 8e: uneven row bands (7 rows over 2 ranks) land on
    rank 0 in pixel order, bit for bit; other ranks get nothing."""
    width, height = 5, 7
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_film, args=(r, port, width, height, result_q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(result_q.get(timeout=240) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = (np.arange(width * height * 3, dtype=np.float64).reshape(-1, 3) * 0.5)
    np.testing.assert_array_equal(res[0], ref)
    assert res[1] is None


def _worker_async(rank, port, result_q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    from paper_2510_07868_b200.rrs import RateControl
    from paper_2510_07868_b200.sharded import sharded_depth, sharded_depth_async
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    local_sum = torch.tensor([10.5 + rank], dtype=torch.float64)
    totals = [700, 650]
    decide = lambda rs: torch.tensor([totals[rank]], dtype=torch.int64)  # noqa: E731
    seen = []
    rc_a, rc_b = RateControl(), RateControl()
    ref = sharded_depth(local_sum, decide, 1200, 1000, None, rc_a)
    pend = sharded_depth_async(local_sum, decide, 1200, 1000, None, None, after_exchange=lambda c: seen.append(c))
    got = pend.resolve(rc_b)
    result_q.put((rank, ref == got, seen == [None], rc_a.alpha == rc_b.alpha < 1.0))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_depth_async_matches_sync():
    """sharded_depth_async (device-side clip on NCCL; host clip on gloo, read at resolve())
    gives the same outcome and RateControl update as sharded_depth, here with a global overflow."""
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_async, args=(r, port, result_q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [result_q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in res:
        assert r[1] and r[2] and r[3], r


def test_sharded_stage_rejects_unknown_exchange():
    from paper_2510_07868_b200.sharded import ShardedRrsStage
    with pytest.raises(ValueError, match="exchange"):
        ShardedRrsStage(16, None, exchange="carrier-pigeon")
