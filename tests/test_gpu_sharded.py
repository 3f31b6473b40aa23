"""GPU: the tile-sharded product path (nrrs_gpu_stage_factors -> all-gather ->
nrrs_gpu_stage_decide -> all-gather -> nrrs_gpu_sharded_clip) with 2 ranks.

Only one GPU is available, so both ranks run on cuda:0 with the gloo backend:
the two per-depth exchanges are host-side collectives and no kernel of one
rank waits on the other.  Parity: the concatenation of the rank queues equals
the single-rank stage on the whole batch.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
WORLD = 2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, port, n, npx, cap, variant, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist
    import oracle as orc
    from helpers import mirror_nets, to_dev
    from paper_2510_07868_b200 import RateControl, Strategy, StrategyKind
    from paper_2510_07868_b200.sharded import ShardedRrsStage

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    torch.cuda.set_device(0)
    nets = orc.OracleNets(variant, seed=1, randomize=True)
    v = orc.gen_vertices(n, n_pixels=npx)
    lo, hi = rank * n // WORLD, (rank + 1) * n // WORLD
    band = {k: np.ascontiguousarray(a[lo:hi]) for k, a in v.items()}
    st = ShardedRrsStage(npx, mirror_nets(nets), capacity=cap, seed=0, device=0)
    rc = RateControl(f_rate=1.2)  # E[S] = 1.2 Npx > capacity: the global tail clip must fire
    dv = to_dev(band)
    out = st.stage.alloc_outputs(hi - lo, full=True)
    kind = StrategyKind.AidNrrs if variant == orc.VARIANT_AID else StrategyKind.Nrrs
    local = st.factors(dv, 2, Strategy(kind), out, 0.0, rc.gain())
    sums = [torch.zeros_like(local.cpu()) for _ in range(WORLD)]  # the exact sums: [2] int64 words
    dist.all_gather(sums, local.cpu())
    rank_sums = torch.cat(sums).cuda()
    total = st.decide(hi - lo, 2, Strategy(kind), out, rank_sums, rc.gain(), 0.0)
    tots = [torch.zeros(1, dtype=torch.int64) for _ in range(WORLD)]
    dist.all_gather(tots, total.cpu())
    from paper_2510_07868_b200.sharded import global_clip
    totals = [int(t.item()) for t in tots]
    base, kept, spawned, dropped = global_clip(totals, rank, st.capacity)
    torch.cuda.synchronize()
    fr = st.stage.fetch_result()
    q.put((rank, base, kept, spawned, dropped, out.k.cpu().numpy(), out.q_norm.cpu().numpy(),
           out.slots.cpu().numpy()[:kept].view(np.uint32), fr.f_norm))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(400)
@pytest.mark.parametrize("variant", [0, 1], ids=["nrrs", "aid"])
def test_two_rank_sharded_stage_matches_single_rank(variant):
    import oracle as orc
    from helpers import mirror_nets, to_dev
    from paper_2510_07868_b200 import RateControl, RrsStage, Strategy, StrategyKind
    n = npx = 40000
    cap = 40000  # slackless queue
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, port, n, npx, cap, variant, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(WORLD)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    nets = orc.OracleNets(variant, seed=1, randomize=True)
    v = orc.gen_vertices(n, n_pixels=npx)
    st = RrsStage(npx, mirror_nets(nets), capacity=cap, seed=0)
    kind = StrategyKind.AidNrrs if variant == orc.VARIANT_AID else StrategyKind.Nrrs
    out, r = st.run(to_dev(v), 2, Strategy(kind), rc=RateControl(f_rate=1.2), full=True)
    assert r.dropped > 0
    k = np.concatenate([x[5] for x in res])
    np.testing.assert_array_equal(k, out.k.cpu().numpy())
    np.testing.assert_array_equal(np.concatenate([x[6] for x in res]), out.q_norm.cpu().numpy())
    assert res[0][3] == res[1][3] == r.spawned and res[0][4] == r.dropped
    assert res[0][8] == res[1][8] == r.f_norm  # exact rank sums: the one-rank F, bit for bit
    # rank queues concatenate to the global queue: rank 1's parents are offset by rank 0's band
    slots = out.slots.cpu().numpy()[: r.spawned].view(np.uint32)
    r0 = res[0][7]
    r1 = res[1][7].copy()
    r1[:, 0] += n // WORLD
    np.testing.assert_array_equal(np.concatenate([r0, r1]), slots)
