"""GPU: the mailbox exchange across PROCESSES -- each rank's mailbox mapped into the other rank's
process through its CUDA IPC handle (nrrs_gpu_mailbox_init / _connect, handles passed over the
process group), the path an N-GPU run takes; test_gpu_mailbox.py connects ranks of one process by
device address instead.

Both ranks share the one reachable GPU, so no kernel may wait on a kernel of the other process
that has not run yet: each phase (factors -> both sums published; decide -> both totals
published; clip) is followed by a device sync and a host barrier, so every mailbox poll finds its
data already there.  Parity: the rank queues concatenate to the single-rank stage, bit for bit,
with the global clip firing (wavefront.cpp:141-154, rrs.cpp:8-24 across ranks).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
WORLD = 2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, port, n, cap, q):
    import ctypes as C
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch
    import torch.distributed as dist
    import oracle as orc
    from helpers import mirror_nets, to_dev
    from paper_2510_07868_b200 import RateControl, Strategy, StrategyKind, _capi
    from paper_2510_07868_b200.sharded import ShardedRrsStage, mailbox_check

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    torch.cuda.set_device(0)
    nets = orc.OracleNets(orc.VARIANT_AID, seed=1, randomize=True)
    v = orc.gen_vertices(n, n_pixels=n)
    lo, hi = rank * n // WORLD, (rank + 1) * n // WORLD
    band = {k: np.ascontiguousarray(a[lo:hi]) for k, a in v.items()}
    sh = ShardedRrsStage(n, mirror_nets(nets), capacity=cap, seed=0, device=0, exchange="mailbox")  # IPC connect
    st = sh.stage
    rc = RateControl(f_rate=1.2)
    out = st.alloc_outputs(hi - lo, full=True)
    kind = Strategy(StrategyKind.AidNrrs)
    sh.factors(to_dev(band), 2, kind, out, 0.0, rc.gain())  # K-A's last CTA publishes the exact sum
    torch.cuda.synchronize()
    dist.barrier()
    total = torch.zeros(1, dtype=torch.int64, device="cuda")
    p = st.params(2, kind, rc.gain(), 0.0, n_pixels=n)
    _capi.check(st.handle, st.ctx.lib.nrrs_gpu_stage_decide_mbox(st.handle, hi - lo, C.byref(p),
                                                                 C.byref(out.c()), total.data_ptr()))
    torch.cuda.synchronize()
    dist.barrier()
    clip = torch.zeros(4, dtype=torch.int64, device="cuda")
    _capi.check(st.handle, st.ctx.lib.nrrs_gpu_sharded_clip_mbox(st.handle, cap, clip.data_ptr(), None, None))
    torch.cuda.synchronize()
    mailbox_check(st)
    fr = st.fetch_result()
    base, kept, spawned, dropped = (int(x) for x in clip.cpu().numpy())
    q.put((rank, base, kept, spawned, dropped, out.k.cpu().numpy(), out.slots.cpu().numpy()[:kept].view(np.uint32),
           fr.f_norm))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(400)
def test_mailbox_over_cuda_ipc_between_processes():
    import oracle as orc
    import torch
    from helpers import mirror_nets, to_dev
    from paper_2510_07868_b200 import RateControl, RrsStage, Strategy, StrategyKind
    n = 40000
    cap = 40000  # slackless: f_rate 1.2 makes the global clip fire
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, port, n, cap, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(WORLD)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    nets = orc.OracleNets(orc.VARIANT_AID, seed=1, randomize=True)
    st = RrsStage(n, mirror_nets(nets), capacity=cap, seed=0)
    out, r = st.run(to_dev(orc.gen_vertices(n, n_pixels=n)), 2, Strategy(StrategyKind.AidNrrs),
                    rc=RateControl(f_rate=1.2), full=True)
    torch.cuda.synchronize()
    assert r.dropped > 0
    assert res[0][7] == res[1][7] == r.f_norm  # exact sums through the IPC-mapped mailboxes
    assert res[0][3] == res[1][3] == r.spawned and res[0][4] == res[1][4] == r.dropped
    assert res[0][1] == 0 and res[0][2] + res[1][2] == r.spawned  # rank 0 first; kept records add up
    np.testing.assert_array_equal(np.concatenate([res[0][5], res[1][5]]), out.k.cpu().numpy())
    r1 = res[1][6].copy()
    r1[:, 0] += n // WORLD
    np.testing.assert_array_equal(np.concatenate([res[0][6], r1]), out.slots.cpu().numpy()[:r.spawned].view(np.uint32))
    st.close()
