"""GPU: the tile-sharded stage over a real NCCL process group (world size 1 -- one GPU is all
this environment reaches).

test_gpu_sharded.py / test_gpu_mailbox.py check the multi-rank arithmetic on one device with gloo
or in-process mailboxes; this one runs the code the N-GPU bench runs on NCCL: the exact sums
exchanged with all_gather_into_tensor straight from the context's words, nrrs_gpu_sharded_clip_dev
on the gathered totals (no host round trip), the device-resident weight broadcast
(nrrs_gpu_set_weights_dev), the per-frame eps_div gather and the film gather -- and the mailbox
exchange with its IPC handles passed over the NCCL group.  Parity: several consecutive depths,
queued without a host wait, equal the plain single-rank stage bit for bit (
wavefront.cpp:141-154, :238-243, rrs.cpp:8-24).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(port, exchange, variant, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch
    import torch.distributed as dist
    import oracle as orc
    from helpers import mirror_nets, to_dev
    from paper_2510_07868_b200 import RateControl, RrsStage, Strategy, StrategyKind
    from paper_2510_07868_b200.sharded import ShardedRrsStage, gather_film

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    assert dist.get_backend() == "nccl"
    n = npx = 50_000
    cap = npx  # slackless: f_rate 1.2 makes the global clip fire
    nets = orc.OracleNets(variant, seed=1, randomize=True)
    kind = StrategyKind.AidNrrs if variant == orc.VARIANT_AID else StrategyKind.Nrrs
    vs = [to_dev(orc.gen_vertices(n, n_pixels=npx, frame=f)) for f in range(3)]
    msgs = []

    ref = RrsStage(npx, mirror_nets(nets), capacity=cap, seed=0)
    refs = []
    for d, v in enumerate(vs):
        o, r = ref.run(v, 2 + d, Strategy(kind), rc=RateControl(f_rate=1.2), full=True)
        refs.append((o.k.cpu().numpy(), o.slots.cpu().numpy()[:r.spawned].copy(), r))

    st = ShardedRrsStage(npx, None, capacity=cap, seed=0, exchange=exchange)
    st.set_weights(mirror_nets(nets))  # NCCL broadcast; the blocks stay on the GPU
    outs, pend = [], []
    for d, v in enumerate(vs):  # three depths queued back to back, no host wait in between
        out = st.stage.alloc_outputs(n, full=True)
        st.factors(v, 2 + d, Strategy(kind), out, 0.0, RateControl(f_rate=1.2).gain())
        pend.append(st.depth_async(n, 2 + d, Strategy(kind), out, RateControl(f_rate=1.2).gain()))
        outs.append(out)
    for d, (out, pd) in enumerate(zip(outs, pend)):
        oc = pd.resolve()
        k_ref, slots_ref, r = refs[d]
        if (oc.spawned, oc.dropped, oc.base, oc.kept) != (r.spawned, r.dropped, 0, r.spawned):
            msgs.append(f"depth {d}: outcome {oc} vs {r}")
        if oc.f_norm != r.f_norm:
            msgs.append(f"depth {d}: F {oc.f_norm!r} vs {r.f_norm!r}")
        if not np.array_equal(out.k.cpu().numpy(), k_ref):
            msgs.append(f"depth {d}: counts differ")
        if not np.array_equal(out.slots.cpu().numpy()[:r.spawned], slots_ref):
            msgs.append(f"depth {d}: slots differ")
    if refs[0][2].dropped == 0:
        msgs.append("the global clip did not fire")
    # per-frame exchanges: eps_div from the band's luminance sum, the film gathered to rank 0
    i_acc = torch.rand(npx, 3, device="cuda") * 4
    eps = st.eps_div(i_acc)
    lum = ref.film_luminance_sum(i_acc)
    from paper_2510_07868_b200.rrs import eps_div_from_luminance_sum
    if eps != eps_div_from_luminance_sum(float(lum.item()), npx):
        msgs.append(f"eps_div {eps} vs {eps_div_from_luminance_sum(float(lum.item()), npx)}")
    film = torch.rand(npx, 3, dtype=torch.float64, device="cuda")
    full = gather_film(film)
    if full is None or not torch.equal(full, film):
        msgs.append("film gather differs")
    torch.cuda.synchronize()
    dist.destroy_process_group()
    q.put(msgs)


@pytest.mark.timeout(400)
@pytest.mark.parametrize("exchange", ["collective", "mailbox"])
@pytest.mark.parametrize("variant", [0, 1], ids=["nrrs", "aid"])
def test_nccl_world1_sharded_depths_match_plain_stage(exchange, variant):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_port(), exchange, variant, q))
    p.start()
    msgs = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert msgs == []
