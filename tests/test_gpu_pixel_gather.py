"""GPU: the stage's film-gather input mode against the per-vertex mode, on every kernel path.

The reference reads i_pixel = film.i_acc[v.pixel] inside the stage (wavefront.cpp:378); the ABI
takes either i_pixel per vertex or (pixel, i_acc) and gathers it on the device (the staged K-A
paths read the pixel index by TMA and gather from L2).  With i_acc[pixel[j]] == i_pixel[j] by
construction (pixels shuffled, several vertices per pixel), both modes must give the same
factors and decisions bit for bit; the per-vertex mode is itself the oracle-pinned one
(test_gpu_parity.py, test_gpu_headline.py).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle as orc
from helpers import mirror_nets, to_dev
from paper_2510_07868_b200 import RateControl, RrsStage, Strategy, StrategyKind

pytestmark = pytest.mark.gpu
FIELDS = ("q_orig", "u", "q_norm", "q_real", "k", "offset", "decided")


@pytest.mark.parametrize("variant,kind,n,fused", [
    (orc.VARIANT_AID, StrategyKind.AidNrrs, 1_000_003, None),  # K-A0 + K-A (staged rows) + K-B
    (orc.VARIANT_AID, StrategyKind.AidNrrs, 65_536, None),     # the fused single-kernel stage
    (orc.VARIANT_NRRS, StrategyKind.Nrrs, 300_001, None),      # StatNet planes + 8-layer chain
    (orc.VARIANT_NRRS, StrategyKind.AdrrsNn, 300_001, None),   # StatNet planes, ADRRS head
    (orc.VARIANT_NRRS, StrategyKind.Throughput, 300_001, None),  # heuristic kernel
], ids=["aid-3k", "aid-fused", "nrrs", "adrrs-nn", "throughput"])
def test_film_gather_equals_per_vertex_i_pixel(variant, kind, n, fused, monkeypatch):
    if fused is not None:
        monkeypatch.setenv("NRRS_FUSED", fused)
    npx = n // 3 + 1
    v = orc.gen_vertices(n, n_pixels=npx)
    g = np.random.default_rng(17)
    pixel = g.permutation(np.arange(n, dtype=np.int64) % npx).astype(np.uint32)
    i_acc = (np.float32(0.25) + g.random((npx, 3), dtype=np.float32)).astype(np.float32)
    v["i_pixel"] = np.ascontiguousarray(i_acc[pixel])
    nets = orc.OracleNets(variant, seed=1, randomize=True)
    st = RrsStage(npx, mirror_nets(nets), capacity=3 * n)
    dv = to_dev(v)
    eps = 1e-3
    ref_o, ref_r = st.run(dv, 2, Strategy(kind), rc=RateControl(), eps_div=eps, full=True)
    torch.cuda.synchronize()
    ref = {f: getattr(ref_o, f).clone() for f in FIELDS}
    gv = {k: t for k, t in dv.items() if k != "i_pixel"}
    gv["pixel"] = torch.from_numpy(pixel.view(np.int32)).cuda()
    gv["i_acc"] = torch.from_numpy(i_acc).cuda()
    out, r = st.run(gv, 2, Strategy(kind), rc=RateControl(), eps_div=eps, full=True)
    torch.cuda.synchronize()
    for f in FIELDS:
        assert torch.equal(getattr(out, f), ref[f]), f
    assert torch.equal(out.slots[:r.spawned], ref_o.slots[:ref_r.spawned])
    assert (r.f_norm, r.sum_q, r.total, r.spawned, r.dropped) == \
        (ref_r.f_norm, ref_r.sum_q, ref_r.total, ref_r.spawned, ref_r.dropped)
    st.close()
