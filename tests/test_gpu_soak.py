"""GPU: a short race soak (the long one is tools/soak_stage.py, profiles/r02_soak.txt).

A CUDA graph of back-to-back stage calls is replayed with the outputs poisoned before every replay;
every replay must reproduce the eager call bit for bit.  This exercises what a race would break:
the single-wave prefix and the decoupled look-back of K-B (epochs across replays), the grid barrier
and the TMEM-parked (q, u) of the fused stage, K-A's mbarrier / TMEM pipelines, and the exact sum.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2510_07868_b200 import (NeuralRrs, NeuralRrsConfig, RateControl, RrsStage, RrsVariant, Strategy,
                                   StrategyKind, synthetic)

pytestmark = pytest.mark.gpu
FIELDS = ("q_orig", "u", "q_norm", "q_real", "k", "offset", "decided")


@pytest.mark.parametrize("variant,kind,n,fused", [
    (RrsVariant.Aid, StrategyKind.AidNrrs, 2_073_600, None),
    (RrsVariant.Aid, StrategyKind.AidNrrs, 65_536, None),
    (RrsVariant.Aid, StrategyKind.AidNrrs, 700_001, "1"),
    (RrsVariant.Nrrs, StrategyKind.Nrrs, 300_001, None),
    (RrsVariant.Nrrs, StrategyKind.Throughput, 4_194_305, None),
], ids=["aid-3k", "aid-fused-small", "aid-fused-forced", "nrrs", "throughput-multiwave"])
def test_graph_replays_reproduce_the_eager_call(variant, kind, n, fused, monkeypatch):
    if fused is not None:
        monkeypatch.setenv("NRRS_FUSED", fused)
    st = RrsStage(n, NeuralRrs(NeuralRrsConfig(variant=variant, seed=1)).randomize_for_benchmark())
    hv = synthetic.gen_vertices(n, n_pixels=n)
    dv = {k: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).cuda() for k, a in hv.items()
          if k != "pixel"}
    ref_o, ref_r = st.run(dv, 2, Strategy(kind), rc=RateControl(), full=True)
    torch.cuda.synchronize()
    ref = {f: getattr(ref_o, f).clone() for f in FIELDS}
    ref_slots = ref_o.slots[:ref_r.spawned].clone()
    out = st.alloc_outputs(n, full=True)
    g = st.capture(dv, 2, Strategy(kind), out, gain=RateControl().gain(), calls=4)
    for _ in range(40):
        for f in FIELDS:
            getattr(out, f).fill_(255 if f == "decided" else -1)
        out.slots.fill_(-1)
        g.replay()
        for f in FIELDS:
            assert torch.equal(getattr(out, f), ref[f]), f
        assert torch.equal(out.slots[:ref_r.spawned], ref_slots)
        r = st.fetch_result()
        assert (r.f_norm, r.sum_q, r.total, r.spawned, r.dropped) == \
            (ref_r.f_norm, ref_r.sum_q, ref_r.total, ref_r.spawned, ref_r.dropped)
    st.close()
