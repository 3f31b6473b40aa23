"""GPU: independent contexts running at the same time on their own streams.

The ABI is one context per device per host thread, stream-ordered; several
contexts share the device.  Every piece of launch bookkeeping (look-back tile states and epochs,
last-CTA-done counters, the fused stage's grid-barrier words, the exact-sum words) lives in its
context, and the single-wave prefix claims tiles dynamically, so kernels of other contexts occupying
SMs cannot deadlock it.  Here three contexts -- the three-kernel AID path, the cooperative fused
stage and NRRS -- are driven round-robin on three streams with no synchronization in between, and
each one's final outputs must equal its own eager, isolated call bit for bit.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2510_07868_b200 import (NeuralRrs, NeuralRrsConfig, RateControl, RrsStage, RrsVariant, Strategy,
                                   StrategyKind, synthetic)

pytestmark = pytest.mark.gpu
FIELDS = ("q_orig", "u", "q_norm", "q_real", "k", "offset", "decided")


def test_three_contexts_on_three_streams():
    cases = [(RrsVariant.Aid, StrategyKind.AidNrrs, 1_000_003), (RrsVariant.Aid, StrategyKind.AidNrrs, 65_536),
             (RrsVariant.Nrrs, StrategyKind.Nrrs, 300_001)]
    setups = []
    for variant, kind, n in cases:
        st = RrsStage(n, NeuralRrs(NeuralRrsConfig(variant=variant, seed=1)).randomize_for_benchmark())
        hv = synthetic.gen_vertices(n, n_pixels=n)
        dv = {k: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).cuda() for k, a in hv.items()
              if k != "pixel"}
        ref_o, ref_r = st.run(dv, 2, Strategy(kind), rc=RateControl(), full=True)
        torch.cuda.synchronize()
        ref = {f: getattr(ref_o, f).clone() for f in FIELDS}
        out = st.alloc_outputs(n, full=True)
        setups.append((st, kind, dv, out, ref, ref_o.slots[:ref_r.spawned].clone(), ref_r))
    streams = [torch.cuda.Stream() for _ in setups]
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    for _ in range(12):  # round-robin, no host wait: the three streams overlap on the device
        for (st, kind, dv, out, *_), s in zip(setups, streams):
            with torch.cuda.stream(s):
                st.run(dv, 2, Strategy(kind), rc=RateControl(), out=out, sync=False)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    for st, kind, dv, out, ref, ref_slots, ref_r in setups:
        for f in FIELDS:
            assert torch.equal(getattr(out, f), ref[f]), f
        assert torch.equal(out.slots[:ref_r.spawned], ref_slots)
        r = st.fetch_result()
        assert (r.f_norm, r.sum_q, r.spawned, r.dropped) == (ref_r.f_norm, ref_r.sum_q, ref_r.spawned, ref_r.dropped)
        st.close()
