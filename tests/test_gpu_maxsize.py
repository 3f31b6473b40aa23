"""GPU: the maximum batch the benchmark configs name -- configs[4]'s 16M-vertex wavefront batch
(3840 x 2160 film, two vertices per pixel: 16,588,800 vertices) -- on ONE GPU.

At this size the 32-bit plane offsets of K-A0 (up to 16 fp32 planes x 16.6M = 1.06 GB), K-A's
~112 tiles per MLP group, K-B's multi-wave decoupled look-back and K-C run far past every other
test.  The oracle cannot run 16.6M vertices in test time on one core, so parity is checked through
size-independent properties:

* q_orig and u on a strided sample of 65,536 vertices against the oracle on the same vertices
  (the factor of a vertex depends only on that vertex: networks.cpp:266-281, rng.hpp);
* the whole decision chain (normalize_factors over all 16.6M q, realize_counts, plan_spawns, slot
  layout: rrs.cpp:8-45, wavefront.cpp:141-154, :390-425) on the GPU's own q and u, bit-exact.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle as orc
from helpers import mirror_nets, oracle_decide, rel_err, to_dev
from paper_2510_07868_b200 import RateControl, RrsStage, Strategy, StrategyKind

pytestmark = pytest.mark.gpu
REL_TOL = 1e-3
NPX = 3840 * 2160
N = 2 * NPX


def _np(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("variant,kind", [(orc.VARIANT_AID, orc.AID_NRRS), (orc.VARIANT_NRRS, orc.NRRS)],
                         ids=["aid", "nrrs"])
def test_configs4_batch_on_one_gpu(variant, kind):
    v = orc.gen_vertices(N, n_pixels=NPX)
    v["weight"][::97] = 0.0  # zero-throughput vertices (undecided, q = 0) spread over every tile
    on = orc.OracleNets(variant, seed=1, randomize=True)
    st = RrsStage(NPX, mirror_nets(on))
    out, res = st.run(to_dev(v), 2, Strategy(StrategyKind(kind)), rc=RateControl(), full=True)
    torch.cuda.synchronize()
    q, u = _np(out.q_orig), _np(out.u)

    idx = np.linspace(0, N - 1, 65_536).astype(np.int64)
    idx[-1] = N - 1  # the last tile's last row
    sub = {k: np.ascontiguousarray(a[idx]) for k, a in v.items()}
    ref = orc.rrs_stage(sub, 2, NPX, st.capacity, kind, on, gain=0.85, seed=0, threads=orc.threads_available())
    err = rel_err(q[idx], ref["q_orig"], 1e-6)
    assert err.max() <= REL_TOL, f"q_orig max rel err {err.max():.3e} at vertex {int(idx[err.argmax()])}"
    np.testing.assert_array_equal(u[idx], ref["u"])
    np.testing.assert_array_equal(_np(out.decided)[idx], ref["decided"])
    assert np.all(q[::97] == 0.0)

    dec = oracle_decide(q, u, NPX, st.capacity, 0.85)
    assert np.float32(res.f_norm) == np.float32(dec["f_norm"])
    np.testing.assert_array_equal(_np(out.q_norm), dec["q_norm"])
    np.testing.assert_array_equal(_np(out.k), dec["k"])
    np.testing.assert_array_equal(_np(out.offset).view(np.uint32), dec["offset"])
    assert res.total == dec["total"] and res.spawned == dec["spawned"] and res.dropped == dec["dropped"]
    assert res.spawned > 1_000_000
    np.testing.assert_array_equal(_np(out.slots)[:res.spawned].view(np.uint32), dec["slots"])
    st.close()
