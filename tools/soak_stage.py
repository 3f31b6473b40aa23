"""Race soak of the stage kernels (race detection; compute-sanitizer is closed
on the GPU pool).  For each configuration one eager call gives the reference outputs; then a CUDA
graph of `calls` back-to-back stage calls is replayed `replays` times, the outputs poisoned before
every replay, and after every replay the outputs (q_orig, u, q_norm, q_real, k, offset, decided,
the spawned slot records) and the result scalars must equal the reference bit for bit.  A race in
the look-back / single-wave prefix, the grid barrier of the fused stage, the mbarrier / TMEM
pipelines of K-A or the epoch reset of the launch bookkeeping shows up as a mismatch.
usage: python tools/soak_stage.py [replays] [calls]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_07868_b200 import (NeuralRrs, NeuralRrsConfig, RateControl, RrsStage, RrsVariant, Strategy,  # noqa
                                   StrategyKind, synthetic)

replays = int(sys.argv[1]) if len(sys.argv) > 1 else 300
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 10
CONFIGS = [  # (name, variant, strategy, n, env)
    ("aid 2073600 (K-A0 + K-A + K-B)", RrsVariant.Aid, StrategyKind.AidNrrs, 2_073_600, {}),
    ("aid 65536 (fused stage)", RrsVariant.Aid, StrategyKind.AidNrrs, 65_536, {}),
    ("aid 196609 (three kernels)", RrsVariant.Aid, StrategyKind.AidNrrs, 196_609, {}),
    ("aid 1000003 (fused, forced)", RrsVariant.Aid, StrategyKind.AidNrrs, 1_000_003, {"NRRS_FUSED": "1"}),
    ("nrrs 300001", RrsVariant.Nrrs, StrategyKind.Nrrs, 300_001, {}),
    ("adrrs-nn 1228800", RrsVariant.Nrrs, StrategyKind.AdrrsNn, 1_228_800, {}),
    ("throughput 4194305 (multi-wave K-B)", RrsVariant.Nrrs, StrategyKind.Throughput, 4_194_305, {}),
]
fields = ("q_orig", "u", "q_norm", "q_real", "k", "offset", "decided")
total_calls, failures = 0, 0
print(f"# {replays} replays x {calls} calls per configuration; outputs poisoned before each replay")
for name, variant, kind, n, env in CONFIGS:
    for k, v in env.items():
        os.environ[k] = v
    try:
        nets = NeuralRrs(NeuralRrsConfig(variant=variant, seed=1)).randomize_for_benchmark()
        st = RrsStage(n, nets)
    finally:
        for k in env:
            del os.environ[k]
    hv = synthetic.gen_vertices(n, n_pixels=n)
    dv = {k: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).cuda() for k, a in hv.items()
          if k != "pixel"}
    gain = RateControl().gain()
    out = st.alloc_outputs(n, full=True)
    ref_o, ref_r = st.run(dv, 2, Strategy(kind), rc=RateControl(), full=True)
    torch.cuda.synchronize()
    ref = {f: getattr(ref_o, f).clone() for f in fields}
    ref_slots = ref_o.slots[:ref_r.spawned].clone()
    g = st.capture(dv, 2, Strategy(kind), out, gain=gain, calls=calls)
    bad = 0
    t0 = time.perf_counter()
    for rep in range(replays):
        for f in fields:
            getattr(out, f).fill_(-1 if getattr(out, f).dtype != torch.uint8 else 255)
        out.slots.fill_(-1)
        g.replay()
        ok = all(torch.equal(getattr(out, f), ref[f]) for f in fields)
        ok = ok and torch.equal(out.slots[:ref_r.spawned], ref_slots)
        r = st.fetch_result()
        ok = ok and (r.f_norm, r.total, r.spawned, r.dropped, r.nonfinite) == \
            (ref_r.f_norm, ref_r.total, ref_r.spawned, ref_r.dropped, ref_r.nonfinite)
        if not ok:
            bad += 1
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    total_calls += replays * calls
    failures += bad
    print(f"{name:38s} {replays * calls:7d} calls  mismatching replays: {bad}  ({dt:.1f} s)")
    st.close()
# the mailbox exchange (one rank, its own mailbox): a graph of 4 depths (factors, mailbox decide,
# mailbox clip), generations advancing on the device across every replay
import ctypes as C  # noqa: E402

from paper_2510_07868_b200 import _capi  # noqa: E402
from paper_2510_07868_b200.sharded import connect_mailboxes_in_process, mailbox_check, mailbox_depth  # noqa: E402
from paper_2510_07868_b200.stage import vertex_soa  # noqa: E402

n = 500_000
nets = NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Aid, seed=1)).randomize_for_benchmark()
hv = synthetic.gen_vertices(n, n_pixels=n)
dv = {k: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).cuda() for k, a in hv.items()
      if k != "pixel"}
ref_st = RrsStage(n, nets)
ref_o, ref_r = ref_st.run(dv, 2, Strategy(StrategyKind.AidNrrs), rc=RateControl(), full=True)
torch.cuda.synchronize()
st = RrsStage(n, nets)
connect_mailboxes_in_process([st])
out = st.alloc_outputs(n, full=True)
local_sum = torch.zeros(1, dtype=torch.float64, device="cuda")
total = torch.zeros(1, dtype=torch.int64, device="cuda")
p = st.params(2, Strategy(StrategyKind.AidNrrs), RateControl().gain(), 0.0, n_pixels=n)
soa = vertex_soa(dv)


def depth():
    st.ctx.bind_stream()
    oc = out.c()
    _capi.check(st.handle, st.ctx.lib.nrrs_gpu_stage_factors(st.handle, C.byref(soa), n, C.byref(p), C.byref(oc),
                                                             local_sum.data_ptr()))
    return mailbox_depth(st, n, p, out, total, 1, 0, st.capacity, n)


side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    depth()
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(4):
        pend = depth()
bad = 0
t0 = time.perf_counter()
for rep in range(replays):
    out.k.fill_(-1)
    out.slots.fill_(-1)
    g.replay()
    o = pend.resolve()
    ok = (o.spawned, o.dropped, o.kept) == (ref_r.spawned, ref_r.dropped, ref_r.spawned)
    ok = ok and torch.equal(out.k, ref_o.k) and torch.equal(out.slots[:ref_r.spawned], ref_o.slots[:ref_r.spawned])
    bad += 0 if ok else 1
mailbox_check(st)
dt = time.perf_counter() - t0
print(f"{'mailbox depths (aid 500000, world 1)':38s} {replays * 4:7d} depths mismatching replays: {bad}  ({dt:.1f} s)")
total_calls += replays * 4
failures += bad
st.close()
ref_st.close()
print(f"# total {total_calls} stage calls / depths, {failures} mismatching replays")
sys.exit(1 if failures else 0)
