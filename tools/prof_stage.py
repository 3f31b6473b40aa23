"""Minimal driver for ncu captures: runs the stage (K-A, K-B) and the slot compaction (K-C, ~10%
invalid slots as in bench.py) on a synthetic batch `reps` times.
usage: python tools/prof_stage.py [aid|nrrs|adrrs|throughput] [n] [reps]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_07868_b200 import (NeuralRrs, NeuralRrsConfig, RateControl, RrsStage, RrsVariant, Strategy,
                                   StrategyKind, _capi, synthetic)

kind = sys.argv[1] if len(sys.argv) > 1 else "aid"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1920 * 1080
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
variant = RrsVariant.Nrrs if kind == "nrrs" else RrsVariant.Aid
nets = NeuralRrs(NeuralRrsConfig(variant=variant, seed=1)).randomize_for_benchmark()
strat = {"aid": StrategyKind.AidNrrs, "nrrs": StrategyKind.Nrrs, "adrrs": StrategyKind.AdrrsNn,
         "throughput": StrategyKind.Throughput}[kind]
hv = synthetic.gen_vertices(n)
dv = {k: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).cuda() for k, a in hv.items()
      if k != "pixel"}
st = RrsStage(n, nets)
out = st.alloc_outputs(n)
cap = st.capacity
idx = torch.arange(cap, dtype=torch.int64, device="cuda")
used = (((idx * 2654435761) >> 7) % 10 != 0).to(torch.uint8)
compacted = torch.empty((cap, 2), dtype=torch.int32, device="cuda")
d_count = torch.zeros(1, dtype=torch.int32, device="cuda")
lib = _capi.lib()


def step():
    res = st.run(dv, 2, Strategy(strat), rc=RateControl(), out=out, sync=False)
    _capi.check(st.handle, lib.nrrs_gpu_compact(st.handle, out.slots.data_ptr(), used.data_ptr(), cap, 2,
                                                compacted.data_ptr(), d_count.data_ptr(), None))
    return res


for _ in range(reps):
    step()
torch.cuda.synchronize()
times = []
for _ in range(max(reps, 1)):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    step()
    b.record()
    torch.cuda.synchronize()
    times.append(a.elapsed_time(b))
times.sort()
print(f"{kind} n={n}: stage+compact {times[len(times) // 2]:.3f} ms (median of {len(times)}, min {times[0]:.3f})")
