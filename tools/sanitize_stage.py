"""Small-n driver for compute-sanitizer (one --tool per gpurun call, B200_PROFILING.md): every kernel
family of the stage once -- AID (K-A0 + K-A + K-B), NRRS and ADRRS-NN (fused-gather K-A), the
throughput heuristic, the slot compaction (K-C), the opt-in fused AID stage -- at ragged sizes.
usage: compute-sanitizer --tool memcheck python tools/sanitize_stage.py"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as orc  # noqa: E402
from helpers import mirror_nets, to_dev  # noqa: E402
from paper_2510_07868_b200 import RateControl, RrsStage, Strategy, StrategyKind, _capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4099
v = to_dev(orc.gen_vertices(n))
for variant, kinds in ((orc.VARIANT_AID, (StrategyKind.AidNrrs, StrategyKind.Throughput)),
                       (orc.VARIANT_NRRS, (StrategyKind.Nrrs, StrategyKind.AdrrsNn))):
    st = RrsStage(n, mirror_nets(orc.OracleNets(variant, seed=1, randomize=True)))
    for kind in kinds:
        out, res = st.run(v, 2, Strategy(kind), rc=RateControl(), full=True)
        used = (torch.arange(st.capacity, device="cuda") % 10 != 0).to(torch.uint8)
        comp = torch.empty((st.capacity, 2), dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
        _capi.check(st.handle, st.ctx.lib.nrrs_gpu_compact(st.handle, out.slots.data_ptr(), used.data_ptr(),
                                                           res.spawned, 2, comp.data_ptr(), cnt.data_ptr(), None))
        torch.cuda.synchronize()
        print(kind.name, "spawned", res.spawned)
    st.close()
os.environ["NRRS_FUSED"] = "1"
m = 8 * 128 * 3 + 77
vm = to_dev(orc.gen_vertices(m))
st = RrsStage(m, mirror_nets(orc.OracleNets(orc.VARIANT_AID, seed=1, randomize=True)))
out, res = st.run(vm, 2, Strategy(StrategyKind.AidNrrs), rc=RateControl(), full=True)
torch.cuda.synchronize()
print("fused spawned", res.spawned)
st.close()
print("sanitize driver ok")
