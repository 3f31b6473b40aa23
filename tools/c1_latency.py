"""C1 / configs[0] latency probe: per-call time of 65,536-vertex stage calls replayed from a CUDA
graph (100 calls per graph), per strategy and routing; env knobs are read at context creation.
usage: python tools/c1_latency.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_07868_b200 import (NeuralRrs, NeuralRrsConfig, RateControl, RrsStage, RrsVariant, Strategy,  # noqa
                                   StrategyKind, synthetic)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
hv = synthetic.gen_vertices(n, n_pixels=n)
dv = {k: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).cuda() for k, a in hv.items()
      if k != "pixel"}


def probe(name, variant, kind, env=None, val="1"):
    if env:
        os.environ[env] = val
    try:
        nets = NeuralRrs(NeuralRrsConfig(variant=variant, seed=1)).randomize_for_benchmark()
        st = RrsStage(n, nets)
    finally:
        if env:
            del os.environ[env]
    o = st.alloc_outputs(n)
    for _ in range(5):
        st.run(dv, 2, Strategy(kind), rc=RateControl(), out=o, sync=False)
    g = st.capture(dv, 2, Strategy(kind), o, gain=RateControl().gain(), calls=100)
    g.replay()
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    z.record()
    torch.cuda.synchronize()
    print(f"{name:34s} {a.elapsed_time(z) * 1e3 / 500:7.2f} us/call")
    st.close()


probe("aid (default routing)", RrsVariant.Aid, StrategyKind.AidNrrs)
probe("aid (fused-gather K-A, no K-A0)", RrsVariant.Aid, StrategyKind.AidNrrs, "NRRS_NO_LEVEL_KERNEL")
probe("aid (fused single kernel)", RrsVariant.Aid, StrategyKind.AidNrrs, "NRRS_FUSED")
probe("aid (K-A0 + K-A + K-B)", RrsVariant.Aid, StrategyKind.AidNrrs, "NRRS_FUSED", "0")
probe("nrrs", RrsVariant.Nrrs, StrategyKind.Nrrs)
probe("nrrs (L2-gather K-A, no K-A0)", RrsVariant.Nrrs, StrategyKind.Nrrs, "NRRS_NO_LEVEL_KERNEL")
probe("adrrs-nn (L2-gather K-A, no K-A0)", RrsVariant.Nrrs, StrategyKind.AdrrsNn, "NRRS_NO_LEVEL_KERNEL")
probe("adrrs-nn", RrsVariant.Nrrs, StrategyKind.AdrrsNn)
probe("throughput", RrsVariant.Nrrs, StrategyKind.Throughput)
