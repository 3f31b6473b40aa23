"""NVTX check: two eager AID stage calls (300,000 vertices), for
ncu --nvtx --nvtx-include "nrrs@nrrs_gpu_rrs_stage/" python tools/nvtx_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_07868_b200 import NeuralRrs, NeuralRrsConfig, RateControl, RrsStage, RrsVariant, Strategy, StrategyKind, synthetic
n = 300_000
hv = synthetic.gen_vertices(n, n_pixels=n)
dv = {k: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).cuda() for k, a in hv.items() if k != "pixel"}
st = RrsStage(n, NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Aid, seed=1)).randomize_for_benchmark())
for _ in range(2):
    st.run(dv, 2, Strategy(StrategyKind.AidNrrs), rc=RateControl())
torch.cuda.synchronize()
print("ok")
