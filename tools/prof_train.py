"""Driver for ncu launch lists of the online-training step: `reps`
StatNetTrainer.step calls and NeuralRrsTrainer.train_frame chunks (AID, full phase) on the bench's
synthetic 65,536-sample batch.  usage: python tools/prof_train.py [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as orc  # noqa: E402  (synthetic TrainSamples, host-side input only)
from paper_2510_07868_b200 import NeuralRrs, NeuralRrsConfig, RrsVariant  # noqa: E402
from paper_2510_07868_b200.training import FULL, NeuralRrsTrainer, StatNetTrainer  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
nb = 1 << 16
hb = orc.gen_train_batch(nb, seed=5)
db = torch.from_numpy(hb.view(np.uint8).reshape(nb, 80).copy()).cuda()
tr = StatNetTrainer(NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Nrrs, seed=1)).randomize_for_benchmark())
for _ in range(reps):
    t0 = time.perf_counter()
    tr.step(db)
    torch.cuda.synchronize()
    print(f"step_statnet {1e3 * (time.perf_counter() - t0):.3f} ms")
nets = NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Aid, seed=1)).randomize_for_benchmark()
ntr = NeuralRrsTrainer(nets, batch=nb)
hb2 = hb.copy()
hb2["q_real"] = np.float32(1.5)
hb2["q_norm"] = np.float32(1.2)
db2 = torch.from_numpy(hb2.view(np.uint8).reshape(nb, 80).copy()).cuda()
errs = torch.rand((1024, 2), dtype=torch.float32, device="cuda")
for _ in range(reps):
    t0 = time.perf_counter()
    ntr.train_frame(db2, errs, 0.5, FULL)
    torch.cuda.synchronize()
    print(f"train_frame {1e3 * (time.perf_counter() - t0):.3f} ms")
ntr.close()
