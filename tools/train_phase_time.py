"""Device time of one StatNet loss_and_grad and one AID RRSNet loss_and_grad (CUDA events, mean of
20 after warm-up) on the bench's 65,536-sample batch -- for A/B of training-kernel variants.
usage: python tools/train_phase_time.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as orc  # noqa: E402  (synthetic TrainSamples, host-side input only)
from paper_2510_07868_b200 import NeuralRrs, NeuralRrsConfig, RrsVariant  # noqa: E402
from paper_2510_07868_b200.training import FULL, NeuralRrsTrainer  # noqa: E402

nb = 1 << 16
hb = orc.gen_train_batch(nb, seed=5)
hb["q_real"] = np.float32(1.5)
hb["q_norm"] = np.float32(1.2)
db = torch.from_numpy(hb.view(np.uint8).reshape(nb, 80).copy()).cuda()
nets = NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Aid, seed=1)).randomize_for_benchmark()
tr = NeuralRrsTrainer(nets, batch=nb)
errs = torch.rand((1024, 2), dtype=torch.float32, device="cuda")


def timed(name, f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    z.record()
    torch.cuda.synchronize()
    print(f"{name:28s} {a.elapsed_time(z) * 1e3 / reps:8.1f} us")


timed("stat loss_and_grad", lambda: tr.stat.loss_and_grad(db))
timed("rrs (AID) loss_and_grad", lambda: tr.rrs.loss_and_grad(db, tr.snap_stat_grid, tr.snap_stat_mlp, errs, 0.5, FULL))
timed("train_frame", lambda: tr.train_frame(db, errs, 0.5, FULL))
tr.close()
