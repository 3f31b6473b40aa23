"""A/B check of the grid-gradient fold: dumps the StatNet and AID RRSNet grid gradients (and the
MLP gradients) of one loss_and_grad on the bench's 65,536-sample batch, so two library builds can
be compared bit for bit.  usage: python tools/fold_ab.py out.npz"""
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
errs = torch.rand((1024, 2), dtype=torch.float32, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
tr.stat.loss_and_grad(db)
tr.rrs.loss_and_grad(db, tr.snap_stat_grid, tr.snap_stat_mlp, errs, 0.5, FULL)
torch.cuda.synchronize()
out = {"stat_g_grid": tr.stat.g_grid.cpu().numpy(), "stat_g_mlp": tr.stat.g_mlp.cpu().numpy(),
       "rrs_g_grid": tr.rrs.g_grid.cpu().numpy(), "rrs_g_mlp": tr.rrs.g_mlp.cpu().numpy()}
for _ in range(3):
    tr.train_frame(db, errs, 0.5, FULL)
torch.cuda.synchronize()
out["stat_grid_after"] = tr.stat.grid.cpu().numpy()
out["rrs_grid_after"] = tr.rrs.grid.cpu().numpy()
np.savez(sys.argv[1], **out)
print({k: (v.shape, float(np.abs(v).sum())) for k, v in out.items()})
tr.close()
