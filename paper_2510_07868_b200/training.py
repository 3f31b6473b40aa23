"""Online training of the StatNet on the GPU (first part).

Mirrors NeuralRrs's StatNet side (networks.hpp:119-271): live parameters, the
two Adam optimizers (grid, MLP), the EMA shadows that become the published
snapshot, and the dynamic loss scale of apply_step / step_statnet
(networks.cpp:462-552).  The loss and gradients run through
nrrs_gpu_stat_loss_grad, the update through nrrs_gpu_adam_ema.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch

from . import _capi
from .networks import NeuralRrs
from .stage import GpuContext

K_MIN_LOSS_SCALE = 1.0 / 65536.0   # networks.cpp:16
K_SCALE_GROWTH_STREAK = 256        # networks.cpp:17


class _Adam:
    """Adam state for one flat parameter vector (optimizer.hpp:13-49)."""

    def __init__(self, n: int, device, lr: float, beta1=0.9, beta2=0.999, eps=1e-8):
        self.m = torch.zeros(n, dtype=torch.float32, device=device)
        self.v = torch.zeros(n, dtype=torch.float32, device=device)
        self.t = 0
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps


class StatNetTrainer:
    """StatNet training on one GPU, starting from a NeuralRrs's live parameters."""

    def __init__(self, nets: NeuralRrs, device: int = 0, ctx: Optional[GpuContext] = None):
        self.ctx = ctx or GpuContext(device)
        self.device = torch.device("cuda", self.ctx.device)
        c = nets.cfg
        self.spec = _capi.GridSpec(c.grid.levels, c.grid.features, c.grid.base_resolution, c.grid.log2_table_size)
        self.grid = torch.from_numpy(np.ascontiguousarray(nets.stat_grid, np.float32)).to(self.device)
        self.mlp = torch.from_numpy(np.ascontiguousarray(nets.stat_mlp, np.float32)).to(self.device)
        self.g_grid = torch.zeros_like(self.grid)
        self.g_mlp = torch.zeros_like(self.mlp)
        lr = getattr(c, "lr_stat", 0.005)
        self.adam_grid = _Adam(self.grid.numel(), self.device, lr)
        self.adam_mlp = _Adam(self.mlp.numel(), self.device, lr)
        self.ema_decay = getattr(c, "ema_decay", 0.99)
        self.shadow_grid = self.grid.clone()  # m_ema_*.reset(theta) (networks.cpp:192-193)
        self.shadow_mlp = self.mlp.clone()
        self.eps = getattr(c, "eps", 0.01)
        self.scale = 1.0
        self.streak = 0
        self.steps = 0
        self.skipped_steps = 0

    def loss_and_grad(self, batch: torch.Tensor, d_scale: float = 1.0):
        """stat_loss_impl on the live parameters -> (loss, finite); gradients in g_mlp / g_grid."""
        self.ctx.bind_stream()
        n = int(batch.shape[0])
        loss, fin = C.c_double(), C.c_int32()
        _capi.check(self.ctx.handle, self.ctx.lib.nrrs_gpu_stat_loss_grad(
            self.ctx.handle, C.byref(self.spec), self.grid.data_ptr(), self.mlp.data_ptr(),
            batch.data_ptr() if n else None, n, float(self.eps), float(d_scale), self.g_mlp.data_ptr(),
            self.g_grid.data_ptr(), C.byref(loss), C.byref(fin)))
        return loss.value, bool(fin.value)

    def _adam(self, adam: "_Adam", theta, grad, shadow, inv_scale: float):
        adam.t += 1
        _capi.check(self.ctx.handle, self.ctx.lib.nrrs_gpu_adam_ema(
            self.ctx.handle, theta.data_ptr(), grad.data_ptr(), adam.m.data_ptr(), adam.v.data_ptr(),
            shadow.data_ptr(), theta.numel(), adam.t, adam.lr, adam.beta1, adam.beta2, adam.eps, float(inv_scale),
            float(self.ema_decay)))

    def step(self, batch: torch.Tensor) -> tuple:
        """NeuralRrs::step_statnet (networks.cpp:532-552) with apply_step (:462-489).
        batch: uint8 [n, 80] TrainSample rows on the device.  Returns (loss, applied)."""
        if batch.shape[0] == 0:
            return 0.0, False
        loss, finite = self.loss_and_grad(batch, self.scale)
        if not np.isfinite(loss) or not finite:
            self.scale = max(self.scale * 0.5, K_MIN_LOSS_SCALE)
            self.streak = 0
            self.skipped_steps += 1
            return loss, False
        inv = np.float32(1.0) / np.float32(self.scale)
        self._adam(self.adam_mlp, self.mlp, self.g_mlp, self.shadow_mlp, inv)
        if self.grid.numel():
            self._adam(self.adam_grid, self.grid, self.g_grid, self.shadow_grid, inv)
        self.streak += 1
        if self.streak >= K_SCALE_GROWTH_STREAK:
            self.scale = min(self.scale * 2.0, 1.0)
            self.streak = 0
        self.steps += 1
        return loss, True

    def publish(self, nets: NeuralRrs) -> NeuralRrs:
        """NeuralRrs::publish (networks.cpp:199-204) for the StatNet: snapshot = EMA shadow."""
        nets.stat_grid = self.shadow_grid.cpu().numpy().copy()
        nets.stat_mlp = self.shadow_mlp.cpu().numpy().copy()
        return nets

    def close(self) -> None:
        self.ctx.close()


PIXEL_ERROR_DTYPE = np.dtype([("e", "<f4"), ("inv_denom", "<f4")])   # PixelError (networks.hpp:89-92)
WARMUP, FULL = 0, 1                                                   # TrainPhase (networks.hpp:84)


class RrsNetTrainer:
    """RRSNet training (NRRS or AID) on one GPU: rrs_loss_impl + apply_step + step_rrsnet
    (networks.cpp:418-460, :462-489, :554-575).  Stats come from the published StatNet snapshot."""

    def __init__(self, nets: NeuralRrs, device: int = 0, ctx: Optional[GpuContext] = None):
        self.ctx = ctx or GpuContext(device)
        self.device = torch.device("cuda", self.ctx.device)
        c = nets.cfg
        self.variant = int(c.variant)
        self.spec = _capi.GridSpec(c.grid.levels, c.grid.features, c.grid.base_resolution, c.grid.log2_table_size)
        dev = self.device
        self.mlp = torch.from_numpy(np.ascontiguousarray(nets.rrs_mlp, np.float32)).to(dev)
        self.grid = torch.from_numpy(np.ascontiguousarray(nets.rrs_grid, np.float32)).to(dev)
        self.g_mlp = torch.zeros_like(self.mlp)
        self.g_grid = torch.zeros_like(self.grid)
        lr = getattr(c, "lr_rrs", 0.0003)
        self.adam_mlp = _Adam(self.mlp.numel(), dev, lr)
        self.adam_grid = _Adam(self.grid.numel(), dev, lr)
        self.ema_decay = getattr(c, "ema_decay", 0.99)
        self.shadow_mlp = self.mlp.clone()
        self.shadow_grid = self.grid.clone()
        self.gamma_min = getattr(c, "gamma_min", 0.05)
        self.gamma_avg = getattr(c, "gamma_avg", 0.01)
        self.gamma_rrs = getattr(c, "gamma_rrs", 0.01)
        self.eps = getattr(c, "eps", 0.01)
        self.scale = 1.0
        self.streak = 0
        self.steps = 0
        self.skipped_steps = 0
        self.skipped_samples = 0

    def loss_and_grad(self, batch: torch.Tensor, snap_stat_grid: torch.Tensor, snap_stat_mlp: torch.Tensor,
                      errors: Optional[torch.Tensor], e_avg: float, phase: int, d_scale: float = 1.0):
        """rrs_loss_impl -> (parts {min, avg, rrs, total}, skipped, finite); gradients in g_mlp / g_grid."""
        self.ctx.bind_stream()
        n = int(batch.shape[0])
        parts = (C.c_double * 4)()
        sk, fin = C.c_uint32(), C.c_int32()
        ne = 0 if errors is None else int(errors.numel() // 2)
        _capi.check(self.ctx.handle, self.ctx.lib.nrrs_gpu_rrs_loss_grad(
            self.ctx.handle, self.variant, C.byref(self.spec), snap_stat_grid.data_ptr(), snap_stat_mlp.data_ptr(),
            self.grid.data_ptr() if self.grid.numel() else None, self.mlp.data_ptr(),
            batch.data_ptr() if n else None, n, errors.data_ptr() if ne else None, ne, float(e_avg), int(phase),
            float(self.gamma_min), float(self.gamma_avg), float(self.gamma_rrs), float(self.eps), float(d_scale),
            self.g_mlp.data_ptr(), self.g_grid.data_ptr() if self.grid.numel() else None, parts, C.byref(sk),
            C.byref(fin)))
        return {"min": parts[0], "avg": parts[1], "rrs": parts[2], "total": parts[3]}, sk.value, bool(fin.value)

    def step(self, batch, snap_stat_grid, snap_stat_mlp, errors, e_avg, phase):
        """NeuralRrs::step_rrsnet -> (parts, applied)."""
        if batch.shape[0] == 0:
            return None, False
        parts, skipped, finite = self.loss_and_grad(batch, snap_stat_grid, snap_stat_mlp, errors, e_avg, phase,
                                                    self.scale)
        self.skipped_samples += skipped
        if not np.isfinite(parts["total"]) or not finite:
            self.scale = max(self.scale * 0.5, K_MIN_LOSS_SCALE)
            self.streak = 0
            self.skipped_steps += 1
            return parts, False
        inv = np.float32(1.0) / np.float32(self.scale)
        StatNetTrainer._adam(self, self.adam_mlp, self.mlp, self.g_mlp, self.shadow_mlp, inv)
        if self.grid.numel():
            StatNetTrainer._adam(self, self.adam_grid, self.grid, self.g_grid, self.shadow_grid, inv)
        self.streak += 1
        if self.streak >= K_SCALE_GROWTH_STREAK:
            self.scale = min(self.scale * 2.0, 1.0)
            self.streak = 0
        self.steps += 1
        return parts, True

    def close(self) -> None:
        self.ctx.close()


class NeuralRrsTrainer:
    """NeuralRrs::train_frame + publish (networks.cpp:199-204, :577-605) on one GPU."""

    def __init__(self, nets: NeuralRrs, device: int = 0, batch: int = 1 << 16):
        self.nets = nets
        self.ctx = GpuContext(device)
        self.stat = StatNetTrainer(nets, ctx=self.ctx)
        self.rrs = RrsNetTrainer(nets, ctx=self.ctx)
        self.batch = int(batch)
        dev = self.stat.device
        # the published snapshot the RRSNet reads its stats from (m_snap_stat_*)
        self.snap_stat_grid = torch.from_numpy(np.ascontiguousarray(nets.stat_grid, np.float32)).to(dev)
        self.snap_stat_mlp = torch.from_numpy(np.ascontiguousarray(nets.stat_mlp, np.float32)).to(dev)

    def train_frame(self, samples: torch.Tensor, errors: Optional[torch.Tensor], e_avg: float, phase: int) -> dict:
        """Chunks of `batch` samples: step_statnet then step_rrsnet per chunk; batch-mean losses."""
        out = {"loss_stat": 0.0, "loss_min": 0.0, "loss_avg": 0.0, "loss_rrs": 0.0, "chunks": 0}
        n = int(samples.shape[0])
        for off in range(0, n, self.batch):
            chunk = samples[off:off + self.batch]
            ls, ok = self.stat.step(chunk)
            if ok:
                out["loss_stat"] += ls
            parts, ok = self.rrs.step(chunk, self.snap_stat_grid, self.snap_stat_mlp, errors, e_avg, phase)
            if ok:
                out["loss_min"] += parts["min"]
                out["loss_avg"] += parts["avg"]
                out["loss_rrs"] += parts["rrs"]
            out["chunks"] += 1
        for k in ("loss_stat", "loss_min", "loss_avg", "loss_rrs"):
            out[k] /= max(out["chunks"], 1)
        return out

    def publish(self) -> NeuralRrs:
        """Snapshot = EMA shadows (networks.cpp:199-204); returns the NeuralRrs for set_weights."""
        self.snap_stat_grid.copy_(self.stat.shadow_grid)
        self.snap_stat_mlp.copy_(self.stat.shadow_mlp)
        self.nets.stat_grid = self.stat.shadow_grid.cpu().numpy().copy()
        self.nets.stat_mlp = self.stat.shadow_mlp.cpu().numpy().copy()
        self.nets.rrs_mlp = self.rrs.shadow_mlp.cpu().numpy().copy()
        if self.rrs.grid.numel():
            self.nets.rrs_grid = self.rrs.shadow_grid.cpu().numpy().copy()
        return self.nets

    def close(self) -> None:
        self.ctx.close()
