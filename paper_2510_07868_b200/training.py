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

    def _adam(self, adam: _Adam, theta, grad, shadow, inv_scale: float):
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
