"""Host mirror of the reference's NeuralRrs snapshot side (networks.hpp).

Only what the inference stage needs: the hash-grid / MLP specs, the constructor
initialisation (networks.cpp:159-197, reproduced bit-for-bit with the same
counter-based RNG through the C ABI's nrrs_rng_fill), the published snapshot
parameter blocks, and the NRRSCK01 checkpoint interchange (networks.cpp:610-705).
Training (losses, Adam, EMA updates) is out of scope.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import math
import struct

import numpy as np

from . import _capi


class RrsVariant(enum.IntEnum):
    Nrrs = 0
    Aid = 1


@dataclasses.dataclass
class HashGridSpec:
    """hashgrid.hpp:13-22."""
    levels: int = 8
    features: int = 2
    base_resolution: int = 16
    log2_table_size: int = 15

    def output_dim(self) -> int:
        return self.levels * self.features

    def resolution(self, level: int) -> int:
        return self.base_resolution << level

    def table_size(self) -> int:
        return 1 << self.log2_table_size

    def param_count(self) -> int:
        return self.levels * self.table_size() * self.features


EMPTY_GRID = HashGridSpec(levels=0, features=0, base_resolution=1, log2_table_size=0)  # networks.cpp:26-35

HIDDEN, HIDDEN_LAYERS = 32, 3
STAT_TAIL_DIM, NRRS_INPUT_DIM, AID_TAIL_DIM = 16, 11, 16


def mlp_param_count(n_in: int, n_out: int) -> int:
    """mlp.cpp:7-16."""
    dims = [n_in] + [HIDDEN] * HIDDEN_LAYERS + [n_out]
    return sum(dims[l + 1] * dims[l] + dims[l + 1] for l in range(HIDDEN_LAYERS + 1))


def mlp_head_offset(n_in: int, n_out: int) -> int:
    return mlp_param_count(n_in, n_out) - (HIDDEN * n_out + n_out)


def softplus_mod_inverse_pos(y: float) -> float:
    """encodings.hpp:85-88 (float32)."""
    return float(np.float32(2.0) * (np.float32(y) - np.float32(0.6931471805599453)))


def rng_uniform(seed: int, seq: int, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """RngStream(seed, seq).next_float() x n mapped to lo + (hi-lo)*u (float32)."""
    out = np.empty(n, dtype=np.float32)
    if n:
        _capi.lib().nrrs_rng_fill(seed, seq, out.ctypes.data_as(C.POINTER(C.c_float)), n, lo, hi)
    return out


def grid_init(spec: HashGridSpec, seed: int, seq: int) -> np.ndarray:
    """hashgrid.cpp:25-28: U(-1e-4, 1e-4) as (u*2-1)*1e-4 in float32."""
    u = rng_uniform(seed, seq, spec.param_count())
    return ((u * np.float32(2.0) - np.float32(1.0)) * np.float32(1e-4)).astype(np.float32)


def mlp_init(n_in: int, n_out: int, seed: int, seq: int) -> np.ndarray:
    """mlp.cpp:34-44: He-uniform hidden layers in column-major order, zero head."""
    theta = np.zeros(mlp_param_count(n_in, n_out), dtype=np.float32)
    dims = [n_in] + [HIDDEN] * HIDDEN_LAYERS
    count = sum(dims[l] * HIDDEN for l in range(HIDDEN_LAYERS))
    u = rng_uniform(seed, seq, count)
    off, used = 0, 0
    for l in range(HIDDEN_LAYERS):
        li = dims[l]
        bound = np.sqrt(np.float32(6.0) / np.float32(li), dtype=np.float32)
        n = li * HIDDEN
        theta[off:off + n] = (u[used:used + n] * np.float32(2.0) - np.float32(1.0)) * bound
        used += n
        off += n + HIDDEN
    return theta


@dataclasses.dataclass
class NeuralRrsConfig:
    """networks.hpp:84-97 (inference-relevant fields; training knobs kept for checkpoint parity)."""
    variant: RrsVariant = RrsVariant.Nrrs
    grid: HashGridSpec = dataclasses.field(default_factory=HashGridSpec)
    seed: int = 0x9E3779B97F4A7C15


class NeuralRrs:
    """Published-snapshot holder mirroring NeuralRrs (networks.hpp:119-271).

    `stat_grid`, `stat_mlp`, `rrs_grid`, `rrs_mlp` are the snapshot blocks that
    predict_q / predict_stats read (networks.cpp:276-279).  A fresh instance
    equals the reference constructor's published state: the RRSNet is exactly
    the constant 1 (zero head weights, bias softplus_inv(1)).
    """

    def __init__(self, cfg: NeuralRrsConfig | None = None):
        self.cfg = cfg or NeuralRrsConfig()
        c = self.cfg
        self.stat_grid = grid_init(c.grid, c.seed, 0)
        self.stat_mlp = mlp_init(self.stat_input_dim(), 6, c.seed, 1)
        self.rrs_grid = grid_init(c.grid, c.seed, 2) if c.variant == RrsVariant.Aid else np.zeros(0, np.float32)
        self.rrs_mlp = mlp_init(self.rrs_input_dim(), 1, c.seed, 3)
        self.rrs_mlp[-1] = np.float32(softplus_mod_inverse_pos(1.0))  # networks.cpp:186-190

    def stat_input_dim(self) -> int:
        return self.cfg.grid.output_dim() + STAT_TAIL_DIM

    def rrs_input_dim(self) -> int:
        return NRRS_INPUT_DIM if self.cfg.variant == RrsVariant.Nrrs else self.cfg.grid.output_dim() + AID_TAIL_DIM

    def randomize_for_benchmark(self) -> "NeuralRrs":
        """SURVEY.md 8d "random-init RRSNet": heads ~ U(-0.5, 0.5) (test_networks.cpp:407-410),
        StatNet head bias 1, RRSNet head bias softplus_inv(2), grids x 1e4 (test_networks.cpp:337-339).
        Identical to oracle orc_init_nets(randomize=1)."""
        seed = self.cfg.seed
        sh = mlp_head_offset(self.stat_input_dim(), 6)
        self.stat_mlp[sh:] = rng_uniform(seed, 100, self.stat_mlp.size - sh) * np.float32(2.0) - np.float32(1.0)
        self.stat_mlp[sh:] *= np.float32(0.5)
        self.stat_mlp[-6:] = np.float32(1.0)
        rh = mlp_head_offset(self.rrs_input_dim(), 1)
        self.rrs_mlp[rh:] = (rng_uniform(seed, 101, self.rrs_mlp.size - rh) * np.float32(2.0) - np.float32(1.0)) \
            * np.float32(0.5)
        self.rrs_mlp[-1] = np.float32(softplus_mod_inverse_pos(2.0))
        self.stat_grid *= np.float32(1e4)
        if self.rrs_grid.size:
            self.rrs_grid *= np.float32(1e4)
        return self

    # ---- NRRSCK01 (networks.cpp:610-705) ----
    _MAGIC = b"NRRSCK01"

    def save_checkpoint(self, path: str) -> None:
        """Writes a NRRSCK01 v1 file whose live, EMA and snapshot blocks all hold the
        snapshot (inference-only state), zero Adam moments and unit loss scales."""
        c = self.cfg
        blocks = [self.stat_grid, self.stat_mlp, self.rrs_grid, self.rrs_mlp]
        with open(path, "wb") as f:
            f.write(self._MAGIC)
            f.write(struct.pack("<II", 1, int(c.variant)))
            f.write(struct.pack("<iiii", c.grid.levels, c.grid.features, c.grid.base_resolution,
                                c.grid.log2_table_size))
            f.write(struct.pack("<ii", self.stat_input_dim(), self.rrs_input_dim()))
            for _ in range(3):  # live, ema shadow, snapshot
                for b in blocks:
                    f.write(struct.pack("<Q", b.size))
                    f.write(np.ascontiguousarray(b, dtype="<f4").tobytes())
            for b in blocks:  # adam moment1, moment2, step per block
                for _ in range(2):
                    f.write(struct.pack("<Q", b.size))
                    f.write(np.zeros(b.size, dtype="<f4").tobytes())
                f.write(struct.pack("<q", 0))
            f.write(struct.pack("<ffIIQQ", 1.0, 1.0, 0, 0, 0, 0))

    def load_checkpoint(self, path: str) -> None:
        """Reads the snapshot blocks; rejects mismatched magic/version/variant/spec (runtime_error)."""
        c = self.cfg
        with open(path, "rb") as f:
            data = f.read()
        pos = 0

        def take(n):
            nonlocal pos
            if pos + n > len(data):
                raise RuntimeError("checkpoint: truncated file")
            out = data[pos:pos + n]
            pos += n
            return out

        if take(8) != self._MAGIC:
            raise RuntimeError("checkpoint: bad magic")
        version, variant = struct.unpack("<II", take(8))
        if version != 1:
            raise RuntimeError("checkpoint: unsupported version")
        if variant != int(c.variant):
            raise RuntimeError("checkpoint: variant mismatch")
        spec = struct.unpack("<iiii", take(16))
        if spec != (c.grid.levels, c.grid.features, c.grid.base_resolution, c.grid.log2_table_size):
            raise RuntimeError("checkpoint: grid spec mismatch")
        if struct.unpack("<ii", take(8)) != (self.stat_input_dim(), self.rrs_input_dim()):
            raise RuntimeError("checkpoint: input layout mismatch")
        sizes = [c.grid.param_count(), mlp_param_count(self.stat_input_dim(), 6),
                 c.grid.param_count() if c.variant == RrsVariant.Aid else 0,
                 mlp_param_count(self.rrs_input_dim(), 1)]
        groups = []
        for _ in range(3):
            g = []
            for s in sizes:
                (n,) = struct.unpack("<Q", take(8))
                if n != s:
                    raise RuntimeError("checkpoint: parameter block size mismatch")
                g.append(np.frombuffer(take(4 * n), dtype="<f4").astype(np.float32))
            groups.append(g)
        snap = groups[2]
        self.stat_grid, self.stat_mlp, self.rrs_grid, self.rrs_mlp = snap

    def weights_c(self):
        """nrrs_net_weights view (keeps numpy buffers alive on the returned object)."""
        c = self.cfg
        arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in
                (self.stat_grid, self.stat_mlp, self.rrs_grid, self.rrs_mlp)]
        fp = C.POINTER(C.c_float)
        w = _capi.NetWeights(
            int(c.variant),
            _capi.GridSpec(c.grid.levels, c.grid.features, c.grid.base_resolution, c.grid.log2_table_size),
            arrs[0].ctypes.data_as(fp), arrs[0].size, arrs[1].ctypes.data_as(fp), arrs[1].size,
            arrs[2].ctypes.data_as(fp) if arrs[2].size else None, arrs[2].size,
            arrs[3].ctypes.data_as(fp), arrs[3].size)
        w._keep = arrs
        return w
