"""Shared test helpers: device transfer, oracle-side decision from given factors."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

import oracle as orc
from paper_2510_07868_b200.networks import HashGridSpec, NeuralRrs, NeuralRrsConfig, RrsVariant


def to_dev(v: dict, device="cuda") -> dict:
    out = {}
    for k, a in v.items():
        if k == "pixel":
            continue
        if a.dtype == np.uint64:
            out[k] = torch.from_numpy(a.view(np.int64)).to(device)
        else:
            out[k] = torch.from_numpy(np.ascontiguousarray(a)).to(device)
    return out


def mirror_nets(on: orc.OracleNets) -> NeuralRrs:
    """Host-mirror NeuralRrs holding exactly the oracle's snapshot arrays."""
    s = on.spec
    cfg = NeuralRrsConfig(variant=RrsVariant(on.variant),
                          grid=HashGridSpec(s.levels, s.features, s.base_resolution, s.log2_table_size), seed=1)
    n = NeuralRrs.__new__(NeuralRrs)
    n.cfg = cfg
    n.stat_grid, n.stat_mlp, n.rrs_grid, n.rrs_mlp = (on.stat_grid.copy(), on.stat_mlp.copy(), on.rrs_grid.copy(),
                                                      on.rrs_mlp.copy())
    return n


def oracle_decide(q_orig: np.ndarray, u: np.ndarray, n_pixels: int, capacity: int, gain: float) -> dict:
    """normalize_factors -> q_real -> realize_counts -> plan_spawns -> slot layout, via the oracle."""
    q = np.ascontiguousarray(q_orig, np.float32).copy()
    f = orc.normalize_factors(q, n_pixels)
    q_real = (q * np.float32(gain)).astype(np.float32)
    k = np.zeros(q.size, np.int32)
    err = C.c_int(0)
    u = np.ascontiguousarray(u, np.float32)
    total = orc.lib().orc_realize_counts(orc.ptr(q_real), orc.ptr(u), orc.ptr(k), q.size, C.byref(err))
    assert err.value == 0
    off, spawned, dropped = orc.plan_spawns(k, capacity)
    rem = spawned - np.minimum(spawned, off.astype(np.int64))
    kept = np.minimum(k.astype(np.int64), rem)
    parents = np.repeat(np.arange(q.size, dtype=np.uint32), kept)
    starts = np.repeat(np.cumsum(kept) - kept, kept)
    child = (np.arange(parents.size) - starts).astype(np.uint32)
    return {"q_norm": q, "q_real": q_real, "k": k, "offset": off, "total": int(total), "spawned": spawned,
            "dropped": dropped, "f_norm": f, "slots": np.stack([parents, child], 1)}


def rel_err(a: np.ndarray, b: np.ndarray, floor: float = 1e-30) -> np.ndarray:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(np.abs(b), floor)
