"""Synthetic path-vertex batches of SURVEY.md 8(d), vectorized (numpy).

Vertex i draws from its own stream RngStream(0xC0FFEE, i) (the per-index
convention of nrrs_cli.cpp:121-125) in the order of test_networks.cpp:37-51:
p01 = (g,g,g), wo01 = (g,g), roughness = g, t_x = 0.2+(g,g,g),
i_pixel = 0.5+(g,g,g); pixel = i mod Npx; path_key = root_path_key(pixel, frame).
The "split bound 4" factors are RngStream(0xACC02, i).next_float()*4.
This is input generation for tests/bench (host side), not part of the stage.
"""
from __future__ import annotations

import numpy as np

_MUL = np.uint64(6364136223846793005)


def mix_bits(x: np.ndarray) -> np.ndarray:
    """rng.hpp:8-13 on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


class VecRng:
    """RngStream (rng.hpp:33-65) for a vector of independent streams."""

    def __init__(self, seed: int, sequence: np.ndarray):
        seq = np.asarray(sequence, dtype=np.uint64)
        self.inc = (seq << np.uint64(1)) | np.uint64(1)
        self.state = np.zeros_like(seq)
        self.next_u32()
        with np.errstate(over="ignore"):
            self.state = self.state + mix_bits(np.uint64(seed))
        self.next_u32()

    def next_u32(self) -> np.ndarray:
        old = self.state
        with np.errstate(over="ignore"):
            self.state = old * _MUL + self.inc
        xs = (((old >> np.uint64(18)) ^ old) >> np.uint64(27)).astype(np.uint32)
        rot = (old >> np.uint64(59)).astype(np.uint32)
        return (xs >> rot) | (xs << ((np.uint32(32) - rot) & np.uint32(31)))

    def next_float(self) -> np.ndarray:
        return (self.next_u32() >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)


def root_path_key(pixel: np.ndarray, frame: int) -> np.ndarray:
    return mix_bits((np.uint64(frame) << np.uint64(32)) | np.asarray(pixel, dtype=np.uint64))


def gen_vertices(n: int, n_pixels: int | None = None, frame: int = 0, first: int = 0, chunk: int = 1 << 20) -> dict:
    """SoA dict of numpy arrays for vertices first .. first+n-1."""
    n_pixels = n if n_pixels is None else n_pixels
    v = {"p01": np.empty((n, 3), np.float32), "wo01": np.empty((n, 2), np.float32),
         "roughness": np.empty(n, np.float32), "weight": np.empty((n, 3), np.float32),
         "i_pixel": np.empty((n, 3), np.float32), "path_key": np.empty(n, np.uint64),
         "pixel": np.empty(n, np.uint32)}
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        idx = np.arange(first + s, first + e, dtype=np.uint64)
        g = VecRng(0xC0FFEE, idx)
        for c in range(3):
            v["p01"][s:e, c] = g.next_float()
        for c in range(2):
            v["wo01"][s:e, c] = g.next_float()
        v["roughness"][s:e] = g.next_float()
        for c in range(3):
            v["weight"][s:e, c] = np.float32(0.2) + g.next_float()
        for c in range(3):
            v["i_pixel"][s:e, c] = np.float32(0.5) + g.next_float()
        px = (idx % np.uint64(max(n_pixels, 1))).astype(np.uint32)
        v["pixel"][s:e] = px
        v["path_key"][s:e] = root_path_key(px, frame)
    return v


def split_bound_factors(n: int, first: int = 0) -> np.ndarray:
    g = VecRng(0xACC02, np.arange(first, first + n, dtype=np.uint64))
    return g.next_float() * np.float32(4.0)
