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


def gen_cornell_vertices(width: int, height: int, frame: int = 0) -> dict:
    """Render-like, spatially coherent depth-2 batch in pixel order (SURVEY.md 8d "render-derived
    batches"): the first surface hit of each pixel's primary ray in a closed unit box seen from
    inside (camera (0.5, 0.5, 0.02) looking +z), walls at 0 and 1 on every axis plus one block.
    p01 is the hit point (walls give p = 0 and p = 1 exactly: the encoder's clamp edge),
    wo01 the spherical direction back to the camera, roughness 1 on diffuse walls and 0.3 on the
    block, t_x the Cornell albedos, i_pixel a smooth per-pixel estimate.  Not a renderer: an input
    generator with the memory-access coherence of a real frame (the stage is otherwise unchanged)."""
    n = width * height
    pix = np.arange(n, dtype=np.uint64)
    px = (pix % np.uint64(width)).astype(np.float64)
    py = (pix // np.uint64(width)).astype(np.float64)
    aspect = width / height
    dx = ((px + 0.5) / width - 0.5) * aspect * 1.2
    dy = (0.5 - (py + 0.5) / height) * 1.2
    d = np.stack([dx, dy, np.ones(n)], axis=1)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = np.array([0.5, 0.5, 0.02])
    with np.errstate(divide="ignore", invalid="ignore"):
        tw = np.full(n, np.inf)
        face = np.zeros(n, np.int64)  # 0 left 1 right 2 floor 3 ceiling 4 back 5 block
        for axis, lo_face, hi_face in ((0, 0, 1), (1, 2, 3)):
            t_lo = np.where(d[:, axis] < 0, (0.0 - o[axis]) / d[:, axis], np.inf)
            t_hi = np.where(d[:, axis] > 0, (1.0 - o[axis]) / d[:, axis], np.inf)
            for t, f in ((t_lo, lo_face), (t_hi, hi_face)):
                m = t < tw
                tw = np.where(m, t, tw)
                face = np.where(m, f, face)
        t_back = (1.0 - o[2]) / d[:, 2]
        m = t_back < tw
        tw = np.where(m, t_back, tw)
        face = np.where(m, 4, face)
        bmin, bmax = np.array([0.18, 0.0, 0.45]), np.array([0.48, 0.55, 0.75])
        t1 = (bmin - o) / d
        t2 = (bmax - o) / d
        tn = np.max(np.minimum(t1, t2), axis=1)
        tf = np.min(np.maximum(t1, t2), axis=1)
        hit_b = (tn <= tf) & (tn > 0) & (tn < tw)
        tw = np.where(hit_b, tn, tw)
        face = np.where(hit_b, 5, face)
    p = np.clip(o + tw[:, None] * d, 0.0, 1.0)
    for axis, lo_face, hi_face in ((0, 0, 1), (1, 2, 3)):  # walls exactly on the boundary
        p[face == lo_face, axis] = 0.0
        p[face == hi_face, axis] = 1.0
    p[face == 4, 2] = 1.0
    w = -d
    theta = np.arccos(np.clip(w[:, 2], -1.0, 1.0)) / np.pi
    phi = (np.arctan2(w[:, 1], w[:, 0]) / (2 * np.pi)) + 0.5
    albedo = np.array([[0.63, 0.065, 0.05], [0.14, 0.45, 0.091], [0.725, 0.71, 0.68], [0.725, 0.71, 0.68],
                       [0.725, 0.71, 0.68], [0.8, 0.8, 0.8]], np.float32)
    rough = np.where(face == 5, 0.3, 1.0).astype(np.float32)
    ipix = 0.5 + 0.3 * np.stack([np.sin(px / width * 6.0 + c) * np.cos(py / height * 4.0 - c)
                                 for c in (0.0, 1.0, 2.0)], axis=1)
    return {"p01": p.astype(np.float32), "wo01": np.stack([theta, phi], axis=1).astype(np.float32),
            "roughness": rough, "weight": albedo[face], "i_pixel": ipix.astype(np.float32),
            "path_key": root_path_key(pix.astype(np.uint32), frame), "pixel": pix.astype(np.uint32)}
