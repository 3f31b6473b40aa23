"""ctypes wrapper of oracle/liborc.so -- the CPU CHECKER (test infrastructure only).

Imported by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs,
never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib
import subprocess

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
ORACLE_DIR = ROOT / "oracle"
LIB = ORACLE_DIR / "liborc.so"

FIXED, THROUGHPUT, ADRRS_TREE, ADRRS_NN, NRRS, AID_NRRS = range(6)
VARIANT_NRRS, VARIANT_AID = 0, 1


class GridSpec(C.Structure):
    _fields_ = [("levels", C.c_int), ("features", C.c_int), ("base_resolution", C.c_int),
                ("log2_table_size", C.c_int)]


class Nets(C.Structure):
    _fields_ = [("variant", C.c_int), ("grid", GridSpec), ("stat_grid", C.c_void_p), ("stat_mlp", C.c_void_p),
                ("rrs_grid", C.c_void_p), ("rrs_mlp", C.c_void_p)]


class Vertices(C.Structure):
    _fields_ = [("p01", C.c_void_p), ("wo01", C.c_void_p), ("roughness", C.c_void_p), ("weight", C.c_void_p),
                ("i_pixel", C.c_void_p), ("path_key", C.c_void_p)]


class StageParams(C.Structure):
    _fields_ = [("depth", C.c_uint32), ("n_pixels", C.c_uint32), ("capacity", C.c_uint32), ("kind", C.c_int),
                ("fixed_value", C.c_float), ("gain", C.c_float), ("eps_div", C.c_float), ("seed", C.c_uint64),
                ("threads", C.c_int)]


class StageOut(C.Structure):
    _fields_ = [("q_orig", C.c_void_p), ("q_norm", C.c_void_p), ("q_real", C.c_void_p), ("u", C.c_void_p),
                ("k", C.c_void_p), ("offset", C.c_void_p), ("decided", C.c_void_p), ("slots", C.c_void_p),
                ("f_norm", C.c_double), ("sum_q", C.c_double), ("total", C.c_uint64), ("spawned", C.c_uint32),
                ("dropped", C.c_uint64), ("nonfinite", C.c_uint64)]


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "liborc.so"], check=True)
    if pathlib.Path("/root/reference/proj/include/nrrs/rng.hpp").exists():
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "ref"], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        src = ORACLE_DIR / "nrrs_oracle.c"
        if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
            build()
        L = C.CDLL(str(LIB))
        f, d, u32, u64, i, p = C.c_float, C.c_double, C.c_uint32, C.c_uint64, C.c_int, C.c_void_p
        sig = {
            "orc_mix_bits": (u64, [u64]), "orc_mix_bits2": (u64, [u64, u64]),
            "orc_rng_init": (None, [p, u64, u64]), "orc_rng_next_u32": (u32, [p]), "orc_rng_next_float": (f, [p]),
            "orc_child_path_key": (u64, [u64, u32]), "orc_root_path_key": (u64, [u32, u32]),
            "orc_rrs_uniform": (f, [u64, u64, u32]), "orc_luminance": (f, [p]),
            "orc_stochastic_round": (i, [f, f]), "orc_one_blob": (None, [f, i, p]), "orc_box_cox": (f, [f]),
            "orc_roughness_remap": (f, [f]), "orc_softplus_mod": (f, [f]),
            "orc_softplus_mod_inverse_pos": (f, [f]), "orc_box_cox_clamps": (u64, []),
            "orc_reset_box_cox_clamps": (None, []),
            "orc_grid_param_count": (C.c_size_t, [p]), "orc_grid_encode": (None, [p, p, p, p]),
            "orc_mlp_param_count": (i, [i, i]), "orc_mlp_head_offset": (i, [i, i]),
            "orc_mlp_forward": (None, [i, i, p, p, p]),
            "orc_build_stat_tail": (None, [p, f, p]), "orc_build_nrrs_input": (None, [p, p, p, p, f, p]),
            "orc_build_aid_tail": (None, [p, p, p, f, p]),
            "orc_predict_stats": (None, [p, p, p, f, p]), "orc_predict_q": (f, [p, p, p, f, p, p]),
            "orc_adrrs_factor": (f, [p, p, p, f]),
            "orc_strategy_factor": (f, [i, f, p, p, p, p, f, p, f]),
            "orc_normalize_factors": (d, [p, C.c_size_t, u64, p]),
            "orc_realize_counts": (u64, [p, p, p, C.c_size_t, p]), "orc_bernstein_bound": (d, [d, u64]),
            "orc_queue_capacity_for": (u32, [u32]), "orc_plan_spawns": (None, [p, C.c_size_t, u32, p, p, p, p]),
            "orc_rrs_stage": (None, [p, C.c_size_t, p, p, p]),
            "orc_compact_slots": (u32, [p, p, u32, p]),
            "orc_gen_vertices": (None, [C.c_size_t, u32, u32, p, p, p, p, p, p, p]),
            "orc_gen_split_bound_factors": (None, [C.c_size_t, p]),
            "orc_init_nets": (None, [i, p, u64, i, p, p, p, p]),
            "orc_fold_ordered": (None, [p, p, p, C.c_size_t]),
            "orc_emit_train": (C.c_size_t, [u32, C.c_size_t, p, p, p, p, p, p, p, p, p, p, p, p]),
            "orc_train_k_i": (None, [p, C.c_size_t, C.c_size_t, u32]),
            "orc_film_add_frame": (None, [p, p, p, p, C.c_size_t]),
            "orc_film_roll_acc": (None, [p, p, C.c_size_t]),
            "orc_relative_l2": (None, [f, f, f, p, p]),
            "orc_stat_loss": (d, [p, p, p, p, C.c_size_t, f, f, p, p]),
            "orc_adam_step": (None, [p, p, p, p, C.c_size_t, C.c_int64, f, f, f, f]),
            "orc_rrs_loss": (None, [i, p, p, p, p, p, p, C.c_size_t, p, C.c_size_t, f, i, f, f, f, f, f, p, p, p]),
            "orc_ema_update": (None, [p, p, C.c_size_t, f]),
            "orc_camera_ray": (None, [p, p, p, f, f, f, f, p, p]),
            "orc_path_floats2": (None, [u64, u64, u32, u64, p, p]),
            "orc_intersect_brute": (None, [p, p, u32, p, p, f, p, p, p, p]),
            "orc_render_depth1": (None, [p, u32, u32, u64, u32, p, p, p, p, p, p, p, p, p]),
            "orc_trace_frame": (i, [p, p, p, p, p, p, p, p, p, C.c_size_t, p, p]),
            "orc_bsdf_sample": (i, [i, p, f, p, p, f, f, p, p, p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


# ---------------------------------------------------------------------------
class OracleNets:
    """Snapshot weights held by the oracle (orc_init_nets)."""

    def __init__(self, variant: int, levels=8, features=2, base=16, log2t=15, seed=1, randomize=True,
                 arrays=None):
        self.variant = variant
        self.spec = GridSpec(levels, features, base, log2t)
        gn = levels * (1 << log2t) * features
        gd = levels * features
        self.stat_in = gd + 16
        self.rrs_in = 11 if variant == VARIANT_NRRS else gd + 16
        L = lib()
        if arrays is not None:
            self.stat_grid, self.stat_mlp, self.rrs_grid, self.rrs_mlp = [np.ascontiguousarray(a, np.float32)
                                                                          for a in arrays]
        else:
            self.stat_grid = np.zeros(gn, np.float32)
            self.stat_mlp = np.zeros(L.orc_mlp_param_count(self.stat_in, 6), np.float32)
            self.rrs_grid = np.zeros(gn if variant == VARIANT_AID else 0, np.float32)
            self.rrs_mlp = np.zeros(L.orc_mlp_param_count(self.rrs_in, 1), np.float32)
            L.orc_init_nets(variant, C.byref(self.spec), seed, int(randomize), ptr(self.stat_grid),
                            ptr(self.stat_mlp), ptr(self.rrs_grid) if self.rrs_grid.size else None,
                            ptr(self.rrs_mlp))
        self.c = Nets(variant, self.spec, ptr(self.stat_grid), ptr(self.stat_mlp),
                      ptr(self.rrs_grid) if self.rrs_grid.size else None, ptr(self.rrs_mlp))


def gen_vertices(n: int, n_pixels: int | None = None, frame: int = 0) -> dict:
    """SURVEY.md 8d synthetic vertex batch (RngStream(0xC0FFEE, i) per vertex)."""
    n_pixels = n if n_pixels is None else n_pixels
    v = {"p01": np.empty((n, 3), np.float32), "wo01": np.empty((n, 2), np.float32),
         "roughness": np.empty(n, np.float32), "weight": np.empty((n, 3), np.float32),
         "i_pixel": np.empty((n, 3), np.float32), "path_key": np.empty(n, np.uint64),
         "pixel": np.empty(n, np.uint32)}
    lib().orc_gen_vertices(n, n_pixels, frame, ptr(v["p01"]), ptr(v["wo01"]), ptr(v["roughness"]),
                           ptr(v["weight"]), ptr(v["i_pixel"]), ptr(v["path_key"]), ptr(v["pixel"]))
    return v


def split_bound_factors(n: int) -> np.ndarray:
    q = np.empty(n, np.float32)
    lib().orc_gen_split_bound_factors(n, ptr(q))
    return q


def rrs_stage(v: dict, depth: int, n_pixels: int, capacity: int, kind: int, nets: OracleNets | None = None,
              fixed_value: float = 1.0, gain: float = 0.85, eps_div: float = 0.0, seed: int = 0,
              threads: int = 1) -> dict:
    """The reference's RRS decision block (wavefront.cpp:363-425) restated in C."""
    n = int(v["roughness"].shape[0])
    vc = Vertices(ptr(v["p01"]), ptr(v["wo01"]), ptr(v["roughness"]), ptr(v["weight"]), ptr(v["i_pixel"]),
                  ptr(v["path_key"]))
    p = StageParams(depth, n_pixels, capacity, kind, fixed_value, gain, eps_div, seed, threads)
    out = {"q_orig": np.zeros(n, np.float32), "q_norm": np.zeros(n, np.float32), "q_real": np.zeros(n, np.float32),
           "u": np.zeros(n, np.float32), "k": np.zeros(n, np.int32), "offset": np.zeros(n, np.uint32),
           "decided": np.zeros(n, np.uint8), "slots": np.zeros((max(capacity, 1), 2), np.uint32)}
    o = StageOut(*(ptr(out[k]) for k in ("q_orig", "q_norm", "q_real", "u", "k", "offset", "decided", "slots")))
    lib().orc_rrs_stage(C.byref(vc), n, C.byref(p), C.byref(nets.c) if nets is not None else None, C.byref(o))
    out.update(f_norm=o.f_norm, sum_q=o.sum_q, total=o.total, spawned=o.spawned, dropped=o.dropped,
               nonfinite=o.nonfinite)
    return out


def normalize_factors(q: np.ndarray, n_pixels: int):
    err = C.c_int(0)
    f = lib().orc_normalize_factors(ptr(q), q.size, n_pixels, C.byref(err))
    if err.value:
        raise RuntimeError("normalize_factors: factors must be finite and >= 0")
    return f


def plan_spawns(counts: np.ndarray, capacity: int):
    counts = np.ascontiguousarray(counts, np.int32)
    off = np.zeros(counts.size, np.uint32)
    sp, dr, err = C.c_uint32(0), C.c_uint64(0), C.c_int(0)
    lib().orc_plan_spawns(ptr(counts), counts.size, capacity, ptr(off), C.byref(sp), C.byref(dr), C.byref(err))
    if err.value:
        raise RuntimeError("plan_spawns: negative count")
    return off, sp.value, dr.value


def compact_slots(slots: np.ndarray, used: np.ndarray, count: int) -> np.ndarray:
    out = np.zeros((max(count, 1), 2), np.uint32)
    slots = np.ascontiguousarray(slots, np.uint32)
    used = np.ascontiguousarray(used, np.uint8)
    w = lib().orc_compact_slots(ptr(slots), ptr(used), count, ptr(out))
    return out[:w]


def predict_q(nets: OracleNets, v: dict) -> np.ndarray:
    n = int(v["roughness"].shape[0])
    q = np.empty(n, np.float32)
    L = lib()
    for i in range(n):
        q[i] = L.orc_predict_q(C.byref(nets.c), ptr(v["p01"][i]), ptr(v["wo01"][i]), float(v["roughness"][i]),
                               ptr(v["weight"][i]), ptr(v["i_pixel"][i]))
    return q


def strategy_factors(kind: int, v: dict, nets: OracleNets | None, eps_div: float, fixed_value: float = 1.0):
    n = int(v["roughness"].shape[0])
    q = np.empty(n, np.float32)
    L = lib()
    for i in range(n):
        q[i] = L.orc_strategy_factor(kind, fixed_value, C.byref(nets.c) if nets else None, ptr(v["weight"][i]),
                                     ptr(v["p01"][i]), ptr(v["wo01"][i]), float(v["roughness"][i]),
                                     ptr(v["i_pixel"][i]), eps_div)
    return q


def grid_encode(spec: GridSpec, theta: np.ndarray, p01: np.ndarray) -> np.ndarray:
    """HashGrid::encode (hashgrid.cpp:38-82) per point: [n, levels * features] float32."""
    L = lib()
    theta = np.ascontiguousarray(theta, np.float32)
    p01 = np.ascontiguousarray(p01, np.float32).reshape(-1, 3)
    out = np.zeros((p01.shape[0], spec.levels * spec.features), np.float32)
    for i in range(p01.shape[0]):
        L.orc_grid_encode(C.byref(spec), ptr(theta), p01[i].ctypes.data, out[i].ctypes.data)
    return out


def predict_stats(nets: OracleNets, v: dict) -> np.ndarray:
    n = int(v["roughness"].shape[0])
    st = np.empty((n, 6), np.float32)
    L = lib()
    for i in range(n):
        L.orc_predict_stats(C.byref(nets.c), ptr(v["p01"][i]), ptr(v["wo01"][i]), float(v["roughness"][i]),
                            ptr(st[i]))
    return st


def threads_available() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---- suffix side of trace_frame ----
TRAIN_SAMPLE_DTYPE = np.dtype([("position", "<f4", 3), ("omega_o", "<f4", 2), ("roughness", "<f4"),
                               ("t_x", "<f4", 3), ("i_pixel", "<f4", 3), ("lo_sample", "<f4", 3),
                               ("q_norm", "<f4"), ("q_real", "<f4"), ("pixel", "<u4"), ("k_i", "<f4"),
                               ("depth", "<u2"), ("pad", "<u2")])


def fold_ordered(dst: np.ndarray, keys: np.ndarray, terms: np.ndarray) -> None:
    """In place: dst[keys[i]] += terms[i] (f64 x3), item order, negative keys skipped."""
    keys = np.ascontiguousarray(keys, dtype=np.int32)
    terms = np.ascontiguousarray(terms, dtype=np.float64)
    assert dst.dtype == np.float64 and dst.flags.c_contiguous
    lib().orc_fold_ordered(ptr(dst), ptr(keys), ptr(terms), keys.size)


def reverse_pass(verts: list) -> None:
    for d in range(len(verts) - 1, 1, -1):
        fold_ordered(verts[d - 1]["s"], verts[d]["parent"], verts[d]["s"])


def emit_train(verts: list, i_acc: np.ndarray, n_pixels: int):
    """TrainSamples for depths 1..B-1 then k_i (wavefront.cpp:510-543) -> (records, nonfinite)."""
    total = sum(int(verts[d]["pixel"].size) for d in range(1, len(verts)))
    out = np.zeros(max(total, 1), TRAIN_SAMPLE_DTYPE)
    nf = C.c_uint64(0)
    w = 0
    for d in range(1, len(verts)):
        v = {k: np.ascontiguousarray(a) for k, a in verts[d].items()}
        n = int(v["pixel"].size)
        sub = out[w:]
        w += lib().orc_emit_train(d, n, ptr(v["p01"]), ptr(v["wo01"]), ptr(v["roughness"]), ptr(v["weight"]),
                                  ptr(v["pixel"]), ptr(v["q_norm"]), ptr(v["q_real"]), ptr(v["decided"]),
                                  ptr(v["s"]), ptr(np.ascontiguousarray(i_acc)), sub.ctypes.data, C.byref(nf))
    lib().orc_train_k_i(out.ctypes.data, 0, w, n_pixels)
    return out[:w], nf.value


def film_add_frame(sum_: np.ndarray, samples: np.ndarray, i_cur: np.ndarray, frame: np.ndarray) -> None:
    lib().orc_film_add_frame(ptr(sum_), ptr(samples), ptr(i_cur), ptr(np.ascontiguousarray(frame)), samples.size)


def film_roll_acc(i_acc: np.ndarray, i_cur: np.ndarray) -> None:
    lib().orc_film_roll_acc(ptr(i_acc), ptr(i_cur), i_acc.size // 3)


def gen_vertex_tree(depth_sizes: list, n_pixels: int, seed: int = 7) -> list:
    """Synthetic per-depth VertexRec SoA in queue order (pixel and parent non-decreasing):
    index 0 unused, depth 1 has one vertex per pixel prefix, deeper vertices pick sorted parents.
    s (f64) holds the vertices' own film terms before the reverse pass."""
    g = np.random.default_rng(seed)
    verts = [None]
    prev_pixel = None
    for d, n in enumerate(depth_sizes, start=1):
        if d == 1:
            pixel = np.sort(g.integers(0, n_pixels, n)).astype(np.uint32)
            parent = np.full(n, -1, np.int32)
        else:
            parent = np.sort(g.integers(0, depth_sizes[d - 2], n)).astype(np.int32)
            pixel = prev_pixel[parent]
        w = (g.random((n, 3), dtype=np.float32) * np.float32(2.0) - np.float32(0.25)).astype(np.float32)
        s = g.standard_normal((n, 3)) * 3.0
        s[g.random(n) < 0.002, 1] = np.inf  # non-finite suffix -> counted, no sample
        verts.append({"parent": parent, "pixel": pixel, "weight": w, "s": s,
                      "p01": g.random((n, 3), dtype=np.float32), "wo01": g.random((n, 2), dtype=np.float32),
                      "roughness": g.random(n, dtype=np.float32),
                      "q_norm": g.random(n, dtype=np.float32) * np.float32(3),
                      "q_real": g.random(n, dtype=np.float32) * np.float32(3),
                      "decided": (g.random(n) < 0.8).astype(np.uint8)})
        prev_pixel = pixel
    return verts


# ---- StatNet training step ----
def stat_loss(nets: "OracleNets", batch: np.ndarray, eps: float = 0.01, d_scale: float = 1.0, grads: bool = True):
    """NeuralRrs::stat_loss_impl -> (loss, g_mlp, g_grid) (gradients None when grads=False)."""
    batch = np.ascontiguousarray(batch, dtype=TRAIN_SAMPLE_DTYPE)
    gm = np.zeros_like(nets.stat_mlp) if grads else None
    gg = np.zeros_like(nets.stat_grid) if grads else None
    loss = lib().orc_stat_loss(C.byref(nets.spec), ptr(nets.stat_grid), ptr(nets.stat_mlp), batch.ctypes.data,
                               batch.size, eps, d_scale, ptr(gm), ptr(gg))
    return loss, gm, gg


def adam_step(theta, grad, m, v, t, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    lib().orc_adam_step(ptr(theta), ptr(np.ascontiguousarray(grad, np.float32)), ptr(m), ptr(v), theta.size, t,
                        lr, beta1, beta2, eps)


def ema_update(shadow, theta, decay=0.99):
    lib().orc_ema_update(ptr(shadow), ptr(theta), theta.size, decay)


def gen_train_batch(n: int, seed: int = 11) -> np.ndarray:
    """Synthetic TrainSamples (position, omega_o, roughness, lo_sample), test_networks.cpp:37-51 style."""
    g = np.random.default_rng(seed)
    b = np.zeros(n, TRAIN_SAMPLE_DTYPE)
    b["position"] = g.random((n, 3), dtype=np.float32)
    b["omega_o"] = g.random((n, 2), dtype=np.float32)
    b["roughness"] = g.random(n, dtype=np.float32)
    b["t_x"] = np.float32(0.2) + g.random((n, 3), dtype=np.float32)
    b["lo_sample"] = np.float32(0.5) + g.random((n, 3), dtype=np.float32)
    b["pixel"] = g.integers(0, 1024, n).astype(np.uint32)
    b["k_i"] = 1.0
    b["depth"] = 2
    return b


class RrsParts(C.Structure):
    _fields_ = [("min", C.c_double), ("avg", C.c_double), ("rrs", C.c_double), ("total", C.c_double),
                ("skipped", C.c_uint32)]


PIXEL_ERROR_DTYPE = np.dtype([("e", "<f4"), ("inv_denom", "<f4")])
GAMMA_MIN, GAMMA_AVG, GAMMA_RRS, LOSS_EPS = 0.05, 0.01, 0.01, 0.01   # NeuralRrsConfig (networks.hpp:94-106)


def rrs_loss(nets: "OracleNets", snap_stat_grid, snap_stat_mlp, batch, errors, e_avg: float, phase: int,
             d_scale: float = 1.0, grads: bool = True):
    """NeuralRrs::rrs_loss_impl -> (parts, g_mlp, g_grid)."""
    batch = np.ascontiguousarray(batch, dtype=TRAIN_SAMPLE_DTYPE)
    errors = np.ascontiguousarray(errors, dtype=PIXEL_ERROR_DTYPE)
    gm = np.zeros_like(nets.rrs_mlp) if grads else None
    gg = np.zeros_like(nets.rrs_grid) if (grads and nets.rrs_grid.size) else None
    parts = RrsParts()
    lib().orc_rrs_loss(nets.variant, C.byref(nets.spec), ptr(snap_stat_grid), ptr(snap_stat_mlp),
                       ptr(nets.rrs_grid) if nets.rrs_grid.size else None, ptr(nets.rrs_mlp), batch.ctypes.data,
                       batch.size, errors.ctypes.data, errors.size, e_avg, phase, GAMMA_MIN, GAMMA_AVG, GAMMA_RRS,
                       LOSS_EPS, d_scale, ptr(gm), ptr(gg), C.byref(parts))
    return parts, gm, gg


def gen_pixel_errors(n_pixels: int, seed: int = 13) -> np.ndarray:
    g = np.random.default_rng(seed)
    e = np.zeros(n_pixels, PIXEL_ERROR_DTYPE)
    e["e"] = g.random(n_pixels, dtype=np.float32) * np.float32(2.0)
    e["inv_denom"] = np.float32(1.0) / (g.random(n_pixels, dtype=np.float32) + np.float32(0.01))
    return e


# ---- render front-end ----
class OrcScene(C.Structure):
    _fields_ = [("pos", C.c_void_p), ("idx", C.c_void_p), ("mat_of_tri", C.c_void_p), ("n_vert", C.c_uint32),
                ("n_tri", C.c_uint32), ("mat_kind", C.c_void_p), ("mat_albedo", C.c_void_p),
                ("mat_roughness", C.c_void_p), ("mat_emission", C.c_void_p), ("cam_pos", C.c_float * 3),
                ("cam_look", C.c_float * 3), ("cam_up", C.c_float * 3), ("vfov", C.c_float)]


def render_depth1(desc, width: int, height: int, seed: int, frame: int) -> dict:
    """orc_render_depth1: camera rays, brute-force closest hits, dispatch class, surface fields."""
    pos, idx, mid = desc.arrays()
    kind = np.array([m.kind for m in desc.materials], np.int32)
    alb = np.array([m.albedo for m in desc.materials], np.float32).reshape(-1)
    rough = np.array([m.roughness for m in desc.materials], np.float32)
    emi = np.array([m.emission for m in desc.materials], np.float32).reshape(-1)
    f3 = lambda v: (C.c_float * 3)(*[float(np.float32(x)) for x in v])
    cam = desc.camera
    sc = OrcScene(pos.ctypes.data, idx.ctypes.data, mid.ctypes.data, pos.shape[0], mid.size, kind.ctypes.data,
                  alb.ctypes.data, rough.ctypes.data, emi.ctypes.data, f3(cam.position), f3(cam.look_at),
                  f3(cam.up), float(np.float32(cam.vfov_deg)))
    n = width * height
    out = {"o": np.zeros((n, 3), np.float32), "d": np.zeros((n, 3), np.float32), "t": np.zeros(n, np.float32),
           "tri": np.zeros(n, np.uint32), "class": np.zeros(n, np.uint8), "p01": np.zeros((n, 3), np.float32),
           "wo01": np.zeros((n, 2), np.float32), "roughness": np.zeros(n, np.float32),
           "path_key": np.zeros(n, np.uint64)}
    lib().orc_render_depth1(C.byref(sc), width, height, seed & (2**64 - 1), frame, ptr(out["o"]), ptr(out["d"]),
                            ptr(out["t"]), ptr(out["tri"]), ptr(out["class"]), ptr(out["p01"]), ptr(out["wo01"]),
                            ptr(out["roughness"]), ptr(out["path_key"]))
    return out


def intersect_brute(pos: np.ndarray, idx: np.ndarray, o: np.ndarray, d: np.ndarray, t_max=None) -> dict:
    """Bvh::intersect_brute_force per ray (geometry.cpp:46-70 in triangle order)."""
    n = o.shape[0]
    pos = np.ascontiguousarray(pos, np.float32)
    idx = np.ascontiguousarray(idx, np.uint32)
    o = np.ascontiguousarray(o, np.float32)
    d = np.ascontiguousarray(d, np.float32)
    t = np.zeros(n, np.float32)
    tri = np.zeros(n, np.uint32)
    u = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    L = lib()
    ft, fu, fv, ut = C.c_float(), C.c_float(), C.c_float(), C.c_uint32()
    n_tri = idx.size // 3
    for r in range(n):
        tm = np.float32(np.inf) if t_max is None else np.float32(t_max[r])
        L.orc_intersect_brute(pos.ctypes.data, idx.ctypes.data, n_tri, o[r].ctypes.data, d[r].ctypes.data,
                              float(tm), C.byref(ft), C.byref(ut), C.byref(fu), C.byref(fv))
        t[r], tri[r], u[r], v[r] = ft.value, ut.value, fu.value, fv.value
    return {"t": t, "tri": tri, "u": u, "v": v}


def _rng(seed: int, seq: int):
    r = (C.c_uint64 * 2)()
    lib().orc_rng_init(r, seed, seq)
    return r


def random_soup(tris: int, seed: int):
    """test_geometry.cpp:14-29 random_soup (arguments drawn left to right): positions [3*tris, 3] f32,
    indices [3*tris] u32, material ids [tris] (all 0)."""
    L = lib()
    r = _rng(seed, 0)
    nf = lambda: np.float32(L.orc_rng_next_float(r))
    pos = np.zeros((3 * tris, 3), np.float32)
    f4, f2, f07, h = np.float32(4), np.float32(2), np.float32(0.7), np.float32(0.5)
    for i in range(tris):
        base = np.array([nf() * f4 - f2 for _ in range(3)], np.float32)
        for k in range(3):
            jit = np.array([nf() - h for _ in range(3)], np.float32)
            pos[3 * i + k] = base + f07 * jit
    return pos, np.arange(3 * tris, dtype=np.uint32), np.zeros(tris, np.uint32)


def random_rays(n: int, seed: int, seq: int, extent: float = 8.0, t_max: bool = False):
    """test_geometry.cpp:47-53 / :70-75: origins in [-extent/2, extent/2)^3, random_unit directions
    (:31-38), optional t_max = 2 + 4u."""
    L = lib()
    r = _rng(seed, seq)
    nf = lambda: np.float32(L.orc_rng_next_float(r))
    e, he = np.float32(extent), np.float32(extent / 2)
    o = np.zeros((n, 3), np.float32)
    d = np.zeros((n, 3), np.float32)
    tm = np.full(n, np.inf, np.float32)
    one, two = np.float32(1), np.float32(2)
    for i in range(n):
        o[i] = [nf() * e - he for _ in range(3)]
        while True:
            v = np.array([nf() * two - one for _ in range(3)], np.float32)
            n2 = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]
            if np.float32(1e-4) < n2 < one:
                d[i] = v / np.sqrt(n2)
                break
        if t_max:
            tm[i] = np.float32(2) + np.float32(4) * nf()
    return o, d, tm


class OrcTraceCfg(C.Structure):
    _fields_ = [("width", C.c_uint32), ("height", C.c_uint32), ("max_depth", C.c_int), ("capacity", C.c_uint32),
                ("seed", C.c_uint64), ("frame_index", C.c_uint32), ("adrrs_eps_scale", C.c_float),
                ("collect_training", C.c_int), ("env", C.c_float * 3)]


class OrcStrategy(C.Structure):
    _fields_ = [("kind", C.c_int), ("fixed_value", C.c_float)]


class OrcRateControl(C.Structure):
    _fields_ = [("f_rate", C.c_float), ("alpha", C.c_float), ("eps", C.c_float), ("enabled", C.c_int),
                ("overflow_events", C.c_uint64)]


class OrcFrameReport(C.Structure):
    _fields_ = [("camera_rays", C.c_uint64), ("scatter_rays", C.c_uint64), ("shadow_rays", C.c_uint64),
                ("nonfinite_drops", C.c_uint64), ("overflow_events", C.c_uint64), ("bias_drop_events", C.c_uint64),
                ("train_samples", C.c_uint64), ("depth_counts", C.c_uint32 * 32)]


def _orc_scene(desc):
    pos, idx, mid = desc.arrays()
    keep = {"pos": pos, "idx": idx, "mid": mid,
            "kind": np.array([m.kind for m in desc.materials], np.int32),
            "alb": np.array([m.albedo for m in desc.materials], np.float32).reshape(-1),
            "rough": np.array([m.roughness for m in desc.materials], np.float32),
            "emi": np.array([m.emission for m in desc.materials], np.float32).reshape(-1)}
    f3 = lambda v: (C.c_float * 3)(*[float(np.float32(x)) for x in v])
    cam = desc.camera
    sc = OrcScene(pos.ctypes.data, idx.ctypes.data, mid.ctypes.data, pos.shape[0], mid.size, keep["kind"].ctypes.data,
                  keep["alb"].ctypes.data, keep["rough"].ctypes.data, keep["emi"].ctypes.data, f3(cam.position),
                  f3(cam.look_at), f3(cam.up), float(np.float32(cam.vfov_deg)))
    return sc, keep


def trace_frame(desc, width: int, height: int, assignment, max_depth: int, seed: int = 0, frame_index: int = 0,
                i_acc: np.ndarray | None = None, rc=None, nets: "OracleNets | None" = None, capacity: int = 0,
                collect_training: bool = False, adrrs_eps_scale: float = 1e-4, train_cap: int = 0):
    """orc_trace_frame: the reference's trace_frame run sequentially (brute-force hits).  assignment:
    list of (kind, fixed_value); rc: dict(f_rate, alpha, eps, enabled) updated in place.  Returns
    dict(frame [n,3] f64, normals, train (structured array), report)."""
    sc, keep = _orc_scene(desc)
    npx = width * height
    i_acc = np.zeros((npx, 3), np.float32) if i_acc is None else np.ascontiguousarray(i_acc, np.float32)
    rc = rc if rc is not None else {"f_rate": 0.85, "alpha": 1.0, "eps": 0.01, "enabled": 1, "overflow_events": 0}
    rcc = OrcRateControl(rc["f_rate"], rc["alpha"], rc["eps"], int(rc["enabled"]), rc.get("overflow_events", 0))
    cfg = OrcTraceCfg(width, height, max_depth, capacity, seed & (2**64 - 1), frame_index,
                      float(np.float32(adrrs_eps_scale)), int(collect_training),
                      (C.c_float * 3)(*[float(np.float32(x)) for x in desc.env_emission]))
    strat = (OrcStrategy * max_depth)(*[OrcStrategy(int(k), float(v)) for k, v in assignment])
    frame = np.zeros((npx, 3), np.float64)
    normals = np.zeros((npx, 3), np.float32)
    from paper_2510_07868_b200.film import TRAIN_SAMPLE_DTYPE
    cap = train_cap if train_cap else (npx * 8 if collect_training else 0)
    train = np.zeros(max(cap, 1), TRAIN_SAMPLE_DTYPE)
    n_train = C.c_size_t(0)
    rep = OrcFrameReport()
    r = lib().orc_trace_frame(C.byref(sc), C.byref(cfg), strat, C.byref(nets.c) if nets is not None else None,
                              C.byref(rcc), ptr(i_acc), ptr(frame), ptr(normals), ptr(train), cap,
                              C.byref(n_train), C.byref(rep))
    if r != 0:
        raise RuntimeError("orc_trace_frame failed")
    rc["alpha"] = float(np.float32(rcc.alpha))
    rc["overflow_events"] = int(rcc.overflow_events)
    report = {k: int(getattr(rep, k)) for k in ("camera_rays", "scatter_rays", "shadow_rays", "nonfinite_drops",
                                                 "overflow_events", "bias_drop_events", "train_samples")}
    report["depth_counts"] = list(rep.depth_counts[:max_depth])
    return {"frame": frame, "normals": normals, "train": train[:n_train.value], "report": report}
