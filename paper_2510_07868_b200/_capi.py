"""ctypes binding of the C ABI in include/nrrs_gpu.h (libnrrs_gpu.so, in-tree).

The product path has no CPU fallback: if the shared library is missing or no
sm_100 device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import pathlib

_PKG = pathlib.Path(__file__).resolve().parent
LIB_PATH = _PKG / "libnrrs_gpu.so"

NRRS_OK, NRRS_EINVAL, NRRS_ESIZE, NRRS_ECUDA, NRRS_ENCCL, NRRS_ESTATE = range(6)

_STATUS_NAMES = {1: "EINVAL", 2: "ESIZE", 3: "ECUDA", 4: "ENCCL", 5: "ESTATE"}


class GridSpec(C.Structure):
    _fields_ = [("levels", C.c_int32), ("features", C.c_int32), ("base_resolution", C.c_int32),
                ("log2_table_size", C.c_int32)]


class NetWeights(C.Structure):
    _fields_ = [("variant", C.c_int32), ("grid", GridSpec),
                ("stat_grid", C.POINTER(C.c_float)), ("stat_grid_len", C.c_uint64),
                ("stat_mlp", C.POINTER(C.c_float)), ("stat_mlp_len", C.c_uint64),
                ("rrs_grid", C.POINTER(C.c_float)), ("rrs_grid_len", C.c_uint64),
                ("rrs_mlp", C.POINTER(C.c_float)), ("rrs_mlp_len", C.c_uint64)]


class StrategyC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("fixed_value", C.c_float)]


class VertexSoA(C.Structure):
    _fields_ = [("p01", C.c_void_p), ("wo01", C.c_void_p), ("roughness", C.c_void_p), ("weight", C.c_void_p),
                ("i_pixel", C.c_void_p), ("path_key", C.c_void_p), ("pixel", C.c_void_p), ("i_acc", C.c_void_p)]


class StageParams(C.Structure):
    _fields_ = [("depth", C.c_uint32), ("n_pixels", C.c_uint32), ("capacity", C.c_uint32),
                ("strategy", StrategyC), ("gain", C.c_float), ("eps_div", C.c_float), ("seed", C.c_uint64)]


class StageOut(C.Structure):
    _fields_ = [("q_norm", C.c_void_p), ("q_real", C.c_void_p), ("slots", C.c_void_p), ("k", C.c_void_p),
                ("offset", C.c_void_p), ("decided", C.c_void_p), ("q_orig", C.c_void_p), ("u", C.c_void_p)]


class StageResultC(C.Structure):
    _fields_ = [("f_norm", C.c_double), ("sum_q", C.c_double), ("total", C.c_uint64), ("dropped", C.c_uint64),
                ("nonfinite", C.c_uint64), ("box_cox_clamps", C.c_uint64), ("spawned", C.c_uint32),
                ("overflow", C.c_uint32)]


class VertexRecSoA(C.Structure):
    _fields_ = [("p01", C.c_void_p), ("wo01", C.c_void_p), ("roughness", C.c_void_p), ("weight", C.c_void_p),
                ("pixel", C.c_void_p), ("q_norm", C.c_void_p), ("q_real", C.c_void_p), ("decided", C.c_void_p),
                ("s", C.c_void_p)]


class MaterialC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("albedo", C.c_float * 3), ("roughness", C.c_float),
                ("emission", C.c_float * 3)]


class CameraC(C.Structure):
    _fields_ = [("position", C.c_float * 3), ("look_at", C.c_float * 3), ("up", C.c_float * 3),
                ("vfov_deg", C.c_float)]


class TraceConfigC(C.Structure):
    _fields_ = [("width", C.c_uint32), ("height", C.c_uint32), ("max_depth", C.c_int32),
                ("queue_capacity", C.c_uint32), ("seed", C.c_uint64), ("frame_index", C.c_uint32),
                ("adrrs_eps_scale", C.c_float), ("collect_training", C.c_int32)]


class RateControlC(C.Structure):
    _fields_ = [("f_rate", C.c_float), ("alpha", C.c_float), ("eps", C.c_float), ("enabled", C.c_int32),
                ("overflow_events", C.c_uint64)]


class FrameReportC(C.Structure):
    _fields_ = [("camera_rays", C.c_uint64), ("scatter_rays", C.c_uint64), ("shadow_rays", C.c_uint64),
                ("nonfinite_drops", C.c_uint64), ("overflow_events", C.c_uint64), ("bias_drop_events", C.c_uint64),
                ("train_samples", C.c_uint64), ("depth_counts", C.c_uint32 * 32)]


class FilmDevC(C.Structure):
    _fields_ = [("sum", C.c_void_p), ("samples", C.c_void_p), ("i_cur", C.c_void_p), ("i_acc", C.c_void_p),
                ("normal", C.c_void_p)]


# (name, restype, argtypes) for every entry point declared in include/nrrs_gpu.h
_P = C.c_void_p
SIGNATURES = [
    ("nrrs_gpu_abi_version", C.c_int, []),
    ("nrrs_gpu_create", C.c_int, [C.c_int, C.POINTER(_P)]),
    ("nrrs_gpu_destroy", C.c_int, [_P]),
    ("nrrs_gpu_last_error", C.c_char_p, [_P]),
    ("nrrs_gpu_set_stream", C.c_int, [_P, _P]),
    ("nrrs_gpu_reserve", C.c_int, [_P, C.c_uint64, C.c_uint32]),
    ("nrrs_gpu_launch_count", C.c_uint64, [_P]),
    ("nrrs_gpu_fetch_result", C.c_int, [_P, C.POINTER(StageResultC)]),
    ("nrrs_gpu_stage_total_dev", C.c_int, [_P, C.POINTER(C.c_void_p)]),
    ("nrrs_gpu_weights_info", C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
    ("nrrs_gpu_film_luminance_sum", C.c_int, [_P, _P, C.c_uint64, _P]),
    ("nrrs_gpu_fold_ordered", C.c_int, [_P, _P, C.c_uint64, _P, _P, C.c_uint64]),
    ("nrrs_gpu_emit_train", C.c_int, [_P, C.c_uint32, C.POINTER(VertexRecSoA), C.c_uint64, _P, _P, C.c_uint64,
                                      _P, _P, _P]),
    ("nrrs_gpu_train_k_i", C.c_int, [_P, _P, C.c_uint64, _P, C.c_uint64, C.c_uint32]),
    ("nrrs_gpu_film_add_frame", C.c_int, [_P, _P, _P, _P, _P, C.c_uint32]),
    ("nrrs_gpu_film_roll_acc", C.c_int, [_P, _P, _P, C.c_uint32]),
    ("nrrs_gpu_stat_loss_grad", C.c_int, [_P, C.POINTER(GridSpec), _P, _P, _P, C.c_uint64, C.c_float, C.c_float, _P,
                                          _P, C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
    ("nrrs_gpu_rrs_loss_grad", C.c_int, [_P, C.c_int32, C.POINTER(GridSpec), _P, _P, _P, _P, _P, C.c_uint64, _P,
                                         C.c_uint64, C.c_float, C.c_int32, C.c_float, C.c_float, C.c_float,
                                         C.c_float, C.c_float, _P, _P, C.POINTER(C.c_double),
                                         C.POINTER(C.c_uint32), C.POINTER(C.c_int32)]),
    ("nrrs_gpu_adam_ema", C.c_int, [_P, _P, _P, _P, _P, _P, C.c_uint64, C.c_int64, C.c_float, C.c_float, C.c_float,
                                    C.c_float, C.c_float, C.c_float]),
    ("nrrs_gpu_scene_create", C.c_int, [_P, _P, C.c_uint32, _P, C.c_uint32, _P, C.POINTER(MaterialC), C.c_uint32,
                                        C.POINTER(CameraC), C.POINTER(_P)]),
    ("nrrs_gpu_scene_destroy", C.c_int, [_P]),
    ("nrrs_gpu_scene_node_count", C.c_uint32, [_P]),
    ("nrrs_gpu_camera_rays", C.c_int, [_P, _P, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, _P, _P, _P]),
    ("nrrs_gpu_intersect", C.c_int, [_P, _P, _P, _P, _P, C.c_uint64, _P, _P, _P, _P]),
    ("nrrs_gpu_render_check", C.c_int, [_P]),
    ("nrrs_gpu_scene_light_count", C.c_uint32, [_P]),
    ("nrrs_gpu_scene_set_env", C.c_int, [_P, C.POINTER(C.c_float)]),
    ("nrrs_gpu_tracer_create", C.c_int, [_P, C.c_uint32, C.c_int32, C.c_uint32, C.POINTER(_P)]),
    ("nrrs_gpu_tracer_destroy", C.c_int, [_P]),
    ("nrrs_gpu_trace_frame", C.c_int, [_P, _P, C.POINTER(TraceConfigC), C.POINTER(StrategyC),
                                       C.POINTER(RateControlC), C.POINTER(FilmDevC), _P, C.c_uint64,
                                       C.POINTER(C.c_uint64), C.POINTER(FrameReportC)]),
    ("nrrs_gpu_tracer_frame_buffer", C.c_int, [_P, C.POINTER(_P)]),
    ("nrrs_gpu_tracer_vertices", C.c_int, [_P, C.c_int32, C.POINTER(VertexRecSoA), C.POINTER(C.c_uint32)]),
    ("nrrs_gpu_surface_records", C.c_int, [_P, _P, _P, _P, _P, _P, C.c_uint64, _P, _P, _P, _P, _P]),
    ("nrrs_gpu_set_weights", C.c_int, [_P, C.POINTER(NetWeights)]),
    ("nrrs_gpu_set_weights_dev", C.c_int, [_P, C.POINTER(NetWeights)]),
    ("nrrs_gpu_rrs_stage", C.c_int, [_P, C.POINTER(VertexSoA), C.c_uint64, C.POINTER(StageParams),
                                     C.POINTER(StageOut), C.POINTER(StageResultC)]),
    ("nrrs_gpu_rrs_stage_host", C.c_int, [_P, C.POINTER(VertexSoA), C.c_uint64, C.POINTER(StageParams),
                                          C.POINTER(StageOut), C.POINTER(StageResultC)]),
    ("nrrs_gpu_rrs_stage_host_async", C.c_int, [_P, C.POINTER(VertexSoA), C.c_uint64, C.POINTER(StageParams),
                                                C.POINTER(StageOut), C.POINTER(C.c_uint64)]),
    ("nrrs_gpu_stage_host_wait", C.c_int, [_P, C.c_uint64, C.POINTER(StageResultC)]),
    ("nrrs_gpu_stage_factors", C.c_int, [_P, C.POINTER(VertexSoA), C.c_uint64, C.POINTER(StageParams),
                                         C.POINTER(StageOut), _P]),
    ("nrrs_gpu_stage_decide", C.c_int, [_P, C.c_uint64, C.POINTER(StageParams), _P, C.c_int32,
                                        C.POINTER(StageOut), _P]),
    ("nrrs_gpu_sharded_clip_dev", C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_uint32, _P]),
    ("nrrs_gpu_stage_local_sum_exact", C.c_int, [_P, _P]),
    ("nrrs_gpu_stage_sum_exact_dev", C.c_int, [_P, C.POINTER(C.c_void_p)]),
    ("nrrs_gpu_stage_decide_exact", C.c_int, [_P, C.c_uint64, C.POINTER(StageParams), _P, C.c_int32,
                                              C.POINTER(StageOut), _P]),
    ("nrrs_gpu_mailbox_init", C.c_int, [_P, C.c_int32, C.c_int32, _P, C.POINTER(C.c_uint64)]),
    ("nrrs_gpu_mailbox_connect", C.c_int, [_P, _P, _P]),
    ("nrrs_gpu_stage_decide_mbox", C.c_int, [_P, C.c_uint64, C.POINTER(StageParams), C.POINTER(StageOut), _P]),
    ("nrrs_gpu_sharded_clip_mbox", C.c_int, [_P, C.c_uint32, _P, _P, _P]),
    ("nrrs_gpu_mailbox_status", C.c_int, [_P, C.POINTER(C.c_int32)]),
    ("nrrs_gpu_sharded_clip", C.c_int, [C.POINTER(C.c_uint64), C.c_int32, C.c_int32, C.c_uint32,
                                        C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                        C.POINTER(C.c_uint64)]),
    ("nrrs_gpu_compact", C.c_int, [_P, _P, _P, C.c_uint32, C.c_uint32, _P, _P, C.POINTER(C.c_uint32)]),
    ("nrrs_gpu_compact_dev", C.c_int, [_P, _P, _P, _P, C.c_uint32, C.c_uint32, _P, _P]),
    ("nrrs_gpu_normalize_factors", C.c_int, [_P, _P, C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]),
    ("nrrs_gpu_realize_counts", C.c_int, [_P, _P, _P, _P, C.c_uint64, C.POINTER(C.c_uint64)]),
    ("nrrs_gpu_plan_spawns", C.c_int, [_P, _P, C.c_uint64, C.c_uint32, _P, C.POINTER(C.c_uint32),
                                       C.POINTER(C.c_uint64)]),
    ("nrrs_gpu_strategy_factor", C.c_int, [_P, C.POINTER(VertexSoA), C.c_uint64, C.POINTER(StrategyC),
                                           C.c_float, _P]),
    ("nrrs_gpu_predict_stats", C.c_int, [_P, C.POINTER(VertexSoA), C.c_uint64, _P]),
    ("nrrs_gpu_encode_levels", C.c_int, [_P, _P, C.c_uint64, _P, C.c_uint64]),
    ("nrrs_queue_capacity_for", C.c_uint32, [C.c_uint32]),
    ("nrrs_rng_fill", None, [C.c_uint64, C.c_uint64, C.POINTER(C.c_float), C.c_uint64, C.c_float, C.c_float]),
    ("nrrs_root_path_key", C.c_uint64, [C.c_uint32, C.c_uint32]),
    ("nrrs_child_path_key", C.c_uint64, [C.c_uint64, C.c_uint32]),
]

_lib = None


def lib() -> C.CDLL:
    """Loads libnrrs_gpu.so (building it first if the sources are newer)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            from . import _build
            _build.build()
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run python -c 'import __graft_entry__ as g; g.build()'")
        handle = C.CDLL(str(LIB_PATH))
        for name, res, args in SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


class NrrsError(RuntimeError):
    """Raised for non-zero nrrs_status codes (std::runtime_error in the reference)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"{_STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def check(ctx, code: int) -> None:
    if code != NRRS_OK:
        msg = lib().nrrs_gpu_last_error(ctx).decode() if ctx else ""
        raise NrrsError(code, msg)
