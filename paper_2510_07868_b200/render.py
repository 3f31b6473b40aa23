"""Render front-end on the GPU (first part): scenes, camera rays,
closest-hit BVH traversal, dispatch and the surface vertex fields the RRS stage reads.

Mirrors the reference's `TriMesh` / `Material` / `Camera` / `Scene` (geometry.hpp,
bsdf.hpp:10-20, scene.hpp:12-20, scene.cpp) and the depth-1 head of `trace_frame`
(wavefront.cpp:253-268 camera rays, :282-290 intersect, :125-138 dispatch, :330-345
surface fields).  The BVH is built on the host exactly as `Bvh::build`
(geometry.cpp:88-137), so traversal returns the reference's hits.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _capi
from .stage import GpuContext

DIFFUSE, CONDUCTOR = 0, 1
NO_HIT = 0xFFFFFFFF
CLASS_MISS, CLASS_LIGHT, CLASS_SURFACE = 0, 1, 2


@dataclass
class Material:
    """bsdf.hpp:10-20 (same defaults)."""
    kind: int = DIFFUSE
    albedo: Sequence[float] = (0.5, 0.5, 0.5)
    roughness: float = 0.5
    emission: Sequence[float] = (0.0, 0.0, 0.0)

    def scattering(self) -> bool:
        return self.kind == CONDUCTOR or max(np.float32(a) for a in self.albedo) > 0.0


@dataclass
class Camera:
    """scene.hpp:12-20 (same defaults)."""
    position: Sequence[float] = (0.0, 0.0, 0.0)
    look_at: Sequence[float] = (0.0, 0.0, -1.0)
    up: Sequence[float] = (0.0, 1.0, 0.0)
    vfov_deg: float = 40.0


@dataclass
class SceneDesc:
    """Host scene: TriMesh (positions, indices, material_ids) + materials + camera."""
    positions: List[np.ndarray] = field(default_factory=list)
    indices: List[int] = field(default_factory=list)
    material_ids: List[int] = field(default_factory=list)
    materials: List[Material] = field(default_factory=list)
    camera: Camera = field(default_factory=Camera)
    env_emission: Sequence[float] = (0.0, 0.0, 0.0)

    def add_quad(self, corner, e1, e2, material_id: int) -> None:
        """add_quad (scene.cpp:98-109): float32 corner + e1 + e2, two triangles."""
        c, a, b = (np.asarray(x, dtype=np.float32) for x in (corner, e1, e2))
        base = len(self.positions)
        self.positions += [c, c + a, (c + a) + b, c + b]
        self.indices += [base, base + 1, base + 2, base, base + 2, base + 3]
        self.material_ids += [material_id, material_id]

    def add_box(self, lo, hi, mat: int) -> None:
        """make_cornell_scene's add_box lambda (scene.cpp:201-209)."""
        lo, hi = np.asarray(lo, np.float32), np.asarray(hi, np.float32)
        z = np.float32(0)
        dx = np.array([hi[0] - lo[0], z, z], np.float32)
        dy = np.array([z, hi[1] - lo[1], z], np.float32)
        dz = np.array([z, z, hi[2] - lo[2]], np.float32)
        self.add_quad(lo, dz, dx, mat)
        self.add_quad([lo[0], hi[1], lo[2]], dx, dz, mat)
        self.add_quad(lo, dx, dy, mat)
        self.add_quad([lo[0], lo[1], hi[2]], dy, dx, mat)
        self.add_quad(lo, dy, dz, mat)
        self.add_quad([hi[0], lo[1], lo[2]], dz, dy, mat)

    def arrays(self):
        pos = np.ascontiguousarray(np.array(self.positions, dtype=np.float32).reshape(-1, 3))
        idx = np.ascontiguousarray(np.array(self.indices, dtype=np.uint32))
        mid = np.ascontiguousarray(np.array(self.material_ids, dtype=np.uint32))
        return pos, idx, mid


def make_cornell_scene() -> SceneDesc:
    """make_cornell_scene (scene.cpp:174-219)."""
    s = SceneDesc()
    white = Material(albedo=(0.73, 0.73, 0.73))
    red = Material(albedo=(0.63, 0.065, 0.05))
    green = Material(albedo=(0.14, 0.45, 0.091))
    metal = Material(kind=CONDUCTOR, albedo=(0.9, 0.75, 0.4), roughness=0.15)
    lamp = Material(albedo=(0.0, 0.0, 0.0), emission=(17.0, 12.0, 4.0))
    s.materials = [white, red, green, metal, lamp]
    s.add_quad((-1, 0, -1), (2, 0, 0), (0, 0, 2), 0)
    s.add_quad((-1, 2, -1), (0, 0, 2), (2, 0, 0), 0)
    s.add_quad((-1, 0, -1), (0, 2, 0), (2, 0, 0), 0)
    s.add_quad((-1, 0, -1), (0, 0, 2), (0, 2, 0), 1)
    s.add_quad((1, 0, -1), (0, 2, 0), (0, 0, 2), 2)
    s.add_quad((-0.25, 1.98, -0.35), (0.5, 0, 0), (0, 0, 0.5), 4)
    s.add_box((-0.65, 0.001, -0.6), (-0.1, 1.1, -0.1), 3)
    s.add_box((0.15, 0.001, 0.0), (0.7, 0.55, 0.55), 0)
    s.camera = Camera(position=(0, 1, 3.2), look_at=(0, 1, 0), up=(0, 1, 0), vfov_deg=38.0)
    return s


def make_caustic_scene() -> SceneDesc:
    """make_caustic_scene (scene.cpp:245-277)."""
    s = SceneDesc()
    s.materials = [Material(kind=CONDUCTOR, albedo=(0.95, 0.93, 0.88), roughness=0.06),
                   Material(albedo=(0.65, 0.65, 0.7)), Material(albedo=(0.55, 0.35, 0.25)),
                   Material(albedo=(0.0, 0.0, 0.0), emission=(60.0, 55.0, 45.0))]
    s.add_quad((-2, 0, -2), (4, 0, 0), (0, 0, 4), 0)
    s.add_quad((-2, 0, -2), (0, 2.5, 0), (4, 0, 0), 1)
    s.add_quad((-2, 0, -2), (0, 0, 4), (0, 2.5, 0), 2)
    s.add_quad((2, 0, -2), (0, 2.5, 0), (0, 0, 4), 2)
    s.add_quad((-2, 2.5, -2), (0, 0, 4), (4, 0, 0), 1)
    s.add_quad((-0.5, 2.2, 1.0), (1.0, 0, 0), (0, -0.45, -0.3), 3)
    s.add_quad((-0.6, 2.3, 1.05), (1.2, 0, 0), (0, -0.6, 0.0), 2)
    s.camera = Camera(position=(0, 1.3, 1.85), look_at=(0, 0.9, -2), vfov_deg=55.0)
    return s


def make_furnace_scene(albedo: float = 0.7, emission: float = 0.5) -> SceneDesc:
    """make_furnace_scene (scene.cpp:221-243)."""
    s = SceneDesc()
    s.materials = [Material(albedo=(albedo,) * 3, emission=(emission,) * 3)]
    s.add_quad((-1, -1, -1), (2, 0, 0), (0, 0, 2), 0)
    s.add_quad((-1, 1, -1), (0, 0, 2), (2, 0, 0), 0)
    s.add_quad((-1, -1, -1), (0, 2, 0), (2, 0, 0), 0)
    s.add_quad((-1, -1, 1), (2, 0, 0), (0, 2, 0), 0)
    s.add_quad((-1, -1, -1), (0, 0, 2), (0, 2, 0), 0)
    s.add_quad((1, -1, -1), (0, 2, 0), (0, 0, 2), 0)
    s.camera = Camera(position=(0, 0, 0), look_at=(0.3, 0.2, -1), vfov_deg=60.0)
    return s


def _f3(v) -> C.Array:
    return (C.c_float * 3)(*[float(np.float32(x)) for x in v])


class GpuScene:
    """A scene resident on one GPU (nrrs_gpu_scene_create)."""

    def __init__(self, desc: SceneDesc, ctx: Optional[GpuContext] = None, device: int = 0):
        self.ctx = ctx or GpuContext(device)
        self.device = torch.device("cuda", self.ctx.device)
        self.desc = desc
        pos, idx, mid = desc.arrays()
        self.n_tri = int(mid.size)
        mats = (_capi.MaterialC * max(1, len(desc.materials)))()
        for i, m in enumerate(desc.materials):
            mats[i].kind = int(m.kind)
            mats[i].albedo = _f3(m.albedo)
            mats[i].roughness = float(np.float32(m.roughness))
            mats[i].emission = _f3(m.emission)
        cam = _capi.CameraC(_f3(desc.camera.position), _f3(desc.camera.look_at), _f3(desc.camera.up),
                            float(np.float32(desc.camera.vfov_deg)))
        h = C.c_void_p()
        _capi.check(self.ctx.handle, self.ctx.lib.nrrs_gpu_scene_create(
            self.ctx.handle, pos.ctypes.data, pos.shape[0], idx.ctypes.data, self.n_tri, mid.ctypes.data, mats,
            len(desc.materials), C.byref(cam), C.byref(h)))
        self.handle = h
        env = (C.c_float * 3)(*[float(np.float32(x)) for x in desc.env_emission])
        _capi.check(self.ctx.handle, self.ctx.lib.nrrs_gpu_scene_set_env(self.handle, env))

    @property
    def light_count(self) -> int:
        return int(self.ctx.lib.nrrs_gpu_scene_light_count(self.handle))

    @property
    def node_count(self) -> int:
        return int(self.ctx.lib.nrrs_gpu_scene_node_count(self.handle))

    def camera_rays(self, width: int, height: int, seed: int, frame: int) -> Dict[str, torch.Tensor]:
        """Depth-1 rays of every pixel (wavefront.cpp:253-268): o, d [n, 3] f32 and path_key [n] u64."""
        self.ctx.bind_stream()
        n = width * height
        o = torch.empty(n, 3, dtype=torch.float32, device=self.device)
        d = torch.empty_like(o)
        keys = torch.empty(n, dtype=torch.int64, device=self.device)
        _capi.check(self.ctx.handle, self.ctx.lib.nrrs_gpu_camera_rays(
            self.ctx.handle, self.handle, width, height, seed & (2**64 - 1), frame, o.data_ptr(), d.data_ptr(),
            keys.data_ptr()))
        return {"o": o, "d": d, "path_key": keys}

    def intersect(self, o: torch.Tensor, d: torch.Tensor, t_max: Optional[torch.Tensor] = None,
                  uv: bool = True, check: bool = False) -> Dict[str, torch.Tensor]:
        """Closest hits (Bvh::intersect): t (inf on miss), tri (NO_HIT as int32 -1), u, v.
        check=True synchronizes and raises on a degenerate ray direction, as the reference does."""
        self.ctx.bind_stream()
        n = int(o.shape[0])
        t = torch.empty(n, dtype=torch.float32, device=self.device)
        tri = torch.empty(n, dtype=torch.int32, device=self.device)
        u = torch.empty(n, dtype=torch.float32, device=self.device) if uv else None
        v = torch.empty(n, dtype=torch.float32, device=self.device) if uv else None
        _capi.check(self.ctx.handle, self.ctx.lib.nrrs_gpu_intersect(
            self.ctx.handle, self.handle, o.data_ptr(), d.data_ptr(), t_max.data_ptr() if t_max is not None else None,
            n, t.data_ptr(), tri.data_ptr(), u.data_ptr() if uv else None, v.data_ptr() if uv else None))
        if check:
            self.check()
        return {"t": t, "tri": tri, "u": u, "v": v}

    def check(self) -> None:
        """Raises NrrsError for a degenerate ray direction seen since the last check."""
        _capi.check(self.ctx.handle, self.ctx.lib.nrrs_gpu_render_check(self.ctx.handle))

    def surface_records(self, o: torch.Tensor, d: torch.Tensor, t: torch.Tensor,
                        tri: torch.Tensor) -> Dict[str, torch.Tensor]:
        """dispatch class (0 miss, 1 light, 2 surface) and p01 / wo01 / roughness / material."""
        self.ctx.bind_stream()
        n = int(o.shape[0])
        cls = torch.empty(n, dtype=torch.uint8, device=self.device)
        p01 = torch.empty(n, 3, dtype=torch.float32, device=self.device)
        wo01 = torch.empty(n, 2, dtype=torch.float32, device=self.device)
        rough = torch.empty(n, dtype=torch.float32, device=self.device)
        mat = torch.empty(n, dtype=torch.int32, device=self.device)
        _capi.check(self.ctx.handle, self.ctx.lib.nrrs_gpu_surface_records(
            self.ctx.handle, self.handle, o.data_ptr(), d.data_ptr(), t.data_ptr(), tri.data_ptr(), n,
            cls.data_ptr(), p01.data_ptr(), wo01.data_ptr(), rough.data_ptr(), mat.data_ptr()))
        return {"class": cls, "p01": p01, "wo01": wo01, "roughness": rough, "material": mat}

    def render_depth1(self, width: int, height: int, seed: int, frame: int) -> Dict[str, torch.Tensor]:
        rays = self.camera_rays(width, height, seed, frame)
        hits = self.intersect(rays["o"], rays["d"])
        rec = self.surface_records(rays["o"], rays["d"], hits["t"], hits["tri"])
        return {**rays, **hits, **rec}

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.ctx.lib.nrrs_gpu_scene_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class TraceConfig:
    """TraceConfig (wavefront.hpp:128-140): the fields trace_frame reads."""
    max_depth: int = 8
    queue_capacity: int = 0
    seed: int = 0
    frame_index: int = 0
    adrrs_eps_scale: float = 1e-4
    collect_training: bool = False


@dataclass
class FrameReport:
    """FrameReport (wavefront.hpp:175-186)."""
    camera_rays: int = 0
    scatter_rays: int = 0
    shadow_rays: int = 0
    nonfinite_drops: int = 0
    overflow_events: int = 0
    bias_drop_events: int = 0
    train_samples: int = 0
    depth_counts: List[int] = field(default_factory=list)


class Tracer:
    """trace_frame on one GPU (wavefront.cpp:217-551) through nrrs_gpu_trace_frame: device
    queues and per-depth vertex records sized for films up to max_pixels."""

    def __init__(self, scene: GpuScene, max_pixels: int, max_depth: int, capacity: int = 0):
        self.scene = scene
        self.ctx = scene.ctx
        self.max_depth = int(max_depth)
        h = C.c_void_p()
        _capi.check(self.ctx.handle, self.ctx.lib.nrrs_gpu_tracer_create(self.ctx.handle, int(max_pixels),
                                                                         self.max_depth, int(capacity), C.byref(h)))
        self.handle = h

    def trace_frame(self, assignment, cfg: TraceConfig, rc, film, train: Optional[torch.Tensor] = None,
                    train_count: int = 0):
        """Renders one frame into `film` (a film.GpuFilm); returns (FrameReport, train_count).
        `assignment` holds one rrs.Strategy per depth; `rc` is an rrs.RateControl (updated)."""
        from . import rrs as _rrs
        if len(assignment) != cfg.max_depth:
            raise RuntimeError("trace_frame: assignment must have one entry per depth")
        self.ctx.bind_stream()
        strat = (_capi.StrategyC * len(assignment))(*[s.c() for s in assignment])
        c = _capi.TraceConfigC(film.width, film.height, cfg.max_depth, cfg.queue_capacity, cfg.seed & (2**64 - 1),
                               cfg.frame_index, float(np.float32(cfg.adrrs_eps_scale)), int(cfg.collect_training))
        rcc = _capi.RateControlC(rc.f_rate, rc.alpha, rc.eps, int(rc.enabled), rc.overflow_events)
        fd = _capi.FilmDevC(film.sum.data_ptr(), film.samples.data_ptr(), film.i_cur.data_ptr(),
                            film.i_acc.data_ptr(), film.normal.data_ptr())
        rep = _capi.FrameReportC()
        cnt = C.c_uint64(train_count)
        cap = 0 if train is None else int(train.numel() * train.element_size() // 80)
        _capi.check(self.ctx.handle, self.ctx.lib.nrrs_gpu_trace_frame(
            self.handle, self.scene.handle, C.byref(c), strat, C.byref(rcc), C.byref(fd),
            train.data_ptr() if train is not None else None, cap, C.byref(cnt), C.byref(rep)))
        rc.alpha = float(np.float32(rcc.alpha))
        rc.overflow_events = int(rcc.overflow_events)
        r = FrameReport(rep.camera_rays, rep.scatter_rays, rep.shadow_rays, rep.nonfinite_drops, rep.overflow_events,
                        rep.bias_drop_events, rep.train_samples, list(rep.depth_counts[:cfg.max_depth]))
        return r, int(cnt.value)

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.ctx.lib.nrrs_gpu_tracer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


__all__ = ["TraceConfig", "FrameReport", "Tracer", "Material", "Camera", "SceneDesc", "GpuScene", "make_cornell_scene", "make_caustic_scene",
           "make_furnace_scene", "DIFFUSE", "CONDUCTOR", "NO_HIT", "CLASS_MISS", "CLASS_LIGHT", "CLASS_SURFACE"]
