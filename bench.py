#!/usr/bin/env python
"""Benchmark of the NRRS per-bounce RRS stage (BASELINE.json metric: path vertices/s
through RRSNet + normalized RRS + compaction).

Workload (N=1): BASELINE.json configs[2] shape -- AID-NRRS, one 1920x1080 film,
one decision depth (depth 2) over 2,073,600 synthetic surface vertices
(SURVEY.md 8d generator), random-init RRSNet (NeuralRrsConfig{AID, seed 1} +
benchmark head randomization), gain f_rate*alpha = 0.85, capacity
queue_capacity_for(Npx).  A step = K-A factors (hash grid + tcgen05 MLP) ->
K-B normalize/realize/scan/slot emission -> K-C order-preserving compaction of
the slot records by a synthetic BSDF-validity mask (~10% invalid).
N>1 (torchrun): each rank owns a 2,073,600-vertex band of an N-band film,
global normalization and capacity clip over NCCL (weak scaling; N=8 is the
16.6M-vertex configs[4] batch).

--impl reference: the reference's CPU implementation of the same path (the C
oracle port: parallel factor pass + serial normalize/realize/plan/slots), all
host threads, bounded samples.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "path vertices/sec (RRSNet+normalized RRS+compaction) at 1/2/4/8 B200"
N_LOCAL = 1920 * 1080
ALG_BYTES_INFER = 56 + 8   # K-A: reads p01 12, wo01 8, rough 4, t_x 12, i_pixel 12, key 8; writes q_orig 4 + u 4
# K-A's binding resource is L2 scattered-gather throughput, counted in random 8-byte
# gather requests per vertex.  AID (fp16 tables): 7 hashed levels x (4 edge pairs + 4/256 unpaired corners,
# 8 edge-paired table copies) + dense level 0 (4 pairs) = 32.1 8-byte requests.  NRRS (fp32 tables): the same
# requests, the pairs 16 bytes wide at 1.28 units each (measured).  Ceiling: 296 G random 8-byte gathers/s from
# a 2 MiB table (profiles/r01_microbench_gather_bw.txt, tools/gather_bw.cu).
GATHER_UNITS_PER_VERTEX = {"aid": 7 * (4 + 4 / 256) + 4, "nrrs": 7 * (4 * 1.28 + 4 / 256) + 4 * 1.28}
GATHER_CEILING_PER_S = 296e9
# AID with fp16 tables runs K-A0 first: one hash-grid level per CTA from shared memory, 8 random 4-byte
# corner loads per vertex and level = 64 per vertex.  Ceiling: 8.54 random 4-byte loads/cycle/SM from a
# 128 KB shared-memory table at 32 warps/SM = 2,484 G loads/s (profiles/r01_microbench_gather_bw.txt).
SMEM_LOADS_PER_VERTEX = 64
SMEM_LOAD_CEILING_PER_S = 2484.46e9
STAGE_READ, STAGE_WRITE = 56, 8  # SURVEY.md 8d per-vertex compulsory bytes (+ 8 B per spawned slot record)


class _DevPtr:
    """A raw device address with the data_ptr() accessor the ABI wrappers use."""

    def __init__(self, addr: int):
        self.addr = addr

    def data_ptr(self) -> int:
        return self.addr


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="aid", choices=["aid", "nrrs"])
    ap.add_argument("--vertices", type=int, default=N_LOCAL, help="vertices per rank")
    ap.add_argument("--no-extra", action="store_true", help="skip the per-strategy side measurements")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling (configs[3]): --vertices is the whole film, split into N row bands "
                         "(default: weak scaling, --vertices per rank; N=8 is the configs[4] 16.6 M batch)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# ---------------------------------------------------------------------------
def cpu_baseline(variant: str, n_sample: int = N_LOCAL):
    """Oracle port of the reference path on this host's cores (rank 0, N=1 only)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle as orc  # CPU checker / baseline only
    threads = orc.threads_available()
    v = orc.gen_vertices(n_sample)
    var = orc.VARIANT_AID if variant == "aid" else orc.VARIANT_NRRS
    kind = orc.AID_NRRS if variant == "aid" else orc.NRRS
    nets = orc.OracleNets(var, seed=1, randomize=True)
    cap = orc.lib().orc_queue_capacity_for(n_sample)
    best = float("inf")
    for _ in range(5):
        t0 = time.perf_counter()
        orc.rrs_stage(v, 2, n_sample, cap, kind, nets, gain=0.85, seed=0, threads=threads)
        best = min(best, time.perf_counter() - t0)
    return {"value": n_sample / best, "unit": "vertices/s", "cores": threads, "kind": "port",
            "host": host_cpu(),
            "sample": f"{n_sample} synthetic vertices (the full workload), {variant}-nrrs, depth 2, best of 5 "
                      f"(factor pass over {threads} threads + serial normalize/realize/plan/slots)"}


def host_cpu() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    world, rank, _ = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        if rank != 0:
            dist.barrier()
            dist.destroy_process_group()
            return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle as orc
    threads = orc.threads_available()
    var = orc.VARIANT_AID if args.variant == "aid" else orc.VARIANT_NRRS
    kind = orc.AID_NRRS if args.variant == "aid" else orc.NRRS
    nets = orc.OracleNets(var, seed=1, randomize=True)
    sample = args.vertices
    v = orc.gen_vertices(sample)
    cap = orc.lib().orc_queue_capacity_for(sample)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        orc.rrs_stage(v, 2, sample, cap, kind, nets, gain=0.85, seed=i, threads=threads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    value = sample / statistics.mean(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "vertices/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (f64 sum; CPU port)", "data": "synthetic",
            "config": {"workload": f"{args.variant}-nrrs stage, 1920x1080 synthetic vertices at depth 2 "
                                   f"(full batch each step)",
                       "n_pixels": args.vertices, "strategy": f"{args.variant}-nrrs", "depth": 2},
            "cpu_baseline": {"value": value, "unit": "vertices/s", "cores": threads, "kind": "port", "host": host_cpu(),
                             "sample": f"the full {sample}-vertex batch per step; C restatement of the reference "
                                       "path (the reference's network code builds here only against this repo's "
                                       "Eigen-subset shim -- a correctness pin, not a performance-representative "
                                       "build of the reference)"},
            "e2e": {"value": value, "unit": "vertices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2510_07868_b200 import (NeuralRrs, NeuralRrsConfig, RateControl, RrsStage, RrsVariant, Strategy,
                                       StrategyKind, queue_capacity_for)
    from paper_2510_07868_b200 import _capi, synthetic
    from paper_2510_07868_b200.sharded import ShardedRrsStage

    world, rank, local = dist_env()
    # test-only knobs: run N ranks on one device with gloo exchanges (functional check of the N>1 path)
    backend = os.environ.get("NRRS_BENCH_BACKEND", "nccl")
    # N > 1 exchange: "collective" (torch.distributed all-gathers, default) or "mailbox" (in-kernel
    # over NVLink peer memory, CUDA IPC; one GPU per rank -- never with NRRS_BENCH_SAME_DEVICE)
    exchange = os.environ.get("NRRS_BENCH_EXCHANGE", "collective")
    if exchange == "mailbox" and os.environ.get("NRRS_BENCH_SAME_DEVICE") and world > 1:
        raise SystemExit("NRRS_BENCH_EXCHANGE=mailbox needs one GPU per rank (its kernels wait on the other ranks)")
    if os.environ.get("NRRS_BENCH_SAME_DEVICE"):
        local = 0
    torch.cuda.set_device(local)
    # test-only: the sharded path with one rank (a 1-rank NCCL group), to see its host and collective
    # overhead on one GPU
    force_sharded = bool(os.environ.get("NRRS_BENCH_FORCE_SHARDED")) and world == 1
    if force_sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29561")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    if world > 1 or force_sharded:
        if backend == "nccl":
            dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend, init_method="env://")
    dev = torch.device("cuda", local)
    if args.strong:  # one film of args.vertices pixels, rank r takes the r-th contiguous band
        first = args.vertices * rank // world
        n = args.vertices * (rank + 1) // world - first
        npx = args.vertices
    else:
        first = rank * args.vertices
        n = args.vertices
        npx = n * world
    cap = queue_capacity_for(npx)
    variant = RrsVariant.Aid if args.variant == "aid" else RrsVariant.Nrrs
    strategy = Strategy(StrategyKind.AidNrrs if args.variant == "aid" else StrategyKind.Nrrs)
    nets = NeuralRrs(NeuralRrsConfig(variant=variant, seed=1)).randomize_for_benchmark()

    # inputs resident in HBM before timing
    hv = synthetic.gen_vertices(n, n_pixels=npx, first=first)
    dv = {k: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).to(dev)
          for k, a in hv.items() if k != "pixel"}
    if world > 1 or force_sharded:
        sh = ShardedRrsStage(npx, nets, device=local, exchange=exchange)
        stage = sh.stage
    else:
        sh = None
        stage = RrsStage(npx, nets, device=local)
    stage.reserve(n)
    _half, _perr = stage.table_precision()
    aid_tables = {"fp16": _half, "error_budget_probe_max_rel_err": _perr, "budget": 2.5e-4}
    _tp = ctypes.c_void_p()
    _capi.check(stage.handle, _capi.lib().nrrs_gpu_stage_total_dev(stage.handle, ctypes.byref(_tp)))
    total_dev = _DevPtr(_tp.value)  # the stage's device-side realized total (compaction bound)
    out = stage.alloc_outputs(n)  # q_norm, q_real, slots (q_orig / u stay context scratch)
    slot_cap = stage.capacity
    slot_idx = torch.arange(slot_cap, dtype=torch.int64, device=dev)
    # synthetic BSDF validity per slot (~10% invalid samples), fixed hash of the slot index
    used = (((slot_idx * 2654435761) >> 7) % 10 != 0).to(torch.uint8)
    compacted = torch.empty((slot_cap, 2), dtype=torch.int32, device=dev)
    d_count = torch.zeros(1, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    lib = _capi.lib()
    import ctypes as C
    rc = RateControl()
    local_sum = torch.zeros(1, dtype=torch.float64, device=dev)
    local_total = torch.zeros(1, dtype=torch.int64, device=dev)

    pending = [None]  # N > 1: the last depth's device-side scalars (sharded_depth_async)

    def step(ev):
        """One stage step.  ev = [start, end] (timed loop: nothing between the kernels, so K-B / K-C
        launch early under programmatic dependent launch) or [start, after K-A, after K-B, end]
        (breakdown loop)."""
        stream = torch.cuda.current_stream()
        ev[0].record(stream)
        gain = rc.gain()
        p = stage.params(2, strategy, gain, 0.0, n_pixels=npx)
        from paper_2510_07868_b200.stage import vertex_soa
        soa = vertex_soa(dv)
        oc = out.c()
        if not (sh is None and len(ev) == 2):
            _capi.check(stage.handle, lib.nrrs_gpu_stage_factors(stage.handle, C.byref(soa), n, C.byref(p),
                                                                 C.byref(oc), local_sum.data_ptr()))
        if len(ev) == 4:
            ev[1].record(stream)
        def compact(count_src):
            if len(ev) == 4:
                ev[2].record(stream)
            _capi.check(stage.handle, lib.nrrs_gpu_compact_dev(stage.handle, out.slots.data_ptr(), used.data_ptr(),
                                                               count_src.data_ptr(), slot_cap, 2, compacted.data_ptr(),
                                                               d_count.data_ptr()))
        if sh is None and len(ev) == 2:
            # the drop-in call (nrrs_gpu_rrs_stage, asynchronous), then the compaction of its slot records
            _capi.check(stage.handle, lib.nrrs_gpu_rrs_stage(stage.handle, C.byref(soa), n, C.byref(p), C.byref(oc),
                                                             None))
            compact(total_dev)
        elif sh is None:
            _capi.check(stage.handle, lib.nrrs_gpu_stage_decide(stage.handle, n, C.byref(p), local_sum.data_ptr(), 1,
                                                                C.byref(oc), local_total.data_ptr()))
            compact(local_total)
        else:
            sh.stage.ctx.bind_stream()
            from paper_2510_07868_b200.sharded import sharded_depth_async
            # no host wait inside the depth: the global clip runs on the device (NCCL path) and this rank's
            # compaction needs only its own queue; the scalars are read after the timed loop
            # this rank's compaction needs only its own total: queued right behind K-B (programmatic
            # dependent launch), ahead of the totals exchange and the clip
            if sh.exchange == "mailbox":
                pending[0] = sh.depth_async(n, 2, strategy, out, gain, 0.0, after_decide=lambda: compact(sh._total))
            else:
                pending[0] = sharded_depth_async(sh._sum_fx, lambda rs: sh.decide(n, 2, strategy, out, rs, gain, 0.0),
                                                 cap, npx, sh.stage, None, after_decide=lambda: compact(sh._total))
        ev[-1].record(stream)

    def events(k=2):
        return [torch.cuda.Event(enable_timing=True) for _ in range(k)]

    stage.ctx.bind_stream()
    if world > 1:
        dist.barrier()  # every rank set up before the first exchange (mailbox waits are bounded)
    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        step(events())
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = []
    launches0 = stage.ctx.launch_count()
    with ClockSampler(local) as clk:
        t_host = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev = events()
            step(ev)
            evs.append(ev)
        host_enqueue_ms = (time.perf_counter() - t_host) * 1e3 / max(args.steps, 1)  # host time per step
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = stage.ctx.launch_count() - launches0
    step_ms = [e[0].elapsed_time(e[1]) for e in evs]
    total_s = sum(step_ms) / 1e3
    # per-kernel breakdown (separate loop: events between the kernels serialize their launches)
    bevs = []
    for _ in range(min(args.steps, 10)):
        flush.zero_()
        ev = events(4)
        step(ev)
        bevs.append(ev)
    torch.cuda.synchronize()
    infer_ms = [e[0].elapsed_time(e[1]) for e in bevs]
    decide_ms = [e[1].elapsed_time(e[2]) for e in bevs]
    compact_ms = [e[2].elapsed_time(e[3]) for e in bevs]
    # K-A0 alone (the level-plane encode the AID stage launches first), same batch, same L2 flush
    levels_ms = []
    if args.variant == "aid":
        planes = torch.empty((8, n, 2), dtype=torch.float32, device=dev)
        for _ in range(min(args.steps, 10)):
            flush.zero_()
            ev = events()
            ev[0].record(torch.cuda.current_stream())
            _capi.check(stage.handle, lib.nrrs_gpu_encode_levels(stage.handle, dv["p01"].data_ptr(), n,
                                                                 planes.data_ptr(), n))
            ev[1].record(torch.cuda.current_stream())
            levels_ms.append(ev)
        torch.cuda.synchronize()
        levels_ms = [e[0].elapsed_time(e[1]) for e in levels_ms]
        del planes
    t = torch.tensor([total_s], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max over ranks
    total_s = float(t.item())
    value = (args.vertices if args.strong else world * n) * args.steps / total_s
    res = _capi.StageResultC()
    if sh is not None and pending[0] is not None:
        po = pending[0].resolve(rc)  # the last timed depth's global outcome (host read after the loop)
        assert po.dropped == 0 or po.spawned == cap
    if sh is None:
        _capi.check(stage.handle, lib.nrrs_gpu_fetch_result(stage.handle, ctypes.byref(res)))
        spawned = int(res.spawned)
    else:
        spawned = int(sh._total.item())

    # ---- e2e: the C ABI host-buffer entry (H2D + stage + D2H every step) ----
    e2e = None
    if world == 1:
        pinned = {k: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).pin_memory().numpy()
                  for k, a in hv.items() if k != "pixel"}
        pinned["path_key"] = pinned["path_key"].view(np.uint64)
        hout = {"q_norm": torch.empty(n, dtype=torch.float32).pin_memory().numpy(),
                "q_real": torch.empty(n, dtype=torch.float32).pin_memory().numpy(),
                "slots": torch.empty((slot_cap, 2), dtype=torch.int32).pin_memory().numpy().view(np.uint32)}
        for _ in range(3):
            stage.run_host(pinned, 2, strategy, rc=RateControl(), out=hout)
        torch.cuda.synchronize()
        e_times, d2h = [], 0
        for _ in range(max(3, args.steps // 2)):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, r = stage.run_host(pinned, 2, strategy, rc=RateControl(), out=hout)
            e_times.append(time.perf_counter() - t0)
            d2h = 8 * n + 8 * r.spawned
        sync_value = n / statistics.mean(e_times)
        sync_d2h = d2h
        # the same calls as a stream of batches, two in flight (nrrs_gpu_rrs_stage_host_async): the inputs
        # of call i+1 stream in while the outputs of call i stream out; every step still copies its inputs
        # in and its outputs (q_norm, q_real, the slot array, the scalars) back
        houts = [hout, {"q_norm": torch.empty(n, dtype=torch.float32).pin_memory().numpy(),
                        "q_real": torch.empty(n, dtype=torch.float32).pin_memory().numpy(),
                        "slots": torch.empty((slot_cap, 2), dtype=torch.int32).pin_memory().numpy()
                        .view(np.uint32)}]
        gain0 = RateControl().gain()
        a_steps = max(6, args.steps)

        def pipelined(k):
            tickets, results = [], []
            for i in range(k):
                if len(tickets) == 2:
                    results.append(stage.wait_host(tickets.pop(0)))
                t, _ = stage.submit_host(pinned, 2, strategy, gain0, out=houts[i % 2])
                tickets.append(t)
            for t in tickets:
                results.append(stage.wait_host(t))
            return results
        pipelined(4)
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rs = pipelined(a_steps)
        a_s = time.perf_counter() - t0
        assert all(r.spawned == rs[0].spawned and r.dropped == 0 for r in rs)
        d2h = 8 * n + 8 * slot_cap
        e2e = {"value": n * a_steps / a_s, "unit": "vertices/s", "h2d_bytes_per_step": 56 * n,
               "d2h_bytes_per_step": d2h,
               "path": "nrrs_gpu_rrs_stage_host_async, two calls in flight (pinned host buffers; chunked H2D "
                       "overlapped with K-A; call i's D2H overlaps call i+1's H2D); wall clock over "
                       f"{a_steps} consecutive steps",
               "sync": {"value": sync_value, "d2h_bytes_per_step": sync_d2h,
                        "path": "nrrs_gpu_rrs_stage_host, one call at a time (H2D, stage, D2H serialized)"}}
        # the floor e2e can reach: the step's bytes over the measured pinned copy bandwidths (H2D and D2H
        # cannot overlap inside one call -- q_norm needs the global F)
        hb = torch.empty(56 * n, dtype=torch.uint8).pin_memory()
        hb.fill_(1)  # touch the pages (an untouched pinned buffer copies at ~35 GB/s)
        db = torch.empty(56 * n, dtype=torch.uint8, device=dev)
        bw = {}
        piece = 16 << 20  # 16 MiB pieces: the link's streaming rate (tools/pcie_bw.py)
        for name, dst, src in (("h2d", db, hb), ("d2h", hb, db)):
            best = 0.0
            for _ in range(3):
                a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for o in range(0, 56 * n, piece):
                    dst[o:o + piece].copy_(src[o:o + piece], non_blocking=True)
                z.record()
                torch.cuda.synchronize()
                best = max(best, 56 * n / (a.elapsed_time(z) / 1e3))
            bw[name] = best
        e2e["copy_gbs"] = {k: v / 1e9 for k, v in bw.items()}
        # full duplex: the pipelined step is bound by the larger direction; one call at a time pays both
        e2e["pcie_floor"] = n / max(56 * n / bw["h2d"], d2h / bw["d2h"])
        e2e["frac_of_floor"] = e2e["value"] / e2e["pcie_floor"]
        e2e["sync"]["pcie_floor"] = n / (56 * n / bw["h2d"] + sync_d2h / bw["d2h"])
        e2e["sync"]["frac_of_floor"] = sync_value / e2e["sync"]["pcie_floor"]
        del hb, db
    else:
        # N>1: each rank copies its band in from pinned host memory, runs the sharded stage (two
        # exchanges) and reads q_norm/q_real and its kept slot records back; max over ranks.
        pinned_t = {k: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).pin_memory()
                    for k, a in hv.items() if k != "pixel"}
        hq = torch.empty(n, dtype=torch.float32).pin_memory()
        hr = torch.empty(n, dtype=torch.float32).pin_memory()
        hs = torch.empty((slot_cap, 2), dtype=torch.int32).pin_memory()
        e_tot, e_steps, d2h = 0.0, max(3, args.steps // 2), 0
        for i in range(3 + e_steps):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            for k in dv:
                dv[k].copy_(pinned_t[k], non_blocking=True)
            _, oc_ = sh.run(dv, 2, strategy, rc=RateControl(), out=out)
            hq.copy_(out.q_norm, non_blocking=True)
            hr.copy_(out.q_real, non_blocking=True)
            if oc_.kept:
                hs[:oc_.kept].copy_(out.slots[:oc_.kept], non_blocking=True)
            torch.cuda.synchronize()
            if i >= 3:
                e_tot += time.perf_counter() - t0
            d2h = 8 * n + 8 * oc_.kept
        te = torch.tensor([e_tot], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": (args.vertices if args.strong else world * n) * e_steps / float(te.item()),
               "unit": "vertices/s",
               "h2d_bytes_per_step": 56 * n, "d2h_bytes_per_step": d2h,
               "path": "ShardedRrsStage.run per rank (pinned host buffers, per-rank bytes, max over ranks)"}

    # ---- side measurements: other strategies (Mix-Depth candidates) on the same batch ----
    extra = {}
    if world == 1 and not args.no_extra:
        alt_nets = NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Nrrs if variant == RrsVariant.Aid
                                             else RrsVariant.Aid, seed=1)).randomize_for_benchmark()
        for name, strat, nn in (("nrrs" if variant == RrsVariant.Aid else "aid-nrrs",
                                 Strategy(StrategyKind.Nrrs), alt_nets),
                                ("adrrs-nn", Strategy(StrategyKind.AdrrsNn), nets),
                                ("throughput", Strategy(StrategyKind.Throughput), nets),
                                ("depth1-fixed", None, nets)):
            stg = RrsStage(npx, nn, device=local)
            o2 = stg.alloc_outputs(n)
            depth = 1 if strat is None else 2
            s2 = strat or Strategy(StrategyKind.Fixed, 1.0)
            for _ in range(3):
                stg.run(dv, depth, s2, rc=None, out=o2, sync=False)
            ts = []
            for _ in range(5):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                stg.run(dv, depth, s2, rc=None, out=o2, sync=False)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            extra[name] = {"vertices_per_s": n / (statistics.mean(ts) / 1e3), "ms": statistics.mean(ts)}
            stg.close()
        # the configs[2] batch again, through alternative AID forms chosen at context creation:
        # fp32 grid tables (no fp16 error budget spent) and the opt-in fused single-kernel stage
        if variant == RrsVariant.Aid:
            for name, env in (("aid-nrrs-fp32-tables", "NRRS_FP32_TABLES"), ("aid-nrrs-fused-kernel", "NRRS_FUSED")):
                os.environ[env] = "1"
                try:
                    stg = RrsStage(npx, nets, device=local)
                finally:
                    del os.environ[env]
                o2 = stg.alloc_outputs(n)
                for _ in range(3):
                    stg.run(dv, 2, strategy, rc=None, out=o2, sync=False)
                ts = []
                for _ in range(5):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    stg.run(dv, 2, strategy, rc=None, out=o2, sync=False)
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                half, perr = stg.table_precision()
                extra[name] = {"vertices_per_s": n / (statistics.mean(ts) / 1e3), "ms": statistics.mean(ts),
                               "aid_fp16_tables": half}
                stg.close()
        # render-like, spatially coherent batch in pixel order, same strategy and nets
        hc = synthetic.gen_cornell_vertices(1920, 1080)
        dc = {k: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).to(dev)
              for k, a in hc.items() if k != "pixel"}
        stg = RrsStage(hc["roughness"].shape[0], nets, device=local)
        o2 = stg.alloc_outputs(hc["roughness"].shape[0])
        for _ in range(3):
            stg.run(dc, 2, strategy, rc=None, out=o2, sync=False)
        ts = []
        for _ in range(5):
            flush.zero_()
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            stg.run(dc, 2, strategy, rc=None, out=o2, sync=False)
            z.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(z))
        extra[f"{args.variant}-nrrs-cornell-coherent"] = {
            "vertices_per_s": hc["roughness"].shape[0] / (statistics.mean(ts) / 1e3), "ms": statistics.mean(ts),
            "batch": "1920x1080 first hits of a closed Cornell-style box, pixel order (synthetic.gen_cornell_vertices)"}
        stg.close()
        del dc

    # ---- C1: 65,536 vertices is launch-bound; single-call latency and CUDA-graph
    # replays of 1000 stage calls (K-A + K-B), same strategy and nets ----
    c1 = None
    if world == 1 and not args.no_extra:
        # configs[0]: NRRS normalized-RRS step on 65,536 synthetic vertices, random-init RRSNet, split
        # bound 4 (C1).  Launch-bound: per-call times from CUDA-graph replays of 100
        # calls, plus the single-call latency; the decision-only variant feeds the split-bound-4
        # factors q = RngStream(0xACC02, i).next_float() * 4 to the decide step alone.
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import oracle as orc_c1  # split-bound-4 factor generator + CPU port (baseline only)
        n1 = 65536
        hv1 = synthetic.gen_vertices(n1, n_pixels=n1)
        dv1 = {k: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).to(dev)
               for k, a in hv1.items() if k != "pixel"}

        def graph_us(st, kind, nets_variant):
            o = st.alloc_outputs(n1)
            for _ in range(5):
                st.run(dv1, 2, Strategy(kind), rc=RateControl(), out=o, sync=False)
            torch.cuda.synchronize()
            lat = []
            for _ in range(30):
                a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                st.run(dv1, 2, Strategy(kind), rc=RateControl(), out=o, sync=False)
                z.record()
                torch.cuda.synchronize()
                lat.append(a.elapsed_time(z) * 1e3)
            g = st.capture(dv1, 2, Strategy(kind), o, gain=RateControl().gain(), calls=100)
            g.replay()
            torch.cuda.synchronize()
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                g.replay()
            z.record()
            torch.cuda.synchronize()
            return statistics.median(lat), a.elapsed_time(z) * 1e3 / 1000

        nrrs_nets = NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Nrrs, seed=1)).randomize_for_benchmark()
        st1 = RrsStage(n1, nrrs_nets, device=local)
        single, per_call = graph_us(st1, StrategyKind.Nrrs, RrsVariant.Nrrs)
        # decision-only: the split-bound-4 factors through the decide step (K-B) alone
        q4 = torch.from_numpy(orc_c1.split_bound_factors(n1)).to(dev)
        o1 = st1.alloc_outputs(n1)
        o1.q_orig = torch.empty(n1, dtype=torch.float32, device=dev)
        o1.u = torch.empty(n1, dtype=torch.float32, device=dev)
        p1 = st1.params(2, Strategy(StrategyKind.Throughput), RateControl().gain())
        from paper_2510_07868_b200.stage import vertex_soa as _vsoa
        soa1, oc1 = _vsoa(dv1), o1.c()
        ls1 = torch.zeros(1, dtype=torch.float64, device=dev)
        tot1 = torch.zeros(1, dtype=torch.int64, device=dev)
        st1.ctx.bind_stream()
        _capi.check(st1.handle, lib.nrrs_gpu_stage_factors(st1.handle, ctypes.byref(soa1), n1, ctypes.byref(p1),
                                                           ctypes.byref(oc1), ls1.data_ptr()))  # u for these keys
        o1.q_orig.copy_(q4)
        s4 = torch.tensor([float(q4.double().sum())], dtype=torch.float64, device=dev)
        torch.cuda.synchronize()

        def decide_only():
            _capi.check(st1.handle, lib.nrrs_gpu_stage_decide(st1.handle, n1, ctypes.byref(p1), s4.data_ptr(), 1,
                                                              ctypes.byref(oc1), tot1.data_ptr()))
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            st1.ctx.bind_stream()
            decide_only()
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize()
        gd = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gd):
            st1.ctx.bind_stream()
            for _ in range(100):
                decide_only()
        st1.ctx.bind_stream()
        gd.replay()
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            gd.replay()
        z.record()
        torch.cuda.synchronize()
        dec_us = a.elapsed_time(z) * 1e3 / 1000
        st1.close()
        # AID at C1 through the default routing (the fused single-kernel stage up to 196,608
        # vertices) and through K-A0 + K-A + K-B (NRRS_FUSED=0)
        st2 = RrsStage(n1, nets, device=local)
        _, aid_call = graph_us(st2, StrategyKind.AidNrrs, RrsVariant.Aid)
        st2.close()
        os.environ["NRRS_FUSED"] = "0"
        try:
            st3 = RrsStage(n1, nets, device=local)
        finally:
            del os.environ["NRRS_FUSED"]
        _, aid_3k_call = graph_us(st3, StrategyKind.AidNrrs, RrsVariant.Aid)
        st3.close()
        # CPU port of the same NRRS step and decision-only step on this host
        vc = orc_c1.gen_vertices(n1)
        onn = orc_c1.OracleNets(orc_c1.VARIANT_NRRS, seed=1, randomize=True)
        thr = orc_c1.threads_available()
        cap1 = orc_c1.lib().orc_queue_capacity_for(n1)
        t0 = time.perf_counter()
        for _ in range(3):
            orc_c1.rrs_stage(vc, 2, n1, cap1, orc_c1.NRRS, onn, gain=0.85, seed=0, threads=thr)
        cpu_stage_s = (time.perf_counter() - t0) / 3
        c1 = {"config": "configs[0]: NRRS normalized-RRS step, 65,536 synthetic vertices, random-init RRSNet, "
                        "split bound 4 (SURVEY.md 8d C1)", "vertices": n1,
              "nrrs_stage": {"graph_us_per_call": per_call, "single_call_us": single,
                             "vertices_per_s": n1 / (per_call / 1e6),
                             "hbm_gbs": (STAGE_READ + STAGE_WRITE + 8 * 0.85) * n1 / (per_call / 1e6) / 1e9},
              "decision_only_split_bound4": {"graph_us_per_call": dec_us, "vertices_per_s": n1 / (dec_us / 1e6),
                                             "kernel": "decide3 (normalize, gain, stochastic round, prefix, slots)"},
              "aid_stage_graph_us_per_call": aid_call, "aid_three_kernel_graph_us_per_call": aid_3k_call,
              "cpu_port": {"nrrs_stage_vertices_per_s": n1 / cpu_stage_s, "cores": thr,
                           "sample": "the same 65,536-vertex NRRS step (oracle port), mean of 3"},
              "note": "launch-bound: ~2-3 kernels per call; the per-call floor of two dependent launches on "
                      "this stream is the throughput-heuristic stage"}

    # ---- suffix side: reverse pass + TrainSample emission + k_i + Film update
    # over a synthetic 4-depth vertex tree in queue order, 2,073,600 depth-1 vertices ----
    suffix = None
    if world == 1 and not args.no_extra:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import oracle as orc_gen  # synthetic tree generator (host-side input only)
        from paper_2510_07868_b200.film import GpuFilm, SuffixStage
        sizes = [n, int(n * 0.85), int(n * 0.6), int(n * 0.4)]
        tree = orc_gen.gen_vertex_tree(sizes, n)
        gv = [None] + [{k: torch.from_numpy(np.ascontiguousarray(a)).to(dev) for k, a in v.items()}
                       for v in tree[1:]]
        s0 = [None] + [v["s"].clone() for v in gv[1:]]
        sx = SuffixStage(local)
        film = GpuFilm(1920, 1080, sx)
        frame = torch.rand((1920 * 1080, 3), dtype=torch.float64, device=dev)
        i_acc = torch.rand((n, 3), dtype=torch.float32, device=dev)
        recs = torch.empty((sum(sizes), 80), dtype=torch.uint8, device=dev)

        def suffix_step():
            for d in range(1, len(gv)):
                gv[d]["s"].copy_(s0[d])
            sx.reverse_pass(gv)
            cnt, _ = sx.emit_train(gv, i_acc, n, recs)
            film.add_frame(frame)
            film.roll_acc()
            return cnt

        for _ in range(3):
            suffix_step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            cnt = suffix_step()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        nv = sum(sizes)
        suffix = {"vertices": nv, "depths": len(sizes), "train_samples": cnt, "ms": 1e3 * statistics.mean(ts),
                  "vertices_per_s": nv / statistics.mean(ts),
                  "note": "wall time per frame incl. the host syncs of fold/k_i error checks; bit-exact vs the "
                          "reference order (tests/test_gpu_film.py)"}
        sx.close()
        del gv, s0, recs

    # ---- online training: one StatNet step at the reference batch (1 << 16) ----
    train = None
    if world == 1 and not args.no_extra:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import oracle as orc_gen  # synthetic TrainSamples (host-side input only)
        from paper_2510_07868_b200.training import FULL, NeuralRrsTrainer, StatNetTrainer
        nb = 1 << 16
        hb = orc_gen.gen_train_batch(nb, seed=5)
        db = torch.from_numpy(hb.view(np.uint8).reshape(nb, 80).copy()).to(dev)
        tr = StatNetTrainer(NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Nrrs, seed=1)).randomize_for_benchmark(),
                            device=local)
        for _ in range(3):
            tr.step(db)
        torch.cuda.synchronize()
        ts, losses = [], []
        for _ in range(10):
            t0 = time.perf_counter()
            loss, _ = tr.step(db)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            losses.append(loss)
        # the same step on the host: the oracle's stat_loss_impl + Adam/EMA (1 thread, C port)
        on = orc_gen.OracleNets(orc_gen.VARIANT_NRRS, seed=1, randomize=True)
        t0 = time.perf_counter()
        _, gm_h, gg_h = orc_gen.stat_loss(on, hb)
        for arr, g in ((on.stat_mlp, gm_h), (on.stat_grid, gg_h)):
            orc_gen.adam_step(arr, g, np.zeros_like(arr), np.zeros_like(arr), 1, 0.005)
            orc_gen.ema_update(arr.copy(), arr)
        cpu_ms = 1e3 * (time.perf_counter() - t0)
        # a whole train_frame chunk: StatNet step + AID RRSNet step (full phase, pixel errors)
        ntr = NeuralRrsTrainer(nets, device=local, batch=nb)
        hb2 = hb.copy()
        hb2["q_real"] = np.float32(1.5)
        hb2["q_norm"] = np.float32(1.2)
        db2 = torch.from_numpy(hb2.view(np.uint8).reshape(nb, 80).copy()).to(dev)
        errs = torch.rand((1024, 2), dtype=torch.float32, device=dev)
        for _ in range(3):
            ntr.train_frame(db2, errs, 0.5, FULL)
        torch.cuda.synchronize()
        tf = []
        for _ in range(10):
            t0 = time.perf_counter()
            ntr.train_frame(db2, errs, 0.5, FULL)
            torch.cuda.synchronize()
            tf.append(time.perf_counter() - t0)
        ntr.close()
        train = {"batch": nb, "ms_per_step": 1e3 * statistics.mean(ts), "samples_per_s": nb / statistics.mean(ts),
                 "train_frame_chunk_ms": 1e3 * statistics.mean(tf),
                 "cpu_port_ms_per_step": cpu_ms,
                 "params": int(tr.grid.numel() + tr.mlp.numel()), "loss_first": losses[0], "loss_last": losses[-1],
                 "note": "ms_per_step: step_statnet (loss + gradients + Adam + EMA); train_frame_chunk_ms: "
                         "step_statnet + step_rrsnet (AID, full phase); wall time incl. the finite-check syncs"}
        tr.close()

    # ---- GPU trace_frame: configs[2] shape C3, AID-NRRS at depths >= 2 on
    # builtin:cornell 1920x1080, B = 16, the RRS stage inside the full wavefront renderer ----
    trace = None
    if world == 1 and not args.no_extra:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import oracle as orc_gen  # CPU port timing only
        from paper_2510_07868_b200 import render as rnd
        from paper_2510_07868_b200.film import GpuFilm, SuffixStage
        from paper_2510_07868_b200.rrs import Strategy as St, StrategyKind as SK
        tw, th, tb = 1920, 1080, 16
        kind = SK.AidNrrs if variant == RrsVariant.Aid else SK.Nrrs
        tst = RrsStage(tw * th, nets, device=local)
        desc = rnd.make_cornell_scene()
        tscene = rnd.GpuScene(desc, ctx=tst.ctx)
        tracer = rnd.Tracer(tscene, tw * th, tb)
        tfilm = GpuFilm(tw, th, SuffixStage(ctx=tst.ctx))
        assign = [St()] + [St(kind)] * (tb - 1)
        trc = RateControl()
        reps, tts = [], []
        for f in range(6):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep_f, _ = tracer.trace_frame(assign, rnd.TraceConfig(max_depth=tb, seed=7, frame_index=f), trc, tfilm)
            torch.cuda.synchronize()
            tts.append(time.perf_counter() - t0)
            reps.append(rep_f)
            tfilm.roll_acc()
        tts, reps = tts[2:], reps[2:]  # frames 0-1 warm up (the first roll_acc'd frame pays one-time costs)
        nverts = statistics.mean(sum(r.depth_counts) for r in reps)
        rays = statistics.mean(r.camera_rays + r.scatter_rays + r.shadow_rays for r in reps)
        ms = 1e3 * statistics.median(tts)
        # the same frame shape through the C port of the reference loop (1 thread, brute-force hits,
        # a 96x54 crop of the film so the sample stays a few seconds)
        on = orc_gen.OracleNets(orc_gen.VARIANT_AID if variant == RrsVariant.Aid else orc_gen.VARIANT_NRRS, seed=1,
                                randomize=True)
        cw, ch = 96, 54
        t0 = time.perf_counter()
        cr = orc_gen.trace_frame(desc, cw, ch, [(0, 1.0)] + [(int(kind), 1.0)] * (tb - 1), tb, seed=7, nets=on)
        cpu_s = time.perf_counter() - t0
        trace = {"config": "C3 shape: builtin:cornell 1920x1080, B=16, fixed at depth 1 then "
                           f"{'aid-nrrs' if kind == SK.AidNrrs else 'nrrs'} (random-init networks), RateControl on",
                 "ms_per_frame": ms, "path_vertices_per_frame": nverts, "path_vertices_per_s": nverts / (ms / 1e3),
                 "rays_per_s": rays / (ms / 1e3), "depth_counts": reps[-1].depth_counts,
                 "shadow_rays": reps[-1].shadow_rays,
                 "cpu_port": {"sample": f"{cw}x{ch} crop, same scene / depth / strategy, 1 thread",
                              "path_vertices_per_s": sum(cr["report"]["depth_counts"]) / cpu_s, "cores": 1},
                 "note": "wall time per frame incl. ~3 host syncs per depth; camera + per-depth shade / compaction "
                         "/ RRS stage / scatter (NEE + BSDF) / folds, reverse pass, Film::add_frame"}
        tracer.close()
        tscene.close()
        tst.close()
        # configs[1]: NRRS full wavefront render, builtin:cornell 512x512, 16 spp (16 frames), B = 12
        cw1, ch1, cb1, nf1 = 512, 512, 12, 16
        nets1 = NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Nrrs, seed=1)).randomize_for_benchmark()
        st1 = RrsStage(cw1 * ch1, nets1, device=local)
        sc1 = rnd.GpuScene(desc, ctx=st1.ctx)
        tr1 = rnd.Tracer(sc1, cw1 * ch1, cb1)
        film1 = GpuFilm(cw1, ch1, SuffixStage(ctx=st1.ctx))
        assign1 = [St()] + [St(SK.Nrrs)] * (cb1 - 1)
        rc1 = RateControl()
        for f in range(2):  # warm-up frames (one-time allocations)
            tr1.trace_frame(assign1, rnd.TraceConfig(max_depth=cb1, seed=11, frame_index=f), rc1, film1)
            film1.roll_acc()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps1 = []
        for f in range(nf1):
            r1, _ = tr1.trace_frame(assign1, rnd.TraceConfig(max_depth=cb1, seed=11, frame_index=2 + f), rc1, film1)
            film1.roll_acc()
            reps1.append(r1)
        torch.cuda.synchronize()
        s1 = time.perf_counter() - t0
        v1 = sum(sum(r.depth_counts) for r in reps1)
        trace["configs1"] = {
            "config": "configs[1]: NRRS full wavefront render, builtin:cornell 512x512, 16 spp (16 frames), max "
                      "depth 12, fixed at depth 1 then nrrs (random-init networks), RateControl on",
            "render_ms": 1e3 * s1, "ms_per_frame": 1e3 * s1 / nf1, "path_vertices": v1,
            "path_vertices_per_s": v1 / s1, "depth_counts_last_frame": reps1[-1].depth_counts,
            "note": "wall time of the 16 frames (camera, per-depth shade / stage / scatter / folds, reverse pass, "
                    "Film::add_frame, roll_acc); path vertices = surface vertices over all depths and frames"}
        tr1.close()
        sc1.close()
        st1.close()

    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    hbm = peaks.get("hbm_gbs")
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    if not hbm:
        hbm, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    infer_avg = statistics.mean(infer_ms) / 1e3
    achieved = ALG_BYTES_INFER * n / infer_avg / 1e9
    prof = load_json(os.path.join(ROOT, "profiles", "ncu_summary.json")) or {}
    traffic = prof.get(f"infer_{args.variant}_dram_bytes_per_launch")
    stage_bytes = (STAGE_READ + STAGE_WRITE) * n + 8 * spawned
    gu = GATHER_UNITS_PER_VERTEX[args.variant]
    line = {
        "metric": METRIC, "value": value, "unit": "vertices/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": 1e3 * total_s / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
        "dtype": "fp16x3-split MMA (fp32 accumulate), fp16 AID grid, f32 encodings; f64 sum", "data": "synthetic",
        "config": {"workload": (f"configs[3] shape: {args.variant}-nrrs stage over ONE {args.vertices}-vertex "
                                f"synthetic film split into {world} row bands at depth 2 (SURVEY.md 8d, 8e), "
                                f"+ compaction (~10% invalid slots)") if args.strong else
                               (f"configs[2] shape: {args.variant}-nrrs stage over a 1920x1080 synthetic vertex "
                                f"batch per GPU at depth 2 (SURVEY.md 8d), + compaction (~10% invalid slots)"
                                + ("; N=8 is the configs[4] 16.6 M-vertex batch" if world > 1 else "")),
                   "vertices_per_gpu": n, "n_pixels": npx, "capacity": cap, "strategy": f"{args.variant}-nrrs",
                   "depth": 2, "gain": 0.85, "parallelism": f"tile-sharded dp{world}",
                   "exchange": (exchange if world > 1 or force_sharded else "none"),
                   "l2": "flushed between timed steps (256 MiB write outside the events)",
                   "aid_tables": aid_tables},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic,
                     "kernel": ("K-A0 grid_level_kernel + K-A infer_aid_fused_kernel<8> (level planes, 8 self-contained "
                                "MLP groups): the strategy-factor step of the stage, timed as one unit"
                                if args.variant == "aid" else
                                "K-A0 grid_level_kernel<true> + K-A infer_stat_planes_kernel<Nrrs> (fp32 StatNet "
                                "grid one (level, feature) table per CTA; StatNet + RRSNet chains)"),
                     "alg_bytes_per_vertex": ALG_BYTES_INFER, "peak_source": peak_src,
                     "stage_frac": (stage_bytes / (statistics.mean(step_ms) / 1e3) / 1e9) / hbm},
        "kernels_ms": {"infer": statistics.mean(infer_ms), "decide": statistics.mean(decide_ms),
                       "compact": statistics.mean(compact_ms)},
        "clocks": clk.summary(),
        "gpu_launches": launches,
        "host_enqueue_ms_per_step": host_enqueue_ms,
        "spawned": spawned,
    }
    if levels_ms:
        lv = statistics.mean(levels_ms) / 1e3
        line["kernels_ms"]["infer_grid_levels"] = 1e3 * lv  # K-A0 alone; "infer" = K-A0 + K-A
        line["gather_roofline"] = {
            "bound": "smem_random_loads", "kernel": "K-A0 grid_level_kernel", "unit": "4-byte loads/s",
            "achieved": SMEM_LOADS_PER_VERTEX * n / lv, "peak": SMEM_LOAD_CEILING_PER_S,
            "frac": SMEM_LOADS_PER_VERTEX * n / lv / SMEM_LOAD_CEILING_PER_S,
            "units_per_vertex": SMEM_LOADS_PER_VERTEX,
            "peak_source": "measured, profiles/r01_microbench_gather_bw.txt (tools/gather_bw.cu)"}
    else:
        line["gather_roofline"] = {
            "bound": "l2_scattered_gathers", "unit": "gathers/s (8-byte equivalents)",
            "achieved": gu * n / infer_avg, "peak": GATHER_CEILING_PER_S,
            "frac": gu * n / infer_avg / GATHER_CEILING_PER_S, "units_per_vertex": gu,
            "peak_source": "measured, profiles/r01_microbench_gather_bw.txt"}
    ipv = prof.get("instructions_per_vertex") if args.variant == "aid" else None
    if ipv:
        # HBM does not bind this stage: every kernel is issue-bound (profiles/r02_stage_kernels.txt);
        # the instruction-issue ceiling = 4 warp-instructions per clock per SM at the max SM clock
        wi = sum(v for k, v in ipv.items() if not k.startswith("_"))
        sm_hz = peaks.get("sm_max_mhz", 1965.0) * 1e6
        issue_peak = 4.0 * 148 * sm_hz / wi
        line["issue_roofline"] = {
            "bound": "instruction issue", "unit": "vertices/s", "achieved": value, "peak": issue_peak,
            "frac": value / issue_peak, "warp_instructions_per_vertex": wi,
            "per_kernel": {k: v for k, v in ipv.items() if not k.startswith("_")},
            "peak_source": "4 warp-instructions/clk/SM x 148 SMs x MEASURED_PEAKS sm_max_mhz; instruction counts: "
                           "smsp__inst_executed.sum of the ncu capture (profiles/ncu_summary.json)"}
    if e2e:
        line["e2e"] = e2e
    if extra:
        line["strategies"] = extra
    if c1:
        c1["nrrs_stage"]["hbm_frac"] = c1["nrrs_stage"]["hbm_gbs"] / hbm
        line["configs0_c1"] = c1
    if suffix:
        line["suffix_stage"] = suffix
    if train:
        line["statnet_train_step"] = train
    if trace is not None:
        line["trace_frame"] = trace
    if world == 1 and rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args.variant)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
    if world > 1 or force_sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
