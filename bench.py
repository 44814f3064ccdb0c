#!/usr/bin/env python
"""Benchmark of the B200 TRS partitioner hot path (BASELINE.json metric).

One STEP = one pass of the hot path over one batch of synthetic input: the
K1 texture pass over the batch's luma frames, K2/K3 tables, and the two-step
search (step 1 + step 2) for every frame of the batch.  Default workload:
BASELINE config 3 (32 frames of 3840x2160 10-bit luma, 30x17 CTU grid,
n=8 slices, exhaustive tile columns) -- the "at 4K" configuration the metric
is quoted on that fits one GPU.  Config 1 is the reference's CPU-runnable
case; configs 2/4/5 are parity cases (tests/).

value  = TRS candidates resolved per second over the whole job, inputs
         resident in HBM (device pointers into sc_partition_frames).  A
         candidate is one (frame, candidate) pair counted by the reference's
         own counters (candidates_step1 + candidates_step2, search.hpp:41-43);
         candidates_scored_by_the_walks_per_s beside it counts only what the
         walks evaluated (step 2 skips subtrees over its budget).
e2e    = the same metric through the public C-ABI call with HOST (pinned)
         buffers: the H2D copy of that step's luma + estimate maps and the D2H
         of the per-frame results happen inside the timed region.
Multi-GPU (torchrun): frames are independent once estimated,
so every rank partitions its own batch (POCs offset by rank) -- weak scaling,
no data-path collective; the timed region is barrier-bracketed and the max
over ranks is reported.  --shard candidates instead splits each frame's
candidate space over the ranks (strong scaling, cfg4/cfg5 style): one
sc_shard_best record per frame is all-gathered after each step.

--impl reference runs the UNMODIFIED reference CPU path (oracle/_ref, built
from /root/reference; the C oracle port when that is absent) on the host
cores: whole frames of the same workload (full enumeration), one frame per
host thread, a step being one frame (bounded sample: --steps frames).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TRS candidates scored/sec & frames partitioned/sec at 4K; texture pass GB/s"
UNIT = "candidates/s"
DATA = "synthetic (seeded; SURVEY.md \u00a78d generator, synth/libscsynth.so; no public dataset)"
VALUE_DEF = ("candidates resolved per second: the reference's own per-frame counters "
             "candidates_step1 + candidates_step2 (search.hpp:41-43) summed over the frames of "
             "a step, per second of step time.  Step 1 scores every candidate; step 2 resolves "
             "the family under the t_min*(1+lambda) budget (the B200 walk skips subtrees whose "
             "fixed slices already exceed it: candidates_scored_by_the_walks_per_s counts what "
             "it actually scored)")


def workload_config(w, counts):
    """The workload-defining config, identical in both arms."""
    cols, rows = -(-w.width // w.ctu), -(-w.height // w.ctu)
    return {"workload": w.name, "frames_per_rank": w.frames, "frame": f"{w.width}x{w.height}",
            "bit_depth": w.bit_depth, "ctu": w.ctu, "grid": f"{cols}x{rows}",
            "n_slices": w.n_slices, "max_tile_cols": w.max_tile_cols, "lambda": 0.0,
            "k_area": 3.0, "coverage": "reference",
            "candidates_per_frame_step": [list(c) for c in counts],
            "l2": "inputs larger than L2 (luma batch %.0f MB per %d frames)"
                  % (w.frames * w.width * w.height * w.bps / 1e6, w.frames)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---- clocks sampler (during the timed region) -----------------------------------
class Clocks:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed
    region: NVML polled every 2 ms from a background thread (a step is a few
    ms, so nvidia-smi's 100 ms loop would often see none); nvidia-smi -lms
    as the fallback where NVML is unavailable."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []
        self.nvml = None
        self.samples = []  # (sm_mhz, reason bitmask)
        self.reason_bits = {}
        try:
            import pynvml as N
            N.nvmlInit()
            self.nvml = N
            self.h = N.nvmlDeviceGetHandleByIndex(gpu)
            self.smax = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
            self.reason_bits = {
                "hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        except Exception:
            self.nvml = None

    def start(self):
        if self.nvml is not None:
            self._stop = threading.Event()
            self.samples = []

            def poll():
                N = self.nvml
                while not self._stop.is_set():
                    try:
                        self.samples.append(
                            (float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)),
                             int(N.nvmlDeviceGetCurrentClocksEventReasons(self.h))))
                    except Exception:
                        pass
                    self._stop.wait(0.002)
            self._t = threading.Thread(target=poll, daemon=True)
            self._t.start()
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:  # first sample in hand
                time.sleep(0.02)
            self.lines.clear()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            self._stop.set()
            self._t.join(timeout=2)
            sm = [c for c, _ in self.samples]
            reasons = set()
            for _, m in self.samples:
                for nm, bit in self.reason_bits.items():
                    if m & bit:
                        reasons.add(nm)
            return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.smax,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


def make_inputs(w, rank, frames, pinned=True):
    import torch
    from paper_2012_14792_b200 import workloads as wl
    first = rank * frames + 1
    dt = torch.uint8 if w.bps == 1 else torch.int16
    luma_t = torch.empty((frames, w.height, w.width), dtype=dt, pin_memory=pinned)
    luma = luma_t.numpy().view(np.uint8 if w.bps == 1 else np.uint16)
    wl.synth_luma(w, frames=frames, first_poc=first, out=luma)
    tr = wl.cost_trace(w, frames=first + frames - 1)
    est_t = torch.empty((frames, w.grid().cell_count()), dtype=torch.float64, pin_memory=pinned)
    est_t.numpy()[:] = tr.est[first - 1:]
    return luma_t, est_t


def count_kernel_launches(fn, attempts=3):
    """Kernels launched by one untimed fn() call, counted from the CUDA
    activity trace (CUPTI via torch.profiler sees every kernel of the process,
    including the ones the C-ABI library launches on its own streams and the
    kernel nodes of its CUDA-graph replays).  CUPTI sometimes delivers an
    empty first session, so the capture is retried.  Returns (count, {name: n},
    source); when the profiler stays unusable, the count of the committed ncu
    launch list of this same command (profiles/launches_per_call.json)."""
    import tempfile
    from torch.profiler import ProfilerActivity, profile
    for _ in range(attempts):
        try:
            torch.cuda.synchronize()
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                fn()
                torch.cuda.synchronize()
            with tempfile.TemporaryDirectory() as td:
                path = os.path.join(td, "trace.json")
                prof.export_chrome_trace(path)
                ev = json.load(open(path)).get("traceEvents", [])
            names = {}
            for e in ev:
                if e.get("cat") == "kernel":
                    n = e.get("name", "?")
                    n = n.split("(")[0].replace("void ", "")[:60]
                    names[n] = names.get(n, 0) + 1
            total = sum(names.values())
            if total > 0:
                return total, names, "CUDA activity trace of one extra untimed call"
        except Exception:
            pass
    try:
        rec = json.load(open(os.path.join(ROOT, "profiles", "launches_per_call.json")))
        return int(rec["launches_per_call"]), rec.get("kernels", {}), \
            "profiles/launches_per_call.json (ncu launch list of this command; CUPTI gave no trace)"
    except Exception:
        return None, {}, "unavailable"


def kernel_src_sha():
    """Hash of the search-kernel sources an ncu instruction count belongs to."""
    import hashlib
    h = hashlib.sha256()
    for f in ("search_walk.cuh", "search.cu", "rank.cu", "plan.h", "trace.cuh", "trace.cu"):
        h.update(open(os.path.join(ROOT, "paper_2012_14792_b200", "csrc", f), "rb").read())
    return h.hexdigest()[:16]


# ---- our arm -------------------------------------------------------------------------
def run_ours(args):
    import ctypes as C

    import torch
    import torch.distributed as dist
    from paper_2012_14792_b200 import Partitioner, lib
    from paper_2012_14792_b200._abi import SearchResult, check
    from paper_2012_14792_b200 import workloads as wl

    rank, world, local = dist_env()
    # SLICECRAFT_BENCH_BACKEND=gloo (test only): exercise the multi-rank path
    # with more ranks than GPUs -- ranks share devices round-robin, their
    # kernels never wait on one another (frame sharding has no data-path
    # collective), and only the timing max crosses ranks, on the host
    backend = os.environ.get("SLICECRAFT_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    w = wl.WORKLOADS[args.config]
    F = w.frames
    g = w.grid()
    over = {}
    if args.lam is not None:
        over["lambda_"] = args.lam
    if args.coverage is not None:
        over["coverage"] = args.coverage
    cfg = w.cfg(mode=args.mode, **over)
    luma_h, est_h = make_inputs(w, rank, F)
    luma_d = luma_h.cuda()
    est_d = est_h.cuda()
    torch.cuda.synchronize()

    part = Partitioner(local)
    stream = torch.cuda.current_stream()
    check(lib().sc_ctx_set_stream(part._h, C.c_void_p(stream.cuda_stream)))
    res = (SearchResult * F)()
    bps = w.bps
    pitch, fstride = w.width * bps, w.width * w.height * bps
    gc, cc = g.c(), cfg.c()
    tim = (C.c_double * 8)()

    def call(luma_ptr, est_ptr):
        check(lib().sc_partition_frames(part._h, C.byref(gc), C.byref(cc), C.c_void_p(luma_ptr),
                                        bps, pitch, fstride, C.c_void_p(est_ptr), F, None,
                                        C.cast(res, C.c_void_p)))
        check(lib().sc_ctx_timings_ex(part._h, 8, tim))
        return [tim[i] for i in range(8)]

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up (device-resident) ----
    for _ in range(max(args.warmup, 0)):
        call(luma_d.data_ptr(), est_d.data_ptr())
    if args.warmup <= 0:
        call(luma_d.data_ptr(), est_d.data_ptr())  # counts for the metric
    # exact counts: the low 64 bits plus candidates_step*_hi (cfg5 is ~6.1e29)
    c1 = [r.candidates_step1 | (r.candidates_step1_hi << 64) for r in res]
    c2 = [r.candidates_step2 | (r.candidates_step2_hi << 64) for r in res]
    cands = sum(c1) + sum(c2)
    counts = sorted(set(zip(c1, c2)))
    # what the walks actually scored (transparency beside the reference-counted
    # value): step-2 leaves under the budget-bounded / pruned walks
    # (the exhaustive step 1 scores every candidate; the pruned and budget-
    # bounded walks count what they score)
    walked = sum((c1[i] if args.mode == 0 else r.leaves_scored_step1) + r.leaves_scored_step2
                 for i, r in enumerate(res))

    # ---- timed: device-resident inputs ----
    clocks = Clocks(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    phase = np.zeros(8)
    lib().sc_kernel_launches.restype = C.c_uint64
    launches0 = int(lib().sc_kernel_launches())
    e0.record(stream)
    for _ in range(args.steps):
        phase += np.array(call(luma_d.data_ptr(), est_d.data_ptr()))
    e1.record(stream)
    launches_timed = int(lib().sc_kernel_launches()) - launches0
    torch.cuda.synchronize()
    barrier()
    ck = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    phase /= args.steps

    # ---- timed: end to end from pinned host buffers ----
    barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(args.steps):
        call(luma_h.data_ptr(), est_h.data_ptr())
    e3.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_e2e = max_over_ranks(e2.elapsed_time(e3)) / args.steps

    # ---- K1 alone (sc_texture_moments, device pointers): the texture roofline ----
    # In the pipeline K1 runs on the low-priority side stream beside the time
    # tables (its in-pipeline time is reported too); here it is timed by itself.
    rec_d = torch.empty(F * g.cell_count() * 24, dtype=torch.uint8, device="cuda")
    tex_alone_us = None
    try:
        def k1():
            check(lib().sc_texture_moments(part._h, C.c_void_p(luma_d.data_ptr()), bps, w.width,
                                           w.height, pitch, fstride, w.ctu, F,
                                           C.c_void_p(rec_d.data_ptr())))
            check(lib().sc_ctx_timings_ex(part._h, 8, tim))
            return tim[0]  # the library's CUDA events around the K1 launch, on its stream
        for _ in range(3):
            k1()
        tex_alone_us = float(np.mean([k1() for _ in range(10)]))
    except Exception:
        tex_alone_us = None

    # launches per step, measured on one more (untimed) device-resident call
    n_launch, launch_names, launch_src = count_kernel_launches(
        lambda: call(luma_d.data_ptr(), est_d.data_ptr()))

    total_cands = cands * world
    value = total_cands / (ms / 1e3)
    e2e = total_cands / (ms_e2e / 1e3)
    frames_total = F * world
    luma_bytes = F * w.width * w.height * bps
    rec_bytes = F * g.cell_count() * 24
    tex_us, tab_us, s1_us, s2_us = phase[0], phase[1], phase[2], phase[3]
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "measured" if "hbm_gbs" in peaks else "fallback"
    tex_gbs = (luma_bytes + rec_bytes) / (tex_us * 1e-6) / 1e9 if tex_us > 0 else None
    # search roofline: integer-ALU issue.  The
    # warp-instruction count per launch comes from the committed ncu capture
    # of this same workload (the walk is frame-independent and warp-uniform,
    # so the count is a property of the workload); time is measured live.
    issue = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "search_issue.json")))
        key = f"cfg{args.config}_mode{args.mode}"
        if key in prof and prof[key].get("kernel_src_sha") != kernel_src_sha():
            issue = {"bound": "alu", "achieved": None, "peak": None, "unit": "Gwarp-inst/s",
                     "frac": None, "traffic": None,
                     "note": "committed ncu instruction count is for an older kernel source"}
        elif key in prof:
            p = prof[key]
            clk = ck.get("sm_mhz") or p.get("sm_mhz_ncu") or 1965.0
            sms = torch.cuda.get_device_properties(local).multi_processor_count
            peak = sms * 4 * clk * 1e6 / 1e9  # G warp-instr / s at the measured clock
            # dominant kernel: the step-1 trace walk (every candidate's time);
            # the step-1 phase is that launch plus its finalize (~15 us)
            ach = p["warp_inst_step1"] / (s1_us * 1e-6) / 1e9
            issue = {"bound": "alu",
                     "kernel": "k_trace_walk<FPW> (exhaustive step 1: the candidate-trace "
                               "interpreter, trace.cu)",
                     "achieved": round(ach, 2), "peak": round(peak, 2),
                     "unit": "Gwarp-inst/s", "frac": round(ach / peak, 4),
                     "traffic": p.get("dram_bytes_per_launch"),
                     "ncu_issue_active_pct": p.get("issue_active_pct"),
                     "source": "instructions: profiles/search_issue.json (ncu); time: live CUDA events"}
    except Exception:
        pass
    if issue is None:
        issue = {"bound": "alu", "achieved": None, "peak": None, "unit": "Gwarp-inst/s",
                 "frac": None, "traffic": None, "note": "no ncu instruction count committed yet"}
    alone_gbs = (luma_bytes + rec_bytes) / (tex_alone_us * 1e-6) / 1e9 if tex_alone_us else None
    tex_roof = {"bound": "hbm", "kernel": "k_texture_vec (K1), timed alone through "
                                          "sc_texture_moments (device pointers, 531 MB > L2)",
                "achieved": round(alone_gbs, 1) if alone_gbs else None,
                "peak": hbm_peak, "unit": "GB/s",
                "frac": round(alone_gbs / hbm_peak, 4) if alone_gbs else None,
                "traffic": None, "peak_source": hbm_src + " (burst: kernel timed alone)",
                "algorithmic_bytes_per_launch": luma_bytes + rec_bytes,
                "launch_us": round(tex_alone_us, 2) if tex_alone_us else None,
                "in_pipeline": {"launch_us": round(tex_us, 2),
                                "achieved": round(tex_gbs, 1) if tex_gbs else None,
                                "frac": round(tex_gbs / hbm_peak, 4) if tex_gbs else None,
                                "note": "on the low-priority side stream, beside the time "
                                        "tables and the step-1 walk of the main stream"}}
    try:
        tp = json.load(open(os.path.join(ROOT, "profiles", "texture_traffic.json")))
        tex_roof["traffic"] = tp.get(f"cfg{args.config}")
    except Exception:
        pass

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64/f64",
        "data": DATA, "config": workload_config(w, counts),
        "parallelism": f"frames sharded, {world} rank(s)",
        "search_mode": "exhaustive" if args.mode == 0 else "pruned",
        "value_definition": VALUE_DEF,
        "frames_per_s": frames_total / (ms / 1e3),
        "candidates_scored_by_the_walks_per_s": walked * world / (ms / 1e3),
        "frames_per_s_e2e": frames_total / (ms_e2e / 1e3),
        "texture_gbs": alone_gbs if alone_gbs else tex_gbs,
        "texture_gbs_in_pipeline": tex_gbs,
        "phase_us": {"texture_k1": round(tex_us, 2), "tables_k2k3": round(tab_us, 2),
                     "step1": round(s1_us, 2), "step2": round(s2_us, 2),
                     "call": round(phase[4], 2), "time_tables_main": round(phase[5], 2),
                     "moment_tables_side": round(phase[6], 2),
                     "postcheck_and_copies": round(phase[7], 2)},
        "roofline": issue,
        "roofline_texture": tex_roof,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": luma_bytes + F * g.cell_count() * 8,
                "d2h_bytes_per_step": 2 * 32 * ((F + 31) // 32) * 168, "ms_per_step": ms_e2e},
        # kernels per step counted from the CUDA activity trace of one extra
        # untimed call (every kernel is the library's own or a CUB kernel
        # instantiated inside it), times the timed steps
        # kernels launched inside the timed region: the library's own count
        # (every launch goes through its SCB_LAUNCH macro; graph replays add
        # their captured kernels); beside it the CUDA activity trace of one
        # extra untimed call, when CUPTI delivers one
        "gpu_launches": launches_timed,
        "gpu_launches_source": "sc_kernel_launches() delta over the timed region",
        "gpu_launches_per_step_traced": launch_names or None,
        "gpu_launches_traced_total": (args.steps * n_launch) if n_launch else None,
        "gpu_launches_trace_source": launch_src,
        "clocks": ck,
    }
    if rank == 0 and world == 1 and not args.no_extra and args.mode == 0:
        out["pruned"] = pruned_extras(part, stream, args, w, luma_d, est_d)
        out["step2_lambda"] = lambda_extras(part, stream, w, luma_d, est_d)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_sample(w, threads=os.cpu_count() or 1)
    if rank == 0:
        print(json.dumps(out), flush=True)
    part.close()
    if world > 1:
        dist.destroy_process_group()


def run_candidates(args):
    """--shard candidates: every rank holds the SAME frames and the library
    shards each frame's candidate space over the ranks with its own exchange
    (sc_comm_init_nccl: NCCL over NVLink; the gloo test backend uses the host
    callback transport): after step 1 the global t_min (all-reduce min) sets
    step 2's budget, pruned shards share their seed incumbents, and the shard
    bests are all-gathered and merged inside the call, so every rank returns
    the global result.  Total work is fixed as N grows: strong scaling.  One
    step = one sc_partition_frames call (K1 + tables + both steps + the
    exchanges), timed with CUDA events between barriers, max over ranks."""
    import ctypes as C

    import torch
    import torch.distributed as dist
    from paper_2012_14792_b200 import Partitioner, lib
    from paper_2012_14792_b200._abi import SearchResult, check
    from paper_2012_14792_b200 import workloads as wl
    from paper_2012_14792_b200.partitioner import comm_unique_id

    rank, world, local = dist_env()
    backend = os.environ.get("SLICECRAFT_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    w = wl.WORKLOADS[args.config]
    F, g, bps = w.frames, w.grid(), w.bps
    cfg = w.cfg(mode=args.mode)
    luma_h, est_h = make_inputs(w, 0, F)  # the same frames on every rank
    luma_d, est_d = luma_h.cuda(), est_h.cuda()
    part = Partitioner(local)
    stream = torch.cuda.current_stream()
    check(lib().sc_ctx_set_stream(part._h, C.c_void_p(stream.cuda_stream)))
    if world > 1:
        if backend == "nccl":
            box = [comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(box, src=0)
            part.comm_init_nccl(rank, world, box[0])
        else:
            def gather(blob: bytes) -> bytes:
                t = torch.frombuffer(bytearray(blob), dtype=torch.uint8)
                out = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(out, t)
                return b"".join(x.numpy().tobytes() for x in out)
            part.comm_init_callback(rank, world, gather)
    gc, cc = g.c(), cfg.c()
    pitch, fstride = w.width * bps, w.width * w.height * bps
    res = (SearchResult * F)()

    def step():
        check(lib().sc_partition_frames(part._h, C.byref(gc), C.byref(cc),
                                        C.c_void_p(luma_d.data_ptr()), bps, pitch, fstride,
                                        C.c_void_p(est_d.data_ptr()), F, None,
                                        C.cast(res, C.c_void_p)))

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 1)):
        step()
    c12 = [((r.candidates_step1 | (r.candidates_step1_hi << 64)),
            (r.candidates_step2 | (r.candidates_step2_hi << 64))) for r in res]
    cands = sum(a + b for a, b in c12)
    digest = hash(tuple((r.t_best_us, r.sse_best) for r in res))
    clocks = Clocks(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    out = {
        "metric": METRIC, "value": cands / (ms / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64/f64", "data": DATA, "config": workload_config(w, sorted(set(c12))),
        "parallelism": f"candidate space sharded over {world} rank(s), the library's own "
                       "exchange (t_min all-reduce, shard bests all-gathered and merged)",
        "search_mode": "pruned" if args.mode else "exhaustive",
        "frames_per_s": F / (ms / 1e3),
        "result_digest": digest,
        "clocks": ck,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    part.close()
    if world > 1:
        dist.destroy_process_group()


def lambda_extras(part, stream, w, luma_d, est_d):
    """Step 2 where it matters: the headline workload at lambda
    0.1 and 0.3 and the covering family at lambda 0.3, in the
    exhaustive mode -- device time per phase, the step-2 leaves actually
    scored, and the whole step."""
    import ctypes as C

    import torch
    from paper_2012_14792_b200 import lib
    from paper_2012_14792_b200._abi import SearchResult, check
    F, g, bps = w.frames, w.grid(), w.bps
    res = (SearchResult * F)()
    tim = (C.c_double * 8)()
    out = {}
    for lam, cov in [(0.1, 0), (0.3, 0), (0.3, 1)]:
        cc = w.cfg(mode=0, lambda_=lam, coverage=cov).c()
        gc = g.c()

        def call():
            check(lib().sc_partition_frames(part._h, C.byref(gc), C.byref(cc),
                                            C.c_void_p(luma_d.data_ptr()), bps, w.width * bps,
                                            w.width * w.height * bps, C.c_void_p(est_d.data_ptr()),
                                            F, None, C.cast(res, C.c_void_p)))
            check(lib().sc_ctx_timings_ex(part._h, 8, tim))
            return np.array([tim[i] for i in range(8)])
        for _ in range(2):
            call()
        steps = 5
        ph = np.zeros(8)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            ph += call()
        e1.record(stream)
        torch.cuda.synchronize()
        ph /= steps
        ms = e0.elapsed_time(e1) / steps
        c1 = sum(r.candidates_step1 for r in res)
        c2 = sum(r.candidates_step2 for r in res)
        out[f"lambda{lam}_{'covering' if cov else 'reference'}"] = {
            "ms_per_step": ms, "step1_us": round(ph[2], 2), "step2_us": round(ph[3], 2),
            "candidates_per_frame_step": [c1 // F, c2 // F],
            "step2_leaves_scored_per_frame": sum(r.leaves_scored_step2 for r in res) // F,
            "candidates_resolved_per_s": (c1 + c2) / (ms / 1e3)}
    return out


def pruned_extras(part, stream, args, w3, luma3_d, est3_d):
    """The exact pruned mode (identical results and counters)
    on the headline workload and on configs 4 and 5, whose candidate spaces
    (5.4e12 and 6.1e29 per step per frame) no exhaustive walk can cover.
    Reported beside the headline, which stays the every-candidate-scored
    exhaustive walk."""
    import ctypes as C

    import torch
    from paper_2012_14792_b200 import lib
    from paper_2012_14792_b200._abi import SearchResult, check
    from paper_2012_14792_b200 import workloads as wl
    out = {}
    for ci in (3, 4, 5):
        w = wl.WORKLOADS[ci]
        if ci == 3:
            luma_d, est_d = luma3_d, est3_d
        else:
            lh, eh = make_inputs(w, 0, w.frames, pinned=False)
            luma_d, est_d = lh.cuda(), eh.cuda()
        F, g, bps = w.frames, w.grid(), w.bps
        gc, cc = g.c(), w.cfg(mode=1).c()
        res = (SearchResult * F)()

        def call():
            check(lib().sc_partition_frames(part._h, C.byref(gc), C.byref(cc),
                                            C.c_void_p(luma_d.data_ptr()), bps, w.width * bps,
                                            w.width * w.height * bps, C.c_void_p(est_d.data_ptr()),
                                            F, None, C.cast(res, C.c_void_p)))
        for _ in range(2):
            call()
        steps = 5
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            call()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        cnt = sum((r.candidates_step1 | (r.candidates_step1_hi << 64)) +
                  (r.candidates_step2 | (r.candidates_step2_hi << 64)) for r in res)
        scored = sum(r.leaves_scored_step1 + r.leaves_scored_step2 for r in res)
        out[w.name] = {"ms_per_step": ms, "frames": F, "frames_per_s": F / (ms / 1e3),
                       "candidates_resolved_per_s": float(cnt) / (ms / 1e3),
                       "leaves_scored_per_step": scored,
                       "note": "exact branch-and-bound: every candidate resolved (counted by the "
                               "exact DP), only leaves_scored actually evaluated"}
        if ci != 3:
            del luma_d, est_d
    return out


# ---- reference (CPU) arm ------------------------------------------------------------
def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_frames(w, threads, steps, warmup):
    """The unmodified reference CPU path (oracle/_ref: ctu_stats +
    two_step_partition, search.cpp:407-434, the FULL enumeration of the
    workload's family -- nothing capped) on whole frames of the workload, one
    frame per task on a pool of `threads` host threads (the reference's own
    `workers` threads are slower than one frame per thread).
    `warmup` frames run first, untimed; then `steps` frames are timed
    together (wall clock): a step is one frame.  Falls back to the C oracle
    port where oracle/_ref was not built."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle.oracle import Oracle, Ref
    from paper_2012_14792_b200 import workloads as wl
    kind = "reference"
    try:
        R = Ref()
    except Exception:
        R, kind = None, "port"
    O = Oracle()
    n_pocs = min(w.frames, max(steps + warmup, 1))
    # inputs from the shared generator only: this arm never loads the product
    # library (the reference estimates from the raw history itself)
    maps, hp, ht = wl.history_maps(w, frames=n_pocs)
    luma = wl.synth_luma(w, frames=n_pocs)
    frame_bytes = w.width * w.height * w.bps

    def est_port(p):  # estimate_ctu_times for the port fallback (cost.cpp:66-95)
        same = [i for i in range(p) if ht[i] == ht[p]]
        return maps[same[-1] if same else p - 1]

    def one(k):
        i = k % n_pocs
        p = i + 1  # POC p, estimated from POCs 0..p-1 (workloads.cost_trace)
        t0 = time.perf_counter()
        if R is not None:
            _, rec = R.ctu_stats(luma[i].astype(np.uint16), w.bit_depth, w.ctu)
            t1 = time.perf_counter()
            st, o = R.two_step(w.width, w.height, w.ctu, 16, maps[:p], hp[:p], ht[:p], rec, p,
                               w.n_slices, 0.0, 3.0, 0, w.max_tile_cols)
        else:
            rec = O.ctu_stats(luma[i], w.ctu)
            t1 = time.perf_counter()
            st, o = O.search(w.width, w.height, w.ctu, est_port(p), rec, w.n_slices, 0.0, 3.0,
                             w.max_tile_cols, 0, 3)
        assert st == 0
        return o.candidates_step1, o.candidates_step2, t1 - t0, time.perf_counter() - t1

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, range(warmup)))
        t0 = time.perf_counter()
        res = list(ex.map(one, range(warmup, warmup + steps)))
        wall = time.perf_counter() - t0
        # ctu_stats alone, one frame per thread, all threads at once
        # (texture.cpp:145-169 is single-threaded by design)
        def tex(k):
            a = time.perf_counter()
            if R is not None:
                R.ctu_stats(luma[k % n_pocs].astype(np.uint16), w.bit_depth, w.ctu)
            else:
                O.ctu_stats(luma[k % n_pocs], w.ctu)
            return time.perf_counter() - a
        t1 = time.perf_counter()
        tex_t = list(ex.map(tex, range(threads)))
        tex_wall = time.perf_counter() - t1
    cands = sum(a + b for a, b, _, _ in res)
    counts = sorted({(a, b) for a, b, _, _ in res})
    per_thread_tex = frame_bytes / float(np.mean([r[2] for r in res]))
    # steady-state rate of the host: every thread busy with a frame.  When the
    # frames do not divide into full waves the wall clock also holds a tail
    # with idle threads, so the rate is taken over the frames' own times (the
    # tail frames run with less contention: this favours the reference).
    busy = min(threads, steps)
    frame_s = sum(r[2] + r[3] for r in res)
    return {"kind": kind, "cands": cands, "wall": wall, "counts": counts,
            "value": busy * cands / frame_s, "wall_value": cands / wall,
            "mean_frame_s": frame_s / max(len(res), 1), "threads_busy": busy,
            "ctu_stats": {"gbs_per_thread": per_thread_tex / 1e9,
                          "gbs_all_threads": threads * frame_bytes / tex_wall / 1e9,
                          "threads": threads, "frame_bytes": frame_bytes,
                          "per_thread_spread_s": [round(min(tex_t), 4), round(max(tex_t), 4)]},
            "frames": steps}


def cpu_baseline_sample(w, threads):
    """cpu_baseline of the GPU line: one wave of whole frames of the workload
    (one per host thread) through the unmodified reference."""
    r = reference_frames(w, threads, steps=threads, warmup=0)
    return {"value": r["value"], "unit": UNIT, "cores": threads, "kind": r["kind"],
            "sample": f"{w.name}: ctu_stats + two_step_partition (full enumeration, "
                      f"{r['counts'][0][0]:,} + {r['counts'][0][1]:,} candidates per frame) on "
                      f"{threads} whole frame(s), one per host thread "
                      f"({r['mean_frame_s']:.1f} s per frame, {r['wall']:.1f} s wall)",
            "wall_value": r["wall_value"], "cpu_model": cpu_model(), "ctu_stats": r["ctu_stats"]}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2012_14792_b200 import workloads as wl
    w = wl.WORKLOADS[args.config]
    threads = os.cpu_count() or 1
    r = reference_frames(w, threads, steps=args.steps, warmup=args.warmup)
    v = r["value"]
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup,
           "ms_per_step": 1e3 * r["mean_frame_s"] / max(r["threads_busy"], 1),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64/f64",
           "data": DATA, "config": workload_config(w, r["counts"]),
           "parallelism": f"{threads} host threads, one whole frame per thread",
           "value_definition": VALUE_DEF,
           "impl": "reference",
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": r["kind"],
                            "sample": f"{args.steps} whole frames of {w.name} (a step is one "
                                      f"frame: ctu_stats + two_step_partition, full "
                                      f"enumeration), {args.warmup} warm-up frames first, "
                                      f"{threads} frames in flight; value = {r['threads_busy']} "
                                      f"busy threads x candidates / the frames' own times "
                                      f"({r['mean_frame_s']:.1f} s per frame)",
                            "wall_value": r["wall_value"],
                            "cpu_model": cpu_model(), "ctu_stats": r["ctu_stats"]},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--mode", type=int, default=0, choices=[0, 1],
                    help="0 exhaustive (every candidate scored), 1 exact branch-and-bound")
    ap.add_argument("--lambda", dest="lam", type=float, default=None,
                    help="profiling only: override the workload's lambda (0)")
    ap.add_argument("--coverage", type=int, default=None, choices=[0, 1],
                    help="profiling only: 1 = the covering family (SPEC.md:254)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the pruned-mode extras")
    ap.add_argument("--shard", default="frames", choices=["frames", "candidates"],
                    help="frames: each rank its own batch (weak scaling); candidates: the "
                         "ranks split each frame's candidate space (strong scaling)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.shard == "candidates":
        run_candidates(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
