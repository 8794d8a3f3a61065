#!/usr/bin/env python
"""Benchmark of the SparseTem Diff Computation hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

Workload (default): cfg5 = BASELINE.json configs[4], the largest config that
fits one GPU -- the EfficientDet-D0 (EfficientNet-B0) backbone on a job of 64
chunks x 16 frames of synthetic 1080p video, with online threshold
adjustment.  The metric names no config, so the N=1 line is the largest one.
One step = one SparseBatch pass (all §8(a) rows: reference-frame dense pass,
Subtraction, masks, compaction, sparse conv, non-linear correction,
truncation, Accumulation, per-site statistics, the controller's all-gather
and update) over one fixed group of 8 chunks; the job is 8 such groups and
step s processes group s mod 8 (reading R15).

Thresholds: the controller (BST) is run UNTIMED on the job's
steps until every site is frozen (in band or at resolution); the timed steps
then run with those thresholds (the controller still observes every step --
the counts copy, the all-gather, the host update are inside the timed region
-- but a frozen BST does not move).  Per-site thresholds and sparsity are
printed.

value  = diff frames / s of the whole job (all ranks), inputs resident in
         HBM (uint8 frames, v/255 in-kernel, R20), L2 flushed between timed
         steps (untimed 256 MiB write), CUDA events on the launch stream, max
         over ranks.
e2e    = the same metric through the C ABI with pinned HOST buffers: H2D of
         every step's frames and D2H of every step's dense tap outputs (all
         taps) inside one timed region, copies pipelined on two copy streams.
roofline = the dominant kernel class (per-launch CUDA events on the library's
         launch stream, a separate profiled pass), algorithmic bytes or flops
         per launch / mean launch time vs MEASURED_PEAKS.json (the burst
         tensor peak when the sampled SM clock sat at max, else the sustained
         one; HBM: the measured copy bandwidth); traffic = ncu dram bytes per
         launch from profiles/ncu_summary.json when it was captured on this
         same command, else null.
cpu_baseline = the oracle (test infrastructure) on a bounded sample.
Multi-GPU (torchrun): rank r of G processes chunks r, r+G, ... of each group
(reading R15), so the job and every output are the same for every G: strong
scaling of a fixed job.  The only collective is the all-gather of the per-site
int64 counts.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "diff-frame frames/sec (SparseBatch Diff Computation step)"
UNIT = "diff-frames/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--policy", default=None, choices=[None, "fixed", "bst", "ibst"],
                    help="threshold policy (default: the config's; bst/ibst are calibrated untimed, then frozen)")
    ap.add_argument("--live", action="store_true", help="keep IBST live in the timed region (no freeze)")
    ap.add_argument("--precision", default="bf16", choices=["fp32", "bf16"],
                    help="fp32: exact CUDA-core path; bf16: tcgen05 tensor-core convs (R22-BF16)")
    ap.add_argument("--groups", type=int, default=None, help="distinct chunk groups resident (default: the job's)")
    ap.add_argument("--no-dense", action="store_true", help="skip the own-dense-path reference timing")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-fp32", action="store_true", help="skip the FP32-mode context timing")
    ap.add_argument("--headroom", type=float, default=1.25,
                    help="row capacity = headroom x the largest row count seen in the untimed steps (a9); 0 = keep "
                         "the all-active bound")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event reasons sampled DURING the timed region
    (B200_PROFILING.md): NVML polled from a thread every ~2 ms, nvidia-smi
    -lms as the fallback."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop_flag = threading.Event()

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.gpu)
            bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            self.nvml = N

            def poll():
                while not self.stop_flag.is_set():
                    try:
                        sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                        rs = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(sm), float(mx), [bool(rs & b_) for b_ in bits]))
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu),
                                          "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                                          "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                                          "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

            def read():
                for line in self.proc.stdout:
                    r = [x.strip() for x in line.split(",")]
                    if len(r) >= 7 and r[0].replace(".", "").isdigit():
                        self.rows.append((float(r[0]), float(r[1]), [x.lower() == "active" for x in r[3:7]]))
            self.t = threading.Thread(target=read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:   # sampler live before the timed region
                time.sleep(0.01)
            self.rows.clear()
        except Exception:
            self.proc = None

    def stop(self):
        if self.nvml is not None:
            self.stop_flag.set()
            self.t.join(timeout=2)
        elif self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)
        else:
            return None
        rows = list(self.rows)
        sm = [r[0] for r in rows]
        reasons = sorted({self.NAMES[k] for r in rows for k in range(4) if r[2][k]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(r[1] for r in rows) if rows else None,
                "reasons": reasons, "samples": len(sm), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    # B200_PROFILING.md fallback figures
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_class, cid, precision):
    """dram bytes per launch of a kernel class from a committed ncu --set full
    capture of THIS bench command (profiles/ncu_summary.json records the
    config and precision it was captured on), else None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        k = d.get("kernels", {}).get(kernel_class, {})
        if k.get("config") != cid or k.get("precision", "bf16") != precision:
            return None
        return k.get("dram_bytes_per_launch")
    except Exception:
        return None


def ncu_issue(kernel_class, cid):
    """Duration-weighted warp-instructions issued per scheduler cycle (of 1.0)
    of the class in the same committed capture, or None: an HBM fraction far
    below 1 with traffic == algorithmic bytes and issue near 1 says the
    kernel is instruction-issue bound, not memory bound."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            k = json.load(f).get("kernels", {}).get(kernel_class, {})
        return k.get("issued_warp_per_scheduler_mean") if k.get("config") == cid else None
    except Exception:
        return None


def gen_chunks(cfg, ids, L):
    """uint8 [len(ids)][L][H][W][C] of the config's chunks (seed per chunk),
    generated in worker processes (the generator is numpy, ~0.1 s per 1080p
    frame)."""
    import concurrent.futures as cf
    import multiprocessing as mpc
    args = [(cfg.video_seed(c), L, cfg.h, cfg.w, cfg.c) for c in ids]
    if len(ids) <= 2:
        return np.stack([W.gen_chunk(*a, **cfg.video) for a in args])
    nw = max(1, min(len(ids), (os.cpu_count() or 2) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))))
    with cf.ProcessPoolExecutor(nw, mp_context=mpc.get_context("spawn")) as ex:
        out = list(ex.map(_gen_one, [(a, cfg.video) for a in args]))
    return np.stack(out)


def _gen_one(a):
    (seed, L, h, w, c), video = a
    return W.gen_chunk(seed, L, h, w, c, **video)


# -------------------------------------------------------------- reference
def ref_sample_frames(cfg):
    """Frames per chunk of the oracle's bounded sample: small configs run
    whole chunks; 1080p / 720p chunks run the reference frame + 3 diff frames."""
    return cfg.L if cfg.h * cfg.w <= 512 * 512 else min(cfg.L, 4)


def run_reference(args, cfg):
    """--impl reference: the oracle (as it stands) on the host cores; each
    step a bounded sample of the same workload (1 chunk)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    net = cfg.build_net()
    Ls = ref_sample_frames(cfg)
    fr = W.to_float(W.gen_chunk(cfg.video_seed(0), Ls, cfg.h, cfg.w, cfg.c, **cfg.video))
    th = cfg.theta_fixed
    oracle.build()
    for _ in range(max(args.warmup, 0)):
        oracle.run_chunk(net, fr, th, want_masks=False)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.run_chunk(net, fr, th, want_masks=False)
    dt = time.perf_counter() - t0
    v = args.steps * (Ls - 1) / dt
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    sample = f"1 chunk x {Ls} frames (reference + {Ls - 1} diff) of cfg{cfg.cid} per step, theta {th} at every site"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"cfg{cfg.cid}: {cfg.note}", "chunks_per_step": 1, "frames_per_chunk": Ls,
                       "sample": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def cpu_baseline(cfg):
    import oracle
    oracle.build()
    net = cfg.build_net()
    Ls = ref_sample_frames(cfg)
    fr = W.to_float(W.gen_chunk(cfg.video_seed(0), Ls, cfg.h, cfg.w, cfg.c, **cfg.video))
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.run_chunk(net, fr, cfg.theta_fixed, want_masks=False)
        reps += 1
        if time.perf_counter() - t0 > 10.0 or reps >= 8:
            break
    dt = time.perf_counter() - t0
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": reps * (Ls - 1) / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{reps} x (1 chunk x {Ls} frames) of cfg{cfg.cid}, theta {cfg.theta_fixed}, {dt:.1f} s"}


# -------------------------------------------------------------------- ours
def main():
    args = parse()
    cfg = W.get_config(args.config)
    if args.impl == "reference":
        return run_reference(args, cfg)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    B, L = cfg.chunks_per_step, cfg.L
    if B % world:
        raise SystemExit(f"cfg{cfg.cid}: {B} chunks per step do not divide over {world} GPUs")
    n_groups = max(1, cfg.steps)
    res_groups = min(n_groups, args.groups or n_groups)
    from paper_2410_20790_b200.sharding import shard
    # the rank's chunks of every resident group, generated before CUDA starts
    host = [gen_chunks(cfg, shard(g, B, rank, world), L) for g in range(res_groups)]

    import torch
    import torch.distributed as dist
    from paper_2410_20790_b200 import Encoder, ThresholdController
    from paper_2410_20790_b200.sharding import StatsExchange, StepLoop

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    policy = args.policy or cfg.policy
    Br = B // world
    net = cfg.build_net()
    enc = Encoder(net, max_chunks=Br, max_frames=L, device=local, precision=args.precision)
    ns = enc.n_sites
    frozen_run = policy != "fixed" and not args.live
    ctl = ThresholdController(ns, policy="bst" if frozen_run else policy, T=cfg.T, eps=cfg.eps,
                              theta_fixed=cfg.theta_fixed, cycle=cfg.cycle)
    ex = StatsExchange(ns, device=dev)
    loop = StepLoop(B, n_groups, rank, world, ctl, ex)
    inputs = [torch.from_numpy(np.ascontiguousarray(h)).to(dev) for h in host]
    frame_bytes = inputs[0].numel() * inputs[0].element_size()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def encode_on(x):
        def encode(group, ids, th):
            enc.encode_reference(x(group)[:, 0], stream)
            enc.encode_diff(x(group)[:, 1:], th, stream)
            if policy != "fixed":
                enc.copy_site_counts(ex.local, stream)   # -> the NCCL all-gather
            return None
        return encode

    resident = encode_on(lambda g: inputs[g % res_groups])
    observe = policy != "fixed"
    step_no = 0

    # ---- untimed calibration: BST until every site is frozen
    calib_steps = 0
    if frozen_run:
        while calib_steps < 40:
            loop.run_step(step_no, resident, observe=True)
            step_no += 1
            calib_steps += 1
            if bool(np.all(ctl.state()[3])):
                break
    # ---- row capacity from measured occupancy: every
    # resident group once at the all-active bound, then the arena is re-planned
    # at headroom x the largest row count of each delta tensor
    mem_bound = dict(enc.memory_report(), device_bytes=enc.device_bytes())
    if args.headroom >= 1.0:
        for _ in range(res_groups):
            loop.run_step(step_no, resident, observe=observe)
            step_no += 1
        enc.fit_capacity(args.headroom)
    reissued = 0

    def checked_step(fn):
        # a step whose rows exceed a fitted capacity is clamped on the device and
        # flagged: re-plan from the counts it saw and run it again
        nonlocal reissued
        while True:
            fn()
            if enc.step_ok():
                return
            reissued += 1
            enc.fit_capacity(args.headroom)

    # ---- warm-up; every resident group twice (the library captures a CUDA
    # graph of the step on the second sight of an input buffer)
    for _ in range(args.warmup + 2 * res_groups):
        checked_step(lambda: loop.run_step(step_no, resident, observe=observe))
        step_no += 1
    torch.cuda.synchronize(dev)
    launches_per_step = enc.last_launch_count()
    theta = [float(v) for v in ctl.thresholds()]

    # ---- timed region: K steps, L2 flushed between steps (untimed)
    clk = ClockSampler(local)
    clk.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    total_ms = 0.0
    k = 0
    while k < args.steps:
        flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        loop.run_step(step_no, resident, observe=observe)
        e1.record(stream)
        e1.synchronize()
        if not enc.step_ok():   # untimed check: a clamped step is re-planned and timed again
            reissued += 1
            enc.fit_capacity(args.headroom)
            for _ in range(2):   # graph capture on the new arena
                checked_step(lambda: loop.run_step(step_no, resident, observe=False))
            continue
        total_ms += e0.elapsed_time(e1)
        step_no += 1
        k += 1
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    diff_frames = B * (L - 1)          # the whole group, all ranks
    value = diff_frames / (ms_step / 1e3)
    theta_timed = [float(v) for v in ctl.thresholds()]

    # ---- statistics of the last step
    act, sa, sp = enc.get_sparsity()
    sa_all, sp_all = ex.exchange(np.concatenate([sa, sp])) if world > 1 else (sa, sp)
    site_sparsity = [round(1 - a / p, 4) if p else None for a, p in zip(sa_all, sp_all)]
    lc = enc.layer_counts()

    # ---- e2e: pinned host buffers through the C ABI; every step copies its
    # frames H2D and ALL its dense tap outputs D2H, pipelined on two copy
    # streams (H2D of step k+1 and D2H of step k overlap step k+1's kernels)
    n_pin = min(2, res_groups)
    host_in = [torch.from_numpy(host[g]).pin_memory() for g in range(n_pin)]
    taps = enc.taps
    out_shapes = [tuple(enc.outputs(tp).shape) for tp in taps]
    host_out = [[torch.empty(s, dtype=torch.float32).pin_memory() for s in out_shapes] for _ in range(2)]
    dev_in = [torch.empty_like(inputs[0]) for _ in range(2)]
    stage = [[torch.empty(s, dtype=torch.float32, device=dev) for s in out_shapes] for _ in range(2)]
    d2h_bytes = sum(int(np.prod(s)) * 4 for s in out_shapes)
    h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    buffered = encode_on(lambda g: dev_in[cur_buf[0]])
    cur_buf = [0]
    for j in range(2):   # graph capture of both device input buffers (untimed)
        cur_buf[0] = j
        for _ in range(2):
            dev_in[j].copy_(host_in[0], non_blocking=True)
            loop.run_step(step_no, buffered, observe=observe)
    torch.cuda.synchronize(dev)
    e2e_steps = max(3, min(args.steps, 10))
    ev = lambda: torch.cuda.Event()  # noqa: E731
    h2d_ev, used_ev, staged_ev, d2h_ev = ([ev() for _ in range(e2e_steps)] for _ in range(4))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def issue_h2d(k):
        if k >= 2:
            h2d_s.wait_event(used_ev[k - 2])   # step k-2 has consumed dev_in[k % 2]
        with torch.cuda.stream(h2d_s):
            dev_in[k % 2].copy_(host_in[k % n_pin], non_blocking=True)
        h2d_ev[k].record(h2d_s)

    if world > 1:
        dist.barrier()
    e0.record(stream)
    h2d_s.wait_stream(stream)
    d2h_s.wait_stream(stream)
    issue_h2d(0)
    for k in range(e2e_steps):
        if k + 1 < e2e_steps:
            issue_h2d(k + 1)
        stream.wait_event(h2d_ev[k])
        flush.fill_(float(k))
        cur_buf[0] = k % 2
        loop.run_step(step_no, buffered, observe=observe)
        step_no += 1
        used_ev[k].record(stream)
        if k >= 2:
            stream.wait_event(d2h_ev[k - 2])   # stage[k % 2] drained to the host
        for j, tp in enumerate(taps):
            stage[k % 2][j].copy_(enc.outputs(tp), non_blocking=True)
        staged_ev[k].record(stream)
        d2h_s.wait_event(staged_ev[k])
        with torch.cuda.stream(d2h_s):
            for j in range(len(taps)):
                host_out[k % 2][j].copy_(stage[k % 2][j], non_blocking=True)
        d2h_ev[k].record(d2h_s)
    stream.wait_stream(d2h_s)
    e1.record(stream)
    e1.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    for j, tp in enumerate(taps):
        assert torch.equal(host_out[(e2e_steps - 1) % 2][j], enc.outputs(tp).cpu()), "e2e output landed on the host"
    te = torch.tensor([e2e_ms / e2e_steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = diff_frames / (float(te.item()) / 1e3)
    del host_in, host_out, stage, dev_in

    # ---- roofline of the dominant kernel (separate profiled pass, same steps)
    enc.set_profiling(True)
    enc.kernel_times(reset=True)
    for k in range(args.steps):
        flush.fill_(float(k))
        loop.run_step(step_no, resident, observe=observe)
        step_no += 1
        enc.kernel_times(reset=False)
    kt = enc.kernel_times(reset=True)
    enc.set_profiling(False)
    kt.pop("prof_stats", None)   # roofline-only statistics launched by the profiled pass, not part of a step
    step_kernel_ms = sum(v["ms"] for v in kt.values()) / args.steps
    peaks, peak_src = measured_peaks()
    at_max = bool(clocks and clocks.get("sm_mhz") and clocks.get("sm_max_mhz")
                  and clocks["sm_mhz"] >= 0.97 * clocks["sm_max_mhz"])
    tc_key = "bf16_tflops" if (at_max or "bf16_tflops_sustained" not in peaks) else "bf16_tflops_sustained"
    p_tc = float(peaks.get(tc_key, 1590.0))                      # TF/s, one denominator everywhere
    p_hbm = float(peaks["hbm_gbs"])                                # GB/s
    p_f32 = 148 * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12   # TF/s, derived
    kroof = {}
    for k, v in kt.items():
        if not v["launches"] or v["ms"] <= 0:
            continue
        s = v["ms"] / 1e3
        if v["flops"] > 0 and k.startswith("conv_tc"):
            tf = v["flops"] / s / 1e12
            kroof[k] = {"TFLOP/s": round(tf, 1), "frac": round(tf / p_tc, 3), "GB/s": round(v["bytes"] / s / 1e9, 1),
                        "hbm_frac": round(v["bytes"] / s / 1e9 / p_hbm, 3)}
        elif v["bytes"] > 0:
            gb = v["bytes"] / s / 1e9
            kroof[k] = {"GB/s": round(gb, 1), "frac": round(gb / p_hbm, 3)}
    # whole-step roofline: T_roof = sum over kernel classes
    # of max(algorithmic bytes / BW, algorithmic flops / P_class), measured counts
    t_roof = 0.0
    for k, v in kt.items():
        p = p_tc if k.startswith("conv_tc") else p_f32
        t_roof += max(v["bytes"] / (p_hbm * 1e9), v["flops"] / (p * 1e12))
    t_roof_ms = t_roof * 1e3 / args.steps
    dom = max(kt, key=lambda k: kt[k]["ms"])
    d = kt[dom]
    nl = max(d["launches"], 1)
    share = d["ms"] / args.steps / step_kernel_ms
    if d["flops"] > 0 and dom.startswith("conv_tc") and d["flops"] / (p_tc * 1e12) >= d["bytes"] / (p_hbm * 1e9):
        ach = d["flops"] / nl / (d["ms"] / nl / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": ach, "peak": p_tc, "unit": "TFLOP/s", "frac": ach / p_tc,
                "peak_source": f"{peak_src} {tc_key}" + (" (SM clock at max)" if at_max else "")}
    elif d["flops"] > 0 and dom.startswith("conv") and not dom.startswith("conv_tc") and \
            d["flops"] / (p_f32 * 1e12) >= d["bytes"] / (p_hbm * 1e9):
        ach = d["flops"] / nl / (d["ms"] / nl / 1e3) / 1e12
        roof = {"bound": "alu", "achieved": ach, "peak": p_f32, "unit": "TFLOP/s", "frac": ach / p_f32,
                "peak_source": f"derived: 148 SM x 128 FP32 lanes x 2 x {peaks.get('sm_max_mhz', 1965.0)} MHz"}
    else:
        ach = (d["bytes"] / nl) / (d["ms"] / nl / 1e3) / 1e9 if d["bytes"] else None
        roof = {"bound": "hbm", "achieved": ach, "peak": p_hbm, "unit": "GB/s", "frac": (ach / p_hbm) if ach else None,
                "peak_source": f"{peak_src} hbm_gbs"}
    roof.update({"traffic": ncu_traffic(dom, cfg.cid, args.precision), "issue_per_scheduler": ncu_issue(dom, cfg.cid),
                 "kernel": dom,
                 "alg_bytes_per_launch": d["bytes"] / nl, "alg_flops_per_launch": d["flops"] / nl,
                 "launches_per_step": d["launches"] / args.steps, "share_of_step": share})

    # ---- own dense path: every frame of the group as a reference frame, same kernels
    dense = None
    if not args.no_dense:
        denc = Encoder(net, max_chunks=Br * L, max_frames=1, device=local, precision=args.precision)
        xd = inputs[0].reshape(Br * L, cfg.h, cfg.w, cfg.c)
        for _ in range(2):
            denc.encode_reference(xd, stream)
            denc.encode_diff(None, theta_timed, stream)
        torch.cuda.synchronize(dev)
        dms = 0.0
        nd = max(3, min(args.steps, 5))
        for k in range(nd):
            flush.fill_(float(k))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            denc.encode_reference(xd, stream)
            denc.encode_diff(None, theta_timed, stream)
            e1.record(stream)
            e1.synchronize()
            dms += e0.elapsed_time(e1)
        dense_fps = Br * L / (dms / nd / 1e3)
        ref_ms = dms / nd / L   # dense time of the Br reference frames
        dense = {"dense_fps_per_gpu": dense_fps, "speedup_vs_dense": (value / world) / dense_fps,
                 "diff_fps_excl_reference": diff_frames / max((ms_step - ref_ms) / 1e3, 1e-9)}
        del denc

    mem = dict(enc.memory_report(), device_bytes=enc.device_bytes(), headroom=args.headroom,
               reissued_steps=reissued, at_all_active_bound=mem_bound)
    # ---- the bit-exact FP32 mode on the same chunks (context for the BF16 headline)
    fp32_exact = None
    if args.precision == "bf16" and not args.no_fp32:
        del enc
        fenc = Encoder(net, max_chunks=Br, max_frames=L, device=local, precision="fp32")
        fms = 0.0
        for k in range(4):
            flush.fill_(float(k))
            x = inputs[k % res_groups]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fenc.encode_reference(x[:, 0], stream)
            fenc.encode_diff(x[:, 1:], theta_timed, stream)
            e1.record(stream)
            e1.synchronize()
            if k:
                fms += e0.elapsed_time(e1)
        fp32_exact = {"value": diff_frames / (fms / 3 / 1e3) if world == 1 else None, "ms_per_step": fms / 3,
                      "note": "FP32 mode (bit-exact with the oracle), CUDA-core convs, same thresholds"}
        del fenc

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "bf16xbf16->f32",
                "data": "synthetic (seeded video, calibrated random weights R30)",
                "config": {"workload": f"cfg{cfg.cid}: {cfg.note}", "chunks_per_step": B,
                           "chunks_per_step_per_gpu": Br, "job_chunks": B * n_groups,
                           "resident_chunk_groups": res_groups, "frames_per_chunk": L,
                           "frame": [cfg.h, cfg.w, cfg.c], "policy": policy,
                           "thresholds": ("BST calibrated untimed for %d steps, frozen" % calib_steps) if frozen_run
                           else policy,
                           "parallelism": f"chunk-sharded dp{world} (R15 fixed groups)",
                           "l2": "flushed between timed steps (256 MiB write, untimed)",
                           "input_bytes_per_step": frame_bytes * world, "frames": "uint8 (v/255, R20)"},
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": frame_bytes * world,
                        "d2h_bytes_per_step": d2h_bytes * world, "steps": e2e_steps,
                        "pipelined": "H2D of step k+1 and D2H of step k (all taps) on copy streams overlap compute"},
                "gpu_launches": launches_per_step * args.steps,
                "roofline": roof,
                "cpu_baseline": cpu,
                "clocks": clocks,
                "theta": [round(v, 5) for v in theta_timed],
                "site_sparsity": site_sparsity,
                "conv_rows_out": int(sum(lc["rows_out"][i] for i, l in enumerate(net.layers) if l["kind"] == W.CONV)),
                "kernel_ms_per_step": {k: round(v["ms"] / args.steps, 4) for k, v in kt.items() if v["launches"]},
                "kernel_roofline": kroof,
                "peaks": {"tensor_tflops": p_tc, "tensor_key": tc_key, "hbm_gbs": p_hbm,
                          "fp32_tflops_derived": p_f32, "source": peak_src},
                "step_roofline": {"t_roof_ms": t_roof_ms, "t_measured_ms": ms_step, "frac": t_roof_ms / ms_step,
                                  "note": "sum over kernel classes of max(alg bytes / HBM peak, alg flops / class "
                                          "peak); classes without a byte model (scan, counts, dense_misc) count 0"},
                "memory": mem, "fp32_exact": fp32_exact}
        if dense:
            line.update(dense)
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
