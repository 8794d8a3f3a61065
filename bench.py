#!/usr/bin/env python
"""Benchmark of the SparseTem Diff Computation hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One step = one SparseBatch pass (all §8(a) rows: reference-frame dense pass,
Subtraction, masks, compaction, sparse conv, non-linear correction,
truncation, Accumulation, per-site statistics) over one batch of synthetic
chunks: BASELINE.json configs[1] = cfg2, the CRNN VGG-7 conv encoder on
64 chunks x 32 frames of 32x128 grayscale synthetic text video.

value  = diff frames / s of the whole job (all ranks), inputs resident in
         HBM, L2 flushed between timed steps (untimed 256 MiB write), CUDA
         events on the launch stream, max over ranks.
e2e    = the same metric through the C ABI with pinned HOST buffers: H2D of
         every step's frames and D2H of every step's dense tap outputs inside
         one timed region, the copies pipelined against compute on two copy
         streams (a serving loop: step k+1's input upload and step k's result
         download overlap step k+1's kernels).
roofline = dominant kernel class (per-launch CUDA events inside the library,
         a separate profiled pass), algorithmic flops or bytes per launch /
         mean launch time vs the measured / derived peak.
cpu_baseline = the oracle (test infrastructure) on a bounded sample.
Multi-GPU (torchrun): rank r processes its own 64 chunks per step (weak
scaling, chunks are independent); no data-path collective for the
fixed-threshold config; with --policy bst/ibst the per-site counts are
all-gathered over NCCL every step for the controller.
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
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--policy", default=None, choices=[None, "fixed", "bst", "ibst"])
    ap.add_argument("--precision", default="bf16", choices=["fp32", "bf16"],
                    help="fp32: exact CUDA-core path; bf16: tcgen05 tensor-core convs (R22-BF16)")
    ap.add_argument("--no-dense", action="store_true", help="skip the own-dense-path reference timing")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event reasons sampled DURING the timed region
    (B200_PROFILING.md).  NVML polled from a thread every ~2 ms (a cfg2
    timed region is only tens of ms); nvidia-smi -lms as the fallback."""

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
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def ncu_traffic(kernel_class, cid):
    """dram bytes per launch of the dominant kernel from a committed ncu --set
    full capture of this config's bench command (profiles/ncu_summary.json),
    else None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f).get("kernels", {}).get(kernel_class, {})
        return d.get("dram_bytes_per_launch") if d.get("config") == cid else None
    except Exception:
        return None


# -------------------------------------------------------------- reference
def run_reference(args, cfg):
    """--impl reference: the oracle (as it stands) on the host cores, each
    step a bounded sample (1 chunk x L frames) of the same workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    net = cfg.build_net()
    u8 = W.gen_video(1, cfg.L, cfg.h, cfg.w, cfg.c, cfg.video_seed(0), **cfg.video)
    fr = W.to_float(u8)[0]
    th = cfg.theta_fixed
    oracle.build()
    for _ in range(max(args.warmup, 0)):
        oracle.run_chunk(net, fr, th, want_masks=False)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.run_chunk(net, fr, th, want_masks=False)
    dt = time.perf_counter() - t0
    v = args.steps * (cfg.L - 1) / dt
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"cfg{cfg.cid}: {cfg.note}", "chunks_per_step": 1, "frames_per_chunk": cfg.L,
                       "sample": "1 chunk per step"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"1 chunk x {cfg.L} frames of cfg{cfg.cid} per step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def cpu_baseline(cfg):
    import oracle
    oracle.build()
    net = cfg.build_net()
    u8 = W.gen_video(1, cfg.L, cfg.h, cfg.w, cfg.c, cfg.video_seed(0), **cfg.video)
    fr = W.to_float(u8)[0]
    oracle.run_chunk(net, fr[:2], cfg.theta_fixed, want_masks=False)   # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.run_chunk(net, fr, cfg.theta_fixed, want_masks=False)
        reps += 1
        if time.perf_counter() - t0 > 10.0 or reps >= 8:
            break
    dt = time.perf_counter() - t0
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": reps * (cfg.L - 1) / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{reps} x (1 chunk x {cfg.L} frames) of cfg{cfg.cid}, {dt:.1f} s"}


# -------------------------------------------------------------------- ours
def main():
    args = parse()
    cfg = W.get_config(args.config)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist
    from paper_2410_20790_b200 import Encoder, ThresholdController

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    policy = args.policy or cfg.policy
    B, L = cfg.chunks_per_step, cfg.L
    net = cfg.build_net()
    enc = Encoder(net, max_chunks=B, max_frames=L, device=local, precision=args.precision)
    ns = enc.n_sites
    ctl = ThresholdController(ns, policy=policy, T=cfg.T, eps=cfg.eps, theta_fixed=cfg.theta_fixed,
                              cycle=cfg.cycle)

    # inputs: distinct synthetic batches per step (rank r owns global chunks r + world*j)
    from paper_2410_20790_b200.sharding import shard
    n_batches = max(1, min(cfg.steps, 4 if cfg.h * cfg.w <= 512 * 512 else 2))
    batches = []
    for s in range(n_batches):
        u8 = np.stack([W.gen_chunk(cfg.video_seed(cid), L, cfg.h, cfg.w, cfg.c, **cfg.video)
                       for cid in shard(s, B * world, rank, world)])
        # uint8 frames, the camera / decoder format (v / 255 inside the
        # Subtraction kernels, reading R20; bit-identical to fp32 frames)
        batches.append(torch.from_numpy(np.ascontiguousarray(u8)).to(dev))
    frame_bytes = batches[0].numel() * batches[0].element_size()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    from paper_2410_20790_b200.sharding import StatsExchange
    ex = StatsExchange(ns, device=dev)

    def step(x):
        th = ctl.thresholds()
        enc.encode_reference(x[:, 0], stream)
        enc.encode_diff(x[:, 1:], th, stream)
        if policy != "fixed":
            # the only collective: NCCL all-gather of int64 per-site counts
            enc.copy_site_counts(ex.local, stream)
            ctl.observe(*ex.exchange())

    for w in range(args.warmup):
        step(batches[w % n_batches])
    # every input batch seen twice before timing: the library captures a CUDA
    # graph of the step on the second sight of a (frames, shape) key
    for w in range(2 * n_batches):
        step(batches[w % n_batches])
    torch.cuda.synchronize(dev)
    launches_per_step = enc.last_launch_count()

    # ---- timed region: K steps, L2 flushed between steps (untimed)
    clk = ClockSampler(local)
    clk.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    total_ms = 0.0
    for k in range(args.steps):
        flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(batches[k % n_batches])
        e1.record(stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    diff_frames = B * (L - 1) * world
    value = diff_frames / (ms_step / 1e3)

    # ---- statistics of the last step
    act, sa, sp = enc.get_sparsity()
    site_sparsity = [round(1 - a / p, 4) if p else None for a, p in zip(sa, sp)]
    lc = enc.layer_counts()

    # ---- e2e: pinned host buffers through the C ABI.  Every step copies its
    # frames H2D and its dense tap outputs D2H; the copies run on two copy
    # streams, pipelined against the compute stream (H2D of step k+1 and D2H
    # of step k overlap step k+1's kernels; double-buffered device inputs, the
    # outputs staged D2D so the next step may overwrite the Accumulation
    # buffer).  One timed region over all e2e steps, end = last D2H landed.
    host_in = [b.cpu().pin_memory() for b in batches]
    tap = enc.taps[0]
    out_shape = tuple(enc.outputs(tap).shape)
    host_out = [torch.empty(out_shape, dtype=torch.float32).pin_memory() for _ in range(2)]
    dev_in = [torch.empty_like(batches[0]) for _ in range(2)]
    stage = [torch.empty(out_shape, dtype=torch.float32, device=dev) for _ in range(2)]
    h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    for j in range(2):   # graph capture of both input buffers' keys (untimed)
        for _ in range(2):
            dev_in[j].copy_(host_in[0], non_blocking=True)
            step(dev_in[j])
    torch.cuda.synchronize(dev)
    e2e_steps = max(3, min(args.steps, 10))
    ev = lambda: torch.cuda.Event()  # noqa: E731
    h2d_ev, used_ev, staged_ev, d2h_ev = ([ev() for _ in range(e2e_steps)] for _ in range(4))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def issue_h2d(k):
        if k >= 2:
            h2d_s.wait_event(used_ev[k - 2])   # step k-2 has consumed dev_in[k % 2]
        with torch.cuda.stream(h2d_s):
            dev_in[k % 2].copy_(host_in[k % n_batches], non_blocking=True)
        h2d_ev[k].record(h2d_s)

    e0.record(stream)
    h2d_s.wait_stream(stream)
    d2h_s.wait_stream(stream)
    issue_h2d(0)
    for k in range(e2e_steps):
        if k + 1 < e2e_steps:
            issue_h2d(k + 1)
        stream.wait_event(h2d_ev[k])
        flush.fill_(float(k))
        step(dev_in[k % 2])
        used_ev[k].record(stream)
        if k >= 2:
            stream.wait_event(d2h_ev[k - 2])   # stage[k % 2] drained to the host
        stage[k % 2].copy_(enc.outputs(tap), non_blocking=True)
        staged_ev[k].record(stream)
        d2h_s.wait_event(staged_ev[k])
        with torch.cuda.stream(d2h_s):
            host_out[k % 2].copy_(stage[k % 2], non_blocking=True)
        d2h_ev[k].record(d2h_s)
    stream.wait_stream(d2h_s)
    e1.record(stream)
    e1.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    assert torch.equal(host_out[(e2e_steps - 1) % 2], enc.outputs(tap).cpu()), "e2e output landed on the host"
    te = torch.tensor([e2e_ms / e2e_steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = diff_frames / (float(te.item()) / 1e3)

    # ---- roofline of the dominant kernel (separate profiled pass)
    enc.set_profiling(True)
    enc.kernel_times(reset=True)
    for k in range(args.steps):
        flush.fill_(float(k))
        step(batches[k % n_batches])
        enc.kernel_times(reset=False)
    kt = enc.kernel_times(reset=True)
    enc.set_profiling(False)
    kt.pop("prof_stats", None)   # roofline-only statistics launched by the profiled pass, not part of a step
    step_kernel_ms = sum(v["ms"] for v in kt.values()) / args.steps
    dom = max(kt, key=lambda k: kt[k]["ms"])
    peaks, peak_src = measured_peaks()
    # per-class achieved rate vs its roofline (algorithmic bytes / flops)
    kroof = {}
    for k, v in kt.items():
        if not v["launches"] or v["ms"] <= 0:
            continue
        if v["flops"] > 0 and k.startswith("conv_tc"):
            tf = v["flops"] / (v["ms"] / 1e3) / 1e12
            kroof[k] = {"TFLOP/s": round(tf, 1), "frac": round(tf / float(peaks.get("bf16_tflops", 1590.0)), 3),
                        "GB/s": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1)}
        elif v["bytes"] > 0:
            gb = v["bytes"] / (v["ms"] / 1e3) / 1e9
            kroof[k] = {"GB/s": round(gb, 1), "frac": round(gb / float(peaks["hbm_gbs"]), 3)}
    # whole-step roofline: T_roof = sum over kernel classes of
    # max(algorithmic bytes / BW, algorithmic flops / P_class), on the measured counts
    bw = float(peaks["hbm_gbs"]) * 1e9
    p_tc = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1590.0))) * 1e12
    p_f32 = 148 * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    t_roof = 0.0
    for k, v in kt.items():
        p = p_tc if k.startswith("conv_tc") else p_f32
        t_roof += max(v["bytes"] / bw, v["flops"] / p)
    t_roof_ms = t_roof * 1e3 / args.steps
    step_roof = {"t_roof_ms": t_roof_ms, "t_measured_ms": None, "frac": None,
                 "note": "sum over kernel classes of max(alg bytes / HBM peak, alg flops / class peak); "
                         "classes without a byte model (scan, counts, dense_misc) contribute 0"}
    d = kt[dom]
    nl = max(d["launches"], 1)
    if d["flops"] > 0 and dom.startswith("conv_tc"):
        # tcgen05 bf16: measured cuBLAS bf16 peak, sustained figure (kernel timed inside a long step)
        peak_key = "bf16_tflops_sustained" if "bf16_tflops_sustained" in peaks else "bf16_tflops"
        peak = float(peaks.get(peak_key, 1590.0))
        ach = d["flops"] / nl / (d["ms"] / nl / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "traffic": ncu_traffic(dom, cfg.cid), "kernel": dom,
                "peak_source": f"{peak_src} {peak_key}",
                "share_of_step": d["ms"] / args.steps / step_kernel_ms}
    elif d["flops"] > 0 and dom.startswith("conv"):
        # FP32 CUDA-core FFMA: 148 SMs x 128 lanes x 2 flop x max SM clock
        peak = 148 * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
        ach = d["flops"] / nl / (d["ms"] / nl / 1e3) / 1e12
        roof = {"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "traffic": ncu_traffic(dom, cfg.cid), "kernel": dom,
                "peak_source": f"derived: 148 SM x 128 FP32 lanes x 2 x {peaks.get('sm_max_mhz', 1965.0)} MHz",
                "share_of_step": d["ms"] / args.steps / step_kernel_ms}
    else:
        peak = float(peaks["hbm_gbs"])
        ach = (d["bytes"] / nl) / (d["ms"] / nl / 1e3) / 1e9 if d["bytes"] else None
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": (ach / peak) if ach else None, "traffic": ncu_traffic(dom, cfg.cid), "kernel": dom,
                "peak_source": peak_src, "share_of_step": d["ms"] / args.steps / step_kernel_ms}

    # ---- own dense path: every frame as a reference frame, same kernels
    dense = None
    if not args.no_dense:
        denc = Encoder(net, max_chunks=B * L, max_frames=1, device=local, precision=args.precision)
        xd = batches[0].reshape(B * L, cfg.h, cfg.w, cfg.c)
        for _ in range(2):
            denc.encode_reference(xd, stream)
            denc.encode_diff(None, ctl.thresholds(), stream)
        torch.cuda.synchronize(dev)
        dms = 0.0
        nd = max(3, min(args.steps, 5))
        for k in range(nd):
            flush.fill_(float(k))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            denc.encode_reference(xd, stream)
            denc.encode_diff(None, ctl.thresholds(), stream)
            e1.record(stream)
            e1.synchronize()
            dms += e0.elapsed_time(e1)
        dense_fps = B * L / (dms / nd / 1e3)
        ref_ms = dms / nd / L   # dense time of B reference frames
        dense = {"dense_fps_per_gpu": dense_fps, "speedup_vs_dense": (value / world) / dense_fps,
                 "diff_fps_excl_reference": diff_frames / max((ms_step - ref_ms) / 1e3, 1e-9)}
        del denc

    mem = enc.memory_report()
    # ---- the bit-exact FP32 mode on the same batches (context for the BF16 headline)
    fp32_exact = None
    if args.precision == "bf16":
        del enc
        fenc = Encoder(net, max_chunks=B, max_frames=L, device=local, precision="fp32")
        th = ctl.thresholds()
        fms = 0.0
        for k in range(4):
            flush.fill_(float(k))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fenc.encode_reference(batches[k % n_batches][:, 0], stream)
            fenc.encode_diff(batches[k % n_batches][:, 1:], th, stream)
            e1.record(stream)
            e1.synchronize()
            if k:
                fms += e0.elapsed_time(e1)
        fp32_exact = {"value": diff_frames / (fms / 3 / 1e3), "ms_per_step": fms / 3,
                      "note": "FP32 mode (bit-exact with the oracle), CUDA-core convs"}
        enc = fenc

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "bf16xbf16->f32",
                "data": "synthetic",
                "config": {"workload": f"cfg{cfg.cid}: {cfg.note}", "chunks_per_step_per_gpu": B,
                           "frames_per_chunk": L, "frame": [cfg.h, cfg.w, cfg.c], "policy": policy,
                           "theta": [float(x) for x in ctl.thresholds()[:3]] + ["..."],
                           "parallelism": f"chunk-sharded dp{world}", "l2": "flushed between timed steps",
                           "input_bytes_per_step": frame_bytes, "frames": "uint8 (v/255, R20)"},
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": frame_bytes,
                        "d2h_bytes_per_step": int(host_out[0].numel() * 4), "steps": e2e_steps,
                        "pipelined": "H2D of step k+1 and D2H of step k on copy streams overlap compute"},
                "gpu_launches": launches_per_step * args.steps,
                "roofline": roof,
                "cpu_baseline": cpu,
                "clocks": clocks,
                "site_sparsity": site_sparsity,
                "conv_rows_out": int(sum(lc["rows_out"][i] for i, l in enumerate(net.layers) if l["kind"] == W.CONV)),
                "kernel_ms_per_step": {k: round(v["ms"] / args.steps, 4) for k, v in kt.items() if v["launches"]},
                "kernel_roofline": kroof,
                "step_roofline": dict(step_roof, t_measured_ms=ms_step, frac=step_roof["t_roof_ms"] / ms_step),
                "memory": mem, "fp32_exact": fp32_exact}
        if dense:
            line.update(dense)
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
