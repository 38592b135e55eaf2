#!/usr/bin/env python
"""BDIS matching-core throughput on B200 (BASELINE.json metric: 640x480 stereo
pairs/sec, fraction of the memory roofline).

A "step" = one batched run_pipeline (pyramid -> per-level patch solves ->
finest fusion -> confidence filter -> depth) over BATCH pairs of the config-2
workload (seeded config-0 generator pairs, 640x480 uint8 gray, exps 3..1, 8x8
patches at stride 4, variance off). Pairs are independent, so under torchrun
each rank processes its own BATCH pairs (seeds rank*BATCH...), no collective on
the data path ("scaling": "weak"); the only NCCL call is the max-over-ranks
reduction of the timings.

  value   device-resident inputs/outputs, CUDA events on the launch stream
  e2e     the same through the public C ABI with pinned HOST buffers: H2D of
          both views and D2H of the disparity map (NaN = invalid, i.e. the
          validity mask folded in) inside every timed step
  roofline  dominant kernel (the finest-level k_patches launch) from live CUDA
          events; traffic from the committed ncu capture (profiles/)
  cpu_baseline  the reference (oracle/_ref, the unmodified reference sources)
          on this host's cores, bounded sample (rank 0, N=1 only)

--impl reference times the reference CPU implementation itself, all host cores,
same metric/config.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

W, H = 640, 480
HBM_FALLBACK_GBS = 6650.0


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return HBM_FALLBACK_GBS, "fallback"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the reference's own sources, or the C port)

def _cpu_oracle():
    from oracle import pyoracle

    kind = "reference" if pyoracle.available("reference") else "port"
    return pyoracle.load(kind), kind


def cpu_throughput(left, right, cfg, threads, focal=500.0, baseline=5.0):
    """Runs run_pipeline on every pair with `threads` workers (threads=1 each,
    pair-level parallelism, the fair CPU throughput per SURVEY.md 8d).
    Returns (pairs/s over the wall time, per-pair runtime_ms list)."""
    orc, _ = _cpu_oracle()
    grays = [(orc.to_grayscale(left[k])[0], orc.to_grayscale(right[k])[0])
             for k in range(left.shape[0])]
    idx = [0]
    lock = threading.Lock()
    times = []

    def worker():
        while True:
            with lock:
                k = idx[0]
                idx[0] += 1
            if k >= len(grays):
                return
            r = orc.run_pipeline(grays[k][0], grays[k][1], cfg, focal, baseline)
            with lock:
                times.append(r["runtime_ms"])

    ths = [threading.Thread(target=worker) for _ in range(threads)]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - t0
    return len(grays) / wall, times


def oracle_cfg():
    from oracle import pyoracle

    return pyoracle.Config(coarsest_exp=3, finest_exp=1, patch_size=8, overlap=0.5)


def run_reference_arm(args):
    import paper_2205_03133_b200 as P

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = host_cores()
    orc, kind = _cpu_oracle()
    n = max(cores, 1)
    left, right = P.synth_batch(0, n * (args.steps + args.warmup), seed0=0, threads=cores)
    cfg = oracle_cfg()
    total_pairs, total_t = 0, 0.0
    for step in range(args.warmup + args.steps):
        sl = slice(step * n, (step + 1) * n)
        rate, _ = cpu_throughput(left[sl], right[sl], cfg, cores)
        if step >= args.warmup:
            total_pairs += n
            total_t += n / rate
    value = total_pairs / total_t
    sample = (f"{args.steps} steps x {n} config-2 pairs (640x480, seeds 0..), one pair per core "
              f"per step, run_pipeline threads=1")
    line = {
        "impl": "reference", "metric": "640x480 stereo pairs/sec", "value": value,
        "unit": "pairs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config2: 640x480 u8 gray, exps 3..1, s=8 stride 4, var off",
                   "global_batch": n, "parallelism": f"{cores} host threads"},
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU clocks during the timed region

class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, fl in rows for i, v in enumerate(fl)
                          if v.lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in rows])),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# our arm

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2205_03133_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the multi-rank logic on a one-GPU box (not a
    # measurement): PSTEREO_BENCH_BACKEND=gloo and ranks folded onto the GPUs
    backend = os.environ.get("PSTEREO_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local %= max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    B = args.batch
    cfg = P.PipelineConfig.baseline(0)
    from paper_2205_03133_b200.shard import max_over_ranks, weak_shard

    shard = weak_shard(B, rank, world)  # pairs are independent: no exchange
    dev = torch.device("cuda", local)
    # inputs generated in HBM by the device generator:
    # the same bytes as the host generator, without host work or PCIe per rank
    dl, dr = P.synth_batch_gpu(0, shard.count, seed0=shard.start, device=local)
    torch.cuda.synchronize(dev)
    left, right = dl.cpu().numpy(), dr.cpu().numpy()  # host copies: e2e leg, CPU baseline
    # output: the filtered disparity map with NaN at invalid pixels (the
    # reference persists maps the same way with a -1 sentinel, src/io.cpp:297-310);
    # the validity mask is exactly isfinite(disparity)
    disp = torch.empty((B, H, W), dtype=torch.float32, device=dev)
    m = P.Matcher(cfg, W, H, B, device=local)
    # a dedicated stream: our kernels and the timing events must share it
    # (NULL would select the context's own stream, not torch's legacy stream)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    outs = {"disparity": disp.data_ptr()}
    NAN = float("nan")

    def step():
        m.run_device_u8(B, W, H, 1, dl.data_ptr(), dr.data_ptr(), outs, stream=sh,
                        invalid_value=NAN)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    launches_per_step = m.launch_count()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    # per-stage device times from a separate, instrumented pass (the stage
    # events serialise the launches, so they stay out of the timed region)
    m.set_device_chunks(1)  # one launch per stage: per-launch durations for the roofline
    step()  # (re)sizes the working set for the unsplit batch outside the profile
    torch.cuda.synchronize(dev)
    m.set_profiling(True)
    prof_steps = min(args.steps, 10)
    for _ in range(prof_steps):
        step()
    torch.cuda.synchronize(dev)
    stages, calls = m.stage_times()
    m.set_profiling(False)
    # a step may run as several sub-batch calls (PSTEREO_DEVICE_CHUNKS)
    pairs_per_call = B * prof_steps / max(calls, 1)
    ms_max = max_over_ranks(ms, device=dev)
    value = world * B * args.steps / (ms_max / 1e3)

    # ---- e2e through the public ABI with pinned host buffers
    hl = torch.from_numpy(left).pin_memory()
    hr = torch.from_numpy(right).pin_memory()
    hd = torch.empty((B, H, W), dtype=torch.float32).pin_memory()
    houts = {"disparity": hd.data_ptr()}

    def step_e2e():
        # async host outputs: step k+1's uploads and kernels run under step k's
        # downloads; every step still moves its own inputs and result
        m.run_host_u8(B, W, H, 1, hl.data_ptr(), hr.data_ptr(), houts, stream=sh,
                      invalid_value=NAN, async_host=True)

    e2e_steps = 0 if args.no_e2e else max(3, min(args.steps, 20))
    for _ in range(2 if e2e_steps else 0):  # both alternating staging sets allocated
        step_e2e()
    m.wait(sh)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_e2e()
    m.wait(sh)  # every step's download has landed in host memory
    torch.cuda.synchronize(dev)
    e2e_s = time.perf_counter() - t0
    e2e_s = max_over_ranks(e2e_s, device=dev)
    e2e_value = world * B * e2e_steps / e2e_s if e2e_steps else None
    # parity spot check of the e2e output against the device-resident run
    if e2e_steps:
        dc = disp.cpu()
        assert torch.equal(torch.isnan(hd), torch.isnan(dc)), "e2e validity differs"
        assert torch.equal(torch.nan_to_num(hd), torch.nan_to_num(dc)), "e2e output differs"

    # ---- roofline of the dominant kernel: the finest-level k_patches launch
    hbm, peak_kind = peaks()
    dims = P.level_dims(cfg, W, H)
    e_f, w_f, h_f = dims[-1]
    s_, st_ = cfg.patch_size, max(1, int(round(cfg.patch_size * (1 - cfg.overlap))))
    npatch_f = len(_axis(w_f, s_, st_)) * len(_axis(h_f, s_, st_))
    # read the left/right/gradient fp32 planes (12 B/px)
    # and the coarser records (16 B/patch), write the records (32 B/patch)
    alg_bytes = pairs_per_call * (12.0 * w_f * h_f + 48.0 * npatch_f)
    patch_ms = stages.get(f"patches_e{e_f}", 0.0) / max(calls, 1)
    achieved = alg_bytes / (patch_ms / 1e3) / 1e9 if patch_ms > 0 else 0.0
    traffic = None
    fp64 = None
    tj = ROOT / "profiles" / "ncu_traffic.json"
    if tj.exists():
        t = json.loads(tj.read_text())["k_patches_finest"]
        traffic = t["dram_bytes_per_launch"] / t["pairs_in_launch"] * pairs_per_call
        if "fp64_inst_per_launch" in t and patch_ms > 0:
            # the pipes this kernel actually runs on: FP64 (DADD/DMUL/DFMA) and
            # XU (float<->double/int conversions); counts from ncu for the same
            # launch scaled to this batch, time from the live CUDA events; peaks
            # are this box's measured per-SM rates (scripts/microbench.cu:
            # DADD 62.6, F2F 15.5 thread-ops/clk/SM) x 148 SMs x max clock
            sm_hz = 148 * 1965e6
            f_ops = (t["fp64_inst_per_launch"] / t["pairs_in_launch"] * pairs_per_call
                     / (patch_ms / 1e3))
            x_ops = (t["conversion_inst_per_launch"] / t["pairs_in_launch"] * pairs_per_call
                     / (patch_ms / 1e3))
            fp64 = {"unit": "T thread-inst/s",
                    "fp64_achieved": f_ops / 1e12, "fp64_peak": 62.6 * sm_hz / 1e12,
                    "fp64_frac": f_ops / (62.6 * sm_hz),
                    "xu_achieved": x_ops / 1e12, "xu_peak": 15.5 * sm_hz / 1e12,
                    "xu_frac": x_ops / (15.5 * sm_hz)}
    step_ms = ms_max / args.steps
    b_pair = W * H * (2 * 1 + 4 + 1)  # inputs + fp32 disparity + u8 mask
    line = {
        "metric": "640x480 stereo pairs/sec", "value": value, "unit": "pairs/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded config-0 generator, see DESIGN.md)",
        "config": {"workload": "config2: batch of 640x480 u8 gray pairs, exps 3..1, 8x8 patches "
                               "stride 4, variance off",
                   "global_batch": world * B, "per_gpu_batch": B,
                   "parallelism": f"pair-sharded x{world} (no collective)",
                   "inputs": "generated on device (pstereo_gpu_synth, byte-identical to the "
                             "host generator)",
                   "l2": (f"inputs {2 * B * W * H / 1e6:.0f} MB/step per GPU "
                          + ("> 126 MB L2 (no flush needed)" if 2 * B * W * H > 126e6
                             else "< 126 MB L2: reduced batch, not a bench number"))},
        "gpu_launches": launches_per_step * args.steps,
        "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": 2 * B * W * H,
                "d2h_bytes_per_step": B * W * H * 4, "steps": e2e_steps,
                "output": "fp32 filtered disparity, NaN at invalid pixels"},
        "roofline": {"bound": "hbm", "kernel": f"k_patches, finest level (exp {e_f})",
                     "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "peak_kind": peak_kind,
                     "alg_bytes_per_launch": alg_bytes, "launch_ms": patch_ms,
                     "pairs_per_launch": pairs_per_call,
                     "kernel_share_of_step": patch_ms * calls / prof_steps / step_ms,
                     "pipes": fp64,
                     "note": "not HBM-bound: a latency/issue-bound FP64 mirror of the "
                             "reference's double arithmetic (ncu: issue 47%, FP64 34%, XU 42%; "
                             "DESIGN.md section 4, profiles/r01)"},
        "path_roofline": {"bytes_per_pair": b_pair, "roofline_pairs_s": hbm * 1e9 / b_pair,
                          "frac": value / (world * hbm * 1e9 / b_pair)},
        "stage_ms_per_step": {k: v / prof_steps for k, v in stages.items()},
        "stage_note": "instrumented pass (stage events serialise launches), outside the timed "
                      "region",
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        n_cpu = min(B, max(16, 16 * cores))
        rate, times = cpu_throughput(left[:n_cpu], right[:n_cpu], oracle_cfg(), cores)
        _, kind = _cpu_oracle()
        line["cpu_baseline"] = {
            "value": rate, "unit": "pairs/s", "cores": cores, "kind": kind,
            "sample": f"first {n_cpu} pairs of this batch, {cores} workers x run_pipeline "
                      f"threads=1; median single-pair runtime_ms {float(np.median(times)):.1f}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    m.close()
    if world > 1:
        dist.destroy_process_group()


def _axis(L, s, stride):
    c0 = (s - 1) * 0.5
    cmax = (L - 1) - c0
    out = []
    k = 0
    while True:
        c = c0 + k * stride
        if c >= cmax - 1e-9:
            out.append(cmax)
            return out
        out.append(c)
        k += 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (profiling)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
