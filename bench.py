#!/usr/bin/env python
"""BDIS matching-core throughput on B200 (BASELINE.json metric: 640x480 stereo
pairs/sec at 1/2/4/8 B200, fraction of the memory roofline).

A "step" = one batched run_pipeline (pyramid -> per-level patch solves ->
finest fusion -> confidence filter -> output) over the workload's batch. The
default workload is BASELINE config 2: 256 seeded config-0 generator pairs,
640x480 uint8 gray, exps 3..1, 8x8 patches at stride 4, variance off. Under
N ranks the batch is split into contiguous pair blocks (strong scaling, the
BASELINE definition: 256 pairs total, 32 per GPU at N=8); pairs are
independent, so there is no collective on the data path -- the only
collective is the max-over-ranks reduction of the timings. A weak-scaling
number (256 pairs per GPU) is reported beside it when N > 1.

  value     device-resident inputs/outputs, CUDA events on the launch stream
  e2e       the same through the public C ABI with pinned HOST buffers: H2D of
            both views and D2H of the output inside every timed step
  roofline  dominant kernel (the finest-level k_patches launch) from live
            CUDA events; DRAM traffic from the committed ncu capture
  cpu_baseline  the reference (oracle/_ref: the unmodified reference sources)
            on this host's cores over the same batch (rank 0, N=1 only)
  parity    the GPU step's outputs against those reference outputs

The timed step's output is the filtered disparity map as fp32 with NaN at
invalid pixels (the validity mask folded in: the BASELINE bytes-per-pair);
`full_outputs` times the same batch writing every plane run_pipeline returns
(disparity + mask, probability, depth + mask).

--impl reference times the reference CPU implementation itself (run_pipeline
from oracle/_ref, all host cores) on the same workload; that process never
loads the product library (its inputs come from oracle/libbdis_synth.so).

`python bench.py --gpus N` with no torchrun environment launches the N ranks
itself (torch.distributed.run, 127.0.0.1).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HBM_FALLBACK_GBS = 6650.0
FOCAL, BASELINE_MM = 500.0, 5.0


# ---------------------------------------------------------------------------
# workloads (BASELINE.json configs): generator config + overrides, the
# PipelineConfig fields (SURVEY.md 8a mapping), the batch

def _c4_levels(w, h, s):
    ce, ws, hs = 1, (w + 1) // 2, (h + 1) // 2
    while ce < 4 and (ws + 1) // 2 >= s and (hs + 1) // 2 >= s:
        ws, hs, ce = (ws + 1) // 2, (hs + 1) // 2, ce + 1
    return ce


def workload(name: str) -> dict:
    c0 = dict(coarsest_exp=3, finest_exp=1, patch_size=8, overlap=0.5)
    if name == "c2":
        return dict(name=name, gen=0, over={}, W=640, H=480, C=1, batch=256, params=c0,
                    desc="config2: 640x480 u8 gray, exps 3..1, 8x8 patches stride 4, "
                         "variance off, seeds 0..255")
    if name == "c1":
        return dict(name=name, gen=1, over={}, W=640, H=480, C=1, batch=256,
                    params=dict(c0, estimate_variance=True),
                    desc="config1 generator (photometric stress), 640x480 u8 gray, exps 3..1, "
                         "8x8 patches stride 4, variance on")
    if name == "c3":
        return dict(name=name, gen=3, over={}, W=1280, H=1024, C=1, batch=128,
                    params=dict(coarsest_exp=4, finest_exp=1, patch_size=12,
                                overlap=1.0 - 4.0 / 12.0, estimate_variance=True),
                    desc="config3: 1280x1024 u8 gray, exps 4..1, 12x12 patches stride 4, "
                         "variance on")
    if name.startswith("c4:"):
        # c4:WxH:size:stride:channels:batch
        dims, s, st, ch, b = name[3:].split(":")
        w, h = (int(v) for v in dims.split("x"))
        s, st, ch, b = int(s), int(st), int(ch), int(b)
        return dict(name=name, gen=4, over=dict(width=w, height=h, channels=ch), W=w, H=h, C=ch,
                    batch=b, params=dict(coarsest_exp=_c4_levels(w, h, s), finest_exp=1,
                                         patch_size=s, overlap=1.0 - st / s),
                    desc=f"config4 sweep: {w}x{h} u8 x{ch}, {s}x{s} patches stride {st}")
    raise SystemExit(f"unknown workload {name!r} (c2, c1, c3, c4:WxH:s:stride:ch:batch)")


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


def metric_name(wl) -> str:
    return f"{wl['W']}x{wl['H']} stereo pairs/sec"


def bytes_per_pair(wl) -> int:
    # u8 input views + fp32 disparity + u8 mask (+ fp32 var)
    var = 4 if wl["params"].get("estimate_variance") else 0
    return wl["W"] * wl["H"] * (2 * wl["C"] + 4 + 1 + var)


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the reference's own sources, else the C port)

def workload_config(wl, B: int, world: int) -> dict:
    """The line's `config`: the workload both arms run, identical in the two
    arms' lines (arm-specific details go under `run`)."""
    nb = -(-B // world)
    step_in = 2 * nb * wl["W"] * wl["H"] * wl["C"]
    n_sets = input_sets(step_in)
    return {"workload": wl["desc"], "global_batch": B, "per_gpu_batch": nb,
            "parallelism": f"pair-sharded x{world}, contiguous blocks, no collective",
            "l2": (f"inputs {step_in / 1e6:.0f} MB/step per GPU "
                   + ("> 126 MB L2 (no flush needed)" if n_sets == 1 else
                      f"< 126 MB L2: steps cycle over {n_sets} input sets "
                      f"({n_sets * step_in / 1e6:.0f} MB > 2x L2)"))}


def input_sets(step_in: int) -> int:
    """Distinct input sets the timed steps cycle over, so that no step reads
    L2-resident inputs: one when a step's inputs exceed the 126 MB L2."""
    return 1 if step_in > 126e6 else -(-int(2 * 126e6) // max(step_in, 1))


def _cpu_oracle():
    from oracle import pyoracle

    kind = "reference" if pyoracle.available("reference") else "port"
    return pyoracle.load(kind), kind


def cpu_run(left, right, params, threads, keep=False):
    """run_pipeline on every pair with `threads` workers (threads=1 each:
    pair-level parallelism, the fair CPU throughput per SURVEY.md 8d).
    Returns (pairs/s over the wall time, per-pair runtime_ms, outputs|None)."""
    from oracle import pyoracle

    orc, _ = _cpu_oracle()
    cfg = pyoracle.Config(**params)
    grays = [(orc.to_grayscale(left[k]), orc.to_grayscale(right[k]))
             for k in range(left.shape[0])]
    idx = [0]
    lock = threading.Lock()
    times = [0.0] * len(grays)
    outs = [None] * len(grays) if keep else None

    def worker():
        while True:
            with lock:
                k = idx[0]
                idx[0] += 1
            if k >= len(grays):
                return
            (lf, lv), (rf, rv) = grays[k]
            r = orc.run_pipeline(lf, rf, cfg, FOCAL, BASELINE_MM, lv, rv)
            times[k] = r["runtime_ms"]
            if keep:
                outs[k] = {n: r[n] for n in ("disparity", "disparity_valid", "probability",
                                             "depth", "depth_valid")}

    ths = [threading.Thread(target=worker) for _ in range(threads)]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - t0
    return len(grays) / wall, times, outs


def run_reference_arm(args, wl):
    """The reference's own CPU implementation (run_pipeline, oracle/_ref) on the
    same workload: every step is the whole batch on all host cores. Never
    imports the product (inputs from the test-side generator library)."""
    from oracle import pyoracle

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = host_cores()
    _, kind = _cpu_oracle()
    B = wl["batch"]
    left, right = pyoracle.synth_batch(wl["gen"], B, seed0=0, threads=cores, **wl["over"])
    step_s = []
    for step in range(args.warmup + args.steps):
        rate, _, _ = cpu_run(left, right, wl["params"], cores)
        if step >= args.warmup:
            step_s.append(B / rate)
    total_t = sum(step_s)
    value = B * args.steps / total_t
    world = int(os.environ.get("WORLD_SIZE", "1"))
    sample = (f"{args.steps} timed steps x {B} pairs ({wl['name']}, seeds 0..{B - 1}), "
              f"{cores} workers, one pair per worker at a time, run_pipeline threads=1")
    line = {
        "impl": "reference", "metric": metric_name(wl), "value": value, "unit": "pairs/s",
        "n_gpus": max(args.gpus, world), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(wl, B, max(args.gpus, world)),
        "run": {"arm": "the reference's run_pipeline on the host", "host_threads": cores},
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


def parity_report(ref_outs, gpu, k0):
    """Pairs k0.. of the GPU's F64 planes (device tensors) against the
    reference's run_pipeline outputs for the same pairs."""
    import torch

    n = len(ref_outs)
    bitexact = 0
    mask_diff = 0
    max_dd = 0.0
    planes = ("disparity", "probability", "depth")
    for k in range(n):
        ro = ref_outs[k]
        g = {name: gpu[name][k0 + k].cpu().numpy() for name in gpu}
        same = True
        for vname in ("disparity_valid", "depth_valid"):
            d = int((g[vname] != ro[vname]).sum())
            same = same and d == 0
            if vname == "disparity_valid":
                mask_diff += d
        for name in planes:
            a = np.ascontiguousarray(g[name]).view(np.uint64)
            b = np.ascontiguousarray(ro[name]).view(np.uint64)
            same = same and bool(np.array_equal(a, b))
        both = (g["disparity_valid"] != 0) & (ro["disparity_valid"] != 0)
        if both.any():
            max_dd = max(max_dd, float(np.abs(g["disparity"][both] - ro["disparity"][both]).max()))
        bitexact += int(same)
        del g
    torch.cuda.synchronize()
    return {"pairs": n, "bitexact": bitexact, "mask_diff_px": mask_diff, "max_abs_dd": max_dd,
            "planes": "disparity, disparity_valid, probability, depth, depth_valid (f64 bits)",
            "against": "oracle/_ref run_pipeline (the unmodified reference)"}


def bind_to_gpu_numa_node(device: int):
    """Pins this rank's host threads to the CPUs of its GPU's NUMA node (from
    the PCI device's local_cpulist), so the pinned staging buffers of the e2e
    leg are first-touched, and copied from, memory next to the GPU's PCIe
    root. Best effort: returns the CPU list used, or None."""
    import torch

    try:
        pr = torch.cuda.get_device_properties(device)
        bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        text = Path(f"/sys/bus/pci/devices/{bdf}/local_cpulist").read_text().strip()
        cpus = set()
        for part in text.split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus and len(cpus) < os.cpu_count():
            os.sched_setaffinity(0, cpus)
            return text
    except Exception:
        pass
    return None


def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    import paper_2205_03133_b200 as P
    from paper_2205_03133_b200.shard import max_over_ranks, strong_shard, weak_shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    # more ranks than GPUs (a one-GPU box): a functional run of the multi-rank
    # logic, not a measurement -- ranks share the GPU, timings reduce over gloo
    folded = world > ndev
    backend = os.environ.get("PSTEREO_BENCH_BACKEND", "gloo" if folded else "nccl")
    local %= max(ndev, 1)
    torch.cuda.set_device(local)
    # N > 1: each rank's host threads on its GPU's NUMA node (N = 1 keeps every
    # core: its cpu_baseline leg runs the reference on all of them)
    numa = bind_to_gpu_numa_node(local) if world > 1 else None
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    W, H, CH, B = wl["W"], wl["H"], wl["C"], wl["batch"]
    cfg = P.PipelineConfig(**wl["params"])
    dev = torch.device("cuda", local)
    # pairs are independent: contiguous blocks, no exchange
    shard = strong_shard(B, rank, world)
    nb = shard.count
    shape = (nb, H, W) if CH == 1 else (nb, H, W, CH)
    # inputs generated in HBM by the device generator:
    # the same bytes as the host generator, without host work or PCIe per rank
    dl, dr = P.synth_batch_gpu(wl["gen"], nb, seed0=shard.start, device=local, **wl["over"])
    torch.cuda.synchronize(dev)
    disp = torch.empty((max(nb, 1), H, W), dtype=torch.float32, device=dev)
    m = P.Matcher(cfg, W, H, max(B, 1), device=local)
    # a dedicated stream: our kernels and the timing events share it (NULL
    # would select the context's own stream, not torch's legacy stream)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    NAN = float("nan")

    def step(n=nb, l=dl, r=dr, outs=None):
        m.run_device_u8(n, W, H, CH, l.data_ptr(), r.data_ptr(),
                        outs or {"disparity": disp.data_ptr()}, stream=sh, invalid_value=NAN)

    # The timed leg keeps `inflight` steps in flight: step k runs on context
    # k % inflight, each with its own stream and output, so one batch's
    # latency-bound coarse levels and finalize overlap the next batch's
    # finest level (a server with several batches queued).
    # Inputs: when one step's views would fit in the 126 MB L2, steps cycle
    # over distinct input sets (more seeds of the same generator) totalling
    # more than twice the L2, so no timed step reads L2-resident inputs.
    inflight = max(1, args.inflight)
    step_in = 2 * nb * W * H * CH
    n_sets = input_sets(step_in)
    sets = [(dl, dr)] + [P.synth_batch_gpu(wl["gen"], nb, seed0=shard.start + k * max(B, 1),
                                           device=local, **wl["over"])
                         for k in range(1, n_sets)]
    ctxs = [m] + [P.Matcher(cfg, W, H, max(B, 1), device=local) for _ in range(1, inflight)]
    if inflight > 1:  # the in-flight batches fill the GPU: no extra band split
        for c in ctxs:
            c.set_fill_target(0)
    outs_k = [disp] + [torch.empty_like(disp) for _ in range(1, inflight)]
    streams = [stream] + [torch.cuda.Stream(dev) for _ in range(1, inflight)]
    kstep = [0]

    def step_inflight():
        k = kstep[0]
        kstep[0] += 1
        j = k % inflight
        l, r = sets[k % n_sets]
        ctxs[j].run_device_u8(nb, W, H, CH, l.data_ptr(), r.data_ptr(),
                              {"disparity": outs_k[j].data_ptr()},
                              stream=streams[j].cuda_stream, invalid_value=NAN)

    def timed_inflight(steps, warmup):
        for _ in range(warmup):
            step_inflight()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for st in streams[1:]:
            st.wait_stream(stream)
        for _ in range(steps):
            step_inflight()
        for st in streams[1:]:
            stream.wait_stream(st)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        return max_over_ranks(e0.elapsed_time(e1), device=None if backend != "nccl" else dev)

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        return max_over_ranks(e0.elapsed_time(e1), device=None if backend != "nccl" else dev)

    # every in-flight context runs at least one untimed step (its first call
    # allocates its working set)
    warm = max(args.warmup, inflight)
    for _ in range(warm):
        step_inflight()
    torch.cuda.synchronize(dev)
    launches_per_step = m.launch_count()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ms_max = timed_inflight(args.steps, 0)
    clk = clocks.stop()
    for c in ctxs[1:]:
        c.close()
    m.set_fill_target(148)
    del ctxs, outs_k
    step()  # `disp` = this rank's batch (input set 0) for the checks below
    torch.cuda.synchronize(dev)
    value = B * args.steps / (ms_max / 1e3)
    step_ms = ms_max / args.steps

    # every plane run_pipeline returns (PipelineOutput: disparity, probability,
    # depth; validity planes) for the same batch
    full = {"disparity": torch.empty((max(nb, 1), H, W), dtype=torch.float32, device=dev),
            "disparity_valid": torch.empty((max(nb, 1), H, W), dtype=torch.uint8, device=dev),
            "probability": torch.empty((max(nb, 1), H, W), dtype=torch.float32, device=dev),
            "depth": torch.empty((max(nb, 1), H, W), dtype=torch.float32, device=dev),
            "depth_valid": torch.empty((max(nb, 1), H, W), dtype=torch.uint8, device=dev)}
    full_ptrs = {k: v.data_ptr() for k, v in full.items()}

    kfull = [0]

    def step_full():
        l, r = sets[kfull[0] % n_sets]
        kfull[0] += 1
        m.run_device_u8(nb, W, H, CH, l.data_ptr(), r.data_ptr(), full_ptrs, stream=sh,
                        focal=FOCAL, baseline=BASELINE_MM)

    full_ms = timed(step_full, max(3, min(args.steps, 10)), 2) / max(3, min(args.steps, 10))
    del full, sets

    # weak scaling beside it (N > 1): every rank matches B pairs
    weak = None
    if world > 1 and not args.no_weak:
        ws = weak_shard(B, rank, world)
        wl_, wr_ = P.synth_batch_gpu(wl["gen"], B, seed0=ws.start, device=local, **wl["over"])
        wdisp = torch.empty((B, H, W), dtype=torch.float32, device=dev)
        wsteps = max(3, min(args.steps, 10))
        wms = timed(lambda: step(B, wl_, wr_, {"disparity": wdisp.data_ptr()}), wsteps, 2)
        weak = {"value": world * B * wsteps / (wms / 1e3), "unit": "pairs/s",
                "per_gpu_batch": B, "global_batch": world * B, "ms_per_step": wms / wsteps}
        del wl_, wr_, wdisp

    # per-stage device times from a separate, instrumented pass (stage events
    # serialise the launches, so they stay out of the timed region)
    m.set_device_chunks(1)  # one launch per stage: per-launch durations for the roofline
    step()
    torch.cuda.synchronize(dev)
    m.set_profiling(True)
    prof_steps = min(args.steps, 10)
    for _ in range(prof_steps):
        step()
    torch.cuda.synchronize(dev)
    stages, calls = m.stage_times()
    m.set_profiling(False)
    m.set_device_chunks(2)
    pairs_per_call = nb * prof_steps / max(calls, 1)

    # ---- e2e through the public ABI with pinned host buffers
    hl = dl.cpu().pin_memory()
    hr = dr.cpu().pin_memory()
    hd = torch.empty((max(nb, 1), H, W), dtype=torch.float32).pin_memory()
    houts = {"disparity": hd.data_ptr()}

    def step_e2e():
        # async host outputs: step k+1's uploads and kernels run under step k's
        # downloads; every step still moves its own inputs and result
        m.run_host_u8(nb, W, H, CH, hl.data_ptr(), hr.data_ptr(), houts, stream=sh,
                      invalid_value=NAN, async_host=True)

    # three times the device leg's steps (at most 60): the host-memory-bound leg
    # is the noisier one on a shared host
    e2e_steps = 0 if args.no_e2e else max(3, min(3 * args.steps, 60))
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
    e2e_s = max_over_ranks(e2e_s, device=None if backend != "nccl" else dev)
    e2e_value = B * e2e_steps / e2e_s if e2e_steps else None
    if e2e_steps:  # the e2e output equals the device-resident run
        dc = disp[:nb].cpu()
        assert torch.equal(torch.isnan(hd[:nb]), torch.isnan(dc)), "e2e validity differs"
        assert torch.equal(torch.nan_to_num(hd[:nb]), torch.nan_to_num(dc)), "e2e output differs"

    # ---- roofline of the dominant kernel: the finest-level k_patches launch
    hbm, peak_kind = peaks()
    dims = P.level_dims(cfg, W, H)
    e_f, w_f, h_f = dims[-1]
    host_expand = os.environ.get("PSTEREO_HOST_EXPAND", "1") != "0" and e_f >= 1
    s_ = cfg.patch_size
    st_ = max(1, int(round(cfg.patch_size * (1 - cfg.overlap))))
    npatch_f = len(_axis(w_f, s_, st_)) * len(_axis(h_f, s_, st_))
    # read the left/right/gradient fp32 planes (12 B/px)
    # and the coarser records (16 B/patch), write the records (32 B/patch)
    alg_bytes = pairs_per_call * (12.0 * w_f * h_f + 48.0 * npatch_f)
    patch_ms = stages.get(f"patches_e{e_f}", 0.0) / max(calls, 1)
    achieved = alg_bytes / (patch_ms / 1e3) / 1e9 if patch_ms > 0 else 0.0
    traffic = None
    pipes = None
    tj = ROOT / "profiles" / "ncu_traffic.json"
    if tj.exists() and wl["name"] == "c2":
        t = json.loads(tj.read_text())["k_patches_finest"]
        traffic = t["dram_bytes_per_launch"] / t["pairs_in_launch"] * pairs_per_call
        if "fp64_inst_per_launch" in t and patch_ms > 0:
            # the pipes this kernel actually runs on: FP64 (DADD/DMUL/DFMA) and
            # XU (conversions); counts from ncu for the same launch scaled to
            # this batch, time from the live CUDA events; peaks are this box's
            # measured per-SM rates (scripts/tools/microbench.cu: DADD 62.6, F2F 15.5
            # thread-ops/clk/SM) x 148 SMs x max clock
            sm_hz = 148 * 1965e6
            scale = pairs_per_call / t["pairs_in_launch"] / (patch_ms / 1e3)
            f_ops = t["fp64_inst_per_launch"] * scale
            x_ops = t["conversion_inst_per_launch"] * scale
            pipes = {"unit": "T thread-inst/s",
                     "fp64_achieved": f_ops / 1e12, "fp64_peak": 62.6 * sm_hz / 1e12,
                     "fp64_frac": f_ops / (62.6 * sm_hz),
                     "xu_achieved": x_ops / 1e12, "xu_peak": 15.5 * sm_hz / 1e12,
                     "xu_frac": x_ops / (15.5 * sm_hz)}
            if "warp_inst_per_launch" in t:
                i_ops = t["warp_inst_per_launch"] * scale
                pipes["issue_frac"] = i_ops / (4 * sm_hz)
    b_pair = bytes_per_pair(wl)
    line = {
        "metric": metric_name(wl), "value": value, "unit": "pairs/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator, see DESIGN.md)",
        "config": workload_config(wl, B, world),
        "run": {"arm": "B200 kernels through the C ABI",
                "inputs": "generated on device (pstereo_gpu_synth, byte-identical to the "
                          "host generator)",
                "output": "fp32 filtered disparity, NaN = invalid (mask folded in)",
                "inflight": inflight,
                "warmup_steps_run": warm,
                "host_cpus": numa or "unpinned"},
        "gpu_launches": launches_per_step * args.steps,
        "full_outputs": {"value": B / (full_ms / 1e3), "unit": "pairs/s", "ms_per_step": full_ms,
                         "planes": "disparity f32 + mask, probability f32, depth f32 + mask"},
        "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": 2 * B * W * H * CH,
                # the link carries the plane at the finest level's resolution; host
                # threads replicate it 2^e x 2^e into the caller's full-size buffer
                "d2h_bytes_per_step": B * w_f * h_f * 4 if host_expand else B * W * H * 4,
                "host_output_bytes_per_step": B * W * H * 4,
                "host_expand": (f"on: finest-resolution download ({w_f}x{h_f}), "
                                f"{P.lib().pstereo_gpu_host_threads()} host threads write the "
                                f"{W}x{H} plane (upsample_to_full's replication)"
                                if host_expand else "off: full-resolution download"),
                "steps": e2e_steps,
                "output": "fp32 filtered disparity, NaN at invalid pixels, full resolution "
                          "in pinned host memory"},
        "roofline": {"bound": "hbm", "kernel": f"k_patches, finest level (exp {e_f})",
                     "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "peak_kind": peak_kind,
                     "alg_bytes_per_launch": alg_bytes, "launch_ms": patch_ms,
                     "pairs_per_launch": pairs_per_call,
                     "kernel_share_of_step": patch_ms * calls / prof_steps / step_ms,
                     "pipes": pipes,
                     "note": "not HBM-bound: an issue/FP64-bound mirror of the reference's "
                             "double arithmetic (DESIGN.md section 4, profiles/)"},
        "path_roofline": {"bytes_per_pair": b_pair, "roofline_pairs_s": world * hbm * 1e9 / b_pair,
                          "frac": value / (world * hbm * 1e9 / b_pair)},
        "stage_ms_per_step": {k: v / prof_steps for k, v in stages.items()},
        "stage_note": "instrumented pass (stage events serialise launches), outside the timed "
                      "region",
        "clocks": clk,
    }
    if weak:
        line["weak_scaling"] = weak
    if folded:
        line["functional_only"] = (f"{world} ranks on {ndev} GPU(s): the multi-rank path ran, "
                                   "the number is not a measurement")
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        left, right = dl.cpu().numpy(), dr.cpu().numpy()
        rate, times, ref_outs = cpu_run(left, right, wl["params"], cores, keep=True)
        _, kind = _cpu_oracle()
        line["cpu_baseline"] = {
            "value": rate, "unit": "pairs/s", "cores": cores, "kind": kind,
            "sample": f"all {nb} pairs of this batch, {cores} workers x run_pipeline threads=1; "
                      f"median single-pair runtime_ms {float(np.median(times)):.1f}"}
        # parity of this batch: the GPU's f64 planes against the reference's
        f64 = {"disparity": torch.empty((nb, H, W), dtype=torch.float64, device=dev),
               "disparity_valid": torch.empty((nb, H, W), dtype=torch.uint8, device=dev),
               "probability": torch.empty((nb, H, W), dtype=torch.float64, device=dev),
               "depth": torch.empty((nb, H, W), dtype=torch.float64, device=dev),
               "depth_valid": torch.empty((nb, H, W), dtype=torch.uint8, device=dev)}
        m.run_device_u8(nb, W, H, CH, dl.data_ptr(), dr.data_ptr(),
                        {k: v.data_ptr() for k, v in f64.items()}, dtype=P.F64, stream=sh,
                        focal=FOCAL, baseline=BASELINE_MM)
        torch.cuda.synchronize(dev)
        line["parity"] = parity_report(ref_outs, f64, 0)
        # the timed step's own output (fp32, NaN = invalid) for the same pairs
        dd = disp[:nb].cpu().numpy()
        ok = all(np.array_equal(~np.isnan(dd[k]), ref_outs[k]["disparity_valid"] != 0) and
                 np.array_equal(dd[k][~np.isnan(dd[k])],
                                ref_outs[k]["disparity"].astype(np.float32)[~np.isnan(dd[k])])
                 for k in range(nb))
        line["parity"]["timed_output_matches"] = bool(ok)
        del f64, ref_outs
    if rank == 0:
        print(json.dumps(line), flush=True)
    m.close()
    if world > 1:
        dist.destroy_process_group()


def run_sweep_c4(args):
    """BASELINE config 4 on one GPU: every resolution at s=8 stride 4 and
    every (patch size, stride) in {8,12,16} x {2,4,6} at 640x480, RGB inputs
    from the device generator; batch 1 (latency: one call at a time, host
    wall clock to a completed output, median of 20) and batch 1024
    (throughput, pairs/s, CUDA events), device-resident. The latency calls
    replay a CUDA graph of the call (pstereo_gpu_set_graphs, --graphs 0 for
    eager calls): the per-call host work and launch gaps a repeated caller
    avoids. Beside it, the
    reference's run_pipeline on one host core for pair 0, whose outputs the
    GPU's batch-1 call must match bit for bit. One JSON line per case."""
    import torch

    import paper_2205_03133_b200 as P

    cases = [(w, h, 8, 4) for w, h in ((320, 240), (640, 480), (1280, 1024), (1920, 1080))]
    cases += [(640, 480, s, st) for s in (8, 12, 16) for st in (2, 4, 6) if (s, st) != (8, 4)]
    if args.sweep_cases:
        cases = [cases[int(i)] for i in args.sweep_cases.split(",")]
    big = args.batch or 1024
    for w, h, s, st in cases:
        wl = workload(f"c4:{w}x{h}:{s}:{st}:3:{big}")
        cfg = P.PipelineConfig(**wl["params"])
        row = {"workload": wl["desc"], "exps": f"{cfg.coarsest_exp}..{cfg.finest_exp}",
               "unit": "pairs/s",
               "latency_mode": "CUDA graph replay" if args.graphs else "eager calls"}
        for B in (1, big):
            dl, dr = P.synth_batch_gpu(4, B, seed0=0, **wl["over"])
            disp = torch.empty((B, h, w), dtype=torch.float32, device="cuda")
            stream = torch.cuda.Stream()
            with P.Matcher(cfg, w, h, B) as m:
                if B == 1 and args.graphs:
                    m.set_graphs(True)  # latency as a repeated-call user sees it

                def step():
                    m.run_device_u8(B, w, h, 3, dl.data_ptr(), dr.data_ptr(),
                                    {"disparity": disp.data_ptr()}, stream=stream.cuda_stream,
                                    invalid_value=float("nan"))
                for _ in range(max(args.warmup, 3)):
                    step()
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                if B == 1:
                    # latency: one call at a time, host wall clock from the call
                    # until its output is complete (median of 20)
                    lat = []
                    for _ in range(20):
                        t0 = time.perf_counter()
                        step()
                        stream.synchronize()
                        lat.append((time.perf_counter() - t0) * 1e3)
                    ms = float(np.median(lat))
                else:
                    reps = max(3, min(args.steps, 5))
                    e0.record(stream)
                    for _ in range(reps):
                        step()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1) / reps
            if B == 1:
                row["latency_ms_b1"] = ms
                left, right = dl.cpu().numpy(), dr.cpu().numpy()
                d1 = disp[0].cpu().numpy()
            else:
                row[f"pairs_s_b{B}"] = B / (ms / 1e3)
            del dl, dr, disp
            torch.cuda.empty_cache()
        _, kind = _cpu_oracle()
        _, times, outs = cpu_run(left, right, wl["params"], 1, keep=True)
        ref = outs[0]
        ok = (np.array_equal(~np.isnan(d1), ref["disparity_valid"] != 0) and
              np.array_equal(d1[~np.isnan(d1)],
                             ref["disparity"].astype(np.float32)[~np.isnan(d1)]))
        row["cpu_baseline"] = {"ms_per_pair": times[0], "cores": 1, "kind": kind,
                               "sample": "pair 0 (seed 0), run_pipeline threads=1"}
        row["parity_pair0"] = bool(ok)
        print(json.dumps(row), flush=True)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2",
                    help="c2 (default, BASELINE config 2), c1, c3, or c4:WxH:size:stride:ch:batch")
    ap.add_argument("--batch", type=int, default=0, help="override the workload's global batch")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (profiling)")
    ap.add_argument("--no-weak", action="store_true", help="skip the weak-scaling leg (N > 1)")
    ap.add_argument("--graphs", type=int, default=1,
                    help="--sweep: measure batch-1 latency with CUDA-graph replay "
                         "(pstereo_gpu_set_graphs; 1) or eager calls (0)")
    ap.add_argument("--inflight", type=int, default=4,
                    help="batches in flight in the timed leg (one context and stream each)")
    ap.add_argument("--sweep", choices=["c4"], help="BASELINE config-4 sweep, one JSON line "
                    "per case (1 GPU; --batch overrides the throughput batch of 1024)")
    ap.add_argument("--sweep-cases", default="", help="comma-separated case indices (sweep)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launch the ranks ourselves: one process per GPU (torchrun semantics)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(_free_port()), str(Path(__file__).resolve()), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    if args.sweep:
        run_sweep_c4(args)
        return
    wl = workload(args.workload)
    if args.batch:
        wl["batch"] = args.batch
    if args.impl == "reference":
        run_reference_arm(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
