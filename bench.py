#!/usr/bin/env python
"""PETRA (arXiv 2406.02052) on B200: one JSON line per run (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--model revnet18|revnet34|revnet50] [--batch B] [--stages J]
                    [--precision bf16|fp32] [--no-cpu-baseline]

A step is one steady-state PETRA tick of the whole pipeline: every stage runs
one forward (theta^t) and one backward (approximate inversion + VJP +
immediate Nesterov update) on different micro-batches, so
one micro-batch of B samples completes per tick.  value = B * K / (max over
ranks of the summed device time of the K ticks).  Default workload: BASELINE
configs[1], RevNet-18 on CIFAR-10-shaped synthetic data, batch 64, J = 4.
--impl reference times the fp64 CPU oracle (oracle/) on a bounded sample of the
same workload.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RevNet-18/50 train samples/s at 1/2/4/8 B200 stages; tensor-pipe % of peak"
IMAGE = {"revnet18": (32, 10), "revnet34": (32, 1000), "revnet50": (224, 1000)}
WD = {"revnet18": 5e-4, "revnet34": 1e-4, "revnet50": 1e-4}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


def workload_name(a):
    H, classes = IMAGE[a.model]
    ds = {"revnet18": "CIFAR-10", "revnet34": "ImageNet32", "revnet50": "ImageNet"}[a.model]
    return (f"{a.model.replace('revnet', 'RevNet-')} PETRA, {ds} shape 3x{H}x{H} ({classes} classes), "
            f"batch {a.batch}, J={a.stages} stages")


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region:
    NVML every 2 ms in a thread (plus one sample at start and one at stop, so a short
    timed region still has samples); nvidia-smi -lms 100 as the fallback."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc, self.nv = index, [], None, None
        self.sm, self.reasons, self.mx = [], set(), None

    def _nvml_sample(self):
        nv, h = self.nv, self.h
        self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        for name, bit in zip(self.NAMES, (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                                          nv.nvmlClocksEventReasonSwThermalSlowdown,
                                          nv.nvmlClocksEventReasonSwPowerCap)):
            if r & bit:
                self.reasons.add(name)

    def _nvml_loop(self):
        while not self.done:
            try:
                self._nvml_sample()
            except Exception:
                return
            time.sleep(0.002)

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.done = False
            self._nvml_sample()
            self.th = threading.Thread(target=self._nvml_loop, daemon=True)
            self.th.start()
            return
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.nv is not None:
            self.done = True
            self.th.join(timeout=2)
            try:
                self._nvml_sample()
            except Exception:
                pass
            return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.mx,
                    "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 9]
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = sorted({n for r in rows for n, v in zip(self.NAMES, r[5:9]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "source": "nvidia-smi"}


# ----------------------------------------------------------------------------- oracle timing
def oracle_tick_seconds(model, batch, J, counts, seed=0):
    """Time the fp64 oracle on the work of one steady-state tick: every stage
    runs one forward and one backward (the tail stage its fused step) at
    `batch`.  Returns (seconds, threads)."""
    import numpy as np
    import synth
    from oracle import engine as E, models as OM
    H, classes = IMAGE[model]
    units = OM.init_params(OM.build_revnet(model, H, classes), 1)
    groups = OM.group(units, counts)
    stages = [E.Stage(g, E.OptConfig(weight_decay=WD[model])) for g in groups]
    x = [synth.images((batch, 3, H, H), seed, 0)]
    y = synth.labels(batch, classes, seed, 0)
    # stage inputs: one untimed forward pass through the stages
    msgs = [E.Fwd(0, x, y)]
    for s in stages[:-1]:
        s.j, s.J = 1, J
        msgs.append(s.forward(msgs[-1]))
    # timed: forward + backward of every stage on the stage-local message
    outs = []
    t0 = time.perf_counter()
    for j, s in enumerate(stages):
        s.lr = 0.025
        if j < J - 1:
            m = s.forward(E.Fwd(1, msgs[j].xs, y))
            s.backward(E.Bwd(0, m.xs, [np.ones_like(a) for a in m.xs]))
        else:
            s.tail_step(E.Fwd(1, msgs[j].xs, y))
    dt = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        threads = os.cpu_count()
    return dt, threads


# ----------------------------------------------------------------------------- our arm
def measure(model, stages, batch, precision, steps, warmup, world, rank, local, partition="", e2e=True):
    """Build the PETRA pipeline of `model` (this rank's stages), fill it, warm it up and
    time `steps` steady-state ticks.  Returns the measurement dict (rank 0 fields)."""
    import torch
    import torch.distributed as dist

    from paper_2406_02052_b200 import Pipeline, petra, _lib as L, models as PM
    from paper_2406_02052_b200.dist import contiguous_stage_ranks

    H, classes = IMAGE[model]
    units = PM.revnet(model, H, classes)
    # one GPU: FLOP-balanced stages (all run concurrently); several: the comm-aware
    # cost model (slowest GPU's compute + its cross-GPU message bytes / NVLink)
    counts = (PM.partition(units, stages, batch, H, H, 3) if world == 1
              else PM.partition_comm(units, stages, world, batch, H, H, 3))
    if partition:  # explicit units per stage
        counts = [int(x) for x in partition.split(",")]
        if len(counts) != stages or sum(counts) != len(units):
            raise SystemExit(f"--partition {partition}: need {stages} counts summing to {len(units)}")
    prec = L.BF16_TC if precision == "bf16" else L.FP32
    specs = PM.stage_specs(units, counts, batch, (H, H, 3), prec, WD[model])
    stage_rank = contiguous_stage_ranks(stages, world)
    if world > 1:  # the library moves the messages: ncclSend / ncclRecv on its own comm streams
        nid = [petra.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        pipe = Pipeline(specs, stage_rank, rank, world, seed=1, transport="nccl", nccl_id=nid[0], join_comm=True)
    else:
        pipe = Pipeline(specs, stage_rank, rank, world, seed=1)
    J, B = stages, batch
    dev = torch.device("cuda", local)
    gen = torch.Generator(device=dev).manual_seed(0)
    ring = 16
    owns_first = stage_rank[0] == rank
    xs = [torch.randn((B, H, H, 3), generator=gen, device=dev) for _ in range(ring)]
    ys = [torch.randint(0, classes, (B,), generator=gen, device=dev, dtype=torch.int32) for _ in range(ring)]
    loss = torch.zeros(1, device=dev)
    lr = 0.1 * 64 / 256  # PAPER.md:256 with k = 1
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    st = torch.cuda.current_stream()
    t = 0
    host_ms = []

    def tick(flush_l2=False, ev=None):
        nonlocal t
        i = t % ring
        if flush_l2:
            flush.fill_(t & 0xFF)
        if ev:
            ev[0].record(st)
        h0 = time.perf_counter()
        # at N > 1 the tick's neighbour exchange is inside the events: the pipeline joins
        # the caller's stream to it (join_comm), after overlapping it with the tick's compute
        pipe.tick(t, True, xs[i] if owns_first else None, ys[i] if owns_first else None, lr, loss, report=False)
        if ev:
            host_ms.append((time.perf_counter() - h0) * 1e3)
            ev[1].record(st)
        t += 1

    # fill the pipeline (2J-2 ticks), then one full cycle of CUDA-graph keys (a stage's
    # graph depends on its FIFO slots and the mailbox parity: period lcm(2, 2(J-j)+1)
    # <= 2(2J-1) ticks, captured once each), then the W warm-up ticks
    graph_cycle = 2 * (2 * J - 1)
    for _ in range(2 * J - 2 + graph_cycle + warmup):
        tick()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    n0 = L.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    wall0 = time.perf_counter()
    for k in range(steps):
        tick(flush_l2=True, ev=evs[k])
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = L.launch_count() - n0
    clk = clocks.stop()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
    tms = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(tms, op=dist.ReduceOp.MAX)
    ms = float(tms.item())
    value = B * steps / (ms / 1e3)

    out = {"value": round(value, 2), "unit": "samples/s", "ms_per_step": round(ms / steps, 4),
           "workload": f"{model.replace('revnet', 'RevNet-')} PETRA, "
                       f"{ {'revnet18': 'CIFAR-10', 'revnet34': 'ImageNet32', 'revnet50': 'ImageNet'}[model]} "
                       f"shape 3x{H}x{H} ({classes} classes), batch {B}, J={J} stages",
           "partition_units": counts, "stage_rank": stage_rank, "lr": lr, "fill_ticks": 2 * J - 2,
           "graph_capture_ticks": graph_cycle, "wall_s_timed": round(wall, 3),
           "host_enqueue_ms_per_step": round(statistics.median(host_ms), 4) if host_ms else None,
           "gpu_launches": launches, "clocks": clk, "prec": prec, "H": H, "classes": classes}

    # ---- e2e through the public API: pinned host inputs copied in, loss read back, every step.
    # The input copy of step k+1 runs on a copy stream under step k (double-buffered device
    # inputs, as a training loop's prefetching loader does); every copy is inside the events.
    if e2e:
        hx = [x.cpu().pin_memory() for x in xs[:4]]
        hy = [y.cpu().pin_memory() for y in ys[:4]]
        hl = torch.zeros(1).pin_memory()
        dx = [torch.empty_like(xs[0]) for _ in range(2)]
        dy = [torch.empty_like(ys[0]) for _ in range(2)]
        cs = torch.cuda.Stream()
        copied = [torch.cuda.Event() for _ in range(2)]
        used = [torch.cuda.Event() for _ in range(2)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

        def stage_in(k):  # H2D of step k's inputs into buffer k % 2 (after step k-2 released it)
            b = k % 2
            with torch.cuda.stream(cs):
                if k >= 2:
                    cs.wait_event(used[b])
                dx[b].copy_(hx[(t0 + k) % 4], non_blocking=True)
                dy[b].copy_(hy[(t0 + k) % 4], non_blocking=True)
                copied[b].record(cs)

        t0 = t
        e0.record(st)
        cs.wait_event(e0)
        if owns_first:
            stage_in(0)
        for k in range(steps):
            b = k % 2
            if owns_first:
                if k + 1 < steps:
                    stage_in(k + 1)
                st.wait_event(copied[b])
            pipe.tick(t, True, dx[b] if owns_first else None, dy[b] if owns_first else None, lr, loss, report=False)
            if owns_first:
                used[b].record(st)
            hl.copy_(loss, non_blocking=True)
            t += 1
        e1.record(st)
        torch.cuda.synchronize()
        ems = torch.tensor([e0.elapsed_time(e1)], device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        out["e2e"] = {"value": round(B * steps / (float(ems.item()) / 1e3), 2), "unit": "samples/s",
                      "h2d_bytes_per_step": (B * H * H * 3 * 4 + B * 4) if owns_first else 0, "d2h_bytes_per_step": 4}

    # ---- per-stage device time per tick (events around each stage's work on its stream)
    pipe.timing(True)
    for _ in range(steps):
        tick()
    out["stage_ms_per_tick"] = [round(x, 4) for x in pipe.stage_ms()]
    pipe.timing(False)

    # ---- per-kernel device time (profiled replay of K more steps: CUDA events on the launch stream)
    L.profile(True)
    for _ in range(steps):
        tick()
    prof = L.profile_read()
    recs = L.profile_records()
    L.profile(False)
    pipe.close()
    peaks, src = load_peaks()
    tot = sum(p["ms"] for p in prof)
    prof.sort(key=lambda p: -p["ms"])
    top = prof[0]
    name = top["name"]
    if name.startswith("conv") and name.endswith("_tc"):
        # a kernel timed alone in the serialised replay: the burst bf16 peak
        bound, peak, unit, ach = "tensor", peaks["bf16_tflops"], "TFLOP/s", top["flops"] / top["ms"] / 1e9
        peak_src = f"bf16_tflops, burst: a kernel timed alone ({src})"
    elif name.startswith("conv"):
        fp32_peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        bound, peak, unit, ach = "alu", fp32_peak, "TFLOP/s", top["flops"] / top["ms"] / 1e9
        peak_src = "148 SM x 128 FP32 lanes x 2 FLOP x sm_max_mhz (DESIGN.md)"
    else:
        bound, peak, unit, ach = "hbm", peaks["hbm_gbs"], "GB/s", top["bytes"] / top["ms"] / 1e6
        peak_src = f"hbm_gbs ({src})"
    traffic, traffic_src = None, None
    tfile = os.path.join(ROOT, "profiles", "r02", f"traffic_{model}.json")
    if not os.path.exists(tfile):
        tfile = os.path.join(ROOT, "profiles", "r01", f"traffic_{model}.json")
    if os.path.exists(tfile) and prec == L.BF16_TC:
        with open(tfile) as f:
            tj = json.load(f)
        if name in tj["categories"]:
            traffic = round(tj["categories"][name]["bytes_per_launch"])
            traffic_src = (f"dram__bytes_read.sum + dram__bytes_write.sum per logical launch, ncu launch list "
                           f"({os.path.relpath(tfile, ROOT)}; {tj['cache']})")
    # per-launch roofline of the dominant category: each logical launch's own bound,
    # max(flops / tensor peak, bytes / HBM peak) (its 1x1 K = 64 convolutions are HBM-bound,
    # the 3x3 ones tensor-bound), summed and divided by the measured time
    mine = [r for r in recs if r["name"] == name]
    t_roof = sum(max(r["flops"] / (peaks["bf16_tflops"] * 1e9), r["bytes"] / (peaks["hbm_gbs"] * 1e6)) for r in mine)
    t_meas = sum(r["ms"] for r in mine)
    n_hbm = sum(1 for r in mine if r["bytes"] / peaks["hbm_gbs"] * 1e3 > r["flops"] / peaks["bf16_tflops"])
    out["roofline"] = {
        "bound": bound, "kernel": name, "achieved": round(ach, 2), "peak": peak, "unit": unit,
        "frac": round(ach / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
        "frac_of_launch_rooflines": round(t_roof / t_meas, 4) if t_meas > 0 else None,
        # the same flops over the SM-time the launches held (duration x min(1, CTAs / 148): the
        # persistent conv CTAs take one SM each): the tensor-pipe fraction of the SMs the
        # kernel occupied -- what the grid cap trades against latency
        "frac_of_occupied_sms": (round(sum(r["flops"] for r in mine) / 1e9 / sum(
            r["ms"] * min(1.0, max(1, r["ctas"]) / 148.0) for r in mine) / peak, 4)
            if bound == "tensor" and mine else None),
        "mean_ctas": round(sum(r["ctas"] for r in mine) / max(1, len(mine)), 1),
        "launch_rooflines": (f"sum over the category's {len(mine)} launches of max(algorithmic flops / "
                             f"{peaks['bf16_tflops']} TFLOP/s, algorithmic bytes / {peaks['hbm_gbs']} GB/s) = "
                             f"{t_roof:.4f} ms over {t_meas:.4f} ms measured; {n_hbm} launches HBM-bound"),
        "algorithmic_bytes_per_launch": round(top["bytes"] / top["launches"]), "peak_source": peak_src,
        "share_of_step": round(top["ms"] / tot, 3), "launches_per_step": top["launches"] / steps,
        "method": ("profiled replay of K further steps with every stage and both directions serialised on "
                   "the launch stream: CUDA events around each logical kernel time it alone (warm L2)"),
        "serial_ms_per_step": round(tot / steps, 4)}
    flops_step = sum(p["flops"] for p in prof) / steps
    bytes_step = sum(p["bytes"] for p in prof) / steps
    step_s = ms / steps / 1e3
    # the whole step against both roofs ("report both fractions"): algorithmic
    # flops of every convolution and algorithmic bytes of every kernel per step, over the
    # device-timed step; burst peaks (the timed region is short and ran unthrottled)
    out["step_roofline"] = {
        "tensor": {"achieved": round(flops_step / step_s / 1e12, 2), "peak": peaks["bf16_tflops"],
                   "unit": "TFLOP/s", "frac": round(flops_step / step_s / 1e12 / peaks["bf16_tflops"], 4),
                   "frac_of_sustained": round(flops_step / step_s / 1e12 / peaks["bf16_tflops_sustained"], 4)},
        "hbm": {"achieved": round(bytes_step / step_s / 1e9, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(bytes_step / step_s / 1e9 / peaks["hbm_gbs"], 4)},
        "algorithmic_gflop_per_step": round(flops_step / 1e9, 2),
        "algorithmic_gbytes_per_step": round(bytes_step / 1e9, 3)}
    out["kernels"] = [{"name": p["name"], "share": round(p["ms"] / tot, 3), "launches": p["launches"],
                       "ms_per_step": round(p["ms"] / steps, 4),
                       "tflops": round(p["flops"] / p["ms"] / 1e9, 2) if p["flops"] else None,
                       "gbs": round(p["bytes"] / p["ms"] / 1e6, 1) if p["bytes"] else None} for p in prof][:12]
    out["dtype"] = "bf16" if prec == L.BF16_TC and any(k["name"].endswith("_tc") for k in out["kernels"]) else "f32"
    return out


def mlp_config1_seconds():
    """BASELINE configs[0]: the 2-stage reversible MLP (d = 64, batch 32, 10 ticks, fp64),
    timed on the host cores with the oracle (reading c16)."""
    import synth
    from oracle import engine as E, models as OM
    units = OM.init_params(OM.build_mlp(64, 10), 1)
    stages = [E.Stage(g, E.OptConfig()) for g in OM.group(units, [2, 3])]

    def batch_fn(m):
        x = synth.images((32, 64, 1, 1), 0, m)
        return [x[:, :32].copy(), x[:, 32:].copy()], synth.labels(32, 10, 0, m)
    t0 = time.perf_counter()
    E.run_petra(stages, batch_fn, 10, lr=0.025, drain=False)
    return time.perf_counter() - t0


def run_ours(a):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    m = measure(a.model, a.stages, a.batch, a.precision, a.steps, a.warmup, world, rank, local, a.partition)
    H, classes, J, B = m["H"], m["classes"], a.stages, a.batch
    out = {"metric": METRIC, "value": m["value"], "unit": "samples/s", "n_gpus": world, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": m["dtype"],
           "data": "synthetic (N(0,1) images, uniform labels; seeded device ring of 16 micro-batches)",
           "config": {"workload": m["workload"], "model": a.model, "global_batch": B, "micro_batch": B,
                      "image": [3, H, H], "classes": classes, "stages": J, "partition_units": m["partition_units"],
                      "stage_rank": m["stage_rank"], "parallelism": f"petra-stages{J}-over-{world}gpu",
                      "partitioner": "flop-balanced" if world == 1 else "comm-aware cost model",
                      "precision_requested": a.precision, "lr": m["lr"], "fill_ticks": m["fill_ticks"],
                      "graph_capture_ticks": m["graph_capture_ticks"],
                      "l2": "flushed between timed steps (256 MiB write, outside the events)",
                      "exchange": ("library NCCL send/recv, inside the per-tick events (join_comm)" if world > 1
                                   else "none (one rank)"),
                      "wall_s_timed": m["wall_s_timed"], "host_enqueue_ms_per_step": m["host_enqueue_ms_per_step"]},
           "roofline": m["roofline"], "step_roofline": m["step_roofline"], "gpu_launches": m["gpu_launches"],
           "clocks": m["clocks"], "e2e": m["e2e"], "kernels": m["kernels"],
           "algorithmic_gflop_per_step": m["step_roofline"]["algorithmic_gflop_per_step"],
           "stage_ms_per_tick": m["stage_ms_per_tick"]}
    if world == 1 and a.north_star and a.model != "revnet50":
        # the north_star workload on the same GPU in the same run (BASELINE configs[3] on one
        # GPU: RevNet-50, ImageNet shape, batch 64, J = 8): value, roofline, clocks
        torch.cuda.empty_cache()
        r = measure("revnet50", 8, 64, a.precision, a.steps, a.warmup, 1, 0, local, e2e=False)
        out["north_star_r50"] = {k: r[k] for k in ("workload", "value", "unit", "ms_per_step", "partition_units",
                                                   "roofline", "step_roofline", "clocks", "gpu_launches",
                                                   "stage_ms_per_tick", "kernels", "dtype")}
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        dt, threads = oracle_tick_seconds(a.model, B if a.model != "revnet50" else 4, J, m["partition_units"])
        bb = B if a.model != "revnet50" else 4
        out["cpu_baseline"] = {"value": round(bb / dt, 3), "unit": "samples/s", "cores": threads, "kind": "oracle",
                               "sample": f"one steady-state tick's work (each of the {J} stages: one forward + "
                                         f"one backward / tail step) at batch {bb}, fp64 numpy, {dt:.1f} s",
                               "config1_mlp_seconds": round(mlp_config1_seconds(), 3),
                               "config1": "BASELINE configs[0]: 2-stage reversible MLP, d=64, batch 32, 10 ticks, "
                                          "fp64 oracle, CPU seconds"}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------- reference arm
def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2406_02052_b200 import models as PM
    H, classes = IMAGE[a.model]
    counts = PM.partition(PM.revnet(a.model, H, classes), a.stages, a.batch, H, H, 3)
    bb = 4 if a.model == "revnet50" else 8
    for _ in range(min(a.warmup, 1)):
        oracle_tick_seconds(a.model, bb, a.stages, counts, seed=1)
    tot, threads = 0.0, 1
    for k in range(a.steps):
        dt, threads = oracle_tick_seconds(a.model, bb, a.stages, counts, seed=k)
        tot += dt
    value = bb * a.steps / tot
    sample = (f"per step: one steady-state tick's work (each of the {a.stages} stages one forward + one backward "
              f"/ tail step) at batch {bb} (bounded sample of batch {a.batch}), fp64 numpy oracle")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "samples/s", "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(tot / a.steps * 1e3, 2),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": workload_name(a), "model": a.model, "global_batch": a.batch,
                                        "partition_units": counts},
        "cpu_baseline": {"value": round(value, 4), "unit": "samples/s", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="revnet18", choices=list(IMAGE))
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--stages", type=int, default=4)
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-north-star", dest="north_star", action="store_false",
                    help="skip the RevNet-50 / ImageNet b64 J=8 sub-record (one GPU only)")
    ap.add_argument("--partition", default="", help="units per stage, e.g. 5,4,5,4 (default: FLOP-balanced)")
    a = ap.parse_args()
    # at least one stage per GPU: J = max(--stages, world) (the paper's RevNets have
    # 10-18 units, so J up to 8 always partitions)
    a.stages = max(a.stages, a.gpus)
    if a.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
