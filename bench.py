#!/usr/bin/env python
"""bench.py — aggregate LoRA training tokens/s of the fused multi-LoRA layer on B200.

Contract (see task / DESIGN.md §Measurement):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]
One step = one LoRA training step of the configured layer set over the whole multi-job
token batch (BASELINE.json configs[1] = C2 by default): fwd + bwd of every adapted
projection and the fused per-job AdamW update of every adapter. Rank 0 prints
ONE JSON line. Under torchrun each rank runs one GPU (weak scaling: data-parallel
replicas, adapter-gradient all-reduce over NCCL — the path's only exchange step).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "aggregate LoRA training tokens/sec (all jobs) at 1/2/4/8 B200; tensor-pipe %"
NANO_DEFAULT = 1  # executor nano-batches per step (0 = AIMD every step); see DESIGN.md §5c
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                  "source": "fallback (B200_PROFILING.md)"}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return dict(FALLBACK_PEAKS)


_SAMPLER_SRC = r"""
import sys, time, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByUUID(sys.argv[1].encode())
mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
out = open(sys.argv[2], "w", buffering=1)
while True:
    try:
        out.write("%.3f,%d,%d,%.1f,%d\n" % (time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx,
                  pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                  pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
    except pynvml.NVMLError:
        pass
    time.sleep(0.05)
"""


def workload_config(wl, world: int) -> dict:
    """The benched workload, named identically by both arms (ours and --impl reference) for
    the same workload and N; implementation details go in each line's own keys."""
    return {"workload": f"{wl.name}: {wl.notes}", "layers_per_step": wl.layers,
            "tokens_per_gpu": wl.tokens,
            "jobs": [[j.job_id, j.rank, j.tokens] for j in wl.jobs],
            "projections": [list(p) for p in wl.projections], "parallelism": f"dp{world}",
            "l2": "inputs larger than L2 (X/dY/W per step >> 126 MB)"}

def gpu_energy_mj(device: int):
    """NVML's total-energy counter of this CUDA device (mJ since driver load), or None."""
    try:
        import pynvml
        import torch
        pynvml.nvmlInit()
        uuid = "GPU-" + str(torch.cuda.get_device_properties(device).uuid)
        h = pynvml.nvmlDeviceGetHandleByUUID(uuid.encode())
        return int(pynvml.nvmlDeviceGetTotalEnergyConsumption(h))
    except Exception:
        return None


class ClockSampler:
    """SM clock, power and clock-event (throttle) reasons sampled every ~50 ms from NVML by
    a separate sampler process (so a busy driver thread cannot starve it), started before
    the warm-up so even a short timed region is covered. The GPU is found by the CUDA
    device's UUID. Falls back to `nvidia-smi -lms 200` when NVML is unavailable."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4),
               ("hw_power_brake_slowdown", 0x80))

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.source = None

    def start(self):
        self.out = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)
        self.out.close()
        try:
            import pynvml  # noqa: F401
            import torch
            uuid = "GPU-" + str(torch.cuda.get_device_properties(self.device).uuid)
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER_SRC, uuid, self.out.name],
                                         stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            self.source = "nvml"
            return
        except Exception:
            self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=timestamp,clocks.sm,clocks.max.sm,"
                 "power.draw,clocks_event_reasons.active", "--format=csv,noheader,nounits",
                 "-lms", "200", "-f", self.out.name], stdout=subprocess.DEVNULL,
                stderr=subprocess.DEVNULL)
            self.source = "nvidia-smi"
        except Exception:
            self.proc = None

    def wait_ready(self, timeout_s: float = 20.0):
        """Block until the sampler has written its first sample (bounded)."""
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < timeout_s:
            try:
                if os.path.getsize(self.out.name) > 0:
                    return True
            except OSError:
                pass
            time.sleep(0.05)
        return False

    def stop(self, window=None):
        """window = (t_start, t_end) wall-clock seconds: statistics over the samples taken
        inside it (the settle steps + the timed region); all samples if it holds < 3."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock source"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.out.name) as f:
            for line in f:
                p = [x.strip() for x in line.split(",")]
                try:
                    if self.source == "nvml":
                        ts = float(p[0])
                    else:  # nvidia-smi timestamp "YYYY/MM/DD HH:MM:SS.mmm"
                        import datetime
                        ts = datetime.datetime.strptime(p[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                    rows.append((float(p[1]), float(p[2]), float(p[3]), int(p[4], 0), ts))
                except (ValueError, IndexError):
                    pass
        if os.environ.get("TLORA_CLOCK_DUMP"):  # debugging aid: keep the raw samples
            import shutil
            shutil.copy(self.out.name, os.environ["TLORA_CLOCK_DUMP"])
        os.unlink(self.out.name)
        n_all = len(rows)
        if window is not None:
            inside = [r for r in rows if window[0] <= r[4] <= window[1]]
            if len(inside) >= 3:
                rows = inside
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        pmax = max(r[2] for r in rows)
        loaded = [r for r in rows if r[2] >= 0.5 * pmax]  # under load: >= half peak power
        reasons = sorted({n for r in loaded for n, bit in self.REASONS if r[3] & bit})
        return {"sm_mhz": statistics.median(r[0] for r in loaded),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "power_w_max": round(pmax, 1), "samples": len(rows), "samples_all": n_all,
                "samples_under_load": len(loaded), "source": self.source,
                "window": "settle steps + timed region" if window is not None else "whole run"}


def nvlink_bytes():
    """NVML NVLink data counters of every visible GPU, summed over links (KiB counters x 1024):
    {gpu index: (tx_bytes, rx_bytes)}; {} when NVML or the counters are unavailable. Sampled
    around a timed region, the difference is the NVLink payload that region moved."""
    try:
        import pynvml
        pynvml.nvmlInit()
        out = {}
        ids = [(pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, 0xFFFFFFFF),
               (pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 0xFFFFFFFF)]
        for i in range(pynvml.nvmlDeviceGetCount()):
            h = pynvml.nvmlDeviceGetHandleByIndex(i)
            v = pynvml.nvmlDeviceGetFieldValues(h, ids)
            if v[0].nvmlReturn != 0 or v[1].nvmlReturn != 0:
                continue
            out[i] = (int(v[0].value.ullVal) * 1024, int(v[1].value.ullVal) * 1024)
        return out
    except Exception:
        return {}


def nvlink_delta(before, after, steps):
    if not before or not after:
        return None
    per = {str(i): {"tx_bytes_per_step": (after[i][0] - before[i][0]) / steps,
                    "rx_bytes_per_step": (after[i][1] - before[i][1]) / steps}
           for i in after if i in before}
    return {"source": "NVML NVLINK_THROUGHPUT_DATA_TX/RX, all links, sampled around the timed "
                      "region (every process on the GPUs counts)", "per_gpu": per}


def bind_host_numa(device: int):
    """Pin this process to the CPUs NVML reports as closest to `device` (NVML CPU
    affinity), so the pinned host buffers of the e2e path are first-touched on the GPU's
    own NUMA node and its host->device copies do not cross the inter-socket link."""
    try:
        import pynvml
        import torch
        pynvml.nvmlInit()
        uuid = "GPU-" + str(torch.cuda.get_device_properties(device).uuid)
        h = pynvml.nvmlDeviceGetHandleByUUID(uuid.encode())
        n = (os.cpu_count() + 63) // 64
        words = pynvml.nvmlDeviceGetCpuAffinity(h, n)
        cpus = {64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
        return sorted(cpus)
    except Exception:
        return None


# ------------------------------------------------------------------------------ CPU arm
def cpu_reference_sample(wl, tokens_per_job: int, seconds_budget: float, threads: int):
    """Time the reference CPU implementation of the path on a bounded sample.

    Uses oracle/_ref/ref_bench (the UNMODIFIED reference fused_forward compiled against
    a self-written Eigen-subset header; backward restated with the same GEMM shim, since
    the reference has none) when present, else the oracle port (oracle/liboracle.so).
    Returns dict(value tokens/s, cores, kind, sample) or None.
    """
    return _bench_cpu().measure(wl, tokens_per_job=tokens_per_job, seconds_budget=seconds_budget,
                                threads=threads)


def _bench_cpu():
    """oracle/bench_cpu.py: the CPU baseline leg (lives with the oracle, outside the
    product package; only this leg and the reference arm execute oracle/)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import bench_cpu
    return bench_cpu


def ref_tokens_per_job(wl, threads: int, per_thread: int = 64) -> int:
    """Reference-arm / cpu_baseline sample: >= per_thread tokens per host thread."""
    return max(8, -(-per_thread * threads // len(wl.jobs)))


# ------------------------------------------------------------------------------ GPU arm
def make_comm(local_rank, rank, world, tp_size=1):
    """tlora_comm (NCCL through the C-ABI) for the executor's data-parallel all-reduce: rank 0
    makes the unique id, torch.distributed broadcasts it (host plumbing only)."""
    import ctypes as C
    import torch
    import torch.distributed as dist
    from paper_2602_07263_b200 import capi
    uid = torch.zeros(capi.UNIQUE_ID_BYTES, dtype=torch.uint8, device="cuda")
    if rank == 0:
        buf = (C.c_uint8 * capi.UNIQUE_ID_BYTES)()
        capi.call("tlora_comm_get_unique_id", buf)
        uid.copy_(torch.tensor(list(bytes(buf)), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    idb = (C.c_uint8 * capi.UNIQUE_ID_BYTES)(*uid.cpu().tolist())
    h = C.c_void_p()
    capi.call("tlora_comm_create", local_rank, idb, world, rank, tp_size, C.byref(h))
    return h


def run_executor(args, rank, world, local_rank):
    """Default arm: the C++ step executor (tlora_step_*) — rank-aware nano-batches, AIMD on
    the measured step time (nano 0) or a fixed N, chained fused GEMMs, side-stream
    gradients, masked AdamW, DP all-reduce through the C-ABI communicator, CUDA graphs at
    one replica. Python only builds inputs, times and reports."""
    import ctypes as C
    import torch
    import torch.distributed as dist
    from paper_2602_07263_b200 import capi
    from paper_2602_07263_b200.step import TrainingStep
    from paper_2602_07263_b200.workload import config

    torch.cuda.set_device(local_rank)
    capi.call("tlora_device_check", local_rank, None)
    clocks = ClockSampler(local_rank)
    clocks.start()
    wl = config(args.config)
    if args.layers > 0:
        wl.layers = args.layers
    comm = make_comm(local_rank, rank, world) if world > 1 else None
    st = TrainingStep(wl, device=local_rank, nano_fixed=max(0, args.nano_batches),
                      nano_init=args.nano_init, graphs=not args.no_graph, input_sets=2,
                      comm=comm, sharded_opt=args.dp_sharded_opt and world > 1)
    st.init_random(seed=wl.seed + rank)
    st.enable_optimizer()
    stream = torch.cuda.current_stream()
    clocks.wait_ready()
    for _ in range(args.warmup):
        st.run(stream=stream)
    torch.cuda.synchronize()
    # untimed settle steps (>= 1 s under load); every rank runs the same count
    t_clk0 = time.time()
    en_settle, n_settle = gpu_energy_mj(local_rank), 0
    while True:
        for _ in range(3):
            st.run(stream=stream)
            n_settle += 1
        el = torch.tensor([time.time() - t_clk0], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        if el.item() >= 1.0:
            break
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    lib = capi.lib()
    graph_launches = n_launch = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    traj = []
    nv0 = nvlink_bytes() if world > 1 and rank == 0 else None
    if world > 1:
        dist.barrier()
    e0.record(stream)
    for i in range(args.steps):
        last = i == args.steps - 1 and os.environ.get("TLORA_BENCH_PROF", "1") != "0"
        if last:  # the LAST timed step runs eagerly with CUDA events around every launch
            capi.call("tlora_profile_begin")
        s_ = st.run(eager=last, stream=stream)
        traj.append([s_.nano_used, round(s_.ms, 3) if s_.ms >= 0 else None])
        n_launch += s_.launches  # kernels of the step (a replay counts its captured kernels)
        if s_.replayed_graph:
            graph_launches += 1
    e1.record(stream)
    torch.cuda.synchronize()
    en1, tw1 = gpu_energy_mj(local_rank), time.time()
    if world > 1:
        dist.barrier()
    nvl = nvlink_delta(nv0, nvlink_bytes(), args.steps) if nv0 is not None else None
    energy = None
    if en_settle is not None and en1 is not None and en1 > en_settle:
        # the counter's update granularity is coarse next to a ~0.2 s timed region, so the
        # window is the >= 1 s of settle steps (the same replayed step) + the timed steps
        nst = n_settle + args.steps
        jps = (en1 - en_settle) / 1e3 / nst
        energy = {"joules_per_step": round(jps, 3), "tokens_per_joule": round(wl.tokens / jps, 1),
                  "avg_power_w": round((en1 - en_settle) / 1e3 / max(tw1 - t_clk0, 1e-9), 1),
                  "steps_in_window": nst,
                  "source": "NVML total-energy counter of this rank's GPU over the settle + "
                            "timed steps (host wall clock for the power)"}
    cnt = (C.c_int32 * 6)()
    ms6 = (C.c_double * 6)()
    fl6 = (C.c_double * 6)()
    capi.call("tlora_profile_end", cnt, ms6, fl6)
    t_clk1 = time.time()
    clk = clocks.stop(window=(t_clk0, t_clk1))
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    ms_per_step = ms / args.steps
    tokens = wl.tokens * world
    value = tokens / (ms_per_step / 1e3)

    # ---- one traced step (eager, a timing event after every op): where the step's time goes
    # per stream, and the reference's monitor() reading (nano_pipeline.hpp:114-126) from
    # measured per-nano-batch main-stream spans (t_comp) and comm-stream spans (t_comm)
    step_trace = None
    if os.environ.get("TLORA_BENCH_TRACE", "1") != "0":
        s_ = st.run(stream=stream, trace=True)
        step_trace = trace_summary(st.trace(), s_.ms)

    # ---- the AIMD-driven executor on the same workload (after the timed region): N chosen
    # every step by the reference's controller from the measured step time
    aimd = None
    if args.aimd_steps > 0 and args.nano_batches > 0:
        st.set_controller(0, args.nano_init)
        at = []
        for _ in range(args.aimd_steps):
            s_ = st.run(stream=stream)
            at.append([s_.nano_used, round(s_.ms, 3)])
        tot = sum(m for _, m in at)
        aimd = {"steps": len(at), "trajectory_n_ms": at,
                "tokens_per_s": round(wl.tokens * len(at) / (tot / 1e3), 1),
                "note": "AIMD every step from N=%d (nano_pipeline.hpp:99-112, clamped as "
                        "sim_engine.hpp:314); first visit of each N is eager, then its graph "
                        "replays" % args.nano_init}
        st.set_controller(args.nano_batches)
        st.run(stream=stream)

    # ---- e2e: host pinned inputs -> H2D (copy stream, double-buffered input sets) -> the
    # executor's step on the set -> D2H of every adapter gradient; step i+1's H2D overlaps
    # step i, step i+1 starts after step i's gradients are on the host.
    bind_host_numa(local_rank)
    sets = [list(st.X[s].values()) + list(st.dY[s].values()) for s in range(2)]
    host_in = [t.cpu().pin_memory() for t in sets[0]]
    grads = [g for lay in st.layers.values() for g in lay.packed_grads()]
    host_out = [torch.empty(g.shape, dtype=g.dtype, pin_memory=True) for g in grads]
    h2d = sum(t.numel() * t.element_size() for t in host_in)
    d2h = sum(t.numel() * t.element_size() for t in host_out)
    copy, copy_out = torch.cuda.Stream(), torch.cuda.Stream()

    def e2e_run(nsteps):
        done = [torch.cuda.Event() for _ in range(nsteps)]
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_out = None
        with torch.cuda.stream(copy):
            for h, d in zip(host_in, sets[0]):
                d.copy_(h, non_blocking=True)
            ev_in[0].record(copy)
        for i in range(nsteps):
            s = i % 2
            stream.wait_event(ev_in[s])
            if ev_out is not None:
                stream.wait_event(ev_out)  # grads of step i-1 are on the host before reuse
            with torch.cuda.stream(copy):  # next step's inputs, while this step runs
                if i + 1 < nsteps:
                    if i >= 1:
                        copy.wait_event(done[i - 1])  # set (i+1)%2 was last read by step i-1
                    for h, d in zip(host_in, sets[(i + 1) % 2]):
                        d.copy_(h, non_blocking=True)
                    ev_in[(i + 1) % 2].record(copy)
            st.run(input_set=s, stream=stream)
            done[i].record(stream)
            with torch.cuda.stream(copy_out):
                copy_out.wait_event(done[i])
                for g, h in zip(grads, host_out):
                    h.copy_(g, non_blocking=True)
                ev_out = torch.cuda.Event()
                ev_out.record(copy_out)
        stream.wait_event(ev_out)

    e2e_run(2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(2, min(args.steps, 10))
    f0.record(stream)
    e2e_run(e2e_steps)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.item()

    roofline = roofline_block(cnt, ms6, fl6, "CUDA-event brackets around every launch of the "
                              "LAST timed step (eager, same kernels as the replayed graph); "
                              "per-launch durations of that step")
    cpu = cpu_f32 = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        tpj = args.cpu_tokens_per_job or ref_tokens_per_job(wl, threads)
        cpu = cpu_reference_sample(wl, tokens_per_job=tpj, seconds_budget=args.cpu_seconds,
                                   threads=threads)
        cpu_f32 = _bench_cpu().measure_oracle_f32(wl, tokens_per_job=tpj,
                                                  seconds_budget=min(10.0, args.cpu_seconds),
                                                  threads=threads)
    flops_step = wl.flops_fwd_bwd() * world
    nano_desc = (f"fixed N={args.nano_batches} (the reference's config.fixed_n)"
                 if args.nano_batches > 0 else
                 f"AIMD every step from N={args.nano_init} (nano_pipeline.hpp:99-112, "
                 "sim_engine.hpp:306-315)")
    return {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded normal activations/grads, random-init W and adapters)",
        "config": workload_config(wl, world),
        "run": {"driver": "C++ step executor (tlora_step_run: libtlora.so)",
                   "nano_batches": nano_desc, "aimd_trajectory_n_ms": traj,
                   "trajectory_note": "per timed step [N used, the library's own event time of "
                                      "its latest completed step]; null = with a fixed N the "
                                      "host runs ahead and no step had completed yet",
                   "dp_allreduce": None if world == 1 else (
                       "sharded optimizer: per key reduce-scatter (fp32) -> AdamW on this rank's "
                       "packed-row shard -> all-gather (bf16 operands), nccl via tlora_comm"
                       if args.dp_sharded_opt else
                       "nccl all-reduce via tlora_comm (C-ABI), per key after its last "
                       "nano-batch, on the executor's comm stream"),
                   "cuda_graph": not args.no_graph and world == 1,
                   "graph_replays_timed": graph_launches,
                   "algorithmic_tflop_per_step": round(flops_step / 1e12, 3),
                   "achieved_tflops_step": round(flops_step / (ms_per_step / 1e3) / 1e12, 1)},
        "e2e": {"value": round(tokens / (e2e_ms / 1e3), 1), "unit": "tokens/s",
                "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "h2d_gb_per_s": round(h2d / (e2e_ms / 1e3) / 1e9, 2),
                "bound": "PCIe host->device (raw pinned copy ~55.5 GB/s, tools/pcie_probe.py)",
                "path": "host pinned inputs -> H2D into the executor's input set -> "
                        "tlora_step_run -> D2H of the adapter gradients (H2D of step i+1 "
                        "overlapped with step i)"},
        "gpu_launches": n_launch,
        "roofline": roofline,
        "aimd": aimd,
        "step_trace": step_trace,
        "nvlink": nvl,
        "cpu_baseline": cpu,
        "cpu_baseline_oracle_f32": cpu_f32,
        "energy": energy,
        "clocks": clk,
    }


def trace_summary(trace, step_ms):
    """Per-stream end times of a traced executor step and monitor()'s reading from measured
    per-nano-batch spans: t_comp[i] = main-stream span of nano-batch i, t_comm[i] = span of
    its comm-stream ops (0 for one replica)."""
    from paper_2602_07263_b200 import capi
    from paper_2602_07263_b200.layer import monitor
    ends = {}
    for op, ms in trace:
        ends[op["stream"]] = max(ends.get(op["stream"], 0.0), ms)
    nanos = sorted({op["nano"] for op, _ in trace if op["nano"] >= 0})
    t_comp, t_comm, prev = [], [], 0.0
    for i in nanos:
        main = [ms for op, ms in trace if op["nano"] == i and op["stream"] == capi.STREAM_MAIN]
        comm = [ms for op, ms in trace if op["nano"] == i and op["stream"] == capi.STREAM_COMM]
        end = max(main) if main else prev
        t_comp.append((end - prev) / 1e3)
        t_comm.append(((max(comm) - end) if comm and max(comm) > end else 0.0) / 1e3)
        prev = end
    analytic = max(sum(t_comp), sum(t_comm))
    eta, stall = monitor(t_comp, t_comm, step_ms / 1e3, analytic, num_stages=1)
    names = {capi.STREAM_MAIN: "main", capi.STREAM_SIDE: "side", capi.STREAM_COMM: "comm"}
    return {"step_ms": round(step_ms, 3),
            "stream_end_ms": {names[k]: round(v, 3) for k, v in sorted(ends.items())},
            "t_comp_ms": [round(x * 1e3, 3) for x in t_comp],
            "t_comm_ms": [round(x * 1e3, 3) for x in t_comm],
            "monitor": {"eta_util": round(eta, 4), "delta_stall_ms": round(stall * 1e3, 3)},
            "note": "eager traced step (an event after every op); the step ends on the main "
                    "stream after the side / comm streams"}


GEMM_SOURCES = ("lora_gemm2.cuh", "lora_gemm.cuh", "sm100_ptx.cuh", "tlora_plan.hpp")


def gemm_sources_sha():
    """sha256 over the fused GEMM's kernel + plan sources (ties profiles/traffic.json's ncu
    capture to the kernel that runs now)."""
    import hashlib
    h = hashlib.sha256()
    for f in GEMM_SOURCES:
        h.update((ROOT / "paper_2602_07263_b200" / "csrc" / f).read_bytes())
    return h.hexdigest()


def traffic_info():
    """(traffic, algorithmic, source) of the fused GEMM from the committed ncu capture."""
    tp = ROOT / "profiles" / "traffic.json"
    if not tp.exists():
        return None, None, "no capture"
    try:
        tj = json.loads(tp.read_text())
    except Exception:
        return None, None, "unreadable profiles/traffic.json"
    src = "profiles/traffic.json (ncu dram bytes, mean per fused-GEMM launch"
    if tj.get("commit"):
        src += f", captured at commit {tj['commit']}"
    if tj.get("gemm_sources_sha256"):
        same = tj["gemm_sources_sha256"] == gemm_sources_sha()
        src += ("; GEMM kernel sources identical to this build" if same else
                "; GEMM kernel sources CHANGED since the capture")
    return (tj.get("dram_bytes_per_launch_mean", tj.get("fwd_bytes_per_launch")),
            tj.get("algorithmic_bytes_per_launch_mean"), src + ")")


def roofline_block(cnt, ms6, fl6, timing):
    """Roofline of the dominant kernel family (the fused base+LoRA GEMM: fwd + dX) from the
    live per-launch CUDA-event times and algorithmic FLOPs of one step."""
    from paper_2602_07263_b200 import capi
    peaks = load_peaks()
    fam_ms = ms6[capi.L_FWD] + ms6[capi.L_DX]
    fam_fl = fl6[capi.L_FWD] + fl6[capi.L_DX]
    achieved = fam_fl / (fam_ms / 1e3) / 1e12 if fam_ms > 0 else 0.0
    peak = float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
    total_ms = sum(ms6)
    names = list(capi.LAUNCH_NAMES)
    if cnt[capi.L_DA] == 0 and cnt[capi.L_DB] > 0:
        names[capi.L_DB] = "dB+dA (one launch)"
    per_launch = {names[i]: {
        "launches": cnt[i], "ms_total": round(ms6[i], 3),
        "tflops": round(fl6[i] / (ms6[i] / 1e3) / 1e12, 1) if ms6[i] > 0 else None,
        "share_of_gemm_time": round(ms6[i] / total_ms, 4) if total_ms > 0 else None}
        for i in range(6)}
    traffic, traffic_alg, traffic_src = traffic_info()
    return {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak,
            "unit": "TFLOP/s", "frac": round(achieved / peak, 4) if peak else None,
            "frac_of_burst": round(achieved / float(peaks["bf16_tflops"]), 4),
            "timing": timing, "traffic": traffic, "traffic_algorithmic_bytes": traffic_alg,
            "traffic_source": traffic_src,
            "kernel": "lora_gemm2_kernel (2-CTA fused base+LoRA GEMM: fwd + dX)",
            "peak_source": peaks["source"] + " sustained bf16", "per_launch": per_launch}


def run_cpp_host(args):
    """--host cpp: the pure C++ host (tests/cpp/_build/step_main: LayerSetTrainer over the
    C-ABI, no Python in the loop) prints its own BENCH-format line; add clocks around it."""
    import torch
    binp = ROOT / "tests" / "cpp" / "_build" / "step_main"
    if not binp.exists():
        subprocess.run(["make", "-C", str(ROOT), "tests/cpp/_build/step_main"], check=True)
    clocks = ClockSampler(0)
    clocks.start()
    clocks.wait_ready()
    t0 = time.time()
    p = subprocess.run([str(binp), "bench", args.config, str(args.steps), str(args.warmup),
                        str(max(0, args.nano_batches)), str(max(0, args.layers))],
                       capture_output=True, text=True, check=True)
    clk = clocks.stop(window=(t0, time.time()))
    out = json.loads(p.stdout.strip().splitlines()[-1])
    out["clocks"] = clk
    out["gpu_launches"] = None
    return out


def run_ours(args, rank, world, local_rank):
    """--driver python: round 1's Python per-launch driver (runner.LayerSetStep), kept as the
    executor's bitwise cross-check and for the shuffled / overlap experiments."""
    import torch
    import torch.distributed as dist
    from paper_2602_07263_b200 import capi
    from paper_2602_07263_b200.runner import LayerSetStep
    from paper_2602_07263_b200.workload import config
    import ctypes as C

    torch.cuda.set_device(local_rank)
    capi.call("tlora_device_check", local_rank, None)
    # the sampler process needs a few seconds to come up: start it before building the
    # layer set so it is sampling well before the warm-up / settle / timed steps
    clocks = ClockSampler(local_rank)
    clocks.start()
    wl = config(args.config)
    if args.layers > 0:  # e.g. one layer of C4's 64-layer stack on a single GPU
        wl.layers = args.layers
    step = LayerSetStep(wl, device=local_rank, seed=wl.seed + rank, shuffle=args.shuffle,
                        chain=not args.no_chain and args.overlap == 0)
    step.enable_optimizer()
    if os.environ.get("TLORA_SIDE_GRADS", "1") == "1" and step.chain:
        step.enable_side_grads()
        g_sms = int(os.environ.get("TLORA_GRAD_SMS", "0"))
        if g_sms > 0:  # experiment knob: GEMMs on (SMs - g), gradients on g (measured much
            # slower: 8 / 16 / 24 SMs -> 14.5 / 12.5 / 12.2 ms vs 10.87 ms per C2 step)
            total = torch.cuda.get_device_properties(local_rank).multi_processor_count
            capi.call("tlora_set_sm_budget", local_rank, total - g_sms, g_sms)
    if args.overlap != 0:
        step.enable_overlap(args.overlap)
    stream = torch.cuda.current_stream()

    comm_stream = torch.cuda.Stream() if world > 1 else None
    pending = []

    bucket_at_end = os.environ.get("TLORA_DP_BUCKET", "per_layer") == "end"
    # DP gradient all-reduce by copy-engine push (paper_2602_07263_b200/dp.py), opt-in with
    # TLORA_DP_CE=1 (NCCL's ring stays the default; A/B in profiles/r1c_summary.md).
    # Skipped when its double-buffered slots would exceed 24 GB per GPU.
    push_ar = None
    if world > 1 and not bucket_at_end and os.environ.get("TLORA_DP_CE", "0") == "1":
        sizes = {key: sum(g.numel() for g in lay.packed_grads()) for key, lay in step.layers.items()}
        if 2 * 2 * 4 * sum(sizes.values()) <= (24 << 30):
            from paper_2602_07263_b200.dp import PushAllReduce
            push_ar = PushAllReduce(world, rank, local_rank)
            for key, n in sizes.items():
                push_ar.register(key, n)

    def allreduce_grads(name, layer, ready=None):
        if bucket_at_end:
            return
        # DP replicas: all-reduce this projection's packed fp32 adapter grads on a comm
        # stream while the next projection's backward runs.
        ev = ready
        if ev is None:
            ev = torch.cuda.Event()
            ev.record(stream)
        with torch.cuda.stream(comm_stream):
            comm_stream.wait_event(ev)
            dAT, dB = layer.packed_grads()
            if push_ar is not None:
                push_ar.allreduce(name, [dAT, dB], comm_stream)
                works = []
            else:
                works = [dist.all_reduce(dAT, async_op=True), dist.all_reduce(dB, async_op=True)]
            pending.extend(works)
            if opt_inline:  # this projection's AdamW right after its all-reduce, overlapping
                for w in works:  # the rest of the backward (comm stream waits, host does not)
                    w.wait()
                layer.optimizer_step(1.0 / world, stream=comm_stream)

    # DP: per-projection AdamW on the comm stream after that projection's all-reduce (knob;
    # bitwise-identical adapters, no measurable gain at DP2: 2.88 M vs 2.90 M tokens/s)
    opt_inline = world > 1 and not bucket_at_end and os.environ.get("TLORA_DP_OPT_INLINE", "0") == "1"
    flat_grads = None
    if world > 1 and bucket_at_end:
        flat_grads = [g for lay in step.layers.values() for g in lay.packed_grads()]

    def fwd():
        if args.overlap != 0:
            step.forward_overlapped(stream)
        else:
            step.forward(stream)

    def bwd():
        cb = allreduce_grads if world > 1 else None
        if push_ar is not None:
            push_ar.next_step()
        if args.overlap != 0:
            step.backward_overlapped(stream, on_layer_done=cb)
        else:
            step.backward(stream, on_layer_done=cb)

    graph = graph_prof = None
    used_graph = False
    if not args.no_graph and world == 1 and args.overlap == 0:
        try:
            # Two captures of the same step: a plain one, and one with CUDA-event nodes
            # around every launch (the live per-launch timing). The LAST timed step replays
            # the profiled graph, so the roofline's kernel durations come from inside the
            # timed region while the event nodes (~3 us each, and they break the PDL chain)
            # cost only 1/K of it. TLORA_BENCH_PROF=0 skips the profiled graph.
            graph = step.capture(warmup=1, profile=False)
            if os.environ.get("TLORA_BENCH_PROF", "1") != "0":
                graph_prof = step.capture(warmup=0, profile=True)
            used_graph = True
        except Exception as e:  # same kernels, launched eagerly instead
            print(f"[bench] CUDA-graph capture failed, running eagerly: {e}", file=sys.stderr)
            torch.cuda.synchronize()
            graph = graph_prof = None

    def one_step(last=False):
        # training step: fwd + bwd (+ DP all-reduce) + fused multi-job AdamW of all adapters
        if graph is not None:
            (graph_prof if last and graph_prof is not None else graph).replay()
            return
        fwd()
        if world == 1 and args.overlap == 0:
            step.backward_and_update(stream)
            return
        bwd()
        if flat_grads is not None:
            for g in flat_grads:
                dist.all_reduce(g)
        if world > 1:
            for w in pending:
                w.wait()
            pending.clear()
            stream.wait_stream(comm_stream)
        if not opt_inline:
            step.optimizer_step(stream, grad_scale=1.0 / world)

    clocks.wait_ready()
    for i in range(args.warmup):
        one_step(last=i == args.warmup - 1)  # the profiled graph is uploaded / warm too
    torch.cuda.synchronize()
    # untimed settle steps for >= 1 s of wall time: clocks settle under load and get
    # sampled. Every rank must run the SAME number of steps (each DP step issues
    # collectives; a per-rank time-based loop deadlocked), so steps run in chunks and the
    # ranks agree after each chunk (MAX of elapsed time) whether to run another.
    t_clk0 = time.time()
    chunk = 3
    while True:
        for _ in range(chunk):
            one_step()
        torch.cuda.synchronize()
        el = torch.tensor([time.time() - t_clk0], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        if el.item() >= 1.0:
            break
    if world > 1:
        dist.barrier()

    lib = capi.lib()
    n0 = lib.tlora_launch_count()
    if graph is None:  # (graph mode: profiling was armed at capture time)
        capi.call("tlora_profile_begin")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        one_step(last=i == args.steps - 1)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n_launch = lib.tlora_launch_count() - n0
    if graph is not None:  # replays bypass the host-side counter: count the captured kernels
        n_launch = step.graph_launches * args.steps
    cnt = (C.c_int32 * 6)()
    ms6 = (C.c_double * 6)()
    fl6 = (C.c_double * 6)()
    capi.call("tlora_profile_end", cnt, ms6, fl6)
    if graph is not None:
        # the captured brackets hold the LAST replayed step of the timed region; scale to K
        for i in range(6):
            cnt[i] *= args.steps
            ms6[i] *= args.steps
            fl6[i] *= args.steps
        graph = graph_prof = None  # event nodes reference events released by profile_end
        step.graph = None
    t_clk1 = time.time()
    clk = clocks.stop(window=(t_clk0, t_clk1))
    if os.environ.get("TLORA_CLOCK_DUMP"):
        print(f"[bench] clock window {t_clk0:.3f} .. {t_clk1:.3f}", file=sys.stderr)
    if os.environ.get("TLORA_BENCH_CHECKSUM") and rank == 0:  # debugging aid: schedule
        tot = 0.0                                             # variants must agree bitwise
        for lay in step.layers.values():
            for s_ in range(len(wl.jobs)):
                A, B = lay.read_adapter(s_)
                tot += float(A.double().sum()) + float(B.double().abs().sum())
        print(f"[bench] adapter checksum {tot!r}", file=sys.stderr)
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    ms_per_step = ms / args.steps
    tokens = wl.tokens * world
    value = tokens / (ms_per_step / 1e3)

    # ---- e2e: the same step through the public API with HOST buffers: every step, H2D of
    # all its inputs (activations + upstream grads) from pinned memory and D2H of the
    # adapter gradients. Inputs are double-buffered on a copy stream so the H2D of step i+1
    # overlaps the compute of step i; step i+1's backward waits for the D2H of step i.
    dev_sets = step.make_input_sets(2)
    bind_host_numa(local_rank)  # pinned host buffers on the GPU's own NUMA node
    host_in = [t.cpu().pin_memory() for t in dev_sets[0]]
    grads = [g for lay in step.layers.values() for g in lay.packed_grads()]
    host_out = [torch.empty(g.shape, dtype=g.dtype, pin_memory=True) for g in grads]
    h2d = sum(t.numel() * t.element_size() for t in host_in)
    d2h = sum(t.numel() * t.element_size() for t in host_out)
    copy = torch.cuda.Stream()
    copy_out = torch.cuda.Stream()  # D2H on its own stream: PCIe is full duplex, so the
                                    # gradient read-back overlaps the next step's H2D

    def e2e_run(nsteps):
        done = [torch.cuda.Event() for _ in range(nsteps)]
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_out = None
        with torch.cuda.stream(copy):
            for h, d in zip(host_in, dev_sets[0]):
                d.copy_(h, non_blocking=True)
            ev_in[0].record(copy)
        for i in range(nsteps):
            s = i % 2
            stream.wait_event(ev_in[s])
            step.use_inputs(s)
            fwd()
            if ev_out is not None:
                stream.wait_event(ev_out)  # grads of step i-1 are on the host before reuse
            if world == 1 and args.overlap == 0:
                step.backward_and_update(stream)
            else:
                bwd()
                if world > 1:
                    for w in pending:
                        w.wait()
                    pending.clear()
                    stream.wait_stream(comm_stream)
                if not opt_inline:
                    step.optimizer_step(stream, grad_scale=1.0 / world)
            done[i].record(stream)
            with torch.cuda.stream(copy):
                if i + 1 < nsteps:
                    if i >= 1:
                        copy.wait_event(done[i - 1])  # set (i+1)%2 was last read by step i-1
                    for h, d in zip(host_in, dev_sets[(i + 1) % 2]):
                        d.copy_(h, non_blocking=True)
                    ev_in[(i + 1) % 2].record(copy)
            with torch.cuda.stream(copy_out):
                copy_out.wait_event(done[i])
                for g, h in zip(grads, host_out):
                    h.copy_(g, non_blocking=True)
                ev_out = torch.cuda.Event()
                ev_out.record(copy_out)
        stream.wait_event(ev_out)

    e2e_run(2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(2, min(args.steps, 10))
    f0.record(stream)
    e2e_run(e2e_steps)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / e2e_steps
    step.use_inputs(0)
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.item()

    # ---- roofline of the dominant kernel family: the fused base+LoRA GEMM (fwd and dX)
    peaks = load_peaks()
    fam_ms = ms6[capi.L_FWD] + ms6[capi.L_DX]
    fam_fl = fl6[capi.L_FWD] + fl6[capi.L_DX]
    achieved = fam_fl / (fam_ms / 1e3) / 1e12 if fam_ms > 0 else 0.0
    peak = float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
    total_ms = sum(ms6)
    names = list(capi.LAUNCH_NAMES)
    if cnt[capi.L_DA] == 0 and cnt[capi.L_DB] > 0:
        names[capi.L_DB] = "dB+dA (one launch)"
    per_launch = {names[i]: {
        "launches": cnt[i], "ms_total": round(ms6[i], 3),
        "tflops": round(fl6[i] / (ms6[i] / 1e3) / 1e12, 1) if ms6[i] > 0 else None,
        "share_of_gemm_time": round(ms6[i] / total_ms, 4) if total_ms > 0 else None}
        for i in range(6)}
    traffic, traffic_alg, traffic_src = traffic_info()
    roofline = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak,
                "unit": "TFLOP/s", "frac": round(achieved / peak, 4) if peak else None,
                "frac_of_burst": round(achieved / float(peaks["bf16_tflops"]), 4),
                "timing": ("CUDA-event brackets captured in a second graph of the step, replayed "
                           "as the LAST timed step; per-launch durations of that step x steps") if used_graph else
                          "CUDA-event brackets around every launch of the timed region",
                "traffic": traffic, "traffic_algorithmic_bytes": traffic_alg,
                "traffic_source": traffic_src,
                "kernel": "lora_gemm2_kernel (2-CTA fused base+LoRA GEMM: fwd + dX)",
                "peak_source": peaks["source"] + " sustained bf16", "per_launch": per_launch}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        cpu = cpu_reference_sample(wl, tokens_per_job=args.cpu_tokens_per_job or
                                   ref_tokens_per_job(wl, threads),
                                   seconds_budget=args.cpu_seconds, threads=threads)

    flops_step = wl.flops_fwd_bwd() * world
    out = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded normal activations/grads, random-init W and adapters)",
        "config": {"workload": f"{wl.name}: {wl.notes}", "layers_per_step": wl.layers,
                   "tokens_per_gpu": wl.tokens,
                   "jobs": [[j.job_id, j.rank, j.tokens] for j in wl.jobs],
                   "projections": wl.projections, "token_order": ("shuffled" + (" (gathered plan)" if step.gathered else " (plain plan)"))
                   if args.shuffle else "job-contiguous",
                   "parallelism": f"dp{world}", "lowrank_side_stream_sms": args.overlap,
                   "dp_allreduce": (None if world == 1 else
                                    "copy-engine push + stream flags" if push_ar is not None
                                    else "nccl"),
                   "dp_sm_reserve": os.environ.get("TLORA_SM_RESERVE") if world > 1 else None,
                   "nccl_max_nchannels": os.environ.get("NCCL_MAX_NCHANNELS") if world > 1 else None,
                   "cuda_graph": used_graph, "chained_lowrank": step.chain,
                   "l2": "inputs larger than L2 (X/dY/W per step >> 126 MB)",
                   "algorithmic_tflop_per_step": round(flops_step / 1e12, 3),
                   "achieved_tflops_step": round(flops_step / (ms_per_step / 1e3) / 1e12, 1)},
        "e2e": {"value": round(tokens / (e2e_ms / 1e3), 1), "unit": "tokens/s",
                "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "h2d_gb_per_s": round(h2d / (e2e_ms / 1e3) / 1e9, 2),
                "bound": "PCIe host->device (raw pinned copy ~55.5 GB/s, tools/pcie_probe.py)",
                "path": "host pinned inputs -> tlora C-ABI fwd/bwd -> host grads (D2H on its "
                        "own stream; H2D of step i+1 overlapped with compute of step i)"},
        "gpu_launches": int(n_launch),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    return out


def run_tp(args, rank, world, local_rank):
    """Tensor-parallel layer set: one layer of the configured model split over
    the TP group, per-nano-batch all-gather / reduce-scatter on a comm stream overlapped
    with the GEMMs; N chosen online by AIMD during warm-up, then frozen for timing.
    Strong scaling: the global token batch is fixed, value = global tokens / step time."""
    import torch
    import torch.distributed as dist
    from paper_2602_07263_b200 import capi
    from paper_2602_07263_b200.tp import TPLayerSetStep
    from paper_2602_07263_b200.workload import config

    torch.cuda.set_device(local_rank)
    wl = config(args.config)
    spec = args.fused_rs
    if spec == "auto":  # fused GEMM + reduce-scatter is the default at TP > 1 (measured
        spec = "o,down" if world > 1 else ""  # 1-3% faster than NCCL at TP2 / TP4)
    fused = [p for p in spec.split(",") if p and p != "none"]
    st = TPLayerSetStep(wl, rank, world, local_rank, nano=args.nano, fused_rs=fused)
    st.enable_optimizer()
    stream = torch.cuda.current_stream()
    clocks = ClockSampler(local_rank)
    clocks.start()
    trajectory = []

    seen = set()

    def timed_step(n):
        st.plans(n)  # host-side plan construction for a new N happens outside the timing
        if n not in seen:  # and so do first-use costs (workspace growth, buffers) of a new N
            st.step(n)
            seen.add(n)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st.step(n)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    for _ in range(args.warmup):
        timed_step(st.n)
    if args.aimd_steps > 0:
        best = (float("inf"), st.n)
        for _ in range(args.aimd_steps):
            n = st.n
            ms = timed_step(n)
            trajectory.append([n, round(ms, 3)])
            best = min(best, (ms, n))
            st.adapt(ms / 1e3)  # identical on all ranks (times are max-reduced)
        st.n = best[1]
    dist.barrier()
    torch.cuda.synchronize()
    lib = capi.lib()
    n0 = lib.tlora_launch_count()
    nv0 = nvlink_bytes() if rank == 0 else None
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    step_ev = os.environ.get("TLORA_BENCH_STEP_EVENTS") == "1"  # diagnostic: per-step spans
    evs = []
    for _ in range(args.steps):
        if step_ev:
            evs.append(torch.cuda.Event(enable_timing=True))
            evs[-1].record(stream)
        st.step(st.n)
    e1.record(stream)
    torch.cuda.synchronize()
    if step_ev:
        spans = [a.elapsed_time(b) for a, b in zip(evs, evs[1:] + [e1])]
        print(f"[rank {rank}] caller-stream step spans ms (N={st.n}): "
              f"{[round(x, 3) for x in spans]}", file=sys.stderr, flush=True)
    dist.barrier()
    nvl = nvlink_delta(nv0, nvlink_bytes(), args.steps) if rank == 0 else None
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = t.item() / args.steps
    flops = wl.flops_fwd_bwd() / wl.layers
    value = wl.tokens / (ms_per_step / 1e3)
    n_launch = int(lib.tlora_launch_count() - n0)
    # one extra step with every launch bracketed by CUDA events (after the timed region):
    # where this rank's step time goes, and the fused GEMM family's achieved TFLOP/s
    import ctypes as C
    capi.call("tlora_profile_begin")
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    st.step(st.n)
    e3.record(stream)
    torch.cuda.synchronize()
    cnt, ms6, fl6 = (C.c_int32 * 6)(), (C.c_double * 6)(), (C.c_double * 6)()
    capi.call("tlora_profile_end", cnt, ms6, fl6)
    prof_ms = e2.elapsed_time(e3)
    # one traced step: per nano-batch compute / boundary-traffic intervals -> the reference's
    # PipelineTrace and monitor() reading (nano_pipeline.hpp:28-34, 114-126), measured
    st.enable_trace(True)
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e4.record(stream)
    st.step(st.n)
    e5.record(stream)
    torch.cuda.synchronize()
    reading = st.trace_reading(e4.elapsed_time(e5))
    st.enable_trace(False)
    reading = {k: (round(v, 6) if isinstance(v, float) else [round(x, 6) for x in v])
               for k, v in reading.items()}
    fam_ms, fam_fl = ms6[capi.L_FWD] + ms6[capi.L_DX], fl6[capi.L_FWD] + fl6[capi.L_DX]
    peaks = load_peaks()
    peak = float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
    ach = fam_fl / (fam_ms / 1e3) / 1e12 if fam_ms > 0 else 0.0
    roofline = {"bound": "tensor", "achieved": round(ach, 1), "peak": peak, "unit": "TFLOP/s",
                "frac": round(ach / peak, 4) if peak else None,
                "kernel": "lora_gemm2_kernel (fused GEMM fwd + dX, per rank, this rank's shards)",
                "timing": "CUDA-event brackets of one extra profiled step after the timed region",
                "gemm_share_of_profiled_step": round(fam_ms / prof_ms, 4) if prof_ms else None,
                "per_launch": {capi.LAUNCH_NAMES[i]: {"launches": cnt[i], "ms": round(ms6[i], 3)}
                               for i in range(6)}}
    return {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded normal activations/grads, random-init W and adapters)",
        "config": {"workload": f"{wl.name}: {wl.notes} (one layer of the stack per step)",
                   "tokens_global": wl.tokens, "parallelism": f"tp{world}",
                   "row_parallel_reduce_scatter": {p: ("fused GEMM epilogue -> NVLink peer "
                                                       "slots" if p in fused else "NCCL")
                                                   for p in ("o", "down")},
                   "nano_batches": st.n, "aimd_trajectory_n_ms": trajectory,
                   "algorithmic_tflop_per_step": round(flops / 1e12, 3),
                   "achieved_tflops_aggregate": round(flops / (ms_per_step / 1e3) / 1e12, 1),
                   "achieved_tflops_per_gpu": round(flops / world / (ms_per_step / 1e3) / 1e12, 1)},
        "gpu_launches": n_launch,
        "roofline": roofline,
        "pipeline_monitor": reading,
        "nvlink": nvl,
        "clocks": clk,
    }


def run_tp_exec(args, rank, world, local_rank):
    """Tensor-parallel layer set through the C++ TP step (tlora_tp_*): one layer of the
    configured model (C4 by default) split over the torchrun group, per-nano-batch
    copy-engine all-gathers / reduce-scatters and the fused GEMM + reduce-scatter over
    NVLink, N chosen by AIMD every step (--nano-batches 0) or fixed. Strong scaling: the
    global token batch is fixed, value = global tokens / step time (max over ranks)."""
    import torch
    import torch.distributed as dist
    from paper_2602_07263_b200 import capi
    from paper_2602_07263_b200.tp_step import TPExecutor
    from paper_2602_07263_b200.workload import config

    torch.cuda.set_device(local_rank)
    wl = config(args.config)
    comm = make_comm(local_rank, rank, world, tp_size=world)
    # TP default: AIMD every step (the nano-batches hide the boundary traffic); an explicit
    # --nano-batches N pins N
    nano_fixed = max(0, args.nano_batches) if "--nano-batches" in sys.argv else 0
    args.nano_batches = nano_fixed
    ex = TPExecutor(wl, rank, world, local_rank, comm, nano_fixed=nano_fixed,
                    nano_init=args.nano, fused_rs=args.fused_rs != "none",
                    copy_engine=os.environ.get("TLORA_TP_CE_AG", "1") != "0")
    ex.enable_optimizer()
    stream = torch.cuda.current_stream()
    clocks = ClockSampler(local_rank)
    clocks.start()
    clocks.wait_ready()
    # AIMD every step: a nano-batch count used for the first time builds its layout (plans,
    # split-K scratch) on the host, so settle untimed until the controller's cycle is warm
    settle = args.warmup if nano_fixed > 0 else max(args.warmup, 12)
    for _ in range(settle):
        ex.run(stream)
    torch.cuda.synchronize()
    nv0 = nvlink_bytes() if rank == 0 else None  # (host-side NVML reads: before the barrier)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    traj, launches = [], 0
    e0.record(stream)
    trace_all = os.environ.get("TLORA_TP_TRACE_ALL") == "1"  # diagnostic: trace every step
    step_ev = os.environ.get("TLORA_BENCH_STEP_EVENTS") == "1"  # diagnostic: per-step spans
    evs = []
    for _ in range(args.steps):
        if step_ev:
            evs.append(torch.cuda.Event(enable_timing=True))
            evs[-1].record(stream)
        s_ = ex.run(stream, trace=trace_all)
        traj.append([s_.nano_used, round(s_.ms, 3) if s_.ms >= 0 else None])
        launches += s_.launches
    e1.record(stream)
    torch.cuda.synchronize()
    if step_ev:
        spans = [a.elapsed_time(b) for a, b in zip(evs, evs[1:] + [e1])]
        print(f"[rank {rank}] caller-stream step spans ms: {[round(x, 3) for x in spans]}",
              file=sys.stderr, flush=True)
    dist.barrier()
    nvl = nvlink_delta(nv0, nvlink_bytes(), args.steps) if rank == 0 else None
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = t.item() / args.steps
    flops = wl.flops_fwd_bwd() / wl.layers
    # one traced step after the timed region: the reference's PipelineTrace / monitor()
    # (nano_pipeline.hpp:28-34, 114-126) from measured per-nano-batch spans
    from paper_2602_07263_b200.layer import monitor
    s_ = ex.run(stream, trace=True)
    comp, comm_ms = ex.trace()
    t_it = s_.ms / 1e3
    t_an = max(sum(comp), sum(comm_ms)) / 1e3
    eta, stall = monitor([c / 1e3 for c in comp], [c / 1e3 for c in comm_ms], t_it, t_an, 1)
    reading = {"t_comp_s": [round(c / 1e3, 6) for c in comp],
               "t_comm_s": [round(c / 1e3, 6) for c in comm_ms], "t_iter_event_s": round(t_it, 6),
               "t_iter_analytic_s": round(t_an, 6), "eta_util": round(eta, 6),
               "delta_stall_s": round(stall, 6)}
    return {
        "metric": METRIC, "value": round(wl.tokens / (ms_per_step / 1e3), 1), "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded normal activations/grads, random-init W and adapters)",
        "config": {"workload": f"{wl.name}: {wl.notes} (one layer of the stack per step)",
                   "tokens_global": wl.tokens, "parallelism": f"tp{world}",
                   "driver": "C++ tensor-parallel step (tlora_tp_run: libtlora.so)",
                   "row_parallel_reduce_scatter": "fused GEMM epilogue -> NVLink peer slots"
                   if args.fused_rs != "none" else "copy engine / NCCL",
                   "nano_batches": ("AIMD every step" if args.nano_batches <= 0
                                    else f"fixed N={args.nano_batches}"),
                   "aimd_trajectory_n_ms": traj, "untimed_steps_before_timing": settle,
                   "trajectory_note": "per timed step [N used, the library's own event time of "
                                      "its latest completed step]; null = with a fixed N the "
                                      "host runs ahead and no step had completed yet",
                   "algorithmic_tflop_per_step": round(flops / 1e12, 3),
                   "achieved_tflops_aggregate": round(flops / (ms_per_step / 1e3) / 1e12, 1)},
        "gpu_launches": int(launches),
        "pipeline_monitor": reading,
        "nvlink": nvl,
        "clocks": clk,
    }


def run_reference(args, rank, world):
    """Reference arm: the reference's own CPU implementation of the path (oracle/_ref/
    ref_bench: unmodified fused_forward for fwd and dX, shim GEMM for dA/dB) on all host
    threads; rank 0 only. One harness process: untimed setup, W warm-up repetitions, then
    K timed repetitions (each = one bounded sample step of the workload)."""
    from paper_2602_07263_b200.workload import config
    wl = config(args.config)
    if rank != 0:
        return None
    threads = os.cpu_count() or 1
    tpj = args.ref_tokens_per_job or ref_tokens_per_job(wl, threads)
    res = _bench_cpu().measure(wl, tokens_per_job=tpj, seconds_budget=0.0, threads=threads,
                               repeats=args.steps)
    if res is None or res.get("value") is None:
        why = (res or {}).get("sample", "reference CPU build missing (make ref)")
        return {"impl": "reference", "unavailable": why}
    per = res.get("per_repeat_s") or []
    ms_per_step = 1e3 * (sum(per) / len(per)) if per else None
    value = res["value"]
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": world, "steps": len(per) or args.steps, "warmup": max(args.warmup, 1),
        "ms_per_step": round(ms_per_step, 3) if ms_per_step else None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": res["dtype"],
        "data": "synthetic (seeded)",
        "config": workload_config(wl, world),
        "sample": {"what": res["sample"], "tokens_per_step": res.get("tokens_per_repeat"),
                   "tokens_per_thread": res.get("tokens_per_thread"), "threads": threads},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": res["cores"],
                         "kind": res["kind"], "sample": res["sample"]},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--layers", type=int, default=0,
                    help="override the config's layer count (0 = as configured)")
    ap.add_argument("--shuffle", action="store_true", help="interleave jobs' tokens")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-tokens-per-job", type=int, default=0,
                    help="cpu_baseline sample per job (0 = 64 tokens per host thread)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-tokens-per-job", type=int, default=0,
                    help="reference-arm sample per job (0 = 64 tokens per host thread)")
    ap.add_argument("--overlap", type=int, default=0,
                    help="low-rank launches on a side stream concurrent with the fused GEMMs: "
                         "N>0 caps them to N SMs (GEMMs get the rest), -1 = uncapped, "
                         "0 = serial schedule")
    ap.add_argument("--no-chain", action="store_true",
                    help="one launch per shrink / dH instead of chaining them into the "
                         "previous fused GEMM launch")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every kernel eagerly instead of replaying the captured "
                         "CUDA graph of the training step (graphs are used at N=1)")
    ap.add_argument("--tp", action="store_true",
                    help="tensor-parallel layer set over the torchrun group (default config C4)")
    ap.add_argument("--nano", type=int, default=4, help="initial nano-batch count (TP mode)")
    ap.add_argument("--tp-driver", default="cpp", choices=["cpp", "python"],
                    help="--tp: the C++ TP step (default) or round 1's Python TP driver")
    ap.add_argument("--driver", default="cpp", choices=["cpp", "python"],
                    help="cpp: the C++ step executor (default); python: runner.LayerSetStep")
    ap.add_argument("--host", default="python", choices=["python", "cpp"],
                    help="cpp: run the pure C++ host binary (tests/cpp/_build/step_main)")
    ap.add_argument("--nano-batches", type=int, default=NANO_DEFAULT,
                    help="executor: fixed nano-batch count N (> 0), or 0 = AIMD every step")
    ap.add_argument("--dp-sharded-opt", action="store_true",
                    help="executor, N > 1 GPUs: sharded optimizer (reduce-scatter, AdamW on 1/N "
                         "of the rows, all-gather) instead of the gradient all-reduce")
    ap.add_argument("--nano-init", type=int, default=4,
                    help="executor: AIMD initial N (reference default 4)")
    ap.add_argument("--fused-rs", default="auto",
                    help="TP mode: comma list of row-parallel projections (o,down) whose "
                         "reduce-scatter is fused into the GEMM epilogue (bulk copies into "
                         "the owner's receive slot over NVLink); the rest use NCCL on the "
                         "comm stream. auto = o,down when TP > 1; none = NCCL for all")
    ap.add_argument("--aimd-steps", type=int, default=12,
                    help="AIMD steps: TP mode exploration; executor: the untimed AIMD phase")
    ap.add_argument("--dp-reserve-sms", type=int, default=0,
                    help="DP (N>1): SMs kept free of the persistent grids for the concurrent "
                         "NCCL all-reduce (NCCL gets half as many channels); 0 = defaults "
                         "(measured best: DP2 2.89 M vs 2.79 M tokens/s with 8 reserved)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("TLORA_BENCH_WATCHDOG"):  # debugging aid: dump every thread's stack
        import faulthandler                      # if the run is still going after N seconds
        faulthandler.dump_traceback_later(float(os.environ["TLORA_BENCH_WATCHDOG"]), exit=True)

    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if rank == 0 and out is not None:
            print(json.dumps(out), flush=True)
        return

    if args.tp and args.config == "C2" and "--config" not in sys.argv:
        args.config = "C4"
    if world > 1 and not args.tp and args.dp_reserve_sms > 0:
        # DP: the gradient all-reduce runs on a comm stream concurrently with the persistent
        # GEMMs. Give NCCL a few channels and keep that many SMs (+ slack, whole CTA pairs)
        # out of the persistent grids, so neither waits for the other to drain an SM.
        # Off by default: 3 A/B runs each at DP2 gave 2.79 M (8 reserved) vs 2.89 M.
        os.environ.setdefault("TLORA_SM_RESERVE", str(args.dp_reserve_sms))
        os.environ.setdefault("NCCL_MAX_NCHANNELS", str(max(1, args.dp_reserve_sms // 2)))
    if world > 1 or args.tp:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29555")
            os.environ.setdefault("RANK", str(rank))
            os.environ.setdefault("WORLD_SIZE", str(world))
            # NCCL_DEBUG / NCCL_DEBUG_FILE stay as the environment sets them (the driver
            # reads NCCL's init lines); the JSON line is the last line rank 0 prints.
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.host == "cpp":
        out = run_cpp_host(args)
    elif args.tp and args.tp_driver == "cpp":
        out = run_tp_exec(args, rank, world, local_rank)
    elif args.tp:
        out = run_tp(args, rank, world, local_rank)
    elif args.driver == "python" or args.shuffle or args.overlap != 0:
        out = run_ours(args, rank, world, local_rank)
    else:
        out = run_executor(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1 or args.tp:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
