#!/usr/bin/env python
"""Benchmark of the data-parallel MLP safety check (BASELINE.json metric: perturbations verified/s,
whole box, and % of roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl mlpv|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step is one mlpv_check (every row of SURVEY.md §8(a): decode / generate, forward, argmax,
property, coverage, reductions) over all base inputs of the config and a fresh slice of S sample
indices per base per GPU, followed at N > 1 by the all-gather + merge of the results.  Each rank
checks its own slice (weak scaling).  Timing: W untimed warm-up steps; then K steps, each
bracketed by barrier + synchronize and timed with CUDA events on the launching stream, with an L2
flush (256 MiB write) between steps; the max over ranks is reported.  The oracle (test
infrastructure) is run only in the cpu_baseline leg and in --impl reference.
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import select
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "perturbations verified/sec (whole box) at 1/2/4/8 B200; % of roofline"
UNIT = "perturbations/s"
DEFAULT_SAMPLES = {"cfg1": None, "cfg2": None, "cfg3": 1 << 20, "cfg4": 1 << 16, "cfg4_box": 1 << 16,
                   "cfg5_bf16": 1 << 12, "cfg5_int8": 1 << 12}
DTYPE = {"cfg1": "fp32", "cfg2": "q4.12", "cfg3": "int8", "cfg4": "bf16", "cfg4_box": "bf16", "cfg5_bf16": "bf16",
         "cfg5_int8": "int8"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="cfg4")
    p.add_argument("--samples", type=int, default=0, help="samples per base per GPU per step (Philox spaces)")
    p.add_argument("--impl", default="mlpv", choices=["mlpv", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


def alg_ops_per_candidate(cfg):
    """Algorithmic operations per candidate: dense MACs x 2 for the Philox
    (dense) spaces; the incremental layer-1 update (|S| x n_1) + dense later layers for subset spaces."""
    s = cfg.net.sizes
    dense_rest = sum(s[l - 1] * s[l] for l in range(2, len(s)))
    if cfg.pert.kind in (3, 4, 5):                  # Philox spaces: every pixel moves
        return 2 * (s[0] * s[1] + dense_rest)
    changed = cfg.pert.tuple if cfg.pert.kind == 0 else len(cfg.pert.pixels)
    return 2 * (changed * s[1] + dense_rest)


def epilogue_ops_per_candidate(cfg):
    """Algorithmic CUDA-core ops per candidate when the contractions run on the tensor pipe (k_tc3):
    2 per subset pixel (digit, value), per potential of every layer an offset / bias add and a sign
    predicate, per hidden neuron a requantisation (round-shift, clamp), per output an argmax compare."""
    s = cfg.net.sizes
    hidden = sum(s[1:-1])
    return 2 * len(cfg.pert.pixels) + 2 * sum(s[1:]) + 2 * hidden + s[-1]


def kernel_name(cfg):
    """The enumeration kernel mlpv_check launches for this config (the dominant kernel)."""
    import mlpv_inputs as M
    s = cfg.net.sizes
    if cfg.pert.kind in (4, 5) and len(s) == 4 and s[1] == 256 and s[2] == 256 and s[0] % 2 == 0 and s[0] <= 1024:
        return "k_fused3"
    if cfg.pert.kind in (3, 4, 5):
        return "k_large"
    if (cfg.net.numeric == M.NUM_INT8 and len(s) == 4 and s[1] <= 64 and s[2] <= 32 and s[3] <= 16
            and cfg.pert.kind in (1, 2) and 1 <= len(cfg.pert.pixels) <= 32):
        return "k_tc3"
    if (cfg.net.numeric == M.NUM_INT8 and len(s) == 4 and s[1] <= 64 and s[2] <= 32 and s[3] <= 32
            and cfg.pert.kind in (1, 2) and len(cfg.pert.pixels) >= 2):
        return "k_warp3"
    return "k_small"


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


REASON_BITS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))


class NvmlSampler:
    """In-process NVML sampler (the library nvidia-smi itself reads): SM clock and the active clock-event
    reasons every `period` seconds from a thread, so that even a 40 ms timed region (cfg5) holds
    samples; the nvidia-smi -lms 200 sampler below is the fallback when NVML is not importable."""

    def __init__(self, nvml, handle, period: float = 0.02):
        self.nvml, self.h, self.period = nvml, handle, period
        self.rows, self.halt, self.thread = [], threading.Event(), None

    @classmethod
    def open(cls, uuid: str, index: str):
        try:
            import pynvml
            pynvml.nvmlInit()
            try:
                h = pynvml.nvmlDeviceGetHandleByUUID(uuid) if uuid else pynvml.nvmlDeviceGetHandleByIndex(int(index))
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(int(index))
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            return cls(pynvml, h)
        except Exception:
            return None

    def _reasons(self) -> int:
        try:
            return int(self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h))
        except Exception:
            return int(self.nvml.nvmlDeviceGetCurrentClocksThrottleReasons(self.h))

    def _run(self):
        while not self.halt.is_set():
            try:
                self.rows.append((time.time(), float(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM)),
                                  self._reasons()))
            except Exception:
                pass
            self.halt.wait(self.period)

    def start(self):
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def stop(self, t_begin: float = None, t_end: float = None):
        self.halt.set()
        if self.thread is not None:
            self.thread.join(timeout=2)
        try:
            mx = float(self.nvml.nvmlDeviceGetMaxClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
        except Exception:
            mx = 0.0
        return self.summarise(self.rows, mx, t_begin, t_end, self.period)

    @staticmethod
    def summarise(rows, mx, t_begin, t_end, period):
        """[(time, sm_mhz, reason bits)] -> the clocks object: samples inside [t_begin, t_end] (all when none)."""
        inside = [r for r in rows if t_begin is not None and t_begin <= r[0] <= t_end]
        use = inside or rows
        if not use:
            return None
        bits = 0
        for r in use:
            bits |= r[2]
        return {"sm_mhz": statistics.median(r[1] for r in use), "sm_max_mhz": mx,
                "reasons": sorted(nm for nm, b in REASON_BITS if bits & b), "samples": len(use),
                "source": f"nvml, {int(1e3 * period)} ms period" + ("" if inside else " (no sample inside the timed region: all samples)")}


class ClockSampler:
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: str):
        self.idx = gpu_index
        self.proc = None

    def start(self):
        if os.environ.get("MLPV_BENCH_SAMPLER") == "off":    # diagnostic runs only (tools/s4_smi_ab.sh)
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", os.environ.get("MLPV_BENCH_SAMPLER_MS", "200"), "-i", self.idx], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        # wait for the first sample (NVML start-up done) so that the sampler is live from here on
        self.t_live = None
        r, _, _ = select.select([self.proc.stdout], [], [], 10.0)
        if r:
            self.proc.stdout.readline()
            self.t_live = time.time()

    def stop(self, t_begin: float = None, t_end: float = None):
        """Median SM clock and the throttle reasons of the samples taken inside [t_begin, t_end]
        (host time.time() bounds of the timed region); when none falls inside, of the samples since the
        sampler went live just before the warm-up (the same kernels under the same load)."""
        if self.proc is None:
            return None
        # (no sleep before the terminate unless the timed region was too short to hold a 200 ms
        # sample: a 0.25 s idle here lets the power-capped GPU recover and lifts the e2e steps that
        # follow 3-5 % above the device-timed ones, tools/s4_smi_ab.sh)
        if t_begin is not None and t_end - t_begin < 0.45:
            time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        return self.summarise(out, t_begin, t_end)

    @staticmethod
    def summarise(out: str, t_begin: float = None, t_end: float = None):
        """nvidia-smi csv lines (FIELDS order) -> {"sm_mhz": median, "sm_max_mhz", "reasons", "samples"}."""
        rows = []
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            rows.append((ts, f))
        inside = [f for ts, f in rows if ts is not None and t_begin is not None and t_begin - 0.05 <= ts <= t_end + 0.05]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for f in (inside or [f for _, f in rows]):       # (the first, idle sample was consumed by start())
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def to_device(bases, device):
    import numpy as np
    import torch
    a = bases.view(np.int16) if bases.dtype == np.uint16 else bases
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def samples_for(cfg, args):
    if cfg.pert.kind not in (3, 4, 5):
        return None
    return args.samples or DEFAULT_SAMPLES[cfg.name]


def step_range(cfg, args, k, rank, world):
    """Index range of step k on `rank`: a fresh slice of S samples per base (Philox spaces), or
    the rank's shard of the whole space (enumerated spaces)."""
    S = samples_for(cfg, args)
    space = cfg.space
    if S is None:
        from paper_1907_12933_b200.dist import shard
        return shard(0, space, rank, world)
    slot = (k * world + rank) % max(1, space // S)
    return slot * S, slot * S + S


def cpu_baseline(cfg, budget_s=12.0):
    """The oracle as it stands, on this host's cores, on a bounded sample of the same workload."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(cores)
    nb = min(16, cfg.n_base)
    m = 64                                       # calibrate on probes of at least ~1 s, then size the
    while True:                                  # timed sample to ~budget_s of oracle work
        probe = cfg.subset(n_base=nb, begin=0, end=min(cfg.space, m))
        t0 = time.perf_counter()
        O.check(probe, nthreads=cores)
        dt = max(time.perf_counter() - t0, 1e-3)
        if dt >= 1.0 or m >= cfg.space:
            break
        m *= 4
    rate = nb * (probe.pert.index_end - probe.pert.index_begin) / dt
    m = int(max(8, min(cfg.space, budget_s * rate / nb)))
    s = cfg.subset(n_base=nb, begin=0, end=m)
    t0 = time.perf_counter()
    ores = O.check(s, nthreads=cores)
    dt = time.perf_counter() - t0
    n = nb * m
    out = {"value": n / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"{cfg.name}: bases 0-{nb - 1} x indices [0, {m}) = {n} candidates in {dt:.1f} s"}
    return out, s, ores


def sample_parity(chk, s, o):
    """The GPU on exactly the oracle's timed sample, compared by the parity rules:
    fixed point bit-exact (counts, counterexamples, every coverage bit); float by reading C20
    (violation counts within the flagged counts, first counterexamples bracketing each other's
    unflagged ones, certain coverage contained in the other side's coverage).  The oracle's tau
    (C20) is the GPU's (both from the sample's base traces)."""
    import numpy as np
    import torch
    import mlpv_inputs as M
    import paper_1907_12933_b200 as P
    bases = to_device(s.bases, "cuda")
    r = chk.check(bases, s.pert, s.prop, s.cov)
    chk.sync()
    torch.cuda.synchronize()
    g = P.result_to_numpy(r, s.n_base, r["n_words"])
    bad = []
    if s.net.numeric in (M.NUM_Q4_12, M.NUM_INT8):
        for k in ("checked", "violated", "first_cex"):
            if not np.array_equal(g[k], getattr(o, k)):
                bad.append(k)
        if not np.array_equal(g["cov_all"], o.cov_all):
            bad.append("cov_all")
        rule = "bit-exact"
    else:
        if not np.array_equal(g["checked"], o.checked):
            bad.append("checked")
        vg, vo = g["violated"].astype(np.int64), o.violated.astype(np.int64)
        if not np.all(np.abs(vg - vo) <= np.minimum(g["flagged"], o.flagged).astype(np.int64)):
            bad.append("violated")
        if not (np.all(g["first_cex"] <= o.first_cex_unflagged) and np.all(o.first_cex <= g["first_cex_unflagged"])):
            bad.append("first_cex")
        if (o.cov_certain & ~g["cov_all"]).any() or (g["cov_certain"] & ~o.cov_all).any():
            bad.append("coverage")
        rule = "C20 float rules"
    return {"status": "ok" if not bad else "FAILED", "rule": rule, "mismatch": bad,
            "violated_gpu": int(g["violated"].sum()), "violated_oracle": int(o.violated.sum()),
            "coverage_bits_gpu": int(np.unpackbits(g["cov_all"].view(np.uint8)).sum())}


def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import mlpv_inputs as M
    from oracle import oracle as O
    cfg = M.make_config(args.config)
    cores = os.cpu_count() or 1
    nb = min(16, cfg.n_base)
    # size each step to ~10 s of oracle work so the whole run stays within a few minutes
    cal, _, _ = cpu_baseline(cfg, budget_s=3.0)
    per_step = int(max(8, min(cfg.space, 10.0 * cal["value"] / nb)))
    times = []
    for k in range(args.warmup + args.steps):
        s = cfg.subset(n_base=nb, begin=k * per_step % max(1, cfg.space - per_step), end=None)
        s = cfg.subset(n_base=nb, begin=s.pert.index_begin, end=s.pert.index_begin + per_step)
        t0 = time.perf_counter()
        O.check(s, nthreads=cores)
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
    T = sum(times)
    n = args.steps * nb * per_step
    v = n / T
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": DTYPE[cfg.name], "data": "synthetic",
            "impl": "reference",
            "config": {"workload": cfg.name, "description": cfg.description,
                       "sample_per_step": f"bases 0-{nb - 1} x {per_step} indices"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} steps of {nb} bases x {per_step} indices"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    import mlpv_inputs as M
    import paper_1907_12933_b200 as P
    from paper_1907_12933_b200 import dist as PD

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # MLPV_BENCH_GLOO=1 (tests only): the N > 1 path with gloo and every rank on the visible GPUs in
    # turn -- exercises the sharding, the exchange and the max-over-ranks timing on a one-GPU box;
    # the driver's multi-GPU runs use NCCL, one rank per GPU
    gloo = bool(os.environ.get("MLPV_BENCH_GLOO"))
    local = local % max(1, torch.cuda.device_count()) if gloo else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    tdev = torch.device("cpu") if gloo else dev          # device of the timing all-reduces
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        from paper_1907_12933_b200 import build as B
        B.build()                                # no-op when libmlpv.so is current
    if world > 1:
        dist.barrier()
    P.lib()                                      # fails loudly if libmlpv.so is missing

    cfg = M.make_config(args.config)
    chk = P.Checker(cfg.net, device=local)
    bases = to_device(cfg.bases, dev)
    nw, _ = chk.coverage_layout(cfg.cov)
    res = P.alloc_result(cfg.n_base, nw, dev)
    stream = torch.cuda.current_stream(dev)

    def one_step(k):
        b, e = step_range(cfg, args, k, rank, world)
        r = chk.check(bases, cfg.pert.with_range(b, e), cfg.prop, cfg.cov, out=res)
        if world > 1:
            r = PD.reduce_results(r, cfg.n_base, nw)
        return r, e - b

    def barrier():
        if world > 1:
            dist.barrier()

    # the clock sampler (nvidia-smi -lms) starts before the warm-up so that its start-up (NVML
    # initialisation) is not inside the timed region; only samples stamped inside it are reported
    gpu_idx = os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local] if os.environ.get("CUDA_VISIBLE_DEVICES") else str(local)
    try:
        uuid = "GPU-" + str(torch.cuda.get_device_properties(local).uuid)
    except Exception:
        uuid = ""
    clocks = (None if os.environ.get("MLPV_BENCH_SAMPLER") in ("smi", "off") else NvmlSampler.open(uuid, gpu_idx)) or ClockSampler(gpu_idx)
    late = os.environ.get("MLPV_BENCH_SAMPLER") == "late"
    if not late:
        clocks.start()
    for k in range(args.warmup):
        one_step(k)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    kev0, kev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kev0.record(stream)                          # materialise the cudaEvent_t handles; the library
    kev1.record(stream)                          # re-records them around the enumeration kernel
    torch.cuda.synchronize()
    launches0 = chk.profile(kev0, kev1)
    if late:
        clocks.start()
    t_begin = time.time()
    step_ms, kern_ms, n_cand = [], [], 0
    for k in range(args.warmup, args.warmup + args.steps):
        flush.fill_(k & 0xFF)                   # L2 flush between timed steps (outside the events)
        torch.cuda.synchronize()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        _, per_base = one_step(k)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        step_ms.append(ev0.elapsed_time(ev1))
        kern_ms.append(kev0.elapsed_time(kev1))
        n_cand += per_base * cfg.n_base
    clk = clocks.stop(t_begin, time.time())
    launches = chk.profile(None, None) - launches0 + (args.steps if world > 1 else 0)
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    total_cand = n_cand * world
    if world > 1:                                # the shards of an enumerated space differ by <= 1 per base
        t = torch.tensor([float(n_cand)], dtype=torch.float64, device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        total_cand = int(t.item())
    value = total_cand / (total_ms / 1e3)

    # ---- end to end through the public API: pinned host inputs -> device, check, results -> host
    e2e = None
    if not args.no_e2e:
        arr = cfg.bases.view(np.int16) if cfg.bases.dtype == np.uint16 else cfg.bases
        host_in = torch.from_numpy(np.ascontiguousarray(arr)).pin_memory()
        dev_in = torch.empty_like(host_in, device=dev)
        keys = ("checked", "violated", "flagged", "first_cex", "first_cex_unflagged", "cov_all", "cov_certain")
        host_out = {k: torch.empty_like(res[k], device="cpu").pin_memory() for k in keys}
        h2d = host_in.numel() * host_in.element_size()
        d2h = sum(v.numel() * v.element_size() for v in host_out.values())
        # host wall clock around the whole sequence a user runs (H2D of the inputs, the check
        # through the C ABI, mlpv_sync, the all-gather + merge, D2H of the results): Python,
        # ctypes marshalling and argument validation included (not device events)
        e2e_ms, e2e_cand = 0.0, 0
        for k in range(args.warmup + args.steps, args.warmup + 2 * args.steps):
            flush.fill_(k & 0xFF)               # the same L2 flush as the device-timed steps
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            dev_in.copy_(host_in, non_blocking=True)
            b, e = step_range(cfg, args, k, rank, world)
            r = chk.check(dev_in, cfg.pert.with_range(b, e), cfg.prop, cfg.cov, out=res)
            if world > 1:
                r = PD.reduce_results(r, cfg.n_base, nw)
            for kk in keys:
                host_out[kk].copy_(r[kk], non_blocking=True)
            chk.sync()                          # waits for the stream; raises on a device fault
            e2e_ms += 1e3 * (time.perf_counter() - t0)
            barrier()
            e2e_cand += (e - b) * cfg.n_base
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=tdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": e2e_cand * world / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h}

    # ---- roofline of the dominant kernel (the enumeration kernel)
    pk, src = peaks()
    ops = alg_ops_per_candidate(cfg)
    kern_avg_s = (sum(kern_ms) / len(kern_ms)) / 1e3
    per_launch = n_cand / args.steps
    if cfg.pert.kind in (3, 4, 5):
        bound, unit = "tensor", "TFLOP/s"
        peak = float(pk["bf16_tflops"])
        peak_note = f"{src} bf16 burst"
        if cfg.net.numeric == M.NUM_INT8:
            # int8: measured on this pool by tools/measure_peaks.py (torch._int_mm 8192^3, burst)
            p8 = os.path.join(ROOT, "profiles", "measured_peaks_r2.json")
            if os.path.exists(p8):
                peak = float(json.load(open(p8))["int8_tops"])
                peak_note = "measured int8 burst (profiles/measured_peaks_r2.json)"
            else:
                peak, peak_note = 2.0 * peak, peak_note + " x2 (int8 nominal ratio; measurement missing)"
        achieved = ops * per_launch / kern_avg_s / 1e12
    elif kernel_name(cfg) == "k_tc3":
        # the contractions run on the tensor pipe (a few % busy); the CUDA-core epilogue binds (ncu:
        # the SMSPs' ALU pipe ~70 % of peak): algorithmic epilogue ops against the lane-op peak
        bound, unit = "alu", "Gop/s"
        peak = 148 * 128 * float(pk.get("sm_max_mhz", 1965.0)) * 1e6 / 1e9
        peak_note = ("148 SM x 128 lanes x sm_max_mhz (one op per lane per clock); ops = the epilogue's "
                     "algorithmic ops, the MACs run on the tensor pipe")
        ops_mac = ops
        ops = epilogue_ops_per_candidate(cfg)
        achieved = ops * per_launch / kern_avg_s / 1e9
    else:
        bound, unit = "alu", "Gop/s"
        peak = 148 * 128 * float(pk.get("sm_max_mhz", 1965.0)) * 1e6 / 1e9
        peak_note = "148 SM x 128 lanes x sm_max_mhz (one op per lane per clock)"
        achieved = ops * per_launch / kern_avg_s / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        traffic = json.load(open(prof)).get(cfg.name)
    roofline = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
                "traffic": traffic, "kernel": kernel_name(cfg),
                "kernel_ms": 1e3 * kern_avg_s, "peak_source": peak_note,
                "alg_ops_per_candidate": ops, "candidates_per_launch": per_launch}
    if bound == "tensor" and cfg.net.numeric != M.NUM_INT8 and pk.get("bf16_tflops_sustained"):
        # (context: the same rate against the pod's sustained bf16 figure -- cuBLAS back to back for
        # 4 s, power-capped; the frac above uses the burst figure)
        roofline["frac_vs_sustained_peak"] = achieved / float(pk["bf16_tflops_sustained"])
    if kernel_name(cfg) == "k_tc3":
        # the same launch against the int8 tensor peak, in the MAC ops (5,504 / candidate for cfg3)
        p8 = os.path.join(ROOT, "profiles", "measured_peaks_r2.json")
        if os.path.exists(p8):
            t8 = float(json.load(open(p8))["int8_tops"])
            roofline["tensor_frac_int8_peak"] = ops_mac * per_launch / kern_avg_s / 1e12 / t8

    if rank == 0:
        cpu = par = None
        if world == 1 and not args.no_cpu_baseline:
            cpu, sample, ores = cpu_baseline(cfg)
            par = sample_parity(chk, sample, ores)
            par["sample"] = cpu["sample"]
        S = samples_for(cfg, args)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": DTYPE[cfg.name], "data": "synthetic",
                "config": {"workload": cfg.name, "description": cfg.description, "bases": cfg.n_base,
                           "samples_per_base_per_gpu_per_step": S,
                           "candidates_per_step": total_cand // args.steps,
                           "l2": "flushed between timed steps (256 MiB write)",
                           "parallelism": f"dp{world} (index-space shards, one all-gather per step)"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk}
        if par is not None:
            line["parity"] = par
        print(json.dumps(line), flush=True)
        if par is not None and par["status"] != "ok":
            raise SystemExit(f"bench: GPU / oracle parity FAILED on the timed sample: {par}")
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
