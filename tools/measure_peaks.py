"""Measured peaks the driver's MEASURED_PEAKS.json does not carry:
dense int8 tensor throughput (torch._int_mm 8192^3, cuBLASLt: best of 10 = burst, back to back for
4 s = sustained) and the L2 -> SM read bandwidth of an L2-resident buffer.  Writes
profiles/measured_peaks_r2.json (tracked; bench.py reads the int8 figures from it).

    python tools/measure_peaks.py
"""
import json
import os
import subprocess
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "measured_peaks_r2.json")
OUT2 = os.path.join(ROOT, "gpurun_out", "measured_peaks_r2.json")   # what gpurun brings back


def timed(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / reps


def main():
    dev = torch.device("cuda:0")
    n = 8192
    a = torch.randint(-127, 127, (n, n), dtype=torch.int8, device=dev)
    b = torch.randint(-127, 127, (n, n), dtype=torch.int8, device=dev).t().contiguous().t()
    for _ in range(3):
        torch._int_mm(a, b)
    best = min(timed(lambda: torch._int_mm(a, b), 1) for _ in range(10))
    burst = 2.0 * n ** 3 / best / 1e12
    t0 = time.time()
    k = 0
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < 4.0:
        for _ in range(20):
            torch._int_mm(a, b)
        k += 20
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    sustained = 2.0 * n ** 3 * k / (s.elapsed_time(e) / 1e3) / 1e12
    # bf16 on the same box for the ratio
    ab = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
    bb = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
    for _ in range(3):
        ab @ bb
    bf = 2.0 * n ** 3 / min(timed(lambda: ab @ bb, 1) for _ in range(10)) / 1e12
    # L2 -> SM read bandwidth: sum over a 48 MiB buffer (fits the 126 MB L2) many times; HBM: 4 GiB
    x = torch.ones(12 * 1024 * 1024, dtype=torch.float32, device=dev)
    for _ in range(5):
        x.sum()
    l2 = x.numel() * 4 / min(timed(lambda: x.sum(), 20) for _ in range(5)) / 1e9
    y = torch.ones(1024 * 1024 * 1024, dtype=torch.float32, device=dev)
    y.sum()
    hbm = y.numel() * 4 / min(timed(lambda: y.sum(), 3) for _ in range(3)) / 1e9
    clocks = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,name", "--format=csv,noheader"],
                            capture_output=True, text=True).stdout.strip()
    d = {"int8_tops": burst, "int8_tops_sustained": sustained, "bf16_tflops_same_run": bf,
         "int8_over_bf16": burst / bf, "l2_read_gbs_48MiB": l2, "hbm_read_gbs_4GiB": hbm,
         "how": "torch._int_mm 8192^3 int8->int32 (2 N^3 ops): best of 10 (burst), back to back 4 s (sustained); "
                "bf16 torch.matmul 8192^3 best of 10; read bandwidth = bytes / time of torch.sum (CUDA events)",
         "nvidia_smi_after": clocks, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    json.dump(d, open(OUT, "w"), indent=1)
    os.makedirs(os.path.dirname(OUT2), exist_ok=True)
    json.dump(d, open(OUT2, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
