#!/usr/bin/env python
"""Measured fp64 peaks on this GPU (the alu roofline of the general Hodge used a derived
37.2 TFLOP/s).  (1) DFMA issue throughput: scripts/fp64_peak.cu, 8 independent FMA chains per thread,
a grid of 4 x 148 CTAs x 256 threads (2 FLOPs per FMA; CUDA events).  (2) cuBLAS DGEMM via
torch.matmul on float64 8192^3 (2 N^3 FLOPs), best of 5.  Writes profiles/<tag>_fp64_peak.json."""
import ctypes
import json
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def dfma():
    so = "/tmp/fp64_peak.so"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    os.path.join(ROOT, "scripts", "fp64_peak.cu"), "-o", so], check=True)
    lib = ctypes.CDLL(so)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    best = None
    for per_sm, threads in ((4, 256), (8, 256), (2, 512)):
        blocks, iters = per_sm * sms, 4096
        ms = ctypes.c_float()
        assert lib.run_dfma(blocks, threads, iters, ctypes.byref(ms)) == 0
        flops = 2.0 * 8 * 16 * iters * blocks * threads
        tf = flops / (ms.value * 1e-3) / 1e12
        rec = {"blocks": blocks, "threads": threads, "ms": ms.value, "tflops": tf}
        if best is None or tf > best["tflops"]:
            best = rec
    return best, sms


def dmma():
    """mma.sync m8n8k4 f64 (DMMA) throughput: 512 FLOPs per warp instruction."""
    so = "/tmp/fp64_peak.so"
    lib = ctypes.CDLL(so)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    best = None
    for per_sm, threads in ((4, 256), (8, 256), (2, 512), (1, 128), (2, 128)):
        blocks, iters = per_sm * sms, 2048
        ms = ctypes.c_float()
        assert lib.run_dmma(blocks, threads, iters, ctypes.byref(ms)) == 0
        flops = 512.0 * 8 * 4 * iters * blocks * (threads // 32)
        tf = flops / (ms.value * 1e-3) / 1e12
        rec = {"blocks": blocks, "threads": threads, "ms": ms.value, "tflops": tf}
        print("dmma", rec)
        if best is None or tf > best["tflops"]:
            best = rec
    return best


def dgemm(n=8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2.0 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def main(tag):
    d, sms = dfma()
    mm = dmma()
    g = dgemm()
    try:
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(0)
        clk = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
        clk_max = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
    except Exception:
        clk = clk_max = None
    out = {"gpu": torch.cuda.get_device_name(0), "sms": sms, "dfma": d, "dmma": mm, "dgemm_tflops": g,
           "sm_mhz_after": clk, "sm_max_mhz": clk_max,
           "dfma_lanes_per_sm_per_cycle": (d["tflops"] * 1e12 / 2 / sms / (clk_max * 1e6)) if clk_max else None,
           "how": "scripts/fp64_peak.py: DFMA chains kernel, DMMA (mma.sync m8n8k4 f64) chains kernel (CUDA events) and torch.matmul float64 8192^3 (cuBLAS)"}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", f"{tag}_fp64_peak.json")  # copied to profiles/ by hand
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r2")
