"""Measured FMA-pipe peak (FP32 FFMA, FP64 DFMA) of this B200, register
operands, all SMs busy; the denominator of the bench's FP roofline."""

import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_1608_03836_b200 import _native  # noqa: E402


def measure(dtype_code, torch_dtype, iters=20000, blocks=148 * 8, flops_per_fma=2.0):
    inp = torch.rand(64, dtype=torch_dtype, device="cuda")
    out = torch.empty(256, dtype=torch_dtype, device="cuda")
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    args = (dtype_code, blocks, iters, ctypes.c_void_p(inp.data_ptr()), ctypes.c_void_p(out.data_ptr()), sp)
    _native.call("wadg_microbench_fma", *args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _native.call("wadg_microbench_fma", *args)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) * 1e-3
    return flops_per_fma * 16 * iters * 256 * blocks / s / 1e12


if __name__ == "__main__":
    print(json.dumps({"fp32_fma_tflops": measure(_native.WADG_F32, torch.float32),
                      "fp32_ffma2_tflops": measure(2, torch.float32, flops_per_fma=4.0),
                      "fp64_fma_tflops": measure(_native.WADG_F64, torch.float64)}))


def measure_mma(iters=20000, blocks=148 * 8):
    lib = _native.load()
    fn = lib.wadg_microbench_mma_tf32
    fn.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    inp = torch.rand(64, device="cuda")
    out = torch.empty(256, device="cuda")
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    args = (blocks, iters, ctypes.c_void_p(inp.data_ptr()), ctypes.c_void_p(out.data_ptr()), sp)
    fn(*args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(*args)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) * 1e-3
    return 2.0 * 16 * 8 * 8 * 8 * iters * (256 // 32) * blocks / s / 1e12


if __name__ == "__main__" and hasattr(_native.load(), "wadg_microbench_mma_tf32"):
    print(json.dumps({"mma_sync_tf32_tflops": measure_mma()}))


def measure_dmma(iters=20000, blocks=148 * 8):
    """mma.sync m8n8k4 f64: 256 FMAs per warp instruction."""
    lib = _native.load()
    fn = lib.wadg_microbench_dmma
    fn.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    inp = torch.rand(64, dtype=torch.float64, device="cuda")
    out = torch.empty(256, dtype=torch.float64, device="cuda")
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    args = (blocks, iters, ctypes.c_void_p(inp.data_ptr()), ctypes.c_void_p(out.data_ptr()), sp)
    fn(*args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(*args)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) * 1e-3
    return 2.0 * 256 * 8 * iters * (256 // 32) * blocks / s / 1e12


if __name__ == "__main__" and hasattr(_native.load(), "wadg_microbench_dmma"):
    print(json.dumps({"dmma_f64_tflops": measure_dmma()}))


def measure_umma(n=256, count=20000, blocks=148, mode=1):
    """tcgen05.mma kind::tf32 M=128 K=8 N=n, A in TMEM (mode 1), one CTA per SM:
    chip-wide dense TF32 throughput (each MMA = 128 n 8 MACs)."""
    lib = _native.load()
    fn = lib.wadg_microbench_umma
    fn.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    args = (blocks, n, count, mode, ctypes.c_void_p(out.data_ptr()), sp)
    fn(*args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(*args)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) * 1e-3
    return 2.0 * 128 * n * 8 * count * blocks / s / 1e12


if __name__ == "__main__" and hasattr(_native.load(), "wadg_microbench_umma"):
    print(json.dumps({"tcgen05_tf32_tflops_TS_N256": measure_umma(256, mode=1),
                      "tcgen05_tf32_tflops_SS_N256": measure_umma(256, mode=0),
                      "tcgen05_tf32_tflops_TS_N48": measure_umma(48, mode=1),
                      "tcgen05_tf32_tflops_SS_N48": measure_umma(48, mode=0)}))
