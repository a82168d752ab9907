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
