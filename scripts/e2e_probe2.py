import json, os, sys, time
import torch
x = torch.randn((4, 1572864, 35), device="cuda")
out = {}
def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3
buf = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
out["prealloc_pinned_copy_ms"] = t(lambda: buf.copy_(x))
def fresh():
    h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    h.copy_(x)
    return h
out["fresh_pinned_alloc_copy_ms"] = t(fresh)
out["pinned_alloc_only_ms"] = t(lambda: torch.empty(x.shape, dtype=x.dtype, pin_memory=True))
out["pageable_copy_ms"] = t(lambda: x.cpu())
def nb():
    h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    h.copy_(x, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return h
out["fresh_pinned_nonblocking_ms"] = t(nb)
print(json.dumps(out))
