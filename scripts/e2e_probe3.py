import json, os, sys, time
import torch
K, Np, Kpad = 1572864, 35, 1572864
Q = torch.randn((4, Np, Kpad), device="cuda")
like = torch.randn((K, Np)).pin_memory()
def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3
out = {}
Qt = Q[:, :, :K].transpose(1, 2)
out["transpose_contig_ms"] = t(lambda: Qt.to(like.dtype).contiguous())
dev = Qt.contiguous()
out["is_pinned_ms"] = t(lambda: like.is_pinned())
def d2h():
    h = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=like.is_pinned())
    h.copy_(dev)
    return h
out["alloc_copy_ms"] = t(d2h)
def whole():
    dv = Qt.to(like.dtype).contiguous()
    h = torch.empty(dv.shape, dtype=dv.dtype, pin_memory=like.is_pinned())
    h.copy_(dv)
    return list(h.unbind(0))
out["whole_ms"] = t(whole)
print(json.dumps(out))
