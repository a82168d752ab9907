"""Rounding behaviour of tcgen05.mma kind::tf32 accumulation (debug tool):
split-TF32 C = A B^T (3 MMAs per K step of 8) against fp64, signed bias
mean((got - exact) sign(exact)) / mean|exact| for positive and mixed-sign data."""
import ctypes, json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__
__graft_entry__.build()
from paper_1608_03836_b200 import _native
lib = _native.load()
rng = np.random.default_rng(0)
vp = lambda t: ctypes.c_void_p(t.data_ptr())
for dist in ("pos", "normal"):
    for K in (8, 16, 32, 64):
        N = 128
        f = (lambda s: rng.uniform(0.5, 1.0, s)) if dist == "pos" else (lambda s: rng.standard_normal(s))
        A = f((128, K)).astype(np.float32)
        B = f((N, K)).astype(np.float32)
        exact = A.astype(np.float64) @ B.astype(np.float64).T
        fp32 = (A @ B.T).astype(np.float64)           # numpy sgemm (fp32 FMA, RN)
        for mode in (0,):
            Ad, Bd = torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda")
            Cd = torch.full((128, N), float("nan"), device="cuda")
            lib.wadg_debug_umma_test(vp(Ad), vp(Bd), vp(Cd), N, K, mode, None)
            torch.cuda.synchronize()
            got = Cd.cpu().numpy().astype(np.float64)
            b = lambda g: float(((g - exact) * np.sign(exact)).mean() / np.abs(exact).mean())
            r = lambda g: float(np.sqrt(((g - exact) ** 2).mean()) / np.abs(exact).mean())
            print(json.dumps({"dist": dist, "K": K, "mma_per_out": 3 * K // 8, "bias": b(got), "rms": r(got),
                              "fp32_bias": b(fp32), "fp32_rms": r(fp32)}), flush=True)
