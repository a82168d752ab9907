"""Validate the tcgen05 split-TF32 primitives (wadg_umma.cuh) on the GPU:
C = A B^T for several N, in every operand mode, against fp64."""
import ctypes, json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__
__graft_entry__.build()
from paper_1608_03836_b200 import _native
lib = _native.load()
lib.wadg_debug_umma_test.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3 + [ctypes.c_void_p]
rng = np.random.default_rng(0)
vp = lambda t: ctypes.c_void_p(t.data_ptr())
out = []
for K in (8, 40):
    for N in (8, 16, 40, 48, 128, 256):
        A = rng.standard_normal((128, K)).astype(np.float32)
        B = rng.standard_normal((N, K)).astype(np.float32)
        exact = A.astype(np.float64) @ B.astype(np.float64).T
        for mode in (0, 1, 2, 3, 4):
            Ad, Bd = torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda")
            Cd = torch.full((128, N), float("nan"), device="cuda")
            rc = lib.wadg_debug_umma_test(vp(Ad), vp(Bd), vp(Cd), N, K, mode, None)
            torch.cuda.synchronize()
            got = Cd.cpu().numpy().astype(np.float64)
            err = float(np.abs(got - exact).max() / np.abs(exact).max())
            out.append({"K": K, "N": N, "mode": mode, "rc": rc, "rel_err": err})
            print(json.dumps(out[-1]), flush=True)
