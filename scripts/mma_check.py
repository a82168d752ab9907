"""Validate the mma.sync split-TF32 fragment layouts and accuracy."""
import ctypes, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__
__graft_entry__.build()
from paper_1608_03836_b200 import _native
lib = _native.load()
lib.wadg_debug_mma_test.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_void_p]
rng = np.random.default_rng(0)
K = 40
A = rng.standard_normal((16, K)).astype(np.float32)
B = rng.standard_normal((K, 8)).astype(np.float32)
Ad = torch.tensor(A.T.copy(), device="cuda")       # column-major (k, r)
Bd = torch.tensor(B, device="cuda")
Cd = torch.zeros((16, 8), device="cuda")
vp = lambda t: ctypes.c_void_p(t.data_ptr())
assert lib.wadg_debug_mma_test(vp(Ad), vp(Bd), vp(Cd), K, None) == 0
torch.cuda.synchronize()
exact = A.astype(np.float64) @ B.astype(np.float64)
fp32 = (A @ B)
got = Cd.cpu().numpy()
print("3xTF32 max rel err", np.abs(got - exact).max() / np.abs(exact).max(),
      " fp32 GEMM max rel err", np.abs(fp32 - exact).max() / np.abs(exact).max())
