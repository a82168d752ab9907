"""tcgen05.mma issue rate from one warp (debug measurement)."""
import ctypes, json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__
__graft_entry__.build()
from paper_1608_03836_b200 import _native
lib = _native.load()
lib.wadg_debug_umma_rate.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
out = torch.zeros(2, dtype=torch.int64, device="cuda")
for mode in (0, 1, 2):
    for n in (16, 48, 128, 256):
        r = []
        for count in (64, 512):
            assert lib.wadg_debug_umma_rate(ctypes.c_void_p(out.data_ptr()), n, count, mode, None) == 0
            torch.cuda.synchronize()
            r.append(out.cpu().tolist())
        # per-MMA cost from the difference of the two counts
        issue = (r[1][0] - r[0][0]) / 448
        total = (r[1][1] - r[0][1]) / 448
        print(json.dumps({"mode": mode, "N": n, "issue_cycles_per_mma": issue, "complete_cycles_per_mma": total,
                          "raw": r}), flush=True)
