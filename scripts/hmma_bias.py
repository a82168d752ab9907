"""Rounding of mma.sync m16n8k8 tf32 accumulation (debug probe, scripts/hmma_bias.cu):
signed bias and rms of split-TF32 products against fp64, chained (mode 0) or
per-k-step fresh accumulators added in fp32 (mode 1); numpy fp32 for scale."""
import ctypes, json, os, subprocess, sys
import numpy as np, torch
HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "_hmma_bias.so")
subprocess.run(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
                os.path.join(HERE, "hmma_bias.cu"), "-o", so], check=True)
lib = ctypes.CDLL(so)
rng = np.random.default_rng(0)
vp = lambda t: ctypes.c_void_p(t.data_ptr())
for dist in ("pos", "normal"):
    for K in (8, 32, 64, 216):
        b = lambda g, ex: float(((g - ex) * np.sign(ex)).mean() / np.abs(ex).mean())
        r = lambda g, ex: float(np.sqrt(((g - ex) ** 2).mean()) / np.abs(ex).mean())
        for mode in (0, 1):
            bs, rs, fb, fr = [], [], [], []
            for rep in range(50):
                f = (lambda s: rng.uniform(0.5, 1.0, s)) if dist == "pos" else (lambda s: rng.standard_normal(s))
                A = f((16, K)).astype(np.float32); B = f((K, 8)).astype(np.float32)
                ex = A.astype(np.float64) @ B.astype(np.float64)
                Ad, Bd = torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda")
                Cd = torch.zeros((16, 8), device="cuda")
                assert lib.hmma_probe(vp(Ad), vp(Bd), vp(Cd), K, mode) == 0
                got = Cd.cpu().numpy().astype(np.float64)
                bs.append(b(got, ex)); rs.append(r(got, ex))
                fp = (A @ B).astype(np.float64); fb.append(b(fp, ex)); fr.append(r(fp, ex))
            print(json.dumps({"dist": dist, "K": K, "mode": mode, "bias": np.mean(bs), "rms": np.mean(rs),
                              "fp32_bias": np.mean(fb), "fp32_rms": np.mean(fr)}), flush=True)
