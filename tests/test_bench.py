"""bench.py: the driver's JSON contract and the roofline arithmetic."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def test_fused_lower_bound_bytes_config4():
    """B_F = w (16 Np + 9 Nq + n_w Nq + 4 F) + 16 per element:
    config 4 (fp32, N = 4, heterogeneous c^2) is 9,356 B per tet, 14.716 GB per
    stage for 1,572,864 tets, the figure behind roofline.achieved."""
    Np, Nq, F, w, n_om = 35, 125, 4 * 25, 4, 2
    per = w * (4 * 4 * Np + 9 * Nq + n_om * Nq + 4 * F) + 4 * 4
    assert per == 9356
    assert abs(per * 1572864 / 1e9 - 14.716) < 1e-3
    B, FL = bench.algorithmic_model(3, 1, Np, Nq, Nq, F, w, n_om)
    assert B["volume"] == w * (2 * 4 * Np + 9 * Nq)
    assert FL["update"] == 4 * (4 * Np * Nq + Nq) + 16 * Np


@pytest.mark.parametrize("N", [2, 3, 4, 5, 6, 7])
def test_issued_flops_cover_the_algorithmic_flops(N):
    """The tensor-core flops the kernels issue (padded extents, three split-TF32
    MMAs per product for tf32) are at least the algorithmic flops."""
    Np = (N + 1) * (N + 2) * (N + 3) // 6
    Nq, F = (N + 1) ** 3, 4 * (N + 1) ** 2
    _, FL = bench.algorithmic_model(3, 1, Np, Nq, Nq, F, 4, 1)
    alg = sum(FL.values())
    kpad = 384
    for fn, mult in ((bench.dmma_issued_flops, 1), (bench.tmma_issued_flops, 3)):
        assert fn(N, kpad) / kpad >= 0.9 * mult * alg
    if N <= 4:
        assert bench.umma_issued_flops(N, kpad) / kpad >= 0.9 * 3 * alg


def _last_json(out):
    return json.loads([ln for ln in out.strip().splitlines() if ln.startswith("{")][-1])


def test_reference_arm_json_line():
    """--impl reference prints one JSON line with the reference keys."""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    d = _last_json(p.stdout)
    assert d["impl"] == "reference"
    assert KEYS <= set(d)
    assert d["value"] > 0 and d["unit"] == "GDOF/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["scaling"] == "strong"


@pytest.mark.gpu
def test_bench_json_line_on_the_gpu():
    """The default arm on a small config: the keys the driver reads, a roofline
    with both roofs, launches counted, clocks sampled, e2e through host buffers."""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c2", "--steps", "2",
                        "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    d = _last_json(p.stdout)
    assert (KEYS - {"cpu_baseline"}) <= set(d)
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "fp") and 0 < r["frac"] <= 1.0
    assert r["hbm"]["frac"] > 0 and r["compute"]["frac"] > 0
    assert d["gpu_launches"] == 5 * 2
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert "sm_mhz" in d["clocks"]
