"""bench.py's contract on CPU: the roofline peak rule and the reference arm's
JSON line (the driver parses both arms' lines and compares their configs)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

PK = {"hbm_gbs": 6549.1, "bf16_tflops": 1661.3, "bf16_tflops_sustained": 1391.1, "fp64_tflops": 37.19}


def _prof(name, flops, ms, launches=3):
    return {name: {"ms": ms, "launches": launches, "flops": flops, "bytes": 0.0}}


def test_roofline_sustained_for_long_regions_burst_for_short():
    # 20 steps x 100 ms = 2 s region: sustained TF32 peak (bf16 sustained / 2)
    r = bench.roofline(_prof("opg_symkr", 600e12 * 1.5, 1500.0), 20, 100.0, PK, "test", "tf32")
    assert r["peak"] == pytest.approx(1391.1 / 2) and r["frac"] == pytest.approx(600 / (1391.1 / 2))
    assert r["frac_burst"] == pytest.approx(600 / (1661.3 / 2))
    # 20 steps x 2 ms = 40 ms: burst
    r = bench.roofline(_prof("hess_symkr", 300e12 * 0.03, 30.0), 20, 2.0, PK, "test", "tf32")
    assert r["peak"] == pytest.approx(1661.3 / 2)


def test_roofline_f16s_uses_the_fp16_peak_only_for_fp16_kernels():
    r = bench.roofline(_prof("opg_symkr", 800e12 * 1.0, 1000.0), 15, 80.0, PK, "test", "f16s")
    assert r["peak"] == pytest.approx(1391.1)
    r = bench.roofline(_prof("hess_fused", 200e12 * 0.5, 500.0), 8, 15.0, PK, "test", "f16s")
    assert r["peak"] == pytest.approx(1661.3 / 2)  # a TF32 kernel inside the F16S mode


def test_roofline_fp64_uses_the_measured_dmma_peak():
    r = bench.roofline(_prof("hess_orbit", 22e12 * 0.015, 15.0), 1, 30.0, PK, "test", "f64")
    assert r["peak"] == pytest.approx(37.19) and r["frac"] == pytest.approx(22 / 37.19)


def test_reference_arm_line():
    from oracle.oracle import Ref
    if not Ref.available():
        pytest.skip("oracle/_ref not built (make -C oracle where /root/reference exists)")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c0",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    from paper_1905_05559_b200.workloads import CONFIGS
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "entries/s"
    assert line["config"] == bench.config_dict(CONFIGS["c0"])  # the GPU arm prints the same dict
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "entries/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["higher_is_better"] is True and line["steps"] == 2 and line["warmup"] == 1
