"""CPU: bench.py's pieces that do not need a GPU -- the metric definitions
match the reference's formulas and the committed evidence it reads, and the
committed bench lines keep the driver's JSON contract."""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2604_25422_b200 import traffic  # noqa: E402


def test_path_bytes_and_flops_follow_the_reference():
    for cfg in bench.CONFIGS.values():
        B, H, L, K = cfg
        assert bench.path_bytes(B, H, L, K) == traffic.logical_traffic("fwd", B, H, L, K)
        assert bench.path_flops(B, H, L, K) == 2 * B * H * L * K  # src/analyzer.cpp:36-49


def test_help_runs_without_a_gpu():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 0 and "--impl" in out.stdout and "--bwd" in out.stdout


def test_committed_bench_lines_keep_the_contract():
    lines = sorted(glob.glob(os.path.join(ROOT, "profiles", "r01_bench_config*.json")))
    assert lines
    for p in lines:
        with open(p) as f:
            d = json.loads(f.read().strip().splitlines()[-1])
        for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                    "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks"):
            assert key in d, (p, key)
        assert d["config"].get("workload"), p
        assert d["warmup"] >= 3, p
        assert d["roofline"]["frac"] > 0 and d["roofline"]["peak"] > 0, p
        assert d["gpu_launches"] > 0, p


def test_headline_line_has_e2e_and_cpu_baseline():
    with open(os.path.join(ROOT, "profiles", "r01_bench_config3.json")) as f:
        d = json.loads(f.read().strip().splitlines()[-1])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["kind"] in ("reference", "port")
