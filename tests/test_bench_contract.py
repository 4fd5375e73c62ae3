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
    lines = sorted(glob.glob(os.path.join(ROOT, "profiles", "r02_bench_config*.json")))
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


def _line(name):
    with open(os.path.join(ROOT, "profiles", name)) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def test_headline_line_has_e2e_and_cpu_baseline():
    d = _line("r02_bench_config3.json")
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert "fwd,dx,dw" in d["e2e"]["path"]  # the drop-in's three host calls are the headline e2e
    assert d["e2e_step"]["h2d_bytes_per_step"] < d["e2e"]["h2d_bytes_per_step"]
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert "Separate" in d["cpu_baseline"]["sample"]


def test_both_arms_share_config_and_bytes():
    """The reference arm and this repo's arm print identical config dicts and
    count the same compulsory bytes, so the driver's value ratio is the time
    ratio and its same_config check holds."""
    ours, ref = _line("r02_bench_config3.json"), _line("r02_bench_reference_config3.json")
    assert ours["config"] == ref["config"]
    assert ours["config"]["mode"] == "separate"  # the reference's default MulAddMode
    B, H, L, K = (ours["config"][k] for k in "BHLK")
    assert ours["config"]["bytes_per_step"] == bench.step_bytes(B, H, L, K) == 20 * B * H * L + 12 * H * K
    assert abs(ours["value"] - ours["config"]["bytes_per_step"] / (ours["ms_per_step"] * 1e-3) / 1e9) < 1.0
    assert ref["impl"] == "reference" and ref["e2e"]["h2d_bytes_per_step"] == 0
    assert ref["side"]["mode"] == "fused"
