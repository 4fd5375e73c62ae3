"""CPU: the B200 traffic model (paper_2604_25422_b200/traffic.py) against the
reference's algorithmic bytes and the committed ncu DRAM measurements."""
import json
import os

from paper_2604_25422_b200 import traffic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_logical_traffic_matches_reference_formula():
    # reference tests/test_exec_model.cpp:124-126: 402,677,760 read + 402,653,184 written
    assert traffic.logical_traffic("fwd", 16384, 128, 48, 48) == 402677760 + 402653184


def test_plan_dispatch_tiers():
    assert traffic.plan("fwd", 256, 512, 8192, 7)["kernel"] == "stencil_ldg"
    assert traffic.plan("fwd", 512, 1024, 16384, 16)["kernel"] == "stencil_short"
    assert traffic.plan("fwd", 64, 128, 4096, 4096)["kernel"] == "stencil_pad"
    assert traffic.plan("fwd", 16384, 128, 48, 48)["kernel"] == "stencil_rows"
    assert traffic.plan("dw", 64, 128, 4096, 4096)["kernel"] == "dw_pad"
    assert traffic.plan("dw", 256, 512, 8192, 7)["kernel"] == "dw_short"
    assert traffic.plan("dw", 256, 512, 8192, 7, "pairwise")["kernel"] == "dw_pairwise_tma"


def test_fused_backward_moves_three_quarters():
    B, H, L, K = 256, 512, 8192, 7
    assert traffic.plan("bwd", B, H, L, K)["kernel"] == "bwd_short"
    assert traffic.plan("bwd", 64, 128, 4096, 4096)["kernel"] == "split"
    split = traffic.memory_traffic("dx", B, H, L, K) + traffic.memory_traffic("dw", B, H, L, K)
    assert abs(traffic.memory_traffic("bwd", B, H, L, K) / split - 0.75) < 0.01


def test_model_matches_ncu_dram_bytes():
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
        meas = json.load(f)["config3"]
    B, H, L, K = 256, 512, 8192, 7
    pairs = [("fwd", "fwd"), ("dx", "dX"), ("dw", "dW")] + ([("bwd", "bwd")] if "bwd" in meas else [])
    for path, key in pairs:
        model = traffic.memory_traffic(path, B, H, L, K)
        got = meas[key]["dram_bytes"]
        assert abs(got - model) / model < 0.01, (path, got, model)


def test_halo_rereads_are_small_at_config3():
    B, H, L, K = 256, 512, 8192, 7
    extra = traffic.l2_traffic("fwd", B, H, L, K) / traffic.memory_traffic("fwd", B, H, L, K) - 1
    assert 0 < extra < 0.02
