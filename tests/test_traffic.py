"""CPU: the B200 traffic model (paper_2604_25422_b200/traffic.py) against the
reference's algorithmic bytes, the committed ncu DRAM measurements and the
library's own launch plans (ks_dwconv1d_plan, dumped on a B200 by
tools/dump_plans.py into profiles/r02_plans.json)."""
import json
import os

import pytest

from paper_2604_25422_b200 import traffic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_logical_traffic_matches_reference_formula():
    # reference tests/test_exec_model.cpp:124-126: 402,677,760 read + 402,653,184 written
    assert traffic.logical_traffic("fwd", 16384, 128, 48, 48) == 402677760 + 402653184


def test_plan_dispatch_tiers():
    assert traffic.plan("fwd", 256, 512, 8192, 7)["kernel"] == "stencil_ldg"
    assert traffic.plan("fwd", 512, 1024, 16384, 16)["kernel"] == "stencil_short"
    assert traffic.plan("fwd", 64, 128, 4096, 4096)["kernel"] == "stencil_bl"  # K >= L / 4, B >= 32
    assert traffic.plan("fwd", 16, 128, 4096, 4096)["kernel"] == "stencil_pad"  # fewer than 32 rows
    # the model follows Separate mode (the reference's default): register tiles below K = 1024
    assert traffic.plan("fwd", 1024, 256, 2048, 256)["kernel"] == "stencil_tma"
    assert traffic.plan("fwd", 512, 1024, 16384, 1024)["kernel"] == "stencil_pad"
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


def _plans():
    with open(os.path.join(ROOT, "profiles", "r02_plans.json")) as f:
        return json.load(f)


def test_launch_geometry_matches_the_library_plans():
    """Every launch of every entry point at every BASELINE config, the
    multi-GPU shards and the paper's shape: kernel family, grid, block and
    dynamic shared memory as the real dispatch chose them.  Persistent grids
    take the occupancy the CUDA occupancy API reported."""
    plans = _plans()
    checked = 0
    for name, d in plans.items():
        B, H, L, K = d["shape"]
        for path in ("fwd", "dx", "dw", "bwd"):
            real = [(traffic.kernel_family(r["kernel"]), r["grid"][0], r["block"][0], r["smem"]) for r in d[path]]
            occ = {(r["block"][0], r["smem"]): r["ctas_per_sm"] for r in d[path]}
            model = [(g["kernel"], g["grid"], g["block"], g["smem"])
                     for g in traffic.launch_geometry(path, B, H, L, K, occ=lambda t, sm: occ[(t, sm)])]
            assert model == real, (name, path, model, real)
            checked += 1
    assert checked >= 50


def test_shared_mem_footprint_and_plan_families():
    plans = _plans()
    for name, d in plans.items():
        B, H, L, K = d["shape"]
        for path in ("fwd", "dx", "dw", "bwd"):
            assert traffic.shared_mem_footprint(path, B, H, L, K) == max(r["smem"] for r in d[path]), (name, path)
        fam = {traffic.kernel_family(r["kernel"]) for r in d["dw"]}
        want = traffic.plan("dw", B, H, L, K)["kernel"]
        assert {"dw_short": "bwd_short"}.get(want, want) in fam, (name, want, fam)


def test_resource_check_matches_the_occupancy_api():
    """The reference's resource_check with sm_100 limits (shared memory with
    the maximum carveout the library requests, threads, registers) gives the
    CTAs/SM the CUDA occupancy API reported for every planned kernel."""
    for name, d in _plans().items():
        for path in ("fwd", "dx", "dw", "bwd", "dw_pairwise"):
            for r in d[path]:
                threads = r["block"][0] * r["block"][1] * r["block"][2]
                got = traffic.resource_check(threads, r["smem"], r["regs"], r["static_smem"])
                assert got == r["ctas_per_sm"], (name, path, r)


L2_BYTES = 132644864  # profiles/b200_device_spec.json: dirty lines can stay in L2 past a kernel's end


@pytest.mark.parametrize("cfg", ["config2", "config3", "config4", "config5a", "config5b", "config5c_g8"])
def test_memory_traffic_matches_ncu_dram_bytes_per_path(cfg):
    """memory_traffic_rw against ncu's DRAM bytes (cold-cache replay) summed
    over every launch of each entry point (tools/ncu_summary.py --shape, from
    the launch lists of tools/run_shape.py at the full config): reads within
    1% of the model, plus at most the halo re-reads (traffic.halo_bytes: L2
    hits at short K, partly DRAM at long K); writes at most the model and at
    least the model less one L2 (a kernel's last dirty lines -- and dW's
    partials, read straight back -- may leave L2 after it ends)."""
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
        meas = json.load(f)[cfg]
    for path, key in (("fwd", "fwd"), ("dx", "dX"), ("dw", "dW"), ("bwd", "bwd")):
        B, H, L, K = meas[key]["shape"]
        rd, wr = traffic.memory_traffic_rw(path, B, H, L, K)
        halo = traffic.halo_bytes(path, B, H, L, K)
        got_rd, got_wr = meas[key]["dram_read"], meas[key]["dram_write"]
        assert 0.99 * rd - (8 << 20) <= got_rd <= 1.01 * (rd + halo) + (16 << 20), (cfg, path, got_rd, rd, halo)
        assert wr - L2_BYTES - (1 << 20) <= got_wr <= 1.01 * wr + (4 << 20), (cfg, path, got_wr, wr)
        assert meas[key]["launches"] == len(traffic.launch_geometry(path, B, H, L, K))
