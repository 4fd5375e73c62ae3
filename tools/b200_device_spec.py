#!/usr/bin/env python3
"""Write the B200's DeviceSpec in the reference's JSON schema
(proj/include/kernelscope/device_spec.hpp:11-27; P100 example
proj/fixtures/p100.json) from the live device, for the reference's analysis
pipeline (oracle/_ref/ks_b200_report).

Roofs follow the reference fixture's convention (datasheet-style peaks):
peak_bw = 8000 GB/s (B200 HBM3e), peak_fp32 = SMs x 128 FP32 lanes x 2 FLOP x
max SM clock.  The measured copy bandwidth (MEASURED_PEAKS.json) is recorded
beside them as an extra key the reference parser ignores.

usage: python tools/b200_device_spec.py [out.json]
"""
import json
import os
import subprocess
import sys

import torch


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "profiles/b200_device_spec.json"
    p = torch.cuda.get_device_properties(0)
    clk = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.max.sm", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    mhz = float(clk) if clk else 1965.0
    spec = {
        "name": p.name,
        "sm_count": p.multi_processor_count,
        "warp_size": p.warp_size,
        "max_threads_per_block": 1024,
        "max_threads_per_sm": p.max_threads_per_multi_processor,
        "smem_per_block": p.shared_memory_per_block_optin,
        "smem_per_sm": p.shared_memory_per_multiprocessor,
        "registers_per_sm": p.regs_per_multiprocessor,
        "l2_bytes": p.L2_cache_size,
        "mem_bytes": p.total_memory,
        "peak_bw": 8000.0,
        "peak_fp32": round(p.multi_processor_count * 128 * 2 * mhz / 1e3, 1),
    }
    mp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        spec["measured_copy_bw_gbs"] = json.load(open(mp))["hbm_gbs"]
    with open(out, "w") as f:
        json.dump(spec, f, indent=2)
        f.write("\n")
    print(json.dumps(spec))


if __name__ == "__main__":
    main()
