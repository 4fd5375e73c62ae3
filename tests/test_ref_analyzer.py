"""CPU: B200 timings through the REFERENCE's own analysis pipeline (SURVEY
§8(f) rank 2).

oracle/_ref/ks_b200_report is the reference's src/timing_log.cpp,
analyzer.cpp, exec_model.cpp, report.cpp and svg.cpp compiled from
/root/reference by oracle/Makefile, driven by oracle/ref_shim/b200_report.cpp
(the CLI's `analyze` front end needs CLI11 / nlohmann-json, absent from the
reference tree).  Inputs are committed evidence from one B200:
profiles/b200_device_spec.json (tools/b200_device_spec.py: the reference's
DeviceSpec schema) and the ablation timing logs of tools/ablation.py in the
reference's timing-CSV schema -- the paper's four designs as sm_100a kernels,
and this library beside the paper's naive design.
"""
import csv
import glob
import io
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "ks_b200_report")
SPEC = os.path.join(ROOT, "profiles", "b200_device_spec.json")
LOGS = sorted(glob.glob(os.path.join(ROOT, "profiles", "r02_ablation_*_paper.csv")) +
              glob.glob(os.path.join(ROOT, "profiles", "r02_ablation_*_library.csv")))

pytestmark = pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/ks_b200_report not built")


def _shape(log):
    with open(log) as f:
        head = f.readline()
    s = head.split("(B,H,L,K)=(", 1)[1].split(")", 1)[0]
    return [int(v) for v in s.split(",")]


def _mean_drop_warmup(vals):
    """The reference's aggregate (src/analyzer.cpp:19-32): drop the first
    sample when there are >= 3, then average."""
    vals = list(vals)
    if len(vals) >= 3:
        vals = vals[1:]
    return sum(vals) / len(vals)


def test_device_spec_has_the_reference_schema():
    spec = json.load(open(SPEC))
    for k in ("name", "sm_count", "warp_size", "max_threads_per_block", "max_threads_per_sm", "smem_per_block",
              "smem_per_sm", "registers_per_sm", "l2_bytes", "mem_bytes", "peak_bw", "peak_fp32"):
        assert k in spec, k
    assert spec["sm_count"] == 148 and spec["peak_bw"] > 0 and spec["peak_fp32"] > 0


@pytest.mark.parametrize("log", LOGS, ids=[os.path.basename(p) for p in LOGS])
def test_reference_report_over_b200_timings(log, tmp_path):
    """parse_timing_csv + build_report accept the B200 logs; the speedups the
    reference computes equal the ones recomputed here from the same rows with
    the reference's warm-up rule."""
    B, H, L, K = _shape(log)
    r = subprocess.run([EXE, log, SPEC, str(B), str(H), str(L), str(K), str(tmp_path)],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    for f in ("report.txt", "speedups.csv", "bandwidth.csv", "roofline.csv", "roofline.svg"):
        assert (tmp_path / f).stat().st_size > 0, f
    rows = list(csv.DictReader(io.StringIO("".join(l for l in open(log) if not l.startswith("#")))))
    ms = {}
    for row in rows:
        ms.setdefault((row["variant"], row["path"]), []).append(float(row["runtime_ms"]))
    mean = {k: _mean_drop_warmup(v) for k, v in ms.items()}
    sp = list(csv.DictReader(open(tmp_path / "speedups.csv")))
    assert sp and sp[0]["variant"] == "naive"
    for row in sp:
        v = row["variant"]
        total = sum(mean[(v, p)] for p in ("fwd", "bwd_in", "bwd_k"))
        base = sum(mean[("naive", p)] for p in ("fwd", "bwd_in", "bwd_k"))
        assert abs(float(row["conv_total"]) - base / total) <= 1e-3 * base / total + 1e-3, (v, row)
    if log.endswith("_library.csv"):  # this library (logged as 'warp') beats the paper's naive design
        lib = next(r_ for r_ in sp if r_["variant"] == "warp")
        assert float(lib["conv_total"]) > 1.0
