#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (committed evidence).

usage: python tools/ncu_summary.py ROUND [--launches gpurun_out/launches.csv]
                                   [--full name=gpurun_out/prof_x.ncu-rep ...]
       python tools/ncu_summary.py ROUND --config NAME --shape B H L K --run-shape LIST.csv

The --shape form reads the launch list of `tools/run_shape.py B H L K --reps 1
--bwd` (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum,launch__grid_size,launch__block_size,
launch__shared_mem_per_block_dynamic): three fill launches, then the fwd, dX,
dW and backward calls, segmented by the B200 traffic model's launch counts
(traffic.launch_geometry), into profiles/<ROUND>_launches_<NAME>.csv and
ncu_summary.json[NAME][fwd|dX|dW|bwd] = {dram_read, dram_write, ...}.

Writes
  profiles/<ROUND>_launches.csv      per-launch device time + DRAM bytes (the
                                     `--metrics gpu__time_duration.sum,...` pass)
  profiles/<ROUND>_<name>_full.txt   key metrics + top stall reasons of one
                                     `ncu --set full` capture per kernel
  profiles/ncu_summary.json          {config3: {fwd|dX|dW: {dram_bytes, ...}}},
                                     read by bench.py for roofline.traffic
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
]


def raw_page(rep):
    """rep: an .ncu-rep, or the `ncu -i rep --page raw --csv` export of one (.csv)."""
    if rep.endswith(".csv"):
        with open(rep) as f:
            out = f.read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def full_summary(name, rep, rnd):
    recs, units = raw_page(rep)
    lines, first = [], None
    for r in recs:
        first = first or r
        lines.append(f"kernel: {r.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in r:
                lines.append(f"  {k} = {r[k]} {units.get(k, '')}")
        stalls = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), num(v)) for k, v in r.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                  and num(v) is not None]
        tot = sum(v for _, v in stalls) or 1.0
        lines.append("  top stall reasons (pc sampling):")
        for k, v in sorted(stalls, key=lambda x: -x[1])[:8]:
            lines.append(f"    {k:28s} {100 * v / tot:5.1f}%")
    path = os.path.join(PROF, f"{rnd}_{name}_full.txt")
    with open(path, "w") as f:
        f.write(f"# ncu --set full --clock-control none --import-source on, capture {os.path.basename(rep)}\n")
        f.write("\n".join(lines) + "\n")
    print("wrote", path)
    return first, units


def launches(csv_path, rnd):
    with open(csv_path) as f:
        text = f.read()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in hdr}
    per = {}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        key = (int(r[ix["ID"]]), r[ix["Kernel Name"]], r[ix["Grid Size"]], r[ix["Block Size"]])
        per.setdefault(key, {})[r[ix["Metric Name"]]] = num(r[ix["Metric Value"]])
    out = os.path.join(PROF, f"{rnd}_launches.csv")
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "grid", "block", "time_us", "dram_read_bytes", "dram_write_bytes", "GB_s"])
        for (i, name, grid, block), m in sorted(per.items()):
            t = m.get("gpu__time_duration.sum") or 0.0
            rd, wr = m.get("dram__bytes_read.sum") or 0.0, m.get("dram__bytes_write.sum") or 0.0
            w.writerow([i, name[:90], grid, block, round(t / 1e3, 2), int(rd), int(wr),
                        round((rd + wr) / t, 1) if t else ""])
    print("wrote", out)
    return per


def run_shape_list(csv_path, rnd, config, shape):
    sys.path.insert(0, ROOT)
    from paper_2604_25422_b200 import traffic
    with open(csv_path) as f:
        text = f.read()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in hdr}
    per = {}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        key = (int(r[ix["ID"]]), r[ix["Kernel Name"]])
        per.setdefault(key, {})[r[ix["Metric Name"]]] = num(r[ix["Metric Value"]])
    launches_ = sorted(per.items())
    B, H, L, K = shape
    segs, i = {}, 3  # make_inputs: three fill launches first
    for path, name in (("fwd", "fwd"), ("dx", "dX"), ("dw", "dW"), ("bwd", "bwd")):
        n = len(traffic.launch_geometry(path, B, H, L, K))
        segs[name] = launches_[i:i + n]
        i += n
    out = os.path.join(PROF, f"{rnd}_launches_{config}.csv")
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["path", "id", "kernel", "grid", "block", "smem", "time_us", "dram_read_bytes", "dram_write_bytes"])
        for name, ls in segs.items():
            for (i_, kname), m in ls:
                w.writerow([name, i_, kname[:110], int(m.get("launch__grid_size") or 0),
                            int(m.get("launch__block_size") or 0), int(m.get("launch__shared_mem_per_block_dynamic") or 0),
                            round((m.get("gpu__time_duration.sum") or 0) / 1e3, 2),
                            int(m.get("dram__bytes_read.sum") or 0), int(m.get("dram__bytes_write.sum") or 0)])
    print("wrote", out)
    res = {}
    for name, ls in segs.items():
        rd = sum(m.get("dram__bytes_read.sum") or 0 for _, m in ls)
        wr = sum(m.get("dram__bytes_write.sum") or 0 for _, m in ls)
        main_ = max(ls, key=lambda kv: kv[1].get("gpu__time_duration.sum") or 0)
        res[name] = {"dram_bytes": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
                     "launches": len(ls), "kernel": traffic.kernel_family(main_[0][1]),
                     "ncu_time_us": round(sum((m.get("gpu__time_duration.sum") or 0) for _, m in ls) / 1e3, 2),
                     "round": rnd, "shape": list(shape)}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("round")
    ap.add_argument("--launches")
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--config", default="config3")
    ap.add_argument("--shape", type=int, nargs=4)
    ap.add_argument("--run-shape")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    summ_path = os.path.join(PROF, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    cfg = summ.setdefault(a.config, {})
    if a.run_shape:
        cfg.update(run_shape_list(a.run_shape, a.round, a.config, a.shape))
        with open(summ_path, "w") as f:
            json.dump(summ, f, indent=1, sort_keys=True)
        print("wrote", summ_path)
        return 0
    if a.launches:
        per = launches(a.launches, a.round)
        # per-path DRAM bytes from the last complete fwd/dX/dW triple
        def short_mode(n):  # bwd_short<K, FUSED, MODE>: 0 dW, 1 fused backward, 2 fwd, 3 dX
            if "bwd_short<" not in n:
                return None
            args = n.split("bwd_short<", 1)[1].split(">", 1)[0].split(",")
            return int(args[2]) if len(args) >= 3 else None

        def is_bwd(n):  # the fused backward: bwd_short MODE 1, or dw_tma<JR, TB, NJ, S, FUSED, BWD, S2>
            if short_mode(n) is not None:
                return short_mode(n) == 1
            if "dw_tma<" not in n:
                return False
            args = n.split("dw_tma<", 1)[1].split(">", 1)[0].split(",")
            return len(args) >= 6 and args[5].strip() in ("1", "true")

        def is_stencil(n):
            return "stencil" in n or "conv_tile" in n or short_mode(n) in (2, 3)

        def is_dw(n):
            return ("dw_tma" in n or "dw_hier" in n or short_mode(n) == 0) and not is_bwd(n)

        stencil = [m for (i, n, g, b), m in sorted(per.items()) if is_stencil(n)]
        dw = [m for (i, n, g, b), m in sorted(per.items()) if is_dw(n)]
        bwd = [m for (i, n, g, b), m in sorted(per.items()) if is_bwd(n)]
        if bwd:
            m = bwd[-1]
            cfg["bwd"] = {"dram_bytes": int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]),
                          "ncu_time_us": round(m["gpu__time_duration.sum"] / 1e3, 2), "round": a.round}
        # with the fused-backward step the list ends ... fwd, dX, dW | fwd, bwd:
        # take fwd and dX from the last split step (the stencils before the last dW)
        if bwd and dw:
            last_dw = max(i for (i, n, g, b) in per if is_dw(n))
            stencil = [m for (i, n, g, b), m in sorted(per.items()) if is_stencil(n) and i < last_dw]
        if len(stencil) >= 2:
            for name, m in (("fwd", stencil[-2]), ("dX", stencil[-1])):
                cfg[name] = {"dram_bytes": int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]),
                             "ncu_time_us": round(m["gpu__time_duration.sum"] / 1e3, 2), "round": a.round}
        if dw:
            m = dw[-1]
            cfg["dW"] = {"dram_bytes": int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]),
                         "ncu_time_us": round(m["gpu__time_duration.sum"] / 1e3, 2), "round": a.round}
    for spec in a.full:
        name, rep = spec.split("=", 1)
        full_summary(name, rep, a.round)
    if a.launches:  # only a launch list updates the per-path DRAM bytes bench.py reads
        with open(summ_path, "w") as f:
            json.dump(summ, f, indent=1, sort_keys=True)
        print("wrote", summ_path)


if __name__ == "__main__":
    sys.exit(main())
