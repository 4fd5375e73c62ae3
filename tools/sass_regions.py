#!/usr/bin/env python3
"""Group an `ncu --page source --csv --print-source sass` dump into basic-block
runs (same execution count) and print each run's share of warp samples and its
top stall reasons -- where a kernel's warps spend their time.

usage: python tools/sass_regions.py dump.csv [min_share=0.005]
"""
import csv
import sys
from collections import Counter


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.005
    kernel = rows[0][1] if len(rows[0]) > 1 else "?"
    hdr, data = rows[1], [r for r in rows[2:] if r and r[0] != "Address"]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_e = hdr.index("Instructions Executed")
    sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r[i_s] or 0) for r in data) or 1
    groups = []
    for r in data:
        if len(r) <= i_e:
            continue
        e, s = int(r[i_e] or 0), int(r[i_s] or 0)
        toks = r[1].split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
        st = {hdr[i][6:]: int(r[i] or 0) for i in sc}
        if groups and groups[-1][1] == e:
            g = groups[-1]
            g[2] += s
            g[3] += 1
            g[4].append(op)
            for k, v in st.items():
                g[5][k] = g[5].get(k, 0) + v
        else:
            groups.append([r[0][-5:], e, s, 1, [op], st])
    print(kernel[:100], "samples", tot)
    for g in groups:
        if g[2] > tot * thr:
            t = sum(g[5].values()) or 1
            top = sorted(((k, round(v / t * 100)) for k, v in g[5].items() if v / t > 0.05), key=lambda x: -x[1])
            print(f"{g[0]} exec {g[1]:>10} {100 * g[2] / tot:5.1f}% n={g[3]:<5} {Counter(g[4]).most_common(3)} {top}")


if __name__ == "__main__":
    main()
