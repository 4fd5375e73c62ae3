#!/usr/bin/env python3
"""Tabulate a tools/_ab*.sh log (time_paths.py output per variant / rep / shape):
median ms per (shape, path, variant).  usage: python tools/ab_table.py ab.log"""
import re
import sys
from collections import defaultdict

d = defaultdict(list)
var = shape = None
for ln in open(sys.argv[1]):
    m = re.match(r"== (\S+)", ln)
    if m:
        var = m.group(1)
        continue
    m = re.match(r"shape ([\d ]+?) env", ln)
    if m:
        shape = m.group(1)
        continue
    m = re.match(r"\s+(\w+)\s+([\d.]+) ms", ln)
    if m and var and m.group(1) != "copy":
        d[(shape, m.group(1), var)].append(float(m.group(2)))
vars_ = sorted({k[2] for k in d})
keys = sorted({(k[0], k[1]) for k in d})
print("shape".ljust(22), "path".ljust(5), *[v.rjust(10) for v in vars_], "  ratio")
for s, p in keys:
    vals = [sorted(d[(s, p, v)])[len(d[(s, p, v)]) // 2] if d[(s, p, v)] else float("nan") for v in vars_]
    print(s.ljust(22), p.ljust(5), *[f"{x:10.4f}" for x in vals], f"  {vals[0] / vals[-1]:.3f}" if len(vals) > 1 else "")
