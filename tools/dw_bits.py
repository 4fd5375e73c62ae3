#!/usr/bin/env python3
"""Write dk (HIERARCHICAL, both modes) at one shape to a .npy, for bitwise A/B
between two builds of the library (KS_LIB): python tools/dw_bits.py B H L K out.npy"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_25422_b200 as ks  # noqa: E402

B, H, L, K = (int(a) for a in sys.argv[1:5])
x, k, gy = ks.make_inputs(5, B, H, L, K)
out = [ks.backward_weight(gy, x, K, ks.HIERARCHICAL, 0, m).cpu().numpy() for m in (ks.SEPARATE, ks.FUSED)]
np.save(sys.argv[5], np.stack(out))
print("wrote", sys.argv[5])
