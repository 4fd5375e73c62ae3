"""Generate the committed golden fixtures from the REFERENCE ITSELF.

Runs the reference's own src/conv_core.cpp (built from /root/reference by
oracle/Makefile into oracle/_ref/libksref.so) -- not our restatement -- on
seeded inputs from the reference's generator, and writes:

* ``small.npz``: inputs and every output (fwd/dX in both MulAddModes, dW under
  every scheme and both modes, fp64 fwd/dX/dW) for a set of small shapes that
  cover odd/even K, K=1, K>L, ragged L and multi-chunk dW;
* ``hashes.json``: SHA-256 of the fp32 outputs at BASELINE config 1
  (B=16,H=64,L=1024,K=64, seed 1) and of a config-3 channel slice, so larger
  cases are pinned without committing megabytes.

Run in a container that has /root/reference:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle.oracle import CHUNKED, FUSED, PAIRWISE, SEPARATE, SEQUENTIAL, Reference  # noqa: E402

SMALL_SHAPES = [  # (B, H, L, K, seed)
    (1, 1, 3, 3, 1), (2, 3, 17, 5, 7), (2, 2, 5, 4, 29), (3, 2, 33, 8, 3), (2, 2, 10, 16, 19),
    (4, 3, 64, 1, 11), (2, 2, 7, 12, 5), (1, 2, 300, 7, 13), (3, 3, 33, 9, 41), (8, 3, 32, 5, 17),
    (2, 1, 130, 64, 23), (4, 2, 48, 48, 1),
]
DW_SCHEMES = [("seq", SEQUENTIAL, 0), ("pair", PAIRWISE, 0), ("chunk7", CHUNKED, 7),
              ("chunk64", CHUNKED, 64), ("chunk1024", CHUNKED, 1024)]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ref = Reference()
    arrays = {}
    for (B, H, L, K, seed) in SMALL_SHAPES:
        tag = f"{B}x{H}x{L}x{K}s{seed}"
        x, k, gy = ref.fill_inputs(seed, B, H, L, K)
        arrays[f"{tag}/x"], arrays[f"{tag}/k"], arrays[f"{tag}/gy"] = x, k, gy
        for mname, m in (("sep", SEPARATE), ("fus", FUSED)):
            arrays[f"{tag}/y_{mname}"] = ref.forward(x, k, m)
            arrays[f"{tag}/dx_{mname}"] = ref.backward_input(gy, k, m)
            for sname, s, c in DW_SCHEMES:
                arrays[f"{tag}/dk_{sname}_{mname}"] = ref.backward_weight(gy, x, K, s, c, m)
        xd, kd, gyd = x.astype(np.float64), k.astype(np.float64), gy.astype(np.float64)
        arrays[f"{tag}/y_f64"] = ref.forward(xd, kd, SEPARATE)
        arrays[f"{tag}/dx_f64"] = ref.backward_input(gyd, kd, SEPARATE)
        arrays[f"{tag}/dk_f64"] = ref.backward_weight(gyd, xd, K, SEQUENTIAL, 0, SEPARATE)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **arrays)

    hashes = {}
    B, H, L, K = 16, 64, 1024, 64
    x, k, gy = ref.fill_inputs(1, B, H, L, K)
    hashes["config1_seed1"] = {
        "shape": [B, H, L, K],
        "x": sha(x), "k": sha(k), "gy": sha(gy),
        "y_sep": sha(ref.forward(x, k, SEPARATE)), "y_fus": sha(ref.forward(x, k, FUSED)),
        "dx_sep": sha(ref.backward_input(gy, k, SEPARATE)),
        "dx_fus": sha(ref.backward_input(gy, k, FUSED)),
        "dk_pair": sha(ref.backward_weight(gy, x, K, PAIRWISE, 0, SEPARATE)),
        "dk_chunk1024_fus": sha(ref.backward_weight(gy, x, K, CHUNKED, 1024, FUSED)),
    }
    with open(os.path.join(HERE, "hashes.json"), "w") as f:
        json.dump(hashes, f, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays, {len(hashes)} hash sets")


if __name__ == "__main__":
    main()
