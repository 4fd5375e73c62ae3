"""B200 variant of the reference's execution/traffic model.

The reference models the paper's four P100 kernels analytically
(/root/reference/proj/src/exec_model.cpp: ``launch_geometry`` :80-105,
``shared_mem_footprint``, ``logical_traffic`` :168-179, ``memory_traffic``
:181-208).  This module gives the same three views for this library's
kernels, so the counter-free methodology of the paper (timings + a traffic
model) extends to B200:

* ``logical_traffic(path, B, H, L, K)`` -- the reference's algorithmic bytes,
  8*B*H*L + 4*H*K per path (unchanged definition);
* ``memory_traffic(path, B, H, L, K, scheme)`` -- modeled DRAM bytes of the
  B200 kernels: the algorithmic bytes plus what the kernels add on top (tap
  staging, dW per-CTA partials written and read back), with halo re-reads
  served from L2 (each halo row is the neighbour tile's body and is resident);
* ``l2_traffic`` -- modeled L2->SM bytes, which *do* include the halo re-reads
  (TMA boxes overlap by 32*HH floats per side per tile);
* ``plan(path, B, H, L, K)`` -- which kernel family runs, its tile and grid
  (mirrors the host dispatch in csrc/: conv_fwd.cu, stencil_ldg.cu,
  stencil_tma.cu, bwd_short.cuh, stencil_pad.cu, rows_short.cu, conv_dw.cu, dw_*.cu).

``tests/test_traffic.py`` checks memory_traffic against the ncu DRAM bytes
committed in profiles/ncu_summary.json.
"""
from __future__ import annotations

import math

SMS = 148


def logical_traffic(path: str, B: int, H: int, L: int, K: int) -> int:
    """Reference src/exec_model.cpp:168-179: read one [B,H,L] tensor and k,
    write one [B,H,L] tensor (dW: read gy and x, write dk)."""
    return 8 * B * H * L + 4 * H * K


def _stencil_tier(L: int, K: int):
    if L < 1024 and L % 4 == 0 and L + K - 1 <= 252:
        return "stencil_rows", 16, None
    if L % 32 != 0 or K > 8192:
        return "conv_tile_f32", 16 if L > 1024 else 4, 256
    if K > 32 and L >= 1024:
        return "stencil_pad", 32, 128  # padded TMA view, 128 FMA threads + 1 producer lane
    if K <= 8 and L >= 1024:
        return "stencil_ldg", 8, 256  # stencil_ldg.cu: CTA = (row, 2048-output tile), register windows
    if K <= 16 and L >= 1024:
        return "stencil_short", 8, 256  # bwd_short.cuh MODE fwd/dX: 2048-output tiles, persistent
    if L >= 1024:
        nt = 256 if L >= 4096 and K <= 8 else 128 if L >= 2048 else 64
        return "stencil_tma", 16, nt
    return "stencil_tma", 4, 256


def _dw_groups(B: int, H: int, L: int, K: int) -> tuple[str, int]:
    if K >= 128 and L >= 2048 and L % 32 == 0:
        njg = 4
        while njg < 32 and njg * 32 < K:
            njg *= 2
        njt = math.ceil(K / (njg * 32))
        G = max(1, min(math.ceil(2048 / (H * njt)), B))
        return "dw_pad", G
    groups8 = math.ceil(K / 8)
    nj = 1
    while nj < 8 and nj < groups8:
        nj *= 2
    njt = math.ceil(K / (nj * 8))
    G = max(1, min(math.ceil(8192 / (H * njt)), B))
    if L < 2048 and L % 4 == 0:
        return "dw_rows", G
    if L % 32 == 0 and K <= 16:
        return "dw_short", G  # bwd_short.cuh MODE dW: dw_tma's decomposition, K-specialised
    return ("dw_tma" if L % 32 == 0 else "dw_hier_stage1"), G


def bwd_fused_applies(L: int, K: int) -> bool:
    """ks_dwconv1d_bwd_f32 runs the one-pass kernel (csrc/bwd_short.cuh MODE fused)."""
    return L % 32 == 0 and L >= 2048 and K <= 16


def plan(path: str, B: int, H: int, L: int, K: int, scheme: str = "hierarchical") -> dict:
    """Kernel family, register tile / threads and tile geometry for a shape.
    ``path`` is fwd, dx, dw or bwd (the fused backward entry point)."""
    if path == "bwd":
        if bwd_fused_applies(L, K):
            _, G = _dw_groups(B, H, L, K)
            return {"kernel": "bwd_short", "row_groups": G, "partials_bytes": 4 * G * H * K}
        return {"kernel": "split", "dx": plan("dx", B, H, L, K), "dw": plan("dw", B, H, L, K)}
    if path in ("fwd", "dx"):
        name, R, NT = _stencil_tier(L, K)
        T = (NT or 0) * R if NT else None
        tiles = B * H * math.ceil(L / T) if T else None
        return {"kernel": name, "R": R, "threads": NT, "outputs_per_tile": T, "tiles": tiles}
    if scheme == "pairwise" and B & (B - 1) == 0 and L & (L - 1) == 0 and L >= 2048:
        return {"kernel": "dw_pairwise_tma", "tree": "perfect binary over b*L+t"}
    name, G = _dw_groups(B, H, L, K)
    return {"kernel": name, "row_groups": G, "partials_bytes": 4 * G * H * K}


def memory_traffic(path: str, B: int, H: int, L: int, K: int, scheme: str = "hierarchical") -> int:
    """Modeled DRAM bytes per launch of the B200 kernels."""
    if path == "bwd":
        p = plan(path, B, H, L, K)
        if p["kernel"] == "split":
            return memory_traffic("dx", B, H, L, K) + memory_traffic("dw", B, H, L, K)
        # one pass: read gy and x, write dx, read k; partials out and back
        return 12 * B * H * L + 4 * H * K + 2 * p["partials_bytes"]
    base = logical_traffic(path, B, H, L, K)
    p = plan(path, B, H, L, K, scheme)
    if path in ("fwd", "dx"):
        kp = 4 * H * (16 if p["kernel"] in ("stencil_short", "stencil_ldg") else math.ceil(K / 32) * 32)
        # prep_taps writes kp, the kernel reads it back
        return base + (2 * kp if p["kernel"] in ("stencil_tma", "stencil_pad", "stencil_short", "stencil_ldg") else 0)
    if p["kernel"] == "dw_pairwise_tma":
        return base
    return base + 2 * p["partials_bytes"]  # partials written by stage 1, read by stage 2


def l2_traffic(path: str, B: int, H: int, L: int, K: int) -> int:
    """Modeled L2->SM bytes of the stencil kernels: each tile re-reads its
    halo (32*HH floats per side) from L2."""
    p = plan(path, B, H, L, K)
    if path not in ("fwd", "dx") or not p["tiles"]:
        return memory_traffic(path, B, H, L, K)
    off = K // 2 if path == "fwd" else K - 1 - K // 2
    if p["kernel"] == "stencil_ldg":  # window quads past each 2048-output tile (the rest hits L1)
        halo = p["tiles"] * 2 * 4 * math.ceil((max(off, K - 1 - off) + 3) / 4) * 4
        return memory_traffic(path, B, H, L, K) + halo
    HH = 1 if p["kernel"] == "stencil_short" else max(1, math.ceil(max(off, K - 1 - off) / 32))
    halo = p["tiles"] * 2 * 32 * HH * 4
    return memory_traffic(path, B, H, L, K) + halo
