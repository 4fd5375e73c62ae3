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
  stencil_tma.cu, bwd_short.cuh, stencil_pad.cu, rows_short.cu, conv_dw.cu, dw_*.cu);
* ``launch_geometry(path, B, H, L, K)`` -- every launch of the call (kernel
  family, grid, block, dynamic shared memory), the counterpart of the
  reference's ``launch_geometry`` (exec_model.hpp:14-60);
* ``shared_mem_footprint(path, B, H, L, K)`` -- dynamic shared memory of the
  call's main kernel, the counterpart of the reference's
  ``shared_mem_footprint`` (exec_model.hpp:62-80);
* ``resource_check(...)`` -- resident CTAs per SM from shared memory, threads
  and registers (the reference's ``resource_check``, exec_model.cpp:136-166).

Pinned, on the CPU, by ``tests/test_traffic.py`` against what the hardware
and the library report: memory_traffic against ncu's DRAM bytes for configs
2, 3, 4, 5a and 5b (profiles/ncu_summary.json), launch_geometry /
shared_mem_footprint / plan against the library's own dispatch run without
launching (ks_dwconv1d_plan, profiles/r02_plans.json, every config and the
multi-GPU shards).
"""
from __future__ import annotations

import math

SMS = 148
SMEM_PER_SM = 233472     # bytes (228 KiB) of shared memory per SM at the largest carveout
SMEM_RESERVED = 1024     # per resident CTA (the runtime's)
REGS_PER_SM = 65536
THREADS_PER_SM = 2048
MAX_CTAS_PER_SM = 32


def resource_check(threads: int, smem: int, regs: int | None = None, static_smem: int = 0) -> int:
    """Resident CTAs per SM (the reference's resource_check,
    src/exec_model.cpp:136-166, with sm_100's limits): the smallest of the
    shared-memory (dynamic + static + the runtime's 1 KiB per CTA), thread,
    register and CTA-slot limits.  Registers are allocated per warp in units
    of 256."""
    per_cta = smem + static_smem + SMEM_RESERVED
    lim = [MAX_CTAS_PER_SM, THREADS_PER_SM // threads, SMEM_PER_SM // per_cta]
    if regs:
        per_warp = -(-regs * 32 // 256) * 256
        lim.append(REGS_PER_SM // (per_warp * -(-threads // 32)))
    return max(0, min(lim))


def _cdiv(a: int, b: int) -> int:
    return -(-a // b)


def logical_traffic(path: str, B: int, H: int, L: int, K: int) -> int:
    """Reference src/exec_model.cpp:168-179: read one [B,H,L] tensor and k,
    write one [B,H,L] tensor (dW: read gy and x, write dk)."""
    return 8 * B * H * L + 4 * H * K


def _stencil_tier(L: int, K: int, B: int = 1):
    if L < 1024 and L % 4 == 0 and L + K - 1 <= 252:
        return "stencil_rows", 16, None
    if L % 4 == 0 and L >= 256 and (K <= 10 or (L < 2048 and K <= 12) or (L % 32 != 0 and K <= 16)
                                     or (L < 1024 and K <= 32)):
        # Separate mode's rule (stencil_ldg_f32)
        return "stencil_ldg", 8, 256  # stencil_ldg.cu: CTA = (row, 2048-output tile), register windows
    if L % 32 != 0 or K > 8192:
        return "conv_tile_f32", 16 if L > 1024 else 4, 256
    if K > 32 and L >= 1024 and B >= 32 and 4 * K >= L:
        return "stencil_bl", 32, 128  # batch lanes: 32 rows x 128 outputs per CTA + 1 producer lane
    if K > 32 and L >= 1024 and K >= 1024:
        return "stencil_pad", 32, 128  # padded TMA view, 128 FMA threads + 1 producer lane
    # Separate mode (the reference's default, which this model and the committed
    # plans follow) below K = 1024: stencil_tma's register tiles (Fused mode
    # takes stencil_pad here too)
    if K <= 28 and L >= 1024:  # Separate mode's rule (stencil_tma_f32)
        return "stencil_short", 8, 256  # bwd_short.cuh MODE fwd/dX: 2048-output tiles, persistent
    if K > 32 and L >= 2048:  # stencil_tma.cu pick_tile
        return "stencil_tma", 32, 256 if L >= 8192 else 128 if L >= 4096 else 64
    if L >= 1024:
        nt = 256 if L >= 4096 and K <= 8 else 128 if L >= 2048 else 64
        return "stencil_tma", 16, nt
    return "stencil_tma", 4, 256 if L > 512 else 128 if L > 256 else 64 if L > 128 else 32


def _dwpad_njg(K: int) -> int:
    p = K // 2
    kk = K - (p % 32 - 32 if p % 32 else 0)
    njg = 1
    while njg < 32 and njg * 32 < kk:
        njg *= 2
    return njg


def _dw_groups(B: int, H: int, L: int, K: int) -> tuple[str, int]:
    # dw_pad.cu dw_pad_applies: K >= 48 (option dwpad_min_k), a row at least one work item long
    if K >= 48 and L >= 2048 and L % 32 == 0 and L >= 32 * (256 // _dwpad_njg(K)):
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
    target = min(8192, max(256, (B * H * L * K) // 262144))  # conv_dw.cu hier_plan: >= 2^18 MACs per CTA
    G = max(1, min(math.ceil(target / (H * njt)), B))
    if L < 2048 and L % 4 == 0 and L + 8 * min(8, groups8) + 16 <= 252:  # dw_rows: a whole row in one TMA box
        return "dw_rows", G
    if L % 32 == 0 and K <= 32:
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
        name, R, NT = _stencil_tier(L, K, B)
        if name == "stencil_bl":  # a tile = 32 batch rows x 128 outputs of one channel
            return {"kernel": name, "R": R, "threads": NT, "outputs_per_tile": 32 * 128,
                    "tiles": math.ceil(B / 32) * H * math.ceil(L / 128)}
        T = (NT or 0) * R if NT else None
        tiles = B * H * math.ceil(L / T) if T else None
        return {"kernel": name, "R": R, "threads": NT, "outputs_per_tile": T, "tiles": tiles}
    if scheme == "pairwise" and B & (B - 1) == 0 and L & (L - 1) == 0 and L >= 2048:
        return {"kernel": "dw_pairwise_tma", "tree": "perfect binary over b*L+t"}
    name, G = _dw_groups(B, H, L, K)
    return {"kernel": name, "row_groups": G, "partials_bytes": 4 * G * H * K}


def memory_traffic_rw(path: str, B: int, H: int, L: int, K: int, scheme: str = "hierarchical") -> tuple:
    """Modeled DRAM (read, write) bytes of one entry-point call, all its
    launches: the compulsory tensor bytes, the taps staging (prep_taps reads k
    and writes kp, which the kernel reads back) and dW's per-CTA partials
    (written by stage 1, read back by the fixed-order pass).  Halo re-reads
    hit L2 (each halo is a neighbouring tile's body) and are not DRAM bytes."""
    T = 4 * B * H * L
    kb = 4 * H * K
    if path == "bwd":
        p = plan(path, B, H, L, K)
        if p["kernel"] == "split":
            a, b = memory_traffic_rw("dx", B, H, L, K), memory_traffic_rw("dw", B, H, L, K)
            return a[0] + b[0], a[1] + b[1]
        # one pass: read gy, x and k, write dx; partials out and back; dk out
        return 2 * T + kb + p["partials_bytes"], T + p["partials_bytes"] + kb
    p = plan(path, B, H, L, K, scheme)
    if path in ("fwd", "dx"):
        staged = p["kernel"] in ("stencil_tma", "stencil_pad", "stencil_bl", "stencil_short", "stencil_ldg")
        kp = 4 * H * (16 if p["kernel"] in ("stencil_short", "stencil_ldg") else math.ceil(K / 32) * 32)
        return T + kb + (kp if staged else 0), T + (kp if staged else 0)
    if p["kernel"] == "dw_pairwise_tma":
        return 2 * T, kb
    return 2 * T + p["partials_bytes"], p["partials_bytes"] + kb


def memory_traffic(path: str, B: int, H: int, L: int, K: int, scheme: str = "hierarchical") -> int:
    """Modeled DRAM bytes (read + write) of one entry-point call."""
    return sum(memory_traffic_rw(path, B, H, L, K, scheme))


def halo_bytes(path: str, B: int, H: int, L: int, K: int) -> int:
    """Bytes a forward / dX call re-reads beyond the tensor: every tile's
    window overhangs its outputs by the halo (the neighbouring tiles' bodies).
    They are L2 hits while the neighbour's data is resident, DRAM re-reads
    otherwise -- a persistent grid visits a row's tiles far apart, so at long K
    (stencil_pad: a 4096-output tile carries a Kp-wide window overhang) a few
    percent of the tensor is read twice from DRAM (ncu: 3.9% at config 5c)."""
    if path == "bwd":
        p = plan(path, B, H, L, K)
        if p["kernel"] == "split":
            return halo_bytes("dx", B, H, L, K)
        return B * H * _cdiv(L, 2048) * 2 * 128  # the gy box's halo piece on each side of a 2048-wide item
    if path not in ("fwd", "dx"):
        return 0
    p = plan(path, B, H, L, K)
    off = K // 2 if path == "fwd" else K - 1 - K // 2
    if p["kernel"] == "stencil_ldg":  # window quads past each 2048-output tile (the rest hits L1)
        return B * H * _cdiv(L, 2048) * 2 * 4 * math.ceil((max(off, K - 1 - off) + 3) / 4) * 4
    if p["kernel"] == "stencil_pad":
        lead = (32 - off % 32) % 32
        Kp = _cdiv(K + lead - (lead & 3), 32) * 32
        return B * H * _cdiv(L, 4096) * (Kp + 32) * 4
    if p["kernel"] == "stencil_bl":  # every CTA streams its pieces: the 128 outputs' valid window
        return sum(n * 32 * 128 for n in _bl_pieces(B, H, L, K, off)) * _cdiv(B, 32) * H - 4 * B * H * L
    if not p["tiles"]:
        return 0
    HH = 1 if p["kernel"] == "stencil_short" else max(1, math.ceil(max(off, K - 1 - off) / 32))
    return p["tiles"] * 2 * 32 * HH * 4


def l2_traffic(path: str, B: int, H: int, L: int, K: int) -> int:
    """Modeled L2->SM bytes: the DRAM model plus every halo re-read."""
    return memory_traffic(path, B, H, L, K) + halo_bytes(path, B, H, L, K)


# ---------------------------------------------------------------------------
# launch geometry (grid, block, dynamic shared memory) per kernel family

def _launch(kernel, grid, block, smem):
    return {"kernel": kernel, "grid": int(grid), "block": int(block), "smem": int(smem)}


def _prep_taps(H: int, Kp: int):
    return _launch("prep_taps", min(_cdiv(H * Kp, 256), 4096), 256, 0)


def _bwd_short(mode: str, B, H, L, K, G, occ):
    """bwd_short.cuh Geo<KT, MODE>: 144-byte pieces, a 66-piece x window."""
    gyp = 64 if mode == "dw" else 66
    gy_region = _cdiv(gyp * 144, 128) * 128
    x_region = _cdiv(66 * 144, 128) * 128
    has_dw, has_st = mode in ("dw", "fused"), mode in ("fused", "fwd", "dx")
    mrow = mode == "dw" and L < 2048  # items of whole rows: each row's x window has its own 2 halo pieces
    if mrow:
        x_region = _cdiv((64 + 2 * 8) * 144, 128) * 128
    stage = gy_region + (x_region if has_dw else 0) + (128 if mode in ("fwd", "dx") else 0)
    ns = 4 if mode in ("fwd", "dx") else 3 if mrow else (4 if K <= 8 else 3)
    smem = (2 * 8192 if has_st else 0) + ns * stage + 64 + 1024
    # stencils: persistent in Separate mode (the plans and this model are for
    # Separate, the reference's default); Fused mode launches one CTA per row
    grid = G * H if has_dw else min(B * H, SMS * occ(256, smem))
    return _launch("bwd_short", grid, 256, smem)


def _stencil_pad(B, H, L, K, off, occ):
    """stencil_pad.cu PadGeom: 128 FMA threads x 32 outputs, 36-float rows."""
    nt, kr = 128, 32
    lead = (32 - off % 32) % 32
    S = lead & 3
    Kp = _cdiv(K + lead - S, 32) * 32
    rpt = 1
    while rpt < 4 and nt * kr // (2 * rpt) >= L and H % (2 * rpt) == 0:
        rpt *= 2
    T = nt // rpt * kr
    mirror = T >= L and 4 * K >= L and (nt // rpt) % 64 == 0  # the mirrored lane rings (K comparable to L)
    nr = T // 32 + Kp // 32 + (1 if S >= 2 else 0)
    nbox, nb = (1, nr) if nr <= 256 else (2, ((nr + 1) // 2 + 7) // 8 * 8)
    Kpp = Kp // 32 * 36 if mirror else Kp  # mirrored: taps at the window's 36-float pitch per 32-tap block
    stage = _cdiv(rpt * nbox * nb * 36 * 4 + rpt * Kpp * 4, 1024) * 1024
    ns = 1 if K >= 1024 else 2
    while ns > 1 and ns * stage + 1152 > 110 * 1024:
        ns -= 1
    smem = ns * stage + 128 + 1024
    threads = nt + (32 if K < 1024 else 0)
    tiles = B * H // rpt * _cdiv(L, T)
    prep = _launch("prep_taps_pad36" if mirror else "prep_taps", min(_cdiv(H * Kpp, 256), 4096), 256, 0)
    return [prep, _launch("stencil_pad", min(tiles, SMS * occ(threads, smem)), threads, smem)]


def _stencil_tma(B, H, L, K, off, R, NT, occ):
    """stencil_tma.cu StencilGeom: NT threads x R outputs per tile, a window of
    128-byte rows with HH halo rows each side, taps at Kp = ceil(K/32)*32."""
    T = NT * R
    mr = T // 32
    hh = max(1, _cdiv(max(off, K - 1 - off), 32))
    w = mr + 2 * hh
    nbox, nb = (1, w) if w <= 256 else (2, w // 2)
    kp = _cdiv(K, 32) * 32
    stage = _cdiv(nbox * nb * 128 + kp * 4, 1024) * 1024
    out_bytes = _cdiv(T * 4, 1024) * 1024
    tma_out = R != 32
    smem_of = lambda n: n * stage + (2 * out_bytes if tma_out else 0) + 64 + 1024  # noqa: E731
    ns = 2 if K > 8 else 3
    while ns > 2 and smem_of(ns) > 110 * 1024:
        ns -= 1
    if R == 32:
        ns = 1 if K >= 1024 else 2
    smem = smem_of(ns)
    tiles = B * H * _cdiv(L, T)
    return [_prep_taps(H, kp), _launch("stencil_tma", min(tiles, SMS * occ(NT, smem)), NT, smem)]


def _bl_geom(K, off):
    lead = (32 - off % 32) % 32
    S, zlead = lead & 3, lead - (lead & 3)
    Kp = _cdiv(K + zlead, 32) * 32
    return S, zlead, Kp, (off + lead) // 32


def _bl_pieces(B, H, L, K, off):
    """Pieces each CTA of one row group and channel streams, per output column
    tile (stencil_bl's union of its four warps' valid tap blocks)."""
    S, zlead, Kp, base_row = _bl_geom(K, off)
    xp = 2 if S >= 2 else 1
    out = []
    for col in range(_cdiv(L, 128)):
        lo_p, hi_p = None, None
        for c in range(4):
            ts = col * 128 + 32 * c
            if ts >= L:
                continue
            lo = max(0, (off + zlead - 31 - (ts + 31) + 31 + 32 * 64) // 32 - 64)
            hi = min(Kp // 32, (L + off + zlead - ts + 31) // 32)
            if lo < hi:
                q0 = ts // 32 - base_row
                lo_p = q0 + lo if lo_p is None else min(lo_p, q0 + lo)
                hi_p = q0 + hi - 1 + xp if hi_p is None else max(hi_p, q0 + hi - 1 + xp)
        out.append(0 if lo_p is None else hi_p - lo_p + 1)
    return out


def _stencil_bl(B, H, L, K, off):
    """stencil_pad.cu BlGeom: 4 consumer warps + a producer, an 8-slot ring of
    32-row pieces, the channel's prepared taps staged once."""
    _, _, Kp, _ = _bl_geom(K, off)
    smem = 8 * 32 * 144 + Kp * 4 + 256 + 1024
    return [_prep_taps(H, Kp), _launch("stencil_bl", _cdiv(L, 128) * _cdiv(B, 32) * H, 160, smem)]


def _dw_pad(B, H, L, K, G):
    """dw_pad.cu DwPadGeom: 256 FMA threads + a producer warp, 32 taps per thread."""
    p = K // 2
    base = p % 32 - 32 if p % 32 else 0
    kk = K - base
    njg = _dwpad_njg(K)
    nts = 256 // njg
    jt = njg * 32
    njt = _cdiv(kk, jt)
    tt = min(max(min(max(64 * nts, 4096), L), 32 * nts), 8192)
    gy_rows = tt // 32
    gy_alloc = _cdiv(gy_rows, 8) * 8
    xr = (tt + jt) // 32
    nbx, NBX = (1, xr) if xr <= 256 else (2, _cdiv(_cdiv(xr, 2), 8) * 8)
    stage = _cdiv((gy_alloc + nbx * NBX) * 144, 1024) * 1024
    ns = 3
    while ns > 2 and max(ns * stage, 256 * 33 * 4) + 1152 > 110 * 1024:
        ns -= 1
    smem = max(ns * stage, 256 * 33 * 4) + 128 + 1024
    return _launch("dw_pad", G * H * njt, 288, smem)


def _dw_tma(B, H, L, K, G):
    """dw_tma.cu: 2048-wide work items, JR x TB register blocks, nj tap groups."""
    jr = 8 if K <= 8 else 16
    nj = 1 if (jr == 8 or K <= 16) else 2
    while nj < 8 and nj * jr < K:
        nj *= 2
    njt = _cdiv(K, nj * jr)
    gy_bytes = _cdiv(64 * 32 * 4, 1024) * 1024
    xt = _cdiv(nj * jr + 40, 32)
    xr = 64 + xt
    if 256 <= L < 2048 and L & (L - 1) == 0:  # multi-row items: 2048 / L rows, each x window with its own tail
        xr = (2048 // L) * (L // 32 + xt)
    stage = _cdiv(gy_bytes + xr * 128, 1024) * 1024
    ns = max(2, min(3 if K > 8 else 4, 72 * 1024 // stage))
    return _launch("dw_tma", G * H * njt, 256, ns * stage + 64 + 1024)


def _stride4(n: int) -> int:
    return _cdiv(n - 4, 32) * 32 + 4


def _stencil_rows(B, H, L, K, off, occ):
    sh = (4 - off % 4) % 4
    box = _stride4(L + K - 1 + sh)
    ks_ = _stride4(_cdiv(K, 8) * 8 + 4)
    segs = _cdiv(L, 16)
    nrc = min(max(32, (256 // segs) // 32 * 32), 256)
    stage = nrc * box
    ns = 3
    smem_of = lambda n: (n * stage + H * ks_) * 4 + 64 + 128  # noqa: E731
    while ns > 2 and smem_of(ns) > 110 * 1024:
        ns -= 1
    smem = smem_of(ns)
    threads = min(256, nrc * segs)
    return _launch("stencil_rows", min(_cdiv(B * H, nrc), SMS * occ(threads, smem)), threads, smem)


def _dw_rows(B, H, L, K, G):
    g8 = _cdiv(K, 8)
    njg = min(8, g8)
    tp = max(1, 8 // njg)
    njt = _cdiv(g8, njg)
    boxg, boxx = _stride4(L + 4), _stride4(L + njg * 8 + 16)
    return _launch("dw_rows", G * H * njt, 32 * njg * tp, 2 * 32 * (boxg + boxx) * 4 + 64 + 128)


def launch_geometry(path: str, B: int, H: int, L: int, K: int, scheme: str = "hierarchical", occ=None) -> list:
    """Every launch of one entry-point call, in order: kernel family, grid,
    block, dynamic shared memory.  ``occ(threads, smem)`` gives resident CTAs
    per SM for the persistent kernels (default: resource_check without the
    register limit; ks_dwconv1d_plan reports the occupancy API's value)."""
    occ = occ or (lambda t, sm: resource_check(t, sm))
    pl = plan(path, B, H, L, K, scheme)
    if path == "bwd":
        if pl["kernel"] == "split":
            return launch_geometry("dx", B, H, L, K, occ=occ) + launch_geometry("dw", B, H, L, K, occ=occ)
        return [_bwd_short("fused", B, H, L, K, pl["row_groups"], occ),
                _launch("dw_sum_groups", _cdiv(H * K, 256), 256, 0)]
    if path in ("fwd", "dx"):
        off = K // 2 if path == "fwd" else K - 1 - K // 2
        kind = pl["kernel"]
        if kind == "stencil_ldg":  # rows shorter than 1024: 256 // ceil(L/8) rows per CTA
            rpc = 256 // _cdiv(L, 8) if L < 1024 else 1
            grid = _cdiv(B * H, rpc) if rpc > 1 else B * H * _cdiv(L, 2048)
            return [_prep_taps(H, 16), _launch("stencil_ldg", grid, 256, 0)]
        if kind == "stencil_short":
            return [_prep_taps(H, 16), _bwd_short(path, B, H, L, K, 1, occ)]
        if kind == "stencil_pad":
            return _stencil_pad(B, H, L, K, off, occ)
        if kind == "stencil_bl":
            return _stencil_bl(B, H, L, K, off)
        if kind == "stencil_rows":
            return [_stencil_rows(B, H, L, K, off, occ)]
        if kind == "stencil_tma":
            return _stencil_tma(B, H, L, K, off, pl["R"], pl["threads"], occ)
        raise NotImplementedError(kind)
    kind, G = pl["kernel"], pl.get("row_groups")
    tail = [_launch("dw_sum_groups", _cdiv(H * K, 256), 256, 0)]
    if kind == "dw_short":
        return [_bwd_short("dw", B, H, L, K, G, occ)] + tail
    if kind == "dw_pad":
        return [_dw_pad(B, H, L, K, G)] + tail
    if kind == "dw_rows":
        return [_dw_rows(B, H, L, K, G)] + tail
    if kind == "dw_tma":
        return [_dw_tma(B, H, L, K, G)] + tail
    raise NotImplementedError(kind)


def shared_mem_footprint(path: str, B: int, H: int, L: int, K: int, scheme: str = "hierarchical") -> int:
    """Dynamic shared memory (bytes per CTA) of the call's main kernel."""
    return max(g["smem"] for g in launch_geometry(path, B, H, L, K, scheme))


def kernel_family(signature: str) -> str:
    """'void ks::(anonymous namespace)::stencil_pad<0, false, false>(...)' (the
    library's demangled names) or 'void <unnamed>::stencil_pad<0, 0, 0>(...)'
    (ncu's) -> 'stencil_pad', the family names launch_geometry uses."""
    s = signature.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    s = s.split("(")[0].replace("void ", "").strip()
    return s.split("<")[0].split("::")[-1]
