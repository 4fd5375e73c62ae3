"""Host-side mirror of the reference operator interface for this path.

Same names, argument meaning and error behaviour as ``kernelscope::conv``
(/root/reference/proj/include/kernelscope/conv_core.hpp:49-69):

* ``forward(x, k, mode)``, ``backward_input(gy, k, mode)``,
  ``backward_weight(gy, x, K, scheme, chunk, mode)`` -- ``x``/``gy`` are
  ``[B,H,L]`` and ``k`` is ``[H,K]``, row-major fp32 or fp64.
* torch CUDA tensors go through the device-pointer C ABI on the current torch
  stream (asynchronous); numpy arrays go through the ``*_host`` entry points
  (host buffers, H2D/D2H inside the call), like the reference's value API.
* shape errors raise ``DimensionError`` naming the axis, as the reference's
  ``check_tensor3`` / ``check_kernel2`` do (tensor.hpp:79-105).

PyTorch is plumbing here (device memory and streams); every op is one of the
library's own sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import CHUNKED, FUSED, HIERARCHICAL, PAIRWISE, SEPARATE, SEQUENTIAL, check

try:  # torch is optional plumbing (device tensors); numpy host buffers work without it
    import torch
except Exception:  # pragma: no cover
    torch = None


class DimensionError(ValueError):
    """Extent mismatch; the message names the axis (reference shape.hpp:10-13)."""


def _is_torch(a) -> bool:
    return torch is not None and isinstance(a, torch.Tensor)


def _dims3(a, name: str, want=None):
    if a.ndim != 3:
        raise DimensionError(f"{name}: expected a [B,H,L] tensor, got {a.ndim} dims")
    B, H, L = (int(v) for v in a.shape)
    if want is not None:
        for axis, got, exp in zip("BHL", (B, H, L), want):
            if got != exp:
                raise DimensionError(f"{name}: axis {axis} is {got}, shape expects {exp}")
    return B, H, L


def _dims_k(k, name: str, H: int):
    if k.ndim != 2:
        raise DimensionError(f"{name}: expected a [H,K] kernel, got {k.ndim} dims")
    if int(k.shape[0]) != H:
        raise DimensionError(f"{name}: axis H is {int(k.shape[0])}, shape expects {H}")
    return int(k.shape[1])


def _ptr(a) -> int:
    if _is_torch(a):
        if not a.is_cuda:
            raise ValueError("torch tensors must live on a CUDA device (no CPU fallback)")
        if not a.is_contiguous():
            raise ValueError("tensors must be contiguous row-major")
        return a.data_ptr()
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("arrays must be C-contiguous")
    return a.ctypes.data


def _stream(a):
    return C.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)


def _suffix(a) -> str:
    dt = a.dtype
    if dt in (np.float32,) or (torch is not None and dt == torch.float32):
        return "f32"
    if dt in (np.float64,) or (torch is not None and dt == torch.float64):
        return "f64"
    raise TypeError(f"unsupported dtype {dt}; fp32 or fp64")


def _empty_like(a, shape):
    if _is_torch(a):
        return torch.empty(shape, dtype=a.dtype, device=a.device)
    return np.empty(shape, dtype=a.dtype)


def _raise_dims(status: int, what: str):
    if status in (1, 2, 3, 4, 5):
        raise DimensionError(f"{what}: {_lib.STATUS_NAMES[status]}")
    check(status, what)


def _stencil(kind: str, inp, k, mode: int, out=None):
    B, H, L = _dims3(inp, f"{kind}: input")
    K = _dims_k(k, f"{kind}: k", H)
    suf = _suffix(inp)
    if _suffix(k) != suf:
        raise TypeError("input and kernel dtypes differ")
    if out is None:
        out = _empty_like(inp, (B, H, L))
    l = _lib.lib()
    if _is_torch(inp):
        fn = getattr(l, f"ks_dwconv1d_{kind}_{suf}")
        st = fn(_ptr(inp), _ptr(k), _ptr(out), B, H, L, K, mode, _stream(inp))
    else:
        fn = getattr(l, f"ks_dwconv1d_{kind}_{suf}_host")
        st = fn(_ptr(inp), _ptr(k), _ptr(out), B, H, L, K, mode)
    _raise_dims(st, {"fwd": "forward", "dx": "backward_input"}[kind])
    return out


def forward(x, k, mode: int = SEPARATE, out=None):
    """y = conv::forward(x, k, shape, mode) (reference src/conv_core.cpp:21-46)."""
    return _stencil("fwd", x, k, mode, out)


def backward_input(gy, k, mode: int = SEPARATE, out=None):
    """dx = conv::backward_input(gy, k, shape, mode) (src/conv_core.cpp:48-75)."""
    return _stencil("dx", gy, k, mode, out)


def workspace_bytes(B: int, H: int, L: int, K: int, scheme: int = HIERARCHICAL,
                    chunk: int = 1024, elem_bytes: int = 4) -> int:
    out = C.c_size_t(0)
    st = _lib.lib().ks_dwconv1d_dw_workspace_bytes(B, H, L, K, scheme, chunk, elem_bytes,
                                                   C.byref(out))
    _raise_dims(st, "dw_workspace_bytes")
    return int(out.value)


def backward_weight(gy, x, K: int, scheme: int = SEQUENTIAL, chunk: int = 1024,
                    mode: int = SEPARATE, out=None, workspace=None):
    """dk = conv::backward_weight(gy, x, shape, scheme, mode) (src/conv_core.cpp:148-181).

    ``scheme``: SEQUENTIAL / PAIRWISE / CHUNKED reproduce the reference's
    association order bitwise; HIERARCHICAL is the fast deterministic path.
    """
    B, H, L = _dims3(gy, "backward_weight: gy")
    _dims3(x, "backward_weight: x", (B, H, L))
    if scheme == CHUNKED and chunk < 1:
        raise DimensionError(f"backward_weight: chunk_size must be >= 1, got {chunk}")
    suf = _suffix(gy)
    if _suffix(x) != suf:
        raise TypeError("gy and x dtypes differ")
    if out is None:
        out = _empty_like(gy, (H, K))
    l = _lib.lib()
    if _is_torch(gy):
        ws_ptr, ws_bytes = None, 0
        if workspace is not None:
            ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
        fn = getattr(l, f"ks_dwconv1d_dw_{suf}")
        st = fn(_ptr(gy), _ptr(x), _ptr(out), B, H, L, K, scheme, chunk, mode, ws_ptr, ws_bytes,
                _stream(gy))
    else:
        fn = getattr(l, f"ks_dwconv1d_dw_{suf}_host")
        st = fn(_ptr(gy), _ptr(x), _ptr(out), B, H, L, K, scheme, chunk, mode)
    _raise_dims(st, "backward_weight")
    return out


def backward(gy, x, k, mode: int = SEPARATE, out=None, workspace=None):
    """(dx, dk) = (conv::backward_input(gy, k), conv::backward_weight(gy, x,
    HIERARCHICAL)) in one call (ks_dwconv1d_bwd_f32): the layer's backward,
    fused so gy and x cross HBM once where the fused kernel applies.  Device
    (torch CUDA) fp32 tensors; bits equal the two separate calls."""
    B, H, L = _dims3(gy, "backward: gy")
    _dims3(x, "backward: x", (B, H, L))
    K = _dims_k(k, "backward: k", H)
    if not _is_torch(gy) or _suffix(gy) != "f32" or _suffix(x) != "f32" or _suffix(k) != "f32":
        raise TypeError("backward: fp32 CUDA tensors")
    if out is None:
        out = (_empty_like(gy, (B, H, L)), _empty_like(gy, (H, K)))
    dx, dk = out
    ws_ptr, ws_bytes = None, 0
    if workspace is not None:
        ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    st = _lib.lib().ks_dwconv1d_bwd_f32(_ptr(gy), _ptr(x), _ptr(k), _ptr(dx), _ptr(dk), B, H, L, K, mode,
                                        ws_ptr, ws_bytes, _stream(gy))
    _raise_dims(st, "backward")
    return dx, dk


def step_host(x, k, gy, K: int | None = None, scheme: int = HIERARCHICAL, chunk: int = 0,
              mode: int = FUSED, out=None):
    """One fwd + dX + dW step on host (numpy) buffers through
    ks_dwconv1d_step_f32_host; returns (y, dx, dk)."""
    B, H, L = _dims3(x, "step: x")
    _dims3(gy, "step: gy", (B, H, L))
    K = _dims_k(k, "step: k", H)
    if out is None:
        out = (np.empty_like(x), np.empty_like(gy), np.empty((H, K), np.float32))
    y, dx, dk = out
    st = _lib.lib().ks_dwconv1d_step_f32_host(_ptr(x), _ptr(k), _ptr(gy), _ptr(y), _ptr(dx), _ptr(dk),
                                              B, H, L, K, scheme, chunk, mode)
    _raise_dims(st, "step")
    return y, dx, dk


VARIANTS = {"naive": 0, "coalesced": 1, "shared": 2, "warp": 3}
PATHS = {"fwd": 0, "dx": 1, "dw": 2}


def variant(name: str, path: str, a, b, K: int | None = None, mode: int = FUSED, out=None):
    """Run one of the paper's four kernel designs on device
    tensors: path 'fwd' (a=x, b=k), 'dx' (a=gy, b=k) or 'dw' (a=gy, b=x, K)."""
    v, p = VARIANTS[name], PATHS[path]
    B, H, L = _dims3(a, f"{name} {path}: a")
    if p == 2:
        _dims3(b, f"{name} dw: x", (B, H, L))
        if K is None:
            raise ValueError("dw needs K")
        shape_out = (H, K)
    else:
        K = _dims_k(b, f"{name} {path}: k", H)
        shape_out = (B, H, L)
    if out is None:
        out = _empty_like(a, shape_out)
    st = _lib.lib().ks_dwconv1d_variant_f32(v, p, _ptr(a), _ptr(b), _ptr(out), B, H, L, K, mode, None, 0,
                                           _stream(a))
    _raise_dims(st, f"variant {name} {path}")
    return out


def fill_pm1(seed: int, first: int, out) -> None:
    """Device splitmix64 fill, bit-identical to the reference SplitMix64 stream
    (include/kernelscope/rng.hpp:12-28): out.flat[i] = draw first+1+i."""
    st = _lib.lib().ks_fill_pm1_f32(seed, first, _ptr(out), out.numel(), _stream(out))
    check(st, "fill_pm1")


def make_inputs(seed: int, B: int, H: int, L: int, K: int, device="cuda", b0: int = 0,
                B_total: int | None = None):
    """validate()'s inputs on the device: x, then k, then gy from one stream
    (src/conv_core.cpp:241-247).  With (b0, B_total) it generates batch rows
    [b0, b0+B) of the B_total-row problem in place (O(1) skip-ahead)."""
    Bt = B if B_total is None else B_total
    n = Bt * H * L
    x = torch.empty((B, H, L), dtype=torch.float32, device=device)
    k = torch.empty((H, K), dtype=torch.float32, device=device)
    gy = torch.empty((B, H, L), dtype=torch.float32, device=device)
    fill_pm1(seed, b0 * H * L, x)
    fill_pm1(seed, n, k)
    fill_pm1(seed, n + H * K + b0 * H * L, gy)
    return x, k, gy


# ---- batch sharding / dW combine -------------------------------------------

def shard_rows(B: int, world: int, rank: int):
    b0, nb = C.c_int64(0), C.c_int64(0)
    st = _lib.lib().ks_shard_rows(B, world, rank, C.byref(b0), C.byref(nb))
    check(st, "shard_rows")
    return int(b0.value), int(nb.value)


class Comm:
    """NCCL communicator owned by the C library (one process per GPU).  The
    128-byte unique id is created on rank 0 and broadcast by the caller (e.g.
    over torch.distributed)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_char * 128)()
        check(_lib.lib().ks_comm_unique_id(C.addressof(buf)), "comm_unique_id")
        return bytes(buf)

    def __init__(self, uid: bytes, world: int, rank: int):
        buf = (C.c_char * 128).from_buffer_copy(uid)
        self.handle = C.c_void_p()
        check(_lib.lib().ks_comm_init(C.byref(self.handle), C.addressof(buf), world, rank),
              "comm_init")
        self.world, self.rank = world, rank

    def allreduce_dw(self, dk) -> None:
        H, K = (int(v) for v in dk.shape)
        check(_lib.lib().ks_dwconv1d_dw_allreduce_f32(_ptr(dk), H, K, self.handle, _stream(dk)),
              "dw_allreduce")

    def allgather_sum_dw(self, dk, gather) -> None:
        H, K = (int(v) for v in dk.shape)
        check(_lib.lib().ks_dwconv1d_dw_allgather_sum_f32(_ptr(dk), _ptr(gather), H, K,
                                                          self.handle, _stream(dk)),
              "dw_allgather_sum")

    def peer(self, B: int, H: int, L: int, K: int) -> "Peer":
        """NVLink peer-memory dW combine for per-rank shape (B,H,L,K)."""
        return Peer(self, workspace_bytes(B, H, L, K, HIERARCHICAL))

    def close(self) -> None:
        if self.handle:
            _lib.lib().ks_comm_destroy(self.handle)
            self.handle = C.c_void_p()


class Peer:
    """ks_peer: dW whose cross-rank sum is fused into the reduction kernel and
    read straight from the peers' memory (no NCCL on the data path)."""

    def __init__(self, comm: Comm, partial_bytes: int):
        self.handle = C.c_void_p()
        check(_lib.lib().ks_peer_create(comm.handle, max(partial_bytes, 4), C.byref(self.handle)),
              "peer_create")

    def backward_weight(self, gy, x, K: int, mode: int = FUSED, out=None):
        B, H, L = _dims3(gy, "peer dw: gy")
        _dims3(x, "peer dw: x", (B, H, L))
        if out is None:
            out = _empty_like(gy, (H, K))
        st = _lib.lib().ks_dwconv1d_dw_f32_peer(_ptr(gy), _ptr(x), _ptr(out), B, H, L, K, mode,
                                               self.handle, _stream(gy))
        _raise_dims(st, "dw_peer")
        return out

    def timed_out(self) -> bool:
        f = C.c_int(0)
        check(_lib.lib().ks_peer_timed_out(self.handle, C.byref(f)), "peer_timed_out")
        return bool(f.value)

    def close(self) -> None:
        if self.handle:
            _lib.lib().ks_peer_destroy(self.handle)
            self.handle = C.c_void_p()
