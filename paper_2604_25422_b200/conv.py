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

import contextlib
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


def _same_kind(a, like, name: str) -> None:
    """`a` must be the same kind of buffer as `like` (torch CUDA tensor on the
    same device, or a host numpy array) with the same dtype: the C ABI takes
    raw pointers, so a host pointer among device pointers (or the reverse)
    would be an illegal address, not an exception."""
    if _is_torch(like):
        if not _is_torch(a):
            raise TypeError(f"{name}: expected a torch CUDA tensor like the input, got {type(a).__name__}")
        if a.device != like.device:
            raise ValueError(f"{name}: on {a.device}, the input is on {like.device}")
    elif _is_torch(a) or not isinstance(a, np.ndarray):
        raise TypeError(f"{name}: expected a numpy array like the input, got {type(a).__name__}")
    if a.dtype != like.dtype:
        raise TypeError(f"{name}: dtype {a.dtype}, the input is {like.dtype}")


def _check_out(out, like, shape, name: str):
    """A caller-supplied output: right kind, device, dtype, shape, contiguous."""
    if out is None:
        return _empty_like(like, shape)
    _same_kind(out, like, name)
    if tuple(int(v) for v in out.shape) != tuple(shape):
        raise DimensionError(f"{name}: shape {tuple(out.shape)}, expected {tuple(shape)}")
    return out


def _check_ws(ws, like):
    """(pointer, bytes) of an optional device workspace."""
    if ws is None:
        return None, 0
    if not (_is_torch(ws) and _is_torch(like)) or ws.device != like.device:
        raise TypeError("workspace: a torch CUDA tensor on the input's device")
    if not ws.is_contiguous():
        raise ValueError("workspace must be contiguous")
    return ws.data_ptr(), ws.numel() * ws.element_size()


def _on_device(a):
    """Launch on the tensor's device, not whatever device is current."""
    return torch.cuda.device(a.device) if _is_torch(a) else contextlib.nullcontext()


def _raise_dims(status: int, what: str):
    if status in (1, 2, 3, 4, 5):
        raise DimensionError(f"{what}: {_lib.STATUS_NAMES[status]}")
    check(status, what)


def _stencil(kind: str, inp, k, mode: int, out=None):
    B, H, L = _dims3(inp, f"{kind}: input")
    K = _dims_k(k, f"{kind}: k", H)
    suf = _suffix(inp)
    _same_kind(k, inp, f"{kind}: k")
    out = _check_out(out, inp, (B, H, L), f"{kind}: out")
    l = _lib.lib()
    if _is_torch(inp):
        fn = getattr(l, f"ks_dwconv1d_{kind}_{suf}")
        with _on_device(inp):
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
    _same_kind(x, gy, "backward_weight: x")
    out = _check_out(out, gy, (H, K), "backward_weight: out")
    l = _lib.lib()
    if _is_torch(gy):
        ws_ptr, ws_bytes = _check_ws(workspace, gy)
        fn = getattr(l, f"ks_dwconv1d_dw_{suf}")
        with _on_device(gy):
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
    if not _is_torch(gy) or _suffix(gy) != "f32":
        raise TypeError("backward: fp32 CUDA tensors")
    _same_kind(x, gy, "backward: x")
    _same_kind(k, gy, "backward: k")
    dx, dk = out if out is not None else (None, None)
    dx = _check_out(dx, gy, (B, H, L), "backward: dx")
    dk = _check_out(dk, gy, (H, K), "backward: dk")
    ws_ptr, ws_bytes = _check_ws(workspace, gy)
    with _on_device(gy):
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
    if _is_torch(x) or _suffix(x) != "f32":
        raise TypeError("step_host: fp32 numpy (host) arrays")
    _same_kind(k, x, "step: k")
    _same_kind(gy, x, "step: gy")
    y, dx, dk = out if out is not None else (None, None, None)
    y = _check_out(y, x, (B, H, L), "step: y")
    dx = _check_out(dx, x, (B, H, L), "step: dx")
    dk = _check_out(dk, x, (H, K), "step: dk")
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
    if not _is_torch(a):
        raise TypeError("variant: torch CUDA tensors")
    _same_kind(b, a, f"{name} {path}: b")
    out = _check_out(out, a, shape_out, f"{name} {path}: out")
    with _on_device(a):
        st = _lib.lib().ks_dwconv1d_variant_f32(v, p, _ptr(a), _ptr(b), _ptr(out), B, H, L, K, mode, None, 0,
                                               _stream(a))
    _raise_dims(st, f"variant {name} {path}")
    return out


def fill_pm1(seed: int, first: int, out) -> None:
    """Device splitmix64 fill, bit-identical to the reference SplitMix64 stream
    (include/kernelscope/rng.hpp:12-28): out.flat[i] = draw first+1+i."""
    if not _is_torch(out) or out.dtype != torch.float32:
        raise TypeError("fill_pm1: an fp32 torch CUDA tensor")
    with _on_device(out):
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
    """A communicator owned by the C library (one process per rank).

    ``Comm(uid, world, rank)`` is an NCCL communicator (one GPU per rank; the
    128-byte unique id is created on rank 0 and broadcast by the caller, e.g.
    over torch.distributed).  ``Comm.host(world, rank, allgather)`` uses the
    caller's host all-gather instead -- ``allgather(data: bytes) -> list[bytes]``
    in rank order, e.g. over a gloo process group -- which only moves bytes
    (every sum stays on the device), so ranks may share one GPU."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_char * 128)()
        check(_lib.lib().ks_comm_unique_id(C.addressof(buf)), "comm_unique_id")
        return bytes(buf)

    def __init__(self, uid: bytes | None, world: int, rank: int, _host=None):
        self.handle = C.c_void_p()
        self.world, self.rank = world, rank
        self._cb = None
        if _host is not None:
            def _allgather(send, recv, nbytes, _ctx):
                try:
                    parts = _host(C.string_at(send, nbytes))
                    if len(parts) != world or any(len(p) != nbytes for p in parts):
                        return 1
                    C.memmove(recv, b"".join(parts), nbytes * world)
                    return 0
                except Exception:  # a Python exception must not unwind through C
                    return 1
            self._cb = _lib.ALLGATHER_FN(_allgather)  # kept alive with the communicator
            check(_lib.lib().ks_comm_init_host(C.byref(self.handle), world, rank, self._cb, None),
                  "comm_init_host")
            return
        buf = (C.c_char * 128).from_buffer_copy(uid)
        check(_lib.lib().ks_comm_init(C.byref(self.handle), C.addressof(buf), world, rank),
              "comm_init")

    @classmethod
    def host(cls, world: int, rank: int, allgather) -> "Comm":
        return cls(None, world, rank, _host=allgather)

    def allgather_bytes(self, data: bytes) -> list:
        """ks_comm_allgather_host: every rank's `data` (same length), rank order."""
        n = len(data)
        recv = (C.c_char * (n * self.world))()
        check(_lib.lib().ks_comm_allgather_host(self.handle, data, C.addressof(recv), n), "comm_allgather_host")
        raw = bytes(recv)
        return [raw[r * n:(r + 1) * n] for r in range(self.world)]

    def allreduce_dw(self, dk) -> None:
        H, K = (int(v) for v in dk.shape)
        with _on_device(dk):
            check(_lib.lib().ks_dwconv1d_dw_allreduce_f32(_ptr(dk), H, K, self.handle, _stream(dk)),
                  "dw_allreduce")

    def allgather_sum_dw(self, dk, gather) -> None:
        H, K = (int(v) for v in dk.shape)
        _same_kind(gather, dk, "allgather_sum_dw: gather")
        if gather.numel() < self.world * H * K:
            raise DimensionError(f"allgather_sum_dw: gather needs {self.world * H * K} floats")
        with _on_device(dk):
            check(_lib.lib().ks_dwconv1d_dw_allgather_sum_f32(_ptr(dk), _ptr(gather), H, K,
                                                              self.handle, _stream(dk)),
                  "dw_allgather_sum")

    def chunked_dw(self, gy, x, K: int, chunk: int, mode: int, b0: int, B_total: int, out=None):
        """ks_dwconv1d_dw_chunked_sharded_f32: this rank holds global rows
        [b0, b0 + B_local) of B_total; dk (every rank) is bitwise the
        single-device CHUNKED(chunk) dW of the whole batch."""
        B, H, L = (int(v) for v in gy.shape)
        if tuple(x.shape) != (B, H, L):
            raise DimensionError(f"chunked_dw: x shape {tuple(x.shape)} != gy shape {(B, H, L)}")
        if chunk < 1:
            raise DimensionError(f"chunked_dw: chunk_size must be >= 1, got {chunk}")
        out = _check_out(out, gy, (H, K), "chunked_dw: out")
        with _on_device(gy):
            check(_lib.lib().ks_dwconv1d_dw_chunked_sharded_f32(_ptr(gy), _ptr(x), _ptr(out), B, b0, B_total, H, L,
                                                                K, chunk, mode, self.handle, _stream(gy)),
                  "dw_chunked_sharded")
        return out

    def peer(self, B: int, H: int, L: int, K: int, B_total: int = 0) -> "Peer":
        """Peer-memory dW combine for per-rank shape (B,H,L,K); with B_total the
        global plan (bitwise = the 1-GPU result when the shards align)."""
        need = workspace_bytes(B, H, L, K, HIERARCHICAL)
        if B_total:
            need = max(need, workspace_bytes(B_total, H, L, K, HIERARCHICAL))
        return Peer(self, need)

    def close(self) -> None:
        if self.handle:
            _lib.lib().ks_comm_destroy(self.handle)
            self.handle = C.c_void_p()


class Peer:
    """ks_peer: dW whose cross-rank sum is fused into the reduction kernel and
    read straight from the peers' memory (no collective on the data path)."""

    def __init__(self, comm: Comm, partial_bytes: int):
        self.handle = C.c_void_p()
        self.comm = comm
        check(_lib.lib().ks_peer_create(comm.handle, max(partial_bytes, 4), C.byref(self.handle)),
              "peer_create")

    def backward_weight(self, gy, x, K: int, mode: int = FUSED, out=None, B_total: int = 0):
        B, H, L = _dims3(gy, "peer dw: gy")
        _dims3(x, "peer dw: x", (B, H, L))
        if not _is_torch(gy) or _suffix(gy) != "f32":
            raise TypeError("peer dw: fp32 torch CUDA tensors")
        _same_kind(x, gy, "peer dw: x")
        out = _check_out(out, gy, (H, K), "peer dw: out")
        with _on_device(gy):
            st = _lib.lib().ks_dwconv1d_dw_f32_peer(_ptr(gy), _ptr(x), _ptr(out), B, H, L, K, B_total, mode,
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


def rank_tree_sum(gather, out) -> None:
    """out[i] = midpoint-split pairwise tree over gather[r, i], r in rank order
    (ks_rank_tree_sum_f32): the fixed cross-rank combine."""
    if not _is_torch(gather) or _suffix(gather) != "f32" or gather.ndim != 2:
        raise TypeError("rank_tree_sum: a [world, n] fp32 torch CUDA tensor")
    world, n = (int(v) for v in gather.shape)
    _same_kind(out, gather, "rank_tree_sum: out")
    if out.numel() != n:
        raise DimensionError(f"rank_tree_sum: out has {out.numel()} floats, expected {n}")
    with _on_device(gather):
        check(_lib.lib().ks_rank_tree_sum_f32(_ptr(gather), _ptr(out), n, world, _stream(gather)),
              "rank_tree_sum")


# ---- library-wide -----------------------------------------------------------

def set_option(name: str, value: int | None = None) -> None:
    """ks_set_option: a tuning option (tier switch / pipeline depth); None
    restores the default."""
    v = _lib.KS_OPTION_DEFAULT if value is None else int(value)
    check(_lib.lib().ks_set_option(name.encode(), v), f"set_option {name}")


def get_option(name: str) -> int:
    v = C.c_int64(0)
    check(_lib.lib().ks_get_option(name.encode(), C.byref(v)), f"get_option {name}")
    return int(v.value)


@contextlib.contextmanager
def options(**kw):
    """Temporarily set tuning options (restored to their previous values)."""
    old = {k: get_option(k) for k in kw}
    try:
        for k, v in kw.items():
            set_option(k, v)
        yield
    finally:
        for k, v in old.items():
            set_option(k, v)


def launch_count() -> int:
    """Kernels this library has launched in this process (ks_launch_count)."""
    v = C.c_uint64(0)
    check(_lib.lib().ks_launch_count(C.byref(v)), "launch_count")
    return int(v.value)


PLAN_PATHS = {"fwd": 0, "dx": 1, "dw": 2, "bwd": 3}


def plan(path: str, B: int, H: int, L: int, K: int, scheme: int = HIERARCHICAL, chunk: int = 0,
         mode: int = SEPARATE) -> list:
    """ks_dwconv1d_plan: the kernels one call would launch for this shape
    (kernel, grid, block, dynamic smem) -- the real dispatch run without
    launching; this library's launch_geometry / shared_mem_footprint
    (reference proj/include/kernelscope/exec_model.hpp:14-127).  Needs a device."""
    cap = 64
    recs = (_lib.LaunchRec * cap)()
    n = C.c_int(0)
    st = _lib.lib().ks_dwconv1d_plan(PLAN_PATHS[path], B, H, L, K, scheme, chunk, mode, C.addressof(recs), cap,
                                     C.byref(n))
    _raise_dims(st, f"plan {path}")
    return [{"kernel": r.kernel.decode(), "grid": tuple(r.grid), "block": tuple(r.block),
             "smem": int(r.smem_bytes), "regs": int(r.regs), "static_smem": int(r.static_smem),
             "ctas_per_sm": int(r.ctas_per_sm)}
            for r in recs[:min(n.value, cap)]]
