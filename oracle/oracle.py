"""oracle.py -- numpy/ctypes front end of the CPU parity checkers.

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs import this module; the
product package (``paper_2604_25422_b200``) never does.

Two back ends with the same numpy interface:

* ``Oracle`` -- ``liboracle.so``, the plain-C restatement in ``ks_oracle.c``
  (each routine cites /root/reference/proj/src/conv_core.cpp lines).
* ``Reference`` -- ``_ref/libksref.so``, the reference's own conv_core.cpp
  compiled from /root/reference by ``oracle/Makefile`` (absent on a box that
  never had the reference and no prebuilt copy).

Enum values follow the reference: MulAddMode Separate=0 / Fused=1
(include/kernelscope/conv_core.hpp:45), SumScheme Sequential=0 /
PairwiseTree=1 / ChunkedTwoStage=2 (conv_core.hpp:14-18).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SEPARATE, FUSED = 0, 1
SEQUENTIAL, PAIRWISE, CHUNKED = 0, 1, 2

_i64 = C.c_int64
_u64 = C.c_uint64
_p = C.c_void_p


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _check_shape(a, B, H, L):
    if a.shape != (B, H, L):
        raise ValueError(f"expected [B,H,L]=({B},{H},{L}), got {a.shape}")


class _Backend:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        self.path = path

    def _fn(self, name, argtypes, restype=C.c_int):
        f = getattr(self.lib, self.prefix + name)
        f.argtypes = argtypes
        f.restype = restype
        return f

    # --- paths ---------------------------------------------------------------
    def forward(self, x: np.ndarray, k: np.ndarray, mode: int = SEPARATE, threads: int = 0):
        B, H, L = x.shape
        K = k.shape[1]
        dt = x.dtype
        y = np.empty_like(x)
        if threads and dt == np.float32:
            f = self._fn("forward_f32_mt", [_p, _p, _p, _i64, _i64, _i64, _i64, C.c_int, C.c_int])
            f(_ptr(x), _ptr(k), _ptr(y), B, H, L, K, mode, threads)
        else:
            suf = "f32" if dt == np.float32 else "f64"
            f = self._fn("forward_" + suf, [_p, _p, _p, _i64, _i64, _i64, _i64, C.c_int])
            f(_ptr(x), _ptr(k), _ptr(y), B, H, L, K, mode)
        return y

    def backward_input(self, gy: np.ndarray, k: np.ndarray, mode: int = SEPARATE, threads: int = 0):
        B, H, L = gy.shape
        K = k.shape[1]
        dx = np.empty_like(gy)
        if threads and gy.dtype == np.float32:
            f = self._fn("backward_input_f32_mt",
                         [_p, _p, _p, _i64, _i64, _i64, _i64, C.c_int, C.c_int])
            f(_ptr(gy), _ptr(k), _ptr(dx), B, H, L, K, mode, threads)
        else:
            suf = "f32" if gy.dtype == np.float32 else "f64"
            f = self._fn("backward_input_" + suf, [_p, _p, _p, _i64, _i64, _i64, _i64, C.c_int])
            f(_ptr(gy), _ptr(k), _ptr(dx), B, H, L, K, mode)
        return dx

    def backward_weight(self, gy: np.ndarray, x: np.ndarray, K: int, scheme: int = SEQUENTIAL,
                        chunk: int = 1024, mode: int = SEPARATE, threads: int = 0):
        B, H, L = gy.shape
        _check_shape(x, B, H, L)
        dk = np.empty((H, K), dtype=gy.dtype)
        if threads and (gy.dtype == np.float32 or self.prefix == "kso_"):
            suf = "f32" if gy.dtype == np.float32 else "f64"
            f = self._fn(f"backward_weight_{suf}_mt",
                         [_p, _p, _p, _i64, _i64, _i64, _i64, C.c_int, _i64, C.c_int, C.c_int])
            rc = f(_ptr(gy), _ptr(x), _ptr(dk), B, H, L, K, scheme, chunk, mode, threads)
        else:
            suf = "f32" if gy.dtype == np.float32 else "f64"
            f = self._fn("backward_weight_" + suf,
                         [_p, _p, _p, _i64, _i64, _i64, _i64, C.c_int, _i64, C.c_int])
            rc = f(_ptr(gy), _ptr(x), _ptr(dk), B, H, L, K, scheme, chunk, mode)
        if rc != 0:
            raise ValueError(f"backward_weight: chunk_size must be >= 1, got {chunk}")
        return dk


class Oracle(_Backend):
    """The C restatement (oracle/ks_oracle.c)."""
    prefix = "kso_"

    def __init__(self, path: str = os.path.join(HERE, "liboracle.so")):
        super().__init__(path)

    def fill_pm1(self, seed: int, first: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float32)
        f = self._fn("fill_pm1", [_u64, _u64, _p, _i64], None)
        f(seed, first, _ptr(out), n)
        return out

    def splitmix64_at(self, seed: int, n: int) -> int:
        f = self._fn("splitmix64_at", [_u64, _u64], _u64)
        return int(f(seed, n))

    def fill_inputs(self, seed: int, B: int, H: int, L: int, K: int):
        """validate()'s stream: x, then k, then gy (src/conv_core.cpp:241-247)."""
        n, m = B * H * L, H * K
        x = self.fill_pm1(seed, 0, n).reshape(B, H, L)
        k = self.fill_pm1(seed, n, m).reshape(H, K)
        gy = self.fill_pm1(seed, n + m, n).reshape(B, H, L)
        return x, k, gy

    def backward_weight_int(self, gy: np.ndarray, x: np.ndarray, K: int) -> np.ndarray:
        B, H, L = gy.shape
        dk = np.empty((H, K), dtype=np.int64)
        f = self._fn("backward_weight_i64", [_p, _p, _p, _i64, _i64, _i64, _i64], None)
        f(_ptr(gy), _ptr(x), _ptr(dk), B, H, L, K)
        return dk


class Reference(_Backend):
    """The reference's own conv_core.cpp (oracle/_ref/libksref.so)."""
    prefix = "ksref_"

    def __init__(self, path: str = os.path.join(HERE, "_ref", "libksref.so")):
        super().__init__(path)

    def fill_inputs(self, seed: int, B: int, H: int, L: int, K: int):
        x = np.empty((B, H, L), np.float32)
        gy = np.empty((B, H, L), np.float32)
        k = np.empty((H, K), np.float32)
        f = self._fn("fill_inputs", [_u64, _p, _p, _p, _i64, _i64, _i64, _i64], None)
        f(seed, _ptr(x), _ptr(k), _ptr(gy), B, H, L, K)
        return x, k, gy

    def validate(self, B, H, L, K, seed, schemes):
        """conv::validate; schemes = [(scheme, chunk), ...]."""
        n = len(schemes)
        sc = (C.c_int * n)(*[s for s, _ in schemes])
        ch = (_i64 * n)(*[c for _, c in schemes])
        out = (C.c_double * (6 + 2 * n))()
        f = self._fn("validate", [_i64, _i64, _i64, _i64, _u64, _p, _p, C.c_int, _p])
        rc = f(B, H, L, K, seed, C.addressof(sc), C.addressof(ch), n, C.addressof(out))
        if rc != 0:
            raise ValueError("validate: at least one accumulation scheme required")
        v = list(out)
        return {"fwd": (v[0], v[1]), "bwd_in": (v[2], v[3]),
                "dk": [(v[4 + 2 * i], v[5 + 2 * i]) for i in range(n)],
                "dk_spread_abs": v[4 + 2 * n], "dk_spread_rel": v[5 + 2 * n]}


def reference_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libksref.so"))


def normwise(got: np.ndarray, ref: np.ndarray) -> float:
    """max|got-ref| / max|ref| -- the reference's dk_spread_rel form
    (src/conv_core.cpp:278); per-element relative error is meaningless on
    near-zero outputs."""
    ref64 = ref.astype(np.float64)
    peak = float(np.max(np.abs(ref64))) if ref64.size else 0.0
    diff = float(np.max(np.abs(got.astype(np.float64) - ref64))) if ref64.size else 0.0
    return diff / max(peak, 1e-12)
