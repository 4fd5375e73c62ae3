"""CPU: the C-ABI library loads, exports every symbol include/ks_dwconv1d.h
declares, validates arguments in the reference's order, and fails loudly
(never computes on the CPU) when there is no device."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "ks_dwconv1d.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ks_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2604_25422_b200 import _lib
    lib = _lib.lib()
    declared = header_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.EXPORTED)
    assert lib.ks_abi_version() == 2
    assert lib.ks_status_string(0) == b"ok"


def test_library_is_sm100a_and_links_nccl():
    import subprocess
    so = os.path.join(ROOT, "paper_2604_25422_b200", "libks_dwconv1d.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    deps = subprocess.run(["ldd", so], capture_output=True, text=True).stdout
    assert "libnccl" in deps


def test_argument_validation_order():
    from paper_2604_25422_b200 import _lib
    lib = _lib.lib()
    p = C.c_void_p(16)
    # shape first (ConvShape ctor order B,H,L,K; shape.hpp:27-31)
    assert lib.ks_dwconv1d_fwd_f32(p, p, p, 0, 1, 1, 1, 0, None) == 1
    assert lib.ks_dwconv1d_fwd_f32(p, p, p, 1, 0, 1, 1, 0, None) == 2
    assert lib.ks_dwconv1d_dx_f32(p, p, p, 1, 1, -3, 1, 0, None) == 3
    assert lib.ks_dwconv1d_dx_f64(p, p, p, 1, 1, 1, 0, 0, None) == 4
    assert lib.ks_dwconv1d_fwd_f32(p, p, p, 1, 1, 1, 1, 7, None) == 6     # mode
    assert lib.ks_dwconv1d_fwd_f32(None, p, p, 1, 1, 1, 1, 0, None) == 8  # null
    # chunk < 1 (src/conv_core.cpp:154-156), unknown scheme
    assert lib.ks_dwconv1d_dw_f32(p, p, p, 1, 1, 4, 3, 2, 0, 0, None, 0, None) == 5
    assert lib.ks_dwconv1d_dw_f32(p, p, p, 1, 1, 4, 3, 9, 1, 0, None, 0, None) == 7
    sz = C.c_size_t(0)
    assert lib.ks_dwconv1d_dw_workspace_bytes(4, 2, 100, 7, 3, 0, 4, C.byref(sz)) == 0
    assert sz.value > 0
    assert lib.ks_dwconv1d_dw_workspace_bytes(4, 2, 100, 7, 1, 0, 4, C.byref(sz)) == 0
    assert sz.value == 0  # pairwise needs no scratch
    assert lib.ks_dwconv1d_dw_workspace_bytes(4, 2, 100, 7, 2, 50, 4, C.byref(sz)) == 0
    assert sz.value == 8 * 2 * 7 * 4  # 400/50 chunks x H x K floats


def test_python_mirror_dimension_errors():
    import paper_2604_25422_b200 as ks
    x = np.zeros((2, 2, 5), np.float32)
    with pytest.raises(ks.DimensionError, match="axis H"):
        ks.forward(x, np.zeros((3, 4), np.float32))
    with pytest.raises(ks.DimensionError, match="axis L"):
        ks.backward_weight(x, np.zeros((2, 2, 6), np.float32), 3)
    with pytest.raises(ks.DimensionError, match="chunk_size"):
        ks.backward_weight(x, x, 3, ks.CHUNKED, 0)


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-device path")
def test_no_cpu_fallback_without_device():
    import paper_2604_25422_b200 as ks
    x = np.ones((1, 1, 8), np.float32)
    k = np.ones((1, 3), np.float32)
    with pytest.raises(ks.KsError, match="NO_DEVICE"):
        ks.forward(x, k)
    with pytest.raises(ks.KsError, match="NO_DEVICE"):
        ks.backward_weight(x, x, 3, ks.HIERARCHICAL)


def test_shard_rows_cover_batch():
    import paper_2604_25422_b200 as ks
    for B in (1, 7, 64, 1024):
        for world in (1, 2, 3, 4, 8):
            if world > B:
                continue
            spans = [ks.shard_rows(B, world, r) for r in range(world)]
            assert spans[0][0] == 0
            assert sum(n for _, n in spans) == B
            for (a, n), (b, _) in zip(spans, spans[1:]):
                assert a + n == b
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1
    with pytest.raises(ks.KsError):
        ks.shard_rows(4, 8, 0)


def test_tuning_options_are_explicit_and_validated():
    """Tier switches are an explicit, validated API (ks_set_option): no
    environment variable changes what the library runs."""
    import paper_2604_25422_b200 as ks
    assert ks.get_option("ldg") == 1 and ks.get_option("bwds") == 1 and ks.get_option("disable_tma") == 0
    with ks.options(ldg=2, bwds=0):
        assert ks.get_option("ldg") == 2 and ks.get_option("bwds") == 0
    assert ks.get_option("ldg") == 1 and ks.get_option("bwds") == 1
    with pytest.raises(ks.KsError, match="BAD_OPTION"):
        ks.set_option("ldg", 9)
    with pytest.raises(ks.KsError, match="BAD_OPTION"):
        ks.set_option("no_such_option", 1)
    ks.set_option("pad_prod", 0)
    ks.set_option("pad_prod")  # back to the default
    assert ks.get_option("pad_prod") == -1
    import subprocess
    import sys
    code = ("import paper_2604_25422_b200 as ks; print(ks.get_option('ldg'), ks.get_option('disable_tma'))")
    env = dict(os.environ, KS_LDG="0", KS_DISABLE_TMA="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True)
    assert out.stdout.split() == ["1", "0"], out.stdout + out.stderr


def test_python_mirror_checks_outputs_before_the_c_abi():
    """Outputs, kernels and workspaces of the wrong kind / dtype / shape are
    rejected in Python: the C ABI takes raw pointers and would otherwise
    write out of bounds or dereference a host pointer on the device."""
    import paper_2604_25422_b200 as ks
    x = np.zeros((2, 3, 16), np.float32)
    k = np.zeros((3, 5), np.float32)
    with pytest.raises(ks.DimensionError, match="out"):
        ks.forward(x, k, out=np.zeros((2, 3, 15), np.float32))
    with pytest.raises(TypeError, match="dtype"):
        ks.forward(x, k, out=np.zeros((2, 3, 16), np.float64))
    with pytest.raises(TypeError, match="dtype"):
        ks.forward(x, k.astype(np.float64))
    with pytest.raises(ks.DimensionError, match="out"):
        ks.backward_weight(x, x, 5, ks.HIERARCHICAL, out=np.zeros((3, 4), np.float32))
    torch = pytest.importorskip("torch")
    with pytest.raises(TypeError, match="numpy"):
        ks.forward(x, torch.zeros((3, 5)))

