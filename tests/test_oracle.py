"""CPU: pin the oracle (oracle/ks_oracle.c) before trusting it.

1. Known answers from the reference's tests/test_conv_core.cpp
   (:61-69 y=[4,7,2], :110-117 dx=[0,2,0], :139-147 dk=[0,1,2], :71-85 K=1).
2. Bitwise equality with the committed golden fixtures, which were produced by
   the reference's own conv_core.cpp (tests/golden/make_golden.py).
3. Bitwise equality with oracle/_ref/libksref.so (the reference compiled from
   its sources) on fresh shapes, and the config-1 SHA-256 pins.
4. The splitmix64 skip-ahead used by the device generator.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle.oracle import CHUNKED, FUSED, PAIRWISE, SEPARATE, SEQUENTIAL, normwise

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def same(a, b):
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(bits(a), bits(b))


def test_known_answers(oracle):
    x = np.array([[[1, 2, 3]]], np.float32)
    k = np.array([[1, 0, 2]], np.float32)
    gy = np.array([[[1, 0, 0]]], np.float32)
    assert oracle.forward(x, k).ravel().tolist() == [4, 7, 2]
    assert oracle.backward_input(gy, k).ravel().tolist() == [0, 2, 0]
    for s, c in ((SEQUENTIAL, 0), (PAIRWISE, 0), (CHUNKED, 2)):
        assert oracle.backward_weight(gy, x, 3, s, c).ravel().tolist() == [0, 1, 2]


def test_k1_identity_bitwise(oracle):
    x, _, gy = oracle.fill_inputs(11, 2, 3, 7, 1)
    ones = np.ones((3, 1), np.float32)
    assert same(oracle.forward(x, ones), x)
    assert same(oracle.backward_input(gy, ones), gy)
    kc = np.array([[2.5], [-0.75], [3.0]], np.float32)
    assert same(oracle.forward(x, kc), (x * kc[None, :, :]).astype(np.float32))


def test_chunk_validation(oracle):
    x, _, gy = oracle.fill_inputs(1, 1, 1, 4, 3)
    with pytest.raises(ValueError):
        oracle.backward_weight(gy, x, 3, CHUNKED, 0)


def test_integer_data_all_schemes_agree(oracle):
    # reference tests/test_conv_core.cpp:161-181
    B, H, L, K = 8, 3, 32, 5
    rng = np.random.default_rng(17)
    x = rng.integers(-8, 9, (B, H, L)).astype(np.float32)
    gy = rng.integers(-8, 9, (B, H, L)).astype(np.float32)
    seq = oracle.backward_weight(gy, x, K, SEQUENTIAL)
    assert same(seq, oracle.backward_weight(gy, x, K, PAIRWISE))
    assert same(seq, oracle.backward_weight(gy, x, K, CHUNKED, 64))
    assert np.array_equal(seq.astype(np.int64), oracle.backward_weight_int(gy, x, K))


def test_oracle_matches_reference_goldens(oracle, golden):
    tags = sorted({k.split("/")[0] for k in golden.files})
    assert len(tags) >= 10
    for tag in tags:
        B, H, L, rest = tag.split("x")
        K, seed = rest.split("s")
        B, H, L, K, seed = int(B), int(H), int(L), int(K), int(seed)
        x, k, gy = oracle.fill_inputs(seed, B, H, L, K)
        assert same(x, golden[f"{tag}/x"]) and same(k, golden[f"{tag}/k"]) and same(gy, golden[f"{tag}/gy"])
        for mname, m in (("sep", SEPARATE), ("fus", FUSED)):
            assert same(oracle.forward(x, k, m), golden[f"{tag}/y_{mname}"]), tag
            assert same(oracle.backward_input(gy, k, m), golden[f"{tag}/dx_{mname}"]), tag
            for sname, s, c in (("seq", SEQUENTIAL, 0), ("pair", PAIRWISE, 0), ("chunk7", CHUNKED, 7),
                                ("chunk64", CHUNKED, 64), ("chunk1024", CHUNKED, 1024)):
                assert same(oracle.backward_weight(gy, x, K, s, c, m), golden[f"{tag}/dk_{sname}_{mname}"]), (tag, sname)
        xd, kd, gyd = x.astype(np.float64), k.astype(np.float64), gy.astype(np.float64)
        assert same(oracle.forward(xd, kd), golden[f"{tag}/y_f64"])
        assert same(oracle.backward_input(gyd, kd), golden[f"{tag}/dx_f64"])
        assert same(oracle.backward_weight(gyd, xd, K, SEQUENTIAL), golden[f"{tag}/dk_f64"])


def test_config1_hash_pins(oracle):
    with open(os.path.join(ROOT, "tests", "golden", "hashes.json")) as f:
        pins = json.load(f)["config1_seed1"]
    B, H, L, K = pins["shape"]
    x, k, gy = oracle.fill_inputs(1, B, H, L, K)
    h = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    assert h(x) == pins["x"] and h(k) == pins["k"] and h(gy) == pins["gy"]
    assert h(oracle.forward(x, k, SEPARATE)) == pins["y_sep"]
    assert h(oracle.forward(x, k, FUSED)) == pins["y_fus"]
    assert h(oracle.backward_input(gy, k, SEPARATE)) == pins["dx_sep"]
    assert h(oracle.backward_input(gy, k, FUSED)) == pins["dx_fus"]
    assert h(oracle.backward_weight(gy, x, K, PAIRWISE, 0, SEPARATE, threads=4)) == pins["dk_pair"]
    assert h(oracle.backward_weight(gy, x, K, CHUNKED, 1024, FUSED, threads=4)) == pins["dk_chunk1024_fus"]


@pytest.mark.parametrize("shape", [(2, 3, 17, 5), (3, 2, 33, 8), (2, 2, 10, 16), (1, 1, 1, 1),
                                   (2, 2, 3, 9), (5, 1, 40, 2), (2, 4, 129, 31)])
def test_oracle_matches_reference_build(oracle, reference, shape):
    B, H, L, K = shape
    x, k, gy = reference.fill_inputs(99, B, H, L, K)
    for m in (SEPARATE, FUSED):
        assert same(oracle.forward(x, k, m), reference.forward(x, k, m))
        assert same(oracle.backward_input(gy, k, m), reference.backward_input(gy, k, m))
        for s, c in ((SEQUENTIAL, 0), (PAIRWISE, 0), (CHUNKED, 3), (CHUNKED, L), (CHUNKED, 10 ** 9)):
            assert same(oracle.backward_weight(gy, x, K, s, c, m), reference.backward_weight(gy, x, K, s, c, m))
    # threaded channel-slice fan-outs are bitwise identical to the single call
    assert same(oracle.forward(x, k, SEPARATE, threads=3), reference.forward(x, k, SEPARATE, threads=3))
    assert same(oracle.backward_weight(gy, x, K, CHUNKED, 3, FUSED, threads=2),
                reference.backward_weight(gy, x, K, CHUNKED, 3, FUSED))


def test_reference_validate_bounds(reference):
    # tests/test_conv_core.cpp:279-290 on the reference build itself
    rep = reference.validate(64, 8, 48, 48, 1, [(SEQUENTIAL, 0), (CHUNKED, 1024)])
    assert 0 < rep["fwd"][0] <= 4e-6 and rep["bwd_in"][0] <= 4e-6 and rep["dk_spread_abs"] > 0


def test_skip_ahead(oracle):
    # draw n of SplitMix64(seed) == mix(seed + n*gamma): rng.hpp:17-21
    seed = 12345
    state = seed
    gamma = 0x9E3779B97F4A7C15
    mask = (1 << 64) - 1
    for n in range(1, 50):
        state = (state + gamma) & mask
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        z ^= z >> 31
        assert oracle.splitmix64_at(seed, n) == z
    full = oracle.fill_pm1(seed, 0, 1000)
    assert same(oracle.fill_pm1(seed, 600, 400), full[600:])


def test_normwise_metric():
    ref = np.array([1.0, -2.0, 0.0], np.float32)
    assert normwise(ref, ref) == 0.0
    assert abs(normwise(ref + np.float32(1e-3), ref) - 5e-4) < 1e-7
