"""GPU, world size >= 2 on ONE B200: the library's own multi-rank dW paths.

This round's boxes have one GPU, and NCCL refuses two ranks on one device, so
the ranks here are processes sharing cuda:0, joined by a gloo group whose
all-gather is handed to the library (ks_comm_init_host).  Only bytes cross
gloo; every sum runs in the library's kernels:

* ks_rank_tree_sum_f32 -- the fixed cross-rank tree, world 1..64, bitwise
  against its definition (the reference's midpoint split over ranks);
* ks_dwconv1d_dw_f32_peer -- stage 1 into CUDA-IPC-exported buffers, then the
  signal / wait / combine kernel reading the other process's partials through
  its IPC mapping.  Several back-to-back calls exercise the epoch-parity
  double buffer; with the global plan dk is bitwise the 1-GPU HIERARCHICAL
  dW of the whole batch; uneven shards (different group counts per rank)
  combine through the published headers;
* ks_dwconv1d_dw_allreduce_f32 on a host communicator (all-gather + tree);
* the host-buffer step ks_dwconv1d_step_f32_host per shard, combined.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from test_dist_gloo import gloo_allgather, rank_tree, run_world  # noqa: E402

HIER_TOL = 1e-4


def same(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8, 16, 64])
def test_rank_tree_sum_bitwise(world):
    import paper_2604_25422_b200 as ks
    g = torch.randn((world, 3000), dtype=torch.float32, device="cuda") * 1e3
    out = torch.empty(3000, dtype=torch.float32, device="cuda")
    ks.rank_tree_sum(g, out)
    torch.cuda.synchronize()
    want = rank_tree([r for r in g.cpu().numpy()])
    assert same(out.cpu().numpy(), want)


def _peer_worker(rank, world, results, B, H, L, K, seeds, mode):
    import paper_2604_25422_b200 as ks
    torch.cuda.set_device(0)
    b0, nb = ks.shard_rows(B, world, rank)
    comm = ks.Comm.host(world, rank, gloo_allgather)
    peer = comm.peer(nb, H, L, K, B_total=B)
    try:
        ins = [ks.make_inputs(s, nb, H, L, K, device="cuda", b0=b0, B_total=B) for s in seeds]
        torch.cuda.synchronize()
        # back to back, no host synchronisation: the epoch parity keeps a rank's
        # partials of call e+2 from overwriting what a peer still reads for e
        outs = [peer.backward_weight(gy, x, K, mode, B_total=B) for x, k, gy in ins]
        torch.cuda.synchronize()
        results[rank] = [o.cpu().numpy() for o in outs]
        results[f"timed_out{rank}"] = peer.timed_out()
    finally:
        peer.close()
        comm.close()


@pytest.mark.parametrize("shape", [(32, 16, 4096, 7), (16, 8, 2048, 200), (8, 4, 1000, 9), (64, 4, 2048, 16)])
@pytest.mark.parametrize("world", [2, 4])
def test_peer_combine_global_plan_equals_one_gpu(shape, world):
    """Two or four processes on one GPU through the fused peer combine: every
    rank's dk is bitwise the 1-GPU HIERARCHICAL dW of the whole batch (the
    global plan puts each rank's row groups exactly where the 1-GPU plan has
    them), over four back-to-back calls with different inputs."""
    import paper_2604_25422_b200 as ks
    B, H, L, K = shape
    seeds = [3, 4, 5, 6]
    mode = ks.FUSED
    res = run_world(world, _peer_worker, B, H, L, K, seeds, mode)
    for r in range(world):
        assert not res[f"timed_out{r}"]
    for e, s in enumerate(seeds):
        x, k, gy = ks.make_inputs(s, B, H, L, K, device="cuda")
        ref = ks.backward_weight(gy, x, K, ks.HIERARCHICAL, 0, mode).cpu().numpy()
        for r in range(world):
            assert same(res[r][e], ref), (e, r)


@pytest.mark.parametrize("shape", [(33, 4, 2048, 7), (5, 6, 4096, 130), (7, 3, 300, 5)])
def test_peer_combine_uneven_shards(oracle, shape):
    """Uneven shards (B % world != 0, so the ranks' row-group counts differ):
    each rank publishes its G with its partials; both ranks end with the same
    bits, within tolerance of the fp64 truth."""
    import paper_2604_25422_b200 as ks
    from oracle.oracle import SEQUENTIAL, normwise
    B, H, L, K = shape
    res = run_world(2, _peer_worker, B, H, L, K, [8, 9, 10], ks.SEPARATE)
    assert not res["timed_out0"] and not res["timed_out1"]
    for e, s in enumerate([8, 9, 10]):
        assert same(res[0][e], res[1][e])
        x, k, gy = oracle.fill_inputs(s, B, H, L, K)
        truth = oracle.backward_weight(gy.astype(np.float64), x.astype(np.float64), K, SEQUENTIAL)
        assert normwise(res[0][e], truth) <= HIER_TOL


def _mismatch_worker(rank, world, results):
    import paper_2604_25422_b200 as ks
    torch.cuda.set_device(0)
    comm = ks.Comm.host(world, rank, gloo_allgather)
    K = 7 if rank == 0 else 9  # ranks disagree on the shape
    peer = comm.peer(4, 4, 2048, 9)
    try:
        x, k, gy = ks.make_inputs(1, 4, 4, 2048, K, device="cuda")
        dk = peer.backward_weight(gy, x, K, ks.FUSED)
        torch.cuda.synchronize()
        results[rank] = (np.isnan(dk.cpu().numpy()).all(), peer.timed_out())
        try:
            peer.backward_weight(gy, x, K, ks.FUSED)
            results[f"err{rank}"] = None
        except ks.KsError as e:
            results[f"err{rank}"] = str(e)
    finally:
        peer.close()
        comm.close()


def test_peer_combine_rejects_mismatched_ranks():
    """A rank whose (H, K) differ from its peer's: both combines write NaN (not
    a plausible wrong gradient), the flag is set, and the next call fails with
    KS_ERR_TIMEOUT."""
    res = run_world(2, _mismatch_worker)
    for r in range(2):
        assert res[r] == (True, True)
        assert "TIMEOUT" in res[f"err{r}"]


def _allreduce_worker(rank, world, results, B, H, L, K):
    import paper_2604_25422_b200 as ks
    torch.cuda.set_device(0)
    b0, nb = ks.shard_rows(B, world, rank)
    comm = ks.Comm.host(world, rank, gloo_allgather)
    try:
        x, k, gy = ks.make_inputs(2, nb, H, L, K, device="cuda", b0=b0, B_total=B)
        dk = ks.backward_weight(gy, x, K, ks.HIERARCHICAL, 0, ks.FUSED)
        local = dk.cpu().numpy()
        comm.allreduce_dw(dk)
        gather = torch.empty((world, H, K), dtype=torch.float32, device="cuda")
        dk2 = torch.from_numpy(local).cuda()
        comm.allgather_sum_dw(dk2, gather)
        torch.cuda.synchronize()
        results[rank] = (local, dk.cpu().numpy(), dk2.cpu().numpy())
    finally:
        comm.close()


@pytest.mark.parametrize("world", [2, 3])
def test_host_comm_allreduce_is_rank_tree(world):
    """ks_dwconv1d_dw_allreduce_f32 / _allgather_sum_f32 over a host
    communicator: every rank ends with the rank tree of the local dks, bit for
    bit, and the sum is within tolerance of the whole batch's dW."""
    B, H, L, K = 12, 8, 2048, 11
    res = run_world(world, _allreduce_worker, B, H, L, K)
    want = rank_tree([res[r][0] for r in range(world)])
    for r in range(world):
        assert same(res[r][1], want) and same(res[r][2], want)


def _step_host_worker(rank, world, results, B, H, L, K):
    import paper_2604_25422_b200 as ks
    from oracle.oracle import Oracle
    torch.cuda.set_device(0)
    b0, nb = ks.shard_rows(B, world, rank)
    x, k, gy = Oracle().fill_inputs(4, B, H, L, K)
    xs, gs = np.ascontiguousarray(x[b0:b0 + nb]), np.ascontiguousarray(gy[b0:b0 + nb])
    y, dx, dk = ks.step_host(xs, k, gs, scheme=ks.HIERARCHICAL, mode=ks.FUSED)
    comm = ks.Comm.host(world, rank, gloo_allgather)
    try:
        dkd = torch.from_numpy(dk).cuda()
        comm.allreduce_dw(dkd)
        results[rank] = (y, dx, dkd.cpu().numpy())
    finally:
        comm.close()


def test_step_host_per_shard_world2(oracle):
    """The host-buffer step (ks_dwconv1d_step_f32_host) on each rank's batch
    shard, dk combined through the library: y and dx of both shards together
    bitwise equal the reference on the whole batch, dk within tolerance and
    identical on both ranks."""
    from oracle.oracle import FUSED, SEQUENTIAL, normwise
    B, H, L, K = 9, 4, 4096, 7
    res = run_world(2, _step_host_worker, B, H, L, K)
    x, k, gy = oracle.fill_inputs(4, B, H, L, K)
    y = np.concatenate([res[0][0], res[1][0]])
    dx = np.concatenate([res[0][1], res[1][1]])
    assert same(y, oracle.forward(x, k, FUSED))
    assert same(dx, oracle.backward_input(gy, k, FUSED))
    assert same(res[0][2], res[1][2])
    truth = oracle.backward_weight(gy.astype(np.float64), x.astype(np.float64), K, SEQUENTIAL)
    assert normwise(res[0][2], truth) <= HIER_TOL


def _chunked_worker(rank, world, results, B, H, L, K, chunk, mode, bounds):
    import paper_2604_25422_b200 as ks
    torch.cuda.set_device(0)
    b0, b1 = bounds[rank], bounds[rank + 1]
    comm = ks.Comm.host(world, rank, gloo_allgather)
    try:
        if b1 > b0:
            x, k, gy = ks.make_inputs(7, b1 - b0, H, L, K, device="cuda", b0=b0, B_total=B)
        else:  # a rank without rows still takes part in the exchange
            x = gy = torch.empty((0, H, L), dtype=torch.float32, device="cuda")
        try:
            dk = comm.chunked_dw(gy, x, K, chunk, mode, b0, B)
            torch.cuda.synchronize()
            results[rank] = dk.cpu().numpy()
        except ks.KsError as e:
            results[rank] = f"error: {e}"
    finally:
        comm.close()


@pytest.mark.parametrize("case", [
    # (B, H, L, K, chunk, mode, rank row bounds)
    (12, 4, 2048, 7, 2048, 1, [0, 4, 8, 12]),        # one row per chunk, 3 ranks
    (12, 3, 2048, 9, 4096, 0, [0, 6, 12]),           # two rows per chunk
    (10, 2, 1000, 33, 2000, 1, [0, 4, 10]),          # uneven shards, ragged L
    (9, 2, 512, 5, 1536, 0, [0, 3, 6, 9]),           # three rows per chunk
    (8, 2, 300, 7, 100, 1, [0, 0, 8]),               # an empty rank, chunks inside rows
    (6, 3, 256, 3, 1 << 20, 0, [0, 6, 6]),           # chunk >= B*L: SEQUENTIAL, all rows on rank 0
])
def test_chunked_dw_sharded_equals_one_gpu(case):
    """ks_dwconv1d_dw_chunked_sharded_f32 on 2-3 processes sharing the GPU:
    every rank's dk is bitwise the single-device CHUNKED(chunk) dW of the whole
    batch (and so independent of the rank count), uneven and empty shards
    included."""
    import paper_2604_25422_b200 as ks
    B, H, L, K, chunk, mode, bounds = case
    world = len(bounds) - 1
    res = run_world(world, _chunked_worker, B, H, L, K, chunk, mode, bounds)
    x, k, gy = ks.make_inputs(7, B, H, L, K, device="cuda")
    ref = ks.backward_weight(gy, x, K, ks.CHUNKED, chunk, mode).cpu().numpy()
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
        assert same(res[r], ref), r


def test_chunked_dw_sharded_rejects_straddling_chunks():
    """A chunk that would straddle two ranks' rows (rank boundary * L not a
    multiple of chunk) is refused on every rank (KS_ERR_SHARD), not summed in a
    different order."""
    res = run_world(2, _chunked_worker, 8, 2, 1024, 7, 3072, 1, [0, 4, 8])
    assert isinstance(res[0], str) and isinstance(res[1], str)
    assert "shard" in res[0].lower() or "13" in res[0]


def _chunked_mismatch_worker(rank, world, results):
    import paper_2604_25422_b200 as ks
    torch.cuda.set_device(0)
    comm = ks.Comm.host(world, rank, gloo_allgather)
    try:
        K = 7 if rank == 0 else 9  # the ranks disagree on K
        x, k, gy = ks.make_inputs(7, 4, 2, 1024, K, device="cuda", b0=4 * rank, B_total=8)
        try:
            comm.chunked_dw(gy, x, K, 1024, ks.FUSED, 4 * rank, 8)
            results[rank] = "ok"
        except ks.KsError as e:
            results[rank] = f"error: {e}"
    finally:
        comm.close()


def test_chunked_dw_sharded_rejects_disagreeing_ranks():
    """Ranks that disagree on the shape are refused on every rank before any
    gather of differently sized partials."""
    res = run_world(2, _chunked_mismatch_worker)
    assert res[0].startswith("error") and res[1].startswith("error")
