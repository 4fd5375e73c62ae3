"""CPU, world_size 2 over gloo: the batch-sharded multi-GPU design, checked
on the host.

The GPU box used for this round has one GPU, so the N>1 path is covered here
by construction: each rank takes the contiguous batch slice the C library's
ks_shard_rows gives it, computes its local fwd / dX / dW (with the oracle
standing in for the kernels), and the ranks exchange dW exactly as the
library does:
* allreduce(sum)  -- ks_dwconv1d_dw_allreduce_f32 (tolerance);
* allgather + midpoint tree in rank order -- ks_dwconv1d_dw_allgather_sum_f32,
  which for PAIRWISE on power-of-two shards is BITWISE the 1-GPU result,
  because every shard's local tree is a node of the global tree.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def rank_tree(vals):
    """Midpoint-split pairwise sum in rank order (dist.cu rank_tree_sum)."""
    if len(vals) == 1:
        return vals[0]
    mid = len(vals) // 2
    return (rank_tree(vals[:mid]) + rank_tree(vals[mid:])).astype(np.float32)


def _entry(rank, world, port, fn, results, args):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, results, *args)
    finally:
        dist.destroy_process_group()


def run_world(world, fn, *args):
    """Run fn(rank, world, results, *args) on `world` processes joined by a
    gloo group (127.0.0.1); returns the shared results dict."""
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_entry, args=(world, _free_port(), fn, results, args), nprocs=world, join=True)
    return dict(results)


def gloo_allgather(data: bytes):
    """A host all-gather over the default (gloo) group: the transport handed
    to the library's ks_comm_init_host."""
    t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.numpy().tobytes() for o in out]


def host_comm_worker(rank, world, results):
    """The library's host communicator on CPU: rank-ordered all-gather of
    uneven payloads' fixed-size records through the caller's gloo transport."""
    import paper_2604_25422_b200 as ks
    comm = ks.Comm.host(world, rank, gloo_allgather)
    try:
        got = comm.allgather_bytes(bytes([rank]) * 5 + rank.to_bytes(4, "little"))
        results[rank] = got
    finally:
        comm.close()
    assert got == [bytes([r]) * 5 + r.to_bytes(4, "little") for r in range(world)]


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import FUSED, PAIRWISE, Oracle
        import paper_2604_25422_b200 as ks
        o = Oracle()
        B, H, L, K = 8, 3, 64, 7
        x, k, gy = o.fill_inputs(5, B, H, L, K)
        b0, nb = ks.shard_rows(B, world, rank)
        xs, gs = np.ascontiguousarray(x[b0:b0 + nb]), np.ascontiguousarray(gy[b0:b0 + nb])
        y = o.forward(xs, k, FUSED)
        dxl = o.backward_input(gs, k, FUSED)
        dkl = o.backward_weight(gs, xs, K, PAIRWISE)
        # fwd/dX: no communication; gather only to check coverage
        ys = [torch.zeros((B // world, H, L)) for _ in range(world)]
        dist.all_gather(ys, torch.from_numpy(y))
        dxs = [torch.zeros((B // world, H, L)) for _ in range(world)]
        dist.all_gather(dxs, torch.from_numpy(dxl))
        # dW exchange, both library variants
        gath = [torch.zeros((H, K)) for _ in range(world)]
        dist.all_gather(gath, torch.from_numpy(dkl))
        exact = rank_tree([g.numpy() for g in gath])
        red = torch.from_numpy(dkl.copy())
        dist.all_reduce(red)
        if rank == 0:
            results["y"] = np.concatenate([t.numpy() for t in ys])
            results["dx"] = np.concatenate([t.numpy() for t in dxs])
            results["exact"] = exact
            results["allreduce"] = red.numpy()
            results["full"] = (x, k, gy)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_batch_sharded_step_world2(world):
    from oracle.oracle import FUSED, PAIRWISE, Oracle, normwise
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    o = Oracle()
    x, k, gy = results["full"]
    K = k.shape[1]
    assert np.array_equal(results["y"], o.forward(x, k, FUSED))
    assert np.array_equal(results["dx"], o.backward_input(gy, k, FUSED))
    full = o.backward_weight(gy, x, K, PAIRWISE)
    assert np.array_equal(results["exact"].view(np.uint32), full.view(np.uint32))
    assert normwise(results["allreduce"], full) <= 1e-6


def test_host_communicator_world2_gloo():
    """ks_comm_init_host over a torch.distributed gloo all-gather, world size
    2 (CPU): the library's own communicator moves every rank's bytes in rank
    order -- the transport the multi-rank dW combines use when ranks share a
    GPU (tests/test_multirank_gpu.py runs those on the B200)."""
    res = run_world(2, host_comm_worker)
    assert res[0] == res[1]
