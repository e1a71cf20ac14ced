"""Row-sharded sketch logic on a 2-rank gloo process group (CPU).

The local products are the CPU oracle (injected through the test hooks of
distributed.sketch_row_sharded); the sharding, the per-destination partial
blocks, the operator restriction and both reductions (NCCL-style
reduce-scatter and the fixed-order one) are the product code.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2302_01977_b200 import distributed as D
from paper_2302_01977_b200 import sketching as sk


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class HostMat:
    """Stand-in for a DeviceMatrix holding a host row shard (F-order)."""

    def __init__(self, a):
        self.a = np.asfortranarray(a)
        self.rows, self.cols = self.a.shape


def _local_right(A, op):
    out = O.apply_right(A.a, op)               # (m, d) F-order
    return torch.from_numpy(np.ascontiguousarray(out.T))


def _local_transposed(A, sub_op, bounds):
    parts = []
    for c0, c1 in bounds:
        part = O.apply_right_transposed(A.a[:, c0:c1], sub_op)   # (m_q, d)
        parts.append(torch.from_numpy(np.ascontiguousarray(part.T)))
    return parts


def _worker(rank, world, port, n, kind, det, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        A = rng.standard_normal((n, n))
        kw = dict(alpha=4, construction=sk.BLOCK) if kind == sk.SJLT else {}
        op = sk.new_operator(kind, n, 32, seed=(0, 0), **kw)
        r0, r1 = D.shard_bounds(n, world)[rank]
        S, St = D.sketch_row_sharded(HostMat(A[r0:r1]), op, rank=rank, world=world, n_rows=n,
                                     deterministic=det, local_right=_local_right,
                                     local_transposed=_local_transposed)
        q.put((rank, r0, r1, S.numpy().T.copy(), St.numpy().T.copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,det", [(sk.SJLT, 96, False), (sk.SJLT, 97, True),
                                         (sk.GAUSSIAN, 64, False), (sk.GAUSSIAN, 63, True)])
def test_two_rank_row_sharding_matches_single_process(kind, n, det):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, kind, det, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(7)
    A = rng.standard_normal((n, n))
    kw = dict(alpha=4, construction=sk.BLOCK) if kind == sk.SJLT else {}
    op = sk.new_operator(kind, n, 32, seed=(0, 0), **kw)
    S_ref = O.apply_right(A, op)
    St_ref = O.apply_right_transposed(A, op)
    for rank, r0, r1, S, St in got:
        np.testing.assert_array_equal(S, S_ref[r0:r1])          # rows are local: exact
        assert O.rel_frobenius(St, St_ref[r0:r1]) <= 1e-13     # partial sums reassociate


def test_shard_bounds_and_restriction():
    assert D.shard_bounds(10, 3) == [(0, 4), (4, 7), (7, 10)]
    op = sk.new_operator(sk.SJLT, 40, 8, seed=1, alpha=2, construction=sk.GRAPH)
    sub = D.restrict_operator(op, 10, 25)
    np.testing.assert_array_equal(sk.dense_rows(sub, np.arange(15), np.arange(8)),
                                  sk.dense_rows(op, np.arange(10, 25), np.arange(8)))
    with pytest.raises(ValueError):
        D.restrict_block(sk.new_operator(sk.SRHT, 16, 4, seed=0).blocks[0], 0, 8)


def test_scaling_model():
    m = D.scaling_model(131072, 2048, 8, 6455.9)
    assert 0 < m["serial_eff"] < m["overlap_eff"] <= 1.0


def test_transport_selection_and_validation():
    """Unknown transports are rejected; the CPU test hooks select the
    collective transport (the p2p transport needs CUDA IPC and is covered by
    tests/test_gpu_p2p.py)."""
    n, d = 64, 16
    A = np.random.default_rng(1).standard_normal((n, n))
    op = sk.new_operator(sk.SJLT, n, d, seed=3, alpha=2, construction=sk.GRAPH)
    with pytest.raises(ValueError, match="unknown transport"):
        D.sketch_row_sharded(HostMat(A), op, rank=0, world=1, n_rows=n, transport="carrier-pigeon",
                             local_right=_local_right)
    S, St = D.sketch_row_sharded(HostMat(A), op, rank=0, world=1, n_rows=n,
                                 local_right=_local_right, local_transposed=_local_transposed)
    np.testing.assert_allclose(St.numpy().T, O.apply_right_transposed(A, op), rtol=0, atol=1e-12)


def _agree_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank 1 "fails to map a peer": every rank must see the failure
        q.put((rank, D._all_ranks_ok(rank != 1, None), D._all_ranks_ok(True, None)))
    finally:
        dist.destroy_process_group()


def test_peer_mapping_failure_is_agreed_by_all_ranks():
    """The p2p S' transport falls back to NCCL only collectively: a peer
    mapping failure on one rank is reported on every rank (no rank may take
    the p2p path while another takes the reduce-scatter)."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_agree_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == [(0, False, True), (1, False, True)]
