"""Peer-store S' exchange (distributed transport "p2p") with real CUDA IPC.

Two processes share the one GPU this run has; a gloo group carries only the
IPC handles and host barriers -- no kernel waits on another rank, so the
ranks never need to be co-scheduled on the device.  Each rank's S' kernel
stores its partial of destination block q into rank q's receive slot through
the IPC mapping; the owner sums its slots in rank order.  Checked against the
single-process product on the full matrix (even and uneven shards, SJLT and
Gaussian operators, and reuse of the receive slots on a second call).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

REL = 1e-12


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, n_rows, n, d, kind, q):
    import torch.distributed as dist
    from paper_2302_01977_b200 import device
    from paper_2302_01977_b200 import distributed as D
    from paper_2302_01977_b200 import sketching as sk
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        rng = np.random.default_rng(n_rows + n + d)
        A = rng.standard_normal((n_rows, n))
        kw = dict(alpha=4, construction=sk.GRAPH) if kind == sk.SJLT else {}
        op = sk.new_operator(kind, n, d, seed=(n, d), **kw)
        r0, r1 = D.shard_bounds(n_rows, world)[rank]
        dA = device.DeviceMatrix.from_host(A[r0:r1])
        results = []
        for _ in range(2):  # second call reuses the receive slots
            S, St = D.sketch_row_sharded(dA, op, rank=rank, world=world, n_rows=n_rows,
                                         transport="p2p")
            results.append((S.cpu().numpy().T.copy(), St.cpu().numpy().T.copy()))
        ref_S = sk.apply_right(A, op)[r0:r1]
        ref_St = sk.apply_right_transposed(A, op)[r0:r1]
        errs = []
        for S, St in results:
            errs.append((float(np.linalg.norm(S - ref_S) / max(np.linalg.norm(ref_S), 1e-300)),
                         float(np.linalg.norm(St - ref_St) / max(np.linalg.norm(ref_St), 1e-300)),
                         bool(np.array_equal(St, results[0][1]))))
        dist.barrier()
        D.release_peer_slots()
        q.put((rank, errs, None))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, None, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_rows,n,d,kind", [(600, 600, 64, "sjlt"), (601, 601, 96, "sjlt"),
                                             (512, 512, 48, "gaussian")])
def test_p2p_row_sharded_transposed(cuda, n_rows, n, d, kind):
    assert n_rows == n  # S' = A^T R^T over the row space
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, n_rows, n, d, kind, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, errs, exc = q.get(timeout=300)
        out[rank] = (errs, exc)
    for p in procs:
        p.join(timeout=60)
    for rank, (errs, exc) in out.items():
        assert exc is None, f"rank {rank}: {exc}"
        for e_s, e_st, same in errs:
            assert e_s <= REL and e_st <= REL
            assert same  # deterministic across calls
