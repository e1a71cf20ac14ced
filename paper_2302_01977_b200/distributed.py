"""Row-block sharded sketching across GPUs (one process per GPU).

BASELINE.json C5 / SURVEY.md §8(e).  GPU g holds rows [r0_g, r1_g) of A (all n
columns) and the full operator R (tiny for SJLT; d x n for Gaussian):

  S  = A R^T      rows are local:  S[r0:r1] = A_g R^T           -- no communication
  S' = A^T R^T  = sum_g A_g^T R_g^T,  R_g = R restricted to input indices [r0, r1)
                   every GPU forms partials for all n output rows, blocked by
                   destination rank, and a reduce-scatter leaves GPU g with
                   S'[r0:r1] (the same row sharding as S).

The destination blocks are produced by separate launches over column
slices of A_g (contiguous in the column-major layout), so each block is a
contiguous (m_q x d) buffer and the reduce-scatter needs no repacking.

Transports for the S' exchange:
  "p2p" (default on GPUs) -- no reduction collective: every rank's S' kernel
        stores destination block q straight into rank q's receive slot
        [rank] through a CUDA-IPC mapping of rank q's buffer (the kernel's
        epilogue writes cross NVLink tile by tile while other tiles are
        still computing); after a barrier each rank sums its slots in rank
        order (hsk_sum_slices) -- deterministic, uneven shards allowed.
  "nccl" -- reduce_scatter_tensor over the process group (the baseline), or
        with `deterministic=True` a gather of every partial of block q on
        rank q summed in rank order.

SRHT mixes all input indices in its FWHT, so only S = A R^T row-shards; its
S' is formed on column shards (`sketch_columns_local`).
"""

from __future__ import annotations

import numpy as np

from . import operators as ops

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = None
    dist = None


def shard_bounds(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous near-equal row blocks [r0, r1) per rank."""
    base, extra = divmod(n, world)
    out, r = [], 0
    for g in range(world):
        m = base + (1 if g < extra else 0)
        out.append((r, r + m))
        r += m
    return out


def restrict_block(block, r0: int, r1: int):
    """The block's operator restricted to input indices [r0, r1)."""
    if block.kind == ops.SJLT:
        sub = ops.SjltBlock.from_pattern(r1 - r0, block.rows, block.alpha,
                                         block._pos[r0:r1], block._signs[r0:r1])
        sub._scale = block._scale
        return sub
    if block.kind == ops.GAUSSIAN:
        sub = ops.GaussianBlock.__new__(ops.GaussianBlock)
        sub.n, sub.rows = r1 - r0, block.rows
        sub.matrix = np.ascontiguousarray(block.matrix[:, r0:r1])
        return sub
    raise ValueError("SRHT does not decompose over input-index shards")


def restrict_operator(op, r0: int, r1: int):
    blocks = tuple(restrict_block(b, r0, r1) for b in op.blocks)
    return ops.SketchOperator(op.kind, r1 - r0, blocks, op.alpha, op.construction)


_RESTRICTED: dict = {}


def _restricted_cached(op, r0: int, r1: int):
    """restrict_operator, memoised per (operator blocks, shard) so the device
    state of the restricted blocks (SJLT plans, Gaussian matrices) is built
    once, not on every sketch call.  Keeps the source blocks alive so ids
    are not reused; an operator grown by append_columns has new blocks and
    therefore a new key."""
    key = (tuple(id(b) for b in op.blocks), r0, r1)
    hit = _RESTRICTED.get(key)
    if hit is None:
        if len(_RESTRICTED) > 64:
            _RESTRICTED.clear()
        hit = (op.blocks, restrict_operator(op, r0, r1))
        _RESTRICTED[key] = hit
    return hit[1]


# --------------------------------------------------------------- local math

def _gpu_local_right(A_shard, op):
    from . import sketching as sk
    return sk.apply_right_device(A_shard, op)


def _gpu_local_transposed_blocks(A_shard, sub_op, bounds):
    """Partials of S' for each destination row block, as torch tensors of
    shape (d, m_q) (column-major m_q x d)."""
    from . import device
    from . import sketching as sk
    outs = []
    for (c0, c1) in bounds:
        view = A_shard.column_view(c0, c1 - c0)
        part = device.DeviceMatrix.empty(c1 - c0, sub_op.d, ld=max(1, c1 - c0))
        sk.apply_right_transposed_device(view, sub_op, out=part)
        outs.append(part.t[:, :c1 - c0] if part.t.shape[1] != c1 - c0 else part.t)
    return outs


class PeerSlots:
    """This rank's receive buffer for the p2p S' exchange -- two sets (calls
    alternate between them) of `world` slots of (ld x d) doubles, column-major,
    slot g written by rank g -- and CUDA-IPC mappings of every peer's buffer
    (one process per GPU on one node)."""

    def __init__(self, world: int, rank: int, ld: int, d: int, group=None):
        import ctypes
        from . import _lib
        self.world, self.rank, self.ld, self.d = world, rank, ld, d
        self.slot_elems = ld * d
        self.set_elems = world * self.slot_elems
        self.phase = 0  # the slot set of the next call
        own = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        _lib.call("hsk_ipc_alloc", 2 * self.set_elems * 8, ctypes.byref(own), handle)
        self.own = own.value
        handles = [None] * world
        if world > 1:
            dist.all_gather_object(handles, bytes(handle), group=group)
        self.peer = []
        err = None
        for q in range(world):
            if q == rank:
                self.peer.append(self.own)
                continue
            p = ctypes.c_void_p()
            buf = ctypes.create_string_buffer(handles[q], 64)
            try:
                _lib.call("hsk_ipc_open", buf, ctypes.byref(p))
            except RuntimeError as e:  # no peer mapping between these GPUs
                err = err or e
                p = ctypes.c_void_p()
            self.peer.append(p.value)
        # every rank must take the same transport: agree on success
        if world > 1 and not _all_ranks_ok(err is None, group):
            self.close()
            raise PeerMappingError(f"CUDA IPC peer mapping failed on some rank ({err or 'peer'})")

    def slot(self, q: int, rows: int):
        """Rank q's slot (current set) for this rank's partial of block q (rows x d)."""
        from . import device
        off = (self.phase * self.set_elems + self.rank * self.slot_elems) * 8
        return device.RawMatrix(self.peer[q] + off, rows, self.d, self.ld)

    def reduce(self, rows: int, out_ptr: int, ldo: int, stream: int):
        """out = sum of this rank's slots of the current set in rank order
        (first `rows` rows); the next call uses the other set."""
        from . import _lib
        _lib.call("hsk_sum_slices", self.own + self.phase * self.set_elems * 8, self.world,
                  self.slot_elems, rows, self.d, self.ld, out_ptr, ldo, stream)
        self.phase ^= 1

    def close(self):
        from . import _lib
        for q, p in enumerate(self.peer):
            if q != self.rank and p:
                _lib.call("hsk_ipc_close", p)
        if self.own:
            _lib.call("hsk_ipc_free", self.own)
        self.peer, self.own = [], 0


class PeerMappingError(RuntimeError):
    """Some rank could not map a peer's receive buffer (collectively raised)."""


def _all_ranks_ok(ok: bool, group) -> bool:
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32)
    if dist.get_backend(group) == "nccl":
        flag = flag.cuda()
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return bool(flag.item())


_SLOTS: dict = {}


def peer_slots(world: int, rank: int, ld: int, d: int, group=None) -> PeerSlots:
    """Receive slots for (group, shape), created collectively once and reused."""
    key = (id(group), world, rank, ld, d, torch.cuda.current_device())
    if key not in _SLOTS:
        _SLOTS[key] = PeerSlots(world, rank, ld, d, group)
    return _SLOTS[key]


def release_peer_slots():
    """Unmap and free every receive buffer (call collectively before exit)."""
    for s in _SLOTS.values():
        s.close()
    _SLOTS.clear()


_FENCE: dict = {}


def _stream_fence(group):
    """A device-side barrier in stream order: a one-element all-reduce that
    no rank completes before every rank's earlier kernels have finished (the
    current stream waits on it; no host synchronisation)."""
    t = _FENCE.get(id(group))
    if t is None:
        t = _FENCE[id(group)] = torch.zeros(1, dtype=torch.int32, device="cuda")
    dist.all_reduce(t, group=group)


def _p2p_transposed(A_shard, sub_op, bounds, rank: int, world: int, group):
    """S' rows of this rank via direct peer stores + rank-ordered local sum.

    Ordering without host round trips: the peer stores of every rank's S'
    kernels land before the stream-ordered fence (a kernel's stores are
    visible at its completion); each rank sums its slots after the fence.
    Calls alternate between two slot sets, so the writes of call t+1 go to
    the other set, and those of call t+2 -- issued after call t+1's fence,
    which every rank reaches only after its call-t sum -- never overwrite
    slots still being summed."""
    from . import device
    from . import sketching as sk
    m_max = max(b1 - b0 for b0, b1 in bounds)
    slots = peer_slots(world, rank, m_max, sub_op.d, group)
    for q, (c0, c1) in enumerate(bounds):
        if c1 > c0:
            view = A_shard.column_view(c0, c1 - c0)
            sk.apply_right_transposed_device(view, sub_op, out=slots.slot(q, c1 - c0))
    if world > 1:
        _stream_fence(group)
    r0, r1 = bounds[rank]
    out = torch.empty((sub_op.d, max(1, r1 - r0)), dtype=torch.float64, device="cuda")
    slots.reduce(r1 - r0, out.data_ptr(), max(1, r1 - r0), device.current_stream_ptr())
    return out[:, :r1 - r0]


def sketch_row_sharded(A_shard, op, *, rank: int, world: int, n_rows: int,
                       transposed: bool = True, group=None, deterministic: bool = False,
                       transport: str | None = None, local_right=None, local_transposed=None):
    """S rows and (optionally) S' rows of this rank's shard.

    A_shard: rows [r0, r1) of the global n_rows x op.n matrix (DeviceMatrix on
    GPU ranks).  Returns (S_local, St_local) as torch tensors of shape
    (d, m_local) -- column-major (m_local x d) -- St_local None unless
    `transposed`.  `local_right` / `local_transposed` replace the GPU kernels
    (test hook for CPU process groups).
    """
    bounds = shard_bounds(n_rows, world)
    r0, r1 = bounds[rank]
    local_right = local_right or (lambda A, o: _gpu_local_right(A, o).t[:, :A.rows])
    S_local = local_right(A_shard, op)
    if not transposed:
        return S_local, None
    if op.n != n_rows:
        raise ValueError("S' = A^T R^T needs a square operator over the row space")
    sub = _restricted_cached(op, r0, r1)
    auto = transport is None
    if auto:
        transport = "nccl" if (local_transposed is not None or deterministic) else "p2p"
    if transport == "p2p":
        try:
            return S_local, _p2p_transposed(A_shard, sub, bounds, rank, world, group)
        except PeerMappingError:
            if not auto:
                raise
            transport = "nccl"  # every rank got the same error: all fall back together
    if transport != "nccl":
        raise ValueError(f"unknown transport {transport!r}")
    local_transposed = local_transposed or _gpu_local_transposed_blocks
    parts = local_transposed(A_shard, sub, bounds)  # list of (d, m_q) tensors
    m_loc = r1 - r0
    d = op.d
    if world == 1:  # the whole S' is local
        return S_local, parts[0]
    if deterministic or any(b[1] - b[0] != m_loc for b in bounds):
        # fixed rank-order summation (bitwise reproducible; uneven shards OK)
        return S_local, _ordered_reduce_scatter(parts, rank, world, group)
    flat = torch.cat([p.contiguous().reshape(-1) for p in parts])
    out = torch.empty(d * m_loc, dtype=torch.float64, device=flat.device)
    dist.reduce_scatter_tensor(out, flat, op=dist.ReduceOp.SUM, group=group)
    return S_local, out.view(d, m_loc)


def _ordered_reduce_scatter(parts, rank: int, world: int, group):
    """out = sum over source ranks g = 0..world-1 (in that order) of the
    partial that rank g computed for this rank's block."""
    mine = None
    for q in range(world):
        # rank q collects everyone's partial for block q
        buf = parts[q].contiguous()
        gathered = [torch.empty_like(buf) for _ in range(world)] if q == rank else None
        if world == 1:
            gathered = [buf]
        else:
            dist.gather(buf, gather_list=gathered, dst=q, group=group)
        if q == rank:
            acc = gathered[0].clone()
            for g in range(1, world):
                acc += gathered[g]
            mine = acc
    return mine


def sketch_columns_local(A_cols, op):
    """S' rows for this rank's column block of A: columns are independent in
    A^T R^T, so column sharding needs no communication (any operator,
    including SRHT)."""
    from . import sketching as sk
    return sk.apply_right_transposed_device(A_cols, op)


def scaling_model(n: int, d: int, world: int, hbm_gbs: float, link_gbs: float = 770.0):
    """Roofline model of the C5 S' step: per-GPU A stream + reduce-scatter."""
    a_bytes = n * n * 8 / world
    t_compute = a_bytes / (hbm_gbs * 1e9)
    rs_bytes = n * d * 8 * (world - 1) / world
    t_comm = rs_bytes / (link_gbs * 1e9) if world > 1 else 0.0
    return {"t_compute_s": t_compute, "t_comm_s": t_comm,
            "serial_eff": t_compute / (t_compute + t_comm) if world > 1 else 1.0,
            "overlap_eff": min(1.0, t_compute / max(t_compute, t_comm)) if world > 1 else 1.0}


__all__ = ["shard_bounds", "restrict_block", "restrict_operator", "sketch_row_sharded",
           "sketch_columns_local", "scaling_model", "PeerSlots", "peer_slots",
           "release_peer_slots"]
