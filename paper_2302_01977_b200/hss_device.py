"""Device-resident HSS compression sweep.

The reference compressor (hsskit/hss_compress.py) sketches A once, then
sweeps the cluster tree bottom-up on the host: per node it forms local
samples from the sketch (`_leaf_windows` :189-196, `_internal_windows`
:198-212), reduced randoms (`_reduced_window` :253-266), gates them with
Householder QR + a two-pass projection (`_gate_side` :270-291,
dense_kernels.py:30-51) and compresses with column-pivoted-QR
interpolative decompositions (`compress_node` :293-315, dense_kernels.py:54-90).
Every adaptation round concatenates the whole n x d sketch on the host
(:181-182) and the nodes' growing samples (:246-251).

`device_driver_class(hss_compress)` returns a subclass of the reference's
own `_Driver` whose sweep logic (`sweep`, `run`, gating decisions, tolerances
per level, sketch schedule and operator draws) is the reference's, unchanged,
while every matrix it touches stays in HBM:

  * the sketch lives in an adaptive.DeviceSketch (S and S' appended in place
    by the libhsk kernels; no host concatenation, no D2H of S);
  * A is the device copy (DeviceAccessor / the accessor's cached upload) for
    the sketch; diagonal and cross blocks are requested through the accessor's
    extract() exactly as the reference requests them (gathered in HBM for a
    DeviceAccessor);
  * the random rows R^T(I_tau, cols) are materialised on the device from the
    operator's device state (bit-identical to the reference's dense_rows);
  * local samples and reduced randoms grow in preallocated column buffers;
    compressed leaves of equal size are updated as one batched GEMM per round
    (all leaves are visited back to back in the reference's topological
    order, deepest level first, :cluster_tree.py:134-141);
  * QR of the gate is cuSOLVER (torch.linalg.qr), the projection and the
    windows are cuBLAS GEMMs, and the interpolative decomposition is the
    hand-written column-pivoted QR kernel hsk_pqr (LAPACK dgeqp3 pivoting,
    stopped at the numerical rank) plus a triangular solve.

Only scalars cross to the host during the sweep (the gate norms, the last
diagonal of the incremental QR, the ID ranks and skeleton indices); the
final HssMatrix gets host copies of D, B12, B21, U_coeff and V_coeff, so the
reference's hss_ops (matvec, reconstruct_dense, relative_error, stats) use it
as is.  Install with `plugin.install(compressor=True)`.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _lib
from . import adaptive as _ad
from . import device as _dev
from . import sketching as _sk

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


class ColBuf:
    """rows x width matrix growing by columns, in a (rows, capacity) row-major
    tensor (appends write a column slice; views are strided)."""

    __slots__ = ("buf", "w")

    def __init__(self, first):
        rows, k = first.shape
        cap = max(2 * k, 64)
        self.buf = torch.empty((rows, cap), dtype=torch.float64, device=first.device)
        self.buf[:, :k] = first
        self.w = k

    def append(self, cols):
        rows, k = cols.shape
        if self.w + k > self.buf.shape[1]:
            nb = torch.empty((rows, max(2 * self.buf.shape[1], self.w + k)), dtype=torch.float64,
                             device=self.buf.device)
            nb[:, :self.w] = self.buf[:, :self.w]
            self.buf = nb
        self.buf[:, self.w:self.w + k] = cols
        self.w += k

    def view(self, c0: int = 0, c1: int | None = None):
        return self.buf[:, c0:self.w if c1 is None else c1]


class _NodeDev:
    __slots__ = ("D", "B12", "B21", "Sr", "Sc", "Rr", "Rc", "Qr", "Qc", "U", "V", "Jr_t", "Jc_t")

    def __init__(self):
        for name in self.__slots__:
            setattr(self, name, None)


def _qr(S):
    """Economic Householder QR (dense_kernels.qr): cuSOLVER geqrf/orgqr."""
    q, r = torch.linalg.qr(S, mode="reduced")
    return q, r


def _project_out(Q, S):
    """dense_kernels.project_out (:38-51): two block Gram-Schmidt passes."""
    if Q.numel() == 0:
        return S.clone()
    resid = torch.addmm(S, Q, Q.T @ S, alpha=-1.0)
    resid.addmm_(Q, Q.T @ resid, alpha=-1.0)
    return resid


_SIDE_STREAM = {}


def _side_stream():
    dev = torch.cuda.current_device()
    side = _SIDE_STREAM.get(dev)
    if side is None:
        side = _SIDE_STREAM[dev] = torch.cuda.Stream()
    return side


def row_interpolative_decompositions(S1, S2, eps_rel: float, eps_abs: float):
    """Two independent row IDs (a node's row and column samples), the second
    on a side stream so the two latency-bound factorisations overlap; both
    ranks and pivot orders come to the host in one copy."""
    side = _side_stream()
    cur = torch.cuda.current_stream()
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        M2 = _pqr_launch(S2, eps_rel, eps_abs)
    M1 = _pqr_launch(S1, eps_rel, eps_abs)
    cur.wait_stream(side)
    if M2 is not None:
        for t in M2:
            t.record_stream(cur)
    host = _pqr_host([M1, M2])
    return _pqr_finish(S1, M1, host[0]), _pqr_finish(S2, M2, host[1])


def _pqr_host(launched):
    """(rank, pivot order) of each queued factorisation, one D2H copy."""
    parts, sizes = [], []
    for L in launched:
        if L is None:
            sizes.append(None)
            continue
        _, perm, _, rank_t, _ = L
        parts += [rank_t.to(torch.int64), perm]
        sizes.append(perm.numel())
    flat = torch.cat(parts).cpu().numpy() if parts else np.empty(0, dtype=np.int64)
    out, o = [], 0
    for sz in sizes:
        if sz is None:
            out.append(None)
            continue
        out.append((int(flat[o]), flat[o + 1:o + 1 + sz]))
        o += 1 + sz
    return out


def _pqr_launch(S, eps_rel: float, eps_abs: float):
    """Queue hsk_pqr on a copy of S on the current stream (no host sync)."""
    if eps_rel < 0 or eps_abs < 0:
        raise ValueError("tolerances must be nonnegative")
    rows, width = S.shape
    if S.numel() == 0:
        return None
    dev = S.device
    M = S.contiguous().clone()           # (rows, width) row-major = S^T column-major, ld width
    m, n = width, rows                   # S^T is m x n
    ldr = max(min(m, n), 1)
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    Rb = torch.empty((n, ldr), dtype=torch.float64, device=dev)  # column-major min(m,n) x n
    rank_t = torch.zeros(1, dtype=torch.int32, device=dev)
    wbytes = int(_lib.load().hsk_pqr_work_bytes(m, n))
    work = torch.empty(wbytes, dtype=torch.uint8, device=dev)
    _lib.call("hsk_pqr", M.data_ptr(), m, n, width, float(eps_rel), float(eps_abs), perm.data_ptr(),
              Rb.data_ptr(), ldr, rank_t.data_ptr(), work.data_ptr(), wbytes,
              _dev.current_stream_ptr())
    return (M, perm, Rb, rank_t, work)


def _pqr_finish(S, launched, host=None):
    """Triangular solve and Y assembly (interpolative_decomposition :70-82)
    from the rank and pivot order; returns (U = Y^T, J)."""
    rows = S.shape[0]
    dev = S.device
    if launched is None:
        return torch.zeros((rows, 0), dtype=torch.float64, device=dev), np.empty(0, dtype=np.intp)
    _, perm, Rb, rank_t, _ = launched
    r, perm_h = host if host is not None else _pqr_host([launched])[0]
    n = rows
    Y = torch.zeros((r, n), dtype=torch.float64, device=dev)
    if r > 0:
        R = Rb[:, :r].T                  # r x n, pivot order
        Y[torch.arange(r, device=dev), perm[:r]] = 1.0
        if r < n:
            T = torch.linalg.solve_triangular(R[:, :r], R[:, r:], upper=True)
            Y[:, perm[r:]] = T
    return Y.T, perm_h[:r].astype(np.intp)


def row_interpolative_decomposition(S, eps_rel: float, eps_abs: float):
    """dense_kernels.row_interpolative_decomposition (:85-90) on the device:
    S ~= U S[J, :], U[J, :] = I.  Returns (U (rows x r) device, J host intp).

    The column ID of S^T (interpolative_decomposition, :54-82) runs the
    column-pivoted QR kernel hsk_pqr on a copy of S (row j of S = column j of
    S^T, contiguous), stopped at the numerical rank, then solves the leading
    triangle against the remaining columns."""
    return _pqr_finish(S, _pqr_launch(S, eps_rel, eps_abs))


def device_driver_class(hc, base=None):
    """A subclass of the reference's `_Driver` (hc: hsskit.hss_compress;
    `base` defaults to hc._Driver) keeping the sweep's matrices on the device."""
    Base = base if base is not None else hc._Driver
    NodeState = hc.NodeState

    class DeviceDriver(Base):
        """hss_compress._Driver with device-resident sketch, samples and bases."""

        def __init__(self, A, tree, opts):
            super().__init__(A, tree, opts)
            _dev.require_cuda()
            self.A_dev = _sk.device_matrix_of(A)
            self.dv = [_NodeDev() for _ in tree.nodes]
            self._nid = {id(nd): i for i, nd in enumerate(self.nodes)}
            self._ds = None
            self._blk_cache = {}
            self._Rt = None           # dense R^T, n x width (ColBuf)
            leaves = [t for t in tree.nodes if t.is_leaf]
            sizes = {t.size for t in leaves}
            # batched leaf updates need equal leaves tiling [0, n) in order
            self._uniform_leaf = None
            if len(sizes) == 1 and len(leaves) > 1:
                b = sizes.pop()
                los = sorted(t.lo for t in leaves)
                if los == list(range(0, self.n, b)):
                    self._uniform_leaf = b
            self._leaf_batch = None   # (c0, c1) -> (sr, sc, R) of every leaf, this round
            self._gate_cache = None   # both sides' gate results of the node being gated
            self._n_leaves = len(leaves)
            self._leaves_with_D = 0

        # -------------------------------------------------------- sketch
        def init_sketch(self) -> None:
            o = self.opts
            sk = hc.sketching
            self.op = sk.new_operator(o.kind, self.n, o.d0 + o.dd, self._block_seed(0),
                                      alpha=o.alpha, construction=o.construction)
            start = time.perf_counter()
            cap = min(self.n + o.dd, max(4 * (o.d0 + o.dd), 256))
            self._ds = _ad.DeviceSketch(self.A_dev, cap, growable=True)
            self._ds.start(self.op)
            torch.cuda.current_stream().synchronize()
            self.sketch_seconds += time.perf_counter() - start
            self._Rt = None
            for blk in self.op.blocks:
                self._append_dense_rows(blk)

        def extend_sketch(self) -> None:
            self.rounds += 1
            self.d += self.opts.dd
            self.op = hc.sketching.append_columns(self.op, self.opts.dd,
                                                  self._block_seed(self.rounds))
            start = time.perf_counter()
            self._ds.extend(self.op)      # only the new block touches A
            torch.cuda.current_stream().synchronize()
            self.sketch_seconds += time.perf_counter() - start
            self._append_dense_rows(self.op.blocks[-1])
            self._leaf_batch = None

        def _sketch_rows(self, which: str, lo: int, hi: int, c0: int, c1: int):
            dm = self._ds.S if which == "r" else self._ds.St
            return dm.t[c0:c1, lo:hi].T   # (hi-lo) x (c1-c0) view

        # ---------------------------------------------------- random rows
        def _block_dev(self, blk):
            st = _dev.block_state(blk)
            ent = self._blk_cache.get(id(blk))
            if ent is None:
                if blk.kind == "sjlt":
                    ent = (st.pos.view(st.n, st.alpha).long(),
                           st.sgn.view(st.n, st.alpha).to(torch.float64) * st.scale)
                elif blk.kind == "srht":
                    ent = (st.signs, st.sample)
                else:
                    ent = (st.R,)
                self._blk_cache[id(blk)] = (blk, ent)
            else:
                ent = ent[1]
            return st, ent

        def _append_dense_rows(self, blk):
            """R^T of a new block for every input index, appended once to the
            device buffer the windows read (the rows a leaf needs are then a
            view) -- the blocks' dense_rows (sketching.py:140-141, :184-191,
            :353-360) for I = all indices: exact values (0, +-scale, the
            Gaussian entries)."""
            st, ent = self._block_dev(blk)
            n = self.n
            if blk.kind == "sjlt":
                pos, val = ent
                full = torch.zeros((n, blk.rows), dtype=torch.float64, device="cuda")
                full.scatter_(1, pos, val)
                cols = full.T
            elif blk.kind == "gaussian":
                cols = ent[0]
            else:
                signs, sample = ent
                i = torch.arange(n, device="cuda", dtype=torch.int64)[None, :]
                x = sample[:, None] & i
                for sh in (32, 16, 8, 4, 2, 1):
                    x = x ^ (x >> sh)
                H = 1.0 - 2.0 * (x & 1).to(torch.float64)
                cols = H * signs[None, :n] * st.scale
            if self._Rt is None:
                self._Rt = ColBuf(cols.T)        # n x width (R^T), column-major rows
            else:
                self._Rt.append(cols.T)

        def _random_rows_dev(self, lo: int, hi: int, c0: int, c1: int):
            """R^T(lo:hi, c0:c1) (sketching.dense_rows, :460-476): a view of the
            dense buffer."""
            return self._Rt.view(c0, c1)[lo:hi]

        # ------------------------------------------------- sample updates
        @staticmethod
        def _range(cols):
            cols = np.asarray(cols)
            c0, c1 = int(cols[0]), int(cols[-1]) + 1
            assert c1 - c0 == cols.size, "column windows are contiguous ranges"
            return c0, c1

        def _leaf_batch_windows(self, c0: int, c1: int):
            """Windows of EVERY leaf for columns [c0, c1) in one batched
            GEMM pair: leaves tile [0, n) in equal blocks of b, so the
            sketch rows and the random rows reshape to (L, b, w)."""
            key = (c0, c1)
            if self._leaf_batch is not None and self._leaf_batch[0] == key:
                return self._leaf_batch[1]
            b = self._uniform_leaf
            L = self.n // b
            w = c1 - c0
            leaves = [t for t in self.tree.nodes if t.is_leaf]
            Ds = torch.stack([self.dv[t.nid].D for t in sorted(leaves, key=lambda t: t.lo)])
            R = self._random_rows_dev(0, self.n, c0, c1).reshape(L, b, w)
            Sr = self._ds.S.t[c0:c1, :self.n].T.reshape(L, b, w)
            Sc = self._ds.St.t[c0:c1, :self.n].T.reshape(L, b, w)
            sr = torch.baddbmm(Sr, Ds, R, alpha=-1.0)
            sc = torch.baddbmm(Sc, Ds.transpose(1, 2), R, alpha=-1.0)
            self._leaf_batch = (key, (sr, sc, R))
            return sr, sc, R

        def _leaf_windows(self, nid: int, cols):
            c0, c1 = cols if isinstance(cols, tuple) else self._range(cols)
            tnode = self.tree.nodes[nid]
            dv = self.dv[nid]
            if (self._uniform_leaf is not None and c0 == self.d and
                    self._leaves_with_D == self._n_leaves):
                sr, sc, R = self._leaf_batch_windows(c0, c1)
                i = tnode.lo // self._uniform_leaf
                return sr[i], sc[i], R[i]
            R = self._random_rows_dev(tnode.lo, tnode.hi, c0, c1)
            sr = torch.addmm(self._sketch_rows("r", tnode.lo, tnode.hi, c0, c1), dv.D, R, alpha=-1.0)
            sc = torch.addmm(self._sketch_rows("c", tnode.lo, tnode.hi, c0, c1), dv.D.T, R, alpha=-1.0)
            return sr, sc, R

        def _idx(self, nid: int, side: str):
            dv = self.dv[nid]
            attr = "Jr_t" if side == "r" else "Jc_t"
            t = getattr(dv, attr)
            if t is None:
                J = self.nodes[nid].J_row if side == "r" else self.nodes[nid].J_col
                t = torch.as_tensor(np.asarray(J, dtype=np.int64), device="cuda")
                setattr(dv, attr, t)
            return t

        def _internal_windows(self, nid: int, cols):
            c0, c1 = cols if isinstance(cols, tuple) else self._range(cols)
            tnode = self.tree.nodes[nid]
            dv = self.dv[nid]
            l, r = tnode.left.nid, tnode.right.nid
            d1, d2 = self.dv[l], self.dv[r]
            sr = torch.cat([
                torch.addmm(d1.Sr.view(c0, c1).index_select(0, self._idx(l, "r")), dv.B12,
                            d2.Rc.view(c0, c1), alpha=-1.0),
                torch.addmm(d2.Sr.view(c0, c1).index_select(0, self._idx(r, "r")), dv.B21,
                            d1.Rc.view(c0, c1), alpha=-1.0),
            ])
            sc = torch.cat([
                torch.addmm(d1.Sc.view(c0, c1).index_select(0, self._idx(l, "c")), dv.B21.T,
                            d2.Rr.view(c0, c1), alpha=-1.0),
                torch.addmm(d2.Sc.view(c0, c1).index_select(0, self._idx(r, "c")), dv.B12.T,
                            d1.Rr.view(c0, c1), alpha=-1.0),
            ])
            return sr, sc

        def _extract(self, rows, cols):
            """A.extract(rows, cols) on the device.  A DeviceAccessor's entries
            are gathered from HBM; any other accessor is asked through its own
            extract() -- the reference's matrix-access contract (the diagonal
            and cross blocks are the only entries requested, hss_compress.py
            module docstring and :213-229) -- and the block uploaded."""
            if isinstance(self.A, _sk.DeviceAccessor):
                t = self.A_dev.t
                r = torch.as_tensor(np.asarray(rows, dtype=np.int64), device="cuda")
                c = torch.as_tensor(np.asarray(cols, dtype=np.int64), device="cuda")
                return t.index_select(0, c).index_select(1, r).T.contiguous()
            blk = np.asarray(self.A.extract(rows, cols), dtype=np.float64)
            return torch.as_tensor(np.ascontiguousarray(blk), device="cuda")

        def _fetch_cross_blocks(self, nid: int) -> None:
            tnode = self.tree.nodes[nid]
            dv = self.dv[nid]
            c1 = self.nodes[tnode.left.nid]
            c2 = self.nodes[tnode.right.nid]
            dv.B12 = self._extract(c1.Itilde_row, c2.Itilde_col)
            dv.B21 = self._extract(c2.Itilde_row, c1.Itilde_col)

        def first_touch(self, nid: int) -> None:
            tnode = self.tree.nodes[nid]
            dv = self.dv[nid]
            rng = (0, self.width)
            if tnode.is_leaf:
                idx = np.arange(tnode.lo, tnode.hi)
                dv.D = self._extract(idx, idx)
                self._leaves_with_D += 1
                sr, sc, _ = self._leaf_windows(nid, rng)
            else:
                self._fetch_cross_blocks(nid)
                sr, sc = self._internal_windows(nid, rng)
            dv.Sr, dv.Sc = ColBuf(sr), ColBuf(sc)

        def append_window(self, nid: int, cols) -> None:
            c0, c1 = self._range(cols)
            tnode = self.tree.nodes[nid]
            node = self.nodes[nid]
            dv = self.dv[nid]
            if tnode.is_leaf:
                sr, sc, R = self._leaf_windows(nid, (c0, c1))
            else:
                sr, sc = self._internal_windows(nid, (c0, c1))
                R = None
            dv.Sr.append(sr)
            dv.Sc.append(sc)
            if node.state is NodeState.COMPRESSED:
                rr, rc = self._reduced_window(nid, (c0, c1), R)
                dv.Rr.append(rr)
                dv.Rc.append(rc)

        def _reduced_window(self, nid: int, cols, R_leaf):
            c0, c1 = cols if isinstance(cols, tuple) else self._range(cols)
            tnode = self.tree.nodes[nid]
            dv = self.dv[nid]
            if tnode.is_leaf:
                R = R_leaf if R_leaf is not None else self._random_rows_dev(tnode.lo, tnode.hi, c0, c1)
                return dv.U.T @ R, dv.V.T @ R
            d1, d2 = self.dv[tnode.left.nid], self.dv[tnode.right.nid]
            rr = dv.U.T @ torch.cat([d1.Rr.view(c0, c1), d2.Rr.view(c0, c1)])
            rc = dv.V.T @ torch.cat([d1.Rc.view(c0, c1), d2.Rc.view(c0, c1)])
            return rr, rc

        # ------------------------------------------- gating / compression
        def _gate_stage1(self, node, side: str):
            """Device part of _gate_side (:270-286) up to the Frobenius test:
            the first QR if the side has no basis yet, the projection and the
            two norms.  Returns (S_hat, [omega_first?, lhs, ref] tensors)."""
            dv = self.dv[self._nid[id(node)]]
            S = (dv.Sr if side == "row" else dv.Sc).view()
            q_attr = "Qr" if side == "row" else "Qc"
            Q = getattr(dv, q_attr)
            first = None
            if Q is None:
                # economic QR of a wide block (rows < d): the reflectors, Q and
                # R's leading diagonal come from the first `rows` columns alone
                # (the rest of R is never read), so factor only those
                Q, om = _qr(S[:, :min(self.d, S.shape[0])])
                setattr(dv, q_attr, Q)
                diag = torch.diagonal(om)
                first = diag[:1].abs() if diag.numel() else torch.zeros(1, dtype=torch.float64,
                                                                        device=S.device)
            window = S[:, self.d:]
            S_hat = _project_out(Q, window)
            norms = torch.stack([torch.linalg.norm(S_hat), torch.linalg.norm(window)])
            return S_hat, first, norms

        def _gate_both(self, node, eps_rel: float, eps_abs: float):
            """Both sides' gates of a node (the reference evaluates row then
            column, :341-342, always both): the column side's device work runs
            on the side stream, and the scalars of both sides cross to the host
            together -- two host syncs per node instead of up to six."""
            cur = torch.cuda.current_stream()
            side = _side_stream()
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                hat_c, first_c, norms_c = self._gate_stage1(node, "col")
            hat_r, first_r, norms_r = self._gate_stage1(node, "row")
            cur.wait_stream(side)
            dv = self.dv[self._nid[id(node)]]
            for t in (hat_c, first_c, norms_c, dv.Qc):   # made on the side stream, used here
                if t is not None:
                    t.record_stream(cur)
            parts = [norms_r, norms_c] + [f for f in (first_r, first_c) if f is not None]
            vals = torch.cat(parts).tolist()
            (lhs_r, ref_r, lhs_c, ref_c), rest = vals[:4], vals[4:]
            if first_r is not None:
                node.omega_first_row = rest.pop(0)
            if first_c is not None:
                node.omega_first_col = rest.pop(0)
            out = {}
            pending = []
            for sname, hat, lhs, ref, q_attr, w_attr in (
                    ("row", hat_r, lhs_r, ref_r, "Qr", "omega_first_row"),
                    ("col", hat_c, lhs_c, ref_c, "Qc", "omega_first_col")):
                # hss_compress.frobenius_stop (:106-117) on the two norms
                if lhs < eps_abs or ref == 0.0 or lhs < eps_rel * ref:
                    out[sname] = True
                    continue
                qi, omi = _qr(hat)
                setattr(dv, q_attr, torch.cat([getattr(dv, q_attr), qi], dim=1))
                pending.append((sname, torch.diagonal(omi), w_attr))
            if pending:
                diags = torch.cat([d for _, d, _ in pending]).cpu().numpy()
                o = 0
                for sname, dg, w_attr in pending:
                    k = dg.numel()
                    out[sname] = hc.rank_deficiency_stop(diags[o:o + k], getattr(node, w_attr),
                                                         eps_rel, eps_abs)
                    o += k
            return out

        def _gate_side(self, node, side: str, eps_rel: float, eps_abs: float) -> bool:
            key = (id(node), self.d, eps_rel, eps_abs)
            if side == "row" or self._gate_cache is None or self._gate_cache[0] != key:
                self._gate_cache = (key, self._gate_both(node, eps_rel, eps_abs))
            return self._gate_cache[1][side]

        def compress_node(self, nid: int, eps_rel: float, eps_abs: float) -> None:
            tnode = self.tree.nodes[nid]
            node = self.nodes[nid]
            dv = self.dv[nid]
            (dv.U, node.J_row), (dv.V, node.J_col) = row_interpolative_decompositions(
                dv.Sr.view(), dv.Sc.view(), eps_rel, eps_abs)
            dv.Jr_t = dv.Jc_t = None
            if tnode.is_leaf:
                base = np.arange(tnode.lo, tnode.hi)
                node.Itilde_row = base[node.J_row]
                node.Itilde_col = base[node.J_col]
            else:
                c1 = self.nodes[tnode.left.nid]
                c2 = self.nodes[tnode.right.nid]
                rows = np.concatenate([c1.Itilde_row, c2.Itilde_row])
                cols = np.concatenate([c1.Itilde_col, c2.Itilde_col])
                node.Itilde_row = rows[node.J_row]
                node.Itilde_col = cols[node.J_col]
            rr, rc = self._reduced_window(nid, (0, self.width), None)
            dv.Rr, dv.Rc = ColBuf(rr), ColBuf(rc)
            node.state = NodeState.COMPRESSED
            dv.Qr = dv.Qc = None

        def finalize_root(self, nid: int) -> None:
            self._fetch_cross_blocks(nid)
            self.nodes[nid].state = NodeState.COMPRESSED

        # --------------------------------------------------------- result
        def run(self):
            H = super().run()
            for tnode in self.tree.nodes:
                node, dv = self.nodes[tnode.nid], self.dv[tnode.nid]
                for name in ("D", "B12", "B21"):
                    t = getattr(dv, name)
                    if t is not None:
                        setattr(node, name, t.cpu().numpy())
                if dv.U is not None:
                    node.U_coeff = dv.U.contiguous().cpu().numpy()
                    node.V_coeff = dv.V.contiguous().cpu().numpy()
            self.dv = None
            self._ds = None
            return H

    DeviceDriver.__name__ = DeviceDriver.__qualname__ = "DeviceDriver"
    return DeviceDriver


def compress(A, tree, opts, hss_compress=None):
    """hsskit.hss_compress.compress (:365-385) with the device driver: the
    reference's validation and single-cluster path, then DeviceDriver.run."""
    import importlib
    hc = hss_compress or importlib.import_module("hsskit.hss_compress")
    saved = hc._Driver
    hc._Driver = device_driver_class(hc, base=saved)
    try:
        return hc.compress(A, tree, opts)
    finally:
        hc._Driver = saved


__all__ = ["device_driver_class", "compress", "row_interpolative_decomposition",
           "row_interpolative_decompositions", "ColBuf"]
