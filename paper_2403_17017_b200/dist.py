"""Row-sharded SpMV across GPUs: nnz-balanced partition, x replicated in a
rank-padded layout, y local, one in-place all-gather per iteration.

Partition (K14, ``kp_shard_partition``): cut p = lower_bound(row_offsets, p*nnz/P), so each
rank owns a contiguous row range with ~nnz/P entries.  Unequal row counts R_p would break
NCCL's equal-count all-gather, so columns are remapped ONCE at partition time into a
rank-padded x layout:

    col' = owner(col) * R_max + (col - cut[owner(col)])

x then has P*R_max slots; rank p writes its y into slots [p*R_max, p*R_max + R_p), and the
all-gather ``all_gather_into_tensor(x_pad, x_pad[p*R_max:(p+1)*R_max])`` is in place (send
buffer = own slice of the receive buffer): no copies, padding slots are never referenced.
Feature partials are exact integers, so global features (and hence the Seer selection) are
identical to the single-matrix pass.

The communicator is torch.distributed (NCCL over NVLink on GPUs, gloo on CPU for tests).
"""

from __future__ import annotations

import os

import numpy as np


def partition_cuts(row_offsets, parts: int) -> np.ndarray:
    """Host restatement of K14 (lower_bound of p*nnz/P), int64 cuts[0..parts]."""
    off = np.asarray(row_offsets, dtype=np.int64)
    n_rows = off.size - 1
    nnz = int(off[-1])
    targets = (np.arange(parts, dtype=object) * nnz // parts).astype(np.int64)
    cuts = np.searchsorted(off, targets, side="left").astype(np.int64)
    cuts = np.minimum(cuts, n_rows)
    return np.concatenate([cuts, [n_rows]])


def device_cuts(A, parts: int):
    """K14 on the device (DeviceCSR) -> int64 CUDA tensor of parts+1 cuts."""
    import torch
    from . import _lib
    _lib.require_cuda()
    out = torch.empty(parts + 1, dtype=torch.int64, device=A.device)
    _lib.check(_lib.load().kp_shard_partition(A.row_offsets.data_ptr(), A.off_type, A.n_rows, parts,
                                              out.data_ptr(), _lib.stream_handle()), "kp_shard_partition")
    return out


def remap_columns(cols, cuts, r_max: int):
    """col -> owner*R_max + (col - cuts[owner]); works on numpy arrays or torch tensors."""
    try:
        import torch
        if isinstance(cols, torch.Tensor):
            c = cols.to(torch.int64)
            cu = cuts.to(c.device)
            owner = torch.searchsorted(cu, c, right=True) - 1
            return (owner * r_max + (c - cu[owner])).to(torch.int32)
    except ImportError:
        pass
    c = np.asarray(cols, dtype=np.int64)
    cu = np.asarray(cuts, dtype=np.int64)
    owner = np.searchsorted(cu, c, side="right") - 1
    return (owner * r_max + (c - cu[owner])).astype(np.int32)


class ShardPlan:
    """This rank's slice of a square matrix in the rank-padded layout."""

    def __init__(self, rank: int, world: int, cuts, n_rows: int):
        self.rank, self.world = rank, world
        self.cuts = np.asarray(cuts, dtype=np.int64)
        self.r0, self.r1 = int(self.cuts[rank]), int(self.cuts[rank + 1])
        self.r_max = int(np.max(np.diff(self.cuts))) if world > 0 else 0
        self.n_rows = n_rows

    @property
    def local_rows(self) -> int:
        return self.r1 - self.r0

    def pad(self, x_full):
        """Full-length x -> rank-padded x (host or torch)."""
        import torch
        if isinstance(x_full, torch.Tensor):
            out = torch.zeros(self.world * self.r_max, dtype=x_full.dtype, device=x_full.device)
        else:
            out = np.zeros(self.world * self.r_max, dtype=np.asarray(x_full).dtype)
        for p in range(self.world):
            a, b = int(self.cuts[p]), int(self.cuts[p + 1])
            out[p * self.r_max: p * self.r_max + (b - a)] = x_full[a:b]
        return out

    def unpad(self, x_pad):
        parts = [x_pad[p * self.r_max: p * self.r_max + int(self.cuts[p + 1] - self.cuts[p])]
                 for p in range(self.world)]
        import torch
        return torch.cat(parts) if isinstance(x_pad, torch.Tensor) else np.concatenate(parts)


def local_csr(row_offsets, col_indices, values, plan: ShardPlan):
    """Rows [r0, r1) rebased, columns remapped into the padded layout (host arrays or tensors)."""
    off = row_offsets[plan.r0: plan.r1 + 1]
    s = off[0]
    loff = off - s
    e = off[-1]
    lc = remap_columns(col_indices[int(s): int(e)], plan.cuts if not hasattr(col_indices, "device")
                       else _as_tensor(plan.cuts, col_indices.device), plan.r_max)
    return loff, lc, values[int(s): int(e)]


def _as_tensor(a, device):
    import torch
    return torch.as_tensor(np.asarray(a), dtype=torch.int64, device=device)


def all_gather_slices(buf, plan: ShardPlan, group=None) -> None:
    """The per-iteration y exchange: every rank's R_max slice of the rank-padded buffer
    ``buf`` reaches every rank, in place.  NCCL: one in-place all_gather_into_tensor over
    NVLink (send buffer = own slice of the receive buffer).  gloo (CPU tensors, or ranks
    sharing GPUs for a control-flow check): through host staging."""
    import torch.distributed as tdist
    p = plan
    if p.world == 1:
        return
    if buf.is_cuda and tdist.get_backend(group) == "nccl":
        tdist.all_gather_into_tensor(buf, buf[p.rank * p.r_max:(p.rank + 1) * p.r_max], group=group)
        return
    host = buf.cpu() if buf.is_cuda else buf
    tdist.all_gather_into_tensor(host, host[p.rank * p.r_max:(p.rank + 1) * p.r_max].clone(), group=group)
    if buf.is_cuda:
        buf.copy_(host)


# ---------------------------------------------------------------------- vertex reordering
# A symmetric permutation P A P^T that numbers the vertices by descending column popularity
# (in-degree; ties by index), applied to the global matrix when it is distributed: the hot
# part of x becomes one contiguous, L2-resident prefix that every rank's gathers share.
# The iteration lives in the permuted index space (x' = P x); inputs are permuted and
# outputs un-permuted at the boundary (``newid``: old id -> new id).  Row lengths are only
# reordered, so the selection features -- and Seer's choice -- are unchanged, and each
# row's entries keep their order.  C5 at N = 1 (tools/probes/reorder_probe.py): unblocked
# CSR,WO 10.43 -> 4.13 ms per SpMV; the column-blocked shard 5.10 -> 4.20 ms, so a reordered
# shard is not blocked.
def degree_order(col_indices, n: int):
    """(order: new id -> old id, newid: old id -> new id), int64 tensors on the columns'
    device, by descending in-degree with index tie-break (deterministic on every rank)."""
    import torch
    deg = torch.bincount(col_indices.to(torch.int64), minlength=n)
    order = torch.argsort(-deg, stable=True)
    newid = torch.empty_like(order)
    newid[order] = torch.arange(n, device=order.device)
    return order, newid


def permute_symmetric(row_offsets, col_indices, values, order, newid):
    """P A P^T of a square CSR: row i of the result is row order[i] of A with its columns
    relabelled by newid (entry order within the row kept).  Returns (int64 offsets, int64
    columns, values) on the input's device."""
    import torch
    off = row_offsets.to(torch.int64)
    n = off.numel() - 1
    ln = (off[1:] - off[:-1])[order]
    out = torch.zeros(n + 1, dtype=torch.int64, device=off.device)
    if n:
        torch.cumsum(ln, 0, out=out[1:])
    z = int(out[-1])
    cols = torch.empty(z, dtype=torch.int64, device=off.device)
    vals = torch.empty(z, dtype=values.dtype, device=off.device)
    # gather the rows in chunks of whole rows (bounded temporaries at 10^9 entries)
    chunk_rows = max(1, int(n * min(1.0, (1 << 27) / max(z, 1))))
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        a, b = int(out[r0]), int(out[r1])
        if a == b:
            continue
        row_of = torch.repeat_interleave(torch.arange(r0, r1, device=off.device), ln[r0:r1], output_size=b - a)
        src = off[order[row_of]] + (torch.arange(a, b, device=off.device) - out[row_of])
        cols[a:b] = newid[col_indices[src].to(torch.int64)]
        vals[a:b] = values[src]
    return out, cols, vals


# ---------------------------------------------------------------------- column blocking
# A rank's SpMV gathers x over the WHOLE padded x (C5: 64M fp32 = 268 MB, twice the 126 MB
# L2): on R-MAT nearly every gather misses, and ncu counts 6.1x the algorithmic DRAM bytes
# (profiles/ncu_C5_blocked_r02.md).  Column blocking keeps each gather window closer to
# L2-resident: the block is split once, at shard time, into S column slices A_0..A_{S-1}
# (each a CSR over the same rows), and an iteration is y = A_0 x + ... + A_{S-1} x,
# accumulated slice by slice in the merge kernel's own row stores (kp_spmv_bcast_acc; the
# last slice's stores are the exchange).  R-MAT leaves most rows of a slice empty (C5: 60 %
# of all rows are empty, 21-32 % have entries in a given slice at S = 6-2), so slices are
# compressed-row blocks -- only their non-empty rows, scattered into the accumulator in
# place through a row map -- except the last one when there are several ranks (its
# full-row stores are the fused exchange).  Per-rank SpMV of C5 (shard_scaling, rank-
# emulated on one GPU; profiles/shard_scaling_r02.txt): P = 1 10.4 -> 5.16 ms at S = 3
# (5.14 at 4, 5.95 at 2); P = 8 1.31 -> 0.83 ms at S = 3 (0.85 at 4, 0.88 at 2).
COL_SLICE_L2_FRACTION = 0.75  # an x slice may be this fraction of the L2 (measured sweep)
MAX_COL_SLICES = 8


def auto_col_slices(x_bytes: int, l2_bytes: int) -> int:
    """Slices so that one x slice fits in COL_SLICE_L2_FRACTION of the L2 (1: no blocking)."""
    budget = max(1, int(COL_SLICE_L2_FRACTION * l2_bytes))
    return int(min(MAX_COL_SLICES, max(1, -(-int(x_bytes) // budget))))


def col_slice_bounds(n_cols: int, slices: int) -> list:
    """Equal-width column ranges [b_s, b_{s+1}) over the (padded) x."""
    if slices < 1:
        raise ValueError("slices must be >= 1")
    return [(int(n_cols) * s) // slices for s in range(slices + 1)]


def split_columns(row_offsets, col_indices, values, lo: int, hi: int):
    """The entries of a CSR with lo <= col < hi, as a CSR over the same rows (int64
    offsets; entry order within each row kept).  Torch tensors on any device."""
    import torch
    off = row_offsets.to(torch.int64)
    n_rows = off.numel() - 1
    keep = (col_indices >= lo) & (col_indices < hi)
    idx = torch.nonzero(keep).squeeze(1)
    del keep
    rows = torch.searchsorted(off, idx, right=True) - 1
    cnt = torch.bincount(rows, minlength=n_rows)
    del rows
    out = torch.zeros(n_rows + 1, dtype=torch.int64, device=off.device)
    if n_rows:
        torch.cumsum(cnt, 0, out=out[1:])
    return out, col_indices[idx], values[idx]


def compress_rows(row_offsets):
    """(offsets over the non-empty rows only, int32 row ids of those rows) of a CSR's
    offsets -- a compressed-row block: its merge pass skips the empty rows entirely."""
    import torch
    off = row_offsets.to(torch.int64)
    ln = off[1:] - off[:-1]
    keep = torch.nonzero(ln > 0).squeeze(1)
    out = torch.zeros(keep.numel() + 1, dtype=torch.int64, device=off.device)
    if keep.numel():
        torch.cumsum(ln[keep], 0, out=out[1:])
    return out, keep.to(torch.int32)


def column_blocks(A, slices: int, compact: bool = True, compact_last: bool = False):
    """DeviceCSR -> ``slices`` column blocks (same n_cols), one per column range, as a list
    of (DeviceCSR, row ids).  With ``compact`` every block but the last keeps only its
    non-empty rows (row ids: int32 tensor mapping them back; R-MAT C5: 21-32 % of the rows
    per block); the last block keeps every row (row ids None), so its stores cover the
    whole y -- they are the exchange -- unless ``compact_last`` (one rank: the blocks
    accumulate straight into the next x)."""
    import torch
    from .device import DeviceCSR
    out = []
    b = col_slice_bounds(A.n_cols, slices)
    for s in range(slices):
        o, c, v = split_columns(A.row_offsets, A.col_indices, A.values, b[s], b[s + 1])
        rid = None
        if compact and (s < slices - 1 or compact_last):
            o, rid = compress_rows(o)
        n = o.numel() - 1
        o = o.to(torch.int32) if int(o[-1]) < 2**31 - 1 else o
        out.append((DeviceCSR(n, A.n_cols, o, c, v), rid))
    return out


class Watchdog:
    """Failure detection for the NCCL path: ``kp_watchdog_*`` polls
    ncclCommGetAsyncError on this rank's communicator and a heartbeat the host sends every
    step; an NCCL error, or no heartbeat within ``timeout_s``, aborts the communicator
    (ncclCommAbort) so blocked collectives return, and the next ``heartbeat()`` raises."""

    def __init__(self, handle, timeout_s: float):
        self._h, self.timeout_s = handle, timeout_s

    @classmethod
    def start(cls, timeout_s: float = 300.0, poll_s: float = 0.05, group=None) -> "Watchdog | None":
        """Start on the NCCL communicator of ``group`` (default: WORLD); None when the
        process group is not NCCL or exposes no communicator."""
        import ctypes
        import torch
        import torch.distributed as tdist
        from . import _lib
        pg = group or tdist.group.WORLD
        if tdist.get_backend(pg) != "nccl":
            return None
        try:
            comm = int(pg._get_backend(torch.device("cuda"))._comm_ptr())
        except Exception:
            return None
        if not comm:
            return None
        h = ctypes.c_void_p()
        rc = _lib.load().kp_watchdog_start(comm, int(timeout_s * 1000), max(1, int(poll_s * 1000)), ctypes.byref(h))
        if rc != _lib.KP_OK:
            return None
        return cls(h, timeout_s)

    def status(self) -> tuple[int, int, str]:
        import ctypes
        from . import _lib
        r = ctypes.c_int32(0)
        msg = ctypes.create_string_buffer(256)
        st = _lib.load().kp_watchdog_status(self._h, ctypes.byref(r), msg, 256)
        return st, int(r.value), msg.value.decode()

    def heartbeat(self) -> None:
        from . import _lib
        if _lib.load().kp_watchdog_heartbeat(self._h) != _lib.KP_WD_OK:
            st, r, msg = self.status()
            raise RuntimeError(f"NCCL watchdog: {msg} (state {st}, ncclResult {r})")

    def stop(self) -> dict:
        from . import _lib
        st, r, msg = self.status()
        _lib.load().kp_watchdog_stop(self._h)
        self._h = None
        return {"state": ["ok", "nccl_error", "timeout"][st], "nccl_result": r, "msg": msg,
                "timeout_s": self.timeout_s}


# ---------------------------------------------------------------------- device path (GPU)
def shard_device(row_offsets, col_indices, values, n_cols: int, rank: int, world: int, dtype=None):
    """This rank's row block of a GLOBAL CSR held in device tensors (any int / float
    dtypes): nnz-balanced cut by K14 on the device, rows rebased, columns remapped into
    the rank-padded x layout, stored in the device layout (int32 offsets when the block's
    nnz < 2^31, int32 cols, fp32/fp64 values).  Returns (DeviceCSR, ShardPlan, cuts)."""
    import torch
    from . import _lib
    from .device import DeviceCSR
    _lib.require_cuda()
    n_rows = int(row_offsets.numel()) - 1
    off = row_offsets.contiguous()
    if off.dtype not in (torch.int32, torch.int64):
        off = off.to(torch.int64)
    cuts_d = torch.empty(world + 1, dtype=torch.int64, device=off.device)
    _lib.check(_lib.load().kp_shard_partition(off.data_ptr(), _lib.KP_I32 if off.dtype == torch.int32 else _lib.KP_I64,
                                              n_rows, world, cuts_d.data_ptr(), _lib.stream_handle()),
               "kp_shard_partition")
    cuts = cuts_d.cpu().numpy()
    plan = ShardPlan(rank, world, cuts, n_rows)
    s, e = int(off[plan.r0]), int(off[plan.r1])
    loff = (off[plan.r0: plan.r1 + 1].to(torch.int64) - s)
    loff = loff.to(torch.int32 if e - s < 2**31 - 1 else torch.int64)
    lc = remap_columns(col_indices[s:e], cuts_d, plan.r_max)
    dt = dtype or torch.float32
    lv = values[s:e].to(dt)
    A = DeviceCSR(plan.local_rows, world * plan.r_max, loff, lc.to(torch.int32), lv)
    return A, plan, cuts_d


def _length_partials(A):
    """(lo, hi, s1, s2) of this rank's row lengths on the device (K1); an empty block
    gives the neutral element of the combine (lo = INT64_MAX, hi = INT64_MIN)."""
    import torch
    from . import _lib
    from .device import reduce_workspace
    if A.n_rows == 0:
        return torch.tensor([2**63 - 1, -2**63, 0, 0], dtype=torch.int64, device=A.device)
    out = torch.empty(4, dtype=torch.int64, device=A.device)
    _lib.check(_lib.load().kp_length_stats(A.row_offsets.data_ptr(), A.off_type, A.n_rows + 1, out.data_ptr(),
                                           reduce_workspace(A.device).data_ptr(), _lib.stream_handle()),
               "kp_length_stats")
    return out


def select_sharded(model, A, world: int, n_rows: int, n_cols: int, nnz: int, k: int, group=None, out=None):
    """Row-sharded seer-core.infer: local K1 partials -> one 32-byte all-gather ->
    kp_seer_select_partials (exact combine + epilogue + trees) on every rank, so the
    outcome equals the single-matrix selection.  Returns the device outcome buffer."""
    import torch
    import torch.distributed as tdist
    from . import _lib
    part = _length_partials(A)
    if world > 1:
        if tdist.get_backend(group) == "nccl":
            parts = torch.empty(4 * world, dtype=torch.int64, device=A.device)
            tdist.all_gather_into_tensor(parts, part, group=group)
        else:  # gloo: host staging
            hp = torch.empty(4 * world, dtype=torch.int64)
            tdist.all_gather_into_tensor(hp, part.cpu(), group=group)
            parts = hp.to(A.device)
    else:
        parts = part
    sel, kn, ga = model.device_trees(A.device)
    if out is None:
        out = torch.empty(_lib.OUTCOME_BYTES, dtype=torch.uint8, device=A.device)
    _lib.check(_lib.load().kp_seer_select_partials(parts.data_ptr(), world, n_rows, n_cols, nnz, int(k),
                                                   sel.data_ptr(), kn.data_ptr(), ga.data_ptr(), out.data_ptr(),
                                                   _lib.stream_handle()), "kp_seer_select_partials")
    return out


class ShardedSeer:
    """Row-sharded Seer + iterative SpMV (power iteration x <- A x) on this rank's block.

    Setup: global selection from the ranks' partials (device), the chosen kernel's
    preprocessing of the local block.  ``step(x_full_pad)``: the chosen kernel's
    preprocessing (charged every step) + k x (local SpMV into this rank's
    slice of the next x, in-place NCCL all-gather of the slices over NVLink)."""

    def __init__(self, model, A, plan: ShardPlan, k: int, n_rows: int, n_cols: int, nnz: int, group=None,
                 exchange: str = "auto", kernel=None, col_slices="auto", compact_blocks: bool = True):
        import torch
        from . import kernels
        from .features import decode_outcome
        self.A, self.plan, self.k, self.group = A, plan, int(k), group
        if kernel is None:  # Seer selection over the whole (sharded) matrix
            self.outcome = decode_outcome(select_sharded(model, A, plan.world, n_rows, n_cols, nnz, k, group))
            self.kernel = int(self.outcome.kernel)
        else:  # a fixed kernel (the sweep's baselines)
            self.outcome = None
            self.kernel = kernels.kernel_index(kernel)
        dt = A.values.dtype
        self._kernels = kernels
        # exchange: "fused" = the SpMV epilogue stores y into every rank's next-x buffer over
        # NVLink peer mappings of a symmetric allocation (kp_spmv_bcast) + a device-side
        # barrier; "nccl" = local SpMV then an in-place all-gather; "host" = the all-gather
        # through host staging (gloo: ranks sharing a GPU).  "auto" = fused when the chosen
        # kernel supports it and symmetric memory rendezvous works.
        if exchange not in ("auto", "fused", "nccl", "host"):
            raise ValueError(f"unknown exchange {exchange!r}")
        self.exchange = "host" if exchange == "host" else "nccl"
        if exchange in ("auto", "fused") and self.kernel in (kernels.CSR_MP, kernels.CSR_WO):
            try:
                self._setup_fused(dt)
                self.exchange = "fused"
            except Exception as exc:  # no peer mappings / symm-mem backend: keep NCCL
                if exchange == "fused":
                    raise
                self.fused_error = repr(exc)
        if self.exchange in ("nccl", "host"):
            self.bufs = [torch.zeros(plan.world * plan.r_max, dtype=dt, device=A.device) for _ in range(2)]
        # column blocking (merge-path kernels: the accumulating store is theirs); "auto" =
        # env KP_COL_SLICES if set, else when the padded x exceeds the L2 budget
        S = os.environ.get("KP_COL_SLICES", "auto") if col_slices == "auto" else col_slices
        if S == "auto":
            l2 = int(getattr(torch.cuda.get_device_properties(A.device), "L2_cache_size", 0) or 126 << 20)
            S = auto_col_slices(plan.world * plan.r_max * A.values.element_size(), l2)
        S = int(S)
        if S < 1:
            raise ValueError("col_slices must be >= 1")
        self.col_slices = S if self.kernel in (kernels.CSR_MP, kernels.CSR_WO) and A.nnz > 0 else 1
        # one rank: every block compressed, accumulating straight into the next x; several
        # ranks: the last block keeps all rows so that its stores are the fused exchange
        # (no separate broadcast pass)
        cb = (column_blocks(A, self.col_slices, compact=compact_blocks,
                            compact_last=compact_blocks and plan.world == 1)
              if self.col_slices > 1 else [(A, None)])
        self.blocks = [B for B, _ in cb]
        self.block_rows = [r for _, r in cb]
        self.acc = torch.empty(max(1, plan.local_rows), dtype=dt, device=A.device) if self.col_slices > 1 else None

    def _setup_fused(self, dt):
        import torch
        import torch.distributed as tdist
        import torch.distributed._symmetric_memory as symm
        if not tdist.is_initialized():
            raise RuntimeError("fused exchange needs an initialised process group")
        p = self.plan
        grp = self.group or tdist.group.WORLD
        n = p.world * p.r_max
        self.bufs = [symm.empty(n, dtype=dt, device=self.A.device) for _ in range(2)]
        for b in self.bufs:
            b.zero_()
        self.hdl = [symm.rendezvous(b, grp.group_name) for b in self.bufs]
        # dests[i][q] = this rank's slice inside rank q's buffer i (peer-mapped)
        self.dests = [[h.get_buffer(q, (n,), dt)[p.rank * p.r_max: p.rank * p.r_max + p.local_rows]
                       for q in range(p.world)] for h in self.hdl]
        self.hdl[0].barrier(channel=0)

    def prepare(self):
        """The chosen kernel's preprocessing of every column block (None: needs none)."""
        K = self._kernels
        return [K.prepare(B, self.kernel, cache=False) if self.kernel in K.NEEDS_PREP else None for B in self.blocks]

    def spmv_into(self, x, dests, self_index: int, Ps) -> None:
        """This rank's y = A x stored into ``dests`` (``dests[self_index]`` the local copy).
        Column-blocked: the blocks accumulate into self.acc (compressed-row blocks scatter
        their non-empty rows into it in place), then either the last full-row block's stores
        (acc + its part) go to the destinations, or -- one rank, every block compressed --
        the single destination is the accumulator.  Unblocked non-merge kernels: kp_spmv."""
        K = self._kernels
        if len(self.blocks) == 1 and self.kernel not in (K.CSR_MP, K.CSR_WO):
            K.spmv(self.A, x, self.kernel, y=dests[self_index], prepared=Ps[0])
            for i, d in enumerate(dests):
                if i != self_index:
                    d.copy_(dests[self_index])
            return
        last_compact = self.block_rows[-1] is not None
        n = self.plan.local_rows
        # one destination and every block compressed: accumulate straight into it
        acc = dests[0][:max(1, n)] if last_compact and len(dests) == 1 else self.acc
        if self.block_rows[0] is not None:  # compressed-row blocks add into a zeroed accumulator
            acc.zero_()
        upto = len(self.blocks) if last_compact else len(self.blocks) - 1
        for s_, (B, Pb, rid) in enumerate(zip(self.blocks[:upto], Ps[:upto], self.block_rows[:upto])):
            if B.n_rows == 0:
                continue
            if rid is not None:  # only this block's non-empty rows, scattered in place
                K.spmv_bcast(B, x, self.kernel, [acc], 0, prepared=Pb, acc=acc, rows=rid)
            elif s_ == 0:  # the first block has nothing to add: the plain kernel (kp_spmv)
                K.spmv(B, x, self.kernel, y=acc, prepared=Pb)
            else:
                K.spmv_bcast(B, x, self.kernel, [acc], 0, prepared=Pb, acc=acc)
        if last_compact:  # every block accumulated: y is the accumulator
            for d in dests:
                if d.data_ptr() != acc.data_ptr():
                    d[:n].copy_(acc[:n])
            return
        K.spmv_bcast(self.blocks[-1], x, self.kernel, dests, self_index, prepared=Ps[-1],
                     acc=self.acc if len(self.blocks) > 1 else None)

    def _slice(self, buf):
        p = self.plan
        return buf[p.rank * p.r_max: p.rank * p.r_max + p.local_rows]

    def step(self, x_pad=None, iters: int | None = None):
        """One timed unit: prep + k iterations (``iters`` overrides k); returns the final
        padded x buffer."""
        K = self._kernels
        p = self.plan
        k = self.k if iters is None else int(iters)
        if x_pad is not None:
            self.bufs[0].copy_(x_pad)
        Ps = self.prepare()
        cur = 0
        spmv_into = lambda x, dests, i: self.spmv_into(x, dests, i, Ps)  # noqa: E731
        if self.exchange == "fused":
            if x_pad is not None:
                self.hdl[0].barrier(channel=0)  # every rank's buffer 0 holds x before anyone reads
            for _ in range(k):
                nxt = 1 - cur
                # y -> every rank's next-x slice from the kernel epilogue; the barrier orders
                # all ranks' stores before the next iteration's reads (and frees buffer cur)
                spmv_into(self.bufs[cur], self.dests[nxt], p.rank)
                self.hdl[nxt].barrier(channel=0)
                cur = nxt
            return self.bufs[cur]
        for _ in range(k):
            nxt = 1 - cur
            if len(self.blocks) > 1:
                spmv_into(self.bufs[cur], [self._slice(self.bufs[nxt])], 0)
            else:  # unblocked: plain kp_spmv (every kernel)
                K.spmv(self.A, self.bufs[cur], self.kernel, y=self._slice(self.bufs[nxt]), prepared=Ps[0])
            all_gather_slices(self.bufs[nxt], p, self.group)
            cur = nxt
        return self.bufs[cur]
