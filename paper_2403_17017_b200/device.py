"""Device-resident CSR and the per-device scratch the C-ABI needs.

``DeviceCSR`` is the HBM layout every kernel reads:
row_offsets int32 (nnz < 2^31) or int64, col_indices int32, values fp32 / fp64,
each a separate 256-byte-aligned torch allocation (so 16-byte vector loads and the
1-D TMA bulk copies of CSR,TM are always legal).  torch only allocates; all compute
goes through libkpb200.so.

Prepared formats (ELL, COO row ids, merge-path partition, adaptive row blocks) are
cached on the matrix per kernel: the amortisation lever of PAPER.md:280.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

_I32_MAX = 2**31 - 1
_red_ws: dict = {}


def reduce_workspace(device=None, stream=None):
    """Zeroed K1/K2 scratch for (`device`, `stream`) -- the kernels leave it zeroed.  One
    per stream: K1's last-CTA ticket counter must never see two grids at once, and launches
    on different streams may overlap."""
    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
    key = (dev, _lib.stream_handle(stream, dev))
    ws = _red_ws.get(key)
    if ws is None:
        n = int(_lib.load().kp_reduce_workspace_bytes())
        ws = torch.zeros(n, dtype=torch.uint8, device=dev)
        _red_ws[key] = ws
    return ws


def _torch_dtype(dtype):
    import torch
    if dtype in (np.float32, "float32", "f32", torch.float32):
        return torch.float32
    if dtype in (np.float64, "float64", "f64", torch.float64):
        return torch.float64
    raise ValueError(f"unsupported value dtype {dtype!r} (fp32 or fp64)")


class DeviceCSR:
    """A CSR matrix resident in HBM.  Construct from torch CUDA tensors, or use
    ``DeviceCSR.from_host`` for a reference ``SparseMatrixCSR`` / numpy arrays."""

    def __init__(self, n_rows: int, n_cols: int, row_offsets, col_indices, values):
        torch = _lib.require_cuda()
        if row_offsets.dtype not in (torch.int32, torch.int64):
            raise ValueError("row_offsets must be int32 or int64")
        if col_indices.dtype != torch.int32:
            raise ValueError("col_indices must be int32 on the device")
        if values.dtype not in (torch.float32, torch.float64):
            raise ValueError("values must be fp32 or fp64")
        if not (row_offsets.is_cuda and col_indices.is_cuda and values.is_cuda):
            raise ValueError("DeviceCSR tensors must live on a CUDA device")
        if row_offsets.numel() != n_rows + 1:
            raise ValueError("row_offsets length must be n_rows + 1")
        if n_rows > _I32_MAX - 1 or n_cols > _I32_MAX:
            raise ValueError("device layout supports < 2^31 rows / columns")
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        # the device layout is 256-byte aligned (vector loads, 1-D TMA); views into a
        # larger tensor (e.g. a row block) are copied once to an aligned allocation
        al = lambda t: t.contiguous() if t.contiguous().data_ptr() % 256 == 0 else t.contiguous().clone()  # noqa: E731
        self.row_offsets = al(row_offsets)
        self.col_indices = al(col_indices)
        self.values = al(values)
        self.nnz = int(col_indices.numel())
        if values.numel() != self.nnz:
            raise ValueError("values and col_indices lengths differ")
        if self.row_offsets.dtype == torch.int32 and self.nnz > _I32_MAX - 1:
            raise ValueError("int32 offsets need nnz < 2^31")
        self.device = self.row_offsets.device
        self.off_type = _lib.KP_I32 if self.row_offsets.dtype == torch.int32 else _lib.KP_I64
        self.val_type = _lib.KP_F32 if self.values.dtype == torch.float32 else _lib.KP_F64
        self._struct = _lib.kp_csr(self.n_rows, self.n_cols, self.nnz, self.off_type, self.val_type,
                                   self.row_offsets.data_ptr(), self.col_indices.data_ptr(),
                                   self.values.data_ptr())
        self._prepared: dict = {}

    # ------------------------------------------------------------------ constructors
    @classmethod
    def from_host(cls, m=None, *, n_rows=None, n_cols=None, row_offsets=None, col_indices=None,
                  values=None, dtype=np.float32, index: str = "auto", device=None, non_blocking=False):
        """Upload a reference-layout matrix (int64 / float64 host arrays).  Offsets are
        narrowed to int32 when nnz < 2^31 (index='auto'), columns always to int32,
        values to ``dtype``."""
        torch = _lib.require_cuda()
        if m is not None:
            n_rows, n_cols = m.n_rows, m.n_cols
            row_offsets, col_indices, values = m.row_offsets, m.col_indices, m.values
        off = np.asarray(row_offsets)
        nnz = int(off[-1]) if off.size else 0
        use32 = index == "int32" or (index == "auto" and nnz < _I32_MAX)
        off_np = np.ascontiguousarray(off, dtype=np.int32 if use32 else np.int64)
        col_np = np.ascontiguousarray(col_indices, dtype=np.int32)
        tdt = _torch_dtype(dtype)
        val_np = np.ascontiguousarray(values, dtype=np.float32 if tdt == torch.float32 else np.float64)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        t = lambda a: torch.from_numpy(a).to(dev, non_blocking=non_blocking)  # noqa: E731
        return cls(int(n_rows), int(n_cols), t(off_np), t(col_np), t(val_np))

    # ------------------------------------------------------------------ views
    @property
    def struct(self) -> _lib.kp_csr:
        return self._struct

    @property
    def dtype(self):
        return self.values.dtype

    def known(self):
        from .sparse import KnownFeatures
        return KnownFeatures(self.n_rows, self.n_cols, self.nnz)

    def to_host(self):
        """(row_offsets, col_indices, values) as numpy (test / oracle use)."""
        return (self.row_offsets.cpu().numpy(), self.col_indices.cpu().numpy(), self.values.cpu().numpy())

    def byte_model(self, kernel: int, ell_width: int | None = None) -> int:
        """Compulsory bytes of one SpMV: x counted once, y written once."""
        sv = self.values.element_size()
        so = self.row_offsets.element_size()
        R, C, Z = self.n_rows, self.n_cols, self.nnz
        if kernel == 6:   # COO,WM: row ids + cols + vals
            return Z * (4 + 4 + sv) + C * sv + R * sv
        if kernel == 7 and ell_width is not None:  # ELL,TM: padded slots
            return R * ell_width * (4 + sv) + C * sv + R * sv
        return Z * (4 + sv) + (R + 1) * so + C * sv + R * sv

    def __repr__(self):
        return (f"DeviceCSR({self.n_rows}x{self.n_cols}, nnz={self.nnz}, "
                f"off={self.row_offsets.dtype}, val={self.values.dtype}, {self.device})")


def csr_from_coo(n_rows: int, n_cols: int, rows, cols, vals, dtype=None, device=None) -> DeviceCSR:
    """``sparse.csr_from_coo`` (sparse.py:87-103) on the device (kp_csr_from_coo): stable
    (row, col) order, duplicates summed bit-identically to np.add.reduceat, offsets from
    the row counts.  ``rows`` / ``cols`` / ``vals``: numpy arrays or torch tensors (any
    device; host inputs are uploaded).  Returns a DeviceCSR in the device layout with fp64
    values (or ``dtype``).  Out-of-range coordinates raise ``ValueError`` like the
    reference's validation (sparse.py:54-71)."""
    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)

    def up(a, dt):
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        return t.to(device=dev, dtype=dt).contiguous().view(-1)

    r, c, v = up(rows, torch.int64), up(cols, torch.int64), up(vals, torch.float64)
    n = int(r.numel())
    if not (c.numel() == n and v.numel() == n):
        raise ValueError("rows, cols and vals must have the same length")
    if n_rows < 0 or n_cols < 0:
        raise ValueError("shape must be non-negative")
    L = _lib.load()
    nb = ctypes.c_size_t(0)
    _lib.check(L.kp_coo_workspace_bytes(n, int(n_rows), int(n_cols), ctypes.byref(nb)), "kp_coo_workspace_bytes")
    ws = torch.empty(max(int(nb.value), 256), dtype=torch.uint8, device=dev)
    off = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    val = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    out2 = torch.zeros(2, dtype=torch.int64, device=dev)
    _lib.check(L.kp_csr_from_coo(int(n_rows), int(n_cols), r.data_ptr(), c.data_ptr(), v.data_ptr(), n,
                                 off.data_ptr(), col.data_ptr(), val.data_ptr(), out2.data_ptr(), ws.data_ptr(),
                                 ws.numel(), _lib.stream_handle()), "kp_csr_from_coo")
    nnz, bad = (int(t) for t in out2.cpu())
    if bad:
        raise ValueError(f"{bad} coordinate(s) outside the {n_rows} x {n_cols} shape")
    del ws
    off_t = off.to(torch.int32) if nnz < _I32_MAX else off
    vv = val[:nnz] if dtype is None else val[:nnz].to(_torch_dtype(dtype))
    return DeviceCSR(n_rows, n_cols, off_t, col[:nnz], vv)


def as_device(m, dtype=None) -> DeviceCSR:
    """DeviceCSR passthrough, or upload a host SparseMatrixCSR."""
    if isinstance(m, DeviceCSR):
        return m
    return DeviceCSR.from_host(m, dtype=dtype or np.float32)


def ptr(t) -> int:
    return int(t.data_ptr())


def cptr(obj) -> ctypes.c_void_p:
    return ctypes.c_void_p(ptr(obj))


class HostPackedCSR:
    """A host-resident CSR in the compact transfer format (csrc/kp_pack.cu): int32 offsets,
    column indices bit-packed to ceil(log2(n_cols)) bits (kp_pack_cols, OpenMP), values,
    all in ONE pinned buffer at 256-byte aligned offsets, so a step moves it with one H2D.
    ``upload`` copies it into a device staging area and restores the int32 columns there
    (kp_unpack_cols); ``staging`` builds that area and the DeviceCSR viewing it.  The
    packing runs once per matrix (like the reference's construction-time validation,
    sparse.py:52-71); every step then pays only the compact bytes over PCIe."""

    def __init__(self, A: DeviceCSR, n_threads: int = 0):
        import ctypes
        torch = _lib.require_cuda()
        L = _lib.load()
        self.n_rows, self.n_cols, self.nnz = A.n_rows, A.n_cols, A.nnz
        self.off_dtype, self.val_dtype = A.row_offsets.dtype, A.values.dtype
        self.bits = int(L.kp_pack_bits(max(1, self.n_cols)))
        pk = int(L.kp_pack_cols_bytes(self.nnz, max(1, self.n_cols)))
        sizes = [A.row_offsets.numel() * A.row_offsets.element_size(), pk, self.nnz * A.values.element_size()]
        self.offsets, o = [], 0
        for nb in sizes:
            self.offsets.append(o)
            o += (nb + 255) // 256 * 256
        self.sizes, self.nbytes = sizes, o
        self.buf = torch.empty(o, dtype=torch.uint8, pin_memory=True)
        b = self.buf.numpy()
        b[self.offsets[0]:self.offsets[0] + sizes[0]] = A.row_offsets.cpu().numpy().view(np.uint8)
        b[self.offsets[2]:self.offsets[2] + sizes[2]] = A.values.cpu().numpy().view(np.uint8)
        cols = np.ascontiguousarray(A.col_indices.cpu().numpy())
        dst = self.buf.data_ptr() + self.offsets[1]
        _lib.check(L.kp_pack_cols(cols.ctypes.data_as(ctypes.c_void_p), self.nnz, max(1, self.n_cols),
                                  ctypes.c_void_p(dst), int(n_threads)), "kp_pack_cols")

    def staging(self, device):
        """(device buffer for the packed bytes, DeviceCSR viewing it with its own int32 column array)."""
        torch = _lib.require_cuda()
        d = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        off = d[self.offsets[0]:self.offsets[0] + self.sizes[0]].view(self.off_dtype)
        val = d[self.offsets[2]:self.offsets[2] + self.sizes[2]].view(self.val_dtype)
        cols = torch.empty(self.nnz, dtype=torch.int32, device=device)
        return d, DeviceCSR(self.n_rows, self.n_cols, off, cols, val)

    def upload(self, d_buf, B: DeviceCSR, copy_stream=None, stream=None):
        """H2D of the packed bytes on `copy_stream` (non-blocking), then the column unpack on
        `stream` after it (stream-ordered through an event)."""
        torch = _lib.require_cuda()
        cs = copy_stream or torch.cuda.current_stream(B.device)
        with torch.cuda.stream(cs):
            d_buf.copy_(self.buf, non_blocking=True)
        st = stream or torch.cuda.current_stream(B.device)
        if st is not cs:
            st.wait_stream(cs)
        self.unpack(d_buf, B, st)

    def unpack(self, d_buf, B: DeviceCSR, stream):
        _lib.check(_lib.load().kp_unpack_cols(d_buf.data_ptr() + self.offsets[1], self.nnz, max(1, self.n_cols),
                                              B.col_indices.data_ptr(), int(stream.cuda_stream)), "kp_unpack_cols")
