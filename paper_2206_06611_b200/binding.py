"""Thin ctypes binding of include/brmerge.h (argument marshalling only).

Every step of the SpGEMM runs in libbrmerge.so's CUDA kernels; this module only
turns torch tensors into (pointer, size) arguments and allocates outputs with
torch's caching allocator. There is no CPU fallback: importing this module
without the built library, or calling it without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path

import torch

_LIB_PATH = Path(__file__).resolve().parent / "libbrmerge.so"

BRM_UPPER = 0
BRM_PRECISE = 1
BRM_NUM_BINS = 8
MODES = {"upper": BRM_UPPER, "precise": BRM_PRECISE, BRM_UPPER: BRM_UPPER, BRM_PRECISE: BRM_PRECISE}

STATUS = {0: "BRM_OK", 1: "BRM_ERR_INVALID", 2: "BRM_ERR_DIM", 3: "BRM_ERR_CUDA", 4: "BRM_ERR_OOM",
          5: "BRM_ERR_OVERFLOW", 6: "BRM_ERR_STATE"}


class BrmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class brm_csr_t(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("rpt", ctypes.c_void_p), ("col", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class brm_stats_t(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("nprod_total", ctypes.c_int64),
                ("nprod_max", ctypes.c_int64), ("nnz_c", ctypes.c_int64),
                ("bin_rows", ctypes.c_int64 * BRM_NUM_BINS),
                ("bin_nprod", ctypes.c_int64 * BRM_NUM_BINS),
                ("mode", ctypes.c_int32), ("timing_enabled", ctypes.c_int32),
                ("ms_nprod_scan", ctypes.c_float), ("ms_symbolic", ctypes.c_float),
                ("ms_numeric", ctypes.c_float), ("ms_rowsize_scan", ctypes.c_float),
                ("ms_compact", ctypes.c_float),
                ("ms_bin_numeric", ctypes.c_float * BRM_NUM_BINS),
                ("launches", ctypes.c_int64),
                ("ms_hv_plan", ctypes.c_float), ("ms_hv_merge", ctypes.c_float),
                ("hv_rows_one", ctypes.c_int64), ("hv_rows_multi", ctypes.c_int64)]

    def as_dict(self) -> dict:
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            d[name] = list(v) if isinstance(v, ctypes.Array) else v
        return d


_P = ctypes.c_void_p
_S = ctypes.c_int
# name -> argtypes (restype brm_status_t unless noted)
SIGNATURES = {
    "brm_create": [ctypes.POINTER(_P), ctypes.c_int, _P],
    "brm_destroy": [_P],
    "brm_set_stream": [_P, _P],
    "brm_set_timing": [_P, ctypes.c_int],
    "brm_set_heavy_route": [_P, ctypes.c_int],
    "brm_set_host_pipeline": [_P, ctypes.c_int64],
    "brm_set_mirrors": [_P, ctypes.c_int, ctypes.POINTER(_P), ctypes.POINTER(_P)],
    "brm_enable_peer_access": [_P, ctypes.c_int],
    "brm_last_error": [_P],
    "brm_status_string": [ctypes.c_int],
    "brm_get_stats": [_P, ctypes.POINTER(brm_stats_t)],
    "brmerge_spgemm": [_P, ctypes.POINTER(brm_csr_t), ctypes.POINTER(brm_csr_t), ctypes.c_int,
                       ctypes.POINTER(brm_csr_t)],
    "brm_csr_free": [_P, ctypes.POINTER(brm_csr_t)],
    "brmerge_spgemm_structure": [_P, ctypes.POINTER(brm_csr_t), ctypes.POINTER(brm_csr_t),
                                 ctypes.c_int, _P, ctypes.POINTER(ctypes.c_int64)],
    "brmerge_spgemm_fill": [_P, ctypes.POINTER(brm_csr_t)],
    "brmerge_spgemm_host": [_P, ctypes.POINTER(brm_csr_t), ctypes.POINTER(brm_csr_t), ctypes.c_int,
                            ctypes.POINTER(brm_csr_t)],
    "brm_row_nprod": [_P, ctypes.POINTER(brm_csr_t), ctypes.POINTER(brm_csr_t), _P],
    "brm_exclusive_scan_i64": [_P, _P, _P, ctypes.c_int64],
    "brm_partition_rows": [_P, _P, ctypes.c_int64, ctypes.c_int, _P],
}

_lib = None


def load_library() -> ctypes.CDLL:
    """Load libbrmerge.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(f"{_LIB_PATH} is missing: run __graft_entry__.build() "
                              "(python -m paper_2206_06611_b200._build); there is no CPU fallback")
        lib = ctypes.CDLL(str(_LIB_PATH))
        for name, args in SIGNATURES.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = ctypes.c_char_p if name in ("brm_last_error", "brm_status_string") else _S
        _lib = lib
    return _lib


@dataclass
class TorchCsr:
    """CSR held in torch tensors (rpt int64, col int32, val float64)."""
    rows: int
    cols: int
    rpt: torch.Tensor
    col: torch.Tensor
    val: torch.Tensor

    @property
    def nnz(self) -> int:
        return int(self.col.numel())

    @property
    def device(self) -> torch.device:
        return self.rpt.device

    @classmethod
    def from_csr(cls, X, device="cuda", pin: bool = False) -> "TorchCsr":
        """From an inputs.Csr (numpy) to tensors on `device` (or pinned host)."""
        def t(a):
            x = torch.from_numpy(a)
            if pin:
                return x.pin_memory()
            return x.to(device)
        return cls(int(X.rows), int(X.cols), t(X.rpt), t(X.col), t(X.val))

    def to(self, device) -> "TorchCsr":
        """The same CSR with its tensors on `device`."""
        return TorchCsr(self.rows, self.cols, self.rpt.to(device), self.col.to(device), self.val.to(device))

    def to_numpy(self):
        return (self.rpt.cpu().numpy(), self.col.cpu().numpy(), self.val.cpu().numpy())

    def c_struct(self) -> brm_csr_t:
        for name, x, dt in (("rpt", self.rpt, torch.int64), ("col", self.col, torch.int32),
                            ("val", self.val, torch.float64)):
            if x.dtype != dt or not x.is_contiguous():
                raise TypeError(f"{name} must be a contiguous {dt} tensor")
        return brm_csr_t(self.rows, self.cols, self.nnz, self.rpt.data_ptr(),
                         self.col.data_ptr() if self.nnz else 0,
                         self.val.data_ptr() if self.nnz else 0)


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class Context:
    """One brm_context_t: device workspace + plan, bound to torch's current stream."""

    def __init__(self, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("libbrmerge needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self._h = _P()
        self._check(self.lib.brm_create(ctypes.byref(self._h), self.device.index,
                                        _stream_ptr(self.device)))

    def _check(self, code: int):
        if code != 0:
            msg = self.lib.brm_last_error(self._h).decode() if self._h else ""
            raise BrmError(code, msg)

    def close(self):
        if self._h:
            self.lib.brm_destroy(self._h)
            self._h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _bind_stream(self):
        self._check(self.lib.brm_set_stream(self._h, _stream_ptr(self.device)))

    def set_timing(self, on: bool):
        self._check(self.lib.brm_set_timing(self._h, int(on)))

    HEAVY_AUTO, HEAVY_GLOBAL = 0, 1

    def brm_set_heavy_route(self, route: int):
        """Route of the heavy rows: HEAVY_AUTO (windowed BRMerge, levels of
        list blocks) or HEAVY_GLOBAL (all on the global-memory tier); include/brmerge.h."""
        self._check(self.lib.brm_set_heavy_route(self._h, int(route)))

    def brm_set_host_pipeline(self, min_products: int):
        """Host-buffer form: pipeline row blocks when A*B has >= min_products
        intermediate products (0: always; A of >= 65,536 rows); include/brmerge.h."""
        self._check(self.lib.brm_set_host_pipeline(self._h, int(min_products)))

    def brm_set_mirrors(self, col_ptrs=(), val_ptrs=()):
        """Peers' copies of C that brmerge_spgemm_fill also writes (device
        pointers as ints; empty: none); include/brmerge.h."""
        n = len(col_ptrs)
        if n != len(val_ptrs):
            raise ValueError("one value pointer per column pointer")
        cols = (_P * max(n, 1))(*[int(x) for x in col_ptrs])
        vals = (_P * max(n, 1))(*[int(x) for x in val_ptrs])
        self._check(self.lib.brm_set_mirrors(self._h, n, cols, vals))

    def brm_enable_peer_access(self, peer_device: int):
        self._check(self.lib.brm_enable_peer_access(self._h, int(peer_device)))

    def stats(self) -> dict:
        s = brm_stats_t()
        self._check(self.lib.brm_get_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    # --- brmerge_spgemm_structure / _fill ----------------------------------
    def brmerge_spgemm_structure(self, A: TorchCsr, B: TorchCsr, mode) -> tuple[torch.Tensor, int]:
        self._bind_stream()
        a, b = A.c_struct(), B.c_struct()
        self._A, self._B = (A, B, a, b), None  # keep alive until fill
        c_rpt = torch.empty(A.rows + 1, dtype=torch.int64, device=self.device)
        nnz = ctypes.c_int64()
        self._check(self.lib.brmerge_spgemm_structure(self._h, ctypes.byref(a), ctypes.byref(b),
                                                      MODES[mode], c_rpt.data_ptr(),
                                                      ctypes.byref(nnz)))
        return c_rpt, int(nnz.value)

    def brmerge_spgemm_fill(self, rows: int, cols: int, c_rpt: torch.Tensor, nnz: int,
                            col: torch.Tensor = None, val: torch.Tensor = None) -> TorchCsr:
        """col / val: caller-owned output arrays of nnz entries (e.g. this
        rank's slice of a whole-C array); allocated here when not given."""
        self._bind_stream()
        if col is None:
            col = torch.empty(max(nnz, 0), dtype=torch.int32, device=self.device)
            val = torch.empty(max(nnz, 0), dtype=torch.float64, device=self.device)
        elif (col.dtype != torch.int32 or val.dtype != torch.float64 or col.numel() != nnz
              or val.numel() != nnz or not col.is_contiguous() or not val.is_contiguous()):
            raise ValueError("col / val must be contiguous int32 / float64 arrays of nnz entries")
        C = TorchCsr(rows, cols, c_rpt, col, val)
        c = brm_csr_t(rows, cols, nnz, c_rpt.data_ptr(), col.data_ptr() if nnz else 0,
                      val.data_ptr() if nnz else 0)
        self._check(self.lib.brmerge_spgemm_fill(self._h, ctypes.byref(c)))
        return C

    def spgemm(self, A: TorchCsr, B: TorchCsr, mode="precise") -> TorchCsr:
        """C = A*B through structure + fill, outputs from torch's allocator."""
        c_rpt, nnz = self.brmerge_spgemm_structure(A, B, mode)
        return self.brmerge_spgemm_fill(A.rows, B.cols, c_rpt, nnz)

    # --- brmerge_spgemm (library-allocated C) -------------------------------
    def brmerge_spgemm(self, A: TorchCsr, B: TorchCsr, mode="precise") -> brm_csr_t:
        """The one-call C entry; returns the raw brm_csr_t (device arrays owned
        by the caller: release with brm_csr_free)."""
        self._bind_stream()
        a, b, c = A.c_struct(), B.c_struct(), brm_csr_t()
        self._check(self.lib.brmerge_spgemm(self._h, ctypes.byref(a), ctypes.byref(b), MODES[mode],
                                            ctypes.byref(c)))
        return c

    def brm_csr_free(self, c: brm_csr_t):
        self._check(self.lib.brm_csr_free(self._h, ctypes.byref(c)))

    # --- brmerge_spgemm_host (host buffers in, host buffers out) ------------
    def brmerge_spgemm_host(self, A: TorchCsr, B: TorchCsr, mode="precise"):
        """A, B on the host (pinned tensors). Returns (rpt, col, val) numpy
        views of the context's pinned output buffer (valid until next call)."""
        import numpy as np
        self._bind_stream()
        a, b, c = A.c_struct(), B.c_struct(), brm_csr_t()
        self._check(self.lib.brmerge_spgemm_host(self._h, ctypes.byref(a), ctypes.byref(b),
                                                 MODES[mode], ctypes.byref(c)))

        def view(ptr, n, ct, dt):
            if n == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ct)), shape=(n,))
        return (c.rows, c.cols, view(c.rpt, c.rows + 1, ctypes.c_int64, np.int64),
                view(c.col, c.nnz, ctypes.c_int32, np.int32),
                view(c.val, c.nnz, ctypes.c_double, np.float64))

    # --- stage entry points --------------------------------------------------
    def brm_row_nprod(self, A: TorchCsr, B: TorchCsr) -> torch.Tensor:
        self._bind_stream()
        out = torch.empty(A.rows, dtype=torch.int64, device=self.device)
        a, b = A.c_struct(), B.c_struct()
        self._check(self.lib.brm_row_nprod(self._h, ctypes.byref(a), ctypes.byref(b),
                                           out.data_ptr() if A.rows else None))
        return out

    def brm_exclusive_scan_i64(self, x: torch.Tensor) -> torch.Tensor:
        self._bind_stream()
        assert x.dtype == torch.int64 and x.is_contiguous()
        out = torch.empty(x.numel() + 1, dtype=torch.int64, device=self.device)
        self._check(self.lib.brm_exclusive_scan_i64(self._h, x.data_ptr() if x.numel() else None,
                                                    out.data_ptr(), x.numel()))
        return out

    def brm_partition_rows(self, nprod_off: torch.Tensor, p: int) -> torch.Tensor:
        self._bind_stream()
        out = torch.empty(p + 1, dtype=torch.int64, device=self.device)
        self._check(self.lib.brm_partition_rows(self._h, nprod_off.data_ptr(), nprod_off.numel() - 1,
                                                p, out.data_ptr()))
        return out
