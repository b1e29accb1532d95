"""Host-side mirror of the reference's algorithm API over the B200 C-ABI.

The reference's entry points (qb.hpp is missing from the snapshot; signatures in
/root/reference/SPEC.md:273-308) and the types they use are mirrored here with the
same names, argument meaning and error behaviour:

    rand_qb_ei(A, stop, b, P, rng)
    rand_qb_fp(A, eps, b, P, l_budget, rng)
    rand_qb_fp_fixed_rank(A, k, s, b, reorth, rng)
    single_pass_fp(A, l, b, rng)
    MatrixHandle / StopRule / RngStream / QBFactorization / validate_epsilon / gaussian
    DimensionError, SingularityError, ToleranceFloorError, FormatError, ResourceError
                                                    /root/reference/proj/include/qbfac/types.hpp:16-66

Every call goes through ``libqbfac_gpu.so`` (include/qbfac_gpu.h); there is no CPU
fallback — importing works anywhere, but any compute call raises if the CUDA
library or a B200 is missing. numpy arrays are the host containers (column-major
``DenseMatrix`` semantics, dense_matrix.hpp:11-26).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QBFAC_LIB") or os.path.join(HERE, "libqbfac_gpu.so")  # QBFAC_LIB: dev builds

# ---- errors (types.hpp:16-66) --------------------------------------------------------


class Error(RuntimeError):
    pass


class DimensionError(Error):
    pass


class SingularityError(Error):
    def __init__(self, msg, diag_index=0):
        super().__init__(msg)
        self.diag_index = diag_index


class ToleranceFloorError(Error):
    def __init__(self, msg, floor=0.0):
        super().__init__(msg)
        self.floor = floor

    def floor_value(self):
        return self.floor


class IoError(Error):
    pass


class FormatError(IoError):
    pass


class ResourceError(Error):
    pass


TERMINATION = {0: "rank_reached", 1: "tolerance_met", 2: "sketch_exhausted", 3: "rank_collapse"}
K_EPS_MACH = 1.1102230246251565e-16  # types.hpp:14


class Params(C.Structure):
    _fields_ = [("alg", C.c_int32), ("mode", C.c_int32), ("b", C.c_int64), ("power", C.c_int64),
                ("k", C.c_int64), ("s", C.c_int64), ("max_rank", C.c_int64), ("l_budget", C.c_int64),
                ("max_restarts", C.c_int64), ("eps_abs", C.c_double), ("seed", C.c_uint64),
                ("stream", C.c_uint64), ("reorth", C.c_int32), ("flags", C.c_int32)]


class Info(C.Structure):
    _fields_ = [("rank", C.c_int64), ("error_indicator", C.c_double), ("norm_a_sq", C.c_double),
                ("passes", C.c_int64), ("terminated_by", C.c_int32), ("status", C.c_int32),
                ("diag_index", C.c_int64), ("floor", C.c_double), ("m", C.c_int64), ("n", C.c_int64),
                ("blocks", C.c_int64), ("gaussians_used", C.c_int64), ("restarts", C.c_int64),
                ("householder_fallbacks", C.c_int64), ("device_ms", C.c_double)]


_lib = None


def library_path() -> str:
    return LIB_PATH


def lib():
    """Load libqbfac_gpu.so (fails loudly when it is missing: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; run __graft_entry__.build() "
                              "(make -C paper_1606_09402_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        P, I64, U64, D, I = C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int
        PP = C.POINTER(C.c_void_p)
        L.qbfac_gpu_create.argtypes = [I, PP]
        L.qbfac_gpu_create_dist.argtypes = [I, I, I, P, PP]
        L.qbfac_gpu_nccl_unique_id.argtypes = [P]
        L.qbfac_gpu_destroy.argtypes = [P]
        L.qbfac_gpu_last_error.argtypes = [P]
        L.qbfac_gpu_last_error.restype = C.c_char_p
        L.qbfac_gpu_synchronize.argtypes = [P]
        L.qbfac_gpu_stream.argtypes = [P]
        L.qbfac_gpu_stream.restype = P
        L.qbfac_gpu_kernel_launches.argtypes = [P]
        L.qbfac_gpu_kernel_launches.restype = I64
        L.qbfac_gpu_matrix_dense.argtypes = [P, I64, I64, P, I64, PP]
        L.qbfac_gpu_matrix_dense_device.argtypes = [P, I64, I64, P, I64, PP]
        L.qbfac_gpu_matrix_dense_async.argtypes = [P, I64, I64, P, I64, I64, PP]
        L.qbfac_gpu_matrix_dense_stream.argtypes = [P, I64, I64, P, I64, I64, PP]
        L.qbfac_gpu_matrix_dense_shard.argtypes = [P, I64, I64, I64, I64, P, I64, PP]
        L.qbfac_gpu_matrix_csr.argtypes = [P, I64, I64, I64, P, P, P, PP]
        L.qbfac_gpu_matrix_csr_shard.argtypes = [P, I64, I64, I64, I64, I64, P, P, P, PP]
        L.qbfac_gpu_matrix_csr_stream.argtypes = [P, I64, I64, I64, P, P, P, I64, PP]
        L.qbfac_gpu_matrix_free.argtypes = [P]
        L.qbfac_gpu_matrix_passes.argtypes = [P]
        L.qbfac_gpu_matrix_passes.restype = I64
        L.qbfac_gpu_frob_norm_sq.argtypes = [P, P, P]
        L.qbfac_gpu_multiply.argtypes = [P, P, P, I64, I, P]
        L.qbfac_gpu_multiply_device.argtypes = [P, P, P, I64, I64, I, P, I64]
        L.qbfac_gpu_gaussian.argtypes = [P, U64, U64, U64, I64, I64, P]
        L.qbfac_gpu_gaussian_device.argtypes = [P, U64, U64, U64, I64, I64, P, I64]
        L.qbfac_gpu_run.argtypes = [P, P, P, PP, P]
        L.qbfac_gpu_result_copy_q.argtypes = [P, P, I64]
        L.qbfac_gpu_result_copy_b.argtypes = [P, P, I64]
        L.qbfac_gpu_result_copy_trace.argtypes = [P, P, I64]
        L.qbfac_gpu_result_copy_trace.restype = I64
        L.qbfac_gpu_result_free.argtypes = [P]
        L.qbfac_gpu_result_svd.argtypes = [P, I64, P, I64, P, P, I64, P]
        L.qbfac_gpu_validate_epsilon.argtypes = [D, D, D, P]
        L.qbfac_mtx_last_error.restype = C.c_char_p
        L.qbfac_mtx_info.argtypes = [C.c_char_p, P, P, P, P]
        L.qbfac_mtx_read_csr.argtypes = [C.c_char_p, P, P, P]
        L.qbfac_mtx_read_dense.argtypes = [C.c_char_p, P, I64]
        L.qbfac_mtx_write_csr.argtypes = [C.c_char_p, I64, I64, I64, P, P, P]
        L.qbfac_mtx_write_dense.argtypes = [C.c_char_p, I64, I64, P, I64]
        L.qbfac_gpu_matrix_mtx.argtypes = [P, C.c_char_p, PP]
        L.qbfac_gpu_matrix_shape.argtypes = [P, P, P, P, P]
        L.qbfac_gpu_matrix_export_csr.argtypes = [P, P, P, P, P]
        L.qbfac_gpu_matrix_export_dense.argtypes = [P, P, P, I64]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _raise(status: int, msg: str, info: Optional[Info] = None):
    if status == 0:
        return
    if status == 1:
        raise DimensionError(msg)
    if status == 2:
        raise SingularityError(msg, info.diag_index if info else 0)
    if status == 3:
        raise ToleranceFloorError(msg, info.floor if info else 0.0)
    if status == 4:
        raise FormatError(msg)
    if status == 5:
        raise ResourceError(msg)
    raise Error(msg)


# ---- context ------------------------------------------------------------------------


class Context:
    """One CUDA device (and, with world > 1, one rank of an NCCL communicator)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None):
        L = lib()
        h = C.c_void_p()
        if world > 1 or nccl_id is not None:
            buf = C.create_string_buffer(bytes(nccl_id), 128)
            st = L.qbfac_gpu_create_dist(device, rank, world, C.cast(buf, C.c_void_p), C.byref(h))
        else:
            st = L.qbfac_gpu_create(device, C.byref(h))
        if st:
            _raise(st, L.qbfac_gpu_last_error(None).decode())
        self._h = h
        self.device, self.rank, self.world = device, rank, world

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        st = lib().qbfac_gpu_nccl_unique_id(C.cast(buf, C.c_void_p))
        if st:
            _raise(st, lib().qbfac_gpu_last_error(None).decode())
        return buf.raw

    @property
    def handle(self):
        return self._h

    def check(self, st: int, info: Optional[Info] = None):
        if st:
            _raise(st, lib().qbfac_gpu_last_error(self._h).decode(), info)

    def synchronize(self):
        self.check(lib().qbfac_gpu_synchronize(self._h))

    def stream(self) -> int:
        return lib().qbfac_gpu_stream(self._h)

    def kernel_launches(self) -> int:
        return lib().qbfac_gpu_kernel_launches(self._h)

    def close(self):
        if getattr(self, "_h", None):
            lib().qbfac_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("QBFAC_DEVICE", "0")))
    return _default_ctx


# ---- RngStream (rng.hpp:16-42) ----------------------------------------------------------


class RngStream:
    """RngStream(seed, stream): the generator state is the pair plus the number of
    next_gaussian() draws consumed so far (the device regenerates any position)."""

    def __init__(self, seed: int, stream: int = 0, consumed: int = 0):
        self.seed_ = int(seed)
        self.stream_ = int(stream)
        self.consumed = int(consumed)

    def seed(self) -> int:
        return self.seed_

    def stream_id(self) -> int:
        return self.stream_

    def substream(self, id_: int) -> "RngStream":  # rng.cpp:68-70
        return RngStream(self.seed_, self.stream_ + 1 + int(id_))


def gaussian(rows: int, cols: int, rng: RngStream, ctx: Optional[Context] = None) -> np.ndarray:
    """gaussian(rows, cols, rng) (rng.cpp:72-79) generated on the device."""
    ctx = ctx or default_context()
    if rows < 1 or cols < 1:
        raise DimensionError("gaussian: dimensions must be at least 1")
    out = np.empty((rows, cols), order="F")
    ctx.check(lib().qbfac_gpu_gaussian(ctx.handle, rng.seed_, rng.stream_, rng.consumed, rows, cols, _p(out)))
    rng.consumed += rows * cols
    return out


# ---- StopRule / QBFactorization -------------------------------------------


@dataclass
class StopRule:
    mode: str = "fixed_precision"
    k: int = 0
    s: int = 0
    eps: float = 0.0

    @staticmethod
    def fixed_rank(k: int, s: int = 0) -> "StopRule":
        return StopRule("fixed_rank", int(k), int(s), 0.0)

    @staticmethod
    def fixed_precision(eps: float) -> "StopRule":
        return StopRule("fixed_precision", 0, 0, float(eps))


@dataclass
class QBFactorization:
    Q: np.ndarray
    B: np.ndarray
    error_indicator: float
    passes: int
    terminated_by: str
    norm_a_sq: float = 0.0
    e_trace: np.ndarray = field(default_factory=lambda: np.zeros(0))
    info: Optional[dict] = None

    @property
    def rank(self) -> int:
        return self.Q.shape[1]


# ---- MatrixHandle (matrix_handle.hpp:41-86) ------------------------------------------------


def _mtx_check(st: int):
    _raise(st, lib().qbfac_mtx_last_error().decode())


def read_matrix_market(path: str):
    """Host read of a Matrix Market file: returns ("csr", m, n, row_ptr,
    col_idx, values) built like SparseCsrMatrix::from_triplets, or ("dense", a) column-major."""
    coord, m, n, nnz = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
    bp = os.fsencode(path)
    _mtx_check(lib().qbfac_mtx_info(bp, C.byref(coord), C.byref(m), C.byref(n), C.byref(nnz)))
    if coord.value:
        rp = np.zeros(m.value + 1, dtype=np.int64)
        ci = np.zeros(max(nnz.value, 1), dtype=np.int32)
        v = np.zeros(max(nnz.value, 1), dtype=np.float64)
        _mtx_check(lib().qbfac_mtx_read_csr(bp, _p(rp), _p(ci), _p(v)))
        return "csr", m.value, n.value, rp, ci[:nnz.value], v[:nnz.value]
    a = np.zeros((m.value, n.value), dtype=np.float64, order="F")
    _mtx_check(lib().qbfac_mtx_read_dense(bp, _p(a), max(m.value, 1)))
    return "dense", a


def write_matrix_market(path: str, a=None, csr=None):
    """write_matrix_market: `a` dense (array format) or `csr` = (m, n,
    row_ptr, col_idx, values) (coordinate format); shortest round-trip decimals."""
    bp = os.fsencode(path)
    if csr is not None:
        m, n, rp, ci, v = csr
        rp = np.ascontiguousarray(rp, dtype=np.int64)
        ci = np.ascontiguousarray(ci, dtype=np.int32)
        v = np.ascontiguousarray(v, dtype=np.float64)
        _mtx_check(lib().qbfac_mtx_write_csr(bp, m, n, len(v), _p(rp), _p(ci), _p(v)))
    else:
        a = np.asfortranarray(a, dtype=np.float64)
        _mtx_check(lib().qbfac_mtx_write_dense(bp, a.shape[0], a.shape[1], _p(a), max(a.shape[0], 1)))


class MatrixHandle:
    """A resident on the device (dense column-major or CSR + device-built transposed CSR)."""

    def __init__(self, h, ctx: Context, m: int, n: int, sparse: bool):
        self._h, self.ctx, self.m, self.n, self.sparse = h, ctx, m, n, sparse

    @staticmethod
    def dense(a: np.ndarray, ctx: Optional[Context] = None) -> "MatrixHandle":
        ctx = ctx or default_context()
        a = np.asfortranarray(a, dtype=np.float64)
        m, n = a.shape
        h = C.c_void_p()
        ctx.check(lib().qbfac_gpu_matrix_dense(ctx.handle, m, n, _p(a), max(m, 1), C.byref(h)))
        return MatrixHandle(h, ctx, m, n, False)

    @staticmethod
    def dense_async(a: np.ndarray, ctx: Optional[Context] = None, chunk_rows: int = 0) -> "MatrixHandle":
        """Chunked asynchronous upload (H2D overlapped with the first pass of the next run).
        `a` must be column-major (Fortran-ordered, ideally pinned) and is kept alive by the handle."""
        ctx = ctx or default_context()
        if not (a.flags.f_contiguous and a.dtype == np.float64):
            a = np.asfortranarray(a, dtype=np.float64)
        m, n = a.shape
        h = C.c_void_p()
        ctx.check(lib().qbfac_gpu_matrix_dense_async(ctx.handle, m, n, _p(a), max(m, 1), chunk_rows, C.byref(h)))
        mh = MatrixHandle(h, ctx, m, n, False)
        mh._host_ref = a
        return mh

    @staticmethod
    def dense_stream(a: np.ndarray, ctx: Optional[Context] = None, chunk_rows: int = 0) -> "MatrixHandle":
        """Host-resident A read as a row stream by single_pass_fp only (matrix_handle.hpp:30-37);
        `a` column-major (ideally pinned), kept alive by the handle."""
        ctx = ctx or default_context()
        if not (a.flags.f_contiguous and a.dtype == np.float64):
            a = np.asfortranarray(a, dtype=np.float64)
        m, n = a.shape
        h = C.c_void_p()
        ctx.check(lib().qbfac_gpu_matrix_dense_stream(ctx.handle, m, n, _p(a), max(m, 1), chunk_rows, C.byref(h)))
        mh = MatrixHandle(h, ctx, m, n, False)
        mh._host_ref = a
        return mh

    @staticmethod
    def dense_device(ptr: int, m: int, n: int, lda: int, ctx: Optional[Context] = None) -> "MatrixHandle":
        """A already in device memory (column-major, leading dimension lda); copied."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        ctx.check(lib().qbfac_gpu_matrix_dense_device(ctx.handle, m, n, C.c_void_p(ptr), lda, C.byref(h)))
        return MatrixHandle(h, ctx, m, n, False)

    @staticmethod
    def dense_shard(a_local: np.ndarray, m_global: int, row0: int, ctx: Context) -> "MatrixHandle":
        a = np.asfortranarray(a_local, dtype=np.float64)
        m, n = a.shape
        h = C.c_void_p()
        ctx.check(lib().qbfac_gpu_matrix_dense_shard(ctx.handle, m_global, row0, m, n, _p(a), max(m, 1),
                                                     C.byref(h)))
        return MatrixHandle(h, ctx, m, n, False)

    @staticmethod
    def csr(m: int, n: int, row_ptr, col_idx, values, ctx: Optional[Context] = None) -> "MatrixHandle":
        ctx = ctx or default_context()
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        v = np.ascontiguousarray(values, dtype=np.float64)
        if len(rp) != m + 1 or len(ci) != len(v):
            raise FormatError("csr: inconsistent structure arrays")
        h = C.c_void_p()
        ctx.check(lib().qbfac_gpu_matrix_csr(ctx.handle, m, n, len(v), _p(rp), _p(ci), _p(v), C.byref(h)))
        return MatrixHandle(h, ctx, m, n, True)

    @staticmethod
    def csr_stream(m: int, n: int, row_ptr, col_idx, values, ctx: Optional[Context] = None,
                   chunk_nnz: int = 0) -> "MatrixHandle":
        """CsrRowStream (matrix_handle.cpp:60-73): A stays in host memory; single_pass_fp
        uploads and validates row chunks of ~chunk_nnz entries one at a time."""
        ctx = ctx or default_context()
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        v = np.ascontiguousarray(values, dtype=np.float64)
        if len(rp) != m + 1 or len(ci) != len(v):
            raise FormatError("csr: inconsistent structure arrays")
        h = C.c_void_p()
        ctx.check(lib().qbfac_gpu_matrix_csr_stream(ctx.handle, m, n, len(v), _p(rp), _p(ci), _p(v), chunk_nnz,
                                                    C.byref(h)))
        mh = MatrixHandle(h, ctx, m, n, True)
        mh._host_ref = (rp, ci, v)
        return mh

    @staticmethod
    def csr_shard(m_global: int, row0: int, n: int, row_ptr, col_idx, values, ctx: Context) -> "MatrixHandle":
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        v = np.ascontiguousarray(values, dtype=np.float64)
        m = len(rp) - 1
        h = C.c_void_p()
        ctx.check(lib().qbfac_gpu_matrix_csr_shard(ctx.handle, m_global, row0, m, n, len(v), _p(rp), _p(ci),
                                                   _p(v), C.byref(h)))
        return MatrixHandle(h, ctx, m, n, True)

    @staticmethod
    def from_mtx(path: str, ctx: Optional[Context] = None) -> "MatrixHandle":
        """read_matrix_market(path) straight into device memory."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        ctx.check(lib().qbfac_gpu_matrix_mtx(ctx.handle, os.fsencode(path), C.byref(h)))
        sp, m, n, nnz = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
        lib().qbfac_gpu_matrix_shape(h, C.byref(sp), C.byref(m), C.byref(n), C.byref(nnz))
        return MatrixHandle(h, ctx, m.value, n.value, bool(sp.value))

    def export(self):
        """Device arrays back to the host: (row_ptr, col_idx, values) or the dense array."""
        sp, m, n, nnz = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
        lib().qbfac_gpu_matrix_shape(self._h, C.byref(sp), C.byref(m), C.byref(n), C.byref(nnz))
        if sp.value:
            rp = np.zeros(m.value + 1, dtype=np.int64)
            ci = np.zeros(max(nnz.value, 1), dtype=np.int32)
            v = np.zeros(max(nnz.value, 1), dtype=np.float64)
            self.ctx.check(lib().qbfac_gpu_matrix_export_csr(self.ctx.handle, self._h, _p(rp), _p(ci), _p(v)))
            return rp, ci[:nnz.value], v[:nnz.value]
        a = np.zeros((m.value, n.value), dtype=np.float64, order="F")
        self.ctx.check(lib().qbfac_gpu_matrix_export_dense(self.ctx.handle, self._h, _p(a), max(m.value, 1)))
        return a

    def rows(self):
        return self.m

    def cols(self):
        return self.n

    def is_sparse(self):
        return self.sparse

    def passes(self) -> int:
        return lib().qbfac_gpu_matrix_passes(self._h)

    def frob_norm_sq(self) -> float:
        out = np.zeros(1)
        self.ctx.check(lib().qbfac_gpu_frob_norm_sq(self.ctx.handle, self._h, _p(out)))
        return float(out[0])

    def multiply(self, x: np.ndarray, transpose_a: bool) -> np.ndarray:
        x = np.asfortranarray(x, dtype=np.float64)
        inner = self.m if transpose_a else self.n
        if x.shape[0] != inner:
            raise DimensionError("multiply: inner dimension mismatch")
        y = np.empty((self.n if transpose_a else self.m, x.shape[1]), order="F")
        self.ctx.check(lib().qbfac_gpu_multiply(self.ctx.handle, self._h, _p(x), x.shape[1], int(transpose_a),
                                                _p(y)))
        return y

    def multiply_device(self, x_ptr: int, ldx: int, w: int, transpose_a: bool, y_ptr: int, ldy: int):
        """Device-buffer product (row-major X, Y) on the context stream; one pass."""
        self.ctx.check(lib().qbfac_gpu_multiply_device(self.ctx.handle, self._h, C.c_void_p(x_ptr), ldx, w,
                                                       int(transpose_a), C.c_void_p(y_ptr), ldy))

    def free(self):
        # a handle whose context is already closed (e.g. finalised after it in a garbage cycle at
        # shutdown) is dropped, not freed: its device memory went with the context's device state
        if getattr(self, "_h", None):
            if getattr(self.ctx, "_h", None):
                lib().qbfac_gpu_matrix_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ---- algorithms ------------------------------------------------------------------------------


@dataclass
class TruncatedSvd:
    """U (m x k), S (k, non-increasing), V (n x k), A ~ U diag(S) V^T."""
    U: np.ndarray
    S: np.ndarray
    V: np.ndarray
    sweeps: int = 0


class DeviceResult:
    """Result resident on the device; Q/B are copied to the host on demand."""

    def svd(self, k: Optional[int] = None, u_out: Optional[np.ndarray] = None,
            v_out: Optional[np.ndarray] = None) -> TruncatedSvd:
        """qb_to_svd(f, k) on the device: orth(B^T), one-sided Jacobi of the
        r x r factor, U = Q U_r, V = Q_b W. `u_out` / `v_out`: caller buffers (e.g. pinned),
        column-major m x k / n x k."""
        k = self.rank if k is None else k
        m, n = int(self.info.m), int(self.info.n)
        u = np.zeros((m, k), order="F") if u_out is None else u_out
        sv = np.zeros(k)
        v = np.zeros((n, k), order="F") if v_out is None else v_out
        if u.shape != (m, k) or v.shape != (n, k) or not (u.flags.f_contiguous and v.flags.f_contiguous):
            raise DimensionError("svd: output buffers must be column-major m x k / n x k")
        sw = C.c_int(0)
        self.ctx.check(lib().qbfac_gpu_result_svd(self._h, k, _p(u), max(m, 1), _p(sv), _p(v), max(n, 1),
                                                  C.byref(sw)))
        return TruncatedSvd(u, sv, v, sw.value)

    def __init__(self, h, ctx: Context, info: Info):
        self._h, self.ctx, self.info = h, ctx, info

    @property
    def rank(self) -> int:
        return int(self.info.rank)

    def q(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Q (m x rank, column-major); `out`: caller buffer (e.g. pinned) with >= m*rank doubles."""
        m = int(self.info.m)
        q = np.empty((m, self.rank), order="F") if out is None else out.reshape(-1)[:m * self.rank].reshape(
            (m, self.rank), order="F")
        self.ctx.check(lib().qbfac_gpu_result_copy_q(self._h, _p(q), max(m, 1)))
        return q

    def b(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """B (rank x n, column-major); `out`: caller buffer with >= rank*n doubles."""
        n = int(self.info.n)
        b = np.empty((self.rank, n), order="F") if out is None else out.reshape(-1)[:self.rank * n].reshape(
            (self.rank, n), order="F")
        self.ctx.check(lib().qbfac_gpu_result_copy_b(self._h, _p(b), max(self.rank, 1)))
        return b

    def trace(self) -> np.ndarray:
        n = lib().qbfac_gpu_result_copy_trace(self._h, None, 0)
        out = np.empty(n)
        if n:
            lib().qbfac_gpu_result_copy_trace(self._h, _p(out), n)
        return out

    def free(self):
        if getattr(self, "_h", None):
            if getattr(self.ctx, "_h", None):
                lib().qbfac_gpu_result_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def info_dict(info: Info) -> dict:
    return {f: getattr(info, f) for f, _ in Info._fields_}


def run_device(a: MatrixHandle, *, alg: int, mode: int = 1, b: int = 10, power: int = 0, k: int = 0, s: int = 0,
               max_rank: int = 0, l_budget: int = 0, max_restarts: int = 8, eps_abs: float = 0.0,
               seed: int = 0, stream: int = 0, reorth: bool = True) -> DeviceResult:
    p = Params(alg, mode, b, power, k, s, max_rank, l_budget, max_restarts, eps_abs, seed, stream, int(reorth), 0)
    info = Info()
    h = C.c_void_p()
    st = lib().qbfac_gpu_run(a.ctx.handle, a._h, C.byref(p), C.byref(h), C.byref(info))
    a.ctx.check(st, info)
    return DeviceResult(h, a.ctx, info)


def _to_host(res: DeviceResult) -> QBFactorization:
    inf = res.info
    out = QBFactorization(res.q(), res.b(), float(inf.error_indicator), int(inf.passes),
                          TERMINATION[int(inf.terminated_by)], float(inf.norm_a_sq), res.trace(),
                          info_dict(inf))
    res.free()
    return out


def rand_qb_ei(A: MatrixHandle, stop: StopRule, b: int, P: int, rng: RngStream,
               max_rank: int = 0) -> QBFactorization:
    """Alg. 2 on the device."""
    if rng.consumed:
        raise Error("rand_qb_ei: the device path regenerates Omega from a fresh RngStream position 0")
    res = run_device(A, alg=0, mode=1 if stop.mode == "fixed_precision" else 0, b=b, power=P, k=stop.k,
                     s=stop.s, max_rank=max_rank, eps_abs=stop.eps, seed=rng.seed_, stream=rng.stream_)
    rng.consumed += int(res.info.gaussians_used)
    return _to_host(res)


def rand_qb(A: MatrixHandle, l: int, P: int, rng: RngStream) -> QBFactorization:
    """randQB (Fig. 1a): Q = orth of the power-iterated sketch, B = Q^T A,
    passes = 2 + 2P, E = -1 (no indicator)."""
    if rng.consumed:
        raise Error("rand_qb: the device path needs a fresh RngStream")
    res = run_device(A, alg=4, mode=0, b=l, power=P, k=l, s=0, seed=rng.seed_, stream=rng.stream_)
    rng.consumed += A.n * l
    return _to_host(res)


def rand_qb_b(A: MatrixHandle, stop: StopRule, b: int, rng: RngStream) -> QBFactorization:
    """randQB_b (Fig. 1b): explicit residual (dense A), 4 passes per block."""
    if rng.consumed:
        raise Error("rand_qb_b: the device path needs a fresh RngStream")
    res = run_device(A, alg=5, mode=1 if stop.mode == "fixed_precision" else 0, b=b, k=stop.k, s=stop.s,
                     eps_abs=stop.eps, seed=rng.seed_, stream=rng.stream_)
    rng.consumed += int(res.info.gaussians_used)
    return _to_host(res)


def adaptive_range_finder(A: MatrixHandle, tol_spectral: float, r: int, rng: RngStream,
                          max_rank: int = 0) -> QBFactorization:
    """Adaptive randomized range finder (Eq. 2.4): one vector at a time until the
    last r residual samples are below tol / (10 sqrt(2/pi)); B = Q^T A at the end."""
    if rng.consumed:
        raise Error("adaptive_range_finder: the device path needs a fresh RngStream")
    res = run_device(A, alg=6, b=r, max_rank=max_rank, eps_abs=tol_spectral, seed=rng.seed_, stream=rng.stream_)
    rng.consumed += int(res.info.gaussians_used)
    return _to_host(res)


def rand_qb_fp(A: MatrixHandle, eps: float, b: int, P: int, l_budget: int, rng: RngStream,
               max_rank: int = 0, max_restarts: int = 8) -> QBFactorization:
    """Alg. 4 on the device."""
    if rng.consumed:
        raise Error("rand_qb_fp: the device path regenerates Omega from a fresh RngStream position 0")
    res = run_device(A, alg=1, b=b, power=P, max_rank=max_rank, l_budget=l_budget, max_restarts=max_restarts,
                     eps_abs=eps, seed=rng.seed_, stream=rng.stream_)
    rng.consumed += int(res.info.gaussians_used)
    return _to_host(res)


def rand_qb_fp_fixed_rank(A: MatrixHandle, k: int, s: int, b: int, reorth: bool, rng: RngStream) -> QBFactorization:
    """Alg. 3, optionally with steps 9a-9c."""
    if rng.consumed:
        raise Error("rand_qb_fp_fixed_rank: the device path needs a fresh RngStream")
    res = run_device(A, alg=2, mode=0, b=b, k=k, s=s, seed=rng.seed_, stream=rng.stream_, reorth=reorth)
    rng.consumed += int(res.info.gaussians_used)
    return _to_host(res)


def single_pass_fp(A: MatrixHandle, l: int, b: int, rng: RngStream) -> QBFactorization:
    """Remark 4.2, with A resident in HBM."""
    if rng.consumed:
        raise Error("single_pass_fp: the device path needs a fresh RngStream")
    res = run_device(A, alg=3, mode=0, b=b, k=l, s=0, seed=rng.seed_, stream=rng.stream_)
    rng.consumed += int(res.info.gaussians_used)
    return _to_host(res)


def validate_epsilon(eps: float, frob_a: float, delta: float = 0.01):
    """Theorem 3: (valid, floor)."""
    fl = np.zeros(1)
    ok = lib().qbfac_gpu_validate_epsilon(eps, frob_a, delta, _p(fl))
    return bool(ok), float(fl[0])
