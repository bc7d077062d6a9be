"""Host-side mirror of the reference operator API over the C ABI.

Same names, argument meaning and error behaviour as the reference's
``dim3::join_project`` family (P = /root/reference/proj):

=======================  =====================================================
this module              reference
=======================  =====================================================
``RawTable``             ``dim3::RawTable`` (u64 columns), relation.hpp:43-46
``EngineConfig``         ``dim3::EngineConfig``, engine.hpp:36-48
``CostConstants``        ``dim3::CostConstants``, costmodel.hpp:21-30
``Strategy``             ``dim3::Strategy``, engine.hpp:25-31
``DensePathMode``        ``dim3::DensePathMode``, denseec.hpp:56
``join_project``         ``dim3::join_project``, engine.hpp:102-103
``result_to_raw``        ``dim3::result_to_raw``, engine.hpp:123
``ExecutionReport``      ``dim3::ExecutionReport`` (+ GPU fields), :59-85
``build_csr``            ``dim3::build_csr``, relation.hpp:108-109
``sparse_bmm``           ``dim3::sparse_bmm``, sparsebmm.hpp:33-36
``dense_ec``             ``dim3::dense_ec``, denseec.hpp:82-85
``f1/f3_threshold``      costmodel.hpp:86-121
``ConfigError`` ...      common.hpp:25-36 (status codes 2/3/4 as the CLI)
=======================  =====================================================

Everything computes on the GPU through ``libdim3_b200.so``; there is no CPU
fallback. Importing works without a GPU (so host-only policy functions and
the ABI can be inspected), but every compute call raises if the library or
a Blackwell device is unavailable.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field, fields

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# D3G_LIB: an experiment build of the same library (other compile-time tile
# constants); the default is the in-tree build
LIB_PATH = os.environ.get("D3G_LIB") or os.path.join(_HERE, "libdim3_b200.so")

U64P = C.POINTER(C.c_uint64)
U32P = C.POINTER(C.c_uint32)


# ---------------------------------------------------------------------------
# Errors (P/include/dim3/common.hpp:25-36); status codes as P/tools/dim3.cpp:675-693.
class Dim3Error(RuntimeError):
    status = 5


class ConfigError(Dim3Error):
    status = 2


class IoError(Dim3Error):
    status = 3


class FormatError(Dim3Error):
    status = 3


class ResourceError(Dim3Error):
    status = 4


class CudaError(Dim3Error):
    status = 5


_STATUS = {2: ConfigError, 3: IoError, 4: ResourceError, 5: CudaError, 6: FormatError}


class Strategy(enum.IntEnum):
    auto_select = 0
    classical = 1
    hybrid = 2
    sparse_only = 3
    dense_only = 4


class DensePathMode(enum.IntEnum):
    cost_based = 0
    force_wide = 1
    force_probe = 2


def strategy_from_name(name: str) -> Strategy:
    """strategy_from_name (P/src/engine.cpp), CLI spellings."""
    table = {"auto": Strategy.auto_select, "classical": Strategy.classical,
             "hybrid": Strategy.hybrid, "sparse": Strategy.sparse_only,
             "dense": Strategy.dense_only}
    if name not in table:
        raise ConfigError(f"unknown strategy {name!r}")
    return table[name]


@dataclass
class SkipFlags:
    x: bool = False
    y: bool = False
    z: bool = False


@dataclass
class CostConstants:
    t_seqR: float = 0.0
    t_randR: float = 0.0
    t_randRW: float = 0.0
    t_hash: float = 0.0
    t_map: float = 0.0
    t_ECs: float = 0.0
    t_ECd: float = 0.0
    w: int = 256

    @staticmethod
    def test_consts() -> "CostConstants":
        """test_consts() (P/tests/support.hpp:27-38)."""
        return CostConstants(0.9e-9, 140e-9, 140e-9, 440e-9, 330e-9, 11e-9, 1.2e-9, 256)


@dataclass
class EngineConfig:
    force: Strategy = Strategy.auto_select
    threads: int = 1
    memory_budget_bytes: int = 3 << 30
    count_only: bool = False
    collect_cache_stats: bool = False
    dense_mode: DensePathMode = DensePathMode.cost_based
    natural_keys_auto: bool = True
    natural_keys_declared: SkipFlags = field(default_factory=SkipFlags)
    # GPU extensions
    checksum: bool = False        # also compute the (sum, xor) set fingerprint
    # also compute the reference's per-pair DenseEC counters (dense_blocks_checked,
    # dense_probes_done): a separate per-pair pass, for tests and W_D
    collect_counters: bool = False
    shard_index: int = 0          # x-range shard handled by this call
    shard_count: int = 1
    # restrict the SparseBMM/DenseEC kernels to engine x codes in [lo, hi)
    # (None: all). Statistics and f2 decisions stay global; shards split it.
    x_code_range: tuple | None = None


class RawTable:
    """Two columns; row i = (left[i], right[i]) (relation.hpp:43-46).

    Integer columns (ColumnType::u64) are numpy uint64 / uint32 arrays (host)
    or CUDA torch tensors of int64 / uint64 (device-resident input, no H2D
    copy). A column of byte strings (ColumnType::bytes, relation.hpp:21: a
    numpy array or list of ``bytes`` / ``str``) is taken by ``join_project``,
    which interns it into surrogate ids on the host."""

    def __init__(self, left=None, right=None):
        self.left = _as_col(left if left is not None else [])
        self.right = _as_col(right if right is not None else [])
        if _length(self.left) != _length(self.right):
            raise FormatError("left and right columns differ in length")
        if not (_is_bytes_col(self.left) or _is_bytes_col(self.right)) and \
                _itemsize(self.left) != _itemsize(self.right):
            raise FormatError("left and right columns differ in width")

    @property
    def has_bytes(self) -> bool:
        return _is_bytes_col(self.left) or _is_bytes_col(self.right)

    def size(self) -> int:
        return _length(self.left)

    __len__ = size

    @property
    def on_device(self) -> bool:
        return _is_cuda(self.left)


def _is_cuda(a) -> bool:
    return getattr(a, "is_cuda", False)


def _itemsize(a) -> int:
    return int(a.element_size()) if _is_cuda(a) else int(a.dtype.itemsize)


def _length(a) -> int:
    return int(a.shape[0]) if hasattr(a, "shape") else len(a)


def _is_bytes_col(a) -> bool:
    """A ColumnType::bytes column: a numpy array of bytes / str values."""
    return isinstance(a, np.ndarray) and a.dtype.kind in "SUO"


def _as_col(a):
    """A column as the library takes it: 64-bit (u64 values), or 32-bit for
    uint32 numpy arrays / int32 tensors (d3g_table.value_bytes = 4: half the
    host->device bytes, widened on the GPU). Byte-string columns are kept as
    numpy arrays of their values."""
    if _is_cuda(a):
        if a.element_size() not in (4, 8) or not a.is_contiguous():
            raise FormatError("device columns must be contiguous 32- or 64-bit tensors")
        return a
    arr = np.asarray(a)
    if arr.dtype.kind in "SUO" and arr.size:
        if not all(isinstance(v, (bytes, str)) for v in arr.tolist()):
            raise FormatError("a byte-string column holds bytes or str values only")
        return arr
    if arr.dtype == np.uint32:
        return np.ascontiguousarray(arr)
    if arr.dtype != np.uint64:
        if arr.size and arr.dtype.kind == "i" and int(arr.min()) < 0:
            raise FormatError("integer columns must be non-negative")
        arr = arr.astype(np.uint64)
    return np.ascontiguousarray(arr)


# ---------------------------------------------------------------------------
# ctypes mirror of include/dim3_b200.h
class _Table(C.Structure):
    _fields_ = [("left", U64P), ("right", U64P), ("n", C.c_uint64), ("on_device", C.c_int32),
                ("value_bytes", C.c_int32)]


class _Consts(C.Structure):
    _fields_ = [(k, C.c_double) for k in
                ("t_seqR", "t_randR", "t_randRW", "t_hash", "t_map", "t_ECs", "t_ECd")] + \
               [("w", C.c_uint32), ("pad", C.c_uint32)]


class _Opts(C.Structure):
    _fields_ = [("force", C.c_int32), ("threads", C.c_int32), ("memory_budget_bytes", C.c_uint64),
                ("count_only", C.c_int32), ("dense_mode", C.c_int32),
                ("natural_keys_auto", C.c_int32), ("declared_x", C.c_int32),
                ("declared_y", C.c_int32), ("declared_z", C.c_int32), ("checksum", C.c_int32),
                ("collect_counters", C.c_int32), ("shard_index", C.c_int32),
                ("shard_count", C.c_int32), ("x_code_lo", C.c_uint32), ("x_code_hi", C.c_uint32)]


_REPORT_U64_A = ["r_rows", "s_rows", "out_j_estimate"]
_REPORT_U64_B = ["out_p", "pairs_sparse", "pairs_dense", "sparse_z", "dense_z", "f2_evaluations",
                 "dropped_r", "x_card", "y_card", "z_card", "r_nnz", "s_nnz", "sparse_nnz",
                 "out_j", "x_live", "panel_bytes", "peak_bytes", "spa_inner_count",
                 "dense_wide_encounters", "dense_probe_encounters", "dense_blocks_checked",
                 "dense_probes_done", "dense_row_bitmaps_built", "checksum_sum", "checksum_xor",
                 "h2d_bytes", "d2h_bytes"]
_REPORT_MS = ["ms_total", "ms_h2d", "ms_estimate", "ms_map", "ms_csr", "ms_stats",
              "ms_partition", "ms_sparse", "ms_dense", "ms_decode"]


class _Report(C.Structure):
    _fields_ = [("strategy", C.c_char * 16), ("swapped", C.c_int32),
                ("f1_gate_classical", C.c_int32), ("natural_x", C.c_int32),
                ("natural_y", C.c_int32), ("natural_z", C.c_int32), ("materialized", C.c_int32)] + \
               [(k, C.c_uint64) for k in _REPORT_U64_A] + [("f1", C.c_double)] + \
               [(k, C.c_uint64) for k in _REPORT_U64_B] + \
               [(k, C.c_double) for k in _REPORT_MS] + [("gpu_launches", C.c_uint64)] + \
               [("pairs_classical", C.c_uint64), ("intermediate_pairs", C.c_uint64),
                ("ms_classical", C.c_double), ("ms_dense_hot", C.c_double),
                ("hot_lds_bytes", C.c_uint64), ("hot_lds_bytes_unshared", C.c_uint64),
                ("hot_direct_pairs", C.c_uint64), ("ms_dense_cold", C.c_double),
                ("cold_bytes", C.c_uint64), ("spa_allocations", C.c_uint64),
                ("spa_entries", C.c_uint64), ("rank_out_p", C.c_uint64),
                ("nranks", C.c_int32), ("rank", C.c_int32),
                ("cold_candidates", C.c_uint64), ("cold_tail_checks", C.c_uint64),
                ("exchange_calls", C.c_uint64), ("exchange_bus_bytes", C.c_uint64),
                ("ms_exchange_host", C.c_double), ("zsplit", C.c_int32), ("pad1", C.c_int32)]


class _Pairs(C.Structure):
    _fields_ = [("x", U64P), ("z", U64P), ("cap", C.c_uint64), ("n", C.c_uint64),
                ("on_device", C.c_int32), ("pad", C.c_int32)]


class _Csr(C.Structure):
    _fields_ = [("row_ptr", U64P), ("col", U32P), ("n_rows", C.c_uint32), ("n_cols", C.c_uint32),
                ("nnz", C.c_uint64)]


class _Panel(C.Structure):
    _fields_ = [("z_ids", U32P), ("m_z", U32P), ("blocks", U64P), ("rows", C.c_uint64),
                ("y_card", C.c_uint32), ("w", C.c_uint32)]


class _KStats(C.Structure):
    _fields_ = [("inner_count", C.c_uint64), ("wide_encounters", C.c_uint64),
                ("probe_encounters", C.c_uint64), ("blocks_checked", C.c_uint64),
                ("probes_done", C.c_uint64), ("row_bitmaps_built", C.c_uint64),
                ("ms_kernel", C.c_double)]


# Every symbol include/dim3_b200.h declares (tests check the export table).
EXPORTED = ["d3g_ctx_create", "d3g_ctx_destroy", "d3g_last_error", "d3g_version",
            "d3g_opts_default", "d3g_join_project", "d3g_build_csr", "d3g_sparse_bmm_csr",
            "d3g_dense_ec_rows", "d3g_generate", "d3g_cfg_rows", "d3g_ctx_device",
            "d3g_f3_threshold", "d3g_f1", "d3g_f2_decide", "d3g_alu_peak",
            "d3g_detect_format", "d3g_binary_rows", "d3g_read_binary", "d3g_save_pairs",
            "d3g_join_aggregate", "d3g_smem_peak", "d3g_map_tables", "d3g_nccl_unique_id",
            "d3g_ctx_set_nccl", "d3g_ctx_set_exchange", "d3g_take_pairs"]

# multi-GPU exchange ops (include/dim3_b200.h D3G_EX_*)
EX_SUM_U64, EX_SUM_U32, EX_MAX_U64, EX_GATHER = 0, 1, 2, 3
_EXFN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_uint64)

_lib = None


def lib():
    """Loads libdim3_b200.so (fails loudly when it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                              "(make -C paper_2206_04995_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        L.d3g_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.d3g_ctx_destroy.argtypes = [C.c_void_p]
        L.d3g_last_error.restype = C.c_char_p
        L.d3g_version.restype = C.c_char_p
        L.d3g_opts_default.argtypes = [C.POINTER(_Opts)]
        L.d3g_join_project.argtypes = [C.c_void_p, C.POINTER(_Table), C.POINTER(_Table),
                                       C.POINTER(_Consts), C.POINTER(_Opts), C.POINTER(_Report),
                                       C.POINTER(_Pairs)]
        L.d3g_build_csr.argtypes = [C.c_void_p, U32P, U32P, C.c_uint64, C.c_uint32, C.c_uint32,
                                    C.c_int, C.POINTER(_Csr)]
        L.d3g_sparse_bmm_csr.argtypes = [C.c_void_p, C.POINTER(_Csr), C.POINTER(_Csr), C.c_uint32,
                                         U32P, U32P, C.c_uint64, U64P, C.POINTER(_KStats)]
        L.d3g_dense_ec_rows.argtypes = [C.c_void_p, C.POINTER(_Csr), C.POINTER(_Panel),
                                        C.POINTER(_Consts), C.c_int, U32P, U32P, C.c_uint64, U64P,
                                        C.POINTER(_KStats)]
        L.d3g_generate.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                   C.c_void_p, C.c_void_p]
        L.d3g_cfg_rows.argtypes = [C.c_int]
        L.d3g_cfg_rows.restype = C.c_uint64
        L.d3g_ctx_device.argtypes = [C.c_void_p]
        L.d3g_alu_peak.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        L.d3g_smem_peak.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        L.d3g_f3_threshold.argtypes = [C.c_uint32, C.c_uint32, C.POINTER(_Consts)]
        L.d3g_f3_threshold.restype = C.c_uint32
        L.d3g_f1.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(_Consts)]
        L.d3g_f1.restype = C.c_double
        L.d3g_f2_decide.argtypes = [U64P, C.c_uint64, U64P, C.c_uint64, C.c_uint64, C.c_uint64,
                                    C.c_uint64, C.c_uint64, C.POINTER(_Consts), C.c_int,
                                    C.POINTER(C.c_uint8), U64P]
        L.d3g_join_aggregate.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                         C.POINTER(_Consts), C.POINTER(_Opts), C.POINTER(_Report),
                                         C.c_void_p]
        L.d3g_map_tables.argtypes = [C.c_void_p, C.POINTER(_Table), C.POINTER(_Table),
                                     C.POINTER(_Opts), C.c_void_p]
        L.d3g_detect_format.argtypes = [C.c_char_p, C.c_int]
        L.d3g_binary_rows.argtypes = [C.c_char_p, U64P]
        L.d3g_read_binary.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_void_p, C.c_uint64]
        L.d3g_save_pairs.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int,
                                     C.c_char_p, C.c_int]
        L.d3g_take_pairs.argtypes = [C.c_void_p, U64P, U64P, C.c_uint64, C.c_int]
        L.d3g_nccl_unique_id.argtypes = [C.c_void_p]
        L.d3g_ctx_set_nccl.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.d3g_ctx_set_exchange.argtypes = [C.c_void_p, C.c_int, C.c_int, _EXFN, C.c_void_p]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        msg = lib().d3g_last_error().decode(errors="replace")
        raise _STATUS.get(rc, Dim3Error)(msg)


def _consts(c: CostConstants) -> _Consts:
    return _Consts(c.t_seqR, c.t_randR, c.t_randRW, c.t_hash, c.t_map, c.t_ECs, c.t_ECd, c.w, 0)


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId for rank 0 to share (128 bytes)."""
    buf = C.create_string_buffer(128)
    _check(lib().d3g_nccl_unique_id(buf))
    return buf.raw


class Context:
    """One CUDA device + stream + device-memory pool (the C ABI's d3g_ctx)."""
    nranks, rank = 1, 0

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        _check(lib().d3g_ctx_create(device, C.byref(self._h)))
        self.device = device

    @property
    def handle(self):
        return self._h

    # -- multi-GPU: this context as one rank of an x-sharded job -------------
    def set_nccl(self, unique_id: bytes, nranks: int, rank: int):
        """NCCL communicator (collective over the job; every rank calls it with
        rank 0's nccl_unique_id())."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(lib().d3g_ctx_set_nccl(self._h, buf, nranks, rank))
        self.nranks, self.rank = nranks, rank

    def set_exchange(self, nranks: int, rank: int, fn):
        """Host-callback transport: fn(op, arr) performs the collective in place
        on a numpy array (u64 / u32 elements; EX_GATHER: nranks * count bytes,
        this rank's block filled). See paper_2206_04995_b200.distributed."""
        def cb(_user, op, buf, count):
            try:
                if op == EX_GATHER:
                    arr = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_uint8)),
                                                shape=(nranks * count,))
                else:
                    ct = C.c_uint32 if op == EX_SUM_U32 else C.c_uint64
                    arr = np.ctypeslib.as_array(C.cast(buf, C.POINTER(ct)), shape=(count,))
                fn(op, arr)
                return 0
            except BaseException as e:  # surfaced as the call's error
                self.exchange_error = e
                return 1
        self._exfn = _EXFN(cb)  # kept alive with the context
        _check(lib().d3g_ctx_set_exchange(self._h, nranks, rank, self._exfn, None))
        self.nranks, self.rank = nranks, rank

    def clear_exchange(self):
        _check(lib().d3g_ctx_set_exchange(self._h, 1, 0, C.cast(None, _EXFN), None))
        self._exfn = None
        self.nranks, self.rank = 1, 0

    def close(self):
        if self._h:
            lib().d3g_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: dict[int, Context] = {}


def default_context(device: int | None = None) -> Context:
    if device is None:
        device = 0
        try:
            import torch
            if torch.cuda.is_available():
                device = torch.cuda.current_device()
        except Exception:
            pass
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


# ---------------------------------------------------------------------------
@dataclass
class ExecutionReport:
    strategy: str = ""
    swapped: bool = False
    f1_gate_classical: bool = False
    natural_x: bool = False
    natural_y: bool = False
    natural_z: bool = False
    materialized: bool = False
    r_rows: int = 0
    s_rows: int = 0
    out_j_estimate: int = 0
    f1_value: float = 0.0
    out_p: int = 0
    pairs_sparse: int = 0
    pairs_dense: int = 0
    sparse_z: int = 0
    dense_z: int = 0
    f2_evaluations: int = 0
    dropped_r: int = 0
    x_card: int = 0
    y_card: int = 0
    z_card: int = 0
    r_nnz: int = 0
    s_nnz: int = 0
    sparse_nnz: int = 0
    out_j: int = 0
    x_live: int = 0
    panel_bytes: int = 0
    peak_bytes: int = 0
    spa_inner_count: int = 0
    dense_wide_encounters: int = 0
    dense_probe_encounters: int = 0
    dense_blocks_checked: int = 0
    dense_probes_done: int = 0
    dense_row_bitmaps_built: int = 0
    checksum_sum: int = 0
    checksum_xor: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    ms_total: float = 0.0
    ms_h2d: float = 0.0
    ms_estimate: float = 0.0
    ms_map: float = 0.0
    ms_csr: float = 0.0
    ms_stats: float = 0.0
    ms_partition: float = 0.0
    ms_sparse: float = 0.0
    ms_dense: float = 0.0
    ms_decode: float = 0.0
    gpu_launches: int = 0
    pairs_classical: int = 0
    intermediate_pairs: int = 0
    ms_classical: float = 0.0
    ms_dense_hot: float = 0.0
    hot_lds_bytes: int = 0
    hot_lds_bytes_unshared: int = 0
    hot_direct_pairs: int = 0
    ms_dense_cold: float = 0.0
    cold_bytes: int = 0
    spa_allocations: int = 0
    spa_entries: int = 0
    rank_out_p: int = 0
    nranks: int = 1
    rank: int = 0
    cold_candidates: int = 0
    cold_tail_checks: int = 0
    exchange_calls: int = 0
    exchange_bus_bytes: int = 0
    ms_exchange_host: float = 0.0
    zsplit: bool = False

    def to_kv(self):
        """Insertion-ordered key/value view with the reference's key names
        first (ExecutionReport::to_kv, P/src/engine.cpp:276-321)."""
        kv = [("strategy", self.strategy), ("swapped", "true" if self.swapped else "false"),
              ("r_rows", str(self.r_rows)), ("s_rows", str(self.s_rows)),
              ("out_j_estimate", str(self.out_j_estimate)), ("f1", f"{self.f1_value:.6g}"),
              ("out_p", str(self.out_p)), ("pairs_classical", str(self.pairs_classical)),
              ("pairs_sparse", str(self.pairs_sparse)), ("pairs_dense", str(self.pairs_dense)),
              ("pairs_cached", "0"), ("sparse_z", str(self.sparse_z)),
              ("dense_z", str(self.dense_z)), ("cached_z", "0"),
              ("f2_evaluations", str(self.f2_evaluations)), ("dropped_r", str(self.dropped_r)),
              ("intermediate_pairs", str(self.intermediate_pairs)), ("x_card", str(self.x_card)),
              ("y_card", str(self.y_card)), ("z_card", str(self.z_card)),
              ("panel_bytes", str(self.panel_bytes)), ("peak_bytes", str(self.peak_bytes)),
              ("spa_inner_count", str(self.spa_inner_count)),
              ("spa_allocations", str(self.spa_allocations)),
              ("spa_entries", str(self.spa_entries)),
              ("dense_wide_encounters", str(self.dense_wide_encounters)),
              ("dense_probe_encounters", str(self.dense_probe_encounters)),
              ("dense_blocks_checked", str(self.dense_blocks_checked)),
              ("dense_probes_done", str(self.dense_probes_done)),
              ("dense_row_bitmaps_built", str(self.dense_row_bitmaps_built))]
        for k in ("ms_total", "ms_estimate", "ms_map", "ms_csr", "ms_partition", "ms_sparse",
                  "ms_dense", "ms_classical", "ms_decode"):
            kv.append((k, f"{getattr(self, k):.3f}"))
        for k in ("f1_gate_classical", "x_live", "out_j", "r_nnz", "s_nnz", "sparse_nnz",
                  "checksum_sum", "checksum_xor", "ms_h2d", "ms_stats", "gpu_launches"):
            kv.append((k, str(getattr(self, k))))
        return kv


@dataclass
class ResultSet:
    """ResultSet after result_to_raw: raw caller-oriented pairs, sorted by
    (x code, z code) — raw value order under natural keys."""
    count: int = 0
    materialized: bool = True
    raw_x: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    raw_z: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))


@dataclass
class JoinProjectOutput:
    result: ResultSet
    report: ExecutionReport


def _table_struct(t: RawTable) -> _Table:
    if t.has_bytes:
        raise ConfigError("byte-string columns are taken by join_project only")
    vb = _itemsize(t.left)
    if t.on_device:
        return _Table(C.cast(C.c_void_p(t.left.data_ptr()), U64P),
                      C.cast(C.c_void_p(t.right.data_ptr()), U64P), t.size(), 1, vb)
    return _Table(C.cast(t.left.ctypes.data, U64P), C.cast(t.right.ctypes.data, U64P), t.size(), 0,
                  vb)


def _opts(cfg: EngineConfig) -> _Opts:
    if cfg.collect_cache_stats:
        raise ConfigError("collect_cache_stats belongs to the partial-result cache, which is "
                          "outside this operator's scope")
    d = cfg.natural_keys_declared
    xr = cfg.x_code_range or (0, 0)
    if len(xr) != 2 or not (0 <= xr[0] <= xr[1] < (1 << 32)):
        raise ConfigError("x_code_range must be (lo, hi) with 0 <= lo <= hi < 2^32")
    return _Opts(int(cfg.force), int(cfg.threads), int(cfg.memory_budget_bytes),
                 int(cfg.count_only), int(cfg.dense_mode), int(cfg.natural_keys_auto),
                 int(d.x), int(d.y), int(d.z), int(cfg.checksum), int(cfg.collect_counters),
                 int(cfg.shard_index),
                 int(cfg.shard_count), int(xr[0]), int(xr[1]))


def join_project(r: RawTable, s: RawTable, cfg: EngineConfig, c: CostConstants,
                 ctx: Context | None = None) -> JoinProjectOutput:
    """dim3::join_project on the GPU. Raises ConfigError / ResourceError like
    the reference. With cfg.count_only the result is not materialized."""
    if cfg.threads < 1:
        raise ConfigError("threads must be >= 1")
    ctx = ctx or default_context()
    dec_x = dec_z = None
    key_flags = 0
    if r.has_bytes or s.has_bytes:
        r, s, dec_x, dec_z, key_flags = _intern_bytes(r, s)
    rt, st = _table_struct(r), _table_struct(s)
    cs, op = _consts(c), _opts(cfg)
    op.natural_keys_auto |= key_flags
    rep = _Report()
    pairs_p = None
    ox = oz = None
    if not cfg.count_only:
        # one pipeline pass: the library keeps the sorted, decoded pairs on the
        # device (d3g_pairs.x == NULL) and they are copied out once sized
        pairs = _Pairs(None, None, 0, 0, 0, 0)
        pairs_p = C.byref(pairs)
    _check(lib().d3g_join_project(ctx.handle, C.byref(rt), C.byref(st), C.byref(cs), C.byref(op),
                                  C.byref(rep), pairs_p))
    if not cfg.count_only:
        n = int(pairs.n)  # a sharded rank materializes its own pairs
        ox = np.zeros(max(n, 1), dtype=np.uint64)
        oz = np.zeros(max(n, 1), dtype=np.uint64)
        _check(lib().d3g_take_pairs(ctx.handle, ox.ctypes.data_as(U64P), oz.ctypes.data_as(U64P),
                                    n, 0))
    report = _to_report(rep)
    if cfg.count_only:
        res = ResultSet(count=report.out_p, materialized=False)
    else:
        n = int(pairs.n)
        rx, rz = ox[:n], oz[:n]
        if dec_x is not None:  # surrogate ids back to the byte strings
            rx = dec_x[rx.astype(np.int64)]
        if dec_z is not None:
            rz = dec_z[rz.astype(np.int64)]
        res = ResultSet(count=n, materialized=True, raw_x=rx, raw_z=rz)
    return JoinProjectOutput(res, report)


KEYS_AUTO, KEYS_BYTES_X, KEYS_BYTES_Y, KEYS_BYTES_Z = 1, 2, 4, 8  # d3g_opts.natural_keys_auto bits


def _intern_bytes(r: RawTable, s: RawTable):
    """Byte-string columns (ColumnType::bytes) as surrogate u64 ids: equal
    strings <-> equal ids. The device dictionary-codes the ids like the
    reference does the strings (they are flagged D3G_KEYS_BYTES_*, in engine
    orientation: the larger table's left column is x), and the result ids are
    mapped back through the returned decode arrays. The two y columns share
    one id space; when their types differ no R row finds its y
    (Dictionary::lookup, mapping.cpp:177-189): disjoint id ranges."""
    if r.on_device or s.on_device:
        raise ConfigError("byte-string columns are host columns")

    def ids_of(col):
        vals, inv = np.unique(col, return_inverse=True)
        return vals, inv.astype(np.uint64)

    def widen(col):
        return col.astype(np.uint64) if col.dtype != np.uint64 else col

    bx, bz = _is_bytes_col(r.left), _is_bytes_col(s.left)
    by_r, by_s = _is_bytes_col(r.right), _is_bytes_col(s.right)
    dec_x = dec_z = None
    rl, sl, rr, sr = r.left, s.left, r.right, s.right
    if bx:
        dec_x, rl = ids_of(rl)
    if bz:
        dec_z, sl = ids_of(sl)
    if by_r and by_s:
        both = np.concatenate([np.asarray(rr, dtype=object), np.asarray(sr, dtype=object)])
        if both.size and not all(type(v) is type(both[0]) for v in both.tolist()):
            raise FormatError("the y columns mix bytes and str values")
        _, inv = np.unique(both, return_inverse=True)
        rr, sr = inv[:len(rr)].astype(np.uint64), inv[len(rr):].astype(np.uint64)
    elif by_r or by_s:
        # different types never compare equal (ColumnData::value_equals)
        ur, rr = np.unique(rr, return_inverse=True)
        _, sr = np.unique(sr, return_inverse=True)
        rr, sr = rr.astype(np.uint64), sr.astype(np.uint64) + np.uint64(len(ur))
    swapped = s.size() > r.size()
    flags = ((KEYS_BYTES_X if (bz if swapped else bx) else 0) |
             (KEYS_BYTES_Y if (by_r or by_s) else 0) |
             (KEYS_BYTES_Z if (bx if swapped else bz) else 0))
    r2 = RawTable(widen(np.ascontiguousarray(rl)), widen(np.ascontiguousarray(rr)))
    s2 = RawTable(widen(np.ascontiguousarray(sl)), widen(np.ascontiguousarray(sr)))
    return r2, s2, dec_x, dec_z, flags


def _to_report(rep: _Report) -> ExecutionReport:
    out = ExecutionReport()
    for f in fields(ExecutionReport):
        src = "f1" if f.name == "f1_value" else f.name
        v = getattr(rep, src)
        if isinstance(v, bytes):
            v = v.decode()
        if f.type in ("bool",):
            v = bool(v)
        setattr(out, f.name, v)
    for b in ("swapped", "f1_gate_classical", "natural_x", "natural_y", "natural_z",
              "materialized", "zsplit"):
        setattr(out, b, bool(getattr(out, b)))
    return out


def result_to_raw(out: JoinProjectOutput) -> ResultSet:
    """Results are already decoded to raw values on the device."""
    return out.result


# ---------------------------------------------------------------------------
# Kernel-level entry points
@dataclass
class CsrMatrix:
    row_ptr: np.ndarray
    col: np.ndarray
    n_rows: int
    n_cols: int

    def nnz(self) -> int:
        return int(self.col.shape[0])

    def _struct(self) -> _Csr:
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.uint64)
        self.col = np.ascontiguousarray(self.col, dtype=np.uint32)
        return _Csr(self.row_ptr.ctypes.data_as(U64P), self.col.ctypes.data_as(U32P),
                    self.n_rows, self.n_cols, self.nnz())


def build_csr(a: np.ndarray, b: np.ndarray, a_card: int, b_card: int, major_is_a: bool = True,
              ctx: Context | None = None) -> CsrMatrix:
    """dim3::build_csr on mapped code columns (a, b)."""
    ctx = ctx or default_context()
    a = np.ascontiguousarray(a, dtype=np.uint32)
    b = np.ascontiguousarray(b, dtype=np.uint32)
    n_rows = a_card if major_is_a else b_card
    rp = np.zeros(n_rows + 1, dtype=np.uint64)
    col = np.zeros(max(a.size, 1), dtype=np.uint32)
    out = _Csr(rp.ctypes.data_as(U64P), col.ctypes.data_as(U32P), 0, 0, 0)
    _check(lib().d3g_build_csr(ctx.handle, a.ctypes.data_as(U32P), b.ctypes.data_as(U32P), a.size,
                               a_card, b_card, int(major_is_a), C.byref(out)))
    return CsrMatrix(rp, col[: out.nnz].copy(), out.n_rows, out.n_cols)


@dataclass
class KernelStats:
    inner_count: int = 0
    wide_encounters: int = 0
    probe_encounters: int = 0
    blocks_checked: int = 0
    probes_done: int = 0
    row_bitmaps_built: int = 0
    ms_kernel: float = 0.0


def sparse_bmm(r_by_x: CsrMatrix, s_sparse_by_y: CsrMatrix, z_card: int, materialize=True,
               ctx: Context | None = None):
    """dim3::sparse_bmm: returns (count, pairs[n,2] sorted by (x, z) or None, stats)."""
    ctx = ctx or default_context()
    r, s = r_by_x._struct(), s_sparse_by_y._struct()
    cnt = C.c_uint64()
    st = _KStats()
    _check(lib().d3g_sparse_bmm_csr(ctx.handle, C.byref(r), C.byref(s), z_card, None, None, 0,
                                    C.byref(cnt), C.byref(st)))
    pairs = None
    if materialize:
        n = cnt.value
        px = np.zeros(max(n, 1), np.uint32)
        pz = np.zeros(max(n, 1), np.uint32)
        _check(lib().d3g_sparse_bmm_csr(ctx.handle, C.byref(r), C.byref(s), z_card,
                                        px.ctypes.data_as(U32P), pz.ctypes.data_as(U32P), n,
                                        C.byref(cnt), C.byref(st)))
        pairs = np.stack([px[:n], pz[:n]], axis=1)
    return cnt.value, pairs, KernelStats(**{k: getattr(st, k) for k, _ in _KStats._fields_})


def dense_ec(r_by_x: CsrMatrix, z_ids: np.ndarray, panel_blocks: np.ndarray, y_card: int,
             c: CostConstants, mode: DensePathMode = DensePathMode.cost_based, materialize=True,
             ctx: Context | None = None):
    """dim3::dense_ec over a BitmapPanel given as (z_ids, rows*row_words u64 blocks)."""
    ctx = ctx or default_context()
    r = r_by_x._struct()
    z_ids = np.ascontiguousarray(z_ids, dtype=np.uint32)
    blocks = np.ascontiguousarray(panel_blocks, dtype=np.uint64)
    # BitmapPanel::m_z: the degree of each row (its popcount)
    row_words = blocks.size // max(z_ids.size, 1)
    mz = np.zeros(max(z_ids.size, 1), np.uint32)
    if z_ids.size:
        bits = np.unpackbits(blocks.view(np.uint8).reshape(z_ids.size, row_words * 8), axis=1)
        mz[:z_ids.size] = bits.sum(axis=1, dtype=np.uint64).astype(np.uint32)
    panel = _Panel(z_ids.ctypes.data_as(U32P), mz.ctypes.data_as(U32P),
                   blocks.ctypes.data_as(U64P), z_ids.size, y_card, c.w)
    cs = _consts(c)
    cnt = C.c_uint64()
    st = _KStats()
    _check(lib().d3g_dense_ec_rows(ctx.handle, C.byref(r), C.byref(panel), C.byref(cs), int(mode),
                                   None, None, 0, C.byref(cnt), C.byref(st)))
    pairs = None
    if materialize:
        n = cnt.value
        px = np.zeros(max(n, 1), np.uint32)
        pz = np.zeros(max(n, 1), np.uint32)
        _check(lib().d3g_dense_ec_rows(ctx.handle, C.byref(r), C.byref(panel), C.byref(cs),
                                       int(mode), px.ctypes.data_as(U32P),
                                       pz.ctypes.data_as(U32P), n, C.byref(cnt), C.byref(st)))
        pairs = np.stack([px[:n], pz[:n]], axis=1)
    return cnt.value, pairs, KernelStats(**{k: getattr(st, k) for k, _ in _KStats._fields_})


# ---------------------------------------------------------------------------
# Host-only policy (no GPU needed)
def smem_peak(ctx: "Context | None" = None) -> float:
    """Measured shared-memory read bandwidth (bytes/s), d3g_smem_peak."""
    ctx = ctx or default_context()
    v = C.c_double()
    _check(lib().d3g_smem_peak(ctx.handle, C.byref(v)))
    return v.value


def f1(size_r: int, size_s: int, out_j: int, c: CostConstants) -> float:
    cs = _consts(c)
    return lib().d3g_f1(size_r, size_s, out_j, C.byref(cs))


def f3_threshold(m_x: int, y_card: int, c: CostConstants) -> int:
    cs = _consts(c)
    return int(lib().d3g_f3_threshold(m_x, y_card, C.byref(cs)))


def f2_decide(mx_hist: np.ndarray, mz_hist: np.ndarray, x_card: int, y_card: int, z_card: int,
              out_j: int, c: CostConstants, force: Strategy = Strategy.hybrid):
    """Per-degree f2 decision table from GLOBAL degree histograms (the
    quantities a multi-GPU run all-reduces). Returns (dense_of_mz, evaluations)."""
    mx = np.ascontiguousarray(mx_hist, dtype=np.uint64)
    mz = np.ascontiguousarray(mz_hist, dtype=np.uint64)
    out = np.zeros(max(mz.size, 1), dtype=np.uint8)
    ev = C.c_uint64()
    cs = _consts(c)
    _check(lib().d3g_f2_decide(mx.ctypes.data_as(U64P), mx.size, mz.ctypes.data_as(U64P), mz.size,
                               x_card, y_card, z_card, out_j, C.byref(cs), int(force),
                               out.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(ev)))
    return out[: mz.size], ev.value


def generate(cfg: int, side: int, lo: int = 0, hi: int | None = None, device=None,
             ctx: Context | None = None):
    """Convention-G rows on the GPU, returned as two int64 CUDA tensors
    (bit patterns of the u64 values)."""
    import torch
    ctx = ctx or default_context(device)
    n = int(lib().d3g_cfg_rows(cfg))
    hi = n if hi is None else hi
    dev = torch.device("cuda", ctx.device)
    left = torch.empty(hi - lo, dtype=torch.int64, device=dev)
    right = torch.empty(hi - lo, dtype=torch.int64, device=dev)
    torch.cuda.synchronize(dev)
    _check(lib().d3g_generate(ctx.handle, cfg, side, lo, hi, C.c_void_p(left.data_ptr()),
                              C.c_void_p(right.data_ptr())))
    return left, right


def alu_peak(ctx: Context | None = None) -> float:
    """Measured 32-bit logic ops/s of the device (DenseEC roofline denominator)."""
    ctx = ctx or default_context()
    v = C.c_double()
    _check(lib().d3g_alu_peak(ctx.handle, C.byref(v)))
    return v.value


def cfg_rows(cfg: int) -> int:
    return int(lib().d3g_cfg_rows(cfg))


# ---------------------------------------------------------------------------
# Table files (P/src/relation.cpp; P/include/dim3/relation.hpp FileFormat).
class FileFormat(enum.IntEnum):
    auto_detect = 0
    tsv = 1
    csv = 2
    binary = 3


def detect_format(path, requested: FileFormat = FileFormat.auto_detect) -> FileFormat:
    """detect_format (relation.cpp:13-20)."""
    return FileFormat(lib().d3g_detect_format(os.fsencode(str(path)), int(requested)))


def binary_rows(path) -> int:
    """Rows of a binary table file; IoError / FormatError like read_binary
    (relation.cpp:98-107). Host-only."""
    n = C.c_uint64()
    _check(lib().d3g_binary_rows(os.fsencode(str(path)), C.byref(n)))
    return n.value


def load_table(path, fmt: FileFormat = FileFormat.auto_detect, ctx: "Context | None" = None,
               device=None) -> RawTable:
    """load_table (relation.cpp:130-139) for binary tables: the file streams
    through pinned chunks into HBM and is de-interleaved on the GPU; returns
    a RawTable of device columns. Text tables (TSV/CSV parsing) are outside
    this path's scope and raise FormatError."""
    import torch
    if detect_format(path, fmt) != FileFormat.binary:
        raise FormatError("only binary tables load on the device path "
                          "(TSV/CSV parsing is outside this operator's scope)")
    n = binary_rows(path)
    ctx = ctx or default_context(device)
    dev = torch.device("cuda", ctx.device)
    left = torch.empty(n, dtype=torch.int64, device=dev)
    right = torch.empty(n, dtype=torch.int64, device=dev)
    torch.cuda.synchronize(dev)
    _check(lib().d3g_read_binary(ctx.handle, os.fsencode(str(path)), C.c_void_p(left.data_ptr()),
                                 C.c_void_p(right.data_ptr()), n))
    return RawTable(left, right)


def save_table(t: RawTable, path, fmt: FileFormat = FileFormat.auto_detect,
               ctx: "Context | None" = None, device=None) -> None:
    """save_table (relation.cpp:164-204): binary = interleaved little-endian
    u64 pairs, tsv/csv = "left<sep>right\\n" in decimal. Interleaving or
    formatting runs on the GPU; host or device columns."""
    ctx = ctx or default_context(device)
    n = t.size()
    on_dev = _is_cuda(t.left)
    if on_dev:
        import torch
        torch.cuda.synchronize(t.left.device)
        lp, rp = C.c_void_p(t.left.data_ptr()), C.c_void_p(t.right.data_ptr())
    else:
        lp, rp = C.c_void_p(t.left.ctypes.data), C.c_void_p(t.right.ctypes.data)
    _check(lib().d3g_save_pairs(ctx.handle, lp, rp, n, int(on_dev), os.fsencode(str(path)),
                                int(fmt)))


def save_result(out: "JoinProjectOutput", path, fmt: FileFormat = FileFormat.auto_detect,
                ctx: "Context | None" = None) -> None:
    """The CLI's --out (P/tools/dim3.cpp:212-218): result_to_raw, then
    save_table of the decoded (x, z) pairs."""
    raw = result_to_raw(out)
    save_table(RawTable(raw.raw_x, raw.raw_z), path, fmt, ctx)


# ---------------------------------------------------------------------------
# Join-aggregate (P/include/dim3/engine.hpp:126-154, P/src/engine.cpp:537-722)
class AggFn(enum.IntEnum):
    sum = 0
    count = 1
    min = 2
    max = 3
    avg = 4


class CombineFn(enum.IntEnum):
    multiply = 0
    add = 1
    abs_diff = 2
    left = 3
    right = 4


def agg_from_name(name: str) -> "AggFn | None":
    return AggFn.__members__.get(name)


def combine_from_name(name: str) -> "CombineFn | None":
    return CombineFn.__members__.get(name)


class ValuedTable:
    """dim3::ValuedTable (relation.hpp:49-53): a RawTable plus one double per
    row (numpy array, or a CUDA float64 tensor when the table is on the
    device)."""

    def __init__(self, base: RawTable, values):
        self.base = base
        if _is_cuda(values):
            if values.dtype.itemsize != 8 or not values.is_contiguous() or \
                    not values.dtype.is_floating_point:
                raise FormatError("device values must be a contiguous float64 tensor")
            self.values = values
        else:
            self.values = np.ascontiguousarray(values, dtype=np.float64)
        if _length(self.values) != base.size():
            raise ConfigError("value column length does not match table length")

    def size(self) -> int:
        return self.base.size()


class _ValuedTable(C.Structure):
    _fields_ = [("base", _Table), ("values", C.c_void_p)]


class _AggPairs(C.Structure):
    _fields_ = [("x", U64P), ("z", U64P), ("values", C.c_void_p), ("cap", C.c_uint64),
                ("n", C.c_uint64), ("on_device", C.c_int32), ("pad", C.c_int32)]


@dataclass
class AggregateResult:
    """AggregateResult (engine.hpp:139-146): base = the (x, z) pairs (raw
    values, already decoded), values[i] belongs to pair i."""
    base: ResultSet
    values: np.ndarray
    report: ExecutionReport


def _valued_struct(t: ValuedTable) -> _ValuedTable:
    base = _table_struct(t.base)
    if t.base.on_device != _is_cuda(t.values):
        raise ConfigError("values must live where the table lives (host or device)")
    vp = C.c_void_p(t.values.data_ptr()) if _is_cuda(t.values) else C.c_void_p(t.values.ctypes.data)
    return _ValuedTable(base, vp)


def join_aggregate_both(r: ValuedTable, s: ValuedTable, combine: CombineFn, agg: AggFn,
                        cfg: EngineConfig, c: CostConstants,
                        ctx: Context | None = None) -> AggregateResult:
    """dim3::join_aggregate_both on the GPU, caller orientation (no swap).
    Values are bit-identical to the reference's; force=classical raises
    ConfigError like the reference."""
    if cfg.threads < 1:
        raise ConfigError("threads must be >= 1")
    if cfg.force == Strategy.classical:
        raise ConfigError("join-aggregate always runs the mapped pipeline")
    ctx = ctx or default_context()
    rt, st = _valued_struct(r), _valued_struct(s)
    cs, op = _consts(c), _opts(cfg)
    rep = _Report()
    out_p = None
    ox = oz = ov = None
    if not cfg.count_only:
        cnt_op = _opts(cfg)
        cnt_op.count_only = 1
        _check(lib().d3g_join_aggregate(ctx.handle, C.byref(rt), C.byref(st), int(combine),
                                        int(agg), C.byref(cs), C.byref(cnt_op), C.byref(rep),
                                        None))
        n = int(rep.out_p)
        ox = np.zeros(max(n, 1), dtype=np.uint64)
        oz = np.zeros(max(n, 1), dtype=np.uint64)
        ov = np.zeros(max(n, 1), dtype=np.float64)
        outs = _AggPairs(ox.ctypes.data_as(U64P), oz.ctypes.data_as(U64P),
                         C.c_void_p(ov.ctypes.data), n, 0, 0, 0)
        out_p = C.byref(outs)
    _check(lib().d3g_join_aggregate(ctx.handle, C.byref(rt), C.byref(st), int(combine), int(agg),
                                    C.byref(cs), C.byref(op), C.byref(rep), out_p))
    report = _to_report(rep)
    n = report.out_p
    if cfg.count_only:
        return AggregateResult(ResultSet(count=n, materialized=False), np.zeros(0), report)
    return AggregateResult(ResultSet(count=n, materialized=True, raw_x=ox[:n], raw_z=oz[:n]),
                           ov[:n], report)


def aggregate_to_raw(out: AggregateResult) -> ResultSet:
    """aggregate_to_raw (engine.cpp:530-532): pairs are already raw."""
    return out.base


# ---------------------------------------------------------------------------
# map_tables (P/include/dim3/mapping.hpp:124-141, P/src/mapping.cpp:342-420)
class _Mapping(C.Structure):
    _fields_ = [(k, U32P) for k in ("r_x", "r_y", "s_z", "s_y", "r_kept")] + \
               [(k, U64P) for k in ("rev_x", "rev_y", "rev_z")] + \
               [(k, C.c_uint64) for k in ("kept", "dropped_r", "x_card", "y_card", "z_card")] + \
               [(k, C.c_int32) for k in ("natural_x", "natural_y", "natural_z", "pad")]


@dataclass
class MappingOutput:
    """MappingOutput on the host: MappedTable r = (r_a = x codes, r_b = y codes)
    of the surviving rows, s = (s_a = z codes, s_b = y codes); cards; r_kept
    (empty when nothing was dropped); rev_* decode codes to values (None for
    identity/natural columns)."""
    r_a: np.ndarray
    r_b: np.ndarray
    s_a: np.ndarray
    s_b: np.ndarray
    r_kept: np.ndarray
    dropped_r: int
    x_card: int
    y_card: int
    z_card: int
    rev_x: "np.ndarray | None"
    rev_y: "np.ndarray | None"
    rev_z: "np.ndarray | None"


def map_tables(r: RawTable, s: RawTable, skip: SkipFlags | None = None,
               natural_keys_auto: bool = False, ctx: "Context | None" = None) -> MappingOutput:
    """dim3::map_tables on the GPU (HBM dictionaries, the reference's codes).
    skip = SkipFlags: columns declared natural (identity codes, no y
    semi-join when y is skipped); natural_keys_auto: map_with_fallback."""
    ctx = ctx or default_context()
    skip = skip or SkipFlags()
    nr, ns = r.size(), s.size()
    bufs = {k: np.zeros(max(n, 1), np.uint32) for k, n in
            (("r_x", nr), ("r_y", nr), ("r_kept", nr), ("s_z", ns), ("s_y", ns))}
    revs = {"rev_x": np.zeros(max(nr, 1), np.uint64), "rev_y": np.zeros(max(nr + ns, 1), np.uint64),
            "rev_z": np.zeros(max(ns, 1), np.uint64)}
    m = _Mapping(*[bufs[k].ctypes.data_as(U32P) for k in ("r_x", "r_y", "s_z", "s_y", "r_kept")],
                 *[revs[k].ctypes.data_as(U64P) for k in ("rev_x", "rev_y", "rev_z")])
    cfg = EngineConfig(natural_keys_auto=natural_keys_auto, natural_keys_declared=skip)
    rt, st = _table_struct(r), _table_struct(s)
    _check(lib().d3g_map_tables(ctx.handle, C.byref(rt), C.byref(st), C.byref(_opts(cfg)),
                                C.byref(m)))
    kept = int(m.kept)
    return MappingOutput(bufs["r_x"][:kept].copy(), bufs["r_y"][:kept].copy(),
                         bufs["s_z"][:ns].copy(), bufs["s_y"][:ns].copy(),
                         bufs["r_kept"][:kept].copy() if m.dropped_r else np.zeros(0, np.uint32),
                         int(m.dropped_r), int(m.x_card), int(m.y_card), int(m.z_card),
                         None if m.natural_x else revs["rev_x"][:m.x_card].copy(),
                         None if m.natural_y else revs["rev_y"][:m.y_card].copy(),
                         None if m.natural_z else revs["rev_z"][:m.z_card].copy())
