"""B200-native DIM^3 Join-Project (arXiv 2206.04995) — the hot path
Π_{x,z}(R(x,y) ⋈_y S(z,y)) behind the reference's operator API.

The compute lives in ``libdim3_b200.so`` (hand-written sm_100a CUDA + C ABI,
``include/dim3_b200.h``); this package is the thin host mirror of the
reference's ``dim3::join_project`` interface.
"""
from .engine import (  # noqa: F401
    EXPORTED,
    LIB_PATH,
    ConfigError,
    Context,
    CostConstants,
    CsrMatrix,
    CudaError,
    DensePathMode,
    Dim3Error,
    EngineConfig,
    ExecutionReport,
    FileFormat,
    FormatError,
    IoError,
    JoinProjectOutput,
    KernelStats,
    RawTable,
    ResourceError,
    ResultSet,
    SkipFlags,
    alu_peak,
    binary_rows,
    detect_format,
    load_table,
    save_result,
    save_table,
    Strategy,
    build_csr,
    cfg_rows,
    default_context,
    dense_ec,
    f1,
    f2_decide,
    f3_threshold,
    generate,
    join_project,
    lib,
    result_to_raw,
    sparse_bmm,
    strategy_from_name,
)

__all__ = [n for n in dir() if not n.startswith("_")]
