"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the two CPU checkers.

* ``liboracle.so``   — our plain-C restatement (oracle/dim3_oracle.c).
* ``_ref/libdim3ref.so`` — the unmodified reference library plus the C-ABI
  driver (oracle/ref_driver.cpp), built by oracle/Makefile from
  /root/reference. It travels to the GPU box as a built artefact.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
reference legs may import this module, and only as the checker or the
timed reference arm — never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdim3ref.so")

U64P = C.POINTER(C.c_uint64)

# test_consts(), P/tests/support.hpp:27-38
TEST_CONSTS = dict(t_seqR=0.9e-9, t_randR=140e-9, t_randRW=140e-9, t_hash=440e-9,
                   t_map=330e-9, t_ECs=11e-9, t_ECd=1.2e-9, w=256)

STRATEGY = {"auto": 0, "classical": 1, "hybrid": 2, "sparse": 3, "dense": 4}
DENSE_MODE = {"cost_based": 0, "force_wide": 1, "force_probe": 2}


class Consts(C.Structure):
    _fields_ = [(k, C.c_double) for k in
                ("t_seqR", "t_randR", "t_randRW", "t_hash", "t_map", "t_ECs", "t_ECd")] + \
               [("w", C.c_uint32)]


def make_consts(d=None) -> Consts:
    d = dict(TEST_CONSTS if d is None else d)
    return Consts(**d)


class OrcOpts(C.Structure):
    _fields_ = [("force", C.c_int32), ("dense_mode", C.c_int32), ("count_only", C.c_int32),
                ("natural_keys_auto", C.c_int32), ("threads", C.c_int32), ("pad", C.c_int32)]


_ORC_U64 = ["r_rows", "s_rows", "out_j_estimate"]
_ORC_U64B = ["out_p", "pairs_sparse", "pairs_dense", "sparse_z", "dense_z", "f2_evaluations",
             "dropped_r", "x_card", "y_card", "z_card", "r_nnz", "s_nnz", "sparse_nnz", "out_j",
             "panel_bytes", "spa_inner_count", "dense_wide_encounters",
             "dense_probe_encounters", "dense_blocks_checked", "dense_probes_done",
             "dense_row_bitmaps_built", "x_live", "checksum_sum", "checksum_xor"]


class OrcReport(C.Structure):
    _fields_ = [("swapped", C.c_int32), ("f1_classical", C.c_int32), ("natural_x", C.c_int32),
                ("natural_y", C.c_int32), ("natural_z", C.c_int32), ("pad", C.c_int32)] + \
               [(k, C.c_uint64) for k in _ORC_U64] + [("f1", C.c_double)] + \
               [(k, C.c_uint64) for k in _ORC_U64B]


_REF_U64 = ["out_p", "pairs_classical", "pairs_sparse", "pairs_dense", "sparse_z", "dense_z",
            "f2_evaluations", "dropped_r", "intermediate_pairs", "x_card", "y_card", "z_card",
            "panel_bytes", "peak_bytes", "spa_inner_count", "dense_wide_encounters",
            "dense_probe_encounters", "dense_blocks_checked", "dense_probes_done",
            "dense_row_bitmaps_built"]
_REF_MS = ["ms_total", "ms_estimate", "ms_map", "ms_csr", "ms_partition", "ms_sparse",
           "ms_dense", "ms_classical"]


class RefReport(C.Structure):
    _fields_ = [("strategy", C.c_char * 16), ("swapped", C.c_int32), ("materialized", C.c_int32),
                ("r_rows", C.c_uint64), ("s_rows", C.c_uint64), ("out_j_estimate", C.c_uint64),
                ("f1", C.c_double)] + [(k, C.c_uint64) for k in _REF_U64] + \
               [(k, C.c_double) for k in _REF_MS] + \
               [("checksum_sum", C.c_uint64), ("checksum_xor", C.c_uint64),
                ("spa_allocations", C.c_uint64), ("spa_entries", C.c_uint64)]


class RefPipeline(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in
                ("x_card", "y_card", "z_card", "r_nnz", "s_nnz", "out_j", "dropped_r",
                 "dense_z", "sparse_z", "sparse_nnz")] + \
               [("natural_x", C.c_int32), ("natural_y", C.c_int32), ("natural_z", C.c_int32),
                ("pad", C.c_int32)]


def _struct_dict(s) -> dict:
    out = {}
    for name, _ in s._fields_:
        if name == "pad":
            continue
        v = getattr(s, name)
        out[name] = v.decode() if isinstance(v, bytes) else v
    return out


_orc = None
_ref = None


def orc_lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"oracle not built: {ORACLE_SO} (run `make -C oracle oracle`)")
        lib = C.CDLL(ORACLE_SO)
        lib.orc_gen.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_uint64, U64P, U64P]
        lib.orc_cfg_rows.argtypes = [C.c_int]
        lib.orc_cfg_rows.restype = C.c_uint64
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_join_project.argtypes = [U64P, U64P, C.c_uint64, U64P, U64P, C.c_uint64,
                                         C.POINTER(Consts), C.POINTER(OrcOpts),
                                         C.POINTER(OrcReport), U64P, C.c_uint64, U64P,
                                         C.c_void_p]
        lib.orc_mix64.argtypes = [C.c_uint64]
        lib.orc_mix64.restype = C.c_uint64
        lib.orc_f3_threshold.argtypes = [C.c_uint32, C.c_uint32, C.POINTER(Consts)]
        lib.orc_f3_threshold.restype = C.c_uint32
        lib.orc_f3.argtypes = [C.c_double, C.c_double, C.c_uint32, C.POINTER(Consts)]
        lib.orc_f3.restype = C.c_double
        lib.orc_f1.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(Consts)]
        lib.orc_f1.restype = C.c_double
        lib.orc_check_nonsimd.argtypes = [C.c_double] * 3
        lib.orc_check_nonsimd.restype = C.c_double
        lib.orc_check_simd.argtypes = [C.c_double] * 3 + [C.c_uint32]
        lib.orc_check_simd.restype = C.c_double
        lib.orc_mx_bucket_key.argtypes = [C.c_uint32]
        lib.orc_mx_bucket_key.restype = C.c_uint32
        lib.orc_mz_bucket_index.argtypes = [C.c_uint32, C.c_uint32]
        lib.orc_mz_bucket_index.restype = C.c_uint32
        lib.orc_estimate_out_j_raw.argtypes = [U64P, C.c_uint64, U64P, C.c_uint64]
        lib.orc_estimate_out_j_raw.restype = C.c_uint64
        _orc = lib
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"reference not built: {REF_SO} (run `make -C oracle ref` "
                               "where /root/reference exists)")
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_join_project.argtypes = [U64P, U64P, C.c_uint64, U64P, U64P, C.c_uint64,
                                         C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                         C.POINTER(Consts), C.POINTER(RefReport), U64P, U64P,
                                         C.c_uint64]
        lib.ref_pipeline.argtypes = [U64P, U64P, C.c_uint64, U64P, U64P, C.c_uint64,
                                     C.POINTER(Consts), C.POINTER(RefPipeline), U64P, C.c_uint64]
        lib.ref_set_checksum.argtypes = [U64P, U64P, C.c_uint64, U64P, U64P, C.c_uint64, C.c_int,
                                         C.c_uint64, U64P, U64P, U64P, C.c_uint64, C.c_uint64,
                                         U64P, U64P, U64P]
        lib.ref_f3_threshold.argtypes = [C.c_uint32, C.c_uint32, C.POINTER(Consts),
                                         C.POINTER(C.c_uint32)]
        lib.ref_timed_sample.argtypes = [U64P, U64P, C.c_uint64, U64P, U64P, C.c_uint64,
                                         C.POINTER(Consts), C.c_int, C.c_uint64, C.c_uint64,
                                         C.POINTER(C.c_double), C.POINTER(C.c_double), U64P, U64P]
        lib.ref_mx_bucket_key.argtypes = [C.c_uint32]
        lib.ref_mx_bucket_key.restype = C.c_uint32
        lib.ref_mz_bucket_index.argtypes = [C.c_uint32, C.c_uint32]
        lib.ref_mz_bucket_index.restype = C.c_uint32
        _ref = lib
    return _ref


def _p(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(U64P)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


@dataclass
class Table:
    left: np.ndarray
    right: np.ndarray

    def __len__(self):
        return int(self.left.shape[0])


def cfg_rows(cfg: int) -> int:
    return int(orc_lib().orc_cfg_rows(cfg))


def gen(cfg: int, side: int, lo: int = 0, hi: int | None = None) -> Table:
    """Convention G rows [lo, hi) of side 0 (R) or 1 (S) — SURVEY Appendix A."""
    n = cfg_rows(cfg)
    hi = n if hi is None else hi
    left = np.empty(hi - lo, dtype=np.uint64)
    right = np.empty(hi - lo, dtype=np.uint64)
    rc = orc_lib().orc_gen(cfg, side, lo, hi, _p(left), _p(right))
    if rc:
        raise RuntimeError(orc_lib().orc_last_error().decode())
    return Table(left, right)


def orc_join_project(r: Table, s: Table, force="hybrid", count_only=True, dense_mode="cost_based",
                     natural_keys_auto=True, threads=1, consts=None, want_pairs=False,
                     pairs_cap=None):
    lib = orc_lib()
    rl, rr, sl, sr = (_u64(a) for a in (r.left, r.right, s.left, s.right))
    c = make_consts(consts)
    o = OrcOpts(STRATEGY[force], DENSE_MODE[dense_mode], int(count_only),
                int(natural_keys_auto), threads, 0)
    rep = OrcReport()
    pairs = None
    n_out = C.c_uint64(0)
    if want_pairs:
        cap = pairs_cap if pairs_cap is not None else len(r) * max(len(s), 1) + 1
        cap = min(cap, 50_000_000)
        pairs = np.zeros(2 * cap, dtype=np.uint64)
        rc = lib.orc_join_project(_p(rl), _p(rr), len(rl), _p(sl), _p(sr), len(sl), C.byref(c),
                                  C.byref(o), C.byref(rep), _p(pairs), cap, C.byref(n_out), None)
    else:
        rc = lib.orc_join_project(_p(rl), _p(rr), len(rl), _p(sl), _p(sr), len(sl), C.byref(c),
                                  C.byref(o), C.byref(rep), None, 0, None, None)
    if rc:
        raise ConfigErrorLike(rc, lib.orc_last_error().decode())
    d = _struct_dict(rep)
    if want_pairs:
        d["pairs"] = pairs[: 2 * n_out.value].reshape(-1, 2)
    return d


class ConfigErrorLike(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"status {status}: {msg}")
        self.status = status


def ref_join_project(r: Table, s: Table, force="hybrid", threads=1, count_only=True,
                     dense_mode="cost_based", budget_bytes=0, natural_keys_auto=True,
                     consts=None, want_pairs=False):
    lib = ref_lib()
    rl, rr, sl, sr = (_u64(a) for a in (r.left, r.right, s.left, s.right))
    c = make_consts(consts)
    rep = RefReport()
    if want_pairs and not count_only:
        cap = 50_000_000
        ox = np.zeros(cap, dtype=np.uint64)
        oz = np.zeros(cap, dtype=np.uint64)
        rc = lib.ref_join_project(_p(rl), _p(rr), len(rl), _p(sl), _p(sr), len(sl),
                                  STRATEGY[force], threads, int(count_only), DENSE_MODE[dense_mode],
                                  budget_bytes, int(natural_keys_auto), C.byref(c), C.byref(rep),
                                  _p(ox), _p(oz), cap)
    else:
        rc = lib.ref_join_project(_p(rl), _p(rr), len(rl), _p(sl), _p(sr), len(sl),
                                  STRATEGY[force], threads, int(count_only), DENSE_MODE[dense_mode],
                                  budget_bytes, int(natural_keys_auto), C.byref(c), C.byref(rep),
                                  None, None, 0)
    if rc:
        raise ConfigErrorLike(rc, lib.ref_last_error().decode())
    d = _struct_dict(rep)
    if want_pairs and not count_only:
        n = min(d["out_p"], cap)
        d["pairs"] = np.stack([ox[:n], oz[:n]], axis=1)
    return d


def ref_pipeline(r: Table, s: Table, consts=None):
    lib = ref_lib()
    rl, rr, sl, sr = (_u64(a) for a in (r.left, r.right, s.left, s.right))
    c = make_consts(consts)
    out = RefPipeline()
    cap = 1 << 24
    dz = np.zeros(cap, dtype=np.uint64)
    rc = lib.ref_pipeline(_p(rl), _p(rr), len(rl), _p(sl), _p(sr), len(sl), C.byref(c),
                          C.byref(out), _p(dz), cap)
    if rc:
        raise ConfigErrorLike(rc, lib.ref_last_error().decode())
    d = _struct_dict(out)
    d["dense_z_raw"] = dz[: d["dense_z"]].copy()
    return d


AGG = {"sum": 0, "count": 1, "min": 2, "max": 3, "avg": 4}
COMBINE = {"multiply": 0, "add": 1, "abs_diff": 2, "left": 3, "right": 4}


def ref_join_aggregate(r: Table, s: Table, rv, sv, combine="multiply", agg="sum", force="hybrid",
                       count_only=False, consts=None):
    """dim3::join_aggregate_both through the reference library: the report
    and, unless count_only, {(raw x, raw z): value}."""
    lib = ref_lib()
    rl, rr, sl, sr = (_u64(a) for a in (r.left, r.right, s.left, s.right))
    rv = np.ascontiguousarray(rv, dtype=np.float64)
    sv = np.ascontiguousarray(sv, dtype=np.float64)
    c = make_consts(consts)
    rep = RefReport()
    cap = max(1, len(rl) * max(1, len(sl)))
    cap = min(cap, 20_000_000)
    ox = np.zeros(cap, dtype=np.uint64)
    oz = np.zeros(cap, dtype=np.uint64)
    ov = np.zeros(cap, dtype=np.float64)
    fn = lib.ref_join_aggregate
    D = C.POINTER(C.c_double)
    fn.argtypes = [U64P, U64P, D, C.c_uint64, U64P, U64P, D, C.c_uint64, C.c_int, C.c_int,
                   C.c_int, C.c_int, C.c_void_p, C.c_void_p, U64P, U64P, D, C.c_uint64]
    rc = fn(_p(rl), _p(rr), rv.ctypes.data_as(D), len(rl), _p(sl), _p(sr), sv.ctypes.data_as(D),
            len(sl), COMBINE[combine], AGG[agg], STRATEGY[force], int(count_only), C.byref(c),
            C.byref(rep), _p(ox), _p(oz), ov.ctypes.data_as(D), cap)
    if rc:
        raise ConfigErrorLike(rc, lib.ref_last_error().decode())
    d = _struct_dict(rep)
    if not count_only:
        n = min(d["out_p"], cap)
        d["cells"] = {(int(a), int(b)): float(v) for a, b, v in zip(ox[:n], oz[:n], ov[:n])}
        d["order"] = [(int(a), int(b)) for a, b in zip(ox[:n], oz[:n])]
    return d


def oracle_aggregate(r: Table, s: Table, rv, sv, combine="multiply", agg="sum"):
    """Brute-force restatement of join_aggregate_both's semantics for small
    inputs (P/tests/test_engine.cpp:42-86 OracleCell): {(x, z): value} with the
    accumulation in the reference's order (R rows of x in input order, S rows
    of y in input order). Pure Python; a checker only."""
    import math
    by_y = {}
    for j, (z, y) in enumerate(zip(np.asarray(s.left).tolist(), np.asarray(s.right).tolist())):
        by_y.setdefault(y, []).append((z, float(sv[j])))
    rows_by_x = {}
    for i, (x, y) in enumerate(zip(np.asarray(r.left).tolist(), np.asarray(r.right).tolist())):
        rows_by_x.setdefault(x, []).append((y, float(rv[i])))
    comb = {"multiply": lambda a, b: a * b, "add": lambda a, b: a + b,
            "abs_diff": lambda a, b: math.fabs(a - b), "left": lambda a, b: a,
            "right": lambda a, b: b}[combine]
    cells = {}
    for x, rows in rows_by_x.items():
        for y, v in rows:
            for z, u in by_y.get(y, ()):
                cv = comb(v, u)
                c = cells.get((x, z))
                if c is None:
                    cells[(x, z)] = [0.0 if agg == "count" else cv, 1]
                else:
                    if agg in ("sum", "avg"):
                        c[0] = c[0] + cv
                    elif agg == "min":
                        c[0] = cv if cv < c[0] else c[0]
                    elif agg == "max":
                        c[0] = cv if c[0] < cv else c[0]
                    c[1] += 1
    out = {}
    for k, (acc, cnt) in cells.items():
        out[k] = float(cnt) if agg == "count" else (acc / cnt if agg == "avg" else acc)
    return out


def ref_map_tables(r: Table, s: Table, skip=None):
    """dim3::map_tables through the reference library. skip = None: the
    engine's natural-key detection with fallback; else (x, y, z) SkipFlags."""
    lib = ref_lib()
    rl, rr, sl, sr = (_u64(a) for a in (r.left, r.right, s.left, s.right))
    nr, ns = len(rl), len(sl)
    ra, rb, rk = (np.zeros(max(nr, 1), np.uint32) for _ in range(3))
    sa, sb = (np.zeros(max(ns, 1), np.uint32) for _ in range(2))
    st = np.zeros(6, np.uint64)
    U32P = C.POINTER(C.c_uint32)
    fn = lib.ref_map_tables
    fn.argtypes = [U64P, U64P, C.c_uint64, U64P, U64P, C.c_uint64, C.c_int, C.c_int, C.c_int,
                   C.c_int, U32P, U32P, U32P, U32P, U32P, U64P]
    sk = skip or (0, 0, 0)
    rc = fn(_p(rl), _p(rr), nr, _p(sl), _p(sr), ns, int(skip is None), int(sk[0]), int(sk[1]),
            int(sk[2]), ra.ctypes.data_as(U32P), rb.ctypes.data_as(U32P), sa.ctypes.data_as(U32P),
            sb.ctypes.data_as(U32P), rk.ctypes.data_as(U32P), _p(st))
    if rc:
        raise ConfigErrorLike(rc, lib.ref_last_error().decode())
    kept = int(st[0])
    return {"r_a": ra[:kept].copy(), "r_b": rb[:kept].copy(), "s_a": sa[:ns].copy(),
            "s_b": sb[:ns].copy(), "r_kept": rk[:int(st[5])].copy(), "dropped_r": int(st[1]),
            "x_card": int(st[2]), "y_card": int(st[3]), "z_card": int(st[4])}


def ref_pipeline_split(r: Table, s: Table, consts=None):
    """ref_pipeline's statistics and dense/sparse split without building the
    panel (F2Evaluator decisions only)."""
    lib = ref_lib()
    rl, rr, sl, sr = (_u64(a) for a in (r.left, r.right, s.left, s.right))
    c = make_consts(consts)
    out = RefPipeline()
    fn = lib.ref_pipeline_split
    fn.argtypes = [U64P, U64P, C.c_uint64, U64P, U64P, C.c_uint64, C.c_void_p, C.c_void_p]
    rc = fn(_p(rl), _p(rr), len(rl), _p(sl), _p(sr), len(sl), C.byref(c), C.byref(out))
    if rc:
        raise ConfigErrorLike(rc, lib.ref_last_error().decode())
    return _struct_dict(out)


def ref_set_checksum(r: Table, s: Table, threads=8, rows_per_slice=1024, block_width=0,
                     n_blocks=0):
    lib = ref_lib()
    rl, rr, sl, sr = (_u64(a) for a in (r.left, r.right, s.left, s.right))
    cnt, sm, xr = C.c_uint64(), C.c_uint64(), C.c_uint64()
    if n_blocks:
        bc = np.zeros(n_blocks, np.uint64)
        bs = np.zeros(n_blocks, np.uint64)
        bx = np.zeros(n_blocks, np.uint64)
        rc = lib.ref_set_checksum(_p(rl), _p(rr), len(rl), _p(sl), _p(sr), len(sl), threads,
                                  rows_per_slice, C.byref(cnt), C.byref(sm), C.byref(xr),
                                  block_width, n_blocks, _p(bc), _p(bs), _p(bx))
    else:
        rc = lib.ref_set_checksum(_p(rl), _p(rr), len(rl), _p(sl), _p(sr), len(sl), threads,
                                  rows_per_slice, C.byref(cnt), C.byref(sm), C.byref(xr), 1, 0,
                                  None, None, None)
    if rc:
        raise ConfigErrorLike(rc, lib.ref_last_error().decode())
    d = dict(count=cnt.value, sum=sm.value, xor=xr.value)
    if n_blocks:
        d.update(blk_count=bc, blk_sum=bs, blk_xor=bx)
    return d


def ref_timed_sample(r: Table, s: Table, threads: int, x_lo: int, x_hi: int, consts=None):
    """Reference prep on the whole tables + reference kernels on x rows [x_lo, x_hi)."""
    lib = ref_lib()
    rl, rr, sl, sr = (_u64(a) for a in (r.left, r.right, s.left, s.right))
    c = make_consts(consts)
    tp, tk = C.c_double(), C.c_double()
    xr, pr = C.c_uint64(), C.c_uint64()
    rc = lib.ref_timed_sample(_p(rl), _p(rr), len(rl), _p(sl), _p(sr), len(sl), C.byref(c),
                              threads, x_lo, x_hi, C.byref(tp), C.byref(tk), C.byref(xr),
                              C.byref(pr))
    if rc:
        raise ConfigErrorLike(rc, lib.ref_last_error().decode())
    return dict(sec_prep=tp.value, sec_kernels=tk.value, x_rows=xr.value, pairs=pr.value)


def mix64(x: int) -> int:
    m = (1 << 64) - 1
    x &= m
    x ^= x >> 30
    x = (x * 0xbf58476d1ce4e5b9) & m
    x ^= x >> 27
    x = (x * 0x94d049bb133111eb) & m
    x ^= x >> 31
    return x


def pair_hash_np(x: np.ndarray, z: np.ndarray) -> np.ndarray:
    """h(x,z) = mix64(mix64(x) ^ z), vectorised (uint64 wraps)."""
    def m(v):
        v = v ^ (v >> np.uint64(30))
        v = v * np.uint64(0xbf58476d1ce4e5b9)
        v = v ^ (v >> np.uint64(27))
        v = v * np.uint64(0x94d049bb133111eb)
        v = v ^ (v >> np.uint64(31))
        return v
    with np.errstate(over="ignore"):
        return m(m(x.astype(np.uint64)) ^ z.astype(np.uint64))


def set_fingerprint(x: np.ndarray, z: np.ndarray):
    h = pair_hash_np(x, z)
    return int(h.size), int(np.bitwise_xor.reduce(h)) if h.size else 0, \
        int(h.sum(dtype=np.uint64)) if h.size else 0
