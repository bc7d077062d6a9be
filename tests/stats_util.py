"""Host-side restatement (numpy) of the quantities the f2 decision consumes,
for tests of the policy entry point and of the sharded (all-reduced) path.

Mirrors map_with_fallback / map_tables (P/src/engine.cpp:25-50,
P/src/mapping.cpp:281-420), build_csr's duplicate collapse
(P/src/relation.cpp:245-256) and compute_degree_stats
(P/src/costmodel.cpp:425-438) on raw u64 tables."""
import numpy as np


def detect_natural(col: np.ndarray) -> bool:
    n = col.size
    if n == 0:
        return False
    bound = 2.0 * float(n)
    samples = min(n, 4096)
    stride = max(n // samples, 1)
    idx = np.minimum(np.arange(samples, dtype=np.int64) * stride, n - 1)
    return bool((col[idx].astype(np.float64) < bound).all())


def mapping_plan(r, s):
    """(skip_x, skip_y, skip_z, swapped) as join_project resolves them."""
    rl, rr = (np.asarray(a, np.uint64) for a in r)
    sl, sr = (np.asarray(a, np.uint64) for a in s)
    swapped = sl.size > rl.size
    if swapped:
        rl, rr, sl, sr = sl, sr, rl, rr
    sx = detect_natural(rl)
    sy = detect_natural(rr) and detect_natural(sr)
    sz = detect_natural(sl)
    fits = lambda c: c.size == 0 or int(c.max()) < (1 << 32)  # noqa: E731
    if (sy and not (fits(rr) and fits(sr))) or (sz and not fits(sl)) or (sx and not fits(rl)):
        sx = sy = sz = False
    return sx, sy, sz, (rl, rr, sl, sr), swapped


def f2_inputs(r, s, x_filter=None):
    """Degree histograms and global sizes. x_filter(x_raw) -> bool restricts
    the R rows (an x shard); cards stay global (as after an all-reduce)."""
    sx, sy, sz, (rl, rr, sl, sr), swapped = mapping_plan(r, s)
    # y filter (dictionary y only): keep R rows whose y occurs in S
    if sy:
        keep = np.ones(rl.size, bool)
        y_card = int(max(int(sr.max()) + 1 if sr.size else 0, int(rr.max()) + 1 if rr.size else 0))
    else:
        keep = np.isin(rr, sr)
        y_card = int(np.unique(sr).size)
    x_card = (int(rl.max()) + 1 if rl.size else 0) if sx else int(np.unique(rl[keep]).size)
    z_card = (int(sl.max()) + 1 if sl.size else 0) if sz else int(np.unique(sl).size)
    rk_l, rk_r = rl[keep], rr[keep]
    # distinct tuples (build_csr collapses duplicates)
    rpairs = np.unique(np.stack([rk_l, rk_r], 1), axis=0) if rk_l.size else np.zeros((0, 2), np.uint64)
    spairs = np.unique(np.stack([sl, sr], 1), axis=0) if sl.size else np.zeros((0, 2), np.uint64)
    if x_filter is not None and rpairs.size:
        rpairs = rpairs[np.array([x_filter(int(v)) for v in rpairs[:, 0]], bool)]
    xs, mx = np.unique(rpairs[:, 0], return_counts=True) if rpairs.size else (np.zeros(0), np.zeros(0, np.int64))
    zs, mz = np.unique(spairs[:, 0], return_counts=True) if spairs.size else (np.zeros(0), np.zeros(0, np.int64))
    mx_hist = np.bincount(mx, minlength=1).astype(np.uint64)
    mz_hist = np.bincount(mz, minlength=1).astype(np.uint64)
    mx_hist[0] = 0
    mz_hist[0] = z_card - zs.size  # gap codes (m_z = 0)
    ry, dr = np.unique(rpairs[:, 1], return_counts=True) if rpairs.size else (np.zeros(0), np.zeros(0))
    sy_, ds = np.unique(spairs[:, 1], return_counts=True) if spairs.size else (np.zeros(0), np.zeros(0))
    dmap = dict(zip(sy_.tolist(), ds.tolist()))
    out_j = int(sum(int(c) * int(dmap.get(y, 0)) for y, c in zip(ry.tolist(), dr.tolist())))
    return {"mx_hist": mx_hist, "mz_hist": mz_hist, "x_card": x_card, "y_card": y_card,
            "z_card": z_card, "out_j": out_j, "dr": dict(zip(ry.tolist(), dr.tolist())),
            "m_z_by_raw": dict(zip(zs.tolist(), mz.tolist())), "swapped": swapped}
