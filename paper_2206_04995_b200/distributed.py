"""Multi-GPU host logic (one process per GPU, torch.distributed for plumbing).

The path shards naturally by x: partitioning R by x is
intersection-free (P/src/sparsebmm.cpp:79-104 chunks threads the same way),
so no cross-GPU dedup exists. Two exchange steps remain:

1. f2 inputs. When each rank holds only its x-shard of R, the dense/sparse
   decision (P/src/costmodel.cpp:515-586) must still see GLOBAL statistics:
   the m_x histogram (sum), dR(y) (sum, for OUT_J = sum_y dR*dS), r_nnz
   (sum), x_card (max under natural keys, sum of disjoint local dictionaries
   otherwise). S is replicated (broadcast once), so m_z / dS / z_card /
   y_card are already global. ``allreduce_f2_inputs`` performs the
   all-reduces; every rank then evaluates the identical decision table with
   ``d3g_f2_decide``.
2. Results: per-rank pair counts and (sum, xor) fingerprints are combined
   with ``reduce_tally``.

With the single-call API (``EngineConfig.shard_index/shard_count``) every
rank receives full R and S (NCCL broadcast), computes the statistics
redundantly and runs the kernels on its x shard only, so step 1 is not
needed; the functions here serve the partitioned-input deployment and are
covered by the gloo tests.
"""
from __future__ import annotations

import numpy as np

U64_MASK = (1 << 64) - 1


def _to_i64(v: int) -> int:
    v &= U64_MASK
    return v - (1 << 64) if v >= (1 << 63) else v


def _pad_allreduce(arr: np.ndarray, dist, group=None, op=None):
    import torch
    n = torch.tensor([arr.size], dtype=torch.int64)
    dist.all_reduce(n, op=dist.ReduceOp.MAX, group=group)
    t = torch.zeros(int(n.item()), dtype=torch.int64)
    t[: arr.size] = torch.from_numpy(arr.astype(np.int64))
    dist.all_reduce(t, op=op or dist.ReduceOp.SUM, group=group)
    return t.numpy().astype(np.uint64)


def allreduce_f2_inputs(local: dict, dist, group=None, natural_x: bool = True) -> dict:
    """local: {"mx_hist", "dr" (array over y codes), "x_card", "r_nnz"} of this
    rank's R shard plus the replicated S-side {"mz_hist", "ds", "y_card",
    "z_card"}. Returns the global inputs of d3g_f2_decide."""
    import torch
    mx = _pad_allreduce(np.asarray(local["mx_hist"], np.uint64), dist, group)
    mx[0] = 0
    dr = _pad_allreduce(np.asarray(local["dr"], np.uint64), dist, group)
    sc = torch.tensor([int(local["x_card"]), int(local["r_nnz"])], dtype=torch.int64)
    xc = sc[:1].clone()
    dist.all_reduce(xc, op=dist.ReduceOp.MAX if natural_x else dist.ReduceOp.SUM, group=group)
    nnz = sc[1:].clone()
    dist.all_reduce(nnz, op=dist.ReduceOp.SUM, group=group)
    ds = np.asarray(local["ds"], np.uint64)
    n = min(dr.size, ds.size)
    out_j = int(np.dot(dr[:n].astype(object), ds[:n].astype(object))) if n else 0
    return {"mx_hist": mx, "mz_hist": np.asarray(local["mz_hist"], np.uint64),
            "x_card": int(xc.item()), "y_card": int(local["y_card"]),
            "z_card": int(local["z_card"]), "out_j": min(out_j, U64_MASK),
            "r_nnz": int(nnz.item())}


def reduce_tally(count: int, csum: int, cxor: int, dist, group=None):
    """Global (count, sum mod 2^64, xor) of per-rank results (intersection-free
    shards: plain sums, no dedup)."""
    import torch
    t = torch.tensor([_to_i64(count), _to_i64(csum)], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    world = dist.get_world_size(group)
    xs = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(xs, torch.tensor([_to_i64(cxor)], dtype=torch.int64), group=group)
    x = 0
    for v in xs:
        x ^= int(v.item()) & U64_MASK
    return int(t[0].item()) & U64_MASK, int(t[1].item()) & U64_MASK, x


def x_shard_bounds(x_card: int, rank: int, world: int):
    """Contiguous x-code range of a rank (natural keys)."""
    return x_card * rank // world, x_card * (rank + 1) // world
