"""Multi-GPU host plumbing for the x-sharded join_project.

The library runs one rank of a sharded job when its context has an exchange
(``Context.set_nccl`` or ``Context.set_exchange``): each rank passes its
x-shard of R and the whole S, and ``d3g_join_project`` performs the few
collectives the global decisions need (column maxima and natural-key tests,
the per-y raw R counts behind f1, the m_x histogram, dR(y), nnz / live x, the
final tallies; see include/dim3_b200.h and csrc/exchange.cuh). Partitioning R
by x is intersection-free (the reference's own x chunking,
P/include/dim3/common.hpp:130-155), so no pair ever crosses ranks.

On GPUs the transport is NCCL over NVLink (``Context.set_nccl``). The
host-callback transport takes any object with ``__call__(op, arr)`` that
performs the collective in place on a numpy array:

* ``TorchExchange``   -- torch.distributed (gloo on CPU tensors): the
  multi-process form, covered by the world-size-2 gloo tests;
* ``ThreadExchange``  -- ranks as threads of one process (a barrier): used to
  run an N-rank job on ONE GPU for parity tests. Only host threads wait on
  one another; no kernel waits for another rank's kernel;
* ``RecordingExchange`` / ``ReplayExchange`` -- record a rank's collective
  results in a threaded run, then replay them so that rank can be re-run
  ALONE on the GPU and timed without contention (scripts/shard_projection.py).

Sharding helpers split R by contiguous x ranges (natural keys) or by a hash of
the raw x value (dictionary keys: local dictionaries stay disjoint).
"""
from __future__ import annotations

import threading

import numpy as np

from .engine import EX_GATHER, EX_MAX_U64, EX_SUM_U32, EX_SUM_U64

U64_MASK = (1 << 64) - 1


def _fold(op: int, parts: list[np.ndarray]) -> np.ndarray:
    if op == EX_MAX_U64:
        return np.maximum.reduce(parts)
    out = parts[0].copy()
    for p in parts[1:]:
        out += p  # modular (uint64 / uint32 wrap like the device sums)
    return out


class ThreadExchange:
    """Collectives among `nranks` threads of one process. Each rank uses
    ``rank_fn(r)`` as its exchange callback."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self.barrier = threading.Barrier(nranks)
        self.slots: list = [None] * nranks

    def rank_fn(self, rank: int):
        def fn(op: int, arr: np.ndarray):
            if op == EX_GATHER:
                nb = arr.size // self.nranks
                self.slots[rank] = arr[rank * nb:(rank + 1) * nb].copy()
                self.barrier.wait()
                for q in range(self.nranks):
                    arr[q * nb:(q + 1) * nb] = self.slots[q]
            else:
                self.slots[rank] = arr.copy()
                self.barrier.wait()
                arr[:] = _fold(op, list(self.slots))
            self.barrier.wait()  # slots are reused by the next collective
        return fn


class TorchExchange:
    """Collectives over a torch.distributed process group (gloo / CPU)."""

    def __init__(self, dist, group=None):
        self.dist, self.group = dist, group
        self.nranks = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def __call__(self, op: int, arr: np.ndarray):
        import torch
        d = self.dist
        if op == EX_GATHER:
            nb = arr.size // self.nranks
            mine = torch.from_numpy(arr[self.rank * nb:(self.rank + 1) * nb].copy())
            outs = [torch.empty_like(mine) for _ in range(self.nranks)]
            d.all_gather(outs, mine, group=self.group)
            for q, t in enumerate(outs):
                arr[q * nb:(q + 1) * nb] = t.numpy()
            return
        if op == EX_MAX_U64:
            # torch has no uint64 max: values here are maxima / flags < 2^63
            t = torch.from_numpy(arr.astype(np.int64))
            d.all_reduce(t, op=d.ReduceOp.MAX, group=self.group)
            arr[:] = t.numpy().astype(np.uint64)
            return
        # sums: int64 two's complement wraps exactly like uint64 (mod 2^64)
        t = torch.from_numpy(arr.astype(np.int64) if op == EX_SUM_U64 else arr.astype(np.int64))
        d.all_reduce(t, op=d.ReduceOp.SUM, group=self.group)
        res = t.numpy()
        arr[:] = (res.astype(np.uint64) if op == EX_SUM_U64
                  else (res & 0xFFFFFFFF).astype(np.uint32))


class RecordingExchange:
    """Wraps an exchange and records every collective's result, in order."""

    def __init__(self, inner):
        self.inner, self.log = inner, []

    def __call__(self, op: int, arr: np.ndarray):
        self.inner(op, arr)
        self.log.append((op, arr.copy()))


class ReplayExchange:
    """Returns recorded results in order (a rank re-run alone, same inputs)."""

    def __init__(self, log):
        self.log, self.i = log, 0

    def __call__(self, op: int, arr: np.ndarray):
        rop, val = self.log[self.i]
        self.i += 1
        if rop != op or val.shape != arr.shape:
            raise RuntimeError("replayed exchange diverged from the recorded run")
        arr[:] = val

    def rewind(self):
        self.i = 0


def x_range_bounds(x_card: int, rank: int, nranks: int):
    """Contiguous raw-x range [lo, hi) of a rank (natural keys)."""
    return x_card * rank // nranks, x_card * (rank + 1) // nranks


def shard_mask(x: np.ndarray, rank: int, nranks: int, x_card: int | None = None) -> np.ndarray:
    """Rows of R owned by `rank`: contiguous ranges when x_card is given
    (natural keys), else a hash of the raw value (mix64 mod nranks)."""
    x = np.asarray(x, dtype=np.uint64)
    if x_card is not None:
        lo, hi = x_range_bounds(x_card, rank, nranks)
        return (x >= lo) & (x < hi)
    h = x.copy()
    h ^= h >> np.uint64(30)
    h *= np.uint64(0xBF58476D1CE4E5B9)
    h ^= h >> np.uint64(27)
    h *= np.uint64(0x94D049BB133111EB)
    h ^= h >> np.uint64(31)
    return (h % np.uint64(nranks)) == np.uint64(rank)
