// The z-split S side of a sharded join_project.
//
// A sharded job partitions R by x (intersection-free: the reference's own
// thread chunks, P/src/sparsebmm.cpp:79-104), so every rank needs every dense
// z row. Building the S side on every rank would replicate the S-by-z CSR,
// the dense lists, the hot records and the cold CSR, the part that does not
// shrink with the rank count. Instead rank q builds them for the z codes
// [z_lo, z_hi) only (dense rows = global rows [row_lo, row_lo + D_q), rank
// blocks concatenated in rank order) and the ranks exchange:
//   * all-reduce: the m_z histogram, dS(y), the per-degree join sizes, the
//     dense-row class counts (inputs of the global f2 / K / plan decisions);
//   * all-gather: per dense row the hot mask hz, the hot record and count
//     word, the z code and the folded-sparse flag; the long rows' list tails;
//     the cold CSR's (variant, part, y) counts and 16-byte records, merged
//     here into the one y-major layout the cold kernels stream.
// The gathers are one ncclAllGather each over NVLink (exchange.cuh).
#pragma once

#include "denseec_cold.cuh"

namespace d3g {

// This rank's S tuples: z codes in [z_lo, z_hi), compacted as (z - z_lo, y)
// (their order is irrelevant: the CSR build sorts). Tiles of 256 x 8 codes;
// one cursor atomic per tile (a per-warp atomic serialised the pass: 5 ms for
// cfg5's 200M codes).
constexpr int kZcThreads = 256, kZcPer = 8;
__global__ void __launch_bounds__(kZcThreads)
zrange_compact_kernel(const uint32_t* __restrict__ sz, const uint32_t* __restrict__ sy, uint64_t n,
                      uint32_t z_lo, uint32_t z_hi, uint32_t* __restrict__ oz,
                      uint32_t* __restrict__ oy, unsigned long long* __restrict__ cursor) {
  __shared__ uint32_t wsum[kZcThreads / 32];
  __shared__ unsigned long long base_s;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  constexpr uint64_t kTile = (uint64_t)kZcThreads * kZcPer;
  for (uint64_t t0 = (uint64_t)blockIdx.x * kTile; t0 < n; t0 += (uint64_t)gridDim.x * kTile) {
    uint32_t z[kZcPer], cnt = 0, inm = 0;
#pragma unroll
    for (int k = 0; k < kZcPer; ++k) {
      const uint64_t i = t0 + threadIdx.x + (uint64_t)k * kZcThreads;
      z[k] = i < n ? sz[i] : z_hi;
      if (z[k] >= z_lo && z[k] < z_hi) {
        inm |= 1u << k;
        ++cnt;
      }
    }
    const uint32_t incl = warp_incl_scan(cnt);
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint32_t v = lane < kZcThreads / 32 ? wsum[lane] : 0u;
      const uint32_t vi = warp_incl_scan(v);
      if (lane < kZcThreads / 32) wsum[lane] = vi - v;
      if (lane == kZcThreads / 32 - 1) base_s = vi ? atomicAdd(cursor, (unsigned long long)vi) : 0ull;
    }
    __syncthreads();
    uint64_t o = base_s + wsum[warp] + incl - cnt;
#pragma unroll
    for (int k = 0; k < kZcPer; ++k)
      if (inm >> k & 1u) {
        const uint64_t i = t0 + threadIdx.x + (uint64_t)k * kZcThreads;
        oz[o] = z[k] - z_lo;
        oy[o] = sy[i];
        ++o;
      }
    __syncthreads();  // wsum / base_s are rewritten by the next tile
  }
}

// The job's cold CSR offsets: the sum of the ranks' exclusive scans is the
// exclusive scan of the summed counts, cptr[k] = sum_q cptr_q[k].
__global__ void sum_rows_u64_kernel(const uint64_t* __restrict__ cp /* [N][keys + 1] */,
                                    uint64_t keys1, int nranks, uint64_t* __restrict__ tot) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < keys1;
       k += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s = 0;
    for (int q = 0; q < nranks; ++q) s += cp[(uint64_t)q * keys1 + k];
    tot[k] = s;
  }
}

// The job's cold CSR from the ranks' gathered parts: key k's segment is rank
// 0's segment of k, then rank 1's, ... A warp takes 32 consecutive keys: for
// each rank q their short segments are ONE contiguous range of q's part
// (its segments are key-major), read coalesced; each record's key is found
// from the warp scan of the 32 lengths and it lands at cptr[k] + (the lower
// ranks' records of k) + its offset in q's segment. Long segments (>= 256
// records: the cold y just past the hot ranks) are queued whole and copied
// by a warp each (cold_merge_long_kernel), so no warp serialises a hot key.
struct LongSeg {
  uint64_t src, dst;
  uint32_t len, pad;
};
constexpr uint32_t kMergeLong = 256;
__global__ void cold_merge_kernel(const uint64_t* __restrict__ cp /* [N][keys + 1] */,
                                  const uint64_t* __restrict__ part_base /* [N] */,
                                  const uint4* __restrict__ src, const uint64_t* __restrict__ cptr,
                                  uint64_t keys, int nranks, uint4* __restrict__ dst,
                                  LongSeg* __restrict__ longs, unsigned int* __restrict__ n_long) {
  const uint32_t lane = lane_id();
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t kb = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; kb * 32 < keys;
       kb += nw) {
    const uint64_t k0 = kb * 32, k = k0 + lane;
    uint64_t d = k < keys ? cptr[k] : 0;  // next free slot of key k
    for (int q = 0; q < nranks; ++q) {
      const uint64_t* c = cp + (uint64_t)q * (keys + 1);
      uint64_t s = 0;
      uint32_t len = 0;
      if (k < keys) {
        s = c[k];
        len = (uint32_t)(c[k + 1] - s);
      }
      const bool is_long = len >= kMergeLong;
      if (is_long) {
        const unsigned int slot = atomicAdd(n_long, 1u);
        longs[slot] = LongSeg{part_base[q] + s, d, len, 0};
      }
      const uint32_t sl = is_long ? 0u : len;  // the short ones, copied here
      const uint32_t incl = warp_incl_scan(sl);
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      // record f of the short segments belongs to lane j (the warp scan of
      // their lengths) at offset f - before in both its source and its slot
      for (uint32_t f = lane; f < ((total + 31) & ~31u); f += 32) {
        uint32_t j = 0;
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1) {
          const uint32_t probe = __shfl_sync(0xffffffffu, incl, j + st - 1);
          if (probe <= f) j += st;
        }
        const uint32_t jj = j & 31;
        const uint32_t before = __shfl_sync(0xffffffffu, incl - sl, jj);
        const uint64_t dj = __shfl_sync(0xffffffffu, d, jj);
        const uint64_t sj = __shfl_sync(0xffffffffu, s, jj);
        if (f < total) dst[dj + (f - before)] = __ldg(src + part_base[q] + sj + (f - before));
      }
      d += len;
    }
  }
}
__global__ void cold_merge_long_kernel(const LongSeg* __restrict__ longs,
                                       const unsigned int* __restrict__ n_long,
                                       const uint4* __restrict__ src, uint4* __restrict__ dst) {
  const uint32_t lane = lane_id();
  const uint32_t n = *n_long;
  for (uint32_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n;
       w += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const LongSeg g = longs[w];
    for (uint32_t f = lane; f < g.len; f += 32) dst[g.dst + f] = __ldg(src + g.src + f);
  }
}

// Long rows (more than 32 listed hot ranks: the record holds the first 32)
// keep the rest of their hot prefix in a tail list; under the z-split the
// tails of all rows are gathered instead of the whole dense lists.
// tlen[i] = listed ranks past the record's 32 (0 for the short rows).
__global__ void tail_len_kernel(const uint32_t* __restrict__ rcnt, uint64_t n,
                                uint32_t* __restrict__ tlen, uint32_t* __restrict__ is_tail) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = rcnt[i] & 0xffffffu;
    tlen[i] = c > 32 ? c - 32 : 0u;
    is_tail[i] = c > 32 ? 1u : 0u;
  }
}
// Tail rows: global row id, start of the tail (local, rebased after the
// gather) and the ranks themselves (the list entries after the top-subset
// ranks and the first 32 listed ones).
__global__ void tail_fill_kernel(const uint32_t* __restrict__ rcnt, uint64_t n,
                                 const uint32_t* __restrict__ is_tail,
                                 const uint64_t* __restrict__ tpos /* scan of is_tail */,
                                 const uint64_t* __restrict__ toff /* scan of tlen */,
                                 const uint64_t* __restrict__ dl_ptr,
                                 const uint32_t* __restrict__ dl_col, uint64_t row_base,
                                 uint32_t* __restrict__ t_rows, uint64_t* __restrict__ t_ptr,
                                 uint32_t* __restrict__ t_col) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (!is_tail[i]) continue;
    const uint32_t cw = rcnt[i], c = cw & 0xffffffu;
    const uint32_t skip = __popc((cw >> 24) & 0x7fu) + 32;
    const uint64_t j = tpos[i], o = toff[i];
    t_rows[j] = (uint32_t)(row_base + i);
    t_ptr[j] = o;
    for (uint32_t t = 0; t < c - 32; ++t) t_col[o + t] = dl_col[dl_ptr[i] + skip + t];
  }
}
// Rebase the gathered tail starts: rank q's entries [r0[q], r0[q+1]) += c0[q].
__global__ void tail_rebase_kernel(uint64_t* __restrict__ t_ptr, const uint64_t* __restrict__ r0,
                                   const uint64_t* __restrict__ c0, int nranks) {
  const uint64_t n = r0[nranks];
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    int q = 0;
    while (q + 1 < nranks && r0[q + 1] <= j) ++q;
    t_ptr[j] += c0[q];
  }
}

}  // namespace d3g
