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
// (their order is irrelevant: the CSR build sorts). Warp-aggregated cursor.
__global__ void zrange_compact_kernel(const uint32_t* __restrict__ sz, const uint32_t* __restrict__ sy,
                                      uint64_t n, uint32_t z_lo, uint32_t z_hi,
                                      uint32_t* __restrict__ oz, uint32_t* __restrict__ oy,
                                      unsigned long long* __restrict__ cursor) {
  const uint32_t lane = lane_id();
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    bool in = false;
    uint32_t z = 0;
    if (i < n) {
      z = sz[i];
      in = z >= z_lo && z < z_hi;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, in);
    unsigned long long base = 0;
    if (lane == 0 && m) base = atomicAdd(cursor, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (in) {
      const uint64_t o = base + __popc(m & ((1u << lane) - 1u));
      oz[o] = z - z_lo;
      oy[o] = sy[i];
    }
  }
}

// Sum of the ranks' count rows: tot[k] = sum_q cnt[q][k].
__global__ void sum_rows_u32_kernel(const uint32_t* __restrict__ cnt, uint64_t keys, int nranks,
                                    uint32_t* __restrict__ tot) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < keys;
       k += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t s = 0;
    for (int q = 0; q < nranks; ++q) s += cnt[(uint64_t)q * keys + k];
    tot[k] = s;
  }
}

// The global cold CSR from the ranks' gathered parts: key k's segment is
// rank 0's segment of k, then rank 1's, ... (src_off[q]: rank q's exclusive
// scan over its counts, part_base[q]: where rank q's records start in src).
// A warp per key: lanes copy the records of each rank's segment in turn.
__global__ void cold_merge_kernel(const uint32_t* __restrict__ cnt /* [N][keys] */,
                                  const uint64_t* __restrict__ src_off /* [N][keys + 1] */,
                                  const uint64_t* __restrict__ part_base /* [N] */,
                                  const uint4* __restrict__ src, const uint64_t* __restrict__ cptr,
                                  uint64_t keys, int nranks, uint4* __restrict__ dst) {
  const uint32_t lane = lane_id();
  const uint64_t w0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t k = w0; k < keys; k += nw) {
    uint64_t d = cptr[k];
    for (int q = 0; q < nranks; ++q) {
      const uint32_t n = cnt[(uint64_t)q * keys + k];
      if (n == 0) continue;
      const uint4* s = src + part_base[q] + src_off[(uint64_t)q * (keys + 1) + k];
      for (uint32_t j = lane; j < n; j += 32) dst[d + j] = s[j];
      d += n;
    }
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
