// Counting-scatter CSR build + warp-level segmented sort/unique.
//
// build_csr (P/src/relation.cpp:206-258) needs rows sorted by minor with
// duplicates collapsed. Rows on the BASELINE configs are short (10-45
// entries), so instead of a full-width LSD radix sort of (major, minor) keys
// (5-6 passes of 24 B/tuple) the GPU path:
//   1. histograms the major codes (one pass),
//   2. exclusive-scans the counts into row offsets,
//   3. scatters the minor codes into their row (atomic per-row cursor),
//   4. sorts and de-duplicates every row in registers: one warp per row,
//      bitonic network over 32*E lanes-elements (E = 1, 2, 4 -> rows <= 128),
//      longer rows by one CTA (shared memory up to 8192 entries, global
//      memory beyond), with no host round trip,
//   5. scans the unique counts and compacts the rows into the final CSR.
// About 5 passes of 4-8 B/tuple.
#pragma once

#include "prims.cuh"

namespace d3g {

__global__ void major_hist_kernel(const uint32_t* __restrict__ maj, uint64_t n,
                                  uint32_t* __restrict__ cnt) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[maj[i]], 1u);
}

__global__ void major_scatter_kernel(const uint32_t* __restrict__ maj,
                                     const uint32_t* __restrict__ mnr, uint64_t n,
                                     const uint64_t* __restrict__ off,
                                     uint32_t* __restrict__ left /* counts, consumed */,
                                     uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t m = maj[i];
    out[off[m] + atomicSub(&left[m], 1u) - 1u] = mnr[i];
  }
}

// Bitonic sort of 32*E elements held striped (element e*32 + lane) by a warp.
template <int E>
__device__ __forceinline__ void warp_bitonic(uint32_t (&v)[E]) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int ej = j / 32;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int p = e ^ ej;
          if (p > e) {
            const uint32_t i = (uint32_t)e * 32 + lane;
            const bool up = (i & k) == 0;
            const uint32_t a = v[e], b = v[p];
            const uint32_t mn = a < b ? a : b, mx = a < b ? b : a;
            v[e] = up ? mn : mx;
            v[p] = up ? mx : mn;
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint32_t i = (uint32_t)e * 32 + lane;
          const uint32_t o = __shfl_xor_sync(0xffffffffu, v[e], j);
          const bool up = (i & k) == 0;
          const bool lower = (lane & j) == 0;
          const uint32_t mn = v[e] < o ? v[e] : o, mx = v[e] < o ? o : v[e];
          v[e] = (lower == up) ? mn : mx;
        }
      }
    }
  }
}

// Sort (and optionally unique) a row of len <= 32*E held in data[base..):
// writes the result back in place, returns the kept count (warp-uniform).
template <int E>
__device__ __forceinline__ uint32_t warp_sort_row(uint32_t* __restrict__ data, uint64_t base,
                                                  uint32_t len, bool unique) {
  const uint32_t lane = lane_id();
  uint32_t v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = (uint32_t)e * 32 + lane;
    v[e] = i < len ? data[base + i] : 0xffffffffu;
  }
  warp_bitonic<E>(v);
  uint32_t written = 0;
  uint32_t prev_last = 0xffffffffu;  // last element of the previous chunk
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = (uint32_t)e * 32 + lane;
    uint32_t prev = __shfl_up_sync(0xffffffffu, v[e], 1);
    if (lane == 0) prev = prev_last;
    const bool valid = i < len;
    const bool keep = valid && (!unique || i == 0 || v[e] != prev);
    const uint32_t m = __ballot_sync(0xffffffffu, keep);
    if (keep) data[base + written + __popc(m & ((1u << lane) - 1))] = v[e];
    written += __popc(m);
    prev_last = __shfl_sync(0xffffffffu, v[e], 31);
  }
  return written;
}

// Half-warp sort of a row of <= 16 entries (lanes 16h..16h+15), in place,
// unique-compacted; returns the kept count (uniform within the half).
__device__ __forceinline__ uint32_t half_sort_row(uint32_t* __restrict__ data, uint64_t base,
                                                  uint32_t len, bool unique) {
  const uint32_t lane = lane_id(), l16 = lane & 15, half = lane >> 4;
  uint32_t v = l16 < len ? data[base + l16] : 0xffffffffu;
#pragma unroll
  for (uint32_t k = 2; k <= 16; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      const uint32_t u = __shfl_xor_sync(0xffffffffu, v, j);
      const bool asc = (l16 & k) == 0, low = (l16 & j) == 0;
      v = (asc == low) ? (u < v ? u : v) : (u > v ? u : v);
    }
  }
  const uint32_t prev = __shfl_up_sync(0xffffffffu, v, 1, 16);
  const bool keep = l16 < len && (!unique || l16 == 0 || v != prev);
  const uint32_t m = (__ballot_sync(0xffffffffu, keep) >> (16 * half)) & 0xffffu;
  if (keep) data[base + __popc(m & ((1u << l16) - 1))] = v;
  return __popc(m);
}

// Sort (+ unique) of a row of len <= 32 by a HALF warp: 16 lanes x 2 elements
// (element e * 16 + l16), so one warp sorts two rows per bitonic network --
// half the issued instructions of a 32-lane network per row (rows are ~20
// long on the BASELINE configs). Both halves must call it (len 0 = idle).
// In place; returns the kept count (uniform within the half).
__device__ __forceinline__ uint32_t half_sort_row32(uint32_t* data, uint64_t base, uint32_t len,
                                                  bool unique) {
  const uint32_t lane = lane_id(), l16 = lane & 15, half = lane >> 4;
  uint32_t v0 = l16 < len ? data[base + l16] : 0xffffffffu;
  uint32_t v1 = l16 + 16 < len ? data[base + l16 + 16] : 0xffffffffu;
#pragma unroll
  for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      if (j == 16) {  // k == 32: elements l16 and 16 + l16, ascending
        const uint32_t mn = v0 < v1 ? v0 : v1, mx = v0 < v1 ? v1 : v0;
        v0 = mn;
        v1 = mx;
      } else {
        const uint32_t o0 = __shfl_xor_sync(0xffffffffu, v0, j);
        const uint32_t o1 = __shfl_xor_sync(0xffffffffu, v1, j);
        const bool lower = (l16 & j) == 0;
        const bool up0 = (l16 & k) == 0, up1 = ((16 + l16) & k) == 0;
        const uint32_t mn0 = v0 < o0 ? v0 : o0, mx0 = v0 < o0 ? o0 : v0;
        const uint32_t mn1 = v1 < o1 ? v1 : o1, mx1 = v1 < o1 ? o1 : v1;
        v0 = (lower == up0) ? mn0 : mx0;
        v1 = (lower == up1) ? mn1 : mx1;
      }
    }
  }
  const uint32_t lt = (1u << l16) - 1;
  // element i = e * 16 + l16; predecessor of (0, 0) is none, of (1, 0) is (0, 15)
  uint32_t p0 = __shfl_up_sync(0xffffffffu, v0, 1, 16);
  uint32_t p1 = __shfl_up_sync(0xffffffffu, v1, 1, 16);
  const uint32_t last0 = __shfl_sync(0xffffffffu, v0, 15, 16);
  if (l16 == 0) p1 = last0;
  const bool k0 = l16 < len && (!unique || l16 == 0 || v0 != p0);
  const bool k1 = l16 + 16 < len && (!unique || v1 != p1);
  const uint32_t m0 = (__ballot_sync(0xffffffffu, k0) >> (16 * half)) & 0xffffu;
  const uint32_t m1 = (__ballot_sync(0xffffffffu, k1) >> (16 * half)) & 0xffffu;
  __syncwarp();
  if (k0) data[base + __popc(m0 & lt)] = v0;
  if (k1) data[base + __popc(m0) + __popc(m1 & lt)] = v1;
  __syncwarp();
  return __popc(m0) + __popc(m1);
}

// One warp per row for rows of length <= 128 (two rows per warp, one per
// half-warp, when both hold <= 16 entries); longer rows are appended to
// long_rows (any order) for row_sort_long_kernel.
__global__ void row_sort_small_kernel(uint32_t* __restrict__ data, const uint64_t* __restrict__ off,
                                      uint64_t n_rows, int unique, uint32_t* __restrict__ kept,
                                      uint32_t* __restrict__ long_rows,
                                      unsigned int* __restrict__ n_long) {
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  const uint32_t lane = lane_id();
  for (uint64_t r2 = ((uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * 2;
       r2 < n_rows; r2 += warps * 2) {
    const uint64_t b0 = off[r2], b1 = off[r2 + 1];
    const uint64_t b2 = r2 + 1 < n_rows ? off[r2 + 2] : b1;
    const uint32_t l0 = (uint32_t)(b1 - b0), l1 = (uint32_t)(b2 - b1);
    if (l0 <= 32 && l1 <= 32) {  // both rows in one pass, a half-warp each
      const uint32_t h = lane >> 4;
      const uint64_t b = h ? b1 : b0;
      const uint32_t len = h ? l1 : l0;
      const uint32_t k = (l0 <= 16 && l1 <= 16) ? half_sort_row(data, b, len, unique)
                                                : half_sort_row32(data, b, len, unique);
      if ((lane & 15) == 0 && r2 + h < n_rows) kept[r2 + h] = k;
      continue;
    }
    for (uint64_t r = r2; r < r2 + 2 && r < n_rows; ++r) {
    const uint64_t b = r == r2 ? b0 : b1;
    const uint32_t len = r == r2 ? l0 : l1;
    uint32_t k = len;
    bool lng = false;
    if (len <= 1) {
      k = len;
    } else if (len <= 32) {
      k = warp_sort_row<1>(data, b, len, unique);
    } else if (len <= 64) {
      k = warp_sort_row<2>(data, b, len, unique);
    } else if (len <= 128) {
      k = warp_sort_row<4>(data, b, len, unique);
    } else {
      lng = true;
    }
    if (lane_id() == 0) {
      kept[r] = k;
      if (lng && long_rows) long_rows[atomicAdd(n_long, 1u)] = (uint32_t)r;
    }
    }
  }
}

// One CTA per long row: rows of 129..8192 entries are sorted by a bitonic
// network in shared memory; longer rows (rare: one x or z holding > 8192
// tuples) in place in global memory by the same CTA, with the direction-free
// network (a mirror step per merge size, then half-cleaners, all ascending)
// so that the virtual +inf padding past the row's end never moves. The row
// count comes from the device (n_long): no host round trip.
constexpr int kLongRowMax = 8192;

__device__ __forceinline__ void cas_global(uint32_t* d, uint64_t a, uint64_t b) {
  const uint32_t x = __ldcg(d + a), y = __ldcg(d + b);
  if (y < x) {
    __stcg(d + a, y);
    __stcg(d + b, x);
  }
}

__device__ void sort_row_global(uint32_t* __restrict__ d, uint64_t len) {
  uint64_t p2 = 1;
  while (p2 < len) p2 <<= 1;
  for (uint64_t k = 2; k <= p2; k <<= 1) {
    const uint64_t hk = k >> 1;
    for (uint64_t i = threadIdx.x; i < p2 / 2; i += blockDim.x) {
      const uint64_t blk = (i / hk) * k, o = i % hk;
      const uint64_t a = blk + o, b = blk + k - 1 - o;
      if (b < len) cas_global(d, a, b);
    }
    __syncthreads();
    for (uint64_t j = k >> 2; j >= 1; j >>= 1) {
      for (uint64_t i = threadIdx.x; i < p2 / 2; i += blockDim.x) {
        const uint64_t a = (i / j) * 2 * j + (i % j), b = a + j;
        if (b < len) cas_global(d, a, b);
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(1024)
row_sort_long_kernel(uint32_t* __restrict__ data, const uint64_t* __restrict__ off,
                     const uint32_t* __restrict__ rows, const unsigned int* __restrict__ n_long,
                     int unique, uint32_t* __restrict__ kept) {
  __shared__ uint32_t s[kLongRowMax];
  __shared__ uint32_t wsum[32];
  const uint64_t n = *n_long;
  for (uint64_t q = blockIdx.x; q < n; q += gridDim.x) {
    const uint32_t r = rows[q];
    const uint64_t b = off[r];
    const uint64_t len = off[r + 1] - b;
    uint64_t written = 0;
    if (len <= (uint64_t)kLongRowMax) {
      uint32_t p2 = 1;
      while (p2 < len) p2 <<= 1;
      for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x)
        s[i] = i < len ? data[b + i] : 0xffffffffu;
      __syncthreads();
      for (uint32_t k = 2; k <= p2; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
          for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x) {
            const uint32_t pj = i ^ j;
            if (pj > i) {
              const bool up = (i & k) == 0;
              const uint32_t a = s[i], c = s[pj];
              if ((a > c) == up) {
                s[i] = c;
                s[pj] = a;
              }
            }
          }
          __syncthreads();
        }
      // unique + compaction in index order (block scan over 1024-element chunks)
      for (uint32_t base = 0; base < len; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        const bool keep = i < len && (!unique || i == 0 || s[i] != s[i - 1]);
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        if (lane_id() == 0) wsum[threadIdx.x >> 5] = __popc(m);
        __syncthreads();
        uint32_t before = 0, tot = 0;
        for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) {
          if (w < (threadIdx.x >> 5)) before += wsum[w];
          tot += wsum[w];
        }
        if (keep) data[b + written + before + __popc(m & ((1u << lane_id()) - 1))] = s[i];
        written += tot;
        __syncthreads();
      }
    } else {
      uint32_t* d = data + b;
      sort_row_global(d, len);
      // in-place compaction: a chunk reads (value, predecessor) before any of
      // its writes, and writes land at or below their source index
      for (uint64_t base = 0; base < len; base += blockDim.x) {
        const uint64_t i = base + threadIdx.x;
        uint32_t v = 0;
        bool keep = false;
        if (i < len) {
          v = __ldcg(d + i);
          keep = !unique || i == 0 || v != __ldcg(d + i - 1);
        }
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        if (lane_id() == 0) wsum[threadIdx.x >> 5] = __popc(m);
        __syncthreads();
        uint32_t before = 0, tot = 0;
        for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) {
          if (w < (threadIdx.x >> 5)) before += wsum[w];
          tot += wsum[w];
        }
        if (keep) __stcg(d + written + before + __popc(m & ((1u << lane_id()) - 1)), v);
        written += tot;
        __syncthreads();
      }
    }
    if (threadIdx.x == 0) kept[r] = (uint32_t)written;
    __syncthreads();
  }
}

// rows compaction: copy kept[r] values of row r from data[off[r]..] to
// col[row_ptr[r]..] (one warp per row)
__global__ void row_compact_kernel(const uint32_t* __restrict__ data, const uint64_t* __restrict__ off,
                                   const uint64_t* __restrict__ row_ptr, uint64_t n_rows,
                                   uint32_t* __restrict__ col) {
  // 8 lanes per row: most rows are short
  const uint32_t gl = threadIdx.x & 7;
  for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x / 8) + (threadIdx.x >> 3); r < n_rows;
       r += (uint64_t)gridDim.x * (blockDim.x / 8)) {
    const uint64_t s = off[r], d = row_ptr[r], k = row_ptr[r + 1] - d;
    for (uint64_t i = gl; i < k; i += 8) col[d + i] = data[s + i];
  }
}

// Sorts every row data[off[r] .. off[r+1]) ascending, optionally dropping
// duplicates; kept[r] receives the resulting length (rows stay in place).
// max_len (when known on the host) skips the long-row launch.
inline void segmented_sort(Ctx& ctx, uint32_t* data, const uint64_t* off, uint64_t n_rows,
                           bool unique, uint32_t* kept, uint64_t max_len = ~0ull) {
  if (n_rows == 0) return;
  const bool may_be_long = max_len > 128;
  DBuf<uint32_t> rows;
  DBuf<unsigned int> n_long;
  if (may_be_long) {
    rows = ctx.alloc<uint32_t>(n_rows);
    n_long = ctx.zeros<unsigned int>(1);
  }
  D3G_LAUNCH(ctx, row_sort_small_kernel, grid_for(n_rows * 32, 256, ctx.sm_count * 64), 256, 0,
             data, off, n_rows, unique ? 1 : 0, kept, rows.p, n_long.p);
  if (may_be_long)
    D3G_LAUNCH(ctx, row_sort_long_kernel,
               (unsigned)std::min<uint64_t>(n_rows, (uint64_t)ctx.sm_count * 2), 1024, 0, data, off,
               rows.p, n_long.p, unique ? 1 : 0, kept);
}

}  // namespace d3g
