// DenseEC (north_star subsystem 3), replacing dense_ec / run_chunk
// (P/src/denseec.cpp:8-153) and the bitmap primitives block_and_any /
// probe_any (P/include/dim3/bitmap.hpp:23-48).
//
// The reference answers "does R[x] intersect S[z]?" once per (live x, dense
// z) with a 256-bit-block AND sweep or scalar probes, early-exiting at the
// first common y. The GPU kernel answers the same existence question for 128
// x at once, bit-sliced:
//
//   * a CTA owns a group of 128 live x (x ordered by m_x descending);
//   * it builds, in shared memory, the transposed bit slice
//     T[y] = {bit i : y in R[x_i]} (uint4 = 128 bits) for the hottest y
//     (y re-ranked by dR(y), ranks < y_hot), and a hash map for the colder y
//     of the group in a per-CTA global-memory slice;
//   * every thread then sweeps dense z lists (hot-first y ranks):
//       acc |= T[y]  until acc == all-live (early exit) or the list ends;
//     popc(acc) is the number of distinct (x, z) pairs for that z and group.
//
// One LOP3 per 32 (x, z) pairs per witness; the z lists are streamed from
// L2, the hot slice is read from shared memory. The output set is exactly
// {(x, z) : R[x] and S[z] share a y} restricted to dense z.
#pragma once

#include "sparsebmm.cuh"

namespace d3g {

constexpr int kDenseThreads = 512;
constexpr uint32_t kColdEmpty = 0xffffffffu;

struct DenseParams {
  const uint32_t* xorder;   // live x codes by position
  uint64_t n_live;
  const uint64_t* r_ptr;    // R by x (original y codes)
  const uint32_t* r_col;
  const uint32_t* y_rank;   // y code -> hotness rank
  const uint64_t* dl_ptr;   // dense lists, by row position
  const uint32_t* dl_col;   // y ranks, ascending within a row
  const uint32_t* dl_z;     // z code per row position
  uint64_t n_dense;
  uint32_t y_hot;           // ranks < y_hot live in shared memory
  uint32_t cold_cap;        // per-CTA cold table capacity (power of 2)
  uint32_t* cold_keys;      // gridDim.x * cold_cap
  uint4* cold_vals;         // gridDim.x * cold_cap
  uint64_t z_lo, z_hi;      // row-position range handled by this launch
};

__device__ __forceinline__ uint32_t cold_hash(uint32_t k, uint32_t mask) {
  return (k * 0x9e3779b1u) & mask;
}

__device__ __forceinline__ void cold_insert(uint32_t* keys, uint4* vals, uint32_t mask, uint32_t k,
                                            uint32_t word, uint32_t bit) {
  uint32_t s = cold_hash(k, mask);
  for (;;) {
    uint32_t prev = atomicCAS(&keys[s], kColdEmpty, k);
    if (prev == kColdEmpty || prev == k) break;
    s = (s + 1) & mask;
  }
  atomicOr(reinterpret_cast<uint32_t*>(&vals[s]) + word, bit);
}

__device__ __forceinline__ uint4 cold_lookup(const uint32_t* keys, const uint4* vals, uint32_t mask,
                                             uint32_t k) {
  uint32_t s = cold_hash(k, mask);
  for (;;) {
    uint32_t key = keys[s];
    if (key == k) return vals[s];
    if (key == kColdEmpty) return make_uint4(0, 0, 0, 0);
    s = (s + 1) & mask;
  }
}

template <int kMode>
__global__ void __launch_bounds__(kDenseThreads, 1)
dense_ec_kernel(DenseParams p, Decode dec, Emit em, Tally* tally) {
  extern __shared__ uint4 hot[];
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  uint32_t* ckeys = p.cold_keys + (uint64_t)blockIdx.x * p.cold_cap;
  uint4* cvals = p.cold_vals + (uint64_t)blockIdx.x * p.cold_cap;
  const uint32_t cmask = p.cold_cap - 1;
  const uint64_t groups = (p.n_live + 127) / 128;
  uint64_t cnt = 0, sum = 0, xr = 0;

  for (uint64_t g = blockIdx.x; g < groups; g += gridDim.x) {
    // fresh hot slice and cold table for every group (the cold table is
    // sized to ~2x the group's cold entries, so wiping it is cheap)
    for (uint32_t i = threadIdx.x; i < p.y_hot; i += blockDim.x) hot[i] = make_uint4(0, 0, 0, 0);
    for (uint32_t i = threadIdx.x; i < p.cold_cap; i += blockDim.x) {
      ckeys[i] = kColdEmpty;
      cvals[i] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    const uint64_t p0 = g * 128;
    const uint32_t members = (uint32_t)((p.n_live - p0) < 128 ? (p.n_live - p0) : 128);
    // build the group's transposed slice: one warp per member x
    for (uint32_t m = warp; m < members; m += nwarps) {
      uint32_t x = p.xorder[p0 + m];
      uint32_t word = m >> 5, bit = 1u << (m & 31);
      for (uint64_t k = p.r_ptr[x] + lane; k < p.r_ptr[x + 1]; k += 32) {
        uint32_t yr = p.y_rank[p.r_col[k]];
        if (yr < p.y_hot)
          atomicOr(reinterpret_cast<uint32_t*>(&hot[yr]) + word, bit);
        else
          cold_insert(ckeys, cvals, cmask, yr, word, bit);
      }
    }
    __syncthreads();
    uint4 full;
    full.x = members >= 32 ? 0xffffffffu : ((1u << members) - 1);
    full.y = members >= 64 ? 0xffffffffu : (members <= 32 ? 0u : ((1u << (members - 32)) - 1));
    full.z = members >= 96 ? 0xffffffffu : (members <= 64 ? 0u : ((1u << (members - 64)) - 1));
    full.w = members >= 128 ? 0xffffffffu : (members <= 96 ? 0u : ((1u << (members - 96)) - 1));

    for (uint64_t i = p.z_lo + threadIdx.x; i < p.z_hi; i += blockDim.x) {
      uint64_t k0 = p.dl_ptr[i], k1 = p.dl_ptr[i + 1];
      uint4 acc = make_uint4(0, 0, 0, 0);
      for (uint64_t k = k0; k < k1; ++k) {
        uint32_t yr = p.dl_col[k];
        uint4 v = yr < p.y_hot ? hot[yr] : cold_lookup(ckeys, cvals, cmask, yr);
        acc.x |= v.x;
        acc.y |= v.y;
        acc.z |= v.z;
        acc.w |= v.w;
        if (acc.x == full.x && acc.y == full.y && acc.z == full.z && acc.w == full.w) break;
      }
      uint32_t c = __popc(acc.x) + __popc(acc.y) + __popc(acc.z) + __popc(acc.w);
      cnt += c;
      if (kMode != kModeCount && c) {
        uint32_t zc = p.dl_z[i];
        uint32_t words[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
        for (int wi = 0; wi < 4; ++wi) {
          uint32_t bits = words[wi];
          while (bits) {
            int b = __ffs(bits) - 1;
            bits &= bits - 1;
            uint32_t xc = p.xorder[p0 + wi * 32 + b];
            if (kMode == kModeChecksum) {
              uint64_t h = dec.hash(xc, zc);
              sum += h;
              xr ^= h;
            } else {
              unsigned long long idx = atomicAdd(em.cursor, 1ull);
              if (idx < em.cap) {
                em.x[idx] = xc;
                em.z[idx] = zc;
              }
            }
          }
        }
      }
    }
    __syncthreads();
  }
  tally_flush(tally, cnt, sum, xr);
}

// ---------------------------------------------------------------------------
// DenseEC v2: z-tile resident. The kernel above re-streams every dense z list
// from L2 once per 128-x group (1,563 groups x 18 MB on cfg2) and looks cold
// y up in a global hash. Here a persistent CTA claims a unit = (z tile,
// x-group range): the tile's lists (y ranks) are staged once into shared
// memory, then for each 128-x group of the range the CTA
//   1. builds the transposed slice from the group's R rows (hot ranks in a
//      direct-indexed uint4 array, cold ranks in a shared-memory hash),
//   2. sweeps every row of the tile: acc |= T[y] until all-live (early exit),
//   3. clears exactly what it set (re-walk for the hot part, full wipe of the
//      small cold table).
// All per-iteration loads hit shared memory; global traffic is one pass over
// the lists per x range plus the R rows of each group per tile.
constexpr int kD2Threads = 512;
constexpr int kHotCandidates = 6;
__constant__ uint32_t kHotCand[kHotCandidates] = {16384, 8192, 4096, 2048, 1024, 512};

struct DenseTileParams {
  const uint32_t* xorder;
  uint64_t n_live;
  const uint64_t* r_ptr;
  const uint32_t* r_col;
  const uint32_t* y_rank;
  const uint64_t* dl_ptr;
  const uint32_t* dl_col;
  const uint32_t* dl_z;
  const uint32_t* tile_begin;  // n_tiles + 1 row boundaries
  uint32_t n_tiles, x_splits, groups;
  uint32_t hot, cold_cap, list_cap, row_cap;
  unsigned int* work;
};

// Max over groups of the number of R entries with y rank >= each candidate
// hot size (bounds the per-group cold table).
__global__ void __launch_bounds__(128)
dense_cold_count_kernel(const uint32_t* __restrict__ xorder, uint64_t n_live,
                        const uint64_t* __restrict__ r_ptr, const uint32_t* __restrict__ r_col,
                        const uint32_t* __restrict__ y_rank, unsigned int* __restrict__ out_max) {
  __shared__ unsigned int c[kHotCandidates];
  const uint64_t groups = (n_live + 127) / 128;
  for (uint64_t g = blockIdx.x; g < groups; g += gridDim.x) {
    if (threadIdx.x < kHotCandidates) c[threadIdx.x] = 0;
    __syncthreads();
    uint64_t p = g * 128 + threadIdx.x;
    if (p < n_live) {
      uint32_t x = xorder[p];
      unsigned int loc[kHotCandidates] = {};
      for (uint64_t k = r_ptr[x]; k < r_ptr[x + 1]; ++k) {
        uint32_t yr = y_rank[r_col[k]];
#pragma unroll
        for (int j = 0; j < kHotCandidates; ++j) loc[j] += yr >= kHotCand[j];
      }
#pragma unroll
      for (int j = 0; j < kHotCandidates; ++j)
        if (loc[j]) atomicAdd(&c[j], loc[j]);
    }
    __syncthreads();
    if (threadIdx.x < kHotCandidates) atomicMax(&out_max[threadIdx.x], c[threadIdx.x]);
    __syncthreads();
  }
}

__device__ __forceinline__ void s_cold_insert(uint32_t* keys, uint4* vals, uint32_t mask,
                                              uint32_t k, uint32_t word, uint32_t bit) {
  uint32_t s = cold_hash(k, mask);
  for (;;) {
    uint32_t prev = atomicCAS(&keys[s], kColdEmpty, k);
    if (prev == kColdEmpty || prev == k) break;
    s = (s + 1) & mask;
  }
  atomicOr(reinterpret_cast<uint32_t*>(&vals[s]) + word, bit);
}

__device__ __forceinline__ uint4 s_cold_lookup(const uint32_t* keys, const uint4* vals,
                                               uint32_t mask, uint32_t k) {
  uint32_t s = cold_hash(k, mask);
  for (;;) {
    uint32_t key = keys[s];
    if (key == k) return vals[s];
    if (key == kColdEmpty) return make_uint4(0, 0, 0, 0);
    s = (s + 1) & mask;
  }
}

template <int kMode>
__global__ void __launch_bounds__(kD2Threads, 1)
dense_ec_tile_kernel(DenseTileParams p, Decode dec, Emit em, Tally* tally) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint4* slice = reinterpret_cast<uint4*>(smem_raw);
  uint4* cvals = slice + p.hot;
  uint32_t* ckeys = reinterpret_cast<uint32_t*>(cvals + p.cold_cap);
  uint32_t* lptr = ckeys + p.cold_cap;
  uint32_t* lcol = lptr + p.row_cap + 1;
  __shared__ unsigned int s_unit;
  __shared__ int s_cold_used;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t cmask = p.cold_cap - 1;
  uint64_t cnt = 0, sum = 0, xr = 0;

  for (uint32_t i = threadIdx.x; i < p.hot; i += blockDim.x) slice[i] = make_uint4(0, 0, 0, 0);
  for (uint32_t i = threadIdx.x; i < p.cold_cap; i += blockDim.x) {
    ckeys[i] = kColdEmpty;
    cvals[i] = make_uint4(0, 0, 0, 0);
  }
  int cur_tile = -1;
  const unsigned int n_units = p.n_tiles * p.x_splits;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_unit = atomicAdd(p.work, 1u);
    __syncthreads();
    const unsigned int unit = s_unit;
    if (unit >= n_units) break;
    const int tile = (int)(unit / p.x_splits);
    const uint32_t split = unit % p.x_splits;
    const uint32_t tb = p.tile_begin[tile], te = p.tile_begin[tile + 1];
    const uint32_t nrows = te - tb;
    if (tile != cur_tile) {
      const uint64_t base = p.dl_ptr[tb];
      for (uint32_t i = threadIdx.x; i <= nrows; i += blockDim.x)
        lptr[i] = (uint32_t)(p.dl_ptr[tb + i] - base);
      const uint32_t nent = (uint32_t)(p.dl_ptr[te] - base);
      for (uint32_t k = threadIdx.x; k < nent; k += blockDim.x) lcol[k] = p.dl_col[base + k];
      cur_tile = tile;
      __syncthreads();
    }
    const uint32_t g_lo = (uint32_t)((uint64_t)p.groups * split / p.x_splits);
    const uint32_t g_hi = (uint32_t)((uint64_t)p.groups * (split + 1) / p.x_splits);
    for (uint32_t g = g_lo; g < g_hi; ++g) {
      const uint64_t p0 = (uint64_t)g * 128;
      const uint32_t members = (uint32_t)((p.n_live - p0) < 128 ? (p.n_live - p0) : 128);
      if (threadIdx.x == 0) s_cold_used = 0;
      __syncthreads();
      // 1. build
      bool used_cold = false;
      for (uint32_t m = warp; m < members; m += nwarps) {
        uint32_t x = p.xorder[p0 + m];
        uint32_t word = m >> 5, bit = 1u << (m & 31);
        for (uint64_t k = p.r_ptr[x] + lane; k < p.r_ptr[x + 1]; k += 32) {
          uint32_t yr = p.y_rank[p.r_col[k]];
          if (yr < p.hot) {
            atomicOr(reinterpret_cast<uint32_t*>(&slice[yr]) + word, bit);
          } else {
            s_cold_insert(ckeys, cvals, cmask, yr, word, bit);
            used_cold = true;
          }
        }
      }
      if (__any_sync(0xffffffffu, used_cold) && lane == 0) s_cold_used = 1;
      __syncthreads();
      const int cold_used = s_cold_used;
      uint4 full;
      full.x = members >= 32 ? 0xffffffffu : ((1u << members) - 1);
      full.y = members >= 64 ? 0xffffffffu : (members <= 32 ? 0u : ((1u << (members - 32)) - 1));
      full.z = members >= 96 ? 0xffffffffu : (members <= 64 ? 0u : ((1u << (members - 64)) - 1));
      full.w = members >= 128 ? 0xffffffffu : (members <= 96 ? 0u : ((1u << (members - 96)) - 1));
      // 2. sweep the tile
      for (uint32_t i = threadIdx.x; i < nrows; i += blockDim.x) {
        const uint32_t k0 = lptr[i], k1 = lptr[i + 1];
        uint4 acc = make_uint4(0, 0, 0, 0);
        for (uint32_t k = k0; k < k1; ++k) {
          const uint32_t yr = lcol[k];
          const uint4 v = yr < p.hot ? slice[yr] : s_cold_lookup(ckeys, cvals, cmask, yr);
          acc.x |= v.x;
          acc.y |= v.y;
          acc.z |= v.z;
          acc.w |= v.w;
          if (acc.x == full.x && acc.y == full.y && acc.z == full.z && acc.w == full.w) break;
        }
        const uint32_t c = __popc(acc.x) + __popc(acc.y) + __popc(acc.z) + __popc(acc.w);
        cnt += c;
        if (kMode != kModeCount && c) {
          const uint32_t zc = p.dl_z[tb + i];
          const uint32_t words[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
          for (int wi = 0; wi < 4; ++wi) {
            uint32_t bits = words[wi];
            while (bits) {
              const int b = __ffs(bits) - 1;
              bits &= bits - 1;
              const uint32_t xc = p.xorder[p0 + wi * 32 + b];
              if (kMode == kModeChecksum) {
                const uint64_t h = dec.hash(xc, zc);
                sum += h;
                xr ^= h;
              } else {
                const unsigned long long idx = atomicAdd(em.cursor, 1ull);
                if (idx < em.cap) {
                  em.x[idx] = xc;
                  em.z[idx] = zc;
                }
              }
            }
          }
        }
      }
      __syncthreads();
      // 3. clear what the build set
      for (uint32_t m = warp; m < members; m += nwarps) {
        uint32_t x = p.xorder[p0 + m];
        for (uint64_t k = p.r_ptr[x] + lane; k < p.r_ptr[x + 1]; k += 32) {
          uint32_t yr = p.y_rank[p.r_col[k]];
          if (yr < p.hot) slice[yr] = make_uint4(0, 0, 0, 0);
        }
      }
      if (cold_used)
        for (uint32_t i = threadIdx.x; i < p.cold_cap; i += blockDim.x) {
          ckeys[i] = kColdEmpty;
          cvals[i] = make_uint4(0, 0, 0, 0);
        }
    }
  }
  tally_flush(tally, cnt, sum, xr);
}

}  // namespace d3g
