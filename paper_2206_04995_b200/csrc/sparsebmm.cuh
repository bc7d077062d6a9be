// SparseBMM (north_star subsystem 2), replacing sparse_bmm / run_chunk
// (P/src/sparsebmm.cpp:11-106). For each x, the distinct union of S_sp[y]
// over y in R[x] (Alg. 2). The reference dedups with an int64 stamp array of
// |Z| entries per thread; here each x is routed by its candidate count
// c_x = sum_y |S_sp[y]| (= the reference's inner-body count for that x):
//   * c_x <= 32: one warp per x gathers the candidates into lanes, sorts them
//     with a 32-wide bitonic network in registers and counts adjacent-unique;
//   * c_x > 32: one CTA per x with a bitmap over the COMPACT sparse-z index
//     space in shared memory (or a per-CTA slice in global memory when it
//     does not fit), atomicOr returning the old word tells whether the pair
//     is new; touched words are cleared by re-walking the candidates.
// Output: count, optional (sum, xor) fingerprint, optional code pairs
// (warp-aggregated append).
#pragma once

#include "common.cuh"

namespace d3g {

struct Decode {
  const uint64_t* rev_x;  // engine x code -> raw (null = identity)
  const uint64_t* rev_z;  // engine z code -> raw (null = identity)
  int swapped;            // caller orientation = engine (z, x)
  __device__ __forceinline__ uint64_t hash(uint32_t xc, uint32_t zc) const {
    uint64_t ex = rev_x ? rev_x[xc] : xc;
    uint64_t ez = rev_z ? rev_z[zc] : zc;
    return swapped ? pair_hash(ez, ex) : pair_hash(ex, ez);
  }
};

struct Emit {
  uint32_t* x;  // engine x codes
  uint32_t* z;  // engine z codes
  unsigned long long* cursor;
  uint64_t cap;
};

enum : int { kModeCount = 0, kModeChecksum = 1, kModeEmit = 2 };

// Warp-aggregated output reservation: every lane of a converged warp passes
// the number of pairs it will write; one atomicAdd reserves the warp's run
// and each lane gets its first slot (exclusive warp scan), so the output
// cursor sees one atomic per warp step instead of one per pair.
__device__ __forceinline__ unsigned long long warp_reserve(const Emit& em, uint32_t n) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t incl = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += u;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  unsigned long long base = 0;
  if (lane == 0 && total) base = atomicAdd(em.cursor, (unsigned long long)total);
  base = __shfl_sync(0xffffffffu, base, 0);
  return base + incl - n;
}

__device__ __forceinline__ void emit_at(const Emit& em, unsigned long long slot, uint32_t x,
                                        uint32_t z) {
  if (slot < em.cap) {
    em.x[slot] = x;
    em.z[slot] = z;
  }
}

// Optional candidate filter used by DenseEC's cold residual pass: a candidate
// (x, zi) is skipped when the hot masks of x and of dense row zi intersect
// (that pair was already produced by the hot bit-sliced pass).
struct Filter {
  const uint64_t* hx;  // [x code][kw]
  const uint64_t* hz;  // [compact index][kw]
  uint32_t kw;
  __device__ __forceinline__ bool skip(uint32_t x, uint32_t zi) const {
    if (hz == nullptr) return false;
    const uint64_t* a = hx + (uint64_t)x * kw;
    const uint64_t* b = hz + (uint64_t)zi * kw;
    for (uint32_t w = 0; w < kw; ++w)
      if (a[w] & b[w]) return true;
    return false;
  }
};

// Warp-aggregated append of (xc, zc) for lanes with `pred`.
__device__ __forceinline__ void emit_pair(const Emit& e, bool pred, uint32_t xc, uint32_t zc) {
  uint32_t m = __ballot_sync(__activemask(), pred);
  if (!pred) return;
  uint32_t lane = lane_id();
  int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if ((int)lane == leader) base = atomicAdd(e.cursor, (unsigned long long)__popc(m));
  base = __shfl_sync(m, base, leader);
  uint64_t idx = base + __popc(m & ((1u << lane) - 1));
  if (idx < e.cap) {
    e.x[idx] = xc;
    e.z[idx] = zc;
  }
}

// c_x per x and the total inner count.
__global__ void sparse_cx_kernel(const uint64_t* __restrict__ r_ptr, const uint32_t* __restrict__ r_col,
                                 uint64_t n_rows, const uint64_t* __restrict__ sp_ptr,
                                 uint64_t* __restrict__ cx, unsigned long long* __restrict__ total) {
  uint64_t acc = 0;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n_rows;
       x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = 0;
    for (uint64_t k = r_ptr[x]; k < r_ptr[x + 1]; ++k) {
      uint32_t y = r_col[k];
      c += sp_ptr[y + 1] - sp_ptr[y];
    }
    cx[x] = c;
    acc += c;
  }
  acc = warp_sum(acc);
  if (lane_id() == 0 && acc) atomicAdd(total, (unsigned long long)acc);
}

__global__ void bin_flags_kernel(const uint64_t* __restrict__ cx, uint64_t n, uint64_t small_max,
                                 uint32_t* __restrict__ small, uint32_t* __restrict__ large) {
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
       x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = cx[x];
    small[x] = (c > 0 && c <= small_max) ? 1u : 0u;
    large[x] = c > small_max ? 1u : 0u;
  }
}

__device__ __forceinline__ uint32_t bitonic32(uint32_t v) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      uint32_t o = __shfl_xor_sync(0xffffffffu, v, j);
      bool up = (lane & k) == 0;
      bool lower = (lane & j) == 0;
      uint32_t mn = v < o ? v : o, mx = v < o ? o : v;
      v = (lower == up) ? mn : mx;
    }
  }
  return v;
}

// Sorted-unique count of one warp-held candidate set of up to 32*E values
// (sentinel 0xffffffff pads), with the pair accounting of the tiers.
template <int kMode, int E>
__device__ __forceinline__ void small_tier_finish(uint32_t (&v)[E], uint32_t x,
                                                  const uint32_t* __restrict__ sparse_ids,
                                                  const Decode& dec, const Emit& em, uint64_t& cnt,
                                                  uint64_t& sum, uint64_t& xr) {
  const uint32_t lane = lane_id();
  if (E == 1) {
    v[0] = bitonic32(v[0]);
  } else {
    // bitonic over 32*E values, element e*32+lane in v[e]
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        if (j >= 32) {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int pe = e ^ (j / 32);
            if (pe > e) {
              const uint32_t i = (uint32_t)e * 32 + lane;
              const bool up = (i & k) == 0;
              const uint32_t a = v[e], bb = v[pe];
              const bool swap = up ? (a > bb) : (a < bb);
              if (swap) {
                v[e] = bb;
                v[pe] = a;
              }
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const uint32_t i = (uint32_t)e * 32 + lane;
            const uint32_t o = __shfl_xor_sync(0xffffffffu, v[e], j);
            const bool up = (i & k) == 0, lower = (lane & j) == 0;
            const uint32_t mn = v[e] < o ? v[e] : o, mx = v[e] < o ? o : v[e];
            v[e] = (lower == up) ? mn : mx;
          }
        }
      }
    }
  }
  uint32_t prev_last = 0xffffffffu;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    uint32_t prev = __shfl_up_sync(0xffffffffu, v[e], 1);
    if (lane == 0) prev = prev_last;
    const bool fresh = v[e] != 0xffffffffu && ((e == 0 && lane == 0) || v[e] != prev);
    cnt += fresh;
    if (kMode == kModeChecksum && fresh) {
      const uint64_t h = dec.hash(x, sparse_ids[v[e]]);
      sum += h;
      xr ^= h;
    }
    if (kMode == kModeEmit) emit_pair(em, fresh, x, fresh ? sparse_ids[v[e]] : 0);
    prev_last = __shfl_sync(0xffffffffu, v[e], 31);
  }
}

// One warp per x with c_x <= 128: the candidates are gathered into a
// per-warp shared buffer, sorted in registers (bitonic over 32, 64 or 128
// values) and counted unique.
constexpr int kSmallMax = 128;
template <int kMode>
__global__ void __launch_bounds__(256)
sparse_small_kernel(const uint32_t* __restrict__ xs, uint64_t n_x,
                    const uint64_t* __restrict__ r_ptr, const uint32_t* __restrict__ r_col,
                    const uint64_t* __restrict__ sp_ptr, const uint32_t* __restrict__ sp_col,
                    const uint32_t* __restrict__ sparse_ids, Decode dec, Emit em, Tally* tally,
                    Filter flt) {
  __shared__ uint32_t buf[8][kSmallMax];
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  uint64_t cnt = 0, sum = 0, xr = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * 8 + w; i < n_x; i += (uint64_t)gridDim.x * 8) {
    uint32_t x = xs[i];
    uint64_t r0 = r_ptr[x], r1 = r_ptr[x + 1];
    uint32_t nc = 0;
    for (uint64_t base = r0; base < r1; base += 32) {
      uint64_t k = base + lane;
      uint32_t len = 0;
      uint64_t s0 = 0;
      if (k < r1) {
        const uint32_t y = r_col[k];
        s0 = sp_ptr[y];
        len = (uint32_t)(sp_ptr[y + 1] - s0);
      }
      uint32_t incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += u;
      }
      uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      uint32_t off = nc + incl - len;
      for (uint32_t t = 0; t < len && off + t < kSmallMax; ++t) buf[w][off + t] = sp_col[s0 + t];
      nc += tot;
    }
    __syncwarp();
    auto load = [&](uint32_t idx) {
      uint32_t v = idx < nc ? buf[w][idx] : 0xffffffffu;
      if (v != 0xffffffffu && flt.skip(x, v)) v = 0xffffffffu;
      return v;
    };
    if (nc <= 32) {
      uint32_t v[1] = {load(lane)};
      __syncwarp();
      small_tier_finish<kMode, 1>(v, x, sparse_ids, dec, em, cnt, sum, xr);
    } else if (nc <= 64) {
      uint32_t v[2] = {load(lane), load(32 + lane)};
      __syncwarp();
      small_tier_finish<kMode, 2>(v, x, sparse_ids, dec, em, cnt, sum, xr);
    } else {
      uint32_t v[4] = {load(lane), load(32 + lane), load(64 + lane), load(96 + lane)};
      __syncwarp();
      small_tier_finish<kMode, 4>(v, x, sparse_ids, dec, em, cnt, sum, xr);
    }
  }
  tally_flush(tally, cnt, sum, xr);
}

// ---------------------------------------------------------------------------
// Warp-private shared-memory hash set, one warp per x with 32 < c_x <= cap/2.
constexpr int kHashWarps = 4;
constexpr uint32_t kHashCap = 2048;  // u32 slots per warp (8 KB)
constexpr uint32_t kHashEmpty = 0xffffffffu;

template <int kMode>
__global__ void __launch_bounds__(kHashWarps * 32)
sparse_hash_kernel(const uint32_t* __restrict__ xs, uint64_t n_x,
                   const uint64_t* __restrict__ r_ptr, const uint32_t* __restrict__ r_col,
                   const uint64_t* __restrict__ sp_ptr, const uint32_t* __restrict__ sp_col,
                   const uint32_t* __restrict__ sparse_ids, Decode dec, Emit em, Tally* tally,
                   Filter flt) {
  __shared__ uint32_t table[kHashWarps][kHashCap];
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  uint32_t* t = table[w];
  for (uint32_t i = lane; i < kHashCap; i += 32) t[i] = kHashEmpty;
  __syncwarp();
  uint64_t cnt = 0, sum = 0, xr = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * kHashWarps + w; i < n_x; i += (uint64_t)gridDim.x * kHashWarps) {
    uint32_t x = xs[i];
    for (uint64_t k = r_ptr[x]; k < r_ptr[x + 1]; ++k) {
      uint32_t y = r_col[k];
      uint64_t s0 = sp_ptr[y], s1 = sp_ptr[y + 1];
      for (uint64_t base = s0; base < s1; base += 32) {
        uint64_t q = base + lane;
        bool fresh = false;
        uint32_t zi = 0;
        if (q < s1 && !flt.skip(x, sp_col[q])) {
          zi = sp_col[q];
          uint32_t s = (zi * 0x9e3779b1u) >> 21;  // 11 bits -> [0, 2048)
          for (;;) {
            uint32_t prev = atomicCAS(&t[s], kHashEmpty, zi);
            if (prev == kHashEmpty) { fresh = true; break; }
            if (prev == zi) break;
            s = (s + 1) & (kHashCap - 1);
          }
        }
        cnt += fresh;
        if (kMode == kModeChecksum && fresh) {
          uint64_t h = dec.hash(x, sparse_ids[zi]);
          sum += h;
          xr ^= h;
        }
        if (kMode == kModeEmit) emit_pair(em, fresh, x, fresh ? sparse_ids[zi] : 0);
      }
    }
    __syncwarp();
    for (uint32_t j = lane; j < kHashCap; j += 32) t[j] = kHashEmpty;
    __syncwarp();
  }
  tally_flush(tally, cnt, sum, xr);
}

// ---------------------------------------------------------------------------
// Bitset-row tier for a small sparse side (n_sparse <= 32 * 32 * kBitsetMaxWords
// bits): S_sp rows are kept as bitsets over the compact sparse index; one warp
// per x ORs the rows of its y in registers (lane l owns words l, l+32, ...)
// and pop-counts. No atomics, no dedup structure.
constexpr int kBitsetMaxWordsPerLane = 8;  // 8192 sparse z

__global__ void sparse_rowbits_build_kernel(const uint64_t* __restrict__ sp_ptr,
                                            const uint32_t* __restrict__ sp_col, uint64_t y_card,
                                            uint32_t n_words, uint32_t* __restrict__ rows) {
  for (uint64_t y = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); y < y_card;
       y += (uint64_t)gridDim.x * (blockDim.x / 32))
    for (uint64_t k = sp_ptr[y] + lane_id(); k < sp_ptr[y + 1]; k += 32) {
      uint32_t zi = sp_col[k];
      atomicOr(&rows[y * n_words + (zi >> 5)], 1u << (zi & 31));
    }
}

template <int kMode, int kWPL>
__global__ void __launch_bounds__(256)
sparse_bitset_kernel(const uint32_t* __restrict__ xs, uint64_t n_x,
                     const uint64_t* __restrict__ r_ptr, const uint32_t* __restrict__ r_col,
                     const uint64_t* __restrict__ sp_ptr, const uint32_t* __restrict__ rows,
                     uint32_t n_words, const uint32_t* __restrict__ sparse_ids, Decode dec, Emit em,
                     Tally* tally) {
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t cnt = 0, sum = 0, xr = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * nw + w; i < n_x; i += (uint64_t)gridDim.x * nw) {
    uint32_t x = xs[i];
    uint32_t acc[kWPL];
#pragma unroll
    for (int j = 0; j < kWPL; ++j) acc[j] = 0;
    for (uint64_t k = r_ptr[x]; k < r_ptr[x + 1]; ++k) {
      uint32_t y = r_col[k];
      if (sp_ptr[y + 1] == sp_ptr[y]) continue;
      const uint32_t* row = rows + (uint64_t)y * n_words;
#pragma unroll
      for (int j = 0; j < kWPL; ++j) {
        uint32_t wi = lane + 32 * j;
        if (wi < n_words) acc[j] |= __ldg(row + wi);
      }
    }
#pragma unroll
    for (int j = 0; j < kWPL; ++j) {
      cnt += __popc(acc[j]);
      if (kMode != kModeCount) {
        uint32_t bits = acc[j];
        while (bits) {
          int b = __ffs(bits) - 1;
          bits &= bits - 1;
          uint32_t zc = sparse_ids[(lane + 32 * j) * 32 + b];
          if (kMode == kModeChecksum) {
            uint64_t h = dec.hash(x, zc);
            sum += h;
            xr ^= h;
          } else {
            unsigned long long idx = atomicAdd(em.cursor, 1ull);
            if (idx < em.cap) {
              em.x[idx] = x;
              em.z[idx] = zc;
            }
          }
        }
      }
    }
  }
  tally_flush(tally, cnt, sum, xr);
}

// One CTA per x with c_x > 32; bitmap of n_words 32-bit words in smem
// (kGlobalBitmap = false) or a per-CTA slice of gbm (true).
template <int kMode, bool kGlobalBitmap>
__global__ void __launch_bounds__(512)
sparse_large_kernel(const uint32_t* __restrict__ xs, uint64_t n_x, const uint64_t* __restrict__ cx,
                    uint64_t cx_base, const uint64_t* __restrict__ r_ptr, const uint32_t* __restrict__ r_col,
                    const uint64_t* __restrict__ sp_ptr, const uint32_t* __restrict__ sp_col,
                    const uint32_t* __restrict__ sparse_ids, uint32_t n_words, uint32_t* gbm,
                    Decode dec, Emit em, Tally* tally, Filter flt) {
  extern __shared__ uint32_t smem_bm[];
  uint32_t* bm = kGlobalBitmap ? gbm + (uint64_t)blockIdx.x * n_words : smem_bm;
  for (uint32_t i = threadIdx.x; i < n_words; i += blockDim.x) bm[i] = 0;
  __syncthreads();
  uint64_t cnt = 0, sum = 0, xr = 0;
  for (uint64_t i = blockIdx.x; i < n_x; i += gridDim.x) {
    uint32_t x = xs[i];
    uint64_t r0 = r_ptr[x], r1 = r_ptr[x + 1];
    for (uint64_t k = r0; k < r1; ++k) {
      uint32_t y = r_col[k];
      uint64_t s0 = sp_ptr[y], s1 = sp_ptr[y + 1];
      for (uint64_t t = s0 + threadIdx.x; t < s1 + ((blockDim.x - (s1 - s0) % blockDim.x) % blockDim.x);
           t += blockDim.x) {
        bool fresh = false;
        uint32_t zi = 0;
        if (t < s1 && !flt.skip(x, sp_col[t])) {
          zi = sp_col[t];
          uint32_t bit = 1u << (zi & 31);
          uint32_t old = atomicOr(&bm[zi >> 5], bit);
          fresh = (old & bit) == 0;
        }
        cnt += fresh;
        if (kMode == kModeChecksum && fresh) {
          uint64_t h = dec.hash(x, sparse_ids[zi]);
          sum += h;
          xr ^= h;
        }
        if (kMode == kModeEmit) emit_pair(em, fresh, x, fresh ? sparse_ids[zi] : 0);
      }
    }
    __syncthreads();
    // clear: whole bitmap when cheaper than re-walking the candidates
    if (cx[x - cx_base] >= n_words) {
      for (uint32_t j = threadIdx.x; j < n_words; j += blockDim.x) bm[j] = 0;
    } else {
      for (uint64_t k = r0; k < r1; ++k) {
        uint32_t y = r_col[k];
        for (uint64_t t = sp_ptr[y] + threadIdx.x; t < sp_ptr[y + 1]; t += blockDim.x)
          bm[sp_col[t] >> 5] = 0;
      }
    }
    __syncthreads();
  }
  tally_flush(tally, cnt, sum, xr);
}

}  // namespace d3g
