// join_aggregate_both (P/src/engine.cpp:537-722): one row per distinct (x, z)
// holding agg over all matches of combine(r.value, s.value), duplicates
// included.
//
// Floating-point parity. For a fixed (x, z) the reference accumulates in one
// order: R entries of x in input order (its valued CSR is a stable counting
// sort), and for each the S entries of that y in input order
// (engine.cpp:637-707; the dense/sparse split does not change the order for a
// given z). Here the candidates of a chunk of x are enumerated in exactly that
// order, sorted by (x, z) with a STABLE radix sort (so equal keys keep the
// enumeration order), and each (x, z) segment is folded sequentially by one
// thread with the reference's cell operations: combine and accumulate use
// round-to-nearest intrinsics (no FMA contraction), min/max the std::min /
// std::max comparisons (NaN and signed-zero behaviour included). The results
// are bit-identical doubles.
#pragma once

#include "common.cuh"
#include "prims.cuh"

namespace d3g {

enum : int { kAggSum = 0, kAggCount = 1, kAggMin = 2, kAggMax = 3, kAggAvg = 4 };
enum : int { kCombMul = 0, kCombAdd = 1, kCombAbsDiff = 2, kCombLeft = 3, kCombRight = 4 };

// combine_val (engine.cpp:128-142)
__device__ __forceinline__ double agg_combine(int f, double v, double u) {
  switch (f) {
    case kCombMul:
      return __dmul_rn(v, u);
    case kCombAdd:
      return __dadd_rn(v, u);
    case kCombAbsDiff:
      return fabs(__dsub_rn(v, u));
    case kCombLeft:
      return v;
    default:
      return u;
  }
}

__global__ void gather_u32_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx,
                                  uint64_t n, uint32_t* __restrict__ dst) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

// dst[i] = vals[ remap ? remap[idx[i]] : idx[i] ]
__global__ void gather_f64_kernel(const double* __restrict__ vals, const uint32_t* __restrict__ idx,
                                  const uint32_t* __restrict__ remap, uint64_t n,
                                  double* __restrict__ dst) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t j = idx[i];
    dst[i] = vals[remap ? remap[j] : j];
  }
}

__global__ void code_key_kernel(const uint32_t* __restrict__ code, uint64_t n,
                                uint64_t* __restrict__ key, uint32_t* __restrict__ idx) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    key[i] = code[i];
    idx[i] = (uint32_t)i;
  }
}

__global__ void count_codes_kernel(const uint32_t* __restrict__ code, uint64_t n,
                                   uint32_t* __restrict__ cnt) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[code[i]], 1u);
}

// candidates of x: sum over its R entries of |S_y|
__global__ void agg_cand_kernel(const uint64_t* __restrict__ rptr, const uint32_t* __restrict__ ry,
                                const uint64_t* __restrict__ sptr, uint64_t x_card,
                                uint64_t* __restrict__ cand) {
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < x_card;
       x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = 0;
    for (uint64_t e = rptr[x]; e < rptr[x + 1]; ++e) c += sptr[ry[e] + 1] - sptr[ry[e]];
    cand[x] = c;
  }
}

// Enumerates the candidates of x in [x0, x1) in the reference's order: key =
// (x - x0) << 32 | z, value = combine(r.value, s.value), written at
// coff[x] - coff[x0] + rank. One warp per x; its R entries 32 at a time, the
// (entry, S entry) space flattened across the lanes.
__global__ void agg_enum_kernel(uint64_t x0, uint64_t x1, const uint64_t* __restrict__ coff,
                                const uint64_t* __restrict__ rptr, const uint32_t* __restrict__ ry,
                                const double* __restrict__ rv, const uint64_t* __restrict__ sptr,
                                const uint32_t* __restrict__ sz, const double* __restrict__ sv,
                                int combine, uint64_t* __restrict__ key, double* __restrict__ val) {
  const uint32_t lane = lane_id();
  const uint64_t base0 = coff[x0];
  for (uint64_t x = x0 + (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); x < x1;
       x += (uint64_t)gridDim.x * (blockDim.x / 32)) {
    uint64_t out = coff[x] - base0;
    const uint64_t r0 = rptr[x], r1 = rptr[x + 1];
    for (uint64_t eb = r0; eb < r1; eb += 32) {
      const uint64_t e = eb + lane;
      uint64_t s0 = 0, s1 = 0;
      double v = 0;
      if (e < r1) {
        const uint32_t y = ry[e];
        s0 = sptr[y];
        s1 = sptr[y + 1];
        v = rv[e];
      }
      const uint32_t len = (uint32_t)(s1 - s0);
      uint32_t incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += u;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      for (uint32_t tb = 0; tb < total; tb += 32) {
        const uint32_t tf = tb + lane;
        uint32_t k = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const uint32_t probe = __shfl_sync(0xffffffffu, incl, k + step - 1);
          if (probe <= tf) k += step;
        }
        const uint32_t before = __shfl_sync(0xffffffffu, incl - len, k);
        const uint64_t sbase = __shfl_sync(0xffffffffu, s0, k);
        const double vk = __shfl_sync(0xffffffffu, v, k);
        if (tf < total) {
          const uint64_t f = sbase + (tf - before);
          const uint64_t pos = out + tf;
          key[pos] = ((x - x0) << 32) | sz[f];
          val[pos] = agg_combine(combine, vk, sv[f]);
        }
      }
      out += total;
    }
  }
}

__global__ void seg_head_kernel(const uint64_t* __restrict__ key, uint64_t n,
                                uint32_t* __restrict__ head) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || key[i] != key[i - 1]) ? 1u : 0u;
}

// One thread per (x, z) segment: cell_init / cell_update (engine.cpp:71-94)
// in enumeration order, then cell_final (:116-127).
__global__ void agg_fold_kernel(const uint64_t* __restrict__ key, const uint32_t* __restrict__ perm,
                                const double* __restrict__ val, const uint32_t* __restrict__ starts,
                                uint64_t nseg, uint64_t n, uint64_t x0, int agg,
                                const uint32_t* __restrict__ is_dense, uint32_t* __restrict__ ox,
                                uint32_t* __restrict__ oz, double* __restrict__ ov,
                                unsigned long long* __restrict__ dense_pairs,
                                unsigned int* __restrict__ too_many) {
  uint64_t nd = 0;
  for (uint64_t sg = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; sg < nseg;
       sg += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = starts[sg], e = sg + 1 < nseg ? starts[sg + 1] : n;
    const double v0 = val[perm[b]];
    double acc = agg == kAggCount ? 0.0 : v0;
    for (uint64_t i = b + 1; i < e; ++i) {
      const double v = val[perm[i]];
      if (agg == kAggSum || agg == kAggAvg)
        acc = __dadd_rn(acc, v);
      else if (agg == kAggMin)
        acc = (v < acc) ? v : acc;  // std::min(acc, v)
      else if (agg == kAggMax)
        acc = (acc < v) ? v : acc;  // std::max(acc, v)
    }
    const uint64_t cnt = e - b;
    if ((agg == kAggCount || agg == kAggAvg) && cnt > (1ull << 53)) atomicOr(too_many, 1u);
    double fin = acc;
    if (agg == kAggCount)
      fin = (double)cnt;
    else if (agg == kAggAvg)
      fin = __ddiv_rn(acc, (double)cnt);
    const uint64_t k = key[b];
    const uint32_t z = (uint32_t)(k & 0xffffffffu);
    if (is_dense && is_dense[z]) ++nd;
    if (ox) {
      ox[sg] = (uint32_t)(x0 + (k >> 32));
      oz[sg] = z;
      ov[sg] = fin;
    }
  }
  nd = warp_sum(nd);
  if (lane_id() == 0 && nd) atomicAdd(dense_pairs, (unsigned long long)nd);
}

}  // namespace d3g
