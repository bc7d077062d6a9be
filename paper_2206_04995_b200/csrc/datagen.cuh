// Convention-G synthetic inputs generated directly in HBM.
// SplitMix64 (P/include/dim3/datagen.hpp:176-193) is a counter generator:
// draw k of a stream is mix64(seed + (k+1) * golden), so every row is
// produced independently by one thread. Zipf draws use the reference's exact
// CDF (sequential double sum of r^-alpha, P/src/datagen.cpp:10-25) computed
// on the host and an upper_bound search on the device, so the bytes match
// the CPU generator bit for bit.
#pragma once

#include "common.cuh"

namespace d3g {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

__device__ __forceinline__ uint64_t sm_draw(uint64_t seed, uint64_t k) {
  return mix64(seed + (k + 1) * kGolden);
}
__device__ __forceinline__ uint64_t sm_bounded(uint64_t r, uint64_t n) { return __umul64hi(r, n); }
__device__ __forceinline__ uint64_t zipf_pick(uint64_t r, const double* __restrict__ cum, uint64_t n) {
  double u = (double)(r >> 11) * 0x1.0p-53 * cum[n - 1];
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (cum[mid] > u)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo == n ? n - 1 : lo;
}

struct GenSpec {
  int cfg;
  uint64_t seed, n_rows, nx, ny;
  int zipf;        // y drawn from Zipf over ny
  int pools;       // cfg4: values drawn through pools
  uint64_t base;   // first draw index of this side's rows
  uint64_t pool_off;
};

__global__ void gen_kernel(GenSpec g, const double* __restrict__ cum, uint64_t lo, uint64_t hi,
                           uint64_t* __restrict__ left, uint64_t* __restrict__ right) {
  const uint64_t NP = 1000000, NY = 100000, P = 2 * NP + NY;
  for (uint64_t i = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t a, b;
    if (!g.pools) {
      a = sm_bounded(sm_draw(g.seed, g.base + 2 * i), g.nx);
      uint64_t rb = sm_draw(g.seed, g.base + 2 * i + 1);
      b = g.zipf ? zipf_pick(rb, cum, g.ny) : sm_bounded(rb, g.ny);
    } else {
      uint64_t ai = sm_bounded(sm_draw(g.seed, P + g.base + 2 * i), NP);
      uint64_t bi = zipf_pick(sm_draw(g.seed, P + g.base + 2 * i + 1), cum, NY);
      a = sm_draw(g.seed, g.pool_off + ai);
      b = sm_draw(g.seed, 2 * NP + bi);
    }
    left[i - lo] = a;
    right[i - lo] = b;
  }
}

inline uint64_t cfg_rows(int cfg) {
  switch (cfg) {
    case 1: return 100000ull;
    case 2: return 5000000ull;
    case 3: return 20000000ull;
    case 4: return 10000000ull;
    case 5: return 200000000ull;
  }
  return 0;
}

inline GenSpec gen_spec(int cfg, int side) {
  GenSpec g{};
  g.cfg = cfg;
  g.seed = (uint64_t)cfg;
  g.n_rows = cfg_rows(cfg);
  if (cfg == 2) side = 0;  // S := R
  g.base = side == 0 ? 0 : 2 * g.n_rows;
  switch (cfg) {
    case 1: g.nx = 10000; g.ny = 1000; break;
    case 2: g.nx = 200000; g.ny = 50000; g.zipf = 1; break;
    case 3: g.nx = 2000000; g.ny = 10000000; break;
    case 4: g.nx = 1000000; g.ny = 100000; g.zipf = 1; g.pools = 1;
            g.pool_off = side == 0 ? 0 : 1000000; break;
    case 5: g.nx = 10000000; g.ny = 1000000; g.zipf = 1; break;
  }
  return g;
}

inline double gen_alpha(int cfg) { return cfg == 2 ? 1.0 : cfg == 4 ? 0.8 : 1.2; }

}  // namespace d3g
