// DenseEC v3: hot bit-sliced existence + cold residual join.
//
// Rank the y codes by R-side degree (hottest first) and fix K (a multiple of
// 64). For a pair (x, dense z):
//   hit  <=>  R_hot[x] & S_hot[z] != 0   OR   R_cold[x] & S_cold[z] != 0.
// P1 (this file, dense_hot_kernel) counts the pairs with a common HOT y,
// bit-sliced over groups of 128 live x: every dense z carries a K-bit mask
// hz[z] of its hot ranks; every x group carries T[g][r] = {x in g : rank r in
// R[x]} (uint4, 128 bits) for r < K. For each (z, group):
//      acc = OR_{r in hz[z]} T[g][r]   (early exit once acc == all-live)
// and popc(acc) pairs are hit. T for a batch of groups is staged into shared
// memory with one TMA bulk copy (cp.async.bulk + mbarrier transaction count).
// P2 (the cold kernels at the end of this file: dense_cold_kernel, or
// dense_cold_hash_kernel with its CTA-hash and global-bitmap overflow tiers)
// counts pairs that share only COLD y: the cold join R_cold x S_cold
// restricted to dense z, dedup'd per x, skipping candidates whose hot masks
// already intersect. The two parts are disjoint and together equal the
// reference's dense_ec output (P/src/denseec.cpp:8-86): {(x, z) : R[x] and
// S[z] share a y}, z dense.
#pragma once

#include "sparsebmm.cuh"

#ifndef D3G_COMPARISON_KERNELS
#define D3G_COMPARISON_KERNELS 0
#endif

namespace d3g {

#ifndef D3G_HOT_THREADS
#define D3G_HOT_THREADS 768  // 24 warps, 80 registers (1024: 64 and twice the spills; cfg5 hot 20.8 -> 20.1 ms)
#endif
constexpr int kHotThreads = D3G_HOT_THREADS;
// pivot classes: up to 6 pivots (the top ranks), 64 classes of x and rows
constexpr uint32_t kMaxPivots = 6, kMaxClasses = 1u << kMaxPivots;

struct HotParams {
  const uint4* T;          // [batch of 32 groups][K][32] (uint4 = 128 member bits)
  const uint64_t* hz;      // [n_dense][K/64]
  const uint32_t* xorder;  // live x codes by position
  const uint32_t* dl_z;    // z code per dense row position
  uint64_t n_live, n_dense;
  uint32_t groups, K, kw;  // kw = K / 64
  uint32_t batch;          // groups per smem batch
  uint32_t z_chunks;       // z ranges per batch (units = batches * z_chunks)
  unsigned int* work;
  // Pivot plan (count-only): x and dense rows are classed by which of the
  // top ranks (pivots) they hold; a batch whose x share the pivot set k (the
  // AND of their classes) tests only the rows of the classes sharing no pivot
  // with k (kind k: those class runs of the class-major row order); every
  // other (x, row) pair of that batch is a hit. plan_units == 0: every batch
  // tests all rows in z_chunks ranges.
  const uint32_t* unit_off = nullptr;  // [n_batches + 1] first unit of each batch
  const uint8_t* batch_kind = nullptr; // [n_batches] row-range kind 0..15
  uint64_t run_lo[kMaxClasses + 1] = {};  // class c's rows: [run_lo[c], run_lo[c + 1]) (class-major)
  uint32_t run_zc[kMaxClasses] = {};      // chunks (units per batch) of class c's run
  uint32_t n_classes = 1;
  uint32_t plan_units = 0;
  uint32_t plan_on = 0;  // 1: units follow the plan (plan_units may be 0)
  // z-split (zsplit.cuh): the long rows' list tails, gathered (sorted row
  // ids, tail starts, ranks); null: the tails are read from dl_ptr / dl_col
  const uint32_t* tail_rows = nullptr;
  const uint64_t* tail_ptr = nullptr;
  const uint32_t* tail_col = nullptr;
  uint32_t n_tail = 0;
};

// Unit -> (batch, row range). Units are batch-major.
__device__ __forceinline__ void hot_unit(const HotParams& p, uint32_t n_batches, uint32_t unit,
                                         uint32_t& bi, uint64_t& z_lo, uint64_t& z_hi) {
  if (!p.plan_on) {
    bi = unit / p.z_chunks;
    const uint32_t zc = unit % p.z_chunks;
    z_lo = p.n_dense * zc / p.z_chunks;
    z_hi = p.n_dense * (zc + 1) / p.z_chunks;
    return;
  }
  uint32_t lo = 0, hi = n_batches;  // last batch whose first unit <= unit
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (p.unit_off[mid] <= unit) lo = mid; else hi = mid;
  }
  bi = lo;
  const uint32_t k = p.batch_kind[lo];
  uint32_t u = unit - p.unit_off[lo];
  z_lo = z_hi = 0;
  for (uint32_t c = 0; c < p.n_classes; ++c) {  // the runs of kind k, in order
    if (c & k) continue;
    const uint32_t zcs = p.run_zc[c];
    if (u < zcs) {
      const uint64_t r0 = p.run_lo[c], n = p.run_lo[c + 1] - r0;
      z_lo = r0 + n * u / zcs;
      z_hi = r0 + n * (u + 1) / zcs;
      return;
    }
    u -= zcs;
  }
}

__device__ __forceinline__ uint32_t hot_units(const HotParams& p, uint32_t n_batches) {
  return p.plan_on ? p.plan_units : n_batches * p.z_chunks;
}

// Pivot class of each live x: bit q = holds y_of_rank[q] (q < n_piv; rows are
// sorted by y, binary search); out[16] counts per class.
__global__ void pivot_class_x_kernel(const uint32_t* __restrict__ xorder, uint64_t n_live,
                                     const uint64_t* __restrict__ r_ptr,
                                     const uint32_t* __restrict__ r_col,
                                     const uint32_t* __restrict__ y_of_rank, uint32_t n_piv,
                                     uint32_t* __restrict__ cls, unsigned long long* __restrict__ out) {
  __shared__ unsigned int c8[kMaxClasses];
  if (threadIdx.x < kMaxClasses) c8[threadIdx.x] = 0;
  __syncthreads();
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n_live;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = xorder[p];
    const uint64_t e = r_ptr[x + 1];
    uint32_t c = 0;
    for (uint32_t q = 0; q < n_piv; ++q) {
      const uint32_t yq = y_of_rank[q];
      uint64_t lo = r_ptr[x], hi = e;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (r_col[mid] < yq) lo = mid + 1; else hi = mid;
      }
      if (lo < e && r_col[lo] == yq) c |= 1u << q;
    }
    cls[p] = c;
    atomicAdd(&c8[c], 1u);
  }
  __syncthreads();
  if (threadIdx.x < kMaxClasses && c8[threadIdx.x])
    atomicAdd(&out[threadIdx.x], (unsigned long long)c8[threadIdx.x]);
}

// Dense rows per pivot class (bit q = holds rank q; the lists are
// rank-ascending, so the pivots sit at the front) and folded sparse rows per
// class: out[0, kMaxClasses) rows, out[kMaxClasses, 2 kMaxClasses) flagged rows.
__global__ void pivot_class_rows_kernel(const uint64_t* __restrict__ dl_ptr,
                                        const uint32_t* __restrict__ dl_col, uint64_t n,
                                        uint32_t n_piv, const uint8_t* __restrict__ row_sp,
                                        unsigned long long* __restrict__ out) {
  __shared__ unsigned int c16[2 * kMaxClasses];
  if (threadIdx.x < 2 * kMaxClasses) c16[threadIdx.x] = 0;
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k0 = dl_ptr[i], k1 = dl_ptr[i + 1];
    uint32_t c = 0;
    for (uint64_t k = k0; k < k1 && k < k0 + n_piv; ++k) {
      const uint32_t r = dl_col[k];
      if (r < n_piv) c |= 1u << r; else break;
    }
    atomicAdd(&c16[c], 1u);
    if (row_sp && row_sp[i]) atomicAdd(&c16[kMaxClasses + c], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 2 * kMaxClasses && c16[threadIdx.x])
    atomicAdd(&out[threadIdx.x], (unsigned long long)c16[threadIdx.x]);
}

// T, hx from the live x in degree order: warp per x position.
__global__ void hot_build_x_kernel(const uint32_t* __restrict__ xorder, uint64_t n_live,
                                   const uint64_t* __restrict__ r_ptr,
                                   const uint32_t* __restrict__ r_col,
                                   const uint32_t* __restrict__ y_rank, uint32_t K, uint32_t kw,
                                   uint32_t* __restrict__ T, unsigned long long* __restrict__ hx,
                                   uint64_t pos_base = 0 /* T position of xorder[0] */) {
  // 8 lanes per x (rows hold ~10-30 entries)
  const uint32_t sl = threadIdx.x & 7;
  for (uint64_t p = (uint64_t)blockIdx.x * (blockDim.x / 8) + (threadIdx.x >> 3); p < n_live;
       p += (uint64_t)gridDim.x * (blockDim.x / 8)) {
    uint32_t x = xorder[p];
    if (x == 0xffffffffu) continue;  // an empty slot of a class-aligned batch
    const uint64_t tp = pos_base + p;
    uint64_t g = tp >> 7;
    uint64_t bi = g >> 5, gl = g & 31;
    uint32_t b = (uint32_t)(tp & 127);
    for (uint64_t k = r_ptr[x] + sl; k < r_ptr[x + 1]; k += 8) {
      uint32_t r = y_rank[r_col[k]];
      if (r < K) {
        atomicOr(&T[((bi * K + r) * 32 + gl) * 4 + (b >> 5)], 1u << (b & 31));
        atomicOr(&hx[(uint64_t)x * kw + (r >> 6)], 1ull << (r & 63));
      }
    }
  }
}

// hx (K = 256: four 64-bit words per x) from the R rows of the live x, 8
// lanes per x each OR-ing its entries' hot ranks into registers, reduced
// across the 8 lanes and stored once (no atomics).
__global__ void hx_build_kernel(const uint32_t* __restrict__ xorder, uint64_t n_live,
                                const uint64_t* __restrict__ r_ptr,
                                const uint32_t* __restrict__ r_col,
                                const uint32_t* __restrict__ y_rank, uint32_t K,
                                uint4* __restrict__ hx4) {
  // xorder null: the x codes [0, n_live) in order (coalesced row reads; rows
  // without entries produce zero masks)
  const uint32_t sl = threadIdx.x & 7;
  for (uint64_t p0 = (uint64_t)blockIdx.x * (blockDim.x / 8); p0 < n_live;
       p0 += (uint64_t)gridDim.x * (blockDim.x / 8)) {
    const uint64_t p = p0 + (threadIdx.x >> 3);
    uint64_t w[4] = {0, 0, 0, 0};
    uint32_t x = 0xffffffffu;
    if (p < n_live) {
      x = xorder ? xorder[p] : (uint32_t)p;
      for (uint64_t k = r_ptr[x] + sl; k < r_ptr[x + 1]; k += 8) {
        const uint32_t r = y_rank[r_col[k]];
        if (r < K) w[r >> 6] |= 1ull << (r & 63);
      }
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1)
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] |= __shfl_xor_sync(0xffffffffu, w[q], o);
    if (p < n_live && sl == 0)
      st256(hx4 + 2 * (uint64_t)x,
            make_uint4((uint32_t)w[0], (uint32_t)(w[0] >> 32), (uint32_t)w[1], (uint32_t)(w[1] >> 32)),
            make_uint4((uint32_t)w[2], (uint32_t)(w[2] >> 32), (uint32_t)w[3], (uint32_t)(w[3] >> 32)));
  }
}

// The same masks, one thread per x code in order (all x of R): a thread walks
// its own row (adjacent threads read adjacent rows: L1 serves the rest of
// each line), four rank lookups in flight, no shuffles; rows without
// entries get zero masks.
__global__ void hx_build_rows_kernel(uint64_t n_rows, const uint64_t* __restrict__ r_ptr,
                                     const uint32_t* __restrict__ r_col,
                                     const uint32_t* __restrict__ y_rank, uint32_t K,
                                     uint4* __restrict__ hx4) {
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n_rows;
       x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t w[4] = {0, 0, 0, 0};
    const uint64_t e = r_ptr[x + 1];
    for (uint64_t k = r_ptr[x]; k < e; k += 4) {
      uint32_t y[4], r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) y[u] = k + u < e ? r_col[k + u] : 0xffffffffu;
#pragma unroll
      for (int u = 0; u < 4; ++u) r[u] = y[u] != 0xffffffffu ? y_rank[y[u]] : K;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (r[u] < K) w[r[u] >> 6] |= 1ull << (r[u] & 63);
    }
    st256(hx4 + 2 * x,
          make_uint4((uint32_t)w[0], (uint32_t)(w[0] >> 32), (uint32_t)w[1], (uint32_t)(w[1] >> 32)),
          make_uint4((uint32_t)w[2], (uint32_t)(w[2] >> 32), (uint32_t)w[3], (uint32_t)(w[3] >> 32)));
  }
}

// Pivot class of each live x read off its hot mask (pivot q = rank q, bit q
// of word 0); out[16] counts per class.
__global__ void pivot_class_hx_kernel(const uint32_t* __restrict__ xorder, uint64_t n_live,
                                      const unsigned long long* __restrict__ hx, uint32_t kw,
                                      uint32_t n_piv, uint32_t* __restrict__ cls,
                                      unsigned long long* __restrict__ out) {
  __shared__ unsigned int c16[kMaxClasses];
  if (threadIdx.x < kMaxClasses) c16[threadIdx.x] = 0;
  __syncthreads();
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n_live;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = (uint32_t)(hx[(uint64_t)xorder[p] * kw] & ((1u << n_piv) - 1u));
    cls[p] = c;
    atomicAdd(&c16[c], 1u);
  }
  __syncthreads();
  if (threadIdx.x < kMaxClasses && c16[threadIdx.x])
    atomicAdd(&out[threadIdx.x], (unsigned long long)c16[threadIdx.x]);
}

// The slice tables T from the hot masks: a warp owns one 128-x group (lane l
// holds positions l, l + 32, l + 64, l + 96: the group's four words), so for
// rank r the group's 16-byte slice is four ballots, kept by lane r % 32 and
// stored with one 16-byte store per lane per 32 ranks. Every slice of every
// batch is written (no memset, no atomics); positions past n or holding the
// empty marker contribute no bits.
__global__ void hot_T_from_hx_kernel(const uint32_t* __restrict__ xorder, uint64_t n,
                                     uint64_t n_pos /* whole batches */,
                                     const uint4* __restrict__ hx4, uint32_t K,
                                     uint4* __restrict__ T) {
  const uint32_t lane = lane_id();
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t g = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g * 128 < n_pos;
       g += nw) {
    uint32_t w[4][8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t p = g * 128 + (uint64_t)j * 32 + lane;
      uint4 a = make_uint4(0, 0, 0, 0), b = a;
      if (p < n) {
        const uint32_t x = xorder[p];
        if (x != 0xffffffffu) ld256(hx4 + 2 * (uint64_t)x, a, b);
      }
      w[j][0] = a.x; w[j][1] = a.y; w[j][2] = a.z; w[j][3] = a.w;
      w[j][4] = b.x; w[j][5] = b.y; w[j][6] = b.z; w[j][7] = b.w;
    }
    const uint64_t bi = g >> 5, gl = g & 31;
    uint4* base = T + (bi * K) * 32 + gl;  // rank r's slice at base + r * 32
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if ((uint32_t)q * 32 >= K) break;
      uint4 mine = make_uint4(0, 0, 0, 0);  // lane t keeps rank q * 32 + t
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const uint32_t m0 = __ballot_sync(0xffffffffu, (w[0][q] >> t) & 1u);
        const uint32_t m1 = __ballot_sync(0xffffffffu, (w[1][q] >> t) & 1u);
        const uint32_t m2 = __ballot_sync(0xffffffffu, (w[2][q] >> t) & 1u);
        const uint32_t m3 = __ballot_sync(0xffffffffu, (w[3][q] >> t) & 1u);
        if (lane == (uint32_t)t) mine = make_uint4(m0, m1, m2, m3);
      }
      base[(uint64_t)(q * 32 + lane) * 32] = mine;
    }
  }
}

// hz from the dense lists (ranks ascending: the hot ranks are a prefix).
__global__ void hot_build_z_kernel(const uint64_t* __restrict__ dl_ptr,
                                   const uint32_t* __restrict__ dl_col, uint64_t n_dense,
                                   uint32_t K, uint32_t kw, unsigned long long* __restrict__ hz) {
  const uint32_t sl = threadIdx.x & 7;  // 8 lanes per row
  for (uint64_t i = (uint64_t)blockIdx.x * (blockDim.x / 8) + (threadIdx.x >> 3); i < n_dense;
       i += (uint64_t)gridDim.x * (blockDim.x / 8)) {
    const uint64_t e = dl_ptr[i + 1];
    for (uint64_t k = dl_ptr[i] + sl; k < e; k += 8) {
      const uint32_t r = dl_col[k];
      if (r >= K) break;  // ranks ascend: the hot prefix ended
      atomicOr(&hz[i * kw + (r >> 6)], 1ull << (r & 63));
    }
  }
}


// Pairs whose dense row is a folded-in SPARSE z (row_sp[i] != 0) are also
// counted separately, so the report keeps the reference's pairs_sparse /
// pairs_dense split when the sparse side runs through this engine.
__device__ __forceinline__ void flush_sp(unsigned long long* cnt_sp, uint64_t v) {
  v = warp_sum(v);
  if (cnt_sp && lane_id() == 0 && v) atomicAdd(cnt_sp, (unsigned long long)v);
}

// --- TMA bulk copy helpers (sm_90+ PTX, used on sm_100a) -------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
// Bounded wait on the TMA transaction barrier: a byte-count or phase mismatch
// traps (the launch fails with an error the host reports) instead of hanging
// the device. try_wait suspends for a bounded time per call, so 2^24 polls
// are seconds, far beyond any real copy.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  for (uint32_t it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(a), "r"(phase)
        : "memory");
    if (ok) return;
    if (it > (1u << 24)) asm volatile("trap;");
  }
}

__device__ __forceinline__ uint4 full_mask(uint32_t members) {
  uint4 f;
  f.x = members >= 32 ? 0xffffffffu : ((1u << members) - 1);
  f.y = members >= 64 ? 0xffffffffu : (members <= 32 ? 0u : ((1u << (members - 32)) - 1));
  f.z = members >= 96 ? 0xffffffffu : (members <= 64 ? 0u : ((1u << (members - 64)) - 1));
  f.w = members >= 128 ? 0xffffffffu : (members <= 96 ? 0u : ((1u << (members - 96)) - 1));
  return f;
}

// P1 kernel. A batch = 32 consecutive 128-x groups; its slice table lives in
// shared memory r-major, Ts[r][lane] (uint4), so for a fixed hot rank r the
// 32 lanes read 512 contiguous bytes (conflict-free LDS.128). One warp owns
// one dense z at a time and walks the hot prefix of z's list (ranks ascending,
// warp-uniform broadcast loads); lane l accumulates group l's 128-bit hit mask.
// The batch table (K * 512 B, contiguous in global memory) is staged by one
// TMA bulk copy per batch change.
template <int kMode>
__global__ void __launch_bounds__(kHotThreads, 1)
dense_hot_kernel(HotParams p, const uint64_t* __restrict__ dl_ptr,
                 const uint32_t* __restrict__ dl_col, Decode dec, Emit em, Tally* tally) {
  extern __shared__ __align__(128) uint4 Ts[];  // [K][32]
  __shared__ __align__(8) uint64_t bar;
  __shared__ unsigned int s_unit;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t n_batches = (p.groups + 31) / 32;
  const unsigned int n_units = n_batches * p.z_chunks;
  uint64_t cnt = 0, sum = 0, xr = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  int cur_batch = -1;
  for (;;) {
    if (threadIdx.x == 0) s_unit = atomicAdd(p.work, 1u);
    __syncthreads();
    const unsigned int unit = s_unit;
    if (unit >= n_units) break;
    const uint32_t bi = unit / p.z_chunks, zc_i = unit % p.z_chunks;
    if ((int)bi != cur_batch) {
      if (threadIdx.x == 0) {
        const uint32_t bytes = p.K * 32u * 16u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar, bytes);
        tma_bulk_g2s(Ts, p.T + (uint64_t)bi * p.K * 32, bytes, &bar);
      }
      mbar_wait(&bar, phase);
      phase ^= 1;
      cur_batch = (int)bi;
    }
    const uint32_t g = bi * 32 + lane;  // this lane's group
    const bool lane_live = g < p.groups;
    const uint64_t gp0 = (uint64_t)g * 128;
    const uint32_t members =
        lane_live ? (uint32_t)((p.n_live - gp0) < 128 ? (p.n_live - gp0) : 128) : 0;
    const uint4 full = full_mask(members);
    const uint64_t z_lo = p.n_dense * zc_i / p.z_chunks, z_hi = p.n_dense * (zc_i + 1) / p.z_chunks;
    for (uint64_t i = z_lo + warp; i < z_hi; i += nwarps) {
      const uint64_t k0 = dl_ptr[i], k1 = dl_ptr[i + 1];
      uint4 acc = make_uint4(0, 0, 0, 0);
      // the hot prefix of z's list, 32 entries per coalesced lane-load,
      // broadcast with shuffles; LDS.128 of successive ranks are independent
      for (uint64_t base = k0; base < k1; base += 32) {
        const uint32_t mine = base + lane < k1 ? dl_col[base + lane] : 0xffffffffu;
        const uint32_t nhot = __popc(__ballot_sync(0xffffffffu, mine < p.K));
#pragma unroll 4
        for (uint32_t j = 0; j < nhot; ++j) {
          const uint32_t r = __shfl_sync(0xffffffffu, mine, j);
          const uint4 v = Ts[r * 32 + lane];
          acc.x |= v.x;
          acc.y |= v.y;
          acc.z |= v.z;
          acc.w |= v.w;
        }
        if (nhot < 32) break;  // ranks ascend: the hot prefix ended
      }
      const uint32_t c = __popc(acc.x) + __popc(acc.y) + __popc(acc.z) + __popc(acc.w);
      cnt += c;
      if (kMode != kModeCount && c) {
        const uint32_t zc = p.dl_z[i];
        const uint32_t words[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
        for (int wi = 0; wi < 4; ++wi) {
          uint32_t bits = words[wi];
          while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const uint32_t xc = p.xorder[gp0 + wi * 32 + b];
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
    __syncthreads();  // Ts may be overwritten by the next unit's copy
  }
  tally_flush(tally, cnt, sum, xr);
}

// --- P1 with packed hot records (K <= 256) ---------------------------------
// Each dense row's hot prefix is packed once into a 32-byte record of u8
// ranks (first 32 hot ranks) plus its hot count. A warp then takes 32 rows per
// step with ONE coalesced 1 KB load (lane j holds row j's record), prefetched a
// step ahead, and broadcasts the ranks with one shuffle per 4 ranks. This
// removes the per-row dependent dl_ptr -> dl_col global loads of the list
// kernel above, which leave it latency-bound when the dense lists do not fit
// in L2 (cfg5: 10M dense rows, 680 MB of lists re-read per batch).
// With tb > 0 the ranks below tb are not listed; their presence mask goes to
// bits 24.. of the count word instead (table kernel below).
__global__ void hot_rec_kernel(const uint64_t* __restrict__ dl_ptr,
                               const uint32_t* __restrict__ dl_col, uint64_t n_dense, uint32_t K,
                               uint32_t tb, uint8_t* __restrict__ rec /* [D][32], zeroed */,
                               uint32_t* __restrict__ rcnt, const uint8_t* __restrict__ row_sp,
                               uint32_t sub = 0 /* stored rank = r - sub */) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_dense;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k0 = dl_ptr[i], k1 = dl_ptr[i + 1];
    uint32_t c = 0, top = 0;
    for (uint64_t k = k0; k < k1; ++k) {
      const uint32_t r = dl_col[k];
      if (r >= K) break;  // ranks ascend: the hot prefix ended
      if (r < tb) {
        top |= 1u << r;
        continue;
      }
      if (c < 32) rec[i * 32 + c] = (uint8_t)(r - sub);
      ++c;
    }
    rcnt[i] = c | (top << 24) | ((row_sp && row_sp[i]) ? 0x80000000u : 0u);
  }
}

// top-rank subset table of the hot kernels (see dense_hot_tab_kernel)
constexpr uint32_t kTabBits = 7;
constexpr uint32_t kTabRows = 1u << kTabBits;

#if D3G_COMPARISON_KERNELS  // record / guarded-step table kernels: measured comparisons
template <int kMode>
__global__ void __launch_bounds__(kHotThreads, 1)
dense_hot_rec_kernel(HotParams p, const uint64_t* __restrict__ dl_ptr,
                     const uint32_t* __restrict__ dl_col, const uint4* __restrict__ rec,
                     const uint32_t* __restrict__ rcnt, Decode dec, Emit em, Tally* tally,
                     unsigned long long* __restrict__ cnt_sp) {
  extern __shared__ __align__(128) uint4 Ts[];  // [K][32]
  __shared__ __align__(8) uint64_t bar;
  __shared__ unsigned int s_unit;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t n_batches = (p.groups + 31) / 32;
  const unsigned int n_units = n_batches * p.z_chunks;
  uint64_t cnt = 0, sum = 0, xr = 0, csp = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  int cur_batch = -1;
  const uint4 zero4 = make_uint4(0, 0, 0, 0);
  for (;;) {
    if (threadIdx.x == 0) s_unit = atomicAdd(p.work, 1u);
    __syncthreads();
    const unsigned int unit = s_unit;
    if (unit >= n_units) break;
    const uint32_t bi = unit / p.z_chunks, zc_i = unit % p.z_chunks;
    if ((int)bi != cur_batch) {
      if (threadIdx.x == 0) {
        const uint32_t bytes = p.K * 32u * 16u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar, bytes);
        tma_bulk_g2s(Ts, p.T + (uint64_t)bi * p.K * 32, bytes, &bar);
      }
      mbar_wait(&bar, phase);
      phase ^= 1;
      cur_batch = (int)bi;
    }
    const uint32_t g = bi * 32 + lane;  // this lane's group
    const uint64_t gp0 = (uint64_t)g * 128;
    const uint64_t z_lo = p.n_dense * zc_i / p.z_chunks, z_hi = p.n_dense * (zc_i + 1) / p.z_chunks;
    // software-pipelined 32-row steps: records of step s+1 load while s runs
    uint64_t cb = z_lo + (uint64_t)warp * 32;
    uint4 na = zero4, nb = zero4;
    uint32_t nc = 0;
    if (cb + lane < z_hi) {
      ld256(rec + 2 * (cb + lane), na, nb);
      nc = rcnt[cb + lane];
    }
    for (; cb < z_hi; cb += (uint64_t)nwarps * 32) {
      const uint4 ra = na, rb = nb;
      const uint32_t rc = nc;
      const uint64_t nx = cb + (uint64_t)nwarps * 32 + lane;
      na = zero4;
      nb = zero4;
      nc = 0;
      if (nx < z_hi) {
        ld256(rec + 2 * nx, na, nb);
        nc = rcnt[nx];
      }
      const uint32_t rows = (uint32_t)((z_hi - cb) < 32 ? (z_hi - cb) : 32);
      for (uint32_t j = 0; j < rows; ++j) {
        const uint32_t cw = __shfl_sync(0xffffffffu, rc, j);
        const uint32_t c = cw & 0xffffffu;
        uint4 acc = zero4;
        const uint32_t words[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (4u * q < c) {
            const uint32_t wv = __shfl_sync(0xffffffffu, words[q], j);
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              if (4u * q + b < c) {
                const uint32_t r = (wv >> (8 * b)) & 0xffu;
                const uint4 v = Ts[r * 32 + lane];
                acc.x |= v.x;
                acc.y |= v.y;
                acc.z |= v.z;
                acc.w |= v.w;
              }
            }
          }
        }
        const uint64_t i = cb + j;
        if (c > 32) {  // rare: hot prefix longer than one record
          const uint64_t k0 = dl_ptr[i] + 32, k1 = dl_ptr[i] + c;
          for (uint64_t base = k0; base < k1; base += 32) {
            const uint32_t mine = base + lane < k1 ? dl_col[base + lane] : 0u;
            const uint32_t n = (uint32_t)((k1 - base) < 32 ? (k1 - base) : 32);
            for (uint32_t t = 0; t < n; ++t) {
              const uint32_t r = __shfl_sync(0xffffffffu, mine, t);
              const uint4 v = Ts[r * 32 + lane];
              acc.x |= v.x;
              acc.y |= v.y;
              acc.z |= v.z;
              acc.w |= v.w;
            }
          }
        }
        const uint32_t hits = __popc(acc.x) + __popc(acc.y) + __popc(acc.z) + __popc(acc.w);
        cnt += hits;
        if (cw >> 31) csp += hits;
        if (kMode != kModeCount && hits) {
          const uint32_t zc = p.dl_z[i];
          const uint32_t ws[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
          for (int wi = 0; wi < 4; ++wi) {
            uint32_t bits = ws[wi];
            while (bits) {
              const int b = __ffs(bits) - 1;
              bits &= bits - 1;
              const uint32_t xc = p.xorder[gp0 + wi * 32 + b];
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
    }
    __syncthreads();  // Ts may be overwritten by the next unit's copy
  }
  flush_sp(cnt_sp, csp);
  tally_flush(tally, cnt, sum, xr);
}

// --- P1 with a subset table over the top ranks -----------------------------
// The top kTabBits ranks sit in most dense rows (cfg5: rank 0 in 95% of rows,
// rank 1 in 70%). Per batch, shared memory holds OR-combinations of their
// slices for every subset (2^kTabBits rows of 512 B, built in kTabBits-1
// rounds from the single-rank rows that TMA drops at the power-of-two
// entries), followed by the slices of ranks kTabBits..K-1. A dense row then
// costs ONE LDS.128 for its whole top-rank subset plus one per further hot
// rank. Records list only the ranks >= kTabBits; the subset mask rides in bits
// 24.. of the count word.

template <int kMode>
__global__ void __launch_bounds__(kHotThreads, 1)
dense_hot_tab_kernel(HotParams p, const uint64_t* __restrict__ dl_ptr,
                     const uint32_t* __restrict__ dl_col, const uint4* __restrict__ rec,
                     const uint32_t* __restrict__ rcnt, Decode dec, Emit em, Tally* tally,
                     unsigned long long* __restrict__ cnt_sp) {
  extern __shared__ __align__(128) uint4 Ts[];  // [kTabRows + K - kTabBits][32]
  __shared__ __align__(8) uint64_t bar;
  __shared__ unsigned int s_unit;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t n_batches = (p.groups + 31) / 32;
  const unsigned int n_units = n_batches * p.z_chunks;
  uint64_t cnt = 0, sum = 0, xr = 0, csp = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) Ts[threadIdx.x] = make_uint4(0, 0, 0, 0);  // entry 0: empty subset
  __syncthreads();
  uint32_t phase = 0;
  int cur_batch = -1;
  const uint4 zero4 = make_uint4(0, 0, 0, 0);
  // rank r >= kTabBits lives at row kTabRows + (r - kTabBits)
  const uint4* rows_hi = Ts + (kTabRows - kTabBits) * 32 + lane;
  for (;;) {
    if (threadIdx.x == 0) s_unit = atomicAdd(p.work, 1u);
    __syncthreads();
    const unsigned int unit = s_unit;
    if (unit >= n_units) break;
    const uint32_t bi = unit / p.z_chunks, zc_i = unit % p.z_chunks;
    if ((int)bi != cur_batch) {
      if (threadIdx.x == 0) {
        const uint4* src = p.T + (uint64_t)bi * p.K * 32;
        const uint32_t hi_bytes = (p.K - kTabBits) * 32u * 16u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar, hi_bytes + kTabBits * 512u);
        for (uint32_t b = 0; b < kTabBits; ++b)
          tma_bulk_g2s(Ts + (1u << b) * 32, src + b * 32, 512u, &bar);
        tma_bulk_g2s(Ts + kTabRows * 32, src + kTabBits * 32, hi_bytes, &bar);
      }
      mbar_wait(&bar, phase);
      phase ^= 1;
      cur_batch = (int)bi;
      // subset rows: round b fills (2^b, 2^(b+1)) from 2^b and the lower rows
      for (uint32_t b = 1; b < kTabBits; ++b) {
        const uint32_t lo = 1u << b, n = (lo - 1) * 32;
        for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
          const uint32_t e = lo + 1 + (t >> 5), l = t & 31;
          const uint4 a = Ts[lo * 32 + l], c = Ts[(e - lo) * 32 + l];
          Ts[e * 32 + l] = make_uint4(a.x | c.x, a.y | c.y, a.z | c.z, a.w | c.w);
        }
        __syncthreads();
      }
    }
    const uint32_t g = bi * 32 + lane;  // this lane's group
    const uint64_t gp0 = (uint64_t)g * 128;
    const uint64_t z_lo = p.n_dense * zc_i / p.z_chunks, z_hi = p.n_dense * (zc_i + 1) / p.z_chunks;
    uint64_t cb = z_lo + (uint64_t)warp * 32;
    uint4 na = zero4, nb = zero4;
    uint32_t nc = 0;
    if (cb + lane < z_hi) {
      ld256(rec + 2 * (cb + lane), na, nb);
      nc = rcnt[cb + lane];
    }
    for (; cb < z_hi; cb += (uint64_t)nwarps * 32) {
      const uint4 ra = na, rb = nb;
      const uint32_t rc = nc;
      const uint64_t nx = cb + (uint64_t)nwarps * 32 + lane;
      na = zero4;
      nb = zero4;
      nc = 0;
      if (nx < z_hi) {
        ld256(rec + 2 * nx, na, nb);
        nc = rcnt[nx];
      }
      const uint32_t rows = (uint32_t)((z_hi - cb) < 32 ? (z_hi - cb) : 32);
      for (uint32_t j = 0; j < rows; ++j) {
        const uint32_t cw = __shfl_sync(0xffffffffu, rc, j);
        const uint32_t c = cw & 0xffffffu, top = (cw >> 24) & 0x7fu;
        uint4 acc = Ts[top * 32 + lane];  // entry 0 is the empty subset
        const uint32_t words[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
        // row address = rows_hi + rank * 512 B: PRMT pulls the rank byte out,
        // one LEA-style add forms the address; full words OR two slices per
        // 3-input LOP3
        const char* hb = reinterpret_cast<const char*>(rows_hi);
#define D3G_ROW(wv, b) \
  (*reinterpret_cast<const uint4*>(hb + (__byte_perm((wv), 0u, 0x4440u + (b)) << 9)))
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (4u * q + 4 <= c) {
            const uint32_t wv = __shfl_sync(0xffffffffu, words[q], j);
            const uint4 v0 = D3G_ROW(wv, 0), v1 = D3G_ROW(wv, 1);
            const uint4 v2 = D3G_ROW(wv, 2), v3 = D3G_ROW(wv, 3);
            acc.x |= v0.x | v1.x;
            acc.y |= v0.y | v1.y;
            acc.z |= v0.z | v1.z;
            acc.w |= v0.w | v1.w;
            acc.x |= v2.x | v3.x;
            acc.y |= v2.y | v3.y;
            acc.z |= v2.z | v3.z;
            acc.w |= v2.w | v3.w;
          } else if (4u * q < c) {
            const uint32_t wv = __shfl_sync(0xffffffffu, words[q], j);
            const uint32_t left = c - 4u * q;  // 1..3
            const uint4 v0 = D3G_ROW(wv, 0);
            uint4 v1 = make_uint4(0, 0, 0, 0), v2 = make_uint4(0, 0, 0, 0);
            if (left > 1) v1 = D3G_ROW(wv, 1);
            if (left > 2) v2 = D3G_ROW(wv, 2);
            acc.x |= v0.x | v1.x;
            acc.y |= v0.y | v1.y;
            acc.z |= v0.z | v1.z;
            acc.w |= v0.w | v1.w;
            acc.x |= v2.x;
            acc.y |= v2.y;
            acc.z |= v2.z;
            acc.w |= v2.w;
          }
        }
#undef D3G_ROW
        const uint64_t i = cb + j;
        if (c > 32) {  // rare: more than 32 listed ranks; the tail is in the list
          const uint64_t k1 = dl_ptr[i + 1];
          uint64_t k = dl_ptr[i];
          // skip the top ranks and the 32 listed ones
          const uint32_t skip = __popc(top) + 32;
          const uint64_t kend = k + skip + (c - 32);
          k += skip;
          for (uint64_t base = k; base < kend && base < k1; base += 32) {
            const uint32_t mine = base + lane < kend ? dl_col[base + lane] : 0u;
            const uint32_t n = (uint32_t)((kend - base) < 32 ? (kend - base) : 32);
            for (uint32_t t = 0; t < n; ++t) {
              const uint32_t r = __shfl_sync(0xffffffffu, mine, t);
              const uint4 v = rows_hi[r * 32];
              acc.x |= v.x;
              acc.y |= v.y;
              acc.z |= v.z;
              acc.w |= v.w;
            }
          }
        }
        const uint32_t hits = __popc(acc.x) + __popc(acc.y) + __popc(acc.z) + __popc(acc.w);
        cnt += hits;
        if (cw >> 31) csp += hits;
        if (kMode != kModeCount && hits) {
          const uint32_t zc = p.dl_z[i];
          const uint32_t ws[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
          for (int wi = 0; wi < 4; ++wi) {
            uint32_t bits = ws[wi];
            while (bits) {
              const int b = __ffs(bits) - 1;
              bits &= bits - 1;
              const uint32_t xc = p.xorder[gp0 + wi * 32 + b];
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
    }
    __syncthreads();  // Ts may be overwritten by the next unit's copy
  }
  flush_sp(cnt_sp, csp);
  tally_flush(tally, cnt, sum, xr);
}

#endif  // D3G_COMPARISON_KERNELS

// Sort key of a record for the prefix-shared kernels: (subset mask, first
// listed rank + 1, second listed rank + 1; 7/9/9 bits), 0 = absent.
__global__ void trie_key_kernel(const uint8_t* __restrict__ rec, const uint32_t* __restrict__ rcnt,
                                uint64_t n, uint64_t* __restrict__ key, uint32_t* __restrict__ idx,
                                uint32_t off /* stored rank byte + off = rank - 6 */,
                                uint32_t class_bits = 0) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t cw = rcnt[i], c = cw & 0xffffffu;
    const uint32_t r1 = c >= 1 ? rec[i * 32] + off : 0u;
    const uint32_t r2 = c >= 2 ? rec[i * 32 + 1] + off : 0u;
    // pivot plan: rows class-major (class = the low class_bits bits of the
    // subset mask), so every class is one contiguous run
    const uint32_t top = (cw >> 24) & 0x7fu, cls = top & ((1u << class_bits) - 1u);
    key[i] = ((uint64_t)cls << 25) | ((uint64_t)top << 18) | (r1 << 9) | r2;
    idx[i] = (uint32_t)i;
  }
}

// Records in sorted order plus the shared-prefix length L with the previous
// sorted row (levels: subset, r1, r2; a level counts only if present).
__global__ void trie_gather_kernel(const uint4* __restrict__ rec, const uint32_t* __restrict__ rcnt,
                                   const uint64_t* __restrict__ key, const uint32_t* __restrict__ perm,
                                   uint64_t n, uint4* __restrict__ rec_s, uint32_t* __restrict__ rcnt_s) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t src = perm[i];
    uint4 a, b;
    ld256(rec + 2 * (uint64_t)src, a, b);
    st256(rec_s + 2 * i, a, b);
    const uint64_t k = key[i];
    uint32_t L = 0;
    if (i > 0) {
      const uint64_t kp = key[i - 1];
      if ((k >> 18) == (kp >> 18)) {
        L = 1;
        if ((k & 0x3fe00u) && ((k >> 9) == (kp >> 9))) {
          L = 2;
          if ((k & 0x1ffu) && k == kp) L = 3;
        }
      }
    }
    rcnt_s[i] = rcnt[src] | (L << 22);
  }
}
// --- P1 with prefix-shared records ----------------------------------------
// Dense rows sorted by (subset mask, first listed rank, second listed rank)
// share their leading slices with the row before them: cfg2's sorted rows
// repeat their first kTrieDepth sequence elements (subset, r1, r2) often
// enough to cut the slice reads per (row, batch) by a third (cfg5: by half).
// The warp keeps the partial ORs after each of those elements in registers
// (a0 = subset entry, a1 = a0 | T[r1], a2 = a1 | T[r2]) and a row whose
// shared-prefix length with its predecessor is L (bits 22-23 of the count
// word, set by trie_gather_kernel) restarts from a_{L-1}. The first row of
// each warp step starts from scratch (its predecessor ran on another warp).
// perm maps a sorted position back to the dense row (dl_z, dl_ptr).
constexpr uint32_t kTrieCntMask = 0x3fffffu;
#ifndef D3G_TRIE_THREADS
#define D3G_TRIE_THREADS 768
#endif
constexpr int kTrieThreads = D3G_TRIE_THREADS;

__device__ __forceinline__ void or4(uint4& a, const uint4& v) {
  a.x |= v.x;
  a.y |= v.y;
  a.z |= v.z;
  a.w |= v.w;
}

#if D3G_COMPARISON_KERNELS  // standalone prefix-shared kernel: measured comparison
template <int kMode>
__global__ void __launch_bounds__(kTrieThreads, 1)
dense_hot_trie_kernel(HotParams p, const uint64_t* __restrict__ dl_ptr,
                      const uint32_t* __restrict__ dl_col, const uint4* __restrict__ rec,
                      const uint32_t* __restrict__ rcnt, const uint32_t* __restrict__ perm,
                      Decode dec, Emit em, Tally* tally, unsigned long long* __restrict__ cnt_sp,
                      unsigned long long* __restrict__ lds_units) {
  extern __shared__ __align__(128) uint4 Ts[];  // [kTabRows + K - kTabBits][32]
  __shared__ __align__(8) uint64_t bar;
  __shared__ unsigned int s_unit;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t n_batches = (p.groups + 31) / 32;
  const unsigned int n_units = n_batches * p.z_chunks;
  uint64_t cnt = 0, sum = 0, xr = 0, csp = 0, lds = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) Ts[threadIdx.x] = make_uint4(0, 0, 0, 0);  // entry 0: empty subset
  __syncthreads();
  uint32_t phase = 0;
  int cur_batch = -1;
  const uint4 zero4 = make_uint4(0, 0, 0, 0);
  const uint4* rows_hi = Ts + (kTabRows - kTabBits) * 32 + lane;
  const char* hb = reinterpret_cast<const char*>(rows_hi);
#define D3G_ROW(wv, b) \
  (*reinterpret_cast<const uint4*>(hb + (__byte_perm((wv), 0u, 0x4440u + (b)) << 9)))
  for (;;) {
    if (threadIdx.x == 0) s_unit = atomicAdd(p.work, 1u);
    __syncthreads();
    const unsigned int unit = s_unit;
    if (unit >= n_units) break;
    const uint32_t bi = unit / p.z_chunks, zc_i = unit % p.z_chunks;
    if ((int)bi != cur_batch) {
      if (threadIdx.x == 0) {
        const uint4* src = p.T + (uint64_t)bi * p.K * 32;
        const uint32_t hi_bytes = (p.K - kTabBits) * 32u * 16u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar, hi_bytes + kTabBits * 512u);
        for (uint32_t b = 0; b < kTabBits; ++b)
          tma_bulk_g2s(Ts + (1u << b) * 32, src + b * 32, 512u, &bar);
        tma_bulk_g2s(Ts + kTabRows * 32, src + kTabBits * 32, hi_bytes, &bar);
      }
      mbar_wait(&bar, phase);
      phase ^= 1;
      cur_batch = (int)bi;
      for (uint32_t b = 1; b < kTabBits; ++b) {
        const uint32_t lo = 1u << b, n = (lo - 1) * 32;
        for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
          const uint32_t e = lo + 1 + (t >> 5), l = t & 31;
          const uint4 a = Ts[lo * 32 + l], c = Ts[(e - lo) * 32 + l];
          Ts[e * 32 + l] = make_uint4(a.x | c.x, a.y | c.y, a.z | c.z, a.w | c.w);
        }
        __syncthreads();
      }
    }
    const uint32_t g = bi * 32 + lane;
    const uint64_t gp0 = (uint64_t)g * 128;
    const uint64_t z_lo = p.n_dense * zc_i / p.z_chunks, z_hi = p.n_dense * (zc_i + 1) / p.z_chunks;
    uint64_t cb = z_lo + (uint64_t)warp * 32;
    uint4 na = zero4, nb = zero4;
    uint32_t nc = 0;
    if (cb + lane < z_hi) {
      ld256(rec + 2 * (cb + lane), na, nb);
      nc = rcnt[cb + lane];
    }
    uint4 a0 = zero4, a1 = zero4, a2 = zero4;
    for (; cb < z_hi; cb += (uint64_t)nwarps * 32) {
      const uint4 ra = na, rb = nb;
      const uint32_t rc = nc;
      const uint64_t nx = cb + (uint64_t)nwarps * 32 + lane;
      na = zero4;
      nb = zero4;
      nc = 0;
      if (nx < z_hi) {
        ld256(rec + 2 * nx, na, nb);
        nc = rcnt[nx];
      }
      const uint32_t rows = (uint32_t)((z_hi - cb) < 32 ? (z_hi - cb) : 32);
      for (uint32_t j = 0; j < rows; ++j) {
        const uint32_t cw = __shfl_sync(0xffffffffu, rc, j);
        const uint32_t c = cw & kTrieCntMask, top = (cw >> 24) & 0x7fu;
        const uint32_t L = j ? (cw >> 22) & 3u : 0u;
        const uint32_t w0 = __shfl_sync(0xffffffffu, ra.x, j);
        if (L == 0) a0 = Ts[top * 32 + lane];  // entry 0 is the empty subset
        if (L <= 1) {
          a1 = a0;
          if (c >= 1) or4(a1, D3G_ROW(w0, 0));
        }
        if (L <= 2) {
          a2 = a1;
          if (c >= 2) or4(a2, D3G_ROW(w0, 1));
        }
        lds += (L == 0 ? 1u : 0u) + c - (L > 1 ? L - 1 : 0u);
        uint4 acc = a2;
        if (c > 2) {
          const uint4 v2 = D3G_ROW(w0, 2);
          uint4 v3 = zero4;
          if (c > 3) v3 = D3G_ROW(w0, 3);
          acc.x |= v2.x | v3.x;
          acc.y |= v2.y | v3.y;
          acc.z |= v2.z | v3.z;
          acc.w |= v2.w | v3.w;
        }
        const uint32_t words[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
#pragma unroll
        for (int q = 1; q < 8; ++q) {
          if (4u * q + 4 <= c) {
            const uint32_t wv = __shfl_sync(0xffffffffu, words[q], j);
            const uint4 v0 = D3G_ROW(wv, 0), v1 = D3G_ROW(wv, 1);
            const uint4 v2 = D3G_ROW(wv, 2), v3 = D3G_ROW(wv, 3);
            acc.x |= v0.x | v1.x;
            acc.y |= v0.y | v1.y;
            acc.z |= v0.z | v1.z;
            acc.w |= v0.w | v1.w;
            acc.x |= v2.x | v3.x;
            acc.y |= v2.y | v3.y;
            acc.z |= v2.z | v3.z;
            acc.w |= v2.w | v3.w;
          } else if (4u * q < c) {
            const uint32_t wv = __shfl_sync(0xffffffffu, words[q], j);
            const uint32_t left = c - 4u * q;  // 1..3
            const uint4 v0 = D3G_ROW(wv, 0);
            uint4 v1 = zero4, v2 = zero4;
            if (left > 1) v1 = D3G_ROW(wv, 1);
            if (left > 2) v2 = D3G_ROW(wv, 2);
            acc.x |= v0.x | v1.x;
            acc.y |= v0.y | v1.y;
            acc.z |= v0.z | v1.z;
            acc.w |= v0.w | v1.w;
            acc.x |= v2.x;
            acc.y |= v2.y;
            acc.z |= v2.z;
            acc.w |= v2.w;
          }
        }
        const uint64_t i = cb + j;
        if (c > 32) {  // rare: more than 32 listed ranks; the tail is in the list
          const uint32_t row = perm[i];
          const uint64_t k1 = dl_ptr[row + 1];
          uint64_t k = dl_ptr[row];
          const uint32_t skip = __popc(top) + 32;
          const uint64_t kend = k + skip + (c - 32);
          k += skip;
          for (uint64_t base = k; base < kend && base < k1; base += 32) {
            const uint32_t mine = base + lane < kend ? dl_col[base + lane] : 0u;
            const uint32_t n = (uint32_t)((kend - base) < 32 ? (kend - base) : 32);
            for (uint32_t t = 0; t < n; ++t) {
              const uint32_t r = __shfl_sync(0xffffffffu, mine, t);
              or4(acc, rows_hi[r * 32]);
            }
          }
        }
        const uint32_t hits = __popc(acc.x) + __popc(acc.y) + __popc(acc.z) + __popc(acc.w);
        cnt += hits;
        if (cw >> 31) csp += hits;
        if (kMode != kModeCount && hits) {
          const uint32_t zc = p.dl_z[perm[i]];
          const uint32_t ws[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
          for (int wi = 0; wi < 4; ++wi) {
            uint32_t bits = ws[wi];
            while (bits) {
              const int b = __ffs(bits) - 1;
              bits &= bits - 1;
              const uint32_t xc = p.xorder[gp0 + wi * 32 + b];
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
    }
    __syncthreads();  // Ts may be overwritten by the next unit's copy
  }
#undef D3G_ROW
  flush_sp(cnt_sp, csp);
  if (lane == 0 && lds) atomicAdd(lds_units, (unsigned long long)lds);
  tally_flush(tally, cnt, sum, xr);
}

#endif  // D3G_COMPARISON_KERNELS

// --- P1 with a jump table over the listed ranks (default with the table) ---
// Same work as dense_hot_tab_kernel, fewer instructions per (row, batch): the
// tab kernel's eight guarded 4-rank steps cost ~30 branch/compare instructions
// per row even when skipped (ncu on cfg2: 140 instructions and 32 branches per
// (row, batch), issue-bound at 71% of peak). Here the listed-rank count picks
// one entry of a switch; the entry ORs the partial top quad and jumps into a
// straight-line run of full 4-rank quads. Listed ranks are stored as r - 7,
// so shared memory is [listed rows 0..K-8][subset table], and byte b reads
// row b directly.
// Slice reads per batch of the prefix-shared jump-table kernel, summed over
// rows: (L == 0) + c - max(L - 1, 0), with L forced to 0 on the first row of
// each warp step (positions z_lo + 32k of the row's z chunk).
__global__ void trie_lds_kernel(const uint32_t* __restrict__ rcnt, uint64_t n, uint32_t z_chunks,
                                uint32_t sub_read, unsigned long long* __restrict__ out_shared,
                                unsigned long long* __restrict__ out_unshared, uint64_t mult = 1,
                                uint64_t row0 = 0) {
  rcnt += row0;  // rows [row0, row0 + n), chunked as the kernel chunks them
  uint64_t acc = 0, acc_u = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t zc = i * z_chunks / n;
    while (zc + 1 < z_chunks && n * (zc + 1) / z_chunks <= i) ++zc;
    while (zc > 0 && n * zc / z_chunks > i) --zc;
    const uint64_t z_lo = n * zc / z_chunks;
    const uint32_t cw = rcnt[i], c = cw & kTrieCntMask;
    const uint32_t L = ((i - z_lo) % 32 == 0) ? 0u : (cw >> 22) & 3u;
    acc += (L == 0 ? sub_read : 0u) + c - (L > 1 ? L - 1 : 0u);
    acc_u += sub_read + c;  // the same row without prefix sharing
  }
  acc = warp_sum(acc);
  acc_u = warp_sum(acc_u);
  if (lane_id() == 0 && acc) atomicAdd(out_shared, (unsigned long long)(acc * mult));
  if (lane_id() == 0 && acc_u && out_unshared)
    atomicAdd(out_unshared, (unsigned long long)(acc_u * mult));
}

// The same accounting over several row runs in ONE launch (the pivot plan's
// class runs: up to 64, each with its own chunking and batch multiplicity;
// one launch per run cost more in launch gaps than in work).
struct TrieRuns {
  uint32_t n_runs;
  uint32_t zc[64];     // z chunks of run q
  uint64_t row0[64];   // its first row
  uint64_t start[65];  // exclusive prefix of the runs' row counts
  uint64_t mult[64];   // batches that test it
};
__global__ void trie_lds_runs_kernel(const uint32_t* __restrict__ rcnt, TrieRuns runs,
                                     uint32_t sub_read, unsigned long long* __restrict__ out_shared,
                                     unsigned long long* __restrict__ out_unshared) {
  uint64_t acc = 0, acc_u = 0;
  const uint64_t total = runs.start[runs.n_runs];
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t q = 0;
    while (q + 1 < runs.n_runs && runs.start[q + 1] <= g) ++q;
    const uint64_t n = runs.start[q + 1] - runs.start[q], i = g - runs.start[q];
    const uint64_t z_chunks = runs.zc[q];
    uint64_t zc = i * z_chunks / n;
    while (zc + 1 < z_chunks && n * (zc + 1) / z_chunks <= i) ++zc;
    while (zc > 0 && n * zc / z_chunks > i) --zc;
    const uint64_t z_lo = n * zc / z_chunks;
    const uint32_t cw = rcnt[runs.row0[q] + i], c = cw & kTrieCntMask;
    const uint32_t L = ((i - z_lo) % 32 == 0) ? 0u : (cw >> 22) & 3u;
    acc += ((L == 0 ? sub_read : 0u) + c - (L > 1 ? L - 1 : 0u)) * runs.mult[q];
    acc_u += (uint64_t)(sub_read + c) * runs.mult[q];
  }
  acc = warp_sum(acc);
  acc_u = warp_sum(acc_u);
  if (lane_id() == 0 && acc) atomicAdd(out_shared, (unsigned long long)acc);
  if (lane_id() == 0 && acc_u && out_unshared) atomicAdd(out_unshared, (unsigned long long)acc_u);
}

template <int kMode, bool kTrie, bool kTab = true>
__global__ void __launch_bounds__(kHotThreads, 1)
dense_hot_jt_kernel(HotParams p, const uint64_t* __restrict__ dl_ptr,
                    const uint32_t* __restrict__ dl_col, const uint4* __restrict__ rec,
                    const uint32_t* __restrict__ rcnt, const uint32_t* __restrict__ perm,
                    Decode dec, Emit em, Tally* tally, unsigned long long* __restrict__ cnt_sp) {
  extern __shared__ __align__(128) uint4 Ts[];  // [K - kTabBits listed][kTabRows subset][32]
  __shared__ __align__(8) uint64_t bar;
  __shared__ unsigned int s_unit;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t n_batches = (p.groups + 31) / 32;
  const unsigned int n_units = hot_units(p, n_batches);
  constexpr uint32_t kTB = kTab ? kTabBits : 0u;  // ranks in the subset table
  const uint32_t n_listed = p.K - kTB;
  uint4* const sub_tab = Ts + n_listed * 32;  // entry e at sub_tab[e * 32 + lane]
  uint64_t cnt = 0, sum = 0, xr = 0, csp = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) sub_tab[threadIdx.x] = make_uint4(0, 0, 0, 0);  // empty subset
  __syncthreads();
  uint32_t phase = 0;
  int cur_batch = -1;
  const uint4 zero4 = make_uint4(0, 0, 0, 0);
  const char* hb = reinterpret_cast<const char*>(Ts + lane);
  const uint4* sub_lane = sub_tab + lane;
#define D3G_ROW(wv, b) \
  (*reinterpret_cast<const uint4*>(hb + (__byte_perm((wv), 0u, 0x4440u + (b)) << 9)))
#define D3G_Q4(W)                                                   \
  {                                                                 \
    const uint32_t wv = __shfl_sync(0xffffffffu, (W), j);           \
    const uint4 v0 = D3G_ROW(wv, 0), v1 = D3G_ROW(wv, 1);           \
    const uint4 v2 = D3G_ROW(wv, 2), v3 = D3G_ROW(wv, 3);           \
    acc.x |= v0.x | v1.x;                                           \
    acc.y |= v0.y | v1.y;                                           \
    acc.z |= v0.z | v1.z;                                           \
    acc.w |= v0.w | v1.w;                                           \
    acc.x |= v2.x | v3.x;                                           \
    acc.y |= v2.y | v3.y;                                           \
    acc.z |= v2.z | v3.z;                                           \
    acc.w |= v2.w | v3.w;                                           \
  }
#define D3G_QP(W, n)                                                \
  {                                                                 \
    const uint32_t wv = __shfl_sync(0xffffffffu, (W), j);           \
    uint4 v0 = D3G_ROW(wv, 0), v1 = zero4, v2 = zero4;              \
    if ((n) > 1) v1 = D3G_ROW(wv, 1);                               \
    if ((n) > 2) v2 = D3G_ROW(wv, 2);                               \
    acc.x |= v0.x | v1.x;                                           \
    acc.y |= v0.y | v1.y;                                           \
    acc.z |= v0.z | v1.z;                                           \
    acc.w |= v0.w | v1.w;                                           \
    acc.x |= v2.x;                                                  \
    acc.y |= v2.y;                                                  \
    acc.z |= v2.z;                                                  \
    acc.w |= v2.w;                                                  \
  }
  for (;;) {
    if (threadIdx.x == 0) s_unit = atomicAdd(p.work, 1u);
    __syncthreads();
    const unsigned int unit = s_unit;
    if (unit >= n_units) break;
    uint32_t bi;
    uint64_t z_lo, z_hi;
    hot_unit(p, n_batches, unit, bi, z_lo, z_hi);
    if ((int)bi != cur_batch) {
      if (threadIdx.x == 0) {
        const uint4* src = p.T + (uint64_t)bi * p.K * 32;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar, (n_listed + kTB) * 512u);
        tma_bulk_g2s(Ts, src + kTB * 32, n_listed * 512u, &bar);
        if constexpr (kTab)
          for (uint32_t b = 0; b < kTB; ++b)
            tma_bulk_g2s(sub_tab + (1u << b) * 32, src + b * 32, 512u, &bar);
      }
      mbar_wait(&bar, phase);
      phase ^= 1;
      cur_batch = (int)bi;
      if constexpr (kTab) for (uint32_t b = 1; b < kTB; ++b) {
        const uint32_t lo = 1u << b, n = (lo - 1) * 32;
        for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
          const uint32_t e = lo + 1 + (t >> 5), l = t & 31;
          const uint4 a = sub_tab[lo * 32 + l], c = sub_tab[(e - lo) * 32 + l];
          sub_tab[e * 32 + l] = make_uint4(a.x | c.x, a.y | c.y, a.z | c.z, a.w | c.w);
        }
        __syncthreads();
      }
    }
    const uint32_t g = bi * 32 + lane;
    const uint64_t gp0 = (uint64_t)g * 128;
    uint64_t cb = z_lo + (uint64_t)warp * 32;
    uint4 na = zero4, nb = zero4;
    uint32_t nc = 0;
    uint4 a0 = zero4, a1 = zero4, a2 = zero4;  // kTrie: prefix ORs (subset, +r1, +r2)
    if (cb + lane < z_hi) {
      ld256(rec + 2 * (cb + lane), na, nb);
      nc = rcnt[cb + lane];
    }
    for (; cb < z_hi; cb += (uint64_t)nwarps * 32) {
      const uint4 ra = na, rb = nb;
      const uint32_t rc = nc;
      const uint64_t nx = cb + (uint64_t)nwarps * 32 + lane;
      na = zero4;
      nb = zero4;
      nc = 0;
      if (nx < z_hi) {
        ld256(rec + 2 * nx, na, nb);
        nc = rcnt[nx];
      }
      const uint32_t rows = (uint32_t)((z_hi - cb) < 32 ? (z_hi - cb) : 32);
      const uint32_t words[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
      for (uint32_t j = 0; j < rows; ++j) {
        const uint32_t cw = __shfl_sync(0xffffffffu, rc, j);
        const uint32_t c = cw & (kTrie ? kTrieCntMask : 0xffffffu), top = (cw >> 24) & 0x7fu;
        const uint32_t cc = c < 32 ? c : 32;
        uint4 acc;
        if constexpr (!kTrie) {
          acc = kTab ? sub_lane[top * 32] : zero4;
          switch (cc) {
            case 0: goto q_done;
            case 1: D3G_QP(words[0], 1); goto q_done;
            case 2: D3G_QP(words[0], 2); goto q_done;
            case 3: D3G_QP(words[0], 3); goto q_done;
            case 4: goto q_full0;
            case 5: D3G_QP(words[1], 1); goto q_full0;
            case 6: D3G_QP(words[1], 2); goto q_full0;
            case 7: D3G_QP(words[1], 3); goto q_full0;
            case 8: goto q_full1;
            case 9: D3G_QP(words[2], 1); goto q_full1;
            case 10: D3G_QP(words[2], 2); goto q_full1;
            case 11: D3G_QP(words[2], 3); goto q_full1;
            case 12: goto q_full2;
            case 13: D3G_QP(words[3], 1); goto q_full2;
            case 14: D3G_QP(words[3], 2); goto q_full2;
            case 15: D3G_QP(words[3], 3); goto q_full2;
            case 16: goto q_full3;
            case 17: D3G_QP(words[4], 1); goto q_full3;
            case 18: D3G_QP(words[4], 2); goto q_full3;
            case 19: D3G_QP(words[4], 3); goto q_full3;
            case 20: goto q_full4;
            case 21: D3G_QP(words[5], 1); goto q_full4;
            case 22: D3G_QP(words[5], 2); goto q_full4;
            case 23: D3G_QP(words[5], 3); goto q_full4;
            case 24: goto q_full5;
            case 25: D3G_QP(words[6], 1); goto q_full5;
            case 26: D3G_QP(words[6], 2); goto q_full5;
            case 27: D3G_QP(words[6], 3); goto q_full5;
            case 28: goto q_full6;
            case 29: D3G_QP(words[7], 1); goto q_full6;
            case 30: D3G_QP(words[7], 2); goto q_full6;
            case 31: D3G_QP(words[7], 3); goto q_full6;
            case 32: goto q_full7;
            default: break;
          }
          q_full7: D3G_Q4(words[7]);
          q_full6: D3G_Q4(words[6]);
          q_full5: D3G_Q4(words[5]);
          q_full4: D3G_Q4(words[4]);
          q_full3: D3G_Q4(words[3]);
          q_full2: D3G_Q4(words[2]);
          q_full1: D3G_Q4(words[1]);
          q_full0: D3G_Q4(words[0]);
          q_done:
          ;
        } else {
          // quads 1.. through the table, then quad 0 with the shared prefix
          acc = zero4;
          switch (cc) {
            case 0: case 1: case 2: case 3: case 4: goto t_done;
            case 5: D3G_QP(words[1], 1); goto t_done;
            case 6: D3G_QP(words[1], 2); goto t_done;
            case 7: D3G_QP(words[1], 3); goto t_done;
            case 8: goto t_full1;
            case 9: D3G_QP(words[2], 1); goto t_full1;
            case 10: D3G_QP(words[2], 2); goto t_full1;
            case 11: D3G_QP(words[2], 3); goto t_full1;
            case 12: goto t_full2;
            case 13: D3G_QP(words[3], 1); goto t_full2;
            case 14: D3G_QP(words[3], 2); goto t_full2;
            case 15: D3G_QP(words[3], 3); goto t_full2;
            case 16: goto t_full3;
            case 17: D3G_QP(words[4], 1); goto t_full3;
            case 18: D3G_QP(words[4], 2); goto t_full3;
            case 19: D3G_QP(words[4], 3); goto t_full3;
            case 20: goto t_full4;
            case 21: D3G_QP(words[5], 1); goto t_full4;
            case 22: D3G_QP(words[5], 2); goto t_full4;
            case 23: D3G_QP(words[5], 3); goto t_full4;
            case 24: goto t_full5;
            case 25: D3G_QP(words[6], 1); goto t_full5;
            case 26: D3G_QP(words[6], 2); goto t_full5;
            case 27: D3G_QP(words[6], 3); goto t_full5;
            case 28: goto t_full6;
            case 29: D3G_QP(words[7], 1); goto t_full6;
            case 30: D3G_QP(words[7], 2); goto t_full6;
            case 31: D3G_QP(words[7], 3); goto t_full6;
            case 32: goto t_full7;
            default: break;
          }
          t_full7: D3G_Q4(words[7]);
          t_full6: D3G_Q4(words[6]);
          t_full5: D3G_Q4(words[5]);
          t_full4: D3G_Q4(words[4]);
          t_full3: D3G_Q4(words[3]);
          t_full2: D3G_Q4(words[2]);
          t_full1: D3G_Q4(words[1]);
          t_done:
          ;
          const uint32_t w0 = __shfl_sync(0xffffffffu, words[0], j);
          const uint32_t L = j ? (cw >> 22) & 3u : 0u;
          if (kTab && L == 0) a0 = sub_lane[top * 32];
          if (L <= 1) {
            a1 = a0;
            if (c >= 1) or4(a1, D3G_ROW(w0, 0));
          }
          if (L <= 2) {
            a2 = a1;
            if (c >= 2) or4(a2, D3G_ROW(w0, 1));
          }
          or4(acc, a2);
          if (c > 2) {
            const uint4 v2 = D3G_ROW(w0, 2);
            uint4 v3 = zero4;
            if (c > 3) v3 = D3G_ROW(w0, 3);
            acc.x |= v2.x | v3.x;
            acc.y |= v2.y | v3.y;
            acc.z |= v2.z | v3.z;
            acc.w |= v2.w | v3.w;
          }
        }
        const uint64_t i = cb + j;
        if (c > 32) {  // rare: more than 32 listed ranks; the tail is in the list
          const uint64_t row = kTrie ? perm[i] : i;
          const uint32_t* tl = dl_col;
          uint64_t k;
          if (p.tail_rows) {  // z-split: the gathered tails (sorted row ids)
            uint32_t lo = 0, hi = p.n_tail;
            while (hi - lo > 1) {
              const uint32_t mid = (lo + hi) >> 1;
              if (p.tail_rows[mid] <= row) lo = mid; else hi = mid;
            }
            k = p.tail_ptr[lo];
            tl = p.tail_col;
          } else {
            k = dl_ptr[row] + __popc(top) + 32;
          }
          const uint64_t kend = k + (c - 32);
          for (uint64_t base = k; base < kend; base += 32) {
            const uint32_t mine = base + lane < kend ? tl[base + lane] : 0u;
            const uint32_t n = (uint32_t)((kend - base) < 32 ? (kend - base) : 32);
            for (uint32_t t = 0; t < n; ++t) {
              const uint32_t r = __shfl_sync(0xffffffffu, mine, t);
              const uint4 v = Ts[(r - kTB) * 32 + lane];
              acc.x |= v.x;
              acc.y |= v.y;
              acc.z |= v.z;
              acc.w |= v.w;
            }
          }
        }
        const uint32_t hits = __popc(acc.x) + __popc(acc.y) + __popc(acc.z) + __popc(acc.w);
        cnt += hits;
        if (cw >> 31) csp += hits;
        // emission: one warp-aggregated reservation per row step (all lanes
        // are converged here: they share the row, each holds one x group)
        unsigned long long slot = kMode == kModeEmit ? warp_reserve(em, hits) : 0ull;
        if (kMode != kModeCount && hits) {
          const uint32_t zc = p.dl_z[kTrie ? perm[i] : i];
          const uint32_t ws[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
          for (int wi = 0; wi < 4; ++wi) {
            uint32_t bits = ws[wi];
            while (bits) {
              const int b = __ffs(bits) - 1;
              bits &= bits - 1;
              const uint32_t xc = p.xorder[gp0 + wi * 32 + b];
              if (kMode == kModeChecksum) {
                const uint64_t h = dec.hash(xc, zc);
                sum += h;
                xr ^= h;
              } else {
                emit_at(em, slot++, xc, zc);
              }
            }
          }
        }
      }
    }
    __syncthreads();  // Ts may be overwritten by the next unit's copy
  }
#undef D3G_QP
#undef D3G_Q4
#undef D3G_ROW
  flush_sp(cnt_sp, csp);
  tally_flush(tally, cnt, sum, xr);
}


}  // namespace d3g
