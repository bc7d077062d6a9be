// Orchestration and C ABI of the B200 DIM^3 Join-Project operator.
//
// d3g_join_project follows join_project_extended's hybrid branch
// (P/src/engine.cpp:351-498) phase by phase, entirely device-resident:
//   swap (engine.cpp:361-366) -> f1 estimate (:368-377, on the host from the
//   same strided samples) -> natural-key resolution + mapping (:401,
//   map_with_fallback :40-50) -> CSR R-by-x / S-by-z (:411-415) -> degree
//   stats -> f2 partition (:425-427) -> SparseBMM (:472-476) -> DenseEC
//   (:478-481) -> count / optional (x, z) set (:483-491, decode :502-529).
// Phases are timed with CUDA events on the context stream.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <limits>
#include <string>
#include <type_traits>
#include <thread>
#include <unordered_map>
#include <vector>

#include "classical.cuh"
#include "counters.cuh"
#include "csr_bucket.cuh"
#include "exchange.cuh"
#include "datagen.cuh"
#include "denseec.cuh"
#include "denseec_hot.cuh"
#include "denseec_cold.cuh"
#include "zsplit.cuh"
#include "denseec_tc.cuh"
#include "io.cuh"
#include "aggregate.cuh"
#include "mapping.cuh"
#include "partition.cuh"
#include "sparsebmm.cuh"

struct d3g_ctx {
  d3g::Ctx c;
  d3g::Exchange ex;  // multi-GPU exchange (exchange.cuh); inactive by default
};

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return D3G_OK;
  } catch (const d3g::Error& e) {
    g_last_error = e.what();
    return e.status;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return D3G_INTERNAL_ERROR;
  }
}

using d3g::Ctx;
using d3g::DBuf;

__global__ void gather_stride_kernel(const uint64_t* __restrict__ src, uint64_t stride, uint64_t m,
                                     uint64_t* __restrict__ dst) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i * stride];
}

__global__ void live_flag_kernel(const uint64_t* __restrict__ row_ptr, uint64_t lo, uint64_t hi,
                                 uint32_t* __restrict__ flag) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi - lo;
       i += (uint64_t)gridDim.x * blockDim.x)
    flag[i] = row_ptr[lo + i + 1] > row_ptr[lo + i];
}

__global__ void add_offset_kernel(uint32_t* __restrict__ v, uint64_t n, uint32_t off) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    v[i] += off;
}

// u32 -> u64 columns, four values per thread (16-byte loads, 2 x 16-byte stores)
__global__ void widen_u32_kernel(const uint32_t* __restrict__ in, uint64_t n,
                                 uint64_t* __restrict__ out) {
  const uint64_t n4 = n / 4;
  const bool aligned = (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n + 3) / 4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (aligned && i < n4) {
      const uint4 v = reinterpret_cast<const uint4*>(in)[i];
      ulonglong2* o = reinterpret_cast<ulonglong2*>(out + 4 * i);
      o[0] = make_ulonglong2(v.x, v.y);
      o[1] = make_ulonglong2(v.z, v.w);
    } else {
      for (uint64_t k = 4 * i; k < 4 * i + 4 && k < n; ++k) out[k] = in[k];
    }
  }
}

__global__ void iota_kernel(uint32_t* __restrict__ v, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = (uint32_t)i;
}

struct Timer {
  Ctx& X;
  std::vector<cudaEvent_t> evs;
  explicit Timer(Ctx& x) : X(x) {}
  void mark() {
    cudaEvent_t e;
    D3G_CUDA(cudaEventCreate(&e));
    D3G_CUDA(cudaEventRecord(e, X.stream));
    evs.push_back(e);
  }
  double ms(size_t a, size_t b) {
    float t = 0;
    if (b < evs.size()) D3G_CUDA(cudaEventElapsedTime(&t, evs[a], evs[b]));
    return t;
  }
  ~Timer() {
    for (auto e : evs) cudaEventDestroy(e);
  }
};

struct DictBundle {
  d3g::DeviceDict x, y, z;
};

inline const uint64_t* rev_or_null(const d3g::DeviceDict& d) { return d.identity ? nullptr : d.rev.p; }

int dense_smem_bytes(Ctx& X) {
  int v = (int)X.smem_optin - 4096;  // leave room for static shared memory
  if (v > 220 * 1024) v = 220 * 1024;
  return v < 48 * 1024 ? 48 * 1024 : v;
}

// ---------------------------------------------------------------------------
// Kernel drivers shared by the pipeline and the kernel-level entry points.

struct SparseInputs {
  const uint64_t* r_ptr;
  const uint32_t* r_col;
  uint64_t n_rows;
  const uint64_t* sp_ptr;
  const uint32_t* sp_col;     // compact sparse index
  const uint32_t* sparse_ids; // compact index -> z code
  uint64_t n_sparse;
  uint64_t y_card;            // rows of sp_ptr
  // shard of x handled (x code range)
  uint64_t x_lo, x_hi;
};

struct KernelOut {
  uint64_t count = 0, sum = 0, xr = 0;
  uint64_t inner = 0;
  uint64_t cold_overflow = 0;  // x handed to the overflow kernel (diagnostics)
  uint64_t cold_overflow2 = 0;  // of those, x past the CTA hash tier
  uint64_t count_sp = 0;      // pairs of rows flagged in DenseInputs::row_sp
  double ms_hot = 0;          // CUDA-event time of the hot-pass launch
  uint64_t hot_lds_bytes = 0;  // its algorithmic shared-memory bytes
  uint64_t hot_lds_bytes_unshared = 0;  // without the prefix sharing
  uint64_t split_direct_pairs = 0;  // hits counted without a test (pivot plan)
  double ms_cold = 0;          // CUDA-event time of the cold-pass kernels
  uint64_t cold_bytes = 0;     // their algorithmic bytes (16 B records + 32 B tail checks)
  uint64_t cold_candidates = 0, cold_tail_checks = 0;
};

template <class F>
void with_mode(int mode, F&& f) {
  if (mode == d3g::kModeCount) f(std::integral_constant<int, d3g::kModeCount>{});
  else if (mode == d3g::kModeChecksum) f(std::integral_constant<int, d3g::kModeChecksum>{});
  else f(std::integral_constant<int, d3g::kModeEmit>{});
}

__global__ void sparse_bin_kernel(const uint64_t* __restrict__ cx, uint64_t n, uint64_t small_max,
                                  uint64_t mid_max, uint32_t* __restrict__ f1,
                                  uint32_t* __restrict__ f2, uint32_t* __restrict__ f3) {
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
       x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = cx[x];
    f1[x] = (c > 0 && c <= small_max) ? 1u : 0u;
    f2[x] = (c > small_max && c <= mid_max) ? 1u : 0u;
    f3[x] = c > mid_max ? 1u : 0u;
  }
}

// SparseBMM driver. Tiers per x by candidate count c_x (= its inner count):
//   c_x <= 32                     warp, register bitonic sort
//   n_sparse <= 8192, c_x > 32    warp, OR of bitset rows in registers
//   32 < c_x <= 1024              warp-private shared-memory hash set
//   c_x > 1024                    CTA bitmap over the sparse index (smem, or
//                                 a per-CTA global slice when too large)
void run_sparse(Ctx& X, const SparseInputs& in, d3g::Decode dec, int mode, d3g::Emit em,
                KernelOut& out, d3g::Filter flt = d3g::Filter{nullptr, nullptr, 0}) {
  using namespace d3g;
  if (in.n_rows == 0 || in.n_sparse == 0 || in.x_hi <= in.x_lo) return;
  const uint64_t nx = in.x_hi - in.x_lo;
  const uint32_t n_words = (uint32_t)((in.n_sparse + 31) / 32);
  const bool bitset_tier = flt.hz == nullptr && n_words <= 32u * kBitsetMaxWordsPerLane;
  const uint64_t mid_max = bitset_tier ? ~0ull : (uint64_t)(kHashCap / 2);
  DBuf<uint64_t> cx = X.alloc<uint64_t>(nx);
  DBuf<unsigned long long> tot = X.zeros<unsigned long long>(1);
  D3G_LAUNCH(X, sparse_cx_kernel, grid_for(nx, 256), 256, 0, in.r_ptr + in.x_lo, in.r_col, nx,
             in.sp_ptr, cx.p, tot.p);
  DBuf<uint32_t> fl[3];
  DBuf<uint64_t> pos[3];
  DBuf<uint32_t> lists[3];
  uint64_t cnt[3];
  for (int b = 0; b < 3; ++b) {
    fl[b] = X.alloc<uint32_t>(nx);
    pos[b] = X.alloc<uint64_t>(nx + 1);
  }
  // the register-sort tier takes c_x <= 128 unless the bitset tier applies
  // (cfg2's 3,406 sparse z), where c_x > 32 goes to the bitset rows
  const uint64_t small_max = bitset_tier ? 32ull : (uint64_t)kSmallMax;
  D3G_LAUNCH(X, sparse_bin_kernel, grid_for(nx, 256), 256, 0, cx.p, nx, small_max, mid_max,
             fl[0].p, fl[1].p, fl[2].p);
  for (int b = 0; b < 3; ++b) exclusive_scan<uint32_t>(X, fl[b].p, nx, pos[b].p);
  {  // the three tier sizes and the candidate total in one round trip
    DBuf<unsigned long long> sizes = X.alloc<unsigned long long>(4);
    for (int b = 0; b < 3; ++b)
      D3G_CUDA(cudaMemcpyAsync(sizes.p + b, pos[b].p + nx, 8, cudaMemcpyDeviceToDevice, X.stream));
    D3G_CUDA(cudaMemcpyAsync(sizes.p + 3, tot.p, 8, cudaMemcpyDeviceToDevice, X.stream));
    unsigned long long hs[4];
    X.to_host(hs, sizes.p, 4);
    for (int b = 0; b < 3; ++b) cnt[b] = hs[b];
    out.inner = hs[3];
  }
  for (int b = 0; b < 3; ++b) {
    lists[b] = X.alloc<uint32_t>(cnt[b]);
    if (cnt[b]) {
      D3G_LAUNCH(X, index_compact_kernel, grid_for(nx, 256), 256, 0, fl[b].p, pos[b].p, nx,
                 lists[b].p);
      if (in.x_lo)
        D3G_LAUNCH(X, add_offset_kernel, grid_for(cnt[b], 256), 256, 0, lists[b].p, cnt[b],
                   (uint32_t)in.x_lo);
    }
  }
  DBuf<Tally> t = X.zeros<Tally>(1);
  const uint64_t* rp = in.r_ptr;
  if (cnt[0]) {
    unsigned g = (unsigned)std::min<uint64_t>((cnt[0] + 7) / 8, (uint64_t)X.sm_count * 16);
    with_mode(mode, [&](auto M) {
      D3G_LAUNCH(X, sparse_small_kernel<M()>, g, 256, 0, lists[0].p, cnt[0], rp, in.r_col,
                 in.sp_ptr, in.sp_col, in.sparse_ids, dec, em, t.p, flt);
    });
  }
  if (cnt[1] && bitset_tier) {
    DBuf<uint32_t> rows = X.zeros<uint32_t>(in.y_card * n_words);
    D3G_LAUNCH(X, sparse_rowbits_build_kernel, grid_for(in.y_card * 32, 256), 256, 0, in.sp_ptr,
               in.sp_col, in.y_card, n_words, rows.p);
    unsigned g = (unsigned)std::min<uint64_t>((cnt[1] + 7) / 8, (uint64_t)X.sm_count * 16);
    with_mode(mode, [&](auto M) {
      int wpl = (int)((n_words + 31) / 32);
      if (wpl <= 1)
        D3G_LAUNCH(X, (sparse_bitset_kernel<M(), 1>), g, 256, 0, lists[1].p, cnt[1], rp, in.r_col,
                   in.sp_ptr, rows.p, n_words, in.sparse_ids, dec, em, t.p);
      else if (wpl <= 2)
        D3G_LAUNCH(X, (sparse_bitset_kernel<M(), 2>), g, 256, 0, lists[1].p, cnt[1], rp, in.r_col,
                   in.sp_ptr, rows.p, n_words, in.sparse_ids, dec, em, t.p);
      else if (wpl <= 4)
        D3G_LAUNCH(X, (sparse_bitset_kernel<M(), 4>), g, 256, 0, lists[1].p, cnt[1], rp, in.r_col,
                   in.sp_ptr, rows.p, n_words, in.sparse_ids, dec, em, t.p);
      else
        D3G_LAUNCH(X, (sparse_bitset_kernel<M(), 8>), g, 256, 0, lists[1].p, cnt[1], rp, in.r_col,
                   in.sp_ptr, rows.p, n_words, in.sparse_ids, dec, em, t.p);
    });
  } else if (cnt[1]) {
    unsigned g = (unsigned)std::min<uint64_t>((cnt[1] + kHashWarps - 1) / kHashWarps,
                                              (uint64_t)X.sm_count * 14);
    with_mode(mode, [&](auto M) {
      D3G_LAUNCH(X, sparse_hash_kernel<M()>, g, kHashWarps * 32, 0, lists[1].p, cnt[1], rp,
                 in.r_col, in.sp_ptr, in.sp_col, in.sparse_ids, dec, em, t.p, flt);
    });
  }
  if (cnt[2]) {
    size_t smem = (size_t)n_words * 4;
    bool use_smem = smem <= (size_t)dense_smem_bytes(X);
    unsigned g = (unsigned)std::min<uint64_t>(cnt[2], (uint64_t)X.sm_count *
                                                         (use_smem && smem <= 48 * 1024 ? 4 : 1));
    DBuf<uint32_t> gbm = X.alloc<uint32_t>(use_smem ? 1 : (uint64_t)g * n_words);
    with_mode(mode, [&](auto M) {
      if (use_smem) {
        auto kfn = sparse_large_kernel<M(), false>;
        if (smem > 48 * 1024)
          D3G_CUDA(raise_smem_attr(kfn, (int)smem));
        D3G_LAUNCH(X, kfn, g, 512, smem, lists[2].p, cnt[2], cx.p, in.x_lo, rp, in.r_col,
                   in.sp_ptr, in.sp_col, in.sparse_ids, n_words, gbm.p, dec, em, t.p, flt);
      } else {
        auto kfn = sparse_large_kernel<M(), true>;
        D3G_LAUNCH(X, kfn, g, 512, 0, lists[2].p, cnt[2], cx.p, in.x_lo, rp, in.r_col, in.sp_ptr,
                   in.sp_col, in.sparse_ids, n_words, gbm.p, dec, em, t.p, flt);
      }
    });
  }
  Tally h;
  X.to_host(&h, t.p, 1);
  out.count = h.count;
  out.sum = h.sum;
  out.xr = h.xr;
}

struct DenseInputs {
  const uint32_t* xorder;
  uint64_t n_live;
  const uint64_t* r_ptr;
  const uint32_t* r_col;
  const uint32_t* y_rank;
  uint64_t y_card;
  const uint64_t* dl_ptr;
  const uint32_t* dl_col;
  const uint32_t* dl_z;
  uint64_t n_dense;
  uint64_t max_group_nnz;  // sum of the 128 largest m_x (group 0)
  uint64_t pos_lo, pos_hi; // x positions (in xorder) handled
  const uint32_t* y_of_rank;
  const uint32_t* dR;      // R-side degree per y code
  uint64_t x_card;
  uint64_t x_lo, x_hi;     // x code range of the cold residual pass
  uint64_t dnnz = ~0ull;   // entries of the dense lists (~0: read dl_ptr[n_dense])
  const uint8_t* row_sp = nullptr;  // per row: a folded-in sparse z (count apart)
  // dS over all of S when the dense rows are every live z row: the dense rows
  // holding y are then simply dS(y) (no histogram over the dense lists)
  const uint32_t* dS_all = nullptr;
  // z-split S side of a sharded job (zsplit.cuh): dl_ptr / dl_col / dl_z /
  // row_sp / dnnz describe only this rank's dense rows, the global rows
  // [row_lo, row_lo + n_dense_local) of n_dense; the S-side products are built
  // for them and gathered over zx. Null zx: every row is local.
  d3g::Exchange* zx = nullptr;
  uint64_t row_lo = 0, n_dense_local = 0;
  std::vector<uint64_t> rows_per_rank;
  uint64_t x_card_job = 0, n_live_job = 0;
};

__global__ void gather_by_rank_kernel(const uint32_t* __restrict__ y_of_rank,
                                      const uint32_t* __restrict__ d, uint64_t n,
                                      uint32_t* __restrict__ out) {
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x)
    out[r] = d[y_of_rank[r]];
}

#if D3G_COMPARISON_KERNELS  // earlier DenseEC designs (D3G_DENSE=v1|v2), measured comparisons
// DenseEC driver: the z-tile-resident kernel (dense_ec_tile_kernel) when the
// group's cold entries and the longest dense list fit in shared memory, the
// list-streaming kernel (dense_ec_kernel) otherwise.
void run_dense_streaming(Ctx& X, const DenseInputs& in, d3g::Decode dec, int mode, d3g::Emit em,
                         KernelOut& out) {
  using namespace d3g;
  DenseParams p{};
  p.xorder = in.xorder + in.pos_lo;
  p.n_live = in.pos_hi - in.pos_lo;
  p.r_ptr = in.r_ptr;
  p.r_col = in.r_col;
  p.y_rank = in.y_rank;
  p.dl_ptr = in.dl_ptr;
  p.dl_col = in.dl_col;
  p.dl_z = in.dl_z;
  p.n_dense = in.n_dense;
  int smem = dense_smem_bytes(X);
  uint64_t y_hot = std::min<uint64_t>(in.y_card, (uint64_t)smem / 16);
  p.y_hot = (uint32_t)y_hot;
  uint64_t cap = 256;
  while (cap < 2 * in.max_group_nnz) cap <<= 1;
  p.cold_cap = (uint32_t)cap;
  uint64_t groups = (p.n_live + 127) / 128;
  unsigned g = (unsigned)std::min<uint64_t>(groups, (uint64_t)X.sm_count);
  DBuf<uint32_t> ck = X.alloc<uint32_t>((uint64_t)g * cap);
  DBuf<uint4> cv = X.alloc<uint4>((uint64_t)g * cap);
  p.cold_keys = ck.p;
  p.cold_vals = cv.p;
  p.z_lo = 0;
  p.z_hi = in.n_dense;
  DBuf<Tally> t = X.zeros<Tally>(1);
  size_t sm = (size_t)std::max<uint64_t>(y_hot, 1) * 16;
  with_mode(mode, [&](auto M) {
    auto kfn = dense_ec_kernel<M()>;
    D3G_CUDA(raise_smem_attr(kfn, (int)sm));
    D3G_LAUNCH(X, kfn, g, kDenseThreads, sm, p, dec, em, t.p);
  });
  Tally h;
  X.to_host(&h, t.p, 1);
  out.count = h.count;
  out.sum = h.sum;
  out.xr = h.xr;
}

void run_dense_tiles(Ctx& X, const DenseInputs& in, d3g::Decode dec, int mode, d3g::Emit em,
                     KernelOut& out) {
  using namespace d3g;
  if (in.n_dense == 0 || in.pos_hi <= in.pos_lo) return;
  const uint64_t n_live = in.pos_hi - in.pos_lo;
  const uint32_t groups = (uint32_t)((n_live + 127) / 128);
  const uint32_t* xorder = in.xorder + in.pos_lo;
  // cold-entry bound per group for each candidate hot size
  DBuf<unsigned int> mc = X.zeros<unsigned int>(kHotCandidates);
  D3G_LAUNCH(X, dense_cold_count_kernel, std::min<uint32_t>(groups, X.sm_count * 16), 128, 0,
             xorder, n_live, in.r_ptr, in.r_col, in.y_rank, mc.p);
  unsigned int maxcold[kHotCandidates];
  X.to_host(maxcold, mc.p, kHotCandidates);
  std::vector<uint64_t> hp(in.n_dense + 1);
  X.to_host(hp.data(), in.dl_ptr, in.n_dense + 1);
  uint64_t max_len = 0;
  for (uint64_t i = 0; i < in.n_dense; ++i) max_len = std::max(max_len, hp[i + 1] - hp[i]);
  const uint64_t budget = (uint64_t)dense_smem_bytes(X);
  static const uint32_t cand[kHotCandidates] = {16384, 8192, 4096, 2048, 1024, 512};
  int pick = -1;
  uint32_t hot = 0, ccap = 0, list_cap = 0, row_cap = 0;
  for (int j = 0; j < kHotCandidates; ++j) {
    uint32_t h = (uint32_t)std::min<uint64_t>(cand[j], in.y_card);
    uint64_t cold = h < in.y_card ? maxcold[j] : 0;
    uint64_t cc = 64;
    while (cc < 2 * cold) cc <<= 1;
    uint64_t fixed = (uint64_t)h * 16 + cc * 20;
    if (fixed + 64 * 1024 > budget) continue;
    uint64_t rest = budget - fixed;
    // 3/4 of the rest for list entries, 1/4 for row pointers
    uint64_t lc = (rest * 3 / 4) / 4, rc = (rest / 4) / 4 - 1;
    if (lc < max_len) continue;
    pick = j;
    hot = h;
    ccap = (uint32_t)cc;
    list_cap = (uint32_t)lc;
    row_cap = (uint32_t)rc;
    break;
  }
  if (pick < 0) {
    run_dense_streaming(X, in, dec, mode, em, out);
    return;
  }
  // greedy z tiles: <= row_cap rows and <= list_cap entries each
  std::vector<uint32_t> tb{0};
  {
    uint64_t r = 0;
    while (r < in.n_dense) {
      uint64_t e = r;
      while (e < in.n_dense && e - r < row_cap && hp[e + 1] - hp[r] <= list_cap) ++e;
      tb.push_back((uint32_t)e);
      r = e;
    }
  }
  const uint32_t n_tiles = (uint32_t)(tb.size() - 1);
  const uint32_t want_units = (uint32_t)X.sm_count * 6;
  uint32_t x_splits = std::max<uint32_t>(1, std::min<uint32_t>(groups, (want_units + n_tiles - 1) / n_tiles));
  DBuf<uint32_t> dtb = X.alloc<uint32_t>(tb.size());
  X.to_device(dtb.p, tb.data(), tb.size());
  DBuf<unsigned int> work = X.zeros<unsigned int>(1);
  DenseTileParams p{};
  p.xorder = xorder;
  p.n_live = n_live;
  p.r_ptr = in.r_ptr;
  p.r_col = in.r_col;
  p.y_rank = in.y_rank;
  p.dl_ptr = in.dl_ptr;
  p.dl_col = in.dl_col;
  p.dl_z = in.dl_z;
  p.tile_begin = dtb.p;
  p.n_tiles = n_tiles;
  p.x_splits = x_splits;
  p.groups = groups;
  p.hot = hot;
  p.cold_cap = ccap;
  p.list_cap = list_cap;
  p.row_cap = row_cap;
  p.work = work.p;
  size_t sm = (size_t)hot * 16 + (size_t)ccap * 20 + (size_t)(row_cap + 1) * 4 + (size_t)list_cap * 4;
  DBuf<Tally> t = X.zeros<Tally>(1);
  unsigned g = (unsigned)std::min<uint64_t>((uint64_t)n_tiles * x_splits, (uint64_t)X.sm_count);
  with_mode(mode, [&](auto M) {
    auto kfn = dense_ec_tile_kernel<M()>;
    D3G_CUDA(raise_smem_attr(kfn, (int)sm));
    D3G_LAUNCH(X, kfn, g, kD2Threads, sm, p, dec, em, t.p);
  });
  Tally h;
  X.to_host(&h, t.p, 1);
  out.count = h.count;
  out.sum = h.sum;
  out.xr = h.xr;
}
#endif  // D3G_COMPARISON_KERNELS

// ---------------------------------------------------------------------------
// DenseEC v3 driver (denseec_hot.cuh): hot bit-sliced pass + cold residual
// join. K is chosen from the measured rank histogram so that the cold join
// stays small relative to the pair tests.
constexpr int kKCand = 5;
__constant__ uint32_t kKValues[kKCand] = {64, 128, 256, 512, 1024};

__global__ void k_estimate_kernel(const uint32_t* __restrict__ y_of_rank,
                                  const uint32_t* __restrict__ dR,
                                  const uint32_t* __restrict__ cnt_rank, uint64_t y_card,
                                  unsigned long long* __restrict__ out /* [2][kKCand] */) {
  uint64_t cold[kKCand] = {}, hot[kKCand] = {};
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < y_card;
       r += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = cnt_rank[r];
    if (!c) continue;
    uint64_t prod = (uint64_t)dR[y_of_rank[r]] * c;
#pragma unroll
    for (int j = 0; j < kKCand; ++j) {
      if (r >= kKValues[j]) cold[j] += prod;
      else hot[j] += c;
    }
  }
#pragma unroll
  for (int j = 0; j < kKCand; ++j) {
    uint64_t a = d3g::warp_sum(cold[j]), b = d3g::warp_sum(hot[j]);
    if (d3g::lane_id() == 0) {
      if (a) atomicAdd(&out[j], (unsigned long long)a);
      if (b) atomicAdd(&out[kKCand + j], (unsigned long long)b);
    }
  }
}

__global__ void rec_sum_kernel(const uint32_t* __restrict__ rcnt, uint64_t n, uint32_t add,
                               unsigned long long* __restrict__ out) {
  uint64_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc += (rcnt[i] & 0x3fffffu) + add;
  acc = d3g::warp_sum(acc);
  if (d3g::lane_id() == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}

// out[0..6] = dense rows holding rank r (cnt_rank), out[7..10] = dR of ranks 0..3
__global__ void hot_small_stats_kernel(const uint32_t* __restrict__ cnt_rank,
                                       const uint32_t* __restrict__ y_of_rank,
                                       const uint32_t* __restrict__ dR, uint64_t y_card,
                                       unsigned long long* __restrict__ out) {
  const uint32_t t = threadIdx.x;
  if (t < 7)
    out[t] = t < y_card ? cnt_rank[t] : 0;
  else if (t < 11)
    out[t] = (t - 7) < y_card ? dR[y_of_rank[t - 7]] : 0;
}

// Class-aligned hot positions: the x at class-split position i (class q =
// cls[i], its rank within the class i - cstart[q]) goes to pstart[q] + that.
struct PadStarts {
  uint64_t cstart[d3g::kMaxClasses], pstart[d3g::kMaxClasses];
};
__global__ void pad_scatter_kernel(const uint32_t* __restrict__ cls, const uint32_t* __restrict__ xs,
                                   uint64_t n, PadStarts ps, uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q = cls[i];
    if (ps.pstart[q] == ~0ull) continue;  // a class handled elsewhere (shared batches)
    out[ps.pstart[q] + (i - ps.cstart[q])] = xs[i];
  }
}

// Test/experiment override of a kernel limit: env value clamped to [lo, hi].
static uint32_t env_u32(const char* name, uint32_t dflt, uint32_t lo, uint32_t hi) {
  const char* v = std::getenv(name);
  if (!v) return dflt;
  const unsigned long x = std::strtoul(v, nullptr, 10);
  return (uint32_t)std::min<unsigned long>(std::max<unsigned long>(x, lo), hi);
}

void run_dense_hot(Ctx& X, const DenseInputs& in, d3g::Decode dec, int mode, d3g::Emit em,
                   KernelOut& out) {
  using namespace d3g;
  // z-split: every rank takes part in the S-side gathers, live x or not
  const bool zs = in.zx != nullptr;
  if (in.n_dense == 0 || (!zs && in.pos_hi <= in.pos_lo)) return;
  const uint64_t n_live = in.pos_hi > in.pos_lo ? in.pos_hi - in.pos_lo : 0;
  const uint32_t* xorder = in.xorder + in.pos_lo;
  const uint32_t groups = (uint32_t)((n_live + 127) / 128);
  const uint64_t D = in.n_dense, Y = in.y_card;
  // this rank's dense rows (all of them unless z-split) and their global base
  const uint64_t DL = zs ? in.n_dense_local : D, row_lo = zs ? in.row_lo : 0;
  const uint64_t dnnz = in.dnnz != ~0ull ? in.dnnz : X.scalar(in.dl_ptr + DL);
  // choose K
  DBuf<uint32_t> cnt_rank;
  if (in.dS_all) {
    cnt_rank = X.alloc<uint32_t>(Y);
    D3G_LAUNCH(X, gather_by_rank_kernel, grid_for(Y, 256), 256, 0, in.y_of_rank, in.dS_all, Y,
               cnt_rank.p);
  } else {
    cnt_rank = X.zeros<uint32_t>(Y);
    if (dnnz)
      D3G_LAUNCH(X, value_hist_kernel, grid_for(dnnz, 512, X.sm_count * 2), 512, 0, in.dl_col,
                 dnnz, cnt_rank.p, (uint32_t)Y);
    if (zs) ex_allreduce(X, *in.zx, cnt_rank.p, Y, D3G_EX_SUM_U32);
  }
  // one read-back: K estimates, then the dense-row counts of ranks 0..6 (the
  // subset-table decision) and dR of ranks 0..3 (the cold variant bits)
  DBuf<unsigned long long> est = X.zeros<unsigned long long>(2 * kKCand + 11);
  D3G_LAUNCH(X, k_estimate_kernel, grid_for(Y, 256), 256, 0, in.y_of_rank, in.dR, cnt_rank.p, Y, est.p);
  D3G_LAUNCH(X, hot_small_stats_kernel, 1, 32, 0, cnt_rank.p, in.y_of_rank, in.dR, Y,
             est.p + 2 * kKCand);
  // the pivot-plan class counts (count-only) ride on the same read-back
  const bool piv_pre = mode == kModeCount && std::getenv("D3G_HOT") == nullptr &&
                       std::getenv("D3G_NO_SPLIT") == nullptr && Y >= 1;
  // (z-split: from a rank's share of the job's live x, so every rank picks
  // the same pivots)
  const uint32_t n_batches_pre =
      zs ? (uint32_t)((in.n_live_job / (uint64_t)in.zx->nranks + 4095) / 4096) : (groups + 31) / 32;
  const double units_pre = (double)n_batches_pre * (double)D;
  // measured: cfg5 (2.4e10 units) 2/3/4 pivots 153/135/132 ms; cfg2 (1e7)
  // 2.30/2.31/2.41 ms
  // (cfg5, 2.4e10 units: 4 / 5 / 6 pivots 93.7 / 93.3 / 93.3 ms; cfg2, 1e7: 2.30 / 2.42 / 2.68)
  // (a rank of the 8-way sharded cfg5, 3e9: 4 pivots; 5 gave it 32 partial
  // class batches)
  const uint32_t piv_dflt = units_pre > 1e10 ? 5u : units_pre > 2e9 ? 4u : units_pre > 1e9 ? 3u : 2u;
  const uint32_t n_piv =
      (uint32_t)std::min<uint64_t>(env_u32("D3G_PIVOTS", piv_dflt, 1, kMaxPivots), std::max<uint64_t>(Y, 1));
  DBuf<uint32_t> cls;
  DBuf<unsigned long long> pcnt;
  // pivot-class counts: x [kMaxClasses] | rows [kMaxClasses] | folded sparse rows [kMaxClasses]
  constexpr uint32_t kMC = kMaxClasses;
  unsigned long long c[3 * kMC] = {0};
  // With the cold kernels (K = 256, known before the K estimates return) the
  // x hot masks come first, built without atomics; the pivot classes are
  // read off them and the slice tables are transposed from them by ballots.
  const uint64_t budget_pre = (uint64_t)dense_smem_bytes(X) - 1024;
  const char* cold_env_pre = std::getenv("D3G_COLD");
  const bool hx_first = std::min<uint64_t>(1024, budget_pre / 512 / 64 * 64) >= 256 &&
                        !(cold_env_pre && std::string(cold_env_pre) == "tiers") &&
                        std::getenv("D3G_K") == nullptr && std::getenv("D3G_HOT") == nullptr;
  DBuf<unsigned long long> hx;
  if (hx_first) {
    hx = X.zeros<unsigned long long>(in.x_card * 4);
    // every x code of R when the call covers them all (rows read in order),
    // else the call's live x
    const bool all_x = in.pos_lo == 0 && in.pos_hi == in.n_live && in.x_lo == 0 &&
                       in.x_hi >= in.x_card;
    if (all_x && in.x_card)
      D3G_LAUNCH(X, hx_build_rows_kernel, grid_for(in.x_card, 256, X.sm_count * 32), 256, 0,
                 in.x_card, in.r_ptr, in.r_col, in.y_rank, 256u, reinterpret_cast<uint4*>(hx.p));
    else if (n_live)
      D3G_LAUNCH(X, hx_build_kernel, grid_for(n_live * 8, 256), 256, 0, xorder, n_live, in.r_ptr,
                 in.r_col, in.y_rank, 256u, reinterpret_cast<uint4*>(hx.p));
  }
  if (piv_pre) {
    cls = X.alloc<uint32_t>(n_live);
    pcnt = X.zeros<unsigned long long>(3 * kMC);
    if (n_live && hx_first)
      D3G_LAUNCH(X, pivot_class_hx_kernel, grid_for(n_live, 256), 256, 0, xorder, n_live, hx.p, 4u,
                 n_piv, cls.p, pcnt.p);
    else if (n_live)
      D3G_LAUNCH(X, pivot_class_x_kernel, grid_for(n_live, 256), 256, 0, xorder, n_live, in.r_ptr,
                 in.r_col, in.y_of_rank, n_piv, cls.p, pcnt.p);
    if (DL)
      D3G_LAUNCH(X, pivot_class_rows_kernel, grid_for(DL, 256), 256, 0, in.dl_ptr, in.dl_col, DL,
                 n_piv, in.row_sp, pcnt.p + kMC);
  }
  unsigned long long e[2 * kKCand + 11];
  X.defer(e, est.p, (2 * kKCand + 11) * 8);
  if (piv_pre) X.defer(c, pcnt.p, 3 * kMC * 8);
  X.sync();
  // z-split: the dense-row class counts of the job (the x classes stay local)
  if (zs && piv_pre)
    ex_allreduce_host(X, *in.zx, reinterpret_cast<uint64_t*>(c + kMC), 2 * kMC, D3G_EX_SUM_U64);
  const unsigned long long* top_rank_rows = e + 2 * kKCand;   // [7]
  const unsigned long long* top_rank_dr = e + 2 * kKCand + 7;  // [4]
  static const uint32_t kv[kKCand] = {64, 128, 256, 512, 1024};
  // K is bounded by the shared-memory slice of a 32-group batch (K * 512 B)
  const uint64_t budget = (uint64_t)dense_smem_bytes(X) - 1024;
  const uint32_t k_cap = (uint32_t)std::min<uint64_t>(1024, budget / 512 / 64 * 64);
  const double units = (double)D * (double)((groups + 31) / 32);
  int best = 0;
  double best_cost = 1e300;
  for (int j = 0; j < kKCand; ++j) {
    if (kv[j] > k_cap) break;
    double hot_per_z = (double)e[kKCand + j] / (double)D;
    double cost = units * hot_per_z * 8.0 + 12.0 * (double)e[j] * ((double)n_live / std::max<uint64_t>(in.x_card, 1));
    if (cost < best_cost) { best_cost = cost; best = j; }
  }
  uint32_t K = kv[best];
  if (K * 2 <= k_cap && K == 256 && k_cap >= 384) K = 384;  // use the slack of the batch slice
  // the warp-bitmap cold kernel carries 256-bit hot signatures: K = 256
  // (the dense rows are split into at most 16 bitmap partitions, see P2)
  // CTAs of the bitmap cold kernel per SM (its per-warp bitmaps share the
  // SM's shared memory): more, smaller partitions raise occupancy for the
  // latency-bound candidate stream
  const char* cc_env = std::getenv("D3G_COLD_CTAS");
  // (16-byte records, window mapping: cfg2 3 CTAs 2.12 ms, 4: 2.27, 2: 2.20)
  uint32_t cold_ctas = 3;
  if (cc_env) cold_ctas = std::max(1, std::atoi(cc_env));
  const uint64_t cold_rows_cap =
      std::max<uint64_t>(32, (budget / cold_ctas / kColdWarps - (kDQ + kSegWords) * 4) * 8 / 32 * 32);
  const char* cpath_env = std::getenv("D3G_COLD_PATH");  // experiments: hash | bitmap
  const bool cold_bitmap = k_cap >= 256 && (D + cold_rows_cap - 1) / cold_rows_cap <= 16 &&
                           !(cpath_env && std::string(cpath_env) == "hash");
  // larger dense blocks: the same candidate stream, survivors in a per-warp
  // hash set (dense_cold_hash_kernel); D3G_COLD=tiers keeps the SparseBMM tiers
  const char* cold_env = std::getenv("D3G_COLD");
  const bool cold_hash = !cold_bitmap && k_cap >= 256 &&
                         !(cold_env && std::string(cold_env) == "tiers");
  const bool cold_kernel_ok = cold_bitmap || cold_hash;
  if (in.row_sp && !cold_kernel_ok)
    throw d3g::Error(D3G_INTERNAL_ERROR, "folded sparse rows need the cold kernels");
  if (cold_kernel_ok) K = 256;
  if (const char* kenv = std::getenv("D3G_K")) {  // experiments: force the hot width
    const uint32_t k = (uint32_t)std::strtoul(kenv, nullptr, 10);
    if (k >= 64 && k % 64 == 0 && k <= (cold_kernel_ok ? 256u : k_cap)) K = k;
  }
  // the cold kernels read 256-bit hot signatures: keep that layout for K < 256
  const uint32_t kw = cold_kernel_ok ? 4u : (K + 63) / 64;
  uint32_t n_batches = (groups + 31) / 32;  // of the hot pass (class-aligned: padded)
  // Rank-0 split (count-only; the table kernel with prefix-shared rows): an x
  // holding the top rank y_of_rank[0] hits every dense row that holds it.
  // Live x are split stably into B (without it) then A (with it); batches made
  // only of A x test only the rows without the top rank (sorted first), and
  // their other pairs are counted as hits without a test. cfg5: 95% of x and
  // rows hold rank 0, so ~10x fewer (batch, row) tests; cfg2: ~4x.
  const char* hot_sel_env = std::getenv("D3G_HOT");
  const std::string hot_sel = hot_sel_env ? hot_sel_env : "";
  double top_rows = 0;
  for (uint32_t r = 0; r < kTabBits; ++r) top_rows += (double)top_rank_rows[r] / (double)D;
  const bool tab_planned = K <= 256 && K > kTabBits && hot_sel.empty() &&
                           (size_t)(kTabRows + K - kTabBits) * 32 * 16 <= (size_t)dense_smem_bytes(X) &&
                           top_rows >= 1.5;
  // Pivot plan (count-only): x and dense rows are classed by which of the
  // n_piv top ranks (pivots) they hold (bit q = rank q). A pair sharing a
  // pivot is a hit without a test. x are split stably by class into batches;
  // a batch whose x share the pivot set k (the AND of their classes) tests
  // only the rows of the classes with no pivot in k. The sorted rows are
  // class-major, so those are a few contiguous class runs (no copies); every
  // other pair of the batch is counted as a hit.
  const uint32_t n_kinds = 1u << n_piv;
  // z-split: pool the ranks' class-0 x (tested against every row) into shared
  // batches, each rank testing them against a slice of the rows
  const bool share0_try = zs && piv_pre && std::getenv("D3G_NO_SHARE0") == nullptr;
  bool share0_local = false;  // this rank's class-0 x left its own batches
  uint64_t n0_local = 0;
  // the hot pass's x positions (class-aligned plan: padded with empty slots)
  const uint32_t* hot_xorder = xorder;
  uint64_t hot_n = n_live;
  DBuf<uint32_t> xpad;
  uint64_t plan_direct = 0, plan_direct_sp = 0;  // untested hits (all / folded sparse rows)
  uint64_t run_lo[kMC + 1] = {0};  // class c's rows [run_lo[c], run_lo[c + 1])
  uint32_t run_zc[kMC] = {0};      // units per batch over class c's run
  uint64_t run_mult[kMC] = {0};    // batches that test class c's run
  std::vector<uint32_t> unit_off_h;
  std::vector<uint8_t> batch_kind_h;
  DBuf<uint32_t> xsplit;
  const bool try_plan = piv_pre && tab_planned && top_rank_rows[0] > 0;
  if (try_plan) {
    const unsigned long long* nx = c;       // x per class
    const unsigned long long* nr = c + kMC;       // dense rows per class
    const unsigned long long* nsp = c + 2 * kMC;  // folded sparse rows per class
    uint64_t kind_rows[kMC] = {}, sp_rows[kMC] = {}, sp_all = 0;
    for (uint32_t q = 0; q < n_kinds; ++q) sp_all += nsp[q];
    for (uint32_t k = 0; k < n_kinds; ++k)
      for (uint32_t q = 0; q < n_kinds; ++q)
        if ((q & k) == 0) {
          kind_rows[k] += nr[q];
          sp_rows[k] += nsp[q];
        }
    // class q occupies x positions [cstart[q], cstart[q + 1]) after the split
    uint64_t cstart[kMC + 1] = {0};
    for (uint32_t q = 0; q < kMC; ++q) cstart[q + 1] = cstart[q] + (q < n_kinds ? nx[q] : 0);
    batch_kind_h.assign(n_batches, 0);
    double tested = 0;
    uint64_t direct = 0, direct_sp = 0;
    for (uint32_t b = 0; b < n_batches; ++b) {
      const uint64_t p0 = (uint64_t)b * 4096, p1 = std::min<uint64_t>(p0 + 4096, n_live);
      uint32_t k = n_kinds - 1;
      for (uint32_t q = 0; q < n_kinds; ++q)
        if (cstart[q + 1] > p0 && cstart[q] < p1) k &= q;  // classes present
      batch_kind_h[b] = (uint8_t)k;
      tested += (double)kind_rows[k];
      direct += (p1 - p0) * (D - kind_rows[k]);
      direct_sp += (p1 - p0) * (sp_all - sp_rows[k]);
    }
    // Class-aligned batches: every class padded to whole batches, so no batch
    // mixes classes. A mixed batch tests the rows of the AND of its classes'
    // pivot sets: a batch straddling classes 1 and 2 (pivot 0 only / pivot 1
    // only) tests EVERY row, and an x shard has such boundaries of its own.
    // (z-split: class 0 -- x holding no pivot, so every row is tested -- is
    // pooled across the ranks into shared batches, see below)
    uint64_t pstart[kMC + 1] = {0};
    double tested_pad = 0;
    for (uint32_t q = 0; q < n_kinds; ++q) {
      const uint64_t nb = (share0_try && q == 0) ? 0 : (nx[q] + 4095) / 4096;
      pstart[q + 1] = pstart[q] + nb * 4096;
      tested_pad += (double)nb * (double)kind_rows[q];
    }
    const bool pad = (share0_try || tested_pad < tested) && std::getenv("D3G_NO_PAD") == nullptr;
    uint32_t n_batches_plan = n_batches;
    if (pad) {
      n_batches_plan = (uint32_t)(pstart[n_kinds] / 4096);
      batch_kind_h.assign(n_batches_plan, 0);
      direct = direct_sp = 0;
      for (uint32_t q = 0; q < n_kinds; ++q) {
        for (uint64_t b = pstart[q] / 4096; b < pstart[q + 1] / 4096; ++b) batch_kind_h[b] = (uint8_t)q;
        direct += nx[q] * (D - kind_rows[q]);
        direct_sp += nx[q] * (sp_all - sp_rows[q]);
      }
      tested = tested_pad;
    }
    if (tested < 0.8 * (double)n_batches_plan * (double)D) {
      xsplit = X.alloc<uint32_t>(n_live);
      DBuf<uint32_t> cls_s = X.alloc<uint32_t>(n_live);
      radix_pass_u32(X, cls.p, xorder, n_live, 0, cls_s.p, xsplit.p);  // stable by class
      xorder = xsplit.p;
      if (pad) {  // the hot pass's x positions: each class from a batch start
        n_batches = n_batches_plan;
        hot_n = pstart[n_kinds];
        xpad = X.alloc<uint32_t>(hot_n);
        D3G_CUDA(cudaMemsetAsync(xpad.p, 0xff, hot_n * 4, X.stream));  // empty positions
        PadStarts ps{};
        for (uint32_t q = 0; q < kMC; ++q) {
          ps.cstart[q] = cstart[q];
          ps.pstart[q] = pstart[q];
        }
        if (share0_try) {  // class 0 goes to the shared batches
          ps.pstart[0] = ~0ull;
          share0_local = true;
          n0_local = nx[0];
        }
        if (n_live)
          D3G_LAUNCH(X, pad_scatter_kernel, grid_for(n_live, 256), 256, 0, cls_s.p, xsplit.p,
                     n_live, ps, xpad.p);
        hot_xorder = xpad.p;
      }
      plan_direct = direct;
      plan_direct_sp = direct_sp;
      for (uint32_t q = 0; q < n_kinds; ++q) run_lo[q + 1] = run_lo[q] + nr[q];
      // units of about equal row counts (~8 per SM over the whole pass), so a
      // few all-row batches do not leave one CTA with millions of rows
      // units per SM grow with the batch count: a unit that switches batch
      // reloads the batch's slice table (193 KB), so few batches want few,
      // large units (cfg2, 49 batches: 3/SM, hot 0.33 -> 0.27 ms) and many
      // batches want finer balance (cfg5, 2442 batches: 8 / 12 / 16 / 24 / 32
      // per SM -> hot 20.49 / 20.07 / 20.09 / 19.81 / 19.85 ms)
      const uint32_t u_dflt = (uint32_t)std::min<double>(
          24.0, std::max<double>(2.0, std::round(8.0 * n_batches / X.sm_count)));
      const double per_unit = std::max(
          256.0, tested / ((double)X.sm_count * env_u32("D3G_UNITS_PER_SM", u_dflt, 1, 64)));
      for (uint32_t q = 0; q < n_kinds; ++q) {
        const uint64_t rows = nr[q];
        run_zc[q] = rows ? std::max<uint32_t>(1, (uint32_t)std::min<double>(
                               std::ceil((double)rows / per_unit), (double)((rows + 255) / 256)))
                         : 0u;
      }
      unit_off_h.assign(n_batches + 1, 0);
      for (uint32_t b = 0; b < n_batches; ++b) {
        uint32_t u = 0;
        for (uint32_t q = 0; q < n_kinds; ++q)
          if ((q & batch_kind_h[b]) == 0) {
            u += run_zc[q];
            ++run_mult[q];
          }
        unit_off_h[b + 1] = unit_off_h[b] + u;
      }
    } else {
      batch_kind_h.clear();
    }
  }
  // hot structures
  if (hx_first && (K != 256 || kw != 4))
    throw d3g::Error(D3G_INTERNAL_ERROR, "hot masks built for K = 256");
  // (from the masks every word of T is written: no memset)
  DBuf<uint4> T = hx_first ? X.alloc<uint4>((uint64_t)n_batches * K * 32)
                           : X.zeros<uint4>((uint64_t)n_batches * K * 32);
  if (!hx_first) hx = X.zeros<unsigned long long>(in.x_card * kw);
  DBuf<unsigned long long> hz = X.zeros<unsigned long long>(D * kw);
  // z-split: this rank's rows' masks, gathered into hz (every rank's rows)
  DBuf<unsigned long long> hz_loc;
  unsigned long long* hzl = hz.p;
  if (zs) {
    hz_loc = X.zeros<unsigned long long>(DL * kw);
    hzl = hz_loc.p;
  }
  if (!xpad.p) hot_xorder = xorder;  // the class-split order when planned
  if (hx_first && n_batches)
    D3G_LAUNCH(X, hot_T_from_hx_kernel, grid_for((uint64_t)n_batches * 32 * 32, 256), 256, 0,
               hot_xorder, hot_n, (uint64_t)n_batches * 4096, reinterpret_cast<const uint4*>(hx.p),
               K, T.p);
  else if (n_live)
    D3G_LAUNCH(X, hot_build_x_kernel, grid_for(hot_n * 8, 256), 256, 0, hot_xorder, hot_n,
               in.r_ptr, in.r_col, in.y_rank, K, kw, reinterpret_cast<uint32_t*>(T.p), hx.p);
  if (DL)
    D3G_LAUNCH(X, hot_build_z_kernel, grid_for(DL * 8, 256), 256, 0, in.dl_ptr, in.dl_col, DL, K,
               kw, hzl);
  // z-split shared class-0 batches: every rank ORs its class-0 x into the
  // pooled slice tables (disjoint bits: a sum all-reduce is the OR), then
  // tests them against rows [D r / N, D (r + 1) / N) of the sorted records
  DBuf<uint4> T0;
  uint64_t n0_job = 0, sh_lo = 0, sh_hi = 0;
  uint32_t nb0 = 0;
  if (share0_try && try_plan) {
    const int N = in.zx->nranks, rk = in.zx->rank;
    uint64_t mine = share0_local ? n0_local : 0;
    std::vector<uint64_t> all(N);
    ex_allgather(X, *in.zx, &mine, all.data(), 8);
    uint64_t off = 0;
    for (int q = 0; q < N; ++q) {
      if (q < rk) off += all[q];
      n0_job += all[q];
    }
    if (n0_job) {
      nb0 = (uint32_t)((n0_job + 4095) / 4096);
      T0 = X.zeros<uint4>((uint64_t)nb0 * K * 32);
      if (mine)  // class 0 leads the class-split order
        D3G_LAUNCH(X, hot_build_x_kernel, grid_for(mine * 8, 256), 256, 0, xorder, mine, in.r_ptr,
                   in.r_col, in.y_rank, K, kw, reinterpret_cast<uint32_t*>(T0.p), hx.p, off);
      ex_allreduce(X, *in.zx, T0.p, (uint64_t)nb0 * K * 32 * 4, D3G_EX_SUM_U32);
      sh_lo = D * (uint64_t)rk / (uint64_t)N;
      sh_hi = D * (uint64_t)(rk + 1) / (uint64_t)N;
    }
  }
  if (zs) ex_allgatherv_dev(X, *in.zx, hzl, in.rows_per_rank, kw * 8, hz.p);
  // z-split: the job's per-row z codes and folded-sparse flags
  DBuf<uint32_t> dlz_g;
  DBuf<uint8_t> rsp_g;
  const uint32_t* dlz = in.dl_z;
  const uint8_t* rsp = in.row_sp;
  if (zs) {
    dlz_g = X.alloc<uint32_t>(D);
    ex_allgatherv_dev(X, *in.zx, in.dl_z, in.rows_per_rank, 4, dlz_g.p);
    dlz = dlz_g.p;
    if (in.row_sp) {
      rsp_g = X.alloc<uint8_t>(D);
      ex_allgatherv_dev(X, *in.zx, in.row_sp, in.rows_per_rank, 1, rsp_g.p);
      rsp = rsp_g.p;
    }
  }
  // P2 setup, enqueued BEFORE the hot pass: the cold CSR's size is read back
  // while P1 runs (the host waits on a mark, not on the stream), so P2's
  // scatter and kernel queue behind P1 without an idle gap. With the
  // warp-bitmap kernel the dense rows are cut into `parts` ranges so that 24
  // warps per SM each hold a part_rows-bit bitmap; the cold CSR is keyed by
  // (variant, part, y).
  // the cold join of the K actually used (its estimate is exact: the job's dR
  // and dense-row counts), so every rank of a z-split job agrees
  int kidx = best;
  for (int j = 0; j < kKCand; ++j)
    if (kv[j] == K) kidx = j;
  const bool run_cold = e[kidx] > 0;
  uint32_t parts = 1, part_rows = (uint32_t)(((D + 31) / 32) * 32);
  uint32_t var_bits = 0, vskip = ~0u;
  uint64_t rows_key = 0, cnnz = 0;
  DBuf<uint32_t> cc, ch;  // (variant, part, y) counts; (part, y, mask) histogram
  // cptr_buf = {0, segment starts...}: the scan is written one slot in
  // (cpos, the scatter's cursors); after the scatter cptr_buf is the cptr
  DBuf<uint64_t> cptr_buf;
  uint64_t* cpos = nullptr;
  if (run_cold) {
    if (cold_bitmap) {
      // bitmap + deferred rows + compacted segments
      const uint64_t per_warp = budget / cold_ctas / kColdWarps - (kDQ + kSegWords) * 4;
      const uint64_t rows_cap = std::max<uint64_t>(32, per_warp * 8 / 32 * 32);
      parts = (uint32_t)((D + rows_cap - 1) / rows_cap);
      part_rows = (uint32_t)((((D + parts - 1) / parts) + 31) / 32 * 32);
    }
    // top-rank variants of the cold CSR (only for the warp-bitmap kernel): one
    // bit per top rank that at least half of the live x contain (cfg2: ranks
    // 0-2; cfg4's flatter Zipf(0.8): none)
    const uint64_t xc_job = zs ? in.x_card_job : in.x_card;  // the same bits on every rank
    if (cold_kernel_ok)
      // (a 4th bit pays on large dense blocks: cfg5 87.3 -> 85.6 ms; cfg2 2.28 -> 2.37)
      // (a sharded job gathers the cold CSR: the 4th bit's extra records cost
      // more NVLink time than they save a rank)
      while (var_bits < (D > (4ull << 20) && !zs ? kMaxVarBits : 3u) && var_bits < Y &&
             2ull * top_rank_dr[var_bits] >= xc_job)
        ++var_bits;
    if (cold_kernel_ok && std::getenv("D3G_VAR_BITS"))  // experiments: 0..4
      var_bits = (uint32_t)std::min<uint64_t>(env_u32("D3G_VAR_BITS", var_bits, 0, 4), Y);
    // with 4 bits the variant of x holding only the 4th top rank is not built
    // (it would copy half of all cold entries for the few x without the top
    // three); those x stream variant 0
    vskip = var_bits == 4 ? 8u : ~0u;
    rows_key = ((uint64_t)1 << var_bits) * parts * Y;
    // per (part, y, top-mask) histogram, then the (variant, part, y) counts
    const uint64_t n_py = (uint64_t)parts * Y;
    ch = X.zeros<uint32_t>(n_py * kHistSlots);
    if (DL)
      D3G_LAUNCH(X, cold_hist_kernel, grid_for(DL, 256), 256, 0, in.dl_ptr, in.dl_col, DL,
                 in.y_of_rank, ch.p, Y, part_rows, reinterpret_cast<const uint64_t*>(hzl), kw,
                 var_bits, row_lo);
    cc = X.alloc<uint32_t>(rows_key);
    if (n_py)
      D3G_LAUNCH(X, cold_cnt_from_hist_kernel, grid_for(n_py, 256), 256, 0, ch.p, n_py, Y, parts,
                 var_bits, vskip, cc.p);
    cptr_buf = X.alloc<uint64_t>(rows_key + 2);
    cpos = cptr_buf.p + 1;
    D3G_CUDA(cudaMemsetAsync(cptr_buf.p, 0, 8, X.stream));
    exclusive_scan<uint32_t>(X, cc.p, rows_key, cpos);
    X.defer(&cnnz, cpos + rows_key, 8);
    X.mark();
  }
  // z-split: the cold CSR is built now, for this rank's rows, and merged with
  // the other ranks' parts into the job's (variant, part, y)-major layout
  DBuf<uint4> crec_g;
  if (zs && run_cold) {
    if (!cold_kernel_ok) throw d3g::Error(D3G_INTERNAL_ERROR, "z-split needs the cold kernels");
    X.wait_mark();  // cnnz of this rank
    const int N = in.zx->nranks;
    // every rank's offsets (its exclusive scan over its counts)
    DBuf<uint64_t> cp_all = X.alloc<uint64_t>((rows_key + 1) * N);
    ex_allgatherv_dev(X, *in.zx, cpos, std::vector<uint64_t>(N, rows_key + 1), 8, cp_all.p);
    DBuf<uint4> crec_l = X.alloc<uint4>(cnnz);
    if (DL)
      D3G_LAUNCH(X, cold_scatter_cur_kernel, grid_for(DL, 256), 256, 0, in.dl_ptr, in.dl_col,
                 DL, in.y_of_rank, reinterpret_cast<unsigned long long*>(cpos), Y, part_rows,
                 parts, reinterpret_cast<const uint64_t*>(hzl), kw, var_bits, vskip, row_lo,
                 crec_l.p, (uint32_t*)nullptr, in.row_sp);
    cc.reset();
    ch.reset();
    // the ranks' record counts, their parts gathered rank-major
    uint64_t mine = cnnz;
    std::vector<uint64_t> part_n(N);
    ex_allgather(X, *in.zx, &mine, part_n.data(), 8);
    std::vector<uint64_t> part_b(N, 0);
    uint64_t tot = 0;
    for (int q = 0; q < N; ++q) {
      part_b[q] = tot;
      tot += part_n[q];
    }
    DBuf<uint4> crec_all = X.alloc<uint4>(tot);
    ex_allgatherv_dev(X, *in.zx, crec_l.p, part_n, 16, crec_all.p);
    crec_l.reset();
    // the job's offsets: the sum of the ranks' scans
    D3G_LAUNCH(X, sum_rows_u64_kernel, grid_for(rows_key + 1, 256), 256, 0, cp_all.p, rows_key + 1,
               N, cptr_buf.p);
    DBuf<uint64_t> pb = X.alloc<uint64_t>(N);
    X.to_device(pb.p, part_b.data(), N);
    crec_g = X.alloc<uint4>(tot);
    // long segments: at most tot / kMergeLong of them
    DBuf<LongSeg> longs = X.alloc<LongSeg>(tot / kMergeLong + 1);
    DBuf<unsigned int> n_long = X.zeros<unsigned int>(1);
    D3G_LAUNCH(X, cold_merge_kernel, grid_for((rows_key + 31) / 32 * 32, 256, X.sm_count * 16), 256,
               0, cp_all.p, pb.p, crec_all.p, cptr_buf.p, rows_key, N, crec_g.p, longs.p, n_long.p);
    D3G_LAUNCH(X, cold_merge_long_kernel, X.sm_count * 8, 256, 0, longs.p, n_long.p, crec_all.p,
               crec_g.p);
    cnnz = tot;
  }
  // P1: hot bit-sliced pass
  DBuf<uint32_t> tail_rows_g, tail_col_g;  // z-split: the long rows' tails
  DBuf<uint64_t> tail_ptr_g;
  HotParams hp{};
  hp.T = T.p;
  hp.hz = reinterpret_cast<const uint64_t*>(hz.p);
  hp.xorder = hot_xorder;
  hp.dl_z = dlz;
  hp.n_live = hot_n;
  hp.n_dense = D;
  hp.groups = (uint32_t)((hot_n + 127) / 128);
  hp.K = K;
  hp.kw = kw;
  hp.batch = 32;
  // (batch, z range) units per SM without the pivot plan (cfg4: 8 -> 16,
  // hot 17.6 -> 16.8 ms)
  const uint64_t zc_per_sm = env_u32("D3G_ZCHUNKS_PER_SM", 16, 1, 64);
  hp.z_chunks = std::max<uint32_t>(1, (uint32_t)std::min<uint64_t>(
      (D + 255) / 256,
      ((uint64_t)X.sm_count * zc_per_sm + n_batches - 1) / std::max<uint32_t>(n_batches, 1)));
  const bool plan = !unit_off_h.empty();
  DBuf<uint32_t> unit_off_d;
  DBuf<uint8_t> batch_kind_d;
  if (plan) {
    unit_off_d = X.alloc<uint32_t>(n_batches + 1);
    batch_kind_d = X.alloc<uint8_t>(n_batches);
    X.to_device(unit_off_d.p, unit_off_h.data(), n_batches + 1);
    X.to_device(batch_kind_d.p, batch_kind_h.data(), n_batches);
    hp.unit_off = unit_off_d.p;
    hp.batch_kind = batch_kind_d.p;
    for (uint32_t q = 0; q <= kMC; ++q) hp.run_lo[q] = run_lo[q];
    for (uint32_t q = 0; q < kMC; ++q) hp.run_zc[q] = run_zc[q];
    hp.n_classes = n_kinds;
    hp.plan_units = unit_off_h[n_batches];
    hp.plan_on = 1;
  }
  DBuf<unsigned int> work = X.zeros<unsigned int>(1);
  hp.work = work.p;
  // the shared class-0 batches: the same kernel on the pooled slice tables,
  // one class run = this rank's row slice, every batch of kind 0
  HotParams h0 = hp;
  DBuf<uint32_t> uoff0;
  DBuf<uint8_t> bkind0;
  DBuf<unsigned int> work0;
  uint32_t zc0 = 0;
  if (n0_job) {
    const uint64_t slice = sh_hi - sh_lo;
    zc0 = (uint32_t)std::max<uint64_t>(
        1, std::min<uint64_t>((slice + 255) / 256, ((uint64_t)X.sm_count * 4 + nb0 - 1) / nb0));
    std::vector<uint32_t> uo(nb0 + 1);
    for (uint32_t b = 0; b <= nb0; ++b) uo[b] = b * (slice ? zc0 : 0u);
    uoff0 = X.alloc<uint32_t>(nb0 + 1);
    bkind0 = X.zeros<uint8_t>(nb0);
    X.to_device(uoff0.p, uo.data(), nb0 + 1);
    work0 = X.zeros<unsigned int>(1);
    h0.T = T0.p;
    h0.n_live = n0_job;
    h0.groups = (uint32_t)((n0_job + 127) / 128);
    h0.unit_off = uoff0.p;
    h0.batch_kind = bkind0.p;
    for (uint32_t q = 0; q <= kMC; ++q) h0.run_lo[q] = q == 0 ? sh_lo : sh_hi;
    for (uint32_t q = 0; q < kMC; ++q) h0.run_zc[q] = q == 0 ? (slice ? zc0 : 0u) : 0u;
    h0.n_classes = 1;
    h0.plan_units = uo[nb0];
    h0.plan_on = 1;
    h0.work = work0.p;
  }
  // [hot tally | cold tally | hot-pass LDS units]: read back once at the end
  // [hot | cold | LDS units | pairs of folded sparse rows]
  // [.. | slice reads without prefix sharing]
  // [.. | folded sparse rows among the rows with the top rank (split)]
  DBuf<Tally> tallies = X.zeros<Tally>(6);
  Tally* t = tallies.p;
  unsigned long long* lds_units = &tallies.p[2].count;
  unsigned long long* cnt_sp = in.row_sp ? &tallies.p[3].count : nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
  bool trie = false, jt_trie = false;
  size_t sm = (size_t)K * 32 * 16;
  const uint64_t n_units = plan ? (uint64_t)hp.plan_units : (uint64_t)n_batches * hp.z_chunks;
  // (a plan can leave nothing to test: every pair shares a pivot)
  unsigned g = (unsigned)std::min<uint64_t>(std::max<uint64_t>(n_units, 1), (uint64_t)X.sm_count);
  const char* hot_impl = std::getenv("D3G_HOT");
  const bool use_tc = hot_impl && std::string(hot_impl) == "tc" && mode == kModeCount &&
                      K % 32 == 0 && K <= 384;
  if (use_tc) {
    // tensor-core comparison path (denseec_tc.cuh): count-only
    const uint32_t n_xt = (uint32_t)((n_live + kTcM - 1) / kTcM);
    const uint32_t n_zt = (uint32_t)((D + kTcN - 1) / kTcN);
    DBuf<uint8_t> A = X.zeros<uint8_t>((uint64_t)n_xt * kTcM * K);
    DBuf<uint8_t> B = X.zeros<uint8_t>((uint64_t)n_zt * kTcN * K);
    D3G_LAUNCH(X, tc_build_a_kernel, grid_for(n_live * 32, 256), 256, 0, xorder, n_live, in.r_ptr,
               in.r_col, in.y_rank, K, A.p);
    D3G_LAUNCH(X, tc_build_b_kernel, grid_for(D * 32, 256), 256, 0, in.dl_ptr, in.dl_col, D, K,
               B.p);
    const uint32_t x_chunks = std::max<uint32_t>(
        1, std::min<uint32_t>(n_xt, ((uint32_t)X.sm_count * 4 + n_zt - 1) / n_zt));
    DBuf<unsigned int> tw = X.zeros<unsigned int>(1);
    const size_t tsm = (size_t)(kTcN + 2 * kTcM) * K;
    auto kfn = dense_tc_kernel<kModeCount>;
    D3G_CUDA(raise_smem_attr(kfn, (int)tsm));
    D3G_LAUNCH(X, kfn, (unsigned)std::min<uint64_t>((uint64_t)n_zt * x_chunks, X.sm_count),
               kTcThreads, tsm, A.p, B.p, K, n_xt, n_zt, n_live, D, x_chunks, tw.p, t);
  } else if (K <= 256 && !(hot_impl && std::string(hot_impl) == "list")) {
    // packed hot records (default; D3G_HOT=list selects the list kernel), with
    // the top-rank subset table when it fits (D3G_HOT=rec disables it)
    // the table pays off when the top ranks are common in the dense rows
    // (cfg2/cfg5: >= 3 of the top 7 per row; cfg4's flat Zipf(0.8): < 1)
    const size_t tsm = (size_t)(kTabRows + K - kTabBits) * 32 * 16;
    double top_per_row = 0;
    for (uint32_t r = 0; r < kTabBits; ++r) top_per_row += (double)top_rank_rows[r] / (double)D;
    const std::string hv = hot_impl ? hot_impl : "";
    const bool force_tab = hv == "tab" || hv == "trie";
    // (z-split: the job-wide plan decision, so every rank's records agree)
    const bool tab = (zs ? try_plan : plan) ||
                     K > kTabBits && tsm <= (size_t)dense_smem_bytes(X) &&
                     !(hot_impl && std::string(hot_impl) == "rec") &&
                     (force_tab || top_per_row >= 1.5);
    DBuf<uint4> rec = X.zeros<uint4>(2 * D);
    DBuf<uint32_t> rcnt = X.alloc<uint32_t>(D);
    // the jump-table kernel by default, with or without the subset table;
    // D3G_HOT=tab|trie|rec select the guarded-step table kernel, the standalone
    // prefix-shared kernel or the guarded-step record kernel (comparison)
    const bool jt = hv != "tab" && hv != "trie" && hv != "rec";
    // prefix-shared rows by default with the table (D3G_HOT=jt keeps the
    // dense-row order; D3G_HOT=jttrie forces them without the table, where
    // they measured slower: cfg4 23.2 vs 17.2 ms)
    jt_trie = jt && ((tab && hv != "jt") || hv == "jttrie");
    trie = jt_trie || (tab && hv == "trie");
    if (!zs) {
      D3G_LAUNCH(X, hot_rec_kernel, grid_for(D, 256), 256, 0, in.dl_ptr, in.dl_col, D, K,
                 tab ? kTabBits : 0u, reinterpret_cast<uint8_t*>(rec.p), rcnt.p, in.row_sp,
                 jt && tab ? kTabBits : 0u);
    } else {
      // z-split: this rank's rows' records and count words, gathered; the long
      // rows' list tails (past the record's 32 listed ranks) gathered apart
      DBuf<uint4> rec_l = X.zeros<uint4>(2 * DL);
      DBuf<uint32_t> rcnt_l = X.alloc<uint32_t>(DL);
      if (DL)
        D3G_LAUNCH(X, hot_rec_kernel, grid_for(DL, 256), 256, 0, in.dl_ptr, in.dl_col, DL, K,
                   tab ? kTabBits : 0u, reinterpret_cast<uint8_t*>(rec_l.p), rcnt_l.p, in.row_sp,
                   jt && tab ? kTabBits : 0u);
      std::vector<uint64_t> rr2(in.rows_per_rank);
      for (auto& v : rr2) v *= 2;
      ex_allgatherv_dev(X, *in.zx, rec_l.p, rr2, 16, rec.p);
      ex_allgatherv_dev(X, *in.zx, rcnt_l.p, in.rows_per_rank, 4, rcnt.p);
      const int N = in.zx->nranks;
      DBuf<uint32_t> tlen = X.alloc<uint32_t>(DL), ist = X.alloc<uint32_t>(DL);
      DBuf<uint64_t> toff = X.alloc<uint64_t>(DL + 1), tpos = X.alloc<uint64_t>(DL + 1);
      if (DL)
        D3G_LAUNCH(X, tail_len_kernel, grid_for(DL, 256), 256, 0, rcnt_l.p, DL, tlen.p, ist.p);
      exclusive_scan<uint32_t>(X, tlen.p, DL, toff.p);
      exclusive_scan<uint32_t>(X, ist.p, DL, tpos.p);
      uint64_t tn[2] = {0, 0};  // tail rows, tail ranks
      X.defer(&tn[0], tpos.p + DL, 8);
      X.defer(&tn[1], toff.p + DL, 8);
      X.sync();
      DBuf<uint32_t> t_rows = X.alloc<uint32_t>(tn[0]), t_col = X.alloc<uint32_t>(tn[1]);
      DBuf<uint64_t> t_ptr = X.alloc<uint64_t>(tn[0]);
      if (DL && tn[0])
        D3G_LAUNCH(X, tail_fill_kernel, grid_for(DL, 256), 256, 0, rcnt_l.p, DL, ist.p, tpos.p,
                   toff.p, in.dl_ptr, in.dl_col, row_lo, t_rows.p, t_ptr.p, t_col.p);
      std::vector<uint64_t> all_tn(2 * N);
      ex_allgather(X, *in.zx, tn, all_tn.data(), 16);
      std::vector<uint64_t> nrows(N), ncols(N), r0(N + 1, 0), c0(N + 1, 0);
      for (int q = 0; q < N; ++q) {
        nrows[q] = all_tn[2 * q];
        ncols[q] = all_tn[2 * q + 1];
        r0[q + 1] = r0[q] + nrows[q];
        c0[q + 1] = c0[q] + ncols[q];
      }
      if (r0[N]) {
        tail_rows_g = X.alloc<uint32_t>(r0[N]);
        tail_ptr_g = X.alloc<uint64_t>(r0[N]);
        tail_col_g = X.alloc<uint32_t>(c0[N]);
        ex_allgatherv_dev(X, *in.zx, t_rows.p, nrows, 4, tail_rows_g.p);
        ex_allgatherv_dev(X, *in.zx, t_ptr.p, nrows, 8, tail_ptr_g.p);
        ex_allgatherv_dev(X, *in.zx, t_col.p, ncols, 4, tail_col_g.p);
        DBuf<uint64_t> dr0 = X.alloc<uint64_t>(N + 1), dc0 = X.alloc<uint64_t>(N + 1);
        X.to_device(dr0.p, r0.data(), N + 1);
        X.to_device(dc0.p, c0.data(), N + 1);
        D3G_LAUNCH(X, tail_rebase_kernel, grid_for(r0[N], 256), 256, 0, tail_ptr_g.p, dr0.p, dc0.p,
                   N);
      }
      hp.tail_rows = tail_rows_g.p;
      hp.tail_ptr = tail_ptr_g.p;
      hp.tail_col = tail_col_g.p;
      hp.n_tail = (uint32_t)r0[N];
      // no long rows anywhere: a non-null table keeps the kernel off the
      // (local) lists; with no row past 32 listed ranks it is never read
      if (!hp.tail_rows) hp.tail_rows = rcnt.p;
    }
    // prefix-shared records: rows sorted by (subset, r1, r2), records gathered
    DBuf<uint32_t> perm;
    if (trie) {
      DBuf<uint64_t> key = X.alloc<uint64_t>(D);
      perm = X.alloc<uint32_t>(D);
      D3G_LAUNCH(X, trie_key_kernel, grid_for(D, 256), 256, 0, reinterpret_cast<const uint8_t*>(rec.p),
                 rcnt.p, D, key.p, perm.p, jt ? 1u : 1u - kTabBits,
                 (zs ? try_plan : plan) ? n_piv : 0u);
      radix_sort(X, key.p, perm.p, D, 25 + ((zs ? try_plan : plan) ? (int)n_piv : 0), true);
      DBuf<uint4> rec_s = X.alloc<uint4>(2 * D);
      DBuf<uint32_t> rcnt_s = X.alloc<uint32_t>(D);
      D3G_LAUNCH(X, trie_gather_kernel, grid_for(D, 256), 256, 0, rec.p, rcnt.p, key.p, perm.p, D,
                 rec_s.p, rcnt_s.p);
      rec = std::move(rec_s);
      rcnt = std::move(rcnt_s);
      if (jt_trie) {
        // slice reads of every (batch, row) the kernel tests, with and without
        // the prefix sharing
        if (plan) {
          TrieRuns tr{};  // each class run, times its batches: one launch
          for (uint32_t q = 0; q < n_kinds; ++q) {
            const uint64_t rows = run_lo[q + 1] - run_lo[q];
            if (!run_mult[q] || !rows) continue;
            const uint32_t k = tr.n_runs++;
            tr.zc[k] = run_zc[q];
            tr.row0[k] = run_lo[q];
            tr.mult[k] = run_mult[q];
            tr.start[k + 1] = tr.start[k] + rows;
          }
          if (tr.n_runs)
            D3G_LAUNCH(X, trie_lds_runs_kernel, grid_for(tr.start[tr.n_runs], 256), 256, 0, rcnt.p,
                       tr, tab ? 1u : 0u, lds_units, &tallies.p[4].count);
        } else {
          D3G_LAUNCH(X, trie_lds_kernel, grid_for(D, 256), 256, 0, rcnt.p, D, hp.z_chunks,
                     tab ? 1u : 0u, lds_units, &tallies.p[4].count, (uint64_t)n_batches, 0ull);
        }
        if (n0_job && sh_hi > sh_lo)  // the shared class-0 batches over this rank's row slice
          D3G_LAUNCH(X, trie_lds_kernel, grid_for(sh_hi - sh_lo, 256), 256, 0, rcnt.p,
                     sh_hi - sh_lo, zc0, tab ? 1u : 0u, lds_units, &tallies.p[4].count,
                     (uint64_t)nb0, sh_lo);
      }
    } else {
      // algorithmic LDS traffic: every (row, batch) reads its listed slices plus
      // (tab) one subset-table entry, 512 B each
      D3G_LAUNCH(X, rec_sum_kernel, grid_for(D, 256), 256, 0, rcnt.p, D, tab ? 1u : 0u, lds_units);
    }
    D3G_CUDA(cudaEventCreate(&ev0));
    D3G_CUDA(cudaEventCreate(&ev1));
    D3G_CUDA(cudaEventRecord(ev0, X.stream));
    with_mode(mode, [&](auto M) {
      if (jt) {
        // without the table: K listed rows plus one (zero) subset row
        const size_t jsm = tab ? tsm : (size_t)(K + 1) * 32 * 16;
        auto run = [&](auto kfn) {
          D3G_CUDA(raise_smem_attr(kfn, (int)jsm));
          D3G_LAUNCH(X, kfn, g, kHotThreads, jsm, hp, in.dl_ptr, in.dl_col, rec.p, rcnt.p, perm.p,
                     dec, em, t, cnt_sp);
          h0.tail_rows = hp.tail_rows;  // (set with the records, after h0 was made)
          h0.tail_ptr = hp.tail_ptr;
          h0.tail_col = hp.tail_col;
          h0.n_tail = hp.n_tail;
          if (n0_job && h0.plan_units)  // the shared class-0 batches
            D3G_LAUNCH(X, kfn, std::min<unsigned>(h0.plan_units, X.sm_count), kHotThreads, jsm, h0,
                       in.dl_ptr, in.dl_col, rec.p, rcnt.p, perm.p, dec, em, t, cnt_sp);
        };
        constexpr int Md = decltype(M)::value;
        if (tab && jt_trie)
          run(dense_hot_jt_kernel<Md, true, true>);
        else if (tab)
          run(dense_hot_jt_kernel<Md, false, true>);
        else if (jt_trie)
          run(dense_hot_jt_kernel<Md, true, false>);
        else
          run(dense_hot_jt_kernel<Md, false, false>);
      } else if (!D3G_COMPARISON_KERNELS) {
        throw ConfigError("D3G_HOT=" + hv + " selects a comparison kernel; build with make "
                          "COMPARE=1");
#if D3G_COMPARISON_KERNELS
      } else if (trie) {
        // the kernel counts its own slice reads (over every batch)
        auto kfn = dense_hot_trie_kernel<decltype(M)::value>;
        D3G_CUDA(raise_smem_attr(kfn, (int)tsm));
        D3G_LAUNCH(X, kfn, g, kTrieThreads, tsm, hp, in.dl_ptr, in.dl_col, rec.p, rcnt.p, perm.p,
                   dec, em, t, cnt_sp, lds_units);
      } else if (tab) {
        auto kfn = dense_hot_tab_kernel<decltype(M)::value>;
        D3G_CUDA(raise_smem_attr(kfn, (int)tsm));
        D3G_LAUNCH(X, kfn, g, kHotThreads, tsm, hp, in.dl_ptr, in.dl_col, rec.p, rcnt.p, dec, em,
                   t, cnt_sp);
      } else {
        auto kfn = dense_hot_rec_kernel<decltype(M)::value>;
        D3G_CUDA(raise_smem_attr(kfn, (int)sm));
        D3G_LAUNCH(X, kfn, g, kHotThreads, sm, hp, in.dl_ptr, in.dl_col, rec.p, rcnt.p, dec, em,
                   t, cnt_sp);
#endif
      }
    });
    D3G_CUDA(cudaEventRecord(ev1, X.stream));
  } else {
    // K > 256 (no cold kernel: D3G_COLD=tiers) or D3G_HOT=list: the list kernel
    with_mode(mode, [&](auto M) {
      auto kfn = dense_hot_kernel<decltype(M)::value>;
      D3G_CUDA(raise_smem_attr(kfn, (int)sm));
      D3G_LAUNCH(X, kfn, g, kHotThreads, sm, hp, in.dl_ptr, in.dl_col, dec, em, t);
    });
  }
  // P2: cold residual join, hot-hit candidates filtered
  KernelOut cold;
  if (run_cold) {
    X.wait_mark();  // cnnz
    // cold kernels: 16-byte records {hz word 0, fold of words 1-3, row}; the
    // scatter writes the row fields, one coalesced pass fills the signatures.
    // D3G_COLD=tiers: a plain column of row ids for the SparseBMM tiers.
    // (z-split: built and merged before the hot pass)
    DBuf<uint32_t> ccol;
    DBuf<uint4> crec;
    if (cold_kernel_ok && D >= kRowMask)
      throw d3g::Error(D3G_INTERNAL_ERROR, "cold records hold row ids below 2^31 - 1");
    const uint4* hz4 = reinterpret_cast<const uint4*>(hz.p);
    if (zs) {
      crec = std::move(crec_g);
    } else {
      if (cold_kernel_ok) crec = X.alloc<uint4>(cnnz);
      else ccol = X.alloc<uint32_t>(cnnz);
      D3G_LAUNCH(X, cold_scatter_cur_kernel, grid_for(D, 256), 256, 0, in.dl_ptr, in.dl_col,
                 D, in.y_of_rank, reinterpret_cast<unsigned long long*>(cpos), Y, part_rows,
                 parts, reinterpret_cast<const uint64_t*>(hz.p), kw, var_bits, vskip, 0ull,
                 cold_kernel_ok ? crec.p : nullptr, ccol.p, rsp);
      cc.reset();
      ch.reset();
    }
    if (cold_kernel_ok) {
      DBuf<unsigned int> next = X.zeros<unsigned int>(1);
      Tally* tc = tallies.p + 1;
      // records streamed (.count) and exact tail checks (.sum)
      unsigned long long* cand = &tallies.p[5].count;
      D3G_CUDA(cudaEventCreate(&ev2));
      D3G_CUDA(cudaEventCreate(&ev3));
      D3G_CUDA(cudaEventRecord(ev2, X.stream));
      // the star segment (x's longest: looked up, never inserted); an x whose
      // star is longer than this is handed to the CTA tier
      const uint32_t star_route = env_u32("D3G_COLD_STAR", D3G_COLD_ROUTE, 1, 0xffffffffu);
      // D3G_TRACE: per-tier wall time (synchronised; diagnostics only)
      const bool ttrace = std::getenv("D3G_TRACE") != nullptr;
      auto tier = [&](const char* name, auto&& launch) {
        if (!ttrace) return launch();
        D3G_CUDA(cudaStreamSynchronize(X.stream));
        const auto t0 = std::chrono::steady_clock::now();
        launch();
        D3G_CUDA(cudaStreamSynchronize(X.stream));
        std::fprintf(stderr, "[cold tier] %s %.3f ms\n", name,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
      };
      if (cold_hash) {
        DBuf<uint32_t> over_x = X.alloc<uint32_t>(n_live);
        DBuf<unsigned int> over_n = X.zeros<unsigned int>(1);
        const size_t hsm = kCHSmem;
        tier("warp hash", [&] { with_mode(mode, [&](auto M) {
          auto kfn = dense_cold_hash_kernel<decltype(M)::value>;
          D3G_CUDA(raise_smem_attr(kfn, (int)hsm));
          D3G_LAUNCH(X, kfn, (unsigned)X.sm_count * (D3G_CH_BITS <= 10 ? D3G_CH_CTAS : 3), kCHWarps * 32, hsm,
                     xorder, n_live, in.r_ptr, in.r_col, cptr_buf.p, crec.p, hz4,
                     reinterpret_cast<const uint4*>(hx.p), Y, var_bits, vskip, dlz, dec, em, next.p,
                     over_x.p, over_n.p, tc, cnt_sp,
                     env_u32("D3G_COLD_HASH_MAX", kCHMax, 1, kCHMax),
                     env_u32("D3G_COLD_ROUTE", D3G_COLD_ROUTE, 1, 0xffffffffu), star_route, cand);
        }); });
        const unsigned int n_over = X.scalar(over_n.p);
        out.cold_overflow = n_over;
        // overflowing x: a CTA-wide shared-memory hash first; the few past its
        // limit go on to the CTA-private global bitmaps (1.25 MB each on cfg5,
        // which thrash L2 when every overflowing x uses one)
        const char* ov_env = std::getenv("D3G_COLD_OVERFLOW");
        const bool cta_tier = !(ov_env && std::string(ov_env) == "bitmap");
        unsigned int n_over2 = n_over;
        DBuf<uint32_t> over2_x;
        DBuf<unsigned int> over2_n;
        if (n_over && cta_tier) {
          over2_x = X.alloc<uint32_t>(n_over);
          over2_n = X.zeros<unsigned int>(1);
          tier("cta hash", [&] { with_mode(mode, [&](auto M) {
            auto kfn = dense_cold_cta_kernel<decltype(M)::value>;
            D3G_CUDA(raise_smem_attr(kfn, (int)kCCSmem));
            D3G_LAUNCH(X, kfn, std::min<unsigned>(n_over, (unsigned)X.sm_count * kCCPerSm), kCCThreads,
                       kCCSmem, over_x.p, over_n.p, in.r_ptr, in.r_col, cptr_buf.p, crec.p, hz4,
                       reinterpret_cast<const uint4*>(hx.p), Y, var_bits, vskip, dlz, dec, em,
                       over2_x.p, over2_n.p, env_u32("D3G_COLD_CTA_MAX", kCCMax, 1, kCCMax), tc,
                       cnt_sp, cand);
          }); });
          n_over2 = X.scalar(over2_n.p);
        }
        if (n_over2) {
          const uint32_t* ox = cta_tier ? over2_x.p : over_x.p;
          const unsigned int* on = cta_tier ? over2_n.p : over_n.p;
          const uint64_t words = (D + 31) / 32;
          if (env_u32("D3G_OV_SHARED", 1, 0, 1)) {
            // shared bitmaps, kOvShare CTAs per x, in rounds of at most ~1 GB
            // of bitmaps (dense_cold_shared_kernel): insert launch, star launch
            const uint32_t per_round = (uint32_t)std::max<uint64_t>(
                1, std::min<uint64_t>(n_over2, (1ull << 30) / (words * 4)));
            DBuf<uint32_t> gbm = X.alloc<uint32_t>((uint64_t)per_round * words);
            tier("bitmap (shared)", [&] {
              for (uint32_t lo = 0; lo < n_over2; lo += per_round) {
                const uint32_t xn = std::min<uint32_t>(per_round, n_over2 - lo);
                D3G_CUDA(cudaMemsetAsync(gbm.p, 0, (uint64_t)xn * words * 4, X.stream));
                for (int phase = 0; phase < 2; ++phase)
                  with_mode(mode, [&](auto M) {
                    D3G_LAUNCH(X, dense_cold_shared_kernel<decltype(M)::value>, xn * kOvShare,
                               kOvThreads, kOvSmem, ox, lo, xn, phase, in.r_ptr, in.r_col,
                               cptr_buf.p, crec.p, hz4, reinterpret_cast<const uint4*>(hx.p), Y,
                               var_bits, vskip, dlz, gbm.p, words, dec, em, tc, cnt_sp, cand);
                  });
              }
            });
          } else {
          const unsigned og = (unsigned)std::min<uint64_t>(
              (uint64_t)n_over2,
              (uint64_t)env_u32("D3G_OVERFLOW_CTAS", X.sm_count * kOvPerSm, 1, X.sm_count * 16));
          DBuf<uint32_t> gbm = X.zeros<uint32_t>((uint64_t)og * words);
          DBuf<uint32_t> touched = X.alloc<uint32_t>((uint64_t)og * kOvTouched);
          tier("bitmap", [&] { with_mode(mode, [&](auto M) {
            D3G_LAUNCH(X, dense_cold_overflow_kernel<decltype(M)::value>, og, kOvThreads, kOvSmem, ox,
                       on, in.r_ptr, in.r_col, cptr_buf.p, crec.p, hz4,
                       reinterpret_cast<const uint4*>(hx.p), Y, var_bits, vskip, dlz, gbm.p, words,
                       dec, em, tc, cnt_sp, touched.p, cand);
          }); });
          }
        }
        out.cold_overflow2 = n_over2;
      } else {
        const size_t csm = ((size_t)(part_rows / 32) + kDQ + kSegWords) * 4 * kColdWarps;
        with_mode(mode, [&](auto M) {
          auto kfn = dense_cold_kernel<decltype(M)::value>;
          if (csm > 48 * 1024)
            D3G_CUDA(raise_smem_attr(kfn, (int)csm));
          D3G_LAUNCH(X, kfn, (unsigned)X.sm_count * cold_ctas, kColdWarps * 32, csm, xorder, n_live,
                     in.r_ptr, in.r_col, cptr_buf.p, crec.p, hz4, reinterpret_cast<const uint4*>(hx.p), Y,
                     parts, part_rows, var_bits, vskip, dlz, dec, em, next.p, tc, cnt_sp, cand);
        });
      }
      D3G_CUDA(cudaEventRecord(ev3, X.stream));
    } else {
      SparseInputs si{in.r_ptr, in.r_col, in.x_card, cptr_buf.p, ccol.p, in.dl_z, D, Y, in.x_lo, in.x_hi};
      Filter flt{reinterpret_cast<const uint64_t*>(hx.p), reinterpret_cast<const uint64_t*>(hz.p), kw};
      run_sparse(X, si, dec, mode, em, cold, flt);
    }
  }
  Tally th[6];
  X.to_host(th, tallies.p, 6);
  // pairs of pure batches with rows sharing a pivot: hits, untested
  const uint64_t direct = plan_direct;
  out.count_sp = th[3].count + plan_direct_sp;
  const Tally& h = th[0];
  if (cold_kernel_ok && run_cold) {
    cold.count = th[1].count;
    cold.sum = th[1].sum;
    cold.xr = th[1].xr;
  }
  if (ev0) {
    float ms = 0;
    D3G_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    out.ms_hot = ms;
    // jump-table kernel with prefix sharing / standalone trie kernel: the
    // counters already cover every batch
    out.hot_lds_bytes = th[2].count * (trie ? 1ull : (uint64_t)n_batches) * 512ull;
    out.hot_lds_bytes_unshared = jt_trie ? th[4].count * 512ull : out.hot_lds_bytes;
    out.split_direct_pairs = plan_direct;
  }
  if (ev2) {
    float ms = 0;
    D3G_CUDA(cudaEventElapsedTime(&ms, ev2, ev3));
    cudaEventDestroy(ev2);
    cudaEventDestroy(ev3);
    out.ms_cold = ms;
    // 16-byte records streamed + 32-byte hz rows of the exact tail checks
    out.cold_bytes = th[5].count * 16ull + th[5].sum * 32ull;
    out.cold_candidates = th[5].count;
    out.cold_tail_checks = th[5].sum;
  }
  if (std::getenv("D3G_TRACE"))
    std::fprintf(stderr, "[dense_hot] D=%llu live=%llu K=%u hot=%llu cold=%llu cold_path=%s over=%llu over2=%llu\n",
                 (unsigned long long)D, (unsigned long long)n_live, K, (unsigned long long)h.count,
                 (unsigned long long)cold.count,
                 cold_bitmap ? "bitmap" : cold_hash ? "hash" : "tiers",
                 (unsigned long long)out.cold_overflow, (unsigned long long)out.cold_overflow2);
  out.count = h.count + direct + cold.count;
  out.sum = h.sum + cold.sum;
  out.xr = h.xr ^ cold.xr;
  out.inner = K;  // reported as the hot width (diagnostics)
}

// DenseEC dispatch: v3 (hot + cold residual) by default; D3G_DENSE=v1|v2
// selects the list-streaming or z-tile-resident kernels (kept for comparison).
void run_dense(Ctx& X, const DenseInputs& in, d3g::Decode dec, int mode, d3g::Emit em,
               KernelOut& out) {
  const char* v = std::getenv("D3G_DENSE");
  std::string which = v ? v : "v3";
#if D3G_COMPARISON_KERNELS
  if (which == "v1")
    run_dense_streaming(X, in, dec, mode, em, out);
  else if (which == "v2")
    run_dense_tiles(X, in, dec, mode, em, out);
  else
    run_dense_hot(X, in, dec, mode, em, out);
#else
  if (which == "v1" || which == "v2")
    throw d3g::ConfigError("D3G_DENSE=" + which + " selects a comparison kernel; build with make "
                           "COMPARE=1");
  run_dense_hot(X, in, dec, mode, em, out);
#endif
}

__global__ void decode_pairs_kernel(const uint32_t* __restrict__ xc, const uint32_t* __restrict__ zc,
                                    uint64_t n, const uint64_t* __restrict__ rev_x,
                                    const uint64_t* __restrict__ rev_z, int swapped,
                                    uint64_t* __restrict__ ox, uint64_t* __restrict__ oz) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t ex = rev_x ? rev_x[xc[i]] : xc[i];
    uint64_t ez = rev_z ? rev_z[zc[i]] : zc[i];
    ox[i] = swapped ? ez : ex;
    oz[i] = swapped ? ex : ez;
  }
}

// Rows of a pair CSR (caller x code -> sorted caller z codes) to decoded
// raw pairs, 8 lanes per row (rev == null: identity codes).
__global__ void csr_decode_kernel(const uint64_t* __restrict__ row_ptr,
                                  const uint32_t* __restrict__ col, uint64_t n_rows,
                                  const uint64_t* __restrict__ rev_a,
                                  const uint64_t* __restrict__ rev_b, uint64_t* __restrict__ ox,
                                  uint64_t* __restrict__ oz) {
  const uint32_t sl = threadIdx.x & 7;
  for (uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3; r < n_rows;
       r += ((uint64_t)gridDim.x * blockDim.x) >> 3) {
    const uint64_t b = row_ptr[r], e = row_ptr[r + 1];
    if (b == e) continue;
    const uint64_t a = rev_a ? rev_a[r] : r;
    for (uint64_t k = b + sl; k < e; k += 8) {
      ox[k] = a;
      oz[k] = rev_b ? rev_b[col[k]] : col[k];
    }
  }
}

__global__ void pair_key_kernel(const uint32_t* __restrict__ xc, const uint32_t* __restrict__ zc,
                                uint64_t n, int swapped, int lo_bits, uint64_t* __restrict__ keys,
                                uint32_t* __restrict__ idx) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t a = swapped ? zc[i] : xc[i], b = swapped ? xc[i] : zc[i];
    keys[i] = (a << lo_bits) | b;
    idx[i] = (uint32_t)i;
  }
}

__global__ void permute_pairs_kernel(const uint32_t* __restrict__ idx, uint64_t n,
                                     const uint32_t* __restrict__ xc, const uint32_t* __restrict__ zc,
                                     uint32_t* __restrict__ oxc, uint32_t* __restrict__ ozc) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    oxc[i] = xc[idx[i]];
    ozc[i] = zc[idx[i]];
  }
}


__global__ void map_through_kernel(uint32_t* __restrict__ v, uint64_t n,
                                   const uint32_t* __restrict__ table) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = table[v[i]];
}

// Device layouts of the dense block consumed by dense_ec_kernel.
struct DenseLayout {
  DBuf<uint32_t> y_rank, y_of_rank, dl_z, dl_col, xorder;
  DBuf<uint64_t> dl_ptr;
  uint64_t n_live = 0, n_dense = 0, max_group_nnz = 0, dnnz = 0;
};

// Rows of a CSR ordered by degree, descending, in one counting scatter whose
// offsets come from the host degree histogram (hist[d] = rows of degree d,
// all rows). mode / table: see degree_scatter_kernel. With want_ptr the rows'
// list offsets are written too (rows of equal degree have equal lengths).
struct DegreeOrder {
  DBuf<uint32_t> rows;
  DBuf<uint64_t> ptr;
  DBuf<uint8_t> sp;
  uint64_t n = 0, nnz = 0;
};

void order_by_degree(Ctx& X, const uint64_t* row_ptr, uint64_t r0, uint64_t r1,
                     const std::vector<uint64_t>& hist, const uint8_t* d_table,
                     const std::vector<uint8_t>* h_table, int mode, bool want_ptr, bool want_sp,
                     DegreeOrder& o) {
  using namespace d3g;
  const uint64_t maxd = hist.empty() ? 0 : hist.size() - 1;
  std::vector<uint64_t> oe(2 * (maxd + 1), 0);
  uint64_t pos = 0, e = 0;
  for (uint64_t d = maxd; d >= 1; --d) {
    const bool sparse = !(h_table && d < h_table->size() && (*h_table)[d]);
    if (!(mode == 0 || (mode == 1 ? !sparse : sparse))) continue;
    oe[d] = pos;
    oe[maxd + 1 + d] = e;
    pos += hist[d];
    e += hist[d] * d;
  }
  o.n = pos;
  o.nnz = e;
  DBuf<uint64_t> doe = X.alloc<uint64_t>(oe.size());
  X.to_device(doe.p, oe.data(), oe.size());
  DBuf<unsigned int> cur = X.zeros<unsigned int>(maxd + 1);
  o.rows = X.alloc<uint32_t>(o.n);
  if (want_ptr) o.ptr = X.alloc<uint64_t>(o.n + 1);
  if (want_sp) o.sp = X.alloc<uint8_t>(o.n);
  if (r1 > r0 || want_ptr)
    D3G_LAUNCH(X, degree_scatter_kernel, grid_for(std::max<uint64_t>(r1 - r0, 1), 256), 256, 0,
               row_ptr, r0, r1, d_table, h_table ? (uint64_t)h_table->size() : 0ull, mode, doe.p,
               doe.p + maxd + 1, cur.p, o.rows.p, want_ptr ? o.ptr.p : nullptr, o.n, o.nnz,
               want_sp ? o.sp.p : nullptr);
}

// Selection of the layout's rows by degree (the f2 table), instead of a
// row-id list: rows come out ordered and with their list offsets in one pass.
struct RowSel {
  const std::vector<uint64_t>* hmz;   // m_z histogram (all rows)
  const uint8_t* d_table;             // f2 table on the device
  const std::vector<uint8_t>* table;  // and on the host
  int mode;                           // degree_scatter_kernel mode
  DBuf<uint8_t>* sp_out;              // mode 0: per layout row, "is a sparse z"
};

// y codes ordered by dR descending (ties in any order): a counting sort when
// the value range is small, else the LSD radix sort.
void order_y_by_degree(Ctx& X, const uint32_t* dR, uint64_t y_card, uint64_t max_dr,
                       DBuf<uint32_t>& order, bool deterministic = false) {
  using namespace d3g;
  order = X.alloc<uint32_t>(y_card);
  if (y_card == 0) return;
  // (the counting scatter orders ties as its atomics land; ranks of a z-split
  // job must agree on the ranking: the stable radix sort then)
  if (max_dr < (1ull << 20) && !deterministic) {
    DBuf<uint32_t> cnt = X.zeros<uint32_t>(max_dr + 1);
    D3G_LAUNCH(X, desc_hist_kernel, grid_for(y_card, 256), 256, 0, dR, y_card, (uint32_t)max_dr,
               cnt.p);
    DBuf<uint64_t> off = X.alloc<uint64_t>(max_dr + 2);
    exclusive_scan<uint32_t>(X, cnt.p, max_dr + 1, off.p);
    D3G_LAUNCH(X, desc_scatter_kernel, grid_for(y_card, 256), 256, 0, dR, y_card,
               (uint32_t)max_dr, off.p, cnt.p, order.p);
    return;
  }
  DBuf<uint64_t> k = X.alloc<uint64_t>(y_card);
  D3G_LAUNCH(X, degree_order_key_kernel, grid_for(y_card, 256), 256, 0, (const uint32_t*)nullptr,
             y_card, (const uint64_t*)nullptr, dR, max_dr, k.p, order.p);
  radix_sort(X, k.p, order.p, y_card, bits_for(max_dr), false);
}

// rows: dense z rows given as (row_ptr, col) indexed by row id; row_ids
// lists the n_dense row ids (or sel selects them by degree); z_of_row
// (nullable) maps a row id to its z code (identity when null). dR: per-y
// R-side degrees (hotness).
void build_dense_layout(Ctx& X, const d3g::DeviceCsr& rx, uint64_t max_mx,
                        const std::vector<uint64_t>& hmx, const uint64_t* zrow_ptr,
                        const uint32_t* zcol, const uint32_t* row_ids, uint64_t n_dense,
                        uint64_t max_mz, const uint32_t* z_of_row, uint64_t y_card,
                        const uint32_t* dR, DenseLayout& L, uint64_t xa = 0,
                        uint64_t xb = ~0ull, uint64_t dnnz_hint = ~0ull,
                        const RowSel* sel = nullptr, uint64_t z_rows = 0,
                        bool stable_x = false, uint64_t dr_bound = 0, uint64_t z_base = 0,
                        bool det_rank = false) {
  using namespace d3g;
  // y ranked by dR descending: hottest witnesses first. dR(y) <= x_card
  // bounds the key without a device round trip (sharded: dR is the job's,
  // bounded by the job's x card, dr_bound).
  const uint64_t max_dr = std::max<uint64_t>(rx.n_rows, dr_bound);
  order_y_by_degree(X, dR, y_card, max_dr, L.y_of_rank, det_rank);
  L.y_rank = X.alloc<uint32_t>(y_card);
  D3G_LAUNCH(X, scatter_rank_kernel, grid_for(y_card, 256), 256, 0, L.y_of_rank.p, y_card,
             L.y_rank.p);
  // dense rows ordered by m_z descending (uniform trip counts per warp)
  DBuf<uint32_t> rows;
  uint64_t dnnz = 0;
  if (sel) {
    DegreeOrder o;
    order_by_degree(X, zrow_ptr, 0, z_rows, *sel->hmz, sel->d_table, sel->table, sel->mode, true,
                    sel->sp_out != nullptr, o);
    n_dense = o.n;
    dnnz = o.nnz;
    rows = std::move(o.rows);
    L.dl_ptr = std::move(o.ptr);
    if (sel->sp_out) *sel->sp_out = std::move(o.sp);
  } else {
    rows = X.alloc<uint32_t>(n_dense);
    {
      DBuf<uint64_t> k = X.alloc<uint64_t>(n_dense);
      D3G_LAUNCH(X, degree_order_key_kernel, grid_for(n_dense, 256), 256, 0, row_ids, n_dense,
                 zrow_ptr, (const uint32_t*)nullptr, max_mz, k.p, rows.p);
      radix_sort(X, k.p, rows.p, n_dense, bits_for(max_mz), false);
    }
    DBuf<uint32_t> len = X.alloc<uint32_t>(n_dense);
    D3G_LAUNCH(X, gather_len_kernel, grid_for(n_dense, 256), 256, 0, rows.p, n_dense, zrow_ptr, len.p);
    L.dl_ptr = X.alloc<uint64_t>(n_dense + 1);
    exclusive_scan<uint32_t>(X, len.p, n_dense, L.dl_ptr.p);
    len.reset();
    dnnz = dnnz_hint != ~0ull ? dnnz_hint : X.scalar(L.dl_ptr.p + n_dense);
  }
  L.n_dense = n_dense;
  L.dnnz = dnnz;
  {
    L.dl_col = X.alloc<uint32_t>(dnnz);
    D3G_LAUNCH(X, dense_list_fill_kernel, grid_for(n_dense * 8, 256), 256, 0, rows.p, n_dense,
               zrow_ptr, zcol, L.dl_ptr.p, L.y_rank.p, L.dl_col.p);
    DBuf<uint32_t> kept = X.alloc<uint32_t>(n_dense);
    segmented_sort(X, L.dl_col.p, L.dl_ptr.p, n_dense, /*unique=*/false, kept.p, max_mz);
  }
  if (z_of_row) D3G_LAUNCH(X, map_through_kernel, grid_for(n_dense, 256), 256, 0, rows.p, n_dense, z_of_row);
  // z-split: the rows are this rank's z codes counted from z_base
  if (z_base && n_dense)
    D3G_LAUNCH(X, add_offset_kernel, grid_for(n_dense, 256), 256, 0, rows.p, n_dense, (uint32_t)z_base);
  L.dl_z = std::move(rows);
  // live x ordered by m_x descending, cut into 128-x groups
  // (restricted to x codes in [xa, xb) when the caller asked for an x range)
  if (xb > rx.n_rows) xb = rx.n_rows;
  if (xa > xb) xa = xb;
  const uint64_t x_card = xb - xa;
  // Every live x: one counting scatter with offsets from the m_x histogram
  // (ties in arbitrary order). x shards split the x ORDER by position, so
  // sharded calls (stable_x) use the stable sort: every rank then sees the
  // same order and the shards partition the x exactly.
  const bool full_range = xa == 0 && xb == rx.n_rows;
  if (full_range && !stable_x) {
    DegreeOrder o;
    order_by_degree(X, rx.row_ptr.p, 0, x_card, hmx, nullptr, nullptr, 0, false, false, o);
    L.n_live = o.n;
    L.xorder = std::move(o.rows);
  } else {
    DBuf<uint32_t> lf = X.alloc<uint32_t>(x_card);
    if (x_card) D3G_LAUNCH(X, live_flag_kernel, grid_for(x_card, 256), 256, 0, rx.row_ptr.p, xa, xb, lf.p);
    DBuf<uint64_t> lp = X.alloc<uint64_t>(x_card + 1);
    exclusive_scan<uint32_t>(X, lf.p, x_card, lp.p);
    if (full_range) {  // the m_x histogram knows how many
      L.n_live = 0;
      for (uint64_t m = 1; m < hmx.size(); ++m) L.n_live += hmx[m];
    } else {
      L.n_live = X.scalar(lp.p + x_card);
    }
    DBuf<uint32_t> live_ids = X.alloc<uint32_t>(L.n_live);
    if (x_card)
      D3G_LAUNCH(X, index_compact_kernel, grid_for(x_card, 256), 256, 0, lf.p, lp.p, x_card, live_ids.p);
    if (xa && L.n_live)
      D3G_LAUNCH(X, add_offset_kernel, grid_for(L.n_live, 256), 256, 0, live_ids.p, L.n_live, (uint32_t)xa);
    DBuf<uint64_t> k = X.alloc<uint64_t>(L.n_live);
    L.xorder = X.alloc<uint32_t>(L.n_live);
    if (L.n_live)
      D3G_LAUNCH(X, degree_order_key_kernel, grid_for(L.n_live, 256), 256, 0, live_ids.p, L.n_live,
                 rx.row_ptr.p, (const uint32_t*)nullptr, max_mx, k.p, L.xorder.p);
    radix_sort(X, k.p, L.xorder.p, L.n_live, bits_for(max_mx), false);
  }
  // group 0 holds the 128 largest m_x: bound for the per-group cold table
  uint64_t top = 0, seen = 0;
  for (uint64_t m = max_mx; m >= 1 && seen < 128; --m) {
    uint64_t take = std::min<uint64_t>(hmx[m], 128 - seen);
    top += take * m;
    seen += take;
  }
  L.max_group_nnz = top;
}

// Materialized output: emit code pairs (emit runs the producing kernels in
// kModeEmit), order them by (x, z) code, decode through the dictionaries
// (identity when rev is null) in the caller's orientation, copy out.
void finish_pairs(Ctx& X, DBuf<uint32_t>& ex, DBuf<uint32_t>& ez, uint64_t total,
                  const uint64_t* rev_x, const uint64_t* rev_z, bool swapped, d3g_pairs* pairs,
                  d3g_report* rep, uint64_t x_card, uint64_t z_card);

void materialize_pairs(Ctx& X, uint64_t total, const std::function<void(d3g::Emit)>& emit,
                       const uint64_t* rev_x, const uint64_t* rev_z, bool swapped,
                       d3g_pairs* pairs, d3g_report* rep, uint64_t x_card, uint64_t z_card) {
  using namespace d3g;
  if (pairs->x && pairs->cap < total)
    throw ResourceError("output buffer holds " + std::to_string(pairs->cap) + " pairs, need " +
                        std::to_string(total));
  DBuf<uint32_t> ex = X.alloc<uint32_t>(total), ez = X.alloc<uint32_t>(total);
  DBuf<unsigned long long> cur = X.zeros<unsigned long long>(1);
  emit(Emit{ex.p, ez.p, cur.p, total});
  {
    // the buffer was sized by the counting pass; the emitting kernels must
    // have produced exactly that many pairs (no truncation, no unwritten slots)
    const uint64_t emitted = X.scalar(cur.p);
    if (emitted != total)
      throw CudaError("materialize: emitted " + std::to_string(emitted) + " pairs, counted " +
                      std::to_string(total));
  }
  finish_pairs(X, ex, ez, total, rev_x, rev_z, swapped, pairs, rep, x_card, z_card);
}

// Emitted code pairs -> sorted by (x, z), decoded to raw values in the
// caller's orientation, copied to the caller's buffers -- or, when the
// caller passed no buffer (pairs->x == NULL), kept on the device for
// d3g_take_pairs (one pipeline pass whatever the output size).
void finish_pairs(Ctx& X, DBuf<uint32_t>& ex, DBuf<uint32_t>& ez, uint64_t total,
                  const uint64_t* rev_x, const uint64_t* rev_z, bool swapped, d3g_pairs* pairs,
                  d3g_report* rep, uint64_t x_card, uint64_t z_card) {
  using namespace d3g;
  const bool trace = std::getenv("D3G_TRACE") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto tr = [&](const char* what) {
    if (!trace) return;
    X.sync();
    auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[materialize] %-8s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - tp).count());
    tp = t1;
  };
  tr("emit");
  DBuf<uint64_t> ox, oz;
  uint64_t* dox = pairs->x;
  uint64_t* doz = pairs->z;
  const bool held = pairs->x == nullptr;  // library-owned result
  auto out_buffers = [&] {
    if (!pairs->on_device || held) {
      ox = X.alloc<uint64_t>(total);
      oz = X.alloc<uint64_t>(total);
      dox = ox.p;
      doz = oz.p;
    }
  };
  // (x, z) order through the bucketed CSR build (the pairs are distinct, so
  // rows of caller-x codes with sorted caller-z codes ARE the sorted list):
  // one scatter + shared-memory sorts instead of a 6-8 pass radix sort
  {
    const uint64_t a_card = swapped ? z_card : x_card, b_card = swapped ? x_card : z_card;
    DeviceCsr g;
    if (total && std::getenv("D3G_PAIR_RADIX") == nullptr &&
        build_csr_bucketed(X, swapped ? ez.p : ex.p, swapped ? ex.p : ez.p, total, a_card, b_card,
                           g, false)) {
      if (g.nnz != total) throw CudaError("materialize: duplicate pairs emitted");
      tr("sort");
      ex.reset();
      ez.reset();
      out_buffers();
      D3G_LAUNCH(X, csr_decode_kernel, grid_for(a_card * 8, 256), 256, 0, g.row_ptr.p, g.col.p,
                 a_card, swapped ? rev_z : rev_x, swapped ? rev_x : rev_z, dox, doz);
      tr("decode");
      if (held) {
        X.held_x = std::move(ox);
        X.held_z = std::move(oz);
        X.held_n = total;
      } else if (!pairs->on_device) {
        X.copy_to_pageable(pairs->x, ox.p, total * 8);
        X.copy_to_pageable(pairs->z, oz.p, total * 8);
      }
      tr("d2h");
      pairs->n = total;
      return;
    }
  }
  DBuf<uint64_t> keys = X.alloc<uint64_t>(total);
  DBuf<uint32_t> idx = X.alloc<uint32_t>(total);
  if (total) {
    // sort key = (caller x code, caller z code) packed in as few bits as the
    // code spaces need (fewer 8-bit radix passes than a 64-bit key)
    const uint64_t a_card = swapped ? z_card : x_card, b_card = swapped ? x_card : z_card;
    const int lo = std::max(1, bits_for(b_card ? b_card - 1 : 0));
    const int hi = std::max(1, bits_for(a_card ? a_card - 1 : 0));
    D3G_LAUNCH(X, pair_key_kernel, grid_for(total, 256), 256, 0, ex.p, ez.p, total,
               swapped ? 1 : 0, lo, keys.p, idx.p);
    radix_sort(X, keys.p, idx.p, total, std::min(64, lo + hi), false);
  }
  tr("sort");
  DBuf<uint32_t> sx2 = X.alloc<uint32_t>(total), sz2 = X.alloc<uint32_t>(total);
  if (total)
    D3G_LAUNCH(X, permute_pairs_kernel, grid_for(total, 256), 256, 0, idx.p, total, ex.p, ez.p,
               sx2.p, sz2.p);
  out_buffers();
  if (total)
    D3G_LAUNCH(X, decode_pairs_kernel, grid_for(total, 256), 256, 0, sx2.p, sz2.p, total, rev_x,
               rev_z, swapped ? 1 : 0, dox, doz);
  tr("decode");
  if (held) {
    ex.reset();
    ez.reset();
    X.held_x = std::move(ox);
    X.held_z = std::move(oz);
    X.held_n = total;
  } else if (!pairs->on_device && total) {
    X.copy_to_pageable(pairs->x, ox.p, total * 8);
    X.copy_to_pageable(pairs->z, oz.p, total * 8);
  }
  tr("d2h");
  pairs->n = total;
}

// estimate_out_j_raw on the device-resident y columns (see classical.cuh).
// Launched early, read at the next round trip (EstimateJob::value).
struct EstimateJob {
  DBuf<uint64_t> smp;
  DBuf<unsigned long long> keys, hits;
  DBuf<unsigned int> counts;
  unsigned long long h = 0;
  bool exact = true, empty = true;
  uint64_t nr = 0, ns = 0, mr = 0, ms = 0;
  uint64_t value(Ctx& X) {
    if (empty) return 0;
    if (X.has_deferred()) X.sync();
    if (exact) return h;
    long double scaled = static_cast<long double>(h) * (static_cast<long double>(ns) / ms) *
                         (static_cast<long double>(nr) / mr);
    if (scaled > static_cast<long double>(std::numeric_limits<uint64_t>::max()))
      return std::numeric_limits<uint64_t>::max();
    return static_cast<uint64_t>(scaled);
  }
};

void estimate_out_j_start(Ctx& X, const uint64_t* r_y, uint64_t nr, const uint64_t* s_y,
                          uint64_t ns, EstimateJob& J) {
  using namespace d3g;
  J.empty = nr == 0 || ns == 0;
  if (J.empty) return;
  const uint64_t exact_limit = 65536, sample_rows = 16384;
  J.exact = nr <= exact_limit && ns <= exact_limit;
  J.nr = nr;
  J.ns = ns;
  J.ms = J.exact ? ns : std::min(ns, sample_rows);
  J.mr = J.exact ? nr : std::min(nr, sample_rows);
  const uint64_t ss = J.exact ? 1 : ns / J.ms, sr = J.exact ? 1 : nr / J.mr;
  J.smp = X.alloc<uint64_t>(J.mr + J.ms);
  D3G_LAUNCH(X, gather_stride_kernel, grid_for(J.mr, 256), 256, 0, r_y, sr, J.mr, J.smp.p);
  D3G_LAUNCH(X, gather_stride_kernel, grid_for(J.ms, 256), 256, 0, s_y, ss, J.ms, J.smp.p + J.mr);
  uint64_t cap = 1024;
  while (cap < 2 * J.ms) cap <<= 1;
  J.keys = X.alloc<unsigned long long>(cap);
  D3G_CUDA(cudaMemsetAsync(J.keys.p, 0xff, cap * 8, X.stream));
  J.counts = X.zeros<unsigned int>(cap + 1);
  J.hits = X.zeros<unsigned long long>(1);
  D3G_LAUNCH(X, est_insert_kernel, grid_for(J.ms, 256), 256, 0, J.smp.p + J.mr, J.ms, J.keys.p,
             J.counts.p, cap - 1);
  D3G_LAUNCH(X, est_probe_kernel, grid_for(J.mr, 256), 256, 0, J.smp.p, J.mr, J.keys.p,
             J.counts.p, cap - 1, J.hits.p);
  X.defer(&J.h, J.hits.p, 8);
}


// hash_join_dedup (P/src/classical.cpp:111-210) on the GPU, in engine
// orientation; pairs swap back through decode.
void classical_impl(Ctx& X, const uint64_t* Rl, const uint64_t* Rr, uint64_t NR,
                    const uint64_t* Sl, const uint64_t* Sr, uint64_t NS, bool swapped, int mode,
                    bool materialize, d3g_report* rep, d3g_pairs* pairs) {
  using namespace d3g;
  const bool trace = std::getenv("D3G_CLS_TRACE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto tr = [&](const char* what) {
    if (!trace) return;
    X.sync();
    auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cls] %-10s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  DictBundle D;
  DBuf<uint32_t> s_y = X.alloc<uint32_t>(NS), s_z = X.alloc<uint32_t>(NS);
  DBuf<uint32_t> r_y = X.alloc<uint32_t>(NR), keep = X.alloc<uint32_t>(NR);
  DBuf<uint32_t> r_x = X.alloc<uint32_t>(NR);
  dict_build(X, Sr, NS, D.y, s_y.p);  // y groups (FlatMap over S.y)
  dict_build(X, Sl, NS, D.z, s_z.p);  // z interner
  dict_build(X, Rl, NR, D.x, r_x.p);  // x interner
  tr("dicts");
  if (NR)
    D3G_LAUNCH(X, dict_lookup_kernel, grid_for(NR, 256), 256, 0, Rr, NR, D.y.keys.p,
               D.y.slot_code.p, D.y.mask, r_y.p, keep.p);
  const uint64_t G = D.y.card;
  DBuf<uint32_t> gcnt = X.zeros<uint32_t>(G);
  if (NS) D3G_LAUNCH(X, group_hist_kernel, grid_for(NS, 256), 256, 0, s_y.p, NS, gcnt.p);
  DBuf<uint64_t> gptr = X.alloc<uint64_t>(G + 1);
  exclusive_scan<uint32_t>(X, gcnt.p, G, gptr.p);
  if (G) D3G_CUDA(cudaMemsetAsync(gcnt.p, 0, G * 4, X.stream));
  DBuf<uint32_t> gz = X.alloc<uint32_t>(NS);
  if (NS)
    D3G_LAUNCH(X, group_scatter_kernel, grid_for(NS, 256), 256, 0, s_y.p, s_z.p, NS, gptr.p,
               gcnt.p, gz.p);
  DBuf<unsigned long long> bag = X.zeros<unsigned long long>(1);
  if (NR)
    D3G_LAUNCH(X, classical_bag_kernel, grid_for(NR, 256), 256, 0, r_y.p, keep.p, NR, gptr.p,
               bag.p);
  const uint64_t inter = X.scalar(bag.p);
  tr("groups");
  rep->intermediate_pairs = inter;
  uint64_t cap = 1024;
  while (cap < 2 * inter) cap <<= 1;
  DBuf<unsigned long long> set = X.alloc<unsigned long long>(cap);  // ResourceError if too big
  Decode dec{rev_or_null(D.x), rev_or_null(D.z), swapped ? 1 : 0};
  auto run = [&](int m, Emit em, Tally* t) {
    D3G_CUDA(cudaMemsetAsync(set.p, 0xff, cap * 8, X.stream));
    if (NR == 0) return;
    const unsigned g = grid_for(NR * 32, 256, X.sm_count * 32);
    with_mode(m, [&](auto M) {
      D3G_LAUNCH(X, classical_probe_kernel<decltype(M)::value>, g, 256, 0, r_x.p, r_y.p, keep.p,
                 NR, gptr.p, gz.p, set.p, cap - 1, dec, em, t);
    });
  };
  tr("set alloc");
  DBuf<Tally> t = X.zeros<Tally>(1);
  run(mode, Emit{nullptr, nullptr, nullptr, 0}, t.p);
  Tally h;
  X.to_host(&h, t.p, 1);
  tr("probe");
  rep->pairs_classical = h.count;
  rep->out_p = h.count;
  rep->rank_out_p = h.count;
  rep->nranks = 1;
  rep->checksum_sum = h.sum;
  rep->checksum_xor = h.xr;
  if (materialize) {
    DBuf<Tally> t2 = X.zeros<Tally>(1);
    materialize_pairs(X, h.count, [&](Emit em) { run(kModeEmit, em, t2.p); }, rev_or_null(D.x),
                      rev_or_null(D.z), swapped, pairs, rep, D.x.card, D.z.card);
  }
}

// ---------------------------------------------------------------------------
// Self-join detection: R and S element-wise identical (cfg2's S := R). Blocks
// stop at the first difference any of them has seen.
__global__ void tables_differ_kernel(const uint64_t* __restrict__ a0, const uint64_t* __restrict__ b0,
                                     const uint64_t* __restrict__ a1, const uint64_t* __restrict__ b1,
                                     uint64_t n, unsigned int* __restrict__ differ) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride * 4) {
    bool d = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t i = base + k * stride + threadIdx.x;
      if (i < n) d |= (a0[i] != b0[i]) | (a1[i] != b1[i]);
    }
    if (__syncthreads_or(d)) {  // block-uniform exits only
      if (threadIdx.x == 0) atomicExch(differ, 1u);
      return;
    }
    if (__syncthreads_or(*(volatile unsigned int*)differ != 0)) return;
  }
}

// Launched early, read at the next round trip (IdentityJob::value).
struct IdentityJob {
  DBuf<unsigned int> differ;
  unsigned int h = 1;
  int known = -1;  // 0/1 when decided on the host
  bool value(Ctx& X) {
    if (known >= 0) return known != 0;
    if (X.has_deferred()) X.sync();
    return h == 0;
  }
};

void tables_identical_start(Ctx& X, const uint64_t* Rl, const uint64_t* Rr, const uint64_t* Sl,
                            const uint64_t* Sr, uint64_t NR, uint64_t NS, IdentityJob& J) {
  using namespace d3g;
  if (NR != NS || NR == 0) {
    J.known = 0;
    return;
  }
  if (Rl == Sl && Rr == Sr) {
    J.known = 1;
    return;
  }
  J.differ = X.zeros<unsigned int>(1);
  D3G_LAUNCH(X, tables_differ_kernel, grid_for(NR, 256, X.sm_count * 4), 256, 0, Rl, Sl, Rr, Sr,
             NR, J.differ.p);
  X.defer(&J.h, J.differ.p, 4);
}

// A read-only view of a (the self-join's S-by-z is R-by-x): b shares a's
// buffers without owning them; a must outlive b.
void view_csr(const d3g::DeviceCsr& a, d3g::DeviceCsr& b) {
  b.n_rows = a.n_rows;
  b.n_cols = a.n_cols;
  b.nnz = a.nnz;
  b.max_deg = a.max_deg;
  b.live_rows = a.live_rows;
  b.row_ptr.p = a.row_ptr.p;
  b.row_ptr.n = a.row_ptr.n;
  b.col.p = a.col.p;
  b.col.n = a.col.n;
}

// ---------------------------------------------------------------------------
// Pipeline stages shared by join_project and join_aggregate_both.

// Steps 3-4: natural-key resolution (engine.cpp:25-50, mapping.cpp:281-338)
// and map_tables (mapping.cpp:342-420). Natural columns use the narrowed
// codes of the one-pass statistics kernel; the others go through HBM
// dictionaries. With want_kept the original indices of the surviving R rows
// are produced too (when the semi-join dropped any).
struct Mapped {
  DictBundle D;
  DBuf<uint32_t> nar, s_y_own, s_z_own, r_y_own, r_x_own, r_kept;
  const uint32_t *r_x = nullptr, *r_y = nullptr, *s_z = nullptr, *s_y = nullptr;
  uint64_t kept = 0, x_card = 0, y_card = 0, z_card = 0;
  uint64_t x_card_job = 0;  // the job's x card (sharded: summed local dictionaries)
  // a declared natural-key skip the data does not allow (require_natural's
  // ConfigError, mapping.cpp:328-338). The reference raises it inside
  // map_tables, which its classical branch never calls (engine.cpp:386-395):
  // the columns are dictionary-coded here and the caller raises the error
  // unless the classical join runs (check_natural).
  std::string natural_error;
  void check_natural() const {
    if (!natural_error.empty()) throw d3g::ConfigError(natural_error);
  }
  void release_codes() {
    r_x_own.reset();
    r_y_own.reset();
    s_z_own.reset();
    s_y_own.reset();
    nar.reset();
  }
};

void map_inputs(Ctx& X, const uint64_t* Rl, const uint64_t* Rr, uint64_t NR, const uint64_t* Sl,
                const uint64_t* Sr, uint64_t NS, const d3g_opts* o, d3g_report* rep, bool want_kept,
                Mapped& M, d3g::Exchange* E = nullptr, uint64_t nr_global = 0) {
  const bool dist = E && E->active();
  using namespace d3g;
  DBuf<ColStat> cs = X.zeros<ColStat>(4);
  const uint64_t* cols[4] = {Rl, Rr, Sl, Sr};
  const uint64_t lens[4] = {NR, NR, NS, NS};
  // one pass over the four columns: statistics + speculative u32 codes
  M.nar = X.alloc<uint32_t>(2 * NR + 2 * NS);
  uint32_t* ncol[4] = {M.nar.p, M.nar.p + NR, M.nar.p + 2 * NR, M.nar.p + 2 * NR + NS};
  {
    Cols4 c4{};
    for (int i = 0; i < 4; ++i) {
      c4.col[i] = cols[i];
      c4.n[i] = lens[i];
      c4.narrow[i] = ncol[i];
      c4.bound_n[i] = (dist && i < 2) ? nr_global : lens[i];
    }
    const uint64_t mx = std::max(NR, NS);
    if (mx) {
      dim3 grid(grid_for(mx, 256, X.sm_count * 4), 4);
      D3G_LAUNCH(X, colstat4_kernel, grid, 256, 0, c4, cs.p);
    }
  }
  ColStat hs[4];
  X.to_host(hs, cs.p, 4);
  bool r_empty = NR == 0;
  if (dist) {
    // R is this rank's shard: the job's column maxima and sample tests (a
    // shard fails the test if any of its strided samples reaches 2|R|)
    uint64_t v[5] = {hs[0].max, hs[1].max, hs[0].sample_fail, hs[1].sample_fail, NR};
    ex_allreduce_host(X, *E, v, 5, D3G_EX_MAX_U64);
    hs[0].max = v[0];
    hs[1].max = v[1];
    hs[0].sample_fail = (unsigned)v[2];
    hs[1].sample_fail = (unsigned)v[3];
    r_empty = nr_global == 0;
  }
  const uint64_t one_r = r_empty ? 0u : 1u;
  const uint64_t lens_job[4] = {one_r, one_r, NS, NS};
  auto det = [&](int i) { return lens_job[i] > 0 && hs[i].sample_fail == 0; };
  auto fits = [&](int i) { return lens_job[i] == 0 || hs[i].max < (1ull << 32); };
  bool sx = o->declared_x != 0, sy = o->declared_y != 0, sz = o->declared_z != 0;
  // columns holding surrogate ids of byte strings (ColumnType::bytes on the
  // caller's side): never natural keys -- detect_natural_keys is false for
  // them (mapping.cpp:284) and a declared skip is require_natural's error
  // (mapping.cpp:328-331)
  const bool bx = (o->natural_keys_auto & D3G_KEYS_BYTES_X) != 0,
             by = (o->natural_keys_auto & D3G_KEYS_BYTES_Y) != 0,
             bz = (o->natural_keys_auto & D3G_KEYS_BYTES_Z) != 0;
  if ((bx && sx) || (by && sy) || (bz && sz)) {
    M.natural_error = std::string("natural-key skip on column ") +
                      (by && sy ? "y" : bz && sz ? "z" : "x") + " requires integer values";
    sx = sx && !bx;
    sy = sy && !by;
    sz = sz && !bz;
  }
  if (o->natural_keys_auto & D3G_KEYS_AUTO) {
    sx = sx || (!bx && det(0));
    sy = sy || (!by && det(1) && det(3));
    sz = sz || (!bz && det(2));
  }
  auto feasible = [&](bool ax, bool ay, bool az) {
    if (ay && (!fits(1) || !fits(3))) return false;
    if (az && !fits(2)) return false;
    if (ax && !fits(0)) return false;
    return true;
  };
  if (!feasible(sx, sy, sz)) {
    bool dx = o->declared_x != 0 && !bx, dy = o->declared_y != 0 && !by,
         dz = o->declared_z != 0 && !bz;
    if ((sx == dx && sy == dy && sz == dz) || !feasible(dx, dy, dz)) {
      if (M.natural_error.empty())
        M.natural_error = "natural-key skip requires integer values below 2^32";
      dx = dx && fits(0);
      dy = dy && fits(1) && fits(3);
      dz = dz && fits(2);
    }
    sx = dx;
    sy = dy;
    sz = dz;
  }
  rep->natural_x = sx;
  rep->natural_y = sy;
  rep->natural_z = sz;

  DictBundle& D = M.D;
  M.s_y = ncol[3];
  M.s_z = ncol[2];
  M.r_y = ncol[1];
  M.r_x = ncol[0];
  if (sy) {
    uint64_t a = NS ? hs[3].max + 1 : 0, b = !r_empty ? hs[1].max + 1 : 0;
    M.y_card = std::max(a, b);
    D.y.identity = true;
    D.y.card = M.y_card;
  } else {
    M.s_y_own = X.alloc<uint32_t>(NS);
    dict_build(X, Sr, NS, D.y, M.s_y_own.p);
    M.s_y = M.s_y_own.p;
    M.y_card = D.y.card;
  }
  if (sz) {
    M.z_card = NS ? hs[2].max + 1 : 0;
    D.z.identity = true;
    D.z.card = M.z_card;
  } else {
    M.s_z_own = X.alloc<uint32_t>(NS);
    dict_build(X, Sl, NS, D.z, M.s_z_own.p);
    M.s_z = M.s_z_own.p;
    M.z_card = D.z.card;
  }
  // R pass: semi-join filter on y, then x over the survivors. With identity y
  // the filter is disabled (every R.y < y_card = max over both sides + 1).
  M.kept = NR;
  const uint64_t* Rx = Rl;
  DBuf<uint64_t> rx_kept;
  if (!sy && NR) {
    M.r_y_own = X.alloc<uint32_t>(NR);
    DBuf<uint32_t> keep = X.alloc<uint32_t>(NR);
    D3G_LAUNCH(X, dict_lookup_kernel, grid_for(NR, 256), 256, 0, Rr, NR, D.y.keys.p,
               D.y.slot_code.p, D.y.mask, M.r_y_own.p, keep.p);
    DBuf<uint64_t> kpos = X.alloc<uint64_t>(NR + 1);
    exclusive_scan<uint32_t>(X, keep.p, NR, kpos.p);
    M.kept = X.scalar(kpos.p + NR);
    if (M.kept != NR) {
      rx_kept = X.alloc<uint64_t>(M.kept);
      DBuf<uint32_t> ry2 = X.alloc<uint32_t>(M.kept);
      D3G_LAUNCH(X, compact_kernel<uint64_t>, grid_for(NR, 256), 256, 0, Rl, keep.p, kpos.p, NR,
                 rx_kept.p);
      D3G_LAUNCH(X, compact_kernel<uint32_t>, grid_for(NR, 256), 256, 0, M.r_y_own.p, keep.p,
                 kpos.p, NR, ry2.p);
      M.r_y_own = std::move(ry2);
      Rx = rx_kept.p;
      if (want_kept) {  // m.r_kept (mapping.hpp): original indices of the survivors
        M.r_kept = X.alloc<uint32_t>(M.kept);
        D3G_LAUNCH(X, index_compact_kernel, grid_for(NR, 256), 256, 0, keep.p, kpos.p, NR,
                   M.r_kept.p);
      }
    }
    M.r_y = M.r_y_own.p;
  }
  rep->dropped_r = NR - M.kept;
  if (sx) {
    M.x_card = !r_empty ? hs[0].max + 1 : 0;  // over all of R.left (mapping.cpp:404-413)
    D.x.identity = true;
    D.x.card = M.x_card;
    if (M.kept != NR) {
      M.r_x_own = X.alloc<uint32_t>(M.kept);
      if (M.kept)
        D3G_LAUNCH(X, narrow_kernel, grid_for(M.kept, 256), 256, 0, Rx, M.kept, M.r_x_own.p);
      M.r_x = M.r_x_own.p;
    }
  } else {
    M.r_x_own = X.alloc<uint32_t>(M.kept);
    dict_build(X, Rx, M.kept, D.x, M.r_x_own.p);
    M.r_x = M.r_x_own.p;
    M.x_card = D.x.card;
  }
  M.x_card_job = M.x_card;
  if (dist) {
    // shards are disjoint in x: a dictionary x card is the sum of the local
    // ones (natural keys: every rank already holds the job's max + 1)
    uint64_t v[2] = {sx ? 0 : M.x_card, rep->dropped_r};
    ex_allreduce_host(X, *E, v, 2, D3G_EX_SUM_U64);
    if (!sx) M.x_card_job = v[0];
    rep->dropped_r = v[1];
  }
  rep->x_card = M.x_card_job;
  rep->y_card = M.y_card;
  rep->z_card = M.z_card;
  if (M.x_card >= (1ull << 32) || M.y_card >= (1ull << 32) || M.z_card >= (1ull << 32))
    throw ConfigError("code space exceeds 2^32");
}

// Step 6: compute_degree_stats (costmodel.cpp:425-438) on the collapsed CSRs:
// degree histograms, dR/dS and the exact OUT_J (128-bit, saturating).
struct DegreeStats {
  uint64_t max_mx = 0, x_live = 0, max_mz = 0;
  std::vector<uint64_t> hmx, hmz;
  // wz[m] = sum over z rows of degree m of sum_{y in S_z} dR(y): the join size
  // of those rows, so OUT_J of any degree-defined row set (the f2 sparse side:
  // SpaStats::inner_count) is known on the host without another round trip
  std::vector<uint64_t> wz;
  DBuf<uint32_t> dR, dS;
  // sharded job (exchange active): hmx/max_mx/x_live above are this rank's;
  // these are the job's (the f2 inputs). Empty / 0 when not sharded.
  std::vector<uint64_t> hmx_job;
  uint64_t x_live_job = 0;
  // z-split (this rank built S-by-z for its z range only): hmz, wz, dS and
  // max_mz above are the job's; hmz_local orders this rank's rows
  std::vector<uint64_t> hmz_local;
  uint64_t z_live_job = 0;
  const std::vector<uint64_t>& hmx_f2() const { return hmx_job.empty() ? hmx : hmx_job; }
};

void degree_stats(Ctx& X, const d3g::DeviceCsr& rx, const d3g::DeviceCsr& sz_csr,
                  uint64_t y_card, d3g_report* rep, DegreeStats& G, bool same = false,
                  d3g::Exchange* E = nullptr, uint64_t x_card_job = 0, bool zsplit = false) {
  using namespace d3g;
  const bool dist = E && E->active();
  const uint64_t x_card = rx.n_rows, z_card = sz_csr.n_rows;
  if (rx.max_deg != ~0ull && sz_csr.max_deg != ~0ull) {  // read back with the CSR's nnz
    G.max_mx = rx.max_deg;
    G.x_live = rx.live_rows;
    G.max_mz = sz_csr.max_deg;
  } else {
    DBuf<unsigned long long> sc = X.zeros<unsigned long long>(4);  // max_mx, live_x, max_mz, live_z
    if (x_card)
      D3G_LAUNCH(X, max_degree_kernel, grid_for(x_card, 256), 256, 0, rx.row_ptr.p, x_card, sc.p,
                 sc.p + 1);
    if (z_card)
      D3G_LAUNCH(X, max_degree_kernel, grid_for(z_card, 256), 256, 0, sz_csr.row_ptr.p, z_card,
                 sc.p + 2, sc.p + 3);
    unsigned long long scal[4];
    X.to_host(scal, sc.p, 4);
    G.max_mx = scal[0];
    G.x_live = scal[1];
    G.max_mz = scal[2];
  }
  if (zsplit) ex_allreduce_host(X, *E, &G.max_mz, 1, D3G_EX_MAX_U64);  // size the job's histogram
  rep->x_live = G.x_live;
  // one buffer, one read-back: [m_x histogram | m_z histogram | wz | OUT_J partials]
  const unsigned gb = grid_for(y_card, 1024, 296);
  const uint64_t nbuf = (G.max_mx + 1) + 2 * (G.max_mz + 1) + 2ull * gb;
  DBuf<unsigned long long> hbuf = X.zeros<unsigned long long>(nbuf);
  unsigned long long* mxh_p = hbuf.p;
  unsigned long long* mzh_p = hbuf.p + G.max_mx + 1;
  unsigned long long* wz_p = mzh_p + G.max_mz + 1;
  unsigned long long* parts_p = wz_p + G.max_mz + 1;
  if (x_card)
    D3G_LAUNCH(X, degree_hist_kernel, grid_for(x_card, 256), 256, 0, rx.row_ptr.p, x_card,
               G.max_mx + 1, mxh_p);
  if (z_card && !same)
    D3G_LAUNCH(X, degree_hist_kernel, grid_for(z_card, 256), 256, 0, sz_csr.row_ptr.p, z_card,
               G.max_mz + 1, mzh_p);
  G.dR = X.zeros<uint32_t>(y_card);
  if (rx.nnz)
    D3G_LAUNCH(X, value_hist_kernel, grid_for(rx.nnz, 512, X.sm_count * 2), 512, 0, rx.col.p, rx.nnz, G.dR.p,
               (uint32_t)y_card);
  if (same) {  // self-join: S-by-z is R-by-x, so dS = dR (a view)
    G.dS.p = G.dR.p;
    G.dS.n = G.dR.n;
  } else {
    G.dS = X.zeros<uint32_t>(y_card);
  }
  if (!same && sz_csr.nnz)
    D3G_LAUNCH(X, value_hist_kernel, grid_for(sz_csr.nnz, 512, X.sm_count * 2), 512, 0, sz_csr.col.p, sz_csr.nnz,
               G.dS.p, (uint32_t)y_card);
  // sharded: dR(y) of the whole job (the y ranking, OUT_J and the per-degree
  // join sizes below all read it); z-split: dS(y) of the whole job too
  if (dist) ex_allreduce(X, *E, G.dR.p, y_card, D3G_EX_SUM_U32);
  if (zsplit) ex_allreduce(X, *E, G.dS.p, y_card, D3G_EX_SUM_U32);
  if (y_card) D3G_LAUNCH(X, outj_kernel, gb, 1024, 0, G.dR.p, G.dS.p, y_card, parts_p);
  if (z_card)
    D3G_LAUNCH(X, row_join_hist_kernel, grid_for(z_card * 8, 256), 256, 0, sz_csr.row_ptr.p,
               sz_csr.col.p, z_card, G.dR.p, G.max_mz + 1, wz_p);
  std::vector<unsigned long long> hb(nbuf);
  X.to_host(hb.data(), hbuf.p, nbuf);
  G.hmx.assign(hb.begin(), hb.begin() + (G.max_mx + 1));
  if (same)
    G.hmz = G.hmx;
  else
    G.hmz.assign(hb.begin() + (G.max_mx + 1), hb.begin() + (G.max_mx + 1) + (G.max_mz + 1));
  G.wz.assign(hb.begin() + (G.max_mx + 1) + (G.max_mz + 1),
              hb.begin() + (G.max_mx + 1) + 2 * (G.max_mz + 1));
  if (zsplit) {
    // the job's m_z histogram and per-degree join sizes (this rank's rows
    // keep their own histogram for the degree order of its layout)
    G.hmz_local = G.hmz;
    std::vector<uint64_t> v(2 * (G.max_mz + 1));
    std::copy(G.hmz.begin(), G.hmz.end(), v.begin());
    std::copy(G.wz.begin(), G.wz.end(), v.begin() + (G.max_mz + 1));
    ex_allreduce_host(X, *E, v.data(), v.size(), D3G_EX_SUM_U64);
    G.hmz.assign(v.begin(), v.begin() + (G.max_mz + 1));
    G.wz.assign(v.begin() + (G.max_mz + 1), v.end());
    for (uint64_t m = 1; m <= G.max_mz; ++m) G.z_live_job += G.hmz[m];
  }
  const unsigned long long* hp = hb.data() + (G.max_mx + 1) + 2 * (G.max_mz + 1);
  unsigned __int128 acc = 0;
  for (unsigned i = 0; i < gb; ++i) acc += ((unsigned __int128)hp[2 * i + 1] << 64) | hp[2 * i];
  rep->out_j = acc > (unsigned __int128)std::numeric_limits<uint64_t>::max()
                   ? std::numeric_limits<uint64_t>::max()
                   : (uint64_t)acc;
  if (dist) {
    // the job's m_x histogram: sized by the job's largest degree, summed;
    // entry 0 (x codes with no R rows) recomputed from the job's x card
    uint64_t mx = G.max_mx;
    ex_allreduce_host(X, *E, &mx, 1, D3G_EX_MAX_U64);
    G.hmx_job.assign(mx + 1, 0);
    for (uint64_t m = 1; m < G.hmx.size(); ++m) G.hmx_job[m] = G.hmx[m];
    ex_allreduce_host(X, *E, G.hmx_job.data(), mx + 1, D3G_EX_SUM_U64);
    uint64_t live = 0;
    for (uint64_t m = 1; m <= mx; ++m) live += G.hmx_job[m];
    G.hmx_job[0] = x_card_job - live;
    G.x_live_job = live;
    rep->x_live = live;
  }
}

// Step 7a: the f2 decision per degree value (policy.cpp) and the per-z
// dense/sparse flags (the partition.cpp:17-38 decision loop).
struct Split {
  DBuf<uint32_t> isd, iss;  // per z: dense / sparse (m_z == 0: neither)
  uint64_t n_dense = 0, n_sparse = 0;
  // sums of m_z over the dense / sparse rows; exact on the host because the
  // decision is a function of m_z alone (read off the m_z histogram)
  uint64_t dense_nnz = 0, sparse_nnz = 0;
  uint64_t outj_sparse = 0;  // join size of the sparse rows (from DegreeStats::wz)
  std::vector<uint8_t> table;  // the f2 decision per m_z (1 = dense)
  DBuf<uint8_t> dtable;        // and on the device
};

void f2_split(Ctx& X, const d3g::DeviceCsr& sz_csr, const DegreeStats& G, uint64_t x_card,
              uint64_t y_card, const d3g_consts* c, int pforce, d3g_report* rep, Split& P,
              DBuf<uint64_t>* pd_out = nullptr, DBuf<uint64_t>* psp_out = nullptr,
              bool flags = true, uint64_t z_card_job = ~0ull) {
  using namespace d3g;
  const uint64_t z_card = z_card_job != ~0ull ? z_card_job : sz_csr.n_rows;
  P.table.assign(G.max_mz + 1, 0);
  std::vector<uint8_t>& table = P.table;
  uint64_t evals = 0;
  if (const char* dump = std::getenv("D3G_DUMP_F2")) {  // debugging aid: the f2 inputs
    if (FILE* f = std::fopen(dump, "wb")) {
      uint64_t hdr[6] = {G.hmx_f2().size(), G.max_mz + 1, x_card, y_card, z_card, rep->out_j};
      std::fwrite(hdr, 8, 6, f);
      std::fwrite(G.hmx_f2().data(), 8, G.hmx_f2().size(), f);
      std::fwrite(G.hmz.data(), 8, G.max_mz + 1, f);
      std::fclose(f);
    }
  }
  const std::vector<uint64_t>& hx = G.hmx_f2();  // the job's (sharded) or this call's
  d3g_f2_decide(hx.data(), hx.size(), G.hmz.data(), G.max_mz + 1, x_card, y_card, z_card,
                rep->out_j, c, pforce, table.data(), &evals);
  rep->f2_evaluations = evals;
  P.dtable = X.alloc<uint8_t>(G.max_mz + 1);
  X.to_device(P.dtable.p, table.data(), G.max_mz + 1);
  if (flags) {
    P.isd = X.alloc<uint32_t>(z_card);
    P.iss = X.alloc<uint32_t>(z_card);
    if (z_card)
      D3G_LAUNCH(X, dense_flag_kernel, grid_for(z_card, 256), 256, 0, sz_csr.row_ptr.p, z_card,
                 P.dtable.p, G.max_mz + 1, P.isd.p, P.iss.p);
    DBuf<uint64_t> pd = X.alloc<uint64_t>(z_card + 1), psp = X.alloc<uint64_t>(z_card + 1);
    exclusive_scan<uint32_t>(X, P.isd.p, z_card, pd.p);
    exclusive_scan<uint32_t>(X, P.iss.p, z_card, psp.p);
    if (pd_out) *pd_out = std::move(pd);
    if (psp_out) *psp_out = std::move(psp);
  }
  for (uint64_t m = 1; m < G.hmz.size(); ++m) {
    if (table[m]) {
      P.n_dense += G.hmz[m];
      P.dense_nnz += m * G.hmz[m];
    } else {
      P.n_sparse += G.hmz[m];
      P.sparse_nnz += m * G.hmz[m];
      if (m < G.wz.size()) P.outj_sparse += G.wz[m];
    }
  }
  rep->dense_z = P.n_dense;
  rep->sparse_z = P.n_sparse;
  const uint64_t row_words = ((y_card + c->w - 1) / c->w * c->w) / 64;
  rep->panel_bytes = P.n_dense * row_words * 8;
}

// ---------------------------------------------------------------------------
// Reference-equivalent work counters (SpaStats, DenseEcStats): what the
// reference's sparse_bmm / dense_ec would count on this input (the GPU
// kernels do different work; see counters.cuh).

// wide/probe threshold per x degree under a DensePathMode
// (P/src/denseec.cpp:26-43): cost_based = f3_threshold(m_x), force_wide = 0
// (every dense z has m_z >= 1 > 0), force_probe = never wide.
std::vector<uint32_t> mode_thresholds(uint64_t max_mx, uint64_t y_card, const d3g_consts* c,
                                      int dense_mode) {
  std::vector<uint32_t> thr(max_mx + 1, 0);
  for (uint64_t m = 1; m <= max_mx; ++m)
    thr[m] = dense_mode == D3G_DENSE_FORCE_WIDE    ? 0u
             : dense_mode == D3G_DENSE_FORCE_PROBE ? 0xffffffffu
                                                   : d3g_f3_threshold((uint32_t)m, (uint32_t)y_card, c);
  return thr;
}

// Encounter counts and row bitmaps from the degree histograms alone:
// hx[m] live x of degree m, hd[m] dense rows of degree m.
void encounter_counts(const std::vector<uint64_t>& hx, const std::vector<uint64_t>& hd,
                      const std::vector<uint32_t>& thr, d3g::DenseCounters& out) {
  // gt[t] = dense rows with m_z > t
  std::vector<uint64_t> gt(hd.size() + 1, 0);
  for (uint64_t t = hd.size(); t-- > 0;) gt[t] = gt[t + 1] + (t + 1 < hd.size() ? hd[t + 1] : 0);
  const uint64_t n_dense = gt[0];
  if (n_dense == 0) return;
  for (uint64_t m = 1; m < hx.size(); ++m) {
    if (!hx[m]) continue;
    const uint64_t t = m < thr.size() ? thr[m] : 0;
    const uint64_t w = t < gt.size() ? gt[t] : 0;
    out.wide += hx[m] * w;
    out.probe += hx[m] * (n_dense - w);
    if (w) out.bitmaps += hx[m];
  }
}

// Per-pair counters (blocks_checked, probes_done) on the device, plus the
// encounter counts, for x codes [x_lo, x_hi) of r against the dense rows.
void dense_counters_device(Ctx& X, const d3g::DeviceCsr& r, uint64_t x_lo, uint64_t x_hi,
                           const uint64_t* zptr, const uint32_t* zcol, uint64_t z_rows,
                           const uint8_t* dsel, uint64_t dsel_n, const std::vector<uint32_t>& thr,
                           uint32_t w, uint64_t y_card, d3g::DenseCounters& out) {
  using namespace d3g;
  if (x_hi <= x_lo || z_rows == 0) return;
  const uint64_t words = (std::max<uint64_t>(y_card, 1) + 31) / 32;
  const uint64_t smem = words * 4;
  if (smem > 220 * 1024)
    throw ConfigError("collect_counters: |Y| = " + std::to_string(y_card) +
                      " does not fit one shared-memory row bitmap");
  DBuf<uint32_t> dthr = X.alloc<uint32_t>(thr.size());
  X.to_device(dthr.p, thr.data(), thr.size());
  DBuf<DenseCounters> dc = X.zeros<DenseCounters>(1);
  DBuf<unsigned int> next = X.zeros<unsigned int>(1);
  D3G_CUDA(raise_smem_attr(dense_counters_kernel, (int)smem));
  const uint64_t n_blocks = (y_card + w - 1) / w;
  const int per_sm = smem <= 48 * 1024 ? 4 : smem <= 100 * 1024 ? 2 : 1;
  const unsigned grid = (unsigned)std::min<uint64_t>(x_hi - x_lo, (uint64_t)X.sm_count * per_sm);
  D3G_LAUNCH(X, dense_counters_kernel, grid, kCntThreads, smem, r.row_ptr.p, r.col.p, x_lo, x_hi,
             zptr, zcol, z_rows, dsel, dsel_n, dthr.p, (uint64_t)thr.size(), w, n_blocks,
             (uint32_t)words, next.p, dc.p);
  DenseCounters h{};
  X.to_host(&h, dc.p, 1);
  out.wide += h.wide;
  out.probe += h.probe;
  out.blocks += h.blocks;
  out.probes += h.probes;
  out.bitmaps += h.bitmaps;
}

// SpaStats::spa_allocations / spa_entries (P/src/sparsebmm.cpp:17-21,
// :79-104): one stamp array of |Z| entries per chunk run_chunked executes.
void spa_counters(uint64_t x_rows, uint64_t z_card, int threads, d3g_report* rep) {
  uint64_t chunks = 0;
  if (x_rows > 0) chunks = (threads <= 1 || x_rows <= 1) ? 1 : std::min<uint64_t>(threads, x_rows);
  rep->spa_allocations = chunks;
  rep->spa_entries = chunks ? z_card : 0;
}

// ---------------------------------------------------------------------------
// Input columns in HBM as u64. d3g_table::value_bytes == 4: the columns are
// uint32_t (the int32 workloads), copied at 4 bytes per value and widened on
// the GPU; u64 host columns are copied as they are.
int table_value_bytes(const d3g_table* t) {
  if (t->value_bytes == 0 || t->value_bytes == 8) return 8;
  if (t->value_bytes == 4) return 4;
  throw d3g::ConfigError("d3g_table.value_bytes must be 0, 4 or 8");
}

void resident_columns(Ctx& X, const d3g_table* t, DBuf<uint64_t>& lb, DBuf<uint64_t>& rb,
                      const uint64_t*& l, const uint64_t*& r, d3g_report* rep) {
  using namespace d3g;
  const uint64_t n = t->n;
  if (table_value_bytes(t) == 8) {
    if (t->on_device) return;
    lb = X.alloc<uint64_t>(n);
    rb = X.alloc<uint64_t>(n);
    X.to_device(lb.p, t->left, n);
    X.to_device(rb.p, t->right, n);
    l = lb.p;
    r = rb.p;
    rep->h2d_bytes += n * 16;
    return;
  }
  lb = X.alloc<uint64_t>(n);
  rb = X.alloc<uint64_t>(n);
  const uint32_t* src[2] = {reinterpret_cast<const uint32_t*>(t->left),
                            reinterpret_cast<const uint32_t*>(t->right)};
  uint64_t* dst[2] = {lb.p, rb.p};
  DBuf<uint32_t> stage;
  if (!t->on_device && n) stage = X.alloc<uint32_t>(n);
  for (int c = 0; c < 2; ++c) {
    const uint32_t* in = src[c];
    if (!t->on_device && n) {
      X.to_device(stage.p, src[c], n);
      in = stage.p;
      rep->h2d_bytes += n * 4;
    }
    if (n) D3G_LAUNCH(X, widen_u32_kernel, grid_for((n + 3) / 4, 256), 256, 0, in, n, dst[c]);
  }
  l = lb.p;
  r = rb.p;
}

// ---------------------------------------------------------------------------
// The pipeline.
void join_project_impl(Ctx& X, const d3g_table* r, const d3g_table* s, const d3g_consts* c,
                       const d3g_opts* o, d3g_report* rep, d3g_pairs* pairs,
                       d3g::Exchange* E = nullptr) {
  using namespace d3g;
  // sharded job: r is this rank's x-shard of R (exchange.cuh)
  const bool dist = E && E->active();
  if (o->threads < 1) throw ConfigError("threads must be >= 1");
  if (c->w == 0 || c->w % 64 != 0) throw ConfigError("block width W must be a positive multiple of 64");
  const int shard_count = o->shard_count < 1 ? 1 : o->shard_count;
  const int shard_index = o->shard_index;
  if (shard_index < 0 || shard_index >= shard_count) throw ConfigError("bad shard index");
  std::memset(rep, 0, sizeof(*rep));
  X.launches = 0;
  X.syncs = 0;
  X.d2h_bytes = 0;
  X.budget = o->memory_budget_bytes ? o->memory_budget_bytes : (3ull << 30);
  if (E) E->reset_stats();
  uint64_t base_live = X.live_bytes;
  X.peak_bytes = X.live_bytes;
  Timer T(X);
  T.mark();  // 0

  uint64_t nr_job = r->n;  // |R| of the whole job
  if (dist) ex_allreduce_host(X, *E, &nr_job, 1, D3G_EX_SUM_U64);
  if (dist && s->n > nr_job)
    throw ConfigError("a sharded join_project needs |R| >= |S| (shard the larger table)");
  const bool swapped = s->n > nr_job;  // engine_will_swap (engine.cpp:341-343)
  const d3g_table* R = swapped ? s : r;
  const d3g_table* S = swapped ? r : s;
  rep->swapped = swapped;
  rep->r_rows = swapped ? R->n : nr_job;
  rep->s_rows = S->n;
  const uint64_t NR = R->n, NS = S->n;
  const bool materialize = pairs != nullptr && !o->count_only;
  rep->materialized = materialize;

  // 1. inputs resident in HBM (u64 columns; 4-byte columns are copied as
  // such and widened on the device)
  DBuf<uint64_t> hb[4];
  const uint64_t* Rl = R->left;
  const uint64_t* Rr = R->right;
  const uint64_t* Sl = S->left;
  const uint64_t* Sr = S->right;
  resident_columns(X, R, hb[0], hb[1], Rl, Rr, rep);
  if (!S->on_device && S->left == R->left && S->right == R->right && NS == NR &&
      S->value_bytes == R->value_bytes) {
    Sl = Rl;  // the same host relation passed twice (a self-join): copied once
    Sr = Rr;
  } else {
    resident_columns(X, S, hb[2], hb[3], Sl, Sr, rep);
  }
  T.mark();  // 1

  // 2. f1 gate (engine.cpp:368-384): auto takes the classical join iff f1 > 0.
  // The estimate and the self-join test are launched now and read back with
  // the column statistics (one round trip for the three).
  // (sharded: no rank holds R's strided samples; f1 takes the exact bag join
  // size, summed over the ranks after the mapping)
  EstimateJob est;
  if (!dist) estimate_out_j_start(X, Rr, NR, Sr, NS, est);
  uint64_t bag_job = 0;
  IdentityJob ident;
  const bool try_selfjoin = !dist && std::getenv("D3G_NO_SELFJOIN") == nullptr;
  if (try_selfjoin) tables_identical_start(X, Rl, Rr, Sl, Sr, NR, NS, ident);
  const char* cls_env = std::getenv("D3G_CLASSICAL");
  const bool global_classical = !dist && cls_env && std::strcmp(cls_env, "global") == 0;
  bool classical = false;
  auto decide_f1 = [&] {
    rep->out_j_estimate = dist ? bag_job : est.value(X);
    rep->f1 = d3g_f1(dist ? nr_job : NR, NS, rep->out_j_estimate, c);
    rep->f1_gate_classical = (o->force == D3G_AUTO && rep->f1 > 0) ? 1 : 0;
    classical = o->force == D3G_CLASSICAL || rep->f1_gate_classical;
    const char* strat = classical                    ? "classical"
                        : o->force == D3G_SPARSE_ONLY ? "sparse"
                        : o->force == D3G_DENSE_ONLY  ? "dense"
                                                      : "hybrid";
    std::snprintf(rep->strategy, sizeof(rep->strategy), "%s", strat);
  };
  if (global_classical) decide_f1();
  T.mark();  // 2
  // On the GPU the classical branch runs x-partitioned: the y-grouped hash
  // join is the sparse probe of the pipeline below with every z sparse, and
  // the dedup is per x in shared memory instead of one global pair set. The
  // global-set hash_join_dedup stays available (D3G_CLASSICAL=global).
  if (global_classical && classical) {
    classical_impl(X, Rl, Rr, NR, Sl, Sr, NS, swapped, o->checksum ? kModeChecksum : kModeCount,
                   materialize, rep, pairs);
    T.mark();  // 3
    X.sync();
    rep->ms_h2d = T.ms(0, 1);
    rep->ms_estimate = T.ms(1, 2);
    rep->ms_classical = T.ms(2, 3);
    rep->ms_total = T.ms(0, 3);
    rep->peak_bytes = X.peak_bytes - base_live;
    rep->gpu_launches = X.launches;
    rep->d2h_bytes += X.d2h_bytes;
    X.reserve_for(X.peak_bytes);
    return;
  }

  // 3-4. natural keys + mapping
  Mapped M;
  map_inputs(X, Rl, Rr, NR, Sl, Sr, NS, o, rep, /*want_kept=*/false, M, E, nr_job);
  if (dist) {
    // the job's bag join size sum_y |R_y| |S_y| (estimate_out_j_raw's exact
    // case, P/src/costmodel.cpp:375-409): per-y raw R counts summed over ranks
    const uint64_t yc = M.y_card;
    DBuf<uint32_t> cr = X.zeros<uint32_t>(yc), cs2 = X.zeros<uint32_t>(yc);
    // (hot y privatised in shared memory: Zipf-skewed y would serialise on
    // plain global atomics)
    if (M.kept)
      D3G_LAUNCH(X, value_hist_kernel, grid_for(M.kept, 512, X.sm_count * 2), 512, 0, M.r_y,
                 M.kept, cr.p, (uint32_t)yc);
    // (every rank holds all of S: each counts a 1/N slice, summed with R's)
    const uint64_t s0 = NS * (uint64_t)E->rank / (uint64_t)E->nranks,
                   s1 = NS * (uint64_t)(E->rank + 1) / (uint64_t)E->nranks;
    if (s1 > s0)
      D3G_LAUNCH(X, value_hist_kernel, grid_for(s1 - s0, 512, X.sm_count * 2), 512, 0,
                 M.s_y + s0, s1 - s0, cs2.p, (uint32_t)yc);
    ex_allreduce(X, *E, cr.p, yc, D3G_EX_SUM_U32);
    ex_allreduce(X, *E, cs2.p, yc, D3G_EX_SUM_U32);
    const unsigned gb = grid_for(yc, 1024, 296);
    DBuf<unsigned long long> parts = X.zeros<unsigned long long>(2ull * gb);
    if (yc) D3G_LAUNCH(X, outj_kernel, gb, 1024, 0, cr.p, cs2.p, yc, parts.p);
    std::vector<unsigned long long> hp(2ull * gb);
    X.to_host(hp.data(), parts.p, 2ull * gb);
    unsigned __int128 acc = 0;
    for (unsigned i = 0; i < gb; ++i) acc += ((unsigned __int128)hp[2 * i + 1] << 64) | hp[2 * i];
    bag_job = acc > (unsigned __int128)~0ull ? ~0ull : (uint64_t)acc;
  }
  if (!global_classical) decide_f1();  // delivered by map_inputs' first round trip
  if (!classical) M.check_natural();
  const bool self_join = try_selfjoin && ident.value(X);
  const uint64_t kept = M.kept, x_card = M.x_card, y_card = M.y_card, z_card = M.z_card;
  const uint64_t x_card_job = M.x_card_job;
  DictBundle& D = M.D;
  if (classical && dist) {
    rep->intermediate_pairs = bag_job;
  } else if (classical) {  // intermediate_pairs = bag join size, duplicates included
    DBuf<uint32_t> cnt = X.zeros<uint32_t>(y_card);
    if (NS) D3G_LAUNCH(X, group_hist_kernel, grid_for(NS, 256), 256, 0, M.s_y, NS, cnt.p);
    DBuf<unsigned long long> bag = X.zeros<unsigned long long>(1);
    if (kept)
      D3G_LAUNCH(X, bag_from_counts_kernel, grid_for(kept, 256), 256, 0, M.r_y, kept, cnt.p,
                 bag.p);
    rep->intermediate_pairs = X.scalar(bag.p);
  }
  T.mark();  // 3

  // 5. CSR (build_csr, relation.cpp:206-258). A self-join (S identical to R)
  // maps both sides identically, so S-by-z is R-by-x: built once.
  // A sharded job splits the S side by z (the z-split, zsplit.cuh): rank q
  // builds S-by-z for the z codes [z_lo, z_hi) only; the statistics are
  // all-reduced and the dense-row products gathered (run_dense_hot). It falls
  // back to the whole S-by-z when the sparse side needs the SparseBMM tiers
  // or a layout of its own (decided after the f2 split).
  DeviceCsr rx, sz_csr;
  build_csr_device(X, M.r_x, M.r_y, kept, x_card, y_card, rx);
  const bool same_csr = self_join && kept == NR && x_card == z_card;
  const bool zsplit_try = dist && !classical && !o->collect_counters &&
                          std::getenv("D3G_NO_ZSPLIT") == nullptr &&
                          std::getenv("D3G_HOT") == nullptr && std::getenv("D3G_COLD") == nullptr &&
                          std::getenv("D3G_DENSE") == nullptr && z_card < (1ull << 31);
  uint64_t z_lo = 0, z_hi = z_card;
  if (zsplit_try) {
    z_lo = z_card * (uint64_t)E->rank / (uint64_t)E->nranks;
    z_hi = z_card * (uint64_t)(E->rank + 1) / (uint64_t)E->nranks;
    DBuf<uint32_t> zs_z = X.alloc<uint32_t>(NS), zs_y = X.alloc<uint32_t>(NS);
    DBuf<unsigned long long> cur = X.zeros<unsigned long long>(1);
    if (NS)
      D3G_LAUNCH(X, zrange_compact_kernel, grid_for(NS, kZcThreads * kZcPer, X.sm_count * 8), kZcThreads, 0, M.s_z,
                 M.s_y, NS, (uint32_t)z_lo, (uint32_t)z_hi, zs_z.p, zs_y.p, cur.p);
    const uint64_t n_loc = X.scalar(cur.p);
    build_csr_device(X, zs_z.p, zs_y.p, n_loc, z_hi - z_lo, y_card, sz_csr);
  } else if (same_csr) {
    view_csr(rx, sz_csr);  // declared after rx: released first
  } else {
    build_csr_device(X, M.s_z, M.s_y, NS, z_card, y_card, sz_csr);
  }
  if (!zsplit_try) M.release_codes();  // (z-split: kept for the fallback)
  rep->r_nnz = rx.nnz;
  rep->s_nnz = sz_csr.nnz;
  if (dist) ex_allreduce_host(X, *E, &rep->r_nnz, 1, D3G_EX_SUM_U64);
  if (zsplit_try) ex_allreduce_host(X, *E, &rep->s_nnz, 1, D3G_EX_SUM_U64);
  T.mark();  // 4

  // 6. degree statistics (compute_degree_stats, costmodel.cpp:425-438)
  DegreeStats G;
  degree_stats(X, rx, sz_csr, y_card, rep, G, same_csr, E, x_card_job, zsplit_try);
  const uint64_t max_mx = G.max_mx, x_live = G.x_live, max_mz = G.max_mz;
  const std::vector<uint64_t>& hmx = G.hmx;
  DBuf<uint32_t>& dR = G.dR;
  T.mark();  // 5

  // 7. f2 decisions per degree value (policy.cpp), then the partition
  const int pforce = (classical || o->force == D3G_SPARSE_ONLY) ? D3G_SPARSE_ONLY
                     : o->force == D3G_DENSE_ONLY ? D3G_DENSE_ONLY
                                                  : D3G_HYBRID;
  Split P;
  f2_split(X, sz_csr, G, x_card_job, y_card, c, pforce, rep, P, nullptr, nullptr,
           /*flags=*/false, z_card);
  const uint64_t n_dense = P.n_dense, n_sparse = P.n_sparse;
  rep->sparse_nnz = P.sparse_nnz;  // known on the host (m_z histogram)
  // optional x-code restriction of the kernels (opts x_code_lo/hi)
  const uint64_t xa = o->x_code_hi ? std::min<uint64_t>(o->x_code_lo, x_card) : 0;
  const uint64_t xb = o->x_code_hi ? std::min<uint64_t>(o->x_code_hi, x_card) : x_card;
  // Heavy sparse side (OUT_J,sparse > 4096 per live x): answer it with the
  // same hot bit-sliced + cold residual engine instead of the SparseBMM
  // tiers. Without a dense side (cfg4: 9.7e10 candidates over > 8192 sparse
  // z) it gets its own layout; next to a dense side (cfg2: 1.25e9 candidates
  // over 3,406 sparse z) the sparse rows are FOLDED into the dense layout and
  // their pairs counted apart, so one pass answers both and pairs_sparse /
  // pairs_dense stay the reference's split. Either way the result is exactly
  // the sparse kernel's output, computed faster. OUT_J,sparse
  // (SpaStats::inner_count) comes from the per-degree join sizes.
  const uint64_t outj_sp = P.outj_sparse;
  const uint64_t x_live_job = dist ? G.x_live_job : x_live;
  const bool heavy_sparse = std::getenv("D3G_SPARSE_TIERS") == nullptr && x_live_job > 0 &&
                            n_sparse > 0 && outj_sp > 4096ull * x_live_job;
  // folded rows need the record-based hot kernels and the cold kernels
  const char* hot_env = std::getenv("D3G_HOT");
  const std::string hot_sel = hot_env ? hot_env : "";
  const bool default_engine = (hot_sel.empty() || hot_sel == "jt" || hot_sel == "jttrie" ||
                               hot_sel == "tab" || hot_sel == "rec") &&
                              std::getenv("D3G_COLD") == nullptr &&
                              std::getenv("D3G_DENSE") == nullptr;
  const bool fold = heavy_sparse && n_dense > 0 && default_engine &&
                    std::getenv("D3G_NO_FOLD") == nullptr;
  const bool sparse_hot = heavy_sparse && !fold && n_sparse > 8192;
  const bool tiers = !fold && !sparse_hot;  // the SparseBMM tiers answer the sparse side
  // the z-split holds when the dense layout (with any folded sparse rows) is
  // all the S side there is; else every rank builds the whole S-by-z now
  const bool zsplit = zsplit_try && n_dense > 0 && (fold || n_sparse == 0) &&
                      G.x_live_job > 0;
  if (zsplit_try && !zsplit) {
    DeviceCsr full;
    build_csr_device(X, M.s_z, M.s_y, NS, z_card, y_card, full);
    sz_csr = std::move(full);
  }
  M.release_codes();
  rep->zsplit = zsplit ? 1 : 0;
  // the sparse z as a compact id list, and the y-major CSR over those ids
  // (partition.cpp:59-78), only when the tiers run
  DBuf<uint32_t> sparse_ids;
  DBuf<uint64_t> sp_ptr = X.alloc<uint64_t>(y_card + 1);
  DBuf<uint32_t> sp_col;
  if (tiers) {
    sparse_ids = X.alloc<uint32_t>(n_sparse);
    if (n_sparse) {
      DBuf<uint32_t> iss = X.alloc<uint32_t>(z_card), isd = X.alloc<uint32_t>(z_card);
      D3G_LAUNCH(X, dense_flag_kernel, grid_for(z_card, 256), 256, 0, sz_csr.row_ptr.p, z_card,
                 P.dtable.p, G.max_mz + 1, isd.p, iss.p);
      DBuf<uint64_t> psp = X.alloc<uint64_t>(z_card + 1);
      exclusive_scan<uint32_t>(X, iss.p, z_card, psp.p);
      D3G_LAUNCH(X, index_compact_kernel, grid_for(z_card, 256), 256, 0, iss.p, psp.p, z_card,
                 sparse_ids.p);
    }
    DBuf<uint32_t> sp_cnt = X.zeros<uint32_t>(y_card);
    if (n_sparse)
      D3G_LAUNCH(X, sparse_y_count_kernel, grid_for(n_sparse * 8, 256), 256, 0, sz_csr.row_ptr.p,
                 sz_csr.col.p, sparse_ids.p, n_sparse, sp_cnt.p);
    exclusive_scan<uint32_t>(X, sp_cnt.p, y_card, sp_ptr.p);
    sp_col = X.alloc<uint32_t>(rep->sparse_nnz);
    if (n_sparse)
      D3G_LAUNCH(X, sparse_y_scatter_kernel, grid_for(n_sparse * 8, 256), 256, 0,
                 sz_csr.row_ptr.p, sz_csr.col.p, sparse_ids.p, n_sparse, sp_ptr.p, sp_cnt.p,
                 sp_col.p);
  }
  // dense side (plus the folded sparse rows): rows selected by m_z through
  // the f2 table and ordered by degree in one counting scatter
  DenseLayout L;
  DBuf<uint8_t> row_sp;
  // (z-split: this rank's z rows, counted from z_lo; every rank builds its
  // part, live x or not: the gathers in run_dense_hot take all of them)
  if (n_dense > 0 && (zsplit || x_live > 0)) {
    RowSel sel{zsplit ? &G.hmz_local : &G.hmz, P.dtable.p, &P.table, fold ? 0 : 1,
               fold ? &row_sp : nullptr};
    build_dense_layout(X, rx, max_mx, hmx, sz_csr.row_ptr.p, sz_csr.col.p, nullptr, 0, max_mz,
                       nullptr, y_card, dR.p, L, xa, xb, ~0ull, &sel, sz_csr.n_rows,
                       shard_count > 1, x_card_job, zsplit ? z_lo : 0, zsplit);
  }
  // z-split: the global dense rows are the ranks' blocks in rank order
  std::vector<uint64_t> rows_per_rank;
  uint64_t row_lo = 0, rows_job = 0;
  if (zsplit) {
    rows_per_rank.assign(E->nranks, 0);
    uint64_t mine = L.n_dense;
    ex_allgather(X, *E, &mine, rows_per_rank.data(), 8);
    uint64_t tot = 0;
    for (int q = 0; q < E->nranks; ++q) {
      if (q == E->rank) row_lo = tot;
      tot += rows_per_rank[q];
    }
    // the layout's rows: the dense z, plus the sparse z folded into it
    const uint64_t want = fold ? n_dense + n_sparse : n_dense;
    if (tot != want) throw CudaError("z-split: layout rows " + std::to_string(tot) +
                                     " != the f2 split's " + std::to_string(want));
    rows_job = tot;
  }
  DenseLayout Ls;
  if (sparse_hot && x_live > 0) {
    RowSel sel{&G.hmz, P.dtable.p, &P.table, 2, nullptr};
    build_dense_layout(X, rx, max_mx, hmx, sz_csr.row_ptr.p, sz_csr.col.p, nullptr, 0, max_mz,
                       nullptr, y_card, dR.p, Ls, xa, xb, ~0ull, &sel, z_card, shard_count > 1,
                       x_card_job);
  }
  T.mark();  // 6

  // 8. kernels
  Decode dec{rev_or_null(D.x), rev_or_null(D.z), swapped ? 1 : 0};
  const int mode = o->checksum ? kModeChecksum : kModeCount;
  Emit no_emit{nullptr, nullptr, nullptr, 0};
  // x shard (x code range for SparseBMM, position range for DenseEC)
  uint64_t x_lo = xa + (xb - xa) * shard_index / shard_count,
           x_hi = xa + (xb - xa) * (shard_index + 1) / shard_count;
  SparseInputs si{rx.row_ptr.p, rx.col.p, x_card, sp_ptr.p, sp_col.p, sparse_ids.p, n_sparse,
                  y_card, x_lo, x_hi};
  // reference-equivalent work counters over this call's x codes (SpaStats,
  // DenseEcStats; counters.cuh)
  if (!classical) {
    spa_counters(x_card_job, z_card, o->threads, rep);
    DenseCounters dc{};
    const std::vector<uint32_t> thr = mode_thresholds(max_mx, y_card, c, o->dense_mode);
    if (o->collect_counters) {
      dense_counters_device(X, rx, x_lo, x_hi, sz_csr.row_ptr.p, sz_csr.col.p, z_card,
                            P.dtable.p, max_mz + 1, thr, c->w, y_card, dc);
    } else if (n_dense > 0 && x_hi > x_lo) {
      std::vector<uint64_t> hd(max_mz + 1, 0);
      for (uint64_t m = 1; m <= max_mz; ++m) hd[m] = P.table[m] ? G.hmz[m] : 0;
      std::vector<uint64_t> hx_range;
      const std::vector<uint64_t>* hx = &hmx;
      if (x_lo != 0 || x_hi != x_card) {  // the m_x histogram of this call's x range
        DBuf<unsigned long long> h = X.zeros<unsigned long long>(max_mx + 1);
        D3G_LAUNCH(X, degree_hist_kernel, grid_for(x_hi - x_lo, 256), 256, 0,
                   rx.row_ptr.p + x_lo, x_hi - x_lo, max_mx + 1, h.p);
        hx_range.resize(max_mx + 1);
        X.to_host(reinterpret_cast<unsigned long long*>(hx_range.data()), h.p, max_mx + 1);
        hx = &hx_range;
      }
      encounter_counts(*hx, hd, thr, dc);
    }
    rep->dense_wide_encounters = dc.wide;
    rep->dense_probe_encounters = dc.probe;
    rep->dense_blocks_checked = dc.blocks;
    rep->dense_probes_done = dc.probes;
    rep->dense_row_bitmaps_built = dc.bitmaps;
  }
  // Materialized calls emit in ONE kernel pass when the join size (an upper
  // bound on the distinct pairs) fits the memory budget: no counting pass
  // first. Otherwise (or with the fingerprint requested) count, then emit.
  bool direct = false;
  uint64_t direct_cap = 0;
  if (materialize && !o->checksum && std::getenv("D3G_COUNT_FIRST") == nullptr) {
    const uint64_t bound = std::min<uint64_t>(rep->out_j, x_live * (n_dense + n_sparse));
    const uint64_t need = bound * 48;  // emit + sort + decode buffers
    if (bound < (1ull << 32) && (X.budget == 0 || X.live_bytes + need <= X.budget)) {
      direct = true;
      direct_cap = bound;
    }
  }
  if (zsplit && materialize) {
    // the ranks run the same kernel passes (one emitting pass, or count then
    // emit): the z-split's gathers pair up only if they agree
    uint64_t no_direct = direct ? 0 : 1;
    ex_allreduce_host(X, *E, &no_direct, 1, D3G_EX_MAX_U64);
    direct = no_direct == 0;
  }
  DBuf<uint32_t> dex, dez;
  DBuf<unsigned long long> dcur;
  Emit em_run = no_emit;
  int kmode = mode;
  if (direct) {
    dex = X.alloc<uint32_t>(direct_cap);
    dez = X.alloc<uint32_t>(direct_cap);
    dcur = X.zeros<unsigned long long>(1);
    em_run = Emit{dex.p, dez.p, dcur.p, direct_cap};
    kmode = kModeEmit;
  }
  KernelOut ks, kd;
  const uint64_t s_lo = Ls.n_live * shard_index / shard_count,
                 s_hi = Ls.n_live * (shard_index + 1) / shard_count;
  DenseInputs dsi{Ls.xorder.p, Ls.n_live, rx.row_ptr.p, rx.col.p, Ls.y_rank.p, y_card,
                  Ls.dl_ptr.p, Ls.dl_col.p, Ls.dl_z.p, Ls.n_dense, Ls.max_group_nnz, s_lo, s_hi,
                  Ls.y_of_rank.p, dR.p, x_card, x_lo, x_hi, Ls.dnnz, nullptr,
                  Ls.n_dense == sz_csr.live_rows ? G.dS.p : nullptr};
  if (sparse_hot)
    run_dense_hot(X, dsi, dec, kmode, em_run, ks);
  else if (!fold)
    run_sparse(X, si, dec, kmode, em_run, ks);
  T.mark();  // 7
  uint64_t pos_lo = L.n_live * shard_index / shard_count,
           pos_hi = L.n_live * (shard_index + 1) / shard_count;
  const uint64_t live_z = zsplit ? G.z_live_job : sz_csr.live_rows;
  DenseInputs di{L.xorder.p, L.n_live, rx.row_ptr.p, rx.col.p, L.y_rank.p, y_card, L.dl_ptr.p,
                 L.dl_col.p, L.dl_z.p, zsplit ? rows_job : L.n_dense, L.max_group_nnz, pos_lo,
                 pos_hi, L.y_of_rank.p, dR.p, x_card, x_lo, x_hi, L.dnnz, row_sp.p,
                 (zsplit ? rows_job : L.n_dense) == live_z ? G.dS.p : nullptr};
  if (zsplit) {
    di.zx = E;
    di.row_lo = row_lo;
    di.n_dense_local = L.n_dense;
    di.rows_per_rank = rows_per_rank;
    di.x_card_job = x_card_job;
    di.n_live_job = G.x_live_job;
  }
  run_dense(X, di, dec, kmode, em_run, kd);
  T.mark();  // 8
  if (fold) {  // the folded sparse rows' pairs, counted apart inside the engine
    ks.count = kd.count_sp;
    kd.count -= kd.count_sp;
  }
  rep->pairs_sparse = ks.count;
  rep->pairs_dense = kd.count;
  rep->ms_dense_hot = ks.ms_hot + kd.ms_hot;
  rep->hot_lds_bytes = ks.hot_lds_bytes + kd.hot_lds_bytes;
  rep->hot_lds_bytes_unshared = ks.hot_lds_bytes_unshared + kd.hot_lds_bytes_unshared;
  rep->hot_direct_pairs = ks.split_direct_pairs + kd.split_direct_pairs;
  rep->ms_dense_cold = ks.ms_cold + kd.ms_cold;
  rep->cold_bytes = ks.cold_bytes + kd.cold_bytes;
  rep->cold_candidates = ks.cold_candidates + kd.cold_candidates;
  rep->cold_tail_checks = ks.cold_tail_checks + kd.cold_tail_checks;
  rep->spa_inner_count = outj_sp;
  rep->out_p = ks.count + kd.count;
  rep->checksum_sum = ks.sum + kd.sum;
  rep->checksum_xor = ks.xr ^ kd.xr;
  rep->rank_out_p = rep->out_p;
  rep->nranks = dist ? E->nranks : 1;
  rep->rank = dist ? E->rank : 0;
  if (dist) {
    // the job's totals: each rank's tally record, gathered and folded
    // (the fingerprint's xor has no NCCL reduction)
    constexpr int kF = 15;
    uint64_t mine[kF] = {rep->out_p, rep->pairs_sparse, rep->pairs_dense, rep->checksum_sum,
                         rep->checksum_xor, rep->hot_direct_pairs, rep->cold_bytes,
                         rep->hot_lds_bytes, rep->dense_wide_encounters,
                         rep->dense_probe_encounters, rep->dense_blocks_checked,
                         rep->dense_probes_done, rep->dense_row_bitmaps_built,
                         rep->cold_candidates, rep->cold_tail_checks};
    std::vector<uint64_t> all((size_t)kF * E->nranks);
    ex_allgather(X, *E, mine, all.data(), sizeof(mine));
    uint64_t tot[kF] = {0};
    for (int q = 0; q < E->nranks; ++q)
      for (int f = 0; f < kF; ++f)
        tot[f] = f == 4 ? (tot[f] ^ all[(size_t)q * kF + f]) : tot[f] + all[(size_t)q * kF + f];
    rep->out_p = tot[0];
    rep->pairs_sparse = tot[1];
    rep->pairs_dense = tot[2];
    rep->checksum_sum = tot[3];
    rep->checksum_xor = tot[4];
    rep->hot_direct_pairs = tot[5];
    rep->cold_bytes = tot[6];
    rep->hot_lds_bytes = tot[7];
    rep->dense_wide_encounters = tot[8];
    rep->dense_probe_encounters = tot[9];
    rep->dense_blocks_checked = tot[10];
    rep->dense_probes_done = tot[11];
    rep->dense_row_bitmaps_built = tot[12];
    rep->cold_candidates = tot[13];
    rep->cold_tail_checks = tot[14];
  }

  // 9. materialization (decode, engine.cpp:502-529)
  if (materialize && direct) {
    const uint64_t emitted = X.scalar(dcur.p);
    if (emitted != rep->rank_out_p)
      throw CudaError("materialize: emitted " + std::to_string(emitted) + " pairs, counted " +
                      std::to_string(rep->rank_out_p));
    if (pairs->x && pairs->cap < emitted)
      throw ResourceError("output buffer holds " + std::to_string(pairs->cap) + " pairs, need " +
                          std::to_string(emitted));
    finish_pairs(X, dex, dez, emitted, rev_or_null(D.x), rev_or_null(D.z), swapped, pairs, rep,
                 x_card, z_card);
  } else if (materialize)
    materialize_pairs(X, rep->rank_out_p, [&](Emit em) {
      KernelOut tmp;
      if (sparse_hot)
        run_dense_hot(X, dsi, dec, kModeEmit, em, tmp);
      else if (!fold)
        run_sparse(X, si, dec, kModeEmit, em, tmp);
      run_dense(X, di, dec, kModeEmit, em, tmp);
    }, rev_or_null(D.x), rev_or_null(D.z), swapped, pairs, rep, x_card, z_card);
  T.mark();  // 9
  X.sync();
  rep->ms_h2d = T.ms(0, 1);
  rep->ms_estimate = T.ms(1, 2);
  rep->ms_map = T.ms(2, 3);
  rep->ms_csr = T.ms(3, 4);
  rep->ms_stats = T.ms(4, 5);
  rep->ms_partition = T.ms(5, 6);
  rep->ms_sparse = T.ms(6, 7);
  rep->ms_dense = T.ms(7, 8);
  rep->ms_decode = T.ms(8, 9);
  rep->ms_total = T.ms(0, 9);
  if (classical) {
    // hash_join_dedup's report (engine.cpp:386-395): no mapping/partition
    // fields; the x-partitioned internals are kept only in the phase times
    rep->pairs_classical = rep->out_p;
    rep->ms_classical = T.ms(2, 9);
    rep->dropped_r = rep->x_card = rep->y_card = rep->z_card = 0;
    rep->sparse_z = rep->dense_z = rep->f2_evaluations = rep->panel_bytes = 0;
    rep->pairs_sparse = rep->pairs_dense = rep->r_nnz = rep->s_nnz = rep->out_j = 0;
    rep->spa_inner_count = rep->x_live = rep->sparse_nnz = 0;
    rep->natural_x = rep->natural_y = rep->natural_z = 0;
  }
  rep->peak_bytes = X.peak_bytes - base_live;
  rep->gpu_launches = X.launches;
  rep->d2h_bytes += X.d2h_bytes;
  if (E) {
    rep->exchange_calls = E->calls;
    rep->exchange_bus_bytes = E->bus_bytes;
    rep->ms_exchange_host = E->host_ms;
  }
  if (std::getenv("D3G_TRACE"))
    std::fprintf(stderr, "[join_project] %llu launches, %llu host round trips\n",
                 (unsigned long long)X.launches, (unsigned long long)X.syncs);
  X.reserve_for(X.peak_bytes);
}

// ---------------------------------------------------------------------------
// join_aggregate_both (engine.cpp:537-722); kernels and the parity argument in
// aggregate.cuh.
// Stable grouping of rows by a u32 code: permutation (input order within a
// code) and row_ptr[n_rows + 1].
void stable_group(Ctx& X, const uint32_t* code, uint64_t n, uint64_t n_rows, DBuf<uint32_t>& perm,
                  DBuf<uint64_t>& row_ptr) {
  using namespace d3g;
  DBuf<uint64_t> key = X.alloc<uint64_t>(n);
  perm = X.alloc<uint32_t>(n);
  if (n) D3G_LAUNCH(X, code_key_kernel, grid_for(n, 256), 256, 0, code, n, key.p, perm.p);
  radix_sort(X, key.p, perm.p, n, bits_for(n_rows ? n_rows - 1 : 0), false);
  DBuf<uint32_t> cnt = X.zeros<uint32_t>(n_rows);
  if (n) D3G_LAUNCH(X, count_codes_kernel, grid_for(n, 256), 256, 0, code, n, cnt.p);
  row_ptr = X.alloc<uint64_t>(n_rows + 1);
  exclusive_scan<uint32_t>(X, cnt.p, n_rows, row_ptr.p);
}

void join_aggregate_impl(Ctx& X, const d3g_valued_table* r, const d3g_valued_table* s,
                         int combine, int agg, const d3g_consts* c, const d3g_opts* o,
                         d3g_report* rep, d3g_agg_pairs* out) {
  if (table_value_bytes(&r->base) != 8 || table_value_bytes(&s->base) != 8)
    throw d3g::ConfigError("join_aggregate takes u64 columns (value_bytes 0 or 8)");
  using namespace d3g;
  if (o->threads < 1) throw ConfigError("threads must be >= 1");
  if (o->force == D3G_CLASSICAL) throw ConfigError("join-aggregate always runs the mapped pipeline");
  if (combine < 0 || combine > 4) throw ConfigError("unknown combine function");
  if (agg < 0 || agg > 4) throw ConfigError("unknown aggregate function");
  if (c->w == 0 || c->w % 64 != 0) throw ConfigError("block width W must be a positive multiple of 64");
  if ((r->base.n && !r->values) || (s->base.n && !s->values))
    throw ConfigError("value column length does not match table length");
  std::memset(rep, 0, sizeof(*rep));
  X.launches = 0;
  X.d2h_bytes = 0;
  X.budget = o->memory_budget_bytes ? o->memory_budget_bytes : (3ull << 30);
  const uint64_t base_live = X.live_bytes;
  X.peak_bytes = X.live_bytes;
  Timer T(X);
  T.mark();  // 0
  std::snprintf(rep->strategy, sizeof(rep->strategy), "hybrid");
  const uint64_t NR = r->base.n, NS = s->base.n;
  rep->r_rows = NR;
  rep->s_rows = NS;
  const bool materialize = out != nullptr && !o->count_only;
  rep->materialized = materialize;

  // inputs and values resident in HBM (caller orientation: no swap)
  DBuf<uint64_t> hb[4];
  DBuf<double> hv[2];
  const uint64_t *Rl = r->base.left, *Rr = r->base.right, *Sl = s->base.left, *Sr = s->base.right;
  const double *Rv = r->values, *Sv = s->values;
  if (!r->base.on_device) {
    hb[0] = X.alloc<uint64_t>(NR);
    hb[1] = X.alloc<uint64_t>(NR);
    hv[0] = X.alloc<double>(NR);
    X.to_device(hb[0].p, Rl, NR);
    X.to_device(hb[1].p, Rr, NR);
    X.to_device(hv[0].p, Rv, NR);
    Rl = hb[0].p;
    Rr = hb[1].p;
    Rv = hv[0].p;
    rep->h2d_bytes += NR * 24;
  }
  if (!s->base.on_device) {
    hb[2] = X.alloc<uint64_t>(NS);
    hb[3] = X.alloc<uint64_t>(NS);
    hv[1] = X.alloc<double>(NS);
    X.to_device(hb[2].p, Sl, NS);
    X.to_device(hb[3].p, Sr, NS);
    X.to_device(hv[1].p, Sv, NS);
    Sl = hb[2].p;
    Sr = hb[3].p;
    Sv = hv[1].p;
    rep->h2d_bytes += NS * 24;
  }
  T.mark();  // 1

  // map_with_fallback; the R values follow the surviving rows (m.r_kept)
  Mapped M;
  map_inputs(X, Rl, Rr, NR, Sl, Sr, NS, o, rep, /*want_kept=*/true, M);
  M.check_natural();
  const uint64_t kept = M.kept, x_card = M.x_card, y_card = M.y_card, z_card = M.z_card;
  T.mark();  // 2

  // collapsed matrices drive the per-z density decision only (engine.cpp:570-577)
  DeviceCsr rx, sz_csr;
  build_csr_device(X, M.r_x, M.r_y, kept, x_card, y_card, rx);
  build_csr_device(X, M.s_z, M.s_y, NS, z_card, y_card, sz_csr);
  rep->r_nnz = rx.nnz;
  rep->s_nnz = sz_csr.nnz;
  DegreeStats G;
  degree_stats(X, rx, sz_csr, y_card, rep, G);
  rep->out_j_estimate = rep->out_j;
  T.mark();  // 3

  const int pforce = o->force == D3G_SPARSE_ONLY ? D3G_SPARSE_ONLY
                     : o->force == D3G_DENSE_ONLY ? D3G_DENSE_ONLY
                                                  : D3G_HYBRID;
  Split P;
  f2_split(X, sz_csr, G, x_card, y_card, c, pforce, rep, P);
  rx = DeviceCsr();
  sz_csr = DeviceCsr();
  // valued CSRs (build_valued_csr, engine.cpp:148-171): duplicates kept,
  // stable, one value per entry
  DBuf<uint32_t> rperm, sperm;
  DBuf<uint64_t> rptr, sptr;
  stable_group(X, M.r_x, kept, x_card, rperm, rptr);
  stable_group(X, M.s_y, NS, y_card, sperm, sptr);
  DBuf<uint32_t> ry = X.alloc<uint32_t>(kept), sz = X.alloc<uint32_t>(NS);
  DBuf<double> rv = X.alloc<double>(kept), sv = X.alloc<double>(NS);
  if (kept) {
    D3G_LAUNCH(X, gather_u32_kernel, grid_for(kept, 256), 256, 0, M.r_y, rperm.p, kept, ry.p);
    D3G_LAUNCH(X, gather_f64_kernel, grid_for(kept, 256), 256, 0, Rv, rperm.p,
               M.r_kept.p ? M.r_kept.p : (const uint32_t*)nullptr, kept, rv.p);
  }
  if (NS) {
    D3G_LAUNCH(X, gather_u32_kernel, grid_for(NS, 256), 256, 0, M.s_z, sperm.p, NS, sz.p);
    D3G_LAUNCH(X, gather_f64_kernel, grid_for(NS, 256), 256, 0, Sv, sperm.p,
               (const uint32_t*)nullptr, NS, sv.p);
  }
  rperm.reset();
  sperm.reset();
  M.release_codes();
  M.r_kept.reset();
  T.mark();  // 4

  // candidates per x, then chunks of x whose candidates fit the buffers
  DBuf<uint64_t> cand = X.alloc<uint64_t>(x_card), coff = X.alloc<uint64_t>(x_card + 1);
  if (x_card)
    D3G_LAUNCH(X, agg_cand_kernel, grid_for(x_card, 256), 256, 0, rptr.p, ry.p, sptr.p, x_card,
               cand.p);
  exclusive_scan<uint64_t>(X, cand.p, x_card, coff.p);
  cand.reset();
  std::vector<uint64_t> hoff(x_card + 1);
  X.to_host(reinterpret_cast<unsigned long long*>(hoff.data()),
            reinterpret_cast<unsigned long long*>(coff.p), x_card + 1);
  rep->intermediate_pairs = hoff[x_card];  // bag join size
  uint64_t max_c = 0;
  for (uint64_t x = 0; x < x_card; ++x) max_c = std::max(max_c, hoff[x + 1] - hoff[x]);
  const uint64_t cap_chunk = std::max<uint64_t>(max_c, 1ull << 25);
  DBuf<uint64_t> key = X.alloc<uint64_t>(std::min(cap_chunk, std::max<uint64_t>(hoff[x_card], 1)));
  const uint64_t kcap = key.n;
  DBuf<double> val = X.alloc<double>(kcap);
  DBuf<uint32_t> perm = X.alloc<uint32_t>(kcap), head = X.alloc<uint32_t>(kcap);
  DBuf<uint64_t> hpos = X.alloc<uint64_t>(kcap + 1);
  DBuf<uint32_t> starts = X.alloc<uint32_t>(kcap);
  DBuf<uint32_t> ox, oz;
  DBuf<double> ov;
  if (materialize) {
    ox = X.alloc<uint32_t>(out->cap);
    oz = X.alloc<uint32_t>(out->cap);
    ov = X.alloc<double>(out->cap);
  }
  DBuf<unsigned long long> dense_pairs = X.zeros<unsigned long long>(1);
  DBuf<unsigned int> too_many = X.zeros<unsigned int>(1);
  uint64_t total = 0;
  for (uint64_t x0 = 0; x0 < x_card;) {
    uint64_t x1 = x0;
    while (x1 < x_card && hoff[x1 + 1] - hoff[x0] <= kcap) ++x1;
    const uint64_t n = hoff[x1] - hoff[x0];
    if (n) {
      D3G_LAUNCH(X, agg_enum_kernel, grid_for((x1 - x0) * 32, 256), 256, 0, x0, x1, coff.p, rptr.p,
                 ry.p, rv.p, sptr.p, sz.p, sv.p, combine, key.p, val.p);
      D3G_LAUNCH(X, iota_kernel, grid_for(n, 256), 256, 0, perm.p, n);
      radix_sort(X, key.p, perm.p, n, 32 + bits_for(x1 - x0 - 1));
      D3G_LAUNCH(X, seg_head_kernel, grid_for(n, 256), 256, 0, key.p, n, head.p);
      exclusive_scan<uint32_t>(X, head.p, n, hpos.p);
      const uint64_t nseg = X.scalar(hpos.p + n);
      D3G_LAUNCH(X, index_compact_kernel, grid_for(n, 256), 256, 0, head.p, hpos.p, n, starts.p);
      if (materialize && total + nseg > out->cap)
        throw ResourceError("output buffer holds " + std::to_string(out->cap) +
                            " aggregate rows, need more");
      D3G_LAUNCH(X, agg_fold_kernel, grid_for(nseg, 256), 256, 0, key.p, perm.p, val.p, starts.p,
                 nseg, n, x0, agg, P.isd.p, materialize ? ox.p + total : nullptr,
                 materialize ? oz.p + total : nullptr, materialize ? ov.p + total : nullptr,
                 dense_pairs.p, too_many.p);
      total += nseg;
    }
    x0 = x1;
  }
  if (X.scalar(too_many.p)) throw ResourceError("count aggregate exceeds exact integer range");
  rep->pairs_dense = X.scalar(dense_pairs.p);
  rep->pairs_sparse = total - rep->pairs_dense;
  rep->out_p = total;
  if (materialize) {
    DBuf<uint64_t> dx, dz;
    uint64_t* px = out->x;
    uint64_t* pz = out->z;
    if (!out->on_device) {
      dx = X.alloc<uint64_t>(total);
      dz = X.alloc<uint64_t>(total);
      px = dx.p;
      pz = dz.p;
    }
    if (total)
      D3G_LAUNCH(X, decode_pairs_kernel, grid_for(total, 256), 256, 0, ox.p, oz.p, total,
                 rev_or_null(M.D.x), rev_or_null(M.D.z), 0, px, pz);
    if (out->on_device) {
      D3G_CUDA(cudaMemcpyAsync(out->values, ov.p, total * 8, cudaMemcpyDeviceToDevice, X.stream));
    } else if (total) {
      X.copy_to_pageable(out->x, dx.p, total * 8);
      X.copy_to_pageable(out->z, dz.p, total * 8);
      X.copy_to_pageable(out->values, ov.p, total * 8);
    }
    out->n = total;
  }
  T.mark();  // 5
  X.sync();
  rep->ms_h2d = T.ms(0, 1);
  rep->ms_map = T.ms(1, 2);
  rep->ms_csr = T.ms(2, 3);
  rep->ms_partition = T.ms(3, 4);
  rep->ms_sparse = T.ms(4, 5);
  rep->ms_total = T.ms(0, 5);
  rep->peak_bytes = X.peak_bytes - base_live;
  rep->gpu_launches = X.launches;
  rep->d2h_bytes += X.d2h_bytes;
  X.reserve_for(X.peak_bytes);
}

}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

const char* d3g_last_error(void) { return g_last_error.c_str(); }

const char* d3g_version(void) {
  return "dim3_b200 sm_100a (hand-written CUDA, bit-sliced DenseEC, bitmap SparseBMM)";
}

void d3g_opts_default(d3g_opts* o) {
  std::memset(o, 0, sizeof(*o));
  o->force = D3G_AUTO;
  o->threads = 1;
  o->memory_budget_bytes = 3ull << 30;
  o->natural_keys_auto = 1;
  o->shard_count = 1;
}

int d3g_ctx_create(int device, d3g_ctx** out) {
  return guarded([&] {
    int n = 0;
    D3G_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw d3g::ConfigError("no such CUDA device");
    D3G_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    D3G_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      throw d3g::ConfigError("dim3_b200 requires an sm_100 (Blackwell) device");
    auto* ctx = new d3g_ctx();
    ctx->c.device = device;
    ctx->c.sm_count = prop.multiProcessorCount;
    ctx->c.smem_optin = prop.sharedMemPerBlockOptin;
    D3G_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    D3G_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = ~0ull;
    D3G_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    *out = ctx;
  });
}

int d3g_nccl_unique_id(void* id128) {
  return guarded([&] {
    ncclUniqueId id;
    D3G_NCCL(d3g::nccl().get_unique_id(&id));
    std::memcpy(id128, &id, sizeof(id));
  });
}

int d3g_ctx_set_nccl(d3g_ctx* ctx, const void* id128, int nranks, int rank) {
  return guarded([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw d3g::ConfigError("bad nranks / rank");
    D3G_CUDA(cudaSetDevice(ctx->c.device));
    if (ctx->ex.comm) {
      d3g::nccl().comm_destroy(ctx->ex.comm);
      ctx->ex.comm = nullptr;
    }
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    D3G_NCCL(d3g::nccl().comm_init_rank(&ctx->ex.comm, nranks, id, rank));
    ctx->ex.nranks = nranks;
    ctx->ex.rank = rank;
    ctx->ex.host_fn = nullptr;
    ctx->ex.host_user = nullptr;
  });
}

int d3g_ctx_set_exchange(d3g_ctx* ctx, int nranks, int rank, d3g_exchange_fn fn, void* user) {
  return guarded([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw d3g::ConfigError("bad nranks / rank");
    if (nranks > 1 && !fn) throw d3g::ConfigError("an exchange over several ranks needs a callback");
    if (ctx->ex.comm) {
      d3g::nccl().comm_destroy(ctx->ex.comm);
      ctx->ex.comm = nullptr;
    }
    ctx->ex.nranks = nranks;
    ctx->ex.rank = rank;
    ctx->ex.host_fn = fn;
    ctx->ex.host_user = user;
  });
}

int d3g_take_pairs(d3g_ctx* ctx, uint64_t* x, uint64_t* z, uint64_t n, int on_device) {
  return guarded([&] {
    d3g::Ctx& X = ctx->c;
    D3G_CUDA(cudaSetDevice(X.device));
    if (n > X.held_n) throw d3g::ConfigError("d3g_take_pairs: only " + std::to_string(X.held_n) +
                                             " pairs are held");
    if (n) {
      if (on_device) {
        D3G_CUDA(cudaMemcpyAsync(x, X.held_x.p, n * 8, cudaMemcpyDeviceToDevice, X.stream));
        D3G_CUDA(cudaMemcpyAsync(z, X.held_z.p, n * 8, cudaMemcpyDeviceToDevice, X.stream));
        X.sync();
      } else {
        X.copy_to_pageable(x, X.held_x.p, n * 8);
        X.copy_to_pageable(z, X.held_z.p, n * 8);
      }
    }
    X.held_x.reset();
    X.held_z.reset();
    X.held_n = 0;
  });
}

void d3g_ctx_destroy(d3g_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  ctx->c.held_x.reset();
  ctx->c.held_z.reset();
  if (ctx->c.pinned) cudaFreeHost(ctx->c.pinned);
  if (ctx->c.defer_host) cudaFreeHost(ctx->c.defer_host);
  ctx->c.release_cache();
  if (ctx->c.zarena) cudaFreeAsync(ctx->c.zarena, ctx->c.stream);
  if (ctx->c.scan_state) cudaFreeAsync(ctx->c.scan_state, ctx->c.stream);
  if (ctx->c.mark_ev) cudaEventDestroy(ctx->c.mark_ev);
  cudaStreamSynchronize(ctx->c.stream);
  for (int b = 0; b < 2; ++b) {
    if (ctx->c.stage[b]) cudaFreeHost(ctx->c.stage[b]);
    if (ctx->c.stage_ev[b]) cudaEventDestroy(ctx->c.stage_ev[b]);
  }
  cudaStreamDestroy(ctx->c.stream);
  // return the memory this context kept reserved in the device pool
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, ctx->c.device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  delete ctx;
}

int d3g_join_project(d3g_ctx* ctx, const d3g_table* r, const d3g_table* s, const d3g_consts* c,
                     const d3g_opts* o, d3g_report* rep, d3g_pairs* pairs) {
  if (!ctx || !r || !s || !c || !o || !rep) {
    g_last_error = "null argument";
    return D3G_CONFIG_ERROR;
  }
  return guarded([&] {
    D3G_CUDA(cudaSetDevice(ctx->c.device));
    ctx->c.begin_call();
    try {
      join_project_impl(ctx->c, r, s, c, o, rep, pairs, &ctx->ex);
    } catch (...) {
      cudaStreamSynchronize(ctx->c.stream);
      ctx->c.budget = 0;  // the memory budget is scoped to one call
      throw;
    }
    ctx->c.budget = 0;
  });
}

int d3g_build_csr(d3g_ctx* ctx, const uint32_t* a, const uint32_t* b, uint64_t n, uint32_t a_card,
                  uint32_t b_card, int major_is_a, d3g_csr* out) {
  return guarded([&] {
    Ctx& X = ctx->c;
    D3G_CUDA(cudaSetDevice(X.device));
    X.begin_call();
    X.budget = 0;
    const uint32_t* maj = major_is_a ? a : b;
    const uint32_t* mnr = major_is_a ? b : a;
    uint64_t n_rows = major_is_a ? a_card : b_card, n_cols = major_is_a ? b_card : a_card;
    DBuf<uint32_t> dm = X.alloc<uint32_t>(n), dn = X.alloc<uint32_t>(n);
    X.to_device(dm.p, maj, n);
    X.to_device(dn.p, mnr, n);
    d3g::DeviceCsr csr;
    d3g::build_csr_device(X, dm.p, dn.p, n, n_rows, n_cols, csr);
    X.to_host(out->row_ptr, csr.row_ptr.p, n_rows + 1);
    X.to_host(out->col, csr.col.p, csr.nnz);
    out->n_rows = (uint32_t)n_rows;
    out->n_cols = (uint32_t)n_cols;
    out->nnz = csr.nnz;
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Kernel-level entry points (parity with sparse_bmm / dense_ec on the
// reference's own CSR / BitmapPanel inputs) and the synthetic generator.
namespace {

__global__ void panel_popc_kernel(const uint64_t* __restrict__ blocks, uint64_t rows,
                                  uint64_t row_words, uint32_t* __restrict__ cnt) {
  for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < rows;
       r += (uint64_t)gridDim.x * (blockDim.x / 32)) {
    uint32_t c = 0;
    for (uint64_t w = d3g::lane_id(); w < row_words; w += 32) c += __popcll(blocks[r * row_words + w]);
    c = d3g::warp_sum(c);
    if (d3g::lane_id() == 0) cnt[r] = c;
  }
}

__global__ void panel_extract_kernel(const uint64_t* __restrict__ blocks, uint64_t rows,
                                     uint64_t row_words, const uint64_t* __restrict__ ptr,
                                     uint32_t* __restrict__ col) {
  // one warp per row; lanes take consecutive words, ranks by warp prefix sum
  for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < rows;
       r += (uint64_t)gridDim.x * (blockDim.x / 32)) {
    uint64_t out = ptr[r];
    for (uint64_t base = 0; base < row_words; base += 32) {
      uint64_t w = base + d3g::lane_id();
      uint64_t bits = w < row_words ? blocks[r * row_words + w] : 0;
      uint32_t c = __popcll(bits), incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (d3g::lane_id() >= (uint32_t)o) incl += u;
      }
      uint64_t o = out + incl - c;
      while (bits) {
        int b = __ffsll((long long)bits) - 1;
        bits &= bits - 1;
        col[o++] = (uint32_t)(w * 64 + b);
      }
      out += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

void sort_and_copy_pairs(Ctx& X, uint32_t* ex, uint32_t* ez, uint64_t total, uint32_t* hx,
                         uint32_t* hz) {
  using namespace d3g;
  if (total == 0) return;
  DBuf<uint64_t> keys = X.alloc<uint64_t>(total);
  DBuf<uint32_t> idx = X.alloc<uint32_t>(total);
  D3G_LAUNCH(X, pair_key_kernel, grid_for(total, 256), 256, 0, ex, ez, total, 0, 32, keys.p, idx.p);
  radix_sort(X, keys.p, idx.p, total, 64, false);
  DBuf<uint32_t> sx = X.alloc<uint32_t>(total), sz = X.alloc<uint32_t>(total);
  D3G_LAUNCH(X, permute_pairs_kernel, grid_for(total, 256), 256, 0, idx.p, total, ex, ez, sx.p, sz.p);
  X.to_host(hx, sx.p, total);
  X.to_host(hz, sz.p, total);
}

void upload_csr(Ctx& X, const d3g_csr* h, d3g::DeviceCsr& d) {
  d.n_rows = h->n_rows;
  d.n_cols = h->n_cols;
  d.nnz = h->nnz;
  d.row_ptr = X.alloc<uint64_t>(d.n_rows + 1);
  d.col = X.alloc<uint32_t>(d.nnz);
  X.to_device(d.row_ptr.p, h->row_ptr, d.n_rows + 1);
  X.to_device(d.col.p, h->col, d.nnz);
}

}  // namespace

extern "C" {

int d3g_sparse_bmm_csr(d3g_ctx* ctx, const d3g_csr* r_by_x, const d3g_csr* s_sparse_by_y,
                       uint32_t z_card, uint32_t* pairs_x, uint32_t* pairs_z, uint64_t pairs_cap,
                       uint64_t* count, d3g_kernel_stats* st) {
  return guarded([&] {
    using namespace d3g;
    Ctx& X = ctx->c;
    D3G_CUDA(cudaSetDevice(X.device));
    X.begin_call();
    X.budget = 0;
    DeviceCsr r, sp;
    upload_csr(X, r_by_x, r);
    upload_csr(X, s_sparse_by_y, sp);
    DBuf<uint32_t> ids = X.alloc<uint32_t>(z_card);
    if (z_card) D3G_LAUNCH(X, iota_kernel, grid_for(z_card, 256), 256, 0, ids.p, (uint64_t)z_card);
    SparseInputs si{r.row_ptr.p, r.col.p, r.n_rows, sp.row_ptr.p, sp.col.p, ids.p, z_card,
                    sp.n_rows, 0, r.n_rows};
    Decode dec{nullptr, nullptr, 0};
    Emit none{nullptr, nullptr, nullptr, 0};
    cudaEvent_t e0, e1;
    D3G_CUDA(cudaEventCreate(&e0));
    D3G_CUDA(cudaEventCreate(&e1));
    D3G_CUDA(cudaEventRecord(e0, X.stream));
    KernelOut ko;
    run_sparse(X, si, dec, kModeCount, none, ko);
    D3G_CUDA(cudaEventRecord(e1, X.stream));
    X.sync();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *count = ko.count;
    if (st) {
      std::memset(st, 0, sizeof(*st));
      st->inner_count = ko.inner;
      st->ms_kernel = ms;
    }
    if (pairs_x && pairs_z) {
      if (pairs_cap < ko.count) throw ResourceError("pair buffer too small");
      DBuf<uint32_t> ex = X.alloc<uint32_t>(ko.count), ez = X.alloc<uint32_t>(ko.count);
      DBuf<unsigned long long> cur = X.zeros<unsigned long long>(1);
      Emit em{ex.p, ez.p, cur.p, ko.count};
      KernelOut t;
      run_sparse(X, si, dec, kModeEmit, em, t);
      if (X.scalar(cur.p) != ko.count) throw CudaError("sparse_bmm: emitted != counted");
      sort_and_copy_pairs(X, ex.p, ez.p, ko.count, pairs_x, pairs_z);
    }
  });
}

int d3g_dense_ec_rows(d3g_ctx* ctx, const d3g_csr* r_by_x, const d3g_panel* panel,
                      const d3g_consts* c, int dense_mode, uint32_t* pairs_x, uint32_t* pairs_z,
                      uint64_t pairs_cap, uint64_t* count, d3g_kernel_stats* st) {
  return guarded([&] {
    using namespace d3g;
    Ctx& X = ctx->c;
    D3G_CUDA(cudaSetDevice(X.device));
    X.begin_call();
    X.budget = 0;
    DeviceCsr r;
    upload_csr(X, r_by_x, r);
    const uint64_t rows = panel->rows;
    const uint64_t y_card = panel->y_card;
    const uint64_t row_words = (y_card + panel->w - 1) / panel->w * panel->w / 64;
    *count = 0;
    if (st) std::memset(st, 0, sizeof(*st));
    if (rows == 0 || r.nnz == 0) return;
    DBuf<uint64_t> blocks = X.alloc<uint64_t>(rows * row_words);
    X.to_device(blocks.p, panel->blocks, rows * row_words);
    DBuf<uint32_t> zids = X.alloc<uint32_t>(rows);
    X.to_device(zids.p, panel->z_ids, rows);
    DBuf<uint32_t> cnt = X.alloc<uint32_t>(rows);
    D3G_LAUNCH(X, panel_popc_kernel, grid_for(rows * 32, 256), 256, 0, blocks.p, rows, row_words, cnt.p);
    DBuf<uint64_t> zptr = X.alloc<uint64_t>(rows + 1);
    exclusive_scan<uint32_t>(X, cnt.p, rows, zptr.p);
    uint64_t pnnz = X.scalar(zptr.p + rows);
    DBuf<uint32_t> zcol = X.alloc<uint32_t>(pnnz);
    D3G_LAUNCH(X, panel_extract_kernel, grid_for(rows * 32, 256), 256, 0, blocks.p, rows, row_words,
               zptr.p, zcol.p);
    DBuf<unsigned long long> mz = X.zeros<unsigned long long>(1);
    D3G_LAUNCH(X, max_u32_kernel, grid_for(rows, 256), 256, 0, cnt.p, rows, mz.p);
    uint64_t max_mz = X.scalar(mz.p);
    DBuf<uint32_t> row_ids = X.alloc<uint32_t>(rows);
    D3G_LAUNCH(X, iota_kernel, grid_for(rows, 256), 256, 0, row_ids.p, rows);
    // R-side degrees
    uint64_t yc = std::max<uint64_t>(y_card, r.n_cols);
    DBuf<uint32_t> dR = X.zeros<uint32_t>(yc);
    D3G_LAUNCH(X, value_hist_kernel, grid_for(r.nnz, 512, X.sm_count * 2), 512, 0, r.col.p, r.nnz, dR.p, (uint32_t)yc);
    uint64_t max_mx = 0;
    for (uint32_t i = 0; i < r_by_x->n_rows; ++i)
      max_mx = std::max<uint64_t>(max_mx, r_by_x->row_ptr[i + 1] - r_by_x->row_ptr[i]);
    std::vector<uint64_t> hmx(max_mx + 1, 0);
    for (uint32_t i = 0; i < r_by_x->n_rows; ++i) hmx[r_by_x->row_ptr[i + 1] - r_by_x->row_ptr[i]]++;
    DenseLayout L;
    build_dense_layout(X, r, max_mx, hmx, zptr.p, zcol.p, row_ids.p, rows, max_mz, zids.p, yc,
                       dR.p, L);
    DenseInputs di{L.xorder.p, L.n_live, r.row_ptr.p, r.col.p, L.y_rank.p, yc, L.dl_ptr.p,
                   L.dl_col.p, L.dl_z.p, L.n_dense, L.max_group_nnz, 0, L.n_live,
                   L.y_of_rank.p, dR.p, r.n_rows, 0, r.n_rows};
    Decode dec{nullptr, nullptr, 0};
    Emit none{nullptr, nullptr, nullptr, 0};
    cudaEvent_t e0, e1;
    D3G_CUDA(cudaEventCreate(&e0));
    D3G_CUDA(cudaEventCreate(&e1));
    D3G_CUDA(cudaEventRecord(e0, X.stream));
    KernelOut ko;
    run_dense(X, di, dec, kModeCount, none, ko);
    D3G_CUDA(cudaEventRecord(e1, X.stream));
    X.sync();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *count = ko.count;
    if (st) {
      st->ms_kernel = ms;
      // DenseEcStats of the reference's dense_ec on this panel under
      // dense_mode (counters.cuh): every panel row is dense
      const std::vector<uint32_t> thr = mode_thresholds(max_mx, y_card, c, dense_mode);
      DenseCounters dc{};
      if ((std::max<uint64_t>(y_card, 1) + 31) / 32 * 4 <= 220 * 1024) {
        dense_counters_device(X, r, 0, r.n_rows, zptr.p, zcol.p, rows, nullptr, 0, thr, panel->w,
                              y_card, dc);
      } else {  // |Y| too large for one smem row bitmap: encounters only
        std::vector<uint64_t> hd(max_mz + 1, 0);
        for (uint64_t j = 0; j < rows; ++j) hd[panel->m_z[j]]++;
        encounter_counts(hmx, hd, thr, dc);
      }
      st->wide_encounters = dc.wide;
      st->probe_encounters = dc.probe;
      st->blocks_checked = dc.blocks;
      st->probes_done = dc.probes;
      st->row_bitmaps_built = dc.bitmaps;
    }
    if (pairs_x && pairs_z) {
      if (pairs_cap < ko.count) throw ResourceError("pair buffer too small");
      DBuf<uint32_t> ex = X.alloc<uint32_t>(ko.count), ez = X.alloc<uint32_t>(ko.count);
      DBuf<unsigned long long> cur = X.zeros<unsigned long long>(1);
      Emit em{ex.p, ez.p, cur.p, ko.count};
      KernelOut t;
      run_dense(X, di, dec, kModeEmit, em, t);
      if (X.scalar(cur.p) != ko.count) throw CudaError("dense_ec: emitted != counted");
      sort_and_copy_pairs(X, ex.p, ez.p, ko.count, pairs_x, pairs_z);
    }
  });
}

// Convention-G rows [lo, hi) of side 0 (R) / 1 (S) of config cfg (1..5),
// written to DEVICE buffers left/right on the context's device.
int d3g_generate(d3g_ctx* ctx, int cfg, int side, uint64_t lo, uint64_t hi, uint64_t* left,
                 uint64_t* right) {
  return guarded([&] {
    using namespace d3g;
    Ctx& X = ctx->c;
    D3G_CUDA(cudaSetDevice(X.device));
    X.begin_call();
    uint64_t n = cfg_rows(cfg);
    if (n == 0 || hi > n || lo > hi) throw ConfigError("bad generator request");
    GenSpec g = gen_spec(cfg, side);
    DBuf<double> cum;
    if (g.zipf) {
      uint64_t ny = g.ny;
      std::vector<double> h(ny);
      double run = 0, alpha = gen_alpha(cfg);
      for (uint64_t r = 1; r <= ny; ++r) {
        run += std::pow(static_cast<double>(r), -alpha);
        h[r - 1] = run;
      }
      cum = X.alloc<double>(ny);
      X.to_device(cum.p, h.data(), ny);
    }
    if (hi > lo)
      D3G_LAUNCH(X, gen_kernel, grid_for(hi - lo, 256, X.sm_count * 32), 256, 0, g, cum.p, lo, hi,
                 left, right);
    X.sync();
  });
}

uint64_t d3g_cfg_rows(int cfg) { return d3g::cfg_rows(cfg); }

int d3g_map_tables(d3g_ctx* ctx, const d3g_table* r, const d3g_table* s, const d3g_opts* o,
                   d3g_mapping* out) {
  d3g::Ctx& X = ctx->c;
  int rc = guarded([&] {
    using namespace d3g;
    if (table_value_bytes(r) != 8 || table_value_bytes(s) != 8)
      throw ConfigError("map_tables takes u64 columns (value_bytes 0 or 8)");
    D3G_CUDA(cudaSetDevice(X.device));
    X.begin_call();
    X.budget = o->memory_budget_bytes ? o->memory_budget_bytes : (3ull << 30);
    const uint64_t NR = r->n, NS = s->n;
    DBuf<uint64_t> hb[4];
    const uint64_t *Rl = r->left, *Rr = r->right, *Sl = s->left, *Sr = s->right;
    if (!r->on_device) {
      hb[0] = X.alloc<uint64_t>(NR);
      hb[1] = X.alloc<uint64_t>(NR);
      X.to_device(hb[0].p, Rl, NR);
      X.to_device(hb[1].p, Rr, NR);
      Rl = hb[0].p;
      Rr = hb[1].p;
    }
    if (!s->on_device) {
      hb[2] = X.alloc<uint64_t>(NS);
      hb[3] = X.alloc<uint64_t>(NS);
      X.to_device(hb[2].p, Sl, NS);
      X.to_device(hb[3].p, Sr, NS);
      Sl = hb[2].p;
      Sr = hb[3].p;
    }
    d3g_report rep{};
    Mapped M;
    map_inputs(X, Rl, Rr, NR, Sl, Sr, NS, o, &rep, /*want_kept=*/true, M);
    M.check_natural();
    out->kept = M.kept;
    out->dropped_r = NR - M.kept;
    out->x_card = M.x_card;
    out->y_card = M.y_card;
    out->z_card = M.z_card;
    out->natural_x = M.D.x.identity;
    out->natural_y = M.D.y.identity;
    out->natural_z = M.D.z.identity;
    if (out->r_x) X.to_host(out->r_x, M.r_x, M.kept);
    if (out->r_y) X.to_host(out->r_y, M.r_y, M.kept);
    if (out->s_z) X.to_host(out->s_z, M.s_z, NS);
    if (out->s_y) X.to_host(out->s_y, M.s_y, NS);
    if (out->r_kept && M.r_kept.p) X.to_host(out->r_kept, M.r_kept.p, M.kept);
    if (out->rev_x && !M.D.x.identity) X.to_host(out->rev_x, M.D.x.rev.p, M.x_card);
    if (out->rev_y && !M.D.y.identity) X.to_host(out->rev_y, M.D.y.rev.p, M.y_card);
    if (out->rev_z && !M.D.z.identity) X.to_host(out->rev_z, M.D.z.rev.p, M.z_card);
  });
  X.budget = 0;
  return rc;
}

int d3g_join_aggregate(d3g_ctx* ctx, const d3g_valued_table* r, const d3g_valued_table* s,
                       int combine, int agg, const d3g_consts* c, const d3g_opts* o,
                       d3g_report* rep, d3g_agg_pairs* out) {
  d3g::Ctx& X = ctx->c;
  int rc = guarded([&] {
    D3G_CUDA(cudaSetDevice(X.device));
    X.begin_call();
    join_aggregate_impl(X, r, s, combine, agg, c, o, rep, out);
  });
  X.budget = 0;  // the memory budget is scoped to one call
  return rc;
}

// ---- table files ------------------------------------------------------------
int d3g_detect_format(const char* path, int requested) {
  if (requested != D3G_FMT_AUTO) return requested;
  std::string p = path ? path : "";
  const size_t slash = p.find_last_of('/');
  const size_t dot = p.find_last_of('.');
  std::string ext = (dot == std::string::npos || (slash != std::string::npos && dot < slash))
                        ? ""
                        : p.substr(dot);
  if (ext == ".tsv" || ext == ".txt") return D3G_FMT_TSV;
  if (ext == ".csv") return D3G_FMT_CSV;
  if (ext == ".bin") return D3G_FMT_BINARY;
  return D3G_FMT_TSV;
}

namespace {
struct FileCloser {
  FILE* f;
  ~FileCloser() {
    if (f) std::fclose(f);
  }
};
uint64_t binary_rows_or_throw(const char* path) {
  FILE* f = std::fopen(path, "rb");
  if (!f) throw d3g::Error(D3G_IO_ERROR, std::string("cannot open ") + path);
  FileCloser fc{f};
  if (std::fseek(f, 0, SEEK_END) != 0) throw d3g::Error(D3G_IO_ERROR, std::string("cannot seek ") + path);
  const long long len = std::ftell(f);
  if (len < 0 || len % 16 != 0)
    throw d3g::Error(D3G_FORMAT_ERROR, std::string(path) + ": binary table length " +
                                           std::to_string(len) + " is not a multiple of 16");
  return (uint64_t)len / 16;
}
// Two pinned staging chunks with their own events (double buffering).
struct Staging {
  d3g::Ctx& X;
  void* host[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  size_t bytes;
  Staging(d3g::Ctx& x, size_t b) : X(x), bytes(b) {
    for (int i = 0; i < 2; ++i) {
      D3G_CUDA(cudaMallocHost(&host[i], bytes));
      D3G_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
  }
  ~Staging() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventSynchronize(ev[i]), cudaEventDestroy(ev[i]);
      if (host[i]) cudaFreeHost(host[i]);
    }
  }
};
}  // namespace

int d3g_binary_rows(const char* path, uint64_t* n) {
  return guarded([&] { *n = binary_rows_or_throw(path); });
}

int d3g_read_binary(d3g_ctx* ctx, const char* path, uint64_t* left, uint64_t* right, uint64_t n) {
  return guarded([&] {
    using namespace d3g;
    Ctx& X = ctx->c;
    D3G_CUDA(cudaSetDevice(X.device));
    X.begin_call();
    const uint64_t rows = binary_rows_or_throw(path);
    if (rows != n)
      throw ConfigError("d3g_read_binary: n = " + std::to_string(n) + " but the file holds " +
                        std::to_string(rows) + " rows");
    if (n == 0) return;
    FILE* f = std::fopen(path, "rb");
    if (!f) throw Error(D3G_IO_ERROR, std::string("cannot open ") + path);
    FileCloser fc{f};
    const uint64_t chunk_rows = std::min<uint64_t>(n, 4ull << 20);  // 64 MB chunks
    Staging st(X, chunk_rows * 16);
    DBuf<uint64_t> dev[2] = {X.alloc<uint64_t>(2 * chunk_rows), X.alloc<uint64_t>(2 * chunk_rows)};
    uint64_t done = 0;
    for (int b = 0; done < n; b ^= 1) {
      const uint64_t take = std::min(chunk_rows, n - done);
      D3G_CUDA(cudaEventSynchronize(st.ev[b]));  // the chunk's previous copy has drained
      if (std::fread(st.host[b], 16, take, f) != take)
        throw Error(D3G_IO_ERROR, std::string("read error on ") + path);
      D3G_CUDA(cudaMemcpyAsync(dev[b].p, st.host[b], take * 16, cudaMemcpyHostToDevice, X.stream));
      D3G_LAUNCH(X, deinterleave_kernel, grid_for(take, 256), 256, 0, dev[b].p, take, left + done,
                 right + done);
      D3G_CUDA(cudaEventRecord(st.ev[b], X.stream));
      done += take;
    }
    X.sync();
  });
}

int d3g_save_pairs(d3g_ctx* ctx, const uint64_t* left, const uint64_t* right, uint64_t n,
                   int on_device, const char* path, int format) {
  return guarded([&] {
    using namespace d3g;
    Ctx& X = ctx->c;
    D3G_CUDA(cudaSetDevice(X.device));
    X.begin_call();
    const int fmt = d3g_detect_format(path, format);
    if (fmt < D3G_FMT_TSV || fmt > D3G_FMT_BINARY) throw ConfigError("unknown table format");
    FILE* f = std::fopen(path, "wb");
    if (!f) throw Error(D3G_IO_ERROR, std::string("cannot open ") + path + " for writing");
    FileCloser fc{f};
    const uint64_t chunk_rows = std::max<uint64_t>(1, std::min<uint64_t>(n, 2ull << 20));
    const size_t out_bytes = fmt == D3G_FMT_BINARY ? chunk_rows * 16 : chunk_rows * 42;
    Staging st(X, out_bytes);
    DBuf<uint64_t> in_l, in_r;
    if (!on_device) {
      in_l = X.alloc<uint64_t>(chunk_rows);
      in_r = X.alloc<uint64_t>(chunk_rows);
    }
    DBuf<char> dout[2] = {X.alloc<char>(out_bytes), X.alloc<char>(out_bytes)};
    DBuf<uint32_t> len = X.alloc<uint32_t>(chunk_rows);
    DBuf<uint64_t> off = X.alloc<uint64_t>(chunk_rows + 1);
    size_t pending[2] = {0, 0};
    auto flush = [&](int b) {
      if (!pending[b]) return;
      D3G_CUDA(cudaEventSynchronize(st.ev[b]));
      if (std::fwrite(st.host[b], 1, pending[b], f) != pending[b])
        throw Error(D3G_IO_ERROR, std::string("write error on ") + path);
      pending[b] = 0;
    };
    uint64_t done = 0;
    int b = 0;
    for (; done < n; b ^= 1) {
      const uint64_t take = std::min(chunk_rows, n - done);
      flush(b);  // staging buffer b is free again
      const uint64_t* l = left + done;
      const uint64_t* r = right + done;
      if (!on_device) {
        X.to_device(in_l.p, l, take);
        X.to_device(in_r.p, r, take);
        l = in_l.p;
        r = in_r.p;
      }
      size_t bytes;
      if (fmt == D3G_FMT_BINARY) {
        D3G_LAUNCH(X, interleave_kernel, grid_for(take, 256), 256, 0, l, r, take,
                   reinterpret_cast<uint64_t*>(dout[b].p));
        bytes = take * 16;
      } else {
        D3G_LAUNCH(X, text_len_kernel, grid_for(take, 256), 256, 0, l, r, take, len.p);
        exclusive_scan<uint32_t>(X, len.p, take, off.p);
        bytes = X.scalar(off.p + take);
        D3G_LAUNCH(X, text_write_kernel, grid_for(take, 256), 256, 0, l, r, take, off.p,
                   fmt == D3G_FMT_CSV ? ',' : '\t', dout[b].p);
      }
      D3G_CUDA(cudaMemcpyAsync(st.host[b], dout[b].p, bytes, cudaMemcpyDeviceToHost, X.stream));
      D3G_CUDA(cudaEventRecord(st.ev[b], X.stream));
      pending[b] = bytes;
      done += take;
      if (!on_device) X.sync();  // the host-input staging is reused next chunk
    }
    flush(b);      // the older of the two pending chunks first
    flush(b ^ 1);
    if (std::fflush(f) != 0) throw Error(D3G_IO_ERROR, std::string("write error on ") + path);
  });
}

int d3g_ctx_device(d3g_ctx* ctx) { return ctx ? ctx->c.device : -1; }

}  // extern "C"

// ---------------------------------------------------------------------------
// Measured integer-pipe peak for the DenseEC roofline: 3-input LOP3 chains,
// 8 independent chains per thread, 148 x 4 CTAs of 256 threads. Returns
// logic ops/s (one LOP3 = one 32-bit op).
namespace {
__global__ void __launch_bounds__(256) alu_peak_kernel(uint32_t seed, int iters, uint32_t* out) {
  uint32_t a[8], b = seed * 0x9e3779b1u + threadIdx.x, c = seed ^ (blockIdx.x * 0x85ebca6bu);
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * (j + 1) + seed;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t r;
      asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a[j]), "r"(b), "r"(c));
      a[j] = r;
      asm volatile("lop3.b32 %0, %1, %2, %3, 0xe8;" : "=r"(r) : "r"(a[j]), "r"(c), "r"(b));
      a[j] = r;
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) x ^= a[j];
  if (x == 0x12345678u) out[0] = x;
}
}  // namespace

namespace {
// conflict-free LDS.128 streams: lane l of warp w reads row (i + w) % rows,
// column l; 8 independent loads per iteration, xor-folded
__global__ void __launch_bounds__(1024) smem_peak_kernel(int iters, uint32_t* out) {
  extern __shared__ __align__(16) uint4 sbuf[];  // [rows][32]
  constexpr int kRows = 256;
  for (int i = threadIdx.x; i < kRows * 32; i += blockDim.x)
    sbuf[i] = make_uint4(i, i * 3u, i ^ 0x55u, i + 7u);
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t row = (uint32_t)(it * 8 + j + w) & (kRows - 1);
      const uint4 v = sbuf[row * 32 + lane];
      acc.x ^= v.x;
      acc.y ^= v.y;
      acc.z ^= v.z;
      acc.w ^= v.w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[0] = acc.x;
}
}  // namespace

extern "C" int d3g_smem_peak(d3g_ctx* ctx, double* bytes_per_sec) {
  return guarded([&] {
    using namespace d3g;
    Ctx& X = ctx->c;
    D3G_CUDA(cudaSetDevice(X.device));
    X.begin_call();
    DBuf<uint32_t> out = X.zeros<uint32_t>(1);
    const size_t sm = 256 * 32 * 16;  // 128 KB: one CTA of 1024 threads per SM
    D3G_CUDA(raise_smem_attr(smem_peak_kernel, (int)sm));
    const unsigned grid = (unsigned)X.sm_count;
    const int iters = 8192;
    smem_peak_kernel<<<grid, 1024, sm, X.stream>>>(64, out.p);  // warm-up
    cudaEvent_t e0, e1;
    D3G_CUDA(cudaEventCreate(&e0));
    D3G_CUDA(cudaEventCreate(&e1));
    D3G_CUDA(cudaEventRecord(e0, X.stream));
    smem_peak_kernel<<<grid, 1024, sm, X.stream>>>(iters, out.p);
    D3G_CUDA(cudaEventRecord(e1, X.stream));
    X.sync();
    D3G_CUDA(cudaGetLastError());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double bytes = (double)grid * 1024.0 * iters * 8.0 * 16.0;
    *bytes_per_sec = bytes / (ms * 1e-3);
  });
}

extern "C" int d3g_alu_peak(d3g_ctx* ctx, double* ops_per_sec) {
  return guarded([&] {
    using namespace d3g;
    Ctx& X = ctx->c;
    D3G_CUDA(cudaSetDevice(X.device));
    X.begin_call();
    DBuf<uint32_t> out = X.zeros<uint32_t>(1);
    const int iters = 4096;
    const unsigned grid = (unsigned)X.sm_count * 8;
    alu_peak_kernel<<<grid, 256, 0, X.stream>>>(1u, 64, out.p);  // warm-up
    cudaEvent_t e0, e1;
    D3G_CUDA(cudaEventCreate(&e0));
    D3G_CUDA(cudaEventCreate(&e1));
    D3G_CUDA(cudaEventRecord(e0, X.stream));
    alu_peak_kernel<<<grid, 256, 0, X.stream>>>(2u, iters, out.p);
    D3G_CUDA(cudaEventRecord(e1, X.stream));
    X.sync();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    double ops = (double)grid * 256.0 * iters * 16.0;
    *ops_per_sec = ops / (ms * 1e-3);
  });
}
