// CSR grouping (north_star subsystem 1, second half) and degree statistics.
//
// build_csr (P/src/relation.cpp:206-258) produces rows sorted by the minor
// code with duplicate pairs collapsed. On the GPU: one stable LSD radix sort
// of the composite key (major << minor_bits | minor), a flag/scan/compact
// pass that drops adjacent duplicates, and a boundary fill that writes
// row_ptr. compute_degree_stats (P/src/costmodel.cpp:425-438) reads m_x/m_z
// off row_ptr, histograms the column codes into dR(y)/dS(y) with
// shared-memory privatised counters, and reduces OUT_J = sum_y dR(y)*dS(y)
// with a 128-bit accumulator (out_j_from_degrees, :350-364).
#pragma once

#include "segsort.cuh"

namespace d3g {

struct DeviceCsr {
  DBuf<uint64_t> row_ptr;  // n_rows + 1
  DBuf<uint32_t> col;      // nnz
  uint64_t n_rows = 0, n_cols = 0, nnz = 0;
  // largest row and number of non-empty rows (~0ull: not known on the host)
  uint64_t max_deg = ~0ull, live_rows = 0;
};

// max and number of non-zero entries of a u32 array (the kept row lengths)
__global__ void len_stats_kernel(const uint32_t* __restrict__ len, uint64_t n,
                                 unsigned long long* __restrict__ out /* max, nonzero */) {
  uint64_t m = 0, live = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t d = len[i];
    m = d > m ? d : m;
    live += d > 0;
  }
  m = warp_max(m);
  live = warp_sum(live);
  if (lane_id() == 0) {
    if (m) atomicMax(out, (unsigned long long)m);
    if (live) atomicAdd(out + 1, (unsigned long long)live);
  }
}

__global__ void composite_key_kernel(const uint32_t* __restrict__ maj,
                                     const uint32_t* __restrict__ mnr, uint64_t n, int minor_bits,
                                     uint64_t* __restrict__ keys) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = ((uint64_t)maj[i] << minor_bits) | (uint64_t)mnr[i];
}

__global__ void uniq_flag_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                 uint32_t* __restrict__ flag) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

__global__ void uniq_write_kernel(const uint64_t* __restrict__ keys,
                                  const uint32_t* __restrict__ flag,
                                  const uint64_t* __restrict__ pos, uint64_t n, int minor_bits,
                                  uint32_t* __restrict__ col, uint32_t* __restrict__ row_of) {
  const uint64_t mmask = minor_bits >= 64 ? ~0ull : ((1ull << minor_bits) - 1);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (!flag[i]) continue;
    uint64_t k = keys[i], o = pos[i];
    col[o] = (uint32_t)(k & mmask);
    row_of[o] = (uint32_t)(k >> minor_bits);
  }
}

// row_ptr[r] = first unique index with row >= r; row_ptr[n_rows] = nnz.
__global__ void row_bounds_kernel(const uint32_t* __restrict__ row_of, uint64_t nnz,
                                  uint64_t n_rows, uint64_t* __restrict__ row_ptr) {
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u <= nnz;
       u += (uint64_t)gridDim.x * blockDim.x) {
    int64_t prev = u == 0 ? -1 : (int64_t)row_of[u - 1];
    int64_t cur = u == nnz ? (int64_t)n_rows : (int64_t)row_of[u];
    for (int64_t r = prev + 1; r <= cur && r <= (int64_t)n_rows; ++r) row_ptr[r] = u;
  }
}

// Large builds go through the bucketed path (csr_bucket.cuh); small ones,
// and skewed majors whose buckets overflow shared memory, through the
// counting scatter + segmented sort/unique below (segsort.cuh).
// D3G_CSR=scatter forces the latter, D3G_CSR=bucket the former at any size.
inline bool build_csr_bucketed(Ctx& ctx, const uint32_t* maj, const uint32_t* mnr, uint64_t n,
                               uint64_t n_rows, uint64_t n_cols, DeviceCsr& out, bool force);

inline void build_csr_device(Ctx& ctx, const uint32_t* maj, const uint32_t* mnr, uint64_t n,
                             uint64_t n_rows, uint64_t n_cols, DeviceCsr& out) {
  {
    const char* e = std::getenv("D3G_CSR");
    const bool force_bucket = e && std::strcmp(e, "bucket") == 0;
    const bool force_scatter = e && std::strcmp(e, "scatter") == 0;
    if (!force_scatter && build_csr_bucketed(ctx, maj, mnr, n, n_rows, n_cols, out, force_bucket))
      return;
  }
  out.n_rows = n_rows;
  out.n_cols = n_cols;
  out.row_ptr = ctx.alloc<uint64_t>(n_rows + 1);
  if (n == 0 || n_rows == 0) {
    D3G_CUDA(cudaMemsetAsync(out.row_ptr.p, 0, (n_rows + 1) * 8, ctx.stream));
    out.col = ctx.alloc<uint32_t>(0);
    out.nnz = 0;
    out.max_deg = out.live_rows = 0;
    return;
  }
  unsigned g = grid_for(n, 256);
  DBuf<uint32_t> cnt = ctx.zeros<uint32_t>(n_rows);
  D3G_LAUNCH(ctx, major_hist_kernel, g, 256, 0, maj, n, cnt.p);
  DBuf<uint64_t> off = ctx.alloc<uint64_t>(n_rows + 1);
  exclusive_scan<uint32_t>(ctx, cnt.p, n_rows, off.p);
  DBuf<uint32_t> tmp = ctx.alloc<uint32_t>(n);
  // Large builds (cfg5: 2 x 200M tuples over 10M rows): one 8-bit radix pass
  // on the high row bits first, so the per-row scatter below writes inside a
  // ~1/256 window that stays in L2 instead of scattering 4-byte writes over
  // the whole array (cfg5: 15 ms per relation). Rows are sorted afterwards,
  // so the order inside a row does not matter.
  const int row_bits = bits_for(n_rows - 1);
  if (n >= (1ull << 24) && row_bits > 12 && std::getenv("D3G_CSR_DIRECT") == nullptr) {
    DBuf<uint32_t> pm = ctx.alloc<uint32_t>(n), pv = ctx.alloc<uint32_t>(n);
    if (std::getenv("D3G_CSR_STABLE_BUCKETS"))
      radix_pass_u32(ctx, maj, mnr, n, row_bits - 8, pm.p, pv.p);
    else
      bucket_pass_u32(ctx, maj, mnr, n, row_bits - 8, pm.p, pv.p);
    D3G_LAUNCH(ctx, major_scatter_kernel, g, 256, 0, pm.p, pv.p, n, off.p, cnt.p, tmp.p);
  } else {
    D3G_LAUNCH(ctx, major_scatter_kernel, g, 256, 0, maj, mnr, n, off.p, cnt.p, tmp.p);
  }
  segmented_sort(ctx, tmp.p, off.p, n_rows, /*unique=*/true, cnt.p);  // cnt <- kept per row
  exclusive_scan<uint32_t>(ctx, cnt.p, n_rows, out.row_ptr.p);
  // one round trip: nnz, the largest row and the non-empty rows (degree stats)
  DBuf<unsigned long long> st = ctx.zeros<unsigned long long>(2);
  D3G_LAUNCH(ctx, len_stats_kernel, grid_for(n_rows, 256), 256, 0, cnt.p, n_rows, st.p);
  unsigned long long hs[2];
  ctx.defer(&out.nnz, out.row_ptr.p + n_rows, 8);
  ctx.defer(hs, st.p, 16);
  ctx.sync();
  out.max_deg = hs[0];
  out.live_rows = hs[1];
  out.col = ctx.alloc<uint32_t>(out.nnz);
  D3G_LAUNCH(ctx, row_compact_kernel, grid_for(n_rows * 8, 256), 256, 0, tmp.p, off.p,
             out.row_ptr.p, n_rows, out.col.p);
}

// ---------------------------------------------------------------------------
// Degree statistics.

// max row degree
__global__ void max_degree_kernel(const uint64_t* __restrict__ row_ptr, uint64_t n_rows,
                                  unsigned long long* __restrict__ out_max,
                                  unsigned long long* __restrict__ out_live) {
  uint64_t m = 0, live = 0;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t d = row_ptr[r + 1] - row_ptr[r];
    m = d > m ? d : m;
    live += d > 0;
  }
  m = warp_max(m);
  live = warp_sum(live);
  if (lane_id() == 0) {
    if (m) atomicMax(out_max, (unsigned long long)m);
    if (live) atomicAdd(out_live, (unsigned long long)live);
  }
}

// hist[d] += #rows with degree d (d <= max_deg). Small degrees privatised in smem.
constexpr int kDegSmem = 4096;
__global__ void degree_hist_kernel(const uint64_t* __restrict__ row_ptr, uint64_t n_rows,
                                   uint64_t hist_len, unsigned long long* __restrict__ hist) {
  __shared__ unsigned int sh[kDegSmem];
  for (int i = threadIdx.x; i < kDegSmem; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t d = row_ptr[r + 1] - row_ptr[r];
    if (d < kDegSmem)
      atomicAdd(&sh[d], 1u);
    else
      atomicAdd(&hist[d], 1ull);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kDegSmem && (uint64_t)i < hist_len; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

// counts[v] += 1 for every v in vals. Warps first merge equal values
// (__match_any_sync: one atomic per distinct value per warp, which matters
// for Zipf-skewed y columns where one code holds ~10% of the entries), then
// codes below kHotSmem count in shared memory, others in global memory.
constexpr int kHotSmem = 12288;
__global__ void value_hist_kernel(const uint32_t* __restrict__ vals, uint64_t n,
                                  uint32_t* __restrict__ counts, uint32_t card) {
  // hot values (the small codes: Zipf-ranked y) in a shared-memory histogram,
  // the rest straight to global; four independent loads in flight per thread
  // (the pass is bound by load latency, not by the atomics)
  __shared__ unsigned int sh[kHotSmem];
  const uint32_t hot = card < kHotSmem ? card : kHotSmem;
  for (uint32_t i = threadIdx.x; i < hot; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
    uint32_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = i + k * stride < n ? vals[i + k * stride] : 0xffffffffu;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (v[k] < hot)
        atomicAdd(&sh[v[k]], 1u);
      else if (v[k] != 0xffffffffu)
        atomicAdd(&counts[v[k]], 1u);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < hot; i += blockDim.x)
    if (sh[i]) atomicAdd(&counts[i], sh[i]);
}

// wz[deg(z)] += sum_{y in row z} dR(y): per-degree join sizes of the rows
// (8 lanes per row; degrees below kDegSmem privatised in shared memory).
__global__ void row_join_hist_kernel(const uint64_t* __restrict__ row_ptr,
                                     const uint32_t* __restrict__ col, uint64_t n_rows,
                                     const uint32_t* __restrict__ dr, uint64_t hist_len,
                                     unsigned long long* __restrict__ wz) {
  constexpr int kW = 2048;
  __shared__ unsigned long long sh[kW];
  for (int i = threadIdx.x; i < kW; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t sl = threadIdx.x & 7;
  const uint64_t stride = (uint64_t)gridDim.x * (blockDim.x / 8);
  const uint64_t first = (uint64_t)blockIdx.x * (blockDim.x / 8) + (threadIdx.x >> 3);
  // uniform trip count per warp so the 8-lane reductions stay converged
  const uint64_t trips = n_rows > first ? (n_rows - first + stride - 1) / stride : 0;
  const uint64_t wtrips = __reduce_max_sync(0xffffffffu, (unsigned)trips);
  for (uint64_t t = 0; t < wtrips; ++t) {
    const uint64_t r = first + t * stride;
    uint64_t sum = 0, d = 0;
    if (r < n_rows) {
      const uint64_t b = row_ptr[r], e = row_ptr[r + 1];
      d = e - b;
      for (uint64_t k = b + sl; k < e; k += 8) sum += dr[col[k]];
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (sl == 0 && sum) {
      if (d < (uint64_t)kW)
        atomicAdd(&sh[d], (unsigned long long)sum);
      else
        atomicAdd(&wz[d], (unsigned long long)sum);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kW && (uint64_t)i < hist_len; i += blockDim.x)
    if (sh[i]) atomicAdd(&wz[i], sh[i]);
}

// OUT_J = sum dR*dS with a (hi, lo) 128-bit accumulator per block.
__global__ void outj_kernel(const uint32_t* __restrict__ dr, const uint32_t* __restrict__ ds,
                            uint64_t y_card, unsigned long long* __restrict__ parts) {
  uint64_t lo = 0, hi = 0;
  for (uint64_t y = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; y < y_card;
       y += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t p = (uint64_t)dr[y] * (uint64_t)ds[y];
    uint64_t nl = lo + p;
    hi += nl < lo;
    lo = nl;
  }
  // reduce (lo, hi) across the block via shared memory
  __shared__ uint64_t slo[1024], shi[1024];
  slo[threadIdx.x] = lo;
  shi[threadIdx.x] = hi;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t L = 0, H = 0;
    for (unsigned i = 0; i < blockDim.x; ++i) {
      uint64_t nl = L + slo[i];
      H += shi[i] + (nl < L);
      L = nl;
    }
    parts[2 * blockIdx.x] = L;
    parts[2 * blockIdx.x + 1] = H;
  }
}

}  // namespace d3g
