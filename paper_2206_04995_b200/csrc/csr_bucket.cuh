// Bucketed CSR build: build_csr (P/src/relation.cpp:206-258 -- two stable
// counting sorts then an adjacent-duplicate collapse per row) as ONE global
// scatter plus CTA-local work in shared memory.
//
// Rows are cut into buckets of 2^r consecutive row codes, with r chosen so a
// bucket holds at most ~7K tuples (28 KB of packed keys). Then:
//   K1 csr_bucket_hist    one read of the major codes: bucket histogram
//                         (shared-memory privatised), and the largest bucket
//   K2 scan               bucket starts
//   K3 two-level scatter  region_bucket_scatter (8-bit bucketing on the high
//                         bucket bits, runs reserved by one atomic per
//                         (tile, region)) then csr_region_scatter (one atomic
//                         per (tile, bucket)): the packed key
//                         (row_low << mb | minor) lands in its bucket.
//                         (csr_bucket_scatter, one returning atomic per pair,
//                         is kept as D3G_CSR_SCATTER=atomic for comparison)
//   K4 csr_bucket_build   one CTA per bucket, all in shared memory: counting
//                         sort by row_low, per-row warp bitonic sort + unique
//                         of the minors, row degrees, bucket-local compaction
//   K5 scan               degrees -> row_ptr
//   K6 csr_bucket_copy    each bucket's unique run to its final offset
//                         (a contiguous copy: rows are in order inside it)
// Compulsory traffic per tuple: 4 (K1) + 8 + 4 (K3) + 4 (K4 read) + ~3 + 3
// (K4 write, K6 copy of the unique entries) + 4 (K6 read) bytes, against
// ~24 B/tuple of atomic per-row scatter + sort passes before. Buckets whose
// tuple count exceeds the shared-memory capacity (skewed majors) make the
// caller fall back to the per-row scatter path (segsort.cuh).
#pragma once

#include "csr.cuh"

namespace d3g {

constexpr int kCbThreads = 512;
constexpr uint32_t kCbCap = 12288;        // packed keys per bucket in smem (2 CTAs/SM)
constexpr uint32_t kCbTarget = 7168;      // expected tuples per bucket (at most)
constexpr uint32_t kCbMaxRowsLog = 11;    // <= 2048 rows per bucket
constexpr uint32_t kCbMaxBuckets = 32768; // privatised histogram (128 KB)
constexpr uint32_t kCbThreadRow = 0;      // rows up to this length: one thread each (measured slower than the warp sort on cfg5: 0 = off)

__global__ void max_u32_kernel(const uint32_t* __restrict__ v, uint64_t n,
                               unsigned long long* __restrict__ out) {
  uint64_t m = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    m = v[i] > m ? v[i] : m;
  m = warp_max(m);
  if (lane_id() == 0 && m) atomicMax(out, (unsigned long long)m);
}

// Latency, not bandwidth, bounds these passes (one dependent load -> atomic
// chain per element): every thread keeps kCbIlp elements in flight, loaded
// as 16-byte vectors when the column is aligned.
constexpr int kCbIlp = 8;

__device__ __forceinline__ bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

// K1: bucket histogram (shared-memory privatised; n_buckets <= kCbMaxBuckets).
__global__ void __launch_bounds__(kCbThreads)
csr_bucket_hist_kernel(const uint32_t* __restrict__ maj, uint64_t n, int r, uint32_t n_buckets,
                       unsigned int* __restrict__ hist) {
  extern __shared__ unsigned int sh[];
  for (uint32_t i = threadIdx.x; i < n_buckets; i += kCbThreads) sh[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * kCbThreads * kCbIlp;
  uint64_t i0 = ((uint64_t)blockIdx.x * kCbThreads + threadIdx.x) * kCbIlp;
  if (aligned16(maj)) {
    for (; i0 + kCbIlp <= n; i0 += stride) {
      uint4 v[kCbIlp / 4];
#pragma unroll
      for (int k = 0; k < kCbIlp / 4; ++k) v[k] = reinterpret_cast<const uint4*>(maj + i0)[k];
#pragma unroll
      for (int k = 0; k < kCbIlp / 4; ++k) {
        atomicAdd(&sh[v[k].x >> r], 1u);
        atomicAdd(&sh[v[k].y >> r], 1u);
        atomicAdd(&sh[v[k].z >> r], 1u);
        atomicAdd(&sh[v[k].w >> r], 1u);
      }
    }
  }
  for (; i0 < n; i0 += stride)  // the tail (and unaligned columns)
    for (uint64_t i = i0; i < i0 + kCbIlp && i < n; ++i) atomicAdd(&sh[maj[i] >> r], 1u);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n_buckets; i += kCbThreads)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// K3: packed key into its bucket (order inside a bucket is irrelevant: K4
// sorts). cursor[b] starts at the bucket's start. kCbIlp independent
// (load, atomic, store) chains per thread.
__global__ void __launch_bounds__(kCbThreads)
csr_bucket_scatter_kernel(const uint32_t* __restrict__ maj, const uint32_t* __restrict__ mnr,
                          uint64_t n, int r, int mb, unsigned long long* __restrict__ cursor,
                          uint32_t* __restrict__ packed) {
  const uint32_t rmask = (1u << r) - 1;
  const uint64_t stride = (uint64_t)gridDim.x * kCbThreads * kCbIlp;
  uint64_t i0 = ((uint64_t)blockIdx.x * kCbThreads + threadIdx.x) * kCbIlp;
  if (aligned16(maj) && aligned16(mnr)) {
    for (; i0 + kCbIlp <= n; i0 += stride) {
      uint32_t a[kCbIlp], b[kCbIlp];
#pragma unroll
      for (int k = 0; k < kCbIlp / 4; ++k) {
        const uint4 va = reinterpret_cast<const uint4*>(maj + i0)[k];
        const uint4 vb = reinterpret_cast<const uint4*>(mnr + i0)[k];
        a[4 * k] = va.x, a[4 * k + 1] = va.y, a[4 * k + 2] = va.z, a[4 * k + 3] = va.w;
        b[4 * k] = vb.x, b[4 * k + 1] = vb.y, b[4 * k + 2] = vb.z, b[4 * k + 3] = vb.w;
      }
      unsigned long long p[kCbIlp];
#pragma unroll
      for (int k = 0; k < kCbIlp; ++k) p[k] = atomicAdd(&cursor[a[k] >> r], 1ull);
#pragma unroll
      for (int k = 0; k < kCbIlp; ++k) packed[p[k]] = ((a[k] & rmask) << mb) | b[k];
    }
  }
  for (; i0 < n; i0 += stride)
    for (uint64_t i = i0; i < i0 + kCbIlp && i < n; ++i) {
      const uint32_t a = maj[i], b = mnr[i];
      const unsigned long long p = atomicAdd(&cursor[a >> r], 1ull);
      packed[p] = ((a & rmask) << mb) | b;
    }
}

// Two-level alternative to K3 for many buckets: after an 8-bit bucketing pass
// on the high bucket bits (prims.cuh bucket_pass_u32: tile-local ranks, runs
// written per digit, no atomics), every 4096-pair tile lies inside one region
// of <= 256 consecutive buckets. The tile is ranked by bucket in shared
// memory, each (tile, bucket) run is reserved with ONE global atomic, and the
// packed keys are written out in runs -- instead of one returning global
// atomic per pair (K3 is bound by L2 atomic throughput: ~45 G/s).
constexpr int kRbThreads = 1024;
constexpr int kRbPer = 4;
constexpr int kRbTile = kRbThreads * kRbPer;

struct RbTile {
  unsigned long long start;  // first pair of the tile (region-ordered arrays)
  uint32_t len;              // <= kRbTile
  uint32_t region;           // high bucket bits (bucket >> sub_bits)
};

// A CTA finds its tile itself: region d (pairs [starts[d], starts[d + 1]) of
// the region-ordered arrays) is cut into tiles of kRbTile pairs, tile_prefix
// is the exclusive prefix of the regions' tile counts (region_starts_kernel),
// and the grid is an upper bound (n / kRbTile + 256): no tile list built on
// the host, no round trip between the two scatter passes.
__global__ void __launch_bounds__(kRbThreads)
csr_region_scatter_kernel(const uint32_t* __restrict__ maj, const uint32_t* __restrict__ mnr,
                          const uint64_t* __restrict__ starts /* [257] */,
                          const uint32_t* __restrict__ tile_prefix /* [257] */, int r, int mb,
                          int sub_bits, unsigned long long* __restrict__ cursor,
                          uint32_t* __restrict__ packed) {
  __shared__ uint32_t s_cnt[256], s_loc[256];
  __shared__ unsigned long long s_glb[256];
  __shared__ uint32_t s_out[kRbTile];
  __shared__ uint32_t s_tp[257];
  const uint32_t t = threadIdx.x;
  if (t < 257) s_tp[t] = tile_prefix[t];
  if (t < 256) s_cnt[t] = 0;
  __syncthreads();
  if (blockIdx.x >= s_tp[256]) return;  // (CTA-uniform)
  uint32_t lo = 0, hi = 256;  // the region whose tiles hold blockIdx.x
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (s_tp[mid] <= blockIdx.x) lo = mid; else hi = mid;
  }
  RbTile tl;
  tl.region = lo;
  tl.start = starts[lo] + (unsigned long long)(blockIdx.x - s_tp[lo]) * kRbTile;
  {
    const unsigned long long left = starts[lo + 1] - tl.start;
    tl.len = left < (unsigned long long)kRbTile ? (uint32_t)left : (uint32_t)kRbTile;
  }
  const uint32_t smask = (1u << sub_bits) - 1, rmask = (1u << r) - 1;
  uint32_t key[kRbPer], sub[kRbPer], rk[kRbPer];
#pragma unroll
  for (int q = 0; q < kRbPer; ++q) {
    const uint32_t i = (uint32_t)q * kRbThreads + t;
    if (i < tl.len) {
      const uint32_t a = maj[tl.start + i], b = mnr[tl.start + i];
      sub[q] = (a >> r) & smask;
      key[q] = ((a & rmask) << mb) | b;
      rk[q] = atomicAdd(&s_cnt[sub[q]], 1u);
    }
  }
  __syncthreads();
  if (t < 32) {  // exclusive scan of the 256 sub-bucket counts, 8 per lane
    uint32_t c[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c[j] = s_cnt[t * 8 + j];
      sum += c[j];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (t >= (uint32_t)o) incl += u;
    }
    uint32_t run = incl - sum;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s_loc[t * 8 + j] = run;
      run += c[j];
    }
  }
  // one global reservation per (tile, bucket)
  if (t < 256 && s_cnt[t])
    s_glb[t] = atomicAdd(&cursor[((uint64_t)tl.region << sub_bits) | t],
                         (unsigned long long)s_cnt[t]);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kRbPer; ++q) {
    const uint32_t i = (uint32_t)q * kRbThreads + t;
    if (i < tl.len) s_out[s_loc[sub[q]] + rk[q]] = key[q];
  }
  __syncthreads();
  // the staged tile out in runs: position p belongs to the last sub-bucket
  // whose local start is <= p (empty sub-buckets start where the next does)
  for (uint32_t p = t; p < tl.len; p += kRbThreads) {
    uint32_t lo = 0, hi = 256;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_loc[mid] <= p) lo = mid; else hi = mid;
    }
    packed[s_glb[lo] + (p - s_loc[lo])] = s_out[p];
  }
}

// The 8-bit bucketing pass with its runs reserved by atomics: the region
// starts are already known (sums of the fine bucket histogram K1 took), so a
// tile ranks itself in shared memory and reserves each digit's run with ONE
// 64-bit atomic on that region's cursor -- no per-tile histogram pass over the
// keys and no scan of 256 x n_tiles counts before the scatter (prims.cuh
// bucket_pass_u32 needs both because it knows no totals). Order inside a
// region is arbitrary: the region scatter and the bucket sort re-rank.
__global__ void __launch_bounds__(kBucketThreads)
region_bucket_scatter_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                             uint64_t n, int shift,
                             unsigned long long* __restrict__ region_cursor /* [256] */,
                             uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out) {
  __shared__ uint32_t s_cnt[256], s_loc[256];
  __shared__ unsigned long long s_glb[256];
  __shared__ uint32_t s_key[kBucketTile], s_val[kBucketTile];
  const uint32_t t = threadIdx.x;
  if (t < 256) s_cnt[t] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kBucketTile;
  uint32_t k[kBucketPer], v[kBucketPer], r[kBucketPer];
#pragma unroll
  for (int q = 0; q < kBucketPer; ++q) {
    const uint64_t i = base + (uint64_t)q * kBucketThreads + t;
    if (i < n) {
      k[q] = keys[i];
      v[q] = vals[i];
      r[q] = atomicAdd(&s_cnt[(k[q] >> shift) & 255], 1u);
    }
  }
  __syncthreads();
  if (t < 32) {  // exclusive scan of the 256 tile counts, 8 per lane
    uint32_t c[8], s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c[j] = s_cnt[t * 8 + j];
      s += c[j];
    }
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (t >= (uint32_t)o) incl += u;
    }
    uint32_t run = incl - s;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s_loc[t * 8 + j] = run;
      run += c[j];
    }
  }
  if (t >= 32 && t < 288) {  // one reservation per (tile, digit)
    const uint32_t d = t - 32;
    if (s_cnt[d]) s_glb[d] = atomicAdd(&region_cursor[d], (unsigned long long)s_cnt[d]);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kBucketPer; ++q) {
    const uint64_t i = base + (uint64_t)q * kBucketThreads + t;
    if (i < n) {
      const uint32_t p = s_loc[(k[q] >> shift) & 255] + r[q];
      s_key[p] = k[q];
      s_val[p] = v[q];
    }
  }
  __syncthreads();
  const uint32_t in_tile = (uint32_t)((n - base) < (uint64_t)kBucketTile ? (n - base) : kBucketTile);
  for (uint32_t p = t; p < in_tile; p += kBucketThreads) {
    const uint32_t key = s_key[p], d = (key >> shift) & 255;
    const unsigned long long g = s_glb[d] + (p - s_loc[d]);
    keys_out[g] = key;
    vals_out[g] = s_val[p];
  }
}

// Region starts from the fine bucket starts: region d holds the buckets
// [d << sub_bits, (d + 1) << sub_bits); out[d] for the host's tile list,
// cursor[d] for the scatter's reservations.
__global__ void region_starts_kernel(const unsigned long long* __restrict__ bstart, uint32_t nb,
                                     int sub_bits, uint64_t* __restrict__ out /* [257] */,
                                     unsigned long long* __restrict__ cursor /* [256] */,
                                     uint32_t* __restrict__ tile_prefix /* [257] */) {
  __shared__ unsigned long long s_st[257];
  const uint32_t d = threadIdx.x;  // 288 threads
  if (d <= 256) {
    const uint64_t b = (uint64_t)d << sub_bits;
    const unsigned long long s = bstart[b < nb ? b : nb];
    s_st[d] = s;
    out[d] = s;
    if (d < 256) cursor[d] = s;
  }
  __syncthreads();
  if (d < 32) {  // exclusive prefix of the regions' tile counts, 8 regions per lane
    uint32_t c[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const unsigned long long len = s_st[d * 8 + j + 1] - s_st[d * 8 + j];
      c[j] = (uint32_t)((len + kRbTile - 1) / kRbTile);
      sum += c[j];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (d >= (uint32_t)o) incl += u;
    }
    uint32_t run = incl - sum;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      tile_prefix[d * 8 + j] = run;
      run += c[j];
    }
    if (d == 31) tile_prefix[256] = run;
  }
}

// In-place exclusive scan of a[0..n) in shared memory by the whole CTA
// (n <= kCbThreads * 8); returns the total. Uses ws[kCbThreads / 32].
__device__ __forceinline__ uint32_t cta_exclusive_scan(uint32_t* a, uint32_t n, uint32_t* ws) {
  const uint32_t per = (n + kCbThreads - 1) / kCbThreads;
  const uint32_t b0 = threadIdx.x * per;
  uint32_t loc = 0;
  for (uint32_t k = 0; k < per; ++k)
    if (b0 + k < n) loc += a[b0 + k];
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  uint32_t incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += u;
  }
  if (lane == 31) ws[w] = incl;
  __syncthreads();
  if (w == 0) {
    const uint32_t v = lane < kCbThreads / 32 ? ws[lane] : 0u;
    uint32_t wi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= (uint32_t)o) wi += u;
    }
    if (lane < kCbThreads / 32) ws[lane] = wi - v;  // exclusive over warps
    if (lane == kCbThreads / 32 - 1) ws[kCbThreads / 32] = wi;
  }
  __syncthreads();
  uint32_t run = ws[w] + incl - loc;
  for (uint32_t k = 0; k < per; ++k)
    if (b0 + k < n) {
      const uint32_t v = a[b0 + k];
      a[b0 + k] = run;
      run += v;
    }
  const uint32_t total = ws[kCbThreads / 32];
  __syncthreads();
  return total;
}

// Sort + unique a row of len entries at data[base..) (shared memory) by one
// warp, in place; returns the kept count. Rows past 256 entries (rare: the
// bucket capacity bounds them) use a rank sort into scratch[base..).
__device__ __forceinline__ uint32_t cb_sort_row(uint32_t* data, uint32_t* scratch, uint32_t base,
                                                uint32_t len) {
  if (len <= 32) return warp_sort_row<1>(data, base, len, true);
  if (len <= 64) return warp_sort_row<2>(data, base, len, true);
  if (len <= 128) return warp_sort_row<4>(data, base, len, true);
  if (len <= 256) return warp_sort_row<8>(data, base, len, true);
  const uint32_t lane = lane_id();
  for (uint32_t i = lane; i < len; i += 32) {
    const uint32_t v = data[base + i];
    uint32_t rank = 0;
    for (uint32_t j = 0; j < len; ++j) {
      const uint32_t u = data[base + j];
      rank += (u < v) || (u == v && j < i);
    }
    scratch[base + rank] = v;
  }
  __syncwarp();
  uint32_t written = 0;
  for (uint32_t i0 = 0; i0 < len; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint32_t v = i < len ? scratch[base + i] : 0u;
    const bool keep = i < len && (i == 0 || v != scratch[base + i - 1]);
    const uint32_t m = __ballot_sync(0xffffffffu, keep);
    if (keep) data[base + written + __popc(m & ((1u << lane) - 1))] = v;
    written += __popc(m);
  }
  __syncwarp();
  return written;
}

// K4: one CTA per bucket. Shared memory: keys[kCbCap] | rows[kCbCap] |
// roff[2^r + 1] | rcur[2^r] | ws[kCbThreads / 32 + 1].
__global__ void __launch_bounds__(kCbThreads)
csr_bucket_build_kernel(const uint32_t* __restrict__ packed,
                        const unsigned long long* __restrict__ bstart, uint64_t n_rows, int r,
                        int mb, uint32_t* __restrict__ uniq /* per bucket, at bstart */,
                        uint32_t* __restrict__ deg, unsigned long long* __restrict__ ustart,
                        unsigned long long* __restrict__ stats /* max deg, live rows */) {
  extern __shared__ uint32_t cbs[];
  uint32_t* keys = cbs;
  uint32_t* rowd = cbs + kCbCap;
  uint32_t* roff = rowd + kCbCap;
  uint32_t* rcur = roff + (1u << r) + 1;
  uint32_t* ws = rcur + (1u << r);
  const uint32_t b = blockIdx.x;
  const unsigned long long s0 = bstart[b];
  const uint32_t cnt = (uint32_t)(bstart[b + 1] - s0);
  const uint64_t row0 = (uint64_t)b << r;
  const uint32_t rows = (uint32_t)((n_rows - row0) < (1ull << r) ? (n_rows - row0) : (1ull << r));
  if (cnt == 0) {  // an empty bucket (an x shard's rows sit in one code range)
    for (uint32_t i = threadIdx.x; i < rows; i += kCbThreads) deg[row0 + i] = 0;
    if (threadIdx.x == 0) ustart[b] = 0;
    return;
  }
  const uint32_t mmask = mb >= 32 ? 0xffffffffu : ((1u << mb) - 1);
  for (uint32_t i = threadIdx.x; i <= rows; i += kCbThreads) roff[i] = 0;
  // the bucket's keys into shared memory: 16-byte loads from the first
  // aligned key on, all issued before any is consumed
  const uint32_t head = (uint32_t)((4 - (s0 & 3)) & 3) < cnt ? (uint32_t)((4 - (s0 & 3)) & 3) : cnt;
  const uint32_t nv = (cnt - head) / 4;
  const uint4* pv = reinterpret_cast<const uint4*>(packed + s0 + head);
  for (uint32_t v0 = threadIdx.x; v0 < nv; v0 += kCbThreads * 4) {
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v0 + u * kCbThreads < nv) q[u] = pv[v0 + u * kCbThreads];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v0 + u * kCbThreads < nv) {
        const uint32_t i = head + 4 * (v0 + u * kCbThreads);
        keys[i] = q[u].x;
        keys[i + 1] = q[u].y;
        keys[i + 2] = q[u].z;
        keys[i + 3] = q[u].w;
      }
  }
  for (uint32_t i = threadIdx.x; i < head; i += kCbThreads) keys[i] = packed[s0 + i];
  for (uint32_t i = head + 4 * nv + threadIdx.x; i < cnt; i += kCbThreads) keys[i] = packed[s0 + i];
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < cnt; i += kCbThreads) atomicAdd(&roff[keys[i] >> mb], 1u);
  __syncthreads();
  cta_exclusive_scan(roff, rows + 1, ws);  // roff[rows] = cnt
  for (uint32_t i = threadIdx.x; i < rows; i += kCbThreads) rcur[i] = roff[i];
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < cnt; i += kCbThreads) {
    const uint32_t k = keys[i];
    rowd[atomicAdd(&rcur[k >> mb], 1u)] = k & mmask;
  }
  __syncthreads();
  // per-row sort + unique; kept counts into rcur. Short rows (the common
  // case: ~20 entries) by one thread each -- an insertion sort in shared
  // memory costs ~len^2/4 moves, far fewer issued instructions than a warp
  // bitonic network per row; rows past kCbThreadRow entries by a warp.
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  uint32_t mx = 0, live = 0;
  for (uint32_t q = threadIdx.x; q < rows; q += kCbThreads) {
    const uint32_t base = roff[q], len = roff[q + 1] - base;
    if (len > kCbThreadRow) continue;
    uint32_t* a = rowd + base;
    for (uint32_t i = 1; i < len; ++i) {
      const uint32_t v = a[i];
      uint32_t j = i;
      while (j > 0 && a[j - 1] > v) {
        a[j] = a[j - 1];
        --j;
      }
      a[j] = v;
    }
    uint32_t kept = len ? 1u : 0u;
    for (uint32_t i = 1; i < len; ++i)
      if (a[i] != a[kept - 1]) a[kept++] = a[i];
    rcur[q] = kept;
    deg[row0 + q] = kept;
    mx = kept > mx ? kept : mx;
    live += kept > 0;
  }
  // rows of <= 32 entries: two per warp (one per half)
  for (uint32_t q0 = 2 * w; q0 < rows; q0 += 2 * (kCbThreads / 32)) {
    const uint32_t q = q0 + (lane >> 4);
    uint32_t base = 0, len = 0;
    if (q < rows) {
      base = roff[q];
      len = roff[q + 1] - base;
    }
    const bool mine = q < rows && len > kCbThreadRow && len <= 32;
    const uint32_t kept = half_sort_row32(rowd, base, mine ? len : 0u, true);
    if (mine && (lane & 15) == 0) {
      rcur[q] = kept;
      deg[row0 + q] = kept;
      mx = kept > mx ? kept : mx;
      live += kept > 0;
    }
  }
  for (uint32_t q = w; q < rows; q += kCbThreads / 32) {
    const uint32_t base = roff[q], len = roff[q + 1] - base;
    if (len <= 32) continue;  // warp-uniform
    const uint32_t kept = cb_sort_row(rowd, keys, base, len);
    if (lane == 0) {
      rcur[q] = kept;
      deg[row0 + q] = kept;
      mx = kept > mx ? kept : mx;
      live += 1;
    }
  }
  __syncthreads();
  // bucket-local compaction: unique offsets of the rows
  for (uint32_t i = threadIdx.x; i < rows; i += kCbThreads) keys[i] = rcur[i];
  __syncthreads();
  const uint32_t total = cta_exclusive_scan(keys, rows, ws);
  for (uint32_t q = w; q < rows; q += kCbThreads / 32) {
    const uint32_t src = roff[q], dst = keys[q], kept = rcur[q];
    for (uint32_t j = lane; j < kept; j += 32) uniq[s0 + dst + j] = rowd[src + j];
  }
  if (threadIdx.x == 0) ustart[b] = total;
  mx = warp_max(mx);  // (per-row values sit in lanes 0 and 16 and the thread-row lanes)
  live = warp_sum(live);
  if (lane == 0) {
    if (mx) atomicMax(&stats[0], (unsigned long long)mx);
    if (live) atomicAdd(&stats[1], (unsigned long long)live);
  }
}

// K6: bucket b's unique run -> col[row_ptr[b << r] ..). One CTA per bucket.
__global__ void __launch_bounds__(kCbThreads)
csr_bucket_copy_kernel(const uint32_t* __restrict__ uniq, const unsigned long long* __restrict__ bstart,
                       const unsigned long long* __restrict__ ucount,
                       const uint64_t* __restrict__ row_ptr, int r, uint32_t* __restrict__ col) {
  const uint32_t b = blockIdx.x;
  const uint64_t s0 = bstart[b], n = ucount[b], d0 = row_ptr[(uint64_t)b << r];
  for (uint64_t j = threadIdx.x; j < n; j += kCbThreads) col[d0 + j] = uniq[s0 + j];
}

inline size_t csr_bucket_smem(int r) {
  return ((size_t)2 * kCbCap + (1u << r) * 2 + 1 + kCbThreads / 32 + 1) * 4;
}

// Returns false (nothing built) when the bucketed path does not apply: the
// packed key does not fit 32 bits, too many buckets, or a bucket exceeds
// the shared-memory capacity (skewed majors).
inline bool build_csr_bucketed(Ctx& ctx, const uint32_t* maj, const uint32_t* mnr, uint64_t n,
                               uint64_t n_rows, uint64_t n_cols, DeviceCsr& out, bool force) {
  if ((!force && n < (1ull << 16)) || n == 0 || n >= (1ull << 32) || n_rows == 0) return false;
  const int mb = std::max(1, bits_for(n_cols ? n_cols - 1 : 0));
  if (mb > 31) return false;
  // rows per bucket: ~kCbTarget tuples, packed key within 32 bits. Long
  // average rows (> 64 tuples) go to the scatter path, whose CTA-wide
  // shared-memory sorts suit them (the bucket kernel sorts rows by warps)
  const double per_row = (double)n / (double)n_rows;
  if (!force && per_row > 64.0) return false;
  int r = 0;
  while (r < (int)kCbMaxRowsLog && r + 1 + mb <= 32 && per_row * (double)(1ull << (r + 1)) <= kCbTarget)
    ++r;
  // fewer, fuller buckets when there would be too many for K1's histogram
  while (((n_rows + (1ull << r) - 1) >> r) > kCbMaxBuckets && r < (int)kCbMaxRowsLog &&
         r + 1 + mb <= 32)
    ++r;
  if (r + mb > 32 || per_row * (double)(1ull << r) > 0.9 * kCbCap) return false;
  // The rows may be far from uniform (an x shard of R: its x sit in one code
  // range of a job-sized row space): when the fullest bucket overflows the
  // shared-memory capacity, halve the bucket (up to 3 times) before giving up
  // to the scatter path.
  uint32_t nb = 0;
  DBuf<unsigned int> hist;
  DBuf<unsigned long long> bstart;
  for (int attempt = 0;; ++attempt) {
    const uint64_t nb64 = (n_rows + (1ull << r) - 1) >> r;
    if (nb64 > kCbMaxBuckets) return false;
    nb = (uint32_t)nb64;
    hist = ctx.zeros<unsigned int>(nb);
    const unsigned g = (unsigned)std::min<uint64_t>(ctx.sm_count * 2ull, (n + kCbThreads - 1) / kCbThreads);
    const size_t hsm = (size_t)nb * 4;
    // (the attribute is per function, shared by every context of the process:
    // set to the largest size any call uses, so concurrent calls -- ranks as
    // threads -- never launch above another call's setting)
    D3G_CUDA(raise_smem_attr(csr_bucket_hist_kernel, (int)((size_t)kCbMaxBuckets * 4)));
    D3G_LAUNCH(ctx, csr_bucket_hist_kernel, g, kCbThreads, hsm, maj, n, r, nb, hist.p);
    DBuf<unsigned long long> mxb = ctx.zeros<unsigned long long>(1);
    D3G_LAUNCH(ctx, max_u32_kernel, grid_for(nb, 256), 256, 0, hist.p, (uint64_t)nb, mxb.p);
    const unsigned long long mx = ctx.scalar(mxb.p);
    if (mx <= kCbCap) break;
    if (attempt == 3 || r == 0) return false;
    r = std::max(0, r - std::max(1, (int)std::ceil(std::log2((double)mx / (0.9 * kCbCap)))));
  }
  bstart = ctx.alloc<unsigned long long>(nb + 1);
  exclusive_scan<unsigned int>(ctx, hist.p, nb, reinterpret_cast<uint64_t*>(bstart.p));
  DBuf<unsigned long long> cursor = ctx.alloc<unsigned long long>(nb);
  D3G_CUDA(cudaMemcpyAsync(cursor.p, bstart.p, (size_t)nb * 8, cudaMemcpyDeviceToDevice, ctx.stream));
  DBuf<uint32_t> packed = ctx.alloc<uint32_t>(n);
  const char* sc = std::getenv("D3G_CSR_SCATTER");
  if (sc && std::strcmp(sc, "atomic") == 0) {  // K3: one global atomic per pair (comparison)
    D3G_LAUNCH(ctx, csr_bucket_scatter_kernel, grid_for(n, kCbThreads, ctx.sm_count * 8),
               kCbThreads, 0, maj, mnr, n, r, mb, cursor.p, packed.p);
  } else {
    // two levels: an 8-bit bucketing pass on the high bucket bits, then the
    // region-local tile scatter with one atomic per (tile, bucket)
    const int bucket_bits = std::max(1, bits_for(nb - 1));
    const int sub_bits = std::max(0, bucket_bits - 8);
    DBuf<uint32_t> am = ctx.alloc<uint32_t>(n), av = ctx.alloc<uint32_t>(n);
    const uint32_t n_tiles = (uint32_t)((n + kBucketTile - 1) / kBucketTile);
    {
      DBuf<uint64_t> rs = ctx.alloc<uint64_t>(257);
      DBuf<unsigned long long> rcur = ctx.alloc<unsigned long long>(256);
      DBuf<uint32_t> tpre = ctx.alloc<uint32_t>(257);
      D3G_LAUNCH(ctx, region_starts_kernel, 1, 288, 0, bstart.p, nb, sub_bits, rs.p, rcur.p,
                 tpre.p);
      D3G_LAUNCH(ctx, region_bucket_scatter_kernel, n_tiles, kBucketThreads, 0, maj, mnr, n,
                 r + sub_bits, rcur.p, am.p, av.p);
      // (every region's last tile may be partial: at most 256 more tiles than n / kRbTile)
      D3G_LAUNCH(ctx, csr_region_scatter_kernel, (unsigned)(n / kRbTile + 257), kRbThreads, 0,
                 am.p, av.p, rs.p, tpre.p, r, mb, sub_bits, cursor.p, packed.p);
    }
  }
  cursor.reset();
  DBuf<uint32_t> uniq = ctx.alloc<uint32_t>(n);
  DBuf<uint32_t> deg = ctx.alloc<uint32_t>(n_rows);
  DBuf<unsigned long long> ucount = ctx.alloc<unsigned long long>(nb);
  DBuf<unsigned long long> st = ctx.zeros<unsigned long long>(2);
  const size_t bsm = csr_bucket_smem(r);
  D3G_CUDA(raise_smem_attr(csr_bucket_build_kernel, (int)csr_bucket_smem((int)kCbMaxRowsLog)));  // (see above)
  D3G_LAUNCH(ctx, csr_bucket_build_kernel, nb, kCbThreads, bsm, packed.p, bstart.p, n_rows, r, mb,
             uniq.p, deg.p, ucount.p, st.p);
  packed.reset();
  out.n_rows = n_rows;
  out.n_cols = n_cols;
  out.row_ptr = ctx.alloc<uint64_t>(n_rows + 1);
  exclusive_scan<uint32_t>(ctx, deg.p, n_rows, out.row_ptr.p);
  unsigned long long hs[2];
  ctx.defer(&out.nnz, out.row_ptr.p + n_rows, 8);
  ctx.defer(hs, st.p, 16);
  ctx.sync();
  out.max_deg = hs[0];
  out.live_rows = hs[1];
  out.col = ctx.alloc<uint32_t>(out.nnz);
  D3G_LAUNCH(ctx, csr_bucket_copy_kernel, nb, kCbThreads, 0, uniq.p, bstart.p, ucount.p,
             out.row_ptr.p, r, out.col.p);
  return true;
}

}  // namespace d3g
