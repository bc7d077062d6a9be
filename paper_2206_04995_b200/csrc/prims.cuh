// Device primitives: tiled exclusive scan (u64 result) and a stable LSD
// radix sort of (u64 key, u32 value) pairs with warp multi-split ranking.
// These are the building blocks for the CSR grouping (counting scatter +
// row offsets), the dictionary code assignment and output ordering.
#pragma once

#include "common.cuh"

namespace d3g {

// ---------------------------------------------------------------------------
// Exclusive scan: out[i] = sum(in[0..i)), out[n] = total; one tile in one
// block, larger inputs in one single-pass launch (decoupled look-back).
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

// Block-wide exclusive scan of one value per thread; returns the prefix and
// writes the block total to *total.
__device__ __forceinline__ uint64_t block_exclusive_scan(uint64_t v, uint64_t* total) {
  __shared__ uint64_t warp_tot[32];
  __shared__ uint64_t block_tot;
  uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += u;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t nw = blockDim.x >> 5;
    uint64_t t = lane < nw ? warp_tot[lane] : 0;
    uint64_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t u = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= (uint32_t)o) ti += u;
    }
    if (lane < nw) warp_tot[lane] = ti - t;
    if (lane == nw - 1) block_tot = ti;
  }
  __syncthreads();
  uint64_t res = warp_tot[warp] + incl - v;
  if (total) *total = block_tot;
  __syncthreads();
  return res;
}

template <class Tin>
__global__ void __launch_bounds__(kScanThreads)
scan_tile_kernel(const Tin* __restrict__ in, uint64_t n, const uint64_t* __restrict__ offsets,
                 uint64_t* __restrict__ out) {
  uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint64_t vals[kScanItems];
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    uint64_t i = base + k;
    vals[k] = i < n ? (uint64_t)in[i] : 0;
    s += vals[k];
  }
  uint64_t tot;
  uint64_t run = block_exclusive_scan(s, &tot) + (offsets ? offsets[blockIdx.x] : 0);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    uint64_t i = base + k;
    if (i < n) out[i] = run;
    run += vals[k];
  }
  // the last element of the whole array writes out[n]
  uint64_t last_tile = n == 0 ? 0 : (n - 1) / kScanTile;
  if (blockIdx.x == last_tile && threadIdx.x == blockDim.x - 1)
    out[n] = tot + (offsets ? offsets[blockIdx.x] : 0);
}

// Single-pass exclusive scan with decoupled look-back: tiles take tickets in
// launch order, publish their aggregate, and warp 0 of each tile walks back
// over its predecessors 32 at a time until it meets an inclusive prefix.
// state[t] = flag << 61 | value, flag = 1 + 2*parity (aggregate) or
// 2 + 2*parity (inclusive prefix); entries of the other parity (the previous
// scan) read as "not yet published". The state persists across scans
// (Ctx::scan_state): tickets count up from `ticket0`, and the blocks clear
// the entries in [tiles, hw) that an earlier, longer scan left behind, so the
// next scan (other parity) sees only its own or empty entries. One launch, no
// memset.
template <class Tin>
__global__ void __launch_bounds__(kScanThreads)
scan_onepass_kernel(const Tin* __restrict__ in, uint64_t n, uint64_t* __restrict__ out,
                    unsigned long long* __restrict__ state, uint32_t tiles,
                    unsigned long long* __restrict__ ticket, unsigned long long ticket0,
                    uint32_t parity, uint32_t hw) {
  const unsigned long long kAgg = (1ull + 2 * parity) << 61, kPre = (2ull + 2 * parity) << 61;
  constexpr unsigned long long kVal = (1ull << 61) - 1;
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_excl;
  if (threadIdx.x == 0) s_tile = (uint32_t)(atomicAdd(ticket, 1ull) - ticket0);
  for (uint64_t t = (uint64_t)tiles + blockIdx.x * blockDim.x + threadIdx.x; t < hw;
       t += (uint64_t)gridDim.x * blockDim.x)
    state[t] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = (uint64_t)tile * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint64_t vals[kScanItems];
  uint64_t sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t i = base + k;
    vals[k] = i < n ? (uint64_t)in[i] : 0;
    sum += vals[k];
  }
  uint64_t tot;
  const uint64_t local = block_exclusive_scan(sum, &tot);
  if (threadIdx.x == 0) {
    if (tile == 0) {
      atomicExch(&state[0], kPre | tot);
      s_excl = 0;
    } else {
      atomicExch(&state[tile], kAgg | tot);
    }
  }
  if (tile > 0 && threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    uint64_t excl = 0;
    int64_t t = (int64_t)tile - 1;
    for (;;) {
      const int64_t my = t - (int64_t)lane;
      unsigned long long st = kPre;  // before tile 0: an empty prefix
      if (my >= 0) {
        do {
          st = atomicAdd(&state[my], 0ull);
        } while ((st & ~kVal) != kAgg && (st & ~kVal) != kPre);
      }
      const unsigned pre = __ballot_sync(0xffffffffu, (st & ~kVal) == kPre);
      const int first = pre ? __ffs(pre) - 1 : 32;
      excl += warp_sum((uint64_t)((int)lane <= first && my >= 0 ? (st & kVal) : 0));
      if (pre) break;
      t -= 32;
    }
    if (lane == 0) {
      atomicExch(&state[tile], kPre | (excl + tot));
      s_excl = excl;
    }
  }
  __syncthreads();
  uint64_t run = s_excl + local;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t i = base + k;
    if (i < n) out[i] = run;
    run += vals[k];
  }
  if (tile == tiles - 1 && threadIdx.x == blockDim.x - 1) out[n] = s_excl + tot;
}

// out must hold n + 1 entries. Returns nothing; out[n] is the total.
template <class Tin>
void exclusive_scan(Ctx& ctx, const Tin* in, uint64_t n, uint64_t* out) {
  if (n == 0) {
    D3G_CUDA(cudaMemsetAsync(out, 0, sizeof(uint64_t), ctx.stream));
    return;
  }
  uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles == 1) {
    D3G_LAUNCH(ctx, scan_tile_kernel<Tin>, 1, kScanThreads, 0, in, n,
               (const uint64_t*)nullptr, out);
    return;
  }
  if (tiles >= (1ull << 31)) throw ResourceError("exclusive_scan: too many tiles");
  ctx.scan_reserve(tiles);
  const uint64_t hw = ctx.scan_hw > tiles ? ctx.scan_hw : tiles;
  D3G_LAUNCH(ctx, scan_onepass_kernel<Tin>, (unsigned)tiles, kScanThreads, 0, in, n, out,
             ctx.scan_state, (uint32_t)tiles, ctx.scan_state + ctx.scan_cap, ctx.scan_tickets,
             ctx.scan_parity, (uint32_t)hw);
  ctx.scan_tickets += tiles;
  ctx.scan_parity ^= 1u;
  ctx.scan_hw = tiles;
}

// ---------------------------------------------------------------------------
// Stable LSD radix sort, 8-bit digits. Each tile of kSortTile keys is split
// into per-warp contiguous chunks; warps rank keys with __match_any_sync so
// the scatter is stable (global index order within each digit).
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortPerLane = 8;
constexpr int kSortChunk = 32 * kSortPerLane;           // keys per warp
constexpr int kSortTile = kSortWarps * kSortChunk;      // 2048 keys per block

template <class KT = uint64_t>
__global__ void __launch_bounds__(kSortThreads)
radix_hist_kernel(const KT* __restrict__ keys, uint64_t n, int shift, uint32_t n_tiles,
                  uint32_t* __restrict__ hist) {
  __shared__ uint32_t cnt[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  uint64_t base = (uint64_t)blockIdx.x * kSortTile;
  for (int k = threadIdx.x; k < kSortTile; k += blockDim.x) {
    uint64_t i = base + k;
    if (i < n) atomicAdd(&cnt[(keys[i] >> shift) & 255], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x)
    hist[(uint64_t)d * n_tiles + blockIdx.x] = cnt[d];
}

template <bool kHasVals, class KT = uint64_t>
__global__ void __launch_bounds__(kSortThreads)
radix_scatter_kernel(const KT* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                     uint64_t n, int shift, uint32_t n_tiles,
                     const uint64_t* __restrict__ offsets,  // scanned hist, digit-major
                     KT* __restrict__ keys_out, uint32_t* __restrict__ vals_out) {
  __shared__ uint32_t whist[kSortWarps][256];
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSortWarps * 256; i += blockDim.x) (&whist[0][0])[i] = 0;
  __syncthreads();
  const uint64_t chunk = (uint64_t)blockIdx.x * kSortTile + (uint64_t)warp * kSortChunk;
  KT k[kSortPerLane];
  uint32_t v[kSortPerLane];
  uint32_t rank[kSortPerLane];
  const uint32_t lt = (1u << lane) - 1;
#pragma unroll
  for (int it = 0; it < kSortPerLane; ++it) {
    uint64_t i = chunk + (uint64_t)it * 32 + lane;
    bool valid = i < n;
    k[it] = valid ? keys_in[i] : 0;
    if (kHasVals) v[it] = valid ? vals_in[i] : 0;
    uint32_t d = valid ? (uint32_t)((k[it] >> shift) & 255) : 256u;
    uint32_t active = __ballot_sync(0xffffffffu, valid);
    uint32_t peers = __match_any_sync(0xffffffffu, d) & active;
    uint32_t before = 0;
    if (valid) before = whist[warp][d];
    __syncwarp();
    if (valid) {
      rank[it] = before + __popc(peers & lt);
      if ((peers & lt) == 0) whist[warp][d] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive scan across warps, plus the tile's global offset
  for (int d = threadIdx.x; d < 256; d += blockDim.x) {
    uint64_t run = offsets[(uint64_t)d * n_tiles + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      uint32_t t = whist[w][d];
      whist[w][d] = (uint32_t)run;  // low 32 bits; positions fit (n < 2^32)
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kSortPerLane; ++it) {
    uint64_t i = chunk + (uint64_t)it * 32 + lane;
    if (i < n) {
      uint32_t d = (uint32_t)((k[it] >> shift) & 255);
      uint32_t pos = whist[warp][d] + rank[it];
      keys_out[pos] = k[it];
      if (kHasVals) vals_out[pos] = v[it];
    }
  }
}

// Sorts keys (and vals, if non-null) by the low `bits` bits of the key.
// Ping-pongs through scratch buffers; the sorted result ends up back in
// keys/vals (keys left unspecified when !keys_needed). Requires n < 2^32.
inline void radix_sort(Ctx& ctx, uint64_t* keys, uint32_t* vals, uint64_t n, int bits,
                       bool keys_needed = true) {
  if (n <= 1 || bits <= 0) return;
  if (n >= (1ull << 32)) throw ResourceError("radix_sort: more than 2^32 keys");
  uint32_t n_tiles = (uint32_t)((n + kSortTile - 1) / kSortTile);
  DBuf<uint64_t> k2 = ctx.alloc<uint64_t>(n);
  DBuf<uint32_t> v2 = ctx.alloc<uint32_t>(vals ? n : 1);
  DBuf<uint32_t> hist = ctx.alloc<uint32_t>((uint64_t)256 * n_tiles);
  DBuf<uint64_t> offs = ctx.alloc<uint64_t>((uint64_t)256 * n_tiles + 1);
  uint64_t* kin = keys;
  uint32_t* vin = vals;
  uint64_t* kout = k2.p;
  uint32_t* vout = v2.p;
  int passes = (bits + 7) / 8;
  for (int p = 0; p < passes; ++p) {
    int shift = 8 * p;
    D3G_LAUNCH(ctx, radix_hist_kernel<uint64_t>, n_tiles, kSortThreads, 0, kin, n, shift, n_tiles, hist.p);
    exclusive_scan<uint32_t>(ctx, hist.p, (uint64_t)256 * n_tiles, offs.p);
    if (vals)
      D3G_LAUNCH(ctx, (radix_scatter_kernel<true, uint64_t>), n_tiles, kSortThreads, 0, kin, vin, n, shift,
                 n_tiles, offs.p, kout, vout);
    else
      D3G_LAUNCH(ctx, (radix_scatter_kernel<false, uint64_t>), n_tiles, kSortThreads, 0, kin, vin, n, shift,
                 n_tiles, offs.p, kout, vout);
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  if (kin != keys) {
    if (keys_needed || !vals)
      D3G_CUDA(cudaMemcpyAsync(keys, kin, n * 8, cudaMemcpyDeviceToDevice, ctx.stream));
    if (vals) D3G_CUDA(cudaMemcpyAsync(vals, vin, n * 4, cudaMemcpyDeviceToDevice, ctx.stream));
  }
}

// One stable 8-bit LSD pass over u32 (key, value) pairs: digit (key >> shift)
// & 255. Used to bucket a large CSR build by its high row bits first, so the
// per-row scatter that follows writes into an L2-sized window.
inline void radix_pass_u32(Ctx& ctx, const uint32_t* keys, const uint32_t* vals, uint64_t n,
                           int shift, uint32_t* keys_out, uint32_t* vals_out) {
  if (n == 0) return;
  if (n >= (1ull << 32)) throw ResourceError("radix_pass_u32: more than 2^32 keys");
  const uint32_t n_tiles = (uint32_t)((n + kSortTile - 1) / kSortTile);
  DBuf<uint32_t> hist = ctx.alloc<uint32_t>((uint64_t)256 * n_tiles);
  DBuf<uint64_t> offs = ctx.alloc<uint64_t>((uint64_t)256 * n_tiles + 1);
  D3G_LAUNCH(ctx, radix_hist_kernel<uint32_t>, n_tiles, kSortThreads, 0, keys, n, shift, n_tiles,
             hist.p);
  exclusive_scan<uint32_t>(ctx, hist.p, (uint64_t)256 * n_tiles, offs.p);
  D3G_LAUNCH(ctx, (radix_scatter_kernel<true, uint32_t>), n_tiles, kSortThreads, 0, keys, vals, n,
             shift, n_tiles, offs.p, keys_out, vals_out);
}

// Unstable one-pass bucketing of u32 (key, value) pairs by the 8-bit digit
// (key >> shift) & 255, for callers that re-sort inside each bucket (the
// large CSR build). A CTA ranks its tile in shared memory (per-digit
// counters), stages the tile in digit order and writes it out in runs, so the
// global writes are contiguous per digit instead of scattered per element.
constexpr int kBucketThreads = 1024;
constexpr int kBucketPer = 4;
constexpr int kBucketTile = kBucketThreads * kBucketPer;  // 4096 pairs per CTA

__global__ void __launch_bounds__(kBucketThreads)
bucket_hist_kernel(const uint32_t* __restrict__ keys, uint64_t n, int shift, uint32_t n_tiles,
                   uint32_t* __restrict__ hist /* [256][n_tiles] */) {
  __shared__ uint32_t cnt[256];
  if (threadIdx.x < 256) cnt[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kBucketTile;
#pragma unroll
  for (int k = 0; k < kBucketPer; ++k) {
    const uint64_t i = base + (uint64_t)k * kBucketThreads + threadIdx.x;
    if (i < n) atomicAdd(&cnt[(keys[i] >> shift) & 255], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 256) hist[(uint64_t)threadIdx.x * n_tiles + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(kBucketThreads)
bucket_scatter_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                      uint64_t n, int shift, uint32_t n_tiles,
                      const uint64_t* __restrict__ offsets /* scanned hist, digit-major */,
                      uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out) {
  __shared__ uint32_t s_cnt[256], s_loc[256];
  __shared__ uint64_t s_glb[256];
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
  if (t < 256) s_glb[t] = offsets[(uint64_t)t * n_tiles + blockIdx.x];
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
    const uint64_t g = s_glb[d] + (p - s_loc[d]);
    keys_out[g] = key;
    vals_out[g] = s_val[p];
  }
}

// Unstable bucketing by one 8-bit digit (see bucket_scatter_kernel).
inline void bucket_pass_u32(Ctx& ctx, const uint32_t* keys, const uint32_t* vals, uint64_t n,
                            int shift, uint32_t* keys_out, uint32_t* vals_out) {
  if (n == 0) return;
  if (n >= (1ull << 32)) throw ResourceError("bucket_pass_u32: more than 2^32 keys");
  const uint32_t n_tiles = (uint32_t)((n + kBucketTile - 1) / kBucketTile);
  DBuf<uint32_t> hist = ctx.alloc<uint32_t>((uint64_t)256 * n_tiles);
  DBuf<uint64_t> offs = ctx.alloc<uint64_t>((uint64_t)256 * n_tiles + 1);
  D3G_LAUNCH(ctx, bucket_hist_kernel, n_tiles, kBucketThreads, 0, keys, n, shift, n_tiles, hist.p);
  exclusive_scan<uint32_t>(ctx, hist.p, (uint64_t)256 * n_tiles, offs.p);
  D3G_LAUNCH(ctx, bucket_scatter_kernel, n_tiles, kBucketThreads, 0, keys, vals, n, shift, n_tiles,
             offs.p, keys_out, vals_out);
}

__global__ void index_compact_kernel(const uint32_t* __restrict__ flag,
                                     const uint64_t* __restrict__ pos, uint64_t n,
                                     uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (flag[i]) out[pos[i]] = (uint32_t)i;
}

inline int bits_for(uint64_t max_value) {
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b;
}

}  // namespace d3g
