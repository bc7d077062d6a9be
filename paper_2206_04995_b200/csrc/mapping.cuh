// Value mapping on the GPU (north_star subsystem 1).
//
// * Natural-key probe + full max scan: detect_natural_keys
//   (P/src/mapping.cpp:281-295) and require_natural (:328-338).
// * Dictionary: an open-addressing table in HBM (linear probing, u64 keys)
//   built with atomicCAS, recording the first row index of every distinct
//   value with atomicMin. Codes are then assigned exactly as the reference's
//   Dictionary::build_partitioned does (P/src/mapping.cpp:191-251): values
//   belong to partition mix64(v) & (2^k - 1) with k = partition_bits_for(n)
//   (:308-316); partitions are numbered in order and, within a partition,
//   values are numbered first-seen. On the GPU that is one radix sort of the
//   distinct values by (partition, first index). Same codes as the reference
//   => identical CSR structure and identical per-x/per-z degrees.
#pragma once

#include "prims.cuh"

namespace d3g {

constexpr uint64_t kEmptyKey = ~0ull;
constexpr uint32_t kNoRow = 0xffffffffu;

// ---------------------------------------------------------------------------
// Column statistics: max over the column and the 4096-sample natural test.
struct ColStat {
  unsigned long long max;
  unsigned int sample_fail;  // 1 if any strided sample >= 2 * n
  unsigned int pad;
};

__global__ void colstat_kernel(const uint64_t* __restrict__ col, uint64_t n, ColStat* st) {
  uint64_t m = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t v = col[i];
    m = v > m ? v : m;
  }
  m = warp_max(m);
  if (lane_id() == 0 && m) atomicMax(&st->max, (unsigned long long)m);
  if (blockIdx.x == 0) {
    // detect_natural_keys: samples = min(n, 4096), stride = max(n/samples,1),
    // sample i reads col[min(i*stride, n-1)], fails when (double)v >= 2n.
    uint64_t samples = n < 4096 ? n : 4096;
    uint64_t stride = samples ? n / samples : 1;
    if (stride < 1) stride = 1;
    double bound = 2.0 * (double)n;
    for (uint64_t i = threadIdx.x; i < samples; i += blockDim.x) {
      uint64_t idx = i * stride;
      if (idx > n - 1) idx = n - 1;
      if ((double)col[idx] >= bound) st->sample_fail = 1;
    }
  }
}

// All four input columns in one launch (blockIdx.y = column): max, the
// detect_natural_keys sample test, and the speculative u32 narrowing the
// natural-key mapping uses (codes = values), written while the values stream
// by so a natural column is read exactly once.
struct Cols4 {
  const uint64_t* col[4];
  uint64_t n[4];
  uint32_t* narrow[4];
  uint64_t bound_n[4];  // the sample test's n (the global |R| for an R shard)
};

__global__ void __launch_bounds__(256) colstat4_kernel(Cols4 c, ColStat* st) {
  const int ci = blockIdx.y;
  const uint64_t* __restrict__ col = c.col[ci];
  uint32_t* __restrict__ out = c.narrow[ci];
  const uint64_t n = c.n[ci];
  uint64_t m = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {  // 4 independent loads in flight
    const uint64_t v0 = col[i], v1 = col[i + stride], v2 = col[i + 2 * stride],
                   v3 = col[i + 3 * stride];
    out[i] = (uint32_t)v0;
    out[i + stride] = (uint32_t)v1;
    out[i + 2 * stride] = (uint32_t)v2;
    out[i + 3 * stride] = (uint32_t)v3;
    const uint64_t a = v0 > v1 ? v0 : v1, b = v2 > v3 ? v2 : v3;
    const uint64_t ab = a > b ? a : b;
    m = ab > m ? ab : m;
  }
  for (; i < n; i += stride) {
    const uint64_t v = col[i];
    out[i] = (uint32_t)v;
    m = v > m ? v : m;
  }
  m = warp_max(m);
  if (lane_id() == 0 && m) atomicMax(&st[ci].max, (unsigned long long)m);
  if (blockIdx.x == 0) {
    uint64_t samples = n < 4096 ? n : 4096;
    uint64_t sstride = samples ? n / samples : 1;
    if (sstride < 1) sstride = 1;
    double bound = 2.0 * (double)c.bound_n[ci];
    for (uint64_t k = threadIdx.x; k < samples; k += blockDim.x) {
      uint64_t idx = k * sstride;
      if (idx > n - 1) idx = n - 1;
      if ((double)col[idx] >= bound) st[ci].sample_fail = 1;
    }
  }
}

// ---------------------------------------------------------------------------
// Dictionary.
struct DeviceDict {
  bool identity = true;
  uint64_t card = 0;
  DBuf<uint64_t> rev;        // code -> value (dictionary only)
  DBuf<uint64_t> keys;       // table keys, capacity + 1 (last = sentinel slot)
  DBuf<uint32_t> slot_code;  // code per slot (after assignment)
  uint64_t mask = 0;         // capacity - 1
};

__device__ __forceinline__ uint64_t dict_slot_of(uint64_t h, uint64_t mask) {
  return (h ^ (h >> 29)) & mask;
}

__global__ void dict_insert_kernel(const uint64_t* __restrict__ vals, uint64_t n,
                                   unsigned long long* __restrict__ keys,
                                   uint32_t* __restrict__ first, uint64_t mask) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t v = vals[i];
    if (v == kEmptyKey) {  // the sentinel value lives in the extra slot
      atomicMin(&first[mask + 1], (uint32_t)i);
      continue;
    }
    uint64_t s = dict_slot_of(mix64(v), mask);
    for (;;) {
      unsigned long long k = keys[s];
      if (k == v) break;
      if (k == kEmptyKey) {
        unsigned long long prev = atomicCAS(&keys[s], kEmptyKey, (unsigned long long)v);
        if (prev == kEmptyKey || prev == v) break;
      }
      s = (s + 1) & mask;
    }
    atomicMin(&first[s], (uint32_t)i);
  }
}

// Occupied slots -> (sort key, slot). sort key = partition << 32 | first row.
__global__ void dict_collect_kernel(const uint64_t* __restrict__ keys,
                                    const uint32_t* __restrict__ first, uint64_t slots,
                                    int part_bits, const uint64_t* __restrict__ pos,
                                    uint64_t* __restrict__ sort_keys,
                                    uint32_t* __restrict__ sort_slots) {
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < slots;
       s += (uint64_t)gridDim.x * blockDim.x) {
    if (first[s] == kNoRow) continue;
    uint64_t v = (s == slots - 1) ? kEmptyKey : keys[s];
    uint64_t part = part_bits == 0 ? 0 : (mix64(v) & ((1ull << part_bits) - 1));
    uint64_t o = pos[s];
    sort_keys[o] = (part << 32) | first[s];
    sort_slots[o] = (uint32_t)s;
  }
}

__global__ void occupied_flag_kernel(const uint32_t* __restrict__ first, uint64_t slots,
                                     uint32_t* __restrict__ flag) {
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < slots;
       s += (uint64_t)gridDim.x * blockDim.x)
    flag[s] = first[s] != kNoRow;
}

__global__ void dict_assign_kernel(const uint32_t* __restrict__ sorted_slots, uint64_t distinct,
                                   const uint64_t* __restrict__ keys, uint64_t slots,
                                   uint32_t* __restrict__ slot_code, uint64_t* __restrict__ rev) {
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < distinct;
       c += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t s = sorted_slots[c];
    slot_code[s] = (uint32_t)c;
    rev[c] = (s == slots - 1) ? kEmptyKey : keys[s];
  }
}

__device__ __forceinline__ bool dict_find(const uint64_t* __restrict__ keys,
                                          const uint32_t* __restrict__ slot_code, uint64_t mask,
                                          uint64_t v, uint32_t* code) {
  if (v == kEmptyKey) {
    uint32_t c = slot_code[mask + 1];
    *code = c;
    return c != kNoRow;
  }
  uint64_t s = dict_slot_of(mix64(v), mask);
  for (;;) {
    uint64_t k = keys[s];
    if (k == v) {
      *code = slot_code[s];
      return true;
    }
    if (k == kEmptyKey) return false;
    s = (s + 1) & mask;
  }
}

// codes[i] = code of vals[i]; keep (optional) = 1 iff found.
__global__ void dict_lookup_kernel(const uint64_t* __restrict__ vals, uint64_t n,
                                   const uint64_t* __restrict__ keys,
                                   const uint32_t* __restrict__ slot_code, uint64_t mask,
                                   uint32_t* __restrict__ codes, uint32_t* __restrict__ keep) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    bool ok = dict_find(keys, slot_code, mask, vals[i], &c);
    codes[i] = ok ? c : 0;
    if (keep) keep[i] = ok;
  }
}

// identity codes: value -> u32 (caller has verified max < 2^32)
__global__ void narrow_kernel(const uint64_t* __restrict__ vals, uint64_t n,
                              uint32_t* __restrict__ codes) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    codes[i] = (uint32_t)vals[i];
}

// identity lookup for the y filter: keep iff value < card
__global__ void identity_keep_kernel(const uint64_t* __restrict__ vals, uint64_t n, uint64_t card,
                                     uint32_t* __restrict__ codes, uint32_t* __restrict__ keep) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t v = vals[i];
    bool ok = v < card;
    codes[i] = ok ? (uint32_t)v : 0;
    keep[i] = ok;
  }
}

// partition_bits_for (P/src/mapping.cpp:308-316), llc 12 MiB, load 0.7.
inline int partition_bits_for(uint64_t len) {
  double est = static_cast<double>(len) / 0.7 * 8.0;
  int k = 0;
  while (k < 12 && est / static_cast<double>(1ull << k) > static_cast<double>(12ull << 20)) ++k;
  return k;
}

// Builds a dictionary over vals[0..n) and writes codes[i]. Codes equal the
// reference's Dictionary::build_partitioned codes for the same input.
inline void dict_build(Ctx& ctx, const uint64_t* vals, uint64_t n, DeviceDict& d,
                       uint32_t* codes) {
  d.identity = false;
  uint64_t cap = 1024;
  while (cap < 2 * n) cap <<= 1;
  d.mask = cap - 1;
  uint64_t slots = cap + 1;
  d.keys = ctx.alloc<uint64_t>(slots);
  D3G_CUDA(cudaMemsetAsync(d.keys.p, 0xff, slots * 8, ctx.stream));
  DBuf<uint32_t> first = ctx.alloc<uint32_t>(slots);
  D3G_CUDA(cudaMemsetAsync(first.p, 0xff, slots * 4, ctx.stream));
  unsigned g = grid_for(n, 256);
  D3G_LAUNCH(ctx, dict_insert_kernel, g, 256, 0, vals, n, (unsigned long long*)d.keys.p,
             first.p, d.mask);
  // compact occupied slots
  DBuf<uint32_t> flag = ctx.alloc<uint32_t>(slots);
  DBuf<uint64_t> pos = ctx.alloc<uint64_t>(slots + 1);
  D3G_LAUNCH(ctx, occupied_flag_kernel, grid_for(slots, 256), 256, 0, first.p, slots, flag.p);
  exclusive_scan<uint32_t>(ctx, flag.p, slots, pos.p);
  uint64_t distinct = ctx.scalar(pos.p + slots);
  d.card = distinct;
  DBuf<uint64_t> sk = ctx.alloc<uint64_t>(distinct);
  DBuf<uint32_t> ss = ctx.alloc<uint32_t>(distinct);
  int k = partition_bits_for(n);
  D3G_LAUNCH(ctx, dict_collect_kernel, grid_for(slots, 256), 256, 0, d.keys.p, first.p, slots, k,
             pos.p, sk.p, ss.p);
  radix_sort(ctx, sk.p, ss.p, distinct, 32 + k, false);
  d.slot_code = ctx.alloc<uint32_t>(slots);
  D3G_CUDA(cudaMemsetAsync(d.slot_code.p, 0xff, slots * 4, ctx.stream));
  d.rev = ctx.alloc<uint64_t>(distinct);
  D3G_LAUNCH(ctx, dict_assign_kernel, grid_for(distinct, 256), 256, 0, ss.p, distinct, d.keys.p,
             slots, d.slot_code.p, d.rev.p);
  if (codes)
    D3G_LAUNCH(ctx, dict_lookup_kernel, g, 256, 0, vals, n, d.keys.p, d.slot_code.p, d.mask,
               codes, (uint32_t*)nullptr);
}

// Stable compaction helpers -------------------------------------------------
template <class T>
__global__ void compact_kernel(const T* __restrict__ in, const uint32_t* __restrict__ keep,
                               const uint64_t* __restrict__ pos, uint64_t n, T* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (keep[i]) out[pos[i]] = in[i];
}

}  // namespace d3g
