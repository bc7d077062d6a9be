// f1 gate estimate and the classical hash-join-dedup branch on the GPU.
//
// * estimate_out_j_raw (P/src/costmodel.cpp:375-423): the exact bag join
//   size when both tables have <= 65,536 rows, else 16,384 strided samples
//   per side, hits scaled by (|S|/ms)(|R|/mr) in long double. The counting is
//   integer and order-free, so the GPU hash count gives the reference's hits
//   exactly; the scaling runs on the host with the reference's expression.
// * hash_join_dedup (P/src/classical.cpp:111-210): group S by y (duplicates
//   kept), probe every R row, and deduplicate the (x, z) output. On the GPU
//   the y groups come from the HBM dictionary (y code = group), x and z are
//   interned by dictionaries too, and the dedup is a global open-addressing
//   set of 64-bit (x code << 32 | z code) keys filled with atomicCAS; a
//   successful insert is a new distinct pair. intermediate_pairs = the bag
//   join size (ClassicalStats, classical.hpp).
#pragma once

#include "mapping.cuh"
#include "sparsebmm.cuh"

namespace d3g {

__device__ __forceinline__ uint64_t est_slot(uint64_t v, uint64_t mask) {
  uint64_t h = mix64(v ^ 0x2545F4914F6CDD1Dull);
  return h & mask;
}

// counts[slot] = multiplicity of key in the S sample. Open addressing with a
// 64-bit atomicCAS on the key (empty = all ones), so the slot a value lands
// in is decided atomically at L2 -- no published-flag protocol, whose
// key reads could be served stale from another SM's L1 and split a value
// across two slots. The value 2^64-1 itself is counted in counts[cap].
__global__ void est_insert_kernel(const uint64_t* __restrict__ vals, uint64_t n,
                                  unsigned long long* __restrict__ keys,
                                  unsigned int* __restrict__ counts, uint64_t mask) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = vals[i];
    if (v == ~0ull) {
      atomicAdd(&counts[mask + 1], 1u);
      continue;
    }
    uint64_t s = est_slot(v, mask);
    for (;;) {
      const unsigned long long prev = atomicCAS(&keys[s], ~0ull, (unsigned long long)v);
      if (prev == ~0ull || prev == v) {
        atomicAdd(&counts[s], 1u);
        break;
      }
      s = (s + 1) & mask;
    }
  }
}

__global__ void est_probe_kernel(const uint64_t* __restrict__ vals, uint64_t n,
                                 const unsigned long long* __restrict__ keys,
                                 const unsigned int* __restrict__ counts, uint64_t mask,
                                 unsigned long long* __restrict__ hits) {
  uint64_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = vals[i];
    if (v == ~0ull) {
      acc += counts[mask + 1];
      continue;
    }
    uint64_t s = est_slot(v, mask);
    for (;;) {
      const uint64_t k = keys[s];
      if (k == ~0ull) break;  // not in the sample
      if (k == v) {
        acc += counts[s];
        break;
      }
      s = (s + 1) & mask;
    }
  }
  acc = warp_sum(acc);
  if (lane_id() == 0 && acc) atomicAdd(hits, (unsigned long long)acc);
}

// --- classical ---------------------------------------------------------------
// bag join size: sum over kept R rows of |group(y)|
__global__ void classical_bag_kernel(const uint32_t* __restrict__ r_yc,
                                     const uint32_t* __restrict__ keep, uint64_t nr,
                                     const uint64_t* __restrict__ gptr,
                                     unsigned long long* __restrict__ out) {
  uint64_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nr;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (keep[i]) acc += gptr[r_yc[i] + 1] - gptr[r_yc[i]];
  acc = warp_sum(acc);
  if (lane_id() == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}

// warp per R row: insert (x code, z code of every group entry) into the set
template <int kMode>
__global__ void classical_probe_kernel(const uint32_t* __restrict__ r_xc,
                                       const uint32_t* __restrict__ r_yc,
                                       const uint32_t* __restrict__ keep, uint64_t nr,
                                       const uint64_t* __restrict__ gptr,
                                       const uint32_t* __restrict__ gz,
                                       unsigned long long* __restrict__ set, uint64_t mask,
                                       Decode dec, Emit em, Tally* tally) {
  const uint32_t lane = lane_id();
  uint64_t cnt = 0, sum = 0, xr = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < nr;
       i += (uint64_t)gridDim.x * (blockDim.x / 32)) {
    if (!keep[i]) continue;
    const uint32_t xc = r_xc[i], g = r_yc[i];
    const uint64_t b = gptr[g], e = gptr[g + 1];
    for (uint64_t j = b + lane; j < e; j += 32) {
      const uint32_t zc = gz[j];
      const uint64_t key = ((uint64_t)xc << 32) | zc;
      uint64_t s = mix64(key) & mask;
      bool fresh = false;
      for (;;) {
        const unsigned long long prev = atomicCAS(&set[s], ~0ull, (unsigned long long)key);
        if (prev == ~0ull) {
          fresh = true;
          break;
        }
        if (prev == key) break;
        s = (s + 1) & mask;
      }
      if (!fresh) continue;
      ++cnt;
      if (kMode == kModeChecksum) {
        const uint64_t h = dec.hash(xc, zc);
        sum += h;
        xr ^= h;
      } else if (kMode == kModeEmit) {
        const unsigned long long idx = atomicAdd(em.cursor, 1ull);
        if (idx < em.cap) {
          em.x[idx] = xc;
          em.z[idx] = zc;
        }
      }
    }
  }
  tally_flush(tally, cnt, sum, xr);
}

// bag join size from raw (duplicate-keeping) S y counts: sum over R rows of
// cnt[y] (intermediate_pairs of the x-partitioned classical branch)
__global__ void bag_from_counts_kernel(const uint32_t* __restrict__ r_yc, uint64_t nr,
                                       const uint32_t* __restrict__ cnt,
                                       unsigned long long* __restrict__ out) {
  uint64_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nr;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc += cnt[r_yc[i]];
  acc = warp_sum(acc);
  if (lane_id() == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}

// counting scatter of S rows into y groups (duplicates kept, no sort)
__global__ void group_hist_kernel(const uint32_t* __restrict__ yc, uint64_t n,
                                  uint32_t* __restrict__ cnt) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[yc[i]], 1u);
}

__global__ void group_scatter_kernel(const uint32_t* __restrict__ yc, const uint32_t* __restrict__ zc,
                                     uint64_t n, const uint64_t* __restrict__ gptr,
                                     uint32_t* __restrict__ fill, uint32_t* __restrict__ gz) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t g = yc[i];
    gz[gptr[g] + atomicAdd(&fill[g], 1u)] = zc[i];
  }
}

}  // namespace d3g
