// Reference-equivalent DenseEC work counters (DenseEcStats,
// P/include/dim3/denseec.hpp:20-29, incremented at P/src/denseec.cpp:46-64).
//
// The GPU never runs the reference's per-pair sweep, so these counters are
// what the reference WOULD have counted on the same input, computed exactly:
//   * for each live x and each dense z, the reference picks wide iff
//     m_z > f3_threshold(m_x) (cost_based; force_wide / force_probe pin it);
//   * wide: block_and_any (P/include/dim3/bitmap.hpp:23-36) examines W-bit
//     blocks in y order up to the first block with a common y, so
//     blocks_checked = first_common_y / W + 1, or every block on a miss;
//   * probe: probe_any (bitmap.hpp:40-48) tests R[x]'s y (ascending) in S[z]'s
//     bitmap until the first hit, so probes_done = rank of the first common
//     y in R[x] + 1, or m_x on a miss;
//   * row_bitmaps_built counts the x with at least one wide encounter.
// Both sweeps stop at the SAME y: the smallest y shared by R[x] and S[z].
// One CTA per live x holds R[x] as a bitmap in shared memory; each thread
// walks one dense row S[z] (ascending y) until its first bit hit. This is a
// counting instrument for parity and roofline work figures (SURVEY 8(d)
// W_D = 8 * blocks_checked + probes_done), not the product path.
#pragma once

#include "common.cuh"

namespace d3g {

struct DenseCounters {
  unsigned long long wide, probe, blocks, probes, bitmaps;
};

constexpr int kCntThreads = 512;

// Dense rows: (zptr, zcol) over z_rows rows; a row is dense iff its degree m
// has dsel[m] != 0 (dsel == nullptr: every non-empty row). thr[m_x] is the
// wide/probe threshold per x degree (< thr_n).
__global__ void __launch_bounds__(kCntThreads)
dense_counters_kernel(const uint64_t* __restrict__ r_ptr, const uint32_t* __restrict__ r_col,
                      uint64_t x_lo, uint64_t x_hi, const uint64_t* __restrict__ zptr,
                      const uint32_t* __restrict__ zcol, uint64_t z_rows,
                      const uint8_t* __restrict__ dsel, uint64_t dsel_n,
                      const uint32_t* __restrict__ thr, uint64_t thr_n, uint32_t w,
                      uint64_t n_blocks, uint32_t words, unsigned int* __restrict__ next,
                      DenseCounters* __restrict__ out) {
  extern __shared__ uint32_t rbm[];  // R[x] as a bitmap over y codes
  __shared__ uint32_t s_x;
  for (uint32_t i = threadIdx.x; i < words; i += kCntThreads) rbm[i] = 0;
  unsigned long long wide = 0, probe = 0, blocks = 0, probes = 0, bitmaps = 0;
  for (;;) {
    if (threadIdx.x == 0) s_x = atomicAdd(next, 1u);
    __syncthreads();
    const uint64_t x = x_lo + s_x;
    __syncthreads();
    if (x >= x_hi) break;
    const uint64_t r0 = r_ptr[x], r1 = r_ptr[x + 1];
    const uint32_t m_x = (uint32_t)(r1 - r0);
    if (m_x == 0) continue;
    for (uint64_t k = r0 + threadIdx.x; k < r1; k += kCntThreads) {
      const uint32_t y = r_col[k];
      atomicOr(&rbm[y >> 5], 1u << (y & 31));
    }
    __syncthreads();
    const uint32_t t = m_x < thr_n ? thr[m_x] : 0xffffffffu;
    bool any_wide = false;
    for (uint64_t z = threadIdx.x; z < z_rows; z += kCntThreads) {
      const uint64_t k0 = zptr[z], k1 = zptr[z + 1];
      const uint64_t m_z = k1 - k0;
      if (m_z == 0) continue;
      if (dsel && (m_z >= dsel_n || !dsel[m_z])) continue;
      uint32_t first = 0xffffffffu;
      for (uint64_t k = k0; k < k1; ++k) {
        const uint32_t y = zcol[k];
        if ((rbm[y >> 5] >> (y & 31)) & 1u) {
          first = y;
          break;
        }
      }
      if (m_z > t) {
        ++wide;
        any_wide = true;
        blocks += first == 0xffffffffu ? n_blocks : (uint64_t)(first / w) + 1;
      } else {
        ++probe;
        if (first == 0xffffffffu) {
          probes += m_x;
        } else {  // rank of first in the sorted R[x]
          uint64_t lo = r0, hi = r1;
          while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (r_col[mid] < first) lo = mid + 1; else hi = mid;
          }
          probes += lo - r0 + 1;
        }
      }
    }
    if (__syncthreads_or(any_wide) && threadIdx.x == 0) ++bitmaps;
    for (uint64_t k = r0 + threadIdx.x; k < r1; k += kCntThreads) rbm[r_col[k] >> 5] = 0;
    __syncthreads();
  }
  wide = warp_sum(wide);
  probe = warp_sum(probe);
  blocks = warp_sum(blocks);
  probes = warp_sum(probes);
  if (lane_id() == 0) {
    if (wide) atomicAdd(&out->wide, wide);
    if (probe) atomicAdd(&out->probe, probe);
    if (blocks) atomicAdd(&out->blocks, blocks);
    if (probes) atomicAdd(&out->probes, probes);
  }
  if (threadIdx.x == 0 && bitmaps) atomicAdd(&out->bitmaps, bitmaps);
}

}  // namespace d3g
