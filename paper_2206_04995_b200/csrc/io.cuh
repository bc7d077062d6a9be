// Table files on the device path: binary ingest and pair writers.
//
// * read_binary (P/src/relation.cpp:98-127): little-endian u64 (left, right)
//   pairs, no header, length a multiple of 16. Here the file streams through
//   two pinned chunks straight into HBM (read of chunk k+1 overlaps the H2D
//   copy and the de-interleave kernel of chunk k); nothing is parsed.
// * save_table (P/src/relation.cpp:164-204): binary = the same interleaved
//   u64 pairs; tsv/csv = "left<sep>right\n" in decimal. Pairs are interleaved
//   or formatted on the GPU (one thread per pair, digits via a multiply-high
//   division by 10), copied back in chunks and written.
// * detect_format (P/src/relation.cpp:13-20): by extension, .tsv/.txt -> tsv,
//   .csv -> csv, .bin -> binary, anything else tsv.
#pragma once

#include "common.cuh"
#include "prims.cuh"

namespace d3g {

__global__ void deinterleave_kernel(const uint64_t* __restrict__ in, uint64_t n,
                                    uint64_t* __restrict__ left, uint64_t* __restrict__ right) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const ulonglong2 v = reinterpret_cast<const ulonglong2*>(in)[i];
    left[i] = v.x;
    right[i] = v.y;
  }
}

__global__ void interleave_kernel(const uint64_t* __restrict__ left,
                                  const uint64_t* __restrict__ right, uint64_t n,
                                  uint64_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    reinterpret_cast<ulonglong2*>(out)[i] = make_ulonglong2(left[i], right[i]);
}

__device__ __forceinline__ uint32_t dec_digits(uint64_t v) {
  uint32_t d = 1;
  uint64_t p = 10;
  while (d < 20 && v >= p) {
    ++d;
    p *= 10;
  }
  return d;
}

__device__ __forceinline__ uint64_t div10(uint64_t v) {
  return __umul64hi(v, 0xCCCCCCCCCCCCCCCDull) >> 3;
}

// characters of one "left<sep>right\n" line
__global__ void text_len_kernel(const uint64_t* __restrict__ left,
                                const uint64_t* __restrict__ right, uint64_t n,
                                uint32_t* __restrict__ len) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    len[i] = dec_digits(left[i]) + dec_digits(right[i]) + 2;
}

__device__ __forceinline__ char* put_dec(char* p, uint64_t v, uint32_t digits) {
  char* e = p + digits;
  char* q = e;
  do {
    const uint64_t t = div10(v);
    *--q = (char)('0' + (v - t * 10));
    v = t;
  } while (q > p);
  return e;
}

__global__ void text_write_kernel(const uint64_t* __restrict__ left,
                                  const uint64_t* __restrict__ right, uint64_t n,
                                  const uint64_t* __restrict__ off, char sep,
                                  char* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    char* p = out + off[i];
    const uint64_t a = left[i], b = right[i];
    p = put_dec(p, a, dec_digits(a));
    *p++ = sep;
    p = put_dec(p, b, dec_digits(b));
    *p = '\n';
  }
}

}  // namespace d3g
