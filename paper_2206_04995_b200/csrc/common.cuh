// Shared internals of the B200 DIM^3 library: error taxonomy (mirrors
// P/include/dim3/common.hpp:25-36), the per-context device arena and stream,
// hashing (mix64, common.hpp:42-49), and small warp/block helpers.
#pragma once

#include <mutex>
#include <unordered_map>

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dim3_b200.h"

namespace d3g {

using code_t = uint32_t;

// ---------------------------------------------------------------------------
// Errors. Thrown inside the library, mapped to D3G_* status codes at the ABI.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};
struct ConfigError : Error {
  explicit ConfigError(const std::string& m) : Error(D3G_CONFIG_ERROR, m) {}
};
struct ResourceError : Error {
  explicit ResourceError(const std::string& m) : Error(D3G_RESOURCE_ERROR, m) {}
};
struct CudaError : Error {
  explicit CudaError(const std::string& m) : Error(D3G_INTERNAL_ERROR, m) {}
};

#define D3G_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess)                                                    \
      throw ::d3g::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + \
                             " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

// Launch bookkeeping: every kernel launch goes through D3G_LAUNCH so the
// context can report how many kernels a call issued.
#define D3G_LAUNCH(ctx, kernel, grid, block, smem, ...)                       \
  do {                                                                        \
    kernel<<<(grid), (block), (smem), (ctx).stream>>>(__VA_ARGS__);           \
    D3G_CUDA(cudaGetLastError());                                             \
    (ctx).launches++;                                                         \
  } while (0)

inline constexpr int kNumSMs = 148;

// ---------------------------------------------------------------------------
// Device arena: stream-ordered allocations from the device's default pool,
// which the context configures to never release memory back to the driver
// (so repeated calls reuse the same HBM without cudaMalloc round trips).
// Tracks the working-set high-water mark against the memory budget.
struct Ctx;

template <class T>
struct DBuf {
  T* p = nullptr;
  uint64_t n = 0;
  Ctx* ctx = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), ctx(o.ctx) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept;
  ~DBuf();
  void reset();
  T* get() const { return p; }
  uint64_t bytes() const { return n * sizeof(T); }
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t launches = 0;
  uint64_t d2h_bytes = 0;  // device->host bytes read back by the current call
  uint64_t live_bytes = 0, peak_bytes = 0, budget = 0;
  uint64_t reserved = 0;  // size of the largest block pre-faulted into the pool
  int sm_count = kNumSMs;
  size_t smem_optin = 0;
  // small pinned host staging area for scalars read back mid-pipeline
  void* pinned = nullptr;
  size_t pinned_bytes = 0;

  // Buffers up to kCacheMax bytes are rounded up to a power of two and
  // recycled through per-size free lists on the host: a pipeline call makes
  // ~100 short-lived allocations, and every API call the host saves while the
  // GPU runs the small prelude kernels is GPU time saved. Reuse needs no
  // event: everything runs on this context's one stream, so a recycled block
  // is only touched after the work that used it before.
  static constexpr uint64_t kCacheMax = 64ull << 20;
  std::vector<void*> cache[40];
  static int size_class(uint64_t bytes) {
    int c = 8;
    while ((1ull << c) < bytes) ++c;
    return c;
  }
  void* raw_alloc(uint64_t bytes) {
    if (bytes == 0) bytes = 16;
    if (budget != 0 && live_bytes + bytes > budget)
      throw ResourceError("device memory budget exceeded: need " +
                          std::to_string(live_bytes + bytes) + " bytes, limit " +
                          std::to_string(budget) + " bytes");
    void* p = nullptr;
    const bool cached = bytes <= kCacheMax;
    const int c = cached ? size_class(bytes) : 0;
    if (cached && !cache[c].empty()) {
      p = cache[c].back();
      cache[c].pop_back();
    } else {
      cudaError_t e = cudaMallocAsync(&p, cached ? (1ull << c) : bytes, stream);
      if (e != cudaSuccess) {
        cudaGetLastError();
        throw ResourceError("device allocation of " + std::to_string(bytes) +
                            " bytes failed: " + cudaGetErrorString(e));
      }
    }
    live_bytes += bytes;
    if (live_bytes > peak_bytes) peak_bytes = live_bytes;
    return p;
  }
  void raw_free(void* p, uint64_t bytes) {
    if (p == nullptr) return;
    if (bytes == 0) bytes = 16;
    if (bytes <= kCacheMax)
      cache[size_class(bytes)].push_back(p);
    else
      cudaFreeAsync(p, stream);
    live_bytes -= bytes;
  }
  void release_cache() {
    for (auto& l : cache) {
      for (void* p : l) cudaFreeAsync(p, stream);
      l.clear();
    }
  }
  template <class T>
  DBuf<T> alloc(uint64_t n) {
    DBuf<T> b;
    b.p = static_cast<T*>(raw_alloc(n * sizeof(T)));
    b.n = n;
    b.ctx = this;
    return b;
  }
  // Zero arena: small zero-filled buffers are carved from one block that
  // begin_call() re-zeroes with a single memset, instead of one memset each.
  // Slices live until the end of the call (DBuf with ctx == nullptr: no free).
  static constexpr uint64_t kZeroArena = 4ull << 20, kZeroSlice = 512ull << 10;
  char* zarena = nullptr;
  uint64_t zused = 0;
  void begin_call() {
    if (!zarena) {
      D3G_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&zarena), kZeroArena, stream));
      D3G_CUDA(cudaMemsetAsync(zarena, 0, kZeroArena, stream));
    } else if (zused) {
      D3G_CUDA(cudaMemsetAsync(zarena, 0, zused, stream));
    }
    zused = 0;
  }
  template <class T>
  DBuf<T> zeros(uint64_t n) {
    const uint64_t bytes = ((n == 0 ? 16 : n * sizeof(T)) + 255) & ~255ull;
    if (zarena && bytes <= kZeroSlice && zused + bytes <= kZeroArena) {
      DBuf<T> b;
      b.p = reinterpret_cast<T*>(zarena + zused);
      b.n = n;
      zused += bytes;
      return b;
    }
    DBuf<T> b = alloc<T>(n);
    D3G_CUDA(cudaMemsetAsync(b.p, 0, n * sizeof(T) + (n == 0 ? 16 : 0), stream));
    return b;
  }
  // Persistent look-back state of scan_onepass_kernel (prims.cuh): tile
  // flags carry the parity of the scan that wrote them and every scan clears
  // the entries past its own tiles, so no scan needs a memset; the ticket
  // counter (entry scan_cap) only grows.
  unsigned long long* scan_state = nullptr;
  uint64_t scan_cap = 0, scan_tickets = 0, scan_hw = 0;
  uint32_t scan_parity = 0;
  void scan_reserve(uint64_t tiles) {
    if (tiles <= scan_cap) return;
    uint64_t cap = 4096;
    while (cap < tiles) cap <<= 1;
    if (scan_state) cudaFreeAsync(scan_state, stream);
    D3G_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scan_state), (cap + 1) * 8, stream));
    D3G_CUDA(cudaMemsetAsync(scan_state, 0, (cap + 1) * 8, stream));
    scan_cap = cap;
    scan_tickets = scan_hw = 0;
  }
  uint64_t syncs = 0;  // host round trips of the current call (diagnostics)
  // Deferred reads: small device values copied into pinned memory now and
  // delivered to their host destinations at the next synchronisation, so
  // independent scalars share one round trip instead of one each.
  void* defer_host = nullptr;
  static constexpr size_t kDeferBytes = 4096;
  struct Deferred {
    void* dst;
    size_t off, bytes;
  };
  std::vector<Deferred> deferred;
  size_t defer_used = 0;
  void defer(void* dst, const void* src, size_t bytes) {
    if (!defer_host) D3G_CUDA(cudaMallocHost(&defer_host, kDeferBytes));
    if (defer_used + bytes > kDeferBytes) sync();  // flush first
    D3G_CUDA(cudaMemcpyAsync(static_cast<char*>(defer_host) + defer_used, src, bytes,
                             cudaMemcpyDeviceToHost, stream));
    deferred.push_back({dst, defer_used, bytes});
    defer_used += (bytes + 7) & ~size_t(7);
    d2h_bytes += bytes;
  }
  bool has_deferred() const { return !deferred.empty(); }
  void deliver(size_t n = ~size_t(0)) {  // the first n deferred reads
    if (n > deferred.size()) n = deferred.size();
    for (size_t i = 0; i < n; ++i)
      std::memcpy(deferred[i].dst, static_cast<const char*>(defer_host) + deferred[i].off,
                  deferred[i].bytes);
    deferred.erase(deferred.begin(), deferred.begin() + n);
    if (deferred.empty()) defer_used = 0;
  }
  void sync() {
    ++syncs;
    D3G_CUDA(cudaStreamSynchronize(stream));
    deliver();
  }
  // Marks the point after the deferred reads issued so far; wait_mark()
  // delivers them once the stream reaches it, while the work enqueued after
  // the mark keeps the GPU busy (the host reads a size during a long kernel).
  cudaEvent_t mark_ev = nullptr;
  size_t mark_n = 0;
  void mark() {
    if (!mark_ev) D3G_CUDA(cudaEventCreateWithFlags(&mark_ev, cudaEventDisableTiming));
    D3G_CUDA(cudaEventRecord(mark_ev, stream));
    mark_n = deferred.size();
  }
  void wait_mark() {
    ++syncs;
    D3G_CUDA(cudaEventSynchronize(mark_ev));
    deliver(mark_n);
    mark_n = 0;
  }
  // After a call whose working set outgrew the pool's largest block, fault in
  // one block of (peak + 25%) and return it to the pool: the stream-ordered
  // allocator then carves later calls' buffers out of it instead of mapping
  // new physical memory mid-pipeline (which stalls the stream for ms).
  void reserve_for(uint64_t peak) {
    if (peak <= reserved) return;
    const uint64_t want = peak + peak / 4 + (64ull << 20);
    void* p = nullptr;
    if (cudaMallocAsync(&p, want, stream) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    cudaFreeAsync(p, stream);
    sync();
    reserved = want;
  }
  // Copies n device values to host (through pinned staging) and syncs.
  template <class T>
  void to_host(T* dst, const T* src, uint64_t n) {
    if (n == 0) return;
    uint64_t bytes = n * sizeof(T);
    if (bytes > pinned_bytes) {
      if (pinned) cudaFreeHost(pinned);
      pinned_bytes = bytes < (1u << 20) ? (1u << 20) : bytes;
      D3G_CUDA(cudaMallocHost(&pinned, pinned_bytes));
    }
    D3G_CUDA(cudaMemcpyAsync(pinned, src, bytes, cudaMemcpyDeviceToHost, stream));
    d2h_bytes += bytes;
    sync();
    std::memcpy(dst, pinned, bytes);
  }
  template <class T>
  T scalar(const T* src) {
    T v;
    to_host(&v, src, 1);
    return v;
  }
  // Device -> pageable host copy of a large buffer: 64 MB chunks through two
  // pinned staging buffers, the D2H of chunk k+1 overlapping the (threaded)
  // host copy of chunk k. A plain cudaMemcpy into pageable memory runs at a
  // few GB/s; this path runs near the PCIe rate.
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  static constexpr size_t kStage = 64ull << 20;
  void copy_to_pageable(void* dst, const void* src, size_t bytes);
  // a materialized result kept on the device for d3g_take_pairs
  DBuf<uint64_t> held_x, held_z;
  uint64_t held_n = 0;
  template <class T>
  void to_device(T* dst, const T* src, uint64_t n) {
    if (n == 0) return;
    D3G_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, stream));
  }
};

inline void Ctx::copy_to_pageable(void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  for (int b = 0; b < 2; ++b)
    if (!stage[b]) {
      D3G_CUDA(cudaMallocHost(&stage[b], kStage));
      D3G_CUDA(cudaEventCreateWithFlags(&stage_ev[b], cudaEventDisableTiming));
    }
  auto host_copy = [](char* d, const char* s, size_t n) {
    const unsigned nt = n >= (8u << 20) ? 8u : 1u;
    if (nt == 1) {
      std::memcpy(d, s, n);
      return;
    }
    std::vector<std::thread> th;
    const size_t part = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
      const size_t o = t * part;
      if (o >= n) break;
      th.emplace_back([=] { std::memcpy(d + o, s + o, (n - o) < part ? (n - o) : part); });
    }
    for (auto& t : th) t.join();
  };
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  size_t issued = 0, done = 0;
  size_t len[2] = {0, 0}, off[2] = {0, 0};
  int b = 0;
  // prime: chunk 0
  len[0] = bytes < kStage ? bytes : kStage;
  D3G_CUDA(cudaMemcpyAsync(stage[0], s, len[0], cudaMemcpyDeviceToHost, stream));
  D3G_CUDA(cudaEventRecord(stage_ev[0], stream));
  off[0] = 0;
  issued = len[0];
  while (done < bytes) {
    const int nb = b ^ 1;
    if (issued < bytes) {  // next chunk into the other buffer (free: copied out before)
      len[nb] = (bytes - issued) < kStage ? (bytes - issued) : kStage;
      off[nb] = issued;
      D3G_CUDA(cudaMemcpyAsync(stage[nb], s + issued, len[nb], cudaMemcpyDeviceToHost, stream));
      D3G_CUDA(cudaEventRecord(stage_ev[nb], stream));
      issued += len[nb];
    }
    D3G_CUDA(cudaEventSynchronize(stage_ev[b]));
    host_copy(d + off[b], static_cast<const char*>(stage[b]), len[b]);
    done += len[b];
    b = nb;
  }
  d2h_bytes += bytes;
}

template <class T>
DBuf<T>& DBuf<T>::operator=(DBuf&& o) noexcept {
  if (this != &o) {
    reset();
    p = o.p;
    n = o.n;
    ctx = o.ctx;
    o.p = nullptr;
    o.n = 0;
  }
  return *this;
}
template <class T>
void DBuf<T>::reset() {
  if (p && ctx) ctx->raw_free(p, n * sizeof(T));
  p = nullptr;
  n = 0;
}
template <class T>
DBuf<T>::~DBuf() {
  reset();
}

// ---------------------------------------------------------------------------
// Device helpers.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}
__host__ __device__ __forceinline__ uint64_t pair_hash(uint64_t x, uint64_t z) {
  return mix64(mix64(x) ^ z);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// 32-byte global accesses in ONE instruction (LDG/STG.E.ENL2.256, sm_100):
// a warp reading 32 B per lane touches each 32 B sector once instead of
// twice (two 16 B loads). p must be 32 B aligned.
__device__ __forceinline__ void ld256(const uint4* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z),
                 "=r"(b.w)
               : "l"(p));
}
__device__ __forceinline__ void st256(uint4* p, const uint4& a, const uint4& b) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y),
               "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint64_t warp_xor(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v ^= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  return v;
}

// Accumulator of the order-independent output fingerprint and count.
struct Tally {
  unsigned long long count;
  unsigned long long sum;
  unsigned long long xr;
};

// Warp-reduce (count, sum, xor) and add once per warp.
__device__ __forceinline__ void tally_flush(Tally* t, uint64_t cnt, uint64_t sum,
                                            uint64_t xr) {
  cnt = warp_sum(cnt);
  sum = warp_sum(sum);
  xr = warp_xor(xr);
  if (lane_id() == 0) {
    if (cnt) atomicAdd(&t->count, (unsigned long long)cnt);
    if (sum) atomicAdd(&t->sum, (unsigned long long)sum);
    if (xr) atomicXor(&t->xr, (unsigned long long)xr);
  }
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is per function, shared by every
// context and thread of the process: only ever RAISE it (a call setting a
// smaller value would break a concurrent call -- ranks as threads -- that
// launches with more).
template <class F>
inline cudaError_t raise_smem_attr(F* kfn, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> cur;
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cur[reinterpret_cast<const void*>(kfn)];
  if (bytes <= c) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) c = bytes;
  return e;
}

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 16u) {
  uint64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

}  // namespace d3g
