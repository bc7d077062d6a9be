// Multi-GPU exchange of the x-sharded join_project.
//
// Partitioning R by x is intersection-free (the reference's own thread
// chunking, P/include/dim3/common.hpp:130-155 and P/src/sparsebmm.cpp:79-104),
// so ranks never exchange pairs. What they must agree on are the inputs of the
// global decisions (f1, natural keys, f2 -- P/src/costmodel.cpp:515-586) and
// the final tallies:
//   * allreduce SUM / MAX of small device buffers: the m_x histogram, dR(y),
//     the per-y raw R counts (the bag join size behind f1), scalars;
//   * allgather of the per-rank tally records (count, sum, xor, ...): XOR has
//     no NCCL reduction, so the records are gathered and folded on the host.
// Two transports behind one interface:
//   * NCCL over NVLink/NVSwitch (ncclAllReduce / ncclAllGather on the
//     context's stream), loaded with dlopen so the library itself does not
//     depend on libnccl;
//   * a host callback (d3g_exchange_fn): device buffers are staged through the
//     host and the caller performs the collective (torch.distributed gloo, a
//     thread barrier for the one-GPU shard projection, a replay of recorded
//     results). Only the host threads wait on one another; no kernel ever
//     waits for another rank's kernel.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <chrono>

#include "common.cuh"

namespace d3g {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

inline NcclApi& nccl() {
  static NcclApi api;
  if (!api.lib) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw Error(D3G_CONFIG_ERROR, std::string("NCCL not loadable: ") + dlerror());
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p) throw Error(D3G_CONFIG_ERROR, std::string("NCCL symbol missing: ") + n);
      return p;
    };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.lib = h;
  }
  return api;
}

#define D3G_NCCL(call)                                                                   \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess)                                                               \
      throw ::d3g::Error(D3G_INTERNAL_ERROR, std::string(#call) + ": " +                 \
                                                 ::d3g::nccl().error_string(r_));        \
  } while (0)

struct Exchange {
  int nranks = 1, rank = 0;
  ncclComm_t comm = nullptr;
  d3g_exchange_fn host_fn = nullptr;
  void* host_user = nullptr;
  // accounting of the current call: collectives, bytes a ring collective
  // moves per rank over the links (all-reduce 2 (N-1)/N B, all-gather the
  // other ranks' parts), and the host time of host-staged collectives (the
  // one-GPU shard projection replaces it by an NVLink estimate)
  uint64_t calls = 0, bus_bytes = 0;
  double host_ms = 0;
  void reset_stats() {
    calls = bus_bytes = 0;
    host_ms = 0;
  }
  bool active() const { return nranks > 1 || comm != nullptr || host_fn != nullptr; }
  ~Exchange() {
    if (comm) nccl().comm_destroy(comm);
  }
};

inline size_t ex_elem_bytes(int op) { return op == D3G_EX_SUM_U32 ? 4 : op == D3G_EX_GATHER ? 1 : 8; }

// Host-time bracket of a host-staged collective: the stream is drained first
// (so earlier kernels are not counted) and after (the upload is counted).
struct ExHostTimer {
  Ctx& X;
  Exchange& E;
  std::chrono::steady_clock::time_point t0;
  ExHostTimer(Ctx& x, Exchange& e) : X(x), E(e) {
    X.sync();
    t0 = std::chrono::steady_clock::now();
  }
  ~ExHostTimer() {
    cudaStreamSynchronize(X.stream);
    E.host_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
};

// In-place collective over a device buffer of `count` elements (op's type):
// SUM_U64 / SUM_U32 / MAX_U64. Stream-ordered on X.stream.
inline void ex_allreduce(Ctx& X, Exchange& E, void* dbuf, uint64_t count, int op) {
  if (count == 0 || !E.active()) return;
  ++E.calls;
  E.bus_bytes += 2 * count * ex_elem_bytes(op) * (E.nranks - 1) / std::max(E.nranks, 1);
  if (E.comm) {
    const ncclDataType_t t = op == D3G_EX_SUM_U32 ? ncclUint32 : ncclUint64;
    const ncclRedOp_t o = op == D3G_EX_MAX_U64 ? ncclMax : ncclSum;
    D3G_NCCL(nccl().all_reduce(dbuf, dbuf, count, t, o, E.comm, X.stream));
    return;
  }
  const size_t bytes = count * ex_elem_bytes(op);
  ExHostTimer timer(X, E);
  std::vector<char> h(bytes);
  X.to_host(h.data(), static_cast<const char*>(dbuf), bytes);
  if (E.host_fn(E.host_user, op, h.data(), count) != 0)
    throw Error(D3G_INTERNAL_ERROR, "exchange callback failed (allreduce)");
  X.to_device(static_cast<char*>(dbuf), h.data(), bytes);
}

// Allgather of `bytes` per rank: out (host) receives nranks * bytes, rank r's
// record at [r * bytes, (r + 1) * bytes).
inline void ex_allgather(Ctx& X, Exchange& E, const void* mine, void* out, uint64_t bytes) {
  if (!E.active()) {
    std::memcpy(out, mine, bytes);
    return;
  }
  ++E.calls;
  E.bus_bytes += bytes * (E.nranks - 1);
  if (E.comm) {
    DBuf<char> din = X.alloc<char>(bytes), dout = X.alloc<char>(bytes * E.nranks);
    X.to_device(din.p, static_cast<const char*>(mine), bytes);
    D3G_NCCL(nccl().all_gather(din.p, dout.p, bytes, ncclUint8, E.comm, X.stream));
    X.to_host(static_cast<char*>(out), dout.p, bytes * E.nranks);
    return;
  }
  ExHostTimer timer(X, E);
  std::memcpy(static_cast<char*>(out) + (size_t)E.rank * bytes, mine, bytes);
  if (E.host_fn(E.host_user, D3G_EX_GATHER, out, bytes) != 0)
    throw Error(D3G_INTERNAL_ERROR, "exchange callback failed (allgather)");
}

// Allgather of variable-size DEVICE segments: rank q contributes counts[q]
// elements of `elem` bytes (`mine` is this rank's); `out` (device, sum of the
// counts) receives them rank-major. NCCL: one ncclAllGather of slots padded
// to the largest part, then one device copy per part; host transport: the
// parts are staged through the host callback.
inline void ex_allgatherv_dev(Ctx& X, Exchange& E, const void* mine,
                              const std::vector<uint64_t>& counts, size_t elem, void* out) {
  const int N = E.nranks;
  uint64_t maxn = 0, total = 0;
  std::vector<uint64_t> off(N + 1, 0);
  for (int q = 0; q < N; ++q) {
    maxn = std::max(maxn, counts[q]);
    off[q + 1] = off[q] + counts[q];
  }
  total = off[N];
  char* o = static_cast<char*>(out);
  const uint64_t slot = maxn * elem;
  if (slot == 0) return;
  ++E.calls;
  E.bus_bytes += (total - counts[E.rank]) * elem;
  if (E.comm) {
    DBuf<char> tin = X.alloc<char>(slot), tout = X.alloc<char>(slot * N);
    if (counts[E.rank])
      D3G_CUDA(cudaMemcpyAsync(tin.p, mine, counts[E.rank] * elem, cudaMemcpyDeviceToDevice, X.stream));
    D3G_NCCL(nccl().all_gather(tin.p, tout.p, slot, ncclUint8, E.comm, X.stream));
    for (int q = 0; q < N; ++q)
      if (counts[q])
        D3G_CUDA(cudaMemcpyAsync(o + off[q] * elem, tout.p + (uint64_t)q * slot, counts[q] * elem,
                                 cudaMemcpyDeviceToDevice, X.stream));
    return;
  }
  ExHostTimer timer(X, E);
  std::vector<char> h(slot * N);
  if (counts[E.rank])
    X.copy_to_pageable(h.data() + (uint64_t)E.rank * slot, mine, counts[E.rank] * elem);
  if (E.host_fn(E.host_user, D3G_EX_GATHER, h.data(), slot) != 0)
    throw Error(D3G_INTERNAL_ERROR, "exchange callback failed (allgatherv)");
  for (int q = 0; q < N; ++q)
    if (counts[q]) X.to_device(o + off[q] * elem, h.data() + (uint64_t)q * slot, counts[q] * elem);
}

// Host scalars through the same transport (a tiny device round trip).
inline void ex_allreduce_host(Ctx& X, Exchange& E, uint64_t* v, uint64_t count, int op) {
  if (count == 0 || !E.active()) return;
  DBuf<uint64_t> d = X.alloc<uint64_t>(count);
  X.to_device(d.p, v, count);
  ex_allreduce(X, E, d.p, count, op);
  X.to_host(v, d.p, count);
}

}  // namespace d3g
