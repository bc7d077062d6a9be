// DenseEC P2: the cold residual pass.
//
// Pairs (x, dense z) with no common HOT y (rank < 256, counted by P1 in
// denseec_hot.cuh) but a common COLD y are the cold join R_cold x S_cold
// restricted to dense z, deduplicated per x, minus the pairs whose hot masks
// intersect. Together with P1 this is the reference's dense_ec output
// (P/src/denseec.cpp:8-86): {(x, z) : R[x] and S[z] share a y}, z dense.
//
// The cold CSR is y-major over dense row positions, keyed (variant, part, y):
// variant v in [0, 2^var_bits) holds only the rows z whose hot mask avoids
// every top rank r < var_bits set in v, and an x streams the variant of its
// own top-rank mask, so candidates that share a top rank with x (hot hits) are
// never read. Each entry is ONE 16-byte record:
//     { hz[z] word 0 (ranks 0-63) lo, hi ;  fold(hz[z] words 1-3) ;  row }
// where fold ORs the 32-bit halves of words 1-3 (bit b <=> z holds a rank
// r in [64, 256) with r % 32 == b). The hot filter reads only the record:
//     (hx[x].w0 & hz[z].w0) != 0          -> hot hit: P1 counted it, drop
//     (fold(hx[x]) & fold(hz[z])) == 0    -> no common hot rank: survivor
//     otherwise ("maybe", ~3% on cfg5)     -> exact test on hz[z] words 1-3
// Maybes are queued per warp and resolved 32 at a time (one coalesced gather
// step), so a lane never stalls the candidate stream on a dependent load.
// (Round 1 stored the whole 32-byte signature inline plus a separate 4-byte
// row id: 36 B and two loads per candidate.)
//
// Survivors are deduplicated per x in a warp-private bitmap (dense blocks of
// at most 16 row partitions: dense_cold_kernel) or a warp-private hash set
// (dense_cold_hash_kernel) with two overflow tiers: a CTA-wide shared-memory
// hash (dense_cold_cta_kernel) and a CTA-private global bitmap
// (dense_cold_overflow_kernel).
#pragma once

#include "denseec_hot.cuh"

namespace d3g {

// ---- cold CSR build --------------------------------------------------------

// Cold CSR build in two passes: per (part, y, zm) -- zm the row's
// top-var_bits hot mask -- a histogram H (one atomic per cold entry); the
// (variant, part, y) counts follow as sums of H over the masks compatible with
// the variant, and their exclusive scan is the segment starts. The scatter
// then takes each record's slot from a per-(variant, part, y) cursor (the
// scan itself, advanced in place by 64-bit atomics), for every variant
// compatible with the row. Slot order inside a segment is arbitrary: every
// consumer (the cold kernels, the z-split merge) treats a segment as a set.
// Four list entries are in flight per lane (the passes are latency-bound).
// Mask slots per (part, y): variant bits up to 4. With 4 bits the variant
// with only the 4th top rank set is skipped (its x use variant 0, a
// superset): the cheapest split for the few x without the top rank.
constexpr uint32_t kHistSlots = 16;
#ifndef D3G_MAX_VAR_BITS
#define D3G_MAX_VAR_BITS 4
#endif
constexpr uint32_t kMaxVarBits = D3G_MAX_VAR_BITS;  // the top ranks that split the cold CSR
__device__ __forceinline__ void load_hist(const uint32_t* __restrict__ H, uint64_t t,
                                          uint32_t (&h)[kHistSlots]) {
  const uint4* p = reinterpret_cast<const uint4*>(H) + 4 * t;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 a = p[q];
    h[4 * q] = a.x;
    h[4 * q + 1] = a.y;
    h[4 * q + 2] = a.z;
    h[4 * q + 3] = a.w;
  }
}
// (variant, part, y) counts from H: thread per (part, y)
__global__ void cold_cnt_from_hist_kernel(const uint32_t* __restrict__ H, uint64_t n_py,
                                          uint64_t y_card, uint32_t parts, uint32_t var_bits,
                                          uint32_t vskip, uint32_t* __restrict__ cnt) {
  const uint32_t nvar = 1u << var_bits;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_py;
       t += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t h[kHistSlots];
    load_hist(H, t, h);
    const uint64_t part = t / y_card, y = t % y_card;
    for (uint32_t v = 0; v < nvar; ++v) {
      uint32_t c = 0;
      if (v != vskip)
        for (uint32_t zm = 0; zm < nvar; ++zm)
          if ((zm & v) == 0) c += h[zm];
      cnt[((uint64_t)v * parts + part) * y_card + y] = c;
    }
  }
}
// One thread per dense row. A row's ranks ascend, so its cold entries are
// the suffix after its popc(hz[row]) hot ones: no lane idles on hot entries
// and four cold entries of a row are in flight together.
__device__ __forceinline__ uint32_t row_hot_count(const uint64_t* __restrict__ hz, uint32_t kw,
                                                  uint64_t i, uint4& a, uint4& b) {
  if (kw == 4) {
    ld256(reinterpret_cast<const uint4*>(hz) + 2 * i, a, b);
    return __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w) + __popc(b.x) + __popc(b.y) +
           __popc(b.z) + __popc(b.w);
  }
  uint32_t n = 0;
  for (uint32_t w = 0; w < kw; ++w) n += __popcll(hz[i * kw + w]);
  const uint64_t w0 = hz[i * kw];
  a = make_uint4((uint32_t)w0, (uint32_t)(w0 >> 32), 0, 0);
  b = make_uint4(0, 0, 0, 0);
  return n;
}
__global__ void cold_hist_kernel(const uint64_t* __restrict__ dl_ptr,
                                 const uint32_t* __restrict__ dl_col, uint64_t n_dense,
                                 const uint32_t* __restrict__ y_of_rank, uint32_t* __restrict__ H,
                                 uint64_t y_card, uint32_t part_rows,
                                 const uint64_t* __restrict__ hz, uint32_t kw, uint32_t var_bits,
                                 uint64_t row_base = 0) {
  const uint32_t vmask = (1u << var_bits) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_dense;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 a, b;
    const uint64_t e = dl_ptr[i + 1];
    uint64_t k = dl_ptr[i] + row_hot_count(hz, kw, i, a, b);
    if (k >= e) continue;
    const uint64_t pb = (row_base + i) / part_rows * y_card;
    const uint32_t zm = a.x & vmask;
    for (; k < e; k += 4) {
      uint32_t r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) r[u] = k + u < e ? dl_col[k + u] : 0u;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k + u < e) atomicAdd(&H[(pb + y_of_rank[r[u]]) * kHistSlots + zm], 1u);
    }
  }
}
// cur: the exclusive scan of the (variant, part, y) counts; on return
// cur[i] is the END of segment i (= the start of segment i + 1), so the
// buffer one slot before cur, with a leading 0, is the finished cptr.
__global__ void cold_scatter_cur_kernel(const uint64_t* __restrict__ dl_ptr,
                                        const uint32_t* __restrict__ dl_col, uint64_t n_dense,
                                        const uint32_t* __restrict__ y_of_rank,
                                        unsigned long long* __restrict__ cur, uint64_t y_card,
                                        uint32_t part_rows, uint32_t parts,
                                        const uint64_t* __restrict__ hz, uint32_t kw,
                                        uint32_t var_bits, uint32_t vskip, uint64_t row_base,
                                        uint4* __restrict__ rec, uint32_t* __restrict__ col,
                                        const uint8_t* __restrict__ row_sp) {
  const uint32_t vmask = (1u << var_bits) - 1;
  const uint64_t n_py = (uint64_t)parts * y_card;  // one variant's keys
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_dense;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 a, b;
    const uint64_t e = dl_ptr[i + 1];
    uint64_t k = dl_ptr[i] + row_hot_count(hz, kw, i, a, b);
    if (k >= e) continue;
    const uint64_t pb = (row_base + i) / part_rows * y_card;
    const uint32_t comp = vmask & ~(a.x & vmask);  // the variants holding the row: v subset of comp
    const uint32_t rowv = (uint32_t)(row_base + i);
    // rec: the whole 16-byte record is written here (its hot word, folded tail
    // and flags are the row's); a scattered 16-byte store costs the same DRAM
    // sector as a 4-byte one
    const uint4 rv = make_uint4(a.x, a.y, a.z | a.w | b.x | b.y | b.z | b.w,
                                rowv | (row_sp && row_sp[i] ? 0x80000000u : 0u));
    for (; k < e; k += 4) {
      uint64_t g[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) g[u] = k + u < e ? pb + y_of_rank[dl_col[k + u]] : 0;
      for (uint32_t v = comp;; v = (v - 1) & comp) {
        if (v != vskip) {
          unsigned long long pos[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (k + u < e) pos[u] = atomicAdd(&cur[v * n_py + g[u]], 1ull);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (k + u < e) {
              if (rec) rec[pos[u]] = rv;
              else col[pos[u]] = rowv;
            }
        }
        if (v == 0) break;
      }
    }
  }
}

// Record row field: the dense row position, bit 31 set for a folded-in SPARSE
// z (row_sp), so the pairs of those rows are counted apart at insertion
// without a per-x readout of the dedup table. Rows < 2^31 - 1 (host check).
constexpr uint32_t kSpFlag = 0x80000000u;
constexpr uint32_t kRowMask = 0x7fffffffu;

__device__ __forceinline__ uint32_t fold_tail(const uint4& a0, const uint4& a1) {
  return a0.z | a0.w | a1.x | a1.y | a1.z | a1.w;
}

// ---- the hot filter on a record ----------------------------------------------

struct ColdX {  // x's side of the filter: hx[x] (ranks 0-127 | 128-255) and its fold
  uint4 a0, a1;
  uint32_t fold;
};
__device__ __forceinline__ ColdX cold_x(const uint4* __restrict__ hx4, uint32_t x) {
  ColdX s;
  ld256(hx4 + 2 * (uint64_t)x, s.a0, s.a1);
  s.fold = fold_tail(s.a0, s.a1);
  return s;
}
// x's cold-CSR variant: its top-var_bits hot mask (the skipped variant's x
// stream variant 0, which holds every row)
__device__ __forceinline__ uint32_t x_variant(uint32_t w0, uint32_t var_bits, uint32_t vskip) {
  const uint32_t v = w0 & ((1u << var_bits) - 1);
  return v == vskip ? 0u : v;
}
enum : uint32_t { kColdHot = 0, kColdSurvivor = 1, kColdMaybe = 2 };
__device__ __forceinline__ uint32_t cold_test(const uint4& c, const ColdX& s) {
  if ((c.x & s.a0.x) | (c.y & s.a0.y)) return kColdHot;
  return (c.z & s.fold) ? kColdMaybe : kColdSurvivor;
}
// exact test of a maybe: does z share a rank in [64, 256) with x?
__device__ __forceinline__ bool cold_tail_hot(uint32_t row, const ColdX& s,
                                              const uint4* __restrict__ hz4) {
  uint4 b0, b1;
  ld256(hz4 + 2 * (uint64_t)(row & kRowMask), b0, b1);
  return ((s.a0.z & b0.z) | (s.a0.w & b0.w) | (s.a1.x & b1.x) | (s.a1.y & b1.y) |
          (s.a1.z & b1.z) | (s.a1.w & b1.w)) != 0;
}
__device__ __forceinline__ uint4 ld_rec(const uint4* __restrict__ p) { return __ldg(p); }

#ifndef D3G_COLD_UNROLL
#define D3G_COLD_UNROLL 2
#endif
constexpr int kColdU = D3G_COLD_UNROLL;         // candidate windows in flight per warp
// The star segment (see warp_cold_x): D3G_STAR=0 compiles it out of the warp
// kernels (the A/B build); windows in flight per warp in its lookup loop.
#ifndef D3G_STAR
#define D3G_STAR 1
#endif
constexpr bool kStar = D3G_STAR != 0;
#ifndef D3G_STAR_WARP_UNROLL
#define D3G_STAR_WARP_UNROLL 1
#endif
#ifndef D3G_STAR_CTA_UNROLL
#define D3G_STAR_CTA_UNROLL 2
#endif
constexpr int kStarWarpU = D3G_STAR_WARP_UNROLL, kStarCtaU = D3G_STAR_CTA_UNROLL;
constexpr uint32_t kDQ = 32u * (kColdU + 1);    // per-warp deferred rows (<= 31 + 32 U)
constexpr uint32_t kSegWords = 32 * 3;          // per-warp compacted segments (u64 + u32)

// Deferred exact checks, per warp (qn warp-uniform).
__device__ __forceinline__ void dq_push(uint32_t* dq, uint32_t& qn, bool maybe, uint32_t row) {
  const uint32_t m = __ballot_sync(0xffffffffu, maybe);
  if (m) {
    if (maybe) dq[qn + __popc(m & ((1u << lane_id()) - 1u))] = row;
    qn += __popc(m);
    __syncwarp();
  }
}
// Resolve queued maybes 32 at a time (all: down to empty); ins(ok, row) is
// called by every lane (it may use warp collectives).
template <class Ins>
__device__ __forceinline__ void dq_drain(uint32_t* dq, uint32_t& qn, bool all, const ColdX& s,
                                         const uint4* __restrict__ hz4, uint64_t& ngat, Ins&& ins) {
  while (qn >= 32 || (all && qn > 0)) {
    const uint32_t n = qn < 32 ? qn : 32u;
    const uint32_t lane = lane_id();
    bool ok = false;
    uint32_t row = 0;
    if (lane < n) {
      row = dq[qn - n + lane];
      ok = !cold_tail_hot(row, s, hz4);
    }
    if (lane == 0) ngat += n;
    __syncwarp();
    qn -= n;
    ins(ok, row);
  }
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (uint32_t)o) v += u;
  }
  return v;
}

// Flattened candidate stream over the NONEMPTY segments of a chunk of x's y
// rows, compacted to sseg (CSR start) / sE (exclusive stream offset; strictly
// increasing). The stream is walked in 32-candidate windows: with c0 the
// segment holding the window start tb, lane j's candidate tb + j lies in
// segment c0 + #{segment starts in (tb, tb + j]}, read off the window's
// boundary mask (one REDUX.OR + one VOTE per window) instead of a
// per-candidate binary search.
__device__ __forceinline__ uint32_t warp_stream_init(uint64_t seg0, uint32_t len, uint64_t* sseg,
                                                     uint32_t* sE, uint32_t& n) {
  const uint32_t lane = lane_id();
  const uint32_t ne = __ballot_sync(0xffffffffu, len > 0);
  const uint32_t incl = warp_incl_scan(len);
  if (len) {
    const uint32_t c = __popc(ne & ((1u << lane) - 1u));
    sseg[c] = seg0;
    sE[c] = incl - len;
  }
  n = __popc(ne);
  __syncwarp();
  return __shfl_sync(0xffffffffu, incl, 31);
}
// CSR position of the lane's candidate in window [tb, tb + 32) (valid iff
// tb + lane < total); c0 advances to the segment holding tb + 32.
__device__ __forceinline__ uint64_t warp_window(uint32_t tb, uint32_t& c0, uint32_t n,
                                                const uint64_t* sseg, const uint32_t* sE) {
  const uint32_t lane = lane_id();
  const uint32_t s = c0 + 1 + lane;
  const uint32_t d = s < n ? sE[s] - tb : 64u;  // >= 1: segments after c0 start after tb
  const uint32_t M = __reduce_or_sync(0xffffffffu, d < 32u ? 1u << d : 0u);
  const uint32_t adv = __popc(__ballot_sync(0xffffffffu, d <= 32u));
  const uint32_t seg = c0 + __popc(M & ((2u << lane) - 1u));
  c0 += adv;
  return sseg[seg] + (tb + lane - sE[seg]);
}
// last segment whose stream offset is <= f (warp-uniform f: broadcast loads)
__device__ __forceinline__ uint32_t seg_search(uint32_t f, uint32_t n, const uint32_t* sE) {
  uint32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (sE[mid] <= f) lo = mid; else hi = mid;
  }
  return lo;
}

// CTA-wide version of warp_stream_init over blockDim.x segments (one per
// thread): a CTA scan of the lengths and of the nonempty flags compacts the
// nonempty segments into s_seg0 / s_off. Returns the chunk's candidate total.
template <int kThreads>
__device__ __forceinline__ uint32_t cta_stream_chunk(uint64_t sg0, uint32_t len, uint64_t* s_seg0,
                                                     uint32_t* s_off, uint32_t* s_wsum /*[2 kW]*/,
                                                     uint32_t* s_tot /*[2]*/, uint32_t& n) {
  constexpr uint32_t kW = kThreads / 32;
  static_assert(kW <= 32, "one warp scans the warp sums");
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t incl = warp_incl_scan(len);
  const uint32_t ne = __ballot_sync(0xffffffffu, len > 0);
  if (lane == 31) {
    s_wsum[warp] = incl;
    s_wsum[kW + warp] = __popc(ne);
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t wv = lane < kW ? s_wsum[lane] : 0u, wc = lane < kW ? s_wsum[kW + lane] : 0u;
    const uint32_t wi = warp_incl_scan(wv), ci = warp_incl_scan(wc);
    if (lane < kW) {
      s_wsum[lane] = wi - wv;  // exclusive over warps
      s_wsum[kW + lane] = ci - wc;
    }
    if (lane == kW - 1) {
      s_tot[0] = wi;
      s_tot[1] = ci;
    }
  }
  __syncthreads();
  if (len) {
    const uint32_t c = s_wsum[kW + warp] + __popc(ne & ((1u << lane) - 1u));
    s_off[c] = s_wsum[warp] + incl - len;
    s_seg0[c] = sg0;
  }
  __syncthreads();
  n = s_tot[1];
  return s_tot[0];
}

// Candidates streamed (16-byte records) and exact tail checks (32-byte hz
// rows): the cold pass's algorithmic traffic, cand[0] and cand[1].
__device__ __forceinline__ void flush_cand(unsigned long long* cand, uint64_t v, uint64_t g) {
  if (!cand) return;
  v = warp_sum(v);
  g = warp_sum(g);
  if (lane_id() == 0) {
    if (v) atomicAdd(cand, (unsigned long long)v);
    if (g) atomicAdd(cand + 1, (unsigned long long)g);
  }
}

template <int kMode>
__device__ __forceinline__ void cold_account(uint32_t x, uint32_t zc, const Decode& dec,
                                             const Emit& em, uint64_t& sum, uint64_t& xr) {
  if (kMode == kModeChecksum) {
    const uint64_t h = dec.hash(x, zc);
    sum += h;
    xr ^= h;
  } else if (kMode == kModeEmit) {
    const unsigned long long idx = atomicAdd(em.cursor, 1ull);
    if (idx < em.cap) {
      em.x[idx] = x;
      em.z[idx] = zc;
    }
  }
}

// The per-x candidate loop shared by the warp kernels: every chunk of 32 of
// x's y rows is compacted and streamed in windows of 32 candidates, kColdU
// windows in flight; `on(st, row)` gets every candidate (st: kColdHot for the
// lanes past the end), `step()` runs after each group of windows and returns
// false to stop x. Returns the candidates streamed (warp-uniform).
//
// The star segment. The rows of ONE segment are distinct (a y's list holds a
// row once), so the last segment an x streams needs no insertion: its
// survivors are new iff the dedup set built from the other segments does not
// hold them. With `defer` the LONGEST segment of x (of its last chunk of 32 y
// rows: nearly every x has one chunk) is left out of the stream and returned in
// (star0, star_len) for cold_star: under Zipf it carries most of x's
// candidates, so the set stays small (fewer overflows to the next tier, shorter
// probe chains) and those candidates cost a lookup, not a CAS. An x whose other
// segments pass route_min, or whose star passes star_route, is handed on
// (`routed`).
template <bool defer, class On, class Step>
__device__ __forceinline__ uint32_t warp_cold_x(uint32_t x, const ColdX& s,
                                                const uint64_t* __restrict__ r_ptr,
                                                const uint32_t* __restrict__ r_col,
                                                const uint64_t* __restrict__ cp,
                                                const uint4* __restrict__ crec, uint64_t* sseg,
                                                uint32_t* sE, uint32_t route_min, bool& routed,
                                                uint32_t star_route, uint64_t& star0,
                                                uint32_t& star_len, On&& on, Step&& step) {
  const uint32_t lane = lane_id();
  const uint64_t r0 = r_ptr[x], r1 = r_ptr[x + 1];
  uint32_t streamed = 0;
  routed = false;
  star0 = 0;
  star_len = 0;
  for (uint64_t kb = r0; kb < r1; kb += 32) {
    const uint64_t kk = kb + lane;
    uint64_t seg0 = 0, seg1 = 0;
    if (kk < r1) {
      const uint32_t y = r_col[kk];
      seg0 = cp[y];
      seg1 = cp[y + 1];
    }
    uint32_t len = (uint32_t)(seg1 - seg0);
    if (defer && kb + 32 >= r1) {  // the last chunk: its longest segment is the star
      const uint32_t m = __reduce_max_sync(0xffffffffu, len);
      if (m > star_route) {
        routed = true;
        return streamed;
      }
      if (m) {
        const int src = __ffs(__ballot_sync(0xffffffffu, len == m)) - 1;
        star0 = __shfl_sync(0xffffffffu, seg0, src);
        star_len = m;
        if ((int)lane == src) len = 0;
      }
    }
    uint32_t n;
    const uint32_t total = warp_stream_init(seg0, len, sseg, sE, n);
    if (streamed + total > route_min) {  // handed on before streaming
      routed = true;
      return streamed;
    }
    streamed += total;
    uint32_t c0 = 0;
    for (uint32_t tb = 0; tb < total; tb += 32 * kColdU) {
      uint64_t t[kColdU];
#pragma unroll
      for (int h = 0; h < kColdU; ++h)
        t[h] = tb + 32 * h < total ? warp_window(tb + 32 * h, c0, n, sseg, sE) : 0;
      uint4 c[kColdU];
#pragma unroll
      for (int h = 0; h < kColdU; ++h)
        if (tb + 32 * h + lane < total) c[h] = ld_rec(crec + t[h]);
#pragma unroll
      for (int h = 0; h < kColdU; ++h) {
        const bool ok = tb + 32 * h + lane < total;
        on(ok ? cold_test(c[h], s) : (uint32_t)kColdHot, ok ? c[h].w : 0u);
      }
      if (!step()) return streamed;
    }
    __syncwarp();  // sseg / sE are rewritten by the next chunk
  }
  return streamed;
}

// The star segment's candidates [first, star_len) in steps of `stride` windows
// groups (a warp alone: first 0, stride 1; a CTA: each warp its own groups):
// one contiguous run of records, so lane j of a window reads record tb + j (no
// segment mapping). fn(ok, row) is the lookup (called by every lane); maybes
// go through the warp's deferred queue as in the stream. Returns the lane's
// candidates read.
template <int kStarU, class Fn>
__device__ __forceinline__ uint32_t cold_star(uint64_t star0, uint32_t star_len, uint32_t first,
                                              uint32_t stride, const ColdX& s,
                                              const uint4* __restrict__ crec, uint32_t* dq,
                                              uint32_t& qn, const uint4* __restrict__ hz4,
                                              uint64_t& ngat, Fn&& fn) {
  const uint32_t lane = lane_id();
  const uint4* p = crec + star0;
  uint32_t mine = 0;
  for (uint32_t tb = first * (32 * kStarU); tb < star_len; tb += stride * (32 * kStarU)) {
    uint4 c[kStarU];
#pragma unroll
    for (int h = 0; h < kStarU; ++h)
      if (tb + 32 * h + lane < star_len) {
        ++mine;
        c[h] = ld_rec(p + tb + 32 * h + lane);
      }
#pragma unroll
    for (int h = 0; h < kStarU; ++h) {
      const bool ok = tb + 32 * h + lane < star_len;
      const uint32_t st = ok ? cold_test(c[h], s) : (uint32_t)kColdHot;
      const uint32_t row = ok ? c[h].w : 0u;
      fn(st == kColdSurvivor, row);
      dq_push(dq, qn, st == kColdMaybe, row);
      dq_drain(dq, qn, false, s, hz4, ngat, fn);  // the queue holds <= 31 + 32
    }
  }
  dq_drain(dq, qn, true, s, hz4, ngat, fn);
  return mine;
}

// The CTA kernels' star: the longest segment among x's y rows [r0, r1), by a
// CTA-wide max of (length, first index). Returns its index in r_col (~0: x has
// no candidates). s_best is zero on entry; the caller syncs before reuse.
template <int kThreads>
__device__ __forceinline__ uint64_t cta_star(uint64_t r0, uint64_t r1,
                                             const uint32_t* __restrict__ r_col,
                                             const uint64_t* __restrict__ cp,
                                             unsigned long long* s_best, uint64_t& star0,
                                             uint32_t& star_len) {
  unsigned long long best = 0;
  for (uint64_t k = r0 + threadIdx.x; k < r1; k += kThreads) {
    const uint32_t y = r_col[k];
    const unsigned long long len = cp[y + 1] - cp[y];
    const unsigned long long key = (len << 32) | (0xffffffffull - (k - r0));
    best = key > best ? key : best;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long u = __shfl_xor_sync(0xffffffffu, best, o);
    best = u > best ? u : best;
  }
  if (lane_id() == 0 && (best >> 32)) atomicMax(s_best, best);
  __syncthreads();
  const unsigned long long b = *(volatile unsigned long long*)s_best;
  star_len = (uint32_t)(b >> 32);
  star0 = 0;
  if (!star_len) return ~0ull;
  const uint64_t kstar = r0 + (0xffffffffull - (b & 0xffffffffull));
  star0 = cp[r_col[kstar]];
  return kstar;
}

// ---- P2 with warp-private bitmaps (at most 16 row partitions: cfg2, cfg4) -----

constexpr int kColdWarps = 8;  // warps per CTA (several CTAs per SM)

template <int kMode>
__global__ void __launch_bounds__(kColdWarps * 32, 4)
dense_cold_kernel(const uint32_t* __restrict__ xs, uint64_t n_x,
                  const uint64_t* __restrict__ r_ptr, const uint32_t* __restrict__ r_col,
                  const uint64_t* __restrict__ cptr /* [var][parts][y_card] + 1 */,
                  const uint4* __restrict__ crec, const uint4* __restrict__ hz4,
                  const uint4* __restrict__ hx4, uint64_t y_card, uint32_t parts,
                  uint32_t part_rows, uint32_t var_bits, uint32_t vskip,
                  const uint32_t* __restrict__ dl_z,
                  Decode dec, Emit em, unsigned int* __restrict__ next, Tally* tally,
                  unsigned long long* __restrict__ cnt_sp,
                  unsigned long long* __restrict__ cand = nullptr) {
  // [kColdWarps][part_rows / 32] bitmaps, [kColdWarps][kDQ] deferred rows,
  // [kColdWarps][kSegWords] compacted segments
  extern __shared__ __align__(16) uint32_t cbm[];
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  const uint32_t pw = part_rows / 32;
  uint32_t* bm = cbm + (uint64_t)w * pw;
  uint32_t* dq = cbm + (uint64_t)kColdWarps * pw + w * kDQ;
  uint64_t* sseg = reinterpret_cast<uint64_t*>(cbm + (uint64_t)kColdWarps * (pw + kDQ)) + w * 32;
  uint32_t* sE = cbm + (uint64_t)kColdWarps * (pw + kDQ + 64) + w * 32;
  for (uint32_t i = lane; i < pw; i += 32) bm[i] = 0;
  __syncwarp();
  uint64_t cnt = 0, sum = 0, xr = 0, csp = 0, ncand = 0, ngat = 0;
  const uint64_t n_items = n_x * parts;
  uint32_t item_next = 0;
  if (lane == 0) item_next = atomicAdd(next, 1u);
  for (;;) {
    const uint32_t item = __shfl_sync(0xffffffffu, item_next, 0);
    if (item >= n_items) break;
    if (lane == 0) item_next = atomicAdd(next, 1u);  // consumed next iteration
    const uint32_t part = (uint32_t)(item / n_x);
    const uint32_t x = xs[item % n_x];
    const uint32_t zbase = part * part_rows;
    const ColdX s = cold_x(hx4, x);
    const uint32_t v = x_variant(s.a0.x, var_bits, vskip);
    const uint64_t* cp = cptr + ((uint64_t)v * parts + part) * y_card;
    bool touched = false;
    uint32_t qn = 0;
    auto ins = [&](bool ok, uint32_t row) {
      bool fresh = false;
      const uint32_t zl = (row & kRowMask) - zbase;
      if (ok) {
        const uint32_t bit = 1u << (zl & 31);
        const uint32_t old = atomicOr(&bm[zl >> 5], bit);
        touched = true;
        fresh = (old & bit) == 0;
      }
      if (fresh) {
        ++cnt;
        if (row & kSpFlag) ++csp;
        if (kMode == kModeChecksum) {
          const uint64_t hh = dec.hash(x, dl_z[row & kRowMask]);
          sum += hh;
          xr ^= hh;
        }
      }
      if (kMode == kModeEmit) {  // warp-aggregated reservation
        const unsigned long long slot = warp_reserve(em, fresh ? 1u : 0u);
        if (fresh) emit_at(em, slot, x, dl_z[row & kRowMask]);
      }
    };
    // no star segment here: an atomicOr on the warp's bitmap costs what a bit
    // test does (cfg2 0.65 -> 0.79 ms with it)
    bool routed;
    uint64_t star0;
    uint32_t star_len;
    ncand += warp_cold_x<false>(
        x, s, r_ptr, r_col, cp, crec, sseg, sE, 0xffffffffu, routed, 0xffffffffu, star0, star_len,
        [&](uint32_t st, uint32_t row) {
          ins(st == kColdSurvivor, row);
          dq_push(dq, qn, st == kColdMaybe, row);
        },
        [&]() {
          dq_drain(dq, qn, false, s, hz4, ngat, ins);
          return true;
        });
    dq_drain(dq, qn, true, s, hz4, ngat, ins);
    __syncwarp();
    if (__any_sync(0xffffffffu, touched))
      for (uint32_t i = lane; i < pw; i += 32) bm[i] = 0;
    __syncwarp();
  }
  if (lane != 0) ncand = 0;
  flush_sp(cnt_sp, csp);
  flush_cand(cand, ncand, ngat);
  tally_flush(tally, cnt, sum, xr);
}

// ---- P2 with warp-private hash sets (larger dense blocks: cfg5's 10M rows) ----
//
// An x whose survivors exceed ch_max abandons the hash (nothing of it was
// counted) and is queued for dense_cold_cta_kernel; so is an x whose candidate
// stream exceeds route_min before it is read (it would overflow: the stream
// is not read twice). Count (and the folded-sparse count) are tallied at
// insertion and credited when x completes; fingerprint and emission are read
// from the table, so abandoning is exact.
constexpr int kCHWarps = 8;
// 1024 slots per warp and 4 CTAs per SM (cfg5 cold pass, round 1: 2048 slots
// x 3 CTAs 61 ms, 1024 x 4 52 ms, 512 x 4 58 ms)
#ifndef D3G_CH_BITS
#define D3G_CH_BITS 10
#endif
constexpr uint32_t kCHSlots = 1u << D3G_CH_BITS;
#ifndef D3G_CH_LOAD
#define D3G_CH_LOAD 84  // percent (double hashing: cfg5 60% 90.5, 75% 87.8, 84% 86.5 ms)
#endif
constexpr uint32_t kCHMax = kCHSlots * D3G_CH_LOAD / 100;  // load limit; < kCHSlots - 160 keeps probing finite
constexpr uint32_t kCHEmpty = 0xffffffffu;
#ifndef D3G_CH_CTAS
#define D3G_CH_CTAS 4
#endif
#ifndef D3G_COLD_ROUTE
#define D3G_COLD_ROUTE 8192
#endif
constexpr size_t kCHSmem = (size_t)kCHWarps * (kCHSlots + kDQ + kSegWords) * 4;

__device__ __forceinline__ uint32_t ch_slot(uint32_t v) { return (v * 0x9E3779B1u) >> (32 - D3G_CH_BITS); }
// odd probe step (covers every slot of a power-of-two table)
__device__ __forceinline__ uint32_t probe_step(uint32_t v) { return ((v * 0x85EBCA6Bu) >> 20) | 1u; }

template <int kMode>
__global__ void __launch_bounds__(kCHWarps * 32, D3G_CH_CTAS)
dense_cold_hash_kernel(const uint32_t* __restrict__ xs, uint64_t n_x,
                       const uint64_t* __restrict__ r_ptr, const uint32_t* __restrict__ r_col,
                       const uint64_t* __restrict__ cptr, const uint4* __restrict__ crec,
                       const uint4* __restrict__ hz4, const uint4* __restrict__ hx4,
                       uint64_t y_card, uint32_t var_bits, uint32_t vskip,
                       const uint32_t* __restrict__ dl_z,
                       Decode dec, Emit em, unsigned int* __restrict__ next,
                       uint32_t* __restrict__ over_x, unsigned int* __restrict__ over_n,
                       Tally* tally, unsigned long long* __restrict__ cnt_sp, uint32_t ch_max,
                       uint32_t route_min, uint32_t star_route,
                       unsigned long long* __restrict__ cand = nullptr) {
  // [kCHWarps][kCHSlots] tables, [kCHWarps][kDQ] deferred rows,
  // [kCHWarps][kSegWords] compacted segments
  extern __shared__ __align__(16) uint32_t chtab[];
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  uint32_t* tab = chtab + (uint64_t)w * kCHSlots;
  uint32_t* dq = chtab + (uint64_t)kCHWarps * kCHSlots + w * kDQ;
  uint64_t* sseg = reinterpret_cast<uint64_t*>(chtab + (uint64_t)kCHWarps * (kCHSlots + kDQ)) + w * 32;
  uint32_t* sE = chtab + (uint64_t)kCHWarps * (kCHSlots + kDQ + 64) + w * 32;
  for (uint32_t i = lane; i < kCHSlots; i += 32) tab[i] = kCHEmpty;
  __syncwarp();
  uint64_t cnt = 0, sum = 0, xr = 0, csp = 0, ncand = 0, ngat = 0;
  uint32_t item_next = 0;
  if (lane == 0) item_next = atomicAdd(next, 1u);
  for (;;) {
    const uint32_t item = __shfl_sync(0xffffffffu, item_next, 0);
    if (item >= n_x) break;
    if (lane == 0) item_next = atomicAdd(next, 1u);  // consumed next iteration
    const uint32_t x = xs[item];
    const ColdX s = cold_x(hx4, x);
    const uint32_t v = x_variant(s.a0.x, var_bits, vskip);
    const uint64_t* cp = cptr + (uint64_t)v * y_card;
    uint32_t inserted = 0;  // warp-uniform
    uint32_t qn = 0;
    uint64_t xgat = 0, xsp = 0;  // credited only if x completes in this tier
    auto ins = [&](bool ok, uint32_t key) {
      bool fresh = false;
      if (ok) {
        uint32_t sl = ch_slot(key);
        const uint32_t step = probe_step(key);  // double hashing: short chains at high load
        for (;;) {
          const uint32_t prev = atomicCAS(&tab[sl], kCHEmpty, key);
          if (prev == kCHEmpty) {
            fresh = true;
            break;
          }
          if (prev == key) break;
          sl = (sl + step) & (kCHSlots - 1);
        }
      }
      if (fresh && (key & kSpFlag)) ++xsp;
      inserted += __popc(__ballot_sync(0xffffffffu, fresh));
    };
    bool routed;
    uint64_t star0;
    uint32_t star_len;
    const uint32_t streamed = warp_cold_x<kStar>(
        x, s, r_ptr, r_col, cp, crec, sseg, sE, route_min, routed, star_route, star0, star_len,
        [&](uint32_t st, uint32_t row) {
          ins(st == kColdSurvivor, row);
          dq_push(dq, qn, st == kColdMaybe, row);
        },
        [&]() {
          dq_drain(dq, qn, false, s, hz4, xgat, ins);
          return inserted <= ch_max;
        });
    bool over = routed || inserted > ch_max;
    if (!over) {
      dq_drain(dq, qn, true, s, hz4, xgat, ins);
      over = inserted > ch_max;
    }
    __syncwarp();
    uint32_t star_new = 0;  // warp-uniform
    if (!over && star_len) {
      // the star segment: looked up in the finished set, never inserted
      auto look = [&](bool ok, uint32_t key) {
        bool fresh = ok;
        if (ok && inserted) {
          uint32_t sl = ch_slot(key);
          const uint32_t step = probe_step(key);
          for (;;) {
            const uint32_t cur = tab[sl];
            if (cur == kCHEmpty) break;
            if (cur == key) {
              fresh = false;
              break;
            }
            sl = (sl + step) & (kCHSlots - 1);
          }
        }
        if (fresh && (key & kSpFlag)) ++xsp;
        star_new += __popc(__ballot_sync(0xffffffffu, fresh));
        if (kMode == kModeChecksum && fresh)
          cold_account<kMode>(x, dl_z[key & kRowMask], dec, em, sum, xr);
        if (kMode == kModeEmit) {
          const unsigned long long slot = warp_reserve(em, fresh ? 1u : 0u);
          if (fresh) emit_at(em, slot, x, dl_z[key & kRowMask]);
        }
      };
      cold_star<kStarWarpU>(star0, star_len, 0, 1, s, crec, dq, qn, hz4, xgat, look);
    }
    if (over) {
      if (lane == 0) over_x[atomicAdd(over_n, 1u)] = x;
    } else {
      cnt += lane == 0 ? inserted + star_new : 0;
      // x's stream counted once, in the tier that finishes it
      ncand += lane == 0 ? streamed + star_len : 0;
      ngat += xgat;
      csp += xsp;
    }
    if (inserted && kMode != kModeCount) {
      for (uint32_t i = lane; i < kCHSlots; i += 32) {  // uniform trip count
        const uint32_t key = tab[i];
        if (kMode == kModeEmit) {  // warp-aggregated reservation
          const bool e = key != kCHEmpty && !over;
          const unsigned long long slot = warp_reserve(em, e ? 1u : 0u);
          if (e) emit_at(em, slot, x, dl_z[key & kRowMask]);
        }
        if (key != kCHEmpty) {
          if (!over && kMode == kModeChecksum)
            cold_account<kMode>(x, dl_z[key & kRowMask], dec, em, sum, xr);
          tab[i] = kCHEmpty;
        }
      }
    } else if (inserted) {
      // count only: nothing to read back, reset the table with 16-byte stores
      uint4* t4 = reinterpret_cast<uint4*>(tab);
      const uint4 e4 = make_uint4(kCHEmpty, kCHEmpty, kCHEmpty, kCHEmpty);
#pragma unroll 4
      for (uint32_t i = lane; i < kCHSlots / 4; i += 32) t4[i] = e4;
    }
    __syncwarp();
  }
  flush_sp(cnt_sp, csp);
  flush_cand(cand, ncand, ngat);
  tally_flush(tally, cnt, sum, xr);
}

// The per-x candidate loop of the CTA kernels: chunks of kThreads of x's y
// rows, compacted across the CTA; each warp walks one contiguous share of the
// chunk's candidates in 32-candidate windows (its first segment by one
// warp-uniform binary search, the rest from the windows' boundary masks). Candidates are handed to on(st, row) as in
// warp_cold_x; step() runs after each group of windows (per warp). The loop
// stops at the next check once *stop is set (CTA-uniform). Returns this
// thread's candidates streamed. The segment of r_col index kstar (the star
// segment, see warp_cold_x) is left out.
template <int kThreads, class On, class Step>
__device__ __forceinline__ uint64_t cta_cold_x(const ColdX& s, uint64_t r0, uint64_t r1,
                                               const uint32_t* __restrict__ r_col,
                                               const uint64_t* __restrict__ cp,
                                               const uint4* __restrict__ crec, uint64_t* s_seg0,
                                               uint32_t* s_off, uint32_t* s_wsum, uint32_t* s_tot,
                                               const volatile unsigned int* stop, uint64_t kstar,
                                               On&& on, Step&& step, uint32_t share = 0,
                                               uint32_t n_shares = 1) {
  // (share / n_shares: this CTA streams that part of every chunk -- several
  // CTAs working on one x, dense_cold_shared_kernel)
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint64_t mine = 0;
  for (uint64_t yb = r0; yb < r1 && !*stop; yb += kThreads) {
    const uint64_t k = yb + threadIdx.x;
    uint64_t sg0 = 0;
    uint32_t len = 0;
    if (k < r1) {
      const uint32_t y = r_col[k];
      sg0 = cp[y];
      len = k == kstar ? 0u : (uint32_t)(cp[y + 1] - sg0);  // the star segment is left out
    }
    uint32_t n;
    const uint32_t total = cta_stream_chunk<kThreads>(sg0, len, s_seg0, s_off, s_wsum, s_tot, n);
    // each warp streams one contiguous share of the chunk: its first segment
    // by one binary search, then the windows advance it from their masks
    constexpr uint32_t kW = kThreads / 32;
    const uint32_t nw = kW * n_shares;
    const uint32_t per = ((total + nw - 1) / nw + 31) & ~31u;
    // (64-bit: (share * kW + warp) * per can pass 2^32 only with total near it)
    const uint32_t beg = (uint32_t)min((uint64_t)total, (uint64_t)(share * kW + warp) * per);
    const uint32_t end = min(total, beg + per);
    uint32_t c0 = beg < end ? seg_search(beg, n, s_off) : 0u;
    for (uint32_t tb = beg; tb < end && !*stop; tb += 32 * kColdU) {
      uint64_t t[kColdU];
#pragma unroll
      for (int u = 0; u < kColdU; ++u) {
        const uint32_t wb = tb + 32 * u;
        t[u] = wb < end ? warp_window(wb, c0, n, s_seg0, s_off) : 0;
      }
      uint4 c[kColdU];
#pragma unroll
      for (int u = 0; u < kColdU; ++u)
        if (tb + 32 * u + lane < end) {
          ++mine;
          c[u] = ld_rec(crec + t[u]);
        }
#pragma unroll
      for (int u = 0; u < kColdU; ++u) {
        const bool ok = tb + 32 * u + lane < end;
        on(ok ? cold_test(c[u], s) : (uint32_t)kColdHot, ok ? c[u].w : 0u);
      }
      step();
    }
    __syncthreads();  // s_off / s_seg0 are rewritten by the next chunk
  }
  return mine;
}

// ---- overflow tier 1: one CTA per x, CTA-wide shared-memory hash -------------
//
// The same candidate stream flattened across the CTA; survivors in a kCCSlots
// CTA-wide hash (no global bitmap: those are 1.25 MB per CTA on cfg5 and
// thrash L2). An x whose survivors pass cc_max is abandoned exactly and
// queued for the bitmap kernel.
#ifndef D3G_CC_BITS
#define D3G_CC_BITS 15
#endif
#ifndef D3G_CC_THREADS
#define D3G_CC_THREADS 1024
#endif
constexpr int kCCThreads = D3G_CC_THREADS;
constexpr uint32_t kCCSlots = 1u << D3G_CC_BITS;  // 128 KB at 15 bits
#ifndef D3G_CC_LOAD
#define D3G_CC_LOAD 85  // percent
#endif
constexpr uint32_t kCCMax = kCCSlots * D3G_CC_LOAD / 100;  // load limit
constexpr int kCCPerSm = (1024 / D3G_CC_THREADS) * (D3G_CC_BITS >= 15 ? 1 : 2) > 2
                             ? 2 : (1024 / D3G_CC_THREADS) * (D3G_CC_BITS >= 15 ? 1 : 2);
constexpr size_t kCCSmem = (size_t)kCCSlots * 4 + (size_t)(kCCThreads / 32) * kDQ * 4;

__device__ __forceinline__ uint32_t cc_slot(uint32_t v) { return (v * 0x9E3779B1u) >> (32 - D3G_CC_BITS); }

template <int kMode>
__global__ void __launch_bounds__(kCCThreads, kCCPerSm)
dense_cold_cta_kernel(const uint32_t* __restrict__ over_x, const unsigned int* __restrict__ over_n,
                      const uint64_t* __restrict__ r_ptr, const uint32_t* __restrict__ r_col,
                      const uint64_t* __restrict__ cptr, const uint4* __restrict__ crec,
                      const uint4* __restrict__ hz4, const uint4* __restrict__ hx4,
                      uint64_t y_card, uint32_t var_bits, uint32_t vskip,
                      const uint32_t* __restrict__ dl_z,
                      Decode dec, Emit em, uint32_t* __restrict__ over2_x,
                      unsigned int* __restrict__ over2_n, uint32_t cc_max, Tally* tally,
                      unsigned long long* __restrict__ cnt_sp,
                      unsigned long long* __restrict__ cand = nullptr) {
  __shared__ uint64_t s_seg0[kCCThreads];
  __shared__ uint32_t s_off[kCCThreads];
  __shared__ uint32_t s_wsum[2 * (kCCThreads / 32)];
  __shared__ uint32_t s_tot[2];
  __shared__ unsigned int s_ins, s_over, s_star;
  __shared__ unsigned long long s_best;
  extern __shared__ __align__(16) uint32_t cctab[];  // [kCCSlots], [warps][kDQ]
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t* dq = cctab + kCCSlots + warp * kDQ;
  for (uint32_t i = threadIdx.x; i < kCCSlots; i += kCCThreads) cctab[i] = kCHEmpty;
  const uint32_t n = *over_n;
  uint64_t cnt = 0, sum = 0, xr = 0, csp = 0, ncand = 0, ngat = 0;
  for (uint32_t it = blockIdx.x; it < n; it += gridDim.x) {
    const uint32_t x = over_x[it];
    const ColdX s = cold_x(hx4, x);
    const uint32_t v = x_variant(s.a0.x, var_bits, vskip);
    const uint64_t* cp = cptr + (uint64_t)v * y_card;
    const uint64_t r0 = r_ptr[x], r1 = r_ptr[x + 1];
    if (threadIdx.x == 0) {
      s_ins = 0;
      s_over = 0;
      s_star = 0;
      s_best = 0;
    }
    __syncthreads();
    uint64_t star0 = 0;
    uint32_t star_len = 0;
    const uint64_t kstar =
        kStar ? cta_star<kCCThreads>(r0, r1, r_col, cp, &s_best, star0, star_len) : ~0ull;
    uint64_t xgat = 0, xsp = 0;  // credited only if x completes in this tier
    uint32_t qn = 0;
    uint32_t nf = 0;  // fresh inserts by this thread since the last flush
    auto ins = [&](bool ok, uint32_t key) {
      if (!ok) return;
      uint32_t sl = cc_slot(key);
      const uint32_t step = probe_step(key);
      for (uint32_t probe = 0; probe < kCCSlots; ++probe) {
        const uint32_t prev = atomicCAS(&cctab[sl], kCHEmpty, key);
        if (prev == kCHEmpty) {
          ++nf;
          if (key & kSpFlag) ++xsp;
          break;
        }
        if (prev == key) break;
        sl = (sl + step) & (kCCSlots - 1);
      }
    };
    auto flush_ins = [&]() {
      const uint32_t wf = warp_sum(nf);
      nf = 0;
      if (lane == 0 && wf && atomicAdd(&s_ins, wf) + wf > cc_max) s_over = 1;
    };
    uint64_t xcand = cta_cold_x<kCCThreads>(
        s, r0, r1, r_col, cp, crec, s_seg0, s_off, s_wsum, s_tot, &s_over, kstar,
        [&](uint32_t st, uint32_t row) {
          ins(st == kColdSurvivor, row);
          dq_push(dq, qn, st == kColdMaybe, row);
        },
        [&]() {
          dq_drain(dq, qn, false, s, hz4, xgat, ins);
          flush_ins();
        });
    if (!*(volatile unsigned int*)&s_over) {
      dq_drain(dq, qn, true, s, hz4, xgat, ins);
      flush_ins();
    }
    __syncthreads();  // the set is complete
    const bool over = s_over != 0;
    if (!over && star_len) {
      // the star segment: looked up in the finished set, never inserted
      uint32_t ns = 0;
      auto look = [&](bool ok, uint32_t key) {
        bool fresh = ok;
        if (ok) {
          uint32_t sl = cc_slot(key);
          const uint32_t step = probe_step(key);
          for (;;) {
            const uint32_t cur = cctab[sl];
            if (cur == kCHEmpty) break;
            if (cur == key) {
              fresh = false;
              break;
            }
            sl = (sl + step) & (kCCSlots - 1);
          }
        }
        if (fresh) {
          ++ns;
          if (key & kSpFlag) ++xsp;
          if (kMode == kModeChecksum)
            cold_account<kMode>(x, dl_z[key & kRowMask], dec, em, sum, xr);
        }
        if (kMode == kModeEmit) {
          const unsigned long long slot = warp_reserve(em, fresh ? 1u : 0u);
          if (fresh) emit_at(em, slot, x, dl_z[key & kRowMask]);
        }
      };
      qn = 0;
      xcand += cold_star<kStarCtaU>(star0, star_len, warp, kCCThreads / 32, s, crec, dq, qn, hz4, xgat, look);
      ns = warp_sum(ns);
      if (lane == 0 && ns) atomicAdd(&s_star, ns);
      __syncthreads();
    }
    if (over) {
      if (threadIdx.x == 0) over2_x[atomicAdd(over2_n, 1u)] = x;
    } else {
      ncand += xcand;
      ngat += xgat;
      csp += xsp;
      if (threadIdx.x == 0) cnt += s_ins + s_star;
    }
    if (kMode != kModeCount) {
      for (uint32_t i = threadIdx.x; i < kCCSlots; i += kCCThreads) {  // uniform trip count
        const uint32_t key = cctab[i];
        if (kMode == kModeEmit) {  // warp-aggregated reservation
          const bool e = key != kCHEmpty && !over;
          const unsigned long long slot = warp_reserve(em, e ? 1u : 0u);
          if (e) emit_at(em, slot, x, dl_z[key & kRowMask]);
        }
        if (key != kCHEmpty) {
          if (!over && kMode == kModeChecksum)
            cold_account<kMode>(x, dl_z[key & kRowMask], dec, em, sum, xr);
          cctab[i] = kCHEmpty;
        }
      }
    } else {
      // count only: reset the table with 16-byte stores
      uint4* t4 = reinterpret_cast<uint4*>(cctab);
      const uint4 e4 = make_uint4(kCHEmpty, kCHEmpty, kCHEmpty, kCHEmpty);
      for (uint32_t i = threadIdx.x; i < kCCSlots / 4; i += kCCThreads) t4[i] = e4;
    }
    __syncthreads();
  }
  flush_sp(cnt_sp, csp);
  flush_cand(cand, ncand, ngat);
  tally_flush(tally, cnt, sum, xr);
}

// ---- overflow tier 2: one CTA per x over a CTA-private global bitmap ---------
//
// The bitmap (one bit per dense row) is zero on entry and on exit: the words
// x made non-zero are listed and cleared; if the list overflows, the stream
// is replayed to clear every word it could have touched.
constexpr int kOvThreads = 512;
#ifndef D3G_OV_CTAS
#define D3G_OV_CTAS 3
#endif
constexpr int kOvPerSm = D3G_OV_CTAS;
constexpr uint32_t kOvTouched = 65536;  // touched-word list per CTA
constexpr size_t kOvSmem = (size_t)(kOvThreads / 32) * kDQ * 4;

template <int kMode>
__global__ void __launch_bounds__(kOvThreads, kOvPerSm)
dense_cold_overflow_kernel(const uint32_t* __restrict__ over_x, const unsigned int* __restrict__ over_n,
                           const uint64_t* __restrict__ r_ptr, const uint32_t* __restrict__ r_col,
                           const uint64_t* __restrict__ cptr, const uint4* __restrict__ crec,
                           const uint4* __restrict__ hz4, const uint4* __restrict__ hx4,
                           uint64_t y_card, uint32_t var_bits, uint32_t vskip,
                           const uint32_t* __restrict__ dl_z,
                           uint32_t* __restrict__ gbm, uint64_t words, Decode dec, Emit em,
                           Tally* tally, unsigned long long* __restrict__ cnt_sp,
                           uint32_t* __restrict__ touched /* [gridDim.x][kOvTouched] */,
                           unsigned long long* __restrict__ cand = nullptr) {
  __shared__ uint64_t s_seg0[kOvThreads];
  __shared__ uint32_t s_off[kOvThreads];
  __shared__ uint32_t s_wsum[2 * (kOvThreads / 32)];
  __shared__ uint32_t s_tot[2];
  __shared__ unsigned int s_nt;  // bitmap words this x made non-zero (touched list)
  __shared__ unsigned int s_never;  // 0: the candidate loop never stops early
  __shared__ unsigned long long s_best;
  extern __shared__ __align__(16) uint32_t ovdq[];  // [warps][kDQ]
  uint32_t* tl = touched + (uint64_t)blockIdx.x * kOvTouched;
  const uint32_t warp = threadIdx.x >> 5;
  uint32_t* dq = ovdq + warp * kDQ;
  uint32_t* bm = gbm + (uint64_t)blockIdx.x * words;
  const uint32_t n = *over_n;
  if (threadIdx.x == 0) s_never = 0;
  uint64_t cnt = 0, sum = 0, xr = 0, csp = 0, ncand = 0, ngat = 0;
  for (uint32_t it = blockIdx.x; it < n; it += gridDim.x) {
    const uint32_t x = over_x[it];
    const ColdX s = cold_x(hx4, x);
    const uint32_t v = x_variant(s.a0.x, var_bits, vskip);
    const uint64_t* cp = cptr + (uint64_t)v * y_card;
    const uint64_t r0 = r_ptr[x], r1 = r_ptr[x + 1];
    if (threadIdx.x == 0) {
      s_nt = 0;
      s_best = 0;
    }
    __syncthreads();
    uint64_t star0 = 0;
    uint32_t star_len = 0;
    const uint64_t kstar =
        kStar ? cta_star<kOvThreads>(r0, r1, r_col, cp, &s_best, star0, star_len) : ~0ull;
    auto ins = [&](bool ok, uint32_t key) {
      if (!ok) return;
      const uint32_t zl = key & kRowMask;
      const uint32_t bit = 1u << (zl & 31);
      const uint32_t old = atomicOr(&bm[zl >> 5], bit);
      if (old & bit) return;
      if (old == 0) {
        const unsigned int slot = atomicAdd(&s_nt, 1u);
        if (slot < kOvTouched) tl[slot] = zl >> 5;
      }
      ++cnt;
      if (key & kSpFlag) ++csp;
      if (kMode != kModeCount) cold_account<kMode>(x, dl_z[zl], dec, em, sum, xr);
    };
    uint32_t qn = 0;
    ncand += cta_cold_x<kOvThreads>(
        s, r0, r1, r_col, cp, crec, s_seg0, s_off, s_wsum, s_tot, &s_never, kstar,
        [&](uint32_t st, uint32_t row) {
          ins(st == kColdSurvivor, row);
          dq_push(dq, qn, st == kColdMaybe, row);
        },
        [&]() { dq_drain(dq, qn, false, s, hz4, ngat, ins); });
    dq_drain(dq, qn, true, s, hz4, ngat, ins);
    __syncthreads();  // the bitmap is complete
    if (star_len) {
      // the star segment: a bit test (L2 reads: the bits were set by atomics),
      // nothing written, so its words need no clearing either
      auto look = [&](bool ok, uint32_t key) {
        if (!ok) return;
        const uint32_t zl = key & kRowMask;
        if ((__ldcg(&bm[zl >> 5]) >> (zl & 31)) & 1u) return;
        ++cnt;
        if (key & kSpFlag) ++csp;
        if (kMode != kModeCount) cold_account<kMode>(x, dl_z[zl], dec, em, sum, xr);
      };
      qn = 0;
      ncand += cold_star<kStarCtaU>(star0, star_len, warp, kOvThreads / 32, s, crec, dq, qn, hz4, ngat, look);
      __syncthreads();
    }
    // clear through the touched list; replay the stream only if it overflowed
    const uint32_t nt = s_nt;
    if (nt <= kOvTouched) {
      for (uint32_t i = threadIdx.x; i < nt; i += kOvThreads) bm[tl[i]] = 0;
    } else {
      uint32_t dummy = 0;
      cta_cold_x<kOvThreads>(
          s, r0, r1, r_col, cp, crec, s_seg0, s_off, s_wsum, s_tot, &s_never, kstar,
          [&](uint32_t st, uint32_t row) {
            if (st != kColdHot) bm[(row & kRowMask) >> 5] = 0;  // clearing an untouched word is harmless
          },
          [&]() { ++dummy; });
    }
    __syncthreads();
  }
  flush_sp(cnt_sp, csp);
  flush_cand(cand, ncand, ngat);
  tally_flush(tally, cnt, sum, xr);
}

// ---- overflow tier 2, shared bitmaps: several CTAs per x ------------------------
//
// The x that reach the bitmap tier are few and huge (cfg5: 436 x, up to ~1M
// candidates each): with one CTA per x the tier lasts as long as its longest
// x. Here every x of a round owns a zeroed global bitmap and kOvShare CTAs
// stream one share each of its candidates; atomicOr's return value makes the
// count exact across CTAs. The star segment needs the finished bitmap, so the
// tier is two launches: phase 0 inserts everything but the star, phase 1
// tests the star's survivors against the bitmap. Nothing is cleared (the
// round's bitmaps are zeroed by one memset).
#ifndef D3G_OV_SHARE
#define D3G_OV_SHARE 4
#endif
constexpr uint32_t kOvShare = D3G_OV_SHARE;

template <int kMode>
__global__ void __launch_bounds__(kOvThreads, kOvPerSm)
dense_cold_shared_kernel(const uint32_t* __restrict__ over_x, uint32_t x_lo, uint32_t x_n,
                         int phase, const uint64_t* __restrict__ r_ptr,
                         const uint32_t* __restrict__ r_col, const uint64_t* __restrict__ cptr,
                         const uint4* __restrict__ crec, const uint4* __restrict__ hz4,
                         const uint4* __restrict__ hx4, uint64_t y_card, uint32_t var_bits,
                         uint32_t vskip, const uint32_t* __restrict__ dl_z,
                         uint32_t* __restrict__ gbm, uint64_t words, Decode dec, Emit em,
                         Tally* tally, unsigned long long* __restrict__ cnt_sp,
                         unsigned long long* __restrict__ cand = nullptr) {
  __shared__ uint64_t s_seg0[kOvThreads];
  __shared__ uint32_t s_off[kOvThreads];
  __shared__ uint32_t s_wsum[2 * (kOvThreads / 32)];
  __shared__ uint32_t s_tot[2];
  __shared__ unsigned int s_never;  // 0: the candidate loop never stops early
  __shared__ unsigned long long s_best;
  extern __shared__ __align__(16) uint32_t ovdq[];  // [warps][kDQ]
  const uint32_t warp = threadIdx.x >> 5;
  uint32_t* dq = ovdq + warp * kDQ;
  const uint32_t xi = blockIdx.x / kOvShare, share = blockIdx.x % kOvShare;
  if (xi >= x_n) return;
  if (threadIdx.x == 0) {
    s_never = 0;
    s_best = 0;
  }
  __syncthreads();
  const uint32_t x = over_x[x_lo + xi];
  uint32_t* bm = gbm + (uint64_t)xi * words;
  const ColdX s = cold_x(hx4, x);
  const uint32_t v = x_variant(s.a0.x, var_bits, vskip);
  const uint64_t* cp = cptr + (uint64_t)v * y_card;
  const uint64_t r0 = r_ptr[x], r1 = r_ptr[x + 1];
  uint64_t star0 = 0;
  uint32_t star_len = 0;
  const uint64_t kstar =
      kStar ? cta_star<kOvThreads>(r0, r1, r_col, cp, &s_best, star0, star_len) : ~0ull;
  uint64_t cnt = 0, sum = 0, xr = 0, csp = 0, ncand = 0, ngat = 0;
  uint32_t qn = 0;
  if (phase == 0) {
    auto ins = [&](bool ok, uint32_t key) {
      if (!ok) return;
      const uint32_t zl = key & kRowMask;
      const uint32_t bit = 1u << (zl & 31);
      if (atomicOr(&bm[zl >> 5], bit) & bit) return;
      ++cnt;
      if (key & kSpFlag) ++csp;
      if (kMode != kModeCount) cold_account<kMode>(x, dl_z[zl], dec, em, sum, xr);
    };
    ncand += cta_cold_x<kOvThreads>(
        s, r0, r1, r_col, cp, crec, s_seg0, s_off, s_wsum, s_tot, &s_never, kstar,
        [&](uint32_t st, uint32_t row) {
          ins(st == kColdSurvivor, row);
          dq_push(dq, qn, st == kColdMaybe, row);
        },
        [&]() { dq_drain(dq, qn, false, s, hz4, ngat, ins); }, share, kOvShare);
    dq_drain(dq, qn, true, s, hz4, ngat, ins);
  } else if (star_len) {
    auto look = [&](bool ok, uint32_t key) {
      if (!ok) return;
      const uint32_t zl = key & kRowMask;
      if ((__ldcg(&bm[zl >> 5]) >> (zl & 31)) & 1u) return;
      ++cnt;
      if (key & kSpFlag) ++csp;
      if (kMode != kModeCount) cold_account<kMode>(x, dl_z[zl], dec, em, sum, xr);
    };
    ncand += cold_star<kStarCtaU>(star0, star_len, share * (kOvThreads / 32) + warp,
                                  kOvShare * (kOvThreads / 32), s, crec, dq, qn, hz4, ngat, look);
  }
  flush_sp(cnt_sp, csp);
  flush_cand(cand, ncand, ngat);
  tally_flush(tally, cnt, sum, xr);
}

}  // namespace d3g
