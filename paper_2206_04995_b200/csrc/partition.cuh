// Intersection-free partition of S (P/src/partition.cpp:5-80) and the
// layouts the two GPU kernels consume.
//
// Decision: dense[z] = table[m_z[z]] where table is the per-degree f2
// decision computed on the host (policy.cpp); m_z == 0 gap codes go nowhere.
//
// Sparse side (SparseBMM input): the y-major CSR of the sparse-z tuples
// (partition.cpp:59-78). Columns hold the COMPACT index of the sparse z
// (rank among sparse z), so the per-x dedup bitmap spans only the sparse z
// count, not |Z|; sparse_ids maps the index back to the z code.
//
// Dense side (DenseEC input). Instead of the reference's |Y|-bit panel rows
// (1.25 TB on cfg5) the GPU keeps the dense block in CSR form and answers
// existence with bit-sliced OR sweeps (denseec.cuh):
//   * y_rank: y codes re-ranked by R-side degree dR(y), hottest first, so a
//     z's list meets its most probable witnesses first (early exit);
//   * dense z lists: S rows of dense z with y replaced by y_rank, sorted
//     ascending, rows ordered by m_z descending (uniform warp trip counts);
//   * x order: live x sorted by m_x descending, cut into 128-x groups.
#pragma once

#include "csr.cuh"
#include "segsort.cuh"

namespace d3g {

__global__ void dense_flag_kernel(const uint64_t* __restrict__ row_ptr, uint64_t n_z,
                                  const uint8_t* __restrict__ table, uint64_t table_len,
                                  uint32_t* __restrict__ is_dense, uint32_t* __restrict__ is_sparse) {
  for (uint64_t z = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; z < n_z;
       z += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t m = row_ptr[z + 1] - row_ptr[z];
    uint32_t d = (m > 0 && m < table_len) ? table[m] : 0;
    is_dense[z] = d;
    is_sparse[z] = (m > 0 && !d) ? 1u : 0u;
  }
}


// Counting scatter of rows by degree, descending (ties in arbitrary order),
// with the first position (off) and first list entry (ent) of every degree
// precomputed on the host from the degree histogram: one launch replaces the
// flag / scan / compact / key / radix-sort chain. Selection by the f2 table:
// mode 0 = every row with d > 0 (sp_flag[pos] = the row is sparse), 1 = dense
// rows (table[d] != 0), 2 = sparse rows (table[d] == 0, d > 0). out_ptr (the
// rows' list offsets, with out_ptr[n_out] = total_ent) is optional.
__global__ void degree_scatter_kernel(const uint64_t* __restrict__ row_ptr, uint64_t r0,
                                      uint64_t r1, const uint8_t* __restrict__ table,
                                      uint64_t table_len, int mode,
                                      const uint64_t* __restrict__ off,
                                      const uint64_t* __restrict__ ent,
                                      unsigned int* __restrict__ cur, uint32_t* __restrict__ out,
                                      uint64_t* __restrict__ out_ptr, uint64_t n_out,
                                      uint64_t total_ent, uint8_t* __restrict__ sp_flag) {
  // Positions inside a degree class come from a cursor per degree. A few
  // dozen degrees take every row, so the cursors are reserved per CTA tile
  // (shared-memory counts, then ONE global atomic per (tile, degree)) for
  // degrees below kSmallDeg; rarer large degrees go warp-aggregated to the
  // global cursor. blockDim.x == 256.
  constexpr uint32_t kSmallDeg = 256;
  __shared__ uint32_t s_cnt[kSmallDeg], s_base[kSmallDeg];
  const uint32_t lane = lane_id();
  const uint64_t n = r1 - r0, n_tiles = (n + blockDim.x - 1) / blockDim.x;
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t i = tile * blockDim.x + threadIdx.x;
    const uint64_t r = r0 + i;
    uint64_t d = 0;
    bool take = false, sparse = false;
    if (i < n) {
      d = row_ptr[r + 1] - row_ptr[r];
      if (d > 0) {
        sparse = !(d < table_len && table[d]);
        take = mode == 0 || (mode == 1 ? !sparse : sparse);
      }
    }
    if (threadIdx.x < kSmallDeg) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const bool small = take && d < kSmallDeg;
    uint32_t rank = 0, base = 0;
    if (small) rank = atomicAdd(&s_cnt[d], 1u);
    const uint32_t key = (take && !small) ? (uint32_t)d : 0xffffffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, key);
    if (take && !small) {
      const int leader = __ffs(peers) - 1;
      rank = __popc(peers & ((1u << lane) - 1));
      if ((int)lane == leader) base = atomicAdd(&cur[d], (unsigned)__popc(peers));
      base = __shfl_sync(peers, base, leader);
    }
    __syncthreads();
    if (threadIdx.x < kSmallDeg && s_cnt[threadIdx.x])
      s_base[threadIdx.x] = atomicAdd(&cur[threadIdx.x], s_cnt[threadIdx.x]);
    __syncthreads();
    if (take) {
      if (small) base = s_base[d];
      const uint64_t pos = off[d] + base + rank;
      out[pos] = (uint32_t)r;
      if (out_ptr) out_ptr[pos] = ent[d] + (uint64_t)(base + rank) * d;
      if (sp_flag) sp_flag[pos] = sparse ? 1 : 0;
    }
    __syncthreads();  // s_cnt / s_base are rewritten by the next tile
  }
  if (out_ptr && blockIdx.x == 0 && threadIdx.x == 0) out_ptr[n_out] = total_ent;
}

// Counting sort of indices by a u32 value, descending (ties in arbitrary
// order): desc_hist_kernel counts key = max_val - val[i] (equal keys merged
// per warp), an exclusive scan gives the offsets, desc_scatter_kernel places
// each index (the counts are consumed as cursors).
__global__ void desc_hist_kernel(const uint32_t* __restrict__ val, uint64_t n, uint32_t max_val,
                                 uint32_t* __restrict__ cnt) {
  const uint64_t n_pad = (n + 31) / 32 * 32;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t key = i < n ? max_val - val[i] : 0xffffffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, key);
    if (key != 0xffffffffu && (peers & ((1u << lane_id()) - 1)) == 0)
      atomicAdd(&cnt[key], (unsigned)__popc(peers));
  }
}

__global__ void desc_scatter_kernel(const uint32_t* __restrict__ val, uint64_t n,
                                    uint32_t max_val, const uint64_t* __restrict__ off,
                                    uint32_t* __restrict__ left, uint32_t* __restrict__ order) {
  const uint32_t lane = lane_id();
  const uint64_t n_pad = (n + 31) / 32 * 32;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t key = i < n ? max_val - val[i] : 0xffffffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, key);
    if (key == 0xffffffffu) continue;
    const int leader = __ffs(peers) - 1;
    const uint32_t k = (uint32_t)__popc(peers);
    uint32_t top = 0;
    if ((int)lane == leader) top = atomicSub(&left[key], k);
    top = __shfl_sync(peers, top, leader);
    order[off[key] + top - k + __popc(peers & ((1u << lane) - 1))] = (uint32_t)i;
  }
}

// per-y count of sparse tuples
// Both passes take four rows per warp (8 lanes each): the sparse rows are
// short (cfg3: ~10 entries), and a warp per row left most lanes idle.
__global__ void sparse_y_count_kernel(const uint64_t* __restrict__ row_ptr,
                                      const uint32_t* __restrict__ col,
                                      const uint32_t* __restrict__ sparse_ids, uint64_t n_sparse,
                                      uint32_t* __restrict__ cnt) {
  const uint32_t gl = threadIdx.x & 7;
  for (uint64_t i = (uint64_t)blockIdx.x * (blockDim.x / 8) + (threadIdx.x >> 3); i < n_sparse;
       i += (uint64_t)gridDim.x * (blockDim.x / 8)) {
    const uint32_t z = sparse_ids[i];
    const uint64_t e = row_ptr[z + 1];
    for (uint64_t k = row_ptr[z] + gl; k < e; k += 8) atomicAdd(&cnt[col[k]], 1u);
  }
}

__global__ void sparse_y_scatter_kernel(const uint64_t* __restrict__ row_ptr,
                                        const uint32_t* __restrict__ col,
                                        const uint32_t* __restrict__ sparse_ids, uint64_t n_sparse,
                                        const uint64_t* __restrict__ base,
                                        uint32_t* __restrict__ left /* counts, consumed */,
                                        uint32_t* __restrict__ out_col) {
  const uint32_t gl = threadIdx.x & 7;
  for (uint64_t i = (uint64_t)blockIdx.x * (blockDim.x / 8) + (threadIdx.x >> 3); i < n_sparse;
       i += (uint64_t)gridDim.x * (blockDim.x / 8)) {
    const uint32_t z = sparse_ids[i];
    const uint64_t e = row_ptr[z + 1];
    for (uint64_t k = row_ptr[z] + gl; k < e; k += 8) {
      const uint32_t y = col[k];
      const uint64_t p = base[y] + atomicSub(&left[y], 1u) - 1u;
      out_col[p] = (uint32_t)i;  // compact sparse index
    }
  }
}

// key = maxd - d for ordering ids by degree descending (the radix sort is
// stable, so equal degrees keep ascending id order).
__global__ void degree_order_key_kernel(const uint32_t* __restrict__ ids, uint64_t n,
                                        const uint64_t* __restrict__ row_ptr,
                                        const uint32_t* __restrict__ deg_arr, uint64_t maxd,
                                        uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t id = ids ? ids[i] : (uint32_t)i;
    uint64_t d = row_ptr ? row_ptr[id + 1] - row_ptr[id] : deg_arr[id];
    keys[i] = maxd - d;  // stable sort keeps equal degrees in id order
    vals[i] = id;
  }
}

__global__ void scatter_rank_kernel(const uint32_t* __restrict__ order, uint64_t n,
                                    uint32_t* __restrict__ rank) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    rank[order[i]] = (uint32_t)i;
}

// dense list lengths in processing order
__global__ void gather_len_kernel(const uint32_t* __restrict__ ids, uint64_t n,
                                  const uint64_t* __restrict__ row_ptr, uint32_t* __restrict__ len) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t id = ids[i];
    len[i] = (uint32_t)(row_ptr[id + 1] - row_ptr[id]);
  }
}

// keys for sorting the dense lists: (row_pos << ybits) | y_rank[y]
__global__ void dense_list_key_kernel(const uint32_t* __restrict__ ids, uint64_t n,
                                      const uint64_t* __restrict__ src_ptr,
                                      const uint32_t* __restrict__ src_col,
                                      const uint64_t* __restrict__ dst_ptr,
                                      const uint32_t* __restrict__ y_rank, int ybits,
                                      uint64_t* __restrict__ keys) {
  for (uint64_t i = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < n;
       i += (uint64_t)gridDim.x * (blockDim.x / 32)) {
    uint32_t id = ids[i];
    uint64_t s0 = src_ptr[id], s1 = src_ptr[id + 1], d0 = dst_ptr[i];
    for (uint64_t k = s0 + lane_id(); k < s1; k += 32)
      keys[d0 + (k - s0)] = ((uint64_t)i << ybits) | y_rank[src_col[k]];
  }
}

// dl_col[dl_ptr[i] + k] = y_rank[src_col[src_ptr[ids[i]] + k]] (8 lanes per row)
__global__ void dense_list_fill_kernel(const uint32_t* __restrict__ ids, uint64_t n,
                                       const uint64_t* __restrict__ src_ptr,
                                       const uint32_t* __restrict__ src_col,
                                       const uint64_t* __restrict__ dst_ptr,
                                       const uint32_t* __restrict__ y_rank,
                                       uint32_t* __restrict__ out) {
  const uint32_t gl = threadIdx.x & 7;
  for (uint64_t i = (uint64_t)blockIdx.x * (blockDim.x / 8) + (threadIdx.x >> 3); i < n;
       i += (uint64_t)gridDim.x * (blockDim.x / 8)) {
    uint32_t id = ids[i];
    uint64_t s0 = src_ptr[id], s1 = src_ptr[id + 1], d0 = dst_ptr[i];
    for (uint64_t k = s0 + gl; k < s1; k += 8) out[d0 + (k - s0)] = y_rank[src_col[k]];
  }
}

__global__ void low_bits_kernel(const uint64_t* __restrict__ keys, uint64_t n, int bits,
                                uint32_t* __restrict__ out) {
  const uint64_t m = (1ull << bits) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)(keys[i] & m);
}

}  // namespace d3g
