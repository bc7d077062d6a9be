// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI driver over the UNMODIFIED reference library (built by
// oracle/Makefile from /root/reference/proj/src/*.cpp into
// oracle/_ref/libdim3ref.so). It lets Python tests, the golden-fixture
// generator and bench.py's reference arm call the reference's own operator
// API:
//   dim3::join_project            P/src/engine.cpp:345-349
//   dim3::result_to_raw           P/src/engine.cpp:527-529
//   dim3::map_tables              P/src/mapping.cpp:342-420
//   dim3::build_csr               P/src/relation.cpp:206-258
//   dim3::compute_degree_stats    P/src/costmodel.cpp:425-438
//   dim3::partition_s_csr         P/src/partition.cpp:5-80
//   dim3::sparse_bmm              P/src/sparsebmm.cpp:53-106
// (P = /root/reference/proj). Nothing here re-implements the algorithm; the
// only arithmetic of our own is the order-independent set checksum
// h(x,z) = mix64(mix64(x) ^ z) summed mod 2^64 and xor-folded (SURVEY
// Appendix A).

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "dim3/costmodel.hpp"
#include "dim3/engine.hpp"
#include "dim3/mapping.hpp"
#include "dim3/partition.hpp"
#include "dim3/relation.hpp"
#include "dim3/sparsebmm.hpp"

namespace {

thread_local std::string g_err;

struct RefConsts {
  double t_seqR, t_randR, t_randRW, t_hash, t_map, t_ECs, t_ECd;
  std::uint32_t w;
};

// Flat mirror of dim3::ExecutionReport (P/include/dim3/engine.hpp:59-85).
struct RefReport {
  char strategy[16];
  std::int32_t swapped;
  std::int32_t materialized;
  std::uint64_t r_rows, s_rows, out_j_estimate;
  double f1;
  std::uint64_t out_p, pairs_classical, pairs_sparse, pairs_dense;
  std::uint64_t sparse_z, dense_z, f2_evaluations, dropped_r;
  std::uint64_t intermediate_pairs, x_card, y_card, z_card;
  std::uint64_t panel_bytes, peak_bytes;
  std::uint64_t spa_inner_count;
  std::uint64_t dense_wide_encounters, dense_probe_encounters;
  std::uint64_t dense_blocks_checked, dense_probes_done, dense_row_bitmaps_built;
  double ms_total, ms_estimate, ms_map, ms_csr, ms_partition, ms_sparse,
      ms_dense, ms_classical;
  std::uint64_t checksum_sum, checksum_xor;  // over decoded pairs, if materialized
  std::uint64_t spa_allocations, spa_entries;
};

dim3::CostConstants to_consts(const RefConsts* c) {
  dim3::CostConstants k;
  k.t_seqR = c->t_seqR;
  k.t_randR = c->t_randR;
  k.t_randRW = c->t_randRW;
  k.t_hash = c->t_hash;
  k.t_map = c->t_map;
  k.t_ECs = c->t_ECs;
  k.t_ECd = c->t_ECd;
  k.w = c->w;
  return k;
}

dim3::RawTable to_table(const std::uint64_t* l, const std::uint64_t* r,
                        std::uint64_t n) {
  dim3::RawTable t;
  t.left.type = dim3::ColumnType::u64;
  t.right.type = dim3::ColumnType::u64;
  t.left.ints.assign(l, l + n);
  t.right.ints.assign(r, r + n);
  return t;
}

inline std::uint64_t pair_hash(std::uint64_t x, std::uint64_t z) {
  return dim3::mix64(dim3::mix64(x) ^ z);
}

int status_of(const std::exception& e) {
  if (dynamic_cast<const dim3::ConfigError*>(&e)) return 2;
  if (dynamic_cast<const dim3::IoError*>(&e)) return 3;
  if (dynamic_cast<const dim3::FormatError*>(&e)) return 3;
  if (dynamic_cast<const dim3::ResourceError*>(&e)) return 4;
  return 5;
}

// The engine's own natural-key resolution (P/src/engine.cpp:25-50) lives in
// an anonymous namespace; the checksum path below mirrors its two calls using
// the public detect_natural_keys / map_tables.
dim3::MappingOutput map_like_engine(const dim3::RawTable& R,
                                    const dim3::RawTable& S) {
  dim3::SkipFlags sk;
  sk.x = dim3::detect_natural_keys(R.left);
  sk.y = dim3::detect_natural_keys(R.right) && dim3::detect_natural_keys(S.right);
  sk.z = dim3::detect_natural_keys(S.left);
  try {
    return dim3::map_tables(R, S, sk);
  } catch (const dim3::ConfigError&) {
    if (!sk.x && !sk.y && !sk.z) throw;
    return dim3::map_tables(R, S, dim3::SkipFlags{});
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// dim3::join_project through the reference API. force: 0 auto, 1 classical,
// 2 hybrid, 3 sparse_only, 4 dense_only (dim3::Strategy order). dense_mode:
// 0 cost_based, 1 force_wide, 2 force_probe. When !count_only and out_x is
// non-null, up to out_cap decoded pairs are copied in emission order.
int ref_join_project(const std::uint64_t* rl, const std::uint64_t* rr,
                     std::uint64_t nr, const std::uint64_t* sl,
                     const std::uint64_t* sr, std::uint64_t ns, int force,
                     int threads, int count_only, int dense_mode,
                     std::uint64_t budget_bytes, int natural_keys_auto,
                     const RefConsts* consts, RefReport* rep,
                     std::uint64_t* out_x, std::uint64_t* out_z,
                     std::uint64_t out_cap) {
  try {
    dim3::RawTable r = to_table(rl, rr, nr);
    dim3::RawTable s = to_table(sl, sr, ns);
    dim3::EngineConfig cfg;
    cfg.force = static_cast<dim3::Strategy>(force);
    cfg.threads = threads;
    cfg.count_only = count_only != 0;
    cfg.dense_mode = static_cast<dim3::DensePathMode>(dense_mode);
    if (budget_bytes != 0) cfg.memory_budget_bytes = budget_bytes;
    cfg.natural_keys_auto = natural_keys_auto != 0;
    auto out = dim3::join_project(r, s, cfg, to_consts(consts));
    const auto& e = out.report;
    std::memset(rep, 0, sizeof(*rep));
    std::strncpy(rep->strategy, e.strategy.c_str(), sizeof(rep->strategy) - 1);
    rep->swapped = e.swapped;
    rep->materialized = out.result.materialized;
    rep->r_rows = e.r_rows;
    rep->s_rows = e.s_rows;
    rep->out_j_estimate = e.out_j_estimate;
    rep->f1 = e.f1_value;
    rep->out_p = e.out_p;
    rep->pairs_classical = e.pairs_classical;
    rep->pairs_sparse = e.pairs_sparse;
    rep->pairs_dense = e.pairs_dense;
    rep->sparse_z = e.sparse_z;
    rep->dense_z = e.dense_z;
    rep->f2_evaluations = e.f2_evaluations;
    rep->dropped_r = e.dropped_r;
    rep->intermediate_pairs = e.intermediate_pairs;
    rep->x_card = e.x_card;
    rep->y_card = e.y_card;
    rep->z_card = e.z_card;
    rep->panel_bytes = e.panel_bytes;
    rep->peak_bytes = e.peak_bytes;
    rep->spa_inner_count = e.spa.inner_count;
    rep->dense_wide_encounters = e.dense.wide_encounters;
    rep->dense_probe_encounters = e.dense.probe_encounters;
    rep->dense_blocks_checked = e.dense.blocks_checked;
    rep->dense_probes_done = e.dense.probes_done;
    rep->dense_row_bitmaps_built = e.dense.row_bitmaps_built;
    rep->spa_allocations = e.spa.spa_allocations;
    rep->spa_entries = e.spa.spa_entries;
    rep->ms_total = e.ms_total;
    rep->ms_estimate = e.ms_estimate;
    rep->ms_map = e.ms_map;
    rep->ms_csr = e.ms_csr;
    rep->ms_partition = e.ms_partition;
    rep->ms_sparse = e.ms_sparse;
    rep->ms_dense = e.ms_dense;
    rep->ms_classical = e.ms_classical;
    if (out.result.materialized) {
      dim3::ResultSet raw = dim3::result_to_raw(out);
      std::uint64_t sum = 0, x = 0;
      std::uint64_t n = raw.raw_x.ints.size();
      for (std::uint64_t i = 0; i < n; ++i) {
        std::uint64_t h = pair_hash(raw.raw_x.ints[i], raw.raw_z.ints[i]);
        sum += h;
        x ^= h;
        if (out_x != nullptr && i < out_cap) {
          out_x[i] = raw.raw_x.ints[i];
          out_z[i] = raw.raw_z.ints[i];
        }
      }
      rep->checksum_sum = sum;
      rep->checksum_xor = x;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// dim3::join_aggregate_both through the reference API (engine.cpp:537-722);
// the decoded pairs (aggregate_to_raw) and values in emission order, up to
// out_cap rows. combine / agg follow dim3::CombineFn / dim3::AggFn order.
int ref_join_aggregate(const std::uint64_t* rl, const std::uint64_t* rr,
                       const double* rv, std::uint64_t nr,
                       const std::uint64_t* sl, const std::uint64_t* sr,
                       const double* sv, std::uint64_t ns, int combine, int agg,
                       int force, int count_only, const RefConsts* consts,
                       RefReport* rep, std::uint64_t* out_x,
                       std::uint64_t* out_z, double* out_v,
                       std::uint64_t out_cap) {
  try {
    dim3::ValuedTable r, s;
    r.base = to_table(rl, rr, nr);
    s.base = to_table(sl, sr, ns);
    r.values.assign(rv, rv + nr);
    s.values.assign(sv, sv + ns);
    dim3::EngineConfig cfg;
    cfg.force = static_cast<dim3::Strategy>(force);
    cfg.count_only = count_only != 0;
    auto out = dim3::join_aggregate_both(r, s, static_cast<dim3::CombineFn>(combine),
                                         static_cast<dim3::AggFn>(agg), cfg,
                                         to_consts(consts));
    const auto& e = out.report;
    std::memset(rep, 0, sizeof(*rep));
    std::strncpy(rep->strategy, e.strategy.c_str(), sizeof(rep->strategy) - 1);
    rep->r_rows = e.r_rows;
    rep->s_rows = e.s_rows;
    rep->out_j_estimate = e.out_j_estimate;
    rep->out_p = e.out_p;
    rep->pairs_sparse = e.pairs_sparse;
    rep->pairs_dense = e.pairs_dense;
    rep->sparse_z = e.sparse_z;
    rep->dense_z = e.dense_z;
    rep->f2_evaluations = e.f2_evaluations;
    rep->dropped_r = e.dropped_r;
    rep->x_card = e.x_card;
    rep->y_card = e.y_card;
    rep->z_card = e.z_card;
    if (out.base.materialized && out_x != nullptr) {
      dim3::ResultSet raw = dim3::aggregate_to_raw(out);
      std::uint64_t n = raw.raw_x.ints.size();
      for (std::uint64_t i = 0; i < n && i < out_cap; ++i) {
        out_x[i] = raw.raw_x.ints[i];
        out_z[i] = raw.raw_z.ints[i];
        out_v[i] = out.values[i];
      }
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// dim3::map_tables with explicit SkipFlags (auto: map_like_engine's natural-key
// detection and fallback). Codes of R (kept rows) and S, r_kept, cards.
int ref_map_tables(const std::uint64_t* rl, const std::uint64_t* rr, std::uint64_t nr,
                   const std::uint64_t* sl, const std::uint64_t* sr, std::uint64_t ns,
                   int auto_skip, int skip_x, int skip_y, int skip_z, std::uint32_t* r_a,
                   std::uint32_t* r_b, std::uint32_t* s_a, std::uint32_t* s_b,
                   std::uint32_t* r_kept, std::uint64_t* stats /* kept, dropped, x, y, z cards, n_kept_list */) {
  try {
    dim3::RawTable R = to_table(rl, rr, nr);
    dim3::RawTable S = to_table(sl, sr, ns);
    dim3::MappingOutput m;
    if (auto_skip) {
      m = map_like_engine(R, S);
    } else {
      dim3::SkipFlags sk;
      sk.x = skip_x != 0;
      sk.y = skip_y != 0;
      sk.z = skip_z != 0;
      m = dim3::map_tables(R, S, sk);
    }
    for (std::size_t i = 0; i < m.r.a.size(); ++i) {
      r_a[i] = m.r.a[i];
      r_b[i] = m.r.b[i];
    }
    for (std::size_t i = 0; i < m.s.a.size(); ++i) {
      s_a[i] = m.s.a[i];
      s_b[i] = m.s.b[i];
    }
    for (std::size_t i = 0; i < m.r_kept.size(); ++i) r_kept[i] = m.r_kept[i];
    stats[0] = m.r.a.size();
    stats[1] = m.dropped_r;
    stats[2] = m.r.a_card;
    stats[3] = m.s.b_card;
    stats[4] = m.s.a_card;
    stats[5] = m.r_kept.size();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// Pipeline facts the parity tests compare against: code-space cards, post-
// collapse nnz, the exact distinct OUT_J (DegreeStats::out_j), and the raw
// values of the z columns f2 marks dense (PartitionResult::panel.z_ids),
// obtained the way join_project_extended does it (P/src/engine.cpp:401-427)
// in engine orientation (no swap when |R| >= |S|).
struct RefPipeline {
  std::uint64_t x_card, y_card, z_card, r_nnz, s_nnz, out_j, dropped_r;
  std::uint64_t dense_z, sparse_z, sparse_nnz;
  std::int32_t natural_x, natural_y, natural_z, pad;
};

int ref_pipeline(const std::uint64_t* rl, const std::uint64_t* rr,
                 std::uint64_t nr, const std::uint64_t* sl,
                 const std::uint64_t* sr, std::uint64_t ns,
                 const RefConsts* consts, RefPipeline* out,
                 std::uint64_t* dense_z_raw, std::uint64_t dense_cap) {
  try {
    dim3::RawTable R0 = to_table(rl, rr, nr);
    dim3::RawTable S0 = to_table(sl, sr, ns);
    const bool swapped = dim3::engine_will_swap(R0, S0);  // engine.cpp:361-366
    const dim3::RawTable& R = swapped ? S0 : R0;
    const dim3::RawTable& S = swapped ? R0 : S0;
    dim3::MappingOutput m = map_like_engine(R, S);
    dim3::CsrMatrix r_by_x = dim3::build_csr(m.r, true);
    dim3::CsrMatrix s_by_z = dim3::build_csr(m.s, true);
    dim3::DegreeStats st = dim3::compute_degree_stats(r_by_x, s_by_z);
    dim3::PartitionResult part =
        dim3::partition_s_csr(s_by_z, st, to_consts(consts));
    std::memset(out, 0, sizeof(*out));
    out->x_card = m.r.a_card;
    out->y_card = m.s.b_card;
    out->z_card = m.s.a_card;
    out->r_nnz = r_by_x.nnz();
    out->s_nnz = s_by_z.nnz();
    out->out_j = st.out_j.value;
    out->dropped_r = m.dropped_r;
    out->dense_z = part.dense_z_count;
    out->sparse_z = part.sparse_z_count;
    out->sparse_nnz = part.s_sparse_by_y.nnz();
    out->natural_x = m.dict_x.is_identity();
    out->natural_y = m.dict_y.is_identity();
    out->natural_z = m.dict_z.is_identity();
    if (dense_z_raw != nullptr) {
      std::uint64_t n = std::min<std::uint64_t>(dense_cap, part.panel.z_ids.size());
      for (std::uint64_t i = 0; i < n; ++i)
        dense_z_raw[i] = m.dict_z.int_value(part.panel.z_ids[i]);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// The same statistics as ref_pipeline with the partition DECISION taken by the
// reference's own F2Evaluator (the loop of P/src/partition.cpp:17-38) but no
// panel allocation, for inputs whose panel cannot be built (cfg5: 1.25 TB).
int ref_pipeline_split(const std::uint64_t* rl, const std::uint64_t* rr,
                       std::uint64_t nr, const std::uint64_t* sl,
                       const std::uint64_t* sr, std::uint64_t ns,
                       const RefConsts* consts, RefPipeline* out) {
  try {
    dim3::RawTable R0 = to_table(rl, rr, nr);
    dim3::RawTable S0 = to_table(sl, sr, ns);
    const bool swapped = dim3::engine_will_swap(R0, S0);
    const dim3::RawTable& R = swapped ? S0 : R0;
    const dim3::RawTable& S = swapped ? R0 : S0;
    dim3::MappingOutput m = map_like_engine(R, S);
    dim3::CsrMatrix r_by_x = dim3::build_csr(m.r, true);
    dim3::CsrMatrix s_by_z = dim3::build_csr(m.s, true);
    dim3::DegreeStats st = dim3::compute_degree_stats(r_by_x, s_by_z);
    std::memset(out, 0, sizeof(*out));
    dim3::F2Evaluator ev(st, to_consts(consts));
    std::uint64_t dense_nnz = 0;
    for (dim3::Code z = 0; z < s_by_z.n_rows; ++z) {
      if (st.m_z[z] == 0) continue;
      if (ev.score(z) > 0) {
        out->dense_z++;
        dense_nnz += st.m_z[z];
      } else {
        out->sparse_z++;
      }
    }
    out->x_card = m.r.a_card;
    out->y_card = m.s.b_card;
    out->z_card = m.s.a_card;
    out->r_nnz = r_by_x.nnz();
    out->s_nnz = s_by_z.nnz();
    out->out_j = st.out_j.value;
    out->dropped_r = m.dropped_r;
    out->sparse_nnz = s_by_z.nnz() - dense_nnz;
    out->natural_x = m.dict_x.is_identity();
    out->natural_y = m.dict_y.is_identity();
    out->natural_z = m.dict_z.is_identity();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// Order-independent fingerprint of the full distinct (x,z) set for outputs
// too large to materialize: force=sparse partition, then
// the reference sparse_bmm on row-sliced copies of r_by_x, decoded through
// the dictionaries and hashed. Optional per-block fingerprints bucket pairs
// by raw x / block_width (natural-key x only).
int ref_set_checksum(const std::uint64_t* rl, const std::uint64_t* rr,
                     std::uint64_t nr, const std::uint64_t* sl,
                     const std::uint64_t* sr, std::uint64_t ns, int threads,
                     std::uint64_t rows_per_slice, std::uint64_t* count,
                     std::uint64_t* sum, std::uint64_t* xr,
                     std::uint64_t block_width, std::uint64_t n_blocks,
                     std::uint64_t* blk_count, std::uint64_t* blk_sum,
                     std::uint64_t* blk_xor) {
  try {
    dim3::RawTable R = to_table(rl, rr, nr);
    dim3::RawTable S = to_table(sl, sr, ns);
    bool swapped = dim3::engine_will_swap(R, S);
    const dim3::RawTable& ER = swapped ? S : R;
    const dim3::RawTable& ES = swapped ? R : S;
    dim3::MappingOutput m = map_like_engine(ER, ES);
    dim3::CsrMatrix r_by_x = dim3::build_csr(m.r, true);
    dim3::CsrMatrix s_by_z = dim3::build_csr(m.s, true);
    dim3::DegreeStats st = dim3::compute_degree_stats(r_by_x, s_by_z);
    dim3::CostConstants c;  // unused by all_sparse
    dim3::PartitionResult part = dim3::partition_s_csr(
        s_by_z, st, c, dim3::PartitionForce::all_sparse);
    // decode ENGINE codes with the engine's dictionaries (row = engine x,
    // pair z = engine z), then swap back to the caller's orientation
    const dim3::Dictionary& dx = m.dict_x;
    const dim3::Dictionary& dz = m.dict_z;
    std::uint64_t n_rows = r_by_x.n_rows;
    if (rows_per_slice == 0) rows_per_slice = 256;
    std::uint64_t n_slices = (n_rows + rows_per_slice - 1) / rows_per_slice;
    std::atomic<std::uint64_t> next{0};
    std::mutex mu;
    std::uint64_t tot_c = 0, tot_s = 0, tot_x = 0;
    if (blk_count != nullptr) {
      std::fill(blk_count, blk_count + n_blocks, 0);
      std::fill(blk_sum, blk_sum + n_blocks, 0);
      std::fill(blk_xor, blk_xor + n_blocks, 0);
    }
    std::vector<std::exception_ptr> errs(std::max(threads, 1));
    auto worker = [&](int tid) {
      try {
        std::uint64_t lc = 0, ls = 0, lx = 0;
        std::vector<std::uint64_t> bc, bs, bx;
        if (blk_count != nullptr) {
          bc.assign(n_blocks, 0);
          bs.assign(n_blocks, 0);
          bx.assign(n_blocks, 0);
        }
        std::vector<std::pair<dim3::Code, dim3::Code>> pairs;
        for (;;) {
          std::uint64_t sl_i = next.fetch_add(1);
          if (sl_i >= n_slices) break;
          std::uint64_t lo = sl_i * rows_per_slice;
          std::uint64_t hi = std::min(n_rows, lo + rows_per_slice);
          // Row-sliced CsrMatrix: rows [lo, hi) re-based to start at 0;
          // x codes are shifted back by lo after the call.
          dim3::CsrMatrix sl_m;
          sl_m.n_rows = static_cast<dim3::Code>(hi - lo);
          sl_m.n_cols = r_by_x.n_cols;
          std::uint64_t b0 = r_by_x.row_ptr[lo], b1 = r_by_x.row_ptr[hi];
          sl_m.row_ptr.resize(hi - lo + 1);
          for (std::uint64_t i = lo; i <= hi; ++i)
            sl_m.row_ptr[i - lo] = r_by_x.row_ptr[i] - b0;
          sl_m.col.assign(r_by_x.col.begin() + b0, r_by_x.col.begin() + b1);
          pairs.clear();
          dim3::sparse_bmm(sl_m, part.s_sparse_by_y, m.s.a_card, {}, &pairs);
          for (auto [xc, zc] : pairs) {
            std::uint64_t ex = dx.int_value(static_cast<dim3::Code>(xc + lo));
            std::uint64_t ez = dz.int_value(zc);
            std::uint64_t cx = swapped ? ez : ex;  // caller orientation
            std::uint64_t cz = swapped ? ex : ez;
            std::uint64_t h = pair_hash(cx, cz);
            ++lc;
            ls += h;
            lx ^= h;
            if (blk_count != nullptr) {
              std::uint64_t b = std::min(cx / block_width, n_blocks - 1);
              bc[b]++;
              bs[b] += h;
              bx[b] ^= h;
            }
          }
        }
        std::lock_guard<std::mutex> g(mu);
        tot_c += lc;
        tot_s += ls;
        tot_x ^= lx;
        if (blk_count != nullptr)
          for (std::uint64_t b = 0; b < n_blocks; ++b) {
            blk_count[b] += bc[b];
            blk_sum[b] += bs[b];
            blk_xor[b] ^= bx[b];
          }
      } catch (...) {
        errs[tid] = std::current_exception();
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(threads, 1); ++t) pool.emplace_back(worker, t);
    for (auto& t : pool) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    *count = tot_c;
    *sum = tot_s;
    *xr = tot_x;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// Reference DenseEC counters on its own panel, for W_D.
int ref_f3_threshold(std::uint32_t m_x, std::uint32_t y_card,
                     const RefConsts* consts, std::uint32_t* out) {
  *out = dim3::f3_threshold(m_x, y_card, to_consts(consts));
  return 0;
}

double ref_f3(double m_x, double m_z, std::uint32_t y_card, const RefConsts* c) {
  return dim3::f3(m_x, m_z, y_card, to_consts(c));
}

std::uint32_t ref_mx_bucket_key(std::uint32_t m) { return dim3::mx_bucket_key(m); }
std::uint32_t ref_mz_bucket_index(std::uint32_t m, std::uint32_t y) {
  return dim3::mz_bucket_index(m, y);
}

}  // extern "C"

// Bounded CPU sample of the reference's own hybrid path for the bench's
// reference arm / cpu_baseline: the full preparation (map_tables, build_csr,
// compute_degree_stats, partition_s_csr — the same calls join_project makes,
// P/src/engine.cpp:401-427) on the WHOLE tables, then the reference kernels
// sparse_bmm / dense_ec (count-only, `threads` workers) on rows
// [x_lo, x_hi) of r_by_x. The caller extrapolates the kernel time linearly
// in x. Seconds are wall-clock (steady_clock).
extern "C" int ref_timed_sample(const std::uint64_t* rl, const std::uint64_t* rr,
                                std::uint64_t nr, const std::uint64_t* sl,
                                const std::uint64_t* sr, std::uint64_t ns,
                                const RefConsts* consts, int threads, std::uint64_t x_lo,
                                std::uint64_t x_hi, double* sec_prep, double* sec_kernels,
                                std::uint64_t* x_rows, std::uint64_t* pairs_in_slice) {
  try {
    using Clk = std::chrono::steady_clock;
    dim3::RawTable R = to_table(rl, rr, nr);
    dim3::RawTable S = to_table(sl, sr, ns);
    dim3::CostConstants c = to_consts(consts);
    auto t0 = Clk::now();
    dim3::MappingOutput m = map_like_engine(R, S);
    dim3::CsrMatrix r_by_x = dim3::build_csr(m.r, true);
    dim3::CsrMatrix s_by_z = dim3::build_csr(m.s, true);
    dim3::DegreeStats st = dim3::compute_degree_stats(r_by_x, s_by_z);
    dim3::PartitionResult part = dim3::partition_s_csr(s_by_z, st, c);
    auto t1 = Clk::now();
    std::uint64_t n_rows = r_by_x.n_rows;
    x_hi = std::min(x_hi, n_rows);
    x_lo = std::min(x_lo, x_hi);
    dim3::CsrMatrix sl_m;
    sl_m.n_rows = static_cast<dim3::Code>(x_hi - x_lo);
    sl_m.n_cols = r_by_x.n_cols;
    std::uint64_t b0 = r_by_x.row_ptr[x_lo], b1 = r_by_x.row_ptr[x_hi];
    sl_m.row_ptr.resize(x_hi - x_lo + 1);
    for (std::uint64_t i = x_lo; i <= x_hi; ++i) sl_m.row_ptr[i - x_lo] = r_by_x.row_ptr[i] - b0;
    sl_m.col.assign(r_by_x.col.begin() + b0, r_by_x.col.begin() + b1);
    auto t2 = Clk::now();
    dim3::SparseOptions so;
    so.threads = threads;
    dim3::DenseOptions dopt;
    dopt.threads = threads;
    std::uint64_t a = dim3::sparse_bmm(sl_m, part.s_sparse_by_y, m.s.a_card, so);
    std::uint64_t b = dim3::dense_ec(sl_m, part.panel, c, dopt);
    auto t3 = Clk::now();
    *sec_prep = std::chrono::duration<double>(t1 - t0).count();
    *sec_kernels = std::chrono::duration<double>(t3 - t2).count();
    *x_rows = n_rows;
    *pairs_in_slice = a + b;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}
