// dim3_gpu.hpp — B200 drop-in for dim3::join_project (P/include/dim3/engine.hpp:102-103).
// Header-only: include it next to the reference headers and link
// paper_2206_04995_b200/libdim3_b200.so. Compiled and run against the unmodified
// reference by integration/shim_check.cpp (oracle/Makefile target `shim`).
#pragma once
#include <string>
#include <unordered_map>
#include <vector>

#include "dim3/engine.hpp"
#include "dim3_b200.h"   // from this repo's include/

namespace dim3::gpu {

inline void throw_status(int rc) {
  const char* m = d3g_last_error();
  switch (rc) {
    case D3G_OK: return;
    case D3G_CONFIG_ERROR: throw ConfigError(m);      // common.hpp:34
    case D3G_IO_ERROR: throw IoError(m);              // common.hpp:26
    case D3G_FORMAT_ERROR: throw FormatError(m);      // common.hpp:30
    case D3G_RESOURCE_ERROR: throw ResourceError(m);  // common.hpp:32
    default: throw std::runtime_error(m);
  }
}

// One context per host thread (owns the CUDA stream and device pool).
inline d3g_ctx* context(int device = 0) {
  thread_local d3g_ctx* ctx = nullptr;
  if (!ctx) throw_status(d3g_ctx_create(device, &ctx));
  return ctx;
}

// GPU-side knobs outside EngineConfig. exact_counters: also run the per-pair
// pass that reproduces DenseEcStats::blocks_checked / probes_done (cost grows
// with the pair tests; the encounter counts, row bitmaps and SpaStats are
// always filled exactly).
struct GpuOptions {
  bool exact_counters = false;
};

// ColumnType::bytes columns (relation.hpp:21): the GPU takes u64 columns, so a
// byte-string column is interned on the host into surrogate ids (equal strings
// <-> equal ids, in first-occurrence order) and flagged D3G_KEYS_BYTES_*; the
// device then dictionary-codes the ids as the reference does the strings, and
// the result ids are mapped back. The two y columns share one interner; when
// their types differ no R row finds its y (Dictionary::lookup,
// mapping.cpp:177-189), which disjoint id ranges reproduce.
class ColumnInterner {
 public:
  // ids of a bytes column; `tag` keeps u64 values and strings apart when the
  // two y columns differ in type
  std::vector<std::uint64_t> intern(const ColumnData& col) {
    std::vector<std::uint64_t> ids(col.size());
    if (col.type == ColumnType::bytes) {
      for (std::size_t i = 0; i < ids.size(); ++i) {
        auto [it, fresh] = str_ids_.try_emplace(col.strs[i], next_);
        if (fresh) {
          rev_.push_back(&it->first);
          ++next_;
        }
        ids[i] = it->second;
      }
    } else {
      for (std::size_t i = 0; i < ids.size(); ++i) {
        auto [it, fresh] = int_ids_.try_emplace(col.ints[i], next_);
        if (fresh) {
          rev_.push_back(nullptr);
          ++next_;
        }
        ids[i] = it->second;
      }
    }
    return ids;
  }
  const std::string& value(std::uint64_t id) const { return *rev_[id]; }

 private:
  std::unordered_map<std::string, std::uint64_t> str_ids_;  // node-based: keys stay put
  std::unordered_map<std::uint64_t, std::uint64_t> int_ids_;
  std::vector<const std::string*> rev_;
  std::uint64_t next_ = 0;
};

inline JoinProjectOutput join_project(const RawTable& r, const RawTable& s,
                                      const EngineConfig& cfg, const CostConstants& c,
                                      const GpuOptions& g = {}) {
  // surrogate ids for byte-string columns (none: the columns are passed as they are)
  ColumnInterner ix, iy, iz;
  std::vector<std::uint64_t> rl_ids, rr_ids, sl_ids, sr_ids;
  const bool bytes_x = r.left.type == ColumnType::bytes, bytes_z = s.left.type == ColumnType::bytes;
  const bool bytes_y = r.right.type == ColumnType::bytes || s.right.type == ColumnType::bytes;
  if (bytes_x) rl_ids = ix.intern(r.left);
  if (bytes_z) sl_ids = iz.intern(s.left);
  if (bytes_y) {
    rr_ids = iy.intern(r.right);
    sr_ids = iy.intern(s.right);
  }
  d3g_table R{bytes_x ? rl_ids.data() : r.left.ints.data(),
              bytes_y ? rr_ids.data() : r.right.ints.data(), r.size(), 0, 0};
  d3g_table S{bytes_z ? sl_ids.data() : s.left.ints.data(),
              bytes_y ? sr_ids.data() : s.right.ints.data(), s.size(), 0, 0};
  d3g_consts k{c.t_seqR, c.t_randR, c.t_randRW, c.t_hash, c.t_map, c.t_ECs, c.t_ECd, c.w, 0};
  d3g_opts o;
  d3g_opts_default(&o);
  o.force = static_cast<int32_t>(cfg.force);             // Strategy, engine.hpp:25-31
  o.threads = cfg.threads;
  o.memory_budget_bytes = cfg.memory_budget_bytes;
  o.count_only = cfg.count_only;
  o.dense_mode = static_cast<int32_t>(cfg.dense_mode);
  // the flags are in engine orientation: the larger table is the engine's R
  const bool swapped = engine_will_swap(r, s);
  o.natural_keys_auto = (cfg.natural_keys_auto ? D3G_KEYS_AUTO : 0) |
                        ((swapped ? bytes_z : bytes_x) ? D3G_KEYS_BYTES_X : 0) |
                        (bytes_y ? D3G_KEYS_BYTES_Y : 0) |
                        ((swapped ? bytes_x : bytes_z) ? D3G_KEYS_BYTES_Z : 0);
  o.declared_x = cfg.natural_keys_declared.x;
  o.declared_y = cfg.natural_keys_declared.y;
  o.declared_z = cfg.natural_keys_declared.z;
  o.collect_counters = g.exact_counters ? 1 : 0;
  d3g_report rep{};
  JoinProjectOutput out;
  out.result.provenance = ResultSet::Provenance::raw;   // decoded on the device
  out.result.raw_x.type = r.left.type;                  // decode_result, engine.cpp:502-523
  out.result.raw_z.type = s.left.type;
  if (cfg.count_only) {
    throw_status(d3g_join_project(context(), &R, &S, &k, &o, &rep, nullptr));
  } else {
    // one pipeline pass: the library holds the result, sized on return
    d3g_pairs p{nullptr, nullptr, 0, 0, 0, 0};
    throw_status(d3g_join_project(context(), &R, &S, &k, &o, &rep, &p));
    out.result.raw_x.ints.resize(p.n);
    out.result.raw_z.ints.resize(p.n);
    throw_status(d3g_take_pairs(context(), out.result.raw_x.ints.data(),
                                out.result.raw_z.ints.data(), p.n, 0));
    auto to_strings = [](ColumnData& col, const ColumnInterner& in) {
      col.strs.reserve(col.ints.size());
      for (std::uint64_t id : col.ints) col.strs.push_back(in.value(id));
      col.ints.clear();
      col.ints.shrink_to_fit();
    };
    if (bytes_x) to_strings(out.result.raw_x, ix);
    if (bytes_z) to_strings(out.result.raw_z, iz);
  }
  out.result.materialized = !cfg.count_only;
  out.result.count = rep.out_p;
  ExecutionReport& e = out.report;                      // engine.hpp:59-85
  e.strategy = rep.strategy;
  e.swapped = rep.swapped;
  e.r_rows = rep.r_rows;
  e.s_rows = rep.s_rows;
  e.out_j_estimate = rep.out_j_estimate;
  e.f1_value = rep.f1;
  e.out_p = rep.out_p;
  e.pairs_sparse = rep.pairs_sparse;
  e.pairs_dense = rep.pairs_dense;
  e.sparse_z = rep.sparse_z;
  e.dense_z = rep.dense_z;
  e.f2_evaluations = rep.f2_evaluations;
  e.dropped_r = rep.dropped_r;
  e.x_card = rep.x_card;
  e.y_card = rep.y_card;
  e.z_card = rep.z_card;
  e.panel_bytes = rep.panel_bytes;
  e.peak_bytes = rep.peak_bytes;
  e.pairs_classical = rep.pairs_classical;
  e.intermediate_pairs = rep.intermediate_pairs;
  e.ms_classical = rep.ms_classical;
  e.spa.inner_count = rep.spa_inner_count;           // sparsebmm.hpp:15-19
  e.spa.spa_allocations = rep.spa_allocations;
  e.spa.spa_entries = rep.spa_entries;
  e.dense.wide_encounters = rep.dense_wide_encounters;  // denseec.hpp:20-29
  e.dense.probe_encounters = rep.dense_probe_encounters;
  e.dense.blocks_checked = rep.dense_blocks_checked;
  e.dense.probes_done = rep.dense_probes_done;
  e.dense.row_bitmaps_built = rep.dense_row_bitmaps_built;
  e.ms_total = rep.ms_total;
  e.ms_estimate = rep.ms_estimate;
  e.ms_map = rep.ms_map;
  e.ms_csr = rep.ms_csr + rep.ms_stats;
  e.ms_partition = rep.ms_partition;
  e.ms_sparse = rep.ms_sparse;
  e.ms_dense = rep.ms_dense;
  e.ms_decode = rep.ms_decode;
  return out;   // result_to_raw(out) passes raw results through (engine.cpp:502-505)
}

}  // namespace dim3::gpu
