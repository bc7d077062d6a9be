// dim3_gpu.hpp — B200 drop-in for dim3::join_project (P/include/dim3/engine.hpp:102-103).
// Header-only: include it next to the reference headers and link
// paper_2206_04995_b200/libdim3_b200.so. Compiled and run against the unmodified
// reference by integration/shim_check.cpp (oracle/Makefile target `shim`).
#pragma once
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

inline JoinProjectOutput join_project(const RawTable& r, const RawTable& s,
                                      const EngineConfig& cfg, const CostConstants& c,
                                      const GpuOptions& g = {}) {
  if (r.left.type != ColumnType::u64 || r.right.type != ColumnType::u64 ||
      s.left.type != ColumnType::u64 || s.right.type != ColumnType::u64)
    throw ConfigError("the GPU path takes integer (u64) columns");
  d3g_table R{r.left.ints.data(), r.right.ints.data(), r.size(), 0, 0};
  d3g_table S{s.left.ints.data(), s.right.ints.data(), s.size(), 0, 0};
  d3g_consts k{c.t_seqR, c.t_randR, c.t_randRW, c.t_hash, c.t_map, c.t_ECs, c.t_ECd, c.w, 0};
  d3g_opts o;
  d3g_opts_default(&o);
  o.force = static_cast<int32_t>(cfg.force);             // Strategy, engine.hpp:25-31
  o.threads = cfg.threads;
  o.memory_budget_bytes = cfg.memory_budget_bytes;
  o.count_only = cfg.count_only;
  o.dense_mode = static_cast<int32_t>(cfg.dense_mode);
  o.natural_keys_auto = cfg.natural_keys_auto;
  o.declared_x = cfg.natural_keys_declared.x;
  o.declared_y = cfg.natural_keys_declared.y;
  o.declared_z = cfg.natural_keys_declared.z;
  o.collect_counters = g.exact_counters ? 1 : 0;
  d3g_report rep{};
  JoinProjectOutput out;
  out.result.provenance = ResultSet::Provenance::raw;   // decoded on the device
  out.result.raw_x.type = out.result.raw_z.type = ColumnType::u64;
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
