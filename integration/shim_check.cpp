// Drop-in check: the reference's own test scaffolding (P/tests/support.hpp:
// random_instance, oracle_pairs, oracle_out_j_bag, result_set) drives both
// dim3::join_project (the unmodified CPU reference) and dim3::gpu::join_project
// (integration/dim3_gpu.hpp over libdim3_b200.so). For every strategy, both
// equal the brute-force oracle, and the reports agree on the decisions
// (strategy, swap, split, OUT_J estimate, dropped rows, intermediate size)
// and on every work counter of the report (SpaStats, DenseEcStats).
// Mirrors P/tests/test_engine.cpp:89-113 and acceptance criterion 1.
// Build: make -C oracle shim (needs /root/reference); run on a B200.
#include <cstdio>
#include <set>
#include <string>

#include "dim3_gpu.hpp"
#include "support.hpp"

namespace {

int g_fail = 0;

#define CHECK_EQ(a, b, what)                                                              \
  do {                                                                                     \
    if (!((a) == (b))) {                                                                   \
      std::fprintf(stderr, "mismatch: %s (%s)\n", what, #a " vs " #b);                     \
      ++g_fail;                                                                            \
    }                                                                                      \
  } while (0)

dim3::EngineConfig forced(dim3::Strategy s, bool count_only) {
  dim3::EngineConfig cfg;
  cfg.force = s;
  cfg.count_only = count_only;
  return cfg;
}

}  // namespace

int main() {
  const dim3::Strategy forces[] = {dim3::Strategy::auto_select, dim3::Strategy::classical,
                                   dim3::Strategy::hybrid, dim3::Strategy::sparse_only,
                                   dim3::Strategy::dense_only};
  const auto c = testsup::test_consts();
  int instances = 0;
  for (std::uint64_t seed : {41ull, 501ull, 502ull}) {
    dim3::SplitMix64 rng{seed};
    for (int it = 0; it < 12; ++it, ++instances) {
      auto inst = testsup::random_instance(rng);
      const auto want = testsup::oracle_pairs(inst.r, inst.s);
      for (dim3::Strategy f : forces) {
        auto cpu = dim3::join_project(inst.r, inst.s, forced(f, false), c);
        dim3::gpu::GpuOptions exact;
        exact.exact_counters = true;
        auto gpu = dim3::gpu::join_project(inst.r, inst.s, forced(f, false), c, exact);
        CHECK_EQ(testsup::result_set(dim3::result_to_raw(cpu)), want, "cpu set");
        CHECK_EQ(testsup::result_set(dim3::result_to_raw(gpu)), want, "gpu set");
        CHECK_EQ(gpu.result.count, (std::uint64_t)want.size(), "gpu count");
        const auto &a = cpu.report, &b = gpu.report;
        CHECK_EQ(a.strategy, b.strategy, "strategy");
        CHECK_EQ(a.swapped, b.swapped, "swapped");
        CHECK_EQ(a.out_j_estimate, b.out_j_estimate, "out_j_estimate");
        CHECK_EQ(a.out_p, b.out_p, "out_p");
        CHECK_EQ(a.dropped_r, b.dropped_r, "dropped_r");
        CHECK_EQ(a.intermediate_pairs, b.intermediate_pairs, "intermediate_pairs");
        if (a.strategy != "classical") {
          CHECK_EQ(a.dense_z, b.dense_z, "dense_z");
          CHECK_EQ(a.sparse_z, b.sparse_z, "sparse_z");
          CHECK_EQ(a.pairs_dense, b.pairs_dense, "pairs_dense");
          CHECK_EQ(a.pairs_sparse, b.pairs_sparse, "pairs_sparse");
          CHECK_EQ(a.x_card, b.x_card, "x_card");
          CHECK_EQ(a.y_card, b.y_card, "y_card");
          CHECK_EQ(a.z_card, b.z_card, "z_card");
          CHECK_EQ(a.f2_evaluations, b.f2_evaluations, "f2_evaluations");
          CHECK_EQ(a.panel_bytes, b.panel_bytes, "panel_bytes");
          // the to_kv work counters (engine.cpp:303-309)
          CHECK_EQ(a.spa.inner_count, b.spa.inner_count, "spa_inner_count");
          CHECK_EQ(a.spa.spa_allocations, b.spa.spa_allocations, "spa_allocations");
          CHECK_EQ(a.spa.spa_entries, b.spa.spa_entries, "spa_entries");
          CHECK_EQ(a.dense.wide_encounters, b.dense.wide_encounters, "dense_wide_encounters");
          CHECK_EQ(a.dense.probe_encounters, b.dense.probe_encounters, "dense_probe_encounters");
          CHECK_EQ(a.dense.blocks_checked, b.dense.blocks_checked, "dense_blocks_checked");
          CHECK_EQ(a.dense.probes_done, b.dense.probes_done, "dense_probes_done");
          CHECK_EQ(a.dense.row_bitmaps_built, b.dense.row_bitmaps_built,
                   "dense_row_bitmaps_built");
        } else {
          CHECK_EQ(a.pairs_classical, b.pairs_classical, "pairs_classical");
          CHECK_EQ(b.intermediate_pairs, testsup::oracle_out_j_bag(
                                              a.swapped ? inst.s : inst.r,
                                              a.swapped ? inst.r : inst.s),
                   "bag size");
        }
        auto cnt = dim3::gpu::join_project(inst.r, inst.s, forced(f, true), c);
        CHECK_EQ(cnt.result.count, (std::uint64_t)want.size(), "count-only");
      }
    }
  }
  // ColumnType::bytes columns (relation.hpp:21): the same instances with
  // their columns turned into byte strings, one column role at a time, all of
  // them, and with the two y columns of different types (no R row finds its
  // y). The GPU shim interns the strings; sets, counts and the decisions of
  // the report equal the reference's run on the same byte-string tables.
  int bytes_runs = 0;
  {
    auto as_bytes = [](dim3::ColumnData& col) {
      col.type = dim3::ColumnType::bytes;
      for (std::uint64_t v : col.ints) col.strs.push_back("k" + std::to_string(v * 7919 % 100003));
      col.ints.clear();
    };
    auto cell = [](const dim3::ColumnData& col, std::size_t i) {
      return col.type == dim3::ColumnType::u64 ? "#" + std::to_string(col.ints[i]) : col.strs[i];
    };
    auto str_set = [&](const dim3::ResultSet& raw) {
      std::set<std::pair<std::string, std::string>> out;
      for (std::size_t i = 0; i < raw.raw_x.size(); ++i)
        out.insert({cell(raw.raw_x, i), cell(raw.raw_z, i)});
      return out;
    };
    dim3::SplitMix64 rng{77};
    for (int it = 0; it < 6; ++it) {
      const auto base = testsup::random_instance(rng);
      for (int variant = 0; variant < 6; ++variant, ++bytes_runs) {
        auto inst = base;
        if (variant == 0 || variant == 3) as_bytes(inst.r.left);
        if (variant == 1 || variant == 3) {
          as_bytes(inst.r.right);
          as_bytes(inst.s.right);
        }
        if (variant == 2 || variant == 3) as_bytes(inst.s.left);
        if (variant == 4) as_bytes(inst.r.right);  // y types differ
        if (variant == 5) as_bytes(inst.s.right);
        for (dim3::Strategy f : {dim3::Strategy::auto_select, dim3::Strategy::hybrid,
                                 dim3::Strategy::classical}) {
          auto cpu = dim3::join_project(inst.r, inst.s, forced(f, false), c);
          auto gpu = dim3::gpu::join_project(inst.r, inst.s, forced(f, false), c);
          const auto cr = dim3::result_to_raw(cpu), gr = dim3::result_to_raw(gpu);
          CHECK_EQ(str_set(gr), str_set(cr), "bytes: set");
          CHECK_EQ(gr.raw_x.type, cr.raw_x.type, "bytes: x type");
          CHECK_EQ(gr.raw_z.type, cr.raw_z.type, "bytes: z type");
          CHECK_EQ(gpu.result.count, cpu.result.count, "bytes: count");
          const auto &a = cpu.report, &b = gpu.report;
          CHECK_EQ(a.strategy, b.strategy, "bytes: strategy");
          CHECK_EQ(a.swapped, b.swapped, "bytes: swapped");
          CHECK_EQ(a.out_j_estimate, b.out_j_estimate, "bytes: out_j_estimate");
          CHECK_EQ(a.dropped_r, b.dropped_r, "bytes: dropped_r");
          if (a.strategy != "classical") {
            CHECK_EQ(a.x_card, b.x_card, "bytes: x_card");
            CHECK_EQ(a.y_card, b.y_card, "bytes: y_card");
            CHECK_EQ(a.z_card, b.z_card, "bytes: z_card");
            CHECK_EQ(a.dense_z, b.dense_z, "bytes: dense_z");
            CHECK_EQ(a.sparse_z, b.sparse_z, "bytes: sparse_z");
            CHECK_EQ(a.pairs_dense, b.pairs_dense, "bytes: pairs_dense");
            CHECK_EQ(a.pairs_sparse, b.pairs_sparse, "bytes: pairs_sparse");
          }
          auto cnt = dim3::gpu::join_project(inst.r, inst.s, forced(f, true), c);
          CHECK_EQ(cnt.result.count, cpu.result.count, "bytes: count-only");
        }
      }
      // declaring a byte-string column natural is the reference's ConfigError
      auto inst = base;
      as_bytes(inst.r.left);
      as_bytes(inst.s.left);
      // (raised inside map_tables: the classical branch, forced or chosen by
      // the f1 gate, never gets there -- in the reference and here alike)
      for (dim3::Strategy f : {dim3::Strategy::hybrid, dim3::Strategy::auto_select,
                               dim3::Strategy::classical}) {
        dim3::EngineConfig decl = forced(f, false);
        decl.natural_keys_declared.x = true;
        bool cpu_threw = false, gpu_threw = false;
        try { dim3::join_project(inst.r, inst.s, decl, c); } catch (const dim3::ConfigError&) { cpu_threw = true; }
        try { dim3::gpu::join_project(inst.r, inst.s, decl, c); } catch (const dim3::ConfigError&) { gpu_threw = true; }
        CHECK_EQ(gpu_threw, cpu_threw, "bytes: declared natural x raises as the reference does");
        if (f == dim3::Strategy::hybrid) CHECK_EQ(cpu_threw, true, "bytes: declared natural x -> ConfigError");
        if (f == dim3::Strategy::classical) CHECK_EQ(cpu_threw, false, "classical ignores the skip flags");
      }
    }
  }

  // errors map back to the reference's exception types
  bool threw = false;
  try {
    auto inst = testsup::random_instance(*new dim3::SplitMix64{7});
    dim3::EngineConfig bad;
    bad.threads = 0;
    dim3::gpu::join_project(inst.r, inst.s, bad, c);
  } catch (const dim3::ConfigError&) {
    threw = true;
  }
  CHECK_EQ(threw, true, "threads < 1 -> ConfigError");
  if (g_fail) {
    std::fprintf(stderr, "shim FAILED: %d mismatches\n", g_fail);
    return 1;
  }
  std::printf("shim ok: %d instances x %zu strategies, GPU == reference == oracle; %d byte-string "
              "column runs, GPU == reference\n", instances, sizeof(forces) / sizeof(forces[0]),
              bytes_runs);
  return 0;
}
