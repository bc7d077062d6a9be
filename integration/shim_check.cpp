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
  std::printf("shim ok: %d instances x %zu strategies, GPU == reference == oracle\n", instances,
              sizeof(forces) / sizeof(forces[0]));
  return 0;
}
