/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the DIM^3 Join-Project hot
 * path. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it, and only as the checker. See dim3_oracle.c for the
 * file:line mapping onto the reference. */
#ifndef DIM3_ORACLE_H
#define DIM3_ORACLE_H
#include <stdint.h>

typedef struct {
  double t_seqR, t_randR, t_randRW, t_hash, t_map, t_ECs, t_ECd;
  uint32_t w;
} orc_consts;

/* force: 0 auto, 1 classical(→ reported only), 2 hybrid, 3 sparse_only,
 * 4 dense_only. dense_mode: 0 cost_based, 1 force_wide, 2 force_probe. */
typedef struct {
  int32_t force, dense_mode, count_only, natural_keys_auto, threads, pad;
} orc_opts;

typedef struct {
  int32_t swapped, f1_classical;   /* f1 > 0 (auto would go classical) */
  int32_t natural_x, natural_y, natural_z, pad;
  uint64_t r_rows, s_rows, out_j_estimate;
  double f1;
  uint64_t out_p, pairs_sparse, pairs_dense;
  uint64_t sparse_z, dense_z, f2_evaluations, dropped_r;
  uint64_t x_card, y_card, z_card, r_nnz, s_nnz, sparse_nnz, out_j;
  uint64_t panel_bytes, spa_inner_count;
  uint64_t dense_wide_encounters, dense_probe_encounters;
  uint64_t dense_blocks_checked, dense_probes_done, dense_row_bitmaps_built;
  uint64_t x_live;
  uint64_t checksum_sum, checksum_xor;
} orc_report;

#endif
