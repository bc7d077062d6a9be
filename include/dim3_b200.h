/*
 * dim3_b200.h — C ABI of the B200-native DIM^3 Join-Project operator.
 *
 * This is the drop-in boundary for the reference's operator API
 * (P = /root/reference/proj):
 *
 *   d3g_join_project   replaces dim3::join_project / join_project_extended
 *                      (P/include/dim3/engine.hpp:102-103, :117-120;
 *                       P/src/engine.cpp:345-498) plus result_to_raw
 *                      (engine.hpp:123, engine.cpp:502-529).
 *   d3g_build_csr      replaces dim3::build_csr (P/include/dim3/relation.hpp:108-109).
 *   d3g_sparse_bmm_csr replaces dim3::sparse_bmm (P/include/dim3/sparsebmm.hpp:33-36).
 *   d3g_dense_ec_rows  replaces dim3::dense_ec (P/include/dim3/denseec.hpp:82-85).
 *   d3g_f2_decide      the F2Evaluator decision loop of partition_s_csr
 *                      (P/src/costmodel.cpp:515-586, P/src/partition.cpp:17-38),
 *                      evaluated on degree histograms (host only, no GPU).
 *   d3g_f3_threshold   dim3::f3_threshold (P/include/dim3/costmodel.hpp:120-121).
 *
 * Plain pointers and sizes only. Tables are caller-owned; every entry point
 * is synchronous with respect to the caller's view of the result.
 *
 * Status codes follow the reference CLI's exception mapping
 * (P/tools/dim3.cpp:675-693): 0 ok, 2 ConfigError, 3 IoError/FormatError,
 * 4 ResourceError, 5 CUDA/internal failure. d3g_last_error() returns the
 * message of the last failure on the calling thread.
 */
#ifndef DIM3_B200_H
#define DIM3_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define D3G_OK 0
#define D3G_CONFIG_ERROR 2
#define D3G_IO_ERROR 3
#define D3G_RESOURCE_ERROR 4
#define D3G_INTERNAL_ERROR 5
#define D3G_FORMAT_ERROR 6   /* dim3::FormatError; the CLI maps it to exit 3 like IoError */

/* dim3::Strategy (P/include/dim3/engine.hpp:25-31). */
#define D3G_AUTO 0
#define D3G_CLASSICAL 1
#define D3G_HYBRID 2
#define D3G_SPARSE_ONLY 3
#define D3G_DENSE_ONLY 4

/* dim3::DensePathMode (P/include/dim3/denseec.hpp:18). The GPU answers every
 * (x, dense z) encounter with its own kernels whatever the mode (the output
 * set is the same); the mode decides which reference sweep the
 * reference-equivalent counters describe: the wide (block_and_any) or probe
 * (probe_any) path per encounter, exactly as P/src/denseec.cpp:26-43 picks. */
#define D3G_DENSE_COST_BASED 0
#define D3G_DENSE_FORCE_WIDE 1
#define D3G_DENSE_FORCE_PROBE 2

typedef struct d3g_ctx d3g_ctx;

/* A two-column relation, row i = (left[i], right[i]); the same shape as
 * dim3::RawTable with ColumnType::u64 columns (P/include/dim3/relation.hpp:21-46).
 * on_device != 0: the pointers are CUDA device pointers on the context's
 * device (no H2D copy is made).
 * value_bytes: 0 or 8 = u64 values (ColumnData::ints); 4 = the columns hold
 * uint32_t values (cast the pointers): the int32 workloads copy half the
 * bytes host -> device and are widened on the GPU (d3g_join_project only;
 * the other entry points take u64 columns and raise ConfigError on 4). */
typedef struct {
  const uint64_t* left;
  const uint64_t* right;
  uint64_t n;
  int32_t on_device;
  int32_t value_bytes;
} d3g_table;

/* dim3::CostConstants (P/include/dim3/costmodel.hpp:21-30). */
typedef struct {
  double t_seqR, t_randR, t_randRW, t_hash, t_map, t_ECs, t_ECd;
  uint32_t w;
  uint32_t pad;
} d3g_consts;

/* d3g_opts.natural_keys_auto bits. D3G_KEYS_AUTO is the reference's
 * natural_keys_auto. A caller holding ColumnType::bytes columns
 * (P/include/dim3/relation.hpp:21) passes surrogate u64 ids for them (equal
 * strings <-> equal ids; integration/dim3_gpu.hpp interns them) and marks the
 * column, in ENGINE orientation (x = the larger table's left column, z = the
 * other's, as natural_keys_declared): such a column is always dictionary-coded
 * (detect_natural_keys is false for bytes, P/src/mapping.cpp:284) and
 * declaring it natural is a ConfigError (require_natural, :328-331). */
enum {
  D3G_KEYS_AUTO = 1,
  D3G_KEYS_BYTES_X = 2,
  D3G_KEYS_BYTES_Y = 4,
  D3G_KEYS_BYTES_Z = 8
};

/* dim3::EngineConfig (P/include/dim3/engine.hpp:36-48) plus GPU options. */
typedef struct {
  int32_t force;              /* D3G_AUTO .. D3G_DENSE_ONLY */
  int32_t threads;            /* accepted for API parity; must be >= 1 */
  uint64_t memory_budget_bytes;  /* device working-set cap; 0 = 3 GiB default */
  int32_t count_only;
  int32_t dense_mode;
  int32_t natural_keys_auto;  /* D3G_KEYS_* bits; 1 = EngineConfig::natural_keys_auto */
  int32_t declared_x, declared_y, declared_z;  /* natural_keys_declared */
  int32_t checksum;           /* also compute (sum, xor) of mix64(mix64(x)^z) */
  int32_t collect_counters;   /* also compute dense_blocks_checked and
                                 dense_probes_done (a per-pair pass: for tests
                                 and W_D; |Y| must fit one smem bitmap) */
  int32_t shard_index;        /* x-range shard of R handled by this call */
  int32_t shard_count;        /* 1 = whole table */
  uint32_t x_code_lo;         /* restrict the kernels to engine x codes in */
  uint32_t x_code_hi;         /* [lo, hi); hi = 0: all. Shards split the range */
} d3g_opts;

/* dim3::ExecutionReport (P/include/dim3/engine.hpp:59-85) flattened, plus
 * GPU-side fields. ms_* are CUDA-event times of each phase. */
typedef struct {
  char strategy[16];
  int32_t swapped;
  int32_t f1_gate_classical;  /* auto + f1 > 0: the reference would run the
                                 classical join (outside this path) */
  int32_t natural_x, natural_y, natural_z;
  int32_t materialized;
  uint64_t r_rows, s_rows, out_j_estimate;
  double f1;
  uint64_t out_p, pairs_sparse, pairs_dense;
  uint64_t sparse_z, dense_z, f2_evaluations, dropped_r;
  uint64_t x_card, y_card, z_card, r_nnz, s_nnz, sparse_nnz, out_j;
  uint64_t x_live;
  uint64_t panel_bytes;       /* reference panel size (dense_z * padded(|Y|)/8) */
  uint64_t peak_bytes;        /* device working set high-water mark */
  uint64_t spa_inner_count;   /* OUT_J over sparse z (SpaStats::inner_count) */
  /* DenseEcStats (P/include/dim3/denseec.hpp:20-29): what the reference's
   * dense_ec counts on this input under opts.dense_mode. Encounters and row
   * bitmaps are always filled (exact, from the degree histograms and the
   * f3 thresholds); blocks_checked / probes_done only with collect_counters
   * (0 otherwise). Over the x codes this call processed. */
  uint64_t dense_wide_encounters, dense_probe_encounters;
  uint64_t dense_blocks_checked, dense_probes_done, dense_row_bitmaps_built;
  uint64_t checksum_sum, checksum_xor;
  uint64_t h2d_bytes, d2h_bytes;
  double ms_total, ms_h2d, ms_estimate, ms_map, ms_csr, ms_stats, ms_partition;
  double ms_sparse, ms_dense, ms_decode;
  uint64_t gpu_launches;      /* kernels launched by this call */
  /* classical branch (hash_join_dedup, P/src/classical.cpp:111-210) */
  uint64_t pairs_classical, intermediate_pairs;
  double ms_classical;
  /* DenseEC P1 (hot bit-sliced pass) alone: CUDA-event time of its launches
   * and their algorithmic shared-memory bytes (one 512 B LDS.128 per
   * (row, batch, slice read)), the roofline inputs. */
  double ms_dense_hot;
  uint64_t hot_lds_bytes;
  /* the same pass without the prefix sharing of sorted rows (every row reads
   * its subset entry and all listed slices): the work the sharing removed */
  uint64_t hot_lds_bytes_unshared;
  /* count-only: (x, z) pairs counted as hits without a test by the rank-0
   * split (x and z both hold the top-ranked y) */
  uint64_t hot_direct_pairs;
  /* DenseEC P2 (cold residual) kernels: CUDA-event time and algorithmic
   * bytes = 16 B per candidate record streamed (hot word 0, folded tail,
   * row id) + 32 B per exact tail check (cold_candidates / cold_tail_checks
   * below), each x's stream counted once, in the tier that completes it */
  double ms_dense_cold;
  uint64_t cold_bytes;
  /* SpaStats::spa_allocations / spa_entries (P/include/dim3/sparsebmm.hpp:15-19):
   * the stamp arrays the reference's run_chunked would allocate for
   * opts.threads over the engine's x rows, and |Z| per array. */
  uint64_t spa_allocations, spa_entries;
  /* sharded job (exchange set): this rank's own pair count (materialized
   * pairs are the rank's), and the job shape; 1 / 0 otherwise */
  uint64_t rank_out_p;
  int32_t nranks, rank;
  /* DenseEC P2: candidate records streamed, exact tail checks (gathers) */
  uint64_t cold_candidates, cold_tail_checks;
  /* sharded job: collectives issued, bytes a ring collective moves per rank
   * over the links, host time of host-staged collectives (callback
   * transport; 0 under NCCL), and whether the S side was split by z */
  uint64_t exchange_calls, exchange_bus_bytes;
  double ms_exchange_host;
  int32_t zsplit, pad1;
} d3g_report;

/* Materialized output: caller-owned host (or device, on_device != 0)
 * buffers of cap entries. On return n = pairs written, sorted by (x, z),
 * raw values in the caller's orientation. x == NULL: the library keeps the
 * result on the device (n is set) for d3g_take_pairs -- one pipeline pass
 * without knowing the output size beforehand. */
typedef struct {
  uint64_t* x;
  uint64_t* z;
  uint64_t cap;
  uint64_t n;
  int32_t on_device;
  int32_t pad;
} d3g_pairs;

/* CSR boolean matrix (dim3::CsrMatrix, P/include/dim3/relation.hpp:87-103). */
typedef struct {
  uint64_t* row_ptr; /* n_rows + 1 */
  uint32_t* col;     /* nnz */
  uint32_t n_rows, n_cols;
  uint64_t nnz;
} d3g_csr;

/* Bitmap panel (dim3::BitmapPanel, P/include/dim3/bitmap.hpp:78-96). */
typedef struct {
  const uint32_t* z_ids;
  const uint32_t* m_z;
  const uint64_t* blocks; /* rows * row_words */
  uint64_t rows;
  uint32_t y_card, w;
} d3g_panel;

/* Reference-equivalent kernel counters (SpaStats, DenseEcStats). */
typedef struct {
  uint64_t inner_count;
  uint64_t wide_encounters, probe_encounters, blocks_checked, probes_done;
  uint64_t row_bitmaps_built;
  double ms_kernel;
} d3g_kernel_stats;

int d3g_ctx_create(int device, d3g_ctx** out);
void d3g_ctx_destroy(d3g_ctx* ctx);
const char* d3g_last_error(void);
/* Identifies the build ("sm_100a ..."); never fails. */
const char* d3g_version(void);
/* Default options = EngineConfig{} (auto, 1 thread, 3 GiB, materialize). */
void d3g_opts_default(d3g_opts* o);

int d3g_join_project(d3g_ctx* ctx, const d3g_table* r, const d3g_table* s,
                     const d3g_consts* c, const d3g_opts* o, d3g_report* rep,
                     d3g_pairs* pairs /* NULL = count only */);
/* Copies the first n pairs of the result the last d3g_join_project kept on
 * the device (d3g_pairs.x == NULL) into x / z (host, or device when
 * on_device) and releases it. */
int d3g_take_pairs(d3g_ctx* ctx, uint64_t* x, uint64_t* z, uint64_t n, int on_device);

/* build_csr over mapped code pairs (a = major when major_is_a). Host arrays
 * in, host CSR out (row_ptr/col must hold n_rows+1 / n entries). */
int d3g_build_csr(d3g_ctx* ctx, const uint32_t* a, const uint32_t* b, uint64_t n,
                  uint32_t a_card, uint32_t b_card, int major_is_a, d3g_csr* out);

/* sparse_bmm over host CSRs; pairs_x/pairs_z (nullable) receive code pairs
 * sorted by (x, z); returns the emitted count through *count. */
int d3g_sparse_bmm_csr(d3g_ctx* ctx, const d3g_csr* r_by_x, const d3g_csr* s_sparse_by_y,
                       uint32_t z_card, uint32_t* pairs_x, uint32_t* pairs_z,
                       uint64_t pairs_cap, uint64_t* count, d3g_kernel_stats* st);

/* dense_ec over a host CSR and a host bitmap panel. */
int d3g_dense_ec_rows(d3g_ctx* ctx, const d3g_csr* r_by_x, const d3g_panel* panel,
                      const d3g_consts* c, int dense_mode, uint32_t* pairs_x,
                      uint32_t* pairs_z, uint64_t pairs_cap, uint64_t* count,
                      d3g_kernel_stats* st);

/* Convention-G synthetic rows [lo, hi) of config cfg (1..5; SURVEY
 * Appendix A), side 0 = R (x, y), 1 = S (z, y), generated on the device into
 * the DEVICE buffers left/right. Bit-identical to the CPU generator. */
int d3g_generate(d3g_ctx* ctx, int cfg, int side, uint64_t lo, uint64_t hi, uint64_t* left,
                 uint64_t* right);
uint64_t d3g_cfg_rows(int cfg);
/* Measured 32-bit logic-op throughput of this device (LOP3 chains, ops/s);
 * the denominator of the DenseEC integer-pipe roofline. */
int d3g_alu_peak(d3g_ctx* ctx, double* ops_per_sec);
/* Measured shared-memory read bandwidth of this device (conflict-free
 * LDS.128 streams on every SM, bytes/s): the roofline denominator of the
 * smem-bound DenseEC hot pass. */
int d3g_smem_peak(d3g_ctx* ctx, double* bytes_per_sec);
int d3g_ctx_device(d3g_ctx* ctx);

/* ---- map_tables (P/src/mapping.cpp:342-420) --------------------------------
 * dim3::MappingOutput (P/include/dim3/mapping.hpp:124-132) in host arrays the
 * caller sizes: r_x/r_y/r_kept hold up to r->n entries, s_z/s_y s->n, and the
 * reverse dictionaries rev_x/rev_y/rev_z (code -> value) up to r->n, r->n + s->n,
 * s->n (filled only for dictionary-coded columns; NULL to skip). Codes are
 * the reference's exact codes. r_kept lists the surviving R rows' original
 * indices (filled only when the semi-join dropped rows). The options use
 * declared_x/y/z (SkipFlags) and natural_keys_auto (map_with_fallback). */
typedef struct {
  uint32_t *r_x, *r_y, *s_z, *s_y, *r_kept;
  uint64_t *rev_x, *rev_y, *rev_z;
  uint64_t kept, dropped_r, x_card, y_card, z_card;
  int32_t natural_x, natural_y, natural_z, pad;
} d3g_mapping;
int d3g_map_tables(d3g_ctx* ctx, const d3g_table* r, const d3g_table* s, const d3g_opts* o,
                   d3g_mapping* out);

/* ---- join-aggregate (P/src/engine.cpp:537-722) -----------------------------
 * dim3::ValuedTable (relation.hpp:49-53): a table plus one double per row;
 * values live in device memory iff base.on_device. */
typedef struct {
  d3g_table base;
  const double* values;
} d3g_valued_table;

/* dim3::AggFn / dim3::CombineFn (P/include/dim3/engine.hpp:129-130). */
#define D3G_AGG_SUM 0
#define D3G_AGG_COUNT 1
#define D3G_AGG_MIN 2
#define D3G_AGG_MAX 3
#define D3G_AGG_AVG 4
#define D3G_COMBINE_MULTIPLY 0
#define D3G_COMBINE_ADD 1
#define D3G_COMBINE_ABS_DIFF 2
#define D3G_COMBINE_LEFT 3
#define D3G_COMBINE_RIGHT 4

/* AggregateResult's pairs (decoded raw x, z) and values; cap rows, n set. */
typedef struct {
  uint64_t* x;
  uint64_t* z;
  double* values;
  uint64_t cap;
  uint64_t n;
  int32_t on_device;
  int32_t pad;
} d3g_agg_pairs;

/* join_aggregate_both (engine.cpp:537-722), caller orientation (no swap):
 * one row per distinct (x, z) with agg over every match of
 * combine(r.value, s.value). Values are bit-identical to the reference's
 * (same accumulation order, round-to-nearest, no FMA). force = classical
 * raises D3G_CONFIG_ERROR like the reference. out == NULL or
 * opts->count_only: the count and report only. Report: strategy "hybrid",
 * cards, dropped_r, out_j (= out_j_estimate, exact), f2_evaluations,
 * dense_z/sparse_z, pairs_sparse/pairs_dense, out_p; ms_sparse is the whole
 * aggregation pass. */
int d3g_join_aggregate(d3g_ctx* ctx, const d3g_valued_table* r, const d3g_valued_table* s,
                       int combine, int agg, const d3g_consts* c, const d3g_opts* o,
                       d3g_report* rep, d3g_agg_pairs* out);

/* ---- table files (P/src/relation.cpp) -------------------------------------
 * Binary table = little-endian u64 (left, right) pairs, no header. Text =
 * "left<sep>right\n" in decimal, sep '\t' (tsv) or ',' (csv). */
#define D3G_FMT_AUTO 0
#define D3G_FMT_TSV 1
#define D3G_FMT_CSV 2
#define D3G_FMT_BINARY 3
/* detect_format (relation.cpp:13-20): requested unless AUTO, else by
 * extension (.tsv/.txt tsv, .csv csv, .bin binary, otherwise tsv). */
int d3g_detect_format(const char* path, int requested);
/* Rows of a binary table file: D3G_IO_ERROR if it cannot be opened,
 * D3G_FORMAT_ERROR if its length is not a multiple of 16 (read_binary,
 * relation.cpp:98-107). Host-only. */
int d3g_binary_rows(const char* path, uint64_t* n);
/* read_binary (relation.cpp:98-127) into the DEVICE columns left/right
 * (n = d3g_binary_rows): the file streams through pinned chunks into HBM and
 * is de-interleaved on the GPU. */
int d3g_read_binary(d3g_ctx* ctx, const char* path, uint64_t* left, uint64_t* right, uint64_t n);
/* save_table (relation.cpp:164-204) of n (left, right) pairs, device or host
 * columns: interleaving (binary) or decimal formatting (tsv/csv) runs on the
 * GPU, the bytes are copied back in chunks and written. The CLI's --out of
 * the decoded (x, z) pairs (P/tools/dim3.cpp:212-218). */
int d3g_save_pairs(d3g_ctx* ctx, const uint64_t* left, const uint64_t* right, uint64_t n,
                   int on_device, const char* path, int format);

/* ---- multi-GPU: the x-sharded join_project --------------------
 * With an exchange set on the context, d3g_join_project runs as one rank of
 * an x-sharded job: r is THIS rank's shard of R (the rows whose x value the
 * rank owns; shards are disjoint in x, e.g. contiguous x ranges or hash(x) mod
 * nranks) and s is the whole of S. Partitioning R by x is intersection-free
 * (the reference's x chunking, P/include/dim3/common.hpp:130-155), so no pair
 * crosses ranks. The ranks exchange only
 *   - the inputs of the global decisions: |R|, the column maxima and natural-
 *     key sample tests of R, the per-y raw R counts (f1's join size), the m_x
 *     histogram, dR(y), nnz and live/distinct x (f2, P/src/costmodel.cpp:515-586);
 *   - the final tallies (count, fingerprint, pairs split, counters).
 * Every rank then reports the JOB's totals (out_p, checksums, cards, split);
 * materialized pairs are the rank's own. f1 uses the exact bag join size (the
 * reference samples it above 65,536 rows); the natural-key sample test runs
 * on each shard's rows against the global |R|. |R| >= |S| is required (no
 * swap: the sharded table must stay the engine's R).
 * Transports: NCCL (ncclAllReduce / ncclAllGather on the context's stream,
 * over NVLink/NVSwitch; libnccl is dlopen'ed), or a host callback that
 * performs each collective on host buffers (gloo, threads, replay). */
#define D3G_EX_SUM_U64 0
#define D3G_EX_SUM_U32 1
#define D3G_EX_MAX_U64 2
#define D3G_EX_GATHER 3  /* buf holds nranks * count bytes; fill the other ranks' blocks */
typedef int (*d3g_exchange_fn)(void* user, int op, void* buf, uint64_t count);
/* A new NCCL unique id (128 bytes) for rank 0 to share with the others. */
int d3g_nccl_unique_id(void* id128);
/* ncclCommInitRank on the context's device (collective over the job). */
int d3g_ctx_set_nccl(d3g_ctx* ctx, const void* id128, int nranks, int rank);
/* Host-callback transport; nranks = 1 and fn = NULL clear the exchange. */
int d3g_ctx_set_exchange(d3g_ctx* ctx, int nranks, int rank, d3g_exchange_fn fn, void* user);

/* Host-only policy entry points (callable without a GPU). */
uint32_t d3g_f3_threshold(uint32_t m_x, uint32_t y_card, const d3g_consts* c);
double d3g_f1(uint64_t size_r, uint64_t size_s, uint64_t out_j, const d3g_consts* c);
/* f2 decisions tabulated per degree value from the global degree
 * histograms: mx_hist[m] = #x with m_x = m (m < mx_len), mz_hist likewise
 * (mz_hist[0] = gap codes). dense_of_mz[m] (mz_len bytes) receives 1 iff a
 * z of degree m goes to the dense panel. force: D3G_HYBRID/AUTO cost-based,
 * D3G_SPARSE_ONLY, D3G_DENSE_ONLY. *evaluations = #z with m_z > 0. */
int d3g_f2_decide(const uint64_t* mx_hist, uint64_t mx_len, const uint64_t* mz_hist,
                  uint64_t mz_len, uint64_t x_card, uint64_t y_card, uint64_t z_card,
                  uint64_t out_j, const d3g_consts* c, int force, uint8_t* dense_of_mz,
                  uint64_t* evaluations);

#ifdef __cplusplus
}
#endif
#endif /* DIM3_B200_H */
