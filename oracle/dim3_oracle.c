/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's hybrid
 * Join-Project path, used as the parity checker for the CUDA product path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library. It is pinned against the reference itself
 * (oracle/_ref/libdim3ref.so, built from /root/reference by oracle/Makefile)
 * and against the golden values in SURVEY §8(c) / tests/golden/.
 *
 * P = /root/reference/proj. Function-by-function:
 *   mix64 ..................... P/include/dim3/common.hpp:42-49
 *   SplitMix64 ................ P/include/dim3/datagen.hpp:176-193
 *   zipf_cum / zipf_draw ...... P/src/datagen.cpp:10-25
 *   convention G (cfg1..cfg5) . SURVEY Appendix A
 *   detect_natural_keys ....... P/src/mapping.cpp:281-295
 *   require_natural ........... P/src/mapping.cpp:328-338
 *   resolve_skips/fallback .... P/src/engine.cpp:25-50
 *   partition_bits_for ........ P/src/mapping.cpp:308-316
 *   Dictionary codes .......... P/src/mapping.cpp:191-251 (partition-major,
 *                               first-seen within a partition)
 *   map_tables ................ P/src/mapping.cpp:342-420
 *   build_csr ................. P/src/relation.cpp:206-258
 *   compute_degree_stats ...... P/src/costmodel.cpp:425-438, 350-364
 *   estimate_out_j_raw, f1 .... P/src/costmodel.cpp:375-423, 442-447
 *   pow1m, check_(non)simd, f3,P/src/costmodel.cpp:17-22, 449-483
 *   mx/mz bucket, F2Evaluator . P/src/costmodel.cpp:499-586
 *   partition_s_csr ........... P/src/partition.cpp:5-80
 *   sparse_bmm ................ P/src/sparsebmm.cpp:11-106
 *   dense_ec, block_and_any, .. P/src/denseec.cpp:8-153,
 *   probe_any                   P/include/dim3/bitmap.hpp:23-48
 *   join_project_extended ..... P/src/engine.cpp:351-498 (hybrid branch)
 */
#define _GNU_SOURCE
#include "dim3_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef uint32_t code_t;
typedef unsigned __int128 u128;

static char g_err[256];
const char* orc_last_error(void) { return g_err; }

static inline uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}
uint64_t orc_mix64(uint64_t x) { return mix64(x); }

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 1);
  if (!p) {
    fprintf(stderr, "oracle: out of memory (%zu bytes)\n", n);
    abort();
  }
  return p;
}
static void* xcalloc(size_t n, size_t s) {
  void* p = calloc(n ? n : 1, s ? s : 1);
  if (!p) {
    fprintf(stderr, "oracle: out of memory\n");
    abort();
  }
  return p;
}

/* ------------------------------------------------------------------------
 * Convention G generator. SplitMix64 draw k (0-based)
 * is mix64(seed + (k+1) * golden), so any row range is generated directly.
 */
#define GOLDEN 0x9e3779b97f4a7c15ull
static inline uint64_t sm_draw(uint64_t seed, uint64_t k) {
  return mix64(seed + (k + 1) * GOLDEN);
}
static inline uint64_t bounded(uint64_t r, uint64_t n) {
  return (uint64_t)(((u128)r * n) >> 64);
}
static inline double unit_of(uint64_t r) {
  return (double)(r >> 11) * 0x1.0p-53;
}

typedef struct {
  double alpha;
  uint64_t n;
  double* cum;
} zipf_t;
static zipf_t g_zipf[4];
static pthread_mutex_t g_zipf_mu = PTHREAD_MUTEX_INITIALIZER;

static const double* zipf_cum(uint64_t n, double alpha) {
  pthread_mutex_lock(&g_zipf_mu);
  for (int i = 0; i < 4; ++i)
    if (g_zipf[i].cum && g_zipf[i].n == n && g_zipf[i].alpha == alpha) {
      pthread_mutex_unlock(&g_zipf_mu);
      return g_zipf[i].cum;
    }
  int slot = 0;
  for (int i = 0; i < 4; ++i)
    if (!g_zipf[i].cum) {
      slot = i;
      break;
    }
  free(g_zipf[slot].cum);
  double* cum = xmalloc(n * sizeof(double));
  double run = 0;
  for (uint64_t r = 1; r <= n; ++r) {
    run += pow((double)r, -alpha);
    cum[r - 1] = run;
  }
  g_zipf[slot].alpha = alpha;
  g_zipf[slot].n = n;
  g_zipf[slot].cum = cum;
  pthread_mutex_unlock(&g_zipf_mu);
  return cum;
}

static inline uint64_t zipf_pick(uint64_t r, const double* cum, uint64_t n) {
  double u = unit_of(r) * cum[n - 1];
  uint64_t lo = 0, hi = n; /* upper_bound: first cum[i] > u */
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (cum[mid] > u)
      hi = mid;
    else
      lo = mid + 1;
  }
  if (lo == n) lo = n - 1;
  return lo;
}

/* Rows per side for cfg 1..5. */
uint64_t orc_cfg_rows(int cfg) {
  switch (cfg) {
    case 1: return 100000ull;
    case 2: return 5000000ull;
    case 3: return 20000000ull;
    case 4: return 10000000ull;
    case 5: return 200000000ull;
  }
  return 0;
}

/* side 0 = R rows (x, y), side 1 = S rows (z, y); rows [lo, hi). */
int orc_gen(int cfg, int side, uint64_t lo, uint64_t hi, uint64_t* left,
            uint64_t* right) {
  uint64_t nr = orc_cfg_rows(cfg);
  if (nr == 0 || hi > nr || lo > hi) {
    snprintf(g_err, sizeof g_err, "bad generator request");
    return 2;
  }
  if (cfg == 2) side = 0; /* S := R */
  uint64_t seed = (uint64_t)cfg;
  uint64_t base = side == 0 ? 0 : 2 * nr;
  if (cfg == 1 || cfg == 3) {
    uint64_t nx = cfg == 1 ? 10000 : 2000000;
    uint64_t ny = cfg == 1 ? 1000 : 10000000;
    for (uint64_t i = lo; i < hi; ++i) {
      left[i - lo] = bounded(sm_draw(seed, base + 2 * i), nx);
      right[i - lo] = bounded(sm_draw(seed, base + 2 * i + 1), ny);
    }
  } else if (cfg == 2 || cfg == 5) {
    uint64_t nx = cfg == 2 ? 200000 : 10000000;
    uint64_t ny = cfg == 2 ? 50000 : 1000000;
    double alpha = cfg == 2 ? 1.0 : 1.2;
    const double* cum = zipf_cum(ny, alpha);
    for (uint64_t i = lo; i < hi; ++i) {
      left[i - lo] = bounded(sm_draw(seed, base + 2 * i), nx);
      right[i - lo] = zipf_pick(sm_draw(seed, base + 2 * i + 1), cum, ny);
    }
  } else { /* cfg 4: pools xpool(1e6), zpool(1e6), ypool(1e5) drawn first */
    const uint64_t NP = 1000000, NY = 100000, P = 2 * NP + NY;
    const double* cum = zipf_cum(NY, 0.8);
    uint64_t pool_off = side == 0 ? 0 : NP;
    for (uint64_t i = lo; i < hi; ++i) {
      uint64_t a = bounded(sm_draw(seed, P + base + 2 * i), NP);
      uint64_t b = zipf_pick(sm_draw(seed, P + base + 2 * i + 1), cum, NY);
      left[i - lo] = sm_draw(seed, pool_off + a);
      right[i - lo] = sm_draw(seed, 2 * NP + b);
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------
 * u64 -> u32 open-addressing map (oracle-internal helper; the reference's
 * slot layout is irrelevant to the codes it assigns, see dict_build).
 */
typedef struct {
  uint64_t* keys;
  uint32_t* vals; /* value + 1, 0 = empty */
  uint64_t mask;
} u64map;

static void map_init(u64map* m, uint64_t expect) {
  uint64_t cap = 16;
  while (cap < 2 * expect + 16) cap <<= 1;
  m->keys = xmalloc(cap * 8);
  m->vals = xcalloc(cap, 4);
  m->mask = cap - 1;
}
static void map_free(u64map* m) {
  free(m->keys);
  free(m->vals);
}
/* Returns pointer to the value slot; *fresh set when inserted. */
static uint32_t* map_slot(u64map* m, uint64_t k, int* fresh) {
  uint64_t i = mix64(k ^ 0x5bd1e995ull) & m->mask;
  for (;;) {
    if (m->vals[i] == 0) {
      m->keys[i] = k;
      *fresh = 1;
      return &m->vals[i];
    }
    if (m->keys[i] == k) {
      *fresh = 0;
      return &m->vals[i];
    }
    i = (i + 1) & m->mask;
  }
}
static int map_get(const u64map* m, uint64_t k, uint32_t* v) {
  uint64_t i = mix64(k ^ 0x5bd1e995ull) & m->mask;
  for (;;) {
    if (m->vals[i] == 0) return 0;
    if (m->keys[i] == k) {
      *v = m->vals[i] - 1;
      return 1;
    }
    i = (i + 1) & m->mask;
  }
}

/* ------------------------------------------------------------------------
 * Mapping (P/src/mapping.cpp). */

/* detect_natural_keys, c = 2, distinct_estimate = n (mapping.cpp:281-295). */
static int detect_natural(const uint64_t* col, uint64_t n) {
  if (n == 0) return 0;
  double bound = 2.0 * (double)n;
  uint64_t samples = n < 4096 ? n : 4096;
  uint64_t stride = n / samples;
  if (stride < 1) stride = 1;
  for (uint64_t i = 0; i < samples; ++i) {
    uint64_t idx = i * stride;
    if (idx > n - 1) idx = n - 1;
    if ((double)col[idx] >= bound) return 0;
  }
  return 1;
}

/* require_natural (mapping.cpp:328-338): max+1, or -1 on values >= 2^32. */
static int64_t natural_card(const uint64_t* col, uint64_t n) {
  uint64_t mx = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (col[i] > mx) mx = col[i];
  if (n > 0 && mx >= (1ull << 32)) return -1;
  return n == 0 ? 0 : (int64_t)(mx + 1);
}

/* partition_bits_for (mapping.cpp:308-316) with llc 12 MiB, load 0.7. */
static int partition_bits_for(uint64_t len) {
  double est = (double)len / 0.7 * 8.0;
  int k = 0;
  while (k < 12 && est / (double)(1ull << k) > (double)(12ull << 20)) ++k;
  return k;
}

typedef struct {
  int identity;
  uint64_t card;
  uint64_t* rev; /* code -> value (dictionary only) */
  u64map map;    /* value -> code (dictionary only) */
} dict_t;

/* Dictionary::build_impl codes (mapping.cpp:191-251): values scatter to
 * partition h & (2^k - 1) in input order; each partition numbers its
 * distinct values first-seen from 0; partitions are then rebased in order.
 * Probe windows and stash placement never change a local code. */
static void dict_build(dict_t* d, const uint64_t* v, uint64_t n,
                       code_t* codes) {
  int k = partition_bits_for(n);
  uint64_t nparts = 1ull << k;
  uint64_t* cnt = xcalloc(nparts, 8);
  code_t* local = xmalloc(n * sizeof(code_t) + 4);
  map_init(&d->map, n);
  d->identity = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t p = k == 0 ? 0 : (mix64(v[i]) & (nparts - 1));
    int fresh;
    uint32_t* s = map_slot(&d->map, v[i], &fresh);
    if (fresh) *s = (uint32_t)(cnt[p]++) + 1;
    local[i] = *s - 1;
  }
  uint64_t* base = xmalloc(nparts * 8);
  uint64_t run = 0;
  for (uint64_t p = 0; p < nparts; ++p) {
    base[p] = run;
    run += cnt[p];
  }
  d->card = run;
  d->rev = xmalloc(run * 8 + 8);
  /* rebase the map's stored local codes into global codes */
  for (uint64_t i = 0; i <= d->map.mask; ++i) {
    if (d->map.vals[i] == 0) continue;
    uint64_t val = d->map.keys[i];
    uint64_t p = k == 0 ? 0 : (mix64(val) & (nparts - 1));
    uint64_t g = base[p] + (d->map.vals[i] - 1);
    d->map.vals[i] = (uint32_t)g + 1;
    d->rev[g] = val;
  }
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t p = k == 0 ? 0 : (mix64(v[i]) & (nparts - 1));
    codes[i] = (code_t)(base[p] + local[i]);
  }
  free(cnt);
  free(local);
  free(base);
}
static void dict_identity(dict_t* d, uint64_t card) {
  memset(d, 0, sizeof *d);
  d->identity = 1;
  d->card = card;
}
static void dict_free(dict_t* d) {
  if (!d->identity) {
    free(d->rev);
    map_free(&d->map);
  }
}
static inline uint64_t dict_value(const dict_t* d, code_t c) {
  return d->identity ? c : d->rev[c];
}

typedef struct {
  code_t *a, *b;
  uint64_t n;
  uint64_t a_card, b_card;
} mtable;

typedef struct {
  mtable r, s;
  dict_t dx, dy, dz;
  uint64_t dropped_r;
} mapping_t;

/* map_tables (mapping.cpp:342-420); returns 0 or 2 (ConfigError). */
static int map_tables(const uint64_t* rl, const uint64_t* rr, uint64_t nr,
                      const uint64_t* sl, const uint64_t* sr, uint64_t ns,
                      int sx, int sy, int sz, mapping_t* m) {
  memset(m, 0, sizeof *m);
  code_t* s_y = xmalloc(ns * 4 + 4);
  code_t* s_z = xmalloc(ns * 4 + 4);
  if (sy) {
    int64_t c1 = natural_card(sr, ns), c2 = natural_card(rr, nr);
    if (c1 < 0 || c2 < 0) goto cfg_err;
    dict_identity(&m->dy, (uint64_t)(c1 > c2 ? c1 : c2));
    for (uint64_t i = 0; i < ns; ++i) s_y[i] = (code_t)sr[i];
  } else {
    dict_build(&m->dy, sr, ns, s_y);
  }
  if (sz) {
    int64_t c = natural_card(sl, ns);
    if (c < 0) goto cfg_err;
    dict_identity(&m->dz, (uint64_t)c);
    for (uint64_t i = 0; i < ns; ++i) s_z[i] = (code_t)sl[i];
  } else {
    dict_build(&m->dz, sl, ns, s_z);
  }
  m->s.a = s_z;
  m->s.b = s_y;
  m->s.n = ns;
  m->s.a_card = m->dz.card;
  m->s.b_card = m->dy.card;
  {
    code_t* r_y = xmalloc(nr * 4 + 4);
    uint64_t* surv_x = xmalloc(nr * 8 + 8);
    uint64_t kept = 0;
    for (uint64_t i = 0; i < nr; ++i) {
      uint32_t yc;
      int ok;
      if (m->dy.identity) {
        ok = rr[i] < m->dy.card;
        yc = (uint32_t)rr[i];
      } else {
        ok = map_get(&m->dy.map, rr[i], &yc);
      }
      if (!ok) {
        m->dropped_r++;
        continue;
      }
      r_y[kept] = yc;
      surv_x[kept] = rl[i];
      kept++;
    }
    code_t* r_x = xmalloc(kept * 4 + 4);
    if (sx) {
      int64_t c = natural_card(rl, nr); /* over all of R.left (:404-413) */
      if (c < 0) {
        free(r_y);
        free(surv_x);
        free(r_x);
        goto cfg_err;
      }
      dict_identity(&m->dx, (uint64_t)c);
      for (uint64_t i = 0; i < kept; ++i) r_x[i] = (code_t)surv_x[i];
    } else {
      dict_build(&m->dx, surv_x, kept, r_x);
    }
    free(surv_x);
    m->r.a = r_x;
    m->r.b = r_y;
    m->r.n = kept;
    m->r.a_card = m->dx.card;
    m->r.b_card = m->dy.card;
  }
  return 0;
cfg_err:
  snprintf(g_err, sizeof g_err, "natural-key skip requires values below 2^32");
  free(s_y);
  free(s_z);
  return 2;
}

static void mapping_free(mapping_t* m) {
  free(m->r.a);
  free(m->r.b);
  free(m->s.a);
  free(m->s.b);
  dict_free(&m->dx);
  dict_free(&m->dy);
  dict_free(&m->dz);
}

/* ------------------------------------------------------------------------
 * CSR (P/src/relation.cpp:206-258). */
typedef struct {
  uint64_t* row_ptr;
  code_t* col;
  uint64_t n_rows, n_cols, nnz;
} csr_t;

static void csr_free(csr_t* c) {
  free(c->row_ptr);
  free(c->col);
}

static void build_csr(const mtable* t, csr_t* m) {
  const code_t* major = t->a;
  const code_t* minor = t->b;
  uint64_t n_rows = t->a_card, n_cols = t->b_card, n = t->n;
  /* pass 1: stable counting sort by minor */
  uint64_t* cnt = xcalloc(n_cols + 1, 8);
  for (uint64_t i = 0; i < n; ++i) cnt[minor[i] + 1]++;
  for (uint64_t i = 1; i <= n_cols; ++i) cnt[i] += cnt[i - 1];
  code_t* maj1 = xmalloc(n * 4 + 4);
  code_t* min1 = xmalloc(n * 4 + 4);
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t pos = cnt[minor[i]]++;
    maj1[pos] = major[i];
    min1[pos] = minor[i];
  }
  free(cnt);
  /* pass 2: stable counting sort by major */
  uint64_t* rp = xcalloc(n_rows + 1, 8);
  for (uint64_t i = 0; i < n; ++i) rp[maj1[i] + 1]++;
  for (uint64_t i = 1; i <= n_rows; ++i) rp[i] += rp[i - 1];
  code_t* min2 = xmalloc(n * 4 + 4);
  uint64_t* cur = xmalloc(n_rows * 8 + 8);
  memcpy(cur, rp, n_rows * 8);
  for (uint64_t i = 0; i < n; ++i) min2[cur[maj1[i]]++] = min1[i];
  free(cur);
  free(maj1);
  free(min1);
  /* collapse duplicates per row */
  m->col = xmalloc(n * 4 + 4);
  m->row_ptr = xcalloc(n_rows + 1, 8);
  uint64_t w = 0;
  for (uint64_t r = 0; r < n_rows; ++r) {
    uint64_t lo = rp[r], hi = rp[r + 1];
    for (uint64_t i = lo; i < hi; ++i) {
      if (i > lo && min2[i] == min2[i - 1]) continue;
      m->col[w++] = min2[i];
    }
    m->row_ptr[r + 1] = w;
  }
  free(rp);
  free(min2);
  m->n_rows = n_rows;
  m->n_cols = n_cols;
  m->nnz = w;
}

/* ------------------------------------------------------------------------
 * Cost model (P/src/costmodel.cpp). */
static double pow1m(double p, double m) {
  if (p >= 1.0) return m > 0 ? 0.0 : 1.0;
  if (p <= 0.0) return 1.0;
  return exp(m * log1p(-p));
}
static inline double dmin(double a, double b) { return (b < a) ? b : a; }

double orc_check_nonsimd(double m_x, double m_z, double y_card) {
  double ps = y_card > 0 ? m_z / y_card : 0.0;
  if (ps <= 0.0) return m_x;
  return (1.0 - pow1m(ps, m_x)) / ps;
}
double orc_check_simd(double m_x, double m_z, double y_card, uint32_t w) {
  double blocks = w > 0 ? y_card / (double)w : 0.0;
  double q = y_card > 0 ? dmin(1.0, (m_x * m_z) / (y_card * y_card)) : 0.0;
  double pd = 1.0 - pow1m(q, (double)w);
  if (pd <= 0.0) return blocks;
  return (1.0 - pow1m(pd, blocks)) / pd;
}
double orc_f3(double m_x, double m_z, uint32_t y_card, const orc_consts* c) {
  return orc_check_nonsimd(m_x, m_z, y_card) * c->t_ECs -
         orc_check_simd(m_x, m_z, y_card, c->w) * c->t_ECd;
}
uint32_t orc_f3_threshold(uint32_t m_x, uint32_t y_card, const orc_consts* c) {
  if (y_card == 0) return 1;
  if (orc_f3(m_x, y_card, y_card, c) <= 0) return y_card + 1;
  if (orc_f3(m_x, 1, y_card, c) > 0) return 0;
  uint32_t lo = 1, hi = y_card;
  while (hi - lo > 1) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (orc_f3(m_x, mid, y_card, c) <= 0)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}
double orc_f1(uint64_t size_r, uint64_t size_s, uint64_t out_j,
              const orc_consts* c) {
  return 2.0 * (double)(size_r + size_s) * c->t_map +
         (double)out_j * c->t_randRW - (double)out_j * c->t_hash;
}
uint32_t orc_mx_bucket_key(uint32_t m) {
  uint32_t d = 0, p10 = 1;
  while (m / p10 >= 10) {
    p10 *= 10;
    ++d;
  }
  return d * 10 + m / p10;
}
uint32_t orc_mz_bucket_index(uint32_t m_z, uint32_t y_card) {
  if (y_card == 0) return 0;
  uint64_t idx = (uint64_t)m_z * 100 / y_card;
  return (uint32_t)(idx < 99 ? idx : 99);
}

/* estimate_out_j_raw (costmodel.cpp:375-423), u64 columns. */
uint64_t orc_estimate_out_j_raw(const uint64_t* r_y, uint64_t nr,
                                const uint64_t* s_y, uint64_t ns) {
  if (nr == 0 || ns == 0) return 0;
  const uint64_t exact_limit = 65536, sample_rows = 16384;
  u64map m;
  if (nr <= exact_limit && ns <= exact_limit) {
    map_init(&m, ns);
    uint64_t* cnt = xcalloc(ns + 1, 8);
    uint32_t next = 0;
    for (uint64_t i = 0; i < ns; ++i) {
      int fresh;
      uint32_t* s = map_slot(&m, s_y[i], &fresh);
      if (fresh) *s = ++next;
      cnt[*s - 1]++;
    }
    uint64_t sum = 0;
    for (uint64_t i = 0; i < nr; ++i) {
      uint32_t v;
      if (map_get(&m, r_y[i], &v)) sum += cnt[v];
    }
    free(cnt);
    map_free(&m);
    return sum;
  }
  uint64_t ms = ns < sample_rows ? ns : sample_rows;
  uint64_t mr = nr < sample_rows ? nr : sample_rows;
  uint64_t ss = ns / ms, sr = nr / mr;
  map_init(&m, ms);
  uint64_t* cnt = xcalloc(ms + 1, 8);
  uint32_t next = 0;
  for (uint64_t i = 0; i < ms; ++i) {
    int fresh;
    uint32_t* s = map_slot(&m, s_y[i * ss], &fresh);
    if (fresh) *s = ++next;
    cnt[*s - 1]++;
  }
  u128 hits = 0;
  for (uint64_t i = 0; i < mr; ++i) {
    uint32_t v;
    if (map_get(&m, r_y[i * sr], &v)) hits += cnt[v];
  }
  free(cnt);
  map_free(&m);
  long double scaled = (long double)(uint64_t)hits *
                       ((long double)ns / ms) * ((long double)nr / mr);
  if (scaled > (long double)UINT64_MAX) return UINT64_MAX;
  return (uint64_t)scaled;
}

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

typedef struct {
  double sparse_fixed, out_unit;
  uint64_t n_mx;
  double* mx_median;
  uint64_t* mx_count;
  double mz_median[100];
  double dense_memo[100];
  int memo_set[100];
  uint64_t y_card;
  orc_consts c;
  uint64_t evaluations;
} f2eval;

/* F2Evaluator (costmodel.cpp:515-562). */
static void f2_init(f2eval* e, const uint32_t* m_x, uint64_t x_card,
                    const uint32_t* m_z, uint64_t z_card, uint64_t y_card,
                    uint64_t out_j, const orc_consts* c) {
  memset(e, 0, sizeof *e);
  e->c = *c;
  e->y_card = y_card;
  uint64_t r_nnz = 0, s_nnz = 0;
  for (uint64_t i = 0; i < x_card; ++i) r_nnz += m_x[i];
  for (uint64_t i = 0; i < z_card; ++i) s_nnz += m_z[i];
  e->sparse_fixed =
      ((2.0 * (double)x_card + (double)r_nnz) * c->t_seqR +
       2.0 * (double)r_nnz * c->t_randR) /
      (double)(z_card > 1 ? z_card : 1);
  e->out_unit = s_nnz > 0 ? (double)out_j / (double)s_nnz *
                                (c->t_seqR + c->t_randRW)
                          : 0.0;
  uint32_t* mx = xmalloc(x_card * 4 + 4);
  uint64_t n = 0;
  for (uint64_t i = 0; i < x_card; ++i)
    if (m_x[i] > 0) mx[n++] = m_x[i];
  qsort(mx, n, 4, cmp_u32);
  e->mx_median = xmalloc(64 * sizeof(double));
  e->mx_count = xmalloc(64 * 8);
  for (uint64_t i = 0; i < n;) {
    uint32_t key = orc_mx_bucket_key(mx[i]);
    uint64_t j = i;
    while (j < n && orc_mx_bucket_key(mx[j]) == key) ++j;
    e->mx_median[e->n_mx] = (double)mx[i + (j - i) / 2];
    e->mx_count[e->n_mx] = j - i;
    e->n_mx++;
    i = j;
  }
  free(mx);
  for (int g = 0; g < 100; ++g) e->mz_median[g] = -1.0;
  uint32_t* mz = xmalloc(z_card * 4 + 4);
  memcpy(mz, m_z, z_card * 4);
  qsort(mz, z_card, 4, cmp_u32);
  for (uint64_t i = 0; i < z_card;) {
    uint32_t g = orc_mz_bucket_index(mz[i], (uint32_t)y_card);
    uint64_t j = i;
    while (j < z_card && orc_mz_bucket_index(mz[j], (uint32_t)y_card) == g) ++j;
    e->mz_median[g] = (double)mz[i + (j - i) / 2];
    i = j;
  }
  free(mz);
}
static void f2_free(f2eval* e) {
  free(e->mx_median);
  free(e->mx_count);
}
/* dense_cost / score (costmodel.cpp:564-586). */
static double f2_score(f2eval* e, uint32_t mz) {
  e->evaluations++;
  double t_sparse = e->sparse_fixed + (double)mz * e->out_unit;
  uint32_t g = orc_mz_bucket_index(mz, (uint32_t)e->y_card);
  if (!e->memo_set[g]) {
    double mzq = e->mz_median[g];
    double total = 0;
    for (uint64_t i = 0; i < e->n_mx; ++i) {
      double scalar = orc_check_nonsimd(e->mx_median[i], mzq, (double)e->y_card) *
                      e->c.t_ECs;
      double wide = orc_check_simd(e->mx_median[i], mzq, (double)e->y_card,
                                   e->c.w) *
                    e->c.t_ECd;
      total += (double)e->mx_count[i] * dmin(scalar, wide);
    }
    e->dense_memo[g] = total;
    e->memo_set[g] = 1;
  }
  return t_sparse - e->dense_memo[g];
}

/* ------------------------------------------------------------------------
 * Kernels (P/src/sparsebmm.cpp, P/src/denseec.cpp). */
typedef struct {
  const csr_t *r, *s;          /* r_by_x, s_sparse_by_y */
  const uint64_t* panel;       /* dense rows, row_words each */
  const uint32_t* panel_mz;
  const code_t* panel_z;
  uint64_t n_dense, row_words, y_card, z_card;
  const orc_consts* c;
  int dense_mode;
  const dict_t *dx, *dz;
  int swapped;
  uint64_t x_lo, x_hi;
  /* outputs */
  uint64_t emitted_sparse, emitted_dense, inner;
  uint64_t wide_enc, probe_enc, blocks, probes, bitmaps_built, x_live;
  uint64_t sum, xr;
  uint64_t* pairs; /* optional (x,z) caller-oriented raw, interleaved */
  uint64_t pairs_n, pairs_cap;
  uint64_t* per_x;  /* optional per engine-x-code pair count */
  int do_sparse, do_dense;
} chunk_t;

static inline void emit(chunk_t* k, code_t xc, code_t zc) {
  uint64_t ex = dict_value(k->dx, xc), ez = dict_value(k->dz, zc);
  uint64_t cx = k->swapped ? ez : ex, cz = k->swapped ? ex : ez;
  uint64_t h = mix64(mix64(cx) ^ cz);
  k->sum += h;
  k->xr ^= h;
  if (k->per_x) k->per_x[xc]++;
  if (k->pairs) {
    if (k->pairs_n == k->pairs_cap) {
      k->pairs_cap = k->pairs_cap ? k->pairs_cap * 2 : 1024;
      k->pairs = realloc(k->pairs, k->pairs_cap * 16);
      if (!k->pairs) abort();
    }
    k->pairs[2 * k->pairs_n] = cx;
    k->pairs[2 * k->pairs_n + 1] = cz;
    k->pairs_n++;
  }
}

static void* run_chunk(void* arg) {
  chunk_t* k = arg;
  const csr_t* r = k->r;
  if (k->do_sparse) { /* sparsebmm.cpp:11-49 */
    int64_t* spa = xmalloc(k->z_card * 8 + 8);
    for (uint64_t z = 0; z < k->z_card; ++z) spa[z] = -1;
    for (uint64_t x = k->x_lo; x < k->x_hi; ++x) {
      int64_t stamp = (int64_t)x;
      for (uint64_t i = r->row_ptr[x]; i < r->row_ptr[x + 1]; ++i) {
        code_t y = r->col[i];
        for (uint64_t j = k->s->row_ptr[y]; j < k->s->row_ptr[y + 1]; ++j) {
          code_t z = k->s->col[j];
          k->inner++;
          if (spa[z] != stamp) {
            spa[z] = stamp;
            k->emitted_sparse++;
            emit(k, (code_t)x, z);
          }
        }
      }
    }
    free(spa);
  }
  if (k->do_dense && k->n_dense > 0) { /* denseec.cpp:8-86 */
    uint64_t rw = k->row_words;
    uint64_t* bm = xcalloc(rw, 8);
    uint64_t n_blocks = rw / (k->c->w / 64);
    uint32_t wpb = k->c->w / 64;
    uint32_t* thr = NULL;
    uint32_t thr_n = 0;
    for (uint64_t x = k->x_lo; x < k->x_hi; ++x) {
      uint64_t lo = r->row_ptr[x], hi = r->row_ptr[x + 1];
      if (hi == lo) continue;
      uint32_t m_x = (uint32_t)(hi - lo);
      uint32_t threshold = 0;
      if (k->dense_mode == 0) {
        if (m_x >= thr_n) {
          uint32_t nn = m_x + 64;
          thr = realloc(thr, nn * 4);
          for (uint32_t i = thr_n; i < nn; ++i) thr[i] = UINT32_MAX;
          thr_n = nn;
        }
        if (thr[m_x] == UINT32_MAX)
          thr[m_x] = orc_f3_threshold(m_x, (uint32_t)k->y_card, k->c);
        threshold = thr[m_x];
      }
      int ready = 0;
      for (uint64_t j = 0; j < k->n_dense; ++j) {
        uint32_t m_z = k->panel_mz[j];
        int wide = k->dense_mode == 1 ? 1 : k->dense_mode == 2 ? 0 : m_z > threshold;
        const uint64_t* row = k->panel + j * rw;
        int hit = 0;
        if (wide) {
          if (!ready) {
            for (uint64_t i = lo; i < hi; ++i)
              bm[r->col[i] >> 6] |= 1ull << (r->col[i] & 63);
            ready = 1;
            k->bitmaps_built++;
          }
          k->wide_enc++;
          for (uint64_t b = 0; b < n_blocks; ++b) {
            uint64_t acc = 0;
            for (uint32_t q = 0; q < wpb; ++q) acc |= bm[b * wpb + q] & row[b * wpb + q];
            k->blocks++;
            if (acc) {
              hit = 1;
              break;
            }
          }
        } else {
          k->probe_enc++;
          for (uint64_t i = lo; i < hi; ++i) {
            code_t y = r->col[i];
            k->probes++;
            if ((row[y >> 6] >> (y & 63)) & 1) {
              hit = 1;
              break;
            }
          }
        }
        if (hit) {
          k->emitted_dense++;
          emit(k, (code_t)x, k->panel_z[j]);
        }
      }
      if (ready)
        for (uint64_t i = lo; i < hi; ++i) bm[r->col[i] >> 6] = 0;
    }
    free(bm);
    free(thr);
  }
  return NULL;
}

/* ------------------------------------------------------------------------
 * join_project_extended, hybrid branch (engine.cpp:351-498), with the f1
 * gate evaluated and reported but the mapped path always taken (the
 * classical branch is outside the GPU scope; both yield the same set).
 *
 * pairs_out (optional): caller-owned buffer of 2*pairs_cap u64; receives
 * caller-oriented raw (x,z) in the reference's emission order (sparse
 * pairs then dense pairs, x ascending within each).
 * per_block (optional): n_blocks entries of {count,sum,xor} keyed by raw
 * caller x / block_width.
 */
int orc_join_project(const uint64_t* rl, const uint64_t* rr, uint64_t nr,
                     const uint64_t* sl, const uint64_t* sr, uint64_t ns,
                     const orc_consts* c, const orc_opts* o, orc_report* rep,
                     uint64_t* pairs_out, uint64_t pairs_cap,
                     uint64_t* pairs_n, uint32_t* dense_z_raw_mask_unused) {
  (void)dense_z_raw_mask_unused;
  memset(rep, 0, sizeof *rep);
  if (pairs_n) *pairs_n = 0;
  int swapped = ns > nr; /* engine_will_swap (engine.cpp:341-343) */
  const uint64_t *Rl = swapped ? sl : rl, *Rr = swapped ? sr : rr;
  const uint64_t *Sl = swapped ? rl : sl, *Sr = swapped ? rr : sr;
  uint64_t NR = swapped ? ns : nr, NS = swapped ? nr : ns;
  rep->swapped = swapped;
  rep->r_rows = NR;
  rep->s_rows = NS;
  rep->out_j_estimate = orc_estimate_out_j_raw(Rr, NR, Sr, NS);
  rep->f1 = orc_f1(NR, NS, rep->out_j_estimate, c);
  rep->f1_classical = rep->f1 > 0;

  /* map_with_fallback (engine.cpp:25-50) */
  int sx = 0, sy = 0, sz = 0;
  if (o->natural_keys_auto) {
    sx = detect_natural(Rl, NR);
    sy = detect_natural(Rr, NR) && detect_natural(Sr, NS);
    sz = detect_natural(Sl, NS);
  }
  mapping_t m;
  if (map_tables(Rl, Rr, NR, Sl, Sr, NS, sx, sy, sz, &m) != 0) {
    if (!sx && !sy && !sz) return 2;
    if (map_tables(Rl, Rr, NR, Sl, Sr, NS, 0, 0, 0, &m) != 0) return 2;
  }
  rep->natural_x = m.dx.identity;
  rep->natural_y = m.dy.identity;
  rep->natural_z = m.dz.identity;
  rep->dropped_r = m.dropped_r;
  rep->x_card = m.r.a_card;
  rep->y_card = m.s.b_card;
  rep->z_card = m.s.a_card;

  csr_t r_by_x, s_by_z;
  build_csr(&m.r, &r_by_x);
  build_csr(&m.s, &s_by_z);
  rep->r_nnz = r_by_x.nnz;
  rep->s_nnz = s_by_z.nnz;

  /* compute_degree_stats */
  uint64_t y_card = r_by_x.n_cols > s_by_z.n_cols ? r_by_x.n_cols : s_by_z.n_cols;
  uint32_t* m_x = xmalloc(r_by_x.n_rows * 4 + 4);
  uint32_t* m_z = xmalloc(s_by_z.n_rows * 4 + 4);
  for (uint64_t i = 0; i < r_by_x.n_rows; ++i) {
    m_x[i] = (uint32_t)(r_by_x.row_ptr[i + 1] - r_by_x.row_ptr[i]);
    rep->x_live += m_x[i] > 0;
  }
  for (uint64_t i = 0; i < s_by_z.n_rows; ++i)
    m_z[i] = (uint32_t)(s_by_z.row_ptr[i + 1] - s_by_z.row_ptr[i]);
  {
    uint32_t* dr = xcalloc(y_card + 1, 4);
    uint32_t* ds = xcalloc(y_card + 1, 4);
    for (uint64_t i = 0; i < r_by_x.nnz; ++i) dr[r_by_x.col[i]]++;
    for (uint64_t i = 0; i < s_by_z.nnz; ++i) ds[s_by_z.col[i]]++;
    u128 sum = 0;
    for (uint64_t y = 0; y < y_card; ++y) sum += (uint64_t)dr[y] * ds[y];
    rep->out_j = sum > (u128)UINT64_MAX ? UINT64_MAX : (uint64_t)sum;
    free(dr);
    free(ds);
  }

  /* partition_s_csr (partition.cpp:5-80) */
  uint64_t n_z = s_by_z.n_rows;
  uint8_t* dense = xcalloc(n_z, 1);
  f2eval ev;
  f2_init(&ev, m_x, r_by_x.n_rows, m_z, n_z, y_card, rep->out_j, c);
  int force = o->force;
  for (uint64_t z = 0; z < n_z; ++z) {
    if (m_z[z] == 0) continue;
    if (force == 3)
      dense[z] = 0;
    else if (force == 4)
      dense[z] = 1;
    else
      dense[z] = f2_score(&ev, m_z[z]) > 0;
    if (dense[z])
      rep->dense_z++;
    else
      rep->sparse_z++;
  }
  rep->f2_evaluations = ev.evaluations;
  f2_free(&ev);

  uint64_t row_words = ((s_by_z.n_cols + c->w - 1) / c->w * c->w) / 64;
  uint64_t* panel = xcalloc(rep->dense_z * row_words + 1, 8);
  uint32_t* panel_mz = xmalloc(rep->dense_z * 4 + 4);
  code_t* panel_z = xmalloc(rep->dense_z * 4 + 4);
  uint64_t sparse_nnz = 0, pr = 0;
  for (uint64_t z = 0; z < n_z; ++z) {
    if (!dense[z]) {
      sparse_nnz += s_by_z.row_ptr[z + 1] - s_by_z.row_ptr[z];
      continue;
    }
    panel_z[pr] = (code_t)z;
    panel_mz[pr] = m_z[z];
    uint64_t* row = panel + pr * row_words;
    for (uint64_t i = s_by_z.row_ptr[z]; i < s_by_z.row_ptr[z + 1]; ++i)
      row[s_by_z.col[i] >> 6] |= 1ull << (s_by_z.col[i] & 63);
    pr++;
  }
  rep->panel_bytes = rep->dense_z * row_words * 8;
  rep->sparse_nnz = sparse_nnz;
  csr_t sp;
  sp.n_rows = s_by_z.n_cols;
  sp.n_cols = s_by_z.n_rows;
  sp.row_ptr = xcalloc(sp.n_rows + 1, 8);
  sp.col = xmalloc(sparse_nnz * 4 + 4);
  sp.nnz = sparse_nnz;
  for (uint64_t z = 0; z < n_z; ++z) {
    if (dense[z]) continue;
    for (uint64_t i = s_by_z.row_ptr[z]; i < s_by_z.row_ptr[z + 1]; ++i)
      sp.row_ptr[s_by_z.col[i] + 1]++;
  }
  for (uint64_t i = 1; i <= sp.n_rows; ++i) sp.row_ptr[i] += sp.row_ptr[i - 1];
  {
    uint64_t* cur = xmalloc(sp.n_rows * 8 + 8);
    memcpy(cur, sp.row_ptr, sp.n_rows * 8);
    for (uint64_t z = 0; z < n_z; ++z) {
      if (dense[z]) continue;
      for (uint64_t i = s_by_z.row_ptr[z]; i < s_by_z.row_ptr[z + 1]; ++i)
        sp.col[cur[s_by_z.col[i]]++] = (code_t)z;
    }
    free(cur);
  }

  /* kernels, chunked over x (run_chunked, common.hpp:130-155): the sparse
   * kernel for every chunk first, then the dense kernel, so concatenated
   * emission equals the reference's (sparse pairs, then dense pairs). */
  int threads = o->threads < 1 ? 1 : o->threads;
  uint64_t n_rows = r_by_x.n_rows;
  uint64_t nchunks = (uint64_t)threads < n_rows ? (uint64_t)threads : n_rows;
  if (nchunks == 0) nchunks = 1;
  int want_pairs = pairs_out != NULL && !o->count_only;
  for (int phase = 0; phase < 2; ++phase) {
    chunk_t* ch = xcalloc(nchunks, sizeof(chunk_t));
    pthread_t* th = xmalloc(nchunks * sizeof(pthread_t));
    for (uint64_t ci = 0; ci < nchunks; ++ci) {
      chunk_t* k = &ch[ci];
      k->r = &r_by_x;
      k->s = &sp;
      k->panel = panel;
      k->panel_mz = panel_mz;
      k->panel_z = panel_z;
      k->n_dense = rep->dense_z;
      k->row_words = row_words;
      k->y_card = y_card;
      k->z_card = n_z;
      k->c = c;
      k->dense_mode = o->dense_mode;
      k->dx = &m.dx;
      k->dz = &m.dz;
      k->swapped = swapped;
      k->x_lo = n_rows * ci / nchunks;
      k->x_hi = n_rows * (ci + 1) / nchunks;
      k->do_sparse = phase == 0;
      k->do_dense = phase == 1;
      if (want_pairs) {
        k->pairs_cap = 1024;
        k->pairs = xmalloc(1024 * 16);
      }
    }
    if (nchunks == 1)
      run_chunk(&ch[0]);
    else {
      for (uint64_t ci = 0; ci < nchunks; ++ci)
        pthread_create(&th[ci], NULL, run_chunk, &ch[ci]);
      for (uint64_t ci = 0; ci < nchunks; ++ci) pthread_join(th[ci], NULL);
    }
    for (uint64_t ci = 0; ci < nchunks; ++ci) {
      chunk_t* k = &ch[ci];
      rep->pairs_sparse += k->emitted_sparse;
      rep->pairs_dense += k->emitted_dense;
      rep->spa_inner_count += k->inner;
      rep->dense_wide_encounters += k->wide_enc;
      rep->dense_probe_encounters += k->probe_enc;
      rep->dense_blocks_checked += k->blocks;
      rep->dense_probes_done += k->probes;
      rep->dense_row_bitmaps_built += k->bitmaps_built;
      rep->checksum_sum += k->sum;
      rep->checksum_xor ^= k->xr;
      if (want_pairs) {
        for (uint64_t i = 0; i < k->pairs_n && *pairs_n < pairs_cap; ++i) {
          pairs_out[2 * *pairs_n] = k->pairs[2 * i];
          pairs_out[2 * *pairs_n + 1] = k->pairs[2 * i + 1];
          (*pairs_n)++;
        }
        free(k->pairs);
      }
    }
    free(ch);
    free(th);
  }
  rep->out_p = rep->pairs_sparse + rep->pairs_dense;

  free(dense);
  free(panel);
  free(panel_mz);
  free(panel_z);
  csr_free(&sp);
  free(m_x);
  free(m_z);
  csr_free(&r_by_x);
  csr_free(&s_by_z);
  mapping_free(&m);
  return 0;
}
