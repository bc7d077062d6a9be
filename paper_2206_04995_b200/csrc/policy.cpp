// Host-side strategy policy: f1 gate, f3 threshold and the f2 dense/sparse
// decision, computed in double with the reference's exact arithmetic order so
// the GPU path makes the SAME decisions as the CPU reference.
//
//   pow1m ............ P/src/costmodel.cpp:17-22
//   f1 ............... P/src/costmodel.cpp:442-447
//   check_nonsimd .... P/src/costmodel.cpp:449-453
//   check_simd ....... P/src/costmodel.cpp:455-461
//   f3, f3_threshold . P/src/costmodel.cpp:463-483
//   mx_bucket_key .... P/src/costmodel.cpp:499-507
//   mz_bucket_index .. P/src/costmodel.cpp:509-513
//   F2Evaluator ...... P/src/costmodel.cpp:515-586
//   decision loop .... P/src/partition.cpp:17-38 (m_z == 0 skipped, tie -> sparse)
//
// F2Evaluator sorts the per-x and per-z degree vectors to take bucket
// medians. Every z with the same m_z gets the same score, so the GPU path
// ships only the two degree HISTOGRAMS to the host and this file evaluates
// the score once per distinct m_z. Medians are read off the cumulative
// histogram at exactly the index the reference uses (i + (j - i) / 2), so the
// result is bit-identical. Compiled with -ffp-contract=off.

#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/dim3_b200.h"

namespace {

double pow1m(double p, double m) {
  if (p >= 1.0) return m > 0 ? 0.0 : 1.0;
  if (p <= 0.0) return 1.0;
  return std::exp(m * std::log1p(-p));
}

inline double dmin(double a, double b) { return (b < a) ? b : a; }

double check_nonsimd(double m_x, double m_z, double y_card) {
  double ps = y_card > 0 ? m_z / y_card : 0.0;
  if (ps <= 0.0) return m_x;
  return (1.0 - pow1m(ps, m_x)) / ps;
}

double check_simd(double m_x, double m_z, double y_card, uint32_t w) {
  double blocks = w > 0 ? y_card / static_cast<double>(w) : 0.0;
  double q = y_card > 0 ? dmin(1.0, (m_x * m_z) / (y_card * y_card)) : 0.0;
  double pd = 1.0 - pow1m(q, static_cast<double>(w));
  if (pd <= 0.0) return blocks;
  return (1.0 - pow1m(pd, blocks)) / pd;
}

double f3(double m_x, double m_z, uint32_t y_card, const d3g_consts* c) {
  return check_nonsimd(m_x, m_z, y_card) * c->t_ECs -
         check_simd(m_x, m_z, y_card, c->w) * c->t_ECd;
}

uint32_t mx_bucket_key(uint32_t m) {
  uint32_t d = 0, p10 = 1;
  while (m / p10 >= 10) {
    p10 *= 10;
    ++d;
  }
  return d * 10 + m / p10;
}

uint32_t mz_bucket_index(uint32_t m_z, uint32_t y_card) {
  if (y_card == 0) return 0;
  uint64_t idx = static_cast<uint64_t>(m_z) * 100 / y_card;
  return static_cast<uint32_t>(idx < 99 ? idx : 99);
}

// Value at sorted position `pos` of the multiset described by hist, starting
// the walk at value `from` with `before` elements strictly below it.
uint64_t value_at(const uint64_t* hist, uint64_t len, uint64_t from, uint64_t before,
                  uint64_t pos) {
  uint64_t run = before;
  for (uint64_t m = from; m < len; ++m) {
    run += hist[m];
    if (run > pos) return m;
  }
  return len ? len - 1 : 0;
}

}  // namespace

extern "C" {

double d3g_f1(uint64_t size_r, uint64_t size_s, uint64_t out_j, const d3g_consts* c) {
  return 2.0 * static_cast<double>(size_r + size_s) * c->t_map +
         static_cast<double>(out_j) * c->t_randRW - static_cast<double>(out_j) * c->t_hash;
}

uint32_t d3g_f3_threshold(uint32_t m_x, uint32_t y_card, const d3g_consts* c) {
  if (y_card == 0) return 1;
  if (f3(m_x, y_card, y_card, c) <= 0) return y_card + 1;
  if (f3(m_x, 1, y_card, c) > 0) return 0;
  uint32_t lo = 1, hi = y_card;
  while (hi - lo > 1) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (f3(m_x, mid, y_card, c) <= 0)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

int d3g_f2_decide(const uint64_t* mx_hist, uint64_t mx_len, const uint64_t* mz_hist,
                  uint64_t mz_len, uint64_t x_card, uint64_t y_card, uint64_t z_card,
                  uint64_t out_j, const d3g_consts* c, int force, uint8_t* dense_of_mz,
                  uint64_t* evaluations) {
  for (uint64_t m = 0; m < mz_len; ++m) dense_of_mz[m] = 0;
  uint64_t evals = 0;
  for (uint64_t m = 1; m < mz_len; ++m) evals += mz_hist[m];
  if (evaluations) *evaluations = (force == D3G_SPARSE_ONLY || force == D3G_DENSE_ONLY) ? 0 : evals;
  if (force == D3G_SPARSE_ONLY) return 0;
  if (force == D3G_DENSE_ONLY) {
    for (uint64_t m = 1; m < mz_len; ++m) dense_of_mz[m] = mz_hist[m] ? 1 : 0;
    return 0;
  }
  // GlobalSizes (costmodel.cpp:517-522): nnz from the histograms.
  uint64_t r_nnz = 0, s_nnz = 0;
  for (uint64_t m = 1; m < mx_len; ++m) r_nnz += m * mx_hist[m];
  for (uint64_t m = 1; m < mz_len; ++m) s_nnz += m * mz_hist[m];
  const double sparse_fixed =
      ((2.0 * static_cast<double>(x_card) + static_cast<double>(r_nnz)) * c->t_seqR +
       2.0 * static_cast<double>(r_nnz) * c->t_randR) /
      static_cast<double>(z_card > 1 ? z_card : 1);
  const double out_unit = s_nnz > 0 ? static_cast<double>(out_j) / static_cast<double>(s_nnz) *
                                          (c->t_seqR + c->t_randRW)
                                    : 0.0;

  // m_x groups over the nonzero degrees (costmodel.cpp:536-548). Bucket keys
  // are non-decreasing in m, so each group is a contiguous value range.
  std::vector<double> mx_median;
  std::vector<uint64_t> mx_count;
  {
    uint64_t before = 0;  // nonzero degrees sorted below the current group
    uint64_t m = 1;
    while (m < mx_len) {
      uint32_t key = mx_bucket_key(static_cast<uint32_t>(m));
      uint64_t cnt = 0, e = m;
      while (e < mx_len && mx_bucket_key(static_cast<uint32_t>(e)) == key) cnt += mx_hist[e++];
      if (cnt > 0) {
        mx_median.push_back(
            static_cast<double>(value_at(mx_hist, mx_len, m, before, before + cnt / 2)));
        mx_count.push_back(cnt);
      }
      before += cnt;
      m = e;
    }
  }
  // m_z groups over ALL degrees including 0 (costmodel.cpp:551-562).
  double mz_median[100];
  for (int g = 0; g < 100; ++g) mz_median[g] = -1.0;
  {
    const uint32_t yc = static_cast<uint32_t>(y_card);
    uint64_t before = 0;
    uint64_t m = 0;
    while (m < mz_len) {
      uint32_t g = mz_bucket_index(static_cast<uint32_t>(m), yc);
      uint64_t cnt = 0, e = m;
      while (e < mz_len && mz_bucket_index(static_cast<uint32_t>(e), yc) == g) cnt += mz_hist[e++];
      if (cnt > 0)
        mz_median[g] = static_cast<double>(value_at(mz_hist, mz_len, m, before, before + cnt / 2));
      before += cnt;
      m = e;
    }
  }
  // dense_cost per m_z group, memoized (costmodel.cpp:564-586).
  double memo[100];
  bool have[100] = {};
  const double yd = static_cast<double>(y_card);
  for (uint64_t m = 1; m < mz_len; ++m) {
    if (mz_hist[m] == 0) continue;
    uint32_t g = mz_bucket_index(static_cast<uint32_t>(m), static_cast<uint32_t>(y_card));
    if (!have[g]) {
      double mzq = mz_median[g];
      double total = 0;
      for (size_t i = 0; i < mx_median.size(); ++i) {
        double scalar = check_nonsimd(mx_median[i], mzq, yd) * c->t_ECs;
        double wide = check_simd(mx_median[i], mzq, yd, c->w) * c->t_ECd;
        total += static_cast<double>(mx_count[i]) * dmin(scalar, wide);
      }
      memo[g] = total;
      have[g] = true;
    }
    double t_sparse = sparse_fixed + static_cast<double>(m) * out_unit;
    dense_of_mz[m] = (t_sparse - memo[g]) > 0 ? 1 : 0;
  }
  return 0;
}

}  // extern "C"
