/*
 * oracle/mla_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * CPU restatement (plain C, no BLAS) of the reference package `mla`'s blocked LU hot path.
 * It exists only so that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs can check (and time) the reference algorithm without Python/numba.
 * Nothing under paper_1611_06365_b200/ may import, link or call it.
 *
 * Parity status: PINNED.  Every function below is checked bit-for-bit against outputs of the
 * unmodified reference (imported from /root/reference/pkg/src in the build container by
 * tests/golden/make_golden.py; vectors committed under tests/golden/) -- see
 * tests/test_oracle_golden.py.  Bitwise equality is possible because the reference's numba
 * kernels are compiled without fastmath (no FMA contraction, pkg/README.md:14-15) and this
 * file is compiled with -ffp-contract=off, keeping one rounding per multiply and per add in
 * the same order.
 *
 * Storage: column-major float64, element (i,j) of a view at a[i + j*ld]; pivots int64,
 * view-local, ipiv[k] >= k (reference matrix.py:74-92).
 *
 * OpenMP is used only across independent columns / C tiles, which leaves every scalar
 * operation and its order untouched (same argument as reference kernels.py:3-9).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define A_(a, ld, i, j) ((a)[(int64_t)(i) + (int64_t)(j) * (int64_t)(ld)])

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_num_threads(int t) {
#ifdef _OPENMP
  if (t >= 1) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

/* reference matrix.py:47-59 (_splitmix64_fill): one SplitMix64 draw per entry, columns left to
 * right, u = ((z >> 11) + 1) / (2^53 + 2) in (0,1).  Draw number k (0-based, k = i + j*rows)
 * uses state seed + (k+1)*gamma, so the stream is counter-based. */
void orc_fill_random(double *a, int64_t rows, int64_t cols, int64_t ld, uint64_t seed) {
  uint64_t state = seed;
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i) {
      state += 0x9E3779B97F4A7C15ULL;
      uint64_t z = state;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
      z = z ^ (z >> 31);
      double u = (double)(z >> 11);
      A_(a, ld, i, j) = (u + 1.0) / 9007199254740994.0;
    }
}

/* reference lu.py:44-72 (_unb_pivoted): unblocked right-looking LU on an m x n view.
 * Strict '>' keeps the lowest row on ties (lu.py:53); an exactly-zero pivot column records
 * piv[j] = j, sets info and skips swap, scaling and the rank-1 update (lu.py:56-59); the swap
 * spans the view's n columns only (lu.py:60-64); multipliers by division (lu.py:65-67);
 * update a[i,t] = a[i,t] - a[i,j]*v, two roundings (lu.py:68-71). */
int orc_unb_pivoted(double *a, int64_t m, int64_t n, int64_t ld, int64_t *piv) {
  int info = 0;
  for (int64_t j = 0; j < n; ++j) {
    int64_t p = j;
    double best = fabs(A_(a, ld, j, j));
    for (int64_t i = j + 1; i < m; ++i) {
      double v = fabs(A_(a, ld, i, j));
      if (v > best) { best = v; p = i; }
    }
    piv[j] = p;
    if (best == 0.0) { info = 1; continue; }
    if (p != j)
      for (int64_t t = 0; t < n; ++t) {
        double tmp = A_(a, ld, j, t);
        A_(a, ld, j, t) = A_(a, ld, p, t);
        A_(a, ld, p, t) = tmp;
      }
    double alpha = A_(a, ld, j, j);
    double *restrict cj = &A_(a, ld, 0, j);
    for (int64_t i = j + 1; i < m; ++i) cj[i] = cj[i] / alpha;
    for (int64_t t = j + 1; t < n; ++t) {
      double v = A_(a, ld, j, t);
      double *restrict ct = &A_(a, ld, 0, t);
      for (int64_t i = j + 1; i < m; ++i) ct[i] = ct[i] - cj[i] * v;
    }
  }
  return info;
}

/* reference kernels.py:296-332 (laswp/_swap_cols): validate 0 <= ipiv < rows BEFORE touching
 * anything (326-327, IndexError -> return -1 here); interchange t <-> ipiv[t], ascending, or
 * descending when reverse. */
int orc_laswp(double *a, int64_t rows, int64_t cols, int64_t ld, const int64_t *ipiv,
              int64_t npiv, int reverse) {
  for (int64_t t = 0; t < npiv; ++t)
    if (ipiv[t] < 0 || ipiv[t] >= rows) return -1;
  if (npiv == 0 || cols == 0) return 0;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < cols; ++j) {
    double *c = &A_(a, ld, 0, j);
    if (reverse) {
      for (int64_t t = npiv - 1; t >= 0; --t) {
        int64_t p = ipiv[t];
        if (p != t) { double tmp = c[t]; c[t] = c[p]; c[p] = tmp; }
      }
    } else {
      for (int64_t t = 0; t < npiv; ++t) {
        int64_t p = ipiv[t];
        if (p != t) { double tmp = c[t]; c[t] = c[p]; c[p] = tmp; }
      }
    }
  }
  return 0;
}

/* reference kernels.py:264-293 (trsm_llu/_trsm_cols): x := trilu(low)^-1 x, unit diagonal never
 * read; dot-product form s = sum_l low[i,l]*x[l,j] ascending from 0.0, then x[i,j] -= s. */
void orc_trsm_llu(const double *low, int64_t w, int64_t ldl, double *x, int64_t c, int64_t ldx) {
  if (w <= 1 || c <= 0) return;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < c; ++j) {
    double *restrict xj = &A_(x, ldx, 0, j);
    for (int64_t i = 1; i < w; ++i) {
      double s = 0.0;
      for (int64_t l = 0; l < i; ++l) s += A_(low, ldl, i, l) * xj[l];
      xj[i] = xj[i] - s;
    }
  }
}

/* reference kernels.py:117-153 (_tile_product/_macro_block) and 195-201, 246-258 (step order):
 * C := alpha*C + beta*(A @ B).  k is cut into k_c-deep slices (config.py:34, default 256); each
 * slice accumulates acc = 0; acc += a*b for p ascending (two roundings per term), then the
 * first slice writes c = alpha*c + beta*acc and later ones c = c + beta*acc.  The m/n tiling
 * does not influence any bit (kernels.py:3-9), so a register tile that suits gcc is used. */
#define ORC_MR 16
#define ORC_NR 4
static void gemm_slice(double *c, int64_t m, int64_t n, int64_t ldc, const double *a, int64_t lda,
                       const double *b, int64_t ldb, int64_t kb, double alpha, double beta,
                       int first) {
  int64_t mt = (m + ORC_MR - 1) / ORC_MR, nt = (n + ORC_NR - 1) / ORC_NR;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t jt = 0; jt < nt; ++jt)
    for (int64_t it = 0; it < mt; ++it) {
      int64_t i0 = it * ORC_MR, j0 = jt * ORC_NR;
      int64_t iw = m - i0 < ORC_MR ? m - i0 : ORC_MR, jw = n - j0 < ORC_NR ? n - j0 : ORC_NR;
      double acc[ORC_NR][ORC_MR];
      for (int jj = 0; jj < ORC_NR; ++jj)
        for (int ii = 0; ii < ORC_MR; ++ii) acc[jj][ii] = 0.0;
      if (iw == ORC_MR && jw == ORC_NR) {
        for (int64_t p = 0; p < kb; ++p) {
          const double *restrict ap = &A_(a, lda, i0, p);
          for (int jj = 0; jj < ORC_NR; ++jj) {
            double bv = A_(b, ldb, p, j0 + jj);
            for (int ii = 0; ii < ORC_MR; ++ii) acc[jj][ii] += ap[ii] * bv;
          }
        }
      } else {
        for (int64_t p = 0; p < kb; ++p)
          for (int jj = 0; jj < jw; ++jj) {
            double bv = A_(b, ldb, p, j0 + jj);
            for (int ii = 0; ii < iw; ++ii) acc[jj][ii] += A_(a, lda, i0 + ii, p) * bv;
          }
      }
      for (int jj = 0; jj < jw; ++jj)
        for (int ii = 0; ii < iw; ++ii) {
          double *cc = &A_(c, ldc, i0 + ii, j0 + jj);
          if (first) *cc = alpha * *cc + beta * acc[jj][ii];
          else *cc = *cc + beta * acc[jj][ii];
        }
    }
}

/* reference kernels.py:205-234 (gemm_malleable): m==0||n==0 -> no-op; k==0 -> scale by alpha
 * when alpha != 1 (226-232). k_c <= 0 selects the reference default 256. */
void orc_gemm(double *c, int64_t m, int64_t n, int64_t ldc, const double *a, int64_t lda,
              const double *b, int64_t ldb, int64_t k, double alpha, double beta, int64_t k_c) {
  if (m <= 0 || n <= 0) return;
  if (k_c <= 0) k_c = 256;
  if (k == 0) {
    if (alpha != 1.0)
      for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) A_(c, ldc, i, j) = alpha * A_(c, ldc, i, j);
    return;
  }
  for (int64_t pc = 0; pc < k; pc += k_c) {
    int64_t kb = k - pc < k_c ? k - pc : k_c;
    gemm_slice(c, m, n, ldc, &A_(a, lda, 0, pc), lda, &A_(b, ldb, pc, 0), ldb, kb, alpha, beta,
               pc == 0);
  }
}

/* reference lu.py:140-180 (lu_blk_ll): left-looking blocked panel.  Per step: pending swaps into
 * the incoming block column (165), trsm against the factored triangle (166), one gemm (167-168),
 * unblocked factor of the block (171), swaps propagated left (173-174), pivots rebased to
 * panel-local (175).  The stop flag is polled once per completed step and only while columns
 * remain (177); here the flag is modelled as "set from poll number stop_trip on" (stop_trip <= 0:
 * no flag), which is exactly the CountingFlag fake of the reference tests (test_lu.py:149-156;
 * a pre-set flag is stop_trip == 1).  On a cut the accumulated swaps reach the untouched columns
 * (178).  Returns cols_factored; *singular is OR-ed. */
int64_t orc_lu_blk_ll(double *a, int64_t m, int64_t n, int64_t ld, int64_t b, int64_t *ipiv,
                      int64_t stop_trip, int *singular, int64_t k_c) {
  int64_t polls = 0;
  int64_t j = 0;
  while (j < n) {
    int64_t w = n - j < b ? n - j : b;
    if (j > 0) {
      orc_laswp(&A_(a, ld, 0, j), m, w, ld, ipiv, j, 0);
      orc_trsm_llu(a, j, ld, &A_(a, ld, 0, j), w, ld);
      orc_gemm(&A_(a, ld, j, j), m - j, w, ld, &A_(a, ld, j, 0), ld, &A_(a, ld, 0, j), ld, j, 1.0,
               -1.0, k_c);
    }
    int info = orc_unb_pivoted(&A_(a, ld, j, j), m - j, w, ld, ipiv + j);
    if (info) *singular = 1;
    if (j > 0) orc_laswp(&A_(a, ld, j, 0), m - j, j, ld, ipiv + j, w, 0);
    for (int64_t t = 0; t < w; ++t) ipiv[j + t] += j;
    j += w;
    if (stop_trip > 0 && j < n) {
      ++polls;
      if (polls >= stop_trip) {
        orc_laswp(&A_(a, ld, 0, j), m, n - j, ld, ipiv, j, 0);
        return j;
      }
    }
  }
  return n;
}

/* reference lu.py:106-137 (lu_blk_rl): right-looking blocked LU; panel by _unb_pivoted or one
 * level of blocked recursion when 0 < inner_b < w (125-130); swaps left and right (131-132),
 * rebase (133), trsm (134), gemm (135-136). */
void orc_lu_blk_rl(double *a, int64_t m, int64_t n, int64_t ld, int64_t b, int64_t inner_b,
                   int64_t *ipiv, int *singular, int64_t k_c) {
  for (int64_t j = 0; j < n; j += b) {
    int64_t w = n - j < b ? n - j : b;
    double *panel = &A_(a, ld, j, j);
    int64_t *pv = ipiv + j;
    if (inner_b > 0 && inner_b < w) {
      orc_lu_blk_rl(panel, m - j, w, ld, inner_b, 0, pv, singular, k_c);
    } else {
      if (orc_unb_pivoted(panel, m - j, w, ld, pv)) *singular = 1;
    }
    orc_laswp(&A_(a, ld, j, 0), m - j, j, ld, pv, w, 0);
    orc_laswp(&A_(a, ld, j, j + w), m - j, n - j - w, ld, pv, w, 0);
    for (int64_t t = 0; t < w; ++t) pv[t] += j;
    orc_trsm_llu(panel, w, ld, &A_(a, ld, j, j + w), n - j - w, ld);
    orc_gemm(&A_(a, ld, j + w, j + w), m - j - w, n - j - w, ld, &A_(a, ld, j + w, j), ld,
             &A_(a, ld, j, j + w), ld, w, 1.0, -1.0, k_c);
  }
}

/* reference lu.py:197-334 (lu_la): the look-ahead driver.  lu / lu_la / lu_ws_static / lu_mb
 * perform identical arithmetic on identical values (lu.py:201-204; test_lu.py:198-212), so one
 * serial schedule restates all four; the PF/RU column split changes no bit.
 *
 * Early termination (lu_et) is timing-dependent in the reference; to make it checkable the
 * schedule is an input: et_sched[it] (it = 1.. in loop order, may be NULL / shorter than the run)
 * gives the poll number at which ru_done is seen set inside iteration it's panel (0 = never), i.e.
 * the panel is cut after et_sched[it] inner blocks.  Bookkeeping follows lu.py:314-326: cut ->
 * b_target = max(b_i, k_new); otherwise b_target = min(b_o, 2*b_target); pend remembers which
 * columns already carry the swaps.  widths_out (optional, capacity widths_cap) receives every
 * panel's factored width in order (prologue first); *n_widths the count.
 * ipiv is global, 0-based (lu.py:236, 317).  Returns the number of ET events. */
int64_t orc_lu_la_clamped(double *a, int64_t m, int64_t n, int64_t ld, int64_t b_o, int64_t b_i,
                          int64_t *ipiv, const int64_t *et_sched, int64_t n_sched, int *singular,
                          int64_t *widths_out, int64_t widths_cap, int64_t *n_widths, int64_t k_c,
                          int64_t clamp);

int64_t orc_lu_la(double *a, int64_t m, int64_t n, int64_t ld, int64_t b_o, int64_t b_i,
                  int64_t *ipiv, const int64_t *et_sched, int64_t n_sched, int *singular,
                  int64_t *widths_out, int64_t widths_cap, int64_t *n_widths, int64_t k_c) {
  return orc_lu_la_clamped(a, m, n, ld, b_o, b_i, ipiv, et_sched, n_sched, singular, widths_out,
                           widths_cap, n_widths, k_c, 0);
}

/* clamp > 0: the panel schedule of the 1-D block-cyclic multi-GPU layout (this spec's design, SURVEY.md
 * 8e; the reference has no multi-device path): a panel never crosses a multiple of `clamp` columns
 * (the column block = the unit of ownership), everything else -- operators, order, ET bookkeeping -- is
 * lu.py:224-332 unchanged.  clamp == 0 is the reference's schedule. */
int64_t orc_lu_la_clamped(double *a, int64_t m, int64_t n, int64_t ld, int64_t b_o, int64_t b_i,
                          int64_t *ipiv, const int64_t *et_sched, int64_t n_sched, int *singular,
                          int64_t *widths_out, int64_t widths_cap, int64_t *n_widths, int64_t k_c,
                          int64_t clamp) {
  int64_t et_events = 0, nw = 0;
  *singular = 0;
  if (n_widths) *n_widths = 0;
  if (n == 0) return 0;
  int64_t *piv_local = (int64_t *)malloc(sizeof(int64_t) * (size_t)(b_o > 0 ? b_o : 1));
  int64_t w0 = b_o < n ? b_o : n;
  if (clamp > 0 && w0 > clamp) w0 = clamp;
  orc_lu_blk_ll(a, m, w0, ld, b_i, piv_local, 0, singular, k_c);
  for (int64_t t = 0; t < w0; ++t) ipiv[t] = piv_local[t];
  if (widths_out && nw < widths_cap) widths_out[nw] = w0;
  ++nw;
  int64_t q0 = 0, q1 = w0, pend = w0, b_target = b_o, npiv_prev = w0, it = 0;
  while (q1 < n) {
    ++it;
    int64_t w = b_target < n - q1 ? b_target : n - q1;
    if (clamp > 0 && w > clamp - q1 % clamp) w = clamp - q1 % clamp;
    /* sync_task, lu.py:251-255 */
    orc_laswp(&A_(a, ld, q0, 0), m - q0, q0, ld, piv_local, npiv_prev, 0);
    orc_laswp(&A_(a, ld, q0, pend), m - q0, n - pend, ld, piv_local, npiv_prev, 0);
    /* whole_task, lu.py:260-267 (== PF1+RU1, PF2+RU2, PF3 of 279-310) */
    orc_trsm_llu(&A_(a, ld, q0, q0), q1 - q0, ld, &A_(a, ld, q0, q1), n - q1, ld);
    orc_gemm(&A_(a, ld, q1, q1), m - q1, n - q1, ld, &A_(a, ld, q1, q0), ld, &A_(a, ld, q0, q1),
             ld, q1 - q0, 1.0, -1.0, k_c);
    int64_t trip = (et_sched && it - 1 < n_sched) ? et_sched[it - 1] : 0;
    int64_t k_new = orc_lu_blk_ll(&A_(a, ld, q1, q1), m - q1, w, ld, b_i, piv_local, trip, singular,
                                  k_c);
    for (int64_t t = 0; t < k_new; ++t) ipiv[q1 + t] = q1 + piv_local[t];
    if (widths_out && nw < widths_cap) widths_out[nw] = k_new;
    ++nw;
    if (k_new < w) {
      ++et_events;
      b_target = b_i > k_new ? b_i : k_new;
    } else {
      b_target = b_o < 2 * b_target ? b_o : 2 * b_target;
    }
    npiv_prev = k_new;
    pend = q1 + w;
    q0 = q1;
    q1 = q1 + k_new;
  }
  /* final_sync, lu.py:329-332 */
  orc_laswp(&A_(a, ld, q0, 0), m - q0, q0, ld, piv_local, npiv_prev, 0);
  free(piv_local);
  if (n_widths) *n_widths = nw;
  return et_events;
}

/* reference matrix.py:95-131 (swap_rows/split_lu/residual_lu): ||P A - L U||_F / ||A||_F from the
 * packed factors; L is m x n unit-lower, U is n x n upper.  Straight triple loop in blocks,
 * long-double free; this is a checker, order of summation is not part of the contract (the
 * reference uses numpy matmul + np.linalg.norm here). */
double orc_residual_lu(const double *a_orig, const double *lu, int64_t m, int64_t n, int64_t ld_a,
                       int64_t ld_lu, const int64_t *ipiv) {
  int64_t *rowmap = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
  for (int64_t i = 0; i < m; ++i) rowmap[i] = i;
  for (int64_t k = 0; k < n; ++k) {
    int64_t p = ipiv[k];
    int64_t t = rowmap[k]; rowmap[k] = rowmap[p]; rowmap[p] = t;
  }
  double num = 0.0, den = 0.0;
#pragma omp parallel for schedule(dynamic, 8) reduction(+ : num, den)
  for (int64_t j = 0; j < n; ++j) {
    double *col = (double *)malloc(sizeof(double) * (size_t)m);
    for (int64_t i = 0; i < m; ++i) col[i] = 0.0;
    /* column j of L*U = sum_{p<=j} L[:,p] * U[p,j] */
    for (int64_t p = 0; p <= j && p < n; ++p) {
      double u = A_(lu, ld_lu, p, j);
      col[p] += u; /* unit diagonal of L */
      for (int64_t i = p + 1; i < m; ++i) col[i] += A_(lu, ld_lu, i, p) * u;
    }
    for (int64_t i = 0; i < m; ++i) {
      double pa = A_(a_orig, ld_a, rowmap[i], j);
      double r = pa - col[i];
      num += r * r;
      den += pa * pa;
    }
    free(col);
  }
  free(rowmap);
  if (den == 0.0) return sqrt(num);
  return sqrt(num) / sqrt(den);
}
