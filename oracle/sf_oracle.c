/* sf_oracle.c -- plain-C restatement of the Sparse Fusion reference path.
 *
 * TEST INFRASTRUCTURE ONLY (see sf_oracle.h): the checker, never the product.
 * Compiled with -ffp-contract=off so every `acc -= v * x` is a separate
 * multiply and subtract, exactly as the reference's ISO C++20 build
 * (-std=c++20 turns GCC's default contraction off; proj/CMakeLists.txt:1-8).
 *
 * Each function cites the reference code it restates.
 */
#include "sf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 + std::uniform_real_distribution<double>(-1, 1) as        */
/* libstdc++ evaluates them (fixtures.hpp:148-155).                          */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64_t;

static void mt64_seed(mt64_t* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) +
               (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64_t* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (s->mt[i] & 0xFFFFFFFF80000000ULL) |
                         (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = s->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL)
        v ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = v;
    }
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* std::generate_canonical<double, 53>: one 64-bit draw divided by 2^64,
 * clamped below 1. */
static double mt64_canonical(mt64_t* s) {
  const double sum = (double)mt64_next(s);
  double r = sum / 18446744073709551616.0;
  if (r >= 1.0)
    r = nextafter(1.0, 0.0);
  return r;
}

void orc_gen_vector(int32_t n, uint64_t seed, double* out) {
  mt64_t s;
  mt64_seed(&s, seed);
  for (int32_t i = 0; i < n; ++i)
    out[i] = mt64_canonical(&s) * (1.0 - (-1.0)) + (-1.0);
}

/* ------------------------------------------------------------------------ */
/* Compressed storage helpers (matrix.hpp:18-173).                           */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t nrows, ncols; /* for CSR: ptr over rows; for CSC: ptr over cols */
  int32_t* ptr;
  int32_t* idx;
  double* val;
  int owns;
} smat;

static void smat_free(smat* m) {
  if (m->owns) {
    free(m->ptr);
    free(m->idx);
    free(m->val);
  }
  memset(m, 0, sizeof(*m));
}

/* to_csr (matrix.hpp:66-86): the CSC matrix `a` (ptr over a->ncols columns)
 * becomes CSR (ptr over a->nrows rows), column order ascending per row. */
static void to_csr(const smat* a, smat* r) {
  const int32_t nnz = a->ptr[a->ncols];
  r->nrows = a->nrows;
  r->ncols = a->ncols;
  r->ptr = (int32_t*)calloc((size_t)a->nrows + 1, sizeof(int32_t));
  r->idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz ? nnz : 1));
  r->val = (double*)malloc(sizeof(double) * (size_t)(nnz ? nnz : 1));
  r->owns = 1;
  for (int32_t p = 0; p < nnz; ++p)
    ++r->ptr[a->idx[p] + 1];
  for (int32_t i = 0; i < a->nrows; ++i)
    r->ptr[i + 1] += r->ptr[i];
  int32_t* next = (int32_t*)malloc(sizeof(int32_t) * ((size_t)a->nrows + 1));
  memcpy(next, r->ptr, sizeof(int32_t) * (size_t)a->nrows);
  for (int32_t j = 0; j < a->ncols; ++j)
    for (int32_t p = a->ptr[j]; p < a->ptr[j + 1]; ++p) {
      const int32_t q = next[a->idx[p]]++;
      r->idx[q] = j;
      r->val[q] = a->val[p];
    }
  free(next);
}

/* lower_triangle (matrix.hpp:98-128). Returns 0 or sets *bad_col. */
static int lower_triangle(const smat* a, smat* l, int32_t* bad_col) {
  const int32_t n = a->ncols;
  const int32_t nnz = a->ptr[n];
  l->nrows = l->ncols = n;
  l->ptr = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  l->idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz ? nnz : 1));
  l->val = (double*)malloc(sizeof(double) * (size_t)(nnz ? nnz : 1));
  l->owns = 1;
  int32_t q = 0;
  for (int32_t j = 0; j < n; ++j) {
    int diag = 0;
    for (int32_t p = a->ptr[j]; p < a->ptr[j + 1]; ++p) {
      const int32_t i = a->idx[p];
      if (i < j)
        continue;
      if (i == j) {
        if (a->val[p] == 0.0) {
          *bad_col = j;
          return ORC_ERR_INVALID_MATRIX;
        }
        diag = 1;
      }
      l->idx[q] = i;
      l->val[q] = a->val[p];
      ++q;
    }
    if (!diag) {
      *bad_col = j;
      return ORC_ERR_INVALID_MATRIX;
    }
    l->ptr[j + 1] = q;
  }
  return ORC_OK;
}

/* LowerRowView / build_lower_rows (kernels.hpp:86-115). */
typedef struct {
  int32_t* ptr;
  int32_t* col;
  int32_t* pos;
} rowview;

static int build_lower_rows(const smat* l, rowview* rv, int32_t* bad) {
  const int32_t n = l->ncols;
  rv->ptr = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  for (int32_t j = 0; j < n; ++j) {
    if (l->ptr[j] == l->ptr[j + 1] || l->idx[l->ptr[j]] != j) {
      *bad = j;
      return ORC_ERR_INVALID_MATRIX;
    }
    for (int32_t p = l->ptr[j] + 1; p < l->ptr[j + 1]; ++p)
      ++rv->ptr[l->idx[p] + 1];
  }
  for (int32_t i = 0; i < n; ++i)
    rv->ptr[i + 1] += rv->ptr[i];
  const int32_t m = rv->ptr[n];
  rv->col = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
  rv->pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
  int32_t* next = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  memcpy(next, rv->ptr, sizeof(int32_t) * (size_t)n);
  for (int32_t j = 0; j < n; ++j)
    for (int32_t p = l->ptr[j] + 1; p < l->ptr[j + 1]; ++p) {
      const int32_t q = next[l->idx[p]]++;
      rv->col[q] = j;
      rv->pos[q] = p;
    }
  free(next);
  return ORC_OK;
}

static void rowview_free(rowview* rv) {
  free(rv->ptr);
  free(rv->col);
  free(rv->pos);
  memset(rv, 0, sizeof(*rv));
}

/* find_diag_positions (kernels.hpp:288-297) on CSR. */
static int32_t* find_diag_positions(const smat* a) {
  int32_t* d = (int32_t*)malloc(sizeof(int32_t) * ((size_t)a->nrows + 1));
  for (int32_t i = 0; i < a->nrows; ++i) {
    d[i] = -1;
    for (int32_t p = a->ptr[i]; p < a->ptr[i + 1]; ++p)
      if (a->idx[p] == i) {
        d[i] = p;
        break;
      }
  }
  return d;
}

/* ------------------------------------------------------------------------ */
/* KernelState (kernels.hpp:409-495).                                        */
/* ------------------------------------------------------------------------ */
typedef struct {
  int combo;
  int32_t n;
  smat M;     /* borrowed CSC input */
  smat L_csr; /* combos 1, 2, 4, 8 */
  smat A_csr; /* combos 2, 3, 6 */
  smat L_csc; /* combos 5, 7, 8 */
  rowview rv; /* combos 5, 7 */
  int32_t* diag_pos;
  double* fac; /* combos 3, 5, 6, 7 */
  int64_t nfac;
  double *vin, *vmid, *vout, *dvec;
  /* IterScratch (kernels.hpp:118-139) */
  double* acc;
  int32_t* mark;
  int32_t* slot;
  int32_t stamp;
} ostate;

static void state_free(ostate* st) {
  smat_free(&st->L_csr);
  smat_free(&st->A_csr);
  smat_free(&st->L_csc);
  rowview_free(&st->rv);
  free(st->diag_pos);
  free(st->fac);
  free(st->vin);
  free(st->vmid);
  free(st->vout);
  free(st->dvec);
  free(st->acc);
  free(st->mark);
  free(st->slot);
  memset(st, 0, sizeof(*st));
}

static double* dalloc0(int64_t n) {
  return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
}

static int make_state(ostate* st, int combo, int32_t n, const int32_t* colptr,
                      const int32_t* rowidx, const double* values,
                      uint64_t seed, const double* vin, int32_t* err_index) {
  memset(st, 0, sizeof(*st));
  st->combo = combo;
  st->n = n;
  st->M.nrows = st->M.ncols = n;
  st->M.ptr = (int32_t*)colptr;
  st->M.idx = (int32_t*)rowidx;
  st->M.val = (double*)values;
  int rc = ORC_OK;
  smat low = {0};
  switch (combo) {
  case 1:
  case 4:
  case 8:
    rc = lower_triangle(&st->M, &low, err_index);
    if (rc)
      break;
    to_csr(&low, &st->L_csr);
    if (combo == 8)
      st->L_csc = low; /* backward solve reads the columns of L */
    else
      smat_free(&low);
    break;
  case 2:
    to_csr(&st->M, &st->A_csr);
    rc = lower_triangle(&st->M, &low, err_index);
    if (rc)
      break;
    to_csr(&low, &st->L_csr);
    smat_free(&low);
    break;
  case 3:
  case 6:
    to_csr(&st->M, &st->A_csr);
    st->diag_pos = find_diag_positions(&st->A_csr);
    st->nfac = st->A_csr.ptr[n];
    st->fac = dalloc0(st->nfac);
    memcpy(st->fac, st->A_csr.val, sizeof(double) * (size_t)st->nfac);
    if (combo == 3) {
      /* scaling_vector (kernels.hpp:299-309) */
      st->dvec = dalloc0(n);
      for (int32_t i = 0; i < n; ++i) {
        const double a =
            st->diag_pos[i] >= 0 ? st->A_csr.val[st->diag_pos[i]] : 0.0;
        if (a == 0.0) {
          *err_index = i;
          return ORC_ERR_ZERO_DIAG_SCALE;
        }
        st->dvec[i] = 1.0 / sqrt(fabs(a));
      }
    }
    break;
  case 5:
  case 7:
    rc = lower_triangle(&st->M, &st->L_csc, err_index);
    if (rc)
      break;
    rc = build_lower_rows(&st->L_csc, &st->rv, err_index);
    if (rc)
      break;
    st->nfac = st->L_csc.ptr[n];
    st->fac = dalloc0(st->nfac);
    memcpy(st->fac, st->L_csc.val, sizeof(double) * (size_t)st->nfac);
    if (combo == 7) {
      st->dvec = dalloc0(n);
      for (int32_t j = 0; j < n; ++j)
        st->dvec[j] = 1.0 / sqrt(fabs(st->L_csc.val[st->L_csc.ptr[j]]));
    }
    break;
  default:
    return ORC_ERR_BAD_ARG;
  }
  if (rc)
    return rc;
  if (combo != 3 && combo != 7) {
    st->vin = dalloc0(n);
    if (vin)
      memcpy(st->vin, vin, sizeof(double) * (size_t)n);
    else
      orc_gen_vector(n, seed, st->vin);
    st->vout = dalloc0(n);
    if (combo == 1 || combo == 2 || combo == 4 || combo == 8)
      st->vmid = dalloc0(n);
  }
  st->acc = dalloc0(n);
  st->mark = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  st->slot = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  st->stamp = 0;
  return ORC_OK;
}

static int32_t next_stamp(ostate* st) {
  if (++st->stamp == 0) {
    memset(st->mark, 0, sizeof(int32_t) * (size_t)st->n);
    st->stamp = 1;
  }
  return st->stamp;
}

/* ------------------------------------------------------------------------ */
/* Per-iteration bodies (kernels.hpp:145-286).                               */
/* ------------------------------------------------------------------------ */

/* spmv_csr_row (kernels.hpp:152-158) */
static void spmv_csr_row(int32_t i, const smat* a, const double* x, double* y) {
  double acc = 0.0;
  for (int32_t p = a->ptr[i]; p < a->ptr[i + 1]; ++p)
    acc += a->val[p] * x[a->idx[p]];
  y[i] = acc;
}

/* spmv_csc_col (kernels.hpp:162-168) */
static void spmv_csc_col(int32_t j, const smat* a, const double* x, double* y) {
  const double xj = x[j];
  for (int32_t p = a->ptr[j]; p < a->ptr[j + 1]; ++p)
    y[a->idx[p]] += a->val[p] * xj;
}

/* trsv_csr_row (kernels.hpp:171-181): diagonal stored last. */
static int trsv_csr_row(int32_t i, const smat* l, const double* vals,
                        const double* rhs, double* x, int32_t* ei) {
  const int32_t end = l->ptr[i + 1] - 1;
  double acc = rhs[i];
  for (int32_t p = l->ptr[i]; p < end; ++p)
    acc -= vals[p] * x[l->idx[p]];
  const double d = vals[end];
  if (d == 0.0) {
    *ei = i;
    return ORC_ERR_ZERO_DIAG_SOLVE;
  }
  x[i] = acc / d;
  return ORC_OK;
}

/* trsv_csr_unit_row (kernels.hpp:184-196) */
static void trsv_csr_unit_row(int32_t i, const smat* a, const int32_t* diag_pos,
                              const double* fac, const double* rhs, double* x) {
  double acc = rhs[i];
  const int32_t end = diag_pos[i] >= 0 ? diag_pos[i] : a->ptr[i + 1];
  for (int32_t p = a->ptr[i]; p < end; ++p) {
    if (a->idx[p] >= i)
      break;
    acc -= fac[p] * x[a->idx[p]];
  }
  x[i] = acc;
}

/* trsv_csc_row (kernels.hpp:200-210) */
static int trsv_csc_row(int32_t i, const smat* l, const rowview* rv,
                        const double* fac, const double* rhs, double* x,
                        int32_t* ei) {
  double acc = rhs[i];
  for (int32_t q = rv->ptr[i]; q < rv->ptr[i + 1]; ++q)
    acc -= fac[rv->pos[q]] * x[rv->col[q]];
  const double d = fac[l->ptr[i]];
  if (d == 0.0) {
    *ei = i;
    return ORC_ERR_ZERO_DIAG_SOLVE;
  }
  x[i] = acc / d;
  return ORC_OK;
}

/* Backward L^T solve for combo 8 (not in the reference):
 * sptrsv(to_csr(permute_symmetric(transpose(L), rev))) row n-1-i visits
 * L(j, i) for j descending from the bottom of column i, diagonal last. */
static int trsv_lt_row(int32_t i, const smat* lcsc, const double* rhs,
                       double* x, int32_t* ei) {
  const int32_t beg = lcsc->ptr[i];
  double acc = rhs[i];
  for (int32_t p = lcsc->ptr[i + 1] - 1; p > beg; --p)
    acc -= lcsc->val[p] * x[lcsc->idx[p]];
  const double d = lcsc->val[beg];
  if (d == 0.0) {
    *ei = i;
    return ORC_ERR_ZERO_DIAG_SOLVE;
  }
  x[i] = acc / d;
  return ORC_OK;
}

static int32_t lower_bound_i32(const int32_t* first, const int32_t* last,
                               int32_t key) {
  const int32_t* lo = first;
  int64_t count = last - first;
  while (count > 0) {
    const int64_t step = count / 2;
    const int32_t* it = lo + step;
    if (*it < key) {
      lo = it + 1;
      count -= step + 1;
    } else {
      count = step;
    }
  }
  return (int32_t)(lo - first);
}

/* ic0_column (kernels.hpp:214-242) */
static int ic0_column(int32_t k, ostate* st, double* fac, int32_t* ei) {
  const smat* l = &st->L_csc;
  const rowview* rv = &st->rv;
  const int32_t stamp = next_stamp(st);
  for (int32_t p = l->ptr[k]; p < l->ptr[k + 1]; ++p) {
    const int32_t i = l->idx[p];
    st->mark[i] = stamp;
    st->acc[i] = fac[p];
  }
  for (int32_t q = rv->ptr[k]; q < rv->ptr[k + 1]; ++q) {
    const int32_t j = rv->col[q];
    const double lkj = fac[rv->pos[q]];
    const int32_t b = l->ptr[j];
    const int32_t e = l->ptr[j + 1];
    const int32_t it = b + lower_bound_i32(l->idx + b, l->idx + e, k);
    for (int32_t p = it; p < e; ++p) {
      const int32_t i = l->idx[p];
      if (st->mark[i] == stamp)
        st->acc[i] -= lkj * fac[p];
    }
  }
  const double d = st->acc[k];
  if (d <= 0.0) {
    *ei = k;
    return ORC_ERR_NONPOS_PIVOT;
  }
  const double lkk = sqrt(d);
  fac[l->ptr[k]] = lkk;
  for (int32_t p = l->ptr[k] + 1; p < l->ptr[k + 1]; ++p)
    fac[p] = st->acc[l->idx[p]] / lkk;
  return ORC_OK;
}

/* ilu0_row (kernels.hpp:246-272) */
static int ilu0_row(int32_t i, ostate* st, double* fac, int32_t* ei) {
  const smat* a = &st->A_csr;
  const int32_t* diag_pos = st->diag_pos;
  const int32_t stamp = next_stamp(st);
  for (int32_t p = a->ptr[i]; p < a->ptr[i + 1]; ++p) {
    const int32_t j = a->idx[p];
    st->mark[j] = stamp;
    st->slot[j] = p;
    st->acc[j] = fac[p];
  }
  for (int32_t p = a->ptr[i]; p < a->ptr[i + 1]; ++p) {
    const int32_t k = a->idx[p];
    if (k >= i)
      break;
    if (diag_pos[k] < 0 || fac[diag_pos[k]] == 0.0) {
      *ei = k;
      return ORC_ERR_ZERO_PIVOT;
    }
    const double lik = st->acc[k] / fac[diag_pos[k]];
    st->acc[k] = lik;
    for (int32_t q = diag_pos[k] + 1; q < a->ptr[k + 1]; ++q) {
      const int32_t j = a->idx[q];
      if (st->mark[j] == stamp)
        st->acc[j] -= lik * fac[q];
    }
  }
  for (int32_t p = a->ptr[i]; p < a->ptr[i + 1]; ++p)
    fac[p] = st->acc[a->idx[p]];
  return ORC_OK;
}

/* dscal_csr_row (kernels.hpp:274-279): (d_i * a) * d_j */
static void dscal_csr_row(int32_t i, const smat* a, const double* d,
                          double* fac) {
  const double di = d[i];
  for (int32_t p = a->ptr[i]; p < a->ptr[i + 1]; ++p)
    fac[p] = di * fac[p] * d[a->idx[p]];
}

/* dscal_csc_col (kernels.hpp:281-286): (d_i * a) * d_j */
static void dscal_csc_col(int32_t j, const smat* a, const double* d,
                          double* fac) {
  const double dj = d[j];
  for (int32_t p = a->ptr[j]; p < a->ptr[j + 1]; ++p)
    fac[p] = d[a->idx[p]] * fac[p] * dj;
}

/* run_iteration (kernels.hpp:508-570); combo 8 kernel 2 = backward L^T. */
static int run_iteration(int which, int32_t i, ostate* st, int32_t* ei) {
  switch (st->combo) {
  case 1:
    if (which == 1)
      return trsv_csr_row(i, &st->L_csr, st->L_csr.val, st->vin, st->vmid, ei);
    return trsv_csr_row(i, &st->L_csr, st->L_csr.val, st->vmid, st->vout, ei);
  case 2:
    if (which == 1) {
      spmv_csr_row(i, &st->A_csr, st->vin, st->vmid);
      return ORC_OK;
    }
    return trsv_csr_row(i, &st->L_csr, st->L_csr.val, st->vmid, st->vout, ei);
  case 3:
    if (which == 1) {
      dscal_csr_row(i, &st->A_csr, st->dvec, st->fac);
      return ORC_OK;
    }
    return ilu0_row(i, st, st->fac, ei);
  case 4:
    if (which == 1)
      return trsv_csr_row(i, &st->L_csr, st->L_csr.val, st->vin, st->vmid, ei);
    spmv_csc_col(i, &st->M, st->vmid, st->vout);
    return ORC_OK;
  case 5:
    if (which == 1)
      return ic0_column(i, st, st->fac, ei);
    return trsv_csc_row(i, &st->L_csc, &st->rv, st->fac, st->vin, st->vout, ei);
  case 6:
    if (which == 1)
      return ilu0_row(i, st, st->fac, ei);
    trsv_csr_unit_row(i, &st->A_csr, st->diag_pos, st->fac, st->vin,
                      st->vout);
    return ORC_OK;
  case 7:
    if (which == 1) {
      dscal_csc_col(i, &st->L_csc, st->dvec, st->fac);
      return ORC_OK;
    }
    return ic0_column(i, st, st->fac, ei);
  case 8:
    if (which == 1)
      return trsv_csr_row(i, &st->L_csr, st->L_csr.val, st->vin, st->vmid, ei);
    /* backward iterations run in descending original row order */
    {
      const int32_t row = st->n - 1 - i;
      return trsv_lt_row(row, &st->L_csc, st->vmid, st->vout, ei);
    }
  default:
    return ORC_ERR_BAD_ARG;
  }
}

static int64_t output_len_state(const ostate* st) {
  switch (st->combo) {
  case 1:
  case 2:
  case 4:
  case 8:
    return 2 * (int64_t)st->n;
  case 3:
  case 5:
  case 6:
  case 7:
    return st->nfac + st->n;
  default:
    return -1;
  }
}

int64_t orc_output_len(int combo, int32_t n, const int32_t* colptr,
                       const int32_t* rowidx) {
  switch (combo) {
  case 1:
  case 2:
  case 4:
  case 8:
    return 2 * (int64_t)n;
  case 3:
  case 6:
    return (int64_t)colptr[n] + n;
  case 5:
  case 7: {
    int64_t low = 0;
    for (int32_t j = 0; j < n; ++j)
      for (int32_t p = colptr[j]; p < colptr[j + 1]; ++p)
        if (rowidx[p] >= j)
          ++low;
    return low + n;
  }
  default:
    return -1;
  }
}

/* collect_outputs (kernels.hpp:585-608) */
static void collect_outputs(const ostate* st, double* out) {
  const int32_t n = st->n;
  switch (st->combo) {
  case 1:
  case 2:
  case 4:
  case 8:
    memcpy(out, st->vmid, sizeof(double) * (size_t)n);
    memcpy(out + n, st->vout, sizeof(double) * (size_t)n);
    break;
  case 3:
  case 7:
    memcpy(out, st->fac, sizeof(double) * (size_t)st->nfac);
    memcpy(out + st->nfac, st->dvec, sizeof(double) * (size_t)n);
    break;
  case 5:
  case 6:
    memcpy(out, st->fac, sizeof(double) * (size_t)st->nfac);
    memcpy(out + st->nfac, st->vout, sizeof(double) * (size_t)n);
    break;
  default:
    break;
  }
}

int64_t orc_run_sequential(int combo, int32_t n, const int32_t* colptr,
                           const int32_t* rowidx, const double* values,
                           uint64_t seed, const double* vin, double* out,
                           int64_t out_cap, int32_t* err_code,
                           int32_t* err_index) {
  *err_code = ORC_OK;
  *err_index = -1;
  ostate st;
  int rc = make_state(&st, combo, n, colptr, rowidx, values, seed, vin,
                      err_index);
  if (rc) {
    *err_code = rc;
    state_free(&st);
    return -1;
  }
  /* run_sequential_reference (kernels.hpp:574-582) */
  for (int which = 1; which <= 2 && rc == ORC_OK; ++which)
    for (int32_t i = 0; i < n; ++i) {
      rc = run_iteration(which, i, &st, err_index);
      if (rc)
        break;
    }
  if (rc) {
    *err_code = rc;
    state_free(&st);
    return -1;
  }
  const int64_t len = output_len_state(&st);
  if (len > out_cap) {
    *err_code = ORC_ERR_BAD_ARG;
    state_free(&st);
    return -1;
  }
  collect_outputs(&st, out);
  state_free(&st);
  return len;
}

/* ------------------------------------------------------------------------ */
/* Inspector structures (dag.hpp).                                           */
/* ------------------------------------------------------------------------ */

/* make_dag (dag.hpp:52-69): edges sorted by (u, v) and made unique. The
 * edges are bucketed by u (counting sort), then each bucket is sorted. */
static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

static void make_dag(int32_t nvert, int64_t ne, const int32_t* us,
                     const int32_t* vs, int64_t* cost, orc_dag* g) {
  g->nvert = nvert;
  g->succptr = (int32_t*)calloc((size_t)nvert + 1, sizeof(int32_t));
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ne ? ne : 1));
  int64_t* cnt = (int64_t*)calloc((size_t)nvert + 1, sizeof(int64_t));
  for (int64_t e = 0; e < ne; ++e)
    ++cnt[us[e] + 1];
  for (int32_t u = 0; u < nvert; ++u)
    cnt[u + 1] += cnt[u];
  int64_t* next = (int64_t*)malloc(sizeof(int64_t) * ((size_t)nvert + 1));
  memcpy(next, cnt, sizeof(int64_t) * ((size_t)nvert + 1));
  for (int64_t e = 0; e < ne; ++e)
    tmp[next[us[e]]++] = vs[e];
  free(next);
  int64_t w = 0;
  for (int32_t u = 0; u < nvert; ++u) {
    const int64_t b = cnt[u], e = cnt[u + 1];
    qsort(tmp + b, (size_t)(e - b), sizeof(int32_t), cmp_i32);
    for (int64_t p = b; p < e; ++p)
      if (p == b || tmp[p] != tmp[p - 1])
        tmp[w++] = tmp[p];
    g->succptr[u + 1] = (int32_t)w;
  }
  free(cnt);
  g->nedges = w;
  g->succ = tmp;
  g->cost = cost;
}

static int64_t* cost_alloc(int32_t n) {
  return (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
}

static int64_t max1(int64_t c) { return c > 1 ? c : 1; }

/* vertex_costs, CSR kinds (dag.hpp:82-110) */
static int64_t* costs_csr(int kind, const smat* a) {
  const int32_t n = a->nrows;
  int64_t* c = cost_alloc(n);
  if (kind == 0) { /* SpMV_CSR, SpTRSV_CSR, DSCAL_CSR */
    for (int32_t i = 0; i < n; ++i)
      c[i] = max1(a->ptr[i + 1] - a->ptr[i]);
  } else { /* SpILU0_CSR */
    int32_t* diag = find_diag_positions(a);
    for (int32_t i = 0; i < n; ++i) {
      int64_t t = a->ptr[i + 1] - a->ptr[i];
      for (int32_t p = a->ptr[i]; p < a->ptr[i + 1]; ++p) {
        const int32_t k = a->idx[p];
        if (k >= i)
          break;
        if (diag[k] >= 0)
          t += a->ptr[k + 1] - diag[k] - 1;
      }
      c[i] = max1(t);
    }
    free(diag);
  }
  return c;
}

/* vertex_costs, CSC kinds (dag.hpp:112-145) */
static int64_t* costs_csc(int kind, const smat* a, const rowview* rv) {
  const int32_t n = a->ncols;
  int64_t* c = cost_alloc(n);
  if (kind == 0) { /* SpMV_CSC, DSCAL_CSC */
    for (int32_t j = 0; j < n; ++j)
      c[j] = max1(a->ptr[j + 1] - a->ptr[j]);
  } else if (kind == 1) { /* SpTRSV_CSC */
    for (int32_t i = 0; i < n; ++i)
      c[i] = 1 + rv->ptr[i + 1] - rv->ptr[i];
  } else { /* SpIC0_CSC */
    for (int32_t k = 0; k < n; ++k) {
      int64_t t = a->ptr[k + 1] - a->ptr[k];
      for (int32_t q = rv->ptr[k]; q < rv->ptr[k + 1]; ++q) {
        const int32_t j = rv->col[q];
        const int32_t b = a->ptr[j], e = a->ptr[j + 1];
        t += (e - b) - lower_bound_i32(a->idx + b, a->idx + e, k);
      }
      c[k] = max1(t);
    }
  }
  return c;
}

/* intra_dag on CSR for SpTRSV/SpILU0 (dag.hpp:155-167). */
static void intra_dag_csr_solve(const smat* a, int64_t* cost, orc_dag* g) {
  const int32_t n = a->nrows;
  const int64_t cap = a->ptr[n];
  int32_t* us = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap ? cap : 1));
  int32_t* vs = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap ? cap : 1));
  int64_t ne = 0;
  for (int32_t i = 0; i < n; ++i)
    for (int32_t p = a->ptr[i]; p < a->ptr[i + 1]; ++p) {
      const int32_t j = a->idx[p];
      if (j < i) {
        us[ne] = j;
        vs[ne] = i;
        ++ne;
      } else {
        break;
      }
    }
  make_dag(n, ne, us, vs, cost, g);
  free(us);
  free(vs);
}

/* intra_dag on CSC for SpTRSV_CSC / SpIC0_CSC (dag.hpp:178-188). */
static void intra_dag_csc_solve(const smat* a, int64_t* cost, orc_dag* g) {
  const int32_t n = a->ncols;
  const int64_t cap = a->ptr[n];
  int32_t* us = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap ? cap : 1));
  int32_t* vs = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap ? cap : 1));
  int64_t ne = 0;
  for (int32_t j = 0; j < n; ++j)
    for (int32_t p = a->ptr[j]; p < a->ptr[j + 1]; ++p) {
      const int32_t i = a->idx[p];
      if (i > j) {
        us[ne] = j;
        vs[ne] = i;
        ++ne;
      }
    }
  make_dag(n, ne, us, vs, cost, g);
  free(us);
  free(vs);
}

static void edgeless(int32_t n, int64_t* cost, orc_dag* g) {
  make_dag(n, 0, NULL, NULL, cost, g);
}

int orc_build_g(int combo, int which, int32_t n, const int32_t* colptr,
                const int32_t* rowidx, const double* values, orc_dag* out) {
  memset(out, 0, sizeof(*out));
  ostate st;
  int32_t ei = -1;
  int rc = make_state(&st, combo, n, colptr, rowidx, values, 7, NULL, &ei);
  if (rc && rc != ORC_ERR_ZERO_DIAG_SCALE) {
    state_free(&st);
    return rc;
  }
  if (which == 1) { /* build_g1 (dag.hpp:319-337) */
    switch (combo) {
    case 1:
    case 4:
    case 8:
      intra_dag_csr_solve(&st.L_csr, costs_csr(0, &st.L_csr), out);
      break;
    case 2:
    case 3:
      edgeless(n, costs_csr(0, &st.A_csr), out);
      break;
    case 5: {
      intra_dag_csc_solve(&st.L_csc, costs_csc(2, &st.L_csc, &st.rv), out);
      break;
    }
    case 6:
      intra_dag_csr_solve(&st.A_csr, costs_csr(1, &st.A_csr), out);
      break;
    case 7:
      edgeless(n, costs_csc(0, &st.L_csc, &st.rv), out);
      break;
    default:
      rc = ORC_ERR_BAD_ARG;
    }
  } else { /* build_g2 (dag.hpp:339-370) */
    switch (combo) {
    case 1:
    case 2:
      intra_dag_csr_solve(&st.L_csr, costs_csr(0, &st.L_csr), out);
      break;
    case 3:
      intra_dag_csr_solve(&st.A_csr, costs_csr(1, &st.A_csr), out);
      break;
    case 4:
      edgeless(n, costs_csc(0, &st.M, NULL), out);
      break;
    case 5:
      intra_dag_csc_solve(&st.L_csc, costs_csc(1, &st.L_csc, &st.rv), out);
      break;
    case 6: {
      /* dag.hpp:350-364: strictly-lower edges, cost = 1 + strictly-lower nnz */
      const smat* a = &st.A_csr;
      int64_t* cost = cost_alloc(n);
      const int64_t cap = a->ptr[n];
      int32_t* us = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap ? cap : 1));
      int32_t* vs = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap ? cap : 1));
      int64_t ne = 0;
      for (int32_t i = 0; i < n; ++i) {
        cost[i] = 1;
        for (int32_t p = a->ptr[i]; p < a->ptr[i + 1]; ++p) {
          const int32_t j = a->idx[p];
          if (j >= i)
            break;
          us[ne] = j;
          vs[ne] = i;
          ++ne;
          ++cost[i];
        }
      }
      make_dag(n, ne, us, vs, cost, out);
      free(us);
      free(vs);
      break;
    }
    case 7:
      intra_dag_csc_solve(&st.L_csc, costs_csc(2, &st.L_csc, &st.rv), out);
      break;
    case 8: {
      /* backward solve in reversed numbering i' = n-1-i: the DAG of
       * intra_dag(SpTRSV_CSR, to_csr(B)), B = P L^T P^T. Row i'
       * of B holds (i', n-1-j) for L(j, i) != 0, j >= i. */
      const smat* l = &st.L_csc;
      int64_t* cost = cost_alloc(n);
      const int64_t cap = l->ptr[n];
      int32_t* us = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap ? cap : 1));
      int32_t* vs = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap ? cap : 1));
      int64_t ne = 0;
      for (int32_t ip = 0; ip < n; ++ip) {
        const int32_t i = n - 1 - ip;
        cost[ip] = max1(l->ptr[i + 1] - l->ptr[i]);
        for (int32_t p = l->ptr[i + 1] - 1; p >= l->ptr[i]; --p) {
          const int32_t j = l->idx[p];
          if (j > i) {
            us[ne] = n - 1 - j;
            vs[ne] = ip;
            ++ne;
          }
        }
      }
      make_dag(n, ne, us, vs, cost, out);
      free(us);
      free(vs);
      break;
    }
    default:
      rc = ORC_ERR_BAD_ARG;
    }
  }
  state_free(&st);
  return rc;
}

int orc_inter_dag(int combo, int32_t n, const int32_t* colptr,
                  const int32_t* rowidx, const double* values,
                  orc_interdep* f) {
  memset(f, 0, sizeof(*f));
  ostate st;
  int32_t ei = -1;
  int rc = make_state(&st, combo, n, colptr, rowidx, values, 7, NULL, &ei);
  if (rc && rc != ORC_ERR_ZERO_DIAG_SCALE) {
    state_free(&st);
    return rc;
  }
  f->nrows = f->ncols = n;
  f->rowptr = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  int64_t cap = 0;
  switch (combo) {
  case 1:
  case 2:
  case 6:
  case 8:
  case 4:
    cap = n;
    break;
  case 3:
    cap = st.A_csr.ptr[n];
    break;
  case 5:
  case 7:
    cap = (int64_t)st.rv.ptr[n] + n;
    break;
  default:
    state_free(&st);
    return ORC_ERR_BAD_ARG;
  }
  f->colidx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap ? cap : 1));
  int64_t w = 0;
  for (int32_t i = 0; i < n; ++i) {
    switch (combo) {
    case 1:
    case 2:
    case 6: /* identity_interdep (dag.hpp:257-267) */
      f->colidx[w++] = i;
      break;
    case 8: /* anti-diagonal in reversed G2 numbering */
      f->colidx[w++] = n - 1 - i;
      break;
    case 4: /* dag.hpp:286-292 */
      if (st.M.ptr[i] < st.M.ptr[i + 1])
        f->colidx[w++] = i;
      break;
    case 3: /* dag.hpp:293-303 */
      for (int32_t p = st.A_csr.ptr[i]; p < st.A_csr.ptr[i + 1]; ++p) {
        const int32_t k = st.A_csr.idx[p];
        if (k > i)
          break;
        f->colidx[w++] = k;
      }
      break;
    case 5:
    case 7: /* dag.hpp:304-313: row-view columns (ascending, < i), then i */
      for (int32_t q = st.rv.ptr[i]; q < st.rv.ptr[i + 1]; ++q)
        f->colidx[w++] = st.rv.col[q];
      f->colidx[w++] = i;
      break;
    }
    f->rowptr[i + 1] = (int32_t)w;
  }
  f->nnz = w;
  state_free(&st);
  return ORC_OK;
}

int orc_joint_dag(const orc_dag* g1, const orc_dag* g2, const orc_interdep* f,
                  orc_dag* out) {
  memset(out, 0, sizeof(*out));
  const int64_t ne = g1->nedges + g2->nedges + f->nnz;
  int32_t* us = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ne ? ne : 1));
  int32_t* vs = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ne ? ne : 1));
  int64_t e = 0;
  for (int32_t u = 0; u < g1->nvert; ++u)
    for (int32_t p = g1->succptr[u]; p < g1->succptr[u + 1]; ++p) {
      us[e] = u;
      vs[e] = g1->succ[p];
      ++e;
    }
  for (int32_t u = 0; u < g2->nvert; ++u)
    for (int32_t p = g2->succptr[u]; p < g2->succptr[u + 1]; ++p) {
      us[e] = g1->nvert + u;
      vs[e] = g1->nvert + g2->succ[p];
      ++e;
    }
  for (int32_t i = 0; i < f->nrows; ++i)
    for (int32_t p = f->rowptr[i]; p < f->rowptr[i + 1]; ++p) {
      us[e] = f->colidx[p];
      vs[e] = g1->nvert + i;
      ++e;
    }
  const int32_t nv = g1->nvert + g2->nvert;
  int64_t* cost = cost_alloc(nv);
  for (int32_t v = 0; v < g1->nvert; ++v)
    cost[v] = g1->cost[v];
  for (int32_t v = 0; v < g2->nvert; ++v)
    cost[g1->nvert + v] = g2->cost[v];
  make_dag(nv, e, us, vs, cost, out);
  free(us);
  free(vs);
  return ORC_OK;
}

int orc_level_info(const orc_dag* g, int32_t* level, int32_t* height,
                   int32_t* slack, int32_t* critical_path) {
  const int32_t n = g->nvert;
  for (int32_t v = 0; v < n; ++v) {
    level[v] = 1;
    height[v] = 0;
  }
  for (int32_t u = 0; u < n; ++u)
    for (int32_t p = g->succptr[u]; p < g->succptr[u + 1]; ++p) {
      const int32_t v = g->succ[p];
      if (v <= u)
        return -1; /* "dependence cycle: edge does not ascend" */
      if (level[u] + 1 > level[v])
        level[v] = level[u] + 1;
    }
  int32_t P = 0;
  for (int32_t v = 0; v < n; ++v)
    if (level[v] > P)
      P = level[v];
  for (int32_t u = n; u-- > 0;)
    for (int32_t p = g->succptr[u]; p < g->succptr[u + 1]; ++p) {
      const int32_t h = height[g->succ[p]] + 1;
      if (h > height[u])
        height[u] = h;
    }
  for (int32_t v = 0; v < n; ++v)
    slack[v] = P - level[v] - height[v];
  *critical_path = P;
  return 0;
}

double orc_compute_reuse(int combo, int32_t n, const int32_t* colptr,
                         const int32_t* rowidx, const double* values) {
  (void)values;
  int64_t size_L = 0, size_A = 0, lower = 0;
  for (int32_t j = 0; j < n; ++j)
    for (int32_t p = colptr[j]; p < colptr[j + 1]; ++p)
      if (rowidx[p] >= j)
        ++lower;
  const int64_t nnzA = colptr[n];
  switch (combo) {
  case 1:
  case 8:
    size_L = lower;
    break;
  case 2:
  case 4:
    size_L = lower;
    size_A = nnzA;
    break;
  case 3:
    size_A = nnzA;
    break;
  case 5:
  case 7:
    size_L = lower;
    break;
  case 6:
    size_A = nnzA;
    size_L = lower; /* entries with col <= row (dag.hpp:419-425) */
    break;
  default:
    return -1.0;
  }
  /* dag.hpp:374-396 */
  const double dn = (double)n, L = (double)size_L, A = (double)size_A;
  double r;
#define DMAX(a, b) ((a) > (b) ? (a) : (b))
  switch (combo) {
  case 1:
  case 8:
    r = (2 * dn + 2 * L) / DMAX(2 * dn + L, L + 2 * dn);
    break;
  case 2:
  case 4:
    r = 2 * dn / DMAX(2 * dn + L, A + 2 * dn);
    break;
  case 3:
    r = 2 * A / DMAX(A, A + 2 * dn);
    break;
  case 5:
  case 7:
    r = 2 * L / DMAX(L, L + 2 * dn);
    break;
  case 6:
    r = 2 * A / DMAX(A, L + 2 * dn);
    break;
  default:
    r = -1.0;
  }
#undef DMAX
  return r;
}

void orc_free_dag(orc_dag* g) {
  free(g->succptr);
  free(g->succ);
  free(g->cost);
  memset(g, 0, sizeof(*g));
}

void orc_free_interdep(orc_interdep* f) {
  free(f->rowptr);
  free(f->colidx);
  memset(f, 0, sizeof(*f));
}
