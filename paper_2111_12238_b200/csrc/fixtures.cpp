// fixtures.cpp -- seeded input generators (the reference's fixtures.hpp,
// fixtures.hpp:19-155, plus the five BASELINE.json configurations).
//
// Random numbers come from std::mt19937_64 and the libstdc++ distributions,
// the same engine and distributions the reference uses, so gen_vector and
// gen_banded_spd reproduce the reference's inputs bit for bit (pinned by
// tests/test_fixtures.py against oracle/_ref).
#include "../../include/sfgpu.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <new>
#include <random>
#include <vector>

#include "matrix_handle.hpp"

namespace {

using Entry = struct {
  int32_t i, j;
  double v;
};

void build_from_entries(std::vector<Entry>& e, int32_t n, sfg_matrix& M) {
  std::sort(e.begin(), e.end(), [](const Entry& a, const Entry& b) {
    return a.j != b.j ? a.j < b.j : a.i < b.i;
  });
  M.n = n;
  M.colptr.assign((size_t)n + 1, 0);
  M.rowidx.resize(e.size());
  M.values.resize(e.size());
  for (size_t k = 0; k < e.size(); ++k) {
    ++M.colptr[(size_t)e[k].j + 1];
    M.rowidx[k] = e[k].i;
    M.values[k] = e[k].v;
  }
  for (int32_t j = 0; j < n; ++j)
    M.colptr[(size_t)j + 1] += M.colptr[j];
}

// Recursive-bisection numbering (fixtures.hpp:19-40).
void nd_number(int32_t x0, int32_t y0, int32_t w, int32_t h, int32_t k,
               std::vector<int32_t>& id, int32_t& next) {
  if (w <= 2 || h <= 2) {
    for (int32_t y = y0; y < y0 + h; ++y)
      for (int32_t x = x0; x < x0 + w; ++x)
        id[(size_t)y * k + x] = next++;
    return;
  }
  if (w >= h) {
    const int32_t mid = x0 + w / 2;
    nd_number(x0, y0, mid - x0, h, k, id, next);
    nd_number(mid + 1, y0, x0 + w - mid - 1, h, k, id, next);
    for (int32_t y = y0; y < y0 + h; ++y)
      id[(size_t)y * k + mid] = next++;
  } else {
    const int32_t mid = y0 + h / 2;
    nd_number(x0, y0, w, mid - y0, k, id, next);
    nd_number(x0, mid + 1, w, y0 + h - mid - 1, k, id, next);
    for (int32_t x = x0; x < x0 + w; ++x)
      id[(size_t)mid * k + x] = next++;
  }
}

// gen_grid_laplacian (fixtures.hpp:49-91): ND-numbered 5-point Laplacian.
bool grid_laplacian_nd(int32_t k, sfg_matrix& M) {
  if (k < 2)
    return false;
  const int32_t n = k * k;
  std::vector<int32_t> id((size_t)n);
  int32_t next = 0;
  nd_number(0, 0, k, k, k, id, next);
  std::vector<Entry> e;
  e.reserve((size_t)5 * n);
  for (int32_t cell = 0; cell < n; ++cell) {
    const int32_t r = cell / k, c = cell % k;
    const int32_t j = id[cell];
    e.push_back({j, j, 4.0});
    if (r > 0)
      e.push_back({id[cell - k], j, -1.0});
    if (c > 0)
      e.push_back({id[cell - 1], j, -1.0});
    if (c + 1 < k)
      e.push_back({id[cell + 1], j, -1.0});
    if (r + 1 < k)
      e.push_back({id[cell + k], j, -1.0});
  }
  build_from_entries(e, n, M);
  return true;
}

// gen_banded_spd (fixtures.hpp:97-141).
bool banded_spd(int32_t n, int32_t bw, uint64_t seed, sfg_matrix& M) {
  if (n < 2 || bw < 1 || bw >= n)
    return false;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> mag(0.1, 1.0);
  std::bernoulli_distribution sign(0.5);
  std::vector<std::vector<double>> lowvals((size_t)n);
  for (int32_t i = 0; i < n; ++i) {
    const int32_t lo = std::max<int32_t>(0, i - bw);
    lowvals[i].resize((size_t)(i - lo));
    for (int32_t j = lo; j < i; ++j)
      lowvals[i][(size_t)(j - lo)] = (sign(rng) ? 1.0 : -1.0) * mag(rng);
  }
  std::vector<double> diag((size_t)n, 0.0);
  for (int32_t i = 0; i < n; ++i) {
    double sum = 0.0;
    const int32_t lo = std::max<int32_t>(0, i - bw);
    for (int32_t j = lo; j < i; ++j)
      sum += std::abs(lowvals[i][(size_t)(j - lo)]);
    for (int32_t i2 = i + 1; i2 < std::min<int32_t>(n, i + bw + 1); ++i2)
      sum += std::abs(lowvals[i2][(size_t)(i - std::max<int32_t>(0, i2 - bw))]);
    diag[i] = sum + 1.0 + mag(rng);
  }
  M.n = n;
  M.colptr.assign((size_t)n + 1, 0);
  for (int32_t j = 0; j < n; ++j) {
    const int32_t lo = std::max<int32_t>(0, j - bw);
    const int32_t hi = std::min<int32_t>(n - 1, j + bw);
    for (int32_t i = lo; i <= hi; ++i) {
      double v;
      if (i == j)
        v = diag[j];
      else if (i > j)
        v = lowvals[i][(size_t)(j - std::max<int32_t>(0, i - bw))];
      else
        v = lowvals[j][(size_t)(i - std::max<int32_t>(0, j - bw))];
      M.rowidx.push_back(i);
      M.values.push_back(v);
    }
    M.colptr[(size_t)j + 1] = (int32_t)M.rowidx.size();
  }
  return true;
}

// Config 1: 5-point Laplacian on an a x a grid in natural row-major order
// (the reference's ND ordering makes its MSP inspector
// infeasible for this combo), diagonal 4, off-diagonals -1.
bool cfg1(int32_t a, sfg_matrix& M) {
  if (a < 2)
    return false;
  const int32_t n = a * a;
  M.n = n;
  M.colptr.assign((size_t)n + 1, 0);
  M.rowidx.reserve((size_t)5 * n);
  M.values.reserve((size_t)5 * n);
  for (int32_t j = 0; j < n; ++j) {
    const int32_t r = j / a, c = j % a;
    auto put = [&](int32_t i, double v) {
      M.rowidx.push_back(i);
      M.values.push_back(v);
    };
    if (r > 0)
      put(j - a, -1.0);
    if (c > 0)
      put(j - 1, -1.0);
    put(j, 4.0);
    if (c + 1 < a)
      put(j + 1, -1.0);
    if (r + 1 < a)
      put(j + a, -1.0);
    M.colptr[(size_t)j + 1] = (int32_t)M.rowidx.size();
  }
  return true;
}

// Config 2: 7-point 3-D Laplacian on a^3, natural order, diagonal 6.01.
bool cfg2(int32_t a, sfg_matrix& M) {
  if (a < 2)
    return false;
  const int64_t n64 = (int64_t)a * a * a;
  if (n64 > INT32_MAX)
    return false;
  const int32_t n = (int32_t)n64, a2 = a * a;
  M.n = n;
  M.colptr.assign((size_t)n + 1, 0);
  M.rowidx.reserve((size_t)7 * n);
  M.values.reserve((size_t)7 * n);
  for (int32_t j = 0; j < n; ++j) {
    const int32_t x = j % a, y = (j / a) % a, z = j / a2;
    auto put = [&](int32_t i, double v) {
      M.rowidx.push_back(i);
      M.values.push_back(v);
    };
    if (z > 0)
      put(j - a2, -1.0);
    if (y > 0)
      put(j - a, -1.0);
    if (x > 0)
      put(j - 1, -1.0);
    put(j, 6.01);
    if (x + 1 < a)
      put(j + 1, -1.0);
    if (y + 1 < a)
      put(j + a, -1.0);
    if (z + 1 < a)
      put(j + a2, -1.0);
    M.colptr[(size_t)j + 1] = (int32_t)M.rowidx.size();
  }
  return true;
}

// Config 3: 7-point 3-D convection-diffusion on a^3, natural order.  For each
// undirected grid edge (i, j), i < j, one beta ~ U[0, 0.5] is drawn (vertex i
// ascending; x, y, z neighbour order); the upper entry A(i, j) = -1 + beta and
// the lower entry A(j, i) = -1 - beta (decision recorded in DESIGN.md).  The
// diagonal is the row's absolute off-diagonal sum plus 0.1.
bool cfg3(int32_t a, uint64_t seed, sfg_matrix& M) {
  if (a < 2)
    return false;
  const int64_t n64 = (int64_t)a * a * a;
  if (n64 > INT32_MAX)
    return false;
  const int32_t n = (int32_t)n64, a2 = a * a;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> ub(0.0, 0.5);
  std::vector<double> beta((size_t)3 * n, 0.0); // beta[3*i + d], neighbour i + step_d
  for (int32_t i = 0; i < n; ++i) {
    const int32_t x = i % a, y = (i / a) % a, z = i / a2;
    if (x + 1 < a)
      beta[(size_t)3 * i + 0] = ub(rng);
    if (y + 1 < a)
      beta[(size_t)3 * i + 1] = ub(rng);
    if (z + 1 < a)
      beta[(size_t)3 * i + 2] = ub(rng);
  }
  // diagonal: sum over upper neighbours (1 - beta) + lower neighbours (1 + beta)
  std::vector<double> diag((size_t)n, 0.0);
  const int32_t step[3] = {1, a, a2};
  for (int32_t i = 0; i < n; ++i) {
    const int32_t c[3] = {i % a, (i / a) % a, i / a2};
    double s = 0.0;
    for (int d = 2; d >= 0; --d) // lower neighbours, ascending column order
      if (c[d] > 0)
        s += std::abs(-1.0 - beta[(size_t)3 * (i - step[d]) + d]);
    for (int d = 0; d < 3; ++d) // upper neighbours, ascending column order
      if (c[d] + 1 < a)
        s += std::abs(-1.0 + beta[(size_t)3 * i + d]);
    diag[i] = s + 0.1;
  }
  M.n = n;
  M.colptr.assign((size_t)n + 1, 0);
  M.rowidx.reserve((size_t)7 * n);
  M.values.reserve((size_t)7 * n);
  for (int32_t j = 0; j < n; ++j) {
    const int32_t c[3] = {j % a, (j / a) % a, j / a2};
    auto put = [&](int32_t i, double v) {
      M.rowidx.push_back(i);
      M.values.push_back(v);
    };
    // rows i < j in column j are upper entries A(i, j), i = j - step_d
    for (int d = 2; d >= 0; --d)
      if (c[d] > 0)
        put(j - step[d], -1.0 + beta[(size_t)3 * (j - step[d]) + d]);
    put(j, diag[j]);
    // rows i > j in column j are lower entries A(i, j) = -1 - beta(j, i)
    for (int d = 0; d < 3; ++d)
      if (c[d] + 1 < a)
        put(j + step[d], -1.0 - beta[(size_t)3 * j + d]);
    M.colptr[(size_t)j + 1] = (int32_t)M.rowidx.size();
  }
  return true;
}

// Config 4: random symmetric band matrix.  Each row i draws 8 column offsets
// uniformly from [-hw, hw] (redrawing 0 and out-of-range columns); the union
// of the pairs is symmetrised, each unordered pair gets one value ~ U[-1, 0]
// (drawn in ascending (row, col) pair order), and the diagonal is the row's
// absolute off-diagonal sum plus 1, which makes the matrix SPD.
bool cfg4(int32_t n, int32_t hw, uint64_t seed, sfg_matrix& M) {
  if (n < 2 || hw < 1)
    return false;
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int32_t> off(-hw, hw);
  std::vector<uint64_t> pairs;
  pairs.reserve((size_t)8 * n);
  for (int32_t i = 0; i < n; ++i)
    for (int d = 0; d < 8; ++d) {
      int32_t j;
      do {
        j = i + off(rng);
      } while (j == i || j < 0 || j >= n);
      const int32_t lo = std::min(i, j), hi = std::max(i, j);
      pairs.push_back(((uint64_t)(uint32_t)hi << 32) | (uint32_t)lo); // (row > col)
    }
  std::sort(pairs.begin(), pairs.end());
  pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
  std::uniform_real_distribution<double> val(-1.0, 0.0);
  std::vector<double> pv(pairs.size());
  for (auto& v : pv)
    v = val(rng);
  std::vector<double> diag((size_t)n, 1.0);
  std::vector<double> absum((size_t)n, 0.0);
  std::vector<int32_t> cnt((size_t)n + 1, 0);
  for (size_t k = 0; k < pairs.size(); ++k) {
    const int32_t r = (int32_t)(pairs[k] >> 32), c = (int32_t)(pairs[k] & 0xffffffffu);
    absum[r] += std::abs(pv[k]);
    absum[c] += std::abs(pv[k]);
    ++cnt[(size_t)c + 1]; // lower entry (r, c) in column c
    ++cnt[(size_t)r + 1]; // upper entry (c, r) in column r
  }
  for (int32_t i = 0; i < n; ++i) {
    diag[i] = absum[i] + 1.0;
    ++cnt[(size_t)i + 1];
  }
  M.n = n;
  M.colptr.assign((size_t)n + 1, 0);
  for (int32_t j = 0; j < n; ++j)
    M.colptr[(size_t)j + 1] = M.colptr[j] + cnt[(size_t)j + 1];
  M.rowidx.assign((size_t)M.colptr[n], 0);
  M.values.assign((size_t)M.colptr[n], 0.0);
  std::vector<int32_t> next(M.colptr.begin(), M.colptr.end() - 1);
  // column j gets rows ascending: upper entries (rows < j) come from pairs
  // with hi == j; iterate pairs in (hi, lo) order for those, then the
  // diagonal, then the lower entries (rows > j) from pairs with lo == j.
  std::vector<std::vector<std::pair<int32_t, double>>> lowers((size_t)n);
  for (size_t k = 0; k < pairs.size(); ++k) {
    const int32_t r = (int32_t)(pairs[k] >> 32), c = (int32_t)(pairs[k] & 0xffffffffu);
    // upper entry (c, r): column r, row c < r; pairs sorted by (r, c)
    M.rowidx[(size_t)next[r]] = c;
    M.values[(size_t)next[r]] = pv[k];
    ++next[r];
    lowers[c].push_back({r, pv[k]});
  }
  for (int32_t j = 0; j < n; ++j) {
    M.rowidx[(size_t)next[j]] = j;
    M.values[(size_t)next[j]] = diag[j];
    ++next[j];
    auto& L = lowers[j];
    std::sort(L.begin(), L.end());
    for (auto& e : L) {
      M.rowidx[(size_t)next[j]] = e.first;
      M.values[(size_t)next[j]] = e.second;
      ++next[j];
    }
    std::vector<std::pair<int32_t, double>>().swap(L);
  }
  return true;
}

// Config 5: 27-point 3-D stencil on a^3, natural order, diagonal 26.5,
// off-diagonals -1.
bool cfg5(int32_t a, sfg_matrix& M) {
  if (a < 2)
    return false;
  const int64_t n64 = (int64_t)a * a * a;
  if (n64 > INT32_MAX)
    return false;
  const int32_t n = (int32_t)n64, a2 = a * a;
  M.n = n;
  M.colptr.assign((size_t)n + 1, 0);
  M.rowidx.reserve((size_t)27 * n);
  M.values.reserve((size_t)27 * n);
  for (int32_t j = 0; j < n; ++j) {
    const int32_t x = j % a, y = (j / a) % a, z = j / a2;
    for (int dz = -1; dz <= 1; ++dz) {
      if (z + dz < 0 || z + dz >= a)
        continue;
      for (int dy = -1; dy <= 1; ++dy) {
        if (y + dy < 0 || y + dy >= a)
          continue;
        for (int dx = -1; dx <= 1; ++dx) {
          if (x + dx < 0 || x + dx >= a)
            continue;
          const int32_t i = j + dz * a2 + dy * a + dx;
          M.rowidx.push_back(i);
          M.values.push_back(i == j ? 26.5 : -1.0);
        }
      }
    }
    M.colptr[(size_t)j + 1] = (int32_t)M.rowidx.size();
  }
  return true;
}

} // namespace

extern "C" {

sfg_status sfg_matrix_gen(int32_t kind, int32_t a, int32_t b, uint64_t seed,
                          sfg_matrix** out) {
  if (!out)
    return SFG_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  auto* M = new (std::nothrow) sfg_matrix();
  if (!M)
    return SFG_ERR_INVALID_ARGUMENT;
  bool ok = false;
  try {
    switch (kind) {
    case 0:
      ok = grid_laplacian_nd(a, *M);
      break;
    case 1:
      ok = banded_spd(a, b, seed, *M);
      break;
    case 10:
      ok = cfg1(a, *M);
      break;
    case 11:
      ok = cfg2(a, *M);
      break;
    case 12:
      ok = cfg3(a, seed, *M);
      break;
    case 13:
      ok = cfg4(a, b, seed, *M);
      break;
    case 14:
      ok = cfg5(a, *M);
      break;
    default:
      ok = false;
    }
  } catch (...) {
    ok = false;
  }
  if (!ok) {
    delete M;
    return SFG_ERR_INVALID_ARGUMENT;
  }
  *out = M;
  return SFG_OK;
}

sfg_status sfg_matrix_dims(const sfg_matrix* m, int32_t* n, int64_t* nnz) {
  if (!m)
    return SFG_ERR_INVALID_ARGUMENT;
  if (n)
    *n = m->n;
  if (nnz)
    *nnz = (int64_t)m->rowidx.size();
  return SFG_OK;
}

sfg_status sfg_matrix_copy(const sfg_matrix* m, int32_t* colptr,
                           int32_t* rowidx, double* values) {
  if (!m)
    return SFG_ERR_INVALID_ARGUMENT;
  if (colptr)
    std::memcpy(colptr, m->colptr.data(), sizeof(int32_t) * m->colptr.size());
  if (rowidx)
    std::memcpy(rowidx, m->rowidx.data(), sizeof(int32_t) * m->rowidx.size());
  if (values)
    std::memcpy(values, m->values.data(), sizeof(double) * m->values.size());
  return SFG_OK;
}

sfg_status sfg_matrix_free(sfg_matrix* m) {
  delete m;
  return SFG_OK;
}

sfg_status sfg_matrix_perturb_diag(const sfg_matrix* m, int32_t nsys,
                                   uint64_t seed0, double* out) {
  if (!m || !out || nsys < 1)
    return SFG_ERR_INVALID_ARGUMENT;
  const size_t nnz = m->values.size();
  for (int32_t s = 0; s < nsys; ++s) {
    double* v = out + (size_t)s * nnz;
    std::memcpy(v, m->values.data(), sizeof(double) * nnz);
    std::mt19937_64 rng(seed0 + (uint64_t)s);
    std::uniform_real_distribution<double> delta(0.0, 0.1);
    for (int32_t j = 0; j < m->n; ++j)
      for (int32_t p = m->colptr[j]; p < m->colptr[(size_t)j + 1]; ++p)
        if (m->rowidx[(size_t)p] == j) {
          v[p] += delta(rng);
          break;
        }
  }
  return SFG_OK;
}

sfg_status sfg_gen_vector(int32_t n, uint64_t seed, double* out) {
  if (n < 0 || (n > 0 && !out))
    return SFG_ERR_INVALID_ARGUMENT;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (int32_t i = 0; i < n; ++i)
    out[i] = dist(rng);
  return SFG_OK;
}

} // extern "C"
