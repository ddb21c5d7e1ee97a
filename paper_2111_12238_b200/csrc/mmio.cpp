// mmio.cpp -- Matrix Market ingest/egest and symmetric permutation for the
// plan inputs (host side, like the reference's own readers): real SuiteSparse
// matrices go through the same make_state path as the synthetic configs.
//
// Follows matrix_market.hpp:59-152 (coordinate real, general or symmetric;
// symmetric expanded to full storage; 1-based indices; duplicates summed;
// column-major sort; validate) and permute_symmetric (matrix.hpp:135-173,
// B = P A P^T with row/column i of A becoming perm[i] of B).
#include <algorithm>
#include <cctype>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/sfgpu.h"

#include "matrix_handle.hpp"

namespace {

struct Entry {
  int32_t i, j;
  double v;
};

void put(char* msg, int32_t len, const std::string& s) {
  if (!msg || len <= 0)
    return;
  const size_t n = std::min<size_t>(s.size(), (size_t)len - 1);
  std::memcpy(msg, s.data(), n);
  msg[n] = 0;
}

std::string lower(std::string s) {
  for (char& c : s)
    c = (char)std::tolower((unsigned char)c);
  return s;
}

// column-major order, duplicates summed in file order
void to_csc(int32_t n, std::vector<Entry>& t, sfg_matrix& M, bool sum_duplicates) {
  std::stable_sort(t.begin(), t.end(), [](const Entry& a, const Entry& b) {
    return a.j != b.j ? a.j < b.j : a.i < b.i;
  });
  M.n = n;
  M.colptr.assign((size_t)n + 1, 0);
  M.rowidx.clear();
  M.values.clear();
  for (size_t k = 0; k < t.size(); ++k) {
    if (sum_duplicates && k > 0 && t[k].i == t[k - 1].i && t[k].j == t[k - 1].j) {
      M.values.back() += t[k].v;
      continue;
    }
    ++M.colptr[(size_t)t[k].j + 1];
    M.rowidx.push_back(t[k].i);
    M.values.push_back(t[k].v);
  }
  for (int32_t j = 0; j < n; ++j)
    M.colptr[(size_t)j + 1] += M.colptr[(size_t)j];
}

bool next_data_line(std::ifstream& in, std::string& line) {
  do {
    if (!std::getline(in, line))
      return false;
  } while (line.empty() || line[0] == '%');
  return true;
}

} // namespace

extern "C" {

sfg_status sfg_matrix_read_mm(const char* path, sfg_matrix** out, char* msg, int32_t msg_len) {
  if (!path || !out)
    return SFG_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  const std::string p(path);
  auto fail = [&](const std::string& why) {
    put(msg, msg_len, p + ": " + why);
    return SFG_ERR_PARSE;
  };
  std::ifstream in(p);
  if (!in) {
    put(msg, msg_len, "cannot open " + p);
    return SFG_ERR_PARSE;
  }
  std::string line;
  if (!std::getline(in, line))
    return fail("empty file");
  std::istringstream hdr(line);
  std::string banner, object, format, field, symmetry;
  hdr >> banner >> object >> format >> field >> symmetry;
  if (banner != "%%MatrixMarket")
    return fail("missing MatrixMarket banner");
  if (lower(object) != "matrix" || lower(format) != "coordinate")
    return fail("only coordinate matrices are supported");
  if (lower(field) != "real")
    return fail("field '" + lower(field) + "' not supported");
  const std::string sym = lower(symmetry);
  if (sym != "general" && sym != "symmetric")
    return fail("symmetry '" + sym + "' not supported");
  if (!next_data_line(in, line))
    return fail("missing size line");
  long long nr = 0, nc = 0, nz = 0;
  {
    std::istringstream sz(line);
    if (!(sz >> nr >> nc >> nz) || nr < 0 || nc < 0 || nz < 0)
      return fail("malformed size line");
  }
  if (nr != nc) {
    put(msg, msg_len, p + ": combination input must be square");
    return SFG_ERR_INVALID_MATRIX;
  }
  std::vector<Entry> t;
  t.reserve((size_t)(sym == "symmetric" ? 2 * nz : nz));
  for (long long k = 0; k < nz; ++k) {
    if (!next_data_line(in, line))
      return fail("unexpected end of file at entry " + std::to_string(k + 1));
    std::istringstream es(line);
    long long i = 0, j = 0;
    double v = 0.0;
    if (!(es >> i >> j >> v))
      return fail("malformed entry " + std::to_string(k + 1));
    if (i < 1 || i > nr || j < 1 || j > nc)
      return fail("index out of bounds in entry " + std::to_string(k + 1));
    t.push_back({(int32_t)(i - 1), (int32_t)(j - 1), v});
    if (sym == "symmetric" && i != j)
      t.push_back({(int32_t)(j - 1), (int32_t)(i - 1), v});
  }
  auto* M = new sfg_matrix();
  to_csc((int32_t)nc, t, *M, true);
  *out = M;
  return SFG_OK;
}

sfg_status sfg_matrix_write_mm(const sfg_matrix* m, const char* path) {
  if (!m || !path)
    return SFG_ERR_INVALID_ARGUMENT;
  std::ofstream out(path);
  if (!out)
    return SFG_ERR_PARSE;
  out << "%%MatrixMarket matrix coordinate real general\n";
  out << m->n << ' ' << m->n << ' ' << m->rowidx.size() << '\n';
  out << std::setprecision(17);
  for (int32_t j = 0; j < m->n; ++j)
    for (int32_t q = m->colptr[(size_t)j]; q < m->colptr[(size_t)j + 1]; ++q)
      out << m->rowidx[(size_t)q] + 1 << ' ' << j + 1 << ' ' << m->values[(size_t)q] << '\n';
  return out ? SFG_OK : SFG_ERR_PARSE;
}

sfg_status sfg_matrix_from_csc(int32_t n, const int32_t* colptr, const int32_t* rowidx,
                               const double* values, sfg_matrix** out) {
  if (!out || n < 0 || !colptr)
    return SFG_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  const int32_t nnz = colptr[n];
  if (nnz > 0 && (!rowidx || !values))
    return SFG_ERR_INVALID_ARGUMENT;
  auto* M = new sfg_matrix();
  M->n = n;
  M->colptr.assign(colptr, colptr + n + 1);
  M->rowidx.assign(rowidx, rowidx + nnz);
  M->values.assign(values, values + nnz);
  *out = M;
  return SFG_OK;
}

sfg_status sfg_matrix_permute(const sfg_matrix* m, const int32_t* perm, sfg_matrix** out) {
  if (!m || !perm || !out)
    return SFG_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  std::vector<char> seen((size_t)m->n, 0);
  for (int32_t i = 0; i < m->n; ++i) {
    const int32_t q = perm[i];
    if (q < 0 || q >= m->n || seen[(size_t)q])
      return SFG_ERR_INVALID_MATRIX; // "not a permutation"
    seen[(size_t)q] = 1;
  }
  std::vector<Entry> t;
  t.reserve(m->rowidx.size());
  for (int32_t j = 0; j < m->n; ++j)
    for (int32_t q = m->colptr[(size_t)j]; q < m->colptr[(size_t)j + 1]; ++q)
      t.push_back({perm[m->rowidx[(size_t)q]], perm[j], m->values[(size_t)q]});
  auto* M = new sfg_matrix();
  to_csc(m->n, t, *M, false);
  *out = M;
  return SFG_OK;
}

sfg_status sfg_read_permutation(const char* path, int32_t n, int32_t* perm) {
  if (!path || !perm || n < 0)
    return SFG_ERR_INVALID_ARGUMENT;
  std::ifstream in(path);
  if (!in)
    return SFG_ERR_PARSE;
  long long v;
  int32_t k = 0;
  while (in >> v) {
    if (k >= n)
      return SFG_ERR_PARSE;
    perm[k++] = (int32_t)v;
  }
  return k == n ? SFG_OK : SFG_ERR_PARSE;
}

} // extern "C"
