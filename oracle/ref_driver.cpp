// ref_driver.cpp -- extern "C" shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile directly against the
// reference sources where they lie (/root/reference/proj/include, and
// proj/tests for the paper's 11-vertex fixture) into oracle/_ref/libsfref.so.
// Nothing from the reference is copied into this repository; this file only
// marshals plain arrays into the reference's own types and calls its own
// functions.  Used (a) to pin the C restatement in oracle/sf_oracle.c,
// (b) to generate tests/golden/ fixtures, and (c) as the CPU baseline
// ("kind": "reference") timed by bench.py.
//
// The BASELINE.json input generators are this repository's own
// (paper_2111_12238_b200/csrc/fixtures.cpp); oracle/Makefile compiles that
// file into this library under renamed symbols (sfg_* -> refgen_*), so the
// reference arm of bench.py generates its inputs without loading
// libsfgpu.so.
#include <sparsefuse/dag.hpp>
#include <sparsefuse/executor.hpp>
#include <sparsefuse/fixtures.hpp>
#include <sparsefuse/kernels.hpp>
#include <sparsefuse/lbc.hpp>
#include <sparsefuse/matrix_market.hpp>
#include <sparsefuse/msp.hpp>

#include "fixture11.hpp"

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

using namespace sparsefuse;

namespace {

void put_msg(char* buf, int len, const std::string& s) {
  if (!buf || len <= 0)
    return;
  const std::size_t n = std::min<std::size_t>(s.size(), (std::size_t)len - 1);
  std::memcpy(buf, s.data(), n);
  buf[n] = 0;
}

CscMatrix from_arrays(int32_t n, const int32_t* colptr, const int32_t* rowidx,
                      const double* values) {
  CscMatrix M;
  M.nrows = M.ncols = n;
  M.colptr.assign(colptr, colptr + n + 1);
  const int32_t nnz = colptr[n];
  M.rowidx.assign(rowidx, rowidx + nnz);
  M.values.assign(values, values + nnz);
  return M;
}

double now_s() {
  return std::chrono::duration<double>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// Returns 0 ok, 1 FactorizationError, 2 InvalidMatrixError, 3 other.
template <typename F> int guarded(F&& f, int32_t* err_index, char* msg, int ml) {
  try {
    f();
    return 0;
  } catch (const FactorizationError& e) {
    if (err_index)
      *err_index = e.index();
    put_msg(msg, ml, e.what());
    return 1;
  } catch (const InvalidMatrixError& e) {
    put_msg(msg, ml, e.what());
    return 2;
  } catch (const std::exception& e) {
    put_msg(msg, ml, e.what());
    return 3;
  }
}

struct Setup {
  DepDag g1, g2;
  InterDep f;
  double reuse = 0;
};

Setup inspect(const KernelState& st) {
  Setup s;
  s.g1 = build_g1(st);
  s.g2 = build_g2(st);
  s.f = inter_dag(st);
  s.reuse = compute_reuse(st);
  return s;
}

} // namespace

extern "C" {

// ---- fixtures.hpp -------------------------------------------------------
void ref_gen_vector(int32_t n, uint64_t seed, double* out) {
  const DenseVector v = gen_vector(n, seed);
  std::memcpy(out, v.data(), sizeof(double) * v.size());
}

// kind 0: gen_grid_laplacian(a); 1: gen_banded_spd(a, b, seed);
// 2: gen_dense_spd(a, seed); 3: fixture11::lower(); 4: fixture11::spmv_matrix()
void* ref_mat_gen(int kind, int32_t a, int32_t b, uint64_t seed) {
  try {
    switch (kind) {
    case 0:
      return new CscMatrix(gen_grid_laplacian(a));
    case 1:
      return new CscMatrix(gen_banded_spd(a, b, seed));
    case 2:
      return new CscMatrix(gen_dense_spd(a, seed));
    case 3:
      return new CscMatrix(fixture11::lower());
    case 4:
      return new CscMatrix(fixture11::spmv_matrix());
    default:
      return nullptr;
    }
  } catch (...) {
    return nullptr;
  }
}

void ref_mat_dims(void* m, int32_t* n, int32_t* nnz) {
  auto* M = static_cast<CscMatrix*>(m);
  *n = M->ncols;
  *nnz = M->nnz();
}

void ref_mat_copy(void* m, int32_t* colptr, int32_t* rowidx, double* values) {
  auto* M = static_cast<CscMatrix*>(m);
  std::copy(M->colptr.begin(), M->colptr.end(), colptr);
  std::copy(M->rowidx.begin(), M->rowidx.end(), rowidx);
  std::copy(M->values.begin(), M->values.end(), values);
}

void ref_mat_free(void* m) { delete static_cast<CscMatrix*>(m); }

// ---- kernels.hpp: make_state ---------------------------------------------
void* ref_state_new(int combo, int32_t n, const int32_t* colptr,
                    const int32_t* rowidx, const double* values, uint64_t seed,
                    const double* vin, int32_t* err_index, char* msg, int ml) {
  KernelState* out = nullptr;
  const int rc = guarded(
      [&] {
        KernelState st =
            make_state(combo, from_arrays(n, colptr, rowidx, values), seed);
        if (vin)
          st.vin.assign(vin, vin + n);
        out = new KernelState(std::move(st));
      },
      err_index, msg, ml);
  (void)rc;
  return out;
}

// The paper's running example state (tests/fixture11.hpp:71-81).
void* ref_state_fixture11(uint64_t seed) {
  return new KernelState(fixture11::state(seed));
}

void ref_state_free(void* s) { delete static_cast<KernelState*>(s); }

int64_t ref_output_len(void* s) {
  auto* st = static_cast<KernelState*>(s);
  return static_cast<int64_t>(collect_outputs(*st).size());
}

// ---- executors (executor.hpp) ---------------------------------------------
// executor: 0 sequential, 1 fused (msp + compile_schedule), 2 unfused,
// 3 joint wavefront.  Writes collect_outputs into out.
int ref_execute(void* s, int executor, int32_t nthreads, double* out,
                int64_t cap, int32_t* err_index, char* msg, int ml) {
  auto* st = static_cast<KernelState*>(s);
  return guarded(
      [&] {
        if (executor == 0) {
          execute_sequential(*st);
        } else {
          const Setup su = inspect(*st);
          if (executor == 1) {
            const FusedPartitioning V =
                msp(su.g1, su.g2, su.f, nthreads, su.reuse);
            const FusedSchedule fs =
                compile_schedule(V, su.reuse, su.g1, su.g2, nthreads);
            execute_fused(fs, *st, nthreads);
          } else if (executor == 2) {
            execute_unfused(su.g1, su.g2, *st, nthreads);
          } else {
            execute_joint_wavefront(su.g1, su.g2, su.f, *st, nthreads);
          }
        }
        const std::vector<double> o = collect_outputs(*st);
        if ((int64_t)o.size() > cap)
          throw std::invalid_argument("output buffer too small");
        std::copy(o.begin(), o.end(), out);
      },
      err_index, msg, ml);
}

// Timing protocol of bench.hpp:188-207: the inspector (DAGs + schedule) runs
// once and is reported separately; then `warmups` untimed and `repeats` timed
// executions.  times[r] = wall seconds of repeat r (ExecStats::wall_ns, the
// parallel region; executor.hpp:296-310).  Returns the ref_execute codes.
int ref_bench(void* s, int executor, int32_t nthreads, int warmups,
              int repeats, double* times, double* inspector_s,
              int32_t* n_spartitions, char* msg, int ml) {
  auto* st = static_cast<KernelState*>(s);
  int32_t ei = -1;
  return guarded(
      [&] {
        const double t0 = now_s();
        const Setup su = inspect(*st);
        FusedSchedule fs;
        UnfusedSchedule us;
        WavefrontSchedule ws;
        int32_t nsp = 0;
        if (executor == 1) {
          const FusedPartitioning V =
              msp(su.g1, su.g2, su.f, nthreads, su.reuse);
          fs = compile_schedule(V, su.reuse, su.g1, su.g2, nthreads);
          nsp = fs.nspartitions();
        } else if (executor == 2) {
          us = build_unfused_schedule(su.g1, su.g2, nthreads);
          nsp = us.k1.nspartitions() + us.k2.nspartitions();
        } else if (executor == 3) {
          ws = build_wavefront_schedule(su.g1, su.g2, su.f);
          nsp = static_cast<int32_t>(ws.levels.size());
        }
        if (inspector_s)
          *inspector_s = now_s() - t0;
        if (n_spartitions)
          *n_spartitions = nsp;
        for (int r = 0; r < warmups + repeats; ++r) {
          ExecStats es;
          if (executor == 0)
            es = execute_sequential(*st);
          else if (executor == 1)
            es = execute_fused(fs, *st, nthreads);
          else if (executor == 2)
            es = execute_unfused(us, *st, nthreads);
          else
            es = execute_joint_wavefront(ws, *st, nthreads);
          if (r >= warmups)
            times[r - warmups] = static_cast<double>(es.wall_ns) * 1e-9;
        }
      },
      &ei, msg, ml);
}

// ---- dag.hpp ----------------------------------------------------------------
void* ref_build_g(void* s, int which) {
  auto* st = static_cast<KernelState*>(s);
  try {
    return new DepDag(which == 1 ? build_g1(*st) : build_g2(*st));
  } catch (...) {
    return nullptr;
  }
}

void* ref_inter_dag(void* s) {
  auto* st = static_cast<KernelState*>(s);
  try {
    return new InterDep(inter_dag(*st));
  } catch (...) {
    return nullptr;
  }
}

void* ref_joint_dag(void* g1, void* g2, void* f) {
  return new DepDag(joint_dag(*static_cast<DepDag*>(g1),
                              *static_cast<DepDag*>(g2),
                              *static_cast<InterDep*>(f)));
}

// Builds a DepDag from CSR arrays (through the reference's make_dag).
void* ref_dag_from_csr(int32_t nvert, const int32_t* succptr,
                       const int32_t* succ, const int64_t* cost) {
  std::vector<std::pair<Index, Index>> edges;
  for (Index u = 0; u < nvert; ++u)
    for (Index p = succptr[u]; p < succptr[u + 1]; ++p)
      edges.push_back({u, succ[p]});
  return new DepDag(detail::make_dag(
      nvert, std::move(edges), std::vector<Cost>(cost, cost + nvert)));
}

void ref_dag_dims(void* g, int32_t* nvert, int64_t* nedges) {
  auto* d = static_cast<DepDag*>(g);
  *nvert = d->nvert;
  *nedges = d->nedges();
}

void ref_dag_copy(void* g, int32_t* succptr, int32_t* succ, int64_t* cost) {
  auto* d = static_cast<DepDag*>(g);
  std::copy(d->succptr.begin(), d->succptr.end(), succptr);
  std::copy(d->succ.begin(), d->succ.end(), succ);
  std::copy(d->cost.begin(), d->cost.end(), cost);
}

void ref_dag_free(void* g) { delete static_cast<DepDag*>(g); }

void ref_inter_dims(void* f, int32_t* nrows, int32_t* ncols, int64_t* nnz) {
  auto* d = static_cast<InterDep*>(f);
  *nrows = d->nrows;
  *ncols = d->ncols;
  *nnz = d->nnz();
}

void ref_inter_copy(void* f, int32_t* rowptr, int32_t* colidx) {
  auto* d = static_cast<InterDep*>(f);
  std::copy(d->rowptr.begin(), d->rowptr.end(), rowptr);
  std::copy(d->colidx.begin(), d->colidx.end(), colidx);
}

void ref_inter_free(void* f) { delete static_cast<InterDep*>(f); }

// level_info: returns 0, or 3 if the DAG has a non-ascending edge.
int ref_level_info(void* g, int32_t* level, int32_t* height, int32_t* slack,
                   int32_t* critical_path) {
  try {
    const LevelInfo li = level_info(*static_cast<DepDag*>(g));
    std::copy(li.level.begin(), li.level.end(), level);
    std::copy(li.height.begin(), li.height.end(), height);
    std::copy(li.slack.begin(), li.slack.end(), slack);
    *critical_path = li.critical_path;
    return 0;
  } catch (...) {
    return 3;
  }
}

double ref_compute_reuse(void* s) {
  return compute_reuse(*static_cast<KernelState*>(s));
}

// Wavefront level sets of the joint DAG (executor.hpp:209-229): entries as
// (tag, iter) in schedule order and the [begin, end) of each level.
int64_t ref_wavefront(void* s, uint8_t* tags, int32_t* iters,
                      int32_t* level_ptr, int32_t* nlevels) {
  auto* st = static_cast<KernelState*>(s);
  const Setup su = inspect(*st);
  const WavefrontSchedule ws = build_wavefront_schedule(su.g1, su.g2, su.f);
  if (tags)
    for (std::size_t e = 0; e < ws.entries.size(); ++e) {
      tags[e] = ws.entries[e].tag;
      iters[e] = ws.entries[e].iter;
    }
  if (level_ptr) {
    for (std::size_t l = 0; l < ws.levels.size(); ++l)
      level_ptr[l] = ws.levels[l].first;
    level_ptr[ws.levels.size()] =
        ws.levels.empty() ? 0 : ws.levels.back().second;
  }
  *nlevels = static_cast<int32_t>(ws.levels.size());
  return static_cast<int64_t>(ws.entries.size());
}

// validate_fused_partitioning (msp.hpp:1108-1237) of a partitioning built
// elsewhere (the GPU inspector): s-partition k = w-partitions
// [s_ptr[k], s_ptr[k+1]), w-partition w = entries [w_ptr[w], w_ptr[w+1]).
// Returns the number of violations; the first one goes to msg.
int64_t ref_validate_partitioning(void* s, int32_t nspart, const int64_t* s_ptr,
                                  const int64_t* w_ptr, const uint8_t* tags,
                                  const int32_t* iters, char* msg, int ml) {
  auto* st = static_cast<KernelState*>(s);
  const Setup su = inspect(*st);
  FusedPartitioning V;
  V.fusion = true;
  V.reuse_ratio = su.reuse;
  V.interleaved = su.reuse >= 1.0;
  V.n1 = su.g1.nvert;
  V.n2 = su.g2.nvert;
  V.spartitions.resize((std::size_t)nspart);
  for (int32_t k = 0; k < nspart; ++k)
    for (int64_t w = s_ptr[k]; w < s_ptr[k + 1]; ++w) {
      std::vector<FusedEntry> es;
      for (int64_t e = w_ptr[w]; e < w_ptr[w + 1]; ++e)
        es.push_back(FusedEntry{tags[e], iters[e], false});
      V.spartitions[(std::size_t)k].push_back(std::move(es));
    }
  const std::vector<std::string> bad = validate_fused_partitioning(V, su.g1, su.g2, su.f);
  if (!bad.empty())
    put_msg(msg, ml, bad.front() + " (" + std::to_string(bad.size()) + " violations)");
  return (int64_t)bad.size();
}

// replay_schedule (executor.hpp:518-553) of an external partitioning in flat
// form: one thread, w-partitions of each s-partition interleaved in a seeded
// random order, then collect_outputs into out.  Returns the ref_execute codes.
int ref_replay_partitioning(void* s, int32_t nspart, const int64_t* s_ptr, const int64_t* w_ptr,
                            const uint8_t* tags, const int32_t* iters, uint64_t seed, double* out,
                            int64_t cap, int32_t* err_index, char* msg, int ml) {
  auto* st = static_cast<KernelState*>(s);
  return guarded(
      [&] {
        FusedPartitioning V;
        V.fusion = true;
        V.n1 = V.n2 = st->n;
        V.spartitions.resize((std::size_t)nspart);
        for (int32_t k = 0; k < nspart; ++k)
          for (int64_t w = s_ptr[k]; w < s_ptr[k + 1]; ++w) {
            std::vector<FusedEntry> es;
            for (int64_t e = w_ptr[w]; e < w_ptr[w + 1]; ++e)
              es.push_back(FusedEntry{tags[e], iters[e], false});
            V.spartitions[(std::size_t)k].push_back(std::move(es));
          }
        std::vector<std::string> dups;
        replay_schedule(V, *st, seed, true, &dups);
        if (!dups.empty())
          throw std::logic_error(dups.front());
        const std::vector<double> o = collect_outputs(*st);
        if ((int64_t)o.size() > cap)
          throw std::invalid_argument("output buffer too small");
        std::copy(o.begin(), o.end(), out);
      },
      err_index, msg, ml);
}

// read_matrix_market (matrix_market.hpp:59-121); nullptr + message on error.
void* ref_read_mm(const char* path, char* msg, int ml) {
  try {
    return new CscMatrix(read_matrix_market(path));
  } catch (const std::exception& e) {
    put_msg(msg, ml, e.what());
    return nullptr;
  }
}

// ---- config 5 (forward L then backward L^T) from the reference's primitives
// (the reference has no backward solve):
//   z = sptrsv(to_csr(lower_triangle(M)), b)                 kernels.hpp:335-342
//   B = permute_symmetric(transpose(lower_triangle(M)), rev) matrix.hpp:130-173
//   x'= sptrsv(to_csr(B), z'),  z'[n-1-i] = z[i],  x[i] = x'[n-1-i]
// out = z ++ x (collect_outputs layout of a solve pair).
int ref_fwd_bwd(int32_t n, const int32_t* colptr, const int32_t* rowidx, const double* values,
                const double* b, double* out, int32_t* err_index, char* msg, int ml) {
  return guarded(
      [&] {
        const CscMatrix L = lower_triangle(from_arrays(n, colptr, rowidx, values));
        const DenseVector z = sptrsv(to_csr(L), DenseVector(b, b + n));
        std::vector<Index> rev((size_t)n);
        for (Index i = 0; i < n; ++i)
          rev[(size_t)i] = n - 1 - i;
        const CscMatrix B = permute_symmetric(transpose(L), rev);
        DenseVector zr((size_t)n);
        for (Index i = 0; i < n; ++i)
          zr[(size_t)(n - 1 - i)] = z[(size_t)i];
        const DenseVector xr = sptrsv(to_csr(B), zr);
        for (Index i = 0; i < n; ++i) {
          out[i] = z[(size_t)i];
          out[n + i] = xr[(size_t)(n - 1 - i)];
        }
      },
      err_index, msg, ml);
}

// B = permute_symmetric(transpose(lower_triangle(M)), rev) as a matrix handle
void* ref_backward_matrix(int32_t n, const int32_t* colptr, const int32_t* rowidx,
                          const double* values) {
  try {
    const CscMatrix L = lower_triangle(from_arrays(n, colptr, rowidx, values));
    std::vector<Index> rev((size_t)n);
    for (Index i = 0; i < n; ++i)
      rev[(size_t)i] = n - 1 - i;
    return new CscMatrix(permute_symmetric(transpose(L), rev));
  } catch (...) {
    return nullptr;
  }
}

// One triangular solve L x = b on the reference's own parallel executor:
// kernel 1 of a combo-1 KernelState under its LBC schedule
// (build_kernel_schedule, executor.hpp:158-202) run by execute_unfused
// (executor.hpp:325-381) with an empty kernel-2 schedule.  The schedule is
// built once (the inspector); each run sets vin and returns x.
struct RefSolver {
  KernelState st;
  UnfusedSchedule us;
  Index nthreads = 1;
};

void* ref_solver_new(int32_t n, const int32_t* colptr, const int32_t* rowidx,
                     const double* values, int32_t nthreads, double* inspector_s) {
  try {
    auto* s = new RefSolver();
    s->st = make_state(1, from_arrays(n, colptr, rowidx, values), 7);
    s->nthreads = nthreads;
    const double t0 = now_s();
    s->us.k1 = build_kernel_schedule(build_g1(s->st), nthreads);
    if (inspector_s)
      *inspector_s = now_s() - t0;
    return s;
  } catch (...) {
    return nullptr;
  }
}

// runs the solve; *wall_s = ExecStats::wall_ns (the parallel region)
int ref_solver_run(void* h, const double* b, double* x, double* wall_s, int32_t* err_index,
                   char* msg, int ml) {
  auto* s = static_cast<RefSolver*>(h);
  return guarded(
      [&] {
        std::copy(b, b + s->st.n, s->st.vin.begin());
        const ExecStats es = execute_unfused(s->us, s->st, s->nthreads);
        if (wall_s)
          *wall_s = (double)es.wall_ns * 1e-9;
        if (x)
          std::copy(s->st.vmid.begin(), s->st.vmid.end(), x);
      },
      err_index, msg, ml);
}

void ref_solver_free(void* h) { delete static_cast<RefSolver*>(h); }

// A solver for the same pattern whose matrix differs only on the diagonal
// (config 5's systems: L_s = L + diag(delta_s)): copies the template's state
// and schedule, then sets row i's diagonal (stored last, trsv_csr_row) to
// diag[i].  Saves rebuilding the same DAG and LBC schedule per system.
void* ref_solver_clone_diag(void* h, const double* diag) {
  try {
    const auto* t = static_cast<RefSolver*>(h);
    auto* s = new RefSolver(*t);
    CsrMatrix& L = s->st.L_csr;
    for (Index i = 0; i < L.nrows; ++i)
      L.values[(size_t)L.rowptr[(size_t)i + 1] - 1] = diag[i];
    return s;
  } catch (...) {
    return nullptr;
  }
}

} // extern "C"
