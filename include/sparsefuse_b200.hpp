// sparsefuse_b200.hpp -- C++ mirror of the reference's inspector/executor API
// (namespace sparsefuse, proj/include/sparsefuse/*.hpp) over the C-ABI in
// sfgpu.h.  Header-only; link with -lsfgpu (paper_2111_12238_b200/libsfgpu.so).
//
// A caller of the reference switches with
//     namespace sparsefuse = sparsefuse_b200;
// and keeps its call sequence:
//     auto st = make_state(combo, M, seed);          // kernels.hpp:429
//     auto g1 = build_g1(st), g2 = build_g2(st);     // dag.hpp:319,339
//     auto f  = inter_dag(st);                       // dag.hpp:279
//     double reuse = compute_reuse(st);              // dag.hpp:398
//     auto sched = make_fused_schedule(st);          // msp + compile_schedule
//     execute_fused(sched, st);                      // executor.hpp:395
//     auto out = collect_outputs(st);                // kernels.hpp:585
// Differences, all deliberate:
//  * KernelState owns device memory (move-only); its operands are not public
//    std::vectors.  collect_outputs copies the results back.
//  * The fused schedule is built on the GPU by the inspector (level order of
//    the joint DAG, claimed by tickets) instead of msp (msp.hpp:825-1082); the
//    r / redundancy / nthreads arguments have no GPU meaning and are accepted
//    and ignored so call sites compile unchanged.
//  * joint_dag / level_info take the state (the GPU builds them); the
//    structures returned have the reference's layout and values bit for bit.
//  * No CPU fallback: without a CUDA device make_state throws NoDeviceError.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sfgpu.h"

namespace sparsefuse_b200 {

using Index = std::int32_t;
using Cost = std::int64_t;
using DenseVector = std::vector<double>;

// types.hpp:17-26 -- what() is "<message> at index <k>" like the reference.
class FactorizationError : public std::runtime_error {
public:
  FactorizationError(const std::string& what, Index index)
      : std::runtime_error(what), index_(index) {}
  Index index() const noexcept { return index_; }

private:
  Index index_;
};

// types.hpp:28-31
class InvalidMatrixError : public std::runtime_error {
public:
  using std::runtime_error::runtime_error;
};

class NoDeviceError : public std::runtime_error {
public:
  using std::runtime_error::runtime_error;
};

class CudaError : public std::runtime_error {
public:
  using std::runtime_error::runtime_error;
};

// types.hpp:33-36
class ParseError : public std::runtime_error {
public:
  using std::runtime_error::runtime_error;
};

// matrix.hpp:18-27
struct CscMatrix {
  Index nrows = 0;
  Index ncols = 0;
  std::vector<Index> colptr;
  std::vector<Index> rowidx;
  std::vector<double> values;
  Index nnz() const { return colptr.empty() ? 0 : colptr.back(); }
};

// dag.hpp:17-30
struct DepDag {
  Index nvert = 0;
  std::vector<Index> succptr;
  std::vector<Index> succ;
  std::vector<Cost> cost;
  Index nedges() const { return succptr.empty() ? 0 : succptr.back(); }
  Cost total_cost() const {
    Cost t = 0;
    for (Cost c : cost)
      t += c;
    return t;
  }
};

// dag.hpp:34-41
struct InterDep {
  Index nrows = 0;
  Index ncols = 0;
  std::vector<Index> rowptr;
  std::vector<Index> colidx;
  Index nnz() const { return rowptr.empty() ? 0 : rowptr.back(); }
};

// dag.hpp:43-48
struct LevelInfo {
  std::vector<Index> level;
  std::vector<Index> height;
  Index critical_path = 0;
  std::vector<Index> slack;
};

// executor.hpp:84-90 (timings of one GPU execution; no per-thread busy times)
struct ExecStats {
  std::int64_t wall_ns = 0;  // device time of the execution (CUDA events)
  Index barriers = 0;        // always 0: the executor has no barriers
  std::int64_t launches = 0; // kernels launched by the execution
};

namespace detail {

inline std::string last_message(const sfg_plan* p, std::int32_t* kind, std::int32_t* index) {
  char buf[512] = {0};
  *kind = 0;
  *index = -1;
  if (p)
    sfg_last_error(p, kind, index, buf, (std::int32_t)sizeof(buf));
  return std::string(buf);
}

inline void check(const sfg_plan* p, sfg_status st, const char* what) {
  if (st == SFG_OK)
    return;
  std::int32_t kind = 0, index = -1;
  std::string msg = last_message(p, &kind, &index);
  if (msg.empty())
    msg = what;
  switch (st) {
  case SFG_ERR_FACTORIZATION:
    throw FactorizationError(msg, index);
  case SFG_ERR_INVALID_MATRIX:
    throw InvalidMatrixError(msg);
  case SFG_ERR_INVALID_ARGUMENT:
    throw std::invalid_argument(msg);
  case SFG_ERR_LOGIC:
    throw std::logic_error(msg);
  case SFG_ERR_NO_DEVICE:
    throw NoDeviceError(msg);
  default:
    throw CudaError(msg);
  }
}

} // namespace detail

// kernels.hpp:409-427 -- one combination's operands and outputs, resident on
// the GPU.  nsys > 1 batches independent systems sharing M's pattern (combos
// 1 and 8).
class KernelState {
public:
  KernelState() = default;
  KernelState(const KernelState&) = delete;
  KernelState& operator=(const KernelState&) = delete;
  KernelState(KernelState&& o) noexcept { *this = std::move(o); }
  KernelState& operator=(KernelState&& o) noexcept {
    if (this != &o) {
      release();
      plan_ = o.plan_;
      combo_ = o.combo_;
      n = o.n;
      nsys_ = o.nsys_;
      nnz_m_ = o.nnz_m_;
      output_len_ = o.output_len_;
      inspected_ = o.inspected_;
      o.plan_ = nullptr;
    }
    return *this;
  }
  ~KernelState() { release(); }

  Index n = 0;
  int combo() const { return combo_; }
  Index nsys() const { return nsys_; }
  std::int64_t output_len() const { return output_len_; } // per system
  sfg_plan* handle() const { return plan_; }

  // st.vin = ... (kernels.hpp:420): nsys*n doubles, system-major
  void set_vin(const std::vector<double>& vin) {
    if ((std::int64_t)vin.size() != (std::int64_t)n * nsys_)
      throw std::invalid_argument("vin must hold nsys * n doubles");
    detail::check(plan_, sfg_set_vin(plan_, vin.data()), "set_vin");
  }
  // new matrix values, same pattern: nsys*nnz(M) doubles
  void set_values(const std::vector<double>& values) {
    if ((std::int64_t)values.size() != nnz_m_ * nsys_)
      throw std::invalid_argument("values must hold nsys * nnz(M) doubles");
    detail::check(plan_, sfg_set_values(plan_, values.data()), "set_values");
  }
  void inspect() {
    if (!inspected_) {
      detail::check(plan_, sfg_inspect(plan_), "inspect");
      inspected_ = true;
    }
  }

private:
  friend KernelState make_state(int, const CscMatrix&, std::uint64_t, Index,
                                const std::vector<double>*, const std::vector<double>*);
  void release() {
    if (plan_)
      sfg_plan_destroy(plan_);
    plan_ = nullptr;
  }
  sfg_plan* plan_ = nullptr;
  int combo_ = 0;
  Index nsys_ = 1;
  std::int64_t nnz_m_ = 0;
  std::int64_t output_len_ = 0;
  bool inspected_ = false;
};

// kernels.hpp:429-495.  values / vin (optional) hold nsys blocks; without vin
// system s uses gen_vector(n, seed + s).
inline KernelState make_state(int combo_id, const CscMatrix& M, std::uint64_t seed = 7,
                              Index nsys = 1, const std::vector<double>* values = nullptr,
                              const std::vector<double>* vin = nullptr) {
  if (M.nrows != M.ncols)
    throw InvalidMatrixError("combination input must be square");
  if (values && (std::int64_t)values->size() != (std::int64_t)M.nnz() * nsys)
    throw std::invalid_argument("values must hold nsys * nnz doubles");
  KernelState st;
  sfg_plan* p = nullptr;
  const sfg_status s =
      sfg_plan_create(combo_id, M.nrows, M.colptr.data(), M.rowidx.data(),
                      values ? values->data() : M.values.data(), nsys,
                      vin ? vin->data() : nullptr, seed, &p);
  if (s != SFG_OK) {
    std::int32_t kind = 0, index = -1;
    const std::string msg = detail::last_message(p, &kind, &index);
    if (p)
      sfg_plan_destroy(p);
    const std::string m = msg.empty() ? std::string("make_state") : msg;
    if (s == SFG_ERR_FACTORIZATION) // combo 3's scaling_vector (kernels.hpp:299-309)
      throw FactorizationError(m, index);
    if (s == SFG_ERR_INVALID_MATRIX)
      throw InvalidMatrixError(m);
    if (s == SFG_ERR_INVALID_ARGUMENT)
      throw std::invalid_argument(m);
    if (s == SFG_ERR_NO_DEVICE)
      throw NoDeviceError(m);
    throw CudaError(m);
  }
  st.plan_ = p;
  st.combo_ = combo_id;
  st.n = M.nrows;
  st.nsys_ = nsys;
  st.nnz_m_ = M.nnz();
  std::int32_t c = 0, nn = 0, ns = 0;
  std::int64_t nnzf = 0, olen = 0;
  detail::check(p, sfg_plan_info(p, &c, &nn, &ns, &nnzf, &olen), "plan_info");
  st.output_len_ = olen;
  return st;
}

namespace detail {
inline DepDag get_dag(KernelState& st, std::int32_t which) {
  st.inspect();
  DepDag g;
  std::int64_t ne = 0;
  check(st.handle(), sfg_get_dag(st.handle(), which, &g.nvert, &ne, nullptr, nullptr, nullptr),
        "get_dag");
  g.succptr.resize((size_t)g.nvert + 1);
  g.succ.resize((size_t)ne);
  g.cost.resize((size_t)g.nvert);
  check(st.handle(),
        sfg_get_dag(st.handle(), which, &g.nvert, &ne, g.succptr.data(), g.succ.data(),
                    g.cost.data()),
        "get_dag");
  return g;
}
} // namespace detail

// dag.hpp:319-370
inline DepDag build_g1(KernelState& st) { return detail::get_dag(st, 1); }
inline DepDag build_g2(KernelState& st) { return detail::get_dag(st, 2); }
// joint_dag(g1, g2, f) (dag.hpp:222-238) as built by the GPU inspector
inline DepDag joint_dag(KernelState& st) { return detail::get_dag(st, 3); }

// dag.hpp:279-317
inline InterDep inter_dag(KernelState& st) {
  st.inspect();
  InterDep f;
  std::int64_t nnz = 0;
  detail::check(st.handle(),
                sfg_get_interdep(st.handle(), &f.nrows, &f.ncols, &nnz, nullptr, nullptr),
                "inter_dag");
  f.rowptr.resize((size_t)f.nrows + 1);
  f.colidx.resize((size_t)nnz);
  detail::check(st.handle(),
                sfg_get_interdep(st.handle(), &f.nrows, &f.ncols, &nnz, f.rowptr.data(),
                                 f.colidx.data()),
                "inter_dag");
  return f;
}

// level_info (dag.hpp:197-218) of G1 (which = 1), G2 (2) or the joint DAG (3)
inline LevelInfo level_info(KernelState& st, int which) {
  st.inspect();
  const std::int32_t nv = which == 3 ? 2 * st.n : st.n;
  LevelInfo li;
  li.level.resize((size_t)nv);
  li.height.resize((size_t)nv);
  li.slack.resize((size_t)nv);
  detail::check(st.handle(),
                sfg_get_levels(st.handle(), which, li.level.data(), li.height.data(),
                               li.slack.data(), &li.critical_path),
                "level_info");
  return li;
}

// dag.hpp:398-431
inline double compute_reuse(KernelState& st) {
  double r = 0.0;
  detail::check(st.handle(), sfg_compute_reuse(st.handle(), &r), "compute_reuse");
  return r;
}

// FusedSchedule (executor.hpp:138-150): the GPU inspector's ticket order --
// every (tag, iter) of both kernels in a linear extension of the joint DAG,
// grouped into wavefronts.  `interleaved` follows compile_schedule's rule
// (reuse >= 1, executor.hpp:240).
struct FusedSchedule {
  bool fusion = true;
  bool interleaved = false;
  std::vector<std::uint8_t> tags; // 1 = kernel-1 iteration, 2 = kernel-2
  std::vector<Index> iters;
  std::vector<std::int64_t> wave_ptr;
  Index nspartitions() const { return wave_ptr.empty() ? 0 : (Index)wave_ptr.size() - 1; }
};

// msp (msp.hpp:825-1082) + compile_schedule (executor.hpp:235-268)
inline FusedSchedule make_fused_schedule(KernelState& st, Index /*r*/ = 0,
                                         double /*redundancy*/ = 2.0) {
  st.inspect();
  FusedSchedule fs;
  std::int64_t ne = 0;
  std::int32_t nw = 0;
  detail::check(st.handle(),
                sfg_get_schedule(st.handle(), &ne, nullptr, nullptr, &nw, nullptr), "schedule");
  fs.tags.resize((size_t)ne);
  fs.iters.resize((size_t)ne);
  fs.wave_ptr.resize((size_t)nw + 1);
  detail::check(st.handle(),
                sfg_get_schedule(st.handle(), &ne, fs.tags.data(), fs.iters.data(), &nw,
                                 fs.wave_ptr.data()),
                "schedule");
  fs.interleaved = compute_reuse(st) >= 1.0;
  return fs;
}

// FusedEntry / FusedPartitioning (msp.hpp:19-63): the same schedule as nested
// s-partitions (run in order) of independent w-partitions (ordered entries),
// checkable with the reference's validate_fused_partitioning.
struct FusedEntry {
  std::uint8_t tag = 1;
  Index iter = 0;
  bool dup = false;
};
struct FusedPartitioning {
  bool fusion = true;
  bool interleaved = false;
  double reuse_ratio = 0.0;
  Index n1 = 0, n2 = 0;
  std::vector<std::vector<std::vector<FusedEntry>>> spartitions;
  Index b() const { return static_cast<Index>(spartitions.size()); }
};

inline FusedPartitioning fused_partitioning(KernelState& st) {
  st.inspect();
  std::int32_t ns = 0;
  std::int64_t nw = 0, ne = 0;
  detail::check(st.handle(),
                sfg_get_partitioning(st.handle(), &ns, &nw, &ne, nullptr, nullptr, nullptr,
                                     nullptr),
                "partitioning");
  std::vector<std::int64_t> sp((size_t)ns + 1), wp((size_t)nw + 1);
  std::vector<std::uint8_t> tg((size_t)ne);
  std::vector<Index> it((size_t)ne);
  detail::check(st.handle(),
                sfg_get_partitioning(st.handle(), nullptr, nullptr, nullptr, sp.data(),
                                     wp.data(), tg.data(), it.data()),
                "partitioning");
  FusedPartitioning V;
  V.reuse_ratio = compute_reuse(st);
  V.interleaved = V.reuse_ratio >= 1.0;
  V.n1 = V.n2 = st.n;
  V.spartitions.resize((size_t)ns);
  for (std::int32_t k = 0; k < ns; ++k)
    for (std::int64_t w = sp[(size_t)k]; w < sp[(size_t)k + 1]; ++w) {
      std::vector<FusedEntry> es;
      for (std::int64_t e = wp[(size_t)w]; e < wp[(size_t)w + 1]; ++e)
        es.push_back(FusedEntry{tg[(size_t)e], it[(size_t)e], false});
      V.spartitions[(size_t)k].push_back(std::move(es));
    }
  return V;
}

namespace detail {
inline ExecStats finish(KernelState& st, std::int64_t launches0) {
  detail::check(st.handle(), sfg_synchronize(st.handle()), "execute");
  float total = 0.f, kernel = 0.f;
  detail::check(st.handle(), sfg_last_exec_ms(st.handle(), &total, &kernel), "execute");
  ExecStats es;
  es.wall_ns = (std::int64_t)((double)total * 1e6);
  es.launches = sfg_launch_count(st.handle()) - launches0;
  return es;
}
} // namespace detail

// executor.hpp:395-461 -- one fused launch; resets the outputs first (reset,
// kernels.hpp:498-502, is part of every execution).  Synchronous like the
// reference; FactorizationError carries the failing index.
inline ExecStats execute_fused(const FusedSchedule& /*sched*/, KernelState& st,
                               Index /*nthreads*/ = 0) {
  st.inspect();
  const std::int64_t l0 = sfg_launch_count(st.handle());
  detail::check(st.handle(), sfg_execute_fused(st.handle()), "execute_fused");
  return detail::finish(st, l0);
}

// executor.hpp:325-383 -- kernel 1 in one launch, then kernel 2
inline ExecStats execute_unfused(KernelState& st, Index /*nthreads*/ = 0) {
  st.inspect();
  const std::int64_t l0 = sfg_launch_count(st.handle());
  detail::check(st.handle(), sfg_execute_unfused(st.handle()), "execute_unfused");
  return detail::finish(st, l0);
}

// One kernel of the pair alone (1 or 2): the halves of execute_unfused, for
// callers that move data between them (config 1's row-sharded SpMV).
inline void execute_kernel(KernelState& st, int which) {
  detail::check(st.handle(), sfg_execute_kernel(st.handle(), which), "execute_kernel");
}

// y[0:r1-r0] = A[r0:r1, :] x on device pointers, bit-identical with combo 4's
// kernel 2 rows (spmv_csc_col, kernels.hpp:162-168).
inline void spmv_rows(KernelState& st, std::int32_t r0, std::int32_t r1, const double* x_device,
                      double* y_device) {
  detail::check(st.handle(), sfg_spmv_rows(st.handle(), r0, r1, x_device, y_device),
                "spmv_rows");
}

// K executions with new right-hand sides (vin[k]: nsys*n doubles), transfers
// overlapped with compute (sfg_execute_batch_ex).  out[k] receives the
// collect_outputs layout (nsys*output_len doubles) or, with final_only,
// kernel 2's output only (nsys*n doubles).  Page-locked buffers
// (sfg_host_alloc) give the overlap; any host memory is correct.
inline void execute_batch(KernelState& st, const std::vector<const double*>& vin,
                          const std::vector<double*>& out, bool final_only = false) {
  if (vin.size() != out.size())
    throw std::invalid_argument("one output buffer per input");
  detail::check(st.handle(),
                sfg_execute_batch_ex(st.handle(), (std::int32_t)vin.size(), vin.data(), out.data(),
                                     final_only ? SFG_OUTPUTS_FINAL : SFG_OUTPUTS_ALL),
                "execute_batch");
}

// kernels.hpp:498-502: a no-op -- every execution re-initialises its outputs
inline void reset(KernelState&) {}

// kernels.hpp:585-608, all systems concatenated system-major
inline std::vector<double> collect_outputs(KernelState& st) {
  std::vector<double> out((size_t)(st.output_len() * st.nsys()));
  detail::check(st.handle(),
                sfg_collect_outputs(st.handle(), out.data(), (std::int64_t)out.size()),
                "collect_outputs");
  return out;
}

namespace detail {
inline CscMatrix from_handle(sfg_matrix* h) {
  CscMatrix M;
  std::int32_t n = 0;
  std::int64_t nnz = 0;
  sfg_matrix_dims(h, &n, &nnz);
  M.nrows = M.ncols = n;
  M.colptr.resize((size_t)n + 1);
  M.rowidx.resize((size_t)nnz);
  M.values.resize((size_t)nnz);
  sfg_matrix_copy(h, M.colptr.data(), M.rowidx.data(), M.values.data());
  sfg_matrix_free(h);
  return M;
}
} // namespace detail

// matrix_market.hpp:59-121 (coordinate real, general/symmetric; square)
inline CscMatrix read_matrix_market(const std::string& path) {
  sfg_matrix* h = nullptr;
  char msg[512] = {0};
  const sfg_status st = sfg_matrix_read_mm(path.c_str(), &h, msg, (std::int32_t)sizeof(msg));
  if (st == SFG_ERR_INVALID_MATRIX)
    throw InvalidMatrixError(msg);
  if (st != SFG_OK)
    throw ParseError(msg[0] ? msg : ("cannot read " + path).c_str());
  return detail::from_handle(h);
}

// matrix_market.hpp:123-138
inline void write_matrix_market(const CscMatrix& A, const std::string& path) {
  sfg_matrix* h = nullptr;
  if (sfg_matrix_from_csc(A.ncols, A.colptr.data(), A.rowidx.data(), A.values.data(), &h) !=
      SFG_OK)
    throw std::invalid_argument("bad CSC arrays");
  const sfg_status st = sfg_matrix_write_mm(h, path.c_str());
  sfg_matrix_free(h);
  if (st != SFG_OK)
    throw ParseError("write failed for " + path);
}

// matrix.hpp:135-173: B = P A P^T, row/column i of A -> perm[i] of B
inline CscMatrix permute_symmetric(const CscMatrix& A, const std::vector<Index>& perm) {
  if (A.nrows != A.ncols || (Index)perm.size() != A.ncols)
    throw InvalidMatrixError("permutation length mismatch");
  sfg_matrix* h = nullptr;
  if (sfg_matrix_from_csc(A.ncols, A.colptr.data(), A.rowidx.data(), A.values.data(), &h) !=
      SFG_OK)
    throw std::invalid_argument("bad CSC arrays");
  sfg_matrix* out = nullptr;
  const sfg_status st = sfg_matrix_permute(h, perm.data(), &out);
  sfg_matrix_free(h);
  if (st != SFG_OK)
    throw InvalidMatrixError("not a permutation");
  return detail::from_handle(out);
}

// fixtures.hpp:148-155
inline DenseVector gen_vector(Index n, std::uint64_t seed) {
  DenseVector v((size_t)n);
  detail::check(nullptr, sfg_gen_vector(n, seed, v.data()), "gen_vector");
  return v;
}

} // namespace sparsefuse_b200
