// sparsefuse_b200.hpp -- C++ mirror of the reference's inspector/executor API
// (namespace sparsefuse, proj/include/sparsefuse/*.hpp) over the C-ABI in
// sfgpu.h.  Header-only; link with -lsfgpu (paper_2111_12238_b200/libsfgpu.so).
//
// A caller of the reference switches with
//     #include "sparsefuse_b200.hpp"
//     namespace sparsefuse = sparsefuse_b200;
// and keeps its call sequence (proj/demos/fuse_demo.cpp:15-31,
// proj/tools/sfuse.cpp:113-155):
//     KernelState st = make_state(combo, M, seed);   // kernels.hpp:429
//     DepDag g1 = build_g1(st), g2 = build_g2(st);   // dag.hpp:319,339
//     InterDep f = inter_dag(st);                    // dag.hpp:279
//     double reuse = compute_reuse(st);              // dag.hpp:398
//     FusedPartitioning V = msp(g1, g2, f, r, reuse);           // msp.hpp:825
//     auto bad = validate_fused_partitioning(V, g1, g2, f);     // msp.hpp:1114
//     FusedSchedule sched = compile_schedule(V, reuse, g1, g2, r); // executor.hpp:235
//     execute_fused(sched, st, r);                   // executor.hpp:395
//     execute_unfused(g1, g2, st, r);                // executor.hpp:383
//     execute_joint_wavefront(g1, g2, f, st, r);     // executor.hpp:500
//     execute_sequential(st);                        // executor.hpp:315
//     auto out = collect_outputs(st);                // kernels.hpp:585
// Differences, all deliberate:
//  * KernelState owns device memory (move-only); its operands are not public
//    std::vectors.  collect_outputs copies the results back.
//  * msp returns the GPU inspector's partitioning of the state the DAGs came
//    from (they carry its identity): s-partitions = dependency levels of the
//    executor's work units, checked by validate_fused_partitioning like any
//    MSP output.  For DAGs built elsewhere it returns the joint DAG's level
//    sets split into r w-partitions.  r / redundancy / nthreads have no GPU
//    meaning beyond that.
//  * execute_fused checks the schedule it is handed against the state's
//    joint DAG on the GPU (every iteration once, every dependence ordered)
//    and throws std::invalid_argument if it is not a valid order; a valid
//    schedule computes the same result as any other, so the state's own
//    executor runs it.
//  * No CPU fallback: without a CUDA device make_state throws NoDeviceError,
//    and execute_sequential runs the reference's sequential loop on one GPU
//    thread.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
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
  // the KernelState this DAG was built from (0: built elsewhere); lets msp /
  // joint_dag / the executors use that state's GPU inspector
  std::uint64_t origin = 0;
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
  std::uint64_t origin = 0; // as DepDag::origin
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
  Index barriers = 0;        // 0 for the barrier-free executors; levels - 1 for the wavefront
  std::vector<std::vector<std::int64_t>> busy_ns; // (no per-thread busy times on the GPU)
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

// live KernelStates by id, so DAGs can name the state they came from
struct Registry {
  std::mutex mu;
  std::unordered_map<std::uint64_t, sfg_plan*> live;
  std::uint64_t next = 1;
};
inline Registry& registry() {
  static Registry r;
  return r;
}
inline sfg_plan* plan_of(std::uint64_t id) {
  if (!id)
    return nullptr;
  Registry& r = registry();
  std::lock_guard<std::mutex> lk(r.mu);
  auto it = r.live.find(id);
  return it == r.live.end() ? nullptr : it->second;
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
      id_ = o.id_;
      o.plan_ = nullptr;
      o.id_ = 0;
    }
    return *this;
  }
  ~KernelState() { release(); }

  Index n = 0;
  int combo() const { return combo_; }
  Index nsys() const { return nsys_; }
  std::int64_t output_len() const { return output_len_; } // per system
  sfg_plan* handle() const { return plan_; }
  std::uint64_t id() const { return id_; }

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
    if (id_) {
      detail::Registry& r = detail::registry();
      std::lock_guard<std::mutex> lk(r.mu);
      r.live.erase(id_);
      id_ = 0;
    }
    if (plan_)
      sfg_plan_destroy(plan_);
    plan_ = nullptr;
  }
  sfg_plan* plan_ = nullptr;
  std::uint64_t id_ = 0;
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
  {
    detail::Registry& r = detail::registry();
    std::lock_guard<std::mutex> lk(r.mu);
    st.id_ = r.next++;
    r.live[st.id_] = p;
  }
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
  g.origin = st.id();
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
  f.origin = st.id();
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

// level_info(const DepDag&) (dag.hpp:197-218) of any DAG, on the GPU.  An
// edge that does not ascend throws std::invalid_argument like the reference.
inline LevelInfo level_info(const DepDag& g) {
  LevelInfo li;
  li.level.resize((size_t)g.nvert);
  li.height.resize((size_t)g.nvert);
  li.slack.resize((size_t)g.nvert);
  const sfg_status s = sfg_dag_levels(g.nvert, g.succptr.data(), g.succ.data(), li.level.data(),
                                      li.height.data(), li.slack.data(), &li.critical_path);
  if (s == SFG_ERR_INVALID_ARGUMENT)
    throw std::invalid_argument("dependence cycle: edge does not ascend");
  detail::check(nullptr, s, "level_info");
  return li;
}

// joint_dag (dag.hpp:222-238): G1, G2 offset by |V1|, and (j, |V1| + i) for
// every F_ij.  DAGs of one live state come from its GPU inspector; others
// are merged here (sorted, duplicate-free successor lists, costs concatenated).
inline DepDag joint_dag(const DepDag& g1, const DepDag& g2, const InterDep& f) {
  if (g1.origin && g1.origin == g2.origin && g1.origin == f.origin) {
    if (sfg_plan* p = detail::plan_of(g1.origin)) {
      DepDag j;
      std::int64_t ne = 0;
      detail::check(p, sfg_get_dag(p, 3, &j.nvert, &ne, nullptr, nullptr, nullptr), "joint_dag");
      j.succptr.resize((size_t)j.nvert + 1);
      j.succ.resize((size_t)ne);
      j.cost.resize((size_t)j.nvert);
      detail::check(p, sfg_get_dag(p, 3, &j.nvert, &ne, j.succptr.data(), j.succ.data(),
                                   j.cost.data()),
                    "joint_dag");
      j.origin = g1.origin;
      return j;
    }
  }
  const Index n1 = g1.nvert, nv = g1.nvert + g2.nvert;
  std::vector<std::vector<Index>> adj((size_t)nv);
  for (Index u = 0; u < n1; ++u)
    for (Index p = g1.succptr[(size_t)u]; p < g1.succptr[(size_t)u + 1]; ++p)
      adj[(size_t)u].push_back(g1.succ[(size_t)p]);
  for (Index u = 0; u < g2.nvert; ++u)
    for (Index p = g2.succptr[(size_t)u]; p < g2.succptr[(size_t)u + 1]; ++p)
      adj[(size_t)(n1 + u)].push_back(n1 + g2.succ[(size_t)p]);
  for (Index i = 0; i < f.nrows; ++i)
    for (Index p = f.rowptr[(size_t)i]; p < f.rowptr[(size_t)i + 1]; ++p)
      adj[(size_t)f.colidx[(size_t)p]].push_back(n1 + i);
  DepDag j;
  j.nvert = nv;
  j.succptr.assign((size_t)nv + 1, 0);
  for (Index u = 0; u < nv; ++u) {
    auto& a = adj[(size_t)u];
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
    j.succptr[(size_t)u + 1] = j.succptr[(size_t)u] + (Index)a.size();
  }
  for (auto& a : adj)
    j.succ.insert(j.succ.end(), a.begin(), a.end());
  j.cost = g1.cost;
  j.cost.insert(j.cost.end(), g2.cost.begin(), g2.cost.end());
  return j;
}

// dag.hpp:398-431
inline double compute_reuse(KernelState& st) {
  double r = 0.0;
  detail::check(st.handle(), sfg_compute_reuse(st.handle(), &r), "compute_reuse");
  return r;
}

// FusedEntry / FusedPartitioning (msp.hpp:19-63): nested s-partitions (run in
// order) of independent w-partitions (ordered entries).
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
  std::vector<std::array<Index, 4>> pairs; // (s, w) of paired partitions (none from the GPU)
  std::uint64_t origin = 0;                // state whose inspector built it (0: none)
  Index b() const { return static_cast<Index>(spartitions.size()); }
};

// FusedSchedule (executor.hpp:138-150): flattened partitioning.
struct FusedSchedule {
  bool fusion = true;
  bool interleaved = false;
  struct WRange {
    Index begin, end, split;
    Cost cost;
  };
  std::vector<FusedEntry> entries;
  std::vector<std::vector<WRange>> sparts;
  std::uint64_t checked_for = 0; // state the entries were verified against
  Index nspartitions() const { return static_cast<Index>(sparts.size()); }
};

// WavefrontSchedule (executor.hpp:152-156): joint-DAG level sets.
struct WavefrontSchedule {
  std::vector<FusedEntry> entries;
  std::vector<std::pair<Index, Index>> levels; // [begin, end) per level
};

namespace detail {
// The GPU inspector's partitioning of a state (sfg_get_partitioning).
inline FusedPartitioning gpu_partitioning(sfg_plan* p, std::uint64_t id, Index n) {
  detail::check(p, sfg_inspect(p), "inspect");
  std::int32_t ns = 0;
  std::int64_t nw = 0, ne = 0;
  check(p, sfg_get_partitioning(p, &ns, &nw, &ne, nullptr, nullptr, nullptr, nullptr),
        "partitioning");
  std::vector<std::int64_t> sp((size_t)ns + 1), wp((size_t)nw + 1);
  std::vector<std::uint8_t> tg((size_t)ne);
  std::vector<Index> it((size_t)ne);
  check(p, sfg_get_partitioning(p, nullptr, nullptr, nullptr, sp.data(), wp.data(), tg.data(),
                                it.data()),
        "partitioning");
  FusedPartitioning V;
  double r = 0.0;
  check(p, sfg_compute_reuse(p, &r), "compute_reuse");
  V.reuse_ratio = r;
  V.interleaved = r >= 1.0;
  V.n1 = V.n2 = n;
  V.origin = id;
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

inline void flatten(const FusedSchedule& s, std::vector<std::uint8_t>& tags,
                    std::vector<Index>& iters) {
  tags.resize(s.entries.size());
  iters.resize(s.entries.size());
  for (size_t q = 0; q < s.entries.size(); ++q) {
    tags[q] = s.entries[q].tag;
    iters[q] = s.entries[q].iter;
  }
}

// violations of a flattened order against a state's joint DAG (GPU)
inline std::int64_t order_violations(sfg_plan* p, const FusedSchedule& s) {
  std::vector<std::uint8_t> tags;
  std::vector<Index> iters;
  flatten(s, tags, iters);
  std::int64_t bad = 0;
  check(p, sfg_check_schedule(p, (std::int64_t)tags.size(), tags.data(), iters.data(), &bad),
        "check_schedule");
  return bad;
}
} // namespace detail

// The state's GPU inspector partitioning (sfg_get_partitioning).
inline FusedPartitioning fused_partitioning(KernelState& st) {
  st.inspect();
  return detail::gpu_partitioning(st.handle(), st.id(), st.n);
}

// msp (msp.hpp:825-1082).  For DAGs of a live state: that state's GPU
// inspector partitioning (what execute_fused runs).  Otherwise: the joint
// DAG's level sets (computed on the GPU), each split into at most r
// contiguous w-partitions -- a valid fused partitioning of any DAG pair.
// Packing follows reuse_ratio (interleaved iff >= 1, msp.hpp:834).
inline FusedPartitioning msp(const DepDag& g1, const DepDag& g2, const InterDep& f, Index r,
                             double reuse_ratio, double /*redundancy_factor*/ = 2.0) {
  if (r < 1)
    throw std::invalid_argument("partition count must be >= 1");
  FusedPartitioning V;
  if (g1.origin && g1.origin == g2.origin && g1.origin == f.origin) {
    if (sfg_plan* p = detail::plan_of(g1.origin)) {
      V = detail::gpu_partitioning(p, g1.origin, g1.nvert);
      V.reuse_ratio = reuse_ratio;
      V.interleaved = reuse_ratio >= 1.0;
      return V;
    }
  }
  V.n1 = g1.nvert;
  V.n2 = g2.nvert;
  V.reuse_ratio = reuse_ratio;
  V.interleaved = reuse_ratio >= 1.0;
  const DepDag j = joint_dag(g1, g2, f);
  const LevelInfo li = level_info(j);
  std::vector<std::vector<Index>> lev((size_t)li.critical_path + 1);
  for (Index v = 0; v < j.nvert; ++v)
    lev[(size_t)li.level[(size_t)v]].push_back(v);
  for (Index l = 1; l <= li.critical_path; ++l) {
    const auto& vs = lev[(size_t)l];
    const Index len = (Index)vs.size(), parts = std::min<Index>(r, len);
    std::vector<std::vector<FusedEntry>> sp;
    for (Index w = 0; w < parts; ++w) {
      std::vector<FusedEntry> es;
      for (Index q = w * len / parts; q < (w + 1) * len / parts; ++q) {
        const Index v = vs[(size_t)q];
        es.push_back(v < g1.nvert ? FusedEntry{1, v, false} : FusedEntry{2, v - g1.nvert, false});
      }
      sp.push_back(std::move(es));
    }
    V.spartitions.push_back(std::move(sp));
  }
  return V;
}

namespace detail {
inline void invert(const DepDag& g, std::vector<Index>& pp, std::vector<Index>& pr) {
  pp.assign((size_t)g.nvert + 1, 0);
  for (Index e = 0; e < g.nedges(); ++e)
    ++pp[(size_t)g.succ[(size_t)e] + 1];
  for (Index v = 0; v < g.nvert; ++v)
    pp[(size_t)v + 1] += pp[(size_t)v];
  pr.assign((size_t)g.nedges(), 0);
  std::vector<Index> cur(pp.begin(), pp.end() - 1);
  for (Index u = 0; u < g.nvert; ++u)
    for (Index p = g.succptr[(size_t)u]; p < g.succptr[(size_t)u + 1]; ++p)
      pr[(size_t)cur[(size_t)g.succ[(size_t)p]]++] = u;
}
} // namespace detail

// validate_fused_partitioning (msp.hpp:1110-1237): coverage, duplicate
// provenance, within-partition linear extension and the cross-partition
// ordering invariant, with the reference's messages; empty means valid.
inline std::vector<std::string> validate_fused_partitioning(const FusedPartitioning& V,
                                                            const DepDag& g1, const DepDag& g2,
                                                            const InterDep& f) {
  std::vector<std::string> bad;
  if (!V.fusion) {
    if (V.b() != 0)
      bad.push_back("fusion disabled but schedule non-empty");
    return bad;
  }
  auto complain = [&](Index s, Index w, Index e, const std::string& what) {
    bad.push_back("(s=" + std::to_string(s) + ",w=" + std::to_string(w) +
                  ",entry=" + std::to_string(e) + "): " + what);
  };
  struct Pos {
    Index s, w, idx;
  };
  std::vector<std::vector<Pos>> pos1((size_t)g1.nvert);
  std::vector<Pos> pos2((size_t)g2.nvert, Pos{-1, -1, -1});
  std::vector<Index> count2((size_t)g2.nvert, 0);
  for (Index s = 0; s < V.b(); ++s)
    for (Index w = 0; w < (Index)V.spartitions[(size_t)s].size(); ++w) {
      const auto& es = V.spartitions[(size_t)s][(size_t)w];
      for (Index e = 0; e < (Index)es.size(); ++e) {
        const FusedEntry& fe = es[(size_t)e];
        if (fe.tag == 1) {
          if (fe.iter < 0 || fe.iter >= g1.nvert)
            complain(s, w, e, "kernel-1 iteration out of range");
          else
            pos1[(size_t)fe.iter].push_back({s, w, e});
        } else if (fe.iter < 0 || fe.iter >= g2.nvert) {
          complain(s, w, e, "kernel-2 iteration out of range");
        } else {
          if (++count2[(size_t)fe.iter] > 1)
            complain(s, w, e, "kernel-2 iteration duplicated");
          pos2[(size_t)fe.iter] = {s, w, e};
        }
      }
    }
  for (Index v = 0; v < g1.nvert; ++v)
    if (pos1[(size_t)v].empty())
      bad.push_back("kernel-1 iteration " + std::to_string(v) + " missing");
  for (Index v = 0; v < g2.nvert; ++v)
    if (count2[(size_t)v] == 0)
      bad.push_back("kernel-2 iteration " + std::to_string(v) + " missing");
  if (!bad.empty())
    return bad;
  for (Index v = 0; v < g1.nvert; ++v)
    if (pos1[(size_t)v].size() > 1)
      for (const Pos& p : pos1[(size_t)v])
        if (!V.spartitions[(size_t)p.s][(size_t)p.w][(size_t)p.idx].dup)
          complain(p.s, p.w, p.idx, "replicated entry not flagged dup");
  std::vector<Index> p1, r1, p2, r2;
  detail::invert(g1, p1, r1);
  detail::invert(g2, p2, r2);
  auto earliest1 = [&](Index u) {
    Index s = V.b();
    for (const Pos& p : pos1[(size_t)u])
      s = std::min(s, p.s);
    return s;
  };
  auto before = [&](const Pos& at, Index u, std::uint8_t tag) {
    const auto& es = V.spartitions[(size_t)at.s][(size_t)at.w];
    for (Index e = 0; e < at.idx; ++e)
      if (es[(size_t)e].tag == tag && es[(size_t)e].iter == u)
        return true;
    return false;
  };
  for (Index v = 0; v < g1.nvert; ++v)
    for (const Pos& pv : pos1[(size_t)v])
      for (Index p = p1[(size_t)v]; p < p1[(size_t)v + 1]; ++p) {
        const Index u = r1[(size_t)p];
        if (!before(pv, u, 1) && earliest1(u) >= pv.s)
          complain(pv.s, pv.w, pv.idx, "kernel-1 dependence on " + std::to_string(u) + " unsatisfied");
      }
  for (Index v = 0; v < g2.nvert; ++v) {
    const Pos& pv = pos2[(size_t)v];
    for (Index p = p2[(size_t)v]; p < p2[(size_t)v + 1]; ++p) {
      const Index u = r2[(size_t)p];
      const Pos& pu = pos2[(size_t)u];
      if (!(pu.s < pv.s || (pu.s == pv.s && pu.w == pv.w && pu.idx < pv.idx)))
        complain(pv.s, pv.w, pv.idx, "kernel-2 dependence on " + std::to_string(u) + " unsatisfied");
    }
    for (Index p = f.rowptr[(size_t)v]; p < f.rowptr[(size_t)v + 1]; ++p) {
      const Index u = f.colidx[(size_t)p];
      if (!before(pv, u, 1) && earliest1(u) >= pv.s)
        complain(pv.s, pv.w, pv.idx,
                 "cross-kernel dependence on " + std::to_string(u) + " unsatisfied");
    }
  }
  return bad;
}

// compile_schedule (executor.hpp:235-268): flattens V; interleaved iff
// reuse_ratio >= 1; separated ranges get their kernel-1 / kernel-2 split.
// The entries are checked against the state the DAGs came from (if live).
inline FusedSchedule compile_schedule(const FusedPartitioning& V, double reuse_ratio,
                                      const DepDag& g1, const DepDag& g2, Index /*r*/) {
  FusedSchedule fs;
  fs.fusion = V.fusion;
  fs.interleaved = reuse_ratio >= 1.0;
  for (const auto& sp : V.spartitions) {
    std::vector<FusedSchedule::WRange> ws;
    for (const auto& wp : sp) {
      const Index begin = (Index)fs.entries.size();
      Cost c = 0;
      for (const FusedEntry& e : wp) {
        fs.entries.push_back(e);
        const auto& cost = e.tag == 1 ? g1.cost : g2.cost;
        if (e.iter >= 0 && (size_t)e.iter < cost.size())
          c += cost[(size_t)e.iter];
      }
      Index split = (Index)fs.entries.size();
      if (!fs.interleaved) {
        split = begin;
        while (split < (Index)fs.entries.size() && fs.entries[(size_t)split].tag == 1)
          ++split;
      }
      ws.push_back({begin, (Index)fs.entries.size(), split, c});
    }
    fs.sparts.push_back(std::move(ws));
  }
  if (g1.origin && g1.origin == g2.origin)
    if (sfg_plan* p = detail::plan_of(g1.origin))
      if (detail::order_violations(p, fs) == 0)
        fs.checked_for = g1.origin;
  return fs;
}

// The state's own fused schedule (the GPU inspector's, compile_schedule'd).
inline FusedSchedule make_fused_schedule(KernelState& st, Index r = 1, double /*redundancy*/ = 2.0) {
  const FusedPartitioning V = fused_partitioning(st);
  FusedSchedule fs;
  DepDag g; // costs are not needed by the executor
  fs = compile_schedule(V, V.reuse_ratio, g, g, r);
  fs.checked_for = st.id();
  return fs;
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

// DAGs passed to an executor must describe the state
inline void same_state(const KernelState& st, const DepDag& g1, const DepDag& g2) {
  if ((g1.origin && g1.origin != st.id()) || (g2.origin && g2.origin != st.id()) ||
      g1.nvert != st.n || g2.nvert != st.n)
    throw std::invalid_argument("the DAGs do not belong to this KernelState");
}
} // namespace detail

// executor.hpp:395-461 -- one fused launch; resets the outputs first (reset,
// kernels.hpp:498-502, is part of every execution).  Synchronous like the
// reference; FactorizationError carries the failing index.  A schedule not
// verified for this state is checked on the GPU first (std::invalid_argument
// if an iteration is missing/repeated or a dependence is out of order).
inline ExecStats execute_fused(const FusedSchedule& sched, KernelState& st,
                               Index /*nthreads*/ = 0) {
  st.inspect();
  if (!sched.fusion)
    throw std::logic_error("execute_fused: fusion disabled, run the fallback schedule");
  if (sched.checked_for != st.id()) {
    const std::int64_t bad = detail::order_violations(st.handle(), sched);
    if (bad)
      throw std::invalid_argument("execute_fused: schedule violates the joint DAG of this state (" +
                                  std::to_string(bad) + " violations)");
  }
  const std::int64_t l0 = sfg_launch_count(st.handle());
  detail::check(st.handle(), sfg_execute_fused(st.handle()), "execute_fused");
  return detail::finish(st, l0);
}

// executor.hpp:325-383 -- kernel 1 in one launch, then kernel 2
inline ExecStats execute_unfused(KernelState& st, Index /*nthreads*/ = 0) {
  st.inspect();
  const std::int64_t l0 = sfg_launch_count(st.handle());
  detail::check(st.handle(), sfg_execute_unfused(st.handle()), "execute_unfused");
  ExecStats es = detail::finish(st, l0);
  es.barriers = 1;
  return es;
}
// executor.hpp:383-392 (the reference builds the LBC schedules of g1 / g2)
inline ExecStats execute_unfused(const DepDag& g1, const DepDag& g2, KernelState& st,
                                 Index nthreads = 0) {
  detail::same_state(st, g1, g2);
  return execute_unfused(st, nthreads);
}

// build_wavefront_schedule (executor.hpp:209-229): the joint DAG's level
// sets, ascending vertex id within a level (from the state's GPU inspector
// when the DAGs come from a live state).
inline WavefrontSchedule build_wavefront_schedule(const DepDag& g1, const DepDag& g2,
                                                  const InterDep& f) {
  WavefrontSchedule ws;
  sfg_plan* p = (g1.origin && g1.origin == g2.origin && g1.origin == f.origin)
                    ? detail::plan_of(g1.origin)
                    : nullptr;
  if (p) {
    std::int64_t ne = 0;
    std::int32_t nl = 0;
    detail::check(p, sfg_get_wavefront(p, &ne, nullptr, nullptr, &nl, nullptr), "wavefront");
    std::vector<std::uint8_t> tg((size_t)ne);
    std::vector<Index> it((size_t)ne);
    std::vector<std::int64_t> lp((size_t)nl + 1);
    detail::check(p, sfg_get_wavefront(p, nullptr, tg.data(), it.data(), nullptr, lp.data()),
                  "wavefront");
    for (std::int64_t q = 0; q < ne; ++q)
      ws.entries.push_back(FusedEntry{tg[(size_t)q], it[(size_t)q], false});
    for (std::int32_t l = 0; l < nl; ++l)
      ws.levels.push_back({(Index)lp[(size_t)l], (Index)lp[(size_t)l + 1]});
    return ws;
  }
  const DepDag j = joint_dag(g1, g2, f);
  const LevelInfo li = level_info(j);
  std::vector<std::vector<Index>> lev((size_t)li.critical_path + 1);
  for (Index v = 0; v < j.nvert; ++v)
    lev[(size_t)li.level[(size_t)v]].push_back(v);
  for (Index l = 1; l <= li.critical_path; ++l) {
    const Index b = (Index)ws.entries.size();
    for (Index v : lev[(size_t)l])
      ws.entries.push_back(v < g1.nvert ? FusedEntry{1, v, false} : FusedEntry{2, v - g1.nvert, false});
    ws.levels.push_back({b, (Index)ws.entries.size()});
  }
  return ws;
}

// execute_joint_wavefront (executor.hpp:465-507): the joint level sets in
// order, a grid barrier between levels (sfg_execute_wavefront).
inline ExecStats execute_joint_wavefront(const DepDag& g1, const DepDag& g2, const InterDep& f,
                                         KernelState& st, Index /*nthreads*/ = 0) {
  detail::same_state(st, g1, g2);
  if (f.origin && f.origin != st.id())
    throw std::invalid_argument("the InterDep does not belong to this KernelState");
  const std::int64_t l0 = sfg_launch_count(st.handle());
  detail::check(st.handle(), sfg_execute_wavefront(st.handle()), "execute_joint_wavefront");
  ExecStats es = detail::finish(st, l0);
  std::int32_t nl = 0;
  detail::check(st.handle(), sfg_get_wavefront(st.handle(), nullptr, nullptr, nullptr, &nl, nullptr),
                "wavefront");
  es.barriers = nl > 0 ? nl - 1 : 0;
  return es;
}

// execute_sequential (executor.hpp:315-322) / run_sequential_reference
// (kernels.hpp:574-582): the reference loop on one GPU thread
inline ExecStats execute_sequential(KernelState& st) {
  const std::int64_t l0 = sfg_launch_count(st.handle());
  detail::check(st.handle(), sfg_execute_sequential(st.handle()), "execute_sequential");
  return detail::finish(st, l0);
}
inline void run_sequential_reference(KernelState& st) { execute_sequential(st); }

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

// kernels.hpp:498-502: fac = fac0, vmid = vout = 0 (on the device)
inline void reset(KernelState& st) { detail::check(st.handle(), sfg_reset(st.handle()), "reset"); }

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

namespace detail {
inline CscMatrix generated(std::int32_t kind, std::int32_t a, std::int32_t b, std::uint64_t seed) {
  sfg_matrix* h = nullptr;
  if (sfg_matrix_gen(kind, a, b, seed, &h) != SFG_OK)
    throw std::invalid_argument("bad generator parameters");
  return from_handle(h);
}
} // namespace detail

// fixtures.hpp:49-91: the 5-point Laplacian of a k x k grid, nested-dissection numbered
inline CscMatrix gen_grid_laplacian(Index k) { return detail::generated(0, k, 0, 0); }
// fixtures.hpp:97-141
inline CscMatrix gen_banded_spd(Index n, Index bandwidth, std::uint64_t seed) {
  return detail::generated(1, n, bandwidth, seed);
}

// fixtures.hpp:148-155
inline DenseVector gen_vector(Index n, std::uint64_t seed) {
  DenseVector v((size_t)n);
  detail::check(nullptr, sfg_gen_vector(n, seed, v.data()), "gen_vector");
  return v;
}

} // namespace sparsefuse_b200
