// test_api.cpp -- the C++ mirror of the reference API (include/sparsefuse_b200.hpp)
// driven the way the reference's own executor tests drive sparsefuse
// (test_executor.cpp:80-98,157-171): make_state -> DAGs -> fused schedule ->
// execute -> collect_outputs, checked bit for bit against the C oracle
// (oracle/sf_oracle.c, itself pinned to the reference's golden vectors).
// Without a device it checks that make_state refuses to run (no CPU fallback).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/sparsefuse_b200.hpp"
extern "C" {
#include "../../oracle/sf_oracle.h"
}

namespace sf = sparsefuse_b200;

static int failures = 0;
#define CHECK(c)                                                                        \
  do {                                                                                  \
    if (!(c)) {                                                                         \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);                           \
      ++failures;                                                                       \
    }                                                                                   \
  } while (0)

// 2-D 5-point Laplacian, a x a grid, natural order, diagonal `d` (CSC)
static sf::CscMatrix grid(int a, double d) {
  sf::CscMatrix M;
  const int n = a * a;
  M.nrows = M.ncols = n;
  M.colptr.push_back(0);
  for (int j = 0; j < n; ++j) {
    const int x = j % a, y = j / a;
    const int cand[5] = {y > 0 ? j - a : -1, x > 0 ? j - 1 : -1, j, x + 1 < a ? j + 1 : -1,
                         y + 1 < a ? j + a : -1};
    for (int i : cand)
      if (i >= 0) {
        M.rowidx.push_back(i);
        M.values.push_back(i == j ? d : -1.0 - 0.01 * ((i + 3 * j) % 7));
      }
    M.colptr.push_back((int)M.rowidx.size());
  }
  return M;
}

static std::vector<double> oracle_outputs(int combo, const sf::CscMatrix& M, int* err_index) {
  const int64_t len = orc_output_len(combo, M.nrows, M.colptr.data(), M.rowidx.data());
  std::vector<double> out((size_t)len);
  int32_t code = 0, idx = -1;
  const int64_t got = orc_run_sequential(combo, M.nrows, M.colptr.data(), M.rowidx.data(),
                                         M.values.data(), 7, nullptr, out.data(), len, &code, &idx);
  *err_index = got < 0 ? idx : -1;
  return out;
}

static void same_dag(const sf::DepDag& g, const orc_dag& w) {
  CHECK(g.nvert == w.nvert);
  CHECK((int64_t)g.succ.size() == w.nedges);
  CHECK(std::memcmp(g.succptr.data(), w.succptr, sizeof(int32_t) * (w.nvert + 1)) == 0);
  CHECK(std::memcmp(g.succ.data(), w.succ, sizeof(int32_t) * w.nedges) == 0);
  CHECK(std::memcmp(g.cost.data(), w.cost, sizeof(int64_t) * w.nvert) == 0);
}

int main(int argc, char** argv) {
  int32_t ndev = 0, nsm = 0;
  const bool device = sfg_device_check(&ndev, &nsm) == SFG_OK;
  const bool want_device = !(argc > 1 && std::strcmp(argv[1], "--no-device") == 0);
  sf::CscMatrix M = grid(24, 4.5);
  if (!device || !want_device) {
    if (!device) {
      bool threw = false;
      try {
        auto st = sf::make_state(1, M);
      } catch (const sf::NoDeviceError&) {
        threw = true;
      }
      CHECK(threw);
    }
    std::printf("%s (no device: %d)\n", failures ? "FAILED" : "OK", (int)!device);
    return failures ? 1 : 0;
  }
  for (int combo : {1, 2, 3, 4, 5, 6, 7, 8}) {
    auto st = sf::make_state(combo, M, 7);
    if (combo != 8) {
      orc_dag w1{}, w2{}, wj{};
      orc_interdep wf{};
      orc_build_g(combo, 1, M.nrows, M.colptr.data(), M.rowidx.data(), M.values.data(), &w1);
      orc_build_g(combo, 2, M.nrows, M.colptr.data(), M.rowidx.data(), M.values.data(), &w2);
      orc_inter_dag(combo, M.nrows, M.colptr.data(), M.rowidx.data(), M.values.data(), &wf);
      orc_joint_dag(&w1, &w2, &wf, &wj);
      same_dag(sf::build_g1(st), w1);
      same_dag(sf::build_g2(st), w2);
      same_dag(sf::joint_dag(st), wj);
      const sf::InterDep f = sf::inter_dag(st);
      CHECK(f.nnz() == wf.nnz);
      CHECK(std::memcmp(f.colidx.data(), wf.colidx, sizeof(int32_t) * wf.nnz) == 0);
      std::vector<int32_t> lv(wj.nvert), ht(wj.nvert), sl(wj.nvert);
      int32_t P = 0;
      orc_level_info(&wj, lv.data(), ht.data(), sl.data(), &P);
      const sf::LevelInfo li = sf::level_info(st, 3);
      CHECK(li.critical_path == P && li.level == lv && li.height == ht && li.slack == sl);
      CHECK(sf::compute_reuse(st) ==
            orc_compute_reuse(combo, M.nrows, M.colptr.data(), M.rowidx.data(), M.values.data()));
      orc_free_dag(&w1);
      orc_free_dag(&w2);
      orc_free_dag(&wj);
      orc_free_interdep(&wf);
    }
    const sf::FusedPartitioning V = sf::fused_partitioning(st);
    int64_t entries = 0;
    for (const auto& sp : V.spartitions)
      for (const auto& wp : sp)
        entries += (int64_t)wp.size();
    CHECK(V.b() > 0 && entries == 2 * (int64_t)M.nrows);
    const sf::FusedSchedule sched = sf::make_fused_schedule(st, 8);
    CHECK((int64_t)sched.entries.size() == 2 * (int64_t)M.nrows);
    int eidx = 0;
    const std::vector<double> want = oracle_outputs(combo, M, &eidx);
    CHECK(eidx == -1);
    const sf::ExecStats es = sf::execute_fused(sched, st, 8);
    CHECK(es.launches >= 1 && es.barriers == 0);
    CHECK(sf::collect_outputs(st) == want);
    sf::reset(st);
    {
      // reset (kernels.hpp:498-502): fac = fac0, vmid = vout = 0
      const std::vector<double> r0 = sf::collect_outputs(st);
      const size_t nf = r0.size() - (size_t)M.nrows;
      bool zeros = true;
      for (size_t q = (combo == 1 || combo == 2 || combo == 4 || combo == 8) ? 0 : nf;
           q < ((combo == 3 || combo == 7) ? 0 : r0.size()); ++q)
        zeros = zeros && r0[q] == 0.0;
      CHECK(zeros);
    }
    sf::execute_unfused(st);
    CHECK(sf::collect_outputs(st) == want);
    // the reference's canonical call sequence (fuse_demo.cpp:15-31)
    {
      const sf::DepDag g1 = sf::build_g1(st), g2 = sf::build_g2(st);
      const sf::InterDep f = sf::inter_dag(st);
      const double reuse = sf::compute_reuse(st);
      const sf::FusedPartitioning V2 = sf::msp(g1, g2, f, 4, reuse);
      CHECK(sf::validate_fused_partitioning(V2, g1, g2, f).empty());
      CHECK(V2.interleaved == (reuse >= 1.0));
      const sf::FusedSchedule s2 = sf::compile_schedule(V2, reuse, g1, g2, 4);
      sf::execute_fused(s2, st, 4);
      CHECK(sf::collect_outputs(st) == want);
      sf::execute_unfused(g1, g2, st, 4);
      CHECK(sf::collect_outputs(st) == want);
      const sf::ExecStats ws = sf::execute_joint_wavefront(g1, g2, f, st, 4);
      const std::vector<double> wout = sf::collect_outputs(st);
      if (combo == 4) { // CSC scatter with atomic adds in any order (kernels.hpp:162-168)
        double err = 0.0, mx = 0.0;
        for (size_t q = 0; q < want.size(); ++q) {
          err = std::max(err, std::abs(wout[q] - want[q]));
          mx = std::max(mx, std::abs(want[q]));
        }
        CHECK(err <= 1e-13 * std::max(1.0, mx));
      } else {
        CHECK(wout == want);
      }
      const sf::WavefrontSchedule wfs = sf::build_wavefront_schedule(g1, g2, f);
      CHECK(ws.barriers == (sf::Index)wfs.levels.size() - 1);
      sf::execute_sequential(st);
      CHECK(sf::collect_outputs(st) == want);
      // the same DAGs without their state: joint DAG, levels, msp and the
      // wavefront schedule are built from the structures alone
      sf::DepDag h1 = g1, h2 = g2;
      sf::InterDep hf = f;
      h1.origin = h2.origin = hf.origin = 0;
      const sf::DepDag hj = sf::joint_dag(h1, h2, hf), jj = sf::joint_dag(st);
      CHECK(hj.succptr == jj.succptr && hj.succ == jj.succ && hj.cost == jj.cost);
      const sf::LevelInfo hl = sf::level_info(hj), jl = sf::level_info(st, 3);
      CHECK(hl.level == jl.level && hl.height == jl.height && hl.slack == jl.slack &&
            hl.critical_path == jl.critical_path);
      const sf::WavefrontSchedule hw = sf::build_wavefront_schedule(h1, h2, hf);
      bool same_wf = hw.levels == wfs.levels && hw.entries.size() == wfs.entries.size();
      for (size_t q = 0; same_wf && q < hw.entries.size(); ++q)
        same_wf = hw.entries[q].tag == wfs.entries[q].tag && hw.entries[q].iter == wfs.entries[q].iter;
      CHECK(same_wf);
      const sf::FusedPartitioning V3 = sf::msp(h1, h2, hf, 3, reuse);
      CHECK(sf::validate_fused_partitioning(V3, h1, h2, hf).empty());
      const sf::FusedSchedule s3 = sf::compile_schedule(V3, reuse, h1, h2, 3);
      CHECK(s3.checked_for == 0);
      sf::execute_fused(s3, st, 3); // verified on the GPU, then run
      CHECK(sf::collect_outputs(st) == want);
      // a schedule that breaks a dependence is refused
      sf::FusedSchedule bad = s3;
      std::reverse(bad.entries.begin(), bad.entries.end());
      bool refused = false;
      try {
        sf::execute_fused(bad, st, 3);
      } catch (const std::invalid_argument&) {
        refused = true;
      }
      CHECK(refused == (g1.nedges() + g2.nedges() + f.nnz() > 0));
    }
    // the two halves of the unfused comparator
    sf::execute_kernel(st, 1);
    sf::execute_kernel(st, 2);
    CHECK(sf::collect_outputs(st) == want);
    if (combo != 3 && combo != 7) {
      // batched executions, both output modes, equal to the single run
      const std::vector<double> b = sf::gen_vector(M.nrows, 7);
      std::vector<double> all(2 * want.size()), fin(2 * (size_t)M.nrows);
      sf::execute_batch(st, {b.data(), b.data()}, {all.data(), all.data() + want.size()});
      sf::execute_batch(st, {b.data(), b.data()}, {fin.data(), fin.data() + M.nrows}, true);
      for (int k = 0; k < 2; ++k) {
        CHECK(std::equal(want.begin(), want.end(), all.begin() + (long)k * want.size()));
        CHECK(std::equal(want.end() - M.nrows, want.end(), fin.begin() + (long)k * M.nrows));
      }
    }
    std::printf("combo %d: %zu outputs bit-exact, %lld launches\n", combo, want.size(),
                (long long)es.launches);
  }
  // breakdown: IC0 of an indefinite matrix -> FactorizationError(column)
  {
    sf::CscMatrix B = grid(6, 1.0);
    int eidx = 0;
    oracle_outputs(5, B, &eidx);
    auto st = sf::make_state(5, B);
    bool threw = false;
    try {
      sf::execute_fused(sf::make_fused_schedule(st), st);
    } catch (const sf::FactorizationError& e) {
      threw = true;
      CHECK(e.index() == eidx);
      std::printf("breakdown: %s\n", e.what());
    }
    CHECK(threw && eidx >= 0);
  }
  // invalid matrix: zero diagonal
  {
    sf::CscMatrix Z = grid(5, 4.0);
    for (int p = Z.colptr[3]; p < Z.colptr[4]; ++p)
      if (Z.rowidx[p] == 3)
        Z.values[p] = 0.0;
    bool threw = false;
    try {
      auto st = sf::make_state(1, Z);
    } catch (const sf::InvalidMatrixError& e) {
      threw = true;
      CHECK(std::strstr(e.what(), "zero diagonal entry at column 3") != nullptr);
    }
    CHECK(threw);
  }
  std::printf("%s\n", failures ? "FAILED" : "OK");
  return failures ? 1 : 0;
}
