// test_api.cpp -- the C++ mirror of the reference API (include/sparsefuse_b200.hpp)
// driven the way the reference's own executor tests drive sparsefuse
// (test_executor.cpp:80-98,157-171): make_state -> DAGs -> fused schedule ->
// execute -> collect_outputs, checked bit for bit against the C oracle
// (oracle/sf_oracle.c, itself pinned to the reference's golden vectors).
// Without a device it checks that make_state refuses to run (no CPU fallback).
#include <algorithm>
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
    CHECK((int64_t)sched.tags.size() == 2 * (int64_t)M.nrows);
    int eidx = 0;
    const std::vector<double> want = oracle_outputs(combo, M, &eidx);
    CHECK(eidx == -1);
    const sf::ExecStats es = sf::execute_fused(sched, st, 8);
    CHECK(es.launches >= 1 && es.barriers == 0);
    CHECK(sf::collect_outputs(st) == want);
    sf::reset(st);
    sf::execute_unfused(st);
    CHECK(sf::collect_outputs(st) == want);
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
