// Exercises the C++ drop-in facade (include/dba/dba_b200.hpp) the way the
// reference's own tests use dba:: (tests/test_partition.cpp,
// tests/test_solver.cpp). `cpu` runs host-only parts, `gpu` also solves.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>

#include "dba/dba_b200.hpp"

#define CHECK(x)                                                 \
  do {                                                           \
    if (!(x)) {                                                  \
      std::fprintf(stderr, "CHECK failed: %s line %d\n", #x, __LINE__); \
      return 1;                                                  \
    }                                                            \
  } while (0)

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  dba::SyntheticOptions opt;
  opt.cameras = 20;
  opt.points = 80;
  opt.obs_per_point = 10;
  const auto problem = dba::generate_synthetic(opt);
  CHECK(problem.num_observations() == 800);
  // partition KATs: contiguous chunks, remainder to low ranks (dba/partition.hpp:76-103)
  const auto parts = dba::partition_edges(problem, 3);
  CHECK(parts.size() == 3);
  CHECK(parts[0].edge_ids.size() == 267 && parts[2].edge_ids.size() == 266);
  CHECK(parts[1].edge_ids.front() == 267);
  bool threw = false;
  try {
    dba::partition_edges(problem, 0);
  } catch (const dba::InvalidArgumentError&) {
    threw = true;
  }
  CHECK(threw);
  // predicted-size pool: host-only, lean variant below FP64, shards below the whole
  const std::uint64_t pool1 = dba::predict_memory(problem), pool_lean = dba::predict_memory(problem, 1, 0, true);
  CHECK(pool1 > 800u * 27 * 8 && pool_lean < pool1 && dba::predict_memory(problem, 3, 1) < pool1);
  // BAL text round trip and the ParseError contract (tests/test_problem.cpp:35-80)
  std::ostringstream bal;
  dba::serialize_bal(problem, bal);
  CHECK(bal.str().substr(0, bal.str().find('\n')) == "20 80 800");
  std::istringstream back(bal.str());
  std::vector<std::string> warnings;
  const auto again = dba::parse_bal<double>(back, &warnings);
  CHECK(warnings.empty());
  CHECK(again.num_observations() == 800 && again.packed_cameras() == problem.packed_cameras());
  std::ostringstream bal2;
  dba::serialize_bal(again, bal2);
  CHECK(bal2.str() == bal.str());
  std::istringstream bad("2 1 1\n5 0 0 0\n");
  threw = false;
  try {
    dba::parse_bal<float>(bad);
  } catch (const dba::ParseError& e) {
    threw = e.line() == 2 && std::string(e.what()).find("camera index 5") != std::string::npos;
  }
  CHECK(threw);
  if (gpu) {
    dba::SolverConfig cfg;
    cfg.max_iterations = 20;
    const auto st = dba::lm_solve(problem, cfg);
    CHECK(!st.history.empty());
    CHECK(st.cost < 0.1 * 40261.97);  // tests/test_solver.cpp:361-384
    double last = 1e300;
    for (const auto& r : st.history)
      if (r.accepted) {
        CHECK(r.cost <= last * (1 + 1e-12));
        last = r.cost;
      }
    cfg.workers = 2;
    const auto st2 = dba::lm_solve(problem, cfg);
    CHECK(st2.history.size() == st.history.size());
    std::printf("facade gpu ok: %d iterations, cost %.6e\n", st.iteration, st.cost);
  }
  std::printf("facade ok\n");
  return 0;
}
