// Host-only checks of include/rd_gpu_harness.hpp (no GPU): the reference's table and CSV
// conventions (bench.cpp:31-51, 251-266, 297-321), config validation / JSON
// (bench.cpp:78-166), the rdbench failed-row rule (rdbench.cpp:19-32) and MatrixMarket I/O
// (io.cpp:14-97) incl. the from_triplets semantics of the reader (linalg.cpp:11-17).
// Prints one line per failure; exit code = failures.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <random>
#include <string>

#include "rd_gpu_harness.hpp"

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                               \
  do {                                                            \
    if (cond) {                                                   \
      ++g_pass;                                                   \
    } else {                                                      \
      ++g_fail;                                                   \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                             \
  } while (0)

template <class F>
static bool throws_invalid(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

using namespace rd_gpu;

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";
  {  // CSV: integer columns %lld, others %.6e, NaN blank (bench.cpp:41-51, 251-266)
    EocTable t;
    t.columns = {"rho", "n", "dofs", "iterations", "converged", "setup_seconds", "solve_seconds"};
    t.rows.push_back({1e-4, 8, 343, 5, 1, 0.00125, 2.5e-3});
    t.rows.push_back({1e-4, 16, 3375, 6, 0, std::numeric_limits<double>::quiet_NaN(), 1.0});
    const std::string csv = to_csv(t);
    CHECK(csv ==
          "rho,n,dofs,iterations,converged,setup_seconds,solve_seconds\n"
          "1.000000e-04,8,343,5,1,1.250000e-03,2.500000e-03\n"
          "1.000000e-04,16,3375,6,0,,1.000000e+00\n");
    CHECK(failed_rows(t) == 1);
    const std::string g = gnuplot_blocks(t, "rho");
    CHECK(g.find("# rho = 1.000000e-04\n") != std::string::npos && g.find("nan") != std::string::npos);
    CHECK(column_index(t, "dofs") == 2);
    bool oor = false;
    try {
      column_index(t, "l2_error");
    } catch (const std::out_of_range&) {
      oor = true;
    }
    CHECK(oor);
  }
  {  // validate (bench.cpp:78-97)
    ExperimentConfig c;
    CHECK(throws_invalid([&] { validate(c); }));  // empty rho list
    c.rho_list = {1.0};
    validate(c);
    c.rho_list = {-1.0};
    CHECK(throws_invalid([&] { validate(c); }));
    c.rho_list = {1.0};
    c.n_list = {0};
    CHECK(throws_invalid([&] { validate(c); }));
    c.n_list = {8};
    c.tol = 0.0;
    CHECK(throws_invalid([&] { validate(c); }));
    c.tol = 1e-8;
    c.theta = 1.5;
    CHECK(throws_invalid([&] { validate(c); }));
    c.theta = 0.5;
    c.precond = PrecondKind::bddc;
    c.p = 1;
    CHECK(throws_invalid([&] { validate(c); }));
    c.precond = PrecondKind::jacobi;
    c.p = 2;
    CHECK(throws_invalid([&] { run_precond_bench(c); }));  // bench.cpp:394-395: amg or bddc only
    CHECK(throws_invalid([&] { precond_from_name("ilu"); }));
    CHECK(throws_invalid([&] { example_from_name("ball"); }));
  }
  {  // config JSON round trip (bench.cpp:133-166)
    ExperimentConfig c;
    c.example = ExampleKind::nonzero_bc;
    c.rho_list = {1.0, 1e-2, 0.1};
    c.n_list = {8, 16};
    c.precond = PrecondKind::amg;
    c.tol = 1e-10;
    c.seed = 42;
    c.output = "out \"q\".csv";
    c.theta = 0.25;
    c.gnuplot = true;
    const std::string j = config_to_json(c);
    CHECK(j.find("\"example\": \"nonzero_bc\"") != std::string::npos);
    CHECK(j.rfind("{\n  \"example\"", 0) == 0);
    const ExperimentConfig d = config_from_json(j);
    CHECK(d.example == c.example && d.rho_list == c.rho_list && d.n_list == c.n_list && d.tol == c.tol);
    CHECK(d.seed == 42 && d.output == c.output && d.theta == 0.25 && d.gnuplot && d.precond == PrecondKind::amg);
    CHECK(config_to_json(d) == j);
    CHECK(throws_invalid([&] { config_from_json("{\"example\": \"smooth\"}"); }));  // missing keys
  }
  {  // MatrixMarket: %.17g round trip, 1-based, comments skipped (io.cpp:42-97)
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> u(-1e3, 1e3);
    std::vector<std::tuple<int, int, double>> trips;
    for (int k = 0; k < 300; ++k) trips.emplace_back(int(rng() % 40), int(rng() % 30), u(rng) * std::pow(10.0, int(rng() % 40) - 20));
    trips.emplace_back(3, 3, 0.0);  // an exact zero: pruned
    const HostCsr A = csr_from_triplets(40, 30, trips);
    const std::string p = dir + "/rd_harness_A.mtx";
    write_matrix_market(p, A);
    const HostCsr B = read_matrix_market(p);
    CHECK(B.rows == 40 && B.cols == 30 && B.row_ptr == A.row_ptr && B.col_idx == A.col_idx && B.values == A.values);
    std::vector<double> v(57);
    for (auto& x : v) x = u(rng) / 3.0;
    v[5] = -0.0;
    v[6] = 1e-308;
    const std::string pv = dir + "/rd_harness_v.mtx";
    write_vector_market(pv, v);
    const std::vector<double> w = read_vector_market(pv);
    CHECK(w.size() == v.size());
    bool same = w.size() == v.size();
    for (size_t k = 0; same && k < v.size(); ++k) same = std::memcmp(&w[k], &v[k], sizeof(double)) == 0;
    CHECK(same);
    // a hand-written file: comment lines, duplicate entries summed, a cancelling pair pruned
    const std::string ph = dir + "/rd_harness_h.mtx";
    {
      std::ofstream f(ph);
      f << "%%MatrixMarket matrix coordinate real general\n% a comment\n3 3 6\n1 1 2.5\n3 2 -1\n1 1 0.5\n"
           "2 3 4\n2 3 -4\n3 1 7\n";
    }
    const HostCsr H = read_matrix_market(ph);
    CHECK(H.row_ptr == std::vector<int32_t>({0, 1, 1, 3}));
    CHECK(H.col_idx == std::vector<int32_t>({0, 0, 1}) && H.values == std::vector<double>({3.0, 7.0, -1.0}));
    bool bad_header = false;
    try {
      std::ofstream(dir + "/rd_harness_bad.mtx") << "not a matrix\n";
      read_matrix_market(dir + "/rd_harness_bad.mtx");
    } catch (const std::runtime_error&) {
      bad_header = true;
    }
    CHECK(bad_header);
  }
  std::printf("harness checks: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
