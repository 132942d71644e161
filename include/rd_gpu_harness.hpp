// rd_gpu_harness.hpp -- the reference's benchmark-harness surface for the AMG-PCG path
// (SURVEY.md §8(f)2), header-only C++17 over rd_gpu.hpp:
//
//   * ExperimentConfig, validate, config_to_json / config_from_json   (bench.hpp:17-35, bench.cpp:78-166)
//   * precond / example names, make_target                              (bench.cpp:99-175)
//   * solve_system (PrecondKind::amg on the device)                     (bench.cpp:185-241)
//   * EocTable, to_csv with the reference's cell conventions            (bench.cpp:36-51, 251-266)
//   * run_precond_bench -- the bench-precond rows                       (bench.cpp:392-423)
//   * MatrixMarket coordinate / array I/O, %.17g round trip            (io.cpp:14-97)
//
// Only what the device path serves is routed: bench-precond with the AMG preconditioner, and
// solve_system with AMG or Jacobi.  BDDC and the unpreconditioned (dense Cholesky) solver are
// not part of the north-star path and throw std::invalid_argument (the reference's exception
// type for a rejected config).
#pragma once

#include <algorithm>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "rd_gpu.hpp"

namespace rd_gpu {

enum class PrecondKind { none, jacobi, amg, bddc };
enum class ExampleKind { smooth, box, nonzero_bc };

// bench.hpp:17-30
struct ExperimentConfig {
  ExampleKind example = ExampleKind::smooth;
  std::vector<double> rho_list;
  std::vector<int> n_list;
  int dof_budget = 0;
  PrecondKind precond = PrecondKind::amg;
  int p = 2;
  double tol = 1e-8;
  int threads = 1;
  unsigned long seed = 0;
  std::string output;
  double theta = 0.5;
  bool gnuplot = false;
};

// bench.cpp:78-97
inline void validate(const ExperimentConfig& cfg) {
  if (cfg.rho_list.empty()) throw std::invalid_argument("config: rho_list must not be empty");
  for (double rho : cfg.rho_list)
    if (!(rho > 0.0)) throw std::invalid_argument("config: rho values must be positive");
  for (int n : cfg.n_list)
    if (n < 1) throw std::invalid_argument("config: mesh resolutions must be >= 1");
  if (!(cfg.tol > 0.0)) throw std::invalid_argument("config: tol must be positive");
  if (cfg.precond == PrecondKind::bddc && cfg.p < 2) throw std::invalid_argument("config: bddc requires p >= 2");
  if (cfg.threads < 1) throw std::invalid_argument("config: threads must be >= 1");
  if (!(cfg.theta > 0.0) || cfg.theta > 1.0) throw std::invalid_argument("config: theta must lie in (0, 1]");
  if (cfg.dof_budget < 0) throw std::invalid_argument("config: dof_budget must be >= 0");
}

// bench.cpp:99-131
inline std::string precond_name(PrecondKind k) {
  switch (k) {
    case PrecondKind::none: return "none";
    case PrecondKind::jacobi: return "jacobi";
    case PrecondKind::amg: return "amg";
    case PrecondKind::bddc: return "bddc";
  }
  throw std::logic_error("unknown preconditioner kind");
}
inline PrecondKind precond_from_name(const std::string& s) {
  if (s == "none") return PrecondKind::none;
  if (s == "jacobi") return PrecondKind::jacobi;
  if (s == "amg") return PrecondKind::amg;
  if (s == "bddc") return PrecondKind::bddc;
  throw std::invalid_argument("unknown preconditioner: " + s);
}
inline std::string example_name(ExampleKind k) {
  switch (k) {
    case ExampleKind::smooth: return "smooth";
    case ExampleKind::box: return "box";
    case ExampleKind::nonzero_bc: return "nonzero_bc";
  }
  throw std::logic_error("unknown example kind");
}
inline ExampleKind example_from_name(const std::string& s) {
  if (s == "smooth") return ExampleKind::smooth;
  if (s == "box") return ExampleKind::box;
  if (s == "nonzero_bc") return ExampleKind::nonzero_bc;
  throw std::invalid_argument("unknown example: " + s);
}
// bench.cpp:168-175
inline Target make_target(ExampleKind k) {
  switch (k) {
    case ExampleKind::smooth: return Target::smooth;
    case ExampleKind::box: return Target::box;
    case ExampleKind::nonzero_bc: return Target::nonzero_bc;
  }
  throw std::logic_error("unknown example kind");
}

// ------------------------------------------------------------------ config JSON
// config_to_json writes the reference's key order (nlohmann ordered_json, dump(2));
// config_from_json reads that flat schema back (every key required, as json::at does).
namespace detail {
inline std::string json_num(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  std::string s = buf;
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";  // nlohmann prints doubles with a '.'
  return s;
}
inline std::string json_str(const std::string& s) {
  std::string o = "\"";
  for (char ch : s) {
    if (ch == '"' || ch == '\\') o += '\\';
    o += ch;
  }
  return o + "\"";
}
struct JsonReader {
  const std::string& t;
  size_t i = 0;
  explicit JsonReader(const std::string& text) : t(text) {}
  void ws() {
    while (i < t.size() && std::isspace(static_cast<unsigned char>(t[i]))) ++i;
  }
  [[noreturn]] void fail(const std::string& what) {
    throw std::invalid_argument("config_from_json: " + what + " at offset " + std::to_string(i));
  }
  void expect(char ch) {
    ws();
    if (i >= t.size() || t[i] != ch) fail(std::string("expected '") + ch + "'");
    ++i;
  }
  bool peek(char ch) {
    ws();
    return i < t.size() && t[i] == ch;
  }
  std::string str() {
    expect('"');
    std::string o;
    while (i < t.size() && t[i] != '"') {
      if (t[i] == '\\' && i + 1 < t.size()) ++i;
      o += t[i++];
    }
    if (i >= t.size()) fail("unterminated string");
    ++i;
    return o;
  }
  double num() {
    ws();
    size_t j = i;
    while (j < t.size() && (std::isdigit(static_cast<unsigned char>(t[j])) || std::strchr("+-.eE", t[j]))) ++j;
    if (j == i) fail("expected a number");
    const double v = std::stod(t.substr(i, j - i));
    i = j;
    return v;
  }
  bool boolean() {
    ws();
    if (t.compare(i, 4, "true") == 0) {
      i += 4;
      return true;
    }
    if (t.compare(i, 5, "false") == 0) {
      i += 5;
      return false;
    }
    fail("expected true or false");
  }
  std::vector<double> nums() {
    std::vector<double> v;
    expect('[');
    if (peek(']')) {
      ++i;
      return v;
    }
    for (;;) {
      v.push_back(num());
      if (peek(',')) {
        ++i;
        continue;
      }
      expect(']');
      return v;
    }
  }
};
}  // namespace detail

// bench.cpp:133-148
inline std::string config_to_json(const ExperimentConfig& cfg) {
  auto list = [](const auto& v, bool as_int) {
    if (v.empty()) return std::string("[]");
    std::string s = "[\n";
    for (size_t k = 0; k < v.size(); ++k) {
      s += "    " + (as_int ? std::to_string(static_cast<long long>(v[k])) : detail::json_num(double(v[k])));
      s += k + 1 < v.size() ? ",\n" : "\n";
    }
    return s + "  ]";
  };
  std::string j = "{\n";
  j += "  \"example\": " + detail::json_str(example_name(cfg.example)) + ",\n";
  j += "  \"rho_list\": " + list(cfg.rho_list, false) + ",\n";
  j += "  \"n_list\": " + list(cfg.n_list, true) + ",\n";
  j += "  \"dof_budget\": " + std::to_string(cfg.dof_budget) + ",\n";
  j += "  \"precond\": " + detail::json_str(precond_name(cfg.precond)) + ",\n";
  j += "  \"p\": " + std::to_string(cfg.p) + ",\n";
  j += "  \"tol\": " + detail::json_num(cfg.tol) + ",\n";
  j += "  \"threads\": " + std::to_string(cfg.threads) + ",\n";
  j += "  \"seed\": " + std::to_string(cfg.seed) + ",\n";
  j += "  \"output\": " + detail::json_str(cfg.output) + ",\n";
  j += "  \"theta\": " + detail::json_num(cfg.theta) + ",\n";
  j += "  \"gnuplot\": " + std::string(cfg.gnuplot ? "true" : "false") + "\n";
  return j + "}\n";
}

// bench.cpp:150-166
inline ExperimentConfig config_from_json(const std::string& text) {
  detail::JsonReader r(text);
  ExperimentConfig cfg;
  bool seen[12] = {};
  const char* keys[12] = {"example", "rho_list", "n_list", "dof_budget", "precond", "p",
                          "tol",     "threads",  "seed",   "output",     "theta",   "gnuplot"};
  r.expect('{');
  if (!r.peek('}')) {
    for (;;) {
      const std::string k = r.str();
      r.expect(':');
      int idx = -1;
      for (int q = 0; q < 12; ++q)
        if (k == keys[q]) idx = q;
      switch (idx) {
        case 0: cfg.example = example_from_name(r.str()); break;
        case 1: cfg.rho_list = r.nums(); break;
        case 2: {
          cfg.n_list.clear();
          for (double v : r.nums()) cfg.n_list.push_back(static_cast<int>(v));
          break;
        }
        case 3: cfg.dof_budget = static_cast<int>(r.num()); break;
        case 4: cfg.precond = precond_from_name(r.str()); break;
        case 5: cfg.p = static_cast<int>(r.num()); break;
        case 6: cfg.tol = r.num(); break;
        case 7: cfg.threads = static_cast<int>(r.num()); break;
        case 8: cfg.seed = static_cast<unsigned long>(r.num()); break;
        case 9: cfg.output = r.str(); break;
        case 10: cfg.theta = r.num(); break;
        case 11: cfg.gnuplot = r.boolean(); break;
        default: r.fail("unknown key \"" + k + "\"");
      }
      seen[idx] = true;
      if (r.peek(',')) {
        ++r.i;
        continue;
      }
      break;
    }
  }
  r.expect('}');
  for (int q = 0; q < 12; ++q)
    if (!seen[q]) throw std::invalid_argument(std::string("config_from_json: missing key \"") + keys[q] + "\"");
  return cfg;
}

// ------------------------------------------------------------------ tables
// bench.hpp:63-70
struct EocTable {
  std::vector<std::string> columns;
  std::vector<std::vector<double>> rows;
};

// bench.cpp:31-51: integer columns print as %lld, everything else as %.6e, NaN blank
inline bool integer_column(const std::string& name) {
  return name == "n" || name == "p" || name == "level" || name == "dofs" || name == "iterations" ||
         name == "converged";
}
inline std::string format_cell(const std::string& name, double v, bool blank_nan) {
  if (std::isnan(v)) return blank_nan ? std::string() : std::string("nan");
  char buf[48];
  if (integer_column(name))
    std::snprintf(buf, sizeof buf, "%lld", static_cast<long long>(std::llround(v)));
  else
    std::snprintf(buf, sizeof buf, "%.6e", v);
  return buf;
}
// bench.cpp:251-266
inline std::string to_csv(const EocTable& t) {
  std::ostringstream out;
  for (size_t c = 0; c < t.columns.size(); ++c) out << (c ? "," : "") << t.columns[c];
  out << '\n';
  for (const auto& row : t.rows) {
    for (size_t c = 0; c < t.columns.size(); ++c) {
      if (c) out << ',';
      out << format_cell(t.columns[c], c < row.size() ? row[c] : std::numeric_limits<double>::quiet_NaN(), true);
    }
    out << '\n';
  }
  return out.str();
}
// bench.cpp:297-321: whitespace-separated blocks per value of group_col (two blank lines
// between blocks), NaN printed as "nan"
inline int column_index(const EocTable& t, const std::string& name);
inline std::string gnuplot_blocks(const EocTable& t, const std::string& group_col) {
  const int gc = column_index(t, group_col);
  std::ostringstream out;
  out << '#';
  for (const auto& c : t.columns) out << ' ' << c;
  out << '\n';
  bool have_group = false;
  double group = 0.0;
  for (const auto& row : t.rows) {
    const double g = row[static_cast<size_t>(gc)];
    if (!have_group || g != group) {
      if (have_group) out << "\n\n";
      out << "# " << group_col << " = " << format_cell(group_col, g, false) << '\n';
      group = g;
      have_group = true;
    }
    for (size_t c = 0; c < t.columns.size(); ++c) {
      if (c) out << ' ';
      out << format_cell(t.columns[c], c < row.size() ? row[c] : std::numeric_limits<double>::quiet_NaN(), false);
    }
    out << '\n';
  }
  return out.str();
}
// bench.cpp:268-273
inline int column_index(const EocTable& t, const std::string& name) {
  auto it = std::find(t.columns.begin(), t.columns.end(), name);
  if (it == t.columns.end()) throw std::out_of_range("table has no column named " + name);
  return static_cast<int>(it - t.columns.begin());
}
// rdbench.cpp:19-32: rows whose converged flag is 0
inline int failed_rows(const EocTable& t) {
  int c = -1;
  try {
    c = column_index(t, "converged");
  } catch (const std::out_of_range&) {
    return 0;
  }
  int bad = 0;
  for (const auto& row : t.rows)
    if (row[static_cast<size_t>(c)] == 0.0) ++bad;
  return bad;
}

// ------------------------------------------------------------------ solve_system / bench
// bench.cpp:185-241 for PrecondKind::amg and ::jacobi (the device path): timing excludes
// build_system, setup_seconds = build_amg / jacobi_precond, solve_seconds = pcg, empty systems
// converge immediately.  none (dense Cholesky) and bddc are not served by the device path.
inline SolveOutcome solve_system(const TetMesh& /*mesh*/, const FemSystem& sys, PrecondKind kind, int /*p*/,
                                 double tol) {
  if (kind == PrecondKind::amg) return solve_system_amg(sys, tol);
  if (kind != PrecondKind::jacobi)
    throw std::invalid_argument("solve_system: the " + precond_name(kind) +
                                " preconditioner is not served by the device path");
  SolveOutcome out;
  if (sys.n_dofs() == 0) {  // bench.cpp:188-192
    out.converged = true;
    return out;
  }
  using clk = std::chrono::steady_clock;
  const std::vector<double> f = sys.f();
  const auto t0 = clk::now();
  const LinOp P = jacobi_precond(sys.A);  // bench.cpp:205-207
  const auto t1 = clk::now();
  PcgResult res = pcg(sys.A, P, f, tol, 500);
  const auto t2 = clk::now();
  out.u = std::move(res.x);
  out.iterations = res.report.iterations;
  out.converged = res.report.converged;
  out.setup_seconds = std::chrono::duration<double>(t1 - t0).count();
  out.solve_seconds = std::chrono::duration<double>(t2 - t1).count();
  return out;
}

// bench.cpp:392-423: one row per (rho, n), rho outer; columns rho,n,dofs,iterations,converged,
// setup_seconds,solve_seconds
inline EocTable run_precond_bench(const ExperimentConfig& cfg, Context* ctx_opt = nullptr) {
  validate(cfg);
  if (cfg.precond != PrecondKind::amg && cfg.precond != PrecondKind::bddc)
    throw std::invalid_argument("preconditioner benchmark needs amg or bddc");
  if (cfg.n_list.empty()) throw std::invalid_argument("preconditioner benchmark needs a mesh list");
  if (cfg.precond == PrecondKind::bddc)
    throw std::invalid_argument("preconditioner benchmark: bddc is not part of the device path");
  const Target target = make_target(cfg.example);
  Context& ctx = ctx_opt ? *ctx_opt : default_context();  // after the config checks
  EocTable t;
  t.columns = {"rho", "n", "dofs", "iterations", "converged", "setup_seconds", "solve_seconds"};
  for (double rho : cfg.rho_list) {
    for (int n : cfg.n_list) {
      TetMesh mesh = build_structured_cube(n, ctx);
      FemSystem sys = build_system(mesh, rho, target);
      const SolveOutcome res = solve_system(mesh, sys, cfg.precond, cfg.p, cfg.tol);
      t.rows.push_back({rho, double(n), double(sys.n_dofs()), double(res.iterations), res.converged ? 1.0 : 0.0,
                        res.setup_seconds, res.solve_seconds});
    }
  }
  return t;
}

// ------------------------------------------------------------------ adaptive experiment (bench.cpp:425-474)
inline double eoc_generic(double e_prev, double e_cur, double x_prev, double x_cur) {  // bench.cpp:243-249
  const double nan = std::numeric_limits<double>::quiet_NaN();
  if (!(e_prev > 0.0) || !(e_cur > 0.0) || !(x_prev > 0.0) || !(x_cur > 0.0)) return nan;
  const double d = std::log(x_prev / x_cur);
  if (d == 0.0) return nan;
  return std::log(e_prev / e_cur) / d;
}

// bench.cpp:425-449: per rho, adaptive_solve from build_structured_cube(8) with the configured
// solver (the device path serves AMG), one row per level
inline EocTable run_adaptive_experiment(const ExperimentConfig& cfg, Context* ctx_opt = nullptr) {
  validate(cfg);
  if (cfg.example == ExampleKind::smooth)
    throw std::invalid_argument("adaptive experiment needs the box or nonzero_bc example");
  if (cfg.dof_budget < 1) throw std::invalid_argument("adaptive experiment needs a dof budget");
  if (cfg.precond != PrecondKind::amg)
    throw std::invalid_argument("adaptive experiment: the device path serves the amg solver (" +
                                precond_name(cfg.precond) + " requested)");
  const Target target = make_target(cfg.example);
  Context& ctx = ctx_opt ? *ctx_opt : default_context();
  const TetMesh initial = build_structured_cube(8, ctx);
  EocTable t;
  t.columns = {"rho", "level", "dofs", "eta", "l2_sq", "hm1_sq", "iterations", "seconds"};
  for (double rho : cfg.rho_list) {
    const AdaptResult res = adaptive_solve(initial, target, rho, cfg.dof_budget, cfg.tol, cfg.theta);
    for (const AdaptLevel& lv : res.history)
      t.rows.push_back({rho, double(lv.level), double(lv.dofs), lv.eta, lv.err_l2_sq, lv.err_hm1_sq,
                        double(lv.iterations), lv.seconds});
  }
  return t;
}

// bench.cpp:451-474: the last level of every rho group, with eoc columns over rho
inline EocTable adaptive_rho_summary(const EocTable& levels) {
  const int rc = column_index(levels, "rho"), dc = column_index(levels, "dofs");
  const int lc = column_index(levels, "l2_sq"), hc = column_index(levels, "hm1_sq");
  EocTable t;
  t.columns = {"rho", "dofs", "l2_sq", "l2_eoc", "hm1_sq", "hm1_eoc"};
  std::vector<std::vector<double>> finals;
  for (size_t i = 0; i < levels.rows.size(); ++i) {
    const bool last = i + 1 == levels.rows.size() || levels.rows[i + 1][(size_t)rc] != levels.rows[i][(size_t)rc];
    if (last) finals.push_back(levels.rows[i]);
  }
  const double nan = std::numeric_limits<double>::quiet_NaN();
  double prev_rho = nan, prev_l2 = nan, prev_hm1 = nan;
  for (const auto& row : finals) {
    const double rho = row[(size_t)rc], l2 = row[(size_t)lc], hm1 = row[(size_t)hc];
    t.rows.push_back({rho, row[(size_t)dc], l2, eoc_generic(prev_l2, l2, prev_rho, rho), hm1,
                      eoc_generic(prev_hm1, hm1, prev_rho, rho)});
    prev_rho = rho;
    prev_l2 = l2;
    prev_hm1 = hm1;
  }
  return t;
}

// ------------------------------------------------------------------ MatrixMarket (io.cpp)
namespace detail {
inline std::string fmt17(double v) {  // io.cpp:14-18
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}
inline std::string next_data_line(std::istream& in) {  // io.cpp:32-38
  std::string line;
  while (std::getline(in, line))
    if (!line.empty() && line[0] != '%') return line;
  throw std::runtime_error("unexpected end of MatrixMarket file");
}
}  // namespace detail

// io.cpp:42-48: coordinate real general, 1-based, values %.17g (exact round trip)
inline void write_matrix_market(const std::string& path, const HostCsr& A) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open for writing: " + path);
  out << "%%MatrixMarket matrix coordinate real general\n";
  out << A.rows << " " << A.cols << " " << A.col_idx.size() << "\n";
  for (int i = 0; i < A.rows; ++i)
    for (int k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k)
      out << i + 1 << " " << A.col_idx[k] + 1 << " " << detail::fmt17(A.values[k]) << "\n";
}

// linalg.cpp:11-17 from_triplets semantics: columns sorted per row, duplicates summed in
// file order, exact zeros pruned
inline HostCsr csr_from_triplets(int rows, int cols, const std::vector<std::tuple<int, int, double>>& trips) {
  for (const auto& e : trips)
    if (std::get<0>(e) < 0 || std::get<0>(e) >= rows || std::get<1>(e) < 0 || std::get<1>(e) >= cols)
      throw std::invalid_argument("from_triplets: index out of range");
  std::vector<std::vector<std::pair<int, double>>> r(static_cast<size_t>(rows));
  for (const auto& e : trips) {  // stable: duplicates keep their file order
    auto& row = r[static_cast<size_t>(std::get<0>(e))];
    row.emplace_back(std::get<1>(e), std::get<2>(e));
  }
  HostCsr A;
  A.rows = rows;
  A.cols = cols;
  A.row_ptr.assign(1, 0);
  for (auto& row : r) {
    std::stable_sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (size_t k = 0; k < row.size();) {
      double v = row[k].second;
      size_t q = k + 1;
      for (; q < row.size() && row[q].first == row[k].first; ++q) v += row[q].second;
      if (v != 0.0) {
        A.col_idx.push_back(row[k].first);
        A.values.push_back(v);
      }
      k = q;
    }
    A.row_ptr.push_back(static_cast<int32_t>(A.col_idx.size()));
  }
  return A;
}

// io.cpp:50-69
inline HostCsr read_matrix_market(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open for reading: " + path);
  std::string header;
  if (!std::getline(in, header) || header.rfind("%%MatrixMarket", 0) != 0)
    throw std::runtime_error("not a MatrixMarket file: " + path);
  if (header.find("coordinate") == std::string::npos) throw std::runtime_error("expected coordinate format: " + path);
  std::istringstream sizes(detail::next_data_line(in));
  long rows = 0, cols = 0, nnz = 0;
  sizes >> rows >> cols >> nnz;
  std::vector<std::tuple<int, int, double>> trips;
  trips.reserve(static_cast<size_t>(nnz));
  for (long k = 0; k < nnz; ++k) {
    std::istringstream entry(detail::next_data_line(in));
    long i = 0, j = 0;
    double v = 0.0;
    entry >> i >> j >> v;
    trips.emplace_back(static_cast<int>(i - 1), static_cast<int>(j - 1), v);
  }
  return csr_from_triplets(static_cast<int>(rows), static_cast<int>(cols), trips);
}

// io.cpp:71-76
inline void write_vector_market(const std::string& path, const std::vector<double>& v) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open for writing: " + path);
  out << "%%MatrixMarket matrix array real general\n";
  out << v.size() << " 1\n";
  for (double x : v) out << detail::fmt17(x) << "\n";
}

// io.cpp:78-97
inline std::vector<double> read_vector_market(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open for reading: " + path);
  std::string header;
  if (!std::getline(in, header) || header.rfind("%%MatrixMarket", 0) != 0)
    throw std::runtime_error("not a MatrixMarket file: " + path);
  if (header.find("array") == std::string::npos) throw std::runtime_error("expected array format: " + path);
  std::istringstream sizes(detail::next_data_line(in));
  long rows = 0, cols = 0;
  sizes >> rows >> cols;
  if (cols != 1) throw std::runtime_error("expected a single column: " + path);
  std::vector<double> v(static_cast<size_t>(rows));
  for (long i = 0; i < rows; ++i) {
    std::istringstream entry(detail::next_data_line(in));
    entry >> v[static_cast<size_t>(i)];
  }
  return v;
}

}  // namespace rd_gpu
