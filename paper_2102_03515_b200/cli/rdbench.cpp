// rdbench -- the reference CLI's bench-precond and adapt subcommands (tools/rdbench.cpp:76-151,
// exit codes :121-125, :186-190) on the device path, through include/rd_gpu_harness.hpp.
//
//   rdbench bench-precond|adapt [--rho R...] [--n N...] [--precond amg] [--tol T] [--threads K]
//                         [--seed S] [--out PATH] [--example smooth|box|nonzero_bc] [--p P]
//                         [--budget B] [--theta X] [--gnuplot] [--config FILE.json]
//
// Defaults are the reference's (bench-precond: rho 1..1e-12, n 8 16 32, amg, tol 1e-8; adapt: rho
// 1e-2 1e-3 1e-4, budget 200000, box).  Output: the CSV of run_precond_bench, or the adaptive
// level history plus its eoc summary (or --gnuplot blocks), to stdout or --out.  Exit codes as
// the reference: 0 all rows converged, 1 some bench-precond row did not (the run still
// completes), 2 an exception (bad config, device error).  table-h, table-rho and export-vtk
// (convergence tables, VTK) are not part of the device path: exit 2.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "rd_gpu_harness.hpp"

namespace {

void emit(const std::string& text, const std::string& out_path) {  // rdbench.cpp:34-42
  if (out_path.empty()) {
    std::cout << text;
    return;
  }
  std::ofstream out(out_path);
  if (!out) throw std::runtime_error("cannot open output file " + out_path);
  out << text;
}

bool is_option(const std::string& a) { return a.size() > 2 && a[0] == '-' && a[1] == '-'; }

// CLI11-style: a vector option takes every following token up to the next --option
std::vector<std::string> values(const std::vector<std::string>& args, size_t& k) {
  std::vector<std::string> v;
  while (k + 1 < args.size() && !is_option(args[k + 1])) v.push_back(args[++k]);
  return v;
}

std::string one(const std::vector<std::string>& args, size_t& k) {
  const auto v = values(args, k);
  if (v.size() != 1) throw std::invalid_argument("option " + args[k - v.size()] + " takes one value");
  return v[0];
}

double to_d(const std::string& s) {
  size_t pos = 0;
  const double v = std::stod(s, &pos);
  if (pos != s.size()) throw std::invalid_argument("not a number: " + s);
  return v;
}
long long to_i(const std::string& s) {
  size_t pos = 0;
  const long long v = std::stoll(s, &pos);
  if (pos != s.size()) throw std::invalid_argument("not an integer: " + s);
  return v;
}

void usage() {
  std::cerr << "usage: rdbench bench-precond|adapt [--rho R...] [--n N...] [--precond amg] [--tol T]\n"
               "                             [--threads K] [--seed S] [--out PATH] [--example NAME]\n"
               "                             [--p P] [--budget B] [--theta X] [--gnuplot] [--config FILE]\n";
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  if (args.empty() || args[0] == "--help" || args[0] == "-h") {
    usage();
    return args.empty() ? 2 : 0;
  }
  try {
    const std::string cmd = args[0];
    if (cmd == "table-h" || cmd == "table-rho" || cmd == "export-vtk")
      throw std::invalid_argument(cmd + " is not part of the device path (convergence tables / VTK)");
    if (cmd != "bench-precond" && cmd != "adapt") throw std::invalid_argument("unknown subcommand " + cmd);
    const bool adapt = cmd == "adapt";
    rd_gpu::ExperimentConfig cfg;
    std::string precond = "amg", example = "smooth";
    if (adapt) {  // rdbench.cpp:99-104 defaults
      cfg.rho_list = {1e-2, 1e-3, 1e-4};
      cfg.dof_budget = 200000;
      example = "box";
    } else {  // rdbench.cpp:94-97 defaults
      cfg.rho_list = {1.0, 1e-2, 1e-4, 1e-6, 1e-8, 1e-10, 1e-12};
      cfg.n_list = {8, 16, 32};
    }
    for (size_t k = 1; k < args.size(); ++k) {
      const std::string& a = args[k];
      if (a == "--rho") {
        cfg.rho_list.clear();
        for (const auto& v : values(args, k)) cfg.rho_list.push_back(to_d(v));
      } else if (a == "--n") {
        cfg.n_list.clear();
        for (const auto& v : values(args, k)) cfg.n_list.push_back(static_cast<int>(to_i(v)));
      } else if (a == "--p") {
        cfg.p = static_cast<int>(to_i(one(args, k)));
      } else if (a == "--precond") {
        precond = one(args, k);
      } else if (a == "--tol") {
        cfg.tol = to_d(one(args, k));
      } else if (a == "--threads") {
        cfg.threads = static_cast<int>(to_i(one(args, k)));
      } else if (a == "--seed") {
        cfg.seed = static_cast<unsigned long>(to_i(one(args, k)));
      } else if (a == "--out") {
        cfg.output = one(args, k);
      } else if (a == "--budget") {
        cfg.dof_budget = static_cast<int>(to_i(one(args, k)));
      } else if (a == "--theta") {
        cfg.theta = to_d(one(args, k));
      } else if (a == "--example") {
        example = one(args, k);
      } else if (a == "--gnuplot") {
        cfg.gnuplot = true;
      } else if (a == "--config") {  // a config_to_json file (bench.cpp:150-166)
        std::ifstream in(one(args, k));
        if (!in) throw std::runtime_error("cannot open config file");
        std::stringstream ss;
        ss << in.rdbuf();
        cfg = rd_gpu::config_from_json(ss.str());
        precond = rd_gpu::precond_name(cfg.precond);
        example = rd_gpu::example_name(cfg.example);
      } else {
        throw std::invalid_argument("unknown option " + a);
      }
    }
    cfg.precond = rd_gpu::precond_from_name(precond);  // rdbench.cpp:55-59 finish()
    cfg.example = rd_gpu::example_from_name(example);
    rd_gpu::validate(cfg);
    if (adapt) {  // rdbench.cpp:140-151: the level history, then the eoc summary
      const rd_gpu::EocTable t = rd_gpu::run_adaptive_experiment(cfg);
      std::string text;
      if (cfg.gnuplot) {
        text = rd_gpu::gnuplot_blocks(t, "rho");
      } else {
        text = rd_gpu::to_csv(t) + "\n" + rd_gpu::to_csv(rd_gpu::adaptive_rho_summary(t));
      }
      emit(text, cfg.output);
      return 0;
    }
    const rd_gpu::EocTable t = rd_gpu::run_precond_bench(cfg);
    emit(cfg.gnuplot ? rd_gpu::gnuplot_blocks(t, "rho") : rd_gpu::to_csv(t), cfg.output);
    const int bad = rd_gpu::failed_rows(t);
    if (bad) {
      std::cerr << bad << " row(s) did not converge\n";
      return 1;
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  }
  return 0;
}
