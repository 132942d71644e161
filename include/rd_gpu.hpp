// rd_gpu.hpp -- header-only C++17 layer over the rd_gpu C-ABI (rd_gpu.h) that
// mirrors the reference rd:: API (/root/reference/proj/include/rd/*.hpp): same
// function names, argument meaning and exception types.  This is what a
// maintainer of the reference includes to route the AMG-PCG path to the B200
// (INTEGRATION.md); status codes are rethrown as the exceptions the reference
// throws: RD_EINVAL -> std::invalid_argument, everything else ->
// std::runtime_error (subclass rd_gpu::Error keeps the code).
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "rd_gpu.h"

namespace rd_gpu {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void check(int rc, const rd_ctx* ctx) {
  if (rc == RD_OK) return;
  const std::string msg = rd_gpu_last_error(ctx);
  if (rc == RD_EINVAL) throw std::invalid_argument(msg);
  throw Error(rc, msg);
}

// ------------------------------------------------------------------ context
class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr) { check(rd_gpu_ctx_create(device, stream, &h_), nullptr); }
  ~Context() { rd_gpu_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  rd_ctx* get() const { return h_; }
  void synchronize() { check(rd_gpu_synchronize(h_), h_); }
  int64_t launch_count() const { return rd_gpu_launch_count(h_); }

 private:
  rd_ctx* h_ = nullptr;
};

inline Context& default_context() {
  static Context ctx(0);
  return ctx;
}

// host CSR view, the storage contract of rd::SpMat (types.hpp:14)
struct HostCsr {
  int rows = 0, cols = 0;
  std::vector<int32_t> row_ptr{0}, col_idx;
  std::vector<double> values;
};

// ------------------------------------------------------------------ matrices
class DeviceMatrix {
 public:
  DeviceMatrix() = default;
  DeviceMatrix(Context& ctx, int rows, int cols, int64_t nnz, const int32_t* rp, const int32_t* ci, const double* v)
      : ctx_(&ctx) {
    rd_csr* h = nullptr;
    check(rd_gpu_csr_create(ctx.get(), rows, cols, nnz, rp, ci, v, &h), ctx.get());
    h_ = std::shared_ptr<rd_csr>(h, rd_gpu_csr_free);
  }
  explicit DeviceMatrix(Context& ctx, const HostCsr& a)
      : DeviceMatrix(ctx, a.rows, a.cols, (int64_t)a.col_idx.size(), a.row_ptr.data(), a.col_idx.data(),
                     a.values.data()) {}
  // borrowed view (system / hierarchy keeps it alive through `owner`)
  DeviceMatrix(Context& ctx, const rd_csr* view, std::shared_ptr<void> owner)
      : ctx_(&ctx), view_(view), owner_(std::move(owner)) {}

  const rd_csr* get() const { return h_ ? h_.get() : view_; }
  int rows() const { int r; rd_gpu_csr_info(get(), &r, nullptr, nullptr); return r; }
  int cols() const { int c; rd_gpu_csr_info(get(), nullptr, &c, nullptr); return c; }
  int64_t nonZeros() const { int64_t z; rd_gpu_csr_info(get(), nullptr, nullptr, &z); return z; }
  HostCsr download() const {
    HostCsr a;
    a.rows = rows();
    a.cols = cols();
    a.row_ptr.resize(a.rows + 1);
    a.col_idx.resize(nonZeros());
    a.values.resize(nonZeros());
    check(rd_gpu_csr_download(get(), a.row_ptr.data(), a.col_idx.data(), a.values.data()), ctx_->get());
    return a;
  }
  Context& context() const { return *ctx_; }

 private:
  Context* ctx_ = nullptr;
  std::shared_ptr<rd_csr> h_;
  const rd_csr* view_ = nullptr;
  std::shared_ptr<void> owner_;
};

// ------------------------------------------------------------------ mesh / system
class TetMesh {
 public:
  TetMesh(Context& ctx, rd_mesh* h) : ctx_(&ctx), h_(h, rd_gpu_mesh_free) {}
  const rd_mesh* get() const { return h_.get(); }
  int n_vertices() const { int v; rd_gpu_mesh_info(get(), &v, nullptr, nullptr); return v; }
  int n_tets() const { int t; rd_gpu_mesh_info(get(), nullptr, &t, nullptr); return t; }
  Context& context() const { return *ctx_; }
  // mesh.hpp:13-24 arrays on the host
  std::vector<double> vertices() const {
    std::vector<double> x(3 * (size_t)n_vertices());
    check(rd_gpu_mesh_download(get(), x.data(), nullptr, nullptr), ctx_->get());
    return x;
  }
  std::vector<int32_t> tets() const {
    std::vector<int32_t> t(4 * (size_t)n_tets());
    check(rd_gpu_mesh_download(get(), nullptr, t.data(), nullptr), ctx_->get());
    return t;
  }
  std::vector<uint8_t> boundary_vertex() const {
    std::vector<uint8_t> b((size_t)n_vertices());
    check(rd_gpu_mesh_download(get(), nullptr, nullptr, b.data()), ctx_->get());
    return b;
  }
  std::vector<uint8_t> refinement_edge() const {
    std::vector<uint8_t> r((size_t)n_tets());
    check(rd_gpu_mesh_tags(get(), r.data(), nullptr), ctx_->get());
    return r;
  }
  std::vector<int32_t> generation() const {
    std::vector<int32_t> g((size_t)n_tets());
    check(rd_gpu_mesh_tags(get(), nullptr, g.data()), ctx_->get());
    return g;
  }

 private:
  Context* ctx_;
  std::shared_ptr<rd_mesh> h_;
};

// mesh.hpp:36
inline TetMesh build_structured_cube(int n, Context& ctx = default_context()) {
  rd_mesh* h = nullptr;
  check(rd_gpu_build_structured_cube(ctx.get(), n, &h), ctx.get());
  return TetMesh(ctx, h);
}

enum class Target { smooth = RD_TARGET_SMOOTH, box = RD_TARGET_BOX, nonzero_bc = RD_TARGET_NONZERO_BC,
                    ball = RD_TARGET_BALL, sine_random = RD_TARGET_SINE_RANDOM };

// assembly.hpp:24-31 FemSystem, resident in HBM
class FemSystem {
 public:
  FemSystem(Context& ctx, rd_system* h, double rho) : ctx_(&ctx), h_(h, rd_gpu_system_free), rho(rho) {
    K = DeviceMatrix(ctx, rd_gpu_system_matrix(h, 0), h_);
    M = DeviceMatrix(ctx, rd_gpu_system_matrix(h, 1), h_);
    A = DeviceMatrix(ctx, rd_gpu_system_matrix(h, 2), h_);
  }
  int n_dofs() const { return rd_gpu_system_n_dofs(h_.get()); }
  const rd_system* get() const { return h_.get(); }
  const double* f_device() const { return rd_gpu_system_load(h_.get()); }
  std::vector<double> f() const {
    std::vector<double> out(n_dofs());
    if (!out.empty()) check(rd_gpu_copy(ctx_->get(), out.data(), f_device(), 8 * out.size()), ctx_->get());
    return out;
  }

 private:
  Context* ctx_;
  std::shared_ptr<rd_system> h_;

 public:
  double rho;
  DeviceMatrix K, M, A;
};

// assembly.hpp:48
inline FemSystem build_system(const TetMesh& mesh, double rho, Target target, uint64_t seed = 0) {
  rd_system* h = nullptr;
  const rd_target t{static_cast<int>(target), seed};
  check(rd_gpu_build_system(mesh.context().get(), mesh.get(), rho, &t, &h), mesh.context().get());
  return FemSystem(mesh.context(), h, rho);
}

// ------------------------------------------------------------------ linalg / amg
// linalg.hpp:30
inline std::vector<double> spmv(const DeviceMatrix& A, const std::vector<double>& x) {
  if ((int)x.size() != A.cols()) throw std::invalid_argument("spmv: dimension mismatch");
  std::vector<double> y(A.rows());
  check(rd_gpu_spmv(A.context().get(), A.get(), x.data(), y.data()), A.context().get());
  return y;
}

// amg.hpp:29
inline std::pair<std::vector<uint8_t>, DeviceMatrix> coarsen_redblack(const DeviceMatrix& A) {
  std::vector<uint8_t> flags(A.rows());
  rd_csr* P = nullptr;
  check(rd_gpu_coarsen_redblack(A.context().get(), A.get(), flags.data(), &P), A.context().get());
  std::shared_ptr<rd_csr> own(P, rd_gpu_csr_free);
  return {std::move(flags), DeviceMatrix(A.context(), P, own)};
}

// amg.hpp:31
inline DeviceMatrix galerkin_coarse(const DeviceMatrix& A, const DeviceMatrix& P) {
  rd_csr* c = nullptr;
  check(rd_gpu_galerkin_coarse(A.context().get(), A.get(), P.get(), &c), A.context().get());
  std::shared_ptr<rd_csr> own(c, rd_gpu_csr_free);
  return DeviceMatrix(A.context(), c, own);
}

// amg.hpp:34
inline std::vector<double> sgs_sweep(const DeviceMatrix& A, const std::vector<double>& f, const std::vector<double>& u) {
  std::vector<double> out(A.rows());
  check(rd_gpu_sgs_sweep(A.context().get(), A.get(), f.data(), u.data(), out.data()), A.context().get());
  return out;
}

// amg.hpp:13-24, 36-42
class AmgHierarchy {
 public:
  AmgHierarchy(const DeviceMatrix& A, int coarsest_threshold = 64, int smoothing_steps = 1) : ctx_(&A.context()) {
    rd_amg* h = nullptr;
    check(rd_gpu_amg_setup(ctx_->get(), A.get(), coarsest_threshold, smoothing_steps, &h), ctx_->get());
    h_ = std::shared_ptr<rd_amg>(h, rd_gpu_amg_free);
  }
  int num_levels() const { return rd_gpu_amg_num_levels(h_.get()); }
  DeviceMatrix level(int l, int which = 0) const { return DeviceMatrix(*ctx_, rd_gpu_amg_level_matrix(h_.get(), l, which), h_); }
  std::vector<uint8_t> coarse_flag(int l) const {
    std::vector<uint8_t> f(level(l).rows());
    check(rd_gpu_amg_level_flags(h_.get(), l, f.data()), ctx_->get());
    return f;
  }
  rd_amg* get() const { return h_.get(); }
  Context& context() const { return *ctx_; }

 private:
  Context* ctx_;
  std::shared_ptr<rd_amg> h_;
};

inline AmgHierarchy build_amg(const DeviceMatrix& A, int coarsest_threshold = 64, int smoothing_steps = 1) {
  return AmgHierarchy(A, coarsest_threshold, smoothing_steps);
}

inline std::vector<double> amg_apply(const AmgHierarchy& h, const std::vector<double>& r) {
  std::vector<double> z(r.size());
  if (r.empty()) return z;
  check(rd_gpu_amg_apply(h.get(), r.data(), z.data()), h.context().get());
  return z;
}

// linalg.hpp:13-24
struct PcgReport {
  int iterations = 0;
  bool converged = false;
  std::vector<double> residual_history;
};
struct PcgResult {
  std::vector<double> x;
  PcgReport report;
};

// linalg.hpp:46-49 with apply_P = amg_precond(h) (h == nullptr: identity)
inline PcgResult pcg(const DeviceMatrix& A, const AmgHierarchy* h, const std::vector<double>& f, double tol = 1e-8,
                     int max_iter = 500) {
  PcgResult out;
  out.x.resize(f.size());
  std::vector<double> hist(max_iter > 0 ? max_iter : 1);
  rd_pcg_report rep{};
  check(rd_gpu_pcg(A.context().get(), A.get(), h ? h->get() : nullptr, f.data(), tol, max_iter, out.x.data(), &rep,
                   hist.data()),
        A.context().get());
  out.report.iterations = rep.iterations;
  out.report.converged = rep.converged != 0;
  out.report.residual_history.assign(hist.begin(), hist.begin() + rep.iterations);
  return out;
}

// linalg.hpp:11 rd::LinOp -- a fixed linear map, here y = op(x) on DEVICE vectors enqueued on the
// context's stream (rd_linop).  Built-ins (identity_precond, spmv_op, amg_precond, jacobi_precond)
// run fused inside pcg; LinOp::device wraps a callable on device pointers, LinOp::host the
// reference's own host-vector LinOp (a copy out and back around each application).
class LinOp {
 public:
  using DeviceFn = std::function<void(const double* x_dev, double* y_dev, int64_t n)>;
  using HostFn = std::function<std::vector<double>(const std::vector<double>&)>;
  LinOp() = default;
  LinOp(rd_linop op, Context* ctx, std::shared_ptr<void> keep) : op_(op), ctx_(ctx), keep_(std::move(keep)) {}

  static LinOp device(Context& ctx, DeviceFn fn) {
    auto f = std::make_shared<DeviceFn>(std::move(fn));
    return LinOp(rd_linop{&device_tramp, f.get()}, &ctx, f);
  }
  static LinOp host(Context& ctx, HostFn fn) {
    auto f = std::make_shared<HostFn>(std::move(fn));
    return LinOp(rd_linop{&host_tramp, f.get()}, &ctx, f);
  }
  // y = op(x) on host vectors (rd_gpu_linop_apply)
  std::vector<double> operator()(const std::vector<double>& x) const {
    Context& c = ctx_ ? *ctx_ : default_context();
    std::vector<double> y(x.size());
    if (!x.empty()) check(rd_gpu_linop_apply(c.get(), op_, (int64_t)x.size(), x.data(), y.data()), c.get());
    return y;
  }
  const rd_linop& c_op() const { return op_; }
  Context* context() const { return ctx_; }

 private:
  static int device_tramp(void* user, rd_ctx*, int64_t n, const double* x, double* y) {
    try {
      (*static_cast<DeviceFn*>(user))(x, y, n);
      return RD_OK;
    } catch (const Error& e) {
      return e.code;
    } catch (const std::invalid_argument&) {
      return RD_EINVAL;
    } catch (...) {
      return RD_ERUNTIME;
    }
  }
  static int host_tramp(void* user, rd_ctx* ctx, int64_t n, const double* x, double* y) {
    try {
      std::vector<double> hx((size_t)n);
      check(rd_gpu_copy(ctx, hx.data(), x, sizeof(double) * (size_t)n), ctx);
      const std::vector<double> hy = (*static_cast<HostFn*>(user))(hx);
      if ((int64_t)hy.size() != n) return RD_EINVAL;
      check(rd_gpu_copy(ctx, y, hy.data(), sizeof(double) * (size_t)n), ctx);
      return RD_OK;
    } catch (const Error& e) {
      return e.code;
    } catch (const std::invalid_argument&) {
      return RD_EINVAL;
    } catch (...) {
      return RD_ERUNTIME;
    }
  }
  rd_linop op_{nullptr, nullptr};
  Context* ctx_ = nullptr;
  std::shared_ptr<void> keep_;
};

// linalg.hpp:39 identity_precond()
inline LinOp identity_precond() {
  rd_linop op{};
  check(rd_gpu_linop_identity(&op), nullptr);
  return LinOp(op, nullptr, nullptr);
}
// linalg.cpp:104-106: the SpMat overload's operator [&A](x) { return spmv(A, x); }
inline LinOp spmv_op(const DeviceMatrix& A) {
  rd_linop op{};
  check(rd_gpu_linop_csr(A.get(), &op), A.context().get());
  return LinOp(op, &A.context(), std::make_shared<DeviceMatrix>(A));
}
// amg.hpp:42 amg_precond(h)
inline LinOp amg_precond(const AmgHierarchy& h) {
  rd_linop op{};
  check(rd_gpu_linop_amg(h.get(), &op), h.context().get());
  return LinOp(op, &h.context(), std::make_shared<AmgHierarchy>(h));
}
// linalg.hpp:40 jacobi_precond(A): throws std::runtime_error on a non-positive diagonal
inline LinOp jacobi_precond(const DeviceMatrix& A) {
  rd_jacobi* j = nullptr;
  check(rd_gpu_jacobi_create(A.context().get(), A.get(), &j), A.context().get());
  std::shared_ptr<rd_jacobi> keep(j, rd_gpu_jacobi_free);
  rd_linop op{};
  check(rd_gpu_linop_jacobi(j, &op), A.context().get());
  return LinOp(op, &A.context(), keep);
}

// linalg.hpp:46-47 pcg(apply_A, apply_P, f, tol, max_iter)
inline PcgResult pcg(const LinOp& apply_A, const LinOp& apply_P, const std::vector<double>& f, double tol = 1e-8,
                     int max_iter = 500) {
  Context& c = apply_A.context() ? *apply_A.context()
               : apply_P.context() ? *apply_P.context()
                                   : default_context();
  PcgResult out;
  out.x.resize(f.size());
  std::vector<double> hist(max_iter > 0 ? max_iter : 1);
  rd_pcg_report rep{};
  check(rd_gpu_pcg_linop(c.get(), (int64_t)f.size(), apply_A.c_op(), apply_P.c_op(), f.empty() ? nullptr : f.data(),
                         tol, max_iter, out.x.empty() ? nullptr : out.x.data(), &rep, hist.data()),
        c.get());
  out.report.iterations = rep.iterations;
  out.report.converged = rep.converged != 0;
  out.report.residual_history.assign(hist.begin(), hist.begin() + rep.iterations);
  return out;
}
// linalg.hpp:48-49 pcg(A, apply_P, f, tol, max_iter)
inline PcgResult pcg(const DeviceMatrix& A, const LinOp& apply_P, const std::vector<double>& f, double tol = 1e-8,
                     int max_iter = 500) {
  return pcg(spmv_op(A), apply_P, f, tol, max_iter);
}

// ------------------------------------------------------------------ adaptivity (adapt.hpp, mesh.hpp:40-44)
// mesh.hpp:44 bisect_marked: throws std::invalid_argument for an id outside [0, n_tets)
inline TetMesh bisect_marked(const TetMesh& mesh, const std::vector<int>& marked) {
  rd_mesh* h = nullptr;
  check(rd_gpu_bisect_marked(mesh.context().get(), mesh.get(), (int)marked.size(),
                             marked.empty() ? nullptr : marked.data(), &h),
        mesh.context().get());
  return TetMesh(mesh.context(), h);
}
// mesh.hpp:40 uniform_refine
inline TetMesh uniform_refine(const TetMesh& mesh) {
  rd_mesh* h = nullptr;
  check(rd_gpu_uniform_refine(mesh.context().get(), mesh.get(), &h), mesh.context().get());
  return TetMesh(mesh.context(), h);
}
// adapt.hpp:13-21
struct Estimate {
  std::vector<double> per_tet;
  double global = 0.0;
};
inline Estimate estimate(const TetMesh& mesh, const FemSystem& sys, const std::vector<double>& coeffs, Target target,
                         uint64_t seed = 0) {
  if ((int)coeffs.size() != sys.n_dofs()) throw std::invalid_argument("estimate: coefficient size mismatch");
  Estimate e;
  e.per_tet.resize((size_t)mesh.n_tets());
  const rd_target t{static_cast<int>(target), seed};
  check(rd_gpu_estimate(mesh.context().get(), mesh.get(), sys.get(), coeffs.empty() ? nullptr : coeffs.data(), &t,
                        e.per_tet.empty() ? nullptr : e.per_tet.data(), &e.global),
        mesh.context().get());
  return e;
}
// adapt.hpp:24
inline std::vector<int> mark_dorfler(const Estimate& est, double theta, Context& ctx = default_context()) {
  std::vector<int> m(est.per_tet.size());
  int k = 0;
  check(rd_gpu_mark_dorfler(ctx.get(), (int)est.per_tet.size(), est.per_tet.empty() ? nullptr : est.per_tet.data(),
                            theta, m.empty() ? nullptr : m.data(), &k),
        ctx.get());
  m.resize((size_t)k);
  return m;
}
// adapt.hpp:26-42
struct AdaptLevel {
  int level = 0, dofs = 0;
  double eta = 0.0, err_l2_sq = 0.0, err_hm1_sq = 0.0;
  int iterations = 0;
  double seconds = 0.0;
};
struct AdaptResult {
  TetMesh mesh;
  std::vector<double> coefficients;
  std::vector<AdaptLevel> history;
};
// adapt.hpp:44-47 with the AMG SystemSolver of bench.cpp:65-74 (solve_system, PrecondKind::amg, tol)
inline AdaptResult adaptive_solve(const TetMesh& initial, Target target, double rho, int dof_budget, double tol,
                                  double theta = 0.5, uint64_t seed = 0) {
  Context& ctx = initial.context();
  std::vector<rd_adapt_level> rows(256);
  int nl = 0;
  rd_mesh* fm = nullptr;
  std::vector<double> co(std::max(dof_budget, 1) * (size_t)16 + 4096);
  const rd_target t{static_cast<int>(target), seed};
  int rc = rd_gpu_adaptive_solve(ctx.get(), initial.get(), &t, rho, dof_budget, tol, theta, rows.data(),
                                 (int)rows.size(), &nl, &fm, co.data(), (int)co.size());
  check(rc, ctx.get());
  AdaptResult out{TetMesh(ctx, fm), {}, {}};
  for (int k = 0; k < nl && k < (int)rows.size(); ++k) {
    const rd_adapt_level& r = rows[(size_t)k];
    out.history.push_back(AdaptLevel{r.level, r.dofs, r.eta, r.err_l2_sq, r.err_hm1_sq, r.iterations, r.seconds});
  }
  const int nd = out.history.empty() ? 0 : out.history.back().dofs;
  if (nd > (int)co.size()) throw std::runtime_error("adaptive_solve: final solution larger than the staging buffer");
  out.coefficients.assign(co.begin(), co.begin() + nd);
  return out;
}

// bench.hpp:48-57 SolveOutcome / solve_system(..., PrecondKind::amg, ...)
struct SolveOutcome {
  std::vector<double> u;
  int iterations = 0;
  bool converged = false;
  double setup_seconds = 0.0;
  double solve_seconds = 0.0;
};

inline SolveOutcome solve_system_amg(const DeviceMatrix& A, const double* f, double tol) {
  SolveOutcome out;
  out.u.resize(A.rows());
  rd_solve_outcome o{};
  check(rd_gpu_solve_system_amg(A.context().get(), A.get(), f, tol, out.u.data(), &o), A.context().get());
  out.iterations = o.iterations;
  out.converged = o.converged != 0;
  out.setup_seconds = o.setup_seconds;
  out.solve_seconds = o.solve_seconds;
  return out;
}

inline SolveOutcome solve_system_amg(const FemSystem& sys, double tol) { return solve_system_amg(sys.A, sys.f_device(), tol); }

// assembly.hpp:59-61 l2_error / h1_semi_error with rd::manufactured_exact(rho) (target.cpp:45-58)
struct ErrorNorms {
  double l2 = 0.0, h1_semi = 0.0;
};
inline ErrorNorms error_norms(const TetMesh& mesh, const FemSystem& sys, const std::vector<double>& coeffs,
                              double rho) {
  if ((int)coeffs.size() != sys.n_dofs()) throw std::invalid_argument("error_norms: coefficient size mismatch");
  ErrorNorms e;
  check(rd_gpu_error_norms(mesh.context().get(), mesh.get(), sys.get(), coeffs.data(), rho, &e.l2, &e.h1_semi),
        mesh.context().get());
  return e;
}

// the same norms with a target field u_bar as the exact function (value and gradient):
// ||u_h - u_bar||_L2 and ||grad(u_h - u_bar)||_L2, the BASELINE error gates
inline ErrorNorms error_norms_target(const TetMesh& mesh, const FemSystem& sys, const std::vector<double>& coeffs,
                                     Target target, uint64_t seed = 0) {
  if ((int)coeffs.size() != sys.n_dofs()) throw std::invalid_argument("error_norms_target: coefficient size mismatch");
  ErrorNorms e;
  const rd_target t{static_cast<int>(target), seed};
  check(rd_gpu_error_norms_target(mesh.context().get(), mesh.get(), sys.get(), coeffs.data(), &t, &e.l2,
                                  &e.h1_semi),
        mesh.context().get());
  return e;
}

}  // namespace rd_gpu
