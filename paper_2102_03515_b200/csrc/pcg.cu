// pcg.cu -- device-resident preconditioned conjugate gradients (linalg.cpp:64-102).
//
// Every vector and scalar stays in HBM.  Per iteration:
//   spmv_dot      Ap = A p, pAp = p.Ap                 (fused SpMV epilogue)
//   pcg_xr        alpha = rz/pAp, x += alpha p, r -= alpha Ap   (one pass)
//   V-cycle       z = M^-1 r, rz_next = r.z            (fused into the last GS sweep)
//   pcg_check     rel = sqrt(rz_next/rz0), history, convergence / SPD checks, beta
//   pcg_p         p = z + beta p
// The host reads back one small status word per iteration.
#include <chrono>
#include <cmath>

#include "internal.hpp"

namespace rdg {

struct PcgState {
  double rz, rz0, pAp, rz_next, beta, rel;
  int done;    // 1 converged
  int status;  // 1: p'Ap <= 0, 2: r'z < 0 (both RD_ENOTSPD)
  int it;
};

namespace {

__global__ void pcg_init_kernel(PcgState* st) {
  pdl_wait();
  pdl_trigger();
  // rz already in st->rz (written by the dot)
  const double rz = st->rz;
  st->done = 0;
  st->status = 0;
  st->it = 0;
  if (rz < 0.0) {
    st->status = RD_ENOTSPD;
    return;
  }
  st->rz0 = rz;
  if (rz == 0.0) st->done = 1;
}

__global__ void pcg_xr_kernel(int64_t n, PcgState* st, const double* __restrict__ p, const double* __restrict__ Ap,
                              double* __restrict__ x, double* __restrict__ r) {
  pdl_wait();
  pdl_trigger();
  if (st->done || st->status) return;
  const double pAp = st->pAp;
  if (!(pAp > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st->status = 1;  // p'Ap <= 0
    return;
  }
  const double alpha = __ddiv_rn(st->rz, pAp);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    r[i] = __dsub_rn(r[i], __dmul_rn(alpha, Ap[i]));
  }
}

__global__ void pcg_check_kernel(PcgState* st, double tol, double* hist, int hist_cap) {
  pdl_wait();
  pdl_trigger();
  if (st->done || st->status) return;
  const double rzn = st->rz_next;
  if (rzn < 0.0) {
    st->status = 2;  // preconditioner lost positive definiteness
    return;
  }
  const double rel = __dsqrt_rn(__ddiv_rn(rzn, st->rz0));
  const int it = st->it + 1;
  st->it = it;
  st->rel = rel;
  if (hist && it - 1 < hist_cap) hist[it - 1] = rel;
  if (rel <= tol) {
    st->done = 1;
    return;
  }
  st->beta = __ddiv_rn(rzn, st->rz);
  st->rz = rzn;
}

__global__ void pcg_p_kernel(int64_t n, const PcgState* st, const double* __restrict__ z, double* __restrict__ p) {
  pdl_wait();
  pdl_trigger();
  if (st->done || st->status) return;
  const double beta = st->beta;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

int vec_grid(Ctx& c, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c.num_sms * 8, (n + 255) / 256));
}

}  // namespace

PcgResultDev pcg_ops(Ctx& c, int64_t n, const PcgOp& apply_A, const PcgOp& apply_P, const double* f, double tol,
                     int max_iter, double* x, double* hist_dev) {
  PcgResultDev out;
  if (n == 0) {
    out.converged = true;
    return out;
  }
  DBuf<double> r(n, c.stream), z(n, c.stream), p(n, c.stream), Ap(n, c.stream);
  DBuf<PcgState> st(1, c.stream);
  RDG_CUDA(cudaMemsetAsync(st.p, 0, sizeof(PcgState), c.stream));
  RDG_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c.stream));
  RDG_CUDA(cudaMemcpyAsync(r.p, f, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
  auto precond = [&](double* dot_out) { apply_P(r.p, z.p, dot_out); };
  precond(&st.p->rz);
  launch_pdl(pcg_init_kernel, 1, 1, 0, c.stream, st.p);
  ++c.launches;
  PcgState* hs = reinterpret_cast<PcgState*>(c.h_pinned);
  RDG_CUDA(cudaMemcpyAsync(hs, st.p, sizeof(PcgState), cudaMemcpyDeviceToHost, c.stream));
  RDG_CUDA(cudaStreamSynchronize(c.stream));
  if (hs->status) throw Error(RD_ENOTSPD, "pcg: preconditioner not positive definite");
  if (hs->done) {
    out.converged = true;
    return out;
  }
  RDG_CUDA(cudaMemcpyAsync(p.p, z.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
  const int g = vec_grid(c, n);
  // A p and the x / r update of iteration it are enqueued before the host waits on the
  // convergence check of iteration it - 1, so the GPU never idles across that round trip;
  // once converged they are no-ops (pcg_xr_kernel reads st->done; Ap and pAp are scratch)
  auto enqueue_ap_xr = [&]() {
    apply_A(p.p, Ap.p, &st.p->pAp);
    launch_pdl(pcg_xr_kernel, g, 256, 0, c.stream, n, st.p, p.p, Ap.p, x, r.p);
    ++c.launches;
  };
  static_assert(sizeof(PcgState) <= 8 * sizeof(double), "PcgState overlaps the pinned scratch");
  int* herr = reinterpret_cast<int*>(c.h_pinned + 10);
  if (max_iter >= 1) enqueue_ap_xr();  // max_iter <= 0: x stays 0 (linalg.cpp:66,77)
  for (int it = 1; it <= max_iter; ++it) {
    precond(&st.p->rz_next);
    launch_pdl(pcg_check_kernel, 1, 1, 0, c.stream, st.p, tol, hist_dev, max_iter);
    launch_pdl(pcg_p_kernel, g, 256, 0, c.stream, n, st.p, z.p, p.p);
    c.launches += 2;
    RDG_CUDA(cudaMemcpyAsync(hs, st.p, sizeof(PcgState), cudaMemcpyDeviceToHost, c.stream));
    RDG_CUDA(cudaMemcpyAsync(herr, c.d_err, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    if (it < max_iter) enqueue_ap_xr();
    RDG_CUDA(cudaStreamSynchronize(c.stream));
    const int derr = *herr;
    if (derr) {
      RDG_CUDA(cudaMemset(c.d_err, 0, sizeof(int)));
      throw Error(derr, derr == RD_EZERODIAG ? "sgs_sweep: zero diagonal" : "device error");
    }
    if (hs->status == 1) throw Error(RD_ENOTSPD, "pcg: operator not positive definite (p'Ap <= 0)");
    if (hs->status) throw Error(RD_ENOTSPD, "pcg: preconditioner not positive definite");
    out.iterations = hs->it;
    if (hs->done) {
      out.converged = true;
      return out;
    }
  }
  return out;
}

PcgResultDev pcg_device(Ctx& c, const DCsr& A, Hierarchy* h, const double* f, double tol, int max_iter, double* x,
                        double* hist_dev) {
  // the hierarchy's level 0 views A's arrays (its stencil facts feed the lattice SpMV)
  const DCsr& As = (h && !h->levels.empty() && h->levels[0].A.v.p == A.v.p && h->levels[0].A.rp.p == A.rp.p &&
                    h->levels[0].A.rows == A.rows)
                       ? h->levels[0].A
                       : A;
  const int64_t n = A.rows;
  const PcgOp apply_A = [&](const double* p, double* Ap, double* pAp) { spmv_dot(c, As, p, Ap, pAp); };
  const PcgOp apply_P = [&](const double* r, double* z, double* rz) {
    if (h) {
      vcycle(c, *h, r, z, rz);
    } else {
      RDG_CUDA(cudaMemcpyAsync(z, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
      dot(c, n, r, z, rz);
    }
  };
  return pcg_ops(c, n, apply_A, apply_P, f, tol, max_iter, x, hist_dev);
}

}  // namespace rdg
