// smoother.cu -- exact lexicographic Gauss-Seidel passes (amg.cpp:67-88) on sm_100a.
//
// The reference relaxes rows strictly in order i = 0..n-1 (forward) and then
// n-1..0 (backward); row i reads new values for already-visited columns and
// old values for the rest, summing s = f_i - sum_k a_ik x_k in column order
// and dividing by the diagonal last.  Both kernels here reproduce that
// arithmetic bit for bit: same operands, same order, IEEE division, no FMA.
//
//  * gs_syncfree_kernel (generic CSR): one thread per row, blocks take rows in
//    ticket order; a row spins on epoch-stamped readiness flags of its
//    already-visited neighbours (acquire/release at gpu scope).  Correct for
//    any matrix, latency bound by the dependency depth.
//  * gs_syncfree_cta_kernel (generic CSR up to kGsCtaMaxRows rows -- the coarsest levels
//    of a non-lattice hierarchy): the same inside ONE thread block, readiness flags in
//    shared memory, so a dependency hop is a shared-memory round trip instead of an L2 one.
//    Measured (C2 renumbered, whose coarse levels are nearly serial chains): 139 rows
//    0.48 -> 0.21 ms, 1944 rows 0.93 -> 0.80 ms, but 26830 rows 0.98 -> 2.1 ms -- hence
//    the small threshold.
//  * the structured lattice kernel (smoother_lattice.cu) handles matrices whose
//    pattern was verified to be the 15-point Kuhn stencil on a box.
#include <cstdlib>

#include "internal.hpp"

namespace rdg {

void gs_pass_lattice(Ctx& c, const DCsr& A, const double* f, const double* xin, double* xout, bool fwd,
                     double* dot_out, const double* dot_with);
void gs_pass_generic(Ctx& c, const DCsr& A, const double* f, const double* xin, double* xout, bool fwd,
                     double* dot_out, const double* dot_with);

namespace {

constexpr int kGsNT = 128;

__global__ void __launch_bounds__(kGsNT) gs_syncfree_kernel(int n, const int* __restrict__ rp,
                                                            const int* __restrict__ ci,
                                                            const double* __restrict__ val,
                                                            const double* __restrict__ f,
                                                            const double* __restrict__ xin, double* xout,
                                                            unsigned* flags, unsigned epoch, int* ticket,
                                                            int* err, int fwd) {
  __shared__ int blk;
  if (threadIdx.x == 0) blk = atomicAdd(ticket, 1);
  __syncthreads();
  const int t = blk * kGsNT + threadIdx.x;
  if (t >= n) return;
  const int i = fwd ? t : n - 1 - t;
  double s = f[i];
  double d = 0.0;
  const int e = rp[i + 1];
  for (int k = rp[i]; k < e; ++k) {
    const int j = ci[k];
    const double a = val[k];
    if (j == i) {
      d = a;
      continue;
    }
    double xj;
    if (fwd ? (j < i) : (j > i)) {
      while (ld_acquire_u32(flags + j) != epoch) {
      }
      xj = ld_relaxed_f64(xout + j);
    } else {
      xj = xin ? __ldg(xin + j) : 0.0;
    }
    s = __dsub_rn(s, __dmul_rn(a, xj));
  }
  if (d == 0.0) atomicCAS(err, 0, RD_EZERODIAG);
  xout[i] = __ddiv_rn(s, d);
  st_release_u32(flags + i, epoch);
}

// one thread block: thread t relaxes rows t, t + NT, ... in sweep order; every wait is on
// a smaller (forward) / larger (backward) row, so the chain of waits always ends
constexpr int kGsCtaNT = 1024;
constexpr int kGsCtaMaxRows = 4096;  // u8 flags in dynamic shared memory
__global__ void __launch_bounds__(kGsCtaNT, 1) gs_syncfree_cta_kernel(int n, const int* __restrict__ rp,
                                                                    const int* __restrict__ ci,
                                                                    const double* __restrict__ val,
                                                                    const double* __restrict__ f,
                                                                    const double* __restrict__ xin, double* xout,
                                                                    int* err, int fwd) {
  extern __shared__ unsigned char ready[];
  for (int k = threadIdx.x; k < n; k += kGsCtaNT) ready[k] = 0;
  __syncthreads();
  const unsigned rbase = (unsigned)__cvta_generic_to_shared(ready);
  for (int t = threadIdx.x; t < n; t += kGsCtaNT) {
    const int i = fwd ? t : n - 1 - t;
    double s = f[i];
    double d = 0.0;
    const int e = rp[i + 1];
    for (int k = rp[i]; k < e; ++k) {
      const int j = ci[k];
      const double a = val[k];
      if (j == i) {
        d = a;
        continue;
      }
      double xj;
      if (fwd ? (j < i) : (j > i)) {
        unsigned r;
        do {
          asm volatile("ld.acquire.cta.shared.u8 %0, [%1];" : "=r"(r) : "r"(rbase + (unsigned)j) : "memory");
        } while (r == 0u);
        asm volatile("ld.relaxed.cta.global.f64 %0, [%1];" : "=d"(xj) : "l"(xout + j) : "memory");
      } else {
        xj = xin ? __ldg(xin + j) : 0.0;
      }
      s = __dsub_rn(s, __dmul_rn(a, xj));
    }
    if (d == 0.0) atomicCAS(err, 0, RD_EZERODIAG);
    const double xi = __ddiv_rn(s, d);
    asm volatile("st.relaxed.cta.global.f64 [%0], %1;" ::"l"(xout + i), "d"(xi) : "memory");
    asm volatile("st.release.cta.shared.u8 [%0], %1;" ::"r"(rbase + (unsigned)i), "r"(1u) : "memory");
  }
}

// s -= p_q for q = 0 .. m-1 in order (d takes the diagonal's entry), the p_q held by lane q.
// (Measured: issuing the shuffles eight at a time ahead of the subtractions was slower.)
__device__ __forceinline__ void row_accumulate(double p, unsigned dmask, int m, double& s, double& d) {
  for (int q = 0; q < m; ++q) {
    const double pq = __shfl_sync(0xffffffffu, p, q);
    if ((dmask >> q) & 1u)
      d = pq;
    else
      s = __dsub_rn(s, pq);
  }
}

// Warp per row (generic CSR, any size): the row's entries are handled 32 at a time, so the
// waits on its already-visited neighbours overlap (lane k polls entry k's flag) instead of one
// L2 round trip per neighbour in sequence, and the new values load in parallel after one
// acquire fence.  The sum then runs sequentially over the entries in column order on every
// lane (products shuffled in): the reference's arithmetic, bit for bit.  Warps take rows in
// ticket order, so every wait is on a row some earlier warp owns: no deadlock.
constexpr int kGswNT = 256;
constexpr int kGsWarpMaxRows = 1 << 19;
__global__ void __launch_bounds__(kGswNT) gs_syncfree_warp_kernel(int n, const int* __restrict__ rp,
                                                                  const int* __restrict__ ci,
                                                                  const double* __restrict__ val,
                                                                  const double* __restrict__ f,
                                                                  const double* __restrict__ xin, double* xout,
                                                                  unsigned* flags, unsigned epoch, int* ticket,
                                                                  int* err, int fwd) {
  __shared__ int blk;
  if (threadIdx.x == 0) blk = atomicAdd(ticket, 1);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int t = blk * (kGswNT / 32) + (threadIdx.x >> 5);
  if (t >= n) return;
  const int i = fwd ? t : n - 1 - t;
  const int b = rp[i], e = rp[i + 1];
  // wait for every visited neighbour (relaxed polls), then one acquire fence
  for (int k0 = b; k0 < e; k0 += 32) {
    const int k = k0 + lane;
    if (k < e) {
      const int j = ci[k];
      if (fwd ? (j < i) : (j > i)) {
        unsigned v;
        do {
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + j) : "memory");
        } while (v != epoch);
      }
    }
  }
  __syncwarp();
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  double s = f[i], d = 0.0;
  for (int k0 = b; k0 < e; k0 += 32) {
    const int k = k0 + lane;
    double p = 0.0;
    bool diag = false;
    if (k < e) {
      const int j = ci[k];
      const double a = val[k];
      diag = j == i;
      if (diag) {
        p = a;
      } else {
        const double xj = (fwd ? (j < i) : (j > i)) ? ld_relaxed_f64(xout + j) : (xin ? __ldg(xin + j) : 0.0);
        p = __dmul_rn(a, xj);
      }
    }
    row_accumulate(p, __ballot_sync(0xffffffffu, diag), min(32, e - k0), s, d);
  }
  if (lane == 0) {
    if (d == 0.0) atomicCAS(err, 0, RD_EZERODIAG);
    xout[i] = __ddiv_rn(s, d);
    st_release_u32(flags + i, epoch);
  }
}

// The same warp-per-row scheme inside ONE block for small levels (<= kGsCtaMaxRows rows): old and
// new values and the readiness flags all in shared memory, so a dependency hop is a shared-memory
// round trip.  Warp w relaxes rows w, w + 32, ... in sweep order.
constexpr int kGscNT = 1024;
__global__ void __launch_bounds__(kGscNT, 1) gs_syncfree_cta_warp_kernel(int n, const int* __restrict__ rp,
                                                                        const int* __restrict__ ci,
                                                                        const double* __restrict__ val,
                                                                        const double* __restrict__ f,
                                                                        const double* __restrict__ xin,
                                                                        double* xout, int* err, int fwd) {
  extern __shared__ __align__(16) unsigned char gsm[];
  double* xo = reinterpret_cast<double*>(gsm);  // old values (xin, or 0)
  double* xn = xo + n;                          // new values
  unsigned char* ready = reinterpret_cast<unsigned char*>(xn + n);
  for (int k = threadIdx.x; k < n; k += kGscNT) {
    xo[k] = xin ? xin[k] : 0.0;
    ready[k] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned rbase = (unsigned)__cvta_generic_to_shared(ready);
  for (int t = w; t < n; t += kGscNT / 32) {
    const int i = fwd ? t : n - 1 - t;
    const int b = rp[i], e = rp[i + 1];
    double s = f[i], d = 0.0;
    for (int k0 = b; k0 < e; k0 += 32) {
      const int k = k0 + lane;
      double p = 0.0, a = 0.0;
      bool diag = false, fresh = false;
      int j = 0;
      if (k < e) {  // everything that does not wait on a neighbour first
        j = ci[k];
        a = val[k];
        diag = j == i;
        fresh = !diag && (fwd ? (j < i) : (j > i));
        p = diag ? a : fresh ? 0.0 : __dmul_rn(a, xo[j]);
      }
      if (fresh) {
        unsigned r;
        do {
          asm volatile("ld.acquire.cta.shared.u8 %0, [%1];" : "=r"(r) : "r"(rbase + (unsigned)j) : "memory");
        } while (r == 0u);
        p = __dmul_rn(a, *reinterpret_cast<volatile double*>(xn + j));
      }
      row_accumulate(p, __ballot_sync(0xffffffffu, diag), min(32, e - k0), s, d);
    }
    if (lane == 0) {
      if (d == 0.0) atomicCAS(err, 0, RD_EZERODIAG);
      *reinterpret_cast<volatile double*>(xn + i) = __ddiv_rn(s, d);
      asm volatile("st.release.cta.shared.u8 [%0], %1;" ::"r"(rbase + (unsigned)i), "r"(1u) : "memory");
    }
    __syncwarp();
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += kGscNT) xout[k] = xn[k];
}

}  // namespace

void gs_pass(Ctx& c, const DCsr& A, const double* f, const double* xin, double* xout, bool fwd, double* dot_out,
             const double* dot_with) {
  if (A.rows == 0) {
    if (dot_out) RDG_CUDA(cudaMemsetAsync(dot_out, 0, sizeof(double), c.stream));
    return;
  }
  if (A.lat.ok)
    gs_pass_lattice(c, A, f, xin, xout, fwd, dot_out, dot_with);
  else
    gs_pass_generic(c, A, f, xin, xout, fwd, dot_out, dot_with);
}

void gs_pass_generic(Ctx& c, const DCsr& A, const double* f, const double* xin, double* xout, bool fwd,
                     double* dot_out, const double* dot_with) {
  const int n = A.rows;
  static const int variant = getenv("RD_GS_GENERIC") ? atoi(getenv("RD_GS_GENERIC")) : 1;  // A/B only
  if (n <= kGsCtaMaxRows) {
    if (variant == 1) {  // warp per row, values and flags in shared memory
      const size_t smem = (size_t)n * (2 * sizeof(double) + 1) + 16;
      static bool attr = false;
      if (!attr) {
        RDG_CUDA(cudaFuncSetAttribute(gs_syncfree_cta_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)((size_t)kGsCtaMaxRows * (2 * sizeof(double) + 1) + 16)));
        attr = true;
      }
      gs_syncfree_cta_warp_kernel<<<1, kGscNT, smem, c.stream>>>(n, A.rp.p, A.ci.p, A.v.p, f, xin, xout, c.d_err,
                                                                 fwd ? 1 : 0);
    } else {
      static bool attr = false;
      if (!attr) {
        RDG_CUDA(cudaFuncSetAttribute(gs_syncfree_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kGsCtaMaxRows));
        attr = true;
      }
      gs_syncfree_cta_kernel<<<1, kGsCtaNT, n, c.stream>>>(n, A.rp.p, A.ci.p, A.v.p, f, xin, xout, c.d_err,
                                                           fwd ? 1 : 0);
    }
    RDG_LAUNCH_CHECK();
    ++c.launches;
    if (dot_out) dot(c, n, dot_with, xout, dot_out);
    return;
  }
  if (!A.gs_flags.p) {
    A.gs_flags.alloc(n, c.stream);
    RDG_CUDA(cudaMemsetAsync(A.gs_flags.p, 0, sizeof(unsigned) * n, c.stream));
    A.gs_epoch = 0;
  }
  if (++A.gs_epoch == 0) {  // wrapped: clear and restart at 1
    RDG_CUDA(cudaMemsetAsync(A.gs_flags.p, 0, sizeof(unsigned) * n, c.stream));
    A.gs_epoch = 1;
  }
  int* ticket = reinterpret_cast<int*>(c.d_counter + 32);
  RDG_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), c.stream));
  // warp per row where the dependency chains bound the sweep; one thread per row keeps more
  // rows in flight on the largest levels (measured: C2 renumbered level 0, 2M rows: thread
  // 0.65 ms, warp 1.27 ms; an adapted 248k-row level: thread 0.22 ms, warp 0.15 ms)
  if (variant == 1 && n < kGsWarpMaxRows)
    gs_syncfree_warp_kernel<<<div_up(n, kGswNT / 32), kGswNT, 0, c.stream>>>(
        n, A.rp.p, A.ci.p, A.v.p, f, xin, xout, A.gs_flags.p, A.gs_epoch, ticket, c.d_err, fwd ? 1 : 0);
  else
    gs_syncfree_kernel<<<div_up(n, kGsNT), kGsNT, 0, c.stream>>>(n, A.rp.p, A.ci.p, A.v.p, f, xin, xout,
                                                                 A.gs_flags.p, A.gs_epoch, ticket, c.d_err,
                                                                 fwd ? 1 : 0);
  RDG_LAUNCH_CHECK();
  ++c.launches;
  if (dot_out) dot(c, n, dot_with, xout, dot_out);
}

}  // namespace rdg
