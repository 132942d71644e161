// amg.cu -- device AMG setup and V-cycle (amg.cpp:7-145) on sm_100a.
//
// Setup runs entirely on the device:
//   * coarsen_redblack (amg.cpp:7-56) is the lexicographically-first maximal
//     independent set: vertex i is coarse iff none of its lower-indexed
//     neighbours is coarse.  A sync-free kernel decides vertices in ticket
//     order, each waiting only on its lower neighbours' decisions, so the
//     C/F splitting is bit-identical to the sequential greedy loop.
//   * P rows: unit for C, 1/count over C neighbours for F (amg.cpp:36-51).
//   * Pt = transpose(P); A_c = prune(Pt * (A * P)) with Eigen's ordered
//     conservative-product accumulation (linalg.cu spgemm).
//   * coarsest level: dense LLT in one CTA.
#include <algorithm>
#include <cmath>

#include "internal.hpp"

namespace rdg {

namespace {

constexpr int kMisNT = 128;
enum : int { kUndecided = 0, kCoarse = 1, kFine = 2 };

// Lexicographically-first MIS over in-neighbours given by G (== A for a
// structurally symmetric A, A^T otherwise).
__global__ void __launch_bounds__(kMisNT) mis_kernel(int n, const int* __restrict__ grp,
                                                     const int* __restrict__ gci, int* state, int* ticket) {
  __shared__ int blk;
  if (threadIdx.x == 0) blk = atomicAdd(ticket, 1);
  __syncthreads();
  const int i = blk * kMisNT + threadIdx.x;
  if (i >= n) return;
  int st = kCoarse;
  for (int k = grp[i]; k < grp[i + 1]; ++k) {
    const int j = gci[k];
    if (j >= i) continue;
    // the state word is the whole message: relaxed loads suffice (no L1 invalidation)
    int sj;
    while ((sj = ld_relaxed_s32(state + j)) == kUndecided) {
    }
    if (sj == kCoarse) {
      st = kFine;
      break;
    }
  }
  st_relaxed_s32(state + i, st);
}

// guard (amg.cpp:22-29): count fine rows without a coarse neighbour
__global__ void guard_count_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                   const int* __restrict__ state, int* nbad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || state[i] != kFine) return;
  for (int k = rp[i]; k < rp[i + 1]; ++k)
    if (ci[k] != i && state[ci[k]] == kCoarse) return;
  atomicAdd(nbad, 1);
}

// exact sequential guard (in-place promotion order matters), only when needed
__global__ void guard_serial_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci, int* state) {
  for (int i = 0; i < n; ++i) {
    if (state[i] != kFine) continue;
    bool has = false;
    for (int k = rp[i]; k < rp[i + 1] && !has; ++k) has = ci[k] != i && state[ci[k]] == kCoarse;
    if (!has) state[i] = kCoarse;
  }
}

__global__ void coarse_flags_kernel(int n, const int* __restrict__ state, int* isc, uint8_t* flags) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = state[i] == kCoarse;
  isc[i] = c;
  flags[i] = (uint8_t)c;
}

__global__ void p_count_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                               const int* __restrict__ state, int* cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (state[i] == kCoarse) {
    cnt[i] = 1;
    return;
  }
  int c = 0;
  for (int k = rp[i]; k < rp[i + 1]; ++k) c += ci[k] != i && state[ci[k]] == kCoarse;
  cnt[i] = c;
}

__global__ void p_fill_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                              const int* __restrict__ state, const int* __restrict__ cidx,
                              const int* __restrict__ prp, int* pci, double* pv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int o = prp[i];
  if (state[i] == kCoarse) {
    pci[o] = cidx[i];
    pv[o] = 1.0;
    return;
  }
  const int count = prp[i + 1] - o;
  const double w = __ddiv_rn(1.0, (double)count);
  for (int k = rp[i]; k < rp[i + 1]; ++k)
    if (ci[k] != i && state[ci[k]] == kCoarse) {
      pci[o] = cidx[ci[k]];
      pv[o] = w;
      ++o;
    }
}

__global__ void to_dense_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                const double* __restrict__ v, double* D) {
  const int r = blockIdx.x;
  for (int k = rp[r] + threadIdx.x; k < rp[r + 1]; k += blockDim.x) D[(size_t)r * n + ci[k]] = v[k];
}

// Left-looking Cholesky in one CTA, operation order identical to the oracle's
// llt_compute (the CPU checker in oracle/).  L overwrites the dense copy.
__global__ void llt_kernel(int n, double* L, int* err) {
  __shared__ double piv;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      double s = L[(size_t)j * n + j];
      for (int k = 0; k < j; ++k) s = __dsub_rn(s, __dmul_rn(L[(size_t)j * n + k], L[(size_t)j * n + k]));
      if (!(s > 0.0)) {
        bad = 1;
      } else {
        piv = __dsqrt_rn(s);
        L[(size_t)j * n + j] = piv;
      }
    }
    __syncthreads();
    if (bad) break;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
      double t = L[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) t = __dsub_rn(t, __dmul_rn(L[(size_t)i * n + k], L[(size_t)j * n + k]));
      L[(size_t)i * n + j] = __ddiv_rn(t, piv);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (bad) *err = 1;
    // zero the strict upper triangle (never read; keeps downloads clean)
  }
}

// LLT solve in one CTA: forward L y = b (row sums ascending in k), then
// L^T x = y (sums descending in k) -- same order as the oracle's llt_solve.
constexpr int kCoarseNT = 256;
__global__ void __launch_bounds__(kCoarseNT) llt_solve_kernel(int n, const double* __restrict__ L,
                                                              const double* __restrict__ b, double* x) {
  extern __shared__ double sh[];  // s[n]
  for (int i = threadIdx.x; i < n; i += kCoarseNT) sh[i] = b[i];
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    // y_k final once all updates from columns < k are applied
    const double yk = __ddiv_rn(sh[k], L[(size_t)k * n + k]);
    __syncthreads();
    if (threadIdx.x == 0) sh[k] = yk;
    for (int i = k + 1 + threadIdx.x; i < n; i += kCoarseNT) sh[i] = __dsub_rn(sh[i], __dmul_rn(L[(size_t)i * n + k], yk));
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {
    const double xk = __ddiv_rn(sh[k], L[(size_t)k * n + k]);
    __syncthreads();
    if (threadIdx.x == 0) sh[k] = xk;
    for (int i = threadIdx.x; i < k; i += kCoarseNT) sh[i] = __dsub_rn(sh[i], __dmul_rn(L[(size_t)k * n + i], xk));
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += kCoarseNT) x[i] = sh[i];
}

// ---------------------------------------------------------------- lattice levels
// On a verified 15-point in-box lattice stencil the greedy MIS is the set of
// all-even points (every odd point p sees p - e_S, S = its odd axes, as a lower
// neighbour; every even point's lower neighbours are odd), and every F point has
// a C neighbour, so the guard never fires.
__global__ void lat_flags_kernel(int n, int L, int* state) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int x = i % L, y = i / L % L, z = i / (L * L);
  state[i] = ((x | y | z) & 1) ? kFine : kCoarse;
}

// Galerkin product on lattice levels.  Eigen's ordered product gives entry
// (i, j) of A*B as the in-order sum over ascending k of A_ik * B_kj (first
// term assigned); here each row accumulates into a dense 3x3x3 window of coarse
// columns around its own position, in exactly that order, instead of searching
// a first-touch list.  Terms of absent entries are never added; a window slot
// that only ever receives exact zeros differs at most in the sign of zero, and
// every zero is pruned from A_c.  A column outside the window (not a lattice
// coarsening) raises the flag and the generic product runs instead.
constexpr int kGalNT = 128;

__global__ void __launch_bounds__(kGalNT) lat_ap_kernel(int nf, int L, int Lc, const int* __restrict__ arp,
                                                        const int* __restrict__ aci, const double* __restrict__ av,
                                                        const int* __restrict__ prp, const int* __restrict__ pci,
                                                        const double* __restrict__ pv, double* ap, int* err) {
  __shared__ double W[27][kGalNT];
  const int t = threadIdx.x;
  const int k = blockIdx.x * kGalNT + t;
  if (k >= nf) return;
#pragma unroll
  for (int s = 0; s < 27; ++s) W[s][t] = 0.0;
  const int x = k % L, y = k / L % L, z = k / (L * L);
  const int bx = (x - 1) >> 1, by = (y - 1) >> 1, bz = (z - 1) >> 1;
  bool bad = false;
  for (int ka = arp[k]; ka < arp[k + 1]; ++ka) {
    const int m = aci[ka];
    const double a = av[ka];
    for (int kb = prp[m]; kb < prp[m + 1]; ++kb) {
      const int J = pci[kb];
      const int dx = J % Lc - bx, dy = J / Lc % Lc - by, dz = J / (Lc * Lc) - bz;
      if ((unsigned)dx > 2u || (unsigned)dy > 2u || (unsigned)dz > 2u) {
        bad = true;
        continue;
      }
      double& w = W[dz * 9 + dy * 3 + dx][t];
      w = __dadd_rn(w, __dmul_rn(pv[kb], a));
    }
  }
  if (bad) atomicExch(err, 1);
#pragma unroll
  for (int s = 0; s < 27; ++s) ap[(size_t)s * nf + k] = W[s][t];
}

__global__ void __launch_bounds__(kGalNT) lat_ptap_kernel(int nc, int Lc, int nf, int L,
                                                          const int* __restrict__ trp, const int* __restrict__ tci,
                                                          const double* __restrict__ tv,
                                                          const double* __restrict__ ap, double* out, int* cnt,
                                                          int* err) {
  __shared__ double W[27][kGalNT];
  const int t = threadIdx.x;
  const int I = blockIdx.x * kGalNT + t;
  if (I >= nc) return;
#pragma unroll
  for (int s = 0; s < 27; ++s) W[s][t] = 0.0;
  const int cx = I % Lc - 1, cy = I / Lc % Lc - 1, cz = I / (Lc * Lc) - 1;  // window origin
  bool bad = false;
  for (int kt = trp[I]; kt < trp[I + 1]; ++kt) {
    const int k = tci[kt];
    const double pw = tv[kt];
    const int x = k % L, y = k / L % L, z = k / (L * L);
    const int ox = ((x - 1) >> 1) - cx, oy = ((y - 1) >> 1) - cy, oz = ((z - 1) >> 1) - cz;
#pragma unroll 3
    for (int s = 0; s < 27; ++s) {
      const double v = ap[(size_t)s * nf + k];
      if (v == 0.0) continue;
      const int dx = ox + s % 3, dy = oy + s / 3 % 3, dz = oz + s / 9;
      if ((unsigned)dx > 2u || (unsigned)dy > 2u || (unsigned)dz > 2u) {
        bad = true;
        continue;
      }
      double& w = W[dz * 9 + dy * 3 + dx][t];
      w = __dadd_rn(w, __dmul_rn(v, pw));
    }
  }
  if (bad) atomicExch(err, 1);
  int c = 0;
#pragma unroll
  for (int s = 0; s < 27; ++s) {
    const double w = W[s][t];
    c += w != 0.0;
    out[(size_t)s * nc + I] = w;
  }
  cnt[I] = c;
}

__global__ void lat_compact_kernel(int nc, int Lc, const double* __restrict__ out, const int* __restrict__ rp,
                                   int* ci, double* v) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= nc) return;
  const int cx = I % Lc - 1, cy = I / Lc % Lc - 1, cz = I / (Lc * Lc) - 1;
  int o = rp[I];
#pragma unroll
  for (int s = 0; s < 27; ++s) {
    const double w = out[(size_t)s * nc + I];
    if (w != 0.0) {
      ci[o] = ((cz + s / 9) * Lc + (cy + s / 3 % 3)) * Lc + (cx + s % 3);
      v[o++] = w;
    }
  }
}

// P^T on a lattice level with the all-even coarsening: the rows of P^T come out
// in ascending fine index by walking each coarse point's 3x3x3 fine neighbourhood
// in (dz, dy, dx) order -- no atomics, no per-row sort (same result as transpose()).
template <bool FILL>
__global__ void lat_pt_kernel(int nc, int Lc, int L, const int* __restrict__ prp, const int* __restrict__ pci,
                              const double* __restrict__ pv, int* cnt, const int* __restrict__ trp, int* tci,
                              double* tv) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= nc) return;
  const int fx = 2 * (I % Lc), fy = 2 * (I / Lc % Lc), fz = 2 * (I / (Lc * Lc));
  int o = FILL ? trp[I] : 0;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int x = fx + dx, y = fy + dy, z = fz + dz;
        if (x < 0 || y < 0 || z < 0 || x >= L || y >= L || z >= L) continue;
        const int k = (z * L + y) * L + x;
        for (int e = prp[k]; e < prp[k + 1]; ++e)
          if (pci[e] == I) {
            if (FILL) {
              tci[o] = k;
              tv[o] = pv[e];
            }
            ++o;
          }
      }
  if (!FILL) cnt[I] = o;
}

int read_int(Ctx& c, const int* d) {
  int h = 0;
  RDG_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  RDG_CUDA(cudaStreamSynchronize(c.stream));
  return h;
}

}  // namespace

std::vector<uint8_t> coarsen(Ctx& c, const DCsr& A, DBuf<uint8_t>& flags, DCsr& P) {
  const int n = A.rows;
  flags.alloc(std::max(n, 1), c.stream);
  P = DCsr{};
  P.rows = n;
  P.rp.alloc(n + 1, c.stream);
  if (n == 0) {
    RDG_CUDA(cudaMemsetAsync(P.rp.p, 0, sizeof(int), c.stream));
    return {};
  }
  DBuf<int> state(n, c.stream), tmp(n + 1, c.stream), cidx(n + 1, c.stream), scratch(4, c.stream);
  RDG_CUDA(cudaMemsetAsync(state.p, 0, sizeof(int) * n, c.stream));
  RDG_CUDA(cudaMemsetAsync(scratch.p, 0, sizeof(int) * 4, c.stream));
  if (A.lat.ok && A.lat.lx == A.lat.ly && A.lat.ly == A.lat.lz) {
    lat_flags_kernel<<<div_up(n, 256), 256, 0, c.stream>>>(n, A.lat.lx, state.p);
    RDG_LAUNCH_CHECK();
    ++c.launches;
  } else {
    DCsr At;
    const bool sym = pattern_symmetric(c, A);
    if (!sym) At = transpose(c, A);
    const DCsr& G = sym ? A : At;
    mis_kernel<<<div_up(n, kMisNT), kMisNT, 0, c.stream>>>(n, G.rp.p, G.ci.p, state.p, scratch.p);
    RDG_LAUNCH_CHECK();
    guard_count_kernel<<<div_up(n, 256), 256, 0, c.stream>>>(n, A.rp.p, A.ci.p, state.p, scratch.p + 1);
    RDG_LAUNCH_CHECK();
    c.launches += 2;
    if (read_int(c, scratch.p + 1) > 0) {
      guard_serial_kernel<<<1, 1, 0, c.stream>>>(n, A.rp.p, A.ci.p, state.p);
      RDG_LAUNCH_CHECK();
      ++c.launches;
    }
  }
  coarse_flags_kernel<<<div_up(n, 256), 256, 0, c.stream>>>(n, state.p, tmp.p, flags.p);
  RDG_LAUNCH_CHECK();
  ++c.launches;
  P.cols = static_cast<int>(exclusive_scan(c, tmp.p, cidx.p, n));
  p_count_kernel<<<div_up(n, 256), 256, 0, c.stream>>>(n, A.rp.p, A.ci.p, state.p, tmp.p);
  RDG_LAUNCH_CHECK();
  ++c.launches;
  P.nnz = exclusive_scan(c, tmp.p, P.rp.p, n);
  P.ci.alloc(P.nnz, c.stream);
  P.v.alloc(P.nnz, c.stream);
  p_fill_kernel<<<div_up(n, 256), 256, 0, c.stream>>>(n, A.rp.p, A.ci.p, state.p, cidx.p, P.rp.p, P.ci.p, P.v.p);
  RDG_LAUNCH_CHECK();
  ++c.launches;
  return {};  // flags stay on the device (rd_gpu_coarsen_redblack downloads them)
}

// Lattice-level Galerkin product (see lat_ap_kernel); false: not applicable.
static bool galerkin_lattice(Ctx& c, const DCsr& A, const DCsr& P, const DCsr& Pt, DCsr& Ac) {
  if (!A.lat.ok || A.lat.lx != A.lat.ly || A.lat.ly != A.lat.lz) return false;
  const int L = A.lat.lx, Lc = (L + 1) / 2;
  const int nf = A.rows, nc = P.cols;
  if ((int64_t)Lc * Lc * Lc != nc || nc == 0 || Pt.rows != nc) return false;
  DBuf<int> err(1, c.stream), cnt(nc, c.stream);
  RDG_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), c.stream));
  DBuf<double> out((size_t)27 * nc, c.stream);
  {
    DBuf<double> ap((size_t)27 * nf, c.stream);
    lat_ap_kernel<<<div_up(nf, kGalNT), kGalNT, 0, c.stream>>>(nf, L, Lc, A.rp.p, A.ci.p, A.v.p, P.rp.p, P.ci.p,
                                                               P.v.p, ap.p, err.p);
    RDG_LAUNCH_CHECK();
    lat_ptap_kernel<<<div_up(nc, kGalNT), kGalNT, 0, c.stream>>>(nc, Lc, nf, L, Pt.rp.p, Pt.ci.p, Pt.v.p, ap.p,
                                                                 out.p, cnt.p, err.p);
    RDG_LAUNCH_CHECK();
    c.launches += 2;
  }
  if (read_int(c, err.p)) return false;
  Ac = DCsr{};
  Ac.rows = Ac.cols = nc;
  Ac.rp.alloc(nc + 1, c.stream);
  Ac.nnz = exclusive_scan(c, cnt.p, Ac.rp.p, nc);
  Ac.ci.alloc(Ac.nnz, c.stream);
  Ac.v.alloc(Ac.nnz, c.stream);
  lat_compact_kernel<<<div_up(nc, 256), 256, 0, c.stream>>>(nc, Lc, out.p, Ac.rp.p, Ac.ci.p, Ac.v.p);
  RDG_LAUNCH_CHECK();
  ++c.launches;
  return true;
}

DCsr galerkin(Ctx& c, const DCsr& A, const DCsr& P, const DCsr& Pt) {
  if (A.cols != P.rows) throw Error(RD_EINVAL, "galerkin_coarse: dims");
  {
    DCsr Ac;
    if (galerkin_lattice(c, A, P, Pt, Ac)) return Ac;
  }
  DCsr AP = spgemm(c, A, P);
  DCsr Ac = spgemm(c, Pt, AP);
  return prune_zeros(c, Ac);
}

void dense_llt(Ctx& c, const DCsr& A, DBuf<double>& L) {
  const int n = A.rows;
  L.alloc((size_t)n * n, c.stream);
  RDG_CUDA(cudaMemsetAsync(L.p, 0, sizeof(double) * n * n, c.stream));
  to_dense_kernel<<<n, 64, 0, c.stream>>>(n, A.rp.p, A.ci.p, A.v.p, L.p);
  RDG_LAUNCH_CHECK();
  DBuf<int> err(1, c.stream);
  RDG_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), c.stream));
  llt_kernel<<<1, 256, 0, c.stream>>>(n, L.p, err.p);
  RDG_LAUNCH_CHECK();
  c.launches += 2;
  if (read_int(c, err.p)) throw Error(RD_ENOTSPD, "build_amg: coarsest level not positive definite");
}

void build_hierarchy(Ctx& c, const DCsr& A, int threshold, int m, Hierarchy& h) {
  h.levels.clear();
  h.smoothing_steps = m;
  DCsr current = csr_copy(c, A);
  while (current.rows > threshold) {
    Level lv;
    lv.A = std::move(current);
    detect_lattice(c, lv.A);  // lattice levels: closed-form C/F split and windowed Galerkin
    DCsr P;
    coarsen(c, lv.A, lv.flags, P);
    if (P.cols >= P.rows) {  // no reduction possible (amg.cpp:98-101)
      current = std::move(lv.A);
      lv.flags.release();
      break;
    }
    lv.P = std::move(P);
    const int Lf = lv.A.lat.lx, Lc = (Lf + 1) / 2;
    if (lv.A.lat.ok && Lf == lv.A.lat.ly && Lf == lv.A.lat.lz && (int64_t)Lc * Lc * Lc == lv.P.cols) {
      DCsr& T = lv.Pt;
      T = DCsr{};
      T.rows = lv.P.cols;
      T.cols = lv.P.rows;
      T.rp.alloc(T.rows + 1, c.stream);
      DBuf<int> cnt(T.rows + 1, c.stream);
      lat_pt_kernel<false><<<div_up(T.rows, 256), 256, 0, c.stream>>>(T.rows, Lc, Lf, lv.P.rp.p, lv.P.ci.p, lv.P.v.p,
                                                                       cnt.p, nullptr, nullptr, nullptr);
      RDG_LAUNCH_CHECK();
      T.nnz = exclusive_scan(c, cnt.p, T.rp.p, T.rows);
      c.launches += 1;
      if (T.nnz == lv.P.nnz) {
        T.ci.alloc(T.nnz, c.stream);
        T.v.alloc(T.nnz, c.stream);
        lat_pt_kernel<true><<<div_up(T.rows, 256), 256, 0, c.stream>>>(T.rows, Lc, Lf, lv.P.rp.p, lv.P.ci.p,
                                                                        lv.P.v.p, nullptr, T.rp.p, T.ci.p, T.v.p);
        RDG_LAUNCH_CHECK();
        ++c.launches;
      } else {  // an entry outside the window: not the all-even coarsening after all
        lv.Pt = transpose(c, lv.P);
      }
    } else {
      lv.Pt = transpose(c, lv.P);
    }
    lv.has_p = true;
    current = galerkin(c, lv.A, lv.P, lv.Pt);
    h.levels.push_back(std::move(lv));
  }
  Level last;
  last.A = std::move(current);
  h.levels.push_back(std::move(last));
  h.nc = h.levels.back().A.rows;
  if (h.nc > 0) dense_llt(c, h.levels.back().A, h.Lc);
  // work vectors; structured-smoother detection per level
  for (size_t l = 0; l < h.levels.size(); ++l) {
    Level& lv = h.levels[l];
    const int n = std::max(lv.A.rows, 1);
    if (l > 0) {
      lv.r.alloc(n, c.stream);
      lv.z.alloc(n, c.stream);
    }
    lv.t.alloc(n, c.stream);
    lv.res.alloc(n, c.stream);
    if (lv.has_p) {
      detect_lattice(c, lv.A);
      lattice_prepare(c, lv.A);
    }
  }
}

void coarse_solve(Ctx& c, Hierarchy& h, const double* r, double* z) {
  const int n = h.nc;
  if (n == 0) return;
  llt_solve_kernel<<<1, kCoarseNT, sizeof(double) * n, c.stream>>>(n, h.Lc.p, r, z);
  RDG_LAUNCH_CHECK();
  ++c.launches;
}

// V-cycle with zero initial guess (amg.cpp:119-132), unrolled over levels.
void vcycle(Ctx& c, Hierarchy& h, const double* r, double* z, double* dot_out) {
  const int L = static_cast<int>(h.levels.size());
  const int m = h.smoothing_steps;
  if (L == 1) {
    coarse_solve(c, h, r, z);
    if (dot_out) dot(c, h.nc, r, z, dot_out);
    return;
  }
  std::vector<const double*> rl(L);
  std::vector<double*> zl(L);
  rl[0] = r;
  zl[0] = z;
  for (int l = 1; l < L; ++l) {
    rl[l] = h.levels[l].r.p;
    zl[l] = h.levels[l].z.p;
  }
  for (int l = 0; l + 1 < L; ++l) {
    Level& lv = h.levels[l];
    const double* cur = nullptr;  // zero initial guess
    for (int s = 0; s < m; ++s) {
      gs_pass(c, lv.A, rl[l], cur, lv.t.p, true);
      gs_pass(c, lv.A, rl[l], lv.t.p, zl[l], false);
      cur = zl[l];
    }
    if (m == 0) RDG_CUDA(cudaMemsetAsync(zl[l], 0, sizeof(double) * lv.A.rows, c.stream));
    residual(c, lv.A, rl[l], zl[l], lv.res.p);
    spmv(c, lv.Pt, lv.res.p, h.levels[l + 1].r.p);
  }
  coarse_solve(c, h, rl[L - 1], zl[L - 1]);
  for (int l = L - 2; l >= 0; --l) {
    Level& lv = h.levels[l];
    prolong_add(c, lv.P, zl[l + 1], zl[l]);
    for (int s = 0; s < m; ++s) {
      gs_pass(c, lv.A, rl[l], zl[l], lv.t.p, true);
      const bool last = (l == 0 && s == m - 1);
      gs_pass(c, lv.A, rl[l], lv.t.p, zl[l], false, last ? dot_out : nullptr, last ? rl[0] : nullptr);
    }
  }
  if (m == 0 && dot_out) dot(c, h.levels[0].A.rows, r, z, dot_out);
}

}  // namespace rdg
