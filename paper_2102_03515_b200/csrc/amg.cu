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
#include <utility>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "internal.hpp"

namespace cg = cooperative_groups;

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
// llt_compute (the CPU checker in oracle/).  L overwrites the dense copy; with
// SMEM the factor is staged in shared memory (row stride n + 1: a warp's column
// reads fall in distinct banks) and written back at the end.
template <bool SMEM>
__global__ void llt_kernel(int n, double* Lg, int* err) {
  extern __shared__ double lsh[];
  __shared__ double piv;
  __shared__ int bad;
  const int ld = SMEM ? n + 1 : n;
  double* L = SMEM ? lsh : Lg;
  if (SMEM) {
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) lsh[(e / n) * ld + e % n] = Lg[e];
  }
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      double s = L[(size_t)j * ld + j];
      for (int k = 0; k < j; ++k) s = __dsub_rn(s, __dmul_rn(L[(size_t)j * ld + k], L[(size_t)j * ld + k]));
      if (!(s > 0.0)) {
        bad = 1;
      } else {
        piv = __dsqrt_rn(s);
        L[(size_t)j * ld + j] = piv;
      }
    }
    __syncthreads();
    if (bad) break;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
      double t = L[(size_t)i * ld + j];
      for (int k = 0; k < j; ++k) t = __dsub_rn(t, __dmul_rn(L[(size_t)i * ld + k], L[(size_t)j * ld + k]));
      L[(size_t)i * ld + j] = __ddiv_rn(t, piv);
    }
    __syncthreads();
  }
  if (SMEM) {
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) Lg[e] = lsh[(e / n) * ld + e % n];
  }
  if (threadIdx.x == 0 && bad) *err = 1;
}
constexpr int kLltSmemMax = 160 * 1024;
size_t llt_smem(int n) { return sizeof(double) * (size_t)n * (n + 1); }

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

// The same factorization for matrices past shared memory (the H^-1 dual norm's dense branch,
// n <= 2000), on the whole GPU, right-looking: after column j is divided by its pivot, every
// trailing lower-triangle entry subtracts L(i,j) L(m,j).  Each entry thus sees its products in
// k order, exactly llt_kernel's (and the oracle's) left-looking sequence -- the factor is
// bit-identical -- while the work per column is a wide parallel update instead of one sequential
// dot product per element.  Cooperative grid: two grid barriers per column; warp per row.
__global__ void __launch_bounds__(256) llt_right_kernel(int n, double* L, int* err) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
  for (int j = 0; j < n; ++j) {
    const double s = L[(size_t)j * n + j];  // every k < j already subtracted
    if (!(s > 0.0)) {
      if (gt == 0) *err = 1;
      return;  // every block sees the same pivot
    }
    const double piv = __dsqrt_rn(s);
    for (int64_t i = j + 1 + gt; i < n; i += gs) L[(size_t)i * n + j] = __ddiv_rn(L[(size_t)i * n + j], piv);
    grid.sync();
    if (gt == 0) L[(size_t)j * n + j] = piv;
    for (int64_t i = j + 1 + gw; i < n; i += nw) {
      const double lij = L[(size_t)i * n + j];
      double* row = L + (size_t)i * n;
      for (int64_t m = j + 1 + lane; m <= i; m += 32) row[m] = __dsub_rn(row[m], __dmul_rn(lij, L[(size_t)m * n + j]));
    }
    grid.sync();
  }
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

// ---------------------------------------------------------------- closed-form lattice level
// With the exact in-box 15-point stencil verified on an L^3 box, the greedy
// C/F split is the all-even set (lat_flags_kernel) and everything the level
// needs follows in closed form:
//   * P row of fine point p with odd axes S: C -> (p/2, 1); F -> p - e_S and,
//     when inside the box, p + e_S, each with weight 1/count (p_fill_kernel);
//   * P^T row of coarse point I: the fine points 2I + d, d in the stencil
//     (ascending), with the same weights (every other fine point misses I);
//   * row offsets of both are lexicographic counts of per-axis predicates;
//   * A_c = P^T (A P) entry (I, J) = sum over ascending k in P^T row I of
//     P_kI * (sum over ascending m in A row k of A_km * P_mJ) -- the order of
//     the two ordered Eigen products (lat_ap_kernel / lat_ptap_kernel), fused
//     per coarse row with every window slot a compile-time register.
namespace latc {
struct Stencil {
  int d[15][3];
};
// ascending linear offset (same table as lattice_check_kernel)
constexpr Stencil kSt = {{{-1, -1, -1}, {0, -1, -1}, {-1, 0, -1}, {0, 0, -1}, {-1, -1, 0},
                          {0, -1, 0},   {-1, 0, 0},  {0, 0, 0},   {1, 0, 0},  {0, 1, 0},
                          {1, 1, 0},    {0, 0, 1},   {1, 0, 1},   {0, 1, 1},  {1, 1, 1}}};
constexpr int st(int j, int a) { return kSt.d[j][a]; }
constexpr int slot(int ox, int oy, int oz) { return (oz + 1) * 9 + (oy + 1) * 3 + (ox + 1); }
// 2I + e inside the fine box along one axis, e in [-2, 2]
struct Ax {
  bool lo, h1, h2;  // I >= 1, 2I + 1 < L, 2I + 2 < L
};
template <int E>
__device__ __forceinline__ bool inb(const Ax& a) {
  static_assert(E >= -2 && E <= 2, "offset");
  if constexpr (E < 0) return a.lo;
  else if constexpr (E == 0) return true;
  else if constexpr (E == 1) return a.h1;
  else return a.h2;
}
// window slots of A_c row I that AP row 2I + d(KD) can reach
constexpr unsigned touched(int kd) {
  unsigned m = 0;
  for (int md = 0; md < 15; ++md) {
    const int e[3] = {st(kd, 0) + st(md, 0), st(kd, 1) + st(md, 1), st(kd, 2) + st(md, 2)};
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int a = 0; a < 3; ++a) {
      const int odd = e[a] & 1;
      lo[a] = (e[a] - odd) / 2;
      hi[a] = (e[a] + odd) / 2;
    }
    m |= 1u << slot(lo[0], lo[1], lo[2]);
    m |= 1u << slot(hi[0], hi[1], hi[2]);
  }
  return m;
}

template <int KD, int MD>
__device__ __forceinline__ void ap_term(double (&V)[27], int& pos, const double* __restrict__ av, const Ax& ax,
                                        const Ax& ay, const Ax& az) {
  constexpr int ex = st(KD, 0) + st(MD, 0), ey = st(KD, 1) + st(MD, 1), ez = st(KD, 2) + st(MD, 2);
  if (!(inb<ex>(ax) && inb<ey>(ay) && inb<ez>(az))) return;
  const double a = av[pos++];
  constexpr int sx = ex & 1, sy = ey & 1, sz = ez & 1;
  if constexpr ((sx | sy | sz) == 0) {  // m is a C point: P row (m/2, 1)
    constexpr int s = slot(ex / 2, ey / 2, ez / 2);
    V[s] = __dadd_rn(V[s], __dmul_rn(1.0, a));
  } else {  // F point: low m - e_S, high m + e_S when inside (only +1 offsets can leave the box)
    const bool hin = (!(sx && ex == 1) || ax.h2) && (!(sy && ey == 1) || ay.h2) && (!(sz && ez == 1) || az.h2);
    const double t = __dmul_rn(hin ? 0.5 : 1.0, a);
    constexpr int sl = slot((ex - sx) / 2, (ey - sy) / 2, (ez - sz) / 2);
    constexpr int sh = slot((ex + sx) / 2, (ey + sy) / 2, (ez + sz) / 2);
    V[sl] = __dadd_rn(V[sl], t);
    if (hin) V[sh] = __dadd_rn(V[sh], t);
  }
}

template <int KD, int... MD>
__device__ __forceinline__ void k_term(double (&W)[27], int k0, int L, const int* __restrict__ arp,
                                       const double* __restrict__ av, const Ax& ax, const Ax& ay, const Ax& az,
                                       std::integer_sequence<int, MD...>) {
  constexpr int dx = st(KD, 0), dy = st(KD, 1), dz = st(KD, 2);
  if (!(inb<dx>(ax) && inb<dy>(ay) && inb<dz>(az))) return;
  const int k = k0 + (dz * L + dy) * L + dx;
  double wk;  // P_kI
  if constexpr (dx == 0 && dy == 0 && dz == 0)
    wk = 1.0;
  else if constexpr (dx <= 0 && dy <= 0 && dz <= 0)
    wk = 0.5;
  else
    wk = (inb<2 * dx>(ax) && inb<2 * dy>(ay) && inb<2 * dz>(az)) ? 0.5 : 1.0;
  double V[27];
#pragma unroll
  for (int s = 0; s < 27; ++s) V[s] = 0.0;
  int pos = arp[k];
  (ap_term<KD, MD>(V, pos, av, ax, ay, az), ...);
  constexpr unsigned tm = touched(KD);
#pragma unroll
  for (int s = 0; s < 27; ++s)
    if ((tm >> s) & 1u) W[s] = __dadd_rn(W[s], __dmul_rn(V[s], wk));
}

template <int... KD>
__device__ __forceinline__ void rap_row(double (&W)[27], int k0, int L, const int* __restrict__ arp,
                                        const double* __restrict__ av, const Ax& ax, const Ax& ay, const Ax& az,
                                        std::integer_sequence<int, KD...>) {
  (k_term<KD>(W, k0, L, arp, av, ax, ay, az, std::make_integer_sequence<int, 15>{}), ...);
}

// Row offsets of a stencil-structured CSR over a box of side n: row I holds the
// offsets d of the 15-point table with pred(d_a, I_a) on every axis, where
// pred(-1, u) = u >= 1, pred(0, u) = true, pred(+1, u) = u < mp.  The offset of
// row I is the lexicographic count of (row, d) pairs before it.
__device__ __forceinline__ long long cnt_pred(int d, int v, int mp) {
  return d < 0 ? (v > 0 ? v - 1 : 0) : d == 0 ? v : min(v, mp);
}
__device__ __forceinline__ bool pred(int d, int u, int mp) { return d < 0 ? u >= 1 : d == 0 ? true : u < mp; }
__device__ __forceinline__ void stencil_offset(const int (&D)[15][3], int n, int mp, int ix, int iy, int iz,
                                               long long& o, long long& tot) {
  o = 0;
  tot = 0;
#pragma unroll
  for (int j = 0; j < 15; ++j) {
    const int dx = D[j][0], dy = D[j][1], dz = D[j][2];
    const long long nx = cnt_pred(dx, n, mp), ny = cnt_pred(dy, n, mp);
    o += cnt_pred(dz, iz, mp) * ny * nx +
         (pred(dz, iz, mp) ? cnt_pred(dy, iy, mp) * nx + (pred(dy, iy, mp) ? cnt_pred(dx, ix, mp) : 0) : 0);
    tot += cnt_pred(dz, n, mp) * ny * nx;
  }
}
}  // namespace latc

constexpr int kRapNT = 128;
#define RD_LAT_D15                                                                                       \
  {{-1, -1, -1}, {0, -1, -1}, {-1, 0, -1}, {0, 0, -1}, {-1, -1, 0}, {0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, \
   {1, 0, 0},    {0, 1, 0},   {1, 1, 0},   {0, 0, 1},  {1, 0, 1},   {0, 1, 1},  {1, 1, 1}}

// DIRECT: write A_c straight into its 15-point lattice CSR (closed-form offsets)
// and only flag a pattern mismatch; otherwise the 27-slot window rows go to
// `out` / `cnt` for the scan + compaction of the exact (pruned) pattern.
template <bool DIRECT>
__global__ void __launch_bounds__(kRapNT) lat_rap_kernel(int nc, int Lc, int L, const int* __restrict__ arp,
                                                         const double* __restrict__ av, double* out, int* cnt,
                                                         int* crp, int* cci, double* cv, int* notlat) {
  const int I = blockIdx.x * kRapNT + threadIdx.x;
  if (I >= nc) return;
  const int ix = I % Lc, iy = I / Lc % Lc, iz = I / (Lc * Lc);
  const latc::Ax ax{ix >= 1, 2 * ix + 1 < L, 2 * ix + 2 < L};
  const latc::Ax ay{iy >= 1, 2 * iy + 1 < L, 2 * iy + 2 < L};
  const latc::Ax az{iz >= 1, 2 * iz + 1 < L, 2 * iz + 2 < L};
  double W[27];
#pragma unroll
  for (int s = 0; s < 27; ++s) W[s] = 0.0;
  latc::rap_row(W, (2 * iz * L + 2 * iy) * L + 2 * ix, L, arp, av, ax, ay, az,
                std::make_integer_sequence<int, 15>{});
  int c = 0;
  bool bad = false;
  long long o = 0;
  if (DIRECT) {
    const int D[15][3] = RD_LAT_D15;
    long long tot;
    latc::stencil_offset(D, Lc, Lc - 1, ix, iy, iz, o, tot);
    crp[I] = (int)o;
    if (I == nc - 1) crp[nc] = (int)tot;
  }
#pragma unroll
  for (int s = 0; s < 27; ++s) {
    const int ox = s % 3 - 1, oy = s / 3 % 3 - 1, oz = s / 9 - 1;
    const bool same = (ox >= 0 && oy >= 0 && oz >= 0) || (ox <= 0 && oy <= 0 && oz <= 0);
    const bool in = (unsigned)(ix + ox) < (unsigned)Lc && (unsigned)(iy + oy) < (unsigned)Lc &&
                    (unsigned)(iz + oz) < (unsigned)Lc;
    const bool nz = W[s] != 0.0;
    bad |= nz != (same && in);  // A_c keeps the exact in-box 15-point pattern?
    if (DIRECT) {
      if (same && in) {  // slots ascend with the column index
        cci[o] = I + (oz * Lc + oy) * Lc + ox;
        cv[o] = W[s];
        ++o;
      }
    } else {
      c += nz;
      out[(size_t)s * nc + I] = W[s];
    }
  }
  if (!DIRECT) cnt[I] = c;
  if (bad) atomicExch(notlat, 1);
}

// P of a lattice level: rows, row offsets (closed form) and the C/F flags
__global__ void lat_p_kernel(int L, int Lc, int* rp, int* ci, double* v, uint8_t* flags) {
  const int n = L * L * L;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int x = i % L, y = i / L % L, z = i / (L * L);
  // row length 1 + [F and p + e_S inside]; [F and inside] = [ok] - [even] with
  // ok(u) = (u != L - 1 or L odd); counts below i in lexicographic order
  const int nok = L - ((L & 1) ? 0 : 1);
  auto okc = [&](int u) { return u; };  // #{u' < u : ok(u')} for u <= L - 1
  auto ok = [&](int u) { return (L & 1) || u != L - 1; };
  const long long below_ok =
      (long long)okc(z) * nok * nok + (ok(z) ? (long long)okc(y) * nok + (ok(y) ? okc(x) : 0) : 0);
  auto evc = [](int u) { return (u + 1) >> 1; };
  const long long below_even = (long long)evc(z) * Lc * Lc + (!(z & 1) ? (long long)evc(y) * Lc + (!(y & 1) ? evc(x) : 0) : 0);
  const int o = (int)(i + below_ok - below_even);
  rp[i] = o;
  if (i == n - 1) rp[n] = (int)((long long)n + (long long)nok * nok * nok - (long long)Lc * Lc * Lc);
  const int sx = x & 1, sy = y & 1, sz = z & 1;
  const int lo = ((z >> 1) * Lc + (y >> 1)) * Lc + (x >> 1);
  if (!(sx | sy | sz)) {
    flags[i] = 1;
    ci[o] = lo;
    v[o] = 1.0;
    return;
  }
  flags[i] = 0;
  const bool hin = (!sx || x + 1 < L) && (!sy || y + 1 < L) && (!sz || z + 1 < L);
  const double w = __ddiv_rn(1.0, hin ? 2.0 : 1.0);
  ci[o] = lo;
  v[o] = w;
  if (hin) {
    ci[o + 1] = (((z + sz) >> 1) * Lc + ((y + sy) >> 1)) * Lc + ((x + sx) >> 1);
    v[o + 1] = w;
  }
}

// P^T of a lattice level (closed form; same rows as transpose(P))
__global__ void lat_pt_kernel(int L, int Lc, int* rp, int* ci, double* v) {
  const int nc = Lc * Lc * Lc;
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= nc) return;
  const int ix = I % Lc, iy = I / Lc % Lc, iz = I / (Lc * Lc);
  const int D[15][3] = RD_LAT_D15;
  long long o, tot;
  latc::stencil_offset(D, Lc, L / 2, ix, iy, iz, o, tot);  // 2I + d inside: I_a < L/2 for d_a = +1
  rp[I] = (int)o;
  if (I == nc - 1) rp[nc] = (int)tot;
  const int k0 = (2 * iz * L + 2 * iy) * L + 2 * ix;
#pragma unroll
  for (int j = 0; j < 15; ++j) {
    const int dx = D[j][0], dy = D[j][1], dz = D[j][2];
    if (!(latc::pred(dx, ix, L / 2) && latc::pred(dy, iy, L / 2) && latc::pred(dz, iz, L / 2))) continue;
    double w = 1.0;
    if (j != 7) {
      const bool neg = dx <= 0 && dy <= 0 && dz <= 0;
      const bool hin = neg || ((dx == 0 || 2 * ix + 2 < L) && (dy == 0 || 2 * iy + 2 < L) && (dz == 0 || 2 * iz + 2 < L));
      w = __ddiv_rn(1.0, hin ? 2.0 : 1.0);
    }
    ci[o] = k0 + (dz * L + dy) * L + dx;
    v[o] = w;
    ++o;
  }
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

void dense_llt(Ctx& c, const DCsr& A, DBuf<double>& L, int* err_dev) {
  const int n = A.rows;
  L.alloc((size_t)n * n, c.stream);
  RDG_CUDA(cudaMemsetAsync(L.p, 0, sizeof(double) * n * n, c.stream));
  to_dense_kernel<<<n, 64, 0, c.stream>>>(n, A.rp.p, A.ci.p, A.v.p, L.p);
  RDG_LAUNCH_CHECK();
  DBuf<int> err;
  if (!err_dev) {
    err.alloc(1, c.stream);
    RDG_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), c.stream));
  }
  if (llt_smem(n) <= (size_t)kLltSmemMax) {
    static bool attr = false;
    if (!attr) {
      RDG_CUDA(cudaFuncSetAttribute(llt_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kLltSmemMax));
      attr = true;
    }
    llt_kernel<true><<<1, 256, llt_smem(n), c.stream>>>(n, L.p, err_dev ? err_dev : err.p);
  } else {  // the whole GPU (cooperative launch: every block resident)
    int per_sm = 0;
    RDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, llt_right_kernel, 256, 0));
    const int blocks = std::max(1, per_sm * c.num_sms);
    int* ep = err_dev ? err_dev : err.p;
    int nn = n;
    double* lp = L.p;
    void* args[] = {&nn, &lp, &ep};
    RDG_CUDA(cudaLaunchCooperativeKernel((const void*)llt_right_kernel, dim3(blocks), dim3(256), args, 0, c.stream));
    ++c.launches;
  }
  RDG_LAUNCH_CHECK();
  c.launches += 2;
  if (!err_dev && read_int(c, err.p)) throw Error(RD_ENOTSPD, "build_amg: coarsest level not positive definite");
}

namespace {
bool lattice_cube(const DCsr& A) { return A.lat.ok && A.lat.lx == A.lat.ly && A.lat.ly == A.lat.lz; }

// total of latc::stencil_offset on the host
int64_t stencil_total(int n, int mp) {
  const int D[15][3] = RD_LAT_D15;
  auto N = [&](int d) -> int64_t { return d < 0 ? std::max(n - 1, 0) : d == 0 ? n : std::min(n, mp); };
  int64_t t = 0;
  for (auto& d : D) t += N(d[0]) * N(d[1]) * N(d[2]);
  return t;
}

// One lattice level in closed form (see lat_rap_kernel): P, P^T and the flags
// without scans or host round trips.  direct: A_c goes straight into the
// 15-point lattice layout and *notlat_dev records whether that was exact (the
// caller checks once, after the whole hierarchy); otherwise A_c is compacted
// from its window rows with one host round trip for its size.
void lattice_level(Ctx& c, Level& lv, DCsr& Ac, int* notlat_dev, bool direct) {
  const DCsr& A = lv.A;
  const int L = A.lat.lx, Lc = (L + 1) / 2, n = A.rows, nc = Lc * Lc * Lc;
  const int nok = L - ((L & 1) ? 0 : 1);
  const int64_t pnnz = (int64_t)n + (int64_t)nok * nok * nok - nc;
  const int64_t cnnz = stencil_total(Lc, Lc - 1);
  if (pnnz > 0x7fffffffLL || cnnz > 0x7fffffffLL)
    throw Error(RD_EINVAL, "index overflow: more than INT32_MAX entries (SpMat<int>)");
  lv.flags.alloc(n, c.stream);
  DCsr& P = lv.P;
  P = DCsr{};
  P.rows = n;
  P.cols = nc;
  P.nnz = pnnz;
  P.rp.alloc(n + 1, c.stream);
  P.ci.alloc(pnnz, c.stream);
  P.v.alloc(pnnz, c.stream);
  lat_p_kernel<<<div_up(n, 256), 256, 0, c.stream>>>(L, Lc, P.rp.p, P.ci.p, P.v.p, lv.flags.p);
  RDG_LAUNCH_CHECK();
  DCsr& T = lv.Pt;
  T = DCsr{};
  T.rows = nc;
  T.cols = n;
  T.nnz = pnnz;
  T.rp.alloc(nc + 1, c.stream);
  T.ci.alloc(pnnz, c.stream);
  T.v.alloc(pnnz, c.stream);
  lat_pt_kernel<<<div_up(nc, 256), 256, 0, c.stream>>>(L, Lc, T.rp.p, T.ci.p, T.v.p);
  RDG_LAUNCH_CHECK();
  c.launches += 2;
  Ac = DCsr{};
  Ac.rows = Ac.cols = nc;
  Ac.rp.alloc(nc + 1, c.stream);
  Ac.lat_checked = true;
  if (direct) {
    Ac.nnz = cnnz;
    Ac.ci.alloc(cnnz, c.stream);
    Ac.v.alloc(cnnz, c.stream);
    lat_rap_kernel<true><<<div_up(nc, kRapNT), kRapNT, 0, c.stream>>>(nc, Lc, L, A.rp.p, A.v.p, nullptr, nullptr,
                                                                       Ac.rp.p, Ac.ci.p, Ac.v.p, notlat_dev);
    RDG_LAUNCH_CHECK();
    ++c.launches;
    Ac.lat = nc >= 8 ? Lattice{Lc, Lc, Lc, true} : Lattice{};
    return;
  }
  DBuf<int> notlat(1, c.stream), cnt(nc, c.stream);
  DBuf<double> out((size_t)27 * nc, c.stream);
  RDG_CUDA(cudaMemsetAsync(notlat.p, 0, sizeof(int), c.stream));
  lat_rap_kernel<false><<<div_up(nc, kRapNT), kRapNT, 0, c.stream>>>(nc, Lc, L, A.rp.p, A.v.p, out.p, cnt.p,
                                                                      nullptr, nullptr, nullptr, notlat.p);
  RDG_LAUNCH_CHECK();
  ++c.launches;
  int nl = 0;
  Ac.nnz = exclusive_scan(c, cnt.p, Ac.rp.p, nc, notlat.p, &nl);
  Ac.ci.alloc(Ac.nnz, c.stream);
  Ac.v.alloc(Ac.nnz, c.stream);
  lat_compact_kernel<<<div_up(nc, 256), 256, 0, c.stream>>>(nc, Lc, out.p, Ac.rp.p, Ac.ci.p, Ac.v.p);
  RDG_LAUNCH_CHECK();
  ++c.launches;
  // the pattern check of detect_lattice, folded into the product
  Ac.lat = (nl == 0 && nc >= 8) ? Lattice{Lc, Lc, Lc, true} : Lattice{};
}
}  // namespace

namespace {
// RD_PROBES builds (compile-time, diagnostics only): synchronise after each setup
// phase and print its host time; compiled out of the shipped library
struct SetupTrace {
  Ctx& c;
  bool on;
  std::chrono::steady_clock::time_point t0;
  explicit SetupTrace(Ctx& cc) : c(cc), on(RD_PROBES != 0) {
    if (on) {
      cudaStreamSynchronize(c.stream);
      t0 = std::chrono::steady_clock::now();
    }
  }
  void mark(const char* what, int level) {
    if (!on) return;
    cudaStreamSynchronize(c.stream);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[setup] L%d %-10s %8.1f us\n", level, what,
            std::chrono::duration<double, std::micro>(t - t0).count());
    t0 = t;
  }
};
}  // namespace

namespace {
// direct: lattice levels write A_c in the lattice layout without host round
// trips; returns false if one of them turned out not to be exact (then the
// caller rebuilds with direct = false).
bool build_levels(Ctx& c, const DCsr& A, int threshold, int m, Hierarchy& h, bool borrow, bool direct) {
  SetupTrace tr(c);
  h.levels.clear();
  h.smoothing_steps = m;
  constexpr int kMaxLat = 64;  // lattice levels halve the side: at most log2(INT_MAX) of them
  DBuf<int> flags_dev(kMaxLat + 64, c.stream);  // [0, kMaxLat): not-lattice per level; then setup errors
  RDG_CUDA(cudaMemsetAsync(flags_dev.p, 0, sizeof(int) * (kMaxLat + 64), c.stream));
  int nlat = 0;
  DCsr current = borrow ? csr_view(A) : csr_copy(c, A);
  tr.mark("copy", 0);
  while (current.rows > threshold) {
    const int li = (int)h.levels.size();
    Level lv;
    lv.A = std::move(current);
    detect_lattice(c, lv.A);  // lattice levels: closed-form P, P^T and fused Galerkin product
    tr.mark("detect", li);
    if (lattice_cube(lv.A) && nlat < kMaxLat) {
      lattice_level(c, lv, current, flags_dev.p + nlat++, direct);
      lv.has_p = true;
      tr.mark("lattice", li);
      h.levels.push_back(std::move(lv));
      continue;
    }
    DCsr P;
    coarsen(c, lv.A, lv.flags, P);
    tr.mark("coarsen", li);
    if (P.cols >= P.rows) {  // no reduction possible (amg.cpp:98-101)
      current = std::move(lv.A);
      lv.flags.release();
      break;
    }
    lv.P = std::move(P);
    lv.Pt = transpose(c, lv.P);
    lv.has_p = true;
    tr.mark("transpose", li);
    current = galerkin(c, lv.A, lv.P, lv.Pt);
    tr.mark("galerkin", li);
    h.levels.push_back(std::move(lv));
  }
  Level last;
  last.A = std::move(current);
  h.levels.push_back(std::move(last));
  h.nc = h.levels.back().A.rows;
  // setup errors stay on the device until the single read-back below:
  // [kMaxLat] coarsest LLT, [kMaxLat + 1 + l] level l's structured-smoother layout
  const size_t nerr = std::min<size_t>(h.levels.size() + 1, 64);
  int* serr = flags_dev.p + kMaxLat;
  if (h.nc > 0) dense_llt(c, h.levels.back().A, h.Lc, serr);
  tr.mark("llt", (int)h.levels.size() - 1);
  // work vectors; structured-smoother layout per level
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
      lattice_prepare(c, lv.A, 1 + l < nerr ? serr + 1 + l : nullptr);
    }
    tr.mark("prepare", (int)l);
  }
  std::vector<int> f(kMaxLat + nerr);
  RDG_CUDA(cudaMemcpyAsync(f.data(), flags_dev.p, sizeof(int) * f.size(), cudaMemcpyDeviceToHost, c.stream));
  DBuf<int> tail_bad(1, c.stream);  // the one-CTA coarse tail's class check, read with the same sync
  RDG_CUDA(cudaMemsetAsync(tail_bad.p, 0, sizeof(int), c.stream));
  coarse_tail_prepare(c, h, tail_bad.p);
  int tail_bad_h = 0;
  RDG_CUDA(cudaMemcpyAsync(&tail_bad_h, tail_bad.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  std::vector<int> uni(2 * h.levels.size(), -1);  // smoother stencil uniformity, read with the same sync
  for (size_t l = 0; l < h.levels.size(); ++l)
    if (h.levels[l].A.lat_uni_state == -2)
      RDG_CUDA(cudaMemcpyAsync(&uni[2 * l], h.levels[l].A.lat_uni_flag.p, 2 * sizeof(int), cudaMemcpyDeviceToHost,
                               c.stream));
  RDG_CUDA(cudaStreamSynchronize(c.stream));
  for (int l = 0; l < nlat; ++l)
    if (f[l]) return false;  // a lattice A_c lost the 15-point pattern: rebuild exactly
  if (f[kMaxLat]) throw Error(RD_ENOTSPD, "build_amg: coarsest level not positive definite");
  for (size_t l = 1; l < nerr; ++l) {
    if (f[kMaxLat + l] == 2) throw Error(RD_EZERODIAG, "sgs_sweep: zero diagonal");
    if (f[kMaxLat + l]) throw Error(RD_ERUNTIME, "lattice smoother: pattern/layout mismatch");
  }
  for (size_t l = 0; l < h.levels.size(); ++l)
    if (uni[2 * l] >= 0) lattice_resolve(c, h.levels[l].A, &uni[2 * l]);  // packs only where needed
  if (tail_bad_h) h.tail_level = -1;
  if (RD_PROBES)
    fprintf(stderr, "coarse tail: level %d (class check %s)\n", h.tail_level, tail_bad_h ? "failed" : "ok");
  return true;
}
}  // namespace

void build_hierarchy(Ctx& c, const DCsr& A, int threshold, int m, Hierarchy& h, bool borrow) {
  if (!build_levels(c, A, threshold, m, h, borrow, /*direct=*/true)) build_levels(c, A, threshold, m, h, borrow, false);
}

void dense_llt_solve(Ctx& c, int n, const double* L, const double* b, double* x) {
  if (n == 0) return;
  llt_solve_kernel<<<1, kCoarseNT, sizeof(double) * n, c.stream>>>(n, L, b, x);
  RDG_LAUNCH_CHECK();
  ++c.launches;
}

void coarse_solve(Ctx& c, Hierarchy& h, const double* r, double* z) {
  const int n = h.nc;
  if (n == 0) return;
  llt_solve_kernel<<<1, kCoarseNT, sizeof(double) * n, c.stream>>>(n, h.Lc.p, r, z);
  RDG_LAUNCH_CHECK();
  ++c.launches;
}

// V-cycle with zero initial guess (amg.cpp:119-132), unrolled over levels.
void vcycle(Ctx& c, Hierarchy& h, const double* r, double* z, double* dot_out, int l0) {
  const int L = static_cast<int>(h.levels.size());
  const int m = h.smoothing_steps;
  if (l0 == L - 1) {
    coarse_solve(c, h, r, z);
    if (dot_out) dot(c, h.nc, r, z, dot_out);
    return;
  }
  const int ct = coarse_tail_level(c, h);
  const int tl = ct >= 0 ? std::max(ct, l0) : -1;  // the one-CTA tail takes levels >= tl
  if (tl == l0) {
    coarse_tail(c, h, l0, r, z);
    if (dot_out) dot(c, h.levels[l0].A.rows, r, z, dot_out);
    return;
  }
  const int lend = tl >= 0 ? tl : L - 1;  // levels [l0, lend) smoothed here
  std::vector<const double*> rl(L);
  std::vector<double*> zl(L);
  rl[l0] = r;
  zl[l0] = z;
  for (int l = l0 + 1; l < L; ++l) {
    rl[l] = h.levels[l].r.p;
    zl[l] = h.levels[l].z.p;
  }
  for (int l = l0; l < lend; ++l) {
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
  if (tl >= 0)
    coarse_tail(c, h, tl, rl[tl], zl[tl]);
  else
    coarse_solve(c, h, rl[L - 1], zl[L - 1]);
  for (int l = lend - 1; l >= l0; --l) {
    Level& lv = h.levels[l];
    prolong_add(c, lv.P, zl[l + 1], zl[l]);
    for (int s = 0; s < m; ++s) {
      gs_pass(c, lv.A, rl[l], zl[l], lv.t.p, true);
      const bool last = (l == l0 && s == m - 1);
      gs_pass(c, lv.A, rl[l], lv.t.p, zl[l], false, last ? dot_out : nullptr, last ? rl[l0] : nullptr);
    }
  }
  if (m == 0 && dot_out) dot(c, h.levels[l0].A.rows, r, z, dot_out);
}

}  // namespace rdg
