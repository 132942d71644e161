// coarse_tail.cu -- the bottom of the V-cycle (amg.cpp:119-132) in ONE thread block.
//
// Below a 16^3 lattice level the multi-CTA smoother is all fixed cost: a launch,
// a prologue and tile hand-offs for a wavefront of at most 46 steps.  From the
// first such level down, every operation of the V-cycle -- symmetric Gauss-Seidel
// pre-smoothing, residual, restriction, the coarsest dense LLT solve,
// prolongation, post-smoothing -- runs in a single CTA with all vectors resident
// in shared memory and one __syncthreads between dependent steps:
//
//  * Gauss-Seidel in place on the shared-memory x, one thread per x-line, as a
//    wavefront over a + y + z (reflected for the backward pass).  Rows of one
//    wavefront step never couple on the 15-point stencil, rows of earlier steps
//    already hold new values and rows of later steps old ones -- exactly the
//    sequential relax(i) of amg.cpp:67-88, same operands in the same order;
//  * matrix values row-major in slot order (the lattice stencil's ascending
//    column order, absent slots predicated away), one 128-byte row per thread per
//    step, prefetched a step ahead;
//  * residual, P^T and P row by row, sums from +0 in column order as spmv does
//    (linalg.cpp:19-33); the LLT substitutions in the order of llt_solve_kernel.
//
// Bit-identical to the multi-launch V-cycle; ~20 launches per V-cycle become one.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "internal.hpp"

namespace rdg {
namespace {

constexpr int kTailNT = 256;
constexpr int kTailMaxL = 16;  // lattice side: L^2 <= kTailNT lines
// shared-memory stride (doubles) of a class row: odd in 8-byte words * 2, so the same slot of
// different rows falls in different banks (a warp's rows of one step span several classes)
constexpr int kTbS = 17;

struct TailLev {
  int n, L;
  const double* table;                              // [64][16] class rows (slot order, recip in 15)
  const int* prp; const int* pci; const double* pv;  // P_l
  const int* trp; const int* tci; const double* tv;  // Pt_l
};

struct TailParams {
  int nlev;  // smoothed levels of the tail
  TailLev lv[kTailMaxLevels];
  int nc;
  const double* Lc;
  const double* r;
  double* z;
  int* err;
  int m;  // smoothing steps
  long long* clk;  // RD_PROBES builds only: phase timestamps of thread 0 (else null)
};

__device__ __forceinline__ unsigned tail_mask(int a, int y, int z, int L) {
  const bool am = a > 0, ap = a < L - 1, ym = y > 0, yp = y < L - 1, zm = z > 0, zp = z < L - 1;
  return (unsigned)(am && ym && zm) | (unsigned)(ym && zm) << 1 | (unsigned)(am && zm) << 2 | (unsigned)zm << 3 |
         (unsigned)(am && ym) << 4 | (unsigned)ym << 5 | (unsigned)am << 6 | 1u << 7 | (unsigned)ap << 8 |
         (unsigned)yp << 9 | (unsigned)(ap && yp) << 10 | (unsigned)zp << 11 | (unsigned)(ap && zp) << 12 |
         (unsigned)(yp && zp) << 13 | (unsigned)(ap && yp && zp) << 14;
}

__device__ __forceinline__ void l2_prefetch(const void* src, unsigned bytes) {
  if (bytes >= 16) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes & ~15u) : "memory");
}



extern __shared__ __align__(16) double tail_sm[];  // every vector of the tail (offsets below)

// z vectors live zero-padded, (L+2)^3 with a +0 halo: an absent slot of a class
// row is +0 and reads a halo +0, so its term is +0 * +0 = +0 and s - (+0) == s for
// every s -- the boundary rows need no predicates and the row sum is a plain chain.
__device__ __forceinline__ int padi(int a, int y, int z, int L) { return (a + 1) + (L + 2) * ((y + 1) + (L + 2) * (z + 1)); }
// (the phases between the sweeps run once per V-cycle from a cold instruction cache, so their
// code is kept compact: no inlined integer divisions, one copy of tail_spmv)
__device__ __noinline__ int padof_div(int i, int L) { return padi(i % L, (i / L) % L, i / (L * L), L); }
__device__ __forceinline__ int padof(int i, int L) {
  if ((L & (L - 1)) == 0) {  // power-of-two side: shifts (uniform branch)
    const int sh = 31 - __clz(L);
    return padi(i & (L - 1), (i >> sh) & (L - 1), i >> (2 * sh), L);
  }
  return padof_div(i, L);
}

// one Gauss-Seidel pass in place on the padded x (shared), f (shared), the level's
// class rows (tb, shared): nothing in the step loop touches global memory (a
// pending global load would hold every step's __syncthreads).
template <bool FWD>
__device__ void tail_sweep(const TailLev& lv, int fo, int xo, int tbo, int* err) {
  const double* f = tail_sm + fo;
  double* x = tail_sm + xo;
  const double* tb = tail_sm + tbo;
  const int L = lv.L, P = L * L, Q = L + 2, QQ = Q * Q;
  const int line = threadIdx.x;
  const bool has = line < P;
  const int y = has ? line % L : 0, z = has ? line / L : 0;
  const int yo = FWD ? y : L - 1 - y, zo = FWD ? z : L - 1 - z;
  const int base = (zo * L + yo) * L, pbase = padi(0, yo, zo, L);
  const int cyz = pos_class(yo, L) * 4 + pos_class(zo, L);
  // Neighbour values by sweep-direction offset (the 15-point set is centrally symmetric,
  // so both directions see the same offsets): per step 7 loads -- the three fresh rows of
  // the y-1 / z-1 / yz-1 lines, the old a+1 rows of this and the +y / +z / +yz lines --
  // and the rest from the previous step's registers (row a-1 fresh, row a old).  The
  // thread runs the loads from row -1 (padding), so the first row starts from them.
  const int sg = FWD ? 1 : -1;
  const int oXp = sg, oY0 = -sg * Q, oZ0 = -sg * QQ, oD0 = -sg * (Q + QQ);
  const int oYp = sg * (1 + Q), oZp = sg * (1 + QQ), oYZp = sg * (1 + Q + QQ);
  double X1 = 0.0, Y1 = 0.0, Z1 = 0.0, D1 = 0.0;  // row a-1 of this / y-1 / z-1 / yz-1 lines (fresh)
  double Yp0 = 0.0, Zp0 = 0.0, YZp0 = 0.0;         // row a of the +y / +z / +yz lines (old)
  // the class row of this line's x-interior rows lives in registers; the rows at a = 0, L-2,
  // L-1 come from the table on a rarely taken branch (every class row starts at the same
  // shared-memory bank, so a warp reading n different rows per step pays an n-way conflict)
  double U[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) U[k] = tb[(1 * 16 + cyz) * kTbS + k];
  const int steps = 3 * (L - 1) + 1;
  for (int s = -1; s < steps; ++s) {
    const int a = s - y - z;
    if (has && a >= -1 && a < L) {
      const int ao = FWD ? a : L - 1 - a;
      const int ip = pbase + ao;
      const double Xp = x[ip + oXp], Y0 = x[ip + oY0], Z0 = x[ip + oZ0], D0 = x[ip + oD0];
      const double Yp1 = x[ip + oYp], Zp1 = x[ip + oZp], YZp1 = x[ip + oYZp];
      double xn = 0.0;
      if (a >= 0) {
        const int cx = pos_class(ao, L);
        double v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = U[k];
        if (cx != 1) {
          const double* row = tb + (cx * 16 + cyz) * kTbS;
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] = row[k];
        }
        // ascending original column order: the sweep-offset slots in the reference's order
        const double nf[15] = {D1, D0, Z1, Z0, Y1, Y0, X1, 0.0, Xp, Yp0, Yp1, Zp0, Zp1, YZp0, YZp1};
        const double nr[15] = {YZp1, YZp0, Zp1, Zp0, Yp1, Yp0, Xp, 0.0, X1, Y0, Y1, Z0, Z1, D0, D1};
        const double(&nb)[15] = FWD ? nf : nr;
        double sum = f[base + ao];
#pragma unroll
        for (int k = 0; k < 15; ++k)
          if (k != 7) sum = __dsub_rn(sum, __dmul_rn(v[k], nb[k]));
        const double d = v[7];
        if (d == 0.0) atomicCAS(err, 0, RD_EZERODIAG);
        double q = div_fast(sum, d, v[15]);
        if (!(sum == 0.0 || div_is_fast(sum, d, q))) q = div_exact(sum, d);
        xn = sum == 0.0 ? __dmul_rn(sum, v[15]) : q;
        x[ip] = xn;
      }
      X1 = xn;  // row -1: the padding's +0
      Y1 = Y0;
      Z1 = Z0;
      D1 = D0;
      Yp0 = Yp1;
      Zp0 = Zp1;
      YZp0 = YZp1;
    }
    __syncthreads();
  }
}

// res = r - A z (the lattice rows; z padded), all in shared memory
__device__ void tail_residual(const TailLev& lv, int ro, int zo, int reso, int tbo) {
  const double* r = tail_sm + ro;
  const double* z = tail_sm + zo;
  double* res = tail_sm + reso;
  const double* tb = tail_sm + tbo;
  const int L = lv.L, P = L * L, Q = L + 2, QQ = Q * Q;
  const int off[15] = {-1 - Q - QQ, -Q - QQ, -1 - QQ, -QQ, -1 - Q, -Q, -1, 0, 1, Q, 1 + Q, QQ, 1 + QQ, Q + QQ, 1 + Q + QQ};
  if ((L & (L - 1)) == 0 && (kTailNT % P == 0 || P % kTailNT == 0)) {
    // power-of-two side: a thread's rows i = tid + j * kTailNT share (a, y) and walk z, so the
    // row of its z-interior class lives in registers; the rows at z = 0, L-2, L-1 come from
    // the table (z is warp-uniform for L >= 8, so the branch does not diverge)
    const int sh = 31 - __clz(L);
    const int a = threadIdx.x & (L - 1), y = (threadIdx.x >> sh) & (L - 1);
    const int cay = (pos_class(a, L) * 4 + pos_class(y, L)) * 4;
    double U[15];
#pragma unroll
    for (int k = 0; k < 15; ++k) U[k] = tb[(cay + 1) * kTbS + k];
    for (int i = threadIdx.x; i < lv.n; i += kTailNT) {
      const int zz = i >> (2 * sh), cz = pos_class(zz, L);
      double v[15];
#pragma unroll
      for (int k = 0; k < 15; ++k) v[k] = U[k];
      if (cz != 1) {
#pragma unroll
        for (int k = 0; k < 15; ++k) v[k] = tb[(cay + cz) * kTbS + k];
      }
      const int ip = padi(a, y, zz, L);
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 15; ++k) s = __dadd_rn(s, __dmul_rn(v[k], z[ip + off[k]]));
      res[i] = __dsub_rn(r[i], s);
    }
    return;
  }
  for (int i = threadIdx.x; i < lv.n; i += kTailNT) {
    const int a = i % L, y = (i / L) % L, zz = i / P;
    const double* v = tb + ((pos_class(a, L) * 4 + pos_class(y, L)) * 4 + pos_class(zz, L)) * kTbS;
    const int ip = padi(a, y, zz, L);
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 15; ++k) s = __dadd_rn(s, __dmul_rn(v[k], z[ip + off[k]]));
    res[i] = __dsub_rn(r[i], s);
  }
}

// y = M x for a CSR block in global memory (x, y shared; xL / yL > 0: that vector is
// padded for a side-L lattice), sums from +0; four rows in flight per thread
template <bool CHUNKED>
__device__ __noinline__ void tail_spmv(int rows, const int* rp, const int* ci, const double* val, int xo, int xL, int yo, int yL,
                          bool add) {
  const double* x = tail_sm + xo;
  double* y = tail_sm + yo;
  constexpr int U = 4;
  for (int i0 = threadIdx.x; i0 < rows; i0 += kTailNT * U) {
    int b[U], e[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * kTailNT;
      b[u] = i < rows ? __ldg(rp + i) : 0;
      e[u] = i < rows ? __ldg(rp + i + 1) : 0;
    }
    if constexpr (!CHUNKED) {  // long rows (P^T: up to 15 entries), few of them per thread
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * kTailNT;
        if (i >= rows) break;
        double s = 0.0;
        for (int k = b[u]; k < e[u]; ++k) {
          const int c = __ldg(ci + k);
          s = __dadd_rn(s, __dmul_rn(__ldg(val + k), x[xL ? padof(c, xL) : c]));
        }
        const int yi = yL ? padof(i, yL) : i;
        y[yi] = add ? __dadd_rn(y[yi], s) : s;
      }
      continue;
    }
    // short rows (P): entries in chunks of E per row, the chunk's loads of all U rows issued
    // before any is used (global latency is paid once per chunk, not once per entry); sums in
    // entry order
    constexpr int E = 4;
    double sacc[U];
    int len = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      sacc[u] = 0.0;
      len = max(len, e[u] - b[u]);
    }
    for (int o = 0; o < len; o += E) {
      int cc[U][E];
      double vv[U][E];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const int k = b[u] + o + j;
          const bool in = k < e[u];
          cc[u][j] = in ? __ldg(ci + k) : 0;
          vv[u][j] = in ? __ldg(val + k) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < E; ++j)
          if (b[u] + o + j < e[u])
            sacc[u] = __dadd_rn(sacc[u], __dmul_rn(vv[u][j], x[xL ? padof(cc[u][j], xL) : cc[u][j]]));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * kTailNT;
      if (i >= rows) break;
      const int yi = yL ? padof(i, yL) : i;
      y[yi] = add ? __dadd_rn(y[yi], sacc[u]) : sacc[u];
    }
  }
}

// the coarsest LLT substitutions (the order of llt_solve_kernel) by warp 0 alone:
// lane l keeps rows l, l+32, ... in registers, the pivot's quotient is broadcast by
// shuffle, divisions on the diagonal's precomputed reciprocal (exact fallback)
// (the factor sits in shared memory with the odd row stride n | 1: the forward substitution
// reads a column, which at stride n = 64 would put all 32 lanes in one bank)
__device__ void tail_llt(int n, const double* Lm, const double* rcp, double* rc) {
  if (threadIdx.x >= 32) return;
  const int ld = n | 1;
  const int lane = threadIdx.x;
  constexpr int R = 4;  // n <= 128
  double v[R];
#pragma unroll
  for (int j = 0; j < R; ++j) v[j] = lane + 32 * j < n ? rc[lane + 32 * j] : 0.0;
  auto quot = [&](double sk, int k) {
    const double d = Lm[k * ld + k], y = rcp[k];
    double q = div_fast(sk, d, y);
    if (!(sk == 0.0 || div_is_fast(sk, d, q))) q = div_exact(sk, d);
    return sk == 0.0 ? __dmul_rn(sk, y) : q;
  };
  for (int k = 0; k < n; ++k) {
    const int ow = k & 31, oj = k >> 5;
    double sk = 0.0;
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (j == oj) sk = v[j];
    sk = __shfl_sync(0xffffffffu, sk, ow);
    const double yk = quot(sk, k);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int i = lane + 32 * j;
      if (i == k) v[j] = yk;
      if (i > k && i < n) v[j] = __dsub_rn(v[j], __dmul_rn(Lm[i * ld + k], yk));
    }
  }
  for (int k = n - 1; k >= 0; --k) {
    const int ow = k & 31, oj = k >> 5;
    double sk = 0.0;
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (j == oj) sk = v[j];
    sk = __shfl_sync(0xffffffffu, sk, ow);
    const double xk = quot(sk, k);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int i = lane + 32 * j;
      if (i == k) v[j] = xk;
      if (i < k) v[j] = __dsub_rn(v[j], __dmul_rn(Lm[k * ld + i], xk));
    }
  }
#pragma unroll
  for (int j = 0; j < R; ++j)
    if (lane + 32 * j < n) rc[lane + 32 * j] = v[j];
}

__global__ void __launch_bounds__(kTailNT, 1) coarse_tail_kernel(TailParams p) {
  // layout (element offsets into tail_sm): per level k: r_k (n_k), z_k ((L_k+2)^3, padded);
  // then res, rc, the coarsest factor and its diagonal reciprocals, the class rows
  auto zlen = [&](int k) { return (p.lv[k].L + 2) * (p.lv[k].L + 2) * (p.lv[k].L + 2); };
  auto ro = [&](int k) {
    int o = 0;
    for (int j = 0; j < k; ++j) o += p.lv[j].n + zlen(j);
    return o;
  };
  auto zo = [&](int k) { return ro(k) + p.lv[k].n; };
  int maxn = 0;
  for (int k = 0; k < p.nlev; ++k) maxn = max(maxn, p.lv[k].n);
  const int ldc = p.nc | 1;
  const int reso = ro(p.nlev), rco = reso + maxn, lo = rco + p.nc, dro = lo + p.nc * ldc;
  auto tbo = [&](int k) { return ((dro + p.nc + 1) & ~1) + k * 64 * kTbS; };  // class rows
  double* Rc = tail_sm + rco;
  const int tid = threadIdx.x;
  int ck = 0;
  auto mark = [&]() {
    if (p.clk && tid == 0) p.clk[ck] = clock64();
    ++ck;
  };
  pdl_wait();
  pdl_trigger();
  mark();
  // pull P / P^T into L2 first: between V-cycles the fine-level streams evict them
  if (tid >= 32 && tid - 32 < p.nlev) {
    const TailLev& lv = p.lv[tid - 32];
    const unsigned np = (unsigned)lv.prp[lv.n];  // nnz(P) = nnz(P^T)
    l2_prefetch(lv.pci, np * 4);
    l2_prefetch(lv.pv, np * 8);
    l2_prefetch(lv.tci, np * 4);
    l2_prefetch(lv.tv, np * 8);
  }
  // r, the class rows and the coarsest factor arrive through cp.async (all in flight at once)
  auto cp8 = [](double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
  };
  for (int i = tid; i < p.lv[0].n; i += kTailNT) cp8(tail_sm + i, p.r + i);
  for (int k = 0; k < p.nlev; ++k)
    for (int i = tid; i < 64 * 16; i += kTailNT) cp8(tail_sm + tbo(k) + (i >> 4) * kTbS + (i & 15), p.lv[k].table + i);
  for (int i = tid; i < p.nc * p.nc; i += kTailNT) cp8(tail_sm + lo + (i / p.nc) * ldc + i % p.nc, p.Lc + i);
  for (int i = tid; i < p.nc; i += kTailNT) tail_sm[dro + i] = div_recip(__ldg(p.Lc + i * p.nc + i));
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  mark();
  // ---- down: pre-smooth from zero, residual, restrict
  for (int k = 0; k < p.nlev; ++k) {
    const TailLev& lv = p.lv[k];
    for (int i = tid; i < zlen(k); i += kTailNT) tail_sm[zo(k) + i] = 0.0;  // +0, halo included
    __syncthreads();
    for (int s = 0; s < p.m; ++s) {
      tail_sweep<true>(lv, ro(k), zo(k), tbo(k), p.err);
      tail_sweep<false>(lv, ro(k), zo(k), tbo(k), p.err);
    }
    mark();
    tail_residual(lv, ro(k), zo(k), reso, tbo(k));
    __syncthreads();
    mark();
    tail_spmv<false>(k + 1 < p.nlev ? p.lv[k + 1].n : p.nc, lv.trp, lv.tci, lv.tv, reso, 0, k + 1 < p.nlev ? ro(k + 1) : rco,
              0, false);
    __syncthreads();
    mark();
  }
  // ---- coarsest: L y = r, L^T x = y in place on rc
  tail_llt(p.nc, tail_sm + lo, tail_sm + dro, Rc);
  __syncthreads();
  mark();
  // ---- up: prolongate, post-smooth
  for (int k = p.nlev - 1; k >= 0; --k) {
    const TailLev& lv = p.lv[k];
    const bool fromc = k + 1 == p.nlev;
    tail_spmv<true>(lv.n, lv.prp, lv.pci, lv.pv, fromc ? rco : zo(k + 1), fromc ? 0 : p.lv[k + 1].L, zo(k), lv.L, true);
    __syncthreads();
    mark();
    for (int s = 0; s < p.m; ++s) {
      tail_sweep<true>(lv, ro(k), zo(k), tbo(k), p.err);
      tail_sweep<false>(lv, ro(k), zo(k), tbo(k), p.err);
    }
    mark();
  }
  for (int i = tid; i < p.lv[0].n; i += kTailNT) p.z[i] = tail_sm[zo(0) + padof(i, p.lv[0].L)];
}

// the 64 class rows of a verified lattice level: slot values of a representative
// row (absent slots +0) and the diagonal's division reciprocal in slot 15
__global__ void tail_table_kernel(int L, const int* __restrict__ rp, const double* __restrict__ v, double* tb) {
  const int c = threadIdx.x;  // 64 threads: class (ca, cy, cz) = c / 16, c / 4 % 4, c % 4
  if (c >= 64) return;
  const int rep[4] = {0, 1, L - 2, L - 1};
  const int ca = c / 16, cy = c / 4 % 4, cz = c % 4;
  double* o = tb + c * 16;
  for (int sl = 0; sl < 16; ++sl) o[sl] = 0.0;
  o[7] = o[15] = 1.0;
  const int a = rep[ca], y = rep[cy], z = rep[cz];
  if (a < 0 || y < 0 || z < 0 || pos_class(a, L) != ca || pos_class(y, L) != cy || pos_class(z, L) != cz) return;
  const int i = (z * L + y) * L + a;
  const unsigned m = tail_mask(a, y, z, L);
  const int b = rp[i];
  for (int sl = 0; sl < 15; ++sl)
    o[sl] = ((m >> sl) & 1u) ? v[b + __popc(m & ((1u << sl) - 1u))] : 0.0;
  o[15] = o[7] != 0.0 ? div_recip(o[7]) : 1.0;  // nvcc's d-only division part
}

// every row equals its class row slot by slot (bit for bit); else *bad = 1
__global__ void tail_check_kernel(int L, const int* __restrict__ rp, const double* __restrict__ v,
                                  const double* __restrict__ tb, int* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L * L * L) return;
  const int a = i % L, y = (i / L) % L, z = i / (L * L);
  const unsigned m = tail_mask(a, y, z, L);
  const int b = rp[i];
  if (rp[i + 1] - b != __popc(m)) {
    *bad = 1;
    return;
  }
  const double* o = tb + ((pos_class(a, L) * 4 + pos_class(y, L)) * 4 + pos_class(z, L)) * 16;
  for (int sl = 0; sl < 15; ++sl)
    if (((m >> sl) & 1u) &&
        __double_as_longlong(v[b + __popc(m & ((1u << sl) - 1u))]) != __double_as_longlong(o[sl]))
      *bad = 1;
}

size_t tail_smem(const Hierarchy& h, int c0) {
  size_t d = 0, maxn = 0;
  for (size_t l = c0; l + 1 < h.levels.size(); ++l) {
    const size_t Q = (size_t)h.levels[l].A.lat.lx + 2;
    d += (size_t)h.levels[l].A.rows + Q * Q * Q;
    maxn = std::max(maxn, (size_t)h.levels[l].A.rows);
  }
  if (h.nc > 128) return SIZE_MAX;  // tail_llt keeps at most 4 rows per lane
  d += maxn + 2 * (size_t)h.nc + (size_t)h.nc * (h.nc | 1) + 1 + (size_t)(h.levels.size() - 1 - c0) * 64 * kTbS;
  return d * sizeof(double);
}

}  // namespace

// Setup: the first level the one-CTA tail can take.  From there down every
// smoothed level must be a verified cubic lattice of side <= 16 whose rows are
// equal within each position class (the class check runs on the device and
// lands in *bad; the caller reads it with its own sync and drops the tail if set),
// at most kTailMaxLevels of them, the vectors fitting in shared memory.
void coarse_tail_prepare(Ctx& c, Hierarchy& h, int* bad) {
  h.tail_checked = true;
  h.tail_level = -1;
  static const bool off = getenv("RD_NO_COARSE_TAIL") && atoi(getenv("RD_NO_COARSE_TAIL")) != 0;
  const int nl = (int)h.levels.size();
  if (off || nl < 2 || h.nc < 1) return;
  int c0 = nl - 1;
  while (c0 - 1 >= 0) {
    const DCsr& A = h.levels[c0 - 1].A;
    if (!(A.lat.ok && A.lat.lx == A.lat.ly && A.lat.lx == A.lat.lz && A.lat.lx <= kTailMaxL)) break;
    --c0;
  }
  if (c0 == nl - 1) return;  // no small lattice level above the coarsest
  while (nl - 1 - c0 > kTailMaxLevels) ++c0;
  int maxsm = 0;
  RDG_CUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
  while (c0 < nl - 1 && tail_smem(h, c0) > (size_t)maxsm) ++c0;
  if (c0 >= nl - 1) return;
  for (int l = c0; l + 1 < nl; ++l) {
    Level& lv = h.levels[l];
    const int L = lv.A.lat.lx;
    lv.tail_table.alloc(64 * 16, c.stream);
    tail_table_kernel<<<1, 64, 0, c.stream>>>(L, lv.A.rp.p, lv.A.v.p, lv.tail_table.p);
    RDG_LAUNCH_CHECK();
    tail_check_kernel<<<div_up(lv.A.rows, 256), 256, 0, c.stream>>>(L, lv.A.rp.p, lv.A.v.p, lv.tail_table.p, bad);
    RDG_LAUNCH_CHECK();
    c.launches += 2;
  }
  static bool attr = false;
  if (!attr) {
    RDG_CUDA(cudaFuncSetAttribute(coarse_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    attr = true;
  }
  h.tail_level = c0;
}

int coarse_tail_level(Ctx& c, Hierarchy& h) {
  if (!h.tail_checked) {  // a hierarchy assembled without build_hierarchy: check here
    DBuf<int> bad(1, c.stream);
    RDG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c.stream));
    coarse_tail_prepare(c, h, bad.p);
    int hb = 0;
    RDG_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    RDG_CUDA(cudaStreamSynchronize(c.stream));
    if (hb) h.tail_level = -1;
  }
  return h.tail_level;
}

void coarse_tail(Ctx& c, Hierarchy& h, int c0, const double* r, double* z) {
  TailParams p{};
  const int nl = (int)h.levels.size();
  p.nlev = nl - 1 - c0;
  for (int k = 0; k < p.nlev; ++k) {
    const Level& lv = h.levels[c0 + k];
    TailLev& t = p.lv[k];
    t.n = lv.A.rows;
    t.L = lv.A.lat.lx;
    t.table = lv.tail_table.p;
    t.prp = lv.P.rp.p;
    t.pci = lv.P.ci.p;
    t.pv = lv.P.v.p;
    t.trp = lv.Pt.rp.p;
    t.tci = lv.Pt.ci.p;
    t.tv = lv.Pt.v.p;
  }
  p.nc = h.nc;
  p.Lc = h.Lc.p;
  p.r = r;
  p.z = z;
  p.err = c.d_err;
  p.m = h.smoothing_steps;
#if RD_PROBES  // compile-time diagnostic builds only: phase clocks of the tail kernel
  DBuf<long long> clk(64, c.stream);
  RDG_CUDA(cudaMemsetAsync(clk.p, 0, 64 * sizeof(long long), c.stream));
  p.clk = clk.p;
#else
  p.clk = nullptr;
#endif

  launch_pdl(coarse_tail_kernel, 1, kTailNT, tail_smem(h, c0), c.stream, p);
  RDG_LAUNCH_CHECK();
  ++c.launches;
#if RD_PROBES
  {
    long long hc[64];
    RDG_CUDA(cudaMemcpyAsync(hc, clk.p, sizeof(hc), cudaMemcpyDeviceToHost, c.stream));
    RDG_CUDA(cudaStreamSynchronize(c.stream));
    fprintf(stderr, "tail clocks:");
    for (int k = 1; k < 64 && hc[k]; ++k) fprintf(stderr, " %lld", hc[k] - hc[k - 1]);
    fprintf(stderr, "\n");
  }
#endif
}

}  // namespace rdg
