// linalg.cu -- CSR SpMV family, deterministic dots, scan, transpose, ordered
// SpGEMM and pruning on sm_100a.
//
// Bit-exactness contract: every fp64 row sum is evaluated
// sequentially in column order starting from 0.0 (linalg.cpp:26-31), and the
// whole library is compiled with --fmad=false so a*b+c never contracts.
#include <algorithm>
#include <cmath>

#include <cstdlib>

#include "internal.hpp"

namespace rdg {

// ============================================================== scan
namespace {
constexpr int kScanNT = 256;
constexpr int kScanPer = 8;
constexpr int kScanTile = kScanNT * kScanPer;

__device__ __forceinline__ long long block_incl_scan_ll(long long v, long long* sh) {
  // inclusive scan across the block (warp shuffles + one smem pass)
  const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long t = __shfl_up_sync(0xffffffffu, v, o);
    if (l >= o) v += t;
  }
  if (l == 31) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    long long s = l < (int)(blockDim.x >> 5) ? sh[l] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long t = __shfl_up_sync(0xffffffffu, s, o);
      if (l >= o) s += t;
    }
    sh[l] = s;
  }
  __syncthreads();
  if (w > 0) v += sh[w - 1];
  __syncthreads();
  return v;
}

__global__ void scan_tile_sums(const int* __restrict__ in, int64_t n, long long* __restrict__ bsum) {
  __shared__ long long sh[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  long long s = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int64_t i = base + (int64_t)k * kScanNT + threadIdx.x;
    if (i < n) s += in[i];
  }
  // block sum
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < kScanNT / 32; ++w) t += sh[w];
    bsum[blockIdx.x] = t;
  }
}

__global__ void scan_block_offsets(long long* __restrict__ bsum, int nb, long long* __restrict__ total,
                                   int* __restrict__ out_last) {
  // single block: exclusive scan of nb block sums in place
  __shared__ long long sh[32];
  long long carry = 0;
  for (int base = 0; base < nb; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const long long v = i < nb ? bsum[i] : 0;
    const long long inc = block_incl_scan_ll(v, sh);
    if (i < nb) bsum[i] = carry + inc - v;
    carry += sh[(blockDim.x >> 5) - 1];  // block total left by the scan
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *total = carry;
    *out_last = carry > 0x7fffffffLL ? 0x7fffffff : (int)carry;  // offsets[n]
  }
}

__global__ void scan_tiles(const int* __restrict__ in, int64_t n, const long long* __restrict__ boff,
                           int* __restrict__ out) {
  __shared__ long long sh[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPer;
  long long loc[kScanPer];
  long long s = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int64_t i = base + k;
    loc[k] = i < n ? in[i] : 0;
    s += loc[k];
  }
  const long long inc = block_incl_scan_ll(s, sh);
  long long run = boff[blockIdx.x] + inc - s;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int64_t i = base + k;
    if (i < n) out[i] = (int)run;
    run += loc[k];
  }
}
}  // namespace

int64_t exclusive_scan(Ctx& c, const int* counts, int* offsets, int64_t n, const int* also_dev, int* also_host) {
  if (n <= 0) {
    RDG_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int), c.stream));
    if (also_dev) {
      RDG_CUDA(cudaMemcpyAsync(also_host, also_dev, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
      RDG_CUDA(cudaStreamSynchronize(c.stream));
    }
    return 0;
  }
  const int nb = div_up(n, kScanTile);
  DBuf<long long> bsum(nb + 1, c.stream);
  scan_tile_sums<<<nb, kScanNT, 0, c.stream>>>(counts, n, bsum.p);
  RDG_LAUNCH_CHECK();
  scan_block_offsets<<<1, 1024, 0, c.stream>>>(bsum.p, nb, bsum.p + nb, offsets + n);
  RDG_LAUNCH_CHECK();
  scan_tiles<<<nb, kScanNT, 0, c.stream>>>(counts, n, bsum.p, offsets);
  RDG_LAUNCH_CHECK();
  c.launches += 3;
  long long* hp = reinterpret_cast<long long*>(c.h_pinned + 8);  // pinned: a true async readback
  RDG_CUDA(cudaMemcpyAsync(hp, bsum.p + nb, sizeof(long long), cudaMemcpyDeviceToHost, c.stream));
  int* ha = reinterpret_cast<int*>(c.h_pinned + 9);
  if (also_dev) RDG_CUDA(cudaMemcpyAsync(ha, also_dev, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  RDG_CUDA(cudaStreamSynchronize(c.stream));
  if (also_dev) *also_host = *ha;
  const long long total = *hp;
  if (total > 0x7fffffffLL) throw Error(RD_EINVAL, "index overflow: more than INT32_MAX entries (SpMat<int>)");
  return total;
}

// ============================================================== SpMV (warp-staged CSR)
// One warp owns 32 consecutive rows.  Their contiguous value/column block is
// staged into shared memory with coalesced 128-bit loads (double2 / int4),
// then every lane sums its own row sequentially in column order -- the exact
// reference order, with a fully coalesced HBM stream.
namespace {
constexpr int kSpmvWarps = 8;
constexpr int kSpmvNT = kSpmvWarps * 32;
#ifndef RD_SPMV_CAP
#define RD_SPMV_CAP 256  // measured at C2: 256 + batch 8 -> A 79 us, Pt 12 us, P 18 us (512, no batch: 90, 14, 23)
#endif
#ifndef RD_SPMV_BATCH
#define RD_SPMV_BATCH 8
#endif
constexpr int kSpmvCap = RD_SPMV_CAP;  // staged nnz per warp per chunk

enum SpmvMode { kPlain = 0, kDot = 1, kResidual = 2 };

struct SpmvSmem {
  double v[kSpmvWarps][kSpmvCap + 2];
  int ci[kSpmvWarps][kSpmvCap + 4];
  double red[kSpmvWarps];
};

template <int MODE>
__global__ void __launch_bounds__(kSpmvNT) spmv_staged_kernel(int rows, const int* __restrict__ rp,
                                                              const int* __restrict__ ci,
                                                              const double* __restrict__ val,
                                                              const double* __restrict__ x,
                                                              double* __restrict__ y,
                                                              const double* __restrict__ r,
                                                              double* partials, unsigned* counter,
                                                              double* dot_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SpmvSmem& sm = *reinterpret_cast<SpmvSmem*>(smem_raw);
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = (blockIdx.x * kSpmvWarps + warp) * 32;
  double contrib = 0.0;
  if (r0 < rows) {
    const int nr = min(32, rows - r0);
    const int s0 = __ldg(rp + r0), s1 = __ldg(rp + r0 + nr);
    const int row = r0 + lane;
    const int rs = lane < nr ? __ldg(rp + row) : 0;
    const int re = lane < nr ? __ldg(rp + row + 1) : 0;
    double sum = 0.0;
    for (int cb = s0; cb < s1; cb += kSpmvCap) {
      const int ce = min(s1, cb + kSpmvCap);
      // 128-bit staged loads from 16-byte aligned bases
      const int va = cb & ~1, ia = cb & ~3;
      const int nv2 = (ce - va + 1) >> 1, ni4 = (ce - ia + 3) >> 2;
      const double2* gv = reinterpret_cast<const double2*>(val + va);
      const int4* gi = reinterpret_cast<const int4*>(ci + ia);
      double2* sv = reinterpret_cast<double2*>(sm.v[warp]);
      int4* si = reinterpret_cast<int4*>(sm.ci[warp]);
      // every 16-byte piece of the block in flight at once (cp.async), then one wait:
      // a load -> shared store per iteration would serialise the DRAM round trips
      for (int t = lane; t < nv2; t += 32)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(sv + t)),
                     "l"(gv + t)
                     : "memory");
      for (int t = lane; t < ni4; t += 32)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(si + t)),
                     "l"(gi + t)
                     : "memory");
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncwarp();
      const int kb = max(rs, cb), ke = min(re, ce);
#if RD_SPMV_BATCH
      // the row's x gathers issued RD_SPMV_BATCH at a time, then summed in column order
      for (int k0 = kb; k0 < ke; k0 += RD_SPMV_BATCH) {
        double xv[RD_SPMV_BATCH];
#pragma unroll
        for (int u = 0; u < RD_SPMV_BATCH; ++u) xv[u] = k0 + u < ke ? __ldg(x + sm.ci[warp][k0 + u - ia]) : 0.0;
#pragma unroll
        for (int u = 0; u < RD_SPMV_BATCH; ++u)
          if (k0 + u < ke) sum = __dadd_rn(sum, __dmul_rn(sm.v[warp][k0 + u - va], xv[u]));
      }
#else
      for (int k = kb; k < ke; ++k) sum = __dadd_rn(sum, __dmul_rn(sm.v[warp][k - va], __ldg(x + sm.ci[warp][k - ia])));
#endif
      __syncwarp();
    }
    if (lane < nr) {
      if (MODE == kResidual) {
        y[row] = __dsub_rn(r[row], sum);
      } else {
        y[row] = sum;
        if (MODE == kDot) contrib = __dmul_rn(x[row], sum);
      }
    }
  }
  if (MODE == kDot) {
    const double bs = block_sum_fixed<kSpmvNT>(contrib, sm.red);
    if (threadIdx.x == 0) partials[blockIdx.x] = bs;
    finish_reduction<kSpmvNT>(partials, counter, sm.red, [&](double t) { *dot_out = t; });
  }
}

// SpMV on a lattice level whose rows are known on chip (smoother_lattice.cu's checks):
// uniform (tab = the 15-slot row) or class-uniform (tab = 64 class rows).  2.5-D blocked: a
// block owns a 32 (x) x 16 (y) column of rows, two rows per thread, and marches up 4-16 planes
// in z.  The x values of each plane (with a one-line halo in x and y, zero outside the box)
// arrive by cp.async in a kStNR-plane shared-memory ring, kStD planes ahead of the plane being
// summed (the residual's r rides in the same copy groups), so several planes per block are in
// flight.  A row reads 7 of its 15 neighbours from shared memory per plane: the plane-(z+1)
// values it read as "above" are its "centre" values at z+1, and its centre-plane values are
// its "below" values at z+1, carried in registers.  Each x value is read from L2 / HBM about
// 1.3 times.  A row sums its 15 slots from +0 in ascending column order; absent slots read
// x = +0 (finite coefficient * +0 = +-0, and a running sum from +0 never becomes -0), so the
// result is the CSR row sum bit for bit.  kDot adds p . (A p) with a fixed-order block
// reduction (deterministic, independent of block completion order).
constexpr int kStTX = 32, kStTY = 16, kStNR = 8, kStD = 5;
constexpr int kStNT = 256, kStRows = kStTX * kStTY / kStNT;  // 2 rows per thread (y and y + 8)
constexpr int kStPX = kStTX + 2, kStPY = kStTY + 2, kStPlane = kStPX * kStPY;
constexpr int kStE = (kStPlane + kStNT - 1) / kStNT;  // staging elements per thread
static_assert(kStNR >= kStD + 3, "a ring slot is refilled only after every thread left the planes it held");
static_assert(kStRows == 2, "two rows per thread");
static_assert((kStNR & (kStNR - 1)) == 0, "ring index by mask");

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

template <int MODE, bool CLS>
__global__ void __launch_bounds__(kStNT) stencil_spmv_tiled_kernel(int L, int gx, int gy, int zc, const double* __restrict__ tab,
                                                                  const double* __restrict__ x,
                                                                  double* __restrict__ y,
                                                                  const double* __restrict__ r, double* partials,
                                                                  unsigned* counter, double* dot_out) {
  __shared__ __align__(16) double st[CLS ? 64 * 16 : 16];
  // dynamic: the x ring [kStNR][kStPlane], then (residual) the r ring [kStNR][kStRows * kStNT]
  extern __shared__ __align__(16) double st_dyn[];
  double(*pl)[kStPlane] = reinterpret_cast<double(*)[kStPlane]>(st_dyn);
  double(*rr)[kStRows * kStNT] = reinterpret_cast<double(*)[kStRows * kStNT]>(st_dyn + kStNR * kStPlane);
  __shared__ double red[kStNT / 32];
  const int tid = threadIdx.x, tx = tid % kStTX, ty = tid / kStTX;
  pdl_wait();
  pdl_trigger();
  for (int k = tid; k < (CLS ? 64 * 16 : 16); k += kStNT) st[k] = __ldg(tab + k);
  const int b = blockIdx.x;
  const int a0 = (b % gx) * kStTX, y0 = ((b / gx) % gy) * kStTY, z0 = (b / (gx * gy)) * zc;
  const int z1 = min(z0 + zc, L);
  const long long P = (long long)L * L;
  const int a = a0 + tx;
  int yy[kStRows];
  bool valid[kStRows];
#pragma unroll
  for (int j = 0; j < kStRows; ++j) {
    yy[j] = y0 + ty + 8 * j;
    valid[j] = a < L && yy[j] < L;
  }
  // this thread's staging elements of a plane: in-plane offset, inside the box or not.  Outside
  // elements are zero in every ring slot (written once here, never copied); planes outside the
  // box are zeroed by stores instead of copied.
  int off[kStE];
  bool inb[kStE];
#pragma unroll
  for (int k = 0; k < kStE; ++k) {
    const int e = tid + k * kStNT;
    const int aa = a0 - 1 + e % kStPX, ye = y0 - 1 + e / kStPX;
    inb[k] = e < kStPlane && aa >= 0 && aa < L && ye >= 0 && ye < L;
    off[k] = inb[k] ? ye * L + aa : 0;
    if (e < kStPlane && !inb[k])
      for (int q = 0; q < kStNR; ++q) pl[q][e] = 0.0;
  }
  const int roff[kStRows] = {valid[0] ? yy[0] * L + a : 0, valid[1] ? yy[1] * L + a : 0};
  // copy group of plane q (planes past z1 commit an empty group: the wait count stays uniform)
  auto issue = [&](int q) {
    if (q <= z1) {
      double* dst = pl[(q + kStNR) & (kStNR - 1)];
      if (q >= 0 && q < L) {
        const double* base = x + (long long)q * P;
#pragma unroll
        for (int k = 0; k < kStE; ++k)
          if (inb[k]) cp_async8(dst + tid + k * kStNT, base + off[k]);
      } else {
#pragma unroll
        for (int k = 0; k < kStE; ++k)
          if (inb[k]) dst[tid + k * kStNT] = 0.0;
      }
      if (MODE == kResidual && q >= z0 && q < z1) {
        const double* rb = r + (long long)q * P;
#pragma unroll
        for (int j = 0; j < kStRows; ++j)
          if (valid[j]) cp_async8(&rr[q & (kStNR - 1)][tid + j * kStNT], rb + roff[j]);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int q = 0; q < kStD; ++q) issue(z0 - 1 + q);
  int cay[kStRows];
#pragma unroll
  for (int j = 0; j < kStRows; ++j)
    cay[j] = CLS ? (pos_class(a < L ? a : 0, L) * 16 + pos_class(yy[j] < L ? yy[j] : 0, L) * 4) : 0;
  double U[CLS ? 1 : 15];
  __syncthreads();  // st
  if (!CLS) {
#pragma unroll
    for (int k = 0; k < 15; ++k) U[k] = st[k];
  }
  double cm[kStRows][4], cp[kStRows][4];  // carried: below (-1-1, 0-1, -10, 00), centre (00, 10, 01, 11)
  double contrib = 0.0;
#pragma unroll 2
  for (int z = z0; z < z1; ++z) {
    issue(z + kStD - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(kStD - 2) : "memory");  // planes <= z + 1 landed
    __syncthreads();
    const double* p0 = pl[z & (kStNR - 1)];
    const double* pp = pl[(z + 1) & (kStNR - 1)];
    if (z == z0) {  // prime the carried values from planes z0 - 1 and z0
      const double* pm = pl[(z - 1 + kStNR) & (kStNR - 1)];
#pragma unroll
      for (int j = 0; j < kStRows; ++j) {
        const int c = (ty + 8 * j + 1) * kStPX + tx + 1;
        cm[j][0] = pm[c - kStPX - 1];
        cm[j][1] = pm[c - kStPX];
        cm[j][2] = pm[c - 1];
        cm[j][3] = pm[c];
        cp[j][0] = p0[c];
        cp[j][1] = p0[c + 1];
        cp[j][2] = p0[c + kStPX];
        cp[j][3] = p0[c + kStPX + 1];
      }
    }
#pragma unroll
    for (int j = 0; j < kStRows; ++j) {
      const int c = (ty + 8 * j + 1) * kStPX + tx + 1;
      const double* v = CLS ? st + (cay[j] + pos_class(z, L)) * 16 : U;
      const double xs[15] = {cm[j][0], cm[j][1], cm[j][2], cm[j][3],
                             p0[c - kStPX - 1], p0[c - kStPX], p0[c - 1], cp[j][0], cp[j][1], cp[j][2], cp[j][3],
                             pp[c], pp[c + 1], pp[c + kStPX], pp[c + kStPX + 1]};
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 15; ++k) acc = __dadd_rn(acc, __dmul_rn(v[k], xs[k]));
      if (valid[j]) {
        const long long i = z * P + (long long)yy[j] * L + a;
        if (MODE == kResidual) {
          y[i] = __dsub_rn(rr[z & (kStNR - 1)][tid + j * kStNT], acc);
        } else {
          y[i] = acc;
          if (MODE == kDot) contrib = __dadd_rn(contrib, __dmul_rn(xs[7], acc));
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        cm[j][k] = xs[4 + (k < 3 ? k : 3)];
        cp[j][k] = xs[11 + k];
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (MODE == kDot) {
    const double bs = block_sum_fixed<kStNT>(contrib, red);
    if (tid == 0) partials[b] = bs;
    finish_reduction<kStNT>(partials, counter, red, [&](double t) { *dot_out = t; });
  }
}

template <int MODE>
void launch_spmv(Ctx& c, const DCsr& A, const double* x, double* y, const double* r, double* dot_out) {
  if (A.rows == 0) {
    if (MODE == kDot) RDG_CUDA(cudaMemsetAsync(dot_out, 0, sizeof(double), c.stream));
    return;
  }
  static const bool nostencil = getenv("RD_NO_STENCIL_SPMV") && atoi(getenv("RD_NO_STENCIL_SPMV")) != 0;
  if (!nostencil && A.lat.ok && (A.lat_uni_state == 1 || A.lat_uni_state == 2) && A.lat.lx == A.lat.ly &&
      A.lat.lx == A.lat.lz && (int64_t)A.lat.lx * A.lat.lx * A.lat.lx == A.rows && A.cols == A.rows) {
    const int L = A.lat.lx;
    const bool cls = A.lat_uni_state == 2;
    const int gx = div_up(L, kStTX), gy = div_up(L, kStTY);
    // planes per block: each block's planes are a dependent chain (one ring step each), so the
    // shortest chain that still fits the grid in the resident slots (2 blocks per SM) wins
    int zc = 4;
    while (zc < 16 && (int64_t)gx * gy * div_up(L, zc) > 2 * (int64_t)c.num_sms) zc *= 2;
    const int64_t nb = (int64_t)gx * gy * div_up(L, zc);
    // the fused dot needs one partial per block
    const bool fused = MODE != kDot || nb <= Ctx::kMaxPartials;
    constexpr int M2 = MODE == kDot ? kPlain : MODE;
    auto* k = fused ? (cls ? stencil_spmv_tiled_kernel<MODE, true> : stencil_spmv_tiled_kernel<MODE, false>)
                    : (cls ? stencil_spmv_tiled_kernel<M2, true> : stencil_spmv_tiled_kernel<M2, false>);
    const size_t smem = sizeof(double) * kStNR * (kStPlane + (MODE == kResidual ? kStRows * kStNT : 0));
    static bool attr = false;  // per MODE instantiation
    if (!attr) {
      for (auto* kk : {stencil_spmv_tiled_kernel<MODE, true>, stencil_spmv_tiled_kernel<MODE, false>,
                       stencil_spmv_tiled_kernel<M2, true>, stencil_spmv_tiled_kernel<M2, false>})
        RDG_CUDA(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = true;
    }
    launch_pdl(k, (unsigned)nb, kStNT, smem, c.stream, L, gx, gy, zc, cls ? A.lat_cls.p : A.lat_uni.p, x, y, r,
               c.d_partials, c.d_counter, dot_out);
    ++c.launches;
    if (!fused) dot(c, A.rows, x, y, dot_out);
    return;
  }
  const int nb = div_up(A.rows, kSpmvNT);
  static bool attr = false;
  const size_t smem = sizeof(SpmvSmem);
  if (!attr) {
    for (auto* k : {spmv_staged_kernel<kPlain>, spmv_staged_kernel<kDot>, spmv_staged_kernel<kResidual>})
      RDG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  if (MODE == kDot && nb > Ctx::kMaxPartials) {
    // too many blocks for one partials array: plain SpMV then a separate dot
    launch_pdl(spmv_staged_kernel<kPlain>, nb, kSpmvNT, smem, c.stream, A.rows, A.rp.p, A.ci.p, A.v.p, x, y, r, nullptr,
               nullptr, nullptr);
    ++c.launches;
    dot(c, A.rows, x, y, dot_out);
    return;
  }
  launch_pdl(spmv_staged_kernel<MODE>, nb, kSpmvNT, smem, c.stream, A.rows, A.rp.p, A.ci.p, A.v.p, x, y, r, c.d_partials,
             c.d_counter, dot_out);
  ++c.launches;
}

// z += P zc, P with a handful of entries per row: thread per row, sequential sum
__global__ void prolong_add_kernel(int rows, const int* __restrict__ rp, const int* __restrict__ ci,
                                   const double* __restrict__ val, const double* __restrict__ zc,
                                   double* __restrict__ z) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  double s = 0.0;
  for (int k = rp[i]; k < rp[i + 1]; ++k) s = __dadd_rn(s, __dmul_rn(val[k], zc[ci[k]]));
  z[i] = __dadd_rn(z[i], s);
}

constexpr int kDotNT = 256;

__global__ void __launch_bounds__(kDotNT) dot_kernel(int64_t n, const double* __restrict__ a,
                                                     const double* __restrict__ b, double* partials,
                                                     unsigned* counter, double* out) {
  __shared__ double sh[kDotNT / 32];
  pdl_wait();
  pdl_trigger();
  // fixed contiguous chunk per block, strided per thread -> deterministic
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t beg = (int64_t)blockIdx.x * per, end = min(n, beg + per);
  double s = 0.0;
  for (int64_t i = beg + threadIdx.x; i < end; i += kDotNT) s = __dadd_rn(s, __dmul_rn(a[i], b[i]));
  const double bs = block_sum_fixed<kDotNT>(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = bs;
  finish_reduction<kDotNT>(partials, counter, sh, [&](double t) { *out = t; });
}
}  // namespace

void spmv(Ctx& c, const DCsr& A, const double* x, double* y) { launch_spmv<kPlain>(c, A, x, y, nullptr, nullptr); }
void spmv_dot(Ctx& c, const DCsr& A, const double* x, double* y, double* dot_out) {
  launch_spmv<kDot>(c, A, x, y, nullptr, dot_out);
}
void residual(Ctx& c, const DCsr& A, const double* r, const double* z, double* res) {
  launch_spmv<kResidual>(c, A, z, res, r, nullptr);
}
void prolong_add(Ctx& c, const DCsr& P, const double* zc, double* z) {
  if (P.rows == 0) return;
  launch_pdl(prolong_add_kernel, div_up(P.rows, 256), 256, 0, c.stream, P.rows, P.rp.p, P.ci.p, P.v.p, zc, z);
  ++c.launches;
}

int dot_grid(int64_t n) {
  // deterministic function of n only
  return (int)std::max<int64_t>(1, std::min<int64_t>(1184, (n + 4095) / 4096));
}

void dot(Ctx& c, int64_t n, const double* a, const double* b, double* out_dev) {
  if (n <= 0) {
    RDG_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double), c.stream));
    return;
  }
  launch_pdl(dot_kernel, dot_grid(n), kDotNT, 0, c.stream, n, a, b, c.d_partials, c.d_counter + 1, out_dev);
  ++c.launches;
}

// ============================================================== Jacobi (linalg.cpp:57-62)
namespace {
// d_i = A(i,i) (0 when the row stores no diagonal, like Eigen's diagonal()); bad = 1 if some d_i <= 0
__global__ void csr_diag_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                const double* __restrict__ v, double* __restrict__ d, int* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double di = 0.0;
  for (int k = rp[i]; k < rp[i + 1]; ++k)
    if (ci[k] == i) {
      di = v[k];
      break;
    }
  d[i] = di;
  if (di <= 0.0) *bad = 1;
}
__global__ void jacobi_kernel(int64_t n, const double* __restrict__ d, const double* __restrict__ r,
                              double* __restrict__ z) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] = __ddiv_rn(r[i], d[i]);
}
}  // namespace

void csr_diagonal(Ctx& c, const DCsr& A, double* d, int* bad_dev) {
  if (A.rows == 0) return;
  csr_diag_kernel<<<div_up(A.rows, 256), 256, 0, c.stream>>>(A.rows, A.rp.p, A.ci.p, A.v.p, d, bad_dev);
  RDG_LAUNCH_CHECK();
  ++c.launches;
}
void jacobi_apply(Ctx& c, int64_t n, const double* d, const double* r, double* z) {
  if (n == 0) return;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c.num_sms * 8, (n + 255) / 256));
  jacobi_kernel<<<g, 256, 0, c.stream>>>(n, d, r, z);
  RDG_LAUNCH_CHECK();
  ++c.launches;
}

// ============================================================== structure ops
namespace {
__global__ void count_cols_kernel(int64_t nnz, const int* __restrict__ ci, int* cnt) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nnz) atomicAdd(cnt + ci[k], 1);
}

__global__ void transpose_fill_kernel(int rows, const int* __restrict__ rp, const int* __restrict__ ci,
                                      const double* __restrict__ v, int* cursor, int* tci, double* tv) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  for (int k = rp[r]; k < rp[r + 1]; ++k) {
    const int pos = atomicAdd(cursor + ci[k], 1);
    tci[pos] = r;
    tv[pos] = v[k];
  }
}

// insertion sort of each row by column (rows are short); carries values
__global__ void sort_rows_kernel(int rows, const int* __restrict__ rp, int* ci, double* v) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int b = rp[r], e = rp[r + 1];
  for (int k = b + 1; k < e; ++k) {
    const int key = ci[k];
    const double kv = v[k];
    int j = k - 1;
    while (j >= b && ci[j] > key) {
      ci[j + 1] = ci[j];
      v[j + 1] = v[j];
      --j;
    }
    ci[j + 1] = key;
    v[j + 1] = kv;
  }
}

__global__ void row_count_kernel(int rows, const int* __restrict__ rp, const double* __restrict__ v, int* cnt) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  int c = 0;
  for (int k = rp[r]; k < rp[r + 1]; ++k) c += v[k] != 0.0;
  cnt[r] = c;
}

__global__ void prune_copy_kernel(int rows, const int* __restrict__ rp, const int* __restrict__ ci,
                                  const double* __restrict__ v, const int* __restrict__ orp, int* oci,
                                  double* ov) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  int o = orp[r];
  for (int k = rp[r]; k < rp[r + 1]; ++k)
    if (v[k] != 0.0) {
      oci[o] = ci[k];
      ov[o] = v[k];
      ++o;
    }
}

// ---- ordered Gustavson SpGEMM (Eigen conservative_sparse_sparse_product order)
__global__ void spgemm_upper_kernel(int rows, const int* __restrict__ arp, const int* __restrict__ aci,
                                    const int* __restrict__ brp, int* ub) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= rows) return;
  int s = 0;
  for (int k = arp[j]; k < arp[j + 1]; ++k) {
    const int c = aci[k];
    s += brp[c + 1] - brp[c];
  }
  ub[j] = s;
}

// Row j: for A's entries (k, y) in order, for B's row-k entries (i, x) in order:
// first touch values[i] = x*y, later values[i] += x*y.  Scratch holds the
// first-touch list; it is then insertion-sorted by column.
__global__ void spgemm_numeric_kernel(int rows, const int* __restrict__ arp, const int* __restrict__ aci,
                                      const double* __restrict__ av, const int* __restrict__ brp,
                                      const int* __restrict__ bci, const double* __restrict__ bv,
                                      const int* __restrict__ uoff, int* scol, double* sval, int* cnt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= rows) return;
  int* cols = scol + uoff[j];
  double* vals = sval + uoff[j];
  int u = 0;
  for (int ka = arp[j]; ka < arp[j + 1]; ++ka) {
    const double y = av[ka];
    const int k = aci[ka];
    for (int kb = brp[k]; kb < brp[k + 1]; ++kb) {
      const int i = bci[kb];
      const double xv = bv[kb];
      int q = 0;
      while (q < u && cols[q] != i) ++q;
      if (q == u) {
        cols[u] = i;
        vals[u] = __dmul_rn(xv, y);
        ++u;
      } else {
        vals[q] = __dadd_rn(vals[q], __dmul_rn(xv, y));
      }
    }
  }
  for (int a = 1; a < u; ++a) {
    const int key = cols[a];
    const double kv = vals[a];
    int b = a - 1;
    while (b >= 0 && cols[b] > key) {
      cols[b + 1] = cols[b];
      vals[b + 1] = vals[b];
      --b;
    }
    cols[b + 1] = key;
    vals[b + 1] = kv;
  }
  cnt[j] = u;
}

__global__ void spgemm_copy_kernel(int rows, const int* __restrict__ uoff, const int* __restrict__ scol,
                                   const double* __restrict__ sval, const int* __restrict__ rp, int* ci,
                                   double* v) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= rows) return;
  const int s = uoff[j], o = rp[j], n = rp[j + 1] - o;
  for (int q = 0; q < n; ++q) {
    ci[o + q] = scol[s + q];
    v[o + q] = sval[s + q];
  }
}

__global__ void symmetric_check_kernel(int rows, const int* __restrict__ rp, const int* __restrict__ ci,
                                       int* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  for (int k = rp[i]; k < rp[i + 1]; ++k) {
    const int j = ci[k];
    // binary search i in row j
    int lo = rp[j], hi = rp[j + 1];
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (ci[mid] < i)
        lo = mid + 1;
      else
        hi = mid;
    }
    if (lo >= rp[j + 1] || ci[lo] != i) {
      atomicExch(bad, 1);
      return;
    }
  }
}

// Verifies the full in-box 15-point Kuhn stencil on an
// lx*ly*lz box in lexicographic order.
__global__ void lattice_check_kernel(int rows, const int* __restrict__ rp, const int* __restrict__ ci, int lx,
                                     int ly, int lz, int* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int a = i % lx, b = (i / lx) % ly, c = i / (lx * ly);
  // stencil offsets in ascending linear-offset order
  const int d[15][3] = {{-1, -1, -1}, {0, -1, -1}, {-1, 0, -1}, {0, 0, -1}, {-1, -1, 0},
                        {0, -1, 0},   {-1, 0, 0},  {0, 0, 0},   {1, 0, 0},  {0, 1, 0},
                        {1, 1, 0},    {0, 0, 1},   {1, 0, 1},   {0, 1, 1},  {1, 1, 1}};
  int k = rp[i];
  const int e = rp[i + 1];
  for (int s = 0; s < 15; ++s) {
    const int aa = a + d[s][0], bb = b + d[s][1], cc = c + d[s][2];
    if (aa < 0 || bb < 0 || cc < 0 || aa >= lx || bb >= ly || cc >= lz) continue;
    const int col = (cc * ly + bb) * lx + aa;
    if (k >= e || ci[k] != col) {
      atomicExch(bad, 1);
      return;
    }
    ++k;
  }
  if (k != e) atomicExch(bad, 1);
}
}  // namespace

DCsr csr_view(const DCsr& A) {
  DCsr B;
  B.rows = A.rows;
  B.cols = A.cols;
  B.nnz = A.nnz;
  B.lat = A.lat;
  B.lat_checked = A.lat_checked;
  B.rp = DBuf<int>::view(A.rp.p, A.rp.n);
  B.ci = DBuf<int>::view(A.ci.p, A.ci.n);
  B.v = DBuf<double>::view(A.v.p, A.v.n);
  return B;
}

DCsr csr_copy(Ctx& c, const DCsr& A) {
  DCsr B;
  B.rows = A.rows;
  B.cols = A.cols;
  B.nnz = A.nnz;
  B.lat = A.lat;
  B.lat_checked = A.lat_checked;
  B.rp.alloc(A.rows + 1, c.stream);
  B.ci.alloc(A.nnz, c.stream);
  B.v.alloc(A.nnz, c.stream);
  RDG_CUDA(cudaMemcpyAsync(B.rp.p, A.rp.p, sizeof(int) * (A.rows + 1), cudaMemcpyDeviceToDevice, c.stream));
  if (A.nnz) {
    RDG_CUDA(cudaMemcpyAsync(B.ci.p, A.ci.p, sizeof(int) * A.nnz, cudaMemcpyDeviceToDevice, c.stream));
    RDG_CUDA(cudaMemcpyAsync(B.v.p, A.v.p, sizeof(double) * A.nnz, cudaMemcpyDeviceToDevice, c.stream));
  }
  return B;
}

// SpMat(P.transpose()) (amg.cpp:104): rows of the result list the source rows ascending.
DCsr transpose(Ctx& c, const DCsr& A) {
  DCsr T;
  T.rows = A.cols;
  T.cols = A.rows;
  T.nnz = A.nnz;
  T.rp.alloc(T.rows + 1, c.stream);
  T.ci.alloc(A.nnz, c.stream);
  T.v.alloc(A.nnz, c.stream);
  DBuf<int> cnt(T.rows + 1, c.stream);
  RDG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (T.rows + 1), c.stream));
  if (A.nnz) {
    count_cols_kernel<<<div_up(A.nnz, 256), 256, 0, c.stream>>>(A.nnz, A.ci.p, cnt.p);
    RDG_LAUNCH_CHECK();
    ++c.launches;
  }
  exclusive_scan(c, cnt.p, T.rp.p, T.rows);
  if (A.nnz) {
    RDG_CUDA(cudaMemcpyAsync(cnt.p, T.rp.p, sizeof(int) * T.rows, cudaMemcpyDeviceToDevice, c.stream));
    transpose_fill_kernel<<<div_up(A.rows, 256), 256, 0, c.stream>>>(A.rows, A.rp.p, A.ci.p, A.v.p, cnt.p, T.ci.p,
                                                                     T.v.p);
    RDG_LAUNCH_CHECK();
    sort_rows_kernel<<<div_up(T.rows, 256), 256, 0, c.stream>>>(T.rows, T.rp.p, T.ci.p, T.v.p);
    RDG_LAUNCH_CHECK();
    c.launches += 2;
  }
  return T;
}

DCsr prune_zeros(Ctx& c, const DCsr& A) {
  DCsr B;
  B.rows = A.rows;
  B.cols = A.cols;
  B.rp.alloc(A.rows + 1, c.stream);
  DBuf<int> cnt(std::max(A.rows, 1), c.stream);
  if (A.rows) {
    row_count_kernel<<<div_up(A.rows, 256), 256, 0, c.stream>>>(A.rows, A.rp.p, A.v.p, cnt.p);
    RDG_LAUNCH_CHECK();
    ++c.launches;
  }
  B.nnz = exclusive_scan(c, cnt.p, B.rp.p, A.rows);
  B.ci.alloc(B.nnz, c.stream);
  B.v.alloc(B.nnz, c.stream);
  if (A.rows) {
    prune_copy_kernel<<<div_up(A.rows, 256), 256, 0, c.stream>>>(A.rows, A.rp.p, A.ci.p, A.v.p, B.rp.p, B.ci.p,
                                                                 B.v.p);
    RDG_LAUNCH_CHECK();
    ++c.launches;
  }
  return B;
}

DCsr spgemm(Ctx& c, const DCsr& A, const DCsr& B) {
  if (A.cols != B.rows) throw Error(RD_EINVAL, "galerkin_coarse: dims");
  DCsr C;
  C.rows = A.rows;
  C.cols = B.cols;
  C.rp.alloc(A.rows + 1, c.stream);
  if (A.rows == 0) {
    RDG_CUDA(cudaMemsetAsync(C.rp.p, 0, sizeof(int), c.stream));
    return C;
  }
  const int nb = div_up(A.rows, 128);
  DBuf<int> ub(A.rows + 1, c.stream), uoff(A.rows + 1, c.stream), cnt(A.rows + 1, c.stream);
  spgemm_upper_kernel<<<nb, 128, 0, c.stream>>>(A.rows, A.rp.p, A.ci.p, B.rp.p, ub.p);
  RDG_LAUNCH_CHECK();
  const int64_t total = exclusive_scan(c, ub.p, uoff.p, A.rows);
  DBuf<int> scol(std::max<int64_t>(total, 1), c.stream);
  DBuf<double> sval(std::max<int64_t>(total, 1), c.stream);
  spgemm_numeric_kernel<<<nb, 128, 0, c.stream>>>(A.rows, A.rp.p, A.ci.p, A.v.p, B.rp.p, B.ci.p, B.v.p, uoff.p,
                                                  scol.p, sval.p, cnt.p);
  RDG_LAUNCH_CHECK();
  C.nnz = exclusive_scan(c, cnt.p, C.rp.p, A.rows);
  C.ci.alloc(C.nnz, c.stream);
  C.v.alloc(C.nnz, c.stream);
  spgemm_copy_kernel<<<nb, 128, 0, c.stream>>>(A.rows, uoff.p, scol.p, sval.p, C.rp.p, C.ci.p, C.v.p);
  RDG_LAUNCH_CHECK();
  c.launches += 3;
  return C;
}

bool pattern_symmetric(Ctx& c, const DCsr& A) {
  if (A.rows != A.cols) return false;
  if (A.rows == 0) return true;
  DBuf<int> bad(1, c.stream);
  RDG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c.stream));
  symmetric_check_kernel<<<div_up(A.rows, 256), 256, 0, c.stream>>>(A.rows, A.rp.p, A.ci.p, bad.p);
  RDG_LAUNCH_CHECK();
  ++c.launches;
  int h = 0;
  RDG_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  RDG_CUDA(cudaStreamSynchronize(c.stream));
  return h == 0;
}

void detect_lattice(Ctx& c, DCsr& A) {
  if (A.lat_checked) return;
  A.lat_checked = true;
  A.lat = Lattice{};
  if (A.rows != A.cols || A.rows < 8) return;
  int L = (int)std::llround(std::cbrt((double)A.rows));
  if ((int64_t)L * L * L != A.rows) return;
  DBuf<int> bad(1, c.stream);
  RDG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c.stream));
  lattice_check_kernel<<<div_up(A.rows, 256), 256, 0, c.stream>>>(A.rows, A.rp.p, A.ci.p, L, L, L, bad.p);
  RDG_LAUNCH_CHECK();
  ++c.launches;
  int h = 0;
  RDG_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  RDG_CUDA(cudaStreamSynchronize(c.stream));
  if (h == 0) A.lat = Lattice{L, L, L, true};
}

}  // namespace rdg
