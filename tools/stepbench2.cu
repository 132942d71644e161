// Microbenchmark of the lattice-GS compute-warp protocol in one CTA (no aux warps):
// 4 warps of 8 (y) x 4 (z) lines in a 2 x 2 arrangement, sentinel rings in shared
// memory exactly as gs_lattice5_kernel (publish, clear ahead, poll until all three
// fresh neighbours are present), the row chain + speculative division, and optional
// features (FEAT bits): 1 stencil values from global (8 LDG.128, 3 steps ahead),
// 2 x stores to global, 4 progress + backpressure every 4 steps, 8 cross-warp
// neighbours (off: every lane reads only its own warp's ring), 16 box reads from
// shared memory, 32 one warp only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o tools/stepbench2 tools/stepbench2.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int R5 = 16;
constexpr unsigned long long kSent = 0x7ff4deadbeef0badull;
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long lds_u64(unsigned a) {
  unsigned long long v;
  asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u64(unsigned a, unsigned long long v) {
  asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ double lds_f64(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
template <int KIND>
__device__ __forceinline__ double2 ldg_k(const double2* q) {
  double2 r;
  if (KIND == 0)
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(q));
  else if (KIND == 1)
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(q));
  else if (KIND == 2)
    asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(q));
  else
    r = __ldg(q);  // plain (compiler-scheduled, no volatile)
  return r;
}

template <int FEAT>
__global__ void __launch_bounds__(128, 1) k2(const double2* __restrict__ vals, double* xout, long long* cyc, int steps) {
  __shared__ __align__(16) unsigned long long rings[6][R5][32];
  __shared__ double box[64][40];
  __shared__ int s_prog[4];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  if ((FEAT & 32) && w > 0) return;
  for (int k = tid; k < 6 * R5 * 32; k += blockDim.x) {
    const int r = k / (R5 * 32), sl = k / 32 % R5;
    (&rings[0][0][0])[k] = (r == 5 || (r < 4 && sl == R5 - 2)) ? 0ull : kSent;
  }
  for (int k = tid; k < 64 * 40; k += blockDim.x) (&box[0][0])[k] = 0.001 * (k & 15);
  if (tid < 4) s_prog[tid] = -1;
  __syncthreads();
  const int wy = w & 1, wz = w >> 1, tyw = lane & 7, tzw = lane >> 3;
  const int ty = wy * 8 + tyw, tz = wz * 4 + tzw;
  const unsigned ring0 = smem_addr(&rings[0][0][0]);
  auto ring_lane = [&](int r, int idx) { return ring0 + (unsigned)r * (R5 * 256) + (unsigned)idx * 8u; };
  auto src_of = [&](int ty2, int tz2) -> unsigned {
    if (ty2 < 0 || tz2 < 0) return ring_lane(5, 0);
    if (!(FEAT & 8) && ((ty2 >> 3) != wy || (tz2 >> 2) != wz)) return ring_lane(5, 0);
    return ring_lane((tz2 >> 2) * 2 + (ty2 >> 3), (tz2 & 3) * 8 + (ty2 & 7));
  };
  const unsigned sY = src_of(ty - 1, tz), sZ = src_of(ty, tz - 1), sD = src_of(ty - 1, tz - 1);
  const unsigned myring = ring_lane(w, lane);
  const unsigned bF = smem_addr(&box[0][lane]);
  double* xo = xout + (size_t)(w * 32 + lane) * 8192;
  const double2* vptr = vals + (size_t)w * 32 * 8 + lane;
  auto load_block = [&](int b, double (&v)[16]) {
    const double2* q = vptr + (size_t)(b & 63) * 4 * 32 * 8;
    if (FEAT & 256) {  // 4 x 256-bit loads (layout: quad k of lane l at (k * 32 + l) * 32 B)
      const double* q4 = reinterpret_cast<const double*>(vals) + (size_t)(b & 63) * 4 * 32 * 16 + (size_t)w * 32 * 16 + lane * 4;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(v[4 * k]), "=d"(v[4 * k + 1]), "=d"(v[4 * k + 2]), "=d"(v[4 * k + 3])
                     : "l"(q4 + k * 128));
      return;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double2 t = ldg_k<(FEAT >> 9) & 3>(q + k * 32);
      v[2 * k] = t.x;
      v[2 * k + 1] = t.y;
    }
  };
  double vbA[16], vbB[16], vbC[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) vbA[k] = vbB[k] = vbC[k] = (k == 7 || k == 15) ? 1.0 : 0.0625;
  if (FEAT & 1) {
    load_block(0, vbB);
    load_block(1, vbC);
  }
  double x1 = 0.0, Y1 = 0.0, Z1 = 0.0, D1 = 0.0, D2 = 0.0, acc = 0.0;
  auto min_prog = [&]() {
    int c = *reinterpret_cast<volatile int*>(&s_prog[0]);
    for (int q = 1; q < 4; ++q) c = min(c, *reinterpret_cast<volatile int*>(&s_prog[q]));
    return c;
  };
  auto step = [&](int s, double (&v)[16]) {
    const unsigned q0 = (unsigned)(s & 63) * 320u, q1 = (unsigned)((s + 1) & 63) * 320u;
    double fa = 1.0, Ox = 0.5, Oy = 0.5, Oz = 0.5, Oxy = 0.5, Oxz = 0.5, Oyz = 0.5, Oxyz = 0.5;
    if (FEAT & 16) {
      fa = lds_f64(bF + q0);
      Ox = lds_f64(bF + q1);
      Oxy = lds_f64(bF + q1 + 8);
      Oxz = lds_f64(bF + q1 + 64);
      Oxyz = lds_f64(bF + q1 + 72);
      Oy = lds_f64(bF + q0 + 8);
      Oz = lds_f64(bF + q0 + 64);
      Oyz = lds_f64(bF + q0 + 72);
    }
    const unsigned sn = (unsigned)(s & (R5 - 1)) * 256u;
    sts_u64(myring + ((sn + (R5 / 2) * 256u) & (R5 * 256u - 1)), kSent);
    double sum = fa;
    sum = __dsub_rn(sum, __dmul_rn(v[0], D2));
    sum = __dsub_rn(sum, __dmul_rn(v[1], D1));
    sum = __dsub_rn(sum, __dmul_rn(v[2], Z1));
    const unsigned so = (unsigned)((s - 1) & (R5 - 1)) * 256u;
    unsigned long long uY = lds_u64(sY + so), uZ = lds_u64(sZ + so), uD = lds_u64(sD + so);
    if (!__all_sync(0xffffffffu, uY != kSent && uZ != kSent && uD != kSent)) {
      int spin = 0;
      do {
        if (++spin > (1 << 22)) break;  // never hang the GPU: timing of a broken run is discarded
        if (uY == kSent) uY = lds_u64(sY + so);
        if (uZ == kSent) uZ = lds_u64(sZ + so);
        if (uD == kSent) uD = lds_u64(sD + so);
      } while (!__all_sync(0xffffffffu, uY != kSent && uZ != kSent && uD != kSent));
    }
    const double Y0 = __longlong_as_double((long long)uY), Z0 = __longlong_as_double((long long)uZ);
    const double D0 = __longlong_as_double((long long)uD);
    sum = __dsub_rn(sum, __dmul_rn(v[3], Z0));
    sum = __dsub_rn(sum, __dmul_rn(v[4], Y1));
    sum = __dsub_rn(sum, __dmul_rn(v[5], Y0));
    sum = __dsub_rn(sum, __dmul_rn(v[6], x1));
    sum = __dsub_rn(sum, __dmul_rn(v[8], Ox));
    sum = __dsub_rn(sum, __dmul_rn(v[9], Oy));
    sum = __dsub_rn(sum, __dmul_rn(v[10], Oxy));
    sum = __dsub_rn(sum, __dmul_rn(v[11], Oz));
    sum = __dsub_rn(sum, __dmul_rn(v[12], Oxz));
    sum = __dsub_rn(sum, __dmul_rn(v[13], Oyz));
    sum = __dsub_rn(sum, __dmul_rn(v[14], Oxyz));
    const double qq = __dmul_rn(sum, v[15]);
    double xv = __fma_rn(-v[15], __fma_rn(v[7], qq, -sum), qq);
    xv = xv * 0.5;  // keep the values bounded
    sts_u64(myring + sn, (unsigned long long)__double_as_longlong(xv));
    if (FEAT & 2) xo[s & 8191] = xv;
    if ((FEAT & 64) && ((lane ^ s) & 1) == 0)  // pairs: half the lanes store 16 B per step
      asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(xo + (s & 8190)), "d"(x1), "d"(xv) : "memory");
    if ((FEAT & 128) && ((lane ^ s) & 3) == 0)  // quads: a quarter of the lanes store 32 B per step
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(xo + (s & 8188)), "d"(Y1), "d"(Z1), "d"(x1),
                   "d"(xv)
                   : "memory");
    acc += xv;
    x1 = xv;
    Y1 = Y0;
    Z1 = Z0;
    D2 = D1;
    D1 = D0;
    if (FEAT & 1) load_block(s + 3, v);
    if ((FEAT & 4) && lane == 0) *reinterpret_cast<volatile int*>(&s_prog[w]) = s + 1;
  };
  auto group_start = [&](int s) {
    if (!(FEAT & 4) || ((s + 1) & 3) != 0 || (FEAT & 32)) return;
    const int need = s + 4 - (R5 / 2 - 2);
    int spin = 0;
    while (min_prog() < need && ++spin < (1 << 22)) {
    }
  };
  const long long t0 = clock64();
#pragma unroll 1
  for (int s = -1; s < steps; s += 3) {
    group_start(s);
    step(s, vbA);
    group_start(s + 1);
    step(s + 1, vbB);
    group_start(s + 2);
    step(s + 2, vbC);
  }
  const long long t1 = clock64();
  if (lane == 0) cyc[w] = t1 - t0;
  xout[(size_t)128 * 8192 + tid] = acc;
}

int main() {
  double2* vals;
  double* xout;
  long long* cyc;
  cudaMalloc(&vals, (size_t)64 * 4 * 32 * 8 * sizeof(double2) + 4096);
  cudaMemset(vals, 0, (size_t)64 * 4 * 32 * 8 * sizeof(double2));
  cudaMalloc(&xout, (size_t)(128 * 8192 + 256) * sizeof(double));
  cudaMallocManaged(&cyc, 4 * sizeof(long long));
  const int steps = 3000;
  auto run = [&](auto kern, const char* name) {
    for (int r = 0; r < 2; ++r) {
      kern<<<1, 128>>>(vals, xout, cyc, steps);
      cudaDeviceSynchronize();
    }
    const cudaError_t e = cudaGetLastError();
    printf("%-44s %s cycles/step per warp: %.0f %.0f %.0f %.0f\n", name, e ? cudaGetErrorString(e) : "",
           cyc[0] / (double)steps, cyc[1] / (double)steps, cyc[2] / (double)steps, cyc[3] / (double)steps);
  };
  run(k2<0>, "4 warps, own rings only");
  run(k2<4>, "4 warps, own rings, backpressure");
  run(k2<8 + 4>, "+ cross-warp neighbours");
  run(k2<8 + 4 + 16>, "+ box LDS");
  run(k2<8 + 4 + 16 + 1>, "+ stencil LDG");
  run(k2<8 + 4 + 16 + 1 + 2>, "+ x stores (all)");
  run(k2<16 + 1 + 2 + 4>, "all but cross-warp");
  run(k2<8 + 16 + 2 + 4>, "all but stencil LDG");
  run(k2<8 + 4 + 16 + 1 + 64>, "all, x stores as 16 B pairs");
  run(k2<8 + 4 + 16 + 1 + 128>, "all, x stores as 32 B quads");
  run(k2<8 + 4 + 16 + 128>, "all but LDG, x stores as 32 B quads");
  run(k2<8 + 4 + 1>, "ring + backpressure + LDG only");
  run(k2<8 + 4 + 1 + 512>, "  LDG .nc (L1 allocate)");
  run(k2<8 + 4 + 1 + 1024>, "  LDG coherent");
  run(k2<8 + 4 + 1 + 1536>, "  LDG __ldg (not volatile)");
  run(k2<8 + 4 + 16 + 1 + 128 + 256>, "all, quads, LDG.256");
  run(k2<8 + 4 + 1 + 2>, "ring + backpressure + LDG + stores");
  return 0;
}
