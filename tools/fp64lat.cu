// Microbenchmark: dependent-chain latency (cycles) of fp64 / fp32 ops, MUFU.RCP64H,
// LDS and a 4-warp named barrier on this GPU (64-op unrolled chains).
#include <cstdio>
#define CH8(op) op; op; op; op; op; op; op; op;
#define CH64(op) CH8(op) CH8(op) CH8(op) CH8(op) CH8(op) CH8(op) CH8(op) CH8(op)
__global__ void lat(double* out, long long* cyc, double a, double b, int iters) {
  __shared__ double sh[64];
  sh[threadIdx.x % 64] = a;
  __syncthreads();
  double x = a, y = b;
  float f = (float)a, g = (float)b;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { CH64(x = __dadd_rn(x, y)) }
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) { CH64(x = __fma_rn(x, y, a)) }
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) { CH64(f = __fadd_rn(f, g)) }
  long long t3 = clock64();
  int idx = threadIdx.x % 64;
  for (int i = 0; i < iters; ++i) { CH64(idx = (int)sh[idx] & 63) }
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) { CH64(asm volatile("bar.sync 1, 128;" ::: "memory")) }
  long long t5 = clock64();
  double r = b;
  for (int i = 0; i < iters; ++i) { CH8(asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(r))) }
  long long t6 = clock64();
  out[threadIdx.x] = x + f + idx + r;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMallocManaged(&c, 64);
  const int it = 100;
  for (int r = 0; r < 2; ++r) { lat<<<1, 128>>>(o, c, 1.0000001, 1e-9, it); cudaDeviceSynchronize(); }
  const double n = 64.0 * it;
  printf("latency cycles: dadd %.1f dfma %.1f fadd %.1f lds %.1f bar4w %.1f mufu.rcp64h %.1f\n", c[0] / n, c[1] / n, c[2] / n, c[3] / n, c[4] / n, c[5] / (8.0 * it));
  return 0;
}
