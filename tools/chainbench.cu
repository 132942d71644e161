// Calibration microbenchmark: cycles per "relaxation step" of a one-CTA wavefront --
// 14 shared-memory loads feeding a dependent DMUL/DADD row sum, the fast division tail,
// a shared store and a block barrier -- with parts switched off.
// usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o /tmp/cb tools/chainbench.cu && /tmp/cb
#include <cstdio>
__device__ __forceinline__ double div_fast(double s, double d, double y) {
  const double q0 = __dmul_rn(s, y);
  const double r = __fma_rn(-d, q0, s);
  return __fma_rn(y, r, q0);
}
template <int V>
__global__ void bench(double* out, long long* cyc, int steps, int nthreads_active) {
  __shared__ double x[6000];
  for (int i = threadIdx.x; i < 6000; i += blockDim.x) x[i] = 1.0 + i * 1e-7;
  __syncthreads();
  const int t = threadIdx.x;
  const int off[15] = {-343, -342, -325, -324, -19, -18, -1, 0, 1, 18, 19, 324, 325, 342, 343};
  double v[16];
  for (int k = 0; k < 16; ++k) v[k] = 0.01 * (k + 1);
  v[7] = 4.0;
  v[15] = 0.25;
  int i = 400 + t * 17;
  double sum = 0.0;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    if (t < nthreads_active) {
      double acc = x[i + 3];
      if (V & 1) {  // the row chain through shared memory
#pragma unroll
        for (int k = 0; k < 15; ++k)
          if (k != 7) acc = __dsub_rn(acc, __dmul_rn(v[k], x[i + off[k]]));
      }
      if (V & 2) acc = div_fast(acc, v[7], v[15]);
      x[i] = acc;
      sum += acc;
    }
    if (V & 4) __syncthreads();
    i = (i + 1) % 5000 + 400;
  }
  long long t1 = clock64();
  if (t == 0) cyc[V] = (t1 - t0) / steps;
  out[t] = sum;
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 8192);
  cudaMallocManaged(&c, 8 * 8);
  for (int act : {32, 64, 256}) {
    bench<1><<<1, 256>>>(o, c, 200, act);
    bench<3><<<1, 256>>>(o, c, 200, act);
    bench<4><<<1, 256>>>(o, c, 200, act);
    bench<5><<<1, 256>>>(o, c, 200, act);
    bench<7><<<1, 256>>>(o, c, 200, act);
    cudaDeviceSynchronize();
    printf("active %3d: chain %lld  chain+div %lld  barrier only %lld  chain+barrier %lld  all %lld cycles/step\n", act,
           c[1], c[3], c[4], c[5], c[7]);
  }
  return 0;
}
