// Microbenchmark: one Gauss-Seidel row step's dependent chain on this GPU, per variant, in cycles
// per step (one warp per block, 4 blocks' worth of warps per SM optional).  Variants:
//  0: 12 dependent DADDs (operands ready)                 1: + the three-op division tail
//  2: + 12 DMULs feeding the chain (as the sweep)          3: + publish (STS) / read back (LDS) of the result
//  4: + sentinel compare, vote, branch on the value read   5: variant 4 with 4 warps per block (one per scheduler)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o tools/chainbench tools/chainbench.cu
#include <cstdio>
__device__ __forceinline__ unsigned long long lds64(unsigned a) {
  unsigned long long v;
  asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts64(unsigned a, unsigned long long v) {
  asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
template <int V>
__global__ void k(double* out, long long* cyc, const double* in, int steps) {
  __shared__ unsigned long long ring[6][32][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double c[16], o[12];
  for (int i = 0; i < 16; ++i) c[i] = in[i];
  for (int i = 0; i < 12; ++i) o[i] = in[16 + i] + lane * 1e-3;
  double x = in[30];
  const double d = c[7], y = 1.0 / d;
  for (int sl = 0; sl < 32; ++sl) ring[w][sl][lane] = 0x7ff4deadbeef0badull;
  __syncthreads();
  const unsigned base = (unsigned)__cvta_generic_to_shared(&ring[w][0][0]);
  const unsigned nb = ((lane + 31) & 31) * 8;  // the neighbour lane's slot entry
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    double xin = x;
    if (V >= 3) {
      const unsigned so = (unsigned)(s & 31) * 256u;
      sts64(base + so + lane * 8, (unsigned long long)__double_as_longlong(x));
      sts64(base + (((s + 16) & 31) * 256u) + lane * 8, 0x7ff4deadbeef0badull);
      unsigned long long u = lds64(base + so + nb);
      if (V >= 4) {
        if (!__all_sync(0xffffffffu, u != 0x7ff4deadbeef0badull)) {
          do {
            u = lds64(base + so + nb);
          } while (!__all_sync(0xffffffffu, u != 0x7ff4deadbeef0badull));
        }
      }
      xin = __longlong_as_double((long long)u);
    }
    double sum = c[15];
    if (V >= 2) {
      sum = __dsub_rn(sum, __dmul_rn(c[0], xin));
#pragma unroll
      for (int i = 1; i < 12; ++i) sum = __dsub_rn(sum, __dmul_rn(c[i], o[i]));
    } else {
      sum = __dsub_rn(sum, xin);
#pragma unroll
      for (int i = 1; i < 12; ++i) sum = __dsub_rn(sum, o[i]);
    }
    if (V >= 1) {
      const double q0 = __dmul_rn(sum, y);
      x = __fma_rn(-y, __fma_rn(d, q0, -sum), q0);
    } else {
      x = sum;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double *o, *in;
  long long* c;
  cudaMalloc(&o, 1 << 20);
  cudaMallocManaged(&c, 64);
  cudaMallocManaged(&in, 64 * 8);
  for (int i = 0; i < 64; ++i) in[i] = 1e-3 * (i + 1);
  in[7] = 2.5;
  const int steps = 4000;
#define RUN(V, NT)                                             \
  for (int r = 0; r < 2; ++r) {                                \
    k<V><<<148, NT>>>(o, c, in, steps);                        \
    cudaDeviceSynchronize();                                   \
  }                                                            \
  printf("variant %d (%d warps/block): %.1f cycles per step\n", V, NT / 32, (double)c[0] / steps);
  RUN(0, 32) RUN(1, 32) RUN(2, 32) RUN(3, 32) RUN(4, 32) RUN(4, 128) RUN(4, 192)
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
