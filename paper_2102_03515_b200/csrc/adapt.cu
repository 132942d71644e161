// adapt.cu -- the adaptive loop's mesh and marking steps on the device:
//   mark_dorfler   adapt.cpp:126-150  (radix sort by indicator, then the reference's sequential
//                                      sums in sorted order -- one thread, so the cut is exact)
//   bisect_marked  mesh.cpp:67-145    (newest-vertex bisection with conforming closure, round by
//                                      round; midpoints numbered by the first splitting tet, tets
//                                      in order -- the reference mesh, vertex for vertex)
// The estimator lives in assembly.cu (it shares the quadrature and geometry there).
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <climits>

#include "internal.hpp"

namespace rdg {
namespace {

constexpr unsigned long long kEmptyKey = ~0ull;

__device__ __forceinline__ unsigned long long edge_key(int a, int b) {  // mesh.cpp:20-23
  if (a > b) {
    const int t = a;
    a = b;
    b = t;
  }
  return ((unsigned long long)(unsigned)a << 32) | (unsigned)b;
}
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// open-addressing map edge key -> int (linear probing, power-of-two capacity)
struct EdgeMap {
  unsigned long long* key;
  int* val;
  uint64_t mask;
  __device__ int find(unsigned long long k) const {
    uint64_t h = mix64(k) & mask;
    for (;;) {
      const unsigned long long s = key[h];
      if (s == k) return val[h];
      if (s == kEmptyKey) return -1;
      h = (h + 1) & mask;
    }
  }
  // slot of k, inserting it when absent
  __device__ uint64_t slot(unsigned long long k) const {
    uint64_t h = mix64(k) & mask;
    for (;;) {
      const unsigned long long prev = atomicCAS(key + h, kEmptyKey, k);
      if (prev == kEmptyKey || prev == k) return h;
      h = (h + 1) & mask;
    }
  }
};

__device__ __forceinline__ bool on_unit_boundary(const double* x) {  // mesh.cpp:14-18
  for (int c = 0; c < 3; ++c)
    if (fabs(x[c]) <= 1e-14 || fabs(__dsub_rn(x[c], 1.0)) <= 1e-14) return true;
  return false;
}

__global__ void mark_flags_kernel(int nm, const int* __restrict__ marked, int nt, int* flag, int* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nm) return;
  const int t = marked[i];
  if (t < 0 || t >= nt)
    atomicExch(bad, 1);
  else
    flag[t] = 1;
}

// flagged tets: the midpoint of edge (p0, pd) from earlier rounds, or a pending entry that
// remembers the lowest splitting tet (which numbers the new vertex)
__global__ void split_lookup_kernel(int nt, const int* __restrict__ flag, const int* __restrict__ tets,
                                    const uint8_t* __restrict__ tag, EdgeMap mid, EdgeMap pend, int* zt) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt || !flag[t]) return;
  const int d = tag[t];
  const unsigned long long k = edge_key(tets[4 * (int64_t)t], tets[4 * (int64_t)t + d]);
  const int z = mid.find(k);
  zt[t] = z;
  if (z < 0) atomicMin(pend.val + pend.slot(k), t);
}

__global__ void first_split_kernel(int nt, const int* __restrict__ flag, const int* __restrict__ tets,
                                   const uint8_t* __restrict__ tag, const int* __restrict__ zt, EdgeMap pend,
                                   int* first) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  int f = 0;
  if (flag[t] && zt[t] < 0) {
    const int d = tag[t];
    f = pend.find(edge_key(tets[4 * (int64_t)t], tets[4 * (int64_t)t + d])) == t ? 1 : 0;
  }
  first[t] = f;
}

// new vertex z = nv + rank of its first splitting tet: 0.5 (x_a + x_b) (mesh.cpp:80-86)
__global__ void new_vertex_kernel(int nt, int nv, const int* __restrict__ first, const int* __restrict__ off,
                                  const int* __restrict__ tets, const uint8_t* __restrict__ tag, double* xyz,
                                  uint8_t* bnd, EdgeMap mid) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt || !first[t]) return;
  const int a = tets[4 * (int64_t)t], b = tets[4 * (int64_t)t + tag[t]];
  const int z = nv + off[t];
  double x[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    x[c] = __dmul_rn(0.5, __dadd_rn(xyz[3 * (int64_t)a + c], xyz[3 * (int64_t)b + c]));
    xyz[3 * (int64_t)z + c] = x[c];
  }
  bnd[z] = on_unit_boundary(x) ? 1 : 0;
  mid.val[mid.slot(edge_key(a, b))] = z;
}

__global__ void child_count_kernel(int nt, const int* __restrict__ flag, int* cnt) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nt) cnt[t] = flag[t] ? 2 : 1;
}

// mesh.cpp:92-124: c1 = p with p[d] -> z; c2 = (p1 .. p_d, z, p_{d+1} ..); tag d -> d == 1 ? 3 : d - 1
__global__ void children_kernel(int nt, const int* __restrict__ flag, const int* __restrict__ off,
                                const int* __restrict__ tets, const uint8_t* __restrict__ tag,
                                const int* __restrict__ gen, const int* __restrict__ zt, EdgeMap mid, int* tets2,
                                uint8_t* tag2, int* gen2) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const int o = off[t];
  int p[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) p[k] = tets[4 * (int64_t)t + k];
  if (!flag[t]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) tets2[4 * (int64_t)o + k] = p[k];
    tag2[o] = tag[t];
    gen2[o] = gen[t];
    return;
  }
  const int d = tag[t];
  int z = zt[t];
  if (z < 0) z = mid.find(edge_key(p[0], p[d]));
  int c1[4], c2[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) c1[k] = p[k];
  c1[d] = z;
  for (int q = 0; q < d; ++q) c2[q] = p[q + 1];
  c2[d] = z;
  for (int q = d + 1; q < 4; ++q) c2[q] = p[q];
  const uint8_t nd = (uint8_t)(d == 1 ? 3 : d - 1);
  const int g = gen[t] + 1;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    tets2[4 * (int64_t)o + k] = c1[k];
    tets2[4 * (int64_t)(o + 1) + k] = c2[k];
  }
  tag2[o] = tag2[o + 1] = nd;
  gen2[o] = gen2[o + 1] = g;
}

// mesh.cpp:127-137: a tet carrying any split edge is bisected in the next round
__global__ void closure_kernel(int nt, const int* __restrict__ tets, EdgeMap mid, int* flag) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  constexpr int kE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  int p[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) p[k] = tets[4 * (int64_t)t + k];
  int f = 0;
#pragma unroll
  for (int e = 0; e < 6; ++e)
    if (!f && mid.find(edge_key(p[kE[e][0]], p[kE[e][1]])) >= 0) f = 1;
  flag[t] = f;
}

__global__ void rehash_kernel(uint64_t cap_old, const unsigned long long* __restrict__ k_old,
                              const int* __restrict__ v_old, EdgeMap mid) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cap_old || k_old[i] == kEmptyKey) return;
  mid.val[mid.slot(k_old[i])] = v_old[i];
}

__global__ void fill_u8_kernel(int64_t n, uint8_t v, uint8_t* a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

// adapt.cpp:139-149 in sorted order: total, goal = theta^2 total, then the prefix that reaches it.
// The sums are sequential (the cut must see the reference's rounding), so one thread runs them;
// the block stages each chunk's squares in shared memory first, so that thread only chains adds.
constexpr int kCutNT = 256, kCutChunk = 4096;
__global__ void __launch_bounds__(kCutNT) dorfler_cut_kernel(int n, const unsigned long long* __restrict__ sorted_bits,
                                                             double theta, int* count) {
  __shared__ double sq[kCutChunk];
  __shared__ int stop;
  double total = 0.0;
  for (int c0 = 0; c0 < n; c0 += kCutChunk) {
    const int m = min(kCutChunk, n - c0);
    for (int k = threadIdx.x; k < m; k += kCutNT) {
      const double e = __longlong_as_double((long long)sorted_bits[c0 + k]);
      sq[k] = __dmul_rn(e, e);
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < m; ++k) total = __dadd_rn(total, sq[k]);
    __syncthreads();
  }
  const double goal = __dmul_rn(__dmul_rn(theta, theta), total);  // thread 0's value is the one used
  double acc = 0.0;
  int kk = 0;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  for (int c0 = 0; c0 < n && !stop; c0 += kCutChunk) {
    const int m = min(kCutChunk, n - c0);
    for (int k = threadIdx.x; k < m; k += kCutNT) {
      const double e = __longlong_as_double((long long)sorted_bits[c0 + k]);
      sq[k] = e == 0.0 ? -1.0 : __dmul_rn(e, e);  // -1: a zero indicator ends the marking
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int k = 0;
      for (; k < m; ++k) {
        if (acc >= goal || sq[k] < 0.0) {
          stop = 1;
          break;
        }
        acc = __dadd_rn(acc, sq[k]);
      }
      kk = c0 + k;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = kk;
}

__global__ void iota_kernel(int n, int* a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

uint64_t pow2_at_least(uint64_t x) {
  uint64_t c = 1024;
  while (c < x) c <<= 1;
  return c;
}

struct MapBuf {
  DBuf<unsigned long long> k;
  DBuf<int> v;
  uint64_t cap = 0;
  void alloc(Ctx& c, uint64_t n, int vinit) {
    cap = n;
    k.alloc(n, c.stream);
    v.alloc(n, c.stream);
    RDG_CUDA(cudaMemsetAsync(k.p, 0xff, sizeof(unsigned long long) * n, c.stream));
    if (vinit == -1)
      RDG_CUDA(cudaMemsetAsync(v.p, 0xff, sizeof(int) * n, c.stream));
    else
      RDG_CUDA(cudaMemsetAsync(v.p, 0x7f, sizeof(int) * n, c.stream));  // 0x7f7f7f7f: above any tet id
  }
  EdgeMap view() const { return EdgeMap{k.p, v.p, cap - 1}; }
};

}  // namespace

void mark_dorfler(Ctx& c, int n, const double* eta, double theta, int* marked, int* count) {
  if (!(theta > 0.0 && theta <= 1.0)) throw Error(RD_EINVAL, "mark_dorfler: theta must be in (0, 1]");
  if (n <= 0) {
    *count = 0;
    return;
  }
  // eta >= 0: the IEEE bit patterns sort like the values; the radix sort is stable, so equal
  // indicators keep ascending tet order (adapt.cpp:131-135's tie-break)
  DBuf<unsigned long long> kout(n, c.stream);
  DBuf<int> idx(n, c.stream), cnt(1, c.stream);
  iota_kernel<<<div_up(n, 256), 256, 0, c.stream>>>(n, idx.p);
  RDG_LAUNCH_CHECK();
  ++c.launches;
  const unsigned long long* kin = reinterpret_cast<const unsigned long long*>(eta);
  size_t tmp_bytes = 0;
  RDG_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, kin, kout.p, idx.p, marked, n, 0, 64,
                                                     c.stream));
  DBuf<char> tmp(std::max<size_t>(tmp_bytes, 1), c.stream);
  RDG_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.p, tmp_bytes, kin, kout.p, idx.p, marked, n, 0, 64,
                                                     c.stream));
  dorfler_cut_kernel<<<1, kCutNT, 0, c.stream>>>(n, kout.p, theta, cnt.p);
  RDG_LAUNCH_CHECK();
  c.launches += 2;
  RDG_CUDA(cudaMemcpyAsync(count, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  RDG_CUDA(cudaStreamSynchronize(c.stream));
}

void bisect_marked(Ctx& c, const DMesh& in, const int* marked, int nm, DMesh& out) {
  int nv = in.nv, nt = in.nt;
  // working mesh (vertex arrays grow by doubling; the tet arrays are rebuilt every round)
  size_t cap_v = std::max<size_t>((size_t)nv * 2, 1024);
  DBuf<double> xyz(3 * cap_v, c.stream);
  DBuf<uint8_t> bnd(cap_v, c.stream);
  DBuf<int> tets(std::max<int64_t>(4 * (int64_t)nt, 4), c.stream), gen(std::max(nt, 1), c.stream);
  DBuf<uint8_t> tag(std::max(nt, 1), c.stream);
  if (nv) {
    RDG_CUDA(cudaMemcpyAsync(xyz.p, in.xyz.p, sizeof(double) * 3 * nv, cudaMemcpyDeviceToDevice, c.stream));
    RDG_CUDA(cudaMemcpyAsync(bnd.p, in.boundary.p, nv, cudaMemcpyDeviceToDevice, c.stream));
  }
  if (nt) {
    RDG_CUDA(cudaMemcpyAsync(tets.p, in.tets.p, sizeof(int) * 4 * (size_t)nt, cudaMemcpyDeviceToDevice, c.stream));
    if (in.tag.p) {
      RDG_CUDA(cudaMemcpyAsync(tag.p, in.tag.p, nt, cudaMemcpyDeviceToDevice, c.stream));
      RDG_CUDA(cudaMemcpyAsync(gen.p, in.gen.p, sizeof(int) * (size_t)nt, cudaMemcpyDeviceToDevice, c.stream));
    } else {  // build_structured_cube / uploaded meshes: tag 3, generation 0 (mesh.cpp:60-61)
      fill_u8_kernel<<<div_up(nt, 256), 256, 0, c.stream>>>(nt, 3, tag.p);
      RDG_LAUNCH_CHECK();
      RDG_CUDA(cudaMemsetAsync(gen.p, 0, sizeof(int) * (size_t)nt, c.stream));
      ++c.launches;
    }
  }
  DBuf<int> flag(std::max(nt, 1), c.stream), bad(1, c.stream);
  RDG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int) * std::max(nt, 1), c.stream));
  RDG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c.stream));
  if (nm > 0) {
    mark_flags_kernel<<<div_up(nm, 256), 256, 0, c.stream>>>(nm, marked, nt, flag.p, bad.p);
    RDG_LAUNCH_CHECK();
    ++c.launches;
  }
  int hbad = 0;
  RDG_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  RDG_CUDA(cudaStreamSynchronize(c.stream));
  if (hbad) throw Error(RD_EINVAL, "bisect_marked: tet index out of range");

  MapBuf mid;
  mid.alloc(c, pow2_at_least(2 * (uint64_t)std::max(nm, 1) + 1024), -1);
  int64_t n_mid = 0;
  DBuf<int> cnt, off;
  for (int round = 0;; ++round) {
    cnt.alloc(std::max(nt, 1), c.stream);
    off.alloc((size_t)nt + 1, c.stream);
    const int64_t nflag = exclusive_scan(c, flag.p, off.p, nt);
    if (nflag == 0) break;
    if (round >= 1000) throw Error(RD_ERUNTIME, "bisect_marked: conforming closure did not terminate");
    if ((uint64_t)(n_mid + nflag) * 2 > mid.cap) {  // keep the midpoint map at most half full
      MapBuf bigger;
      bigger.alloc(c, pow2_at_least(4 * (uint64_t)(n_mid + nflag)), -1);
      rehash_kernel<<<div_up((int64_t)mid.cap, 256), 256, 0, c.stream>>>(mid.cap, mid.k.p, mid.v.p, bigger.view());
      RDG_LAUNCH_CHECK();
      ++c.launches;
      mid = std::move(bigger);
    }
    MapBuf pend;
    pend.alloc(c, pow2_at_least(2 * (uint64_t)nflag), 0x7f7f7f7f);
    DBuf<int> zt(std::max(nt, 1), c.stream), first(std::max(nt, 1), c.stream);
    const int g = div_up(nt, 256);
    split_lookup_kernel<<<g, 256, 0, c.stream>>>(nt, flag.p, tets.p, tag.p, mid.view(), pend.view(), zt.p);
    first_split_kernel<<<g, 256, 0, c.stream>>>(nt, flag.p, tets.p, tag.p, zt.p, pend.view(), first.p);
    RDG_LAUNCH_CHECK();
    c.launches += 2;
    const int64_t nnew = exclusive_scan(c, first.p, off.p, nt);
    if ((size_t)nv + (size_t)nnew > cap_v) {  // grow the vertex arrays
      const size_t cap2 = std::max(cap_v * 2, (size_t)nv + (size_t)nnew);
      DBuf<double> x2(3 * cap2, c.stream);
      DBuf<uint8_t> b2(cap2, c.stream);
      RDG_CUDA(cudaMemcpyAsync(x2.p, xyz.p, sizeof(double) * 3 * (size_t)nv, cudaMemcpyDeviceToDevice, c.stream));
      RDG_CUDA(cudaMemcpyAsync(b2.p, bnd.p, (size_t)nv, cudaMemcpyDeviceToDevice, c.stream));
      xyz = std::move(x2);
      bnd = std::move(b2);
      cap_v = cap2;
    }
    if (nnew + (int64_t)nv > INT_MAX) throw Error(RD_EINVAL, "bisect_marked: vertex count exceeds int32");
    new_vertex_kernel<<<g, 256, 0, c.stream>>>(nt, nv, first.p, off.p, tets.p, tag.p, xyz.p, bnd.p, mid.view());
    RDG_LAUNCH_CHECK();
    child_count_kernel<<<g, 256, 0, c.stream>>>(nt, flag.p, cnt.p);
    RDG_LAUNCH_CHECK();
    c.launches += 2;
    const int64_t nt2 = exclusive_scan(c, cnt.p, off.p, nt);
    DBuf<int> tets2(std::max<int64_t>(4 * nt2, 4), c.stream), gen2(std::max<int64_t>(nt2, 1), c.stream);
    DBuf<uint8_t> tag2(std::max<int64_t>(nt2, 1), c.stream);
    children_kernel<<<g, 256, 0, c.stream>>>(nt, flag.p, off.p, tets.p, tag.p, gen.p, zt.p, mid.view(), tets2.p,
                                             tag2.p, gen2.p);
    RDG_LAUNCH_CHECK();
    ++c.launches;
    nv += (int)nnew;
    n_mid += nnew;
    nt = (int)nt2;
    tets = std::move(tets2);
    tag = std::move(tag2);
    gen = std::move(gen2);
    flag.alloc(std::max(nt, 1), c.stream);
    closure_kernel<<<div_up(nt, 256), 256, 0, c.stream>>>(nt, tets.p, mid.view(), flag.p);
    RDG_LAUNCH_CHECK();
    ++c.launches;
  }
  out.nv = nv;
  out.nt = nt;
  out.lattice_n = -1;
  out.xyz.alloc(std::max<int64_t>(3 * (int64_t)nv, 1), c.stream);
  out.boundary.alloc(std::max(nv, 1), c.stream);
  if (nv) {
    RDG_CUDA(cudaMemcpyAsync(out.xyz.p, xyz.p, sizeof(double) * 3 * (size_t)nv, cudaMemcpyDeviceToDevice, c.stream));
    RDG_CUDA(cudaMemcpyAsync(out.boundary.p, bnd.p, (size_t)nv, cudaMemcpyDeviceToDevice, c.stream));
  }
  out.tets = std::move(tets);
  out.tag = std::move(tag);
  out.gen = std::move(gen);
  RDG_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace rdg
