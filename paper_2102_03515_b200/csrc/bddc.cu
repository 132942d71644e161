// bddc.cu -- BDDC on the device (reference bddc.cpp:45-456).
//
// Setup: the combinatorial part (RCB partition of tet centroids, interface / corner / face-class
// sets, per-subdomain index lists) runs on the host from the mesh arrays, as in the reference.
// Each subdomain's Neumann matrix rho K + M over its own tets is assembled on the device by the
// generic assembly kernels (a mesh view holding only those tets), gathered into one dense
// column-major block [[A_II, A_IB], [A_BI, A_BB]], and the local problems are dense on the B200:
// A_II Cholesky (cuSOLVER potrf), X = A_II^-1 A_IB (potrs), S = A_BB - A_BI X (cuBLAS dgemm),
// symmetrised; the saddle matrix [[S, C'], [C, 0]] LU-factored (getrf) and the constrained basis
// Phi from it; the coarse matrix sum_s Phi' S Phi (dgemm) factored by the whole-GPU Cholesky.
// Applies (schur_apply / reduce_rhs / expand_solution / bddc_apply) run per subdomain in the
// reference's order s = 0 .. p-1 (scatter-adds in that order: deterministic).
// Parity with the reference is to rounding (its own tests' bars, 1e-10 .. 1e-7): Eigen's
// SimplicialLLT / PartialPivLU orders are not restated.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <functional>
#include <map>
#include <numeric>
#include <string>

#include "internal.hpp"

namespace rdg {

#define RDG_CUBLAS(x)                                                                   \
  do {                                                                                  \
    const cublasStatus_t st_ = (x);                                                     \
    if (st_ != CUBLAS_STATUS_SUCCESS) throw Error(RD_ECUDA, std::string("cuBLAS: ") + #x); \
  } while (0)
#define RDG_CUSOLVER(x)                                                                     \
  do {                                                                                      \
    const cusolverStatus_t st_ = (x);                                                       \
    if (st_ != CUSOLVER_STATUS_SUCCESS) throw Error(RD_ECUDA, std::string("cuSOLVER: ") + #x); \
  } while (0)

namespace {

__global__ void gather_tets_kernel(int n, const int* __restrict__ ids, const int* __restrict__ tets, int* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  reinterpret_cast<int4*>(out)[k] = reinterpret_cast<const int4*>(tets)[ids[k]];
}

// dense column-major local matrix (nloc x nloc) from the subdomain CSR (global dof numbering)
__global__ void local_dense_kernel(int nloc, const int* __restrict__ dofs, const int* __restrict__ gloc,
                                   const int* __restrict__ rp, const int* __restrict__ ci,
                                   const double* __restrict__ v, double* D) {
  const int r = blockIdx.x;
  const int g = dofs[r];
  for (int k = rp[g] + threadIdx.x; k < rp[g + 1]; k += blockDim.x) {
    const int lc = gloc[ci[k]];
    if (lc >= 0) D[(size_t)lc * nloc + r] = v[k];
  }
}
__global__ void set_map_kernel(int n, const int* __restrict__ dofs, int* gloc, int val_is_index) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) gloc[dofs[k]] = val_is_index ? k : -1;
}
// out (col-major nB x nB) = 0.5 (B + B') from a block inside a larger column-major matrix
__global__ void symmetrize_kernel(int nB, const double* __restrict__ B, int ldb, double* S) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nB * nB) return;
  const int i = (int)(e % nB), j = (int)(e / nB);
  S[(size_t)j * nB + i] = __dmul_rn(0.5, __dadd_rn(B[(size_t)j * ldb + i], B[(size_t)i * ldb + j]));
}
// saddle (col-major m x m) = [[S, C'], [C, 0]]
__global__ void saddle_kernel(int nB, int nc, const double* __restrict__ S, const double* __restrict__ C, double* M) {
  const int m = nB + nc;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)m * m) return;
  const int i = (int)(e % m), j = (int)(e / m);
  double v = 0.0;
  if (i < nB && j < nB) v = S[(size_t)j * nB + i];
  else if (i < nB && j >= nB) v = C[(size_t)i * nc + (j - nB)];  // C' (C stored col-major nc x nB: C[b*nc + r])
  else if (i >= nB && j < nB) v = C[(size_t)j * nc + (i - nB)];
  M[e] = v;
}
__global__ void unit_rhs_kernel(int nB, int nc, double* R) {  // m x nc: [0; I]
  const int m = nB + nc;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)m * nc) return;
  const int i = (int)(e % m), j = (int)(e / m);
  R[e] = i == nB + j ? 1.0 : 0.0;
}
__global__ void coarse_add_kernel(int nc, int np, const int* __restrict__ pidx, const double* __restrict__ Q,
                                  double* Cm) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nc * nc) return;
  const int r = e % nc, c = e / nc;  // Q col-major
  double* t = Cm + (size_t)pidx[c] * np + pidx[r];
  *t = __dadd_rn(*t, Q[e]);
}
__global__ void gather_kernel(int n, const int* __restrict__ idx, const double* __restrict__ x, double* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = x[idx[k]];
}
__global__ void gather_scaled_kernel(int n, const int* __restrict__ idx, const double* __restrict__ sc,
                                     const double* __restrict__ x, double* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = __dmul_rn(sc[k], x[idx[k]]);
}
__global__ void scatter_kernel(int n, const int* __restrict__ idx, const double* __restrict__ x, double* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[idx[k]] = x[k];
}
// out[idx[k]] op= x[k] (sign -1: subtract), optionally scaled
__global__ void scatter_add_kernel(int n, const int* __restrict__ idx, const double* __restrict__ sc,
                                   const double* __restrict__ x, double sign, double* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double v = sc ? __dmul_rn(sc[k], x[k]) : x[k];
  out[idx[k]] = sign > 0 ? __dadd_rn(out[idx[k]], v) : __dsub_rn(out[idx[k]], v);
}
__global__ void sub_kernel(int n, const double* __restrict__ a, double* b) {  // b = a - b
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) b[k] = __dsub_rn(a[k], b[k]);
}

}  // namespace

struct BddcSubDev {
  int nI = 0, nB = 0, ncon = 0;
  std::vector<int> interior, boundary, bidx, pidx;
  DBuf<int> d_interior, d_bidx, d_pidx;
  DBuf<double> scaling;
  DBuf<double> A;    // (nI + nB)^2 col-major: A_II factored in place, A_IB, A_BI, (A_BB - A_BI X)
  DBuf<double> S;    // nB x nB
  DBuf<double> sad;  // (nB + ncon)^2 LU
  DBuf<int> ipiv;
  DBuf<double> Phi;  // nB x ncon
  DBuf<double> C;    // ncon x nB col-major (for the saddle assembly)
};

struct Bddc {
  Ctx* c = nullptr;
  int p = 0, n_dofs = 0, nC = 0, n_primal = 0;
  std::vector<int> owner, interface_dofs, interface_index;
  std::vector<std::vector<int>> dof_subdomains;
  DBuf<int> d_iface;
  DCsr A_CC;
  std::vector<BddcSubDev> subs;
  DBuf<double> coarse;  // np x np (lower factor after setup, row-major as dense_llt_solve reads it)
  DBuf<double> coarse_raw;
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t sol = nullptr;
  DBuf<int> info;
  DBuf<double> w1, w2, w3, rp;  // scratch
  ~Bddc() {
    if (blas) cublasDestroy(blas);
    if (sol) cusolverDnDestroy(sol);
  }
};

namespace {

// bddc.cpp:45-111 (the RCB partition of tet centroids; host setup)
void partition_host(const std::vector<double>& xyz, const std::vector<int>& tets, int nt, int p,
                    std::vector<int>& owner) {
  std::vector<double> cen((size_t)nt * 3);
  for (int t = 0; t < nt; ++t)
    for (int c = 0; c < 3; ++c) {
      const double* v[4];
      for (int k = 0; k < 4; ++k) v[k] = &xyz[3 * (size_t)tets[4 * (size_t)t + k]];
      cen[3 * (size_t)t + c] = 0.25 * (((v[0][c] + v[1][c]) + v[2][c]) + v[3][c]);
    }
  owner.assign((size_t)nt, -1);
  std::function<void(std::vector<int>&, int, int)> rcb = [&](std::vector<int>& ids, int parts, int label) {
    if (parts == 1) {
      for (int t : ids) owner[(size_t)t] = label;
      return;
    }
    double lo[3], hi[3];
    for (int c = 0; c < 3; ++c) lo[c] = hi[c] = cen[3 * (size_t)ids.front() + c];
    for (int t : ids)
      for (int c = 0; c < 3; ++c) {
        lo[c] = std::min(lo[c], cen[3 * (size_t)t + c]);
        hi[c] = std::max(hi[c], cen[3 * (size_t)t + c]);
      }
    int axis = 0;
    double ext = hi[0] - lo[0];
    for (int a = 1; a < 3; ++a)
      if (hi[a] - lo[a] > ext) {
        ext = hi[a] - lo[a];
        axis = a;
      }
    std::sort(ids.begin(), ids.end(), [&](int a, int b) {
      const double ca = cen[3 * (size_t)a + axis], cb = cen[3 * (size_t)b + axis];
      if (ca != cb) return ca < cb;
      return a < b;
    });
    const int p1 = parts / 2;
    const int64_t n1 = (int64_t)ids.size() * p1 / parts;
    std::vector<int> left(ids.begin(), ids.begin() + n1), right(ids.begin() + n1, ids.end());
    rcb(left, p1, label);
    rcb(right, parts - p1, label + p1);
  };
  std::vector<int> all((size_t)nt);
  std::iota(all.begin(), all.end(), 0);
  rcb(all, p, 0);
}

template <class T>
std::vector<T> download(Ctx& c, const T* d, size_t n) {
  std::vector<T> h(n);
  if (n) RDG_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost, c.stream));
  RDG_CUDA(cudaStreamSynchronize(c.stream));
  return h;
}
template <class T>
void upload(Ctx& c, DBuf<T>& d, const std::vector<T>& h) {
  d.alloc(std::max<size_t>(h.size(), 1), c.stream);
  if (!h.empty()) RDG_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, c.stream));
}

void check_info(Ctx& c, Bddc& b, const char* what) {
  int h = 0;
  RDG_CUDA(cudaMemcpyAsync(&h, b.info.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  RDG_CUDA(cudaStreamSynchronize(c.stream));
  if (h != 0) throw Error(RD_ERUNTIME, what);
}

inline int g256(int64_t n) { return (int)std::max<int64_t>(1, (n + 255) / 256); }

}  // namespace

void partition_geometric(Ctx& c, const DMesh& m, const DSystem& s, int p, std::vector<int>& owner,
                         std::vector<std::vector<int>>& dof_subdomains) {
  if (p < 2) throw Error(RD_EINVAL, "partition_geometric: p must be >= 2");
  if (p > m.nt) throw Error(RD_EINVAL, "partition_geometric: more subdomains than tets");
  const auto xyz = download(c, m.xyz.p, 3 * (size_t)m.nv);
  const auto tets = download(c, m.tets.p, 4 * (size_t)m.nt);
  const auto v2d = download(c, s.v2d.p, (size_t)m.nv);
  partition_host(xyz, tets, m.nt, p, owner);
  dof_subdomains.assign((size_t)s.n_dofs, {});
  for (int t = 0; t < m.nt; ++t)
    for (int k = 0; k < 4; ++k) {
      const int d = v2d[(size_t)tets[4 * (size_t)t + k]];
      if (d >= 0) dof_subdomains[(size_t)d].push_back(owner[(size_t)t]);
    }
  for (auto& ss : dof_subdomains) {
    std::sort(ss.begin(), ss.end());
    ss.erase(std::unique(ss.begin(), ss.end()), ss.end());
  }
}

// bddc.cpp:113-301
Bddc* build_bddc(Ctx& c, const DMesh& m, const DSystem& sys, int p) {
  auto op = std::make_unique<Bddc>();
  Bddc& b = *op;
  b.c = &c;
  b.p = p;
  b.n_dofs = sys.n_dofs;
  partition_geometric(c, m, sys, p, b.owner, b.dof_subdomains);
  const int nd = sys.n_dofs;
  b.interface_index.assign((size_t)nd, -1);
  for (int d = 0; d < nd; ++d)
    if (b.dof_subdomains[(size_t)d].size() >= 2) {
      b.interface_index[(size_t)d] = (int)b.interface_dofs.size();
      b.interface_dofs.push_back(d);
    }
  b.nC = (int)b.interface_dofs.size();
  upload(c, b.d_iface, b.interface_dofs);
  RDG_CUBLAS(cublasCreate(&b.blas));
  RDG_CUBLAS(cublasSetStream(b.blas, c.stream));
  RDG_CUSOLVER(cusolverDnCreate(&b.sol));
  RDG_CUSOLVER(cusolverDnSetStream(b.sol, c.stream));
  b.info.alloc(1, c.stream);

  // A_CC (bddc.cpp:16-30): the interface rows of A, interface columns, from the host copy
  {
    const auto rp = download(c, sys.A.rp.p, (size_t)sys.A.rows + 1);
    const auto ci = download(c, sys.A.ci.p, (size_t)sys.A.nnz);
    const auto va = download(c, sys.A.v.p, (size_t)sys.A.nnz);
    std::vector<int> crp(1, 0), cci;
    std::vector<double> cv;
    for (int d : b.interface_dofs) {
      for (int k = rp[(size_t)d]; k < rp[(size_t)d + 1]; ++k) {
        const int col = b.interface_index[(size_t)ci[(size_t)k]];
        if (col >= 0 && va[(size_t)k] != 0.0) {
          cci.push_back(col);
          cv.push_back(va[(size_t)k]);
        }
      }
      crp.push_back((int)cci.size());
    }
    DCsr& A = b.A_CC;
    A.rows = A.cols = b.nC;
    A.nnz = (int64_t)cci.size();
    upload(c, A.rp, crp);
    upload(c, A.ci, cci);
    upload(c, A.v, cv);
  }

  // corners and face classes (bddc.cpp:130-178)
  const auto tets_h = download(c, m.tets.p, 4 * (size_t)m.nt);
  const auto bnd = download(c, m.boundary.p, (size_t)m.nv);
  const auto v2d = download(c, sys.v2d.p, (size_t)m.nv);
  std::vector<uint8_t> near_boundary((size_t)nd, 0);
  constexpr int edges[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  for (int t = 0; t < m.nt; ++t)
    for (const auto& e : edges) {
      const int a = tets_h[4 * (size_t)t + e[0]], bb = tets_h[4 * (size_t)t + e[1]];
      if (bnd[(size_t)a] != bnd[(size_t)bb]) near_boundary[(size_t)v2d[(size_t)(bnd[(size_t)a] ? bb : a)]] = 1;
    }
  std::vector<uint8_t> is_corner((size_t)nd, 0);
  for (int d : b.interface_dofs) {
    const size_t mult = b.dof_subdomains[(size_t)d].size();
    is_corner[(size_t)d] = (mult >= 3 || (mult >= 2 && near_boundary[(size_t)d])) ? 1 : 0;
  }
  std::map<std::vector<int>, int> class_of_key;
  std::vector<std::vector<int>> class_dofs, class_key;
  for (int d : b.interface_dofs) {
    if (is_corner[(size_t)d]) continue;
    const auto& key = b.dof_subdomains[(size_t)d];
    auto it = class_of_key.find(key);
    if (it == class_of_key.end()) {
      it = class_of_key.emplace(key, (int)class_dofs.size()).first;
      class_dofs.emplace_back();
      class_key.push_back(key);
    }
    class_dofs[(size_t)it->second].push_back(d);
  }
  std::vector<int> corner_primal((size_t)nd, -1);
  int np = 0;
  for (int d : b.interface_dofs)
    if (is_corner[(size_t)d]) corner_primal[(size_t)d] = np++;
  const int first_class = np;
  np += (int)class_dofs.size();
  b.n_primal = np;
  std::vector<std::vector<int>> sub_classes((size_t)p);
  for (size_t k = 0; k < class_key.size(); ++k)
    for (int sdx : class_key[k]) sub_classes[(size_t)sdx].push_back((int)k);

  b.subs.resize((size_t)p);
  std::vector<std::vector<int>> sub_tets((size_t)p);
  for (int t = 0; t < m.nt; ++t) sub_tets[(size_t)b.owner[(size_t)t]].push_back(t);
  for (int d = 0; d < nd; ++d) {
    const auto& ss = b.dof_subdomains[(size_t)d];
    if (ss.size() == 1)
      b.subs[(size_t)ss[0]].interior.push_back(d);
    else
      for (int sdx : ss) b.subs[(size_t)sdx].boundary.push_back(d);
  }
  DBuf<int> gloc(std::max(nd, 1), c.stream);
  RDG_CUDA(cudaMemsetAsync(gloc.p, 0xff, sizeof(int) * std::max(nd, 1), c.stream));
  b.coarse_raw.alloc(std::max<size_t>((size_t)np * np, 1), c.stream);
  RDG_CUDA(cudaMemsetAsync(b.coarse_raw.p, 0, sizeof(double) * std::max<size_t>((size_t)np * np, 1), c.stream));
  const double one = 1.0, zero = 0.0, mone = -1.0;

  for (int sdx = 0; sdx < p; ++sdx) {
    BddcSubDev& sd = b.subs[(size_t)sdx];
    const int nI = sd.nI = (int)sd.interior.size();
    const int nB = sd.nB = (int)sd.boundary.size();
    const int nloc = nI + nB;
    sd.bidx.resize((size_t)nB);
    std::vector<double> scal((size_t)nB);
    for (int k = 0; k < nB; ++k) {
      const int d = sd.boundary[(size_t)k];
      sd.bidx[(size_t)k] = b.interface_index[(size_t)d];
      scal[(size_t)k] = 1.0 / (double)b.dof_subdomains[(size_t)d].size();
    }
    upload(c, sd.d_interior, sd.interior);
    upload(c, sd.d_bidx, sd.bidx);
    upload(c, sd.scaling, scal);
    // constraint rows: local corners then face classes (bddc.cpp:233-254)
    std::vector<int> local_corners;
    for (int d : sd.boundary)
      if (is_corner[(size_t)d]) local_corners.push_back(d);
    const auto& cls = sub_classes[(size_t)sdx];
    const int nc = sd.ncon = (int)(local_corners.size() + cls.size());
    std::vector<double> Ch((size_t)nc * nB, 0.0);  // col-major nc x nB: C(r, b) at b * nc + r
    auto lbi = [&](int d) { return (int)(std::lower_bound(sd.boundary.begin(), sd.boundary.end(), d) - sd.boundary.begin()); };
    int row = 0;
    for (int d : local_corners) {
      Ch[(size_t)lbi(d) * nc + row] = 1.0;
      sd.pidx.push_back(corner_primal[(size_t)d]);
      ++row;
    }
    for (int k : cls) {
      const auto& members = class_dofs[(size_t)k];
      const double w = 1.0 / (double)members.size();
      for (int d : members) Ch[(size_t)lbi(d) * nc + row] = w;
      sd.pidx.push_back(first_class + k);
      ++row;
    }
    upload(c, sd.C, Ch);
    upload(c, sd.d_pidx, sd.pidx);
    if (nloc == 0) continue;

    // the subdomain's Neumann matrix rho K + M (assembly.cpp:250-263) on a mesh view of its tets
    DMesh sub;
    sub.nv = m.nv;
    sub.nt = (int)sub_tets[(size_t)sdx].size();
    sub.lattice_n = -1;
    sub.xyz = DBuf<double>::view(m.xyz.p, 3 * (size_t)m.nv);
    sub.boundary = DBuf<uint8_t>::view(m.boundary.p, (size_t)m.nv);
    {
      DBuf<int> ids;
      upload(c, ids, sub_tets[(size_t)sdx]);
      sub.tets.alloc(std::max<int64_t>(4 * (int64_t)sub.nt, 4), c.stream);
      if (sub.nt) {
        gather_tets_kernel<<<g256(sub.nt), 256, 0, c.stream>>>(sub.nt, ids.p, m.tets.p, sub.tets.p);
        RDG_LAUNCH_CHECK();
        ++c.launches;
      }
      RDG_CUDA(cudaStreamSynchronize(c.stream));
    }
    DSystem ss;
    build_system(c, sub, sys.rho, RD_TARGET_ZERO, 0, ss);
    std::vector<int> dofs = sd.interior;
    dofs.insert(dofs.end(), sd.boundary.begin(), sd.boundary.end());
    DBuf<int> d_dofs;
    upload(c, d_dofs, dofs);
    sd.A.alloc((size_t)nloc * nloc, c.stream);
    RDG_CUDA(cudaMemsetAsync(sd.A.p, 0, sizeof(double) * (size_t)nloc * nloc, c.stream));
    set_map_kernel<<<g256(nloc), 256, 0, c.stream>>>(nloc, d_dofs.p, gloc.p, 1);
    local_dense_kernel<<<nloc, 64, 0, c.stream>>>(nloc, d_dofs.p, gloc.p, ss.A.rp.p, ss.A.ci.p, ss.A.v.p, sd.A.p);
    set_map_kernel<<<g256(nloc), 256, 0, c.stream>>>(nloc, d_dofs.p, gloc.p, 0);
    RDG_LAUNCH_CHECK();
    c.launches += 3;
    double* AII = sd.A.p;
    double* AIB = sd.A.p + (size_t)nI * nloc;
    double* ABI = sd.A.p + nI;
    double* ABB = sd.A.p + (size_t)nI * nloc + nI;
    if (nI > 0) {  // A_II = L L' (potrf), X = A_II^-1 A_IB (potrs), A_BB -= A_BI X (dgemm)
      int lw = 0;
      RDG_CUSOLVER(cusolverDnDpotrf_bufferSize(b.sol, CUBLAS_FILL_MODE_LOWER, nI, AII, nloc, &lw));
      DBuf<double> work(std::max(lw, 1), c.stream);
      RDG_CUSOLVER(cusolverDnDpotrf(b.sol, CUBLAS_FILL_MODE_LOWER, nI, AII, nloc, work.p, lw, b.info.p));
      check_info(c, b, ("build_bddc: interior factorization failed in subdomain " + std::to_string(sdx)).c_str());
      if (nB > 0) {
        DBuf<double> X((size_t)nI * nB, c.stream);
        RDG_CUDA(cudaMemcpy2DAsync(X.p, sizeof(double) * nI, AIB, sizeof(double) * nloc, sizeof(double) * nI, nB,
                                   cudaMemcpyDeviceToDevice, c.stream));
        RDG_CUSOLVER(cusolverDnDpotrs(b.sol, CUBLAS_FILL_MODE_LOWER, nI, nB, AII, nloc, X.p, nI, b.info.p));
        RDG_CUBLAS(cublasDgemm(b.blas, CUBLAS_OP_N, CUBLAS_OP_N, nB, nB, nI, &mone, ABI, nloc, X.p, nI, &one, ABB,
                               nloc));
      }
    }
    sd.S.alloc(std::max<size_t>((size_t)nB * nB, 1), c.stream);
    if (nB > 0) {
      symmetrize_kernel<<<g256((int64_t)nB * nB), 256, 0, c.stream>>>(nB, ABB, nloc, sd.S.p);
      RDG_LAUNCH_CHECK();
      ++c.launches;
    }
    const int msz = nB + nc;
    if (msz > 0) {  // saddle [[S, C'], [C, 0]] = LU; Phi = top rows of saddle^-1 [0; I]
      sd.sad.alloc((size_t)msz * msz, c.stream);
      sd.ipiv.alloc(msz, c.stream);
      saddle_kernel<<<g256((int64_t)msz * msz), 256, 0, c.stream>>>(nB, nc, sd.S.p, sd.C.p, sd.sad.p);
      RDG_LAUNCH_CHECK();
      ++c.launches;
      int lw = 0;
      RDG_CUSOLVER(cusolverDnDgetrf_bufferSize(b.sol, msz, msz, sd.sad.p, msz, &lw));
      DBuf<double> work(std::max(lw, 1), c.stream);
      RDG_CUSOLVER(cusolverDnDgetrf(b.sol, msz, msz, sd.sad.p, msz, work.p, sd.ipiv.p, b.info.p));
      check_info(c, b, ("build_bddc: singular saddle system in subdomain " + std::to_string(sdx)).c_str());
      sd.Phi.alloc(std::max<size_t>((size_t)nB * nc, 1), c.stream);
      if (nc > 0) {
        DBuf<double> R((size_t)msz * nc, c.stream);
        unit_rhs_kernel<<<g256((int64_t)msz * nc), 256, 0, c.stream>>>(nB, nc, R.p);
        RDG_LAUNCH_CHECK();
        ++c.launches;
        RDG_CUSOLVER(cusolverDnDgetrs(b.sol, CUBLAS_OP_N, msz, nc, sd.sad.p, msz, sd.ipiv.p, R.p, msz, b.info.p));
        RDG_CUDA(cudaMemcpy2DAsync(sd.Phi.p, sizeof(double) * nB, R.p, sizeof(double) * msz, sizeof(double) * nB, nc,
                                   cudaMemcpyDeviceToDevice, c.stream));
        // coarse += Phi' S Phi on the primal ids (bddc.cpp:290-297), subdomains in order
        DBuf<double> SP((size_t)nB * nc, c.stream), Q((size_t)nc * nc, c.stream);
        RDG_CUBLAS(cublasDgemm(b.blas, CUBLAS_OP_N, CUBLAS_OP_N, nB, nc, nB, &one, sd.S.p, nB, sd.Phi.p, nB, &zero, SP.p,
                               nB));
        RDG_CUBLAS(cublasDgemm(b.blas, CUBLAS_OP_T, CUBLAS_OP_N, nc, nc, nB, &one, sd.Phi.p, nB, SP.p, nB, &zero, Q.p,
                               nc));
        coarse_add_kernel<<<g256((int64_t)nc * nc), 256, 0, c.stream>>>(nc, np, sd.d_pidx.p, Q.p, b.coarse_raw.p);
        RDG_LAUNCH_CHECK();
        ++c.launches;
      }
    }
    RDG_CUDA(cudaStreamSynchronize(c.stream));
  }
  if (np > 0) {  // coarse Cholesky (row-major lower factor, the layout dense_llt_solve reads)
    DCsr Cd;  // dense_llt takes a CSR: build the dense coarse matrix's CSR on the host
    const auto cm = download(c, b.coarse_raw.p, (size_t)np * np);
    std::vector<int> crp(1, 0), cci;
    std::vector<double> cv;
    for (int r = 0; r < np; ++r) {
      for (int k = 0; k < np; ++k)
        if (cm[(size_t)k * np + r] != 0.0) {  // coarse_raw is col-major: (r, k) at k * np + r
          cci.push_back(k);
          cv.push_back(cm[(size_t)k * np + r]);
        }
      crp.push_back((int)cci.size());
    }
    Cd.rows = Cd.cols = np;
    Cd.nnz = (int64_t)cci.size();
    upload(c, Cd.rp, crp);
    upload(c, Cd.ci, cci);
    upload(c, Cd.v, cv);
    DBuf<int> err(1, c.stream);
    RDG_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), c.stream));
    dense_llt(c, Cd, b.coarse, err.p);
    int he = 0;
    RDG_CUDA(cudaMemcpyAsync(&he, err.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    RDG_CUDA(cudaStreamSynchronize(c.stream));
    if (he) throw Error(RD_ENOTSPD, "build_bddc: coarse matrix not positive definite");
  }
  size_t mx = 1;
  for (auto& sd : b.subs) mx = std::max<size_t>(mx, (size_t)std::max(sd.nI, sd.nB + sd.ncon));
  b.w1.alloc(mx, c.stream);
  b.w2.alloc(mx, c.stream);
  b.w3.alloc(mx, c.stream);
  b.rp.alloc(std::max(np, 1), c.stream);
  RDG_CUDA(cudaStreamSynchronize(c.stream));
  return op.release();
}

void bddc_free(Bddc* b) {
  if (!b) return;
  cudaStreamSynchronize(b->c->stream);
  delete b;
}
int bddc_n_interface(const Bddc& b) { return b.nC; }
int bddc_n_primal(const Bddc& b) { return b.n_primal; }
int bddc_n_dofs(const Bddc& b) { return b.n_dofs; }
const std::vector<int>& bddc_interface(const Bddc& b) { return b.interface_dofs; }
std::vector<double> bddc_coarse_matrix(const Bddc& b) {  // row-major np x np (before factorization)
  const int np = b.n_primal;
  const auto cm = download(*b.c, b.coarse_raw.p, (size_t)np * np);
  std::vector<double> out((size_t)np * np);
  for (int r = 0; r < np; ++r)
    for (int k = 0; k < np; ++k) out[(size_t)r * np + k] = cm[(size_t)k * np + r];
  return out;
}

// bddc.cpp:303-324: y = A_CC x - sum_s scatter(A_BI A_II^-1 A_IB x_b), subdomains in order
void bddc_schur_apply(Bddc& b, const double* x, double* y) {
  Ctx& c = *b.c;
  const double one = 1.0, zero = 0.0;
  spmv(c, b.A_CC, x, y);
  for (auto& sd : b.subs) {
    if (!sd.nB || !sd.nI) continue;
    const int nloc = sd.nI + sd.nB;
    gather_kernel<<<g256(sd.nB), 256, 0, c.stream>>>(sd.nB, sd.d_bidx.p, x, b.w1.p);
    RDG_CUBLAS(cublasDgemv(b.blas, CUBLAS_OP_N, sd.nI, sd.nB, &one, sd.A.p + (size_t)sd.nI * nloc, nloc, b.w1.p, 1,
                           &zero, b.w2.p, 1));
    RDG_CUSOLVER(cusolverDnDpotrs(b.sol, CUBLAS_FILL_MODE_LOWER, sd.nI, 1, sd.A.p, nloc, b.w2.p, sd.nI, b.info.p));
    RDG_CUBLAS(cublasDgemv(b.blas, CUBLAS_OP_N, sd.nB, sd.nI, &one, sd.A.p + sd.nI, nloc, b.w2.p, 1, &zero, b.w3.p, 1));
    scatter_add_kernel<<<g256(sd.nB), 256, 0, c.stream>>>(sd.nB, sd.d_bidx.p, nullptr, b.w3.p, -1.0, y);
    RDG_LAUNCH_CHECK();
    c.launches += 2;
  }
}

// bddc.cpp:326-345: g = f_C - sum_s scatter(A_BI A_II^-1 f_I)
void bddc_reduce_rhs(Bddc& b, const double* f, double* g) {
  Ctx& c = *b.c;
  const double one = 1.0, zero = 0.0;
  if (b.nC) {
    gather_kernel<<<g256(b.nC), 256, 0, c.stream>>>(b.nC, b.d_iface.p, f, g);
    RDG_LAUNCH_CHECK();
    ++c.launches;
  }
  for (auto& sd : b.subs) {
    if (!sd.nB || !sd.nI) continue;
    const int nloc = sd.nI + sd.nB;
    gather_kernel<<<g256(sd.nI), 256, 0, c.stream>>>(sd.nI, sd.d_interior.p, f, b.w2.p);
    RDG_CUSOLVER(cusolverDnDpotrs(b.sol, CUBLAS_FILL_MODE_LOWER, sd.nI, 1, sd.A.p, nloc, b.w2.p, sd.nI, b.info.p));
    RDG_CUBLAS(cublasDgemv(b.blas, CUBLAS_OP_N, sd.nB, sd.nI, &one, sd.A.p + sd.nI, nloc, b.w2.p, 1, &zero, b.w3.p, 1));
    scatter_add_kernel<<<g256(sd.nB), 256, 0, c.stream>>>(sd.nB, sd.d_bidx.p, nullptr, b.w3.p, -1.0, g);
    RDG_LAUNCH_CHECK();
    c.launches += 2;
  }
}

// bddc.cpp:347-370: u_C = x; u_I = A_II^-1 (f_I - A_IB u_C) per subdomain
void bddc_expand(Bddc& b, const double* uC, const double* f, double* u) {
  Ctx& c = *b.c;
  const double one = 1.0, zero = 0.0;
  RDG_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * std::max(b.n_dofs, 1), c.stream));
  if (b.nC) {
    scatter_kernel<<<g256(b.nC), 256, 0, c.stream>>>(b.nC, b.d_iface.p, uC, u);
    RDG_LAUNCH_CHECK();
    ++c.launches;
  }
  for (auto& sd : b.subs) {
    if (!sd.nI) continue;
    const int nloc = sd.nI + sd.nB;
    gather_kernel<<<g256(sd.nI), 256, 0, c.stream>>>(sd.nI, sd.d_interior.p, f, b.w2.p);
    if (sd.nB) {
      gather_kernel<<<g256(sd.nB), 256, 0, c.stream>>>(sd.nB, sd.d_bidx.p, uC, b.w1.p);
      RDG_CUBLAS(cublasDgemv(b.blas, CUBLAS_OP_N, sd.nI, sd.nB, &one, sd.A.p + (size_t)sd.nI * nloc, nloc, b.w1.p, 1,
                             &zero, b.w3.p, 1));
      sub_kernel<<<g256(sd.nI), 256, 0, c.stream>>>(sd.nI, b.w2.p, b.w3.p);  // w3 = w2 - w3
      RDG_CUDA(cudaMemcpyAsync(b.w2.p, b.w3.p, sizeof(double) * sd.nI, cudaMemcpyDeviceToDevice, c.stream));
      c.launches += 2;
    }
    RDG_CUSOLVER(cusolverDnDpotrs(b.sol, CUBLAS_FILL_MODE_LOWER, sd.nI, 1, sd.A.p, nloc, b.w2.p, sd.nI, b.info.p));
    scatter_kernel<<<g256(sd.nI), 256, 0, c.stream>>>(sd.nI, sd.d_interior.p, b.w2.p, u);
    RDG_LAUNCH_CHECK();
    c.launches += 2;
  }
}

// bddc.cpp:372-430: scaled local saddle corrections with vanishing primal values, then the coarse
// correction through the constrained basis
void bddc_apply(Bddc& b, const double* r, double* z) {
  Ctx& c = *b.c;
  const double one = 1.0, zero = 0.0;
  RDG_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * std::max(b.nC, 1), c.stream));
  if (b.n_primal) RDG_CUDA(cudaMemsetAsync(b.rp.p, 0, sizeof(double) * b.n_primal, c.stream));
  for (auto& sd : b.subs) {
    if (!sd.nB) continue;
    const int msz = sd.nB + sd.ncon;
    gather_scaled_kernel<<<g256(sd.nB), 256, 0, c.stream>>>(sd.nB, sd.d_bidx.p, sd.scaling.p, r, b.w1.p);  // rb
    RDG_CUDA(cudaMemsetAsync(b.w2.p, 0, sizeof(double) * msz, c.stream));
    RDG_CUDA(cudaMemcpyAsync(b.w2.p, b.w1.p, sizeof(double) * sd.nB, cudaMemcpyDeviceToDevice, c.stream));
    RDG_CUSOLVER(cusolverDnDgetrs(b.sol, CUBLAS_OP_N, msz, 1, sd.sad.p, msz, sd.ipiv.p, b.w2.p, msz, b.info.p));
    scatter_add_kernel<<<g256(sd.nB), 256, 0, c.stream>>>(sd.nB, sd.d_bidx.p, sd.scaling.p, b.w2.p, 1.0, z);
    c.launches += 2;
    if (sd.ncon) {  // r_primal[pidx] += Phi' rb
      RDG_CUBLAS(cublasDgemv(b.blas, CUBLAS_OP_T, sd.nB, sd.ncon, &one, sd.Phi.p, sd.nB, b.w1.p, 1, &zero, b.w3.p, 1));
      scatter_add_kernel<<<g256(sd.ncon), 256, 0, c.stream>>>(sd.ncon, sd.d_pidx.p, nullptr, b.w3.p, 1.0, b.rp.p);
      ++c.launches;
    }
    RDG_LAUNCH_CHECK();
  }
  if (b.n_primal > 0) {
    DBuf<double> lam(b.n_primal, c.stream);
    dense_llt_solve(c, b.n_primal, b.coarse.p, b.rp.p, lam.p);
    for (auto& sd : b.subs) {
      if (!sd.ncon) continue;
      gather_kernel<<<g256(sd.ncon), 256, 0, c.stream>>>(sd.ncon, sd.d_pidx.p, lam.p, b.w1.p);
      RDG_CUBLAS(cublasDgemv(b.blas, CUBLAS_OP_N, sd.nB, sd.ncon, &one, sd.Phi.p, sd.nB, b.w1.p, 1, &zero, b.w3.p, 1));
      scatter_add_kernel<<<g256(sd.nB), 256, 0, c.stream>>>(sd.nB, sd.d_bidx.p, sd.scaling.p, b.w3.p, 1.0, z);
      RDG_LAUNCH_CHECK();
      c.launches += 2;
    }
  }
}

}  // namespace rdg
