// dist.cu -- per-rank pieces of the distributed (z-slab) AMG-PCG solve, SURVEY.md §8(e).
//
// The lattice of every distributed level is cut into z-slabs (contiguous row
// ranges: z is the slowest lattice index, so a slab plus one ghost plane per
// side is one contiguous range of the global numbering).  Each rank keeps
//   * row blocks of A_l, P_l, Pt_l with columns renumbered into its local
//     (slab + ghost planes) vector: the same row sums in the same order as the
//     whole-box SpMV, so residuals, restrictions and prolongations are the
//     single-GPU ones bit for bit;
//   * a slab smoother (smoother_lattice.cu) whose upstream ghost plane enters as
//     tagged cells: fresh neighbour values reproduce the single-GPU sweep
//     exactly (the ranks hand the wavefront on), old ones give the concurrent
//     block variant;
//   * the PCG vector updates with host scalars (the dots are reduced across
//     ranks by the caller, paper_2102_03515_b200/dist.py, over NCCL).
// The coarse levels below the gather threshold stay whole on rank 0 and run
// through rd_gpu_amg_apply_from.  Halo exchange and reductions are the
// caller's (torch.distributed / NCCL over NVLink); nothing here communicates.
#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.hpp"

using namespace rdg;

namespace {

__global__ void rowblock_kernel(int rows, const int* __restrict__ rp, const int* __restrict__ ci,
                                const double* __restrict__ v, int r0, int c0, int c1, int* __restrict__ orp,
                                int* __restrict__ oci, double* __restrict__ ov, int* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > rows) return;
  const int base = rp[r0];
  orp[i] = rp[r0 + i] - base;
  if (i == rows) return;
  for (int k = rp[r0 + i]; k < rp[r0 + i + 1]; ++k) {
    const int c = ci[k];
    if (c < c0 || c >= c1) atomicExch(err, 1);
    oci[k - base] = c - c0;
    ov[k - base] = v[k];
  }
}

// x += alpha p, r -= alpha Ap (linalg.cpp:84-85: Eigen's x += alpha*p, no FMA)
__global__ void dist_xr_kernel(int64_t n, double alpha, const double* __restrict__ p, const double* __restrict__ Ap,
                               double* __restrict__ x, double* __restrict__ r) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    r[i] = __dsub_rn(r[i], __dmul_rn(alpha, Ap[i]));
  }
}

// p = z + beta p (linalg.cpp:99)
__global__ void dist_p_kernel(int64_t n, double beta, const double* __restrict__ z, double* __restrict__ p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

// ---- device-resident distributed PCG scalars (rd_pcg_state): rank-ordered sums of the
// all-gathered partials, so every rank computes the same bits
__device__ __forceinline__ double rank_sum(int world, const double* __restrict__ parts) {
  double s = 0.0;
  for (int k = 0; k < world; ++k) s = __dadd_rn(s, parts[k]);
  return s;
}
__global__ void dpcg_begin_kernel(int world, const double* parts, rd_pcg_state* st) {
  const double rz = rank_sum(world, parts);
  st->rz = rz;
  st->rz0 = rz;
  st->done = 0;
  st->status = 0;
  st->iterations = 0;
  if (rz < 0.0) st->status = 2;  // linalg.cpp:71
  else if (rz == 0.0) st->done = 1;  // linalg.cpp:73-76
}
__global__ void dpcg_alpha_kernel(int world, const double* parts, rd_pcg_state* st) {
  if (st->done || st->status) return;
  const double pAp = rank_sum(world, parts);
  st->pap = pAp;
  if (!(pAp > 0.0)) {  // linalg.cpp:80-82
    st->status = 1;
    return;
  }
  st->alpha = __ddiv_rn(st->rz, pAp);
}
__global__ void dpcg_xr_kernel(int64_t n, const rd_pcg_state* st, const double* __restrict__ p,
                               const double* __restrict__ Ap, double* __restrict__ x, double* __restrict__ r) {
  if (st->done || st->status) return;
  const double alpha = st->alpha;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    r[i] = __dsub_rn(r[i], __dmul_rn(alpha, Ap[i]));
  }
}
__global__ void dpcg_check_kernel(int world, const double* parts, rd_pcg_state* st, double tol, double* hist,
                                  int cap) {
  if (st->done || st->status) return;
  const double rzn = rank_sum(world, parts);
  st->rz_next = rzn;
  if (rzn < 0.0) {  // linalg.cpp:87-89
    st->status = 2;
    return;
  }
  const double rel = __dsqrt_rn(__ddiv_rn(rzn, st->rz0));
  const int it = st->iterations + 1;
  st->iterations = it;
  st->rel = rel;
  if (hist && it - 1 < cap) hist[it - 1] = rel;
  if (rel <= tol) {
    st->done = 1;
    return;
  }
  st->beta = __ddiv_rn(rzn, st->rz);
  st->rz = rzn;
}
__global__ void dpcg_p_kernel(int64_t n, const rd_pcg_state* st, const double* __restrict__ z,
                              double* __restrict__ p) {
  if (st->done || st->status) return;
  const double beta = st->beta;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

int vgrid(Ctx& c, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c.num_sms * 8, (n + 255) / 256));
}

template <class F>
int guard(rd_ctx* ctx, F&& fn) {
  try {
    PoolScope ps(ctx->c.pool);
    fn();
    return RD_OK;
  } catch (const Error& e) {
    ctx->c.err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    ctx->c.err = e.what();
    return RD_ERUNTIME;
  }
}

void require(bool ok, const char* msg) {
  if (!ok) throw Error(RD_EINVAL, msg);
}

}  // namespace

struct rd_slab {
  rd_ctx* ctx = nullptr;
  SlabSmoother s;
};

extern "C" {

int rd_gpu_csr_rowblock(rd_ctx* ctx, const rd_csr* a, int row0, int row1, int col0, int col1, rd_csr** out) {
  return guard(ctx, [&] {
    const DCsr& A = *a->a;
    require(0 <= row0 && row0 <= row1 && row1 <= A.rows && 0 <= col0 && col0 <= col1 && col1 <= A.cols,
            "csr_rowblock: range outside the matrix");
    Ctx& c = ctx->c;
    int nnz2[2];
    RDG_CUDA(cudaMemcpyAsync(&nnz2[0], A.rp.p + row0, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    RDG_CUDA(cudaMemcpyAsync(&nnz2[1], A.rp.p + row1, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    RDG_CUDA(cudaStreamSynchronize(c.stream));
    auto h = std::make_unique<rd_csr>();
    h->ctx = ctx;
    h->owned = std::make_unique<DCsr>();
    DCsr& B = *h->owned;
    B.rows = row1 - row0;
    B.cols = col1 - col0;
    B.nnz = nnz2[1] - nnz2[0];
    B.rp.alloc(B.rows + 1, c.stream);
    B.ci.alloc(B.nnz, c.stream);
    B.v.alloc(B.nnz, c.stream);
    B.lat_checked = true;  // a row block is never a whole-box stencil
    DBuf<int> err(1, c.stream);
    RDG_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), c.stream));
    rowblock_kernel<<<div_up(B.rows + 1, 256), 256, 0, c.stream>>>(B.rows, A.rp.p, A.ci.p, A.v.p, row0, col0, col1,
                                                                  B.rp.p, B.ci.p, B.v.p, err.p);
    RDG_LAUNCH_CHECK();
    ++c.launches;
    int e = 0;
    RDG_CUDA(cudaMemcpyAsync(&e, err.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    RDG_CUDA(cudaStreamSynchronize(c.stream));
    if (e) throw Error(RD_EINVAL, "csr_rowblock: a column lies outside [col0, col1)");
    h->a = h->owned.get();
    *out = h.release();
  });
}

int rd_gpu_residual(rd_ctx* ctx, const rd_csr* a, const double* r, const double* z, double* res) {
  return guard(ctx, [&] { residual(ctx->c, *a->a, r, z, res); });
}

int rd_gpu_prolong_add(rd_ctx* ctx, const rd_csr* p, const double* zc, double* z) {
  return guard(ctx, [&] { prolong_add(ctx->c, *p->a, zc, z); });
}

int rd_gpu_dot_async(rd_ctx* ctx, int n, const double* a, const double* b, double* out_dev) {
  return guard(ctx, [&] { dot(ctx->c, n, a, b, out_dev); });
}

int rd_gpu_pcg_update_xr(rd_ctx* ctx, int64_t n, double alpha, const double* p, const double* ap, double* x,
                         double* r) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (n == 0) return;
    dist_xr_kernel<<<vgrid(c, n), 256, 0, c.stream>>>(n, alpha, p, ap, x, r);
    RDG_LAUNCH_CHECK();
    ++c.launches;
  });
}

int rd_gpu_pcg_update_p(rd_ctx* ctx, int64_t n, double beta, const double* z, double* p) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (n == 0) return;
    dist_p_kernel<<<vgrid(c, n), 256, 0, c.stream>>>(n, beta, z, p);
    RDG_LAUNCH_CHECK();
    ++c.launches;
  });
}

int rd_gpu_pcg_dist_begin(rd_ctx* ctx, int world, const double* parts, rd_pcg_state* st) {
  return guard(ctx, [&] {
    require(world >= 1 && parts && st, "pcg_dist_begin: bad argument");
    dpcg_begin_kernel<<<1, 1, 0, ctx->c.stream>>>(world, parts, st);
    RDG_LAUNCH_CHECK();
    ++ctx->c.launches;
  });
}
int rd_gpu_pcg_dist_alpha(rd_ctx* ctx, int world, const double* parts, rd_pcg_state* st) {
  return guard(ctx, [&] {
    require(world >= 1 && parts && st, "pcg_dist_alpha: bad argument");
    dpcg_alpha_kernel<<<1, 1, 0, ctx->c.stream>>>(world, parts, st);
    RDG_LAUNCH_CHECK();
    ++ctx->c.launches;
  });
}
int rd_gpu_pcg_dist_xr(rd_ctx* ctx, int64_t n, const rd_pcg_state* st, const double* p, const double* ap, double* x,
                       double* r) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (n == 0) return;
    dpcg_xr_kernel<<<vgrid(c, n), 256, 0, c.stream>>>(n, st, p, ap, x, r);
    RDG_LAUNCH_CHECK();
    ++c.launches;
  });
}
int rd_gpu_pcg_dist_check(rd_ctx* ctx, int world, const double* parts, rd_pcg_state* st, double tol, double* hist,
                          int cap) {
  return guard(ctx, [&] {
    require(world >= 1 && parts && st, "pcg_dist_check: bad argument");
    dpcg_check_kernel<<<1, 1, 0, ctx->c.stream>>>(world, parts, st, tol, hist, cap);
    RDG_LAUNCH_CHECK();
    ++ctx->c.launches;
  });
}
int rd_gpu_pcg_dist_p(rd_ctx* ctx, int64_t n, const rd_pcg_state* st, const double* z, double* p) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (n == 0) return;
    dpcg_p_kernel<<<vgrid(c, n), 256, 0, c.stream>>>(n, st, z, p);
    RDG_LAUNCH_CHECK();
    ++c.launches;
  });
}

int rd_gpu_ctx_set_exact_sweeps(rd_ctx* ctx, int exact) {
  return guard(ctx, [&] { ctx->c.gs_exact = exact != 0; });
}

int rd_gpu_amg_apply_from(rd_amg* h, int level, const double* r, double* z) {
  return guard(h->ctx, [&] {
    require(level >= 0 && level < (int)h->h.levels.size(), "amg_apply_from: bad level");
    vcycle(h->ctx->c, h->h, r, z, nullptr, level);
  });
}

int rd_gpu_slab_create(rd_ctx* ctx, const rd_csr* a, int zlo, int zhi, rd_slab** out) {
  return guard(ctx, [&] {
    auto s = std::make_unique<rd_slab>();
    s->ctx = ctx;
    DCsr& A = *a->a;
    if (!A.lat_checked) detect_lattice(ctx->c, A);
    slab_prepare(ctx->c, A, zlo, zhi, s->s);
    *out = s.release();
  });
}

void rd_gpu_slab_free(rd_slab* s) { delete s; }

int rd_gpu_slab_info(const rd_slab* s, int* L, int* g0, int* g1) {
  if (L) *L = s->s.L;
  if (g0) *g0 = s->s.g0;
  if (g1) *g1 = s->s.g1;
  return RD_OK;
}

int rd_gpu_slab_sweep(rd_slab* s, int forward, const double* f, const double* xin, double* xout,
                      const double* in_plane) {
  return guard(s->ctx, [&] { gs_pass_slab(s->ctx->c, s->s, f, xin, xout, forward != 0, in_plane); });
}

namespace {
unsigned long long* virt(void* base, int g0, int L) {
  return reinterpret_cast<unsigned long long*>(base) - 2ll * g0 * (long long)L * L;
}
}  // namespace

int rd_gpu_slab_link(rd_slab* s, const rd_slab* next, const rd_slab* prev) {
  return guard(s->ctx, [&] {
    for (const rd_slab* o : {next, prev})
      require(!o || (o->s.L == s->s.L && o->s.device == s->s.device), "slab_link: neighbour of another level/device");
    require(!next || next->s.zlo == s->s.zhi, "slab_link: next slab must start at this slab's end");
    require(!prev || prev->s.zhi == s->s.zlo, "slab_link: previous slab must end at this slab's start");
    s->s.peer_v[0] = next ? virt(next->s.cells, next->s.g0, s->s.L) : nullptr;
    s->s.peer_v[1] = prev ? virt(prev->s.cells, prev->s.g0, s->s.L) : nullptr;
  });
}

int rd_gpu_slab_ipc_handle(rd_slab* s, void* handle) {
  return guard(s->ctx, [&] {
    require(handle != nullptr, "slab_ipc_handle: null output");
    cudaIpcMemHandle_t h;
    RDG_CUDA(cudaIpcGetMemHandle(&h, s->s.cells));
    static_assert(sizeof(h) == RD_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(handle, &h, sizeof(h));
  });
}

int rd_gpu_slab_open_peer(rd_slab* s, int which, const void* handle, int peer_g0) {
  return guard(s->ctx, [&] {
    require(which == 0 || which == 1, "slab_open_peer: which is 0 (next) or 1 (previous)");
    require(handle != nullptr, "slab_open_peer: null handle");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* q = nullptr;
    RDG_CUDA(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
    if (s->s.peer_ipc[which]) cudaIpcCloseMemHandle(s->s.peer_ipc[which]);
    s->s.peer_ipc[which] = q;
    s->s.peer_v[which] = virt(q, peer_g0, s->s.L);
  });
}

int rd_gpu_slab_sweep_pipelined(rd_slab* s, int forward, const double* f, const double* xin, double* xout) {
  return guard(s->ctx, [&] { gs_pass_slab(s->ctx->c, s->s, f, xin, xout, forward != 0, nullptr, true); });
}

int rd_gpu_slab_sweep_multi(int n, rd_slab* const* s, int forward, const double* const* f,
                            const double* const* xin, double* const* xout) {
  if (n < 1 || !s || !s[0]) return RD_EINVAL;
  return guard(s[0]->ctx, [&] {
    std::vector<Ctx*> cs(n);
    std::vector<SlabSmoother*> ss(n);
    for (int q = 0; q < n; ++q) {
      require(s[q] && s[q]->s.device == s[0]->s.device, "slab_sweep_multi: slabs of one device");
      cs[q] = &s[q]->ctx->c;
      ss[q] = &s[q]->s;
    }
    gs_pass_slabs_multi(s[0]->ctx->c, n, cs.data(), ss.data(), f, xin, xout, forward != 0);
  });
}

}  // extern "C"
