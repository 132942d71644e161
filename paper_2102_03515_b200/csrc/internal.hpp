// internal.hpp -- device-side objects behind the opaque C-ABI handles and the
// host-callable entry points shared between translation units.
#pragma once

#include <functional>
#include <memory>

#include "common.cuh"

namespace rdg {

// ---------------------------------------------------------------- CSR on device
// Layout in HBM: row_ptr int32[rows+1], col int32[nnz], val fp64[nnz]
// (Eigen RowMajor<int> storage contract, types.hpp:14).  `lat` records the
// lattice box when the pattern was verified to be a monotone box stencil
// (SURVEY.md Appendix A); the structured smoother keys off it.
struct Lattice {
  int lx = 0, ly = 0, lz = 0;  // box sides; lx*ly*lz == rows
  bool ok = false;
};

struct DCsr {
  int rows = 0, cols = 0;
  int64_t nnz = 0;
  DBuf<int> rp, ci;
  DBuf<double> v;
  Lattice lat;
  bool lat_checked = false;  // detect_lattice ran on the current pattern
  // generic (sync-free) Gauss-Seidel readiness flags, epoch-stamped so they
  // never need clearing between sweeps
  mutable DBuf<unsigned> gs_flags;
  mutable unsigned gs_epoch = 0;
  // structured smoother: step-major packed values (fwd, bwd) and tagged halo
  // cells {value, sweep tag} (2 words per row), built by lattice_prepare
  mutable DBuf<double> lat_pack[2];
  mutable DBuf<unsigned long long> lat_xh;
  mutable unsigned lat_epoch = 0;
  // uniform stencil: every row equals the box-centre row slot by slot (absent slots
  // aside) -- then the smoother keeps the row in registers and streams no values.
  // class-uniform stencil: every row equals its position class's row (64 classes,
  // pos_class of each coordinate) -- the smoother reads rows from an 8 KB table.
  // state: -1 not prepared, -2 checks pending on the device, 0 packed, 1 uniform, 2 class
  mutable DBuf<double> lat_uni;     // 15 slot values + the diagonal's division reciprocal
  mutable DBuf<int> lat_uni_flag;   // device: [0] 1 = some row differs from the centre row,
                                    //         [1] 1 = some row differs from its class row
  mutable DBuf<double> lat_cls;     // [64][16] class rows (slot order, absent +0, reciprocal in 15)
  mutable DBuf<int> lat_order;      // ticket -> tile, wavefront order (levels with more tiles than SMs)
  mutable int lat_uni_state = -1;
};

// ---------------------------------------------------------------- scan
// Exclusive prefix sum of n int32 counts into int32 offsets[n+1]; returns the
// total (throws RD_EINVAL if it exceeds INT32_MAX, the reference's index type).
// `also_dev` (optional): one more device int read back with the same sync.
int64_t exclusive_scan(Ctx& c, const int* counts, int* offsets, int64_t n, const int* also_dev = nullptr,
                       int* also_host = nullptr);

// ---------------------------------------------------------------- linalg.cu
void spmv(Ctx& c, const DCsr& A, const double* x, double* y);
// y = A x and *dot_out = p . y (deterministic), both on device
void spmv_dot(Ctx& c, const DCsr& A, const double* x, double* y, double* dot_out);
// res = r - A z
void residual(Ctx& c, const DCsr& A, const double* r, const double* z, double* res);
// z += P zc
void prolong_add(Ctx& c, const DCsr& P, const double* zc, double* z);
void dot(Ctx& c, int64_t n, const double* a, const double* b, double* out_dev);
// jacobi_precond (linalg.cpp:57-62): d = diag(A) (0 where absent), *bad_dev = 1 if some d_i <= 0
void csr_diagonal(Ctx& c, const DCsr& A, double* d, int* bad_dev);
void jacobi_apply(Ctx& c, int64_t n, const double* d, const double* r, double* z);  // z = r ./ d
DCsr transpose(Ctx& c, const DCsr& A);
DCsr spgemm(Ctx& c, const DCsr& A, const DCsr& B);  // Eigen conservative product order
DCsr prune_zeros(Ctx& c, const DCsr& A);
DCsr csr_copy(Ctx& c, const DCsr& A);
DCsr csr_view(const DCsr& A);  // non-owning view of A's arrays (lattice facts carried over)
bool pattern_symmetric(Ctx& c, const DCsr& A);
// detect a monotone (15-point Kuhn or sub-) stencil on a box; fills A.lat
void detect_lattice(Ctx& c, DCsr& A);

// ---------------------------------------------------------------- smoother.cu
// one forward (fwd=true) or backward Gauss-Seidel pass: xout from xin (xin may be
// nullptr = zero vector).  Optionally accumulates dot(r, xout) into dot_out.
void gs_pass(Ctx& c, const DCsr& A, const double* f, const double* xin, double* xout, bool fwd,
             double* dot_out = nullptr, const double* dot_with = nullptr);
// setup-time layout for the structured smoother (no-op unless A.lat.ok); with
// err_dev the layout check is left on the device (1 mismatch, 2 zero diagonal)
void lattice_prepare(Ctx& c, const DCsr& A, int* err_dev = nullptr);
// after lattice_prepare: flags_host = the host copy of lat_uni_flag[0..1] (null: read it here);
// builds the packed layout for a non-uniform level when build_packs
void lattice_resolve(Ctx& c, const DCsr& A, const int* flags_host = nullptr, bool build_packs = true);

// distributed z-slab smoother (dist.cu): one rank's planes [zlo, zhi) of a lattice
// level; local vectors hold planes [g0, g1) (the slab plus one ghost plane per side)
struct SlabSmoother {
  int L = 0, zlo = 0, zhi = 0, g0 = 0, g1 = 0, ntz = 0;
  DBuf<double> pack[2];            // fwd, bwd step-major packed stencil of the slab's tiles
  DBuf<double> uni;                // or the stencil on chip (then no packs): the uniform row
  int vm = 0;                      // (vm 1) or the 64 class rows (vm 2); 0 packed
  // tagged cells {value, tag} of planes [g0, g1): plain cudaMalloc, so a peer
  // process can map them (cudaIpcGetMemHandle) for the pipelined hand-off
  unsigned long long* cells = nullptr;
  size_t cells_bytes = 0;
  // the neighbours' cells as virtual global pointers: [0] next slab (downstream of a
  // forward sweep), [1] previous slab (downstream of a backward sweep); null: none
  unsigned long long* peer_v[2] = {nullptr, nullptr};
  void* peer_ipc[2] = {nullptr, nullptr};  // IPC mappings to close
  unsigned epoch = 0;
  int device = 0;
  SlabSmoother() = default;
  SlabSmoother(const SlabSmoother&) = delete;
  SlabSmoother& operator=(const SlabSmoother&) = delete;
  ~SlabSmoother();
};
// A: the level's whole-box matrix (verified lattice)
void slab_prepare(Ctx& c, const DCsr& A, int zlo, int zhi, SlabSmoother& s);
// in_plane: the upstream ghost plane's values (L*L; null = zeros), fresh (exact) or old (block).
// pipelined: no in_plane; the upstream neighbour's kernel writes the cells (peer_v), and
// this sweep writes its downstream boundary plane into the downstream neighbour's.
void gs_pass_slab(Ctx& c, SlabSmoother& s, const double* f, const double* xin, double* xout, bool fwd,
                  const double* in_plane, bool pipelined = false);
// all slabs of a distributed level (linked neighbours, one device) in one cooperative
// launch on c's stream: the single-GPU emulation of the pipelined hand-off
void gs_pass_slabs_multi(Ctx& c, int n, Ctx* const* cs, SlabSmoother* const* s, const double* const* f,
                         const double* const* xin, double* const* xout, bool fwd);

// ---------------------------------------------------------------- amg.cu
struct Level {
  DCsr A, P, Pt;
  DBuf<uint8_t> flags;
  bool has_p = false;
  // work vectors
  DBuf<double> r, z, t, res;
  DBuf<double> tail_table;  // coarse_tail.cu: the 64 position-class rows of a small lattice level
};

constexpr int kTailMaxLevels = 6;
struct Hierarchy {
  std::vector<Level> levels;
  int smoothing_steps = 1;
  int nc = 0;              // coarsest dimension
  DBuf<double> Lc;         // coarsest LLT factor (row-major, lower)
  bool tail_checked = false;
  int tail_level = -1;     // first level of the one-CTA coarse tail (-1: none)
};

// coarse_tail.cu: the V-cycle from level c0 down and back up in one thread block
void coarse_tail_prepare(Ctx& c, Hierarchy& h, int* bad_dev);  // setup (device-side check)
int coarse_tail_level(Ctx& c, Hierarchy& h);
void coarse_tail(Ctx& c, Hierarchy& h, int c0, const double* r, double* z);

std::vector<uint8_t> coarsen(Ctx& c, const DCsr& A, DBuf<uint8_t>& flags_dev, DCsr& P);
DCsr galerkin(Ctx& c, const DCsr& A, const DCsr& P, const DCsr& Pt);
// borrow: level 0 views A's arrays (A must outlive the hierarchy and stay unchanged)
void build_hierarchy(Ctx& c, const DCsr& A, int threshold, int m, Hierarchy& h, bool borrow = false);
// z = V(r) on device; if dot_out, also writes r.z (deterministic)
// l0 > 0: the V-cycle of the sub-hierarchy from level l0 (r, z of level l0's size)
void vcycle(Ctx& c, Hierarchy& h, const double* r, double* z, double* dot_out, int l0 = 0);
// throws RD_ENOTSPD, or (err_dev) leaves the failure flag on the device
void dense_llt(Ctx& c, const DCsr& A, DBuf<double>& L, int* err_dev = nullptr);
// x = L^-T L^-1 b with the dense factor of dense_llt (llt_solve_kernel's order), device vectors
void dense_llt_solve(Ctx& c, int n, const double* L, const double* b, double* x);

// ---------------------------------------------------------------- pcg.cu
struct PcgResultDev {
  int iterations = 0;
  bool converged = false;
};
// An operator of the PCG loop: out = op(in) and *dot_out = in . out (device pointers, stream-ordered).
using PcgOp = std::function<void(const double* in, double* out, double* dot_out)>;
// linalg.cpp:64-102 over any pair of operators (rd_gpu_pcg_linop)
PcgResultDev pcg_ops(Ctx& c, int64_t n, const PcgOp& apply_A, const PcgOp& apply_P, const double* f, double tol,
                     int max_iter, double* x, double* hist_dev);
// x (device, n) receives the solution; hist_dev (device, >= max_iter) may be null.
PcgResultDev pcg_device(Ctx& c, const DCsr& A, Hierarchy* h, const double* f, double tol, int max_iter, double* x,
                        double* hist_dev);

// ---------------------------------------------------------------- assembly.cu
struct DMesh {
  int nv = 0, nt = 0, lattice_n = -1;
  // set while the tets upload on another stream (rd_gpu_solve_host_mesh): the generic
  // assembly path waits on it before reading tets; the lattice path reads none
  cudaEvent_t tets_ready = nullptr;
  DBuf<double> xyz;
  DBuf<int> tets;
  DBuf<uint8_t> boundary;
  // bisection state (mesh.hpp:17-20): refinement edge (0, tag) and generation per tet; empty
  // for build_structured_cube / uploaded meshes, which carry tag 3 and generation 0
  DBuf<uint8_t> tag;
  DBuf<int> gen;
};

struct DSystem {
  double rho = 1.0;
  DCsr K, M, A;
  DBuf<double> f;
  DBuf<int> v2d, d2v;
  int n_dofs = 0;
  int nv = 0;
};

void build_structured_cube(Ctx& c, int n, DMesh& m);
// sets m.lattice_n when the tets are exactly the build_structured_cube enumeration
void detect_cube_lattice(Ctx& c, DMesh& m);
// n when (nv, nt) are the sizes of build_structured_cube(n), else -1 (no check of the tets)
int cube_lattice_candidate(int nv, int nt);
// bad[0] = 1 unless tets[0, nt) is the Kuhn enumeration of build_structured_cube(n); on stream st
void launch_lattice_tets_check(Ctx& c, cudaStream_t st, int n, const int* tets, int nt, int* bad);
void launch_cube_vertices(Ctx& c, cudaStream_t st, int n, double* xyz, uint8_t* bnd);
void launch_verts_equal(Ctx& c, cudaStream_t st, int64_t nv, const double* a, const double* b, const uint8_t* fa,
                        const uint8_t* fb, int* bad);
// a_only: the caller needs A and f only (rd_gpu_solve_host_mesh returns u); on the lattice path
// K and M are then not written (left empty), two thirds of the system's bytes
void build_system(Ctx& c, const DMesh& m, double rho, int target_kind, uint64_t seed, DSystem& s,
                  bool a_only = false);
// l2 / h1-semi error of the P1 field `coeffs` (device, n_dofs) vs the manufactured exact solution
void error_norms(Ctx& c, const DMesh& m, const DSystem& s, const double* coeffs, double rho, double* l2, double* h1);
// l2 / h1-semi error of `coeffs` vs a target field u_bar (value and exact gradient)
void error_norms_target(Ctx& c, const DMesh& m, const DSystem& s, const double* coeffs, int kind, uint64_t seed,
                        double* l2, double* h1);
// assembly.cpp:312-331: squared L2 distance of the P1 field to the target (the target's rule)
double l2_error_target_squared(Ctx& c, const DMesh& m, const DSystem& s, const double* coeffs, int kind,
                               uint64_t seed);
// adapt.cu -- adapt.cpp:126-150 (marked: device, >= n ints; *count on the host) and
// mesh.cpp:67-145 (out: a new mesh; marked: device ids)
void mark_dorfler(Ctx& c, int n, const double* eta, double theta, int* marked, int* count);
void bisect_marked(Ctx& c, const DMesh& in, const int* marked, int n_marked, DMesh& out);
// bddc.cu -- bddc.cpp:45-456 (setup on the host's index lists, numerics on the device)
struct Bddc;
void partition_geometric(Ctx& c, const DMesh& m, const DSystem& s, int p, std::vector<int>& owner,
                         std::vector<std::vector<int>>& dof_subdomains);
Bddc* build_bddc(Ctx& c, const DMesh& m, const DSystem& sys, int p);  // free with bddc_free
void bddc_free(Bddc* b);
int bddc_n_interface(const Bddc& b);
int bddc_n_primal(const Bddc& b);
int bddc_n_dofs(const Bddc& b);
const std::vector<int>& bddc_interface(const Bddc& b);
std::vector<double> bddc_coarse_matrix(const Bddc& b);
// device vectors, stream-ordered on the Bddc's context
void bddc_schur_apply(Bddc& b, const double* x, double* y);            // n_interface -> n_interface
void bddc_reduce_rhs(Bddc& b, const double* f, double* g);             // n_dofs -> n_interface
void bddc_expand(Bddc& b, const double* uC, const double* f, double* u);  // -> n_dofs
void bddc_apply(Bddc& b, const double* r, double* z);                  // n_interface -> n_interface
// adapt.cpp:35-124: per_tet (device, n_tets) = eta_tau, optional eta_tau^2 copy, global = sqrt(sum eta^2)
void estimate(Ctx& c, const DMesh& m, const DSystem& s, const double* coeffs, int kind, double* per_tet,
              double* eta_sq_out, double* global);

}  // namespace rdg

// opaque handles
struct rd_ctx {
  rdg::Ctx c;
};
struct rd_csr {
  rd_ctx* ctx = nullptr;
  std::unique_ptr<rdg::DCsr> owned;  // null for borrowed views
  rdg::DCsr* a = nullptr;
};
struct rd_mesh {
  rd_ctx* ctx = nullptr;
  rdg::DMesh m;
};
struct rd_system {
  rd_ctx* ctx = nullptr;
  rdg::DSystem s;
  rd_csr views[3];
};
struct rd_amg {
  rd_ctx* ctx = nullptr;
  rdg::Hierarchy h;
  std::vector<rd_csr> views;  // 3 per level
};
