/*
 * rd_gpu.h -- C-ABI of the B200-native AMG-PCG solve path (arXiv 2102.03515).
 *
 * This is the drop-in boundary.  Each entry point replaces one function of
 * the reference C++ library rdsolve; the replaced interface is cited as
 * file:line relative to /root/reference/proj.  Plain pointers and sizes
 * only: no torch, no Eigen, no C++ types.  INTEGRATION.md shows the thin
 * rd:: C++ layer a maintainer adds on the reference side.
 *
 * Vectors (double*) may be HOST or DEVICE pointers; the library inspects
 * them (cudaPointerGetAttributes).  Calls that take host pointers are
 * synchronous; calls on device pointers are stream-ordered on the context's
 * stream, and device-detected errors (zero diagonal, loss of positive
 * definiteness) are returned by the call itself when it must synchronise
 * anyway (pcg, solve_system) or by the next rd_gpu_synchronize().
 *
 * Status codes map one-to-one onto the reference's exceptions
 * (SURVEY.md §8(b)); a thin C++ layer rethrows them.
 */
#ifndef RD_GPU_H
#define RD_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status */
#define RD_OK 0
#define RD_EINVAL 1       /* std::invalid_argument (dimension / parameter errors)        */
#define RD_ERUNTIME 2     /* std::runtime_error (generic)                                */
#define RD_ENOTSPD 3      /* runtime_error: pcg "operator/preconditioner not positive
                             definite", build_amg "coarsest level not positive definite",
                             dense_cholesky_solve "matrix not positive definite"          */
#define RD_EZERODIAG 4    /* runtime_error: "sgs_sweep: zero diagonal" (amg.cpp:82)       */
#define RD_ECUDA 5        /* CUDA runtime failure                                         */
#define RD_ENCCL 6        /* NCCL failure (multi-GPU)                                     */
#define RD_EDEGENERATE 7  /* runtime_error: "assembly: degenerate tet" (assembly.cpp:46)  */

typedef struct rd_ctx rd_ctx;
typedef struct rd_mesh rd_mesh;
typedef struct rd_csr rd_csr;
typedef struct rd_system rd_system;
typedef struct rd_amg rd_amg;

/* ------------------------------------------------------------ context */
/* One device, one stream (NULL: the library creates a non-blocking stream). */
int rd_gpu_ctx_create(int device, void* cuda_stream, rd_ctx** out);
void rd_gpu_ctx_destroy(rd_ctx* ctx);
const char* rd_gpu_last_error(const rd_ctx* ctx);
void* rd_gpu_ctx_stream(rd_ctx* ctx);
/* Waits for the stream; returns the first device-detected error, if any. */
int rd_gpu_synchronize(rd_ctx* ctx);
/* Number of rd_gpu kernels launched on this context so far. */
int64_t rd_gpu_launch_count(const rd_ctx* ctx);
/* Bytes of the library's stream-ordered pool on the context's device: in use by live objects
 * (*used) and held from the driver (*reserved).  One pool per device and process: with one
 * process per GPU this is the rank's device footprint (the smoother's peer-mappable cell
 * buffers, plain allocations, are not counted).  No reference counterpart. */
int rd_gpu_pool_bytes(rd_ctx* ctx, uint64_t* used, uint64_t* reserved);
const char* rd_gpu_version(void);
/* cudaMemcpyDefault between any host/device buffers, ordered on the ctx stream, synchronous */
int rd_gpu_copy(rd_ctx* ctx, void* dst, const void* src, size_t bytes);

/* ------------------------------------------------------------ mesh */
/* replaces rd::build_structured_cube(int n)            mesh.hpp:36, mesh.cpp:29-65 */
int rd_gpu_build_structured_cube(rd_ctx* ctx, int n, rd_mesh** out);
/* uploads a host rd::TetMesh (vertices AoS xyz, tets int[4], boundary flags)  mesh.hpp:13-24 */
int rd_gpu_mesh_create(rd_ctx* ctx, int n_vertices, const double* xyz, int n_tets,
                       const int32_t* tets, const uint8_t* boundary, rd_mesh** out);
void rd_gpu_mesh_free(rd_mesh* mesh);
/* lattice_n = n for build_structured_cube meshes, -1 otherwise */
int rd_gpu_mesh_info(const rd_mesh* mesh, int* n_vertices, int* n_tets, int* lattice_n);
int rd_gpu_mesh_download(const rd_mesh* mesh, double* xyz, int32_t* tets, uint8_t* boundary);

/* ------------------------------------------------------------ assembly */
/* TargetField (target.hpp:12-16).  kinds 0-2 are the reference's targets
 * (target.cpp:17-43); 3 (ball) and 4 (sine + 0.1 * seeded random P1 field)
 * are the BASELINE.json config targets; 5-7 are the reference tests'
 * zero / one / x*y+2z loads (test_assembly.cpp:37,102-154).               */
enum {
  RD_TARGET_SMOOTH = 0,
  RD_TARGET_BOX = 1,
  RD_TARGET_NONZERO_BC = 2,
  RD_TARGET_BALL = 3,
  RD_TARGET_SINE_RANDOM = 4,
  RD_TARGET_ZERO = 5,
  RD_TARGET_ONE = 6,
  RD_TARGET_QUADRATIC = 7
};
typedef struct {
  int kind;
  uint64_t seed; /* splitmix64 seed for RD_TARGET_SINE_RANDOM (tests/oracles.hpp:97-108) */
} rd_target;

/* replaces rd::build_system(mesh, rho, target)   assembly.hpp:48, assembly.cpp:225-238
 * K (pruned), M (pruned), A = rho*K + M (not pruned), load f -- all on device. */
int rd_gpu_build_system(rd_ctx* ctx, const rd_mesh* mesh, double rho, const rd_target* target,
                        rd_system** out);
void rd_gpu_system_free(rd_system* sys);
int rd_gpu_system_n_dofs(const rd_system* sys);
/* which: 0 = K, 1 = M, 2 = A.  Borrowed; lives as long as sys. */
const rd_csr* rd_gpu_system_matrix(const rd_system* sys, int which);
/* device pointer to the load vector f (n_dofs doubles); borrowed */
const double* rd_gpu_system_load(const rd_system* sys);
/* DofMap (assembly.hpp:15-22); either pointer may be NULL */
int rd_gpu_system_dofmap(const rd_system* sys, int32_t* vertex_to_dof, int32_t* dof_to_vertex);

/* ------------------------------------------------------------ CSR */
/* SpMat = Eigen::SparseMatrix<double, RowMajor, int> (types.hpp:14): row_ptr
 * int32[rows+1], col_idx int32[nnz] (ascending per row), values fp64[nnz].
 * Arrays may be host or device pointers; the handle owns a device copy. */
int rd_gpu_csr_create(rd_ctx* ctx, int rows, int cols, int64_t nnz, const int32_t* row_ptr,
                      const int32_t* col_idx, const double* values, rd_csr** out);
void rd_gpu_csr_free(rd_csr* a);
int rd_gpu_csr_info(const rd_csr* a, int* rows, int* cols, int64_t* nnz);
int rd_gpu_csr_download(const rd_csr* a, int32_t* row_ptr, int32_t* col_idx, double* values);

/* ------------------------------------------------------------ kernels */
/* replaces rd::spmv(A, x)                                linalg.hpp:30, linalg.cpp:19-33 */
int rd_gpu_spmv(rd_ctx* ctx, const rd_csr* a, const double* x, double* y);
/* deterministic device dot product (fixed reduction tree) */
int rd_gpu_dot(rd_ctx* ctx, int n, const double* a, const double* b, double* out);
/* replaces rd::coarsen_redblack(A)                       amg.hpp:29, amg.cpp:7-56 */
int rd_gpu_coarsen_redblack(rd_ctx* ctx, const rd_csr* a, uint8_t* flags, rd_csr** p_out);
/* replaces rd::galerkin_coarse(A, P)                     amg.hpp:31, amg.cpp:58-65 */
int rd_gpu_galerkin_coarse(rd_ctx* ctx, const rd_csr* a, const rd_csr* p, rd_csr** out);
/* replaces rd::sgs_sweep(A, f, u)                        amg.hpp:34, amg.cpp:67-88 */
int rd_gpu_sgs_sweep(rd_ctx* ctx, const rd_csr* a, const double* f, const double* u, double* out);

/* ------------------------------------------------------------ AMG */
/* replaces rd::build_amg(A, coarsest_threshold, smoothing_steps)  amg.hpp:36-37, amg.cpp:90-117.
 * The handle keeps its own copy of A; A may be freed afterwards. */
int rd_gpu_amg_setup(rd_ctx* ctx, const rd_csr* a, int coarsest_threshold, int smoothing_steps,
                     rd_amg** out);
void rd_gpu_amg_free(rd_amg* h);
int rd_gpu_amg_num_levels(const rd_amg* h);
/* which: 0 = A_l, 1 = P_l, 2 = Pt_l (NULL on the coarsest level); borrowed */
const rd_csr* rd_gpu_amg_level_matrix(const rd_amg* h, int level, int which);
/* coarse_flag of level l (1 = C), host buffer of rows(A_l) bytes */
int rd_gpu_amg_level_flags(const rd_amg* h, int level, uint8_t* flags);
/* level l's smoother: 0 generic, 1 structured lattice kernel streaming the packed stencil,
 * 2 structured with the uniform stencil held in registers (every row = the centre row),
 * 3 structured with the 64 position-class rows in shared memory                          */
int rd_gpu_amg_level_structured(const rd_amg* h, int level);
/* replaces rd::amg_apply(h, r) / amg_precond(h)          amg.hpp:39-42, amg.cpp:119-145 */
int rd_gpu_amg_apply(rd_amg* h, const double* r, double* z);
/* one Gauss-Seidel pass (forward != 0: i ascending) on level l's matrix with the
 * kernel the V-cycle uses there; DEVICE pointers, stream-ordered (xin may be NULL =
 * zero vector).  Half of rd::sgs_sweep (amg.cpp:67-88); used to time the smoother. */
int rd_gpu_amg_level_sweep(rd_amg* h, int level, int forward, const double* f, const double* xin,
                           double* xout);

/* ------------------------------------------------------------ PCG */
typedef struct {
  int iterations;
  int converged;
} rd_pcg_report;

/* replaces rd::pcg(A, amg_precond(h), f, tol, max_iter)  linalg.hpp:46-49, linalg.cpp:64-102.
 * amg == NULL selects the identity preconditioner.  residual_history (host,
 * >= max_iter doubles) may be NULL.  Zero initial guess. */
int rd_gpu_pcg(rd_ctx* ctx, const rd_csr* a, rd_amg* amg, const double* f, double tol, int max_iter,
               double* x, rd_pcg_report* report, double* residual_history);

/* ------------------------------------------------------------ adaptivity */
/* bisection state of a mesh (mesh.hpp:17-20): refinement edge (0, d), d in {1,2,3}, and
 * generation per tet; build_structured_cube / rd_gpu_mesh_create meshes carry d = 3, gen 0.
 * Host or device arrays; either may be NULL. */
int rd_gpu_mesh_tags(const rd_mesh* mesh, uint8_t* refinement_edge, int32_t* generation);
int rd_gpu_mesh_set_tags(rd_mesh* mesh, const uint8_t* refinement_edge, const int32_t* generation);
/* replaces rd::bisect_marked(mesh, marked)             mesh.hpp:44, mesh.cpp:67-145: newest-vertex
 * bisection of the marked tets with conforming closure; a new mesh (vertex, tet, tag and
 * generation arrays identical to the reference's).  RD_EINVAL for an id outside [0, n_tets)
 * (the reference throws std::out_of_range). */
int rd_gpu_bisect_marked(rd_ctx* ctx, const rd_mesh* mesh, int n_marked, const int32_t* marked, rd_mesh** out);
/* replaces rd::uniform_refine(mesh)                     mesh.hpp:40, mesh.cpp:147-156 */
int rd_gpu_uniform_refine(rd_ctx* ctx, const rd_mesh* mesh, rd_mesh** out);
/* replaces rd::estimate(sol, target)                    adapt.hpp:21, adapt.cpp:35-124: eta per tet
 * (n_tets doubles, host or device) and the global sqrt(sum eta^2).  The system carries rho. */
int rd_gpu_estimate(rd_ctx* ctx, const rd_mesh* mesh, const rd_system* sys, const double* coeffs,
                    const rd_target* target, double* per_tet, double* global);
/* replaces rd::mark_dorfler(est, theta)                 adapt.hpp:24, adapt.cpp:126-150: the marked
 * tets in marking order (>= n ints, host or device) and their count; RD_EINVAL unless 0 < theta <= 1 */
int rd_gpu_mark_dorfler(rd_ctx* ctx, int n, const double* per_tet, double theta, int32_t* marked, int* n_marked);
/* replaces rd::adaptive_solve(initial, target, rho, dof_budget, solver, theta)  adapt.hpp:44-47,
 * adapt.cpp:152-205, with the AMG solver of bench.cpp:65-74 (build_amg + pcg(tol, 500)).
 * history: >= cap rows (the level count is returned in *n_levels even when it exceeds cap);
 * final_mesh (may be NULL) receives the last mesh; coeffs (host or device, may be NULL) the last
 * solution when it fits coeffs_cap. */
typedef struct {
  int level, dofs, iterations;
  double eta, err_l2_sq, err_hm1_sq, seconds;
} rd_adapt_level;
int rd_gpu_adaptive_solve(rd_ctx* ctx, const rd_mesh* initial, const rd_target* target, double rho, int dof_budget,
                          double tol, double theta, rd_adapt_level* history, int cap, int* n_levels,
                          rd_mesh** final_mesh, double* coeffs, int coeffs_cap);

/* ------------------------------------------------------------ LinOp (linalg.hpp:11) */
/* rd::LinOp = std::function<Vec(const Vec&)>: a fixed linear map.  Here y = op(x) on DEVICE
 * vectors of n doubles, enqueued on the context's stream (rd_gpu_ctx_stream); x and y never
 * alias.  The callback returns RD_OK or an RD_E* code, which the caller propagates.  Built-in
 * operators are recognised by rd_gpu_pcg_linop and run fused (no callback round trip). */
typedef int (*rd_linop_fn)(void* user, rd_ctx* ctx, int64_t n, const double* x, double* y);
typedef struct {
  rd_linop_fn apply;
  void* user;
} rd_linop;
typedef struct rd_jacobi rd_jacobi;
/* identity_precond()                                     linalg.hpp:39, linalg.cpp:53-55 */
int rd_gpu_linop_identity(rd_linop* out);
/* [&A](x) { return spmv(A, x); }                         linalg.cpp:104-106 (borrows a) */
int rd_gpu_linop_csr(const rd_csr* a, rd_linop* out);
/* amg_precond(h)                                         amg.hpp:42, amg.cpp:143-145 (borrows h) */
int rd_gpu_linop_amg(rd_amg* h, rd_linop* out);
/* jacobi_precond(A): d = diag(A), RD_ENOTSPD ("non-positive diagonal") when some d_i <= 0,
 * apply r ./ d                                           linalg.hpp:40, linalg.cpp:57-62 */
int rd_gpu_jacobi_create(rd_ctx* ctx, const rd_csr* a, rd_jacobi** out);
void rd_gpu_jacobi_free(rd_jacobi* j);
int rd_gpu_linop_jacobi(rd_jacobi* j, rd_linop* out);
/* y = op(x), host or device vectors, synchronous */
int rd_gpu_linop_apply(rd_ctx* ctx, rd_linop op, int64_t n, const double* x, double* y);
/* replaces rd::pcg(apply_A, apply_P, f, tol, max_iter)   linalg.hpp:46-47, linalg.cpp:64-102
 * (and pcg(A, apply_P, ...) with apply_A = rd_gpu_linop_csr(A), linalg.cpp:104-106).
 * f / x host or device; residual_history host (>= max_iter doubles) or NULL. */
int rd_gpu_pcg_linop(rd_ctx* ctx, int64_t n, rd_linop apply_a, rd_linop apply_p, const double* f, double tol,
                     int max_iter, double* x, rd_pcg_report* report, double* residual_history);

/* ------------------------------------------------------------ BDDC (bddc.hpp) */
typedef struct rd_bddc rd_bddc;
/* replaces rd::partition_geometric(mesh, dof_map, p)    bddc.hpp:30, bddc.cpp:45-111: the RCB owner
 * of every tet (n_tets ints, host); RD_EINVAL for p < 2 or p > n_tets */
int rd_gpu_partition_geometric(rd_ctx* ctx, const rd_mesh* mesh, const rd_system* sys, int p, int32_t* owner);
/* replaces rd::build_bddc(mesh, sys, partition_geometric(mesh, dof_map, p))   bddc.hpp:58-59, bddc.cpp:113-301 */
int rd_gpu_bddc_create(rd_ctx* ctx, const rd_mesh* mesh, const rd_system* sys, int p, rd_bddc** out);
void rd_gpu_bddc_free(rd_bddc* b);
int rd_gpu_bddc_info(const rd_bddc* b, int* n_interface, int* n_primal);
int rd_gpu_bddc_interface_dofs(const rd_bddc* b, int32_t* dofs);    /* ascending interior-dof ids (host) */
int rd_gpu_bddc_coarse_matrix(const rd_bddc* b, double* out);       /* n_primal^2, row-major (host) */
/* schur_apply / reduce_rhs / expand_solution / bddc_apply   bddc.hpp:61-75, bddc.cpp:303-430;
 * host or device vectors (n_interface, n_dofs as the reference's) */
int rd_gpu_bddc_schur_apply(rd_bddc* b, const double* x, double* y);
int rd_gpu_bddc_reduce_rhs(rd_bddc* b, const double* f, double* g);
int rd_gpu_bddc_expand(rd_bddc* b, const double* u_interface, const double* f, double* u);
int rd_gpu_bddc_apply(rd_bddc* b, const double* r, double* z);
/* schur_op(op), bddc_precond(op) as rd_linop operators (borrow b)   bddc.hpp:77-78 */
int rd_gpu_linop_bddc_schur(rd_bddc* b, rd_linop* out);
int rd_gpu_linop_bddc(rd_bddc* b, rd_linop* out);
/* replaces rd::bddc_solve(mesh, sys, p, tol, max_iter)   bddc.hpp:85-87, bddc.cpp:440-456:
 * u = n_dofs (host or device), residual_history host (>= max_iter) or NULL */
int rd_gpu_bddc_solve(rd_ctx* ctx, const rd_mesh* mesh, const rd_system* sys, int p, double tol, int max_iter,
                      double* u, rd_pcg_report* report, double* residual_history);


/* replaces rd::solve_system(mesh, sys, PrecondKind::amg, p, tol)  bench.hpp:48-57, bench.cpp:185-225:
 * build_amg(A) [setup_seconds], pcg(A, amg, f, tol, 500) [solve_seconds]. */
typedef struct {
  int iterations;
  int converged;
  double setup_seconds;
  double solve_seconds;
} rd_solve_outcome;
int rd_gpu_solve_system_amg(rd_ctx* ctx, const rd_csr* a, const double* f, double tol, double* u,
                            rd_solve_outcome* out);

/* The bench-precond row end to end from a host TetMesh (mesh.hpp:13-24 arrays, as for
 * rd_gpu_mesh_create) in one call: upload, rd::build_system (assembly.cpp:225-238), then
 * solve_system's AMG branch (bench.cpp:185-225) with u (n_dofs doubles, host or device) read
 * back.  The host arrays need only live for the call.  A mesh of Kuhn-lattice size is solved
 * provisionally as rd::build_structured_cube's mesh (vertices and boundary flags generated on
 * the device, tets by formula) while the host arrays upload on a second stream; the uploaded
 * vertices and flags are compared bit for bit with the generated ones (any difference restarts
 * on the uploaded arrays) and the uploaded tets with the Kuhn enumeration (a mismatch reruns on
 * the generic path) before the call returns.  u may be written by a provisional attempt and is
 * always overwritten by the attempt that stands.  Same results, errors and timing split as
 * rd_gpu_build_system + rd_gpu_solve_system_amg.  n_dofs_out may be NULL. */
int rd_gpu_solve_host_mesh(rd_ctx* ctx, int nv, const double* xyz, int nt, const int32_t* tets, const uint8_t* bnd,
                           double rho, const rd_target* target, double tol, double* u, int* n_dofs_out,
                           rd_solve_outcome* out);

/* replaces rd::l2_error / rd::h1_semi_error (assembly.hpp:59-61, assembly.cpp:265-310) for the
 * manufactured exact solution u = c sin(pi x) sin(pi y) sin(pi z), c = 1/(3 rho pi^2 + 1)
 * (rd::manufactured_exact(rho), target.cpp:45-58): the P1 field with interior coefficients
 * `coeffs` (n_dofs, host or device) and zero boundary values, degree-5 rule per tet.  Either
 * output may be null.  RD_EINVAL if rho < 0 or sizes mismatch. */
int rd_gpu_error_norms(rd_ctx* ctx, const rd_mesh* mesh, const rd_system* sys, const double* coeffs,
                       double rho, double* l2_error, double* h1_semi_error);

/* replaces rd::l2_error_target_squared(sol, target)  assembly.hpp:62, assembly.cpp:312-331:
 * the SQUARED L2 distance of the P1 field (interior coefficients `coeffs`, host or device)
 * to the target field, with the target's own rule (rule_for: 64-point subdivision for the
 * discontinuous box / ball, degree-5 otherwise).  The BASELINE error gate ||u_rho,h - u_bar||_L2
 * for every target; ||grad(u - u_bar)|| of the smooth target is rd_gpu_error_norms(rho = 0). */
int rd_gpu_l2_error_target_squared(rd_ctx* ctx, const rd_mesh* mesh, const rd_system* sys, const double* coeffs,
                                   const rd_target* target, double* err2);

/* replaces rd::l2_error(sol, target.evaluator) / rd::h1_semi_error(sol, grad u_bar)  (assembly.hpp:59-61,
 * assembly.cpp:265-310) with the TARGET field u_bar as the exact function: l2 = ||u_h - u_bar||_L2,
 * h1 = ||grad(u_h - u_bar)||_L2, degree-5 rule per tet.  grad u_bar: sin^3 as manufactured_exact(0)
 * (smooth, nonzero_bc, and the sine part of sine+random), the P1 interpolant's gradient on the
 * Kuhn tet its point location picks (sine+random), (y, x, 2) (quadratic), 0 a.e. (indicators,
 * constants).  The BASELINE C3 gate ||grad(u_rho,h - u_bar)||.  Either output may be null. */
int rd_gpu_error_norms_target(rd_ctx* ctx, const rd_mesh* mesh, const rd_system* sys, const double* coeffs,
                              const rd_target* target, double* l2_error, double* h1_semi_error);

/* replaces the rho-coupled table's target_dual_norm(sys, sol)  bench.cpp:55-63 with
 * target_residual (assembly.cpp:354-356) and hminus1_norm[_with] (assembly.cpp:333-352):
 * r = f - M u, w = K^-1 r (dense LLT for n <= 2000, else AMG(K)-PCG to 1e-11), sqrt(r . w).
 * RD_ERUNTIME on a negative pairing, RD_ENOTSPD if K is not SPD.                      */
int rd_gpu_target_dual_norm(rd_ctx* ctx, const rd_system* sys, const double* coeffs, double* out);

/* ------------------------------------------------------------ distributed (z-slab) pieces
 * SURVEY.md §8(e).  The reference has no distributed solver (its parallelism is
 * the thread pool of parallel.cpp:12-73); these calls are the per-rank device
 * work of the slab-partitioned AMG-PCG that paper_2102_03515_b200/dist.py drives
 * over torch.distributed (NCCL halo planes + dot reductions).  DEVICE pointers
 * only; every call is stream-ordered on the context's stream and asynchronous
 * (device-detected errors surface at the next rd_gpu_synchronize).              */

/* speculative-division miss of a lattice sweep, reported by rd_gpu_synchronize
 * after asynchronous sweeps: rerun the computation with exact sweeps.        */
#define RD_GS_SPECULATION_MISS 0x5ec
int rd_gpu_ctx_set_exact_sweeps(rd_ctx* ctx, int exact);

/* rows [row0, row1) of a, keeping columns [col0, col1) renumbered from 0 (RD_EINVAL
 * if a kept row has a column outside): a rank's block of A_l / P_l / Pt_l.       */
int rd_gpu_csr_rowblock(rd_ctx* ctx, const rd_csr* a, int row0, int row1, int col0, int col1, rd_csr** out);
/* res = r - A z  (the V-cycle residual, amg.cpp:127) */
int rd_gpu_residual(rd_ctx* ctx, const rd_csr* a, const double* r, const double* z, double* res);
/* z += P zc  (the V-cycle correction, amg.cpp:130) */
int rd_gpu_prolong_add(rd_ctx* ctx, const rd_csr* p, const double* zc, double* z);
/* *out_dev = a . b (deterministic fixed-order reduction; out_dev on the device) */
int rd_gpu_dot_async(rd_ctx* ctx, int n, const double* a, const double* b, double* out_dev);
/* x += alpha p, r -= alpha Ap  /  p = z + beta p   (linalg.cpp:84-85,99) */
int rd_gpu_pcg_update_xr(rd_ctx* ctx, int64_t n, double alpha, const double* p, const double* ap, double* x,
                         double* r);
int rd_gpu_pcg_update_p(rd_ctx* ctx, int64_t n, double beta, const double* z, double* p);

/* The distributed PCG's scalars on the device (linalg.cpp:64-102 split across ranks): every
 * rank all-gathers its local dot partials into `parts` [world] (NCCL, on the stream) and these
 * calls sum them in rank order -- the same bits on every rank -- and keep rz, alpha, beta,
 * the relative residual and the convergence / SPD status in a device-resident rd_pcg_state,
 * so no scalar crosses to the host inside the loop; the host reads the 64-byte state once
 * per iteration.  After done or a status, alpha / xr / check / p calls are no-ops.
 *   status 1: p'Ap <= 0 (runtime_error "pcg: operator not positive definite (p'Ap <= 0)")
 *   status 2: r'z < 0   (runtime_error "pcg: preconditioner not positive definite")       */
typedef struct rd_pcg_state {
  double rz, rz0, pap, rz_next, alpha, beta, rel, reserved;
  int32_t done, status, iterations, reserved2;
} rd_pcg_state;
int rd_gpu_pcg_dist_begin(rd_ctx* ctx, int world, const double* parts, rd_pcg_state* st);   /* rz0 = sum */
int rd_gpu_pcg_dist_alpha(rd_ctx* ctx, int world, const double* parts, rd_pcg_state* st);   /* pAp, alpha */
int rd_gpu_pcg_dist_xr(rd_ctx* ctx, int64_t n, const rd_pcg_state* st, const double* p, const double* ap, double* x,
                       double* r);
/* rz_next = sum, history[it-1] = rel = sqrt(rz_next / rz0), done if rel <= tol, else beta */
int rd_gpu_pcg_dist_check(rd_ctx* ctx, int world, const double* parts, rd_pcg_state* st, double tol, double* history,
                          int history_cap);
int rd_gpu_pcg_dist_p(rd_ctx* ctx, int64_t n, const rd_pcg_state* st, const double* z, double* p);
/* the V-cycle of the sub-hierarchy from `level` (amg.cpp:121-132 entered at level l):
 * r, z of rows(A_level); the coarse tail of a distributed V-cycle, on rank 0   */
int rd_gpu_amg_apply_from(rd_amg* h, int level, const double* r, double* z);

/* One rank's z-slab [zlo, zhi) of a lattice level (a: the level's whole-box matrix,
 * e.g. rd_gpu_amg_level_matrix(h, l, 0)).  Local vectors hold planes [g0, g1):
 * the slab plus one ghost plane on each side where the box has one.           */
typedef struct rd_slab rd_slab;
int rd_gpu_slab_create(rd_ctx* ctx, const rd_csr* a, int zlo, int zhi, rd_slab** out);
void rd_gpu_slab_free(rd_slab* s);
int rd_gpu_slab_info(const rd_slab* s, int* lattice_side, int* g0, int* g1);
/* One Gauss-Seidel pass (half of sgs_sweep, amg.cpp:67-88) over the slab's rows.
 * f, xin (NULL = zero vector), xout: local vectors (planes [g0, g1); xin's
 * downstream ghost plane = old values).  in_plane: the L*L values of the upstream
 * ghost plane (zlo-1 forward, zhi backward; NULL = zeros) -- the neighbour's
 * fresh values reproduce the whole-box sweep bit for bit.                       */
int rd_gpu_slab_sweep(rd_slab* s, int forward, const double* f, const double* xin, double* xout,
                      const double* in_plane);

/* Pipelined hand-off (exact, no host round trip): the sweep kernel itself stores
 * its downstream boundary plane as tagged {value, sweep} cells into the
 * downstream neighbour's cell buffer -- another GPU's memory mapped over NVLink
 * -- while the neighbour's kernel is already running and polls them.  The
 * single-GPU sweep, bit for bit, with the wavefront crossing GPUs row by row.
 *   same process / device:  rd_gpu_slab_link(s, next, prev)
 *   one process per GPU:    rd_gpu_slab_ipc_handle on every rank, exchange the
 *                           64-byte handles, rd_gpu_slab_open_peer(s, 0 = next /
 *                           1 = previous, handle, the neighbour's g0)
 * Every rank must run the same sequence of slab sweeps (the cell tags count
 * them).  Ranks on one device must not launch waiting kernels separately:
 * rd_gpu_slab_sweep_multi relaxes all linked slabs in one cooperative launch.  */
#define RD_IPC_HANDLE_BYTES 64
int rd_gpu_slab_link(rd_slab* s, const rd_slab* next, const rd_slab* prev);
int rd_gpu_slab_ipc_handle(rd_slab* s, void* handle /* RD_IPC_HANDLE_BYTES */);
int rd_gpu_slab_open_peer(rd_slab* s, int which, const void* handle, int peer_g0);
int rd_gpu_slab_sweep_pipelined(rd_slab* s, int forward, const double* f, const double* xin, double* xout);
int rd_gpu_slab_sweep_multi(int n, rd_slab* const* s, int forward, const double* const* f,
                            const double* const* xin, double* const* xout);

#ifdef __cplusplus
}
#endif

#endif /* RD_GPU_H */
