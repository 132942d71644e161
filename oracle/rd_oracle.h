/*
 * rd_oracle.h -- TEST INFRASTRUCTURE ONLY (parity checker), never the product.
 *
 * C-callable surface of the CPU restatement of the reference's AMG-PCG solve
 * path (rdsolve, arXiv 2102.03515).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so.
 *
 * Every object is an opaque heap handle freed with or_free().  Functions that
 * can fail return an int status (0 = ok, 1 = invalid_argument, 2 =
 * runtime_error, mirroring the reference's exception types) and leave the
 * message in or_last_error().
 */
#ifndef RD_ORACLE_H
#define RD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_mesh or_mesh;
typedef struct or_system or_system;
typedef struct or_csr or_csr;
typedef struct or_amg or_amg;

const char* or_last_error(void);
void or_set_num_threads(int n);
int or_num_threads(void);

/* mesh.cpp:29-65 */
int or_build_structured_cube(int n, or_mesh** out);
void or_mesh_free(or_mesh* m);
/* a hand-built mesh (test_assembly.cpp:23-33 reference tet) */
int or_mesh_new(int nv, const double* xyz, int nt, const int* tets, const uint8_t* boundary,
                or_mesh** out);
void or_mesh_info(const or_mesh* m, int* n_vertices, int* n_tets);
void or_mesh_get(const or_mesh* m, double* xyz, int* tets, uint8_t* boundary,
                 uint8_t* refinement_edge, int* generation);
double or_tet_volume(const or_mesh* m, int t);

/* quadrature.cpp: rule 0 centroid, 1 degree2, 2 degree5 (14pt), 3 subdivision64 */
int or_rule_size(int rule);
void or_rule_get(int rule, double* points /* size x 4 */, double* weights);

/* target.cpp + the two BASELINE targets (ball, sine+random) */
enum { OR_TARGET_SMOOTH = 0, OR_TARGET_BOX = 1, OR_TARGET_NONZERO_BC = 2,
       OR_TARGET_BALL = 3, OR_TARGET_SINE_RANDOM = 4,
       /* test-only targets from the reference's assembly tests */
       OR_TARGET_ZERO = 5, OR_TARGET_ONE = 6, OR_TARGET_QUADRATIC = 7 };
int or_target_eval(int kind, int n, uint64_t seed, int npts, const double* xyz,
                   double* out);
void or_pseudo_random_vec(int n, uint64_t seed, double* out);

/* assembly.cpp:225-238 build_system */
int or_build_system(const or_mesh* m, double rho, int target_kind, uint64_t seed,
                    or_system** out);
void or_system_free(or_system* s);
int or_system_n_dofs(const or_system* s);
/* which: 0 = K, 1 = M, 2 = A */
or_csr* or_system_csr(or_system* s, int which); /* borrowed */
void or_system_get_f(const or_system* s, double* f);
void or_system_get_dofmap(const or_system* s, int* vertex_to_dof, int* dof_to_vertex);
/* assembly.cpp full (pre-elimination) matrices: which 0 = K, 1 = M */
int or_assemble_full(const or_mesh* m, int which, or_csr** out);
int or_assemble_load(const or_mesh* m, int target_kind, uint64_t seed, double* f);

/* CSR containers (types.hpp:14, linalg.cpp:11-17) */
int or_csr_new(int rows, int cols, int64_t nnz, const int* rp, const int* ci,
               const double* v, or_csr** out);
int or_from_triplets(int rows, int cols, int64_t n, const int* ti, const int* tj,
                     const double* tv, or_csr** out);
void or_csr_free(or_csr* a);
void or_csr_info(const or_csr* a, int* rows, int* cols, int64_t* nnz);
void or_csr_get(const or_csr* a, int* rp, int* ci, double* v);

/* linalg.cpp */
int or_spmv(const or_csr* a, int nx, const double* x, double* y);
int or_dense_cholesky_solve(int n, const double* a_rowmajor, const double* b, double* x);
double or_dot(int n, const double* a, const double* b);

/* amg.cpp */
int or_coarsen_redblack(const or_csr* a, uint8_t* flags, or_csr** p_out);
int or_galerkin_coarse(const or_csr* a, const or_csr* p, or_csr** out);
int or_sgs_sweep(const or_csr* a, const double* f, const double* u, double* out);
int or_build_amg(const or_csr* a, int coarsest_threshold, int smoothing_steps,
                 or_amg** out);
void or_amg_free(or_amg* h);
int or_amg_num_levels(const or_amg* h);
/* which: 0 = A, 1 = P, 2 = Pt ; borrowed, NULL when absent */
or_csr* or_amg_level_csr(or_amg* h, int level, int which);
int or_amg_level_flags(const or_amg* h, int level, uint8_t* flags);
int or_amg_apply(const or_amg* h, int n, const double* r, double* z);
int or_amg_apply_from(const or_amg* h, int level, int n, const double* r, double* z);

/* linalg.cpp:64-102; precond: 0 identity, 1 jacobi, 2 amg (uses h) */
int or_pcg(const or_csr* a, int precond, const or_amg* h, const double* f,
           double tol, int max_iter, double* x, int* iterations, int* converged,
           double* history /* >= max_iter entries, may be NULL */);

/* bench.cpp:185-241 solve_system, AMG branch */
int or_solve_system_amg(const or_system* s, double tol, double* u, int* iterations,
                        int* converged, double* setup_seconds, double* solve_seconds);

/* the whole BASELINE step on the CPU (mesh + build_system, build_amg, pcg), timed in C++ */
int or_pipeline(int n, double rho, int target_kind, uint64_t seed, double tol, int* iterations,
                int* converged, int* n_dofs, double* t_build, double* t_setup, double* t_solve);

/* assembly.cpp:265-310 error norms against the closed form (manufactured_exact) */
int or_l2_error_manufactured(const or_mesh* m, const or_system* s, const double* coeffs,
                             double rho_exact, double* out);
int or_target_dual_norm(const or_system* s, const double* coeffs, double* out);
int or_l2_error_target_squared(const or_mesh* m, const or_system* s, const double* coeffs, int kind, int n,
                               uint64_t seed, double* out);
int or_h1_semi_error_manufactured(const or_mesh* m, const or_system* s,
                                  const double* coeffs, double rho_exact, double* out);
/* assembly.cpp:265-310 with the TARGET field as the exact function (value = target evaluator,
 * gradient = Target::grad): l2 = ||u_h - u_bar||_L2, h1 = ||grad(u_h - u_bar)||_L2 (degree-5 rule;
 * either output may be null) -- the BASELINE error gates for every target, C3 included */
int or_error_norms_target(const or_mesh* m, const or_system* s, const double* coeffs, int kind, int n,
                          uint64_t seed, double* l2, double* h1);
/* the target's exact gradient at npts points (xyz [npts][3] -> g [npts][3]) */
int or_target_grad(int kind, int n, uint64_t seed, int npts, const double* xyz, double* g);

/* §8(f)3 adaptivity: estimate (adapt.cpp:35-124), mark_dorfler (:126-150), bisect_marked
 * (mesh.cpp:67-145), uniform_refine (:147-156), adaptive_solve (adapt.cpp:152-205, AMG solver) */
int or_estimate(const or_mesh* m, const or_system* s, const double* coeffs, int kind, uint64_t seed,
                double* per_tet, double* global);
int or_mark_dorfler(int n, const double* eta, double theta, int* marked, int* n_marked);
int or_bisect_marked(const or_mesh* m, int n_marked, const int* marked, or_mesh** out);
int or_uniform_refine(const or_mesh* m, or_mesh** out);
int or_adaptive_solve(const or_mesh* initial, int kind, uint64_t seed, double rho, int dof_budget, double tol,
                      double theta, int cap, int* n_levels, int* hist_i, double* hist_d, or_mesh** final_mesh,
                      double* coeffs, int coeffs_cap);

/* §8(f)4 BDDC (bddc.hpp / bddc.cpp:45-456) */
typedef struct or_bddc or_bddc;
int or_partition_geometric(const or_mesh* m, const or_system* s, int p, int* owner, int* n_subdomains_per_dof,
                           int* subdomains);
int or_bddc_create(const or_mesh* m, const or_system* s, int p, or_bddc** out);
void or_bddc_free(or_bddc* b);
void or_bddc_info(const or_bddc* b, int* n_interface, int* n_primal, int* p);
void or_bddc_interface(const or_bddc* b, int* dofs);
void or_bddc_coarse(const or_bddc* b, double* out);
void or_bddc_sub_info(const or_bddc* b, int s, int* nI, int* nB, int* ncon);
void or_bddc_sub_get(const or_bddc* b, int s, int* boundary, int* bidx, int* pidx, double* scaling, double* C,
                     double* Phi, double* S);
int or_bddc_op(const or_bddc* b, int which, int n_in, const double* in, const double* f, double* out);
int or_bddc_solve(const or_mesh* m, const or_system* s, int p, double tol, int max_iter, double* u, int* iterations,
                  int* converged, double* history);

#ifdef __cplusplus
}
#endif

#endif
