/*
 * ldg_b200.h — C ABI of the B200-native LDG diffusion path.
 *
 * Drop-in boundary for the per-time-step hot path of the reference LDG
 * solver (arXiv 1408.3877, FESTUNG Part I; C++ reference proj/include/ldg):
 * mesh geometry/topology precompute, L2 projection of d(t) and f(t), the
 * fused reassembly of the coefficient-dependent block operator, the
 * right-hand side, and the Krylov solve of each implicit-Euler step.
 *
 * The reference has no FFI layer: its "interface" is the set of header-only
 * free functions and LdgSystem methods.  Each entry point below names the
 * reference function(s) it replaces (file:line under proj/include/ldg/).
 * The C++ host wrapper paper_1408_3877_b200/host/ldg_host.hpp re-exposes
 * these with the reference's signatures and exception types.
 *
 * Conventions
 *  - plain pointers and sizes; no torch or CUDA types in signatures;
 *  - host arrays are in the reference layout: coordinates V x 2, triangles
 *    K x 3 (counter-clockwise), dof vectors k-major (index k*N + j, the
 *    vec_dof order of fields.hpp:26-32), stacked state Y = [Z1; Z2; C];
 *  - operator exports use the global numbering of system.hpp:120-135:
 *    row (u*K + k)*N + i, column (v*K + k')*N + j, u,v in {Z1=0, Z2=1, C=2};
 *  - every call returns an ldg_status; ldg_last_error() has the message;
 *  - one handle per GPU (rank); a handle is not thread-safe; work is
 *    stream-ordered on the handle's own CUDA stream.
 */
#ifndef LDG_B200_H
#define LDG_B200_H

#include <stdint.h>

#include "ldg_b200_coeffs.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ldg_status {
  LDG_OK = 0,
  LDG_EINVAL = 1,   /* std::invalid_argument in the reference             */
  LDG_EMESH = 2,    /* ldg::MeshError (mesh.hpp:25-27)                     */
  LDG_ECUDA = 3,    /* CUDA runtime error / no device                      */
  LDG_ENCCL = 4,    /* NCCL error                                          */
  LDG_ENOCONV = 5   /* std::runtime_error: solve failed / residual > tol   */
} ldg_status;

enum { LDG_BC_DIRICHLET = 0, LDG_BC_NEUMANN = 1 };
enum { LDG_MAX_BC = 16 };

/* ProblemSpec (system.hpp:26-37) with compiled-in coefficients. */
typedef struct ldg_problem {
  ldg_coeff d, f, c_d, g_n, c0;
  double eta;
  int n_bc;
  int bc_id[LDG_MAX_BC];
  int bc_kind[LDG_MAX_BC];
} ldg_problem;

/* Krylov options for the implicit-Euler solve that replaces SparseLU
 * (system.hpp:190-205).  The reference residual contract
 * ||lhs*y - rhs|| / max(||rhs||, 1) <= contract_tol is checked after every
 * solve when check_residual != 0 (default 1e-10).  The default stopping
 * rule (ldg_default_solver_opts) is rtol = 1e-14 on the Schur residual, met
 * together with the contract; it keeps states within 1e-10 relative L2 of the
 * reference's direct solve (tests/test_gpu_parity_scale.py).  FGMRES stops
 * early only when the residual stagnates at the rounding floor after the
 * contract is met. */
typedef struct ldg_solver_opts {
  double rtol;          /* Schur-system relative residual target (1e-14)   */
  double atol;          /* absolute target on the Schur residual           */
  int maxit;            /* Krylov iterations per solve                     */
  int precond;          /* 0 none, 1 block-Jacobi, 2 multigrid V(2,2) (FK)  */
  int check_residual;   /* 1: enforce the reference residual contract      */
  double contract_tol;  /* 1e-10 in the reference                          */
  int krylov;           /* 0 FGMRES(restart) (default), 1 BiCGStab          */
  int restart;          /* FGMRES basis size (<= 78; 0: 30)                 */
} ldg_solver_opts;

typedef struct ldg_step_stats {
  int iterations;       /* Krylov iterations (summed over steps)           */
  int applies;          /* Schur operator applications                     */
  double schur_relres;  /* final relative Schur residual (last step)       */
  double residual;      /* reference contract residual (last step)         */
  double ms_assemble;   /* device time: projection + assembly + rhs        */
  double ms_solve;      /* device time: Krylov solve + Z recovery + check  */
  double ms_setup;      /* part of ms_solve: rhs, preconditioner setup      */
  double ms_krylov;     /* part of ms_solve: the Krylov iterations          */
} ldg_step_stats;

typedef struct ldg_info_t {
  int p, n_local;       /* degree and N                                    */
  int num_t;            /* K (global)                                      */
  int num_owned;        /* elements owned by this rank                     */
  int num_ghost;        /* halo elements                                   */
  int num_v;
  int rank, size;
  int64_t bytes_device; /* device memory held by the handle                */
  int64_t launches;     /* sm_100a kernel launches issued by this handle   */
} ldg_info_t;

typedef struct ldg_handle ldg_handle;

/* Host-only (no GPU needed): the reference tensors this library uploads,
 * build_ref_tensors (reftensors.hpp:55-154), in the reference index layout:
 * m n*n, h n*n*2, g n^3*2, sd n*n*3, so n*n*9, rd n^3*3, ro n^3*9. */
int ldg_reference_tensors(int n_local, double* m, double* h, double* g, double* sd, double* so, double* rd,
                          double* ro);

/* The RefTensors argument of the reference's LdgSystem(mesh, spec, rt)
 * (system.hpp:67): replaces the handle's own reference tensors (same layout
 * as ldg_reference_tensors; rd / ro may be NULL -- R^m is assembled in the
 * exact rank-Q edge form).  With the tensors of the caller's
 * build_ref_tensors, every static block and G^m come out of the same
 * tables the reference multiplies, so the stored patterns of
 * ldg_export_operator_csc coincide with the reference's to the last
 * explicit zero.  Invalidates the assembled operators. */
int ldg_set_reference_tensors(ldg_handle* h, const double* m, const double* hh, const double* g, const double* sd,
                              const double* so, const double* rd, const double* ro);

/* Host-only: do these reference tensors (NULL, NULL, ...: the library's own)
 * have the structure the rank-Q_e operator kernels assume -- s_diag /
 * s_offdiag (reftensors.hpp:106-128) equal to the Q_e-point edge quadrature
 * of the basis traces to 1e-13, h_hat (reftensors.hpp:76-84) zero unless
 * deg phi_i > deg phi_j?  When not, the handle applies the operator from the
 * N x N tables instead (same results, more work).  *supported = 1 / 0. */
int ldg_rank_form_supported(int n_local, const double* m, const double* hh, const double* g, const double* sd,
                            const double* so, int* supported);

/* Selects the CUDA device used by handles created afterwards on this thread
 * (one process per GPU: the rank's local device). */
int ldg_set_device(int device);

/* ---- creation (replaces generate_grid_data mesh.hpp:103-221 + the
 *      LdgSystem ctor system.hpp:67-88: static operators, selectors) ---- */

/* General triangulation given on the host.  id_e0t (K x 3, nullable) holds
 * boundary IDs per (triangle, local edge); NULL applies the unit-square
 * rule of domain_square (mesh.hpp:245-252). */
int ldg_create(const double* coords, int num_v, const int* v0t, int num_t, const int* id_e0t, int p,
               const ldg_problem* prob, ldg_handle** out);

/* Friedrichs-Keller mesh of the unit square with dim x dim squares
 * (domain_square, mesh.hpp:225-254), generated on the device.  jitter > 0
 * moves interior vertices by U(-jitter*h, jitter*h) per coordinate from a
 * splitmix64 stream keyed by (seed, vertex id) — BASELINE config 4. */
int ldg_create_square(int dim, double jitter, uint64_t seed, int p, const ldg_problem* prob,
                      ldg_handle** out);

/* ---- multi-GPU strips --------------------------------------
 * FK(dim) is split into `size` strips of dim/size element columns; each rank
 * owns its strip plus one ghost column per side.  One process per GPU:
 * rank 0 calls ldg_nccl_unique_id, broadcasts the 128 bytes (e.g. with
 * torch.distributed), every rank calls ldg_create_square_dist.  Halos of the
 * operator applies go through ncclSend/Recv, Krylov dot products through
 * ncclAllReduce.  All other calls are collective over the ranks and keep
 * their single-GPU meaning; host arrays use global numbering and each rank
 * fills / reads its owned rows. */
int ldg_nccl_unique_id(char* out /* 128 bytes */);
int ldg_create_square_dist(int dim, double jitter, uint64_t seed, int p, const ldg_problem* prob, int rank, int size,
                           const char* nccl_id, ldg_handle** out);

/* The same decomposition with all `nranks` ranks in this process on the
 * current GPU ("virtual ranks", halos by device copies): validates the
 * distributed algorithm on one device; results match ldg_create_square. */
int ldg_create_square_group(int dim, double jitter, uint64_t seed, int p, const ldg_problem* prob, int nranks,
                            ldg_handle** out);

void ldg_destroy(ldg_handle* h);

/* Message of the last failure on this thread (or of handle h if given). */
const char* ldg_last_error(const ldg_handle* h);

int ldg_get_info(const ldg_handle* h, ldg_info_t* out);

/* Mesh lists for parity (mesh.hpp:35-98): b K*4 (b11,b12,b21,b22), area K,
 * len K*3, nu K*3*2, nbr/nbr_n K*3 (-1 on the boundary), id_e0t K*3,
 * coords V*2, v0t K*3.  Any pointer may be NULL. */
int ldg_mesh_lists(ldg_handle* h, double* coords, int* v0t, double* b, double* area, double* len, double* nu,
                   int* nbr, int* nbr_n, int* id_e0t);

/* ---- per-step path ---------------------------------------------------- */

/* L2 projection (fields.hpp:53-82) of fn at time t with a quad_rule_2d of
 * order q_ord; out is K x N k-major on the host. */
int ldg_project(ldg_handle* h, const ldg_coeff* fn, double t, int q_ord, double* out);

/* Everything build_blocks(t) computes (system.hpp:110-152): projection of d
 * and f, the fused time-dependent assembly of E^m = -G^m + R^m + R_D^m
 * (assembly.hpp:113-136, 214-252) and V = [-J1; -J2; eta K_D - K_N + L]
 * (assembly.hpp:256-338).  Device-resident; nothing is copied back. */
int ldg_assemble(ldg_handle* h, double t);

/* The time-dependent C-row blocks as the reference assembles them: all 8 N x N
 * blocks per element (E^m_kk and E^m_{k,nbr(k)}, device layout
 * [m][s][i*N+j][Kp]) together with the projection of d, f and the right-hand
 * side -- the assembly-only workload (BASELINE config 3).  The solver path
 * (ldg_assemble) stores only the diagonal blocks and evaluates the others
 * from D.  Device-resident (library buffer, allocated on first use); *ms
 * (optional) receives the device time of the call. */
int ldg_assemble_blocks(ldg_handle* h, double t, double* ms);

enum ldg_operator {
  LDG_OP_MASS = 0, LDG_OP_H1, LDG_OP_H2, LDG_OP_G1, LDG_OP_G2, LDG_OP_R1, LDG_OP_RD1, LDG_OP_R2,
  LDG_OP_RD2, LDG_OP_Q1, LDG_OP_QN1, LDG_OP_Q2, LDG_OP_QN2, LDG_OP_S, LDG_OP_SD,
  LDG_OP_A,      /* the assembled 3KN x 3KN operator of build_blocks          */
  LDG_OP_COUNT
};
enum ldg_vector {
  LDG_VEC_D = 0, LDG_VEC_F, LDG_VEC_JD1, LDG_VEC_JD2, LDG_VEC_KD, LDG_VEC_KN, LDG_VEC_L,
  LDG_VEC_V,     /* 3KN */
  LDG_VEC_Y,     /* 3KN state */
  LDG_VEC_COUNT
};

/* Operator export in COO (global numbering above) of the operators at the
 * time of the last ldg_assemble.  Returns the entry count in *nnz; arrays
 * (capacity cap) may be NULL to query the size.  Entries are whole N x N
 * blocks (explicit zeros kept). */
int ldg_export_operator(ldg_handle* h, int which, int64_t* nnz, int64_t* rows, int64_t* cols, double* vals,
                        int64_t cap);
int ldg_export_vector(ldg_handle* h, int which, double* out, int64_t cap);

/* The same operators in the reference's own storage: a column-major
 * Eigen::SparseMatrix<double> with 32-bit indices after setFromTriplets +
 * makeCompressed (SparseOperator, assembly.hpp:21-22,62-67; A as built by
 * system.hpp:120-140).  colptr has n + 1 entries (n = K*N, or 3*K*N for
 * LDG_OP_A), rows ascend within a column, and the stored pattern follows the
 * reference's rules: M, H^m, G^m drop exact zeros (assembly.hpp:84,103-104,
 * 130-131), S, S_D, Q^m, Q_N^m, R^m, R_D^m store whole blocks (explicit zeros
 * kept).  Pass rowind/vals NULL to query *nnz.  Maps directly onto
 * Eigen::Map<const Eigen::SparseMatrix<double>>(n, n, nnz, colptr, rowind, vals). */
int ldg_export_operator_csc(ldg_handle* h, int which, int64_t* nnz, int32_t* colptr, int32_t* rowind, double* vals,
                            int64_t cap);

/* Block compressed sparse rows of an operator: block row b = u*K + k in the
 * reference's element order (system.hpp:120-135), block columns ascending,
 * each block N x N row-major with its explicit zeros; blocks in which the
 * reference stores no entry are omitted.  rowptr has K+1 (3K+1 for A)
 * entries; vals holds nblocks*N*N doubles.  NULL arrays query *nblocks. */
int ldg_export_operator_bsr(ldg_handle* h, int which, int64_t* nblocks, int32_t* rowptr, int32_t* colind,
                            double* vals, int64_t cap_blocks);

/* Per-operator assembly with the caller's coefficients (one-rank handles).
 * d_disc is the discrete coefficient D, K x N k-major (vec_dof order);
 * the result is CSC as above.  The handle's assembled state is unchanged.
 *   assemble_dphi_phi_coeff(mesh, rt, d_disc) -> G^m   (assembly.hpp:113-136)
 *   assemble_edge_avg_coeff_nu(mesh, m, d_disc, sel_int, sel_dir, rt)
 *       -> R^m (dirichlet = 0) or R_D^m (dirichlet = 1) (assembly.hpp:214-252)
 * m is the normal component, 1 or 2 (else LDG_EINVAL, as the reference's
 * std::invalid_argument). */
int ldg_assemble_dphi_phi_coeff(ldg_handle* h, const double* d_disc, int m, int64_t* nnz, int32_t* colptr,
                                int32_t* rowind, double* vals, int64_t cap);
int ldg_assemble_edge_avg_coeff_nu(ldg_handle* h, const double* d_disc, int m, int dirichlet, int64_t* nnz,
                                   int32_t* colptr, int32_t* rowind, double* vals, int64_t cap);

/* State (SystemState, system.hpp:40-43): y is 3KN k-major per block. */
int ldg_initial_state(ldg_handle* h);  /* system.hpp:99-107 */
int ldg_set_state(ldg_handle* h, const double* y, double t);
int ldg_get_state(ldg_handle* h, double* y, double* t);

/* ---- post-processing of the device-resident state (fields.hpp:84-123) -- */

/* l2_error (fields.hpp:100-123): ||u_h - exact(t, .)||_{L2} of state
 * component `component` (0 Z1, 1 Z2, 2 C, the SystemState order of
 * system.hpp:40-43) with a quad_rule_2d of order q_ord; the convergence
 * study uses order 2p + 2 on C (convergence.hpp:96).  Summed over all ranks. */
int ldg_l2_error(ldg_handle* h, int component, const ldg_coeff* exact, double t, int q_ord, double* err);

/* to_lagrange (fields.hpp:87-97) of state component `component`: values at
 * the 3 vertices (p <= 1) or vertices + edge midpoints (p >= 2) of every
 * element, K x nodes k-major on the host (global element order); *nodes
 * receives 3 or 6. */
int ldg_to_lagrange(ldg_handle* h, int component, double* out, int* nodes);

/* write_vtu (vtkout.hpp:42-108) of state component `component` (0 Z1, 1 Z2,
 * 2 C): writes `<basename>.<t_lvl>.vtu` (ASCII VTK unstructured grid, every
 * triangle its own 3 (p <= 1) or 6 points, the reference's file byte for
 * byte) from the device-resident state; the path is copied to path_out
 * (nullable, path_cap bytes).  One-process handles only. */
int ldg_write_vtu(ldg_handle* h, int component, const char* var_name, const char* basename, int t_lvl,
                  char* path_out, int path_cap);

ldg_solver_opts ldg_default_solver_opts(void);

/* nsteps implicit Euler steps of length dt (system.hpp:155-174), entirely on
 * the device; the state is read/written with ldg_get_state/ldg_set_state. */
int ldg_euler_steps(ldg_handle* h, double dt, int nsteps, const ldg_solver_opts* opts, ldg_step_stats* stats);

/* The reference-facing step with HOST buffers (euler_step, system.hpp:155):
 * copies y_in (3KN, k-major, ideally pinned) to the device, runs nsteps
 * steps from time t, copies the state back to y_out.  *ms_total is the
 * device time of the whole sequence, copies included (CUDA events). */
int ldg_euler_steps_host(ldg_handle* h, const double* y_in, double t, double dt, int nsteps, double* y_out,
                         const ldg_solver_opts* opts, ldg_step_stats* stats, double* ms_total);

/* Stationary solve A Y = V at time t (system.hpp:177-185); result in the state. */
int ldg_solve_stationary(ldg_handle* h, double t, const ldg_solver_opts* opts, ldg_step_stats* stats);

/* y = (W + dt A) x on host vectors (3KN, k-major) with the operators of the
 * last ldg_assemble (the block-SpMV of system.hpp:162-167 / :199). */
int ldg_apply_lhs(ldg_handle* h, double dt, const double* x, double* y);

/* y = S_c c with S_c = M + dt (eta (S + S_D) - sum_m E^m M^-1 B^m) on host
 * C-space vectors (KN, k-major): the Schur complement of W + dt A on the
 * primary unknown that the Krylov solve applies in place of the reference's
 * SparseLU (system.hpp:161-172).  E^m = -G^m + R^m + R_D^m and
 * B^m = -H^m + Q^m + Q_N^m are the operators of the last ldg_assemble. */
int ldg_apply_schur(ldg_handle* h, double dt, const double* c, double* y);

/* ---- measurement --------------------------------------------------------- */

typedef struct ldg_kernel_times {
  double ms_project;    /* K2 projection of d, f + RHS                   */
  double ms_assemble;   /* K3 fused E^m assembly                          */
  double ms_spmv;       /* K6 full (W + dt A) block-SpMV                  */
  double ms_schur;      /* one Schur operator application (2 launches)     */
  int reps;
  int levels;           /* multigrid levels timed below (0: no FK hierarchy) */
  double ms_vcycle;     /* one preconditioner V-cycle (FP32 smoother), graph replay, L2 warm */
  double ms_level[8];   /* one smoothing sweep (residual + block-Jacobi) on level l, graph replay */
  double ms_sweep_s2;   /* level-0 smoother stage 2 + block-Jacobi update, one launch (L2 flushed if asked) */
  int s2_per_vcycle;    /* launches of that kernel per V-cycle (level-0 sweeps + residual) */
} ldg_kernel_times;

/* Times each hot kernel over reps launches with CUDA events on the handle's
 * stream (after warm-up), flushing L2 between launches when flush != 0. */
int ldg_time_kernels(ldg_handle* h, double t, double dt, int reps, int flush, ldg_kernel_times* out);

/* Synchronises the handle's stream. */
int ldg_sync(ldg_handle* h);

#ifdef __cplusplus
}
#endif

#endif /* LDG_B200_H */
