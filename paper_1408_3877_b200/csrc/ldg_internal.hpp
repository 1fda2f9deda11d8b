// Internal host-side state of an ldg_handle and the kernel launchers shared
// by the translation units of libldg_b200.so.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <memory>
#include <functional>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/ldg_b200.h"
#include "ldg_device.cuh"
#include "ldg_tables.hpp"

namespace ldgb {

constexpr int kMaxRed = 80;        // dot products per reduction (FGMRES basis + 1)
constexpr int kMaxLocalRanks = 16; // ranks of one process (virtual ranks share a GPU)
constexpr int kExtrapMax = 7;      // history of the extrapolated Euler start (team_solve)

// NVTX range over a scope (phases of a step in Nsight timelines; header-only
// NVTX v3, a no-op unless a tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Exceptions carry the ABI status they map to.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define LDG_CUDA(call)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      throw ::ldgb::Error(LDG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

// Device buffer owned by a handle.
template <typename T>
struct DBuf {
  T* ptr = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (ptr) cudaFree(ptr);
  }
  void alloc(size_t count, int64_t* counter) {
    release(counter);
    if (count == 0) return;
    LDG_CUDA(cudaMalloc(&ptr, count * sizeof(T)));
    // cudaMemset runs on the legacy default stream, which does not order
    // against the library's non-blocking streams: wait for it, or a kernel
    // launched right after the allocation can be overtaken by the zeroing
    // (seen as FP16 smoother copies full of inf on a second handle)
    LDG_CUDA(cudaMemset(ptr, 0, count * sizeof(T)));
    LDG_CUDA(cudaDeviceSynchronize());
    n = count;
    if (counter) *counter += static_cast<int64_t>(count * sizeof(T));
  }
  void release(int64_t* counter) {
    if (ptr) {
      cudaFree(ptr);
      if (counter) *counter -= static_cast<int64_t>(n * sizeof(T));
    }
    ptr = nullptr;
    n = 0;
  }
};

struct Handle {
  // sizes
  int p = 0, N = 0;
  int K = 0;       // owned elements
  int Kg = 0;      // owned + ghost
  long Kp = 0;     // plane stride
  int Kglobal = 0;
  int V = 0;
  int rank = 0, size = 1;
  ldg_problem prob{};
  int64_t bytes = 0;
  int64_t launches = 0;  // kernels issued (bench evidence: gpu_launches)

  HostTables tables;
  DBuf<double> tab;
  DBuf<float> ftab;      // FP32 smoother tables (build_f32_tables)
  DevTables dtab{};

  // mesh
  DBuf<double> coords;   // V*2 (interleaved)
  DBuf<int> v0t;         // Kg*3 (local vertex ids)
  DBuf<double> geom;     // kGeomCount * Kp
  DBuf<int> nbr, nbrn, kind, bid;  // 3 * Kp
  std::vector<int> gid;  // local -> global element id
  // host lists of a general mesh (ldg_create): the red-refinement hierarchy
  // of the multigrid is detected from them (ldg_mg.cu mg_build_general)
  std::vector<double> host_xy;
  std::vector<int> host_v0t, host_ids;

  // per-step operators / vectors
  DBuf<double> D, F;     // N * Kp
  DBuf<double> E;        // 2 * N*N * Kp (diagonal blocks; see ldg_device.cuh)
  DBuf<double> Efull;    // 2 * 4 * N*N * Kp, ldg_assemble_blocks only
  DBuf<double> Bst;      // 2 * 4 * N*N * Kp
  DBuf<double> Sst;      // 4 * N*N * Kp
  DBuf<double> Vv;       // 3 * N * Kp
  DBuf<double> Y, Yold;  // 3 * N * Kp
  // initial guess of the next implicit-Euler solve: C^{n-1}, C^{n-2} of the
  // last steps (Chist[i] at time hist_time[i]) extrapolate C^n in time
  // (team_solve).  hist_dev (device int) counts the valid history
  // vectors as the device sees them; hist_ok (host) says Y is the output of
  // the last solve at time hist_t0 + hist_dt, cleared by any external state
  // write.  hist_same (host-buffer calls): device flag "uploaded state == last
  // output", 0 drops the history on the device.
  DBuf<double> Chist[kExtrapMax];  // C^{n-1}, C^{n-2}, ... (kExtrapMax)
  DBuf<int> hist_dev;     // [0] valid history vectors, [1] order used by the last start
  double hist_time[kExtrapMax] = {}, hist_dt = 0.0;
  bool hist_ok = false;
  const int* hist_same = nullptr;
  DBuf<int> in_same;
  DBuf<double> host_in;            // k-major upload of a host state (host_stage keeps the last output)
  bool stage_is_output = false;
  double t = 0.0;
  double t_assembled = -1.0;
  bool assembled = false;

  // Krylov workspace (N * Kp each)
  DBuf<double> kr_r, kr_rh, kr_p, kr_v, kr_s, kr_t, kr_ph, kr_sh, kr_b;
  DBuf<double> tz;       // 2 * N * Kp : M^-1 B^m x
  DBuf<float> tz32;      // the same for the FP32 smoother on single-rank thread-per-element levels
  // edge traces of the FP32 smoother (single rank, ldg_smooth.cu): values at the Qe points of
  // each local edge, [n][q][Kp]: tr32 = x | -(c1 t^1 + c2 t^2) of the current sweep, dtr32 = d_h (per step)
  DBuf<float> tr32, dtr32;
  int xtr_cur = 0;  // which x-trace buffer of tr32 belongs to the vector stage 1 sees next
  DBuf<double> Pinv;     // N*N * Kp : block-Jacobi inverse
  DBuf<double> full_r, full_y;  // 3 * N * Kp : reference residual contract
  DBuf<double> red;      // reduction scratch
  DBuf<double> gs;       // FGMRES Gram-Schmidt coefficients on the device (h1 | h2 | hn)
  double* red_host = nullptr;  // pinned
  DBuf<double> flush;    // L2 flush buffer (measurement only)
  DBuf<double> host_stage;  // k-major staging of host states (3KN)
  DBuf<double> rule_elem;  // projection rule of order max(2p,1)
  int rule_elem_R = 0;

  cudaStream_t stream = nullptr;
  bool owns_stream = true;
  cudaEvent_t ev[6] = {};  // 0-2 step timing, 3-4 solve phases (team_solve), 5 host-buffer call span
  std::string err;

  // geometric multigrid hierarchy (ldg_mg.cu).  The top handle is level 0;
  // coarse levels are Handles of their own (same p, tables and stream shared)
  // on FK(dim / 2^l), with coordinates subsampled from the finer level.
  int dim = 0;                                   // FK dim (0: general mesh)
  const double* rule_shared = nullptr;           // coarse levels use level 0's rule
  int rule_shared_R = 0;
  std::vector<std::unique_ptr<Handle>> coarse;   // levels 1 .. L-1 (top handle only)
  bool mg_pcoarse = false;                       // same mesh as the finer level at a lower degree:
                                                 // transfers truncate / pad the modal coefficients
  DBuf<int> mg_parent;                           // element -> parent in the next coarser level
  DBuf<int> mg_children;                         // [4][Kp] children in the next finer level
  DBuf<float> mg_P;                              // [4][N*N][Kp] prolongation blocks (on the coarse level, FP32)
  DBuf<double> mg_x, mg_b, mg_r;                 // V-cycle work vectors (N * Kp)
  DBuf<float> E32, Pinv32;                       // FP32 copies read by the row-kernel smoother (small levels)
  DBuf<uint2> Eh;                                // packed FP16 copy of E (4 values per uint2), scaled per element
  DBuf<float> Escale;                            // per-element scale of Eh
  DBuf<uint2> Ph;                                // packed FP16 P^-1, scaled per element (Pscale)
  DBuf<float> Pscale;
  DBuf<double> mg_s;                             // V-cycle ping-pong partner of x (fused smoother)
  DBuf<double> mg_zero;                          // zeros (Chebyshev eigenvalue estimate)
  double cheb_lmax = 0.0;                        // estimated largest eigenvalue of P^-1 S_c (0: not yet)
  // dense coarsest level (ldg_dense.cu): -S_c as a column-major n x n matrix,
  // its LU and inverse; dense_level on the top handle (0: none)
  int dense_level = 0;
  // strip teams: the whole coarsest strip level replicated on every rank as a
  // one-rank mesh with a dense inverse (top handle; ldg_team.cu replica_solve)
  std::unique_ptr<Handle> replica;
  int replica_level = 0;                         // the strip level it replaces (0: none)
  int dn_n = 0;
  DBuf<double> dn_A, dn_inv, dn_X, dn_T, dn_zero, dn_work, dn_T2, dn_X2, dn_res;
  DBuf<int> dn_ipiv, dn_info, dn_cnt;
  DBuf<double> dn_part;                          // GEMV partial sums (deterministic split reduction)
  void* dn_solver = nullptr;                     // cusolverDnHandle_t
  void* dn_blas = nullptr;                       // cublasHandle_t (Newton-Schulz refinement)
  double* dn_res_host = nullptr;                 // pinned: last Newton-Schulz residual
  bool dn_valid = false;                         // dn_inv inverts a recent operator (same wm, dt)
  double dn_dt = 0.0, dn_wm = 0.0;
  DBuf<double> gm_V, gm_Z;                       // FGMRES basis and preconditioned basis ((m+1) and m vectors)
  int gm_m = 0, gm_req = 0;  // basis length in use, restart length it was sized for
  bool mg_f32 = true;                            // smoother on FP32 copies (precond 2) or FP64 (3)
  bool mg_ready = false;
  struct VGraph {                                // a captured V-cycle (CUDA graph)
    cudaGraphExec_t exec = nullptr;
    const double* b = nullptr;
    double* x = nullptr;
    double wm = 0.0, dt = 0.0;
    int64_t kernels = 0;
  };
  std::vector<VGraph> vgraphs;

  // strip decomposition of FK meshes: this handle owns element
  // columns [strip_a, strip_b) of FK(dim); local numbering is owned lowers
  // ((ix-a)*dim+iy), owned uppers (W*dim + ...), then the ghost uppers of
  // column a-1 and the ghost lowers of column b (one halo column per side).
  // Vertex (ix, iy) of this level is vertex (ix*stride, iy*stride) of the
  // finest mesh FK(dim_fine), so every level and rank regenerates identical
  // (jittered) coordinates from the same splitmix64 stream.
  int strip_a = 0, strip_b = 0;
  int ghost_left = 0, ghost_right = 0;  // ghost element counts (dim or 0)
  int stride = 1, dim_fine = 0;
  double jitter = 0.0;
  uint64_t seed = 0;
  int strip_w() const { return strip_b - strip_a; }
  long own_left_off() const { return 0; }                                                // lowers of column a
  long own_right_off() const { return static_cast<long>(2 * strip_w() - 1) * dim; }     // uppers of column b-1
  long ghost_left_off() const { return 2L * strip_w() * dim; }
  long ghost_right_off() const { return 2L * strip_w() * dim + ghost_left; }

  DevMesh mesh() const { return DevMesh{K, Kg, Kp, geom.ptr, nbr.ptr, nbrn.ptr, kind.ptr}; }
  long vec_len() const { return static_cast<long>(N) * Kp; }
  const double* rule_ptr() const { return rule_shared ? rule_shared : rule_elem.ptr; }
  int rule_R() const { return rule_shared ? rule_shared_R : rule_elem_R; }
};

// A group of ranks driven in lockstep: the local ranks of this process
// (one per GPU in a real multi-GPU run, or several "virtual" ranks sharing
// one GPU and one stream, used to validate the decomposition on one device)
// plus the NCCL communicator to remote ranks.  Halo values of local
// neighbours move with device copies, of remote ones with ncclSend/Recv;
// dot products are summed over local ranks, then ncclAllReduce'd.
struct Team {
  std::vector<std::unique_ptr<Handle>> ranks;
  int size = 1;        // global rank count
  int first = 0;       // global rank of ranks[0]
  void* nccl = nullptr;  // ncclComm_t when size > local ranks
  bool owns_nccl = false;
  cudaStream_t stream = nullptr;
  DBuf<double> send_l, send_r, recv_l, recv_r;  // NCCL halo staging
  cudaStream_t comm_stream = nullptr;           // NCCL halo exchange, overlapping the interior elements
  cudaEvent_t comm_ev[2] = {};                  // packed (main -> comm), landed (comm -> main)
  DBuf<double> rep_send, rep_recv;              // coarsest-level gather (replicated dense solve)
  DBuf<double> red_all;                         // allreduce scratch
  double* red_host = nullptr;                   // pinned
  double* gs_host = nullptr;                    // pinned: FGMRES Gram-Schmidt slots (kMaxRed x (2 kMaxRed + 1))
  cudaEvent_t gs_ev[2] = {};                    // completion of FGMRES iterations j (ping-pong)
  cudaStream_t in_stream = nullptr;             // host-buffer state upload, overlapping assembly + setup
  cudaStream_t setup_stream[2] = {};            // multigrid setup of level 0 / of the coarse levels, overlapping
  cudaEvent_t setup_ev[3] = {};                 // the right-hand side (team_solve): fork, two joins
  bool setup_pending = false;
  cudaEvent_t in_ev[4] = {};                    // [0] call start, [1] state uploaded, [2] Y final, [3] state downloaded
  bool y_pending = false;                       // team_solve waits for in_ev[1] before reading Y
  // host-buffer time loop, one rank: the last step's state leaves for the caller's buffer on
  // in_stream as soon as the flux recovery has written it, under the residual-contract check
  double* early_out = nullptr;
  bool early_out_sent = false;
  std::string err;
  Handle& h0() { return *ranks[0]; }
  const Handle& h0() const { return *ranks[0]; }
  int nlocal() const { return static_cast<int>(ranks.size()); }
  Handle* local(int global_rank) {
    const int i = global_rank - first;
    return (i >= 0 && i < nlocal()) ? ranks[i].get() : nullptr;
  }
};

// Launch with programmatic stream serialisation (PDL): the kernel must call
// pdl_wait() before reading what its predecessor wrote (ldg_device.cuh).
// Used for the latency-bound multigrid kernels; LDG_PDL=0 disables it.
bool pdl_enabled();
void launch_fill_hash(Handle& h, double* v);  // fixed pseudo-random vector
bool debug_nan();  // LDG_DEBUG_NAN=1
int debug_count_nonfinite(cudaStream_t st, const void* v, long n, bool half, const char* what);
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LDG_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// ---- launchers (defined in the .cu files) ----------------------------------
// mesh (ldg_mesh.cu)
void build_square_mesh(Handle& h, int dim, double jitter, uint64_t seed);
// strip [a, b) of FK(dim) (level with vertex stride `stride` of FK(dim_fine))
void build_square_strip(Handle& h, int dim, int a, int b, int stride, int dim_fine, double jitter, uint64_t seed);
void build_general_mesh(Handle& h, const double* coords, int nv, const int* v0t, int nt, const int* id_e0t);

// assembly (ldg_assemble.cu)
// kModeE: all 8 blocks [m][s] (exports); kModeEdiag: the diagonal blocks
// [m] the solver stores (off-diagonal ones are matrix-free, ldg_offdiag.cuh)
enum AsmMode { kModeE = 0, kModeG = 1, kModeR = 2, kModeRD = 3, kModeEdiag = 4 };
enum StaticMode { kStB = 0, kStS = 1, kStM = 2, kStH = 3, kStQ = 4, kStQN = 5, kStSint = 6, kStSD = 7 };
void launch_project(Handle& h, const ldg_coeff& fn, double t, const double* rule_dev, int R, double* out,
                    int count);
void launch_rhs(Handle& h, double t);
void launch_rhs_which(Handle& h, double t, int which, double* out);
void launch_project_df(Handle& h, double t, const double* rule_dev, int R);
void launch_assemble(Handle& h, int mode, double* out);
void launch_static(Handle& h, int mode, double* out);
void upload_rule(Handle& h, int q_ord, DBuf<double>& buf, int* R);

// field post-processing (ldg_fields.cu; fields.hpp:84-123)
void launch_l2err(Handle& h, const double* rule, int R, const ldg_coeff& f, double t, const double* u,
                  double* out);  // out (Kp plane): per-element error, owned-entry self-dot = squared error
int lagrange_nodes(int p);     // 3 (p <= 1) or 6 output nodes per element
void upload_lagrange_phi(Handle& h, DBuf<double>& buf);
void launch_lagrange(Handle& h, const double* phi, const double* u, double* out);  // out: K x nodes k-major

// solver (ldg_solve.cu)
// [k0, k1): owned element range (default all; thread-per-element levels only)
void launch_stage1(Handle& h, const double* vz, double sigma, const double* x, double tau, double* tout, int k0 = 0,
                   int k1 = -1);
void launch_stage2(Handle& h, const double* x, double alpha_m, double beta_s, const double* tz, double gamma_e,
                   const double* w, double delta, double* y, int k0 = 0, int k1 = -1);
void launch_full_apply(Handle& h, const double* Y, double wm, double dt, double* out);
void launch_bjac_setup(Handle& h, double wm, double dt);
void launch_bjac_apply(Handle& h, const double* x, double* y);
void launch_axpby(Handle& h, long n, double a, const double* x, double b, double* y);
// out = Krylov start from C^n (c) and the history (ldg_vec.cu k_extrap)
// w[o - 1][j]: Lagrange weights of order o for c (j = 0) and c_j (j >= 1)
void launch_extrap(Handle& h, long n, int order, const double (*w)[kExtrapMax + 1], const double* c,
                   const double* const* hist_vec, int* hist, const int* same, double* out);
void launch_hist_shift(Handle& h, long n, const double* c, double* const* hist_vec, int* hist);
void launch_same(Handle& h, long n, const double* a, const double* b, int* same, cudaStream_t stream);
void launch_dots(Handle& h, long n, int ndots, const double* const* xs, const double* const* ys, double* out_host);
void launch_soa_to_kmajor(Handle& h, const double* soa, int nvec, double* kmajor_dev, cudaStream_t stream = nullptr);
void launch_kmajor_to_soa(Handle& h, const double* kmajor_dev, int nvec, double* soa, cudaStream_t stream = nullptr);

void launch_bjac_axpy(Handle& h, const double* x, double omega, double beta, double* y);
void launch_bjac_axpy_f32(Handle& h, const double* x, double omega, double beta, double* y);
void launch_to_f32(Handle& h, long n, const double* src, float* dst);
void launch_bjac(Handle& h, double wm, double dt, int out_kind);     // ldg_bjac.cu: 0 Pinv, 1 Pinv32, 3 Ph
void launch_bjac_setup_f32_from64(Handle& h, double wm, double dt);  // Pinv32 from E (FP64)
bool level_uses_rows(const Handle& h);
bool level_is_small(const Handle& h);

// fused mixed-precision smoother (ldg_smooth.cu)
long packed_p_quads(int p);                                           // float4 quads of one packed P^-1 block
void smooth_pack_alloc(Handle& h);  // Eh / Escale of the level (filled by launch_bjac, kind 3)
void smooth_dtraces(Handle& h);     // d_h at the edge points for the trace-form smoother
// chained: x is the output of the preceding smooth_stage2 (mode 1) launch on this level
void smooth_stage1(Handle& h, const double* x, int k0 = 0, int k1 = -1, bool chained = false);  // tz = M^-1 B x (FP32 arithmetic)
// mode 0: out = b - S_c x;  mode 1: out = x + omega P^-1 (b - S_c x)
// cheb_beta != 0: Chebyshev step out <- x + omega P^-1 r + cheb_beta (x - out_old)
// (out_old = x_{k-1}, taken as 0 when prev_zero)
void smooth_stage2(Handle& h, int mode, const double* x, const double* b, double wm, double dt, double omega,
                   double* out, double cheb_beta = 0.0, int prev_zero = 0, int k0 = 0, int k1 = -1);
int smooth_trace_min_p();  // degrees >= this exchange edge traces between the smoother's stages
void smooth_zero(Handle& h, const double* b, double omega, double* out);  // out = omega P^-1 b
// the same three operations for small levels (ldg_small.cu; E32 / Pinv32 SoA copies)
void small_stage1(Handle& h, const double* x);
void small_stage2(Handle& h, int mode, const double* x, const double* b, double wm, double dt, double omega,
                  double* out);
void small_zero(Handle& h, const double* b, double omega, double* out);

// row-parallel operator kernels (ldg_rows.cu), used by the launchers above
void rows_stage1(Handle& h, const double* vz, double sigma, const double* x, double tau, double* tout);
template <typename TE>
void rows_stage2(Handle& h, const TE* E, const double* x, double alpha, double beta, const double* tz, double gamma,
                 const double* w, double delta, double* y);
template <typename TP>
void rows_bjac(Handle& h, const TP* Pinv, const double* x, double omega, double beta, double* y);
void launch_lincomb3(Handle& h, long n, double a, const double* x, double b, const double* y, double c,
                     const double* z, double* out);
void launch_mdots_async(Handle& h, int nv, const double* const* v, const double* w);
void launch_maxpy(Handle& h, int nv, const double* const* v, const double* c, double alpha, double* w);
void launch_mdots_to(Handle& h, int nv, const double* const* v, const double* w, double* out);  // results on device
void launch_maxpy_dev(Handle& h, int nv, const double* const* v, const double* c, bool final, double* w, double* w2,
                      double* hn_out);  // device coefficients (Gram-Schmidt without a host round trip)

// per-rank assembly step (ldg_vec.cu)
void assemble_step(Handle& h, double t);
size_t reduction_scratch();

// team driver (ldg_team.cu)
void team_assemble(Team& T, double t);
int team_solve(Team& T, double wm, double dt, const ldg_solver_opts& o, ldg_step_stats* st);
void team_full_apply(Team& T, double wm, double dt);        // full_y = (W + dt A) Y, halos refreshed
void team_schur_apply_c(Team& T, double wm, double dt);     // kr_v = S_c C (kernel timing)
int team_time_mg(Team& T, double wm, double dt, int reps, double* ms_vcycle, double* ms_level, int max_levels);
void team_sweep_s2_prepare(Team& T, double wm, double dt);  // multigrid set up, level-0 stage 1 done
void team_sweep_s2(Team& T, double wm, double dt);          // one level-0 smoother stage-2 launch
int team_s2_per_vcycle(Team& T);                            // level-0 stage-2 launches per V-cycle
double team_sum_sq(Team& T, const std::function<const double*(Handle&)>& v);  // owned entries, all ranks

void init_handle_tables(Handle& h, int p);  // reference tables + element rule of degree p (ldg_capi.cu)

// multigrid (ldg_mg.cu)
int mg_depth(int dim, int team_size);
// dense coarsest level (ldg_dense.cu)
long dense_max();
bool dense_candidate(const Handle& L);
bool replica_candidate(const Handle& coarsest);  // strip level whose global mesh can be solved densely
void launch_rep_scatter(Handle& R, int size, int W, const double* recv);  // packed owned rows -> R.mg_b
void launch_rep_gather(Handle& R, Handle& L, int q, double* x);           // R.mg_x -> owned rows of strip q
void dense_alloc(Handle& L);
void dense_release(Handle& L);
void dense_setup(Handle& L, double wm, double dt, bool f32);
void dense_solve(Handle& L, const double* b, double* x);
bool mg_build(Handle& h, int team_size);                    // false: no hierarchy for this mesh
void mg_setup_step(Handle& h, double t, double wm, double dt, bool f32);  // per step: coarse E, block-Jacobi
void mg_setup_top(Handle& h, double wm, double dt, bool f32);               // level 0's part of mg_setup_step
void mg_setup_coarse(Handle& h, double t, double wm, double dt, bool f32);  // the coarse levels' part
void mg_restrict(Handle& fine, Handle& coarse);             // coarse.mg_b = P^T fine.mg_r
void mg_prolong_add(Handle& fine, Handle& coarse, double* x);  // x += P coarse.mg_x
int mg_levels(const Handle& h);
void mg_release(Handle& h);  // destroys captured graphs

}  // namespace ldgb
