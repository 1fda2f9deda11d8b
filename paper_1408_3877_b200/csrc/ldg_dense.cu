// Dense solve on the coarsest multigrid level.
//
// Below ~32^2 elements a multigrid level is a chain of latency-bound phases:
// each of the ~11 kernels of a level's V(2,2) visit costs 3-4 us whatever the
// level size (a few dependent L2 round trips plus the launch), so the 8^2,
// 4^2 and 2^2 levels of the 256^2 hierarchy cost ~30 kernels / ~100 us per
// V-cycle.  Here the hierarchy stops at the first level whose operator has at
// most dense_max() unknowns (8^2 at degree 1, 2: 384 / 768 unknowns; 16^2 at
// degree 0): per time step its Schur operator is formed column by column
// (S_c e_c with the level's own stage kernels, ldg_small.cu) and inverted on
// the setup stream, and every V-cycle applies the inverse with one
// matrix-vector kernel.  Single rank only: a strip team keeps the smoothed
// coarsest level.
//
// Inversion: the operator changes by a few per cent per time step (d(t)), so
// the previous step's inverse X is refined by two Newton-Schulz steps
// X <- X (2I - B X) (4 DGEMMs, cuBLAS), quadratically convergent: an
// initial ||I - B X|| of 3e-2 ends at ~1e-6.  The first step, and any step
// after one whose Newton-Schulz residual (checked on the device, read back one
// step later without a synchronisation) exceeded 1e-2, inverts from scratch
// with a pivoted LU (cuSOLVER getrf / getrs against the identity: ~1.5-2.7 ms
// at 512-768 unknowns, latency-bound).
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <cstdlib>

#include "ldg_internal.hpp"

namespace ldgb {

void small_dense_columns(Handle& h, const double* X, double* Tz, const double* zero, double wm, double dt, double* out,
                         int ncols);

namespace {

#define LDG_CUSOLVER(call)                                                                        \
  do {                                                                                            \
    cusolverStatus_t s_ = (call);                                                                 \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                            \
      throw Error(LDG_ECUDA, std::string(#call) + ": cusolver status " + std::to_string(s_));    \
  } while (0)

// *out = max |T - I| (T = 2I - B X: the Newton-Schulz residual I - B X)
__global__ void k_ns_residual(long n, const double* __restrict__ t, double* out) {
  double m = 0.0;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n * n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    m = fmax(m, fabs(t[i] - ((i % (n + 1) == 0) ? 1.0 : 0.0)));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(out), static_cast<unsigned long long>(__double_as_longlong(m)));
}

// B[u][u] = 1 for the unknowns of padding elements (u = i Kp + k, k >= K):
// their columns and rows are otherwise zero
__global__ void k_pad_identity(int N, int K, long Kp, double* __restrict__ a) {
  const long n = N * Kp;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < N * (Kp - K);
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    const long u = (t / (Kp - K)) * Kp + K + t % (Kp - K);
    a[u * n + u] = 1.0;
  }
}

__global__ void k_identity(long n, double* __restrict__ a) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n * n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    a[i] = (i % (n + 1) == 0) ? 1.0 : 0.0;
}

// y = alpha A x, A column-major n x n (n a multiple of 32): 32 rows x
// n / kGemvSplit columns per block (the columns of a block split over its 8
// warps, partial sums reduced in shared memory); the last block of a row
// group to finish (arrival counter, reset by it for the next replay) adds the
// kGemvSplit partials in a fixed order, so the result is deterministic.  The
// inverse (1.2-2 MB) comes from HBM once per V-cycle: 12 blocks over all
// columns streamed it at a few hundred GB/s, 12 x 8 blocks fill the GPU.
constexpr int kGemvSplit = 8;
__global__ void __launch_bounds__(256) k_dense_gemv(int n, const double* __restrict__ a, const double* x,
                                                    double alpha, double* y, double* part_g, int* arrivals) {
  __shared__ double part[8][33];
  __shared__ bool last;
  pdl_wait();
  pdl_trigger();
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  const int row = blockIdx.x * 32 + lx;
  const int c0 = blockIdx.y * (n / kGemvSplit), c1 = blockIdx.y + 1 == kGemvSplit ? n : c0 + n / kGemvSplit;
  double s = 0.0;
  for (int c = c0 + ly; c < c1; c += 8) s = fma(a[static_cast<long>(c) * n + row], x[c], s);
  part[ly][lx] = s;
  __syncthreads();
  if (ly == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += part[w][lx];
    part_g[static_cast<long>(blockIdx.y) * n + row] = t;
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int done = atomicAdd(arrivals + blockIdx.x, 1);
    last = done == kGemvSplit - 1;
    if (last) arrivals[blockIdx.x] = 0;
  }
  __syncthreads();
  if (last && ly == 0) {
    __threadfence();
    double t = 0.0;
    for (int b = 0; b < kGemvSplit; ++b) t += __ldcg(part_g + static_cast<long>(b) * n + row);
    y[row] = alpha * t;
  }
}

// global FK id of local element k of strip q (W columns from q W; local
// order: owned lowers then owned uppers, mesh.hpp:237-242 / ldg_mesh.cu)
__device__ __forceinline__ int strip_gid(int q, int W, int dim, int k) {
  const int a = q * W;
  if (k < W * dim) return (a + k / dim) * dim + k % dim;
  const int kk = k - W * dim;
  return dim * dim + (a + kk / dim) * dim + kk % dim;
}

// the packed owned rows of all ranks ([q][i][k], k < 2 W dim) -> global SoA
__global__ void k_rep_scatter(int size, int W, int dim, int N, long KpR, const double* __restrict__ recv,
                              double* __restrict__ out) {
  const long Kown = 2L * W * dim, n = static_cast<long>(size) * N * Kown;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    const int q = static_cast<int>(t / (N * Kown));
    const long rem = t % (N * Kown);
    const int i = static_cast<int>(rem / Kown), k = static_cast<int>(rem % Kown);
    out[i * KpR + strip_gid(q, W, dim, k)] = recv[t];
  }
}

// global SoA -> the owned rows of strip q (plane stride Kp)
__global__ void k_rep_gather(int q, int W, int dim, int N, long KpR, long Kp, const double* __restrict__ xr,
                             double* __restrict__ x) {
  const long Kown = 2L * W * dim, n = static_cast<long>(N) * Kown;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(t / Kown), k = static_cast<int>(t % Kown);
    x[i * Kp + k] = xr[i * KpR + strip_gid(q, W, dim, k)];
  }
}

}  // namespace

void launch_rep_scatter(Handle& R, int size, int W, const double* recv) {
  k_rep_scatter<<<64, 256, 0, R.stream>>>(size, W, R.dim, R.N, R.Kp, recv, R.mg_b.ptr);
  LDG_CUDA(cudaGetLastError());
  ++R.launches;
}

void launch_rep_gather(Handle& R, Handle& L, int q, double* x) {
  k_rep_gather<<<64, 256, 0, R.stream>>>(q, L.strip_w(), R.dim, R.N, R.Kp, L.Kp, R.mg_x.ptr, x);
  LDG_CUDA(cudaGetLastError());
  ++R.launches;
}

// largest dense coarsest level (unknowns); LDG_DENSE_MAX for tuning runs, 0 off
long dense_max() {
  static const long v = [] {
    const char* e = std::getenv("LDG_DENSE_MAX");
    return e ? std::atol(e) : 800L;
  }();
  return v;
}

// Degree <= 1 only: with the degree-2 levels of a p = 4 hierarchy the exact
// solve of the rediscretised (non-Galerkin) coarse operator raised the FGMRES
// iterations (9.6 -> 10.4 per step on C2, at 8^2 and at 4^2 alike), while at
// degree 0 / 1 it lowered them (p = 0..3: 10.8 / 8.0 / 8.2 / 8.2 -> 10.4 /
// 7.6 / 8.0 / 7.6; ms per step 4.67 / 4.73 / 6.62 / 11.25 -> 3.94 / 4.13 /
// 6.11 / 10.13).
bool dense_candidate(const Handle& L) {
  const long n = static_cast<long>(L.N) * L.Kp;  // padding elements carry identity rows
  return !L.mg_pcoarse && L.size == 1 && L.p <= 1 && n <= dense_max();
}

// Strip teams: the coarsest level of a truncated strip hierarchy (every
// rank keeps a column) was smoothed with 2 dim sweeps, each with a halo
// exchange, and left the distributed solves ~2x the single-rank iterations.
// Its global mesh is tiny (2 dim^2 elements), so every rank holds it whole
// (a one-rank Handle regenerated from the same vertex stream) with a dense
// inverse; the V-cycle gathers the coarsest right-hand side from all ranks
// (ncclAllGather of the owned rows), solves redundantly, and keeps its rows.
// Degree <= 2 (the alternative here is the smoothed truncated level).
bool replica_candidate(const Handle& C) {
  const long K = 2L * C.dim * C.dim, n = static_cast<long>(C.N) * K;
  return C.size > 1 && C.dim > 0 && C.p <= 2 && K % 32 == 0 && n <= dense_max();
}

void dense_alloc(Handle& L) {
  const long n = static_cast<long>(L.N) * L.Kp;
  L.dn_n = static_cast<int>(n);
  L.dn_A.alloc(n * n, &L.bytes);
  L.dn_inv.alloc(n * n, &L.bytes);
  L.dn_X.alloc(n * n, &L.bytes);
  L.dn_T.alloc(2 * n * n, &L.bytes);
  L.dn_zero.alloc(n, &L.bytes);
  L.dn_ipiv.alloc(n, &L.bytes);
  L.dn_info.alloc(1, &L.bytes);
  cusolverDnHandle_t s = nullptr;
  LDG_CUSOLVER(cusolverDnCreate(&s));
  L.dn_solver = s;
  int lwork = 0;
  LDG_CUSOLVER(cusolverDnDgetrf_bufferSize(s, L.dn_n, L.dn_n, L.dn_A.ptr, L.dn_n, &lwork));
  L.dn_work.alloc(static_cast<size_t>(lwork > 0 ? lwork : 1), &L.bytes);
  L.dn_T2.alloc(n * n, &L.bytes);
  L.dn_part.alloc(kGemvSplit * n, &L.bytes);
  L.dn_cnt.alloc(n / 32, &L.bytes);  // zeroed: arrival counters of k_dense_gemv
  L.dn_X2.alloc(n * n, &L.bytes);
  L.dn_res.alloc(1, &L.bytes);
  cublasHandle_t b = nullptr;
  if (cublasCreate(&b) != CUBLAS_STATUS_SUCCESS) throw Error(LDG_ECUDA, "cublasCreate failed");
  L.dn_blas = b;
  if (!L.dn_res_host) LDG_CUDA(cudaMallocHost(&L.dn_res_host, sizeof(double)));
  *L.dn_res_host = 1.0;
  L.dn_valid = false;
  k_identity<<<256, 256, 0, L.stream>>>(n, L.dn_X.ptr);
  LDG_CUDA(cudaGetLastError());
  LDG_CUDA(cudaStreamSynchronize(L.stream));
}

void dense_release(Handle& L) {
  if (L.dn_solver) cusolverDnDestroy(static_cast<cusolverDnHandle_t>(L.dn_solver));
  L.dn_solver = nullptr;
  if (L.dn_blas) cublasDestroy(static_cast<cublasHandle_t>(L.dn_blas));
  L.dn_blas = nullptr;
  if (L.dn_res_host) cudaFreeHost(L.dn_res_host);
  L.dn_res_host = nullptr;
}

// per step, after the level's operator copies (E32) are built: B = -S_c
// column by column, B = LU, inverse = B^-1 (getrs against the identity)
void dense_setup(Handle& L, double wm, double dt, bool f32) {
  const int n = L.dn_n;
  if (!f32 || !level_uses_rows(L)) {  // no FP32 SoA copy of E on this level: make one for the column kernels
    const long nn = 2L * L.N * L.N * L.Kp;
    if (!L.E32.ptr) L.E32.alloc(nn, &L.bytes);
    launch_to_f32(L, nn, L.E.ptr, L.E32.ptr);
  }
  small_dense_columns(L, L.dn_X.ptr, L.dn_T.ptr, L.dn_zero.ptr, wm, dt, L.dn_A.ptr, n);
  if (L.Kp > L.K) {
    k_pad_identity<<<32, 256, 0, L.stream>>>(L.N, L.K, L.Kp, L.dn_A.ptr);
    LDG_CUDA(cudaGetLastError());
    ++L.launches;
  }
  const size_t bytes = sizeof(double) * n * n;
  // the previous step's Newton-Schulz residual (its pinned copy completed
  // with that step) decides between refinement and a fresh factorisation
  if (L.dn_valid && *L.dn_res_host <= 1e-2 && dt == L.dn_dt && wm == L.dn_wm) {
    auto b = static_cast<cublasHandle_t>(L.dn_blas);
    if (cublasSetStream(b, L.stream) != CUBLAS_STATUS_SUCCESS) throw Error(LDG_ECUDA, "cublasSetStream failed");
    const double m1 = -1.0, two = 2.0, one = 1.0, zero = 0.0;
    LDG_CUDA(cudaMemsetAsync(L.dn_res.ptr, 0, sizeof(double), L.stream));
    for (int it = 0; it < 2; ++it) {
      // T2 = 2I - B X;  X <- X T2
      LDG_CUDA(cudaMemcpyAsync(L.dn_T2.ptr, L.dn_X.ptr, bytes, cudaMemcpyDeviceToDevice, L.stream));
      if (cublasDgemm(b, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &m1, L.dn_A.ptr, n, L.dn_inv.ptr, n, &two, L.dn_T2.ptr,
                      n) != CUBLAS_STATUS_SUCCESS)
        throw Error(LDG_ECUDA, "cublasDgemm failed");
      if (it == 1) {
        k_ns_residual<<<64, 256, 0, L.stream>>>(n, L.dn_T2.ptr, L.dn_res.ptr);
        LDG_CUDA(cudaGetLastError());
        ++L.launches;
      }
      if (cublasDgemm(b, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, L.dn_inv.ptr, n, L.dn_T2.ptr, n, &zero, L.dn_X2.ptr,
                      n) != CUBLAS_STATUS_SUCCESS)
        throw Error(LDG_ECUDA, "cublasDgemm failed");
      LDG_CUDA(cudaMemcpyAsync(L.dn_inv.ptr, L.dn_X2.ptr, bytes, cudaMemcpyDeviceToDevice, L.stream));
    }
    LDG_CUDA(cudaMemcpyAsync(L.dn_res_host, L.dn_res.ptr, sizeof(double), cudaMemcpyDeviceToHost, L.stream));
    return;
  }
  auto s = static_cast<cusolverDnHandle_t>(L.dn_solver);
  LDG_CUSOLVER(cusolverDnSetStream(s, L.stream));
  LDG_CUDA(cudaMemcpyAsync(L.dn_T2.ptr, L.dn_A.ptr, bytes, cudaMemcpyDeviceToDevice, L.stream));  // B kept for refinement
  LDG_CUSOLVER(cusolverDnDgetrf(s, n, n, L.dn_T2.ptr, n, L.dn_work.ptr, L.dn_ipiv.ptr, L.dn_info.ptr));
  LDG_CUDA(cudaMemcpyAsync(L.dn_inv.ptr, L.dn_X.ptr, bytes, cudaMemcpyDeviceToDevice, L.stream));
  LDG_CUSOLVER(cusolverDnDgetrs(s, CUBLAS_OP_N, n, n, L.dn_T2.ptr, n, L.dn_ipiv.ptr, L.dn_inv.ptr, n, L.dn_info.ptr));
  L.dn_valid = true;
  L.dn_dt = dt;
  L.dn_wm = wm;
  *L.dn_res_host = 0.0;
}

// x = S_c^-1 b = -(B^-1) b on the dense level
void dense_solve(Handle& L, const double* b, double* x) {
  launch_pdl(k_dense_gemv, dim3(L.dn_n / 32, kGemvSplit), dim3(256), 0, L.stream, L.dn_n,
             static_cast<const double*>(L.dn_inv.ptr), b, -1.0, x, L.dn_part.ptr, L.dn_cnt.ptr);
  LDG_CUDA(cudaGetLastError());
  ++L.launches;
}

}  // namespace ldgb
