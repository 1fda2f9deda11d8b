// K7 vector kernels of the Krylov solve: fused linear combinations,
// deterministic dot-product reductions (fixed grid, fixed order; owned
// entries only, so strip ghosts never count twice), layout conversion
// between the element-interleaved device vectors and the reference's
// k-major host vectors, and the per-rank assembly step.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ldg_internal.hpp"

namespace ldgb {

namespace {

inline unsigned grid_of(long n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

__global__ void k_lincomb3(long n, double a, const double* x, double b, const double* y, double c, const double* z,
                           double* out) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    double v = a * x[i];
    if (y) v += b * y[i];
    if (z) v += c * z[i];
    out[i] = v;
  }
}

__global__ void k_axpby(long n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    y[i] = a * x[i] + b * y[i];
}

constexpr int kRedBlocks = 296;  // 2 x 148 SMs
constexpr int kMaxDots = 4;
constexpr int kMdotChunk = 8;    // dots per block row of the multi-dot kernel

struct DotArgs {
  const double* x[kMaxDots];
  const double* y[kMaxDots];
};

// Deterministic two-pass reduction: fixed grid, fixed per-block order.
__global__ void __launch_bounds__(256) k_dots_partial(long n, int nd, DotArgs a, double* __restrict__ part) {
  double s[kMaxDots] = {0.0, 0.0, 0.0, 0.0};
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    for (int d = 0; d < nd; ++d) s[d] += a.x[d][i] * a.y[d][i];
  __shared__ double sh[kMaxDots][8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int d = 0; d < nd; ++d) {
    double v = s[d];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sh[d][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < nd) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += sh[threadIdx.x][w];
    part[threadIdx.x * kRedBlocks + blockIdx.x] = v;
  }
}

// dots over planes j < N, elements k < K of vectors laid out [j][Kp]
__global__ void __launch_bounds__(256) k_dots_owned(int N, long Kp, int K, int nd, DotArgs a,
                                                    double* __restrict__ part) {
  double s[kMaxDots] = {0.0, 0.0, 0.0, 0.0};
  for (int j = 0; j < N; ++j)
    for (long k = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; k < K;
         k += static_cast<long>(gridDim.x) * blockDim.x) {
      const long i = j * Kp + k;
      for (int d = 0; d < nd; ++d) s[d] += a.x[d][i] * a.y[d][i];
    }
  __shared__ double sh[kMaxDots][8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int d = 0; d < nd; ++d) {
    double v = s[d];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sh[d][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < nd) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += sh[threadIdx.x][w];
    part[threadIdx.x * kRedBlocks + blockIdx.x] = v;
  }
}

// (v_d, w) for d < nv over the owned entries; block row y handles dots
// [8y, 8y + 8) (w re-read per row, from L2 for the small row counts used)
struct MDotArgs {
  const double* v[kMaxRed];
};
__global__ void __launch_bounds__(256) k_mdot_owned(int N, long Kp, int K, int nv, MDotArgs a,
                                                    const double* __restrict__ w, double* __restrict__ part) {
  const int d0 = blockIdx.y * kMdotChunk;
  const int nd = min(kMdotChunk, nv - d0);
  double s[kMdotChunk];
#pragma unroll
  for (int d = 0; d < kMdotChunk; ++d) s[d] = 0.0;
  // owned entries: planes j < N, elements k < K (no division in the loop)
  for (int j = 0; j < N; ++j)
    for (long k = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; k < K;
         k += static_cast<long>(gridDim.x) * blockDim.x) {
      const long i = j * Kp + k;
      const double wi = w[i];
#pragma unroll
      for (int d = 0; d < kMdotChunk; ++d)
        if (d < nd) s[d] = fma(a.v[d0 + d][i], wi, s[d]);
    }
  __shared__ double sh[kMdotChunk][8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int d = 0; d < kMdotChunk; ++d) {
    double v = s[d];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sh[d][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < nd) {
    double v = 0.0;
    for (int ww = 0; ww < 8; ++ww) v += sh[threadIdx.x][ww];
    part[(d0 + threadIdx.x) * kRedBlocks + blockIdx.x] = v;
  }
}

// (v_d, w) for d < nv when every entry of the vectors is owned (one rank,
// K == Kp: no ghosts, no padding): one flat 128-bit stream per vector, 16 dots
// per block row (w read at most twice for the FGMRES basis sizes), 512
// threads per block.  The (j, k) form above moves 64-bit values with a
// 1.73-iteration inner loop per plane at 256^2 and ran at ~2.4 TB/s.
constexpr int kMdotFlatChunk = 16;
__global__ void __launch_bounds__(512) k_mdot_flat(long n2, int nv, MDotArgs a, const double* __restrict__ w,
                                                   double* __restrict__ part) {
  const int d0 = blockIdx.y * kMdotFlatChunk;
  const int nd = min(kMdotFlatChunk, nv - d0);
  double s[kMdotFlatChunk];
#pragma unroll
  for (int d = 0; d < kMdotFlatChunk; ++d) s[d] = 0.0;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n2;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const double2 wi = w2[i];
#pragma unroll
    for (int d = 0; d < kMdotFlatChunk; ++d)
      if (d < nd) {
        const double2 v = reinterpret_cast<const double2*>(a.v[d0 + d])[i];
        s[d] = fma(v.x, wi.x, fma(v.y, wi.y, s[d]));
      }
  }
  __shared__ double sh[kMdotFlatChunk][16];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int d = 0; d < kMdotFlatChunk; ++d) {
    double v = s[d];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sh[d][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < nd) {
    double v = 0.0;
    for (int ww = 0; ww < 16; ++ww) v += sh[threadIdx.x][ww];
    part[(d0 + threadIdx.x) * kRedBlocks + blockIdx.x] = v;
  }
}

// w = alpha w + sum_d c_d v_d over the whole vector (n values)
struct MAxpyArgs {
  const double* v[kMaxRed];
  double c[kMaxRed];
};
__global__ void __launch_bounds__(256) k_maxpy(long n, int nv, MAxpyArgs a, double alpha, double* __restrict__ w) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    double acc = alpha == 0.0 ? 0.0 : alpha * w[i];
#pragma unroll 4
    for (int d = 0; d < nv; ++d) acc = fma(a.c[d], a.v[d][i], acc);
    w[i] = acc;
  }
}

// one warp per dot product: lane l sums partials l, l+32, ... then a fixed
// shuffle tree (deterministic; the former one-thread-per-dot loop over the
// 296 partials took ~17 us, twice per Krylov iteration)
__global__ void k_dots_final(int nd, const double* __restrict__ part, double* __restrict__ out) {
  const int d = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (d >= nd) return;
  double v = 0.0;
  for (int b = lane; b < kRedBlocks; b += 32) v += part[d * kRedBlocks + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) out[d] = v;
}

// Gram-Schmidt update with device-resident coefficients (no host round
// trip between the projection and the update):
//   FINAL 0: w -= sum_d c_d v_d
//   FINAL 1: w = (w - sum_d c_d v_d) / hn, hn = sqrt(c_nv - sum_d c_d^2) (the
//            norm of the updated w by Pythagoras: c_nv holds (w, w)); w2 (if
//            set) receives a copy; block 0 stores hn at *hn_out
template <int FINAL>
__global__ void __launch_bounds__(256) k_maxpy_dev(long n, int nv, MDotArgs a, const double* __restrict__ c,
                                                   double* __restrict__ w, double* __restrict__ w2,
                                                   double* __restrict__ hn_out) {
  __shared__ double s_c[kMaxRed];
  __shared__ double s_inv;
  for (int d = threadIdx.x; d < nv; d += blockDim.x) s_c[d] = -c[d];
  if (FINAL && threadIdx.x == 0) {
    double ss = c[nv];
    for (int d = 0; d < nv; ++d) ss = fma(-c[d], c[d], ss);
    const double hn = ss > 0.0 ? sqrt(ss) : 0.0;
    s_inv = hn > 0.0 ? 1.0 / hn : 0.0;
    if (blockIdx.x == 0) *hn_out = hn;
  }
  __syncthreads();
  // 128-bit stream (n even: N Kp, Kp a multiple of 32)
  const long n2 = n / 2;
  double2* wv = reinterpret_cast<double2*>(w);
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n2;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    double2 acc = wv[i];
#pragma unroll 4
    for (int d = 0; d < nv; ++d) {
      const double2 v = reinterpret_cast<const double2*>(a.v[d])[i];
      acc.x = fma(s_c[d], v.x, acc.x);
      acc.y = fma(s_c[d], v.y, acc.y);
    }
    if (FINAL) {
      acc.x *= s_inv;
      acc.y *= s_inv;
      if (w2) reinterpret_cast<double2*>(w2)[i] = acc;
    }
    wv[i] = acc;
  }
}

inline unsigned final_blocks(int nd) { return static_cast<unsigned>((nd + 7) / 8); }  // 8 warps per block

// SoA [nvec][N][Kp] <-> k-major [nvec][K][N]
__global__ void k_soa_to_kmajor(int K, int N, long Kp, int nvec, const double* __restrict__ soa,
                                double* __restrict__ km) {
  const long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  const long total = static_cast<long>(nvec) * K * N;
  if (idx >= total) return;
  const long v = idx / (static_cast<long>(K) * N);
  const long r = idx % (static_cast<long>(K) * N);
  const long k = r / N, j = r % N;
  km[idx] = soa[(v * N + j) * Kp + k];
}

__global__ void k_kmajor_to_soa(int K, int N, long Kp, int nvec, const double* __restrict__ km,
                                double* __restrict__ soa) {
  const long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  const long total = static_cast<long>(nvec) * K * N;
  if (idx >= total) return;
  const long v = idx / (static_cast<long>(K) * N);
  const long r = idx % (static_cast<long>(K) * N);
  const long k = r / N, j = r % N;
  soa[(v * N + j) * Kp + k] = km[idx];
}

#define LDG_DISPATCH_P(p, CALL) \
  switch (p) {                  \
    case 0: { CALL(0); break; } \
    case 1: { CALL(1); break; } \
    case 2: { CALL(2); break; } \
    case 3: { CALL(3); break; } \
    default: { CALL(4); break; } \
  }

__global__ void k_count_nonfinite(long n, const double* __restrict__ v, int* __restrict__ out) {
  int c = 0;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    c += isfinite(v[i]) ? 0 : 1;
  if (c) atomicAdd(out, c);
}

__global__ void k_count_nonfinite_h(long n, const __half* __restrict__ v, int* __restrict__ out) {
  int c = 0;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    c += isfinite(__half2float(v[i])) ? 0 : 1;
  if (c) atomicAdd(out, c);
}

}  // namespace

// LDG_DEBUG_NAN=1 (diagnostics): count non-finite values of a device array
// (synchronises the stream) and report them on stderr under `what`
bool debug_nan() {
  static const bool on = [] {
    const char* s = std::getenv("LDG_DEBUG_NAN");
    return s && std::atoi(s) != 0;
  }();
  return on;
}

int debug_count_nonfinite(cudaStream_t st, const void* v, long n, bool half, const char* what) {
  int* d = nullptr;
  int h = 0;
  LDG_CUDA(cudaMallocAsync(&d, sizeof(int), st));
  LDG_CUDA(cudaMemsetAsync(d, 0, sizeof(int), st));
  if (half)
    k_count_nonfinite_h<<<256, 256, 0, st>>>(n, static_cast<const __half*>(v), d);
  else
    k_count_nonfinite<<<256, 256, 0, st>>>(n, static_cast<const double*>(v), d);
  LDG_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, st));
  LDG_CUDA(cudaFreeAsync(d, st));
  LDG_CUDA(cudaStreamSynchronize(st));
  if (h) fprintf(stderr, "[ldg nan] %s: %d non-finite of %ld\n", what, h, n);
  return h;
}

namespace {
// a fixed pseudo-random vector in [-0.5, 0.5) on the owned entries (halo and
// padding slots zero: start of power iterations)
__global__ void k_fill_hash(long n, long Kp, int K, double* __restrict__ v) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    unsigned long long z = static_cast<unsigned long long>(i) + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    v[i] = i % Kp < K ? static_cast<double>(z >> 11) * 0x1.0p-53 - 0.5 : 0.0;
  }
}
}  // namespace

void launch_fill_hash(Handle& h, double* v) {
  k_fill_hash<<<kRedBlocks * 4, 256, 0, h.stream>>>(h.vec_len(), h.Kp, h.K, v);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

// programmatic dependent launch for the latency-bound multigrid kernels
bool pdl_enabled() { return true; }

void launch_lincomb3(Handle& h, long n, double a, const double* x, double b, const double* y, double c,
                     const double* z, double* out) {
  k_lincomb3<<<kRedBlocks * 4, 256, 0, h.stream>>>(n, a, x, b, y, c, z, out);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

// Krylov start of an implicit-Euler solve: Lagrange extrapolation in time of
// C^n (c) and the history C^{n-1..n-3} at the order min(order, hist[0]),
// dropped to the plain start c where *same == 0 (a host-buffer state that does
// not continue the last output); the order used goes to hist[1].
struct ExtrapArgs {
  double w[kExtrapMax][kExtrapMax + 1];
  const double* v[kExtrapMax];
};
__global__ void k_extrap(long n, int order, ExtrapArgs a, const double* __restrict__ c, int* hist,
                         const int* __restrict__ same, double* __restrict__ out) {
  int o = min(order, hist[0]);
  if (same && *same == 0) o = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) hist[1] = o;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    double r = c[i];
    if (o > 0) {
      const double* w = a.w[o - 1];
      r *= w[0];
      for (int j = 1; j <= o; ++j) r = fma(w[j], a.v[j - 1][i], r);
    }
    out[i] = r;
  }
}

// after a solve from C^n: the history moves down one slot and C^n enters
// slot 0; valid count hist[0] = 1 after a plain start, else one more
struct HistArgs {
  double* v[kExtrapMax];
};
__global__ void k_hist_shift(long n, const double* __restrict__ c, HistArgs a, int* hist) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    for (int j = kExtrapMax - 1; j > 0; --j) a.v[j][i] = a.v[j - 1][i];
    a.v[0][i] = c[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) hist[0] = hist[1] == 0 ? 1 : min(hist[0] + 1, kExtrapMax);
}

// *same = 0 unless a[i] == b[i] for every i (bitwise state continuity)
__global__ void k_same(long n, const double* __restrict__ a, const double* __restrict__ b, int* same) {
  bool eq = true;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    eq &= __double_as_longlong(a[i]) == __double_as_longlong(b[i]);
  if (__syncthreads_and(eq) == 0 && threadIdx.x == 0) *same = 0;
}

void launch_extrap(Handle& h, long n, int order, const double (*w)[kExtrapMax + 1], const double* c,
                   const double* const* hist_vec, int* hist, const int* same, double* out) {
  ExtrapArgs a{};
  for (int o = 0; o < kExtrapMax; ++o)
    for (int j = 0; j <= kExtrapMax; ++j) a.w[o][j] = w[o][j];
  for (int j = 0; j < kExtrapMax; ++j) a.v[j] = hist_vec[j];
  k_extrap<<<kRedBlocks * 4, 256, 0, h.stream>>>(n, order, a, c, hist, same, out);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void launch_hist_shift(Handle& h, long n, const double* c, double* const* hist_vec, int* hist) {
  HistArgs a{};
  for (int j = 0; j < kExtrapMax; ++j) a.v[j] = hist_vec[j];
  k_hist_shift<<<kRedBlocks * 4, 256, 0, h.stream>>>(n, c, a, hist);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void launch_same(Handle& h, long n, const double* a, const double* b, int* same, cudaStream_t stream) {
  LDG_CUDA(cudaMemsetAsync(same, 0xff, sizeof(int), stream));
  k_same<<<kRedBlocks * 4, 256, 0, stream>>>(n, a, b, same);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void launch_axpby(Handle& h, long n, double a, const double* x, double b, double* y) {
  k_axpby<<<kRedBlocks * 4, 256, 0, h.stream>>>(n, a, x, b, y);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void launch_dots(Handle& h, long n, int nd, const double* const* xs, const double* const* ys, double* out_host) {
  DotArgs a{};
  for (int d = 0; d < nd; ++d) {
    a.x[d] = xs[d];
    a.y[d] = ys[d];
  }
  k_dots_partial<<<kRedBlocks, 256, 0, h.stream>>>(n, nd, a, h.red.ptr);
  k_dots_final<<<final_blocks(nd), 256, 0, h.stream>>>(nd, h.red.ptr, h.red.ptr + kMaxRed * kRedBlocks);
  LDG_CUDA(cudaGetLastError());
  h.launches += 2;
  LDG_CUDA(cudaMemcpyAsync(h.red_host, h.red.ptr + kMaxRed * kRedBlocks, sizeof(double) * nd,
                           cudaMemcpyDeviceToHost, h.stream));
  LDG_CUDA(cudaStreamSynchronize(h.stream));
  for (int d = 0; d < nd; ++d) out_host[d] = h.red_host[d];
}

void launch_soa_to_kmajor(Handle& h, const double* soa, int nvec, double* km, cudaStream_t stream) {
  const long total = static_cast<long>(nvec) * h.K * h.N;
  k_soa_to_kmajor<<<grid_of(total, 256), 256, 0, stream ? stream : h.stream>>>(h.K, h.N, h.Kp, nvec, soa, km);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

void launch_kmajor_to_soa(Handle& h, const double* km, int nvec, double* soa, cudaStream_t stream) {
  const long total = static_cast<long>(nvec) * h.K * h.N;
  k_kmajor_to_soa<<<grid_of(total, 256), 256, 0, stream ? stream : h.stream>>>(h.K, h.N, h.Kp, nvec, km, soa);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

size_t reduction_scratch() { return static_cast<size_t>(kMaxRed) * kRedBlocks + kMaxRed; }

void assemble_step(Handle& h, double t) {
  launch_project_df(h, t, h.rule_ptr(), h.rule_R());        // K2: d, f (system.hpp:112-113)
  launch_rhs(h, t);                                          // K5: V (system.hpp:142-150)
  launch_assemble(h, kModeEdiag, h.E.ptr);                   // K3: E^m diagonal blocks (system.hpp:115-117)
  h.assembled = true;
  h.t_assembled = t;
}

// Partial dots over the OWNED entries of N-plane vectors (ghost columns of
// a strip are skipped); result left on the device at dots_result(h).
void launch_dots_async(Handle& h, int nd, const double* const* xs, const double* const* ys) {
  DotArgs a{};
  for (int d = 0; d < nd; ++d) {
    a.x[d] = xs[d];
    a.y[d] = ys[d];
  }
  k_dots_owned<<<kRedBlocks, 256, 0, h.stream>>>(h.N, h.Kp, h.K, nd, a, h.red.ptr);
  k_dots_final<<<final_blocks(nd), 256, 0, h.stream>>>(nd, h.red.ptr, h.red.ptr + kMaxRed * kRedBlocks);
  LDG_CUDA(cudaGetLastError());
  h.launches += 2;
}

double* dots_result(Handle& h) { return h.red.ptr + kMaxRed * kRedBlocks; }

// (v_d, w), d < nv (<= kMaxRed), owned entries; result at dots_result(h)
void launch_mdots_async(Handle& h, int nv, const double* const* v, const double* w) {
  if (nv < 1 || nv > kMaxRed) throw Error(LDG_EINVAL, "multi-dot count out of range");
  MDotArgs a{};
  for (int d = 0; d < nv; ++d) a.v[d] = v[d];
  const dim3 grid(kRedBlocks, (nv + kMdotChunk - 1) / kMdotChunk);
  k_mdot_owned<<<grid, 256, 0, h.stream>>>(h.N, h.Kp, h.K, nv, a, w, h.red.ptr);
  k_dots_final<<<final_blocks(nv), 256, 0, h.stream>>>(nv, h.red.ptr, h.red.ptr + kMaxRed * kRedBlocks);
  LDG_CUDA(cudaGetLastError());
  h.launches += 2;
}

// w = alpha w + sum_d c[d] v[d] over all n = N * Kp entries
void launch_maxpy(Handle& h, int nv, const double* const* v, const double* c, double alpha, double* w) {
  if (nv < 0 || nv > kMaxRed) throw Error(LDG_EINVAL, "multi-axpy count out of range");
  MAxpyArgs a{};
  for (int d = 0; d < nv; ++d) {
    a.v[d] = v[d];
    a.c[d] = c[d];
  }
  k_maxpy<<<kRedBlocks * 4, 256, 0, h.stream>>>(h.vec_len(), nv, a, alpha, w);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

// (v_d, w), d < nv, owned entries; the results land at out (device)
void launch_mdots_to(Handle& h, int nv, const double* const* v, const double* w, double* out) {
  if (nv < 1 || nv > kMaxRed) throw Error(LDG_EINVAL, "multi-dot count out of range");
  MDotArgs a{};
  for (int d = 0; d < nv; ++d) a.v[d] = v[d];
  if (h.K == h.Kp) {
    const dim3 grid(kRedBlocks, (nv + kMdotFlatChunk - 1) / kMdotFlatChunk);
    k_mdot_flat<<<grid, 512, 0, h.stream>>>(static_cast<long>(h.N) * h.Kp / 2, nv, a, w, h.red.ptr);
  } else {
    const dim3 grid(kRedBlocks, (nv + kMdotChunk - 1) / kMdotChunk);
    k_mdot_owned<<<grid, 256, 0, h.stream>>>(h.N, h.Kp, h.K, nv, a, w, h.red.ptr);
  }
  k_dots_final<<<final_blocks(nv), 256, 0, h.stream>>>(nv, h.red.ptr, out);
  LDG_CUDA(cudaGetLastError());
  h.launches += 2;
}

// w -= sum c_d v_d (final = false) or w = (w - sum c_d v_d) / hn with the
// Pythagorean norm from c[nv] = (w, w) (final = true; copy into w2, hn at
// *hn_out); c on the device
void launch_maxpy_dev(Handle& h, int nv, const double* const* v, const double* c, bool final, double* w, double* w2,
                      double* hn_out) {
  if (nv < 1 || nv > kMaxRed - 1) throw Error(LDG_EINVAL, "multi-axpy count out of range");
  MDotArgs a{};
  for (int d = 0; d < nv; ++d) a.v[d] = v[d];
  const long n = h.vec_len();
  const unsigned grid = static_cast<unsigned>(std::min<long>(grid_of(n / 2, 256), 4L * kRedBlocks));
  if (final)
    k_maxpy_dev<1><<<grid, 256, 0, h.stream>>>(n, nv, a, c, w, w2, hn_out);
  else
    k_maxpy_dev<0><<<grid, 256, 0, h.stream>>>(n, nv, a, c, w, nullptr, nullptr);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

}  // namespace ldgb
