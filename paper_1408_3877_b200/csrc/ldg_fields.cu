// Post-processing of a device-resident DG field (fields.hpp:84-123):
//  * l2_error  — ||u_h - u(t, .)||_{L2(Omega)} with a quad_rule_2d of order
//                q_ord (fields.hpp:100-123), used by the convergence study
//                (convergence.hpp:96, order 2p + 2);
//  * to_lagrange — u_h at the output nodes: the three vertices for p <= 1,
//                vertices + edge midpoints for p >= 2 (fields.hpp:87-97).
// One thread per element, element-interleaved coefficients (ldg_device.cuh).
#include <vector>

#include "ldg_internal.hpp"
#include "ldg_tables.hpp"

namespace ldgb {
namespace {

inline unsigned grid_of(long n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

// Physical point of reference point (s1, s2) on element k: map_to_physical
// (mesh.hpp:64-68), same operation order, no contraction.
__device__ __forceinline__ void to_physical(const double* __restrict__ g, long Kp, int k, double s1, double s2,
                                            double* x1, double* x2) {
  *x1 = __dadd_rn(__dadd_rn(__dmul_rn(g[kB11 * Kp + k], s1), __dmul_rn(g[kB12 * Kp + k], s2)), g[kA1x * Kp + k]);
  *x2 = __dadd_rn(__dadd_rn(__dmul_rn(g[kB21 * Kp + k], s1), __dmul_rn(g[kB22 * Kp + k], s2)), g[kA1y * Kp + k]);
}

// rule = [x1(R) | x2(R) | w(R) | phi(R x N)] (upload_rule).  out[k] =
// sqrt(2|T_k| sum_r w_r (u_h - u)^2) on owned k, so that the owned-entry
// self-dot of out is the squared error (deterministic reduction).
template <int N>
__global__ void __launch_bounds__(128) k_l2err(DevMesh m, const double* __restrict__ rule, int R,
                                               ldg_coeff f, double t, const double* __restrict__ u,
                                               double* __restrict__ out) {
  extern __shared__ double s_rule[];
  for (int i = threadIdx.x; i < R * (3 + N); i += blockDim.x) s_rule[i] = rule[i];
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m.Kp) return;
  if (k >= m.K) {
    out[k] = 0.0;
    return;
  }
  double c[N];
#pragma unroll
  for (int j = 0; j < N; ++j) c[j] = u[j * m.Kp + k];
  const double* phi = s_rule + 3 * R;
  double acc = 0.0;
  for (int r = 0; r < R; ++r) {
    double vh = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) vh = fma(c[j], phi[r * N + j], vh);
    double x1, x2;
    to_physical(m.geom, m.Kp, k, s_rule[r], s_rule[R + r], &x1, &x2);
    const double d = vh - ldg_coeff_eval(f.id, f.p, t, x1, x2);
    acc = fma(s_rule[2 * R + r] * d, d, acc);
  }
  out[k] = sqrt(2.0 * m.geom[kArea * m.Kp + k] * acc);
}

// nodes: phi(M x N) at the output nodes; out k-major K x M (owned elements)
template <int N>
__global__ void __launch_bounds__(128) k_lagrange(DevMesh m, const double* __restrict__ phi, int M,
                                                  const double* __restrict__ u, double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m.K) return;
  double c[N];
#pragma unroll
  for (int j = 0; j < N; ++j) c[j] = u[j * m.Kp + k];
  for (int i = 0; i < M; ++i) {
    double v = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) v = fma(c[j], __ldg(phi + i * N + j), v);
    out[static_cast<long>(k) * M + i] = v;
  }
}

template <int N>
void l2err_n(Handle& h, const double* rule, int R, const ldg_coeff& f, double t, const double* u, double* out) {
  const size_t smem = sizeof(double) * R * (3 + N);
  LDG_CUDA(cudaFuncSetAttribute(k_l2err<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  k_l2err<N><<<grid_of(static_cast<int>(h.Kp), 128), 128, smem, h.stream>>>(h.mesh(), rule, R, f, t, u, out);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

template <int N>
void lagrange_n(Handle& h, const double* phi, int M, const double* u, double* out) {
  k_lagrange<N><<<grid_of(h.K, 128), 128, 0, h.stream>>>(h.mesh(), phi, M, u, out);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
}

}  // namespace

void launch_l2err(Handle& h, const double* rule, int R, const ldg_coeff& f, double t, const double* u,
                  double* out) {
  switch (h.N) {
    case 1: l2err_n<1>(h, rule, R, f, t, u, out); break;
    case 3: l2err_n<3>(h, rule, R, f, t, u, out); break;
    case 6: l2err_n<6>(h, rule, R, f, t, u, out); break;
    case 10: l2err_n<10>(h, rule, R, f, t, u, out); break;
    default: l2err_n<15>(h, rule, R, f, t, u, out); break;
  }
}

int lagrange_nodes(int p) { return p <= 1 ? 3 : 6; }

void upload_lagrange_phi(Handle& h, DBuf<double>& buf) {
  // output nodes of fields.hpp:91-92 (vertices, then edge midpoints)
  static const double l1[6] = {0.0, 1.0, 0.0, 0.5, 0.0, 0.5};
  static const double l2[6] = {0.0, 0.0, 1.0, 0.5, 0.5, 0.0};
  const int M = lagrange_nodes(h.p);
  std::vector<double> host(static_cast<size_t>(M) * h.N);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < h.N; ++j) host[i * h.N + j] = basis_value(j, l1[i], l2[i]);
  buf.alloc(host.size(), nullptr);
  LDG_CUDA(cudaMemcpy(buf.ptr, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice));
}

void launch_lagrange(Handle& h, const double* phi, const double* u, double* out) {
  const int M = lagrange_nodes(h.p);
  switch (h.N) {
    case 1: lagrange_n<1>(h, phi, M, u, out); break;
    case 3: lagrange_n<3>(h, phi, M, u, out); break;
    case 6: lagrange_n<6>(h, phi, M, u, out); break;
    case 10: lagrange_n<10>(h, phi, M, u, out); break;
    default: lagrange_n<15>(h, phi, M, u, out); break;
  }
}

}  // namespace ldgb
