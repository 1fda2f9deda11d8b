// Geometric multigrid preconditioner for the Schur system of each implicit-
// Euler step (the reference has none: it factorises with SparseLU every step,
// system.hpp:190-205).
//
// Friedrichs-Keller meshes nest: FK(dim) is the red refinement of FK(dim/2)
// (each coarse triangle holds 4 fine ones).  Coarse levels are rediscretised:
// every level is a Handle of its own on FK(dim/2^l) with vertex coordinates
// generated from the finest mesh's stream (jittered meshes: a reduced jitter,
// see coarse_jitter_scale),
// d projected on that level, and the same assembly / Schur kernels.  Transfer
// is the exact L2 embedding of the coarse polynomial space: per fine element
// one N x N block P_k (fine coeffs = P_k coarse coeffs of the parent),
// restriction is P^T (residuals are integrated quantities).  V(2,2) cycle
// with damped block-Jacobi smoothing (omega = 0.7) on every level; the
// coarsest level (dim 2) gets two smoothing sweeps.  Prototyped in numpy
// against the oracle first: 12-27 BiCGStab iterations for p = 1..4
// independent of h, against 170-2100 with block-Jacobi alone.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "ldg_internal.hpp"

namespace ldgb {

namespace {

template <int P>
struct Cfg {
  static constexpr int N = (P + 1) * (P + 2) / 2;
};

inline unsigned grid_of(long n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

#define LDG_DISPATCH_P(p, CALL) \
  switch (p) {                  \
    case 0: { CALL(0); break; } \
    case 1: { CALL(1); break; } \
    case 2: { CALL(2); break; } \
    case 3: { CALL(3); break; } \
    default: { CALL(4); break; } \
  }

// Parent of every owned fine element and the 4 children of every owned
// coarse element, in strip-local numbering (fine strip [2a, 2b) of FK(dim_f)
// over coarse strip [a, b)).  Coarse lower (cx,cy) holds fine lower
// (0,0),(1,0),(0,1) and upper (0,0) of its 2x2 block; coarse upper holds fine
// lower (1,1) and upper (1,0),(0,1),(1,1).
__global__ void k_fk_parent(int dim_f, int a_c, int w_c, long Kp_c, int* __restrict__ parent,
                            int* __restrict__ slots, int* __restrict__ children) {
  const int w_f = 2 * w_c, a_f = 2 * a_c, dim_c = dim_f / 2;
  const long Kf = 2L * w_f * dim_f;
  const long k = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (k >= Kf) return;
  const bool lower = k < static_cast<long>(w_f) * dim_f;
  const long q = lower ? k : k - static_cast<long>(w_f) * dim_f;
  const int ix = a_f + static_cast<int>(q / dim_f), iy = static_cast<int>(q % dim_f);
  const int cx = ix >> 1, cy = iy >> 1, lx = ix & 1, ly = iy & 1;
  bool clower;
  int slot;
  if (lower) {
    clower = !(lx && ly);
    slot = clower ? (lx ? 1 : (ly ? 2 : 0)) : 0;
  } else {
    clower = !lx && !ly;
    slot = clower ? 3 : (lx && !ly ? 1 : (!lx && ly ? 2 : 3));
  }
  const int kc = (clower ? 0 : w_c * dim_c) + (cx - a_c) * dim_c + cy;
  parent[k] = kc;
  slots[k] = slot;
  children[slot * Kp_c + kc] = static_cast<int>(k);
}

template <int N>
__device__ __forceinline__ void eval_basis(const double* __restrict__ mono, double x1, double x2, double* phi) {
  // monomials x1^a x2^b in the order (0,0),(1,0),(0,1),(2,0),(1,1),(0,2),...
  double m[15];
  m[0] = 1.0;
  int at = 1;
  double p1[5] = {1.0, x1, x1 * x1, x1 * x1 * x1, x1 * x1 * x1 * x1};
  double p2[5] = {1.0, x2, x2 * x2, x2 * x2 * x2, x2 * x2 * x2 * x2};
  for (int d = 1; d <= 4; ++d)
    for (int a = d; a >= 0; --a) m[at++] = p1[a] * p2[d - a];
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
    for (int q = 0; q < 15; ++q) s += mono[i * 15 + q] * m[q];
    phi[i] = s;
  }
}

// P_k[i][j] = sum_a minv[i][a] int_ref phi_a(xh) phi_j(xi(xh)), xi = parent
// reference coordinates of the fine point; exact with the order-2p rule.
// Pm (FP32: a preconditioner transfer; half the bytes of the level-0/1
// transfers, the largest of them) is stored on the coarse level, [slot][N*N][Kp_c], so restriction and
// prolongation (both driven from the coarse side) read it coalesced.
template <int P>
__global__ void __launch_bounds__(128) k_prolong_blocks(DevMesh f, DevMesh c, DevTables T, const int* __restrict__ parent,
                                                        const int* __restrict__ slots, float* __restrict__ Pm) {
  constexpr int N = Cfg<P>::N, NN = N * N;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= f.K) return;
  const double* base = T.base;
  const int R = T.R;
  const int kc = parent[k];
  const double* gf = f.geom;
  const double* gc = c.geom;
  const long Kf = f.Kp, Kc = c.Kp;
  const double b11 = gc[kB11 * Kc + kc], b12 = gc[kB12 * Kc + kc], b21 = gc[kB21 * Kc + kc], b22 = gc[kB22 * Kc + kc];
  const double det = b11 * b22 - b12 * b21;
  double acc[NN];
  for (int ij = 0; ij < NN; ++ij) acc[ij] = 0.0;
  for (int r = 0; r < R; ++r) {
    const double r1 = base[T.proj_x + 2 * r], r2 = base[T.proj_x + 2 * r + 1], w = base[T.proj_w + r];
    const double x1 = gf[kB11 * Kf + k] * r1 + gf[kB12 * Kf + k] * r2 + gf[kA1x * Kf + k];
    const double x2 = gf[kB21 * Kf + k] * r1 + gf[kB22 * Kf + k] * r2 + gf[kA1y * Kf + k];
    const double d1 = x1 - gc[kA1x * Kc + kc], d2 = x2 - gc[kA1y * Kc + kc];
    const double xi1 = (b22 * d1 - b12 * d2) / det, xi2 = (b11 * d2 - b21 * d1) / det;
    double pc[N];
    eval_basis<N>(base + T.mono, xi1, xi2, pc);
    const double* pf = base + T.proj_phi + r * N;
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) acc[i * N + j] += w * pf[i] * pc[j];
  }
  const double* minv = base + T.minv;
  float* out = Pm + static_cast<long>(slots[k]) * NN * Kc;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0.0;
      for (int a = 0; a < N; ++a) s += minv[i * N + a] * acc[a * N + j];
      out[static_cast<long>(i * N + j) * Kc + kc] = static_cast<float>(s);
    }
}

// bc[j][kc] = sum over the 4 children s, rows i of P_s[i][j] rf[i][child_s]:
// one thread per (j, kc) output value (coarse levels hold too few elements
// for a thread per element to hide the load latency)
template <int P>
__global__ void __launch_bounds__(256) k_restrict(int Kc, long Kpc, long Kpf, const int* __restrict__ children,
                                                  const float* __restrict__ Pm, const double* __restrict__ rf,
                                                  double* __restrict__ bc) {
  constexpr int N = Cfg<P>::N, NN = N * N;
  pdl_wait();
  pdl_trigger();
  const long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (t >= static_cast<long>(N) * Kc) return;
  const int kc = static_cast<int>(t % Kc), j = static_cast<int>(t / Kc);
  int ch[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) ch[s] = children[s * Kpc + kc];
  double acc = 0.0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {  // loads of a child first, then its FMA chain (latency-bound on coarse levels)
    const float* Ps = Pm + (static_cast<long>(s) * NN + j) * Kpc + kc;
    double pv[N], rv[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      pv[i] = __ldcs(Ps + static_cast<long>(i) * N * Kpc);
      rv[i] = rf[i * Kpf + ch[s]];
    }
#pragma unroll
    for (int i = 0; i < N; ++i) acc = fma(pv[i], rv[i], acc);
  }
  bc[j * Kpc + kc] = acc;
}

// xf[i][child_s] += sum_j P_s[i][j] xc[j][kc]: one thread per (i, s, kc)
template <int P>
__global__ void __launch_bounds__(256) k_prolong_add(int Kc, long Kpc, long Kpf, const int* __restrict__ children,
                                                     const float* __restrict__ Pm, const double* __restrict__ xc,
                                                     double* __restrict__ xf, double theta) {
  constexpr int N = Cfg<P>::N, NN = N * N;
  pdl_wait();
  pdl_trigger();
  const long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (t >= 4L * N * Kc) return;
  const int kc = static_cast<int>(t % Kc);
  const int rest = static_cast<int>(t / Kc);
  const int s = rest % 4, i = rest / 4;
  const int k = children[s * Kpc + kc];
  const float* Ps = Pm + (static_cast<long>(s) * NN + static_cast<long>(i) * N) * Kpc + kc;
  double pv[N], xv[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    pv[j] = __ldcs(Ps + static_cast<long>(j) * Kpc);
    xv[j] = xc[j * Kpc + kc];
  }
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) acc = fma(pv[j], xv[j], acc);
  xf[i * Kpf + k] = fma(theta, acc, xf[i * Kpf + k]);
}

}  // namespace

int mg_levels(const Handle& h) { return 1 + static_cast<int>(h.coarse.size()); }

double coarse_jitter_scale();

// Number of coarse levels for FK(dim) split into `size` equal strips: halve
// while dim stays even, the coarse mesh keeps dim >= 2, and every rank keeps
// at least one whole column with even strip boundaries.  Every rank computes
// the same count, so the distributed V-cycle stays in lockstep.
int mg_depth(int dim, int size) {
  if (dim % size != 0) return 0;
  int w = dim / size, d = dim, n = 0;
  while (d % 2 == 0 && d / 2 >= 2 && w % 2 == 0) {
    d /= 2;
    w /= 2;
    ++n;
  }
  return n;
}

// Degrees of the p-coarsened levels: the first coarse levels are the fine
// mesh itself at the degrees of this chain (descending, each < p); the
// h-coarsened levels below run at the last one.  The modal basis is
// hierarchical and L2-orthonormal on the reference element (basis.hpp), so
// the embedding of a lower-degree space is the identity on its first N
// coefficients: restriction truncates, prolongation pads with zeros.
std::vector<int> mg_pcoarse_chain(int p) {
  // A/B runs: LDG_MG_PC<p>="2,1" overrides the chain of degree p
  char name[16];
  snprintf(name, sizeof(name), "LDG_MG_PC%d", p);
  if (const char* e = std::getenv(name)) {
    std::vector<int> chain;
    int last = p;
    for (const char* q = e; *q;) {
      char* end = nullptr;
      const long v = std::strtol(q, &end, 10);
      if (end == q) break;
      if (v >= 0 && v < last) chain.push_back(static_cast<int>(last = static_cast<int>(v)));
      q = *end == ',' ? end + 1 : end;
    }
    return chain;
  }
  // p = 4: 4 -> 2 -> 1 (with the dense degree-1 coarsest level: 23.0 ->
  // 19.8 ms per step, 9.6 -> 8.4 iterations on C2 against 4 -> 2)
  if (p >= 4) return {2, 1};
  return p >= 2 ? std::vector<int>{1} : std::vector<int>{};
}

namespace {

// coarse-level buffers shared by both kinds of level
void alloc_coarse(Handle& c) {
  const long n = c.vec_len();
  const long NN = static_cast<long>(c.N) * c.N;
  c.D.alloc(n, &c.bytes);
  c.E.alloc(2 * NN * c.Kp, &c.bytes);  // diagonal blocks (off-diagonal ones matrix-free)
  c.Pinv.alloc(NN * c.Kp, &c.bytes);
  c.tz.alloc(2 * n, &c.bytes);
  c.mg_x.alloc(n, &c.bytes);
  c.mg_b.alloc(n, &c.bytes);
  c.mg_r.alloc(n, &c.bytes);
  c.mg_s.alloc(n, &c.bytes);
}

std::unique_ptr<Handle> coarse_shell(const Handle& h, const Handle& fine) {
  auto c = std::make_unique<Handle>();
  c->p = fine.p;
  c->N = fine.N;
  c->prob = h.prob;
  c->dtab = fine.dtab;
  c->stream = h.stream;
  c->owns_stream = false;
  c->rule_shared = fine.rule_ptr();
  c->rule_shared_R = fine.rule_R();
  c->rank = h.rank;
  c->size = h.size;
  return c;
}

}  // namespace

// The coarse mesh of a red refinement (refine_uniform, mesh.hpp:258-293):
// parent c's children are 4c..4c+3 = (a1, m3, m2), (m3, a2, m1), (m2, m1,
// a3), (m3, m1, m2) with m_n the midpoint of the edge opposite a_n, the
// parent's vertices numbered before every midpoint, and a parent edge's
// boundary ID on its child edges.  False when the mesh is not one.
bool coarsen_red(const std::vector<double>& xy, const std::vector<int>& t, const std::vector<int>& ids, int K,
                 std::vector<double>* cxy, std::vector<int>* ct, std::vector<int>* cids) {
  if (K < 4 || K % 4 != 0) return false;
  const int Kc = K / 4;
  ct->assign(3L * Kc, 0);
  int amax = -1, mmin = 1 << 30;
  double scale = 0.0;
  for (double v : xy) scale = std::max(scale, std::fabs(v));
  const double tol = 1e-12 * std::max(scale, 1.0);
  auto mid_ok = [&](int m, int a, int b) {
    return std::fabs(xy[2 * m] - 0.5 * (xy[2 * a] + xy[2 * b])) <= tol &&
           std::fabs(xy[2 * m + 1] - 0.5 * (xy[2 * a + 1] + xy[2 * b + 1])) <= tol;
  };
  for (int c = 0; c < Kc; ++c) {
    const int* t0 = &t[3L * (4 * c)];
    const int* t1 = t0 + 3;
    const int* t2 = t0 + 6;
    const int* t3 = t0 + 9;
    const int a1 = t0[0], m3 = t0[1], m2 = t0[2], a2 = t1[1], m1 = t1[2], a3 = t2[2];
    if (t1[0] != m3 || t2[0] != m2 || t2[1] != m1 || t3[0] != m3 || t3[1] != m1 || t3[2] != m2) return false;
    if (!mid_ok(m1, a2, a3) || !mid_ok(m2, a3, a1) || !mid_ok(m3, a1, a2)) return false;
    (*ct)[3 * c] = a1;
    (*ct)[3 * c + 1] = a2;
    (*ct)[3 * c + 2] = a3;
    amax = std::max({amax, a1, a2, a3});
    mmin = std::min({mmin, m1, m2, m3});
  }
  if (mmin <= amax) return false;  // parent vertices first, then the midpoints
  cxy->assign(xy.begin(), xy.begin() + 2L * (amax + 1));
  cids->clear();
  if (!ids.empty()) {
    cids->assign(3L * Kc, 0);
    for (int c = 0; c < Kc; ++c) {
      (*cids)[3 * c] = ids[3L * (4 * c + 1)];         // edge a2-a3: child (m3, a2, m1), edge 0
      (*cids)[3 * c + 1] = ids[3L * (4 * c + 2) + 1];  // edge a3-a1: child (m2, m1, a3), edge 1
      (*cids)[3 * c + 2] = ids[3L * (4 * c) + 2];      // edge a1-a2: child (a1, m3, m2), edge 2
    }
  }
  return true;
}

// General meshes (ldg_create, one rank): the p-coarsened levels on the same
// mesh, then h-levels while the mesh is a red refinement of a coarser one
// (the reference's convergence ladder is domain_square refined by
// refine_uniform), then the dense coarsest level when small enough.  Without
// a red-refinement hierarchy there is no multigrid (block-Jacobi).
bool mg_build_general(Handle& h) {
  std::vector<double> xy = h.host_xy, cxy;
  std::vector<int> t = h.host_v0t, ids = h.host_ids, ct, cids;
  std::vector<std::vector<double>> lxy;
  std::vector<std::vector<int>> lt, lids;
  int K = h.K;
  while (lt.size() < 12 && coarsen_red(xy, t, ids, K, &cxy, &ct, &cids)) {
    lxy.push_back(cxy);
    lt.push_back(ct);
    lids.push_back(cids);
    xy.swap(cxy);
    t.swap(ct);
    ids.swap(cids);
    K /= 4;
  }
  if (lt.empty()) return false;
  h.mg_r.alloc(h.vec_len(), &h.bytes);
  h.mg_s.alloc(h.vec_len(), &h.bytes);
  Handle* fine = &h;
  for (const int pc : mg_pcoarse_chain(h.p)) {  // the same mesh at degree pc
    auto c = std::make_unique<Handle>();
    c->p = pc;
    c->N = dofs_of(pc);
    c->prob = h.prob;
    c->stream = h.stream;
    c->owns_stream = false;
    c->rank = h.rank;
    c->size = h.size;
    init_handle_tables(*c, pc);
    build_general_mesh(*c, h.host_xy.data(), static_cast<int>(h.host_xy.size() / 2), h.host_v0t.data(), h.K,
                       h.host_ids.empty() ? nullptr : h.host_ids.data());
    alloc_coarse(*c);
    c->mg_pcoarse = true;
    fine = c.get();
    h.coarse.push_back(std::move(c));
  }
  for (size_t l = 0; l < lt.size(); ++l) {
    auto c = coarse_shell(h, *fine);
    const int Kc = static_cast<int>(lt[l].size() / 3);
    build_general_mesh(*c, lxy[l].data(), static_cast<int>(lxy[l].size() / 2), lt[l].data(), Kc,
                       lids[l].empty() ? nullptr : lids[l].data());
    alloc_coarse(*c);
    const long NN = static_cast<long>(c->N) * c->N;
    // parent f / 4, slot f % 4 (refine_uniform's child order)
    std::vector<int> parent(fine->Kp, 0), slot(fine->Kp, 0), children(4L * c->Kp, 0);
    for (int f = 0; f < fine->K; ++f) {
      parent[f] = f / 4;
      slot[f] = f % 4;
      children[static_cast<long>(f % 4) * c->Kp + f / 4] = f;
    }
    c->mg_children.alloc(4 * c->Kp, &c->bytes);
    fine->mg_parent.alloc(fine->Kp, &fine->bytes);
    DBuf<int> slots;
    slots.alloc(fine->Kp, nullptr);
    LDG_CUDA(cudaMemcpy(c->mg_children.ptr, children.data(), sizeof(int) * children.size(), cudaMemcpyHostToDevice));
    LDG_CUDA(cudaMemcpy(fine->mg_parent.ptr, parent.data(), sizeof(int) * parent.size(), cudaMemcpyHostToDevice));
    LDG_CUDA(cudaMemcpy(slots.ptr, slot.data(), sizeof(int) * slot.size(), cudaMemcpyHostToDevice));
    c->mg_P.alloc(4 * NN * c->Kp, &c->bytes);
#define CALL(PP)                                                                                              \
  k_prolong_blocks<PP><<<grid_of(fine->K, 128), 128, 0, h.stream>>>(fine->mesh(), c->mesh(), fine->dtab,     \
                                                                   fine->mg_parent.ptr, slots.ptr, c->mg_P.ptr)
    LDG_DISPATCH_P(fine->p, CALL)
#undef CALL
    LDG_CUDA(cudaGetLastError());
    LDG_CUDA(cudaStreamSynchronize(h.stream));
    fine = c.get();
    h.coarse.push_back(std::move(c));
  }
  for (size_t i = 0; i < h.coarse.size(); ++i) {
    Handle& c = *h.coarse[i];
    if (!dense_candidate(c)) continue;
    dense_alloc(c);
    h.dense_level = static_cast<int>(i) + 1;
    break;
  }
  h.mg_ready = true;
  return true;
}

bool mg_build(Handle& h, int team_size) {
  if (h.mg_ready) return true;
  if (h.dim == 0 && team_size == 1 && !h.host_v0t.empty()) return mg_build_general(h);
  if (h.dim < 4 || h.dim_fine == 0) return false;
  const int depth = mg_depth(h.dim, team_size);
  if (depth < 1) return false;
  h.mg_r.alloc(h.vec_len(), &h.bytes);
  h.mg_s.alloc(h.vec_len(), &h.bytes);
  Handle* fine = &h;
  for (const int pc : mg_pcoarse_chain(h.p)) {  // the fine mesh again at degree pc (same vertices, numbering, strip)
    auto c = std::make_unique<Handle>();
    c->p = pc;
    c->N = dofs_of(pc);
    c->prob = h.prob;
    c->stream = h.stream;
    c->owns_stream = false;
    c->rank = h.rank;
    c->size = h.size;
    init_handle_tables(*c, pc);
    build_square_strip(*c, h.dim, h.strip_a, h.strip_b, h.stride, h.dim_fine, h.jitter, h.seed);
    alloc_coarse(*c);
    c->mg_pcoarse = true;
    fine = c.get();
    h.coarse.push_back(std::move(c));
  }
  for (int l = 0; l < depth; ++l) {
    const int dc = fine->dim / 2;
    auto c = coarse_shell(h, *fine);
    const long NN = static_cast<long>(c->N) * c->N;
    // coarse vertices are the finest mesh's vertices (stride 2^l): jittered
    // meshes coarsen consistently on every rank
    const double cj = coarse_jitter_scale() * h.jitter;
    build_square_strip(*c, dc, fine->strip_a / 2, fine->strip_b / 2, fine->stride * 2, h.dim_fine, cj, h.seed);
    alloc_coarse(*c);
    c->mg_children.alloc(4 * c->Kp, &c->bytes);
    fine->mg_parent.alloc(fine->Kp, &fine->bytes);
    DBuf<int> slots;
    slots.alloc(fine->Kp, nullptr);
    c->mg_P.alloc(4 * NN * c->Kp, &c->bytes);
    k_fk_parent<<<grid_of(fine->K, 256), 256, 0, h.stream>>>(fine->dim, c->strip_a, c->strip_w(), c->Kp,
                                                             fine->mg_parent.ptr, slots.ptr, c->mg_children.ptr);
    LDG_CUDA(cudaGetLastError());
#define CALL(PP)                                                                                              \
  k_prolong_blocks<PP><<<grid_of(fine->K, 128), 128, 0, h.stream>>>(fine->mesh(), c->mesh(), fine->dtab,     \
                                                                   fine->mg_parent.ptr, slots.ptr, c->mg_P.ptr)
    LDG_DISPATCH_P(fine->p, CALL)
#undef CALL
    LDG_CUDA(cudaGetLastError());
    LDG_CUDA(cudaStreamSynchronize(h.stream));
    fine = c.get();
    h.coarse.push_back(std::move(c));
  }
  // strip team: the coarsest strip level replicated whole on this rank
  // (the first h-level small enough; the levels below it are never visited)
  int rl = 0;
  for (size_t i = 0; team_size > 1 && i < h.coarse.size() && !rl; ++i)
    if (!h.coarse[i]->mg_pcoarse && replica_candidate(*h.coarse[i])) rl = static_cast<int>(i) + 1;
  if (rl > 0) {
    const Handle& C = *h.coarse[rl - 1];
    h.replica_level = rl;
    auto r = std::make_unique<Handle>();
    r->p = C.p;
    r->N = C.N;
    r->prob = C.prob;
    r->dtab = C.dtab;
    r->stream = h.stream;
    r->owns_stream = false;
    r->rule_shared = C.rule_ptr();
    r->rule_shared_R = C.rule_R();
    r->rank = 0;
    r->size = 1;
    build_square_strip(*r, C.dim, 0, C.dim, C.stride, C.dim_fine, C.jitter, C.seed);
    alloc_coarse(*r);
    dense_alloc(*r);
    h.replica = std::move(r);
  }
  // dense coarsest level: the first h-level small enough (single rank)
  for (size_t i = 0; i < h.coarse.size(); ++i) {
    Handle& c = *h.coarse[i];
    if (!dense_candidate(c)) continue;
    dense_alloc(c);
    h.dense_level = static_cast<int>(i) + 1;
    break;
  }
  h.mg_ready = true;
  return true;
}

// Per step: rediscretise every coarse level at time t (projection of d on
// owned + ghost elements, E^m assembly) and build the block-Jacobi inverses.
// Mixed precision (f32): every level gets FP32 copies of E and of the
// inverses (built from the FP64 E) — packed float4 for the levels the fused
// smoother runs on, plain SoA for the small levels on the row kernels.
// All-FP64 (precond 3): level 0's inverse is built by the caller.
void mg_setup_f32_level(Handle& L, double wm, double dt) {
  const long NN = static_cast<long>(L.N) * L.N;
  if (!level_uses_rows(L)) {
    // stage-1 output of the smoother in FP32 (no halo of it across ranks: single rank only)
    if (L.size == 1 && !L.tz32.ptr) {
      L.tz32.alloc(2 * L.vec_len(), &L.bytes);
      if (L.p >= smooth_trace_min_p()) {
        const long q = (3 * L.p + 2) / 2;  // edge rule of the rank-Qe form
        L.tr32.alloc(9 * q * L.Kp, &L.bytes);  // x traces A | u traces | x traces B
        L.dtr32.alloc(3 * q * L.Kp, &L.bytes);
      }
    }
    if (!L.Ph.ptr) {  // FP16 packed P^-1, scaled per element
      L.Ph.alloc(packed_p_quads(L.p) * L.Kp, &L.bytes);
      L.Pscale.alloc(L.Kp, &L.bytes);
    }
    launch_bjac(L, wm, dt, 3);  // also writes the FP16 copy of E (Eh, Escale) from its staged blocks
    smooth_dtraces(L);
  } else {
    if (!L.E32.ptr) {
      L.E32.alloc(2 * NN * L.Kp, &L.bytes);
      L.Pinv32.alloc(NN * L.Kp, &L.bytes);
    }
    launch_to_f32(L, 2 * NN * L.Kp, L.E.ptr, L.E32.ptr);
    launch_bjac_setup_f32_from64(L, wm, dt);
  }
}

void debug_level(Handle& L, int l) {
  char w[64];
  const long NN = static_cast<long>(L.N) * L.N;
  snprintf(w, sizeof(w), "level %d E", l);
  debug_count_nonfinite(L.stream, L.E.ptr, 2 * NN * L.Kp, false, w);
  if (L.Eh.ptr) {
    snprintf(w, sizeof(w), "level %d Eh", l);
    debug_count_nonfinite(L.stream, L.Eh.ptr, 4 * L.Eh.n, true, w);
  }
  if (L.Ph.ptr) {
    snprintf(w, sizeof(w), "level %d Ph", l);
    debug_count_nonfinite(L.stream, L.Ph.ptr, 4 * L.Ph.n, true, w);
  }
  snprintf(w, sizeof(w), "level %d D", l);
  debug_count_nonfinite(L.stream, L.D.ptr, L.vec_len(), false, w);
}

void mg_setup_step(Handle& h, double t, double wm, double dt, bool f32) {
  mg_setup_top(h, wm, dt, f32);
  mg_setup_coarse(h, t, wm, dt, f32);
}

void mg_setup_top(Handle& h, double wm, double dt, bool f32) {
  if (f32) mg_setup_f32_level(h, wm, dt);
  if (debug_nan()) debug_level(h, 0);
}

// every coarse level is rediscretised from d(t) on its own mesh: independent
// of level 0 and of each other
void mg_setup_coarse(Handle& h, double t, double wm, double dt, bool f32) {
  for (auto& cp : h.coarse) {
    const int lvl = static_cast<int>(&cp - &h.coarse[0]) + 1;
    if (h.dense_level > 0 && lvl > h.dense_level) break;  // below the dense level: never visited
    if (h.replica_level > 0 && lvl > h.replica_level) break;
    Handle& c = *cp;
    launch_project(c, h.prob.d, t, c.rule_ptr(), c.rule_R(), c.D.ptr, c.Kg);
    launch_assemble(c, kModeEdiag, c.E.ptr);
    if (f32)
      mg_setup_f32_level(c, wm, dt);
    else
      launch_bjac_setup(c, wm, dt);
    if (lvl == h.dense_level) dense_setup(c, wm, dt, f32);
    if (debug_nan()) debug_level(c, lvl);
  }
  if (h.replica) {  // the replicated coarsest strip level: same operator, whole mesh
    Handle& r = *h.replica;
    launch_project(r, h.prob.d, t, r.rule_ptr(), r.rule_R(), r.D.ptr, r.Kg);
    launch_assemble(r, kModeEdiag, r.E.ptr);
    dense_setup(r, wm, dt, false);
  }
}

// C.mg_b = P^T L.mg_r (restriction of the fine residual to the coarse level)
void mg_restrict(Handle& L, Handle& C) {
  if (C.mg_pcoarse) {  // same mesh, lower degree: the first C.N coefficient planes
    LDG_CUDA(cudaMemcpyAsync(C.mg_b.ptr, L.mg_r.ptr, sizeof(double) * C.vec_len(), cudaMemcpyDeviceToDevice,
                             L.stream));
    return;
  }
#define CALL(PP)                                                                                             \
  launch_pdl(k_restrict<PP>, grid_of(static_cast<long>(L.N) * C.K, 256), 256, 0, L.stream, C.K, C.Kp, L.Kp,      \
             C.mg_children.ptr, C.mg_P.ptr, L.mg_r.ptr, C.mg_b.ptr)
  LDG_DISPATCH_P(L.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++L.launches;
}

// Jitter of the coarse levels' vertices as a fraction of the finest mesh's
// displacement (same splitmix64 stream): on a jittered FK mesh the fine
// triangles do not tile the coarse ones whatever the coarse vertices are, and
// subsampling the fine vertices (1.0) made the rediscretised coarse operators
// a poor match -- measured at 512^2, p = 3, jitter 0.2, mixed BCs: 93
// iterations with 1.0, 60 with a regular coarse lattice (0.0), 52.5 with 0.4
// (0.25..0.75 swept).
double coarse_jitter_scale() { return 0.4; }

// x += P C.mg_x (prolongation of the coarse correction)
void mg_prolong_add(Handle& L, Handle& C, double* x) {
  if (C.mg_pcoarse) {  // pad: the first C.N coefficient planes
    launch_lincomb3(L, C.vec_len(), 1.0, x, 1.0, C.mg_x.ptr, 0.0, nullptr, x);
    return;
  }
#define CALL(PP)                                                                                              \
  launch_pdl(k_prolong_add<PP>, grid_of(4L * L.N * C.K, 256), 256, 0, L.stream, C.K, C.Kp, L.Kp,                \
             C.mg_children.ptr, C.mg_P.ptr, C.mg_x.ptr, x, 1.0)
  LDG_DISPATCH_P(L.p, CALL)
#undef CALL
  LDG_CUDA(cudaGetLastError());
  ++L.launches;
}

void mg_release(Handle& h) {
  for (auto& g : h.vgraphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  h.vgraphs.clear();
}

}  // namespace ldgb
