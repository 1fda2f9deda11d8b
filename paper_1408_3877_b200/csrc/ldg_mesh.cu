// K1 — mesh geometry and topology precompute on the device, once per handle.
//
// Replaces generate_grid_data (mesh.hpp:103-221) and domain_square
// (mesh.hpp:225-254).  The reference numbers edges through a std::map
// (O(E log E) on one core, 2.7 s at K = 2.1M); here each (triangle, local
// edge) emits a 64-bit key min(v)*V + max(v), one device radix sort groups
// the two sides of every interior edge, and a pairing pass writes the
// neighbour (k+, n+) both ways.  Geometry (B_k, |T_k|, |E_kn|, outward nu_kn)
// is computed per element with the reference's exact operation order
// (explicit round-to-nearest intrinsics, no FMA contraction), so the lists
// match the reference bit-for-bit up to hypot().
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "ldg_internal.hpp"

namespace ldgb {

namespace {

struct BcMap {
  int n;
  int id[LDG_MAX_BC];
  int kind[LDG_MAX_BC];
};

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// FK vertices: id = ix*(dim+1)+iy at (ix h, iy h) (mesh.hpp:231-233), with
// optional interior jitter U(-jitter h, jitter h) (BASELINE config 4).
__global__ void k_fk_vertices(int dim, double jitter, uint64_t seed, double* coords) {
  const long V = static_cast<long>(dim + 1) * (dim + 1);
  const long v = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (v >= V) return;
  const int ix = static_cast<int>(v / (dim + 1)), iy = static_cast<int>(v % (dim + 1));
  const double h = 1.0 / dim;
  double x = ix * h, y = iy * h;
  if (jitter > 0.0 && ix > 0 && ix < dim && iy > 0 && iy < dim) {
    const uint64_t base = seed << 32;
    const double amp = __dmul_rn(jitter, h);
    const uint64_t rx = splitmix64(base + 2ull * static_cast<uint64_t>(v));
    const uint64_t ry = splitmix64(base + 2ull * static_cast<uint64_t>(v) + 1ull);
    const double ux = static_cast<double>(rx >> 11) * (1.0 / 9007199254740992.0);
    const double uy = static_cast<double>(ry >> 11) * (1.0 / 9007199254740992.0);
    x = __dadd_rn(x, __dmul_rn(__dsub_rn(__dmul_rn(2.0, ux), 1.0), amp));
    y = __dadd_rn(y, __dmul_rn(__dsub_rn(__dmul_rn(2.0, uy), 1.0), amp));
  }
  coords[2 * v] = x;
  coords[2 * v + 1] = y;
}

// FK triangles: all lower (ix,iy) first, then all upper ones (mesh.hpp:237-242).
__global__ void k_fk_triangles(int dim, int* v0t) {
  const long K = 2L * dim * dim;
  const long k = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (k >= K) return;
  const long q = k < static_cast<long>(dim) * dim ? k : k - static_cast<long>(dim) * dim;
  const int ix = static_cast<int>(q / dim), iy = static_cast<int>(q % dim);
  auto vid = [dim](int a, int b) { return a * (dim + 1) + b; };
  if (k < static_cast<long>(dim) * dim) {
    v0t[3 * k] = vid(ix, iy);
    v0t[3 * k + 1] = vid(ix + 1, iy);
    v0t[3 * k + 2] = vid(ix, iy + 1);
  } else {
    v0t[3 * k] = vid(ix + 1, iy);
    v0t[3 * k + 1] = vid(ix + 1, iy + 1);
    v0t[3 * k + 2] = vid(ix, iy + 1);
  }
}

// Per-element geometry (mesh.hpp:123-143, 167-188) + edge keys.
__global__ void k_geometry(int Kg, long Kp, int V, double bbox_area, const double* __restrict__ coords,
                           const int* __restrict__ v0t, double* __restrict__ geom, uint64_t* __restrict__ keys,
                           int* __restrict__ vals, int* __restrict__ errs) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= Kg) return;
  int vv[3];
  double px[3], py[3];
  for (int i = 0; i < 3; ++i) {
    vv[i] = v0t[3 * k + i];
    if (vv[i] < 0 || vv[i] >= V) {
      atomicCAS(&errs[0], 0, 1);
      atomicCAS(&errs[1], -1, k);
      return;
    }
    px[i] = coords[2 * vv[i]];
    py[i] = coords[2 * vv[i] + 1];
  }
  if (vv[0] == vv[1] || vv[1] == vv[2] || vv[2] == vv[0]) {
    atomicCAS(&errs[0], 0, 2);
    atomicCAS(&errs[1], -1, k);
    return;
  }
  const double b11 = __dsub_rn(px[1], px[0]), b12 = __dsub_rn(px[2], px[0]);
  const double b21 = __dsub_rn(py[1], py[0]), b22 = __dsub_rn(py[2], py[0]);
  const double signed2 = __dsub_rn(__dmul_rn(b11, b22), __dmul_rn(b12, b21));
  if (!(signed2 > 2e-14 * bbox_area)) {
    atomicCAS(&errs[0], 0, 3);
    atomicCAS(&errs[1], -1, k);
  }
  geom[kB11 * Kp + k] = b11;
  geom[kB12 * Kp + k] = b12;
  geom[kB21 * Kp + k] = b21;
  geom[kB22 * Kp + k] = b22;
  geom[kArea * Kp + k] = 0.5 * signed2;
  geom[kA1x * Kp + k] = px[0];
  geom[kA1y * Kp + k] = py[0];
  const double btx = __ddiv_rn(__dadd_rn(__dadd_rn(px[0], px[1]), px[2]), 3.0);
  const double bty = __ddiv_rn(__dadd_rn(__dadd_rn(py[0], py[1]), py[2]), 3.0);
  for (int n = 0; n < 3; ++n) {
    const int va = vv[(n + 1) % 3], vb = vv[(n + 2) % 3];
    const int lo = min(va, vb), hi = max(va, vb);
    const double ax = coords[2 * lo], ay = coords[2 * lo + 1];
    const double bx = coords[2 * hi], by = coords[2 * hi + 1];
    const double dx = __dsub_rn(bx, ax), dy = __dsub_rn(by, ay);
    const double len = hypot(dx, dy);
    const double nx = __ddiv_rn(dy, len), ny = __ddiv_rn(-dx, len);
    const double mx = __dmul_rn(0.5, __dadd_rn(ax, bx)), my = __dmul_rn(0.5, __dadd_rn(ay, by));
    const double dot = __dadd_rn(__dmul_rn(nx, __dsub_rn(mx, btx)), __dmul_rn(ny, __dsub_rn(my, bty)));
    const double sgn = dot > 0.0 ? 1.0 : -1.0;
    geom[(kLen0 + n) * Kp + k] = len;
    geom[(kNux0 + n) * Kp + k] = sgn * nx;
    geom[(kNuy0 + n) * Kp + k] = sgn * ny;
    keys[3L * k + n] = static_cast<uint64_t>(lo) * static_cast<uint64_t>(V) + static_cast<uint64_t>(hi);
    vals[3L * k + n] = 3 * k + n;
  }
}

// Groups of equal keys: 2 = interior edge, 1 = boundary, >2 = non-manifold.
__global__ void k_pair_edges(long M, const uint64_t* __restrict__ keys, const int* __restrict__ vals,
                             const int* __restrict__ v0t, long Kp, int* __restrict__ nbr, int* __restrict__ nbrn,
                             int* __restrict__ errs) {
  const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (i >= M) return;
  const uint64_t key = keys[i];
  if (i > 0 && keys[i - 1] == key) return;  // not the first of its run
  const int a = vals[i];
  const int ka = a / 3, na = a % 3;
  if (i + 1 < M && keys[i + 1] == key) {
    if (i + 2 < M && keys[i + 2] == key) {
      atomicCAS(&errs[0], 0, 4);
      atomicCAS(&errs[1], -1, ka);
      return;
    }
    const int b = vals[i + 1];
    const int kb = b / 3, nb = b % 3;
    // Both sides traverse the edge: consistent ccw orientation needs them reversed.
    if (v0t[3 * ka + (na + 1) % 3] == v0t[3 * kb + (nb + 1) % 3]) {
      atomicCAS(&errs[0], 0, 5);
      atomicCAS(&errs[1], -1, ka);
    }
    nbr[na * Kp + ka] = kb;
    nbrn[na * Kp + ka] = nb;
    nbr[nb * Kp + kb] = ka;
    nbrn[nb * Kp + kb] = na;
  } else {
    nbr[na * Kp + ka] = -1;
    nbrn[na * Kp + ka] = -1;
  }
}

// Boundary IDs (given per (k,n), or the unit-square rule of mesh.hpp:245-252
// on the edge barycentre) and the edge kind through the boundary map.
__global__ void k_edge_kinds(int K, long Kp, const double* __restrict__ coords, const int* __restrict__ v0t,
                             const int* __restrict__ id_in, const int* __restrict__ nbr, BcMap bc,
                             int* __restrict__ kind, int* __restrict__ bid, int* __restrict__ errs) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  for (int n = 0; n < 3; ++n) {
    if (nbr[n * Kp + k] >= 0) {
      kind[n * Kp + k] = kInterior;
      bid[n * Kp + k] = 0;
      continue;
    }
    int id;
    if (id_in) {
      id = id_in[3 * k + n];
    } else {
      const int va = v0t[3 * k + (n + 1) % 3], vb = v0t[3 * k + (n + 2) % 3];
      const double mx = __dmul_rn(0.5, __dadd_rn(coords[2 * va], coords[2 * vb]));
      const double my = __dmul_rn(0.5, __dadd_rn(coords[2 * va + 1], coords[2 * vb + 1]));
      const double tol = 1e-12;
      id = 0;
      if (fabs(my) < tol) id = 1;
      else if (fabs(mx - 1.0) < tol) id = 2;
      else if (fabs(my - 1.0) < tol) id = 3;
      else if (fabs(mx) < tol) id = 4;
    }
    bid[n * Kp + k] = id;
    int kd = kUnmapped;
    for (int q = 0; q < bc.n; ++q)
      if (bc.id[q] == id) kd = bc.kind[q] == LDG_BC_DIRICHLET ? kDirichlet : kNeumann;
    kind[n * Kp + k] = kd;
    if (kd == kUnmapped) {
      atomicCAS(&errs[0], 0, 6);
      atomicCAS(&errs[1], -1, id);
    }
  }
}

inline unsigned grid_of(long n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

void topology_and_geometry(Handle& h, double bbox_area, const int* id_in_dev) {
  const int Kg = h.Kg;
  const long Kp = h.Kp;
  h.geom.alloc(static_cast<size_t>(kGeomCount) * Kp, &h.bytes);
  h.nbr.alloc(3 * Kp, &h.bytes);
  h.nbrn.alloc(3 * Kp, &h.bytes);
  h.kind.alloc(3 * Kp, &h.bytes);
  h.bid.alloc(3 * Kp, &h.bytes);
  LDG_CUDA(cudaMemsetAsync(h.nbr.ptr, 0xff, 3 * Kp * sizeof(int), h.stream));
  LDG_CUDA(cudaMemsetAsync(h.nbrn.ptr, 0xff, 3 * Kp * sizeof(int), h.stream));

  const long M = 3L * Kg;
  DBuf<uint64_t> keys, keys2;
  DBuf<int> vals, vals2, errs;
  keys.alloc(M, nullptr);
  keys2.alloc(M, nullptr);
  vals.alloc(M, nullptr);
  vals2.alloc(M, nullptr);
  errs.alloc(2, nullptr);
  int init[2] = {0, -1};
  LDG_CUDA(cudaMemcpyAsync(errs.ptr, init, sizeof(init), cudaMemcpyHostToDevice, h.stream));

  k_geometry<<<grid_of(Kg, 256), 256, 0, h.stream>>>(Kg, Kp, h.V, bbox_area, h.coords.ptr, h.v0t.ptr, h.geom.ptr,
                                                     keys.ptr, vals.ptr, errs.ptr);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
  int end_bit = 1;
  while (end_bit < 64 && (1ull << end_bit) <= static_cast<uint64_t>(h.V) * static_cast<uint64_t>(h.V)) ++end_bit;
  size_t temp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys.ptr, keys2.ptr, vals.ptr, vals2.ptr, M, 0, end_bit,
                                  h.stream);
  DBuf<unsigned char> temp;
  temp.alloc(std::max<size_t>(temp_bytes, 1), nullptr);
  LDG_CUDA(cub::DeviceRadixSort::SortPairs(temp.ptr, temp_bytes, keys.ptr, keys2.ptr, vals.ptr, vals2.ptr, M, 0,
                                           end_bit, h.stream));
  k_pair_edges<<<grid_of(M, 256), 256, 0, h.stream>>>(M, keys2.ptr, vals2.ptr, h.v0t.ptr, Kp, h.nbr.ptr,
                                                      h.nbrn.ptr, errs.ptr);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
  int herr[2];
  LDG_CUDA(cudaMemcpyAsync(herr, errs.ptr, sizeof(herr), cudaMemcpyDeviceToHost, h.stream));
  LDG_CUDA(cudaStreamSynchronize(h.stream));
  if (herr[0] != 0) {
    static const char* what[] = {"", "references a vertex out of range", "has a repeated vertex",
                                 "is degenerate or not counter-clockwise", "shares an edge with two other triangles",
                                 "claims an edge from the same side as its neighbour"};
    throw Error(LDG_EMESH, "triangle " + std::to_string(herr[1]) + " " + what[herr[0] < 6 ? herr[0] : 0]);
  }
  BcMap bc{};
  bc.n = h.prob.n_bc;
  for (int i = 0; i < bc.n; ++i) {
    bc.id[i] = h.prob.bc_id[i];
    bc.kind[i] = h.prob.bc_kind[i];
  }
  LDG_CUDA(cudaMemcpyAsync(errs.ptr, init, sizeof(init), cudaMemcpyHostToDevice, h.stream));
  k_edge_kinds<<<grid_of(h.K, 256), 256, 0, h.stream>>>(h.K, Kp, h.coords.ptr, h.v0t.ptr, id_in_dev, h.nbr.ptr, bc,
                                                        h.kind.ptr, h.bid.ptr, errs.ptr);
  LDG_CUDA(cudaGetLastError());
  ++h.launches;
  LDG_CUDA(cudaMemcpyAsync(herr, errs.ptr, sizeof(herr), cudaMemcpyDeviceToHost, h.stream));
  LDG_CUDA(cudaStreamSynchronize(h.stream));
  if (herr[0] != 0)
    throw Error(LDG_EINVAL, "boundary ID " + std::to_string(herr[1]) + " has no boundary condition assigned");
  keys.release(nullptr);
  keys2.release(nullptr);
  vals.release(nullptr);
  vals2.release(nullptr);
  errs.release(nullptr);
  temp.release(nullptr);
}

long padded(long k) { return ((k + 31) / 32) * 32; }

// Vertices of columns [vx0, vx1] of FK(dim) on one level: vertex (ix, iy) is
// vertex (ix*stride, iy*stride) of the finest FK(dim_fine), coordinates and
// jitter computed exactly as k_fk_vertices does for that finest vertex.
__global__ void k_fk_vertices_strip(int dim, int vx0, int vx1, int stride, int dim_fine, double jitter,
                                    uint64_t seed, double* coords) {
  const long V = static_cast<long>(vx1 - vx0 + 1) * (dim + 1);
  const long v = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (v >= V) return;
  const int fx = (vx0 + static_cast<int>(v / (dim + 1))) * stride;
  const int fy = static_cast<int>(v % (dim + 1)) * stride;
  const double h = 1.0 / dim_fine;
  double x = fx * h, y = fy * h;
  if (jitter > 0.0 && fx > 0 && fx < dim_fine && fy > 0 && fy < dim_fine) {
    const uint64_t vf = static_cast<uint64_t>(fx) * static_cast<uint64_t>(dim_fine + 1) + static_cast<uint64_t>(fy);
    const uint64_t base = seed << 32;
    const double amp = __dmul_rn(jitter, h);
    const double ux = static_cast<double>(splitmix64(base + 2ull * vf) >> 11) * (1.0 / 9007199254740992.0);
    const double uy = static_cast<double>(splitmix64(base + 2ull * vf + 1ull) >> 11) * (1.0 / 9007199254740992.0);
    x = __dadd_rn(x, __dmul_rn(__dsub_rn(__dmul_rn(2.0, ux), 1.0), amp));
    y = __dadd_rn(y, __dmul_rn(__dsub_rn(__dmul_rn(2.0, uy), 1.0), amp));
  }
  coords[2 * v] = x;
  coords[2 * v + 1] = y;
}

// FK triangles of the strip in local numbering: owned lowers, owned uppers,
// ghost uppers of column a-1 (gl of them), ghost lowers of column b.
__global__ void k_fk_triangles_strip(int dim, int a, int b, int gl, int gr, int vx0, int* v0t) {
  const long W = b - a;
  const long Kg = 2 * W * dim + gl + gr;
  const long k = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (k >= Kg) return;
  bool upper;
  int ix, iy;
  if (k < W * dim) {
    upper = false;
    ix = a + static_cast<int>(k / dim);
    iy = static_cast<int>(k % dim);
  } else if (k < 2 * W * dim) {
    upper = true;
    ix = a + static_cast<int>((k - W * dim) / dim);
    iy = static_cast<int>((k - W * dim) % dim);
  } else if (k < 2 * W * dim + gl) {
    upper = true;
    ix = a - 1;
    iy = static_cast<int>(k - 2 * W * dim);
  } else {
    upper = false;
    ix = b;
    iy = static_cast<int>(k - 2 * W * dim - gl);
  }
  auto vid = [dim, vx0](int x, int y) { return (x - vx0) * (dim + 1) + y; };
  if (!upper) {
    v0t[3 * k] = vid(ix, iy);
    v0t[3 * k + 1] = vid(ix + 1, iy);
    v0t[3 * k + 2] = vid(ix, iy + 1);
  } else {
    v0t[3 * k] = vid(ix + 1, iy);
    v0t[3 * k + 1] = vid(ix + 1, iy + 1);
    v0t[3 * k + 2] = vid(ix, iy + 1);
  }
}

}  // namespace

// Columns [a, b) of FK(dim) plus one ghost column per side (the full mesh
// when a = 0, b = dim).  Element order within the owned part matches the
// reference's (lowers then uppers, column-major), so a single strip is
// exactly domain_square's numbering (mesh.hpp:237-242).
void build_square_strip(Handle& h, int dim, int a, int b, int stride, int dim_fine, double jitter, uint64_t seed) {
  if (dim < 1) throw Error(LDG_EINVAL, "maximum edge length must be positive");
  if (!(jitter >= 0.0 && jitter < 0.5)) throw Error(LDG_EINVAL, "jitter must be in [0, 0.5)");
  if (a < 0 || b > dim || b <= a) throw Error(LDG_EINVAL, "empty or invalid strip");
  if (2L * dim * dim > 0x7fffffffL / 3) throw Error(LDG_EINVAL, "mesh too large for 32-bit element indices");
  const int W = b - a;
  const int gl = a > 0 ? dim : 0, gr = b < dim ? dim : 0;
  const int vx0 = a > 0 ? a - 1 : a, vx1 = b < dim ? b + 1 : b;
  const long V = static_cast<long>(vx1 - vx0 + 1) * (dim + 1);
  const long K = 2L * W * dim;
  const long Kg = K + gl + gr;
  h.dim = dim;
  h.strip_a = a;
  h.strip_b = b;
  h.ghost_left = gl;
  h.ghost_right = gr;
  h.stride = stride;
  h.dim_fine = dim_fine;
  h.jitter = jitter;
  h.seed = seed;
  h.V = static_cast<int>(V);
  h.K = static_cast<int>(K);
  h.Kg = static_cast<int>(Kg);
  h.Kglobal = 2 * dim * dim;
  h.Kp = padded(Kg);
  h.coords.alloc(2 * V, &h.bytes);
  h.v0t.alloc(3 * Kg, &h.bytes);
  k_fk_vertices_strip<<<grid_of(V, 256), 256, 0, h.stream>>>(dim, vx0, vx1, stride, dim_fine, jitter, seed,
                                                             h.coords.ptr);
  k_fk_triangles_strip<<<grid_of(Kg, 256), 256, 0, h.stream>>>(dim, a, b, gl, gr, vx0, h.v0t.ptr);
  LDG_CUDA(cudaGetLastError());
  h.launches += 2;
  // global element index (reference numbering) of every local element,
  // ghosts included (exports resolve neighbour columns through it)
  h.gid.resize(Kg);
  const long dd = static_cast<long>(dim) * dim;
  for (long k = 0; k < K; ++k) {
    const long q = k < static_cast<long>(W) * dim ? k : k - static_cast<long>(W) * dim;
    const long ix = a + q / dim, iy = q % dim;
    h.gid[k] = static_cast<int>((k < static_cast<long>(W) * dim ? 0 : dd) + ix * dim + iy);
  }
  for (long iy = 0; iy < gl; ++iy) h.gid[K + iy] = static_cast<int>(dd + static_cast<long>(a - 1) * dim + iy);
  for (long iy = 0; iy < gr; ++iy) h.gid[K + gl + iy] = static_cast<int>(static_cast<long>(b) * dim + iy);
  topology_and_geometry(h, 1.0, nullptr);
}

void build_square_mesh(Handle& h, int dim, double jitter, uint64_t seed) {
  build_square_strip(h, dim, 0, dim, 1, dim, jitter, seed);
}

void build_general_mesh(Handle& h, const double* coords, int nv, const int* v0t, int nt, const int* id_e0t) {
  if (nv < 3 || nt < 1 || !coords || !v0t) throw Error(LDG_EINVAL, "empty mesh");
  double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
  for (int i = 0; i < nv; ++i) {
    xmin = std::min(xmin, coords[2 * i]);
    xmax = std::max(xmax, coords[2 * i]);
    ymin = std::min(ymin, coords[2 * i + 1]);
    ymax = std::max(ymax, coords[2 * i + 1]);
  }
  const double bbox = std::max((xmax - xmin) * (ymax - ymin), 1e-300);
  h.V = nv;
  h.K = h.Kg = h.Kglobal = nt;
  h.Kp = padded(nt);
  h.coords.alloc(2L * nv, &h.bytes);
  h.v0t.alloc(3L * nt, &h.bytes);
  LDG_CUDA(cudaMemcpyAsync(h.coords.ptr, coords, sizeof(double) * 2 * nv, cudaMemcpyHostToDevice, h.stream));
  LDG_CUDA(cudaMemcpyAsync(h.v0t.ptr, v0t, sizeof(int) * 3L * nt, cudaMemcpyHostToDevice, h.stream));
  DBuf<int> ids;
  if (id_e0t) {
    ids.alloc(3L * nt, nullptr);
    LDG_CUDA(cudaMemcpyAsync(ids.ptr, id_e0t, sizeof(int) * 3L * nt, cudaMemcpyHostToDevice, h.stream));
  }
  h.gid.resize(nt);
  for (int k = 0; k < nt; ++k) h.gid[k] = k;
  h.host_xy.assign(coords, coords + 2L * nv);
  h.host_v0t.assign(v0t, v0t + 3L * nt);
  if (id_e0t)
    h.host_ids.assign(id_e0t, id_e0t + 3L * nt);
  else
    h.host_ids.clear();
  topology_and_geometry(h, bbox, ids.ptr);
  ids.release(nullptr);
}

}  // namespace ldgb
