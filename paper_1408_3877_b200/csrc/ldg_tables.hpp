// Host-side reference-element math for the LDG path: the modal basis, the
// quadrature rules, the reference integral tensors and the flat tables the
// sm_100a kernels read.  Computed once per (p) at ldg_create, uploaded once.
//
// Mirrors (behaviour, not code) of the reference:
//   basis              proj/include/ldg/basis.hpp:42-158
//   quadrature rules   proj/include/ldg/quadrature.hpp:39-174
//   reference tensors  proj/include/ldg/reftensors.hpp:55-154
#pragma once

#include <array>
#include <vector>

namespace ldgb {

constexpr int kMaxP = 4;
constexpr int kMaxN = 15;

inline int dofs_of(int p) { return (p + 1) * (p + 2) / 2; }

// phi_i and grad phi_i (i = 0..14) at a reference point, table-driven.
double basis_value(int i, double x1, double x2);
void basis_gradient(int i, double x1, double x2, double* g1, double* g2);

struct Rule1D {
  std::vector<double> s, w;  // nodes on (0,1), weights sum to 1
};
struct Rule2D {
  std::vector<double> x1, x2, w;  // weights sum to 1/2
};

Rule1D gauss_unit(int npts);       // Newton on Legendre P_n
Rule1D rule_1d(int order);         // reference quad_rule_1d(order)
Rule2D rule_2d(int order);         // reference quad_rule_2d(order)
void edge_point(int n, double s, double* x1, double* x2);                 // gamma_n, n = 0..2
void edge_to_edge(int nm, int np, double x1, double x2, double* y1, double* y2);  // theta

struct RefTensors {
  int n = 0;
  std::vector<double> m, h, g, sd, so, rd, ro;  // same index layout as reftensors.hpp:36-50
};
RefTensors reference_tensors(int n);

// Flat device tables; every array is an offset (in doubles) into one buffer.
struct TableLayout {
  int p = 0, N = 0;
  int R = 0;    // projection rule points (order max(2p,1))
  int Qe = 0;   // exact edge rule for the rank-Q R assembly (degree 3p)
  int Qb = 0;   // boundary-vector edge rule (order 2p+1, reference BasisQuadCache)
  long proj_phi, proj_w, proj_x;     // [R][N], [R], [R][2]
  long mhat, minv;                   // [N][N]
  long ghat;                         // [i][j][l][m]  (reftensors.hpp:38-40)
  long hhat, sdiag, soff;            // [i][j][m], [i][j][n], [i][j][nm][np]
  long pe, pth, we;                  // [n][q][i], [nm][np][q][j], [q]   (rank-Q edge form)
  long pb, sb, wb;                   // [n][q][i], [q], [q]              (RHS edge rule)
  long mono;                         // [i][15] scaled monomial coefficients of phi_i
  // matrix-free static operators: reference matrices transposed and padded
  // to NP = N rounded up to even, T^t[j][i] at j*NP + i (16-byte rows)
  int NP = 0;
  long tH;                           // [2][N][NP]  h_hat(.,.,m)^t
  long tSd;                          // [3][N][NP]  s_diag(.,.,n)^t
  long tSo;                          // [9][N][NP]  s_offdiag(.,.,nm,np)^t
  long tM;                           // [N][NP]     m_hat^t
  long tMinv;                        // [N][NP]     m_hat^-1 ^t
  long tmH, tmSd, tmSo;              // the same with m_hat^-1 applied: (m_hat^-1 T)^t,
                                     // for stage 1 (t = M^-1 B x in one pass)
  // rank-Qe edge block of the FP64 operator kernels (ldg_apply.cu), contiguous,
  // QP = Qe rounded up to even:
  //   rkR  [3][Qe][NP]   phi_i at the points of edge n (rows of pe, padded)
  //   rkRm [3][Qe][NP]   the same with m_hat^-1 applied (stage 1 output)
  //   rkT  [3][N][QP]    pe transposed (own projection)
  //   rkV  [9][N][QP]    pth transposed (neighbour projection)
  //   rkW  [QP]          weights
  int QP = 0;
  long rkR = 0, rkRm = 0, rkT = 0, rkV = 0, rkW = 0, rkEnd = 0;
  // the caller's s_diag / s_offdiag equal pe^t diag(we) pe / pth to 1e-13 and
  // h_hat is degree-lower-triangular (true for the library's own tensors):
  // the operator kernels may use the rank-Qe edge form and skip the zero
  // chunks of the derivative tables
  bool rank_ok = false;
  // block-Jacobi setup (ldg_bjac.cu): bjG2[n*3+np][q][j] = sum_i pth_{n,np}[q][i] (m_hat^-1 s_off(np, n))[i][j],
  // the row space of an off-diagonal E block (rank Qe) carried through the neighbour's M^-1 B block
  long bjG2 = 0;
  long total = 0;
};

struct HostTables {
  TableLayout lay;
  std::vector<double> data;
};

// caller_rt: the caller's RefTensors (the rt argument of the reference's
// LdgSystem(mesh, spec, rt), system.hpp:67) instead of the library's own
HostTables build_tables(int p, const RefTensors* caller_rt = nullptr);

// FP32 copies of the transposed static tables for the mixed-precision
// multigrid smoother (ldg_smooth.cu), rows padded to NF = N rounded up to 4
// (one 128-bit shared load per 4 entries), T^t[j][i] at j*NF + i:
//   [tmH 2 | tmSd 3 | tmSo 9]  stage 1 (m_hat^-1 applied)
//   [tM 1 | tSd 3 | tSo 9]     stage 2
//   [pe 3*Qe*N | pth 9*Qe*N | we Qe (padded to 4)]  matrix-free off-diagonal E
// and the rank-Qe edge block every edge term of the smoother is applied from
// (s_diag_n = pe_n^t diag(we) pe_n, s_offdiag_{n,np} = pe_n^t diag(we) pth_{n,np}:
// the Qe-point rule is exact for degree 3p >= 2p), QF = Qe rounded up to 4:
//   [peR 3][Qe][NF]    phi_i at the points of edge n, one row per point (the output product)
//   [peT 3][N][QF]     the same transposed, one row per basis function (own projection)
//   [pthT 9][N][QF]    phi_j at the theta-mapped points of the pair (n, np) (neighbour projection)
//   [weR QF]           rule weights
struct FTables {
  int NF = 0, QF = 0;
  long fmH = 0, fmSd = 0, fmSo = 0, fM = 0, fSd = 0, fSo = 0, fpe = 0, fpth = 0, fwe = 0, total = 0;
  long fR = 0, fpeT = 0, fpthT = 0, fweR = 0, fRend = 0;
  std::vector<float> data;
};
FTables build_f32_tables(const HostTables& ht);

}  // namespace ldgb
