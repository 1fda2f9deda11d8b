// Device-side data layout of the LDG path (sm_100a, FP64).
//
// Everything per element is stored element-interleaved ("SoA"): value v of
// element k lives at v * Kp + k, Kp = K rounded up to a multiple of 32.  A
// thread owns one element, so a warp touches 32 consecutive doubles (256 B)
// for every value: every load and store of the hot kernels is coalesced, and
// no padding is needed for odd block sizes N^2 = 1, 9, 225.
//
//  geometry   G[g][k]          g < kGeomCount (B, |T|, a_1, |E_n|, nu_n)
//  topology   nbr[n][k], nbrn[n][k], kind[n][k]   (neighbour k+, its edge n+,
//             edge kind: interior / Dirichlet / Neumann)
//  D, F       [N][Kp]          projected d(t) and f(t)
//  E          [m][i*N+j][Kp]     diagonal blocks E^m_kk of the time-dependent
//                              C-row operator E^m = -G^m + R^m + R_D^m; the
//                              off-diagonal blocks (pure R^m, rank Qe) are
//                              evaluated from D in the kernels (ldg_offdiag.cuh)
//  Bst        [m][s][i*N+j][Kp]  static Z-row blocks B^m = -H^m + Q^m + Q_N^m
//  Sst        [s][i*N+j][Kp]     static penalty S + S_D (eta applied in SpMV)
//  vectors    [u][j][Kp]       u = Z1, Z2, C
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/ldg_b200_coeffs.h"

namespace ldgb {

enum GeomField : int {
  kB11 = 0, kB12, kB21, kB22, kArea, kA1x, kA1y,
  kLen0, kLen1, kLen2, kNux0, kNux1, kNux2, kNuy0, kNuy1, kNuy2,
  kGeomCount
};

enum EdgeKind : int { kInterior = 0, kDirichlet = 1, kNeumann = 2, kUnmapped = 3 };

// Flat, read-only tables (offsets from TableLayout) in one device buffer.
struct DevTables {
  const double* base;
  int p, N, R, Qe, Qb;
  long proj_phi, proj_w, proj_x, mhat, minv, ghat, hhat, sdiag, soff, pe, pth, we, pb, sb, wb, total, mono;
  int NP;
  long tH, tSd, tSo, tM, tMinv;
  long tmH, tmSd, tmSo;
  // rank-Qe edge block (TableLayout rkR..rkW), usable when rank_ok
  int QP, rank_ok;
  long rkR, rkRm, rkT, rkV, rkW, rkEnd;
  long bjG2;  // block-Jacobi setup table (TableLayout::bjG2)
  // FP32 smoother tables (FTables in ldg_tables.hpp), offsets in floats
  const float* fbase;
  int NF;
  long fmH, fmSd, fmSo, fM, fSd, fSo, fpe, fpth, fwe;
  // rank-Qe edge block (FTables): peR | peT | pthT | weR, rows padded to NF / QF
  int QF;
  long fR, fpeT, fpthT, fweR, fRend;
};

struct DevMesh {
  int K;        // owned elements (rows this rank assembles / applies)
  int Kg;       // owned + ghost elements (D is projected on all of them)
  long Kp;      // plane stride
  const double* geom;
  const int* nbr;
  const int* nbrn;
  const int* kind;
};

__host__ __device__ inline long plane(long v, long Kp) { return v * Kp; }

// Programmatic dependent launch (launch_pdl, ldg_internal.hpp): a kernel
// launched with it may start while its stream predecessor drains; it calls
// pdl_wait() before touching the predecessor's output (everything before the
// wait may only read launch-invariant data such as the reference tables) and
// pdl_trigger() to let its own successor start.  Both are no-ops otherwise.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

}  // namespace ldgb
