/*
 * ldg_b200_coeffs.h — compiled-in coefficient functions of the LDG path.
 *
 * The reference passes d, f, c_D, g_N and c0 as std::function ScalarFunc
 * (proj/include/ldg/fields.hpp:19; ProblemSpec system.hpp:26-37), built from
 * closures or the expression language (exprlang.hpp, OUT OF SCOPE here).  A
 * std::function cannot cross to the device, so the C ABI names a coefficient
 * by an id plus four double parameters; this header evaluates it identically
 * on host (C/C++) and device (CUDA).  The set covers the BASELINE.json problem
 * and every closure the reference's tests and drivers use.
 */
#ifndef LDG_B200_COEFFS_H
#define LDG_B200_COEFFS_H

#include <math.h>

#if defined(__CUDACC__)
#define LDG_HD __host__ __device__ __forceinline__
#else
#define LDG_HD static inline
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* A coefficient: f(t, x1, x2) = ldg_coeff_eval(id, p, t, x1, x2). */
typedef struct ldg_coeff {
  int id;
  double p[4];
} ldg_coeff;

enum ldg_coeff_id {
  LDG_FN_ZERO = 0,             /* 0                                                  */
  LDG_FN_CONST = 1,            /* p0                                                 */
  LDG_FN_POLY = 2,             /* p0 + p1 x1 + p2 x2 + p3 x1 x2                      */
  LDG_FN_EXP_SUM = 3,          /* exp(x1 + x2)         (test_assembly.cpp:140)        */
  LDG_FN_COS7X1_X2 = 4,        /* cos(7 x1) x2         (test_assembly.cpp:141)        */
  LDG_FN_MMS_EXACT = 5,        /* cos(7x1) cos(7x2)    (convergence.hpp:29-31)        */
  LDG_FN_MMS_F = 6,            /* manufactured f       (convergence.hpp:44-49)        */
  LDG_FN_MMS_GN = 7,           /* manufactured g_N     (convergence.hpp:53-56)        */
  LDG_FN_BASE_C = 8,           /* cos7x1 cos7x2 + e^-t (BASELINE.json configs, §8d)   */
  LDG_FN_BASE_D = 9,           /* e^(x1+x2) (1 + 0.5 sin t)                           */
  LDG_FN_BASE_F = 10,          /* dc/dt - div(d grad c) of the two above              */
  LDG_FN_BASE_GN = 11,         /* -grad c . nu on x1=1 (east) / x2=1 (north)          */
  LDG_FN_SIN_X1X2 = 12,        /* 1 + 0.5 sin(x1 x2)   (test_system.cpp:130)          */
  LDG_FN_COS3X1_PLUS_X2 = 13,  /* cos(3 x1) + x2       (test_system.cpp:134)          */
  LDG_FN_MMS_Z1 = 14,          /* 7 sin(7x1) cos(7x2)  (convergence.hpp:33-35)        */
  LDG_FN_MMS_Z2 = 15,          /* 7 cos(7x1) sin(7x2)  (convergence.hpp:36-38)        */
  LDG_FN_SIN3X1_X2SQ = 16,     /* sin(3 x1) + x2^2     (test_fields.cpp:82)           */
  LDG_FN_EXP_X1_MINUS_X2 = 17, /* exp(x1 - x2)         (test_fields.cpp:100)          */
  LDG_FN_COUNT = 18
};

LDG_HD double ldg_coeff_eval(int id, const double* p, double t, double x1, double x2) {
  switch (id) {
    case LDG_FN_ZERO: return 0.0;
    case LDG_FN_CONST: return p[0];
    case LDG_FN_POLY: return p[0] + p[1] * x1 + p[2] * x2 + p[3] * x1 * x2;
    case LDG_FN_EXP_SUM: return exp(x1 + x2);
    case LDG_FN_COS7X1_X2: return cos(7.0 * x1) * x2;
    case LDG_FN_MMS_EXACT: return cos(7.0 * x1) * cos(7.0 * x2);
    case LDG_FN_MMS_F: {
      const double d = exp(x1 + x2);
      return d * (98.0 * cos(7.0 * x1) * cos(7.0 * x2) + 7.0 * sin(7.0 * x1) * cos(7.0 * x2) +
                  7.0 * cos(7.0 * x1) * sin(7.0 * x2));
    }
    case LDG_FN_MMS_GN: {
      const double sign = (x2 > 0.5) ? 1.0 : -1.0;
      return sign * 7.0 * cos(7.0 * x1) * sin(7.0 * x2);
    }
    case LDG_FN_BASE_C: return cos(7.0 * x1) * cos(7.0 * x2) + exp(-t);
    case LDG_FN_BASE_D: return exp(x1 + x2) * (1.0 + 0.5 * sin(t));
    case LDG_FN_BASE_F: {
      const double d = exp(x1 + x2) * (1.0 + 0.5 * sin(t));
      return -exp(-t) + d * (98.0 * cos(7.0 * x1) * cos(7.0 * x2) +
                             7.0 * sin(7.0 * x1) * cos(7.0 * x2) +
                             7.0 * cos(7.0 * x1) * sin(7.0 * x2));
    }
    case LDG_FN_BASE_GN:
      /* Quadrature nodes are interior to boundary edges, so x1 > x2 holds
         exactly on the east edge (x1 = 1) and fails on the north edge. */
      return (x1 > x2) ? 7.0 * sin(7.0 * x1) * cos(7.0 * x2) : 7.0 * cos(7.0 * x1) * sin(7.0 * x2);
    case LDG_FN_SIN_X1X2: return 1.0 + 0.5 * sin(x1 * x2);
    case LDG_FN_COS3X1_PLUS_X2: return cos(3.0 * x1) + x2;
    case LDG_FN_MMS_Z1: return 7.0 * sin(7.0 * x1) * cos(7.0 * x2);
    case LDG_FN_MMS_Z2: return 7.0 * cos(7.0 * x1) * sin(7.0 * x2);
    case LDG_FN_SIN3X1_X2SQ: return sin(3.0 * x1) + x2 * x2;
    case LDG_FN_EXP_X1_MINUS_X2: return exp(x1 - x2);
    default: return NAN;
  }
}

#ifdef __cplusplus
}
#endif

#endif /* LDG_B200_COEFFS_H */
