/*
 * hdc_oracle.c -- plain, slow, obviously-correct CPU oracle for batched HDC
 * inference (ScalableHD, arXiv 2506.09282).  TEST INFRASTRUCTURE ONLY: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  It shares no code, header, table or
 * helper with the CUDA path (paper_2506_09282_b200/).
 *
 * What it computes (PAPER.md = P:line):
 *   Alg. 1 "Two-Stage HDC Inference":
 *     V = X B                      eq. batch_encode, encoding P:117-124
 *     H = HardSign(V)              eq. hardsign: +1 if v >= 0 else -1
 *     S = H M^T   (M = C, K x D)   eq. batch_sim
 *     y = argmax(S, axis=1)        eq. pred_batch; ties -> lowest k
 *                                  (paper silent; reading R2)
 * Arithmetic: float64.  Each fp32 x fp32 product is exact in float64; sums run
 * in the plain definition's order (f ascending for V, d ascending for S).
 * Non-finite inputs are rejected, return code 1.
 *
 * Parity pins: see tests/test_oracle.py (worked examples S:52-54, S:97-99,
 * S:106-108; exact-rational brute force; D-chunk / linearity /
 * permutation / scaling invariants).  No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int all_finite(const float* a, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(a[i])) return 0;
  return 1;
}

/* HardSign: +1 if x >= 0 else -1.  -0.0 >= 0.0 is true -> +1. */
double oracle_hardsign(double x) { return x >= 0.0 ? 1.0 : -1.0; }

/* Operand formats of the low-precision paths (not in the paper, which is fp32-only,
 * P:143; the TF32 / BF16 paths are BASELINE north_star's additions, DESIGN.md
 * reading R15).  Both keep fp32's 8-bit exponent and shorten the significand:
 *   ORACLE_FMT_TF32: 10 explicit mantissa bits, round to nearest, ties AWAY from zero;
 *   ORACLE_FMT_BF16:  7 explicit mantissa bits, round to nearest, ties to EVEN.
 * Definition: for x != 0 with 2^(e-1) <= |x| < 2^e (frexp), the representable
 * neighbours are the multiples of q = 2^(e-1-p) (p = explicit bits; q >= 2^(-126-p)
 * below the normal range); the result is q * round(x / q).  x / q is exact in double. */
#define ORACLE_FMT_FP32 0
#define ORACLE_FMT_TF32 1
#define ORACLE_FMT_BF16 2
double oracle_round_fmt(double x, int fmt) {
  if (fmt == ORACLE_FMT_FP32 || x == 0.0 || !isfinite(x)) return x;
  const int p = (fmt == ORACLE_FMT_TF32) ? 10 : 7;
  int e;
  frexp(x, &e);
  int qe = e - 1 - p;
  if (qe < -126 - p) qe = -126 - p;
  const double q = ldexp(1.0, qe);
  const double t = x / q;                      /* exact: a power-of-two scaling */
  double r;
  if (fmt == ORACLE_FMT_TF32) {
    r = round(t);                              /* C99 round(): halfway cases away from zero */
  } else {
    r = floor(t);                              /* nearest, ties to even */
    const double frac = t - r;
    if (frac > 0.5 || (frac == 0.5 && fmod(r, 2.0) != 0.0)) r += 1.0;
  }
  return r * q;
}

/* Pre-activation V = X B for rows [0,N): V[n,d] = sum_f X[n,f] * B[f,d]
 * (eq. nonlinenc: bind x_i to b_i, bundle over i).  Loop n -> f -> d. */
int oracle_preact(const float* X, const float* B, int64_t N, int64_t F, int64_t D, double* V) {
  if (!all_finite(X, N * F) || !all_finite(B, F * D)) return 1;
  for (int64_t n = 0; n < N; ++n) {
    double* v = V + n * D;
    for (int64_t d = 0; d < D; ++d) v[d] = 0.0;
    for (int64_t f = 0; f < F; ++f) {
      const double x = (double)X[n * F + f];
      const float* b = B + f * D;
      for (int64_t d = 0; d < D; ++d) v[d] += x * (double)b[d];
    }
  }
  return 0;
}

/* Full inference, Alg. 1, one row at a time.
 *   S      [N*K] float64 scores (required)
 *   y      [N]   int32 labels (required), lowest index among equal maxima
 *   allow  [N*K] nullable: sum over the float64-ambiguous set
 *          A64(n) = { d : W[n,d] > 0, |V[n,d]| <= (F+1) 2^-53 W[n,d] },
 *          W = sum_f |x||b| (W = 0 means V is exactly 0 in any arithmetic -> +1),
 *          of 2|C[k,d]| -- the only score movement a correct fp64-exact sign
 *          decision could differ by (DESIGN.md tolerance policy).
 *   namb   [N] nullable: |A64(n)|
 *   nthreads: OpenMP threads over rows (<=0: runtime default).  Rows are
 *          independent, so the result does not depend on it. */
int oracle_infer_ex(const float* X, const float* B, const float* C, int64_t N, int64_t F, int64_t D,
                    int64_t K, int fmt, double gamma, double* S, int32_t* y, double* allow,
                    int32_t* namb, int nthreads);

int oracle_infer(const float* X, const float* B, const float* C, int64_t N, int64_t F, int64_t D,
                 int64_t K, double* S, int32_t* y, double* allow, int32_t* namb, int nthreads) {
  return oracle_infer_ex(X, B, C, N, F, D, K, ORACLE_FMT_FP32, (double)(F + 1) * ldexp(1.0, -53),
                         S, y, allow, namb, nthreads);
}

/* Generalised form (test infrastructure for the TF32 / BF16 paths, R15, R16):
 *   fmt   ORACLE_FMT_FP32: X and B as given (the paper's fp32 operands).
 *         ORACLE_FMT_TF32 / ORACLE_FMT_BF16: every element of X and B is first rounded
 *         to that format (oracle_round_fmt), then Alg. 1 runs unchanged in float64 on
 *         the rounded operands; C is not rounded.
 *   gamma the ambiguity set is A(n) = { d : W[n,d] > 0, |V[n,d]| <= gamma W[n,d] }, with
 *         V and W = sum_f |x||b| both of the (rounded) operands; allow[n,k] =
 *         sum_{d in A(n)} 2|C[k,d]| (the score movement of flipping every sign in A). */
int oracle_infer_ex(const float* X, const float* B, const float* C, int64_t N, int64_t F, int64_t D,
                    int64_t K, int fmt, double gamma, double* S, int32_t* y, double* allow,
                    int32_t* namb, int nthreads) {
  if (N < 0 || F < 1 || D < 1 || K < 1) return 2;
  if (fmt != ORACLE_FMT_FP32 && fmt != ORACLE_FMT_TF32 && fmt != ORACLE_FMT_BF16) return 2;
  if (!all_finite(X, N * F) || !all_finite(B, F * D) || !all_finite(C, K * D)) return 1;
  const double amb_c = gamma;
  /* the operands Stage I sees: rounded copies when fmt asks for them */
  float* Xr = NULL;
  float* Br = NULL;
  if (fmt != ORACLE_FMT_FP32) {
    Xr = (float*)malloc(sizeof(float) * (size_t)(N * F > 0 ? N * F : 1));
    Br = (float*)malloc(sizeof(float) * (size_t)(F * D));
    if (!Xr || !Br) {
      free(Xr);
      free(Br);
      return 3;
    }
    for (int64_t i = 0; i < N * F; ++i) Xr[i] = (float)oracle_round_fmt((double)X[i], fmt);
    for (int64_t i = 0; i < F * D; ++i) Br[i] = (float)oracle_round_fmt((double)B[i], fmt);
    X = Xr;
    B = Br;
  }
  int err = 0;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
  {
    double* v = (double*)malloc(sizeof(double) * (size_t)D);
    double* w = allow ? (double*)malloc(sizeof(double) * (size_t)D) : NULL;
    if (!v || (allow && !w)) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
      err = 3;
    } else {
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
      for (int64_t n = 0; n < N; ++n) {
        /* Stage I: v = sum_f x_f b_f  (Alg. 1 line 2) */
        for (int64_t d = 0; d < D; ++d) v[d] = 0.0;
        if (w) for (int64_t d = 0; d < D; ++d) w[d] = 0.0;
        for (int64_t f = 0; f < F; ++f) {
          const double x = (double)X[n * F + f];
          const float* b = B + f * D;
          for (int64_t d = 0; d < D; ++d) v[d] += x * (double)b[d];
          if (w) for (int64_t d = 0; d < D; ++d) w[d] += fabs(x) * fabs((double)b[d]);
        }
        /* Stage II: s_k = <HardSign(v), m_k>  (Alg. 1 line 4) */
        for (int64_t k = 0; k < K; ++k) {
          const float* c = C + k * D;
          double s = 0.0;
          for (int64_t d = 0; d < D; ++d) s += oracle_hardsign(v[d]) * (double)c[d];
          S[n * K + k] = s;
        }
        /* argmax, lowest index wins ties (Alg. 1 line 5) */
        int32_t best = 0;
        for (int64_t k = 1; k < K; ++k)
          if (S[n * K + k] > S[n * K + best]) best = (int32_t)k;
        y[n] = best;
        if (allow) {
          int32_t cnt = 0;
          for (int64_t k = 0; k < K; ++k) allow[n * K + k] = 0.0;
          for (int64_t d = 0; d < D; ++d) {
            if (w[d] > 0.0 && fabs(v[d]) <= amb_c * w[d]) {
              ++cnt;
              for (int64_t k = 0; k < K; ++k) allow[n * K + k] += 2.0 * fabs((double)C[k * D + d]);
            }
          }
          if (namb) namb[n] = cnt;
        }
      }
    }
    free(v);
    free(w);
  }
  free(Xr);
  free(Br);
  return err;
}

/* Element-wise oracle_round_fmt over an fp32 array (out may alias in). */
int oracle_round_array(const float* in, int64_t n, int fmt, float* out) {
  if (fmt != ORACLE_FMT_FP32 && fmt != ORACLE_FMT_TF32 && fmt != ORACLE_FMT_BF16) return 2;
  for (int64_t i = 0; i < n; ++i) out[i] = (float)oracle_round_fmt((double)in[i], fmt);
  return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Encoding alone, H = HardSign(X B) (eq. batch_encode P:173-176 with the HardSign
 * activation P:126-131), as int8 +1 / -1, rows [0,N).  Same float64 sum as
 * oracle_preact (f ascending). */
int oracle_encode(const float* X, const float* B, int64_t N, int64_t F, int64_t D, int8_t* H) {
  if (!all_finite(X, N * F) || !all_finite(B, F * D)) return 1;
  double* v = (double*)malloc(sizeof(double) * (D > 0 ? D : 1));
  if (!v) return 2;
  for (int64_t n = 0; n < N; ++n) {
    for (int64_t d = 0; d < D; ++d) v[d] = 0.0;
    for (int64_t f = 0; f < F; ++f) {
      const double x = (double)X[n * F + f];
      const float* b = B + f * D;
      for (int64_t d = 0; d < D; ++d) v[d] += x * (double)b[d];
    }
    for (int64_t d = 0; d < D; ++d) H[n * D + d] = (int8_t)oracle_hardsign(v[d]);
  }
  free(v);
  return 0;
}

/* Single-pass training: the class codebook by constrained bundling of the
 * encoded HVs of each class.  Bundling is element-wise addition, so
 *   counts[k,d] = sum_{n : y[n] = k} H[n,d]        (exact integers)
 * and the normalised class HV is M[k,d] = HardSign(counts[k,d]) (a tie,
 * count 0, gives +1).  Labels outside [0,K) return 3. */
int oracle_train(const int8_t* H, const int32_t* y, int64_t N, int64_t D, int64_t K, int64_t* counts,
                 double* M) {
  for (int64_t i = 0; i < K * D; ++i) counts[i] = 0;
  for (int64_t n = 0; n < N; ++n) {
    if (y[n] < 0 || y[n] >= K) return 3;
    for (int64_t d = 0; d < D; ++d) counts[(int64_t)y[n] * D + d] += H[n * D + d];
  }
  if (M)
    for (int64_t i = 0; i < K * D; ++i) M[i] = oracle_hardsign((double)counts[i]);
  return 0;
}
