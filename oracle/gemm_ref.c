/* Plain GEMM references for arXiv 1909.10616 (oracle; TEST INFRASTRUCTURE ONLY).
 *
 * PAPER.md P:113 (Fig. 2 "three-for-loop" computation) and P:166: "Multiplication of two
 * matrices A(m x k) and B(k x n) produces matrix C(m x n)"; "A resulted matrix is
 * initialized with zeros ... accumulates".  Row-major A[m][k], B[k][n], C[m][n] (reading Z14).
 *
 *   oracle_gemm_f64   R_ij = sum_{l=0}^{k-1} A_il * B_lj in double, sequential l
 *   oracle_gemm_fmaf  C_ij = fmaf(A_il, B_lj, acc) for l = 0..k-1 in float, acc0 = 0
 *   oracle_gemm_f64_rows / _entries   the same definition on sampled rows / (i,j) pairs
 *
 * OpenMP over rows only: each output is still one sequential sum in k order.
 * Shares no code or header with the CUDA library.
 */
#include <math.h>
#include <stdint.h>

void oracle_gemm_f64(int64_t m, int64_t n, int64_t k, const double* A, const double* B, double* C) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t j = 0; j < n; ++j) C[i * n + j] = 0.0;
    for (int64_t l = 0; l < k; ++l) {          /* i-l-j order: same per-entry sum order as i-j-l */
      const double a = A[i * k + l];
      const double* b = B + l * n;
      double* c = C + i * n;
      for (int64_t j = 0; j < n; ++j) c[j] += a * b[j];
    }
  }
}

void oracle_gemm_fmaf(int64_t m, int64_t n, int64_t k, const float* A, const float* B, float* C) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t j = 0; j < n; ++j) C[i * n + j] = 0.0f;
    for (int64_t l = 0; l < k; ++l) {
      const float a = A[i * k + l];
      const float* b = B + l * n;
      float* c = C + i * n;
      for (int64_t j = 0; j < n; ++j) c[j] = fmaf(a, b[j], c[j]);
    }
  }
}

/* rows[r] selects row i of the product; out is [nrows][n]. */
void oracle_gemm_f64_rows(int64_t n, int64_t k, const double* A, const double* B,
                          const int64_t* rows, int64_t nrows, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < nrows; ++r) {
    const int64_t i = rows[r];
    double* c = out + r * n;
    for (int64_t j = 0; j < n; ++j) c[j] = 0.0;
    for (int64_t l = 0; l < k; ++l) {
      const double a = A[i * k + l];
      const double* b = B + l * n;
      for (int64_t j = 0; j < n; ++j) c[j] += a * b[j];
    }
  }
}

/* one entry at a time: R_ij for the listed (i, j). */
void oracle_gemm_f64_entries(int64_t n, int64_t k, const double* A, const double* B,
                             const int64_t* ii, const int64_t* jj, int64_t cnt, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < cnt; ++t) {
    double s = 0.0;
    for (int64_t l = 0; l < k; ++l) s += A[ii[t] * k + l] * B[l * n + jj[t]];
    out[t] = s;
  }
}

/* Direct convolution (cross-correlation, as in DL frameworks), the operation P:105 lowers to a GEMM:
 * y[n][f][p][q] = sum_{c,r,s} x[n][c][p*st - pad + r][q*st - pad + s] * w[f][c][r][s], taps outside
 * the image contribute 0.  Plain seven-deep loop in double, sequential over (c, r, s). */
void oracle_conv2d_f64(int64_t Nb, int64_t C, int64_t H, int64_t W, int64_t F, int64_t R, int64_t S,
                       int64_t st, int64_t pad, const double* x, const double* w, double* y) {
  const int64_t P = (H + 2 * pad - R) / st + 1, Q = (W + 2 * pad - S) / st + 1;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t n = 0; n < Nb; ++n)
    for (int64_t f = 0; f < F; ++f)
      for (int64_t p = 0; p < P; ++p)
        for (int64_t q = 0; q < Q; ++q) {
          double acc = 0.0;
          for (int64_t c = 0; c < C; ++c)
            for (int64_t r = 0; r < R; ++r)
              for (int64_t s = 0; s < S; ++s) {
                const int64_t ih = p * st - pad + r, iw = q * st - pad + s;
                if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
                acc += x[((n * C + c) * H + ih) * W + iw] * w[((f * C + c) * R + r) * S + s];
              }
          y[((n * F + f) * P + p) * Q + q] = acc;
        }
}
