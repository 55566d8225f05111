/* Strict-order GEMM oracle -- TEST INFRASTRUCTURE ONLY.
 *
 * Restates the reference matmul (pkg/src/ssagrad/tensor.py:351-361):
 *   C[i,j] = (((a_i0*b_0j) + a_i1*b_1j) + ...) in ascending k,
 * every product and every sum rounded separately (no FMA contraction:
 * build with -ffp-contract=off).  In float64 this is bit-identical to the
 * reference's cumsum kernel; in float32 it is the strict-fp32 mode the GPU
 * must match bit for bit.  Row-major; j is the inner loop so each C[i,j]
 * still folds over k in ascending order.
 */
#include <stddef.h>
#include <string.h>

void oracle_gemm_f32(const float* A, const float* B, float* C, long m, long k, long n) {
  for (long i = 0; i < m; ++i) {
    float* c = C + i * n;
    for (long j = 0; j < n; ++j) c[j] = 0.0f;
    for (long kk = 0; kk < k; ++kk) {
      const float a = A[i * k + kk];
      const float* b = B + kk * n;
      if (kk == 0) {
        for (long j = 0; j < n; ++j) c[j] = a * b[j];
      } else {
        for (long j = 0; j < n; ++j) {
          float p = a * b[j];
          c[j] = c[j] + p;
        }
      }
    }
  }
}

void oracle_gemm_f64(const double* A, const double* B, double* C, long m, long k, long n) {
  for (long i = 0; i < m; ++i) {
    double* c = C + i * n;
    for (long kk = 0; kk < k; ++kk) {
      const double a = A[i * k + kk];
      const double* b = B + kk * n;
      if (kk == 0) {
        for (long j = 0; j < n; ++j) c[j] = a * b[j];
      } else {
        for (long j = 0; j < n; ++j) {
          double p = a * b[j];
          c[j] = c[j] + p;
        }
      }
    }
  }
}
