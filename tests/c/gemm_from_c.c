/* The C ABI used from plain C (no Python, no torch): a bf16 tensor-core GEMM
 * with the bias + sigmoid epilogue through sg_gemm, checked against a double
 * precision product of the same bf16 values, and an argument error reported
 * through sg_last_error.  Built and run by tests/test_c_abi_gpu.py. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "sgb200.h"

static unsigned short f2bf(float f) {
  unsigned u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (unsigned short)(u >> 16);
}
static float bf2f(unsigned short h) {
  unsigned u = ((unsigned)h) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main(void) {
  const int M = 300, N = 200, K = 136;
  sg_ctx* ctx = NULL;
  if (sg_create(0, &ctx) != SG_OK) {
    fprintf(stderr, "sg_create failed\n");
    return 1;
  }
  unsigned short* a = malloc(sizeof(unsigned short) * M * K);
  unsigned short* b = malloc(sizeof(unsigned short) * N * K);
  float* bias = malloc(sizeof(float) * N);
  float* out = malloc(sizeof(float) * M * N);
  srand(7);
  for (int i = 0; i < M * K; ++i) a[i] = f2bf((float)rand() / RAND_MAX * 2.0f - 1.0f);
  for (int i = 0; i < N * K; ++i) b[i] = f2bf(((float)rand() / RAND_MAX * 2.0f - 1.0f) * 0.1f);
  for (int j = 0; j < N; ++j) bias[j] = (float)rand() / RAND_MAX * 0.2f - 0.1f;
  void *da, *db, *dbias, *dout;
  cudaMalloc(&da, sizeof(unsigned short) * M * K);
  cudaMalloc(&db, sizeof(unsigned short) * N * K);
  cudaMalloc(&dbias, sizeof(float) * N);
  cudaMalloc(&dout, sizeof(float) * M * N);
  cudaMemcpy(da, a, sizeof(unsigned short) * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b, sizeof(unsigned short) * N * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dbias, bias, sizeof(float) * N, cudaMemcpyHostToDevice);

  sg_gemm_desc d;
  memset(&d, 0, sizeof d);
  d.M = M, d.N = N, d.K = K;
  d.A = da, d.lda = K;
  d.B = db, d.ldb = K;
  d.precision = SG_PREC_BF16;
  d.epilogue = SG_EPI_BIAS_ACT;
  d.act = SG_ACT_SIGMOID;
  d.bias = dbias;
  d.out = dout, d.ld_out = N;
  d.batch = 1;
  if (sg_gemm(ctx, &d, NULL) != SG_OK) {
    char msg[256];
    sg_last_error(msg, sizeof msg);
    fprintf(stderr, "sg_gemm failed: %s\n", msg);
    return 1;
  }
  cudaDeviceSynchronize();
  cudaMemcpy(out, dout, sizeof(float) * M * N, cudaMemcpyDeviceToHost);
  double worst = 0.0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double z = bias[j];
      for (int k = 0; k < K; ++k) z += (double)bf2f(a[i * K + k]) * (double)bf2f(b[j * K + k]);
      const double y = 1.0 / (1.0 + exp(-z));
      const double e = fabs(out[i * N + j] - y);
      if (e > worst) worst = e;
    }
  /* argument errors come back as SG_EINVAL with a message, no launch */
  d.K = 0;
  const int rc = sg_gemm(ctx, &d, NULL);
  char msg[256] = {0};
  sg_last_error(msg, sizeof msg);
  printf("max_abs_err %.3e einval %d msg %s\n", worst, rc == SG_EINVAL, msg);
  sg_destroy(ctx);
  return (worst <= 1e-5 && rc == SG_EINVAL) ? 0 : 2;
}
