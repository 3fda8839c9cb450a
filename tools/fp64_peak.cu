// FP64 peak probe for the roofline denominator (MEASURED_PEAKS.json has no FP64 key).
// (1) DFMA-chain microkernel, (2) cuBLAS DGEMM / ZGEMM 8192^3 best-of-10.
#include <cstdio>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cuComplex.h>

__global__ void dfma_chain(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

// (3) DMMA (mma.sync.m8n8k4.f64) chain: 8 independent accumulators per warp
__global__ void dmma_chain(double* out, int iters) {
  double a = 1e-3 * (threadIdx.x & 31), b = 1.0 - a;
  double c[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = q;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096; int threads = 512; int blocks = sms * 4;
  dfma_chain<<<blocks, threads>>>(d, 16, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_chain<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
  printf("{\"probe\":\"dfma_chain\",\"tflops\":%.3f,\"ms\":%.3f,\"sms\":%d}\n", flops / best / 1e9, best, sms);

  for (int wpb = 4; wpb <= 16; wpb *= 2) {
    const int th = 32 * wpb, bl = sms * (wpb == 4 ? 8 : wpb == 8 ? 4 : 2);
    dmma_chain<<<bl, th>>>(d, 16);
    cudaDeviceSynchronize();
    best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      dmma_chain<<<bl, th>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double fl = 512.0 * 8 * (double)iters * (th / 32) * bl;
    printf("{\"probe\":\"dmma_chain\",\"warps_per_sm\":%d,\"tflops\":%.3f,\"ms\":%.3f}\n", th / 32 * bl / sms, fl / best / 1e9, best);
  }

  cublasHandle_t h; cublasCreate(&h);
  for (int z = 0; z < 2; ++z) {
    int n = 8192; size_t es = z ? 16 : 8;
    void *A, *B, *C; cudaMalloc(&A, es * n * n); cudaMalloc(&B, es * n * n); cudaMalloc(&C, es * n * n);
    cudaMemset(A, 0, es * n * n); cudaMemset(B, 0, es * n * n);
    double one = 1, zero = 0; cuDoubleComplex cone = make_cuDoubleComplex(1, 0), czero = make_cuDoubleComplex(0, 0);
    best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0);
      if (z) cublasZgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &cone, (cuDoubleComplex*)A, n, (cuDoubleComplex*)B, n, &czero, (cuDoubleComplex*)C, n);
      else cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, (double*)A, n, (double*)B, n, &zero, (double*)C, n);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r > 0 && ms < best) best = ms;
    }
    double fl = (z ? 8.0 : 2.0) * n * (double)n * n;
    printf("{\"probe\":\"%s\",\"n\":%d,\"tflops\":%.3f,\"ms\":%.3f}\n", z ? "cublas_zgemm" : "cublas_dgemm", n, fl / best / 1e9, best);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
