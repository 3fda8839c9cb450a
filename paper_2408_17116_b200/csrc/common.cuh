// common.cuh — shared types for libcbie (sm_100a): complex128 helpers, device
// tables, physics parameters, error handling, device buffers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cbie.h"

// ---------------------------------------------------------------------------
// complex128 on double2 (16-byte aligned, == numpy complex128 == cbie_c128)
// ---------------------------------------------------------------------------
typedef double2 zc;

__host__ __device__ __forceinline__ zc zmk(double a, double b) { return make_double2(a, b); }
__host__ __device__ __forceinline__ zc zadd(zc a, zc b) { return zmk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ zc zsub(zc a, zc b) { return zmk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ zc zmul(zc a, zc b) {
  return zmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ zc zscale(zc a, double s) { return zmk(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ zc zconj(zc a) { return zmk(a.x, -a.y); }
__host__ __device__ __forceinline__ double zabs2(zc a) { return a.x * a.x + a.y * a.y; }
// a * conj(b)
__host__ __device__ __forceinline__ zc zmulc(zc a, zc b) {
  return zmk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
// conj(a) * b
__host__ __device__ __forceinline__ zc zcmul(zc a, zc b) {
  return zmk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__host__ __device__ __forceinline__ zc zdiv(zc a, zc b) {
  double d = b.x * b.x + b.y * b.y;
  return zmk((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
// acc += a * b
__host__ __device__ __forceinline__ void zfma(zc& acc, zc a, zc b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}
// FP64 tensor-core MMA (DMMA, mma.sync.m8n8k4.f64): D(8x8) += A(8x4) B(4x8) per warp.
// Fragments: a = A[lane / 4][lane % 4], b = B[lane % 4][lane / 4],
// (c0, c1) = C[lane / 4][2 (lane % 4) + {0, 1}].  512 flops per instruction (DFMA: 64).
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
// complex 8x8x4 step: C += A B (4 DMMA; c = {Cr0, Cr1, Ci0, Ci1})
__device__ __forceinline__ void zdmma(double* c, zc a, zc b) {
  dmma(c[0], c[1], a.x, b.x);
  dmma(c[0], c[1], -a.y, b.y);
  dmma(c[2], c[3], a.x, b.y);
  dmma(c[2], c[3], a.y, b.x);
}
// complex 8x8x4 step with the A operand conjugated: C += conj(A) B
__device__ __forceinline__ void zdmma_ca(double* c, zc a, zc b) {
  dmma(c[0], c[1], a.x, b.x);
  dmma(c[0], c[1], a.y, b.y);
  dmma(c[2], c[3], a.x, b.y);
  dmma(c[2], c[3], -a.y, b.x);
}

// Executed FP64 work of the H-LU kernels (SURVEY 8(d) flop convention): every task
// adds its own algorithmic count once, with the ranks it actually saw on the device.
// One counter per translation unit (static), read / reset by CBIE_FLOP_API below.
static __device__ double g_tu_flops;
__device__ __forceinline__ void flop_add(double f) { atomicAdd(&g_tu_flops, f); }
__host__ __device__ inline double flops_qr(double m, double k) {   // thin QR incl. Q formation
  return 16.0 * m * k * k - 16.0 * k * k * k / 3.0;
}
__host__ __device__ inline double flops_trunc(int m, int n, int k, bool dense) {
  if (dense) {   // SVD with vectors of a dense m x n block (R-SVD x 4 for complex)
    const double a = m > n ? m : n, b = m > n ? n : m;
    return 4.0 * (4.0 * a * b * b + 22.0 * b * b * b);
  }
  const double kk = (double)min(min(m, n), k);
  return flops_qr(m, min(m, k)) + flops_qr(n, min(n, k)) + 112.0 * kk * kk * kk;
}
#define CBIE_FLOP_API(name)                                                         \
  double name##_flops_read() {                                                      \
    double v = 0.0;                                                                 \
    cudaMemcpyFromSymbol(&v, g_tu_flops, sizeof(double));                           \
    return v;                                                                       \
  }                                                                                 \
  void name##_flops_reset() {                                                       \
    const double z = 0.0;                                                           \
    cudaMemcpyToSymbol(g_tu_flops, &z, sizeof(double));                             \
  }
// e^{-j k R} for complex k (Im k <= 0 for physical media)
__device__ __forceinline__ zc zexp_mjkR(zc k, double R) {
  double s, c;
  sincos(k.x * R, &s, &c);
  double m = (k.y == 0.0) ? 1.0 : exp(k.y * R);
  return zmk(m * c, -m * s);
}

// ---------------------------------------------------------------------------
// Tables shared by every kernel (passed by value as __grid_constant__).
// ---------------------------------------------------------------------------
#define CBIE_MAXO 16      // max patch order per direction
#define CBIE_MAXS 32      // max oversampled singular-rule order

struct Tables {
  int nu, nv, np, ns;          // patch orders, nodes per patch, rule order
  int npatch, npts, C;
  double xu[CBIE_MAXO], xv[CBIE_MAXO];          // Fejer-1 nodes (descending)
  double wu[CBIE_MAXO], wv[CBIE_MAXO];          // Fejer-1 weights
  double Au[CBIE_MAXO * CBIE_MAXO];             // analysis [m][l]: coeff m from value l
  double Av[CBIE_MAXO * CBIE_MAXO];
  double Du[CBIE_MAXO * CBIE_MAXO];             // node differentiation [l][m]
  double Dv[CBIE_MAXO * CBIE_MAXO];
  double rs[CBIE_MAXS], rw[CBIE_MAXS];          // graded rule: s = sigma^p, w_s
};

struct Phys {
  int kind, C;
  double omega, tau;
  zc k1, k2, eps1, mu1, eps2, mu2;
  zc jump[16];                 // C x C jump matrix (kernels.py:85-100)
  zc rsc[4], csc[4];           // per-component equilibration (solver.py:107-117)
};

// Device-side geometry pointers (all device memory owned by the ctx).
struct Geom {
  const int* kind;             // [npatch] chart kind
  const double* cpar;          // [npatch][8]
  const double* coef;          // [npatch][6][3][nu*nv]; tensors pos,du,dv,duu,duv,dvv; c[n*nv+m]
  const double* star;          // [25] star-body Y_lm coefficients (or null)
  const double* pos;           // node frames [npts][3]
  const double* au;
  const double* av;
  const double* sg;            // [npts]
  const double* wg;            // [npts] Fejer weight * sqrt_g
  const double* bbox;          // [npatch][6]
  const double* diam;          // [npatch]
};

// Near-field table (classification output).
struct NearTab {
  const int32_t* idx;          // [npts][npatch] -> record or -1 (FAR)
  const zc* blk;               // [n_near][C][np*C]
};

// ---------------------------------------------------------------------------
// Host-side errors and buffers
// ---------------------------------------------------------------------------
struct cbie_error : std::runtime_error {
  int code;
  cbie_error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw cbie_error(e_ == cudaErrorMemoryAllocation ? CBIE_EOOM : CBIE_ECUDA,          \
                       std::string(#call) + ": " + cudaGetErrorString(e_) + " @" +         \
                           __FILE__ + ":" + std::to_string(__LINE__));                    \
  } while (0)

// every kernel launch site calls CKL(); it also counts launches (cbie_launch_count)
#include <atomic>
extern std::atomic<long long> g_cbie_launches;
extern std::atomic<long long> g_cbie_frees;   // cudaFree calls (each one synchronises the device)
#define CKL()                 \
  do {                        \
    ++g_cbie_launches;        \
    CK(cudaGetLastError());   \
  } while (0)

// Device allocations come from the device's default stream-ordered memory pool with
// an unbounded release threshold: freed blocks stay mapped and are handed out again,
// so repeated fills / factorisations never unmap memory (cudaFree of large blocks
// stalled concurrently running kernels by up to 2x).  Allocation is ordered on a
// private stream and completed before use; release keeps cudaFree's semantics
// (device-wide synchronisation first).  mem_free_bytes() counts pool-held blocks.
cudaStream_t cbie_alloc_stream();
size_t mem_free_bytes(size_t* total = nullptr);
cudaError_t cbie_malloc(void** p, size_t bytes);
void cbie_free(void* p);

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  bool borrowed = false;   // p is not ours (mapped host memory, cbie_hmatrix_offload): never freed here
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p && !borrowed) {
      cbie_free(p);
      ++g_cbie_frees;
    }
    borrowed = false;
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    if (count == 0) return;
    if (count * sizeof(T) >= ((size_t)1 << 28) && getenv("CBIE_MEMLOG"))   // debug: large allocations
      fprintf(stderr, "[cbie] alloc %zu MiB (free %zu MiB)\n", (count * sizeof(T)) >> 20, mem_free_bytes() >> 20);
    cudaError_t e = cbie_malloc(reinterpret_cast<void**>(&p), count * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      const size_t fr = mem_free_bytes();
      throw cbie_error(e == cudaErrorMemoryAllocation ? CBIE_EOOM : CBIE_ECUDA,
                       std::string("cudaMalloc of ") + std::to_string(count * sizeof(T) >> 20) +
                           " MiB failed (" + cudaGetErrorString(e) + "; free " +
                           std::to_string(fr >> 20) + " MiB)");
    }
    n = count;
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    alloc(count);
    if (count) CK(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& h, cudaStream_t s) { upload(h.data(), h.size(), s); }
  std::vector<T> download(cudaStream_t s) const {
    std::vector<T> h(n);
    if (n) CK(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return h;
  }
};

// Elapsed-time helper on one stream (CUDA events).
struct EvTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  EvTimer() {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
  }
  ~EvTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  void start(cudaStream_t s) { cudaEventRecord(a, s); }
  double stop_ms(cudaStream_t s) {
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
  }
};

static inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }
