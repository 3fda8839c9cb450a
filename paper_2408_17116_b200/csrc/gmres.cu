// gmres.cu — restarted GMRES on the device H-matvec (the
// reference's iterative path solver.gmres / solve_gmres, solver.py:206-307).
//
// Same algorithm as the reference: zero initial guess, restart length m, Arnoldi
// with one re-orthogonalisation pass, complex Givens rotations, stop when
// |g_{j+1}| / |b| <= tol, true residual checked after every cycle.  The Krylov
// basis V ((m+1) x N), the operator (H-matvec over the compressed leaves) and
// every N-length vector operation stay on the device, in the H-matrix's
// permuted dof order (inner products are permutation invariant); only the
// (m+1) x m Hessenberg matrix and the rotations live on the host.  The
// orthogonalisation is classical Gram-Schmidt applied twice (CGS2: one batched
// projection kernel per pass) instead of the reference's two modified
// Gram-Schmidt sweeps -- the same "one re-orthogonalisation", rounding-level
// different, and one launch per pass instead of j + 1.
#include <algorithm>
#include <cmath>
#include <complex>

#include "hmatrix.h"

void hmat_apply(cbie_hmat* H, const zc* d_xp, zc* d_yp, int nrhs, cudaStream_t s);

namespace {

constexpr int GM_NT = 512;

// out[i] = sum_n conj(V[i][n]) w[n], i < nv (one CTA per basis vector)
__global__ void __launch_bounds__(GM_NT) k_dots(const zc* __restrict__ V, int64_t ld, int nv,
                                                const zc* __restrict__ w, int64_t n, zc* __restrict__ out) {
  const int i = blockIdx.x;
  if (i >= nv) return;
  const zc* v = V + (int64_t)i * ld;
  double sr = 0.0, si = 0.0;
  for (int64_t e = threadIdx.x; e < n; e += GM_NT) {
    const zc a = v[e], b = w[e];
    sr = fma(a.x, b.x, fma(a.y, b.y, sr));
    si = fma(a.x, b.y, fma(-a.y, b.x, si));
  }
  __shared__ double rr[GM_NT / 32], ri[GM_NT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, o);
    si += __shfl_xor_sync(0xffffffffu, si, o);
  }
  if ((threadIdx.x & 31) == 0) {
    rr[threadIdx.x >> 5] = sr;
    ri[threadIdx.x >> 5] = si;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < GM_NT / 32; ++q) {
      a += rr[q];
      b += ri[q];
    }
    out[i] = zmk(a, b);
  }
}

// w[n] -= sum_i h[i] V[i][n]
__global__ void k_project(const zc* __restrict__ V, int64_t ld, int nv, const zc* __restrict__ h, zc* w, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    zc acc = w[e];
    for (int i = 0; i < nv; ++i) acc = zsub(acc, zmul(h[i], V[(int64_t)i * ld + e]));
    w[e] = acc;
  }
}

// y = a x + b y (complex a, b)
__global__ void k_axpby(zc a, const zc* __restrict__ x, zc b, zc* y, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    y[e] = zadd(zmul(a, x[e]), zmul(b, y[e]));
}

// x[n] += sum_j y[j] V[j][n]
__global__ void k_update(const zc* __restrict__ V, int64_t ld, int nv, const zc* __restrict__ y, zc* x, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    zc acc = x[e];
    for (int j = 0; j < nv; ++j) acc = zadd(acc, zmul(y[j], V[(int64_t)j * ld + e]));
    x[e] = acc;
  }
}

using cd = std::complex<double>;

struct Gmres {
  cbie_hmat* H;
  cudaStream_t s;
  int64_t n;
  int grid;
  DBuf<zc> dots, hv;
  explicit Gmres(cbie_hmat* h) : H(h), s(h->ctx->stream), n(h->N) {
    grid = (int)std::min<int64_t>(4 * 148, (n + 255) / 256);
    dots.alloc(1024);
    hv.alloc(1024);
  }
  // host copies of sum conj(V_i) w, i < nv
  std::vector<cd> proj(const zc* V, int64_t ld, int nv, const zc* w) {
    k_dots<<<nv, GM_NT, 0, s>>>(V, ld, nv, w, n, dots.p);
    CKL();
    std::vector<cd> h(nv);
    CK(cudaMemcpyAsync(h.data(), dots.p, sizeof(zc) * nv, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return h;
  }
  void project(const zc* V, int64_t ld, const std::vector<cd>& h, zc* w) {
    CK(cudaMemcpyAsync(hv.p, h.data(), sizeof(zc) * h.size(), cudaMemcpyHostToDevice, s));
    k_project<<<grid, 256, 0, s>>>(V, ld, (int)h.size(), hv.p, w, n);
    CKL();
  }
  double norm(const zc* w) { return std::sqrt(std::max(0.0, proj(w, 0, 1, w)[0].real())); }
  void axpby(cd a, const zc* x, cd b, zc* y) {
    k_axpby<<<grid, 256, 0, s>>>(zmk(a.real(), a.imag()), x, zmk(b.real(), b.imag()), y, n);
    CKL();
  }
};

}  // namespace

extern "C" int cbie_gmres(cbie_hmat* h, const cbie_c128* b, double tol, int restart, int max_iters, cbie_c128* x,
                          int* iterations, double* rel_residual, int* converged) {
  try {
    cudaSetDevice(h->ctx->device);
    if (h->partial) throw cbie_error(CBIE_ESTATE, "partial (sharded) H-matrix: exchange the shards first");
    if (restart < 1 || restart > 1000 || max_iters < 0) throw cbie_error(CBIE_EINVALID, "restart in [1, 1000]");
    Gmres G(h);
    const int64_t n = G.n;
    const Tree& T = h->tree;
    const int C = T.C;
    cudaStream_t s = G.s;
    // permuted right-hand side
    std::vector<zc> bp(n);
    const zc* bb = reinterpret_cast<const zc*>(b);
    for (size_t p = 0; p < T.pperm.size(); ++p)
      for (int c = 0; c < C; ++c) bp[(int64_t)p * C + c] = bb[(int64_t)T.pperm[p] * C + c];
    const int m0 = std::max(1, std::min(restart, std::max(max_iters, 1)));
    DBuf<zc> db, dx, dr, dV;
    db.upload(bp, s);
    dx.alloc(n);
    dr.alloc(n);
    dV.alloc((size_t)(m0 + 1) * n);
    CK(cudaMemsetAsync(dx.p, 0, sizeof(zc) * n, s));
    const double bnorm = G.norm(db.p);
    int total = 0;
    double rel = 0.0;
    bool ok = bnorm == 0.0;
    // r = b - A x
    auto residual = [&]() {
      hmat_apply(h, dx.p, dr.p, 1, s);
      G.axpby(cd(1.0, 0.0), db.p, cd(-1.0, 0.0), dr.p);
      return G.norm(dr.p);
    };
    while (!ok && total < max_iters) {
      const double beta = residual();
      if (beta / bnorm <= tol) {
        rel = beta / bnorm;
        ok = true;
        break;
      }
      const int m = std::min(restart, max_iters - total);
      std::vector<cd> Hm((size_t)(m + 1) * m, cd(0.0)), cs(m), sn(m), g(m + 1, cd(0.0));
      auto Hij = [&](int i, int j) -> cd& { return Hm[(size_t)j * (m + 1) + i]; };
      g[0] = beta;
      G.axpby(cd(1.0 / beta, 0.0), dr.p, cd(0.0, 0.0), dV.p);   // V_0 = r / beta
      int jd = 0;
      for (int j = 0; j < m; ++j) {
        zc* w = dV.p + (int64_t)(j + 1) * n;
        hmat_apply(h, dV.p + (int64_t)j * n, w, 1, s);
        for (int pass = 0; pass < 2; ++pass) {   // Gram-Schmidt + one re-orthogonalisation
          const std::vector<cd> hp = G.proj(dV.p, n, j + 1, w);
          G.project(dV.p, n, hp, w);
          for (int i = 0; i <= j; ++i) Hij(i, j) += hp[i];
        }
        const double hn = G.norm(w);
        Hij(j + 1, j) = hn;
        for (int i = 0; i < j; ++i) {
          const cd t = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
          Hij(i + 1, j) = -std::conj(sn[i]) * Hij(i, j) + std::conj(cs[i]) * Hij(i + 1, j);
          Hij(i, j) = t;
        }
        const double den = std::sqrt(std::norm(Hij(j, j)) + std::norm(Hij(j + 1, j)));
        if (den == 0.0) {
          cs[j] = 1.0;
          sn[j] = 0.0;
        } else {
          cs[j] = std::conj(Hij(j, j)) / den;
          sn[j] = std::conj(Hij(j + 1, j)) / den;
        }
        Hij(j, j) = cs[j] * Hij(j, j) + sn[j] * Hij(j + 1, j);
        Hij(j + 1, j) = 0.0;
        g[j + 1] = -std::conj(sn[j]) * g[j];
        g[j] = cs[j] * g[j];
        ++total;
        jd = j + 1;
        if (std::abs(g[j + 1]) / bnorm <= tol || hn == 0.0 || total >= max_iters) break;
        G.axpby(cd(1.0 / hn, 0.0), w, cd(0.0, 0.0), w);   // V_{j+1} = w / |w|
      }
      // y = Hm[:jd, :jd]^{-1} g[:jd] (upper triangular), x += V[:jd]^T y
      std::vector<cd> y(jd);
      for (int i = jd - 1; i >= 0; --i) {
        cd acc = g[i];
        for (int k = i + 1; k < jd; ++k) acc -= Hij(i, k) * y[k];
        y[i] = acc / Hij(i, i);
      }
      CK(cudaMemcpyAsync(G.hv.p, y.data(), sizeof(zc) * jd, cudaMemcpyHostToDevice, s));
      k_update<<<G.grid, 256, 0, s>>>(dV.p, n, jd, G.hv.p, dx.p, n);
      CKL();
      rel = residual() / bnorm;
      if (rel <= tol) ok = true;
    }
    if (!ok && total >= max_iters) rel = residual() / bnorm;
    std::vector<zc> xp(n);
    CK(cudaMemcpyAsync(xp.data(), dx.p, sizeof(zc) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    zc* xx = reinterpret_cast<zc*>(x);
    for (size_t p = 0; p < T.pperm.size(); ++p)
      for (int c = 0; c < C; ++c) xx[(int64_t)T.pperm[p] * C + c] = xp[(int64_t)p * C + c];
    if (iterations) *iterations = total;
    if (rel_residual) *rel_residual = rel;
    if (converged) *converged = ok ? 1 : 0;
  } catch (const cbie_error& e) {
    h->ctx->err = e.what();
    return e.code;
  }
  return CBIE_OK;
}
