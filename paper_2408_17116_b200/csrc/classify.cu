// classify.cu — K1: FAR/NEAR/SELF classification of every (point, patch) pair.
//
// Restates EntryGenerator._classify_patch_column (assembly.py:106-143) and the
// lock-step damped Newton closest point (quadrature.py:87-140).  This file is
// compiled with -fmad=false so the Newton arithmetic rounds like the numpy
// reference (its convergence flag decides which singular rule is used).
//
// Pipeline (all on device, deterministic):
//   k_screen    bbox prescreen over npts*npatch pairs (point-major) -> flags
//   select      cub::DeviceSelect::Flagged -> candidate pair ids (sorted)
//   k_newton    closest point for every candidate -> tag, uv, converged
//   select      non-FAR candidates -> near records (sorted by (point, patch))
//   k_index     [npts][npatch] -> record index table (-1 = FAR)
#include <cub/cub.cuh>

#include "context.h"
#include "geometry.cuh"

namespace {

__global__ void k_screen(const __grid_constant__ Tables t, Geom g, double tau, uint8_t* flags) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)t.npts * t.npatch;
  if (idx >= total) return;
  int p = (int)(idx / t.npatch), q = (int)(idx % t.npatch);
  uint8_t f;
  if (p / t.np == q) {
    f = 1;   // SELF from the dof map, never from geometry (assembly.py:110-111)
  } else {
    const double* lo = g.bbox + 6 * q;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double x = g.pos[3 * p + i];
      double gap = fmax(0.0, fmax(lo[i] - x, x - lo[3 + i]));
      s += gap * gap;
    }
    // FAR if |gap| >= tau * diam * 1.25  (assembly.py:117-119, quadrature.py:28)
    f = (sqrt(s) >= tau * g.diam[q] * 1.25) ? 0 : 1;
  }
  flags[idx] = f;
}

// numpy's einsum("mx,mx->m") over a length-3 axis sums (x0 + x2) + x1 (its
// SIMD pairing); the Newton dots follow that order (quadrature.py:112-119).
__device__ __forceinline__ double dot3(const double a[3], const double b[3]) {
  return (a[0] * b[0] + a[2] * b[2]) + a[1] * b[1];
}

__global__ void k_newton(const __grid_constant__ Tables t, Geom g, double tau,
                         const int64_t* __restrict__ cand, int64_t ncand, int8_t* tag, double* uo,
                         double* vo, int8_t* oko, unsigned long long* nfallback) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncand) return;
  int64_t idx = cand[c];
  int p = (int)(idx / t.npatch), q = (int)(idx % t.npatch);
  if (p / t.np == q) {   // SELF: uv of the point's own node
    int node = p % t.np;
    tag[c] = CBIE_SELF;
    uo[c] = t.xu[node % t.nu];
    vo[c] = t.xv[node / t.nu];
    oko[c] = 1;
    return;
  }
  double x[3] = {g.pos[3 * p], g.pos[3 * p + 1], g.pos[3 * p + 2]};
  // seed = argmin |x|^2 - (2x) @ r^T + |r|^2 over the patch nodes (quadrature.py:96-99).
  // The symmetric cube-sphere mesh makes exact ties common, so the rounding
  // must match the reference: einsum order for the squares and the FMA chain
  // of the BLAS dgemm that evaluates (2 obs) @ nodes.T on the build host.
  const double xx = dot3(x, x);
  const double x2[3] = {2.0 * x[0], 2.0 * x[1], 2.0 * x[2]};
  int seed = 0;
  double best = 0.0;
  for (int n = 0; n < t.np; ++n) {
    const double* r = g.pos + 3 * ((int64_t)q * t.np + n);
    double xr = fma(x2[2], r[2], fma(x2[1], r[1], x2[0] * r[0]));
    double rr = dot3(r, r);
    double d2 = (xx - xr) + rr;
    if (n == 0 || d2 < best) {
      best = d2;
      seed = n;
    }
  }
  const double u0 = t.xu[seed % t.nu], v0 = t.xv[seed / t.nu];
  double u = u0, v = v0;
  bool ok = false;
  for (int it = 0; it < 30; ++it) {
    double pos[3], au[3], av[3], ruu[3], ruv[3], rvv[3], d[3];
    patch_eval(g, t, q, u, v, pos, au, av);
    patch_hessian(g, t, q, u, v, ruu, ruv, rvv);
    for (int i = 0; i < 3; ++i) d[i] = pos[i] - x[i];
    double g0 = 2.0 * dot3(au, d), g1 = 2.0 * dot3(av, d);
    double auu = dot3(au, au), auv = dot3(au, av), avv = dot3(av, av);
    double h00 = 2.0 * (auu + dot3(ruu, d));
    double h01 = 2.0 * (auv + dot3(ruv, d));
    double h11 = 2.0 * (avv + dot3(rvv, d));
    double det = h00 * h11 - h01 * h01;
    if (det <= 1e-30 || h00 <= 0) {   // Gauss-Newton fallback (quadrature.py:121-126)
      h00 = 2.0 * auu;
      h01 = 2.0 * auv;
      h11 = 2.0 * avv;
      det = h00 * h11 - h01 * h01;
    }
    double su = -(h11 * g0 - h01 * g1) / det;
    double sv = -(-h01 * g0 + h00 * g1) / det;
    double un = fmin(fmax(u + su, -1.05), 1.05);
    double vn = fmin(fmax(v + sv, -1.05), 1.05);
    double moved = fmax(fabs(un - u), fabs(vn - v));
    u = un;
    v = vn;
    if (moved < 1e-12) {
      ok = true;
      break;
    }
  }
  if (!ok) {   // non-converged points fall back to the seed node (quadrature.py:136)
    u = u0;
    v = v0;
    atomicAdd(nfallback, 1ull);
  }
  u = fmin(fmax(u, -1.0), 1.0);
  v = fmin(fmax(v, -1.0), 1.0);
  double pos[3], au[3], av[3];
  patch_eval(g, t, q, u, v, pos, au, av);
  double d0 = pos[0] - x[0], d1 = pos[1] - x[1], d2 = pos[2] - x[2];
  double dist = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
  tag[c] = (dist < tau * g.diam[q]) ? CBIE_NEAR : CBIE_FAR;
  uo[c] = u;
  vo[c] = v;
  oko[c] = ok ? 1 : 0;
}

__global__ void k_count(const uint8_t* f, int64_t n, unsigned long long* out) {
  int64_t base = (int64_t)blockIdx.x * 1024;
  unsigned v = 0;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x)
    if (base + i < n) v += f[base + i];
  typedef cub::BlockReduce<unsigned, 256> BR;
  __shared__ typename BR::TempStorage ts;
  unsigned tot = BR(ts).Sum(v);
  if (threadIdx.x == 0 && tot) atomicAdd(out, (unsigned long long)tot);
}

__global__ void k_nonfar(const int8_t* tag, int64_t n, uint8_t* f) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = tag[i] != CBIE_FAR;
}

__global__ void k_gather(const int64_t* sel, int64_t nsel, const int64_t* cand, const int8_t* tag,
                         const double* u, const double* v, const int8_t* ok, int npatch,
                         int32_t* pt, int32_t* pq, int8_t* otag, double* ou, double* ov,
                         int8_t* ook, int32_t* idxtab) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nsel) return;
  int64_t c = sel[r];
  int64_t idx = cand[c];
  pt[r] = (int32_t)(idx / npatch);
  pq[r] = (int32_t)(idx % npatch);
  otag[r] = tag[c];
  ou[r] = u[c];
  ov[r] = v[c];
  ook[r] = ok[c];
  idxtab[idx] = (int32_t)r;
}

}  // namespace

void ctx_classify(cbie_ctx* c) {
  cudaStream_t s = c->stream;
  EvTimer tm;
  tm.start(s);
  const int64_t total = (int64_t)c->npts * c->npatch;
  const double tau = c->ph.tau;
  DBuf<uint8_t> flags;
  flags.alloc(total);
  k_screen<<<ceil_div(total, 256), 256, 0, s>>>(c->tab, c->geom(), tau, flags.p);
  CKL();
  DBuf<int64_t> cand, nsel;
  nsel.alloc(1);
  size_t tmp_bytes = 0;
  cub::CountingInputIterator<int64_t> it(0);
  {
    // exact candidate count first, so the candidate list is sized exactly
    CK(cudaMemsetAsync(nsel.p, 0, 8, s));
    k_count<<<ceil_div(total, 1024), 256, 0, s>>>(flags.p, total,
                                                 reinterpret_cast<unsigned long long*>(nsel.p));
    CKL();
    int64_t nc = 0;
    CK(cudaMemcpyAsync(&nc, nsel.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cand.alloc(std::max<int64_t>(nc, 1));
  }
  CK(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, it, flags.p, cand.p, nsel.p, total, s));
  DBuf<char> tmp;
  tmp.alloc(tmp_bytes);
  CK(cub::DeviceSelect::Flagged(tmp.p, tmp_bytes, it, flags.p, cand.p, nsel.p, total, s));
  int64_t ncand = 0;
  CK(cudaMemcpyAsync(&ncand, nsel.p, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  c->n_cand = ncand;
  DBuf<int8_t> tag, ok;
  DBuf<double> u, v;
  DBuf<unsigned long long> nfb;
  tag.alloc(ncand);
  ok.alloc(ncand);
  u.alloc(ncand);
  v.alloc(ncand);
  nfb.alloc(1);
  CK(cudaMemsetAsync(nfb.p, 0, 8, s));
  if (ncand)
    k_newton<<<ceil_div(ncand, 128), 128, 0, s>>>(c->tab, c->geom(), tau, cand.p, ncand, tag.p,
                                                   u.p, v.p, ok.p, nfb.p);
  CKL();
  DBuf<uint8_t> f2;
  f2.alloc(std::max<int64_t>(ncand, 1));
  if (ncand) k_nonfar<<<ceil_div(ncand, 256), 256, 0, s>>>(tag.p, ncand, f2.p);
  CKL();
  DBuf<int64_t> sel;
  sel.alloc(std::max<int64_t>(ncand, 1));
  size_t tb2 = 0;
  cub::CountingInputIterator<int64_t> it2(0);
  CK(cub::DeviceSelect::Flagged(nullptr, tb2, it2, f2.p, sel.p, nsel.p, ncand, s));
  DBuf<char> tmp2;
  tmp2.alloc(std::max<size_t>(tb2, 1));
  CK(cub::DeviceSelect::Flagged(tmp2.p, tb2, it2, f2.p, sel.p, nsel.p, ncand, s));
  int64_t nnear = 0;
  unsigned long long hfb = 0;
  CK(cudaMemcpyAsync(&nnear, nsel.p, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&hfb, nfb.p, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  c->n_near = nnear;
  c->n_self = c->npts;   // every point is SELF against its own patch
  c->n_fallback = (int64_t)hfb;
  c->d_nearidx.alloc(total);
  CK(cudaMemsetAsync(c->d_nearidx.p, 0xFF, total * sizeof(int32_t), s));
  c->d_near_pt.alloc(nnear);
  c->d_near_q.alloc(nnear);
  c->d_near_tag.alloc(nnear);
  c->d_near_u.alloc(nnear);
  c->d_near_v.alloc(nnear);
  c->d_near_ok.alloc(nnear);
  if (nnear)
    k_gather<<<ceil_div(nnear, 256), 256, 0, s>>>(sel.p, nnear, cand.p, tag.p, u.p, v.p, ok.p,
                                                  c->npatch, c->d_near_pt.p, c->d_near_q.p,
                                                  c->d_near_tag.p, c->d_near_u.p, c->d_near_v.p,
                                                  c->d_near_ok.p, c->d_nearidx.p);
  CKL();
  c->stat["classify_ms"] = tm.stop_ms(s);
  c->stat["n_candidates"] = (double)ncand;
  c->stat["n_near_records"] = (double)nnear;
  c->stat["n_fallback"] = (double)hfb;
  c->has_class = true;
}
