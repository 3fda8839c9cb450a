// context.cu — context, geometry upload, node frames, formulation, C-ABI glue.
//
// Geometry restates geometry.py:100-220 (Patch, eval_frames, node weights) and
// chebyshev.py:32-108 (Fejer-1 rule, transform tables).
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>

#include "context.h"
#include "geometry.cuh"

// ---------------------------------------------------------------------------
// host Chebyshev tables (chebyshev.py:32-108)
// ---------------------------------------------------------------------------
static void fejer_host(int n, double* x, double* w) {
  for (int l = 0; l < n; ++l) {
    double th = (2.0 * l + 1.0) * M_PI / (2.0 * n);
    x[l] = std::cos(th);
    double acc = 1.0;
    for (int m = 1; m <= n / 2; ++m) acc -= 2.0 * std::cos(2.0 * m * th) / (4.0 * m * m - 1.0);
    w[l] = (2.0 / n) * acc;
  }
}

static std::vector<double> vander_host(const double* x, int npts, int n) {
  std::vector<double> V((size_t)npts * n);
  for (int i = 0; i < npts; ++i) {
    V[i * n + 0] = 1.0;
    if (n > 1) V[i * n + 1] = x[i];
    for (int k = 2; k < n; ++k) V[i * n + k] = 2.0 * x[i] * V[i * n + k - 1] - V[i * n + k - 2];
  }
  return V;
}

// analysis[m][l] = (alpha_m / n) T_m(x_l)
static std::vector<double> analysis_host(int n) {
  std::vector<double> x(n), w(n);
  fejer_host(n, x.data(), w.data());
  auto V = vander_host(x.data(), n, n);
  std::vector<double> A((size_t)n * n);
  for (int m = 0; m < n; ++m)
    for (int l = 0; l < n; ++l) A[m * n + l] = ((m == 0 ? 1.0 : 2.0) / n) * V[l * n + m];
  return A;
}

static std::vector<double> dcoef_host(int n) {
  std::vector<double> D((size_t)n * n, 0.0);
  for (int k = 1; k < n; ++k)
    for (int j = k - 1; j >= 0; j -= 2) D[j * n + k] = 2.0 * k;
  for (int k = 0; k < n; ++k) D[0 * n + k] *= 0.5;
  return D;
}

static std::vector<double> matmul(const std::vector<double>& A, const std::vector<double>& B,
                                  int m, int k, int n) {
  std::vector<double> C((size_t)m * n, 0.0);
  for (int i = 0; i < m; ++i)
    for (int p = 0; p < k; ++p) {
      double a = A[i * k + p];
      for (int j = 0; j < n; ++j) C[i * n + j] += a * B[p * n + j];
    }
  return C;
}
static std::vector<double> transpose(const std::vector<double>& A, int m, int n) {
  std::vector<double> T((size_t)n * m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) T[j * m + i] = A[i * n + j];
  return T;
}

static void build_tables(Tables& t, int nu, int nv, int ns, int grading) {
  t.nu = nu;
  t.nv = nv;
  t.np = nu * nv;
  t.ns = ns;
  fejer_host(nu, t.xu, t.wu);
  fejer_host(nv, t.xv, t.wv);
  auto Au = analysis_host(nu), Av = analysis_host(nv);
  std::memcpy(t.Au, Au.data(), sizeof(double) * nu * nu);
  std::memcpy(t.Av, Av.data(), sizeof(double) * nv * nv);
  for (int dir = 0; dir < 2; ++dir) {
    int n = dir == 0 ? nu : nv;
    const double* x = dir == 0 ? t.xu : t.xv;
    auto S = vander_host(x, n, n);
    auto Dn = matmul(matmul(S, dcoef_host(n), n, n, n), dir == 0 ? Au : Av, n, n, n);
    std::memcpy(dir == 0 ? t.Du : t.Dv, Dn.data(), sizeof(double) * n * n);
  }
  // graded rule base on (0,1): s = sigma^p, w_s = (w/2) p sigma^(p-1)  (quadrature.py:154-158)
  double x[CBIE_MAXS], w[CBIE_MAXS];
  fejer_host(ns, x, w);
  for (int i = 0; i < ns; ++i) {
    double sig = 0.5 * (x[i] + 1.0);
    t.rs[i] = std::pow(sig, grading);
    t.rw[i] = 0.5 * w[i] * grading * std::pow(sig, grading - 1);
  }
}

// ---------------------------------------------------------------------------
// node frames kernel (geometry.py:157-174, 196-220)
// ---------------------------------------------------------------------------
__global__ void k_node_frames(const __grid_constant__ Tables t, Geom g, double* pos, double* au,
                              double* av, double* sg, double* wg, int* flag) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= t.npts) return;
  int q = p / t.np, node = p % t.np, l = node % t.nu, k = node / t.nu;
  double x[3], a[3], b[3];
  patch_eval(g, t, q, t.xu[l], t.xv[k], x, a, b);
  double s = cross_norm(a, b);
  double dq = g.diam[q];
  if (!(s >= 1e-14 * dq * dq)) atomicOr(flag, 1);
  for (int i = 0; i < 3; ++i) {
    pos[3 * p + i] = x[i];
    au[3 * p + i] = a[i];
    av[3 * p + i] = b[i];
  }
  sg[p] = s;
  wg[p] = (t.wv[k] * t.wu[l]) * s;
}

void ctx_set_geometry(cbie_ctx* c, int npatch, int nu, int nv, const double* samples,
                      const int* kind, const double* cpar, const double* star,
                      const double* cheb_coef) {
  if (npatch <= 0 || nu < 2 || nv < 2 || nu > CBIE_MAXO || nv > CBIE_MAXO)
    throw cbie_error(CBIE_EINVALID, "invalid patch count or orders (2..16 supported)");
  cudaStream_t s = c->stream;
  c->npatch = npatch;
  c->nu = nu;
  c->nv = nv;
  c->np = nu * nv;
  c->npts = npatch * c->np;
  const int np = c->np;
  c->h_kind.assign(kind, kind + npatch);
  c->h_cpar.assign(cpar, cpar + 8 * (size_t)npatch);
  c->h_samples.assign(samples, samples + (size_t)npatch * np * 3);
  c->h_star.assign(CBIE_STAR_TABLE, 0.0);
  if (star) c->h_star.assign(star, star + CBIE_STAR_TABLE);
  for (int q = 0; q < npatch; ++q)
    if (kind[q] < 0 || kind[q] > 2) throw cbie_error(CBIE_EINVALID, "unknown chart kind");
  // bbox + diameter of the samples (geometry.py:128-135, quadrature.py:73)
  c->h_bbox.assign(6 * (size_t)npatch, 0.0);
  c->h_diam.assign(npatch, 0.0);
  for (int q = 0; q < npatch; ++q) {
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int n = 0; n < np; ++n)
      for (int i = 0; i < 3; ++i) {
        double v = samples[((size_t)q * np + n) * 3 + i];
        lo[i] = std::min(lo[i], v);
        hi[i] = std::max(hi[i], v);
      }
    double d2 = 0;
    for (int i = 0; i < 3; ++i) {
      c->h_bbox[6 * q + i] = lo[i];
      c->h_bbox[6 * q + 3 + i] = hi[i];
      d2 += (hi[i] - lo[i]) * (hi[i] - lo[i]);
    }
    c->h_diam[q] = std::sqrt(d2);
  }
  // Chebyshev coefficient tensors: pos, d/du, d/dv, d2/du2, d2/dudv, d2/dv2
  // (chebyshev.py:133-140, 205-209; geometry.py:137-143, 228-238)
  auto Au = analysis_host(nu), Av = analysis_host(nv);
  auto AvT = transpose(Av, nv, nv);
  auto Dcu = dcoef_host(nu), Dcv = dcoef_host(nv);
  auto DcvT = transpose(Dcv, nv, nv);
  std::vector<double> coef((size_t)npatch * 18 * np);
  std::vector<double> vals((size_t)nu * nv);
  if (cheb_coef) std::memcpy(coef.data(), cheb_coef, sizeof(double) * coef.size());
  for (int q = 0; q < npatch && !cheb_coef; ++q)
    for (int i = 0; i < 3; ++i) {
      for (int l = 0; l < nu; ++l)
        for (int k = 0; k < nv; ++k) vals[l * nv + k] = samples[(((size_t)q * nu + l) * nv + k) * 3 + i];
      auto cc = matmul(matmul(Au, vals, nu, nu, nv), AvT, nu, nv, nv);
      auto cu = matmul(Dcu, cc, nu, nu, nv);
      auto cv = matmul(cc, DcvT, nu, nv, nv);
      auto cuu = matmul(Dcu, cu, nu, nu, nv);
      auto cuv = matmul(cu, DcvT, nu, nv, nv);
      auto cvv = matmul(cv, DcvT, nu, nv, nv);
      const std::vector<double>* T[6] = {&cc, &cu, &cv, &cuu, &cuv, &cvv};
      for (int tt = 0; tt < 6; ++tt)
        std::memcpy(&coef[((size_t)q * 18 + tt * 3 + i) * np], T[tt]->data(), sizeof(double) * np);
    }
  c->d_kind.upload(c->h_kind, s);
  c->d_cpar.upload(c->h_cpar, s);
  c->d_coef.upload(coef, s);
  c->d_star.upload(c->h_star, s);
  c->d_bbox.upload(c->h_bbox, s);
  c->d_diam.upload(c->h_diam, s);
  int ns = c->oversample > 0 ? c->oversample : std::max(2 * std::max(nu, nv), 16);
  build_tables(c->tab, nu, nv, ns, c->grading);
  c->tab.npatch = npatch;
  c->tab.npts = c->npts;
  c->tab.C = c->C;
  c->d_pos.alloc(3 * (size_t)c->npts);
  c->d_au.alloc(3 * (size_t)c->npts);
  c->d_av.alloc(3 * (size_t)c->npts);
  c->d_sg.alloc(c->npts);
  c->d_wg.alloc(c->npts);
  c->d_flag.alloc(4);
  CK(cudaMemsetAsync(c->d_flag.p, 0, 4 * sizeof(int), s));
  k_node_frames<<<ceil_div(c->npts, 128), 128, 0, s>>>(c->tab, c->geom(), c->d_pos.p, c->d_au.p,
                                                        c->d_av.p, c->d_sg.p, c->d_wg.p,
                                                        c->d_flag.p);
  CKL();
  int flag = 0;
  CK(cudaMemcpyAsync(&flag, c->d_flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  c->h_pos.resize(3 * (size_t)c->npts);
  CK(cudaMemcpyAsync(c->h_pos.data(), c->d_pos.p, sizeof(double) * c->h_pos.size(),
                     cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (flag) throw cbie_error(CBIE_EDEGENERATE_PATCH, "patch Jacobian below 1e-14 diam^2 at a node");
  c->has_geom = true;
  c->has_class = false;
}

void ctx_set_formulation(cbie_ctx* c, int kind, double omega, zc k1, zc k2, zc eps1, zc mu1,
                         zc eps2, zc mu2, double tau, int grading, int oversample,
                         const zc* rsc, const zc* csc) {
  if (kind != CBIE_MFIE_PEC && kind != CBIE_MULLER) throw cbie_error(CBIE_EINVALID, "formulation");
  if (grading < 2) throw cbie_error(CBIE_EINVALID, "grading power must be >= 2");
  Phys& p = c->ph;
  p = Phys{};
  p.kind = kind;
  p.C = kind == CBIE_MFIE_PEC ? 2 : 4;
  p.omega = omega;
  p.tau = tau;
  p.k1 = k1;
  p.k2 = k2;
  p.eps1 = eps1;
  p.mu1 = mu1;
  p.eps2 = eps2;
  p.mu2 = mu2;
  for (int i = 0; i < 16; ++i) p.jump[i] = zmk(0, 0);
  if (kind == CBIE_MFIE_PEC) {
    p.jump[0] = p.jump[1 * 4 + 1] = zmk(0.5, 0.0);
  } else {   // kernels.py:95-100
    zc e = zscale(zadd(eps1, eps2), -0.5), m = zscale(zadd(mu1, mu2), 0.5);
    p.jump[0 * 4 + 2] = p.jump[1 * 4 + 3] = e;
    p.jump[2 * 4 + 0] = p.jump[3 * 4 + 1] = m;
  }
  for (int i = 0; i < p.C; ++i) {
    p.rsc[i] = rsc ? rsc[i] : zmk(1, 0);
    p.csc[i] = csc ? csc[i] : zmk(1, 0);
  }
  c->C = p.C;
  c->grading = grading;
  c->oversample = oversample;
  if (oversample > CBIE_MAXS) throw cbie_error(CBIE_EINVALID, "oversample > 32 unsupported");
  c->has_form = true;
  c->has_class = false;
  if (c->has_geom) {
    int ns = oversample > 0 ? oversample : std::max(2 * std::max(c->nu, c->nv), 16);
    build_tables(c->tab, c->nu, c->nv, ns, grading);
    c->tab.npatch = c->npatch;
    c->tab.npts = c->npts;
  }
  c->tab.C = p.C;
  c->N = (int64_t)c->npts * p.C;
}

std::atomic<long long> g_cbie_launches{0};
std::atomic<long long> g_cbie_frees{0};

namespace {
struct PoolState {
  cudaStream_t st = nullptr;
  cudaMemPool_t pool = nullptr;
};
PoolState& pool_state() {
  // never destroyed: buffers held by static objects are released during exit
  static std::mutex* mu = new std::mutex;
  static std::map<int, PoolState>* m = new std::map<int, PoolState>;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(*mu);
  PoolState& P = (*m)[dev];
  if (!P.st) {
    cudaStreamCreateWithFlags(&P.st, cudaStreamNonBlocking);
    cudaDeviceGetDefaultMemPool(&P.pool, dev);
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(P.pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  return P;
}
}  // namespace

cudaStream_t cbie_alloc_stream() { return pool_state().st; }

size_t mem_free_bytes(size_t* total) {
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  PoolState& P = pool_state();
  uint64_t res = 0, used = 0;
  cudaMemPoolGetAttribute(P.pool, cudaMemPoolAttrReservedMemCurrent, &res);
  cudaMemPoolGetAttribute(P.pool, cudaMemPoolAttrUsedMemCurrent, &used);
  if (total) *total = tot;
  return fr + (res > used ? (size_t)(res - used) : 0);
}

cudaError_t cbie_malloc(void** p, size_t bytes) {
  PoolState& P = pool_state();
  cudaError_t e = cudaMallocAsync(p, bytes, P.st);
  if (e == cudaErrorMemoryAllocation) {   // blocks held by the pool of other sizes: give them back, retry
    cudaGetLastError();
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(P.pool, 0);
    e = cudaMallocAsync(p, bytes, P.st);
  }
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(P.st);
}

void cbie_free(void* p) {
  cudaDeviceSynchronize();   // cudaFree semantics: no kernel may still use the block
  cudaFreeAsync(p, pool_state().st);
}

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
#define API_BEGIN(ctx) \
  try {
#define API_END(ctx)                                   \
  }                                                    \
  catch (const cbie_error& e) {                        \
    if (ctx) (ctx)->err = e.what();                    \
    return e.code;                                     \
  }                                                    \
  catch (const std::exception& e) {                    \
    if (ctx) (ctx)->err = e.what();                    \
    return CBIE_EINVALID;                              \
  }                                                    \
  return CBIE_OK;

extern "C" {

int cbie_create(int device, cbie_ctx** out) {
  cbie_ctx* c = nullptr;
  try {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw cbie_error(CBIE_EINVALID, "no such CUDA device");
    CK(cudaSetDevice(device));
    c = new cbie_ctx();
    c->device = device;
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    *out = c;
  } catch (const cbie_error& e) {
    delete c;
    *out = nullptr;
    return e.code;
  }
  return CBIE_OK;
}

void cbie_destroy(cbie_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  cudaStream_t s = c->stream;
  delete c;
  cudaStreamDestroy(s);
}

const char* cbie_last_error(const cbie_ctx* c) { return c ? c->err.c_str() : "null context"; }

int64_t cbie_launch_count(void) { return g_cbie_launches.load(); }

void* cbie_stream(cbie_ctx* c) { return c ? (void*)c->stream : nullptr; }

int cbie_set_geometry(cbie_ctx* c, int npatch, int nu, int nv, const double* samples,
                      const int* chart_kind, const double* chart_params, const double* star_coef,
                      const double* cheb_coef) {
  API_BEGIN(c)
  cudaSetDevice(c->device);
  ctx_set_geometry(c, npatch, nu, nv, samples, chart_kind, chart_params, star_coef, cheb_coef);
  if (c->has_form) c->N = (int64_t)c->npts * c->C;
  API_END(c)
}

int cbie_node_frames(cbie_ctx* c, double* pos, double* au, double* av, double* sg) {
  API_BEGIN(c)
  cudaSetDevice(c->device);
  c->require(c->has_geom, "set geometry first");
  cudaStream_t s = c->stream;
  size_t n = c->npts;
  if (pos) CK(cudaMemcpyAsync(pos, c->d_pos.p, 24 * n, cudaMemcpyDeviceToHost, s));
  if (au) CK(cudaMemcpyAsync(au, c->d_au.p, 24 * n, cudaMemcpyDeviceToHost, s));
  if (av) CK(cudaMemcpyAsync(av, c->d_av.p, 24 * n, cudaMemcpyDeviceToHost, s));
  if (sg) CK(cudaMemcpyAsync(sg, c->d_sg.p, 8 * n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  API_END(c)
}

int cbie_set_formulation(cbie_ctx* c, int kind, double omega, cbie_c128 k1, cbie_c128 k2,
                         cbie_c128 eps1, cbie_c128 mu1, cbie_c128 eps2, cbie_c128 mu2,
                         double tau, int grading, int oversample, const cbie_c128* rsc,
                         const cbie_c128* csc) {
  API_BEGIN(c)
  cudaSetDevice(c->device);
  auto Z = [](cbie_c128 a) { return zmk(a.re, a.im); };
  ctx_set_formulation(c, kind, omega, Z(k1), Z(k2), Z(eps1), Z(mu1), Z(eps2), Z(mu2), tau,
                      grading, oversample, reinterpret_cast<const zc*>(rsc),
                      reinterpret_cast<const zc*>(csc));
  API_END(c)
}

int cbie_classify(cbie_ctx* c, int64_t* n_near, int64_t* n_self, int64_t* n_fallback) {
  API_BEGIN(c)
  cudaSetDevice(c->device);
  c->require(c->has_geom && c->has_form, "cbie_classify needs geometry and formulation");
  ctx_classify(c);
  ctx_near_fill(c);
  if (n_near) *n_near = c->n_near - c->n_self;
  if (n_self) *n_self = c->n_self;
  if (n_fallback) *n_fallback = c->n_fallback;
  API_END(c)
}

int cbie_export_classification(cbie_ctx* c, int64_t cap, int32_t* point, int32_t* patch,
                               int8_t* tag, double* u, double* v, int8_t* ok) {
  API_BEGIN(c)
  cudaSetDevice(c->device);
  c->require(c->has_class, "classify first");
  if (cap < c->n_near) throw cbie_error(CBIE_EINVALID, "export capacity too small");
  size_t n = c->n_near;
  cudaStream_t s = c->stream;
  if (n) {
    CK(cudaMemcpyAsync(point, c->d_near_pt.p, n * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(patch, c->d_near_q.p, n * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(tag, c->d_near_tag.p, n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ok, c->d_near_ok.p, n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(u, c->d_near_u.p, n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(v, c->d_near_v.p, n * 8, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  API_END(c)
}

int cbie_pair_block(cbie_ctx* c, int64_t point, int patch, cbie_c128* out) {
  API_BEGIN(c)
  cudaSetDevice(c->device);
  c->require(c->has_class, "classify first");
  if (point < 0 || point >= c->npts || patch < 0 || patch >= c->npatch)
    throw cbie_error(CBIE_EINVALID, "pair index out of range");
  ctx_pair_block(c, point, patch, reinterpret_cast<zc*>(out));
  API_END(c)
}

int cbie_fill_block(cbie_ctx* c, const int64_t* rows, int64_t m, const int64_t* cols, int64_t n,
                    int scaled, cbie_c128* out) {
  API_BEGIN(c)
  cudaSetDevice(c->device);
  c->require(c->has_class, "classify first");
  ctx_fill_block(c, rows, m, cols, n, scaled, reinterpret_cast<zc*>(out));
  API_END(c)
}

int cbie_fill_dense(cbie_ctx* c, int64_t cap, cbie_c128* out) {
  API_BEGIN(c)
  cudaSetDevice(c->device);
  c->require(c->has_class, "classify first");
  if (c->N > cap) throw cbie_error(CBIE_ECAP_EXCEEDED, "N exceeds dense cap");
  ctx_fill_dense(c, reinterpret_cast<zc*>(out));
  API_END(c)
}

}  // extern "C"

std::string stats_to_json(const std::map<std::string, double>& m) {
  std::ostringstream o;
  o.precision(17);
  o << "{";
  bool first = true;
  for (auto& kv : m) {
    if (!first) o << ",";
    first = false;
    o << "\"" << kv.first << "\":" << kv.second;
  }
  o << "}";
  return o.str();
}

std::string hmat_stats(const cbie_hmat* h);
std::string hlu_stats(const cbie_hlu* f);

extern "C" int cbie_stats_json(const void* h, int which, char* buf, size_t cap) {
  if (!h || !buf || cap == 0) return CBIE_EINVALID;
  std::string s = which == 0   ? stats_to_json(((const cbie_ctx*)h)->stat)
                  : which == 1 ? hmat_stats((const cbie_hmat*)h)
                               : hlu_stats((const cbie_hlu*)h);
  if (s.size() + 1 > cap) return CBIE_EINVALID;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return CBIE_OK;
}
