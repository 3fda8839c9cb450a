// farfield.cu — radiation sums of the far field / bistatic RCS on the device
// (postprocess.far_field, postprocess.py:193-212).
//
// The reference forms the phase matrix exp(j k rhat @ pos^T) (angles x nodes,
// 880 MB at config 5 for a 361-angle cut) and multiplies it with the quadrature
// tables (w a_u F^u + w a_v F^v, w div F, and the M tables for Muller).  Here
// every CTA takes one angle and a chunk of nodes, evaluates the phase with one
// sincos per node (node positions resident from cbie_set_geometry, tables read
// once, coalesced) and reduces its ntab complex sums; a second pass adds the
// chunk partials in a fixed order (deterministic, no atomics).
#include <algorithm>

#include "context.h"

#define API_BEGIN(ctx) \
  try {
#define API_END(ctx)                \
  }                                 \
  catch (const cbie_error& e) {     \
    if (ctx) (ctx)->err = e.what(); \
    return e.code;                  \
  }                                 \
  catch (const std::exception& e) { \
    if (ctx) (ctx)->err = e.what(); \
    return CBIE_EINVALID;           \
  }                                 \
  return CBIE_OK;

namespace {

constexpr int FF_NT = 256;
constexpr int FF_CHUNK = 8192;   // nodes per CTA
constexpr int FF_MAXTAB = 8;

__global__ void __launch_bounds__(FF_NT) k_far_partial(const double* __restrict__ pos, int64_t npts,
                                                       const zc* __restrict__ tab, int ntab,
                                                       const double* __restrict__ rhat, double k, int nchunk,
                                                       zc* __restrict__ part) {
  const int a = blockIdx.x, ch = blockIdx.y;
  const double rx = rhat[3 * a], ry = rhat[3 * a + 1], rz = rhat[3 * a + 2];
  double sr[FF_MAXTAB], si[FF_MAXTAB];
#pragma unroll
  for (int t = 0; t < FF_MAXTAB; ++t) sr[t] = si[t] = 0.0;
  const int64_t n0 = (int64_t)ch * FF_CHUNK, n1 = min(npts, n0 + FF_CHUNK);
  for (int64_t n = n0 + threadIdx.x; n < n1; n += FF_NT) {
    const double ph = k * (rx * pos[3 * n] + ry * pos[3 * n + 1] + rz * pos[3 * n + 2]);
    double s, c;
    sincos(ph, &s, &c);
#pragma unroll
    for (int t = 0; t < FF_MAXTAB; ++t)
      if (t < ntab) {
        const zc w = tab[n * ntab + t];
        sr[t] = fma(c, w.x, fma(-s, w.y, sr[t]));
        si[t] = fma(c, w.y, fma(s, w.x, si[t]));
      }
  }
  __shared__ double red[2][FF_MAXTAB][FF_NT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < FF_MAXTAB; ++t) {
    double x = sr[t], y = si[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      x += __shfl_xor_sync(0xffffffffu, x, o);
      y += __shfl_xor_sync(0xffffffffu, y, o);
    }
    if (lane == 0) {
      red[0][t][w] = x;
      red[1][t][w] = y;
    }
  }
  __syncthreads();
  if (threadIdx.x < ntab) {
    const int t = threadIdx.x;
    double x = 0.0, y = 0.0;
    for (int q = 0; q < FF_NT / 32; ++q) {
      x += red[0][t][q];
      y += red[1][t][q];
    }
    part[((int64_t)a * nchunk + ch) * ntab + t] = zmk(x, y);
  }
}

__global__ void k_far_sum(const zc* __restrict__ part, int nang, int nchunk, int ntab, zc* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nang * ntab) return;
  const int a = e / ntab, t = e % ntab;
  zc s = zmk(0.0, 0.0);
  for (int c = 0; c < nchunk; ++c) s = zadd(s, part[((int64_t)a * nchunk + c) * ntab + t]);
  out[e] = s;
}

}  // namespace

extern "C" int cbie_far_field_sums(cbie_ctx* c, const cbie_c128* tab, int ntab, const double* rhat, int nang,
                                   double k, cbie_c128* out) {
  API_BEGIN(c)
  cudaSetDevice(c->device);
  c->require(c->has_geom, "set geometry first");
  if (ntab < 1 || ntab > FF_MAXTAB) throw cbie_error(CBIE_EINVALID, "ntab in [1, 8]");
  if (nang < 0) throw cbie_error(CBIE_EINVALID, "nang >= 0");
  if (nang > 0) {
  cudaStream_t s = c->stream;
  const int64_t npts = c->npts;
  const int nchunk = (int)std::max<int64_t>(1, (npts + FF_CHUNK - 1) / FF_CHUNK);
  DBuf<zc> dtab, dpart, dout;
  DBuf<double> drh;
  dtab.alloc((size_t)npts * ntab);
  CK(cudaMemcpyAsync(dtab.p, tab, sizeof(zc) * npts * ntab, cudaMemcpyHostToDevice, s));
  drh.alloc((size_t)3 * nang);
  CK(cudaMemcpyAsync(drh.p, rhat, sizeof(double) * 3 * nang, cudaMemcpyHostToDevice, s));
  dpart.alloc((size_t)nang * nchunk * ntab);
  dout.alloc((size_t)nang * ntab);
  k_far_partial<<<dim3(nang, nchunk), FF_NT, 0, s>>>(c->d_pos.p, npts, dtab.p, ntab, drh.p, k, nchunk, dpart.p);
  CKL();
  k_far_sum<<<(nang * ntab + 255) / 256, 256, 0, s>>>(dpart.p, nang, nchunk, ntab, dout.p);
  CKL();
  CK(cudaMemcpyAsync(out, dout.p, sizeof(zc) * nang * ntab, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  }
  API_END(c)
}
