// physics.cuh — tested Helmholtz integrands (complex128) for one
// (observation point, source point) pair.
//
// Restates kernels.py:181-287 (greens, grad_greens, greens_diff,
// grad_greens_diff, mfie_tested_fields, muller_tested_fields) and the
// vectorised far path assembly.py:378-431.
#pragma once
#include "common.cuh"

#define CBIE_INV4PI 0.079577471545947667884   // 1/(4 pi)

__device__ __forceinline__ zc zsin(zc z) {
  if (z.y == 0.0) return zmk(sin(z.x), 0.0);
  double s, c;
  sincos(z.x, &s, &c);
  return zmk(s * cosh(z.y), c * sinh(z.y));
}
__device__ __forceinline__ zc zcos(zc z) {
  if (z.y == 0.0) return zmk(cos(z.x), 0.0);
  double s, c;
  sincos(z.x, &s, &c);
  return zmk(c * cosh(z.y), -s * sinh(z.y));
}
// sin x - x cos x with the |x| < 0.05 series (kernels.py:196-203)
__device__ __forceinline__ zc zsin_minus_xcos(zc x) {
  if (sqrt(zabs2(x)) < 0.05) {
    zc x2 = zmul(x, x);
    zc t = zsub(zmk(1.0 / 840.0, 0.0), zscale(x2, 1.0 / 45360.0));
    t = zadd(zmk(-1.0 / 30.0, 0.0), zmul(x2, t));
    t = zadd(zmk(1.0 / 3.0, 0.0), zmul(x2, t));
    return zmul(zmul(x, x2), t);
  }
  return zsub(zsin(x), zmul(x, zcos(x)));
}

// MFIE tested curl kernel B[b][c] / sqrt(g') (kernels.py:234-246):
//   grad G = -(1 + jkR) e^{-jkR} rel / (4 pi R^3),  K_c = -grad G x a_c',
//   row 0 = -a_v(obs) . K_c,  row 1 = +a_u(obs) . K_c.
__device__ __forceinline__ void mfie_block(zc k, const double xo[3], const double auo[3],
                                           const double avo[3], const double ys[3],
                                           const double aus[3], const double avs[3],
                                           double sgs, zc B[2][2]) {
  const double r0 = xo[0] - ys[0], r1 = xo[1] - ys[1], r2 = xo[2] - ys[2];
  const double R = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
  const zc e = zexp_mjkR(k, R);
  // (1 + j k R)
  const zc one_jkR = zmk(1.0 - k.y * R, k.x * R);
  const double inv = -CBIE_INV4PI / (R * R * R);
  const zc f = zscale(zmul(one_jkR, e), inv);
  // K_c = -(g x a_c) = a_c x g,  g = f rel.  tested: t . (a_c x rel) f
  // row 0: -a_v(obs) . (a_c x rel) ; row 1: a_u(obs) . (a_c x rel)
  const double inv_sg = 1.0 / sgs;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const double* a = c == 0 ? aus : avs;
    const double x0 = a[1] * r2 - a[2] * r1;
    const double x1 = a[2] * r0 - a[0] * r2;
    const double x2 = a[0] * r1 - a[1] * r0;
    const double t0 = -(avo[0] * x0 + avo[1] * x1 + avo[2] * x2) * inv_sg;
    const double t1 = (auo[0] * x0 + auo[1] * x1 + auo[2] * x2) * inv_sg;
    B[0][c] = zscale(f, t0);
    B[1][c] = zscale(f, t1);
  }
}

// Muller compact generators (kernels.py:249-287):
//   T6[g][b], g = sJ a_u, sJ a_v, cM x a_u, cM x a_v, cJ x a_u, cJ x a_v;
//   TdG[b] divergence kernel; all / sqrt(g').
__device__ __forceinline__ void muller_fields(const Phys& ph, const double xo[3],
                                              const double auo[3], const double avo[3],
                                              const double ys[3], const double aus[3],
                                              const double avs[3], double sgs, zc T6[6][2],
                                              zc TdG[2]) {
  const double rel[3] = {xo[0] - ys[0], xo[1] - ys[1], xo[2] - ys[2]};
  const double R = sqrt(rel[0] * rel[0] + rel[1] * rel[1] + rel[2] * rel[2]);
  const zc k1 = ph.k1, k2 = ph.k2;
  const zc s = zscale(zadd(k1, k2), 0.5), d = zscale(zsub(k1, k2), 0.5);
  const zc e2 = zexp_mjkR(k2, R), es = zexp_mjkR(s, R);
  const zc dR = zscale(d, R);
  const zc sdR = zsin(dR);
  const double i4piR = CBIE_INV4PI / R, i4piR3 = CBIE_INV4PI / (R * R * R);
  const zc G2 = zscale(e2, i4piR);
  const zc Gd = zscale(zmul(zmul(es, zmk(0.0, -2.0)), sdR), i4piR);
  const zc f2 = zscale(zmul(zmk(1.0 - k2.y * R, k2.x * R), e2), -i4piR3);
  // 2 e^{-jsR} (j S(dR) - R s sin(dR)) / (4 pi R^3)
  const zc S = zsin_minus_xcos(dR);
  const zc fd = zscale(zmul(es, zsub(zmul(zmk(0.0, 1.0), S), zmul(zscale(s, R), sdR))),
                       2.0 * i4piR3);
  const zc em1 = zmul(ph.eps1, ph.mu1), em2 = zmul(ph.eps2, ph.mu2);
  const zc sJ = zmul(zmk(0.0, ph.omega), zadd(zmul(em1, Gd), zmul(zsub(em1, em2), G2)));
  // cM = eps1 gd + (eps1-eps2) g2 = (eps1 fd + (eps1-eps2) f2) rel
  const zc fM = zadd(zmul(ph.eps1, fd), zmul(zsub(ph.eps1, ph.eps2), f2));
  const zc fJ = zscale(zadd(zmul(ph.mu1, fd), zmul(zsub(ph.mu1, ph.mu2), f2)), -1.0);
  const double inv_sg = 1.0 / sgs;
  // tested projections of real vectors
  auto tst = [&](const double X[3], int b) {
    return b == 0 ? -(avo[0] * X[0] + avo[1] * X[1] + avo[2] * X[2])
                  : (auo[0] * X[0] + auo[1] * X[1] + auo[2] * X[2]);
  };
  double ru[3], rv[3];   // rel x a_u', rel x a_v'
  ru[0] = rel[1] * aus[2] - rel[2] * aus[1];
  ru[1] = rel[2] * aus[0] - rel[0] * aus[2];
  ru[2] = rel[0] * aus[1] - rel[1] * aus[0];
  rv[0] = rel[1] * avs[2] - rel[2] * avs[1];
  rv[1] = rel[2] * avs[0] - rel[0] * avs[2];
  rv[2] = rel[0] * avs[1] - rel[1] * avs[0];
  // TdG = t(gd / (-j omega)) = fd t(rel) / (-j omega)
  const zc fdG = zdiv(fd, zmk(0.0, -ph.omega));
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    const double tu = tst(aus, b) * inv_sg, tv = tst(avs, b) * inv_sg;
    const double tru = tst(ru, b) * inv_sg, trv = tst(rv, b) * inv_sg;
    T6[0][b] = zscale(sJ, tu);
    T6[1][b] = zscale(sJ, tv);
    T6[2][b] = zscale(fM, tru);
    T6[3][b] = zscale(fM, trv);
    T6[4][b] = zscale(fJ, tru);
    T6[5][b] = zscale(fJ, trv);
    TdG[b] = zscale(fdG, tst(rel, b) * inv_sg);
  }
}
