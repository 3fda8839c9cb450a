// geometry.cuh — device evaluation of patch charts and Chebyshev interpolants.
//
// Restates geometry.py:48-97 (CubeSphereFace), 196-220 (eval_frames),
// 228-245 (second_derivatives) and chebyshev.py:163-202 (Clenshaw order).
#pragma once
#include "common.cuh"

// Positions feed rel = x_obs - y_src at rule nodes ~1e-10 from the singular
// point, where one ulp of position changes the tested kernel by O(1)
// relative.  Chart and Clenshaw arithmetic therefore use explicitly rounded
// operations (no FMA contraction), in numpy's evaluation order, so positions
// are bit-identical to the reference's.
#define RN_ADD(a, b) __dadd_rn((a), (b))
#define RN_SUB(a, b) __dsub_rn((a), (b))
#define RN_MUL(a, b) __dmul_rn((a), (b))
#define RN_DIV(a, b) __ddiv_rn((a), (b))

__device__ __constant__ static const int kFace[6][4] = {
    {0, +1, 1, 2}, {0, -1, 2, 1}, {1, +1, 2, 0}, {1, -1, 0, 2}, {2, +1, 0, 1}, {2, -1, 1, 0}};

// sum c[n][m] T_n(u) T_m(v); Clenshaw along v first, then u (chebyshev.py:163-202).
__device__ __forceinline__ double clenshaw2(const double* __restrict__ c, int nu, int nv,
                                            double u, double v) {
  double inner[CBIE_MAXO];
  for (int n = 0; n < nu; ++n) {
    const double* cn = c + n * nv;
    double b1 = 0.0, b2 = 0.0;
    for (int m = nv - 1; m > 0; --m) {
      double t = RN_SUB(RN_ADD(cn[m], RN_MUL(RN_MUL(2.0, v), b1)), b2);
      b2 = b1;
      b1 = t;
    }
    inner[n] = RN_SUB(RN_ADD(cn[0], RN_MUL(v, b1)), b2);
  }
  double b1 = 0.0, b2 = 0.0;
  for (int n = nu - 1; n > 0; --n) {
    double t = RN_SUB(RN_ADD(inner[n], RN_MUL(RN_MUL(2.0, u), b1)), b2);
    b2 = b1;
    b1 = t;
  }
  return RN_SUB(RN_ADD(inner[0], RN_MUL(u, b1)), b2);
}

// Cube-sphere chart position + covariant tangents (geometry.py:70-97).
__device__ __forceinline__ void cube_sphere(const double* __restrict__ par, double u, double v,
                                            double pos[3], double au[3], double av[3]) {
  const double R = par[0];
  const int face = (int)par[1];
  const double ulo = par[2], uhi = par[3], vlo = par[4], vhi = par[5];
  const int ax = kFace[face][0], ua = kFace[face][2], va = kFace[face][3];
  const double sg = (double)kFace[face][1];
  double x[3];
  x[ax] = sg;
  x[ua] = RN_ADD(ulo, RN_MUL(RN_MUL(RN_ADD(u, 1.0), 0.5), RN_SUB(uhi, ulo)));
  x[va] = RN_ADD(vlo, RN_MUL(RN_MUL(RN_ADD(v, 1.0), 0.5), RN_SUB(vhi, vlo)));
  const double hu = RN_MUL(0.5, RN_SUB(uhi, ulo)), hv = RN_MUL(0.5, RN_SUB(vhi, vlo));
  const double nrm =
      __dsqrt_rn(RN_ADD(RN_ADD(RN_MUL(x[0], x[0]), RN_MUL(x[1], x[1])), RN_MUL(x[2], x[2])));
  double unit[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    pos[i] = RN_DIV(RN_MUL(R, x[i]), nrm);
    unit[i] = RN_DIV(x[i], nrm);
  }
  const double scale = RN_DIV(R, nrm);
  const double pu = RN_MUL(unit[ua], hu), pv = RN_MUL(unit[va], hv);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double du = (i == ua) ? hu : 0.0, dv = (i == va) ? hv : 0.0;
    au[i] = RN_MUL(scale, RN_SUB(du, RN_MUL(unit[i], pu)));
    av[i] = RN_MUL(scale, RN_SUB(dv, RN_MUL(unit[i], pv)));
  }
}

// Real orthonormal spherical harmonics l = 0..4 (25 functions) as polynomials of
// the unit vector and their Cartesian gradients (extended homogeneously: the
// polynomial form is differentiated, then the tangential chain rule above
// projects it).  Index i = l*l + (m + l).
__device__ __forceinline__ void star_basis(const double xh[3], double Y[25], double dY[25][3]) {
  const double x = xh[0], y = xh[1], z = xh[2];
  const double PI = 3.14159265358979323846;
  // normalisation constants
  const double c00 = 0.5 * sqrt(1.0 / PI);
  const double c1 = sqrt(3.0 / (4.0 * PI));
  const double c2a = 0.5 * sqrt(15.0 / PI), c2b = 0.25 * sqrt(5.0 / PI), c2c = 0.25 * sqrt(15.0 / PI);
  const double c3a = 0.25 * sqrt(35.0 / (2.0 * PI)), c3b = 0.5 * sqrt(105.0 / PI),
               c3c = 0.25 * sqrt(21.0 / (2.0 * PI)), c3d = 0.25 * sqrt(7.0 / PI),
               c3e = 0.25 * sqrt(105.0 / PI);
  const double c4a = 0.75 * sqrt(35.0 / PI), c4b = 0.75 * sqrt(35.0 / (2.0 * PI)),
               c4c = 0.75 * sqrt(5.0 / PI), c4d = 0.75 * sqrt(5.0 / (2.0 * PI)),
               c4e = (3.0 / 16.0) * sqrt(1.0 / PI), c4f = (3.0 / 8.0) * sqrt(5.0 / PI),
               c4g = (3.0 / 16.0) * sqrt(35.0 / PI);
  for (int i = 0; i < 25; ++i) dY[i][0] = dY[i][1] = dY[i][2] = 0.0;
  // l = 0
  Y[0] = c00;
  // l = 1 : m=-1 y, m=0 z, m=1 x
  Y[1] = c1 * y; dY[1][1] = c1;
  Y[2] = c1 * z; dY[2][2] = c1;
  Y[3] = c1 * x; dY[3][0] = c1;
  // l = 2
  Y[4] = c2a * x * y; dY[4][0] = c2a * y; dY[4][1] = c2a * x;
  Y[5] = c2a * y * z; dY[5][1] = c2a * z; dY[5][2] = c2a * y;
  Y[6] = c2b * (3 * z * z - 1); dY[6][2] = c2b * 6 * z;
  Y[7] = c2a * x * z; dY[7][0] = c2a * z; dY[7][2] = c2a * x;
  Y[8] = c2c * (x * x - y * y); dY[8][0] = c2c * 2 * x; dY[8][1] = -c2c * 2 * y;
  // l = 3
  Y[9] = c3a * y * (3 * x * x - y * y); dY[9][0] = c3a * 6 * x * y; dY[9][1] = c3a * (3 * x * x - 3 * y * y);
  Y[10] = c3b * x * y * z; dY[10][0] = c3b * y * z; dY[10][1] = c3b * x * z; dY[10][2] = c3b * x * y;
  Y[11] = c3c * y * (5 * z * z - 1); dY[11][1] = c3c * (5 * z * z - 1); dY[11][2] = c3c * 10 * y * z;
  Y[12] = c3d * z * (5 * z * z - 3); dY[12][2] = c3d * (15 * z * z - 3);
  Y[13] = c3c * x * (5 * z * z - 1); dY[13][0] = c3c * (5 * z * z - 1); dY[13][2] = c3c * 10 * x * z;
  Y[14] = c3e * z * (x * x - y * y); dY[14][0] = c3e * 2 * x * z; dY[14][1] = -c3e * 2 * y * z; dY[14][2] = c3e * (x * x - y * y);
  Y[15] = c3a * x * (x * x - 3 * y * y); dY[15][0] = c3a * (3 * x * x - 3 * y * y); dY[15][1] = -c3a * 6 * x * y;
  // l = 4
  Y[16] = c4a * x * y * (x * x - y * y); dY[16][0] = c4a * (3 * x * x * y - y * y * y); dY[16][1] = c4a * (x * x * x - 3 * x * y * y);
  Y[17] = c4b * y * z * (3 * x * x - y * y); dY[17][0] = c4b * 6 * x * y * z; dY[17][1] = c4b * z * (3 * x * x - 3 * y * y); dY[17][2] = c4b * y * (3 * x * x - y * y);
  Y[18] = c4c * x * y * (7 * z * z - 1); dY[18][0] = c4c * y * (7 * z * z - 1); dY[18][1] = c4c * x * (7 * z * z - 1); dY[18][2] = c4c * 14 * x * y * z;
  Y[19] = c4d * y * z * (7 * z * z - 3); dY[19][1] = c4d * z * (7 * z * z - 3); dY[19][2] = c4d * y * (21 * z * z - 3);
  Y[20] = c4e * (35 * z * z * z * z - 30 * z * z + 3); dY[20][2] = c4e * (140 * z * z * z - 60 * z);
  Y[21] = c4d * x * z * (7 * z * z - 3); dY[21][0] = c4d * z * (7 * z * z - 3); dY[21][2] = c4d * x * (21 * z * z - 3);
  Y[22] = c4f * (x * x - y * y) * (7 * z * z - 1); dY[22][0] = c4f * 2 * x * (7 * z * z - 1); dY[22][1] = -c4f * 2 * y * (7 * z * z - 1); dY[22][2] = c4f * (x * x - y * y) * 14 * z;
  Y[23] = c4b * x * z * (x * x - 3 * y * y); dY[23][0] = c4b * z * (3 * x * x - 3 * y * y); dY[23][1] = -c4b * 6 * x * y * z; dY[23][2] = c4b * x * (x * x - 3 * y * y);
  Y[24] = c4g * (x * x * (x * x - 3 * y * y) - y * y * (3 * x * x - y * y)); dY[24][0] = c4g * (4 * x * x * x - 12 * x * y * y); dY[24][1] = c4g * (4 * y * y * y - 12 * x * x * y);
}

// Star body: r(xhat) = a (1 + amp * f(xhat)) xhat with f a real Y_lm sum, l <= 4,
// composed with the cube -> sphere direction map.  star[0] = a*amp scale folded
// on the host: rad(xhat) = par[0] * (1 + sum_i star[i] Y_i(xhat)).
__device__ __forceinline__ void star_chart(const double* __restrict__ par,
                                           const double* __restrict__ star, double u, double v,
                                           double pos[3], double au[3], double av[3]) {
  const double a = par[0];
  const int face = (int)par[1];
  const double ulo = par[2], uhi = par[3], vlo = par[4], vhi = par[5];
  const int ax = kFace[face][0], ua = kFace[face][2], va = kFace[face][3];
  double x[3];
  x[ax] = (double)kFace[face][1];
  x[ua] = ulo + (u + 1.0) * 0.5 * (uhi - ulo);
  x[va] = vlo + (v + 1.0) * 0.5 * (vhi - vlo);
  const double hu = 0.5 * (uhi - ulo), hv = 0.5 * (vhi - vlo);
  const double nrm = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
  double xh[3], tu[3], tv[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) xh[i] = x[i] / nrm;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    tu[i] = (((i == ua) ? hu : 0.0) - xh[i] * xh[ua] * hu) / nrm;   // d xhat / du
    tv[i] = (((i == va) ? hv : 0.0) - xh[i] * xh[va] * hv) / nrm;
  }
  double Y[25], dY[25][3];
  star_basis(xh, Y, dY);
  double f = 0.0, gf[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < 25; ++i) {
    f += star[i] * Y[i];
    gf[0] += star[i] * dY[i][0];
    gf[1] += star[i] * dY[i][1];
    gf[2] += star[i] * dY[i][2];
  }
  const double r = a * (1.0 + f);
  const double dru = a * (gf[0] * tu[0] + gf[1] * tu[1] + gf[2] * tu[2]);
  const double drv = a * (gf[0] * tv[0] + gf[1] * tv[1] + gf[2] * tv[2]);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    pos[i] = r * xh[i];
    au[i] = dru * xh[i] + r * tu[i];
    av[i] = drv * xh[i] + r * tv[i];
  }
}

// Position + tangents at (u,v) of patch q (chart or Chebyshev interpolant).
__device__ __forceinline__ void patch_eval(const Geom& g, const Tables& t, int q, double u,
                                           double v, double pos[3], double au[3], double av[3]) {
  const int kind = g.kind[q];
  if (kind == CBIE_CHART_CUBE_SPHERE) {
    cube_sphere(g.cpar + 8 * q, u, v, pos, au, av);
  } else if (kind == CBIE_CHART_STAR) {
    star_chart(g.cpar + 8 * q, g.star, u, v, pos, au, av);
  } else {
    const double* c = g.coef + (size_t)q * 18 * t.np;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      pos[i] = clenshaw2(c + (0 * 3 + i) * t.np, t.nu, t.nv, u, v);
      au[i] = clenshaw2(c + (1 * 3 + i) * t.np, t.nu, t.nv, u, v);
      av[i] = clenshaw2(c + (2 * 3 + i) * t.np, t.nu, t.nv, u, v);
    }
  }
}

// r_uu, r_uv, r_vv from the interpolant (geometry.py:228-245).
__device__ __forceinline__ void patch_hessian(const Geom& g, const Tables& t, int q, double u,
                                              double v, double ruu[3], double ruv[3],
                                              double rvv[3]) {
  const double* c = g.coef + (size_t)q * 18 * t.np;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    ruu[i] = clenshaw2(c + (3 * 3 + i) * t.np, t.nu, t.nv, u, v);
    ruv[i] = clenshaw2(c + (4 * 3 + i) * t.np, t.nu, t.nv, u, v);
    rvv[i] = clenshaw2(c + (5 * 3 + i) * t.np, t.nu, t.nv, u, v);
  }
}

__device__ __forceinline__ double cross_norm(const double a[3], const double b[3]) {
  double c0 = a[1] * b[2] - a[2] * b[1];
  double c1 = a[2] * b[0] - a[0] * b[2];
  double c2 = a[0] * b[1] - a[1] * b[0];
  return sqrt(c0 * c0 + c1 * c1 + c2 * c2);
}
