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

// Star body (config 4): r(xhat) = a (1 + f(xhat)) xhat, f = sum_lm c_lm Y_lm, l <= 4,
// composed with the cube -> sphere direction map.  The host expands f and its
// Cartesian gradient into the 35 monomials x^a y^b z^c of degree <= 4
// (geometry.py star_tables: star[0..34] = f, [35..69] = df/dx, [70..104] = df/dy,
// [105..139] = df/dz) and evaluates them with the same explicitly rounded
// operation order (geometry.py star_eval), so chart positions and tangents are
// bit-identical on host and device.
__device__ __forceinline__ double star_poly(const double* __restrict__ F, const double px[5],
                                            const double py[5], const double pz[5]) {
  double s = 0.0;
  int m = 0;
#pragma unroll
  for (int deg = 0; deg <= 4; ++deg)
#pragma unroll
    for (int a = deg; a >= 0; --a)
#pragma unroll
      for (int b = deg - a; b >= 0; --b, ++m)
        s = RN_ADD(s, RN_MUL(RN_MUL(RN_MUL(F[m], px[a]), py[b]), pz[deg - a - b]));
  return s;
}

__device__ __forceinline__ void star_chart(const double* __restrict__ par,
                                           const double* __restrict__ star, double u, double v,
                                           double pos[3], double au[3], double av[3]) {
  const double a = par[0];
  const int face = (int)par[1];
  const double ulo = par[2], uhi = par[3], vlo = par[4], vhi = par[5];
  const int ax = kFace[face][0], ua = kFace[face][2], va = kFace[face][3];
  double x[3];
  x[ax] = (double)kFace[face][1];
  x[ua] = RN_ADD(ulo, RN_MUL(RN_MUL(RN_ADD(u, 1.0), 0.5), RN_SUB(uhi, ulo)));
  x[va] = RN_ADD(vlo, RN_MUL(RN_MUL(RN_ADD(v, 1.0), 0.5), RN_SUB(vhi, vlo)));
  const double hu = RN_MUL(0.5, RN_SUB(uhi, ulo)), hv = RN_MUL(0.5, RN_SUB(vhi, vlo));
  const double nrm =
      __dsqrt_rn(RN_ADD(RN_ADD(RN_MUL(x[0], x[0]), RN_MUL(x[1], x[1])), RN_MUL(x[2], x[2])));
  double xh[3], tu[3], tv[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) xh[i] = RN_DIV(x[i], nrm);
#pragma unroll
  for (int i = 0; i < 3; ++i) {    // d xhat / du, d xhat / dv
    tu[i] = RN_DIV(RN_SUB((i == ua) ? hu : 0.0, RN_MUL(RN_MUL(xh[i], xh[ua]), hu)), nrm);
    tv[i] = RN_DIV(RN_SUB((i == va) ? hv : 0.0, RN_MUL(RN_MUL(xh[i], xh[va]), hv)), nrm);
  }
  double px[5], py[5], pz[5];
  px[0] = py[0] = pz[0] = 1.0;
  px[1] = xh[0]; py[1] = xh[1]; pz[1] = xh[2];
#pragma unroll
  for (int k = 2; k <= 4; ++k) {
    px[k] = RN_MUL(px[k - 1], xh[0]);
    py[k] = RN_MUL(py[k - 1], xh[1]);
    pz[k] = RN_MUL(pz[k - 1], xh[2]);
  }
  const double f = star_poly(star, px, py, pz);
  const double gx = star_poly(star + 35, px, py, pz);
  const double gy = star_poly(star + 70, px, py, pz);
  const double gz = star_poly(star + 105, px, py, pz);
  const double r = RN_MUL(a, RN_ADD(1.0, f));
  const double dru = RN_MUL(a, RN_ADD(RN_ADD(RN_MUL(gx, tu[0]), RN_MUL(gy, tu[1])), RN_MUL(gz, tu[2])));
  const double drv = RN_MUL(a, RN_ADD(RN_ADD(RN_MUL(gx, tv[0]), RN_MUL(gy, tv[1])), RN_MUL(gz, tv[2])));
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    pos[i] = RN_MUL(r, xh[i]);
    au[i] = RN_ADD(RN_MUL(dru, xh[i]), RN_MUL(r, tu[i]));
    av[i] = RN_ADD(RN_MUL(drv, xh[i]), RN_MUL(r, tv[i]));
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
