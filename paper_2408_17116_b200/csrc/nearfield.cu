// nearfield.cu — K3: near/self pair blocks with the graded corner-split rule.
//
// One CTA per NEAR/SELF record (point p, source patch q).  For each of the <= 4
// rectangles of the singular rule (quadrature.py:143-183) every thread
// evaluates the chart frame and the tested kernel at one rule node
// (kernels.py:234-287), the weighted integrand goes to shared memory, and the
// rule -> cardinal contraction (assembly.py:337-370, chebyshev.py:217-236) is
// done sum-factorised: first over the v-nodes against Pv, then over the
// u-nodes against Pu, accumulating the C x (np*C) pair block in registers.
// SELF records add the jump matrix (assembly.py:211-212).
#include "context.h"
#include "geometry.cuh"
#include "physics.cuh"

namespace {

constexpr int NT = 256;

// rows contracted per node: MFIE 4 (b*2+c) vs P; Muller 12 (g*2+b) vs P + 2 TdG rows
template <int C> struct Rows;
template <> struct Rows<2> { static constexpr int Y = 4, Z = 4, O = 4; };
template <> struct Rows<4> { static constexpr int Y = 14, Z = 16, O = 16; };

template <int C>
__global__ void __launch_bounds__(NT) k_near_blocks(const __grid_constant__ Tables t, Geom g,
                                                    const __grid_constant__ Phys ph,
                                                    const int32_t* __restrict__ rpt,
                                                    const int32_t* __restrict__ rq,
                                                    const int8_t* __restrict__ rtag,
                                                    const double* __restrict__ ru,
                                                    const double* __restrict__ rv, zc* out) {
  constexpr int RY = Rows<C>::Y, RZ = Rows<C>::Z, RO = Rows<C>::O;
  constexpr int MAXNODE = CBIE_MAXS * CBIE_MAXS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ns = t.ns, nu = t.nu, nv = t.nv, np = t.np;
  zc* Y = reinterpret_cast<zc*>(smem_raw);                 // [ns*ns][RY]
  zc* Z = Y + (size_t)ns * ns * RY;                          // [ns][nv][RZ]
  double* Pu = reinterpret_cast<double*>(Z + (size_t)ns * nv * RZ);   // [ns][nu]
  double* dPu = Pu + ns * nu;
  double* Pv = dPu + ns * nu;                                // [ns][nv]
  double* dPv = Pv + ns * nv;
  __shared__ double s_ru[CBIE_MAXS], s_rv[CBIE_MAXS];
  (void)MAXNODE;

  const int rec = blockIdx.x;
  const int p = rpt[rec], q = rq[rec];
  const double us = ru[rec], vs = rv[rec];
  const double xo[3] = {g.pos[3 * p], g.pos[3 * p + 1], g.pos[3 * p + 2]};
  const double auo[3] = {g.au[3 * p], g.au[3 * p + 1], g.au[3 * p + 2]};
  const double avo[3] = {g.av[3 * p], g.av[3 * p + 1], g.av[3 * p + 2]};

  // outputs owned by this thread: o = tid + NT*i over RO*np entries, layout [r][k*nu+l]
  constexpr int MAXO = (RO * CBIE_MAXO * CBIE_MAXO + NT - 1) / NT;
  zc acc[MAXO];
#pragma unroll
  for (int i = 0; i < MAXO; ++i) acc[i] = zmk(0.0, 0.0);
  const int nout = RO * np;

  for (int su = 0; su < 2; ++su) {
    const double ulo = su == 0 ? -1.0 : us, uhi = su == 0 ? us : 1.0;
    if (fabs(uhi - ulo) < 1e-12) continue;
    const double fu = su == 0 ? -1.0 : 1.0;
    for (int sv = 0; sv < 2; ++sv) {
      const double vlo = sv == 0 ? -1.0 : vs, vhi = sv == 0 ? vs : 1.0;
      if (fabs(vhi - vlo) < 1e-12) continue;
      const double fv = sv == 0 ? -1.0 : 1.0;
      __syncthreads();   // previous rectangle's consumers are done
      if (threadIdx.x < ns) {
        // u = u* + s (far - u*), rounded like numpy (quadrature.py:166, 173)
        s_ru[threadIdx.x] = __dadd_rn(us, __dmul_rn(t.rs[threadIdx.x], __dsub_rn(fu, us)));
        s_rv[threadIdx.x] = __dadd_rn(vs, __dmul_rn(t.rs[threadIdx.x], __dsub_rn(fv, vs)));
      }
      __syncthreads();
      // 1-D cardinal tables at this rectangle's nodes (chebyshev.py:217-236)
      for (int e = threadIdx.x; e < ns * (nu + nv); e += NT) {
        const bool isu = e < ns * nu;
        const int n = isu ? nu : nv;
        const int a = isu ? e / nu : (e - ns * nu) / nv;
        const int l = isu ? e % nu : (e - ns * nu) % nv;
        const double x = isu ? s_ru[a] : s_rv[a];
        const double* A = isu ? t.Au : t.Av;
        // T_m(x) and T_m'(x) = m U_{m-1}(x)
        double T0 = 1.0, T1 = x, U0 = 1.0, U1 = 2.0 * x;
        double val = A[0 * n + l], dval = 0.0;
        if (n > 1) {
          val += T1 * A[1 * n + l];
          dval += U0 * A[1 * n + l];
        }
        for (int m = 2; m < n; ++m) {
          double T2 = 2.0 * x * T1 - T0;
          val += T2 * A[m * n + l];
          dval += m * U1 * A[m * n + l];
          double U2 = 2.0 * x * U1 - U0;
          T0 = T1;
          T1 = T2;
          U0 = U1;
          U1 = U2;
        }
        if (isu) {
          Pu[a * nu + l] = val;
          dPu[a * nu + l] = dval;
        } else {
          Pv[a * nv + l] = val;
          dPv[a * nv + l] = dval;
        }
      }
      // rule nodes: weighted integrand into Y
      const double lu = fabs(fu - us), lv = fabs(fv - vs);
      for (int nd = threadIdx.x; nd < ns * ns; nd += NT) {
        const int a = nd / ns, b = nd % ns;
        const double u = s_ru[a], v = s_rv[b];
        const double w = (t.rw[a] * lu) * (t.rw[b] * lv);
        double ys[3], aus[3], avs[3];
        patch_eval(g, t, q, u, v, ys, aus, avs);
        const double sgs = cross_norm(aus, avs);
        const double d0 = ys[0] - xo[0], d1 = ys[1] - xo[1], d2 = ys[2] - xo[2];
        const bool keep = (d0 * d0 + d1 * d1 + d2 * d2) > 1e-28;   // assembly.py:196-201
        const double wg = keep ? w * sgs : 0.0;
        zc* y = Y + (size_t)nd * RY;
        if (!keep) {
#pragma unroll
          for (int r = 0; r < RY; ++r) y[r] = zmk(0.0, 0.0);
          continue;
        }
        if constexpr (C == 2) {
          zc B[2][2];
          mfie_block(ph.k1, xo, auo, avo, ys, aus, avs, sgs, B);
          y[0] = zscale(B[0][0], wg);
          y[1] = zscale(B[0][1], wg);
          y[2] = zscale(B[1][0], wg);
          y[3] = zscale(B[1][1], wg);
        } else {
          zc T6[6][2], TdG[2];
          muller_fields(ph, xo, auo, avo, ys, aus, avs, sgs, T6, TdG);
#pragma unroll
          for (int gg = 0; gg < 6; ++gg)
#pragma unroll
            for (int bb = 0; bb < 2; ++bb) y[gg * 2 + bb] = zscale(T6[gg][bb], wg);
          y[12] = zscale(TdG[0], wg);
          y[13] = zscale(TdG[1], wg);
        }
      }
      __syncthreads();
      // step 1: Z[a][k][r] = sum_b Y[a][b][r] * (Pv or dPv)[b][k]
      for (int e = threadIdx.x; e < ns * nv * RZ; e += NT) {
        const int r = e % RZ, k = (e / RZ) % nv, a = e / (RZ * nv);
        int ry = r;
        const double* Tv = Pv;
        if (C == 4 && r >= 14) {   // TdG rows against dP/dv
          ry = r - 2;
          Tv = dPv;
        }
        zc s = zmk(0.0, 0.0);
        const zc* y = Y + (size_t)a * ns * RY + ry;
        for (int b = 0; b < ns; ++b) {
          const double pv = Tv[b * nv + k];
          const zc yy = y[(size_t)b * RY];
          s.x = fma(yy.x, pv, s.x);
          s.y = fma(yy.y, pv, s.y);
        }
        Z[e] = s;
      }
      __syncthreads();
      // step 2: acc[r][k][l] += sum_a Z[a][k][r] * (Pu or dPu)[a][l]
#pragma unroll
      for (int i = 0; i < MAXO; ++i) {
        const int o = threadIdx.x + NT * i;
        if (o >= nout) break;
        const int r = o / np, j = o % np, k = j / nu, l = j % nu;
        const double* Tu = (C == 4 && r >= 12 && r < 14) ? dPu : Pu;
        zc s = acc[i];
        for (int a = 0; a < ns; ++a) {
          const double pu = Tu[a * nu + l];
          const zc z = Z[((size_t)a * nv + k) * RZ + r];
          s.x = fma(z.x, pu, s.x);
          s.y = fma(z.y, pu, s.y);
        }
        acc[i] = s;
      }
    }
  }
  // scatter rows into the C x (np*C) pair block
  zc* blk = out + (size_t)rec * C * np * C;
  if constexpr (C == 2) {
#pragma unroll
    for (int i = 0; i < MAXO; ++i) {
      const int o = threadIdx.x + NT * i;
      if (o >= nout) break;
      const int r = o / np, j = o % np, b = r / 2, c = r % 2;
      blk[(size_t)b * np * 2 + j * 2 + c] = acc[i];
    }
    __syncthreads();
    if (rtag[rec] == CBIE_SELF && threadIdx.x < 4) {
      const int n0 = p % np, b = threadIdx.x / 2, c = threadIdx.x % 2;
      zc* e = blk + (size_t)b * np * 2 + n0 * 2 + c;
      *e = zadd(*e, ph.jump[b * 4 + c]);
    }
  } else {
    // stage W (12 rows), Wu (2), Wv (2) through shared memory, then assemble
    __syncthreads();
    zc* W = Y;   // reuse: [16][np]
#pragma unroll
    for (int i = 0; i < MAXO; ++i) {
      const int o = threadIdx.x + NT * i;
      if (o >= nout) break;
      W[o] = acc[i];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 4 * np * 4; e += NT) {
      const int b = e / (np * 4), j = (e / 4) % np, c = e % 4;
      const int bb = b & 1;
      int gsel;
      bool div = false;
      if (b < 2) {
        gsel = c;                 // W[0..3]
        div = c < 2;
      } else {
        const int m[4] = {4, 5, 0, 1};
        gsel = m[c];
        div = c >= 2;
      }
      zc v = W[(gsel * 2 + bb) * np + j];
      if (div) {
        const int dr = (c % 2 == 0) ? 12 : 14;   // Wu rows 12..13, Wv rows 14..15
        v = zadd(v, W[(dr + bb) * np + j]);
      }
      if (rtag[rec] == CBIE_SELF && j == p % np) v = zadd(v, ph.jump[b * 4 + c]);
      blk[(size_t)b * np * 4 + j * 4 + c] = v;
    }
  }
}

template <int C>
size_t near_smem(const Tables& t) {
  return (size_t)t.ns * t.ns * Rows<C>::Y * sizeof(zc) + (size_t)t.ns * t.nv * Rows<C>::Z * sizeof(zc) +
         (size_t)2 * t.ns * (t.nu + t.nv) * sizeof(double);
}

}  // namespace

void ctx_near_fill(cbie_ctx* c) {
  cudaStream_t s = c->stream;
  const int C = c->C;
  const int64_t n = c->n_near;
  c->d_near_blk.alloc((size_t)std::max<int64_t>(n, 1) * C * c->np * C);
  if (n == 0) return;
  EvTimer tm;
  tm.start(s);
  if (C == 2) {
    size_t sm = near_smem<2>(c->tab);
    CK(cudaFuncSetAttribute(k_near_blocks<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_near_blocks<2><<<(unsigned)n, NT, sm, s>>>(c->tab, c->geom(), c->ph, c->d_near_pt.p,
                                                 c->d_near_q.p, c->d_near_tag.p, c->d_near_u.p,
                                                 c->d_near_v.p, c->d_near_blk.p);
  } else {
    size_t sm = near_smem<4>(c->tab);
    sm = std::max(sm, (size_t)16 * c->np * sizeof(zc));
    CK(cudaFuncSetAttribute(k_near_blocks<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_near_blocks<4><<<(unsigned)n, NT, sm, s>>>(c->tab, c->geom(), c->ph, c->d_near_pt.p,
                                                 c->d_near_q.p, c->d_near_tag.p, c->d_near_u.p,
                                                 c->d_near_v.p, c->d_near_blk.p);
  }
  CKL();
  c->stat["near_fill_ms"] = tm.stop_ms(s);
}
