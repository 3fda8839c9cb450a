// entry.cuh — the on-the-fly matrix entry generator shared by the dense fill,
// the dense-leaf fill and the ACA row/column generators.
//
// For (observation point p, source point j): if (p, patch(j)) is NEAR/SELF the
// C x C block is gathered from the near pair-block table (computed once by
// nearfield.cu); otherwise the FAR formula is evaluated on the source patch's
// native Fejer grid (assembly.py:182-190, 305-334, 378-431).  For Muller the
// FAR derivative columns go through the node-differentiation matrices along
// the source node's u-line / v-line (assembly.py:215-226).
#pragma once
#include "geometry.cuh"
#include "physics.cuh"

template <int C>
__device__ __forceinline__ void entry_block(const Tables& t, const Geom& g, const Phys& ph,
                                            const NearTab& nt, int p, int j, zc out[C][C]) {
  const int np = t.np;
  const int q = j / np, node = j % np;
  const int rec = nt.idx[(int64_t)p * t.npatch + q];
  if (rec >= 0) {
    const zc* blk = nt.blk + (size_t)rec * C * np * C + (size_t)node * C;
#pragma unroll
    for (int b = 0; b < C; ++b)
#pragma unroll
      for (int c = 0; c < C; ++c) out[b][c] = blk[(size_t)b * np * C + c];
    return;
  }
  const double xo[3] = {g.pos[3 * p], g.pos[3 * p + 1], g.pos[3 * p + 2]};
  const double auo[3] = {g.au[3 * p], g.au[3 * p + 1], g.au[3 * p + 2]};
  const double avo[3] = {g.av[3 * p], g.av[3 * p + 1], g.av[3 * p + 2]};
  if constexpr (C == 2) {
    const double ys[3] = {g.pos[3 * j], g.pos[3 * j + 1], g.pos[3 * j + 2]};
    const double aus[3] = {g.au[3 * j], g.au[3 * j + 1], g.au[3 * j + 2]};
    const double avs[3] = {g.av[3 * j], g.av[3 * j + 1], g.av[3 * j + 2]};
    zc B[2][2];
    mfie_block(ph.k1, xo, auo, avo, ys, aus, avs, g.sg[j], B);
    const double w = g.wg[j];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) out[b][c] = zscale(B[b][c], w);
  } else {
    auto fields = [&](int jj, zc T6[6][2], zc TdG[2]) {
      const double ys[3] = {g.pos[3 * jj], g.pos[3 * jj + 1], g.pos[3 * jj + 2]};
      const double aus[3] = {g.au[3 * jj], g.au[3 * jj + 1], g.au[3 * jj + 2]};
      const double avs[3] = {g.av[3 * jj], g.av[3 * jj + 1], g.av[3 * jj + 2]};
      muller_fields(ph, xo, auo, avo, ys, aus, avs, g.sg[jj], T6, TdG);
    };
    zc T6[6][2], TdG[2];
    fields(j, T6, TdG);
    const double w = g.wg[j];
    // value block (kernels.py:290-302)
    const int gmap[2][4] = {{0, 1, 2, 3}, {4, 5, 0, 1}};
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) out[b][c] = zscale(T6[gmap[b >> 1][c]][b & 1], w);
    // derivative columns: u-line for even c, v-line for odd c
    const int base = q * np, k = node / t.nu, m = node % t.nu;
    zc du[2] = {zmk(0, 0), zmk(0, 0)}, dv[2] = {zmk(0, 0), zmk(0, 0)};
    for (int l = 0; l < t.nu; ++l) {
      const int jj = base + k * t.nu + l;
      zc T6b[6][2], Tb[2];
      fields(jj, T6b, Tb);
      const double f = g.wg[jj] * t.Du[l * t.nu + m];
      du[0] = zadd(du[0], zscale(Tb[0], f));
      du[1] = zadd(du[1], zscale(Tb[1], f));
    }
    for (int kk = 0; kk < t.nv; ++kk) {
      const int jj = base + kk * t.nu + m;
      zc T6b[6][2], Tb[2];
      fields(jj, T6b, Tb);
      const double f = g.wg[jj] * t.Dv[kk * t.nv + k];
      dv[0] = zadd(dv[0], zscale(Tb[0], f));
      dv[1] = zadd(dv[1], zscale(Tb[1], f));
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int c0 = (b < 2) ? 0 : 2;
      out[b][c0] = zadd(out[b][c0], du[b & 1]);
      out[b][c0 + 1] = zadd(out[b][c0 + 1], dv[b & 1]);
    }
  }
}
