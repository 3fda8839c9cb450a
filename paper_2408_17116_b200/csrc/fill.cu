// fill.cu — K2/K4: dense-block fill kernels built on entry_block().
//
//   k_fill_entries   arbitrary (rows, cols) sub-block, row-major: EntryGenerator.block /
//                    row_segment / col_segment / entry (assembly.py:229-271) and the
//                    EquilibratedGenerator scaling (solver.py:119-129)
//   k_fill_dense     full matrix in row chunks: assemble_dense (assembly.py:438-460)
//   k_fill_tiles     H-matrix dense leaves in permuted order, column-major tiles
//                    (HMatrix._fill_leaf dense branch, hmatrix.py:245-248)
#include "context.h"
#include "entry.cuh"

namespace {

template <int C>
__global__ void k_fill_entries(const __grid_constant__ Tables t, Geom g,
                               const __grid_constant__ Phys ph, NearTab nt,
                               const int64_t* __restrict__ rows, int64_t m,
                               const int64_t* __restrict__ cols, int64_t n, int scaled, zc* out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * n) return;
  const int64_t i = rows[e / n], j = cols[e % n];
  const int p = (int)(i / C), b = (int)(i % C), pj = (int)(j / C), c = (int)(j % C);
  zc blk[C][C];
  entry_block<C>(t, g, ph, nt, p, pj, blk);
  zc v = blk[b][c];
  if (scaled) v = zmul(v, zmul(ph.rsc[b], ph.csc[c]));
  out[e] = v;
}

// one thread per (row point, column point) pair; rows [p0, p0+nrow) x all points
template <int C>
__global__ void k_fill_dense(const __grid_constant__ Tables t, Geom g,
                             const __grid_constant__ Phys ph, NearTab nt, int p0, int nrow,
                             zc* out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int npts = t.npts;
  if (e >= (int64_t)nrow * npts) return;
  const int p = p0 + (int)(e / npts), j = (int)(e % npts);
  zc blk[C][C];
  entry_block<C>(t, g, ph, nt, p, j, blk);
  const int64_t N = (int64_t)npts * C;
#pragma unroll
  for (int b = 0; b < C; ++b)
#pragma unroll
    for (int c = 0; c < C; ++c) out[((int64_t)(p - p0) * C + b) * N + (int64_t)j * C + c] = blk[b][c];
}

// one CTA per tile; column-major tile (ld = rows), optional equilibration
template <int C>
__global__ void __launch_bounds__(256) k_fill_tiles(const __grid_constant__ Tables t, Geom g,
                                                    const __grid_constant__ Phys ph, NearTab nt,
                                                    const TileDesc* __restrict__ tiles,
                                                    const int32_t* __restrict__ pperm,
                                                    zc* arena, int scaled) {
  const TileDesc td = tiles[blockIdx.x];
  const int mr = td.r_hi - td.r_lo, nc = td.c_hi - td.c_lo;
  const int ld = mr * C;
  zc* T = arena + td.out_off;
  for (int e = threadIdx.x; e < mr * nc; e += blockDim.x) {
    const int a = e % mr, bcol = e / mr;   // consecutive threads -> consecutive rows
    const int p = pperm[td.r_lo + a], j = pperm[td.c_lo + bcol];
    zc blk[C][C];
    entry_block<C>(t, g, ph, nt, p, j, blk);
#pragma unroll
    for (int b = 0; b < C; ++b)
#pragma unroll
      for (int c = 0; c < C; ++c) {
        zc v = blk[b][c];
        if (scaled) v = zmul(v, zmul(ph.rsc[b], ph.csc[c]));
        T[(int64_t)(bcol * C + c) * ld + a * C + b] = v;
      }
  }
}

}  // namespace

void launch_fill_tiles(const cbie_ctx* c, const TileDesc* d_tiles, int ntiles,
                       const int32_t* d_pperm, zc* d_arena, int scaled, cudaStream_t s) {
  if (ntiles == 0) return;
  if (c->C == 2)
    k_fill_tiles<2><<<ntiles, 256, 0, s>>>(c->tab, c->geom(), c->ph, c->near(), d_tiles, d_pperm,
                                           d_arena, scaled);
  else
    k_fill_tiles<4><<<ntiles, 256, 0, s>>>(c->tab, c->geom(), c->ph, c->near(), d_tiles, d_pperm,
                                           d_arena, scaled);
  CKL();
}

void ctx_fill_block(cbie_ctx* c, const int64_t* rows, int64_t m, const int64_t* cols, int64_t n,
                    int scaled, zc* out_host) {
  for (int64_t i = 0; i < m; ++i)
    if (rows[i] < 0 || rows[i] >= c->N) throw cbie_error(CBIE_EINVALID, "row index out of range");
  for (int64_t j = 0; j < n; ++j)
    if (cols[j] < 0 || cols[j] >= c->N) throw cbie_error(CBIE_EINVALID, "col index out of range");
  if (m == 0 || n == 0) return;
  cudaStream_t s = c->stream;
  DBuf<int64_t> dr, dc;
  DBuf<zc> d;
  dr.upload(rows, m, s);
  dc.upload(cols, n, s);
  d.alloc(m * n);
  if (c->C == 2)
    k_fill_entries<2><<<ceil_div(m * n, 128), 128, 0, s>>>(c->tab, c->geom(), c->ph, c->near(),
                                                           dr.p, m, dc.p, n, scaled, d.p);
  else
    k_fill_entries<4><<<ceil_div(m * n, 128), 128, 0, s>>>(c->tab, c->geom(), c->ph, c->near(),
                                                           dr.p, m, dc.p, n, scaled, d.p);
  CKL();
  CK(cudaMemcpyAsync(out_host, d.p, sizeof(zc) * m * n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
}

void ctx_pair_block(cbie_ctx* c, int64_t point, int patch, zc* out_host) {
  const int C = c->C, np = c->np;
  std::vector<int64_t> rows(C), cols((size_t)np * C);
  for (int b = 0; b < C; ++b) rows[b] = point * C + b;
  for (int j = 0; j < np * C; ++j) cols[j] = ((int64_t)patch * np) * C + j;
  ctx_fill_block(c, rows.data(), C, cols.data(), (int64_t)np * C, 0, out_host);
}

// whole unscaled matrix, row-major, into device memory (the dense solve keeps it there)
void ctx_fill_dense_device(cbie_ctx* c, zc* d_out) {
  cudaStream_t s = c->stream;
  const int64_t work = (int64_t)c->npts * c->npts;
  if (c->C == 2)
    k_fill_dense<2><<<ceil_div(work, 128), 128, 0, s>>>(c->tab, c->geom(), c->ph, c->near(), 0, c->npts, d_out);
  else
    k_fill_dense<4><<<ceil_div(work, 128), 128, 0, s>>>(c->tab, c->geom(), c->ph, c->near(), 0, c->npts, d_out);
  CKL();
}

void ctx_fill_dense(cbie_ctx* c, zc* out_host) {
  cudaStream_t s = c->stream;
  const int64_t N = c->N;
  const int C = c->C;
  // row chunks of <= 1 GiB on device
  int64_t chunk_pts = std::max<int64_t>(1, ((int64_t)1 << 30) / (16 * N * C));
  chunk_pts = std::min<int64_t>(chunk_pts, c->npts);
  DBuf<zc> d;
  d.alloc((size_t)chunk_pts * C * N);
  EvTimer tm;
  tm.start(s);
  double kernel_ms = 0;
  for (int64_t p0 = 0; p0 < c->npts; p0 += chunk_pts) {
    int nrow = (int)std::min<int64_t>(chunk_pts, c->npts - p0);
    int64_t work = (int64_t)nrow * c->npts;
    if (C == 2)
      k_fill_dense<2><<<ceil_div(work, 128), 128, 0, s>>>(c->tab, c->geom(), c->ph, c->near(),
                                                          (int)p0, nrow, d.p);
    else
      k_fill_dense<4><<<ceil_div(work, 128), 128, 0, s>>>(c->tab, c->geom(), c->ph, c->near(),
                                                          (int)p0, nrow, d.p);
    CKL();
    CK(cudaMemcpyAsync(out_host + p0 * C * N, d.p, sizeof(zc) * nrow * C * N,
                       cudaMemcpyDeviceToHost, s));
  }
  kernel_ms = tm.stop_ms(s);
  c->stat["fill_dense_ms"] = kernel_ms;
}
