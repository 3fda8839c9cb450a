// context.h — host-side state of a cbie_ctx (one CUDA device).
#pragma once
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

struct cbie_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;

  // geometry -----------------------------------------------------------------
  bool has_geom = false;
  Tables tab{};
  int npatch = 0, nu = 0, nv = 0, np = 0, npts = 0;
  std::vector<int> h_kind;
  std::vector<double> h_cpar, h_samples, h_bbox, h_diam, h_pos, h_star;
  DBuf<int> d_kind;
  DBuf<double> d_cpar, d_coef, d_star, d_pos, d_au, d_av, d_sg, d_wg, d_bbox, d_diam;
  DBuf<int> d_flag;               // device error flags (degenerate patch, ...)

  // formulation -----------------------------------------------------------------
  bool has_form = false;
  Phys ph{};
  int grading = 3, oversample = 16;
  int C = 2;
  int64_t N = 0;

  // classification / near table ---------------------------------------------------
  bool has_class = false;
  int64_t n_near = 0, n_self = 0, n_fallback = 0, n_cand = 0;
  DBuf<int32_t> d_nearidx;        // [npts][npatch]
  DBuf<int32_t> d_near_pt, d_near_q;
  DBuf<double> d_near_u, d_near_v;
  DBuf<int8_t> d_near_tag, d_near_ok;
  DBuf<zc> d_near_blk;            // [n_near][C][np*C]

  // stats -------------------------------------------------------------------------
  std::map<std::string, double> stat;

  Geom geom() const {
    Geom g;
    g.kind = d_kind.p;
    g.cpar = d_cpar.p;
    g.coef = d_coef.p;
    g.star = d_star.p;
    g.pos = d_pos.p;
    g.au = d_au.p;
    g.av = d_av.p;
    g.sg = d_sg.p;
    g.wg = d_wg.p;
    g.bbox = d_bbox.p;
    g.diam = d_diam.p;
    return g;
  }
  NearTab near() const { return NearTab{d_nearidx.p, d_near_blk.p}; }
  void require(bool cond, const char* what) const {
    if (!cond) throw cbie_error(CBIE_ESTATE, what);
  }
};

// implemented in the .cu files
void ctx_set_geometry(cbie_ctx* c, int npatch, int nu, int nv, const double* samples,
                      const int* kind, const double* cpar, const double* star,
                      const double* cheb_coef);
void ctx_set_formulation(cbie_ctx* c, int kind, double omega, zc k1, zc k2, zc eps1, zc mu1,
                         zc eps2, zc mu2, double tau, int grading, int oversample,
                         const zc* rsc, const zc* csc);
void ctx_classify(cbie_ctx* c);
void ctx_near_fill(cbie_ctx* c);
void ctx_fill_block(cbie_ctx* c, const int64_t* rows, int64_t m, const int64_t* cols, int64_t n,
                    int scaled, zc* out_host);
void ctx_fill_dense(cbie_ctx* c, zc* out_host);
void ctx_fill_dense_device(cbie_ctx* c, zc* d_out);
void ctx_pair_block(cbie_ctx* c, int64_t point, int patch, zc* out_host);

// entry generation for a list of H-matrix dense leaves / arbitrary tiles (fill.cu)
struct TileDesc {                 // one dense tile of the permuted system
  int64_t out_off;                // offset (in zc) of the column-major tile in the output arena
  int32_t r_lo, r_hi, c_lo, c_hi; // point ranges in permuted order
};
void launch_fill_tiles(const cbie_ctx* c, const TileDesc* d_tiles, int ntiles, const int32_t* d_pperm,
                       zc* d_arena, int scaled, cudaStream_t s);
