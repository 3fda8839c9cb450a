// tree.cpp — cluster tree and block tree on the host (native C++).
//
// Restates ClusterTree._split (hmatrix.py:62-75): median bisection on the
// longest bounding-box axis with a STABLE sort, leaf if points*C <= n_leaf or
// fewer than 2 points; admissible (hmatrix.py:87-89); HMatrix._descend
// (hmatrix.py:194-204): admissible -> low rank, leaf x leaf -> dense, else
// subdivide over the children grid.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "hmatrix.h"

void Tree::build_clusters(const double* pts, int npts, int C_, int n_leaf) {
  C = C_;
  cl.clear();
  pperm.resize(npts);
  std::iota(pperm.begin(), pperm.end(), 0);
  std::vector<int32_t> tmp(npts);
  // explicit stack: (lo, hi, level, parent slot)
  struct Job { int lo, hi, level, parent, which; };
  std::vector<Job> stack{{0, npts, 0, -1, 0}};
  // depth-first, children in order (ids are creation order; only structure matters)
  while (!stack.empty()) {
    Job j = stack.back();
    stack.pop_back();
    Cluster c;
    c.lo = j.lo;
    c.hi = j.hi;
    c.level = j.level;
    for (int i = 0; i < 3; ++i) {
      c.blo[i] = 1e300;
      c.bhi[i] = -1e300;
    }
    for (int a = j.lo; a < j.hi; ++a)
      for (int i = 0; i < 3; ++i) {
        double v = pts[3 * (size_t)pperm[a] + i];
        c.blo[i] = std::min(c.blo[i], v);
        c.bhi[i] = std::max(c.bhi[i], v);
      }
    int id = (int)cl.size();
    cl.push_back(c);
    if (j.parent >= 0) {
      cl[j.parent].kid[j.which] = id;
    }
    if ((j.hi - j.lo) * C <= n_leaf || j.hi - j.lo < 2) continue;
    int ax = 0;
    double ext[3];
    for (int i = 0; i < 3; ++i) ext[i] = c.bhi[i] - c.blo[i];
    for (int i = 1; i < 3; ++i)
      if (ext[i] > ext[ax]) ax = i;   // np.argmax: first maximum
    std::stable_sort(pperm.begin() + j.lo, pperm.begin() + j.hi, [&](int32_t a, int32_t b) {
      return pts[3 * (size_t)a + ax] < pts[3 * (size_t)b + ax];
    });
    int mid = j.lo + (j.hi - j.lo) / 2;
    cl[id].nkid = 2;
    // push right first so the left child is processed (and numbered) first
    stack.push_back({mid, j.hi, j.level + 1, id, 1});
    stack.push_back({j.lo, mid, j.level + 1, id, 0});
  }
  root_cl = 0;
}

static double box_diam(const Cluster& a) {
  double s = 0;
  for (int i = 0; i < 3; ++i) s += (a.bhi[i] - a.blo[i]) * (a.bhi[i] - a.blo[i]);
  return std::sqrt(s);
}
static double box_dist(const Cluster& a, const Cluster& b) {
  double s = 0;
  for (int i = 0; i < 3; ++i) {
    double g = std::max(0.0, std::max(a.blo[i] - b.bhi[i], b.blo[i] - a.bhi[i]));
    s += g * g;
  }
  return std::sqrt(s);
}

void Tree::build_blocks(double eta) {
  nodes.clear();
  leaves.clear();
  struct Job { int r, c, parent, slot; };
  std::vector<Job> stack{{root_cl, root_cl, -1, 0}};
  std::vector<int> order;   // leaves in depth-first (row-major children) order
  while (!stack.empty()) {
    Job j = stack.back();
    stack.pop_back();
    BNode b;
    b.r = j.r;
    b.c = j.c;
    const Cluster &R = cl[j.r], &Cc = cl[j.c];
    double d = box_dist(R, Cc);
    bool adm = d > 0 && std::min(box_diam(R), box_diam(Cc)) <= eta * d;
    int id = (int)nodes.size();
    if (adm) {
      b.kind = BLK_LR;
    } else if (R.nkid == 0 && Cc.nkid == 0) {
      b.kind = BLK_DENSE;
    } else {
      b.kind = BLK_H;
      b.nr = R.nkid ? 2 : 1;
      b.nc = Cc.nkid ? 2 : 1;
    }
    nodes.push_back(b);
    if (j.parent >= 0) nodes[j.parent].kid[j.slot] = id;
    if (b.kind == BLK_H) {
      // push in reverse so children are visited row-major (a, b)
      for (int a = b.nr - 1; a >= 0; --a)
        for (int bb = b.nc - 1; bb >= 0; --bb) {
          int rk = R.nkid ? R.kid[a] : j.r;
          int ck = Cc.nkid ? Cc.kid[bb] : j.c;
          stack.push_back({rk, ck, id, a * b.nc + bb});
        }
    } else {
      LeafInfo L;
      L.node = id;
      L.r = j.r;
      L.c = j.c;
      L.m = dofs(j.r);
      L.n = dofs(j.c);
      L.kind = b.kind;
      nodes[id].leaf = (int)leaves.size();
      leaves.push_back(L);
    }
  }
  root_node = 0;
}
