// Native host runtime of the level pipeline: the per-level bookkeeping the
// reference does in Python per box (tree queries, far-field DOF lists, proxy
// rings), done here for a whole quadtree level in one call.  Plain C ABI over
// host arrays (numpy buffers); no CUDA.  Compiled with -ffp-contract=off so
// every floating-point expression rounds like the reference's NumPy code.
//
// Tree arrays follow tree.py (paper_2001_11619_b200): boxes indexed globally
// level by level, keys (lev, ix, iy) sorted within a level, children in
// SW, SE, NW, NE order, neighbours (nbox x 8) in sorted key order.

#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "../../include/skelb200.h"

namespace {

struct TreeView {
  const double* center;     // nbox x 2
  const double* hw;         // nbox
  const int64_t* nbr;       // nbox x 8
  const int64_t* lev;
  const int64_t* ix;
  const int64_t* iy;
  const uint8_t* is_leaf;
  const int64_t* level_start;  // depth + 2
  int64_t depth;
  double root_cx, root_cy, root_hw;
};

inline int64_t find_code(const TreeView& t, int64_t lp, int64_t code) {
  // boxes of level lp are sorted by code ix * 2^lp + iy
  int64_t lo = t.level_start[lp], hi = t.level_start[lp + 1];
  const int64_t side = (int64_t)1 << lp;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int64_t c = t.ix[mid] * side + t.iy[mid];
    if (c < code) lo = mid + 1;
    else hi = mid;
  }
  if (lo < t.level_start[lp + 1] && t.ix[lo] * side + t.iy[lo] == code) return lo;
  return -1;
}

// Coarser leaves meeting the disc (c, r) of a level-L box, sorted by index
// (reference Tree.shallow_leaves_near, tree.py:83-99; same cell walk and
// box-disc test as Tree.coarse_leaves in tree.py).
void coarse_leaves(const TreeView& t, int64_t L, double cx, double cy, double r,
                   std::vector<int64_t>& out) {
  const double ox = t.root_cx - t.root_hw, oy = t.root_cy - t.root_hw;
  const int64_t side = (int64_t)1 << L;
  const double cell = 2.0 * t.root_hw / (double)side;
  auto clip = [&](int64_t v) { return v < 0 ? 0 : (v > side - 1 ? side - 1 : v); };
  const int64_t lox = clip((int64_t)floor(((cx - r) - ox) / cell));
  const int64_t loy = clip((int64_t)floor(((cy - r) - oy) / cell));
  const int64_t hix = clip((int64_t)floor(((cx + r) - ox) / cell));
  const int64_t hiy = clip((int64_t)floor(((cy + r) - oy) / cell));
  const double r2 = r * r;
  for (int64_t lp = 0; lp < L; ++lp) {
    if (t.level_start[lp + 1] == t.level_start[lp]) continue;
    const int64_t sh = L - lp, sl = (int64_t)1 << lp;
    for (int64_t x = lox >> sh; x <= (hix >> sh); ++x)
      for (int64_t y = loy >> sh; y <= (hiy >> sh); ++y) {
        const int64_t j = find_code(t, lp, x * sl + y);
        if (j < 0 || !t.is_leaf[j]) continue;
        double dx = fabs(cx - t.center[2 * j]) - t.hw[j];
        double dy = fabs(cy - t.center[2 * j + 1]) - t.hw[j];
        dx = dx > 0.0 ? dx : 0.0;
        dy = dy > 0.0 ? dy : 0.0;
        if (!(dx * dx + dy * dy > r2)) out.push_back(j);
      }
  }
}

}  // namespace

extern "C" {

int skb_host_far_lists(int64_t nb, const int64_t* idx, const double* center, const double* hw,
                       const int64_t* nbr, const int64_t* lev, const int64_t* ix,
                       const int64_t* iy, const uint8_t* is_leaf, const int64_t* level_start,
                       int64_t depth, const double* root, double factor, const int64_t* big,
                       const int64_t* a_start, const int64_t* a_len, const double* px,
                       const double* py, int64_t* far_off, int64_t* far, int64_t cap,
                       int64_t* need) {
  TreeView t{center, hw, nbr, lev, ix, iy, is_leaf, level_start, depth, root[0], root[1], root[2]};
  const double s2 = sqrt(2.0);
  std::vector<int64_t> src;
  int64_t o = 0;
  far_off[0] = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t i = idx[b];
    const double rp = factor * hw[i] * s2;          // proxy_radius, tree.py:158-160
    const double cx = center[2 * i], cy = center[2 * i + 1];
    src.clear();
    for (int s = 0; s < 8; ++s)                     // colleagues, sorted keys
      if (nbr[8 * i + s] >= 0) src.push_back(nbr[8 * i + s]);
    coarse_leaves(t, lev[i], cx, cy, rp, src);     // then coarser leaves, sorted keys
    const double r2 = rp * rp;
    for (int64_t j : src) {
      const int64_t* a = big + a_start[j];
      for (int64_t q = 0; q < a_len[j]; ++q) {
        const int64_t node = a[q] >> 1;
        const double dx = px[node] - cx, dy = py[node] - cy;
        if (dx * dx + dy * dy < r2) {               // skel.py:279 strict distance filter
          if (o < cap) far[o] = a[q];
          ++o;
        }
      }
    }
    far_off[b + 1] = o;
  }
  *need = o;
  return o <= cap ? 0 : 1;
}

// Proxy rings with radial normals about the ring centroid and weights
// (kernels.py:263-273, 340-342); pts/pn: nb x P x 2, pw: nb.
int skb_host_proxies(int64_t nb, const int64_t* idx, const double* center, const double* hw,
                     double factor, int64_t P, const double* cs, double* pts, double* pn,
                     double* pw) {
  const double s2 = sqrt(2.0);
  const double two_pi = 2.0 * M_PI;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t i = idx[b];
    const double rp = factor * hw[i] * s2;
    const double cx = center[2 * i], cy = center[2 * i + 1];
    double* p = pts + 2 * P * b;
    double sx = 0.0, sy = 0.0;
    for (int64_t j = 0; j < P; ++j) {
      p[2 * j] = cx + rp * cs[2 * j];
      p[2 * j + 1] = cy + rp * cs[2 * j + 1];
      if (j == 0) { sx = p[0]; sy = p[1]; }
      else { sx = sx + p[2 * j]; sy = sy + p[2 * j + 1]; }
    }
    const double mx = sx / (double)P, my = sy / (double)P;
    double* n = pn + 2 * P * b;
    for (int64_t j = 0; j < P; ++j) {
      const double ux = p[2 * j] - mx, uy = p[2 * j + 1] - my;
      const double nn = sqrt(ux * ux + uy * uy);
      n[2 * j] = ux / nn;
      n[2 * j + 1] = uy / nn;
    }
    pw[b] = two_pi * rp / (double)P;
  }
  return 0;
}

}  // extern "C"
