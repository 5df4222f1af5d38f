// Native host runtime of the level pipeline: the per-level bookkeeping the
// reference does in Python per box (tree queries, far-field DOF lists, proxy
// rings), done here for a whole quadtree level in one call.  Plain C ABI over
// host arrays (numpy buffers); no CUDA.  Compiled with -ffp-contract=off so
// every floating-point expression rounds like the reference's NumPy code.
//
// Tree arrays follow tree.py (paper_2001_11619_b200): boxes indexed globally
// level by level, keys (lev, ix, iy) sorted within a level, children in
// SW, SE, NW, NE order, neighbours (nbox x 8) in sorted key order.

#include <malloc.h>
#include <math.h>
#include <stdint.h>
#include <chrono>
#include <functional>
#include <thread>
#include <stdio.h>
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

// Host allocator tuning for the level pipeline: per-level descriptor arrays
// (host vectors, NumPy buffers) of 0.1-10 MB are allocated and freed at every
// level; keeping freed blocks in the heap avoids an mmap/munmap + page-fault
// cycle per allocation (the dominant host cost of a native tree build).
int skb_host_init(void) {
  static bool done = false;
  if (!done) {
    mallopt(M_MMAP_THRESHOLD, 256 << 20);
    mallopt(M_TRIM_THRESHOLD, 512 << 20);
    done = true;
  }
  return 0;
}

int skb_host_far_lists(int64_t nb, const int64_t* idx, const double* center, const double* hw,
                       const int64_t* nbr, const int64_t* lev, const int64_t* ix,
                       const int64_t* iy, const uint8_t* is_leaf, const int64_t* level_start,
                       int64_t depth, const double* root, double factor, const int64_t* big,
                       const int64_t* a_start, const int64_t* a_len, const double* px,
                       const double* py, int64_t* far_off, int64_t* far, int64_t cap,
                       int64_t* need, int32_t dof_shift) {
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
        const int64_t node = a[q] >> dof_shift;     // dof -> node (dpn 2: >> 1, dpn 1: id)
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

// Leaf active sets (skel.py:243-249): DOFs dpn * node + {0 .. dpn-1} of each
// leaf's owned nodes (ascending), appended to `big` level by level, leaves in
// index order; a_start / a_len per box (0 for internal boxes).  Returns the
// fill, or -1 when `big` (capacity cap) is too small.
int64_t skb_host_leaf_actives(int64_t nbox, int64_t depth, const int64_t* lev, const uint8_t* is_leaf,
                              const int64_t* node_start, const int64_t* node_cnt,
                              const int64_t* level_nodes, const int64_t* level_nodes_off,
                              const int64_t* level_start, int64_t dpn, int64_t* big, int64_t cap,
                              int64_t* a_start, int64_t* a_len) {
  int64_t fill = 0;
  for (int64_t i = 0; i < nbox; ++i) { a_start[i] = 0; a_len[i] = 0; }
  for (int64_t l = 0; l <= depth; ++l)
    for (int64_t i = level_start[l]; i < level_start[l + 1]; ++i) {
      if (!is_leaf[i]) continue;
      (void)lev;
      const int64_t* nd = level_nodes + level_nodes_off[l] + node_start[i];
      const int64_t n = node_cnt[i];
      if (fill + dpn * n > cap) return -1;
      a_start[i] = fill;
      a_len[i] = dpn * n;
      for (int64_t t = 0; t < n; ++t)
        for (int64_t e = 0; e < dpn; ++e) big[fill++] = dpn * nd[t] + e;
    }
  return fill;
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

// ---------------------------------------------------------------------------
// Quadtree build (reference build_tree, tree.py:110-155; same rules as the
// NumPy restatement tree.build_tree): split while a box holds more than
// leaf_cap nodes, east = x >= cx, north = y >= cy, empty children pruned,
// boxes of a level sorted by key, nodes of a child in their parent order.
// ---------------------------------------------------------------------------
struct NativeTree {
  int64_t n_nodes = 0, nbox = 0, depth = 0;
  std::vector<int64_t> level_start, lev, ix, iy, parent, children, nchild, node_start, node_cnt;
  std::vector<int64_t> level_nodes, level_nodes_off, nbr, node_leaf;
  std::vector<double> center, hw;
};

int skb_tree_build(const double* pos, int64_t N, int64_t leaf_cap, int64_t max_depth,
                   const double* root, int64_t* handle) {
  NativeTree* T = new NativeTree();
  T->n_nodes = N;
  const bool tt_on = getenv("SKB_TREE_TIMING") != nullptr;
  auto tt0 = std::chrono::steady_clock::now();
  auto tt = [&](const char* nm) {
    if (!tt_on) return;
    auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, " %s %.0f", nm, std::chrono::duration<double, std::micro>(t1 - tt0).count());
    tt0 = t1;
  };
  // Level-by-level split.  The node lists of all levels are written straight
  // into the flat level_nodes array (level l at level_nodes_off[l]); a level's
  // nodes are the nodes of the split boxes of the level above, so only those
  // are visited.  Working indices are 32-bit (N < 2^31).
  struct Lv { std::vector<int64_t> ix, iy, par, cnt; std::vector<double> cx, cy, half; int64_t noff; };
  std::vector<Lv> levels;
  levels.reserve(64);
  std::vector<std::vector<int64_t>> L_children;   // per level, nb x 4 (local child idx, by quadrant)
  T->level_nodes.reserve((size_t)N * 14);     // ~ nodes x levels (grows if a tree is deeper)
  T->level_nodes.resize((size_t)N);
  for (int64_t i = 0; i < N; ++i) T->level_nodes[i] = i;
  T->level_nodes_off.assign(1, 0);
  {
    Lv L0;
    L0.ix = {0}; L0.iy = {0}; L0.par = {-1}; L0.cnt = {N};
    L0.cx = {root[0]}; L0.cy = {root[1]}; L0.half = {root[2]};
    L0.noff = 0;
    levels.push_back(std::move(L0));
  }
  std::vector<uint8_t> quad((size_t)N);
  double ph[4] = {0, 0, 0, 0};
  auto pnow = [] { return std::chrono::steady_clock::now(); };
  auto pus = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
  std::vector<int64_t> start, qcnt, slot, fillp;
  struct Kid { int64_t code, b, q; };
  std::vector<Kid> kids;
  int64_t l = 0;
  while (true) {
    const Lv& cur = levels.back();
    const int64_t nb = (int64_t)cur.ix.size();
    const auto& ix = cur.ix; const auto& iy = cur.iy; const auto& cnt = cur.cnt;
    const auto& cx = cur.cx; const auto& cy = cur.cy; const auto& half = cur.half;
    const int64_t* nodes = T->level_nodes.data() + cur.noff;
    int64_t nn = 0;
    for (int64_t b = 0; b < nb; ++b) nn += cnt[b];
    T->level_nodes_off.push_back(cur.noff + nn);
    std::vector<int64_t> ch(4 * nb, -1);
    bool any = false;
    for (int64_t b = 0; b < nb; ++b) any |= (cnt[b] > leaf_cap) && (l < max_depth);
    if (!any) { L_children.push_back(std::move(ch)); break; }
    // children of all split boxes, keyed by code = cix * side + ciy; nodes of
    // a child keep their order in the parent (counting sort per quadrant)
    const int64_t side = (int64_t)1 << (l + 1);
    start.assign(nb + 1, 0);
    for (int64_t b = 0; b < nb; ++b) start[b + 1] = start[b] + cnt[b];
    qcnt.assign(4 * nb, 0);
    int64_t nnext = 0;
    auto p0 = pnow();
    for (int64_t b = 0; b < nb; ++b) {
      if (!((cnt[b] > leaf_cap) && (l < max_depth))) continue;
      const double bx = cx[b], by = cy[b];
      // counters in registers (a per-quadrant array increment would serialise
      // the loop on store-to-load forwarding)
      int64_t ne = 0, nn_ = 0, nne = 0;
      for (int64_t t = start[b]; t < start[b + 1]; ++t) {
        const double* pp = pos + 2 * nodes[t];
        const int dx = pp[0] >= bx ? 1 : 0, dy = pp[1] >= by ? 1 : 0;
        quad[t] = (uint8_t)(dx + 2 * dy);
        ne += dx; nn_ += dy; nne += dx & dy;
      }
      qcnt[4 * b + 3] = nne;
      qcnt[4 * b + 1] = ne - nne;
      qcnt[4 * b + 2] = nn_ - nne;
      qcnt[4 * b + 0] = cnt[b] - ne - nn_ + nne;
    }
    for (int64_t b = 0; b < nb; ++b)
      if ((cnt[b] > leaf_cap) && (l < max_depth)) nnext += cnt[b];
    auto p1 = pnow();
    kids.clear();
    for (int64_t b = 0; b < nb; ++b)
      for (int64_t q = 0; q < 4; ++q)
        if (qcnt[4 * b + q] > 0)
          kids.push_back(Kid{(2 * ix[b] + (q & 1)) * side + (2 * iy[b] + (q >> 1)), b, q});
    std::sort(kids.begin(), kids.end(), [](const Kid& a, const Kid& b) { return a.code < b.code; });
    const size_t nk = kids.size();
    Lv nx;
    nx.ix.resize(nk); nx.iy.resize(nk); nx.par.resize(nk); nx.cnt.resize(nk);
    nx.cx.resize(nk); nx.cy.resize(nk); nx.half.resize(nk);
    nx.noff = cur.noff + nn;
    slot.assign(4 * nb, -1);
    fillp.assign(nk + 1, 0);
    for (size_t c = 0; c < nk; ++c) {
      const int64_t b = kids[c].b, q = kids[c].q, dx = q & 1, dy = q >> 1;
      ch[4 * b + q] = (int64_t)c;
      slot[4 * b + q] = (int64_t)c;
      nx.ix[c] = 2 * ix[b] + dx;
      nx.iy[c] = 2 * iy[b] + dy;
      nx.par[c] = b;
      nx.cnt[c] = qcnt[4 * b + q];
      fillp[c + 1] = fillp[c] + nx.cnt[c];
      nx.cx[c] = cx[b] + ((double)dx - 0.5) * half[b];
      nx.cy[c] = cy[b] + ((double)dy - 0.5) * half[b];
      nx.half[c] = half[b] / 2;
    }
    auto p2 = pnow();
    const size_t base = (size_t)nx.noff;
    T->level_nodes.resize(base + (size_t)nnext);
    auto p3 = pnow();
    nodes = T->level_nodes.data() + cur.noff;          // (resize may have moved the array)
    int64_t* out = T->level_nodes.data() + base;
    for (int64_t b = 0; b < nb; ++b) {
      if (!((cnt[b] > leaf_cap) && (l < max_depth))) continue;
      int64_t f[4];
      for (int q = 0; q < 4; ++q) f[q] = slot[4 * b + q] >= 0 ? fillp[slot[4 * b + q]] : 0;
      int64_t f0 = f[0], f1 = f[1], f2 = f[2], f3 = f[3];     // write cursors in registers
      for (int64_t t = start[b]; t < start[b + 1]; ++t) {
        const int q = quad[t];
        const int64_t at = q == 0 ? f0 : (q == 1 ? f1 : (q == 2 ? f2 : f3));
        out[at] = nodes[t];
        f0 += q == 0; f1 += q == 1; f2 += q == 2; f3 += q == 3;
      }
    }
    auto p4 = pnow();
    ph[0] += pus(p0, p1); ph[1] += pus(p1, p2); ph[2] += pus(p2, p3); ph[3] += pus(p3, p4);
    L_children.push_back(std::move(ch));
    levels.push_back(std::move(nx));
    ++l;
  }
  if (tt_on) fprintf(stderr, " [quad %.0f kids %.0f resize %.0f scatter %.0f]", ph[0], ph[1], ph[2], ph[3]);
  tt("levels");
  T->depth = l;
  const int64_t nlev = l + 1;
  T->level_start.assign(nlev + 1, 0);
  for (int64_t q = 0; q < nlev; ++q) T->level_start[q + 1] = T->level_start[q] + (int64_t)levels[q].ix.size();
  const int64_t nbox = T->level_start[nlev];
  T->nbox = nbox;
  T->lev.resize(nbox); T->ix.resize(nbox); T->iy.resize(nbox); T->parent.resize(nbox);
  T->center.resize(2 * nbox); T->hw.resize(nbox); T->children.assign(4 * nbox, -1);
  T->nchild.assign(nbox, 0); T->node_start.resize(nbox); T->node_cnt.resize(nbox);
  for (int64_t q = 0; q < nlev; ++q) {
    const Lv& L = levels[q];
    const int64_t base = T->level_start[q];
    int64_t st = 0;
    for (size_t b = 0; b < L.ix.size(); ++b) {
      const int64_t g = base + (int64_t)b;
      T->lev[g] = q; T->ix[g] = L.ix[b]; T->iy[g] = L.iy[b];
      T->parent[g] = L.par[b] >= 0 ? L.par[b] + T->level_start[q > 0 ? q - 1 : 0] : -1;
      T->center[2 * g] = L.cx[b]; T->center[2 * g + 1] = L.cy[b]; T->hw[g] = L.half[b];
      T->node_start[g] = st; T->node_cnt[g] = L.cnt[b]; st += L.cnt[b];
      int nc = 0;
      for (int qd = 0; qd < 4; ++qd) {
        const int64_t c = L_children[q][4 * b + qd];
        if (c >= 0) T->children[4 * g + nc++] = c + T->level_start[q + 1];
      }
      T->nchild[g] = nc;
    }
  }
  tt("flatten");
  // same-level neighbours in sorted key order (tree.py:70-81): a box's three
  // neighbours in cell column ix + dx are consecutive keys, found by one
  // binary search per column restricted to the level
  T->nbr.assign(8 * nbox, -1);
  for (int64_t q = 0; q < nlev; ++q) {
    const int64_t lo0 = T->level_start[q], hi0 = T->level_start[q + 1], side = (int64_t)1 << q;
    const int64_t* ixp = T->ix.data();
    const int64_t* iyp = T->iy.data();
    for (int64_t g = lo0; g < hi0; ++g) {
      for (int dx = -1; dx <= 1; ++dx) {
        const int64_t nxc = ixp[g] + dx;
        if (nxc < 0 || nxc >= side) continue;
        const int64_t ylo = iyp[g] - 1;
        // first box of the level with key >= nxc * side + max(ylo, 0)
        const int64_t want = nxc * side + (ylo < 0 ? 0 : ylo);
        int64_t lo = lo0, hi = hi0;
        if (dx == 0) { lo = g > lo0 ? g - 1 : g; hi = g + 2 < hi0 ? g + 2 : hi0; }   // own column: adjacent keys
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (ixp[mid] * side + iyp[mid] < want) lo = mid + 1;
          else hi = mid;
        }
        for (int64_t j = lo; j < hi0 && ixp[j] == nxc && iyp[j] <= iyp[g] + 1; ++j) {
          const int dy = (int)(iyp[j] - iyp[g]);
          if (dx == 0 && dy == 0) continue;
          // slot order of the reference loop: dx outer, dy inner, (0, 0) skipped
          int sl = (dx + 1) * 3 + (dy + 1);
          if (sl > 4) --sl;
          T->nbr[8 * g + sl] = j;
        }
      }
    }
  }
  tt("nbr");
  T->node_leaf.assign(N, -1);
  for (int64_t g = 0; g < nbox; ++g)
    if (T->nchild[g] == 0) {
      const int64_t* nd = T->level_nodes.data() + T->level_nodes_off[T->lev[g]] + T->node_start[g];
      for (int64_t t = 0; t < T->node_cnt[g]; ++t) T->node_leaf[nd[t]] = g;
    }
  tt("node_leaf");
  if (tt_on) fprintf(stderr, " us\n");
  *handle = (int64_t)T;
  return 0;
}

// sizes: {nbox, depth, total level-node entries}
int skb_tree_sizes(int64_t handle, int64_t* sizes) {
  const NativeTree* T = (const NativeTree*)handle;
  sizes[0] = T->nbox; sizes[1] = T->depth; sizes[2] = (int64_t)T->level_nodes.size();
  return 0;
}

int skb_tree_export(int64_t handle, int64_t* level_start, int64_t* lev, int64_t* ix, int64_t* iy,
                    int64_t* parent, double* center, double* hw, int64_t* children,
                    int64_t* nchild, int64_t* node_start, int64_t* node_cnt, int64_t* level_nodes,
                    int64_t* level_nodes_off, int64_t* nbr, int64_t* node_leaf) {
  const NativeTree* T = (const NativeTree*)handle;
  auto cp = [](int64_t* d, const std::vector<int64_t>& v) { memcpy(d, v.data(), v.size() * 8); };
  cp(level_start, T->level_start); cp(lev, T->lev); cp(ix, T->ix); cp(iy, T->iy);
  cp(parent, T->parent); cp(children, T->children); cp(nchild, T->nchild);
  cp(node_start, T->node_start); cp(node_cnt, T->node_cnt); cp(level_nodes, T->level_nodes);
  cp(level_nodes_off, T->level_nodes_off); cp(nbr, T->nbr); cp(node_leaf, T->node_leaf);
  memcpy(center, T->center.data(), T->center.size() * 8);
  memcpy(hw, T->hw.data(), T->hw.size() * 8);
  return 0;
}

int skb_tree_free(int64_t handle) {
  delete (NativeTree*)handle;
  return 0;
}

// ---------------------------------------------------------------------------
// Dirty set of an update (reference skel.py:476-491, 517-534; tree.py:215-270;
// same rules as tree.dirty_set): ownership changes, proxy discs holding an
// old/new moved position, ancestors of the moved nodes' new leaves, closed
// under parents + colleagues.  Trees as flat arrays (tree.py layout);
// out_mask: new-tree boxes (uint8).
// ---------------------------------------------------------------------------
struct FlatTree {
  const int64_t *level_start, *lev, *ix, *iy, *parent, *node_start, *node_cnt, *level_nodes,
      *level_nodes_off, *nbr, *node_leaf;
  const double* center;
  int64_t depth;
  double root_cx, root_cy, root_hw;
};

static int64_t flat_find(const FlatTree& t, int64_t lp, int64_t code) {
  if (lp > t.depth) return -1;
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

static FlatTree flat(const int64_t* const* a, const double* center, int64_t depth, const double* root) {
  return FlatTree{a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], a[9], a[10],
                  center, depth, root[0], root[1], root[2]};
}

// arrays: {level_start, lev, ix, iy, parent, node_start, node_cnt, level_nodes,
//          level_nodes_off, nbr, node_leaf}
int skb_dirty_set(const int64_t* const* new_arrays, const double* new_center, int64_t new_depth,
                  const int64_t* const* old_arrays, int64_t old_depth, const double* root,
                  const int64_t* old_to_new, const double* pts, int64_t npts,
                  const int64_t* mod_new, int64_t nmod, double proxy_factor, uint8_t* out_mask) {
  const FlatTree tn = flat(new_arrays, new_center, new_depth, root);
  const FlatTree to = flat(old_arrays, nullptr, old_depth, root);
  const int64_t nbn = tn.level_start[new_depth + 1];
  std::vector<uint8_t> content(nbn, 0);
  // ownership changes (tree.py:251-270)
  for (int64_t l = 0; l <= std::max(new_depth, old_depth); ++l) {
    const int64_t side = (int64_t)1 << l;
    if (l <= new_depth)
      for (int64_t g = tn.level_start[l]; g < tn.level_start[l + 1]; ++g) {
        const int64_t o = flat_find(to, l, tn.ix[g] * side + tn.iy[g]);
        if (o < 0 || tn.node_cnt[g] != to.node_cnt[o]) { content[g] = 1; continue; }
        const int64_t* nn = tn.level_nodes + tn.level_nodes_off[l] + tn.node_start[g];
        const int64_t* oo = to.level_nodes + to.level_nodes_off[l] + to.node_start[o];
        for (int64_t t = 0; t < tn.node_cnt[g]; ++t)
          if (nn[t] != old_to_new[oo[t]]) { content[g] = 1; break; }
      }
    if (l <= old_depth)
      for (int64_t o = to.level_start[l]; o < to.level_start[l + 1]; ++o) {
        if (flat_find(tn, l, to.ix[o] * side + to.iy[o]) >= 0) continue;
        int64_t p = o;                 // vanished: nearest surviving ancestor changed
        while (p >= 0) {
          const int64_t lp = to.lev[p], sp = (int64_t)1 << lp;
          const int64_t g = flat_find(tn, lp, to.ix[p] * sp + to.iy[p]);
          if (g >= 0) { content[g] = 1; break; }
          p = to.parent[p];
        }
      }
  }
  // proxy discs holding a moved position (tree.py:215-236)
  if (npts > 0) {
    const double ox = tn.root_cx - tn.root_hw, oy = tn.root_cy - tn.root_hw;
    std::vector<int64_t> cand;
    for (int64_t l = 0; l <= new_depth; ++l) {
      if (tn.level_start[l + 1] == tn.level_start[l]) continue;
      const double hw = tn.root_hw / (double)((int64_t)1 << l);
      const double rad = proxy_factor * hw * sqrt(2.0);
      const double step = 2 * hw;
      const int64_t reach = (int64_t)ceil(rad / step) + 1, side = (int64_t)1 << l;
      std::vector<int64_t> cells(npts);
      const int64_t W = side + 2 * reach + 2;
      for (int64_t i = 0; i < npts; ++i)
        cells[i] = (int64_t)floor((pts[2 * i] - ox) / step) * W + (int64_t)floor((pts[2 * i + 1] - oy) / step);
      std::sort(cells.begin(), cells.end());
      cells.erase(std::unique(cells.begin(), cells.end()), cells.end());
      cand.clear();
      for (int64_t uc : cells) {
        // floor division matching numpy's // for negative codes
        int64_t cxl = uc / W, cyl = uc - cxl * W;
        if (cyl < 0) { cxl -= 1; cyl += W; }
        for (int64_t dx = -reach; dx <= reach; ++dx)
          for (int64_t dy = -reach; dy <= reach; ++dy) {
            const int64_t nx = cxl + dx, ny = cyl + dy;
            if (nx < 0 || ny < 0 || nx >= side || ny >= side) continue;
            const int64_t g = flat_find(tn, l, nx * side + ny);
            if (g >= 0) cand.push_back(g);
          }
      }
      std::sort(cand.begin(), cand.end());
      cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
      const double r2 = rad * rad;
      for (int64_t g : cand) {
        if (content[g]) continue;
        const double bx = tn.center[2 * g], by = tn.center[2 * g + 1];
        for (int64_t i = 0; i < npts; ++i) {
          const double dx = pts[2 * i] - bx, dy = pts[2 * i + 1] - by;
          if (dx * dx + dy * dy <= r2) { content[g] = 1; break; }
        }
      }
    }
  }
  // ancestors of the moved nodes' new leaves (skel.py:486-490)
  for (int64_t t = 0; t < nmod; ++t) {
    int64_t i = tn.node_leaf[mod_new[t]];
    while (i >= 0 && !content[i]) { content[i] = 1; i = tn.parent[i]; }
  }
  // closure under parents + colleagues, bottom-up (skel.py:517-534)
  std::vector<uint8_t> marked(content);
  for (int64_t l = new_depth; l >= 0; --l) {
    std::vector<int64_t> grew;
    for (int64_t g = tn.level_start[l]; g < tn.level_start[l + 1]; ++g)
      if (marked[g]) grew.push_back(g);
    if (l + 1 <= new_depth)
      for (int64_t g = tn.level_start[l + 1]; g < tn.level_start[l + 2]; ++g)
        if (marked[g] && tn.parent[g] >= 0 && !marked[tn.parent[g]]) {
          marked[tn.parent[g]] = 1;
          grew.push_back(tn.parent[g]);
        }
    for (int64_t g : grew)
      for (int s = 0; s < 8; ++s)
        if (tn.nbr[8 * g + s] >= 0) marked[tn.nbr[8 * g + s]] = 1;
  }
  memcpy(out_mask, marked.data(), nbn);
  return 0;
}

}  // extern "C"
