// Host-side mesh preparation (C++17): 2:1 balance, canonical numbering,
// hanging-node constraints, Dirichlet DOFs, consistent loads and filter
// neighbour lists.  See include/tomesh_host.h for the contract and the paper
// passages (PAPER.md:564-571, :640-663 Eq. 6, :600-609 Eq. 4).
//
// Algorithms (independent of the oracle's):
//   balance   worklist ripple on a hash set of leaves; point location by
//             walking ancestors from the finest level;
//   numbering LSD radix sort of (Morton key, slot) pairs;
//   hanging   node-centric: locate the leaves around every node and test
//             whether the node is a corner of each of them;
//   filter    uniform binning of element centres (OpenMP).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <unordered_map>
#include <unordered_set>
#include <vector>
#include <deque>
#include <array>
#include <atomic>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../../include/tomesh.h"
#include "../../include/tomesh_host.h"
#include "common.h"

using namespace tomesh;

struct tomesh_host {
  int dim = 0, L = 0;
  double h0 = 1.0;
  int32_t ext[3] = {1, 1, 1};
  std::vector<int32_t> elem_node, elem_anchor, node_coord;
  std::vector<int8_t> elem_level;
  std::vector<uint64_t> node_key;       // sorted Morton keys of nodes
  std::vector<int32_t> hang_node, hang_ptr, hang_parent;
  std::vector<double> hang_weight, load;
  std::vector<int64_t> fixed_dof, filt_ptr;
  std::vector<int32_t> filt_idx;
  bool has_filter = false;
};

namespace {

struct LeafKey {
  // level in bits 58..62, coords 19 bits each
  static uint64_t make(int l, const int32_t *a, int dim) {
    uint64_t k = (uint64_t)l << 58;
    for (int c = 0; c < dim; ++c) k |= (uint64_t)(uint32_t)a[c] << (19 * c);
    return k;
  }
  static int level(uint64_t k) { return (int)(k >> 58); }
  static void anchor(uint64_t k, int dim, int32_t *a) {
    for (int c = 0; c < dim; ++c) a[c] = (int32_t)((k >> (19 * c)) & 0x7ffff);
  }
};

struct Splitmix {
  size_t operator()(uint64_t x) const {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return (size_t)(x ^ (x >> 31));
  }
};
using LeafSet = std::unordered_set<uint64_t, Splitmix>;

// Leaf containing the finest cell with anchor q (q inside the domain).
static bool locate(const LeafSet &S, int dim, int L, const int32_t *q, int *lev, int32_t *anc) {
  for (int l = L; l >= 0; --l) {
    int32_t s = 1 << (L - l);
    int32_t a[3] = {0, 0, 0};
    for (int c = 0; c < dim; ++c) a[c] = q[c] & ~(s - 1);
    if (S.count(LeafKey::make(l, a, dim))) {
      *lev = l;
      for (int c = 0; c < dim; ++c) anc[c] = a[c];
      return true;
    }
  }
  return false;
}

// Neighbour directions of the balance rule: edges (2D); faces + edges (3D).
static std::vector<std::array<int, 3>> balance_dirs(int dim) {
  std::vector<std::array<int, 3>> out;
  for (int dz = (dim == 3 ? -1 : 0); dz <= (dim == 3 ? 1 : 0); ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int nz = (dx != 0) + (dy != 0) + (dz != 0);
        if ((dim == 2 && nz == 1) || (dim == 3 && (nz == 1 || nz == 2))) out.push_back({dx, dy, dz});
      }
  return out;
}

// LSD radix sort of (key, val) pairs by key.
static void radix_sort_pairs(std::vector<uint64_t> &key, std::vector<int64_t> &val) {
  size_t n = key.size();
  uint64_t mx = 0;
  for (auto k : key) mx |= k;
  int bits = 0;
  while (bits < 64 && (mx >> bits)) ++bits;
  std::vector<uint64_t> k2(n);
  std::vector<int64_t> v2(n);
  const int R = 11;
  for (int sh = 0; sh < bits; sh += R) {
    std::vector<size_t> cnt((1u << R) + 1, 0);
    for (size_t i = 0; i < n; ++i) cnt[((key[i] >> sh) & ((1u << R) - 1)) + 1]++;
    for (size_t b = 1; b < cnt.size(); ++b) cnt[b] += cnt[b - 1];
    for (size_t i = 0; i < n; ++i) {
      size_t d = cnt[(key[i] >> sh) & ((1u << R) - 1)]++;
      k2[d] = key[i];
      v2[d] = val[i];
    }
    key.swap(k2);
    val.swap(v2);
  }
}

static int64_t find_node(const std::vector<uint64_t> &keys, int dim, const int32_t *p) {
  uint64_t k = morton(dim, p);
  auto it = std::lower_bound(keys.begin(), keys.end(), k);
  if (it == keys.end() || *it != k) return -1;
  return (int64_t)(it - keys.begin());
}

static int build_filter(tomesh_host *H, double rmin) {
  H->filt_ptr.clear();
  H->filt_idx.clear();
  H->has_filter = false;
  if (!(rmin > 0.0)) return 0;
  const int dim = H->dim, L = H->L;
  const int64_t ne = (int64_t)H->elem_level.size();
  const double hL = H->h0 / (double)(1 << L);
  std::vector<double> cen((size_t)ne * dim);
  for (int64_t e = 0; e < ne; ++e) {
    double s = (double)(1 << (L - H->elem_level[e]));
    for (int c = 0; c < dim; ++c) cen[e * dim + c] = ((double)H->elem_anchor[e * dim + c] + 0.5 * s) * hL;
  }
  // bins of edge >= rmin
  int64_t nb[3] = {1, 1, 1};
  for (int c = 0; c < dim; ++c) {
    double extent = H->ext[c] * hL;
    nb[c] = std::max<int64_t>(1, (int64_t)std::floor(extent / rmin));
  }
  double bw[3];
  for (int c = 0; c < dim; ++c) bw[c] = H->ext[c] * hL / (double)nb[c];
  auto binof = [&](const double *p, int64_t *b) {
    for (int c = 0; c < dim; ++c) {
      int64_t t = (int64_t)std::floor(p[c] / bw[c]);
      b[c] = std::min<int64_t>(std::max<int64_t>(t, 0), nb[c] - 1);
    }
  };
  int64_t nbins = nb[0] * nb[1] * nb[2];
  std::vector<int64_t> head(nbins + 1, 0), ebin(ne);
  for (int64_t e = 0; e < ne; ++e) {
    int64_t b[3] = {0, 0, 0};
    binof(&cen[e * dim], b);
    ebin[e] = b[0] + nb[0] * (b[1] + nb[1] * b[2]);
    head[ebin[e] + 1]++;
  }
  for (int64_t i = 0; i < nbins; ++i) head[i + 1] += head[i];
  std::vector<int64_t> fillp(head.begin(), head.end() - 1);
  std::vector<int32_t> members(ne);
  for (int64_t e = 0; e < ne; ++e) members[fillp[ebin[e]]++] = (int32_t)e;  // ascending e within a bin
  const double r2 = rmin * rmin;
  std::vector<int64_t> cnt(ne + 1, 0);
  std::vector<std::vector<int32_t>> rows(ne);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t e = 0; e < ne; ++e) {
    int64_t b[3] = {0, 0, 0};
    binof(&cen[e * dim], b);
    std::vector<int32_t> &row = rows[e];
    for (int64_t z = (dim == 3 ? b[2] - 1 : 0); z <= (dim == 3 ? b[2] + 1 : 0); ++z) {
      if (z < 0 || z >= nb[2]) continue;
      for (int64_t y = b[1] - 1; y <= b[1] + 1; ++y) {
        if (y < 0 || y >= nb[1]) continue;
        for (int64_t x = b[0] - 1; x <= b[0] + 1; ++x) {
          if (x < 0 || x >= nb[0]) continue;
          int64_t bi = x + nb[0] * (y + nb[1] * z);
          for (int64_t t = head[bi]; t < head[bi + 1]; ++t) {
            int32_t d = members[t];
            double d2 = 0.0;
            for (int c = 0; c < dim; ++c) {
              double df = cen[(int64_t)d * dim + c] - cen[e * dim + c];
              d2 += df * df;
            }
            if (d2 < r2) row.push_back(d);
          }
        }
      }
    }
    std::sort(row.begin(), row.end());
  }
  H->filt_ptr.assign(ne + 1, 0);
  for (int64_t e = 0; e < ne; ++e) H->filt_ptr[e + 1] = H->filt_ptr[e] + (int64_t)rows[e].size();
  H->filt_idx.resize(H->filt_ptr[ne]);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < ne; ++e) {
    std::copy(rows[e].begin(), rows[e].end(), H->filt_idx.begin() + H->filt_ptr[e]);
    std::vector<int32_t>().swap(rows[e]);
  }
  H->has_filter = true;
  return 0;
}

// C10 2:1 balance of a leaf set in place: worklist ripple, refining the
// coarser leaf of any face/edge (3D) or edge (2D) pair more than one level apart.
static int balance_set(LeafSet &S, int dim, int L, const int32_t *ext) {
  const int nc = 1 << dim;
  auto dirs = balance_dirs(dim);
  std::deque<uint64_t> work(S.begin(), S.end());
  while (!work.empty()) {
    uint64_t k = work.front();
    work.pop_front();
    if (!S.count(k)) continue;
    int l = LeafKey::level(k);
    int32_t a[3] = {0, 0, 0};
    LeafKey::anchor(k, dim, a);
    int32_t s = 1 << (L - l);
    for (auto &d : dirs) {
      int32_t q[3] = {0, 0, 0};
      bool inside = true;
      for (int c = 0; c < dim; ++c) {
        q[c] = a[c] + d[c] * s;
        if (q[c] < 0 || q[c] >= ext[c]) inside = false;
      }
      if (!inside) continue;
      for (;;) {
        int lb;
        int32_t ab[3] = {0, 0, 0};
        if (!locate(S, dim, L, q, &lb, ab)) { set_error("point location failed"); return TO_EINVAL; }
        if (lb >= l - 1) break;
        S.erase(LeafKey::make(lb, ab, dim));
        int32_t half = 1 << (L - lb - 1);
        for (int ch = 0; ch < nc; ++ch) {
          int32_t ca[3] = {0, 0, 0};
          for (int c = 0; c < dim; ++c) ca[c] = ab[c] + ((ch >> c) & 1) * half;
          uint64_t ck = LeafKey::make(lb + 1, ca, dim);
          S.insert(ck);
          work.push_back(ck);
        }
      }
    }
  }
  return 0;
}

static int build(const tomesh_host_spec *sp, tomesh_host *H) {
  const int dim = sp->dim, L = sp->max_level;
  if (dim != 2 && dim != 3) { set_error("dim must be 2 or 3"); return TO_EINVAL; }
  if (L < 0 || L > 16) { set_error("max_level out of range"); return TO_EINVAL; }
  H->dim = dim;
  H->L = L;
  H->h0 = sp->h0;
  for (int c = 0; c < 3; ++c) H->ext[c] = (c < dim) ? (sp->base[c] << L) : 1;
  for (int c = 0; c < dim; ++c)
    if (sp->base[c] < 1 || H->ext[c] >= (1 << 19)) { set_error("bad base extent"); return TO_EINVAL; }
  const int nc = 1 << dim;

  // ---- C10: 2:1 balance -------------------------------------------------------
  LeafSet S;
  S.reserve((size_t)sp->n_leaf * 2 + 16);
  int64_t vol = 0, dvol = 1;
  for (int c = 0; c < dim; ++c) dvol *= H->ext[c];
  for (int64_t i = 0; i < sp->n_leaf; ++i) {
    int l = sp->leaf_level[i];
    const int32_t *a = sp->leaf_anchor + i * dim;
    if (l < 0 || l > L) { set_error("leaf %lld: level out of range", (long long)i); return TO_EINVAL; }
    int32_t s = 1 << (L - l);
    for (int c = 0; c < dim; ++c)
      if (a[c] < 0 || a[c] % s != 0 || a[c] + s > H->ext[c]) {
        set_error("leaf %lld: anchor off the lattice or outside the box", (long long)i);
        return TO_EINVAL;
      }
    if (!S.insert(LeafKey::make(l, a, dim)).second) { set_error("duplicate leaf"); return TO_EINVAL; }
    int64_t v = 1;
    for (int c = 0; c < dim; ++c) v *= s;
    vol += v;
  }
  if (vol != dvol) { set_error("leaves do not tile the box (volume %lld vs %lld)", (long long)vol, (long long)dvol); return TO_EINVAL; }
  bool one_level = true;
  for (int64_t i = 1; i < sp->n_leaf; ++i)
    if (sp->leaf_level[i] != sp->leaf_level[0]) { one_level = false; break; }
  if (!one_level) {  // a single-level tiling is trivially balanced
    const int rc = balance_set(S, dim, L, H->ext);
    if (rc != 0) return rc;
  }

  // ---- C2: Morton order of leaves ----------------------------------------------
  const int64_t ne = (int64_t)S.size();
  {
    std::vector<uint64_t> key;
    std::vector<int64_t> val;
    std::vector<uint64_t> lk(S.begin(), S.end());
    key.reserve(ne);
    val.reserve(ne);
    for (int64_t i = 0; i < ne; ++i) {
      int32_t a[3] = {0, 0, 0};
      LeafKey::anchor(lk[i], dim, a);
      key.push_back(morton(dim, a));
      val.push_back(i);
    }
    radix_sort_pairs(key, val);
    H->elem_level.resize(ne);
    H->elem_anchor.resize(ne * dim);
    for (int64_t e = 0; e < ne; ++e) {
      uint64_t k = lk[val[e]];
      H->elem_level[e] = (int8_t)LeafKey::level(k);
      int32_t a[3] = {0, 0, 0};
      LeafKey::anchor(k, dim, a);
      for (int c = 0; c < dim; ++c) H->elem_anchor[e * dim + c] = a[c];
    }
  }

  // ---- C3/C4: nodes and connectivity ---------------------------------------------
  {
    std::vector<uint64_t> key((size_t)ne * nc);
    std::vector<int64_t> slot((size_t)ne * nc);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < ne; ++e) {
      int32_t s = 1 << (L - H->elem_level[e]);
      for (int ch = 0; ch < nc; ++ch) {
        int32_t p[3] = {0, 0, 0};
        for (int c = 0; c < dim; ++c) p[c] = H->elem_anchor[e * dim + c] + ((ch >> c) & 1) * s;
        key[e * nc + ch] = morton(dim, p);
        slot[e * nc + ch] = e * nc + ch;
      }
    }
    radix_sort_pairs(key, slot);
    H->elem_node.resize((size_t)ne * nc);
    H->node_key.clear();
    H->node_coord.clear();
    int64_t id = -1;
    uint64_t prev = ~0ULL;
    for (size_t i = 0; i < key.size(); ++i) {
      if (key[i] != prev) {
        ++id;
        prev = key[i];
        H->node_key.push_back(key[i]);
        int64_t e = slot[i] / nc;
        int ch = (int)(slot[i] % nc);
        int32_t s = 1 << (L - H->elem_level[e]);
        for (int c = 0; c < dim; ++c) H->node_coord.push_back(H->elem_anchor[e * dim + c] + ((ch >> c) & 1) * s);
      }
      H->elem_node[slot[i]] = (int32_t)id;
    }
  }
  const int64_t nn = (int64_t)H->node_key.size();
  if (nn >= (1LL << 31) / dim) { set_error("too many nodes"); return TO_EINVAL; }

  // ---- C6: hanging nodes (node-centric) ------------------------------------------
  std::vector<uint8_t> is_hang(nn, 0);
  {
    bool uniform = true;
    for (int64_t e = 0; e < ne; ++e)
      if (H->elem_level[e] != H->elem_level[0]) { uniform = false; break; }
    std::vector<std::array<int32_t, 4>> par(uniform ? 0 : nn);
    std::vector<int8_t> npar(uniform ? 0 : nn, 0);
    if (!uniform) {
      std::atomic<int> err{0};
#pragma omp parallel for schedule(dynamic, 1024)
      for (int64_t n = 0; n < nn; ++n) {
        const int32_t *p = &H->node_coord[n * dim];
        for (int cell = 0; cell < nc; ++cell) {
          int32_t q[3] = {0, 0, 0};
          bool inside = true;
          for (int c = 0; c < dim; ++c) {
            q[c] = p[c] - ((cell >> c) & 1);
            if (q[c] < 0 || q[c] >= H->ext[c]) inside = false;
          }
          if (!inside) continue;
          int lb;
          int32_t ab[3] = {0, 0, 0};
          if (!locate(S, dim, L, q, &lb, ab)) { err = 1; continue; }
          int32_t sb = 1 << (L - lb);
          int nfree = 0, freeax[3] = {0, 0, 0};
          bool mid_ok = true;
          for (int c = 0; c < dim; ++c) {
            if (p[c] != ab[c] && p[c] != ab[c] + sb) {
              freeax[nfree++] = c;
              if (2 * (p[c] - ab[c]) != sb) mid_ok = false;
            }
          }
          if (nfree == 0) continue;            // p is a corner of this leaf
          if (!mid_ok || nfree == dim) { err = 2; continue; }
          int np = 1 << nfree;
          if (np > 4) { err = 2; continue; }
          std::array<int32_t, 4> pp = {-1, -1, -1, -1};
          for (int m = 0; m < np; ++m) {
            int32_t r[3] = {p[0], p[1], dim == 3 ? p[2] : 0};
            for (int t = 0; t < nfree; ++t) r[freeax[t]] = ab[freeax[t]] + ((m >> t) & 1) * sb;
            pp[m] = (int32_t)find_node(H->node_key, dim, r);
            if (pp[m] < 0) err = 3;
          }
          for (int u = 1; u < np; ++u)   // insertion sort, np <= 4
            for (int v = u; v > 0 && pp[v - 1] > pp[v]; --v) std::swap(pp[v - 1], pp[v]);
          if (npar[n] == 0) {
            npar[n] = (int8_t)np;
            par[n] = pp;
          } else if (npar[n] != np || par[n] != pp) {
            err = 4;
          }
        }
      }
      if (err.load()) { set_error("hanging-node classification failed (code %d): mesh not 2:1 balanced?", err.load()); return TO_EMESH; }
      int32_t ptr = 0;
      H->hang_ptr.push_back(0);
      for (int64_t n = 0; n < nn; ++n) {
        if (!npar[n]) continue;
        is_hang[n] = 1;
        H->hang_node.push_back((int32_t)n);
        for (int m = 0; m < npar[n]; ++m) {
          H->hang_parent.push_back(par[n][m]);
          H->hang_weight.push_back(1.0 / npar[n]);
        }
        ptr += npar[n];
        H->hang_ptr.push_back(ptr);
      }
      for (int32_t p : H->hang_parent)
        if (npar[p]) { set_error("chained constraint: parent %d is hanging", p); return TO_EMESH; }
    } else {
      H->hang_ptr.push_back(0);
    }
  }

  // ---- C7: Dirichlet DOFs ----------------------------------------------------------
  for (int64_t n = 0; n < nn; ++n) {
    if (is_hang[n]) continue;
    const int32_t *p = &H->node_coord[n * dim];
    int mask = 0;
    for (int b = 0; b < sp->n_fixed_box; ++b) {
      const int32_t *bx = sp->fixed_box + (size_t)b * 2 * dim;
      bool in = true;
      for (int c = 0; c < dim; ++c)
        if (p[c] < bx[c] || p[c] > bx[dim + c]) in = false;
      if (in) mask |= sp->fixed_mask[b];
    }
    for (int c = 0; c < dim; ++c)
      if ((mask >> c) & 1) H->fixed_dof.push_back(n * dim + c);
  }

  // ---- C8: consistent loads ----------------------------------------------------------
  H->load.assign((size_t)nn * dim, 0.0);
  const double hL = sp->h0 / (double)(1 << L);
  for (int i = 0; i < sp->n_load; ++i) {
    const int32_t *bx = sp->load_box + (size_t)i * 2 * dim;
    const double *vec = sp->load_vec + (size_t)i * dim;
    int kind = sp->load_kind[i];
    if (kind == TOH_LOAD_POINT) {
      int64_t n = find_node(H->node_key, dim, bx);
      if (n < 0) { set_error("point load %d is not on a node", i); return TO_EINVAL; }
      for (int c = 0; c < dim; ++c) H->load[n * dim + c] += vec[c];
      continue;
    }
    int span[3], nspan = 0, fixax[3], nfix = 0;
    for (int c = 0; c < dim; ++c) {
      if (bx[c] != bx[dim + c]) span[nspan++] = c; else fixax[nfix++] = c;
    }
    if ((kind == TOH_LOAD_LINE && nspan != 1) || (kind == TOH_LOAD_FACE && (nspan != 2 || dim != 3))) {
      set_error("load %d: region has the wrong dimension", i);
      return TO_EINVAL;
    }
    for (int64_t e = 0; e < ne; ++e) {
      int32_t s = 1 << (L - H->elem_level[e]);
      const int32_t *a = &H->elem_anchor[e * dim];
      bool hit = true;
      for (int t = 0; t < nfix; ++t) {
        int c = fixax[t];
        if (a[c] != bx[c] && a[c] + s != bx[c]) hit = false;
      }
      for (int t = 0; t < nspan; ++t) {
        int c = span[t];
        if (a[c] < bx[c] || a[c] + s > bx[dim + c]) hit = false;
      }
      if (!hit) continue;
      double meas = 1.0;
      for (int t = 0; t < nspan; ++t) meas *= (double)s * hL;
      int np = 1 << nspan;
      for (int m = 0; m < np; ++m) {
        int32_t r[3] = {0, 0, 0};
        for (int t = 0; t < nfix; ++t) r[fixax[t]] = bx[fixax[t]];
        for (int t = 0; t < nspan; ++t) r[span[t]] = a[span[t]] + ((m >> t) & 1) * s;
        int64_t n = find_node(H->node_key, dim, r);
        if (n < 0) { set_error("load %d: corner not a node", i); return TO_EINVAL; }
        for (int c = 0; c < dim; ++c) H->load[n * dim + c] += vec[c] * (meas / np);
      }
    }
  }

  // ---- C9: filter neighbour lists ----------------------------------------------------
  return build_filter(H, sp->rmin);
}

}  // namespace

extern "C" int tomesh_host_build(const tomesh_host_spec *spec, tomesh_host **out) {
  clear_error();
  if (!spec || !out) { set_error("NULL argument"); return TO_EINVAL; }
  *out = nullptr;
  tomesh_host *H = new (std::nothrow) tomesh_host();
  if (!H) { set_error("out of host memory"); return TO_ENOMEM; }
  int rc;
  try {
    rc = build(spec, H);
  } catch (const std::bad_alloc &) {
    set_error("out of host memory");
    rc = TO_ENOMEM;
  } catch (...) {
    set_error("internal error in tomesh_host_build");
    rc = TO_EINVAL;
  }
  if (rc != 0) { delete H; return rc; }
  *out = H;
  return 0;
}

extern "C" int tomesh_host_get(const tomesh_host *H, tomesh_host_arrays *o) {
  if (!H || !o) { set_error("NULL argument"); return TO_EINVAL; }
  o->dim = H->dim;
  o->max_level = H->L;
  o->h0 = H->h0;
  o->n_elem = (int64_t)H->elem_level.size();
  o->n_node = (int64_t)H->node_key.size();
  o->n_hang = (int64_t)H->hang_node.size();
  o->n_hang_nnz = (int64_t)H->hang_parent.size();
  o->n_fixed = (int64_t)H->fixed_dof.size();
  o->filt_nnz = H->has_filter ? (int64_t)H->filt_idx.size() : 0;
  o->elem_node = H->elem_node.data();
  o->elem_anchor = H->elem_anchor.data();
  o->elem_level = H->elem_level.data();
  o->node_coord = H->node_coord.data();
  o->hang_node = H->hang_node.data();
  o->hang_ptr = H->hang_ptr.data();
  o->hang_parent = H->hang_parent.data();
  o->hang_weight = H->hang_weight.data();
  o->fixed_dof = H->fixed_dof.data();
  o->load = H->load.data();
  o->filt_ptr = H->has_filter ? H->filt_ptr.data() : nullptr;
  o->filt_idx = H->has_filter ? H->filt_idx.data() : nullptr;
  return 0;
}

extern "C" int tomesh_host_filter(tomesh_host *H, double rmin) {
  if (!H) { set_error("NULL argument"); return TO_EINVAL; }
  try {
    return build_filter(H, rmin);
  } catch (...) {
    set_error("out of host memory");
    return TO_ENOMEM;
  }
}

extern "C" void tomesh_host_free(tomesh_host *H) { delete H; }

// ======================================================================================
// Dynamic AMR: compatibility sweeps on the device-computed
// marks, refine/derefine, density transfer.  Readings R21-R23.
// ======================================================================================

struct tomesh_adapt {
  int dim = 0, L = 0;
  std::vector<int8_t> leaf_level, marks;
  std::vector<int32_t> leaf_anchor;
  std::vector<double> leaf_x;
  int64_t n_refined = 0, n_groups = 0, n_unmarked_sibling = 0, n_unmarked_incompat = 0;
};

namespace {

static int adapt(const tomesh_host *H, const int8_t *marks_in, const double *x, tomesh_adapt *A) {
  const int dim = H->dim, L = H->L, nc = 1 << dim;
  const int64_t ne = (int64_t)H->elem_level.size();
  A->dim = dim;
  A->L = L;
  std::vector<int8_t> m(marks_in, marks_in + ne);
  for (int64_t e = 0; e < ne; ++e) {
    const int l = H->elem_level[e];
    if (m[e] < -1 || m[e] > 1) { set_error("marks must be -1, 0 or +1"); return TO_EINVAL; }
    if ((m[e] == 1 && l >= L) || (m[e] == -1 && l == 0)) { set_error("mark beyond the level range"); return TO_EINVAL; }
  }
  std::unordered_map<uint64_t, int64_t, Splitmix> where;
  where.reserve((size_t)ne * 2);
  for (int64_t e = 0; e < ne; ++e) where[LeafKey::make(H->elem_level[e], &H->elem_anchor[e * dim], dim)] = e;
  // siblings of e in corner order (-1 where the sibling is not a leaf)
  auto group = [&](int64_t e, int32_t *pa, int64_t *sib) {
    const int l = H->elem_level[e];
    const int32_t s = 1 << (L - l);
    for (int c = 0; c < dim; ++c) pa[c] = H->elem_anchor[e * dim + c] & ~(2 * s - 1);
    for (int ch = 0; ch < nc; ++ch) {
      int32_t a[3] = {0, 0, 0};
      for (int c = 0; c < dim; ++c) a[c] = pa[c] + ((ch >> c) & 1) * s;
      auto it = where.find(LeafKey::make(l, a, dim));
      sib[ch] = it == where.end() ? -1 : it->second;
    }
  };
  // sweep 1: every sibling a leaf marked for derefinement
  {
    std::vector<int8_t> m1(m);
    for (int64_t e = 0; e < ne; ++e) {
      if (m[e] != -1) continue;
      int32_t pa[3];
      int64_t sib[8];
      group(e, pa, sib);
      for (int ch = 0; ch < nc; ++ch)
        if (sib[ch] < 0 || m[sib[ch]] != -1) {
          m1[e] = 0;
          A->n_unmarked_sibling++;
          break;
        }
    }
    m.swap(m1);
  }
  // sweep 2: no leaf two or more levels finer than the parent across a face/edge,
  // in the 2:1 closure of this pass's refinements
  {
    LeafSet C;
    C.reserve((size_t)ne * 2 + 16);
    for (int64_t e = 0; e < ne; ++e) {
      const int l = H->elem_level[e];
      const int32_t *a = &H->elem_anchor[e * dim];
      if (m[e] == 1) {
        const int32_t half = 1 << (L - l - 1);
        for (int ch = 0; ch < nc; ++ch) {
          int32_t ca[3] = {0, 0, 0};
          for (int c = 0; c < dim; ++c) ca[c] = a[c] + ((ch >> c) & 1) * half;
          C.insert(LeafKey::make(l + 1, ca, dim));
        }
      } else {
        C.insert(LeafKey::make(l, a, dim));
      }
    }
    const int rc = balance_set(C, dim, L, H->ext);
    if (rc != 0) return rc;
    auto dirs = balance_dirs(dim);
    std::vector<char> seen(ne, 0);
    for (int64_t e = 0; e < ne; ++e) {
      if (m[e] != -1 || seen[e]) continue;
      int32_t pa[3] = {0, 0, 0};
      int64_t sib[8];
      group(e, pa, sib);
      for (int ch = 0; ch < nc; ++ch) seen[sib[ch]] = 1;
      const int l = H->elem_level[e];
      bool bad = false;
      if (l < L) {
        const int32_t S2 = 2 * (1 << (L - l)), t = (1 << (L - l)) / 2;
        for (auto &d : dirs) {
          // probe cells of edge t along the parent's side(s) in direction d
          int32_t lo[3] = {0, 0, 0}, cnt[3] = {1, 1, 1};
          for (int c = 0; c < dim; ++c) {
            if (d[c] < 0) lo[c] = pa[c] - t;
            else if (d[c] > 0) lo[c] = pa[c] + S2;
            else { lo[c] = pa[c]; cnt[c] = S2 / t; }
          }
          for (int32_t k2 = 0; k2 < cnt[2] && !bad; ++k2)
            for (int32_t k1 = 0; k1 < cnt[1] && !bad; ++k1)
              for (int32_t k0 = 0; k0 < cnt[0] && !bad; ++k0) {
                int32_t q[3] = {lo[0] + k0 * t, lo[1] + k1 * t, lo[2] + k2 * t};
                bool inside = true;
                for (int c = 0; c < dim; ++c)
                  if (q[c] < 0 || q[c] >= H->ext[c]) inside = false;
                if (!inside) continue;
                int lb;
                int32_t ab[3];
                if (!locate(C, dim, L, q, &lb, ab)) { set_error("point location failed"); return TO_EINVAL; }
                if (lb >= l + 1) bad = true;
              }
          if (bad) break;
        }
      }
      if (bad)
        for (int ch = 0; ch < nc; ++ch)
          if (m[sib[ch]] == -1) {
            m[sib[ch]] = 0;
            A->n_unmarked_incompat++;
          }
    }
  }
  // the new pre-balance leaf set with transferred densities
  std::vector<uint64_t> key;
  std::vector<int64_t> val;
  std::vector<int8_t> lv;
  std::vector<int32_t> an;
  std::vector<double> xv;
  auto emit = [&](int l, const int32_t *a, double xe) {
    key.push_back(morton(dim, a));
    val.push_back((int64_t)lv.size());
    lv.push_back((int8_t)l);
    for (int c = 0; c < dim; ++c) an.push_back(a[c]);
    xv.push_back(xe);
  };
  for (int64_t e = 0; e < ne; ++e) {
    const int l = H->elem_level[e];
    const int32_t *a = &H->elem_anchor[e * dim];
    const int32_t s = 1 << (L - l);
    if (m[e] == 1) {
      A->n_refined++;
      for (int ch = 0; ch < nc; ++ch) {
        int32_t ca[3] = {0, 0, 0};
        for (int c = 0; c < dim; ++c) ca[c] = a[c] + ((ch >> c) & 1) * (s / 2);
        emit(l + 1, ca, x[e]);
      }
    } else if (m[e] == -1) {
      int32_t pa[3] = {0, 0, 0};
      int64_t sib[8];
      group(e, pa, sib);
      bool first = true;
      for (int c = 0; c < dim; ++c) first = first && (pa[c] == a[c]);
      if (first) {
        double acc = 0.0;   // mean of the children in corner order
        for (int ch = 0; ch < nc; ++ch) acc += x[sib[ch]];
        A->n_groups++;
        emit(l - 1, pa, acc / nc);
      }
    } else {
      emit(l, a, x[e]);
    }
  }
  radix_sort_pairs(key, val);
  const int64_t n = (int64_t)val.size();
  A->leaf_level.resize(n);
  A->leaf_anchor.resize(n * dim);
  A->leaf_x.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t j = val[i];
    A->leaf_level[i] = lv[j];
    for (int c = 0; c < dim; ++c) A->leaf_anchor[i * dim + c] = an[j * dim + c];
    A->leaf_x[i] = xv[j];
  }
  A->marks.swap(m);
  return 0;
}

}  // namespace

extern "C" int tomesh_host_adapt(const tomesh_host *H, const int8_t *marks, const double *x, tomesh_adapt **out) {
  clear_error();
  if (!H || !marks || !x || !out) { set_error("NULL argument"); return TO_EINVAL; }
  *out = nullptr;
  tomesh_adapt *A = new (std::nothrow) tomesh_adapt();
  if (!A) { set_error("out of host memory"); return TO_ENOMEM; }
  int rc;
  try {
    rc = adapt(H, marks, x, A);
  } catch (const std::bad_alloc &) {
    set_error("out of host memory");
    rc = TO_ENOMEM;
  } catch (...) {
    set_error("internal error in tomesh_host_adapt");
    rc = TO_EINVAL;
  }
  if (rc != 0) { delete A; return rc; }
  *out = A;
  return 0;
}

extern "C" int tomesh_adapt_get(const tomesh_adapt *A, tomesh_adapt_result *o) {
  if (!A || !o) { set_error("NULL argument"); return TO_EINVAL; }
  o->n_leaf = (int64_t)A->leaf_level.size();
  o->leaf_level = A->leaf_level.data();
  o->leaf_anchor = A->leaf_anchor.data();
  o->leaf_x = A->leaf_x.data();
  o->marks = A->marks.data();
  o->n_refined = A->n_refined;
  o->n_groups = A->n_groups;
  o->n_unmarked_sibling = A->n_unmarked_sibling;
  o->n_unmarked_incompat = A->n_unmarked_incompat;
  return 0;
}

extern "C" int tomesh_host_transfer(const tomesh_host *H, const tomesh_adapt *A, double *x_out) {
  clear_error();
  if (!H || !A || !x_out) { set_error("NULL argument"); return TO_EINVAL; }
  if (H->dim != A->dim || H->L != A->L) { set_error("mesh and adaptation differ in dim or max_level"); return TO_EINVAL; }
  const int dim = H->dim;
  std::unordered_map<uint64_t, double, Splitmix> xs;
  LeafSet P;
  const int64_t n = (int64_t)A->leaf_level.size();
  xs.reserve((size_t)n * 2);
  P.reserve((size_t)n * 2);
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t k = LeafKey::make(A->leaf_level[i], &A->leaf_anchor[i * dim], dim);
    xs[k] = A->leaf_x[i];
    P.insert(k);
  }
  const int64_t ne = (int64_t)H->elem_level.size();
  for (int64_t e = 0; e < ne; ++e) {
    int lb;
    int32_t ab[3];
    if (!locate(P, dim, H->L, &H->elem_anchor[e * dim], &lb, ab) || lb > H->elem_level[e]) {
      set_error("element %lld is not inside a leaf of the adaptation", (long long)e);
      return TO_EINVAL;
    }
    x_out[e] = xs[LeafKey::make(lb, ab, dim)];
  }
  return 0;
}

extern "C" void tomesh_adapt_free(tomesh_adapt *A) { delete A; }
