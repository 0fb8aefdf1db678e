// libtomesh — C ABI entry points (include/tomesh.h) and the host side of the
// device path: validation, upload, the PCG driver loop, sensitivities, filter,
// AMR marks and the operator-level calls.  MINRES / IC(0): tomesh_minres.cu;
// OC update and the Fig. 1 loop: tomesh_opt.cu.
#include "tomesh_impl.cuh"
#include "kernels_cg.cuh"
#include "kernels_general.cuh"
#include "kernels_genfused.cuh"
#include "kernels_gencluster.cuh"
#include "kernels_genep.cuh"
#include "kernels_struct3d.cuh"

using namespace tomesh;

int validate(const to_mesh_desc *d) {
  if (d->dim != 2 && d->dim != 3) { set_error("dim must be 2 or 3"); return TO_EINVAL; }
  if (d->n_elem <= 0 || d->n_node <= 0) { set_error("empty mesh"); return TO_EINVAL; }
  if (d->max_level < 0 || d->max_level > 20) { set_error("max_level out of range"); return TO_EINVAL; }
  if (!d->elem_node || !d->elem_anchor || !d->elem_level || !d->load) { set_error("NULL mesh array"); return TO_EINVAL; }
  if (d->n_node * d->dim >= (1LL << 31)) { set_error("too many DOFs for int32 node ids"); return TO_EINVAL; }
  if (!(d->h0 > 0.0) || !(d->E0 > 0.0) || !(d->Emin >= 0.0) || !(d->nu > -1.0 && d->nu < 0.5)) {
    set_error("bad material or geometry constants");
    return TO_EINVAL;
  }
  const int nc = 1 << d->dim;
  for (int64_t i = 0; i < d->n_elem * nc; ++i)
    if (d->elem_node[i] < 0 || d->elem_node[i] >= d->n_node) {
      set_error("elem_node[%lld] = %d out of range", (long long)i, d->elem_node[i]);
      return TO_EMESH;
    }
  for (int64_t e = 0; e < d->n_elem; ++e)
    if (d->elem_level[e] < 0 || d->elem_level[e] > d->max_level) { set_error("elem_level out of range"); return TO_EMESH; }
  if (d->n_hang < 0 || (d->n_hang > 0 && (!d->hang_node || !d->hang_ptr || !d->hang_parent || !d->hang_weight))) {
    set_error("bad hanging arrays");
    return TO_EINVAL;
  }
  std::vector<char> hang(d->n_node, 0);
  for (int64_t h = 0; h < d->n_hang; ++h) {
    int32_t n = d->hang_node[h];
    if (n < 0 || n >= d->n_node || (h > 0 && n <= d->hang_node[h - 1])) { set_error("hang_node not ascending / out of range"); return TO_EMESH; }
    hang[n] = 1;
  }
  if (d->n_hang > 0 && d->hang_ptr[0] != 0) { set_error("hang_ptr[0] != 0"); return TO_EMESH; }
  for (int64_t h = 0; h < d->n_hang; ++h) {
    int32_t a = d->hang_ptr[h], b = d->hang_ptr[h + 1];
    if (b <= a || b - a > 4) { set_error("hanging node %lld has %d parents", (long long)h, b - a); return TO_EMESH; }
    double wsum = 0.0;
    for (int32_t k = a; k < b; ++k) {
      int32_t p = d->hang_parent[k];
      if (p < 0 || p >= d->n_node) { set_error("hang_parent out of range"); return TO_EMESH; }
      if (hang[p]) { set_error("constraint parent %d of hanging node %d is itself hanging", p, d->hang_node[h]); return TO_EMESH; }
      if (k > a && p <= d->hang_parent[k - 1]) { set_error("hang_parent not ascending"); return TO_EMESH; }
      wsum += d->hang_weight[k];
    }
    if (std::fabs(wsum - 1.0) > 1e-12) { set_error("hanging weights of node %d sum to %.17g", d->hang_node[h], wsum); return TO_EMESH; }
  }
  if (d->n_fixed < 0 || (d->n_fixed > 0 && !d->fixed_dof)) { set_error("bad fixed_dof"); return TO_EINVAL; }
  for (int64_t i = 0; i < d->n_fixed; ++i) {
    int64_t f = d->fixed_dof[i];
    if (f < 0 || f >= d->n_node * d->dim || (i > 0 && f <= d->fixed_dof[i - 1])) { set_error("fixed_dof not ascending / out of range"); return TO_EMESH; }
    if (hang[f / d->dim]) { set_error("fixed DOF %lld is on a hanging node", (long long)f); return TO_EMESH; }
  }
  if ((d->options & ~(uint32_t)(TO_UPLOAD_GENERAL | TO_UPLOAD_LAUNCHED | TO_UPLOAD_NO_CLUSTER | TO_UPLOAD_EP |
                                TO_UPLOAD_NO_EP)) != 0) {
    set_error("unknown upload option bits 0x%x", d->options);
    return TO_EINVAL;
  }
  if (d->n_owned < 0 || d->n_owned > d->n_node) { set_error("n_owned outside [0, n_node]"); return TO_EINVAL; }
  if (d->rmin > 0.0) {
    if (!d->filt_ptr || !d->filt_idx) { set_error("rmin > 0 but no filter lists"); return TO_EINVAL; }
    if (d->filt_ptr[0] != 0 || d->filt_ptr[d->n_elem] != d->filt_nnz) { set_error("bad filt_ptr"); return TO_EMESH; }
    for (int64_t e = 0; e < d->n_elem; ++e)
      if (d->filt_ptr[e + 1] < d->filt_ptr[e]) { set_error("filt_ptr not monotone"); return TO_EMESH; }
    for (int64_t k = 0; k < d->filt_nnz; ++k)
      if (d->filt_idx[k] < 0 || d->filt_idx[k] >= d->n_elem) { set_error("filt_idx out of range"); return TO_EMESH; }
  }
  return 0;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    else
      cudaGetLastError();
  }
  return fn;
}

// 3D fp64 tensor map over [d2][d1][d0] with a (b0 x b1 x 1) box; OOB reads are 0.
int make_tensor_map(CUtensorMap *map, const double *base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0,
                    uint32_t b1) {
  auto enc = tensor_map_encoder();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return TO_ECUDA; }
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * 8, d0 * d1 * 8};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d)", (int)r); return TO_ECUDA; }
  return 0;
}

// Uniform 3D meshes (one level, leaves tiling a box, no hanging nodes) use the
// structured fast path: lexicographic internal vectors, implicit connectivity.
// Host-planned K1 grid: z segments of two lengths by x tile column so that
// the CTA count fills whole waves of resident slots; long CTAs are dispatched
// first, so each slot pairs a long with a short one.  Chosen only if the
// simulated in-order list schedule beats the uniform segmentation.
// [z0, z1): the node planes to own (a shard's owned range); force: always
// install a plan (uniform segments if nothing beats them).
int plan_s3(to_mesh *m, cudaStream_t st, int z0, int z1, bool force, const int4 **plan_out, int *ncta_out) {
  const GridView &G = m->G;
  const int NZo = z1 - z0;
  const int slots = kNumSMs * kS3CtasPerSM, over = 3;   // ~3 planes of start-up per CTA
  auto makespan = [&](const std::vector<int> &len) {
    std::vector<int64_t> fin(slots, 0);
    int64_t t_max = 0;
    for (size_t c = 0; c < len.size(); ++c) {
      auto it = std::min_element(fin.begin(), fin.end());
      *it += len[c] + over;
      t_max = std::max(t_max, *it);
    }
    return t_max;
  };
  std::vector<int> uni;
  std::vector<int4> uni_plan;
  {
    const int zl = std::min(G.zlen, NZo), nzs = (NZo + zl - 1) / zl;
    for (int z = 0; z < nzs; ++z)
      for (int ty = 0; ty < G.nty; ++ty)
        for (int tx = 0; tx < G.ntx; ++tx) {
          const int lo = z0 + z * zl, hi = std::min(z1, lo + zl);
          uni.push_back(hi - lo);
          uni_plan.push_back(make_int4(tx, ty, lo, hi));
        }
  }
  int64_t best = makespan(uni);
  std::vector<int4> best_plan;
  if (force) best_plan = uni_plan;
  const int tiles = G.ntx * G.nty;
  for (int W = 1; W <= 6; ++W) {
    const int T = W * slots, n_lo = T / tiles;
    if (n_lo < 1) continue;
    int a = (T - tiles * n_lo) / G.nty;          // columns with n_lo + 1 segments
    a = std::min(a, G.ntx);
    std::vector<int4> plan;
    std::vector<int> len;
    for (int pass = 0; pass < 2; ++pass) {         // long CTAs (n_lo segments) first
      for (int seg = 0; seg < n_lo + 1; ++seg)
        for (int ty = 0; ty < G.nty; ++ty)
          for (int tx = 0; tx < G.ntx; ++tx) {
            const int ns = tx < a ? n_lo + 1 : n_lo;
            if ((pass == 0) != (ns == n_lo) || seg >= ns) continue;
            const int zl = (NZo + ns - 1) / ns;
            const int lo = z0 + seg * zl, hi = std::min(z1, lo + zl);
            if (lo >= hi) continue;
            plan.push_back(make_int4(tx, ty, lo, hi));
            len.push_back(hi - lo);
          }
    }
    const int64_t ms = makespan(len);
    if (ms < best) {
      best = ms;
      best_plan = plan;
    }
  }
  if (best_plan.empty()) return 0;
  int4 *d = nullptr;
  RC(upload_array(m, &d, best_plan.data(), best_plan.size(), st));
  *plan_out = d;
  *ncta_out = (int)best_plan.size();
  RC(ensure_partials(m, best_plan.size() * 5));
  return 0;
}

int setup_structured(const to_mesh_desc *d, const std::vector<uint8_t> &free_dof, cudaStream_t st, to_mesh *m) {
  m->structured = false;
  if (d->dim != 3 || d->n_hang != 0 || m->force_general) return 0;
  const int8_t lev0 = d->elem_level[0];
  for (int64_t e = 1; e < d->n_elem; ++e)
    if (d->elem_level[e] != lev0) return 0;
  const int32_t sz = 1 << (d->max_level - lev0);
  int64_t ext[3] = {0, 0, 0};
  for (int64_t e = 0; e < d->n_elem; ++e)
    for (int c = 0; c < 3; ++c) ext[c] = std::max<int64_t>(ext[c], d->elem_anchor[e * 3 + c] / sz + 1);
  if (ext[0] * ext[1] * ext[2] != d->n_elem) return 0;
  if ((ext[0] + 1) * (ext[1] + 1) * (ext[2] + 1) != d->n_node) return 0;
  if (ext[0] + 1 >= (1 << 30) / 4) return 0;
  GridView G{};
  G.EX = (int)ext[0]; G.EY = (int)ext[1]; G.EZ = (int)ext[2];
  G.NX = G.EX + 1; G.NY = G.EY + 1; G.NZ = G.EZ + 1;
  G.NXP = G.NX + (G.NX & 1);              // even node count per row: node pairs never straddle rows
  G.RS = 3 * G.NXP;                       // every node row 16-byte aligned
  if ((int64_t)G.RS * G.NY * G.NZ >= (1LL << 31) - kS3PadBack) return 0;
  G.ntx = (G.NX + 30) / 31;
  G.nty = (G.NY + kS3TYW - 2) / (kS3TYW - 1);
  // z segmentation: balance full waves (2 CTAs/SM) against the one recomputed layer per segment
  {
    const int64_t base = (int64_t)G.ntx * G.nty, slots = (int64_t)kNumSMs * kS3CtasPerSM;
    double best = 1e300;
    int best_n = 1;
    for (int nz = 1; nz <= G.NZ; ++nz) {
      int zlen = (G.NZ + nz - 1) / nz;
      int nseg = (G.NZ + zlen - 1) / zlen;
      double waves = std::ceil((double)(base * nseg) / (double)slots);
      double cost = waves * (zlen + 1);
      if (cost < best - 1e-9) { best = cost; best_n = nseg; }
    }
    G.zlen = (G.NZ + best_n - 1) / best_n;
    G.nzs = (G.NZ + G.zlen - 1) / G.zlen;
  }
  // all 24 diagonal entries of the cube's K0 are equal (symmetry); Dinv uses one
  for (int a = 1; a < 24; ++a)
    if (std::fabs(m->K3.K[a * 24 + a] - m->K3.K[0]) > 1e-14 * std::fabs(m->K3.K[0])) return 0;
  // Dirichlet conditions must clamp whole nodes (one Dinv per node)
  for (int64_t n = 0; n < d->n_node; ++n)
    if (free_dof[n * 3] != free_dof[n * 3 + 1] || free_dof[n * 3] != free_dof[n * 3 + 2]) return 0;
  std::vector<int32_t> perm_el(d->n_elem), perm_node(d->n_node, -1);
  for (int64_t e = 0; e < d->n_elem; ++e) {
    const int32_t *a = d->elem_anchor + e * 3;
    const int64_t ei = a[0] / sz, ej = a[1] / sz, ek = a[2] / sz;
    perm_el[e] = (int32_t)(ei + G.EX * (ej + (int64_t)G.EY * ek));
    for (int c = 0; c < 8; ++c) {
      const int64_t ni = ei + (c & 1), nj = ej + ((c >> 1) & 1), nk = ek + (c >> 2);
      perm_node[d->elem_node[e * 8 + c]] = (int32_t)((nj + (int64_t)G.NY * nk) * G.RS + 3 * ni);
    }
  }
  m->n_int = (int64_t)G.RS * G.NY * G.NZ;
  m->n_int_nodes = (int64_t)G.NXP * G.NY * G.NZ;
  std::vector<uint8_t> free_lex(m->n_int, 0), free_node(m->n_int_nodes, 0);
  for (int64_t n = 0; n < d->n_node; ++n) {
    if (perm_node[n] < 0) return 0;
    for (int c = 0; c < 3; ++c) free_lex[(int64_t)perm_node[n] + c] = free_dof[n * 3 + c];
    free_node[perm_node[n] / 3] = free_dof[n * 3];
  }
  RC(upload_array(m, &m->perm_el, perm_el.data(), perm_el.size(), st));
  RC(upload_array(m, &m->perm_node, perm_node.data(), perm_node.size(), st));
  RC(upload_array(m, &m->free_lex, free_lex.data(), free_lex.size(), st));
  RC(upload_array(m, &m->free_node_lex, free_node.data(), free_node.size(), st));
  {
    double *base = nullptr;
    const size_t cnt = (size_t)(m->n_int_nodes + kS3PadFront + kS3PadBack);
    RC(m->alloc(&base, cnt));
    CK(cudaMemsetAsync(base, 0, sizeof(double) * cnt, st));
    m->dn = base + kS3PadFront;
  }
  // K1 reduces 5 values per CTA (grid_sum<5>), on the uniform grid or the plan
  const int64_t grid = (int64_t)G.ntx * G.nty * G.nzs;
  RC(ensure_partials(m, (size_t)grid * 5));
  m->G = G;
  RC(plan_s3(m, st, 0, G.NZ, false, &m->G.plan, &m->s3_ncta));
  m->k0d = m->K3.K[0];
  m->h_struct = m->hL * (double)sz;
  m->structured = true;
  m->matvec_variant = 1;
  const size_t smem = sizeof(S3Smem<kS3TYW>);
  CK(cudaFuncSetAttribute(k_apply_s3<kS3TYW, S3_CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_apply_s3<kS3TYW, S3_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return 0;
}


// General path: node -> (element, corner, weight) incidence CSR, the transpose
// of the gather C_e P_e: a non-hanging corner contributes to its node with
// weight 1, a hanging corner to each parent with the Eq. 6 weight.  Entries
// per node in ascending (element, corner) order (deterministic sums).
int setup_incidence(const to_mesh_desc *d, const std::vector<int32_t> &node_hang, cudaStream_t st, to_mesh *m,
                    std::vector<int64_t> &ptr, std::vector<uint32_t> &inc) {
  const int nc = 1 << d->dim;
  if ((int64_t)d->n_elem * nc >= (1LL << 30)) { set_error("mesh too large for the packed incidence list"); return TO_EINVAL; }
  ptr.assign(d->n_node + 1, 0);
  for (int64_t e = 0; e < d->n_elem; ++e)
    for (int c = 0; c < nc; ++c) {
      const int32_t n = d->elem_node[e * nc + c];
      const int32_t h = node_hang[n];
      if (h < 0) ptr[n + 1]++;
      else
        for (int32_t k = d->hang_ptr[h]; k < d->hang_ptr[h + 1]; ++k) ptr[d->hang_parent[k] + 1]++;
    }
  for (int64_t n = 0; n < d->n_node; ++n) ptr[n + 1] += ptr[n];
  inc.assign(ptr[d->n_node], 0u);
  std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
  auto code = [](double w) -> uint32_t { return w == 1.0 ? 0u : w == 0.5 ? 1u : 2u; };
  for (int64_t e = 0; e < d->n_elem; ++e)
    for (int c = 0; c < nc; ++c) {
      const int32_t n = d->elem_node[e * nc + c];
      const int32_t h = node_hang[n];
      const uint32_t idx = (uint32_t)(e * nc + c);
      if (h < 0) inc[fill[n]++] = idx;
      else
        for (int32_t k = d->hang_ptr[h]; k < d->hang_ptr[h + 1]; ++k) {
          const double w = d->hang_weight[k];
          if (w != 1.0 && w != 0.5 && w != 0.25) { set_error("hanging weight %g not in {1, 1/2, 1/4}", w); return TO_EMESH; }
          inc[fill[d->hang_parent[k]]++] = idx | (code(w) << 30);
        }
    }
  RC(upload_array(m, &m->inc_ptr, ptr.data(), ptr.size(), st));
  RC(upload_array(m, &m->inc, inc.data(), inc.size(), st));
  return 0;
}

// Owner-computes decomposition of the single-kernel general iteration
// (kernels_genfused.cuh).  Canonical nodes are cut into contiguous ranges of
// about `own_target` nodes (Morton order keeps a range compact in space);
// a range whose staged elements or local slots exceed the kernel's limits
// is split in halves until it fits.  Every array is ordered deterministically
// (elements and halo / hanging nodes ascending), so the decomposition, and
// with it every summation order, depends on the mesh only.
struct HostBlocks {
  std::vector<GfMeta> meta;
  std::vector<uint8_t> rec;
  std::vector<int32_t> el_id;
  int max_loc = 0, max_own = 0, max_rec16 = 0, max_el = 0;
};
// max_blocks > 0: stop (return 1) as soon as the cut has more ranges.
int make_gen_blocks(const to_mesh_desc *d, const std::vector<int32_t> &node_hang, const std::vector<int64_t> &iptr,
                    const std::vector<uint32_t> &inc, int64_t N, int own_target, int el_max, int loc_max, int own_max,
                    int max_blocks, int ch, HostBlocks &hb, size_t smem_max = 0) {
  const int nc = 1 << d->dim;
  std::vector<int32_t> el_mark(d->n_elem, -1), nd_mark(d->n_node, -1), el_le(d->n_elem, 0), nd_slot(d->n_node, 0);
  int stamp = 0;
  auto elem_of = [&](uint32_t t) { return (int64_t)((t & 0x3fffffffu) / (uint32_t)nc); };
  auto fits = [&](int64_t a, int64_t b) {
    if (b - a > own_max) return false;
    const int sp = ++stamp;
    int64_t nE = 0, nOut = 0;
    for (int64_t n = a; n < b; ++n)
      for (int64_t k = iptr[n]; k < iptr[n + 1]; ++k) {
        const int64_t e = elem_of(inc[k]);
        if (el_mark[e] == sp) continue;
        el_mark[e] = sp;
        ++nE;
        for (int c = 0; c < nc; ++c) {
          const int32_t g = d->elem_node[e * nc + c];
          const int32_t h = node_hang[g];
          if (h < 0) {
            if ((g < a || g >= b) && nd_mark[g] != sp) { nd_mark[g] = sp; ++nOut; }
          } else {
            if (nd_mark[g] != sp) { nd_mark[g] = sp; ++nOut; }
            for (int32_t q = d->hang_ptr[h]; q < d->hang_ptr[h + 1]; ++q) {
              const int32_t pn = d->hang_parent[q];
              if ((pn < a || pn >= b) && nd_mark[pn] != sp) { nd_mark[pn] = sp; ++nOut; }
            }
          }
        }
      }
    if (nE > el_max || (b - a) + nOut > loc_max) return false;
    if (smem_max) {   // k_gen_fused's shared memory for this block alone (halo / virtual ids bounded by 8 bytes)
      const int64_t ninc = iptr[b] - iptr[a];
      const int64_t rec = 2 * gf_pad16((int)(8 * nOut)) + gf_pad16((int)(2 * nc * nE)) +
                          gf_pad16((int)(2 * gf_nchunks((int)nE, ch) * (b - a + 1))) + gf_pad16((int)(2 * ninc));
      const int ys = nc * d->dim + 1;
      const int64_t sm = rec + 8 * ((nE + 1) & ~1) + 8 * (((b - a) + nOut) * d->dim + 2 * (int64_t)own_max * d->dim +
                                                          (int64_t)ch * ys) + 16;
      if ((size_t)sm > smem_max) return false;
    }
    return true;
  };
  std::vector<int32_t> node0;
  {
    std::vector<std::pair<int64_t, int64_t>> todo;
    // block starts are even node ids (3D: 16-byte aligned bulk copies of the owned DOFs)
    const int64_t tgt = (own_target + 1) & ~1;
    for (int64_t a = 0; a < N; a += tgt) todo.push_back({a, std::min<int64_t>(N, a + tgt)});
    std::reverse(todo.begin(), todo.end());
    while (!todo.empty()) {
      auto [a, b] = todo.back();
      todo.pop_back();
      if (fits(a, b)) {
        node0.push_back((int32_t)a);
        if (max_blocks > 0 && (int)node0.size() > max_blocks) return 1;
        continue;
      }
      if (b - a <= 2) { set_error("general-path block of node %lld exceeds the kernel limits", (long long)a); return TO_EINVAL; }
      const int64_t mid = a + ((b - a) / 2 & ~(int64_t)1);
      todo.push_back({mid, b});
      todo.push_back({a, mid});
    }
    node0.push_back((int32_t)N);
  }
  const int nb = (int)node0.size() - 1;
  std::vector<GfMeta> &meta = hb.meta;
  std::vector<uint8_t> &rec = hb.rec;
  std::vector<int32_t> &el_id = hb.el_id;
  meta.assign(nb, GfMeta{});
  rec.clear();
  el_id.clear();
  int &max_loc = hb.max_loc, &max_own = hb.max_own, &max_rec16 = hb.max_rec16, &max_el = hb.max_el;
  max_loc = max_own = max_rec16 = max_el = 0;
  std::vector<int64_t> elems;
  std::vector<int32_t> hl, vt;
  std::vector<uint16_t> iptr_l, inc_l;
  auto put = [&](const void *src, size_t bytes) {
    const size_t at = rec.size();
    rec.resize(at + ((bytes + 15) & ~(size_t)15), 0);
    if (bytes) std::memcpy(rec.data() + at, src, bytes);
  };
  for (int bk = 0; bk < nb; ++bk) {
    const int64_t a = node0[bk], b = node0[bk + 1];
    const int sp = ++stamp;
    elems.clear();
    hl.clear();
    vt.clear();
    for (int64_t n = a; n < b; ++n)
      for (int64_t k = iptr[n]; k < iptr[n + 1]; ++k) {
        const int64_t e = elem_of(inc[k]);
        if (el_mark[e] != sp) { el_mark[e] = sp; elems.push_back(e); }
      }
    std::sort(elems.begin(), elems.end());
    for (size_t i = 0; i < elems.size(); ++i) el_le[elems[i]] = (int32_t)i;
    for (int64_t e : elems)
      for (int c = 0; c < nc; ++c) {
        const int32_t g = d->elem_node[e * nc + c];
        const int32_t h = node_hang[g];
        if (h < 0) {
          if ((g < a || g >= b) && nd_mark[g] != sp) { nd_mark[g] = sp; hl.push_back(g); }
        } else {
          if (nd_mark[g] != sp) { nd_mark[g] = sp; vt.push_back(g); }
          for (int32_t q = d->hang_ptr[h]; q < d->hang_ptr[h + 1]; ++q) {
            const int32_t pn = d->hang_parent[q];
            if ((pn < a || pn >= b) && nd_mark[pn] != sp) { nd_mark[pn] = sp; hl.push_back(pn); }
          }
        }
      }
    std::sort(hl.begin(), hl.end());
    std::sort(vt.begin(), vt.end());
    const int nOwn = (int)(b - a), nHalo = (int)hl.size(), nVirt = (int)vt.size(), nE = (int)elems.size();
    for (int i = 0; i < nHalo; ++i) nd_slot[hl[i]] = nOwn + i;
    for (int i = 0; i < nVirt; ++i) nd_slot[vt[i]] = nOwn + nHalo + i;
    auto slot = [&](int32_t g) { return (g >= a && g < b && node_hang[g] < 0) ? (int)(g - a) : nd_slot[g]; };
    std::vector<ushort4> vrec(nVirt);
    for (int i = 0; i < nVirt; ++i) {
      const int32_t g = vt[i], h = node_hang[g];
      const int np = d->hang_ptr[h + 1] - d->hang_ptr[h];
      if (np != 2 && np != 4) { set_error("hanging node %d has %d parents (2 or 4 expected)", g, np); return TO_EMESH; }
      uint16_t ps[4] = {0xffff, 0xffff, 0xffff, 0xffff};
      for (int q = 0; q < np; ++q) {
        const double w = d->hang_weight[d->hang_ptr[h] + q];
        if (w != 1.0 / np) { set_error("hanging node %d: weight %g with %d parents", g, w, np); return TO_EMESH; }
        ps[q] = (uint16_t)slot(d->hang_parent[d->hang_ptr[h] + q]);
      }
      vrec[i] = make_ushort4(ps[0], ps[1], ps[2], ps[3]);
    }
    std::vector<uint16_t> crec((size_t)nE * nc);
    for (int i = 0; i < nE; ++i)
      for (int c = 0; c < nc; ++c) crec[(size_t)i * nc + c] = (uint16_t)slot(d->elem_node[elems[i] * nc + c]);
    // chunk-major incidence CSR: for each chunk of `ch` elements, each owned
    // node's incidences with that chunk's elements (ascending element order,
    // as the global list), as offsets into the kernel's chunk buffer
    const int nch = gf_nchunks(nE, ch), ys = nc * d->dim + 1;
    if ((ch - 1) * ys + (nc - 1) * d->dim >= (1 << 14)) { set_error("internal: chunk buffer offset range"); return TO_EINVAL; }
    iptr_l.clear();
    inc_l.clear();
    {
      std::vector<std::vector<uint16_t>> by_chunk(nch);
      std::vector<int> cnt((size_t)nch * nOwn, 0);
      for (int64_t n = a; n < b; ++n)
        for (int64_t k = iptr[n]; k < iptr[n + 1]; ++k) {
          const uint32_t t = inc[k];
          const int le = el_le[elem_of(t)];
          const uint32_t c = (t & 0x3fffffffu) % (uint32_t)nc, code = t >> 30;
          const int cix = le / ch;
          by_chunk[cix].push_back((uint16_t)((uint32_t)((le - cix * ch) * ys + (int)c * d->dim) | (code << 14)));
          ++cnt[(size_t)cix * nOwn + (n - a)];
        }
      // by_chunk[c] holds chunk c's entries node by node (nodes ascending,
      // each node's entries ascending): concatenate chunk after chunk
      for (int cix = 0; cix < nch; ++cix) {
        iptr_l.push_back((uint16_t)inc_l.size());
        size_t at = 0;
        for (int o = 0; o < nOwn; ++o) {
          const int c_o = cnt[(size_t)cix * nOwn + o];
          inc_l.insert(inc_l.end(), by_chunk[cix].begin() + at, by_chunk[cix].begin() + at + c_o);
          at += c_o;
          if (inc_l.size() > 0xffff) { set_error("general-path block with more than 65535 incidences"); return TO_EINVAL; }
          iptr_l.push_back((uint16_t)inc_l.size());
        }
      }
    }
    GfMeta &mt = meta[bk];
    mt.node0 = (int32_t)a;
    mt.n_own = nOwn;
    mt.n_halo = nHalo;
    mt.n_virt = nVirt;
    mt.n_el = nE;
    mt.n_inc = (int32_t)inc_l.size();
    mt.el_off = (int32_t)el_id.size();
    mt.rec_off16 = (int32_t)(rec.size() / 16);
    const size_t r0 = rec.size();
    put(hl.data(), 4 * hl.size());
    put(vrec.data(), 8 * vrec.size());
    put(crec.data(), 2 * crec.size());
    put(iptr_l.data(), 2 * iptr_l.size());
    put(inc_l.data(), 2 * inc_l.size());
    const GfSections sec = d->dim == 3 ? gf_sections<3>(nOwn, nHalo, nVirt, nE, mt.n_inc, ch)
                                       : gf_sections<2>(nOwn, nHalo, nVirt, nE, mt.n_inc, ch);
    if ((size_t)sec.total != rec.size() - r0) { set_error("internal: block record layout"); return TO_EINVAL; }
    for (int64_t e : elems) el_id.push_back((int32_t)e);
    if (nE & 1) el_id.push_back(-1);   // every block's s_e starts 16-byte aligned
    max_loc = std::max(max_loc, nOwn + nHalo + nVirt);
    max_own = std::max(max_own, nOwn);
    max_rec16 = std::max(max_rec16, sec.total / 16);
    max_el = std::max(max_el, nE);
  }
  if (rec.size() / 16 >= (size_t)INT32_MAX || el_id.size() >= (size_t)INT32_MAX) { set_error("mesh too large for the general-path records"); return TO_EINVAL; }
  return 0;
}

// Device copies of a decomposition; s_loc (s_e in block-local order, filled
// per solve by k_gather_s) allocated to match.
int upload_gen_blocks(to_mesh *m, const HostBlocks &hb, GenBlocks &B, int32_t **el_id, int64_t *n_loc_el,
                      double **s_loc, cudaStream_t st) {
  B.n_blk = (int)hb.meta.size();
  B.max_loc = hb.max_loc;
  B.max_own = hb.max_own;
  B.max_rec16 = hb.max_rec16;
  B.max_el = hb.max_el;
  GfMeta *dmeta;
  uint4 *drec;
  RC(upload_array(m, &dmeta, hb.meta.data(), hb.meta.size(), st));
  RC(upload_array(m, &drec, reinterpret_cast<const uint4 *>(hb.rec.data()), hb.rec.size() / 16, st));
  RC(upload_array(m, el_id, hb.el_id.data(), hb.el_id.size(), st));
  B.meta = dmeta;
  B.rec = drec;
  *n_loc_el = (int64_t)hb.el_id.size();
  RC(m->alloc(s_loc, (size_t)std::max<int64_t>(2, *n_loc_el)));
  return 0;
}

// the attribute is per function, not per handle: allow the device's opt-in
// maximum (less the kernel's static shared memory) so that a later upload of
// a smaller mesh cannot lower it below what an earlier handle launches with
int allow_smem(to_mesh *m, const void *fn, size_t need) {
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, m->device));
  cudaFuncAttributes fa{};
  CK(cudaFuncGetAttributes(&fa, fn));
  const int dyn = optin - (int)fa.sharedSizeBytes;
  if (need > (size_t)dyn) { set_error("general-path blocks need %zu bytes of shared memory", need); return TO_EINVAL; }
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
  return 0;
}

int build_gen_blocks(const to_mesh_desc *d, const std::vector<int32_t> &node_hang, const std::vector<int64_t> &iptr,
                     const std::vector<uint32_t> &inc, cudaStream_t st, to_mesh *m) {
  const int nc = 1 << d->dim;
  const int64_t N = m->n_owned;   // blocks cover the owned nodes (all, unless a shard's local mesh)
  // mid-size 3D meshes get smaller blocks, about two per SM slot pair (a
  // grid that fills the GPU beats the lower halo overhead of big blocks:
  // 6k / 12k-element octree meshes 16.8 / 17.2 -> 12.1 / 13.9 us per
  // iteration; c4 unchanged; in 2D it lost, c2 9.0 -> 10.0, so 2D keeps its
  // target; profiles/r2/general_midsize_ab.txt)
  const int own_target = d->dim == 3 ? (int)std::max<int64_t>(kGfOwnMin, std::min<int64_t>(kGfOwnTarget3,
                                                                                           N / (2 * kNumSMs)))
                                     : kGfOwnTarget2;
  // (incidence encoding: le * 2^dim < 2^14)
  HostBlocks hb;
  // the kernel's shared memory is the sum of per-section maxima over the
  // blocks (from different blocks), so the per-block cap is tightened until
  // the total fits as well
  size_t cap = (size_t)TOMESH_GF_SMEMMAX;
  for (int attempt = 0;; ++attempt) {
    RC(make_gen_blocks(d, node_hang, iptr, inc, N, own_target, std::min(kGfElMax, (1 << 14) / nc - 1), kGfMaxLoc,
                       std::min(kGfMaxOwn, (own_target + 1) & ~1), 0, d->dim == 3 ? GfChunk<3>::CH : GfChunk<2>::CH,
                       hb, cap));
    const size_t tot = d->dim == 3 ? gf_smem_bytes<3>(hb.max_rec16, hb.max_el, hb.max_loc, hb.max_own)
                                   : gf_smem_bytes<2>(hb.max_rec16, hb.max_el, hb.max_loc, hb.max_own);
    if (!cap || tot <= (size_t)TOMESH_GF_SMEMMAX || attempt == 4) break;
    cap -= std::min(cap / 2, tot - (size_t)TOMESH_GF_SMEMMAX + 1024);
  }
  GenBlocks &B = m->GB;
  RC(upload_gen_blocks(m, hb, B, &m->gb_el_id, &m->gb_n_loc_el, &m->s_loc, st));
  const int nb = B.n_blk;
  m->gb_smem = d->dim == 3 ? gf_smem_bytes<3>(B.max_rec16, B.max_el, B.max_loc, B.max_own)
                           : gf_smem_bytes<2>(B.max_rec16, B.max_el, B.max_loc, B.max_own);
  if (d->dim == 3) {
    RC(allow_smem(m, (const void *)k_gen_fused<3, G_CG>, m->gb_smem));
    RC(allow_smem(m, (const void *)k_gen_fused<3, G_PLAIN>, m->gb_smem));
    RC(allow_smem(m, (const void *)k_gen_persist<3>, m->gb_smem));
  } else {
    RC(allow_smem(m, (const void *)k_gen_fused<2, G_CG>, m->gb_smem));
    RC(allow_smem(m, (const void *)k_gen_fused<2, G_PLAIN>, m->gb_smem));
    RC(allow_smem(m, (const void *)k_gen_persist<2>, m->gb_smem));
  }
  // next-wave L2 prefetch distance: the CTAs resident at once (a block's
  // successor in its SM slot is about one full residency later).  Only when
  // what one iteration streams (records, s_e, the owned r, q, p, Dinv, x)
  // exceeds the L2: an L2-resident mesh gains nothing (c4: 47.2 -> 48.1 us
  // with it, c4L: 256-265 -> 241; profiles/r2/general_l2prefetch_ab.txt).  A size rule, not a
  // timing: the prefetch is a cache fill and never changes a result.
  B.pf = 0;
#if TOMESH_GF_PF
  int l2 = 0;
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, m->device));
  const size_t streamed = hb.rec.size() + 8 * (size_t)m->gb_n_loc_el + 5 * 8 * (size_t)m->n_owned * d->dim;
  if (streamed > (size_t)l2) {
    int per_sm = 0;
    const void *fn = d->dim == 3 ? (const void *)k_gen_fused<3, G_CG> : (const void *)k_gen_fused<2, G_CG>;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kGfThreads, m->gb_smem));
    if (per_sm > 0 && (int64_t)per_sm * kNumSMs * TOMESH_GF_PF < nb) B.pf = per_sm * kNumSMs * TOMESH_GF_PF;
  }
#endif
  RC(ensure_partials(m, (size_t)nb * 10));   // dots of two launches (parity)
  m->gb_local_el = m->gb_local_nodes = 0;
  for (const GfMeta &mt : hb.meta) {
    m->gb_local_el += mt.n_el;
    m->gb_local_nodes += mt.n_own + mt.n_halo + mt.n_virt;
  }
  m->gen_fused = true;
  return 0;
}

// Element-partitioned decomposition (kernels_genep.cuh): node ranges as in
// build_gen_blocks; element e is assigned to the block owning its smallest
// contributed node (non-hanging corner or parent of a hanging corner); node
// n's operator output is the sum of one partial per contributor block, in
// ascending block order (slot_ptr[n] .. slot_ptr[n+1]).  Deterministic: every
// list is built in ascending order from the mesh alone.
int build_gen_ep(const to_mesh_desc *d, const std::vector<int32_t> &node_hang, cudaStream_t st, to_mesh *m) {
  const int nc = 1 << d->dim, dim = d->dim;
  const int64_t N = d->n_node, E = d->n_elem;
  const int ch = dim == 3 ? GfChunk<3>::CH : GfChunk<2>::CH, ys = nc * dim + 1;
  if (N >= INT32_MAX / 8) { set_error("mesh too large for the element-partitioned path"); return TO_EINVAL; }
  auto code = [](double w) -> uint32_t { return w == 1.0 ? 0u : w == 0.5 ? 1u : 2u; };
  // smallest contributed node of every element; elements bucketed by it
  std::vector<int32_t> emin(E);
  for (int64_t e = 0; e < E; ++e) {
    int32_t mn = INT32_MAX;
    for (int c = 0; c < nc; ++c) {
      const int32_t g = d->elem_node[e * nc + c], h = node_hang[g];
      if (h < 0) mn = std::min(mn, g);
      else
        for (int32_t q = d->hang_ptr[h]; q < d->hang_ptr[h + 1]; ++q) mn = std::min(mn, d->hang_parent[q]);
    }
    emin[e] = mn;
  }
  std::vector<int64_t> bptr(N + 1, 0);
  for (int64_t e = 0; e < E; ++e) bptr[emin[e] + 1]++;
  for (int64_t n = 0; n < N; ++n) bptr[n + 1] += bptr[n];
  std::vector<int32_t> bel(E);
  {
    std::vector<int64_t> f(bptr.begin(), bptr.end() - 1);
    for (int64_t e = 0; e < E; ++e) bel[f[emin[e]]++] = (int32_t)e;
  }
  std::vector<int32_t> mark(N, -1), hmark(N, -1);
  int stamp = 0;
  // local node counts of a candidate range [a, b)
  struct Cnt { int64_t nE, nHalo, nVirt, nInc; };
  auto count = [&](int64_t a, int64_t b) {
    const int sp = ++stamp;
    Cnt c{bptr[b] - bptr[a], 0, 0, 0};
    for (int64_t k = bptr[a]; k < bptr[b]; ++k) {
      const int64_t e = bel[k];
      for (int cc = 0; cc < nc; ++cc) {
        const int32_t g = d->elem_node[e * nc + cc], h = node_hang[g];
        if (h < 0) {
          ++c.nInc;
          if ((g < a || g >= b) && mark[g] != sp) { mark[g] = sp; ++c.nHalo; }
        } else {
          if (hmark[g] != sp) { hmark[g] = sp; ++c.nVirt; }
          for (int32_t q = d->hang_ptr[h]; q < d->hang_ptr[h + 1]; ++q) {
            const int32_t pn = d->hang_parent[q];
            ++c.nInc;
            if ((pn < a || pn >= b) && mark[pn] != sp) { mark[pn] = sp; ++c.nHalo; }
          }
        }
      }
    }
    return c;
  };
  const size_t cap = (size_t)TOMESH_GF_SMEMMAX;
  auto fits = [&](int64_t a, int64_t b) {
    const Cnt c = count(a, b);
    const int64_t nOwn = b - a, nAcc = nOwn + c.nHalo, nLoc = nAcc + c.nVirt;
    if (nOwn > kGfMaxOwn || nAcc > kEpMaxAcc || nLoc > kGfMaxLoc || c.nE > kGfElMax || c.nInc > 0xffff) return false;
    const int64_t rec = gf_pad16((int)(4 * c.nHalo)) + gf_pad16((int)(8 * c.nVirt)) + gf_pad16((int)(2 * nc * c.nE)) +
                        gf_pad16((int)(2 * gf_nchunks((int)c.nE, ch) * (nAcc + 1))) + gf_pad16((int)(2 * c.nInc)) +
                        gf_pad16((int)(4 * nAcc)) + gf_pad16((int)(4 * c.nHalo)) + gf_pad16((int)c.nHalo);
    const size_t sm = (size_t)rec + 8 * (size_t)((c.nE + 1) & ~1) + 8 * ((size_t)nLoc * dim + (size_t)ch * ys) + 16;
    return sm <= cap;
  };
  const int own_target = dim == 3 ? TOMESH_EP_OWN3 : TOMESH_EP_OWN2;
  std::vector<int32_t> node0;
  {
    std::vector<std::pair<int64_t, int64_t>> todo;
    const int64_t tgt = (own_target + 1) & ~1;
    for (int64_t a = 0; a < N; a += tgt) todo.push_back({a, std::min<int64_t>(N, a + tgt)});
    std::reverse(todo.begin(), todo.end());
    while (!todo.empty()) {
      auto [a, b] = todo.back();
      todo.pop_back();
      if (fits(a, b)) { node0.push_back((int32_t)a); continue; }
      if (b - a <= 2) { set_error("element-partitioned block of node %lld exceeds the kernel limits", (long long)a); return TO_EINVAL; }
      const int64_t mid = a + ((b - a) / 2 & ~(int64_t)1);
      todo.push_back({mid, b});
      todo.push_back({a, mid});
    }
    node0.push_back((int32_t)N);
  }
  const int nb = (int)node0.size() - 1;
  // contributors per node (ascending block): counts, then slot pointers
  std::vector<int32_t> lastb(N, -1);
  std::vector<int64_t> sptr(N + 1, 0);
  auto for_contrib = [&](int64_t e, auto f) {
    for (int cc = 0; cc < nc; ++cc) {
      const int32_t g = d->elem_node[e * nc + cc], h = node_hang[g];
      if (h < 0) f(g);
      else
        for (int32_t q = d->hang_ptr[h]; q < d->hang_ptr[h + 1]; ++q) f(d->hang_parent[q]);
    }
  };
  for (int b = 0; b < nb; ++b)
    for (int64_t k = bptr[node0[b]]; k < bptr[node0[b + 1]]; ++k)
      for_contrib(bel[k], [&](int32_t g) {
        if (lastb[g] != b) { lastb[g] = b; sptr[g + 1]++; }
      });
  for (int64_t n = 0; n < N; ++n) {
    if (sptr[n + 1] > 255) { set_error("node %lld has more than 255 contributor blocks", (long long)n); return TO_EINVAL; }
    sptr[n + 1] += sptr[n];
  }
  const int64_t n_slots = sptr[N];
  if (n_slots * dim >= INT32_MAX) { set_error("too many slots for the element-partitioned path"); return TO_EINVAL; }
  std::vector<int64_t> sfill(sptr.begin(), sptr.end() - 1);
  std::vector<GfMeta> meta(nb);
  std::vector<uint8_t> rec;
  std::vector<int32_t> el_id;
  int max_loc = 0, max_rec16 = 0, max_el = 0;
  int64_t loc_el = 0, loc_nodes = 0;
  std::vector<int32_t> slot_of(N, 0);
  auto put = [&](const void *src, size_t bytes) {
    const size_t at = rec.size();
    rec.resize(at + ((bytes + 15) & ~(size_t)15), 0);
    if (bytes) std::memcpy(rec.data() + at, src, bytes);
  };
  std::vector<int32_t> elems, hl, vt;
  for (int bk = 0; bk < nb; ++bk) {
    const int64_t a = node0[bk], b = node0[bk + 1];
    const int sp = ++stamp;
    elems.assign(bel.begin() + bptr[a], bel.begin() + bptr[b]);
    std::sort(elems.begin(), elems.end());
    hl.clear();
    vt.clear();
    for (int32_t e : elems)
      for (int cc = 0; cc < nc; ++cc) {
        const int32_t g = d->elem_node[(int64_t)e * nc + cc], h = node_hang[g];
        if (h < 0) {
          if ((g < a || g >= b) && mark[g] != sp) { mark[g] = sp; hl.push_back(g); }
        } else {
          if (hmark[g] != sp) { hmark[g] = sp; vt.push_back(g); }
          for (int32_t q = d->hang_ptr[h]; q < d->hang_ptr[h + 1]; ++q) {
            const int32_t pn = d->hang_parent[q];
            if ((pn < a || pn >= b) && mark[pn] != sp) { mark[pn] = sp; hl.push_back(pn); }
          }
        }
      }
    std::sort(hl.begin(), hl.end());
    std::sort(vt.begin(), vt.end());
    const int nOwn = (int)(b - a), nHalo = (int)hl.size(), nVirt = (int)vt.size(), nE = (int)elems.size();
    const int nAcc = nOwn + nHalo;
    for (int i = 0; i < nHalo; ++i) slot_of[hl[i]] = nOwn + i;
    for (int i = 0; i < nVirt; ++i) slot_of[vt[i]] = nAcc + i;
    auto slot = [&](int32_t g) { return (g >= a && g < b && node_hang[g] < 0) ? (int)(g - a) : slot_of[g]; };
    std::vector<ushort4> vrec(nVirt);
    for (int i = 0; i < nVirt; ++i) {
      const int32_t g = vt[i], h = node_hang[g];
      const int np = d->hang_ptr[h + 1] - d->hang_ptr[h];
      if (np != 2 && np != 4) { set_error("hanging node %d has %d parents (2 or 4 expected)", g, np); return TO_EMESH; }
      uint16_t ps[4] = {0xffff, 0xffff, 0xffff, 0xffff};
      for (int q = 0; q < np; ++q) {
        const double w = d->hang_weight[d->hang_ptr[h] + q];
        if (w != 1.0 / np) { set_error("hanging node %d: weight %g with %d parents", g, w, np); return TO_EMESH; }
        ps[q] = (uint16_t)slot(d->hang_parent[d->hang_ptr[h] + q]);
      }
      vrec[i] = make_ushort4(ps[0], ps[1], ps[2], ps[3]);
    }
    std::vector<uint16_t> crec((size_t)nE * nc);
    // incidences grouped by (chunk, local accumulating node), in (element, corner, parent) order
    const int nch = gf_nchunks(nE, ch);
    std::vector<std::vector<uint16_t>> lists((size_t)nch * nAcc);
    std::vector<uint32_t> wslot(nAcc, 0xffffffffu);
    for (int le = 0; le < nE; ++le) {
      const int64_t e = elems[le];
      const int cix = le / ch;
      for (int cc = 0; cc < nc; ++cc) {
        const int32_t g = d->elem_node[e * nc + cc], h = node_hang[g];
        crec[(size_t)le * nc + cc] = (uint16_t)slot(g);
        const uint32_t off = (uint32_t)((le - cix * ch) * ys + cc * dim);
        auto add = [&](int32_t t, uint32_t cd) {
          const int l = slot(t);
          lists[(size_t)cix * nAcc + l].push_back((uint16_t)(off | (cd << 14)));
          if (wslot[l] == 0xffffffffu) wslot[l] = (uint32_t)(sfill[t]++);
        };
        if (h < 0) add(g, 0u);
        else
          for (int32_t q = d->hang_ptr[h]; q < d->hang_ptr[h + 1]; ++q)
            add(d->hang_parent[q], code(d->hang_weight[q]));
      }
    }
    std::vector<uint16_t> iptr_l, inc_l;
    for (int cix = 0; cix < nch; ++cix) {
      iptr_l.push_back((uint16_t)inc_l.size());
      for (int l = 0; l < nAcc; ++l) {
        const auto &L = lists[(size_t)cix * nAcc + l];
        inc_l.insert(inc_l.end(), L.begin(), L.end());
        if (inc_l.size() > 0xffff) { set_error("element-partitioned block with more than 65535 incidences"); return TO_EINVAL; }
        iptr_l.push_back((uint16_t)inc_l.size());
      }
    }
    std::vector<uint32_t> hslot(nHalo);
    std::vector<uint8_t> hcnt(nHalo);
    for (int i = 0; i < nHalo; ++i) {
      hslot[i] = (uint32_t)sptr[hl[i]];
      hcnt[i] = (uint8_t)(sptr[hl[i] + 1] - sptr[hl[i]]);
    }
    GfMeta &mt = meta[bk];
    mt.node0 = (int32_t)a;
    mt.n_own = nOwn;
    mt.n_halo = nHalo;
    mt.n_virt = nVirt;
    mt.n_el = nE;
    mt.n_inc = (int32_t)inc_l.size();
    mt.el_off = (int32_t)el_id.size();
    mt.rec_off16 = (int32_t)(rec.size() / 16);
    const size_t r0 = rec.size();
    put(hl.data(), 4 * hl.size());
    put(vrec.data(), 8 * vrec.size());
    put(crec.data(), 2 * crec.size());
    put(iptr_l.data(), 2 * iptr_l.size());
    put(inc_l.data(), 2 * inc_l.size());
    put(wslot.data(), 4 * wslot.size());
    put(hslot.data(), 4 * hslot.size());
    put(hcnt.data(), hcnt.size());
    const EpSections sec = ep_sections(dim, nOwn, nHalo, nVirt, nE, mt.n_inc, ch);
    if ((size_t)sec.total != rec.size() - r0) { set_error("internal: element-partitioned record layout"); return TO_EINVAL; }
    for (int32_t e : elems) el_id.push_back(e);
    if (nE & 1) el_id.push_back(-1);
    max_loc = std::max(max_loc, nAcc + nVirt);
    max_rec16 = std::max(max_rec16, sec.total / 16);
    max_el = std::max(max_el, nE);
    loc_el += nE;
    loc_nodes += nAcc + nVirt;
  }
  for (int64_t n = 0; n < N; ++n)
    if (sfill[n] != sptr[n + 1]) { set_error("internal: element-partitioned slot count"); return TO_EINVAL; }
  if (rec.size() / 16 >= (size_t)INT32_MAX) { set_error("mesh too large for the element-partitioned records"); return TO_EINVAL; }
  GenBlocks &B = m->EB;
  B.n_blk = nb;
  B.max_loc = max_loc;
  B.max_own = kGfMaxOwn;
  B.max_rec16 = max_rec16;
  B.max_el = max_el;
  GfMeta *dmeta;
  uint4 *drec;
  RC(upload_array(m, &dmeta, meta.data(), meta.size(), st));
  RC(upload_array(m, &drec, reinterpret_cast<const uint4 *>(rec.data()), rec.size() / 16, st));
  RC(upload_array(m, &m->ep_el_id, el_id.data(), el_id.size(), st));
  B.meta = dmeta;
  B.rec = drec;
  m->ep_n_loc_el = (int64_t)el_id.size();
  RC(m->alloc(&m->ep_s_loc, (size_t)std::max<int64_t>(2, m->ep_n_loc_el)));
  std::vector<int32_t> sp32(sptr.begin(), sptr.end());
  RC(upload_array(m, &m->ep_slot_ptr, sp32.data(), sp32.size(), st));
  for (int k = 0; k < 2; ++k) {
    RC(m->alloc(&m->ep_W[k], (size_t)std::max<int64_t>(1, n_slots * dim)));
    CK(cudaMemsetAsync(m->ep_W[k], 0, sizeof(double) * (size_t)std::max<int64_t>(1, n_slots * dim), st));
  }
  m->ep_smem = dim == 3 ? ep_smem_bytes<3>(max_rec16, max_el, max_loc) : ep_smem_bytes<2>(max_rec16, max_el, max_loc);
  RC(allow_smem(m, dim == 3 ? (const void *)k_gen_ep<3> : (const void *)k_gen_ep<2>, m->ep_smem));
  RC(ensure_partials(m, (size_t)nb * 5));
  m->ep_n_slots = n_slots;
  RC(m->alloc(&m->ep_w, (size_t)std::max<int64_t>(1, m->n_dof)));
  m->ep_local_el = loc_el;
  m->ep_local_nodes = loc_nodes;
  m->gen_ep = true;
  return 0;
}

const void *gc_kernel(int dim, int T) {
  if (dim == 2) return T == 128 ? (const void *)k_gen_cluster<2, 128> : T == 256 ? (const void *)k_gen_cluster<2, 256>
                                                                              : (const void *)k_gen_cluster<2, 512>;
  return T == 128 ? (const void *)k_gen_cluster<3, 128> : T == 256 ? (const void *)k_gen_cluster<3, 256>
                                                                   : (const void *)k_gen_cluster<3, 512>;
}
size_t gc_smem(int dim, int T, const HostBlocks &hb, int max_halo, int max_send) {
  auto f = [&](auto lay) { return lay(hb.max_rec16, hb.max_el, hb.max_loc, hb.max_own, max_halo, max_send).total; };
  if (dim == 2) return T == 128 ? f(gc_layout<2, 128>) : T == 256 ? f(gc_layout<2, 256>) : f(gc_layout<2, 512>);
  return T == 128 ? f(gc_layout<3, 128>) : T == 256 ? f(gc_layout<3, 256>) : f(gc_layout<3, 512>);
}

// Small meshes: a second decomposition into at most kGcMaxBlocks blocks for
// the cluster-resident solver (kernels_gencluster.cuh), if one cluster of
// that many CTAs with the state of its owned nodes in shared memory fits
// (shared memory, and a cluster placement the device reports possible).
// Leaves m->gen_cluster false otherwise.
int build_gen_cluster(const to_mesh_desc *d, const std::vector<int32_t> &node_hang, const std::vector<int64_t> &iptr,
                      const std::vector<uint32_t> &inc, cudaStream_t st, to_mesh *m) {
  const int nc = 1 << d->dim;
  const int64_t N = m->n_owned;
  if (N > (int64_t)kGcMaxBlocks * kGcMaxOwn) return 0;
  const int64_t nb_t = std::min<int64_t>(kGcMaxBlocks, std::max<int64_t>(1, (N + kGcOwnMin - 1) / kGcOwnMin));
  const int own_target = (int)((N + nb_t - 1) / nb_t);
  // 2 T >= the target; beyond 512 owned nodes per CTA (T = 512) one kernel
  // per iteration over the whole GPU is faster (c2: 1,184 nodes per CTA,
  // 10.7 us per iteration in the cluster against 8.6 launched)
  if (own_target > kGcOwnMaxTarget) return 0;
  const int T = own_target <= 256 ? 128 : own_target <= 512 ? 256 : 512;
  HostBlocks hb;
  const int rc = make_gen_blocks(d, node_hang, iptr, inc, N, own_target, (1 << 14) / nc - 1, 0xfffe,
                                 kGcOwnPerThread * T, kGcMaxBlocks,
                                 d->dim == 3 ? (T == 512 ? GcChunk<3, 512>::CH : T == 256 ? GcChunk<3, 256>::CH : GcChunk<3, 128>::CH)
                                             : (T == 512 ? GcChunk<2, 512>::CH : T == 256 ? GcChunk<2, 256>::CH : GcChunk<2, 128>::CH),
                                 hb);
  if (rc == 1) return 0;     // the limits split it into more blocks than one cluster holds
  RC(rc);
  // send lists: for every halo node of block b (index i in b's halo list), an
  // entry in its owner's list; each list sorted by (destination, index)
  const int nbk = (int)hb.meta.size();
  std::vector<std::vector<uint32_t>> lists(nbk);
  int max_halo = 0;
  for (int b = 0; b < nbk; ++b) {
    const GfMeta &mb = hb.meta[b];
    max_halo = std::max(max_halo, mb.n_halo);
    const int32_t *hl = reinterpret_cast<const int32_t *>(hb.rec.data() + (size_t)16 * mb.rec_off16);   // section 0
    for (int i = 0; i < mb.n_halo; ++i) {
      const int32_t g = hl[i];
      int o = 0;
      while (o + 1 < nbk && hb.meta[o + 1].node0 <= g) ++o;
      const int src = g - hb.meta[o].node0;
      if (o == b || src < 0 || src >= hb.meta[o].n_own || src > 0xfff || i > 0x7fff) {
        set_error("internal: cluster send list (block %d, halo %d)", b, i);
        return TO_EINVAL;
      }
      lists[o].push_back((uint32_t)src | ((uint32_t)i << 12) | ((uint32_t)b << 27));
    }
  }
  std::vector<uint32_t> ent;
  std::vector<int32_t> off(1, 0);
  int max_send = 0;
  for (int o = 0; o < nbk; ++o) {
    std::sort(lists[o].begin(), lists[o].end(), [](uint32_t a, uint32_t b) {
      return (a >> 27) != (b >> 27) ? (a >> 27) < (b >> 27) : ((a >> 12) & 0x7fff) < ((b >> 12) & 0x7fff);
    });
    ent.insert(ent.end(), lists[o].begin(), lists[o].end());
    off.push_back((int32_t)ent.size());
    max_send = std::max(max_send, (int)lists[o].size());
  }
  const size_t smem = gc_smem(d->dim, T, hb, max_halo, max_send);
  const void *fn = gc_kernel(d->dim, T);
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, m->device));
  cudaFuncAttributes fa{};
  CK(cudaFuncGetAttributes(&fa, fn));
  if (smem > (size_t)(optin - (int)fa.sharedSizeBytes)) return 0;
  RC(allow_smem(m, fn, smem));
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  const int nb = (int)hb.meta.size();
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)nb;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(nb);
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclu = 0;
  if (cudaOccupancyMaxActiveClusters(&nclu, fn, &cfg) != cudaSuccess || nclu < 1) {
    (void)cudaGetLastError();
    return 0;
  }
  RC(upload_gen_blocks(m, hb, m->GC, &m->gc_el_id, &m->gc_n_loc_el, &m->gc_s_loc, st));
  uint32_t *dent;
  int32_t *doff;
  if (ent.empty()) ent.push_back(0u);   // (a single-block cluster sends nothing)
  RC(upload_array(m, &dent, ent.data(), ent.size(), st));
  RC(upload_array(m, &doff, off.data(), off.size(), st));
  m->GCS = GcSend{dent, doff, max_halo, max_send};
  m->gc_smem = smem;
  m->gc_threads = T;
  m->gen_cluster = true;
  return 0;
}

int do_upload(const to_mesh_desc *d, int device, cudaStream_t st, to_mesh *m) {
  CK(cudaSetDevice(device));
  m->device = device;
  m->dim = d->dim;
  m->L = d->max_level;
  {
    const double hL = d->h0 / (double)(1 << d->max_level);
    double vt = 0.0;   // sum of exact dyadic element volumes (C1)
    for (int64_t e = 0; e < d->n_elem; ++e) {
      const double hs = std::ldexp(hL, d->max_level - d->elem_level[e]);
      vt += d->dim == 2 ? hs * hs : hs * hs * hs;
    }
    m->vol_total = vt;
  }
  m->h0 = d->h0;
  m->hL = d->h0 / (double)(1 << d->max_level);
  m->E0 = d->E0;
  m->Emin = d->Emin;
  m->nu = d->nu;
  m->rmin = d->rmin;
  m->n_el = d->n_elem;
  m->n_node = d->n_node;
  m->n_dof = d->n_node * d->dim;
  m->n_hang = d->n_hang;
  m->n_fixed = d->n_fixed;
  m->filt_nnz = d->rmin > 0.0 ? d->filt_nnz : 0;
  const int dim = d->dim, nc = 1 << dim;

  // host-derived encodings
  std::vector<int32_t> node_hang(m->n_node, -1);
  for (int64_t h = 0; h < d->n_hang; ++h) node_hang[d->hang_node[h]] = (int32_t)h;
  std::vector<uint8_t> free_dof(m->n_dof, 1);
  for (int64_t h = 0; h < d->n_hang; ++h)
    for (int c = 0; c < dim; ++c) free_dof[(int64_t)d->hang_node[h] * dim + c] = 0;
  for (int64_t i = 0; i < d->n_fixed; ++i) free_dof[d->fixed_dof[i]] = 0;
  // parent -> hanging children (transpose of P), children ascending
  std::vector<int32_t> cptr(m->n_node + 1, 0), chang, ccount(m->n_node, 0);
  std::vector<double> cw;
  if (d->n_hang > 0) {
    for (int64_t h = 0; h < d->n_hang; ++h)
      for (int32_t k = d->hang_ptr[h]; k < d->hang_ptr[h + 1]; ++k) cptr[d->hang_parent[k] + 1]++;
    for (int64_t n = 0; n < m->n_node; ++n) cptr[n + 1] += cptr[n];
    chang.resize(cptr[m->n_node]);
    cw.resize(cptr[m->n_node]);
    for (int64_t h = 0; h < d->n_hang; ++h)
      for (int32_t k = d->hang_ptr[h]; k < d->hang_ptr[h + 1]; ++k) {
        int32_t p = d->hang_parent[k];
        int32_t pos = cptr[p] + ccount[p]++;
        chang[pos] = d->hang_node[h];
        cw[pos] = d->hang_weight[k];
      }
  }

  RC(upload_array(m, &m->elem_node, d->elem_node, (size_t)m->n_el * nc, st));
  RC(upload_array(m, &m->elem_anchor, d->elem_anchor, (size_t)m->n_el * dim, st));
  RC(upload_array(m, &m->elem_level, d->elem_level, (size_t)m->n_el, st));
  RC(upload_array(m, &m->node_hang, node_hang.data(), node_hang.size(), st));
  RC(upload_array(m, &m->free_dof, free_dof.data(), free_dof.size(), st));
  RC(upload_array(m, &m->load, d->load, (size_t)m->n_dof, st));
  if (d->n_hang > 0) {
    const size_t nnz = (size_t)d->hang_ptr[d->n_hang];
    RC(upload_array(m, &m->hang_ptr, d->hang_ptr, (size_t)d->n_hang + 1, st));
    RC(upload_array(m, &m->hang_parent, d->hang_parent, nnz, st));
    RC(upload_array(m, &m->hang_weight, d->hang_weight, nnz, st));
    RC(upload_array(m, &m->child_ptr, cptr.data(), cptr.size(), st));
    RC(upload_array(m, &m->child_hang, chang.data(), chang.size(), st));
    RC(upload_array(m, &m->child_weight, cw.data(), cw.size(), st));
  }

  RC(ensure_partials(m, (size_t)kMaxPartialBlocks * 4));
  RC(m->alloc(&m->S, 1));
  CK(cudaMemsetAsync(m->S, 0, sizeof(CgScalars), st));
  CK(cudaMallocHost(&m->S_host, sizeof(CgScalars)));
  CK(cudaEventCreate(&m->ev0));
  CK(cudaEventCreate(&m->ev1));
  // element matrices (closed form, element.cpp)
  build_K0(2, d->nu, m->K2.K);
  build_K0(3, d->nu, m->K3.K);
  if (build_K0_hadamard(d->nu, &m->KH) != 0) { set_error("Hadamard factorisation check failed"); return TO_EINVAL; }
  if (build_K0_hadamard_sym(m->KH, &m->KS) != 0) { set_error("Hadamard coefficient classes check failed"); return TO_EINVAL; }
  m->n_int = m->n_dof;
  // TO_UPLOAD_GENERAL keeps uniform H8 meshes on the general path
  m->force_general = (d->options & TO_UPLOAD_GENERAL) != 0 || d->n_owned > 0;
  m->n_owned = d->n_owned > 0 ? d->n_owned : d->n_node;
  RC(setup_structured(d, free_dof, st, m));
  // (the structured path filters with a lattice stencil and needs no lists)
  if ((m->filt_nnz > 0 || d->rmin > 0.0) && !m->structured) {
    RC(upload_array(m, &m->filt_ptr, d->filt_ptr, (size_t)m->n_el + 1, st));
    RC(upload_array(m, &m->filt_idx, d->filt_idx, (size_t)std::max<int64_t>(1, m->filt_nnz), st));
  }
  if (d->rmin > 0.0 && m->structured) {
    const double h = m->h_struct, r2 = d->rmin * d->rmin, V = h * h * h;
    const int R = (int)std::ceil(d->rmin / h) + 1;
    std::vector<S3FilterOffset> offs;
    for (int dk = -R; dk <= R; ++dk)
      for (int dj = -R; dj <= R; ++dj)
        for (int di = -R; di <= R; ++di) {
          const double d2 = (double)(di * di + dj * dj + dk * dk) * h * h;   // exact: integer times h^2
          if (d2 < r2) offs.push_back({di, dj, dk, (d->rmin - std::sqrt(d2)) * V});
        }
    m->n_foffs = (int)offs.size();
    RC(upload_array(m, &m->foffs, offs.data(), offs.size(), st));
    RC(m->alloc(&m->ftmp, (size_t)m->n_el));
  }
  if (!m->structured) {
    std::vector<int64_t> iptr;
    std::vector<uint32_t> incv;
    RC(setup_incidence(d, node_hang, st, m, iptr, incv));
    RC(build_gen_blocks(d, node_hang, iptr, incv, st, m));
    // large meshes (the launched path with a step kernel): the element-
    // partitioned iteration (kernels_genep.cuh), unless TO_UPLOAD_NO_EP or a
    // shard's local mesh; TO_UPLOAD_EP forces it
    const bool ep_auto = TOMESH_EP_AUTO && m->GB.n_blk > kGfStepInMaxBlocks;
    if (d->n_owned == 0 && !(d->options & TO_UPLOAD_NO_EP) && ((d->options & TO_UPLOAD_EP) || ep_auto))
      RC(build_gen_ep(d, node_hang, st, m));
    // the smallest meshes: one thread-block cluster holds the whole solve
    // (k_gen_cluster), unless TO_UPLOAD_LAUNCHED / NO_CLUSTER or a shard's local mesh
    if (!(d->options & (TO_UPLOAD_LAUNCHED | TO_UPLOAD_NO_CLUSTER)) && d->n_owned == 0 && !m->gen_ep)
      RC(build_gen_cluster(d, node_hang, iptr, incv, st, m));
    // small meshes (at most kGfPersistMaxBlocks blocks): the whole loop in one
    // cooperative kernel, unless TO_UPLOAD_LAUNCHED.  Measured: c1 (6 blocks)
    // 5.8 vs 6.9 us per iteration launched; c2 (85 blocks) 13.8 vs 9.0 -- the
    // grid barrier and the partial sums in every block cost more than the two
    // PDL-chained launches once there are more than a few dozen blocks
    int coop = 0;
    CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
    if (coop && !m->gen_cluster && !m->gen_ep && !(d->options & TO_UPLOAD_LAUNCHED) && d->n_owned == 0 &&
        m->GB.n_blk <= kGfPersistMaxBlocks) {
      int per_sm = 0;
      const void *fn = d->dim == 2 ? (const void *)k_gen_persist<2> : (const void *)k_gen_persist<3>;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kGfThreads, m->gb_smem));
      if ((int64_t)per_sm * kNumSMs >= m->GB.n_blk) {
        m->gen_persist = true;
        RC(ensure_partials(m, (size_t)m->GB.n_blk * 10));   // part[2][n_blk][5]
      }
    }
  }
  // workspace: internal-order vectors with zero pads on both sides (the
  // structured kernels read whole aligned row windows)
  RC(m->alloc(&m->s, m->n_el));
  std::vector<double **> vecs = {&m->x, &m->r, &m->pb[0], &m->pb[1], &m->q, &m->dinv, &m->D};
  if (m->structured || m->gen_fused) {
    vecs.push_back(&m->rb[1]);
    vecs.push_back(&m->qb[1]);
  }
  for (double **v : vecs) {
    double *base = nullptr;
    RC(m->alloc(&base, (size_t)(m->n_int + kS3PadFront + kS3PadBack)));
    CK(cudaMemsetAsync(base, 0, sizeof(double) * (m->n_int + kS3PadFront + kS3PadBack), st));
    *v = base + kS3PadFront;
  }
  m->rb[0] = m->r;
  m->qb[0] = m->q;
  if (m->structured) {
    const GridView &G = m->G;
    const uint32_t PY = kS3TYW + 1;
    RC(make_tensor_map(&m->tm_x, m->x, G.RS, G.NY, G.NZ, kS3RowD, PY));
    for (int b = 0; b < 2; ++b) {
      RC(make_tensor_map(&m->tm_rb[b], m->rb[b], G.RS, G.NY, G.NZ, kS3RowD, PY));
      RC(make_tensor_map(&m->tm_qb[b], m->qb[b], G.RS, G.NY, G.NZ, kS3RowD, PY));
      RC(make_tensor_map(&m->tm_pb[b], m->pb[b], G.RS, G.NY, G.NZ, kS3RowD, PY));
    }
    RC(make_tensor_map(&m->tm_dn, m->dn, G.NXP, G.NY, G.NZ, kS3RowN, PY));
  }
  CK(cudaStreamSynchronize(st));
  return 0;
}

// ---- operator pieces -------------------------------------------------------------------

int launch_simp(to_mesh *m, double penal, const double *x, cudaStream_t st) {
  int g = grid_for(m->n_el);
  if (m->dim == 2)
    k_simp<2><<<g, kBlock, 0, st>>>(m->n_el, x, m->elem_level, penal, m->E0, m->Emin, m->L, m->hL, m->s, m->S);
  else
    k_simp<3><<<g, kBlock, 0, st>>>(m->n_el, x, m->elem_level, penal, m->E0, m->Emin, m->L, m->hL, m->s, m->S);
  m->last_launches++;
  return check_launch();
}

// D = diag(Pi_F C^T K C Pi_F) from s; Dinv (free mask) and optional diag(A).
int launch_diag(to_mesh *m, double *d_out, cudaStream_t st) {
  const int g = grid_for(m->n_node);
  if (m->dim == 2) k_diag_node<2><<<g, kBlock, 0, st>>>(m->n_node, m->inc_ptr, m->inc, m->s, m->K2, m->D);
  else k_diag_node<3><<<g, kBlock, 0, st>>>(m->n_node, m->inc_ptr, m->inc, m->s, m->K3, m->D);
  k_dinv<<<grid_for(m->n_dof), kBlock, 0, st>>>(m->n_dof, m->free_dof, m->D, m->dinv, d_out, m->S);
  m->last_launches += 2;
  return check_launch();
}

int launch_rhs(to_mesh *m, double *b, cudaStream_t st) {
  int g = grid_for(m->n_node);
  if (m->dim == 2) k_rhs<2><<<g, kBlock, 0, st>>>(m->view(), m->load, b);
  else k_rhs<3><<<g, kBlock, 0, st>>>(m->view(), m->load, b);
  m->last_launches++;
  return check_launch();
}

// q = C^T K C p for p vanishing on non-free DOFs (values on non-free DOFs of
// q are not meaningful; callers mask): the single-kernel general operator in
// its plain mode.
int launch_matvec(to_mesh *m, const double *p, double *q, cudaStream_t st) {
  if (m->dim == 2)
    RC(launch_pdl(k_gen_fused<2, G_PLAIN>, dim3(m->GB.n_blk), dim3(kGfThreads), m->gb_smem, st, m->GB,
                  (const double *)m->s_loc, (const double *)nullptr, (const double *)nullptr, p,
                  (const double *)nullptr, (double *)nullptr, (double *)nullptr, q, (double *)nullptr, m->K2, m->KS,
                  (CgScalars *)nullptr, (double *)nullptr, 0, 0.0, (double *)nullptr, 0));
  else
    RC(launch_pdl(k_gen_fused<3, G_PLAIN>, dim3(m->GB.n_blk), dim3(kGfThreads), m->gb_smem, st, m->GB,
                  (const double *)m->s_loc, (const double *)nullptr, (const double *)nullptr, p,
                  (const double *)nullptr, (double *)nullptr, (double *)nullptr, q, (double *)nullptr, m->K2, m->KS,
                  (CgScalars *)nullptr, (double *)nullptr, 0, 0.0, (double *)nullptr, 0));
  m->last_launches++;
  return check_launch();
}

int launch_recover(to_mesh *m, const double *v, double *u, cudaStream_t st) {
  int g = grid_for(m->n_node);
  if (m->dim == 2) k_recover<2><<<g, kBlock, 0, st>>>(m->view(), v, u);
  else k_recover<3><<<g, kBlock, 0, st>>>(m->view(), v, u);
  m->last_launches++;
  return check_launch();
}

int reset_scalars(to_mesh *m, int max_iter, bool fixed, bool history, cudaStream_t st) {
  CgScalars h;
  std::memset(&h, 0, sizeof(h));
  h.max_iter = max_iter;
  h.fixed = fixed ? 1 : 0;
  h.history = history ? 1 : 0;
  *m->S_host = h;
  CK(cudaMemcpyAsync(m->S, m->S_host, sizeof(CgScalars), cudaMemcpyHostToDevice, st));
  return 0;
}

int read_scalars(to_mesh *m, cudaStream_t st) {
  CK(cudaMemcpyAsync(m->S_host, m->S, sizeof(CgScalars), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

// ---- internal-order operations --------------------------------------------------------
// The CG vectors are in "internal" order: lexicographic for the structured path,
// canonical (Morton, C3) otherwise.

const uint8_t *free_int(const to_mesh *m) { return m->structured ? m->free_lex : m->free_dof; }

// s_e and Dinv (internal order); d_int (optional) = diag(A) in internal order.
int op_scale_and_diag(to_mesh *m, double penal, const double *x, double *d_int, cudaStream_t st) {
  if (!m->structured) {
    RC(launch_simp(m, penal, x, st));
    RC(launch_diag(m, d_int, st));
    k_gather_s<<<grid_for(m->gb_n_loc_el), kBlock, 0, st>>>(m->gb_n_loc_el, m->gb_el_id, m->s, m->s_loc);
    m->last_launches++;
    if (m->gen_cluster) {
      k_gather_s<<<grid_for(m->gc_n_loc_el), kBlock, 0, st>>>(m->gc_n_loc_el, m->gc_el_id, m->s, m->gc_s_loc);
      m->last_launches++;
    }
    if (m->gen_ep) {
      k_gather_s<<<grid_for(m->ep_n_loc_el), kBlock, 0, st>>>(m->ep_n_loc_el, m->ep_el_id, m->s, m->ep_s_loc);
      m->last_launches++;
    }
    return check_launch();
  }
  k_simp_s3<<<grid_for(m->n_el), kBlock, 0, st>>>(m->n_el, x, m->perm_el, penal, m->E0, m->Emin, m->h_struct,
                                                   m->s, m->S);
  k_diag_s3<<<grid_for(m->n_node), kBlock, 0, st>>>(m->G, m->s, m->free_node_lex, m->k0d, m->dn, d_int, m->S);
  m->last_launches += 2;
  return check_launch();
}

// b = Pi_F C^T f in internal order
int op_rhs(to_mesh *m, double *b_int, cudaStream_t st) {
  if (!m->structured) return launch_rhs(m, b_int, st);
  k_to_int<<<grid_for(m->n_node), kBlock, 0, st>>>(m->n_node, m->perm_node, m->load, m->free_dof, b_int);
  m->last_launches++;
  return check_launch();
}

int s3_grid(const to_mesh *m) { return m->s3_ncta > 0 ? m->s3_ncta : m->G.ntx * m->G.nty * m->G.nzs; }

int op_apply(to_mesh *m, const double *in, double *out, cudaStream_t st) {
  if (!m->structured) return launch_matvec(m, in, out, st);
  const CUtensorMap *tin = in == m->x        ? &m->tm_x
                           : in == m->pb[0]  ? &m->tm_pb[0]
                           : in == m->rb[0]  ? &m->tm_rb[0]
                           : in == m->rb[1]  ? &m->tm_rb[1]
                                             : nullptr;
  if (!tin) { set_error("internal: unmapped apply input"); return TO_EINVAL; }
  S3Maps M;
  M.a = M.q = M.p = M.d = *tin;
  dim3 block(32, kS3TYW);
  k_apply_s3<kS3TYW, S3_PLAIN><<<s3_grid(m), block, sizeof(S3Smem<kS3TYW>), st>>>(
      m->G, m->s, M, nullptr, nullptr, nullptr, out, m->KS, nullptr, nullptr, 0, 0.0, nullptr, ShardComm{}, 0ull);
  m->last_launches++;
  return check_launch();
}

// General path, iteration k (kernels_genfused.cuh): the block kernel.
// step_in: it evaluates the step of iteration k-1 itself (the unsharded
// solve; op_cg_gen_step after the loop evaluates the last one); otherwise the
// shard group's exchange and step kernels follow it.
int op_cg_gen(to_mesh *m, int k, double rtol, cudaStream_t st, bool step_in) {
  const int o = (k + 1) & 1, w = k & 1;
  const dim3 grid(m->GB.n_blk);
  if (m->dim == 2)
    RC(launch_pdl(k_gen_fused<2, G_CG>, grid, dim3(kGfThreads), m->gb_smem, st, m->GB,
                  (const double *)m->s_loc, (const double *)m->rb[o], (const double *)m->qb[o],
                  (const double *)m->pb[o], (const double *)m->dinv, m->rb[w], m->pb[w], m->qb[w], m->x, m->K2,
                  m->KS, m->S, m->partials, k, rtol, m->hist, step_in ? 1 : 0));
  else
    RC(launch_pdl(k_gen_fused<3, G_CG>, grid, dim3(kGfThreads), m->gb_smem, st, m->GB,
                  (const double *)m->s_loc, (const double *)m->rb[o], (const double *)m->qb[o],
                  (const double *)m->pb[o], (const double *)m->dinv, m->rb[w], m->pb[w], m->qb[w], m->x, m->K2,
                  m->KS, m->S, m->partials, k, rtol, m->hist, step_in ? 1 : 0));
  m->last_launches++;
  return 0;
}
// The step of iteration k from the dots of launch k (partials[k & 1] when
// the launches evaluate the steps themselves, else partials[0]).
int op_cg_gen_step(to_mesh *m, int k, double rtol, cudaStream_t st, bool step_in) {
  RC(launch_pdl(k_gen_step, dim3(1), dim3(512), 0, st, m->GB.n_blk,
                (const double *)(m->partials + (step_in ? (size_t)5 * m->GB.n_blk * (k & 1) : 0)), m->S, k, rtol,
                m->hist));
  m->last_launches++;
  return 0;
}

// General path, x_N and the final residual after N iterations.
// Element-partitioned path (kernels_genep.cuh): iteration k and its step.
int op_cg_ep(to_mesh *m, int k, cudaStream_t st) {
  const int o = (k + 1) & 1, w = k & 1;
  if (m->dim == 2)
    RC(launch_pdl(k_gen_ep<2>, dim3(m->EB.n_blk), dim3(kGfThreads), m->ep_smem, st, m->EB,
                  (const double *)m->ep_s_loc, (const int32_t *)m->ep_slot_ptr, (const double *)m->ep_W[o],
                  m->ep_W[w], (const double *)m->rb[o], (const double *)m->qb[o], (const double *)m->pb[o],
                  (const double *)m->dinv, m->rb[w], m->qb[w], m->pb[w], m->x, m->K2, m->KS, m->S, m->partials,
                  (const double *)m->ep_w));
  else
    RC(launch_pdl(k_gen_ep<3>, dim3(m->EB.n_blk), dim3(kGfThreads), m->ep_smem, st, m->EB,
                  (const double *)m->ep_s_loc, (const int32_t *)m->ep_slot_ptr, (const double *)m->ep_W[o],
                  m->ep_W[w], (const double *)m->rb[o], (const double *)m->qb[o], (const double *)m->pb[o],
                  (const double *)m->dinv, m->rb[w], m->qb[w], m->pb[w], m->x, m->K2, m->KS, m->S, m->partials,
                  (const double *)m->ep_w));
  m->last_launches++;
  return 0;
}
int op_ep_reduce(to_mesh *m, int k, cudaStream_t st) {
  if (!TOMESH_EP_REDUCE) return 0;
  const int w = k & 1;
  const int g = std::min<int64_t>(grid_for(m->n_dof), (int64_t)4 * kNumSMs);
  if (m->dim == 2)
    RC(launch_pdl(k_ep_reduce<2>, dim3(g), dim3(kBlock), 0, st, (int64_t)m->n_dof, (const int32_t *)m->ep_slot_ptr,
                  (const double *)m->ep_W[w], (const double *)m->dinv, m->ep_w, (const CgScalars *)m->S));
  else
    RC(launch_pdl(k_ep_reduce<3>, dim3(g), dim3(kBlock), 0, st, (int64_t)m->n_dof, (const int32_t *)m->ep_slot_ptr,
                  (const double *)m->ep_W[w], (const double *)m->dinv, m->ep_w, (const CgScalars *)m->S));
  m->last_launches++;
  return 0;
}
int op_cg_ep_step(to_mesh *m, int k, double rtol, cudaStream_t st) {
  RC(launch_pdl(k_gen_ep_step, dim3(1), dim3(512), 0, st, m->EB.n_blk, (const double *)m->partials, m->S, k, rtol,
                m->hist));
  m->last_launches++;
  return 0;
}
// x_N after exactly N element-partitioned iterations (s = A p recurrence).
int op_final_ep(to_mesh *m, int n_iter, double rtol, cudaStream_t st) {
  const int o = (n_iter + 1) & 1;
  if (m->dim == 2)
    k_final_ep<2><<<grid_for(m->n_dof), kBlock, 0, st>>>(m->n_dof, m->ep_slot_ptr, m->ep_W[o], m->rb[o], m->qb[o],
                                                         m->pb[o], m->dinv, m->x, m->partials, m->S, n_iter, rtol,
                                                         m->hist);
  else
    k_final_ep<3><<<grid_for(m->n_dof), kBlock, 0, st>>>(m->n_dof, m->ep_slot_ptr, m->ep_W[o], m->rb[o], m->qb[o],
                                                         m->pb[o], m->dinv, m->x, m->partials, m->S, n_iter, rtol,
                                                         m->hist);
  m->last_launches++;
  return check_launch();
}

int op_final_gen(to_mesh *m, int n_iter, double rtol, cudaStream_t st) {
  const int o = (n_iter + 1) & 1;
  k_final_gen<false><<<grid_for(m->n_dof), kBlock, 0, st>>>(m->n_dof, m->rb[o], m->qb[o], m->pb[o], m->dinv,
                                                           m->x, m->partials, m->S, n_iter, rtol, m->hist,
                                                           ShardComm{}, 0ull);
  m->last_launches++;
  return check_launch();
}

// Structured path, the whole iteration k in one kernel (kernels_struct3d.cuh).
int op_cg_s3(to_mesh *m, int k, double rtol, cudaStream_t st) {
  const int o = (k + 1) & 1, w = k & 1;
  S3Maps M;
  M.a = m->tm_rb[o];
  M.q = m->tm_qb[o];
  M.p = m->tm_pb[o];
  M.d = m->tm_dn;
  dim3 block(32, kS3TYW);
  RC(launch_pdl(k_apply_s3<kS3TYW, S3_CG>, dim3(s3_grid(m)), block, sizeof(S3Smem<kS3TYW>), st, m->G,
                (const double *)m->s, M, m->rb[w], m->pb[w], m->x, m->qb[w], m->KS, m->S, m->partials, k, rtol,
                m->hist, ShardComm{}, 0ull));
  m->last_launches++;
  return 0;
}

// Structured path, x_N and the final residual after N iterations.
int op_final_s3(to_mesh *m, int n_iter, double rtol, cudaStream_t st) {
  const int o = (n_iter + 1) & 1;
  k_final_s3<false><<<kNumSMs * 4, 512, 0, st>>>((int)m->n_int, m->rb[o], m->qb[o], m->pb[o], m->dn, m->x,
                                                 m->partials, m->S, n_iter, rtol, m->hist, ShardComm{}, 0ull,
                                                 m->rb[1], m->pb[1]);
  m->last_launches++;
  return check_launch();
}

// dst = Pi_F u (canonical -> internal), used for warm starts
int op_masked_in(to_mesh *m, const double *u_canon, double *dst, cudaStream_t st) {
  if (!m->structured) {
    k_mask_free<<<grid_for(m->n_dof), kBlock, 0, st>>>(m->n_dof, m->free_dof, u_canon, dst);
  } else {
    k_to_int<<<grid_for(m->n_node), kBlock, 0, st>>>(m->n_node, m->perm_node, u_canon, m->free_dof, dst);
  }
  m->last_launches++;
  return check_launch();
}

// u = C v (internal -> canonical, hanging DOFs interpolated, Eq. 9)
int op_recover_out(to_mesh *m, const double *v_int, double *u_canon, cudaStream_t st) {
  if (!m->structured) return launch_recover(m, v_int, u_canon, st);
  k_from_int<<<grid_for(m->n_node), kBlock, 0, st>>>(m->n_node, m->perm_node, v_int, u_canon);
  m->last_launches++;
  return check_launch();
}

// ||b - A x||^2 over free DOFs for the internal x in m->x (true residual)
int op_resid2_x(to_mesh *m, double *r2, cudaStream_t st) {
  RC(op_rhs(m, m->r, st));                      // r := b
  RC(op_apply(m, m->x, m->q, st));              // q := C^T K C x
  k_resid2<<<grid_for(m->n_int), kBlock, 0, st>>>(m->n_int, m->r, m->q, free_int(m), m->partials, m->S);
  m->last_launches++;
  RC(read_scalars(m, st));
  *r2 = m->S_host->tmp[0];
  return 0;
}

int solve(to_mesh *m, double penal, const double *x_dev, double *u_dev, double rtol, int32_t max_iter,
          uint32_t flags, to_cg_stats *st_out, cudaStream_t st) {
  const bool fixed = (flags & TO_FIXED_ITERS) != 0;
  const bool warm = (flags & TO_WARM) != 0;
  const bool hist = (flags & TO_HISTORY) != 0;
  const int64_t n = m->n_int;
  m->last_launches = 0;
  if (hist && max_iter > m->hist_cap) {
    RC(m->alloc(&m->hist, (size_t)max_iter));
    m->hist_cap = max_iter;
  }
  CK(cudaEventRecord(m->ev0, st));
  RC(reset_scalars(m, max_iter, fixed, hist, st));
  RC(op_scale_and_diag(m, penal, x_dev, nullptr, st));
  // single-kernel iterations (launched, or the general path's cooperative
  // kernel for small meshes): iteration 0 reads r0 = b from rb[1]
  const bool cluster = !m->structured && m->gen_cluster;
  const bool persistent = !m->structured && !cluster && m->gen_persist;
  // element-partitioned iteration (large general meshes, kernels_genep.cuh)
  const bool ep = !m->structured && m->gen_ep;
  // launched general path: the step inside the block kernel for small grids
  const bool step_in = !m->structured && !ep && m->GB.n_blk <= kGfStepInMaxBlocks;
  double *r0 = m->rb[1];
  if (!m->structured) {   // q_{-1} = p_{-1} = 0 (finite whatever an earlier solve left)
    CK(cudaMemsetAsync(m->qb[1], 0, sizeof(double) * n, st));
    CK(cudaMemsetAsync(m->pb[1], 0, sizeof(double) * n, st));
    // element-partitioned: s_{-2} = qb[1] = 0, p_{-2} = 0, w_{-1} = 0 (slots of buffer 1)
    if (ep) CK(cudaMemsetAsync(m->ep_W[1], 0, sizeof(double) * (size_t)m->ep_n_slots * m->dim, st));
    if (ep) CK(cudaMemsetAsync(m->ep_w, 0, sizeof(double) * n, st));
  }
  RC(op_rhs(m, r0, st));
  const int gv = grid_for(n);
  k_norm2_b<<<gv, kBlock, 0, st>>>(n, r0, m->partials, m->S);
  m->last_launches++;
  if (warm) {
    RC(op_masked_in(m, u_dev, m->x, st));
    RC(op_apply(m, m->x, m->q, st));
    k_sub_masked<<<gv, kBlock, 0, st>>>(n, m->q, free_int(m), r0);
    m->last_launches++;
  } else {
    CK(cudaMemsetAsync(m->x, 0, sizeof(double) * n, st));
  }
  RC(check_launch());

  const bool prof = (flags & TO_PROFILE) != 0;
  if (prof) {
    size_t need = (size_t)3 * std::max(1, max_iter);
    while (m->prof_ev.size() < need) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      m->prof_ev.push_back(e);
    }
  }
  int launched = 0;
  int chunk = fixed ? std::max(1, max_iter) : 16;
  bool stop = false;
  const bool loop_prof = (flags & TO_PROFILE_LOOP) != 0;
  if (loop_prof) {
    for (auto &e : m->loop_ev)
      if (!e) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(m->loop_ev[0], st));
  }
  if (persistent && !stop) {
    // the whole loop in one cooperative kernel (no launches, no host polling)
    if (prof) CK(cudaEventRecord(m->prof_ev[0], st));
    const double *sl = m->s_loc, *dv = m->dinv;
    double *rb0 = m->rb[0], *rb1 = m->rb[1], *pb0 = m->pb[0], *pb1 = m->pb[1], *qb0 = m->qb[0], *qb1 = m->qb[1];
    int mi = max_iter;
    double rt = rtol;
    void *args[] = {&m->GB, &sl, &rb0, &rb1, &pb0, &pb1, &qb0, &qb1, &dv, &m->x, &m->K2, &m->KS, &m->S,
                    &m->partials, &mi, &rt, &m->hist};
    const void *fn = m->dim == 2 ? (const void *)k_gen_persist<2> : (const void *)k_gen_persist<3>;
    CK(cudaLaunchCooperativeKernel(fn, dim3(m->GB.n_blk), dim3(kGfThreads), args, m->gb_smem, st));
    m->last_launches++;
    if (prof) CK(cudaEventRecord(m->prof_ev[1], st));
    if (prof) CK(cudaEventRecord(m->prof_ev[2], st));
    stop = true;
    launched = max_iter;
  }
  if (cluster && !stop) {
    // the whole loop in one thread-block cluster (kernels_gencluster.cuh)
    if (prof) CK(cudaEventRecord(m->prof_ev[0], st));
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)m->GC.n_blk;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(m->GC.n_blk);
    cfg.blockDim = dim3(m->gc_threads);
    cfg.dynamicSmemBytes = m->gc_smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const double *sl = m->gc_s_loc, *dv = m->dinv;
    int mi = max_iter;
    double rt = rtol;
    void *args[] = {&m->GC, &m->GCS, &sl, &m->rb[0], &m->rb[1], &m->pb[0], &m->pb[1], &m->qb[0], &m->qb[1], &dv,
                    &m->x, &m->K2, &m->KS, &m->S, &mi, &rt, &m->hist};
    CK(cudaLaunchKernelExC(&cfg, gc_kernel(m->dim, m->gc_threads), args));
    m->last_launches++;
    if (prof) CK(cudaEventRecord(m->prof_ev[1], st));
    if (prof) CK(cudaEventRecord(m->prof_ev[2], st));
    stop = true;
    launched = max_iter;
  }
  while (!stop && launched < max_iter) {
    int cnt = std::min(chunk, max_iter - launched);
    for (int k = 0; k < cnt; ++k) {
      cudaEvent_t *E = prof ? &m->prof_ev[(size_t)3 * (launched + k)] : nullptr;
      if (prof) CK(cudaEventRecord(E[0], st));
      if (m->structured) {
        RC(op_cg_s3(m, launched + k, rtol, st));
        if (prof) CK(cudaEventRecord(E[1], st));
        if (prof) CK(cudaEventRecord(E[2], st));
      } else if (ep) {
        RC(op_cg_ep(m, launched + k, st));
        if (prof) CK(cudaEventRecord(E[1], st));
        RC(op_ep_reduce(m, launched + k, st));
        RC(op_cg_ep_step(m, launched + k, rtol, st));
        if (prof) CK(cudaEventRecord(E[2], st));
      } else if (step_in) {
        RC(op_cg_gen(m, launched + k, rtol, st, true));
        if (prof) CK(cudaEventRecord(E[1], st));
        if (prof) CK(cudaEventRecord(E[2], st));
      } else {
        RC(op_cg_gen(m, launched + k, rtol, st, false));
        if (prof) CK(cudaEventRecord(E[1], st));
        RC(op_cg_gen_step(m, launched + k, rtol, st, false));
        if (prof) CK(cudaEventRecord(E[2], st));
      }
    }
    RC(check_launch());
    launched += cnt;
    if (!fixed) {
      RC(read_scalars(m, st));
      stop = m->S_host->done || m->S_host->done_next;
      chunk = std::min(chunk * 2, 256);
    }
  }
  // general path, one launch per iteration: the step of the last launch (a
  // no-op if the solve has stopped)
  if (step_in && !persistent && !cluster && launched > 0) RC(op_cg_gen_step(m, launched - 1, rtol, st, true));
  if (loop_prof) CK(cudaEventRecord(m->loop_ev[1], st));
  // x_N after exactly N iterations (a no-op if an iteration already converged)
  if (m->structured) RC(op_final_s3(m, max_iter, rtol, st));
  else if (ep) RC(op_final_ep(m, max_iter, rtol, st));
  else RC(op_final_gen(m, max_iter, rtol, st));
  RC(check_launch());
  RC(read_scalars(m, st));
  CgScalars res = *m->S_host;
  if (loop_prof) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, m->loop_ev[0], m->loop_ev[1]));
    if (!prof)
      for (int j = 0; j < 4; ++j) m->prof_ms[j] = 0.0;
    m->prof_ms[5] = t;
    m->prof_ms[4] = std::min(launched, res.iter);
  }
  if (prof) {
    for (int j = 0; j < 5; ++j) m->prof_ms[j] = 0.0;
    int nit = std::min(launched, res.iter);
    for (int it = 0; it < (persistent || cluster ? std::min(nit, 1) : nit); ++it) {
      const int slot[2] = {0, 2};   // K1 (p/x update + apply + alpha), K2 (r update + reductions)
      for (int j = 0; j < 2; ++j) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, m->prof_ev[(size_t)3 * it + j], m->prof_ev[(size_t)3 * it + j + 1]));
        m->prof_ms[slot[j]] += t;
      }
    }
    m->prof_ms[4] = nit;
  }
  double relres_true = -1.0;
  if (!(flags & TO_NO_TRUE_RES) && res.status == 0) {
    double r2 = 0.0;
    RC(op_resid2_x(m, &r2, st));
    relres_true = res.bnorm2 > 0.0 ? std::sqrt(r2 / res.bnorm2) : 0.0;
  }
  RC(op_recover_out(m, m->x, u_dev, st));
  CK(cudaEventRecord(m->ev1, st));
  CK(cudaStreamSynchronize(st));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
  m->hist_len = hist ? res.iter : 0;
  int rc = res.status;
  if (rc == 0 && !fixed && !(res.rr <= res.thresh2) && res.bnorm2 > 0.0) rc = TO_NOT_CONVERGED;
  if (st_out) {
    st_out->iters = res.iter;
    st_out->status = rc;
    st_out->relres = res.bnorm2 > 0.0 ? std::sqrt(res.rr / res.bnorm2) : 0.0;
    st_out->relres_true = relres_true;
    st_out->ms = ms;
    st_out->bnorm = std::sqrt(res.bnorm2);
  }
  if (rc < 0) {
    const char *why = rc == TO_EBREAKDOWN ? "CG breakdown (p^T A p <= 0)"
                      : rc == TO_ENAN     ? "NaN/Inf in the CG recurrences"
                      : rc == TO_ENONPOS_DIAG ? "non-positive diagonal on a free DOF"
                      : rc == TO_EINVAL   ? "density outside (0, 1]"
                                          : "solver failure";
    set_error("%s", why);
  }
  return rc;
}

// ======================================================================================
// C ABI
// ======================================================================================

extern "C" int tomesh_upload(const to_mesh_desc *desc, int device, void *cuda_stream, to_mesh **out) {
  clear_error();
  if (!desc || !out) { set_error("NULL argument"); return TO_EINVAL; }
  *out = nullptr;
  int rc = validate(desc);
  if (rc) return rc;
  to_mesh *m = new (std::nothrow) to_mesh();
  if (!m) { set_error("out of host memory"); return TO_ENOMEM; }
  try {
    rc = do_upload(desc, device, (cudaStream_t)cuda_stream, m);
  } catch (...) {
    set_error("out of host memory during upload");
    rc = TO_ENOMEM;
  }
  if (rc) { delete m; return rc; }
  *out = m;
  return 0;
}

extern "C" void tomesh_free(to_mesh *m) {
  if (!m) return;
  cudaSetDevice(m->device);
  delete m;
}

extern "C" int tomesh_get_info(const to_mesh *m, to_mesh_info *info) {
  if (!m || !info) { set_error("NULL argument"); return TO_EINVAL; }
  std::memset(info, 0, sizeof(*info));
  info->dim = m->dim;
  info->structured = m->structured ? 1 : 0;
  info->grid[0] = m->structured ? m->G.EX : 0;
  info->grid[1] = m->structured ? m->G.EY : 0;
  info->grid[2] = m->structured ? m->G.EZ : 0;
  info->n_elem = m->n_el;
  info->n_node = m->n_node;
  info->n_dof = m->n_dof;
  info->n_hang = m->n_hang;
  info->n_fixed = m->n_fixed;
  info->filt_nnz = m->filt_nnz;
  info->device_bytes = m->dev_bytes;
  info->kernel_launches = m->last_launches;
  info->matvec_variant = m->structured ? 1 : m->gen_cluster ? 5 : m->gen_persist ? 3 : m->gen_ep ? 6 : 4;
  info->launches_total = m->launches_total;
  if (m->gen_ep) {   // the CG iteration runs on the element-partitioned blocks
    info->gen_blocks = m->EB.n_blk;
    info->gen_smem_bytes = (int32_t)m->ep_smem;
    info->gen_max_loc = m->EB.max_loc;
    info->gen_max_el = m->EB.max_el;
    info->gen_local_el = m->ep_local_el;
    info->gen_local_nodes = m->ep_local_nodes;
  } else if (m->gen_fused) {
    info->gen_blocks = m->GB.n_blk;
    info->gen_smem_bytes = (int32_t)m->gb_smem;
    info->gen_max_loc = m->GB.max_loc;
    info->gen_max_el = m->GB.max_el;
    info->gen_local_el = m->gb_local_el;
    info->gen_local_nodes = m->gb_local_nodes;
  }
  return 0;
}

extern "C" int tosolve_cg(to_mesh *m, double penal, const double *x_dev, double *u_dev, double rtol,
                          int32_t max_iter, uint32_t flags, to_cg_stats *st, void *cuda_stream) {
  clear_error();
  if (!m || !x_dev || !u_dev) { set_error("NULL argument"); return TO_EINVAL; }
  if (!(penal > 0.0) || max_iter < 0 || (!(flags & TO_FIXED_ITERS) && !(rtol >= 0.0))) {
    set_error("bad solver parameters");
    return TO_EINVAL;
  }
  if (cudaSetDevice(m->device) != cudaSuccess) { set_error("cudaSetDevice failed"); return TO_ECUDA; }
  const int rc = solve(m, penal, x_dev, u_dev, rtol, max_iter, flags, st, (cudaStream_t)cuda_stream);
  m->launches_total += m->last_launches;
  return rc;
}

extern "C" int tosolve_history(const to_mesh *m, double *out, int32_t n) {
  if (!m || !out || n < 0) { set_error("NULL argument"); return TO_EINVAL; }
  int cnt = std::min(n, m->hist_len);
  if (cnt > 0 && cudaMemcpy(out, m->hist, sizeof(double) * cnt, cudaMemcpyDeviceToHost) != cudaSuccess) {
    set_error("history copy failed");
    return TO_ECUDA;
  }
  return cnt;
}

extern "C" int tosolve_profile(const to_mesh *m, double *out, int32_t n) {
  if (!m || !out || n < 5) { set_error("bad argument"); return TO_EINVAL; }
  for (int j = 0; j < 5; ++j) out[j] = m->prof_ms[j];
  if (n >= 6) out[5] = m->prof_ms[5];
  return 0;
}

extern "C" int to_sensitivity(to_mesh *m, double penal, const double *x_dev, const double *u_dev, double *dc_dev,
                              double *compliance_host, void *cuda_stream) {
  clear_error();
  if (!m || !x_dev || !u_dev || !dc_dev) { set_error("NULL argument"); return TO_EINVAL; }
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int g = grid_for(m->n_el);
  if (m->dim == 2) k_sens<2><<<g, kBlock, 0, st>>>(m->view(), x_dev, u_dev, penal, m->E0, m->Emin, dc_dev, m->K2);
  else k_sens_had3<<<g, kBlock, 0, st>>>(m->view(), x_dev, u_dev, penal, m->E0, m->Emin, dc_dev, m->KS);
  m->launches_total++;
  RC(check_launch());
  if (compliance_host && m->sharded) return shard_compliance_partial(m, u_dev, compliance_host, st);
  if (compliance_host) {
    m->launches_total++;
    k_dot<<<grid_for(m->n_dof), kBlock, 0, st>>>(m->n_dof, m->load, u_dev, m->partials, m->S, 1);
    RC(check_launch());
    CK(cudaMemcpyAsync(m->S_host, m->S, sizeof(CgScalars), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *compliance_host = m->S_host->tmp[1];
  }
  return 0;
}

extern "C" int to_filter(to_mesh *m, int32_t mode, const double *x_dev, const double *in_dev, double *out_dev,
                         void *cuda_stream) {
  clear_error();
  if (!m || !in_dev || !out_dev || (mode == TO_FILTER_SENS && !x_dev)) { set_error("NULL argument"); return TO_EINVAL; }
  if (mode != TO_FILTER_SENS && mode != TO_FILTER_DENS) { set_error("bad filter mode"); return TO_EINVAL; }
  if (out_dev == in_dev || out_dev == x_dev) { set_error("out_dev aliases an input"); return TO_EINVAL; }
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (!(m->rmin > 0.0)) {   // filter deactivated: identity
    CK(cudaMemcpyAsync(out_dev, in_dev, sizeof(double) * m->n_el, cudaMemcpyDeviceToDevice, st));
    return 0;
  }
  int g = grid_for(m->n_el);
  if (m->structured) {
    k_filter_s3_scatter<<<g, kBlock, 0, st>>>(m->n_el, m->perm_el, mode, x_dev, in_dev, m->ftmp);
    k_filter_s3<<<g, kBlock, 0, st>>>(m->G, m->n_el, m->perm_el, m->foffs, m->n_foffs, mode, x_dev, m->ftmp, out_dev);
    m->launches_total += 2;
    return check_launch();
  }
  m->launches_total++;
  if (m->dim == 2) k_filter<2><<<g, kBlock, 0, st>>>(m->view(), m->filt_ptr, m->filt_idx, m->rmin, mode, x_dev, in_dev, out_dev);
  else k_filter<3><<<g, kBlock, 0, st>>>(m->view(), m->filt_ptr, m->filt_idx, m->rmin, mode, x_dev, in_dev, out_dev);
  return check_launch();
}

extern "C" int to_amr_mark(to_mesh *m, const double *x_dev, double rho_s, int8_t *marks_dev, void *cuda_stream) {
  clear_error();
  if (!m || !x_dev || !marks_dev) { set_error("NULL argument"); return TO_EINVAL; }
  if (!(rho_s > 0.0 && rho_s <= 1.0)) { set_error("rho_s must lie in (0, 1]"); return TO_EINVAL; }
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int g = grid_for(m->n_el);
  if (m->structured) {
    // structured meshes are one level: read it back once from the uploaded levels
    int8_t lev = 0;
    CK(cudaMemcpyAsync(&lev, m->elem_level, 1, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const bool filt = m->rmin > 0.0;
    if (filt) k_filter_s3_scatter<<<g, kBlock, 0, st>>>(m->n_el, m->perm_el, 1, x_dev, x_dev, m->ftmp);
    k_amr_mark_s3<<<g, kBlock, 0, st>>>(m->G, m->n_el, m->perm_el, m->foffs, filt ? m->n_foffs : 0,
                                        filt ? m->ftmp : nullptr, rho_s, lev, m->L, marks_dev);
    m->launches_total += filt ? 2 : 1;
    if (!filt) {   // no neighbourhood: only the element itself (reading R21 with r_amr = 0)
      k_amr_mark<<<g, kBlock, 0, st>>>(m->n_el, m->elem_level, m->L, nullptr, nullptr, x_dev, rho_s, marks_dev);
      m->launches_total++;
    }
    return check_launch();
  }
  k_amr_mark<<<g, kBlock, 0, st>>>(m->n_el, m->elem_level, m->L, m->rmin > 0.0 ? m->filt_ptr : nullptr,
                                   m->filt_idx, x_dev, rho_s, marks_dev);
  m->launches_total++;
  return check_launch();
}

extern "C" int to_apply_A(to_mesh *m, double penal, const double *x_dev, const double *v_dev, double *q_dev,
                          void *cuda_stream) {
  LaunchCounter lc_{m, m ? m->last_launches : 0};
  clear_error();
  if (!m || !x_dev || !v_dev || !q_dev || q_dev == v_dev) { set_error("bad argument"); return TO_EINVAL; }
  cudaStream_t st = (cudaStream_t)cuda_stream;
  RC(reset_scalars(m, 0, false, false, st));
  RC(op_scale_and_diag(m, penal, x_dev, nullptr, st));
  int gv = grid_for(m->n_dof);
  if (!m->structured) {
    k_mask_free<<<gv, kBlock, 0, st>>>(m->n_dof, m->free_dof, v_dev, m->pb[0]);
    m->last_launches++;
    RC(op_apply(m, m->pb[0], q_dev, st));
  } else {
    RC(op_masked_in(m, v_dev, m->pb[0], st));        // Pi_F v, internal order
    RC(op_apply(m, m->pb[0], m->q, st));
    RC(op_recover_out(m, m->q, q_dev, st));          // back to canonical order
  }
  k_fix_nonfree<<<gv, kBlock, 0, st>>>(m->n_dof, m->free_dof, v_dev, q_dev);
  m->last_launches++;
  return check_launch();
}

extern "C" int to_jacobi_diag(to_mesh *m, double penal, const double *x_dev, double *d_dev, void *cuda_stream) {
  LaunchCounter lc_{m, m ? m->last_launches : 0};
  clear_error();
  if (!m || !x_dev || !d_dev) { set_error("NULL argument"); return TO_EINVAL; }
  cudaStream_t st = (cudaStream_t)cuda_stream;
  RC(reset_scalars(m, 0, false, false, st));
  if (!m->structured) return op_scale_and_diag(m, penal, x_dev, d_dev, st);
  RC(op_scale_and_diag(m, penal, x_dev, m->D, st));
  return op_recover_out(m, m->D, d_dev, st);
}

extern "C" int to_project_rhs(to_mesh *m, double *b_dev, void *cuda_stream) {
  LaunchCounter lc_{m, m ? m->last_launches : 0};
  clear_error();
  if (!m || !b_dev) { set_error("NULL argument"); return TO_EINVAL; }
  return launch_rhs(m, b_dev, (cudaStream_t)cuda_stream);
}

extern "C" int to_recover(to_mesh *m, const double *v_dev, double *u_dev, void *cuda_stream) {
  LaunchCounter lc_{m, m ? m->last_launches : 0};
  clear_error();
  if (!m || !v_dev || !u_dev) { set_error("NULL argument"); return TO_EINVAL; }
  return launch_recover(m, v_dev, u_dev, (cudaStream_t)cuda_stream);
}

extern "C" int to_element_matrix(int32_t dim, double nu, double *K_host) {
  if ((dim != 2 && dim != 3) || !K_host) { set_error("bad argument"); return TO_EINVAL; }
  build_K0(dim, nu, K_host);
  return 0;
}

extern "C" int to_element_hadamard(double nu, double *diag_host, double *off_host) {
  if (!diag_host || !off_host) { set_error("NULL argument"); return TO_EINVAL; }
  K0Had3 h;
  int bad = build_K0_hadamard(nu, &h);
  std::memcpy(diag_host, h.diag, sizeof(h.diag));
  std::memcpy(off_host, h.off, sizeof(h.off));
  return bad;
}

#ifdef TOMESH_GF_TRACE
// A/B instrumentation build only: the per-block phase timestamps of the last
// k_gen_fused launch (16384 x 8 u64).
extern "C" int to_debug_gf_trace(unsigned long long *out) {
  return cudaMemcpyFromSymbol(out, g_gf_trace, sizeof(g_gf_trace)) == cudaSuccess ? 0 : TO_ECUDA;
}

#endif
