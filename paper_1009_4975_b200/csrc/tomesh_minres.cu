// libtomesh — the paper's own solver (tosolve_minres):
// MINRES on the rescaled system and IC(0) of the rescaled matrix.
#include "tomesh_impl.cuh"
#include "kernels_minres.cuh"
#include "kernels_ic0.cuh"

using namespace tomesh;

int alloc_padded(to_mesh *m, double **v, cudaStream_t st) {
  double *base = nullptr;
  RC(m->alloc(&base, (size_t)(m->n_int + kS3PadFront + kS3PadBack)));
  CK(cudaMemsetAsync(base, 0, sizeof(double) * (m->n_int + kS3PadFront + kS3PadBack), st));
  *v = base + kS3PadFront;
  return 0;
}

int read_mr(to_mesh *m, cudaStream_t st) {
  CK(cudaMemcpyAsync(m->MS_host, m->MS, sizeof(MrScalars), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

int op_ic0_solve(to_mesh *m, const double *v, double *z, cudaStream_t st);   // below
int op_ic0_setup(to_mesh *m, cudaStream_t st, double *shift);

// MINRES on the rescaled system (header comment of kernels_minres.cuh).
int solve_minres(to_mesh *m, double penal, const double *x_dev, double *u_dev, double rtol, int32_t max_iter,
                 int32_t precond, uint32_t flags, to_minres_stats *st_out, cudaStream_t st) {
  const int64_t n = m->n_int;
  const bool ic0 = precond == TO_PC_IC0;
  m->last_launches = 0;
  if (!m->MS) {
    for (int b = 0; b < 3; ++b) {
      RC(alloc_padded(m, &m->mr_v[b], st));
      RC(alloc_padded(m, &m->mr_w[b], st));
    }
    for (int b = 0; b < 2; ++b) {
      RC(alloc_padded(m, &m->mr_zn[b], st));
      RC(alloc_padded(m, &m->mr_z[b], st));
    }
    RC(alloc_padded(m, &m->mr_xt, st));
    RC(alloc_padded(m, &m->mr_msc, st));
    RC(alloc_padded(m, &m->mr_az, st));
    if (!m->structured) RC(alloc_padded(m, &m->mr_t, st));
    RC(m->alloc(&m->MS, 1));
    CK(cudaMallocHost(&m->MS_host, sizeof(MrScalars)));
  }
  double *t = m->structured ? m->rb[0] : m->mr_t;   // the apply input (TMA-mapped when structured)
  CK(cudaEventRecord(m->ev0, st));
  RC(reset_scalars(m, 0, false, false, st));
  RC(op_scale_and_diag(m, penal, x_dev, nullptr, st));
  const int gv = grid_for(n);
  if (m->structured) {
    k_mr_scale_s3<<<grid_for((int64_t)m->G.NX * m->G.NY * m->G.NZ), kBlock, 0, st>>>(m->G, m->dn, m->mr_msc);
  } else {
    k_mr_scale<<<gv, kBlock, 0, st>>>(n, m->dinv, m->mr_msc);
  }
  m->last_launches++;
  RC(read_scalars(m, st));
  if (m->S_host->status != 0) {
    set_error(m->S_host->status == TO_EINVAL ? "density outside (0, 1]" : "non-positive diagonal on a free DOF");
    return m->S_host->status;
  }
  double shift = 0.0;
  if (ic0) RC(op_ic0_setup(m, st, &shift));
  std::memset(m->MS_host, 0, sizeof(MrScalars));
  m->MS_host->max_iter = max_iter;
  CK(cudaMemcpyAsync(m->MS, m->MS_host, sizeof(MrScalars), cudaMemcpyHostToDevice, st));
  for (int b = 0; b < 3; ++b) {
    CK(cudaMemsetAsync(m->mr_v[b], 0, sizeof(double) * n, st));
    CK(cudaMemsetAsync(m->mr_w[b], 0, sizeof(double) * n, st));
  }
  CK(cudaMemsetAsync(m->mr_xt, 0, sizeof(double) * n, st));
  RC(op_rhs(m, m->r, st));                                   // b (internal order)
  if (!ic0) {
    k_mr_init<true><<<gv, kBlock, 0, st>>>(n, m->r, m->mr_msc, m->mr_v[1], m->partials, m->MS, rtol);
    m->last_launches++;
  } else {
    k_mr_init<false><<<gv, kBlock, 0, st>>>(n, m->r, m->mr_msc, m->mr_v[1], m->partials, m->MS, rtol);
    m->last_launches++;
    RC(op_ic0_solve(m, m->mr_v[1], m->mr_z[1], st));
    k_mr_init_gamma<<<gv, kBlock, 0, st>>>(n, m->mr_z[1], m->mr_v[1], m->partials, m->MS, rtol);
    m->last_launches++;
  }
  RC(check_launch());
  // iteration it performs Lanczos / Givens step j = it + 1 and, first, the
  // w / x~ update of step it (buffers: v(k) in mr_v[k%3], w(k) in mr_w[k%3],
  // zn(k) in mr_zn[k%2], z(k) in mr_z[k%2])
  auto iteration = [&](int it) -> int {
    const double *z_j = ic0 ? m->mr_z[(it + 1) % 2] : m->mr_v[(it + 1) % 3];
    k_mr_wx_prep<<<gv, kBlock, 0, st>>>(n, m->mr_zn[(it + 1) % 2], m->mr_w[(it + 2) % 3], m->mr_w[it % 3],
                                        m->mr_w[(it + 1) % 3], m->mr_xt, z_j, m->mr_msc, m->mr_zn[it % 2], t, m->MS);
    m->last_launches++;
    RC(op_apply(m, t, m->q, st));
    k_mr_delta<<<gv, kBlock, 0, st>>>(n, m->q, m->mr_msc, m->mr_zn[it % 2], m->mr_az, m->partials, m->MS);
    m->last_launches++;
    double *v_new = m->mr_v[(it + 2) % 3];
    if (!ic0) {
      k_mr_lanczos<true><<<gv, kBlock, 0, st>>>(n, m->mr_az, m->mr_v[(it + 1) % 3], m->mr_v[it % 3], v_new,
                                                m->partials, m->MS);
      m->last_launches++;
    } else {
      k_mr_lanczos<false><<<gv, kBlock, 0, st>>>(n, m->mr_az, m->mr_v[(it + 1) % 3], m->mr_v[it % 3], v_new,
                                                 m->partials, m->MS);
      m->last_launches++;
      RC(op_ic0_solve(m, v_new, m->mr_z[it % 2], st));
      k_mr_gamma<<<gv, kBlock, 0, st>>>(n, m->mr_z[it % 2], v_new, m->partials, m->MS);
      m->last_launches++;
    }
    return 0;
  };
  RC(read_mr(m, st));
  int launched = 0, chunk = 16;
  bool stop = m->MS_host->done != 0;
  while (!stop && launched < max_iter) {
    const int cnt = std::min(chunk, max_iter - launched);
    for (int k = 0; k < cnt; ++k) RC(iteration(launched + k));
    RC(check_launch());
    launched += cnt;
    RC(read_mr(m, st));
    stop = m->MS_host->done != 0;
    chunk = std::min(chunk * 2, 256);
  }
  // the w / x~ update of the last step (a no-op if an enqueued iteration did it)
  {
    const int it = launched;
    k_mr_wx_prep<<<gv, kBlock, 0, st>>>(n, m->mr_zn[(it + 1) % 2], m->mr_w[(it + 2) % 3], m->mr_w[it % 3],
                                        m->mr_w[(it + 1) % 3], m->mr_xt, m->mr_v[0], m->mr_msc, m->mr_zn[it % 2], t,
                                        m->MS);
    m->last_launches++;
  }
  k_mr_unscale<<<gv, kBlock, 0, st>>>(n, m->mr_msc, m->mr_xt, m->x);
  m->last_launches++;
  RC(read_mr(m, st));
  MrScalars res = *m->MS_host;
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
  int rc = res.status;
  const bool converged = res.eta0 == 0.0 || std::fabs(res.eta) <= res.thresh;
  if (rc == 0 && !converged) rc = TO_NOT_CONVERGED;
  if (st_out) {
    st_out->iters = res.iter;
    st_out->status = rc;
    st_out->eta_rel = res.eta0 > 0.0 ? std::fabs(res.eta) / res.eta0 : 0.0;
    st_out->relres_true = relres_true;
    st_out->ms = ms;
    st_out->ic0_shift = ic0 ? shift : -1.0;
    st_out->ic0_levels[0] = ic0 ? m->ic_nlvl : 0;
    st_out->ic0_levels[1] = ic0 ? m->ic_nblvl : 0;
  }
  if (rc < 0) set_error("%s", rc == TO_EBREAKDOWN ? "MINRES breakdown" : "NaN/Inf in the MINRES recurrences");
  return rc;
}

template <typename T>
int download(std::vector<T> &h, const T *d, size_t n) {
  h.resize(n);
  if (n) CK(cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost));
  return 0;
}

// Host symbolic phase of IC(0) (general path): the lower pattern of K~ over
// free-free couplings (through the Eq. 6 interpolation) plus unit rows of the
// non-free DOFs, the element contributions of every nonzero, the transposed
// pattern and the dependency levels of both triangular solves.
int ic0_build(to_mesh *m, cudaStream_t st) {
  const int dim = m->dim, nc = 1 << dim, ND = dim * nc;
  const int64_t n = m->n_dof, ne = m->n_el;
  if (ne * (int64_t)(ND * (ND + 1) / 2) > (int64_t)250000000) {
    set_error("IC(0): %lld elements give more than 2.5e8 element contributions (host symbolic phase too large)",
              (long long)ne);
    return TO_ENOMEM;
  }
  CK(cudaStreamSynchronize(st));
  std::vector<int32_t> en, nh, hp, hpar;
  std::vector<double> hw;
  std::vector<uint8_t> fr;
  RC(download(en, m->elem_node, (size_t)ne * nc));
  RC(download(nh, m->node_hang, (size_t)m->n_node));
  RC(download(fr, m->free_dof, (size_t)n));
  if (m->n_hang > 0) {
    RC(download(hp, m->hang_ptr, (size_t)m->n_hang + 1));
    RC(download(hpar, m->hang_parent, (size_t)hp[m->n_hang]));
    RC(download(hw, m->hang_weight, (size_t)hp[m->n_hang]));
  }
  auto wcode = [](double w) -> int { return w == 1.0 ? 0 : w == 0.5 ? 1 : w == 0.25 ? 2 : -1; };
  // expansions of every local DOF of an element: (global free DOF, log2(1/w))
  auto expand = [&](int64_t e, int a, std::vector<std::pair<int64_t, int>> &out) {
    out.clear();
    const int32_t node = en[e * nc + a / dim], c = a % dim;
    if (nh[node] < 0) {
      const int64_t g = (int64_t)node * dim + c;
      if (fr[g]) out.push_back({g, 0});
      return;
    }
    const int32_t h = nh[node];
    for (int32_t k = hp[h]; k < hp[h + 1]; ++k) {
      const int64_t g = (int64_t)hpar[k] * dim + c;
      if (fr[g]) out.push_back({g, wcode(hw[k])});
    }
  };
  std::vector<std::vector<std::pair<int64_t, int>>> ex(ND);
  // per row: (column, packed contribution), then sorted by column
  std::vector<std::vector<std::pair<int32_t, uint64_t>>> rows(n);
  for (int64_t e = 0; e < ne; ++e) {
    for (int a = 0; a < ND; ++a) expand(e, a, ex[a]);
    for (int a = 0; a < ND; ++a)
      for (const auto &pa : ex[a])
        for (int b = 0; b < ND; ++b)
          for (const auto &pb : ex[b]) {
            if (pb.first > pa.first) continue;   // lower triangle (column <= row)
            const uint64_t code = (uint64_t)(pa.second + pb.second);
            rows[pa.first].push_back({(int32_t)pb.first, ((uint64_t)e << 16) | ((uint64_t)(a * ND + b) << 3) | code});
          }
  }
  std::vector<int64_t> ptr(n + 1, 0), cptr(1, 0);
  std::vector<int32_t> col, row;
  std::vector<uint64_t> contrib;
  for (int64_t i = 0; i < n; ++i) {
    auto &R = rows[i];
    std::stable_sort(R.begin(), R.end(), [](const std::pair<int32_t, uint64_t> &x, const std::pair<int32_t, uint64_t> &y) {
      return x.first < y.first;
    });
    if (R.empty()) {                         // non-free DOF: unit diagonal, no contributions
      col.push_back((int32_t)i);
      row.push_back((int32_t)i);
      cptr.push_back((int64_t)contrib.size());
    } else {
      for (size_t u = 0; u < R.size();) {
        size_t v = u;
        while (v < R.size() && R[v].first == R[u].first) contrib.push_back(R[v++].second);
        col.push_back(R[u].first);
        row.push_back((int32_t)i);
        cptr.push_back((int64_t)contrib.size());
        u = v;
      }
      if (col.back() != (int32_t)i) { set_error("IC(0): free row %lld without a diagonal", (long long)i); return TO_EMESH; }
    }
    ptr[i + 1] = (int64_t)col.size();
    std::vector<std::pair<int32_t, uint64_t>>().swap(R);
  }
  const int64_t nnz = (int64_t)col.size();
  // dependency levels: forward (row i after its columns k < i), backward (row k of L^T after rows i > k)
  std::vector<int32_t> lv(n, 0), blv(n, 0);
  int nl = 0, nbl = 0;
  for (int64_t i = 0; i < n; ++i) {
    int l = 0;
    for (int64_t t = ptr[i]; t < ptr[i + 1] - 1; ++t) l = std::max(l, lv[col[t]] + 1);
    lv[i] = l;
    nl = std::max(nl, l + 1);
  }
  std::vector<int64_t> ut_ptr(n + 1, 0);
  for (int64_t t = 0; t < nnz; ++t)
    if (col[t] != row[t]) ut_ptr[col[t] + 1]++;
  for (int64_t k = 0; k < n; ++k) ut_ptr[k + 1] += ut_ptr[k];
  std::vector<int32_t> ut_row(ut_ptr[n]);
  std::vector<int64_t> ut_pos(ut_ptr[n]), ufill(ut_ptr.begin(), ut_ptr.end() - 1);
  for (int64_t i = 0; i < n; ++i)          // rows ascending: each column's entries ascending in i
    for (int64_t t = ptr[i]; t < ptr[i + 1] - 1; ++t) {
      const int64_t q = ufill[col[t]]++;
      ut_row[q] = (int32_t)i;
      ut_pos[q] = t;
    }
  for (int64_t k = n - 1; k >= 0; --k) {
    int l = 0;
    for (int64_t t = ut_ptr[k]; t < ut_ptr[k + 1]; ++t) l = std::max(l, blv[ut_row[t]] + 1);
    blv[k] = l;
    nbl = std::max(nbl, l + 1);
  }
  auto bucket = [&](const std::vector<int32_t> &lvl, int nlev, std::vector<int64_t> &lptr, std::vector<int32_t> &lrows) {
    lptr.assign(nlev + 1, 0);
    for (int64_t i = 0; i < n; ++i) lptr[lvl[i] + 1]++;
    for (int l = 0; l < nlev; ++l) lptr[l + 1] += lptr[l];
    lrows.resize(n);
    std::vector<int64_t> f(lptr.begin(), lptr.end() - 1);
    for (int64_t i = 0; i < n; ++i) lrows[f[lvl[i]]++] = (int32_t)i;
  };
  std::vector<int64_t> lptr, blptr;
  std::vector<int32_t> lrows, blrows;
  bucket(lv, nl, lptr, lrows);
  bucket(blv, nbl, blptr, blrows);
  // the solve kernels (k_ic0_tri: ic_warps warps, a row each) walk "steps": the
  // levels cut into pieces of at most ic_warps rows, so that every row goes through
  // the software pipeline (a barrier between two pieces of one level is
  // redundant but cheap; arithmetic and order are the level schedule's)
  // warps per CTA: about twice the mean rows per level (idle warps still pay
  // the per-step bookkeeping and the barrier: c1, 5.6 rows per level, 130 ms
  // with 32 warps, 112 with 16; c2, 14 rows per level, 3.54 s with 32, 3.65 s
  // with 16; profiles/r2/ic0_tri_ab.txt)
  const double mean_rows = (double)n / std::max(1, std::max(nl, nbl));
  int W = 8;
  while (W < kIc0Warps && W < 2.0 * mean_rows) W *= 2;
  m->ic_warps = W;
  auto split = [&](const std::vector<int64_t> &lp, std::vector<int64_t> &sp) {
    sp.assign(1, 0);
    for (size_t l = 0; l + 1 < lp.size(); ++l)
      for (int64_t r = lp[l]; r < lp[l + 1]; r += W) sp.push_back(std::min<int64_t>(r + W, lp[l + 1]));
  };
  std::vector<int64_t> slptr, sblptr;
  split(lptr, slptr);
  split(blptr, sblptr);
  // device copies
  int64_t *d_ptr, *d_cptr;
  int32_t *d_col, *d_row;
  uint64_t *d_contrib;
  RC(upload_array(m, &d_ptr, ptr.data(), ptr.size(), st));
  RC(upload_array(m, &d_col, col.data(), col.size(), st));
  RC(upload_array(m, &d_row, row.data(), row.size(), st));
  RC(upload_array(m, &d_cptr, cptr.data(), cptr.size(), st));
  RC(upload_array(m, &d_contrib, contrib.data(), std::max<size_t>(1, contrib.size()), st));
  RC(upload_array(m, &m->ic_lvl_rows, lrows.data(), lrows.size(), st));
  RC(upload_array(m, &m->ic_blvl_rows, blrows.data(), blrows.size(), st));
  RC(upload_array(m, &m->ic_step_ptr, slptr.data(), slptr.size(), st));
  RC(upload_array(m, &m->ic_bstep_ptr, sblptr.data(), sblptr.size(), st));
  m->ic_nstep = (int)slptr.size() - 1;
  m->ic_nbstep = (int)sblptr.size() - 1;
  RC(upload_array(m, &m->ic_ut_ptr, ut_ptr.data(), ut_ptr.size(), st));
  RC(upload_array(m, &m->ic_ut_row, ut_row.data(), std::max<size_t>(1, ut_row.size()), st));
  RC(upload_array(m, &m->ic_ut_pos, ut_pos.data(), std::max<size_t>(1, ut_pos.size()), st));
  const double *K0 = dim == 2 ? m->K2.K : m->K3.K;
  RC(upload_array(m, &m->ic_K0, K0, (size_t)ND * ND, st));
  RC(m->alloc(&m->ic_kt, (size_t)nnz));
  RC(m->alloc(&m->ic_L, (size_t)nnz));
  RC(m->alloc(&m->ic_y, (size_t)n));
  RC(m->alloc(&m->ic_fail, 1));
  m->IC.n = n;
  m->IC.nnz = nnz;
  m->IC.ptr = d_ptr;
  m->IC.col = d_col;
  m->IC.row = d_row;
  m->IC.cptr = d_cptr;
  m->IC.contrib = d_contrib;
  m->ic_lvl_host = lptr;
  m->ic_nlvl = nl;
  m->ic_nblvl = nbl;
  m->ic_ready = true;
  CK(cudaStreamSynchronize(st));
  return 0;
}

// K~ (+ a I) assembled and factored; a = 0, then 1e-3 2^t until no pivot fails
int op_ic0_setup(to_mesh *m, cudaStream_t st, double *shift) {
  if (m->structured) {
    set_error("IC(0) needs the general (canonical-order) operator path; upload with the TO_UPLOAD_GENERAL option");
    return TO_EINVAL;
  }
  if (!m->ic_ready) RC(ic0_build(m, st));
  const int g = grid_for(m->IC.nnz);
  for (int t = -1; t < 30; ++t) {
    const double a = t < 0 ? 0.0 : 1e-3 * std::ldexp(1.0, t);
    if (m->dim == 2) k_ic0_assemble<2><<<g, kBlock, 0, st>>>(m->IC, m->s, m->mr_msc, m->ic_K0, a, m->ic_L);
    else k_ic0_assemble<3><<<g, kBlock, 0, st>>>(m->IC, m->s, m->mr_msc, m->ic_K0, a, m->ic_L);
    m->last_launches++;
    CK(cudaMemsetAsync(m->ic_fail, 0, sizeof(int), st));
    for (int l = 0; l < m->ic_nlvl; ++l) {
      const int64_t r0 = m->ic_lvl_host[l], r1 = m->ic_lvl_host[l + 1];
      k_ic0_factor<<<(int)std::min<int64_t>((r1 - r0 + 127) / 128, 4 * kNumSMs), 128, 0, st>>>(
          m->IC, m->ic_lvl_rows, r0, r1, m->ic_L, m->ic_fail);
    }
    m->last_launches += m->ic_nlvl;
    RC(check_launch());
    int fail = 0;
    CK(cudaMemcpyAsync(&fail, m->ic_fail, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!fail) {
      *shift = a;
      return 0;
    }
  }
  set_error("IC(0) breaks down for every shift tried");
  return TO_EBREAKDOWN;
}

// z = (L L^T)^-1 v
int op_ic0_solve(to_mesh *m, const double *v, double *z, cudaStream_t st) {
  k_ic0_tri<false><<<1, 32 * m->ic_warps, 0, st>>>(m->IC, nullptr, nullptr, nullptr, m->ic_step_ptr, m->ic_nstep,
                                                 m->ic_lvl_rows, m->ic_L, v, m->ic_y);
  k_ic0_tri<true><<<1, 32 * m->ic_warps, 0, st>>>(m->IC, m->ic_ut_ptr, m->ic_ut_row, m->ic_ut_pos, m->ic_bstep_ptr,
                                                m->ic_nbstep, m->ic_blvl_rows, m->ic_L, m->ic_y, z);
  m->last_launches += 2;
  return check_launch();
}

extern "C" int tosolve_minres(to_mesh *m, double penal, const double *x_dev, double *u_dev, double rtol,
                              int32_t max_iter, int32_t precond, uint32_t flags, to_minres_stats *st,
                              void *cuda_stream) {
  LaunchCounter lc_{m, 0};
  clear_error();
  if (!m || !x_dev || !u_dev || !(penal > 0.0) || max_iter < 0 || !(rtol >= 0.0)) {
    set_error("bad argument");
    return TO_EINVAL;
  }
  if (precond != TO_PC_JACOBI && precond != TO_PC_IC0) { set_error("unknown preconditioner"); return TO_EINVAL; }
  if (flags & ~(uint32_t)TO_NO_TRUE_RES) { set_error("tosolve_minres supports TO_NO_TRUE_RES only"); return TO_EINVAL; }
  return solve_minres(m, penal, x_dev, u_dev, rtol, max_iter, precond, flags, st, (cudaStream_t)cuda_stream);
}
