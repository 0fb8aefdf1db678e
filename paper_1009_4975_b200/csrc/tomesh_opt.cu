// libtomesh — the OC design update (to_oc_update) and the Fig. 1 loop
// (to_optimize).
#include "tomesh_impl.cuh"
#include "kernels_oc.cuh"

using namespace tomesh;

extern "C" int to_oc_update(to_mesh *m, const double *x_dev, const double *dc_dev, double volfrac, double move,
                            double eta, double rho_o, double *x_new_dev, to_oc_stats *st, void *cuda_stream) {
  clear_error();
  if (!m || !x_dev || !dc_dev || !x_new_dev) { set_error("NULL argument"); return TO_EINVAL; }
  if (x_new_dev == dc_dev) { set_error("x_new_dev aliases dc_dev"); return TO_EINVAL; }
  if (!(volfrac > 0.0 && volfrac <= 1.0) || !(move >= 0.0 && move <= 1.0) || !(eta > 0.0 && eta <= 4.0) ||
      !(rho_o > 0.0 && rho_o < 1.0)) {
    set_error("OC parameters out of range (volfrac in (0,1], move in [0,1], eta in (0,4], rho_o in (0,1))");
    return TO_EINVAL;
  }
  if (m->L > 23) { set_error("max_level too large for the OC volume table"); return TO_EINVAL; }
  cudaStream_t st_ = (cudaStream_t)cuda_stream;
  if (!m->oc_a) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_oc_update, kOcBlock, 0));
    if (per_sm < 1) { set_error("OC kernel cannot be resident"); return TO_ECUDA; }
    const int64_t need = (m->n_el + kOcBlock - 1) / kOcBlock;
    m->oc_blocks = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)per_sm * kNumSMs));
    if (m->n_el <= 16 * kOcBlock) m->oc_blocks = 1;   // latency-bound: one block, block-level sums only
    RC(m->alloc(&m->oc_a, (size_t)m->n_el));
    RC(m->alloc(&m->oc_part, (size_t)kOcCand * m->oc_blocks));
    RC(m->alloc(&m->oc_state, 1));
    if (!m->oc_state_host) CK(cudaMallocHost(&m->oc_state_host, sizeof(OcState)));
  }
  OcArgs A{};
  A.n = m->n_el;
  A.x = x_dev;
  A.dc = dc_dev;
  A.level = m->structured ? nullptr : m->elem_level;
  A.a = m->oc_a;
  A.xn = x_new_dev;
  A.target = volfrac * m->vol_total;
  A.move = move;
  A.eta = eta;
  A.rho_o = rho_o;
  A.lam_hi = 1e9;
  A.tol = 1e-12;
  A.max_steps = 200;
  for (int l = 0; l < 24; ++l) {
    const double hs = l <= m->L ? std::ldexp(m->hL, m->L - l) : 0.0;   // (2^(L-l) h_L)
    A.vtab[l] = m->dim == 2 ? hs * hs : hs * hs * hs;
  }
  if (m->structured) A.vtab[0] = m->dim == 2 ? m->h_struct * m->h_struct : m->h_struct * m->h_struct * m->h_struct;
  CK(cudaEventRecord(m->ev0, st_));
  CK(cudaMemsetAsync(m->oc_state, 0, sizeof(OcState), st_));   // reduction counters, flag, max
  void *args[] = {(void *)&A, (void *)&m->oc_part, (void *)&m->oc_state};
  CK(cudaLaunchCooperativeKernel((const void *)k_oc_update, dim3(m->oc_blocks), dim3(kOcBlock), args, 0, st_));
  m->launches_total++;
  CK(cudaEventRecord(m->ev1, st_));
  RC(check_launch());
  if (!st) return 0;
  CK(cudaMemcpyAsync(m->oc_state_host, m->oc_state, sizeof(OcState), cudaMemcpyDeviceToHost, st_));
  CK(cudaStreamSynchronize(st_));
  const OcState &S = *m->oc_state_host;
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
  st->lambda = S.lam;
  st->volume = S.volume_abs / m->vol_total;
  st->change = S.change;
  st->ms = ms;
  st->steps = S.steps;
  st->state = S.state;
  st->passes = S.passes;
  if (S.state < 0) { set_error("NaN/Inf in x or dc"); return TO_ENAN; }
  return 0;
}

extern "C" int to_optimize(to_mesh *m, const to_opt_params *P, int32_t n_steps, double *x_dev, double *u_dev,
                           to_opt_step *hist, int32_t *steps_done, to_opt_state *state, void *cuda_stream) {
  clear_error();
  if (steps_done) *steps_done = 0;
  if (!m || !P || !x_dev || !u_dev || n_steps < 0) { set_error("bad argument"); return TO_EINVAL; }
  if (!(P->penal0 > 0.0) || !(P->penal_max >= P->penal0) || !(P->penal_step >= 0.0) || P->stage_steps < 1 ||
      !(P->rtol > 0.0) || P->max_iter < 1 || P->adapt_min_steps < 0 || P->adapt_max_steps < 0) {
    set_error("bad continuation, solver or adaptation parameters");
    return TO_EINVAL;
  }
  if (!m->opt_dc) {
    RC(m->alloc(&m->opt_dc, (size_t)m->n_el));
    RC(m->alloc(&m->opt_dcf, (size_t)m->n_el));
  }
  double penal = state ? state->penal : P->penal0;
  int at_stage = state ? state->at_stage : 0, since = state ? state->since_adapt : 0;
  if (!(penal > 0.0)) { set_error("state->penal must be > 0"); return TO_EINVAL; }
  if (state) state->adapt_due = state->converged = 0;
  const bool amr = P->adapt_max_steps > 0;
  int k = 0, result = TO_OK;
  for (; k < n_steps; ++k) {
    to_cg_stats cs{};
    const int rc = tosolve_cg(m, penal, x_dev, u_dev, P->rtol, P->max_iter, (k > 0 ? TO_WARM : 0) | TO_NO_TRUE_RES,
                              &cs, cuda_stream);
    if (rc < 0) return rc;
    if (rc > 0) result = TO_NOT_CONVERGED;
    double c = 0.0;
    RC(to_sensitivity(m, penal, x_dev, u_dev, m->opt_dc, &c, cuda_stream));
    const double *dcf = m->opt_dc;
    if (P->filter && m->rmin > 0.0) {
      RC(to_filter(m, TO_FILTER_SENS, x_dev, m->opt_dc, m->opt_dcf, cuda_stream));
      dcf = m->opt_dcf;
    }
    to_oc_stats os{};
    RC(to_oc_update(m, x_dev, dcf, P->volfrac, P->move, P->eta, P->rho_o, x_dev, &os, cuda_stream));
    if (hist) {
      to_opt_step &h = hist[k];
      h.compliance = c;
      h.penal = penal;
      h.volume = os.volume;
      h.change = os.change;
      h.lambda = os.lambda;
      h.solve_ms = cs.ms;
      h.oc_ms = os.ms;
      h.cg_iters = cs.iters;
      h.status = rc;
    }
    ++at_stage;
    ++since;
    const bool conv = os.change < P->change_tol;
    if (P->stop_on_converge && penal >= P->penal_max && conv) {
      ++k;
      if (state) state->converged = 1;
      break;
    }
    if (penal < P->penal_max && (conv || at_stage >= P->stage_steps)) {
      penal = std::min(P->penal_max, penal + P->penal_step);
      at_stage = 0;
    }
    if (amr && ((conv && since >= P->adapt_min_steps) || since >= P->adapt_max_steps)) {
      ++k;
      if (state) state->adapt_due = 1;
      break;
    }
  }
  if (state) {
    state->penal = penal;
    state->at_stage = at_stage;
    state->since_adapt = since;
  }
  if (steps_done) *steps_done = k;
  return result;
}
