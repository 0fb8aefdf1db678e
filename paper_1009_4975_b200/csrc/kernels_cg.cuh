// Jacobi-PCG scalar logic and vector kernels shared by both paths (textbook
// Hestenes-Stiefel recurrences on the rescaled system, PAPER.md:511-523 with
// reading Q3).  The iteration kernels themselves live in kernels_struct3d.cuh
// (uniform H8: one kernel per iteration) and kernels_general.cuh (AMR: an
// element pass and a node pass per iteration).  Dinv == 0 marks hanging and
// fixed DOFs: r, p, x stay 0 there (A is the identity on them and b vanishes
// there, so this is exact).
#pragma once
#include "device_common.cuh"

namespace tomesh {


// Scalars after the initial residual: rho0 = r0.z0, rr0, thresholds.
__device__ __forceinline__ void cg_init_scalars(CgScalars *S, double rho, double rr, double rtol) {
  S->rho = rho;
  S->rr = rr;
  S->thresh2 = rtol * rtol * S->bnorm2;
  S->alpha = 0.0;
  S->beta = 0.0;
  if (S->bnorm2 == 0.0 || S->status != 0) S->done = 1;
  if (!S->fixed && rr <= S->thresh2) S->done = 1;
  if (S->max_iter <= 0) S->done = 1;
  if (!(rho == rho) || !(rr == rr)) {
    cg_fail(S, -5);
    S->done = 1;
  }
}

// Scalars after the r update of iteration k (one completed iteration).
__device__ __forceinline__ void cg_after_rupdate(CgScalars *S, double rz, double rr, double *hist) {
  const int it = S->iter + 1;
  S->iter = it;
  if (!(rz == rz) || !(rr == rr)) {
    cg_fail(S, -5);
    S->done = 1;
    return;
  }
  S->beta = rz / S->rho;
  S->rho = rz;
  S->rr = rr;
  if (S->history && hist) hist[it - 1] = sqrt(rr / S->bnorm2);
  if ((!S->fixed && rr <= S->thresh2) || it >= S->max_iter) S->done_next = 1;
}

// Structured path, end of the single-kernel iteration k (last block).
// d = {rho_k = r_k.Dinv r_k, rr_k = r_k.r_k, p_k.q_k, q_k.z_k, q_k.Dinv q_k},
// all exact dots of the vectors formed in this kernel.  x_k is complete.
//   stop if rr_k <= rtol^2 ||b||^2 (x_k is the answer, k iterations);
//   alpha_k = rho_k / p_k.q_k;
//   rho_{k+1} = (r_k - alpha q).Dinv (r_k - alpha q)
//             = rho_k - 2 alpha q.z_k + alpha^2 q.Dinv q   (one-step expansion:
//     the next kernel needs beta_k = rho_{k+1}/rho_k before it can form r_{k+1};
//     its own exact rho_{k+1} then feeds alpha_{k+1}, so the expansion error,
//     ~eps rho_k / rho_{k+1}, enters beta_k only and does not accumulate).
__device__ __forceinline__ void cg_single_step(CgScalars *S, int k, const double (&d)[5], double rtol, double *hist) {
  const double rho = d[0], rr = d[1], pq = d[2], qz = d[3], qdq = d[4];
  if (k == 0) {
    S->thresh2 = rtol * rtol * S->bnorm2;
    if (S->status != 0) {
      S->done = 1;
      return;
    }
  }
  S->iter = k;
  S->rho = rho;
  S->rr = rr;
  if (!(rho == rho) || !(rr == rr) || !(pq == pq) || !(qz == qz) || !(qdq == qdq)) {
    cg_fail(S, -5);
    S->done = 1;
    return;
  }
  if (S->history && hist && k >= 1) hist[k - 1] = sqrt(rr / S->bnorm2);
  if ((!S->fixed && rr <= S->thresh2) || S->bnorm2 == 0.0) {
    S->done = 1;
    return;
  }
  if (!(pq > 0.0)) {
    cg_fail(S, -6);
    S->done = 1;
    return;
  }
  const double alpha = rho / pq;
  const double rho_next = fma(alpha * alpha, qdq, fma(-2.0 * alpha, qz, rho));
  S->alpha = alpha;
  S->beta = rho_next / rho;
  S->ab[k & 1][0] = S->alpha;
  S->ab[k & 1][1] = S->beta;
}

// Element-partitioned general path (kernels_genep.cuh), end of iteration k in
// the Chronopoulos-Gear form: d = {gamma_k = r_k.u_k, rr_k, delta_k = A u_k .
// u_k}, u_k = Dinv r_k, all of kernel k's vectors.  x_k is complete.
//   stop if rr_k <= rtol^2 ||b||^2;
//   beta_k = gamma_k / gamma_{k-1} (beta_0 = 0),
//   alpha_k = gamma_k / (delta_k - beta_k gamma_k / alpha_{k-1}) (alpha_0 = gamma_0 / delta_0)
// (the denominator is p_k . A p_k: <= 0 is a breakdown, status -6).
__device__ __forceinline__ void cg_cgear_step(CgScalars *S, int k, const double (&d)[5], double rtol, double *hist) {
  const double gam = d[0], rr = d[1], del = d[2];
  if (k == 0) {
    S->thresh2 = rtol * rtol * S->bnorm2;
    if (S->status != 0) {
      S->done = 1;
      return;
    }
  }
  const double gam_prev = S->rho, alpha_prev = S->alpha;
  S->iter = k;
  S->rho = gam;
  S->rr = rr;
  if (!(gam == gam) || !(rr == rr) || !(del == del)) {
    cg_fail(S, -5);
    S->done = 1;
    return;
  }
  if (S->history && hist && k >= 1) hist[k - 1] = sqrt(rr / S->bnorm2);
  if ((!S->fixed && rr <= S->thresh2) || S->bnorm2 == 0.0) {
    S->done = 1;
    return;
  }
  double beta = 0.0, den = del;
  if (k > 0) {
    beta = gam / gam_prev;
    den = del - beta * gam / alpha_prev;
  }
  if (!(den > 0.0)) {
    cg_fail(S, -6);
    S->done = 1;
    return;
  }
  S->alpha = gam / den;
  S->beta = beta;
  S->ab[k & 1][0] = S->alpha;
  S->ab[k & 1][1] = S->beta;
}

// cg_single_step split for the sharded K1, where EVERY CTA of iteration k+1
// forms the step of iteration k from the same gathered dots (no separate step
// kernel): cg_step_eval is the pure decision (reads only fields that are
// constant during the solve, or that every CTA writes with the same value),
// cg_step_commit writes it to S (one CTA).  Same arithmetic as cg_single_step.
struct CgStepOut {
  double alpha, beta, rho, rr, thresh2;
  int done, fail, early;   // early: k == 0 with a failed status (nothing else is written)
};
__device__ __forceinline__ void cg_step_eval(const CgScalars *S, int k, const double (&d)[5], double rtol,
                                             CgStepOut &o) {
  const double rho = d[0], rr = d[1], pq = d[2], qz = d[3], qdq = d[4];
  const double bnorm2 = __ldcg(&S->bnorm2);
  o.alpha = o.beta = 0.0;
  o.rho = rho;
  o.rr = rr;
  o.done = o.fail = o.early = 0;
  o.thresh2 = k == 0 ? rtol * rtol * bnorm2 : __ldcg(&S->thresh2);
  if (k == 0 && __ldcg(&S->status) != 0) {
    o.done = o.early = 1;
    return;
  }
  if (!(rho == rho) || !(rr == rr) || !(pq == pq) || !(qz == qz) || !(qdq == qdq)) {
    o.fail = -5;
    o.done = 1;
    return;
  }
  if ((!S->fixed && rr <= o.thresh2) || bnorm2 == 0.0) {
    o.done = 1;
    return;
  }
  if (!(pq > 0.0)) {
    o.fail = -6;
    o.done = 1;
    return;
  }
  const double alpha = rho / pq;
  const double rho_next = fma(alpha * alpha, qdq, fma(-2.0 * alpha, qz, rho));
  o.alpha = alpha;
  o.beta = rho_next / rho;
}
// cg_step_eval with the fields it reads from S loaded once per solve (a
// kernel that runs the whole loop): bnorm2, fixed, the status before the
// loop, thresh2 = rtol^2 bnorm2 (what step 0 computes).  Same arithmetic.
struct CgConst {
  double bnorm2, thresh2;
  int fixed, status;
};
__device__ __forceinline__ CgConst cg_const(const CgScalars *S, double rtol) {
  CgConst c;
  c.bnorm2 = __ldcg(&S->bnorm2);
  c.thresh2 = rtol * rtol * c.bnorm2;
  c.fixed = __ldcg(&S->fixed);
  c.status = __ldcg(&S->status);
  return c;
}
__device__ __forceinline__ void cg_step_eval_c(const CgConst &c, int k, const double (&d)[5], CgStepOut &o) {
  const double rho = d[0], rr = d[1], pq = d[2], qz = d[3], qdq = d[4];
  o.alpha = o.beta = 0.0;
  o.rho = rho;
  o.rr = rr;
  o.done = o.fail = o.early = 0;
  o.thresh2 = c.thresh2;
  if (k == 0 && c.status != 0) {
    o.done = o.early = 1;
    return;
  }
  if (!(rho == rho) || !(rr == rr) || !(pq == pq) || !(qz == qz) || !(qdq == qdq)) {
    o.fail = -5;
    o.done = 1;
    return;
  }
  if ((!c.fixed && rr <= o.thresh2) || c.bnorm2 == 0.0) {
    o.done = 1;
    return;
  }
  if (!(pq > 0.0)) {
    o.fail = -6;
    o.done = 1;
    return;
  }
  const double alpha = rho / pq;
  const double rho_next = fma(alpha * alpha, qdq, fma(-2.0 * alpha, qz, rho));
  o.alpha = alpha;
  o.beta = rho_next / rho;
}
__device__ __forceinline__ void cg_step_commit(CgScalars *S, int k, const CgStepOut &o, double *hist) {
  if (k == 0) S->thresh2 = o.thresh2;
  if (o.early) {
    S->done = 1;
    return;
  }
  S->iter = k;
  S->rho = o.rho;
  S->rr = o.rr;
  if (o.fail) cg_fail(S, o.fail);
  if (o.fail == -5) {
    S->done = 1;
    return;
  }
  if (S->history && hist && k >= 1) hist[k - 1] = sqrt(o.rr / S->bnorm2);
  if (o.done) {
    S->done = 1;
    return;
  }
  S->alpha = o.alpha;
  S->beta = o.beta;
  S->ab[k & 1][0] = o.alpha;
  S->ab[k & 1][1] = o.beta;
}

// Deferred x update of the structured kernel (kernels_struct3d.cuh).  Kernel
// k stages p_{k-1} and r_{k-1} (z_{k-1} = Dinv r_{k-1}); the textbook update
// there is x_k = x_{k-1} + alpha_{k-1} p_{k-1}.  An odd kernel k skips x (one
// read and one write of x saved) and the next kernel applies both terms:
//   alpha_{k-1} p_{k-1} = (alpha_{k-1} / beta_{k-1}) (p_k - z_k)
// since p_k = z_k + beta_{k-1} p_{k-1}.  Only when |beta_{k-1}| is not tiny
// (a deterministic test on the step's own scalars, so every CTA, rank and the
// final kernel take the same decision); x's rounding differs from the
// textbook order by the reconstruction only (it never feeds back into r, p).
constexpr double kXDeferMinBeta = 1e-6;
__device__ __forceinline__ bool cg_x_deferred(int k, double alpha_km1, double beta_km1) {
  return (k & 1) && alpha_km1 != 0.0 && fabs(beta_km1) >= kXDeferMinBeta;
}
// x += cp p_{k-1} + cz z_{k-1} in kernel k (touch = false: x untouched).
// a1 = alpha_{k-1}; (a2, b2) = (alpha_{k-2}, beta_{k-2}); defer = false
// forces the update (the final kernel).
struct XCoef {
  double cp, cz;
  bool touch;
};
__device__ __forceinline__ XCoef cg_x_coef(int k, double a1, double b1, double a2, double b2, bool defer) {
  XCoef c{a1, 0.0, a1 != 0.0};
  if (defer && cg_x_deferred(k, a1, b1)) {
    c.touch = false;
    return c;
  }
  if (k >= 2 && cg_x_deferred(k - 1, a2, b2)) {   // kernel k-1 left alpha_{k-2} p_{k-2} pending
    const double t = a2 / b2;
    c.cp = a1 + t;
    c.cz = -t;
    c.touch = true;
  }
  return c;
}

// Structured path, final step after N = max_iter iterations (or 0): r_N =
// r_{N-1} - alpha q_{N-1}, x_N = x_{N-1} + alpha p_{N-1}, rho_N, rr_N.
// Elementwise over node pairs (no operator needed).
__device__ __forceinline__ void cg_final_step(CgScalars *S, int n_iter, double rho, double rr, double rtol,
                                              double *hist) {
  if (n_iter == 0) S->thresh2 = rtol * rtol * S->bnorm2;
  S->iter = n_iter;
  S->rho = rho;
  S->rr = rr;
  if (!(rho == rho) || !(rr == rr)) cg_fail(S, -5);
  if (S->history && hist && n_iter >= 1) hist[n_iter - 1] = sqrt(rr / S->bnorm2);
  S->done = 1;
}

// ||v||^2 -> S->bnorm2 (used for b).
static __global__ void k_norm2_b(int64_t n, const double *__restrict__ v, double *partials, CgScalars *S) {
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) { double t = v[i]; acc[0] = fma(t, t, acc[0]); }
  if (grid_sum<1>(acc, partials, &S->counter[CNT_MISC])) S->bnorm2 = acc[0];
}

// r = r - q on free DOFs (warm start: r = b - A x0); `free` per DOF.
static __global__ void k_sub_masked(int64_t n, const double *__restrict__ q, const uint8_t *__restrict__ free_dof,
                             double *__restrict__ r) {
  GRID_STRIDE(i, n) { r[i] = free_dof[i] ? r[i] - q[i] : 0.0; }
}

// sum over free DOFs of (b - t)^2 -> S->tmp[0]
static __global__ void k_resid2(int64_t n, const double *__restrict__ b, const double *__restrict__ t,
                         const uint8_t *__restrict__ free_dof, double *partials, CgScalars *S) {
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) {
    if (free_dof[i]) { double d = b[i] - t[i]; acc[0] = fma(d, d, acc[0]); }
  }
  if (grid_sum<1>(acc, partials, &S->counter[CNT_MISC])) S->tmp[0] = acc[0];
}

// a . b -> S->tmp[slot]
static __global__ void k_dot(int64_t n, const double *__restrict__ a, const double *__restrict__ b, double *partials,
                      CgScalars *S, int slot) {
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) { acc[0] = fma(a[i], b[i], acc[0]); }
  if (grid_sum<1>(acc, partials, &S->counter[CNT_MISC2])) S->tmp[slot] = acc[0];
}

// q_i = free ? q_i : v_i   (completes A v = Pi_F C^T K C Pi_F v + (I - Pi_F) v)
static __global__ void k_fix_nonfree(int64_t n, const uint8_t *__restrict__ free_dof, const double *__restrict__ v,
                              double *__restrict__ q) {
  GRID_STRIDE(i, n) { if (!free_dof[i]) q[i] = v[i]; }
}

static __global__ void k_mask_free(int64_t n, const uint8_t *__restrict__ free_dof, const double *__restrict__ v,
                            double *__restrict__ w) {
  GRID_STRIDE(i, n) { w[i] = free_dof[i] ? v[i] : 0.0; }
}

}  // namespace tomesh
