// Fused Jacobi-PCG vector kernels (textbook Hestenes-Stiefel recurrences on
// the rescaled system, PAPER.md:511-523 with SURVEY reading Q3).
//
// Per iteration (V = 12 fp64 vector passes):
//   matvec            q = A p                         (p read, q written)
//   k_pq              alpha = rho / (p.q)             (p, q read) [v0 only; fused later]
//   k_u1              r -= alpha q; rho' = r.(Dinv r); rr = r.r      (r, q, Dinv -> r)
//   k_u2              x += alpha p;  p = Dinv r + beta p            (r, Dinv, p, x -> p, x)
// Dinv == 0 marks hanging and fixed DOFs: r, p, x stay 0 there (A is the
// identity on them and b vanishes there, so this is exact).
#pragma once
#include "device_common.cuh"

namespace tomesh {

#define GRID_STRIDE(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ||v||^2 -> S->bnorm2 (used for b).
__global__ void k_norm2_b(int64_t n, const double *__restrict__ v, double *partials, CgScalars *S) {
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) { double t = v[i]; acc[0] = fma(t, t, acc[0]); }
  if (grid_sum<1>(acc, partials, &S->counter[CNT_MISC])) S->bnorm2 = acc[0];
}

// x = Pi_F u (warm start), masked copy using Dinv as the free mask.
__global__ void k_mask_copy(int64_t n, const double *__restrict__ u, const double *__restrict__ Dinv,
                            double *__restrict__ x) {
  GRID_STRIDE(i, n) { x[i] = (Dinv[i] != 0.0) ? u[i] : 0.0; }
}

// r = r - q on free DOFs (warm start: r = b - A x0).
__global__ void k_sub_masked(int64_t n, const double *__restrict__ q, const double *__restrict__ Dinv,
                             double *__restrict__ r) {
  GRID_STRIDE(i, n) { r[i] = (Dinv[i] != 0.0) ? r[i] - q[i] : 0.0; }
}

// z = Dinv r; p = z; rho = r.z; rr = r.r; thresholds.
__global__ void k_init(int64_t n, const double *__restrict__ r, const double *__restrict__ Dinv,
                       double *__restrict__ p, double *partials, CgScalars *S, double rtol) {
  double acc[2] = {0.0, 0.0};
  GRID_STRIDE(i, n) {
    double ri = r[i], z = Dinv[i] * ri;
    p[i] = z;
    acc[0] = fma(ri, z, acc[0]);
    acc[1] = fma(ri, ri, acc[1]);
  }
  if (grid_sum<2>(acc, partials, &S->counter[CNT_INIT])) {
    S->rho = acc[0];
    S->rr = acc[1];
    S->thresh2 = rtol * rtol * S->bnorm2;
    S->alpha = 0.0;
    S->beta = 0.0;
    if (S->bnorm2 == 0.0 || S->status != 0) S->done = 1;
    if (!S->fixed && acc[1] <= S->thresh2) S->done = 1;
    if (S->max_iter <= 0) S->done = 1;
  }
}

// alpha = rho / (p . q)
__global__ void k_pq(int64_t n, const double *__restrict__ p, const double *__restrict__ q, double *partials,
                     CgScalars *S) {
  if (cg_stopped(S)) return;
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) { acc[0] = fma(p[i], q[i], acc[0]); }
  if (grid_sum<1>(acc, partials, &S->counter[CNT_PQ])) {
    double pq = acc[0];
    if (!(pq > 0.0)) {
      S->status = (pq != pq) ? -5 : -6;   // TO_ENAN / TO_EBREAKDOWN
      S->done = 1;
    } else {
      S->alpha = S->rho / pq;
    }
  }
}

__global__ void k_u1(int64_t n, const double *__restrict__ q, const double *__restrict__ Dinv,
                     double *__restrict__ r, double *partials, CgScalars *S, double *hist) {
  if (cg_stopped(S)) return;
  const double alpha = S->alpha;
  double acc[2] = {0.0, 0.0};
  GRID_STRIDE(i, n) {
    double di = Dinv[i];
    double ri = r[i];
    if (di != 0.0) ri = fma(-alpha, q[i], ri);
    r[i] = ri;
    acc[0] = fma(ri, di * ri, acc[0]);
    acc[1] = fma(ri, ri, acc[1]);
  }
  if (grid_sum<2>(acc, partials, &S->counter[CNT_U1])) {
    double rz = acc[0], rr = acc[1];
    int it = S->iter + 1;
    S->iter = it;
    if (!(rz == rz) || !(rr == rr)) {
      S->status = -5;
      S->done = 1;
      return;
    }
    S->beta = rz / S->rho;
    S->rho = rz;
    S->rr = rr;
    if (S->history && hist) hist[it - 1] = sqrt(rr / S->bnorm2);
    if ((!S->fixed && rr <= S->thresh2) || it >= S->max_iter) S->done_next = 1;
  }
}

__global__ void k_u2(int64_t n, const double *__restrict__ r, const double *__restrict__ Dinv,
                     double *__restrict__ p, double *__restrict__ x, const CgScalars *S) {
  if (*((volatile const int32_t *)&S->done)) return;
  const double alpha = S->alpha, beta = S->beta;
  GRID_STRIDE(i, n) {
    double pi = p[i];
    x[i] = fma(alpha, pi, x[i]);
    p[i] = fma(beta, pi, Dinv[i] * r[i]);
  }
}

// sum over free DOFs of (b - t)^2 -> S->tmp[0]
__global__ void k_resid2(int64_t n, const double *__restrict__ b, const double *__restrict__ t,
                         const uint8_t *__restrict__ free_dof, double *partials, CgScalars *S) {
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) {
    if (free_dof[i]) { double d = b[i] - t[i]; acc[0] = fma(d, d, acc[0]); }
  }
  if (grid_sum<1>(acc, partials, &S->counter[CNT_MISC])) S->tmp[0] = acc[0];
}

// a . b -> S->tmp[slot]
__global__ void k_dot(int64_t n, const double *__restrict__ a, const double *__restrict__ b, double *partials,
                      CgScalars *S, int slot) {
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) { acc[0] = fma(a[i], b[i], acc[0]); }
  if (grid_sum<1>(acc, partials, &S->counter[CNT_MISC2])) S->tmp[slot] = acc[0];
}

// q_i = free ? q_i : v_i   (completes A v = Pi_F C^T K C Pi_F v + (I - Pi_F) v)
__global__ void k_fix_nonfree(int64_t n, const uint8_t *__restrict__ free_dof, const double *__restrict__ v,
                              double *__restrict__ q) {
  GRID_STRIDE(i, n) { if (!free_dof[i]) q[i] = v[i]; }
}

__global__ void k_mask_free(int64_t n, const uint8_t *__restrict__ free_dof, const double *__restrict__ v,
                            double *__restrict__ w) {
  GRID_STRIDE(i, n) { w[i] = free_dof[i] ? v[i] : 0.0; }
}

}  // namespace tomesh
