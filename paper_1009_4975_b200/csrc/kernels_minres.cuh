// The paper's own Krylov method (§5): preconditioned MINRES
// on the explicitly rescaled system K~ = D^-1/2 A D^-1/2 (:511-523), in the
// Lanczos / Givens form of Paige and Saunders (oracle/minres.py follows the
// same steps).  Vectors live in the handle's internal order and vanish on
// non-free DOFs, where K~ is the identity and b~ = 0.  With the plain
// rescaling, M = I on K~ (z = v); with IC(0), z = (L~ L~^T)^-1 v
// (kernels_ic0.cuh).  One iteration:
//   k_mr_wx_prep   the w / x~ update of the previous step (if pending), then
//                  zn = z_j / gamma_j and t = D^-1/2 zn (the apply input)
//   op_apply       q = C^T K C t
//   k_mr_delta     az = D^-1/2 q (= K~ zn), delta_j = az . zn
//   k_mr_lanczos   v_{j+1} = az - (delta/gamma) v_j - (gamma/gamma_{j-1}) v_{j-1}
//                  [M = I: gamma_{j+1}^2 = v.v reduced here]
//   k_mr_gamma     [IC(0): gamma_{j+1}^2 = z_{j+1} . v_{j+1}]
// and the last block of the gamma reduction applies the Givens rotation
// (mr_givens).  Deterministic: last-block-done reductions in block order.
#pragma once
#include "device_common.cuh"
#include "tomesh_types.cuh"

namespace tomesh {


// Givens step after gamma_{j+1}^2 is known (last block only).
__device__ __forceinline__ void mr_givens(MrScalars *S, double g2) {
  if (!(g2 == g2) || g2 < -1e300) {
    S->status = -5;
    S->done = 1;
    return;
  }
  const double gn = sqrt(fmax(g2, 0.0));
  const double gamma = S->gamma, delta = S->delta, c = S->c, c_old = S->c_old, s = S->s, s_old = S->s_old;
  const double a0 = c * delta - c_old * s * gamma;
  const double a1 = sqrt(a0 * a0 + gn * gn);
  const double a2 = s * delta + c_old * c * gamma;
  const double a3 = s_old * gamma;
  if (!(a1 > 0.0) || !(a1 == a1)) {
    S->status = (a1 == a1) ? -6 : -5;
    S->done = 1;
    return;
  }
  const double cn = a0 / a1, sn = gn / a1;
  S->a1 = a1;
  S->a2 = a2;
  S->a3 = a3;
  S->cn = cn;
  S->eta_prev = S->eta;
  S->eta = -sn * S->eta;
  S->gamma_old = gamma;
  S->gamma = gn;
  S->c_old = c;
  S->c = cn;
  S->s_old = s;
  S->s = sn;
  S->iter += 1;
  if (fabs(S->eta) <= S->thresh || gn == 0.0 || S->iter >= S->max_iter) S->done = 1;
}

// v1 = D^-1/2 b (internal order); with M = I also gamma_1 = ||v1|| and the
// initial scalars.  ||b||^2 -> bnorm2 (for the true residual).
template <bool IDENT>
__global__ void k_mr_init(int64_t n, const double *__restrict__ b, const double *__restrict__ msc,
                          double *__restrict__ v1, double *partials, MrScalars *S, double rtol) {
  double acc[2] = {0.0, 0.0};
  GRID_STRIDE(i, n) {
    const double bi = b[i];
    const double v = msc[i] * bi;
    v1[i] = v;
    acc[0] = fma(v, v, acc[0]);
    acc[1] = fma(bi, bi, acc[1]);
  }
  if (grid_sum<2>(acc, partials, &S->counter[MRC_MISC])) {
    S->bnorm2 = acc[1];
    if (IDENT) {
      const double g = sqrt(acc[0]);
      S->gamma = g;
      S->eta = S->eta0 = g;
      S->thresh = rtol * g;
      S->gamma_old = 1.0;
      S->c = S->c_old = 1.0;
      S->s = S->s_old = 0.0;
      if (!(g > 0.0) || S->max_iter <= 0) S->done = 1;
      if (!(g == g)) {
        S->status = -5;
        S->done = 1;
      }
    }
  }
}

// IC(0) start: gamma_1^2 = z1 . v1 and the initial scalars.
__global__ void k_mr_init_gamma(int64_t n, const double *__restrict__ z, const double *__restrict__ v, double *partials,
                                MrScalars *S, double rtol) {
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) { acc[0] = fma(z[i], v[i], acc[0]); }
  if (grid_sum<1>(acc, partials, &S->counter[MRC_MISC])) {
    const double g = sqrt(fmax(acc[0], 0.0));
    S->gamma = g;
    S->eta = S->eta0 = g;
    S->thresh = rtol * g;
    S->gamma_old = 1.0;
    S->c = S->c_old = 1.0;
    S->s = S->s_old = 0.0;
    if (!(g > 0.0) || S->max_iter <= 0) S->done = 1;
    if (!(g == g)) {
      S->status = -5;
      S->done = 1;
    }
  }
}

// w_new = (zn_prev - a3 w_old - a2 w) / a1, x~ += cn eta_prev w_new (if a step
// is pending), then zn = z_j / gamma_j, t = D^-1/2 zn (if not done).
__global__ void k_mr_wx_prep(int64_t n, const double *__restrict__ zn_prev, const double *__restrict__ w_old,
                             const double *__restrict__ w, double *__restrict__ w_new, double *__restrict__ xt,
                             const double *__restrict__ z, const double *__restrict__ msc, double *__restrict__ zn,
                             double *__restrict__ t, MrScalars *S) {
  const bool wx = __ldcg(&S->wx_done) < __ldcg(&S->iter);
  const bool prep = !__ldcg(&S->done);
  if (!wx && !prep) return;
  const double a1i = wx ? 1.0 / __ldcg(&S->a1) : 0.0, a2 = __ldcg(&S->a2), a3 = __ldcg(&S->a3);
  const double ce = wx ? __ldcg(&S->cn) * __ldcg(&S->eta_prev) : 0.0;
  const double gi = prep ? 1.0 / __ldcg(&S->gamma) : 0.0;
  GRID_STRIDE(i, n) {
    if (wx) {
      const double wn = (zn_prev[i] - a3 * w_old[i] - a2 * w[i]) * a1i;
      w_new[i] = wn;
      xt[i] = fma(ce, wn, xt[i]);
    }
    if (prep) {
      const double zz = z[i] * gi;
      zn[i] = zz;
      t[i] = msc[i] * zz;
    }
  }
  if (wx) {
    // the last block to finish records the update (the host rotates buffers
    // in step with S->iter, so exactly one update per step)
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(&S->counter[MRC_WX], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      S->counter[MRC_WX] = 0;
      S->wx_done = S->iter;
    }
  }
}

// az = D^-1/2 q, delta_j = az . zn
__global__ void k_mr_delta(int64_t n, const double *__restrict__ q, const double *__restrict__ msc,
                           const double *__restrict__ zn, double *__restrict__ az, double *partials, MrScalars *S) {
  if (__ldcg(&S->done)) return;
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) {
    const double a = msc[i] * q[i];
    az[i] = a;
    acc[0] = fma(a, zn[i], acc[0]);
  }
  if (grid_sum<1>(acc, partials, &S->counter[MRC_DELTA])) S->delta = acc[0];
}

// v_new = az - (delta/gamma) v - (gamma/gamma_old) v_old;  IDENT: gamma_new^2 = v_new . v_new + Givens
template <bool IDENT>
__global__ void k_mr_lanczos(int64_t n, const double *__restrict__ az, const double *__restrict__ v,
                             const double *__restrict__ v_old, double *__restrict__ v_new, double *partials,
                             MrScalars *S) {
  if (__ldcg(&S->done)) return;
  const double g = __ldcg(&S->gamma);
  const double f1 = __ldcg(&S->delta) / g, f2 = g / __ldcg(&S->gamma_old);
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) {
    const double vn = az[i] - f1 * v[i] - f2 * v_old[i];
    v_new[i] = vn;
    acc[0] = fma(vn, vn, acc[0]);
  }
  if (IDENT) {
    if (grid_sum<1>(acc, partials, &S->counter[MRC_GAMMA])) mr_givens(S, acc[0]);
  }
}

// IC(0): gamma_new^2 = z_new . v_new + Givens
__global__ void k_mr_gamma(int64_t n, const double *__restrict__ z, const double *__restrict__ v, double *partials,
                           MrScalars *S) {
  if (__ldcg(&S->done)) return;
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) { acc[0] = fma(z[i], v[i], acc[0]); }
  if (grid_sum<1>(acc, partials, &S->counter[MRC_GAMMA])) mr_givens(S, acc[0]);
}

// u_int = D^-1/2 x~
__global__ void k_mr_unscale(int64_t n, const double *__restrict__ msc, const double *__restrict__ xt,
                             double *__restrict__ u) {
  GRID_STRIDE(i, n) { u[i] = msc[i] * xt[i]; }
}

// D^-1/2 per internal DOF: general path from Dinv per DOF (0 on non-free)
__global__ void k_mr_scale(int64_t n, const double *__restrict__ dinv, double *__restrict__ msc) {
  GRID_STRIDE(i, n) { msc[i] = sqrt(dinv[i]); }
}

// D^-1/2 per internal DOF on the structured layout, from Dinv per node
__global__ void k_mr_scale_s3(GridView G, const double *__restrict__ dn, double *__restrict__ msc) {
  const int64_t nn = (int64_t)G.NX * G.NY * G.NZ;
  GRID_STRIDE(t, nn) {
    const int i = (int)(t % G.NX);
    const int64_t rest = t / G.NX;
    const int j = (int)(rest % G.NY), k = (int)(rest / G.NY);
    const double v = sqrt(dn[((int64_t)j + (int64_t)G.NY * k) * G.NXP + i]);
    double *o = msc + ((int64_t)j + (int64_t)G.NY * k) * G.RS + 3 * i;
    o[0] = o[1] = o[2] = v;
  }
}

}  // namespace tomesh
