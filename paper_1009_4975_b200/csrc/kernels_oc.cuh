// OC design update ("we use Optimality Criteria (OC)",
// formula per DESIGN.md reading R18) in ONE cooperative kernel: the whole
// bisection on the volume multiplier runs on the device with one grid-wide
// reduction per pass over the elements (block sums -> per-block partials ->
// the last block to arrive adds them in a fixed order and releases the
// totals to every block, so all blocks take the same branch), 3 bisection
// steps per pass, no host round trip.
//
//   x_e(lam) = min(hi_e, max(lo_e, x_e (max(-dc_e, 0) / (lam V_e))^eta))
//   lo_e = max(rho_o, x_e - move), hi_e = min(1, x_e + move)
//   vol(lam) = sum_e V_e x_e(lam)  == target = V0 sum_e V_e   (Eq. 1)
//
// B200 formulation: the lam dependence factors out of the element term,
// x_e (g_e / lam)^eta = a_e lam^-eta with a_e = x_e g_e^eta, g_e = max(-dc_e,0)/V_e,
// so the first pass stores a_e once (one pow per element) and every
// bisection pass is a clamp + fma per element over (x, a) that stays resident
// in the 126 MB L2 for meshes up to ~7M elements, with t = lam^-eta computed
// once per pass.  The bracket and the step sequence are exactly those of the
// oracle (oracle/oc.py), so both take the same decisions except when vol(lam)
// lies within rounding of the target.
#pragma once
#include "device_common.cuh"
#include "tomesh_types.cuh"

namespace tomesh {


struct OcArgs {
  int64_t n;
  const double *x, *dc;
  const int8_t *level;    // nullptr: every element has volume vtab[0]
  double *a;              // [n] workspace
  double *xn;             // [n] output (may alias x)
  double target, move, eta, rho_o, lam_hi, tol;
  int32_t max_steps;
  double vtab[24];        // V_e by level (exact dyadics, host-computed)
};

__device__ __forceinline__ double oc_block_max(double v) {
  __shared__ double sh[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  return v;
}

__device__ __forceinline__ uint32_t oc_ld_acquire(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ double oc_V(const OcArgs &A, int64_t e) {
  return A.level ? A.vtab[A.level[e]] : A.vtab[0];
}

__device__ __forceinline__ double oc_clamp(double xe, double v, const OcArgs &A) {
  const double lo = fmax(A.rho_o, xe - A.move), hi = fmin(1.0, xe + A.move);
  return fmin(hi, fmax(lo, v));
}

__device__ __forceinline__ double oc_pow_neg(double l, double eta) {   // l^-eta
  return eta == 0.5 ? 1.0 / sqrt(l) : pow(l, -eta);
}

// Speculative bisection: one pass over the elements evaluates vol() at the
// 2^kOcDepth - 1 midpoints the next kOcDepth sequential bisection steps could
// visit (heap order: node i spans (L_i, R_i), candidate c_i = (L_i + R_i)/2,
// children 2i+1 = (L_i, c_i) taken when vol(c_i) <= target, 2i+2 = (c_i, R_i)
// otherwise).  Walking the tree with the totals takes exactly the decisions,
// in the same arithmetic, of the oracle's one-midpoint-per-step loop, so lam
// is unchanged while the grid-wide reductions drop by kOcDepth.
constexpr int kOcDepth = 3;
constexpr int kOcCand = (1 << kOcDepth) - 1;
static_assert(kOcDepth == 3, "the candidate heap below is written out for depth 3");
constexpr int kOcBlock = 1024;   // one block per SM: fewer partials for every block to add

// Cooperative launch (all blocks co-resident) so that blocks may wait on each
// other; the reductions themselves do not use grid.sync.
__global__ void __launch_bounds__(kOcBlock, 1) k_oc_update(const __grid_constant__ OcArgs A, double *part, OcState *S) {
  const int nb = gridDim.x;
  const int64_t tid0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)nb * blockDim.x;
  uint32_t round = 0;
  __shared__ bool s_last;
  __shared__ double s_tot[kOcCand];
  // Grid-wide sums, one round per pass: every block deposits its partials and
  // arrives on a counter; the last to arrive adds the partials in block order
  // (deterministic) and publishes the totals with a release flag that the
  // other blocks acquire.  Totals alternate between two slots by round parity;
  // one partial buffer suffices since a block writes round r+1's partials only
  // after it has acquired round r's flag, i.e. after the last block's reads.
  auto grid_totals = [&](double(&v)[kOcCand]) {
    block_sum<kOcCand>(v);
    if (nb == 1) {   // small meshes: a single block, no grid-level step
      if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < kOcCand; ++k) s_tot[k] = v[k];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kOcCand; ++k) v[k] = s_tot[k];
      __syncthreads();
      ++round;
      return;
    }
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < kOcCand; ++k) __stcg(&part[(size_t)kOcCand * blockIdx.x + k], v[k]);
      __threadfence();
      const uint32_t old = atomicAdd(&S->arrive, 1u);
      s_last = (old == (round + 1) * (uint32_t)nb - 1);
    }
    __syncthreads();
    if (s_last && threadIdx.x < 32) {   // warp 0 of the last block adds the partials
      __threadfence();
      double a[kOcCand];
#pragma unroll
      for (int k = 0; k < kOcCand; ++k) a[k] = 0.0;
      for (int b = threadIdx.x; b < nb; b += 32)
#pragma unroll
        for (int k = 0; k < kOcCand; ++k) a[k] += __ldcg(&part[(size_t)kOcCand * b + k]);
#pragma unroll
      for (int k = 0; k < kOcCand; ++k) a[k] = warp_sum(a[k]);
      if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < kOcCand; ++k) __stcg(&S->tot[round & 1][k], a[k]);
        __threadfence();
        atomicExch(&S->flag, round + 1);
      }
    }
    if (threadIdx.x == 0) {
      while (oc_ld_acquire(&S->flag) < round + 1) __nanosleep(32);
#pragma unroll
      for (int k = 0; k < kOcCand; ++k) s_tot[k] = __ldcg(&S->tot[round & 1][k]);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kOcCand; ++k) v[k] = s_tot[k];
    __syncthreads();
    ++round;
  };
  // vol() at every candidate lam of `cand` in one pass over (x, a)
  auto vols = [&](const double(&cand)[kOcCand], double(&v)[kOcCand]) {
    // t_j = cand_j^-eta once per block (fp64 sqrt/div or pow), broadcast via smem
    __shared__ double s_t[kOcCand];
    if (threadIdx.x < kOcCand) {
      double c = 0.0;
#pragma unroll
      for (int j = 0; j < kOcCand; ++j)
        if (j == (int)threadIdx.x) c = cand[j];
      s_t[threadIdx.x] = oc_pow_neg(c, A.eta);
    }
    __syncthreads();
    double t[kOcCand];
#pragma unroll
    for (int j = 0; j < kOcCand; ++j) {
      t[j] = s_t[j];
      v[j] = 0.0;
    }
    for (int64_t e = tid0; e < A.n; e += stride) {
      const double xe = A.x[e], ae = A.a[e], V = oc_V(A, e);
      const double lo = fmax(A.rho_o, xe - A.move), hi = fmin(1.0, xe + A.move);
#pragma unroll
      for (int j = 0; j < kOcCand; ++j) v[j] = fma(V, fmin(hi, fmax(lo, ae * t[j])), v[j]);
    }
    grid_totals(v);
  };

  // pass 0: a_e, and vol at the lam -> 0+ limit (every loaded element at hi)
  double v[kOcCand];
#pragma unroll
  for (int j = 0; j < kOcCand; ++j) v[j] = 0.0;
  for (int64_t e = tid0; e < A.n; e += stride) {
    const double xe = A.x[e], dce = A.dc[e], V = oc_V(A, e);
    const double g = fmax(-dce, 0.0) / V;
    const double ae = xe * (A.eta == 0.5 ? sqrt(g) : pow(g, A.eta));
    A.a[e] = ae;
    if (!(ae == ae) || !(xe == xe) || !(dce == dce)) v[1] = 1.0;
    v[0] = fma(V, dce < 0.0 ? fmin(1.0, xe + A.move) : fmax(A.rho_o, xe - A.move), v[0]);
  }
  grid_totals(v);
  const double vol0 = v[0];
  int state = 0, steps = 0, passes = 1;
  double t = 0.0, lam = 0.0;   // t = lam^-eta; state 1 uses the limit values
  if (v[1] != 0.0) {
    state = -5;
  } else if (vol0 <= A.target) {
    state = 1;
  } else {
    // bracket: the oracle's  while vol(l2) > target and l2 < 1e300: l2 *= 1e3,
    // kOcCand consecutive upper ends per pass
    double l1 = 0.0, l2 = A.lam_hi;
    bool found = false, capped = false;
    double cand[kOcCand];
    while (!found && !capped) {
      double c = l2;
#pragma unroll
      for (int j = 0; j < kOcCand; ++j) {
        cand[j] = c;
        c *= 1e3;
      }
      vols(cand, v);
      ++passes;
#pragma unroll
      for (int j = 0; j < kOcCand; ++j) {
        if (found || capped) continue;
        l2 = cand[j];
        if (v[j] <= A.target) found = true;
        else if (!(l2 < 1e300)) capped = true;
        else ++steps;
      }
      if (!found && !capped) l2 = cand[kOcCand - 1] * 1e3;
    }
    if (!found) {
      state = 2;
      lam = l2;
    } else {
      int nbis = 0;
      bool done = false;
      while (!done) {
        // candidates of the next 3 bisection levels below (l1, l2), heap order
        cand[0] = 0.5 * (l1 + l2);
        cand[1] = 0.5 * (l1 + cand[0]);
        cand[2] = 0.5 * (cand[0] + l2);
        cand[3] = 0.5 * (l1 + cand[1]);
        cand[4] = 0.5 * (cand[1] + cand[0]);
        cand[5] = 0.5 * (cand[0] + cand[2]);
        cand[6] = 0.5 * (cand[2] + l2);
        if (!(nbis < A.max_steps && !(l2 - l1 <= A.tol * (l1 + l2)))) break;
        vols(cand, v);
        ++passes;
        int i = 0;
        for (int d = 0; d < kOcDepth; ++d) {
          if (!(nbis < A.max_steps && !(l2 - l1 <= A.tol * (l1 + l2)))) { done = true; break; }
          double vi = 0.0, ci = 0.0;   // v[i], cand[i] without dynamic register indexing
#pragma unroll
          for (int j = 0; j < kOcCand; ++j)
            if (j == i) {
              vi = v[j];
              ci = cand[j];
            }
          const bool right = vi > A.target;
          if (right) l1 = ci; else l2 = ci;
          ++nbis;
          i = right ? 2 * i + 2 : 2 * i + 1;
        }
      }
      steps += nbis;
      lam = 0.5 * (l1 + l2);
    }
    t = oc_pow_neg(lam, A.eta);
  }
  // final pass: x_new, its volume and the design change (Condition 1)
  double vs = 0.0, ch = 0.0;
  if (state >= 0) {
    for (int64_t e = tid0; e < A.n; e += stride) {
      const double xe = A.x[e];
      const double xne = state == 1 ? (A.dc[e] < 0.0 ? fmin(1.0, xe + A.move) : fmax(A.rho_o, xe - A.move))
                                    : oc_clamp(xe, A.a[e] * t, A);
      A.xn[e] = xne;
      vs = fma(oc_V(A, e), xne, vs);
      ch = fmax(ch, fabs(xne - xe));
    }
  }
  ch = oc_block_max(ch);
  if (threadIdx.x == 0) atomicMax(&S->change_bits, (unsigned long long)__double_as_longlong(ch));
#pragma unroll
  for (int j = 0; j < kOcCand; ++j) v[j] = 0.0;
  v[0] = vs;
  grid_totals(v);   // the arrivals order the change maxima before the last block reads them
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    S->lam = lam;
    S->volume_abs = v[0];
    S->change = __longlong_as_double((long long)atomicAdd(&S->change_bits, 0ull));
    S->steps = steps;
    S->state = state;
    S->passes = passes + 1;
  }
}

}  // namespace tomesh
