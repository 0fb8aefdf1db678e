// Zero-fill incomplete Cholesky of the rescaled matrix K~ = D^-1/2 A D^-1/2
// ("an incomplete Cholesky preconditioner with zero
// fill-in to the explicitly rescaled system"), shifted on breakdown
// (reading R24), for MINRES (kernels_minres.cuh).  General
// (canonical DOF order) handles only; the order is the oracle's.
//
// The lower pattern and, per nonzero, the list of element contributions
// (element, local DOF pair, Eq. 6 weight product) are built once on the host;
// per solve:
//   k_ic0_assemble   K~_ij (+ shift on the diagonal) = s_i s_j sum w s_e K0[a][b]
//                    in a fixed order (deterministic, no atomics)
//   k_ic0_factor     one launch per dependency level, one thread per row:
//                    L_ik = (K~_ik - sum_{j<k} L_ij L_kj) / L_kk,
//                    L_ii = sqrt(K~_ii - sum L_ik^2); a non-positive pivot
//                    raises the breakdown flag (the host retries with a shift)
//   k_ic0_fwd/bwd    L y = v and L^T z = y, level-scheduled inside ONE CTA
//                    (a warp per row, __syncthreads between levels): the solves are
//                    sequential chains of short rows, the dependency depth,
//                    not bandwidth, bounds them — the reason the B200 path
//                    keeps the plain rescaling.
#pragma once
#include "device_common.cuh"
#include "tomesh_types.cuh"

namespace tomesh {


template <int DIM>
__global__ void k_ic0_assemble(Ic0View V, const double *__restrict__ s, const double *__restrict__ msc,
                               const double *__restrict__ K0, double shift, double *__restrict__ kt) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < V.nnz; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = V.row[t], j = V.col[t];
    double a = 0.0;
    for (int64_t u = V.cptr[t]; u < V.cptr[t + 1]; ++u) {
      const uint64_t c = V.contrib[u];
      const int64_t e = (int64_t)(c >> 16);
      const int ab = (int)((c >> 3) & 0x1fff);
      const double w = ldexp(1.0, -(int)(c & 7));
      a += w * K0[ab] * s[e];
    }
    double v;
    if (V.cptr[t] == V.cptr[t + 1]) v = (i == j) ? 1.0 : 0.0;   // a non-free row: unit diagonal
    else v = __dmul_rn(__dmul_rn(msc[i], a), msc[j]);
    if (i == j) v += shift;
    kt[t] = v;
  }
}

// rows lvl_rows[r0 .. r1) (one dependency level)
__global__ void k_ic0_factor(Ic0View V, const int32_t *__restrict__ lvl_rows, int64_t r0, int64_t r1,
                             double *__restrict__ L, int *fail) {
  for (int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r1; r += (int64_t)gridDim.x * blockDim.x) {
    const int i = lvl_rows[r];
    const int64_t a = V.ptr[i], b = V.ptr[i + 1];
    for (int64_t t = a; t < b - 1; ++t) {
      const int k = V.col[t];
      double acc = L[t];
      const int64_t ka = V.ptr[k], kb = V.ptr[k + 1];
      // j < k common to rows i and k: merge of the two ascending column lists
      int64_t pk = ka;
      for (int64_t u = a; u < t; ++u) {
        const int j = V.col[u];
        while (pk < kb - 1 && V.col[pk] < j) ++pk;
        if (pk < kb - 1 && V.col[pk] == j) acc = __dsub_rn(acc, __dmul_rn(L[u], L[pk]));
      }
      L[t] = __ddiv_rn(acc, L[kb - 1]);
    }
    double d = L[b - 1];
    for (int64_t u = a; u < b - 1; ++u) d = __dsub_rn(d, __dmul_rn(L[u], L[u]));
    if (!(d > 0.0)) {
      atomicExch(fail, 1);
      d = 1.0;
    }
    L[b - 1] = sqrt(d);
  }
}

// L y = v, one CTA, levels in order; a warp per row (lanes split the row's
// entries, xor-shuffle sum)
__global__ void __launch_bounds__(1024) k_ic0_fwd(Ic0View V, const int64_t *__restrict__ lvl_ptr, int n_lvl,
                                                  const int32_t *__restrict__ lvl_rows, const double *__restrict__ L,
                                                  const double *__restrict__ v, double *__restrict__ y) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int l = 0; l < n_lvl; ++l) {
    for (int64_t r = lvl_ptr[l] + warp; r < lvl_ptr[l + 1]; r += nw) {
      const int i = lvl_rows[r];
      const int64_t a = V.ptr[i], b = V.ptr[i + 1];
      double acc = 0.0;
      for (int64_t t = a + lane; t < b - 1; t += 32) acc = fma(L[t], __ldcg(&y[V.col[t]]), acc);
      acc = warp_sum(acc);
      if (lane == 0) __stcg(&y[i], (v[i] - acc) / L[b - 1]);
    }
    __syncthreads();
  }
}

// L^T z = y through the transposed pattern (rows of L^T: the entries below
// the diagonal in column k of L), levels in order, a warp per row
__global__ void __launch_bounds__(1024) k_ic0_bwd(Ic0View V, const int64_t *__restrict__ ut_ptr,
                                                  const int32_t *__restrict__ ut_row, const int64_t *__restrict__ ut_pos,
                                                  const int64_t *__restrict__ lvl_ptr, int n_lvl,
                                                  const int32_t *__restrict__ lvl_rows, const double *__restrict__ L,
                                                  const double *__restrict__ y, double *__restrict__ z) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int l = 0; l < n_lvl; ++l) {
    for (int64_t r = lvl_ptr[l] + warp; r < lvl_ptr[l + 1]; r += nw) {
      const int k = lvl_rows[r];
      double acc = 0.0;
      for (int64_t t = ut_ptr[k] + lane; t < ut_ptr[k + 1]; t += 32)
        acc = fma(L[ut_pos[t]], __ldcg(&z[ut_row[t]]), acc);
      acc = warp_sum(acc);
      if (lane == 0) __stcg(&z[k], (y[k] - acc) / L[V.ptr[k + 1] - 1]);
    }
    __syncthreads();
  }
}

}  // namespace tomesh
