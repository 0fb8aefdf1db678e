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
//   k_ic0_tri        L y = v and L^T z = y, level-scheduled inside ONE CTA
//                    (a warp per row, __syncthreads between levels, the rows'
//                    static data software-pipelined three levels ahead): the
//                    solves are sequential chains of short rows, the
//                    dependency depth, not bandwidth, bounds them — the reason
//                    the B200 path keeps the plain rescaling.
#pragma once
#include "device_common.cuh"
#include "tomesh_types.cuh"

namespace tomesh {

constexpr int kIc0Warps = 32;   // most warps of the one-CTA triangular solves (= rows per step); per mesh: to_mesh::ic_warps

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

// L y = v (BWD = false) and L^T z = y (BWD = true), one CTA, levels in order,
// a warp per row (lanes split the row's entries, xor-shuffle sum).  The
// static data of a row (its index, pointers, coefficients and column
// indices, right-hand side and pivot) does not depend on the solution, so
// each warp loads it through a 3-level-deep software pipeline: at level l it
// loads the row index of level l+3, the row pointers of level l+2 and the
// entries of level l+1, all independent of one another.  What is left on the
// critical path of a level is the gather of the solution entries, the warp
// sum, the division and the CTA barrier (round 1: four dependent loads per
// level, ~2.7 us; the arithmetic and its order are unchanged).  The host
// hands over the levels cut into steps of at most blockDim / 32 rows, so every
// row is a warp's first of its step; entries beyond 64 of a row (and rows
// beyond the first, if a caller passes whole levels) take the plain loop.
//   BWD: the rows of L^T through the transposed pattern (ut_ptr, ut_row,
//   ut_pos: the entries below the diagonal in column k of L).
template <bool BWD>
__global__ void __launch_bounds__(1024) k_ic0_tri(Ic0View V, const int64_t *__restrict__ ut_ptr,
                                                  const int32_t *__restrict__ ut_row, const int64_t *__restrict__ ut_pos,
                                                  const int64_t *__restrict__ lvl_ptr, int n_lvl,
                                                  const int32_t *__restrict__ lvl_rows, const double *__restrict__ L,
                                                  const double *__restrict__ rhs, double *__restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  auto lp = [&](int j) { return __ldg(&lvl_ptr[min(max(j, 0), n_lvl)]); };
  // one row, start to end, nothing prefetched
  auto plain_row = [&](int i) {
    const int64_t a = BWD ? ut_ptr[i] : V.ptr[i];
    const int64_t dpos = V.ptr[i + 1] - 1;
    const int64_t e = BWD ? ut_ptr[i + 1] : dpos;
    double acc = 0.0;
    for (int64_t t = a + lane; t < e; t += 32)
      acc = BWD ? fma(L[ut_pos[t]], __ldcg(&out[ut_row[t]]), acc) : fma(L[t], __ldcg(&out[V.col[t]]), acc);
    acc = warp_sum(acc);
    if (lane == 0) __stcg(&out[i], (rhs[i] - acc) / L[dpos]);
  };
  // pipeline registers: w_j = first row position of level l + j
  int64_t w0 = 0, w1 = 0, w2 = 0, w3 = lp(0), w4 = lp(1);
  int i2 = -1;                                            // level l+2: row index
  int i1 = -1;                                            // level l+1: row index, pointers
  int64_t a1 = 0, e1 = 0, d1 = 0;
  int i0 = -1;                                            // level l: row index, pointers, first 2 entries per lane
  int64_t a0 = 0, e0 = 0;
  double c0a = 0.0, c0b = 0.0, rh0 = 0.0, dg0 = 1.0;
  int64_t q0a = 0, q0b = 0;                               // BWD: positions in L of the two entries
  int x0a = -1, x0b = -1;
  for (int l = -3; l < n_lvl; ++l) {
    // ---- loads for the levels ahead (independent of the solution) ----
    const int64_t w5 = lp(l + 5);
    const int i3 = (l + 3 < n_lvl && w3 + warp < w4) ? __ldg(&lvl_rows[w3 + warp]) : -1;
    int64_t a2 = 0, e2 = 0, d2 = 0;
    if (i2 >= 0) {
      d2 = __ldg(&V.ptr[i2 + 1]) - 1;
      a2 = BWD ? __ldg(&ut_ptr[i2]) : __ldg(&V.ptr[i2]);
      e2 = BWD ? __ldg(&ut_ptr[i2 + 1]) : d2;
    }
    double n_ca = 0.0, n_cb = 0.0, n_rh = 0.0, n_dg = 1.0;
    int64_t n_qa = 0, n_qb = 0;
    int n_xa = -1, n_xb = -1;
    if (i1 >= 0) {
      const int64_t ta = a1 + lane, tb = ta + 32;
      if (ta < e1) {
        if (BWD) {
          n_qa = __ldg(&ut_pos[ta]);
          n_xa = __ldg(&ut_row[ta]);
        } else {
          n_ca = L[ta];
          n_xa = __ldg(&V.col[ta]);
        }
      }
      if (tb < e1) {
        if (BWD) {
          n_qb = __ldg(&ut_pos[tb]);
          n_xb = __ldg(&ut_row[tb]);
        } else {
          n_cb = L[tb];
          n_xb = __ldg(&V.col[tb]);
        }
      }
      if (lane == 0) {
        n_rh = rhs[i1];
        n_dg = L[d1];
      }
    }
    // ---- level l ----
    if (l >= 0) {
      if (i0 >= 0) {
        double acc = 0.0;
        if (BWD) {
          if (x0a >= 0) acc = fma(L[q0a], __ldcg(&out[x0a]), acc);
          if (x0b >= 0) acc = fma(L[q0b], __ldcg(&out[x0b]), acc);
        } else {
          if (x0a >= 0) acc = fma(c0a, __ldcg(&out[x0a]), acc);
          if (x0b >= 0) acc = fma(c0b, __ldcg(&out[x0b]), acc);
        }
        for (int64_t t = a0 + 64 + lane; t < e0; t += 32)
          acc = BWD ? fma(L[ut_pos[t]], __ldcg(&out[ut_row[t]]), acc) : fma(L[t], __ldcg(&out[V.col[t]]), acc);
        acc = warp_sum(acc);
        if (lane == 0) __stcg(&out[i0], (rh0 - acc) / dg0);
      }
      for (int64_t r = w0 + warp + nw; r < w1; r += nw) plain_row(lvl_rows[r]);
      __syncthreads();
    }
    // ---- rotate ----
    i0 = i1, a0 = a1, e0 = e1;
    c0a = n_ca, c0b = n_cb, q0a = n_qa, q0b = n_qb, x0a = n_xa, x0b = n_xb, rh0 = n_rh, dg0 = n_dg;
    i1 = i2, a1 = a2, e1 = e2, d1 = d2;
    i2 = i3;
    w0 = w1, w1 = w2, w2 = w3, w3 = w4, w4 = w5;
  }
}

}  // namespace tomesh
