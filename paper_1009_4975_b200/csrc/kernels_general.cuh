// General (unstructured, AMR) kernels of the hot path.  Work from the
// canonical flat arrays: elem_node, per-node hanging index, hanging CSR.
//
//   k_simp        a1  s_e = (E_min + x_e^p (E0 - E_min)) h_e^(d-2)       (Eq. 2)
//   k_diag_*      a2  D = diag(Pi_F C^T K C Pi_F) (cross terms included)  (:515-521)
//   k_rhs         a3  b = Pi_F C^T f                                      (Eq. 7 rhs)
//   (one PCG iteration, a4-a7: kernels_genfused.cuh)                        (Eq. 8)
//   k_recover     a8  u = C u_hat                                         (Eq. 9)
//   k_sens        a10 dc_e = -p x^(p-1)(E0-Emin) h^(d-2) u_e^T K0 u_e    (:343-346)
//   k_filter      a11 Eq. 5 / density variant                             (:613-616)
#pragma once
#include <cooperative_groups.h>

#include "device_common.cuh"
#include "element.h"
#include "kernels_cg.cuh"
#include "tomesh_types.cuh"

namespace tomesh {


template <int DIM>
__global__ void k_simp(int64_t n, const double *__restrict__ x, const int8_t *__restrict__ lev,
                       double penal, double E0, double Emin, int L, double hL,
                       double *__restrict__ s, CgScalars *S) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double xe = x[e];
    if (!(xe > 0.0) || !(xe <= 1.0)) cg_fail(S, -1);  // TO_EINVAL
    double v = Emin + pow(xe, penal) * (E0 - Emin);
    if (DIM == 3) v *= hL * (double)(1 << (L - lev[e]));
    s[e] = v;
  }
}

// ---- Jacobi diagonal (a2) ---------------------------------------------------------
// D_(n,i) = sum_e s_e sum_{a,b} w_a w_b K0[(a,i),(b,i)] over the corners a, b of
// element e that map to node n (directly with w = 1, or as a hanging corner
// with its Eq. 6 weight): the diagonal of C^T K C with the cross terms of two
// hanging corners sharing a parent (reading Q4).  Node-centric over the
// incidence CSR (entries of one element are consecutive): no atomics, so D is
// bit-reproducible.
template <int DIM>
__global__ void k_diag_node(int64_t n_node, const int64_t *__restrict__ inc_ptr, const uint32_t *__restrict__ inc,
                            const double *__restrict__ s,
                            const __grid_constant__ typename std::conditional<DIM == 2, K0Dense2, K0Dense3>::type K0,
                            double *__restrict__ D) {
  constexpr int NC = 1 << DIM, ND = DIM * NC;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_node; n += (int64_t)gridDim.x * blockDim.x) {
    double acc[DIM];
#pragma unroll
    for (int i = 0; i < DIM; ++i) acc[i] = 0.0;
    const int64_t k1 = inc_ptr[n + 1];
    int64_t k = inc_ptr[n];
    while (k < k1) {
      const uint32_t e = (inc[k] & 0x3fffffffu) / NC;
      int64_t kend = k;
      while (kend < k1 && (inc[kend] & 0x3fffffffu) / NC == e) ++kend;   // this element's corners
      double el[DIM];
#pragma unroll
      for (int i = 0; i < DIM; ++i) el[i] = 0.0;
      for (int64_t a = k; a < kend; ++a)
        for (int64_t b = k; b < kend; ++b) {
          const uint32_t ta = inc[a], tb = inc[b];
          const int ca = (int)((ta & 0x3fffffffu) % NC), cb = (int)((tb & 0x3fffffffu) % NC);
          const double wa = (ta >> 30) == 0 ? 1.0 : (ta >> 30) == 1 ? 0.5 : 0.25;
          const double wb = (tb >> 30) == 0 ? 1.0 : (tb >> 30) == 1 ? 0.5 : 0.25;
#pragma unroll
          for (int i = 0; i < DIM; ++i) el[i] += wa * wb * K0.K[(DIM * ca + i) * ND + DIM * cb + i];
        }
      const double se = s[e];
#pragma unroll
      for (int i = 0; i < DIM; ++i) acc[i] = fma(se, el[i], acc[i]);
      k = kend;
    }
#pragma unroll
    for (int i = 0; i < DIM; ++i) D[n * DIM + i] = acc[i];
  }
}

// Dinv = 1/D on free DOFs, 0 elsewhere (the zero doubles as the free mask of the
// CG loop); d_out (optional) = diag(A) with 1 on non-free DOFs.
static __global__ void k_dinv(int64_t ndof, const uint8_t *__restrict__ free_dof, const double *__restrict__ D,
                       double *__restrict__ Dinv, double *__restrict__ d_out, CgScalars *S) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ndof; i += (int64_t)gridDim.x * blockDim.x) {
    double d = D[i];
    if (free_dof[i]) {
      if (!(d > 0.0)) cg_fail(S, -7);  // TO_ENONPOS_DIAG
      if (Dinv) Dinv[i] = 1.0 / d;
      if (d_out) d_out[i] = d;
    } else {
      if (Dinv) Dinv[i] = 0.0;
      if (d_out) d_out[i] = 1.0;
    }
  }
}

// ---- rhs b = Pi_F C^T f (a3), deterministic via the parent->children CSR ------------
template <int DIM>
__global__ void k_rhs(MeshView M, const double *__restrict__ f, double *__restrict__ b) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < M.n_node; n += (int64_t)gridDim.x * blockDim.x) {
    for (int i = 0; i < DIM; ++i) {
      int64_t dof = n * DIM + i;
      double v = 0.0;
      if (M.free_dof[dof]) {
        v = f[dof];
        if (M.child_ptr)
          for (int k = M.child_ptr[n]; k < M.child_ptr[n + 1]; ++k)
            v += M.child_weight[k] * f[(int64_t)M.child_hang[k] * DIM + i];
      }
      b[dof] = v;
    }
  }
}

// ---- recovery u = C v (a8) --------------------------------------------------------------
template <int DIM>
__global__ void k_recover(MeshView M, const double *__restrict__ v, double *__restrict__ u) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < M.n_node; n += (int64_t)gridDim.x * blockDim.x) {
    int h = M.node_hang[n];
    for (int i = 0; i < DIM; ++i) {
      double val;
      if (h < 0) {
        val = v[n * DIM + i];
      } else {
        val = 0.0;
        for (int k = M.hang_ptr[h]; k < M.hang_ptr[h + 1]; ++k)
          val += M.hang_weight[k] * v[(int64_t)M.hang_parent[k] * DIM + i];
      }
      u[n * DIM + i] = val;
    }
  }
}

// ---- element gather through C (hanging corners interpolated) ------------------------
template <int DIM>
__device__ __forceinline__ void gather_C(const MeshView &M, int64_t e, const double *__restrict__ p,
                                         double (&ue)[DIM << DIM], int (&node)[1 << DIM], int (&hang)[1 << DIM]) {
  constexpr int NC = 1 << DIM;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    int n = M.elem_node[e * NC + c];
    int h = M.node_hang[n];
    node[c] = n;
    hang[c] = h;
    if (h < 0) {
#pragma unroll
      for (int i = 0; i < DIM; ++i) ue[DIM * c + i] = p[(int64_t)n * DIM + i];
    } else {
      double acc[DIM];
#pragma unroll
      for (int i = 0; i < DIM; ++i) acc[i] = 0.0;
      for (int k = M.hang_ptr[h]; k < M.hang_ptr[h + 1]; ++k) {
        double w = M.hang_weight[k];
        int64_t pn = M.hang_parent[k];
#pragma unroll
        for (int i = 0; i < DIM; ++i) acc[i] += w * p[pn * DIM + i];
      }
#pragma unroll
      for (int i = 0; i < DIM; ++i) ue[DIM * c + i] = acc[i];
    }
  }
}

template <int ND>
__device__ __forceinline__ void dense_apply(const double *__restrict__ K, const double (&x)[ND], double (&y)[ND]) {
#pragma unroll
  for (int a = 0; a < ND; ++a) {
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < ND; ++b) acc = fma(K[a * ND + b], x[b], acc);
    y[a] = acc;
  }
}

// In-place Walsh-Hadamard transform over the 8 corners of each component.
__device__ __forceinline__ void wht8x3(double (&v)[24]) {
#pragma unroll
  for (int bit = 1; bit < 8; bit <<= 1) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c & bit) continue;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double a = v[3 * c + i], b = v[3 * (c | bit) + i];
        v[3 * c + i] = a + b;
        v[3 * (c | bit) + i] = a - b;
      }
    }
  }
}

// One output of the Hadamard-basis product: yhat(m,i) = diag[i][m] xhat(m,i) +
// sum_{j != i, bit_i(m) != bit_j(m)} off[i][j][m] xhat(m ^ e_i ^ e_j, j).
__device__ __forceinline__ double had_mid_one(const K0Had3 &H, const double (&x)[24], int m, int i) {
  double acc = H.diag[i][m] * x[3 * m + i];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    if (j == i || ((m >> i) & 1) == ((m >> j) & 1)) continue;
    acc = fma(H.off[i][j][m], x[3 * (m ^ ((1 << i) | (1 << j))) + j], acc);
  }
  return acc;
}

// xhat := Khat xhat in place.  The coupling (m,i) -> (m ^ e_i ^ e_j, j) splits
// the 24 Hadamard coordinates into closed groups: two triples, six pairs,
// three singletons (m = 7) and the rigid-translation mode m = 0, whose
// output is zero.  Each group is evaluated from its inputs before it is
// written back, so no second 24-vector is live (register pressure).
template <typename HC>
__device__ __forceinline__ void had_mid_inplace(const HC &H, double (&x)[24]) {
#define HAD_G3(m0, i0, m1, i1, m2, i2)                                                                      \
  {                                                                                                         \
    const double a = had_mid_one(H, x, m0, i0), b = had_mid_one(H, x, m1, i1), c = had_mid_one(H, x, m2, i2); \
    x[3 * m0 + i0] = a;                                                                                     \
    x[3 * m1 + i1] = b;                                                                                     \
    x[3 * m2 + i2] = c;                                                                                     \
  }
#define HAD_G2(m0, i0, m1, i1)                                                   \
  {                                                                              \
    const double a = had_mid_one(H, x, m0, i0), b = had_mid_one(H, x, m1, i1); \
    x[3 * m0 + i0] = a;                                                          \
    x[3 * m1 + i1] = b;                                                          \
  }
  HAD_G3(1, 0, 2, 1, 4, 2)
  HAD_G2(1, 1, 2, 0)
  HAD_G2(1, 2, 4, 0)
  HAD_G2(2, 2, 4, 1)
  HAD_G3(6, 0, 5, 1, 3, 2)
  HAD_G2(6, 1, 5, 0)
  HAD_G2(6, 2, 3, 0)
  HAD_G2(5, 2, 3, 1)
#pragma unroll
  for (int i = 0; i < 3; ++i) x[21 + i] = had_mid_one(H, x, 7, i);
  x[0] = x[1] = x[2] = 0.0;
#undef HAD_G3
#undef HAD_G2
}

// Same products with the 9 class values of the coefficients (element.h
// K0HadSym): the compiler keeps 9 doubles live instead of reloading 45.
__device__ __forceinline__ double had_mid_one(const K0HadSym &H, const double (&x)[24], int m, int i) {
  const int b = (m >> i) & 1;
  const int n = (m & 1) + ((m >> 1) & 1) + ((m >> 2) & 1) - b;
  double acc = H.d[b][n] * x[3 * m + i];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    if (j == i || ((m >> j) & 1) == b) continue;
    acc = fma(H.o[b][(m >> (3 - i - j)) & 1], x[3 * (m ^ ((1 << i) | (1 << j))) + j], acc);
  }
  return acc;
}

// In-place middle product that also accumulates x^T K0 x = sum xhat . yhat
// (K0 = H Khat H with the 1/64 folded into Khat), group by group.
template <typename HC>
__device__ __forceinline__ void had_mid_inplace_energy(const HC &H, double (&x)[24], double &en) {
#define HAD_E3(m0, i0, m1, i1, m2, i2)                                                                      \
  {                                                                                                         \
    const double a = had_mid_one(H, x, m0, i0), b = had_mid_one(H, x, m1, i1), c = had_mid_one(H, x, m2, i2); \
    en = fma(a, x[3 * m0 + i0], fma(b, x[3 * m1 + i1], fma(c, x[3 * m2 + i2], en)));                         \
    x[3 * m0 + i0] = a;                                                                                     \
    x[3 * m1 + i1] = b;                                                                                     \
    x[3 * m2 + i2] = c;                                                                                     \
  }
#define HAD_E2(m0, i0, m1, i1)                                                   \
  {                                                                              \
    const double a = had_mid_one(H, x, m0, i0), b = had_mid_one(H, x, m1, i1); \
    en = fma(a, x[3 * m0 + i0], fma(b, x[3 * m1 + i1], en));                     \
    x[3 * m0 + i0] = a;                                                          \
    x[3 * m1 + i1] = b;                                                          \
  }
  HAD_E3(1, 0, 2, 1, 4, 2)
  HAD_E2(1, 1, 2, 0)
  HAD_E2(1, 2, 4, 0)
  HAD_E2(2, 2, 4, 1)
  HAD_E3(6, 0, 5, 1, 3, 2)
  HAD_E2(6, 1, 5, 0)
  HAD_E2(6, 2, 3, 0)
  HAD_E2(5, 2, 3, 1)
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double a = had_mid_one(H, x, 7, i);
    en = fma(a, x[21 + i], en);
    x[21 + i] = a;
  }
  x[0] = x[1] = x[2] = 0.0;
#undef HAD_E3
#undef HAD_E2
}

// x := K0 x for H8 via the Hadamard factorisation (element.h), in place.
template <typename HC>
__device__ __forceinline__ void had_apply_inplace(const HC &H, double (&x)[24]) {
  wht8x3(x);
  had_mid_inplace(H, x);
  wht8x3(x);
}

// y = K0 x (x is destroyed).
__device__ __forceinline__ void had_apply(const K0Had3 &H, double (&x)[24], double (&y)[24]) {
  had_apply_inplace(H, x);
#pragma unroll
  for (int a = 0; a < 24; ++a) y[a] = x[a];
}

// ---- grid-wide sums inside a cooperative kernel ---------------------------------------
enum { G_PLAIN = 0, G_CG = 1 };

// Sum of the per-block partials, computed by warp 0 of every block in the same
// fixed order (lane-strided partial sums, then the xor-shuffle tree) and
// broadcast through shared memory: every block obtains bit-identical totals.
template <int NV>
__device__ __forceinline__ void g_sum_partials(const double *part, int nb, double (&out)[NV]) {
  if (nb <= 32) {                                       // small grids: every thread, same order
#pragma unroll
    for (int k = 0; k < NV; ++k) out[k] = 0.0;
    for (int b = 0; b < nb; ++b)
#pragma unroll
      for (int k = 0; k < NV; ++k) out[k] += __ldcg(&part[NV * b + k]);
    return;
  }
  __shared__ double bc[NV];
  if (threadIdx.x < 32) {
    double a[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) a[k] = 0.0;
    for (int b = threadIdx.x; b < nb; b += 32)
#pragma unroll
      for (int k = 0; k < NV; ++k) a[k] += __ldcg(&part[NV * b + k]);
#pragma unroll
    for (int k = 0; k < NV; ++k) a[k] = warp_sum(a[k]);
    if (threadIdx.x == 0)
#pragma unroll
      for (int k = 0; k < NV; ++k) bc[k] = a[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = bc[k];
  __syncthreads();
}

// ---- sensitivities (a10) ----------------------------------------------------------------
// 3D: u_e^T K0 u_e from the Hadamard middle product (sum xhat . yhat).
static __global__ void __launch_bounds__(256) k_sens_had3(MeshView M, const double *__restrict__ x,
                                                   const double *__restrict__ u, double penal, double E0, double Emin,
                                                   double *__restrict__ dc, const __grid_constant__ K0HadSym H) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M.n_el; e += (int64_t)gridDim.x * blockDim.x) {
    double ue[24];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int64_t n = M.elem_node[e * 8 + c];
#pragma unroll
      for (int i = 0; i < 3; ++i) ue[3 * c + i] = u[n * 3 + i];
    }
    wht8x3(ue);
    double en = 0.0;
    had_mid_inplace_energy(H, ue, en);
    const double h = M.hL * (double)(1 << (M.L - M.elem_level[e]));
    const double xe = x[e];
    dc[e] = -penal * pow(xe, penal - 1.0) * (E0 - Emin) * h * en;
  }
}

template <int DIM>
__global__ void k_sens(MeshView M, const double *__restrict__ x, const double *__restrict__ u, double penal,
                       double E0, double Emin, double *__restrict__ dc,
                       const __grid_constant__ typename std::conditional<DIM == 2, K0Dense2, K0Dense3>::type K0) {
  constexpr int NC = 1 << DIM, ND = DIM * NC;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M.n_el; e += (int64_t)gridDim.x * blockDim.x) {
    double ue[ND], ye[ND];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      int64_t n = M.elem_node[e * NC + c];
#pragma unroll
      for (int i = 0; i < DIM; ++i) ue[DIM * c + i] = u[n * DIM + i];
    }
    dense_apply<ND>(K0.K, ue, ye);
    double en = 0.0;
#pragma unroll
    for (int a = 0; a < ND; ++a) en = fma(ue[a], ye[a], en);
    double h = (DIM == 3) ? M.hL * (double)(1 << (M.L - M.elem_level[e])) : 1.0;
    double xe = x[e];
    dc[e] = -penal * pow(xe, penal - 1.0) * (E0 - Emin) * h * en;
  }
}

// ---- filter (a11) -------------------------------------------------------------------------
template <int DIM>
__global__ void k_filter(MeshView M, const int64_t *__restrict__ fptr, const int32_t *__restrict__ fidx,
                         double rmin, int mode, const double *__restrict__ x, const double *__restrict__ in,
                         double *__restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M.n_el; e += (int64_t)gridDim.x * blockDim.x) {
    double ce[DIM];
    const double se = (double)(1 << (M.L - M.elem_level[e]));
#pragma unroll
    for (int c = 0; c < DIM; ++c) ce[c] = ((double)M.elem_anchor[e * DIM + c] + 0.5 * se) * M.hL;
    double num = 0.0, den = 0.0;
    for (int64_t k = fptr[e]; k < fptr[e + 1]; ++k) {
      int64_t d = fidx[k];
      const double sd = (double)(1 << (M.L - M.elem_level[d]));
      double d2 = 0.0;
#pragma unroll
      for (int c = 0; c < DIM; ++c) {
        double df = ((double)M.elem_anchor[d * DIM + c] + 0.5 * sd) * M.hL - ce[c];
        d2 += df * df;
      }
      double H = fmax(rmin - sqrt(d2), 0.0);
      double V = sd * M.hL;
      V = (DIM == 2) ? V * V : V * V * V;
      double w = H * V;
      num += (mode == 0) ? w * (x[d] * in[d]) : w * in[d];
      den += w;
    }
    out[e] = (mode == 0) ? num / (x[e] * den) : num / den;
  }
}

// Dynamic AMR marking (reading R21): +1 when a solid
// element (x >= rho_s) lies in e's neighbour list (|c_d - c_e| < r_amr =
// rmin, self included), else -1; refinement capped at level L, derefinement
// at level 0.  Integer output, no floating-point decisions beyond x >= rho_s.
static __global__ void k_amr_mark(int64_t n_el, const int8_t *__restrict__ level, int L, const int64_t *__restrict__ fptr,
                           const int32_t *__restrict__ fidx, const double *__restrict__ x, double rho_s,
                           int8_t *__restrict__ marks) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x) {
    bool near = false;
    if (fptr) {
      for (int64_t k = fptr[e]; k < fptr[e + 1] && !near; ++k) near = x[fidx[k]] >= rho_s;
    } else {
      near = x[e] >= rho_s;
    }
    const int l = level[e];
    marks[e] = near ? (l < L ? 1 : 0) : (l > 0 ? -1 : 0);
  }
}

}  // namespace tomesh
