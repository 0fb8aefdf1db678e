// General (unstructured, AMR) kernels of the hot path.  Work from the
// canonical flat arrays: elem_node, per-node hanging index, hanging CSR.
//
//   k_simp        a1  s_e = (E_min + x_e^p (E0 - E_min)) h_e^(d-2)       (Eq. 2)
//   k_diag_*      a2  D = diag(Pi_F C^T K C Pi_F) (cross terms included)  (:515-521)
//   k_rhs         a3  b = Pi_F C^T f                                      (Eq. 7 rhs)
//   k_matvec_*    a4  q = C^T K C p for p vanishing on non-free DOFs       (Eq. 8)
//   k_recover     a8  u = C u_hat                                         (Eq. 9)
//   k_sens        a10 dc_e = -p x^(p-1)(E0-Emin) h^(d-2) u_e^T K0 u_e    (:343-346)
//   k_filter      a11 Eq. 5 / density variant                             (:613-616)
#pragma once
#include "device_common.cuh"
#include "element.h"

namespace tomesh {

struct MeshView {
  int64_t n_el, n_node;
  const int32_t *elem_node;     // [n_el][NC]
  const int8_t *elem_level;
  const int32_t *elem_anchor;   // [n_el][DIM]
  const int32_t *node_hang;     // [n_node] index into hang rows or -1
  const int32_t *hang_ptr, *hang_parent;
  const double *hang_weight;
  const int32_t *child_ptr, *child_hang;  // transpose: parent node -> hanging children
  const double *child_weight;
  const uint8_t *free_dof;      // [n_dof] 1 = neither hanging nor fixed
  int L;
  double hL;
};

template <int DIM>
__global__ void k_simp(int64_t n, const double *__restrict__ x, const int8_t *__restrict__ lev,
                       double penal, double E0, double Emin, int L, double hL,
                       double *__restrict__ s, CgScalars *S) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double xe = x[e];
    if (!(xe > 0.0) || !(xe <= 1.0)) S->status = -1;  // TO_EINVAL
    double v = Emin + pow(xe, penal) * (E0 - Emin);
    if (DIM == 3) v *= hL * (double)(1 << (L - lev[e]));
    s[e] = v;
  }
}

// ---- Jacobi diagonal (a2) ---------------------------------------------------------
template <int DIM>
__global__ void k_diag(MeshView M, const double *__restrict__ s, double *__restrict__ D,
                       const __grid_constant__ typename std::conditional<DIM == 2, K0Dense2, K0Dense3>::type K0) {
  constexpr int NC = 1 << DIM, ND = DIM * NC;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M.n_el; e += (int64_t)gridDim.x * blockDim.x) {
    const double se = s[e];
    int tgt[NC * 4], cor[NC * 4];
    double w[NC * 4];
    int nt = 0;
    bool any_h = false;
    for (int c = 0; c < NC; ++c) {
      int n = M.elem_node[e * NC + c];
      int h = M.node_hang[n];
      if (h < 0) {
        tgt[nt] = n; cor[nt] = c; w[nt] = 1.0; ++nt;
      } else {
        any_h = true;
        for (int k = M.hang_ptr[h]; k < M.hang_ptr[h + 1]; ++k) {
          tgt[nt] = M.hang_parent[k]; cor[nt] = c; w[nt] = M.hang_weight[k]; ++nt;
        }
      }
    }
    if (!any_h) {
      for (int c = 0; c < NC; ++c)
        for (int i = 0; i < DIM; ++i)
          atomicAdd(&D[(int64_t)tgt[c] * DIM + i], se * K0.K[(DIM * c + i) * ND + DIM * c + i]);
      continue;
    }
    for (int t1 = 0; t1 < nt; ++t1) {
      bool first = true;
      for (int t0 = 0; t0 < t1; ++t0)
        if (tgt[t0] == tgt[t1]) first = false;
      if (!first) continue;
      for (int i = 0; i < DIM; ++i) {
        double acc = 0.0;
        for (int a = 0; a < nt; ++a) {
          if (tgt[a] != tgt[t1]) continue;
          for (int b = 0; b < nt; ++b) {
            if (tgt[b] != tgt[t1]) continue;
            acc += w[a] * w[b] * K0.K[(DIM * cor[a] + i) * ND + DIM * cor[b] + i];
          }
        }
        atomicAdd(&D[(int64_t)tgt[t1] * DIM + i], se * acc);
      }
    }
  }
}

// Dinv = 1/D on free DOFs, 0 elsewhere (the zero doubles as the free mask of the
// CG loop); d_out (optional) = diag(A) with 1 on non-free DOFs.
__global__ void k_dinv(int64_t ndof, const uint8_t *__restrict__ free_dof, const double *__restrict__ D,
                       double *__restrict__ Dinv, double *__restrict__ d_out, CgScalars *S) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ndof; i += (int64_t)gridDim.x * blockDim.x) {
    double d = D[i];
    if (free_dof[i]) {
      if (!(d > 0.0)) S->status = -7;  // TO_ENONPOS_DIAG
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
__device__ __forceinline__ void had_mid_inplace(const K0Had3 &H, double (&x)[24]) {
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
  for (int i = 0; i < 3; ++i) x[21 + i] *= H.diag[i][7];
  x[0] = x[1] = x[2] = 0.0;
#undef HAD_G3
#undef HAD_G2
}

// x := K0 x for H8 via the Hadamard factorisation (element.h), in place.
__device__ __forceinline__ void had_apply_inplace(const K0Had3 &H, double (&x)[24]) {
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

// ---- operator apply, atomic scatter ------------------------------------------------------
// q += C^T (s_e K0) C p per element (q zeroed by the caller).  With S (CG
// mode): p^T A p = sum_e s_e pbar_e^T K0 pbar_e (pbar_e = C_e p, p vanishing
// on non-free DOFs) is reduced in the same pass and the last block forms
// alpha_k = rho_k / p^T A p, so no separate p.q pass is needed.
template <int DIM>
__global__ void k_matvec_atomic(MeshView M, const double *__restrict__ s, const double *__restrict__ p,
                                double *__restrict__ q,
                                const __grid_constant__ typename std::conditional<DIM == 2, K0Dense2, K0Dense3>::type K0,
                                CgScalars *S, double *partials) {
  constexpr int NC = 1 << DIM, ND = DIM * NC;
  if (S && cg_stopped(S)) return;
  double pq = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M.n_el; e += (int64_t)gridDim.x * blockDim.x) {
    double ue[ND], ye[ND];
    int node[NC], hang[NC];
    gather_C<DIM>(M, e, p, ue, node, hang);
    dense_apply<ND>(K0.K, ue, ye);
    const double se = s[e];
    if (S) {
      double en = 0.0;
#pragma unroll
      for (int a = 0; a < ND; ++a) en = fma(ue[a], ye[a], en);
      pq = fma(se, en, pq);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (hang[c] < 0) {
#pragma unroll
        for (int i = 0; i < DIM; ++i) atomicAdd(&q[(int64_t)node[c] * DIM + i], se * ye[DIM * c + i]);
      } else {
        int h = hang[c];
        for (int k = M.hang_ptr[h]; k < M.hang_ptr[h + 1]; ++k) {
          double w = se * M.hang_weight[k];
          int64_t pn = M.hang_parent[k];
#pragma unroll
          for (int i = 0; i < DIM; ++i) atomicAdd(&q[pn * DIM + i], w * ye[DIM * c + i]);
        }
      }
    }
  }
  if (S) {
    double v[1] = {pq};
    if (grid_sum<1>(v, partials, &S->counter[CNT_PQ])) {
      if (!(v[0] > 0.0)) {
        S->status = (v[0] != v[0]) ? -5 : -6;
        S->done = 1;
      } else {
        S->alpha = S->rho / v[0];
      }
    }
  }
}

// ---- sensitivities (a10) ----------------------------------------------------------------
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

}  // namespace tomesh
