// Structured fast path for uniform H8 meshes (every leaf at one level and
// the leaves tiling the box: configs 3 and 5).  Same operator as the general
// path (Eq. 8 with Dirichlet rows); only the data layout
// and the work decomposition change:
//
//  * CG vectors live in lexicographic node order (i fastest), DOF-interleaved
//    (3 doubles per node); the canonical Morton numbering (C3) is applied once
//    per solve at the boundary (f in, u out).  Connectivity is implicit:
//    element (i,j,k) has corner c at node (i+cx, j+cy, k+cz).
//  * s_e lives in lexicographic element order.
//  * One CTA owns a (31 x (TYW-1)) patch of node columns and a range of node
//    planes; it sweeps the element layers in z.  Thread (tx, ty) computes the
//    element whose minimum corner is node (i0+tx-1, j0+ty-1) and accumulates
//    the node at that corner.  Element results reach their 4 in-plane nodes
//    by a warp shuffle (x) and a shared-memory exchange between warps (y);
//    the z neighbour is carried in registers to the next layer.  No atomics:
//    every node is written by exactly one thread, so the result is
//    deterministic.  The halo element row/column of each patch is recomputed
//    (32/31 x TYW/(TYW-1) extra work) instead of exchanged.
//  * The p plane tile (33 x (TYW+1) nodes) is staged in shared memory with
//    cp.async one layer ahead (triple buffer).
//  * The element product uses the Hadamard factorisation of K0 (element.h):
//    ~215 fp64 operations instead of 576 FMAs.
//  * p.q of the owned nodes is reduced in the same kernel (last-block-done),
//    and the last block forms alpha = rho / p.q (CG scalars stay on device).
#pragma once
#include "device_common.cuh"
#include "element.h"
#include "kernels_general.cuh"

namespace tomesh {

struct GridView {
  int EX, EY, EZ;        // elements per axis
  int NX, NY, NZ;        // nodes per axis
  int ntx, nty, nzs;     // CTA tiles in x, y and z segments
  int zlen;              // node planes per z segment
};

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

template <int TYW>
struct S3Smem {
  static constexpr int PX = 33;            // node columns staged per row
  static constexpr int PY = TYW + 1;       // node rows staged
  double plane[3][3][PY][PX];              // [buffer][component][row][col]
  double xch[TYW][6][32];                  // y-exchange: 2 planes x 3 components
};

// Stage node plane k of p (tile origin i0-1, j0-1) into buf; zero outside the mesh.
template <int TYW>
__device__ __forceinline__ void stage_plane(S3Smem<TYW> &sm, int buf, const GridView &G, const double *__restrict__ p,
                                            int i0, int j0, int k) {
  constexpr int PX = S3Smem<TYW>::PX, PY = S3Smem<TYW>::PY;
  const int tid = threadIdx.x + 32 * threadIdx.y;
  constexpr int NT = 32 * TYW;
  const bool kin = (k >= 0 && k < G.NZ);
  for (int t = tid; t < PY * PX * 3; t += NT) {
    int row = t / (PX * 3);
    int rem = t - row * (PX * 3);
    int col = rem / 3;
    int c = rem - col * 3;
    int i = i0 - 1 + col, j = j0 - 1 + row;
    double *dst = &sm.plane[buf][c][row][col];
    if (kin && i >= 0 && i < G.NX && j >= 0 && j < G.NY) {
      cp_async8(dst, p + ((int64_t)i + (int64_t)G.NX * ((int64_t)j + (int64_t)G.NY * k)) * 3 + c);
    } else {
      *dst = 0.0;
    }
  }
}

template <int TYW>
__global__ void __launch_bounds__(32 * TYW, 2)
k_apply_s3(GridView G, const double *__restrict__ s, const double *__restrict__ p, double *__restrict__ q,
           const __grid_constant__ K0Had3 H, CgScalars *S, double *partials) {
  if (S && cg_stop_at_apply(S)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S3Smem<TYW> &sm = *reinterpret_cast<S3Smem<TYW> *>(smem_raw);
  const int tx = threadIdx.x, ty = threadIdx.y;
  int b = blockIdx.x;
  const int zs = b % G.nzs;
  b /= G.nzs;
  const int ty_t = b % G.nty;
  const int tx_t = b / G.nty;
  const int i0 = tx_t * 31, j0 = ty_t * (TYW - 1);
  const int k_lo = zs * G.zlen;
  const int k_hi = min(G.NZ, k_lo + G.zlen);
  const int ei = i0 - 1 + tx, ej = j0 - 1 + ty;        // this thread's element column / node column
  const bool col_el = (ei >= 0 && ei < G.EX && ej >= 0 && ej < G.EY);
  const bool owner = (tx >= 1 && ty >= 1 && ei < G.NX && ej < G.NY);
  double pq = 0.0;

  // prologue: planes k_lo-1 (buffer 0) and k_lo (buffer 1)
  stage_plane<TYW>(sm, 0, G, p, i0, j0, k_lo - 1);
  stage_plane<TYW>(sm, 1, G, p, i0, j0, k_lo);
  cp_async_commit();
  double acc_cur[3] = {0.0, 0.0, 0.0};   // node plane ek (owned column)
  int bo = 0, bn = 1, bf = 2;            // buffers of planes ek, ek+1, ek+2

  for (int ek = k_lo - 1; ek < k_hi; ++ek) {
    cp_async_wait_all();
    __syncthreads();
    // prefetch plane ek+2 (its buffer was last read in layer ek-1)
    if (ek + 2 <= k_hi) stage_plane<TYW>(sm, bf, G, p, i0, j0, ek + 2);
    cp_async_commit();

    const bool el = col_el && ek >= 0 && ek < G.EZ;
    double y[24];
    if (el) {
      const double se = s[(int64_t)ei + (int64_t)G.EX * ((int64_t)ej + (int64_t)G.EY * ek)];
      double xv[24];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int cx = c & 1, cy = (c >> 1) & 1, cz = c >> 2;
        const int buf = cz ? bn : bo;
#pragma unroll
        for (int d = 0; d < 3; ++d) xv[3 * c + d] = sm.plane[buf][d][ty + cy][tx + cx];
      }
      had_apply(H, xv, y);
#pragma unroll
      for (int a = 0; a < 24; ++a) y[a] *= se;
    } else {
#pragma unroll
      for (int a = 0; a < 24; ++a) y[a] = 0.0;
    }
    // x routing: corner (1,cy,cz) of element ei goes to node ei+1 (lane + 1)
    double a_row[2][2][3];   // [cy][cz][comp] after the x merge, at node column ei
#pragma unroll
    for (int cy = 0; cy < 2; ++cy)
#pragma unroll
      for (int cz = 0; cz < 2; ++cz)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          double from_left = __shfl_up_sync(0xffffffffu, y[3 * (1 + 2 * cy + 4 * cz) + d], 1);
          if (tx == 0) from_left = 0.0;
          a_row[cy][cz][d] = y[3 * (2 * cy + 4 * cz) + d] + from_left;
        }
    // y routing: row ty's (cy = 1) part goes to row ty+1
#pragma unroll
    for (int cz = 0; cz < 2; ++cz)
#pragma unroll
      for (int d = 0; d < 3; ++d) sm.xch[ty][3 * cz + d][tx] = a_row[1][cz][d];
    __syncthreads();
    double tot[2][3];
#pragma unroll
    for (int cz = 0; cz < 2; ++cz)
#pragma unroll
      for (int d = 0; d < 3; ++d) tot[cz][d] = a_row[0][cz][d] + (ty > 0 ? sm.xch[ty - 1][3 * cz + d][tx] : 0.0);
    // node plane ek is complete: cz=1 part of layer ek-1 (acc_cur) + cz=0 part of layer ek
    if (ek >= k_lo && owner) {
      const int64_t node = (int64_t)ei + (int64_t)G.NX * ((int64_t)ej + (int64_t)G.NY * ek);
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double qv = acc_cur[d] + tot[0][d];
        q[node * 3 + d] = qv;
        pq = fma(sm.plane[bo][d][ty][tx], qv, pq);
      }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) acc_cur[d] = tot[1][d];
    const int t = bo;
    bo = bn;
    bn = bf;
    bf = t;
  }
  cp_async_wait_all();
  if (S) {
    double v[1] = {pq};
    // grid_sum needs a 1-D block index space; blockIdx.x is already linear
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

// ---- setup kernels of the structured path ------------------------------------------------

// s in lexicographic element order from x in canonical (Morton) element order.
__global__ void k_simp_s3(int64_t n, const double *__restrict__ x, const int32_t *__restrict__ perm_el,
                          double penal, double E0, double Emin, double h, double *__restrict__ s_lex,
                          CgScalars *S) {
  GRID_STRIDE(e, n) {
    double xe = x[e];
    if (!(xe > 0.0) || !(xe <= 1.0)) S->status = -1;
    s_lex[perm_el[e]] = (Emin + pow(xe, penal) * (E0 - Emin)) * h;
  }
}

// D = K0_diag * sum of s over the <= 8 elements around each node (all 24
// diagonal entries of the cube's K0 are equal); Dinv = free ? 1/D : 0.
__global__ void k_diag_s3(GridView G, const double *__restrict__ s_lex, const uint8_t *__restrict__ free_lex,
                          double k0d, double *__restrict__ Dinv, double *__restrict__ d_out, CgScalars *S) {
  const int64_t nn = (int64_t)G.NX * G.NY * G.NZ;
  GRID_STRIDE(n, nn) {
    int i = (int)(n % G.NX);
    int64_t r = n / G.NX;
    int j = (int)(r % G.NY);
    int k = (int)(r / G.NY);
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      int ei = i - (c & 1), ej = j - ((c >> 1) & 1), ek = k - (c >> 2);
      if (ei >= 0 && ei < G.EX && ej >= 0 && ej < G.EY && ek >= 0 && ek < G.EZ)
        acc += s_lex[(int64_t)ei + (int64_t)G.EX * ((int64_t)ej + (int64_t)G.EY * ek)];
    }
    const double d = k0d * acc;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t dof = n * 3 + c;
      if (free_lex[dof]) {
        if (!(d > 0.0)) S->status = -7;
        if (Dinv) Dinv[dof] = 1.0 / d;
        if (d_out) d_out[dof] = d;
      } else {
        if (Dinv) Dinv[dof] = 0.0;
        if (d_out) d_out[dof] = 1.0;
      }
    }
  }
}

// out_lex[perm[n]*3+c] = mask ? in[n*3+c] : 0   (canonical -> internal)
__global__ void k_to_lex(int64_t n_node, const int32_t *__restrict__ perm, const double *__restrict__ in,
                         const uint8_t *__restrict__ free_canon, double *__restrict__ out_lex) {
  GRID_STRIDE(n, n_node) {
    const int64_t l = perm[n];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t d = n * 3 + c;
      out_lex[l * 3 + c] = (free_canon == nullptr || free_canon[d]) ? in[d] : 0.0;
    }
  }
}

// out[n*3+c] = in_lex[perm[n]*3+c]   (internal -> canonical)
__global__ void k_from_lex(int64_t n_node, const int32_t *__restrict__ perm, const double *__restrict__ in_lex,
                           double *__restrict__ out) {
  GRID_STRIDE(n, n_node) {
    const int64_t l = perm[n];
#pragma unroll
    for (int c = 0; c < 3; ++c) out[n * 3 + c] = in_lex[l * 3 + c];
  }
}

}  // namespace tomesh
