// Structured fast path for uniform H8 meshes (every leaf at one level and
// the leaves tiling the box: configs 3 and 5).  Same operator as the general
// path (Eq. 8 with Dirichlet rows); only the data layout
// and the work decomposition change:
//
//  * CG vectors live in "internal" order: lexicographic nodes (i fastest),
//    3 interleaved doubles per node, each node row padded to an even number
//    of doubles (RS) so every row starts 16-byte aligned, plus zero pads in
//    front of and behind the vector.  The canonical Morton numbering (C3) is
//    applied once per solve at the boundary (f in, u out).  Connectivity is
//    implicit: element (i,j,k) has corner c at node (i+cx, j+cy, k+cz).
//  * s_e lives in lexicographic element order.
//  * One CTA owns a (31 x (TYW-1)) patch of node columns and a range of node
//    planes; it sweeps the element layers in z.  Thread (tx, ty) computes the
//    element whose minimum corner is node (i0+tx-1, j0+ty-1) and accumulates
//    the node at that corner.  Element results reach their 4 in-plane nodes
//    by a warp shuffle (x) and a shared-memory exchange between warps (y);
//    the z neighbour is carried in registers to the next layer.  No atomics:
//    every node is written by exactly one thread, so the result is
//    deterministic.  The halo element row/column of each patch is recomputed
//    instead of exchanged.
//  * The p plane tile (33 x (TYW+1) nodes) arrives by TMA 1D bulk copies
//    (cp.async.bulk, one 800-byte row each, issued by one thread, completion
//    on an mbarrier), NBUF-deep so the copy of plane k+3 overlaps the
//    compute of layer k.  The lower plane of each element is carried in
//    registers, so each layer reads one plane from shared memory.
//  * The element product uses the Hadamard factorisation of K0 (element.h):
//    ~215 fp64 operations instead of 576 FMAs.
//  * p.q of the owned nodes is reduced in the same kernel (last-block-done),
//    and the last block forms alpha = rho / p.q (CG scalars stay on device).
#pragma once
#include "device_common.cuh"
#include "element.h"
#include "kernels_cg.cuh"
#include "kernels_general.cuh"

namespace tomesh {

struct GridView {
  int EX, EY, EZ;        // elements per axis
  int NX, NY, NZ;        // nodes per axis
  int RS;                // doubles per node row in the internal layout (even)
  int ntx, nty, nzs;     // CTA tiles in x, y and z segments
  int zlen;              // node planes per z segment
};

constexpr int kS3PadFront = 16;    // doubles before / after an internal vector
constexpr int kS3PadBack = 128;
constexpr int kS3RowD = 100;       // doubles staged per node row: 33 nodes + alignment (800 B)
constexpr int kS3NBuf = 4;

__device__ __forceinline__ int64_t s3_row(const GridView &G, int j, int k) {
  return ((int64_t)j + (int64_t)G.NY * k) * G.RS;
}

template <int TYW>
struct S3Smem {
  static constexpr int PY = TYW + 1;                // node rows staged
  double plane[kS3NBuf][PY][kS3RowD];
  double xch[TYW][6][32];                           // y-exchange: 2 planes x 3 components
  unsigned long long mbar[kS3NBuf];
};

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// One thread: copy the node rows of plane k (tile origin i0-1, j0-1) into buffer b.
// Rows outside the mesh are skipped (they only feed elements outside the mesh,
// whose s_e is 0; their stale values are finite).
template <int TYW>
__device__ __forceinline__ void s3_issue_plane(S3Smem<TYW> &sm, int b, const GridView &G, const double *p, int i0,
                                               int j0, int k, int off) {
  constexpr int PY = TYW + 1;
  unsigned bytes = 0;
  const bool kin = (k >= 0 && k < G.NZ);
  if (kin)
    for (int row = 0; row < PY; ++row) {
      const int j = j0 - 1 + row;
      if (j >= 0 && j < G.NY) bytes += kS3RowD * 8;
    }
  fence_proxy_async();
  mbar_arrive_expect_tx(&sm.mbar[b], bytes);
  if (kin)
    for (int row = 0; row < PY; ++row) {
      const int j = j0 - 1 + row;
      if (j < 0 || j >= G.NY) continue;
      const double *src = p + s3_row(G, j, k) + 3 * (i0 - 1) - off;
      bulk_g2s(&sm.plane[b][row][0], src, kS3RowD * 8, &sm.mbar[b]);
    }
}

template <int TYW>
__global__ void __launch_bounds__(32 * TYW, 2)
k_apply_s3(GridView G, const double *__restrict__ s, const double *__restrict__ p, double *__restrict__ q,
           const __grid_constant__ K0Had3 H, CgScalars *S, double *partials) {
  if (S && cg_stop_at_apply(S)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  S3Smem<TYW> &sm = *reinterpret_cast<S3Smem<TYW> *>(smem_raw);
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = tx + 32 * ty;
  int b = blockIdx.x;
  const int zs = b % G.nzs;
  b /= G.nzs;
  const int ty_t = b % G.nty;
  const int tx_t = b / G.nty;
  const int i0 = tx_t * 31, j0 = ty_t * (TYW - 1);
  const int k_lo = zs * G.zlen;
  const int k_hi = min(G.NZ, k_lo + G.zlen);
  const int off = (i0 - 1) & 1;                         // window starts on an even double
  const int ei = i0 - 1 + tx, ej = j0 - 1 + ty;        // this thread's element column / node column
  const bool col_el = (ei >= 0 && ei < G.EX && ej >= 0 && ej < G.EY);
  const bool owner = (tx >= 1 && ty >= 1 && ei < G.NX && ej < G.NY);

  // zero the staging buffers once (rows that are never copied must hold finite values)
  for (int t = tid; t < kS3NBuf * (TYW + 1) * kS3RowD; t += 32 * TYW) (&sm.plane[0][0][0])[t] = 0.0;
  if (tid == 0)
    for (int bb = 0; bb < kS3NBuf; ++bb) mbar_init(&sm.mbar[bb], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  // prologue: planes k_lo-1, k_lo, k_lo+1
  if (tid == 0)
    for (int t = 0; t < 3; ++t) s3_issue_plane<TYW>(sm, t, G, p, i0, j0, k_lo - 1 + t, off);
  unsigned phase = 0;                                   // parity bit per buffer

  double pq = 0.0;
  double acc_cur[3] = {0.0, 0.0, 0.0};                  // node plane ek (owned column)
  int64_t s_idx = (int64_t)ei + (int64_t)G.EX * ((int64_t)ej + (int64_t)G.EY * (k_lo - 1));
  const int64_t s_stride = (int64_t)G.EX * G.EY;
  double s_next = 0.0;
  {
    const int ek = k_lo - 1;
    if (col_el && ek >= 0 && ek < G.EZ) s_next = __ldg(&s[s_idx]);
  }

  for (int ek = k_lo - 1; ek < k_hi; ++ek) {
    const int bo = (ek - (k_lo - 1)) % kS3NBuf;         // buffer of plane ek
    const int bn = (bo + 1) % kS3NBuf;                  // buffer of plane ek+1
    // keep the copy engine NBUF-1 planes ahead: plane ek+3 into the buffer of plane ek-1
    if (tid == 0 && ek + 3 <= k_hi) s3_issue_plane<TYW>(sm, (bo + 3) % kS3NBuf, G, p, i0, j0, ek + 3, off);
    if (ek == k_lo - 1) {
      mbar_wait(&sm.mbar[bo], (phase >> bo) & 1);
      phase ^= 1u << bo;
    }
    mbar_wait(&sm.mbar[bn], (phase >> bn) & 1);
    phase ^= 1u << bn;
    const double se = s_next;
    s_idx += s_stride;
    {
      const int ekn = ek + 1;
      s_next = (col_el && ekn >= 0 && ekn < G.EZ && ekn < k_hi) ? __ldg(&s[s_idx]) : 0.0;
    }
    const bool el = col_el && ek >= 0 && ek < G.EZ;
    double y[24];
    if (el) {
      double xv[24];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int cx = c & 1, cy = (c >> 1) & 1, cz = c >> 2;
        const double *row = &sm.plane[cz ? bn : bo][ty + cy][off + 3 * (tx + cx)];
#pragma unroll
        for (int d = 0; d < 3; ++d) xv[3 * c + d] = row[d];
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
      const int64_t dof = s3_row(G, ej, ek) + 3 * ei;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double qv = acc_cur[d] + tot[0][d];
        q[dof + d] = qv;
        pq = fma(sm.plane[bo][ty][off + 3 * tx + d], qv, pq);
      }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) acc_cur[d] = tot[1][d];
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
__global__ void k_diag_s3(GridView G, const double *__restrict__ s_lex, const uint8_t *__restrict__ free_int,
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
    const int64_t base = s3_row(G, j, k) + 3 * i;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t dof = base + c;
      if (free_int[dof]) {
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

// out_int[base(n)+c] = mask ? in[n*3+c] : 0   (canonical -> internal)
__global__ void k_to_int(int64_t n_node, const int32_t *__restrict__ base_of, const double *__restrict__ in,
                         const uint8_t *__restrict__ free_canon, double *__restrict__ out_int) {
  GRID_STRIDE(n, n_node) {
    const int64_t l = base_of[n];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t d = n * 3 + c;
      out_int[l + c] = (free_canon == nullptr || free_canon[d]) ? in[d] : 0.0;
    }
  }
}

// out[n*3+c] = in_int[base(n)+c]   (internal -> canonical)
__global__ void k_from_int(int64_t n_node, const int32_t *__restrict__ base_of, const double *__restrict__ in_int,
                           double *__restrict__ out) {
  GRID_STRIDE(n, n_node) {
    const int64_t l = base_of[n];
#pragma unroll
    for (int c = 0; c < 3; ++c) out[n * 3 + c] = in_int[l + c];
  }
}

}  // namespace tomesh
