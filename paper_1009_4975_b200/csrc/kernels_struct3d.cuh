// Structured fast path for uniform H8 meshes (every leaf at one level and
// the leaves tiling the box: configs 3 and 5).  Same operator as the general
// path (Eq. 8 with Dirichlet rows); only the data layout
// and the work decomposition change:
//
//  * CG vectors live in "internal" order: lexicographic nodes (i fastest),
//    NXP = NX rounded up to even nodes per row, 3 interleaved doubles per
//    node (row stride RS = 3 NXP doubles, 16-byte aligned), plus zero pads
//    in front of and behind the vector.  Node-valued arrays (the Jacobi
//    inverse diagonal Dinv, one value per node because the 24 diagonal
//    entries of the cube's K0 are equal and Dirichlet conditions clamp whole
//    nodes) use the same node order.  The canonical Morton numbering (C3) is
//    applied once per solve at the boundary (f in, u out).  Connectivity is
//    implicit: element (i,j,k) has corner c at node (i+cx, j+cy, k+cz).
//  * One PCG iteration is ONE kernel (k_apply_s3<S3_CG>, Hestenes-Stiefel
//    recurrences on the rescaled system, PAPER.md:511-523 with reading Q3):
//      r_k = r_{k-1} - alpha_{k-1} q_{k-1}      (all staged nodes)
//      p_k = Dinv r_k + beta_{k-1} p_{k-1}      (all staged nodes)
//      x  += alpha_{k-1} p_{k-1}               (owned nodes)
//      q_k = A p_k                              (owned nodes)
//      one grid reduction of r_k.Dinv r_k, r_k.r_k, p_k.q_k, q_k.z_k, q_k.Dinv q_k
//    after which the last block forms alpha_k and beta_k (cg_single_step, with
//    rho_{k+1} from the one-step expansion) and tests rr_k.  r, p and q
//    ping-pong between two buffers each (iteration k reads buffer (k+1)&1 at
//    neighbours' nodes while they write buffer k&1).  k_final_s3 completes
//    x_N after exactly N iterations.  Vector traffic per iteration: read r,
//    q, p, x, write r, p, q, x (+ s, Dinv/3): 8.67 passes (12 for the
//    unfused textbook scheme).
//  * One CTA owns a (31 x (TYW-1)) patch of node columns and a range of node
//    planes; it sweeps the element layers in z.  Thread (tx, ty) computes the
//    element whose minimum corner is node (i0+tx-1, j0+ty-1) and accumulates
//    the node at that corner.  Element results reach their 4 in-plane nodes
//    by a warp shuffle (x) and a shared-memory exchange between warps (y);
//    the z neighbour is carried in registers to the next layer.  No atomics:
//    every node is written by exactly one thread, so the result is
//    deterministic.  The halo element row/column of each patch is recomputed
//    instead of exchanged.
//  * The r_{k-1}, q_{k-1}, p_{k-1} and Dinv plane tiles (33 x (TYW+1) nodes)
//    arrive as TMA boxes (cp.async.bulk.tensor.3d over tensor maps encoded at
//    upload, out-of-range rows and columns zero-filled), issued by one thread
//    with completion on an mbarrier, NBUF planes ahead of the compute; a
//    buffer is refilled right after the layer barrier that follows its form.
//    p_k is formed from them into a 4-plane shared-memory ring, so the gather
//    of the element corners never touches global memory.
//  * The element product uses the Hadamard factorisation of K0 (element.h):
//    ~215 fp64 operations instead of 576 FMAs.
//  * The 5 dots of the owned nodes are reduced in the same kernel
//    (last-block-done), and the last block forms the step (CG scalars stay on
//    device; sharded: the partials go to every rank, kernels_shard.cuh).
#pragma once
#include <cuda.h>

#include "device_common.cuh"
#include "element.h"
#include "kernels_cg.cuh"
#include "kernels_general.cuh"
#include "kernels_shard.cuh"
#include "tomesh_types.cuh"

namespace tomesh {



__device__ __forceinline__ int64_t s3_row(const GridView &G, int j, int k) {
  return ((int64_t)j + (int64_t)G.NY * k) * G.RS;
}
__device__ __forceinline__ int64_t s3_nrow(const GridView &G, int j, int k) {
  return ((int64_t)j + (int64_t)G.NY * k) * G.NXP;
}

constexpr int s3_pad128(int doubles) { return (doubles + 15) / 16 * 16; }   // 128-byte multiple


enum { S3_PLAIN = 0, S3_CG = 1 };

template <int TYW>
struct S3Smem {
  static constexpr int PY = TYW + 1;                          // node rows staged
  static constexpr int PD = s3_pad128(PY * kS3RowD);          // doubles per staged DOF plane
  static constexpr int PN = s3_pad128(PY * kS3RowN);          // doubles per staged node plane
  double ra[kS3NBuf][PD];                                     // r_{k-1} (CG) or v (plain), TMA box
  double qa[kS3NBuf][PD];                                     // q_{k-1}, TMA box
  double pa[kS3NBuf][PD];                                     // p_{k-1}, TMA box
  double dn[kS3NBuf][PN];                                     // Dinv per node, TMA box
  double pn[4][PY][kS3RowD];                                  // p_k ring: planes k mod 4
  double own[3][4][TYW * 32];                                 // owned node of plane k mod 3: z_k (3), Dinv
  double xch[2][TYW - 1][3][32];                              // y-exchange (layer parity); row TYW-1 sends to nobody
  unsigned long long mbar[kS3NBuf];
};

// 3D tiled TMA load of one box (OOB elements zero-filled; the transaction
// count is always the full box).
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

struct S3Maps {           // TMA maps of the arrays one K1 launch stages
  CUtensorMap a, q, p, d;   // r_{k-1} (or v), q_{k-1}, p_{k-1}, Dinv
};

// One thread: stage plane k (tile origin node (i0-1, j0-1)) into buffer b:
// one TMA box per array.  Rows and columns outside the vector come back as 0.
template <int TYW, int MODE>
__device__ __forceinline__ void s3_issue_plane(S3Smem<TYW> &sm, int b, const S3Maps &M, int i0, int j0, int k,
                                               int off, int noff) {
  constexpr int PY = TYW + 1;
  constexpr bool CG = MODE == S3_CG;
  constexpr unsigned bytes = PY * kS3RowD * 8 * (CG ? 3 : 1) + (CG ? PY * kS3RowN * 8 : 0);
  fence_proxy_async();
  mbar_arrive_expect_tx(&sm.mbar[b], bytes);
  tma_load_3d(sm.ra[b], &M.a, 3 * (i0 - 1) - off, j0 - 1, k, &sm.mbar[b]);
  if (CG) {
    tma_load_3d(sm.qa[b], &M.q, 3 * (i0 - 1) - off, j0 - 1, k, &sm.mbar[b]);
    tma_load_3d(sm.pa[b], &M.p, 3 * (i0 - 1) - off, j0 - 1, k, &sm.mbar[b]);
    tma_load_3d(sm.dn[b], &M.d, (i0 - 1) - noff, j0 - 1, k, &sm.mbar[b]);
  }
}

// r_k and p_k of node (col, row) of staged plane k.  CG:
//   r_k = r_{k-1} - alpha_{k-1} q_{k-1}   (free nodes, Dinv != 0; r stays 0 elsewhere)
//   p_k = Dinv r_k + beta_{k-1} p_{k-1}
// plain: p = the staged v.  pin = false (plane outside the mesh): zeros.
template <int TYW, int MODE>
__device__ __forceinline__ void s3_form_node(const S3Smem<TYW> &sm, int b, int row, int col, int off, int noff,
                                             double alpha, double beta, bool pin, double (&rv)[3], double (&pv)[3],
                                             double &dv) {
  // The staged q and p are finite (every buffer is zeroed at upload and only
  // ever holds finite iterates), so alpha = 0 / beta = 0 need no special case.
  const int o = row * kS3RowD + off + 3 * col;
  if (!pin) {
    dv = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) rv[d] = pv[d] = 0.0;
    return;
  }
  dv = MODE == S3_CG ? sm.dn[b][row * kS3RowN + noff + col] : 0.0;
  const double a_eff = dv != 0.0 ? -alpha : 0.0;   // r changes on free nodes only
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double r = sm.ra[b][o + d];
    double p = r;
    if (MODE == S3_CG) {
      r = fma(a_eff, sm.qa[b][o + d], r);
      p = fma(dv, r, beta * sm.pa[b][o + d]);
    }
    rv[d] = r;
    pv[d] = p;
  }
}

// K1.  MODE = S3_CG: iteration k of the single-kernel Jacobi-PCG (header comment):
//   form r_k, p_k on every staged node; owners write r_k, p_k and do
//   x += alpha_{k-1} p_{k-1}; q_k = A p_k (owners write it); reduce
//   rho_k = r_k.Dinv r_k, rr_k = r_k.r_k, p_k.q_k, q_k.z_k, q_k.Dinv q_k; the
//   last block forms alpha_k, beta_k (rho_{k+1} by the one-step expansion)
//   and the stop test on rr_k.
// MODE = S3_PLAIN: q = C^T K C v for a v that vanishes on non-free DOFs.
//
// Per CTA the layers ek = k_lo-1 .. k_hi-1 run with one CTA barrier each:
//   1. element ek from p planes ek, ek+1 (ring slots ek%4, (ek+1)%4); x routing
//      by warp shuffle; upper-row corners to the y-exchange (layer parity)
//   2. form plane ek+3 into ring slot (ek+3)%4 (last read by layer ek-1,
//      before the previous barrier) from the TMA staging; owners write r_k,
//      p_k, update x, keep z_k, Dinv.  The last warp done with a staging buffer
//      issues its next plane (+NBUF).  Runs before the barrier, overlapping
//      the other warps' element work.
//   3. barrier
//   4. y-exchange read: q and the dots of the owned node of plane ek
// (A variant with neighbour-only progress counters instead of the barrier was
// measured 18% slower: the counter handshakes cost more than the barrier.)
//
// SHARD (z-slab sharding, kernels_shard.cuh): the owners of planes own_lo and
// own_hi-1 also store r_k, p_k and q_k into the neighbours' ghost planes, and
// the last block pushes the 5 partial dots to every rank instead of forming
// the step.  Iteration k+1 starts with the step of iteration k: thread 0 of
// every CTA waits for the flags of sequence seq-1, sums the ranks' dots in
// rank order and evaluates the step (cg_step_eval, the same on every CTA and
// rank); CTA 0 also commits it to S.  One kernel per iteration, as unsharded.
template <int TYW, int MODE, bool SHARD = false>
__global__ void __launch_bounds__(32 * TYW, TYW <= 8 ? 2 : 1)
k_apply_s3(GridView G, const double *__restrict__ s, const __grid_constant__ S3Maps M, double *__restrict__ rnew,
           double *__restrict__ pnew, double *__restrict__ x, double *__restrict__ q,
           const __grid_constant__ K0HadSym H, CgScalars *S, double *partials, int kit, double rtol, double *hist,
           const __grid_constant__ ShardComm C, unsigned long long seq) {
  constexpr bool CG = MODE == S3_CG;
  pdl_wait();
  pdl_release();
  if (CG && cg_stopped(S)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  S3Smem<TYW> &sm = *reinterpret_cast<S3Smem<TYW> *>(smem_raw);
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = tx + 32 * ty;
  // x tiles fastest: the CTAs resident together cover whole node rows of the
  // same z range, so their TMA boxes (and stores) of a plane are adjacent in
  // memory (DRAM page locality)
  int tx_t, ty_t, k_lo, k_hi;
  if (G.plan) {
    const int4 pl = G.plan[blockIdx.x];
    tx_t = pl.x;
    ty_t = pl.y;
    k_lo = pl.z;
    k_hi = pl.w;
  } else {
    int bid = blockIdx.x;
    tx_t = bid % G.ntx;
    bid /= G.ntx;
    ty_t = bid % G.nty;
    const int zs = bid / G.nty;
    k_lo = zs * G.zlen;
    k_hi = min(G.NZ, k_lo + G.zlen);
  }
  const int i0 = tx_t * 31, j0 = ty_t * (TYW - 1);
  const int off = (i0 - 1) & 1;                         // DOF window starts on an even double
  const int noff = (i0 - 1) & 1;                        // node window starts on an even node
  const int ei = i0 - 1 + tx, ej = j0 - 1 + ty;        // this thread's element column / node column
  const bool col_el = (ei >= 0 && ei < G.EX && ej >= 0 && ej < G.EY);
  const bool owner = (tx >= 1 && ty >= 1 && ei < G.NX && ej < G.NY);
  double beta = CG ? __ldcg(&S->beta) : 0.0;
  double alpha_old = CG ? __ldcg(&S->alpha) : 0.0;
  if (SHARD && kit > 0) {
    __shared__ double s_ab[2];
    __shared__ int s_go;
    if (tid == 0) {
      double d[5];
      CgStepOut o;
      if (shard_gather(C, seq - 1, d, 5)) {
        // the neighbours' ghost planes (generic stores, ordered before their
        // flags) are read below by TMA (async proxy): cross-proxy fence
        asm volatile("fence.proxy.async;\n" ::: "memory");
        cg_step_eval(S, kit - 1, d, rtol, o);
      } else {
        o = CgStepOut{0.0, 0.0, 0.0, 0.0, 0.0, 1, -2, 0};
        o.thresh2 = __ldcg(&S->thresh2);
      }
      if (blockIdx.x == 0) cg_step_commit(S, kit - 1, o, hist);
      s_ab[0] = o.alpha;
      s_ab[1] = o.beta;
      s_go = !o.done;
    }
    __syncthreads();
    if (!s_go) return;
    alpha_old = s_ab[0];
    beta = s_ab[1];
  }
  // x += cp p_{k-1} + cz z_{k-1}, or x untouched in a deferring (odd) kernel
  // (cg_x_coef, kernels_cg.cuh).  (alpha, beta)_{k-2} sit in slot k & 1 of S,
  // which neither this kernel nor a sharded CTA 0 committing step k-1 writes.
  XCoef xc{0.0, 0.0, false};
  if (CG) xc = cg_x_coef(kit, alpha_old, beta, __ldcg(&S->ab[kit & 1][0]), __ldcg(&S->ab[kit & 1][1]), true);
  const bool xupd = CG && owner && xc.touch;
  const int64_t plane_d = (int64_t)G.NY * G.RS;        // doubles per node plane

  auto buf_of = [&](int k) { return (k - (k_lo - 1)) % kS3NBuf; };
  auto staged = [&](int k) { return k >= 0 && k < G.NZ && k <= k_hi; };
  if (tid == 0) {
    for (int bb = 0; bb < kS3NBuf; ++bb) {
      mbar_init(&sm.mbar[bb], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // initial staging: planes k_lo-1 .. k_lo-2+NBUF; afterwards plane P is
  // issued after the CTA barrier that follows the form of plane P-NBUF
  if (tid == 0)
    for (int k = k_lo - 1; k < k_lo - 1 + kS3NBuf; ++k)
      if (staged(k)) s3_issue_plane<TYW, MODE>(sm, buf_of(k), M, i0, j0, k, off, noff);
  unsigned phase = 0;                                   // parity bit per buffer

  // x of the owned node, two planes ahead: slot xa holds planes k_lo, k_lo+2,
  // ..., slot xb planes k_lo+1, k_lo+3, ... (each slot is a fixed register
  // triple: the 2x-unrolled layer loop alternates them)
  double xa[3] = {0.0, 0.0, 0.0}, xb[3] = {0.0, 0.0, 0.0};
  if (xupd) {
    const int64_t dof = s3_row(G, ej, k_lo) + 3 * ei;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (k_lo < k_hi) xa[d] = __ldcs(&x[dof + d]);
      if (k_lo + 1 < k_hi) xb[d] = __ldcs(&x[dof + plane_d + d]);
    }
  }
  double dots[5] = {0.0, 0.0, 0.0, 0.0, 0.0};           // rho, rr, p.q, q.z, q.Dinv q

  // form plane k into ring slot k%3.  Every thread forms its own node
  // (tx, ty), which is the node it owns (if it owns one).  The 41 halo nodes
  // of row TYW and column 32 go to warp 0, which owns no node (no stores, no
  // x update): two extra rounds there instead of one divergent round in
  // every warp.
  const int xe_row = tx == 0 ? TYW : tx - 1;            // warp 0, round 2 (lanes 0..TYW): column 32
  auto form_plane = [&](int k, double(&xs)[3]) {
    const bool pin = k >= 0 && k < G.NZ;
    const int bb = buf_of(k);
    if (pin) {
      mbar_wait(&sm.mbar[bb], (phase >> bb) & 1);
      phase ^= 1u << bb;
    }
    const int slot = (k + 3) % 3;                       // own ring slot
    double(*dst)[kS3RowD] = sm.pn[(k + 4) & 3];
    double rv[3], pv[3], dv;
    s3_form_node<TYW, MODE>(sm, bb, ty, tx, off, noff, alpha_old, beta, pin, rv, pv, dv);
#pragma unroll
    for (int d = 0; d < 3; ++d) dst[ty][off + 3 * tx + d] = pv[d];
    if (CG) {
      const bool mine = owner && k >= k_lo && k < k_hi;
#pragma unroll
      for (int d = 0; d < 3; ++d) sm.own[slot][d][tid] = dv * rv[d];   // read back only if mine
      sm.own[slot][3][tid] = dv;
      if (mine) {
        const int64_t dof = s3_row(G, ej, k) + 3 * ei;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          __stcs(&rnew[dof + d], rv[d]);
          __stcs(&pnew[dof + d], pv[d]);
          dots[0] = fma(dv * rv[d], rv[d], dots[0]);
          dots[1] = fma(rv[d], rv[d], dots[1]);
        }
        if (xupd) {
          const double *pp = &sm.pa[bb][ty * kS3RowD + off + 3 * tx];
          const double *rp = &sm.ra[bb][ty * kS3RowD + off + 3 * tx];
#pragma unroll
          for (int d = 0; d < 3; ++d) __stcs(&x[dof + d], fma(xc.cp, pp[d], fma(xc.cz * dv, rp[d], xs[d])));
          if (k + 2 < k_hi) {
#pragma unroll
            for (int d = 0; d < 3; ++d) xs[d] = __ldcs(&x[dof + 2 * plane_d + d]);
          }
        }
      }
    }
    if (ty == 0) {
      s3_form_node<TYW, MODE>(sm, bb, TYW, tx, off, noff, alpha_old, beta, pin, rv, pv, dv);
#pragma unroll
      for (int d = 0; d < 3; ++d) dst[TYW][off + 3 * tx + d] = pv[d];
      if (tx <= TYW) {
        s3_form_node<TYW, MODE>(sm, bb, xe_row, 32, off, noff, alpha_old, beta, pin, rv, pv, dv);
#pragma unroll
        for (int d = 0; d < 3; ++d) dst[xe_row][off + 3 * 32 + d] = pv[d];
      }
    }
  };
  // staging buffer of plane k is free once every warp has formed plane k,
  // i.e. after the CTA barrier that follows the form: thread 0 then refills it
  // with plane k+NBUF (no per-warp completion count on the critical path)
  auto refill = [&](int k) {
    if (tid == 0 && staged(k + kS3NBuf)) s3_issue_plane<TYW, MODE>(sm, buf_of(k), M, i0, j0, k + kS3NBuf, off, noff);
  };
  // prologue: planes k_lo-1 .. k_lo+1 (no element has read a ring slot yet)
  form_plane(k_lo - 1, xa);
  if (k_lo <= k_hi) form_plane(k_lo, xa);
  __syncthreads();
  refill(k_lo - 1);
  refill(k_lo);
  if (k_lo + 1 <= k_hi) form_plane(k_lo + 1, xb);
  __syncthreads();
  refill(k_lo + 1);

  // z carry at the face level: the top-face half of layer ek-1's inverse
  // transform (still in the x-y Hadamard basis of the 4 face nodes), added to
  // layer ek's bottom-face half before the face's own inverse x-y transform
  double gcar[12];
#pragma unroll
  for (int t = 0; t < 12; ++t) gcar[t] = 0.0;
  // s_e of this thread's element column, loaded two layers ahead (register ring)
  const int64_t s_stride = (int64_t)G.EX * G.EY;
  // the load itself is unconditional (clamped to a valid element) so that no
  // select waits on it; the validity mask is applied two layers later
  const int64_t s_col_c = (int64_t)min(max(ei, 0), G.EX - 1) + (int64_t)G.EX * min(max(ej, 0), G.EY - 1);
  auto load_s = [&](int ek) { return __ldg(&s[s_col_c + s_stride * min(max(ek, 0), G.EZ - 1)]); };
  auto s_valid = [&](int ek) { return col_el && ek >= 0 && ek < G.EZ && ek < k_hi; };
  // two slots, used alternately by even/odd layers of the 2x-unrolled loop
  // below, so the prefetch lands in its own register (no rotation moves that
  // would wait on the load)
  double s_a = load_s(k_lo - 1), s_b = load_s(k_lo);

  // One layer; no CTA barrier: warp w synchronises with rows w-1 and w+1 only
  // through the progress counters (it reads row w+1 of the p ring, sends its
  // upper corners to row w+1 and receives row w-1's).
  auto layer = [&](const int ek, double &s_slot, double(&x_slot)[3]) {
    const double se = s_valid(ek) ? s_slot : 0.0;
    s_slot = load_s(ek + 2);
    const int slo = (ek + 4) & 3, shi = (ek + 5) & 3;
    double y[24];
    {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int cx = c & 1, cy = (c >> 1) & 1, cz = c >> 2;
        const double *row = &sm.pn[cz ? shi : slo][ty + cy][off + 3 * (tx + cx)];
#pragma unroll
        for (int d = 0; d < 3; ++d) y[3 * c + d] = row[d];
      }
    }
    // element product in the Hadamard basis (mode m = mx + 2 my + 4 mz), with
    // s_e folded into the 10 class coefficients (se = 0 for elements outside
    // the mesh / segment)
    K0HadSym Hs;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
#pragma unroll
      for (int t = 0; t < 3; ++t) Hs.d[b][t] = H.d[b][t] * se;
#pragma unroll
      for (int t = 0; t < 2; ++t) Hs.o[b][t] = H.o[b][t] * se;
    }
    wht8x3(y);
    had_mid_inplace(Hs, y);
    // inverse transform, z stage: bottom face (plane ek) and top face (plane ek+1)
    double face[12];
#pragma unroll
    for (int t = 0; t < 12; ++t) {
      const double a = y[t], b = y[12 + t];
      face[t] = a + b + gcar[t];                        // plane ek: this layer's bottom + last layer's top
      gcar[t] = a - b;
    }
    // inverse y stage then x stage on the 4 face nodes (corner cx + 2 cy)
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double a = face[3 * m + d], b = face[3 * (m + 2) + d];
        face[3 * m + d] = a + b;
        face[3 * (m + 2) + d] = a - b;
      }
#pragma unroll
    for (int m = 0; m < 4; m += 2)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double a = face[3 * m + d], b = face[3 * (m + 1) + d];
        face[3 * m + d] = a + b;
        face[3 * (m + 1) + d] = a - b;
      }
    // x routing: corner (1, cy) of element column ei goes to node ei+1 (lane + 1);
    // lane 0 receives its own value: garbage, but lane 0 is the halo column
    double a_row[2][3];                                 // [cy][comp] at node column ei, plane ek
#pragma unroll
    for (int cy = 0; cy < 2; ++cy)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double from_left = __shfl_up_sync(0xffffffffu, face[3 * (1 + 2 * cy) + d], 1);
        a_row[cy][d] = face[3 * (2 * cy) + d] + from_left;
      }
    // y routing: the cy = 1 row goes to node row ty+1
    if (ty < TYW - 1) {
#pragma unroll
      for (int d = 0; d < 3; ++d) sm.xch[ek & 1][ty][d][tx] = a_row[1][d];
    }
    // the owned node's z_k and Dinv for plane ek (own ring slot ek%3, which the
    // form of plane ek+3 below overwrites)
    const bool qmine = ek >= k_lo && owner;
    double zown[3] = {0.0, 0.0, 0.0}, dvown = 0.0;
    if (CG && qmine) {
      const int os = (ek + 3) % 3;
#pragma unroll
      for (int d = 0; d < 3; ++d) zown[d] = sm.own[os][d][tid];
      dvown = sm.own[os][3][tid];
    }
    // plane ek+3 goes to ring slot (ek+3)%4, last read by layer ek-1's elements
    // (before the previous barrier), so the form runs before this layer's
    // barrier and overlaps the other warps' element work
    if (ek + 3 <= k_hi) form_plane(ek + 3, x_slot);
    __syncthreads();                                    // the one CTA barrier of the layer
    refill(ek + 3);
    // node plane ek is complete: (cz=0) parts of layer ek + (cz=1) parts of layer ek-1
    if (qmine) {
      const int64_t dof = s3_row(G, ej, ek) + 3 * ei;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double qv = a_row[0][d] + sm.xch[ek & 1][ty - 1][d][tx];
        __stcs(&q[dof + d], qv);
        if (CG) {
          dots[2] = fma(sm.pn[slo][ty][off + 3 * tx + d], qv, dots[2]);   // p_k of the own node (this thread formed it)
          dots[3] = fma(zown[d], qv, dots[3]);
          dots[4] = fma(dvown * qv, qv, dots[4]);
        }
      }
    }
  };
  // ek = k_lo-1+2t forms plane k_lo+2+2t (x slot xa); ek+1 forms k_lo+3+2t (xb)
  for (int ek = k_lo - 1; ek < k_hi; ek += 2) {
    layer(ek, s_a, xa);
    if (ek + 1 < k_hi) layer(ek + 1, s_b, xb);
  }
  if (SHARD) {
    // a CTA owning a boundary plane copies its tile of r_k, p_k, q_k there to
    // the neighbour's ghost plane (row segments, coalesced; the values were
    // stored by this CTA, so after the barrier they are read back from L2),
    // then fences at system scope before its arrival (kernels_shard.cuh)
    const bool lo_b = C.lo_r[0] && k_lo <= C.own_lo && C.own_lo < k_hi;
    const bool hi_b = C.hi_r[0] && k_lo <= C.own_hi - 1 && C.own_hi - 1 < k_hi;
    if (lo_b || hi_b) {
      __syncthreads();
      const int w = kit & 1;
      for (int side = 0; side < 2; ++side) {
        if (!(side ? hi_b : lo_b)) continue;
        const int kb = side ? C.own_hi - 1 : C.own_lo;
        double *tr = side ? C.hi_r[w] : C.lo_r[w], *tp = side ? C.hi_p[w] : C.lo_p[w];
        double *tq = side ? C.hi_q[w] : C.lo_q[w];
        for (int t = tid; t < (TYW - 1) * 93; t += 32 * TYW) {
          const int row = t / 93, e = t - 93 * row;
          const int j = j0 + row, i = i0 + e / 3;
          if (i < G.NX && j < G.NY) {
            const int64_t idx = s3_row(G, j, kb) + 3 * i0 + e;
            tr[idx] = __ldcg(&rnew[idx]);
            tp[idx] = __ldcg(&pnew[idx]);
            tq[idx] = __ldcg(&q[idx]);
          }
        }
      }
      __threadfence_system();
    }
  }
  if (CG) {
    if (grid_sum<5>(dots, partials, &S->counter[CNT_PQ])) {
      if (SHARD) shard_push(C, seq, dots, 5);
      else cg_single_step(S, kit, dots, rtol, hist);
    }
  }
}

// ---- final step of a structured solve (after N iterations) ----------------------------
// r_N = r_{N-1} - alpha q_{N-1} (free nodes), x_N = x_{N-1} + alpha p_{N-1},
// rho_N, rr_N -> cg_final_step.  Coalesced double2 streams; Dinv gathered
// per node (node = DOF / 3, an L1 hit).  r_N itself is not stored.
// SHARD: over the owned planes only (the caller offsets the pointers), and
// the partial rho_N, rr_N are pushed for k_shard_final.
// The deferred x update (cg_x_coef): x_N also takes the term kernel N-1 left
// pending.  A solve that stopped at an odd iteration k whose kernel deferred
// gets that term here too (x += (alpha_{k-1}/beta_{k-1}) (p_k - z_k), from
// r_k, p_k in buffer 1 = rk, pk); nothing else happens then.
template <bool SHARD = false>
__global__ void __launch_bounds__(512) k_final_s3(int n, const double *__restrict__ ro, const double *__restrict__ qo,
                                                  const double *__restrict__ po, const double *__restrict__ dn,
                                                  double *__restrict__ x, double *partials, CgScalars *S, int n_iter,
                                                  double rtol, double *hist, const __grid_constant__ ShardComm C,
                                                  unsigned long long seq, const double *__restrict__ rk,
                                                  const double *__restrict__ pk) {
  const int n2 = n >> 1;
  double2 *x2 = reinterpret_cast<double2 *>(x);
  if (cg_stopped(S)) {
    const int k = __ldcg(&S->iter);
    if (__ldcg(&S->status) == 0 && cg_x_deferred(k, __ldcg(&S->alpha), __ldcg(&S->beta))) {
      const double t = __ldcg(&S->alpha) / __ldcg(&S->beta);
      const double2 *r2 = reinterpret_cast<const double2 *>(rk);
      const double2 *p2 = reinterpret_cast<const double2 *>(pk);
      for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n2; j += gridDim.x * blockDim.x) {
        const unsigned e = 2u * (unsigned)j;
        const double d0 = __ldg(&dn[e / 3u]), d1 = __ldg(&dn[(e + 1u) / 3u]);
        const double2 rv = __ldcs(&r2[j]), pv = __ldcs(&p2[j]);
        double2 xv = x2[j];
        xv.x = fma(t, pv.x, fma(-t * d0, rv.x, xv.x));
        xv.y = fma(t, pv.y, fma(-t * d1, rv.y, xv.y));
        x2[j] = xv;
      }
    }
    // sharded: every rank pushes every tail sequence (kernels_shard.cuh)
    if (SHARD && blockIdx.x == 0 && threadIdx.x == 0) {
      const double zero[2] = {0.0, 0.0};
      shard_push(C, seq, zero, 2);
    }
    return;
  }
  const double alpha = __ldcg(&S->alpha);
  const XCoef xc = cg_x_coef(n_iter, alpha, __ldcg(&S->beta), __ldcg(&S->ab[n_iter & 1][0]),
                             __ldcg(&S->ab[n_iter & 1][1]), false);
  double acc[2] = {0.0, 0.0};
  const double2 *r2 = reinterpret_cast<const double2 *>(ro);
  const double2 *q2 = reinterpret_cast<const double2 *>(qo);
  const double2 *p2 = reinterpret_cast<const double2 *>(po);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n2; j += gridDim.x * blockDim.x) {
    double2 rv = __ldcs(&r2[j]);
    const unsigned e = 2u * (unsigned)j;
    const double d0 = __ldg(&dn[e / 3u]), d1 = __ldg(&dn[(e + 1u) / 3u]);
    if (xc.touch) {
      const double2 pv = __ldcs(&p2[j]);
      double2 xv = x2[j];
      xv.x = fma(xc.cp, pv.x, fma(xc.cz * d0, rv.x, xv.x));
      xv.y = fma(xc.cp, pv.y, fma(xc.cz * d1, rv.y, xv.y));
      x2[j] = xv;
    }
    if (alpha != 0.0) {
      const double2 qv = __ldcs(&q2[j]);
      if (d0 != 0.0) rv.x = fma(-alpha, qv.x, rv.x);
      if (d1 != 0.0) rv.y = fma(-alpha, qv.y, rv.y);
    }
    acc[0] = fma(rv.x, d0 * rv.x, fma(rv.y, d1 * rv.y, acc[0]));
    acc[1] = fma(rv.x, rv.x, fma(rv.y, rv.y, acc[1]));
  }
  if (grid_sum<2>(acc, partials, &S->counter[CNT_U1])) {
    if (SHARD) shard_push(C, seq, acc, 2);
    else cg_final_step(S, n_iter, acc[0], acc[1], rtol, hist);
  }
}

// ---- filter on the uniform lattice (a11; Eqs. 3-5) --------------------
// On a uniform grid H_de = rmin - |c_d - c_e| depends only on the lattice
// offset d - e, so the neighbour set of C9 is a fixed stencil of offsets with
// |offset|^2 h^2 < rmin^2 (exact on these dyadic values), truncated at the
// box boundary; V_d = h^3 for every element.  Two passes: the filtered
// quantity (x in for SENS, in for DENS) is scattered to lexicographic order,
// then each element (canonical order) sums its stencil.

static __global__ void k_filter_s3_scatter(int64_t n, const int32_t *__restrict__ perm_el, int mode,
                                    const double *__restrict__ x, const double *__restrict__ in,
                                    double *__restrict__ t_lex) {
  GRID_STRIDE(e, n) { t_lex[perm_el[e]] = mode == 0 ? x[e] * in[e] : in[e]; }
}

static __global__ void k_filter_s3(GridView G, int64_t n, const int32_t *__restrict__ perm_el,
                            const S3FilterOffset *__restrict__ offs, int n_off, int mode,
                            const double *__restrict__ x, const double *__restrict__ t_lex, double *__restrict__ out) {
  GRID_STRIDE(e, n) {
    const int64_t l = perm_el[e];
    const int i = (int)(l % G.EX);
    const int64_t rest = l / G.EX;
    const int j = (int)(rest % G.EY), k = (int)(rest / G.EY);
    double num = 0.0, den = 0.0;
    for (int o = 0; o < n_off; ++o) {
      const S3FilterOffset f = offs[o];
      const int ii = i + f.di, jj = j + f.dj, kk = k + f.dk;
      if (ii < 0 || ii >= G.EX || jj < 0 || jj >= G.EY || kk < 0 || kk >= G.EZ) continue;
      num = fma(f.w, __ldg(&t_lex[ii + (int64_t)G.EX * (jj + (int64_t)G.EY * kk)]), num);
      den += f.w;
    }
    out[e] = mode == 0 ? num / (x[e] * den) : num / den;
  }
}

// Dynamic AMR marking on the uniform box (reading R21): x scattered to
// lexicographic order in t_lex, then any solid element within the filter
// stencil (the same exact |o|^2 h^2 < rmin^2 offsets).  lev = the mesh level.
static __global__ void k_amr_mark_s3(GridView G, int64_t n, const int32_t *__restrict__ perm_el,
                              const S3FilterOffset *__restrict__ offs, int n_off, const double *__restrict__ t_lex,
                              double rho_s, int lev, int L, int8_t *__restrict__ marks) {
  GRID_STRIDE(e, n) {
    const int64_t l = perm_el[e];
    const int i = (int)(l % G.EX);
    const int64_t rest = l / G.EX;
    const int j = (int)(rest % G.EY), k = (int)(rest / G.EY);
    bool near = false;
    for (int o = 0; o < n_off && !near; ++o) {
      const S3FilterOffset f = offs[o];
      const int ii = i + f.di, jj = j + f.dj, kk = k + f.dk;
      if (ii < 0 || ii >= G.EX || jj < 0 || jj >= G.EY || kk < 0 || kk >= G.EZ) continue;
      near = __ldg(&t_lex[ii + (int64_t)G.EX * (jj + (int64_t)G.EY * kk)]) >= rho_s;
    }
    marks[e] = near ? (lev < L ? 1 : 0) : (lev > 0 ? -1 : 0);
  }
}

// ---- setup kernels of the structured path ------------------------------------------------

// s in lexicographic element order from x in canonical (Morton) element order.
static __global__ void k_simp_s3(int64_t n, const double *__restrict__ x, const int32_t *__restrict__ perm_el,
                          double penal, double E0, double Emin, double h, double *__restrict__ s_lex,
                          CgScalars *S) {
  GRID_STRIDE(e, n) {
    double xe = x[e];
    if (!(xe > 0.0) || !(xe <= 1.0)) cg_fail(S, -1);
    s_lex[perm_el[e]] = (Emin + pow(xe, penal) * (E0 - Emin)) * h;
  }
}

// D = K0_diag * sum of s over the <= 8 elements around each node (all 24
// diagonal entries of the cube's K0 are equal); Dinv = free ? 1/D : 0 per
// node; d_out (optional, per DOF) = diag(A) with 1 on non-free DOFs.
static __global__ void k_diag_s3(GridView G, const double *__restrict__ s_lex, const uint8_t *__restrict__ free_node,
                          double k0d, double *__restrict__ dn, double *__restrict__ d_out, CgScalars *S) {
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
    const int64_t node = s3_nrow(G, j, k) + i;
    const bool fr = free_node[node] != 0;
    if (fr && !(d > 0.0)) cg_fail(S, -7);
    if (dn) dn[node] = fr ? 1.0 / d : 0.0;
    if (d_out) {
      const int64_t base = s3_row(G, j, k) + 3 * i;
#pragma unroll
      for (int c = 0; c < 3; ++c) d_out[base + c] = fr ? d : 1.0;
    }
  }
}

// out_int[base(n)+c] = mask ? in[n*3+c] : 0   (canonical -> internal)
static __global__ void k_to_int(int64_t n_node, const int32_t *__restrict__ base_of, const double *__restrict__ in,
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
static __global__ void k_from_int(int64_t n_node, const int32_t *__restrict__ base_of, const double *__restrict__ in_int,
                           double *__restrict__ out) {
  GRID_STRIDE(n, n_node) {
    const int64_t l = base_of[n];
#pragma unroll
    for (int c = 0; c < 3; ++c) out[n * 3 + c] = in_int[l + c];
  }
}

}  // namespace tomesh
