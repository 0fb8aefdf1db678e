// General (AMR) path, small meshes: the whole PCG loop in ONE thread-block
// cluster (k_gen_cluster).  Same operator (Eq. 8 with Dirichlet rows,
// PAPER.md:678-682, the hanging-node interpolation C of Eq. 6, :653-663),
// same recurrences and step (the one-step rho expansion of kernels_cg.cuh)
// and the same owner-computes block records as k_gen_fused
// (kernels_genfused.cuh), built with at most kGcMaxBlocks blocks so that one
// cluster holds the mesh.  What changes is where the vectors live and how
// the CTAs exchange them:
//   * each CTA keeps the CG state of its owned nodes -- r, p, x, q, z, Dinv --
//     in its shared memory for the whole solve (loaded once, written back
//     once); nothing goes through global memory per iteration;
//   * halo values of p_k are PUSHED by their owner into the consumers' shared
//     memory (st.async over distributed shared memory, completion counted in
//     bytes on the consumer's mbarrier), from a send list built at upload;
//   * the 5 dots: every CTA pushes its block sums to every CTA the same way;
//     each CTA then adds the nb partials in rank order and evaluates the step
//     itself (same values, same order: the same alpha, beta and stop decision
//     everywhere).  The step is committed to S once, after the loop.
// No cluster barrier inside the loop: a CTA waits only on its own mbarriers.
// Receive buffers are double-buffered by iteration parity.  Reuse is safe
// because every CTA's push of iteration k+2 comes after its step k+1, which
// needs every CTA's dots of iteration k+1, which each CTA pushes only after it
// has consumed its halo and dots of iteration k.  For the same reason no
// complete-tx of iteration k+2 reaches an mbarrier before its phase of
// iteration k has completed.  Deterministic: fixed orders, no atomics.
#pragma once
#include <cooperative_groups.h>

#include "kernels_genfused.cuh"

namespace tomesh {

// CTA size T in {128, 256, 512} (the smallest whose 2 T covers a block's
// owned nodes: fewer warps make the CTA barriers and the block reduction
// cheaper); up to kGcOwnPerThread owned nodes per thread.
constexpr int kGcMaxThreads = 512;
constexpr int kGcOwnPerThread = 4;
constexpr int kGcMaxOwn = kGcMaxThreads * kGcOwnPerThread;   // owned nodes per CTA
#ifndef TOMESH_GC_MAXB
#define TOMESH_GC_MAXB 16
#endif
constexpr int kGcMaxBlocks = TOMESH_GC_MAXB;             // cluster size (16: non-portable, opted in at upload)
#ifndef TOMESH_GC_OWN_MIN
#define TOMESH_GC_OWN_MIN 128
#endif
constexpr int kGcOwnMin = TOMESH_GC_OWN_MIN;             // fewer, larger blocks below nb * kGcOwnMin nodes
#ifndef TOMESH_GC_OWN_MAXT
#define TOMESH_GC_OWN_MAXT 512
#endif
constexpr int kGcOwnMaxTarget = TOMESH_GC_OWN_MAXT;      // larger meshes: not the cluster solver

// (send lists: GcSend, tomesh_types.cuh)

template <int DIM, int T>
struct GcChunk {
  static constexpr int NC = 1 << DIM;
  static constexpr int CH = DIM == 3 && T > 256 ? 256 : T;   // elements per chunk (one per thread)
  static constexpr int YS = NC * DIM + 1;
};

// Byte offsets of the dynamic shared memory of k_gen_cluster (host and
// device): record, s_e, local node values P, the owned r, x, q, z, Dinv, one
// chunk of element results, the halo receive buffers [2], the dot receive
// slots [2][16][8], the step broadcast [10], the send list, 5 mbarriers.
struct GcLayout {
  size_t sl, P, R, X, Q, Zs, Ds, Y, PH, PT, bc, send, bar, total;
};
__host__ __device__ inline size_t gc_even8(size_t doubles) { return 8 * ((doubles + 1) & ~(size_t)1); }
template <int DIM, int T>
__host__ __device__ inline GcLayout gc_layout(int max_rec16, int max_el, int max_loc, int max_own, int max_halo,
                                              int max_send) {
  GcLayout L;
  size_t o = (size_t)16 * max_rec16;
  const size_t own = gc_even8((size_t)max_own * DIM);
  L.sl = o;
  o += gc_even8(max_el);
  L.P = o;
  o += gc_even8((size_t)max_loc * DIM);
  L.R = o;
  o += own;
  L.X = o;
  o += own;
  L.Q = o;
  o += own;
  L.Zs = o;
  o += own;
  L.Ds = o;
  o += own;
  L.Y = o;
  o += gc_even8((size_t)GcChunk<DIM, T>::CH * GcChunk<DIM, T>::YS);
  L.PH = o;
  o += 2 * gc_even8((size_t)max_halo * DIM);
  L.PT = o;
  o += (size_t)2 * 16 * 8 * 8;
  L.bc = o;
  o += 8 * 10;
  L.send = o;
  o += (size_t)4 * ((max_send + 3) & ~3);
  L.bar = o;
  o += 8 * 6;
  L.total = o;
  return L;
}

// shared::cluster address of `p` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t gc_mapa(const void *p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void gc_st_async(uint32_t addr, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(addr), "d"(v),
               "r"(bar)
               : "memory");
}
__device__ __forceinline__ void gc_st_async2(uint32_t addr, double a, double b, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(addr),
               "d"(a), "d"(b), "r"(bar)
               : "memory");
}

#ifdef TOMESH_GC_TRACE
// A/B instrumentation build only: phase timestamps of iteration 10 in CTA 0, printed.
#define GC_MARK(j)                                 \
  do {                                             \
    if (k == 10 && tid == 0) gct[j] = global_ns(); \
  } while (0)
#else
#define GC_MARK(j) \
  do {             \
  } while (0)
#endif

template <int DIM, int T>
__global__ void __launch_bounds__(T, 1)
k_gen_cluster(const __grid_constant__ GenBlocks B, const __grid_constant__ GcSend SL, const double *__restrict__ s_loc,
              double *rb0, double *rb1, double *pb0, double *pb1, double *qb0, double *qb1,
              const double *__restrict__ Dinv, double *x, const __grid_constant__ K0Dense2 K2,
              const __grid_constant__ K0HadSym H, CgScalars *S, int max_iter, double rtol, double *hist) {
  namespace cg = cooperative_groups;
  constexpr int NC = 1 << DIM, ND = NC * DIM, CH = GcChunk<DIM, T>::CH, YS = GcChunk<DIM, T>::YS;
  constexpr int OPT = kGcOwnPerThread;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  const int tid = threadIdx.x, nb = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const GfMeta mt = B.meta[rank];
  const GfSections sec = gf_sections<DIM>(mt.n_own, mt.n_halo, mt.n_virt, mt.n_el, mt.n_inc, CH);
  const GcLayout L = gc_layout<DIM, T>(B.max_rec16, B.max_el, B.max_loc, B.max_own, SL.max_halo, SL.max_send);
  unsigned char *rec = gsm_raw;
  double *sl = reinterpret_cast<double *>(gsm_raw + L.sl);
  double *P = reinterpret_cast<double *>(gsm_raw + L.P);
  double *R = reinterpret_cast<double *>(gsm_raw + L.R);
  double *X = reinterpret_cast<double *>(gsm_raw + L.X);
  double *Q = reinterpret_cast<double *>(gsm_raw + L.Q);
  double *Zs = reinterpret_cast<double *>(gsm_raw + L.Zs);
  double *Ds = reinterpret_cast<double *>(gsm_raw + L.Ds);
  double *Y = reinterpret_cast<double *>(gsm_raw + L.Y);
  double *PH = reinterpret_cast<double *>(gsm_raw + L.PH);   // [2][max_halo * DIM]
  double *PT = reinterpret_cast<double *>(gsm_raw + L.PT);   // [2][16][8]
  double *bc = reinterpret_cast<double *>(gsm_raw + L.bc);   // alpha, beta, done, -, the 5 summed dots
  uint32_t *send = reinterpret_cast<uint32_t *>(gsm_raw + L.send);
  unsigned long long *bar = reinterpret_cast<unsigned long long *>(gsm_raw + L.bar);   // record, halo[2], dots[2]
  const size_t ph_stride = gc_even8((size_t)SL.max_halo * DIM) / 8;
  const ushort4 *virt = reinterpret_cast<const ushort4 *>(rec + sec.virt);
  const uint16_t *corner = reinterpret_cast<const uint16_t *>(rec + sec.corner);
  const uint16_t *iptr = reinterpret_cast<const uint16_t *>(rec + sec.iptr);
  const uint16_t *inc = reinterpret_cast<const uint16_t *>(rec + sec.inc);
  const int nOwn = mt.n_own, nHalo = mt.n_halo, nVirt = mt.n_virt, nE = mt.n_el;
  const int s0 = SL.off[rank], nSend = SL.off[rank + 1] - s0;
  GF_CHECK(sec.total <= 16 * B.max_rec16 && nE <= B.max_el && nOwn <= B.max_own && nOwn <= OPT * T);
  GF_CHECK(nOwn + nHalo + nVirt <= B.max_loc && nb == B.n_blk && nHalo <= SL.max_halo && nSend <= SL.max_send);
  if (tid == 0) {
    const unsigned s_bytes = 8u * (unsigned)((nE + 1) & ~1);
#pragma unroll
    for (int j = 0; j < 5; ++j) mbar_init(&bar[j], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    fence_proxy_async();
    mbar_arrive_expect_tx(&bar[0], (unsigned)sec.total + s_bytes);
    bulk_load_1d(rec, B.rec + mt.rec_off16, (unsigned)sec.total, &bar[0]);
    if (s_bytes) bulk_load_1d(sl, s_loc + mt.el_off, s_bytes, &bar[0]);
  }
  // the owned state: r_{-1} = r0 (rb1), p_{-1} = pb1, q_{-1} = qb1, x, Dinv;
  // this CTA's send list
  const int64_t g0 = (int64_t)mt.node0 * DIM;
#pragma unroll
  for (int u = 0; u < OPT; ++u) {
    const int o = tid + u * T;
    if (o >= nOwn) continue;
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      const int64_t g = g0 + (int64_t)o * DIM + i;
      R[o * DIM + i] = rb1[g];
      P[o * DIM + i] = pb1[g];
      Q[o * DIM + i] = qb1[g];
      X[o * DIM + i] = x[g];
      Ds[o * DIM + i] = Dinv[g];
    }
  }
  for (int e = tid; e < nSend; e += T) send[e] = SL.ent[s0 + e];
  double alpha = __ldcg(&S->alpha), beta = __ldcg(&S->beta);
  const bool stopped = cg_stopped(S);   // the same in every CTA (S is written after the loop only)
  // the fields cg_step_eval reads that stay constant during the solve
  const CgConst cc = cg_const(S, rtol);
  int klast = -1;
  CgStepOut so_last{};                  // CTA 0, thread 0: the last step, committed to S after the loop
  const bool hist_on = rank == 0 && tid == 0 && hist && __ldcg(&S->history);
#ifdef TOMESH_GC_TRACE
  unsigned long long gct[12] = {};
#endif
  mbar_wait(&bar[0], 0);
  cl.sync();   // every CTA's mbarriers initialised and state loaded before the first push
  if (!stopped) {
    for (int k = 0; k < max_iter; ++k) {
      klast = k;
      const int par = k & 1;
      const unsigned ph = (k >> 1) & 1;
      double *phb = PH + par * ph_stride;
      double *ptb = PT + par * 16 * 8;
      GC_MARK(0);
      if (tid == 0) {   // this iteration's expected bytes: the halo values, nb x 5 dots
        mbar_arrive_expect_tx(&bar[1 + par], (unsigned)(8 * DIM * nHalo));
        mbar_arrive_expect_tx(&bar[3 + par], (unsigned)(40 * nb));
      }
      // 1. owned nodes: r_k, z_k, p_k, x += alpha p_{k-1}; rho_k, rr_k
      double rho = 0.0, rr = 0.0;
#pragma unroll
      for (int u = 0; u < OPT; ++u) {
        const int o = tid + u * T;
        if (o >= nOwn) continue;
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
          const int a = o * DIM + i;
          const double rn = fma(-alpha, Q[a], R[a]);   // q is 0 on non-free DOFs, so r stays 0 there
          const double z = Ds[a] * rn;
          const double pold = P[a];
          R[a] = rn;
          Zs[a] = z;
          P[a] = fma(beta, pold, z);
          if (alpha != 0.0) X[a] = fma(alpha, pold, X[a]);
          rho = fma(rn, z, rho);
          rr = fma(rn, rn, rr);
        }
      }
      __syncthreads();
      GC_MARK(1);
      // 2. push the owned p_k the other CTAs need into their halo buffers
      for (int e = tid; e < nSend; e += T) {
        const uint32_t ent = send[e];
        const int src = (int)(ent & 0xfffu), dst = (int)((ent >> 12) & 0x7fffu), r = (int)(ent >> 27);
        GF_CHECK(src < nOwn && r < nb && r != rank && dst < SL.max_halo);
        const uint32_t ra = gc_mapa(phb + (size_t)dst * DIM, r), rb = gc_mapa(&bar[1 + par], r);
        if (DIM == 2) {
          gc_st_async2(ra, P[src * DIM], P[src * DIM + 1], rb);
        } else {
#pragma unroll
          for (int i = 0; i < DIM; ++i) gc_st_async(ra + 8 * i, P[src * DIM + i], rb);
        }
      }
      // ... and wait for this CTA's halo values; they go to the local slots
      mbar_wait(&bar[1 + par], ph);
      GC_MARK(2);
      for (int j = tid; j < nHalo * DIM; j += T) P[nOwn * DIM + j] = phb[j];
      __syncthreads();
      GC_MARK(3);
      {
        const int vb = (nOwn + nHalo) * DIM;
        for (int v = tid; v < nVirt; v += T) {
          const ushort4 pv = virt[v];
          const int np = pv.z == 0xffff ? 2 : 4;
          const double w = np == 2 ? 0.5 : 0.25;
          const int par4[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
          for (int i = 0; i < DIM; ++i) {
            double acc = 0.0;
            for (int q = 0; q < np; ++q) acc = fma(w, P[par4[q] * DIM + i], acc);
            P[vb + v * DIM + i] = acc;
          }
        }
      }
      __syncthreads();
      // 3. elements by chunks of CH; owned nodes sum their incidences of the
      //    chunk in ascending order (C^T, weights 1, 1/2, 1/4)
      double qa[OPT][DIM];
#pragma unroll
      for (int u = 0; u < OPT; ++u)
#pragma unroll
        for (int i = 0; i < DIM; ++i) qa[u][i] = 0.0;
      for (int c0 = 0; c0 < nE; c0 += CH) {
        const int le = c0 + tid;
        if (tid < CH && le < nE) {
          double y[ND];
          if constexpr (DIM == 3) {
            const uint4 cs = *reinterpret_cast<const uint4 *>(corner + (size_t)le * NC);
            const unsigned sw[4] = {cs.x, cs.y, cs.z, cs.w};
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              const int slot = (int)((sw[c >> 1] >> (16 * (c & 1))) & 0xffffu);
#pragma unroll
              for (int i = 0; i < DIM; ++i) y[DIM * c + i] = P[slot * DIM + i];
            }
            had_apply_inplace(H, y);
          } else {
            const uint2 cs = *reinterpret_cast<const uint2 *>(corner + (size_t)le * NC);
            const unsigned sw[2] = {cs.x, cs.y};
            double v[ND];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              const int slot = (int)((sw[c >> 1] >> (16 * (c & 1))) & 0xffffu);
#pragma unroll
              for (int i = 0; i < DIM; ++i) v[DIM * c + i] = P[slot * DIM + i];
            }
            dense_apply<ND>(K2.K, v, y);
          }
          const double se = sl[le];
          double *dst = Y + (size_t)tid * YS;
#pragma unroll
          for (int a = 0; a < ND; ++a) dst[a] = se * y[a];
        }
        __syncthreads();
        gf_ct_chunk<DIM, OPT, T>(iptr, inc, Y, nOwn, c0 / CH, qa);
        __syncthreads();
      }
      GC_MARK(4);
      // 4. owners: q_k (0 on non-free DOFs), p.q, q.z, q.Dinv q
      double dots[5] = {rho, rr, 0.0, 0.0, 0.0};
#pragma unroll
      for (int u = 0; u < OPT; ++u) {
        const int o = tid + u * T;
        if (o >= nOwn) continue;
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
          const int a = o * DIM + i;
          const double d = Ds[a];
          const double q = d != 0.0 ? qa[u][i] : 0.0;
          Q[a] = q;
          dots[2] = fma(P[a], q, dots[2]);
          dots[3] = fma(Zs[a], q, dots[3]);
          dots[4] = fma(d * q, q, dots[4]);
        }
      }
      GC_MARK(5);
      block_sum<5>(dots);   // the block's sums end up in every lane of warp 0
      GC_MARK(6);
      // 5. this CTA's dots to slot `rank` of every CTA (lane b of warp 0 to
      //    CTA b); wait for all nb
      if (tid < nb) {
        const uint32_t ra = gc_mapa(ptb + 8 * rank, tid), rb = gc_mapa(&bar[3 + par], tid);
        gc_st_async2(ra, dots[0], dots[1], rb);
        gc_st_async2(ra + 16, dots[2], dots[3], rb);
        gc_st_async(ra + 32, dots[4], rb);
      }
      mbar_wait(&bar[3 + par], ph);
      GC_MARK(7);
      // 6. the step: lane j < 5 adds dot j over the nb slots in rank order;
      //    lane 0 evaluates it
      if (tid < 5) {
        double t = 0.0;
        for (int b = 0; b < nb; ++b) t += ptb[8 * b + tid];
        bc[4 + tid] = t;
      }
      __syncwarp();
      if (tid == 0) {
        const double tot[5] = {bc[4], bc[5], bc[6], bc[7], bc[8]};
        CgStepOut so;
        cg_step_eval_c(cc, k, tot, so);
        // S is read by nobody during the loop: the step is committed once,
        // after it; the residual history (if asked for) is written as it comes
        so_last = so;
        if (hist_on && k >= 1 && so.fail != -5) hist[k - 1] = sqrt(so.rr / cc.bnorm2);
        bc[0] = so.alpha;
        bc[1] = so.beta;
        bc[2] = so.done ? 1.0 : 0.0;
      }
      __syncthreads();
      GC_MARK(8);
#ifdef TOMESH_GC_TRACE
      if (k == 10 && tid == 0 && (rank == 0 || rank == nb - 1))
        printf("gc trace rank %d/%d own %d el %d halo %d send %d: upd %llu push+wait %llu copy %llu elem %llu "
               "q %llu bsum %llu dots %llu step %llu ns\n",
               rank, nb, nOwn, nE, nHalo, nSend, gct[1] - gct[0], gct[2] - gct[1], gct[3] - gct[2],
               gct[4] - gct[3], gct[5] - gct[4], gct[6] - gct[5], gct[7] - gct[6], gct[8] - gct[7]);
#endif
      if (bc[2] != 0.0) break;
      alpha = bc[0];
      beta = bc[1];
    }
  }
  if (klast >= 0 && rank == 0 && tid == 0) {
    S->thresh2 = cc.thresh2;
    cg_step_commit(S, klast, so_last, nullptr);
  }
  // write back: x; r, p, q of the last iteration into buffer klast & 1 (what
  // k_final_gen reads after a fixed count)
  if (klast >= 0) {
    double *rw = (klast & 1) ? rb1 : rb0, *pw = (klast & 1) ? pb1 : pb0, *qw = (klast & 1) ? qb1 : qb0;
#pragma unroll
    for (int u = 0; u < OPT; ++u) {
      const int o = tid + u * T;
      if (o >= nOwn) continue;
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        const int a = o * DIM + i;
        const int64_t g = g0 + a;
        x[g] = X[a];
        rw[g] = R[a];
        pw[g] = P[a];
        qw[g] = Q[a];
      }
    }
  }
  cl.sync();   // no CTA leaves while a push to it may be in flight
}

}  // namespace tomesh
