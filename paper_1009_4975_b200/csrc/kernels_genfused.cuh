// General (AMR) path, one PCG iteration = ONE kernel (k_gen_fused).  Same
// operator as every other path (Eq. 8 with Dirichlet rows, PAPER.md:678-682:
// A = Pi_F C^T K C Pi_F + (I - Pi_F), the hanging-node interpolation C of
// Eq. 6, :653-663, applied at the element gather and transposed at the
// scatter), same Hestenes-Stiefel recurrences on the rescaled system
// (reading R3) in the single-kernel form of the structured
// path (kernels_struct3d.cuh, kernels_cg.cuh cg_single_step).
//
// Decomposition ("owner computes", built on the host at upload, tomesh.cu
// build_gen_blocks): the canonical node order (Morton, C3) is cut into
// contiguous ranges; CTA b OWNS the nodes [node0[b], node0[b+1]).  It stages
//   * every element that contributes to an owned node (directly, or through a
//     hanging corner whose parent is owned) -- the halo elements are
//     recomputed by each CTA that needs them, so no element result ever
//     leaves the CTA and no atomics or element buffers are needed;
//   * the "local nodes": owned nodes (slots [0, nOwn), contiguous in global
//     memory), halo nodes (the other non-hanging corners and parents,
//     ascending global id) and one virtual slot per hanging corner node
//     (ascending id) holding the Eq. 6 interpolation of its parents.
// Per iteration k (alpha_{k-1}, beta_{k-1} from the previous kernel's last
// block; buffers ping-pong as in K1: read (k+1)&1, write k&1):
//   1. every local node: r_k = r_{k-1} - alpha q_{k-1}, z_k = Dinv r_k,
//      p_k = z_k + beta p_{k-1} into shared memory; owners also store r_k,
//      p_k, x += alpha p_{k-1} and reduce rho_k = r_k.z_k, rr_k;
//   2. virtual slots: p of a hanging node = sum_parents w p_parent (Eq. 6);
//   3. elements in chunks of kGfChunk: lane c of an element group gathers
//      corner c from shared memory, the element product (Hadamard form of K0
//      in 3D, dense in 2D, across the group by warp shuffles) times s_e goes
//      to a shared chunk buffer; then every owned node sums its block-local
//      incidences (element, corner, weight 1 or the Eq. 6 weight: C^T) of that
//      chunk in ascending order -- a fixed summation order, so the result is
//      bit-reproducible;
//   4. owners store q_k (0 on non-free DOFs) and reduce p.q, q.z, q.Dinv q;
//      one grid reduction; the last block forms alpha_k and beta_k
//      (cg_single_step, one-step rho expansion) and tests rr_k.
// PLAIN mode (operator-level calls, warm start, true residual, MINRES):
// step 1 loads v, step 4 stores q = C^T K C v on the owned nodes, no dots.
#pragma once
#include <cooperative_groups.h>

#include "device_common.cuh"
#include "element.h"
#include "kernels_cg.cuh"
#include "kernels_general.cuh"
#include "kernels_shard.cuh"
#include "tomesh_types.cuh"

namespace tomesh {

#ifndef TOMESH_GF_THREADS
#define TOMESH_GF_THREADS 256
#endif
constexpr int kGfThreads = TOMESH_GF_THREADS;
constexpr int kGfOwnPerThread = 1;                       // owned nodes per thread in the C^T sums
constexpr int kGfMaxOwn = kGfThreads * kGfOwnPerThread;  // (block targets are <= 224 nodes)
#ifndef TOMESH_GF_LOCMAX
#define TOMESH_GF_LOCMAX 1536
#endif
constexpr int kGfMaxLoc = TOMESH_GF_LOCMAX;              // local node slots per block (uint16 slots)
constexpr int kGfPersistMaxBlocks = 32;                  // k_gen_persist only up to this many blocks
// Launched path: every block evaluates the previous step itself (no step
// kernel) up to this many blocks; beyond, the O(blocks^2) partial reads cost
// more than the step launch (c2, 85 blocks: 8.98 -> 8.07 us per iteration;
// c4, 1,131 blocks: 62.4 -> 78.2; c4L, 7,099 blocks: 320 -> 772)
constexpr int kGfStepInMaxBlocks = 256;
#ifndef TOMESH_GF_OWN3
#define TOMESH_GF_OWN3 256      // with the 2-CTA shared-memory cap (TOMESH_GF_SMEMMAX): c4L 224 / 240 / 256: 270 / 264 / 259 us
#endif
#ifndef TOMESH_GF_OWN2
#define TOMESH_GF_OWN2 224
#endif
constexpr int kGfOwnTarget3 = TOMESH_GF_OWN3;           // owned nodes per block before splitting (3D)
constexpr int kGfOwnTarget2 = TOMESH_GF_OWN2;           // (2D)
#ifndef TOMESH_GF_OWN_MIN
#define TOMESH_GF_OWN_MIN 64
#endif
constexpr int kGfOwnMin = TOMESH_GF_OWN_MIN;             // smallest block target (mid-size meshes)
#ifndef TOMESH_GF_CH
#define TOMESH_GF_CH 256
#endif
#ifndef TOMESH_GF_MINB
#define TOMESH_GF_MINB 2
#endif
#ifndef TOMESH_GF_SMEMMAX
// blocks are split until their shared memory fits two CTAs per SM (228 KB
// less 1 KB reserved and the static shared memory per CTA): one block above
// it would halve the residency of the whole grid (c4L with 240-node blocks:
// one CTA per SM, 426 vs 270 us per iteration)
#define TOMESH_GF_SMEMMAX 113664
#endif
#ifndef TOMESH_GF_HPRE
#define TOMESH_GF_HPRE 3        // halo DOFs per thread loaded ahead of the owned update (0, 3, 4, 5: c4L 293, 292, 295, 307 us)
#endif
#ifndef TOMESH_GF_PF
#define TOMESH_GF_PF 1          // next-wave L2 prefetch, in residencies ahead (GenBlocks::pf, set at upload; 0: off)
#endif
#ifndef TOMESH_GF_ELMAX
#define TOMESH_GF_ELMAX 2047    // capping blocks at one chunk (256) split them too finely: c4 62 -> 92 us
#endif
constexpr int kGfElMax = TOMESH_GF_ELMAX;               // elements per block (chunks of TOMESH_GF_CH)

template <int DIM>
struct GfChunk {
  static constexpr int NC = 1 << DIM;
  static constexpr int CH = TOMESH_GF_CH;               // elements per chunk: one per thread (threads < CH)
  static constexpr int YS = NC * DIM + 1;               // doubles per element result (odd: no bank conflicts)
};

// Byte offsets of the sections of a block record (tomesh_types.cuh GfMeta).
struct GfSections {
  int halo, virt, corner, iptr, inc, total;
};
// ch: elements per chunk of the kernel that reads the record (the incidence
// lists are chunk-major, tomesh_types.cuh GfMeta).
__host__ __device__ inline int gf_nchunks(int n_el, int ch) { return (n_el + ch - 1) / ch; }
template <int DIM>
__host__ __device__ inline GfSections gf_sections(int n_own, int n_halo, int n_virt, int n_el, int n_inc, int ch) {
  GfSections s;
  s.halo = 0;
  s.virt = s.halo + gf_pad16(4 * n_halo);
  s.corner = s.virt + gf_pad16(8 * n_virt);
  s.iptr = s.corner + gf_pad16(2 * (1 << DIM) * n_el);
  s.inc = s.iptr + gf_pad16(2 * gf_nchunks(n_el, ch) * (n_own + 1));
  s.total = s.inc + gf_pad16(2 * n_inc);
  return s;
}

// Dynamic shared memory of k_gen_fused in bytes: the block record, s_e of
// the block's elements, local node values P, one chunk of element results,
// the mbarrier.
template <int DIM>
__host__ __device__ constexpr size_t gf_smem_bytes(int max_rec16, int max_el, int max_loc, int max_own) {
  return (size_t)16 * max_rec16 + 8 * (size_t)((max_el + 1) & ~1) +
         8 * ((size_t)max_loc * DIM + 2 * (size_t)max_own * DIM + (size_t)GfChunk<DIM>::CH * GfChunk<DIM>::YS) + 16;
}

// Lane c of an 2^DIM-lane group holds v = the element's corner c values;
// returns y = (K0 v)[corner c] (unit modulus, h = 1).  3D: Walsh-Hadamard
// stages as xor-shuffles, lane c = Hadamard mode c (element.h); 2D: dense.
template <int DIM>
__device__ __forceinline__ void gf_elem_lane(const double (&v_in)[DIM], int c, const K0Dense2 &K2, const K0HadSym &H,
                                             double (&y)[DIM]) {
  double v[DIM];
#pragma unroll
  for (int i = 0; i < DIM; ++i) v[i] = v_in[i];
  if constexpr (DIM == 3) {
#pragma unroll
    for (int b = 1; b < 8; b <<= 1)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double o = __shfl_xor_sync(0xffffffffu, v[i], b);
        v[i] = (c & b) ? o - v[i] : v[i] + o;
      }
    const int m = c;
    const int bit[3] = {m & 1, (m >> 1) & 1, (m >> 2) & 1};
    const int pop = bit[0] + bit[1] + bit[2];
    double xo[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = i + 1; j < 3; ++j) {
        const int mask = (1 << i) | (1 << j);
        xo[i][j] = __shfl_xor_sync(0xffffffffu, v[j], mask);
        xo[j][i] = __shfl_xor_sync(0xffffffffu, v[i], mask);
      }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int b = bit[i], nn = pop - b;
      const double dco = b ? (nn == 0 ? H.d[1][0] : nn == 1 ? H.d[1][1] : H.d[1][2])
                           : (nn == 0 ? 0.0 : nn == 1 ? H.d[0][1] : H.d[0][2]);
      double acc = dco * v[i];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if (j == i) continue;
        const int t = 3 - i - j;
        const double oco = b ? (bit[t] ? H.o[1][1] : H.o[1][0]) : (bit[t] ? H.o[0][1] : H.o[0][0]);
        acc = (bit[j] != b) ? fma(oco, xo[i][j], acc) : acc;
      }
      y[i] = acc;
    }
#pragma unroll
    for (int b = 1; b < 8; b <<= 1)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double o = __shfl_xor_sync(0xffffffffu, y[i], b);
        y[i] = (c & b) ? o - y[i] : y[i] + o;
      }
  } else {
    const int base = (threadIdx.x & 31) & ~3;
    double vv[4][2];
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
#pragma unroll
      for (int j = 0; j < 2; ++j) vv[cc][j] = __shfl_sync(0xffffffffu, v[j], base + cc);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc = fma(K2.K[(2 * c + i) * 8 + 2 * cc + j], vv[cc][j], acc);
      y[i] = acc;
    }
  }
}

#ifdef TOMESH_GF_TRACE
// A/B instrumentation build only: per-block phase timestamps of the last launch.
__device__ unsigned long long g_gf_trace[16384][8];
#define GF_MARK(k)                                                                     \
  do {                                                                                 \
    if (threadIdx.x == 0 && blockIdx.x < 16384) g_gf_trace[blockIdx.x][k] = global_ns(); \
  } while (0)
#else
#define GF_MARK(k) \
  do {             \
  } while (0)
#endif

#ifdef TOMESH_DEBUG_CHECKS
// checking build (sanitizer substitute): trap on an index outside its array
#define GF_CHECK(cond)                                                                            \
  do {                                                                                            \
    if (!(cond)) {                                                                                \
      printf("k_gen_fused check failed: %s (block %d thread %d)\n", #cond, blockIdx.x, threadIdx.x); \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define GF_CHECK(cond) \
  do {                 \
  } while (0)
#endif

// weight code 0, 1, 2 -> 1, 1/2, 1/4 (2^-code: the exponent field alone)
__device__ __forceinline__ double gf_weight(unsigned code) {
  return __longlong_as_double((long long)(0x3ffu - code) << 52);
}

// C^T of one chunk: owned node o = tid + u * T adds its incidences of chunk
// `ch` (chunk-major CSR: cp = iptr + ch (n_own + 1); entry = double offset of
// the corner's result row in Y | weight code << 14), in ascending element
// order -- the same order across chunks as one ascending list, so the sum
// is fixed by the mesh.
template <int DIM, int OPT, int T>
__device__ __forceinline__ void gf_ct_chunk(const uint16_t *__restrict__ iptr, const uint16_t *__restrict__ inc,
                                            const double *__restrict__ Y, int nOwn, int ch, double (&qa)[OPT][DIM]) {
  const uint16_t *cp = iptr + (size_t)ch * (nOwn + 1);
#pragma unroll
  for (int u = 0; u < OPT; ++u) {
    const int o = threadIdx.x + u * T;
    if (o >= nOwn) continue;
    const int kb = cp[o], ke = cp[o + 1];
#pragma unroll 2
    for (int k = kb; k < ke; ++k) {
      const unsigned ent = inc[k];
      const double w = gf_weight(ent >> 14);
      const double *src = Y + (ent & 0x3fffu);
#pragma unroll
      for (int i = 0; i < DIM; ++i) qa[u][i] = fma(w, src[i], qa[u][i]);
    }
  }
}

// Shared-memory view of one block of the general path (its record, s_e, the
// staging arrays) -- set up once per kernel.
struct GfView {
  GfMeta mt;
  double *sl, *P, *Zs, *Ds, *Y;
  unsigned long long *bar;
  const int32_t *halo;
  const ushort4 *virt;
  const uint16_t *corner, *iptr, *inc;
};
template <int DIM>
__device__ __forceinline__ GfView gf_view(const GenBlocks &B, const GfMeta &mt, unsigned char *gsm_raw, GfSections &sec) {
  constexpr int CH = GfChunk<DIM>::CH, YS = GfChunk<DIM>::YS;
  GfView V;
  V.mt = mt;
  sec = gf_sections<DIM>(mt.n_own, mt.n_halo, mt.n_virt, mt.n_el, mt.n_inc, CH);
  unsigned char *rec = gsm_raw;
  V.sl = reinterpret_cast<double *>(gsm_raw + 16 * (size_t)B.max_rec16);
  V.P = V.sl + ((B.max_el + 1) & ~1);
  V.Zs = V.P + (size_t)B.max_loc * DIM;
  V.Ds = V.Zs + (size_t)B.max_own * DIM;
  V.Y = V.Ds + (size_t)B.max_own * DIM;
  V.bar = reinterpret_cast<unsigned long long *>(V.Y + (size_t)CH * YS);
  V.halo = reinterpret_cast<const int32_t *>(rec + sec.halo);
  V.virt = reinterpret_cast<const ushort4 *>(rec + sec.virt);
  V.corner = reinterpret_cast<const uint16_t *>(rec + sec.corner);
  V.iptr = reinterpret_cast<const uint16_t *>(rec + sec.iptr);
  V.inc = reinterpret_cast<const uint16_t *>(rec + sec.inc);
  return V;
}

// Thread 0: issue the bulk copies of the block record and s_e (one mbarrier phase).
template <int DIM>
__device__ __forceinline__ void gf_issue_record(const GenBlocks &B, const GfView &V, const GfSections &sec,
                                                const double *s_loc, unsigned char *gsm_raw) {
  const unsigned s_bytes = 8u * (unsigned)((V.mt.n_el + 1) & ~1);
  mbar_init(V.bar, 1);
  fence_proxy_async();
  mbar_arrive_expect_tx(V.bar, (unsigned)sec.total + s_bytes);
  bulk_load_1d(gsm_raw, B.rec + V.mt.rec_off16, (unsigned)sec.total, V.bar);
  if (s_bytes) bulk_load_1d(V.sl, s_loc + V.mt.el_off, s_bytes, V.bar);
}

// Lanes 0-6 of warp 0: bulk L2 prefetch of block bn's record, s_e and owned
// r, q, p, Dinv, x ranges.  bn = blockIdx.x + B.pf is the block that will
// take over this SM slot about one residency later, so its dependent load
// chain (meta -> record -> owned/halo loads) starts from L2 instead of HBM;
// its halo rows are mostly owned rows of the blocks next to it, prefetched
// by their own predecessors.  Blocks of the last residency prefetch the
// first ones of the NEXT launch (from the buffers this launch writes, which
// that launch reads).  Only a cache fill: no effect on results.
template <int DIM>
__device__ __forceinline__ void gf_prefetch_block(const GenBlocks &B, int bn, const double *s_loc,
                                                  const double *ro, const double *qo, const double *po,
                                                  const double *Dinv, const double *x) {
  const int lane = threadIdx.x;
  if (lane >= 7 || bn >= B.n_blk) return;
  const GfMeta mn = B.meta[bn];
  uintptr_t a, e;
  if (lane == 0) {
    const GfSections sec = gf_sections<DIM>(mn.n_own, mn.n_halo, mn.n_virt, mn.n_el, mn.n_inc, GfChunk<DIM>::CH);
    a = reinterpret_cast<uintptr_t>(B.rec + mn.rec_off16);
    e = a + (unsigned)sec.total;
  } else if (lane == 1) {
    a = reinterpret_cast<uintptr_t>(s_loc + mn.el_off);
    e = a + 8u * (unsigned)((mn.n_el + 1) & ~1);
  } else {
    const double *v = lane == 2 ? ro : lane == 3 ? qo : lane == 4 ? po : lane == 5 ? Dinv : x;
    a = reinterpret_cast<uintptr_t>(v + (int64_t)mn.node0 * DIM) & ~(uintptr_t)15;
    e = (reinterpret_cast<uintptr_t>(v + (int64_t)(mn.node0 + mn.n_own) * DIM) + 15) & ~(uintptr_t)15;
  }
  if (e > a) bulk_prefetch_l2(reinterpret_cast<const void *>(a), (unsigned)(e - a));
}

// Loads of vectors another block may have written in the same kernel (the
// persistent solver: after a grid barrier) go through L2; otherwise the
// read-only path.
template <bool COH>
__device__ __forceinline__ double gf_ld(const double *p) { return COH ? __ldcg(p) : __ldg(p); }

// The owned DOFs' r, q, p, Dinv of one block, DOF-linear (owned DOF j = tid +
// v * kGfThreads: coalesced), loaded before the stop test and the step are
// known (they do not depend on alpha, beta): gf_block_iter takes them from here.
template <int DIM>
struct GfOwned {
  static constexpr int OD = kGfMaxOwn * DIM / kGfThreads;   // owned DOFs per thread
  double r[OD], q[OD], p[OD], d[OD], x[OD];
};
template <int DIM, bool COH>
__device__ __forceinline__ void gf_load_owned(const GfMeta &mt, const double *__restrict__ ro,
                                              const double *__restrict__ qo, const double *__restrict__ po,
                                              const double *__restrict__ Dinv, const double *__restrict__ x,
                                              GfOwned<DIM> &w) {
  const int64_t g0 = (int64_t)mt.node0 * DIM;
  const int nd = mt.n_own * DIM;
#pragma unroll
  for (int v = 0; v < GfOwned<DIM>::OD; ++v) {
    const int j = threadIdx.x + v * kGfThreads;
    w.r[v] = w.q[v] = w.p[v] = w.d[v] = w.x[v] = 0.0;
    if (j < nd) {
      w.r[v] = gf_ld<COH>(ro + g0 + j);
      w.q[v] = gf_ld<COH>(qo + g0 + j);
      w.p[v] = gf_ld<COH>(po + g0 + j);
      w.d[v] = __ldg(Dinv + g0 + j);
      w.x[v] = __ldcg(x + g0 + j);   // written by this block only (owned DOFs)
    }
  }
}

// The first HB halo DOFs of each thread (j = tid + v * kGfThreads of the
// block's halo DOF list): r, q, p, Dinv loaded before the stop test and the
// owned update, so they are in flight while S arrives and the owned stores go
// out (needs the block record: halo ids).
constexpr int kGfHaloPre = TOMESH_GF_HPRE;
struct GfHaloPre {
  double r[kGfHaloPre > 0 ? kGfHaloPre : 1], q[kGfHaloPre > 0 ? kGfHaloPre : 1], p[kGfHaloPre > 0 ? kGfHaloPre : 1],
      d[kGfHaloPre > 0 ? kGfHaloPre : 1];
};
template <int DIM, bool COH>
__device__ __forceinline__ void gf_load_halo(const GfView &V, const double *__restrict__ ro,
                                             const double *__restrict__ qo, const double *__restrict__ po,
                                             const double *__restrict__ Dinv, GfHaloPre &h) {
  const int nh = V.mt.n_halo * DIM;
#pragma unroll
  for (int v = 0; v < kGfHaloPre; ++v) {
    const int j = threadIdx.x + v * kGfThreads;
    h.r[v] = h.q[v] = h.p[v] = h.d[v] = 0.0;
    if (j < nh) {
      const int64_t g = (int64_t)V.halo[j / DIM] * DIM + (j % DIM);
      h.r[v] = gf_ld<COH>(ro + g);
      h.q[v] = gf_ld<COH>(qo + g);
      h.p[v] = gf_ld<COH>(po + g);
      h.d[v] = __ldg(Dinv + g);
    }
  }
}

// One PCG iteration of one block (steps 1-4 of the header comment); the
// block's dots (unreduced, per thread) in `dots`.  wait_par >= 0: the
// record's mbarrier phase of that parity is still outstanding.
// PRE: the owned r, q, p, Dinv come preloaded in `pre` (CG mode).
template <int DIM, int MODE, bool COH, bool PRE = false>
__device__ __forceinline__ void gf_block_iter(const GfView &V, int wait_par, const double *__restrict__ ro,
                                              const double *__restrict__ qo, const double *__restrict__ po,
                                              const double *__restrict__ Dinv, double *__restrict__ rw,
                                              double *__restrict__ pw, double *__restrict__ qw,
                                              double *__restrict__ x, const K0Dense2 &K2, const K0HadSym &H,
                                              double alpha, double beta, double (&dots)[5],
                                              const GfOwned<DIM> *pre = nullptr, const GfHaloPre *hpre = nullptr) {
  constexpr bool CG = MODE == G_CG;
  constexpr int NC = 1 << DIM, ND = NC * DIM, CH = GfChunk<DIM>::CH, YS = GfChunk<DIM>::YS;
  constexpr int OPT = kGfOwnPerThread;
  const int tid = threadIdx.x;
  const GfMeta &mt = V.mt;
  const int nOwn = mt.n_own, nHalo = mt.n_halo, nVirt = mt.n_virt, nE = mt.n_el;
  double *P = V.P, *Zs = V.Zs, *Ds = V.Ds, *Y = V.Y;
  const double *sl = V.sl;
  const int32_t *halo = V.halo;
  const ushort4 *virt = V.virt;
  const uint16_t *corner = V.corner, *iptr = V.iptr, *inc = V.inc;
  const int64_t g0 = (int64_t)mt.node0 * DIM;
  double rho = 0.0, rr = 0.0;
  constexpr int HB = kGfHaloPre;
  GfHaloPre h;
  if (CG && HB > 0) {
    if (hpre) {
      h = *hpre;
    } else {
      if (wait_par >= 0) mbar_wait(V.bar, (unsigned)wait_par);
      wait_par = -1;
      gf_load_halo<DIM, COH>(V, ro, qo, po, Dinv, h);
    }
  }
  // 1. owned DOFs j = tid + v * kGfThreads (DOF-linear, coalesced)
  if (CG) {
    GfOwned<DIM> w;
    if (PRE) w = *pre;
    else gf_load_owned<DIM, COH>(mt, ro, qo, po, Dinv, x, w);
#pragma unroll
    for (int v = 0; v < GfOwned<DIM>::OD; ++v) {
      const int j = tid + v * kGfThreads;
      if (j >= nOwn * DIM) continue;
      const int64_t g = g0 + j;
      const double rn = fma(-alpha, w.q[v], w.r[v]);   // q is 0 on non-free DOFs, so r stays 0 there
      const double z = w.d[v] * rn;
      const double pn = fma(beta, w.p[v], z);
      rw[g] = rn;
      pw[g] = pn;
      if (alpha != 0.0) x[g] = fma(alpha, w.p[v], w.x[v]);
      rho = fma(rn, z, rho);
      rr = fma(rn, rn, rr);
      P[j] = pn;
      Zs[j] = z;
      Ds[j] = w.d[v];
    }
  } else {
    for (int j = tid; j < nOwn * DIM; j += kGfThreads) P[j] = gf_ld<COH>(po + g0 + j);
  }
  GF_MARK(2);
  if (wait_par >= 0) mbar_wait(V.bar, (unsigned)wait_par);
  // ... and the halo nodes
  if (CG) {
#pragma unroll
    for (int v = 0; v < HB; ++v) {
      const int j = tid + v * kGfThreads;
      if (j < nHalo * DIM) P[nOwn * DIM + j] = fma(beta, h.p[v], h.d[v] * fma(-alpha, h.q[v], h.r[v]));
    }
  }
#pragma unroll 4
  for (int j = tid + (CG ? HB : 0) * kGfThreads; j < nHalo * DIM; j += kGfThreads) {
    const int node = halo[j / DIM];
    GF_CHECK(node >= 0 && (node < mt.node0 || node >= mt.node0 + nOwn));
    const int64_t g = (int64_t)node * DIM + (j % DIM);
    double pn;
    if (CG) {
      const double r_o = gf_ld<COH>(ro + g), q_o = gf_ld<COH>(qo + g), p_o = gf_ld<COH>(po + g), d = __ldg(Dinv + g);
      pn = fma(beta, p_o, d * fma(-alpha, q_o, r_o));
    } else {
      pn = gf_ld<COH>(po + g);
    }
    P[nOwn * DIM + j] = pn;
  }
  __syncthreads();
  GF_MARK(3);
  // 2. hanging corners: Eq. 6 interpolation of the parents (ascending parent order)
  {
    const int vb = (nOwn + nHalo) * DIM;
    for (int v = tid; v < nVirt; v += kGfThreads) {
      const ushort4 pv = virt[v];
      const int np = pv.z == 0xffff ? 2 : 4;
      const double w = np == 2 ? 0.5 : 0.25;
      const int par[4] = {pv.x, pv.y, pv.z, pv.w};
      for (int k = 0; k < np; ++k) GF_CHECK(par[k] < nOwn + nHalo);
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        double acc = 0.0;
        for (int k = 0; k < np; ++k) acc = fma(w, P[par[k] * DIM + i], acc);
        P[vb + v * DIM + i] = acc;
      }
    }
  }
  __syncthreads();
  // 3. elements by chunks of CH (one per thread); then owned nodes sum their
  //    incidences of the chunk in ascending order
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
          GF_CHECK(slot < nOwn + nHalo + nVirt);
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
#ifdef TOMESH_DEBUG_CHECKS
    for (int o = tid; o < nOwn; o += kGfThreads) {
      const uint16_t *cp = iptr + (size_t)(c0 / CH) * (nOwn + 1);
      GF_CHECK(cp[o] <= cp[o + 1] && cp[o + 1] <= mt.n_inc);
      for (int k = cp[o]; k < cp[o + 1]; ++k)
        GF_CHECK((inc[k] & 0x3fffu) + DIM <= (unsigned)(min(CH, nE - c0) * YS) && (inc[k] >> 14) <= 2);
    }
#endif
    gf_ct_chunk<DIM, OPT, kGfThreads>(iptr, inc, Y, nOwn, c0 / CH, qa);
    __syncthreads();
  }
  GF_MARK(4);
  // 4. owners: q (masked), dots
  double pq = 0.0, qz = 0.0, qdq = 0.0;
#pragma unroll
  for (int u = 0; u < OPT; ++u) {
    const int o = tid + u * kGfThreads;
    if (o >= nOwn) continue;
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      const int64_t g = g0 + (int64_t)o * DIM + i;
      if (CG) {
        const double d = Ds[o * DIM + i];
        const double q = d != 0.0 ? qa[u][i] : 0.0;
        qw[g] = q;
        pq = fma(P[o * DIM + i], q, pq);
        qz = fma(Zs[o * DIM + i], q, qz);
        qdq = fma(d * q, q, qdq);
      } else {
        qw[g] = qa[u][i];
      }
    }
  }
  dots[0] = rho;
  dots[1] = rr;
  dots[2] = pq;
  dots[3] = qz;
  dots[4] = qdq;
}

// The blocks' dots of one launch summed in a fixed order (thread t takes
// blocks t, t + blockDim, ...; then block_sum): every caller with the same
// blockDim gets the same bits.  Block-wide (barriers); the sums in warp 0.
__device__ __forceinline__ void gf_step_sum(const double *part, int nb, double (&d)[5]) {
#pragma unroll
  for (int k = 0; k < 5; ++k) d[k] = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
#pragma unroll
    for (int k = 0; k < 5; ++k) d[k] += __ldcg(&part[(size_t)5 * b + k]);
  block_sum<5>(d);
}

// This block's dots (summed in a fixed order by the next launch / k_gen_step).
__device__ __forceinline__ void gf_block_dots(double (&dots)[5], double *partials, int nbk, int kit, int step_in,
                                              int b) {
  block_sum<5>(dots);
  double *pk = partials + (step_in ? (size_t)5 * nbk * (kit & 1) : 0);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < 5; ++k) pk[(size_t)5 * b + k] = dots[k];
}

// step_in = 1 (the unsharded solve): the step of iteration kit-1 is evaluated
// at the start of this launch by EVERY block from the previous launch's
// block dots (partials[(kit-1) & 1], the same sum and the same cg_step_eval
// everywhere, so every block takes the same alpha, beta and stop decision);
// block 0 commits it to S.  This launch's dots go to partials[kit & 1].  One
// launch per iteration; k_gen_step evaluates the last step after the loop.
// step_in = 0 (large grids, the shard group): alpha, beta from S, dots to
// partials[0..nb).
template <int DIM, int MODE>
__global__ void __launch_bounds__(kGfThreads, TOMESH_GF_MINB)
k_gen_fused(const __grid_constant__ GenBlocks B, const double *__restrict__ s_loc, const double *__restrict__ ro,
            const double *__restrict__ qo, const double *__restrict__ po, const double *__restrict__ Dinv,
            double *__restrict__ rw, double *__restrict__ pw, double *__restrict__ qw, double *__restrict__ x,
            const __grid_constant__ K0Dense2 K2, const __grid_constant__ K0HadSym H, CgScalars *S,
            double *partials, int kit, double rtol, double *hist, int step_in) {
  constexpr bool CG = MODE == G_CG;
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  const int tid = threadIdx.x;
  GF_MARK(0);
  const GfMeta mt = B.meta[blockIdx.x];
  GfSections sec;
  const GfView V = gf_view<DIM>(B, mt, gsm_raw, sec);
  GF_CHECK(sec.total <= 16 * B.max_rec16 && mt.n_el <= B.max_el && mt.n_own <= B.max_own && mt.n_own <= kGfMaxOwn);
  GF_CHECK(mt.n_own + mt.n_halo + mt.n_virt <= B.max_loc && (mt.el_off & 1) == 0);
  // static block data and s_e (written before the first iteration's launch):
  // one bulk copy each, issued before the wait on the previous iteration
  if (tid == 0) gf_issue_record<DIM>(B, V, sec, s_loc, gsm_raw);
  __syncthreads();
  pdl_wait();
  pdl_release();
  const int nbk = B.n_blk;
  if constexpr (CG) {
    // the owned vectors do not depend on the step or the stop test: their
    // loads are in flight while S is read and the step is evaluated
    GfOwned<DIM> pre;
    gf_load_owned<DIM, false>(mt, ro, qo, po, Dinv, x, pre);
    const bool stopped = cg_stopped(S);
    double alpha = __ldcg(&S->alpha);
    double beta = __ldcg(&S->beta);
#if TOMESH_GF_PF
    if (B.pf > 0 && tid < 32) {
      int bn = blockIdx.x + B.pf;
      const bool wrap = bn >= B.n_blk;   // the next launch's first wave: it reads this launch's write buffers
      if (wrap) bn -= B.n_blk;
      gf_prefetch_block<DIM>(B, bn, s_loc, wrap ? rw : ro, wrap ? qw : qo, wrap ? pw : po, Dinv, x);
    }
#endif
    // the halo prefetch needs the record; the stop test is taken after it so
    // that the S round trip overlaps the halo loads (harmless reads if stopped)
    mbar_wait(V.bar, 0);   // (also: no bulk copy may still be writing when the CTA exits)
    GfHaloPre hpre;
    gf_load_halo<DIM, false>(V, ro, qo, po, Dinv, hpre);
    if (stopped) return;
    GF_MARK(1);
    if (step_in && kit > 0) {
      __shared__ double s_st[3];
      double d[5];
      gf_step_sum(partials + (size_t)5 * nbk * ((kit - 1) & 1), nbk, d);
      if (tid == 0) {
        CgStepOut so;
        cg_step_eval(S, kit - 1, d, rtol, so);
        if (blockIdx.x == 0) cg_step_commit(S, kit - 1, so, hist);
        s_st[0] = so.alpha;
        s_st[1] = so.beta;
        s_st[2] = so.done ? 1.0 : 0.0;
      }
      __syncthreads();
      if (s_st[2] != 0.0) return;
      alpha = s_st[0];
      beta = s_st[1];
    }
    double dots[5];
    gf_block_iter<DIM, MODE, false, true>(V, -1, ro, qo, po, Dinv, rw, pw, qw, x, K2, H, alpha, beta, dots, &pre,
                                          &hpre);
    GF_MARK(5);
    gf_block_dots(dots, partials, nbk, kit, step_in, blockIdx.x);
    GF_MARK(6);
  } else {
    GF_MARK(1);
    double dots[5];
    gf_block_iter<DIM, MODE, false>(V, 0, ro, qo, po, Dinv, rw, pw, qw, x, K2, H, 0.0, 0.0, dots);
  }
}

// The whole general-path PCG loop in one cooperative kernel, for meshes whose
// blocks are all co-resident (c1, c2 and other small meshes: launch and
// drain latency dominate there).  Each block keeps its record in shared
// memory across iterations; per iteration: the block iteration (vectors other
// blocks wrote are read through L2), its dots to part[k & 1], a grid barrier,
// then EVERY block sums the partials in block order and evaluates the step
// (cg_step_eval: the same arithmetic on the same values, hence the same
// alpha, beta and stop decision everywhere); block 0 commits it to S.  x_N
// after a fixed count is completed by k_final_gen, as on the launched path.
template <int DIM>
__global__ void __launch_bounds__(kGfThreads, TOMESH_GF_MINB)
k_gen_persist(const __grid_constant__ GenBlocks B, const double *__restrict__ s_loc, double *rb0, double *rb1,
              double *pb0, double *pb1, double *qb0, double *qb1, const double *__restrict__ Dinv, double *x,
              const __grid_constant__ K0Dense2 K2, const __grid_constant__ K0HadSym H, CgScalars *S, double *part,
              int max_iter, double rtol, double *hist) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  const int tid = threadIdx.x, nb = gridDim.x;
  const GfMeta mt = B.meta[blockIdx.x];
  GfSections sec;
  const GfView V = gf_view<DIM>(B, mt, gsm_raw, sec);
  if (tid == 0) gf_issue_record<DIM>(B, V, sec, s_loc, gsm_raw);
  __syncthreads();
  if (cg_stopped(S)) {   // read by every block before block 0 writes S (after the first barrier)
    mbar_wait(V.bar, 0);
    return;
  }
  double alpha = __ldcg(&S->alpha), beta = __ldcg(&S->beta);
  for (int k = 0; k < max_iter; ++k) {
    const bool odd = k & 1;                           // writes buffer k & 1, reads (k + 1) & 1
    double dots[5];
    gf_block_iter<DIM, G_CG, true>(V, k == 0 ? 0 : -1, odd ? rb0 : rb1, odd ? qb0 : qb1, odd ? pb0 : pb1, Dinv,
                                   odd ? rb1 : rb0, odd ? pb1 : pb0, odd ? qb1 : qb0, x, K2, H, alpha, beta, dots);
    block_sum<5>(dots);
    double *pk = part + (size_t)(k & 1) * 5 * nb;
    if (tid == 0)
#pragma unroll
      for (int j = 0; j < 5; ++j) __stcg(&pk[(size_t)5 * blockIdx.x + j], dots[j]);
    grid.sync();
    double d[5];
    g_sum_partials<5>(pk, nb, d);
    CgStepOut so;
    cg_step_eval(S, k, d, rtol, so);
    if (blockIdx.x == 0 && tid == 0) cg_step_commit(S, k, so, hist);
    if (so.done) break;
    alpha = so.alpha;
    beta = so.beta;
  }
}

// The step of general-path iteration k: the blocks' dots summed in block
// order (thread t adds blocks t, t + 512, ... then a fixed tree), then
// cg_single_step (alpha_k, beta_k, stop test).  One CTA.
// The step of iteration kit from the block dots at `partials` (every
// iteration on large grids; after the last launch of a solve on small ones).
static __global__ void __launch_bounds__(512) k_gen_step(int nb, const double *__restrict__ partials,
                                                                CgScalars *S, int kit, double rtol, double *hist) {
  pdl_wait();
  if (cg_stopped(S)) {
    pdl_release();
    return;
  }
  double acc[5];
  gf_step_sum(partials, nb, acc);
  if (threadIdx.x == 0) cg_single_step(S, kit, acc, rtol, hist);
  __syncthreads();
  pdl_release();
}

// After exactly N iterations (general path): r_N = r_{N-1} - alpha q_{N-1},
// x_N = x_{N-1} + alpha p_{N-1}, rho_N, rr_N (per-DOF Dinv).
// SHARD (general-path shard group, kernels_gshard.cuh): over the owned DOFs
// [0, n); the partial rho_N, rr_N are pushed for k_shard_final (zeros when
// the solve had stopped: every rank pushes every tail sequence).
template <bool SHARD = false>
__global__ void k_final_gen(int64_t n, const double *__restrict__ ro, const double *__restrict__ qo,
                            const double *__restrict__ po, const double *__restrict__ Dinv,
                            double *__restrict__ x, double *partials, CgScalars *S, int n_iter, double rtol,
                            double *hist, const __grid_constant__ ShardComm C, unsigned long long seq) {
  if (cg_stopped(S)) {
    if (SHARD && blockIdx.x == 0 && threadIdx.x == 0) {
      const double zero[2] = {0.0, 0.0};
      shard_push(C, seq, zero, 2);
    }
    return;
  }
  const double alpha = __ldcg(&S->alpha);
  double acc[2] = {0.0, 0.0};
  GRID_STRIDE(i, n) {
    const double d = __ldg(Dinv + i);
    const double rn = fma(-alpha, __ldg(qo + i), __ldg(ro + i));
    if (alpha != 0.0) x[i] = fma(alpha, __ldg(po + i), x[i]);
    acc[0] = fma(rn, d * rn, acc[0]);
    acc[1] = fma(rn, rn, acc[1]);
  }
  if (grid_sum<2>(acc, partials, &S->counter[CNT_U1])) {
    if (SHARD) shard_push(C, seq, acc, 2);
    else cg_final_step(S, n_iter, acc[0], acc[1], rtol, hist);
  }
}

// s_loc[j] = s[el_id[j]]: the SIMP factors in block-local element order (once
// per solve; el_id = -1 on the padding slots, which get 0).
static __global__ void k_gather_s(int64_t n, const int32_t *__restrict__ el_id, const double *__restrict__ s,
                                  double *__restrict__ s_loc) {
  GRID_STRIDE(j, n) {
    const int32_t e = el_id[j];
    s_loc[j] = e >= 0 ? __ldg(s + e) : 0.0;
  }
}

}  // namespace tomesh
