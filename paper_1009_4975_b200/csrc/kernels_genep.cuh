// General (AMR) path, element-partitioned PCG iteration (k_gen_ep): the same
// operator (Eq. 8 with Dirichlet rows; the hanging-node
// interpolation C of Eq. 6, :653-663, at the element gather and C^T at the
// sum) and the same Jacobi preconditioning of the rescaled system
// (reading R3) as k_gen_fused, with the work split so that
// every element is computed exactly once:
//
//  * block b owns the canonical node range [node0, node0 + n_own) (as in
//    k_gen_fused: contiguous, coalesced) and is ASSIGNED the elements whose
//    smallest contributed node (non-hanging corner, or parent of a hanging
//    corner) it owns -- each element in exactly one block, no recompute;
//  * its element results reach every node they contribute to: a node's
//    operator output w(n) = sum over its contributor blocks (ascending) of the
//    block's partial, each partial in its own slot of the slot array W
//    (slot_ptr: node -> its slots).  Nothing is added atomically and every sum
//    has a fixed order, so the result is bit-reproducible.
//
// Because w = A u is only complete one launch later, the iteration is the
// Chronopoulos-Gear form of PCG (one reduction per iteration, both of whose
// inner products are linear in w's partials):
//   s_{K-1} = w_{K-1} + beta_{K-1} s_{K-2}         (s = A p)
//   r_K     = r_{K-1} - alpha_{K-1} s_{K-1}
//   u_K     = Dinv r_K
//   p_{K-1} = u_{K-1} + beta_{K-1} p_{K-2},   x_K = x_{K-1} + alpha_{K-1} p_{K-1}
//   w_K     = A u_K                                 (partials)
//   gamma_K = r_K . u_K,  delta_K = w_K . u_K  (= sum of u . partial), rr_K
//   beta_K  = gamma_K / gamma_{K-1},  alpha_K = gamma_K / (delta_K - beta_K gamma_K / alpha_{K-1})
// (alpha_0 = gamma_0 / delta_0, beta_0 = 0; cg_cgear_step).  In exact
// arithmetic these are the Hestenes-Stiefel iterates (the same x_K, r_K);
// kernel K completes x_K and r_K, so the iteration count and the stop test
// keep the meaning they have on the other paths.
//
// Per block (one kernel per iteration, k_gen_step forms the step):
//   1. owned DOFs (DOF-linear): the slots of w_{K-1}, r_{K-1}, s_{K-2},
//      p_{K-2}, x, Dinv -> s, r, u, p, x (stored), u into shared memory;
//   2. halo nodes (other contributed nodes of the assigned elements): the
//      same u from their slots, r, s, Dinv (the record carries their slot
//      ranges);  3. virtual slots: Eq. 6 interpolation of u;
//   4. assigned elements in chunks (Hadamard K0, x s_e) -> chunk buffer; every
//      local node sums its incidences of the chunk (chunk-major CSR, C^T
//      weights 1, 1/2, 1/4);
//   5. each contributed local node writes its partial to its slot; the dots.
#pragma once
#include "device_common.cuh"
#include "element.h"
#include "kernels_cg.cuh"
#include "kernels_genfused.cuh"
#include "tomesh_types.cuh"

namespace tomesh {

constexpr int kEpAccPerThread = 3;                                  // accumulated local nodes per thread
constexpr int kEpMaxAcc = kGfThreads * kEpAccPerThread;            // owned + halo nodes per block
#ifndef TOMESH_EP_AUTO
#define TOMESH_EP_AUTO 0        // 1: meshes with more than kGfStepInMaxBlocks blocks use k_gen_ep by default
#endif
#ifndef TOMESH_EP_REDUCE
#define TOMESH_EP_REDUCE 1      // the shared nodes' partials summed by k_ep_reduce into a w vector
#endif
#ifndef TOMESH_EP_OWN3
#define TOMESH_EP_OWN3 256
#endif
#ifndef TOMESH_EP_OWN2
#define TOMESH_EP_OWN2 256
#endif

// Sections of an element-partitioned block record (byte offsets; each
// padded to 16).  n_acc = n_own + n_halo local nodes accumulate C^T sums.
//   halo   int32  [n_halo]          canonical node ids, ascending
//   virt   ushort4[n_virt]          parent slots of a hanging corner node
//   corner uint16 [n_el][2^dim]     local slot of every corner (assigned elements, ascending)
//   iptr   uint16 [nch][n_acc + 1]  chunk-major CSR of the local nodes' incidences
//   inc    uint16 [n_inc]           chunk-buffer double offset | weight code << 14
//   wslot  uint32 [n_acc]           slot this block writes for the node (~0: none)
//   hslot  uint32 [n_halo]          first slot of a halo node
//   hcnt   uint8  [n_halo]          its slot count
struct EpSections {
  int halo, virt, corner, iptr, inc, wslot, hslot, hcnt, total;
};
__host__ __device__ inline EpSections ep_sections(int dim, int n_own, int n_halo, int n_virt, int n_el, int n_inc,
                                                  int ch) {
  EpSections s;
  const int nacc = n_own + n_halo;
  s.halo = 0;
  s.virt = s.halo + gf_pad16(4 * n_halo);
  s.corner = s.virt + gf_pad16(8 * n_virt);
  s.iptr = s.corner + gf_pad16(2 * (1 << dim) * n_el);
  s.inc = s.iptr + gf_pad16(2 * gf_nchunks(n_el, ch) * (nacc + 1));
  s.wslot = s.inc + gf_pad16(2 * n_inc);
  s.hslot = s.wslot + gf_pad16(4 * nacc);
  s.hcnt = s.hslot + gf_pad16(4 * n_halo);
  s.total = s.hcnt + gf_pad16(n_halo);
  return s;
}

// Dynamic shared memory: record, s_e, local u values, one chunk of element
// results, the mbarrier.
template <int DIM>
__host__ __device__ constexpr size_t ep_smem_bytes(int max_rec16, int max_el, int max_loc) {
  return (size_t)16 * max_rec16 + 8 * (size_t)((max_el + 1) & ~1) +
         8 * ((size_t)max_loc * DIM + (size_t)GfChunk<DIM>::CH * GfChunk<DIM>::YS) + 16;
}

// w of one DOF from its slots (ascending), 0 on non-free DOFs (Dinv = 0).
// w of one DOF from its slots s0 .. s0 + cnt (its contributor blocks in
// ascending order), 0 on non-free DOFs (Dinv = 0).  The first four slots are
// loaded predicated (independent loads in flight together); the sum is the
// same left-to-right order everywhere (owner, halo readers, k_final_ep).
template <int DIM>
__device__ __forceinline__ double ep_wsum(const double *__restrict__ W, uint32_t s0, int cnt, int i, double d) {
  const double *w = W + (size_t)s0 * DIM + i;
  const double a0 = cnt > 0 ? __ldg(w) : 0.0, a1 = cnt > 1 ? __ldg(w + DIM) : 0.0;
  const double a2 = cnt > 2 ? __ldg(w + 2 * DIM) : 0.0, a3 = cnt > 3 ? __ldg(w + 3 * DIM) : 0.0;
  double acc = a0;
  if (cnt > 1) acc += a1;
  if (cnt > 2) acc += a2;
  if (cnt > 3) acc += a3;
  for (int t = 4; t < cnt; ++t) acc += __ldg(w + (size_t)t * DIM);
  return d != 0.0 ? acc : 0.0;
}

template <int DIM>
__global__ void __launch_bounds__(kGfThreads, TOMESH_GF_MINB)
k_gen_ep(const __grid_constant__ GenBlocks B, const double *__restrict__ s_loc, const int32_t *__restrict__ slot_ptr,
         const double *__restrict__ Wo, double *__restrict__ Ww, const double *__restrict__ ro,
         const double *__restrict__ so, const double *__restrict__ po, const double *__restrict__ Dinv,
         double *__restrict__ rw, double *__restrict__ sw, double *__restrict__ pw, double *__restrict__ x,
         const __grid_constant__ K0Dense2 K2, const __grid_constant__ K0HadSym H, CgScalars *S,
         double *partials, const double *__restrict__ wv) {
  constexpr int NC = 1 << DIM, ND = NC * DIM, CH = GfChunk<DIM>::CH, YS = GfChunk<DIM>::YS;
  constexpr int OA = kEpAccPerThread;
  constexpr int OD = kGfMaxOwn * DIM / kGfThreads;   // owned DOFs per thread
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  const int tid = threadIdx.x;
  GF_MARK(0);
  const GfMeta mt = B.meta[blockIdx.x];
  const int nOwn = mt.n_own, nHalo = mt.n_halo, nVirt = mt.n_virt, nE = mt.n_el, nAcc = nOwn + nHalo;
  const EpSections sec = ep_sections(DIM, nOwn, nHalo, nVirt, nE, mt.n_inc, CH);
  unsigned char *rec = gsm_raw;
  double *sl = reinterpret_cast<double *>(gsm_raw + 16 * (size_t)B.max_rec16);
  double *P = sl + ((B.max_el + 1) & ~1);
  double *Y = P + (size_t)B.max_loc * DIM;
  unsigned long long *bar = reinterpret_cast<unsigned long long *>(Y + (size_t)CH * YS);
  const int32_t *halo = reinterpret_cast<const int32_t *>(rec + sec.halo);
  const ushort4 *virt = reinterpret_cast<const ushort4 *>(rec + sec.virt);
  const uint16_t *corner = reinterpret_cast<const uint16_t *>(rec + sec.corner);
  const uint16_t *iptr = reinterpret_cast<const uint16_t *>(rec + sec.iptr);
  const uint16_t *inc = reinterpret_cast<const uint16_t *>(rec + sec.inc);
  const uint32_t *wslot = reinterpret_cast<const uint32_t *>(rec + sec.wslot);
  const uint32_t *hslot = reinterpret_cast<const uint32_t *>(rec + sec.hslot);
  const uint8_t *hcnt = reinterpret_cast<const uint8_t *>(rec + sec.hcnt);
  GF_CHECK(sec.total <= 16 * B.max_rec16 && nE <= B.max_el && nOwn <= kGfMaxOwn && nAcc <= kEpMaxAcc);
  GF_CHECK(nAcc + nVirt <= B.max_loc && (mt.el_off & 1) == 0);
  if (tid == 0) {
    const unsigned s_bytes = 8u * (unsigned)((nE + 1) & ~1);
    mbar_init(bar, 1);
    fence_proxy_async();
    mbar_arrive_expect_tx(bar, (unsigned)sec.total + s_bytes);
    bulk_load_1d(rec, B.rec + mt.rec_off16, (unsigned)sec.total, bar);
    if (s_bytes) bulk_load_1d(sl, s_loc + mt.el_off, s_bytes, bar);
  }
  __syncthreads();
  pdl_wait();
  pdl_release();
  // 1. owned DOFs: everything is loaded before the stop test and the step
  const int64_t g0 = (int64_t)mt.node0 * DIM;
  double r_o[OD], s_o[OD], p_o[OD], d_o[OD], x_o[OD], w_o[OD];
#pragma unroll
  for (int v = 0; v < OD; ++v) {
    const int j = tid + v * kGfThreads;
    r_o[v] = s_o[v] = p_o[v] = d_o[v] = x_o[v] = w_o[v] = 0.0;
    if (j < nOwn * DIM) {
      const int64_t g = g0 + j;
      const int n = mt.node0 + j / DIM;
      r_o[v] = __ldg(ro + g);
      s_o[v] = __ldg(so + g);
      p_o[v] = __ldg(po + g);
      d_o[v] = __ldg(Dinv + g);
      x_o[v] = __ldcg(x + g);
      if (TOMESH_EP_REDUCE) {
        w_o[v] = __ldg(wv + g);   // summed and masked by k_ep_reduce
      } else {
        const int32_t sa = __ldg(slot_ptr + n), sb = __ldg(slot_ptr + n + 1);
        w_o[v] = ep_wsum<DIM>(Wo, (uint32_t)sa, sb - sa, j % DIM, d_o[v]);
      }
    }
  }
  const bool stopped = cg_stopped(S);
  const double alpha = __ldcg(&S->alpha), beta = __ldcg(&S->beta);
  if (stopped) {
    mbar_wait(bar, 0);
    return;
  }
  GF_MARK(1);
  double gam = 0.0, rr = 0.0, del = 0.0;
#pragma unroll
  for (int v = 0; v < OD; ++v) {
    const int j = tid + v * kGfThreads;
    if (j >= nOwn * DIM) continue;
    const int64_t g = g0 + j;
    const double s = fma(beta, s_o[v], w_o[v]);
    const double r = fma(-alpha, s, r_o[v]);
    const double u = d_o[v] * r;
    const double p = fma(beta, p_o[v], d_o[v] * r_o[v]);
    rw[g] = r;
    sw[g] = s;
    pw[g] = p;
    if (alpha != 0.0) x[g] = fma(alpha, p, x_o[v]);
    gam = fma(r, u, gam);
    rr = fma(r, r, rr);
    P[j] = u;
  }
  GF_MARK(2);
  // 2. halo nodes: the same u from their slots, r, s, Dinv
  mbar_wait(bar, 0);
#pragma unroll 2
  for (int j = tid; j < nHalo * DIM; j += kGfThreads) {
    const int h = j / DIM, i = j % DIM;
    const int64_t g = (int64_t)halo[h] * DIM + i;
    const double d = __ldg(Dinv + g);
    const double w = TOMESH_EP_REDUCE ? __ldg(wv + g) : ep_wsum<DIM>(Wo, hslot[h], hcnt[h], i, d);
    const double s = fma(beta, __ldg(so + g), w);
    const double r = fma(-alpha, s, __ldg(ro + g));
    P[nOwn * DIM + j] = d * r;
  }
  __syncthreads();
  GF_MARK(3);
  // 3. hanging corners: Eq. 6 interpolation of the parents
  {
    const int vb = nAcc * DIM;
    for (int v = tid; v < nVirt; v += kGfThreads) {
      const ushort4 pv = virt[v];
      const int np = pv.z == 0xffff ? 2 : 4;
      const double wgt = np == 2 ? 0.5 : 0.25;
      const int par[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        double acc = 0.0;
        for (int k = 0; k < np; ++k) acc = fma(wgt, P[par[k] * DIM + i], acc);
        P[vb + v * DIM + i] = acc;
      }
    }
  }
  __syncthreads();
  // 4. assigned elements by chunks; local nodes sum their incidences
  double qa[OA][DIM];
  int node_of[OA];
#pragma unroll
  for (int a = 0; a < OA; ++a) {
    node_of[a] = tid + a * kGfThreads;
#pragma unroll
    for (int i = 0; i < DIM; ++i) qa[a][i] = 0.0;
  }
  for (int c0 = 0; c0 < nE; c0 += CH) {
    const int le = c0 + tid;
    if (tid < CH && le < nE) {
      double y[ND];
      if constexpr (DIM == 3) {
        const uint4 cs = *reinterpret_cast<const uint4 *>(corner + (size_t)le * NC);
        const unsigned swd[4] = {cs.x, cs.y, cs.z, cs.w};
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int slot = (int)((swd[c >> 1] >> (16 * (c & 1))) & 0xffffu);
          GF_CHECK(slot < nAcc + nVirt);
#pragma unroll
          for (int i = 0; i < DIM; ++i) y[DIM * c + i] = P[slot * DIM + i];
        }
        had_apply_inplace(H, y);
      } else {
        const uint2 cs = *reinterpret_cast<const uint2 *>(corner + (size_t)le * NC);
        const unsigned swd[2] = {cs.x, cs.y};
        double vv[ND];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int slot = (int)((swd[c >> 1] >> (16 * (c & 1))) & 0xffffu);
#pragma unroll
          for (int i = 0; i < DIM; ++i) vv[DIM * c + i] = P[slot * DIM + i];
        }
        dense_apply<ND>(K2.K, vv, y);
      }
      const double se = sl[le];
      double *dst = Y + (size_t)tid * YS;
#pragma unroll
      for (int a = 0; a < ND; ++a) dst[a] = se * y[a];
    }
    __syncthreads();
    gf_ct_chunk<DIM, OA, kGfThreads>(iptr, inc, Y, nAcc, c0 / CH, qa);
    __syncthreads();
  }
  GF_MARK(4);
  // 5. partials to the slots this block writes; delta = sum of u . partial
#pragma unroll
  for (int a = 0; a < OA; ++a) {
    const int l = node_of[a];
    if (l >= nAcc) continue;
    const uint32_t ws = wslot[l];
    if (ws == 0xffffffffu) continue;
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      Ww[(size_t)ws * DIM + i] = qa[a][i];
      del = fma(P[l * DIM + i], qa[a][i], del);
    }
  }
  GF_MARK(5);
  double dots[5] = {gam, rr, del, 0.0, 0.0};
  block_sum<5>(dots);
  if (tid == 0)
#pragma unroll
    for (int k = 0; k < 5; ++k) partials[(size_t)5 * blockIdx.x + k] = dots[k];
  GF_MARK(6);
}

// w_K = the sum of every node's partial slots (ascending block order, the
// same arithmetic as ep_wsum everywhere), 0 on non-free DOFs: one coalesced
// pass between the block kernel of iteration K and the next one, so that the
// block kernel reads w as a plain vector.
template <int DIM>
__global__ void k_ep_reduce(int64_t n, const int32_t *__restrict__ slot_ptr, const double *__restrict__ W,
                            const double *__restrict__ Dinv, double *__restrict__ wv, const CgScalars *S) {
  pdl_wait();
  pdl_release();
  if (cg_stopped(S)) return;
  GRID_STRIDE(j, n) {
    const int64_t node = j / DIM;
    const int32_t sa = __ldg(slot_ptr + node), sb = __ldg(slot_ptr + node + 1);
    wv[j] = ep_wsum<DIM>(W, (uint32_t)sa, sb - sa, (int)(j % DIM), __ldg(Dinv + j));
  }
}

// After exactly N iterations: r_N, x_N (no operator), rho_N = r_N.Dinv r_N,
// rr_N -> cg_final_step.  Every DOF of the (unsharded) mesh.
template <int DIM>
__global__ void k_final_ep(int64_t n, const int32_t *__restrict__ slot_ptr, const double *__restrict__ Wo,
                           const double *__restrict__ ro, const double *__restrict__ so,
                           const double *__restrict__ po, const double *__restrict__ Dinv, double *__restrict__ x,
                           double *partials, CgScalars *S, int n_iter, double rtol, double *hist) {
  if (cg_stopped(S)) return;
  const double alpha = __ldcg(&S->alpha), beta = __ldcg(&S->beta);
  double acc[2] = {0.0, 0.0};
  GRID_STRIDE(j, n) {
    const double d = __ldg(Dinv + j);
    const int64_t node = j / DIM;
    const int32_t sa = __ldg(slot_ptr + node), sb = __ldg(slot_ptr + node + 1);
    const double w = ep_wsum<DIM>(Wo, (uint32_t)sa, sb - sa, (int)(j % DIM), d);
    const double s = fma(beta, __ldg(so + j), w);
    const double r = fma(-alpha, s, __ldg(ro + j));
    const double p = fma(beta, __ldg(po + j), d * __ldg(ro + j));
    if (alpha != 0.0) x[j] = fma(alpha, p, x[j]);
    acc[0] = fma(r, d * r, acc[0]);
    acc[1] = fma(r, r, acc[1]);
  }
  if (grid_sum<2>(acc, partials, &S->counter[CNT_U1])) cg_final_step(S, n_iter, acc[0], acc[1], rtol, hist);
}

// The step of element-partitioned iteration k (Chronopoulos-Gear, header):
// the blocks' dots {gamma_k, rr_k, delta_k} summed in block order, then
// cg_cgear_step.  One CTA.
static __global__ void __launch_bounds__(512) k_gen_ep_step(int nb, const double *__restrict__ partials,
                                                            CgScalars *S, int kit, double rtol, double *hist) {
  pdl_wait();
  if (cg_stopped(S)) {
    pdl_release();
    return;
  }
  double acc[5];
  gf_step_sum(partials, nb, acc);
  if (threadIdx.x == 0) cg_cgear_step(S, kit, acc, rtol, hist);
  __syncthreads();
  pdl_release();
}

}  // namespace tomesh
