// Device-side helpers: reductions, scalar block of the CG loop.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tomesh {

constexpr int kNumSMs = 148;          // B200
constexpr int kBlock = 256;

// Device-resident state of one Jacobi-PCG solve.  Every scalar of the
// recurrences lives here so that no iteration needs the host.
struct CgScalars {
  double rho;        // r_k . z_k
  double alpha;      // rho / (p . A p)
  double beta;       // rho_{k+1} / rho_k
  double rr;         // ||r_k||^2
  double bnorm2;     // ||b||^2
  double thresh2;    // rtol^2 ||b||^2
  double tmp[4];     // scratch reductions (true residual, compliance, ...)
  int32_t iter;      // completed iterations
  int32_t max_iter;
  int32_t fixed;     // 1: ignore rtol
  int32_t done;      // 1: stop now (set on breakdown / before the first iteration)
  int32_t done_next; // 1: stop after the x/p update of the current iteration
  int32_t status;    // TO_OK or a negative code
  int32_t history;   // record ||r||/||b|| per iteration
  int32_t pad;
  uint32_t counter[8];   // last-block-done counters, one per reduction site
  double ab[2][2];       // {alpha_k, beta_k} of step k in slot k & 1 (the structured kernel's deferred x update)
};

enum { CNT_PQ = 0, CNT_U1 = 1, CNT_INIT = 2, CNT_MISC = 3, CNT_MISC2 = 4, CNT_XCHG = 5 };

#define GRID_STRIDE(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// Programmatic dependent launch (PDL): a kernel launched with the
// programmatic-serialization attribute may be scheduled while its predecessor
// in the stream is still draining; pdl_wait() blocks until the predecessor
// has completed and its memory is visible (a no-op for a normal launch), and
// pdl_release() lets the successor be scheduled as blocks of this kernel free
// their SM resources.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Shared-memory address, mbarrier and bulk-copy (TMA) helpers.
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
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// 1D bulk copy global -> shared (the async proxy, TMA), completion counted in
// bytes on `bar`; dst, src and bytes multiples of 16.
__device__ __forceinline__ void bulk_load_1d(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Bulk prefetch of [src, src + bytes) into L2 (src and bytes multiples of 16).
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

// 8-byte asynchronous copy global -> shared (LDGSTS), and an mbarrier arrival
// triggered when all of this thread's prior cp.async copies have completed
// (.noinc: the arrival is part of the barrier's initial count).
__device__ __forceinline__ void cp_async_8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_arrive_noinc(unsigned long long *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// Named barrier over the first `nthreads` threads (warp-aligned), id 1..15.
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
  return t;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of NV values; the result is valid in thread 0.
__device__ __forceinline__ int lin_tid() { return threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z); }
__device__ __forceinline__ int lin_nthr() { return blockDim.x * blockDim.y * blockDim.z; }

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV]) {
  __shared__ double sh[NV][32];
  const int tid = lin_tid();
  const int lane = tid & 31, wid = tid >> 5;
  const int nw = (lin_nthr() + 31) >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) sh[k][wid] = v[k];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double t = lane < nw ? sh[k][lane] : 0.0;
      v[k] = warp_sum(t);
    }
  }
}

// Grid-wide deterministic sum: every block deposits its partial, the last
// block to arrive adds the partials in a fixed order.  Returns true in
// thread 0 of the last block, with the totals in `v`.
template <int NV>
__device__ __forceinline__ bool grid_sum(double (&v)[NV], double *partials, uint32_t *counter) {
  __shared__ bool s_last;
  block_sum<NV>(v);
  const int tid = lin_tid();
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) partials[(size_t)blockIdx.x * NV + k] = v[k];
    // release: this block's partials (and everything its threads wrote before
    // the barrier in block_sum) are visible before the arrival is counted
    uint32_t t;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(counter) : "memory");
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (int b = tid; b < (int)gridDim.x; b += lin_nthr()) {
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] += __ldcg(&partials[(size_t)b * NV + k]);
  }
  block_sum<NV>(acc);
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = acc[k];
    *counter = 0u;
  }
  return tid == 0;
}

// Record a failure status; the first one wins (an invalid density makes the
// diagonal and then the recurrences NaN too, and the user needs the cause).
__device__ __forceinline__ void cg_fail(CgScalars *S, int code) {
  atomicCAS(reinterpret_cast<int *>(&S->status), 0, code);
}

__device__ __forceinline__ bool cg_stopped(const CgScalars *S) {
  return *((volatile const int32_t *)&S->done) | *((volatile const int32_t *)&S->done_next);
}

// Called by the first kernel of every iteration (the operator apply).  When
// the previous iteration converged (done_next), promote it to `done` so that
// the x/p update kernel of this overshoot iteration is skipped as well.
__device__ __forceinline__ bool cg_stop_at_apply(CgScalars *S) {
  if (!cg_stopped(S)) return false;
  if (blockIdx.x == 0 && threadIdx.x == 0) S->done = 1;
  return true;
}

}  // namespace tomesh
