// z-slab sharding of the structured path ("one exchange step
// per matvec plus scalar reductions").  The exchange is fused into K1 (the
// owners of the first and last owned plane also store r_k, p_k and q_k into
// the neighbour's ghost plane, over NVLink when the neighbour is another GPU),
// and the scalar all-reduce is a push of each rank's partial dots into every
// rank's slot array followed by a flag store; the next K1 waits (one thread
// per CTA) for all flags of that sequence number and sums the slots in rank
// order, so every CTA of every rank forms the same alpha, beta and stop
// decision and an iteration stays one kernel.
//
// Ordering: the writer stores its data, fence.sc.sys, then stores the flag
// with release semantics at system scope; the reader loads the flag with
// acquire semantics at system scope.  A CTA that stored into a neighbour's
// ghost plane fences at system scope before it arrives at the grid reduction,
// so the ghost data is ordered before the flag the last block publishes.
// Slots and flags are double-buffered by sequence parity: a rank can push
// sequence s+1 only after its own gather of s, so the slot of s is not
// overwritten before every rank has read it.  That argument needs every rank
// to push every sequence number of a bank.  K1 stops pushing once the solve
// has stopped (the same iteration on every rank), so the collectives around
// the iteration loop (||b||, the final step, the x ghost planes) use a bank
// pair of their own (sequence numbers tagged kShardTail), which every rank
// pushes on every solve, stopped or not: a rank that runs ahead into them
// can never overwrite a flag a lagging peer's K1 still waits for.
#pragma once
#include "device_common.cuh"
#include "kernels_cg.cuh"
#include "tomesh_types.cuh"

namespace tomesh {

__device__ __forceinline__ void st_release_sys_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Bank of a sequence number: 0/1 = K1 (parity), 2/3 = tail collectives.
__device__ __forceinline__ int shard_bank(unsigned long long seq) {
  return (int)(seq & 1ull) + ((seq & kShardTail) ? 2 : 0);
}

// One thread: push n values of sequence `seq` into every rank's slot.
__device__ __forceinline__ void shard_push(const ShardComm &C, unsigned long long seq, const double *v, int n) {
  const int par = shard_bank(seq);
  for (int r = 0; r < C.nranks; ++r) {
    double *dst = C.slots[r] + ((size_t)par * kShardMax + C.rank) * kShardVals;
    for (int k = 0; k < n; ++k) dst[k] = v[k];
  }
  __threadfence_system();
  for (int r = 0; r < C.nranks; ++r) st_release_sys_u64(C.flags[r] + par * kShardMax + C.rank, seq);
}

// One thread: wait for sequence `seq` from every rank, then sum their n
// values in rank order.  Returns false after ~20 s without all flags (a peer
// that never arrives): the caller records a failure instead of hanging.
__device__ __forceinline__ bool shard_gather(const ShardComm &C, unsigned long long seq, double *out, int n) {
  const int par = shard_bank(seq);
  const unsigned long long t0 = global_ns();
  for (int r = 0; r < C.nranks; ++r) {
    const unsigned long long *f = C.my_flags + par * kShardMax + r;
    while (ld_acquire_sys_u64(f) != seq) {
      if (global_ns() - t0 > 20000000000ull) return false;
      __nanosleep(64);
    }
  }
  for (int k = 0; k < n; ++k) out[k] = 0.0;
  for (int r = 0; r < C.nranks; ++r) {
    const double *src = C.my_slots + ((size_t)par * kShardMax + r) * kShardVals;
    for (int k = 0; k < n; ++k) out[k] += __ldcv(&src[k]);
  }
  return true;
}

// The step of the LAST launched iteration k (every earlier step is formed at
// the start of the next K1): the global dots, then cg_single_step.
static __global__ void k_shard_step(const __grid_constant__ ShardComm C, unsigned long long seq, CgScalars *S, int k,
                             double rtol, double *hist) {
  pdl_wait();
  pdl_release();
  if (threadIdx.x != 0 || cg_stopped(S)) return;
  double d[5];
  if (!shard_gather(C, seq, d, 5)) {
    cg_fail(S, -2);
    S->done = 1;
    return;
  }
  cg_single_step(S, k, d, rtol, hist);
}

// ||b||^2 over the owned range [0, n) of b, pushed as this rank's partial
// together with a failure count (an invalid density found by k_simp_s3 on
// any rank then stops every rank at iteration 0).
static __global__ void k_shard_norm2_push(int64_t n, const double *__restrict__ v, double *partials, CgScalars *S,
                                   const __grid_constant__ ShardComm C, unsigned long long seq) {
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) {
    const double t = v[i];
    acc[0] = fma(t, t, acc[0]);
  }
  if (grid_sum<1>(acc, partials, &S->counter[CNT_MISC])) {
    const double out[2] = {acc[0], __ldcg(&S->status) != 0 ? 1.0 : 0.0};
    shard_push(C, seq, out, 2);
  }
}

static __global__ void k_shard_set_bnorm(const __grid_constant__ ShardComm C, unsigned long long seq, CgScalars *S) {
  if (threadIdx.x != 0) return;
  double b2[2];
  if (!shard_gather(C, seq, b2, 2)) {
    cg_fail(S, -2);
    S->done = 1;
    return;
  }
  S->bnorm2 = b2[0];
  if (b2[1] > 0.0) cg_fail(S, -1);   // a density outside (0, 1] on some rank
}

// After N iterations: the global rho_N, rr_N (k_final_s3<true> pushed them;
// a stopped solve pushed zeros, which are gathered and dropped).
static __global__ void k_shard_final(const __grid_constant__ ShardComm C, unsigned long long seq, CgScalars *S, int n_iter,
                              double rtol, double *hist) {
  if (threadIdx.x != 0) return;
  const bool stopped = cg_stopped(S);
  double d[2];
  if (!shard_gather(C, seq, d, 2)) {
    cg_fail(S, -2);
    S->done = 1;
    return;
  }
  if (!stopped) cg_final_step(S, n_iter, d[0], d[1], rtol, hist);
}

// After the solve: the owned planes the neighbours need for sensitivities and
// the filter (their ghost planes a-1, b, b+1): planes own_lo, own_lo+1 to the
// lower neighbour, plane own_hi-1 to the upper one; then a zero-value
// collective as the barrier (fence + flag in the last block).
static __global__ void k_shard_push_x(const double *__restrict__ x, int64_t plane_d, double *partials, CgScalars *S,
                               const __grid_constant__ ShardComm C, unsigned long long seq) {
  const int64_t lo0 = (int64_t)C.own_lo * plane_d, hi0 = (int64_t)(C.own_hi - 1) * plane_d;
  const int64_t n = 3 * plane_d;
  GRID_STRIDE(t, n) {
    if (t < 2 * plane_d) {
      if (C.lo_x) C.lo_x[lo0 + t] = x[lo0 + t];
    } else if (C.hi_x) {
      const int64_t i = hi0 + (t - 2 * plane_d);
      C.hi_x[i] = x[i];
    }
  }
  __threadfence_system();
  double none[1] = {0.0};
  if (grid_sum<1>(none, partials, &S->counter[CNT_MISC])) shard_push(C, seq, none, 0);
}

static __global__ void k_shard_wait(const __grid_constant__ ShardComm C, unsigned long long seq, CgScalars *S) {
  if (threadIdx.x != 0) return;
  double none[1];
  if (!shard_gather(C, seq, none, 0)) cg_fail(S, -2);
}

}  // namespace tomesh
