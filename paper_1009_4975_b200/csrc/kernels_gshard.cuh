// Morton node-range sharding of the general (AMR) path (DESIGN.md
// §9; host side paper_1009_4975_b200/amr_shard.py).  Rank r's handle holds its
// local mesh: owned nodes [0, n_owned), then ghosts, then non-owned hanging
// nodes.  Its iteration kernel (k_gen_fused) computes the owned nodes from
// the local vectors, ghosts included; k_gshard_xchg then stores the values
// the peers hold as ghosts into their buffers (send entries: local owned node
// -> remote ghost node of rank send_rank) and its last block pushes the
// rank's dots with the slot / flag all-reduce of kernels_shard.cuh;
// k_shard_step on every rank gathers them in rank order and forms the same
// step.  Ordering: every block fences its peer stores at system scope before
// it arrives on the counter, and the last block's push fences again before
// its flag, so a peer that has seen the flag reads complete ghosts.
#pragma once
#include "device_common.cuh"
#include "kernels_cg.cuh"
#include "kernels_shard.cuh"
#include "tomesh_types.cuh"

namespace tomesh {


enum { GX_ITER = 0, GX_SETUP = 1, GX_X = 2, GX_BARRIER = 3 };

// MODE GX_ITER: r_k, p_k, q_k (buffer w) to the peers' buffer w, then the
//   rank's dots (its k_gen_fused blocks' partials summed in block order);
//   skipped entirely once the solve has stopped (the same iteration on every
//   rank; the tail collectives use their own bank).
// MODE GX_SETUP: Dinv and r_0 = b (buffer 1), then {||b||^2 over the owned
//   DOFs (S->bnorm2 of this rank), status != 0}.
// MODE GX_X: the iterate x after the solve, then an empty push (a barrier).
// MODE GX_BARRIER: no stores, an empty push (every rank's local setup -- its
//   Jacobi diagonal and b, ghosts included -- is done before any rank stores
//   the owners' values into those ghosts).
template <int DIM, int MODE>
__global__ void __launch_bounds__(256) k_gshard_xchg(const __grid_constant__ GShardComm G, const double *__restrict__ a,
                                                     const double *__restrict__ b, const double *__restrict__ c,
                                                     int w, const double *__restrict__ blk_partials, int nblk,
                                                     CgScalars *S, unsigned long long seq) {
  if (MODE == GX_ITER && cg_stopped(S)) return;
  if (MODE != GX_BARRIER) GRID_STRIDE(i, G.n_send) {
    const int s = G.send_rank[i];
    const int64_t src = (int64_t)G.send_local[i] * DIM, dst = (int64_t)G.send_remote[i] * DIM;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      if (MODE == GX_ITER) {
        G.peer_r[w][s][dst + d] = __ldcg(a + src + d);
        G.peer_p[w][s][dst + d] = __ldcg(b + src + d);
        G.peer_q[w][s][dst + d] = __ldcg(c + src + d);
      } else if (MODE == GX_SETUP) {
        G.peer_d[s][dst + d] = __ldcg(a + src + d);
        G.peer_r[1][s][dst + d] = __ldcg(b + src + d);
      } else {
        G.peer_x[s][dst + d] = __ldcg(a + src + d);
      }
    }
  }
  __threadfence_system();
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t t = atomicAdd(&S->counter[CNT_XCHG], 1u);
    s_last = t == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (MODE == GX_ITER) {
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int bk = threadIdx.x; bk < nblk; bk += blockDim.x)
#pragma unroll
      for (int k = 0; k < 5; ++k) acc[k] += __ldcg(&blk_partials[(size_t)5 * bk + k]);
    block_sum<5>(acc);
    if (threadIdx.x == 0) {
      S->counter[CNT_XCHG] = 0u;
      shard_push(G.C, seq, acc, 5);
    }
  } else if (threadIdx.x == 0) {
    S->counter[CNT_XCHG] = 0u;
    if (MODE == GX_SETUP) {
      const double v[2] = {__ldcg(&S->bnorm2), __ldcg(&S->status) != 0 ? 1.0 : 0.0};
      shard_push(G.C, seq, v, 2);
    } else {
      shard_push(G.C, seq, nullptr, 0);
    }
  }
}

}  // namespace tomesh
