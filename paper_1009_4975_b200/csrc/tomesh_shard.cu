// libtomesh — z-slab sharding of the structured path: one
// handle per slab (per GPU), a per-iteration exchange fused into K1 plus
// device-side scalar all-reduces (kernels_shard.cuh), and the group solve
// tosolve_cg_group that drives one or several handles in lockstep.
//
// Slab layout (the caller's partition, paper_1009_4975_b200/shard.py): rank r
// owns the global node planes [a_r, b_r); its local box holds the element
// layers [a_r - 2, b_r + 1) and node planes [a_r - 2, b_r + 2), clipped to the
// mesh.  With these two ghost layers the Jacobi diagonal of the ghost planes
// a_r - 1 and b_r (which K1 stages) is complete locally, and after the solve
// the filter of every owned element finds its neighbours (reach 1 layer,
// rmin <= 2 element edges) in the local box.
#include "tomesh_impl.cuh"
#include "kernels_cg.cuh"
#include "kernels_shard.cuh"
#include "kernels_struct3d.cuh"
#include "kernels_genfused.cuh"
#include "kernels_gshard.cuh"

using namespace tomesh;

namespace {

__global__ void k_own_dof(int64_t n_node, const int32_t *__restrict__ perm_node, int64_t plane_d, int own_lo,
                          int own_hi, uint8_t *__restrict__ own) {
  GRID_STRIDE(n, n_node) {
    const int64_t kp = (int64_t)perm_node[n] / plane_d;
    const uint8_t o = (kp >= own_lo && kp < own_hi) ? 1 : 0;
    own[3 * n] = own[3 * n + 1] = own[3 * n + 2] = o;
  }
}

__global__ void k_dot_masked(int64_t n, const double *__restrict__ a, const double *__restrict__ b,
                             const uint8_t *__restrict__ mask, double *partials, CgScalars *S, int slot) {
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) {
    if (mask[i]) acc[0] = fma(a[i], b[i], acc[0]);
  }
  if (grid_sum<1>(acc, partials, &S->counter[CNT_MISC2])) S->tmp[slot] = acc[0];
}

int64_t plane_doubles(const to_mesh *m) { return (int64_t)m->G.NY * m->G.RS; }

int ensure_shard_mem(to_mesh *m, cudaStream_t st) {
  if (m->shard_slots) return 0;
  RC(m->alloc(&m->shard_slots, (size_t)kShardBanks * kShardMax * kShardVals));
  RC(m->alloc(&m->shard_flags, (size_t)kShardBanks * kShardMax));
  CK(cudaMemsetAsync(m->shard_slots, 0, sizeof(double) * kShardBanks * kShardMax * kShardVals, st));
  CK(cudaMemsetAsync(m->shard_flags, 0, sizeof(unsigned long long) * kShardBanks * kShardMax, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

// Iteration k of a sharded solve: K1 (SHARD) then the step.
int op_cg_s3_shard(to_mesh *m, int k, double rtol, cudaStream_t st) {
  const int o = (k + 1) & 1, w = k & 1;
  S3Maps M;
  M.a = m->tm_rb[o];
  M.q = m->tm_qb[o];
  M.p = m->tm_pb[o];
  M.d = m->tm_dn;
  GridView G = m->G;
  G.plan = m->shard_plan;
  dim3 block(32, kS3TYW);
  RC(launch_pdl(k_apply_s3<kS3TYW, S3_CG, true>, dim3(m->shard_ncta), block, sizeof(S3Smem<kS3TYW>), st, G,
                (const double *)m->s, M, m->rb[w], m->pb[w], m->x, m->qb[w], m->KS, m->S, m->partials, k, rtol,
                m->hist, m->SC, m->shard_seq));
  m->shard_seq++;   // K1 k pushes this sequence; K1 k+1 gathers it and forms the step of iteration k
  m->last_launches++;
  return 0;
}

// The step of the last launched iteration k (no K1 follows to form it).
int op_step_shard(to_mesh *m, int k, double rtol, cudaStream_t st) {
  RC(launch_pdl(k_shard_step, dim3(1), dim3(32), 0, st, m->SC, m->shard_seq - 1, m->S, k, rtol, m->hist));
  m->last_launches++;
  return 0;
}

int check_group(to_mesh *const *ms, int n) {
  if (!ms || n <= 0) { set_error("empty group"); return TO_EINVAL; }
  for (int i = 0; i < n; ++i) {
    if (!ms[i]) { set_error("NULL handle in group"); return TO_EINVAL; }
    if (!ms[i]->sharded) { set_error("handle %d of the group is not attached (to_shard_attach)", i); return TO_EINVAL; }
    if (ms[i]->shard_seq != ms[0]->shard_seq || ms[i]->tail_seq != ms[0]->tail_seq) {
      set_error("group handles out of step (sequence numbers differ)");
      return TO_EINVAL;
    }
  }
  return 0;
}

}  // namespace

extern "C" int to_shard_buffers(to_mesh *m, to_shard_bufs *out, void *cuda_stream) {
  clear_error();
  if (!m || !out) { set_error("NULL argument"); return TO_EINVAL; }
  if (!m->structured && !m->gen_fused) { set_error("sharding needs the structured or the general single-kernel path"); return TO_EINVAL; }
  CK(cudaSetDevice(m->device));
  RC(ensure_shard_mem(m, (cudaStream_t)cuda_stream));
  std::memset(out, 0, sizeof(*out));
  out->dinv = m->dinv;
  for (int w = 0; w < 2; ++w) {
    out->rb[w] = m->rb[w];
    out->pb[w] = m->pb[w];
    out->qb[w] = m->qb[w];
  }
  out->x = m->x;
  out->slots = m->shard_slots;
  out->flags = m->shard_flags;
  if (m->structured) {
    out->nx = m->G.NX;
    out->ny = m->G.NY;
    out->nz = m->G.NZ;
    out->plane_doubles = plane_doubles(m);
  }
  return 0;
}

extern "C" int to_shard_attach(to_mesh *m, int32_t rank, int32_t nranks, const int32_t *gz_lo, int32_t own_lo,
                               int32_t own_hi, const to_shard_bufs *peers, void *cuda_stream) {
  clear_error();
  if (!m || !gz_lo || !peers) { set_error("NULL argument"); return TO_EINVAL; }
  if (!m->structured) { set_error("sharding needs the structured path (uniform H8 box)"); return TO_EINVAL; }
  if (nranks < 1 || nranks > kShardMax || rank < 0 || rank >= nranks) {
    set_error("rank %d of %d outside [0, %d)", rank, nranks, kShardMax);
    return TO_EINVAL;
  }
  const GridView &G = m->G;
  const int64_t pd = plane_doubles(m);
  if (own_hi - own_lo < 2 || own_lo < 0 || own_hi > G.NZ) { set_error("owned planes [%d, %d) invalid (>= 2 planes inside the box)", own_lo, own_hi); return TO_EINVAL; }
  if ((rank > 0) != (own_lo >= 1) || (rank > 0 && own_lo < 2)) { set_error("rank %d needs two ghost planes below its owned range", rank); return TO_EINVAL; }
  if ((rank < nranks - 1) && own_hi > G.NZ - 2) { set_error("rank %d needs two ghost planes above its owned range", rank); return TO_EINVAL; }
  if (rank == 0 && own_lo != 0) { set_error("rank 0 must own its first plane"); return TO_EINVAL; }
  if (rank == nranks - 1 && own_hi != G.NZ) { set_error("the last rank must own its last plane"); return TO_EINVAL; }
  for (int r = 0; r < nranks; ++r) {
    const to_shard_bufs &p = peers[r];
    const bool nb = r == rank - 1 || r == rank + 1;   // neighbours: their vectors are written too
    if (!p.slots || !p.flags || p.nx != G.NX || p.ny != G.NY || p.plane_doubles != pd ||
        (nb && (!p.x || !p.rb[0] || !p.rb[1] || !p.pb[0] || !p.pb[1] || !p.qb[0] || !p.qb[1]))) {
      set_error("peer %d: missing buffers or a different x-y box", r);
      return TO_EINVAL;
    }
  }
  CK(cudaSetDevice(m->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  RC(ensure_shard_mem(m, st));
  if (peers[rank].x != m->x || peers[rank].slots != m->shard_slots) { set_error("peers[rank] is not this handle"); return TO_EINVAL; }
  ShardComm C{};
  C.rank = rank;
  C.nranks = nranks;
  C.own_lo = own_lo;
  C.own_hi = own_hi;
  // neighbour r' sees this rank's local plane kp at its own plane kp + gz_lo[rank] - gz_lo[r']
  auto shifted = [&](double *base, int rp) { return base + (int64_t)(gz_lo[rank] - gz_lo[rp]) * pd; };
  if (rank > 0) {
    const to_shard_bufs &p = peers[rank - 1];
    const int g0 = gz_lo[rank] + own_lo;   // pushed planes g0, g0 + 1 must lie in the lower box's ghost region
    if (g0 + 1 - gz_lo[rank - 1] >= p.nz) { set_error("lower neighbour box too small"); return TO_EINVAL; }
    for (int w = 0; w < 2; ++w) {
      C.lo_r[w] = shifted(p.rb[w], rank - 1);
      C.lo_p[w] = shifted(p.pb[w], rank - 1);
      C.lo_q[w] = shifted(p.qb[w], rank - 1);
    }
    C.lo_x = shifted(p.x, rank - 1);
  }
  if (rank < nranks - 1) {
    const to_shard_bufs &p = peers[rank + 1];
    const int g1 = gz_lo[rank] + own_hi - 1;
    if (g1 - gz_lo[rank + 1] < 0) { set_error("upper neighbour box does not reach below its owned range"); return TO_EINVAL; }
    for (int w = 0; w < 2; ++w) {
      C.hi_r[w] = shifted(p.rb[w], rank + 1);
      C.hi_p[w] = shifted(p.pb[w], rank + 1);
      C.hi_q[w] = shifted(p.qb[w], rank + 1);
    }
    C.hi_x = shifted(p.x, rank + 1);
  }
  for (int r = 0; r < nranks; ++r) {
    C.slots[r] = peers[r].slots;
    C.flags[r] = peers[r].flags;
  }
  // a group spread over several GPUs of one process: this device stores into
  // the others' memory, so enable peer access to every device a peer buffer
  // lives on (buffers mapped by CUDA IPC already belong to this context)
  for (int r = 0; r < nranks; ++r) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, peers[r].slots) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (at.type == cudaMemoryTypeDevice && at.device != m->device) {
      int can = 0;
      CK(cudaDeviceCanAccessPeer(&can, m->device, at.device));
      if (!can) { set_error("device %d cannot access peer device %d", m->device, at.device); return TO_ECUDA; }
      const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
      cudaGetLastError();
    }
  }
  C.my_slots = m->shard_slots;
  C.my_flags = m->shard_flags;
  if (m->shard_plan) {   // re-attach: the previous plan is no longer referenced
    CK(cudaStreamSynchronize(st));
    m->release(m->shard_plan);
    m->shard_plan = nullptr;
  }
  RC(plan_s3(m, st, own_lo, own_hi, true, &m->shard_plan, &m->shard_ncta));
  CK(cudaFuncSetAttribute(k_apply_s3<kS3TYW, S3_CG, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)sizeof(S3Smem<kS3TYW>)));
  if (!m->own_dof) RC(m->alloc(&m->own_dof, (size_t)m->n_dof));
  k_own_dof<<<grid_for(m->n_node), kBlock, 0, st>>>(m->n_node, m->perm_node, pd, own_lo, own_hi, m->own_dof);
  RC(check_launch());
  // a (re)attached group restarts its sequence numbers at 1: clear this
  // handle's flags so that no flag of an earlier attachment can match
  // (every rank attaches before any rank solves; ShardRank barriers on it)
  CK(cudaMemsetAsync(m->shard_flags, 0, sizeof(unsigned long long) * kShardBanks * kShardMax, st));
  CK(cudaStreamSynchronize(st));
  m->SC = C;
  m->sharded = true;
  m->shard_seq = 1;
  m->tail_seq = 1;
  return 0;
}

// Compliance partial of a sharded handle: sum of f.u over the owned DOFs.
int shard_compliance_partial(to_mesh *m, const double *u_dev, double *out, cudaStream_t st) {
  k_dot_masked<<<grid_for(m->n_dof), kBlock, 0, st>>>(m->n_dof, m->load, u_dev, m->own_dof, m->partials, m->S, 1);
  m->launches_total++;
  RC(check_launch());
  CK(cudaMemcpyAsync(m->S_host, m->S, sizeof(CgScalars), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *out = m->S_host->tmp[1];
  return 0;
}

int gshard_solve_group(to_mesh *const *ms, int32_t n, double penal, const double *const *x_dev,
                       double *const *u_dev, double rtol, int32_t max_iter, uint32_t flags, to_cg_stats *st_out,
                       void *const *streams);

extern "C" int tosolve_cg_group(to_mesh *const *ms, int32_t n, double penal, const double *const *x_dev,
                                double *const *u_dev, double rtol, int32_t max_iter, uint32_t flags,
                                to_cg_stats *st_out, void *const *streams) {
  clear_error();
  RC(check_group(ms, n));
  if (ms[0]->gshard) return gshard_solve_group(ms, n, penal, x_dev, u_dev, rtol, max_iter, flags, st_out, streams);
  if (!x_dev || !u_dev || !streams) { set_error("NULL argument"); return TO_EINVAL; }
  for (int i = 0; i < n; ++i)
    if (!x_dev[i] || !u_dev[i]) { set_error("NULL density or output of handle %d", i); return TO_EINVAL; }
  if (!(penal > 0.0)) { set_error("penal must be > 0"); return TO_EINVAL; }
  if (max_iter < 0) { set_error("max_iter < 0"); return TO_EINVAL; }
  if (flags & (TO_WARM | TO_PROFILE)) { set_error("TO_WARM / TO_PROFILE are not supported on sharded handles"); return TO_EINVAL; }
  const bool fixed = (flags & TO_FIXED_ITERS) != 0;
  const bool hist = (flags & TO_HISTORY) != 0;
  auto S_ = [&](int i) { return (cudaStream_t)streams[i]; };
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    m->last_launches = 0;
    if (hist && max_iter > m->hist_cap) {
      RC(m->alloc(&m->hist, (size_t)max_iter));
      m->hist_cap = max_iter;
    }
    CK(cudaEventRecord(m->ev0, S_(i)));
    RC(reset_scalars(m, max_iter, fixed, hist, S_(i)));
    RC(op_scale_and_diag(m, penal, x_dev[i], nullptr, S_(i)));
    RC(op_rhs(m, m->rb[1], S_(i)));   // r0 = b (iteration 0 reads rb[1]), ghost planes included
    CK(cudaMemsetAsync(m->x, 0, sizeof(double) * m->n_int, S_(i)));
    const int64_t pd = plane_doubles(m), n_own = (int64_t)(m->SC.own_hi - m->SC.own_lo) * pd;
    k_shard_norm2_push<<<grid_for(n_own), kBlock, 0, S_(i)>>>(n_own, m->rb[1] + m->SC.own_lo * pd, m->partials,
                                                               m->S, m->SC, kShardTail | m->tail_seq);
    m->last_launches++;
    RC(check_launch());
  }
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    k_shard_set_bnorm<<<1, 32, 0, S_(i)>>>(m->SC, kShardTail | m->tail_seq, m->S);
    m->tail_seq++;
    m->last_launches++;
    RC(check_launch());
  }
  const bool loop_prof = (flags & TO_PROFILE_LOOP) != 0;
  if (loop_prof)
    for (int i = 0; i < n; ++i) {
      CK(cudaSetDevice(ms[i]->device));
      for (auto &e : ms[i]->loop_ev)
        if (!e) CK(cudaEventCreate(&e));
      CK(cudaEventRecord(ms[i]->loop_ev[0], S_(i)));
    }
  int launched = 0, chunk = fixed ? std::max(1, max_iter) : 16;
  bool stop = false;
  while (!stop && launched < max_iter) {
    const int cnt = std::min(chunk, max_iter - launched);
    for (int k = 0; k < cnt; ++k)
      for (int i = 0; i < n; ++i) {
        CK(cudaSetDevice(ms[i]->device));
        RC(op_cg_s3_shard(ms[i], launched + k, rtol, S_(i)));
      }
    RC(check_launch());
    launched += cnt;
    if (!fixed) {
      int done = -1;
      for (int i = 0; i < n; ++i) {
        CK(cudaSetDevice(ms[i]->device));
        RC(read_scalars(ms[i], S_(i)));
        const int d = (ms[i]->S_host->done || ms[i]->S_host->done_next) ? 1 : 0;
        if (done >= 0 && d != done) { set_error("sharded solve: ranks disagree on the stop test"); return TO_ECUDA; }
        done = d;
      }
      stop = done == 1;
      chunk = std::min(chunk * 2, 256);
    }
  }
  if (launched > 0)
    for (int i = 0; i < n; ++i) {
      CK(cudaSetDevice(ms[i]->device));
      RC(op_step_shard(ms[i], launched - 1, rtol, S_(i)));
    }
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    if (loop_prof) CK(cudaEventRecord(m->loop_ev[1], S_(i)));
    const int o = (max_iter + 1) & 1;
    const int64_t pd = plane_doubles(m), off = m->SC.own_lo * pd, nodes_off = off / 3;
    const int n_own = (int)((m->SC.own_hi - m->SC.own_lo) * pd);
    k_final_s3<true><<<kNumSMs * 4, 512, 0, S_(i)>>>(n_own, m->rb[o] + off, m->qb[o] + off, m->pb[o] + off,
                                                     m->dn + nodes_off, m->x + off, m->partials, m->S, max_iter, rtol,
                                                     m->hist, m->SC, kShardTail | m->tail_seq, m->rb[1] + off,
                                                     m->pb[1] + off);
    m->last_launches++;
    RC(check_launch());
  }
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    k_shard_final<<<1, 32, 0, S_(i)>>>(m->SC, kShardTail | m->tail_seq, m->S, max_iter, rtol, m->hist);
    m->tail_seq++;
    m->last_launches++;
    RC(check_launch());
  }
  // the neighbours' ghost planes of x (sensitivities and filter of their owned elements)
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    const int64_t pd = plane_doubles(m);
    k_shard_push_x<<<grid_for(3 * pd), kBlock, 0, S_(i)>>>(m->x, pd, m->partials, m->S, m->SC,
                                                           kShardTail | m->tail_seq);
    m->last_launches++;
    RC(check_launch());
  }
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    k_shard_wait<<<1, 32, 0, S_(i)>>>(m->SC, kShardTail | m->tail_seq, m->S);
    m->tail_seq++;
    m->last_launches++;
    RC(check_launch());
    RC(op_recover_out(m, m->x, u_dev[i], S_(i)));
    CK(cudaEventRecord(m->ev1, S_(i)));
  }
  int rc_all = 0;
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    CK(cudaStreamSynchronize(S_(i)));
    RC(read_scalars(m, S_(i)));
    const CgScalars res = *m->S_host;
    float ms_ = 0.f;
    CK(cudaEventElapsedTime(&ms_, m->ev0, m->ev1));
    if (loop_prof) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, m->loop_ev[0], m->loop_ev[1]));
      for (int j = 0; j < 4; ++j) m->prof_ms[j] = 0.0;
      m->prof_ms[4] = std::min(launched, res.iter);
      m->prof_ms[5] = t;
    }
    m->hist_len = hist ? res.iter : 0;
    m->launches_total += m->last_launches;
    int rc = res.status;
    if (rc == 0 && !fixed && !(res.rr <= res.thresh2) && res.bnorm2 > 0.0) rc = TO_NOT_CONVERGED;
    if (st_out) {
      st_out[i].iters = res.iter;
      st_out[i].status = rc;
      st_out[i].relres = res.bnorm2 > 0.0 ? std::sqrt(res.rr / res.bnorm2) : 0.0;
      st_out[i].relres_true = -1.0;
      st_out[i].ms = ms_;
      st_out[i].bnorm = std::sqrt(res.bnorm2);
    }
    if (rc < 0 && rc_all >= 0) rc_all = rc;
    else if (rc > 0 && rc_all == 0) rc_all = rc;
  }
  if (rc_all < 0) set_error("sharded solve failed (status %d)", rc_all);
  return rc_all;
}

// ---- CUDA IPC of the exchange buffers (one process per GPU) ---------------------------

// The driver may place several small cudaMalloc allocations in one IPC-able
// block, and an IPC handle maps the whole block: the offset is taken from the
// block's base as the driver reports it (cuMemGetAddressRange).
using PFN_memrange = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
static PFN_memrange mem_range_fn() {
  static PFN_memrange fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_memrange)p;
    else
      cudaGetLastError();
  }
  return fn;
}

extern "C" int to_ipc_export(to_mesh *m, const void *dev_ptr, void *handle64, uint64_t *offset) {
  clear_error();
  if (!m || !dev_ptr || !handle64 || !offset) { set_error("NULL argument"); return TO_EINVAL; }
  bool mine = false;
  for (const DevBuf &b : m->bufs)
    if ((const char *)dev_ptr >= (const char *)b.p && (const char *)dev_ptr < (const char *)b.p + b.bytes) mine = true;
  if (!mine) { set_error("pointer is not inside a buffer of this handle"); return TO_EINVAL; }
  CK(cudaSetDevice(m->device));
  auto range = mem_range_fn();
  if (!range) { set_error("cuMemGetAddressRange unavailable"); return TO_ECUDA; }
  CUdeviceptr base = 0;
  size_t bytes = 0;
  if (range(&base, &bytes, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS) { set_error("cuMemGetAddressRange failed"); return TO_ECUDA; }
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, (void *)base));
  std::memcpy(handle64, &h, sizeof(h));
  *offset = (uint64_t)((CUdeviceptr)dev_ptr - base);
  return 0;
}

extern "C" int to_ipc_open(int device, const void *handle64, uint64_t offset, void **dev_ptr) {
  clear_error();
  if (!handle64 || !dev_ptr) { set_error("NULL argument"); return TO_EINVAL; }
  CK(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  void *p = nullptr;
  CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *dev_ptr = (char *)p + offset;
  return 0;
}

extern "C" int to_ipc_close(int device, void *base_ptr) {
  clear_error();
  CK(cudaSetDevice(device));
  CK(cudaIpcCloseMemHandle(base_ptr));
  return 0;
}

// ---- Morton node-range sharding of the general path (kernels_gshard.cuh) --------------

__global__ void k_own_nodes(int64_t n_dof, int64_t owned_dofs, uint8_t *__restrict__ own) {
  GRID_STRIDE(i, n_dof) { own[i] = i < owned_dofs ? 1 : 0; }
}

extern "C" int to_gshard_attach(to_mesh *m, int32_t rank, int32_t nranks, const to_shard_bufs *peers, int64_t n_send,
                                const int32_t *send_rank, const int32_t *send_local, const int32_t *send_remote,
                                void *cuda_stream) {
  clear_error();
  if (!m || !peers || n_send < 0 || (n_send > 0 && (!send_rank || !send_local || !send_remote))) {
    set_error("NULL argument");
    return TO_EINVAL;
  }
  if (!m->gen_fused || m->structured) { set_error("to_gshard_attach needs a general-path handle"); return TO_EINVAL; }
  if (nranks < 1 || nranks > kShardMax || rank < 0 || rank >= nranks) {
    set_error("rank %d of %d outside [0, %d)", rank, nranks, kShardMax);
    return TO_EINVAL;
  }
  for (int64_t i = 0; i < n_send; ++i) {
    const int s = send_rank[i];
    if (s < 0 || s >= nranks || s == rank) { set_error("send entry %lld: bad rank %d", (long long)i, s); return TO_EINVAL; }
    if (send_local[i] < 0 || send_local[i] >= m->n_owned) { set_error("send entry %lld: not an owned node", (long long)i); return TO_EINVAL; }
    if (send_remote[i] < 0) { set_error("send entry %lld: bad remote node", (long long)i); return TO_EINVAL; }
  }
  for (int r = 0; r < nranks; ++r) {
    const to_shard_bufs &p = peers[r];
    if (!p.slots || !p.flags || !p.x || !p.dinv || !p.rb[0] || !p.rb[1] || !p.pb[0] || !p.pb[1] || !p.qb[0] ||
        !p.qb[1] || p.nx != 0) {
      set_error("peer %d: missing buffers or not a general handle", r);
      return TO_EINVAL;
    }
  }
  CK(cudaSetDevice(m->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  RC(ensure_shard_mem(m, st));
  if (peers[rank].x != m->x || peers[rank].slots != m->shard_slots) { set_error("peers[rank] is not this handle"); return TO_EINVAL; }
  GShardComm G{};
  G.C.rank = rank;
  G.C.nranks = nranks;
  for (int r = 0; r < nranks; ++r) {
    G.C.slots[r] = peers[r].slots;
    G.C.flags[r] = peers[r].flags;
    for (int w = 0; w < 2; ++w) {
      G.peer_r[w][r] = peers[r].rb[w];
      G.peer_p[w][r] = peers[r].pb[w];
      G.peer_q[w][r] = peers[r].qb[w];
    }
    G.peer_x[r] = peers[r].x;
    G.peer_d[r] = peers[r].dinv;
  }
  G.C.my_slots = m->shard_slots;
  G.C.my_flags = m->shard_flags;
  // peer access for groups spread over several GPUs of one process
  for (int r = 0; r < nranks; ++r) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, peers[r].slots) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (at.type == cudaMemoryTypeDevice && at.device != m->device) {
      int can = 0;
      CK(cudaDeviceCanAccessPeer(&can, m->device, at.device));
      if (!can) { set_error("device %d cannot access peer device %d", m->device, at.device); return TO_ECUDA; }
      const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
      cudaGetLastError();
    }
  }
  int32_t *d_rank = nullptr, *d_loc = nullptr, *d_rem = nullptr;
  RC(upload_array(m, &d_rank, send_rank, (size_t)n_send, st));
  RC(upload_array(m, &d_loc, send_local, (size_t)n_send, st));
  RC(upload_array(m, &d_rem, send_remote, (size_t)n_send, st));
  G.n_send = n_send;
  G.send_rank = d_rank;
  G.send_local = d_loc;
  G.send_remote = d_rem;
  if (!m->own_dof) RC(m->alloc(&m->own_dof, (size_t)m->n_dof));
  k_own_nodes<<<grid_for(m->n_dof), kBlock, 0, st>>>(m->n_dof, m->n_owned * m->dim, m->own_dof);
  RC(check_launch());
  CK(cudaMemsetAsync(m->shard_flags, 0, sizeof(unsigned long long) * kShardBanks * kShardMax, st));
  CK(cudaStreamSynchronize(st));
  m->GS = G;
  m->gshard = true;
  m->sharded = true;
  m->shard_seq = 1;
  m->tail_seq = 1;
  return 0;
}

template <int MODE>
int launch_gxchg(to_mesh *m, const double *a, const double *b, const double *c, int w, unsigned long long seq,
                 cudaStream_t st) {
  const int g = grid_for(std::max<int64_t>(1, m->GS.n_send));
  if (m->dim == 2)
    k_gshard_xchg<2, MODE><<<g, 256, 0, st>>>(m->GS, a, b, c, w, m->partials, m->GB.n_blk, m->S, seq);
  else
    k_gshard_xchg<3, MODE><<<g, 256, 0, st>>>(m->GS, a, b, c, w, m->partials, m->GB.n_blk, m->S, seq);
  m->last_launches++;
  return check_launch();
}

// The general-path group solve (one handle per rank; n of them in lockstep in
// this process, or 1 per process).  Same device-side protocol as the slabs:
// iteration collectives on the sequence-parity banks, the setup / final / x
// collectives on the tail banks.
int gshard_solve_group(to_mesh *const *ms, int32_t n, double penal, const double *const *x_dev,
                       double *const *u_dev, double rtol, int32_t max_iter, uint32_t flags, to_cg_stats *st_out,
                       void *const *streams) {
  if (!x_dev || !u_dev || !streams) { set_error("NULL argument"); return TO_EINVAL; }
  for (int i = 0; i < n; ++i) {
    if (!ms[i]->gshard) { set_error("handle %d is not an attached general handle", i); return TO_EINVAL; }
    if (!x_dev[i] || !u_dev[i]) { set_error("NULL density or output of handle %d", i); return TO_EINVAL; }
  }
  if (!(penal > 0.0)) { set_error("penal must be > 0"); return TO_EINVAL; }
  if (max_iter < 0) { set_error("max_iter < 0"); return TO_EINVAL; }
  if (flags & (TO_WARM | TO_PROFILE)) { set_error("TO_WARM / TO_PROFILE are not supported on sharded handles"); return TO_EINVAL; }
  const bool fixed = (flags & TO_FIXED_ITERS) != 0;
  const bool hist = (flags & TO_HISTORY) != 0;
  auto S_ = [&](int i) { return (cudaStream_t)streams[i]; };
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    m->last_launches = 0;
    if (hist && max_iter > m->hist_cap) {
      RC(m->alloc(&m->hist, (size_t)max_iter));
      m->hist_cap = max_iter;
    }
    CK(cudaEventRecord(m->ev0, S_(i)));
    RC(reset_scalars(m, max_iter, fixed, hist, S_(i)));
    RC(op_scale_and_diag(m, penal, x_dev[i], nullptr, S_(i)));
    RC(op_rhs(m, m->rb[1], S_(i)));              // r0 = b (owned rows exact; ghosts come from their owners)
    CK(cudaMemsetAsync(m->x, 0, sizeof(double) * m->n_int, S_(i)));
    CK(cudaMemsetAsync(m->qb[1], 0, sizeof(double) * m->n_int, S_(i)));
    CK(cudaMemsetAsync(m->pb[1], 0, sizeof(double) * m->n_int, S_(i)));
    const int64_t n_own = m->n_owned * m->dim;
    k_norm2_b<<<grid_for(n_own), kBlock, 0, S_(i)>>>(n_own, m->rb[1], m->partials, m->S);   // this rank's ||b||^2
    m->last_launches++;
    RC(check_launch());
    RC(launch_gxchg<GX_BARRIER>(m, nullptr, nullptr, nullptr, 0, kShardTail | m->tail_seq, S_(i)));
  }
  for (int i = 0; i < n; ++i) {   // every rank's local Dinv and b are written ...
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    k_shard_wait<<<1, 32, 0, S_(i)>>>(m->GS.C, kShardTail | m->tail_seq, m->S);
    m->tail_seq++;
    m->last_launches++;
    RC(check_launch());
    // ... before the owners store theirs into the ghosts
    RC(launch_gxchg<GX_SETUP>(m, m->dinv, m->rb[1], nullptr, 0, kShardTail | m->tail_seq, S_(i)));
  }
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    k_shard_set_bnorm<<<1, 32, 0, S_(i)>>>(m->GS.C, kShardTail | m->tail_seq, m->S);
    m->tail_seq++;
    m->last_launches++;
    RC(check_launch());
  }
  const bool loop_prof = (flags & TO_PROFILE_LOOP) != 0;
  if (loop_prof)
    for (int i = 0; i < n; ++i) {
      CK(cudaSetDevice(ms[i]->device));
      for (auto &e : ms[i]->loop_ev)
        if (!e) CK(cudaEventCreate(&e));
      CK(cudaEventRecord(ms[i]->loop_ev[0], S_(i)));
    }
  int launched = 0, chunk = fixed ? std::max(1, max_iter) : 16;
  bool stop = false;
  while (!stop && launched < max_iter) {
    const int cnt = std::min(chunk, max_iter - launched);
    for (int k = 0; k < cnt; ++k) {
      const int kk = launched + k, w = kk & 1;
      // every rank's push before any rank's gather in launch order (the
      // handles of one process may share a stream)
      for (int i = 0; i < n; ++i) {
        to_mesh *m = ms[i];
        CK(cudaSetDevice(m->device));
        RC(op_cg_gen(m, kk, rtol, S_(i), false));
        RC(launch_gxchg<GX_ITER>(m, m->rb[w], m->pb[w], m->qb[w], w, m->shard_seq, S_(i)));
      }
      for (int i = 0; i < n; ++i) {
        to_mesh *m = ms[i];
        CK(cudaSetDevice(m->device));
        k_shard_step<<<1, 32, 0, S_(i)>>>(m->GS.C, m->shard_seq, m->S, kk, rtol, m->hist);
        m->shard_seq++;
        m->last_launches++;
      }
    }
    RC(check_launch());
    launched += cnt;
    if (!fixed) {
      int done = -1;
      for (int i = 0; i < n; ++i) {
        CK(cudaSetDevice(ms[i]->device));
        RC(read_scalars(ms[i], S_(i)));
        const int d = (ms[i]->S_host->done || ms[i]->S_host->done_next) ? 1 : 0;
        if (done >= 0 && d != done) { set_error("sharded solve: ranks disagree on the stop test"); return TO_ECUDA; }
        done = d;
      }
      stop = done == 1;
      chunk = std::min(chunk * 2, 256);
    }
  }
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    if (loop_prof) CK(cudaEventRecord(m->loop_ev[1], S_(i)));
    const int o = (max_iter + 1) & 1;
    const int64_t n_own = m->n_owned * m->dim;
    k_final_gen<true><<<grid_for(n_own), kBlock, 0, S_(i)>>>(n_own, m->rb[o], m->qb[o], m->pb[o], m->dinv, m->x,
                                                             m->partials, m->S, max_iter, rtol, m->hist, m->GS.C,
                                                             kShardTail | m->tail_seq);
    m->last_launches++;
    RC(check_launch());
  }
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    k_shard_final<<<1, 32, 0, S_(i)>>>(m->GS.C, kShardTail | m->tail_seq, m->S, max_iter, rtol, m->hist);
    m->tail_seq++;
    m->last_launches++;
    RC(check_launch());
  }
  // the ghosts of x (sensitivities of every local element)
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    RC(launch_gxchg<GX_X>(m, m->x, nullptr, nullptr, 0, kShardTail | m->tail_seq, S_(i)));
  }
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    k_shard_wait<<<1, 32, 0, S_(i)>>>(m->GS.C, kShardTail | m->tail_seq, m->S);
    m->tail_seq++;
    m->last_launches++;
    RC(check_launch());
    RC(op_recover_out(m, m->x, u_dev[i], S_(i)));
    CK(cudaEventRecord(m->ev1, S_(i)));
  }
  int rc_all = 0;
  for (int i = 0; i < n; ++i) {
    to_mesh *m = ms[i];
    CK(cudaSetDevice(m->device));
    CK(cudaStreamSynchronize(S_(i)));
    RC(read_scalars(m, S_(i)));
    const CgScalars res = *m->S_host;
    float ms_ = 0.f;
    CK(cudaEventElapsedTime(&ms_, m->ev0, m->ev1));
    if (loop_prof) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, m->loop_ev[0], m->loop_ev[1]));
      for (int j = 0; j < 4; ++j) m->prof_ms[j] = 0.0;
      m->prof_ms[4] = std::min(launched, res.iter);
      m->prof_ms[5] = t;
    }
    m->hist_len = hist ? res.iter : 0;
    m->launches_total += m->last_launches;
    int rc = res.status;
    if (rc == 0 && !fixed && !(res.rr <= res.thresh2) && res.bnorm2 > 0.0) rc = TO_NOT_CONVERGED;
    if (st_out) {
      st_out[i].iters = res.iter;
      st_out[i].status = rc;
      st_out[i].relres = res.bnorm2 > 0.0 ? std::sqrt(res.rr / res.bnorm2) : 0.0;
      st_out[i].relres_true = -1.0;
      st_out[i].ms = ms_;
      st_out[i].bnorm = std::sqrt(res.bnorm2);
    }
    if (rc < 0 && rc_all >= 0) rc_all = rc;
    else if (rc > 0 && rc_all == 0) rc_all = rc;
  }
  if (rc_all < 0) set_error("sharded solve failed (status %d)", rc_all);
  return rc_all;
}
