// Data types shared by the kernels and the host side of libtomesh (the
// handle in tomesh_impl.cuh holds them), kept apart from the kernel
// definitions so that each translation unit includes only the kernels it
// launches.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "device_common.cuh"

namespace tomesh {

// General (AMR) path: the mesh arrays a kernel reads (kernels_general.cuh).
struct MeshView {
  int64_t n_el, n_node;
  const int32_t *elem_node;     // [n_el][NC]
  const int8_t *elem_level;
  const int32_t *elem_anchor;   // [n_el][DIM]
  const int32_t *node_hang;     // [n_node] index into hang rows or -1
  const int32_t *hang_ptr, *hang_parent;
  const double *hang_weight;
  const int32_t *child_ptr, *child_hang;  // transpose: parent node -> hanging children
  const double *child_weight;
  const uint8_t *free_dof;      // [n_dof] 1 = neither hanging nor fixed
  int L;
  double hL;
};

// General path, single-kernel iteration (kernels_genfused.cuh): the
// owner-computes decomposition built at upload (tomesh.cu build_gen_blocks).
// CTA b owns the canonical nodes [node0, node0 + n_own).  Its local node
// slots are [0, n_own) owned, then n_halo halo nodes, then n_virt virtual
// slots (hanging corner nodes).  Everything static about the block is one
// contiguous 16-byte-aligned record (one bulk copy into shared memory), with
// sections, each padded to 16 bytes, in this order:
//   halo    int32  [n_halo]       global node ids, ascending
//   virt    ushort4[n_virt]       the parents' local slots of a hanging corner
//                                 node (.z = 0xffff: two parents), ascending
//                                 hanging node id
//   corner  uint16 [n_el][2^dim]  local slot of every corner of the block's
//                                 elements (ascending element id)
//   iptr    uint16 [nch][n_own+1] chunk-major CSR (nch = ceil(n_el / ch), ch =
//                                 the reading kernel's elements per chunk):
//                                 owned node o's incidences with the elements
//                                 of chunk c are inc[iptr[c][o] .. iptr[c][o+1])
//   inc     uint16 [n_inc]        double offset of the corner's result in the
//                                 chunk buffer ((local element - c ch) * YS +
//                                 corner * dim, YS = 2^dim dim + 1) | weight
//                                 code << 14 (0: 1, 1: 1/2, 2: 1/4); per node
//                                 and chunk in ascending element order
// s_e of the block's elements: s_loc[el_off .. el_off + n_el) (el_off even).
struct GfMeta {
  int32_t node0, n_own, n_halo, n_virt, n_el, n_inc, el_off, rec_off16;
};
struct GenBlocks {
  int n_blk, max_loc, max_own, max_rec16, max_el;   // shared-memory sizing: maxima over the blocks
  const GfMeta *meta;
  const uint4 *rec;
  int pf;   // k_gen_fused: block b prefetches block b + pf's static data and owned vectors into L2 (0: off)
};

// Send lists of the cluster solver's halo exchange (kernels_gencluster.cuh),
// built at upload: entry = src owned node (12 bits) | index in the
// destination's halo list (15 bits) << 12 | destination rank (4 bits) << 27.
struct GcSend {
  const uint32_t *ent;
  const int32_t *off;   // [n_blk + 1]
  int max_halo, max_send;
};

__host__ __device__ constexpr int gf_pad16(int bytes) { return (bytes + 15) & ~15; }

// Structured path (kernels_struct3d.cuh): the uniform H8 box and its CTA grid.
struct GridView {
  int EX, EY, EZ;        // elements per axis
  int NX, NY, NZ;        // nodes per axis
  int NXP;               // nodes per internal row (NX rounded up to even)
  int RS;                // doubles per node row in the internal layout (3 NXP)
  int ntx, nty, nzs;     // CTA tiles in x, y and z segments
  int zlen;              // node planes per z segment
  const int4 *plan;      // nullptr, or per CTA {x tile, y tile, k_lo, k_hi} (host-planned waves)
};

constexpr int kS3PadFront = 16;    // doubles (or nodes) before an internal vector
constexpr int kS3PadBack = 128;    // doubles (or nodes) after it
constexpr int kS3RowD = 100;       // doubles staged per node row: 33 nodes + alignment (800 B)
constexpr int kS3RowN = 34;        // node values staged per row: 33 + alignment (272 B)
constexpr int kS3NBuf = 2;         // staging depth: plane P is issued ~1.5 layers before it is formed

// z-slab sharding of the structured path (kernels_shard.cuh).
// Rank r owns the node planes [own_lo, own_hi) of its local box; the box adds
// up to two ghost node planes (and element layers) on each side.  Every
// collective is a push into every rank's slots plus a flag store
// (release, system scope) and a wait on the local flags (acquire): deterministic
// (the gather sums the ranks in rank order on every rank).
constexpr int kShardMax = 16;          // ranks per group
constexpr int kShardVals = 8;          // doubles per slot
constexpr int kShardBanks = 4;         // slot / flag banks: K1 parity 0/1, tail collectives 2/3
constexpr unsigned long long kShardTail = 1ull << 62;   // sequence tag of the tail collectives
struct ShardComm {
  int rank, nranks;
  int own_lo, own_hi;                  // owned local node planes
  // neighbours' vectors as seen from this device, pre-offset so that this
  // rank's internal index i addresses the same global node there (nullptr at
  // the ends of the stack); [w] = ping-pong buffer w
  double *lo_r[2], *lo_p[2], *lo_q[2], *lo_x;
  double *hi_r[2], *hi_p[2], *hi_q[2], *hi_x;
  double *slots[kShardMax];            // rank r's slots [kShardBanks][kShardMax][kShardVals]
  unsigned long long *flags[kShardMax];   // rank r's flags [kShardBanks][kShardMax]
  double *my_slots;
  unsigned long long *my_flags;
};

// Morton node-range sharding of the general path (kernels_gshard.cuh): the
// collectives' ShardComm plus the ghost-store list and the peers' vectors.
struct GShardComm {
  ShardComm C;                                     // rank, nranks, slots / flags of every rank
  int64_t n_send;
  const int32_t *send_rank, *send_local, *send_remote;
  double *peer_r[2][kShardMax], *peer_p[2][kShardMax], *peer_q[2][kShardMax];
  double *peer_x[kShardMax], *peer_d[kShardMax];
};

// One offset of the uniform-box filter stencil (k_filter_s3).
struct S3FilterOffset {
  int di, dj, dk;
  double w;          // H * V
};

// OC update (kernels_oc.cuh): results and the grid-reduction words.
struct OcState {
  double lam, volume_abs, change;
  int32_t steps, state;   // state: 0 active, 1 inactive, 2 infeasible, -5 NaN
  int32_t passes;         // passes over the elements (grid-wide reductions)
  // grid-wide reduction words; zeroed by the host before every launch
  uint32_t arrive, flag;
  unsigned long long change_bits;   // max |x_new - x| as the bits of a non-negative double
  double tot[2][8];
};

// MINRES (kernels_minres.cuh): device scalars.
struct MrScalars {
  double gamma, gamma_old, delta, c, c_old, s, s_old, eta, eta0, thresh;
  double a1, a2, a3, cn, eta_prev;      // w / x~ update coefficients of the last completed step
  double bnorm2, tmp;
  int32_t iter, wx_done, max_iter, done, status, pad;
  uint32_t counter[6];
};
enum { MRC_GAMMA = 0, MRC_DELTA = 1, MRC_WX = 2, MRC_MISC = 3 };

// IC(0) of the rescaled matrix (kernels_ic0.cuh).
struct Ic0View {
  int64_t n, nnz;
  const int64_t *ptr;      // [n+1] lower CSR, columns ascending, diagonal last
  const int32_t *col;      // [nnz]
  const int32_t *row;      // [nnz]
  const int64_t *cptr;     // [nnz+1] contributions of each nonzero
  const uint64_t *contrib; // element << 16 | (a * ND + b) << 3 | log2(1/w)
};

}  // namespace tomesh
