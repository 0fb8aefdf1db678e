/*
 * tomesh_host.h — C ABI of the host-side mesh preparation (C++17, CPU).
 *
 * The paper keeps mesh adaptation, compatibility enforcement and DOF
 * numbering in libMesh on the host (PAPER.md:564-571 §6, :640-663); so does
 * this build.  tomesh_host_build turns a pre-balance leaf set and geometric
 * boundary/load predicates into the flat arrays tomesh_upload consumes,
 * following the canonical contract of SURVEY.md §8(b):
 *   C10 2:1 balance across edges (2D) / faces and edges (3D) — the paper's
 *       "level-one mesh incompatibility" only;
 *   C2  elements in ascending Morton order of their anchors;
 *   C3  nodes = all leaf corners (hanging included), ascending Morton order;
 *   C4  elem_node corner order c = cx + 2cy + 4cz;
 *   C6  hanging nodes (a node inside an edge, or a 3D face, of some leaf):
 *       parents = that edge's 2 endpoints (w = 1/2) / face's 4 corners
 *       (w = 1/4), the linear interpolation of PAPER.md:656-663 (Eq. 6);
 *   C7  fixed DOFs: nodes inside a fixed box, hanging nodes excluded;
 *   C8  consistent nodal loads (point / line / face);
 *   C9  filter neighbour lists |c_d - c_e| < rmin (Eq. 4).
 * All outputs are owned by the returned handle (host memory) and stay valid
 * until tomesh_host_free.  No CUDA is used.
 */
#ifndef TOMESH_HOST_H
#define TOMESH_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tomesh_host tomesh_host;

enum { TOH_LOAD_POINT = 0, TOH_LOAD_LINE = 1, TOH_LOAD_FACE = 2 };

typedef struct {
  int32_t dim;                /* 2 or 3                                           */
  int32_t max_level;          /* L: finest lattice level, 0 <= L <= 16            */
  int32_t base[3];            /* level-0 cells per axis                           */
  double  h0;                 /* level-0 cell edge                                */
  int64_t n_leaf;
  const int8_t  *leaf_level;  /* [n_leaf] pre-balance leaves tiling the box       */
  const int32_t *leaf_anchor; /* [n_leaf][dim] lattice anchors                    */
  int32_t n_fixed_box;
  const int32_t *fixed_box;   /* [n_fixed_box][2*dim]: lo[0..dim), hi[0..dim),
                                 inclusive lattice coordinates                    */
  const int32_t *fixed_mask;  /* [n_fixed_box] bit c = component c is fixed       */
  int32_t n_load;
  const int32_t *load_kind;   /* [n_load] TOH_LOAD_*                              */
  const int32_t *load_box;    /* [n_load][2*dim] region (a point, a boundary
                                 segment or a boundary rectangle of the domain)   */
  const double  *load_vec;    /* [n_load][dim] force (point), force per unit
                                 length (line) or per unit area (face)           */
  double rmin;                /* physical filter radius; <= 0: no lists           */
} tomesh_host_spec;

typedef struct {
  int32_t dim, max_level;
  double  h0;
  int64_t n_elem, n_node, n_hang, n_hang_nnz, n_fixed, filt_nnz;
  const int32_t *elem_node;   /* [n_elem][2^dim]                                  */
  const int32_t *elem_anchor; /* [n_elem][dim]                                    */
  const int8_t  *elem_level;  /* [n_elem]                                         */
  const int32_t *node_coord;  /* [n_node][dim] lattice coordinates                */
  const int32_t *hang_node;   /* [n_hang]                                         */
  const int32_t *hang_ptr;    /* [n_hang+1]                                       */
  const int32_t *hang_parent; /* [n_hang_nnz]                                     */
  const double  *hang_weight; /* [n_hang_nnz]                                     */
  const int64_t *fixed_dof;   /* [n_fixed]                                        */
  const double  *load;        /* [dim*n_node]                                     */
  const int64_t *filt_ptr;    /* [n_elem+1] (NULL if rmin <= 0)                   */
  const int32_t *filt_idx;    /* [filt_nnz]                                       */
} tomesh_host_arrays;

/* Returns 0 on success, TO_EINVAL (-1) for a bad spec (leaves not tiling the
 * box, anchors off the lattice, a point load not on a node ...), with the
 * message in to_last_error(). */
int  tomesh_host_build(const tomesh_host_spec *spec, tomesh_host **out);
int  tomesh_host_get(const tomesh_host *h, tomesh_host_arrays *out);
/* Recompute the filter neighbour lists for another radius (replaces them). */
int  tomesh_host_filter(tomesh_host *h, double rmin);
void tomesh_host_free(tomesh_host *h);

#ifdef __cplusplus
}
#endif
#endif /* TOMESH_HOST_H */
