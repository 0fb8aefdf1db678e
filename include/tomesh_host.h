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

/* Dynamic AMR mesh update (§4; readings R21-R23).
 * tomesh_host_adapt takes per-element marks of the mesh h (+1 refine, -1
 * derefine, 0 keep; from to_amr_mark) and the element densities x, applies
 *   sweep 1: a derefinement survives only if all 2^dim siblings are leaves
 *            marked -1 ("unmark ... if they have a sibling that is not marked");
 *   sweep 2: a sibling group survives only if no leaf two or more levels finer
 *            than the would-be parent touches it across a face/edge (3D) or an
 *            edge (2D) in the 2:1 closure (C10) of this pass's refinements
 *            ("level two or higher edge incompatibility");
 * and returns the new pre-balance leaf set (ascending Morton order):
 * refined leaves become their children with the parent's density; a
 * derefined group becomes the parent with the children's mean density
 * (summed in corner order).  Build the new mesh from it with
 * tomesh_host_build (same boundary and load boxes), then
 * tomesh_host_transfer gives every new (balanced) element the density of
 * the pre-balance leaf containing it.  Marks beyond the level range
 * (refine at max_level, derefine at level 0) are rejected (TO_EINVAL). */
typedef struct tomesh_adapt tomesh_adapt;
typedef struct {
  int64_t n_leaf;
  const int8_t  *leaf_level;   /* [n_leaf]                                         */
  const int32_t *leaf_anchor;  /* [n_leaf][dim]                                    */
  const double  *leaf_x;       /* [n_leaf] transferred densities                   */
  const int8_t  *marks;        /* [n_elem of h] marks after the two sweeps         */
  int64_t n_refined, n_groups, n_unmarked_sibling, n_unmarked_incompat;
} tomesh_adapt_result;
int  tomesh_host_adapt(const tomesh_host *h, const int8_t *marks, const double *x, tomesh_adapt **out);
int  tomesh_adapt_get(const tomesh_adapt *a, tomesh_adapt_result *out);
int  tomesh_host_transfer(const tomesh_host *h_new, const tomesh_adapt *a, double *x_out);
void tomesh_adapt_free(tomesh_adapt *a);

#ifdef __cplusplus
}
#endif
#endif /* TOMESH_HOST_H */
