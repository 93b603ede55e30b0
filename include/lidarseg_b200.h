/*
 * lidarseg_b200 — C ABI of the B200 (sm_100a) implementation of the lidarseg
 * per-scan hot path: points -> range grid -> 6-neighbour mesh -> normals ->
 * normal-homogeneity segments -> label completion.
 *
 * The reference (arXiv 2005.02704's `lidarseg` package) is pure Python and
 * has no FFI; its operator API for this path is the set of Python functions
 * re-exported at reference pkg/src/lidarseg/__init__.py:21-35.  Each entry
 * point below replaces one of them (cited per function); the Python mirror in
 * paper_2005_02704_b200/ binds them with ctypes.
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer unless noted "host".  The library never
 *    allocates device memory: the caller owns every buffer, including the
 *    scratch `workspace` sized by lseg_workspace_bytes().
 *  - All work is enqueued asynchronously on `stream` (a cudaStream_t, NULL =
 *    legacy default stream).  Nothing synchronises.
 *  - Batched: F frames share one sensor (R rings x S azimuth steps).  Grids are
 *    dense row-major (F, R, S) / (F, R, S'), S' = lseg_kept_count(S, k).
 *    Node-level arrays are padded per frame to cap = R * S' nodes, node ids are
 *    frame-local (0..n_nodes[f]-1), exactly the reference's numbering.
 *  - Return value: 0 on success, negative on error (LSEG_E*); the message is
 *    available from lseg_last_error() (thread-local).  No exception crosses
 *    the ABI.  Calls are stateless and re-entrant.
 */
#ifndef LIDARSEG_B200_H
#define LIDARSEG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSEG_OK 0
#define LSEG_EINVAL (-1)     /* bad argument (reference raises ValueError) */
#define LSEG_EWORKSPACE (-2) /* workspace too small */
#define LSEG_ECUDA (-3)      /* CUDA launch / runtime error */

/* Sensor geometry (reference scan.py:51-139, SensorConfig).  The four angle
 * tables are DEVICE arrays computed on the host exactly as the reference does
 * (cos/sin of ring_elevations, and of phi_j = (2*pi*j)/S, scan.py:119-139) so
 * positions dir*r are bit-identical to the reference's. */
typedef struct lseg_sensor {
  int32_t rings;          /* R >= 2, ring 0 = top beam                        */
  int32_t steps;          /* S >= 3 azimuth steps per revolution              */
  double r_min, r_max;    /* valid window, inclusive (scan.py:177-182)        */
  const double* cos_el;   /* (R)                                               */
  const double* sin_el;   /* (R)                                               */
  const double* cos_az;   /* (S)                                               */
  const double* sin_az;   /* (S)                                               */
} lseg_sensor;

const char* lseg_last_error(void);
const char* lseg_version(void);

/* Stage profiler for the calling thread: after lseg_profile_begin(), every
 * kernel stage enqueued by this library records a CUDA event on its stream;
 * lseg_profile_end() synchronises on the last event and returns, per stage in
 * first-seen order, the summed device milliseconds and the launch count.
 * names_csv (host) receives the comma-separated stage names. */
int lseg_profile_begin(void);
int lseg_profile_end(char* names_csv, size_t names_cap, double* ms, int32_t* counts,
                     int32_t max_stages, int32_t* n_stages);

/* S' = number of kept azimuth steps {0, k, 2k, ...} <= S-1
 * (reference scan.py:215-225 subsample_steps); -1 if k is not in [1, S-1]. */
int32_t lseg_kept_count(int32_t steps, int32_t interval);

/* Scratch bytes needed by any entry point below for this batch shape.
 * label_bound: exclusive bound on label values for lseg_prune_small
 * (pass 0 to size for the pipeline, whose labels are <= R*S'). */
size_t lseg_workspace_bytes(int32_t frames, int32_t rings, int32_t steps, int32_t interval,
                            int64_t label_bound);

/* NEW op (no reference function; inverse of ScanGrid.valid_points,
 * reference scan.py:192-195; definition SURVEY.md §8(a) A2).
 * xyz (P,3) f32, ring (P) i32, frame_offsets (F+1) i64 into the point arrays.
 * Writes ranges (F,R,S) f64: smallest binned r per cell, NaN elsewhere.
 * cell (P) i32 optional (NULL): R*S-local cell of each point or -1. */
int lseg_bin_points(const lseg_sensor* sensor, int32_t frames, const float* xyz,
                    const int32_t* ring, const int64_t* frame_offsets, int64_t total_points,
                    double* ranges, int32_t* cell, void* stream);

/* Replaces build_mesh (reference mesh.py:105-136, _neighbor_grid :83-102).
 * max_edge_length NaN means None (the reference default); otherwise an edge
 * survives iff its fp64 3-D length d <= max_edge_length.
 * Out: node_ids (F,R,S') i32 (-1 absent), neighbors (F,cap,6) i32 slots N0..N5
 * (-1 absent), n_nodes (F) i32; node_rings / node_steps (F,cap) i32 optional. */
int lseg_build_mesh(const lseg_sensor* sensor, int32_t frames, int32_t interval,
                    double max_edge_length, const double* ranges, int32_t* node_ids,
                    int32_t* neighbors, int32_t* node_rings, int32_t* node_steps,
                    int32_t* n_nodes, void* workspace, size_t workspace_bytes, void* stream);

/* Replaces mesh_triangles (reference mesh.py:173-189): per frame all type-A
 * (p, down, diag) faces in row-major order, then all type-B (p, diag, right).
 * tris (F, 2*R*S', 3) i32 padded, n_tris (F). */
int lseg_mesh_triangles(int32_t frames, int32_t rings, int32_t kept, const int32_t* node_ids,
                        int32_t* tris, int32_t* n_tris, void* stream);

/* Replaces estimate_normals (reference normals.py:94-145, node_positions
 * :42-46).  fp64 arithmetic in the reference's operation order.  Writes
 * normals64 (F,cap,3) f64 and/or normals32 (F,cap,3) f32 (either may be
 * NULL; absent rows are NaN) and nmask (F,cap) u8. */
int lseg_estimate_normals(const lseg_sensor* sensor, int32_t frames, int32_t interval,
                          const double* ranges, const int32_t* node_ids, const int32_t* neighbors,
                          const int32_t* n_nodes, double* normals64, float* normals32,
                          uint8_t* nmask, void* stream);

/* Replaces segment (reference segment.py:43-88).  Union-find connected
 * components over mesh edges passing the strict component-wise test
 * |n_p - n_q| < thresholds (host array of 3); label = 1 + rank of the
 * component's minimum node id (identical to the reference's DFS first-touch
 * numbering).  labels (F,R,S) dense i32, 0 off-node; n_labels (F). */
int lseg_segment(int32_t frames, int32_t rings, int32_t steps, int32_t interval,
                 const int32_t* node_ids, const int32_t* neighbors, const int32_t* n_nodes,
                 const double* normals64, const uint8_t* nmask, const double* thresholds,
                 int32_t* labels, int32_t* n_labels, void* workspace, size_t workspace_bytes,
                 void* stream);

/* Replaces backfill (reference segment.py:109-124, _nearest_donor_steps
 * :91-106).  labels_in / labels_out (F,R,S) i32 (must not alias). */
int lseg_backfill(const lseg_sensor* sensor, int32_t frames, const double* ranges,
                  const int32_t* labels_in, int32_t* labels_out, void* stream);

/* Replaces prune_small (reference segment.py:127-160).  label_bound is an
 * exclusive upper bound on label values (the caller knows max+1).  Labels
 * >= label_bound are a caller error: they are not counted, never index the
 * workspace, and come out as -1. */
int lseg_prune_small(int32_t frames, int32_t rings, int32_t steps, const int32_t* labels_in,
                     int32_t min_segment_size, int64_t label_bound, int32_t* labels_out,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Replaces run_pipeline (reference pipeline.py:47-70) preceded by
 * bin_points: the whole hot path for F frames of points in one call.
 * Outputs as in the individual ops; normals32 (F,cap,3) f32;
 * node_labels (F,R,S) optional (NULL) = segment() output before completion;
 * labels (F,R,S) = after backfill + prune_small; n_nodes (F) mesh nodes;
 * n_labels (F) = number of segment() labels (before completion).
 * node_ids and normals32 may be NULL (not written). */
int lseg_run_pipeline(const lseg_sensor* sensor, int32_t frames, int32_t interval,
                      const double* thresholds, int32_t min_segment_size, const float* xyz,
                      const int32_t* ring, const int64_t* frame_offsets, int64_t total_points,
                      double* ranges, int32_t* node_ids, int32_t* neighbors, float* normals32,
                      uint8_t* nmask, int32_t* node_labels, int32_t* labels, int32_t* n_nodes,
                      int32_t* n_labels, void* workspace, size_t workspace_bytes, void* stream);

/* Same as lseg_run_pipeline with one-byte ring ids (every real spinning
 * sensor has <= 256 rings): 13 instead of 16 bytes per input point, which is
 * what bounds the host-to-device copy of a streamed batch. */
int lseg_run_pipeline_r8(const lseg_sensor* sensor, int32_t frames, int32_t interval,
                         const double* thresholds, int32_t min_segment_size, const float* xyz,
                         const uint8_t* ring, const int64_t* frame_offsets, int64_t total_points,
                         double* ranges, int32_t* node_ids, int32_t* neighbors, float* normals32,
                         uint8_t* nmask, int32_t* node_labels, int32_t* labels, int32_t* n_nodes,
                         int32_t* n_labels, void* workspace, size_t workspace_bytes, void* stream);

/* Flags of lseg_run_pipeline_ex. */
#define LSEG_PIPE_CERT_NORMALS 1u /* certified fp32 normals (see below) instead of exact fp64 ones */
#define LSEG_PIPE_RING_U8 2u      /* ring ids are uint8_t (as lseg_run_pipeline_r8) */
#define LSEG_PIPE_RING_SEGMENTS 4u /* points are ring-major and `ring` is an int64_t (frames, rings + 1)
                                      table of absolute point offsets (ring i of frame f = points
                                      [seg[f][i], seg[f][i+1])) instead of a ring id per point:
                                      12 instead of 13 or 16 input bytes per point */

/* lseg_run_pipeline with flags.  By default (and in lseg_run_pipeline / _r8)
 * normals are computed in fp64 with the reference's operation order, so
 * normals32 is the exact float32 rounding of the reference's fp64 normals.
 * With LSEG_PIPE_CERT_NORMALS they are computed in fp32 with a rigorous
 * per-node error bound; every homogeneity decision the bound cannot settle,
 * and every degenerate or ill-conditioned node, is recomputed with the exact
 * fp64 arithmetic, so node_labels / labels are identical in both modes
 * (bit-exact with the reference) while normals32 then agrees with the
 * reference to well within 1e-5 per component (SURVEY.md §8(c) tolerance). */
int lseg_run_pipeline_ex(const lseg_sensor* sensor, int32_t frames, int32_t interval,
                         const double* thresholds, int32_t min_segment_size, uint32_t flags,
                         const float* xyz, const void* ring, const int64_t* frame_offsets,
                         int64_t total_points, double* ranges, int32_t* node_ids, int32_t* neighbors,
                         float* normals32, uint8_t* nmask, int32_t* node_labels, int32_t* labels,
                         int32_t* n_nodes, int32_t* n_labels, void* workspace, size_t workspace_bytes,
                         void* stream);

/* Batched run_pipeline on range grids (reference run_pipeline(scan, cfg),
 * pipeline.py:47-70, over F frames): ranges (F, R, S) f64 with NaN = INVALID
 * as input instead of points; outputs and flags (LSEG_PIPE_CERT_NORMALS) as
 * in lseg_run_pipeline_ex. */
int lseg_run_pipeline_grid(const lseg_sensor* sensor, int32_t frames, int32_t interval,
                           const double* thresholds, int32_t min_segment_size, uint32_t flags,
                           const double* ranges, int32_t* node_ids, int32_t* neighbors, float* normals32,
                           uint8_t* nmask, int32_t* node_labels, int32_t* labels, int32_t* n_nodes,
                           int32_t* n_labels, void* workspace, size_t workspace_bytes, void* stream);

/* The drop-in single-scan path (reference run_pipeline(scan, cfg),
 * pipeline.py:47-70, returning its PipelineResult fields) for F scans in ONE
 * call: ranges (F, R, S) f64 in; mesh node_ids (F,R,S') and neighbors
 * (F,cap,6), fp64 normals64 (F,cap,3) (the reference's NormalMap values,
 * bit-identical; NaN rows where nmask is 0), node_cells (F,cap,2) i32
 * optional (ring, step) of each node = Mesh.node_rings / node_steps,
 * segment() node_labels (F,R,S) optional, final labels (F,R,S).  Exact
 * fp64 normals only. */
int lseg_run_scans(const lseg_sensor* sensor, int32_t frames, int32_t interval, const double* thresholds,
                   int32_t min_segment_size, const double* ranges, int32_t* node_ids, int32_t* neighbors,
                   double* normals64, uint8_t* nmask, int32_t* node_cells, int32_t* node_labels, int32_t* labels,
                   int32_t* n_nodes, int32_t* n_labels, void* workspace, size_t workspace_bytes, void* stream);

/* ---- streaming mesh builder (reference MeshBuilder, mesh.py:139-170;
 * streaming contract SPEC.md:200).  Columns are fed in sweep order; when
 * kept column j arrives (its R ranges, device f64), the valid bits and
 * per-ring ranks of column j are recorded and every slot of column j-1 is
 * emitted (slots reference (ring, rank) pairs).  State: runcnt (R) i32,
 * zeroed before column 0; colrank (R, kept) i32; slots (R, kept, 6) i32. */
int lseg_mb_column(int32_t rings, int32_t kept, int32_t column, double r_min, double r_max, const double* ranges,
                   int32_t* runcnt, int32_t* colrank, int32_t* slots, void* stream);

/* Closes the wrap (slots of columns 0 and kept-1), scans the per-ring
 * counts into row offsets (rowoff (R) i32) and resolves every slot to the
 * reference's row-major node ids: node_ids (R, kept), neighbors
 * (n_nodes, 6), n_nodes (1) -- identical to lseg_build_mesh on the grid. */
int lseg_mb_finish(int32_t rings, int32_t kept, const int32_t* runcnt, const int32_t* colrank, int32_t* slots,
                   int32_t* rowoff, int32_t* node_ids, int32_t* neighbors, int32_t* n_nodes, void* stream);

/* ---- edge-based evaluation (reference evaluate.py:40-94).
 * Label grids (F,R,S) i32, 0 = unlabelled.  Scratch sized by
 * lseg_eval_workspace_bytes. */
size_t lseg_eval_workspace_bytes(int32_t frames, int32_t rings, int32_t steps);

/* Replaces the counting inside edge_prf (evaluate.py:73-94): per frame
 * counts[f] = {n_pred_edges, n_truth_edges, pred edges within the Chebyshev
 * radius of a truth edge, truth edges within the radius of a pred edge}. */
int lseg_edge_counts(int32_t frames, int32_t rings, int32_t steps, const int32_t* pred,
                     const int32_t* truth, int32_t radius, int32_t* counts, void* workspace,
                     size_t workspace_bytes, void* stream);

/* Replaces extract_edges (evaluate.py:40-55): edges (F,R,S) u8. */
int lseg_extract_edges(int32_t frames, int32_t rings, int32_t steps, const int32_t* labels,
                       uint8_t* edges, void* workspace, size_t workspace_bytes, void* stream);

/* Replaces dilate_chebyshev (evaluate.py:58-70): out (F,R,S) u8. */
int lseg_dilate_chebyshev(int32_t frames, int32_t rings, int32_t steps, const uint8_t* mask,
                          int32_t radius, uint8_t* out, void* workspace, size_t workspace_bytes,
                          void* stream);

/* ---- scan simulator (reference simulate.py:59-448).
 * A scene is n_prims packed records of LSEG_PRIM_STRIDE doubles (layout in
 * csrc/lseg_sim.cu, built by simulate.py:_pack); ties between primitives keep
 * the earlier one, as cast_grid does. */
#define LSEG_PRIM_STRIDE 24

/* Replaces cast_grid (simulate.py:383-401), batched: frames x (rings, steps)
 * beams, t_out = nearest hit (+inf if none), ids_out = surface id (0 if none).
 * poses (frames, 12) = row-major rotation of the beam directions then the
 * sensor origin, or NULL for the reference's origin-centred scan. */
int lseg_cast_grid(const lseg_sensor* sensor, int32_t frames, const double* prims, int32_t n_prims,
                   const double* poses, double* t_out, int32_t* ids_out, void* stream);

/* Replaces ray_intersect (simulate.py:364-380) for n_rays arbitrary rays
 * (origins, unit directions: (n_rays, 3) each). */
int lseg_cast_rays(const double* prims, int32_t n_prims, int64_t n_rays, const double* origins,
                   const double* dirs, double* t_out, int32_t* ids_out, void* stream);

/* scan_scene's noise + range window (simulate.py:404-421): ranges = t
 * (+ noise where the beam hit; noise may be NULL), NaN + label 0 outside
 * [r_min, r_max]. */
int lseg_apply_scan(int64_t n_cells, double r_min, double r_max, const double* t, const int32_t* ids,
                    const double* noise, double* ranges, int32_t* labels, void* stream);

/* Replaces scene_normals (simulate.py:424-448): (rings, steps, 3) f64,
 * oriented toward the sensor, NaN where labels == 0. */
int lseg_scene_normals(const lseg_sensor* sensor, const double* prims, int32_t n_prims,
                       const double* ranges, const int32_t* labels, double* normals, void* stream);

/* ---- text formats (reference io.py).  Host-side, no
 * device needed.  Formats n_rows rows of n_cols values (row-major doubles):
 * col_kind[c] = 0 -> Python repr(float) text (io.py:42-47, shortest
 * round-trip), 1 -> integer; cells joined by ' ', rows ended by '\n'.
 * out = NULL returns an upper bound of the bytes needed; otherwise returns the
 * bytes written (-2 if capacity is too small, -1 on bad arguments).
 * threads <= 0: all hardware threads. */
int64_t lseg_format_rows(int64_t n_rows, int32_t n_cols, const double* values, const uint8_t* col_kind,
                         char* out, int64_t capacity, int32_t threads);

#ifdef __cplusplus
}
#endif
#endif /* LIDARSEG_B200_H */
