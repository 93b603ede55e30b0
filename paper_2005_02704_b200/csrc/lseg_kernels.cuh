// Kernel launchers (lseg_kernels.cu) used by the C ABI (lseg_abi.cu).
#pragma once
#include "lseg_internal.cuh"

namespace lseg {
void launch_bin(const lseg_sensor& sn, int F, const float* xyz, const int32_t* ring, const int64_t* off,
                int64_t P, double* ranges, int32_t* cell, cudaStream_t st);
void launch_mesh(const lseg_sensor& sn, const Shape& sh, double max_edge, const double* ranges,
                 const Workspace& ws, int32_t* node_ids, int32_t* neighbors, int32_t* node_rings,
                 int32_t* node_steps, int32_t* n_nodes, cudaStream_t st);
void launch_normals(const lseg_sensor& sn, const Shape& sh, const double* ranges, const int32_t* node_ids,
                    const int32_t* neighbors, double* n64, float* n32, uint8_t* nmask, cudaStream_t st);
void launch_segment(const Shape& sh, int nslots, const int32_t* node_ids, const int32_t* neighbors,
                    const int32_t* n_nodes, const double* n64, const uint8_t* nmask, const double* thr,
                    int32_t* labels, int32_t* n_labels, const Workspace& ws, int32_t* hist, cudaStream_t st);
void launch_ring_fill(int mode, const lseg_sensor& sn, const Shape& sh, const double* ranges,
                      const int32_t* in, int32_t* out, int32_t* hist, const int32_t* remap,
                      const int32_t* fscal, int64_t K, int32_t m, cudaStream_t st);
void launch_prune_plan(const Shape& sh, const int32_t* n_labels, int64_t K, int32_t m, const int32_t* hist,
                       int32_t* remap, int32_t* fscal, cudaStream_t st);
void launch_hist(const Shape& sh, int64_t K, const int32_t* labels, int32_t* hist, cudaStream_t st);
void launch_triangles(int F, int R, int Sk, const int32_t* node_ids, int32_t* tris, int32_t* n_tris,
                      cudaStream_t st);
void launch_valid_scan(const lseg_sensor& sn, const Shape& sh, const double* ranges, const Workspace& ws,
                       int32_t* n_nodes, cudaStream_t st);
void launch_root_rank(const Shape& sh, const int32_t* n_nodes, const int32_t* parent, const uint8_t* nmask,
                      int32_t* rank, int32_t* n_labels, int32_t* hist, int64_t K, cudaStream_t st);
void launch_fused_graph(const lseg_sensor& sn, const Shape& sh, const Workspace& ws, const double* ranges,
                        const double* thr, int32_t* node_ids, int32_t* neighbors, float* n32, uint8_t* nmask,
                        int32_t* n_nodes, int32_t* n_labels, int32_t* node_labels, bool fbits_valid,
                        bool exact_normals, float* dbg_err, cudaStream_t st, double* n64 = nullptr,
                        int32_t* node_rc = nullptr);
void launch_bin_fused(const lseg_sensor& sn, const Shape& sh, const float* xyz, const void* ring, int ring_bytes,
                      const int64_t* off, const Workspace& ws, double* ranges, int32_t* n_nodes, cudaStream_t st);
void launch_frame_scan(const Shape& sh, const Workspace& ws, int32_t* n_nodes, cudaStream_t st);
void launch_scan_bits(const Shape& sh, const uint32_t* bits, int32_t* pre, int32_t* counts, int32_t* hist, int64_t K,
                      cudaStream_t st);
void launch_prune_fused(const Shape& sh, const Workspace& ws, int32_t min_size, int32_t* labels, cudaStream_t st);
void debug_phases(double* out);
size_t eval_workspace_bytes(int F, int R, int S);
int eval_counts(int F, int R, int S, const int32_t* pred, const int32_t* truth, int r, int32_t* counts, void* ws,
                cudaStream_t st);
int eval_extract(int F, int R, int S, const int32_t* labels, uint8_t* out, void* ws, cudaStream_t st);
int eval_dilate(int F, int R, int S, const uint8_t* mask, int r, uint8_t* out, void* ws, cudaStream_t st);
void launch_cast_grid(const lseg_sensor& sn, int F, const double* prims, int n_prims, const double* poses,
                      double* t, int32_t* id, cudaStream_t st);
void launch_cast_rays(const double* prims, int n_prims, int64_t n, const double* origins, const double* dirs,
                      double* t, int32_t* id, cudaStream_t st);
void launch_apply_scan(int64_t n, double r_min, double r_max, const double* t, const int32_t* id,
                       const double* noise, double* ranges, int32_t* labels, cudaStream_t st);
void launch_scene_normals(const lseg_sensor& sn, const double* prims, int n_prims, const double* ranges,
                          const int32_t* labels, double* out, cudaStream_t st);
void launch_selftest_math(int64_t n, uint64_t seed, unsigned long long* bad, cudaStream_t st);
void launch_mb_column(int R, int Sk, int j, double r_min, double r_max, const double* col, int32_t* runcnt,
                      int32_t* colrank, int32_t* slots, cudaStream_t st);
void launch_mb_finish(int R, int Sk, const int32_t* runcnt, const int32_t* colrank, int32_t* slots, int32_t* rowoff,
                      int32_t* node_ids, int32_t* neighbors, int32_t* n_nodes, cudaStream_t st);

}  // namespace lseg
