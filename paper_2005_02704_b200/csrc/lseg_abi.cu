// C ABI of lidarseg_b200 (declared in include/lidarseg_b200.h).
//
// Host-side validation mirrors the reference's ValueError contract
// (scan.py:76-88, :223-224; segment.py:32-36); every entry point enqueues on
// the caller's stream and returns without synchronising.

#include <math.h>
#include <stdio.h>

#include <string>
#include <vector>
#include <cstring>

#include "lseg_internal.cuh"
#include "lseg_kernels.cuh"

namespace lseg {
void debug_tile_cc(int n, const unsigned long long* masks, int32_t* parent, uint32_t* lroots);

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LSEG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return LSEG_OK;
}

// ---------------------------------------------------------------- profiler
struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<const char*> names;  // names[i] = stage that ended at event i (nullptr = start mark)
  size_t used = 0;
};
static thread_local Profiler g_prof;

void prof_mark(const char* stage, cudaStream_t st) {
  Profiler& p = g_prof;
  if (!p.on) return;
  if (p.used == p.pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    p.pool.push_back(e);
  }
  cudaEventRecord(p.pool[p.used], st);
  if (p.names.size() <= p.used) p.names.resize(p.used + 1);
  p.names[p.used] = stage;
  ++p.used;
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

Workspace carve(const Shape& s, int64_t label_bound, void* base) {
  Workspace w{};
  const int64_t K = label_bound > 0 ? label_bound : s.cap + 1;
  w.K = K;
  size_t off = 0;
  char* b = static_cast<char*>(base);
  auto take = [&](size_t bytes) -> char* {
    char* p = b ? b + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  const size_t words = (size_t)s.F * s.R * s.Wk;
  w.vbits = reinterpret_cast<uint32_t*>(take(words * 4));
  w.wpre = reinterpret_cast<int32_t*>(take(words * 4));
  w.parent = reinterpret_cast<int32_t*>(take((size_t)s.F * s.cap * 4));
  w.rank = reinterpret_cast<int32_t*>(take((size_t)s.F * s.cap * 4));
  w.normals64 = reinterpret_cast<double*>(take((size_t)s.F * s.cap * 3 * 8));
  w.hist = reinterpret_cast<int32_t*>(take((size_t)s.F * K * 4));
  w.remap = reinterpret_cast<int32_t*>(take((size_t)s.F * K * 4));
  w.fscal = reinterpret_cast<int32_t*>(take((size_t)s.F * 4 * 4));
  w.lab_tmp = reinterpret_cast<int32_t*>(take((size_t)s.F * s.R * s.S * 4));
  w.bnorm = reinterpret_cast<double*>(
      take((size_t)s.F * (2 * ((s.R + kTileR - 1) / kTileR) * (size_t)s.Sk + 2 * ((s.Sk + kTileC - 1) / kTileC) * (size_t)s.R) * 3 * 8));
  {
    const size_t tiles = (size_t)s.F * ((s.R + kTileR - 1) / kTileR) * ((s.Sk + kTileC - 1) / kTileC);
    w.masks = reinterpret_cast<unsigned long long*>(take(tiles * kTileR * 5 * 8));
  }
  w.fallback = reinterpret_cast<int32_t*>(take((size_t)s.F * 4));
  w.seg = reinterpret_cast<int64_t*>(take((size_t)s.F * (s.R + 1) * 8));
  w.fbits = reinterpret_cast<uint32_t*>(take((size_t)s.F * s.R * ((s.S + 31) / 32) * 4));
  w.rbits = reinterpret_cast<uint32_t*>(take(words * 4));
  w.lroots = reinterpret_cast<uint32_t*>(take(words * 4));
  w.rpre = reinterpret_cast<int32_t*>(take(words * 4));
  w.rcnt = reinterpret_cast<int32_t*>(take((size_t)s.F * s.R * 4));
  w.ucnt = reinterpret_cast<unsigned long long*>(take(2 * 8));
  w.bytes = off;
  return w;
}

static int check_sensor(const lseg_sensor* sn) {
  if (!sn) return fail(LSEG_EINVAL, "sensor is NULL");
  if (sn->rings < 2) return fail(LSEG_EINVAL, "ring_elevations needs at least 2 entries");
  if (sn->steps < 3) return fail(LSEG_EINVAL, "azimuth_steps must be >= 3");
  if (sn->steps > 16384) return fail(LSEG_EINVAL, "azimuth_steps > 16384 not supported");
  if (!(0.0 < sn->r_min && sn->r_min < sn->r_max)) return fail(LSEG_EINVAL, "require 0 < r_min < r_max");
  if (!sn->cos_el || !sn->sin_el || !sn->cos_az || !sn->sin_az)
    return fail(LSEG_EINVAL, "sensor angle tables must be device pointers");
  return LSEG_OK;
}

static int check_shape(int F, int R, int S, int k, Shape* out) {
  if (F < 0) return fail(LSEG_EINVAL, "frames must be >= 0");
  if (F > 65535) return fail(LSEG_EINVAL, "at most 65535 frames per call");
  if (kept_count(S, k) < 0)
    return fail(LSEG_EINVAL, "interval " + std::to_string(k) + " not in [1, " + std::to_string(S - 1) + "]");
  *out = make_shape(F, R, S, k);
  if (out->cap >= (int64_t)1 << 30) return fail(LSEG_EINVAL, "grid too large for int32 node ids");
  return LSEG_OK;
}

static int check_ws(const Shape& s, int64_t label_bound, void* ws, size_t ws_bytes, Workspace* out) {
  *out = carve(s, label_bound, ws);
  if (!ws || ws_bytes < out->bytes)
    return fail(LSEG_EWORKSPACE, "workspace too small: need " + std::to_string(out->bytes) + " bytes");
  return LSEG_OK;
}

}  // namespace lseg

using namespace lseg;

extern "C" {

const char* lseg_last_error(void) { return g_last_error.c_str(); }

// Self-test of the branch-free sqrt / reciprocal used by the pipeline kernels
// (not part of the public header): mismatch counts vs __dsqrt_rn / __drcp_rn.
int lseg_selftest_math(int64_t n, uint64_t seed, unsigned long long* bad, void* stream) {
  if (n < 0 || !bad) return fail(LSEG_EINVAL, "bad arguments");
  launch_selftest_math(n, seed, bad, (cudaStream_t)stream);
  return check_launch("selftest_math");
}

// Debug hook: summed per-phase SM cycles of k_tile (builds with LSEG_PHASES=1).
void lseg_debug_tile_phases(double* out8) { lseg::debug_phases(out8); }

const char* lseg_version(void) { return "lidarseg_b200 0.1.0 sm_100a"; }

int lseg_profile_begin(void) {
  g_prof.on = true;
  g_prof.used = 0;
  return LSEG_OK;
}

int lseg_profile_end(char* names_csv, size_t names_cap, double* ms, int32_t* counts, int32_t max_stages,
                     int32_t* n_stages) {
  Profiler& p = g_prof;
  p.on = false;
  std::vector<std::string> order;
  std::vector<double> tot;
  std::vector<int> cnt;
  if (p.used > 0 && cudaEventSynchronize(p.pool[p.used - 1]) != cudaSuccess)
    return fail(LSEG_ECUDA, "profile_end: event sync failed");
  for (size_t i = 1; i < p.used; ++i) {
    if (!p.names[i]) continue;  // a start mark closes nothing
    float t = 0.f;
    cudaEventElapsedTime(&t, p.pool[i - 1], p.pool[i]);
    size_t j = 0;
    while (j < order.size() && order[j] != p.names[i]) ++j;
    if (j == order.size()) { order.push_back(p.names[i]); tot.push_back(0.0); cnt.push_back(0); }
    tot[j] += t;
    cnt[j] += 1;
  }
  std::string csv;
  const int n = (int)order.size() < max_stages ? (int)order.size() : max_stages;
  for (int j = 0; j < n; ++j) {
    if (j) csv += ",";
    csv += order[j];
    if (ms) ms[j] = tot[j];
    if (counts) counts[j] = cnt[j];
  }
  if (names_csv && names_cap) {
    strncpy(names_csv, csv.c_str(), names_cap - 1);
    names_csv[names_cap - 1] = 0;
  }
  if (n_stages) *n_stages = n;
  p.used = 0;
  return LSEG_OK;
}

int32_t lseg_kept_count(int32_t steps, int32_t interval) { return kept_count(steps, interval); }

size_t lseg_workspace_bytes(int32_t frames, int32_t rings, int32_t steps, int32_t interval,
                            int64_t label_bound) {
  if (kept_count(steps, interval) < 0 || frames < 0 || rings < 1) return 0;
  return carve(make_shape(frames, rings, steps, interval), label_bound, nullptr).bytes;
}

int lseg_bin_points(const lseg_sensor* sensor, int32_t frames, const float* xyz, const int32_t* ring,
                    const int64_t* frame_offsets, int64_t total_points, double* ranges, int32_t* cell,
                    void* stream) {
  if (int e = check_sensor(sensor)) return e;
  if (frames < 0 || total_points < 0) return fail(LSEG_EINVAL, "negative sizes");
  if (frames == 0) return LSEG_OK;
  if (!ranges || !frame_offsets || (total_points > 0 && (!xyz || !ring)))
    return fail(LSEG_EINVAL, "NULL buffer");
  launch_bin(*sensor, frames, xyz, ring, frame_offsets, total_points, ranges, cell, (cudaStream_t)stream);
  return check_launch("bin_points");
}

int lseg_build_mesh(const lseg_sensor* sensor, int32_t frames, int32_t interval, double max_edge_length,
                    const double* ranges, int32_t* node_ids, int32_t* neighbors, int32_t* node_rings,
                    int32_t* node_steps, int32_t* n_nodes, void* workspace, size_t workspace_bytes,
                    void* stream) {
  if (int e = check_sensor(sensor)) return e;
  Shape sh;
  if (int e = check_shape(frames, sensor->rings, sensor->steps, interval, &sh)) return e;
  if (frames == 0) return LSEG_OK;
  Workspace ws;
  if (int e = check_ws(sh, 0, workspace, workspace_bytes, &ws)) return e;
  if (!ranges || !node_ids || !neighbors || !n_nodes) return fail(LSEG_EINVAL, "NULL buffer");
  launch_mesh(*sensor, sh, max_edge_length, ranges, ws, node_ids, neighbors, node_rings, node_steps, n_nodes,
              (cudaStream_t)stream);
  return check_launch("build_mesh");
}

int lseg_mesh_triangles(int32_t frames, int32_t rings, int32_t kept, const int32_t* node_ids, int32_t* tris,
                        int32_t* n_tris, void* stream) {
  if (frames < 0 || rings < 1 || kept < 1) return fail(LSEG_EINVAL, "bad shape");
  if (frames == 0) return LSEG_OK;
  if (!node_ids || !tris || !n_tris) return fail(LSEG_EINVAL, "NULL buffer");
  launch_triangles(frames, rings, kept, node_ids, tris, n_tris, (cudaStream_t)stream);
  return check_launch("mesh_triangles");
}

int lseg_estimate_normals(const lseg_sensor* sensor, int32_t frames, int32_t interval, const double* ranges,
                          const int32_t* node_ids, const int32_t* neighbors, const int32_t* n_nodes,
                          double* normals64, float* normals32, uint8_t* nmask, void* stream) {
  (void)n_nodes;
  if (int e = check_sensor(sensor)) return e;
  Shape sh;
  if (int e = check_shape(frames, sensor->rings, sensor->steps, interval, &sh)) return e;
  if (frames == 0) return LSEG_OK;
  if (!ranges || !node_ids || !neighbors || !nmask) return fail(LSEG_EINVAL, "NULL buffer");
  launch_normals(*sensor, sh, ranges, node_ids, neighbors, normals64, normals32, nmask, (cudaStream_t)stream);
  return check_launch("estimate_normals");
}

int lseg_segment(int32_t frames, int32_t rings, int32_t steps, int32_t interval, const int32_t* node_ids,
                 const int32_t* neighbors, const int32_t* n_nodes, const double* normals64,
                 const uint8_t* nmask, const double* thresholds, int32_t* labels, int32_t* n_labels,
                 void* workspace, size_t workspace_bytes, void* stream) {
  Shape sh;
  if (int e = check_shape(frames, rings, steps, interval, &sh)) return e;
  if (!thresholds) return fail(LSEG_EINVAL, "thresholds is NULL");
  for (int c = 0; c < 3; ++c)
    if (!(thresholds[c] > 0.0 && thresholds[c] <= 2.0)) return fail(LSEG_EINVAL, "thresholds must be in (0, 2]");
  if (frames == 0) return LSEG_OK;
  Workspace ws;
  if (int e = check_ws(sh, 0, workspace, workspace_bytes, &ws)) return e;
  if (!node_ids || !neighbors || !n_nodes || !normals64 || !nmask || !labels || !n_labels)
    return fail(LSEG_EINVAL, "NULL buffer");
  // all 6 slots: correct for any symmetric-or-not neighbour table a caller passes
  launch_segment(sh, 6, node_ids, neighbors, n_nodes, normals64, nmask, thresholds, labels, n_labels, ws,
                 nullptr, (cudaStream_t)stream);
  return check_launch("segment");
}

int lseg_backfill(const lseg_sensor* sensor, int32_t frames, const double* ranges, const int32_t* labels_in,
                  int32_t* labels_out, void* stream) {
  if (int e = check_sensor(sensor)) return e;
  if (frames < 0) return fail(LSEG_EINVAL, "frames must be >= 0");
  if (frames == 0) return LSEG_OK;
  if (!ranges || !labels_in || !labels_out) return fail(LSEG_EINVAL, "NULL buffer");
  if (labels_in == labels_out) return fail(LSEG_EINVAL, "labels_in and labels_out must not alias");
  const Shape sh = make_shape(frames, sensor->rings, sensor->steps, 1);
  launch_ring_fill(0, *sensor, sh, ranges, labels_in, labels_out, nullptr, nullptr, nullptr, 0, 0,
                   (cudaStream_t)stream);
  return check_launch("backfill");
}

int lseg_prune_small(int32_t frames, int32_t rings, int32_t steps, const int32_t* labels_in,
                     int32_t min_segment_size, int64_t label_bound, int32_t* labels_out, void* workspace,
                     size_t workspace_bytes, void* stream) {
  if (frames < 0 || rings < 1 || steps < 1) return fail(LSEG_EINVAL, "bad shape");
  if (min_segment_size < 0) return fail(LSEG_EINVAL, "min_segment_size must be >= 0");
  if (label_bound < 1) return fail(LSEG_EINVAL, "label_bound must be >= 1");
  if (steps > 16384) return fail(LSEG_EINVAL, "steps > 16384 not supported");
  if (frames == 0) return LSEG_OK;
  if (!labels_in || !labels_out) return fail(LSEG_EINVAL, "NULL buffer");
  if (labels_in == labels_out) return fail(LSEG_EINVAL, "labels_in and labels_out must not alias");
  Shape shr = make_shape(frames, rings, steps < 2 ? 2 : steps, 1);
  Workspace ws;
  if (int e = check_ws(shr, label_bound, workspace, workspace_bytes, &ws)) return e;
  shr.S = steps;
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(ws.hist, 0, sizeof(int32_t) * (size_t)frames * label_bound, st);
  launch_hist(shr, label_bound, labels_in, ws.hist, st);
  launch_prune_plan(shr, nullptr, label_bound, min_segment_size, ws.hist, ws.remap, ws.fscal, st);
  lseg_sensor dummy{};
  dummy.rings = rings;
  dummy.steps = steps;
  launch_ring_fill(1, dummy, shr, nullptr, labels_in, labels_out, ws.hist, ws.remap, ws.fscal, label_bound,
                   min_segment_size, st);
  return check_launch("prune_small");
}

// Test hook (not in the public header): per-node certified error bounds of the
// next fused pipeline launch on this thread (0 for nodes that took the exact
// path, -1 without a normal).
static thread_local float* g_dbg_err = nullptr;

static int run_pipeline_impl(const lseg_sensor* sensor, int32_t frames, int32_t interval, const double* thresholds,
                             int32_t min_segment_size, uint32_t flags, const float* xyz, const void* ring,
                             int ring_bytes,
                             const int64_t* frame_offsets, int64_t total_points, double* ranges, int32_t* node_ids,
                             int32_t* neighbors, float* normals32, uint8_t* nmask, int32_t* node_labels,
                             int32_t* labels, int32_t* n_nodes, int32_t* n_labels, void* workspace,
                             size_t workspace_bytes, void* stream) {
  if (int e = check_sensor(sensor)) return e;
  Shape sh;
  if (int e = check_shape(frames, sensor->rings, sensor->steps, interval, &sh)) return e;
  if (!thresholds) return fail(LSEG_EINVAL, "thresholds is NULL");
  for (int c = 0; c < 3; ++c)
    if (!(thresholds[c] > 0.0 && thresholds[c] <= 2.0)) return fail(LSEG_EINVAL, "thresholds must be in (0, 2]");
  if (min_segment_size < 0) return fail(LSEG_EINVAL, "min_segment_size must be >= 0");
  if (frames == 0) return LSEG_OK;
  Workspace ws;
  if (int e = check_ws(sh, 0, workspace, workspace_bytes, &ws)) return e;
  if (!ranges || !neighbors || !nmask || !labels || !n_nodes || !n_labels || !frame_offsets)
    return fail(LSEG_EINVAL, "NULL buffer");  // node_ids / normals32 / node_labels optional
  cudaStream_t st = (cudaStream_t)stream;
  prof_mark(nullptr, st);
  const bool fused_bin = sensor->steps <= 8192;
  if (!fused_bin && ring_bytes != 4)
    return fail(LSEG_EINVAL, "byte ring ids / ring segments need azimuth_steps <= 8192");
  if (ring_bytes == 0 && !ring) return fail(LSEG_EINVAL, "ring segment table is NULL");
  if (fused_bin) {
    launch_bin_fused(*sensor, sh, xyz, ring, ring_bytes, frame_offsets, ws, ranges, n_nodes, st);
  } else {
    launch_bin(*sensor, frames, xyz, static_cast<const int32_t*>(ring), frame_offsets, total_points, ranges, nullptr,
               st);
    launch_valid_scan(*sensor, sh, ranges, ws, n_nodes, st);
  }
  float* dbg = g_dbg_err;
  g_dbg_err = nullptr;
  launch_fused_graph(*sensor, sh, ws, ranges, thresholds, node_ids, neighbors, normals32, nmask, n_nodes, n_labels,
                     node_labels, fused_bin, (flags & LSEG_PIPE_CERT_NORMALS) == 0, dbg, st);
  launch_prune_fused(sh, ws, min_segment_size, labels, st);
  return check_launch("run_pipeline");
}

int lseg_run_pipeline(const lseg_sensor* sensor, int32_t frames, int32_t interval, const double* thresholds,
                      int32_t min_segment_size, const float* xyz, const int32_t* ring,
                      const int64_t* frame_offsets, int64_t total_points, double* ranges, int32_t* node_ids,
                      int32_t* neighbors, float* normals32, uint8_t* nmask, int32_t* node_labels,
                      int32_t* labels, int32_t* n_nodes, int32_t* n_labels, void* workspace,
                      size_t workspace_bytes, void* stream) {
  return run_pipeline_impl(sensor, frames, interval, thresholds, min_segment_size, 0u, xyz, ring, 4, frame_offsets,
                           total_points, ranges, node_ids, neighbors, normals32, nmask, node_labels, labels, n_nodes,
                           n_labels, workspace, workspace_bytes, stream);
}

int lseg_run_pipeline_r8(const lseg_sensor* sensor, int32_t frames, int32_t interval, const double* thresholds,
                         int32_t min_segment_size, const float* xyz, const uint8_t* ring,
                         const int64_t* frame_offsets, int64_t total_points, double* ranges, int32_t* node_ids,
                         int32_t* neighbors, float* normals32, uint8_t* nmask, int32_t* node_labels,
                         int32_t* labels, int32_t* n_nodes, int32_t* n_labels, void* workspace,
                         size_t workspace_bytes, void* stream) {
  return run_pipeline_impl(sensor, frames, interval, thresholds, min_segment_size, 0u, xyz, ring, 1, frame_offsets,
                           total_points, ranges, node_ids, neighbors, normals32, nmask, node_labels, labels, n_nodes,
                           n_labels, workspace, workspace_bytes, stream);
}

int lseg_run_pipeline_ex(const lseg_sensor* sensor, int32_t frames, int32_t interval, const double* thresholds,
                         int32_t min_segment_size, uint32_t flags, const float* xyz, const void* ring,
                         const int64_t* frame_offsets, int64_t total_points, double* ranges, int32_t* node_ids,
                         int32_t* neighbors, float* normals32, uint8_t* nmask, int32_t* node_labels,
                         int32_t* labels, int32_t* n_nodes, int32_t* n_labels, void* workspace,
                         size_t workspace_bytes, void* stream) {
  if (flags & ~(LSEG_PIPE_CERT_NORMALS | LSEG_PIPE_RING_U8 | LSEG_PIPE_RING_SEGMENTS))
    return fail(LSEG_EINVAL, "unknown pipeline flags");
  if ((flags & LSEG_PIPE_RING_U8) && (flags & LSEG_PIPE_RING_SEGMENTS))
    return fail(LSEG_EINVAL, "LSEG_PIPE_RING_U8 and LSEG_PIPE_RING_SEGMENTS are exclusive");
  const int ring_bytes = (flags & LSEG_PIPE_RING_SEGMENTS) ? 0 : (flags & LSEG_PIPE_RING_U8) ? 1 : 4;
  return run_pipeline_impl(sensor, frames, interval, thresholds, min_segment_size, flags, xyz, ring,
                           ring_bytes, frame_offsets, total_points, ranges, node_ids,
                           neighbors, normals32, nmask, node_labels, labels, n_nodes, n_labels, workspace,
                           workspace_bytes, stream);
}

int lseg_run_pipeline_grid(const lseg_sensor* sensor, int32_t frames, int32_t interval, const double* thresholds,
                           int32_t min_segment_size, uint32_t flags, const double* ranges, int32_t* node_ids,
                           int32_t* neighbors, float* normals32, uint8_t* nmask, int32_t* node_labels,
                           int32_t* labels, int32_t* n_nodes, int32_t* n_labels, void* workspace,
                           size_t workspace_bytes, void* stream) {
  if (int e = check_sensor(sensor)) return e;
  if (flags & ~LSEG_PIPE_CERT_NORMALS) return fail(LSEG_EINVAL, "unknown pipeline flags");
  Shape sh;
  if (int e = check_shape(frames, sensor->rings, sensor->steps, interval, &sh)) return e;
  if (!thresholds) return fail(LSEG_EINVAL, "thresholds is NULL");
  for (int c = 0; c < 3; ++c)
    if (!(thresholds[c] > 0.0 && thresholds[c] <= 2.0)) return fail(LSEG_EINVAL, "thresholds must be in (0, 2]");
  if (min_segment_size < 0) return fail(LSEG_EINVAL, "min_segment_size must be >= 0");
  if (frames == 0) return LSEG_OK;
  Workspace ws;
  if (int e = check_ws(sh, 0, workspace, workspace_bytes, &ws)) return e;
  if (!ranges || !neighbors || !nmask || !labels || !n_nodes || !n_labels)
    return fail(LSEG_EINVAL, "NULL buffer");  // node_ids / normals32 / node_labels optional
  cudaStream_t st = (cudaStream_t)stream;
  prof_mark(nullptr, st);
  float* dbg = g_dbg_err;
  g_dbg_err = nullptr;
  launch_valid_scan(*sensor, sh, ranges, ws, n_nodes, st);
  launch_fused_graph(*sensor, sh, ws, ranges, thresholds, node_ids, neighbors, normals32, nmask, n_nodes, n_labels,
                     node_labels, false, (flags & LSEG_PIPE_CERT_NORMALS) == 0, dbg, st);
  launch_prune_fused(sh, ws, min_segment_size, labels, st);
  return check_launch("run_pipeline_grid");
}

int lseg_run_scans(const lseg_sensor* sensor, int32_t frames, int32_t interval, const double* thresholds,
                   int32_t min_segment_size, const double* ranges, int32_t* node_ids, int32_t* neighbors,
                   double* normals64, uint8_t* nmask, int32_t* node_cells, int32_t* node_labels, int32_t* labels,
                   int32_t* n_nodes, int32_t* n_labels, void* workspace, size_t workspace_bytes, void* stream) {
  if (int e = check_sensor(sensor)) return e;
  Shape sh;
  if (int e = check_shape(frames, sensor->rings, sensor->steps, interval, &sh)) return e;
  if (!thresholds) return fail(LSEG_EINVAL, "thresholds is NULL");
  for (int c = 0; c < 3; ++c)
    if (!(thresholds[c] > 0.0 && thresholds[c] <= 2.0)) return fail(LSEG_EINVAL, "thresholds must be in (0, 2]");
  if (min_segment_size < 0) return fail(LSEG_EINVAL, "min_segment_size must be >= 0");
  if (frames == 0) return LSEG_OK;
  Workspace ws;
  if (int e = check_ws(sh, 0, workspace, workspace_bytes, &ws)) return e;
  if (!ranges || !node_ids || !neighbors || !normals64 || !nmask || !labels || !n_nodes || !n_labels)
    return fail(LSEG_EINVAL, "NULL buffer");
  cudaStream_t st = (cudaStream_t)stream;
  prof_mark(nullptr, st);
  launch_valid_scan(*sensor, sh, ranges, ws, n_nodes, st);
  launch_fused_graph(*sensor, sh, ws, ranges, thresholds, node_ids, neighbors, nullptr, nmask, n_nodes, n_labels,
                     node_labels, false, true, nullptr, st, normals64, node_cells);
  launch_prune_fused(sh, ws, min_segment_size, labels, st);
  return check_launch("run_scans");
}

int lseg_mb_column(int32_t rings, int32_t kept, int32_t column, double r_min, double r_max, const double* ranges,
                   int32_t* runcnt, int32_t* colrank, int32_t* slots, void* stream) {
  if (rings < 1 || kept < 2 || kept > 65535 || rings > 32767) return fail(LSEG_EINVAL, "bad shape");
  if (column < 0 || column >= kept) return fail(LSEG_EINVAL, "column out of range");
  if (!ranges || !runcnt || !colrank || !slots) return fail(LSEG_EINVAL, "NULL buffer");
  launch_mb_column(rings, kept, column, r_min, r_max, ranges, runcnt, colrank, slots, (cudaStream_t)stream);
  return check_launch("mb_column");
}

int lseg_mb_finish(int32_t rings, int32_t kept, const int32_t* runcnt, const int32_t* colrank, int32_t* slots,
                   int32_t* rowoff, int32_t* node_ids, int32_t* neighbors, int32_t* n_nodes, void* stream) {
  if (rings < 1 || kept < 2 || kept > 65535 || rings > 32767) return fail(LSEG_EINVAL, "bad shape");
  if (!runcnt || !colrank || !slots || !rowoff || !node_ids || !neighbors || !n_nodes)
    return fail(LSEG_EINVAL, "NULL buffer");
  launch_mb_finish(rings, kept, runcnt, colrank, slots, rowoff, node_ids, neighbors, n_nodes, (cudaStream_t)stream);
  return check_launch("mb_finish");
}

void lseg_debug_cert_err(float* per_node_err) { g_dbg_err = per_node_err; }

void lseg_debug_tile_cc(int n, const unsigned long long* masks, int32_t* parent, uint32_t* lroots) {
  lseg::debug_tile_cc(n, masks, parent, lroots);
}

// ---------------------------------------------------------------- evaluator (F1)
size_t lseg_eval_workspace_bytes(int32_t frames, int32_t rings, int32_t steps) {
  if (frames < 0 || rings < 1 || steps < 1) return 0;
  return eval_workspace_bytes(frames, rings, steps);
}

static int check_eval(int32_t frames, int32_t rings, int32_t steps, int32_t radius, void* ws, size_t ws_bytes) {
  if (frames < 0 || rings < 1 || steps < 1) return fail(LSEG_EINVAL, "bad shape");
  if (radius < 0) return fail(LSEG_EINVAL, "dilation_radius must be >= 0");
  if (frames > 0 && (!ws || ws_bytes < eval_workspace_bytes(frames, rings, steps)))
    return fail(LSEG_EWORKSPACE, "workspace too small");
  return LSEG_OK;
}

int lseg_edge_counts(int32_t frames, int32_t rings, int32_t steps, const int32_t* pred, const int32_t* truth,
                     int32_t radius, int32_t* counts, void* workspace, size_t workspace_bytes, void* stream) {
  if (int e = check_eval(frames, rings, steps, radius, workspace, workspace_bytes)) return e;
  if (frames == 0) return LSEG_OK;
  if (!pred || !truth || !counts) return fail(LSEG_EINVAL, "NULL buffer");
  return eval_counts(frames, rings, steps, pred, truth, radius, counts, workspace, (cudaStream_t)stream);
}

int lseg_extract_edges(int32_t frames, int32_t rings, int32_t steps, const int32_t* labels, uint8_t* edges,
                       void* workspace, size_t workspace_bytes, void* stream) {
  if (int e = check_eval(frames, rings, steps, 0, workspace, workspace_bytes)) return e;
  if (frames == 0) return LSEG_OK;
  if (!labels || !edges) return fail(LSEG_EINVAL, "NULL buffer");
  return eval_extract(frames, rings, steps, labels, edges, workspace, (cudaStream_t)stream);
}

int lseg_dilate_chebyshev(int32_t frames, int32_t rings, int32_t steps, const uint8_t* mask, int32_t radius,
                          uint8_t* out, void* workspace, size_t workspace_bytes, void* stream) {
  if (int e = check_eval(frames, rings, steps, radius, workspace, workspace_bytes)) return e;
  if (frames == 0) return LSEG_OK;
  if (!mask || !out) return fail(LSEG_EINVAL, "NULL buffer");
  return eval_dilate(frames, rings, steps, mask, radius, out, workspace, (cudaStream_t)stream);
}


// ---------------------------------------------------------------- simulator (F3)
static int check_prims(const double* prims, int32_t n_prims) {
  if (n_prims < 0) return fail(LSEG_EINVAL, "n_prims must be >= 0");
  if (n_prims > 0 && !prims) return fail(LSEG_EINVAL, "prims is NULL");
  return LSEG_OK;
}

int lseg_cast_grid(const lseg_sensor* sensor, int32_t frames, const double* prims, int32_t n_prims,
                   const double* poses, double* t_out, int32_t* ids_out, void* stream) {
  if (!sensor || !sensor->cos_el || !sensor->sin_el || !sensor->cos_az || !sensor->sin_az)
    return fail(LSEG_EINVAL, "sensor angle tables must be device pointers");
  if (frames < 0 || sensor->rings < 1 || sensor->steps < 1) return fail(LSEG_EINVAL, "bad shape");
  if (int e = check_prims(prims, n_prims)) return e;
  if (frames == 0) return LSEG_OK;
  if (!t_out || !ids_out) return fail(LSEG_EINVAL, "NULL buffer");
  launch_cast_grid(*sensor, frames, prims, n_prims, poses, t_out, ids_out, (cudaStream_t)stream);
  return check_launch("cast_grid");
}

int lseg_cast_rays(const double* prims, int32_t n_prims, int64_t n_rays, const double* origins, const double* dirs,
                   double* t_out, int32_t* ids_out, void* stream) {
  if (n_rays < 0) return fail(LSEG_EINVAL, "n_rays must be >= 0");
  if (int e = check_prims(prims, n_prims)) return e;
  if (n_rays == 0) return LSEG_OK;
  if (!origins || !dirs || !t_out || !ids_out) return fail(LSEG_EINVAL, "NULL buffer");
  launch_cast_rays(prims, n_prims, n_rays, origins, dirs, t_out, ids_out, (cudaStream_t)stream);
  return check_launch("cast_rays");
}

int lseg_apply_scan(int64_t n_cells, double r_min, double r_max, const double* t, const int32_t* ids,
                    const double* noise, double* ranges, int32_t* labels, void* stream) {
  if (n_cells < 0) return fail(LSEG_EINVAL, "n_cells must be >= 0");
  if (n_cells == 0) return LSEG_OK;
  if (!t || !ids || !ranges || !labels) return fail(LSEG_EINVAL, "NULL buffer");
  launch_apply_scan(n_cells, r_min, r_max, t, ids, noise, ranges, labels, (cudaStream_t)stream);
  return check_launch("apply_scan");
}

int lseg_scene_normals(const lseg_sensor* sensor, const double* prims, int32_t n_prims, const double* ranges,
                       const int32_t* labels, double* normals, void* stream) {
  if (!sensor || !sensor->cos_el || !sensor->sin_el || !sensor->cos_az || !sensor->sin_az)
    return fail(LSEG_EINVAL, "sensor angle tables must be device pointers");
  if (int e = check_prims(prims, n_prims)) return e;
  if (!ranges || !labels || !normals) return fail(LSEG_EINVAL, "NULL buffer");
  launch_scene_normals(*sensor, prims, n_prims, ranges, labels, normals, (cudaStream_t)stream);
  return check_launch("scene_normals");
}

}  // extern "C"
