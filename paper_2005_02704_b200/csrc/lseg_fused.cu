// Fused pipeline kernels (sm_100a): the batched hot path of lseg_run_pipeline
// (DESIGN.md §4 has the table with bytes and bounds).  Per batch, in order:
//
//   k_ring_bounds, k_bin_rows  per (frame, ring): the ring's points binned
//              into a shared-memory row (smallest range wins), row + valid bits
//              written once; non-ring-major frames are flagged
//   k_bin_finish   per frame: generic re-binning of flagged frames, then the
//              valid-bit prefix -> node numbering
//   k_tile / k_tile_cert  per 16 x 64 tile: halo staging, normals (exact fp64,
//              or certified fp32 with exact fallback), mesh outputs, pass
//              masks of the internal edges, border normals for k_merge
//   k_tile_cc  per tile: components of the pass masks (lock-free union-find
//              over horizontal runs in shared memory) -> parent = tile-local root
//   k_merge(_cert, _exact)  global union-find over tile-border edges only
//   k_labels_backfill  per ring row: tile-local roots chased to the final
//              roots (root bits, label count), labels (root cell + 1),
//              nearest-donor backfill, label histogram (slots zeroed by
//              k_tile_cc).  With the segment() output requested, k_root_flatten
//              + the root-rank scan run first instead.
//   k_prune_rows  per ring row: surviving roots (published per row), row
//              bases from the earlier rows, compacted final ids (reference
//              segment.py:127-160)
#include <cub/block/block_scan.cuh>
#include <cuda_fp16.h>
#include <stdio.h>
#include <stdlib.h>

#include "lseg_internal.cuh"
#include "lseg_kernels.cuh"

namespace lseg {

#ifndef LSEG_PHASES
#define LSEG_PHASES 0
#endif
#if LSEG_PHASES
__device__ unsigned long long g_ph[8];
#endif
#ifndef LSEG_UNR
#define LSEG_UNR 1
#endif
static constexpr int kUnrollNormals = LSEG_UNR;
#ifndef LSEG_FAST_MATH
#define LSEG_FAST_MATH 1
#endif
static constexpr bool kFastMath = LSEG_FAST_MATH;
#ifndef LSEG_BIN_B
#define LSEG_BIN_B 2  // points per thread in flight in k_bin_rows (4: register spills, -5 %)
#endif
#ifndef LSEG_BIN_MINB
#define LSEG_BIN_MINB 8
#endif
#ifndef LSEG_CC_TBIG
#define LSEG_CC_TBIG 128
#endif
#ifndef LSEG_FOLD_FLATTEN
#define LSEG_FOLD_FLATTEN 1
#endif
// loads in flight per thread in the row kernels (measured: labels 2, pruning 16)
#ifndef LSEG_PF_LAB
#define LSEG_PF_LAB 2
#endif
#ifndef LSEG_PF_PRUNE
#define LSEG_PF_PRUNE 16
#endif
// resident threads per SM the row kernels are compiled for (2048: 32 registers)
#ifndef LSEG_CC_TSM
#define LSEG_CC_TSM 2048
#endif
#ifndef LSEG_MERGE_PER
#define LSEG_MERGE_PER 2  // border cells per merge thread in large batches (grid-stride; measured 1: 0.181, 2: 0.171, 4: 0.179 ms)
#endif
#ifndef LSEG_MERGE_T
#define LSEG_MERGE_T 128
#endif
#ifndef LSEG_LAB_T
#define LSEG_LAB_T 128  // labels threads per row in large batches
#endif
#ifndef LSEG_LAB_TSM
#define LSEG_LAB_TSM 1280  // measured: 0.356 ms vs 0.367 at 2048, 0.405 at 1024
#endif
#ifndef LSEG_PRUNE_TSM
#define LSEG_PRUNE_TSM 2048
#endif
#ifndef LSEG_CERT_MINB
#define LSEG_CERT_MINB 4
#endif
static constexpr int TILE_R = kTileR;
static constexpr int TILE_C = kTileC;
#ifndef LSEG_TILE_T
#define LSEG_TILE_T 256
#endif
static constexpr int TILE_T = LSEG_TILE_T;

__device__ __forceinline__ int wrapc(int c, int Sk) { return c < 0 ? c + Sk : (c >= Sk ? c - Sk : c); }

__device__ __forceinline__ int id_at(const uint32_t* vbf, const int32_t* wpf, int Wk, int r, int c) {
  return node_id_at(vbf + (int64_t)r * Wk, wpf + (int64_t)r * Wk, c);
}

// Is the forward edge (r, c) -> slot s internal to the (TR x TC) tile that
// owns (r, c)?  Shared by k_tile (local unions) and k_merge (the rest).
template <int TR, int TC>
__device__ __forceinline__ bool edge_internal(int r, int c, int s, int Sk) {
  const int tr = r + slot_dr(s);
  int tc = c + slot_dc(s);
  if (tc >= Sk) tc -= Sk;
  return (tr / TR == r / TR) && (tc / TC == c / TC);
}

// Border-normal store of one frame: for each tile row, its first and last
// ring rows (all S' columns), then for each tile column its first and last
// columns (all R rows); 3 doubles per cell, so every write run is contiguous.
__device__ __forceinline__ int64_t bn_frame(const Shape& sh, int TR, int TC) {
  return ((int64_t)2 * ((sh.R + TR - 1) / TR) * sh.Sk + (int64_t)2 * ((sh.Sk + TC - 1) / TC) * sh.R) * 3;
}
// (offsets within one frame's store fit 32 bits: 6 (R/TR + S'/TC) doubles per cell row / column)
__device__ __forceinline__ int bn_row(const Shape& sh, int slot, int c) { return (slot * sh.Sk + c) * 3; }
__device__ __forceinline__ int bn_col(const Shape& sh, int TR, int slot, int r) {
  return (2 * ((sh.R + TR - 1) / TR) * sh.Sk + slot * sh.R + r) * 3;
}
__device__ __forceinline__ void bn_put(double* o, double a, double b, double c) { o[0] = a; o[1] = b; o[2] = c; }

// One CTA per (frame, TR x TC tile of kept cells).
//   A  ranges + node ids of the tile and a 1-cell halo into shared memory
//   B  fp64 normals of the tile's nodes (shared memory)
//   C  neighbours / normals / mask out; fp64 normals of the tile's border
//      cells to `bnorm` for k_merge
//   D  homogeneity test + shared-memory union-find on internal forward edges
//   E  parent[cell] = tile-local root cell (-1 for cells without a normal)
template <int TR, int TC, int T>
#ifndef LSEG_TILE_MINB
#define LSEG_TILE_MINB 4
#endif
__global__ void __launch_bounds__(T, LSEG_TILE_MINB) k_tile(lseg_sensor sn, Shape sh, const double* __restrict__ ranges,
                                                const uint32_t* __restrict__ vbits, const int32_t* __restrict__ wpre,
                                                double t0, double t1, double t2, int32_t* __restrict__ node_ids,
                                                int32_t* __restrict__ neighbors, float* __restrict__ n32,
                                                uint8_t* __restrict__ nmask, unsigned long long* __restrict__ masks,
                                                double* __restrict__ bnorm, int32_t* __restrict__ parent,
                                                uint32_t* __restrict__ lroots, int32_t* __restrict__ n_labels,
                                                double* __restrict__ n64, int32_t* __restrict__ node_rc) {
  pdl_trigger();
  pdl_wait();
  constexpr int GR = TR + 2, GC = TC + 2;  // halo rows r0-1..r0+TR, cols c0-1..c0+TC
  constexpr int NT = TR * TC;
#if LSEG_PHASES
  long long ph_prev = clock64();
#define PH_MARK(i)                                                   \
  do {                                                               \
    if (threadIdx.x == 0) {                                          \
      const long long now = clock64();                               \
      atomicAdd(&g_ph[i], (unsigned long long)(now - ph_prev));       \
      ph_prev = now;                                                 \
    }                                                                \
  } while (0)
#else
#define PH_MARK(i) do {} while (0)
#endif
  // dynamic shared memory (58 KB > the 48 KB static limit), see tile_smem_bytes()
  extern __shared__ __align__(16) unsigned char s_dyn[];
  // ranges + separable direction tables; positions are rebuilt on use
  // (5 multiplies) -- 19 KB less shared memory buys a 4th CTA per SM
  double* s_r = reinterpret_cast<double*>(s_dyn);
  double2* s_el = reinterpret_cast<double2*>(s_r + GR * GC);  // (cos, sin)(elev) per halo row
  double2* s_az = s_el + GR;                                  // (cos, sin)(az) per halo column
  double* s_nend = reinterpret_cast<double*>(s_az + GC);
  // position of halo cell (row yy, column xx): one 16-B load per table
  auto posyx = [&](int yy, int xx) -> Vec3 {
    const double2 el = s_el[yy], az = s_az[xx];
    const double r = s_r[yy * GC + xx];
    Vec3 q;
    q.x = __dmul_rn(__dmul_rn(el.x, az.x), r);
    q.y = __dmul_rn(__dmul_rn(el.x, az.y), r);
    q.z = __dmul_rn(el.y, r);
    return q;
  };
  // tile normals: (x, y) as one 16-B element, z apart
  double2* s_nxy = reinterpret_cast<double2*>(s_nend);
  double* s_nz = reinterpret_cast<double*>(s_nxy + NT);
  auto nput = [&](int e, double x, double y, double z) { s_nxy[e] = make_double2(x, y); s_nz[e] = z; };
  auto nget = [&](int e) -> Vec3 { const double2 v = s_nxy[e]; Vec3 q; q.x = v.x; q.y = v.y; q.z = s_nz[e]; return q; };
  int* s_id = reinterpret_cast<int*>(s_nz + NT);
  unsigned short* s_list = reinterpret_cast<unsigned short*>(s_id + GR * GC);  // fan6 list from the front, rest from the back
  uint8_t* s_has = reinterpret_cast<uint8_t*>(s_list + NT);
  uint8_t* s_m = s_has + NT;  // presence mask of general-path nodes

  const int tilesC = (sh.Sk + TC - 1) / TC;
  const int tilesR = (sh.R + TR - 1) / TR;
  // grid (tile column, tile row, frame): per-CTA values straight from the
  // block index (uniform registers, no division)
  const int f = blockIdx.z;
  const int rem = blockIdx.y * tilesC + blockIdx.x;  // tile within the frame
  const int64_t b = (int64_t)f * tilesR * tilesC + rem;
  const int r0 = blockIdx.y * TR, c0 = blockIdx.x * TC;
  const int TRe = min(TR, sh.R - r0), TCe = min(TC, sh.Sk - c0);
  const double* rf = ranges + (int64_t)f * sh.R * sh.S;
  const uint32_t* vbf = vbits + (int64_t)f * sh.R * sh.Wk;
  const int32_t* wpf = wpre + (int64_t)f * sh.R * sh.Wk;
  const int64_t nbase = (int64_t)f * sh.cap;
  const int tid = threadIdx.x;
  if (rem == 0 && tid == 0) n_labels[f] = 0;  // counted by k_labels_backfill (or k_root_flatten)

  // A. halo positions dir*r (reference product order) and node ids (-1 absent).
  // All of a thread's loads are issued before any is used (one memory round
  // trip for the whole halo instead of one per cell).
  // row-structured: thread (column xi, row group g) loads rows g, g + NG, ...
  // of tile column xi (per-thread column offsets, one row pointer per row),
  // then threads 0 .. 2 GR - 1 load the two halo columns
  {
    static_assert(T % TC == 0, "whole row groups");
    constexpr int NG = T / TC, NRA = (GR + NG - 1) / NG;
    const int xi = tid % TC, g = tid / TC;
    const bool colok = xi < TCe;
    const int cc = c0 + (colok ? xi : 0);
    const int64_t coff = (int64_t)cc * sh.k;
    const int wo = cc >> 5;
    const uint32_t bit = 1u << (cc & 31);
    double rv[NRA];
    uint32_t wv[NRA];
    int32_t pv[NRA];
    // frame bases opaque to the optimiser (phase-local copies): 32-bit
    // frame-local offsets, one wide multiply-add per load
    const double* rfa = rf;
    const uint32_t* vba = vbf;
    const int32_t* wpa = wpf;
    asm volatile("" : "+l"(rfa), "+l"(vba), "+l"(wpa));
#pragma unroll
    for (int j = 0; j < NRA; ++j) {
      const int y = g + NG * j, rr = r0 - 1 + y;
      rv[j] = 0.0;
      wv[j] = 0u;
      pv[j] = 0;
      if (y < GR && colok && rr >= 0 && rr < sh.R) {
        rv[j] = __ldg(rfa + (rr * sh.S + (int)coff));
        wv[j] = __ldg(vba + (rr * sh.Wk + wo));
        pv[j] = __ldg(wpa + (rr * sh.Wk + wo));
      }
    }
    // halo columns: halo index 0 = column c0 - 1, index TCe + 1 = column
    // c0 + TCe (both cyclic)
    const bool hthr = tid < 2 * GR;
    const int hy = tid >> 1, hside = tid & 1, hrr = r0 - 1 + hy;
    const int hcol = hside ? (c0 + TCe == sh.Sk ? 0 : c0 + TCe) : (c0 == 0 ? sh.Sk - 1 : c0 - 1);
    double hr = 0.0;
    uint32_t hw = 0u;
    int32_t hp = 0;
    if (hthr && hrr >= 0 && hrr < sh.R) {
      hr = __ldg(rf + (int64_t)hrr * sh.S + (int64_t)hcol * sh.k);
      hw = __ldg(vbf + (int64_t)hrr * sh.Wk + (hcol >> 5));
      hp = __ldg(wpf + (int64_t)hrr * sh.Wk + (hcol >> 5));
    }
#pragma unroll
    for (int j = 0; j < NRA; ++j) {
      const int y = g + NG * j;
      if (y < GR && colok) {
        const int id = (wv[j] & bit) ? pv[j] + __popc(wv[j] & (bit - 1u)) : -1;
        const int e = y * GC + xi + 1;
        s_r[e] = id >= 0 ? rv[j] : 0.0;
        s_id[e] = id;
      }
    }
    if (hthr) {
      const uint32_t hb = 1u << (hcol & 31);
      const int id = (hw & hb) ? hp + __popc(hw & (hb - 1u)) : -1;
      const int e = hy * GC + (hside ? TCe + 1 : 0);
      s_r[e] = id >= 0 ? hr : 0.0;
      s_id[e] = id;
    }
    for (int e = tid; e < GR + GC; e += T) {
      if (e < GR) {
        const int rr = min(max(r0 - 1 + e, 0), sh.R - 1);
        s_el[e] = make_double2(__ldg(sn.cos_el + rr), __ldg(sn.sin_el + rr));
      } else {
        int c = (c0 - 1 + (e - GR)) % sh.Sk;
        if (c < 0) c += sh.Sk;
        s_az[e - GR] = make_double2(__ldg(sn.cos_az + (int64_t)c * sh.k), __ldg(sn.sin_az + (int64_t)c * sh.k));
      }
    }
  }
  __syncthreads();
  PH_MARK(1);

  // B. fp64 normals (reference normals.py:94-145 operation order).  Nodes are
  // first sorted into two work lists so that no warp runs both code paths:
  // nodes with all 6 slots (the common case) take the straight-line fan6,
  // the rest the streaming Fan over their present slots.
  __shared__ int s_cnt[2 * (T / 32) + 2];
  {
    const int lane = tid & 31, warp = tid >> 5;
    unsigned char ml[(NT + T - 1) / T];
    int kind[(NT + T - 1) / T];  // 0 none, 1 fan6, 2 general
    int na = 0, nb = 0;
#pragma unroll
    for (int j = 0; j < (NT + T - 1) / T; ++j) {
      const int e = tid + j * T;
      const int y = e / TC, x = e - y * TC;
      const int g = (y + 1) * GC + (x + 1);
      unsigned m = 0;
      kind[j] = 0;
      if (e < NT && y < TRe && x < TCe) {
        // the mesh outputs (node ids, neighbours, node cells) need no
        // normal: written here, while the neighbour ids are at hand
        const int id = s_id[g];
        if (node_ids) node_ids[nbase + (int64_t)(r0 + y) * sh.Sk + c0 + x] = id;
        if (id >= 0) {
          int nb[6];
#pragma unroll
          for (int s = 0; s < 6; ++s) {
            nb[s] = (s == 5 && sh.Sk == 2) ? -1 : s_id[g + slot_dr(s) * GC + slot_dc(s)];  // mesh.py:96-101
            if (nb[s] >= 0) m |= 1u << s;
          }
          kind[j] = (m == 0x3fu) ? 1 : 2;
          int2* o2 = reinterpret_cast<int2*>(neighbors + (nbase + id) * 6);  // 24 B rows, 8-B aligned
          o2[0] = make_int2(nb[0], nb[1]);
          o2[1] = make_int2(nb[2], nb[3]);
          o2[2] = make_int2(nb[4], nb[5]);
          if (node_rc) {  // the single-scan Mesh's node_rings / node_steps (mesh.py:115-117)
            node_rc[(nbase + id) * 2] = r0 + y;
            node_rc[(nbase + id) * 2 + 1] = (c0 + x) * sh.k;
          }
        }
      }
      ml[j] = (unsigned char)m;
      na += kind[j] == 1;
      nb += kind[j] == 2;
      if (e < NT) { s_has[e] = 0; nput(e, 0.0, 0.0, 0.0); }
    }
    // block-wide exclusive offsets of (na, nb): warp scan + per-warp totals
    int ia = na, ib = nb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ta = __shfl_up_sync(0xffffffffu, ia, o), tb = __shfl_up_sync(0xffffffffu, ib, o);
      if (lane >= o) { ia += ta; ib += tb; }
    }
    if (lane == 31) { s_cnt[warp] = ia; s_cnt[T / 32 + warp] = ib; }
    __syncthreads();
    int oa = 0, ob = 0, ta = 0, tb = 0;
    for (int w = 0; w < T / 32; ++w) {
      if (w < warp) { oa += s_cnt[w]; ob += s_cnt[T / 32 + w]; }
      ta += s_cnt[w];
      tb += s_cnt[T / 32 + w];
    }
    oa += ia - na;
    ob += ib - nb;
#pragma unroll
    for (int j = 0; j < (NT + T - 1) / T; ++j) {
      const int e = tid + j * T;
      if (kind[j] == 1) s_list[oa++] = (unsigned short)e;
      else if (kind[j] == 2) { s_list[NT - 1 - ob] = (unsigned short)e; s_m[e] = ml[j]; ++ob; }
    }
    if (tid == 0) { s_cnt[2 * (T / 32)] = ta; s_cnt[2 * (T / 32) + 1] = tb; }
  }
  __syncthreads();
  PH_MARK(2);
  const int nfan6 = s_cnt[2 * (T / 32)], ngen = s_cnt[2 * (T / 32) + 1];
#pragma unroll kUnrollNormals
  for (int i = tid; i < nfan6; i += T) {
    const int e = s_list[i];
    const int y = e / TC, x = e - y * TC;
    const Vec3 p = posyx(y + 1, x + 1);
    double nv[3];
    // streamed: only first / previous / current vectors live (fewer registers,
    // more resident warps)
    FanT<kFastMath> fan;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const Vec3 q = posyx(y + 1 + slot_dr(s), x + 1 + slot_dc(s));
      fan.add(__dsub_rn(q.x, p.x), __dsub_rn(q.y, p.y), __dsub_rn(q.z, p.z));
    }
    const bool okn = fan.finish(p, nv);
    if (okn) {
      nput(e, nv[0], nv[1], nv[2]);
      s_has[e] = 1;
    }
  }
  // the general nodes start at the first warp after the last fan6 node's
  // warp, i.e. on the warps with one fan6 node fewer per lane
  const int gstart = (((nfan6 % T) + 31) & ~31) % T;
  for (int i = (tid - gstart + T) % T; i < ngen; i += T) {
    const int e = s_list[NT - 1 - i];
    const int y = e / TC, x = e - y * TC;
    const unsigned m = s_m[e];
    const Vec3 p = posyx(y + 1, x + 1);
    double nv[3];
    // straight-line six-slot sequence with absent slots substituted
    // (fan_subst): slot s -> (row, column) offsets from packed tables
    // (dr + 1, dc + 1 in 2-bit fields)
    auto pos = [&](int sl) -> Vec3 {
      const int dr = (int)((0x41Au >> (2 * sl)) & 3u) - 1, dc = (int)((0x069u >> (2 * sl)) & 3u) - 1;
      return posyx(y + 1 + dr, x + 1 + dc);
    };
    if (fan_subst<kFastMath>(p, m, pos, nv)) {
      nput(e, nv[0], nv[1], nv[2]);
      s_has[e] = 1;
    }
  }
  __syncthreads();
  PH_MARK(3);

  // C. per-node normal outputs (phase-local opaque frame bases: 32-bit node
  // ids, one wide multiply-add per store)
  {
    float* n32f = n32 ? n32 + nbase * 3 : nullptr;
    uint8_t* nmf = nmask + nbase;
    asm volatile("" : "+l"(n32f), "+l"(nmf));
#pragma unroll
    for (int j = 0; j < (NT + T - 1) / T; ++j) {
      const int e = tid + j * T;
      const int y = e / TC, x = e - y * TC;
      if (e >= NT || y >= TRe || x >= TCe) continue;
      const int id = s_id[(y + 1) * GC + (x + 1)];
      if (id < 0) continue;  // (mesh outputs: written by the classification)
      const bool has = s_has[e];
      const Vec3 nv = nget(e);
      if (n32f) {
        float* o = n32f + id * 3;
        const float qn = __int_as_float(0x7fc00000);
        o[0] = has ? (float)nv.x : qn;
        o[1] = has ? (float)nv.y : qn;
        o[2] = has ? (float)nv.z : qn;
      }
      if (n64) {  // fp64 normals (the single-scan drop-in: reference NormalMap values)
        double* o = n64 + (nbase + id) * 3;
        const double qn = __longlong_as_double(0x7ff8000000000000LL);
        o[0] = has ? nv.x : qn;
        o[1] = has ? nv.y : qn;
        o[2] = has ? nv.z : qn;
      }
      nmf[id] = has ? 1 : 0;
    }
  }
  // fp64 normals of the tile's border rows / columns for k_merge: only the
  // 2 TC + 2 TR border cells, one thread each (row stores coalesced)
  {
    double* bf = bnorm + (int64_t)f * bn_frame(sh, TR, TC);
    const int tr = r0 / TR, tc = c0 / TC;
    for (int u = tid; u < 2 * TC + 2 * TR; u += T) {
      int y, x, slot;
      bool rowside;
      if (u < 2 * TC) {
        rowside = true;
        slot = u / TC;
        x = u - slot * TC;
        y = slot ? TRe - 1 : 0;
      } else {
        rowside = false;
        slot = (u - 2 * TC) / TR;
        y = u - 2 * TC - slot * TR;
        x = slot ? TCe - 1 : 0;
      }
      if (y >= TRe || x >= TCe) continue;
      const int e = y * TC + x;
      if (!s_has[e]) continue;
      double* o = rowside ? bf + bn_row(sh, 2 * tr + slot, c0 + x) : bf + bn_col(sh, TR, 2 * tc + slot, r0 + y);
      const Vec3 nv = nget(e);
      bn_put(o, nv.x, nv.y, nv.z);
    }
  }

#if LSEG_PHASES
  __syncthreads();
#endif
  PH_MARK(4);
  // D. homogeneity test on the tile's internal forward edges, one warp per
  // tile row, as 64-bit masks per row (bit x = column x):
  //   H  (y,x)->(y,x+1)   V0 (y,x)->(y+1,x)   V1 (y,x)->(y+1,x+1)
  //   HAS  node with a normal;  W bit0/bit1 = column-wrap right / diagonal edge
  //   of x = S'-1 in a full-width tile (S' <= TC).
  // k_tile_cc turns them into tile-local components.
  static_assert(TC == 64, "row masks assume 64-column tiles");
  const int lane = tid & 31;
  const bool full_width = (c0 == 0 && TCe == sh.Sk);
  unsigned long long* mrow = masks + (((int64_t)f * tilesR + r0 / TR) * tilesC + c0 / TC) * (TR * 5);
  static_assert(TR % (T / 32) == 0, "whole rows per warp");
#pragma unroll
  for (int yy = 0; yy < TR / (T / 32); ++yy) {
    const int y = (tid >> 5) + yy * (T / 32);
    uint32_t H[2], V0[2], V1[2], HS[2];  // 32-bit halves of the row masks
    bool w0 = false, w1 = false;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int x = lane + 32 * half;
      const int e = y * TC + x;
      bool h = false, v0 = false, v1 = false;
      const bool has = (y < TRe) && s_has[e];
      // branch-free: every test runs (an absent partner reads the node's own
      // normal, a test that is then masked off), no short-circuit
      {
        const bool ph = has && x + 1 < TCe && s_has[e + 1];
        const bool pv0 = has && y + 1 < TRe && s_has[e + TC];
        const bool pv1 = has && y + 1 < TRe && x + 1 < TCe && s_has[e + TC + 1];
        const Vec3 a = nget(e);
        auto pass = [&](int q) -> bool {
          const Vec3 b = nget(q);
          const bool c0 = fabs(__dsub_rn(b.x, a.x)) < t0;
          const bool c1 = fabs(__dsub_rn(b.y, a.y)) < t1;
          const bool c2 = fabs(__dsub_rn(b.z, a.z)) < t2;
          return c0 & c1 & c2;
        };
        h = ph & pass(ph ? e + 1 : e);
        v0 = pv0 & pass(pv0 ? e + TC : e);
        v1 = pv1 & pass(pv1 ? e + TC + 1 : e);
      }
      if (has && full_width && x == TCe - 1) {  // the column wrap of a full-width tile (rare)
        const Vec3 av = nget(e);
        const double a[3] = {av.x, av.y, av.z};
        if (full_width && x == TCe - 1) {
          const int e0 = y * TC;  // (y, 0)
          if (TCe > 1 && s_has[e0]) {
            const Vec3 qv = nget(e0);
            const double q[3] = {qv.x, qv.y, qv.z};
            w0 = normals_pass(a, q, t0, t1, t2);
          }
          if (y + 1 < TRe && s_has[e0 + TC]) {
            const Vec3 qv = nget(e0 + TC);
            const double q[3] = {qv.x, qv.y, qv.z};
            w1 = normals_pass(a, q, t0, t1, t2);
          }
        }
      }
      H[half] = __ballot_sync(0xffffffffu, h);
      V0[half] = __ballot_sync(0xffffffffu, v0);
      V1[half] = __ballot_sync(0xffffffffu, v1);
      HS[half] = __ballot_sync(0xffffffffu, has);
    }
    unsigned W = 0u;
    if (full_width)  // block-uniform: the wrap bits exist only in a full-width tile
      W = (__ballot_sync(0xffffffffu, w0) ? 1u : 0u) | (__ballot_sync(0xffffffffu, w1) ? 2u : 0u);
    if (lane == 0) {  // little-endian: the low half first
      uint2* m2 = reinterpret_cast<uint2*>(mrow + y * 5);
      m2[0] = make_uint2(H[0], H[1]);
      m2[1] = make_uint2(V0[0], V0[1]);
      m2[2] = make_uint2(V1[0], V1[1]);
      m2[3] = make_uint2(HS[0], HS[1]);
      m2[4] = make_uint2(W, 0u);
    }
  }
#if LSEG_PHASES
  __syncthreads();
#endif
  PH_MARK(5);
}

// ---------------------------------------------------------------- certified fp32 normals
// The exact fp64 normals above are bound by the FP64 pipe (~350 DP ops per
// node).  The certified variant computes each normal in fp32 from exactly
// formed edge vectors, together with a rigorous bound `err` on
// |n_fp32 - n_reference| per component; every homogeneity decision that the
// bound cannot settle (and every node whose normal is degenerate or badly
// conditioned) is redone with the exact fp64 path, so segment labels stay
// bit-identical to the reference.  Output normals (fp32) are then within the
// north-star tolerance (1e-5), not bit-identical.
//
// Error model (u = 2^-24, all fp32 ops round-to-nearest except the PTX
// approximations rcp.approx (<= 1 ulp) and rsqrt.approx (<= 2^-22.9 rel.)):
//   the edge vectors V = q - p are formed in fp64 exactly as the reference
//   forms them and rounded once to fp32: |v - V| <= u|V| (|V| >= 1e-15, else
//   the node is "degenerate" -> exact path).  Then |l - |V|| <= 6u|V|,
//   w = 1/(la+lb) within 9u, |c - A x B| <= 6u|A||B|, each term w*c within
//   15u W|A||B|, and six fma accumulations add <= 11u B, so
//   |acc - ACC| <= E = kAcc u B with B = sum W|A||B| (kAcc = 32 > 26 + slack).
//   The unit normal then deviates by <= 2E/|acc| + 5u (normalisation), and
//   err = u (2 kAcc B/|acc| + 8) bounds every component, including the
//   reference's own fp64 rounding (2^-29 smaller).
static constexpr float kU32 = 5.9604645e-08f;  // 2^-24
static constexpr float kAcc = 32.0f;
static constexpr float kOutCond = 64.0f;  // B/|acc| above this -> exact path (fp32 output accuracy)

__device__ __forceinline__ float rcp_apx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_apx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct Fan32 {
  float fx, fy, fz, fl;  // first vector and its length
  float qx, qy, qz, ql;  // previous vector
  float a0, a1, a2, ws, bs;
  int cnt;
  bool deg;

  __device__ __forceinline__ Fan32() : a0(0.f), a1(0.f), a2(0.f), ws(0.f), bs(0.f), cnt(0), deg(false) {}

  __device__ __forceinline__ void pair(float ax, float ay, float az, float la, float bx, float by, float bz,
                                       float lb) {
    const float w = rcp_apx(la + lb);
    const float c0 = fmaf(ay, bz, -(az * by));
    const float c1 = fmaf(az, bx, -(ax * bz));
    const float c2 = fmaf(ax, by, -(ay * bx));
    a0 = fmaf(w, c0, a0);
    a1 = fmaf(w, c1, a1);
    a2 = fmaf(w, c2, a2);
    ws += w;
    bs = fmaf(w, la * lb, bs);
  }

  __device__ __forceinline__ void add(float vx, float vy, float vz, float deg2) {
    const float s = fmaf(vz, vz, fmaf(vy, vy, vx * vx));
    deg |= !(s >= deg2);
    const float l = s * rsqrt_apx(s);
    if (cnt == 0) { fx = vx; fy = vy; fz = vz; fl = l; }
    else pair(qx, qy, qz, ql, vx, vy, vz, l);
    qx = vx; qy = vy; qz = vz; ql = l;
    ++cnt;
  }

  // 0: no normal (certain), 1: normal + bound, >= 2: undecided -> exact fp64
  // path (the value says why: 2 short edge vector, 3 cancelling fan, 4 |mean|
  // near 1e-12, 5 ill-conditioned, 6 orientation)
  __device__ __forceinline__ int finish(float px, float py, float pz, float n[3], float& err) {
    if (cnt < 2) return 0;
    if (cnt >= 3) pair(qx, qy, qz, ql, fx, fy, fz, fl);
    if (deg) return 2;
    const float A2 = fmaf(a2, a2, fmaf(a1, a1, a0 * a0));
    const float inv = rsqrt_apx(A2);
    const float alen = A2 * inv;
    const float E = kAcc * kU32 * bs;
    if (!(alen > 2.0f * E)) return 3;                 // cancelling fan (or underflow)
    if (alen - E < 1.0001e-12f * ws) return 4;        // |mean| >= 1e-12 undecided (normals.py:138)
    if (bs > kOutCond * alen) return 5;               // ill-conditioned: exact output
    err = kU32 * (2.0f * kAcc * bs * rcp_apx(alen) + 8.0f) * 1.01f;
    float n0 = a0 * inv, n1 = a1 * inv, n2 = a2 * inv;
    const float dot = fmaf(n2, pz, fmaf(n1, py, n0 * px));
    const float pm = fabsf(px) + fabsf(py) + fabsf(pz);
    if (fabsf(dot) <= pm * (err + 8.0f * kU32)) return 6;  // orientation undecided (normals.py:142-143)
    if (dot > 0.0f) { n0 = -n0; n1 = -n1; n2 = -n2; }
    n[0] = n0; n[1] = n1; n[2] = n2;
    return 1;
  }
};

// Exact reference normal of kept cell (r, c) of one frame, straight from the
// range grid and valid bits in global memory (the same operation sequence as
// the fp64 tile path).  Used for the rare nodes / edges the fp32 bound cannot
// settle.
__device__ __noinline__ bool exact_normal_at(const lseg_sensor& sn, const Shape& sh, const double* __restrict__ rf,
                                             const uint32_t* __restrict__ vbf, int r, int c, double out[3]) {
  const Vec3 p = cell_pos(sn, r, c * sh.k, __ldg(rf + (int64_t)r * sh.S + (int64_t)c * sh.k));
  FanT<kFastMath> fan;
#pragma unroll 1
  for (int s = 0; s < 6; ++s) {
    const int rr = r + slot_dr(s);
    if (rr < 0 || rr >= sh.R) continue;
    if (s == 5 && sh.Sk == 2) continue;  // mesh.py:96-101
    const int cc = wrapc(c + slot_dc(s), sh.Sk);
    if (!((__ldg(vbf + (int64_t)rr * sh.Wk + (cc >> 5)) >> (cc & 31)) & 1u)) continue;
    const Vec3 q = cell_pos(sn, rr, cc * sh.k, __ldg(rf + (int64_t)rr * sh.S + (int64_t)cc * sh.k));
    fan.add(__dsub_rn(q.x, p.x), __dsub_rn(q.y, p.y), __dsub_rn(q.z, p.z));
  }
  return fan.finish(p, out);
}

struct CertParams {
  double t[3];   // thresholds (fp64, for the exact decisions)
  float tf[3];   // thresholds rounded to fp32
  float mt[3];   // per-component decision slack: rounding of T and of the fp32 difference
  float deg2;    // shorter squared edge vectors take the exact path
};

// Homogeneity decision from certified normals: 1 pass, 0 fail, 2 undecided.
__device__ __forceinline__ int cert_pass(const CertParams& cp, float ax, float ay, float az, float ea, float bx,
                                         float by, float bz, float eb) {
  const float m = ea + eb;
  const float d0 = fabsf(ax - bx), d1 = fabsf(ay - by), d2 = fabsf(az - bz);
  const float m0 = m + cp.mt[0], m1 = m + cp.mt[1], m2 = m + cp.mt[2];
  if (d0 - m0 >= cp.tf[0] || d1 - m1 >= cp.tf[1] || d2 - m2 >= cp.tf[2]) return 0;
  if (d0 + m0 < cp.tf[0] && d1 + m1 < cp.tf[1] && d2 + m2 < cp.tf[2]) return 1;
  return 2;
}

// Border-normal store of the certified path: one float4 {n, err} per cell,
// same slot layout as bn_row / bn_col.
__device__ __forceinline__ int64_t bn4_frame(const Shape& sh, int TR, int TC) {
  return (int64_t)2 * ((sh.R + TR - 1) / TR) * sh.Sk + (int64_t)2 * ((sh.Sk + TC - 1) / TC) * sh.R;
}
__device__ __forceinline__ int64_t bn4_row(const Shape& sh, int slot, int c) { return (int64_t)slot * sh.Sk + c; }
__device__ __forceinline__ int64_t bn4_col(const Shape& sh, int TR, int slot, int r) {
  return (int64_t)2 * ((sh.R + TR - 1) / TR) * sh.Sk + (int64_t)slot * sh.R + r;
}

// One CTA per (frame, TR x TC tile), certified normals.  Phases (4 barriers
// when nothing needs the exact path):
//   A  halo positions (fp64, reference product order) + node ids in smem,
//      then per halo row a presence bitmask (slot masks by bit arithmetic)
//   L  work lists: all-six-slot nodes / the rest (warp-aggregated atomics)
//   B  fp32 normals + bounds from the exactly formed fp64 edge vectors;
//      uncertified nodes are listed for X0
//   X0 exact fp64 normals of the uncertified nodes (lane-dense, from smem)
//   D  per row: edge decisions (certain pass / fail / undecided) and the
//      per-node outputs; undecided edges list their endpoints for X1
//   X1 + D2 (rare): exact normals of those endpoints, undecided edges settled
// Exact fp64 normals also go to the global scratch `xn` (read back by D2).
template <int TR, int TC, int T>
__global__ void __launch_bounds__(T, LSEG_CERT_MINB) k_tile_cert(
    lseg_sensor sn, Shape sh, const double* __restrict__ ranges, const uint32_t* __restrict__ vbits,
    const int32_t* __restrict__ wpre, CertParams cp, int32_t* __restrict__ node_ids, int32_t* __restrict__ neighbors,
    float* __restrict__ n32, uint8_t* __restrict__ nmask, unsigned long long* __restrict__ masks,
    float4* __restrict__ bn4, double* __restrict__ xn, float* __restrict__ dbg_err, int32_t* __restrict__ fscal,
    int32_t* __restrict__ n_labels) {
  pdl_trigger();
  pdl_wait();
  constexpr int GR = TR + 2, GC = TC + 2, NH = GR * GC;
  constexpr int NT = TR * TC;
  static_assert(TC == 64, "row masks assume 64-column tiles");
  extern __shared__ __align__(16) unsigned char s_dyn[];
  double* s_px = reinterpret_cast<double*>(s_dyn);
  double* s_py = s_px + NH;
  double* s_pz = s_py + NH;
  float* s_nx = reinterpret_cast<float*>(s_pz + NH);
  auto posg = [&](int gi) -> Vec3 { return Vec3{s_px[gi], s_py[gi], s_pz[gi]}; };
  float* s_ny = s_nx + NT;
  float* s_nz = s_ny + NT;
  __half* s_eh = reinterpret_cast<__half*>(s_nz + NT);  // err / u, rounded up (<= 64 kAcc + 8 < 65504)
  int* s_id = reinterpret_cast<int*>(s_eh + NT);
  unsigned short* s_list = reinterpret_cast<unsigned short*>(s_id + NH);  // fan6 from the front, rest from the back
  unsigned short* s_xl = s_list + NT;                                     // exact-path list (X0, then X1)
  uint8_t* s_has = reinterpret_cast<uint8_t*>(s_xl + NT);  // 0 none, 1 normal, 2 uncertified
  uint8_t* s_m = s_has + NT;                                // slot mask
  uint8_t* s_req = s_m + NT;                                // exact path: 1 edge request, >= 2 reason
  __shared__ unsigned long long s_hm[GR];                   // presence of halo columns 1..64 per halo row
  __shared__ unsigned s_he[GR];                             // bit 0: halo column 0, bit 1: column 65
  __shared__ unsigned long long s_U[TR * 3];
  __shared__ unsigned s_UW[TR];
  __shared__ int s_cnt[5];  // fan6, general, X0, X1 list sizes; undecided edges

  const int tilesC = (sh.Sk + TC - 1) / TC;
  const int tilesR = (sh.R + TR - 1) / TR;
  // grid (tile column, tile row, frame): per-CTA values straight from the
  // block index (uniform registers, no division)
  const int f = blockIdx.z;
  const int rem = blockIdx.y * tilesC + blockIdx.x;  // tile within the frame
  const int64_t b = (int64_t)f * tilesR * tilesC + rem;
  const int r0 = blockIdx.y * TR, c0 = blockIdx.x * TC;
  const int TRe = min(TR, sh.R - r0), TCe = min(TC, sh.Sk - c0);
  const double* rf = ranges + (int64_t)f * sh.R * sh.S;
  const uint32_t* vbf = vbits + (int64_t)f * sh.R * sh.Wk;
  const int32_t* wpf = wpre + (int64_t)f * sh.R * sh.Wk;
  const int64_t nbase = (int64_t)f * sh.cap;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
#if LSEG_PHASES
  long long ph_prev = clock64();
#endif
  if (tid < 5) s_cnt[tid] = 0;
  if (rem == 0 && tid == 0) {
    fscal[f * 4 + 2] = 0;  // k_merge_cert's undecided-edge counter
    n_labels[f] = 0;       // counted by k_labels_backfill (or k_root_flatten)
  }

  // A. halo positions dir*r (reference product order) and node ids
  {
    constexpr int NA = (NH + T - 1) / T;
    double rv[NA];
    uint32_t wv[NA];
    int32_t pv[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) {
      const int e = tid + j * T;
      const int y = e / GC, x = e - y * GC;
      const int rr = r0 - 1 + y;
      rv[j] = 0.0;
      wv[j] = 0u;
      pv[j] = 0;
      if (e < NH && rr >= 0 && rr < sh.R) {
        const int cc = wrapc(c0 - 1 + x, sh.Sk);
        rv[j] = __ldg(rf + (int64_t)rr * sh.S + (int64_t)cc * sh.k);
        wv[j] = __ldg(vbf + (int64_t)rr * sh.Wk + (cc >> 5));
        pv[j] = __ldg(wpf + (int64_t)rr * sh.Wk + (cc >> 5));
      }
    }
#pragma unroll
    for (int j = 0; j < NA; ++j) {
      const int e = tid + j * T;
      if (e >= NH) break;
      const int y = e / GC, x = e - y * GC;
      const int rr = r0 - 1 + y;
      const int cc = wrapc(c0 - 1 + x, sh.Sk);
      const uint32_t bit = 1u << (cc & 31);
      const int id = (wv[j] & bit) ? pv[j] + __popc(wv[j] & (bit - 1u)) : -1;
      Vec3 q = {0.0, 0.0, 0.0};
      if (id >= 0) q = cell_pos(sn, rr, cc * sh.k, rv[j]);
      s_px[e] = q.x;
      s_py[e] = q.y;
      s_pz[e] = q.z;
      s_id[e] = id;
    }
  }
  __syncthreads();
  for (int hy = warp; hy < GR; hy += T / 32) {
    const int* row = s_id + hy * GC;
    const unsigned lo = __ballot_sync(0xffffffffu, row[1 + lane] >= 0);
    const unsigned hi = __ballot_sync(0xffffffffu, row[33 + lane] >= 0);
    if (lane == 0) {
      s_hm[hy] = ((unsigned long long)hi << 32) | lo;
      s_he[hy] = (row[0] >= 0 ? 1u : 0u) | (row[GC - 1] >= 0 ? 2u : 0u);
    }
  }
  __syncthreads();
  PH_MARK(1);

  // L. slot masks (mesh.py:83-102) from the presence bits, work lists
  auto pres = [&](int hy, int xx) -> unsigned {  // xx = tile column (-1..64)
    return xx < 0 ? (s_he[hy] & 1u) : xx > 63 ? ((s_he[hy] >> 1) & 1u) : (unsigned)((s_hm[hy] >> xx) & 1ull);
  };
#pragma unroll
  for (int j = 0; j < NT / T; ++j) {
    const int e = tid + j * T;
    const int y = e / TC, x = e - y * TC;
    const int hy = y + 1;
    unsigned m = 0;
    const bool node = y < TRe && x < TCe && pres(hy, x);
    if (node) {
      const int g = hy * GC + x + 1;
#pragma unroll
      for (int s = 0; s < 6; ++s)
        if (s_id[g + slot_dr(s) * GC + slot_dc(s)] >= 0 && !(s == 5 && sh.Sk == 2)) m |= 1u << s;
    }
    s_m[e] = (uint8_t)m;
    s_has[e] = 0;
    s_req[e] = 0;
    const bool six = node && m == 0x3fu, gen = node && m != 0x3fu;
    const unsigned b6 = __ballot_sync(0xffffffffu, six), bg = __ballot_sync(0xffffffffu, gen);
    int o6 = 0, og = 0;
    if (lane == 0) {
      if (b6) o6 = atomicAdd(&s_cnt[0], __popc(b6));
      if (bg) og = atomicAdd(&s_cnt[1], __popc(bg));
    }
    o6 = __shfl_sync(0xffffffffu, o6, 0);
    og = __shfl_sync(0xffffffffu, og, 0);
    const unsigned below = (1u << lane) - 1u;
    if (six) s_list[o6 + __popc(b6 & below)] = (unsigned short)e;
    if (gen) s_list[NT - 1 - (og + __popc(bg & below))] = (unsigned short)e;
  }
  __syncthreads();
  PH_MARK(2);

  // B. certified fp32 normals
  const int nfan6 = s_cnt[0], ngen = s_cnt[1];
  auto node_normal = [&](int e, unsigned m) {
    const int y = e / TC, x = e - y * TC;
    const int g = (y + 1) * GC + (x + 1);
    const Vec3 p = posg(g);
    Fan32 fan;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      if (!((m >> s) & 1u)) continue;
      const Vec3 q = posg(g + slot_dr(s) * GC + slot_dc(s));
      fan.add(__double2float_rn(__dsub_rn(q.x, p.x)), __double2float_rn(__dsub_rn(q.y, p.y)),
              __double2float_rn(__dsub_rn(q.z, p.z)), cp.deg2);
    }
    float nv[3] = {0.f, 0.f, 0.f}, err = 0.f;
    const int st = fan.finish(__double2float_rn(p.x), __double2float_rn(p.y), __double2float_rn(p.z), nv, err);
    if (st == 1) {
      s_nx[e] = nv[0];
      s_ny[e] = nv[1];
      s_nz[e] = nv[2];
      s_eh[e] = __float2half_ru(err * (1.0f / kU32));
      s_has[e] = 1;
    } else if (st >= 2) {
      s_has[e] = 2;
      s_req[e] = (uint8_t)st;
      s_xl[atomicAdd(&s_cnt[2], 1)] = (unsigned short)e;
    }
  };
  for (int i = tid; i < nfan6; i += T) node_normal(s_list[i], 0x3fu);  // straight-line: all six slots
  // the rest from the first warp after the six-slot list's last partial warp
  // (as in k_tile)
  const int gstart = (((nfan6 % T) + 31) & ~31) % T;
  for (int i = (tid - gstart + T) % T; i < ngen; i += T) {
    const int e = s_list[NT - 1 - i];
    node_normal(e, s_m[e]);
  }
  __syncthreads();
  PH_MARK(3);

  // X. exact fp64 normals of the listed nodes, from the smem positions
  double* xf = xn + nbase * 3;
  auto run_exact = [&](int n) {
    for (int i = tid; i < n; i += T) {
      const int e = s_xl[i];
      const int y = e / TC, x = e - y * TC;
      const int g = (y + 1) * GC + (x + 1);
      const unsigned m = s_m[e];
      const Vec3 p = posg(g);
      FanT<kFastMath> fan;
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        if (!((m >> s) & 1u)) continue;
        const Vec3 q = posg(g + slot_dr(s) * GC + slot_dc(s));
        fan.add(__dsub_rn(q.x, p.x), __dsub_rn(q.y, p.y), __dsub_rn(q.z, p.z));
      }
      double nv[3];
      const bool has = fan.finish(p, nv);
      const double qn = __longlong_as_double(0x7ff8000000000000LL);
      const int64_t cell = (int64_t)(r0 + y) * sh.Sk + c0 + x;
      xf[cell * 3] = has ? nv[0] : qn;
      xf[cell * 3 + 1] = has ? nv[1] : qn;
      xf[cell * 3 + 2] = has ? nv[2] : qn;
      if (s_req[e] >= 2) {  // X0: the exact normal is the node's output
        s_has[e] = has ? 1 : 0;
        if (has) {
          s_nx[e] = __double2float_rn(nv[0]);
          s_ny[e] = __double2float_rn(nv[1]);
          s_nz[e] = __double2float_rn(nv[2]);
          s_eh[e] = __float2half_ru(0.5f);  // rounding of the exact normal to fp32
        }
      }
    }
  };
  const int nx0 = s_cnt[2];
  if (nx0) {
    run_exact(nx0);
    __syncthreads();
    if (tid == 0) s_cnt[2] = 0;  // no reader before the next barrier
  }
  PH_MARK(4);

  // D. per row: edge decisions + per-node outputs.  One warp per row, lane x
  // and x + 32.  Undecided edges list their not-yet-exact endpoints for X1.
  const bool full_width = (c0 == 0 && TCe == sh.Sk);
  unsigned long long* mrow = masks + (((int64_t)f * tilesR + r0 / TR) * tilesC + c0 / TC) * (TR * 5);
  float4* bf = bn4 + (int64_t)f * bn4_frame(sh, TR, TC);
  const int tr = r0 / TR, tc = c0 / TC;
  auto request = [&](int e) {
    const unsigned sft = (e & 3) * 8;
    const unsigned old = atomicOr(reinterpret_cast<unsigned*>(s_req) + (e >> 2), 1u << sft);
    if (!((old >> sft) & 0xffu)) s_xl[atomicAdd(&s_cnt[3], 1)] = (unsigned short)e;
  };
  auto decide = [&](int ea, int eb) -> int {  // 1 pass, 0 fail, 2 undecided
    if (!s_has[eb]) return 0;
    const int r = cert_pass(cp, s_nx[ea], s_ny[ea], s_nz[ea], __half2float(s_eh[ea]) * kU32, s_nx[eb], s_ny[eb],
                            s_nz[eb], __half2float(s_eh[eb]) * kU32);
    if (r == 2) {
      request(ea);
      request(eb);
    }
    return r;
  };
  for (int y = warp; y < TR; y += T / 32) {
    unsigned long long H = 0, V0 = 0, V1 = 0, HS = 0, UH = 0, UV0 = 0, UV1 = 0;
    unsigned W = 0, UW = 0;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int x = lane + 32 * half;
      const int e = y * TC + x;
      const bool in = y < TRe && x < TCe;
      const bool hs = in && s_has[e];
      int h = 0, v0 = 0, v1 = 0, w0 = 0, w1 = 0;
      if (hs) {
        if (x + 1 < TCe) h = decide(e, e + 1);
        if (y + 1 < TRe) {
          v0 = decide(e, e + TC);
          if (x + 1 < TCe) v1 = decide(e, e + TC + 1);
        }
        if (full_width && x == TCe - 1) {
          if (TCe > 1) w0 = decide(e, y * TC);
          if (y + 1 < TRe) w1 = decide(e, (y + 1) * TC);
        }
      }
      const int sh_ = half ? 32 : 0;
      H |= (unsigned long long)__ballot_sync(0xffffffffu, h == 1) << sh_;
      V0 |= (unsigned long long)__ballot_sync(0xffffffffu, v0 == 1) << sh_;
      V1 |= (unsigned long long)__ballot_sync(0xffffffffu, v1 == 1) << sh_;
      HS |= (unsigned long long)__ballot_sync(0xffffffffu, hs) << sh_;
      W |= (__ballot_sync(0xffffffffu, w0 == 1) ? 1u : 0u) | (__ballot_sync(0xffffffffu, w1 == 1) ? 2u : 0u);
      if (__any_sync(0xffffffffu, (h | v0 | v1 | w0 | w1) & 2)) {  // rare
        UH |= (unsigned long long)__ballot_sync(0xffffffffu, h == 2) << sh_;
        UV0 |= (unsigned long long)__ballot_sync(0xffffffffu, v0 == 2) << sh_;
        UV1 |= (unsigned long long)__ballot_sync(0xffffffffu, v1 == 2) << sh_;
        UW |= (__ballot_sync(0xffffffffu, w0 == 2) ? 1u : 0u) | (__ballot_sync(0xffffffffu, w1 == 2) ? 2u : 0u);
      }
      // per-node outputs
      if (in) {
        const int rr = r0 + y, cc = c0 + x;
        const int g = (y + 1) * GC + (x + 1);
        const int id = s_id[g];
        if (node_ids) node_ids[nbase + (int64_t)rr * sh.Sk + cc] = id;
        if (id >= 0) {
          int nb[6];
#pragma unroll
          for (int s = 0; s < 6; ++s) nb[s] = s_id[g + slot_dr(s) * GC + slot_dc(s)];
          if (sh.Sk == 2 && nb[5] == nb[2]) nb[5] = -1;
          int2* o2 = reinterpret_cast<int2*>(neighbors + (nbase + id) * 6);
          o2[0] = make_int2(nb[0], nb[1]);
          o2[1] = make_int2(nb[2], nb[3]);
          o2[2] = make_int2(nb[4], nb[5]);
          const float qn = __int_as_float(0x7fc00000);
          const float4 v = hs ? make_float4(s_nx[e], s_ny[e], s_nz[e], __half2float(s_eh[e]) * kU32)
                              : make_float4(qn, qn, qn, -1.0f);
          if (n32) {
            float* o = n32 + (nbase + id) * 3;
            o[0] = v.x;
            o[1] = v.y;
            o[2] = v.z;
          }
          if (dbg_err) dbg_err[nbase + id] = s_req[e] >= 2 ? -10.0f - s_req[e] : v.w;
          nmask[nbase + id] = hs ? 1 : 0;
          if (hs) {
            if (y == 0) bf[bn4_row(sh, 2 * tr, cc)] = v;
            if (y == TRe - 1) bf[bn4_row(sh, 2 * tr + 1, cc)] = v;
            if (x == 0) bf[bn4_col(sh, TR, 2 * tc, rr)] = v;
            if (x == TCe - 1) bf[bn4_col(sh, TR, 2 * tc + 1, rr)] = v;
          }
        }
      }
    }
    if (lane == 0) {
      mrow[y * 5 + 0] = H;
      mrow[y * 5 + 1] = V0;
      mrow[y * 5 + 2] = V1;
      mrow[y * 5 + 3] = HS;
      mrow[y * 5 + 4] = W;
      s_U[y * 3] = UH;
      s_U[y * 3 + 1] = UV0;
      s_U[y * 3 + 2] = UV1;
      s_UW[y] = UW;
      if ((UH | UV0 | UV1) || UW) atomicAdd(&s_cnt[4], 1);
    }
  }
  __syncthreads();
  PH_MARK(5);


  // X1 + D2 (rare; block-uniform): settle the undecided edges on exact normals
  if (s_cnt[4]) {
    const int nx1 = s_cnt[3];
    if (nx1) {
      run_exact(nx1);
      __syncthreads();
    }
    auto exact_pass = [&](int ea, int eb) -> bool {
      const int ya = ea / TC, yb = eb / TC;
      const int64_t ca = (int64_t)(r0 + ya) * sh.Sk + c0 + (ea - ya * TC);
      const int64_t cb = (int64_t)(r0 + yb) * sh.Sk + c0 + (eb - yb * TC);
      const double a[3] = {xf[ca * 3], xf[ca * 3 + 1], xf[ca * 3 + 2]};
      const double q[3] = {xf[cb * 3], xf[cb * 3 + 1], xf[cb * 3 + 2]};
      return normals_pass(a, q, cp.t[0], cp.t[1], cp.t[2]);
    };
    for (int y = warp; y < TR; y += T / 32) {
      const unsigned long long UH = s_U[y * 3], UV0 = s_U[y * 3 + 1], UV1 = s_U[y * 3 + 2];
      const unsigned UW = s_UW[y];
      if (!(UH | UV0 | UV1) && !UW) continue;  // warp-uniform
      unsigned long long H = 0, V0 = 0, V1 = 0;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int x = lane + 32 * half;
        const int e = y * TC + x;
        const int sh_ = half ? 32 : 0;
        bool h = false, v0 = false, v1 = false;
        if ((UH >> x) & 1ull) h = exact_pass(e, e + 1);
        if ((UV0 >> x) & 1ull) v0 = exact_pass(e, e + TC);
        if ((UV1 >> x) & 1ull) v1 = exact_pass(e, e + TC + 1);
        H |= (unsigned long long)__ballot_sync(0xffffffffu, h) << sh_;
        V0 |= (unsigned long long)__ballot_sync(0xffffffffu, v0) << sh_;
        V1 |= (unsigned long long)__ballot_sync(0xffffffffu, v1) << sh_;
      }
      if (lane == 0) {
        unsigned W = 0;
        if ((UW & 1u) && exact_pass(y * TC + TCe - 1, y * TC)) W |= 1u;
        if ((UW & 2u) && exact_pass(y * TC + TCe - 1, (y + 1) * TC)) W |= 2u;
        mrow[y * 5 + 0] |= H;
        mrow[y * 5 + 1] |= V0;
        mrow[y * 5 + 2] |= V1;
        mrow[y * 5 + 4] |= W;
      }
    }
  }
#if LSEG_PHASES
  __syncthreads();
#endif
  PH_MARK(0);
}

// Global union over tile-border edges from the certified border normals;
// undecided edges recompute both exact normals (exact_normal_at).
// Undecided edges go to a per-frame list (unc, counter fscal[f*4+2]) that
// k_merge_exact settles afterwards, keeping the fp64 path (and its registers)
// out of this kernel.  overflow_pass = true re-enumerates every border edge
// and settles the undecided ones inline (only for a frame whose list overflowed).
template <int TR, int TC>
__device__ __forceinline__ void merge_cert_frame(const lseg_sensor& sn, const Shape& sh, const double* ranges,
                                                 const uint32_t* vbits, const float4* bn4, const CertParams& cp,
                                                 int32_t* parent, int32_t* unc, int32_t* fscal, int f, int u0,
                                                 int ustep, bool overflow_pass) {
  const int nbr = (sh.R + TR - 1) / TR;
  const int nbc = (sh.Sk + TC - 1) / TC;
  const int per = nbr * sh.Sk + nbc * sh.R;
  const int64_t capp = sh.cap / 2;  // undecided-list capacity (pairs) per frame
  int32_t* par = parent + (int64_t)f * sh.cap;
  const float4* bn = bn4 + (int64_t)f * bn4_frame(sh, TR, TC);
  for (int u = u0; u < per; u += ustep) {
    int r, c;
    if (u < nbr * sh.Sk) {
      const int br = u / sh.Sk;
      r = min(br * TR + TR - 1, sh.R - 1);
      c = u - br * sh.Sk;
    } else {
      const int v = u - nbr * sh.Sk;
      const int bc = v / sh.R;
      c = min(bc * TC + TC - 1, sh.Sk - 1);
      r = v - bc * sh.R;
    }
    const int p = r * sh.Sk + c;
    const int pp = __ldcg(par + p);
    if (pp < 0) continue;  // no normal
    const int tr = r / TR;
    const bool last_row = (r == min(tr * TR + TR - 1, sh.R - 1));
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      if (r + slot_dr(s) >= sh.R) continue;
      if (edge_internal<TR, TC>(r, c, s, sh.Sk)) continue;
      const int rq = r + slot_dr(s), cq = wrapc(c + slot_dc(s), sh.Sk);
      const int q = rq * sh.Sk + cq;
      const int pq = __ldcg(par + q);
      if (pq < 0) continue;
      float4 a, bq;
      if (slot_dr(s) == 1 && last_row) {
        a = __ldcg(bn + bn4_row(sh, 2 * tr + 1, c));
        bq = __ldcg(bn + bn4_row(sh, 2 * (rq / TR), cq));
      } else {
        a = __ldcg(bn + bn4_col(sh, TR, 2 * (c / TC) + 1, r));
        bq = __ldcg(bn + bn4_col(sh, TR, 2 * (cq / TC), rq));
      }
      int d = cert_pass(cp, a.x, a.y, a.z, a.w, bq.x, bq.y, bq.z, bq.w);
      if (d == 2) {
        if (overflow_pass) {
          const double* rf = ranges + (int64_t)f * sh.R * sh.S;
          const uint32_t* vbf = vbits + (int64_t)f * sh.R * sh.Wk;
          double na[3], nq[3];
          const bool ha = exact_normal_at(sn, sh, rf, vbf, r, c, na);
          const bool hq = exact_normal_at(sn, sh, rf, vbf, rq, cq, nq);
          d = (ha && hq && normals_pass(na, nq, cp.t[0], cp.t[1], cp.t[2])) ? 1 : 0;
        } else {
          const int idx = atomicAdd(fscal + f * 4 + 2, 1);
          if (idx < capp) {
            unc[(int64_t)f * sh.cap + 2 * idx] = p;
            unc[(int64_t)f * sh.cap + 2 * idx + 1] = q;
          }
        }
      }
      if (d == 1) uf_union_pre(par, p, pp, q, pq);  // a stale parent is still an ancestor
    }
  }
}

template <int TR, int TC>
__global__ void k_merge_cert(lseg_sensor sn, Shape sh, const double* __restrict__ ranges,
                             const uint32_t* __restrict__ vbits, const float4* __restrict__ bn4, CertParams cp,
                             int32_t* __restrict__ parent, int32_t* __restrict__ unc, int32_t* __restrict__ fscal) {
  pdl_trigger();
  pdl_wait();
  merge_cert_frame<TR, TC>(sn, sh, ranges, vbits, bn4, cp, parent, unc, fscal, blockIdx.y,
                           blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, false);
}

// Settles the undecided border edges of k_merge_cert with exact normals.
template <int TR, int TC>
__global__ void k_merge_exact(lseg_sensor sn, Shape sh, const double* __restrict__ ranges,
                              const uint32_t* __restrict__ vbits, const float4* __restrict__ bn4, CertParams cp,
                              int32_t* __restrict__ parent, const int32_t* __restrict__ unc,
                              int32_t* __restrict__ fscal) {
  pdl_trigger();
  pdl_wait();
  const int f = blockIdx.y;
  const int n = fscal[f * 4 + 2];
  if (n == 0) return;
  if (n > sh.cap / 2) {  // list overflowed: redo the frame's border edges inline
    merge_cert_frame<TR, TC>(sn, sh, ranges, vbits, bn4, cp, parent, nullptr, fscal, f, threadIdx.x, blockDim.x,
                             true);
    return;
  }
  const double* rf = ranges + (int64_t)f * sh.R * sh.S;
  const uint32_t* vbf = vbits + (int64_t)f * sh.R * sh.Wk;
  int32_t* par = parent + (int64_t)f * sh.cap;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int p = unc[(int64_t)f * sh.cap + 2 * i], q = unc[(int64_t)f * sh.cap + 2 * i + 1];
    const int r = p / sh.Sk, c = p - r * sh.Sk, rq = q / sh.Sk, cq = q - rq * sh.Sk;
    double na[3], nq[3];
    const bool ha = exact_normal_at(sn, sh, rf, vbf, r, c, na);
    const bool hq = exact_normal_at(sn, sh, rf, vbf, rq, cq, nq);
    if (ha && hq && normals_pass(na, nq, cp.t[0], cp.t[1], cp.t[2])) uf_union(par, p, q);
  }
}

// Tile-local connected components from the tile's pass masks (the body of
// k_tile_cc, one small CTA per tile): each node's parent starts as the first
// cell of its horizontal run (bit arithmetic); vertical / diagonal edges --
// minus those whose parallel edge one column to the left already joins the
// same two runs -- join runs by union-find in shared memory; each
// labelled cell gets parent[cell] = minimum cell of its tile-local component
// (-1 without a normal).
template <int TR, int TC, int T>
__device__ __forceinline__ void tile_cc_body(const Shape& sh, int f, int r0, int c0, int TRe, int TCe,
                                             const unsigned long long* s_m, int* s_par, int32_t* __restrict__ parent,
                                             uint32_t* __restrict__ lroots, int32_t* __restrict__ hist, int64_t K) {
  constexpr int NT = TR * TC;
  // run starts: parent of every cell = first cell of its horizontal run (the
  // cell after the highest failing row edge below it), branch-free on the
  // 32-bit halves of the row mask
  static_assert(NT % T == 0 && TC == 64 && T % 32 == 0, "each warp step covers a 32-cell chunk of one row");
  constexpr int NJ = NT / T;
  unsigned starts = 0;  // which of this thread's cells (tid + j T) are run starts
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int e = threadIdx.x + j * T;
    const int y = e / TC, x = e - y * TC;
    const unsigned long long Hm = s_m[y * 5];
    const uint32_t hl = (uint32_t)Hm, hh = (uint32_t)(Hm >> 32);
    // branch-free: the cell's own half first, then (upper half) the lower one
    const bool up = x >= 32;
    const uint32_t Z = ~(up ? hh : hl) & ((1u << (x & 31)) - 1u);
    const int lowst = (up && ~hl) ? 32 - __clz(~hl) : 0;
    const int st = Z ? (up ? 64 : 32) - __clz(Z) : lowst;
    s_par[e] = y * TC + st;
    if (st == x) starts |= 1u << j;
  }
  __syncthreads();
  // vertical / diagonal unions: an edge is dropped (64-bit mask arithmetic,
  // one thread per row pair) when another kept edge joins the same two runs:
  // the parallel edge one column to the left, or -- for a diagonal (y,x) ->
  // (y+1,x+1) -- the vertical edge into (y+1,x) or out of (y,x+1) when the
  // row edge between them passes (vertical edges are only ever dropped for
  // vertical edges further left, so no drop depends on itself); the rest are
  // unioned cell-parallel
  __shared__ unsigned long long s_U[TR * 2];
  for (int y = threadIdx.x; y < TR; y += T) {
    unsigned long long U0 = 0, U1 = 0;
    if (y + 1 < TRe) {
      const unsigned long long Hy = s_m[y * 5], V0 = s_m[y * 5 + 1], V1 = s_m[y * 5 + 2];
      const unsigned long long Hn = s_m[(y + 1) * 5];
      U0 = V0 & ~((Hy << 1) & (Hn << 1) & (V0 << 1));
      U1 = V1 & ~((V0 & Hn) | ((Hy << 1) & Hn & (V1 << 1)) | (Hy & (V0 >> 1)));
    }
    s_U[2 * y] = U0;
    s_U[2 * y + 1] = U1;
  }
  __syncthreads();
  // Union-find over runs: labels live at run starts (every other cell keeps
  // s_par = its run start throughout).  The tile's run-to-run edges are
  // gathered into one dense shared-memory list (packed per thread first as
  // a | b0 << 10 | b1 << 20 | valid bits << 30, 10-bit tile cell indices);
  // all threads then union them lock-free (atomicCAS, larger root hooked
  // under the smaller, so each root is its component's minimum run start)
  // and compress the run starts -- two barriers, no rounds.
  static_assert(NT <= 1024, "10-bit cell indices");

  // each warp's edges as a dense list (a | b << 10) in its own shared-memory
  // segment (appended without atomics), then unioned by the same warp:
  // no block barrier between gathering and union.  At step j the warp's
  // lanes are one 32-cell chunk of a row, so the chunk's edge bits are read
  // straight from the row masks and chunks without edges are skipped.
  constexpr int SEG = 2 * NT / (T / 32);  // >= 2 edges per cell of the warp (+ the wraps, see below)
  __shared__ unsigned s_el[2 * NT];
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  unsigned* el = s_el + (threadIdx.x >> 5) * SEG;
  int ne = 0;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int e0 = (threadIdx.x & ~31) + j * T;
    const int y = e0 / TC, x0 = e0 - y * TC;
    const int e = e0 + lane;
    const uint32_t* sU32 = reinterpret_cast<const uint32_t*>(s_U);  // 32-bit halves (little-endian)
    const unsigned c0 = sU32[4 * y + (x0 >> 5)], c1 = sU32[4 * y + 2 + (x0 >> 5)];
    // unconditional (chunks without edges are rare; no branch / reconvergence)
    const unsigned a = (unsigned)s_par[e];
    // (the last row's reads past the tile land in s_par's padding: unused)
    if ((c0 >> lane) & 1u) el[ne + __popc(c0 & lt)] = a | (unsigned)s_par[e + TC] << 10;
    ne += __popc(c0);
    if ((c1 >> lane) & 1u) el[ne + __popc(c1 & lt)] = a | (unsigned)s_par[e + TC + 1] << 10;
    ne += __popc(c1);
  }
  // full-width column wrap (x = S'-1 -> 0), added by the last warp (fewest
  // edges: it holds row TR-1)
  if (threadIdx.x >= T - 32) {
    const int y = lane;
    const unsigned W = (y < TRe) ? (unsigned)s_m[y * 5 + 4] : 0u;
    const bool w0 = W & 1u, w1 = (W & 2u) && (y + 1 < TRe);
    const unsigned b0 = __ballot_sync(0xffffffffu, w0), b1 = __ballot_sync(0xffffffffu, w1);
    if (b0 | b1) {
      const unsigned a = (y < TRe) ? (unsigned)s_par[y * TC + TCe - 1] : 0u;
      if (w0) el[ne + __popc(b0 & lt)] = a | (unsigned)(y * TC) << 10;
      ne += __popc(b0);
      // (y + 1) * TC is 1024 on the last row: only when that edge exists
      if (w1) el[ne + __popc(b1 & lt)] = a | (unsigned)((y + 1) * TC) << 10;
      ne += __popc(b1);
    }
  }
  __syncwarp();
  const int any_edge = __syncthreads_or(ne);
  if (any_edge) {
    // lock-free union-find over the run-start labels (larger root hooked
    // under the smaller: root = component minimum; path halving on the way),
    // then full compression at run starts
    auto find = [&](int x) -> int {  // with path halving: unions only
      int p = s_par[x];
      while (p != x) {
        const int g = s_par[p];
        if (g != p) s_par[x] = g;  // x is not a root: only ever points further up
        x = p;
        p = g;
      }
      return x;
    };
    // read-only find for the compression (a halving store there could
    // overwrite a run start another thread has already compressed)
    auto root = [&](int x) -> int {
      int p = s_par[x];
      while (p != x) {
        x = p;
        p = s_par[x];
      }
      return x;
    };
    for (int k = lane; k < ne; k += 32) {
      const unsigned v = el[k];
      int ra = find(v & 1023u), rb = find(v >> 10);
      while (ra != rb) {
        if (ra < rb) { const int t = ra; ra = rb; rb = t; }
        const int old = atomicCAS(s_par + ra, ra, rb);
        if (old == ra) break;
        ra = find(old);
        rb = find(rb);
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NJ; ++j)
      if ((starts >> j) & 1u) s_par[threadIdx.x + j * T] = root(threadIdx.x + j * T);
    __syncthreads();
  }
  // ... and give every labelled cell its run start's root; tile-local roots
  // (cells that are their own root) also get a bit in `lroots`, so the global
  // flatten only has to chase those
  const int64_t nbase = (int64_t)f * sh.cap;
  // frame-local cell of the tile's first cell; per-tile base pointers, opaque
  // to the optimiser (32-bit tile-local offsets: one wide multiply-add per store)
  const int Sk = sh.Sk, Wk = sh.Wk;
  const int tbase = r0 * Sk + c0;
  int32_t* pbase = parent + nbase + tbase;
  int32_t* hbase = hist ? hist + (int64_t)f * K + 1 + tbase : nullptr;
  uint32_t* lbase = lroots + ((int64_t)f * sh.R + r0) * Wk + (c0 >> 5);
  asm volatile("" : "+l"(pbase), "+l"(hbase), "+l"(lbase));
  const int wrem = Wk - (c0 >> 5);  // words of the row from the tile's first
  const uint32_t* sm32 = reinterpret_cast<const uint32_t*>(s_m);
#pragma unroll
  for (int j = 0; j < NJ; ++j) {  // whole warps: cell e = tid + j T, one 32-cell half-row per warp
    const int e = threadIdx.x + j * T;
    const int y = e / TC, x = e - y * TC;
    const bool in = (y < TRe && x < TCe);
    const int loc = y * Sk + x;
    int pc = -1;
    if (in && ((sm32[(y * 5 + 3) * 2 + (x >> 5)] >> (x & 31)) & 1u)) {
      const int lr = s_par[s_par[e]];  // run start -> its label
      pc = tbase + (lr / TC) * Sk + lr % TC;
    }
    const bool isroot = in && pc == tbase + loc;
    if (in) pbase[loc] = pc;
    // histogram slot of every tile-local root zeroed here (a superset of the
    // final roots k_labels_backfill counts into)
    if (hbase && isroot) hbase[loc] = 0;
    const uint32_t b = __ballot_sync(0xffffffffu, isroot);
    if ((threadIdx.x & 31) == 0 && y < TRe && (x >> 5) < wrem) lbase[y * Wk + (x >> 5)] = b;
  }
}

// Test hook (lseg_debug_tile_cc): the tile CC body on given pass masks, one
// 16 x 64 tile per "frame" (tests/test_gpu_math.py checks it against a CPU
// union-find over the same edges).
template <int TR, int TC, int T>
__global__ void k_tile_cc_dbg(Shape sh, const unsigned long long* __restrict__ masks, int32_t* parent,
                              uint32_t* lroots) {
  __shared__ int s_par[TR * TC + TC + 1];  // + padding: the edge gathering's reads below the last row
  __shared__ unsigned long long s_m[TR * 5];
  const int f = blockIdx.x;
  for (int j = threadIdx.x; j < TR * 5; j += T) s_m[j] = masks[(int64_t)f * TR * 5 + j];
  __syncthreads();
  tile_cc_body<TR, TC, T>(sh, f, 0, 0, TR, TC, s_m, s_par, parent, lroots, nullptr, 0);
}
void debug_tile_cc(int n, const unsigned long long* masks, int32_t* parent, uint32_t* lroots) {
  const Shape sh = make_shape(n, TILE_R, TILE_C, 1);
  k_tile_cc_dbg<TILE_R, TILE_C, 256><<<n, 256>>>(sh, masks, parent, lroots);
}

template <int TR, int TC, int T>
__global__ void __launch_bounds__(T, LSEG_CC_TSM / T) k_tile_cc(Shape sh, const unsigned long long* __restrict__ masks,
                                               int32_t* __restrict__ parent, uint32_t* __restrict__ lroots,
                                               int32_t* __restrict__ hist, int64_t K) {
  pdl_trigger();
  pdl_wait();
  __shared__ int s_par[TR * TC + TC + 1];  // + padding: the edge gathering's reads below the last row
  __shared__ unsigned long long s_m[TR * 5];
  const int tilesC = (sh.Sk + TC - 1) / TC;
  const int tilesR = (sh.R + TR - 1) / TR;
  // grid (tile column, tile row, frame): per-CTA values straight from the
  // block index (uniform registers, no division)
  const int f = blockIdx.z;
  const int rem = blockIdx.y * tilesC + blockIdx.x;  // tile within the frame
  const int64_t b = (int64_t)f * tilesR * tilesC + rem;
  const int r0 = blockIdx.y * TR, c0 = blockIdx.x * TC;
  const int TRe = min(TR, sh.R - r0), TCe = min(TC, sh.Sk - c0);
  const unsigned long long* mrow = masks + b * (TR * 5);
  for (int j = threadIdx.x; j < TR * 5; j += T) s_m[j] = __ldg(mrow + j);
  __syncthreads();
  tile_cc_body<TR, TC, T>(sh, f, r0, c0, TRe, TCe, s_m, s_par, parent, lroots, hist, K);
}

// Global union over the forward edges that leave a tile.  Threads enumerate
// the cells of each tile's last row and last column (corner duplicates are
// harmless); both endpoints' fp64 normals come from `bnorm`.  Along a tile
// border most passing edges join the same two tile-local components, so a
// warp first collapses edges with equal (parent of p, parent of q) -- the
// same union -- and only one lane per distinct pair runs it: far fewer CAS
// on the few large roots.
template <int TR, int TC>
__global__ void k_merge(Shape sh, const double* __restrict__ bnorm, double t0, double t1, double t2,
                        int32_t* __restrict__ parent) {
  pdl_trigger();
  pdl_wait();
  // blockIdx.y = frame; threads enumerate the frame's border cells
  const int f = blockIdx.y;
  const int nbr = (sh.R + TR - 1) / TR;
  const int nbc = (sh.Sk + TC - 1) / TC;
  const int per = nbr * sh.Sk + nbc * sh.R;
  int32_t* par = parent + (int64_t)f * sh.cap;
  const double* bn = bnorm + (int64_t)f * bn_frame(sh, TR, TC);
  asm volatile("" : "+l"(par), "+l"(bn));  // frame bases opaque: one wide multiply-add per access
  const int lane = threadIdx.x & 31;
  // warp-uniform trip count (the dedup below needs whole warps)
  for (int u0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); u0 < per; u0 += gridDim.x * blockDim.x) {
    const int u = u0 + lane;
    int r = 0, c = 0, pp = -1;
    if (u < per) {
      if (u < nbr * sh.Sk) {
        const int br = fdiv(u, sh.Sk, sh.inv_Sk);
        r = min(br * TR + TR - 1, sh.R - 1);
        c = u - br * sh.Sk;
      } else {
        const int v = u - nbr * sh.Sk;
        const int bc = fdiv(v, sh.R, sh.inv_R);
        c = min(bc * TC + TC - 1, sh.Sk - 1);
        r = v - bc * sh.R;
      }
      pp = __ldcg(par + r * sh.Sk + c);  // -1: no normal
    }
    const int p = r * sh.Sk + c;
    const int tr = r / TR, tc = c / TC;
    const bool last_row = (r == min(tr * TR + TR - 1, sh.R - 1));
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      bool want = false;
      int q = 0, pq = -1;
      if (pp >= 0 && r + slot_dr(s) < sh.R && !edge_internal<TR, TC>(r, c, s, sh.Sk)) {
        const int rq = r + slot_dr(s), cq = wrapc(c + slot_dc(s), sh.Sk);
        q = rq * sh.Sk + cq;
        pq = __ldcg(par + q);
        if (pq >= 0) {
          // an edge that crosses a tile-row boundary reads both normals from
          // the row border store, one that only crosses a column boundary
          // from the column border store
          const double *pa, *pb;
          if (slot_dr(s) == 1 && last_row) {
            pa = bn + bn_row(sh, 2 * tr + 1, c);
            pb = bn + bn_row(sh, 2 * (rq / TR), cq);
          } else {
            pa = bn + bn_col(sh, TR, 2 * tc + 1, r);
            pb = bn + bn_col(sh, TR, 2 * (cq / TC), rq);
          }
          const double a[3] = {__ldcg(pa), __ldcg(pa + 1), __ldcg(pa + 2)};
          const double b[3] = {__ldcg(pb), __ldcg(pb + 1), __ldcg(pb + 2)};
          want = normals_pass(a, b, t0, t1, t2);
        }
      }
      const unsigned long long key =
          want ? ((unsigned long long)(unsigned)pp << 32 | (unsigned)pq) : ~0ull;
      const unsigned m = __match_any_sync(0xffffffffu, key);
      if (want && lane == __ffs(m) - 1) uf_union_pre(par, p, pp, q, pq);  // stale parents are ancestors
    }
  }
}

// Read-only root chase (parent[x] <= x, so it terminates).
__device__ __forceinline__ int root_of(const int32_t* __restrict__ par, int x) {
  int p = __ldcg(par + x);
  while (p != x) { x = p; p = __ldcg(par + x); }
  return x;
}

// After k_merge: point every labelled cell straight at its final root, mark
// roots with a bit per kept cell (k_frame_scan over these gives label ranks)
// and zero each root's histogram slot (labels are root cell + 1 until pruning).
__global__ void k_root_flatten(Shape sh, int32_t* __restrict__ parent, const uint32_t* __restrict__ lroots,
                               uint32_t* __restrict__ rbits, int32_t* __restrict__ hist, int64_t K,
                               int32_t* __restrict__ fscal, int32_t* __restrict__ rstat,
                               int32_t* __restrict__ n_labels) {
  pdl_trigger();
  pdl_wait();
  // after k_merge: point every tile-local root straight at its final root
  // (the only cells whose chains can be long; every other cell points at its
  // tile-local root, so its final root is parent[parent[cell]]), mark final
  // roots and zero their histogram slots.  One CTA per ring row, one warp per
  // 32-cell word, no 64-bit division.
  const int row = blockIdx.x;
  const int f = row / sh.R, i = row - f * sh.R;
  const int lane = threadIdx.x & 31;
  int32_t* par = parent + (int64_t)f * sh.cap;
  int32_t* hf = hist + (int64_t)f * K;
  if (threadIdx.x == 0) {
    rstat[row] = 0;                   // k_prune_rows' per-row survivor count (+ ready flag)
    if (row == 0) fscal[3] = 0;       // k_prune_rows' row ticket
  }
  __shared__ int s_nroot;
  if (threadIdx.x == 0) s_nroot = 0;
  __syncthreads();
  int nroot = 0;
  for (int w = threadIdx.x >> 5; w < sh.Wk; w += blockDim.x >> 5) {
    const uint32_t lr = __ldg(lroots + (int64_t)row * sh.Wk + w);
    bool root = false;
    if ((lr >> lane) & 1u) {
      const int cell = i * sh.Sk + w * 32 + lane;
      const int p = __ldcg(par + cell);
      const int r = root_of(par, p);
      if (r != p) par[cell] = r;
      root = (r == cell);
      if (root) hf[cell + 1] = 0;
    }
    const uint32_t b = __ballot_sync(0xffffffffu, root);
    if (lane == 0) {
      rbits[(int64_t)row * sh.Wk + w] = b;
      nroot += __popc(b);
    }
  }
  // segment() label count of the frame (zeroed by the tile kernel): one
  // global atomic per row
  if (lane == 0 && nroot) atomicAdd(&s_nroot, nroot);
  __syncthreads();
  if (threadIdx.x == 0 && s_nroot) atomicAdd(n_labels + f, s_nroot);
}

// 1 + rank of root cell rc among the set bits of (bits, pre) = its label.
__device__ __forceinline__ int rank_label(const uint32_t* bf, const int32_t* pf, int Wk, int Sk, int rc,
                                          double inv_Sk) {
  const int rr = fdiv(rc, Sk, inv_Sk), cc = rc - rr * Sk;
  return 1 + node_id_at(bf + (int64_t)rr * Wk, pf + (int64_t)rr * Wk, cc);
}

// Nearest donor of target cell s in a ring row (reference segment.py:91-106:
// cyclic step distance, ties to the smaller actual step index), from the
// row's donor bitmask in shared memory.  Scans 32-cell words outward from s;
// the row must hold at least one donor.
__device__ __forceinline__ int nearest_donor(const uint32_t* s_dm, int nw, int S, int s) {
  const int w = s >> 5, b = s & 31;
  // left: highest donor < s (cyclic)
  int left;
  {
    uint32_t m = s_dm[w] & ((1u << b) - 1u);
    int ww = w;
    while (!m) {
      ww = (ww == 0) ? nw - 1 : ww - 1;
      m = s_dm[ww];
      if (ww == w) m &= ~((1u << b) - 1u) & ~(1u << b);  // wrapped to own word: only cells > s remain
    }
    left = ww * 32 + 31 - __clz(m);
  }
  int right;
  {
    uint32_t m = (b == 31) ? 0u : (s_dm[w] & ~((2u << b) - 1u));
    int ww = w;
    while (!m) {
      ww = (ww + 1 == nw) ? 0 : ww + 1;
      m = s_dm[ww];
      if (ww == w) m &= (1u << b) - 1u;  // wrapped to own word: only cells < s remain
    }
    right = ww * 32 + __ffs(m) - 1;
  }
  int dl = s - left;
  if (dl <= 0) dl += S;
  int dr = right - s;
  if (dr <= 0) dr += S;
  return dl < dr ? left : (dr < dl ? right : min(left, right));
}

// Nearest donor of cell s when the donors are kept cells (cell = column * k):
// the highest donor column <= cl0 and the lowest >= cr0, both cyclic over the
// kept-column bits, then the reference rule (segment.py:91-106: cyclic step
// distance, ties to the smaller step index).  cl0 = the last column whose
// cell is < s (-1 wraps), cr0 = the first whose cell is > s.  The row must
// hold at least one donor.  Returns the donor column.
__device__ __forceinline__ int nearest_kept_donor(const uint32_t* s_kdm, int nwk, int k, int S, int s, int cl0,
                                                  int cr0) {
  int cl;
  {
    int ww;
    uint32_t m;
    if (cl0 < 0) {
      ww = nwk - 1;
      m = s_kdm[ww];
    } else {
      ww = cl0 >> 5;
      const int b = cl0 & 31;
      m = s_kdm[ww] & (b == 31 ? 0xffffffffu : ((2u << b) - 1u));
    }
    while (!m) {
      ww = (ww == 0) ? nwk - 1 : ww - 1;
      m = s_kdm[ww];
    }
    cl = ww * 32 + 31 - __clz(m);
  }
  int cr;
  {
    int ww = cr0 >> 5;
    uint32_t m = (ww < nwk) ? (s_kdm[ww] & ~((1u << (cr0 & 31)) - 1u)) : 0u;
    if (ww >= nwk) ww = nwk - 1;
    while (!m) {
      ww = (ww + 1 == nwk) ? 0 : ww + 1;
      m = s_kdm[ww];
    }
    cr = ww * 32 + __ffs(m) - 1;
  }
  const int L = cl * k, Rc = cr * k;
  int dl = s - L;
  if (dl <= 0) dl += S;
  int dr = Rc - s;
  if (dr <= 0) dr += S;
  return dl < dr ? cl : (dr < dl ? cr : (L < Rc ? cl : cr));
}

// nearest_donor with per-word tables: P[w] / N[w] = the nearest word at or
// before / after word w (cyclic) holding a donor.  O(1) per target instead of
// a word-by-word search (rows of fragmented frames have few, far donors).
// Same result as nearest_donor (the row must hold at least one donor).
__device__ __forceinline__ int nearest_donor_tab(const uint32_t* s_dm, const short* P, const short* N, int nw, int S,
                                                 int s) {
  const int w = s >> 5, b = s & 31;
  int left;
  {
    const uint32_t m = s_dm[w] & ((1u << b) - 1u);
    if (m) {
      left = w * 32 + 31 - __clz(m);
    } else {  // the nearest earlier donor word; if that wrapped back to w, its donors are all above s
      const int pw = P[w == 0 ? nw - 1 : w - 1];
      left = pw * 32 + 31 - __clz(s_dm[pw]);
    }
  }
  int right;
  {
    const uint32_t m = (b == 31) ? 0u : (s_dm[w] & ~((2u << b) - 1u));
    if (m) {
      right = w * 32 + __ffs(m) - 1;
    } else {
      const int nx = N[w + 1 == nw ? 0 : w + 1];
      right = nx * 32 + __ffs(s_dm[nx]) - 1;
    }
  }
  int dl = s - left;
  if (dl <= 0) dl += S;
  int dr = right - s;
  if (dr <= 0) dr += S;
  return dl < dr ? left : (dr < dl ? right : min(left, right));
}

// Shared body of k_prune_rows' fill: s_val[s] holds a donor label (> 0),
// 0 (passive: stays 0) or -2 (target: nearest donor's label, 0 if the row has
// no donor); s_dm the donor bits.  Returns the filled label of cell s.
__device__ __forceinline__ int fill_one(const int* s_val, const uint32_t* s_dm, int nw, int S, int s, bool any) {
  const int v = s_val[s];
  if (v != -2) return v > 0 ? v : 0;
  return any ? s_val[nearest_donor(s_dm, nw, S, s)] : 0;
}

// Warp-aggregated histogram increment (adjacent cells mostly share a label).
__device__ __forceinline__ void hist_add(int32_t* hw, int lab) {
  const unsigned m = __match_any_sync(0xffffffffu, lab);
  if (lab > 0 && (threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(hw + lab, __popc(m));
}

// Node labels + backfill + histogram, one CTA per ring row.  Provisional
// label ids are root cell + 1 (ascending root cell == ascending reference
// label, so the compaction in k_prune_rows reproduces the reference ids).
// Donors are kept cells only, so the row is classified per kept column
// (label / valid-without-label target / invalid) and every cell then takes
// its value: a non-kept valid cell between two donor columns picks the nearer
// one directly, the rest search the donor-column bits.
template <int T, bool DIRECT>
__global__ void __launch_bounds__(T, LSEG_LAB_TSM / T) k_labels_backfill(lseg_sensor sn, Shape sh, const double* __restrict__ ranges,
                                                       const uint32_t* __restrict__ vbits,
                                                       const uint32_t* __restrict__ fbits,
                                                       const int32_t* __restrict__ parent,
                                                       const uint32_t* __restrict__ rbits,
                                                       const int32_t* __restrict__ rpre,
                                                       int32_t* __restrict__ node_labels, int32_t* __restrict__ out,
                                                       int32_t* __restrict__ hist, int64_t K,
                                                       uint32_t* __restrict__ rbits_out, int32_t* __restrict__ n_labels,
                                                       int32_t* __restrict__ rstat, int32_t* __restrict__ ticket) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ int s_dynrow[];
  const int S = sh.S, Sk = sh.Sk, k = sh.k, nwk = sh.Wk, nw = (S + 31) / 32;
  int* s_kv = s_dynrow;                                                 // per kept column
  uint32_t* s_kdm = reinterpret_cast<uint32_t*>(s_dynrow + nwk * 32);  // donor columns
  uint32_t* s_ktw = s_kdm + nwk;                                        // k = 1: backfill-target columns
  __shared__ int s_any;
  const int row = blockIdx.x;
  const int f = fdiv(row, sh.R, sh.inv_R), i = row - f * sh.R;
  const uint32_t* vbr = vbits + (int64_t)row * sh.Wk;
  const uint32_t* fbr = fbits ? fbits + (int64_t)row * nw : nullptr;
  const int32_t* parf = parent + (int64_t)f * sh.cap;
  // opaque to the optimiser: frame-local indices then cost one wide multiply-add
  // per load instead of a re-associated 64-bit index computation
  int32_t* hw = hist + (int64_t)f * K;
  asm volatile("" : "+l"(parf), "+l"(hw));
  const int32_t* par = parf + (int64_t)i * sh.Sk;
  const uint32_t* rbf = rbits + (int64_t)f * sh.R * sh.Wk;
  const int32_t* rpf = rpre + (int64_t)f * sh.R * sh.Wk;
  const int64_t rb = (int64_t)row * S;
  int32_t* outr = out + rb;
  // rbits_out != nullptr: k_root_flatten's work folded in (no node_labels
  // output): each column chases its tile-local root to the final root
  // itself, the row's final roots go to rbits_out and n_labels, and the
  // pruning's per-row counters are reset here
  const bool fold = DIRECT || rbits_out != nullptr;  // the direct (k = 1) variant is only launched folded
  // k = 1 without the segment() output: labelled / passive cells are written
  // and counted while the columns are classified; the second pass only
  // handles the backfill targets (valid cells without a normal: rare at k = 1)
  constexpr bool direct = DIRECT;  // the launcher's choice: k == 1 && !node_labels
  __shared__ int s_nroot;
  if (threadIdx.x == 0) {
    s_any = 0;
    s_nroot = 0;
    if (fold) {
      rstat[row] = 0;
      if (row == 0) *ticket = 0;
    }
  }
  __syncthreads();
  bool any = false;
  int nroot = 0;
  // classify the kept columns: donor label / target -2 / passive 0.  Chunks
  // of PF columns per thread with all loads of a chunk issued before they
  // are used (the two dependent parent loads would otherwise serialise).
  constexpr int PF = LSEG_PF_LAB;
  for (int c0 = 0; c0 < nwk * 32; c0 += T * PF) {
    int pv[PF], lv[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) {
      const int c = c0 + threadIdx.x + j * T;
      pv[j] = (c < Sk) ? __ldcg(par + c) : -1;  // tile-local root
    }
#pragma unroll
    for (int j = 0; j < PF; ++j) lv[j] = pv[j] >= 0 ? __ldcg(parf + pv[j]) : 0;  // its parent: the final root
    if (fold) {
#pragma unroll
      for (int j = 0; j < PF; ++j)
        if (pv[j] >= 0 && lv[j] != pv[j]) lv[j] = root_of(parf, lv[j]);  // merged across tiles
    }
#pragma unroll
    for (int j = 0; j < PF; ++j) {
      const int c = c0 + threadIdx.x + j * T;
      if (c >= nwk * 32) break;
      if (fold) {
        const uint32_t rm = __ballot_sync(0xffffffffu, pv[j] >= 0 && lv[j] == i * Sk + c);
        if ((c & 31) == 0) {
          rbits_out[(int64_t)row * nwk + (c >> 5)] = rm;
          nroot += __popc(rm);
        }
      }
      int v = 0;
      if (pv[j] >= 0) v = lv[j] + 1;
      else if (c < Sk) v = ((__ldg(vbr + (c >> 5)) >> (c & 31)) & 1u) ? -2 : 0;  // valid, no normal
      s_kv[c] = v;
      const uint32_t dm = __ballot_sync(0xffffffffu, v > 0);
      if ((c & 31) == 0) s_kdm[c >> 5] = dm;
      any |= dm != 0;
      if (direct) {  // k = 1: every cell but the backfill targets is final here
        const uint32_t tm = __ballot_sync(0xffffffffu, v == -2);
        if ((c & 31) == 0) s_ktw[c >> 5] = tm;
        if (c < S && v != -2) outr[c] = v > 0 ? v : 0;
        hist_add(hw, v > 0 ? v : 0);
      }
    }
  }
  if (any && (threadIdx.x & 31) == 0) s_any = 1;
  if (nroot) atomicAdd(&s_nroot, nroot);
  __syncthreads();
  if (fold && threadIdx.x == 0 && s_nroot) atomicAdd(n_labels + f, s_nroot);
  const bool rany = s_any != 0;
  // s / k as a multiply-high: exact for s < 2^32 / k (S <= 16384 here)
  const unsigned kmag = 0xffffffffu / (unsigned)k + 1u;
  // k = 1: only the words holding backfill targets (one shared load per word)
  for (int s = threadIdx.x; s < nw * 32; s += T) {  // whole warps (hist_add)
    if (direct && s_ktw[s >> 5] == 0u) continue;  // warp-uniform
    int r = 0;
    if (s < S) {
      const int c = (k == 1) ? s : (int)__umulhi((unsigned)s, kmag);
      const int j = s - c * k;
      int v;
      if (j == 0) v = s_kv[c];
      else  // not a kept cell: valid full-resolution cell? (bits from k_bin_rows)
        v = fbr ? (((__ldg(fbr + (s >> 5)) >> (s & 31)) & 1u) ? -2 : 0)
                : (in_window(__ldg(ranges + rb + s), sn.r_min, sn.r_max) ? -2 : 0);
      if (v > 0) {
        r = v;
      } else if (v == -2 && rany) {
        bool done = false;
        if (j > 0) {  // between donor columns c and c + 1 (cyclic): nearer one, ties to the smaller cell
          const bool wrap = (c + 1 == Sk);
          const int vl = s_kv[c], vr = s_kv[wrap ? 0 : c + 1];
          if (vl > 0 && vr > 0) {
            const int dr = wrap ? S - s : k - j;
            r = (j < dr) ? vl : (dr < j ? vr : (wrap ? vr : vl));
            done = true;
          }
        }
        if (!done) r = s_kv[nearest_kept_donor(s_kdm, nwk, k, S, s, j > 0 ? c : c - 1, c + 1)];
      }
      if (node_labels)  // reference segment() output: 1 + rank of the root
        node_labels[rb + s] = (j == 0 && v > 0) ? rank_label(rbf, rpf, sh.Wk, sh.Sk, v - 1, sh.inv_Sk) : 0;
      if (!direct || v == -2) outr[s] = r;
      else r = 0;  // written and counted in the first pass
    }
    hist_add(hw, r);
  }
}

// ---------------------------------------------------------------- binning
static constexpr double kTwoPiF = 6.283185307179586;  // == 2.0 * np.pi

// First index in [lo, hi) whose ring id is >= v, found by one warp with a
// 32-ary search (4 dependent probes for a 124 k-point frame instead of 17).
// Exact for ring-major input; for other orders the result is arbitrary but in
// range, and k_bin_rows' segment check sends the frame to the generic path.
template <typename RT>
__device__ __forceinline__ int64_t warp_lower_bound(const RT* __restrict__ ring, int64_t lo, int64_t hi, int v,
                                                    int lane) {
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t q = lo + (int64_t)lane * step;
    const bool less = (q < hi) && ((int)__ldg(ring + q) < v);
    const unsigned m = __ballot_sync(0xffffffffu, less);
    const int c = (~m == 0u) ? 32 : __ffs(~m) - 1;  // leading lanes with ring < v
    const int64_t nlo = (c == 0) ? lo : lo + (int64_t)(c - 1) * step + 1;
    const int64_t nhi = (c == 32) ? hi : min(hi, lo + (int64_t)c * step);
    lo = nlo;
    hi = nhi;
  }
  const int64_t q = lo + lane;
  const unsigned m = __ballot_sync(0xffffffffu, (q < hi) && ((int)__ldg(ring + q) < v));
  const int c = (~m == 0u) ? 32 : __ffs(~m) - 1;
  return min(hi, lo + c);
}

// Same definition as k_bin_points: r and step of one point.
// The step is rint(phi*S/2pi) of the fp64 phi; a float atan2 of the (exact,
// float) inputs decides it whenever phi*S/2pi is clearly away from a
// half-integer (its error is < 1e-5 rad, far inside the guard), otherwise the
// fp64 formula runs -- the result is the fp64 formula's either way.
// atan2 from one reciprocal and a degree-9 odd minimax polynomial for atan on
// [0, 1] (Abramowitz & Stegun 4.4.49, |error| <= 1e-5 rad) plus octant
// reduction; float rounding adds < 2e-7 rad.  Only used to pick the azimuth
// step away from half-step boundaries (see the guard in bin_xyz).
__device__ __forceinline__ float fast_atan2(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  const float a = mx > 0.0f ? __fdividef(mn, mx) : 0.0f;
  const float s = a * a;
  float r = fmaf(fmaf(fmaf(fmaf(0.0208351f, s, -0.0851330f), s, 0.1801410f), s, -0.3302995f), s, 0.9998660f) * a;
  if (ay > ax) r = 1.57079637f - r;
  if (x < 0.0f) r = 3.14159274f - r;
  return y < 0.0f ? -r : r;
}

__device__ __forceinline__ bool bin_xyz(const lseg_sensor& sn, float xf, float yf, float zf, double& r, int& step) {
  const double x = (double)xf, y = (double)yf, z = (double)zf;
  // squares of float inputs are exact and their sum is 0 or >= 2^-298: the
  // branch-free sqrt is exact here (0 gives NaN, rejected like r = 0)
  r = sqrt_pos(__dadd_rn(__dadd_rn(x * x, y * y), z * z));
  if (!in_window(r, sn.r_min, sn.r_max)) return false;
  const float scale = (float)sn.steps * 0.15915494309189535f;  // S / (2 pi)
  float ph = fast_atan2(yf, xf);  // |error| <= 1.2e-5 rad
  if (ph < 0.0f) ph += 6.283185307179586f;
  const float t = ph * scale;
  const float fr = t - floorf(t);
  // guard: 2x the angle error in step units + float rounding of t
  if (fabsf(fr - 0.5f) > 1e-3f + 2.6e-5f * scale) {
    int st = (int)rintf(t);
    step = st >= sn.steps ? st - sn.steps : st;
    return true;
  }
  double phi = atan2(y, x);
  if (phi < 0.0) phi = __dadd_rn(phi, kTwoPiF);
  step = (int)rint(__ddiv_rn(__dmul_rn(phi, (double)sn.steps), kTwoPiF)) % sn.steps;
  return true;
}

__device__ __forceinline__ bool bin_one(const lseg_sensor& sn, const float* __restrict__ xyz, int64_t p, double& r,
                                        int& step) {
  return bin_xyz(sn, __ldg(xyz + 3 * p), __ldg(xyz + 3 * p + 1), __ldg(xyz + 3 * p + 2), r, step);
}

// Fast path for ring-major input (the sensor's firing order): one CTA per
// (frame, ring) bins that ring's points into a shared-memory row with 64-bit
// shared atomics, then writes the f64 row and the kept-cell valid bits once
// (no memset, no global atomics).  The CTA verifies that its binary-searched
// segment really holds only its ring (and ring 0 / R-1 check the prefix /
// suffix), so any other input order flips the frame to the generic path.
template <int T, typename RT, bool RINGS = true>
__global__ void __launch_bounds__(T, LSEG_BIN_MINB) k_bin_rows(lseg_sensor sn, Shape sh, const float* __restrict__ xyz,
                                                const RT* __restrict__ ring, const int64_t* __restrict__ off,
                                                const int64_t* __restrict__ seg, double* __restrict__ ranges,
                                                uint32_t* __restrict__ vbits, uint32_t* __restrict__ fbits,
                                                int32_t* __restrict__ fallback) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ unsigned long long s_cell[];
  __shared__ int s_bad;
  const int64_t row = blockIdx.x;
  const int f = (int)(row / sh.R), i = (int)(row - (int64_t)f * sh.R);
  const int S = sh.S;
  const int64_t p0 = __ldg(off + f), p1 = __ldg(off + f + 1);
  const int64_t lo = __ldg(seg + f * (sh.R + 1) + i);
  int64_t hi = __ldg(seg + f * (sh.R + 1) + i + 1);
  if (!RINGS) hi = max(hi, lo);  // caller-given segments: nothing to verify against
  for (int s = threadIdx.x; s < S; s += T) s_cell[s] = ~0ull;
  if (threadIdx.x == 0) s_bad = (hi < lo) ? 1 : 0;
  __syncthreads();
  int bad = 0;
  // batches of B points per thread: all loads of a batch are issued first
  constexpr int B = LSEG_BIN_B;
  for (int64_t base = lo; base < hi; base += (int64_t)T * B) {
    float px[B], py[B], pz[B];
    int pr[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int64_t p = base + threadIdx.x + (int64_t)j * T;
      pr[j] = i;
      px[j] = py[j] = pz[j] = 0.0f;
      if (p < hi) {
        if (RINGS) pr[j] = (int)__ldg(ring + p);
        px[j] = __ldg(xyz + 3 * p);
        py[j] = __ldg(xyz + 3 * p + 1);
        pz[j] = __ldg(xyz + 3 * p + 2);
      }
    }
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int64_t p = base + threadIdx.x + (int64_t)j * T;
      if (p >= hi) break;
      if (pr[j] != i) { bad = 1; continue; }
      double r;
      int st;
      if (bin_xyz(sn, px[j], py[j], pz[j], r, st)) atomicMin(s_cell + st, (unsigned long long)__double_as_longlong(r));
    }
  }
  if (RINGS && i == 0)
    for (int64_t p = p0 + threadIdx.x; p < lo; p += T) bad |= ((int)__ldg(ring + p) >= 0) ? 1 : 0;
  if (RINGS && i == sh.R - 1)
    for (int64_t p = hi + threadIdx.x; p < p1; p += T) bad |= ((int)__ldg(ring + p) < sh.R) ? 1 : 0;
  if (bad) s_bad = 1;
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) atomicExch(fallback + f, 1);
    return;
  }
  double* out = ranges + row * S;
  uint32_t* vbr = vbits + row * sh.Wk;
  asm volatile("" : "+l"(out), "+l"(vbr));  // row bases opaque: 32-bit offsets
  const int lane = threadIdx.x & 31;
  // every binned range passed the window test in bin_xyz: a cell is valid
  // iff it received a point (the empty pattern ~0 is a NaN)
  if (sh.k == 1) {  // row out + valid bits in one pass (kept cells = cells)
    for (int w = threadIdx.x >> 5; w < sh.Wk; w += T / 32) {
      const int c = w * 32 + lane;
      const unsigned long long v = c < S ? s_cell[c] : ~0ull;
      if (c < S) out[c] = __longlong_as_double((long long)v);
      const uint32_t b = __ballot_sync(0xffffffffu, v != ~0ull);
      if (lane == 0) vbr[w] = b;
    }
    return;
  }
  {  // row out + full-resolution valid bits (the backfill's target test) in one pass
    const int Wf = (S + 31) / 32;
    for (int w = threadIdx.x >> 5; w < Wf; w += T / 32) {
      const int c = w * 32 + lane;
      const unsigned long long v = c < S ? s_cell[c] : ~0ull;
      if (c < S) out[c] = __longlong_as_double((long long)v);
      const uint32_t b = __ballot_sync(0xffffffffu, v != ~0ull);
      if (fbits && lane == 0) fbits[row * Wf + w] = b;
    }
  }
  for (int w = threadIdx.x >> 5; w < sh.Wk; w += T / 32) {
    const int c = w * 32 + lane;
    const bool v = (c < sh.Sk) && s_cell[c * sh.k] != ~0ull;
    const uint32_t b = __ballot_sync(0xffffffffu, v);
    if (lane == 0) vbits[row * sh.Wk + w] = b;
  }
}

// Ring segment bounds of ring-major input: seg[f][i] = first point of frame f
// with ring >= i, i = 0..R, one warp per entry (32-ary search).
template <typename RT>
__global__ void k_ring_bounds(Shape sh, const RT* __restrict__ ring, const int64_t* __restrict__ off,
                             int64_t* __restrict__ seg) {
  pdl_trigger();
  pdl_wait();
  const int f = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);  // one warp per bound
  if (i > sh.R) return;
  const int64_t b = warp_lower_bound(ring, __ldg(off + f), __ldg(off + f + 1), i, lane);
  if (lane == 0) seg[(int64_t)f * (sh.R + 1) + i] = b;
}

// After k_bin_rows, one CTA per frame: a frame that k_bin_rows flagged (not
// ring-major) is re-binned here by the generic path (reset, then global
// atomics over its points -- the rare case), then the kept-cell valid bits
// are scanned into node ids (the work of k_frame_scan).  One launch instead
// of three on the common path.
template <int T, int ITEMS, typename RT>
__global__ void __launch_bounds__(T) k_bin_finish(lseg_sensor sn, Shape sh, const float* __restrict__ xyz,
                                                  const RT* __restrict__ ring, const int64_t* __restrict__ off,
                                                  const int32_t* __restrict__ fallback, double* __restrict__ ranges,
                                                  uint32_t* __restrict__ vbits, uint32_t* __restrict__ fbits,
                                                  int32_t* __restrict__ wpre, int32_t* __restrict__ n_nodes) {
  pdl_trigger();
  pdl_wait();
  const int f = blockIdx.x;
  if (ring && fallback[f]) {
    const int Wf = (sh.S + 31) / 32;
    for (int64_t q = threadIdx.x; q < (int64_t)sh.R * sh.S; q += T)
      ranges[(int64_t)f * sh.R * sh.S + q] = __longlong_as_double(~0ll);
    for (int q = threadIdx.x; q < sh.R * sh.Wk; q += T) vbits[(int64_t)f * sh.R * sh.Wk + q] = 0u;
    for (int q = threadIdx.x; q < sh.R * Wf; q += T) fbits[(int64_t)f * sh.R * Wf + q] = 0u;
    __syncthreads();
    const int64_t p0 = __ldg(off + f), p1 = __ldg(off + f + 1);
    for (int64_t p = p0 + threadIdx.x; p < p1; p += T) {
      const int rg = (int)__ldg(ring + p);
      double r;
      int stp;
      if (rg < 0 || rg >= sh.R || !bin_one(sn, xyz, p, r, stp)) continue;
      const int64_t row = (int64_t)f * sh.R + rg;
      atomicMin(reinterpret_cast<unsigned long long*>(ranges + row * sh.S + stp),
                (unsigned long long)__double_as_longlong(r));
      if (stp % sh.k == 0) atomicOr(vbits + row * sh.Wk + (stp / sh.k >> 5), 1u << ((stp / sh.k) & 31));
      atomicOr(fbits + row * Wf + (stp >> 5), 1u << (stp & 31));
    }
    __syncthreads();
  }
  // valid-bit word prefix -> node ids (as k_frame_scan)
  using Scan = cub::BlockScan<int, T>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  const int64_t n = (int64_t)sh.R * sh.Wk;
  const uint32_t* vb = vbits + f * n;
  int32_t* wp = wpre + f * n;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += (int64_t)T * ITEMS) {
    int v[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const int64_t idx = base + (int64_t)threadIdx.x * ITEMS + j;
      v[j] = idx < n ? __popc(vb[idx]) : 0;
    }
    int total;
    Scan(tmp).ExclusiveSum(v, v, total);
    const int c0 = carry;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const int64_t idx = base + (int64_t)threadIdx.x * ITEMS + j;
      if (idx < n) wp[idx] = c0 + v[j];
    }
    __syncthreads();
    if (threadIdx.x == 0) carry = c0 + total;
    __syncthreads();
  }
  if (threadIdx.x == 0) n_nodes[f] = carry;
}

template <typename RT>
static void bin_fused_t(const lseg_sensor& sn, const Shape& sh, const float* xyz, const RT* ring, const int64_t* off,
                        const Workspace& ws, double* ranges, cudaStream_t st) {
  cudaMemsetAsync(ws.fallback, 0, sizeof(int32_t) * sh.F, st);
  const size_t smem = sizeof(unsigned long long) * sh.S;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_bin_rows<256, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_pdl(k_ring_bounds<RT>, dim3((sh.R + 1 + 7) / 8, sh.F), 256, 0, st, sh, ring, off, ws.seg);
  launch_pdl(k_bin_rows<256, RT>, sh.F * sh.R, 256, smem, st, sn, sh, xyz, ring, off, ws.seg, ranges, ws.vbits, ws.fbits,
                                                     ws.fallback);
  prof_mark("bin_rows", st);
}

// Ring-major points whose per-frame ring segments the caller passes
// ((F, R+1) absolute point offsets) instead of a ring id per point: no bounds
// search, no verification, no generic path.
static void bin_fused_seg(const lseg_sensor& sn, const Shape& sh, const float* xyz, const int64_t* segs,
                          const int64_t* off, const Workspace& ws, double* ranges, cudaStream_t st) {
  const size_t smem = sizeof(unsigned long long) * sh.S;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_bin_rows<256, uint8_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_pdl(k_bin_rows<256, uint8_t, false>, sh.F * sh.R, 256, smem, st, sn, sh, xyz, nullptr, off, segs, ranges, ws.vbits,
                                                                  ws.fbits, ws.fallback);
  prof_mark("bin_rows", st);
}

void launch_bin_fused(const lseg_sensor& sn, const Shape& sh, const float* xyz, const void* ring, int ring_bytes,
                      const int64_t* off, const Workspace& ws, double* ranges, int32_t* n_nodes, cudaStream_t st) {
  if (ring_bytes == 0) {  // caller-given ring segments: nothing can fall back
    bin_fused_seg(sn, sh, xyz, static_cast<const int64_t*>(ring), off, ws, ranges, st);
    launch_pdl(k_bin_finish<1024, 4, uint8_t>, sh.F, 1024, 0, st, sn, sh, xyz, nullptr, off, ws.fallback, ranges, ws.vbits,
                                                          ws.fbits, ws.wpre, n_nodes);
  } else if (ring_bytes == 1) {
    const uint8_t* r8 = static_cast<const uint8_t*>(ring);
    bin_fused_t(sn, sh, xyz, r8, off, ws, ranges, st);
    launch_pdl(k_bin_finish<1024, 4, uint8_t>, sh.F, 1024, 0, st, sn, sh, xyz, r8, off, ws.fallback, ranges, ws.vbits,
                                                          ws.fbits, ws.wpre, n_nodes);
  } else {
    const int32_t* r32 = static_cast<const int32_t*>(ring);
    bin_fused_t(sn, sh, xyz, r32, off, ws, ranges, st);
    launch_pdl(k_bin_finish<1024, 4, int32_t>, sh.F, 1024, 0, st, sn, sh, xyz, r32, off, ws.fallback, ranges, ws.vbits,
                                                          ws.fbits, ws.wpre, n_nodes);
  }
  prof_mark("frame_scan", st);
}

// Dissolve small segments into the nearest surviving ring donor (reference
// segment.py:136-154) and write the final compacted ids, one CTA per ring row,
// in one pass:
//   A  the row's roots survive unless their post-backfill count is below
//      min_size: survivor bits and row-local word prefix (shared memory);
//      the row's survivor count is published in rstat[row] (ready flag);
//   B  row base = the published counts of the frame's earlier rows;
//   C  final id of each of the row's roots (1 + rank among the frame's
//      survivors, -2 = dissolved) into remap[root cell], then a second flag;
//   D  once the earlier rows' ids are published (every label of a row has
//      its root in that row or an earlier one: roots are component minima and
//      donors lie in the same row), each labelled cell reads its root's id
//      and the dissolved cells are filled from the nearest surviving donor.
// Rows are claimed in ticket order, so every earlier row belongs to a CTA
// that is already running; a row waits only for earlier rows' counts before
// publishing its ids, so no wait chain forms and nothing deadlocks.
// rstat and the ticket are zeroed by k_root_flatten.
template <int T>
__global__ void __launch_bounds__(T, LSEG_PRUNE_TSM / T) k_prune_rows(Shape sh, const int32_t* __restrict__ lab_in,
                                                  int32_t* __restrict__ out, const int32_t* __restrict__ hist,
                                                  int64_t K, int32_t min_size, const uint32_t* __restrict__ rbits,
                                                  int32_t* __restrict__ remap, int32_t* __restrict__ rstat,
                                                  int32_t* __restrict__ ticket) {
  pdl_trigger();
  pdl_wait();
  constexpr int NW = T / 32;
  constexpr int kReady = 1 << 30, kIds = 1 << 29;
  extern __shared__ int s_dynrow[];
  const int S = sh.S, nw = (S + 31) / 32;
  int* s_val = s_dynrow;
  uint32_t* s_dm = reinterpret_cast<uint32_t*>(s_dynrow + nw * 32);
  int* s_wc = reinterpret_cast<int*>(s_dm + nw);  // per-word survivor counts -> row-local prefix
  uint32_t* s_sb = reinterpret_cast<uint32_t*>(s_wc + sh.Wk);  // survivor bits of the row
  short* s_pw = reinterpret_cast<short*>(s_sb + sh.Wk);  // nearest donor word at / before each word (cyclic)
  short* s_nx = s_pw + nw;                              // ... at / after
  uint32_t* s_rbw = reinterpret_cast<uint32_t*>(s_nx + nw);  // the row's root bits (s_pw is 4-B aligned, 2 nw shorts)
  __shared__ int s_any, s_row, s_base, s_part[NW];
  if (threadIdx.x == 0) {
    s_row = atomicAdd(ticket, 1);
    s_any = 0;
  }
  __syncthreads();
  const int row = s_row;
  const int f = fdiv(row, sh.R, sh.inv_R), i = row - f * sh.R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const volatile int32_t* rs = rstat + (int64_t)f * sh.R;
  int32_t* rmf = remap + (int64_t)f * K;
  asm volatile("" : "+l"(rmf));  // frame base opaque: one wide multiply-add per lookup
  // A. survivors of this row's roots, one warp per 32-cell word (the
  // histogram reads of a word are one coalesced load)
  {
    const int32_t* hf = hist + (int64_t)f * K + (int64_t)i * sh.Sk + 1;
    const uint32_t* rbr = rbits + (int64_t)row * sh.Wk;
    asm volatile("" : "+l"(hf), "+l"(rbr));  // row bases opaque: 32-bit offsets, one wide multiply-add each
    // the warp's words are w = warp + NW q: lane q loads word q's root bits,
    // then the histogram reads go out PA words at a time (3 dependent loads
    // per 32 words instead of 2 per word)
    constexpr int PA = 4;
    for (int wb = warp; wb < sh.Wk; wb += NW * 32) {
      const int wl = wb + lane * NW;
      const uint32_t rbl = wl < sh.Wk ? __ldg(rbr + wl) : 0u;
      if (wl < sh.Wk) s_rbw[wl] = rbl;
      for (int q0 = 0; q0 < 32 && wb + q0 * NW < sh.Wk; q0 += PA) {
        uint32_t rq[PA];
        int hv[PA];
#pragma unroll
        for (int j = 0; j < PA; ++j) {
          rq[j] = __shfl_sync(0xffffffffu, rbl, q0 + j);
          hv[j] = ((rq[j] >> lane) & 1u) ? __ldcg(hf + (wb + (q0 + j) * NW) * 32 + lane) : 0;
        }
#pragma unroll
        for (int j = 0; j < PA; ++j) {
          const int w = wb + (q0 + j) * NW;
          const bool surv = ((rq[j] >> lane) & 1u) && !((min_size > 0) && (hv[j] < min_size));
          const uint32_t b = __ballot_sync(0xffffffffu, surv);
          if (lane == 0 && w < sh.Wk) {
            s_sb[w] = b;
            s_wc[w] = __popc(b);
          }
        }
      }
    }
    __syncthreads();
    // row-local exclusive prefix over the words: each warp scans a
    // contiguous block of words, then the block totals are offset
    const int per = (sh.Wk + NW - 1) / NW;
    const int w0 = warp * per, w1 = min(sh.Wk, w0 + per);
    int carry = 0;
    for (int c = w0; c < w1; c += 32) {
      const int w = c + lane;
      const int v = (w < w1) ? s_wc[w] : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
      }
      if (w < w1) s_wc[w] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) s_part[warp] = carry;
    __syncthreads();
    int base = 0;
    for (int q = 0; q < warp; ++q) base += s_part[q];
    for (int w = w0 + lane; w < w1; w += 32) s_wc[w] += base;
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int q = 0; q < NW; ++q) tot += s_part[q];
      atomicExch(rstat + row, kReady | tot);  // only the count: no data behind it
    }
  }
  // B. row base: the published counts of the frame's earlier rows
  if (warp == 0) {
    int sum = 0;
    for (int r = lane; r < i; r += 32) {
      int v;
      while (((v = rs[r]) & kReady) == 0) {
      }
      sum += v & (kIds - 1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) s_base = sum;
  }
  __syncthreads();
  // C. final ids of this row's roots, then the second flag
  {
    const int base = s_base;
    for (int w = warp; w < sh.Wk; w += NW) {
      const uint32_t rb = s_rbw[w];
      if ((rb >> lane) & 1u) {
        const uint32_t sb = s_sb[w], bit = 1u << lane;
        rmf[i * sh.Sk + w * 32 + lane] = (sb & bit) ? 1 + base + s_wc[w] + __popc(sb & (bit - 1u)) : -2;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();  // this row's ids before its flag
      atomicOr(rstat + row, kIds);
    }
  }
  // D. wait for the earlier rows' ids, then pass 1: each labelled cell's
  // root id (L2 loads: written by other CTAs of this launch) -- dissolved
  // -> target (-2), survivor -> its final id, so the fill only copies ids
  if (warp == 0) {
    for (int r = lane; r < i; r += 32)
      while ((rs[r] & kIds) == 0) {
      }
    __threadfence();  // acquire: the earlier rows' ids
  }
  __syncthreads();
  const int64_t rb = (int64_t)row * S;
  const int32_t* lin = lab_in + rb;
  asm volatile("" : "+l"(lin));
  bool any = false;
  constexpr int PF = LSEG_PF_PRUNE;
  for (int s0 = 0; s0 < nw * 32; s0 += T * PF) {
    int lv[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) {
      const int s = s0 + threadIdx.x + j * T;
      lv[j] = (s < S) ? __ldcg(lin + s) : 0;
    }
#pragma unroll
    for (int j = 0; j < PF; ++j) lv[j] = lv[j] > 0 ? __ldcg(rmf + lv[j] - 1) : 0;
#pragma unroll
    for (int j = 0; j < PF; ++j) {
      const int s = s0 + threadIdx.x + j * T;
      if (s >= nw * 32) break;
      s_val[s] = lv[j];
      const uint32_t dm = __ballot_sync(0xffffffffu, lv[j] > 0);
      if ((s & 31) == 0) s_dm[s >> 5] = dm;
      any |= dm != 0;
    }
  }
  if (any && lane == 0) s_any = 1;
  __syncthreads();
  const bool rany = s_any != 0;
  if (rany) {
    // donor-word tables (one warp): running max / min of donor word indices,
    // entries before the first / after the last donor word wrap around
    if (warp == 0) {
      int carry = -1;
      for (int c0 = 0; c0 < nw; c0 += 32) {
        const int w = c0 + lane;
        int x = (w < nw && s_dm[w]) ? w : -1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) x = max(x, __shfl_up_sync(0xffffffffu, x, o));
        x = max(x, carry);
        if (w < nw) s_pw[w] = (short)x;
        carry = __shfl_sync(0xffffffffu, x, 31);
      }
      const int last = carry;
      carry = 0x7fffffff;
      for (int c0 = ((nw - 1) & ~31); c0 >= 0; c0 -= 32) {
        const int w = c0 + 31 - lane;  // lane 0 holds the highest word of the chunk
        int x = (w < nw && s_dm[w]) ? w : 0x7fffffff;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) x = min(x, __shfl_up_sync(0xffffffffu, x, o));
        x = min(x, carry);
        if (w < nw) s_nx[w] = (short)(x == 0x7fffffff ? -1 : x);
        carry = __shfl_sync(0xffffffffu, x, 31);
      }
      const int first = carry;
      __syncwarp();
      for (int w = lane; w < nw; w += 32) {
        if (s_pw[w] < 0) s_pw[w] = (short)last;
        if (s_nx[w] < 0) s_nx[w] = (short)first;
      }
    }
    __syncthreads();
  }
  for (int s = threadIdx.x; s < S; s += T) {
    const int v = s_val[s];
    out[rb + s] = v != -2 ? (v > 0 ? v : 0) : (rany ? s_val[nearest_donor_tab(s_dm, s_pw, s_nx, nw, S, s)] : 0);
  }
}

void launch_prune_fused(const Shape& sh, const Workspace& ws, int32_t min_size, int32_t* labels, cudaStream_t st) {
  // 128-thread CTAs (16 per SM) for throughput; one-wave batches (single
  // scans) use 256 threads per row to cut the per-row latency
  const bool wide = (int64_t)sh.F * sh.R < num_sms() * 8;
  const int nwr = (sh.S + 31) / 32;
  const size_t smem = sizeof(int) * ((size_t)nwr * 33 + 3 * (size_t)sh.Wk) + sizeof(short) * 2 * ((size_t)nwr + 1);
  if (smem > 48 * 1024)
    for (auto fn : {k_prune_rows<128>, k_prune_rows<256>})
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (wide)
    launch_pdl(k_prune_rows<256>, sh.F * sh.R, 256, smem, st, sh, ws.lab_tmp, labels, ws.hist, ws.K, min_size, ws.rbits,
                                                      ws.remap, ws.rcnt, ws.fscal + 3);
  else
    launch_pdl(k_prune_rows<128>, sh.F * sh.R, 128, smem, st, sh, ws.lab_tmp, labels, ws.hist, ws.K, min_size, ws.rbits,
                                                      ws.remap, ws.rcnt, ws.fscal + 3);
  prof_mark("prune_apply", st);
}

// ---------------------------------------------------------------- launchers
void debug_phases(double* out) {
#if LSEG_PHASES
  unsigned long long h[8];
  cudaMemcpyFromSymbol(h, g_ph, sizeof(h));
  for (int i = 0; i < 8; ++i) out[i] = (double)h[i];
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(g_ph, z, sizeof(z));
#else
  for (int i = 0; i < 8; ++i) out[i] = -1.0;
#endif
}
void launch_fused_graph(const lseg_sensor& sn, const Shape& sh, const Workspace& ws, const double* ranges,
                        const double* thr, int32_t* node_ids, int32_t* neighbors, float* n32, uint8_t* nmask,
                        int32_t* n_nodes, int32_t* n_labels, int32_t* node_labels, bool fbits_valid,
                        bool exact_normals, float* dbg_err, cudaStream_t st, double* n64, int32_t* node_rc) {
  const int tilesC = (sh.Sk + TILE_C - 1) / TILE_C, tilesR = (sh.R + TILE_R - 1) / TILE_R;
  const int64_t nt = (int64_t)sh.F * tilesR * tilesC;
  const dim3 tgrid(tilesC, tilesR, sh.F);  // frames <= 65535 (check_shape)
  const int per = tilesR * sh.Sk + tilesC * sh.R;
  const int mt = sh.F < 8 ? 64 : LSEG_MERGE_T;  // border-merge threads per CTA (more CTAs for single scans)
  if (!exact_normals) {
    CertParams cp;
    for (int c = 0; c < 3; ++c) {
      cp.t[c] = thr[c];
      cp.tf[c] = (float)thr[c];
      cp.mt[c] = 5.9604645e-08f * (8.0f + 4.0f * (float)thr[c]);
    }
    cp.deg2 = 1e-30f;  // |V| < 1e-15: fp32 squares would leave the normal range
    constexpr int NH = (TILE_R + 2) * (TILE_C + 2), NT = TILE_R * TILE_C;
    const size_t csmem = (size_t)NH * (3 * 8 + 4) + (size_t)NT * (3 * 4 + 2 + 2 + 2 + 3);  // see k_tile_cert
    // per launch: cheap, and correct for every device / thread (a static
    // "done" flag would not be)
    cudaFuncSetAttribute(k_tile_cert<TILE_R, TILE_C, TILE_T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)csmem);
    float4* bn4 = reinterpret_cast<float4*>(ws.bnorm);
    launch_pdl(k_tile_cert<TILE_R, TILE_C, TILE_T>, tgrid, TILE_T, csmem, st, 
        sn, sh, ranges, ws.vbits, ws.wpre, cp, node_ids, neighbors, n32, nmask, ws.masks, bn4, ws.normals64, dbg_err,
        ws.fscal, n_labels);
    prof_mark("tile", st);
    if (nt < num_sms() * 16)  // one-wave batches: 256 threads per tile for latency
      launch_pdl(k_tile_cc<TILE_R, TILE_C, 256>, tgrid, 256, 0, st, sh, ws.masks, ws.parent, ws.lroots, ws.hist, ws.K);
    else
      launch_pdl(k_tile_cc<TILE_R, TILE_C, LSEG_CC_TBIG>, tgrid, LSEG_CC_TBIG, 0, st, sh, ws.masks, ws.parent, ws.lroots, ws.hist, ws.K);
    prof_mark("tile_cc", st);
    launch_pdl(k_merge_cert<TILE_R, TILE_C>, dim3((per + mt - 1) / mt, sh.F), mt, 0, st, sn, sh, ranges, ws.vbits, bn4, cp,
                                                                                ws.parent, ws.rank, ws.fscal);
    launch_pdl(k_merge_exact<TILE_R, TILE_C>, dim3(1, sh.F), 128, 0, st, sn, sh, ranges, ws.vbits, bn4, cp, ws.parent,
                                                                 ws.rank, ws.fscal);
    prof_mark("merge", st);
  } else {
  const size_t tsmem =
      (size_t)((TILE_R + 2) * (TILE_C + 2) + 2 * (TILE_R + 2) + 2 * (TILE_C + 2) + 3 * TILE_R * TILE_C) * 8 +
      (size_t)(TILE_R + 2) * (TILE_C + 2) * 4 + (size_t)TILE_R * TILE_C * 4;
  cudaFuncSetAttribute(k_tile<TILE_R, TILE_C, TILE_T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
  launch_pdl(k_tile<TILE_R, TILE_C, TILE_T>, tgrid, TILE_T, tsmem, st, sn, sh, ranges, ws.vbits, ws.wpre, thr[0], thr[1],
                                                                  thr[2], node_ids, neighbors, n32, nmask, ws.masks,
                                                                  ws.bnorm, ws.parent, ws.lroots, n_labels, n64, node_rc);
  prof_mark("tile", st);
  if (nt < num_sms() * 16)  // one-wave batches: 256 threads per tile for latency
    launch_pdl(k_tile_cc<TILE_R, TILE_C, 256>, tgrid, 256, 0, st, sh, ws.masks, ws.parent, ws.lroots, ws.hist, ws.K);
  else
    launch_pdl(k_tile_cc<TILE_R, TILE_C, LSEG_CC_TBIG>, tgrid, LSEG_CC_TBIG, 0, st, sh, ws.masks, ws.parent, ws.lroots, ws.hist, ws.K);
  prof_mark("tile_cc", st);
  const int mper = sh.F < 8 ? 1 : LSEG_MERGE_PER;  // single scans: one cell per thread (more CTAs in flight)
  launch_pdl(k_merge<TILE_R, TILE_C>, dim3((per + mt * mper - 1) / (mt * mper), sh.F), mt, 0, st, 
      sh, ws.bnorm, thr[0], thr[1], thr[2], ws.parent);
  prof_mark("merge", st);
  }
  const bool fold = !node_labels && LSEG_FOLD_FLATTEN;
  if (!fold) {
    const int ft = (int64_t)sh.F * sh.R < num_sms() * 8 ? 256 : 128;  // one-wave batches: wider CTAs
    const int thr = sh.Wk >= ft / 32 ? ft : 32 * sh.Wk;
    launch_pdl(k_root_flatten, sh.F * sh.R, thr, 0, st, sh, ws.parent, ws.lroots, ws.rbits, ws.hist, ws.K, ws.fscal,
                                                ws.rcnt, n_labels);
    prof_mark("root_flatten", st);
    if (node_labels) {  // frame-level root ranks: only the segment() output needs them
      launch_scan_bits(sh, ws.rbits, ws.rpre, n_labels, nullptr, 0, st);
      prof_mark("root_scan", st);
    }
  }
  // labels + backfill -> lab_tmp (+ histogram)
  const size_t smem = sizeof(int) * (size_t)sh.Wk * 34;
  const uint32_t* fb = (sh.k > 1 && fbits_valid) ? ws.fbits : nullptr;
  const bool wide = (int64_t)sh.F * sh.R < num_sms() * 8;  // one-wave batches: 256 threads per row for latency
  const bool direct = sh.k == 1 && fold;  // (fold implies no segment() output)
  auto kern = wide ? (direct ? k_labels_backfill<256, true> : k_labels_backfill<256, false>)
                   : (direct ? k_labels_backfill<LSEG_LAB_T, true> : k_labels_backfill<LSEG_LAB_T, false>);
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_pdl(kern, sh.F * sh.R, wide ? 256 : LSEG_LAB_T, smem, st, sn, sh, ranges, ws.vbits, fb, ws.parent, ws.rbits, ws.rpre,
             node_labels, ws.lab_tmp, ws.hist, ws.K, fold ? ws.rbits : nullptr, n_labels, ws.rcnt, ws.fscal + 3);
  prof_mark("labels_backfill", st);
}

}  // namespace lseg
