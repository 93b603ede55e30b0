// Fused pipeline kernels (sm_100a): the batched hot path of lseg_run_pipeline.
//
//   k_tile     one CTA per (frame, TR x TC tile of kept cells): stages the
//              ranges halo in shared memory, computes fp64 normals for the tile
//              plus its forward halo, writes the mesh slots / normals, evaluates
//              the homogeneity test on every forward edge and runs union-find
//              in shared memory.  Edges leaving the tile are recorded as flag
//              bits for k_merge.  No fp64 normals ever reach HBM.
//   k_merge    global union-find over the tile-boundary edges only.
//   k_labels_backfill  per ring row: node label = 1 + rank[root] (read-only
//              root chase), then the nearest-donor backfill and the label
//              histogram, in one pass (replaces label_dense + backfill).
#include <cub/block/block_scan.cuh>
#include <stdlib.h>

#include "lseg_internal.cuh"
#include "lseg_kernels.cuh"

namespace lseg {

static constexpr int TILE_R = 16;
static constexpr int TILE_C = 64;
static constexpr int TILE_T = 256;

__device__ __forceinline__ int wrapc(int c, int Sk) { return c < 0 ? c + Sk : (c >= Sk ? c - Sk : c); }

__device__ __forceinline__ int id_at(const uint32_t* vbf, const int32_t* wpf, int Wk, int r, int c) {
  return node_id_at(vbf + (int64_t)r * Wk, wpf + (int64_t)r * Wk, c);
}

// local (shared-memory) union-find, same min-root invariant as the global one
__device__ __forceinline__ int lfind(volatile int* par, int x) {
  int p = par[x];
  while (p != x) {
    const int g = par[p];
    if (g != p) par[x] = g;  // halving
    x = p;
    p = g;
  }
  return x;
}

__device__ __forceinline__ void lunion(int* par, int a, int b) {
  volatile int* vp = par;
  int ra = lfind(vp, a), rb = lfind(vp, b);
  while (ra != rb) {
    if (ra < rb) { const int t = ra; ra = rb; rb = t; }
    const int old = atomicCAS(par + ra, ra, rb);
    if (old == ra) break;
    ra = lfind(vp, old);
    rb = lfind(vp, rb);
  }
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

// Normal of a node whose 6 slots are all present: the same operation sequence
// as Fan (pairs (0,1)..(4,5),(5,0) accumulated in order) but straight-line, so
// the six square roots / reciprocals are independent and can overlap.
__device__ __forceinline__ bool fan6(const double* vx, const double* vy, const double* vz, const Vec3& p,
                                     double out[3]) {
  double l[6];
#pragma unroll
  for (int a = 0; a < 6; ++a) l[a] = norm3(vx[a], vy[a], vz[a]);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, ws = 0.0;
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    const int b = (a + 1) % 6;
    const double L = __dadd_rn(l[a], l[b]);
    const double w = (L > 0.0) ? __drcp_rn(L) : 0.0;
    a0 = __dadd_rn(a0, __dmul_rn(w, __dsub_rn(__dmul_rn(vy[a], vz[b]), __dmul_rn(vz[a], vy[b]))));
    a1 = __dadd_rn(a1, __dmul_rn(w, __dsub_rn(__dmul_rn(vz[a], vx[b]), __dmul_rn(vx[a], vz[b]))));
    a2 = __dadd_rn(a2, __dmul_rn(w, __dsub_rn(__dmul_rn(vx[a], vy[b]), __dmul_rn(vy[a], vx[b]))));
    ws = __dadd_rn(ws, w);
  }
  if (!(ws > 0.0)) return false;
  const double m0 = __ddiv_rn(a0, ws), m1 = __ddiv_rn(a1, ws), m2 = __ddiv_rn(a2, ws);
  const double mag = norm3(m0, m1, m2);
  if (!(mag >= 1e-12)) return false;
  double u0 = __ddiv_rn(m0, mag), u1 = __ddiv_rn(m1, mag), u2 = __ddiv_rn(m2, mag);
  const double dot = __dadd_rn(__dadd_rn(__dmul_rn(u0, p.x), __dmul_rn(u2, p.z)), __dmul_rn(u1, p.y));
  if (dot > 0.0) { u0 = -u0; u1 = -u1; u2 = -u2; }
  out[0] = u0; out[1] = u1; out[2] = u2;
  return true;
}

// One CTA per (frame, TR x TC tile of kept cells).
//   A  ranges + node ids of the tile and a 1-cell halo into shared memory
//   B  fp64 normals of the tile's nodes (shared memory)
//   C  neighbours / normals / mask out; fp64 normals of the tile's border
//      cells to `bnorm` for k_merge
//   D  homogeneity test + shared-memory union-find on internal forward edges
//   E  parent[cell] = tile-local root cell (-1 for cells without a normal)
template <int TR, int TC, int T>
#ifndef LSEG_TILE_MINB
#define LSEG_TILE_MINB 3
#endif
__global__ void __launch_bounds__(T, LSEG_TILE_MINB) k_tile(lseg_sensor sn, Shape sh, const double* __restrict__ ranges,
                                                const uint32_t* __restrict__ vbits, const int32_t* __restrict__ wpre,
                                                double t0, double t1, double t2, int32_t* __restrict__ node_ids,
                                                int32_t* __restrict__ neighbors, float* __restrict__ n32,
                                                uint8_t* __restrict__ nmask, unsigned long long* __restrict__ masks,
                                                double* __restrict__ bnorm) {
  constexpr int GR = TR + 2, GC = TC + 2;  // halo rows r0-1..r0+TR, cols c0-1..c0+TC
  constexpr int NT = TR * TC;
  // dynamic shared memory (58 KB > the 48 KB static limit), see tile_smem_bytes()
  extern __shared__ __align__(16) unsigned char s_dyn[];
  double* s_px = reinterpret_cast<double*>(s_dyn);
  double* s_py = s_px + GR * GC;
  double* s_pz = s_py + GR * GC;
  double* s_nx = s_pz + GR * GC;
  double* s_ny = s_nx + NT;
  double* s_nz = s_ny + NT;
  int* s_id = reinterpret_cast<int*>(s_nz + NT);
  unsigned short* s_list = reinterpret_cast<unsigned short*>(s_id + GR * GC);  // fan6 list from the front, rest from the back
  uint8_t* s_has = reinterpret_cast<uint8_t*>(s_list + NT);
  uint8_t* s_m = s_has + NT;  // presence mask of general-path nodes

  const int tilesC = (sh.Sk + TC - 1) / TC;
  const int tilesR = (sh.R + TR - 1) / TR;
  const int64_t b = blockIdx.x;
  const int f = (int)(b / ((int64_t)tilesR * tilesC));
  const int rem = (int)(b - (int64_t)f * tilesR * tilesC);
  const int r0 = (rem / tilesC) * TR, c0 = (rem % tilesC) * TC;
  const int TRe = min(TR, sh.R - r0), TCe = min(TC, sh.Sk - c0);
  const double* rf = ranges + (int64_t)f * sh.R * sh.S;
  const uint32_t* vbf = vbits + (int64_t)f * sh.R * sh.Wk;
  const int32_t* wpf = wpre + (int64_t)f * sh.R * sh.Wk;
  const int64_t nbase = (int64_t)f * sh.cap;
  const int tid = threadIdx.x;

  // A. halo positions dir*r (reference product order) and node ids (-1 absent)
  for (int e = tid; e < GR * GC; e += T) {
    const int y = e / GC, x = e - y * GC;
    const int rr = r0 - 1 + y;
    Vec3 q = {0.0, 0.0, 0.0};
    int id = -1;
    if (rr >= 0 && rr < sh.R) {
      const int cc = wrapc(c0 - 1 + x, sh.Sk);
      id = id_at(vbf, wpf, sh.Wk, rr, cc);
      if (id >= 0) q = cell_pos(sn, rr, cc * sh.k, __ldg(rf + (int64_t)rr * sh.S + (int64_t)cc * sh.k));
    }
    s_px[e] = q.x;
    s_py[e] = q.y;
    s_pz[e] = q.z;
    s_id[e] = id;
  }
  __syncthreads();

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
      if (e < NT && y < TRe && x < TCe && s_id[g] >= 0) {
#pragma unroll
        for (int s = 0; s < 6; ++s)
          if (s_id[g + slot_dr(s) * GC + slot_dc(s)] >= 0 && !(s == 5 && sh.Sk == 2)) m |= 1u << s;  // mesh.py:96-101
        kind[j] = (m == 0x3fu) ? 1 : 2;
      }
      ml[j] = (unsigned char)m;
      na += kind[j] == 1;
      nb += kind[j] == 2;
      if (e < NT) { s_has[e] = 0; s_nx[e] = s_ny[e] = s_nz[e] = 0.0; }
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
  const int nfan6 = s_cnt[2 * (T / 32)], ngen = s_cnt[2 * (T / 32) + 1];
  for (int i = tid; i < nfan6; i += T) {
    const int e = s_list[i];
    const int y = e / TC, x = e - y * TC;
    const int g = (y + 1) * GC + (x + 1);
    const Vec3 p = {s_px[g], s_py[g], s_pz[g]};
    double vx[6], vy[6], vz[6], nv[3];
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int gq = g + slot_dr(s) * GC + slot_dc(s);
      vx[s] = __dsub_rn(s_px[gq], p.x);
      vy[s] = __dsub_rn(s_py[gq], p.y);
      vz[s] = __dsub_rn(s_pz[gq], p.z);
    }
    if (fan6(vx, vy, vz, p, nv)) {
      s_nx[e] = nv[0];
      s_ny[e] = nv[1];
      s_nz[e] = nv[2];
      s_has[e] = 1;
    }
  }
  for (int i = tid; i < ngen; i += T) {
    const int e = s_list[NT - 1 - i];
    const int y = e / TC, x = e - y * TC;
    const int g = (y + 1) * GC + (x + 1);
    const unsigned m = s_m[e];
    const Vec3 p = {s_px[g], s_py[g], s_pz[g]};
    Fan fan;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      if (!((m >> s) & 1u)) continue;
      const int gq = g + slot_dr(s) * GC + slot_dc(s);
      fan.add(__dsub_rn(s_px[gq], p.x), __dsub_rn(s_py[gq], p.y), __dsub_rn(s_pz[gq], p.z));
    }
    double nv[3];
    if (fan.finish(p, nv)) {
      s_nx[e] = nv[0];
      s_ny[e] = nv[1];
      s_nz[e] = nv[2];
      s_has[e] = 1;
    }
  }
  __syncthreads();

  // C. per-node outputs
  for (int e = tid; e < NT; e += T) {
    const int y = e / TC, x = e - y * TC;
    if (y >= TRe || x >= TCe) continue;
    const int rr = r0 + y, cc = c0 + x;
    const int g = (y + 1) * GC + (x + 1);
    const int id = s_id[g];
    const int64_t cell = (int64_t)rr * sh.Sk + cc;
    if (node_ids) node_ids[nbase + cell] = id;
    if (id < 0) continue;
    int nb[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) nb[s] = s_id[g + slot_dr(s) * GC + slot_dc(s)];
    if (sh.Sk == 2 && nb[5] == nb[2]) nb[5] = -1;
    int2* o2 = reinterpret_cast<int2*>(neighbors + (nbase + id) * 6);  // 24 B rows, 8-B aligned
    o2[0] = make_int2(nb[0], nb[1]);
    o2[1] = make_int2(nb[2], nb[3]);
    o2[2] = make_int2(nb[4], nb[5]);
    const bool has = s_has[e];
    if (n32) {
      float* o = n32 + (nbase + id) * 3;
      const float qn = __int_as_float(0x7fc00000);
      o[0] = has ? (float)s_nx[e] : qn;
      o[1] = has ? (float)s_ny[e] : qn;
      o[2] = has ? (float)s_nz[e] : qn;
    }
    nmask[nbase + id] = has ? 1 : 0;
    if (has && (y == 0 || y == TRe - 1 || x == 0 || x == TCe - 1)) {
      double* o = bnorm + (nbase + cell) * 3;
      o[0] = s_nx[e];
      o[1] = s_ny[e];
      o[2] = s_nz[e];
    }
  }

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
  for (int y = tid >> 5; y < TR; y += T / 32) {
    unsigned long long H = 0, V0 = 0, V1 = 0, HS = 0;
    bool w0 = false, w1 = false;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int x = lane + 32 * half;
      const int e = y * TC + x;
      bool h = false, v0 = false, v1 = false;
      const bool has = (y < TRe) && s_has[e];
      if (has) {
        const double a[3] = {s_nx[e], s_ny[e], s_nz[e]};
        if (x + 1 < TCe && s_has[e + 1]) {
          const double q[3] = {s_nx[e + 1], s_ny[e + 1], s_nz[e + 1]};
          h = normals_pass(a, q, t0, t1, t2);
        }
        if (y + 1 < TRe) {
          if (s_has[e + TC]) {
            const double q[3] = {s_nx[e + TC], s_ny[e + TC], s_nz[e + TC]};
            v0 = normals_pass(a, q, t0, t1, t2);
          }
          if (x + 1 < TCe && s_has[e + TC + 1]) {
            const double q[3] = {s_nx[e + TC + 1], s_ny[e + TC + 1], s_nz[e + TC + 1]};
            v1 = normals_pass(a, q, t0, t1, t2);
          }
        }
        if (full_width && x == TCe - 1) {
          const int e0 = y * TC;  // (y, 0)
          if (TCe > 1 && s_has[e0]) {
            const double q[3] = {s_nx[e0], s_ny[e0], s_nz[e0]};
            w0 = normals_pass(a, q, t0, t1, t2);
          }
          if (y + 1 < TRe && s_has[e0 + TC]) {
            const double q[3] = {s_nx[e0 + TC], s_ny[e0 + TC], s_nz[e0 + TC]};
            w1 = normals_pass(a, q, t0, t1, t2);
          }
        }
      }
      const unsigned long long sh_ = half ? 32 : 0;
      H |= (unsigned long long)__ballot_sync(0xffffffffu, h) << sh_;
      V0 |= (unsigned long long)__ballot_sync(0xffffffffu, v0) << sh_;
      V1 |= (unsigned long long)__ballot_sync(0xffffffffu, v1) << sh_;
      HS |= (unsigned long long)__ballot_sync(0xffffffffu, has) << sh_;
    }
    const unsigned W = (__ballot_sync(0xffffffffu, w0) ? 1u : 0u) | (__ballot_sync(0xffffffffu, w1) ? 2u : 0u);
    if (lane == 0) {
      mrow[y * 5 + 0] = H;
      mrow[y * 5 + 1] = V0;
      mrow[y * 5 + 2] = V1;
      mrow[y * 5 + 3] = HS;
      mrow[y * 5 + 4] = W;
    }
  }
}

// Tile-local connected components from k_tile's masks (one small CTA per
// tile): each node's parent starts as the first cell of its horizontal run
// (bit arithmetic), vertical / diagonal edges join runs with shared-memory
// union-find -- skipping an edge when the parallel edge one column to the left
// already joins the same two runs -- and each labelled cell gets
// parent[cell] = minimum cell of its tile-local component (-1 without normal).
template <int TR, int TC, int T>
__global__ void __launch_bounds__(T) k_tile_cc(Shape sh, const unsigned long long* __restrict__ masks,
                                               int32_t* __restrict__ parent) {
  constexpr int NT = TR * TC;
  __shared__ int s_par[NT];
  __shared__ unsigned long long s_m[TR * 5];
  const int tilesC = (sh.Sk + TC - 1) / TC;
  const int tilesR = (sh.R + TR - 1) / TR;
  const int64_t b = blockIdx.x;
  const int f = (int)(b / ((int64_t)tilesR * tilesC));
  const int rem = (int)(b - (int64_t)f * tilesR * tilesC);
  const int r0 = (rem / tilesC) * TR, c0 = (rem % tilesC) * TC;
  const int TRe = min(TR, sh.R - r0), TCe = min(TC, sh.Sk - c0);
  const unsigned long long* mrow = masks + b * (TR * 5);
  for (int j = threadIdx.x; j < TR * 5; j += T) s_m[j] = __ldg(mrow + j);
  __syncthreads();
  for (int e = threadIdx.x; e < NT; e += T) {
    const int y = e / TC, x = e - y * TC;
    const unsigned long long Z = ~s_m[y * 5] & ((1ull << x) - 1ull);
    s_par[e] = y * TC + (Z ? 64 - __clzll((long long)Z) : 0);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NT; e += T) {
    const int y = e / TC, x = e - y * TC;
    if (y + 1 >= TRe) continue;
    const unsigned long long Hy = s_m[y * 5], V0 = s_m[y * 5 + 1], V1 = s_m[y * 5 + 2];
    const unsigned long long Hn = s_m[(y + 1) * 5];
    const unsigned long long bx = 1ull << x, bl = bx >> 1;
    if (V0 & bx) {
      const bool dup = x > 0 && (Hy & bl) && (Hn & bl) && (V0 & bl);
      if (!dup) lunion(s_par, e, e + TC);
    }
    if (V1 & bx) {
      const bool dup = ((V0 & bx) && (Hn & bx)) || (x > 0 && (Hy & bl) && (Hn & bx) && (V1 & bl));
      if (!dup) lunion(s_par, e, e + TC + 1);
    }
  }
  for (int y = threadIdx.x; y < TRe; y += T) {  // full-width column wrap (x = S'-1 -> 0)
    const unsigned W = (unsigned)s_m[y * 5 + 4];
    if (W & 1u) lunion(s_par, y * TC + TCe - 1, y * TC);
    if (W & 2u) lunion(s_par, y * TC + TCe - 1, (y + 1) * TC);
  }
  __syncthreads();
  const int64_t nbase = (int64_t)f * sh.cap;
  for (int e = threadIdx.x; e < NT; e += T) {
    const int y = e / TC, x = e - y * TC;
    if (y >= TRe || x >= TCe) continue;
    int pc = -1;
    if ((s_m[y * 5 + 3] >> x) & 1ull) {
      const int lr = lfind(s_par, e);
      pc = (r0 + lr / TC) * sh.Sk + c0 + lr % TC;
    }
    parent[nbase + (int64_t)(r0 + y) * sh.Sk + c0 + x] = pc;
  }
}

// Global union over the forward edges that leave a tile.  Threads enumerate
// the cells of each tile's last row and last column (corner duplicates are
// harmless); both endpoints' fp64 normals come from `bnorm`.
template <int TR, int TC>
__global__ void k_merge(Shape sh, const double* __restrict__ bnorm, double t0, double t1, double t2,
                        int32_t* __restrict__ parent) {
  const int nbr = (sh.R + TR - 1) / TR;
  const int nbc = (sh.Sk + TC - 1) / TC;
  const int64_t per = (int64_t)nbr * sh.Sk + (int64_t)nbc * sh.R;
  const int64_t n = per * sh.F;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(t / per);
    int64_t u = t - (int64_t)f * per;
    int r, c;
    if (u < (int64_t)nbr * sh.Sk) {
      const int br = (int)(u / sh.Sk);
      r = min(br * TR + TR - 1, sh.R - 1);
      c = (int)(u - (int64_t)br * sh.Sk);
    } else {
      u -= (int64_t)nbr * sh.Sk;
      const int bc = (int)(u / sh.R);
      c = min(bc * TC + TC - 1, sh.Sk - 1);
      r = (int)(u - (int64_t)bc * sh.R);
    }
    int32_t* par = parent + (int64_t)f * sh.cap;
    const int p = r * sh.Sk + c;
    if (__ldcg(par + p) < 0) continue;  // no normal
    const double* bn = bnorm + (int64_t)f * sh.cap * 3;
    const double a[3] = {__ldcg(bn + 3 * p), __ldcg(bn + 3 * p + 1), __ldcg(bn + 3 * p + 2)};
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      if (r + slot_dr(s) >= sh.R) continue;
      if (edge_internal<TR, TC>(r, c, s, sh.Sk)) continue;
      const int q = (r + slot_dr(s)) * sh.Sk + wrapc(c + slot_dc(s), sh.Sk);
      if (__ldcg(par + q) < 0) continue;
      const double b[3] = {__ldcg(bn + 3 * q), __ldcg(bn + 3 * q + 1), __ldcg(bn + 3 * q + 2)};
      if (normals_pass(a, b, t0, t1, t2)) uf_union(par, p, q);
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
__global__ void k_root_flatten(Shape sh, int32_t* __restrict__ parent, uint32_t* __restrict__ rbits,
                               int32_t* __restrict__ hist, int64_t K) {
  const int64_t nwords = (int64_t)sh.F * sh.R * sh.Wk;
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nwords;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t row = w / sh.Wk;
    const int c = (int)(w - row * sh.Wk) * 32 + lane;
    const int f = (int)(row / sh.R);
    bool root = false;
    if (c < sh.Sk) {
      int32_t* par = parent + (int64_t)f * sh.cap;
      const int cell = (int)(row - (int64_t)f * sh.R) * sh.Sk + c;
      const int p = __ldcg(par + cell);
      if (p >= 0) {
        const int r = root_of(par, p);
        if (r != p) par[cell] = r;
        root = (r == cell);
        if (root) hist[(int64_t)f * K + cell + 1] = 0;
      }
    }
    const uint32_t b = __ballot_sync(0xffffffffu, root);
    if (lane == 0) rbits[w] = b;
  }
}

// 1 + rank of root cell rc among the set bits of (bits, pre) = its label.
__device__ __forceinline__ int rank_label(const uint32_t* bf, const int32_t* pf, int Wk, int Sk, int rc) {
  const int rr = rc / Sk, cc = rc - rr * Sk;
  return 1 + node_id_at(bf + (int64_t)rr * Wk, pf + (int64_t)rr * Wk, cc);
}

// Node labels + backfill + histogram for one ring row per CTA.
template <int T, int ITEMS>
__global__ void __launch_bounds__(T) k_labels_backfill(lseg_sensor sn, Shape sh, const double* __restrict__ ranges,
                                                       const uint32_t* __restrict__ vbits,
                                                       const int32_t* __restrict__ parent,
                                                       const uint32_t* __restrict__ rbits,
                                                       const int32_t* __restrict__ rpre,
                                                       int32_t* __restrict__ node_labels, int32_t* __restrict__ out,
                                                       int32_t* __restrict__ hist, int64_t K) {
  using Scan = cub::BlockScan<int, T>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_first[T];
  __shared__ int s_next[T];
  __shared__ int s_gfirst, s_glast;
  extern __shared__ int s_row[];
  const int64_t row = blockIdx.x;
  const int f = (int)(row / sh.R), i = (int)(row - (int64_t)f * sh.R);
  const int S = sh.S;
  const uint32_t* vbr = vbits + row * sh.Wk;
  const int32_t* par = parent + (int64_t)f * sh.cap;

  // node labels of this row, provisional ids = root cell + 1 (ascending root
  // cell == ascending reference label, so the final compaction in
  // k_prune_rows reproduces the reference ids); -1 marks an invalid kept cell
  // (so k = 1 needs no ranges read for validity)
  const uint32_t* rbf = rbits + (int64_t)f * sh.R * sh.Wk;
  const int32_t* rpf = rpre + (int64_t)f * sh.R * sh.Wk;
  for (int s = threadIdx.x; s < S; s += T) {
    int lab = 0;
    if (s % sh.k == 0) {
      const int c = s / sh.k;
      const int p = __ldcg(par + i * sh.Sk + c);  // flattened: p is the root cell
      if (p >= 0) lab = p + 1;
      else if (!((__ldg(vbr + (c >> 5)) >> (c & 31)) & 1u)) lab = -1;
    }
    s_row[s] = lab;
  }
  __syncthreads();
  if (node_labels)  // reference segment() output: 1 + rank of the root
    for (int s = threadIdx.x; s < S; s += T) {
      const int v = s_row[s];
      node_labels[row * S + s] = v > 0 ? rank_label(rbf, rpf, sh.Wk, sh.Sk, v - 1) : 0;
    }

  const int s0 = threadIdx.x * ITEMS;
  int lab[ITEMS];
  bool valid[ITEMS];
  int last = INT_MIN, first = INT_MAX;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int s = s0 + j;
    lab[j] = 0;
    valid[j] = false;
    if (s < S) {
      const int v = s_row[s];
      if (sh.k == 1) valid[j] = (v >= 0);
      else valid[j] = (v > 0) || in_window(__ldg(ranges + row * S + s), sn.r_min, sn.r_max);
      lab[j] = max(v, 0);
      if (lab[j] > 0) { if (first == INT_MAX) first = s; last = s; }
    }
  }
  int prev;
  Scan(tmp).ExclusiveScan(last, prev, INT_MIN, cub::Max());
  __syncthreads();
  s_first[threadIdx.x] = first;
  __syncthreads();
  int rout;
  Scan(tmp).ExclusiveScan(s_first[T - 1 - threadIdx.x], rout, INT_MAX, cub::Min());
  s_next[T - 1 - threadIdx.x] = rout;
  if (threadIdx.x == T - 1) s_glast = (last != INT_MIN) ? last : prev;
  __syncthreads();
  const int next = s_next[threadIdx.x];
  if (threadIdx.x == 0) s_gfirst = (first != INT_MAX) ? first : next;
  __syncthreads();
  const int gfirst = s_gfirst, glast = s_glast;
  const bool has_donor = (gfirst != INT_MAX);
  int nxt[ITEMS];
  {
    int nd = next;
#pragma unroll
    for (int j = ITEMS - 1; j >= 0; --j) {
      nxt[j] = nd;
      if (lab[j] > 0) nd = s0 + j;
    }
  }
  int pd = prev;
  int run_lab = -1, run_len = 0;
  int32_t* hw = hist + (int64_t)f * K;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int s = s0 + j;
    if (s >= S) break;
    int res = lab[j];
    if (res == 0 && valid[j] && has_donor) {
      const int left = (pd != INT_MIN) ? pd : glast - S;
      const int right = (nxt[j] != INT_MAX) ? nxt[j] : gfirst + S;
      const int dl = s - left, dr = right - s;
      const int ls = left < 0 ? left + S : left;
      const int rs = right >= S ? right - S : right;
      res = max(s_row[dl < dr ? ls : (dr < dl ? rs : min(ls, rs))], 0);
    }
    if (lab[j] > 0) pd = s;
    out[row * S + s] = res;
    if (res == run_lab) ++run_len;
    else {
      if (run_len > 0 && run_lab > 0) atomicAdd(hw + run_lab, run_len);
      run_lab = res;
      run_len = 1;
    }
  }
  if (run_len > 0 && run_lab > 0) atomicAdd(hw + run_lab, run_len);
  (void)i;
}


// ---------------------------------------------------------------- binning
static constexpr double kTwoPiF = 6.283185307179586;  // == 2.0 * np.pi

// First index in [lo, hi) whose ring id is >= v, found by one warp with a
// 32-ary search (4 dependent probes for a 124 k-point frame instead of 17).
// Exact for ring-major input; for other orders the result is arbitrary but in
// range, and k_bin_rows' segment check sends the frame to the generic path.
__device__ __forceinline__ int64_t warp_lower_bound(const int32_t* __restrict__ ring, int64_t lo, int64_t hi, int v,
                                                    int lane) {
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t q = lo + (int64_t)lane * step;
    const bool less = (q < hi) && (__ldg(ring + q) < v);
    const unsigned m = __ballot_sync(0xffffffffu, less);
    const int c = (~m == 0u) ? 32 : __ffs(~m) - 1;  // leading lanes with ring < v
    const int64_t nlo = (c == 0) ? lo : lo + (int64_t)(c - 1) * step + 1;
    const int64_t nhi = (c == 32) ? hi : min(hi, lo + (int64_t)c * step);
    lo = nlo;
    hi = nhi;
  }
  const int64_t q = lo + lane;
  const unsigned m = __ballot_sync(0xffffffffu, (q < hi) && (__ldg(ring + q) < v));
  const int c = (~m == 0u) ? 32 : __ffs(~m) - 1;
  return min(hi, lo + c);
}

// Same definition as k_bin_points: r and step of one point.
// The step is rint(phi*S/2pi) of the fp64 phi; a float atan2 of the (exact,
// float) inputs decides it whenever phi*S/2pi is clearly away from a
// half-integer (its error is < 1e-5 rad, far inside the guard), otherwise the
// fp64 formula runs -- the result is the fp64 formula's either way.
__device__ __forceinline__ bool bin_one(const lseg_sensor& sn, const float* __restrict__ xyz, int64_t p, double& r,
                                        int& step) {
  const float xf = __ldg(xyz + 3 * p), yf = __ldg(xyz + 3 * p + 1), zf = __ldg(xyz + 3 * p + 2);
  const double x = (double)xf, y = (double)yf, z = (double)zf;
  r = __dsqrt_rn(__dadd_rn(__dadd_rn(x * x, y * y), z * z));
  if (!in_window(r, sn.r_min, sn.r_max)) return false;
  const float scale = (float)sn.steps * 0.15915494309189535f;  // S / (2 pi)
  float ph = atan2f(yf, xf);
  if (ph < 0.0f) ph += 6.283185307179586f;
  const float t = ph * scale;
  const float fr = t - floorf(t);
  if (fabsf(fr - 0.5f) > 1e-3f + 2e-5f * scale) {
    int st = (int)rintf(t);
    step = st >= sn.steps ? st - sn.steps : st;
    return true;
  }
  double phi = atan2(y, x);
  if (phi < 0.0) phi = __dadd_rn(phi, kTwoPiF);
  step = (int)rint(__ddiv_rn(__dmul_rn(phi, (double)sn.steps), kTwoPiF)) % sn.steps;
  return true;
}

// Fast path for ring-major input (the sensor's firing order): one CTA per
// (frame, ring) bins that ring's points into a shared-memory row with 64-bit
// shared atomics, then writes the f64 row and the kept-cell valid bits once
// (no memset, no global atomics).  The CTA verifies that its binary-searched
// segment really holds only its ring (and ring 0 / R-1 check the prefix /
// suffix), so any other input order flips the frame to the generic path.
template <int T>
__global__ void __launch_bounds__(T) k_bin_rows(lseg_sensor sn, Shape sh, const float* __restrict__ xyz,
                                                const int32_t* __restrict__ ring, const int64_t* __restrict__ off,
                                                double* __restrict__ ranges, uint32_t* __restrict__ vbits,
                                                int32_t* __restrict__ fallback) {
  extern __shared__ unsigned long long s_cell[];
  __shared__ int s_bad;
  const int64_t row = blockIdx.x;
  const int f = (int)(row / sh.R), i = (int)(row - (int64_t)f * sh.R);
  const int S = sh.S;
  __shared__ int64_t s_lohi[2];
  const int64_t p0 = __ldg(off + f), p1 = __ldg(off + f + 1);
  const int warp = threadIdx.x >> 5;
  if (warp < 2) {
    const int64_t b = warp_lower_bound(ring, p0, p1, i + warp, threadIdx.x & 31);
    if ((threadIdx.x & 31) == 0) s_lohi[warp] = b;
  }
  for (int s = threadIdx.x; s < S; s += T) s_cell[s] = ~0ull;
  __syncthreads();
  const int64_t lo = s_lohi[0], hi = s_lohi[1];
  if (threadIdx.x == 0) s_bad = (hi < lo) ? 1 : 0;
  __syncthreads();
  int bad = 0;
  for (int64_t p = lo + threadIdx.x; p < hi; p += T) {
    if (__ldg(ring + p) != i) { bad = 1; continue; }
    double r;
    int st;
    if (bin_one(sn, xyz, p, r, st)) atomicMin(s_cell + st, (unsigned long long)__double_as_longlong(r));
  }
  if (i == 0)
    for (int64_t p = p0 + threadIdx.x; p < lo; p += T) bad |= (__ldg(ring + p) >= 0) ? 1 : 0;
  if (i == sh.R - 1)
    for (int64_t p = hi + threadIdx.x; p < p1; p += T) bad |= (__ldg(ring + p) < sh.R) ? 1 : 0;
  if (bad) s_bad = 1;
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) atomicExch(fallback + f, 1);
    return;
  }
  double* out = ranges + row * S;
  for (int s = threadIdx.x; s < S; s += T) out[s] = __longlong_as_double((long long)s_cell[s]);
  const int lane = threadIdx.x & 31;
  for (int w = threadIdx.x >> 5; w < sh.Wk; w += T / 32) {
    const int c = w * 32 + lane;
    const bool v = (c < sh.Sk) && in_window(__longlong_as_double((long long)s_cell[c * sh.k]), sn.r_min, sn.r_max);
    const uint32_t b = __ballot_sync(0xffffffffu, v);
    if (lane == 0) vbits[row * sh.Wk + w] = b;
  }
}

// Generic path for frames flagged by k_bin_rows: reset the frame's row / bits.
__global__ void k_bin_reset(Shape sh, const int32_t* __restrict__ fallback, double* __restrict__ ranges,
                            uint32_t* __restrict__ vbits) {
  const int64_t row = blockIdx.x;
  const int f = (int)(row / sh.R);
  if (!__ldg(fallback + f)) return;
  for (int s = threadIdx.x; s < sh.S; s += blockDim.x)
    ranges[row * sh.S + s] = __longlong_as_double(~0ll);
  for (int w = threadIdx.x; w < sh.Wk; w += blockDim.x) vbits[row * sh.Wk + w] = 0u;
}

// Generic path: global 64-bit atomicMin per point + atomicOr of the kept bit.
__global__ void k_bin_atomic(lseg_sensor sn, Shape sh, const float* __restrict__ xyz, const int32_t* __restrict__ ring,
                             const int64_t* __restrict__ off, const int32_t* __restrict__ fallback,
                             double* __restrict__ ranges, uint32_t* __restrict__ vbits) {
  const int f = blockIdx.y;
  if (!__ldg(fallback + f)) return;
  const int64_t p0 = __ldg(off + f), p1 = __ldg(off + f + 1);
  for (int64_t p = p0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < p1; p += (int64_t)gridDim.x * blockDim.x) {
    const int rg = __ldg(ring + p);
    double r;
    int st;
    if (rg < 0 || rg >= sh.R || !bin_one(sn, xyz, p, r, st)) continue;
    const int64_t row = (int64_t)f * sh.R + rg;
    atomicMin(reinterpret_cast<unsigned long long*>(ranges + row * sh.S + st),
              (unsigned long long)__double_as_longlong(r));
    if (st % sh.k == 0) {
      const int c = st / sh.k;
      atomicOr(vbits + row * sh.Wk + (c >> 5), 1u << (c & 31));
    }
  }
}

void launch_bin_fused(const lseg_sensor& sn, const Shape& sh, const float* xyz, const int32_t* ring,
                      const int64_t* off, const Workspace& ws, double* ranges, int32_t* n_nodes, cudaStream_t st) {
  cudaMemsetAsync(ws.fallback, 0, sizeof(int32_t) * sh.F, st);
  const size_t smem = sizeof(unsigned long long) * sh.S;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_bin_rows<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_bin_rows<256><<<sh.F * sh.R, 256, smem, st>>>(sn, sh, xyz, ring, off, ranges, ws.vbits, ws.fallback);
  prof_mark("bin_rows", st);
  k_bin_reset<<<sh.F * sh.R, 256, 0, st>>>(sh, ws.fallback, ranges, ws.vbits);
  k_bin_atomic<<<dim3(8, sh.F), 256, 0, st>>>(sn, sh, xyz, ring, off, ws.fallback, ranges, ws.vbits);
  prof_mark("bin_fallback", st);
  launch_frame_scan(sh, ws, n_nodes, st);
}

// Pruning plan over roots: a root survives unless its (post-backfill) count is
// below min_size; survivor bits -> k_frame_scan gives the compaction ranks.
// fscal[f*4] = 1 when some label of frame f is small (reference
// segment.py:136-140: otherwise labels stay as they are).
__global__ void k_survivors(Shape sh, const uint32_t* __restrict__ rbits, const int32_t* __restrict__ hist, int64_t K,
                            int32_t min_size, uint32_t* __restrict__ sbits, int32_t* __restrict__ fscal) {
  const int64_t nwords = (int64_t)sh.F * sh.R * sh.Wk;
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nwords;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t row = w / sh.Wk;
    const int f = (int)(row / sh.R);
    const uint32_t rb = __ldg(rbits + w);
    bool surv = false, small = false;
    if ((rb >> lane) & 1u) {
      const int cell = (int)(row - (int64_t)f * sh.R) * sh.Sk + (int)(w - row * sh.Wk) * 32 + lane;
      const int cnt = __ldg(hist + (int64_t)f * K + cell + 1);
      small = (min_size > 0) && (cnt < min_size);
      surv = !small;
    }
    const uint32_t b = __ballot_sync(0xffffffffu, surv);
    const uint32_t sm = __ballot_sync(0xffffffffu, small);
    if (lane == 0) {
      sbits[w] = b;
      if (sm) atomicOr(fscal + f * 4, 1);
    }
  }
}

// Dissolve small segments into the nearest surviving ring donor (reference
// segment.py:141-154) and write the final compacted ids, one CTA per ring row.
template <int T, int ITEMS>
__global__ void __launch_bounds__(T) k_prune_rows(Shape sh, const int32_t* __restrict__ lab_in,
                                                  int32_t* __restrict__ out, const int32_t* __restrict__ hist,
                                                  int64_t K, int32_t min_size, const int32_t* __restrict__ fscal,
                                                  const uint32_t* __restrict__ rbits, const int32_t* __restrict__ rpre,
                                                  const uint32_t* __restrict__ sbits,
                                                  const int32_t* __restrict__ spre) {
  using Scan = cub::BlockScan<int, T>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_first[T];
  __shared__ int s_next[T];
  __shared__ int s_gfirst, s_glast;
  extern __shared__ int s_row[];
  const int64_t row = blockIdx.x;
  const int f = (int)(row / sh.R);
  const int S = sh.S;
  const bool any_small = fscal[f * 4] != 0;
  const int32_t* hf = hist + (int64_t)f * K;
  const uint32_t* bb = (any_small ? sbits : rbits) + (int64_t)f * sh.R * sh.Wk;
  const int32_t* bp = (any_small ? spre : rpre) + (int64_t)f * sh.R * sh.Wk;
  const int s0 = threadIdx.x * ITEMS;
  int lab[ITEMS];
  bool gone[ITEMS];
  int last = INT_MIN, first = INT_MAX;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int s = s0 + j;
    lab[j] = 0;
    gone[j] = false;
    if (s < S) {
      lab[j] = __ldcg(lab_in + row * S + s);
      gone[j] = any_small && lab[j] > 0 && __ldg(hf + lab[j]) < min_size;
      if (lab[j] > 0 && !gone[j]) { if (first == INT_MAX) first = s; last = s; }
      s_row[s] = gone[j] ? 0 : lab[j];  // donor labels only
    }
  }
  __syncthreads();
  int prev;
  Scan(tmp).ExclusiveScan(last, prev, INT_MIN, cub::Max());
  __syncthreads();
  s_first[threadIdx.x] = first;
  __syncthreads();
  int rout;
  Scan(tmp).ExclusiveScan(s_first[T - 1 - threadIdx.x], rout, INT_MAX, cub::Min());
  s_next[T - 1 - threadIdx.x] = rout;
  if (threadIdx.x == T - 1) s_glast = (last != INT_MIN) ? last : prev;
  __syncthreads();
  const int next = s_next[threadIdx.x];
  if (threadIdx.x == 0) s_gfirst = (first != INT_MAX) ? first : next;
  __syncthreads();
  const int gfirst = s_gfirst, glast = s_glast;
  const bool has_donor = (gfirst != INT_MAX);
  int nxt[ITEMS];
  {
    int nd = next;
#pragma unroll
    for (int j = ITEMS - 1; j >= 0; --j) {
      nxt[j] = nd;
      if (lab[j] > 0 && !gone[j]) nd = s0 + j;
    }
  }
  int pd = prev;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int s = s0 + j;
    if (s >= S) break;
    int res = lab[j];
    if (gone[j]) {
      res = 0;
      if (has_donor) {
        const int left = (pd != INT_MIN) ? pd : glast - S;
        const int right = (nxt[j] != INT_MAX) ? nxt[j] : gfirst + S;
        const int dl = s - left, dr = right - s;
        const int ls = left < 0 ? left + S : left;
        const int rs = right >= S ? right - S : right;
        res = s_row[dl < dr ? ls : (dr < dl ? rs : min(ls, rs))];
      }
    } else if (res > 0) {
      pd = s;
    }
    out[row * S + s] = res > 0 ? rank_label(bb, bp, sh.Wk, sh.Sk, res - 1) : 0;
  }
}

void launch_prune_fused(const Shape& sh, const Workspace& ws, int32_t min_size, int32_t* labels, cudaStream_t st) {
  cudaMemsetAsync(ws.fscal, 0, sizeof(int32_t) * 4 * sh.F, st);
  const int64_t nwords = (int64_t)sh.F * sh.R * sh.Wk;
  const int64_t blocks = (nwords * 32 + 255) / 256;
  k_survivors<<<(unsigned)(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0, st>>>(sh, ws.rbits, ws.hist, ws.K, min_size,
                                                                                ws.sbits, ws.fscal);
  launch_scan_bits(sh, ws.sbits, ws.spre, ws.fscal_cnt, nullptr, 0, st);
  prof_mark("prune_plan", st);
  const size_t smem = sizeof(int) * sh.S;
#define PR(T_, I_)                                                                                            \
  do {                                                                                                        \
    if (smem > 48 * 1024)                                                                                     \
      cudaFuncSetAttribute(k_prune_rows<T_, I_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    k_prune_rows<T_, I_><<<sh.F * sh.R, T_, smem, st>>>(sh, ws.lab_tmp, labels, ws.hist, ws.K, min_size,      \
                                                        ws.fscal, ws.rbits, ws.rpre, ws.sbits, ws.spre);      \
  } while (0)
  if (sh.S <= 1024) PR(256, 4);
  else if (sh.S <= 2048) PR(256, 8);
  else if (sh.S <= 4096) PR(256, 16);
  else PR(512, 32);
#undef PR
  prof_mark("prune_apply", st);
}

// ---------------------------------------------------------------- launchers
void launch_fused_graph(const lseg_sensor& sn, const Shape& sh, const Workspace& ws, const double* ranges,
                        const double* thr, int32_t* node_ids, int32_t* neighbors, float* n32, uint8_t* nmask,
                        int32_t* n_nodes, int32_t* n_labels, int32_t* node_labels, cudaStream_t st) {
  const int tilesC = (sh.Sk + TILE_C - 1) / TILE_C, tilesR = (sh.R + TILE_R - 1) / TILE_R;
  const int64_t nt = (int64_t)sh.F * tilesR * tilesC;
  const size_t tsmem = (size_t)(3 * (TILE_R + 2) * (TILE_C + 2) + 3 * TILE_R * TILE_C) * 8 +
                       (size_t)(TILE_R + 2) * (TILE_C + 2) * 4 + (size_t)TILE_R * TILE_C * 4;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_tile<TILE_R, TILE_C, TILE_T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
    attr_set = true;
  }
  k_tile<TILE_R, TILE_C, TILE_T><<<(unsigned)nt, TILE_T, tsmem, st>>>(sn, sh, ranges, ws.vbits, ws.wpre, thr[0], thr[1],
                                                                  thr[2], node_ids, neighbors, n32, nmask, ws.masks,
                                                                  ws.bnorm);
  prof_mark("tile", st);
  k_tile_cc<TILE_R, TILE_C, 128><<<(unsigned)nt, 128, 0, st>>>(sh, ws.masks, ws.parent);
  prof_mark("tile_cc", st);
  const int64_t nb = ((int64_t)tilesR * sh.Sk + (int64_t)tilesC * sh.R) * sh.F;
  k_merge<TILE_R, TILE_C><<<(unsigned)((nb + 255) / 256 < 148 * 32 ? (nb + 255) / 256 : 148 * 32), 256, 0, st>>>(
      sh, ws.bnorm, thr[0], thr[1], thr[2], ws.parent);
  prof_mark("merge", st);
  {
    const int64_t nwords = (int64_t)sh.F * sh.R * sh.Wk;
    const int64_t blocks = (nwords * 32 + 255) / 256;
    k_root_flatten<<<(unsigned)(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0, st>>>(sh, ws.parent, ws.rbits,
                                                                                     ws.hist, ws.K);
    prof_mark("root_flatten", st);
    launch_scan_bits(sh, ws.rbits, ws.rpre, n_labels, nullptr, 0, st);
    prof_mark("root_scan", st);
  }
  // labels + backfill -> lab_tmp (+ histogram)
  const size_t smem = sizeof(int) * sh.S;
#define LB(T_, I_)                                                                                              \
  do {                                                                                                          \
    if (smem > 48 * 1024)                                                                                       \
      cudaFuncSetAttribute(k_labels_backfill<T_, I_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
    k_labels_backfill<T_, I_><<<sh.F * sh.R, T_, smem, st>>>(sn, sh, ranges, ws.vbits, ws.parent, ws.rbits,      \
                                                             ws.rpre, node_labels, ws.lab_tmp, ws.hist, ws.K);  \
  } while (0)
  if (sh.S <= 1024) LB(256, 4);
  else if (sh.S <= 2048) LB(256, 8);
  else if (sh.S <= 4096) LB(256, 16);
  else LB(512, 32);
#undef LB
  prof_mark("labels_backfill", st);
}

}  // namespace lseg
