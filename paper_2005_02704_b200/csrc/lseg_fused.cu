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

#include "lseg_internal.cuh"
#include "lseg_kernels.cuh"

namespace lseg {

static constexpr int TILE_R = 8;
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

template <int TR, int TC, int T>
__global__ void __launch_bounds__(T) k_tile(lseg_sensor sn, Shape sh, const double* __restrict__ ranges,
                                             const uint32_t* __restrict__ vbits, const int32_t* __restrict__ wpre,
                                             double t0, double t1, double t2, int32_t* __restrict__ node_ids,
                                             int32_t* __restrict__ neighbors, float* __restrict__ n32,
                                             uint8_t* __restrict__ nmask, int32_t* __restrict__ parent,
                                             uint8_t* __restrict__ bflags) {
  constexpr int GR = TR + 3, GC = TC + 3;  // ranges halo: rows r0-1..r0+TR+1, cols c0-1..c0+TC+1
  constexpr int NR = TR + 1, NC = TC + 1;  // normals: rows r0..r0+TR, cols c0..c0+TC
  __shared__ double s_r[GR][GC];
  __shared__ double s_n[NR][NC][3];
  __shared__ uint8_t s_has[NR][NC];
  __shared__ int s_gid[TR * TC];
  __shared__ int s_par[TR * TC];

  const int tilesC = (sh.Sk + TC - 1) / TC;
  const int tilesR = (sh.R + TR - 1) / TR;
  const int64_t b = blockIdx.x;
  const int f = (int)(b / ((int64_t)tilesR * tilesC));
  const int rem = (int)(b - (int64_t)f * tilesR * tilesC);
  const int r0 = (rem / tilesC) * TR, c0 = (rem % tilesC) * TC;
  const int TRe = min(TR, sh.R - r0), TCe = min(TC, sh.Sk - c0);
  const bool full_width = (c0 == 0 && TCe == sh.Sk);
  const double* rf = ranges + (int64_t)f * sh.R * sh.S;
  const uint32_t* vbf = vbits + (int64_t)f * sh.R * sh.Wk;
  const int32_t* wpf = wpre + (int64_t)f * sh.R * sh.Wk;
  const int64_t nbase = (int64_t)f * sh.cap;
  const int tid = threadIdx.x;

  // A. ranges halo (NaN outside the ring range)
  for (int e = tid; e < GR * GC; e += T) {
    const int y = e / GC, x = e - y * GC;
    const int rr = r0 - 1 + y;
    double v = __longlong_as_double(0x7ff8000000000000LL);
    if (rr >= 0 && rr < sh.R) v = __ldg(rf + (int64_t)rr * sh.S + (int64_t)wrapc(c0 - 1 + x, sh.Sk) * sh.k);
    s_r[y][x] = v;
  }
  __syncthreads();

  // B. fp64 normals for tile + forward halo (reference normals.py:94-145 order)
  for (int e = tid; e < NR * NC; e += T) {
    const int y = e / NC, x = e - y * NC;
    const int rr = r0 + y;
    bool ok = false;
    double nv[3] = {0.0, 0.0, 0.0};
    const double rp = s_r[y + 1][x + 1];
    if (rr < sh.R && in_window(rp, sn.r_min, sn.r_max)) {
      const int cc = wrapc(c0 + x, sh.Sk);
      const Vec3 p = cell_pos(sn, rr, cc * sh.k, rp);
      Fan fan;
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const int dy = slot_dr(s), dx = slot_dc(s);
        const double rq = s_r[y + 1 + dy][x + 1 + dx];
        bool present = in_window(rq, sn.r_min, sn.r_max);
        if (s == 5 && sh.Sk == 2) present = false;  // duplicate of slot 2 (mesh.py:96-101)
        if (present) {
          const Vec3 q = cell_pos(sn, rr + dy, wrapc(cc + dx, sh.Sk) * sh.k, rq);
          fan.add(__dsub_rn(q.x, p.x), __dsub_rn(q.y, p.y), __dsub_rn(q.z, p.z));
        }
      }
      ok = fan.finish(p, nv);
    }
    s_n[y][x][0] = nv[0];
    s_n[y][x][1] = nv[1];
    s_n[y][x][2] = nv[2];
    s_has[y][x] = ok ? 1 : 0;
  }

  // C. tile nodes: ids, slots, outputs
  for (int e = tid; e < TR * TC; e += T) {
    const int y = e / TC, x = e - y * TC;
    int id = -1;
    if (y < TRe && x < TCe) {
      const int rr = r0 + y, cc = c0 + x;
      id = id_at(vbf, wpf, sh.Wk, rr, cc);
      if (node_ids) node_ids[((int64_t)f * sh.R + rr) * sh.Sk + cc] = id;
      if (id >= 0) {
        int nb[6];
#pragma unroll
        for (int s = 0; s < 6; ++s) {
          const int r2 = rr + slot_dr(s);
          nb[s] = (r2 >= 0 && r2 < sh.R) ? id_at(vbf, wpf, sh.Wk, r2, wrapc(cc + slot_dc(s), sh.Sk)) : -1;
        }
        if (sh.Sk == 2 && nb[5] == nb[2]) nb[5] = -1;
        int4* o4 = reinterpret_cast<int4*>(neighbors + (nbase + id) * 6);  // 24 B, 8-B aligned
        int2* o2 = reinterpret_cast<int2*>(o4);
        o2[0] = make_int2(nb[0], nb[1]);
        o2[1] = make_int2(nb[2], nb[3]);
        o2[2] = make_int2(nb[4], nb[5]);
      }
    }
    s_gid[e] = id;
    s_par[e] = e;
  }
  __syncthreads();  // s_n / s_has / s_gid / s_par complete

  // D. outputs that need the normals + local union over passing forward edges
  for (int e = tid; e < TR * TC; e += T) {
    const int y = e / TC, x = e - y * TC;
    const int id = s_gid[e];
    if (id < 0) continue;
    const bool has = s_has[y][x];
    if (n32) {
      float* o = n32 + (nbase + id) * 3;
      const float nanf_ = __int_as_float(0x7fc00000);
      o[0] = has ? (float)s_n[y][x][0] : nanf_;
      o[1] = has ? (float)s_n[y][x][1] : nanf_;
      o[2] = has ? (float)s_n[y][x][2] : nanf_;
    }
    nmask[nbase + id] = has ? 1 : 0;
  }
  uint8_t myflags[(TR * TC + T - 1) / T];
#pragma unroll
  for (int j = 0; j < (TR * TC + T - 1) / T; ++j) myflags[j] = 0;
#pragma unroll
  for (int j = 0; j < (TR * TC + T - 1) / T; ++j) {
    const int e = tid + j * T;
    if (e >= TR * TC) break;
    const int y = e / TC, x = e - y * TC;
    if (s_gid[e] < 0 || !s_has[y][x]) continue;
    const double* a = s_n[y][x];
#pragma unroll
    for (int s = 0; s < 3; ++s) {  // forward slots N0 (+1,0), N1 (+1,+1), N2 (0,+1)
      const int ty = y + slot_dr(s), tx = x + slot_dc(s);
      if (r0 + ty >= sh.R) continue;        // no ring below the bottom ring
      if (!s_has[ty][tx]) continue;         // target absent or without a normal
      if (!normals_pass(a, s_n[ty][tx], t0, t1, t2)) continue;
      int lx = tx;
      bool local = (ty < TRe);
      if (local) {
        if (tx >= TCe) {
          if (full_width) lx = tx - TCe; else local = false;
        }
      }
      if (local) lunion(s_par, e, ty * TC + lx);
      else myflags[j] |= (uint8_t)(1u << s);
    }
  }
  __syncthreads();

  // E. local roots -> global parent; boundary flags for k_merge
#pragma unroll
  for (int j = 0; j < (TR * TC + T - 1) / T; ++j) {
    const int e = tid + j * T;
    if (e >= TR * TC) break;
    const int y = e / TC, x = e - y * TC;
    if (y >= TRe || x >= TCe) continue;
    const int id = s_gid[e];
    // union-find runs on frame-local kept-cell indices (row-major, so the
    // minimum cell of a component is also its minimum node id)
    int pc = -1;
    if (id >= 0 && s_has[y][x]) {
      const int lr = lfind(s_par, e);
      pc = (r0 + lr / TC) * sh.Sk + c0 + lr % TC;
    }
    parent[nbase + (int64_t)(r0 + y) * sh.Sk + c0 + x] = pc;
    if (y == TR - 1 || y == TRe - 1 || x == TC - 1 || x == TCe - 1)
      bflags[((int64_t)f * sh.R + r0 + y) * sh.Sk + c0 + x] = (id >= 0) ? myflags[j] : 0;
  }
}

// Global union over tile-boundary edges.  Threads enumerate the cells of the
// tiles' last rows and last columns (duplicates at corners are harmless).
template <int TR, int TC>
__global__ void k_merge(Shape sh, const uint8_t* __restrict__ bflags, int32_t* __restrict__ parent) {
  const int nbr = (sh.R + TR - 1) / TR;                // boundary rows per frame (last row of each tile row)
  const int nbc = (sh.Sk + TC - 1) / TC;               // boundary cols per frame
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
    const uint8_t fl = bflags[((int64_t)f * sh.R + r) * sh.Sk + c];
    if (!fl) continue;
    int32_t* par = parent + (int64_t)f * sh.cap;
    const int p = r * sh.Sk + c;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      if (!(fl & (1u << s))) continue;
      const int q = (r + slot_dr(s)) * sh.Sk + wrapc(c + slot_dc(s), sh.Sk);
      uf_union(par, p, q);
    }
  }
}

// Final roots as a bit per kept cell (a labelled cell whose parent is itself);
// k_frame_scan over these bits gives every root its rank = label - 1.
__global__ void k_root_bits(Shape sh, const int32_t* __restrict__ parent, uint32_t* __restrict__ rbits) {
  const int64_t nwords = (int64_t)sh.F * sh.R * sh.Wk;
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nwords;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t row = w / sh.Wk;
    const int c = (int)(w - row * sh.Wk) * 32 + lane;
    bool root = false;
    if (c < sh.Sk) {
      const int f = (int)(row / sh.R);
      const int64_t cell = row * sh.Sk + c;  // == f*cap + frame-local cell
      root = (__ldg(parent + cell) == (int)(cell - (int64_t)f * sh.cap));
    }
    const uint32_t b = __ballot_sync(0xffffffffu, root);
    if (lane == 0) rbits[w] = b;
  }
}

// Read-only root chase (parent[x] <= x, so it terminates).
__device__ __forceinline__ int root_of(const int32_t* __restrict__ par, int x) {
  int p = __ldcg(par + x);
  while (p != x) { x = p; p = __ldcg(par + x); }
  return x;
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

  // node labels of this row (reference segment.py:86-88); -1 marks an invalid
  // kept cell (so k = 1 needs no ranges read for validity)
  const uint32_t* rbf = rbits + (int64_t)f * sh.R * sh.Wk;
  const int32_t* rpf = rpre + (int64_t)f * sh.R * sh.Wk;
  for (int s = threadIdx.x; s < S; s += T) {
    int lab = 0;
    if (s % sh.k == 0) {
      const int c = s / sh.k;
      const int p = __ldcg(par + i * sh.Sk + c);
      if (p >= 0) {
        const int rc = root_of(par, p);
        const int rr = rc / sh.Sk, cc = rc - rr * sh.Sk;
        lab = 1 + node_id_at(rbf + (int64_t)rr * sh.Wk, rpf + (int64_t)rr * sh.Wk, cc);
      } else if (!((__ldg(vbr + (c >> 5)) >> (c & 31)) & 1u)) {
        lab = -1;
      }
    }
    s_row[s] = lab;
  }
  __syncthreads();
  if (node_labels)
    for (int s = threadIdx.x; s < S; s += T) node_labels[row * S + s] = max(s_row[s], 0);

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

__device__ __forceinline__ int64_t lower_bound_ring(const int32_t* __restrict__ ring, int64_t lo, int64_t hi, int v) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(ring + mid) < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Same definition as k_bin_points: r and step of one point.
__device__ __forceinline__ bool bin_one(const lseg_sensor& sn, const float* __restrict__ xyz, int64_t p, double& r,
                                        int& step) {
  const double x = (double)__ldg(xyz + 3 * p), y = (double)__ldg(xyz + 3 * p + 1), z = (double)__ldg(xyz + 3 * p + 2);
  r = __dsqrt_rn(__dadd_rn(__dadd_rn(x * x, y * y), z * z));
  if (!in_window(r, sn.r_min, sn.r_max)) return false;
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
  const int64_t p0 = __ldg(off + f), p1 = __ldg(off + f + 1);
  const int64_t lo = lower_bound_ring(ring, p0, p1, i);
  const int64_t hi = lower_bound_ring(ring, p0, p1, i + 1);
  for (int s = threadIdx.x; s < S; s += T) s_cell[s] = ~0ull;
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

// ---------------------------------------------------------------- launchers
void launch_fused_graph(const lseg_sensor& sn, const Shape& sh, const Workspace& ws, const double* ranges,
                        const double* thr, int32_t* node_ids, int32_t* neighbors, float* n32, uint8_t* nmask,
                        int32_t* n_nodes, int32_t* n_labels, int32_t* node_labels, cudaStream_t st) {
  const int tilesC = (sh.Sk + TILE_C - 1) / TILE_C, tilesR = (sh.R + TILE_R - 1) / TILE_R;
  const int64_t nt = (int64_t)sh.F * tilesR * tilesC;
  k_tile<TILE_R, TILE_C, TILE_T><<<(unsigned)nt, TILE_T, 0, st>>>(sn, sh, ranges, ws.vbits, ws.wpre, thr[0], thr[1],
                                                                  thr[2], node_ids, neighbors, n32, nmask, ws.parent,
                                                                  ws.bflags);
  prof_mark("tile", st);
  const int64_t nb = ((int64_t)tilesR * sh.Sk + (int64_t)tilesC * sh.R) * sh.F;
  k_merge<TILE_R, TILE_C><<<(unsigned)((nb + 255) / 256 < 148 * 32 ? (nb + 255) / 256 : 148 * 32), 256, 0, st>>>(
      sh, ws.bflags, ws.parent);
  prof_mark("merge", st);
  {
    const int64_t nwords = (int64_t)sh.F * sh.R * sh.Wk;
    const int64_t blocks = (nwords * 32 + 255) / 256;
    k_root_bits<<<(unsigned)(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0, st>>>(sh, ws.parent, ws.rbits);
    prof_mark("root_bits", st);
    launch_scan_bits(sh, ws.rbits, ws.rpre, n_labels, ws.hist, ws.K, st);
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
  else if (sh.S <= 4096) LB(256, 16);
  else LB(512, 32);
#undef LB
  prof_mark("labels_backfill", st);
}

}  // namespace lseg
