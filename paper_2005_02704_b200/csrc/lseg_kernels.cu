// lidarseg_b200 kernels for sm_100a.
//
// Hot path: bin points -> valid bits + node numbering ->
// mesh slots -> fp64 normals -> union-find segments -> per-ring backfill ->
// small-segment pruning.  All kernels take a frame axis F; grids are dense
// row-major (F, R, S) and node arrays are per-frame slabs of cap = R*S'.
//
// Nothing here is a dense contraction, so no tensor cores: every kernel is
// bounded by HBM/L2 bandwidth or by fp64 issue (normals); see DESIGN.md for
// the byte model per kernel.

#include <cub/block/block_scan.cuh>
#include <cub/block/block_reduce.cuh>

#include "lseg_internal.cuh"
#include "lseg_kernels.cuh"

namespace lseg {

static constexpr double kTwoPi = 6.283185307179586;  // == 2.0 * np.pi

// --------------------------------------------------------------------------
// K1: bin points into the f64 range grid.  Grid pre-filled with all-ones bits
// (a NaN whose u64 image exceeds every finite positive double), so a u64
// atomicMin on the bit pattern keeps the smallest r per cell.
// --------------------------------------------------------------------------
__global__ void k_bin_points(lseg_sensor sn, int F, const float* __restrict__ xyz,
                             const int32_t* __restrict__ ring, const int64_t* __restrict__ off,
                             int64_t P, double* __restrict__ ranges, int32_t* __restrict__ cell_out) {
  const int R = sn.rings, S = sn.steps;
  const double dS = (double)S;
  // only the points the frames own: [off[0], off[F]) read on the device (the
  // buffer behind xyz may be longer than the frames' points, e.g. a reused
  // chunk buffer, and off[0] need not be 0 for a sub-batch of a larger one)
  const int64_t pb = __ldg(off), pe = min(__ldg(off + F), P);
  for (int64_t p = pb + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < pe;
       p += (int64_t)gridDim.x * blockDim.x) {
    // frame of point p: binary search in off[0..F]
    int lo = 0, hi = F;  // off[lo] <= p < off[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(off + mid) <= p) lo = mid; else hi = mid;
    }
    const double x = (double)__ldg(xyz + 3 * p), y = (double)__ldg(xyz + 3 * p + 1),
                 z = (double)__ldg(xyz + 3 * p + 2);
    const int rg = __ldg(ring + p);
    // products of f32 values are exact in f64, so FMA contraction cannot change r
    const double r = __dsqrt_rn(__dadd_rn(__dadd_rn(x * x, y * y), z * z));
    int c = -1;
    if (in_window(r, sn.r_min, sn.r_max) && rg >= 0 && rg < R) {
      double phi = atan2(y, x);
      if (phi < 0.0) phi = __dadd_rn(phi, kTwoPi);
      int st = (int)rint(__ddiv_rn(__dmul_rn(phi, dS), kTwoPi));
      st %= S;
      c = rg * S + st;
      atomicMin(reinterpret_cast<unsigned long long*>(ranges + (int64_t)lo * R * S + c),
                (unsigned long long)__double_as_longlong(r));
    }
    if (cell_out) cell_out[p] = c;
  }
}

// --------------------------------------------------------------------------
// K2a: valid bits of kept cells, one warp per 32 consecutive kept cells of a row.
// --------------------------------------------------------------------------
__global__ void k_valid_bits(lseg_sensor sn, Shape sh, const double* __restrict__ ranges,
                             uint32_t* __restrict__ vbits) {
  pdl_trigger();
  pdl_wait();
  const int64_t nwords = (int64_t)sh.F * sh.R * sh.Wk;
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nwords;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t row = w / sh.Wk;  // f*R + i
    const int c = (int)(w - row * sh.Wk) * 32 + lane;
    bool v = false;
    if (c < sh.Sk) v = in_window(__ldg(ranges + row * sh.S + (int64_t)c * sh.k), sn.r_min, sn.r_max);
    const uint32_t b = __ballot_sync(0xffffffffu, v);
    if (lane == 0) vbits[w] = b;
  }
}

// --------------------------------------------------------------------------
// K2b: per-frame exclusive scan of valid counts over (R, Wk) words -> word
// prefix = frame-local node id of each word's first valid cell.  One CTA per
// frame (node numbering is row-major per frame, reference mesh.py:115-117).
// --------------------------------------------------------------------------
template <int T, int ITEMS>
__global__ void __launch_bounds__(T) k_frame_scan(Shape sh, const uint32_t* __restrict__ vbits,
                                                  int32_t* __restrict__ wpre, int32_t* __restrict__ n_nodes,
                                                  int32_t* __restrict__ hist, int64_t K) {
  pdl_trigger();
  pdl_wait();
  using Scan = cub::BlockScan<int, T>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  const int f = blockIdx.x;
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
  if (hist) {  // zero the histogram slots 0..count this frame's labels will use
    int32_t* h = hist + (int64_t)f * K;
    for (int64_t l = threadIdx.x; l <= carry; l += T) h[l] = 0;
  }
}

// --------------------------------------------------------------------------
// K2c: mesh slots.  One thread per kept cell; writes node_ids (F,R,S') and,
// for nodes, the 6 slots (reference _neighbor_grid, mesh.py:83-102) plus the
// optional 3-D edge-length filter (mesh.py:122-126).
// --------------------------------------------------------------------------
__global__ void k_mesh(lseg_sensor sn, Shape sh, double max_edge, const double* __restrict__ ranges,
                       const uint32_t* __restrict__ vbits, const int32_t* __restrict__ wpre,
                       int32_t* __restrict__ node_ids, int32_t* __restrict__ neighbors,
                       int32_t* __restrict__ node_rings, int32_t* __restrict__ node_steps) {
  const int64_t ncell = (int64_t)sh.F * sh.R * sh.Sk;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ncell;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / sh.Sk;
    const int c = (int)(t - row * sh.Sk);
    const int f = (int)(row / sh.R), i = (int)(row - (int64_t)f * sh.R);
    const uint32_t* vbf = vbits + (int64_t)f * sh.R * sh.Wk;
    const int32_t* wpf = wpre + (int64_t)f * sh.R * sh.Wk;
    const int id = node_id_at(vbf + (int64_t)i * sh.Wk, wpf + (int64_t)i * sh.Wk, c);
    node_ids[t] = id;
    if (id < 0) continue;
    int nb[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int i2 = i + slot_dr(s);
      int c2 = c + slot_dc(s);
      c2 = c2 < 0 ? c2 + sh.Sk : (c2 >= sh.Sk ? c2 - sh.Sk : c2);
      nb[s] = (i2 >= 0 && i2 < sh.R) ? node_id_at(vbf + (int64_t)i2 * sh.Wk, wpf + (int64_t)i2 * sh.Wk, c2) : -1;
    }
    if (sh.Sk == 2) {  // j+ == j-: drop a slot repeating an earlier one (mesh.py:96-101)
#pragma unroll
      for (int s = 1; s < 6; ++s) {
        bool dup = false;
#pragma unroll
        for (int u = 0; u < s; ++u) dup |= (nb[s] >= 0 && nb[u] == nb[s]);
        if (dup) nb[s] = -1;
      }
    }
    if (!isnan(max_edge)) {
      const double* rf = ranges + (int64_t)f * sh.R * sh.S;
      const Vec3 p = cell_pos(sn, i, c * sh.k, rf[(int64_t)i * sh.S + (int64_t)c * sh.k]);
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        if (nb[s] < 0) continue;
        const int i2 = i + slot_dr(s);
        int c2 = c + slot_dc(s);
        c2 = c2 < 0 ? c2 + sh.Sk : (c2 >= sh.Sk ? c2 - sh.Sk : c2);
        const Vec3 q = cell_pos(sn, i2, c2 * sh.k, rf[(int64_t)i2 * sh.S + (int64_t)c2 * sh.k]);
        const double d = norm3(__dsub_rn(q.x, p.x), __dsub_rn(q.y, p.y), __dsub_rn(q.z, p.z));
        if (!(d <= max_edge)) nb[s] = -1;
      }
    }
    int32_t* out = neighbors + ((int64_t)f * sh.cap + id) * 6;
#pragma unroll
    for (int s = 0; s < 6; ++s) out[s] = nb[s];
    if (node_rings) node_rings[(int64_t)f * sh.cap + id] = i;
    if (node_steps) node_steps[(int64_t)f * sh.cap + id] = c * sh.k;
  }
}

// --------------------------------------------------------------------------
// K3: normals.  One thread per kept cell; neighbour positions come from the
// slot's cell (the slot table fixes which cell a present slot refers to).
// --------------------------------------------------------------------------
__global__ void k_normals(lseg_sensor sn, Shape sh, const double* __restrict__ ranges,
                          const int32_t* __restrict__ node_ids, const int32_t* __restrict__ neighbors,
                          double* __restrict__ n64, float* __restrict__ n32, uint8_t* __restrict__ nmask) {
  const int64_t ncell = (int64_t)sh.F * sh.R * sh.Sk;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ncell;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int id = __ldg(node_ids + t);
    if (id < 0) continue;
    const int64_t row = t / sh.Sk;
    const int c = (int)(t - row * sh.Sk);
    const int f = (int)(row / sh.R), i = (int)(row - (int64_t)f * sh.R);
    const double* rf = ranges + (int64_t)f * sh.R * sh.S;
    const Vec3 p = cell_pos(sn, i, c * sh.k, __ldg(rf + (int64_t)i * sh.S + (int64_t)c * sh.k));
    const int64_t node = (int64_t)f * sh.cap + id;
    Fan fan;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      if (__ldg(neighbors + node * 6 + s) < 0) continue;
      const int i2 = i + slot_dr(s);
      int c2 = c + slot_dc(s);
      c2 = c2 < 0 ? c2 + sh.Sk : (c2 >= sh.Sk ? c2 - sh.Sk : c2);
      const Vec3 q = cell_pos(sn, i2, c2 * sh.k, __ldg(rf + (int64_t)i2 * sh.S + (int64_t)c2 * sh.k));
      fan.add(__dsub_rn(q.x, p.x), __dsub_rn(q.y, p.y), __dsub_rn(q.z, p.z));
    }
    double n[3];
    const bool ok = fan.finish(p, n);
    if (!ok) n[0] = n[1] = n[2] = __longlong_as_double(0x7ff8000000000000LL);
    if (n64) { n64[node * 3] = n[0]; n64[node * 3 + 1] = n[1]; n64[node * 3 + 2] = n[2]; }
    if (n32) { n32[node * 3] = (float)n[0]; n32[node * 3 + 1] = (float)n[1]; n32[node * 3 + 2] = (float)n[2]; }
    nmask[node] = ok ? 1 : 0;
  }
}

// --------------------------------------------------------------------------
// K4: union-find connected components (replaces the DFS of segment.py:63-84).
// --------------------------------------------------------------------------
__global__ void k_uf_init(Shape sh, const int32_t* __restrict__ n_nodes, int32_t* __restrict__ parent) {
  const int64_t n = (int64_t)sh.F * sh.cap;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(t / sh.cap);
    const int p = (int)(t - (int64_t)f * sh.cap);
    if (p < __ldg(n_nodes + f)) parent[t] = p;
  }
}

__global__ void k_uf_union(Shape sh, int nslots, const int32_t* __restrict__ n_nodes,
                           const int32_t* __restrict__ neighbors, const double* __restrict__ n64,
                           const uint8_t* __restrict__ nmask, double t0, double t1, double t2,
                           int32_t* __restrict__ parent) {
  const int64_t n = (int64_t)sh.F * sh.cap;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(t / sh.cap);
    const int p = (int)(t - (int64_t)f * sh.cap);
    if (p >= __ldg(n_nodes + f) || !__ldg(nmask + t)) continue;
    double a[3] = {__ldg(n64 + t * 3), __ldg(n64 + t * 3 + 1), __ldg(n64 + t * 3 + 2)};
    int32_t* par = parent + (int64_t)f * sh.cap;
    for (int s = 0; s < nslots; ++s) {
      const int q = __ldg(neighbors + t * 6 + s);
      if (q < 0) continue;
      const int64_t tq = (int64_t)f * sh.cap + q;
      if (!__ldg(nmask + tq)) continue;
      const double b[3] = {__ldg(n64 + tq * 3), __ldg(n64 + tq * 3 + 1), __ldg(n64 + tq * 3 + 2)};
      if (normals_pass(a, b, t0, t1, t2)) uf_union(par, p, q);
    }
  }
}

__global__ void k_uf_flatten(Shape sh, const int32_t* __restrict__ n_nodes, int32_t* __restrict__ parent) {
  const int64_t n = (int64_t)sh.F * sh.cap;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(t / sh.cap);
    const int p = (int)(t - (int64_t)f * sh.cap);
    if (p >= __ldg(n_nodes + f)) continue;
    int32_t* par = parent + (int64_t)f * sh.cap;
    int r = par[p];
    while (true) { const int g = par[r]; if (g == r) break; r = g; }
    par[p] = r;
  }
}

// rank[root] = number of labelled roots before it in node order (per frame);
// also zeroes the label histogram slots this frame will use.
template <int T, int ITEMS>
__global__ void __launch_bounds__(T) k_root_rank(Shape sh, const int32_t* __restrict__ n_nodes,
                                                 const int32_t* __restrict__ parent,
                                                 const uint8_t* __restrict__ nmask, int32_t* __restrict__ rank,
                                                 int32_t* __restrict__ n_labels, int32_t* __restrict__ hist,
                                                 int64_t K) {
  using Scan = cub::BlockScan<int, T>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  const int f = blockIdx.x;
  const int n = n_nodes[f];
  const int32_t* par = parent + (int64_t)f * sh.cap;
  const uint8_t* msk = nmask + (int64_t)f * sh.cap;
  int32_t* rk = rank + (int64_t)f * sh.cap;
  int32_t* h = hist ? hist + (int64_t)f * K : nullptr;
  if (threadIdx.x == 0) { carry = 0; if (h) h[0] = 0; }
  __syncthreads();
  for (int base = 0; base < n; base += T * ITEMS) {
    int v[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const int idx = base + threadIdx.x * ITEMS + j;
      v[j] = (idx < n && msk[idx] && par[idx] == idx) ? 1 : 0;
    }
    int x[ITEMS], total;
    Scan(tmp).ExclusiveSum(v, x, total);
    const int c0 = carry;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const int idx = base + threadIdx.x * ITEMS + j;
      if (v[j]) {
        rk[idx] = c0 + x[j];
        if (h) h[1 + c0 + x[j]] = 0;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) carry = c0 + total;
    __syncthreads();
  }
  if (threadIdx.x == 0) n_labels[f] = carry;
}

// Dense label grid: 1 + rank[root] at node cells with a normal, 0 elsewhere
// (reference segment.py:86-88).
__global__ void k_label_dense(Shape sh, const int32_t* __restrict__ node_ids,
                              const int32_t* __restrict__ parent, const uint8_t* __restrict__ nmask,
                              const int32_t* __restrict__ rank, int32_t* __restrict__ labels) {
  const int64_t n = (int64_t)sh.F * sh.R * sh.S;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / sh.S;
    const int s = (int)(t - row * sh.S);
    int lab = 0;
    if (s % sh.k == 0) {
      const int f = (int)(row / sh.R);
      const int id = __ldg(node_ids + row * sh.Sk + s / sh.k);
      if (id >= 0) {
        const int64_t node = (int64_t)f * sh.cap + id;
        if (__ldg(nmask + node)) lab = 1 + __ldg(rank + (int64_t)f * sh.cap + __ldg(parent + node));
      }
    }
    labels[t] = lab;
  }
}

// --------------------------------------------------------------------------
// K5: per-ring nearest-donor fill (backfill, and the dissolve step of
// prune_small).  One CTA per (frame, ring) row; cyclic distance with the tie
// going to the smaller actual step index (reference segment.py:91-106).
//   mode 0 (backfill):  donors = label > 0, targets = valid & label == 0
//   mode 1 (prune):     donors = label > 0 & !small, targets = label > 0 & small;
//                       outputs remap[label]; rings without donors give 0.
// In mode 0 the kernel also accumulates the per-frame label histogram.
// --------------------------------------------------------------------------
template <int T, int ITEMS>
__global__ void __launch_bounds__(T) k_ring_fill(int mode, lseg_sensor sn, Shape sh,
                                                 const double* __restrict__ ranges,
                                                 const int32_t* __restrict__ lab_in, int32_t* __restrict__ lab_out,
                                                 int32_t* __restrict__ hist, const int32_t* __restrict__ remap,
                                                 const int32_t* __restrict__ fscal, int64_t K, int32_t min_size) {
  using Scan = cub::BlockScan<int, T>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_first[T];
  __shared__ int s_next[T];
  extern __shared__ int s_row[];
  const int64_t row = blockIdx.x;
  const int f = (int)(row / sh.R);
  const int S = sh.S;
  const int32_t* in = lab_in + row * S;
  int32_t* out = lab_out + row * S;
  const int32_t* hf = hist ? hist + (int64_t)f * K : nullptr;
  const int32_t* rm = remap ? remap + (int64_t)f * K : nullptr;
  const bool any_small = (mode == 1) ? (fscal[f * 4] != 0) : false;

  for (int s = threadIdx.x; s < S; s += T) s_row[s] = in[s];
  __syncthreads();

  // donor predicate
  auto is_donor = [&](int lab) -> bool {
    if (lab <= 0) return false;
    if (mode == 0) return true;
    return lab >= K || !(any_small && hf[lab] < min_size);  // >= K: caller error, see below
  };
  const int s0 = threadIdx.x * ITEMS;
  int last = INT_MIN, first = INT_MAX;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int s = s0 + j;
    if (s < S && is_donor(s_row[s])) { if (first == INT_MAX) first = s; last = s; }
  }
  // prev donor before my chunk: exclusive max-scan
  int prev;
  Scan(tmp).ExclusiveScan(last, prev, INT_MIN, cub::Max());
  __syncthreads();
  // next donor after my chunk: exclusive min-scan over reversed thread order
  s_first[threadIdx.x] = first;
  __syncthreads();
  int rin = s_first[T - 1 - threadIdx.x], rout;
  Scan(tmp).ExclusiveScan(rin, rout, INT_MAX, cub::Min());
  s_next[T - 1 - threadIdx.x] = rout;
  __syncthreads();
  int next = s_next[threadIdx.x];
  // row-wide first / last donor for the cyclic wrap
  __shared__ int s_gfirst, s_glast;
  if (threadIdx.x == T - 1) s_glast = (last != INT_MIN) ? last : prev;
  if (threadIdx.x == 0) s_gfirst = (first != INT_MAX) ? first : next;
  __syncthreads();
  const int gfirst = s_gfirst, glast = s_glast;
  const bool has_donor = (gfirst != INT_MAX);

  // walk my chunk backward to get the next donor for each cell
  int nxt[ITEMS];
  {
    int nd = next;
#pragma unroll
    for (int j = ITEMS - 1; j >= 0; --j) {
      const int s = s0 + j;
      nxt[j] = nd;
      if (s < S && is_donor(s_row[s])) nd = s;
    }
  }
  const double* rrow = ranges ? ranges + row * S : nullptr;
  int pd = prev;
  int run_lab = -1, run_len = 0;
  int32_t* hw = (mode == 0 && hist) ? hist + (int64_t)f * K : nullptr;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int s = s0 + j;
    if (s >= S) break;
    const int lab = s_row[s];
    int res = lab;
    bool target;
    if (mode == 0) target = (lab == 0) && in_window(__ldg(rrow + s), sn.r_min, sn.r_max);
    else target = (lab > 0) && lab < K && any_small && hf[lab] < min_size;
    if (target) {
      if (!has_donor) {
        res = (mode == 0) ? lab : 0;
      } else {
        const int left = (pd != INT_MIN) ? pd : glast - S;
        const int right = (nxt[j] != INT_MAX) ? nxt[j] : gfirst + S;
        const int dl = s - left, dr = right - s;
        const int ls = left < 0 ? left + S : left;
        const int rs = right >= S ? right - S : right;
        const int pick = dl < dr ? ls : (dr < dl ? rs : min(ls, rs));
        res = s_row[pick];
      }
    }
    if (is_donor(lab)) pd = s;
    // a label >= K (label_bound too small, a caller error) comes out as -1:
    // no histogram / remap access outside the workspace
    if (mode == 1) res = res >= K ? -1 : (any_small ? rm[res] : res);
    out[s] = res;
    if (hw) {  // run-length aggregated histogram of the backfilled row
      if (res == run_lab) ++run_len;
      else {
        if (run_len > 0 && run_lab > 0) atomicAdd(hw + run_lab, run_len);
        run_lab = res; run_len = 1;
      }
    }
  }
  if (hw && run_len > 0 && run_lab > 0) atomicAdd(hw + run_lab, run_len);
}

// Per frame: any_small flag and the survivor remap (compaction to 1..k in
// ascending old-id order, segment.py:155-160).  remap[0] = 0.
template <int T, int ITEMS>
__global__ void __launch_bounds__(T) k_prune_plan(const int32_t* __restrict__ n_labels, int64_t K,
                                                  int32_t min_size, const int32_t* __restrict__ hist,
                                                  int32_t* __restrict__ remap, int32_t* __restrict__ fscal) {
  using Scan = cub::BlockScan<int, T>;
  using Red = cub::BlockReduce<int, T>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ typename Red::TempStorage rtmp;
  __shared__ int carry, anys;
  const int f = blockIdx.x;
  const int64_t L = n_labels ? (int64_t)n_labels[f] + 1 : K;  // label values < L
  const int32_t* h = hist + (int64_t)f * K;
  int32_t* rm = remap + (int64_t)f * K;
  if (threadIdx.x == 0) { carry = 0; anys = 0; }
  __syncthreads();
  // Compaction happens iff some id in 1..L-1 has count < m, absent ids included
  // (reference bincount semantics, segment.py:136-140).
  int local = 0;
  if (min_size > 0)
    for (int64_t l = 1 + threadIdx.x; l < L; l += T) local |= (h[l] < min_size) ? 1 : 0;
  const int any = Red(rtmp).Reduce(local, cub::Max());
  if (threadIdx.x == 0) anys = any;
  __syncthreads();
  const int do_prune = anys;
  for (int64_t base = 0; base < L; base += (int64_t)T * ITEMS) {
    int v[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const int64_t l = base + (int64_t)threadIdx.x * ITEMS + j;
      v[j] = (l > 0 && l < L && h[l] >= min_size && h[l] > 0) ? 1 : 0;
    }
    int x[ITEMS], total;
    Scan(tmp).ExclusiveSum(v, x, total);
    const int c0 = carry;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const int64_t l = base + (int64_t)threadIdx.x * ITEMS + j;
      if (l < L) rm[l] = do_prune ? (v[j] ? 1 + c0 + x[j] : 0) : (int)l;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry = c0 + total;
    __syncthreads();
  }
  if (threadIdx.x == 0) { fscal[f * 4] = do_prune; fscal[f * 4 + 1] = do_prune ? carry : -1; }
}

// Histogram of arbitrary label grids (standalone prune_small).
__global__ void k_hist(Shape sh, int64_t K, const int32_t* __restrict__ labels, int32_t* __restrict__ hist) {
  const int64_t n = (int64_t)sh.F * sh.R * sh.S;
  const int64_t per = (int64_t)sh.R * sh.S;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int lab = labels[t];
    // labels outside [1, K) are a caller error (label_bound too small): not
    // counted, flagged in hist[frame * K + 0] (slot 0 is never a label)
    if (lab > 0 && lab < K) atomicAdd(hist + (t / per) * K + lab, 1);
    else if (lab >= K) atomicOr(hist + (t / per) * K, 1);
  }
}

// --------------------------------------------------------------------------
// mesh_triangles (export only): one CTA per frame, type-A faces then type-B.
// --------------------------------------------------------------------------
template <int T>
__global__ void __launch_bounds__(T) k_triangles(int R, int Sk, const int32_t* __restrict__ node_ids,
                                                 int32_t* __restrict__ tris, int32_t* __restrict__ n_tris) {
  using Scan = cub::BlockScan<int, T>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  const int f = blockIdx.x;
  const int64_t ncell = (int64_t)R * Sk;
  const int32_t* ids = node_ids + f * ncell;
  int32_t* out = tris + f * ncell * 2 * 3;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int type = 0; type < 2; ++type) {
    for (int64_t base = 0; base < ncell; base += T) {
      const int64_t t = base + threadIdx.x;
      int a = -1, b = -1, c = -1;
      if (t < ncell) {
        const int i = (int)(t / Sk), j = (int)(t - (int64_t)i * Sk);
        const int jn = (j + 1 == Sk) ? 0 : j + 1;
        a = ids[t];
        const int down = (i + 1 < R) ? ids[(int64_t)(i + 1) * Sk + j] : -1;
        const int diag = (i + 1 < R) ? ids[(int64_t)(i + 1) * Sk + jn] : -1;
        const int right = ids[(int64_t)i * Sk + jn];
        if (type == 0) { b = down; c = diag; } else { b = diag; c = right; }
      }
      const int ok = (a >= 0 && b >= 0 && c >= 0) ? 1 : 0;
      int pos, total;
      Scan(tmp).ExclusiveSum(ok, pos, total);
      const int c0 = carry;
      if (ok) {
        int32_t* o = out + (int64_t)(c0 + pos) * 3;
        o[0] = a; o[1] = b; o[2] = c;
      }
      __syncthreads();
      if (threadIdx.x == 0) carry = c0 + total;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) n_tris[f] = carry;
}

// --------------------------------------------------------------------------
// Self-test of sqrt_pos / rcp_pos against the IEEE intrinsics on n random
// doubles (random mantissas; log-uniform exponents in [2^-40, 2^40] for odd
// seeds, [2^-300, 2^300] for even seeds).
__global__ void k_selftest_math(int64_t n, uint64_t seed, unsigned long long* bad) {
  unsigned long long b0 = 0, b1 = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (uint64_t)t * 0x9E3779B97F4A7C15ull ^ seed;
    h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
    const uint64_t mant = h & 0x000FFFFFFFFFFFFFull;
    const int ex = (seed & 1) ? (int)((h >> 52) % 81) - 40 : (int)((h >> 52) % 601) - 300;
    const double x = __longlong_as_double((long long)(((uint64_t)(1023 + ex) << 52) | mant));
    b0 += sqrt_pos(x) != __dsqrt_rn(x);
    b1 += rcp_pos(x) != __drcp_rn(x);
  }
  if (b0) atomicAdd(bad, b0);
  if (b1) atomicAdd(bad + 1, b1);
}

void launch_selftest_math(int64_t n, uint64_t seed, unsigned long long* bad, cudaStream_t st) {
  cudaMemsetAsync(bad, 0, 16, st);
  k_selftest_math<<<num_sms() * 16, 256, 0, st>>>(n, seed, bad);
}

// --------------------------------------------------------------------------
// host-side launchers
// --------------------------------------------------------------------------
static inline int grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 64;  // persistent-ish grid-stride cap
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

void launch_bin(const lseg_sensor& sn, int F, const float* xyz, const int32_t* ring, const int64_t* off,
                int64_t P, double* ranges, int32_t* cell, cudaStream_t st) {
  cudaMemsetAsync(ranges, 0xFF, sizeof(double) * (size_t)F * sn.rings * sn.steps, st);
  prof_mark("bin_fill", st);
  if (P > 0) k_bin_points<<<grid_for(P, 256), 256, 0, st>>>(sn, F, xyz, ring, off, P, ranges, cell);
  prof_mark("bin", st);
}

void launch_mesh(const lseg_sensor& sn, const Shape& sh, double max_edge, const double* ranges,
                 const Workspace& ws, int32_t* node_ids, int32_t* neighbors, int32_t* node_rings,
                 int32_t* node_steps, int32_t* n_nodes, cudaStream_t st) {
  const int64_t nwords = (int64_t)sh.F * sh.R * sh.Wk;
  launch_pdl(k_valid_bits, grid_for(nwords * 32, 256), 256, 0, st, sn, sh, ranges, ws.vbits);
  prof_mark("valid_bits", st);
  launch_pdl(k_frame_scan<1024, 4>, sh.F, 1024, 0, st, sh, ws.vbits, ws.wpre, n_nodes, nullptr, 0);
  prof_mark("frame_scan", st);
  const int64_t ncell = (int64_t)sh.F * sh.R * sh.Sk;
  k_mesh<<<grid_for(ncell, 256), 256, 0, st>>>(sn, sh, max_edge, ranges, ws.vbits, ws.wpre, node_ids,
                                               neighbors, node_rings, node_steps);
  prof_mark("mesh", st);
}

void launch_valid_scan(const lseg_sensor& sn, const Shape& sh, const double* ranges, const Workspace& ws,
                       int32_t* n_nodes, cudaStream_t st) {
  const int64_t nwords = (int64_t)sh.F * sh.R * sh.Wk;
  launch_pdl(k_valid_bits, grid_for(nwords * 32, 256), 256, 0, st, sn, sh, ranges, ws.vbits);
  prof_mark("valid_bits", st);
  launch_pdl(k_frame_scan<1024, 4>, sh.F, 1024, 0, st, sh, ws.vbits, ws.wpre, n_nodes, nullptr, 0);
  prof_mark("frame_scan", st);
}

void launch_frame_scan(const Shape& sh, const Workspace& ws, int32_t* n_nodes, cudaStream_t st) {
  launch_pdl(k_frame_scan<1024, 4>, sh.F, 1024, 0, st, sh, ws.vbits, ws.wpre, n_nodes, nullptr, 0);
  prof_mark("frame_scan", st);
}

void launch_scan_bits(const Shape& sh, const uint32_t* bits, int32_t* pre, int32_t* counts, int32_t* hist, int64_t K,
                      cudaStream_t st) {
  launch_pdl(k_frame_scan<1024, 4>, sh.F, 1024, 0, st, sh, bits, pre, counts, hist, K);
}

void launch_root_rank(const Shape& sh, const int32_t* n_nodes, const int32_t* parent, const uint8_t* nmask,
                      int32_t* rank, int32_t* n_labels, int32_t* hist, int64_t K, cudaStream_t st) {
  k_root_rank<1024, 4><<<sh.F, 1024, 0, st>>>(sh, n_nodes, parent, nmask, rank, n_labels, hist, K);
}

void launch_normals(const lseg_sensor& sn, const Shape& sh, const double* ranges, const int32_t* node_ids,
                    const int32_t* neighbors, double* n64, float* n32, uint8_t* nmask, cudaStream_t st) {
  const int64_t ncell = (int64_t)sh.F * sh.R * sh.Sk;
  k_normals<<<grid_for(ncell, 128), 128, 0, st>>>(sn, sh, ranges, node_ids, neighbors, n64, n32, nmask);
}

void launch_segment(const Shape& sh, int nslots, const int32_t* node_ids, const int32_t* neighbors,
                    const int32_t* n_nodes, const double* n64, const uint8_t* nmask, const double* thr,
                    int32_t* labels, int32_t* n_labels, const Workspace& ws, int32_t* hist, cudaStream_t st) {
  const int64_t nn = (int64_t)sh.F * sh.cap;
  k_uf_init<<<grid_for(nn, 256), 256, 0, st>>>(sh, n_nodes, ws.parent);
  prof_mark("uf_init", st);
  k_uf_union<<<grid_for(nn, 256), 256, 0, st>>>(sh, nslots, n_nodes, neighbors, n64, nmask, thr[0], thr[1],
                                                 thr[2], ws.parent);
  prof_mark("uf_union", st);
  k_uf_flatten<<<grid_for(nn, 256), 256, 0, st>>>(sh, n_nodes, ws.parent);
  prof_mark("uf_flatten", st);
  k_root_rank<1024, 4><<<sh.F, 1024, 0, st>>>(sh, n_nodes, ws.parent, nmask, ws.rank, n_labels, hist, ws.K);
  prof_mark("root_rank", st);
  const int64_t ncell = (int64_t)sh.F * sh.R * sh.S;
  k_label_dense<<<grid_for(ncell, 256), 256, 0, st>>>(sh, node_ids, ws.parent, nmask, ws.rank, labels);
  prof_mark("label_dense", st);
}

template <int T, int ITEMS>
static void ring_fill(int mode, const lseg_sensor& sn, const Shape& sh, const double* ranges,
                      const int32_t* in, int32_t* out, int32_t* hist, const int32_t* remap,
                      const int32_t* fscal, int64_t K, int32_t m, cudaStream_t st) {
  const size_t smem = sizeof(int) * sh.S;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_ring_fill<T, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_ring_fill<T, ITEMS><<<sh.F * sh.R, T, smem, st>>>(mode, sn, sh, ranges, in, out, hist, remap,
                                                                     fscal, K, m);
}

void launch_ring_fill(int mode, const lseg_sensor& sn, const Shape& sh, const double* ranges,
                      const int32_t* in, int32_t* out, int32_t* hist, const int32_t* remap,
                      const int32_t* fscal, int64_t K, int32_t m, cudaStream_t st) {
  if (sh.S <= 1024) ring_fill<256, 4>(mode, sn, sh, ranges, in, out, hist, remap, fscal, K, m, st);
  else if (sh.S <= 4096) ring_fill<256, 16>(mode, sn, sh, ranges, in, out, hist, remap, fscal, K, m, st);
  else ring_fill<512, 32>(mode, sn, sh, ranges, in, out, hist, remap, fscal, K, m, st);  // S <= 16384
}

void launch_prune_plan(const Shape& sh, const int32_t* n_labels, int64_t K, int32_t m, const int32_t* hist,
                       int32_t* remap, int32_t* fscal, cudaStream_t st) {
  k_prune_plan<512, 8><<<sh.F, 512, 0, st>>>(n_labels, K, m, hist, remap, fscal);
}

void launch_hist(const Shape& sh, int64_t K, const int32_t* labels, int32_t* hist, cudaStream_t st) {
  const int64_t n = (int64_t)sh.F * sh.R * sh.S;
  k_hist<<<grid_for(n, 256), 256, 0, st>>>(sh, K, labels, hist);
}

void launch_triangles(int F, int R, int Sk, const int32_t* node_ids, int32_t* tris, int32_t* n_tris,
                      cudaStream_t st) {
  k_triangles<512><<<F, 512, 0, st>>>(R, Sk, node_ids, tris, n_tris);
}

}  // namespace lseg
