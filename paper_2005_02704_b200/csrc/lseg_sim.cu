// Scan simulator: ray casting of scenes of geometric
// primitives, reference simulate.py:59-421.  One thread per beam; each
// primitive's intersection follows the reference's formulas (Plane
// :86-101, Sphere :121-133, Cylinder :161-200, Box :243-271, Cone :312-353)
// in fp64 with the same branch structure, and the nearest hit keeps the first
// primitive on ties (cast_grid :383-401, strict `t < best_t`).  The
// reference evaluates its dot products with numpy/BLAS, whose summation
// order and FMA use depend on the host CPU, so ranges agree to ~1 ulp rather
// than bit-for-bit (tests/test_sim.py states the tolerance).
//
// Packed primitive record (kPrimStride doubles, built by simulate.py:_pack):
//   [0] kind  0 plane, 1 sphere, 2 cylinder, 3 box, 4 cone
//   [1..6] surface id of face 0..5
//   plane    [7..9] point [10..12] normal [13] has extent [14,15] half sizes
//            [16..18] u [19..21] v   (_plane_axes, computed on the host)
//   sphere   [7..9] center [10] radius
//   cylinder [7..9] base [10..12] axis [13] radius [14] height
//   box      [7..9] center [10..12] half extents [13..21] rotation (row-major)
//   cone     [7..9] apex [10..12] axis [13] cos(half_angle)^2 [14] height
//            [15] height*tan(half_angle) [16] cos(half_angle) [17] sin(half_angle)

#include <math.h>

#include "lseg_internal.cuh"
#include "lseg_kernels.cuh"

namespace lseg {

static constexpr double kSimEps = 1e-12;  // simulate.py:23 _EPS
static constexpr double kInf = __builtin_huge_val();

struct V3 {
  double x, y, z;
};
__device__ __forceinline__ V3 v3(const double* p) { return V3{__ldg(p), __ldg(p + 1), __ldg(p + 2)}; }
__device__ __forceinline__ double dot3(const V3& a, const V3& b) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}
__device__ __forceinline__ V3 sub3(const V3& a, const V3& b) {
  return V3{__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)};
}
__device__ __forceinline__ V3 axpy3(double t, const V3& d, const V3& o) {  // o + t*d
  return V3{__dadd_rn(o.x, __dmul_rn(t, d.x)), __dadd_rn(o.y, __dmul_rn(t, d.y)), __dadd_rn(o.z, __dmul_rn(t, d.z))};
}
__device__ __forceinline__ V3 radial3(const V3& p, const V3& u) {  // p - (p.u) u
  const double s = dot3(p, u);
  return V3{__dsub_rn(p.x, __dmul_rn(s, u.x)), __dsub_rn(p.y, __dmul_rn(s, u.y)), __dsub_rn(p.z, __dmul_rn(s, u.z))};
}
__device__ __forceinline__ double norm_np(const V3& a) {  // numpy einsum / norm association
  return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.z, a.z)), __dmul_rn(a.y, a.y)));
}
__device__ __forceinline__ double dd_np(const V3& a) {  // einsum("ij,ij->i") of a row with itself
  return __dadd_rn(__dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.z, a.z)), __dmul_rn(a.y, a.y));
}
__device__ __forceinline__ double np_min(double a, double b) { return (isnan(a) || isnan(b)) ? NAN : (a < b ? a : b); }
__device__ __forceinline__ double np_max(double a, double b) { return (isnan(a) || isnan(b)) ? NAN : (a > b ? a : b); }

// Smallest t > eps of ray o + t d against primitive `rec`, and the face hit.
__device__ double prim_hit(const double* __restrict__ rec, const V3& o, const V3& d, int& face) {
  const int kind = (int)__ldg(rec);
  face = 0;
  if (kind == 0) {  // Plane
    const V3 pt = v3(rec + 7), n = v3(rec + 10);
    const double denom = dot3(d, n);
    const double offset = dot3(sub3(pt, o), n);
    double t = fabs(denom) > kSimEps ? __ddiv_rn(offset, denom) : kInf;
    t = t > kSimEps ? t : kInf;
    if (__ldg(rec + 13) != 0.0) {
      const V3 hit = axpy3(t, d, o);
      const V3 rel = sub3(hit, pt);
      const bool inside = fabs(dot3(rel, v3(rec + 16))) <= __ldg(rec + 14) &&
                          fabs(dot3(rel, v3(rec + 19))) <= __ldg(rec + 15);
      t = inside ? t : kInf;
    }
    return t;
  }
  if (kind == 1) {  // Sphere
    const V3 oc = sub3(o, v3(rec + 7));
    const double r = __ldg(rec + 10);
    const double b = dot3(d, oc);
    const double c = __dsub_rn(dot3(oc, oc), __dmul_rn(r, r));
    const double disc = __dsub_rn(__dmul_rn(b, b), c);
    const double sq = sqrt(fmax(disc, 0.0));
    const double t0 = __dsub_rn(-b, sq), t1 = __dadd_rn(-b, sq);
    double t = t0 > kSimEps ? t0 : (t1 > kSimEps ? t1 : kInf);
    return disc >= 0.0 ? t : kInf;
  }
  if (kind == 2) {  // Cylinder: faces 0 side, 1 bottom cap, 2 top cap
    const V3 u = v3(rec + 10);
    const double rad = __ldg(rec + 13), h = __ldg(rec + 14);
    const V3 ob = sub3(o, v3(rec + 7));
    const double os_ax = dot3(ob, u);
    const double d_ax = dot3(d, u);
    const V3 oc = {__dsub_rn(ob.x, __dmul_rn(os_ax, u.x)), __dsub_rn(ob.y, __dmul_rn(os_ax, u.y)),
                   __dsub_rn(ob.z, __dmul_rn(os_ax, u.z))};
    const V3 dc = {__dsub_rn(d.x, __dmul_rn(d_ax, u.x)), __dsub_rn(d.y, __dmul_rn(d_ax, u.y)),
                   __dsub_rn(d.z, __dmul_rn(d_ax, u.z))};
    const double a = dd_np(dc);
    const double b = dot3(dc, oc);
    const double c = __dsub_rn(dot3(oc, oc), __dmul_rn(rad, rad));
    const double disc = __dsub_rn(__dmul_rn(b, b), __dmul_rn(a, c));
    const double sq = sqrt(fmax(disc, 0.0));
    const double t0 = a > kSimEps ? __ddiv_rn(__dsub_rn(-b, sq), a) : kInf;
    const double t1 = a > kSimEps ? __ddiv_rn(__dadd_rn(-b, sq), a) : kInf;
    double best = kInf;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double tc = k ? t1 : t0;
      const double s = __dadd_rn(os_ax, __dmul_rn(tc, d_ax));
      if (disc >= 0.0 && tc > kSimEps && s >= 0.0 && s <= h && tc < best) best = tc;
    }
#pragma unroll
    for (int k = 1; k <= 2; ++k) {
      const double s_cap = (k == 1) ? 0.0 : h;
      const double tc = fabs(d_ax) > kSimEps ? __ddiv_rn(__dsub_rn(s_cap, os_ax), d_ax) : kInf;
      const bool fin = isfinite(tc);
      const V3 hit = axpy3(fin ? tc : 0.0, d, ob);
      const V3 radial = radial3(hit, u);
      if (fin && tc > kSimEps && dd_np(radial) <= __dmul_rn(rad, rad) && tc < best) {
        best = tc;
        face = k;
      }
    }
    return best;
  }
  if (kind == 3) {  // Box: slab method in the box frame, faces (+x,-x,+y,-y,+z,-z)
    const V3 oc = sub3(o, v3(rec + 7));
    const double* R = rec + 13;
    // (row vector) @ rotation: component j = sum_i v_i R[i][j]
    double ol[3], dl[3], hv[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      ol[j] = __dadd_rn(__dadd_rn(__dmul_rn(oc.x, __ldg(R + j)), __dmul_rn(oc.y, __ldg(R + 3 + j))),
                        __dmul_rn(oc.z, __ldg(R + 6 + j)));
      dl[j] = __dadd_rn(__dadd_rn(__dmul_rn(d.x, __ldg(R + j)), __dmul_rn(d.y, __ldg(R + 3 + j))),
                        __dmul_rn(d.z, __ldg(R + 6 + j)));
      hv[j] = __ldg(rec + 10 + j);
    }
    double tn[3], tf[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double inv = __drcp_rn(dl[j]);  // 1/0 -> inf like numpy
      const double tlo = __dmul_rn(__dsub_rn(-hv[j], ol[j]), inv);
      const double thi = __dmul_rn(__dsub_rn(hv[j], ol[j]), inv);
      const bool parallel = fabs(dl[j]) < kSimEps;
      const bool inside = fabs(ol[j]) <= hv[j];
      tn[j] = parallel ? (inside ? -kInf : kInf) : np_min(tlo, thi);
      tf[j] = parallel ? (inside ? kInf : -kInf) : np_max(tlo, thi);
    }
    const double t_near = np_max(np_max(tn[0], tn[1]), tn[2]);
    const double t_far = np_min(np_min(tf[0], tf[1]), tf[2]);
    const bool hit = t_near <= t_far && t_far > kSimEps;
    double t = t_near > kSimEps ? t_near : t_far;
    t = hit ? t : kInf;
    // argmax / argmin: first index of the extreme value
    int ax = 0, ex = 0;
    if (tn[1] > tn[ax]) ax = 1;
    if (tn[2] > tn[ax]) ax = 2;
    if (tf[1] < tf[ex]) ex = 1;
    if (tf[2] < tf[ex]) ex = 2;
    const int axis = t_near > kSimEps ? ax : ex;
    const double tt = isfinite(t) ? t : 0.0;
    const double hp = __dadd_rn(ol[axis], __dmul_rn(tt, dl[axis]));
    face = axis * 2 + (hp >= 0.0 ? 0 : 1);
    return t;
  }
  // Cone: faces 0 lateral, 1 base cap
  const V3 u = v3(rec + 10);
  const double cos2 = __ldg(rec + 13), h = __ldg(rec + 14), rb = __ldg(rec + 15);
  const V3 oa = sub3(o, v3(rec + 7));
  const double d_ax = dot3(d, u);
  const double o_ax = dot3(oa, u);
  const double d_o = dot3(d, oa);
  const double a = __dsub_rn(__dmul_rn(d_ax, d_ax), cos2);
  const double b = __dsub_rn(__dmul_rn(d_ax, o_ax), __dmul_rn(cos2, d_o));
  const double c = __dsub_rn(__dmul_rn(o_ax, o_ax), __dmul_rn(cos2, dot3(oa, oa)));
  const double disc = __dsub_rn(__dmul_rn(b, b), __dmul_rn(a, c));
  const double sq = sqrt(fmax(disc, 0.0));
  double roots[3];
  roots[0] = fabs(a) > kSimEps ? __ddiv_rn(__dsub_rn(-b, sq), a) : kInf;
  roots[1] = fabs(a) > kSimEps ? __ddiv_rn(__dadd_rn(-b, sq), a) : kInf;
  roots[2] = (fabs(a) <= kSimEps && fabs(b) > kSimEps) ? __ddiv_rn(-c, __dmul_rn(2.0, b)) : kInf;
  double best = kInf;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double tc = roots[k];
    const double s = __dadd_rn(o_ax, __dmul_rn(tc, d_ax));
    if (disc >= 0.0 && tc > kSimEps && s >= 0.0 && s <= h && tc < best) best = tc;
  }
  const double tc = fabs(d_ax) > kSimEps ? __ddiv_rn(__dsub_rn(h, o_ax), d_ax) : kInf;
  const bool fin = isfinite(tc);
  const V3 hit = axpy3(fin ? tc : 0.0, d, oa);
  const V3 radial = radial3(hit, u);
  if (fin && tc > kSimEps && dd_np(radial) <= __dmul_rn(rb, rb) && tc < best) {
    best = tc;
    face = 1;
  }
  return best;
}

__device__ __forceinline__ void cast_one(const double* __restrict__ prims, int n_prims, const V3& o, const V3& d,
                                         double& best_t, int& best_id) {
  best_t = kInf;
  best_id = 0;
  for (int p = 0; p < n_prims; ++p) {
    const double* rec = prims + (int64_t)p * kPrimStride;
    int face;
    const double t = prim_hit(rec, o, d, face);
    if (t < best_t) {
      best_t = t;
      best_id = (int)__ldg(rec + 1 + face);
    }
  }
}

// Beam directions from the sensor tables (reference ray_directions,
// scan.py:130-139), optionally rotated / offset by a per-frame pose
// (R row-major 3x3, then origin): world ray = origin + t * (R d).
__global__ void k_cast_grid(lseg_sensor sn, int F, const double* __restrict__ prims, int n_prims,
                            const double* __restrict__ poses, double* __restrict__ t_out,
                            int32_t* __restrict__ id_out) {
  const int64_t n = (int64_t)F * sn.rings * sn.steps;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = i % ((int64_t)sn.rings * sn.steps);
    const int f = (int)(i / ((int64_t)sn.rings * sn.steps));
    const int ring = (int)(cell / sn.steps), step = (int)(cell - (int64_t)ring * sn.steps);
    const double ct = __ldg(sn.cos_el + ring);
    V3 d = {__dmul_rn(ct, __ldg(sn.cos_az + step)), __dmul_rn(ct, __ldg(sn.sin_az + step)), __ldg(sn.sin_el + ring)};
    V3 o = {0.0, 0.0, 0.0};
    if (poses) {
      const double* P = poses + (int64_t)f * 12;
      const V3 dw = {dot3(v3(P), d), dot3(v3(P + 3), d), dot3(v3(P + 6), d)};
      d = dw;
      o = v3(P + 9);
    }
    double t;
    int id;
    cast_one(prims, n_prims, o, d, t, id);
    t_out[i] = t;
    id_out[i] = id;
  }
}

__global__ void k_cast_rays(const double* __restrict__ prims, int n_prims, int64_t n,
                            const double* __restrict__ origins, const double* __restrict__ dirs,
                            double* __restrict__ t_out, int32_t* __restrict__ id_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double t;
    int id;
    cast_one(prims, n_prims, v3(origins + 3 * i), v3(dirs + 3 * i), t, id);
    t_out[i] = t;
    id_out[i] = id;
  }
}

// scan_scene's noise + window (simulate.py:404-421): r = t (+ noise where the
// beam hit), invalid -> NaN with label 0.
__global__ void k_apply_scan(int64_t n, double r_min, double r_max, const double* __restrict__ t,
                             const int32_t* __restrict__ id, const double* __restrict__ noise,
                             double* __restrict__ ranges, int32_t* __restrict__ labels) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double r = t[i];
    if (noise && isfinite(r)) r = __dadd_rn(r, noise[i]);
    const bool valid = isfinite(r) && r >= r_min && r <= r_max;
    ranges[i] = valid ? r : __longlong_as_double(0x7ff8000000000000LL);
    labels[i] = valid ? id[i] : 0;
  }
}

// Analytic surface normal per labelled cell, oriented toward the sensor
// (scene_normals, simulate.py:424-448); NaN rows for label 0.
__global__ void k_scene_normals(lseg_sensor sn, const double* __restrict__ prims, int n_prims,
                                const double* __restrict__ ranges, const int32_t* __restrict__ labels,
                                double* __restrict__ out) {
  const int64_t n = (int64_t)sn.rings * sn.steps;
  const double qn = __longlong_as_double(0x7ff8000000000000LL);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int lab = labels[i];
    double* o = out + 3 * i;
    o[0] = o[1] = o[2] = qn;
    if (lab == 0) continue;
    const int ring = (int)(i / sn.steps), step = (int)(i - (int64_t)ring * sn.steps);
    const double r = ranges[i];
    const double ct = __ldg(sn.cos_el + ring);
    const V3 p = {__dmul_rn(__dmul_rn(ct, __ldg(sn.cos_az + step)), r),
                  __dmul_rn(__dmul_rn(ct, __ldg(sn.sin_az + step)), r), __dmul_rn(__ldg(sn.sin_el + ring), r)};
    // the primitive / face owning the label (ids are unique scene-wide)
    const double* rec = nullptr;
    int face = -1;
    for (int q = 0; q < n_prims && face < 0; ++q) {
      const double* rq = prims + (int64_t)q * kPrimStride;
      for (int fc = 0; fc < 6; ++fc)
        if ((int)__ldg(rq + 1 + fc) == lab) { rec = rq; face = fc; break; }
    }
    if (!rec) continue;
    const int kind = (int)__ldg(rec);
    V3 nv;
    if (kind == 0) {
      nv = v3(rec + 10);
    } else if (kind == 1) {
      const V3 rel = sub3(p, v3(rec + 7));
      const double l = norm_np(rel);
      nv = V3{__ddiv_rn(rel.x, l), __ddiv_rn(rel.y, l), __ddiv_rn(rel.z, l)};
    } else if (kind == 2) {
      const V3 u = v3(rec + 10);
      if (face == 0) {
        const V3 rad = radial3(sub3(p, v3(rec + 7)), u);
        const double l = norm_np(rad);
        nv = V3{__ddiv_rn(rad.x, l), __ddiv_rn(rad.y, l), __ddiv_rn(rad.z, l)};
      } else {
        nv = face == 1 ? V3{-u.x, -u.y, -u.z} : u;
      }
    } else if (kind == 3) {
      const int axis = face / 2;
      const double sg = (face % 2 == 0) ? 1.0 : -1.0;
      const double* R = rec + 13;  // local one-hot @ R^T: column `axis` of R
      nv = V3{__dmul_rn(sg, __ldg(R + axis)), __dmul_rn(sg, __ldg(R + 3 + axis)), __dmul_rn(sg, __ldg(R + 6 + axis))};
      nv = V3{__dadd_rn(nv.x, 0.0), __dadd_rn(nv.y, 0.0), __dadd_rn(nv.z, 0.0)};
    } else {
      const V3 u = v3(rec + 10);
      if (face == 0) {
        const V3 rad = radial3(sub3(p, v3(rec + 7)), u);
        const double l = norm_np(rad);
        const double ch = __ldg(rec + 16), shh = __ldg(rec + 17);
        nv = V3{__dsub_rn(__dmul_rn(__ddiv_rn(rad.x, l), ch), __dmul_rn(u.x, shh)),
                __dsub_rn(__dmul_rn(__ddiv_rn(rad.y, l), ch), __dmul_rn(u.y, shh)),
                __dsub_rn(__dmul_rn(__ddiv_rn(rad.z, l), ch), __dmul_rn(u.z, shh))};
        if (isnan(nv.x)) nv.x = 0.0;  // nan_to_num (apex)
        if (isnan(nv.y)) nv.y = 0.0;
        if (isnan(nv.z)) nv.z = 0.0;
      } else {
        nv = u;
      }
    }
    const double dt = __dadd_rn(__dadd_rn(__dmul_rn(nv.x, p.x), __dmul_rn(nv.z, p.z)), __dmul_rn(nv.y, p.y));
    if (dt > 0.0) nv = V3{-nv.x, -nv.y, -nv.z};
    o[0] = nv.x;
    o[1] = nv.y;
    o[2] = nv.z;
  }
}

static int sim_grid(int64_t n) {
  const int64_t b = (n + 127) / 128;
  return (int)(b > num_sms() * 16 ? num_sms() * 16 : (b < 1 ? 1 : b));
}

void launch_cast_grid(const lseg_sensor& sn, int F, const double* prims, int n_prims, const double* poses,
                      double* t, int32_t* id, cudaStream_t st) {
  const int64_t n = (int64_t)F * sn.rings * sn.steps;
  if (n == 0) return;
  k_cast_grid<<<sim_grid(n), 128, 0, st>>>(sn, F, prims, n_prims, poses, t, id);
}

void launch_cast_rays(const double* prims, int n_prims, int64_t n, const double* origins, const double* dirs,
                      double* t, int32_t* id, cudaStream_t st) {
  if (n == 0) return;
  k_cast_rays<<<sim_grid(n), 128, 0, st>>>(prims, n_prims, n, origins, dirs, t, id);
}

void launch_apply_scan(int64_t n, double r_min, double r_max, const double* t, const int32_t* id,
                       const double* noise, double* ranges, int32_t* labels, cudaStream_t st) {
  if (n == 0) return;
  k_apply_scan<<<sim_grid(n), 128, 0, st>>>(n, r_min, r_max, t, id, noise, ranges, labels);
}

void launch_scene_normals(const lseg_sensor& sn, const double* prims, int n_prims, const double* ranges,
                          const int32_t* labels, double* out, cudaStream_t st) {
  const int64_t n = (int64_t)sn.rings * sn.steps;
  if (n == 0) return;
  k_scene_normals<<<sim_grid(n), 128, 0, st>>>(sn, prims, n_prims, ranges, labels, out);
}

}  // namespace lseg
