// Edge precision / recall evaluator, reference
// evaluate.py:40-94: a labelled cell is an edge cell when one of its 4 grid
// neighbours (azimuth wraps, rings clamp) holds a different nonzero label;
// predicted and truth edge sets are matched after a Chebyshev dilation.
// Batched over frames; edge sets are kept as bit words (1 bit per cell).

#include "lseg_internal.cuh"
#include "lseg_kernels.cuh"

namespace lseg {

struct EvalShape {
  int F, R, S, W;  // frames, rings, steps, 32-bit words per row
};

__device__ __forceinline__ bool edge_at(const int32_t* __restrict__ lab, const EvalShape& e, int64_t fr, int i,
                                        int c) {
  const int32_t* row = lab + (fr * e.R + i) * e.S;
  const int v = __ldg(row + c);
  if (v <= 0) return false;
  const int l = __ldg(row + (c == 0 ? e.S - 1 : c - 1));
  const int r = __ldg(row + (c + 1 == e.S ? 0 : c + 1));
  bool edge = (l > 0 && l != v) || (r > 0 && r != v);
  if (i > 0) {
    const int u = __ldg(row - e.S + c);
    edge |= (u > 0 && u != v);
  }
  if (i + 1 < e.R) {
    const int d = __ldg(row + e.S + c);
    edge |= (d > 0 && d != v);
  }
  return edge;
}

// Edge bit words of a label grid (blockIdx.y selects one of two grids).
__global__ void k_edge_bits(EvalShape e, const int32_t* __restrict__ a, const int32_t* __restrict__ b,
                            uint32_t* __restrict__ bits_a, uint32_t* __restrict__ bits_b) {
  const int32_t* lab = blockIdx.y ? b : a;
  uint32_t* bits = blockIdx.y ? bits_b : bits_a;
  if (!lab) return;
  const int64_t nwords = (int64_t)e.F * e.R * e.W;
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nwords;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t row = w / e.W;
    const int c = (int)(w - row * e.W) * 32 + lane;
    const int64_t fr = row / e.R;
    const int i = (int)(row - fr * e.R);
    const bool ed = (c < e.S) && edge_at(lab, e, fr, i, c);
    const uint32_t m = __ballot_sync(0xffffffffu, ed);
    if (lane == 0) bits[w] = m;
  }
}

__device__ __forceinline__ bool bit_at(const uint32_t* __restrict__ bits, const EvalShape& e, int64_t fr, int i,
                                       int c) {
  return (__ldg(bits + (fr * e.R + i) * e.W + (c >> 5)) >> (c & 31)) & 1u;
}

// Is any bit set within Chebyshev radius r of (i, c)?  Rings clamp, azimuth wraps
// (reference dilate_chebyshev, evaluate.py:58-70).
__device__ __forceinline__ bool dilated(const uint32_t* __restrict__ bits, const EvalShape& e, int64_t fr, int i,
                                        int c, int r) {
  const int i0 = max(0, i - r), i1 = min(e.R - 1, i + r);
  for (int ii = i0; ii <= i1; ++ii)
    for (int dc = -r; dc <= r; ++dc) {
      int cc = c + dc;
      cc = ((cc % e.S) + e.S) % e.S;
      if (bit_at(bits, e, fr, ii, cc)) return true;
    }
  return false;
}

// Per frame: n_pred, n_truth, pred edges near a truth edge, truth edges near a pred edge.
__global__ void k_edge_counts(EvalShape e, const uint32_t* __restrict__ pe, const uint32_t* __restrict__ te, int r,
                              int32_t* __restrict__ counts) {
  const int64_t n = (int64_t)e.F * e.R * e.S;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / e.S;
    const int c = (int)(t - row * e.S);
    const int64_t fr = row / e.R;
    const int i = (int)(row - fr * e.R);
    const bool p = bit_at(pe, e, fr, i, c), q = bit_at(te, e, fr, i, c);
    int v0 = p, v1 = q, v2 = 0, v3 = 0;
    if (p) v2 = dilated(te, e, fr, i, c, r);
    if (q) v3 = dilated(pe, e, fr, i, c, r);
    if (v0 | v1) {
      int32_t* cf = counts + fr * 4;
      if (v0) atomicAdd(cf + 0, 1);
      if (v1) atomicAdd(cf + 1, 1);
      if (v2) atomicAdd(cf + 2, 1);
      if (v3) atomicAdd(cf + 3, 1);
    }
  }
}

// Byte masks for the single-grid API functions.
__global__ void k_bits_to_bytes(EvalShape e, const uint32_t* __restrict__ bits, uint8_t* __restrict__ out) {
  const int64_t n = (int64_t)e.F * e.R * e.S;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / e.S;
    const int c = (int)(t - row * e.S);
    out[t] = (__ldg(bits + row * e.W + (c >> 5)) >> (c & 31)) & 1u;
  }
}

__global__ void k_bytes_to_bits(EvalShape e, const uint8_t* __restrict__ in, uint32_t* __restrict__ bits) {
  const int64_t nwords = (int64_t)e.F * e.R * e.W;
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nwords;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t row = w / e.W;
    const int c = (int)(w - row * e.W) * 32 + lane;
    const uint32_t m = __ballot_sync(0xffffffffu, c < e.S && in[row * e.S + c]);
    if (lane == 0) bits[w] = m;
  }
}

__global__ void k_dilate_bytes(EvalShape e, const uint32_t* __restrict__ bits, int r, uint8_t* __restrict__ out) {
  const int64_t n = (int64_t)e.F * e.R * e.S;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / e.S;
    const int c = (int)(t - row * e.S);
    const int64_t fr = row / e.R;
    out[t] = dilated(bits, e, fr, (int)(row - fr * e.R), c, r) ? 1 : 0;
  }
}

static int grid_of(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)(b > num_sms() * 32 ? num_sms() * 32 : (b < 1 ? 1 : b));
}

size_t eval_workspace_bytes(int F, int R, int S) {
  const size_t words = (size_t)F * R * ((S + 31) / 32);
  return 2 * ((words * 4 + 255) & ~(size_t)255);
}

int eval_counts(int F, int R, int S, const int32_t* pred, const int32_t* truth, int r, int32_t* counts, void* ws,
                cudaStream_t st) {
  EvalShape e{F, R, S, (S + 31) / 32};
  const size_t words = (size_t)F * R * e.W;
  uint32_t* pe = static_cast<uint32_t*>(ws);
  uint32_t* te = pe + ((words * 4 + 255) & ~(size_t)255) / 4;
  cudaMemsetAsync(counts, 0, sizeof(int32_t) * 4 * F, st);
  k_edge_bits<<<dim3(grid_of((int64_t)words * 32), 2), 256, 0, st>>>(e, pred, truth, pe, te);
  k_edge_counts<<<grid_of((int64_t)F * R * S), 256, 0, st>>>(e, pe, te, r, counts);
  return check_launch("edge_counts");
}

int eval_extract(int F, int R, int S, const int32_t* labels, uint8_t* out, void* ws, cudaStream_t st) {
  EvalShape e{F, R, S, (S + 31) / 32};
  const size_t words = (size_t)F * R * e.W;
  uint32_t* bits = static_cast<uint32_t*>(ws);
  k_edge_bits<<<dim3(grid_of((int64_t)words * 32), 1), 256, 0, st>>>(e, labels, nullptr, bits, nullptr);
  k_bits_to_bytes<<<grid_of((int64_t)F * R * S), 256, 0, st>>>(e, bits, out);
  return check_launch("extract_edges");
}

int eval_dilate(int F, int R, int S, const uint8_t* mask, int r, uint8_t* out, void* ws, cudaStream_t st) {
  EvalShape e{F, R, S, (S + 31) / 32};
  const size_t words = (size_t)F * R * e.W;
  uint32_t* bits = static_cast<uint32_t*>(ws);
  k_bytes_to_bits<<<grid_of((int64_t)words * 32), 256, 0, st>>>(e, mask, bits);
  k_dilate_bytes<<<grid_of((int64_t)F * R * S), 256, 0, st>>>(e, bits, r, out);
  return check_launch("dilate_chebyshev");
}

}  // namespace lseg
