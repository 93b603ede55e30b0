// Streaming mesh builder (reference MeshBuilder,
// mesh.py:139-170, streaming contract SPEC.md:200): one kept azimuth column
// at a time, in sweep order, while the sensor spins.
//
// The join rules (mesh.py:83-102) relate a kept column only to its
// neighbouring kept columns, so when column j arrives every slot of column
// j-1 is known (N0 / N3 in column j-1, N1 / N2 in column j, N4 / N5 in column
// j-2) and is emitted right away; only the wrap (column S'-1 -> 0) waits for
// finish().  Node ids are row-major (mesh.py:115-117), i.e. id(i, c) =
// rowoff[i] + colrank(i, c) where colrank counts row i's valid cells before
// column c -- known when column c arrives -- and rowoff[i] needs every column
// of the rows above.  So slots are emitted as (ring, colrank) references and
// finish() resolves them: an O(R) scan of the per-ring counts plus one
// parallel renumbering pass over the kept cells.
//
// State (caller-owned device buffers; runcnt zeroed by the caller before column 0):
//   runcnt  (R) i32        valid cells per ring so far
//   colrank (R, S') i32    colrank of each valid kept cell, -1 invalid
//   slots   (R, S', 6) i32 (ring << 16 | colrank) of each present slot, -1 absent

#include "lseg_internal.cuh"
#include "lseg_kernels.cuh"

namespace lseg {

__device__ __forceinline__ int mb_ref(const int32_t* colrank, int Sk, int r, int c) {
  const int cr = colrank[r * Sk + c];
  return cr < 0 ? -1 : (r << 16) | cr;
}

// Slots N0..N5 of valid kept cell (i, c) (mesh.py:27, 87-101): (+1,0),
// (+1,+1), (0,+1), (-1,0), (-1,-1), (0,-1) in (ring, kept position), kept
// positions cyclic, rings not; with S' = 2 a slot equal to an earlier one
// (N5 == N2) is dropped.
__device__ __forceinline__ void mb_emit(const int32_t* colrank, int32_t* slots, int R, int Sk, int i, int c) {
  const int cp = c + 1 == Sk ? 0 : c + 1, cm = c == 0 ? Sk - 1 : c - 1;
  int32_t* o = slots + ((int64_t)i * Sk + c) * 6;
  o[0] = i + 1 < R ? mb_ref(colrank, Sk, i + 1, c) : -1;
  o[1] = i + 1 < R ? mb_ref(colrank, Sk, i + 1, cp) : -1;
  o[2] = mb_ref(colrank, Sk, i, cp);
  o[3] = i > 0 ? mb_ref(colrank, Sk, i - 1, c) : -1;
  o[4] = i > 0 ? mb_ref(colrank, Sk, i - 1, cm) : -1;
  o[5] = (Sk == 2) ? -1 : mb_ref(colrank, Sk, i, cm);
}

// Column j arrives: its valid bits and colranks, then the slots of column
// j-1 (all of whose neighbours now exist).  One CTA; the ring loop strides.
__global__ void k_mb_column(int R, int Sk, int j, double r_min, double r_max, const double* __restrict__ col,
                            int32_t* __restrict__ runcnt, int32_t* __restrict__ colrank, int32_t* __restrict__ slots) {
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    const bool v = in_window(col[i], r_min, r_max);
    const int n = runcnt[i];
    colrank[i * Sk + j] = v ? n : -1;
    runcnt[i] = n + (v ? 1 : 0);
  }
  __syncthreads();
  // column j-1 is complete once j arrives, except column 0 (its N4 / N5 wrap
  // to column S'-1): that one and the last column are finish()'s
  if (j >= 2)
    for (int i = threadIdx.x; i < R; i += blockDim.x)
      if (colrank[i * Sk + j - 1] >= 0) mb_emit(colrank, slots, R, Sk, i, j - 1);
}

// finish(): slots of column 0 and column S'-1 (the wrap), the per-ring
// offsets (exclusive scan of runcnt, O(R)), the frame's node count.
__global__ void k_mb_wrap(int R, int Sk, const int32_t* __restrict__ runcnt, const int32_t* __restrict__ colrank,
                          int32_t* __restrict__ slots, int32_t* __restrict__ rowoff, int32_t* __restrict__ n_nodes) {
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    if (colrank[i * Sk] >= 0) mb_emit(colrank, slots, R, Sk, i, 0);
    if (Sk > 1 && colrank[i * Sk + Sk - 1] >= 0) mb_emit(colrank, slots, R, Sk, i, Sk - 1);
  }
  if (threadIdx.x == 0) {  // R is small (rings of one sensor)
    int acc = 0;
    for (int i = 0; i < R; ++i) {
      rowoff[i] = acc;
      acc += runcnt[i];
    }
    *n_nodes = acc;
  }
}

// finish(): resolve (ring, colrank) references to row-major node ids.
__global__ void k_mb_resolve(int R, int Sk, const int32_t* __restrict__ colrank, const int32_t* __restrict__ slots,
                             const int32_t* __restrict__ rowoff, int32_t* __restrict__ node_ids,
                             int32_t* __restrict__ neighbors) {
  const int64_t n = (int64_t)R * Sk;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / Sk);
    const int cr = colrank[t];
    const int id = cr < 0 ? -1 : rowoff[i] + cr;
    node_ids[t] = id;
    if (id < 0) continue;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int ref = slots[t * 6 + s];
      neighbors[(int64_t)id * 6 + s] = ref < 0 ? -1 : rowoff[ref >> 16] + (ref & 0xffff);
    }
  }
}

void launch_mb_column(int R, int Sk, int j, double r_min, double r_max, const double* col, int32_t* runcnt,
                      int32_t* colrank, int32_t* slots, cudaStream_t st) {
  k_mb_column<<<1, R < 256 ? ((R + 31) / 32) * 32 : 256, 0, st>>>(R, Sk, j, r_min, r_max, col, runcnt, colrank, slots);
}

void launch_mb_finish(int R, int Sk, const int32_t* runcnt, const int32_t* colrank, int32_t* slots, int32_t* rowoff,
                      int32_t* node_ids, int32_t* neighbors, int32_t* n_nodes, cudaStream_t st) {
  k_mb_wrap<<<1, R < 256 ? ((R + 31) / 32) * 32 : 256, 0, st>>>(R, Sk, runcnt, colrank, slots, rowoff, n_nodes);
  const int64_t n = (int64_t)R * Sk;
  int64_t blocks = (n + 255) / 256;
  if (blocks > num_sms() * 16) blocks = num_sms() * 16;
  k_mb_resolve<<<(int)blocks, 256, 0, st>>>(R, Sk, colrank, slots, rowoff, node_ids, neighbors);
}

}  // namespace lseg
