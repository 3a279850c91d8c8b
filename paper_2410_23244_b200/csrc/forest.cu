// Forest kernels outside the per-iteration sweep.
//
//   traverse   trees.traverse_forest (trees.py:174-203): D-1 fixed levels, a
//              point stops at the first node with cutpoint 0, goes right iff
//              x[axis] >= cutpoint (trees.py:154-171).  Output in the (m, n)
//              tree-major cache layout.
//   predict    trees.sum_leaf_values (trees.py:206-218): f64 accumulation in
//              tree order, so cached and fresh-traversal predictions agree
//              bit for bit with the reference.
//   evaluate   trees.evaluate_forest (trees.py:221-223) fused: traverse + sum
//              per point without materialising the (m, n) index matrix.
//   transpose  byte-matrix layout changes at the host boundary: the
//              reference's (n, p) X and (n, m) leaf index <-> our (p, n) / (m, n).
#include "common.cuh"
#include "internal.h"

namespace bart {

// dst[c * dst_ld + r] = src[r * src_ld + c] for r < rows, c < cols; one
// 32x32 tile per CTA over a 1-D grid (either dimension may exceed 65535 tiles)
__global__ void transpose_u8_kernel(const uint8_t *__restrict__ src, int64_t rows, int64_t cols, int64_t src_ld,
                                    uint8_t *__restrict__ dst, int64_t dst_ld, int64_t col_tiles) {
  __shared__ uint8_t tile[32][33];
  const int64_t tr = (int64_t)blockIdx.x / col_tiles, tc = (int64_t)blockIdx.x % col_tiles;
  const int64_t r0 = tr * 32, c0 = tc * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = r0 + k, cc = c0 + tx;
    if (r < rows && cc < cols) tile[k][tx] = src[r * src_ld + cc];
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int64_t cc = c0 + k, r = r0 + tx;
    if (r < rows && cc < cols) dst[cc * dst_ld + r] = tile[tx][k];
  }
}

void launch_transpose_u8(const uint8_t *src, int64_t rows, int64_t cols, int64_t src_ld, uint8_t *dst,
                         int64_t dst_ld, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  const int64_t rt = (rows + 31) / 32, ct = (cols + 31) / 32;
  transpose_u8_kernel<<<(unsigned)(rt * ct), 256, 0, s>>>(src, rows, cols, src_ld, dst, dst_ld, ct);
}

__global__ void fill_root_kernel(uint8_t *L, int m, int64_t n, int64_t n_pad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i < n_pad && j < m) L[(size_t)j * n_pad + i] = i < n ? 1 : 0;
}

void launch_fill_root(uint8_t *L, int m, int64_t n, int64_t n_pad, cudaStream_t s) {
  const dim3 grid((unsigned)((n_pad + 255) / 256), (unsigned)m);
  fill_root_kernel<<<grid, 256, 0, s>>>(L, m, n, n_pad);
}

__device__ __forceinline__ int descend(const uint8_t *cut, const uint16_t *axis, const uint8_t *Xt, int64_t ld,
                                       int64_t i, int D) {
  int idx = 1;
  bool done = false;
  for (int lvl = 0; lvl < D - 1; ++lvl) {
    const int split = cut[idx];
    done = done || split == 0;
    const int x = Xt[(size_t)axis[idx] * ld + i];
    const int child = 2 * idx + (x >= split ? 1 : 0);
    idx = done ? idx : child;
  }
  return idx;
}

// grid (words, m): one thread per 4 points of one tree
__global__ void traverse_kernel(const uint8_t *__restrict__ Xt, int64_t n, int64_t ld, int D, int half,
                                const uint16_t *__restrict__ axis, const uint8_t *__restrict__ cut,
                                uint8_t *__restrict__ L) {
  __shared__ uint8_t s_cut[kSlotsMax];
  __shared__ uint16_t s_ax[kSlotsMax];
  const int j = blockIdx.y;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    s_cut[i] = cut[(size_t)j * half + i];
    s_ax[i] = axis[(size_t)j * half + i];
  }
  __syncthreads();
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w * 4 >= ld) return;
  uint32_t out = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int64_t i = w * 4 + b;
    const uint32_t v = i < n ? (uint32_t)descend(s_cut, s_ax, Xt, ld, i, D) : 0u;
    out |= v << (8 * b);
  }
  reinterpret_cast<uint32_t *>(L + (size_t)j * ld)[w] = out;
}

void launch_traverse(const uint8_t *Xt, int64_t n, int64_t ld, int D, int half, int m, const uint16_t *axis,
                     const uint8_t *cut, uint8_t *L, cudaStream_t s) {
  const int64_t words = ld / 4;
  const dim3 grid((unsigned)((words + 255) / 256), (unsigned)m);
  traverse_kernel<<<grid, 256, 0, s>>>(Xt, n, ld, D, half, axis, cut, L);
}

// yhat[i] = sum_j leaf[j, L[j, i]] accumulated in f64, j ascending
__global__ void predict_cached_kernel(const uint8_t *__restrict__ L, int64_t n, int64_t ld, int m, int size,
                                      const float *__restrict__ leaf, double *__restrict__ out) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w * 4 >= ld) return;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int j = 0; j < m; ++j) {
    const uint32_t l = reinterpret_cast<const uint32_t *>(L + (size_t)j * ld)[w];
    const float *row = leaf + (size_t)j * size;
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[b] = __dadd_rn(acc[b], (double)__ldg(row + ((l >> (8 * b)) & 0xffu)));
  }
#pragma unroll
  for (int b = 0; b < 4; ++b)
    if (w * 4 + b < n) out[w * 4 + b] = acc[b];
}

void launch_predict_cached(const uint8_t *L, int64_t n, int64_t ld, int m, int size, const float *leaf,
                           double *out, cudaStream_t s) {
  const int64_t words = ld / 4;
  predict_cached_kernel<<<(unsigned)((words + 255) / 256), 256, 0, s>>>(L, n, ld, m, size, leaf, out);
}

// fused traverse + sum over all trees (forest staged through shared memory)
__global__ void evaluate_kernel(const uint8_t *__restrict__ Xt, int64_t n, int64_t ld, int D, int half, int m,
                                const uint16_t *__restrict__ axis, const uint8_t *__restrict__ cut,
                                const float *__restrict__ leaf, double *__restrict__ out) {
  constexpr int kTreesPerStage = 32;
  __shared__ uint8_t s_cut[kTreesPerStage][kSlotsMax];
  __shared__ uint16_t s_ax[kTreesPerStage][kSlotsMax];
  __shared__ float s_leaf[kTreesPerStage][2 * kSlotsMax];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int size = 2 * half;
  double acc = 0.0;
  for (int j0 = 0; j0 < m; j0 += kTreesPerStage) {
    const int nt = m - j0 < kTreesPerStage ? m - j0 : kTreesPerStage;
    __syncthreads();
    for (int k = threadIdx.x; k < nt * half; k += blockDim.x) {
      const int jj = k / half, h = k % half;
      s_cut[jj][h] = cut[(size_t)(j0 + jj) * half + h];
      s_ax[jj][h] = axis[(size_t)(j0 + jj) * half + h];
    }
    for (int k = threadIdx.x; k < nt * size; k += blockDim.x) {
      const int jj = k / size, h = k % size;
      s_leaf[jj][h] = leaf[(size_t)(j0 + jj) * size + h];
    }
    __syncthreads();
    if (i < n)
      for (int jj = 0; jj < nt; ++jj) {
        const int l = descend(s_cut[jj], s_ax[jj], Xt, ld, i, D);
        acc = __dadd_rn(acc, (double)s_leaf[jj][l]);
      }
  }
  if (i < n) out[i] = acc;
}

void launch_evaluate(const uint8_t *Xt, int64_t n, int64_t ld, int D, int half, int m, const uint16_t *axis,
                     const uint8_t *cut, const float *leaf, double *out, cudaStream_t s) {
  evaluate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(Xt, n, ld, D, half, m, axis, cut, leaf, out);
}

// r = f32(f64(y) - pred)  (tests/util.py:19-23 recomputation)
__global__ void resid_kernel(const float *__restrict__ y, const double *__restrict__ pred, float *__restrict__ r,
                             int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) r[i] = __double2float_rn(__dsub_rn((double)y[i], pred[i]));
}

void launch_resid(const float *y, const double *pred, float *r, int64_t n, cudaStream_t s) {
  resid_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(y, pred, r, n);
}

}  // namespace bart

namespace bart {

// fit() trace, one kept draw (regression.py:191-200): the sum of trees at the
// training rows from the cached leaf index (f64, tree order, as sum_leaf_values,
// trees.py:206-218), folded into per-point running moments (Welford, draw
// number k >= 1), optionally stored whole and at the first npts rows.
__global__ void trace_train_kernel(const uint8_t *__restrict__ L, int64_t n, int64_t ld, int m, int size,
                                   const float *__restrict__ leaf, double k, double *__restrict__ mean,
                                   double *__restrict__ m2, double *__restrict__ draw, double *__restrict__ pts,
                                   int npts) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w * 4 >= ld) return;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int j = 0; j < m; ++j) {
    const uint32_t l = reinterpret_cast<const uint32_t *>(L + (size_t)j * ld)[w];
    const float *row = leaf + (size_t)j * size;
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[b] = __dadd_rn(acc[b], (double)__ldg(row + ((l >> (8 * b)) & 0xffu)));
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int64_t i = w * 4 + b;
    if (i >= n) break;
    const double x = acc[b], mu = mean[i], d = x - mu, mu2 = mu + d / k;
    mean[i] = mu2;
    m2[i] += d * (x - mu2);
    if (draw) draw[i] = x;
    if (i < npts) pts[i] = x;
  }
}

// leaves per tree, averaged: every nonzero cutpoint is an internal node of a
// valid heap tree, and a binary tree has one more leaf than internal nodes
__global__ void mean_leaves_kernel(const uint8_t *__restrict__ cut, int m, int half, double *__restrict__ out) {
  __shared__ int part[32];
  int cnt = 0;
  for (int i = threadIdx.x; i < m * half; i += blockDim.x) cnt += cut[i] != 0;
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += part[k];
    *out = (double)(t + m) / (double)m;
  }
}

void launch_trace_train(const uint8_t *L, int64_t n, int64_t ld, int m, int size, const float *leaf, int64_t k,
                        double *mean, double *m2, double *draw, double *pts, int npts, cudaStream_t s) {
  const int64_t words = ld / 4;
  trace_train_kernel<<<(unsigned)((words + 255) / 256), 256, 0, s>>>(L, n, ld, m, size, leaf, (double)k, mean, m2,
                                                                     draw, pts, npts);
}

void launch_mean_leaves(const uint8_t *cut, int m, int half, double *out, cudaStream_t s) {
  mean_leaves_kernel<<<1, 1024, 0, s>>>(cut, m, half, out);
}

}  // namespace bart
