// Forest kernels outside the per-iteration sweep.
//
//   traverse   trees.traverse_forest (trees.py:174-203): a point stops at the
//              first node with cutpoint 0 and goes right iff x[axis] >= cutpoint
//              (trees.py:154-171).  Output in the (m, n) tree-major cache layout.
//
// Layout of the traverse / evaluate kernels: each thread owns 16 consecutive
// points (one 16-byte vector of every X column and cache row) and walks all
// trees.
// A tree is applied node by node in heap order, SWAR over the 16 point bytes
// (common.cuh swar_step, 11 integer ops per 4 points; the root, where every
// point starts, in 5): points at internal node t move to 2t + (x >= cut) --
// equivalent to the reference's per-point descent, since parents precede
// children in heap order.  traverse: the warp finds the tree's internal nodes
// with one ballot per 32 heap slots and broadcasts (node, axis, cut) by
// shuffle; evaluate: from a per-block node list in shared memory.  X is read as
// one coalesced 16-byte load per (internal node, thread) and the cache written
// as one 16-byte store per (tree, thread).
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

// dst[c * dst_ld + r] = src[r * src_ld + c] for r < rows, c < cols.
// 64 x 64-byte tiles over a 1-D grid (either dimension may exceed 65535
// tiles); 256 threads.  Loads: 4-byte words when rows are 4-byte aligned
// (W4), else bytes; stores: 16-byte vectors when destination rows are 16-byte
// aligned (V16), else bytes.  Out-of-range source bytes read as 0, so the
// destination's padding (dst_ld > rows) is written with zeros.
template <bool W4, bool V16>
__global__ void __launch_bounds__(256) transpose_u8_kernel(const uint8_t *__restrict__ src, int64_t rows, int64_t cols,
                                                           int64_t src_ld, uint8_t *__restrict__ dst, int64_t dst_ld,
                                                           int64_t col_tiles) {
  __shared__ uint8_t tile[64][68];
  const int64_t tr = (int64_t)blockIdx.x / col_tiles, tc = (int64_t)blockIdx.x % col_tiles;
  const int64_t r0 = tr * 64, c0 = tc * 64;
  const int t = threadIdx.x;
  {  // load: thread t -> source row t / 4, 16 columns from (t % 4) * 16
    const int rr = t >> 2, cc = (t & 3) * 16;
    const int64_t r = r0 + rr;
    uint8_t b[16];
    if (W4 && r < rows && c0 + cc + 16 <= cols) {
      const uint32_t *p = reinterpret_cast<const uint32_t *>(src + r * src_ld + c0 + cc);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t w = __ldg(p + k);
#pragma unroll
        for (int q = 0; q < 4; ++q) b[4 * k + q] = (uint8_t)(w >> (8 * q));
      }
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int64_t c = c0 + cc + k;
        b[k] = (r < rows && c < cols) ? __ldg(src + r * src_ld + c) : (uint8_t)0;
      }
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[rr][cc + k] = b[k];
  }
  __syncthreads();
  {  // store: thread t -> destination row (source column) t / 4, 16 source rows from (t % 4) * 16
    const int cc = t >> 2, rr = (t & 3) * 16;
    const int64_t c = c0 + cc, r = r0 + rr;
    if (c >= cols) return;
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      w[k] = (uint32_t)tile[rr + 4 * k][cc] | ((uint32_t)tile[rr + 4 * k + 1][cc] << 8) |
             ((uint32_t)tile[rr + 4 * k + 2][cc] << 16) | ((uint32_t)tile[rr + 4 * k + 3][cc] << 24);
    if (V16) {
      if (r < dst_ld) *reinterpret_cast<uint4 *>(dst + c * dst_ld + r) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (r + k < dst_ld && r + k < rows) dst[c * dst_ld + r + k] = (uint8_t)(w[k >> 2] >> (8 * (k & 3)));
    }
  }
}

void launch_transpose_u8(const uint8_t *src, int64_t rows, int64_t cols, int64_t src_ld, uint8_t *dst,
                         int64_t dst_ld, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  const int64_t rt = (rows + 63) / 64, ct = (cols + 63) / 64;
  const bool w4 = src_ld % 4 == 0 && reinterpret_cast<uintptr_t>(src) % 4 == 0;
  const bool v16 = dst_ld % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0;
  const unsigned g = (unsigned)(rt * ct);
  if (w4 && v16)
    transpose_u8_kernel<true, true><<<g, 256, 0, s>>>(src, rows, cols, src_ld, dst, dst_ld, ct);
  else if (w4)
    transpose_u8_kernel<true, false><<<g, 256, 0, s>>>(src, rows, cols, src_ld, dst, dst_ld, ct);
  else if (v16)
    transpose_u8_kernel<false, true><<<g, 256, 0, s>>>(src, rows, cols, src_ld, dst, dst_ld, ct);
  else
    transpose_u8_kernel<false, false><<<g, 256, 0, s>>>(src, rows, cols, src_ld, dst, dst_ld, ct);
}

// every point at the root (1), padding points 0: two strided memsets run at
// copy bandwidth (the per-byte kernel they replace ran at 0.5 TB/s)
void launch_fill_root(uint8_t *L, int m, int64_t n, int64_t n_pad, cudaStream_t s) {
  if (m <= 0 || n_pad <= 0) return;
  if (n > 0) cudaMemset2DAsync(L, (size_t)n_pad, 1, (size_t)n, (size_t)m, s);
  if (n_pad > n) cudaMemset2DAsync(L + n, (size_t)n_pad, 0, (size_t)(n_pad - n), (size_t)m, s);
}

// K words (4K points) per thread: the X column / cache-row vector type
template <int K> struct Vec;
template <> struct Vec<1> { typedef uint32_t T; };
template <> struct Vec<2> { typedef uint2 T; };
template <> struct Vec<4> { typedef uint4 T; };
template <> struct Vec<8> { typedef uint4 T; };  // (vload: two vectors)
template <int K>
__device__ __forceinline__ void vload(uint32_t (&w)[K], const uint8_t *p) {
  if constexpr (K == 8) {  // two 16-byte vectors
    const uint4 a = __ldg(reinterpret_cast<const uint4 *>(p)), b = __ldg(reinterpret_cast<const uint4 *>(p) + 1);
    w[0] = a.x, w[1] = a.y, w[2] = a.z, w[3] = a.w, w[4] = b.x, w[5] = b.y, w[6] = b.z, w[7] = b.w;
  } else {
    const typename Vec<K>::T v = __ldg(reinterpret_cast<const typename Vec<K>::T *>(p));
    memcpy(w, &v, sizeof(w));
  }
}
template <int K>
__device__ __forceinline__ void vstore(uint8_t *p, const uint32_t (&w)[K]) {
  typename Vec<K>::T v;
  memcpy(&v, w, sizeof(w));
  *reinterpret_cast<typename Vec<K>::T *>(p) = v;
}

// Leaf indices (bytes of l) of the thread's 4K points in tree j.  Every lane
// of the warp must call it (ballot / shuffle); lanes past the row read nothing.
// The internal nodes are taken kNodeBatch at a time: all their X column loads
// are issued before the first SWAR step, so a tree of several internal nodes
// waits for one memory latency instead of one per node (heap order, hence the
// reference's descent, is kept: nodes are applied in ascending index).
#ifndef BART_NODE_BATCH
#define BART_NODE_BATCH 1
#endif
constexpr int kNodeBatch = BART_NODE_BATCH;

template <int K>
__device__ __forceinline__ void traverse_pts(uint32_t (&l)[K], const uint8_t *__restrict__ Xt, int64_t ld, int64_t i0,
                                             bool live, const uint8_t *__restrict__ cut_j,
                                             const uint16_t *__restrict__ ax_j, int half, int lane) {
#pragma unroll
  for (int k = 0; k < K; ++k) l[k] = 0x01010101u;
  for (int base = 0; base < half; base += 32) {
    const int t = base + lane;
    const uint32_t ct = t < half ? __ldg(cut_j + t) : 0u, at = t < half ? __ldg(ax_j + t) : 0u;
    uint32_t msk = __ballot_sync(0xffffffffu, ct != 0u && t >= 1);
    while (msk) {  // warp-uniform
      uint32_t x[kNodeBatch][K], node[kNodeBatch], cv[kNodeBatch];
      bool use[kNodeBatch];
#pragma unroll
      for (int g = 0; g < kNodeBatch; ++g) {
        use[g] = msk != 0u;
        node[g] = 0u;
        cv[g] = 0u;
        if (use[g]) {
          const int src = __ffs(msk) - 1;
          msk &= msk - 1u;
          node[g] = (uint32_t)(base + src);
          cv[g] = __shfl_sync(0xffffffffu, ct, src);
          const uint32_t av = __shfl_sync(0xffffffffu, at, src);
          if (live) vload<K>(x[g], Xt + (size_t)av * ld + i0);
        }
      }
#pragma unroll
      for (int g = 0; g < kNodeBatch; ++g) {
        if (use[g] && live) {
          const uint32_t t4 = 0x01010101u * node[g], c4 = 0x01010101u * cv[g], b4 = 0x01010101u * (2u * node[g]);
          if (node[g] == 1u) {  // the root (first in heap order): every point is there
#pragma unroll
            for (int k = 0; k < K; ++k) l[k] = swar_child(x[g][k], c4, c4 & 0x7f7f7f7fu, b4);
          } else {
#pragma unroll
            for (int k = 0; k < K; ++k) l[k] = swar_step(l[k], x[g][k], t4, c4, b4);
          }
        }
      }
    }
  }
}

// bytes of the thread's points that lie below n (padding points -> 0)
template <int K>
__device__ __forceinline__ void valid_pts(uint32_t (&v)[K], int64_t i0, int64_t n) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int64_t left = n - (i0 + 4 * k);
    v[k] = left >= 4 ? 0xffffffffu : (left <= 0 ? 0u : (0xffffffffu >> (8 * (4 - (int)left))));
  }
}

constexpr int kTravWords = 4;  // 16 points per thread (tools: 8 measured 20% slower at n = 1e6)
constexpr int kTravTrees = 4;  // trees per traverse block (grid y)
// leaf values staged in shared memory as f64, kLeafStage doubles per block
// (the conversion once per leaf instead of once per point and tree)
constexpr int kLeafStage = 4096;

__global__ void __launch_bounds__(256) traverse_kernel(const uint8_t *__restrict__ Xt, int64_t n, int64_t ld, int half,
                                                       int m, const uint16_t *__restrict__ axis,
                                                       const uint8_t *__restrict__ cut, uint8_t *__restrict__ L) {
  constexpr int K = kTravWords;
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4 * K;
  const bool live = i0 < ld;
  const int lane = threadIdx.x & 31;
  uint32_t v[K], l[K];
  valid_pts<K>(v, i0, n);
  // blockIdx.y: a group of kTravTrees trees (independent outputs), so enough
  // warps are in flight to cover the X column loads' latency
  const int j0 = blockIdx.y * kTravTrees, j1 = j0 + kTravTrees < m ? j0 + kTravTrees : m;
  for (int j = j0; j < j1; ++j) {
    traverse_pts<K>(l, Xt, ld, i0, live, cut + (size_t)j * half, axis + (size_t)j * half, half, lane);
    if (live) {
#pragma unroll
      for (int k = 0; k < K; ++k) l[k] &= v[k];
      vstore<K>(L + (size_t)j * ld + i0, l);
    }
  }
}

static unsigned grid_for(int64_t ld, int words) { return (unsigned)((ld / (4 * words) + 255) / 256); }

void launch_traverse(const uint8_t *Xt, int64_t n, int64_t ld, int D, int half, int m, const uint16_t *axis,
                     const uint8_t *cut, uint8_t *L, cudaStream_t s) {
  (void)D;
  if (m <= 0) return;
  const dim3 grid(grid_for(ld, kTravWords), (unsigned)((m + kTravTrees - 1) / kTravTrees));
  traverse_kernel<<<grid, 256, 0, s>>>(Xt, n, ld, half, m, axis, cut, L);
}

// trees [j0, j0 + nt) of the leaf table -> shared memory as f64 (whole block)
__device__ __forceinline__ int stage_leaves(double *s_leaf, const float *__restrict__ leaf, int j0, int m, int size,
                                            int cap = kLeafStage) {
  const int per = kLeafStage / size < cap ? kLeafStage / size : cap, nt = m - j0 < per ? m - j0 : per;
  __syncthreads();  // the previous chunk is consumed
  for (int i = threadIdx.x; i < nt * size; i += blockDim.x) s_leaf[i] = (double)__ldg(leaf + (size_t)j0 * size + i);
  __syncthreads();
  return nt;
}

template <int K>
__device__ __forceinline__ void add_leaves_s(double (&acc)[4 * K], const uint32_t (&l)[K], const double *row) {
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[4 * k + b] = __dadd_rn(acc[4 * k + b], row[(l[k] >> (8 * b)) & 0xffu]);
}

template <int K>
__device__ __forceinline__ void store_pts(double *__restrict__ out, int64_t i0, int64_t n, const double (&acc)[4 * K]) {
#pragma unroll
  for (int b = 0; b < 4 * K; ++b)
    if (i0 + b < n) out[i0 + b] = acc[b];
}

// the same sum for rows wider than 64 slots (D = 7, 8): leaf values gathered
// through L1, kSumUnroll trees' cache words in flight per thread
__device__ __forceinline__ void sum_trees_gather(double (&acc)[4], const uint8_t *__restrict__ L, int64_t ld, int64_t w,
                                                 int m, int size, const float *__restrict__ leaf) {
  int j = 0;
  for (; j + 8 <= m; j += 8) {
    uint32_t l[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) l[u] = __ldg(reinterpret_cast<const uint32_t *>(L + (size_t)(j + u) * ld) + w);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float *row = leaf + (size_t)(j + u) * size;
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[b] = __dadd_rn(acc[b], (double)__ldg(row + ((l[u] >> (8 * b)) & 0xffu)));
    }
  }
  for (; j < m; ++j) {
    const uint32_t l = __ldg(reinterpret_cast<const uint32_t *>(L + (size_t)j * ld) + w);
    const float *row = leaf + (size_t)j * size;
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[b] = __dadd_rn(acc[b], (double)__ldg(row + ((l >> (8 * b)) & 0xffu)));
  }
}

// yhat[i] = sum_j leaf[j, L[j, i]] accumulated in f64, j ascending.  Four
// points per thread, leaf values gathered through L1: at n = 1e6 this beat
// 16 points per thread (206 us vs 136 us) and shared-memory f64 leaf tables
// (233 us, the staging is amortised over too few points per block).
__global__ void __launch_bounds__(256) predict_cached_kernel(const uint8_t *__restrict__ L, int64_t n, int64_t ld, int m,
                                                             int size, const float *__restrict__ leaf,
                                                             double *__restrict__ out) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w * 4 >= ld) return;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  sum_trees_gather(acc, L, ld, w, m, size, leaf);
#pragma unroll
  for (int b = 0; b < 4; ++b)
    if (w * 4 + b < n) out[w * 4 + b] = acc[b];
}

// Trees of <= 64 leaf slots (D <= 6): the warp holds the tree's leaf row in
// registers (lane k: slots k and k + 32) and looks values up by shuffle
// instead of gathering them through L1.
// sum over trees (ascending, f64) of the 4 points of cache word w; leaf rows
// of <= 64 slots, looked up by shuffle (the whole warp must call it).
// kSumUnroll trees' cache words and leaf rows are loaded before any of them is
// used, so each warp keeps kSumUnroll independent row loads in flight (the
// loop is bound by memory latency, not by the shuffles: one 128 B load per
// warp and tree would leave HBM mostly idle).  The upper half of a row
// (heap slots 32..63, leaves at depth 5) is shuffled only when a lane of the
// warp indexes it -- rarely, trees are shallow.
#ifndef BART_SUM_UNROLL
#define BART_SUM_UNROLL 8
#endif
constexpr int kSumUnroll = BART_SUM_UNROLL;

template <int U>
__device__ __forceinline__ void sum_trees_block(double (&acc)[4], const uint32_t *__restrict__ Lw, int64_t ldw,
                                                bool live, const float *__restrict__ lrow, int size, int lane) {
  uint32_t l[U];
  float lo[U], hi[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    lo[u] = lane < size ? __ldg(lrow + u * size) : 0.f;
    hi[u] = lane + 32 < size ? __ldg(lrow + u * size + 32) : 0.f;
    l[u] = live ? __ldg(Lw) : 0u;
    Lw += ldw;
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    // each lane widens its own leaf slot(s) once per tree, and the points
    // fetch f64 values by shuffle: the f32->f64 conversion runs on the XU
    // pipe, which a conversion per point and tree saturates (ncu)
    const double dlo = (double)lo[u];
    if (!__any_sync(0xffffffffu, (l[u] & 0xe0e0e0e0u) != 0u)) {  // no index >= 32 in the warp (shallow tree)
#pragma unroll
      for (int b = 0; b < 4; ++b)
        acc[b] = __dadd_rn(acc[b], __shfl_sync(0xffffffffu, dlo, (l[u] >> (8 * b)) & 31u));
    } else {
      const double dhi = (double)hi[u];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t h = (l[u] >> (8 * b)) & 0xffu;
        const double a = __shfl_sync(0xffffffffu, dlo, h & 31u), c = __shfl_sync(0xffffffffu, dhi, h & 31u);
        acc[b] = __dadd_rn(acc[b], h < 32u ? a : c);
      }
    }
  }
}

__device__ __forceinline__ void sum_trees_shfl(double (&acc)[4], const uint8_t *__restrict__ L, int64_t ld, int64_t w,
                                               bool live, int m, int size, const float *__restrict__ leaf, int lane) {
#pragma unroll
  for (int b = 0; b < 4; ++b) acc[b] = 0.0;
  const int64_t ldw = ld / 4;  // cache row stride in words
  const uint32_t *Lw = reinterpret_cast<const uint32_t *>(L) + w;
  const float *lrow = leaf + lane;
  int j = 0;
  for (; j + kSumUnroll <= m; j += kSumUnroll) {
    sum_trees_block<kSumUnroll>(acc, Lw, ldw, live, lrow, size, lane);
    Lw += kSumUnroll * ldw;
    lrow += kSumUnroll * size;
  }
  for (; j < m; ++j) {
    sum_trees_block<1>(acc, Lw, ldw, live, lrow, size, lane);
    Lw += ldw;
    lrow += size;
  }
}

// f64 leaf table in shared memory: every kSTrees trees the block widens the
// trees' leaf rows to f64 once (one conversion per leaf value and block,
// instead of one per point and tree on the slow XU conversion pipe), then each
// point's lookup is one shared-memory gather of the f64 value.  Cache words
// are loaded kSumUnroll trees ahead (memory-level parallelism).
constexpr int kSTrees = 32;
#ifndef BART_SMEM64_UNROLL
#define BART_SMEM64_UNROLL 8
#endif
constexpr int kS64Unroll = BART_SMEM64_UNROLL;
template <int SIZE, int P>
__device__ __forceinline__ void sum_trees_smem64(double (&acc)[4 * P], const uint8_t *__restrict__ L, int64_t ld,
                                                 int64_t w, bool live, int m, const float *__restrict__ leaf,
                                                 double *s_tab) {
  // P cache words (4P points) per thread: word w*P+p
  typedef typename Vec<P>::T VT;
#pragma unroll
  for (int b = 0; b < 4 * P; ++b) acc[b] = 0.0;
  const int64_t ldv = ld / (4 * P);
  const VT *Lv = reinterpret_cast<const VT *>(L) + w;
  for (int j0 = 0; j0 < m; j0 += kSTrees) {
    const int nt = m - j0 < kSTrees ? m - j0 : kSTrees;
    __syncthreads();  // the previous chunk's table is consumed
    for (int i = threadIdx.x; i < nt * SIZE; i += blockDim.x) s_tab[i] = (double)__ldg(leaf + (size_t)j0 * SIZE + i);
    __syncthreads();
    if (!live) continue;
    int jj = 0;
    for (; jj + kS64Unroll <= nt; jj += kS64Unroll) {
      uint32_t l[kS64Unroll][P];
#pragma unroll
      for (int u = 0; u < kS64Unroll; ++u) {
        const VT v = __ldg(Lv + (size_t)(j0 + jj + u) * ldv);
        memcpy(l[u], &v, sizeof(VT));
      }
#pragma unroll
      for (int u = 0; u < kS64Unroll; ++u) {
        const double *row = s_tab + (jj + u) * SIZE;
#pragma unroll
        for (int p = 0; p < P; ++p)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[4 * p + b] = __dadd_rn(acc[4 * p + b], row[(l[u][p] >> (8 * b)) & 0xffu]);
      }
    }
    for (; jj < nt; ++jj) {
      uint32_t l[P];
      const VT v = __ldg(Lv + (size_t)(j0 + jj) * ldv);
      memcpy(l, &v, sizeof(VT));
      const double *row = s_tab + jj * SIZE;
#pragma unroll
      for (int p = 0; p < P; ++p)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[4 * p + b] = __dadd_rn(acc[4 * p + b], row[(l[p] >> (8 * b)) & 0xffu]);
    }
  }
}

#ifndef BART_SMEM64_WORDS
#define BART_SMEM64_WORDS 1
#endif
constexpr int kS64Words = BART_SMEM64_WORDS;

__global__ void __launch_bounds__(256) predict_smem64_kernel(const uint8_t *__restrict__ L, int64_t n, int64_t ld, int m,
                                                             const float *__restrict__ leaf, double *__restrict__ out) {
  constexpr int P = kS64Words;
  __shared__ double s_tab[kSTrees * 64];
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = w * 4 * P < ld;
  double acc[4 * P];
  sum_trees_smem64<64, P>(acc, L, ld, w, live, m, leaf, s_tab);
  if (live)
#pragma unroll
    for (int b = 0; b < 4 * P; ++b)
      if (w * 4 * P + b < n) out[w * 4 * P + b] = acc[b];
}

__global__ void __launch_bounds__(256) predict_shfl_kernel(const uint8_t *__restrict__ L, int64_t n, int64_t ld, int m,
                                                           int size, const float *__restrict__ leaf,
                                                           double *__restrict__ out) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = w * 4 < ld;
  double acc[4];
  sum_trees_shfl(acc, L, ld, w, live, m, size, leaf, threadIdx.x & 31);
  if (live)
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (w * 4 + b < n) out[w * 4 + b] = acc[b];
}

void launch_predict_cached(const uint8_t *L, int64_t n, int64_t ld, int m, int size, const float *leaf,
                           double *out, cudaStream_t s) {
#ifndef BART_PREDICT_SHFL
#define BART_PREDICT_SHFL 1
#endif
#ifndef BART_PREDICT_SMEM64
#define BART_PREDICT_SMEM64 1
#endif
  if (BART_PREDICT_SMEM64 && size == 64) {
    predict_smem64_kernel<<<grid_for(ld, kS64Words), 256, 0, s>>>(L, n, ld, m, leaf, out);
    return;
  }
  if (BART_PREDICT_SHFL && size <= 64) {
    predict_shfl_kernel<<<grid_for(ld, 1), 256, 0, s>>>(L, n, ld, m, size, leaf, out);
    return;
  }
  predict_cached_kernel<<<grid_for(ld, 1), 256, 0, s>>>(L, n, ld, m, size, leaf, out);
}

// Fused traverse + sum over all trees, without materialising the (m, n)
// cache.  A column's address depends only on the tree (axis of the node), never
// on the data, so each chunk of trees is flattened into a shared-memory list of
// internal nodes in (tree, heap) order -- one 32-bit entry: axis | last-of-tree
// | cut | node -- and every thread keeps the loads of the next P entries in
// flight while it applies the current one (no per-tree ballot / shuffle on the
// path).  A tree with no internal node gets a no-op entry (node 0 matches no
// point).  Leaf values are added per tree in ascending order (trees.py:206-
// 218), so the result is bit-identical to traverse + sum_leaf_values.
// Measured at n=1e6, m=200 (steady state): 4 words x 1 entry ahead 172 us;
// 8 x 1 171; 4 x 2 185; 4 x 4 191; 2 x 8 213 (more loads in flight lose: the
// kernel is ALU-bound on the SWAR steps, not waiting on L2).
#ifndef BART_EVAL_PIPE
#define BART_EVAL_PIPE 1
#endif
#ifndef BART_EVAL_PIPE_WORDS
#define BART_EVAL_PIPE_WORDS 4
#endif
constexpr int kEvalPipe = BART_EVAL_PIPE;
constexpr int kEvalPipeWords = BART_EVAL_PIPE_WORDS;
constexpr int kNodeStage = 2048;  // >= trees per leaf chunk x entries per tree (64 x 31 at D = 6, 16 x 127 at D = 8)
constexpr int kNodeTrees = 1024;  // trees per chunk (D = 1's 2048-tree leaf chunks are halved: static smem < 48 KB)
constexpr uint32_t kEntryEnd = 1u << 15;

__device__ __forceinline__ uint32_t make_entry(uint32_t node, uint32_t cutv, uint32_t ax, bool end) {
  return (ax << 16) | (end ? kEntryEnd : 0u) | (cutv << 7) | node;
}

// the internal nodes of trees [j0, j0 + nt) -> s_nodes (whole block); returns the entry count
__device__ __forceinline__ int stage_nodes(uint32_t *s_nodes, int *s_off, const uint8_t *__restrict__ cut,
                                           const uint16_t *__restrict__ axis, int j0, int nt, int half) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int jj = warp; jj < nt; jj += nwarps) {  // entries per tree (>= 1)
    const uint8_t *cj = cut + (size_t)(j0 + jj) * half;
    int cnt = 0;
    for (int base = 0; base < half; base += 32) {
      const int t = base + lane;
      cnt += __popc(__ballot_sync(0xffffffffu, t >= 1 && t < half && __ldg(cj + t) != 0));
    }
    if (lane == 0) s_off[jj + 1] = cnt > 0 ? cnt : 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive scan (nt <= 64 at D = 6; a serial scan is noise next to the chunk)
    s_off[0] = 0;
    for (int jj = 0; jj < nt; ++jj) s_off[jj + 1] += s_off[jj];
  }
  __syncthreads();
  for (int jj = warp; jj < nt; jj += nwarps) {
    const uint8_t *cj = cut + (size_t)(j0 + jj) * half;
    const uint16_t *aj = axis + (size_t)(j0 + jj) * half;
    const int o = s_off[jj], last = s_off[jj + 1] - 1;
    int k = o;
    for (int base = 0; base < half; base += 32) {
      const int t = base + lane;
      const uint32_t ct = t < half ? __ldg(cj + t) : 0u;
      const bool in = t >= 1 && ct != 0u;
      const uint32_t msk = __ballot_sync(0xffffffffu, in);
      if (in) {
        const int pos = k + __popc(msk & ((1u << lane) - 1u));
        s_nodes[pos] = make_entry((uint32_t)t, ct, __ldg(aj + t), pos == last);
      }
      k += __popc(msk);
    }
    if (k == o && lane == 0) s_nodes[o] = make_entry(0u, 0u, 0u, true);  // no internal node: a no-op step
  }
  __syncthreads();
  return s_off[nt];
}

template <int K, int P>
__global__ void __launch_bounds__(256) evaluate_kernel(const uint8_t *__restrict__ Xt, int64_t n, int64_t ld,
                                                            int half, int m, const uint16_t *__restrict__ axis,
                                                            const uint8_t *__restrict__ cut,
                                                            const float *__restrict__ leaf, double *__restrict__ out) {
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4 * K;
  const bool live = i0 < ld;
  const int size = 2 * half;
  const size_t f = blockIdx.y;  // one forest of a stacked batch
  axis += f * (size_t)m * half;
  cut += f * (size_t)m * half;
  leaf += f * (size_t)m * size;
  out += f * (size_t)n;
  __shared__ double s_leaf[kLeafStage];
  __shared__ uint32_t s_nodes[kNodeStage];
  __shared__ int s_off[kNodeTrees + 1];
  const uint8_t *xp = Xt + (live ? i0 : 0);
  double acc[4 * K];
#pragma unroll
  for (int b = 0; b < 4 * K; ++b) acc[b] = 0.0;
  for (int j0 = 0; j0 < m;) {
    const int nt = stage_leaves(s_leaf, leaf, j0, m, size, kNodeTrees);
    const int total = stage_nodes(s_nodes, s_off, cut, axis, j0, nt, half);
    uint32_t xq[P][K];
#pragma unroll
    for (int g = 0; g < P; ++g)
      if (g < total && live) vload<K>(xq[g], xp + (size_t)(s_nodes[g] >> 16) * ld);
    uint32_t l[K];
#pragma unroll
    for (int k = 0; k < K; ++k) l[k] = 0x01010101u;
    const double *row = s_leaf;
    for (int e0 = 0; e0 < total; e0 += P) {
#pragma unroll
      for (int g = 0; g < P; ++g) {
        const int e = e0 + g;
        if (e < total) {  // warp-uniform
          const uint32_t ent = s_nodes[e];
          uint32_t x[K];
#pragma unroll
          for (int k = 0; k < K; ++k) x[k] = xq[g][k];
          if (e + P < total && live) vload<K>(xq[g], xp + (size_t)(s_nodes[e + P] >> 16) * ld);
          const uint32_t node = ent & 0x7fu, cv = (ent >> 7) & 0xffu;
          const uint32_t t4 = 0x01010101u * node, c4 = 0x01010101u * cv, b4 = 0x01010101u * (2u * node);
          if (node == 1u) {  // the root (a tree's first entry): every point is there
#pragma unroll
            for (int k = 0; k < K; ++k) l[k] = swar_child(x[k], c4, c4 & 0x7f7f7f7fu, b4);
          } else {
#pragma unroll
            for (int k = 0; k < K; ++k) l[k] = swar_step(l[k], x[k], t4, c4, b4);
          }
          if (ent & kEntryEnd) {
            if (live) add_leaves_s<K>(acc, l, row);
            row += size;
#pragma unroll
            for (int k = 0; k < K; ++k) l[k] = 0x01010101u;
          }
        }
      }
    }
    j0 += nt;
  }
  if (live) store_pts<K>(out, i0, n, acc);
}

void launch_evaluate(const uint8_t *Xt, int64_t n, int64_t ld, int D, int half, int m, const uint16_t *axis,
                     const uint8_t *cut, const float *leaf, double *out, cudaStream_t s) {
  launch_evaluate_batch(Xt, n, ld, D, half, m, 1, axis, cut, leaf, out, s);
}

void launch_evaluate_batch(const uint8_t *Xt, int64_t n, int64_t ld, int D, int half, int m, int n_forests,
                           const uint16_t *axis, const uint8_t *cut, const float *leaf, double *out, cudaStream_t s) {
  (void)D;
  if (n_forests <= 0 || n <= 0) return;
  const dim3 grid(grid_for(ld, kEvalPipeWords), (unsigned)n_forests);
  evaluate_kernel<kEvalPipeWords, kEvalPipe><<<grid, 256, 0, s>>>(Xt, n, ld, half, m, axis, cut, leaf, out);
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
__global__ void __launch_bounds__(256) trace_train_kernel(const uint8_t *__restrict__ L, int64_t n, int64_t ld, int m,
                                                          int size, const float *__restrict__ leaf, double k,
                                                          double *__restrict__ mean, double *__restrict__ m2,
                                                          double *__restrict__ draw, double *__restrict__ pts,
                                                          int npts) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = w * 4 < ld;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  __shared__ double s_tab[kSTrees * 64];
  if (size == 64) {  // block-uniform (D = 6, the default depth)
    sum_trees_smem64<64, 1>(acc, L, ld, w, live, m, leaf, s_tab);
  } else if (size < 64) {
    sum_trees_shfl(acc, L, ld, w, live, m, size, leaf, threadIdx.x & 31);
  } else if (live) {
    sum_trees_gather(acc, L, ld, w, m, size, leaf);
  }
  if (!live) return;
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
  trace_train_kernel<<<grid_for(ld, 1), 256, 0, s>>>(L, n, ld, m, size, leaf, (double)k, mean, m2, draw, pts, npts);
}

void launch_mean_leaves(const uint8_t *cut, int m, int half, double *out, cudaStream_t s) {
  mean_leaves_kernel<<<1, 1024, 0, s>>>(cut, m, half, out);
}

}  // namespace bart
