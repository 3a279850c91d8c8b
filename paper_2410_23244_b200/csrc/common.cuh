// Shared device definitions for the B200 BART step (sm_100a).
//
// Layout in HBM, per chain handle:
//   Xt   uint8  (p, n_pad)   predictors, transposed from the reference's (n, p)
//                            (grid.py:121-134) so a split column is one row
//   L    uint8  (m, n_pad)   leaf-index cache, transposed from the reference's
//                            (n, m) (sampler.py:137): tree j is one n-byte row
//   r, y float  (n_pad)      residuals / response (sampler.py:134-136)
//   axis uint16 (m, half), cut uint8 (m, half), leaf float (m, size)
//                            heap forest (trees.py:1-17), half = 2^(D-1), size = 2^D
// n_pad is n rounded up to 16 so every CTA chunk starts 16-B aligned for TMA.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bart {

constexpr int kMaxDepth = 8;
constexpr int kSlotsMax = 128;        // leaves of a depth-8 tree
constexpr int kWorkers = 480;                 // threads that own points (15 warps)
constexpr int kWorkWarps = kWorkers / 32;
constexpr int kSweepThreads = kWorkers + 32;  // + one producer warp (TMA / stage loads)
constexpr int kSweepWarps = kSweepThreads / 32;
constexpr int kMaxCtas = 256;         // mailbox gather unroll bound
constexpr int kGatherUnroll = kMaxCtas / 32;
constexpr int kProposeWarps = 4;
constexpr int kAccWords = 8;       // per slot: 4 fixed-point limbs, 1 count, pad (64 B)

enum : int { KIND_NONE = 0, KIND_GROW = 1, KIND_PRUNE = 2 };

struct HP {
  double leaf_sd, lam, alpha, beta, leaf_mean, nu, p_grow;
  int update_sigma;
  double depth_prob[kMaxDepth];
};

// One tree's proposal (sampler.py:263-306) plus the leaf list of the larger
// tree of the move pair, which the sweep histograms over.
struct __align__(16) TreeMove {
  int32_t kind, node, axis, cut;
  int32_t depth, n_axes, n_splits, w_small;
  int32_t w_prime_big, growable_big, gl, gr;
  int32_t nslots, pad0;
  double struct_log;
  double log_u;  // log(accept_u): lets the sweep decide without exp() off the near-tie band
  uint8_t slot_node[kSlotsMax];
};

// Compact per-tree header the sweep keeps in shared memory for all trees.
struct __align__(8) TreeHdr {
  uint8_t kind, node, cut, nslots;  // nslots in [1, 128]
  uint16_t axis;
  uint8_t slot_l, slot_r;  // slot indices of children 2t, 2t+1 in the larger tree (moves only)
};

// Everything a kernel needs about one chain (passed by value).
struct ChainDev {
  int64_t n, n_pad;
  int p, m, D, half, size;
  const uint8_t *Xt;
  uint8_t *L;
  float *r;
  const float *y;
  uint16_t *axis;
  uint8_t *cut;
  float *leaf;
  const int32_t *max_cuts;
  const uint32_t *open_bits;  // bit a set iff max_cuts[a] > 0
  int P_open;                 // popcount of open_bits
  TreeMove *moves;
  TreeHdr *hdr;
  double *rand_move, *rand_acc, *rand_z, *rand_chi2;
  double *sigma2, *sigma2_draw;
  uint8_t *accepted;
  int64_t *tap_counts;
  double *tap_sums;
  int taps;
  unsigned long long *accum;    // [kSlotsMax+1][kAccWords] monotonic fixed-point slot accumulators
  unsigned long long *counter;  // monotonic exchange arrival counter (own 128-B line)
  unsigned long long *accum_base;  // accumulator + counter values at the end of the last sweep
  unsigned long long *iter_dev;
  uint64_t seed;
  int nblk, chunk;
  long long *timeline;        // optional per-tree phase stamps (clock64), CTA 0 and last CTA
  long long *trace;           // optional (m+1, nblk, 2) globaltimer: publish, gathered
  HP hp;
};

// ------------------------------------------------------------ Philox4x32-10
__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t lo0 = c.x * 0xD2511F53u, hi0 = __umulhi(c.x, 0xD2511F53u);
    const uint32_t lo1 = c.z * 0xCD9E8D57u, hi1 = __umulhi(c.z, 0xCD9E8D57u);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}
// 53-bit uniform in [0, 1)
__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
  return (double)((((uint64_t)(a >> 5)) << 26) | (uint64_t)(b >> 6)) * 0x1.0p-53;
}

// ------------------------------------------------------------ misc
__device__ __forceinline__ int heap_depth(int h) { return 31 - __clz(h); }

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
  return v;  // valid in lane 0
}

}  // namespace bart
