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
constexpr int kSweepThreads = 512;
constexpr int kSweepWarps = kSweepThreads / 32;
constexpr int kMaxCtas = 256;         // mailbox gather unroll bound
constexpr int kGatherUnroll = kMaxCtas / 32;
constexpr int kProposeWarps = 4;

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
  uint8_t slot_node[kSlotsMax];
};

// Compact per-tree header the sweep keeps in shared memory for all trees.
struct __align__(8) TreeHdr {
  uint8_t kind, node, cut, pad;
  uint16_t axis, nslots;
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
  unsigned long long *mbox;   // [2][kSlotsMax+1][nblk][4] LL mailbox
  uint32_t *tagbase;
  unsigned long long *iter_dev;
  uint64_t seed;
  int nblk, chunk;
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

// ------------------------------------------------------------ LL mailbox
// Low-latency exchange: every 64-bit word carries a 32-bit tag in its high
// half, so a reader validates data and arrival with one load (no fences).
__device__ __forceinline__ void ll_store(unsigned long long *p, uint32_t tag, uint32_t cnt, double s) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(s);
  const unsigned long long t = ((unsigned long long)tag) << 32;
  const unsigned long long w0 = t | cnt, w1 = t | (bits & 0xffffffffull), w2 = t | (bits >> 32);
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p + 2), "l"(w2) : "memory");
}
__device__ __forceinline__ void ll_load(const unsigned long long *p, unsigned long long &w0,
                                        unsigned long long &w1, unsigned long long &w2) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(w2) : "l"(p + 2) : "memory");
}

// ------------------------------------------------------------ misc
__device__ __forceinline__ int heap_depth(int h) { return 31 - __clz(h); }

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
  return v;  // valid in lane 0
}

}  // namespace bart
