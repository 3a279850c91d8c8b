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
constexpr int kWorkers = 448;                 // threads that own points (14 warps)
constexpr int kWorkWarps = kWorkers / 32;
constexpr int kSweepThreads = kWorkers + 64;  // + control warp (exchange, decision) + helper warp
constexpr int kSweepWarps = kSweepThreads / 32;
constexpr int kMaxCtas = 256;         // CTAs per shard (one per SM)
constexpr int kProposeWarps = 4;
constexpr int kMaxShards = 8;         // n-shards whose exchange words a sweep adds into
// Exchange accumulators: kXSets sets (exchange X uses set X % kXSets), each
// kSlotsMax+1 slots of 3 tagged fixed-point limbs of the slot's f64 residual
// sum.  Slots sit kXSlotWords (256 B) apart, so the slots of one exchange
// hit different L2 lines and slices: same-line atomics from 148 CTAs
// serialise (tools/xbench2.cu; +2.4% end to end over 32-B slots).  One warp
// instruction adds (and polls) 8 slots: lane 4s+q owns word q of slot s.
constexpr int kXSets = 3;
constexpr int kXSlotWords = 32;
constexpr size_t kXSetWords = (size_t)(kSlotsMax + 1) * kXSlotWords;
constexpr size_t kXPrevWords = (size_t)(kSlotsMax + 1) * 4;  // per set: baselines of the used words (s*4+q)
// Count channel: the per-leaf point counts of tree j (needed one exchange
// before tree j's decision) travel through their own tagged words, set j % 4,
// one u64 per slot, added and polled by the helper warps.
constexpr int kCSets = 4;
constexpr size_t kCSetWords = (size_t)kSlotsMax;

enum : int { KIND_NONE = 0, KIND_GROW = 1, KIND_PRUNE = 2 };

struct HP {
  double leaf_sd, lam, alpha, beta, leaf_mean, nu, p_grow;
  int update_sigma;
  double depth_prob[kMaxDepth];
};

// One tree's proposal (sampler.py:263-306) plus everything the sweep needs
// about the tree, as one contiguous per-tree RECORD the sweep fetches with a
// single TMA bulk copy: this header, then float old_leaf[size] (the tree's
// leaf row before the sweep) and double z[size] (its leaf_z draws).
struct __align__(16) TreeMove {
  int32_t kind, node, axis, cut;
  int32_t depth, n_axes, n_splits, w_small;
  int32_t w_prime_big, growable_big, gl, gr;
  int32_t nslots, pad0, pad1, pad2;
  double struct_log;
  double log_u;  // log(accept_u): lets the sweep decide without exp() off the near-tie band
  double acc_u;  // accept_u (sampler.py:833)
  double pad3;
  uint8_t slot_node[kSlotsMax];  // leaves of the larger tree of the move pair, heap order
};
static_assert(sizeof(TreeMove) == 224, "record header layout");

__host__ __device__ __forceinline__ int rec_stride(int size) { return (224 + 12 * size + 15) & ~15; }
__device__ __forceinline__ const TreeMove &rec_hdr(const uint8_t *rec) { return *reinterpret_cast<const TreeMove *>(rec); }
__device__ __forceinline__ const float *rec_leaf(const uint8_t *rec) { return reinterpret_cast<const float *>(rec + 224); }
__device__ __forceinline__ const double *rec_z(const uint8_t *rec, int size) {
  return reinterpret_cast<const double *>(rec + 224 + 4 * size);
}

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
  uint8_t *rec;   // (m, rec_stride(size)) per-tree records
  int rstride;
  TreeHdr *hdr;
  double *rand_move, *rand_acc, *rand_z, *rand_chi2;
  double *sigma2, *sigma2_draw;
  uint8_t *accepted;
  int64_t *tap_counts;
  double *tap_sums;
  int taps;
  unsigned long long *xacc;     // this shard's exchange sets [kXSets][kXSetWords] (polled)
  unsigned long long *xpeer[kMaxShards];  // every shard's xacc (own included): where partials are added
  int n_shards;                 // copies in xpeer (= shards of the chain)
  int nblk_total;               // CTAs over all shards = arrival tag of a complete word
  int shard_sys;                // 1: peers on other devices (system-scope atomics and polls)
  int copy_base, copy_groups;   // CTA c polls copy copy_base + c % copy_groups (copy_groups > 1 only
                                // when one launch emulates several shards on one device)
  int64_t n_total;              // points of the whole chain (chi-square df, sampler.py:259)
  int *err;                     // device error flags (bit 0: exchange value out of fixed-point range)
  int *err_out;                 // bart_step: the sigma CTA copies *err here at the end (pinned host), or null
  unsigned long long *xsnap;    // [1 + kXSets*kXPrevWords]: exchange count, then every polled
                                // word's last complete value (the next sweep's baseline)
  unsigned long long *cacc;     // this shard's count channel [kCSets][kCSetWords] (polled)
  unsigned long long *cpeer[kMaxShards];  // every shard's cacc
  unsigned long long *csnap;    // [kCSets*kCSetWords] last complete count words
  // Two-level (hierarchical) exchange, n-sharded chains: a CTA adds into its
  // own shard's STAGE words (device scope); one forwarder CTA per shard polls
  // them complete and adds the shard's total, tagged once, into every shard's
  // copy -- n_shards arrivals per word instead of one per CTA of every shard.
  // With copy groups (one-device emulation) every group has its own stage.
  int hier;                      // 1: two-level exchange (bart_set_exchange)
  unsigned long long *xstage;    // [groups][kXSets][kXSetWords] (groups = copy_groups, or 1 per shard)
  unsigned long long *cstage;    // [groups][kCSets][kCSetWords]
  unsigned long long *xssnap;    // [groups][kXSets*kXPrevWords] forwarders' stage baselines
  unsigned long long *cssnap;    // [groups][kCSets*kCSetWords]
  unsigned long long *iter_dev;
  uint64_t seed;
  int nblk, chunk;
  int stream;     // 1: chunk beyond the register budget -- residuals in global (L2) memory
  size_t persist_bytes;  // stream mode: bytes of r in the launch's persisting L2 window (0: none)
  uint8_t *Lref;  // stream mode: (3, n_pad) refreshed larger-tree rows of trees e-1, e, e+1
  long long *timeline;        // optional per-tree phase stamps (clock64), CTA 0 and last CTA
  long long *trace;           // optional (m+1, nblk, 2) globaltimer: publish, gathered
  HP hp;
  int dbg;  // experiment switches (BART_DBG env var at create; 0 in production)
  int propose_in_sweep;  // per launch: 0 proposals already made, 1 propose with device RNG, 2 with injected randoms
  // on-device trace (bart_trace_begin): per-iteration accept flags and sigma2,
  // rows [iter - hist_base] of (hist_cap, m) / (hist_cap)
  uint8_t *acc_hist;
  double *sig_hist;
  int64_t hist_base, hist_cap;
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

// ------------------------------------------------------------ async copies (TMA bulk), mbarriers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *b, uint32_t count = 1) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// phase of tree t on a per-parity mbarrier
__device__ __forceinline__ uint32_t par2(int t) { return (uint32_t)((t >> 1) & 1); }
__device__ __forceinline__ void mbar_expect(unsigned long long *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------ misc
__device__ __forceinline__ int heap_depth(int h) { return 31 - __clz(h); }

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
  return v;  // valid in lane 0
}

// SWAR on 4 point bytes.  A node step: bytes of l equal to t become
// 2t + (x >= cut).  Per word: equality in 4 integer ops (high bit of each
// equal byte), the 0xff byte mask by one sign-replicating byte permute, the
// unsigned x >= cut per byte in 3 (bit 7 of each byte, Hacker's Delight:
// (x7 & ~c7) | (~(x7 ^ c7) & bit 7 of (x | 0x80) - (c & 0x7f))), the child
// byte in 2 and the merge in 1 (forest.cu's traversals; the sweep's B pass,
// sweep.cu grow4s, takes the byte mask but keeps its 9-bit-lane compare, which
// measured 1% faster there).
__device__ __forceinline__ uint32_t swar_eq(uint32_t a, uint32_t b4) {
  const uint32_t x = a ^ b4;
  return ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x) & 0x80808080u;
}
template <int LUT>
__device__ __forceinline__ uint32_t lop3t(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return d;
}
// every byte -> its sign bit replicated (prmt's sign mode: selector nibbles 8 + i)
__device__ __forceinline__ uint32_t sign_bytes(uint32_t a) {
  uint32_t d;
  asm("prmt.b32 %0, %1, 0, 0xba98;" : "=r"(d) : "r"(a));
  return d;
}
// child bytes 2t + (x >= cut): c4 = cut per byte, c7 = c4 & 0x7f7f7f7f, b4 = 2t per byte
__device__ __forceinline__ uint32_t swar_child(uint32_t x, uint32_t c4, uint32_t c7, uint32_t b4) {
  const uint32_t d = (x | 0x80808080u) - c7;
  // (x & ~c) | (~(x ^ c) & d), bit 7 of each byte is x >= cut (LUT of f(a=x, b=c, c=d))
  constexpr int A = 0xf0, B = 0xcc, C = 0xaa;
  const uint32_t ge = lop3t<((A & ~B) | (~(A ^ B) & C)) & 0xff>(x, c4, d);
  return ((ge >> 7) & 0x01010101u) | b4;
}
__device__ __forceinline__ uint32_t swar_step(uint32_t l, uint32_t x, uint32_t t4, uint32_t c4, uint32_t b4) {
  const uint32_t msk = sign_bytes(swar_eq(l, t4));
  const uint32_t nw = swar_child(x, c4, c4 & 0x7f7f7f7fu, b4);
  return (l & ~msk) | (msk & nw);
}

}  // namespace bart
