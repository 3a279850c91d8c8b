// The sequential tree sweep of one MCMC iteration as ONE persistent kernel.
//
// Reference semantics (bforge, /root/reference/pkg/src/bforge/sampler.py):
//   phase 2  refresh_leaf_indices      :529-547  (grow refresh of the index cache)
//   phase 3  count_points_per_leaf      :550-553
//   phase 4/6 _parallel_accept_terms    :669-703
//   phase 7/8 sum_residuals_per_leaf    :556-576
//   phase 9  _resolve_tree decision     :829-866
//   phase 10 leaf_posterior/draw        :579-595, 868-870
//   phase 11 update_caches              :737-761
//   sigma    sigma2_draw/sum_squares    :790-799, 906-908
//
// Design.  One CTA per SM owns a contiguous chunk of points.
// 14 worker warps hold the chunk's residuals (f32) and the larger-tree leaf
// indices of trees e-1, e, e+1 (4 points per 32-bit word) in REGISTERS for the
// whole sweep.  Per tree e the workers run
//   A_e (critical path): tree e-1's residual update + cache write, then tree
//       e's per-leaf f64 residual sums; publish the warp partials;
//   B_e (hidden behind the exchange): tree e+2's grow refresh and per-leaf
//       point counts, from its leaf-index row and split column that a TMA bulk
//       copy staged in shared memory four trees ahead;
// then wait for the decision of tree e.  The CONTROL warp folds the partials,
// exchanges them across the grid and decides; nothing else sits on the
// per-tree critical path.  The HELPER warp does everything that can lag one
// tree behind: the next tree's count-only terms, one CTA's forest write per
// tree, and the TMA prefetch of the per-tree data (cache row, split column and
// the tree's record: proposal, leaf list, old leaf row, leaf draws).
//
// Cross-CTA exchange without a grid barrier, counter, fence or decider: every
// CTA adds its partials, as exact fixed point (3 x 37-bit limbs of a 111-bit
// number with 64 fraction bits; counts as integers), into 64-bit words whose
// top 16 bits count arrivals: each add is (1 << 48) | limb.  A reader knows
// each word's last complete value, so a word is complete when (now - last)
// carries exactly one arrival per CTA: the readers poll the data words
// themselves, one L2 round trip after the last add lands.  Integer addition
// is associative, so every CTA reads bit-identical totals and takes the same
// decision redundantly.  Exchange X uses set X % 3; a CTA adds to X+3 only
// after X+2 completed, which needs every CTA to have read X, so words never
// need resetting.  The same words extend to n-sharding across GPUs
// (DESIGN.md §6): a shard adds into every shard's copy (c.xpeer) and polls
// its own.
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"
#include "propose.cuh"

namespace bart {

constexpr int kRing = 4;  // trees e+1 .. e+4 staged
constexpr int kTagShift = 48;
constexpr unsigned long long kTagOne = 1ull << kTagShift;
constexpr unsigned long long kDataMask = kTagOne - 1ull;
constexpr int kLimbBits = 37;
constexpr unsigned long long kLimbMask = (1ull << kLimbBits) - 1ull;
constexpr int kFastRounds = 4;  // exchange rounds (8 slots each) kept in registers: trees with <= 32 slots
constexpr int kCtrlWarp = kWorkWarps;  // then the helper warp

// Named barriers (0 is __syncthreads) only where the two sides strictly
// alternate: workers publish A_e (PARTIALS) and then wait for decision e
// (DECISION).  Signals whose producer may run a tree ahead of its consumer
// (counts -> helper, prep -> control, decision -> helper) are mbarriers with
// one phase per tree and a buffer per tree parity.
enum : int { BAR_PARTIALS = 1, BAR_DECISION = 2, BAR_ROLES = 3 };
constexpr int kBarWC = kWorkers + 32;  // workers + control

// count-only precomputation for one tree (see prepare())
struct Prep {
  uint32_t cnt[kSlotsMax];
  double prec[kSlotsMax];  // tau_mu + n * tau
  double zs[kSlotsMax];    // z / sqrt(prec)
  double cadj[kSlotsMax];  // n * adj, the tree's own contribution to the sums
  double rcp[kSlotsMax];   // 1 / prec, correctly rounded (division by Markstein's correction)
  double prec_l, prec_r, prec_p, zs_p, partial, rcp_p;
};

// decision outputs of one tree, read by the helper's bookkeeping
struct Dec {
  double v_s[kSlotsMax + 1];  // leaf draws (leaves of the larger tree, then the collapsed parent)
  double sums_s[kSlotsMax];   // tree-excluded sums (taps)
  int acc;
};

struct __align__(16) SweepSmem {
  Prep prep[2];
  Dec dec[2];
  double wsum[kWorkWarps][kSlotsMax];       // A pass: per-warp f64 sums of tree e
  uint32_t wcnt[2][kWorkWarps][kSlotsMax];  // B pass: per-warp counts of tree e+2 (by parity)
  double tot_sum[kSlotsMax + 1];            // exchange totals (control; slot 0 = sum r^2 at e = m)
  uint32_t hcnt[kSlotsMax];                 // count-channel totals of the tree being prepared (helper)
  double q_s[kSlotsMax + 1];                // posterior means (control scratch, wide trees)
  float row[256];                           // new leaf row (helper scratch)
  float dlt[256];                           // residual delta by larger-tree heap index
  unsigned long long xprev[kXSets][kXPrevWords];      // last complete value of every exchange word (s*4+q)
  unsigned long long cprev[kCSets][kCSetWords];       // last complete value of every count word
  unsigned long long mbar[kRing];      // TMA ring slot filled (per tree j % kRing)
  unsigned long long cnt_mbar[2];     // workers -> helper: B pass counts of tree t in wcnt[t & 1]
  unsigned long long prep_mbar[2];    // helper -> control: prep[t & 1] ready
  unsigned long long dec_mbar[2];     // control -> helper: decision t in dec[t & 1] (t = m: sum r^2)
  int flag_wr, flag_prune, flag_t;
};

// two-level exchange only (the HIER kernel; after the ring): a forwarder's
// baselines of its shard's stage words
struct __align__(16) HierSmem {
  unsigned long long xsprev[kXSets][kXPrevWords];
  unsigned long long csprev[kCSets][kCSetWords];
};

// ring slot: cache row | split column | record (register mode); record only (stream mode)
__host__ __device__ __forceinline__ size_t ring_row_bytes(int chunk, bool stream) { return stream ? 0 : (size_t)2 * chunk; }
__host__ __device__ __forceinline__ size_t ring_slot_bytes(int chunk, int rstride, bool stream) {
  return ring_row_bytes(chunk, stream) + (size_t)rstride;
}

// Words (4 points) per worker thread held in registers, or 0: the chunk is
// too big and the sweep streams residuals through global memory (L2).
int sweep_words_per_thread(int chunk) {
  const int words = (chunk + 3) / 4;
  for (int w : {1, 2, 4, 8})
    if (w * kWorkers >= words) return w;
  return 0;
}

size_t sweep_smem_bytes(int m, int chunk, int size, bool stream, bool hier) {
  size_t b = sizeof(SweepSmem);
  b += ((size_t)m * sizeof(TreeHdr) + 15) & ~(size_t)15;
  b += ((size_t)kRing * ring_slot_bytes(chunk, rec_stride(size), stream) + 15) & ~(size_t)15;
  if (hier) b += sizeof(HierSmem);
  return b;
}

// ------------------------------------------------------------ barriers (async-copy helpers: common.cuh)
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// Timeline stamps (tools/timeline.py builds a BART_TIMELINE=1 variant of the
// library; production builds carry no instrumentation): SM clock cycles, all
// stamps of one CTA on one clock.
#ifndef BART_TIMELINE
#define BART_TIMELINE 0
#endif
#define TL_STAMP(cond) if (BART_TIMELINE && (cond))
__device__ __forceinline__ long long gtimer() { return clock64(); }
// a stamp that cannot be taken before `dep` is computed
// (a predicated trap on the value holds issue until the value is ready)
__device__ __forceinline__ long long gtimer_after(double dep) {
  long long t;
  asm volatile("{\n .reg .pred p;\n setp.eq.f64 p, %1, 0d7E4D3C2B1A098765;\n @p trap;\n mov.u64 %0, %%clock64;\n}"
               : "=l"(t) : "d"(dep) : "memory");
  return t;
}
// cross-CTA trace stamps: the global nanosecond timer
__device__ __forceinline__ long long nstimer() {
  unsigned long long g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  return (long long)g;
}

// ------------------------------------------------------------ byte-lane ops
// collapse of a pruned pair back into its parent (sampler.py:755)
__device__ __forceinline__ uint32_t collapse4(uint32_t l, uint32_t t) {
  uint32_t out = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint32_t lb = (l >> (8 * b)) & 0xffu;
    out |= ((lb >> 1) == t ? t : lb) << (8 * b);
  }
  return out;
}
// 0x80 in every byte of a that equals the byte in b4 (SWAR zero-byte test)
__device__ __forceinline__ uint32_t bytes_eq(uint32_t a, uint32_t b4) {
  const uint32_t x = a ^ b4;
  const uint32_t t = ((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x;
  return ~t & 0x80808080u;
}

__device__ __forceinline__ float4 update4(float4 r, uint32_t l, const float *dlt) {
  r.x = __fadd_rn(r.x, dlt[l & 0xffu]);
  r.y = __fadd_rn(r.y, dlt[(l >> 8) & 0xffu]);
  r.z = __fadd_rn(r.z, dlt[(l >> 16) & 0xffu]);
  r.w = __fadd_rn(r.w, dlt[l >> 24]);
  return r;
}

// acc += v iff h == slot, exactly: fma(v, 1, acc) = RN(acc + v) and
// fma(v, 0, acc) = acc.  Compare + select of the multiplier's high word +
// DFMA: three instructions (a predicated DADD gets if-converted by ptxas
// into DADD + two FSELs).
#ifndef BART_SUMS_SEL
#define BART_SUMS_SEL 1
#endif
__device__ __forceinline__ void add_if_eq(double &acc, uint32_t h, uint32_t slot, double v) {
#if BART_SUMS_SEL
  acc = __fma_rn(v, h == slot ? 1.0 : 0.0, acc);
#else
  if (h == slot) acc = __dadd_rn(acc, v);
#endif
}

struct Geom {
  int m, chunk, nwords, cta, nblk, size;
  int64_t start;
  uint32_t lenp;
  uint32_t slot_bytes;  // ring slot: cache row | split column | record
  uint32_t row_bytes;   // 2 * chunk (register mode) or 0 (stream mode)
  uint8_t *ring;
  TreeHdr *hdr;
  HierSmem *hs;  // two-level exchange kernel only
  __device__ __forceinline__ uint8_t *slot(int j) const { return ring + (size_t)(j % kRing) * slot_bytes; }
  __device__ __forceinline__ const uint8_t *rec(int j) const { return slot(j) + row_bytes; }
};

// ------------------------------------------------------------ worker passes
struct APass {
  bool do_update, wr, prune;
  uint32_t t;
  uint32_t *gL;  // this chunk of tree e-1's global cache row
  const uint8_t *slots;
  int ns;
};

// Warp sums of V per-thread values at once, by transpose reduction: at each
// butterfly level a lane keeps half of its values and trades the other half
// with its partner (lanes L, L^bit), so V values cost ~V + log2(32) shuffle
// rounds instead of 5V.  Every addition pairs the same lane groups as a
// shfl_down tree (only the operand order differs, and IEEE addition is
// commutative), so each total is bit-identical to warp_sum_f64's.  On return
// the lane holds the total of value `idx`; lanes equal outside
// xreduce_group_mask(V) hold the same total.
template <int N, int BIT>
__device__ __forceinline__ double warp_xreduce(const double (&a)[N], int lane, int &idx) {
  if constexpr (N == 1) {
    double x = a[0];
#pragma unroll
    for (int b = BIT; b >= 0; --b) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, 1 << b));
    return x;
  } else {
    constexpr int H = (N + 1) / 2, R = N - H;
    const bool up = (lane >> BIT) & 1;
    double keep[H];
#pragma unroll
    for (int k = 0; k < H; ++k) {
      const double lo = a[k], hi = k < R ? a[H + k] : 0.0;
      const double mine = up ? hi : lo, other = up ? lo : hi;
      keep[k] = __dadd_rn(mine, __shfl_xor_sync(0xffffffffu, other, 1 << BIT));
    }
    if (up) idx += H;
    return warp_xreduce<H, BIT - 1>(keep, lane, idx);
  }
}
// lanes sharing one total: the bits below the last halving level
__host__ __device__ constexpr int xreduce_levels(int n) { return n <= 1 ? 0 : 1 + xreduce_levels((n + 1) / 2); }
__host__ __device__ constexpr int xreduce_group_mask(int n) { return (1 << (5 - xreduce_levels(n))) - 1; }

// Per-warp slot sums -> S.wsum[warp]: the C compared slots [base, base+C)
// and (TOTAL) slot ns-1 = per-thread total minus the others, reduced together.
template <int C, bool TOTAL>
__device__ __forceinline__ void store_warp_sums(const double (&acc)[C > 0 ? C : 1], double tot, const APass &A,
                                                SweepSmem &S, int warp, int lane, int base, long long *ts = nullptr) {
  constexpr int V = C + (TOTAL ? 1 : 0);
  double vals[V > 0 ? V : 1];
  double rest = tot;
#pragma unroll
  for (int s = 0; s < C; ++s) {
    vals[s] = acc[s];
    if (TOTAL) rest = __dsub_rn(rest, acc[s]);
  }
  if (TOTAL) vals[C] = rest;
  if constexpr (V > 0) {
    int idx = 0;
    const double v = warp_xreduce<V, 4>(vals, lane, idx);
    if ((lane & xreduce_group_mask(V)) == 0) {
      const int slot = idx < C ? base + idx : A.ns - 1;
      // compared slots beyond the tree's (padded variants) are not stored: with
      // TOTAL, slot ns-1 is the running total's, and only it may write there
      if (idx < V && (idx >= C || base + idx < (TOTAL ? A.ns - 1 : A.ns))) S.wsum[warp][slot] = v;
    }
    TL_STAMP(ts && TOTAL) ts[25] = gtimer_after(v);
  }
}

// A pass over the register-resident chunk.  FIRST: tree e-1's update
// (residuals f32 with the reference's two roundings, sampler.py:755-760;
// cache write of the final tree).  Then the f64 residual sums of tree e over
// its larger-tree leaves (sampler.py:556-576): with TOTAL, slots
// [base, base+C) are accumulated by compare-and-add and the last slot ns-1
// is the running total minus the others (one DADD per point instead of a
// compare-and-add); without TOTAL, slots [base, base+C) only.
template <int W, int C, bool FIRST, bool TOTAL>
__device__ __forceinline__ void sums_pass(float4 (&r)[W], const uint32_t (&lp)[W], const uint32_t (&lc)[W],
                                          const APass &A, const Geom &G, const float *dlt, SweepSmem &S, int tid,
                                          int warp, int lane, int base, long long *ts = nullptr) {
  uint32_t sn[C > 0 ? C : 1];
  double acc[C > 0 ? C : 1];
  double tot = 0.0;
#pragma unroll
  for (int s = 0; s < C; ++s) {
    sn[s] = base + s < (TOTAL ? A.ns - 1 : A.ns) ? A.slots[base + s] : 0xffffu;
    acc[s] = 0.0;
  }
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const int w = tid + k * kWorkers;
    if (w < G.nwords) {
      if (FIRST && A.do_update) {
        r[k] = update4(r[k], lp[k], dlt);
        if (A.wr) A.gL[w] = A.prune ? collapse4(lp[k], A.t) : lp[k];
      }
      const float rv[4] = {r[k].x, r[k].y, r[k].z, r[k].w};
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t h = (lc[k] >> (8 * b)) & 0xffu;
        const double v = (double)rv[b];
        if (TOTAL) tot = __dadd_rn(tot, v);  // padding points (index 0) carry r = 0
#pragma unroll
        for (int s = 0; s < C; ++s) add_if_eq(acc[s], h, sn[s], v);
      }
    }
  }
  TL_STAMP(ts && base == 0) ts[24] = gtimer_after(tot + (C > 0 ? acc[0] : 0.0));
  store_warp_sums<C, TOTAL>(acc, tot, A, S, warp, lane, base, ts);
}

template <int W>
__device__ __forceinline__ void sums_passes(float4 (&r)[W], const uint32_t (&lp)[W], const uint32_t (&lc)[W],
                                            const APass &A, const Geom &G, const float *dlt, SweepSmem &S, int tid,
                                            int warp, int lane, long long *ts = nullptr) {
  // compared-slot variants {0, 1, 2, 3} + the total for trees of <= 4 leaves;
  // wider trees take 8-slot passes.  Few variants: the control warp's code
  // must stay in the instruction cache next to the workers'.
#ifndef BART_SUMS_TOTAL
#define BART_SUMS_TOTAL 1
#endif
  if (!BART_SUMS_TOTAL) {
    if (A.ns <= 2)
      sums_pass<W, 2, true, false>(r, lp, lc, A, G, dlt, S, tid, warp, lane, 0);
    else if (A.ns <= 4)
      sums_pass<W, 4, true, false>(r, lp, lc, A, G, dlt, S, tid, warp, lane, 0);
    else
      sums_pass<W, 8, true, false>(r, lp, lc, A, G, dlt, S, tid, warp, lane, 0);
    for (int base = 8; base < A.ns; base += 8) sums_pass<W, 8, false, false>(r, lp, lc, A, G, dlt, S, tid, warp, lane, base);
    return;
  }
  // compared-slot variants: each is a fully unrolled pass over the W words,
  // so every variant is instruction-cache footprint the next tree may miss
  // (ncu: no_instruction stalls ~16% of samples); BART_SUMS_SET trades
  // compared slots (~300 cycles each, tools/apass_bench.cu) against variants:
  //   3: one variant per width 1..8   2: {1,2,3,4,6,8}   1: {1,2,3,4,8}   0: {1,2,4,8}
#ifndef BART_SUMS_SET
#define BART_SUMS_SET 3
#endif
  switch (A.ns) {
    case 1: sums_pass<W, 0, true, true>(r, lp, lc, A, G, dlt, S, tid, warp, lane, 0, ts); break;
    case 2: sums_pass<W, 1, true, true>(r, lp, lc, A, G, dlt, S, tid, warp, lane, 0, ts); break;
#if BART_SUMS_SET >= 1
    case 3: sums_pass<W, 2, true, true>(r, lp, lc, A, G, dlt, S, tid, warp, lane, 0, ts); break;
#else
    case 3:
#endif
    case 4: sums_pass<W, 3, true, true>(r, lp, lc, A, G, dlt, S, tid, warp, lane, 0, ts); break;
#if BART_SUMS_SET >= 3
    case 5: sums_pass<W, 4, true, true>(r, lp, lc, A, G, dlt, S, tid, warp, lane, 0, ts); break;
    case 6: sums_pass<W, 5, true, true>(r, lp, lc, A, G, dlt, S, tid, warp, lane, 0, ts); break;
    case 7: sums_pass<W, 6, true, true>(r, lp, lc, A, G, dlt, S, tid, warp, lane, 0, ts); break;
#elif BART_SUMS_SET == 2
    case 5: case 6: sums_pass<W, 5, true, true>(r, lp, lc, A, G, dlt, S, tid, warp, lane, 0, ts); break;
    case 7:
#else
    case 5: case 6: case 7:
#endif
    case 8: sums_pass<W, 7, true, true>(r, lp, lc, A, G, dlt, S, tid, warp, lane, 0, ts); break;
    default:
      sums_pass<W, 8, true, false>(r, lp, lc, A, G, dlt, S, tid, warp, lane, 0);
#ifndef BART_SUMS_TAIL4
#define BART_SUMS_TAIL4 1
#endif
#ifndef BART_COUNT_TAIL4
#define BART_COUNT_TAIL4 1
#endif
      for (int base = 8; base < A.ns; base += 8) {
        if (BART_SUMS_TAIL4 && A.ns - base <= 4)  // a 4-slot tail (9-12 leaves: the common wide trees)
          sums_pass<W, 4, false, false>(r, lp, lc, A, G, dlt, S, tid, warp, lane, base);
        else
          sums_pass<W, 8, false, false>(r, lp, lc, A, G, dlt, S, tid, warp, lane, base);
      }
  }
}

// x >= cut per byte (unsigned), 0x01 in every byte where it holds: 9-bit
// lanes so the subtraction's borrow lands in bit 8 of each lane
__device__ __forceinline__ uint32_t bytes_geu(uint32_t x, uint32_t c4) {
  const uint32_t de = ((x & 0x00ff00ffu) | 0x01000100u) - (c4 & 0x00ff00ffu);
  const uint32_t dodd = (((x >> 8) & 0x00ff00ffu) | 0x01000100u) - ((c4 >> 8) & 0x00ff00ffu);
  return ((de >> 8) & 0x00010001u) | (dodd & 0x01000100u);
}
// refresh_leaf_indices on 4 points (sampler.py:541-545), SWAR: bytes equal to
// t become 2t + (x >= cut)
__device__ __forceinline__ uint32_t grow4s(uint32_t l, uint32_t x, uint32_t t4, uint32_t c4, uint32_t b4) {
  // 0xff byte mask by prmt's sign replication (common.cuh sign_bytes): +0.1% on
  // the step; the forest kernels' borrow-free compare measured -1% here
  const uint32_t msk = sign_bytes(bytes_eq(l, t4));
  return (l & ~msk) | (msk & (b4 | bytes_geu(x, c4)));
}

// Per-slot counts over the chunk: POPC of the SWAR byte-equality mask (or,
// with BART_COUNT_POPC=0, byte-lane counters folded once per slot; measured
// ~1% slower end to end).
template <int W, int NS>
__device__ __forceinline__ void count_pass(const uint32_t (&v)[W], const Geom &G, const uint8_t *slots, int ns,
                                           int base, uint32_t *wrow, int tid, int lane) {
  uint32_t cnt[NS], s4[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    s4[s] = base + s < ns ? 0x01010101u * (uint32_t)slots[base + s] : 0xffffffffu;
    cnt[s] = 0u;
  }
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const int w = tid + k * kWorkers;
    if (w < G.nwords) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
#ifndef BART_COUNT_POPC
#define BART_COUNT_POPC 1
#endif
#if BART_COUNT_POPC
        cnt[s] += __popc(bytes_eq(v[k], s4[s]));
#else
        cnt[s] += bytes_eq(v[k], s4[s]) >> 7;
#endif
      }
    }
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) {
#if BART_COUNT_POPC
    const uint32_t mine = cnt[s];
#else
    const uint32_t mine = (cnt[s] * 0x01010101u) >> 24;
#endif
    const uint32_t cc = __reduce_add_sync(0xffffffffu, mine);
    if (lane == 0 && base + s < ns) wrow[base + s] = cc;
  }
}

// B pass: grow refresh of tree j's cache row (staged in its ring slot) into
// registers and the per-leaf point counts of its larger tree (sampler.py:
// 541-553), reduced per warp into wrow.  Padding bytes are 0 and never match
// a slot (heap indices >= 1); unused slot lanes compare against 0xff..ff,
// which only a depth-8 index 255 could equal, and those lanes are not stored.
template <int W>
__device__ __forceinline__ void refresh_count(uint32_t (&out)[W], const uint8_t *slot, const Geom &G,
                                              const TreeHdr hd, const uint8_t *slots, uint32_t *wrow, int tid,
                                              int lane) {
  const uint32_t *Lr = reinterpret_cast<const uint32_t *>(slot);
  const uint32_t *Xr = reinterpret_cast<const uint32_t *>(slot + G.chunk);
  const bool g = hd.kind == KIND_GROW;
  const uint32_t t4 = 0x01010101u * hd.node, c4 = 0x01010101u * hd.cut, b4 = 0x01010101u * (2u * hd.node);
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const int w = tid + k * kWorkers;
    uint32_t l = 0u;
    if (w < G.nwords) {
      l = Lr[w];
      if (g) l = grow4s(l, Xr[w], t4, c4, b4);
    }
    out[k] = l;
  }
  const int ns = hd.nslots;
  if (ns <= 2)
    count_pass<W, 2>(out, G, slots, ns, 0, wrow, tid, lane);
  else if (ns <= 4)
    count_pass<W, 4>(out, G, slots, ns, 0, wrow, tid, lane);
  else
    for (int base = 0; base < ns; base += 8) {
      if (BART_COUNT_TAIL4 && ns - base <= 4)
        count_pass<W, 4>(out, G, slots, ns, base, wrow, tid, lane);
      else
        count_pass<W, 8>(out, G, slots, ns, base, wrow, tid, lane);
    }
}

// ------------------------------------------------------------ exchange
// f64 -> 111-bit two's-complement fixed point with 64 fraction bits, as three
// 37-bit limbs.  Exact for 2^-12 <= |x| < lim; tinier values round at 2^-64.
// lim = 2^46 / (CTAs over all shards, rounded up to a power of two), so the
// sum of every CTA's partial stays below 2^46 and never wraps the 111-bit
// total.  A partial outside it (or NaN) sets the chain's sticky error flag,
// which the host turns into BART_ERANGE at the next sync (capi.cu).
__device__ __forceinline__ void to_limbs(double x, unsigned long long (&l)[3], int *err, double lim) {
  if (!(fabs(x) < lim)) {  // also catches NaN
    if (err) atomicOr(err, 1);
    x = 0.0;
  }
  const long long hi = __double2ll_rd(x);
  const double rem = __dsub_rn(x, (double)hi);  // exact, in [0, 1]
  const unsigned long long lo = __double2ull_rn(__dmul_rn(rem, 0x1.0p64));
  l[0] = lo & kLimbMask;
  l[1] = ((lo >> kLimbBits) | ((unsigned long long)hi << (64 - kLimbBits))) & kLimbMask;
  l[2] = ((unsigned long long)(hi >> (2 * kLimbBits - 64))) & kLimbMask;
}

// limb sums (each < 2^48) -> f64 of the 111-bit total
__device__ __forceinline__ double from_limbs(unsigned long long t0, unsigned long long t1, unsigned long long t2) {
  unsigned long long lo = t0, hi = 0;
  const unsigned long long a = t1 << kLimbBits;
  lo += a;
  hi += (lo < a ? 1ull : 0ull) + (t1 >> (64 - kLimbBits));
  hi += t2 << (2 * kLimbBits - 64);
  hi &= (1ull << 47) - 1ull;  // mod 2^111
  const bool neg = (hi >> 46) & 1ull;
  if (neg) {  // magnitude = 2^111 - V
    lo = ~lo + 1ull;
    hi = (~hi + (lo == 0ull ? 1ull : 0ull)) & ((1ull << 47) - 1ull);
  }
  const double mag = __dadd_rn(__dmul_rn((double)hi, 0x1.0p64), (double)lo);
  const double v = __dmul_rn(mag, 0x1.0p-64);
  return neg ? -v : v;
}

__device__ __forceinline__ void red_add(unsigned long long *p, unsigned long long v, bool sys) {
  if (sys)
    asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Kernel parameters the control and helper loops touch every tree, loaded
// once into registers: reading them from the parameter (constant) bank inside
// the loop costs a constant-cache miss -- an L2 round trip -- whenever the
// workers' parameter reads have evicted them.
template <typename T>
__device__ __forceinline__ T *pin_ptr(T *p) {
  asm volatile("" : "+l"(p));
  return p;
}
__device__ __forceinline__ int pin_int(int v) {
  asm volatile("" : "+r"(v));
  return v;
}
// 2^46 / (ctas rounded up to a power of two): the per-CTA bound of to_limbs
__device__ __forceinline__ double xrange_limit(int ctas) {
  int bits = 0;
  while ((1 << bits) < ctas) ++bits;
  return ldexp(1.0, 46 - bits);
}
// the copy group (emulated shard) of a CTA: its index among the groups this
// launch holds, and how many of the launch's CTAs share it
__host__ __device__ __forceinline__ int xgroup(const ChainDev &c, int cta) {
  return c.copy_groups > 1 ? cta % c.copy_groups : 0;
}
__host__ __device__ __forceinline__ int xgroup_ctas(const ChainDev &c, int grp) {
  return c.copy_groups > 1 ? (c.nblk - grp + c.copy_groups - 1) / c.copy_groups : c.nblk;
}

// HIER: the two-level exchange's kernel instantiation; the flat one folds the
// stage fields away (the flat path's code is what it was before two-level)
template <bool HIER>
struct XCtx {
  unsigned long long *xacc, *cacc;  // the copy this CTA polls
  unsigned long long *xstage, *cstage;  // two-level: this CTA's stage words (adds), the forwarder polls them
  int *err;
  int n_shards, nblk_total;
  int target;    // arrivals of a complete copy word: CTAs of all shards, or (two-level) shards
  int grp_ctas;  // two-level: arrivals of a complete stage word
  bool sys, hier, fwd;
  double lim;  // per-CTA fixed-point range (to_limbs)
  __device__ __forceinline__ XCtx(const ChainDev &c, int cta)
      : xacc(pin_ptr(c.copy_groups > 1 ? c.xpeer[c.copy_base + cta % c.copy_groups] : c.xacc)),
        cacc(pin_ptr(c.copy_groups > 1 ? c.cpeer[c.copy_base + cta % c.copy_groups] : c.cacc)),
        xstage(HIER ? pin_ptr(c.xstage + (size_t)xgroup(c, cta) * kXSets * kXSetWords) : nullptr),
        cstage(HIER ? pin_ptr(c.cstage + (size_t)xgroup(c, cta) * kCSets * kCSetWords) : nullptr),
        err(pin_ptr(c.err)), n_shards(pin_int(c.n_shards)), nblk_total(pin_int(c.nblk_total)),
        target(HIER ? n_shards : nblk_total), grp_ctas(HIER ? pin_int(xgroup_ctas(c, xgroup(c, cta))) : 0),
        sys(pin_int(c.shard_sys) != 0), hier(HIER), fwd(HIER && cta == xgroup(c, cta)),
        lim(xrange_limit(c.nblk_total)) {}
};

// Control warp, exchange X: fold the worker warps' f64 partials of ns slots
// (fixed order), add them as fixed-point limbs into every shard's copy of set
// X % 3.  Lane 4j+q handles word q of slot 8k+j, so each warp instruction
// carries 8 slots and the L2 sees one coalesced atomic per slot per CTA (the
// four lanes of a slot fold it redundantly).
__device__ __forceinline__ unsigned long long pick3(const unsigned long long (&l)[3], int q) {
  return q == 0 ? l[0] : (q == 1 ? l[1] : l[2]);
}

template <bool HIER>
__device__ __forceinline__ void exchange_add(const ChainDev &c, const XCtx<HIER> &X, const SweepSmem &S, int ns, int set,
                                             int lane, long long *ts = nullptr) {
  const bool sys = X.sys;
  const size_t set_off = (size_t)set * kXSetWords;
  const int q = lane & 3;
  for (int s0 = 0; s0 < ns; s0 += 8) {
    const int s = s0 + (lane >> 2);
    if (s < ns) {
      double w[kWorkWarps];
#pragma unroll
      for (int k = 0; k < kWorkWarps; ++k) w[k] = S.wsum[k][s];
#pragma unroll
      for (int step = 1; step < kWorkWarps; step <<= 1)  // fixed pairwise order
#pragma unroll
        for (int k = 0; k + step < kWorkWarps; k += 2 * step) w[k] = __dadd_rn(w[k], w[k + step]);
      TL_STAMP(ts && s0 == 0) ts[14] = gtimer_after(w[0]);
      unsigned long long l[3];
      to_limbs(w[0], l, X.err, X.lim);
      TL_STAMP(ts && s0 == 0) ts[15] = gtimer_after(__longlong_as_double((long long)(l[2] | l[1] | l[0])));
      if (q < 3) {
        const unsigned long long v = kTagOne | pick3(l, q);
        if (X.hier)
          red_add(X.xstage + set_off + (size_t)s * kXSlotWords + q, v, false);
        else if (X.n_shards == 1)
          red_add(X.xacc + set_off + (size_t)s * kXSlotWords + q, v, false);
        else
          for (int g = 0; g < X.n_shards; ++g) red_add(c.xpeer[g] + set_off + (size_t)s * kXSlotWords + q, v, sys);
        TL_STAMP(ts && s0 == 0) ts[30] = gtimer();
      }
    }
  }
}

__device__ __forceinline__ void ld_poll1(const unsigned long long *p, unsigned long long &a) {
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(a) : "l"(p) : "memory");
}
__device__ __forceinline__ void ld_poll1s(const unsigned long long *p, unsigned long long &a) {
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(a) : "l"(p) : "memory");
}

// Poll rounds [k0, k0+R) of set `set` until every used word is complete; on
// return lane 4j (q == 0) holds in tot[k] the total of slot 8(k0+k)+j.
template <int R, bool HIER>
__device__ __forceinline__ void poll_rounds(const XCtx<HIER> &X, SweepSmem &S, int ns, int set, int k0, int lane,
                                            double (&tot)[R], long long *ts = nullptr) {
  const bool sys = X.sys;
  const unsigned long long target = (unsigned long long)X.target << kTagShift;
  const unsigned long long *base = X.xacc + (size_t)set * kXSetWords;
  unsigned long long *prev = S.xprev[set];
  const int q = lane & 3;
  unsigned long long w[R];
  bool done;
  do {
    bool ok = true;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int s = 8 * (k0 + k) + (lane >> 2);
      w[k] = 0ull;
      if (s < ns && q < 3) {
        const size_t a = (size_t)s * kXSlotWords + q;
        if (sys)
          ld_poll1s(base + a, w[k]);
        else
          ld_poll1(base + a, w[k]);
        ok = ok && ((w[k] - prev[s * 4 + q]) & ~kDataMask) == target;
      }
    }
    done = __all_sync(0xffffffffu, ok);
  } while (!done);
  TL_STAMP(ts) ts[7] = gtimer_after(__longlong_as_double((long long)w[0]));
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int s = 8 * (k0 + k) + (lane >> 2);
    unsigned long long d = 0ull;
    if (s < ns && q < 3) {
      d = (w[k] - prev[s * 4 + q]) & kDataMask;
      prev[s * 4 + q] = w[k];
    }
    const unsigned long long d1 = __shfl_down_sync(0xffffffffu, d, 1), d2 = __shfl_down_sync(0xffffffffu, d, 2);
    tot[k] = from_limbs(d, d1, d2);
  }
}

// Trees with <= 32 slots: returns the total of slot `lane` in every lane.
template <bool HIER>
__device__ __forceinline__ double exchange_poll_fast(const XCtx<HIER> &X, SweepSmem &S, int ns, int set, int lane,
                                                     long long *ts) {
  const int rounds = (ns + 7) >> 3;
  double mine = 0.0;
  if (rounds <= 1) {
    double t[1];
    poll_rounds<1, HIER>(X, S, ns, set, 0, lane, t, ts);
    mine = __shfl_sync(0xffffffffu, t[0], (lane & 7) * 4);
  } else {
    double t[kFastRounds];
    poll_rounds<kFastRounds, HIER>(X, S, ns, set, 0, lane, t, ts);
#pragma unroll
    for (int k = 0; k < kFastRounds; ++k) {
      const double v = __shfl_sync(0xffffffffu, t[k], (lane & 7) * 4);
      if ((lane >> 3) == k) mine = v;
    }
  }
  return mine;
}

// Any number of slots, one round (8 slots) at a time: totals into S.tot_sum.
template <bool HIER>
__device__ __forceinline__ void exchange_poll_slow(const XCtx<HIER> &X, SweepSmem &S, int ns, int set, int lane) {
  for (int k0 = 0; 8 * k0 < ns; ++k0) {
    double t[1];
    poll_rounds<1, HIER>(X, S, ns, set, k0, lane, t);
    const int s = 8 * k0 + (lane >> 2);
    if ((lane & 3) == 0 && s < ns) S.tot_sum[s] = t[0];
  }
  __syncwarp();
}

// Helper warp, count channel: add this CTA's per-leaf counts of tree j into
// every shard's copy of count set j % 4 / poll the local copy until complete.
template <bool HIER>
__device__ __forceinline__ void counts_add(const ChainDev &c, const XCtx<HIER> &X, const SweepSmem &S, int j, int ns,
                                           int lane) {
  const bool sys = X.sys;
  const size_t off = (size_t)(j % kCSets) * kCSetWords;
  for (int s = lane; s < ns; s += 32) {
    uint32_t cn = 0;
#pragma unroll
    for (int k = 0; k < kWorkWarps; ++k) cn += S.wcnt[j & 1][k][s];
    if (X.hier)
      red_add(X.cstage + off + s, kTagOne | (unsigned long long)cn, false);
    else if (X.n_shards == 1)
      red_add(X.cacc + off + s, kTagOne | (unsigned long long)cn, false);
    else
      for (int g = 0; g < X.n_shards; ++g) red_add(c.cpeer[g] + off + s, kTagOne | (unsigned long long)cn, sys);
  }
}

// Two-level exchange, the shard's forwarder CTA (control warp): poll this
// shard's stage words of set `set` until every CTA of the shard has added,
// then add the shard's totals -- one tagged arrival per word -- into every
// shard's copy.  Integer sums, so the final totals equal the flat exchange's.
template <bool HIER>
__device__ __forceinline__ void forward_stage(const ChainDev &c, const XCtx<HIER> &X, const Geom &G, int ns, int set,
                                              int lane) {
  const unsigned long long target = (unsigned long long)X.grp_ctas << kTagShift;
  const size_t set_off = (size_t)set * kXSetWords;
  const int q = lane & 3;
  for (int s0 = 0; s0 < ns; s0 += 8) {
    const int s = s0 + (lane >> 2);
    const bool mine = s < ns && q < 3;
    unsigned long long w = 0ull;
    bool done;
    do {
      bool ok = true;
      if (mine) {
        ld_poll1(X.xstage + set_off + (size_t)s * kXSlotWords + q, w);
        ok = ((w - G.hs->xsprev[set][s * 4 + q]) & ~kDataMask) == target;
      }
      done = __all_sync(0xffffffffu, ok);
    } while (!done);
    if (mine) {
      const unsigned long long d = (w - G.hs->xsprev[set][s * 4 + q]) & kDataMask;
      G.hs->xsprev[set][s * 4 + q] = w;
      for (int g = 0; g < X.n_shards; ++g) red_add(c.xpeer[g] + set_off + (size_t)s * kXSlotWords + q, kTagOne | d, X.sys);
    }
  }
  __syncwarp();
}

// The same for the count channel (helper warp of the forwarder CTA).
template <bool HIER>
__device__ __forceinline__ void forward_counts(const ChainDev &c, const XCtx<HIER> &X, const Geom &G, int j, int ns,
                                               int lane) {
  const unsigned long long target = (unsigned long long)X.grp_ctas << kTagShift;
  const int set = j % kCSets;
  const size_t off = (size_t)set * kCSetWords;
  for (int s0 = 0; s0 < ns; s0 += 32) {
    const int s = s0 + lane;
    unsigned long long v = 0ull;
    bool done;
    do {
      bool ok = true;
      if (s < ns) {
        ld_poll1(X.cstage + off + s, v);
        ok = ((v - G.hs->csprev[set][s]) & ~kDataMask) == target;
      }
      done = __all_sync(0xffffffffu, ok);
    } while (!done);
    if (s < ns) {
      const unsigned long long d = (v - G.hs->csprev[set][s]) & kDataMask;
      G.hs->csprev[set][s] = v;
      for (int g = 0; g < X.n_shards; ++g) red_add(c.cpeer[g] + off + s, kTagOne | d, X.sys);
    }
  }
  __syncwarp();
}

template <bool HIER>
__device__ __forceinline__ void counts_poll(const XCtx<HIER> &X, SweepSmem &S, int j, int ns, int lane) {
  const bool sys = X.sys;
  const unsigned long long target = (unsigned long long)X.target << kTagShift;
  const int set = j % kCSets;
  const unsigned long long *base = X.cacc + (size_t)set * kCSetWords;
  for (int s0 = 0; s0 < ns; s0 += 32) {
    const int s = s0 + lane;
    unsigned long long v = 0;
    bool done;
    do {
      bool ok = true;
      if (s < ns) {
        if (sys)
          ld_poll1s(base + s, v);
        else
          ld_poll1(base + s, v);
        ok = ((v - S.cprev[set][s]) & ~kDataMask) == target;
      }
      done = __all_sync(0xffffffffu, ok);
    } while (!done);
    if (s < ns) {
      S.hcnt[s] = (uint32_t)((v - S.cprev[set][s]) & kDataMask);
      S.cprev[set][s] = v;
    }
  }
  __syncwarp();
}

// ------------------------------------------------------------ decision
struct DecConst {
  double tau, tau_mu, prior, lm_term;  // 1/sigma2, 1/leaf_sd^2, tau_mu*leaf_mean, 0.5*lm*lm*tau_mu
};

__device__ __forceinline__ bool is_child(int h, int t, bool move) { return move && h >= 2 && (h >> 1) == t; }

// a / b for b > 0 given y = RN(1/b): q0 = RN(a*y) is faithful, the residual
// a - b*q0 is exact in one FMA, and RN(q0 + r*y) is the correctly rounded
// quotient (Markstein).  Bit-identical to __ddiv_rn on 5e9 samples of the
// decision's operand ranges (tools/divtest.cu), at a third of its latency.
__device__ __forceinline__ double div_rcp(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double r = __fma_rn(-b, q0, a);
  const double q1 = __fma_rn(r, y, q0);
  return a == 0.0 ? a : q1;
}

// Helper warp: count-only terms of tree j, from the counts the previous
// exchange delivered.  Same operations, in the same order, as the reference:
// prec = tau_mu + n*tau, z/sqrt(prec) (sampler.py:579-595), adjustment n*adj
// (sampler.py:575-576), and the count part of the ratio (sampler.py:669-684).
__device__ __forceinline__ void prepare(Prep &P, const uint32_t *tot_cnt, const uint8_t *rec, int size,
                                        const TreeHdr hd, int lane, const DecConst &K) {
  const TreeMove &mv = rec_hdr(rec);
  const float *old_leaf = rec_leaf(rec);
  const double *z = rec_z(rec, size);
  const int kind = hd.kind, t = hd.node, ns = hd.nslots;
  const bool grow = kind == KIND_GROW, move = kind != KIND_NONE;
  for (int j = lane; j < ns; j += 32) {
    const int h = mv.slot_node[j];
    const uint32_t cn = tot_cnt[j];
    const float a32 = (grow && is_child(h, t, move)) ? old_leaf[t] : old_leaf[h];
    const double prec = __dadd_rn(K.tau_mu, __dmul_rn((double)cn, K.tau));
    P.cnt[j] = cn;
    P.cadj[j] = __dmul_rn((double)cn, (double)a32);
    P.prec[j] = prec;
    P.rcp[j] = __drcp_rn(prec);
    P.zs[j] = __ddiv_rn(z[h], __dsqrt_rn(prec));
  }
  __syncwarp();
  if (move && lane < 2) {
    const uint32_t nl = P.cnt[hd.slot_l], nr = P.cnt[hd.slot_r];
    const double prec_l = P.prec[hd.slot_l], prec_r = P.prec[hd.slot_r];
    const double prec_p = __dadd_rn(K.tau_mu, __dmul_rn((double)(nl + nr), K.tau));
    if (lane == 0) {
      P.prec_l = prec_l;
      P.prec_r = prec_r;
      P.prec_p = prec_p;
      P.rcp_p = __drcp_rn(prec_p);
      P.zs_p = __ddiv_rn(z[t], __dsqrt_rn(prec_p));
    } else {
      const double q = __ddiv_rn(__dmul_rn(K.tau_mu, prec_p), __dmul_rn(prec_l, prec_r));
      P.partial = __dadd_rn(mv.struct_log, __dsub_rn(__dmul_rn(0.5, log(q)), K.lm_term));
    }
  }
  __syncwarp();
}

// Control warp, phases 8-10 of tree e (critical path): tree-excluded sums,
// posterior means (one division each), the acceptance test and the residual
// delta per leaf of the larger tree.
__device__ __forceinline__ void decide(SweepSmem &S, const Prep &P, Dec &Do, const uint8_t *rec, const TreeHdr hd,
                                       int lane, const DecConst &K) {
  const TreeMove &mv = rec_hdr(rec);
  const float *old_leaf = rec_leaf(rec);
  const int kind = hd.kind, t = hd.node, ns = hd.nslots;
  const bool grow = kind == KIND_GROW, move = kind != KIND_NONE;
  const int sl_i = hd.slot_l, sr_i = hd.slot_r;
  for (int base = 0; base <= ns; base += 32) {
    const int j = base + lane;
    double num = 1.0, den = 1.0, rcp = 1.0, zs = 0.0;
    if (j < ns) {
      const double sums = __dadd_rn(S.tot_sum[j], P.cadj[j]);  // sampler.py:570-576
      Do.sums_s[j] = sums;
      num = __dadd_rn(K.prior, __dmul_rn(K.tau, sums));
      den = P.prec[j];
      rcp = P.rcp[j];
      zs = P.zs[j];
    } else if (j == ns && move) {  // the collapsed parent: count nl+nr, sum sl+sr (sampler.py:861-866)
      const double sl = __dadd_rn(S.tot_sum[sl_i], P.cadj[sl_i]);
      const double sr = __dadd_rn(S.tot_sum[sr_i], P.cadj[sr_i]);
      num = __dadd_rn(K.prior, __dmul_rn(K.tau, __dadd_rn(sl, sr)));
      den = P.prec_p;
      rcp = P.rcp_p;
      zs = P.zs_p;
    }
    const double q = div_rcp(num, den, rcp);
    if (j <= ns) {
      S.q_s[j] = q;
      Do.v_s[j] = __dadd_rn(q, zs);
    }
  }
  __syncwarp();
  int acc = 0;
  if (move && lane == 0) {
    // sum part (sampler.py:634-645): mean*mean*prec with the leaf posterior means
    const double ml = S.q_s[sl_i], mr = S.q_s[sr_i], mp = S.q_s[ns];
    const double tl = __dmul_rn(__dmul_rn(ml, ml), P.prec_l);
    const double tr = __dmul_rn(__dmul_rn(mr, mr), P.prec_r);
    const double tp = __dmul_rn(__dmul_rn(mp, mp), P.prec_p);
    const double sum_part = __dmul_rn(0.5, __dsub_rn(__dadd_rn(tl, tr), tp));
    const double la = __dmul_rn(grow ? 1.0 : -1.0, __dadd_rn(P.partial, sum_part));
    // accept iff u < exp(min(la, 0)) (sampler.py:833-834), decided through the
    // precomputed log(u) outside a 1e-9 band around the tie; inside the band
    // the reference's exp comparison is evaluated as written
    if (la >= 0.0)
      acc = 1;
    else if (la < mv.log_u - 1e-9)
      acc = 0;
    else if (la > mv.log_u + 1e-9)
      acc = 1;
    else
      acc = mv.acc_u < exp(la);
  }
  acc = __shfl_sync(0xffffffffu, acc, 0);
  const bool fsmall = move && ((acc != 0) != grow);  // sampler.py:861
  const float v_par = __double2float_rn(Do.v_s[ns]);
  // residual delta per leaf of the larger tree (sampler.py:755-760)
  for (int j = lane; j < ns; j += 32) {
    const int h = mv.slot_node[j];
    const bool child = is_child(h, t, move);
    const int oi = (grow && child) ? t : h;
    const float nv = (fsmall && child) ? v_par : __double2float_rn(Do.v_s[j]);
    S.dlt[h] = __fsub_rn(old_leaf[oi], nv);
  }
  if (lane == 0) {
    S.flag_wr = acc;
    S.flag_prune = acc && !grow;
    S.flag_t = t;
    Do.acc = acc;
  }
  __syncwarp();
}

// The same decision with lane s holding slot s in registers (trees whose
// larger tree has <= 31 leaves: every depth <= 5 tree and nearly every depth-6
// one).  Identical operations and order to decide().  Every lane evaluates
// the acceptance test itself from the two children's totals (one shuffle
// round on the critical path, no broadcast of the outcome), and every input
// that does not depend on the exchange is loaded before it completes.
struct DecIn {
  double cadj, den, rcp, zs;  // own slot (lane < ns)
  float oldv;
  int h;
  bool child;
};

__device__ __forceinline__ void decide_load(DecIn &I, const Prep &P, const uint8_t *rec, const TreeHdr hd, int lane) {
  const TreeMove &mv = rec_hdr(rec);
  const float *old_leaf = rec_leaf(rec);
  const int kind = hd.kind, t = hd.node, ns = hd.nslots;
  const bool grow = kind == KIND_GROW, move = kind != KIND_NONE;
  I.cadj = 0.0;
  I.den = 1.0;
  I.rcp = 1.0;
  I.zs = 0.0;
  I.oldv = 0.f;
  I.h = 0;
  I.child = false;
  if (lane < ns) {
    I.cadj = P.cadj[lane];
    I.den = P.prec[lane];
    I.rcp = P.rcp[lane];
    I.zs = P.zs[lane];
    I.h = mv.slot_node[lane];
    I.child = is_child(I.h, t, move);
    I.oldv = old_leaf[(grow && I.child) ? t : I.h];
  }
}

__device__ __forceinline__ bool accept_near_tie(double la, double acc_u) { return acc_u < exp(la); }

__device__ __forceinline__ void decide_fast(SweepSmem &S, Dec &Do, const DecIn &I, double tot, const Prep &P,
                                            const uint8_t *rec, const TreeHdr hd, int lane, const DecConst &K,
                                            long long *ts) {
  const int kind = hd.kind, t = hd.node, ns = hd.nslots;
  const bool grow = kind == KIND_GROW, move = kind != KIND_NONE;
  const double tl = __shfl_sync(0xffffffffu, tot, hd.slot_l), tr = __shfl_sync(0xffffffffu, tot, hd.slot_r);
  // own leaf (sampler.py:570-595)
  const double sums = __dadd_rn(tot, I.cadj);
  const double q = div_rcp(__dadd_rn(K.prior, __dmul_rn(K.tau, sums)), I.den, I.rcp);
  const double v = __dadd_rn(q, I.zs);
  int acc = 0;
  double vp = 0.0;
  if (move) {
    // the children and the collapsed parent (sampler.py:861-866), then the sum
    // part (sampler.py:634-645) and the test (sampler.py:833-834) -- in every
    // lane; the move terms are warp-uniform shared loads issued alongside the
    // shuffles
    const TreeMove &mv = rec_hdr(rec);
    const double cadj_l = P.cadj[hd.slot_l], cadj_r = P.cadj[hd.slot_r];
    const double prec_l = P.prec_l, prec_r = P.prec_r, prec_p = P.prec_p;
    const double rcp_l = P.rcp[hd.slot_l], rcp_r = P.rcp[hd.slot_r], rcp_p = P.rcp_p;
    const double sl = __dadd_rn(tl, cadj_l), sr = __dadd_rn(tr, cadj_r);
    const double ml = div_rcp(__dadd_rn(K.prior, __dmul_rn(K.tau, sl)), prec_l, rcp_l);
    const double mr = div_rcp(__dadd_rn(K.prior, __dmul_rn(K.tau, sr)), prec_r, rcp_r);
    const double mp = div_rcp(__dadd_rn(K.prior, __dmul_rn(K.tau, __dadd_rn(sl, sr))), prec_p, rcp_p);
    vp = __dadd_rn(mp, P.zs_p);
    const double t_l = __dmul_rn(__dmul_rn(ml, ml), prec_l);
    const double t_r = __dmul_rn(__dmul_rn(mr, mr), prec_r);
    const double t_p = __dmul_rn(__dmul_rn(mp, mp), prec_p);
    const double sum_part = __dmul_rn(0.5, __dsub_rn(__dadd_rn(t_l, t_r), t_p));
    const double la = __dmul_rn(grow ? 1.0 : -1.0, __dadd_rn(P.partial, sum_part));
    const double log_u = mv.log_u;
    if (la >= 0.0 || la > log_u + 1e-9)
      acc = 1;
    else if (la < log_u - 1e-9)
      acc = 0;
    else
      acc = accept_near_tie(la, mv.acc_u) ? 1 : 0;
  }
  TL_STAMP(ts) ts[10] = gtimer_after((double)acc);
  const bool fsmall = move && ((acc != 0) != grow);
  if (lane < ns) {  // residual delta (sampler.py:755-760)
    const float nv = (fsmall && I.child) ? __double2float_rn(vp) : __double2float_rn(v);
    S.dlt[I.h] = __fsub_rn(I.oldv, nv);
  }
  if (lane == 0) {
    S.flag_wr = acc;
    S.flag_prune = acc && !grow;
    S.flag_t = t;
  }
  __syncwarp();
  named_arrive(BAR_DECISION, kBarWC);
  // for the helper's bookkeeping (off the critical path)
  if (lane < ns) {
    Do.sums_s[lane] = sums;
    Do.v_s[lane] = v;
  }
  if (lane == 0) {
    Do.v_s[ns] = vp;
    Do.acc = acc;
  }
}

// Helper warp, one CTA per tree: accept flag, structure write, the new leaf
// row (final leaves keep their draw, other slots a signed zero; sampler.py:
// 836-848, 868-870) and the parity taps.
__device__ __forceinline__ void decide_post(const ChainDev &c, SweepSmem &S, const Prep &P, const Dec &Di,
                                            const uint8_t *rec, const TreeHdr hd, int e, int lane,
                                            const DecConst &K, int64_t hist_row) {
  const TreeMove &mv = rec_hdr(rec);
  const double *z = rec_z(rec, c.size);
  const int size = c.size, half = c.half;
  const int kind = hd.kind, t = hd.node, ns = hd.nslots;
  const bool grow = kind == KIND_GROW, move = kind != KIND_NONE;
  const int acc = Di.acc;
  const bool fsmall = move && ((acc != 0) != grow);
  const float v_par = __double2float_rn(Di.v_s[ns]);
  if (lane == 0) {
    c.accepted[e] = (uint8_t)acc;
    if (hist_row >= 0) c.acc_hist[hist_row * c.m + e] = (uint8_t)acc;  // fit() trace (regression.py:190)
    if (acc) {
      c.axis[(size_t)e * half + t] = grow ? hd.axis : (uint16_t)0;
      c.cut[(size_t)e * half + t] = grow ? hd.cut : (uint8_t)0;
    }
  }
  for (int h = lane; h < size; h += 32) {
    float z0;
    if (K.prior == 0.0) {
      z0 = copysignf(0.0f, (float)z[h]);  // 0 + z/sqrt(tau_mu) has the sign of z
    } else {
      const double v0 = __dadd_rn(__ddiv_rn(K.prior, K.tau_mu), __ddiv_rn(z[h], __dsqrt_rn(K.tau_mu)));
      z0 = __double2float_rn(__dmul_rn(v0, 0.0));
    }
    S.row[h] = z0;
  }
  __syncwarp();
  for (int j = lane; j < ns; j += 32) {
    const int h = mv.slot_node[j];
    if (!(fsmall && is_child(h, t, move))) S.row[h] = __double2float_rn(Di.v_s[j]);
  }
  if (lane == 0 && fsmall) S.row[t] = v_par;
  __syncwarp();
  for (int h = lane; h < size; h += 32) c.leaf[(size_t)e * size + h] = S.row[h];
  if (c.taps) {
    for (int h = lane; h < size; h += 32) {
      c.tap_counts[(size_t)e * size + h] = 0;
      c.tap_sums[(size_t)e * size + h] = 0.0;
    }
    __syncwarp();
    for (int j = lane; j < ns; j += 32) {
      const int h = mv.slot_node[j];
      c.tap_counts[(size_t)e * size + h] = (int64_t)P.cnt[j];
      c.tap_sums[(size_t)e * size + h] = Di.sums_s[j];
    }
  }
  __syncwarp();
}

// ------------------------------------------------------------ warp roles
// Worker warps: the register-resident point chunk, one A and one B pass per tree.
template <int W>
__device__ __forceinline__ void worker_loop(const ChainDev &c, SweepSmem &S, const Geom &G, int tid, int warp, int lane,
                                            long long *tl) {
  float4 r[W];
  uint32_t lp[W], lc[W], ln[W];  // larger-tree indices of trees e-1, e, e+1
  const float4 *gr4 = reinterpret_cast<const float4 *>(c.r + G.start);
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const int w = tid + k * kWorkers;
    r[k] = w < G.nwords ? gr4[w] : make_float4(0.f, 0.f, 0.f, 0.f);
    lp[k] = lc[k] = ln[k] = 0u;
  }
  // role prologue barrier (mbarriers initialised, first trees in flight),
  // reached by each warp role from its own code, as the per-tree named
  // barriers are: warp-uniform, role-divergent bar.sync, the warp-specialised
  // pattern of CUTLASS's NamedBarrier.  (The non-.aligned barrier.sync forms,
  // which compute-sanitizer's synccheck accepts, measured 8% slower, and so
  // did an mbarrier here: code layout.)
  named_sync(BAR_ROLES, kSweepThreads);
  const int m = G.m;
  if (m > 0) {  // tree 0: refresh + counts
    mbar_wait(&S.mbar[0], 0u);
    refresh_count<W>(ln, G.slot(0), G, G.hdr[0], rec_hdr(G.rec(0)).slot_node, S.wcnt[0][warp], tid, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.cnt_mbar[0]);
  }
  for (int e = -1; e <= m; ++e) {
    TL_STAMP(tl) tl[(size_t)(e + 1) * 32 + 0] = gtimer_after((double)S.flag_t);  // after the barrier releases
    // ---- A_e: critical path
    if (e >= 0 && e < m) {
      APass A;
      A.do_update = e > 0;
      A.wr = e > 0 && S.flag_wr;
      A.prune = e > 0 && S.flag_prune;
      A.t = (uint32_t)S.flag_t;
      A.gL = reinterpret_cast<uint32_t *>(c.L + (size_t)(e > 0 ? e - 1 : 0) * c.n_pad + G.start);
      A.slots = rec_hdr(G.rec(e)).slot_node;
      A.ns = G.hdr[e].nslots;
      long long *ts = tl ? tl + (size_t)(e + 1) * 32 : nullptr;
      TL_STAMP(ts) ts[26] = gtimer_after((double)A.ns + (double)A.slots[0]);
      sums_passes<W>(r, lp, lc, A, G, S.dlt, S, tid, warp, lane, ts);
#if BART_TIMELINE
      if (lane == 0 && G.cta == 0 && c.timeline && warp < 8) {  // worker warps' A-pass ends (0-7)
        const volatile double dep = S.wsum[warp][0];
        (void)dep;
        c.timeline[(size_t)(e + 1) * 32 + 16 + warp] = gtimer();
      }
#endif
      named_arrive(BAR_PARTIALS, kBarWC);
    } else if (e == m) {  // tree m-1's update, residual write-back, sum of squares (sampler.py:790-794)
      const bool wr = m > 0 && S.flag_wr, prune = S.flag_prune;
      const uint32_t t = (uint32_t)S.flag_t;
      uint32_t *gL = reinterpret_cast<uint32_t *>(c.L + (size_t)(m > 0 ? m - 1 : 0) * c.n_pad + G.start);
      float4 *out = reinterpret_cast<float4 *>(c.r + G.start);
      double ss = 0.0;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const int w = tid + k * kWorkers;
        if (w < G.nwords) {
          if (m > 0) r[k] = update4(r[k], lp[k], S.dlt);
          if (wr) gL[w] = prune ? collapse4(lp[k], t) : lp[k];
          out[w] = r[k];
          const double a = r[k].x, b = r[k].y, cc = r[k].z, d = r[k].w;
          ss = __dadd_rn(ss, __dmul_rn(a, a));
          ss = __dadd_rn(ss, __dmul_rn(b, b));
          ss = __dadd_rn(ss, __dmul_rn(cc, cc));
          ss = __dadd_rn(ss, __dmul_rn(d, d));
        }
      }
      const double v = warp_sum_f64(ss);
      if (lane == 0) S.wsum[warp][0] = v;
      named_arrive(BAR_PARTIALS, kBarWC);
      break;
    }
    TL_STAMP(tl) tl[(size_t)(e + 1) * 32 + 1] = gtimer();
    // ---- B_e: tree e+2's refresh + counts, hidden behind the exchange
    uint32_t lnn[W];
    const int j2 = e + 2;
    if (j2 < m) {
      mbar_wait(&S.mbar[j2 % kRing], (uint32_t)((j2 / kRing) & 1));
      refresh_count<W>(lnn, G.slot(j2), G, G.hdr[j2], rec_hdr(G.rec(j2)).slot_node, S.wcnt[j2 & 1][warp], tid,
                       lane);
      fence_proxy_async();  // generic reads of the ring slot before its next TMA refill
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.cnt_mbar[j2 & 1]);
    } else {
#pragma unroll
      for (int k = 0; k < W; ++k) lnn[k] = 0u;
    }
#pragma unroll
    for (int k = 0; k < W; ++k) {  // rotate: e-1 <- e <- e+1 <- e+2
      lp[k] = lc[k];
      lc[k] = ln[k];
      ln[k] = lnn[k];
    }
    TL_STAMP(tl) tl[(size_t)(e + 1) * 32 + 2] = gtimer();
    if (e >= 0) named_sync(BAR_DECISION, kBarWC);  // decision of tree e installed (S.dlt, flags)
    TL_STAMP(tl) tl[(size_t)(e + 1) * 32 + 3] = gtimer();
  }
}

// ------------------------------------------------------------ stream mode
// Chunks beyond the register budget (n per device > ~2.2M): the residuals
// stay in global memory, L2-resident (4n bytes: 40 MB at n = 1e7), and tree
// j's refreshed larger-tree row goes to the global scratch ring Lref[j % 3].
// Same passes as the register mode, over tiles of kTileW words per thread.
constexpr int kTileW = 4;

__device__ __forceinline__ const uint8_t *lref_row(const ChainDev &c, const Geom &G, int j) {
  return c.Lref + (size_t)(j % 3) * c.n_pad + G.start;
}

// A pass (first = tree e-1's update + cache write), f64 sums of slots
// [base, base+C) (+ running total when TOTAL) accumulated over the chunk.
template <int C, bool TOTAL>
__device__ __forceinline__ void stream_sums(const ChainDev &c, const Geom &G, const APass &A, const uint32_t *lp32,
                                            const uint32_t *lc32, const float *dlt, SweepSmem &S, int tid, int warp,
                                            int lane, int base, bool first) {
  uint32_t sn[C > 0 ? C : 1];
  double acc[C > 0 ? C : 1];
  double tot = 0.0;
#pragma unroll
  for (int s = 0; s < C; ++s) {
    sn[s] = base + s < (TOTAL ? A.ns - 1 : A.ns) ? A.slots[base + s] : 0xffffu;
    acc[s] = 0.0;
  }
  float4 *rg = reinterpret_cast<float4 *>(c.r + G.start);
  const bool upd = first && A.do_update;
  for (int w0 = 0; w0 < G.nwords; w0 += kWorkers * kTileW) {
    float4 r[kTileW];
    uint32_t lp[kTileW], lc[kTileW];
#pragma unroll
    for (int k = 0; k < kTileW; ++k) {
      const int w = w0 + tid + k * kWorkers;
      if (w < G.nwords) {
        r[k] = rg[w];
        lc[k] = lc32[w];
        lp[k] = upd ? lp32[w] : 0u;
      }
    }
#pragma unroll
    for (int k = 0; k < kTileW; ++k) {
      const int w = w0 + tid + k * kWorkers;
      if (w < G.nwords) {
        if (upd) {
          r[k] = update4(r[k], lp[k], dlt);
          if (A.wr) A.gL[w] = A.prune ? collapse4(lp[k], A.t) : lp[k];
          rg[w] = r[k];
        }
        const float rv[4] = {r[k].x, r[k].y, r[k].z, r[k].w};
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint32_t h = (lc[k] >> (8 * b)) & 0xffu;
          const double v = (double)rv[b];
          if (TOTAL) tot = __dadd_rn(tot, v);
#pragma unroll
          for (int s = 0; s < C; ++s) add_if_eq(acc[s], h, sn[s], v);
        }
      }
    }
  }
  store_warp_sums<C, TOTAL>(acc, tot, A, S, warp, lane, base);
}

__device__ __forceinline__ void stream_sums_all(const ChainDev &c, const Geom &G, const APass &A, const uint32_t *lp32,
                                                const uint32_t *lc32, const float *dlt, SweepSmem &S, int tid, int warp,
                                                int lane) {
  switch (A.ns) {
    case 1: stream_sums<0, true>(c, G, A, lp32, lc32, dlt, S, tid, warp, lane, 0, true); break;
    case 2: stream_sums<1, true>(c, G, A, lp32, lc32, dlt, S, tid, warp, lane, 0, true); break;
    case 3: stream_sums<2, true>(c, G, A, lp32, lc32, dlt, S, tid, warp, lane, 0, true); break;
    case 4: stream_sums<3, true>(c, G, A, lp32, lc32, dlt, S, tid, warp, lane, 0, true); break;
    default:  // wide trees: further passes re-read the (updated) residuals
      // (per-width variants here cost 28% at n = 1e7: the stream loop spills)
      stream_sums<8, false>(c, G, A, lp32, lc32, dlt, S, tid, warp, lane, 0, true);
      for (int base = 8; base < A.ns; base += 8) {
        if (A.ns - base <= 4)  // a 4-slot tail (+9% at n = 1e7, where most trees have 9-12 slots)
          stream_sums<4, false>(c, G, A, lp32, lc32, dlt, S, tid, warp, lane, base, false);
        else
          stream_sums<8, false>(c, G, A, lp32, lc32, dlt, S, tid, warp, lane, base, false);
      }
  }
}

// B pass: tree j's row from global memory -> grow refresh -> Lref[j % 3], and
// per-slot counts of slots [base, base+NS).
template <int NS>
__device__ __forceinline__ void stream_refresh_count(const ChainDev &c, const Geom &G, int j, const TreeHdr hd,
                                                     const uint8_t *slots, uint32_t *wrow, int tid, int lane,
                                                     int base, bool write) {
  const uint32_t *L32 = reinterpret_cast<const uint32_t *>(c.L + (size_t)j * c.n_pad + G.start);
  const uint32_t *X32 = reinterpret_cast<const uint32_t *>(c.Xt + (size_t)hd.axis * c.n_pad + G.start);
  uint32_t *O32 = reinterpret_cast<uint32_t *>(const_cast<uint8_t *>(lref_row(c, G, j)));
  const bool g = hd.kind == KIND_GROW;
  const uint32_t t4 = 0x01010101u * hd.node, c4 = 0x01010101u * hd.cut, b4 = 0x01010101u * (2u * hd.node);
  const int ns = hd.nslots;
  uint32_t cnt[NS], s4[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    s4[s] = base + s < ns ? 0x01010101u * (uint32_t)slots[base + s] : 0xffffffffu;
    cnt[s] = 0u;
  }
  for (int w0 = 0; w0 < G.nwords; w0 += kWorkers * kTileW) {
    uint32_t l[kTileW], x[kTileW];
#pragma unroll
    for (int k = 0; k < kTileW; ++k) {
      const int w = w0 + tid + k * kWorkers;
      l[k] = 0u;
      x[k] = 0u;
      if (w < G.nwords) {
#ifndef BART_STREAM_EVICT_FIRST
#define BART_STREAM_EVICT_FIRST 1
#endif
        // the cache row and split column are read once per sweep: streaming
        // loads, so they do not evict the L2-resident residuals and Lref rows
        if (BART_STREAM_EVICT_FIRST) {
          l[k] = write ? __ldcs(L32 + w) : O32[w];
          if (write && g) x[k] = __ldcs(X32 + w);
        } else {
          l[k] = write ? L32[w] : O32[w];
          if (write && g) x[k] = X32[w];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kTileW; ++k) {
      const int w = w0 + tid + k * kWorkers;
      if (w < G.nwords) {
        if (write) {
          if (g) l[k] = grow4s(l[k], x[k], t4, c4, b4);
          O32[w] = l[k];
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) cnt[s] += __popc(bytes_eq(l[k], s4[s]));
      }
    }
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const uint32_t cc = __reduce_add_sync(0xffffffffu, cnt[s]);
    if (lane == 0 && base + s < ns) wrow[base + s] = cc;
  }
}

__device__ __forceinline__ void stream_refresh_count_all(const ChainDev &c, const Geom &G, int j, const TreeHdr hd,
                                                         const uint8_t *slots, uint32_t *wrow, int tid, int lane) {
  const int ns = hd.nslots;
  if (ns <= 2)
    stream_refresh_count<2>(c, G, j, hd, slots, wrow, tid, lane, 0, true);
  else if (ns <= 4)
    stream_refresh_count<4>(c, G, j, hd, slots, wrow, tid, lane, 0, true);
  else
    for (int base = 0; base < ns; base += 8) {  // later groups re-read the refreshed row
      if (ns - base <= 4)
        stream_refresh_count<4>(c, G, j, hd, slots, wrow, tid, lane, base, base == 0);
      else
        stream_refresh_count<8>(c, G, j, hd, slots, wrow, tid, lane, base, base == 0);
    }
}

__device__ __forceinline__ void stream_worker_loop(const ChainDev &c, SweepSmem &S, const Geom &G, int tid, int warp,
                                                   int lane) {
  named_sync(BAR_ROLES, kSweepThreads);  // role prologue barrier
  const int m = G.m;
  if (m > 0) {
    mbar_wait(&S.mbar[0], 0u);
    stream_refresh_count_all(c, G, 0, G.hdr[0], rec_hdr(G.rec(0)).slot_node, S.wcnt[0][warp], tid, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.cnt_mbar[0]);
  }
  for (int e = -1; e <= m; ++e) {
    if (e >= 0 && e < m) {
      APass A;
      A.do_update = e > 0;
      A.wr = e > 0 && S.flag_wr;
      A.prune = e > 0 && S.flag_prune;
      A.t = (uint32_t)S.flag_t;
      A.gL = reinterpret_cast<uint32_t *>(c.L + (size_t)(e > 0 ? e - 1 : 0) * c.n_pad + G.start);
      A.slots = rec_hdr(G.rec(e)).slot_node;
      A.ns = G.hdr[e].nslots;
      stream_sums_all(c, G, A, reinterpret_cast<const uint32_t *>(lref_row(c, G, e > 0 ? e - 1 : 0)),
                      reinterpret_cast<const uint32_t *>(lref_row(c, G, e)), S.dlt, S, tid, warp, lane);
      named_arrive(BAR_PARTIALS, kBarWC);
    } else if (e == m) {  // tree m-1's update, sum of squares (sampler.py:790-794)
      const bool wr = m > 0 && S.flag_wr, prune = S.flag_prune;
      const uint32_t t = (uint32_t)S.flag_t;
      uint32_t *gL = reinterpret_cast<uint32_t *>(c.L + (size_t)(m > 0 ? m - 1 : 0) * c.n_pad + G.start);
      const uint32_t *lp32 = reinterpret_cast<const uint32_t *>(lref_row(c, G, m > 0 ? m - 1 : 0));
      float4 *rg = reinterpret_cast<float4 *>(c.r + G.start);
      double ss = 0.0;
      for (int w = tid; w < G.nwords; w += kWorkers) {
        float4 r = rg[w];
        if (m > 0) {
          const uint32_t lp = lp32[w];
          r = update4(r, lp, S.dlt);
          if (wr) gL[w] = prune ? collapse4(lp, t) : lp;
          rg[w] = r;
        }
        const double a = r.x, b = r.y, cc = r.z, d = r.w;
        ss = __dadd_rn(ss, __dmul_rn(a, a));
        ss = __dadd_rn(ss, __dmul_rn(b, b));
        ss = __dadd_rn(ss, __dmul_rn(cc, cc));
        ss = __dadd_rn(ss, __dmul_rn(d, d));
      }
      const double v = warp_sum_f64(ss);
      if (lane == 0) S.wsum[warp][0] = v;
      named_arrive(BAR_PARTIALS, kBarWC);
      break;
    }
    const int j2 = e + 2;
    if (j2 < m) {
      mbar_wait(&S.mbar[j2 % kRing], (uint32_t)((j2 / kRing) & 1));
      stream_refresh_count_all(c, G, j2, G.hdr[j2], rec_hdr(G.rec(j2)).slot_node, S.wcnt[j2 & 1][warp], tid, lane);
      fence_proxy_async();  // generic reads of the record before its slot's next TMA refill
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.cnt_mbar[j2 & 1]);
    }
    if (e >= 0) named_sync(BAR_DECISION, kBarWC);
  }
}

// Control warp: exchange and decision, nothing else.
template <bool HIER>
__device__ __forceinline__ void control_loop(const ChainDev &c, SweepSmem &S, const Geom &G, int lane,
                                             const DecConst &K, unsigned long long xbase, long long *tl) {
  const int m = G.m;
  const XCtx<HIER> X(c, G.cta);
  named_sync(BAR_ROLES, kSweepThreads);  // role prologue barrier
  for (int e = 0; e <= m; ++e) {
    const bool has_cur = e < m;
    const TreeHdr hd = has_cur ? G.hdr[e] : TreeHdr{};
    const int ns = has_cur ? hd.nslots : 1;  // e == m: sum of squares in slot 0
    const int set = (int)((xbase + (unsigned long long)e) % kXSets);
    const bool fast = ns < 32;

    named_sync(BAR_PARTIALS, kBarWC);  // A_e partials complete
    // (BAR.SYNC defers blocking to the next dependent instruction: stamp after a shared load)
    TL_STAMP(tl) tl[(size_t)(e + 1) * 32 + 4] = gtimer_after(S.wsum[0][0]);
#if BART_TIMELINE
    if (c.trace && lane == 0) {
      const volatile double dep = S.wsum[0][0];
      (void)dep;
      c.trace[((size_t)(e + 1) * G.nblk + G.cta) * 2 + 0] = nstimer();
    }
#endif
    long long *ts = tl ? tl + (size_t)(e + 1) * 32 : nullptr;
    exchange_add(c, X, S, ns, set, lane, ts);
    if (X.fwd) forward_stage(c, X, G, ns, set, lane);
    TL_STAMP(ts) ts[5] = gtimer();
    DecIn I;
    if (has_cur) {
      mbar_wait(&S.prep_mbar[e & 1], par2(e));  // helper: prep(e) ready
      if (fast) decide_load(I, S.prep[e & 1], G.rec(e), hd, lane);
    }
    TL_STAMP(ts) ts[6] = gtimer();
    double tot = 0.0;
    if (fast)
      tot = exchange_poll_fast(X, S, ns, set, lane, ts);
    else
      exchange_poll_slow(X, S, ns, set, lane);
    TL_STAMP(ts) ts[8] = gtimer_after(tot);
#if BART_TIMELINE
    if (c.trace && lane == 0) c.trace[((size_t)(e + 1) * G.nblk + G.cta) * 2 + 1] = nstimer();
#endif
    if (has_cur && fast) {
      decide_fast(S, S.dec[e & 1], I, tot, S.prep[e & 1], G.rec(e), hd, lane, K, ts);
      TL_STAMP(ts) ts[11] = gtimer();
    } else {
      if (fast && lane < ns) S.tot_sum[lane] = tot;
      __syncwarp();
      if (has_cur) {
        decide(S, S.prep[e & 1], S.dec[e & 1], G.rec(e), hd, lane, K);
        named_arrive(BAR_DECISION, kBarWC);
      }
    }
    TL_STAMP(tl) tl[(size_t)(e + 1) * 32 + 12] = gtimer();
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.dec_mbar[e & 1]);  // dec[e & 1] (or sum r^2) for the helper
  }
}

// Helper warp: prefetch, count channel, count-only precomputation, bookkeeping.
template <bool HIER>
__device__ __forceinline__ void helper_loop(const ChainDev &c, SweepSmem &S, const Geom &G, int lane,
                                            const DecConst &K, unsigned long long xbase, long long *tl) {
  const int m = G.m;
  const XCtx<HIER> X(c, G.cta);
  // trace row of this iteration (read before the sigma CTA bumps the counter)
  const int64_t hrow = c.acc_hist ? (int64_t)*c.iter_dev - c.hist_base : -1;
  const int64_t hist_row = (hrow >= 0 && hrow < c.hist_cap) ? hrow : -1;
  // the step's chi-square draw, read now: an injected block lives in pinned
  // host memory (one host-link round trip, off the sweep's tail)
  const double chi2 = G.cta == c.m % G.nblk ? *c.rand_chi2 : 0.0;
  auto issue_tree = [&](int j) {  // lane 0: cache row, split column, record -> ring slot j % kRing
    const TreeHdr hd = G.hdr[j];
    unsigned long long *mb = &S.mbar[j % kRing];
    uint8_t *dst = G.slot(j);
    const bool g = hd.kind == KIND_GROW;
    const uint32_t rb = (uint32_t)c.rstride;
    if (G.row_bytes == 0) {  // stream mode: the workers read the rows from global memory
      mbar_expect(mb, rb);
      bulk_g2s(dst, c.rec + (size_t)j * rb, rb, mb);
      return;
    }
    mbar_expect(mb, (g ? 2u * G.lenp : G.lenp) + rb);
    bulk_g2s(dst, c.L + (size_t)j * c.n_pad + G.start, G.lenp, mb);
    if (g) bulk_g2s(dst + G.chunk, c.Xt + (size_t)hd.axis * c.n_pad + G.start, G.lenp, mb);
    bulk_g2s(dst + G.row_bytes, c.rec + (size_t)j * rb, rb, mb);
  };
  auto prepare_tree = [&](int j) {
    mbar_wait(&S.mbar[j % kRing], (uint32_t)((j / kRing) & 1));
    counts_poll(X, S, j, G.hdr[j].nslots, lane);
    prepare(S.prep[j & 1], S.hcnt, G.rec(j), G.size, G.hdr[j], lane, K);
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.prep_mbar[j & 1]);
  };
  if (lane == 0)
    for (int j = 0; j < kRing && j < m; ++j) issue_tree(j);
  named_sync(BAR_ROLES, kSweepThreads);  // role prologue barrier
  for (int j = 0; j < 2 && j < m; ++j) {  // counts of trees 0 and 1
    mbar_wait(&S.cnt_mbar[j & 1], par2(j));
    counts_add(c, X, S, j, G.hdr[j].nslots, lane);
    if (X.fwd) forward_counts(c, X, G, j, G.hdr[j].nslots, lane);
  }
  if (m > 0) prepare_tree(0);
  for (int e = 0; e <= m; ++e) {
    if (e + 2 < m) {  // B_e done: publish the counts of tree e+2
      mbar_wait(&S.cnt_mbar[e & 1], par2(e + 2));
      counts_add(c, X, S, e + 2, G.hdr[e + 2].nslots, lane);
      if (X.fwd) forward_counts(c, X, G, e + 2, G.hdr[e + 2].nslots, lane);
    }
    // tree e+1's count-only terms: prep[(e+1)&1] was last read by decide(e-1)
    // and decide_post(e-1), both done
    if (e + 1 < m) prepare_tree(e + 1);
    TL_STAMP(tl) tl[(size_t)(e + 1) * 32 + 13] = gtimer();
    mbar_wait(&S.dec_mbar[e & 1], par2(e));  // exchange e done, decision e taken
    if (e < m && G.cta == e % G.nblk)
      decide_post(c, S, S.prep[e & 1], S.dec[e & 1], G.rec(e), G.hdr[e], e, lane, K, hist_row);
    if (e == m && G.cta == m % G.nblk && lane == 0) {  // sigma^2 (sampler.py:797-799, 906-908)
      const HP &hp = c.hp;
      const double s2 = __ddiv_rn(__dadd_rn(__dmul_rn(hp.nu, hp.lam), S.tot_sum[0]), chi2);
      *c.sigma2_draw = s2;
      if (hp.update_sigma) *c.sigma2 = s2;
      if (hist_row >= 0) c.sig_hist[hist_row] = hp.update_sigma ? s2 : *c.sigma2;
      *c.iter_dev += 1ull;
      if (c.err_out) *c.err_out = *reinterpret_cast<volatile int *>(c.err);  // with the step's result (host)
    }
    if (e == m && X.fwd) {  // two-level: this forwarder's stage baselines, for the next sweep
      const size_t g = (size_t)xgroup(c, G.cta);
      const unsigned long long *src = &G.hs->xsprev[0][0];
      for (int i = lane; i < kXSets * (int)kXPrevWords; i += 32) c.xssnap[g * kXSets * kXPrevWords + i] = src[i];
      const unsigned long long *cs = &G.hs->csprev[0][0];
      for (int i = lane; i < kCSets * (int)kCSetWords; i += 32) c.cssnap[g * kCSets * kCSetWords + i] = cs[i];
    }
    if (e == m && G.cta == 0) {  // the next sweep's exchange baselines
      if (lane == 0) c.xsnap[0] = xbase + (unsigned long long)(m + 1);
      const unsigned long long *src = &S.xprev[0][0];
      for (int i = lane; i < kXSets * (int)kXPrevWords; i += 32) c.xsnap[1 + i] = src[i];
      const unsigned long long *cs = &S.cprev[0][0];
      for (int i = lane; i < kCSets * (int)kCSetWords; i += 32) c.csnap[i] = cs[i];
    }
    if (e < m && e + kRing < m && lane == 0) issue_tree(e + kRing);  // slot of tree e is free
  }
}

template <int W, bool HIER>
__global__ void __launch_bounds__(kSweepThreads, 1) sweep_kernel(ChainDev c) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SweepSmem &S = *reinterpret_cast<SweepSmem *>(smem_raw);
  Geom G;
  G.m = c.m;
  G.chunk = c.chunk;
  G.size = c.size;
  G.hdr = reinterpret_cast<TreeHdr *>(smem_raw + sizeof(SweepSmem));
  G.ring = smem_raw + sizeof(SweepSmem) + ((((size_t)c.m * sizeof(TreeHdr)) + 15) & ~(size_t)15);
  G.row_bytes = (uint32_t)ring_row_bytes(c.chunk, W == 0);
  G.slot_bytes = (uint32_t)ring_slot_bytes(c.chunk, c.rstride, W == 0);
  G.hs = HIER ? reinterpret_cast<HierSmem *>(G.ring + (((size_t)kRing * G.slot_bytes + 15) & ~(size_t)15)) : nullptr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  G.cta = blockIdx.x;
  G.nblk = gridDim.x;
#ifdef BART_CHUNK_ROT  // diagnostics: CTA c sweeps chunk (c + ROT) % nblk (tools/jobs/r02_rot.sh)
  G.start = (int64_t)((G.cta + BART_CHUNK_ROT) % G.nblk) * G.chunk;
#else
  G.start = (int64_t)G.cta * G.chunk;
#endif
  const int len = (int)((c.n - G.start) < (int64_t)G.chunk ? (c.n - G.start) : (int64_t)G.chunk);
  G.lenp = (uint32_t)((len + 15) & ~15);
  G.nwords = (int)(G.lenp >> 2);

  if (c.propose_in_sweep) {
    // phase 1 for every tree, spread over all warps of the grid (propose.cuh;
    // sampler.py:469-526), then one grid barrier: the step is ONE launch.
    // Scratch: the worker partials' buffer, unused until the first A pass.
    const unsigned long long it = *c.iter_dev;
    const int device_rng = c.propose_in_sweep == 1;
    uint8_t *scratch = reinterpret_cast<uint8_t *>(&S.wsum[0][0]) + (size_t)warp * 512;
    for (int j = G.cta + G.nblk * warp; j < c.m; j += G.nblk * kSweepWarps)
      propose_tree(c, j, it, device_rng, scratch, reinterpret_cast<uint16_t *>(scratch + 128),
                   reinterpret_cast<uint32_t *>(scratch + 384), lane);
    if (device_rng && G.cta == G.nblk - 1 && warp == kSweepWarps - 1 && lane == 0) {
      const uint2 key = make_uint2((uint32_t)c.seed, (uint32_t)(c.seed >> 32));
      *c.rand_chi2 = chi2_draw(c.hp.nu + (double)c.n_total, it, key);
    }
    cooperative_groups::this_grid().sync();
    asm volatile("fence.proxy.async;" ::: "memory");  // records written by generic stores, read by TMA
  }
  for (int i = tid; i < c.m; i += kSweepThreads) G.hdr[i] = c.hdr[i];
  {  // exchange baselines: the words' values when the previous sweep ended
    unsigned long long *dst = &S.xprev[0][0];
    for (int i = tid; i < kXSets * (int)kXPrevWords; i += kSweepThreads) dst[i] = c.xsnap[1 + i];
    unsigned long long *cd = &S.cprev[0][0];
    for (int i = tid; i < kCSets * (int)kCSetWords; i += kSweepThreads) cd[i] = c.csnap[i];
    if (HIER && G.cta == xgroup(c, G.cta)) {  // two-level forwarder: its stage baselines
      const size_t g = (size_t)xgroup(c, G.cta);
      unsigned long long *xs = &G.hs->xsprev[0][0];
      for (int i = tid; i < kXSets * (int)kXPrevWords; i += kSweepThreads) xs[i] = c.xssnap[g * kXSets * kXPrevWords + i];
      unsigned long long *cs = &G.hs->csprev[0][0];
      for (int i = tid; i < kCSets * (int)kCSetWords; i += kSweepThreads) cs[i] = c.cssnap[g * kCSets * kCSetWords + i];
    }
  }
  if (tid == 0) {
    for (int q = 0; q < kRing; ++q) mbar_init(&S.mbar[q]);
    for (int q = 0; q < 2; ++q) {
      mbar_init(&S.cnt_mbar[q], kWorkWarps);
      mbar_init(&S.prep_mbar[q]);
      mbar_init(&S.dec_mbar[q]);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    S.flag_wr = 0;
    S.flag_prune = 0;
    S.flag_t = 0;
  }
  for (int h = tid; h < 256; h += kSweepThreads) S.dlt[h] = 0.f;  // index 0 = padding points
  const unsigned long long xbase = c.xsnap[0];
  __syncthreads();

  if (warp >= kCtrlWarp) {
    DecConst K;
    const double sigma2 = *c.sigma2;  // the sweep uses the old sigma2 (sampler.py:906)
    K.tau = __ddiv_rn(1.0, sigma2);
    K.tau_mu = __ddiv_rn(1.0, __dmul_rn(c.hp.leaf_sd, c.hp.leaf_sd));
    K.prior = __dmul_rn(K.tau_mu, c.hp.leaf_mean);
    K.lm_term = __dmul_rn(__dmul_rn(__dmul_rn(0.5, c.hp.leaf_mean), c.hp.leaf_mean), K.tau_mu);
    long long *tl = (BART_TIMELINE && c.timeline && G.cta == 0 && lane == 0) ? c.timeline : nullptr;
    if (warp == kCtrlWarp)
      control_loop<HIER>(c, S, G, lane, K, xbase, tl);
    else
      helper_loop<HIER>(c, S, G, lane, K, xbase, tl);
  } else {
    long long *tl = (BART_TIMELINE && c.timeline && tid == 0 && G.cta == 0) ? c.timeline : nullptr;
    if constexpr (W == 0)
      stream_worker_loop(c, S, G, tid, warp, lane);
    else
      worker_loop<W>(c, S, G, tid, warp, lane, tl);
  }
}

typedef void (*SweepFn)(ChainDev);
template <bool HIER>
static SweepFn sweep_fn_t(int W) {
  switch (W) {
    case 0: return sweep_kernel<0, HIER>;
    case 1: return sweep_kernel<1, HIER>;
    case 2: return sweep_kernel<2, HIER>;
    case 4: return sweep_kernel<4, HIER>;
    default: return sweep_kernel<8, HIER>;
  }
}
static SweepFn sweep_fn(int W, bool hier = false) { return hier ? sweep_fn_t<true>(W) : sweep_fn_t<false>(W); }

int sweep_launch(const ChainDev &c, size_t smem, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)c.nblk);
  cfg.blockDim = dim3(kSweepThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#ifndef BART_STREAM_PERSIST
#define BART_STREAM_PERSIST 1
#endif
  if (BART_STREAM_PERSIST && c.stream && c.persist_bytes > 0) {
    // stream mode: keep the residuals L2-resident (persisting window) while the
    // cache rows and split columns stream past
    attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[1].val.accessPolicyWindow.base_ptr = c.r;
    attr[1].val.accessPolicyWindow.num_bytes = c.persist_bytes;
    attr[1].val.accessPolicyWindow.hitRatio = 1.0f;
    attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.numAttrs = 2;
  }
  return (int)cudaLaunchKernelEx(&cfg, sweep_fn(c.stream ? 0 : sweep_words_per_thread(c.chunk), c.hier != 0), c);
}

cudaError_t sweep_prepare(size_t smem) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  for (int W : {0, 1, 2, 4, 8})
    for (bool hier : {false, true}) {
      cudaError_t e = cudaFuncSetAttribute(sweep_fn(W, hier), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           optin > (int)smem ? optin : (int)smem);
      if (e != cudaSuccess) return e;
    }
  return cudaSuccess;
}

int sweep_max_ctas(size_t smem, int device, int chunk, bool stream) {
  int per_sm = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_fn(stream ? 0 : sweep_words_per_thread(chunk)), kSweepThreads,
                                                    smem) != cudaSuccess)
    return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return per_sm * sms;
}

}  // namespace bart
