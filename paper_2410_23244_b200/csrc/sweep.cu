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
// 15 worker warps hold the chunk's residuals and leaf indices in REGISTERS
// for the whole sweep (4 points per 32-bit word, W words per thread) and run
// one pass per tree: tree j-1's residual/cache update, tree j's per-leaf f64
// residual sums, and tree j+1's grow refresh and leaf counts (counts one
// tree early).  A 16th warp is the CTA's control warp: it streams each tree's
// n-byte leaf-index row and split column into shared memory with TMA bulk
// copies two trees ahead, publishes the CTA's partials, and decides.
//
// Cross-CTA reduction without a grid barrier or a decider: each CTA adds its
// f64 partial, as an exact 64.64 fixed-point number split into 32-bit limbs,
// into monotonic 64-bit accumulators with red.add (integer addition is
// associative, so the total is bit-identical whatever the arrival order),
// then bumps an arrival counter with red.release.  Every CTA acquires the
// counter, reads the few accumulator words and, holding identical totals,
// takes the same accept decision and leaf draws redundantly.  Count-only
// terms of the ratio and draws are precomputed one tree early, so the
// decision's critical path is one division per leaf.  m+2 exchanges per sweep.
#include "common.cuh"
#include "internal.h"

namespace bart {

constexpr int kRing = 3;  // TMA / stage ring depth: trees j, j+1, j+2

// count-only precomputation for one tree (see prepare())
struct Prep {
  unsigned long long cnt[kSlotsMax];
  double prec[kSlotsMax];  // tau_mu + n * tau
  double zs[kSlotsMax];    // z / sqrt(prec)
  double cadj[kSlotsMax];  // n * adj, the tree's own contribution to the sums
  double prec_l, prec_r, prec_p, zs_p, partial;
};

struct __align__(16) Stage {
  double z[256];
  float old_leaf[256];
  uint8_t slot_node[kSlotsMax];
  double struct_log;
  double log_u;
  double acc_u;
  double pad;
};

struct __align__(16) SweepSmem {
  Stage stage[kRing];
  Prep prep[2];
  double wsum[kSlotsMax][kWorkWarps];
  uint32_t wcnt[kSlotsMax][kWorkWarps];
  unsigned long long prev[kSlotsMax + 1][5];  // accumulator values after the last exchange
  unsigned long long prev_counter;
  double tot_sum[kSlotsMax];
  unsigned long long tot_cnt[kSlotsMax];
  double sums_s[kSlotsMax];   // tree-excluded sums of the decided tree (taps)
  double q_s[kSlotsMax + 1];  // posterior means (leaves, then collapsed parent)
  double v_s[kSlotsMax + 1];  // leaf draws
  float row[256];             // new leaf row
  float dlt[256];             // residual delta by larger-tree heap index
  unsigned long long mbar[kRing];
  int flag_wr, flag_prune, flag_t, acc_e;
};

size_t sweep_smem_bytes(int m, int chunk) {
  size_t b = sizeof(SweepSmem);
  b += ((size_t)m * sizeof(TreeHdr) + 15) & ~(size_t)15;
  b += (size_t)chunk * 2 * kRing;  // leaf-index rows + split columns, ring of 3
  return b;
}

int sweep_words_per_thread(int chunk) {
  const int words = (chunk + 3) / 4;
  for (int w : {1, 2, 4, 8, 16})
    if (w * kWorkers >= words) return w;
  return -1;
}

// ------------------------------------------------------------ async copies
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)) : "memory");
}
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
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------ byte-lane ops
// refresh_leaf_indices on 4 points: L==t -> 2t + (x >= cut) (sampler.py:541-545)
__device__ __forceinline__ uint32_t grow4(uint32_t l, uint32_t x, uint32_t t, uint32_t cut) {
  uint32_t out = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint32_t lb = (l >> (8 * b)) & 0xffu, xb = (x >> (8 * b)) & 0xffu;
    out |= (lb == t ? 2u * t + (xb >= cut ? 1u : 0u) : lb) << (8 * b);
  }
  return out;
}
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

__device__ __forceinline__ float4 update4(float4 r, uint32_t l, const float *dlt) {
  r.x = __fadd_rn(r.x, dlt[l & 0xffu]);
  r.y = __fadd_rn(r.y, dlt[(l >> 8) & 0xffu]);
  r.z = __fadd_rn(r.z, dlt[(l >> 16) & 0xffu]);
  r.w = __fadd_rn(r.w, dlt[l >> 24]);
  return r;
}

struct PassArgs {
  int nwords;
  // tree e-1: residual update and cache write
  bool do_update, wr_prev, prune_prev;
  uint32_t t_prev;
  uint32_t *gLprev;
  // tree e: residual sums over its larger-tree indices (already refreshed)
  const uint8_t *slots_cur;
  int ns_cur;
  // tree e+1: grow refresh of its cache row and point counts
  bool has_next, grow_next;
  const uint32_t *Lnext, *Xnext;
  uint32_t t_next, cut_next;
  const uint8_t *slots_next;
  int ns_next;
};

// One register pass over the chunk.  FIRST: tree e-1's update (residuals
// f32, cache write) and tree e+1's grow refresh.  Every pass: for slot group
// [base, base+NS) the f64 residual sums of tree e and the counts of tree e+1.
// Counts one tree early let the decider precompute every count-only term of
// the acceptance ratio and leaf draws off the critical path.
template <int W, int NS, bool FIRST>
__device__ __forceinline__ void tree_pass(float4 (&r)[W], const uint32_t (&lbp)[W], const uint32_t (&lbc)[W],
                                          uint32_t (&lbn)[W], const PassArgs &A, const float *dlt, SweepSmem &S,
                                          int tid, int warp, int lane, int base) {
  uint32_t sn[8], gn[8];
  double acc[8];
  uint32_t cnt[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    sn[s] = (s < NS && base + s < A.ns_cur) ? A.slots_cur[base + s] : 0xffffu;
    gn[s] = (s < NS && base + s < A.ns_next) ? A.slots_next[base + s] : 0xffffu;
    acc[s] = 0.0;
    cnt[s] = 0u;
  }
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const int w = tid + k * kWorkers;
    if (w < A.nwords) {
      if (FIRST) {
        if (A.do_update) {
          r[k] = update4(r[k], lbp[k], dlt);
          if (A.wr_prev) A.gLprev[w] = A.prune_prev ? collapse4(lbp[k], A.t_prev) : lbp[k];
        }
        if (A.has_next) {
          uint32_t l = A.Lnext[w];
          if (A.grow_next) l = grow4(l, A.Xnext[w], A.t_next, A.cut_next);
          lbn[k] = l;
        }
      }
      const float rv[4] = {r[k].x, r[k].y, r[k].z, r[k].w};
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t h = (lbc[k] >> (8 * b)) & 0xffu, g = (lbn[k] >> (8 * b)) & 0xffu;
        const double v = (double)rv[b];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          if (h == sn[s]) acc[s] = __dadd_rn(acc[s], v);
          if (g == gn[s]) cnt[s] += 1u;
        }
      }
    }
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const double v = warp_sum_f64(acc[s]);
    const uint32_t cc = __reduce_add_sync(0xffffffffu, cnt[s]);
    if (lane == 0) {
      S.wsum[base + s][warp] = v;
      S.wcnt[base + s][warp] = cc;
    }
  }
}

template <int W>
__device__ __forceinline__ void tree_passes(int nsx, float4 (&r)[W], const uint32_t (&lbp)[W],
                                            const uint32_t (&lbc)[W], uint32_t (&lbn)[W], const PassArgs &A,
                                            const float *dlt, SweepSmem &S, int tid, int warp, int lane) {
  // slot-count variants limited to {2, 4, 8} (+ 8-wide follow-up passes) so
  // that the code a tree executes stays inside the instruction cache
  if (nsx <= 2)
    tree_pass<W, 2, true>(r, lbp, lbc, lbn, A, dlt, S, tid, warp, lane, 0);
  else if (nsx <= 4)
    tree_pass<W, 4, true>(r, lbp, lbc, lbn, A, dlt, S, tid, warp, lane, 0);
  else
    tree_pass<W, 8, true>(r, lbp, lbc, lbn, A, dlt, S, tid, warp, lane, 0);
  for (int base = 8; base < nsx; base += 8) tree_pass<W, 8, false>(r, lbp, lbc, lbn, A, dlt, S, tid, warp, lane, base);
}

// ------------------------------------------------------------ exchange
// f64 -> 64.64 fixed point, two's complement, as four 32-bit limbs.  Exact
// for |x| >= 2^-12 with |x| < 2^63 (CTA partials); tinier values round at 2^-64.
__device__ __forceinline__ void to_limbs(double x, unsigned long long (&l)[4]) {
  const long long hi = __double2ll_rd(x);
  const double rem = __dsub_rn(x, (double)hi);  // exact, in [0, 1)
  const unsigned long long lo = __double2ull_rn(__dmul_rn(rem, 0x1.0p64));
  l[0] = lo & 0xffffffffull;
  l[1] = lo >> 32;
  l[2] = (unsigned long long)hi & 0xffffffffull;
  l[3] = (unsigned long long)hi >> 32;
}

// accumulated limb deltas (mod 2^64 each) -> the f64 total (mod 2^128 value)
__device__ __forceinline__ double from_limbs(const unsigned long long (&d)[4]) {
  unsigned long long lo = d[0], hi = 0;
  unsigned long long t = d[1] << 32;
  lo += t;
  hi += (lo < t) + (d[1] >> 32);
  hi += d[2] + (d[3] << 32);
  const bool neg = (long long)hi < 0;
  if (neg) {  // negate the 128-bit value
    lo = ~lo + 1ull;
    hi = ~hi + (lo == 0ull ? 1ull : 0ull);
  }
  const double mag = __dadd_rn(__dmul_rn((double)hi, 0x1.0p64), (double)lo);
  const double v = __dmul_rn(mag, 0x1.0p-64);
  return neg ? -v : v;
}

// Control warp: fold the worker warps' partials of nsx slots (fixed order),
// add them into the accumulators, release the arrival, wait for every CTA,
// and read back the totals (sums, counts) of this exchange.
__device__ __forceinline__ void exchange(const ChainDev &c, SweepSmem &S, int nsx, unsigned long long target,
                                         int lane) {
  for (int s = lane; s < nsx; s += 32) {
    double v = 0.0;
    uint32_t cn = 0;
#pragma unroll
    for (int w = 0; w < kWorkWarps; ++w) {
      v = __dadd_rn(v, S.wsum[s][w]);
      cn += S.wcnt[s][w];
    }
    unsigned long long l[4];
    to_limbs(v, l);
    unsigned long long *a = c.accum + (size_t)s * kAccWords;
#pragma unroll
    for (int k = 0; k < 4; ++k) asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(a + k), "l"(l[k]) : "memory");
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(a + 4), "l"((unsigned long long)cn) : "memory");
  }
  __syncwarp();
  if (lane == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(c.counter) : "memory");
  unsigned long long v;
  do {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(c.counter) : "memory");
  } while (v < target);
  for (int s = lane; s < nsx; s += 32) {
    const unsigned long long *a = c.accum + (size_t)s * kAccWords;
    unsigned long long now[5], d[4];
#pragma unroll
    for (int k = 0; k < 5; ++k) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(now[k]) : "l"(a + k) : "memory");
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      d[k] = now[k] - S.prev[s][k];
      S.prev[s][k] = now[k];
    }
    S.tot_sum[s] = from_limbs(d);
    S.tot_cnt[s] = now[4] - S.prev[s][4];
    S.prev[s][4] = now[4];
  }
  __syncwarp();
}

// ------------------------------------------------------------ decision
struct DecConst {
  double tau, tau_mu, prior, lm_term;  // 1/sigma2, 1/leaf_sd^2, tau_mu*leaf_mean, 0.5*lm*lm*tau_mu
};

__device__ __forceinline__ bool is_child(int h, int t, bool move) { return move && h >= 2 && (h >> 1) == t; }

// Count-only terms of tree j, from the counts gathered one exchange early
// (every CTA's control warp, off the critical path).  Same operations, in the
// same order, as the reference: prec = tau_mu + n*tau, z/sqrt(prec)
// (sampler.py:579-595), adjustment n*adj (sampler.py:575-576), and the count
// part of the ratio (sampler.py:669-684).
__device__ __forceinline__ void prepare(SweepSmem &S, Prep &P, const Stage &st, const TreeHdr hd, int lane,
                                     const DecConst &K) {
  const int kind = hd.kind, t = hd.node, ns = hd.nslots;
  const bool grow = kind == KIND_GROW, move = kind != KIND_NONE;
  for (int j = lane; j < ns; j += 32) {
    const int h = st.slot_node[j];
    const unsigned long long cn = S.tot_cnt[j];
    const float a32 = (grow && is_child(h, t, move)) ? st.old_leaf[t] : st.old_leaf[h];
    const double prec = __dadd_rn(K.tau_mu, __dmul_rn((double)cn, K.tau));
    P.cnt[j] = cn;
    P.cadj[j] = __dmul_rn((double)cn, (double)a32);
    P.prec[j] = prec;
    P.zs[j] = __ddiv_rn(st.z[h], __dsqrt_rn(prec));
  }
  __syncwarp();
  if (move && lane < 2) {
    const unsigned long long nl = P.cnt[hd.slot_l], nr = P.cnt[hd.slot_r];
    const double prec_l = P.prec[hd.slot_l], prec_r = P.prec[hd.slot_r];
    const double prec_p = __dadd_rn(K.tau_mu, __dmul_rn((double)(nl + nr), K.tau));
    if (lane == 0) {
      P.prec_l = prec_l;
      P.prec_r = prec_r;
      P.prec_p = prec_p;
      P.zs_p = __ddiv_rn(st.z[t], __dsqrt_rn(prec_p));
    } else {
      const double q = __ddiv_rn(__dmul_rn(K.tau_mu, prec_p), __dmul_rn(prec_l, prec_r));
      P.partial = __dadd_rn(st.struct_log, __dsub_rn(__dmul_rn(0.5, log(q)), K.lm_term));
    }
  }
  __syncwarp();
}

// Phases 8-10 of tree e, on every CTA's control warp (critical path):
// tree-excluded sums, posterior means (one division each), the acceptance
// test and the residual delta per leaf of the larger tree.
__device__ __forceinline__ void decide(SweepSmem &S, const Prep &P, const Stage &st, const TreeHdr hd, int lane,
                                       const DecConst &K) {
  const int kind = hd.kind, t = hd.node, ns = hd.nslots;
  const bool grow = kind == KIND_GROW, move = kind != KIND_NONE;
  for (int j = lane; j < ns; j += 32) S.sums_s[j] = __dadd_rn(S.tot_sum[j], P.cadj[j]);  // sampler.py:570-576
  __syncwarp();
  const double sl = move ? S.sums_s[hd.slot_l] : 0.0, sr = move ? S.sums_s[hd.slot_r] : 0.0;
  for (int base = 0; base <= ns; base += 32) {
    const int j = base + lane;
    double num = 1.0, den = 1.0, zs = 0.0;
    if (j < ns) {
      num = __dadd_rn(K.prior, __dmul_rn(K.tau, S.sums_s[j]));
      den = P.prec[j];
      zs = P.zs[j];
    } else if (j == ns && move) {  // the collapsed parent: count nl+nr, sum sl+sr
      num = __dadd_rn(K.prior, __dmul_rn(K.tau, __dadd_rn(sl, sr)));
      den = P.prec_p;
      zs = P.zs_p;
    }
    const double q = __ddiv_rn(num, den);
    if (j <= ns) {
      S.q_s[j] = q;
      S.v_s[j] = __dadd_rn(q, zs);
    }
  }
  __syncwarp();
  int acc = 0;
  if (move && lane == 0) {
    // sum part (sampler.py:634-645): mean*mean*prec with the leaf posterior means
    const double ml = S.q_s[hd.slot_l], mr = S.q_s[hd.slot_r], mp = S.q_s[ns];
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
    else if (la < st.log_u - 1e-9)
      acc = 0;
    else if (la > st.log_u + 1e-9)
      acc = 1;
    else
      acc = st.acc_u < exp(la);
  }
  acc = __shfl_sync(0xffffffffu, acc, 0);
  const bool fsmall = move && ((acc != 0) != grow);  // sampler.py:861
  const float v_par = __double2float_rn(S.v_s[ns]);
  // residual delta per leaf of the larger tree (sampler.py:755-760)
  for (int j = lane; j < ns; j += 32) {
    const int h = st.slot_node[j];
    const bool child = is_child(h, t, move);
    const int oi = (grow && child) ? t : h;
    const float nv = (fsmall && child) ? v_par : __double2float_rn(S.v_s[j]);
    S.dlt[h] = __fsub_rn(st.old_leaf[oi], nv);
  }
  if (lane == 0) {
    S.flag_wr = acc;
    S.flag_prune = acc && !grow;
    S.flag_t = t;
    S.acc_e = acc;
  }
  __syncwarp();
}

// CTA 0's bookkeeping for tree e, off the critical path: accept flag,
// structure write, the new leaf row (final leaves keep their draw, other
// slots a signed zero; sampler.py:836-848, 868-870) and the parity taps.
__device__ __forceinline__ void decide_post(const ChainDev &c, SweepSmem &S, const Prep &P, const Stage &st,
                                         const TreeHdr hd, int e, int lane, const DecConst &K) {
  const int size = c.size, half = c.half;
  const int kind = hd.kind, t = hd.node, ns = hd.nslots;
  const bool grow = kind == KIND_GROW, move = kind != KIND_NONE;
  const int acc = S.acc_e;
  const bool fsmall = move && ((acc != 0) != grow);
  const float v_par = __double2float_rn(S.v_s[ns]);
  if (lane == 0) {
    c.accepted[e] = (uint8_t)acc;
    if (acc) {
      c.axis[(size_t)e * half + t] = grow ? hd.axis : (uint16_t)0;
      c.cut[(size_t)e * half + t] = grow ? hd.cut : (uint8_t)0;
    }
  }
  for (int h = lane; h < size; h += 32) {
    float z0;
    if (K.prior == 0.0) {
      z0 = copysignf(0.0f, (float)st.z[h]);  // 0 + z/sqrt(tau_mu) has the sign of z
    } else {
      const double v0 = __dadd_rn(__ddiv_rn(K.prior, K.tau_mu), __ddiv_rn(st.z[h], __dsqrt_rn(K.tau_mu)));
      z0 = __double2float_rn(__dmul_rn(v0, 0.0));
    }
    S.row[h] = z0;
  }
  __syncwarp();
  for (int j = lane; j < ns; j += 32) {
    const int h = st.slot_node[j];
    if (!(fsmall && is_child(h, t, move))) S.row[h] = __double2float_rn(S.v_s[j]);
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
      const int h = st.slot_node[j];
      c.tap_counts[(size_t)e * size + h] = (int64_t)P.cnt[j];
      c.tap_sums[(size_t)e * size + h] = S.sums_s[j];
    }
  }
  __syncwarp();
}

// ------------------------------------------------------------ the kernel
__device__ __forceinline__ void stage_load(const ChainDev &c, Stage &st, int j, int lane) {
  const int size = c.size;
  for (int h = lane; h < size; h += 32) {
    cp_async8(&st.z[h], c.rand_z + (size_t)j * size + h);
    cp_async4(&st.old_leaf[h], c.leaf + (size_t)j * size + h);
  }
  cp_async4(reinterpret_cast<uint32_t *>(st.slot_node) + lane,
            reinterpret_cast<const uint32_t *>(c.moves[j].slot_node) + lane);
  if (lane == 0) {
    cp_async8(&st.struct_log, &c.moves[j].struct_log);
    cp_async8(&st.log_u, &c.moves[j].log_u);
    cp_async8(&st.acc_u, c.rand_acc + j);
  }
  cp_async_commit();
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct Geom {
  int m, chunk, nwords, cta, nblk;
  int64_t start;
  uint32_t lenp;
  uint8_t *ring;
  TreeHdr *hdr;
};

// Worker warps: the register-resident point chunk, one pass per exchange.
template <int W>
__device__ __forceinline__ void worker_loop(const ChainDev &c, SweepSmem &S, const Geom &G, int tid, int warp, int lane,
                                            long long *tl) {
  float4 r[W];
  uint32_t lbp[W], lbc[W], lbn[W];  // larger-tree indices of trees e-1, e, e+1
  const float4 *gr4 = reinterpret_cast<const float4 *>(c.r + G.start);
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const int w = tid + k * kWorkers;
    r[k] = w < G.nwords ? gr4[w] : make_float4(0.f, 0.f, 0.f, 0.f);
    lbp[k] = lbc[k] = lbn[k] = 0u;
  }
  __syncthreads();  // prologue barrier (control warp: ring and stages 0, 1 issued)
  const int m = G.m;
  for (int e = -1; e <= m; ++e) {
    const bool has_cur = e >= 0 && e < m, has_next = e + 1 < m;
    const int ns_cur = has_cur ? G.hdr[e].nslots : 0, ns_next = has_next ? G.hdr[e + 1].nslots : 0;
    if (tl && e >= 0) tl[(size_t)e * 8 + 0] = clock64();
    PassArgs A;
    A.nwords = G.nwords;
    A.do_update = e > 0;
    A.wr_prev = e > 0 && S.flag_wr;
    A.prune_prev = e > 0 && S.flag_prune;
    A.t_prev = (uint32_t)S.flag_t;
    A.gLprev = reinterpret_cast<uint32_t *>(c.L + (size_t)(e > 0 ? e - 1 : 0) * c.n_pad + G.start);
    A.ns_cur = ns_cur;
    A.slots_cur = has_cur ? S.stage[e % kRing].slot_node : S.stage[0].slot_node;
    A.has_next = has_next;
    A.ns_next = ns_next;
    A.slots_next = A.slots_cur;
    if (has_next) {
      const TreeHdr hn = G.hdr[e + 1];
      const uint8_t *slot = G.ring + (size_t)((e + 1) % kRing) * 2 * G.chunk;
      A.Lnext = reinterpret_cast<const uint32_t *>(slot);
      A.Xnext = reinterpret_cast<const uint32_t *>(slot + G.chunk);
      A.grow_next = hn.kind == KIND_GROW;
      A.t_next = hn.node;
      A.cut_next = hn.cut;
      A.slots_next = S.stage[(e + 1) % kRing].slot_node;
      mbar_wait(&S.mbar[(e + 1) % kRing], (uint32_t)(((e + 1) / kRing) & 1));
    }
    if (tl && e >= 0) tl[(size_t)e * 8 + 1] = clock64();
    if (e < m) {
      const int nsx = ns_cur > ns_next ? ns_cur : ns_next;
      tree_passes<W>(nsx, r, lbp, lbc, lbn, A, S.dlt, S, tid, warp, lane);
    } else {  // tree m-1's update, residual write-back, sum of squares (sampler.py:790-794)
      float4 *out = reinterpret_cast<float4 *>(c.r + G.start);
      double ss = 0.0;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const int w = tid + k * kWorkers;
        if (w < G.nwords) {
          r[k] = update4(r[k], lbp[k], S.dlt);
          if (A.wr_prev) A.gLprev[w] = A.prune_prev ? collapse4(lbp[k], A.t_prev) : lbp[k];
          out[w] = r[k];
          const double a = r[k].x, b = r[k].y, cc = r[k].z, d = r[k].w;
          ss = __dadd_rn(ss, __dmul_rn(a, a));
          ss = __dadd_rn(ss, __dmul_rn(b, b));
          ss = __dadd_rn(ss, __dmul_rn(cc, cc));
          ss = __dadd_rn(ss, __dmul_rn(d, d));
        }
      }
      const double v = warp_sum_f64(ss);
      if (lane == 0) {
        S.wsum[0][warp] = v;
        S.wcnt[0][warp] = 0u;
      }
    }
#pragma unroll
    for (int k = 0; k < W; ++k) {  // rotate: e-1 <- e <- e+1
      lbp[k] = lbc[k];
      lbc[k] = lbn[k];
    }
    if (tl && e >= 0) tl[(size_t)e * 8 + 2] = clock64();
    fence_proxy_async();
    __syncthreads();                // partials complete
    named_sync(1, kSweepThreads);   // decision of tree e installed (S.dlt, flags)
    if (tl && e >= 0) tl[(size_t)e * 8 + 3] = clock64();
  }
}

// Control warp: TMA/stage streaming, exchange, decision, bookkeeping.
__device__ __forceinline__ void control_loop(const ChainDev &c, SweepSmem &S, const Geom &G, int lane,
                                             const DecConst &K, long long *dtl) {
  const int m = G.m;
  auto issue_tree = [&](int j) {  // lane 0
    const TreeHdr hd = G.hdr[j];
    unsigned long long *mb = &S.mbar[j % kRing];
    uint8_t *dst = G.ring + (size_t)(j % kRing) * 2 * G.chunk;
    const bool g = hd.kind == KIND_GROW;
    fence_proxy_async();
    mbar_expect(mb, g ? 2u * G.lenp : G.lenp);
    bulk_g2s(dst, c.L + (size_t)j * c.n_pad + G.start, G.lenp, mb);
    if (g) bulk_g2s(dst + G.chunk, c.Xt + (size_t)hd.axis * c.n_pad + G.start, G.lenp, mb);
  };
  // baseline of the monotonic accumulators: CTA 0 saved their values at the
  // end of the previous sweep (the live words may already be moving)
  for (int i = lane; i < (kSlotsMax + 1) * 5; i += 32) S.prev[i / 5][i % 5] = c.accum_base[i];
  unsigned long long counter = c.accum_base[(kSlotsMax + 1) * 5];
  for (int j = 0; j < 2 && j < m; ++j) {
    if (lane == 0) issue_tree(j);
    stage_load(c, S.stage[j], j, lane);
  }
  cp_async_wait_all();
  __syncthreads();  // prologue barrier

  for (int e = -1; e <= m; ++e) {
    const bool has_cur = e >= 0 && e < m, has_next = e + 1 < m;
    const TreeHdr hc = has_cur ? G.hdr[e] : TreeHdr{};
    const TreeHdr hn = has_next ? G.hdr[e + 1] : TreeHdr{};
    const int nsx = e == m ? 1 : (hc.nslots > hn.nslots ? hc.nslots : hn.nslots);
    // two trees ahead: ring slot / stage (e+2)%3 held tree e-1, whose last
    // users (pass e-2, decide_post(e-1)) are done
    if (e >= 0 && e + 2 < m) {
      if (lane == 0) issue_tree(e + 2);
      stage_load(c, S.stage[(e + 2) % kRing], e + 2, lane);
    }
    __syncthreads();  // worker partials complete
    if (dtl && e >= 0) dtl[(size_t)e * 8 + 0] = clock64();
    counter += (unsigned long long)G.nblk;
    exchange(c, S, nsx, counter, lane);
    if (dtl && e >= 0) dtl[(size_t)e * 8 + 1] = clock64();
    if (has_cur) decide(S, S.prep[e & 1], S.stage[e % kRing], hc, lane, K);
    if (dtl && e >= 0) dtl[(size_t)e * 8 + 2] = clock64();
    if (e + 1 < m) cp_async_wait_all();  // stage e+2 before pass e+1 reads its leaf list
    named_arrive(1, kSweepThreads);       // workers may start the next pass
    if (has_next) prepare(S, S.prep[(e + 1) & 1], S.stage[(e + 1) % kRing], hn, lane, K);
    if (G.cta == 0) {
      if (has_cur) decide_post(c, S, S.prep[e & 1], S.stage[e % kRing], hc, e, lane, K);
      if (e == m && lane == 0) {  // sigma^2 (sampler.py:797-799, 906-908)
        const HP &hp = c.hp;
        const double s2 = __ddiv_rn(__dadd_rn(__dmul_rn(hp.nu, hp.lam), S.tot_sum[0]), *c.rand_chi2);
        *c.sigma2_draw = s2;
        if (hp.update_sigma) *c.sigma2 = s2;
        *c.iter_dev += 1ull;
      }
      if (e == m) {  // baseline for the next sweep: every accumulator's final value
        __syncwarp();
        for (int i = lane; i < (kSlotsMax + 1) * 5; i += 32) c.accum_base[i] = S.prev[i / 5][i % 5];
        if (lane == 0) c.accum_base[(kSlotsMax + 1) * 5] = counter;
      }
    }
    if (dtl && e >= 0) dtl[(size_t)e * 8 + 3] = clock64();
    if (c.trace && lane == 0 && e >= 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      c.trace[((size_t)e * G.nblk + G.cta) * 2 + 1] = (long long)g;
    }
  }
}

template <int W>
__global__ void __launch_bounds__(kSweepThreads, 1) sweep_kernel(ChainDev c) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SweepSmem &S = *reinterpret_cast<SweepSmem *>(smem_raw);
  Geom G;
  G.m = c.m;
  G.chunk = c.chunk;
  G.hdr = reinterpret_cast<TreeHdr *>(smem_raw + sizeof(SweepSmem));
  // ring slot q: leaf-index row at ring + q*2*chunk, split column right after it
  G.ring = smem_raw + sizeof(SweepSmem) + ((((size_t)c.m * sizeof(TreeHdr)) + 15) & ~(size_t)15);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  G.cta = blockIdx.x;
  G.nblk = gridDim.x;
  G.start = (int64_t)G.cta * G.chunk;
  const int len = (int)((c.n - G.start) < (int64_t)G.chunk ? (c.n - G.start) : (int64_t)G.chunk);
  G.lenp = (uint32_t)((len + 15) & ~15);
  G.nwords = (int)(G.lenp >> 2);

  for (int i = tid; i < c.m; i += kSweepThreads) G.hdr[i] = c.hdr[i];
  if (tid == 0) {
    for (int q = 0; q < kRing; ++q) mbar_init(&S.mbar[q]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int h = tid; h < 256; h += kSweepThreads) S.dlt[h] = 0.f;  // index 0 = padding points
  __syncthreads();

  if (warp == kWorkWarps) {
    DecConst K;
    const double sigma2 = *c.sigma2;  // the sweep uses the old sigma2 (sampler.py:906)
    K.tau = __ddiv_rn(1.0, sigma2);
    K.tau_mu = __ddiv_rn(1.0, __dmul_rn(c.hp.leaf_sd, c.hp.leaf_sd));
    K.prior = __dmul_rn(K.tau_mu, c.hp.leaf_mean);
    K.lm_term = __dmul_rn(__dmul_rn(__dmul_rn(0.5, c.hp.leaf_mean), c.hp.leaf_mean), K.tau_mu);
    long long *dtl = (c.timeline && G.cta == 0 && lane == 0) ? c.timeline + (size_t)2 * (c.m + 1) * 8 : nullptr;
    control_loop(c, S, G, lane, K, dtl);
  } else {
    long long *tl = nullptr;
    if (c.timeline && tid == 0 && (G.cta == 0 || G.cta == G.nblk - 1))
      tl = c.timeline + (size_t)(G.cta == 0 ? 0 : 1) * (c.m + 1) * 8;
    worker_loop<W>(c, S, G, tid, warp, lane, tl);
  }
}

typedef void (*SweepFn)(ChainDev);
static SweepFn sweep_fn(int W) {
  switch (W) {
    case 1: return sweep_kernel<1>;
    case 2: return sweep_kernel<2>;
    case 4: return sweep_kernel<4>;
    case 8: return sweep_kernel<8>;
    default: return sweep_kernel<16>;
  }
}

int sweep_launch(const ChainDev &c, size_t smem, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)c.nblk);
  cfg.blockDim = dim3(kSweepThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, sweep_fn(sweep_words_per_thread(c.chunk)), c);
}

cudaError_t sweep_prepare(size_t smem) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  for (int W : {1, 2, 4, 8, 16}) {
    cudaError_t e = cudaFuncSetAttribute(sweep_fn(W), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         optin > (int)smem ? optin : (int)smem);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int sweep_max_ctas(size_t smem, int device, int chunk) {
  int per_sm = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_fn(sweep_words_per_thread(chunk)), kSweepThreads,
                                                    smem) != cudaSuccess)
    return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return per_sm * sms;
}

}  // namespace bart
