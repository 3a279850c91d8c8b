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
// Design: one CTA per SM owns a contiguous chunk of points.
// Its residuals live in shared memory for the whole sweep; per tree it
// streams only the tree's n-byte leaf-index row and (for GROW moves) the
// split column of X, prefetched one tree ahead with TMA bulk copies.  One
// pass over the chunk applies tree j-1's residual update and, on the updated
// residuals, builds tree j's per-leaf (count, f64 sum) histogram in
// registers.  CTA partials are exchanged through a tagged low-latency
// mailbox in L2 (one 64-bit store per word, tag in the high half: no
// fences, no grid barrier); every CTA reduces all partials in a fixed order
// and so computes bit-identical totals, the same accept decision and the
// same leaf draws redundantly.  One exchange per tree, m+1 per iteration.
#include "common.cuh"
#include "internal.h"

namespace bart {

struct __align__(16) Stage {
  double z[256];
  float old_leaf[256];
  uint8_t slot_node[kSlotsMax];
  double struct_log;
  double acc_u;
};

struct __align__(16) SweepSmem {
  Stage stage[2];
  double wsum[kSlotsMax][kSweepWarps];
  uint32_t wcnt[kSlotsMax][kSweepWarps];
  double tot_sum[kSlotsMax];
  unsigned long long tot_cnt[kSlotsMax];
  unsigned long long cnt_h[256];
  double sums_h[256];
  float dlt[256];
  float new_leaf[256];
  uint8_t bigleaf[256];
  unsigned long long mbar[2];
  int flag_wr, flag_prune, flag_t, pad;
};

size_t sweep_smem_bytes(int m, int chunk) {
  size_t b = sizeof(SweepSmem);
  b += ((size_t)m * sizeof(TreeHdr) + 15) & ~(size_t)15;
  b += (size_t)chunk * 4;  // residuals
  b += (size_t)chunk * 3;  // leaf-index ring (tree j-1, j, j+1)
  b += (size_t)chunk * 2;  // split-column double buffer
  return b;
}

// ------------------------------------------------------------ async copies
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
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
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------ byte-lane ops
// refresh_leaf_indices on 4 points: L==t -> 2t + (x >= cut) (sampler.py:541-545)
__device__ __forceinline__ uint32_t grow4(uint32_t l, uint32_t x, uint32_t t, uint32_t cut) {
  uint32_t out = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint32_t lb = (l >> (8 * b)) & 0xffu, xb = (x >> (8 * b)) & 0xffu;
    const uint32_t nb = lb == t ? 2u * t + (xb >= cut ? 1u : 0u) : lb;
    out |= nb << (8 * b);
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

// per-leaf histogram of 4 points into NS register slots
template <int NS>
__device__ __forceinline__ void accumulate4(uint32_t l, const float4 &r, const uint32_t (&sn)[8], double (&acc)[8],
                                            uint32_t (&cnt)[8]) {
  const float rv[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint32_t h = (l >> (8 * b)) & 0xffu;
    const double v = (double)rv[b];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (h == sn[s]) {
        acc[s] = __dadd_rn(acc[s], v);
        cnt[s] += 1u;
      }
    }
  }
}

template <int NS>
__device__ __forceinline__ void flush_partials(SweepSmem &S, int base, const double (&acc)[8],
                                               const uint32_t (&cnt)[8], int warp, int lane) {
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

struct PassCtx {
  int tid, warp, lane, nwords;
  float4 *r4;
  // previous tree (update)
  bool do_update, wr_prev, prune_prev;
  uint32_t t_prev;
  const uint32_t *Lprev;
  uint32_t *gLprev;
  const float *dlt;
  // current tree (histogram)
  uint32_t *Lcur;
  const uint32_t *Xc;
  bool grow;
  uint32_t t, cut;
  const uint8_t *slots;
};

// One pass: tree j-1's residual/cache update fused with tree j's grow refresh
// and the first NS slots of its histogram.
template <int NS>
__device__ __noinline__ void pass_first(const PassCtx &P, SweepSmem &S) {
  uint32_t sn[8];
  double acc[8];
  uint32_t cnt[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    sn[s] = s < NS ? P.slots[s] : 0xffffu;
    acc[s] = 0.0;
    cnt[s] = 0u;
  }
  for (int w = P.tid; w < P.nwords; w += kSweepThreads) {
    float4 r = P.r4[w];
    if (P.do_update) {
      const uint32_t lp = P.Lprev[w];
      r.x = __fadd_rn(r.x, P.dlt[lp & 0xffu]);
      r.y = __fadd_rn(r.y, P.dlt[(lp >> 8) & 0xffu]);
      r.z = __fadd_rn(r.z, P.dlt[(lp >> 16) & 0xffu]);
      r.w = __fadd_rn(r.w, P.dlt[lp >> 24]);
      P.r4[w] = r;
      if (P.wr_prev) P.gLprev[w] = P.prune_prev ? collapse4(lp, P.t_prev) : lp;
    }
    uint32_t l = P.Lcur[w];
    if (P.grow) {
      l = grow4(l, P.Xc[w], P.t, P.cut);
      P.Lcur[w] = l;
    }
    accumulate4<NS>(l, r, sn, acc, cnt);
  }
  flush_partials<NS>(S, 0, acc, cnt, P.warp, P.lane);
}

// further histogram slots (trees with more than 8 leaves)
template <int NS>
__device__ __noinline__ void pass_more(const PassCtx &P, SweepSmem &S, int base) {
  uint32_t sn[8];
  double acc[8];
  uint32_t cnt[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    sn[s] = s < NS ? P.slots[base + s] : 0xffffu;
    acc[s] = 0.0;
    cnt[s] = 0u;
  }
  for (int w = P.tid; w < P.nwords; w += kSweepThreads) accumulate4<NS>(P.Lcur[w], P.r4[w], sn, acc, cnt);
  flush_partials<NS>(S, base, acc, cnt, P.warp, P.lane);
}

// last pass: tree m-1's update, write-back, and sum of squares (sampler.py:790-794)
__device__ __noinline__ void pass_last(const PassCtx &P, SweepSmem &S, float4 *gr) {
  double ss = 0.0;
  for (int w = P.tid; w < P.nwords; w += kSweepThreads) {
    float4 r = P.r4[w];
    if (P.do_update) {
      const uint32_t lp = P.Lprev[w];
      r.x = __fadd_rn(r.x, P.dlt[lp & 0xffu]);
      r.y = __fadd_rn(r.y, P.dlt[(lp >> 8) & 0xffu]);
      r.z = __fadd_rn(r.z, P.dlt[(lp >> 16) & 0xffu]);
      r.w = __fadd_rn(r.w, P.dlt[lp >> 24]);
      if (P.wr_prev) P.gLprev[w] = P.prune_prev ? collapse4(lp, P.t_prev) : lp;
    }
    gr[w] = r;
    const double a = r.x, b = r.y, c = r.z, d = r.w;
    ss = __dadd_rn(ss, __dmul_rn(a, a));
    ss = __dadd_rn(ss, __dmul_rn(b, b));
    ss = __dadd_rn(ss, __dmul_rn(c, c));
    ss = __dadd_rn(ss, __dmul_rn(d, d));
  }
  const double v = warp_sum_f64(ss);
  if (P.lane == 0) {
    S.wsum[0][P.warp] = v;
    S.wcnt[0][P.warp] = 0u;
  }
}

// ------------------------------------------------------------ exchange
__device__ __forceinline__ void gather_slot(const unsigned long long *box, int nblk, uint32_t tag, int lane,
                                            double &tot, unsigned long long &ctot) {
  unsigned long long a[kGatherUnroll], b[kGatherUnroll], d[kGatherUnroll];
  bool ok;
  do {
    ok = true;
#pragma unroll
    for (int k = 0; k < kGatherUnroll; ++k) {
      const int i = lane + 32 * k;
      if (i < nblk) {
        ll_load(box + (size_t)i * 4, a[k], b[k], d[k]);
        ok = ok && (uint32_t)(a[k] >> 32) == tag && (uint32_t)(b[k] >> 32) == tag && (uint32_t)(d[k] >> 32) == tag;
      }
    }
  } while (!__all_sync(0xffffffffu, ok));
  double s = 0.0;
  unsigned long long cn = 0;
#pragma unroll
  for (int k = 0; k < kGatherUnroll; ++k) {
    const int i = lane + 32 * k;
    if (i < nblk) {
      cn += a[k] & 0xffffffffull;
      s = __dadd_rn(s, __longlong_as_double((long long)((d[k] << 32) | (b[k] & 0xffffffffull))));
    }
  }
  s = warp_sum_f64(s);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) cn += __shfl_down_sync(0xffffffffu, cn, off);
  tot = s;
  ctot = cn;
}

// ------------------------------------------------------------ decision
// Phases 8-10 for tree e, executed redundantly by warp 0 of every CTA.
__device__ __noinline__ void decide(const ChainDev &c, SweepSmem &S, const TreeHdr hd, int e, int lane,
                                    double sigma2) {
  const Stage &st = S.stage[e & 1];
  const int size = c.size, half = c.half;
  const int kind = hd.kind, t = hd.node, ns = hd.nslots;
  const bool grow = kind == KIND_GROW;
  for (int h = lane; h < size; h += 32) {
    S.cnt_h[h] = 0ull;
    S.sums_h[h] = 0.0;
    S.bigleaf[h] = 0;
  }
  __syncwarp();
  for (int s = lane; s < ns; s += 32) {
    const int h = st.slot_node[s];
    S.cnt_h[h] = S.tot_cnt[s];
    S.sums_h[h] = S.tot_sum[s];
    S.bigleaf[h] = 1;
  }
  __syncwarp();
  // sums = raw + counts * adj, grown children inherit the split leaf's value (sampler.py:570-576)
  for (int h = lane; h < size; h += 32) {
    float a32 = st.old_leaf[h];
    if (grow && h >= 2 && (h >> 1) == t) a32 = st.old_leaf[t];
    S.sums_h[h] = __dadd_rn(S.sums_h[h], __dmul_rn((double)S.cnt_h[h], (double)a32));
  }
  __syncwarp();
  const HP &hp = c.hp;
  const double tau = __ddiv_rn(1.0, sigma2);
  const double tau_mu = __ddiv_rn(1.0, __dmul_rn(hp.leaf_sd, hp.leaf_sd));
  int acc = 0;
  if (lane == 0 && kind != KIND_NONE) {
    const unsigned long long nl = S.cnt_h[2 * t], nr = S.cnt_h[2 * t + 1];
    const double sl = S.sums_h[2 * t], sr = S.sums_h[2 * t + 1];
    // count part (sampler.py:669-684)
    const double prec_l = __dadd_rn(tau_mu, __dmul_rn((double)nl, tau));
    const double prec_r = __dadd_rn(tau_mu, __dmul_rn((double)nr, tau));
    const double prec_p = __dadd_rn(tau_mu, __dmul_rn((double)(nl + nr), tau));
    const double q = __ddiv_rn(__dmul_rn(tau_mu, prec_p), __dmul_rn(prec_l, prec_r));
    const double count_part =
        __dsub_rn(__dmul_rn(0.5, log(q)), __dmul_rn(__dmul_rn(__dmul_rn(0.5, hp.leaf_mean), hp.leaf_mean), tau_mu));
    const double partial = __dadd_rn(st.struct_log, count_part);
    // sum part (sampler.py:634-645)
    const double shift = __dmul_rn(tau_mu, hp.leaf_mean);
    double tl, tr, tp;
    {
      const double m_ = __ddiv_rn(__dadd_rn(shift, __dmul_rn(tau, sl)), prec_l);
      tl = __dmul_rn(__dmul_rn(m_, m_), prec_l);
    }
    {
      const double m_ = __ddiv_rn(__dadd_rn(shift, __dmul_rn(tau, sr)), prec_r);
      tr = __dmul_rn(__dmul_rn(m_, m_), prec_r);
    }
    {
      const double m_ = __ddiv_rn(__dadd_rn(shift, __dmul_rn(tau, __dadd_rn(sl, sr))), prec_p);
      tp = __dmul_rn(__dmul_rn(m_, m_), prec_p);
    }
    const double sum_part = __dmul_rn(0.5, __dsub_rn(__dadd_rn(tl, tr), tp));
    const double log_alpha = __dmul_rn(grow ? 1.0 : -1.0, __dadd_rn(partial, sum_part));
    acc = st.acc_u < exp(log_alpha < 0.0 ? log_alpha : 0.0);  // sampler.py:833-834
  }
  acc = __shfl_sync(0xffffffffu, acc, 0);
  const bool fsmall = kind != KIND_NONE && ((acc != 0) != grow);  // sampler.py:861
  if (c.taps && blockIdx.x == 0) {
    for (int h = lane; h < size; h += 32) {
      c.tap_counts[(size_t)e * size + h] = (int64_t)S.cnt_h[h];
      c.tap_sums[(size_t)e * size + h] = S.sums_h[h];
    }
  }
  __syncwarp();
  if (fsmall && lane == 0) {  // sampler.py:862-866
    S.cnt_h[t] = S.cnt_h[2 * t] + S.cnt_h[2 * t + 1];
    S.cnt_h[2 * t] = S.cnt_h[2 * t + 1] = 0ull;
    S.sums_h[t] = __dadd_rn(S.sums_h[2 * t], S.sums_h[2 * t + 1]);
    S.sums_h[2 * t] = S.sums_h[2 * t + 1] = 0.0;
  }
  __syncwarp();
  // leaf redraw over every heap slot, masked by the final tree's leaves (sampler.py:868-870)
  const double prior = __dmul_rn(tau_mu, hp.leaf_mean);
  for (int h = lane; h < size; h += 32) {
    const bool leaf_f = fsmall ? ((S.bigleaf[h] && (h >> 1) != t) || h == t) : (S.bigleaf[h] != 0);
    const double prec = __dadd_rn(tau_mu, __dmul_rn((double)S.cnt_h[h], tau));
    const double mean = __ddiv_rn(__dadd_rn(prior, __dmul_rn(tau, S.sums_h[h])), prec);
    const double v = __dadd_rn(mean, __ddiv_rn(st.z[h], __dsqrt_rn(prec)));
    S.new_leaf[h] = __double2float_rn(__dmul_rn(v, leaf_f ? 1.0 : 0.0));
  }
  __syncwarp();
  // residual delta per larger-tree index (sampler.py:755-760)
  for (int h = lane; h < size; h += 32) {
    const int coll = (h >> 1) == t ? t : h;
    const int oi = grow ? coll : h;
    const int fi = fsmall ? coll : h;
    S.dlt[h] = __fsub_rn(st.old_leaf[oi], S.new_leaf[fi]);
    if (blockIdx.x == 0) c.leaf[(size_t)e * size + h] = S.new_leaf[h];
  }
  if (lane == 0) {
    S.flag_wr = acc;
    S.flag_prune = acc && !grow;
    S.flag_t = t;
    if (blockIdx.x == 0) {
      c.accepted[e] = (uint8_t)acc;
      if (acc) {  // structure write (sampler.py:836-848)
        c.axis[(size_t)e * half + t] = grow ? hd.axis : (uint16_t)0;
        c.cut[(size_t)e * half + t] = grow ? hd.cut : (uint8_t)0;
      }
    }
  }
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
    cp_async8(&st.acc_u, c.rand_acc + j);
  }
  cp_async_commit();
}

__global__ void __launch_bounds__(kSweepThreads, 1) sweep_kernel(ChainDev c) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SweepSmem &S = *reinterpret_cast<SweepSmem *>(smem_raw);
  TreeHdr *s_hdr = reinterpret_cast<TreeHdr *>(smem_raw + sizeof(SweepSmem));
  const int m = c.m, chunk = c.chunk;
  unsigned char *dyn = smem_raw + sizeof(SweepSmem) + ((((size_t)m * sizeof(TreeHdr)) + 15) & ~(size_t)15);
  float *s_r = reinterpret_cast<float *>(dyn);
  uint8_t *s_L[3] = {dyn + (size_t)chunk * 4, dyn + (size_t)chunk * 5, dyn + (size_t)chunk * 6};
  uint8_t *s_X[2] = {dyn + (size_t)chunk * 7, dyn + (size_t)chunk * 8};

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cta = blockIdx.x, nblk = gridDim.x;
  const int64_t start = (int64_t)cta * chunk;
  const int len = (int)((c.n - start) < (int64_t)chunk ? (c.n - start) : (int64_t)chunk);
  const uint32_t lenp = (uint32_t)((len + 15) & ~15);
  const int nwords = (int)(lenp >> 2);
  const uint32_t base_tag = *reinterpret_cast<volatile uint32_t *>(c.tagbase);
  const double sigma2 = *c.sigma2;

  // ---- prologue
  for (int i = tid; i < m; i += kSweepThreads) s_hdr[i] = c.hdr[i];
  float4 *r4 = reinterpret_cast<float4 *>(s_r);
  const float4 *gr4 = reinterpret_cast<const float4 *>(c.r + start);
  for (int w = tid; w < nwords; w += kSweepThreads) r4[w] = gr4[w];
  if (tid == 0) {
    mbar_init(&S.mbar[0]);
    mbar_init(&S.mbar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kSweepWarps - 1) {
    stage_load(c, S.stage[0], 0, lane);
    cp_async_wait_all();
  }
  __syncthreads();

  auto issue_tree = [&](int j) {
    const TreeHdr hd = s_hdr[j];
    unsigned long long *mb = &S.mbar[j & 1];
    const bool g = hd.kind == KIND_GROW;
    fence_proxy_async();
    mbar_expect(mb, g ? 2u * lenp : lenp);
    bulk_g2s(s_L[j % 3], c.L + (size_t)j * c.n_pad + start, lenp, mb);
    if (g) bulk_g2s(s_X[j & 1], c.Xt + (size_t)hd.axis * c.n_pad + start, lenp, mb);
  };
  if (tid == 0) issue_tree(0);

  for (int e = 0; e <= m; ++e) {
    const bool has_tree = e < m;
    if (tid == 0 && e + 1 < m) issue_tree(e + 1);
    if (warp == kSweepWarps - 1 && e + 1 < m) stage_load(c, S.stage[(e + 1) & 1], e + 1, lane);

    PassCtx P;
    P.tid = tid;
    P.warp = warp;
    P.lane = lane;
    P.nwords = nwords;
    P.r4 = r4;
    P.do_update = e > 0;
    P.wr_prev = e > 0 && S.flag_wr;
    P.prune_prev = e > 0 && S.flag_prune;
    P.t_prev = (uint32_t)S.flag_t;
    P.Lprev = reinterpret_cast<const uint32_t *>(s_L[(e + 2) % 3]);
    P.gLprev = reinterpret_cast<uint32_t *>(c.L + (size_t)(e > 0 ? e - 1 : 0) * c.n_pad + start);
    P.dlt = S.dlt;

    TreeHdr hd = {};
    int ns = 1;
    if (has_tree) {
      hd = s_hdr[e];
      ns = hd.nslots;
      P.Lcur = reinterpret_cast<uint32_t *>(s_L[e % 3]);
      P.Xc = reinterpret_cast<const uint32_t *>(s_X[e & 1]);
      P.grow = hd.kind == KIND_GROW;
      P.t = hd.node;
      P.cut = hd.cut;
      P.slots = S.stage[e & 1].slot_node;
      mbar_wait(&S.mbar[e & 1], (uint32_t)((e >> 1) & 1));
      switch (ns < 8 ? ns : 8) {
        case 1: pass_first<1>(P, S); break;
        case 2: pass_first<2>(P, S); break;
        case 3: pass_first<3>(P, S); break;
        case 4: pass_first<4>(P, S); break;
        case 5: pass_first<5>(P, S); break;
        case 6: pass_first<6>(P, S); break;
        case 7: pass_first<7>(P, S); break;
        default: pass_first<8>(P, S); break;
      }
      for (int base = 8; base < ns; base += 8) {
        switch (ns - base < 8 ? ns - base : 8) {
          case 1: pass_more<1>(P, S, base); break;
          case 2: pass_more<2>(P, S, base); break;
          case 3: pass_more<3>(P, S, base); break;
          case 4: pass_more<4>(P, S, base); break;
          case 5: pass_more<5>(P, S, base); break;
          case 6: pass_more<6>(P, S, base); break;
          case 7: pass_more<7>(P, S, base); break;
          default: pass_more<8>(P, S, base); break;
        }
      }
    } else {
      pass_last(P, S, reinterpret_cast<float4 *>(c.r + start));
    }
    fence_proxy_async();
    __syncthreads();

    // ---- publish this CTA's partials, gather everyone's (fixed order)
    const uint32_t tag = base_tag + (uint32_t)e + 1u;
    unsigned long long *box = c.mbox + (size_t)(e & 1) * (kSlotsMax + 1) * nblk * 4;
    for (int s = tid; s < ns; s += kSweepThreads) {
      double ps = 0.0;
      uint32_t pc = 0;
#pragma unroll
      for (int w = 0; w < kSweepWarps; ++w) {
        ps = __dadd_rn(ps, S.wsum[s][w]);
        pc += S.wcnt[s][w];
      }
      ll_store(box + ((size_t)s * nblk + cta) * 4, tag, pc, ps);
    }
    for (int s = warp; s < ns; s += kSweepWarps) {
      double tot;
      unsigned long long ct;
      gather_slot(box + (size_t)s * nblk * 4, nblk, tag, lane, tot, ct);
      if (lane == 0) {
        S.tot_sum[s] = tot;
        S.tot_cnt[s] = ct;
      }
    }
    __syncthreads();

    if (has_tree) {
      if (warp == 0) decide(c, S, hd, e, lane, sigma2);
    } else if (cta == 0 && tid == 0) {  // sigma^2 (sampler.py:797-799, 906-908)
      const HP &hp = c.hp;
      const double s2 = __ddiv_rn(__dadd_rn(__dmul_rn(hp.nu, hp.lam), S.tot_sum[0]), *c.rand_chi2);
      *c.sigma2_draw = s2;
      if (hp.update_sigma) *c.sigma2 = s2;
      *c.tagbase = base_tag + (uint32_t)m + 1u;
      *c.iter_dev += 1ull;
    }
    if (warp == kSweepWarps - 1 && e + 1 < m) cp_async_wait_all();
    __syncthreads();
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
  return (int)cudaLaunchKernelEx(&cfg, sweep_kernel, c);
}

cudaError_t sweep_prepare(size_t smem) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin > (int)smem ? optin : (int)smem);
}

int sweep_max_ctas(size_t smem, int device) {
  int per_sm = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel, kSweepThreads, smem) != cudaSuccess)
    return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return per_sm * sms;
}

}  // namespace bart
