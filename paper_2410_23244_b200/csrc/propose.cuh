// Phase 1 of the step, per tree (device code shared by the standalone
// propose kernel and the sweep, which proposes tree j of the NEXT iteration
// as soon as it has finalised tree j -- see csrc/sweep.cu).
//
// Reference semantics: bforge sampler._propose_kernel (sampler.py:326-466)
// and propose_moves (sampler.py:469-526).  The reference keeps per-node
// availability caches avail_lo/avail_hi of shape (m, 2^D, p) (sampler.py:
// 142-143, 171-198, 850-859); here availability is recomputed from the
// node's ancestors (<= D-1 of them), which equals the cached value on every
// present node (the only nodes the reference reads), and avoids 2*m*2^D*p
// bytes of state (64 MB each at m=1000, p=1000).
//
// With device RNG the random block (sampler.py:244-260 layout: move_u (m,5),
// accept_u (m), leaf_z (m,2^D), one chi-square) comes from Philox4x32-10
// keyed by (seed, iteration).
#pragma once
#include "common.cuh"

namespace bart {


// Distinct split axes on the path from the root to node h, with the open
// interval (lo, hi] of cutpoints each leaves at h (oracles.py:44-59 walk).
struct PathInfo {
  int n;
  int axis[kMaxDepth];
  int lo[kMaxDepth];
  int hi[kMaxDepth];
};

__device__ __forceinline__ void path_info(const uint8_t *cut, const uint16_t *axis,
                                          const int32_t *max_cuts, int h, PathInfo &P) {
  P.n = 0;
  const int d = heap_depth(h);
  for (int k = d; k >= 1; --k) {  // root first, deeper splits override
    const int anc = h >> k;
    const int a = axis[anc];
    const int c = cut[anc];
    int idx = -1;
    for (int i = 0; i < P.n; ++i)
      if (P.axis[i] == a) idx = i;
    if (idx < 0) {
      idx = P.n++;
      P.axis[idx] = a;
      P.lo[idx] = 0;
      P.hi[idx] = max_cuts[a];
    }
    if ((h >> (k - 1)) & 1)
      P.lo[idx] = c;
    else
      P.hi[idx] = c - 1;
  }
}

// number of axes with a non-empty interval at the node (sampler.py:397-400)
__device__ __forceinline__ int open_axes(const PathInfo &P, const int32_t *max_cuts, int P_open) {
  int on_path_splittable = 0, open_on_path = 0;
  for (int i = 0; i < P.n; ++i) {
    on_path_splittable += max_cuts[P.axis[i]] > 0;
    open_on_path += P.hi[i] > P.lo[i];
  }
  return P_open - on_path_splittable + open_on_path;
}

__device__ __forceinline__ int nth_set_bit(uint32_t m, int k) {
  for (int i = 0; i < k; ++i) m &= m - 1;
  return __ffs(m) - 1;
}

__device__ __forceinline__ bool mask_bit(const uint32_t *mask, int h) { return (mask[h >> 5] >> (h & 31)) & 1u; }

// chi-square(df) draw by Marsaglia-Tsang on Gamma(df/2), 2x.
static __device__ __noinline__ double chi2_draw(double df, unsigned long long it, uint2 key) {
  double a = 0.5 * df;
  const bool boost = a < 1.0;
  const double a0 = a;
  if (boost) a += 1.0;
  const double d = a - 1.0 / 3.0, cc = 1.0 / sqrt(9.0 * d);
  double g = d;
  for (uint32_t att = 0; att < 256; ++att) {
    const uint4 r = philox(make_uint4((uint32_t)it, (uint32_t)(it >> 32), 0xFFFFFFFFu, att), key);
    const double u1 = 1.0 - u53(r.x, r.y), u2 = u53(r.z, r.w);
    const double z = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    double v = 1.0 + cc * z;
    if (v <= 0.0) continue;
    v = v * v * v;
    const uint4 q = philox(make_uint4((uint32_t)it, (uint32_t)(it >> 32), 0xFFFFFFFEu, att), key);
    const double u = 1.0 - u53(q.x, q.y);
    if (u < 1.0 - 0.0331 * z * z * z * z || log(u) < 0.5 * z * z + d * (1.0 - v + log(v))) {
      g = d * v;
      if (boost) g *= pow(1.0 - u53(q.z, q.w), 1.0 / a0);
      break;
    }
  }
  return 2.0 * g;
}

// Phase 1 for tree j, by one warp: the tree's random numbers (device RNG:
// Philox keyed by (seed, iteration `it`); else the injected block), the
// proposal and its bookkeeping, and the tree's record for the sweep.  `cut`
// and `ax` are per-warp shared-memory scratch of kSlotsMax entries.
// (The loops over 32-node chunks stay rolled and keep their masks in shared
// memory: this code runs once per tree, cold in the instruction cache, so its
// size matters more than its instruction count.)
__device__ __forceinline__ void propose_tree(const ChainDev &c, int j, unsigned long long it, int device_rng,
                                             uint8_t *cut, uint16_t *ax, uint32_t *masks, int lane) {
  const uint2 key = make_uint2((uint32_t)c.seed, (uint32_t)(c.seed >> 32));
  const int D = c.D, half = c.half, size = c.size;
  uint8_t *rec = c.rec + (size_t)j * c.rstride;
  float *rec_old = reinterpret_cast<float *>(rec + 224);
  double *rec_zz = reinterpret_cast<double *>(rec + 224 + 4 * size);
  for (int h = lane; h < size; h += 32) rec_old[h] = c.leaf[(size_t)j * size + h];
  for (int i = lane; i < half; i += 32) {
    cut[i] = c.cut[(size_t)j * half + i];
    ax[i] = c.axis[(size_t)j * half + i];
  }
  __syncwarp();

  // ---- the tree's random numbers (sampler.py:253-260 block layout)
  double u[5], acc_u;
  if (device_rng) {
    double ra = 0.0, rb = 0.0;
    if (lane < 3) {
      const uint4 r = philox(make_uint4((uint32_t)it, (uint32_t)(it >> 32), (uint32_t)j, (uint32_t)lane), key);
      ra = u53(r.x, r.y);
      rb = u53(r.z, r.w);
    }
    u[0] = __shfl_sync(0xffffffffu, ra, 0);
    u[1] = __shfl_sync(0xffffffffu, rb, 0);
    u[2] = __shfl_sync(0xffffffffu, ra, 1);
    u[3] = __shfl_sync(0xffffffffu, rb, 1);
    u[4] = __shfl_sync(0xffffffffu, ra, 2);
    acc_u = __shfl_sync(0xffffffffu, rb, 2);
    if (lane < 5) c.rand_move[(size_t)j * 5 + lane] = u[lane];
    if (lane == 0) c.rand_acc[j] = acc_u;
    for (int q = lane; 2 * q < size; q += 32) {  // Box-Muller pairs
      const uint4 r = philox(make_uint4((uint32_t)it, (uint32_t)(it >> 32), (uint32_t)j, 16u + (uint32_t)q), key);
      const double u1 = 1.0 - u53(r.x, r.y), u2 = u53(r.z, r.w);
      const double rad = sqrt(-2.0 * log(u1));
      double sn, cs;
      sincospi(2.0 * u2, &sn, &cs);
      c.rand_z[(size_t)j * size + 2 * q] = rad * cs;
      rec_zz[2 * q] = rad * cs;
      if (2 * q + 1 < size) {
        c.rand_z[(size_t)j * size + 2 * q + 1] = rad * sn;
        rec_zz[2 * q + 1] = rad * sn;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < 5; ++k) u[k] = c.rand_move[(size_t)j * 5 + k];
    acc_u = c.rand_acc[j];
    for (int h = lane; h < size; h += 32) rec_zz[h] = c.rand_z[(size_t)j * size + h];
  }

  // ---- candidate sets in heap order (sampler.py:342-360)
  const int npl = (size + 31) >> 5;
  uint32_t *gmask = masks, *pmask = masks + 8, *lmask = masks + 16;
  int w = 0, wp = 0;
#pragma unroll 1
  for (int k = 0; k < 8; ++k) {
    if (k < npl) {
      const int h = lane + 32 * k;
      const bool valid = h >= 1 && h < size;
      bool present = valid;
      for (int a = h >> 1; a >= 1; a >>= 1) present = present && cut[a] != 0;
      const bool internal = valid && h < half && cut[h] != 0;
      const bool leaf = present && !internal;
      bool growable = false;
      if (leaf && heap_depth(h) < D - 1) {
        PathInfo P;
        path_info(cut, ax, c.max_cuts, h, P);
        growable = open_axes(P, c.max_cuts, c.P_open) > 0;
      }
      bool prunable = false;
      if (internal) {
        const bool kids_internal = 2 * h < half && (cut[2 * h] != 0 || cut[2 * h + 1] != 0);
        prunable = !kids_internal;
      }
      const uint32_t gm = __ballot_sync(0xffffffffu, growable), pm = __ballot_sync(0xffffffffu, prunable);
      const uint32_t lm = __ballot_sync(0xffffffffu, leaf);
      if (lane == 0) {
        gmask[k] = gm;
        pmask[k] = pm;
        lmask[k] = lm;
      }
      w += __popc(gm);
      wp += __popc(pm);
    } else if (lane == 0) {
      gmask[k] = pmask[k] = lmask[k] = 0u;
    }
  }
  __syncwarp();

  // ---- move kind and target (sampler.py:362-395)
  int kind = KIND_NONE, t = 0;
  if (w > 0 || wp > 0) {
    const bool grow = w > 0 && (wp == 0 || u[0] < c.hp.p_grow);
    kind = grow ? KIND_GROW : KIND_PRUNE;
    const int cnt = grow ? w : wp;
    int kk = (int)__dmul_rn(grow ? u[1] : u[4], (double)cnt);
    if (kk > cnt - 1) kk = cnt - 1;
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
      const uint32_t mk = grow ? gmask[k] : pmask[k];
      const int pc = __popc(mk);
      if (kk >= 0 && kk < pc) {
        t = 32 * k + nth_set_bit(mk, kk);
        kk = -1;
      } else if (kk >= 0) {
        kk -= pc;
      }
    }
  }
  const bool grow = kind == KIND_GROW;

  int na = 0, a_sel = 0, la = 0, ha = 0, ns = 0, c_sel = 0, depth = 0;
  int gl = 0, gr = 0, w_small = 0, w_prime_big = 0, growable_big = 0;
  double struct_log = 0.0;
  if (kind != KIND_NONE) {
    PathInfo P;
    path_info(cut, ax, c.max_cuts, t, P);
    na = open_axes(P, c.max_cuts, c.P_open);
    if (grow) {  // floor(u2*na)-th open axis in index order (sampler.py:401-411)
      int ka = (int)__dmul_rn(u[2], (double)na);
      if (ka > na - 1) ka = na - 1;
      int found = -1;
      for (int base = 0; base < c.p && found < 0; base += 32) {
        const int a = base + lane;
        bool op = false;
        if (a < c.p) {
          int idx = -1;
          for (int i = 0; i < P.n; ++i)
            if (P.axis[i] == a) idx = i;
          op = idx >= 0 ? (P.hi[idx] > P.lo[idx]) : (((c.open_bits[a >> 5] >> (a & 31)) & 1u) != 0u);
        }
        const uint32_t b = __ballot_sync(0xffffffffu, op);
        const int pc = __popc(b);
        if (ka < pc)
          found = base + nth_set_bit(b, ka);
        else
          ka -= pc;
      }
      a_sel = found;
    } else {
      a_sel = ax[t];
    }
    int idx = -1;
    for (int i = 0; i < P.n; ++i)
      if (P.axis[i] == a_sel) idx = i;
    la = idx >= 0 ? P.lo[idx] : 0;
    ha = idx >= 0 ? P.hi[idx] : c.max_cuts[a_sel];
    ns = ha - la;
    if (grow) {  // sampler.py:417-421
      int kc = (int)__dmul_rn(u[3], (double)ns);
      if (kc > ns - 1) kc = ns - 1;
      c_sel = la + 1 + kc;
    } else {
      c_sel = cut[t];
    }
    // bookkeeping (sampler.py:425-440)
    depth = heap_depth(t);
    const bool child_ok = depth < D - 2;
    if (grow) {
      const bool other = na >= 2;
      gl = child_ok && (other || c_sel - 1 > la);
      gr = child_ok && (other || ha > c_sel);
      w_small = w;
      const bool par_pr = t > 1 && mask_bit(pmask, t >> 1);
      w_prime_big = wp + 1 - (par_pr ? 1 : 0);
      growable_big = w - 1 + gl + gr;
    } else {
      gl = mask_bit(gmask, 2 * t);
      gr = mask_bit(gmask, 2 * t + 1);
      w_small = w - gl - gr + 1;
      w_prime_big = wp;
      growable_big = w;
    }
    // structural log-ratio, grow direction (sampler.py:453-466)
    const double dp = c.hp.depth_prob[depth];
    const double cp = c.hp.depth_prob[depth + 1 < D ? depth + 1 : D - 1];
    const double ppe = growable_big == 0 ? 1.0 : __dsub_rn(1.0, c.hp.p_grow);
    const double pge = t == 1 ? 1.0 : c.hp.p_grow;
    const double ws = (double)(w_small > 1 ? w_small : 1);
    const double wpb = (double)(w_prime_big > 1 ? w_prime_big : 1);
    const double core = __ddiv_rn(__dmul_rn(__dmul_rn(dp, ppe), ws),
                                  __dmul_rn(__dmul_rn(__dsub_rn(1.0, dp), pge), wpb));
    struct_log = __dadd_rn(__dadd_rn(log(core), log1p(__dmul_rn(-cp, gl ? 1.0 : 0.0))),
                           log1p(__dmul_rn(-cp, gr ? 1.0 : 0.0)));
  }

  // ---- leaves of the larger tree, heap order: the sweep's histogram slots
  TreeMove &mv = *reinterpret_cast<TreeMove *>(rec);
  int nslots = 0, slot_l = 0, slot_r = 0;
#pragma unroll 1
  for (int k = 0; k < 8; ++k) {
    if (k < npl) {
      const int h = lane + 32 * k;
      bool big = (lmask[k] >> lane) & 1u;
      if (grow && h == t) big = false;
      if (grow && (h == 2 * t || h == 2 * t + 1)) big = true;
      const uint32_t b = __ballot_sync(0xffffffffu, big);
      const int idx = nslots + __popc(b & ((1u << lane) - 1u));
      if (big) mv.slot_node[idx] = (uint8_t)h;
      if (big && kind != KIND_NONE && h == 2 * t) slot_l = idx;
      if (big && kind != KIND_NONE && h == 2 * t + 1) slot_r = idx;
      nslots += __popc(b);
    }
  }
  slot_l = __reduce_max_sync(0xffffffffu, (unsigned)slot_l);
  slot_r = __reduce_max_sync(0xffffffffu, (unsigned)slot_r);
  if (lane == 0) {
    mv.kind = kind;
    mv.node = t;
    mv.axis = a_sel;
    mv.cut = c_sel;
    mv.depth = depth;
    mv.n_axes = na;
    mv.n_splits = ns;
    mv.w_small = w_small;
    mv.w_prime_big = w_prime_big;
    mv.growable_big = growable_big;
    mv.gl = gl;
    mv.gr = gr;
    mv.nslots = nslots;
    mv.struct_log = struct_log;
    mv.log_u = log(acc_u);
    mv.acc_u = acc_u;
    TreeHdr hd;
    hd.kind = (uint8_t)kind;
    hd.node = (uint8_t)t;
    hd.cut = (uint8_t)c_sel;
    hd.nslots = (uint8_t)nslots;
    hd.axis = (uint16_t)a_sel;
    hd.slot_l = (uint8_t)slot_l;
    hd.slot_r = (uint8_t)slot_r;
    c.hdr[j] = hd;
  }
}


}  // namespace bart
