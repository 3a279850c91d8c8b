// Phase 1 of the step: one move proposal per tree, one warp per tree.
//
// Reference semantics: bforge sampler._propose_kernel (sampler.py:326-466)
// and propose_moves (sampler.py:469-526).  The reference keeps per-node
// availability caches avail_lo/avail_hi of shape (m, 2^D, p) (sampler.py:
// 142-143, 171-198, 850-859); here availability is recomputed from the
// node's ancestors (<= D-1 of them), which equals the cached value on every
// present node (the only nodes the reference reads), and avoids 2*m*2^D*p
// bytes of state (64 MB each at m=1000, p=1000).
//
// With device RNG the same kernel also draws the step's random block
// (sampler.py:244-260 layout: move_u (m,5), accept_u (m), leaf_z (m,2^D),
// one chi-square) from Philox4x32-10 keyed by (seed, iteration).
#include "propose.cuh"
#include "internal.h"

namespace bart {

__global__ void __launch_bounds__(kProposeWarps * 32) propose_kernel(ChainDev c, int device_rng) {
  __shared__ uint8_t s_cut[kProposeWarps][kSlotsMax];
  __shared__ uint16_t s_axis[kProposeWarps][kSlotsMax];
  __shared__ uint32_t s_masks[kProposeWarps][24];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const unsigned long long it = *c.iter_dev;
  if (device_rng && blockIdx.x == gridDim.x - 1) {  // the chi-square block
    const uint2 key = make_uint2((uint32_t)c.seed, (uint32_t)(c.seed >> 32));
    if (threadIdx.x == 0) *c.rand_chi2 = chi2_draw(c.hp.nu + (double)c.n_total, it, key);
    return;
  }
  const int j = blockIdx.x * kProposeWarps + wl;
  if (j >= c.m) return;
  propose_tree(c, j, it, device_rng, s_cut[wl], s_axis[wl], s_masks[wl], lane);
}

void launch_propose(const ChainDev &c, int device_rng, cudaStream_t s) {
  const int blocks = (c.m + kProposeWarps - 1) / kProposeWarps + (device_rng ? 1 : 0);
  propose_kernel<<<blocks, kProposeWarps * 32, 0, s>>>(c, device_rng);
}

__global__ void philox_kernel(const uint4 *ctr, const uint2 *key, uint4 *out, int64_t count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = philox(ctr[i], key[i]);
}

void launch_philox(const uint32_t *ctr, const uint32_t *key, uint32_t *out, int64_t count, cudaStream_t s) {
  const int threads = 256;
  const int64_t blocks = (count + threads - 1) / threads;
  philox_kernel<<<(unsigned)blocks, threads, 0, s>>>(reinterpret_cast<const uint4 *>(ctr),
                                                    reinterpret_cast<const uint2 *>(key),
                                                    reinterpret_cast<uint4 *>(out), count);
}

}  // namespace bart
