// Cost of the control warp's exchange-add step in isolation: f64 -> 3 fixed-point
// limbs (to_limbs) -> 3 coalesced red.add.u64, one warp, no contention.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int kLimbBits = 37;
constexpr unsigned long long kLimbMask = (1ull << kLimbBits) - 1ull;
__device__ __forceinline__ void to_limbs(double x, unsigned long long (&l)[3]) {
  const long long hi = __double2ll_rd(x);
  const double rem = __dsub_rn(x, (double)hi);
  const unsigned long long lo = __double2ull_rn(__dmul_rn(rem, 0x1.0p64));
  l[0] = lo & kLimbMask;
  l[1] = ((lo >> kLimbBits) | ((unsigned long long)hi << (64 - kLimbBits))) & kLimbMask;
  l[2] = ((unsigned long long)(hi >> (2 * kLimbBits - 64))) & kLimbMask;
}
template <int MODE>
__global__ void k(unsigned long long *acc, long long *out, double seed) {
  const int lane = threadIdx.x, q = lane & 3, s = lane >> 2;
  double x = seed + lane * 0.001;
  unsigned long long sink = 0;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) {
    unsigned long long l[3] = {0, 0, 0};
    if (MODE == 3) out[64 + lane] = sink;  // a plain global store before the reds
    if (MODE == 4) { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); out[64 + lane] = t; }
    if (MODE != 2) to_limbs(x, l);
    else l[0] = __double_as_longlong(x) & 0xff, l[1] = l[0], l[2] = l[0];
    const unsigned long long v = (1ull << 48) | (q == 0 ? l[0] : (q == 1 ? l[1] : l[2]));
    if (MODE >= 1 && q < 3) asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(acc + s * 4 + q), "l"(v) : "memory");
    sink += v;
    x = __dadd_rn(x, (double)(sink & 1));  // next iteration depends on this one's limbs
  }
  long long t1 = clock64();
  if (lane == 0) out[MODE] = (t1 - t0) / 256;
  if (sink == 1) out[10] = 1;
}
int main() {
  unsigned long long *acc; long long *out, h[5];
  cudaMalloc(&acc, 4096); cudaMalloc(&out, 4096); cudaMemset(acc, 0, 4096);
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<1, 32>>>(acc, out, 1.25); k<1><<<1, 32>>>(acc, out, 1.25); k<2><<<1, 32>>>(acc, out, 1.25);
    k<3><<<1, 32>>>(acc, out, 1.25); k<4><<<1, 32>>>(acc, out, 1.25);
  }
  cudaDeviceSynchronize();
  cudaMemcpy(h, out, 40, cudaMemcpyDeviceToHost);
  printf("to_limbs chain: %lld cyc/iter; to_limbs + 3 red: %lld; red only: %lld; st.global then limbs+red: %lld; clock+st then limbs+red: %lld\n", h[0], h[1], h[2], h[3], h[4]);
  return 0;
}
