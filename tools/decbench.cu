// decide_fast in isolation: one warp, a loop of decisions on fake data, to
// compare its latency with the in-sweep timeline.
#define BART_DECBENCH 1
#include <cstdio>
#include "../paper_2410_23244_b200/csrc/sweep.cu"
using namespace bart;

__global__ void decbench(long long *out, double seed) {
  extern __shared__ __align__(128) unsigned char raw[];
  SweepSmem &S = *reinterpret_cast<SweepSmem *>(raw);
  const int lane = threadIdx.x;
  DecConst K{0.9, 4.0, 0.0, 0.0};
  TreeHdr hd{};
  hd.kind = KIND_GROW; hd.node = 1; hd.nslots = 2; hd.slot_l = 0; hd.slot_r = 1;
  DecIn I{};
  I.cadj = 0.1 * lane; I.den = 100.0 + lane; I.rcp = __drcp_rn(I.den); I.zs = 0.01; I.h = 2 + lane; I.oldv = 0.5f;
  I.prec_l = 100.0; I.prec_r = 101.0; I.prec_p = 201.0; I.partial = -0.3; I.log_u = -1.0; I.acc_u = 0.3;
  double tot = seed + lane;
  long long t0 = clock64();
  for (int i = 0; i < 64; ++i) {
    decide_fast(S, S.dec[i & 1], I, tot, hd, lane, K, nullptr);
    tot = tot + (double)S.dlt[2] * 1e-9;  // next decision depends on this one
  }
  long long t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0) / 64;
}

int main() {
  long long *d, h;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(decbench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SweepSmem));
  for (int r = 0; r < 2; ++r) decbench<<<1, 32, sizeof(SweepSmem)>>>(d, 1.0);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("decide_fast in isolation: %lld cycles per decision (incl. bar.arrive on an unmatched barrier)\n", h);
  return 0;
}
