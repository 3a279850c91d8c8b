// Does the control warp's decision (a dependent FP64 chain of ~40 ops) slow
// down when the worker warps of its SM sub-partition run the B pass (SWAR
// byte compares + POPC, integer-heavy) at the same time?
// One CTA per SM, 16 warps (the sweep's 512 threads): warp 14 runs the
// dependent chain and times it; warps w % 4 == 2 (its sub-partition) and the
// others optionally run a B-pass-like loop meanwhile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/bin/contention_bench tools/contention_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t bytes_eq(uint32_t a, uint32_t b4) {
  const uint32_t x = a ^ b4;
  const uint32_t t = ((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x;
  return ~t & 0x80808080u;
}

__global__ void __launch_bounds__(512, 1) bench(int mode, int iters, long long *out, uint32_t *sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ volatile int go;
  if (threadIdx.x == 0) go = 0;
  __syncthreads();
  if (warp == 14) {
    double x = 1.0 + lane * 1e-9, y = 0.999;
    long long tot = 0;
    for (int it = 0; it < iters; ++it) {
      if (lane == 0) go = it + 1;
      __syncwarp();
      const long long t0 = clock64();
#pragma unroll 1
      for (int k = 0; k < 40; ++k) x = __fma_rn(x, y, 1e-3);  // dependent chain
      x = __shfl_sync(0xffffffffu, x, 0);
      const long long t1 = clock64();
      tot += t1 - t0;
      // gap between decisions
      const long long w0 = clock64();
      while (clock64() - w0 < 3000) {
      }
    }
    if (lane == 0) {
      out[blockIdx.x] = tot / iters;
      go = -1;
    }
    if (x == 123.0) sink[0] = 1;
  } else if (warp < 14 && (mode == 2 || (mode == 1 && (warp & 3) == 2))) {
    uint32_t acc = 0, v = threadIdx.x * 2654435761u;
    while (go >= 0) {
#pragma unroll 8
      for (int k = 0; k < 64; ++k) {
        v = v * 1664525u + 1013904223u;
        acc += __popc(bytes_eq(v, 0x03030303u)) + __popc(bytes_eq(v, 0x05050505u));
      }
    }
    if (acc == 0xdeadbeef) sink[1] = acc;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long *out;
  uint32_t *sink;
  cudaMalloc(&out, sms * 8);
  cudaMalloc(&sink, 16);
  const char *names[] = {"alone", "3 busy warps on its sub-partition", "13 busy warps on the SM"};
  for (int mode = 0; mode < 3; ++mode) {
    bench<<<sms, 512>>>(mode, 200, out, sink);
    cudaDeviceSynchronize();
    long long h[256];
    cudaMemcpy(h, out, sms * 8, cudaMemcpyDeviceToHost);
    long long s = 0;
    for (int i = 0; i < sms; ++i) s += h[i];
    printf("40-op dependent DFMA chain + shuffle, %-36s %6lld cycles\n", names[mode], s / sms);
  }
  return 0;
}
