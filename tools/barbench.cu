// Hand-off latency inside one CTA, the sweep's DECISION pattern: one warp
// (the "control") publishes, 14 waiting warps wake and read shared memory.
// Variants: named barrier (bar.arrive / bar.sync over 480 threads), mbarrier
// (arrive / try_wait.parity), shared-memory flag spin.  Reported: cycles from
// the control's publish to the last waiter's first dependent read, median
// over rounds.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/barbench tools/barbench.cu
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>

constexpr int kRounds = 256;
constexpr int kWaiters = 14;

__device__ __forceinline__ void mbar_init(unsigned long long *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"((uint32_t)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(
          (uint32_t)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}

template <int MODE>
__global__ void handoff(long long *out, int spin) {
  __shared__ volatile int flag;
  __shared__ int payload[kRounds];
  __shared__ long long t_pub[kRounds], t_wake[kRounds][kWaiters];
  __shared__ unsigned long long mb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    flag = -1;
    mbar_init(&mb, 1);
  }
  __syncthreads();
  for (int r = 0; r < kRounds; ++r) {
    if (warp == kWaiters) {  // control
      const long long t0 = clock64();
      while (clock64() - t0 < spin) {
      }
      if (lane == 0) payload[r] = r;
      __syncwarp();
      const long long tp = clock64();
      if (MODE == 0) asm volatile("bar.arrive 1, %0;" ::"r"((kWaiters + 1) * 32) : "memory");
      if (MODE == 1 && lane == 0) mbar_arrive(&mb);
      if (MODE == 2 && lane == 0) flag = r;
      if (lane == 0) t_pub[r] = tp;
      // the waiters' next round needs the control ahead of them: wait for them
      asm volatile("bar.sync 2, %0;" ::"r"((kWaiters + 1) * 32) : "memory");
    } else {
      int v;
      if (MODE == 0) {
        asm volatile("bar.sync 1, %0;" ::"r"((kWaiters + 1) * 32) : "memory");
        v = payload[r];
      } else if (MODE == 1) {
        mbar_wait(&mb, (uint32_t)(r & 1));
        v = payload[r];
      } else {
        while (flag != r) {
        }
        v = payload[r];
      }
      const long long tw = clock64() + (v < 0 ? 1 : 0);
      if (lane == 0) t_wake[r][warp] = tw;
      asm volatile("bar.sync 2, %0;" ::"r"((kWaiters + 1) * 32) : "memory");
    }
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int r = 0; r < kRounds; ++r) {
      long long mx = 0;
      for (int w = 0; w < kWaiters; ++w) { const long long dd = t_wake[r][w] - t_pub[r]; mx = dd > mx ? dd : mx; }
      out[r] = mx;
    }
}

template <int MODE>
void run(const char *name) {
  long long *d;
  cudaMalloc(&d, kRounds * 8);
  handoff<MODE><<<1, (kWaiters + 1) * 32>>>(d, 2000);
  std::vector<long long> h(kRounds);
  cudaMemcpy(h.data(), d, kRounds * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin() + 8, h.end());
  printf("%-16s publish -> last waiter read: median %lld, p90 %lld cycles\n", name, h[8 + (kRounds - 8) / 2],
         h[8 + (kRounds - 8) * 9 / 10]);
  cudaFree(d);
}

int main() {
  run<0>("named barrier");
  run<1>("mbarrier");
  run<2>("smem flag spin");
  return 0;
}
