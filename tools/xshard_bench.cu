// One-GPU emulation of the n-sharded exchange's ARRIVALS:
// flat vs two-level, at N = 1, 2, 4, 8 shards of 148 CTAs.
//
// 148 CTAs, one warp each, one CTA per SM, the sweep's word layout (lane 4s+q
// owns word q of slot s, slots 256 B apart, tagged adds (1 << 48) | value).
// Per round (one tree's exchange, ns slots):
//   flat       every CTA plays its counterpart CTA on each of the N shards:
//              it adds N times into the copy it polls (the N arrivals a word
//              receives per CTA index), and N-1 times into each of N-1 other
//              copies (the remote copies' traffic), then polls its copy until
//              148*N arrivals are in -- a word sees 148*N atomics.
//   two-level  every CTA adds once into the stage words (its shard's); CTA 0
//              (the forwarder) polls the stage complete (148 arrivals), then
//              adds the shard total into the polled copy N times (the N
//              shards' forwarders) and into N-1 other copies; everyone polls
//              its copy until N arrivals are in.
// Not emulated: NVLink latency between GPUs (one device here).  Reported:
// cycles per round (max over CTAs, median over rounds).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/xshard_bench tools/xshard_bench.cu
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kTagShift = 48;
constexpr unsigned long long kOne = 1ull << kTagShift, kMask = kOne - 1;
constexpr int kSlotWords = 32;                  // 256 B between slots
constexpr size_t kSetWords = 33 * kSlotWords;   // 32 slots + spare
constexpr int kSets = 3;
constexpr int kRounds = 200;

__device__ __forceinline__ void red(unsigned long long *p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ldr(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// copies: [N][kSets][kSetWords] (copy 0 polled), stage: [kSets][kSetWords]
__global__ void rounds_kernel(unsigned long long *copies, unsigned long long *stage, int N, int ns, int two_level,
                              int work, long long *cyc) {
  const int lane = threadIdx.x, cta = blockIdx.x, nb = gridDim.x;
  const int q = lane & 3, s = lane >> 2;
  const bool mine = s < ns && q < 3;
  unsigned long long prev[kSets] = {0, 0, 0}, sprev[kSets] = {0, 0, 0};
  const unsigned long long target = (unsigned long long)(two_level ? N : nb * N) << kTagShift;
  for (int r = 0; r < kRounds; ++r) {
    const int set = r % kSets;
    const long long w0 = clock64();
    while (clock64() - w0 < work + (cta * 37 + r * 11) % 300) {  // A pass stand-in, CTA skew
    }
    const long long t0 = clock64();
    const size_t off = (size_t)set * kSetWords + (size_t)s * kSlotWords + q;
    const unsigned long long val = kOne | (unsigned long long)(cta + 1);
    if (mine) {
      if (!two_level) {
        for (int k = 0; k < N; ++k) red(copies + off, val);
        for (int g = 1; g < N; ++g)
          for (int k = 0; k < N; ++k) red(copies + (size_t)g * kSets * kSetWords + off, val);
      } else {
        red(stage + off, val);
      }
    }
    if (two_level && cta == 0) {  // the forwarder
      unsigned long long w = 0;
      bool done;
      do {
        bool ok = true;
        if (mine) {
          w = ldr(stage + off);
          ok = ((w - sprev[set]) & ~kMask) == ((unsigned long long)nb << kTagShift);
        }
        done = __all_sync(0xffffffffu, ok);
      } while (!done);
      if (mine) {
        const unsigned long long d = (w - sprev[set]) & kMask;
        sprev[set] = w;
        for (int k = 0; k < N; ++k) red(copies + off, kOne | d);
        for (int g = 1; g < N; ++g)
          for (int k = 0; k < N; ++k) red(copies + (size_t)g * kSets * kSetWords + off, kOne | d);
      }
    }
    unsigned long long w = 0;
    bool done;
    do {
      bool ok = true;
      if (mine) {
        w = ldr(copies + off);
        ok = ((w - prev[set]) & ~kMask) == target;
      }
      done = __all_sync(0xffffffffu, ok);
    } while (!done);
    if (mine) prev[set] = w;
    if (lane == 0) cyc[(size_t)r * nb + cta] = clock64() - t0;
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int ns = 4, work = 3000;
  unsigned long long *copies, *stage;
  long long *cyc;
  CK(cudaMalloc(&copies, (size_t)8 * kSets * kSetWords * 8));
  CK(cudaMalloc(&stage, (size_t)kSets * kSetWords * 8));
  CK(cudaMalloc(&cyc, (size_t)kRounds * sms * 8));
  std::vector<long long> h((size_t)kRounds * sms);
  printf("exchange emulation: %d CTAs per shard, %d slots, per-round cycles (max over CTAs, median of rounds)\n", sms,
         ns);
  for (int two = 0; two < 2; ++two)
    for (int N : {1, 2, 4, 8}) {
      CK(cudaMemset(copies, 0, (size_t)8 * kSets * kSetWords * 8));
      CK(cudaMemset(stage, 0, (size_t)kSets * kSetWords * 8));
      rounds_kernel<<<sms, 32>>>(copies, stage, N, ns, two, work, cyc);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost));
      std::vector<long long> mx;
      for (int r = 10; r < kRounds; ++r) {
        long long m = 0;
        for (int c = 0; c < sms; ++c) m = std::max(m, h[(size_t)r * sms + c]);
        mx.push_back(m);
      }
      std::sort(mx.begin(), mx.end());
      printf("  %-9s N=%d: %6lld cycles per exchange (%d arrivals per polled word)\n", two ? "two-level" : "flat", N,
             mx[mx.size() / 2], two ? N : sms * N);
    }
  return 0;
}
