// Exchange microbenchmark in the sweep's own pattern: one warp per CTA, one
// CTA per SM; per round, lane 4s+q adds tagged word q (< 3) of slot s (one
// coalesced red per warp instruction, 8 slots), then polls until every word
// is complete.  Variants:
//   stride: words between consecutive slots (4 = one 32-B sector per slot,
//           16 = one 128-B line per slot, 32 = two lines)
//   G:      CTA c adds only into group copy c % G; readers load all G copies
//           and sum them (integer sums: exact, order-free), so each word sees
//           nblk / G atomics instead of nblk.
// Reported: cycles per round minus the compute spin, max over CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/xbench2 tools/xbench2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kTagShift = 48;
constexpr unsigned long long kMask = (1ull << kTagShift) - 1;
constexpr size_t kCopyWords = 8 * 32 * 32;  // up to 32 slots x stride 32

template <int G>
__global__ void xround(unsigned long long *acc, int ns, int stride, int rounds, int work, long long *cyc) {
  const int lane = threadIdx.x, nb = gridDim.x, cta = blockIdx.x;
  __shared__ unsigned long long prev[3][G][32];
  for (int i = lane; i < 3 * G * 32; i += 32) (&prev[0][0][0])[i] = 0;
  __syncwarp();
  const int q = lane & 3, s = lane >> 2;
  const bool mine = s < ns && q < 3;
  // arrivals per group copy
  const int gsz_base = nb / G, gextra = nb % G;
  unsigned long long sink = 0;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const int set = r % 3;
    const long long w0 = clock64();
    while (clock64() - w0 < work) {
    }
    unsigned long long *base = acc + (size_t)set * G * kCopyWords;
    if (mine) {
      unsigned long long *a = base + (size_t)(cta % G) * kCopyWords + (size_t)s * stride + q;
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(a), "l"((1ull << kTagShift) | (unsigned long long)(cta + r)) : "memory");
    }
    unsigned long long v[G];
    bool done;
    do {
      bool ok = true;
      if (mine) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const unsigned long long *a = base + (size_t)g * kCopyWords + (size_t)s * stride + q;
          asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v[g]) : "l"(a) : "memory");
          const unsigned long long want = (unsigned long long)(gsz_base + (g < gextra ? 1 : 0)) << kTagShift;
          ok = ok && ((v[g] - prev[set][g][lane]) & ~kMask) == want;
        }
      }
      done = __all_sync(0xffffffffu, ok);
    } while (!done);
    if (mine)
#pragma unroll
      for (int g = 0; g < G; ++g) {
        sink += (v[g] - prev[set][g][lane]) & kMask;
        prev[set][g][lane] = v[g];
      }
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[cta] = (t1 - t0) / rounds;
  if (sink == 42) cyc[4000] = 1;
}

template <int G>
int run(int nb, int ns, int stride, int work) {
  unsigned long long *acc;
  long long *cyc;
  const size_t words = (size_t)3 * G * kCopyWords;
  CK(cudaMalloc(&acc, words * 8));
  CK(cudaMemset(acc, 0, words * 8));
  CK(cudaMalloc(&cyc, 4096 * 8));
  int rounds = 3000;
  void *args[] = {&acc, &ns, &stride, &rounds, &work, &cyc};
  CK(cudaLaunchCooperativeKernel((void *)xround<G>, nb, 32, args, 0, 0));
  CK(cudaDeviceSynchronize());
  std::vector<long long> c(nb);
  CK(cudaMemcpy(c.data(), cyc, nb * 8, cudaMemcpyDeviceToHost));
  long long mc = 0;
  for (int i = 0; i < nb; ++i) mc = c[i] > mc ? c[i] : mc;
  printf("ctas %3d slots %2d stride %2d groups %2d work %4d: exchange %5lld cyc\n", nb, ns, stride, G, work, mc - work);
  cudaFree(acc);
  cudaFree(cyc);
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int work = 2000;
  for (int ns : {2, 4, 8}) {
    for (int stride : {4, 16, 32}) {
      run<1>(sms, ns, stride, work);
      run<2>(sms, ns, stride, work);
      run<4>(sms, ns, stride, work);
      run<8>(sms, ns, stride, work);
    }
  }
  for (int nb : {1, 8, 37, 74}) run<1>(nb, 4, 4, work);
  return 0;
}
