// Microbenchmark of the sweep's cross-CTA exchange (one warp per CTA, one CTA
// per SM): R rounds of [spin WORK cycles] -> red.add NS slots x 3 tagged words
// -> poll until every word carries one more arrival per CTA than last round.
// Reported: cycles per round minus WORK (= exchange cost incl. skew).
// Variants: K copies of the words (every CTA adds into all K, polls copy
// cta % K), poll backoff, slot layout (3 words in one sector vs one line each).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/xbench tools/xbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kTagShift = 48;
constexpr int kMaxK = 8;
constexpr size_t kSetWords = 64 * 16 * 4;  // slots x line x (3 words spread over up to 4 lines)

template <int K, int SPREAD, int BACKOFF>
__global__ void xround(unsigned long long *acc, int ns, int rounds, int work, long long *cyc) {
  const int lane = threadIdx.x, nb = gridDim.x, cta = blockIdx.x;
  __shared__ unsigned long long prev[3][32][3];
  for (int i = lane; i < 3 * 32 * 3; i += 32) (&prev[0][0][0])[i] = 0;
  __syncwarp();
  const unsigned long long target = (unsigned long long)nb << kTagShift;
  unsigned long long sink = 0;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const int set = r % 3;
    // the compute between exchanges
    const long long w0 = clock64();
    while (clock64() - w0 < work) {
    }
    // adds: lane s owns slot s
    if (lane < ns) {
      for (int k = 0; k < K; ++k) {
        unsigned long long *base = acc + ((size_t)k * 3 + set) * kSetWords;
        for (int q = 0; q < 3; ++q) {
          unsigned long long *a = base + (SPREAD ? ((size_t)q * 64 + lane) * 16 : (size_t)lane * 16 + q);
          asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(a), "l"((1ull << kTagShift) | (unsigned long long)(cta + r)) : "memory");
        }
      }
    }
    // poll own copy
    const unsigned long long *base = acc + ((size_t)(cta % K) * 3 + set) * kSetWords;
    unsigned long long v[3];
    bool done;
    do {
      bool ok = true;
      if (lane < ns) {
        for (int q = 0; q < 3; ++q) {
          const unsigned long long *a = base + (SPREAD ? ((size_t)q * 64 + lane) * 16 : (size_t)lane * 16 + q);
          asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v[q]) : "l"(a) : "memory");
          ok = ok && ((v[q] - prev[set][lane][q]) & ~((1ull << kTagShift) - 1)) == target;
        }
      }
      done = __all_sync(0xffffffffu, ok);
      if (!done && BACKOFF) __nanosleep(BACKOFF);
    } while (!done);
    if (lane < ns)
      for (int q = 0; q < 3; ++q) {
        prev[set][lane][q] = v[q];
        sink += v[q];
      }
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[cta] = (t1 - t0) / rounds;
  if (sink == 42) cyc[4000] = 1;
}

template <int K, int SPREAD, int BACKOFF>
int run(int nb, int ns, int work, const char *label) {
  unsigned long long *acc;
  long long *cyc;
  const size_t words = (size_t)kMaxK * 3 * kSetWords;
  CK(cudaMalloc(&acc, words * 8));
  CK(cudaMemset(acc, 0, words * 8));
  CK(cudaMalloc(&cyc, 4096 * 8));
  int rounds = 2000;
  void *args[] = {&acc, &ns, &rounds, &work, &cyc};
  CK(cudaLaunchCooperativeKernel((void *)xround<K, SPREAD, BACKOFF>, nb, 32, args, 0, 0));
  CK(cudaDeviceSynchronize());
  std::vector<long long> c(nb);
  CK(cudaMemcpy(c.data(), cyc, nb * 8, cudaMemcpyDeviceToHost));
  long long mc = 0;
  for (int i = 0; i < nb; ++i) mc = c[i] > mc ? c[i] : mc;
  printf("%-40s ctas %3d slots %2d work %5d: exchange %5lld cyc\n", label, nb, ns, work, mc - work);
  cudaFree(acc);
  cudaFree(cyc);
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int work : {0, 2000}) {
    for (int ns : {1, 4, 8}) {
      run<1, 0, 0>(sms, ns, work, "sector per slot");
      run<1, 1, 0>(sms, ns, work, "line per word");
      run<2, 0, 0>(sms, ns, work, "sector per slot, 2 copies");
      run<4, 0, 0>(sms, ns, work, "sector per slot, 4 copies");
      run<8, 0, 0>(sms, ns, work, "sector per slot, 8 copies");
      run<1, 0, 100>(sms, ns, work, "sector per slot, backoff 100ns");
      run<4, 1, 0>(sms, ns, work, "line per word, 4 copies");
    }
  }
  for (int nb : {1, 2, 8, 37, 74, 98})
    run<1, 0, 0>(nb, 4, 2000, "sector per slot");
  return 0;
}
