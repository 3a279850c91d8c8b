// Microbenchmark of the sweep's cross-CTA exchange: 148 CTAs, one warp each,
// R rounds of (red.add NW tagged words per CTA -> poll until every word
// carries nblk more arrivals than last round).  Variants: words per line
// layout, load scope, replicated words, poll backoff.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/xbench tools/xbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kTagShift = 48;

// word w of the round's set lives at: SPREAD=0 -> set + w (packed),
// SPREAD=1 -> set + w*16 (one 128-B line per word).  REPL copies of every
// word; CTA c adds into copy c % REPL.  SYS: poll loads at .sys scope.
template <int SPREAD, int REPL, int SYS, int BACKOFF>
__global__ void xround(unsigned long long *acc, int nw, int rounds, long long *cyc, long long *ns) {
  const int lane = threadIdx.x, nb = gridDim.x, cta = blockIdx.x;
  __shared__ unsigned long long prev[3][64 * REPL];
  for (int i = lane; i < 3 * 64 * REPL; i += 32) (&prev[0][0])[i] = 0;
  __syncwarp();
  const int stride = SPREAD ? 16 : 1;
  const size_t set_words = (size_t)64 * REPL * 16;
  long long t0 = clock64(), g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  unsigned long long sink = 0;
  for (int r = 0; r < rounds; ++r) {
    const int set = r % 3;
    unsigned long long *base = acc + set * set_words;
    // adds
    for (int w = lane; w < nw; w += 32) {
      unsigned long long *a = base + (size_t)(w * REPL + cta % REPL) * stride;
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(a), "l"((1ull << kTagShift) | (unsigned long long)(cta + r)) : "memory");
    }
    // poll
    unsigned long long vals[4];
    bool done;
    do {
      bool ok = true;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = lane + 32 * k;
        if (i < nw * REPL) {
          const int w = i / REPL, rep = i % REPL;
          const unsigned long long *a = base + (size_t)(w * REPL + rep) * stride;
          unsigned long long v;
          if (SYS)
            asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
          else
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
          const unsigned long long expect = (unsigned long long)(nb / REPL + (rep < nb % REPL ? 1 : 0));
          ok = ok && ((v - prev[set][i]) >> kTagShift) == expect;
          vals[k] = v;
        }
      }
      done = __all_sync(0xffffffffu, ok);
      if (!done && BACKOFF) __nanosleep(BACKOFF);
    } while (!done);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = lane + 32 * k;
      if (i < nw * REPL) {
        prev[set][i] = vals[k];
        sink += vals[k];
      }
    }
    __syncwarp();
  }
  long long t1 = clock64(), g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (lane == 0) {
    cyc[cta] = (t1 - t0) / rounds;
    ns[cta] = (g1 - g0) / rounds;
  }
  if (sink == 42) cyc[1000] = 1;
}

template <int SPREAD, int REPL, int SYS, int BACKOFF>
int run(int nb, int nw, const char *label) {
  unsigned long long *acc;
  long long *cyc, *ns;
  const size_t words = (size_t)3 * 64 * REPL * 16;
  CK(cudaMalloc(&acc, words * 8));
  CK(cudaMemset(acc, 0, words * 8));
  CK(cudaMalloc(&cyc, 2048 * 8));
  CK(cudaMalloc(&ns, 2048 * 8));
  int rounds = 3000;
  void *args[] = {&acc, &nw, &rounds, &cyc, &ns};
  // note: prev[] is only updated when a word is seen complete, so a word
  // completes exactly once per round (the poll re-reads until all are).
  CK(cudaLaunchCooperativeKernel((void *)xround<SPREAD, REPL, SYS, BACKOFF>, nb, 32, args, 0, 0));
  CK(cudaDeviceSynchronize());
  std::vector<long long> c(nb), n(nb);
  CK(cudaMemcpy(c.data(), cyc, nb * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(n.data(), ns, nb * 8, cudaMemcpyDeviceToHost));
  long long mc = 0, mn = 0;
  for (int i = 0; i < nb; ++i) {
    mc = c[i] > mc ? c[i] : mc;
    mn = n[i] > mn ? n[i] : mn;
  }
  printf("%-44s ctas %3d words %3d: %6lld cyc/round %6lld ns/round\n", label, nb, nw, mc, mn);
  cudaFree(acc);
  cudaFree(cyc);
  cudaFree(ns);
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int nw : {4, 16, 20, 32}) {
    run<0, 1, 0, 0>(sms, nw, "packed, gpu loads");
    run<0, 1, 1, 0>(sms, nw, "packed, sys loads");
    run<1, 1, 0, 0>(sms, nw, "line per word, gpu loads");
    run<1, 4, 0, 0>(sms, nw, "line per word, 4 replicas, gpu loads");
    run<1, 1, 0, 64>(sms, nw, "line per word, gpu loads, 64ns backoff");
  }
  for (int nb : {2, 16, 74})
    run<1, 1, 0, 0>(nb, 16, "line per word, gpu loads");
  return 0;
}
