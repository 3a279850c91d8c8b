// Latency microbenchmarks that size the sweep's critical path on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void fp64_lat(double *out, long long *cyc, double seed) {
  double x = seed, y = 1.0000001;
  long long t0, t1;
  const int N = 256;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = __dadd_rn(x, y);
  t1 = clock64(); cyc[0] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = __dmul_rn(x, y);
  t1 = clock64(); cyc[1] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = __ddiv_rn(x, y + (double)i * 1e-9);
  t1 = clock64(); cyc[2] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = __dsqrt_rn(x + 2.0);
  t1 = clock64(); cyc[3] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = log(x + 3.0);
  t1 = clock64(); cyc[4] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = exp(-x);
  t1 = clock64(); cyc[5] = (t1 - t0) / N;
  float f = (float)x;
  t0 = clock64();
  for (int i = 0; i < N; ++i) { double d = (double)f; f = (float)(d * 1.0000001); }
  t1 = clock64(); cyc[6] = (t1 - t0) / N;
  out[threadIdx.x] = x + f;
}

__global__ void smem_lat(int *out, long long *cyc) {
  __shared__ int buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < 512; ++i) p = buf[p];
  long long t1 = clock64();
  cyc[0] = (t1 - t0) / 512;
  // __syncthreads cost with all warps
  t0 = clock64();
  for (int i = 0; i < 256; ++i) __syncthreads();
  t1 = clock64();
  cyc[1] = (t1 - t0) / 256;
  // __syncwarp
  t0 = clock64();
  for (int i = 0; i < 256; ++i) __syncwarp();
  t1 = clock64();
  cyc[2] = (t1 - t0) / 256;
  out[threadIdx.x] = p;
}

// L2 pointer chase (strong loads)
__global__ void l2_lat(const unsigned long long *chain, long long *cyc, unsigned long long *sink) {
  unsigned long long p = 0;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(p) : "l"(chain + p));
  long long t1 = clock64();
  cyc[0] = (t1 - t0) / 256;
  t0 = clock64();
  for (int i = 0; i < 256; ++i) asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(p) : "l"(chain + p));
  t1 = clock64();
  cyc[1] = (t1 - t0) / 256;
  sink[0] = p;
}

// ping-pong between CTA 0 and CTA b (different SMs): round trips of flag handoff
__global__ void pingpong(unsigned long long *flags, long long *cyc, int iters, int peer) {
  if (threadIdx.x != 0) return;
  volatile unsigned long long *f = flags;
  if (blockIdx.x == 0) {
    long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
      f[0] = i;
      while (f[16] != (unsigned long long)i) {}
    }
    cyc[0] = (clock64() - t0) / iters;
  } else if (blockIdx.x == peer) {
    for (int i = 1; i <= iters; ++i) {
      while (f[0] != (unsigned long long)i) {}
      f[16] = i;
    }
  }
}

// all-to-all exchange: each CTA publishes one tagged entry per round and
// gathers all entries (one warp), MODE 0 = poll every entry (LL),
// MODE 1 = red.add counter then one LL read, MODE 2 = counter with acquire.
template <int MODE>
__global__ void exchange(unsigned long long *box, unsigned long long *counter, long long *cyc, int rounds, double *sink) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = gridDim.x, cta = blockIdx.x;
  double acc = 0;
  long long t0 = clock64();
  for (int r = 1; r <= rounds; ++r) {
    unsigned long long *row = box + (size_t)(r & 1) * nb * 4;
    if (warp == 0) {
      if (lane == 0) {
        const unsigned long long t = ((unsigned long long)r) << 32;
        asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(row + cta * 4), "l"(t | 1ull), "l"(t | 2ull) : "memory");
        asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(row + cta * 4 + 2), "l"(t | 3ull) : "memory");
        if (MODE >= 1) asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(counter) : "memory");
      }
      if (MODE >= 1) {
        if (lane == 0) {
          unsigned long long v;
          const unsigned long long target = (unsigned long long)r * nb;
          if (MODE == 1) {
            do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(counter) : "memory"); } while (v < target);
          } else {
            do { asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(counter) : "memory"); } while (v < target);
          }
        }
        __syncwarp();
      }
      bool ok;
      unsigned long long a[8], b[8], d[8];
      do {
        ok = true;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int i = lane + 32 * k;
          if (i < nb) {
            asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a[k]), "=l"(b[k]) : "l"(row + i * 4) : "memory");
            asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(d[k]) : "l"(row + i * 4 + 2) : "memory");
            ok = ok && (a[k] >> 32) == (unsigned long long)r && (b[k] >> 32) == (unsigned long long)r && (d[k] >> 32) == (unsigned long long)r;
          }
        }
      } while (!__all_sync(0xffffffffu, ok));
      for (int k = 0; k < 8; ++k) if (lane + 32 * k < nb) acc += (double)(a[k] & 0xff);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[cta] = (t1 - t0) / rounds;
  if (threadIdx.x == 0) sink[cta] = acc;
}

// decider protocol: everyone publishes, CTA 0 gathers all (LL), broadcasts
// one tagged word to 8 replicas, the others poll their replica.
template <int VARIANT>
__global__ void decider_proto(unsigned long long *box, unsigned long long *bc, long long *cyc, int rounds, double *sink) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = gridDim.x, cta = blockIdx.x;
  double acc = 0;
  long long tg = 0, tb = 0;
  long long t0 = clock64();
  for (int r = 1; r <= rounds; ++r) {
    unsigned long long *row = box + (size_t)(r & 1) * nb * 4;
    unsigned long long *b = bc + (size_t)(r & 1) * 8 * 160;
    const unsigned long long t = ((unsigned long long)r) << 32;
    if (warp == 0 && lane == 0) {
      asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(row + cta * 4), "l"(t | 1ull), "l"(t | 2ull) : "memory");
      asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(row + cta * 4 + 2), "l"(t | 3ull) : "memory");
    }
    if (cta == 0) {
      if (warp == 0) {
        long long a0 = clock64();
        bool ok;
        unsigned long long a[8], bb[8], d[8];
        do {
          ok = true;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int i = lane + 32 * k;
            if (i < nb) {
              if (VARIANT == 0) {
                asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a[k]), "=l"(bb[k]) : "l"(row + i * 4) : "memory");
                asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(d[k]) : "l"(row + i * 4 + 2) : "memory");
              } else {
                asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a[k]), "=l"(bb[k]) : "l"(row + i * 4));
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(d[k]) : "l"(row + i * 4 + 2));
              }
              ok = ok && (a[k] >> 32) == (unsigned long long)r && (bb[k] >> 32) == (unsigned long long)r && (d[k] >> 32) == (unsigned long long)r;
            }
          }
        } while (!__all_sync(0xffffffffu, ok));
        tg += clock64() - a0;
        for (int k = 0; k < 8; ++k) if (lane + 32 * k < nb) acc += (double)(a[k] & 0xff);
        if (lane < 8) asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(b + lane * 160), "l"(t | 5ull) : "memory");
      }
    } else if (warp == 0) {
      long long a0 = clock64();
      unsigned long long w;
      do {
        asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(w) : "l"(b + (cta % 8) * 160) : "memory");
      } while ((w >> 32) != (unsigned long long)r);
      tb += clock64() - a0;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[cta] = (t1 - t0) / rounds; cyc[1024 + cta] = tg / rounds; cyc[2048 + cta] = tb / rounds; }
  if (threadIdx.x == 0) sink[cta] = acc;
}

// variants of the decider protocol.  SPREAD: stride between CTA entries in
// 64-bit words (4 = packed 32 B, 16 = one per 128 B line); WARPS: decider
// warps splitting the entries; BACKOFF: receivers sleep between polls (ns).
template <int SPREAD, int WARPS, int BACKOFF>
__global__ void proto2(unsigned long long *box, unsigned long long *bc, long long *cyc, int rounds, double *sink) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = gridDim.x, cta = blockIdx.x;
  double acc = 0;
  long long t0 = clock64();
  __shared__ int go;
  for (int r = 1; r <= rounds; ++r) {
    unsigned long long *row = box + (size_t)(r & 1) * 256 * SPREAD;
    unsigned long long *b = bc + (size_t)(r & 1) * 8 * 160;
    const unsigned long long t = ((unsigned long long)r) << 32;
    if (warp == 0 && lane == 0) {
      asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(row + cta * SPREAD), "l"(t | 1ull), "l"(t | 2ull) : "memory");
      asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(row + cta * SPREAD + 2), "l"(t | 3ull) : "memory");
    }
    if (cta == 0) {
      if (warp < WARPS) {
        bool ok;
        unsigned long long a[8], bb[8], d[8];
        do {
          ok = true;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int i = warp * 32 + lane + 32 * WARPS * k;
            if (i < nb) {
              asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a[k]), "=l"(bb[k]) : "l"(row + i * SPREAD) : "memory");
              asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(d[k]) : "l"(row + i * SPREAD + 2) : "memory");
              ok = ok && (a[k] >> 32) == (unsigned long long)r && (bb[k] >> 32) == (unsigned long long)r && (d[k] >> 32) == (unsigned long long)r;
            }
          }
        } while (!__all_sync(0xffffffffu, ok));
        for (int k = 0; k < 8; ++k) acc += (double)(a[k] & 0xff);
      }
      __syncthreads();
      if (warp == 0 && lane < 8) asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(b + lane * 160), "l"(t | 5ull) : "memory");
    } else if (warp == 0) {
      unsigned long long w;
      do {
        asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(w) : "l"(b + (cta % 8) * 160) : "memory");
        if (BACKOFF && (w >> 32) != (unsigned long long)r) __nanosleep(BACKOFF);
      } while ((w >> 32) != (unsigned long long)r);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[cta] = (t1 - t0) / rounds;
  if (threadIdx.x == 0) sink[cta] = acc;
}

template <int SPREAD, int WARPS, int BACKOFF>
int run_proto2(unsigned long long *box, long long *cyc, double *dout, int nb, const char *label) {
  unsigned long long *bc;
  CK(cudaMalloc(&bc, 2 * 8 * 160 * 8));
  CK(cudaMemset(bc, 0, 2 * 8 * 160 * 8));
  CK(cudaMemset(box, 0, 2 * 256 * 16 * 8));
  int rounds = 2000;
  void *args[] = {&box, &bc, &cyc, &rounds, &dout};
  CK(cudaLaunchCooperativeKernel((void *)proto2<SPREAD, WARPS, BACKOFF>, nb, 512, args, 0, 0));
  CK(cudaDeviceSynchronize());
  std::vector<long long> all(nb);
  CK(cudaMemcpy(all.data(), cyc, nb * 8, cudaMemcpyDeviceToHost));
  long long mx = 0;
  for (int i = 0; i < nb; ++i) mx = all[i] > mx ? all[i] : mx;
  printf("proto2 %-34s ctas %3d: %lld cyc/round\n", label, nb, mx);
  cudaFree(bc);
  return 0;
}

// atomic-accumulator protocol: every CTA red.adds NW words (spread over
// separate 128-B lines), then red.release on a counter; everyone polls the
// counter with ld.acquire and reads the NW words.  LINES: words per line.
template <int NW, int STRIDE>
__global__ void accum_proto(unsigned long long *acc, unsigned long long *counter, long long *cyc, int rounds,
                            double *sink) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = gridDim.x, cta = blockIdx.x;
  unsigned long long sum = 0;
  long long tw = 0;
  long long t0 = clock64();
  for (int r = 1; r <= rounds; ++r) {
    if (warp == 0) {
      if (lane < NW) asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(acc + lane * STRIDE), "l"((unsigned long long)(cta + 1)) : "memory");
      __syncwarp();
      if (lane == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(counter) : "memory");
      long long a0 = clock64();
      if (lane == 0) {
        unsigned long long v;
        const unsigned long long target = (unsigned long long)r * nb;
        do { asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(counter) : "memory"); } while (v < target);
      }
      __syncwarp();
      unsigned long long v = 0;
      if (lane < NW) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(acc + lane * STRIDE) : "memory");
      sum += v;
      tw += clock64() - a0;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[cta] = (t1 - t0) / rounds; cyc[1024 + cta] = tw / rounds; }
  if (threadIdx.x == 0) sink[cta] = (double)sum;
}

template <int NW, int STRIDE>
int run_accum(long long *cyc, double *dout, int nb) {
  unsigned long long *acc, *counter;
  CK(cudaMalloc(&acc, 64 * 16 * 8 * 4));
  CK(cudaMalloc(&counter, 256));
  CK(cudaMemset(acc, 0, 64 * 16 * 8 * 4));
  CK(cudaMemset(counter, 0, 256));
  int rounds = 2000;
  void *args[] = {&acc, &counter, &cyc, &rounds, &dout};
  CK(cudaLaunchCooperativeKernel((void *)accum_proto<NW, STRIDE>, nb, 512, args, 0, 0));
  CK(cudaDeviceSynchronize());
  std::vector<long long> all(2048);
  CK(cudaMemcpy(all.data(), cyc, 2048 * 8, cudaMemcpyDeviceToHost));
  long long mx = 0;
  for (int i = 0; i < nb; ++i) mx = all[i] > mx ? all[i] : mx;
  printf("accum protocol words %2d stride %2d ctas %3d: %lld cyc/round (cta0 wait %lld)\n", NW, STRIDE, nb, mx, all[1024]);
  cudaFree(acc); cudaFree(counter);
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long *cyc;
  double *dout;
  CK(cudaMalloc(&cyc, 4096 * sizeof(long long)));
  CK(cudaMalloc(&dout, 4096 * sizeof(double)));
  long long h[16];
  fp64_lat<<<1, 32>>>(dout, cyc, 1.5);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, cyc, 7 * 8, cudaMemcpyDeviceToHost));
  printf("fp64 latency (cyc, 1 warp): dadd %lld dmul %lld ddiv %lld dsqrt %lld log %lld exp %lld f2f(f32->f64->f32 + dmul) %lld\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
  int *iout;
  CK(cudaMalloc(&iout, 4096 * 4));
  smem_lat<<<1, 512>>>(iout, cyc);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, cyc, 3 * 8, cudaMemcpyDeviceToHost));
  printf("smem dependent load %lld cyc, __syncthreads(512 thr) %lld cyc, __syncwarp %lld cyc\n", h[0], h[1], h[2]);
  // L2 chain
  std::vector<unsigned long long> chain(1 << 20);
  for (size_t i = 0; i < chain.size(); ++i) chain[i] = (i * 7919 + 4099) % chain.size();
  unsigned long long *dchain, *sink;
  CK(cudaMalloc(&dchain, chain.size() * 8));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemcpy(dchain, chain.data(), chain.size() * 8, cudaMemcpyHostToDevice));
  l2_lat<<<1, 1>>>(dchain, cyc, sink);  // warm
  l2_lat<<<1, 1>>>(dchain, cyc, sink);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, cyc, 2 * 8, cudaMemcpyDeviceToHost));
  printf("L2-resident strong load latency: relaxed.gpu %lld cyc, volatile %lld cyc\n", h[0], h[1]);
  // ping-pong
  unsigned long long *flags;
  CK(cudaMalloc(&flags, 4096));
  for (int peer : {1, 2, 37, 74, 100, 147}) {
    CK(cudaMemset(flags, 0, 4096));
    pingpong<<<sms, 32>>>(flags, cyc, 2000, peer);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost));
    printf("ping-pong CTA0<->CTA%d: %lld cyc per round trip (two one-way handoffs)\n", peer, h[0]);
  }
  unsigned long long *box, *counter;
  CK(cudaMalloc(&box, 2 * 256 * 16 * 8));
  CK(cudaMalloc(&counter, 256));
  std::vector<long long> hc(sms);
  for (int mode = 0; mode < 0; ++mode)
    for (int nb : {1, 16, 74, sms}) {
      CK(cudaMemset(box, 0, 2 * 256 * 4 * 8));
      CK(cudaMemset(counter, 0, 256));
      void *args[] = {&box, &counter, &cyc, nullptr, &dout};
      int rounds = 2000;
      args[3] = &rounds;
      void (*fn)(unsigned long long *, unsigned long long *, long long *, int, double *) =
          mode == 0 ? exchange<0> : (mode == 1 ? exchange<1> : exchange<2>);
      CK(cudaLaunchCooperativeKernel((void *)fn, nb, 512, args, 0, 0));
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(hc.data(), cyc, nb * 8, cudaMemcpyDeviceToHost));
      long long mx = 0;
      for (int i = 0; i < nb; ++i) mx = hc[i] > mx ? hc[i] : mx;
      printf("exchange mode %d (%s) ctas %3d: %lld cyc per round (publish+gather+__syncthreads)\n", mode,
             mode == 0 ? "poll all LL" : (mode == 1 ? "counter+LL" : "counter acquire+LL"), nb, mx);
    }
  for (int variant = 0; variant < 1; ++variant)
    for (int nb : {2, 16, 74, sms}) {
      CK(cudaMemset(box, 0, 2 * 256 * 4 * 8));
      unsigned long long *bc;
      CK(cudaMalloc(&bc, 2 * 8 * 160 * 8));
      CK(cudaMemset(bc, 0, 2 * 8 * 160 * 8));
      int rounds = 2000;
      void *args[] = {&box, &bc, &cyc, &rounds, &dout};
      CK(cudaLaunchCooperativeKernel((void *)(variant == 0 ? decider_proto<0> : decider_proto<1>), nb, 512, args, 0, 0));
      CK(cudaDeviceSynchronize());
      std::vector<long long> all(3072);
      CK(cudaMemcpy(all.data(), cyc, 3072 * 8, cudaMemcpyDeviceToHost));
      long long mx = 0, mb = 0;
      for (int i = 0; i < nb; ++i) mx = all[i] > mx ? all[i] : mx;
      for (int i = 1; i < nb; ++i) mb = all[2048 + i] > mb ? all[2048 + i] : mb;
      printf("decider protocol (%s loads) ctas %3d: %lld cyc/round; decider gather wait %lld; max receiver wait %lld\n",
             variant == 0 ? "volatile" : "relaxed.gpu", nb, mx, all[1024], mb);
      cudaFree(bc);
    }
  for (int nb : {sms}) {
    run_proto2<4, 1, 0>(box, cyc, dout, nb, "packed, 1 warp, spin");
    run_proto2<16, 1, 0>(box, cyc, dout, nb, "line-spread, 1 warp, spin");
    run_proto2<16, 4, 0>(box, cyc, dout, nb, "line-spread, 4 warps, spin");
    run_proto2<16, 4, 100>(box, cyc, dout, nb, "line-spread, 4 warps, backoff 100ns");
    run_proto2<4, 4, 0>(box, cyc, dout, nb, "packed, 4 warps, spin");
  }
  for (int nb : {sms}) {
    run_proto2<4, 1, 0>(box, cyc, dout, nb, "packed, 1 warp, spin");
    run_proto2<16, 1, 0>(box, cyc, dout, nb, "line-spread, 1 warp, spin");
    run_proto2<16, 4, 0>(box, cyc, dout, nb, "line-spread, 4 warps, spin");
    run_proto2<16, 4, 100>(box, cyc, dout, nb, "line-spread, 4 warps, backoff 100ns");
    run_proto2<4, 4, 0>(box, cyc, dout, nb, "packed, 4 warps, spin");
  }
  for (int nb : {16, 74, sms}) {
    run_accum<5, 16>(cyc, dout, nb);
    run_accum<20, 16>(cyc, dout, nb);
    run_accum<20, 1>(cyc, dout, nb);
  }
  return 0;
}
