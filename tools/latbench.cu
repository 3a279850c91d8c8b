// Dependent-chain latencies (cycles) of the primitives on the sweep's
// per-tree critical path, one warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/latbench tools/latbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N 128
__global__ void lat(long long *out, double seed, unsigned long long useed) {
  __shared__ unsigned long long mb;
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  long long t0, t1;
  int k = 0;
  double x = seed + lane;
  unsigned long long u = useed + lane;
#define TIME(name, body)                          \
  t0 = clock64();                                 \
  for (int i = 0; i < N; ++i) { body; }          \
  t1 = clock64();                                 \
  if (lane == 0) out[k] = (t1 - t0) / N;          \
  ++k;
  TIME("dadd", x = __dadd_rn(x, 1.0000001))
  TIME("dfma", x = __fma_rn(x, 0.999999, 1e-9))
  TIME("f2i.s64 floor", { long long h = __double2ll_rd(x); x = (double)(h & 7) + 1.5; })
  TIME("i2f.f64.s64", { x = (double)(long long)u; u = (unsigned long long)(x) + 3; })
  TIME("f2i.u64 rn", { u = __double2ull_rn(x) + 1; x = (double)(u & 15); })
  TIME("shfl f64", x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31) + 1.0)
  TIME("shfl u32", { uint32_t v = __shfl_sync(0xffffffffu, (uint32_t)u, (lane + 1) & 31); u = v + 1; })
  TIME("redux add", { uint32_t v = __reduce_add_sync(0xffffffffu, (uint32_t)u); u = v + lane; })
  if (lane < 64) sm[lane] = 1.0;
  __syncwarp();
  TIME("lds f64", x = sm[((int)x) & 31] + 1.0)
  TIME("int64 add+shift", { u = (u << 3) + (u >> 7) + 1; })
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mb)));
  __syncwarp();
  if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&mb)));
  __syncwarp();
  TIME("mbar try_wait (complete)", {
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&mb)) : "memory");
  })
  TIME("syncwarp", __syncwarp())
  TIME("ld.relaxed.gpu L2 (same line)", {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"((unsigned long long *)out + 100 + (u & 1)) : "memory");
    u += v & 1;
  })
  if (lane == 0) out[k] = (long long)(x + (double)u);
}

int main() {
  long long *d, h[32];
  cudaMalloc(&d, 4096);
  cudaMemset(d, 0, 4096);
  lat<<<1, 32>>>(d, 1.5, 7);
  lat<<<1, 32>>>(d, 1.5, 7);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char *names[] = {"dadd", "dfma", "f2i.s64 floor (+i2f)", "i2f.f64.s64 (+f2i)", "f2i.u64 rn (+i2f)", "shfl f64 (+dadd)",
                         "shfl u32 (+iadd)", "redux add (+iadd)", "lds f64 (+dadd,f2i)", "int64 shift/add", "mbar try_wait complete",
                         "syncwarp", "ld.relaxed.gpu L2 hit"};
  for (int i = 0; i < 13; ++i) printf("%-28s %lld cyc\n", names[i], h[i]);
  return 0;
}
