// Does q = fma(fma(-b, RN(a*y), a), y, RN(a*y)) with y = RN(1/b) (Markstein)
// reproduce __ddiv_rn(a, b) bit for bit on the decision's operand ranges?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/divtest tools/divtest.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cstring>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}
__device__ __forceinline__ double u01(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

__global__ void test(uint64_t seed, unsigned long long *bad, unsigned long long *example, int iters) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned long long nb = 0;
  for (int i = 0; i < iters; ++i) {
    const uint64_t h1 = mix(seed ^ (tid * 0x9E3779B97F4A7C15ull + i)), h2 = mix(h1 + 0x1234567ull), h3 = mix(h2);
    // a: prior + tau * sums, any sign, magnitudes 1e-6 .. 1e9 ; b: prec in 1e-3 .. 1e10
    const double ea = -20.0 + 50.0 * u01(h1), eb = -10.0 + 43.0 * u01(h2);
    double a = exp2(ea) * (1.0 + u01(h3));
    if (h3 & 1) a = -a;
    const double b = exp2(eb) * (1.0 + u01(mix(h3 + 7)));
    const double q = __ddiv_rn(a, b);
    const double y = __drcp_rn(b);
    const double q0 = __dmul_rn(a, y);
    const double r = __fma_rn(-b, q0, a);
    const double q1 = __fma_rn(r, y, q0);
    if (__double_as_longlong(q1) != __double_as_longlong(q)) {
      ++nb;
      example[0] = __double_as_longlong(a);
      example[1] = __double_as_longlong(b);
    }
  }
  if (nb) atomicAdd(bad, nb);
}

__global__ void lat(double a, double b, long long *cyc, double *sink) {
  double x = a, y = __drcp_rn(b);
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) x = __ddiv_rn(x, b) + 1.0;
  long long t1 = clock64();
  double z = a;
  for (int i = 0; i < 256; ++i) {
    const double q0 = __dmul_rn(z, y);
    const double r = __fma_rn(-b, q0, z);
    z = __fma_rn(r, y, q0) + 1.0;
  }
  long long t2 = clock64();
  cyc[0] = (t1 - t0) / 256;
  cyc[1] = (t2 - t1) / 256;
  sink[0] = x + z;
}

int main() {
  unsigned long long *bad, *ex;
  cudaMalloc(&bad, 8); cudaMalloc(&ex, 16);
  cudaMemset(bad, 0, 8);
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  for (int s = 0; s < 4; ++s) test<<<blocks, threads>>>(1000 + s, bad, ex, iters);
  cudaDeviceSynchronize();
  unsigned long long h = 0, e[2] = {0, 0};
  cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(e, ex, 16, cudaMemcpyDeviceToHost);
  printf("markstein vs __ddiv_rn: %llu mismatches in %.3g samples\n", h, 4.0 * blocks * threads * iters);
  if (h) { double a, b; memcpy(&a, &e[0], 8); memcpy(&b, &e[1], 8); printf("  e.g. a=%.17g b=%.17g\n", a, b); }
  long long *cyc; double *sink;
  cudaMalloc(&cyc, 16); cudaMalloc(&sink, 8);
  lat<<<1, 1>>>(3.7, 1.3, cyc, sink);
  long long c[2];
  cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
  printf("latency: __ddiv_rn %lld cyc, markstein %lld cyc (chained, +1 dadd each)\n", c[0], c[1]);
  return 0;
}
