// The sweep's A pass in isolation: 14 worker warps per CTA, one CTA per SM,
// W register words (4 points each) per thread; per pass: residual update
// from a leaf-delta table in shared memory, f64 per-slot sums (C compared
// slots + running total), warp reductions, per-warp partials to shared
// memory, one CTA barrier.  Reported: cycles per pass (CTA 0, median), for
// variants of the inner loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/bin/apass_bench tools/apass_bench.cu
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>

constexpr int kWorkers = 448;
constexpr int kWarps = kWorkers / 32;
constexpr int kPasses = 64;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

// f32 -> f64 by integer ops (normal numbers and zero; denormals flush, which
// the real kernel would route to F2F)
__device__ __forceinline__ double f2d_int(float f) {
  const uint32_t b = __float_as_uint(f);
  const uint32_t mag = b & 0x7fffffffu;
  const uint32_t hi = (b & 0x80000000u) | (mag ? ((mag >> 3) + 0x38000000u) : 0u);
  const uint32_t lo = b << 29;
  return __hiloint2double((int)hi, (int)lo);
}

template <int W, int C, int VAR>
__global__ void __launch_bounds__(kWorkers, 1) apass(const float *rin, const uint32_t *lin, int nwords, long long *out, double *sink) {
  __shared__ float dlt[256];
  __shared__ double wsum[kWarps][16];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int h = tid; h < 256; h += kWorkers) dlt[h] = h ? 1e-3f * (float)(h % 7) - 2e-3f : 0.f;
  float4 r[W];
  uint32_t lc[W];
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const int w = tid + k * kWorkers;
    r[k] = w < nwords ? reinterpret_cast<const float4 *>(rin)[w + blockIdx.x * W * kWorkers] : make_float4(0, 0, 0, 0);
    lc[k] = w < nwords ? lin[w + blockIdx.x * W * kWorkers] : 0u;
  }
  __syncthreads();
  long long t[kPasses];
  for (int p = 0; p < kPasses; ++p) {
    const long long t0 = clock64();
    double acc[C], tot = 0.0;
    uint32_t sn[C];
#pragma unroll
    for (int s = 0; s < C; ++s) {
      acc[s] = 0.0;
      sn[s] = 1 + s + (p & 1);
    }
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int w = tid + k * kWorkers;
      const bool guard = VAR & 1;
      if (!guard || w < nwords) {
        const uint32_t l = lc[k];
        r[k].x = __fadd_rn(r[k].x, dlt[l & 0xffu]);
        r[k].y = __fadd_rn(r[k].y, dlt[(l >> 8) & 0xffu]);
        r[k].z = __fadd_rn(r[k].z, dlt[(l >> 16) & 0xffu]);
        r[k].w = __fadd_rn(r[k].w, dlt[l >> 24]);
        const float rv[4] = {r[k].x, r[k].y, r[k].z, r[k].w};
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint32_t h = (l >> (8 * b)) & 0xffu;
          const double v = (VAR & 2) ? f2d_int(rv[b]) : (double)rv[b];
          tot = __dadd_rn(tot, v);
#pragma unroll
          for (int s = 0; s < C; ++s) {
            if (VAR & 4)
              asm("{.reg .pred p; setp.eq.u32 p, %1, %2; @p add.rn.f64 %0, %0, %3;}" : "+d"(acc[s]) : "r"(h), "r"(sn[s]), "d"(v));
            else if (VAR & 8)
              acc[s] = __dadd_rn(acc[s], h == sn[s] ? v : 0.0);
            else
              acc[s] = __fma_rn(v, h == sn[s] ? 1.0 : 0.0, acc[s]);
          }
        }
      }
    }
    double rest = tot;
#pragma unroll
    for (int s = 0; s < C; ++s) {
      const double v = warp_sum(acc[s]);
      rest = __dsub_rn(rest, acc[s]);
      if (lane == 0) wsum[warp][s] = v;
    }
    const double v = warp_sum(rest);
    if (lane == 0) wsum[warp][C] = v;
    __syncthreads();
    t[p] = clock64() - t0;
    if (tid == 0) sink[blockIdx.x] += wsum[3][0];
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid == 0) {
    for (int p = 0; p < kPasses; ++p) out[p] = t[p];
  }
#pragma unroll
  for (int k = 0; k < W; ++k) sink[1000 + tid] += r[k].x + r[k].y + r[k].z + r[k].w;
}

template <int W, int C, int VAR>
void run(const float *r, const uint32_t *l, int nwords, long long *d, double *sink, const char *name) {
  apass<W, C, VAR><<<148, kWorkers>>>(r, l, nwords, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  std::vector<long long> h(kPasses);
  cudaMemcpy(h.data(), d, kPasses * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin() + 4, h.end());
  printf("W %d C %d %-28s %6lld cycles per pass\n", W, C, name, h[4 + (kPasses - 4) / 2]);
}

int main() {
  const int W = 4, nwords = 1692;
  const size_t words = (size_t)148 * W * kWorkers;
  float *r;
  uint32_t *l;
  long long *d;
  double *sink;
  cudaMalloc(&r, words * 16);
  cudaMalloc(&l, words * 4);
  cudaMalloc(&d, kPasses * 8);
  cudaMalloc(&sink, 4096 * 8);
  std::vector<float> hr(words * 4);
  std::vector<uint32_t> hl(words);
  uint32_t x = 12345;
  for (auto &v : hr) {
    x = x * 1664525u + 1013904223u;
    v = ((x >> 8) & 0xffff) / 65536.f - 0.5f;
  }
  for (auto &v : hl) {
    uint32_t o = 0;
    for (int b = 0; b < 4; ++b) {
      x = x * 1664525u + 1013904223u;
      o |= (1u + ((x >> 16) % 4u)) << (8 * b);
    }
    v = o;
  }
  cudaMemcpy(r, hr.data(), words * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(l, hl.data(), words * 4, cudaMemcpyHostToDevice);
  run<4, 1, 5>(r, l, nwords, d, sink, "guarded, predicated DADD");
  run<4, 3, 5>(r, l, nwords, d, sink, "guarded, predicated DADD");
  run<4, 7, 5>(r, l, nwords, d, sink, "guarded, predicated DADD");
  run<4, 3, 9>(r, l, nwords, d, sink, "guarded, select DADD");
  run<4, 1, 1>(r, l, nwords, d, sink, "guarded (sweep v8)");
  run<4, 1, 0>(r, l, nwords, d, sink, "unguarded");
  run<4, 1, 3>(r, l, nwords, d, sink, "guarded, int f2d");
  run<4, 1, 2>(r, l, nwords, d, sink, "unguarded, int f2d");
  run<4, 3, 1>(r, l, nwords, d, sink, "guarded (sweep v8)");
  run<4, 3, 0>(r, l, nwords, d, sink, "unguarded");
  run<4, 3, 3>(r, l, nwords, d, sink, "guarded, int f2d");
  run<4, 3, 2>(r, l, nwords, d, sink, "unguarded, int f2d");
  run<4, 7, 1>(r, l, nwords, d, sink, "guarded (sweep v8)");
  run<4, 7, 0>(r, l, nwords, d, sink, "unguarded");
  return 0;
}
