// Per-SM throughput and dependent latency of the instructions on the sweep's
// critical paths (B200): DFMA, DADD, F2F.F64.F32, F2I.S64.F64, I2F.F64.U64,
// ISETP+FSEL, SHFL.  Throughput: 16 warps per SM, 8 independent chains per
// thread; latency: one warp, one chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/bin/pipe_bench tools/pipe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int N = 512;  // iterations per chain

template <int OP, int CH>
__global__ void kern(double *out, long long *cyc, float seed) {
  double d[CH];
  float f[CH];
  long long l[CH];
  for (int c = 0; c < CH; ++c) {
    d[c] = 1.0 + threadIdx.x * 1e-7 + c * 1e-3;
    f[c] = seed + c;
    l[c] = threadIdx.x + c;
  }
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) d[c] = __fma_rn(d[c], 0.9999, 1e-4);
      if (OP == 1) d[c] = __dadd_rn(d[c], 1e-4);
      if (OP == 2) { f[c] = __fadd_rn(f[c], 1.0f); d[c] = __dadd_rn(d[c], (double)f[c]); }  // F2F + DADD
      if (OP == 3) { l[c] = __double2ll_rd(d[c]); d[c] = __dadd_rn(d[c], 1.0) ; d[c] += (double)(l[c] & 1); }
      if (OP == 4) d[c] = __fma_rn(d[c], (threadIdx.x + i + c) & 1 ? 1.0 : 0.0, 1e-4);  // ISETP/FSEL + DFMA
      if (OP == 5) d[c] = __shfl_xor_sync(0xffffffffu, d[c], 1 + (c & 15)) + 1e-4;
    }
  }
  const long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c] + f[c] + l[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char *name, double *out, long long *cyc, int sms) {
  long long h[1];
  kern<OP, 8><<<sms, 512>>>(out, cyc, 1.f);
  cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  const double ops = 512.0 * 8 * N;  // thread-ops per SM
  const double tput = ops / h[0];
  kern<OP, 1><<<1, 32>>>(out, cyc, 1.f);
  cudaDeviceSynchronize();
  cudaMemcpy(h + 0, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-34s throughput %6.1f lanes/clk/SM   dependent latency %5.1f cycles\n", name, tput, (double)h[0] / N);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  long long *cyc;
  cudaMalloc(&out, (size_t)sms * 512 * 8);
  cudaMalloc(&cyc, sms * 8);
  run<0>("DFMA", out, cyc, sms);
  run<1>("DADD", out, cyc, sms);
  run<2>("FADD + F2F.F64.F32 + DADD", out, cyc, sms);
  run<3>("F2I.S64.F64 + DADD + I2F + DADD", out, cyc, sms);
  run<4>("select multiplier + DFMA", out, cyc, sms);
  run<5>("SHFL (f64) + DADD", out, cyc, sms);
  return 0;
}
