// Does an SM see different L2 latency for different lines (near vs far die)?
// One CTA per SM (one thread); each measures the latency of an L2-hitting
// relaxed load (the exchange's poll) to K candidate 256-B slots, median of
// reps.  Prints per-SM-group statistics and how well a 2-way split of the
// slots by latency separates the SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/l2_near_far tools/l2_near_far.cu
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

constexpr int K = 256;      // candidate slots
constexpr int kStride = 32; // u64 words (256 B) between slots
constexpr int REPS = 16;

__global__ void probe(unsigned long long *buf, int *lat, int *smid_out) {
  if (threadIdx.x) return;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  smid_out[blockIdx.x] = (int)smid;
  for (int k = 0; k < K; ++k) {
    unsigned long long *p = buf + (size_t)k * kStride;
    int best[REPS];
    for (int r = 0; r < REPS; ++r) {
      unsigned long long v;
      const long long t0 = clock64();
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
      long long t1;  // a clock read that cannot issue before the load's value is back
      asm volatile("{\n .reg .pred q;\n setp.eq.u64 q, %1, 0x7E4D3C2B1A098765;\n @q trap;\n mov.u64 %0, %%clock64;\n}"
                   : "=l"(t1) : "l"(v) : "memory");
      best[r] = (int)(t1 - t0);
    }
    // median
    for (int i = 1; i < REPS; ++i)
      for (int j = i; j > 0 && best[j - 1] > best[j]; --j) {
        int t = best[j];
        best[j] = best[j - 1];
        best[j - 1] = t;
      }
    lat[blockIdx.x * K + k] = best[REPS / 2];
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *buf;
  int *lat, *smid;
  cudaMalloc(&buf, (size_t)K * kStride * 8);
  cudaMemset(buf, 0, (size_t)K * kStride * 8);
  cudaMalloc(&lat, (size_t)sms * K * 4);
  cudaMalloc(&smid, sms * 4);
  probe<<<sms, 32>>>(buf, lat, smid);
  cudaDeviceSynchronize();
  std::vector<int> h((size_t)sms * K), sm(sms);
  cudaMemcpy(h.data(), lat, h.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(sm.data(), smid, sms * 4, cudaMemcpyDeviceToHost);
  // per slot: mean latency from SMs with smid < sms/2 vs >= sms/2
  int lo_near = 0;
  std::vector<double> diff(K);
  for (int k = 0; k < K; ++k) {
    double a = 0, b = 0;
    int na = 0, nb = 0;
    for (int c = 0; c < sms; ++c) {
      if (sm[c] < sms / 2) {
        a += h[(size_t)c * K + k];
        ++na;
      } else {
        b += h[(size_t)c * K + k];
        ++nb;
      }
    }
    diff[k] = a / na - b / nb;
    lo_near += diff[k] < 0;
  }
  std::vector<int> all(h);
  std::sort(all.begin(), all.end());
  printf("L2-hit load latency (cycles) over %d SMs x %d slots: min %d p10 %d median %d p90 %d max %d\n", sms, K,
         all[0], all[all.size() / 10], all[all.size() / 2], all[all.size() * 9 / 10], all.back());
  printf("slots faster from smid < %d: %d of %d\n", sms / 2, lo_near, K);
  std::vector<double> d(diff);
  std::sort(d.begin(), d.end());
  printf("per-slot mean latency difference (low-smid half minus high half): min %.0f p25 %.0f median %.0f p75 %.0f max %.0f\n",
         d[0], d[K / 4], d[K / 2], d[3 * K / 4], d[K - 1]);
  printf("first 32 slots' differences:");
  for (int k = 0; k < 32; ++k) printf(" %.0f", diff[k]);
  printf("\n");
  // one SM's latencies for the first 32 slots, low and high smid
  for (int c = 0; c < sms; ++c)
    if (sm[c] == 0 || sm[c] == sms - 1) {
      printf("smid %3d:", sm[c]);
      for (int k = 0; k < 32; ++k) printf(" %d", h[(size_t)c * K + k]);
      printf("\n");
    }
  return 0;
}
