// Predictor binning on the GPU (reference bforge/grid.py).
//
//   minmax    per-column min / max of the raw (n, p) matrix: the range a
//             uniform grid spans (build_grid_uniform, grid.py:77-95); exact
//             (min/max do not round), so the host computes the identical
//             cutpoints lo + (hi - lo) * k / (K + 1) from them
//   quantize  value -> number of cutpoints <= value (grid.py:121-134,
//             np.searchsorted(side="right")): a branchless binary search over
//             the axis's sorted cutpoints; f64 comparisons, bit-exact
//
// Both stream X once (HBM-bound: 8 B read per element, 1 B written).
#include <cfloat>

#include "common.cuh"
#include "internal.h"

namespace bart {

// double -> int64 whose signed order is the double order (negatives: flip all
// but the sign bit), so min/max combine with integer atomics, order-free
__device__ __forceinline__ long long ord_key(double v) {
  const long long b = __double_as_longlong(v);
  return b >= 0 ? b : (b ^ 0x7fffffffffffffffll);
}
__device__ __forceinline__ double ord_val(long long k) {
  return __longlong_as_double(k >= 0 ? k : (k ^ 0x7fffffffffffffffll));
}

// keys[0..p) = min, keys[p..2p) = max (initialised to LLONG_MAX / LLONG_MIN);
// *bad counts non-finite values (the reference raises, grid.py:_ranges)
__global__ void minmax_kernel(const double *__restrict__ X, int64_t n, int p, int64_t rows_per_block,
                              long long *__restrict__ keys, unsigned long long *__restrict__ bad) {
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = r0 + rows_per_block < n ? r0 + rows_per_block : n;
  for (int a = threadIdx.x; a < p; a += blockDim.x) {
    double mn = DBL_MAX, mx = -DBL_MAX;
    unsigned long long nb = 0;
    for (int64_t i = r0; i < r1; ++i) {
      const double v = X[i * p + a];
      nb += isfinite(v) ? 0ull : 1ull;
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    }
    if (r1 > r0) {
      atomicMin(keys + a, ord_key(mn));
      atomicMax(keys + p + a, ord_key(mx));
    }
    if (nb) atomicAdd(bad, nb);
  }
}

__global__ void minmax_decode_kernel(const long long *__restrict__ keys, int p, double *__restrict__ lo,
                                     double *__restrict__ hi) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= p) return;
  lo[a] = ord_val(keys[a]);
  hi[a] = ord_val(keys[p + a]);
}

__global__ void quantize_kernel(const double *__restrict__ X, int64_t total, int p, const double *__restrict__ cuts,
                                const int64_t *__restrict__ off, uint8_t *__restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int a = (int)(e % p);
  const double v = X[e];
  const double *c = cuts + off[a];
  int hi = (int)(off[a + 1] - off[a]);  // count of cutpoints <= v, in [0, hi]
  int lo = 0;
  if (v != v) lo = hi;  // NaN sorts after every cutpoint (np.searchsorted side="right", grid.py:127-128)
  while (lo < hi) {  // first index with c[idx] > v
    const int mid = (lo + hi) >> 1;
    if (__ldg(c + mid) <= v)
      lo = mid + 1;
    else
      hi = mid;
  }
  out[e] = (uint8_t)lo;
}

__global__ void minmax_init_kernel(long long *keys, int p, unsigned long long *bad) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a < p) {
    keys[a] = 0x7fffffffffffffffll;
    keys[p + a] = (long long)0x8000000000000000ull;
  }
  if (a == 0) *bad = 0ull;
}

// keys: scratch of 2p int64; bad: one u64
void launch_minmax(const double *X, int64_t n, int p, long long *keys, unsigned long long *bad, double *lo, double *hi,
                   cudaStream_t s) {
  const int64_t rpb = 64;
  minmax_init_kernel<<<(p + 127) / 128, 128, 0, s>>>(keys, p, bad);
  minmax_kernel<<<(unsigned)((n + rpb - 1) / rpb), 128, 0, s>>>(X, n, p, rpb, keys, bad);
  minmax_decode_kernel<<<(p + 127) / 128, 128, 0, s>>>(keys, p, lo, hi);
}

void launch_quantize(const double *X, int64_t n, int p, const double *cuts, const int64_t *off, uint8_t *out,
                     cudaStream_t s) {
  const int64_t total = n * p;
  if (total <= 0) return;
  quantize_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(X, total, p, cuts, off, out);
}

}  // namespace bart
