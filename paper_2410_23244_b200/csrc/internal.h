// Host-side launchers shared between the CUDA translation units.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace bart {

void launch_propose(const ChainDev &c, int device_rng, cudaStream_t s);
// the step's Philox4x32-10 (common.cuh) on explicit counters/keys: known-answer tests
void launch_philox(const uint32_t *ctr, const uint32_t *key, uint32_t *out, int64_t count, cudaStream_t s);
size_t sweep_smem_bytes(int m, int chunk, int size, bool stream, bool hier);
cudaError_t sweep_prepare(size_t smem);
int sweep_max_ctas(size_t smem, int device, int chunk, bool stream);
int sweep_words_per_thread(int chunk);
int sweep_launch(const ChainDev &c, size_t smem, cudaStream_t s);

void launch_transpose_u8(const uint8_t *src, int64_t rows, int64_t cols, int64_t src_ld, uint8_t *dst,
                         int64_t dst_ld, cudaStream_t s);
void launch_fill_root(uint8_t *L, int m, int64_t n, int64_t n_pad, cudaStream_t s);
void launch_traverse(const uint8_t *Xt, int64_t n, int64_t ld, int D, int half, int m, const uint16_t *axis,
                     const uint8_t *cut, uint8_t *L, cudaStream_t s);
void launch_predict_cached(const uint8_t *L, int64_t n, int64_t ld, int m, int size, const float *leaf,
                           double *out, cudaStream_t s);
void launch_evaluate(const uint8_t *Xt, int64_t n, int64_t ld, int D, int half, int m, const uint16_t *axis,
                     const uint8_t *cut, const float *leaf, double *out, cudaStream_t s);
// n_forests stacked forests (F, m, ...) evaluated at once (grid y = forest), out (F, n)
void launch_evaluate_batch(const uint8_t *Xt, int64_t n, int64_t ld, int D, int half, int m, int n_forests,
                           const uint16_t *axis, const uint8_t *cut, const float *leaf, double *out, cudaStream_t s);
void launch_resid(const float *y, const double *pred, float *r, int64_t n, cudaStream_t s);
void launch_trace_train(const uint8_t *L, int64_t n, int64_t ld, int m, int size, const float *leaf, int64_t k,
                        double *mean, double *m2, double *draw, double *pts, int npts, cudaStream_t s);
void launch_mean_leaves(const uint8_t *cut, int m, int half, double *out, cudaStream_t s);
void launch_minmax(const double *X, int64_t n, int p, long long *keys, unsigned long long *bad, double *lo, double *hi,
                   cudaStream_t s);
void launch_quantize(const double *X, int64_t n, int p, const double *cuts, const int64_t *off, uint8_t *out,
                     cudaStream_t s);

}  // namespace bart
