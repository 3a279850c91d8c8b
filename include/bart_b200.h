/*
 * bart_b200.h — C ABI of the B200-native BART MCMC step.
 *
 * The reference (`bforge`, /root/reference/pkg/src/bforge) is pure Python and
 * has no FFI layer; its hot-path boundary is the Python pair
 *     init_state(X, max_cuts, y, hp, rng, sigma2=None) -> SamplerState   (sampler.py:201-241)
 *     step(state, hp, rng=None) -> SamplerState                           (sampler.py:878-912)
 * plus the forest kernels traverse_forest / sum_leaf_values / evaluate_forest
 * (trees.py:174-223).  Each entry point below names the reference function it
 * replaces.  Plain pointers and sizes only: host arrays in the reference's own
 * layouts ((n,p) X, (n,m) leaf index, (m,2^(D-1)) axis/cutpoint, (m,2^D) leaf
 * values); the library owns all device memory.  A ctypes binding is in
 * INTEGRATION.md and paper_2410_23244_b200/_native.py.
 *
 * Errors: every function returns BART_OK (0) or a status code; the message of
 * the last failure on the calling thread is returned by bart_last_error().
 * BART_EINVAL maps to the reference's ValueError (shape/config checks,
 * sampler.py:214-217, trees.py:63-67), BART_ECUDA / BART_ESTATE / BART_ERANGE to
 * RuntimeError.
 * Threading: one writer per handle; handles are independent.
 */
#ifndef BART_B200_H
#define BART_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BART_OK 0
#define BART_EINVAL 1
#define BART_ECUDA 2
#define BART_ESTATE 3
/* The step's cross-CTA exchange met a non-finite value or one outside its
 * exact fixed-point range (per-CTA partial >= 2^46 / CTAs, e.g. an
 * unstandardised y with sum(r^2) ~ 1e14, or a NaN residual).  Sticky: the
 * chain's state is no longer the reference's; every later call that syncs
 * returns it until bart_set_state resets the chain. */
#define BART_ERANGE 4

#define BART_MAX_DEPTH 8 /* trees.py:27-28: leaf heap index fits one byte */

typedef struct bart_chain bart_chain; /* one chain (or one n-shard of it) on one device */

typedef struct {
  int64_t n;         /* points held by this handle */
  int32_t p;         /* predictors (axes) */
  int32_t m;         /* trees */
  int32_t max_depth; /* D in [1, 8] */
  int32_t _pad;
} bart_dims;

/* sampler.Hyperparams (sampler.py:62-104).  depth_prob[d] = alpha/(1+d)**beta
 * with depth_prob[D-1] = 0, computed by the host exactly as sampler.py:107-113. */
typedef struct {
  double leaf_sd, lam, alpha, beta, leaf_mean, nu, p_grow;
  int32_t update_sigma;
  int32_t _pad;
  double depth_prob[BART_MAX_DEPTH];
} bart_hparams;

/* sampler.StepRandoms (sampler.py:244-260), host pointers. */
typedef struct {
  const double *move_u;   /* (m, 5): move coin, leaf, axis, cut, prune picks */
  const double *accept_u; /* (m,) */
  const double *leaf_z;   /* (m, 2^D) */
  double chi2;
} bart_randoms;

/* Number of int64 rows written by bart_get_proposals (sampler.Proposals,
 * sampler.py:286-306): kind, node, axis, cut, depth, n_axes, n_splits,
 * w_small, w_prime_big, growable_big, left_child_growable, right_child_growable. */
#define BART_PROPOSAL_ROWS 12

/* ---- chain lifecycle (replaces sampler.init_state, sampler.py:201-241) ---- */

/* Root-only zero forest, leaf index == 1, resid = y (sampler.py:218-241).
 * X is (n, p) row-major uint8 grid indices; max_cuts (p,) <= 255; y (n,) f32.
 * seed keys the on-device Philox stream used when bart_step gets no randoms. */
int bart_create(const bart_dims *dims, const bart_hparams *hp, const uint8_t *X,
                const int64_t *max_cuts, const float *y, double sigma2, uint64_t seed,
                int device, bart_chain **out);
/* Multi-chain batching: the same, with the chain's sweep
 * limited to max_ctas CTAs (= SMs; 0: no limit), so several chains, each on
 * its own stream, co-run on one GPU instead of taking turns. */
int bart_device_sms(int device); /* SM count (-1 without a device) */
int bart_create_ex(const bart_dims *dims, const bart_hparams *hp, const uint8_t *X, const int64_t *max_cuts,
                   const float *y, double sigma2, uint64_t seed, int device, int max_ctas, bart_chain **out);
int bart_destroy(bart_chain *h);

/* ---- n-sharding across GPUs (the reference has none: PAPER.md:405-409) ----
 * One process per GPU holds the contiguous points [offset, offset + dims->n) of
 * a chain of n_total points; forest, proposals and random draws are replicated
 * (seed identical on every shard), so every shard takes identical decisions.
 * The per-tree leaf statistics travel inside the sweep kernel: each shard adds
 * its fixed-point partials into every shard's exchange words over NVLink
 * (peer-mapped with CUDA IPC) and polls its own copy.  Protocol:
 *   bart_create_shard on every rank -> bart_shard_export -> all-gather the
 *   handles (any host transport, e.g. torch.distributed) -> bart_shard_connect
 *   with the n_shards handles in shard order -> bart_step / bart_run. */
#define BART_SHARD_HANDLE_BYTES 256
int bart_create_shard(const bart_dims *dims /* n = this shard's points */, int64_t n_total, int shard,
                      int n_shards, const bart_hparams *hp, const uint8_t *X, const int64_t *max_cuts,
                      const float *y, double sigma2, uint64_t seed, int device, bart_chain **out);
int bart_shard_export(bart_chain *h, void *out /* BART_SHARD_HANDLE_BYTES */);
int bart_shard_connect(bart_chain *h, const void *all /* n_shards * BART_SHARD_HANDLE_BYTES, shard order */);
/* Test hook: emulate `groups` shards inside one launch on one device (CTA c
 * polls copy c % groups; every CTA adds into every copy). */
int bart_set_copy_groups(bart_chain *h, int groups);
/* Cross-CTA / cross-shard exchange of the per-tree leaf sums and counts.
 * FLAT: every CTA of every shard adds into every shard's words (n_shards x CTAs
 * arrivals per word).  TWO_LEVEL: CTAs add into their own shard's stage words;
 * one forwarder CTA per shard adds the shard's total into every shard's words
 * (n_shards arrivals per word, one remote add per shard).  Totals, hence every
 * decision, are bit-identical between the two.  Set between steps. */
#define BART_EXCHANGE_FLAT 0
#define BART_EXCHANGE_TWO_LEVEL 1
int bart_set_exchange(bart_chain *h, int mode);

/* Direct state edit + SamplerState.rebuild_structure_caches (sampler.py:157-168,
 * tests/util.py:11-24).  axis (m, 2^(D-1)) as uint16; leaf_index (n, m) or NULL
 * (then recomputed by traversal); resid (n,) or NULL (then y - forest in f64,
 * cast to f32).  sigma2 < 0 keeps the current value. */
int bart_set_state(bart_chain *h, const uint16_t *axis, const uint8_t *cutpoint,
                   const float *leaf_value, const uint8_t *leaf_index, const float *resid,
                   double sigma2);
int bart_set_hparams(bart_chain *h, const bart_hparams *hp);
int bart_set_sigma2(bart_chain *h, double sigma2);

/* ---- the hot path (replaces sampler.step, sampler.py:878-912) ----
 * randoms != NULL: use the caller's StepRandoms (parity mode, bit-compatible
 * with the reference's Generator stream).  randoms == NULL: draw them on the
 * device from counter-based Philox4x32-10 keyed by (seed, iteration). */
int bart_step(bart_chain *h, const bart_randoms *randoms);
/* Phase 1 alone (sampler.propose_moves, sampler.py:469-526): proposals for the
 * current forest from the given (m, 5) uniforms; the state is not changed.
 * Read them with bart_get_proposals. */
int bart_propose(bart_chain *h, const double *move_u);
/* n_iter device-RNG iterations, replayed from a captured CUDA graph. Async. */
int bart_run(bart_chain *h, int64_t n_iter);
int bart_sync(bart_chain *h);

/* ---- state readback (reference layouts) ---- */
int bart_get_forest(bart_chain *h, uint16_t *axis, uint8_t *cutpoint, float *leaf_value);
int bart_get_leaf_index(bart_chain *h, uint8_t *out_nm); /* (n, m) */
int bart_get_resid(bart_chain *h, float *out);
int bart_get_sigma2(bart_chain *h, double *out);
int bart_get_accepted(bart_chain *h, uint8_t *out); /* last_accepted (m,) */
/* last_accepted (m,) and sigma2 after the last step in one synchronisation
 * (either pointer may be NULL): the per-step read of the end-to-end loop */
int bart_get_step_result(bart_chain *h, uint8_t *accepted, double *sigma2);
/* The result (accept flags, sigma2) of bart_step number `iteration` (0-based),
 * for either of the last two steps: every bart_step enqueues a copy of its
 * result into pinned memory behind the step, so a caller can launch step k+1
 * (and draw its randoms on the host meanwhile) before reading step k. */
int bart_read_step_result(bart_chain *h, int64_t iteration, uint8_t *accepted, double *sigma2);
int bart_get_proposals(bart_chain *h, int64_t *rows /* (12, m) */, double *struct_log /* (m,) */);
/* The StepRandoms block (sampler.py:244-260 layout) the latest step consumed:
 * the injected one, or the one drawn on the device from Philox4x32-10.  Any
 * pointer may be NULL.  move_u (m,5), accept_u (m,), leaf_z (m,2^D), chi2 (1). */
int bart_get_randoms(bart_chain *h, double *move_u, double *accept_u, double *leaf_z, double *chi2);
/* Test hook: the device Philox4x32-10 bijection of the step (Random123's
 * philox4x32_10) on `count` explicit (counter, key) pairs: ctr (count,4),
 * key (count,2), out (count,4), uint32.  For known-answer tests. */
int bart_philox4x32_10(const uint32_t *ctr, const uint32_t *key, uint32_t *out, int64_t count, int device);
/* Phase taps for parity (enable with bart_set_taps before the step):
 * counts (m, 2^D) after the grow refresh (sampler.py:894-897) and the
 * tree-excluded sums (m, 2^D) each tree resolved with (sampler.py:828). */
int bart_set_taps(bart_chain *h, int on);
int bart_get_taps(bart_chain *h, int64_t *counts, double *sums);
int64_t bart_iteration(bart_chain *h);
/* Resume support (checkpoints): set the iteration counter, which is also the
 * device random stream's Philox counter, so a restored chain continues the
 * stream it was saved from. */
int bart_set_iteration(bart_chain *h, int64_t iteration);
/* Tracing: per-tree phase stamps (clock64) of the last sweep, (m+2) rows of 32 (buffer 4*(m+2)*8 words):
 * [0] CTA 0 and [1] last CTA: start, data-ready, pass-done, block-reduced, -,
 * gathered, gathered-synced, decided; [2] CTA 0 stamps inside the decision. */
int bart_set_timeline(bart_chain *h, int on);
int bart_get_timeline(bart_chain *h, int64_t *out);
/* globaltimer (ns) of every CTA's partial publish and gather completion per
 * exchange of the last sweep: (m+1, ctas, 2). */
int bart_get_trace(bart_chain *h, int64_t *out);

/* ---- fit() trace kept on the device (regression.fit's chain loop, regression.py:183-201) ----
 * Instead of reading last_accepted / sigma2 / predictions back after every
 * iteration, the sweep writes each iteration's accept flags and sigma2 into
 * device history rows, and bart_trace_keep records a kept draw
 * asynchronously: per-point running mean/variance of the training-row sum of
 * trees (Welford, f64), optionally the whole draw, the draw at the first
 * BART_TRACE_POINTS rows (cross-chain diagnostics), test-row predictions,
 * sigma2, mean leaves per tree, and the forest.  One read at the end. */
#define BART_TRACE_POINTS 8
typedef struct {
  int64_t n_iter, n_keep, n_test;  /* capacities; n_test rows of X_test */
  int32_t store_train_draws, store_forests;
  /* training-row draws kept on the device: 0 = all n_keep; else a ring of
   * train_ring rows (kept draw k in row k % train_ring), drained by the
   * caller with bart_trace_read_draws before it is overwritten -- a streamed
   * trace file then needs train_ring * n * 8 B of device memory, not n_keep * n * 8 */
  int64_t train_ring;
} bart_trace_opts;
int bart_trace_begin(bart_chain *h, const bart_trace_opts *opts, const uint8_t *X_test /* (n_test, p) or NULL */);
int bart_trace_keep(bart_chain *h);
int bart_trace_counts(bart_chain *h, int64_t *n_iter, int64_t *n_keep);
/* any pointer may be NULL; shapes: accepted (n_iter, m), sigma2_iter (n_iter), sigma2_keep (n_keep),
 * train_mean/var (n), train_draws (n_keep, n), train_points (n_keep, min(n, 8)), test_draws (n_keep, n_test),
 * mean_leaves (n_keep), axis/cutpoint (n_keep, m, 2^(D-1)), leaf_value (n_keep, m, 2^D) */
int bart_trace_read(bart_chain *h, uint8_t *accepted, double *sigma2_iter, double *sigma2_keep, double *train_mean,
                    double *train_var, double *train_draws, double *train_points, double *test_draws,
                    double *mean_leaves, uint16_t *axis, uint8_t *cutpoint, float *leaf_value);
/* kept draws [k0, k1) only: train (k1-k0, n) / test (k1-k0, n_test), either NULL
 * (streams a BFTRACE1 file from the device without one host array of every draw);
 * with a train ring, [k0, k1) must still be in it (k0 >= kept - train_ring) */
int bart_trace_read_draws(bart_chain *h, int64_t k0, int64_t k1, double *train, double *test);
int bart_trace_end(bart_chain *h);

/* ---- predictions (trees.sum_leaf_values / evaluate_forest, trees.py:206-223) ---- */
/* sum of trees from the cached leaf index, f64 in tree order: (n,) */
int bart_predict_cached(bart_chain *h, double *out);
/* evaluate the chain's current forest on a new (n_new, p) matrix */
int bart_predict_matrix(bart_chain *h, const uint8_t *X, int64_t n_new, double *out);

/* ---- stateless forest kernels (trees.traverse_forest, trees.py:174-203) ---- */
int bart_traverse(const bart_dims *dims, const uint16_t *axis, const uint8_t *cutpoint,
                  const uint8_t *X, uint8_t *out_nm, int device);
int bart_evaluate(const bart_dims *dims, const uint16_t *axis, const uint8_t *cutpoint,
                  const float *leaf_value, const uint8_t *X, double *out, int device);
/* n_forests forests stacked (F, m, ...) on one (n, p) matrix: out (F, n)
 * (regression.predict over kept forests, regression.py:252-258). */
int bart_evaluate_many(const bart_dims *dims, int64_t n_forests, const uint16_t *axis, const uint8_t *cutpoint,
                       const float *leaf_value, const uint8_t *X, double *out, int device);
/* trees.sum_leaf_values (trees.py:206-218) on host arrays: leaf (m, 2^D), L (n, m) */
int bart_sum_leaf_values(const bart_dims *dims, const float *leaf_value, const uint8_t *leaf_index_nm,
                         double *out, int device);

/* ---- measurement hooks used by bench.py ---- */
/* Runs n_iter device-RNG iterations with CUDA events on the chain's stream:
 * ms[0] = total elapsed, ms[1] = summed sweep-kernel time, ms[2] = summed
 * propose-kernel time (per-launch events, not graph-replayed). */
int bart_profile(bart_chain *h, int64_t n_iter, float *ms);
/* Per-launch time (ms, CUDA events on the chain's stream, `reps` back-to-back
 * launches after a warm-up) of the forest kernels on the chain's own state:
 * ms[0] traverse (trees.traverse_forest into a scratch cache), ms[1] cached
 * sum of trees (trees.sum_leaf_values), ms[2] fused traverse + sum
 * (trees.evaluate_forest). */
int bart_profile_forest(bart_chain *h, int reps, float *ms);
/* n_iter graph-replayed device-RNG iterations bracketed by CUDA events on the
 * chain's stream (synchronised on both sides); *ms = elapsed. */
int bart_run_timed(bart_chain *h, int64_t n_iter, float *ms);
/* kernels this library launched on the handle since creation */
int64_t bart_kernel_launches(bart_chain *h);
/* 1 if bart_run replays a captured CUDA graph, 0 if it falls back to launches */
int bart_graph_active(bart_chain *h);
int bart_sweep_config(bart_chain *h, int32_t *out /* [ctas, threads, chunk, smem_bytes, stream] */);

/* ---- binning (bforge/grid.py) ----
 * column min / max of the raw (n, p) row-major f64 matrix (the span of
 * build_grid_uniform, grid.py:77-95; EINVAL on non-finite values), and
 * quantize (grid.py:121-134): out[i, a] = #{cutpoints of axis a <= X[i, a]}
 * (np.searchsorted side="right"), cutpoints of axis a at
 * cutpoints[offsets[a] .. offsets[a+1]), <= 255 per axis. */
int bart_grid_minmax(const double *X, int64_t n, int32_t p, double *lo, double *hi, int device);
int bart_quantize(const double *X, int64_t n, int32_t p, const double *cutpoints, const int64_t *offsets,
                  uint8_t *out, int device);
/* both for a uniform grid with X uploaded once (regression.fit's binning,
 * regression.py:136 -> grid.py:77-95 + 121-134): lo / hi as bart_grid_minmax,
 * the cutpoints lo + (hi - lo) * (k / (n_cutpoints + 1)), k = 1..n_cutpoints
 * (none where lo == hi), and out as bart_quantize with them. */
int bart_grid_uniform_quantize(const double *X, int64_t n, int32_t p, int32_t n_cutpoints, double *lo, double *hi,
                               uint8_t *out, int device);

const char *bart_last_error(void);
const char *bart_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BART_B200_H */
