// C ABI (include/bart_b200.h): chain handles, host<->device layout changes,
// step orchestration (propose kernel + persistent sweep, optionally replayed
// from a CUDA graph), readback taps and measurement hooks.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/bart_b200.h"
#include "common.cuh"
#include "internal.h"

using namespace bart;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                              \
  do {                                                                                              \
    cudaError_t e_ = (expr);                                                                        \
    if (e_ != cudaSuccess) return fail(BART_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <typename T>
cudaError_t dalloc(T **p, size_t count) {
  return cudaMalloc(reinterpret_cast<void **>(p), count * sizeof(T) > 0 ? count * sizeof(T) : 16);
}

struct DevBuf {  // scoped temporary device buffer
  void *p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 16); }
  template <typename T>
  T *as() {
    return reinterpret_cast<T *>(p);
  }
};

int64_t round16(int64_t v) { return (v + 15) & ~int64_t(15); }

constexpr const char *kRangeMsg =
    "the step's exchange met a NaN/inf or a per-CTA partial outside its exact fixed-point range "
    "(|partial| < 2^46 / CTAs; e.g. an unstandardised y whose sum of squared residuals exceeds ~1e11 "
    "per SM, or a non-finite residual): the chain state is invalid; reset it with set_state";

int check_dims(const bart_dims *d) {
  if (!d) return fail(BART_EINVAL, "dims is NULL");
  if (d->max_depth < 1 || d->max_depth > BART_MAX_DEPTH)
    return fail(BART_EINVAL, "max_depth must be in [1, 8], got " + std::to_string(d->max_depth));
  if (d->m < 1) return fail(BART_EINVAL, "n_trees must be >= 1, got " + std::to_string(d->m));
  if (d->n < 1) return fail(BART_EINVAL, "need at least one point");
  if (d->p < 1 || d->p > 65536) return fail(BART_EINVAL, "p must be in [1, 65536]");
  return BART_OK;
}

HP to_hp(const bart_hparams *h) {
  HP o;
  o.leaf_sd = h->leaf_sd;
  o.lam = h->lam;
  o.alpha = h->alpha;
  o.beta = h->beta;
  o.leaf_mean = h->leaf_mean;
  o.nu = h->nu;
  o.p_grow = h->p_grow;
  o.update_sigma = h->update_sigma;
  for (int i = 0; i < kMaxDepth; ++i) o.depth_prob[i] = h->depth_prob[i];
  return o;
}

}  // namespace

struct TraceState {  // fit() trace kept on the device (bart_trace_begin)
  bool on = false;
  int64_t iter_cap = 0, keep_cap = 0, n_test = 0, ld_test = 0, iter0 = 0, kept = 0;
  int64_t train_rows = 0;  // device rows of training-row draws: keep_cap, or the ring size
  int store_train = 0, store_forests = 0, npts = 0;
  uint8_t *acc = nullptr, *Xt_test = nullptr, *f_cut = nullptr;
  uint16_t *f_axis = nullptr;
  float *f_leaf = nullptr;
  double *sig_iter = nullptr, *sig_keep = nullptr, *mean = nullptr, *m2 = nullptr, *train = nullptr, *pts = nullptr,
         *test = nullptr, *mleaves = nullptr;
  std::vector<void *> bufs;
};

struct bart_chain {
  int device = 0;
  cudaStream_t stream = nullptr;
  ChainDev c{};
  size_t smem = 0;
  int64_t iteration = 0;
  int64_t launches = 0;
  bool taps_on = false;
  long long *timeline_buf = nullptr;
  long long *trace_buf = nullptr;
  cudaGraphExec_t graph = nullptr;
  bool graph_failed = false;
  std::vector<void *> owned;
  std::vector<void *> ipc_opened;  // peer shards' exchange buffers (cudaIpcOpenMemHandle)
  bool shard_pending = false;      // created as a shard, not yet connected
  TraceState tr;
  uint8_t *result_stage = nullptr;  // pinned: last_accepted (m) + sigma2
  // bart_step pipeline, two slots (slot = iteration % 2): the injected random
  // block is written into the slot's pinned stage, which the step kernel
  // reads directly (zero-copy) while the host prepares the next step; the
  // kernel writes the step's accept flags, sigma2 draw and error flag straight
  // into the slot's pinned step_out, so the host reads step k after launching
  // step k+1 -- no copy engine, no second stream, no cross-stream event.
  double *rstage[2] = {nullptr, nullptr};
  double *rblock[2] = {nullptr, nullptr};
  uint8_t *acc_base = nullptr;  // the chain's device result buffers (bart_run's graph writes them)
  double *sdraw_base = nullptr;
  uint8_t *res_acc = nullptr;  // where the latest step's accept flags are
  double *res_sdraw = nullptr;
  double *res_block = nullptr;  // the random block (StepRandoms) the latest step consumed
  uint8_t *step_out = nullptr;
  cudaEvent_t kernel_done[2] = {nullptr, nullptr};
  bool update_sigma = true;
  cudaGraphExec_t graph_step[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [slot][injected randoms]
  int64_t slot_iter[2] = {-1, -1};  // which iteration each result slot holds
};

namespace {

void drop_graphs(bart_chain *h) {
  if (h->graph) cudaGraphExecDestroy(h->graph);
  h->graph = nullptr;
  for (auto &row : h->graph_step)
    for (auto &g : row) {
      if (g) cudaGraphExecDestroy(g);
      g = nullptr;
    }
}

void free_chain(bart_chain *h) {
  if (!h) return;
  cudaSetDevice(h->device);
  drop_graphs(h);
  for (void *p : h->tr.bufs) cudaFree(p);
  for (void *p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  for (void *p : h->owned)
    if (p) cudaFree(p);
  if (h->stream) cudaStreamSynchronize(h->stream);
  // a stream-mode chain pinned its residuals in L2: release the persisting lines
  if (h->c.persist_bytes > 0) cudaCtxResetPersistingL2Cache();
  for (auto *p : h->rstage)
    if (p) cudaFreeHost(p);
  if (h->result_stage) cudaFreeHost(h->result_stage);
  if (h->step_out) cudaFreeHost(h->step_out);
  for (int k = 0; k < 2; ++k) {
    if (h->kernel_done[k]) cudaEventDestroy(h->kernel_done[k]);
  }
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

template <typename T>
cudaError_t own(bart_chain *h, T **p, size_t count) {
  cudaError_t e = dalloc(p, count);
  if (e == cudaSuccess) {
    h->owned.push_back(*p);
    e = cudaMemsetAsync(*p, 0, count * sizeof(T) > 0 ? count * sizeof(T) : 16, h->stream);
  }
  return e;
}

// One iteration = ONE launch: the sweep kernel proposes every tree first
// (injected or device randoms), then sweeps.
ChainDev step_args(const bart_chain *h, int device_rng) {
  ChainDev c = h->c;
  c.propose_in_sweep = device_rng ? 1 : 2;
  return c;
}

int launch_iteration(bart_chain *h, int device_rng) {
  CUDA_TRY((cudaError_t)sweep_launch(step_args(h, device_rng), h->smem, h->stream));
  h->launches += 1;
  h->iteration += 1;
  return BART_OK;
}

int ensure_graph(bart_chain *h) {
  if (h->graph || h->graph_failed) return BART_OK;
  cudaGraph_t g = nullptr;
  if (cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    h->graph_failed = true;
    cudaGetLastError();
    return BART_OK;
  }
  cudaError_t e1 = cudaGetLastError();
  cudaError_t e2 = (cudaError_t)sweep_launch(step_args(h, 1), h->smem, h->stream);
  cudaError_t e3 = cudaStreamEndCapture(h->stream, &g);
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess || !g ||
      cudaGraphInstantiate(&h->graph, g, 0) != cudaSuccess) {
    h->graph = nullptr;
    h->graph_failed = true;
    cudaGetLastError();
  }
  if (g) cudaGraphDestroy(g);
  return BART_OK;
}

}  // namespace

// ---- fit() trace on the device ----
namespace {
void trace_free(bart_chain *h) {
  for (void *p : h->tr.bufs) cudaFree(p);
  h->tr = TraceState{};
  h->c.acc_hist = nullptr;
  h->c.sig_hist = nullptr;
  h->c.hist_cap = 0;
  drop_graphs(h);  // captured launches carry the chain parameters
}
template <typename T>
cudaError_t trace_alloc(bart_chain *h, T **p, size_t count) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void **>(p), count * sizeof(T) > 0 ? count * sizeof(T) : 16);
  if (e == cudaSuccess) {
    h->tr.bufs.push_back(*p);
    e = cudaMemsetAsync(*p, 0, count * sizeof(T) > 0 ? count * sizeof(T) : 16, h->stream);
  }
  return e;
}
}  // namespace

extern "C" {

const char *bart_last_error(void) { return g_err.c_str(); }
const char *bart_version(void) { return "bart_b200 0.1 sm_100a"; }

static int create_impl(const bart_dims *dims, int64_t n_total, int shard, int n_shards, const bart_hparams *hp,
                       const uint8_t *X, const int64_t *max_cuts, const float *y, double sigma2, uint64_t seed,
                       int device, bart_chain **out, int max_ctas = 0) {
  if (int rc = check_dims(dims)) return rc;
  if (n_shards < 1 || n_shards > kMaxShards || shard < 0 || shard >= n_shards)
    return fail(BART_EINVAL, "shard must be in [0, n_shards), n_shards in [1, " + std::to_string(kMaxShards) + "]");
  if (n_total < dims->n) return fail(BART_EINVAL, "n_total < points of this shard");
  if (!hp || !X || !max_cuts || !y || !out) return fail(BART_EINVAL, "NULL argument");
  for (int a = 0; a < dims->p; ++a)
    if (max_cuts[a] < 0 || max_cuts[a] > 255)
      return fail(BART_EINVAL, "max_cuts must be in [0, 255] (grid.py:18)");
  CUDA_TRY(cudaSetDevice(device));
  bart_chain *h = new bart_chain();
  h->device = device;
  auto bail = [&](int rc) {
    free_chain(h);
    return rc;
  };
  if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(BART_ECUDA, "cudaStreamCreate failed"));

  ChainDev &c = h->c;
  c.n = dims->n;
  c.n_pad = round16(dims->n);
  c.p = dims->p;
  c.m = dims->m;
  c.D = dims->max_depth;
  c.half = 1 << (c.D - 1);
  c.size = 1 << c.D;
  c.hp = to_hp(hp);
  c.seed = seed;
  if (const char *dbg = getenv("BART_DBG")) c.dbg = atoi(dbg);

  // sweep geometry: one CTA per SM, contiguous 16-aligned chunks
  int sms = 0, optin = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  int64_t want = (c.n + 1023) / 1024;
  int nblk = (int)(want < sms ? (want > 0 ? want : 1) : sms);
  if (nblk > kMaxCtas) nblk = kMaxCtas;
  if (max_ctas > 0 && nblk > max_ctas) nblk = max_ctas;  // multi-chain batching: leave SMs to other chains
  int64_t chunk = round16((c.n + nblk - 1) / nblk);
  nblk = (int)((c.n + chunk - 1) / chunk);
  c.nblk = nblk;
  c.chunk = (int)chunk;
  // register mode while the chunk fits the workers' registers, else stream
  // mode (residuals in global memory / L2, refreshed rows in Lref)
  c.stream = sweep_words_per_thread(c.chunk) == 0 ? 1 : 0;
  if (const char *fs = getenv("BART_FORCE_STREAM")) c.stream |= atoi(fs) != 0;  // tests: stream mode at small n
  c.persist_bytes = 0;
  if (c.stream) {  // L2 set-aside for the residuals (stream mode's persisting window, sweep_launch)
    int max_persist = 0, max_window = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device);
    size_t want = (size_t)4 * round16(c.n);
    if (want > (size_t)max_window) want = (size_t)max_window;
    if (want > (size_t)max_persist) want = (size_t)max_persist;
    if (want > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) c.persist_bytes = want;
    cudaGetLastError();
  }
  h->smem = sweep_smem_bytes(c.m, c.chunk, c.size, c.stream != 0, false);
  if ((int64_t)h->smem > optin)
    return bail(fail(BART_EINVAL, "sweep needs " + std::to_string(h->smem) + " B shared memory > " +
                                      std::to_string(optin) + " (n_trees too large?)"));
  if (cudaError_t e = sweep_prepare(h->smem); e != cudaSuccess)
    return bail(fail(BART_ECUDA, std::string("sweep_prepare: ") + cudaGetErrorString(e)));
  const int maxc = sweep_max_ctas(h->smem, device, c.chunk, c.stream != 0);
  if (maxc < nblk) return bail(fail(BART_ECUDA, "sweep grid cannot be co-resident"));

  const size_t np = (size_t)c.n_pad;
  uint8_t *Xt = nullptr, *L = nullptr, *cut = nullptr, *acc = nullptr;
  float *r = nullptr, *yy = nullptr, *leaf = nullptr;
  uint16_t *axis = nullptr;
  int32_t *mc = nullptr;
  uint32_t *ob = nullptr;
  uint8_t *recs = nullptr;
  TreeHdr *hdr = nullptr;
  double *rm = nullptr, *ra = nullptr, *rz = nullptr, *rc2 = nullptr, *s2 = nullptr, *s2d = nullptr;
  unsigned long long *xacc = nullptr, *itd = nullptr, *xsnap = nullptr;
  int *errf = nullptr;
  unsigned long long *cacc = nullptr, *csnap = nullptr;
  cudaError_t e = cudaSuccess;
#define OWN(ptr, cnt) \
  if (e == cudaSuccess) e = own(h, &ptr, cnt)
  OWN(Xt, (size_t)c.p * np);
  OWN(L, (size_t)c.m * np);
  uint8_t *Lref = nullptr;
  if (c.stream) OWN(Lref, 3 * np);
  OWN(r, np);
  OWN(yy, np);
  OWN(axis, (size_t)c.m * c.half);
  OWN(cut, (size_t)c.m * c.half);
  OWN(leaf, (size_t)c.m * c.size);
  OWN(mc, (size_t)c.p);
  OWN(ob, (size_t)(c.p + 31) / 32);
  c.rstride = rec_stride(c.size);
  OWN(recs, (size_t)c.m * c.rstride);
  OWN(hdr, (size_t)c.m);
  // one StepRandoms block (move_u | accept_u | leaf_z | chi2), so an injected
  // block is one host->device copy from the pinned staging buffer
  const size_t rwords = (size_t)c.m * 5 + (size_t)c.m + (size_t)c.m * c.size + 1;
  OWN(rm, rwords);
  if (e == cudaSuccess) {
    ra = rm + (size_t)c.m * 5;
    rz = ra + c.m;
    rc2 = rz + (size_t)c.m * c.size;
    h->rblock[0] = rm;
  }
  OWN(s2, 1);
  OWN(s2d, 1);
  OWN(acc, (size_t)c.m);
  OWN(xacc, (size_t)kXSets * kXSetWords);
  OWN(xsnap, 1 + (size_t)kXSets * kXPrevWords);
  OWN(errf, 32);
  OWN(cacc, (size_t)kCSets * kCSetWords);
  OWN(csnap, (size_t)kCSets * kCSetWords);
  OWN(itd, 1);
#undef OWN
  if (e != cudaSuccess) return bail(fail(BART_ECUDA, std::string("allocation: ") + cudaGetErrorString(e)));
  c.Xt = Xt;
  c.L = L;
  c.Lref = Lref;
  c.r = r;
  c.y = yy;
  c.axis = axis;
  c.cut = cut;
  c.leaf = leaf;
  c.max_cuts = mc;
  c.open_bits = ob;
  c.rec = recs;
  c.hdr = hdr;
  c.rand_move = rm;
  c.rand_acc = ra;
  c.rand_z = rz;
  c.rand_chi2 = rc2;
  c.sigma2 = s2;
  c.sigma2_draw = s2d;
  c.accepted = acc;
  h->acc_base = acc;
  h->sdraw_base = s2d;
  h->res_acc = acc;
  h->res_sdraw = s2d;
  h->res_block = rm;
  h->update_sigma = hp->update_sigma != 0;
  c.xacc = xacc;
  c.xpeer[0] = xacc;
  c.n_shards = 1;
  c.nblk_total = c.nblk;
  c.shard_sys = 0;
  c.copy_base = shard;
  c.copy_groups = 1;
  c.n_total = n_total;
  if (n_shards > 1) {  // peers come with bart_shard_connect
    c.n_shards = n_shards;
    c.xpeer[shard] = xacc;
    c.cpeer[shard] = cacc;
    h->shard_pending = true;
  }
  c.xsnap = xsnap;
  c.err = errf;
  c.cacc = cacc;
  c.cpeer[0] = cacc;
  c.csnap = csnap;
  c.iter_dev = itd;

  // predictors: (n, p) row-major -> (p, n_pad)
  {
    DevBuf tmp;
    if (tmp.alloc((size_t)c.n * c.p) != cudaSuccess) return bail(fail(BART_ECUDA, "X staging alloc"));
    if (cudaMemcpyAsync(tmp.p, X, (size_t)c.n * c.p, cudaMemcpyHostToDevice, h->stream) != cudaSuccess)
      return bail(fail(BART_ECUDA, "X upload"));
    launch_transpose_u8(tmp.as<uint8_t>(), c.n, c.p, c.p, Xt, c.n_pad, h->stream);
    if (cudaStreamSynchronize(h->stream) != cudaSuccess) return bail(fail(BART_ECUDA, "X transpose"));
  }
  std::vector<int32_t> mc32(c.p);
  std::vector<uint32_t> bits((c.p + 31) / 32, 0u);
  int popen = 0;
  for (int a = 0; a < c.p; ++a) {
    mc32[a] = (int32_t)max_cuts[a];
    if (max_cuts[a] > 0) {
      bits[a >> 5] |= 1u << (a & 31);
      ++popen;
    }
  }
  c.P_open = popen;
  bool ok = cudaMemcpyAsync(mc, mc32.data(), mc32.size() * 4, cudaMemcpyHostToDevice, h->stream) == cudaSuccess &&
            cudaMemcpyAsync(ob, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice, h->stream) == cudaSuccess &&
            cudaMemcpyAsync(yy, y, (size_t)c.n * 4, cudaMemcpyHostToDevice, h->stream) == cudaSuccess &&
            cudaMemcpyAsync(r, y, (size_t)c.n * 4, cudaMemcpyHostToDevice, h->stream) == cudaSuccess &&
            cudaMemcpyAsync(s2, &sigma2, 8, cudaMemcpyHostToDevice, h->stream) == cudaSuccess;
  if (!ok) return bail(fail(BART_ECUDA, "state upload"));
  launch_fill_root(L, c.m, c.n, c.n_pad, h->stream);
  if (cudaStreamSynchronize(h->stream) != cudaSuccess || cudaGetLastError() != cudaSuccess)
    return bail(fail(BART_ECUDA, "init kernels failed"));
  *out = h;
  return BART_OK;
}

int bart_create(const bart_dims *dims, const bart_hparams *hp, const uint8_t *X, const int64_t *max_cuts,
                const float *y, double sigma2, uint64_t seed, int device, bart_chain **out) {
  return create_impl(dims, dims ? dims->n : 0, 0, 1, hp, X, max_cuts, y, sigma2, seed, device, out);
}

int bart_device_sms(int device) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    fail(BART_ECUDA, "no CUDA device");
    return -1;
  }
  return sms;
}

int bart_create_ex(const bart_dims *dims, const bart_hparams *hp, const uint8_t *X, const int64_t *max_cuts,
                   const float *y, double sigma2, uint64_t seed, int device, int max_ctas, bart_chain **out) {
  if (max_ctas < 0) return fail(BART_EINVAL, "max_ctas must be >= 0");
  return create_impl(dims, dims ? dims->n : 0, 0, 1, hp, X, max_cuts, y, sigma2, seed, device, out, max_ctas);
}

int bart_create_shard(const bart_dims *dims, int64_t n_total, int shard, int n_shards, const bart_hparams *hp,
                      const uint8_t *X, const int64_t *max_cuts, const float *y, double sigma2, uint64_t seed,
                      int device, bart_chain **out) {
  return create_impl(dims, n_total, shard, n_shards, hp, X, max_cuts, y, sigma2, seed, device, out);
}

namespace {
struct ShardHandle {  // what one shard tells the others (bart_shard_export)
  cudaIpcMemHandle_t xacc, cacc;
  int32_t nblk, shard, n_shards, magic;
  int64_t n_local, n_total;
};
static_assert(sizeof(ShardHandle) <= BART_SHARD_HANDLE_BYTES, "handle size");
constexpr int32_t kShardMagic = 0x42415254;  // "BART"
}  // namespace

int bart_shard_export(bart_chain *h, void *out) {
  if (!h || !out) return fail(BART_EINVAL, "NULL argument");
  CUDA_TRY(cudaSetDevice(h->device));
  ShardHandle sh{};
  CUDA_TRY(cudaIpcGetMemHandle(&sh.xacc, h->c.xpeer[h->c.copy_base]));
  CUDA_TRY(cudaIpcGetMemHandle(&sh.cacc, h->c.cpeer[h->c.copy_base]));
  sh.nblk = h->c.nblk;
  sh.shard = h->c.copy_base;
  sh.n_shards = h->c.n_shards;
  sh.magic = kShardMagic;
  sh.n_local = h->c.n;
  sh.n_total = h->c.n_total;
  std::memset(out, 0, BART_SHARD_HANDLE_BYTES);
  std::memcpy(out, &sh, sizeof(sh));
  return BART_OK;
}

int bart_shard_connect(bart_chain *h, const void *all) {
  if (!h || !all) return fail(BART_EINVAL, "NULL argument");
  if (!h->shard_pending) return fail(BART_ESTATE, "not an unconnected shard (bart_create_shard)");
  CUDA_TRY(cudaSetDevice(h->device));
  ChainDev &c = h->c;
  int total = 0;
  int64_t points = 0;
  for (int g = 0; g < c.n_shards; ++g) {
    ShardHandle sh;
    std::memcpy(&sh, static_cast<const uint8_t *>(all) + (size_t)g * BART_SHARD_HANDLE_BYTES, sizeof(sh));
    if (sh.magic != kShardMagic || sh.shard != g || sh.n_shards != c.n_shards || sh.n_total != c.n_total)
      return fail(BART_EINVAL, "shard handle " + std::to_string(g) + " does not belong to this chain");
    total += sh.nblk;
    points += sh.n_local;
    if (g == c.copy_base) continue;
    void *px = nullptr, *pc = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&px, sh.xacc, cudaIpcMemLazyEnablePeerAccess));
    h->ipc_opened.push_back(px);
    CUDA_TRY(cudaIpcOpenMemHandle(&pc, sh.cacc, cudaIpcMemLazyEnablePeerAccess));
    h->ipc_opened.push_back(pc);
    c.xpeer[g] = static_cast<unsigned long long *>(px);
    c.cpeer[g] = static_cast<unsigned long long *>(pc);
  }
  if (points != c.n_total) return fail(BART_EINVAL, "shards cover " + std::to_string(points) + " points, n_total " +
                                                        std::to_string(c.n_total));
  if (total >= 2048) return fail(BART_EINVAL, "too many CTAs over all shards for the exchange tags");
  c.nblk_total = total;
  c.shard_sys = 1;
  h->shard_pending = false;
  drop_graphs(h);  // captured launches carry the chain parameters
  // from 4 shards the flat exchange's arrivals (CTAs x shards per word)
  // outgrow the two-level exchange's extra hop (tools/xshard_bench.cu:
  // 3295 vs 3002 cycles at N=4, 4989 vs 3091 at N=8)
  if (c.n_shards >= 4) return bart_set_exchange(h, BART_EXCHANGE_TWO_LEVEL);
  return BART_OK;
}

int bart_set_copy_groups(bart_chain *h, int groups) {
  if (!h) return fail(BART_EINVAL, "NULL handle");
  ChainDev &c = h->c;
  if (c.n_shards != 1 || h->iteration != 0)
    return fail(BART_ESTATE, "copy groups are set on a fresh, unsharded chain");
  if (groups < 1 || groups > kMaxShards || groups > c.nblk)
    return fail(BART_EINVAL, "groups must be in [1, min(8, CTAs)]");
  CUDA_TRY(cudaSetDevice(h->device));
  for (int g = 1; g < groups; ++g) {
    unsigned long long *x = nullptr, *cc = nullptr;
    CUDA_TRY(own(h, &x, (size_t)kXSets * kXSetWords));
    CUDA_TRY(own(h, &cc, (size_t)kCSets * kCSetWords));
    c.xpeer[g] = x;
    c.cpeer[g] = cc;
  }
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  c.n_shards = groups;
  c.copy_groups = groups;
  c.copy_base = 0;
  drop_graphs(h);  // captured launches carry the chain parameters
  return BART_OK;
}


int bart_set_exchange(bart_chain *h, int mode) {
  if (!h) return fail(BART_EINVAL, "NULL handle");
  if (mode != BART_EXCHANGE_FLAT && mode != BART_EXCHANGE_TWO_LEVEL)
    return fail(BART_EINVAL, "exchange mode must be BART_EXCHANGE_FLAT or BART_EXCHANGE_TWO_LEVEL");
  CUDA_TRY(cudaSetDevice(h->device));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  ChainDev &c = h->c;
  if (mode == BART_EXCHANGE_TWO_LEVEL && !c.xstage) {
    // stage words and forwarder baselines for up to kMaxShards copy groups
    // (one per emulated shard; a real shard uses group 0), zero: a fresh stage
    CUDA_TRY(own(h, &c.xstage, (size_t)kMaxShards * kXSets * kXSetWords));
    CUDA_TRY(own(h, &c.cstage, (size_t)kMaxShards * kCSets * kCSetWords));
    CUDA_TRY(own(h, &c.xssnap, (size_t)kMaxShards * kXSets * kXPrevWords));
    CUDA_TRY(own(h, &c.cssnap, (size_t)kMaxShards * kCSets * kCSetWords));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  // the two-level kernel keeps its forwarder baselines after the TMA ring
  const size_t smem = sweep_smem_bytes(c.m, c.chunk, c.size, c.stream != 0, mode == BART_EXCHANGE_TWO_LEVEL);
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
  if ((int64_t)smem > optin) return fail(BART_EINVAL, "two-level exchange needs " + std::to_string(smem) +
                                                         " B of shared memory > " + std::to_string(optin));
  if (cudaError_t e = sweep_prepare(smem); e != cudaSuccess)
    return fail(BART_ECUDA, std::string("sweep_prepare: ") + cudaGetErrorString(e));
  h->smem = smem;
  c.hier = mode == BART_EXCHANGE_TWO_LEVEL ? 1 : 0;
  drop_graphs(h);  // captured launches carry the chain parameters
  return BART_OK;
}

int bart_trace_begin(bart_chain *h, const bart_trace_opts *o, const uint8_t *X_test) {
  if (!h || !o) return fail(BART_EINVAL, "NULL argument");
  if (o->n_iter < 0 || o->n_keep < 0 || o->n_test < 0 || o->train_ring < 0 || (o->n_test > 0 && !X_test))
    return fail(BART_EINVAL, "bad trace options");
  CUDA_TRY(cudaSetDevice(h->device));
  trace_free(h);
  ChainDev &c = h->c;
  TraceState &t = h->tr;
  t.iter_cap = o->n_iter;
  t.keep_cap = o->n_keep;
  t.n_test = o->n_test;
  t.ld_test = round16(o->n_test);
  t.store_train = o->store_train_draws;
  t.store_forests = o->store_forests;
  t.npts = (int)(c.n < BART_TRACE_POINTS ? c.n : BART_TRACE_POINTS);
  t.iter0 = h->iteration;
  const size_t K = (size_t)t.keep_cap, n = (size_t)c.n;
  CUDA_TRY(trace_alloc(h, &t.acc, (size_t)t.iter_cap * c.m));
  CUDA_TRY(trace_alloc(h, &t.sig_iter, (size_t)t.iter_cap));
  CUDA_TRY(trace_alloc(h, &t.sig_keep, K));
  CUDA_TRY(trace_alloc(h, &t.mean, n));
  CUDA_TRY(trace_alloc(h, &t.m2, n));
  CUDA_TRY(trace_alloc(h, &t.pts, K * t.npts));
  CUDA_TRY(trace_alloc(h, &t.mleaves, K));
  t.train_rows = (o->train_ring > 0 && o->train_ring < t.keep_cap) ? o->train_ring : t.keep_cap;
  if (t.store_train) CUDA_TRY(trace_alloc(h, &t.train, (size_t)t.train_rows * n));
  if (t.n_test) {
    CUDA_TRY(trace_alloc(h, &t.test, K * (size_t)t.n_test));
    CUDA_TRY(trace_alloc(h, &t.Xt_test, (size_t)t.ld_test * c.p));
    DevBuf xs;
    CUDA_TRY(xs.alloc((size_t)t.n_test * c.p));
    CUDA_TRY(cudaMemcpyAsync(xs.p, X_test, (size_t)t.n_test * c.p, cudaMemcpyHostToDevice, h->stream));
    launch_transpose_u8(xs.as<uint8_t>(), t.n_test, c.p, c.p, t.Xt_test, t.ld_test, h->stream);
    CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  if (t.store_forests) {
    CUDA_TRY(trace_alloc(h, &t.f_axis, K * c.m * c.half));
    CUDA_TRY(trace_alloc(h, &t.f_cut, K * c.m * c.half));
    CUDA_TRY(trace_alloc(h, &t.f_leaf, K * c.m * c.size));
  }
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  c.acc_hist = t.acc;
  c.sig_hist = t.sig_iter;
  c.hist_base = h->iteration;
  c.hist_cap = t.iter_cap;
  t.on = true;
  drop_graphs(h);  // captured launches carry the chain parameters
  return BART_OK;
}

int bart_trace_keep(bart_chain *h) {
  if (!h) return fail(BART_EINVAL, "NULL handle");
  TraceState &t = h->tr;
  if (!t.on) return fail(BART_ESTATE, "no trace (bart_trace_begin)");
  if (t.kept >= t.keep_cap) return fail(BART_EINVAL, "trace full: n_keep draws already kept");
  CUDA_TRY(cudaSetDevice(h->device));
  ChainDev &c = h->c;
  cudaStream_t s = h->stream;
  const size_t k = (size_t)t.kept;
  launch_trace_train(c.L, c.n, c.n_pad, c.m, c.size, c.leaf, t.kept + 1, t.mean, t.m2,
                     t.store_train ? t.train + (k % (size_t)t.train_rows) * c.n : nullptr, t.pts + k * t.npts, t.npts, s);
  if (t.n_test)
    launch_evaluate(t.Xt_test, t.n_test, t.ld_test, c.D, c.half, c.m, c.axis, c.cut, c.leaf, t.test + k * t.n_test, s);
  launch_mean_leaves(c.cut, c.m, c.half, t.mleaves + k, s);
  h->launches += t.n_test ? 3 : 2;
  CUDA_TRY(cudaMemcpyAsync(t.sig_keep + k, c.sigma2, 8, cudaMemcpyDeviceToDevice, s));
  if (t.store_forests) {
    CUDA_TRY(cudaMemcpyAsync(t.f_axis + k * c.m * c.half, c.axis, (size_t)c.m * c.half * 2, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(t.f_cut + k * c.m * c.half, c.cut, (size_t)c.m * c.half, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(t.f_leaf + k * c.m * c.size, c.leaf, (size_t)c.m * c.size * 4, cudaMemcpyDeviceToDevice, s));
  }
  CUDA_TRY(cudaGetLastError());
  t.kept += 1;
  return BART_OK;
}

int bart_trace_counts(bart_chain *h, int64_t *n_iter, int64_t *n_keep) {
  if (!h || !n_iter || !n_keep) return fail(BART_EINVAL, "NULL argument");
  const TraceState &t = h->tr;
  if (!t.on) return fail(BART_ESTATE, "no trace (bart_trace_begin)");
  const int64_t it = h->iteration - t.iter0;
  *n_iter = it < t.iter_cap ? it : t.iter_cap;
  *n_keep = t.kept;
  return BART_OK;
}

int bart_trace_read(bart_chain *h, uint8_t *accepted, double *sigma2_iter, double *sigma2_keep, double *train_mean,
                    double *train_var, double *train_draws, double *train_points, double *test_draws,
                    double *mean_leaves, uint16_t *axis, uint8_t *cutpoint, float *leaf_value) {
  int64_t ni = 0, nk = 0;
  if (int rc = bart_trace_counts(h, &ni, &nk)) return rc;
  if (int rc = bart_sync(h)) return rc;
  const TraceState &t = h->tr;
  const ChainDev &c = h->c;
  auto d2h = [](void *dst, const void *src, size_t bytes) {
    return dst && bytes ? cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost) : cudaSuccess;
  };
  CUDA_TRY(d2h(accepted, t.acc, (size_t)ni * c.m));
  CUDA_TRY(d2h(sigma2_iter, t.sig_iter, (size_t)ni * 8));
  CUDA_TRY(d2h(sigma2_keep, t.sig_keep, (size_t)nk * 8));
  CUDA_TRY(d2h(train_mean, t.mean, (size_t)c.n * 8));
  if (train_var) {  // sample variance over the kept draws
    CUDA_TRY(d2h(train_var, t.m2, (size_t)c.n * 8));
    for (int64_t i = 0; i < c.n; ++i) train_var[i] = nk > 1 ? train_var[i] / (double)(nk - 1) : 0.0;
  }
  if (t.store_train && train_draws) {
    if (t.train_rows < t.keep_cap) return fail(BART_ESTATE, "training-row draws are in a ring: read them with bart_trace_read_draws");
    CUDA_TRY(d2h(train_draws, t.train, (size_t)nk * c.n * 8));
  }
  CUDA_TRY(d2h(train_points, t.pts, (size_t)nk * t.npts * 8));
  if (t.n_test) CUDA_TRY(d2h(test_draws, t.test, (size_t)nk * t.n_test * 8));
  CUDA_TRY(d2h(mean_leaves, t.mleaves, (size_t)nk * 8));
  if (t.store_forests) {
    CUDA_TRY(d2h(axis, t.f_axis, (size_t)nk * c.m * c.half * 2));
    CUDA_TRY(d2h(cutpoint, t.f_cut, (size_t)nk * c.m * c.half));
    CUDA_TRY(d2h(leaf_value, t.f_leaf, (size_t)nk * c.m * c.size * 4));
  }
  return BART_OK;
}

int bart_trace_read_draws(bart_chain *h, int64_t k0, int64_t k1, double *train, double *test) {
  int64_t ni = 0, nk = 0;
  if (int rc = bart_trace_counts(h, &ni, &nk)) return rc;
  if (k0 < 0 || k1 < k0 || k1 > nk) return fail(BART_EINVAL, "draw range outside the kept draws");
  const TraceState &t = h->tr;
  if (train && !t.store_train) return fail(BART_ESTATE, "training-row draws were not stored (store_train_draws)");
  if (test && !t.n_test) return fail(BART_ESTATE, "no test rows in this trace");
  if (int rc = bart_sync(h)) return rc;
  const size_t rows = (size_t)(k1 - k0);
  if (train && rows) {
    if (k0 < nk - t.train_rows) return fail(BART_EINVAL, "draw range no longer in the device ring (train_ring)");
    const size_t n = (size_t)h->c.n;
    for (size_t k = (size_t)k0; k < (size_t)k1;) {  // contiguous runs of ring rows
      const size_t r = k % (size_t)t.train_rows, run = std::min((size_t)k1 - k, (size_t)t.train_rows - r);
      CUDA_TRY(cudaMemcpy(train + (k - (size_t)k0) * n, t.train + r * n, run * n * 8, cudaMemcpyDeviceToHost));
      k += run;
    }
  }
  if (test && rows)
    CUDA_TRY(cudaMemcpy(test, t.test + (size_t)k0 * t.n_test, rows * t.n_test * 8, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int bart_trace_end(bart_chain *h) {
  if (!h) return fail(BART_EINVAL, "NULL handle");
  CUDA_TRY(cudaSetDevice(h->device));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  trace_free(h);
  return BART_OK;
}

// ---- binning (grid.py) ----
int bart_grid_minmax(const double *X, int64_t n, int32_t p, double *lo, double *hi, int device) {
  if (!X || !lo || !hi || n < 1 || p < 1) return fail(BART_EINVAL, "bad minmax arguments");
  CUDA_TRY(cudaSetDevice(device));
  DevBuf dx, keys, bad, dlo, dhi;
  CUDA_TRY(dx.alloc((size_t)n * p * 8));
  CUDA_TRY(keys.alloc((size_t)2 * p * 8));
  CUDA_TRY(bad.alloc(8));
  CUDA_TRY(dlo.alloc((size_t)p * 8));
  CUDA_TRY(dhi.alloc((size_t)p * 8));
  CUDA_TRY(cudaMemcpy(dx.p, X, (size_t)n * p * 8, cudaMemcpyHostToDevice));
  launch_minmax(dx.as<double>(), n, p, keys.as<long long>(), bad.as<unsigned long long>(), dlo.as<double>(),
                dhi.as<double>(), 0);
  unsigned long long nbad = 0;
  CUDA_TRY(cudaMemcpy(&nbad, bad.p, 8, cudaMemcpyDeviceToHost));
  if (nbad) return fail(BART_EINVAL, "predictors must be finite (" + std::to_string(nbad) + " non-finite values)");
  CUDA_TRY(cudaMemcpy(lo, dlo.p, (size_t)p * 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(hi, dhi.p, (size_t)p * 8, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int bart_quantize(const double *X, int64_t n, int32_t p, const double *cutpoints, const int64_t *offsets,
                  uint8_t *out, int device) {
  if (!X || !cutpoints || !offsets || !out || n < 0 || p < 1) return fail(BART_EINVAL, "bad quantize arguments");
  for (int a = 0; a < p; ++a)
    if (offsets[a + 1] < offsets[a] || offsets[a + 1] - offsets[a] > 255)
      return fail(BART_EINVAL, "each axis needs 0..255 cutpoints (grid.py:18)");
  if (n == 0) return BART_OK;
  CUDA_TRY(cudaSetDevice(device));
  const int64_t nc = offsets[p];
  DevBuf dx, dc, doff, dout;
  CUDA_TRY(dx.alloc((size_t)n * p * 8));
  CUDA_TRY(dc.alloc((size_t)(nc > 0 ? nc : 1) * 8));
  CUDA_TRY(doff.alloc((size_t)(p + 1) * 8));
  CUDA_TRY(dout.alloc((size_t)n * p));
  CUDA_TRY(cudaMemcpy(dx.p, X, (size_t)n * p * 8, cudaMemcpyHostToDevice));
  if (nc > 0) CUDA_TRY(cudaMemcpy(dc.p, cutpoints, (size_t)nc * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(doff.p, offsets, (size_t)(p + 1) * 8, cudaMemcpyHostToDevice));
  launch_quantize(dx.as<double>(), n, p, dc.as<double>(), doff.as<int64_t>(), dout.as<uint8_t>(), 0);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpy(out, dout.p, (size_t)n * p, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int bart_grid_uniform_quantize(const double *X, int64_t n, int32_t p, int32_t n_cutpoints, double *lo, double *hi,
                               uint8_t *out, int device) {
  if (!X || !lo || !hi || !out || n < 2 || p < 1) return fail(BART_EINVAL, "bad grid arguments");
  if (n_cutpoints < 1 || n_cutpoints > 255) return fail(BART_EINVAL, "n_cutpoints must be in [1, 255]");
  CUDA_TRY(cudaSetDevice(device));
  DevBuf dx, keys, bad, dlo, dhi, dc, doff, dout;
  CUDA_TRY(dx.alloc((size_t)n * p * 8));
  CUDA_TRY(keys.alloc((size_t)2 * p * 8));
  CUDA_TRY(bad.alloc(8));
  CUDA_TRY(dlo.alloc((size_t)p * 8));
  CUDA_TRY(dhi.alloc((size_t)p * 8));
  CUDA_TRY(dc.alloc((size_t)p * n_cutpoints * 8));
  CUDA_TRY(doff.alloc((size_t)(p + 1) * 8));
  CUDA_TRY(dout.alloc((size_t)n * p));
  CUDA_TRY(cudaMemcpy(dx.p, X, (size_t)n * p * 8, cudaMemcpyHostToDevice));
  launch_minmax(dx.as<double>(), n, p, keys.as<long long>(), bad.as<unsigned long long>(), dlo.as<double>(),
                dhi.as<double>(), 0);
  unsigned long long nbad = 0;
  CUDA_TRY(cudaMemcpy(&nbad, bad.p, 8, cudaMemcpyDeviceToHost));
  if (nbad) return fail(BART_EINVAL, "predictors must be finite (" + std::to_string(nbad) + " non-finite values)");
  CUDA_TRY(cudaMemcpy(lo, dlo.p, (size_t)p * 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(hi, dhi.p, (size_t)p * 8, cudaMemcpyDeviceToHost));
  // the cutpoints as grid.build_grid_uniform computes them in numpy: frac_k =
  // k / (K + 1) correctly rounded, then lo + (hi - lo) * frac_k, two roundings
  // (x86-64 host code: no FMA contraction)
  std::vector<double> cuts;
  std::vector<int64_t> off(p + 1, 0);
  cuts.reserve((size_t)p * n_cutpoints);
  for (int a = 0; a < p; ++a) {
    if (lo[a] != hi[a]) {
      const double span = hi[a] - lo[a];
      for (int k = 1; k <= n_cutpoints; ++k) {
        const double frac = (double)k / (double)(n_cutpoints + 1);
        const double step = span * frac;
        cuts.push_back(lo[a] + step);
      }
    }
    off[a + 1] = (int64_t)cuts.size();
  }
  if (!cuts.empty()) CUDA_TRY(cudaMemcpy(dc.p, cuts.data(), cuts.size() * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(doff.p, off.data(), (size_t)(p + 1) * 8, cudaMemcpyHostToDevice));
  launch_quantize(dx.as<double>(), n, p, dc.as<double>(), doff.as<int64_t>(), dout.as<uint8_t>(), 0);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpy(out, dout.p, (size_t)n * p, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int bart_destroy(bart_chain *h) {
  free_chain(h);
  return BART_OK;
}

int bart_set_hparams(bart_chain *h, const bart_hparams *hp) {
  if (!h || !hp) return fail(BART_EINVAL, "NULL argument");
  h->c.hp = to_hp(hp);
  h->update_sigma = hp->update_sigma != 0;
  drop_graphs(h);  // captured launches carry the chain parameters
  return BART_OK;
}

int bart_set_sigma2(bart_chain *h, double sigma2) {
  if (!h) return fail(BART_EINVAL, "NULL handle");
  CUDA_TRY(cudaSetDevice(h->device));
  CUDA_TRY(cudaMemcpyAsync(h->c.sigma2, &sigma2, 8, cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return BART_OK;
}

int bart_set_state(bart_chain *h, const uint16_t *axis, const uint8_t *cutpoint, const float *leaf_value,
                   const uint8_t *leaf_index, const float *resid, double sigma2) {
  if (!h || !axis || !cutpoint || !leaf_value) return fail(BART_EINVAL, "NULL argument");
  CUDA_TRY(cudaSetDevice(h->device));
  ChainDev &c = h->c;
  cudaStream_t s = h->stream;
  CUDA_TRY(cudaMemcpyAsync(c.axis, axis, (size_t)c.m * c.half * 2, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(c.cut, cutpoint, (size_t)c.m * c.half, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(c.leaf, leaf_value, (size_t)c.m * c.size * 4, cudaMemcpyHostToDevice, s));
  if (leaf_index) {
    DevBuf tmp;
    CUDA_TRY(tmp.alloc((size_t)c.n * c.m));
    CUDA_TRY(cudaMemcpyAsync(tmp.p, leaf_index, (size_t)c.n * c.m, cudaMemcpyHostToDevice, s));
    launch_transpose_u8(tmp.as<uint8_t>(), c.n, c.m, c.m, c.L, c.n_pad, s);
    CUDA_TRY(cudaStreamSynchronize(s));
  } else {
    launch_traverse(c.Xt, c.n, c.n_pad, c.D, c.half, c.m, c.axis, c.cut, c.L, s);
  }
  h->launches += 1;
  if (resid) {
    CUDA_TRY(cudaMemcpyAsync(c.r, resid, (size_t)c.n * 4, cudaMemcpyHostToDevice, s));
  } else {
    DevBuf pred;
    CUDA_TRY(pred.alloc((size_t)c.n_pad * 8));
    launch_predict_cached(c.L, c.n, c.n_pad, c.m, c.size, c.leaf, pred.as<double>(), s);
    launch_resid(c.y, pred.as<double>(), c.r, c.n, s);
    h->launches += 2;
    CUDA_TRY(cudaStreamSynchronize(s));
  }
  if (sigma2 >= 0.0) CUDA_TRY(cudaMemcpyAsync(c.sigma2, &sigma2, 8, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemsetAsync(c.err, 0, sizeof(int), s));  // a reset chain is valid again (BART_ERANGE)
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  return BART_OK;
}

// The sweep's sticky exchange-range flag (sweep.cu to_limbs), read after the
// stream has synchronised.
static int check_range(bart_chain *h) {
  int err = 0;
  CUDA_TRY(cudaMemcpy(&err, h->c.err, sizeof(err), cudaMemcpyDeviceToHost));
  if (err) return fail(BART_ERANGE, kRangeMsg);
  return BART_OK;
}

// the bart_step pipeline's second slot, pinned stages, copy streams and
// events, made on the first bart_step (device-RNG chains driven by bart_run,
// like fit()'s, never pay for them)
// one bart_step result in pinned memory: accept flags (m, padded to 8) |
// sigma2 draw (8 B) | exchange error flag (8 B)
static size_t step_out_stride(int m) { return ((size_t)m + 7) / 8 * 8 + 16; }

static cudaError_t ensure_step_pipeline(bart_chain *h) {
  if (h->step_out) return cudaSuccess;
  const ChainDev &c = h->c;
  const size_t rwords = (size_t)c.m * 5 + (size_t)c.m + (size_t)c.m * c.size + 1;
  cudaError_t e = own(h, &h->rblock[1], rwords);
  for (int k = 0; k < 2 && e == cudaSuccess; ++k) e = cudaHostAlloc(&h->rstage[k], rwords * 8, cudaHostAllocMapped);
  for (int k = 0; k < 2 && e == cudaSuccess; ++k)
    e = cudaEventCreateWithFlags(&h->kernel_done[k], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);  // the new buffers' zero fill
  if (e == cudaSuccess) e = cudaHostAlloc(&h->step_out, 2 * step_out_stride(c.m), cudaHostAllocMapped);
  if (e == cudaSuccess) std::memset(h->step_out, 0, 2 * step_out_stride(c.m));
  return e;
}

int bart_step(bart_chain *h, const bart_randoms *rnd) {
  if (!h) return fail(BART_EINVAL, "NULL handle");
  if (h->shard_pending) return fail(BART_ESTATE, "shard not connected (bart_shard_connect)");
  CUDA_TRY(cudaSetDevice(h->device));
  ChainDev &c = h->c;
  CUDA_TRY(ensure_step_pipeline(h));
  const int slot = (int)(h->iteration & 1);
  ChainDev args = step_args(h, rnd ? 0 : 1);
  const size_t nm = (size_t)c.m * 5, na = (size_t)c.m, nz = (size_t)c.m * c.size;
  // injected randoms: the kernel reads the block straight from the slot's
  // pinned stage (zero-copy over the host link: the block's 8(6m + m*2^D) + 8
  // bytes are the step's host->device transfer, with no copy-engine hop and
  // no cross-stream event between the copy and the kernel); device randoms:
  // the slot's device block, which the kernel writes
  double *blk = h->rblock[slot];
  if (rnd) CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void **>(&blk), h->rstage[slot], 0));
  args.rand_move = blk;
  args.rand_acc = blk + nm;
  args.rand_z = blk + nm + na;
  args.rand_chi2 = blk + nm + na + nz;
  // the step's result, written by the kernel into the slot's pinned step_out
  const size_t stride = step_out_stride(c.m);
  uint8_t *out_host = h->step_out + (size_t)slot * stride, *out_dev = nullptr;
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void **>(&out_dev), out_host, 0));
  args.accepted = out_dev;
  args.sigma2_draw = reinterpret_cast<double *>(out_dev + stride - 16);
  args.err_out = reinterpret_cast<int *>(out_dev + stride - 8);
  if (rnd) {
    if (!rnd->move_u || !rnd->accept_u || !rnd->leaf_z) return fail(BART_EINVAL, "incomplete randoms");
    // the slot's stage (and result) is free once the step two back is done
    CUDA_TRY(cudaEventSynchronize(h->kernel_done[slot]));
    double *st = h->rstage[slot];
    std::memcpy(st, rnd->move_u, nm * 8);
    std::memcpy(st + nm, rnd->accept_u, na * 8);
    std::memcpy(st + nm + na, rnd->leaf_z, nz * 8);
    st[nm + na + nz] = rnd->chi2;
  }
  // one captured launch per (slot, randoms kind): graph replay skips the
  // cooperative launch's per-call validation
  cudaGraphExec_t &gx = h->graph_step[slot][rnd ? 1 : 0];
  if (!gx && !h->graph_failed) {
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      const cudaError_t e1 = (cudaError_t)sweep_launch(args, h->smem, h->stream);
      const cudaError_t e2 = cudaStreamEndCapture(h->stream, &g);
      if (e1 != cudaSuccess || e2 != cudaSuccess || !g || cudaGraphInstantiate(&gx, g, 0) != cudaSuccess) gx = nullptr;
      if (g) cudaGraphDestroy(g);
    }
    cudaGetLastError();
  }
  if (gx)
    CUDA_TRY(cudaGraphLaunch(gx, h->stream));
  else
    CUDA_TRY((cudaError_t)sweep_launch(args, h->smem, h->stream));
  h->launches += 1;
  h->iteration += 1;
  CUDA_TRY(cudaEventRecord(h->kernel_done[slot], h->stream));
  h->res_acc = out_host;
  h->res_sdraw = reinterpret_cast<double *>(out_host + stride - 16);
  h->res_block = blk;
  h->slot_iter[slot] = h->iteration - 1;
  return BART_OK;
}

int bart_read_step_result(bart_chain *h, int64_t iteration, uint8_t *accepted, double *sigma2) {
  if (!h) return fail(BART_EINVAL, "NULL handle");
  if (iteration < 0 || iteration < h->iteration - 2 || iteration >= h->iteration)
    return fail(BART_EINVAL, "only the last two bart_step results are kept");
  if (!h->step_out || h->slot_iter[iteration & 1] != iteration)
    return fail(BART_ESTATE, "iteration " + std::to_string(iteration) + " did not run through bart_step");
  CUDA_TRY(cudaSetDevice(h->device));
  CUDA_TRY(cudaEventSynchronize(h->kernel_done[iteration & 1]));
  const size_t stride = step_out_stride(h->c.m);
  const uint8_t *src = h->step_out + (size_t)(iteration & 1) * stride;
  int err = 0;
  std::memcpy(&err, src + stride - 8, 4);
  if (err) return fail(BART_ERANGE, kRangeMsg);
  if (accepted) std::memcpy(accepted, src, (size_t)h->c.m);
  if (sigma2) {
    if (h->update_sigma) {
      std::memcpy(sigma2, src + stride - 16, 8);  // the step's draw became sigma2 (sampler.py:906-908)
    } else {  // sigma2 is not sampled: the (unchanged) state value
      CUDA_TRY(cudaMemcpy(sigma2, h->c.sigma2, 8, cudaMemcpyDeviceToHost));
    }
  }
  return BART_OK;
}

int bart_propose(bart_chain *h, const double *move_u) {
  if (!h || !move_u) return fail(BART_EINVAL, "NULL argument");
  CUDA_TRY(cudaSetDevice(h->device));
  CUDA_TRY(cudaMemcpyAsync(h->c.rand_move, move_u, (size_t)h->c.m * 5 * 8, cudaMemcpyHostToDevice, h->stream));
  launch_propose(h->c, 0, h->stream);
  h->launches += 1;
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  CUDA_TRY(cudaGetLastError());
  return BART_OK;
}

int bart_run(bart_chain *h, int64_t n_iter) {
  if (!h) return fail(BART_EINVAL, "NULL handle");
  if (h->shard_pending) return fail(BART_ESTATE, "shard not connected (bart_shard_connect)");
  CUDA_TRY(cudaSetDevice(h->device));
  ensure_graph(h);
  h->res_acc = h->acc_base;  // the graph's kernels use the base buffers
  h->res_sdraw = h->sdraw_base;
  h->res_block = h->rblock[0];
  for (int64_t i = 0; i < n_iter; ++i) {
    if (h->graph) {
      CUDA_TRY(cudaGraphLaunch(h->graph, h->stream));
      h->launches += 1;
      h->iteration += 1;
    } else if (int rc = launch_iteration(h, 1)) {
      return rc;
    }
  }
  CUDA_TRY(cudaGetLastError());
  return BART_OK;
}

int bart_sync(bart_chain *h) {
  if (!h) return fail(BART_EINVAL, "NULL handle");
  CUDA_TRY(cudaSetDevice(h->device));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  CUDA_TRY(cudaGetLastError());
  return check_range(h);
}

int bart_get_forest(bart_chain *h, uint16_t *axis, uint8_t *cutpoint, float *leaf_value) {
  if (int rc = bart_sync(h)) return rc;
  ChainDev &c = h->c;
  if (axis) CUDA_TRY(cudaMemcpy(axis, c.axis, (size_t)c.m * c.half * 2, cudaMemcpyDeviceToHost));
  if (cutpoint) CUDA_TRY(cudaMemcpy(cutpoint, c.cut, (size_t)c.m * c.half, cudaMemcpyDeviceToHost));
  if (leaf_value) CUDA_TRY(cudaMemcpy(leaf_value, c.leaf, (size_t)c.m * c.size * 4, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int bart_get_leaf_index(bart_chain *h, uint8_t *out) {
  if (int rc = bart_sync(h)) return rc;
  ChainDev &c = h->c;
  DevBuf tmp;
  CUDA_TRY(tmp.alloc((size_t)c.n * c.m));
  launch_transpose_u8(c.L, c.m, c.n, c.n_pad, tmp.as<uint8_t>(), c.m, h->stream);
  h->launches += 1;
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  CUDA_TRY(cudaMemcpy(out, tmp.p, (size_t)c.n * c.m, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int bart_get_resid(bart_chain *h, float *out) {
  if (int rc = bart_sync(h)) return rc;
  CUDA_TRY(cudaMemcpy(out, h->c.r, (size_t)h->c.n * 4, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int bart_get_sigma2(bart_chain *h, double *out) {
  if (int rc = bart_sync(h)) return rc;
  CUDA_TRY(cudaMemcpy(out, h->c.sigma2, 8, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int bart_get_step_result(bart_chain *h, uint8_t *accepted, double *sigma2) {
  if (!h) return fail(BART_EINVAL, "NULL handle");
  CUDA_TRY(cudaSetDevice(h->device));
  const size_t m = (size_t)h->c.m;
  if (!h->result_stage) CUDA_TRY(cudaMallocHost(&h->result_stage, m + 24));
  uint8_t *st = h->result_stage;
  const size_t m8 = (m + 7) & ~(size_t)7;
  if (accepted) CUDA_TRY(cudaMemcpyAsync(st, h->res_acc, m, cudaMemcpyDefault, h->stream));
  if (sigma2) CUDA_TRY(cudaMemcpyAsync(st + m8, h->c.sigma2, 8, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaMemcpyAsync(st + m8 + 8, h->c.err, 4, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  CUDA_TRY(cudaGetLastError());
  int err = 0;
  std::memcpy(&err, st + m8 + 8, 4);
  if (err) return fail(BART_ERANGE, kRangeMsg);
  if (accepted) std::memcpy(accepted, st, m);
  if (sigma2) std::memcpy(sigma2, st + m8, 8);
  return BART_OK;
}

int bart_get_accepted(bart_chain *h, uint8_t *out) {
  if (int rc = bart_sync(h)) return rc;
  CUDA_TRY(cudaMemcpy(out, h->res_acc, (size_t)h->c.m, cudaMemcpyDefault));
  return BART_OK;
}

int bart_get_randoms(bart_chain *h, double *move_u, double *accept_u, double *leaf_z, double *chi2) {
  if (int rc = bart_sync(h)) return rc;
  const ChainDev &c = h->c;
  const size_t nm = (size_t)c.m * 5, na = (size_t)c.m, nz = (size_t)c.m * c.size;
  const double *b = h->res_block;  // a device block, or (injected) a pinned stage
  if (move_u) CUDA_TRY(cudaMemcpy(move_u, b, nm * 8, cudaMemcpyDefault));
  if (accept_u) CUDA_TRY(cudaMemcpy(accept_u, b + nm, na * 8, cudaMemcpyDefault));
  if (leaf_z) CUDA_TRY(cudaMemcpy(leaf_z, b + nm + na, nz * 8, cudaMemcpyDefault));
  if (chi2) CUDA_TRY(cudaMemcpy(chi2, b + nm + na + nz, 8, cudaMemcpyDefault));
  return BART_OK;
}

int bart_philox4x32_10(const uint32_t *ctr, const uint32_t *key, uint32_t *out, int64_t count, int device) {
  if (!ctr || !key || !out || count < 0) return fail(BART_EINVAL, "bad philox arguments");
  if (count == 0) return BART_OK;
  CUDA_TRY(cudaSetDevice(device));
  DevBuf dc, dk, dout;
  CUDA_TRY(dc.alloc((size_t)count * 16));
  CUDA_TRY(dk.alloc((size_t)count * 8));
  CUDA_TRY(dout.alloc((size_t)count * 16));
  CUDA_TRY(cudaMemcpy(dc.p, ctr, (size_t)count * 16, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dk.p, key, (size_t)count * 8, cudaMemcpyHostToDevice));
  launch_philox(dc.as<uint32_t>(), dk.as<uint32_t>(), dout.as<uint32_t>(), count, 0);
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpy(out, dout.p, (size_t)count * 16, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int bart_get_proposals(bart_chain *h, int64_t *rows, double *struct_log) {
  if (int rc = bart_sync(h)) return rc;
  const int m = h->c.m;
  std::vector<TreeMove> mv(m);
  CUDA_TRY(cudaMemcpy2D(mv.data(), sizeof(TreeMove), h->c.rec, (size_t)h->c.rstride, sizeof(TreeMove), m,
                        cudaMemcpyDeviceToHost));
  for (int j = 0; j < m; ++j) {
    const TreeMove &t = mv[j];
    const int64_t vals[BART_PROPOSAL_ROWS] = {t.kind,    t.node,        t.axis,         t.cut,
                                              t.depth,   t.n_axes,      t.n_splits,     t.w_small,
                                              t.w_prime_big, t.growable_big, t.gl, t.gr};
    for (int k = 0; k < BART_PROPOSAL_ROWS; ++k) rows[(size_t)k * m + j] = vals[k];
    if (struct_log) struct_log[j] = t.struct_log;
  }
  return BART_OK;
}

int bart_set_taps(bart_chain *h, int on) {
  if (!h) return fail(BART_EINVAL, "NULL handle");
  CUDA_TRY(cudaSetDevice(h->device));
  ChainDev &c = h->c;
  if (on && !c.tap_counts) {
    CUDA_TRY(own(h, &c.tap_counts, (size_t)c.m * c.size));
    CUDA_TRY(own(h, &c.tap_sums, (size_t)c.m * c.size));
  }
  c.taps = on ? 1 : 0;
  drop_graphs(h);  // captured launches carry the chain parameters
  return BART_OK;
}

int bart_set_timeline(bart_chain *h, int on) {
  if (!h) return fail(BART_EINVAL, "NULL handle");
  CUDA_TRY(cudaSetDevice(h->device));
  ChainDev &c = h->c;
  if (on && !h->timeline_buf) CUDA_TRY(own(h, &h->timeline_buf, (size_t)4 * (c.m + 2) * 8));
  if (on && !h->trace_buf) CUDA_TRY(own(h, &h->trace_buf, (size_t)(c.m + 2) * c.nblk * 2));
  c.timeline = on ? h->timeline_buf : nullptr;
  c.trace = on ? h->trace_buf : nullptr;
  drop_graphs(h);  // captured launches carry the chain parameters
  return BART_OK;
}

int bart_get_timeline(bart_chain *h, int64_t *out) {
  if (int rc = bart_sync(h)) return rc;
  if (!h->timeline_buf) return fail(BART_ESTATE, "timeline not enabled (bart_set_timeline)");
  CUDA_TRY(cudaMemcpy(out, h->timeline_buf, (size_t)4 * (h->c.m + 2) * 8 * 8, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int bart_get_trace(bart_chain *h, int64_t *out) {
  if (int rc = bart_sync(h)) return rc;
  if (!h->trace_buf) return fail(BART_ESTATE, "timeline not enabled (bart_set_timeline)");
  CUDA_TRY(cudaMemcpy(out, h->trace_buf, (size_t)(h->c.m + 2) * h->c.nblk * 2 * 8, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int bart_get_taps(bart_chain *h, int64_t *counts, double *sums) {
  if (int rc = bart_sync(h)) return rc;
  ChainDev &c = h->c;
  if (!c.tap_counts) return fail(BART_ESTATE, "taps not enabled (bart_set_taps)");
  CUDA_TRY(cudaMemcpy(counts, c.tap_counts, (size_t)c.m * c.size * 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(sums, c.tap_sums, (size_t)c.m * c.size * 8, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int64_t bart_iteration(bart_chain *h) { return h ? h->iteration : -1; }

int bart_set_iteration(bart_chain *h, int64_t iteration) {
  if (!h) return fail(BART_EINVAL, "NULL handle");
  if (iteration < 0) return fail(BART_EINVAL, "iteration must be >= 0");
  if (h->tr.on) return fail(BART_ESTATE, "cannot move the iteration counter while a trace is recording");
  CUDA_TRY(cudaSetDevice(h->device));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  const unsigned long long it = (unsigned long long)iteration;  // the device Philox counter
  CUDA_TRY(cudaMemcpy(h->c.iter_dev, &it, sizeof(it), cudaMemcpyHostToDevice));
  h->iteration = iteration;
  return BART_OK;
}
int64_t bart_kernel_launches(bart_chain *h) { return h ? h->launches : -1; }

int bart_sweep_config(bart_chain *h, int32_t *out) {
  if (!h || !out) return fail(BART_EINVAL, "NULL argument");
  out[0] = h->c.nblk;
  out[1] = kSweepThreads;
  out[2] = h->c.chunk;
  out[3] = (int32_t)h->smem;
  out[4] = h->c.stream;
  return BART_OK;
}

int bart_predict_cached(bart_chain *h, double *out) {
  if (int rc = bart_sync(h)) return rc;
  ChainDev &c = h->c;
  DevBuf pred;
  CUDA_TRY(pred.alloc((size_t)c.n_pad * 8));
  launch_predict_cached(c.L, c.n, c.n_pad, c.m, c.size, c.leaf, pred.as<double>(), h->stream);
  h->launches += 1;
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpy(out, pred.p, (size_t)c.n * 8, cudaMemcpyDeviceToHost));
  return BART_OK;
}

static int evaluate_on(int device, cudaStream_t s, const ChainDev &c, const uint16_t *d_axis, const uint8_t *d_cut,
                       const float *d_leaf, const uint8_t *X, int64_t n_new, double *out, int64_t *launches) {
  const int64_t ld = round16(n_new);
  DevBuf xs, xt, pred;
  CUDA_TRY(xs.alloc((size_t)n_new * c.p));
  CUDA_TRY(xt.alloc((size_t)ld * c.p));
  CUDA_TRY(pred.alloc((size_t)n_new * 8));
  CUDA_TRY(cudaMemsetAsync(xt.p, 0, (size_t)ld * c.p, s));
  CUDA_TRY(cudaMemcpyAsync(xs.p, X, (size_t)n_new * c.p, cudaMemcpyHostToDevice, s));
  launch_transpose_u8(xs.as<uint8_t>(), n_new, c.p, c.p, xt.as<uint8_t>(), ld, s);
  launch_evaluate(xt.as<uint8_t>(), n_new, ld, c.D, c.half, c.m, d_axis, d_cut, d_leaf, pred.as<double>(), s);
  if (launches) *launches += 2;
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpy(out, pred.p, (size_t)n_new * 8, cudaMemcpyDeviceToHost));
  (void)device;
  return BART_OK;
}

int bart_predict_matrix(bart_chain *h, const uint8_t *X, int64_t n_new, double *out) {
  if (int rc = bart_sync(h)) return rc;
  if (n_new <= 0) return BART_OK;
  return evaluate_on(h->device, h->stream, h->c, h->c.axis, h->c.cut, h->c.leaf, X, n_new, out, &h->launches);
}

int bart_traverse(const bart_dims *dims, const uint16_t *axis, const uint8_t *cutpoint, const uint8_t *X,
                  uint8_t *out_nm, int device) {
  if (int rc = check_dims(dims)) return rc;
  CUDA_TRY(cudaSetDevice(device));
  const int64_t n = dims->n, ld = round16(n);
  const int m = dims->m, D = dims->max_depth, half = 1 << (D - 1), p = dims->p;
  DevBuf da, dc, xs, xt, L, Lt;
  CUDA_TRY(da.alloc((size_t)m * half * 2));
  CUDA_TRY(dc.alloc((size_t)m * half));
  CUDA_TRY(xs.alloc((size_t)n * p));
  CUDA_TRY(xt.alloc((size_t)ld * p));
  CUDA_TRY(L.alloc((size_t)ld * m));
  CUDA_TRY(Lt.alloc((size_t)n * m));
  CUDA_TRY(cudaMemset(xt.p, 0, (size_t)ld * p));
  CUDA_TRY(cudaMemcpy(da.p, axis, (size_t)m * half * 2, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dc.p, cutpoint, (size_t)m * half, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(xs.p, X, (size_t)n * p, cudaMemcpyHostToDevice));
  launch_transpose_u8(xs.as<uint8_t>(), n, p, p, xt.as<uint8_t>(), ld, 0);
  launch_traverse(xt.as<uint8_t>(), n, ld, D, half, m, da.as<uint16_t>(), dc.as<uint8_t>(), L.as<uint8_t>(), 0);
  launch_transpose_u8(L.as<uint8_t>(), m, n, ld, Lt.as<uint8_t>(), m, 0);
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpy(out_nm, Lt.p, (size_t)n * m, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int bart_evaluate(const bart_dims *dims, const uint16_t *axis, const uint8_t *cutpoint, const float *leaf_value,
                  const uint8_t *X, double *out, int device) {
  if (int rc = check_dims(dims)) return rc;
  CUDA_TRY(cudaSetDevice(device));
  ChainDev c{};
  c.p = dims->p;
  c.m = dims->m;
  c.D = dims->max_depth;
  c.half = 1 << (c.D - 1);
  c.size = 1 << c.D;
  DevBuf da, dc, dl;
  CUDA_TRY(da.alloc((size_t)c.m * c.half * 2));
  CUDA_TRY(dc.alloc((size_t)c.m * c.half));
  CUDA_TRY(dl.alloc((size_t)c.m * c.size * 4));
  CUDA_TRY(cudaMemcpy(da.p, axis, (size_t)c.m * c.half * 2, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dc.p, cutpoint, (size_t)c.m * c.half, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dl.p, leaf_value, (size_t)c.m * c.size * 4, cudaMemcpyHostToDevice));
  return evaluate_on(device, 0, c, da.as<uint16_t>(), dc.as<uint8_t>(), dl.as<float>(), X, dims->n, out, nullptr);
}

int bart_evaluate_many(const bart_dims *dims, int64_t n_forests, const uint16_t *axis, const uint8_t *cutpoint,
                       const float *leaf_value, const uint8_t *X, double *out, int device) {
  if (int rc = check_dims(dims)) return rc;
  if (n_forests < 0) return fail(BART_EINVAL, "n_forests < 0");
  CUDA_TRY(cudaSetDevice(device));
  const int64_t n = dims->n, ld = round16(n);
  const int m = dims->m, D = dims->max_depth, half = 1 << (D - 1), size = 1 << D, p = dims->p;
  // forests go up and are evaluated a batch at a time (one launch per batch,
  // grid y = forest): enough forests to give the GPU ~4 blocks per SM when
  // one forest's point tiles are fewer (small n); a batch's output <= 512 MB
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int64_t tiles = (ld / 16 + 255) / 256;
  const int64_t want = std::max<int64_t>(1, (4 * (int64_t)sms + tiles - 1) / tiles);
  const int64_t batch = std::max<int64_t>(
      1, std::min<int64_t>({n_forests, want, (512ll << 20) / std::max<int64_t>(1, n * 8), (int64_t)65535}));
  DevBuf xs, xt, da, dc, dl, pred;
  CUDA_TRY(xs.alloc((size_t)n * p));
  CUDA_TRY(xt.alloc((size_t)ld * p));
  CUDA_TRY(da.alloc((size_t)batch * m * half * 2));
  CUDA_TRY(dc.alloc((size_t)batch * m * half));
  CUDA_TRY(dl.alloc((size_t)batch * m * size * 4));
  CUDA_TRY(pred.alloc((size_t)batch * n * 8));
  CUDA_TRY(cudaMemset(xt.p, 0, (size_t)ld * p));
  CUDA_TRY(cudaMemcpy(xs.p, X, (size_t)n * p, cudaMemcpyHostToDevice));
  launch_transpose_u8(xs.as<uint8_t>(), n, p, p, xt.as<uint8_t>(), ld, 0);
  for (int64_t f0 = 0; f0 < n_forests; f0 += batch) {
    const int64_t nf = std::min<int64_t>(batch, n_forests - f0);
    CUDA_TRY(cudaMemcpy(da.p, axis + (size_t)f0 * m * half, (size_t)nf * m * half * 2, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(dc.p, cutpoint + (size_t)f0 * m * half, (size_t)nf * m * half, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(dl.p, leaf_value + (size_t)f0 * m * size, (size_t)nf * m * size * 4, cudaMemcpyHostToDevice));
    launch_evaluate_batch(xt.as<uint8_t>(), n, ld, D, half, m, (int)nf, da.as<uint16_t>(), dc.as<uint8_t>(),
                          dl.as<float>(), pred.as<double>(), 0);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpy(out + (size_t)f0 * n, pred.p, (size_t)nf * n * 8, cudaMemcpyDeviceToHost));
  }
  return BART_OK;
}

int bart_sum_leaf_values(const bart_dims *dims, const float *leaf_value, const uint8_t *leaf_index_nm, double *out,
                         int device) {
  if (int rc = check_dims(dims)) return rc;
  CUDA_TRY(cudaSetDevice(device));
  const int64_t n = dims->n, ld = round16(n);
  const int m = dims->m, size = 1 << dims->max_depth;
  DevBuf ls, L, dl, pred;
  CUDA_TRY(ls.alloc((size_t)n * m));
  CUDA_TRY(L.alloc((size_t)ld * m));
  CUDA_TRY(dl.alloc((size_t)m * size * 4));
  CUDA_TRY(pred.alloc((size_t)ld * 8));
  CUDA_TRY(cudaMemset(L.p, 0, (size_t)ld * m));
  CUDA_TRY(cudaMemcpy(ls.p, leaf_index_nm, (size_t)n * m, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dl.p, leaf_value, (size_t)m * size * 4, cudaMemcpyHostToDevice));
  launch_transpose_u8(ls.as<uint8_t>(), n, m, m, L.as<uint8_t>(), ld, 0);
  launch_predict_cached(L.as<uint8_t>(), n, ld, m, size, dl.as<float>(), pred.as<double>(), 0);
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpy(out, pred.p, (size_t)n * 8, cudaMemcpyDeviceToHost));
  return BART_OK;
}

int bart_run_timed(bart_chain *h, int64_t n_iter, float *ms) {
  if (!h || !ms) return fail(BART_EINVAL, "NULL argument");
  CUDA_TRY(cudaSetDevice(h->device));
  ensure_graph(h);
  cudaEvent_t a, b;
  CUDA_TRY(cudaEventCreate(&a));
  CUDA_TRY(cudaEventCreate(&b));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  CUDA_TRY(cudaEventRecord(a, h->stream));
  for (int64_t i = 0; i < n_iter; ++i) {
    if (h->graph) {
      CUDA_TRY(cudaGraphLaunch(h->graph, h->stream));
      h->launches += 1;
      h->iteration += 1;
    } else if (int rc = launch_iteration(h, 1)) {
      return rc;
    }
  }
  CUDA_TRY(cudaEventRecord(b, h->stream));
  CUDA_TRY(cudaEventSynchronize(b));
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventElapsedTime(ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return check_range(h);
}

int bart_graph_active(bart_chain *h) { return h && h->graph ? 1 : 0; }



int bart_profile_forest(bart_chain *h, int reps, float *ms) {
  if (!h || !ms || reps < 1) return fail(BART_EINVAL, "bad arguments");
  if (int rc = bart_sync(h)) return rc;
  const ChainDev &c = h->c;
  DevBuf L2, pred;
  CUDA_TRY(L2.alloc((size_t)c.m * c.n_pad));
  CUDA_TRY(pred.alloc((size_t)c.n_pad * 8));
  cudaEvent_t e[4];
  for (auto &x : e) CUDA_TRY(cudaEventCreate(&x));
  auto traverse = [&] { launch_traverse(c.Xt, c.n, c.n_pad, c.D, c.half, c.m, c.axis, c.cut, L2.as<uint8_t>(), h->stream); };
  auto predict = [&] { launch_predict_cached(c.L, c.n, c.n_pad, c.m, c.size, c.leaf, pred.as<double>(), h->stream); };
  auto evaluate = [&] {
    launch_evaluate(c.Xt, c.n, c.n_pad, c.D, c.half, c.m, c.axis, c.cut, c.leaf, pred.as<double>(), h->stream);
  };
  traverse();  // warm-up
  predict();
  evaluate();
  CUDA_TRY(cudaEventRecord(e[0], h->stream));
  for (int i = 0; i < reps; ++i) traverse();
  CUDA_TRY(cudaEventRecord(e[1], h->stream));
  for (int i = 0; i < reps; ++i) predict();
  CUDA_TRY(cudaEventRecord(e[2], h->stream));
  for (int i = 0; i < reps; ++i) evaluate();
  CUDA_TRY(cudaEventRecord(e[3], h->stream));
  CUDA_TRY(cudaEventSynchronize(e[3]));
  CUDA_TRY(cudaGetLastError());
  for (int k = 0; k < 3; ++k) {
    CUDA_TRY(cudaEventElapsedTime(&ms[k], e[k], e[k + 1]));
    ms[k] /= (float)reps;
  }
  for (auto &x : e) cudaEventDestroy(x);
  h->launches += 3 * (int64_t)(reps + 1);
  return BART_OK;
}

int bart_profile(bart_chain *h, int64_t n_iter, float *ms) {
  if (!h || !ms) return fail(BART_EINVAL, "NULL argument");
  CUDA_TRY(cudaSetDevice(h->device));
  std::vector<cudaEvent_t> ev((size_t)(3 * n_iter + 2));
  for (auto &e : ev) CUDA_TRY(cudaEventCreate(&e));
  CUDA_TRY(cudaEventRecord(ev[0], h->stream));
  for (int64_t i = 0; i < n_iter; ++i) {
    CUDA_TRY(cudaEventRecord(ev[1 + 3 * i], h->stream));
    CUDA_TRY(cudaEventRecord(ev[2 + 3 * i], h->stream));
    CUDA_TRY((cudaError_t)sweep_launch(step_args(h, 1), h->smem, h->stream));
    CUDA_TRY(cudaEventRecord(ev[3 + 3 * i], h->stream));
    h->launches += 1;
    h->iteration += 1;
  }
  CUDA_TRY(cudaEventRecord(ev.back(), h->stream));
  CUDA_TRY(cudaEventSynchronize(ev.back()));
  float tot = 0.f, sw = 0.f, pr = 0.f, x = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&tot, ev[0], ev.back()));
  for (int64_t i = 0; i < n_iter; ++i) {
    CUDA_TRY(cudaEventElapsedTime(&x, ev[1 + 3 * i], ev[2 + 3 * i]));
    pr += x;
    CUDA_TRY(cudaEventElapsedTime(&x, ev[2 + 3 * i], ev[3 + 3 * i]));
    sw += x;
  }
  for (auto &e : ev) cudaEventDestroy(e);
  ms[0] = tot;
  ms[1] = sw;
  ms[2] = pr;
  return check_range(h);
}

}  // extern "C"
