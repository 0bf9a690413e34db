// capi.cu -- context lifetime, deferred error reporting, scratch arenas and
// the host-buffer (end-to-end) entry points of include/skx.h.
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <random>
#include <vector>

#include "skx_internal.cuh"

namespace skx {

int set_error(skx_ctx* ctx, int status, const char* fmt, ...) {
  if (!ctx) return status;
  ctx->last.status = status;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(ctx->last.message, sizeof ctx->last.message, fmt, ap);
  va_end(ap);
  return status;
}

int cuda_fail(skx_ctx* ctx, cudaError_t e, const char* where) {
  return set_error(ctx, SKX_CUDA_ERROR, "%s: %s", where, cudaGetErrorString(e));
}

// Stream-ordered growth: the old arena is released after the work already
// queued on s, the new one is valid for everything enqueued on s afterwards.
static void* grow(Scratch& sc, size_t bytes, cudaStream_t s) {
  if (sc.bytes >= bytes && sc.ptr) return sc.ptr;
  // Inside a CUDA Graph capture an allocation would belong to the graph, not
  // to the context: scratch must be reserved (skx_reserve) before capturing.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return nullptr;
  }
  if (sc.ptr) {
    cudaFreeAsync(sc.ptr, s);
    sc.ptr = nullptr;
    sc.bytes = 0;
  }
  size_t want = bytes < 4096 ? 4096 : bytes;
  if (cudaMallocAsync(&sc.ptr, want, s) != cudaSuccess) {
    cudaGetLastError();
    sc.ptr = nullptr;
    return nullptr;
  }
  sc.bytes = want;
  return sc.ptr;
}

static ScratchSet* set_for(skx_ctx* ctx, cudaStream_t s) {
  for (auto& st : ctx->sets)
    if (st.used && st.stream == s) return &st;
  for (auto& st : ctx->sets)
    if (!st.used) {
      st.used = true;
      st.stream = s;
      return &st;
    }
  // More streams than sets: recycle the least recently added set (rare;
  // callers normally use one or two streams).  Its stream may already be
  // destroyed, so drain the whole device before freeing its arenas.
  ScratchSet* victim = &ctx->sets[0];
  cudaDeviceSynchronize();
  for (auto& sc : victim->slot) {
    if (sc.ptr) cudaFree(sc.ptr);
    sc = Scratch{};
  }
  for (int i = 0; i + 1 < kScratchSets; ++i) ctx->sets[i] = ctx->sets[i + 1];
  ScratchSet* st = &ctx->sets[kScratchSets - 1];
  *st = ScratchSet{};
  st->used = true;
  st->stream = s;
  return st;
}

ScratchSet* scratch_set(skx_ctx* ctx, cudaStream_t s) { return set_for(ctx, s); }

void* scratch(skx_ctx* ctx, int slot, size_t bytes, cudaStream_t s) {
  return grow(set_for(ctx, s)->slot[slot], bytes, s);
}
void* host_scratch_dev(skx_ctx* ctx, int slot, size_t bytes, cudaStream_t s) {
  return grow(ctx->hb[slot], bytes, s);
}

static void reset_err_host(DevErr* e) {
  for (int i = 0; i < kViolSlots; ++i) e->viol[i] = ~0ull;
  e->invalid = 0;
  e->pad = 0;
  e->sum = 0;
}

}  // namespace skx

using namespace skx;

extern "C" {

int skx_version(void) { return 2; }

int skx_device_count(int* count) {
  if (!count) return SKX_INVALID_ARGUMENT;
  *count = 0;
  if (cudaGetDeviceCount(count) != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
  }
  return SKX_OK;
}

int skx_ctx_create(int device, skx_ctx** out) {
  if (!out) return SKX_INVALID_ARGUMENT;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return SKX_CUDA_ERROR;
  }
  if ((e = cudaSetDevice(device)) != cudaSuccess) return SKX_CUDA_ERROR;
  skx_ctx* ctx = new skx_ctx();
  ctx->device = device;
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major != 10) {
    delete ctx;
    fprintf(stderr, "skx: device %d is sm_%d%d; libskx.so is built for sm_100a only\n", device,
            prop.major, prop.minor);
    return SKX_CUDA_ERROR;
  }
  ctx->num_sms = prop.multiProcessorCount;
  ctx->smem_optin = prop.sharedMemPerBlockOptin;
  ctx->l2_bytes = prop.l2CacheSize;
  // Limits for the optional persisting L2 window (gather policy bit 4).  The
  // set-aside itself is only reserved while that bit is on: a reserved
  // set-aside shrinks the L2 available to normal accesses (measured).
  int pmax = 0, wmax = 0;
  cudaDeviceGetAttribute(&pmax, cudaDevAttrMaxPersistingL2CacheSize, device);
  cudaDeviceGetAttribute(&wmax, cudaDevAttrMaxAccessPolicyWindowSize, device);
  if (pmax > 0 && wmax > 0) {
    ctx->persist_max = (size_t)pmax;
    ctx->window_max = (size_t)wmax;
  }
  cudaGetLastError();
  if (cudaMalloc(&ctx->err, sizeof(DevErr)) != cudaSuccess ||
      cudaMallocHost(&ctx->err_host, sizeof(DevErr)) != cudaSuccess) {
    delete ctx;
    return SKX_CUDA_ERROR;
  }
  reset_err_host(ctx->err_host);
  cudaMemcpy(ctx->err, ctx->err_host, sizeof(DevErr), cudaMemcpyHostToDevice);
  for (auto& s : ctx->hstream) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (auto& ev : ctx->hevent) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  *out = ctx;
  return SKX_OK;
}

int skx_ctx_destroy(skx_ctx* ctx) {
  if (!ctx) return SKX_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  for (auto& st : ctx->sets)
    for (auto& sc : st.slot)
      if (sc.ptr) cudaFree(sc.ptr);
  for (auto& sc : ctx->hb)
    if (sc.ptr) cudaFree(sc.ptr);
  for (auto& s : ctx->hstream)
    if (s) cudaStreamDestroy(s);
  for (auto& ev : ctx->hevent)
    if (ev) cudaEventDestroy(ev);
  for (auto& pe : ctx->pg_cache)
    if (pe.ev) cudaEventDestroy(pe.ev);
  if (ctx->pg_host) cudaFreeHost(ctx->pg_host);
  if (ctx->pg_dev) cudaFree(ctx->pg_dev);
  cudaFree(ctx->err);
  cudaFreeHost(ctx->err_host);
  delete ctx;
  return SKX_OK;
}

uint64_t skx_launch_count(const skx_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

int skx_reserve(skx_ctx* ctx, int slot, uint64_t bytes, void* stream) {
  if (!ctx || slot < -1 || slot >= kScratchSlots) return SKX_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  cudaStream_t s = as_stream(stream);
  for (int i = (slot < 0 ? 0 : slot); i < (slot < 0 ? kScratchSlots : slot + 1); ++i)
    if (!scratch(ctx, i, bytes, s))
      return set_error(ctx, SKX_CUDA_ERROR, "reserve: out of device memory (%llu bytes)",
                       (unsigned long long)bytes);
  return SKX_OK;
}

int skx_scratch_bytes(const skx_ctx* ctx, void* stream, uint64_t* bytes) {
  if (!ctx || !bytes) return SKX_INVALID_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  for (int i = 0; i < kScratchSlots; ++i) bytes[i] = 0;
  for (const auto& st : ctx->sets)
    if (st.used && st.stream == s)
      for (int i = 0; i < kScratchSlots; ++i) bytes[i] = st.slot[i].bytes;
  return SKX_OK;
}

int skx_set_gather_policy(skx_ctx* ctx, int policy) {
  if (!ctx || policy < 0 || policy > 32767) return SKX_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  const bool want = (policy & 4) != 0 && ctx->persist_max > 0;
  if (want != ctx->setaside_on) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want ? ctx->persist_max : 0);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "set persisting L2 limit");
    if (!want) cudaCtxResetPersistingL2Cache();
    ctx->setaside_on = want;
  }
  ctx->gather_policy = policy;
  for (auto& pe : ctx->pg_cache)  // plans were made under the old policy; copies in flight finish
    if (!pe.pending) pe.state = 0;
    else pe.fact = nullptr;  // matches no launch; the slot is reused once its copy has landed
  return SKX_OK;
}

int skx_set_gather_tiers(skx_ctx* ctx, uint64_t smem_bytes, uint64_t l1_bytes, double l2_fraction) {
  if (!ctx || !(l2_fraction >= 0.0 && l2_fraction <= 1.0)) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  ctx->tier_smem_bytes = smem_bytes;
  ctx->tier_l1_bytes = l1_bytes;
  ctx->tier_l2_frac = l2_fraction;
  return SKX_OK;
}

int skx_set_histogram_mode(skx_ctx* ctx, int mode) {
  if (!ctx || mode < 0 || mode > 2) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  ctx->hist_mode = mode;
  return SKX_OK;
}

int skx_set_aggregate_mode(skx_ctx* ctx, int mode) {
  if (!ctx || mode < 0 || mode > 2) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  ctx->agg_mode = mode;
  return SKX_OK;
}

int skx_reset_persisting_l2(skx_ctx* ctx) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaCtxResetPersistingL2Cache();
  return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "reset_persisting_l2");
}

int skx_set_l2_fetch_granularity(skx_ctx* ctx, int bytes) {
  if (!ctx || (bytes != 32 && bytes != 64 && bytes != 128)) return SKX_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes);
  return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "set_l2_fetch_granularity");
}

int skx_device_info(skx_ctx* ctx, uint64_t* info, int n) {
  // [num_sms, smem_optin, l2_bytes, persist_max, window_max, l2_fetch_granularity]
  if (!ctx || !info) return SKX_INVALID_ARGUMENT;
  size_t gran = 0;
  cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
  const uint64_t v[6] = {(uint64_t)ctx->num_sms, ctx->smem_optin, ctx->l2_bytes, ctx->persist_max,
                         ctx->window_max, gran};
  for (int i = 0; i < n && i < 6; ++i) info[i] = v[i];
  return SKX_OK;
}

int skx_last_error(const skx_ctx* ctx, skx_error_info* info) {
  if (!ctx || !info) return SKX_INVALID_ARGUMENT;
  *info = ctx->last;
  return SKX_OK;
}

int skx_sync(skx_ctx* ctx, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaMemcpyAsync(ctx->err_host, ctx->err, sizeof(DevErr), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "skx_sync");
  DevErr h = *ctx->err_host;
  bool dirty = h.invalid != 0;
  for (int i = 0; i < kViolSlots; ++i) dirty |= h.viol[i] != ~0ull;
  if (!dirty) return SKX_OK;
  reset_err_host(ctx->err_host);
  cudaMemcpy(ctx->err, ctx->err_host, sizeof(DevErr), cudaMemcpyHostToDevice);
  for (int i = 0; i < kViolSlots; ++i) {
    if (h.viol[i] != ~0ull) {
      const uint64_t row = (uint64_t(i) << 32) | (h.viol[i] >> 32);
      const uint32_t value = static_cast<uint32_t>(h.viol[i]);
      ctx->last.row = row;
      ctx->last.value = value;
      ctx->last.domain = ctx->last_domain;
      return set_error(ctx, SKX_DOMAIN_VIOLATION, "domain violation at row %llu: value %u outside 1..%llu",
                       (unsigned long long)row, value, (unsigned long long)ctx->last_domain);
    }
  }
  return set_error(ctx, SKX_INVALID_ARGUMENT, "frequency profile counts do not sum to its total");
}

// ---- generator host side (column.cpp:44-71) --------------------------------

// simulate_lru (cachemodel.cpp:125-173): exact fully associative LRU over a
// trace of dense line ids -- a sequential recency list, host-side analysis
// code as in the reference.  stats = {accesses, hits, distinct lines}.
int skx_simulate_lru_host(const uint32_t* trace, uint64_t n, uint64_t cache_lines,
                          uint64_t* stats) {
  if (cache_lines == 0 || !stats || (n && !trace)) return SKX_INVALID_ARGUMENT;
  stats[0] = n;
  stats[1] = 0;
  stats[2] = 0;
  if (n == 0) return SKX_OK;
  uint32_t mx = 0;
  for (uint64_t i = 0; i < n; ++i) mx = trace[i] > mx ? trace[i] : mx;
  const size_t u = (size_t)mx + 1;
  constexpr uint32_t nil = 0xFFFFFFFFu;
  std::vector<uint32_t> prv(u, nil), nxt(u, nil);
  std::vector<uint8_t> resident(u, 0), seen(u, 0);
  uint32_t head = nil, tail = nil;
  uint64_t size = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t x = trace[i];
    if (!seen[x]) {
      seen[x] = 1;
      ++stats[2];
    }
    if (resident[x]) {
      ++stats[1];
      if (x == head) continue;
      if (prv[x] != nil) nxt[prv[x]] = nxt[x]; else head = nxt[x];
      if (nxt[x] != nil) prv[nxt[x]] = prv[x]; else tail = prv[x];
    } else {
      resident[x] = 1;
      ++size;
    }
    prv[x] = nil;
    nxt[x] = head;
    if (head != nil) prv[head] = x; else tail = x;
    head = x;
    if (size > cache_lines) {
      const uint32_t v = tail;
      tail = prv[v];
      if (tail != nil) nxt[tail] = nil; else head = nil;
      resident[v] = 0;
      --size;
    }
  }
  return SKX_OK;
}

int skx_zipf_cdf_host(uint32_t d, double z, double* cdf) {
  if (d == 0 || d > SKX_MAX_DOMAIN_CARDINALITY || !(z >= 0.0) || !cdf) return SKX_INVALID_ARGUMENT;
  // zipf_frequencies: Kahan-summed normaliser, column.cpp:44-60.
  double sum = 0.0, carry = 0.0;
  for (uint32_t r = 1; r <= d; ++r) {
    const double w = std::pow(static_cast<double>(r), -z);
    cdf[r - 1] = w;
    const double y = w - carry;
    const double t = sum + y;
    carry = (t - sum) - y;
    sum = t;
  }
  for (uint32_t i = 0; i < d; ++i) cdf[i] /= sum;
  // std::partial_sum, then cdf.back() = 1.0 (column.cpp:77-79).
  for (uint32_t i = 1; i < d; ++i) cdf[i] = cdf[i - 1] + cdf[i];
  cdf[d - 1] = 1.0;
  return SKX_OK;
}

int skx_random_bijection_host(uint32_t n, uint64_t seed, uint32_t* map) {
  if (!map && n) return SKX_INVALID_ARGUMENT;
  // Fisher-Yates with mt19937_64(seed), j = rng() % i (column.cpp:62-71).
  for (uint32_t i = 0; i < n; ++i) map[i] = i + 1;
  std::mt19937_64 rng(seed);
  for (uint32_t i = n; i > 1; --i) {
    const uint32_t j = static_cast<uint32_t>(rng() % i);
    const uint32_t t = map[i - 1];
    map[i - 1] = map[j];
    map[j] = t;
  }
  return SKX_OK;
}

// ---- host-buffer entry points ---------------------------------------------
// Chunked pipeline over two streams: H2D(fact chunk) -> kernel -> D2H(out
// chunk); chunk i+1's copy-in overlaps chunk i's kernel and copy-out.

int skx_materialize_host(skx_ctx* ctx, int w, const uint32_t* fact, uint64_t n, const void* dim,
                         uint64_t dim_len, void* out) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  if (w != 2 && w != 4 && w != 8) return set_error(ctx, SKX_INVALID_ARGUMENT, "bad value width");
  cudaSetDevice(ctx->device);
  const uint64_t chunk = uint64_t(1) << 25;  // rows per pipeline stage
  void* d_dim = host_scratch_dev(ctx, 0, dim_len * w + 16, ctx->hstream[0]);
  void* d_fact[2] = {host_scratch_dev(ctx, 1, chunk * 4, ctx->hstream[0]), host_scratch_dev(ctx, 2, chunk * 4, ctx->hstream[0])};
  void* d_out[2] = {host_scratch_dev(ctx, 3, chunk * w, ctx->hstream[0]), host_scratch_dev(ctx, 4, chunk * w, ctx->hstream[0])};
  if (!d_dim || !d_fact[0] || !d_fact[1] || !d_out[0] || !d_out[1])
    return set_error(ctx, SKX_CUDA_ERROR, "materialize_host: out of device memory");
  cudaError_t e = cudaMemcpyAsync(d_dim, dim, dim_len * w, cudaMemcpyHostToDevice, ctx->hstream[0]);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "materialize_host H2D dim");
  cudaEventRecord(ctx->hevent[2], ctx->hstream[0]);
  cudaStreamWaitEvent(ctx->hstream[1], ctx->hevent[2], 0);
  int rc = SKX_OK;
  for (uint64_t b = 0, i = 0; b < n; b += chunk, ++i) {
    const int s = static_cast<int>(i & 1);
    const uint64_t m = (n - b) < chunk ? (n - b) : chunk;
    cudaStream_t st = ctx->hstream[s];
    cudaMemcpyAsync(d_fact[s], fact + b, m * 4, cudaMemcpyHostToDevice, st);
    rc = launch_gather(ctx, w, static_cast<const uint32_t*>(d_fact[s]), m, d_dim, dim_len, d_out[s], st);
    if (rc) break;
    cudaMemcpyAsync(static_cast<char*>(out) + b * w, d_out[s], m * w, cudaMemcpyDeviceToHost, st);
  }
  cudaStreamSynchronize(ctx->hstream[0]);
  cudaStreamSynchronize(ctx->hstream[1]);
  if (rc) return rc;
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "materialize_host");
  rc = skx_sync(ctx, ctx->hstream[0]);
  if (rc == SKX_DOMAIN_VIOLATION) {
    // Chunk launches record chunk-local rows; find the first offending global
    // row on the host (cold path only).
    for (uint64_t k = 0; k < n; ++k) {
      if (fact[k] - 1u >= dim_len) {
        ctx->last.row = k;
        ctx->last.value = fact[k];
        ctx->last.domain = dim_len;
        return set_error(ctx, SKX_DOMAIN_VIOLATION, "domain violation at row %llu: value %u outside 1..%llu",
                         (unsigned long long)k, fact[k], (unsigned long long)dim_len);
      }
    }
  }
  return rc;
}

int skx_aggregate_host(skx_ctx* ctx, const uint32_t* fact, const void* measure, int mw, uint64_t n,
                       uint32_t d, uint32_t hot, uint64_t* counts, uint64_t* sums) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  if (mw != 0 && mw != 4 && mw != 8) return set_error(ctx, SKX_INVALID_ARGUMENT, "bad measure width");
  cudaSetDevice(ctx->device);
  void* d_fact = host_scratch_dev(ctx, 1, n * 4 + 16, ctx->hstream[0]);
  void* d_meas = mw ? host_scratch_dev(ctx, 3, n * mw + 16, ctx->hstream[0]) : nullptr;
  void* d_out = host_scratch_dev(ctx, 0, uint64_t(d) * 16 + 16, ctx->hstream[0]);
  if (!d_fact || (mw && !d_meas) || !d_out)
    return set_error(ctx, SKX_CUDA_ERROR, "aggregate_host: out of device memory");
  cudaStream_t st = ctx->hstream[0];
  cudaMemcpyAsync(d_fact, fact, n * 4, cudaMemcpyHostToDevice, st);
  if (mw) cudaMemcpyAsync(d_meas, measure, n * mw, cudaMemcpyHostToDevice, st);
  uint64_t* dc = static_cast<uint64_t*>(d_out);
  uint64_t* ds = dc + d;
  int rc = launch_aggregate(ctx, static_cast<const uint32_t*>(d_fact), d_meas, mw, n, d, hot,
                            counts ? dc : nullptr, sums ? ds : nullptr, st);
  if (rc) return rc;
  if (counts) cudaMemcpyAsync(counts, dc, uint64_t(d) * 8, cudaMemcpyDeviceToHost, st);
  if (sums) cudaMemcpyAsync(sums, ds, uint64_t(d) * 8, cudaMemcpyDeviceToHost, st);
  return skx_sync(ctx, st);
}

}  // extern "C"

// ---- device memory for host-side callers -----------------------------------
namespace skx {
namespace {
__global__ void k_domain_scan(const uint32_t* __restrict__ fact, uint64_t n, uint64_t d,
                              DevErr* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    const uint32_t id = fact[k];
    if ((uint64_t)(uint32_t)(id - 1u) >= d) record_violation(err, k, id);
  }
}
}  // namespace
}  // namespace skx

extern "C" {

int skx_device_alloc(skx_ctx* ctx, uint64_t bytes, void** ptr) {
  if (!ctx || !ptr) return SKX_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  *ptr = nullptr;
  cudaError_t e = cudaMalloc(ptr, bytes ? bytes : 16);
  return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "device_alloc");
}

int skx_device_free(skx_ctx* ctx, void* ptr) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (!ptr) return SKX_OK;
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "device_free");
}

int skx_copy_to_device(skx_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (!bytes) return SKX_OK;
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
  return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "copy_to_device");
}

int skx_copy_to_host(skx_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (!bytes) return SKX_OK;
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "copy_to_host");
}

int skx_pinned_alloc(skx_ctx* ctx, uint64_t bytes, void** ptr) {
  if (!ctx || !ptr) return SKX_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  *ptr = nullptr;
  cudaError_t e = cudaHostAlloc(ptr, bytes ? bytes : 16, cudaHostAllocPortable);
  return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "pinned_alloc");
}

int skx_pinned_free(skx_ctx* ctx, void* ptr) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  if (!ptr) return SKX_OK;
  cudaError_t e = cudaFreeHost(ptr);
  return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "pinned_free");
}

void* skx_ctx_stream(skx_ctx* ctx, int slot) {
  if (!ctx || slot < 0 || slot > 1) return nullptr;
  skx::bind(ctx);
  return ctx->hstream[slot];
}

int skx_copy_to_device_async(skx_ctx* ctx, void* dst, const void* src, uint64_t bytes,
                             void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (!bytes) return SKX_OK;
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream));
  return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "copy_to_device_async");
}

int skx_copy_to_host_async(skx_ctx* ctx, void* dst, const void* src, uint64_t bytes,
                           void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (!bytes) return SKX_OK;
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream));
  return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "copy_to_host_async");
}

int skx_find_domain_violation(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint64_t d,
                              uint64_t* row_out) {
  if (!ctx || !row_out) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  *row_out = ~0ull;
  if (n == 0) return SKX_OK;
  if (n > (uint64_t(1) << 34)) return set_error(ctx, SKX_INVALID_ARGUMENT, "more than 2^34 rows");
  cudaSetDevice(ctx->device);
  ctx->last_domain = d;
  k_domain_scan<<<grid_for(ctx, n, 256, 8), 256>>>(fact, n, d, ctx->err);
  ctx->launches++;
  const int rc = skx_sync(ctx, nullptr);
  if (rc == SKX_DOMAIN_VIOLATION) {
    *row_out = ctx->last.row;
    return SKX_OK;
  }
  return rc;
}

}  // extern "C"
