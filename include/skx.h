/*
 * skx.h -- C-ABI of the B200-native skew-aware repositioning index and the
 * operators it accelerates (libskx.so, built from paper_1910_10063_b200/csrc).
 *
 * This is the drop-in boundary for the reference library "skewdx"
 * (/root/reference/proj).  The reference exposes its hot path two ways:
 *   (1) the C function-pointer plugin table skewdx::kernels::KernelTable
 *       (proj/include/skewdx/kernels.hpp:16-41), and
 *   (2) the C++ operator API in permindex.hpp:34-59, operators.hpp:57-122 and
 *       parallel.hpp:34-61.
 * Each entry below names the reference interface it replaces.  Plain
 * pointers and sizes only; no torch or C++ types cross this boundary.
 *
 * Conventions
 *  - Identifiers are 1-based; id 0 and id > D are domain violations
 *    (operators.cpp:33-38: `fact[k] - 1 >= D` in u32 arithmetic).
 *  - Device entry points take DEVICE pointers and a cudaStream_t passed as
 *    `void* stream` (NULL = legacy default stream).  They are asynchronous:
 *    they enqueue work and return SKX_OK unless an argument is rejected on
 *    the host.  Device-detected errors (domain violations, a frequency profile
 *    whose counts do not sum to its total) are recorded in the context and
 *    reported by the next skx_sync() on that context -- the first offending
 *    row, exactly as DomainViolation::row() reports it (error.hpp:20-33).
 *    Enqueue one operator and skx_sync() to attribute an error to it; the
 *    C++ drop-in (the cpp/include/skewdx headers over libskewdx_b200.so) does that and rethrows the
 *    reference's exception types.
 *  - A context belongs to one device and one host thread.  It owns the
 *    scratch memory, kept as one set of arenas per stream: operators enqueued
 *    on the same stream share that stream's set (so they are ordered), and
 *    operators on different streams never share scratch.  Arenas grow
 *    stream-ordered (cudaMallocAsync / cudaFreeAsync on the operator's
 *    stream), so no operator synchronises the device; skx_reserve() grows
 *    them up front -- required before capturing operators into a CUDA Graph
 *    (an arena cannot grow during capture: the operator returns
 *    SKX_CUDA_ERROR "out of device memory").  Callers own every input and
 *    output buffer.
 *  - Host-buffer entry points (suffix _host) copy host -> device, run the
 *    kernel and copy back, pipelined in chunks over two streams; they are
 *    synchronous and report errors directly.
 */
#ifndef SKX_H_
#define SKX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (mirror error.hpp:12-49). */
#define SKX_OK 0
#define SKX_INVALID_ARGUMENT 1 /* skewdx::InvalidArgument */
#define SKX_DOMAIN_VIOLATION 2 /* skewdx::DomainViolation{row, value, domain} */
#define SKX_CUDA_ERROR 3
#define SKX_NCCL_ERROR 4 /* a collective failed (multi-GPU combine steps) */
#define SKX_ERROR 5 /* any other skewdx::Error */

/* kMaxDomainCardinality, column.hpp:17 */
#define SKX_MAX_DOMAIN_CARDINALITY 0xFFFFFFFEu

typedef struct skx_ctx skx_ctx;
typedef struct skx_comm skx_comm;

typedef struct skx_error_info {
  int32_t status;
  uint64_t row;    /* DomainViolation::row()   */
  uint32_t value;  /* DomainViolation::value() */
  uint64_t domain; /* the D the row was checked against */
  char message[256];
} skx_error_info;

/* ---- context ------------------------------------------------------------ */
int skx_version(void);
/* Number of visible CUDA devices (0 when none). */
int skx_device_count(int* count);
int skx_ctx_create(int device, skx_ctx** out);
int skx_ctx_destroy(skx_ctx* ctx);
/* Waits for `stream`, then reports (and clears) any deferred device error. */
int skx_sync(skx_ctx* ctx, void* stream);
/* Details of the last non-OK status returned on this context. */
int skx_last_error(const skx_ctx* ctx, skx_error_info* info);
/* Number of kernels this context has launched since creation (bench evidence). */
uint64_t skx_launch_count(const skx_ctx* ctx);
/* Grow scratch arena `slot` (0..3, or -1 = all four) of `stream`'s set to at
 * least `bytes`, stream-ordered on `stream`.  Operators grow their arenas on
 * demand the same way; reserving first keeps allocation out of a timed or
 * captured region.  Slots: 0 histogram / index sort / group-by staging,
 * 1 rebuild counters / group-by accumulators / cache model, 2 selection,
 * 3 spare.  No reference counterpart (the reference allocates per call). */
int skx_reserve(skx_ctx* ctx, int slot, uint64_t bytes, void* stream);
/* Current arena sizes (bytes[0..4)) of `stream`'s set (0 when it has none). */
int skx_scratch_bytes(const skx_ctx* ctx, void* stream, uint64_t* bytes);

/* ---- device memory for host-side callers (the C++ drop-in) --------------- */
int skx_device_alloc(skx_ctx* ctx, uint64_t bytes, void** ptr);
int skx_device_free(skx_ctx* ctx, void* ptr);
/* Synchronous copies on the context's device. */
int skx_copy_to_device(skx_ctx* ctx, void* dst, const void* src, uint64_t bytes);
int skx_copy_to_host(skx_ctx* ctx, void* dst, const void* src, uint64_t bytes);
/* Streamed callers (SKDX columns streamed host -> device
 * through pinned memory; no reference counterpart -- the reference reads a
 * whole column into a std::vector, column_io.cpp:89-95).  Pinned host
 * buffers, the context's two host-side streams (slot 0 / 1), and
 * asynchronous copies on a stream; completion and deferred device errors
 * are reported by skx_sync(ctx, stream). */
int skx_pinned_alloc(skx_ctx* ctx, uint64_t bytes, void** ptr);
int skx_pinned_free(skx_ctx* ctx, void* ptr);
void* skx_ctx_stream(skx_ctx* ctx, int slot);
int skx_copy_to_device_async(skx_ctx* ctx, void* dst, const void* src, uint64_t bytes,
                             void* stream);
int skx_copy_to_host_async(skx_ctx* ctx, void* dst, const void* src, uint64_t bytes,
                           void* stream);

/* find_domain_violation (operators.cpp:32-41): *row_out (host) = the first k
 * with fact[k]-1 >= d, or UINT64_MAX.  Synchronous. */
int skx_find_domain_violation(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint64_t d,
                              uint64_t* row_out);

/* ---- Q1 gather: out[k] = dim[fact[k]-1] --------------------------------- *
 * Replaces KernelTable::gather_u32 (kernels.hpp:21-23; scalar.cpp:13-29,
 * avx2.cpp:43-57) and the operator materialize() (operators.cpp:60-66) /
 * parallel_materialize() (parallel.cpp:87-100), with the domain check of
 * find_domain_violation (operators.cpp:32-41) fused into the same pass.
 * Unlike the table entry it carries dim_len, so the device can bound-check.
 * u16/u64 widths restate the same contract for BASELINE's int16/int64/f32
 * value columns (bit moves; f32 and i32 go through _u32). */
int skx_gather_u16(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint16_t* dim,
                   uint64_t dim_len, uint16_t* out, void* stream);
int skx_gather_u32(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint32_t* dim,
                   uint64_t dim_len, uint32_t* out, void* stream);
int skx_gather_u64(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint64_t* dim,
                   uint64_t dim_len, uint64_t* out, void* stream);

/* Threshold-split materialize: materialize_split
 * (operators.cpp:68-85) over KernelTable::gather_split_pass1 (kernels.hpp:
 * 32-39): pass 1 gathers rows with id <= threshold and queues the others,
 * pass 2 patches the queued rows.  Same result as skx_gather_*; threshold
 * must lie in 1..dim_len (SKX_INVALID_ARGUMENT otherwise), n < 2^32. */
int skx_gather_split_u32(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint32_t* dim,
                         uint64_t dim_len, uint32_t threshold, uint32_t* out, void* stream);
int skx_gather_split_u64(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint64_t* dim,
                         uint64_t dim_len, uint32_t threshold, uint64_t* out, void* stream);

/* ---- index build (permindex.cpp) ---------------------------------------- */
/* count_frequencies (permindex.cpp:18-30): counts[id-1] = #rows with id.
 * `counts` (u64[d]) is overwritten. */
int skx_count_frequencies(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d,
                          uint64_t* counts, void* stream);
/* Same histogram into u32 counters (the per-GPU partial that is NCCL
 * all-reduced before the sort, BASELINE config 4).  accumulate != 0 adds to
 * the existing counters instead of overwriting them. */
int skx_histogram_u32(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d,
                      uint32_t* counts, int accumulate, void* stream);
/* build_index (permindex.cpp:32-58): offsets = ids ordered by (count desc,
 * id asc), zero-count ids last in ascending order; ranks = inverse
 * (ranks[offsets[r]-1] = r+1).  Counts must sum to `total` (deferred
 * SKX_INVALID_ARGUMENT otherwise, permindex.cpp:36-40). */
int skx_build_index(skx_ctx* ctx, const uint64_t* counts, uint32_t d, uint64_t total,
                    uint32_t* offsets, uint32_t* ranks, void* stream);
int skx_build_index_u32(skx_ctx* ctx, const uint32_t* counts, uint32_t d, uint64_t total,
                        uint32_t* offsets, uint32_t* ranks, void* stream);
/* rebuild (permindex.cpp:86-88) = count_frequencies + build_index. */
int skx_rebuild(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d, uint32_t* offsets,
                uint32_t* ranks, void* stream);
/* recode_fact (permindex.cpp:60-64): out[k] = ranks[fact[k]-1]. */
int skx_recode_fact(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint32_t* ranks,
                    uint32_t d, uint32_t* out, void* stream);
/* permute_dimension (permindex.cpp:66-73): out[r] = dim[offsets[r]-1];
 * dim_len must equal d (SKX_INVALID_ARGUMENT otherwise). */
int skx_permute_dimension_u16(skx_ctx* ctx, const uint16_t* dim, uint64_t dim_len,
                              const uint32_t* offsets, uint32_t d, uint16_t* out, void* stream);
int skx_permute_dimension_u32(skx_ctx* ctx, const uint32_t* dim, uint64_t dim_len,
                              const uint32_t* offsets, uint32_t d, uint32_t* out, void* stream);
int skx_permute_dimension_u64(skx_ctx* ctx, const uint64_t* dim, uint64_t dim_len,
                              const uint32_t* offsets, uint32_t d, uint64_t* out, void* stream);

/* ---- Q3 group-by --------------------------------------------------------- *
 * aggregate_count / aggregate_sum (operators.cpp:100-118) and the hybrid
 * parallel_aggregate (parallel.cpp:178-207): ids <= hot_threshold are
 * accumulated in per-CTA shared-memory bins, the tail in global atomics.
 * measure_width is 0 (no measure; sums ignored), 4 (u32, the reference's
 * Column measure) or 8 (u64, BASELINE config 3's int64 quantity).
 * counts and/or sums (u64[d]) may be NULL; both are overwritten.
 * hot_threshold 0 = automatic (as many ids as fit shared memory).  Results
 * do not depend on it (parallel.hpp:51-53). */
int skx_aggregate(skx_ctx* ctx, const uint32_t* fact, const void* measure, int measure_width,
                  uint64_t n, uint32_t d, uint32_t hot_threshold, uint64_t* counts,
                  uint64_t* sums, void* stream);

/* ---- Q2 selection -------------------------------------------------------- *
 * KernelTable::select_offsets (kernels.hpp:25-30; scalar.cpp:31-42) and
 * select()/parallel_select() (operators.cpp:87-98, parallel.cpp:102-129):
 * ascending base+k for every row whose bit fact[k]-1 is set in the packed
 * little-endian bitmap of `bits` bits.  n must be <= UINT32_MAX.  The number
 * written goes to *count_dev (device u64). */
int skx_select_offsets(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint64_t* words,
                       uint64_t bits, uint32_t base, uint32_t* out, uint64_t* count_dev,
                       void* stream);
/* permute_bitmap (operators.cpp:21-30): out bit r = in bit offsets[r]-1. */
int skx_permute_bitmap(skx_ctx* ctx, const uint64_t* words, uint64_t bits,
                       const uint32_t* offsets, uint32_t d, uint64_t* out_words, void* stream);
/* build_bitmap(dim, v < threshold) (operators.hpp:38-45) for an int32 column. */
int skx_build_bitmap_lt_i32(skx_ctx* ctx, const int32_t* dim, uint64_t d, int32_t threshold,
                            uint64_t* out_words, void* stream);
/* BASELINE config 5, fused: select rows whose bit is set, gather the four
 * dimension columns (i32 category, f32 price, u64 supplier, u16 flag) for
 * the selected rows in ascending row order, and SUM(price) per category
 * (sums[n_categories] as fp64, overwritten; categories outside
 * [0, n_categories) are not summed): exact 96-bit fixed point when the
 * prices are finite, span <= 2^30 in exponent and n_categories <= 4096,
 * else an fp64 reduction (decided on the device).  Offsets get `base` added.
 * The output columns hold `capacity` rows: *count_dev always receives the
 * true number of selected rows; when it exceeds capacity only the first
 * capacity rows are written (and the sums are unspecified) -- call again
 * with capacity >= *count_dev (the reference returns exactly-sized vectors,
 * operators.cpp:87-98; a device caller sizes its buffers up front). */
int skx_select_gather_sum(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint64_t* words,
                          uint32_t d, const int32_t* cat, const float* price,
                          const uint64_t* supp, const uint16_t* flag, uint32_t base,
                          uint32_t n_categories, uint64_t capacity, uint32_t* out_off,
                          int32_t* out_cat, float* out_price, uint64_t* out_supp,
                          uint16_t* out_flag, double* sums, uint64_t* count_dev, void* stream);

/* Cross-GPU combine of config 5's category sums: the exact
 * partial of the last skx_select_gather_sum enqueued on `stream`, as int64
 * out[2 + 3 * n_categories]: out[0] = 1 if that call summed in 96-bit fixed
 * point (else 0), out[1] = its scale S, out[2 + 3c ...] = the low / middle
 * (unsigned) and high (signed) 32-bit limbs of category c's sum.  An
 * element-wise integer SUM of these over ranks (skx_reduce, SKX_DT_I64) is
 * exact; skx_select_sums_from_partials then writes sums[c] = total * 2^-S when
 * all `nranks` ranks summed in fixed point with the same S, and leaves
 * `sums` (the fp64-reduced sums) untouched otherwise.  The reference sums
 * nothing across workers for this config; its fold order is the chunk order
 * of parallel.cpp:102-129. */
int skx_select_sum_partials(skx_ctx* ctx, uint32_t n_categories, int64_t* out, void* stream);
int skx_select_sums_from_partials(skx_ctx* ctx, const int64_t* partials, uint32_t n_categories,
                                  uint32_t nranks, double* sums, void* stream);

/* ---- Q3a heavy hitters (operators.cpp:184-203) ---------------------------- *
 * counts[i] = #rows with id i+1 for i < min(k, d) on a recoded column. */
int skx_heavy_hitter_count(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d,
                           uint32_t k, uint64_t* counts, void* stream);

/* ---- workload generator (column.cpp:44-125) ------------------------------ */
/* zipf_frequencies + partial_sum with cdf[d-1] = 1.0 (column.cpp:44-60,
 * 77-79), on the host, bit-identical to the reference's doubles. */
int skx_zipf_cdf_host(uint32_t d, double z, double* cdf);
/* random_bijection (column.cpp:62-71), host, bit-identical (mt19937_64). */
int skx_random_bijection_host(uint32_t n, uint64_t seed, uint32_t* out);
/* Counter-based parallel Zipf draw on the device:
 * u_k = (splitmix64(splitmix64(seed^0x5ca1ab1e) + k*0x9e3779b97f4a7c15)>>11)
 * * 2^-53 for global row k = row_begin + i, rank = upper_bound(cdf, u)
 * (clamped to d-1), out[i] = rank_to_id[rank] (or rank+1 when NULL). */
int skx_generate_zipf(skx_ctx* ctx, const double* cdf, uint32_t d, const uint32_t* rank_to_id,
                      uint64_t seed, uint64_t row_begin, uint64_t n, uint32_t* out,
                      void* stream);

/* Value-column fixtures for the BASELINE configs (device).  kind 0: raw
 * splitmix64(seed ^ (0xd1000000 + i)) truncated to width bytes (the reference
 * bench's dimension column, dataset.cpp:35-38); kind 1: integer
 * p0 + splitmix64(seed + i*0x9e3779b97f4a7c15) % p1; kind 2: float32
 * lognormal(mu=p0, sigma=p1) (Box-Muller in fp64), width must be 4. */
int skx_fill_column(skx_ctx* ctx, int kind, int width, uint64_t seed, uint64_t n, double p0,
                    double p1, void* out, void* stream);

/* ---- cache model (cachemodel.hpp) ------------------------ *
 * line_frequencies (cachemodel.cpp:22-45): out[l] = sum of value_freqs[r]
 * over the ranks r whose element lands in line l, accumulated in ascending
 * rank order (bit-identical to the reference).  rank_to_id NULL = freq layout
 * (rank r is element r); else element rank_to_id[r]-1 (the rand layout's
 * random_bijection, skx_random_bijection_host).  per_line = line_bytes /
 * element_bytes (1..256 with a bijection).  Device pointers, d doubles in,
 * ceil(d / per_line) doubles out. */
int skx_line_frequencies(skx_ctx* ctx, const double* value_freqs, uint32_t d,
                         const uint32_t* rank_to_id, uint32_t per_line, double* out,
                         void* stream);
/* estimate_hit_rate (cachemodel.cpp:76-123): analytical LRU hit rate of an
 * access stream with independent per-line frequencies, for a cache of
 * cache_lines lines; *result (device double) written on `stream`.  Matches
 * the reference to rounding (parallel prefix sums). */
int skx_estimate_hit_rate(skx_ctx* ctx, const double* line_freqs, uint64_t nlines,
                          uint64_t cache_lines, double* result, void* stream);
/* trace_from_column (cachemodel.cpp:175-186): out[k] = (fact[k]-1)/per_line;
 * an id 0 is a DomainViolation (deferred to skx_sync, domain 0xFFFFFFFE). */
int skx_trace_from_column(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t per_line,
                          uint32_t* out, void* stream);
/* simulate_lru (cachemodel.cpp:125-173), host: exact LRU over a host trace;
 * stats[0..3) = {accesses, hits, distinct lines}. */
int skx_simulate_lru_host(const uint32_t* trace, uint64_t n, uint64_t cache_lines,
                          uint64_t* stats);

/* ---- host-buffer entry points (what a reference caller hands over) ------- *
 * materialize() with host vectors: value_width 2, 4 or 8.  fact/dim/out are
 * HOST pointers (pinned or pageable).  Synchronous. */
int skx_materialize_host(skx_ctx* ctx, int value_width, const uint32_t* fact, uint64_t n,
                         const void* dim, uint64_t dim_len, void* out);
/* aggregate with host buffers (counts/sums are host u64[d]). */
int skx_aggregate_host(skx_ctx* ctx, const uint32_t* fact, const void* measure,
                       int measure_width, uint64_t n, uint32_t d, uint32_t hot_threshold,
                       uint64_t* counts, uint64_t* sums);

/* ---- multi-GPU: NCCL communicators and the combine steps ---------------- *
 * SURVEY §8(b)/(e).  The reference combines per-worker partials on the host
 * after its fork-join (parallel.cpp:147-207 fold; parallel_select's ordered
 * concatenation, parallel.cpp:102-129); across GPUs those folds are NCCL
 * collectives over NVLink / NVSwitch.  A communicator spans either several
 * devices of this process (skx_comm_init_all: ncclCommInitAll, one context and
 * one stream per device -- the C++ drop-in's multi-device overloads) or one
 * device of a process-per-GPU job (skx_comm_init_rank with the 128-byte id
 * from skx_comm_unique_id on rank 0).  Collectives take one buffer per LOCAL
 * device (bufs[0..nlocal)) and optional per-device streams (NULL = the
 * communicator's own streams), are asynchronous, and are group-launched
 * across local devices.  Failures return SKX_NCCL_ERROR with the message in
 * skx_comm_error() and in every local context's skx_last_error(). */
#define SKX_COMM_MAX_LOCAL 16
#define SKX_DT_U32 0
#define SKX_DT_I32 1
#define SKX_DT_U64 2
#define SKX_DT_I64 3
#define SKX_DT_F64 4
#define SKX_OP_SUM 0
#define SKX_OP_MIN 1
#define SKX_OP_MAX 2
int skx_comm_init_all(int ndev, const int* devices, skx_comm** out);
int skx_comm_unique_id(void* id128);
int skx_comm_init_rank(int device, int nranks, int rank, const void* id128, skx_comm** out);
int skx_comm_destroy(skx_comm* comm);
int skx_comm_info(const skx_comm* comm, int* nranks, int* rank0, int* nlocal);
skx_ctx* skx_comm_ctx(skx_comm* comm, int local);
void* skx_comm_stream(skx_comm* comm, int local);
const char* skx_comm_error(const skx_comm* comm);
/* Waits for every local stream and reports asynchronous NCCL errors. */
int skx_comm_sync(skx_comm* comm);
int skx_allreduce(skx_comm* comm, void* const* bufs, uint64_t count, int dtype, int op,
                  void* const* streams);
int skx_reduce(skx_comm* comm, void* const* bufs, uint64_t count, int dtype, int op, int root,
               void* const* streams);
int skx_reduce_scatter(skx_comm* comm, void* const* send, void* const* recv, uint64_t recvcount,
                       int dtype, int op, void* const* streams);
int skx_allgather(skx_comm* comm, void* const* send, void* const* recv, uint64_t sendcount,
                  int dtype, void* const* streams);
int skx_broadcast(skx_comm* comm, void* const* bufs, uint64_t count, int dtype, int root,
                  void* const* streams);

/* Group-by partials in the combine layout (config 3's per-GPU partials
 * reduced to a root): buf (u64[d + hot]) = [counts[0..hot) | sums[0..hot) |
 * packed[hot..d)] with packed[i] = counts[i] << 40 | sums[i] -- 8 B per tail
 * key instead of 16.  guard (device u64[2]) = max tail count and max tail
 * sum of this rank; after a SUM all-reduce of the guards over ranks,
 * skx_groupby_packed_ok(host copy) says whether a u64 SUM-reduce of the
 * packed buffers is exact (no field can overflow: counts < 2^24, sums <
 * 2^40).  Otherwise reduce counts and sums directly.  sums may be NULL
 * (COUNT only).  The reference's fold is parallel.cpp:155-157. */
int skx_groupby_pack(skx_ctx* ctx, const uint64_t* counts, const uint64_t* sums, uint32_t d,
                     uint32_t hot, uint64_t* buf, uint64_t* guard, void* stream);
int skx_groupby_unpack(skx_ctx* ctx, const uint64_t* buf, uint32_t d, uint32_t hot,
                       uint64_t* counts, uint64_t* sums, void* stream);
int skx_groupby_packed_ok(const uint64_t* guard_sum);

/* ---- tuning / evidence ---------------------------------------------------- *
 * Cache policy of the gathers (materialize/recode/permute), a bit set:
 *   1 = evict_first on the streamed FK/output, evict_last on dimension reads;
 *   2 = hot prefix in shared memory: the leading dimension values (the most
 *       popular ids after reordering) are staged per CTA and served on chip;
 *   4 = L2 access-policy window (persisting) over the dimension bytes after
 *       the shared-memory tier;
 *   8 = dimension loads bypass L1 allocation;
 *  16 = FK stream software-pipelined one iteration ahead;
 *  32 = tiered: the reordered id selects the cache class of each dimension
 *       load -- ids below t1 allocate in L1, ids below t2 are L2 evict_last,
 *       colder ids are L2 evict_first and skip L1 (skx_set_gather_tiers);
 *  64 = diagnostic: loads only, output stores dropped (NOT a valid gather);
 * 128 = FK stream / output use the .cs (streaming) cache operator;
 * 256, 512 = int64 dimension loads via the coherent / .cg (L2-only) path;
 * 2048 = output staged per CTA and written with 8 KB bulk stores;
 * 4096 = int64 output as 256-bit stores;
 * 8192 = partitioned gather for columns whose rows mostly miss L2: the cold
 *       rows are radix-partitioned by key range and their values fetched
 *       slice by slice while each dimension slice is L2-resident (the GPU form
 *       of a partitioned join; needs ~4 + 4 + 2 x width bytes of scratch per
 *       row, and falls back to the one-pass kernel without it).  Whether a
 *       column takes it is planned on the device: the first launch over a
 *       (fact pointer, rows, dimension pointer, length) pair runs the one-pass
 *       kernel and a plan kernel that samples 64 K rows; the plan is copied
 *       back asynchronously, and once it has landed later launches over the
 *       same pair follow it -- partitioned when >= 30% of the sample are first
 *       touches of dimension lines past the L2-resident prefix, the launch
 *       touches each such line >= 4 times and the ids do not walk the
 *       dimension in order; one pass otherwise (skew-reordered columns at
 *       s >= ~1, in-order permutes, heavy-hitter recodes).  Plans are
 *       refreshed in the background every 16 launches and dropped by
 *       skx_set_gather_policy; a stale plan (the buffer now holds another
 *       column) can cost time but never changes a result.  Inside a CUDA
 *       Graph capture the one-pass kernel runs;
 * 16384 = with 8192: take the partitioned path at once, whatever a plan says.
 * Default 8321 (= 1 | 128 | 8192); measurements in profiles/r1_experiments.md
 * and profiles/r2_experiments.md. */
int skx_set_gather_policy(skx_ctx* ctx, int policy);
/* Evidence: the last gather launched on this context, after draining `stream`
 * (which must be the stream it ran on): info[0] = 1 when it ran the
 * partitioned kernels; info[3] = its column's plan (1 = partitioned: what the
 * next launches over the same column take); info[1] = sampled rows (of 65536)
 * the plan counted as miss candidates, info[2] = ascending adjacent id pairs
 * inside the sampled 4-row vectors (of 49152; >= 80% marks an in-order walk).
 * info must hold 4 words; info[1..3] are 0 for launches that were not planned
 * (policy bit off, small or narrow columns, forced path: info[3] = info[0]). */
int skx_gather_last_plan(skx_ctx* ctx, uint32_t* info, void* stream);
/* cudaLimitMaxL2FetchGranularity (32, 64 or 128 bytes): device-wide. */
int skx_set_l2_fetch_granularity(skx_ctx* ctx, int bytes);
/* Tier sizes: shared-memory tier (policy bit 2) capped at smem_bytes (0 = all
 * opt-in shared memory); for policy bit 32, t1 = hot + l1_bytes / width and
 * t2 = l2_fraction * L2 size / width. */
int skx_set_gather_tiers(skx_ctx* ctx, uint64_t smem_bytes, uint64_t l1_bytes,
                         double l2_fraction);
/* Histogram cold-key handling for domains whose counters exceed half of L2:
 * 0 = default: beyond 3x L2, packed 16-bit counters (two keys per word)
 *     checked on the device against the exact cold-row count, with a gated
 *     direct recount on a wrap (only when the call starts from zeroed
 *     counts); otherwise direct reductions,
 * 1 = cold keys staged per key-range bucket and applied while L2-resident,
 * 2 = direct 32/64-bit reductions. */
int skx_set_histogram_mode(skx_ctx* ctx, int mode);
/* Group-by (measure_width 4/8) cold-tail strategy:
 * 0 = packed (default): one 64-bit reduction of (1 << 40 | m) per cold row
 *     into an 8 B/key accumulator, decoded and validated on the device
 *     against exact per-launch totals; rows with m >= 2^16 or a failed check
 *     rerun the call through mode 2 on the device (no host round trip);
 * 1 = staged per key-range bucket and folded while L2-resident, when the
 *     tail pairs exceed half of L2 (else mode 2);
 * 2 = direct: two 64-bit reductions per cold row on an interleaved
 *     {count, sum} pair. */
int skx_set_aggregate_mode(skx_ctx* ctx, int mode);
/* cudaCtxResetPersistingL2Cache: demote lines left persisting by windows. */
int skx_reset_persisting_l2(skx_ctx* ctx);
/* info[0..n): num_sms, smem_optin, l2_bytes, persisting-L2 max, access-policy
 * window max, current L2 fetch granularity. */
int skx_device_info(skx_ctx* ctx, uint64_t* info, int n);

#ifdef __cplusplus
}
#endif
#endif /* SKX_H_ */
