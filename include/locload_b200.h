/*
 * locload_b200.h -- C-ABI of the B200-native locality-aware loader hot path.
 *
 * This is the drop-in boundary.  The reference (/root/reference/proj) exposes
 * the path as a C++ static library (namespace locload); every entry point
 * below replaces one reference interface (cited as file:line) and is what a
 * binding of that interface calls.  Plain pointers and sizes only; all
 * "host_*" pointers are host memory (pageable or pinned), device memory is
 * owned by the library.  Every function returns LL_OK or an error code and
 * leaves a message in ll_last_error() (per thread).  There is no CPU fallback:
 * without a CUDA device every compute entry point fails with LL_ERR_CUDA.
 *
 * Error mapping (reference exception -> status):
 *   std::invalid_argument -> LL_ERR_INVALID   (message text identical where the
 *                                               reference defines one)
 *   std::runtime_error    -> LL_ERR_RUNTIME
 */
#ifndef LOCLOAD_B200_H
#define LOCLOAD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    LL_OK = 0,
    LL_ERR_INVALID = 1,   /* std::invalid_argument in the reference           */
    LL_ERR_RUNTIME = 2,   /* std::runtime_error in the reference              */
    LL_ERR_CUDA = 3,      /* CUDA runtime / no device                         */
    LL_ERR_NCCL = 4,      /* NCCL                                             */
    LL_ERR_UNSUPPORTED = 5
};

/* SchemeKind, proj/include/locload/equivalence.hpp:34-38 */
enum { LL_SCHEME_REGULAR = 0, LL_SCHEME_LOCALITY = 1, LL_SCHEME_LOCALITY_BALANCED = 2 };
/* how remote (moved) samples reach their receiver (no reference: SPEC.md:219) */
enum { LL_EXCHANGE_NONE = 0, LL_EXCHANGE_NCCL = 1, LL_EXCHANGE_P2P = 2 };
enum { LL_OUT_F32 = 0, LL_OUT_BF16 = 1 };
enum { LL_AUG_CROP = 0, LL_AUG_RESIZE = 1 };
enum { LL_GEOM_FIXED = 0, LL_GEOM_VARIABLE = 1 };

typedef struct ll_ctx ll_ctx;       /* one CUDA device + stream + workspace   */
typedef struct ll_loader ll_loader; /* one learner's HBM shard + epoch plan   */
typedef struct ll_store ll_store;   /* HBM sample store (SampleCache)         */

int ll_version(void);
const char* ll_last_error(void);
int ll_device_count(int* out);

/* ---- context ----------------------------------------------------------- */
int ll_ctx_create(ll_ctx** out, int device);
int ll_ctx_destroy(ll_ctx* ctx);
int ll_ctx_sync(ll_ctx* ctx);
/* the cudaStream_t all work of this context is issued on */
int ll_ctx_stream(ll_ctx* ctx, uintptr_t* out);
/* number of kernels this context launched so far */
int ll_ctx_launch_count(ll_ctx* ctx, uint64_t* out);
/* per-kernel CUDA-event timing (off by default) */
int ll_ctx_set_timing(ll_ctx* ctx, int enable);
int ll_ctx_kernel_stats(ll_ctx* ctx, const char* kernel, uint64_t* launches, double* total_ms);
int ll_ctx_reset_stats(ll_ctx* ctx);
/* synchronous device -> host copy of library-owned device memory (e.g. a
 * step's device_out) for host consumers and tests */
int ll_ctx_copy_to_host(ll_ctx* ctx, void* host_dst, uintptr_t device_src, uint64_t bytes);

/* ---- core: proj/include/locload/core.hpp -------------------------------- */
/* permute_epoch, core.hpp:25-28 / core.cpp:11-27.  host_order[d]. */
int ll_permute_epoch(ll_ctx* ctx, uint64_t seed, uint64_t epoch, uint64_t d,
                     uint64_t* host_order);
/* permutation_prefix, core.hpp:30-33 / core.cpp:29-55.  host_prefix[k]. */
int ll_permutation_prefix(ll_ctx* ctx, uint64_t seed, uint64_t epoch, uint64_t d, uint64_t k,
                          uint64_t* host_prefix);
/* test hook: the same permutation with the listed 0-based draw indices forced
 * to fail the Lemire test (rng.hpp:41-50), exercising the retry path. */
int ll_permute_epoch_forced(ll_ctx* ctx, uint64_t seed, uint64_t epoch, uint64_t d,
                            const uint64_t* host_forced, uint64_t n_forced,
                            uint64_t* host_order);
/* rounds of the last permutation (deterministic-reservation commit rounds) */
int ll_last_permute_rounds(ll_ctx* ctx, uint32_t* out);
/* phase profile of the last permutation (globaltimer): {rounds, grid-wide
 * rounds, ns draws+repair, ns grid-wide rounds, ns single-CTA rounds, ns total} */
int ll_last_permute_profile(ll_ctx* ctx, uint64_t* out6);

/* ---- sampling + balance: sampling.hpp:42-67, balance.hpp:20-50,
 *      equivalence.cpp:66-91 ------------------------------------------------ */
typedef struct ll_move {
    uint32_t sender;
    uint32_t receiver;
    uint32_t count;    /* samples moved (Move::count, balance.hpp:24-28)        */
    uint32_t src_off;  /* first moved index in the sender's pre-balance list     */
    uint32_t dst_off;  /* first index of the run in the receiver's final list    */
    uint32_t nvlink;   /* moved samples that are cached (cross NVLink)           */
    uint32_t reserved[2];
} ll_move;

/* Assignment of one global batch (host ids) to p learners.
 *  scheme REGULAR            -> reg_slice for every learner (sampling.cpp:27-42)
 *  scheme LOCALITY           -> loc_distribution (sampling.cpp:44-63) with the
 *                               k-th uncached sample dealt to learner k mod p
 *                               (counts: sampling.cpp:65-72)
 *  scheme LOCALITY_BALANCED  -> + targets/balance/tail moves (balance.cpp:14-84,
 *                               equivalence.cpp:77-88)
 * Outputs (host): final_ids[B], final_off[p+1], kept[p], counts[p],
 * moves[p] (n_moves <= p-1), optional stats4 = {moved, moved over NVLink,
 * uncached, remote under the regular scheme (UINT64_MAX when p does not
 * divide B)}. */
int ll_assign(ll_ctx* ctx, const uint64_t* host_batch, uint64_t B, uint64_t d, uint32_t p,
              double alpha, int scheme, uint64_t* final_ids, uint64_t* final_off,
              uint64_t* kept, uint64_t* counts, ll_move* moves, uint32_t* n_moves,
              uint64_t* stats4);

/* A whole epoch's plan on the device, no shard needed: permute_epoch
 * (core.cpp:11-27) + batches (core.cpp:57-73, remainder dropped) + the
 * ll_assign composition for every one of steps = d / B batches -- the
 * sampler half of Loader::run_epoch (pipeline.cpp:251-252) composed with
 * equivalence.cpp:66-91.  Outputs (host, each may be NULL):
 * final_ids[steps*B], final_off[steps*(p+1)], kept[steps*p], counts[steps*p],
 * moves[steps*p] (step s's n_moves[s] moves at s*p), stats4 = epoch totals
 * {moved, moved over NVLink, uncached, regular-scheme remote (UINT64_MAX when
 * p does not divide B)}. */
int ll_plan_epoch(ll_ctx* ctx, uint64_t seed, uint64_t epoch, uint64_t d, uint32_t p,
                  uint64_t B, double alpha, int scheme, uint64_t* steps_out,
                  uint64_t* final_ids, uint64_t* final_off, uint64_t* kept, uint64_t* counts,
                  ll_move* moves, uint32_t* n_moves, uint64_t* stats4);

/* balance() on n independent instances (balance.cpp:58-84): counts/targets are
 * [n][p] row-major; moves [n][p]; n_moves[n].  Rejects mismatched sums with
 * balance.cpp:38-39's message. */
int ll_balance_batch(ll_ctx* ctx, const int64_t* counts, const int64_t* targets, uint32_t p,
                     uint64_t n, ll_move* moves, uint32_t* n_moves);

/* Host-side exchange plan of one learner for one step (no device work): for
 * every move of the schedule that involves learner `me`, one transfer.
 * Sends pack the receiver's list run [list_first, list_first+count) of the
 * step's final ids (all learners, offsets final_off[p+1]) contiguously at
 * buf_first (in samples) of the send buffer; receives land at buf_first of the
 * receive buffer, which is exactly the learner's final-list entries
 * [kept, n_local) in order.  Returns the number of transfers in *n_xfers. */
typedef struct ll_xfer {
    uint32_t peer;
    uint32_t is_send;
    uint64_t count;       /* samples (all cross NVLink when alpha = 1)          */
    uint64_t buf_first;   /* first sample slot in the send / receive buffer      */
    uint64_t list_first;  /* first index into the step's final ids (all learners) */
} ll_xfer;
int ll_exchange_plan(const ll_move* moves, uint32_t n_moves, const uint64_t* final_off,
                     uint32_t p, uint32_t me, ll_xfer* out, uint32_t* n_xfers);

/* ---- dataset: pipeline.cpp:208-234 (generate_dataset byte formula) ------- */
int ll_generate_samples(ll_ctx* ctx, uint64_t data_seed, const uint64_t* host_ids, uint64_t n,
                        uint64_t sample_bytes, uint8_t* host_out);

/* ---- augment (replaces PreprocessPacer, pipeline.cpp:87-108) ------------- */
typedef struct ll_augment_spec {
    int32_t mode;        /* LL_AUG_CROP | LL_AUG_RESIZE                        */
    int32_t out_dtype;   /* LL_OUT_F32 | LL_OUT_BF16                           */
    uint32_t out_h, out_w;
    double mean[3];
    double std[3];
} ll_augment_spec;

/* n HWC u8 samples (each height*width*3 bytes, concatenated) with ids (they
 * key the per-sample crop/flip stream derive_seed(seed, epoch, id)) ->
 * host_out[n][3][out_h][out_w]. */
int ll_augment(ll_ctx* ctx, const ll_augment_spec* spec, uint64_t seed, uint64_t epoch,
               const uint8_t* host_src, const uint64_t* host_ids, uint64_t n, uint32_t height,
               uint32_t width, void* host_out);
/* The same on device buffers (asynchronous on the context stream): n samples
 * at device_src + k*height*width*3 -- which may be a peer GPU's memory after
 * ll_ctx_enable_peer -- with ids device_ids[k], into device_out. */
int ll_augment_device(ll_ctx* ctx, const ll_augment_spec* spec, uint64_t seed, uint64_t epoch,
                      uintptr_t device_src, uintptr_t device_ids, uint64_t n, uint32_t height,
                      uint32_t width, uintptr_t device_out);
/* let kernels of this context read `peer_device`'s memory (NVLink P2P) */
int ll_ctx_enable_peer(ll_ctx* ctx, int peer_device);
/* crop/flip parameters the augment uses (y0, x0, ch, cw, flip per sample) */
int ll_augment_params(ll_ctx* ctx, const ll_augment_spec* spec, uint64_t seed, uint64_t epoch,
                      const uint64_t* host_ids, uint64_t n, uint32_t height, uint32_t width,
                      uint32_t* host_params5);

/* ---- equivalence: proj/include/locload/equivalence.hpp ----------------- */
/* Consumer side: synchronous SGD of p learners on the least-squares toy
 * objective (per-sample loss 0.5 (w.x_i - y_i)^2), run_training
 * (equivalence.cpp:95-174) on the device.  host_xs[n*dims] / host_ys[n] are
 * ToyObjective::synthesize's data (equivalence.cpp:12-37).  Every step the
 * epoch's batch goes through the scheme's assignment; aggregation CANONICAL
 * sums per-sample gradients in ascending sample id, LEARNER_ORDER sums per
 * learner list then across learners.  Outputs host_final_w[dims] and, if not
 * NULL, host_step_grads[steps*dims] (each normalised by B).  Bit-identical to
 * the reference.  Errors: p = 0, B outside [1, n], p not dividing B under the
 * regular scheme (the reference's messages); p > 64; n >= 2^32. */
enum { LL_AGG_CANONICAL = 0, LL_AGG_LEARNER_ORDER = 1 };
int ll_train_run(ll_ctx* ctx, const double* host_xs, const double* host_ys, uint64_t n,
                 uint32_t dims, int scheme, uint32_t p, uint64_t batch_size, uint64_t steps,
                 uint64_t seed, double learning_rate, int aggregation, double* host_final_w,
                 double* host_step_grads);
/* ToyObjective::synthesize (equivalence.cpp:12-37), host-only: host_xs[n*dims],
 * host_ys[n] from the seeded streams, bit-identical to the reference (same
 * Box-Muller draws through the host libm). */
int ll_toy_synthesize(uint64_t n, uint32_t dims, uint64_t seed, double* host_xs, double* host_ys);
/* full_batch_gradient (equivalence.cpp:190-205): the batch's mean gradient at
 * host_w, summed in batch-sequence order.  host_grad[dims]. */
int ll_full_batch_gradient(ll_ctx* ctx, const double* host_xs, const double* host_ys, uint64_t n,
                           uint32_t dims, const double* host_w, const uint64_t* host_batch,
                           uint64_t batch_size, double* host_grad);

/* ---- sample store: SampleCache, pipeline.hpp:68-94 ---------------------- */
/* The populate-on-first-touch cache of the reference's Loader, held in HBM:
 * at most capacity_samples samples of one fixed size, no replacement
 * (SampleCache::insert ignores inserts at capacity, pipeline.hpp:78-83); slabs
 * are allocated as it fills, and an exhausted device also ends inserts.
 * Lookups may run concurrently with each other and with inserts (the
 * reference's shared_mutex, pipeline.hpp:90); every call is thread-safe. */
int ll_store_create(ll_store** out, int device, uint64_t capacity_samples);
int ll_store_destroy(ll_store* st);
int ll_store_size(ll_store* st, uint64_t* out);              /* SampleCache::size  */
/* the stored sample size (fixed by the first insert; 0 while empty) */
int ll_store_sample_bytes(ll_store* st, uint64_t* out);
/* found[i] = 1 when ids[i] is held (SampleCache::find, pipeline.hpp:72-76) */
int ll_store_lookup(ll_store* st, const uint64_t* ids, uint64_t n, uint8_t* found);
/* SampleCache::insert for n samples of sample_bytes each at host_ptrs[i]
 * (copied on ctx's stream; complete and visible to every thread on return);
 * held ids and ids past capacity are skipped; inserted[i] (may be NULL). */
int ll_store_insert(ll_store* st, ll_ctx* ctx, const uint64_t* ids, uint64_t n,
                    uint64_t sample_bytes, const uint8_t* const* host_ptrs, uint8_t* inserted);
/* host copies of n held samples, contiguous in host_dst[n * sample_bytes]
 * (one device gather + one D2H); LL_ERR_INVALID if an id is not held */
int ll_store_gather(ll_store* st, ll_ctx* ctx, const uint64_t* ids, uint64_t n,
                    uint8_t* host_dst);

/* ---- distributed consumer: run_training's aggregation (equivalence.cpp:
 *      121-166) with one learner per process, on caller-owned device buffers
 *      (e.g. torch tensors), asynchronous on the context's stream ---------- */
/* grads[i][*] = the toy objective's gradient of sample ids[i] (int64) at w
 * (equivalence.cpp:52-64); xs[n*dims], ys[n] as ll_toy_synthesize made them */
int ll_toy_grads_device(ll_ctx* ctx, uintptr_t xs, uintptr_t ys, uint32_t dims, uintptr_t w,
                        uintptr_t ids, uint64_t n_ids, uintptr_t grads);
/* out[k] = sum over i of grads[order[i]][k] (order = 0: i), sequentially from
 * 0.0 -- the deterministic half of the gradient all-reduce: rows gathered
 * from every rank and summed in ascending sample id (canonical) or per-learner
 * partials summed in learner order (learner_order) equal the reference's sums
 * bit for bit (equivalence.cpp:132-148) */
int ll_ordered_sum_device(ll_ctx* ctx, uintptr_t grads, uint64_t n, uint32_t dims,
                          uintptr_t order, uintptr_t out);
/* g = gsum * scale; step_grad = g (if non-zero); w -= lr * g (:157-166) */
int ll_sgd_apply_device(ll_ctx* ctx, uintptr_t gsum, uint32_t dims, double scale, double lr,
                        uintptr_t w, uintptr_t step_grad);

/* ---- loader: pipeline.hpp:46-128 ---------------------------------------- */
typedef struct ll_loader_config {
    uint64_t d;               /* DatasetSpec::n                                 */
    uint32_t height, width;   /* HWC u8 sample geometry; sample_bytes = h*w*3    */
    uint32_t learners;        /* p                                             */
    uint32_t rank;            /* this learner                                  */
    uint64_t batch_size;      /* GLOBAL batch, LoaderConfig::batch_size          */
    double alpha;             /* cached fraction (CacheDirectory); alpha < 1
                                 keeps ids [alpha*d, d) in a pinned host
                                 storage tier (fixed geometry; any exchange)   */
    uint64_t seed;            /* run_epoch seed: shuffle + augment streams       */
    uint64_t data_seed;       /* generate_dataset seed                           */
    int32_t scheme;           /* LL_SCHEME_*                                     */
    int32_t exchange;         /* LL_EXCHANGE_*: P2P (peer HBM read by the
                                 augment) or NCCL (grouped send/recv of crop /
                                 resize windows; the regular scheme over NCCL
                                 needs crop mode)                              */
    uint32_t prefetch_depth;  /* LoaderConfig::prefetch_depth: output ring depth */
    uint32_t geometry;        /* LL_GEOM_FIXED: every sample height x width;
                                 LL_GEOM_VARIABLE: sample id is H x W with
                                 H, W = 128 + bounded(385) from
                                 SplitMix64(derive_seed(data_seed, id, 1))
                                 (cfg5; needs augment.mode = LL_AUG_RESIZE) */
    ll_augment_spec augment;
} ll_loader_config;

typedef struct ll_step_info {
    uint64_t epoch, step;
    uint64_t n_local;         /* samples in this learner's final list           */
    uint64_t kept;            /* of which assembled from its own shard          */
    uint64_t received;        /* of which received from other learners          */
    uint64_t moved_total;     /* samples moved box-wide this step               */
    uint64_t nvlink_bytes;    /* bytes this learner received over NVLink: the
                                 NCCL message slots, or (P2P) the samples      */
    uint64_t uncached;        /* samples of the global batch not cached         */
    uint64_t reg_remote;      /* remote samples the regular scheme would need   */
    uintptr_t device_out;     /* this step's [n_local][3][out_h][out_w] tensor  */
    uintptr_t device_ids;     /* [n_local] u32 sample ids, final list order     */
    uint64_t h2d_bytes;       /* host->device bytes this call copied (host step) */
    uint64_t d2h_bytes;       /* device->host bytes this call copied (host step) */
} ll_step_info;

int ll_loader_create(ll_loader** out, ll_ctx* ctx, const ll_loader_config* cfg);
int ll_loader_destroy(ll_loader* ld);
/* NCCL bootstrap for LL_EXCHANGE_NCCL: rank 0 makes the id, every rank inits */
int ll_nccl_unique_id(uint8_t* out128);
int ll_loader_comm_init(ll_loader* ld, const uint8_t* id128);
/* P2P bootstrap for LL_EXCHANGE_P2P: export this rank's shard handle (64 B),
 * all-gather them, then open the peers' shards ([p][64] bytes). */
int ll_loader_ipc_handle(ll_loader* ld, uint8_t* out64);
int ll_loader_open_peers(ll_loader* ld, const uint8_t* handles);
/* Same-process learners (tests, single-process multi-learner runs): give each
 * loader the others' shard pointers for LL_EXCHANGE_P2P.  All loaders must sit
 * on one device or on devices with peer access. */
int ll_loader_link_peers(ll_loader* const* loaders, uint32_t n);
/* Fill this learner's HBM shard (CacheDirectory block, sampling.cpp:19-25)
 * with the generate_dataset bytes -- the populated cache of epoch 0. */
int ll_loader_populate(ll_loader* ld);
/* Fill the shard (and, for alpha < 1, the host storage tier) from the
 * reference's on-disk dataset: files <root>/%08llu.bin written by
 * generate_dataset (pipeline.cpp:202-234), read by `threads` host threads
 * (0 = all cores) through pinned staging.  Missing / short files fail with
 * LL_ERR_RUNTIME and read_sample's messages ("sample N: cannot open PATH",
 * "sample N: truncated file PATH (read X of Y bytes)", pipeline.cpp:110-126). */
int ll_loader_populate_from_files(ll_loader* ld, const char* root, uint32_t threads);
/* Fill the shard from host memory instead: owned_count(rank) samples. */
int ll_loader_populate_from_host(ll_loader* ld, const uint8_t* host_samples);
int ll_loader_shard_range(ll_loader* ld, uint64_t* first_id, uint64_t* count);
int ll_loader_steps_per_epoch(ll_loader* ld, uint64_t* out);
/* Epoch plan on the device: permutation + assignment of every step. */
int ll_loader_plan_epoch(ll_loader* ld, uint64_t epoch);
/* One step, asynchronous on the context stream: exchange + augment of this
 * learner's share of global batch `step` (plans the epoch if needed). */
int ll_loader_step(ll_loader* ld, uint64_t epoch, uint64_t step, ll_step_info* info);
/* Reference-facing host call (Loader::run_epoch per batch, pipeline.cpp:
 * 247-336): the global batch comes in from host memory (GlobalBatch::samples,
 * core.hpp:20-23), is assigned/exchanged/augmented on the device, and the
 * learner's final id list is returned to host memory; synchronous. */
int ll_loader_step_host(ll_loader* ld, uint64_t epoch, uint64_t step,
                        const uint64_t* host_batch, uint64_t* host_local_ids,
                        ll_step_info* info);
/* The same, pipelined like the reference's prefetching Loader (pipeline.hpp:
 * 46-53 prefetch_depth, pipeline.cpp:283-318 in-order delivery): submit
 * returns once the step is queued (the batch ids are copied out of
 * host_batch), at most prefetch_depth steps may be outstanding, and wait
 * delivers the oldest one (its local ids and info), in submission order.
 * The step's device_out stays valid until prefetch_depth later steps. */
int ll_loader_submit_host(ll_loader* ld, uint64_t epoch, uint64_t step,
                          const uint64_t* host_batch);
int ll_loader_wait_host(ll_loader* ld, uint64_t* host_local_ids, ll_step_info* info);
/* host copies of the current epoch plan for step `step` (tests) */
int ll_loader_plan_step(ll_loader* ld, uint64_t step, uint64_t* final_ids, uint64_t* final_off,
                        uint64_t* kept, uint64_t* counts, ll_move* moves, uint32_t* n_moves);
/* DLPack view (a DLManagedTensor*, DLPack v0.8 ABI) of a step's augmented
 * batch: kDLCUDA device, float32 or bfloat16, shape [n_local][3][out_h][out_w],
 * compact -- the zero-copy hand-off to any DLPack consumer (torch, JAX, CuPy,
 * a C++ trainer).  The memory stays the loader's (valid until prefetch_depth
 * later steps); the tensor's deleter frees only the view.  Order the
 * consumer's stream after ll_ctx_stream before reading. */
int ll_loader_batch_dlpack(ll_loader* ld, const ll_step_info* info, void** out_managed);
/* per-epoch totals of the current plan: moved, nvlink-moved, uncached, reg_remote */
int ll_loader_epoch_totals(ll_loader* ld, uint64_t* out4);
/* NCCL exchange accounting since the last reset: out8 = {steps, bytes sent,
 * bytes received (message bytes on the wire), steps timed, bytes received in
 * the timed steps, ms in the pack kernel, ms from the grouped send/recv's
 * issue to its completion, 0}; the times cover steps issued while the
 * context's timing (ll_ctx_set_timing) was on, measured by CUDA events on
 * the exchange's stream.  NVLink GB/s = timed bytes received / ms on the wire. */
int ll_loader_exchange_stats(ll_loader* ld, double* out8, int reset);

#ifdef __cplusplus
}
#endif
#endif
