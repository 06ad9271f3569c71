/*
 * locload_oracle.h -- CPU restatement of the locality-aware loader hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_1910_01196_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product never links or calls it (no CPU fallback).
 *
 * Parity status
 *   - rng, permutation, directory, distribution, balance, tail moves and the
 *     synthetic dataset bytes restate /root/reference/proj (file:line cited
 *     per function) and are PINNED: tests/test_oracle.py checks them against
 *     the reference's own known-answer tests and against golden vectors that
 *     tests/golden/make_golden.py produced by running the compiled reference
 *     (oracle/_ref, built from the reference sources by oracle/Makefile).
 *   - The uncached-list ORDER for alpha < 1 (the reference materialises only
 *     counts, sampling.cpp:65-72) and the augment stage (crop / flip /
 *     bilinear / normalise; the reference has none) have no
 *     reference code: here this restatement IS the specification.  Parity
 *     for those parts is "unpinned" in the sense of DESIGN.md section 3.
 */
#ifndef LOCLOAD_ORACLE_H
#define LOCLOAD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng (proj/include/locload/rng.hpp) ------------------------------- */
uint64_t lo_mix64(uint64_t z);                                   /* rng.hpp:9-13  */
uint64_t lo_derive_seed(uint64_t seed, uint64_t a);              /* rng.hpp:19-22 */
uint64_t lo_derive_seed3(uint64_t seed, uint64_t a, uint64_t b); /* rng.hpp:24-26 */

typedef struct {
    uint64_t state;
    uint64_t draws;                 /* 0-based index of the next draw        */
    const uint64_t* forced;         /* sorted draw indices treated as        */
    uint64_t n_forced;              /* rejected by bounded() (test hook)     */
} lo_rng;

void lo_rng_init(lo_rng* r, uint64_t seed);
uint64_t lo_rng_next(lo_rng* r);                                 /* rng.hpp:35-38 */
uint64_t lo_rng_bounded(lo_rng* r, uint64_t n);                  /* rng.hpp:41-50 */

/* ---- core (proj/src/core.cpp) ------------------------------------------ */
/* Returns 0, or -1 for d == 0 (std::invalid_argument in core.cpp:12-14). */
int lo_permute_epoch(uint64_t seed, uint64_t epoch, uint64_t d, uint64_t* order);
/* Same with a list of draw indices forced to be rejected (exercises the
 * Lemire retry path, which real inputs essentially never hit). */
int lo_permute_epoch_forced(uint64_t seed, uint64_t epoch, uint64_t d, uint64_t* order,
                            const uint64_t* forced, uint64_t n_forced);

/* ---- sampling (proj/src/sampling.cpp) ---------------------------------- */
uint64_t lo_cached_count(uint64_t d, double alpha);              /* sampling.cpp:15-16 */
/* owner of s, or p when s is not cached (sampling.hpp:22-25) */
uint32_t lo_owner(uint64_t s, uint32_t p, uint64_t cached);
uint64_t lo_owned_begin(uint32_t j, uint32_t p, uint64_t cached);/* sampling.cpp:21-23 */

/* ---- balance (proj/src/balance.cpp) ------------------------------------ */
typedef struct {
    uint32_t sender;
    uint32_t receiver;
    uint64_t count;
    uint64_t src_off;   /* first index of the moved tail in the sender's list   */
    uint64_t dst_off;   /* first index of the moved run in the receiver's list  */
} lo_move;

void lo_targets(uint64_t b, uint32_t p, int64_t* out);           /* balance.cpp:14-28 */
/* Algorithm 1 (balance.cpp:58-84).  Returns the number of moves, or -1 when
 * counts and targets disagree in sum (balance.cpp:32-41). */
int lo_balance(const int64_t* counts, const int64_t* targets, uint32_t p, lo_move* moves);

/* ---- one step of assignment (equivalence.cpp:66-91 composed with
 *      sampling.cpp:44-72 and balance.cpp:14-84) ------------------------- */
enum { LO_MODE_REGULAR = 0, LO_MODE_LOCALITY = 1, LO_MODE_LOCALITY_BALANCED = 2 };

/* final_ids[B]   : learner j's final list is final_ids[final_off[j] .. final_off[j+1])
 * final_off[p+1] : list offsets
 * kept[p]        : leading entries of learner j's list that it assembled itself
 * counts[p]      : pre-balance list sizes (cached-owned + round-robin uncached)
 * moves[p]       : schedule (at most p-1 moves), *n_moves its length
 * Returns 0, or -1 on invalid arguments (regular mode needs p | B). */
int lo_assign_step(const uint64_t* batch, uint64_t B, uint32_t p, uint64_t cached, int mode,
                   uint64_t* final_ids, uint64_t* final_off, uint64_t* kept, uint64_t* counts,
                   lo_move* moves, uint32_t* n_moves);

/* ---- dataset (proj/src/pipeline.cpp:208-234) --------------------------- */
void lo_gen_sample(uint64_t data_seed, uint64_t id, uint64_t nbytes, uint8_t* out);
/* cfg5 variable-size sources: H, W = 128 + bounded(385) each from
 * SplitMix64(derive_seed(data_seed, id, 1)) (new semantics). */
void lo_sample_hw(uint64_t data_seed, uint64_t id, uint32_t* h, uint32_t* w);

/* ---- augment (new semantics) ------------------ */
typedef struct {
    uint32_t y0, x0;    /* crop origin in the source                      */
    uint32_t ch, cw;    /* crop extent in the source                      */
    uint32_t flip;      /* horizontal flip                                */
} lo_aug_params;

/* CROP mode: region = out_h x out_w at a random origin; RESIZE mode: region =
 * the largest centred-size square min(H,W) at a random origin, bilinearly
 * resized to out_h x out_w.  Stream SplitMix64(derive_seed(seed, epoch, id)):
 * draw y0 = bounded(H-ch+1), x0 = bounded(W-cw+1), flip = next() >> 63. */
enum { LO_AUG_CROP = 0, LO_AUG_RESIZE = 1 };
void lo_aug_params_for(uint64_t seed, uint64_t epoch, uint64_t id, uint32_t H, uint32_t W,
                       uint32_t out_h, uint32_t out_w, int mode, lo_aug_params* prm);

/* Normalisation constants: out = (float(v) - mean255[c]) * inv_std255[c] with
 * mean255 = (float)(mean*255), inv_std255 = (float)(1/(std*255)), both formed
 * in double and rounded once to float. */
void lo_norm_constants(const double mean[3], const double std_[3], float mean255[3],
                       float inv_std255[3]);

uint16_t lo_bf16_rne(float f);

/* RESIZE source tap along one axis: output index o of n_out over a crop of
 * `extent` source pixels.  f = floor((2o+1)*extent*64 / n_out) - 64 (the
 * half-pixel-centre position in 1/128 px), clamped at 0; lo = f >> 7,
 * w = f & 127; at the far edge (lo >= extent-1) lo = extent-1 and w = 0.
 * The second tap is lo+1 (weight w), used only when w > 0. */
void lo_resize_tap(uint32_t o, uint32_t n_out, uint32_t extent, uint32_t* lo, uint32_t* w);

/* src is HWC u8 (H x W x 3).  out is CHW (3 x out_h x out_w), fp32 when
 * out_bf16 == 0, else bf16 bits (uint16). */
void lo_augment_one(const uint8_t* src, uint32_t H, uint32_t W, const lo_aug_params* prm,
                    uint32_t out_h, uint32_t out_w, int mode, const float mean255[3],
                    const float inv_std255[3], int out_bf16, void* out);

/* Multi-threaded batch driver for the CPU baseline: n samples with the given
 * source pointers / sizes / params into out (n x 3 x out_h x out_w). */
void lo_augment_batch_mt(const uint8_t* const* srcs, const uint32_t* Hs, const uint32_t* Ws,
                         const lo_aug_params* prms, uint64_t n, uint32_t out_h, uint32_t out_w,
                         int mode, const float mean255[3], const float inv_std255[3],
                         int out_bf16, void* out, int threads);

/* CPU-baseline driver (bench.py's reference arm): one step's augment of n
 * samples on `threads` threads.  Sample ids[i] reads pool[ids[i] % pool_n]
 * (a warm host cache of pool_n samples of H*W*3 bytes); parameters come from
 * lo_aug_params_for (CROP mode); the normalisation is a per-channel 256-entry
 * table of exactly the values lo_augment_one computes, so the output is
 * bit-identical to lo_augment_one. */
void lo_cpu_crop_step(const uint8_t* pool, uint64_t pool_n, const uint64_t* ids, uint64_t n,
                      uint32_t H, uint32_t W, uint64_t seed, uint64_t epoch, uint32_t out_h,
                      uint32_t out_w, const float mean255[3], const float inv_std255[3],
                      int out_bf16, void* out, int threads);

/* CPU-baseline driver for the variable-size workload (cfg5): sample ids[i]
 * reads pool slot ids[i] % pool_n (srcs[slot], Hs[slot] x Ws[slot]); RESIZE
 * parameters and lo_augment_one per sample, on `threads` threads. */
void lo_cpu_resize_step(const uint8_t* const* srcs, const uint32_t* Hs, const uint32_t* Ws,
                        uint64_t pool_n, const uint64_t* ids, uint64_t n, uint64_t seed,
                        uint64_t epoch, uint32_t out_h, uint32_t out_w, const float mean255[3],
                        const float inv_std255[3], int out_bf16, void* out, int threads);

#ifdef __cplusplus
}
#endif
#endif
