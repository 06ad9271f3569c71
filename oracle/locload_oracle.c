/*
 * locload_oracle.c -- CPU restatement of the loader hot path.
 * TEST INFRASTRUCTURE ONLY; see locload_oracle.h for the contract.
 * Compiled by oracle/Makefile with -ffp-contract=off so every float
 * operation is one IEEE-rounded op, matching the __f*_rn sequence the CUDA
 * kernels use.
 */
#include "locload_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define GAMMA 0x9e3779b97f4a7c15ULL

/* rng.hpp:9-13 */
uint64_t lo_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.hpp:19-22 */
uint64_t lo_derive_seed(uint64_t seed, uint64_t a) {
    uint64_t s = lo_mix64(seed + GAMMA);
    return lo_mix64(s ^ (a + 0xbf58476d1ce4e5b9ULL));
}

/* rng.hpp:24-26 */
uint64_t lo_derive_seed3(uint64_t seed, uint64_t a, uint64_t b) {
    return lo_mix64(lo_derive_seed(seed, a) ^ (b + 0x94d049bb133111ebULL));
}

void lo_rng_init(lo_rng* r, uint64_t seed) {
    r->state = seed;
    r->draws = 0;
    r->forced = NULL;
    r->n_forced = 0;
}

/* rng.hpp:35-38: the k-th (0-based) draw is mix64(seed + (k+1)*gamma). */
uint64_t lo_rng_next(lo_rng* r) {
    r->state += GAMMA;
    r->draws += 1;
    return lo_mix64(r->state);
}

static int is_forced(const lo_rng* r, uint64_t k) {
    uint64_t lo = 0, hi = r->n_forced;
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (r->forced[mid] < k) lo = mid + 1; else hi = mid;
    }
    return lo < r->n_forced && r->forced[lo] == k;
}

/* rng.hpp:41-50 (Lemire multiply-shift with rejection) */
uint64_t lo_rng_bounded(lo_rng* r, uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
        const uint64_t k = r->draws;
        const uint64_t x = lo_rng_next(r);
        const unsigned __int128 m = (unsigned __int128)x * n;
        if ((uint64_t)m >= threshold && !(r->forced && is_forced(r, k))) {
            return (uint64_t)(m >> 64);
        }
    }
}

/* core.cpp:11-27 (forward Fisher-Yates on iota(d)) */
int lo_permute_epoch_forced(uint64_t seed, uint64_t epoch, uint64_t d, uint64_t* order,
                            const uint64_t* forced, uint64_t n_forced) {
    if (d == 0) return -1;
    for (uint64_t i = 0; i < d; ++i) order[i] = i;
    lo_rng r;
    lo_rng_init(&r, lo_derive_seed(seed, epoch));
    r.forced = forced;
    r.n_forced = n_forced;
    for (uint64_t i = 0; i < d; ++i) {
        const uint64_t j = i + lo_rng_bounded(&r, d - i);
        const uint64_t t = order[i];
        order[i] = order[j];
        order[j] = t;
    }
    return 0;
}

int lo_permute_epoch(uint64_t seed, uint64_t epoch, uint64_t d, uint64_t* order) {
    return lo_permute_epoch_forced(seed, epoch, d, order, NULL, 0);
}

/* sampling.cpp:15-16 */
uint64_t lo_cached_count(uint64_t d, double alpha) {
    uint64_t c = (uint64_t)(alpha * (double)d);
    return c > d ? d : c;
}

/* sampling.hpp:22-25 */
uint32_t lo_owner(uint64_t s, uint32_t p, uint64_t cached) {
    if (s >= cached) return p;
    return (uint32_t)(s * p / cached);
}

/* sampling.cpp:21-23: first index owned by learner j */
uint64_t lo_owned_begin(uint32_t j, uint32_t p, uint64_t cached) {
    return ((uint64_t)j * cached + p - 1) / p;
}

/* balance.cpp:14-28 */
void lo_targets(uint64_t b, uint32_t p, int64_t* out) {
    const int64_t base = (int64_t)(b / p);
    const int64_t rem = (int64_t)(b % p);
    for (uint32_t j = 0; j < p; ++j) out[j] = base + ((int64_t)j < rem ? 1 : 0);
}

/* balance.cpp:58-84.  The reference keeps two max-heaps ordered by
 * (imbalance, lowest id) (HeapLess, balance.cpp:49-54).  Ids are unique, so
 * the heap top is the unique maximum of that strict order and an argmax scan
 * over the live entries selects exactly the same element every round. */
int lo_balance(const int64_t* counts, const int64_t* targets, uint32_t p, lo_move* moves) {
    int64_t cs = 0, ts = 0;
    for (uint32_t j = 0; j < p; ++j) { cs += counts[j]; ts += targets[j]; }
    if (cs != ts) return -1;
    int64_t* imb = (int64_t*)malloc(sizeof(int64_t) * (p ? p : 1));
    for (uint32_t j = 0; j < p; ++j) imb[j] = counts[j] - targets[j];
    int n = 0;
    for (;;) {
        int s = -1, r = -1;
        for (uint32_t j = 0; j < p; ++j) {
            if (imb[j] > 0 && (s < 0 || imb[j] > imb[s])) s = (int)j;
            if (imb[j] < 0 && (r < 0 || -imb[j] > -imb[r])) r = (int)j;
        }
        if (s < 0) break;
        const int64_t m = imb[s] < -imb[r] ? imb[s] : -imb[r];
        moves[n].sender = (uint32_t)s;
        moves[n].receiver = (uint32_t)r;
        moves[n].count = (uint64_t)m;
        moves[n].src_off = 0;
        moves[n].dst_off = 0;
        ++n;
        imb[s] -= m;
        imb[r] += m;
    }
    free(imb);
    return n;
}

/* One step of assignment.
 *   regular            : reg_slice, sampling.cpp:27-42
 *   locality(_balanced): loc_distribution (sampling.cpp:44-63) -- each cached
 *     sample to its owner in batch order -- then the k-th uncached sample (in
 *     batch order) dealt to learner k mod p (sampling.cpp:65-72 deals the
 *     COUNTS that way; the reference never materialises those lists, so their
 *     placement -- appended after the learner's cached samples, in batch
 *     order -- is this build's definition).  Balanced mode then runs targets
 *     + Algorithm 1 and applies every move as "receiver appends the sender's
 *     last `count` samples" (equivalence.cpp:77-88). */
int lo_assign_step(const uint64_t* batch, uint64_t B, uint32_t p, uint64_t cached, int mode,
                   uint64_t* final_ids, uint64_t* final_off, uint64_t* kept, uint64_t* counts,
                   lo_move* moves, uint32_t* n_moves) {
    if (p == 0) return -1;
    *n_moves = 0;
    if (mode == LO_MODE_REGULAR) {
        if (B % p != 0) return -1;
        const uint64_t slice = B / p;
        for (uint32_t j = 0; j <= p; ++j) final_off[j] = slice * j;
        for (uint32_t j = 0; j < p; ++j) { kept[j] = slice; counts[j] = slice; }
        memcpy(final_ids, batch, sizeof(uint64_t) * B);
        return 0;
    }
    /* pre-balance lists */
    uint64_t* owned = (uint64_t*)calloc(p, sizeof(uint64_t));
    uint64_t n_unc = 0;
    for (uint64_t e = 0; e < B; ++e) {
        const uint32_t o = lo_owner(batch[e], p, cached);
        if (o < p) owned[o]++; else n_unc++;
    }
    for (uint32_t j = 0; j < p; ++j) counts[j] = owned[j] + n_unc / p + (j < n_unc % p ? 1 : 0);
    uint64_t* pre_off = (uint64_t*)calloc(p + 1, sizeof(uint64_t));
    for (uint32_t j = 0; j < p; ++j) pre_off[j + 1] = pre_off[j] + counts[j];
    uint64_t* pre = (uint64_t*)malloc(sizeof(uint64_t) * (B ? B : 1));
    uint64_t* fill = (uint64_t*)calloc(p, sizeof(uint64_t));
    uint64_t k_unc = 0;
    for (uint64_t e = 0; e < B; ++e) {
        const uint32_t o = lo_owner(batch[e], p, cached);
        if (o < p) {
            pre[pre_off[o] + fill[o]++] = batch[e];
        } else {
            const uint32_t j = (uint32_t)(k_unc % p);
            pre[pre_off[j] + owned[j] + k_unc / p] = batch[e];
            k_unc++;
        }
    }
    if (mode == LO_MODE_LOCALITY) {
        memcpy(final_ids, pre, sizeof(uint64_t) * B);
        memcpy(final_off, pre_off, sizeof(uint64_t) * (p + 1));
        for (uint32_t j = 0; j < p; ++j) kept[j] = counts[j];
    } else {
        int64_t* tg = (int64_t*)malloc(sizeof(int64_t) * p);
        int64_t* cn = (int64_t*)malloc(sizeof(int64_t) * p);
        lo_targets(B, p, tg);
        for (uint32_t j = 0; j < p; ++j) cn[j] = (int64_t)counts[j];
        const int n = lo_balance(cn, tg, p, moves);
        uint64_t* taken = (uint64_t*)calloc(p, sizeof(uint64_t));
        uint64_t* recvd = (uint64_t*)calloc(p, sizeof(uint64_t));
        for (int m = 0; m < n; ++m) {
            const uint32_t s = moves[m].sender, r = moves[m].receiver;
            moves[m].src_off = counts[s] - taken[s] - moves[m].count;
            moves[m].dst_off = counts[r] + recvd[r];
            taken[s] += moves[m].count;
            recvd[r] += moves[m].count;
        }
        final_off[0] = 0;
        for (uint32_t j = 0; j < p; ++j) {
            final_off[j + 1] = final_off[j] + (uint64_t)tg[j];
            kept[j] = counts[j] - taken[j];
            memcpy(final_ids + final_off[j], pre + pre_off[j], sizeof(uint64_t) * kept[j]);
        }
        for (int m = 0; m < n; ++m) {
            memcpy(final_ids + final_off[moves[m].receiver] + moves[m].dst_off,
                   pre + pre_off[moves[m].sender] + moves[m].src_off,
                   sizeof(uint64_t) * moves[m].count);
        }
        *n_moves = (uint32_t)n;
        free(tg); free(cn); free(taken); free(recvd);
    }
    free(owned); free(pre_off); free(pre); free(fill);
    return 0;
}

/* pipeline.cpp:221-226: byte i of sample id = byte (i mod 8) of draw i/8 of
 * SplitMix64(derive_seed(seed, id)). */
void lo_gen_sample(uint64_t data_seed, uint64_t id, uint64_t nbytes, uint8_t* out) {
    lo_rng r;
    lo_rng_init(&r, lo_derive_seed(data_seed, id));
    uint64_t word = 0;
    for (uint64_t i = 0; i < nbytes; ++i) {
        if (i % 8 == 0) word = lo_rng_next(&r);
        out[i] = (uint8_t)(word >> ((i % 8) * 8));
    }
}

void lo_sample_hw(uint64_t data_seed, uint64_t id, uint32_t* h, uint32_t* w) {
    lo_rng r;
    lo_rng_init(&r, lo_derive_seed3(data_seed, id, 1));
    *h = 128u + (uint32_t)lo_rng_bounded(&r, 385);
    *w = 128u + (uint32_t)lo_rng_bounded(&r, 385);
}

void lo_aug_params_for(uint64_t seed, uint64_t epoch, uint64_t id, uint32_t H, uint32_t W,
                       uint32_t out_h, uint32_t out_w, int mode, lo_aug_params* prm) {
    uint32_t ch, cw;
    if (mode == LO_AUG_CROP) {
        ch = out_h;
        cw = out_w;
    } else {
        ch = cw = H < W ? H : W;
    }
    lo_rng r;
    lo_rng_init(&r, lo_derive_seed3(seed, epoch, id));
    prm->ch = ch;
    prm->cw = cw;
    prm->y0 = (uint32_t)lo_rng_bounded(&r, (uint64_t)(H - ch) + 1);
    prm->x0 = (uint32_t)lo_rng_bounded(&r, (uint64_t)(W - cw) + 1);
    prm->flip = (uint32_t)(lo_rng_next(&r) >> 63);
}

void lo_norm_constants(const double mean[3], const double std_[3], float mean255[3],
                       float inv_std255[3]) {
    for (int c = 0; c < 3; ++c) {
        mean255[c] = (float)(mean[c] * 255.0);
        inv_std255[c] = (float)(1.0 / (std_[c] * 255.0));
    }
}

uint16_t lo_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) return (uint16_t)((u >> 16) | 0x40);
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}

static inline void store_px(void* out, uint64_t idx, float v, int out_bf16) {
    if (out_bf16) ((uint16_t*)out)[idx] = lo_bf16_rne(v);
    else ((float*)out)[idx] = v;
}

void lo_resize_tap(uint32_t o, uint32_t n_out, uint32_t extent, uint32_t* lo, uint32_t* w) {
    /* f = 128 * ((o + 0.5) * extent / n_out - 0.5), floored, in exact integers */
    const int64_t f = (int64_t)(((uint64_t)(2 * o + 1) * extent * 64) / n_out) - 64;
    uint32_t l = 0, ww = 0;
    if (f > 0) {
        l = (uint32_t)(f >> 7);
        ww = (uint32_t)(f & 127);
    }
    if (l >= extent - 1) {
        l = extent - 1;
        ww = 0;
    }
    *lo = l;
    *w = ww;
}

void lo_augment_one(const uint8_t* src, uint32_t H, uint32_t W, const lo_aug_params* prm,
                    uint32_t out_h, uint32_t out_w, int mode, const float mean255[3],
                    const float inv_std255[3], int out_bf16, void* out) {
    (void)H;
    const uint64_t plane = (uint64_t)out_h * out_w;
    if (mode == LO_AUG_CROP) {
        for (uint32_t oy = 0; oy < out_h; ++oy) {
            const uint8_t* row = src + ((uint64_t)(prm->y0 + oy) * W) * 3;
            for (uint32_t ox = 0; ox < out_w; ++ox) {
                const uint32_t sx = prm->flip ? prm->x0 + out_w - 1 - ox : prm->x0 + ox;
                for (int c = 0; c < 3; ++c) {
                    const float v = (float)row[(uint64_t)sx * 3 + c];
                    const float o = (v - mean255[c]) * inv_std255[c];
                    store_px(out, c * plane + (uint64_t)oy * out_w + ox, o, out_bf16);
                }
            }
        }
        return;
    }
    /* RESIZE: fixed-point bilinear.  Source positions
     * in 1/128 px, half-pixel centres, edge clamp; the four tap weights are
     * products of 7-bit axis weights, so v is an exact integer < 2^22 and
     * out = (v * 2^-14 - mean255) * inv_std255.  Column taps are tabulated
     * once per sample. */
    uint32_t* txl = (uint32_t*)malloc(sizeof(uint32_t) * out_w);
    uint32_t* txw = (uint32_t*)malloc(sizeof(uint32_t) * out_w);
    for (uint32_t ox = 0; ox < out_w; ++ox) {
        const uint32_t mx = prm->flip ? out_w - 1 - ox : ox;
        lo_resize_tap(mx, out_w, prm->cw, &txl[ox], &txw[ox]);
    }
    for (uint32_t oy = 0; oy < out_h; ++oy) {
        uint32_t ylo, wy;
        lo_resize_tap(oy, out_h, prm->ch, &ylo, &wy);
        const uint32_t yhi = wy ? ylo + 1 : ylo;
        const uint8_t* r0 = src + ((uint64_t)(prm->y0 + ylo) * W) * 3;
        const uint8_t* r1 = src + ((uint64_t)(prm->y0 + yhi) * W) * 3;
        for (uint32_t ox = 0; ox < out_w; ++ox) {
            const uint32_t wx = txw[ox];
            const uint64_t a = (uint64_t)(prm->x0 + txl[ox]) * 3;
            const uint64_t b = wx ? a + 3 : a;
            const uint32_t w00 = (128 - wx) * (128 - wy), w01 = wx * (128 - wy);
            const uint32_t w10 = (128 - wx) * wy, w11 = wx * wy;
            for (int c = 0; c < 3; ++c) {
                const uint32_t v = w00 * r0[a + c] + w01 * r0[b + c] + w10 * r1[a + c] +
                                   w11 * r1[b + c];
                const float o = ((float)v * 0x1p-14f - mean255[c]) * inv_std255[c];
                store_px(out, c * plane + (uint64_t)oy * out_w + ox, o, out_bf16);
            }
        }
    }
    free(txl);
    free(txw);
}

typedef struct {
    const uint8_t* const* srcs;
    const uint32_t* Hs;
    const uint32_t* Ws;
    const lo_aug_params* prms;
    uint64_t begin, end;
    uint32_t out_h, out_w;
    int mode;
    const float* mean255;
    const float* inv_std255;
    int out_bf16;
    void* out;
} aug_job;

static void* aug_worker(void* arg) {
    const aug_job* j = (const aug_job*)arg;
    const uint64_t per = 3ull * j->out_h * j->out_w * (j->out_bf16 ? 2 : 4);
    for (uint64_t i = j->begin; i < j->end; ++i) {
        lo_augment_one(j->srcs[i], j->Hs[i], j->Ws[i], &j->prms[i], j->out_h, j->out_w, j->mode,
                       j->mean255, j->inv_std255, j->out_bf16, (uint8_t*)j->out + i * per);
    }
    return NULL;
}

void lo_augment_batch_mt(const uint8_t* const* srcs, const uint32_t* Hs, const uint32_t* Ws,
                         const lo_aug_params* prms, uint64_t n, uint32_t out_h, uint32_t out_w,
                         int mode, const float mean255[3], const float inv_std255[3],
                         int out_bf16, void* out, int threads) {
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > n) threads = n ? (int)n : 1;
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    aug_job* jobs = (aug_job*)malloc(sizeof(aug_job) * threads);
    for (int t = 0; t < threads; ++t) {
        jobs[t].srcs = srcs; jobs[t].Hs = Hs; jobs[t].Ws = Ws; jobs[t].prms = prms;
        jobs[t].begin = n * t / threads;
        jobs[t].end = n * (t + 1) / threads;
        jobs[t].out_h = out_h; jobs[t].out_w = out_w; jobs[t].mode = mode;
        jobs[t].mean255 = mean255; jobs[t].inv_std255 = inv_std255;
        jobs[t].out_bf16 = out_bf16; jobs[t].out = out;
        if (t > 0) pthread_create(&tid[t], NULL, aug_worker, &jobs[t]);
    }
    aug_worker(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    free(tid);
    free(jobs);
}

typedef struct {
    const uint8_t* pool;
    uint64_t pool_n;
    const uint64_t* ids;
    uint64_t begin, end;
    uint32_t H, W, out_h, out_w;
    uint64_t seed, epoch;
    const float* lut;      /* [3][256] */
    const uint16_t* lut16; /* [3][256] */
    int out_bf16;
    void* out;
} crop_job;

static void* crop_worker(void* arg) {
    const crop_job* j = (const crop_job*)arg;
    const uint64_t plane = (uint64_t)j->out_h * j->out_w;
    const uint64_t S = (uint64_t)j->H * j->W * 3;
    for (uint64_t i = j->begin; i < j->end; ++i) {
        lo_aug_params prm;
        lo_aug_params_for(j->seed, j->epoch, j->ids[i], j->H, j->W, j->out_h, j->out_w,
                          LO_AUG_CROP, &prm);
        const uint8_t* src = j->pool + (j->ids[i] % j->pool_n) * S;
        for (uint32_t oy = 0; oy < j->out_h; ++oy) {
            const uint8_t* row = src + ((uint64_t)(prm.y0 + oy) * j->W + prm.x0) * 3;
            for (int c = 0; c < 3; ++c) {
                const uint64_t o = (i * 3 + c) * plane + (uint64_t)oy * j->out_w;
                if (j->out_bf16) {
                    const uint16_t* t = j->lut16 + 256 * c;
                    uint16_t* dst = (uint16_t*)j->out + o;
                    if (prm.flip)
                        for (uint32_t x = 0; x < j->out_w; ++x)
                            dst[x] = t[row[(j->out_w - 1 - x) * 3 + c]];
                    else
                        for (uint32_t x = 0; x < j->out_w; ++x) dst[x] = t[row[x * 3 + c]];
                } else {
                    const float* t = j->lut + 256 * c;
                    float* dst = (float*)j->out + o;
                    if (prm.flip)
                        for (uint32_t x = 0; x < j->out_w; ++x)
                            dst[x] = t[row[(j->out_w - 1 - x) * 3 + c]];
                    else
                        for (uint32_t x = 0; x < j->out_w; ++x) dst[x] = t[row[x * 3 + c]];
                }
            }
        }
    }
    return NULL;
}

void lo_cpu_crop_step(const uint8_t* pool, uint64_t pool_n, const uint64_t* ids, uint64_t n,
                      uint32_t H, uint32_t W, uint64_t seed, uint64_t epoch, uint32_t out_h,
                      uint32_t out_w, const float mean255[3], const float inv_std255[3],
                      int out_bf16, void* out, int threads) {
    float lut[3 * 256];
    uint16_t lut16[3 * 256];
    for (int c = 0; c < 3; ++c)
        for (int v = 0; v < 256; ++v) {
            lut[256 * c + v] = ((float)v - mean255[c]) * inv_std255[c];
            lut16[256 * c + v] = lo_bf16_rne(lut[256 * c + v]);
        }
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > n) threads = n ? (int)n : 1;
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    crop_job* jobs = (crop_job*)malloc(sizeof(crop_job) * threads);
    for (int t = 0; t < threads; ++t) {
        crop_job* j = &jobs[t];
        j->pool = pool; j->pool_n = pool_n; j->ids = ids;
        j->begin = n * t / threads; j->end = n * (t + 1) / threads;
        j->H = H; j->W = W; j->out_h = out_h; j->out_w = out_w;
        j->seed = seed; j->epoch = epoch; j->lut = lut; j->lut16 = lut16;
        j->out_bf16 = out_bf16; j->out = out;
        if (t > 0) pthread_create(&tid[t], NULL, crop_worker, j);
    }
    crop_worker(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    free(tid);
    free(jobs);
}

typedef struct {
    const uint8_t* const* srcs;
    const uint32_t* Hs;
    const uint32_t* Ws;
    uint64_t pool_n;
    const uint64_t* ids;
    uint64_t begin, end, seed, epoch;
    uint32_t out_h, out_w;
    const float* mean255;
    const float* inv_std255;
    int out_bf16;
    void* out;
} resize_job;

static void* resize_worker(void* arg) {
    const resize_job* j = (const resize_job*)arg;
    const uint64_t per = 3ull * j->out_h * j->out_w * (j->out_bf16 ? 2 : 4);
    for (uint64_t i = j->begin; i < j->end; ++i) {
        const uint64_t slot = j->ids[i] % j->pool_n;
        lo_aug_params prm;
        lo_aug_params_for(j->seed, j->epoch, j->ids[i], j->Hs[slot], j->Ws[slot], j->out_h,
                          j->out_w, LO_AUG_RESIZE, &prm);
        lo_augment_one(j->srcs[slot], j->Hs[slot], j->Ws[slot], &prm, j->out_h, j->out_w,
                       LO_AUG_RESIZE, j->mean255, j->inv_std255, j->out_bf16,
                       (uint8_t*)j->out + i * per);
    }
    return NULL;
}

void lo_cpu_resize_step(const uint8_t* const* srcs, const uint32_t* Hs, const uint32_t* Ws,
                        uint64_t pool_n, const uint64_t* ids, uint64_t n, uint64_t seed,
                        uint64_t epoch, uint32_t out_h, uint32_t out_w, const float mean255[3],
                        const float inv_std255[3], int out_bf16, void* out, int threads) {
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > n) threads = n ? (int)n : 1;
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    resize_job* jobs = (resize_job*)malloc(sizeof(resize_job) * threads);
    for (int t = 0; t < threads; ++t) {
        resize_job* j = &jobs[t];
        j->srcs = srcs; j->Hs = Hs; j->Ws = Ws; j->pool_n = pool_n; j->ids = ids;
        j->begin = n * t / threads; j->end = n * (t + 1) / threads;
        j->seed = seed; j->epoch = epoch; j->out_h = out_h; j->out_w = out_w;
        j->mean255 = mean255; j->inv_std255 = inv_std255; j->out_bf16 = out_bf16; j->out = out;
        if (t > 0) pthread_create(&tid[t], NULL, resize_worker, j);
    }
    resize_worker(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    free(tid);
    free(jobs);
}
