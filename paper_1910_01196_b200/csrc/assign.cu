// assign.cu -- K4: locality-aware assignment of every step of an epoch.
//
// One CTA per global batch.  Composes, bit-exactly:
//   loc_distribution          proj/src/sampling.cpp:44-63  (owner = s*p/cached,
//                             lists in batch order -> STABLE partition)
//   counts_with_uncached      sampling.cpp:65-72           (k-th uncached -> k mod p)
//   targets                   balance.cpp:14-28
//   balance (Algorithm 1)     balance.cpp:58-84            (heap order (imbalance,
//                             lowest id) == argmax scan, ids unique)
//   tail moves                equivalence.cpp:77-88        (receiver appends the
//                             sender's last `count`, in schedule order)
//   reg_slice                 sampling.cpp:27-42           (REGULAR scheme)
//
// Pass 1 tiles the batch 1024 samples at a time: __match_any_sync groups the
// lanes of a warp by owner, popc gives warp-local ranks and counts, a per-group
// scan over the 32 warps gives the stable rank of every sample inside its
// owner's list.  Thread 0 then runs Algorithm 1 on <= 64 learners.  Pass 2
// maps every sample (owner, rank) -> (final learner, final index) through the
// move table and scatters it.  The uncached samples of the batch are placed,
// in batch order, after their dealt learner's cached ones (this build's
// definition; the reference only deals counts), so tail moves hand them over
// first -- they cost no NVLink bytes.
#include "ll_internal.h"
#include "locload_rng.cuh"

namespace ll {
namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;

// Algorithm 1 on imb[0..p) (modified in place).  Returns #moves.
template <typename I>
__device__ __forceinline__ uint32_t greedy_balance(I* imb, uint32_t p, ll_move* out) {
    uint32_t n = 0;
    for (;;) {
        int s = -1, r = -1;
        for (uint32_t j = 0; j < p; ++j) {
            const I v = imb[j];
            if (v > 0 && (s < 0 || v > imb[s])) s = static_cast<int>(j);
            if (v < 0 && (r < 0 || -v > -imb[r])) r = static_cast<int>(j);
        }
        if (s < 0) break;
        const I m = imb[s] < -imb[r] ? imb[s] : -imb[r];
        ll_move mv{};
        mv.sender = static_cast<uint32_t>(s);
        mv.receiver = static_cast<uint32_t>(r);
        mv.count = static_cast<uint32_t>(m);
        out[n++] = mv;
        imb[s] -= m;
        imb[r] += m;
    }
    return n;
}

struct AssignArgs {
    const uint32_t* order;
    uint64_t B;
    uint32_t p;
    uint64_t cached;
    int scheme;
    AugPlan aug;
};

// Crop parameters of sample s (lo_aug_params_for, CROP mode), packed.
__device__ __forceinline__ uint32_t crop_params(const AugPlan& g, uint32_t s) {
    SplitMix r(derive_seed(g.seed, g.epoch, s));
    const uint32_t y0 = static_cast<uint32_t>(r.bounded(static_cast<uint64_t>(g.H - g.ch) + 1));
    const uint32_t x0 = static_cast<uint32_t>(r.bounded(static_cast<uint64_t>(g.W - g.cw) + 1));
    const uint32_t flip = static_cast<uint32_t>(r.next() >> 63);
    return y0 | (x0 << 15) | (flip << 31);
}

__global__ void __launch_bounds__(kThreads) k_assign(AssignArgs a, PlanDev P) {
    const uint32_t st = blockIdx.x;
    const uint64_t B = a.B;
    const uint32_t p = a.p;
    const uint32_t* batch = a.order + st * B;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    __shared__ uint32_t wcnt[kWarps][kMaxP + 2];
    __shared__ uint32_t total[kMaxP + 1];
    __shared__ uint32_t off[kMaxP + 1];
    __shared__ uint32_t kept[kMaxP];
    __shared__ uint32_t cnt[kMaxP];
    __shared__ ll_move mv[kMaxP];
    __shared__ uint32_t nmv;
    __shared__ uint32_t mv_nvl[kMaxP];
    __shared__ uint32_t reg_remote;
    __shared__ long long imb[kMaxP];
    __shared__ uint32_t rc[kMaxP * kMaxP];  // regular + NCCL: [slice][owner] counts

    uint32_t* scratch = P.scratch + st * B;
    uint32_t* final_ids = P.final_ids + st * B;
    const uint64_t slice = (B % p == 0) ? B / p : 0;

    if (tid <= p) total[tid] = 0;
    if (tid < kMaxP) mv_nvl[tid] = 0;
    if (tid == 0) reg_remote = 0;
    const bool want_rc = slice && P.regcnt != nullptr;
    if (want_rc)
        for (uint32_t i = tid; i < p * p; i += kThreads) rc[i] = 0;
    __syncthreads();

    // ---- pass 1: stable rank of every sample inside its owner group -------
    uint32_t my_reg_remote = 0;
    for (uint64_t t0 = 0; t0 < B; t0 += kThreads) {
        const uint64_t e = t0 + tid;
        const bool valid = e < B;
        uint32_t g = 0xFFFFFFFFu;
        if (valid) {
            const uint64_t s = batch[e];
            g = s < a.cached ? static_cast<uint32_t>(s * p / a.cached) : p;
            if (slice && g != static_cast<uint32_t>(e / slice) && g < p) ++my_reg_remote;
            if (want_rc && g < p) atomicAdd(&rc[static_cast<uint32_t>(e / slice) * p + g], 1u);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, g);
        const uint32_t lrank = __popc(peers & ((1u << lane) - 1u));
        for (uint32_t q = lane; q <= p; q += 32) wcnt[warp][q] = 0;
        __syncwarp();
        if (valid && lrank == 0) wcnt[warp][g] = __popc(peers);
        __syncthreads();
        if (tid <= p) {
            uint32_t run = total[tid];
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t c = wcnt[w][tid];
                wcnt[w][tid] = run;
                run += c;
            }
            total[tid] = run;
        }
        __syncthreads();
        if (valid) scratch[e] = (g << 24) | (wcnt[warp][g] + lrank);
        __syncthreads();
    }
    if (my_reg_remote) atomicAdd(&reg_remote, my_reg_remote);

    // ---- schedule (one thread; p <= 64) -----------------------------------
    if (tid == 0) {
        const uint32_t U = total[p];
        for (uint32_t j = 0; j < p; ++j) cnt[j] = total[j] + U / p + (j < U % p ? 1u : 0u);
        nmv = 0;
        if (a.scheme == LL_SCHEME_LOCALITY_BALANCED) {
            const uint32_t base = static_cast<uint32_t>(B / p), rem = static_cast<uint32_t>(B % p);
            for (uint32_t j = 0; j < p; ++j)
                imb[j] = static_cast<long long>(cnt[j]) -
                         static_cast<long long>(base + (j < rem ? 1u : 0u));
            nmv = greedy_balance(imb, p, mv);
            LL_DCHECK(nmv + 1 <= p || nmv == 0);
            uint32_t taken[kMaxP], recvd[kMaxP];
            for (uint32_t j = 0; j < p; ++j) taken[j] = recvd[j] = 0;
            for (uint32_t m = 0; m < nmv; ++m) {
                const uint32_t s = mv[m].sender, r = mv[m].receiver;
                mv[m].src_off = cnt[s] - taken[s] - mv[m].count;
                mv[m].dst_off = cnt[r] + recvd[r];
                taken[s] += mv[m].count;
                recvd[r] += mv[m].count;
            }
            off[0] = 0;
            for (uint32_t j = 0; j < p; ++j) {
                kept[j] = cnt[j] - taken[j];
                off[j + 1] = off[j] + base + (j < rem ? 1u : 0u);
            }
        } else if (a.scheme == LL_SCHEME_LOCALITY) {
            off[0] = 0;
            for (uint32_t j = 0; j < p; ++j) {
                kept[j] = cnt[j];
                off[j + 1] = off[j] + cnt[j];
            }
        } else {  // regular
            for (uint32_t j = 0; j <= p; ++j) off[j] = static_cast<uint32_t>(slice * j);
            for (uint32_t j = 0; j < p; ++j) kept[j] = cnt[j] = static_cast<uint32_t>(slice);
        }
    }
    __syncthreads();

    // ---- pass 2: scatter into the final lists -------------------------------
    uint32_t my_nvl_moved = 0;
    for (uint64_t e = tid; e < B; e += kThreads) {
        const uint32_t s = batch[e];
        if (a.scheme == LL_SCHEME_REGULAR) {
            final_ids[e] = s;
            if (a.aug.enabled) P.aug[st * B + e] = crop_params(a.aug, s);
            continue;
        }
        const uint32_t v = scratch[e];
        const uint32_t g = v >> 24, r = v & 0xFFFFFFu;
        uint32_t j, k;
        if (g < p) {
            j = g;
            k = r;
        } else {
            j = r % p;
            k = total[j] + r / p;
        }
        uint32_t fj = j, fk = k;
        if (k >= kept[j]) {
            for (uint32_t m = 0; m < nmv; ++m) {
                if (mv[m].sender == j && k >= mv[m].src_off && k < mv[m].src_off + mv[m].count) {
                    fj = mv[m].receiver;
                    fk = mv[m].dst_off + (k - mv[m].src_off);
                    if (g < p) atomicAdd(&mv_nvl[m], 1u);
                    ++my_nvl_moved;
                    break;
                }
            }
        }
        LL_DCHECK(fj < p && off[fj] + fk < off[fj + 1] && off[fj + 1] <= B);
        final_ids[off[fj] + fk] = s;
        if (a.aug.enabled) P.aug[st * B + off[fj] + fk] = crop_params(a.aug, s);
    }
    (void)my_nvl_moved;
    __syncthreads();

    // ---- plan records -------------------------------------------------------
    if (want_rc)
        for (uint32_t i = tid; i < p * p; i += kThreads) P.regcnt[st * p * p + i] = rc[i];
    if (tid <= p) P.off[st * (kMaxP + 1) + tid] = off[tid];
    if (tid < p) {
        P.kept[st * kMaxP + tid] = kept[tid];
        P.counts[st * kMaxP + tid] = cnt[tid];
    }
    if (tid < nmv) {
        ll_move m = mv[tid];
        m.nvlink = mv_nvl[tid];
        P.moves[st * kMaxP + tid] = m;
    }
    if (tid == 0) {
        P.n_moves[st] = nmv;
        uint32_t moved = 0, nvl = 0;
        for (uint32_t m = 0; m < nmv; ++m) {
            moved += mv[m].count;
            nvl += mv_nvl[m];
        }
        P.stats[st * 4 + 0] = moved;
        P.stats[st * 4 + 1] = nvl;
        P.stats[st * 4 + 2] = total[p];
        P.stats[st * 4 + 3] = slice ? reg_remote : 0xFFFFFFFFu;
    }
}

__global__ void k_balance_batch(const int64_t* __restrict__ counts,
                                const int64_t* __restrict__ targets, uint32_t p, uint64_t n,
                                ll_move* __restrict__ moves, uint32_t* __restrict__ n_moves) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    long long imb[kMaxP];
    for (uint32_t j = 0; j < p; ++j) imb[j] = counts[i * p + j] - targets[i * p + j];
    ll_move mv[kMaxP];
    const uint32_t m = greedy_balance(imb, p, mv);
    for (uint32_t k = 0; k < m; ++k) moves[i * p + k] = mv[k];
    n_moves[i] = m;
}

} // namespace

PlanDev PlanBufs::view() const {
    PlanDev v;
    v.final_ids = final_ids.as<uint32_t>();
    v.off = off.as<uint32_t>();
    v.kept = kept.as<uint32_t>();
    v.counts = counts.as<uint32_t>();
    v.moves = moves.as<ll_move>();
    v.n_moves = n_moves.as<uint32_t>();
    v.stats = stats.as<uint32_t>();
    v.scratch = scratch.as<uint32_t>();
    v.aug = aug.as<uint32_t>();
    v.regcnt = regcnt.as<uint32_t>();
    return v;
}

void PlanBufs::reserve_regcnt(uint64_t steps, uint32_t p) {
    regcnt.reserve(sizeof(uint32_t) * steps * p * p);
}

void PlanBufs::reserve(uint64_t steps, uint64_t B) {
    final_ids.reserve(sizeof(uint32_t) * steps * B);
    scratch.reserve(sizeof(uint32_t) * steps * B);
    aug.reserve(sizeof(uint32_t) * steps * B);
    off.reserve(sizeof(uint32_t) * steps * (kMaxP + 1));
    kept.reserve(sizeof(uint32_t) * steps * kMaxP);
    counts.reserve(sizeof(uint32_t) * steps * kMaxP);
    moves.reserve(sizeof(ll_move) * steps * kMaxP);
    n_moves.reserve(sizeof(uint32_t) * steps);
    stats.reserve(sizeof(uint32_t) * steps * 4);
}

void assign_device(ll_ctx* ctx, const uint32_t* d_order, uint64_t steps, uint64_t B, uint32_t p,
                   uint64_t cached, int scheme, const PlanDev& plan, const AugPlan& aug) {
    require(p >= 1 && p <= kMaxP, "assign: learner count must be in [1, 64]");
    require(B < (1ull << 24), "assign: batch size must be < 2^24");
    if (scheme == LL_SCHEME_REGULAR)
        require(B % p == 0, "reg_slice: learner count must divide the batch size");
    if (steps == 0) return;
    require(!aug.enabled || (plan.aug != nullptr && aug.H >= aug.ch && aug.W >= aug.cw &&
                             aug.H < 32768 && aug.W < 32768),
            "assign: bad crop-parameter plan");
    AssignArgs a{d_order, B, p, cached, scheme, aug};
    launch(ctx, "assign", [&] {
        k_assign<<<static_cast<unsigned>(steps), kThreads, 0, ctx->stream>>>(a, plan);
    });
}

void balance_device(ll_ctx* ctx, const int64_t* d_counts, const int64_t* d_targets, uint32_t p,
                    uint64_t n, ll_move* d_moves, uint32_t* d_n) {
    if (n == 0) return;
    launch(ctx, "balance", [&] {
        k_balance_batch<<<static_cast<unsigned>((n + 127) / 128), 128, 0, ctx->stream>>>(
            d_counts, d_targets, p, n, d_moves, d_n);
    });
}

} // namespace ll
