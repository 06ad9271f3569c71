// permute.cu -- K2 + K3: bit-exact parallel forward Fisher-Yates.
//
// Reference: permute_epoch, proj/src/core.cpp:11-27.  Sequentially,
//     for i in [0, d): j = i + bounded(d - i); swap(order[i], order[j])
// over SplitMix64(derive_seed(seed, epoch)).
//
// Two observations make it parallel and still bit-exact:
//  1. The stream is counter based (rng.hpp:35-38), so draw i is
//     mix64(s0 + (i+1)*gamma) as long as no earlier Lemire trial rejected.
//     All d draws J[i] are computed at once; the (probability < d/2^64)
//     rejection is detected and repaired exactly by re-drawing the rejected
//     index and shifting every later draw index (fix-up loop below).
//  2. Deterministic reservations (Shun, Gu, Blelloch, Fineman, Gibbons,
//     SODA'15): iteration i touches positions {i, J[i]}.  Each round every
//     pending iteration priority-writes its index into R[i] and R[J[i]]; the
//     ones that own both slots have no pending predecessor touching their
//     positions, so they swap now, in any order, exactly as the sequential
//     loop would.  Rounds continue on the survivors.  Iterations with
//     J[i] == i are no-ops and are dropped.
//
// Priorities are (round << 32 | ~i) under atomicMax, so R needs no reset
// between rounds.  One cooperative persistent kernel runs everything; once the
// survivor list is small, CTA 0 finishes alone with block barriers.
#include <cooperative_groups.h>

#include "ll_internal.h"
#include "locload_rng.cuh"

namespace cg = cooperative_groups;

namespace ll {
namespace {

constexpr int kThreads = 512;
constexpr uint32_t kSmallList = 16384;  // survivors handed to a single CTA
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kMaxRounds = 4096;   // O(log d) expected (~50 at d = 1.28 M); hang guard

struct PermArgs {
    uint64_t s0;
    uint32_t d;
    uint32_t* A;               // order being permuted
    uint32_t* J;               // swap partner of iteration i
    unsigned long long* R;     // reservations
    uint32_t* L0;              // survivor lists
    uint32_t* L1;
    unsigned int* ctl;         // [0..1] reject cells, [2] rounds, [4..6] list counters
    unsigned long long* shift; // extra draws consumed before the current index
    const uint64_t* forced;    // sorted forced-reject draw indices (test hook)
    uint32_t n_forced;
};

__device__ __forceinline__ uint32_t ldcg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ldcg64(const unsigned long long* p) {
    return __ldcg(p);
}

__device__ __forceinline__ bool is_forced(const uint64_t* f, uint32_t n, uint64_t k) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (f[mid] < k) lo = mid + 1; else hi = mid;
    }
    return lo < n && f[lo] == k;
}

// Draw with 0-based stream index k0 for range n; false when rejected.
__device__ __forceinline__ bool fy_draw(const PermArgs& a, uint64_t k0, uint32_t n,
                                        uint32_t* off) {
    uint64_t v;
    bool ok = lemire_accept(draw_at(a.s0, k0), n, &v);
    if (a.n_forced && is_forced(a.forced, a.n_forced, k0)) ok = false;
    *off = static_cast<uint32_t>(v);
    return ok;
}

__device__ __forceinline__ unsigned long long prio(uint32_t round, uint32_t i) {
    return (static_cast<unsigned long long>(round) << 32) | (0xFFFFFFFFu - i);
}

// One reserve+commit round over `n` pending iterations read from `cur`
// (or the identity when cur == nullptr) by threads [t0, t0+nth).
template <typename Sync>
__device__ __forceinline__ uint32_t run_round(const PermArgs& a, const uint32_t* cur, uint32_t n,
                                              uint32_t* next, unsigned int* next_cnt,
                                              uint32_t round, uint32_t gtid, uint32_t nth,
                                              Sync&& sync) {
    for (uint32_t t = gtid; t < n; t += nth) {
        const uint32_t i = cur ? ldcg(cur + t) : t;
        const uint32_t j = ldcg(a.J + i);
        if (j == i) continue;
        const unsigned long long key = prio(round, i);
        atomicMax(a.R + i, key);
        atomicMax(a.R + j, key);
    }
    sync();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nth_w = nth & ~31u;  // nth is a multiple of 32
    for (uint32_t tb = gtid - lane; tb < n; tb += nth_w) {
        const uint32_t t = tb + lane;
        bool pend = false;
        uint32_t i = 0;
        if (t < n) {
            i = cur ? ldcg(cur + t) : t;
            const uint32_t j = ldcg(a.J + i);
            if (j != i) {
                const unsigned long long key = prio(round, i);
                if (ldcg64(a.R + i) == key && ldcg64(a.R + j) == key) {
                    const uint32_t vi = ldcg(a.A + i), vj = ldcg(a.A + j);
                    a.A[i] = vj;
                    a.A[j] = vi;
                } else {
                    pend = true;
                }
            }
        }
        const unsigned mask = __ballot_sync(0xffffffffu, pend);
        if (mask) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(next_cnt, __popc(mask));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (pend) next[base + __popc(mask & ((1u << lane) - 1u))] = i;
        }
    }
    sync();
    return ldcg(next_cnt);
}

__global__ void __launch_bounds__(kThreads) k_permute(PermArgs a) {
    cg::grid_group grid = cg::this_grid();
    const uint32_t d = a.d;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t nth = gridDim.x * blockDim.x;

    // K2: identity, reservations cleared, all draws with shift 0.
    for (uint32_t i = gtid; i < d; i += nth) {
        a.A[i] = i;
        a.R[i] = 0ull;
        uint32_t off;
        const bool ok = fy_draw(a, i, d - i, &off);
        a.J[i] = i + off;
        if (!ok) atomicMin(&a.ctl[0], i);
    }

    // Exact repair of Lemire rejections (core.cpp:22 via rng.hpp:45-49): the
    // first rejected index re-draws sequentially, every later index shifts.
    uint64_t shift = 0;
    for (uint32_t it = 0;; ++it) {
        grid.sync();
        const uint32_t i0 = ldcg(&a.ctl[it & 1]);
        if (i0 >= d) break;
        if (gtid == 0) {
            uint64_t k = i0 + shift + 1;
            uint32_t off;
            while (!fy_draw(a, k, d - i0, &off)) ++k;
            a.J[i0] = i0 + off;
            *a.shift = k - i0;
            a.ctl[(it + 1) & 1] = kNone;
        }
        grid.sync();
        shift = ldcg64(a.shift);
        for (uint64_t i = static_cast<uint64_t>(i0) + 1 + gtid; i < d; i += nth) {
            uint32_t off;
            const bool ok = fy_draw(a, i + shift, d - static_cast<uint32_t>(i), &off);
            a.J[i] = static_cast<uint32_t>(i) + off;
            if (!ok) atomicMin(&a.ctl[(it + 1) & 1], static_cast<uint32_t>(i));
        }
    }

    // K3: deterministic-reservation rounds over the whole grid.
    const uint32_t* cur = nullptr;
    uint32_t n = d;
    uint32_t round = 1;
    auto gsync = [&] { grid.sync(); };
    while (n > kSmallList && round < kMaxRounds) {
        uint32_t* next = (cur == a.L0) ? a.L1 : a.L0;
        unsigned int* cnt = &a.ctl[4 + round % 3];
        if (gtid == 0) a.ctl[4 + (round + 1) % 3] = 0;
        n = run_round(a, cur, n, next, cnt, round, gtid, nth, gsync);
        cur = next;
        ++round;
    }
    if (blockIdx.x != 0) return;
    // Tail rounds inside CTA 0 (all grid writes are visible after grid.sync).
    auto bsync = [] { __syncthreads(); };
    while (n > 0 && round < kMaxRounds) {
        uint32_t* next = (cur == a.L0) ? a.L1 : a.L0;
        unsigned int* cnt = &a.ctl[4 + round % 3];
        if (threadIdx.x == 0) a.ctl[4 + (round + 1) % 3] = 0;
        n = run_round(a, cur, n, next, cnt, round, threadIdx.x, blockDim.x, bsync);
        cur = next;
        ++round;
    }
    if (threadIdx.x == 0) {
        a.ctl[2] = round - 1;
        a.ctl[3] = n;  // survivors left: non-zero only if the round guard tripped
    }
}

__global__ void k_widen(const uint32_t* __restrict__ in, uint64_t* __restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = in[i];
}

} // namespace

void permute_device(ll_ctx* ctx, uint64_t seed, uint64_t epoch, uint32_t d, uint32_t* d_order,
                    const uint64_t* host_forced, uint64_t n_forced) {
    DevBuf& J = ctx->buf("perm.J", sizeof(uint32_t) * d);
    DevBuf& R = ctx->buf("perm.R", sizeof(unsigned long long) * d);
    DevBuf& L0 = ctx->buf("perm.L0", sizeof(uint32_t) * d);
    DevBuf& L1 = ctx->buf("perm.L1", sizeof(uint32_t) * d);
    DevBuf& ctl = ctx->buf("perm.ctl", 64);
    unsigned int init[16] = {kNone, kNone, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    LL_CUDA(cudaMemcpyAsync(ctl.ptr, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
    PermArgs a{};
    a.s0 = derive_seed(seed, epoch);
    a.d = d;
    a.A = d_order;
    a.J = J.as<uint32_t>();
    a.R = R.as<unsigned long long>();
    a.L0 = L0.as<uint32_t>();
    a.L1 = L1.as<uint32_t>();
    a.ctl = ctl.as<unsigned int>();
    a.shift = reinterpret_cast<unsigned long long*>(ctl.as<unsigned int>() + 8);
    a.n_forced = static_cast<uint32_t>(n_forced);
    if (n_forced) {
        DevBuf& forced = ctx->buf("perm.forced", sizeof(uint64_t) * n_forced);
        LL_CUDA(cudaMemcpyAsync(forced.ptr, host_forced, sizeof(uint64_t) * n_forced,
                                cudaMemcpyHostToDevice, ctx->stream));
        LL_CUDA(cudaStreamSynchronize(ctx->stream));  // host_forced may be pageable
        a.forced = forced.as<uint64_t>();
    }
    int per_sm = 0;
    LL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_permute, kThreads, 0));
    if (per_sm < 1) fail(LL_ERR_CUDA, "permute: kernel cannot be resident");
    const uint64_t want = (static_cast<uint64_t>(d) + kThreads - 1) / kThreads;
    const uint64_t cap = static_cast<uint64_t>(per_sm) * ctx->sm_count;
    const unsigned grid = static_cast<unsigned>(want < cap ? (want ? want : 1) : cap);
    void* args[] = {&a};
    launch(ctx, "permute", [&] {
        LL_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_permute), dim3(grid),
                                            dim3(kThreads), args, 0, ctx->stream));
    });
}

uint32_t permute_rounds(ll_ctx* ctx) {
    unsigned int ctl[2] = {0, 0};
    LL_CUDA(cudaMemcpyAsync(ctl, ctx->buf("perm.ctl", 64).as<unsigned int>() + 2, sizeof(ctl),
                            cudaMemcpyDeviceToHost, ctx->stream));
    LL_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctl[1] != 0) fail(LL_ERR_RUNTIME, "permute: round limit exceeded (internal error)");
    return ctl[0];
}

void widen_device(ll_ctx* ctx, const uint32_t* in, uint64_t* out, uint64_t n) {
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148u * 8u));
    launch(ctx, "widen", [&] { k_widen<<<grid ? grid : 1, 256, 0, ctx->stream>>>(in, out, n); });
}

} // namespace ll
