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
// between rounds.  One cooperative persistent kernel runs everything; once at
// most 2,048 iterations survive, CTA 0 finishes them in shared memory.
#include <cooperative_groups.h>

#include "ll_internal.h"
#include "locload_rng.cuh"

namespace cg = cooperative_groups;

namespace ll {
namespace {

constexpr int kThreads = 512;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kMaxRounds = 4096;   // O(log d) expected (~50 at d = 1.28 M); hang guard

struct PermArgs {
    uint64_t s0;
    uint32_t d;
    uint32_t* A;               // order being permuted
    uint32_t* J;               // swap partner of iteration i
    unsigned long long* R;     // reservations
    uint2* L0;                 // survivor lists of (i, J[i])
    uint2* L1;
    unsigned int* ctl;         // [0..1] reject cells, [2] rounds, [4..6] list counters
    unsigned long long* shift; // extra draws consumed before the current index
    const uint64_t* forced;    // sorted forced-reject draw indices (test hook)
    uint32_t n_forced;
};

__device__ __forceinline__ uint32_t ldcg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
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
// (or the identity when cur == nullptr) by threads [gtid, +nth).  Each thread
// works on kU iterations at a time with every load of the batch issued before
// any is consumed (memory-level parallelism: the loads are dependent chains
// cur -> J -> R -> A through L2).
constexpr uint32_t kU = 4;

// Survivor lists hold (i, J[i]) pairs so a round needs no J lookup; the first
// round walks the identity and reads J.
__device__ __forceinline__ void load_pairs(const PermArgs& a, const uint2* cur, uint32_t n,
                                           uint32_t t0, uint32_t nth, uint32_t* i, uint32_t* j) {
#pragma unroll
    for (uint32_t u = 0; u < kU; ++u) {
        const uint32_t t = t0 + u * nth;
        if (t >= n) {
            i[u] = j[u] = 0xFFFFFFFFu;
        } else if (cur) {
            const uint2 v = __ldcg(cur + t);
            i[u] = v.x;
            j[u] = v.y;
        } else {
            i[u] = t;
            j[u] = ldcg(a.J + t);
        }
    }
}

__device__ __forceinline__ uint32_t run_round(const PermArgs& a, const uint2* cur, uint32_t n,
                                              uint2* next, unsigned int* next_cnt,
                                              uint32_t round, uint32_t gtid, uint32_t nth,
                                              cg::grid_group& grid) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t wbase = gtid - lane;  // nth is a multiple of 32
    for (uint32_t tb = wbase; tb < n; tb += nth * kU) {
        uint32_t i[kU], j[kU];
        load_pairs(a, cur, n, tb + lane, nth, i, j);
#pragma unroll
        for (uint32_t u = 0; u < kU; ++u) {
            if (j[u] == i[u]) continue;  // padding or a no-op swap
            LL_DCHECK(i[u] < a.d && j[u] < a.d && j[u] > i[u]);
            const unsigned long long key = prio(round, i[u]);
            atomicMax(a.R + i[u], key);
            atomicMax(a.R + j[u], key);
        }
    }
    grid.sync();
    for (uint32_t tb = wbase; tb < n; tb += nth * kU) {
        uint32_t i[kU], j[kU];
        unsigned long long ri[kU], rj[kU];
        load_pairs(a, cur, n, tb + lane, nth, i, j);
#pragma unroll
        for (uint32_t u = 0; u < kU; ++u) {
            ri[u] = rj[u] = 0;
            if (j[u] != i[u]) {
                ri[u] = ldcg64(a.R + i[u]);
                rj[u] = ldcg64(a.R + j[u]);
            }
        }
        bool win[kU];
        uint32_t vi[kU], vj[kU];
#pragma unroll
        for (uint32_t u = 0; u < kU; ++u) {
            const unsigned long long key = prio(round, i[u]);
            win[u] = j[u] != i[u] && ri[u] == key && rj[u] == key;
            if (win[u]) {
                vi[u] = ldcg(a.A + i[u]);
                vj[u] = ldcg(a.A + j[u]);
            }
        }
#pragma unroll
        for (uint32_t u = 0; u < kU; ++u) {
            if (win[u]) {
                a.A[i[u]] = vj[u];
                a.A[j[u]] = vi[u];
            }
            const bool pend = j[u] != i[u] && !win[u];
            const unsigned mask = __ballot_sync(0xffffffffu, pend);
            if (mask) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(next_cnt, __popc(mask));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (pend) next[base + __popc(mask & ((1u << lane) - 1u))] = make_uint2(i[u], j[u]);
            }
        }
    }
    grid.sync();
    return ldcg(next_cnt);
}

// The last <= kTail survivors, inside CTA 0 and its shared memory: the <= 2*kTail
// positions they touch are gathered into an open-addressing table (position ->
// slot holding its current order value), the remaining rounds reserve with
// shared-memory atomicMin on the iteration index and swap slot values, and the
// slots are written back at the end.  Same deterministic-reservation rule,
// so the result is unchanged; only the memory the rounds run in differs.
constexpr uint32_t kTail = 2048;
constexpr uint32_t kTab = 8192;            // power of two >= 2 * kTail / 0.5
constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr size_t kTailSmem = (3ull * kTab + 5ull * kTail + 4) * sizeof(uint32_t);

__device__ __forceinline__ uint32_t tab_slot(uint32_t* keys, uint32_t* aval, const uint32_t* A,
                                             uint32_t pos) {
    uint32_t h = (pos * 2654435761u) >> (32 - 13);  // log2(kTab) = 13
    for (;;) {
        const uint32_t prev = atomicCAS(&keys[h], kEmpty, pos);
        if (prev == kEmpty) {
            aval[h] = ldcg(A + pos);
            return h;
        }
        if (prev == pos) return h;
        h = (h + 1) & (kTab - 1);
    }
}

__device__ uint32_t smem_tail(const PermArgs& a, const uint2* cur, uint32_t n, uint32_t round) {
    extern __shared__ uint32_t sm[];
    uint32_t* keys = sm;
    uint32_t* aval = keys + kTab;
    uint32_t* rsv = aval + kTab;
    uint32_t* sidx = rsv + kTab;               // iteration index i of local survivor t
    uint32_t* si = sidx + kTail;               // slot of position i
    uint32_t* sj = si + kTail;                 // slot of position J[i]
    uint32_t* lst = sj + kTail;                // two survivor lists (local ids)
    uint32_t* cnt = lst + 2 * kTail;           // [0..1] list counters
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    for (uint32_t h = tid; h < kTab; h += blockDim.x) keys[h] = kEmpty;
    if (tid < 2) cnt[tid] = 0;
    __syncthreads();
    LL_DCHECK(n <= kTail);
    for (uint32_t t = tid; t < n; t += blockDim.x) {
        const uint2 v = __ldcg(cur + t);
        const uint32_t i = v.x, j = v.y;
        LL_DCHECK(i < a.d && j < a.d);
        sidx[t] = i;
        si[t] = tab_slot(keys, aval, a.A, i);
        sj[t] = tab_slot(keys, aval, a.A, j);
        lst[t] = t;
    }
    __syncthreads();
    uint32_t which = 0;
    while (n > 0 && round < kMaxRounds) {
        const uint32_t* in = lst + which * kTail;
        uint32_t* out = lst + (which ^ 1) * kTail;
        for (uint32_t q = tid; q < n; q += blockDim.x) {
            const uint32_t t = in[q];
            rsv[si[t]] = kEmpty;
            rsv[sj[t]] = kEmpty;
        }
        if (tid == 0) cnt[which ^ 1] = 0;
        __syncthreads();
        for (uint32_t q = tid; q < n; q += blockDim.x) {
            const uint32_t t = in[q];
            atomicMin(&rsv[si[t]], sidx[t]);
            atomicMin(&rsv[sj[t]], sidx[t]);
        }
        __syncthreads();
        for (uint32_t qb = tid - lane; qb < n; qb += blockDim.x) {
            const uint32_t q = qb + lane;
            bool pend = false;
            uint32_t t = 0;
            if (q < n) {
                t = in[q];
                const uint32_t x = si[t], y = sj[t], i = sidx[t];
                if (rsv[x] == i && rsv[y] == i) {
                    const uint32_t v = aval[x];
                    aval[x] = aval[y];
                    aval[y] = v;
                } else {
                    pend = true;
                }
            }
            const unsigned mask = __ballot_sync(0xffffffffu, pend);
            if (mask) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(&cnt[which ^ 1], __popc(mask));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (pend) out[base + __popc(mask & ((1u << lane) - 1u))] = t;
            }
        }
        __syncthreads();
        n = cnt[which ^ 1];
        which ^= 1;
        ++round;
        __syncthreads();
    }
    for (uint32_t h = tid; h < kTab; h += blockDim.x)
        if (keys[h] != kEmpty) a.A[keys[h]] = aval[h];
    if (tid == 0) a.ctl[3] = n;  // non-zero only if the round guard tripped
    return round;
}

__global__ void __launch_bounds__(kThreads) k_permute(PermArgs a) {
    cg::grid_group grid = cg::this_grid();
    const uint32_t d = a.d;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t nth = gridDim.x * blockDim.x;
    // phase timestamps (globaltimer ns) for ll_last_permute_profile
    uint64_t* ts = reinterpret_cast<uint64_t*>(a.ctl + 16);
    if (gtid == 0) ts[0] = gtimer();

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

    if (gtid == 0) ts[1] = gtimer();
    // K3: deterministic-reservation rounds over the whole grid ...
    const uint2* cur = nullptr;
    uint32_t n = d;
    uint32_t round = 1;
    while (n > kTail && round < kMaxRounds) {
        uint2* next = (cur == a.L0) ? a.L1 : a.L0;
        unsigned int* cnt = &a.ctl[4 + round % 3];
        if (gtid == 0) a.ctl[4 + (round + 1) % 3] = 0;
        n = run_round(a, cur, n, next, cnt, round, gtid, nth, grid);
        cur = next;
        ++round;
    }
    if (blockIdx.x != 0) return;
    if (threadIdx.x == 0) {
        ts[2] = gtimer();
        a.ctl[12] = round - 1;  // grid-wide rounds
    }
    // ... then the tail in CTA 0's shared memory (grid writes are visible after
    // the last grid.sync).  The first round may still run over the identity
    // list when d itself is small.
    if (n > 0 && cur == nullptr) {
        // d <= kTail: materialise the identity survivor list (no-op swaps dropped)
        uint2* next = a.L0;
        if (threadIdx.x == 0) a.ctl[4] = 0;
        __syncthreads();
        for (uint32_t tb = threadIdx.x - (threadIdx.x & 31); tb < n; tb += blockDim.x) {
            const uint32_t t = tb + (threadIdx.x & 31);
            const uint32_t jt = t < n ? ldcg(a.J + t) : t;
            const bool keep = t < n && jt != t;
            const unsigned mask = __ballot_sync(0xffffffffu, keep);
            if (mask) {
                uint32_t base = 0;
                if ((threadIdx.x & 31) == 0) base = atomicAdd(&a.ctl[4], __popc(mask));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (keep) next[base + __popc(mask & ((1u << (threadIdx.x & 31)) - 1u))] = make_uint2(t, jt);
            }
        }
        __syncthreads();
        n = ldcg(&a.ctl[4]);
        cur = next;
    }
    round = smem_tail(a, cur, n, round);
    if (threadIdx.x == 0) {
        a.ctl[2] = round - 1;
        ts[3] = gtimer();
    }
}

__global__ void k_widen(const uint32_t* __restrict__ in, uint64_t* __restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = in[i];
}

} // namespace

void permute_device(ll_ctx* ctx, uint64_t seed, uint64_t epoch, uint32_t d, uint32_t* d_order,
                    const uint64_t* host_forced, uint64_t n_forced, const char* tag) {
    const std::string t(tag);
    DevBuf& J = ctx->buf(t + ".J", sizeof(uint32_t) * d);
    DevBuf& R = ctx->buf(t + ".R", sizeof(unsigned long long) * d);
    DevBuf& L0 = ctx->buf(t + ".L0", sizeof(uint2) * d);
    DevBuf& L1 = ctx->buf(t + ".L1", sizeof(uint2) * d);
    DevBuf& ctl = ctx->buf(t + ".ctl", 128);
    unsigned int init[16] = {kNone, kNone, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    LL_CUDA(cudaMemcpyAsync(ctl.ptr, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
    PermArgs a{};
    a.s0 = derive_seed(seed, epoch);
    a.d = d;
    a.A = d_order;
    a.J = J.as<uint32_t>();
    a.R = R.as<unsigned long long>();
    a.L0 = L0.as<uint2>();
    a.L1 = L1.as<uint2>();
    a.ctl = ctl.as<unsigned int>();
    a.shift = reinterpret_cast<unsigned long long*>(ctl.as<unsigned int>() + 8);
    a.n_forced = static_cast<uint32_t>(n_forced);
    if (n_forced) {
        DevBuf& forced = ctx->buf(t + ".forced", sizeof(uint64_t) * n_forced);
        LL_CUDA(cudaMemcpyAsync(forced.ptr, host_forced, sizeof(uint64_t) * n_forced,
                                cudaMemcpyHostToDevice, ctx->stream));
        LL_CUDA(cudaStreamSynchronize(ctx->stream));  // host_forced may be pageable
        a.forced = forced.as<uint64_t>();
    }
    ensure_smem_attr(k_permute, ctx->device, kTailSmem);
    int per_sm = 0;
    LL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_permute, kThreads, kTailSmem));
    if (per_sm < 1) fail(LL_ERR_CUDA, "permute: kernel cannot be resident");
    const uint64_t want = (static_cast<uint64_t>(d) + kThreads - 1) / kThreads;
    const uint64_t cap = static_cast<uint64_t>(per_sm) * ctx->sm_count;
    const unsigned grid = static_cast<unsigned>(want < cap ? (want ? want : 1) : cap);
    void* args[] = {&a};
    launch(ctx, "permute", [&] {
        LL_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_permute), dim3(grid),
                                            dim3(kThreads), args, kTailSmem, ctx->stream));
    });
}

uint32_t permute_rounds(ll_ctx* ctx, const char* tag) {
    const std::string t(tag);
    unsigned int ctl[2] = {0, 0};
    LL_CUDA(cudaMemcpyAsync(ctl, ctx->buf(t + ".ctl", 128).as<unsigned int>() + 2, sizeof(ctl),
                            cudaMemcpyDeviceToHost, ctx->stream));
    LL_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctl[1] != 0) fail(LL_ERR_RUNTIME, "permute: round limit exceeded (internal error)");
    return ctl[0];
}

void widen_device(ll_ctx* ctx, const uint32_t* in, uint64_t* out, uint64_t n) {
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148u * 8u));
    launch(ctx, "widen", [&] { k_widen<<<grid ? grid : 1, 256, 0, ctx->stream>>>(in, out, n); });
}

// {rounds, grid-wide rounds, ns draws+repair, ns grid rounds, ns CTA-0 rounds, ns total}
void permute_profile(ll_ctx* ctx, uint64_t* out6, const char* tag) {
    const std::string t(tag);
    unsigned int ctl[32];
    LL_CUDA(cudaMemcpyAsync(ctl, ctx->buf(t + ".ctl", 128).ptr, sizeof(ctl),
                            cudaMemcpyDeviceToHost, ctx->stream));
    LL_CUDA(cudaStreamSynchronize(ctx->stream));
    const uint64_t* ts = reinterpret_cast<const uint64_t*>(ctl + 16);
    out6[0] = ctl[2];
    out6[1] = ctl[12];
    out6[2] = ts[1] - ts[0];
    out6[3] = ts[2] - ts[1];
    out6[4] = ts[3] - ts[2];
    out6[5] = ts[3] - ts[0];
}

} // namespace ll
