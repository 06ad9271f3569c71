// exchange.cu -- K5: gather the samples this learner sends in a step.
//
// The schedule comes from Algorithm 1 (balance.cpp:58-84) with the tail-move
// rule of equivalence.cpp:77-88: move m hands the receiver's final-list run
// [dst_off, dst_off+count) over from the sender.  The reference stops at the
// schedule; here the sender packs those samples' bytes from its
// HBM shard, in move order, into one contiguous send buffer so each move is a
// single ncclSend (loader.cu issues the grouped send/recv).  Copy-bound:
// 128-bit loads and streaming stores, one CTA per (sample, 16 KB chunk).
#include <vector>

#include "ll_internal.h"

namespace ll {
namespace {

constexpr uint32_t kChunk = 16384;

struct PackArgs {
    const uint32_t* final_step;  // final ids of the step, all learners
    uint32_t n_sends;
    uint32_t list_first[kMaxP];  // first final-list index of each send's run
    uint32_t count[kMaxP];       // samples in each send
    const uint8_t* shard;
    uint64_t shard_first;
    uint64_t sample_bytes;
    uint64_t chunks;             // per sample
    uint8_t* out;
};

__global__ void __launch_bounds__(256) k_pack(PackArgs a) {
    const uint64_t t = blockIdx.x / a.chunks;
    const uint64_t c = blockIdx.x - t * a.chunks;
    uint64_t rem = t;
    uint32_t m = 0;
    while (m + 1 < a.n_sends && rem >= a.count[m]) rem -= a.count[m++];
    const uint32_t id = a.final_step[a.list_first[m] + rem];
    const uint8_t* src = a.shard + (id - a.shard_first) * a.sample_bytes;
    uint8_t* dst = a.out + t * a.sample_bytes;
    const uint64_t b0 = c * kChunk;
    const uint64_t b1 = b0 + kChunk < a.sample_bytes ? b0 + kChunk : a.sample_bytes;
    for (uint64_t b = b0 + 16ull * threadIdx.x; b + 16 <= b1; b += 16ull * blockDim.x) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + b));
        __stcs(reinterpret_cast<uint4*>(dst + b), v);
    }
}

// Regular scheme (reg_slice, sampling.cpp:27-42) over NCCL: learner j's slice
// is batch positions [j*L, (j+1)*L) in batch order, and every sample is read
// from its owner.  The pair (slice j, owner o) exchanges regcnt[j][o] samples;
// a sample's index inside that message is its rank among the owner-o samples
// of slice j (its rank in the owner's whole-batch group, scratch[e] from K4
// pass 1, minus the owner-o samples of earlier slices).  One CTA per batch
// position: the sender copies its own samples of other slices into their
// message (pack segment j of L samples), the receiver records for each slice
// position the receive-segment index, or kLocal for its own samples.
constexpr uint32_t kLocal = 0xFFFFFFFFu;

struct RegPrepArgs {
    const uint32_t* batch;    // final ids of the step (regular: the batch itself)
    const uint32_t* scratch;  // K4 pass 1: owner << 24 | rank in the owner's batch group
    const uint32_t* regcnt;   // [p][p] of the step
    uint32_t p, me, L;
    const uint8_t* shard;
    uint64_t shard_first, sample_bytes;
    uint8_t* pack;            // [p][L] samples
    uint32_t* ridx;           // [L]: my slice position -> receive index or kLocal
};

__global__ void __launch_bounds__(256) k_reg_prep(RegPrepArgs a) {
    const uint32_t e = blockIdx.x;
    const uint32_t j = e / a.L;
    const uint32_t v = a.scratch[e];
    const uint32_t o = v >> 24;
    if (j != a.me && o != a.me) return;  // neither mine to send nor in my slice
    __shared__ uint32_t s_rank;
    if (threadIdx.x == 0) {
        uint32_t before = 0;
        for (uint32_t jj = 0; jj < j; ++jj) before += a.regcnt[jj * a.p + o];
        s_rank = (v & 0xFFFFFFu) - before;
    }
    __syncthreads();
    const uint32_t rank = s_rank;
    if (j == a.me) {
        if (threadIdx.x == 0) a.ridx[e - j * a.L] = o == a.me ? kLocal : o * a.L + rank;
        return;
    }
    // o == me, j != me: copy the sample into message (j), slot rank
    const uint32_t id = a.batch[e];
    const uint4* src = reinterpret_cast<const uint4*>(a.shard + (id - a.shard_first) * a.sample_bytes);
    uint4* dst = reinterpret_cast<uint4*>(a.pack + (static_cast<uint64_t>(j) * a.L + rank) *
                                                       a.sample_bytes);
    const uint64_t n16 = a.sample_bytes / 16;
    for (uint64_t c = threadIdx.x; c < n16; c += blockDim.x) __stcs(dst + c, __ldg(src + c));
}

} // namespace

void reg_prep_device(ll_ctx* ctx, const uint32_t* d_batch, const uint32_t* d_scratch,
                     const uint32_t* d_regcnt, uint32_t p, uint32_t me, uint64_t B,
                     const uint8_t* shard, uint64_t shard_first, uint64_t sample_bytes,
                     uint8_t* pack, uint32_t* ridx) {
    require(sample_bytes % 16 == 0, "exchange: sample bytes must be a multiple of 16");
    require(B % p == 0, "reg_slice: learner count must divide the batch size");
    RegPrepArgs a{d_batch, d_scratch, d_regcnt, p, me, static_cast<uint32_t>(B / p), shard,
                  shard_first, sample_bytes, pack, ridx};
    launch(ctx, "reg_prep", [&] {
        k_reg_prep<<<static_cast<unsigned>(B), 256, 0, ctx->stream>>>(a);
    });
}

void pack_device(ll_ctx* ctx, const std::vector<ll_xfer>& xfers, const uint32_t* d_final_step,
                 const uint8_t* shard, uint64_t shard_first, uint64_t sample_bytes,
                 uint8_t* packbuf) {
    PackArgs a{};
    uint64_t n_pack = 0;
    for (const ll_xfer& x : xfers) {
        if (!x.is_send || x.count == 0) continue;
        a.list_first[a.n_sends] = static_cast<uint32_t>(x.list_first);
        a.count[a.n_sends] = static_cast<uint32_t>(x.count);
        a.n_sends++;
        n_pack += x.count;
    }
    if (n_pack == 0) return;
    require(sample_bytes % 16 == 0, "exchange: sample bytes must be a multiple of 16");
    a.final_step = d_final_step;
    a.shard = shard;
    a.shard_first = shard_first;
    a.sample_bytes = sample_bytes;
    a.chunks = (sample_bytes + kChunk - 1) / kChunk;
    a.out = packbuf;
    launch(ctx, "pack", [&] {
        k_pack<<<static_cast<unsigned>(n_pack * a.chunks), 256, 0, ctx->stream>>>(a);
    });
}

// Host logic shared by the loader and the ll_exchange_plan entry point.
template <typename Off>
std::vector<ll_xfer> exchange_plan_t(const ll_move* moves, uint32_t n_moves, const Off* off,
                                     uint32_t me) {
    std::vector<ll_xfer> out;
    uint64_t so = 0, ro = 0;
    for (uint32_t m = 0; m < n_moves; ++m) {
        const ll_move& mv = moves[m];
        if (mv.sender == me) {
            ll_xfer x{};
            x.peer = mv.receiver;
            x.is_send = 1;
            x.count = mv.count;
            x.buf_first = so;
            x.list_first = static_cast<uint64_t>(off[mv.receiver]) + mv.dst_off;
            so += mv.count;
            out.push_back(x);
        }
        if (mv.receiver == me) {
            ll_xfer x{};
            x.peer = mv.sender;
            x.is_send = 0;
            x.count = mv.count;
            x.buf_first = ro;
            x.list_first = static_cast<uint64_t>(off[me]) + mv.dst_off;
            ro += mv.count;
            out.push_back(x);
        }
    }
    return out;
}

std::vector<ll_xfer> exchange_plan(const ll_move* moves, uint32_t n, const uint32_t* off,
                                   uint32_t me) {
    return exchange_plan_t(moves, n, off, me);
}
std::vector<ll_xfer> exchange_plan(const ll_move* moves, uint32_t n, const uint64_t* off,
                                   uint32_t me) {
    return exchange_plan_t(moves, n, off, me);
}

} // namespace ll
