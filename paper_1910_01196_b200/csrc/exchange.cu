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

} // namespace

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
