// exchange.cu -- K5: gather the samples this learner sends in a step.
//
// The schedule comes from Algorithm 1 (balance.cpp:58-84) with the tail-move
// rule of equivalence.cpp:77-88: move m hands the receiver's final-list run
// [dst_off, dst_off+count) over from the sender.  The reference stops at the
// schedule; here the sender packs those samples' bytes from its
// HBM shard, in move order, into one contiguous send buffer so each move is a
// single ncclSend (loader.cu issues the grouped send/recv).  Copy-bound:
// 128-bit loads and streaming stores, one CTA per (sample, 16 KB chunk).
#include <algorithm>
#include <vector>

#include "geometry.cuh"
#include "ll_internal.h"

namespace ll {
namespace {

constexpr uint32_t kChunk = 16384;

// One sample into a message slot: the whole sample, or (win) its crop
// window's 224 rows as the 16-byte-aligned spans K6 reads, at kWinRow pitch
// (157,696 B instead of 196,608 B on the wire).  CTA part of parts.
__device__ __forceinline__ void copy_slot(const uint8_t* src, uint8_t* dst, uint64_t sample_bytes,
                                          bool win, uint32_t crop, uint32_t row_bytes,
                                          uint32_t part, uint32_t parts) {
    if (!win) {
        const uint64_t n16 = sample_bytes / 16;
        for (uint64_t c = part * blockDim.x + threadIdx.x; c < n16;
             c += static_cast<uint64_t>(parts) * blockDim.x)
            __stcs(reinterpret_cast<uint4*>(dst) + c, __ldg(reinterpret_cast<const uint4*>(src) + c));
        return;
    }
    const uint32_t y0 = crop & 0x7FFFu, x0 = (crop >> 15) & 0xFFFFu;
    const uint32_t a0 = (3 * x0) & ~15u;
    const uint32_t nch = ((3 * x0 + 3 * kWinRows + 15u) & ~15u) / 16 - a0 / 16;
    const uint8_t* s0 = src + static_cast<uint64_t>(y0) * row_bytes + a0;
    if ((row_bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        for (uint32_t t = part * blockDim.x + threadIdx.x; t < kWinRows * nch;
             t += parts * blockDim.x) {
            const uint32_t r = t / nch, c = t - r * nch;
            __stcs(reinterpret_cast<uint4*>(dst + r * kWinRow) + c,
                   __ldg(reinterpret_cast<const uint4*>(s0 + static_cast<uint64_t>(r) * row_bytes) + c));
        }
        return;
    }
    // unaligned rows (e.g. 250-px sources): the same bytes, realigned so the
    // receiver reads every slot row from its start (K6's window-slot path)
    const uint32_t nb = 16 * nch;
    for (uint32_t t = part * blockDim.x + threadIdx.x; t < kWinRows * nb; t += parts * blockDim.x) {
        const uint32_t r = t / nb, c = t - r * nb;
        dst[r * kWinRow + c] = s0[static_cast<uint64_t>(r) * row_bytes + c];
    }
}

// One sample's resize window into a message slot (resize mode): source rows
// [y0, y0 + ch) at the sample's pitch, from byte kRecvPad of the slot, as
// 32-bit copies (word-aligned rows) or bytes.  CTA part of parts.
__device__ __forceinline__ void copy_resize_window(const uint8_t* sample, uint32_t pitch,
                                                   uint32_t y0, uint32_t ch, uint8_t* slot,
                                                   uint32_t part, uint32_t parts) {
    const uint8_t* s0 = sample + static_cast<uint64_t>(y0) * pitch;
    uint8_t* d0 = slot + kRecvPad;
    const uint64_t bytes = static_cast<uint64_t>(ch) * pitch;
    const uint64_t stride = static_cast<uint64_t>(parts) * blockDim.x;
    if ((reinterpret_cast<uintptr_t>(s0) & 3) == 0 && (pitch & 3) == 0) {
        const uint64_t nw = bytes / 4;
        for (uint64_t c = part * blockDim.x + threadIdx.x; c < nw; c += stride)
            reinterpret_cast<uint32_t*>(d0)[c] = __ldg(reinterpret_cast<const uint32_t*>(s0) + c);
    } else {
        for (uint64_t c = part * blockDim.x + threadIdx.x; c < bytes; c += stride) d0[c] = s0[c];
    }
}

// where sample `id` of this learner's shard starts, and its resize window
__device__ __forceinline__ void resize_source(const ResizeWin& rw, const uint8_t* shard,
                                              uint64_t shard_first, uint64_t sample_bytes,
                                              uint64_t id, const uint8_t** sample,
                                              uint32_t* pitch, uint32_t* y0, uint32_t* ch) {
    uint32_t H = rw.H, W = rw.W;
    if (rw.prefix) {
        var_hw(rw.data_seed, id, &H, &W);
        *sample = shard + (rw.prefix[id] - rw.prefix[shard_first]);
        *pitch = var_pitch(W);
    } else {
        *sample = shard + (id - shard_first) * sample_bytes;
        *pitch = 3 * W;
    }
    const Params q = aug_params(rw.seed, rw.epoch, id, H, W, rw.out_h, rw.out_w, LL_AUG_RESIZE);
    *y0 = q.y0;
    *ch = q.ch;
}

struct PackArgs {
    const uint32_t* final_step;  // final ids of the step, all learners
    uint32_t n_sends;
    uint32_t list_first[kMaxP];  // first final-list index of each send's run
    uint32_t count[kMaxP];       // samples in each send
    const uint8_t* shard;
    uint64_t shard_first;
    uint64_t sample_bytes;
    uint64_t chunks;
    uint8_t* out;
    const uint32_t* aug;
    uint32_t row_bytes;
    uint64_t slot_bytes;
    ResizeWin rw;
};

__global__ void __launch_bounds__(256) k_pack(PackArgs a) {
    const uint64_t t = blockIdx.x / a.chunks;
    const uint64_t c = blockIdx.x - t * a.chunks;
    uint64_t rem = t;
    uint32_t m = 0;
    while (m + 1 < a.n_sends && rem >= a.count[m]) rem -= a.count[m++];
    const uint32_t fi = a.list_first[m] + static_cast<uint32_t>(rem);
    const uint32_t id = a.final_step[fi];
    LL_DCHECK(m < a.n_sends && rem < a.count[m] && id >= a.shard_first);
    if (a.rw.enabled) {
        const uint8_t* sample;
        uint32_t pitch, y0, ch;
        resize_source(a.rw, a.shard, a.shard_first, a.sample_bytes, id, &sample, &pitch, &y0,
                      &ch);
        copy_resize_window(sample, pitch, y0, ch, a.out + t * a.slot_bytes,
                           static_cast<uint32_t>(c), static_cast<uint32_t>(a.chunks));
        return;
    }
    const uint8_t* src = a.shard + (id - a.shard_first) * a.sample_bytes;
    copy_slot(src, a.out + t * a.slot_bytes, a.sample_bytes, a.aug != nullptr,
              a.aug ? a.aug[fi] : 0u, a.row_bytes, static_cast<uint32_t>(c),
              static_cast<uint32_t>(a.chunks));
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
    uint8_t* pack;
    uint32_t* ridx;
    const uint32_t* aug;
    uint32_t row_bytes;
    uint64_t slot_bytes;
};

__global__ void __launch_bounds__(256) k_reg_prep(RegPrepArgs a) {
    const uint32_t e = blockIdx.x;
    const uint32_t j = e / a.L;
    const uint32_t v = a.scratch[e];
    const uint32_t o = v >> 24;
    if (j != a.me && o != a.me) return;  // neither mine to send nor in my slice
    __shared__ uint32_t s_rank;
    if (threadIdx.x == 0 && o < a.p) {
        uint32_t before = 0;
        for (uint32_t jj = 0; jj < j; ++jj) before += a.regcnt[jj * a.p + o];
        s_rank = (v & 0xFFFFFFu) - before;
    }
    __syncthreads();
    const uint32_t rank = s_rank;
    if (j == a.me) {
        // own samples and uncached ones (o == p: the storage tier) are not received
        if (threadIdx.x == 0) a.ridx[e - j * a.L] = o == a.me || o >= a.p ? kLocal : o * a.L + rank;
        return;
    }
    if (o >= a.p) return;  // uncached: every learner reads it from the storage tier
    // o == me, j != me: copy the sample into message (j), slot rank
    const uint32_t id = a.batch[e];
    copy_slot(a.shard + (id - a.shard_first) * a.sample_bytes,
              a.pack + (static_cast<uint64_t>(j) * a.L + rank) * a.slot_bytes, a.sample_bytes,
              a.aug != nullptr, a.aug ? a.aug[e] : 0u, a.row_bytes, 0, 1);
}

} // namespace

void reg_prep_device(ll_ctx* ctx, const uint32_t* d_batch, const uint32_t* d_scratch,
                     const uint32_t* d_regcnt, uint32_t p, uint32_t me, uint64_t B,
                     const uint8_t* shard, uint64_t shard_first, uint64_t sample_bytes,
                     uint8_t* pack, uint32_t* ridx, const uint32_t* d_aug, uint32_t row_bytes) {
    require(d_aug != nullptr || sample_bytes % 16 == 0,
            "exchange: whole-sample messages need sample bytes that are a multiple of 16");
    require(B % p == 0, "reg_slice: learner count must divide the batch size");
    RegPrepArgs a{d_batch, d_scratch, d_regcnt, p, me, static_cast<uint32_t>(B / p), shard,
                  shard_first, sample_bytes, pack, ridx, d_aug, row_bytes,
                  d_aug ? kWinBytes : sample_bytes};
    launch(ctx, "reg_prep", [&] {
        k_reg_prep<<<static_cast<unsigned>(B), 256, 0, ctx->stream>>>(a);
    });
}

uint64_t resize_slot_bytes(bool variable, uint32_t H, uint32_t W) {
    const uint64_t side = variable ? kVarMin + kVarSpan - 1 : std::min(H, W);
    const uint64_t pitch = variable ? var_pitch(kVarMin + kVarSpan - 1) : 3ull * W;
    return pad16(side * pitch) + kRecvPad + 64;  // + K7's read slack past a window row
}

void pack_device(ll_ctx* ctx, const std::vector<ll_xfer>& xfers, const uint32_t* d_final_step,
                 const uint8_t* shard, uint64_t shard_first, uint64_t sample_bytes,
                 uint8_t* packbuf, const uint32_t* d_aug, uint32_t row_bytes,
                 const ResizeWin& rw) {
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
    require(rw.enabled || d_aug != nullptr || sample_bytes % 16 == 0,
            "exchange: whole-sample messages need sample bytes that are a multiple of 16");
    a.final_step = d_final_step;
    a.shard = shard;
    a.shard_first = shard_first;
    a.sample_bytes = sample_bytes;
    a.rw = rw;
    a.slot_bytes = rw.enabled ? rw.slot : d_aug ? kWinBytes : sample_bytes;
    a.chunks = (a.slot_bytes + kChunk - 1) / kChunk;
    a.out = packbuf;
    a.aug = d_aug;
    a.row_bytes = row_bytes;
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
