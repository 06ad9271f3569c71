// loader.cu -- one learner of the locality-aware loader on one B200.
//
// Reference shape: Loader (proj/include/locload/pipeline.hpp:106-123,
// pipeline.cpp:236-336) + SampleCache (pipeline.hpp:68-94), with the
// locality-aware composition of equivalence.cpp:66-91.  What changes:
//   * the cache is this learner's CacheDirectory block (sampling.cpp:19-25)
//     held densely in HBM: sample s lives at shard + (s - first) * bytes --
//     no hash map, no lock, no shared_ptr;
//   * the epoch plan (permute_epoch + per-step assignment, schedule and tail
//     moves) is computed on the device, identically on every learner, so
//     learners agree on it without communicating (as in the reference's
//     replicated directory, sampling.hpp:11-14);
//   * per step, moved samples travel learner-to-learner (NCCL grouped
//     send/recv over NVLink, or direct peer-HBM reads inside the augment
//     kernel), then the fused augment writes the learner's NCHW batch;
//   * delivery order is stream order; prefetch_depth is the output ring.
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <cstring>
#include <vector>

#include "geometry.cuh"
#include "ll_internal.h"

namespace ll {
void widen_device(ll_ctx* ctx, const uint32_t* in, uint64_t* out, uint64_t n);
}

#define LL_NCCL(x)                                                                        \
    do {                                                                                  \
        ncclResult_t r_ = (x);                                                            \
        if (r_ != ncclSuccess)                                                            \
            ::ll::fail(LL_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_));     \
    } while (0)

struct ll_loader {
    ll_ctx* ctx = nullptr;
    // names this loader's context scratch that its own streams (plan, side)
    // write: loaders on one device share the context
    std::string tag;
    ll_loader_config cfg{};
    uint64_t S = 0;               // sample bytes
    uint64_t cached = 0;          // CacheDirectory::cached_count
    uint64_t first = 0, owned = 0;
    uint64_t steps = 0;           // per epoch
    uint64_t max_local = 0;
    ll::DevBuf shard;
    bool populated = false;
    ll::DevBuf prefix;            // variable geometry: global padded-size prefix [d+1]
    uint8_t* storage = nullptr;   // alpha < 1: pinned+mapped host copy of ids [cached, d)
    std::vector<uint64_t> h_prefix_ends;  // prefix at first and first+owned
    // epoch plans: two slots, the current epoch's and the next one being
    // prefetched on plan_stream (host tables in pinned memory)
    struct PlanSlot {
        ll::DevBuf order;
        ll::PlanBufs plan;
        int64_t epoch = -1;          // epoch held (or being computed)
        cudaEvent_t ready = nullptr; // tables landed in host memory
        ll_move* moves = nullptr;    // pinned host tables
        uint32_t *off = nullptr, *kept = nullptr, *counts = nullptr, *nmoves = nullptr,
                 *stats = nullptr;
        uint32_t* regcnt = nullptr;  // regular + NCCL: [steps][p][p]
    } slot[2];
    int cur = 0;
    cudaStream_t plan_stream = nullptr;
    int64_t plan_epoch = -1;
    ll::PlanBufs& plan() { return slot[cur].plan; }
    // current epoch's host tables
    ll_move* h_moves = nullptr;
    uint32_t* h_regcnt = nullptr;  // regular + NCCL: [steps][p][p]
    uint32_t *h_off = nullptr, *h_kept = nullptr, *h_counts = nullptr, *h_nmoves = nullptr,
             *h_stats = nullptr;
    // exchange
    ncclComm_t comm = nullptr;
    // one step's exchange buffers: send messages, receive buffer and, for the
    // regular scheme, the slice-position -> receive-index map
    struct ExSet {
        ll::DevBuf pack, recv, ridx;
    };
    // NCCL exchange of step t+1 issued on the side stream while step t's
    // augment runs (two buffer sets, alternating by step parity)
    ExSet xset[2];
    // exchange buffers from ncclMemAlloc, registered with the communicator
    // (user-buffer registration: NVLink send/recv may copy between them
    // directly instead of through NCCL's staging FIFO); freed after the
    // communicator lets go of them
    std::vector<std::pair<void*, void*>> nccl_mem;  // {ptr, registration handle}
    cudaEvent_t xdone[2] = {nullptr, nullptr}, augdone[2] = {nullptr, nullptr};
    // the pack kernel of a set runs on its own stream, so step t+1's pack
    // overlaps step t's grouped send/recv on the side stream
    cudaStream_t pack_stream = nullptr;
    cudaEvent_t packdone[2] = {nullptr, nullptr};
    // the grouped send/recv of every step, on a stream of its own so a
    // host-driven step's prologue (side stream) never queues behind them
    cudaStream_t wire_stream = nullptr;
    struct Pending {
        bool valid = false;
        uint64_t epoch = 0, step = 0;
    } xpending[2];
    // resize prologue (K7 prep + far pull) of step t+1 issued on the side
    // stream while step t's augment runs (buffer sets 0/1 by step parity)
    cudaEvent_t rready[2] = {nullptr, nullptr}, rdone[2] = {nullptr, nullptr};
    Pending rpending[2];
    std::vector<void*> peer_open;  // opened IPC mappings (excluding self)
    ll::DevBuf d_peers;
    bool peers_ready = false;
    // output ring
    std::vector<std::unique_ptr<ll::DevBuf>> out;
    uint32_t out_slot = 0;
    // host-driven steps in flight (ll_loader_submit_host / wait_host), at most
    // prefetch_depth outstanding, delivered in submission order
    struct Tables {  // one step's plan tables as delivered to the host
        ll_move moves[ll::kMaxP];
        uint32_t off[ll::kMaxP + 1], kept[ll::kMaxP], n, stats[4];
    };
    struct HostSlot {
        uint64_t* pin = nullptr;         // pinned: [Tables][B x u64 local ids]
        uint64_t* pin_batch = nullptr;   // pinned copy of the caller's GlobalBatch
        ll::DevBuf batch64, order, stage;  // device: batch, narrowed batch, staging
        ll::PlanBufs plan;               // this step's single-step plan
        cudaEvent_t pro_done = nullptr;  // prologue (H2D + assign) finished (side stream)
        cudaEvent_t done = nullptr;      // whole step finished (main stream)
        bool used = false;
        ll_step_info info{};
        uint64_t n_local = 0;
        bool synchronous = false;
        std::string rtag;                // owner name of this slot's K7 prologue set
        int rslot = -1;                  // K7 prologue prepared into (rtag, 0), or -1
        uint32_t* pin_rc = nullptr;      // regular + NCCL: the step's [slice][owner] counts
                                         // (pinned: the D2H is queued behind the
                                         // side stream's work, never a blocking copy)
        Tables* tab() const { return reinterpret_cast<Tables*>(pin); }
        uint64_t* ids() const { return pin + sizeof(Tables) / 8; }
    };
    std::vector<std::unique_ptr<HostSlot>> hslots;
    uint64_t submitted = 0, waited = 0;
    cudaStream_t side = nullptr;     // prologue stream of host-driven steps
    // NCCL exchange accounting: bytes every step; with the context's timing
    // on, events around each step's pack and wire phase on its stream
    struct XTimes {
        cudaEvent_t t0, t1, t2, t3;  // pack start / end (pack stream), wire start / end
        uint64_t recvd;
    };
    std::vector<XTimes> xtimes;
    uint64_t x_steps = 0, x_sent = 0, x_recv = 0, x_timed = 0, x_timed_recv = 0;
    double x_ms_pack = 0, x_ms_wire = 0;
};

namespace ll {
namespace {

uint64_t out_elem_bytes(const ll_loader_config& c) {
    return c.augment.out_dtype == LL_OUT_BF16 ? 2 : 4;
}

// Queue the D2H of slot `k`'s step tables on `stream` (pinned destination) and
// mark the slot's ready event.
// the regular scheme's full-volume exchange over NCCL
bool reg_nccl(const ll_loader_config& c) {
    return c.learners > 1 && c.scheme == LL_SCHEME_REGULAR && c.exchange == LL_EXCHANGE_NCCL;
}

void copy_tables(ll_loader* ld, int k, cudaStream_t stream) {
    auto& sl = ld->slot[k];
    const uint64_t steps = ld->steps;
    const PlanBufs& plan = sl.plan;
    auto d2h = [&](void* dst, const DevBuf& b, size_t n) {
        LL_CUDA(cudaMemcpyAsync(dst, b.ptr, n, cudaMemcpyDeviceToHost, stream));
    };
    d2h(sl.moves, plan.moves, sizeof(ll_move) * steps * kMaxP);
    d2h(sl.off, plan.off, sizeof(uint32_t) * steps * (kMaxP + 1));
    d2h(sl.kept, plan.kept, sizeof(uint32_t) * steps * kMaxP);
    d2h(sl.counts, plan.counts, sizeof(uint32_t) * steps * kMaxP);
    d2h(sl.nmoves, plan.n_moves, sizeof(uint32_t) * steps);
    d2h(sl.stats, plan.stats, sizeof(uint32_t) * steps * 4);
    if (sl.regcnt) {
        const uint64_t p = ld->cfg.learners;
        d2h(sl.regcnt, plan.regcnt, sizeof(uint32_t) * steps * p * p);
    }
    LL_CUDA(cudaEventRecord(sl.ready, stream));
}

AugPlan aug_plan(const ll_loader* ld, uint64_t epoch);

// Compute epoch `epoch`'s plan into slot k on `stream`: permutation (scratch
// tagged per slot, so a prefetch and an API call never share buffers),
// assignment, host tables.
void plan_into(ll_loader* ld, int k, uint64_t epoch, cudaStream_t stream) {
    ll_ctx* ctx = ld->ctx;
    const ll_loader_config& c = ld->cfg;
    auto& sl = ld->slot[k];
    const std::string tag = ld->tag + (k ? "plan1" : "plan0");
    cudaStream_t main = ctx->stream;
    ctx->stream = stream;  // the device helpers launch on the context stream
    try {
        permute_device(ctx, c.seed, epoch, static_cast<uint32_t>(c.d), sl.order.as<uint32_t>(),
                       nullptr, 0, tag.c_str());
        assign_device(ctx, sl.order.as<uint32_t>(), ld->steps, c.batch_size, c.learners,
                      ld->cached, c.scheme, sl.plan.view(), aug_plan(ld, epoch));
        copy_tables(ld, k, stream);
    } catch (...) {
        ctx->stream = main;
        throw;
    }
    ctx->stream = main;
    sl.epoch = static_cast<int64_t>(epoch);
}

AugPlan aug_plan(const ll_loader* ld, uint64_t epoch) {
    AugPlan g;
    const ll_loader_config& c = ld->cfg;
    if (c.augment.mode != LL_AUG_CROP) return g;
    g.enabled = true;
    g.seed = c.seed;
    g.epoch = epoch;
    g.H = c.height;
    g.W = c.width;
    g.ch = c.augment.out_h;
    g.cw = c.augment.out_w;
    return g;
}

void ensure_out(ll_loader* ld) {
    if (!ld->out.empty()) return;
    const ll_loader_config& c = ld->cfg;
    const uint64_t bytes =
        ld->max_local * 3ull * c.augment.out_h * c.augment.out_w * out_elem_bytes(c);
    for (uint32_t f = 0; f < std::max<uint32_t>(1, c.prefetch_depth); ++f) {
        ld->out.emplace_back(new DevBuf());
        ld->out.back()->reserve(bytes ? bytes : 16);
    }
}

// One step's exchange on `stream`, NCCL grouped send/recv.
//  * balanced / locality schemes: K5 packs the tail moves this learner sends
//    (Algorithm 1 + equivalence.cpp:77-88); received samples land in x.recv
//    in the learner's final-list order;
//  * regular scheme (reg_slice, sampling.cpp:27-42): every learner exchanges
//    with every other its owned samples of their slices (h_regcnt: this
//    step's [slice][owner] counts); x.ridx maps slice positions to x.recv.
// Brackets one step's exchange: the pack kernel on the pack stream (t0 -> t1)
// and the NCCL grouped send/recv on the wire stream (t2 -> t3, from the point
// the wire stream has the packed set), while the context's timing is on.
struct ExchangeTimer {
    ll_loader* ld;
    cudaStream_t pstream, wstream;
    ll_loader::XTimes t{nullptr, nullptr, nullptr, nullptr, 0};
    ExchangeTimer(ll_loader* l, cudaStream_t ps, cudaStream_t ws) : ld(l), pstream(ps), wstream(ws) {
        if (!ld->ctx->timing) return;
        t.t0 = ld->ctx->take_event();
        LL_CUDA(cudaEventRecord(t.t0, pstream));
    }
    void packed() {
        if (!t.t0) return;
        t.t1 = ld->ctx->take_event();
        LL_CUDA(cudaEventRecord(t.t1, pstream));
    }
    void wire_start() {
        if (!t.t0) return;
        t.t2 = ld->ctx->take_event();
        LL_CUDA(cudaEventRecord(t.t2, wstream));
    }
    void done(uint64_t sent, uint64_t recvd) {
        ++ld->x_steps;
        ld->x_sent += sent;
        ld->x_recv += recvd;
        if (!t.t0) return;
        t.t3 = ld->ctx->take_event();
        LL_CUDA(cudaEventRecord(t.t3, wstream));
        t.recvd = recvd;
        ld->xtimes.push_back(t);
        t = ll_loader::XTimes{nullptr, nullptr, nullptr, nullptr, 0};  // owned by xtimes now
    }
    ~ExchangeTimer() {  // an exception before done(): hand the events back
        for (cudaEvent_t e : {t.t0, t.t1, t.t2, t.t3})
            if (e) ld->ctx->event_pool.push_back(e);
    }
};

// Bytes per NCCL message slot: a crop window (crop mode) or the largest
// resize window (resize mode, rows at the sample's pitch after kRecvPad).
uint64_t msg_slot(const ll_loader* ld) {
    const ll_loader_config& c = ld->cfg;
    if (c.augment.mode == LL_AUG_CROP) return kWinBytes;
    return resize_slot_bytes(c.geometry == LL_GEOM_VARIABLE, c.height, c.width);
}

void ensure_pack_stream(ll_loader* ld) {
    if (ld->pack_stream) return;
    int lo = 0, hi = 0;
    LL_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    LL_CUDA(cudaStreamCreateWithPriority(&ld->pack_stream, cudaStreamNonBlocking, hi));
    for (int i = 0; i < 2; ++i)
        LL_CUDA(cudaEventCreateWithFlags(&ld->packdone[i], cudaEventDisableTiming));
}

cudaStream_t wire_stream(ll_loader* ld) {
    if (!ld->wire_stream) {
        int lo = 0, hi = 0;
        LL_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        LL_CUDA(cudaStreamCreateWithPriority(&ld->wire_stream, cudaStreamNonBlocking, hi));
    }
    return ld->wire_stream;
}

// Exchange set `set` (xset[set]) for one step: the pack kernel on the pack
// stream once the set is free again (its previous grouped send/recv,
// xdone[set], and the augment that read it, augdone[set], are done), then the
// grouped send/recv on `stream` after the pack.  So the pack of step t+1
// overlaps the send/recv of step t.
void issue_exchange(ll_loader* ld, const PlanDev& pd, uint64_t epoch, uint64_t step,
                    const ll_move* h_moves, uint32_t h_nmoves, const uint32_t* h_off,
                    const uint32_t* h_regcnt, int set, cudaStream_t stream,
                    cudaEvent_t plan_ready = nullptr) {
    ll_loader::ExSet& x = ld->xset[set];
    ensure_pack_stream(ld);
    cudaStream_t ps = ld->pack_stream;
    if (plan_ready) LL_CUDA(cudaStreamWaitEvent(ps, plan_ready, 0));  // host-driven step's plan
    if (ld->xdone[set]) LL_CUDA(cudaStreamWaitEvent(ps, ld->xdone[set], 0));
    if (ld->augdone[set]) LL_CUDA(cudaStreamWaitEvent(ps, ld->augdone[set], 0));
    ll_ctx* ctx = ld->ctx;
    const ll_loader_config& c = ld->cfg;
    const uint32_t me = c.rank, p = c.learners;
    const uint64_t B = c.batch_size;
    require(ld->comm != nullptr, "loader: NCCL exchange needs ll_loader_comm_init");
    const uint32_t* d_final_step = pd.final_ids + step * B;
    cudaStream_t main = ctx->stream;
    // crop mode: messages carry crop windows (K6 reads nothing else of a
    // sample); resize mode: resize windows (K7 reads nothing else)
    const bool crop = c.augment.mode == LL_AUG_CROP;
    const uint64_t slot = msg_slot(ld);
    const uint32_t* d_aug = crop ? pd.aug + step * B : nullptr;
    const uint32_t row_bytes = 3 * c.width;
    ExchangeTimer tm(ld, ps, stream);
    // after the pack: the wire stream picks the set up
    auto handoff = [&] {
        tm.packed();
        LL_CUDA(cudaEventRecord(ld->packdone[set], ps));
        LL_CUDA(cudaStreamWaitEvent(stream, ld->packdone[set], 0));
        tm.wire_start();
    };
    if (c.scheme == LL_SCHEME_REGULAR) {
        require(crop, "loader: the regular scheme over NCCL needs crop mode (resize windows of "
                      "a full slice exchange go over the P2P exchange)");
        require(h_regcnt != nullptr && pd.regcnt != nullptr, "loader: regular plan lacks counts");
        const uint64_t L = B / p;
        x.pack.need(B * slot, "exchange send buffer");
        x.recv.need(B * slot, "exchange receive buffer");
        x.ridx.need(sizeof(uint32_t) * std::max<uint64_t>(L, 1), "exchange receive map");
        ctx->stream = ps;
        try {
            reg_prep_device(ctx, d_final_step, pd.scratch + step * B, pd.regcnt + step * p * p, p,
                            me, B, ld->shard.as<uint8_t>(), ld->first, ld->S,
                            x.pack.as<uint8_t>(), x.ridx.as<uint32_t>(), d_aug, row_bytes);
        } catch (...) {
            ctx->stream = main;
            throw;
        }
        ctx->stream = main;
        handoff();
        uint64_t sent = 0, recvd = 0;
        LL_NCCL(ncclGroupStart());
        for (uint32_t r = 0; r < p; ++r) {
            if (r == me) continue;
            const uint64_t ns = h_regcnt[r * p + me], nr = h_regcnt[me * p + r];
            if (ns)
                LL_NCCL(ncclSend(x.pack.as<uint8_t>() + r * L * slot, ns * slot, ncclUint8,
                                 static_cast<int>(r), ld->comm, stream));
            if (nr)
                LL_NCCL(ncclRecv(x.recv.as<uint8_t>() + r * L * slot, nr * slot, ncclUint8,
                                 static_cast<int>(r), ld->comm, stream));
            sent += ns * slot;
            recvd += nr * slot;
        }
        LL_NCCL(ncclGroupEnd());
        tm.done(sent, recvd);
        return;
    }
    // balanced / locality schemes: one message per tail move involving me
    // (equivalence.cpp:77-88).  A run hands the sender's cached samples over
    // first and its uncached ones (storage tier, alpha < 1) last, so only the
    // run's first `nvlink` samples cross the wire; the receive slots stay
    // indexed by whole runs (slot = final-list position - kept), and K6 / K7
    // read uncached samples from the storage tier.
    std::vector<ll_xfer> xs;
    uint64_t so = 0, ro = 0;
    for (uint32_t m = 0; m < h_nmoves; ++m) {
        const ll_move& mv = h_moves[m];
        if (mv.sender == me) {
            xs.push_back(ll_xfer{mv.receiver, 1, mv.nvlink, so,
                                 static_cast<uint64_t>(h_off[mv.receiver]) + mv.dst_off});
            so += mv.nvlink;
        }
        if (mv.receiver == me) {
            xs.push_back(ll_xfer{mv.sender, 0, mv.nvlink, ro,
                                 static_cast<uint64_t>(h_off[me]) + mv.dst_off});
            ro += mv.count;
        }
    }
    x.pack.need(so * slot, "exchange send buffer");
    x.recv.need(ro * slot, "exchange receive buffer");
    ResizeWin rw;
    if (!crop) {
        rw.enabled = true;
        rw.seed = c.seed;
        rw.epoch = epoch;
        rw.data_seed = c.data_seed;
        rw.prefix = c.geometry == LL_GEOM_VARIABLE ? ld->prefix.as<uint64_t>() : nullptr;
        rw.H = c.height;
        rw.W = c.width;
        rw.out_h = c.augment.out_h;
        rw.out_w = c.augment.out_w;
        rw.slot = slot;
    }
    ctx->stream = ps;  // pack_device launches on the context stream
    try {
        pack_device(ctx, xs, d_final_step, ld->shard.as<uint8_t>(), ld->first, ld->S,
                    x.pack.as<uint8_t>(), d_aug, row_bytes, rw);
    } catch (...) {
        ctx->stream = main;
        throw;
    }
    ctx->stream = main;
    handoff();
    uint64_t sent = 0, recvd = 0;
    LL_NCCL(ncclGroupStart());
    for (const ll_xfer& xf : xs) {
        if (xf.count == 0) continue;
        if (xf.is_send) {
            LL_NCCL(ncclSend(x.pack.as<uint8_t>() + xf.buf_first * slot, xf.count * slot,
                             ncclUint8, static_cast<int>(xf.peer), ld->comm, stream));
            sent += xf.count * slot;
        } else {
            LL_NCCL(ncclRecv(x.recv.as<uint8_t>() + xf.buf_first * slot, xf.count * slot,
                             ncclUint8, static_cast<int>(xf.peer), ld->comm, stream));
            recvd += xf.count * slot;
        }
    }
    LL_NCCL(ncclGroupEnd());
    tm.done(sent, recvd);
}

// Where this learner's samples of `step` come from (own shard, storage tier,
// peer shards), for every exchange but NCCL (run_step adds the receive buffer).
struct StepSrc {
    SrcMap src;
    uint64_t n_local = 0, n_send = 0, n_recv = 0, nvl_recv = 0;
};

StepSrc step_src(ll_loader* ld, const PlanDev& pd, uint64_t step, const ll_move* h_moves,
                 const uint32_t* h_off, const uint32_t* h_kept, uint32_t h_nmoves) {
    const ll_loader_config& c = ld->cfg;
    const uint32_t me = c.rank, p = c.learners;
    const uint64_t B = c.batch_size;
    const uint32_t* d_final_step = pd.final_ids + step * B;
    StepSrc r;
    r.n_local = h_off[me + 1] - h_off[me];
    const uint64_t kept = h_kept[me];
    for (uint32_t m = 0; m < h_nmoves; ++m) {
        if (h_moves[m].sender == me) r.n_send += h_moves[m].count;
        if (h_moves[m].receiver == me) {
            r.n_recv += h_moves[m].count;
            r.nvl_recv += h_moves[m].nvlink;
        }
    }
    SrcMap& src = r.src;
    src.kind = 1;
    src.list = d_final_step + h_off[me];
    src.kept = static_cast<uint32_t>(kept);
    src.shard = ld->shard.as<uint8_t>();
    src.shard_end = ld->shard.as<uint8_t>() + ld->shard.bytes;
    src.storage_end = ld->storage ? ld->storage + (ld->cfg.d - ld->cached) * ld->S + 64 : nullptr;
    src.shard_first = ld->first;
    src.p = p;
    src.cached = ld->cached;
    src.sample_bytes = ld->S;
    src.storage = ld->storage;
    if (c.geometry == LL_GEOM_VARIABLE) {
        src.prefix = ld->prefix.as<uint64_t>();
        src.data_seed = c.data_seed;
    }
    if (c.augment.mode == LL_AUG_CROP) src.aug = pd.aug + step * B + h_off[me];
    if (p > 1 && c.scheme == LL_SCHEME_REGULAR) {
        // reg_slice (sampling.cpp:27-42) ignores ownership: every sample of the
        // slice is read from its owner's shard (the owner may be this learner),
        // over P2P, or received over NCCL (run_step adds the receive buffer)
        require((c.exchange == LL_EXCHANGE_P2P && ld->peers_ready) ||
                    c.exchange == LL_EXCHANGE_NCCL,
                "loader: the regular scheme needs an exchange (P2P peer shards or NCCL)");
        src.kept = 0;
        if (c.exchange == LL_EXCHANGE_P2P) src.peers = ld->d_peers.as<const uint8_t*>();
        r.n_recv = r.n_local;
    } else if (p > 1 && (r.n_send || r.n_recv)) {
        if (c.exchange == LL_EXCHANGE_P2P) {
            require(ld->peers_ready, "loader: P2P exchange needs peer shards (open/link)");
            src.peers = ld->d_peers.as<const uint8_t*>();
        } else if (c.exchange != LL_EXCHANGE_NCCL) {
            fail(LL_ERR_INVALID, "loader: remote samples need an exchange (NCCL or P2P)");
        }
    }
    return r;
}

uint32_t geom_h(const ll_loader_config& c) {
    return c.geometry == LL_GEOM_VARIABLE ? kVarMin + kVarSpan - 1 : c.height;
}
uint32_t geom_w(const ll_loader_config& c) {
    return c.geometry == LL_GEOM_VARIABLE ? kVarMin + kVarSpan - 1 : c.width;
}

// prepared_slot >= 0: the resize prologue of this step is in that buffer set
void run_step(ll_loader* ld, uint64_t epoch, const PlanDev& pd, uint64_t step,
              const ll_move* h_moves, const uint32_t* h_off, const uint32_t* h_kept,
              uint32_t h_nmoves, const uint32_t* h_stats, ll_step_info* info,
              const ll_loader::ExSet* prefetched = nullptr, int prepared_slot = -1,
              const uint32_t* h_regcnt = nullptr, const std::string* owner = nullptr) {
    ll_ctx* ctx = ld->ctx;
    const ll_loader_config& c = ld->cfg;
    const uint32_t me = c.rank, p = c.learners;
    const uint64_t B = c.batch_size;
    const uint32_t* d_final_step = pd.final_ids + step * B;
    StepSrc ss = step_src(ld, pd, step, h_moves, h_off, h_kept, h_nmoves);
    SrcMap& src = ss.src;
    const uint64_t n_local = ss.n_local;
    uint64_t n_recv = ss.n_recv, nvl_recv = ss.nvl_recv;
    const bool reg = p > 1 && c.scheme == LL_SCHEME_REGULAR;
    if (p > 1 && c.exchange == LL_EXCHANGE_NCCL && (reg || ss.n_send || ss.n_recv)) {
        const ll_loader::ExSet* x = prefetched;
        require(x != nullptr, "loader: NCCL step without an issued exchange");
        src.recv = x->recv.as<uint8_t>();
        if (c.augment.mode == LL_AUG_CROP)
            src.recv_row = kWinRow;  // crop-window slots
        else
            src.recv_slot = msg_slot(ld);  // resize-window slots
        if (reg) {
            src.recv_idx = x->ridx.as<uint32_t>();
            n_recv = nvl_recv = 0;  // this slice's samples owned by the others
            for (uint32_t o = 0; o < p; ++o)
                if (o != me) n_recv += h_regcnt[me * p + o];
            nvl_recv = n_recv;
        }
    }
    ensure_out(ld);
    void* out = ld->out[ld->out_slot]->ptr;
    ld->out_slot = (ld->out_slot + 1) % ld->out.size();
    augment_device(ctx, c.augment, c.seed, epoch, src, n_local, geom_h(c), geom_w(c), out,
                   prepared_slot, owner ? *owner : ld->tag);
    if (info) {
        info->epoch = epoch;
        info->step = step;
        info->n_local = n_local;
        info->kept = src.kept;
        info->received = n_recv;
        info->moved_total = h_stats[0];
        // bytes that crossed NVLink into this learner: NCCL message slots, or
        // (P2P, crop mode) the crop windows K6 read from peer shards
        uint64_t per = ld->S;
        if (p > 1 && c.exchange == LL_EXCHANGE_NCCL)
            per = msg_slot(ld);
        else if (c.augment.mode == LL_AUG_CROP)
            per = 3ull * c.augment.out_h * c.augment.out_w;
        // regular scheme over P2P: the box's remote samples of the step
        // (K4's count) spread over the learners -- no per-learner count exists
        if (reg && c.exchange == LL_EXCHANGE_P2P && h_stats[3] != 0xFFFFFFFFu)
            nvl_recv = h_stats[3] / p;
        info->nvlink_bytes = nvl_recv * per;
        info->uncached = h_stats[2];
        info->reg_remote = h_stats[3] == 0xFFFFFFFFu ? UINT64_MAX : h_stats[3];
        info->device_out = reinterpret_cast<uintptr_t>(out);
        info->device_ids = reinterpret_cast<uintptr_t>(d_final_step + h_off[me]);
    }
}

// A step whose plan tables stay on the device (host-driven path): the list
// offset and kept count are read by the kernel, n_local is the balanced
// target (or the regular slice), so no mid-step host sync is needed.
SrcMap devplan_src(ll_loader* ld, const PlanDev& pd) {
    const ll_loader_config& c = ld->cfg;
    const uint32_t me = c.rank, p = c.learners;
    SrcMap src;
    src.kind = 1;
    src.list = pd.final_ids;
    src.list_off = pd.off + me;
    src.kept_dev = pd.kept + me;
    src.shard = ld->shard.as<uint8_t>();
    src.shard_end = ld->shard.as<uint8_t>() + ld->shard.bytes;
    src.storage_end = ld->storage ? ld->storage + (ld->cfg.d - ld->cached) * ld->S + 64 : nullptr;
    src.shard_first = ld->first;
    src.p = p;
    src.cached = ld->cached;
    src.sample_bytes = ld->S;
    src.storage = ld->storage;
    if (c.geometry == LL_GEOM_VARIABLE) {
        src.prefix = ld->prefix.as<uint64_t>();
        src.data_seed = c.data_seed;
    }
    if (c.augment.mode == LL_AUG_CROP) src.aug = pd.aug;
    if (p > 1) {
        require(ld->peers_ready, "loader: P2P exchange needs peer shards (open/link)");
        src.peers = ld->d_peers.as<const uint8_t*>();
        if (c.scheme == LL_SCHEME_REGULAR) {
            src.kept_dev = nullptr;
            src.kept = 0;
        }
    }
    return src;
}

// prepared_slot >= 0: the resize prologue ran into set (owner, prepared_slot)
void* run_step_devplan(ll_loader* ld, uint64_t epoch, const PlanDev& pd, uint64_t n_local,
                       int prepared_slot = -1, const std::string& owner = std::string()) {
    ll_ctx* ctx = ld->ctx;
    const ll_loader_config& c = ld->cfg;
    const SrcMap src = devplan_src(ld, pd);
    ensure_out(ld);
    void* out = ld->out[ld->out_slot]->ptr;
    ld->out_slot = (ld->out_slot + 1) % ld->out.size();
    augment_device(ctx, c.augment, c.seed, epoch, src, n_local, geom_h(c), geom_w(c), out,
                   prepared_slot, owner);
    return out;
}

// Stage one host-driven step's results for a single D2H copy:
// [Tables][n_local x u64 ids].
__global__ void k_stage(PlanDev pd, uint32_t me, uint32_t p, uint8_t* __restrict__ stage,
                        uint64_t n) {
    auto* t = reinterpret_cast<ll_loader::Tables*>(stage);
    uint64_t* ids = reinterpret_cast<uint64_t*>(stage + sizeof(ll_loader::Tables));
    const uint32_t base = pd.off[me];
    const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    for (uint64_t i = tid; i < n; i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        ids[i] = pd.final_ids[base + i];
    if (blockIdx.x == 0) {
        const uint32_t nm = *pd.n_moves;
        for (uint32_t j = threadIdx.x; j < kMaxP; j += blockDim.x) {
            if (j < nm) t->moves[j] = pd.moves[j];
            if (j < p) {
                t->kept[j] = pd.kept[j];
            }
        }
        for (uint32_t j = threadIdx.x; j <= p; j += blockDim.x) t->off[j] = pd.off[j];
        if (threadIdx.x < 4) t->stats[threadIdx.x] = pd.stats[threadIdx.x];
        if (threadIdx.x == 0) t->n = nm;
    }
}

} // namespace

void loader_create(ll_loader** out, ll_ctx* ctx, const ll_loader_config* cfg) {
    require(cfg != nullptr, "Loader: null config");
    const ll_loader_config& c = *cfg;
    // pipeline.cpp:237-241
    require(c.batch_size >= 1 && c.prefetch_depth >= 1,
            "Loader: workers, parallelism, prefetch and batch size must all be >= 1");
    require(c.learners >= 1, "CacheDirectory: learner count must be >= 1");
    require(c.alpha > 0.0 && c.alpha <= 1.0, "CacheDirectory: cached fraction must be in (0, 1]");
    require(c.d >= 1, "permute_epoch: dataset must contain at least one sample");
    require(c.batch_size <= c.d, "batches: batch size must be in [1, dataset size]");
    require(c.learners <= kMaxP, "Loader: at most 64 learners per box");
    require(c.rank < c.learners, "Loader: rank out of range");
    require(c.d < 0xFFFFFFFFull, "Loader: dataset size must be < 2^32 - 1 on the device");
    require(c.geometry == LL_GEOM_VARIABLE || (c.height >= 1 && c.width >= 1),
            "Loader: empty sample geometry");
    require(c.scheme >= LL_SCHEME_REGULAR && c.scheme <= LL_SCHEME_LOCALITY_BALANCED,
            "Loader: unknown scheme");
    if (c.scheme == LL_SCHEME_REGULAR)
        require(c.batch_size % c.learners == 0,
                "reg_slice: learner count must divide the batch size");
    auto ld = std::make_unique<ll_loader>();
    static std::atomic<uint64_t> serial{0};
    ld->tag = "ld" + std::to_string(serial++) + ".";
    ld->ctx = ctx;
    ld->cfg = c;
    require(c.geometry == LL_GEOM_FIXED || c.geometry == LL_GEOM_VARIABLE,
            "Loader: unknown geometry");
    if (c.geometry == LL_GEOM_VARIABLE)
        require(c.augment.mode == LL_AUG_RESIZE,
                "Loader: variable-size samples need augment.mode = LL_AUG_RESIZE");
    ld->S = c.geometry == LL_GEOM_FIXED ? static_cast<uint64_t>(c.height) * c.width * 3 : 0;
    ld->cached = static_cast<uint64_t>(c.alpha * static_cast<double>(c.d));  // sampling.cpp:15
    if (ld->cached > c.d) ld->cached = c.d;
    require(ld->cached >= 1, "Loader: alpha * d must cache at least one sample");
    if (ld->cached < c.d) {
        require(c.geometry == LL_GEOM_FIXED,
                "Loader: the storage tier (alpha < 1) supports fixed-size samples");
        require(c.learners == 1 || c.exchange != LL_EXCHANGE_NONE,
                "Loader: the storage tier (alpha < 1) with several learners needs an exchange");
    }
    const uint64_t p = c.learners, j = c.rank;
    ld->first = (j * ld->cached + p - 1) / p;
    ld->owned = ((j + 1) * ld->cached + p - 1) / p - ld->first;
    ld->steps = c.d / c.batch_size;
    ld->max_local = c.scheme == LL_SCHEME_LOCALITY ? c.batch_size
                                                   : (c.batch_size + p - 1) / p;
    set_device(ctx);
    uint64_t shard_bytes = ld->owned * ld->S;
    if (c.geometry == LL_GEOM_VARIABLE) {
        // every learner computes the same global prefix of padded sample sizes
        ld->prefix.reserve(sizeof(uint64_t) * (c.d + 1));
        var_prefix_device(ctx, ld->prefix.as<uint64_t>(), c.d, c.data_seed);
        uint64_t ends[2];
        LL_CUDA(cudaMemcpyAsync(&ends[0], ld->prefix.as<uint64_t>() + ld->first, 8,
                                cudaMemcpyDeviceToHost, ctx->stream));
        LL_CUDA(cudaMemcpyAsync(&ends[1], ld->prefix.as<uint64_t>() + ld->first + ld->owned, 8,
                                cudaMemcpyDeviceToHost, ctx->stream));
        LL_CUDA(cudaStreamSynchronize(ctx->stream));
        ld->h_prefix_ends.assign(ends, ends + 2);
        shard_bytes = ends[1] - ends[0];
    }
    // + 64: K7 reads up to 27 bytes past a crop row (word-aligned taps, TMA spans)
    ld->shard.reserve(std::max<uint64_t>(shard_bytes, 16) + 64);
    for (auto& sl : ld->slot) {
        sl.order.reserve(sizeof(uint32_t) * c.d);
        sl.plan.reserve(ld->steps, c.batch_size);
        const uint64_t st = std::max<uint64_t>(ld->steps, 1);
        LL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&sl.moves), sizeof(ll_move) * st * kMaxP, 0));
        LL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&sl.off), sizeof(uint32_t) * st * (kMaxP + 1), 0));
        LL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&sl.kept), sizeof(uint32_t) * st * kMaxP, 0));
        LL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&sl.counts), sizeof(uint32_t) * st * kMaxP, 0));
        LL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&sl.nmoves), sizeof(uint32_t) * st, 0));
        LL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&sl.stats), sizeof(uint32_t) * st * 4, 0));
        if (reg_nccl(c)) {
            sl.plan.reserve_regcnt(st, c.learners);
            LL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&sl.regcnt),
                                  sizeof(uint32_t) * st * c.learners * c.learners, 0));
        }
        LL_CUDA(cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
    }
    *out = ld.release();
}

void loader_destroy(ll_loader* ld) {
    if (!ld) return;
    cudaSetDevice(ld->ctx->device);
    for (void* p : ld->peer_open) cudaIpcCloseMemHandle(p);
    for (auto& hp : ld->hslots) {
        auto& h = *hp;
        if (h.pin) cudaFreeHost(h.pin);
        if (h.pin_batch) cudaFreeHost(h.pin_batch);
        if (h.pin_rc) cudaFreeHost(h.pin_rc);
        if (h.pro_done) cudaEventDestroy(h.pro_done);
        if (h.done) cudaEventDestroy(h.done);
    }
    if (ld->side) cudaStreamDestroy(ld->side);
    if (ld->pack_stream) cudaStreamDestroy(ld->pack_stream);
    if (ld->wire_stream) cudaStreamDestroy(ld->wire_stream);
    for (int i = 0; i < 2; ++i) {
        if (ld->packdone[i]) cudaEventDestroy(ld->packdone[i]);
        if (ld->xdone[i]) cudaEventDestroy(ld->xdone[i]);
        if (ld->rready[i]) cudaEventDestroy(ld->rready[i]);
        if (ld->rdone[i]) cudaEventDestroy(ld->rdone[i]);
        if (ld->augdone[i]) cudaEventDestroy(ld->augdone[i]);
    }
    if (ld->storage) cudaFreeHost(ld->storage);
    for (auto& sl : ld->slot) {
        for (void* q : {static_cast<void*>(sl.moves), static_cast<void*>(sl.off),
                        static_cast<void*>(sl.kept), static_cast<void*>(sl.counts),
                        static_cast<void*>(sl.nmoves), static_cast<void*>(sl.stats),
                        static_cast<void*>(sl.regcnt)})
            if (q) cudaFreeHost(q);
        if (sl.ready) cudaEventDestroy(sl.ready);
    }
    if (ld->plan_stream) cudaStreamDestroy(ld->plan_stream);
    if (ld->comm) {
        for (auto& m : ld->nccl_mem) ncclCommDeregister(ld->comm, m.second);
        ncclCommDestroy(ld->comm);
    }
    for (auto& m : ld->nccl_mem) ncclMemFree(m.first);
    delete ld;
}

void loader_comm_init(ll_loader* ld, const uint8_t* id128) {
    set_device(ld->ctx);
    // The regular scheme's full all-to-all (large messages every step) runs
    // on registered buffers with 128 KB NVLink P2P chunks; the balanced
    // schemes' few small tail moves keep cudaMalloc buffers and NCCL's
    // default chunks, which registration and small chunks slowed at N = 4
    // (profiles/r2_nccl_exchange.md).  The chunk size takes effect only if no
    // communicator of this process has read NCCL's parameters yet (bench.py
    // sets it before torch.distributed for cfg4); a user's own value wins.
    const bool regular = ld->cfg.scheme == LL_SCHEME_REGULAR;
    if (regular) setenv("NCCL_P2P_NVL_CHUNKSIZE", "131072", 0);
    ncclUniqueId id;
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(&id, id128, sizeof(id));
    LL_NCCL(ncclCommInitRank(&ld->comm, static_cast<int>(ld->cfg.learners), id,
                             static_cast<int>(ld->cfg.rank)));
    // Every exchange buffer at its largest size now: a buffer grown on the step
    // path is a cudaFree + cudaMalloc, which synchronises the device while peer
    // ranks' NCCL kernels wait on this rank's next send/recv -- a deadlock.
    // Sends are at most the batch, receives at most this learner's share.
    const ll_loader_config& c = ld->cfg;
    const uint64_t B = c.batch_size, p = c.learners;
    const uint64_t share = (B + p - 1) / p;
    // the message slot issue_exchange uses: a crop window (which may exceed a
    // small source's whole sample, e.g. 224 x 224) or the whole sample
    const uint64_t slot = msg_slot(ld);
    // sends: at most the batch in crop mode; resize slots are large (a whole
    // resize window), so there a learner's sends are capped at its share --
    // a learner sends count - target <= B - B/p, which exceeds B/p only when
    // it owns over half of a p > 2 batch (need() fails loudly if it ever does)
    const uint64_t max_send = c.augment.mode == LL_AUG_CROP ? B : share;
    // LL_NCCL_REGISTER=0 / 1: plain / registered buffers for every scheme (A/B)
    const char* reg_env = std::getenv("LL_NCCL_REGISTER");
    const bool reg = reg_env && reg_env[0] ? reg_env[0] != '0' : regular;
    auto alloc = [&](ll::DevBuf& b, uint64_t n) {
        if (!reg) {
            b.reserve(n);
            return;
        }
        void* ptr = nullptr;
        void* handle = nullptr;
        LL_NCCL(ncclMemAlloc(&ptr, n));
        const ncclResult_t r = ncclCommRegister(ld->comm, ptr, n, &handle);
        if (r != ncclSuccess) {
            ncclMemFree(ptr);
            LL_NCCL(r);
        }
        ld->nccl_mem.emplace_back(ptr, handle);
        b.release();
        b.ptr = ptr;
        b.bytes = n;
        b.borrowed = true;
    };
    for (ll_loader::ExSet* x : {&ld->xset[0], &ld->xset[1]}) {
        alloc(x->pack, std::max<uint64_t>(max_send * slot, 16));
        alloc(x->recv, std::max<uint64_t>((c.scheme == LL_SCHEME_REGULAR ? B : share) * slot, 16));
        x->ridx.reserve(sizeof(uint32_t) * std::max<uint64_t>(share, 1));
    }
    LL_CUDA(cudaDeviceSynchronize());
}

void loader_ipc_handle(ll_loader* ld, uint8_t* out64) {
    set_device(ld->ctx);
    cudaIpcMemHandle_t h;
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
    LL_CUDA(cudaIpcGetMemHandle(&h, ld->shard.ptr));
    std::memcpy(out64, &h, sizeof(h));
}

void loader_open_peers(ll_loader* ld, const uint8_t* handles) {
    set_device(ld->ctx);
    const uint32_t p = ld->cfg.learners;
    std::vector<const uint8_t*> ptrs(p);
    for (uint32_t j = 0; j < p; ++j) {
        if (j == ld->cfg.rank) {
            ptrs[j] = ld->shard.as<uint8_t>();
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handles + 64ull * j, sizeof(h));
        void* ptr = nullptr;
        LL_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        ld->peer_open.push_back(ptr);
        ptrs[j] = static_cast<const uint8_t*>(ptr);
    }
    ld->d_peers.reserve(sizeof(void*) * p);
    LL_CUDA(cudaMemcpy(ld->d_peers.ptr, ptrs.data(), sizeof(void*) * p, cudaMemcpyHostToDevice));
    ld->peers_ready = true;
}

void loader_link_peers(ll_loader* const* lds, uint32_t n) {
    require(n >= 1, "link_peers: no loaders");
    const uint32_t p = lds[0]->cfg.learners;
    require(n == p, "link_peers: need one loader per learner");
    std::vector<const uint8_t*> ptrs(p, nullptr);
    for (uint32_t i = 0; i < n; ++i) {
        require(lds[i]->cfg.learners == p, "link_peers: learner counts differ");
        ptrs[lds[i]->cfg.rank] = lds[i]->shard.as<uint8_t>();
    }
    for (uint32_t j = 0; j < p; ++j) require(ptrs[j] != nullptr, "link_peers: missing rank");
    for (uint32_t i = 0; i < n; ++i) {
        set_device(lds[i]->ctx);
        lds[i]->d_peers.reserve(sizeof(void*) * p);
        LL_CUDA(cudaMemcpy(lds[i]->d_peers.ptr, ptrs.data(), sizeof(void*) * p,
                           cudaMemcpyHostToDevice));
        lds[i]->peers_ready = true;
    }
}

// Storage tier for alpha < 1: every uncached sample (ids [cached, d)) in one
// pinned, device-mapped host buffer, filled with the generate_dataset bytes in
// device-generated chunks.  The augment kernel reads crop windows from it
// directly (zero-copy over PCIe / NVLink-C2C) -- the "storage system" path of
// the paper's cost model (model.hpp:65-74), counted separately from NVLink.
void populate_storage(ll_loader* ld) {
    const uint64_t n = ld->cfg.d - ld->cached;
    if (n == 0 || ld->storage) return;
    ll_ctx* ctx = ld->ctx;
    // + 64: window rows are read from the 16-byte-aligned address at or below
    // them and may run up to 31 bytes past the last sample (K6, unaligned rows)
    LL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ld->storage), n * ld->S + 64,
                          cudaHostAllocMapped | cudaHostAllocPortable));
    const uint64_t chunk = std::max<uint64_t>(1, (1ull << 30) / ld->S);
    DevBuf& tmp = ctx->buf("storage.stage", chunk * ld->S);
    for (uint64_t i = 0; i < n; i += chunk) {
        const uint64_t m = std::min(chunk, n - i);
        generate_range_device(ctx, tmp.as<uint8_t>(), ld->cached + i, m, ld->S, ld->cfg.data_seed);
        LL_CUDA(cudaMemcpyAsync(ld->storage + i * ld->S, tmp.ptr, m * ld->S,
                                cudaMemcpyDeviceToHost, ctx->stream));
    }
    LL_CUDA(cudaStreamSynchronize(ctx->stream));
}

void ensure_plan_stream(ll_loader* ld);
void ensure_side_stream(ll_loader* ld);

// Steady state from the first step on: the output ring, the plan stream and
// the second plan slot (device scratch, pinned host tables) are created here,
// not on the step path, where an allocation would synchronise the device.
// Slot 1 is left holding epoch 1's plan, which the mid-epoch prefetch reuses.
void prime(ll_loader* ld) {
    ensure_out(ld);
    ensure_plan_stream(ld);
    ensure_side_stream(ld);
    if (ld->slot[1].epoch < 0) {
        plan_into(ld, 1, 1, ld->plan_stream);
        LL_CUDA(cudaStreamSynchronize(ld->plan_stream));
    }
}

void loader_populate(ll_loader* ld) {
    set_device(ld->ctx);
    populate_storage(ld);
    if (ld->cfg.geometry == LL_GEOM_VARIABLE)
        generate_var_device(ld->ctx, ld->shard.as<uint8_t>(), ld->first, ld->owned,
                            ld->prefix.as<uint64_t>(), ld->cfg.data_seed);
    else
        generate_range_device(ld->ctx, ld->shard.as<uint8_t>(), ld->first, ld->owned, ld->S,
                          ld->cfg.data_seed);
    LL_CUDA(cudaStreamSynchronize(ld->ctx->stream));
    prime(ld);
    ld->populated = true;
}

void loader_populate_from_host(ll_loader* ld, const uint8_t* host) {
    set_device(ld->ctx);
    require(ld->cached == ld->cfg.d, "Loader: populate_from_host needs alpha = 1");
    require(ld->cfg.geometry == LL_GEOM_FIXED,
            "Loader: populate_from_host supports fixed-size samples");
    LL_CUDA(cudaMemcpyAsync(ld->shard.ptr, host, ld->owned * ld->S, cudaMemcpyHostToDevice,
                            ld->ctx->stream));
    LL_CUDA(cudaStreamSynchronize(ld->ctx->stream));
    prime(ld);
    ld->populated = true;
}

// Cache population from the reference's on-disk dataset (generate_dataset /
// sample_path: `<root>/%08llu.bin`, pipeline.cpp:202-234): the learner's
// CacheDirectory block goes to its HBM shard and, for alpha < 1, ids
// [cached, d) to the host storage tier.  `threads` host threads read files
// into a pinned staging window that is copied to the device while the next
// window is read.  Errors name the sample like read_sample (pipeline.cpp:110-126).
namespace {

std::string sample_file(const std::string& root, uint64_t id) {
    char name[32];
    std::snprintf(name, sizeof(name), "%08llu.bin", static_cast<unsigned long long>(id));
    return root.empty() || root.back() == '/' ? root + name : root + "/" + name;
}

uint64_t sample_size(const ll_loader* ld, uint64_t id) {
    if (ld->cfg.geometry == LL_GEOM_FIXED) return ld->S;
    uint32_t h, w;
    var_hw(ld->cfg.data_seed, id, &h, &w);
    return 3ull * h * w;
}

// Reads ids [lo, hi) into dst (host) at offsets off(id); parallel over files.
// Variable geometry: the flat file rows land at the HBM row pitch (var_pitch).
template <typename Off>
void read_files(const ll_loader* ld, const std::string& root, uint64_t lo, uint64_t hi,
                uint8_t* dst, Off off, uint32_t threads) {
    std::atomic<uint64_t> next{lo};
    std::mutex err_mu;
    std::string err;
    const bool pitched = ld->cfg.geometry == LL_GEOM_VARIABLE;
    auto work = [&] {
        std::vector<uint8_t> flat;
        for (;;) {
            const uint64_t id = next.fetch_add(1);
            if (id >= hi) return;
            const std::string path = sample_file(root, id);
            const uint64_t want = sample_size(ld, id);
            FILE* f = std::fopen(path.c_str(), "rb");
            std::string e;
            if (!f) {
                e = "sample " + std::to_string(id) + ": cannot open " + path;
            } else {
                if (pitched) flat.resize(want);
                uint8_t* to = pitched ? flat.data() : dst + off(id);
                const size_t got = std::fread(to, 1, want, f);
                std::fclose(f);
                if (got != want) {
                    e = "sample " + std::to_string(id) + ": truncated file " + path + " (read " +
                        std::to_string(got) + " of " + std::to_string(want) + " bytes)";
                } else if (pitched) {
                    uint32_t h, w;
                    var_hw(ld->cfg.data_seed, id, &h, &w);
                    const uint32_t row = 3 * w, pitch = var_pitch(w);
                    uint8_t* out = dst + off(id);
                    for (uint32_t y = 0; y < h; ++y) {
                        std::memcpy(out + static_cast<uint64_t>(y) * pitch,
                                    flat.data() + static_cast<uint64_t>(y) * row, row);
                        std::memset(out + static_cast<uint64_t>(y) * pitch + row, 0, pitch - row);
                    }
                }
            }
            if (!e.empty()) {
                std::lock_guard<std::mutex> g(err_mu);
                if (err.empty()) err = e;
                next.store(hi);
                return;
            }
        }
    };
    std::vector<std::thread> pool;
    for (uint32_t t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    if (!err.empty()) fail(LL_ERR_RUNTIME, err);
}

} // namespace

void loader_populate_from_files(ll_loader* ld, const char* root_c, uint32_t threads) {
    require(root_c != nullptr, "Loader: null dataset root");
    set_device(ld->ctx);
    ll_ctx* ctx = ld->ctx;
    const std::string root(root_c);
    if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
    const ll_loader_config& c = ld->cfg;
    // HBM shard: windows of ~256 MiB through two pinned staging buffers
    const uint64_t first = ld->first, end = ld->first + ld->owned;
    std::vector<uint64_t> prefix;  // variable geometry: host copy of the shard's prefix
    if (c.geometry == LL_GEOM_VARIABLE) {
        prefix.resize(ld->owned + 1);
        LL_CUDA(cudaMemcpy(prefix.data(), ld->prefix.as<uint64_t>() + first,
                           sizeof(uint64_t) * (ld->owned + 1), cudaMemcpyDeviceToHost));
    }
    auto off_in_shard = [&](uint64_t id) -> uint64_t {
        return c.geometry == LL_GEOM_FIXED ? (id - first) * ld->S : prefix[id - first] - prefix[0];
    };
    const uint64_t window = 256ull << 20;
    uint8_t* stage[2] = {nullptr, nullptr};
    cudaEvent_t copied[2] = {nullptr, nullptr};
    try {
        for (int i = 0; i < 2; ++i) {
            LL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&stage[i]), window + (4ull << 20), 0));
            LL_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
        }
        uint64_t id = first;
        int b = 0;
        while (id < end) {
            // ids [id, stop) fit the window (at least one sample always)
            uint64_t stop = id, bytes = 0;
            while (stop < end) {
                const uint64_t sz = off_in_shard(stop + 1) - off_in_shard(stop);  // padded size
                if (bytes && bytes + sz > window) break;
                bytes += sz;
                ++stop;
            }
            LL_CUDA(cudaEventSynchronize(copied[b]));  // staging buffer b free again
            const uint64_t base = off_in_shard(id);
            read_files(ld, root, id, stop, stage[b],
                       [&](uint64_t s) { return off_in_shard(s) - base; }, threads);
            LL_CUDA(cudaMemcpyAsync(ld->shard.as<uint8_t>() + base, stage[b], bytes,
                                    cudaMemcpyHostToDevice, ctx->stream));
            LL_CUDA(cudaEventRecord(copied[b], ctx->stream));
            id = stop;
            b ^= 1;
        }
        LL_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        cudaStreamSynchronize(ctx->stream);
        for (int i = 0; i < 2; ++i) {
            if (stage[i]) cudaFreeHost(stage[i]);
            if (copied[i]) cudaEventDestroy(copied[i]);
        }
        throw;
    }
    for (int i = 0; i < 2; ++i) {
        cudaFreeHost(stage[i]);
        cudaEventDestroy(copied[i]);
    }
    // storage tier: straight into the pinned host buffer
    const uint64_t n_unc = c.d - ld->cached;
    if (n_unc) {
        if (!ld->storage)
            LL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ld->storage), n_unc * ld->S + 64,
                                  cudaHostAllocMapped | cudaHostAllocPortable));
        read_files(ld, root, ld->cached, c.d, ld->storage,
                   [&](uint64_t s) { return (s - ld->cached) * ld->S; }, threads);
    }
    prime(ld);
    ld->populated = true;
}

void loader_shard_range(ll_loader* ld, uint64_t* first, uint64_t* count) {
    *first = ld->first;
    *count = ld->owned;
}

uint64_t loader_steps(ll_loader* ld) { return ld->steps; }

// Make `epoch` the current plan: take the prefetched slot when it holds it
// (waiting only for its tables), else compute it now on the loader stream.
void loader_plan_epoch(ll_loader* ld, uint64_t epoch) {
    set_device(ld->ctx);
    ll_ctx* ctx = ld->ctx;
    // a prefetched exchange may still be packing from the old plan
    for (int i = 0; i < 2; ++i) {
        if (ld->xdone[i]) LL_CUDA(cudaStreamWaitEvent(ctx->stream, ld->xdone[i], 0));
        ld->xpending[i].valid = false;
        if (ld->rready[i]) LL_CUDA(cudaStreamWaitEvent(ctx->stream, ld->rready[i], 0));
        ld->rpending[i].valid = false;
    }
    const int k = ld->plan_epoch >= 0 ? ld->cur ^ 1 : ld->cur;
    auto& sl = ld->slot[k];
    if (sl.epoch != static_cast<int64_t>(epoch) || ld->plan_epoch < 0) {
        LL_CUDA(cudaEventSynchronize(sl.ready));  // any prefetch into this slot is done
        plan_into(ld, k, epoch, ctx->stream);
    } else {
        LL_CUDA(cudaStreamWaitEvent(ctx->stream, sl.ready, 0));  // prefetched
    }
    LL_CUDA(cudaEventSynchronize(sl.ready));
    permute_rounds(ctx, (ld->tag + (k ? "plan1" : "plan0")).c_str());  // raises if the round guard tripped
    ld->cur = k;
    ld->h_moves = sl.moves;
    ld->h_off = sl.off;
    ld->h_kept = sl.kept;
    ld->h_counts = sl.counts;
    ld->h_nmoves = sl.nmoves;
    ld->h_stats = sl.stats;
    ld->h_regcnt = sl.regcnt;
    ld->plan_epoch = static_cast<int64_t>(epoch);
}

// The side stream carries the prefetched exchange (K5 pack + NCCL) and the
// host-driven prologue (H2D + single-step K4).  Highest priority: its small
// grids are scheduled ahead of the pending CTAs of the running augment grid,
// so they complete under that augment instead of after it.
void ensure_side_stream(ll_loader* ld) {
    if (ld->side) return;
    int lo = 0, hi = 0;
    LL_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    LL_CUDA(cudaStreamCreateWithPriority(&ld->side, cudaStreamNonBlocking, hi));
}

void ensure_plan_stream(ll_loader* ld) {
    if (ld->plan_stream) return;
    // highest priority: the permutation is a cooperative launch, and its
    // blocks must win SMs back from the running augment grids promptly
    int lo = 0, hi = 0;
    LL_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    LL_CUDA(cudaStreamCreateWithPriority(&ld->plan_stream, cudaStreamNonBlocking, hi));
}

// Start planning epoch + 1 into the other slot on plan_stream, after
// everything already issued on the loader stream (which includes every step
// that read that slot's previous plan).
void prefetch_plan(ll_loader* ld, uint64_t next_epoch) {
    ll_ctx* ctx = ld->ctx;
    const int k = ld->cur ^ 1;
    auto& sl = ld->slot[k];
    if (sl.epoch == static_cast<int64_t>(next_epoch)) return;
    // LL_PLAN_PREFETCH: "stream" (default) / "inline" (loader stream) / "off"
    static const char* mode_env = std::getenv("LL_PLAN_PREFETCH");
    const std::string mode = mode_env ? mode_env : "stream";
    if (mode == "off") return;
    if (mode == "inline") {
        plan_into(ld, k, next_epoch, ctx->stream);
        return;
    }
    ensure_plan_stream(ld);
    cudaEvent_t issued = ctx->take_event();
    LL_CUDA(cudaEventRecord(issued, ctx->stream));
    LL_CUDA(cudaStreamWaitEvent(ld->plan_stream, issued, 0));
    ctx->event_pool.push_back(issued);
    plan_into(ld, k, next_epoch, ld->plan_stream);
}

void loader_step(ll_loader* ld, uint64_t epoch, uint64_t step, ll_step_info* info) {
    require(ld->populated, "Loader: shard not populated");
    require(step < ld->steps, "Loader: step out of range");
    if (ld->plan_epoch != static_cast<int64_t>(epoch)) loader_plan_epoch(ld, epoch);
    set_device(ld->ctx);
    ll_ctx* ctx = ld->ctx;
    const ll_loader_config& c = ld->cfg;
    const bool nccl = c.learners > 1 && c.exchange == LL_EXCHANGE_NCCL;
    auto tables = [&](uint64_t st) {
        return std::make_tuple(&ld->h_moves[st * kMaxP], &ld->h_off[st * (kMaxP + 1)],
                               &ld->h_kept[st * kMaxP], ld->h_nmoves[st], &ld->h_stats[st * 4]);
    };
    const uint64_t pp = static_cast<uint64_t>(c.learners) * c.learners;
    auto regcnt = [&](uint64_t st) -> const uint32_t* {
        return ld->h_regcnt ? ld->h_regcnt + st * pp : nullptr;
    };
    const ll_loader::ExSet* pre = nullptr;
    const uint32_t slot = step & 1;
    if (nccl) {
        if (!ld->xdone[0]) {
            for (int i = 0; i < 2; ++i) {
                LL_CUDA(cudaEventCreateWithFlags(&ld->xdone[i], cudaEventDisableTiming));
                LL_CUDA(cudaEventCreateWithFlags(&ld->augdone[i], cudaEventDisableTiming));
            }
            ensure_side_stream(ld);
        }
        auto& pend = ld->xpending[slot];
        if (pend.valid && pend.epoch == epoch && pend.step == step) {
            LL_CUDA(cudaStreamWaitEvent(ctx->stream, ld->xdone[slot], 0));
        } else {
            // not prefetched (first step of an epoch): exchange on the side
            // stream into this slot's buffers, after the step that last read them
            cudaStream_t ws = wire_stream(ld);
            LL_CUDA(cudaStreamWaitEvent(ws, ld->augdone[slot], 0));
            auto [mv, off, kept, nm, st] = tables(step);
            (void)kept;
            (void)st;
            issue_exchange(ld, ld->plan().view(), epoch, step, mv, nm, off, regcnt(step),
                           static_cast<int>(slot), ws);
            LL_CUDA(cudaEventRecord(ld->xdone[slot], ws));
            LL_CUDA(cudaStreamWaitEvent(ctx->stream, ld->xdone[slot], 0));
        }
        pend.valid = false;
        pre = &ld->xset[slot];
    }
    // resize (K7): the prologue of this step was prefetched under the previous
    // step's augment, or runs now; that of the next step is issued after it
    const bool rpre = c.augment.mode == LL_AUG_RESIZE;
    // NCCL: the prologue only computes where a received sample's window will
    // sit (its slot in the step's receive set, xset[step & 1]); it reads no
    // received bytes, so it may run before the send/recv completes
    auto with_recv = [&](StepSrc ss, uint64_t st) {
        if (nccl && (ss.n_send || ss.n_recv)) {
            ss.src.recv = ld->xset[st & 1].recv.as<uint8_t>();
            ss.src.recv_slot = msg_slot(ld);
        }
        return ss;
    };
    int pslot = -1;
    if (rpre) {
        if (!ld->rready[0]) {
            for (int i = 0; i < 2; ++i) {
                LL_CUDA(cudaEventCreateWithFlags(&ld->rready[i], cudaEventDisableTiming));
                LL_CUDA(cudaEventCreateWithFlags(&ld->rdone[i], cudaEventDisableTiming));
            }
            ensure_side_stream(ld);
        }
        const int rs = static_cast<int>(step & 1);
        auto& rp = ld->rpending[rs];
        // any side-stream write into this set has landed before it is read or rewritten
        LL_CUDA(cudaStreamWaitEvent(ctx->stream, ld->rready[rs], 0));
        if (rp.valid && rp.epoch == epoch && rp.step == step) {
            pslot = rs;
        } else {
            auto [mv, off, kept, nm, st] = tables(step);
            (void)st;
            const StepSrc ss =
                with_recv(step_src(ld, ld->plan().view(), step, mv, off, kept, nm), step);
            if (resize_prepare(ctx, c.augment, c.seed, epoch, ss.src, ss.n_local, geom_h(c),
                               geom_w(c), rs, ld->tag))
                pslot = rs;
        }
        rp.valid = false;
    }
    {
        auto [mv, off, kept, nm, st] = tables(step);
        run_step(ld, epoch, ld->plan().view(), step, mv, off, kept, nm, st, info, pre, pslot,
                 regcnt(step));
    }
    if (rpre) {
        LL_CUDA(cudaEventRecord(ld->rdone[step & 1], ctx->stream));
        if (step + 1 < ld->steps) {
            const int ns = static_cast<int>((step + 1) & 1);
            auto [mv, off, kept, nm, st] = tables(step + 1);
            (void)st;
            const StepSrc ss =
                with_recv(step_src(ld, ld->plan().view(), step + 1, mv, off, kept, nm), step + 1);
            // set ns was last read by step - 1's augment
            LL_CUDA(cudaStreamWaitEvent(ld->side, ld->rdone[ns], 0));
            cudaStream_t main = ctx->stream;
            ctx->stream = ld->side;
            bool ok = false;
            try {
                ok = resize_prepare(ctx, c.augment, c.seed, epoch, ss.src, ss.n_local, geom_h(c),
                                    geom_w(c), ns, ld->tag);
            } catch (...) {
                ctx->stream = main;
                throw;
            }
            ctx->stream = main;
            LL_CUDA(cudaEventRecord(ld->rready[ns], ld->side));
            ld->rpending[ns] = {ok, epoch, step + 1};
        }
    }
    // halfway through the epoch, start the next epoch's plan on its own stream
    if (step == ld->steps / 2) prefetch_plan(ld, epoch + 1);
    if (nccl) {
        LL_CUDA(cudaEventRecord(ld->augdone[slot], ctx->stream));
        if (step + 1 < ld->steps) {
            // prefetch the next step's exchange while this augment runs
            const uint32_t ns = (step + 1) & 1;
            cudaStream_t ws = wire_stream(ld);
            LL_CUDA(cudaStreamWaitEvent(ws, ld->augdone[ns], 0));
            auto [mv, off, kept, nm, st] = tables(step + 1);
            (void)kept;
            (void)st;
            issue_exchange(ld, ld->plan().view(), epoch, step + 1, mv, nm, off, regcnt(step + 1),
                           static_cast<int>(ns), ws);
            LL_CUDA(cudaEventRecord(ld->xdone[ns], ws));
            ld->xpending[ns] = {true, epoch, step + 1};
        }
    }
}

void loader_submit_host(ll_loader* ld, uint64_t epoch, uint64_t step, const uint64_t* host_batch) {
    require(ld->populated, "Loader: shard not populated");
    set_device(ld->ctx);
    ll_ctx* ctx = ld->ctx;
    const ll_loader_config& c = ld->cfg;
    const uint64_t B = c.batch_size;
    const uint32_t p = c.learners, me = c.rank;
    const uint32_t F = std::max<uint32_t>(1, c.prefetch_depth);
    require(ld->submitted - ld->waited < F,
            "Loader: prefetch_depth host steps already outstanding (wait first)");
    if (ld->hslots.empty()) {
        for (uint32_t f = 0; f < F; ++f) {
            ld->hslots.emplace_back(new ll_loader::HostSlot());
            ld->hslots.back()->rtag = ld->tag + "h" + std::to_string(f) + ".";
        }
        for (auto& hp : ld->hslots) {
            auto& h = *hp;
            LL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h.pin),
                                  sizeof(ll_loader::Tables) + sizeof(uint64_t) * B, 0));
            LL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h.pin_batch), sizeof(uint64_t) * B, 0));
            LL_CUDA(cudaEventCreateWithFlags(&h.pro_done, cudaEventDisableTiming));
            LL_CUDA(cudaEventCreateWithFlags(&h.done, cudaEventDisableTiming));
            h.batch64.reserve(sizeof(uint64_t) * B);
            h.order.reserve(sizeof(uint32_t) * B);
            h.stage.reserve(sizeof(ll_loader::Tables) + sizeof(uint64_t) * B);
            h.plan.reserve(1, B);
            if (reg_nccl(c)) {
                h.plan.reserve_regcnt(1, p);
                LL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h.pin_rc),
                                      sizeof(uint32_t) * p * p, 0));
            }
        }
        ensure_side_stream(ld);
    }
    auto& h = *ld->hslots[ld->submitted % F];
    h.info = ll_step_info{};
    h.rslot = -1;
    h.info.epoch = epoch;
    h.info.step = step;
    // the caller's GlobalBatch: ids index the shard and the storage tier, so
    // an id outside [0, d) would read past them -- refuse it here
    for (uint64_t i = 0; i < B; ++i) {
        const uint64_t id = host_batch[i];
        if (id >= c.d)
            fail(LL_ERR_INVALID, "Loader: batch sample id " + std::to_string(id) +
                                     " out of range (dataset has " + std::to_string(c.d) +
                                     " samples)");
        h.pin_batch[i] = id;
    }
    // prologue (H2D + assignment) on the side stream, so it overlaps the
    // previous step's augment; it may reuse this slot only after the step that
    // last used it has finished on the main stream
    cudaStream_t main = ctx->stream;
    if (h.used) LL_CUDA(cudaStreamWaitEvent(ld->side, h.done, 0));
    const PlanDev pd = h.plan.view();
    const bool devplan = (c.scheme == LL_SCHEME_LOCALITY_BALANCED ||
                          c.scheme == LL_SCHEME_REGULAR) &&
                         (p == 1 || c.exchange == LL_EXCHANGE_P2P);
    h.synchronous = !devplan;
    const size_t tab = sizeof(ll_loader::Tables);
    // devplan: n_local is the balanced target / regular slice, known up front
    if (devplan) h.n_local = B / p + (me < B % p ? 1 : 0);
    ctx->stream = ld->side;
    try {
        LL_CUDA(cudaMemcpyAsync(h.batch64.ptr, h.pin_batch, sizeof(uint64_t) * B,
                                cudaMemcpyHostToDevice, ctx->stream));
        narrow_device(ctx, h.batch64.as<uint64_t>(), h.order.as<uint32_t>(), B);
        assign_device(ctx, h.order.as<uint32_t>(), 1, B, p, ld->cached, c.scheme, pd,
                      aug_plan(ld, epoch));
        if (devplan && c.augment.mode == LL_AUG_RESIZE) {
            // K7's prologue (geometry, far pulls, row table) too: it needs the plan only
            h.rslot = resize_prepare(ctx, c.augment, c.seed, epoch, devplan_src(ld, pd),
                                     h.n_local, geom_h(c), geom_w(c), 0, h.rtag)
                          ? 0
                          : -1;
        }
        if (devplan) {
            // the step's tables and local ids back to the host, also under the
            // previous step's augment (they depend on the plan only)
            launch(ctx, "stage", [&] {
                k_stage<<<static_cast<unsigned>(
                              std::min<uint64_t>((h.n_local + 255) / 256 + 1, 1184)),
                          256, 0, ctx->stream>>>(pd, me, p, h.stage.as<uint8_t>(), h.n_local);
            });
            LL_CUDA(cudaMemcpyAsync(h.pin, h.stage.ptr, tab + sizeof(uint64_t) * h.n_local,
                                    cudaMemcpyDeviceToHost, ctx->stream));
        } else {
            // NCCL exchange / unbalanced lists: the host needs the counts to
            // size the grid and the messages; staged here on the side stream so
            // the host waits for this step's plan only, not for the previous
            // step's augment on the main stream
            launch(ctx, "stage", [&] {
                k_stage<<<1, 256, 0, ctx->stream>>>(pd, me, p, h.stage.as<uint8_t>(), 0);
            });
            LL_CUDA(cudaMemcpyAsync(h.pin, h.stage.ptr, tab, cudaMemcpyDeviceToHost, ctx->stream));
            if (pd.regcnt)
                LL_CUDA(cudaMemcpyAsync(h.pin_rc, pd.regcnt, sizeof(uint32_t) * p * p,
                                        cudaMemcpyDeviceToHost, ctx->stream));
        }
        LL_CUDA(cudaEventRecord(h.pro_done, ctx->stream));
    } catch (...) {
        ctx->stream = main;
        throw;
    }
    ctx->stream = main;
    LL_CUDA(cudaStreamWaitEvent(main, h.pro_done, 0));
    h.used = true;
    h.info.h2d_bytes = sizeof(uint64_t) * B;
    if (devplan) {
        // fully asynchronous: the kernel reads the list offset and kept count
        // from the device plan
        void* out = run_step_devplan(ld, epoch, pd, h.n_local, h.rslot, h.rtag);
        h.info.d2h_bytes = tab + sizeof(uint64_t) * h.n_local;
        h.info.device_out = reinterpret_cast<uintptr_t>(out);
    } else {
        // the tables staged on the side stream (prologue above)
        LL_CUDA(cudaEventSynchronize(h.pro_done));
        const uint32_t* rc = pd.regcnt ? h.pin_rc : nullptr;  // regular + NCCL
        const auto* t = h.tab();
        ll_step_info local{};
        // NCCL: the exchange goes on the side stream behind this step's
        // prologue, into one of two buffer sets, so it overlaps the previous
        // step's augment on the main stream
        const ll_loader::ExSet* pre = nullptr;
        int xs = -1;
        if (p > 1 && c.exchange == LL_EXCHANGE_NCCL) {
            if (!ld->xdone[0]) {
                for (int i = 0; i < 2; ++i) {
                    LL_CUDA(cudaEventCreateWithFlags(&ld->xdone[i], cudaEventDisableTiming));
                    LL_CUDA(cudaEventCreateWithFlags(&ld->augdone[i], cudaEventDisableTiming));
                }
            }
            xs = static_cast<int>(ld->submitted & 1);
            cudaStream_t ws = wire_stream(ld);
            LL_CUDA(cudaStreamWaitEvent(ws, ld->augdone[xs], 0));
            // a loader_step prefetch parked in this set is clobbered now
            ld->xpending[xs].valid = false;
            issue_exchange(ld, pd, epoch, 0, t->moves, t->n, t->off, rc, xs, ws, h.pro_done);
            LL_CUDA(cudaEventRecord(ld->xdone[xs], ws));
            LL_CUDA(cudaStreamWaitEvent(ctx->stream, ld->xdone[xs], 0));
            pre = &ld->xset[xs];
        }
        // resize: K7's prologue on the side stream too (it needs the tables
        // and, over NCCL, where the receive slots are -- not their bytes), so
        // it overlaps the previous step's augment instead of running inline
        int pslot = -1;
        if (c.augment.mode == LL_AUG_RESIZE) {
            StepSrc ss = step_src(ld, pd, 0, t->moves, t->off, t->kept, t->n);
            if (pre && (ss.n_send || ss.n_recv)) {
                ss.src.recv = pre->recv.as<uint8_t>();
                ss.src.recv_slot = msg_slot(ld);
            }
            cudaStream_t main_s = ctx->stream;
            ctx->stream = ld->side;
            bool ok = false;
            try {
                ok = resize_prepare(ctx, c.augment, c.seed, epoch, ss.src, ss.n_local, geom_h(c),
                                    geom_w(c), 0, h.rtag);
            } catch (...) {
                ctx->stream = main_s;
                throw;
            }
            ctx->stream = main_s;
            if (ok) {
                cudaEvent_t ev = ctx->take_event();
                LL_CUDA(cudaEventRecord(ev, ld->side));
                LL_CUDA(cudaStreamWaitEvent(ctx->stream, ev, 0));
                ctx->event_pool.push_back(ev);
                pslot = 0;
            }
        }
        run_step(ld, epoch, pd, 0, t->moves, t->off, t->kept, t->n, t->stats, &local, pre,
                 pslot, rc, &h.rtag);
        if (xs >= 0) LL_CUDA(cudaEventRecord(ld->augdone[xs], ctx->stream));
        local.h2d_bytes = h.info.h2d_bytes;
        local.d2h_bytes = tab + (rc ? sizeof(uint32_t) * p * p : 0);
        h.info = local;
        h.n_local = local.n_local;
        launch(ctx, "stage", [&] {
            k_stage<<<static_cast<unsigned>(std::min<uint64_t>((h.n_local + 255) / 256 + 1, 1184)),
                      256, 0, ctx->stream>>>(pd, me, p, h.stage.as<uint8_t>(), h.n_local);
        });
        LL_CUDA(cudaMemcpyAsync(h.ids(), h.stage.as<uint8_t>() + tab,
                                sizeof(uint64_t) * h.n_local, cudaMemcpyDeviceToHost,
                                ctx->stream));
        h.info.d2h_bytes += sizeof(uint64_t) * h.n_local;
    }
    h.info.step = step;
    h.info.epoch = epoch;
    LL_CUDA(cudaEventRecord(h.done, ctx->stream));
    ++ld->submitted;
}

void loader_wait_host(ll_loader* ld, uint64_t* host_local_ids, ll_step_info* info) {
    require(ld->waited < ld->submitted, "Loader: no host step outstanding");
    set_device(ld->ctx);
    const uint32_t F = std::max<uint32_t>(1, ld->cfg.prefetch_depth);
    auto& h = *ld->hslots[ld->waited % F];
    LL_CUDA(cudaEventSynchronize(h.done));
    const uint32_t me = ld->cfg.rank, p = ld->cfg.learners;
    if (!h.synchronous) {
        const auto* t = h.tab();
        uint64_t recv = 0, nvl = 0;
        for (uint32_t m = 0; m < t->n; ++m)
            if (t->moves[m].receiver == me) {
                recv += t->moves[m].count;
                nvl += t->moves[m].nvlink;
            }
        const bool reg = p > 1 && ld->cfg.scheme == LL_SCHEME_REGULAR;
        h.info.n_local = h.n_local;
        h.info.kept = reg ? 0 : t->kept[me];
        h.info.received = reg ? h.n_local : recv;
        h.info.moved_total = t->stats[0];
        h.info.nvlink_bytes = nvl * ld->S;
        h.info.uncached = t->stats[2];
        h.info.reg_remote = t->stats[3] == 0xFFFFFFFFu ? UINT64_MAX : t->stats[3];
        h.info.device_ids = reinterpret_cast<uintptr_t>(h.plan.final_ids.as<uint32_t>() + t->off[me]);
    }
    if (host_local_ids) std::memcpy(host_local_ids, h.ids(), sizeof(uint64_t) * h.n_local);
    if (info) *info = h.info;
    ++ld->waited;
}

void loader_step_host(ll_loader* ld, uint64_t epoch, uint64_t step, const uint64_t* host_batch,
                      uint64_t* host_local_ids, ll_step_info* info) {
    require(ld->waited == ld->submitted, "Loader: host steps still outstanding");
    loader_submit_host(ld, epoch, step, host_batch);
    loader_wait_host(ld, host_local_ids, info);
}

void loader_plan_step(ll_loader* ld, uint64_t step, uint64_t* final_ids, uint64_t* final_off,
                      uint64_t* kept, uint64_t* counts, ll_move* moves, uint32_t* n_moves) {
    require(ld->plan_epoch >= 0, "Loader: no epoch planned");
    require(step < ld->steps, "Loader: step out of range");
    set_device(ld->ctx);
    const uint64_t B = ld->cfg.batch_size;
    const uint32_t p = ld->cfg.learners;
    std::vector<uint32_t> ids(B);
    LL_CUDA(cudaMemcpy(ids.data(), ld->plan().final_ids.as<uint32_t>() + step * B,
                       sizeof(uint32_t) * B, cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < B; ++i) final_ids[i] = ids[i];
    for (uint32_t j = 0; j <= p; ++j) final_off[j] = ld->h_off[step * (kMaxP + 1) + j];
    for (uint32_t j = 0; j < p; ++j) {
        kept[j] = ld->h_kept[step * kMaxP + j];
        counts[j] = ld->h_counts[step * kMaxP + j];
    }
    *n_moves = ld->h_nmoves[step];
    for (uint32_t m = 0; m < *n_moves; ++m) moves[m] = ld->h_moves[step * kMaxP + m];
}

// {steps, bytes sent, bytes received, timed steps, bytes received in timed
// steps, ms packing, ms on the wire, 0}
void loader_exchange_stats(ll_loader* ld, double* out8, int reset) {
    set_device(ld->ctx);
    for (const auto& t : ld->xtimes) {
        float a = 0, b = 0;
        LL_CUDA(cudaEventSynchronize(t.t3));
        LL_CUDA(cudaEventElapsedTime(&a, t.t0, t.t1));
        LL_CUDA(cudaEventElapsedTime(&b, t.t2, t.t3));
        ld->x_ms_pack += a;
        ld->x_ms_wire += b;
        ++ld->x_timed;
        ld->x_timed_recv += t.recvd;
        for (cudaEvent_t e : {t.t0, t.t1, t.t2, t.t3}) ld->ctx->event_pool.push_back(e);
    }
    ld->xtimes.clear();
    out8[0] = static_cast<double>(ld->x_steps);
    out8[1] = static_cast<double>(ld->x_sent);
    out8[2] = static_cast<double>(ld->x_recv);
    out8[3] = static_cast<double>(ld->x_timed);
    out8[4] = static_cast<double>(ld->x_timed_recv);
    out8[5] = ld->x_ms_pack;
    out8[6] = ld->x_ms_wire;
    out8[7] = 0;
    if (reset) {
        ld->x_steps = ld->x_sent = ld->x_recv = ld->x_timed = ld->x_timed_recv = 0;
        ld->x_ms_pack = ld->x_ms_wire = 0;
    }
}

// ---- DLPack view of a step's batch (the C-level trainer hand-off) --------
// The DLPack (v0.8) ABI, restated: a consumer of another framework takes the
// tensor without copying; the deleter frees the view only.
namespace dl {
struct Device {
    int32_t device_type;  // kDLCUDA = 2
    int32_t device_id;
};
struct DataType {
    uint8_t code;  // kDLFloat = 2, kDLBfloat = 4
    uint8_t bits;
    uint16_t lanes;
};
struct Tensor {
    void* data;
    Device device;
    int32_t ndim;
    DataType dtype;
    int64_t* shape;
    int64_t* strides;
    uint64_t byte_offset;
};
struct Managed {
    Tensor dl_tensor;
    void* manager_ctx;
    void (*deleter)(Managed*);
};
struct Holder {
    Managed m;
    int64_t shape[4];
};
void release(Managed* m) { delete reinterpret_cast<Holder*>(m); }
} // namespace dl

void loader_batch_dlpack(ll_loader* ld, const ll_step_info* info, void** out) {
    require(info != nullptr && out != nullptr, "dlpack: null argument");
    const ll_loader_config& c = ld->cfg;
    auto* h = new dl::Holder();
    h->shape[0] = static_cast<int64_t>(info->n_local);
    h->shape[1] = 3;
    h->shape[2] = c.augment.out_h;
    h->shape[3] = c.augment.out_w;
    h->m.dl_tensor.data = reinterpret_cast<void*>(info->device_out);
    h->m.dl_tensor.device = dl::Device{2, ld->ctx->device};
    h->m.dl_tensor.ndim = 4;
    h->m.dl_tensor.dtype = c.augment.out_dtype == LL_OUT_BF16 ? dl::DataType{4, 16, 1}
                                                              : dl::DataType{2, 32, 1};
    h->m.dl_tensor.shape = h->shape;
    h->m.dl_tensor.strides = nullptr;  // compact row-major
    h->m.dl_tensor.byte_offset = 0;
    h->m.manager_ctx = nullptr;
    h->m.deleter = dl::release;
    *out = &h->m;
}

void loader_epoch_totals(ll_loader* ld, uint64_t* out4) {
    require(ld->plan_epoch >= 0, "Loader: no epoch planned");
    for (int k = 0; k < 4; ++k) out4[k] = 0;
    for (uint64_t s = 0; s < ld->steps; ++s)
        for (int k = 0; k < 4; ++k) {
            const uint32_t v = ld->h_stats[s * 4 + k];
            out4[k] += (v == 0xFFFFFFFFu) ? 0 : v;
        }
}

} // namespace ll
