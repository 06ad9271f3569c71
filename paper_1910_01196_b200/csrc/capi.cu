// capi.cu -- the extern "C" boundary declared in include/locload_b200.h.
//
// Each entry point validates its arguments with the reference's own
// std::invalid_argument messages (cited per function), runs the device
// implementation and converts exceptions into status codes + ll_last_error().
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ll_internal.h"
#include "locload/equivalence.hpp"

namespace ll {
void widen_device(ll_ctx* ctx, const uint32_t* in, uint64_t* out, uint64_t n);
void loader_create(ll_loader** out, ll_ctx* ctx, const ll_loader_config* cfg);
void loader_destroy(ll_loader* ld);
void loader_comm_init(ll_loader* ld, const uint8_t* id128);
void loader_ipc_handle(ll_loader* ld, uint8_t* out64);
void loader_open_peers(ll_loader* ld, const uint8_t* handles);
void loader_populate(ll_loader* ld);
void loader_link_peers(ll_loader* const* lds, uint32_t n);
void loader_populate_from_host(ll_loader* ld, const uint8_t* host);
void loader_populate_from_files(ll_loader* ld, const char* root, uint32_t threads);
void loader_shard_range(ll_loader* ld, uint64_t* first, uint64_t* count);
uint64_t loader_steps(ll_loader* ld);
void loader_plan_epoch(ll_loader* ld, uint64_t epoch);
void loader_step(ll_loader* ld, uint64_t epoch, uint64_t step, ll_step_info* info);
void loader_step_host(ll_loader* ld, uint64_t epoch, uint64_t step, const uint64_t* host_batch,
                      uint64_t* host_local_ids, ll_step_info* info);
void loader_submit_host(ll_loader* ld, uint64_t epoch, uint64_t step, const uint64_t* host_batch);
void loader_wait_host(ll_loader* ld, uint64_t* host_local_ids, ll_step_info* info);
void loader_plan_step(ll_loader* ld, uint64_t step, uint64_t* final_ids, uint64_t* final_off,
                      uint64_t* kept, uint64_t* counts, ll_move* moves, uint32_t* n_moves);
void loader_epoch_totals(ll_loader* ld, uint64_t* out4);
void loader_exchange_stats(ll_loader* ld, double* out8, int reset);
void loader_batch_dlpack(ll_loader* ld, const ll_step_info* info, void** out);
// store.cu
void store_create(ll_store** out, int device, uint64_t capacity_samples);
void store_destroy(ll_store* st);
void store_size(ll_store* st, uint64_t* out);
void store_sample_bytes(ll_store* st, uint64_t* out);
void store_lookup(ll_store* st, const uint64_t* ids, uint64_t n, uint8_t* found);
void store_insert(ll_store* st, ll_ctx* ctx, const uint64_t* ids, uint64_t n,
                  uint64_t sample_bytes, const uint8_t* const* host_ptrs, uint8_t* inserted);
void store_gather(ll_store* st, ll_ctx* ctx, const uint64_t* ids, uint64_t n, uint8_t* host_dst);

namespace {
thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return LL_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return LL_ERR_RUNTIME;
    }
}

__global__ void k_narrow(const uint64_t* __restrict__ in, uint32_t* __restrict__ out,
                         uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<uint32_t>(in[i]);
}

void h2d(ll_ctx* ctx, void* dst, const void* src, size_t n) {
    if (n) LL_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, ctx->stream));
}
void d2h_sync(ll_ctx* ctx, void* dst, const void* src, size_t n) {
    if (n) LL_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, ctx->stream));
    LL_CUDA(cudaStreamSynchronize(ctx->stream));
}

void check_ctx(ll_ctx* ctx) {
    require(ctx != nullptr, "null context");
    set_device(ctx);
}

} // namespace

void set_device(ll_ctx* ctx) { LL_CUDA(cudaSetDevice(ctx->device)); }

void narrow_device(ll_ctx* ctx, const uint64_t* in, uint32_t* out, uint64_t n) {
    if (!n) return;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148u * 8u));
    launch(ctx, "narrow", [&] { k_narrow<<<grid, 256, 0, ctx->stream>>>(in, out, n); });
}

} // namespace ll

cudaEvent_t ll_ctx::take_event() {
    cudaEvent_t e;
    if (!event_pool.empty()) {
        e = event_pool.back();
        event_pool.pop_back();
        return e;
    }
    LL_CUDA(cudaEventCreate(&e));
    return e;
}

using namespace ll;

extern "C" {

int ll_version(void) { return 1; }

const char* ll_last_error(void) { return g_last_error.c_str(); }

int ll_device_count(int* out) {
    return guarded([&] {
        int n = 0;
        const cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) n = 0;
        *out = n;
    });
}

int ll_ctx_create(ll_ctx** out, int device) {
    return guarded([&] {
        require(out != nullptr, "null output");
        int n = 0;
        LL_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) fail(LL_ERR_CUDA, "no such CUDA device");
        auto ctx = std::make_unique<ll_ctx>();
        ctx->device = device;
        LL_CUDA(cudaSetDevice(device));
        LL_CUDA(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device));
        LL_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        *out = ctx.release();
    });
}

int ll_ctx_destroy(ll_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        for (auto& kv : ctx->times)
            for (auto& pr : kv.second.pending) {
                cudaEventDestroy(pr.first);
                cudaEventDestroy(pr.second);
            }
        for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
        ctx->scratch.clear();
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int ll_ctx_sync(ll_ctx* ctx) {
    return guarded([&] {
        check_ctx(ctx);
        LL_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int ll_ctx_stream(ll_ctx* ctx, uintptr_t* out) {
    return guarded([&] {
        require(ctx != nullptr, "null context");
        *out = reinterpret_cast<uintptr_t>(ctx->stream);
    });
}

int ll_ctx_launch_count(ll_ctx* ctx, uint64_t* out) {
    return guarded([&] {
        require(ctx != nullptr, "null context");
        *out = ctx->launches;
    });
}

int ll_ctx_set_timing(ll_ctx* ctx, int enable) {
    return guarded([&] {
        require(ctx != nullptr, "null context");
        ctx->timing = enable != 0;
    });
}

int ll_ctx_kernel_stats(ll_ctx* ctx, const char* kernel, uint64_t* launches, double* total_ms) {
    return guarded([&] {
        check_ctx(ctx);
        LL_CUDA(cudaStreamSynchronize(ctx->stream));
        auto& t = ctx->times[kernel];
        for (auto& pr : t.pending) {
            float ms = 0;
            LL_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
            t.total_ms += ms;
            t.launches += 1;
            ctx->event_pool.push_back(pr.first);
            ctx->event_pool.push_back(pr.second);
        }
        t.pending.clear();
        *launches = t.launches;
        *total_ms = t.total_ms;
    });
}

int ll_ctx_reset_stats(ll_ctx* ctx) {
    return guarded([&] {
        check_ctx(ctx);
        LL_CUDA(cudaStreamSynchronize(ctx->stream));
        for (auto& kv : ctx->times) {
            for (auto& pr : kv.second.pending) {
                ctx->event_pool.push_back(pr.first);
                ctx->event_pool.push_back(pr.second);
            }
            kv.second = KernelTimes();
        }
        ctx->launches = 0;
    });
}

int ll_ctx_copy_to_host(ll_ctx* ctx, void* host_dst, uintptr_t device_src, uint64_t bytes) {
    return guarded([&] {
        check_ctx(ctx);
        d2h_sync(ctx, host_dst, reinterpret_cast<const void*>(device_src), bytes);
    });
}

static void permute_to_host(ll_ctx* ctx, uint64_t seed, uint64_t epoch, uint64_t d,
                            const uint64_t* forced, uint64_t n_forced, uint64_t* host_order,
                            uint64_t k_out) {
    require(d < 0xFFFFFFFFull, "permute_epoch: device path needs d < 2^32 - 1");
    DevBuf& order = ctx->buf("api.order", sizeof(uint32_t) * d);
    DevBuf& wide = ctx->buf("api.order64", sizeof(uint64_t) * d);
    permute_device(ctx, seed, epoch, static_cast<uint32_t>(d), order.as<uint32_t>(), forced,
                   n_forced);
    widen_device(ctx, order.as<uint32_t>(), wide.as<uint64_t>(), k_out);
    d2h_sync(ctx, host_order, wide.ptr, sizeof(uint64_t) * k_out);
    permute_rounds(ctx);  // raises if the kernel's round guard tripped
}

// core.cpp:11-27
int ll_permute_epoch(ll_ctx* ctx, uint64_t seed, uint64_t epoch, uint64_t d,
                     uint64_t* host_order) {
    return guarded([&] {
        check_ctx(ctx);
        require(d != 0, "permute_epoch: dataset must contain at least one sample");
        permute_to_host(ctx, seed, epoch, d, nullptr, 0, host_order, d);
    });
}

int ll_permute_epoch_forced(ll_ctx* ctx, uint64_t seed, uint64_t epoch, uint64_t d,
                            const uint64_t* host_forced, uint64_t n_forced,
                            uint64_t* host_order) {
    return guarded([&] {
        check_ctx(ctx);
        require(d != 0, "permute_epoch: dataset must contain at least one sample");
        permute_to_host(ctx, seed, epoch, d, host_forced, n_forced, host_order, d);
    });
}

// core.cpp:29-55: the prefix of the dense permutation.
int ll_permutation_prefix(ll_ctx* ctx, uint64_t seed, uint64_t epoch, uint64_t d, uint64_t k,
                          uint64_t* host_prefix) {
    return guarded([&] {
        check_ctx(ctx);
        require(d != 0, "permutation_prefix: dataset must contain at least one sample");
        require(k <= d, "permutation_prefix: prefix length exceeds dataset size");
        if (k == 0) return;
        permute_to_host(ctx, seed, epoch, d, nullptr, 0, host_prefix, k);
    });
}

int ll_last_permute_profile(ll_ctx* ctx, uint64_t* out6) {
    return guarded([&] {
        check_ctx(ctx);
        permute_profile(ctx, out6);
    });
}

int ll_last_permute_rounds(ll_ctx* ctx, uint32_t* out) {
    return guarded([&] {
        check_ctx(ctx);
        *out = permute_rounds(ctx);
    });
}

// sampling.cpp:7-17 (CacheDirectory), :27-72, balance.cpp:14-84,
// equivalence.cpp:66-91
int ll_assign(ll_ctx* ctx, const uint64_t* host_batch, uint64_t B, uint64_t d, uint32_t p,
              double alpha, int scheme, uint64_t* final_ids, uint64_t* final_off,
              uint64_t* kept, uint64_t* counts, ll_move* moves, uint32_t* n_moves,
              uint64_t* stats4) {
    return guarded([&] {
        check_ctx(ctx);
        require(p != 0, "CacheDirectory: learner count must be >= 1");
        require(alpha > 0.0 && alpha <= 1.0, "CacheDirectory: cached fraction must be in (0, 1]");
        require(p <= kMaxP, "assign: learner count must be in [1, 64]");
        require(scheme >= LL_SCHEME_REGULAR && scheme <= LL_SCHEME_LOCALITY_BALANCED,
                "assign: unknown scheme");
        if (scheme == LL_SCHEME_REGULAR)
            require(B % p == 0, "reg_slice: learner count must divide the batch size");
        uint64_t cached = static_cast<uint64_t>(alpha * static_cast<double>(d));
        if (cached > d) cached = d;
        for (uint64_t i = 0; i < B; ++i)
            require(host_batch[i] < 0xFFFFFFFFull, "assign: sample ids must be < 2^32 - 1");
        const uint64_t Bs = B ? B : 1;
        DevBuf& b64 = ctx->buf("api.batch64", sizeof(uint64_t) * Bs);
        DevBuf& b32 = ctx->buf("api.batch32", sizeof(uint32_t) * Bs);
        auto& pb = ctx->api_plan;
        if (!pb) pb.reset(new PlanBufs());
        pb->reserve(1, Bs);
        h2d(ctx, b64.ptr, host_batch, sizeof(uint64_t) * B);
        narrow_device(ctx, b64.as<uint64_t>(), b32.as<uint32_t>(), B);
        assign_device(ctx, b32.as<uint32_t>(), 1, B, p, cached, scheme, pb->view());
        std::vector<uint32_t> ids(B), off(kMaxP + 1), kp(kMaxP), cn(kMaxP);
        std::vector<ll_move> mv(kMaxP);
        uint32_t nm = 0, st[4] = {0, 0, 0, 0};
        LL_CUDA(cudaMemcpyAsync(st, pb->stats.ptr, sizeof(st), cudaMemcpyDeviceToHost,
                                ctx->stream));
        if (B) LL_CUDA(cudaMemcpyAsync(ids.data(), pb->final_ids.ptr, sizeof(uint32_t) * B,
                                       cudaMemcpyDeviceToHost, ctx->stream));
        LL_CUDA(cudaMemcpyAsync(off.data(), pb->off.ptr, sizeof(uint32_t) * (kMaxP + 1),
                                cudaMemcpyDeviceToHost, ctx->stream));
        LL_CUDA(cudaMemcpyAsync(kp.data(), pb->kept.ptr, sizeof(uint32_t) * kMaxP,
                                cudaMemcpyDeviceToHost, ctx->stream));
        LL_CUDA(cudaMemcpyAsync(cn.data(), pb->counts.ptr, sizeof(uint32_t) * kMaxP,
                                cudaMemcpyDeviceToHost, ctx->stream));
        LL_CUDA(cudaMemcpyAsync(mv.data(), pb->moves.ptr, sizeof(ll_move) * kMaxP,
                                cudaMemcpyDeviceToHost, ctx->stream));
        d2h_sync(ctx, &nm, pb->n_moves.ptr, sizeof(uint32_t));
        for (uint64_t i = 0; i < B; ++i) final_ids[i] = ids[i];
        for (uint32_t j = 0; j <= p; ++j) final_off[j] = off[j];
        for (uint32_t j = 0; j < p; ++j) {
            kept[j] = kp[j];
            counts[j] = cn[j];
        }
        for (uint32_t m = 0; m < nm; ++m) moves[m] = mv[m];
        *n_moves = nm;
        if (stats4)
            for (int q = 0; q < 4; ++q) stats4[q] = st[q] == 0xFFFFFFFFu ? UINT64_MAX : st[q];
    });
}

// A whole epoch's plan with no shard attached: K2+K3 permute_epoch
// (core.cpp:11-27), batches (core.cpp:57-73) and K4 over every step -- the
// same kernels and device tables a loader plans its epochs with
// (loader.cu plan_into), so tests can pin the headline configuration's plan
// (cfg2: d = 1.28 M, p = 8, B = 8,192) and the bench can count remote samples
// per epoch for any p on one GPU.
int ll_plan_epoch(ll_ctx* ctx, uint64_t seed, uint64_t epoch, uint64_t d, uint32_t p,
                  uint64_t B, double alpha, int scheme, uint64_t* steps_out,
                  uint64_t* final_ids, uint64_t* final_off, uint64_t* kept, uint64_t* counts,
                  ll_move* moves, uint32_t* n_moves, uint64_t* stats4) {
    return guarded([&] {
        check_ctx(ctx);
        require(d != 0, "permute_epoch: dataset must contain at least one sample");
        require(B != 0 && B <= d, "batches: batch size must be in [1, dataset size]");
        require(p != 0, "CacheDirectory: learner count must be >= 1");
        require(alpha > 0.0 && alpha <= 1.0, "CacheDirectory: cached fraction must be in (0, 1]");
        require(p <= kMaxP, "assign: learner count must be in [1, 64]");
        require(d < 0xFFFFFFFFull, "plan_epoch: dataset size must be < 2^32 - 1 on the device");
        require(scheme >= LL_SCHEME_REGULAR && scheme <= LL_SCHEME_LOCALITY_BALANCED,
                "assign: unknown scheme");
        if (scheme == LL_SCHEME_REGULAR)
            require(B % p == 0, "reg_slice: learner count must divide the batch size");
        uint64_t cached = static_cast<uint64_t>(alpha * static_cast<double>(d));  // sampling.cpp:15
        if (cached > d) cached = d;
        const uint64_t steps = d / B;
        if (steps_out) *steps_out = steps;
        DevBuf& order = ctx->buf("epoch.order", sizeof(uint32_t) * d);
        PlanBufs pb;
        pb.reserve(steps, B);
        permute_device(ctx, seed, epoch, static_cast<uint32_t>(d), order.as<uint32_t>(), nullptr,
                       0, "epoch");
        assign_device(ctx, order.as<uint32_t>(), steps, B, p, cached, scheme, pb.view());
        std::vector<uint32_t> ids(final_ids ? steps * B : 0), off(steps * (kMaxP + 1)),
            kp(steps * kMaxP), cn(steps * kMaxP), nm(steps), st(steps * 4);
        std::vector<ll_move> mv(steps * kMaxP);
        auto d2h = [&](void* dst, const DevBuf& b, size_t n) {
            if (n) LL_CUDA(cudaMemcpyAsync(dst, b.ptr, n, cudaMemcpyDeviceToHost, ctx->stream));
        };
        d2h(ids.data(), pb.final_ids, sizeof(uint32_t) * ids.size());
        d2h(off.data(), pb.off, sizeof(uint32_t) * off.size());
        d2h(kp.data(), pb.kept, sizeof(uint32_t) * kp.size());
        d2h(cn.data(), pb.counts, sizeof(uint32_t) * cn.size());
        d2h(mv.data(), pb.moves, sizeof(ll_move) * mv.size());
        d2h(nm.data(), pb.n_moves, sizeof(uint32_t) * nm.size());
        d2h(st.data(), pb.stats, sizeof(uint32_t) * st.size());
        LL_CUDA(cudaStreamSynchronize(ctx->stream));
        permute_rounds(ctx, "epoch");  // raises if the round guard tripped
        for (uint64_t i = 0; i < ids.size(); ++i) final_ids[i] = ids[i];
        if (stats4)
            for (int q = 0; q < 4; ++q) stats4[q] = 0;
        for (uint64_t s = 0; s < steps; ++s) {
            if (final_off)
                for (uint32_t j = 0; j <= p; ++j)
                    final_off[s * (p + 1) + j] = off[s * (kMaxP + 1) + j];
            for (uint32_t j = 0; j < p; ++j) {
                if (kept) kept[s * p + j] = kp[s * kMaxP + j];
                if (counts) counts[s * p + j] = cn[s * kMaxP + j];
            }
            if (n_moves) n_moves[s] = nm[s];
            if (moves)
                for (uint32_t m = 0; m < nm[s]; ++m) moves[s * p + m] = mv[s * kMaxP + m];
            if (stats4)
                for (int q = 0; q < 4; ++q) {
                    const uint32_t v = st[s * 4 + q];
                    if (v == 0xFFFFFFFFu) stats4[q] = UINT64_MAX;
                    else if (stats4[q] != UINT64_MAX) stats4[q] += v;
                }
        }
    });
}

// balance.cpp:32-41 (validate) + :58-84
int ll_balance_batch(ll_ctx* ctx, const int64_t* counts, const int64_t* targets, uint32_t p,
                     uint64_t n, ll_move* moves, uint32_t* n_moves) {
    return guarded([&] {
        check_ctx(ctx);
        require(p <= kMaxP, "balance: at most 64 learners");
        for (uint64_t i = 0; i < n; ++i) {
            int64_t cs = 0, ts = 0;
            for (uint32_t j = 0; j < p; ++j) {
                cs += counts[i * p + j];
                ts += targets[i * p + j];
            }
            require(cs == ts, "balance: counts and targets must sum to the same total");
        }
        if (n == 0) return;
        if (p == 0) {
            for (uint64_t i = 0; i < n; ++i) n_moves[i] = 0;
            return;
        }
        DevBuf& c = ctx->buf("bal.counts", sizeof(int64_t) * n * p);
        DevBuf& t = ctx->buf("bal.targets", sizeof(int64_t) * n * p);
        DevBuf& m = ctx->buf("bal.moves", sizeof(ll_move) * n * p);
        DevBuf& k = ctx->buf("bal.n", sizeof(uint32_t) * n);
        h2d(ctx, c.ptr, counts, sizeof(int64_t) * n * p);
        h2d(ctx, t.ptr, targets, sizeof(int64_t) * n * p);
        balance_device(ctx, c.as<int64_t>(), t.as<int64_t>(), p, n, m.as<ll_move>(),
                       k.as<uint32_t>());
        LL_CUDA(cudaMemcpyAsync(moves, m.ptr, sizeof(ll_move) * n * p, cudaMemcpyDeviceToHost,
                                ctx->stream));
        d2h_sync(ctx, n_moves, k.ptr, sizeof(uint32_t) * n);
    });
}

// pipeline.cpp:208-234
int ll_generate_samples(ll_ctx* ctx, uint64_t data_seed, const uint64_t* host_ids, uint64_t n,
                        uint64_t sample_bytes, uint8_t* host_out) {
    return guarded([&] {
        check_ctx(ctx);
        require(sample_bytes != 0, "generate_dataset: need n >= 1 and sample_bytes >= 1");
        if (n == 0) return;
        DevBuf& ids = ctx->buf("gen.ids", sizeof(uint64_t) * n);
        DevBuf& out = ctx->buf("gen.out", n * sample_bytes);
        h2d(ctx, ids.ptr, host_ids, sizeof(uint64_t) * n);
        generate_ids_device(ctx, out.as<uint8_t>(), ids.as<uint64_t>(), n, sample_bytes,
                            data_seed);
        d2h_sync(ctx, host_out, out.ptr, n * sample_bytes);
    });
}

int ll_augment(ll_ctx* ctx, const ll_augment_spec* spec, uint64_t seed, uint64_t epoch,
               const uint8_t* host_src, const uint64_t* host_ids, uint64_t n, uint32_t height,
               uint32_t width, void* host_out) {
    return guarded([&] {
        check_ctx(ctx);
        require(spec != nullptr, "augment: null spec");
        if (n == 0) return;
        const uint64_t S = static_cast<uint64_t>(height) * width * 3;
        const uint64_t ob = 3ull * spec->out_h * spec->out_w *
                            (spec->out_dtype == LL_OUT_BF16 ? 2 : 4);
        DevBuf& src = ctx->buf("aug.src", n * S + 16);
        DevBuf& ids = ctx->buf("aug.ids", sizeof(uint64_t) * n);
        DevBuf& out = ctx->buf("aug.out", n * ob);
        h2d(ctx, src.ptr, host_src, n * S);
        h2d(ctx, ids.ptr, host_ids, sizeof(uint64_t) * n);
        SrcMap m;
        m.kind = 0;
        m.base = src.as<uint8_t>();
        m.ids = ids.as<uint64_t>();
        m.sample_bytes = S;
        augment_device(ctx, *spec, seed, epoch, m, n, height, width, out.ptr);
        d2h_sync(ctx, host_out, out.ptr, n * ob);
    });
}

int ll_augment_device(ll_ctx* ctx, const ll_augment_spec* spec, uint64_t seed, uint64_t epoch,
                      uintptr_t device_src, uintptr_t device_ids, uint64_t n, uint32_t height,
                      uint32_t width, uintptr_t device_out) {
    return guarded([&] {
        check_ctx(ctx);
        require(spec != nullptr, "augment: null spec");
        if (n == 0) return;
        SrcMap m;
        m.kind = 0;
        m.base = reinterpret_cast<const uint8_t*>(device_src);
        m.ids = reinterpret_cast<const uint64_t*>(device_ids);
        m.sample_bytes = static_cast<uint64_t>(height) * width * 3;
        augment_device(ctx, *spec, seed, epoch, m, n, height, width,
                       reinterpret_cast<void*>(device_out));
    });
}

int ll_ctx_enable_peer(ll_ctx* ctx, int peer_device) {
    return guarded([&] {
        check_ctx(ctx);
        int can = 0;
        LL_CUDA(cudaDeviceCanAccessPeer(&can, ctx->device, peer_device));
        if (!can) fail(LL_ERR_UNSUPPORTED, "no peer access between these devices");
        const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
            cudaGetLastError();
            return;
        }
        LL_CUDA(e);
    });
}

int ll_augment_params(ll_ctx* ctx, const ll_augment_spec* spec, uint64_t seed, uint64_t epoch,
                      const uint64_t* host_ids, uint64_t n, uint32_t height, uint32_t width,
                      uint32_t* host_params5) {
    return guarded([&] {
        check_ctx(ctx);
        require(spec != nullptr, "augment: null spec");
        if (n == 0) return;
        DevBuf& ids = ctx->buf("augp.ids", sizeof(uint64_t) * n);
        DevBuf& out = ctx->buf("augp.out", sizeof(uint32_t) * 5 * n);
        h2d(ctx, ids.ptr, host_ids, sizeof(uint64_t) * n);
        augment_params_device(ctx, *spec, seed, epoch, ids.as<uint64_t>(), n, height, width,
                              out.as<uint32_t>());
        d2h_sync(ctx, host_params5, out.ptr, sizeof(uint32_t) * 5 * n);
    });
}

int ll_loader_create(ll_loader** out, ll_ctx* ctx, const ll_loader_config* cfg) {
    return guarded([&] {
        check_ctx(ctx);
        loader_create(out, ctx, cfg);
    });
}

int ll_loader_destroy(ll_loader* ld) {
    return guarded([&] { loader_destroy(ld); });
}

int ll_nccl_unique_id(uint8_t* out128) {
    return guarded([&] {
        ncclUniqueId id;
        const ncclResult_t r = ncclGetUniqueId(&id);
        if (r != ncclSuccess) fail(LL_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
        std::memcpy(out128, &id, sizeof(id));
    });
}

int ll_loader_comm_init(ll_loader* ld, const uint8_t* id128) {
    return guarded([&] { loader_comm_init(ld, id128); });
}
int ll_loader_ipc_handle(ll_loader* ld, uint8_t* out64) {
    return guarded([&] { loader_ipc_handle(ld, out64); });
}
int ll_loader_open_peers(ll_loader* ld, const uint8_t* handles) {
    return guarded([&] { loader_open_peers(ld, handles); });
}
int ll_loader_link_peers(ll_loader* const* loaders, uint32_t n) {
    return guarded([&] { loader_link_peers(loaders, n); });
}

// equivalence.cpp:95-174 (run_training) and :190-205 (full_batch_gradient)
int ll_train_run(ll_ctx* ctx, const double* host_xs, const double* host_ys, uint64_t n,
                 uint32_t dims, int scheme, uint32_t p, uint64_t batch_size, uint64_t steps,
                 uint64_t seed, double learning_rate, int aggregation, double* host_final_w,
                 double* host_step_grads) {
    return guarded([&] {
        check_ctx(ctx);
        require(n >= 1 && dims >= 1, "ToyObjective: need n >= 1 and dims >= 1");
        require(p != 0, "run_training: need at least one learner");
        require(batch_size != 0 && batch_size <= n, "run_training: batch size must be in [1, n]");
        require(scheme >= LL_SCHEME_REGULAR && scheme <= LL_SCHEME_LOCALITY_BALANCED,
                "run_training: unknown scheme");
        require(aggregation == LL_AGG_CANONICAL || aggregation == LL_AGG_LEARNER_ORDER,
                "run_training: unknown aggregation");
        if (scheme == LL_SCHEME_REGULAR)
            require(batch_size % p == 0, "reg_slice: learner count must divide the batch size");
        require(p <= kMaxP, "run_training: learner count must be in [1, 64] on the device");
        require(n < 0xFFFFFFFFull, "run_training: sample count must be < 2^32 - 1");
        require(host_xs && host_ys && host_final_w, "run_training: null buffer");
        train_run_device(ctx, host_xs, host_ys, n, dims, scheme, p, batch_size, steps, seed,
                         learning_rate, aggregation, host_final_w, host_step_grads);
    });
}

// pure host logic (no device)
int ll_toy_synthesize(uint64_t n, uint32_t dims, uint64_t seed, double* host_xs, double* host_ys) {
    return guarded([&] {
        require(n >= 1 && dims >= 1, "ToyObjective: need n >= 1 and dims >= 1");
        const locload::ToyObjective obj = locload::ToyObjective::synthesize(n, dims, seed);
        std::copy(obj.xs().begin(), obj.xs().end(), host_xs);
        std::copy(obj.ys().begin(), obj.ys().end(), host_ys);
    });
}

int ll_full_batch_gradient(ll_ctx* ctx, const double* host_xs, const double* host_ys, uint64_t n,
                           uint32_t dims, const double* host_w, const uint64_t* host_batch,
                           uint64_t batch_size, double* host_grad) {
    return guarded([&] {
        check_ctx(ctx);
        require(n >= 1 && dims >= 1, "ToyObjective: need n >= 1 and dims >= 1");
        require(n < 0xFFFFFFFFull, "full_batch_gradient: sample count must be < 2^32 - 1");
        for (uint64_t i = 0; i < batch_size; ++i)
            require(host_batch[i] < n, "full_batch_gradient: sample id out of range");
        if (batch_size == 0) {  // 0 * (1.0 / 0) per coordinate, as the reference computes
            for (uint32_t k = 0; k < dims; ++k) host_grad[k] = 0.0 * (1.0 / 0.0);
            return;
        }
        full_batch_gradient_device(ctx, host_xs, host_ys, n, dims, host_w, host_batch,
                                   batch_size, host_grad);
    });
}

// pure host logic (no device): usable on CPU-only hosts
int ll_exchange_plan(const ll_move* moves, uint32_t n_moves, const uint64_t* final_off,
                     uint32_t p, uint32_t me, ll_xfer* out, uint32_t* n_xfers) {
    return guarded([&] {
        require(me < p, "exchange_plan: learner out of range");
        const std::vector<ll_xfer> xs = exchange_plan(moves, n_moves, final_off, me);
        for (size_t i = 0; i < xs.size(); ++i) out[i] = xs[i];
        *n_xfers = static_cast<uint32_t>(xs.size());
    });
}

int ll_loader_populate(ll_loader* ld) {
    return guarded([&] { loader_populate(ld); });
}
int ll_loader_populate_from_files(ll_loader* ld, const char* root, uint32_t threads) {
    return guarded([&] { loader_populate_from_files(ld, root, threads); });
}
int ll_loader_populate_from_host(ll_loader* ld, const uint8_t* host_samples) {
    return guarded([&] { loader_populate_from_host(ld, host_samples); });
}
int ll_loader_shard_range(ll_loader* ld, uint64_t* first_id, uint64_t* count) {
    return guarded([&] { loader_shard_range(ld, first_id, count); });
}
int ll_loader_steps_per_epoch(ll_loader* ld, uint64_t* out) {
    return guarded([&] { *out = loader_steps(ld); });
}
int ll_loader_plan_epoch(ll_loader* ld, uint64_t epoch) {
    return guarded([&] { loader_plan_epoch(ld, epoch); });
}
int ll_loader_step(ll_loader* ld, uint64_t epoch, uint64_t step, ll_step_info* info) {
    return guarded([&] { loader_step(ld, epoch, step, info); });
}
int ll_loader_step_host(ll_loader* ld, uint64_t epoch, uint64_t step,
                        const uint64_t* host_batch, uint64_t* host_local_ids,
                        ll_step_info* info) {
    return guarded([&] { loader_step_host(ld, epoch, step, host_batch, host_local_ids, info); });
}
int ll_loader_submit_host(ll_loader* ld, uint64_t epoch, uint64_t step,
                          const uint64_t* host_batch) {
    return guarded([&] { loader_submit_host(ld, epoch, step, host_batch); });
}
int ll_loader_wait_host(ll_loader* ld, uint64_t* host_local_ids, ll_step_info* info) {
    return guarded([&] { loader_wait_host(ld, host_local_ids, info); });
}
int ll_loader_plan_step(ll_loader* ld, uint64_t step, uint64_t* final_ids, uint64_t* final_off,
                        uint64_t* kept, uint64_t* counts, ll_move* moves, uint32_t* n_moves) {
    return guarded(
        [&] { loader_plan_step(ld, step, final_ids, final_off, kept, counts, moves, n_moves); });
}
int ll_loader_epoch_totals(ll_loader* ld, uint64_t* out4) {
    return guarded([&] { loader_epoch_totals(ld, out4); });
}

int ll_loader_batch_dlpack(ll_loader* ld, const ll_step_info* info, void** out_managed) {
    return guarded([&] {
        require(ld != nullptr, "null loader");
        loader_batch_dlpack(ld, info, out_managed);
    });
}

int ll_loader_exchange_stats(ll_loader* ld, double* out8, int reset) {
    return guarded([&] {
        require(ld != nullptr, "null loader");
        loader_exchange_stats(ld, out8, reset);
    });
}

// ---- sample store: SampleCache (pipeline.hpp:68-94) in HBM (store.cu) ----
int ll_store_create(ll_store** out, int device, uint64_t capacity_samples) {
    return guarded([&] { store_create(out, device, capacity_samples); });
}

int ll_store_destroy(ll_store* st) {
    return guarded([&] { store_destroy(st); });
}

int ll_store_size(ll_store* st, uint64_t* out) {
    return guarded([&] { store_size(st, out); });
}

int ll_store_sample_bytes(ll_store* st, uint64_t* out) {
    return guarded([&] { store_sample_bytes(st, out); });
}

int ll_store_lookup(ll_store* st, const uint64_t* ids, uint64_t n, uint8_t* found) {
    return guarded([&] { store_lookup(st, ids, n, found); });
}

int ll_store_insert(ll_store* st, ll_ctx* ctx, const uint64_t* ids, uint64_t n,
                    uint64_t sample_bytes, const uint8_t* const* host_ptrs, uint8_t* inserted) {
    return guarded([&] { store_insert(st, ctx, ids, n, sample_bytes, host_ptrs, inserted); });
}

int ll_store_gather(ll_store* st, ll_ctx* ctx, const uint64_t* ids, uint64_t n,
                    uint8_t* host_dst) {
    return guarded([&] { store_gather(st, ctx, ids, n, host_dst); });
}

// ---- distributed consumer (one learner per rank), device buffers --------
int ll_toy_grads_device(ll_ctx* ctx, uintptr_t xs, uintptr_t ys, uint32_t dims, uintptr_t w,
                        uintptr_t ids, uint64_t n_ids, uintptr_t grads) {
    return guarded([&] {
        check_ctx(ctx);
        require(dims >= 1, "ToyObjective: need n >= 1 and dims >= 1");
        toy_grads_device(ctx, reinterpret_cast<const double*>(xs),
                         reinterpret_cast<const double*>(ys), dims,
                         reinterpret_cast<const double*>(w), reinterpret_cast<const int64_t*>(ids),
                         n_ids, reinterpret_cast<double*>(grads));
    });
}

int ll_ordered_sum_device(ll_ctx* ctx, uintptr_t grads, uint64_t n, uint32_t dims,
                          uintptr_t order, uintptr_t out) {
    return guarded([&] {
        check_ctx(ctx);
        ordered_sum_device(ctx, reinterpret_cast<const double*>(grads), n, dims,
                           reinterpret_cast<const int64_t*>(order),
                           reinterpret_cast<double*>(out));
    });
}

int ll_sgd_apply_device(ll_ctx* ctx, uintptr_t gsum, uint32_t dims, double scale, double lr,
                        uintptr_t w, uintptr_t step_grad) {
    return guarded([&] {
        check_ctx(ctx);
        sgd_apply_device(ctx, reinterpret_cast<const double*>(gsum), dims, scale, lr,
                         reinterpret_cast<double*>(w), reinterpret_cast<double*>(step_grad));
    });
}

} // extern "C"
