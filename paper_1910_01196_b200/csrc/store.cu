// store.cu -- the HBM sample store behind locload::SampleCache.
//
// Reference: SampleCache (proj/include/locload/pipeline.hpp:68-94), a host
// unordered_map<SampleId, shared_ptr<vector<u8>>> with a capacity in samples,
// populate on first touch, no replacement, concurrent readers and exclusive
// writers.  Here the payloads live in device memory:
//   * slots of the (fixed) sample size are carved from slabs of about 1 GiB,
//     allocated as the store fills -- capacity is only an upper bound, so a
//     capacity of the whole dataset costs nothing up front; when HBM runs out
//     the store behaves as full (inserts are skipped, as the reference skips
//     them at capacity);
//   * the id -> slot index is host metadata under a shared mutex (lookups run
//     concurrently, inserts exclusively);
//   * an insert's copy completes before its ids are published, so any thread
//     that finds an id can gather it on its own stream;
//   * gathers run one kernel that packs the requested slots contiguously
//     (16-byte vector copies when the sample size allows), then one D2H.
#include <algorithm>
#include <shared_mutex>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "ll_internal.h"

struct ll_store {
    int device = 0;
    uint64_t capacity = 0;  // samples
    uint64_t S = 0;         // sample bytes, fixed by the first insert
    uint64_t per_slab = 0;  // slots per slab
    std::vector<void*> slabs;
    uint64_t used = 0;      // slots handed out
    bool hbm_full = false;  // a slab allocation failed: treat as full
    std::unordered_map<uint64_t, uint64_t> slot;  // published ids
    std::unordered_set<uint64_t> pending;         // being copied in
    mutable std::shared_mutex mu;

    uint8_t* slot_ptr(uint64_t k) const {
        return static_cast<uint8_t*>(slabs[k / per_slab]) + (k % per_slab) * S;
    }
};

namespace ll {
namespace {

constexpr uint64_t kSlabBytes = 1ull << 30;

// one CTA row per sample, 16-byte copies (S % 16 == 0) or bytes otherwise
__global__ void k_store_gather(const uint8_t* const* __restrict__ src, uint64_t n, uint64_t S,
                               uint8_t* __restrict__ dst) {
    for (uint64_t i = blockIdx.y; i < n; i += gridDim.y) {
        const uint8_t* s = src[i];
        uint8_t* d = dst + i * S;
        if ((S & 15) == 0) {
            const uint64_t w = S >> 4;
            for (uint64_t k = blockIdx.x * blockDim.x + threadIdx.x; k < w;
                 k += static_cast<uint64_t>(gridDim.x) * blockDim.x)
                reinterpret_cast<uint4*>(d)[k] = __ldg(reinterpret_cast<const uint4*>(s) + k);
        } else {
            for (uint64_t k = blockIdx.x * blockDim.x + threadIdx.x; k < S;
                 k += static_cast<uint64_t>(gridDim.x) * blockDim.x)
                d[k] = s[k];
        }
    }
}

void check_store(ll_store* st) { require(st != nullptr, "null sample store"); }
void check_ctx(ll_ctx* ctx) {
    require(ctx != nullptr, "null context");
    set_device(ctx);
}

} // namespace

void store_create(ll_store** out, int device, uint64_t capacity_samples) {
    require(out != nullptr, "null output");
    auto st = std::make_unique<ll_store>();
    st->device = device;
    st->capacity = capacity_samples;
    *out = st.release();
}

void store_destroy(ll_store* st) {
    if (!st) return;
    cudaSetDevice(st->device);
    for (void* p : st->slabs) cudaFree(p);
    delete st;
}

void store_size(ll_store* st, uint64_t* out) {
    check_store(st);
    std::shared_lock<std::shared_mutex> g(st->mu);
    *out = st->slot.size();
}

void store_sample_bytes(ll_store* st, uint64_t* out) {
    check_store(st);
    std::shared_lock<std::shared_mutex> g(st->mu);
    *out = st->S;
}

void store_lookup(ll_store* st, const uint64_t* ids, uint64_t n, uint8_t* found) {
    check_store(st);
    std::shared_lock<std::shared_mutex> g(st->mu);
    for (uint64_t i = 0; i < n; ++i) found[i] = st->slot.count(ids[i]) ? 1 : 0;
}

void store_insert(ll_store* st, ll_ctx* ctx, const uint64_t* ids, uint64_t n,
                  uint64_t sample_bytes, const uint8_t* const* host_ptrs, uint8_t* inserted) {
    check_store(st);
    check_ctx(ctx);
    require(ctx->device == st->device, "store: context on another device");
    require(sample_bytes >= 1, "store: empty samples");
    std::vector<std::pair<uint64_t, uint64_t>> take;  // (index in ids, slot)
    {
        std::unique_lock<std::shared_mutex> g(st->mu);
        if (st->S == 0) {
            st->S = sample_bytes;
            st->per_slab = std::max<uint64_t>(1, kSlabBytes / sample_bytes);
        }
        require(sample_bytes == st->S, "store: samples must all have the same size");
        for (uint64_t i = 0; i < n; ++i) {
            if (inserted) inserted[i] = 0;
            const uint64_t id = ids[i];
            if (st->slot.count(id) || st->pending.count(id)) continue;
            if (st->used >= st->capacity || st->hbm_full) continue;
            const uint64_t k = st->used;
            if (k / st->per_slab >= st->slabs.size()) {
                const uint64_t left = st->capacity - k;
                const uint64_t slots = std::min<uint64_t>(st->per_slab, left);
                void* p = nullptr;
                set_device(ctx);
                if (cudaMalloc(&p, slots * st->S) != cudaSuccess) {
                    cudaGetLastError();  // out of HBM: the store is full from here on
                    st->hbm_full = true;
                    continue;
                }
                st->slabs.push_back(p);
            }
            ++st->used;
            st->pending.insert(id);
            take.emplace_back(i, k);
            if (inserted) inserted[i] = 1;
        }
    }
    if (take.empty()) return;
    set_device(ctx);
    cudaError_t err = cudaSuccess;
    for (const auto& t : take) {
        err = cudaMemcpyAsync(st->slot_ptr(t.second), host_ptrs[t.first], st->S,
                              cudaMemcpyHostToDevice, ctx->stream);
        if (err != cudaSuccess) break;
    }
    if (err == cudaSuccess) err = cudaStreamSynchronize(ctx->stream);
    std::unique_lock<std::shared_mutex> g(st->mu);
    for (const auto& t : take) {
        st->pending.erase(ids[t.first]);
        if (err == cudaSuccess) st->slot.emplace(ids[t.first], t.second);
    }
    cuda_check(err, "store insert copy");
}

void store_gather(ll_store* st, ll_ctx* ctx, const uint64_t* ids, uint64_t n,
                  uint8_t* host_dst) {
    check_store(st);
    check_ctx(ctx);
    require(ctx->device == st->device, "store: context on another device");
    if (n == 0) return;
    std::vector<const uint8_t*> src(n);
    uint64_t S = 0;
    {
        std::shared_lock<std::shared_mutex> g(st->mu);
        S = st->S;
        for (uint64_t i = 0; i < n; ++i) {
            auto it = st->slot.find(ids[i]);
            require(it != st->slot.end(),
                    "store: sample " + std::to_string(ids[i]) + " is not held");
            src[i] = st->slot_ptr(it->second);
        }
    }
    set_device(ctx);
    DevBuf& dsrc = ctx->buf("store.src", sizeof(void*) * n);
    DevBuf& dout = ctx->buf("store.out", n * S);
    LL_CUDA(cudaMemcpyAsync(dsrc.ptr, src.data(), sizeof(void*) * n, cudaMemcpyHostToDevice,
                            ctx->stream));
    const uint64_t units = (S & 15) == 0 ? S >> 4 : S;
    const unsigned bx = static_cast<unsigned>(std::min<uint64_t>((units + 255) / 256, 64));
    const unsigned by = static_cast<unsigned>(std::min<uint64_t>(n, 65535));
    launch(ctx, "store_gather", [&] {
        k_store_gather<<<dim3(bx, by), 256, 0, ctx->stream>>>(
            dsrc.as<const uint8_t* const>(), n, S, dout.as<uint8_t>());
    });
    LL_CUDA(cudaMemcpyAsync(host_dst, dout.ptr, n * S, cudaMemcpyDeviceToHost, ctx->stream));
    LL_CUDA(cudaStreamSynchronize(ctx->stream));
}

} // namespace ll
