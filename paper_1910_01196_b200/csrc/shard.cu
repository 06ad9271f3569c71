// shard.cu -- K1: synthesize dataset samples straight into HBM.
//
// Byte formula of generate_dataset, proj/src/pipeline.cpp:221-226: byte i of
// sample `id` is byte (i mod 8), little-endian, of draw i/8 of
// SplitMix64(derive_seed(seed, id)).  Because the stream is counter based,
// every 16-byte chunk (draws 2c, 2c+1) is independent: one thread writes one
// 128-bit chunk with a streaming store.  Write-bound: HBM roofline.
#include <algorithm>

#include "ll_internal.h"
#include "geometry.cuh"
#include "locload_rng.cuh"

namespace ll {
namespace {

__device__ __forceinline__ void st_cs_v4(void* p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ void gen_chunk(uint8_t* dst_sample, uint64_t key, uint64_t c,
                                          uint64_t sample_bytes, bool vec) {
    const uint64_t w0 = draw_at(key, 2 * c), w1 = draw_at(key, 2 * c + 1);
    const uint64_t byte0 = 16 * c;
    if (vec && byte0 + 16 <= sample_bytes) {
        st_cs_v4(dst_sample + byte0,
                 make_uint4(static_cast<uint32_t>(w0), static_cast<uint32_t>(w0 >> 32),
                            static_cast<uint32_t>(w1), static_cast<uint32_t>(w1 >> 32)));
    } else {  // unaligned sample sizes, or the sample's tail chunk
        const uint64_t end = byte0 + 16 < sample_bytes ? byte0 + 16 : sample_bytes;
        for (uint64_t b = byte0; b < end; ++b) {
            const uint64_t w = (b - byte0) < 8 ? w0 : w1;
            dst_sample[b] = static_cast<uint8_t>(w >> (((b - byte0) & 7) * 8));
        }
    }
}

// dst is [n][sample_bytes]; sample t has id first_id + t (or ids[t]).
__global__ void k_generate(uint8_t* __restrict__ dst, uint64_t first_id,
                           const uint64_t* __restrict__ ids, uint64_t n, uint64_t sample_bytes,
                           uint64_t chunks_per_sample, uint64_t data_seed, bool vec) {
    const uint64_t total = n * chunks_per_sample;
    for (uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; g < total;
         g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t t = g / chunks_per_sample, c = g - t * chunks_per_sample;
        const uint64_t id = ids ? ids[t] : first_id + t;
        gen_chunk(dst + t * sample_bytes, derive_seed(data_seed, id), c, sample_bytes, vec);
    }
}

void run(ll_ctx* ctx, uint8_t* dst, uint64_t first_id, const uint64_t* ids, uint64_t n,
         uint64_t sample_bytes, uint64_t data_seed) {
    if (n == 0 || sample_bytes == 0) return;
    const uint64_t cps = (sample_bytes + 15) / 16;
    const uint64_t total = n * cps;
    const uint64_t cap = static_cast<uint64_t>(ctx->sm_count) * 8;  // 8 x 256-thread CTAs / SM
    const uint64_t want = (total + 255) / 256;
    const unsigned grid = static_cast<unsigned>(want < cap ? want : cap);
    const bool vec = (reinterpret_cast<uintptr_t>(dst) % 16 == 0) && (sample_bytes % 16 == 0);
    launch(ctx, "generate", [&] {
        k_generate<<<grid, 256, 0, ctx->stream>>>(dst, first_id, ids, n, sample_bytes, cps,
                                                  data_seed, vec);
    });
}

// Variable geometry: padded byte size of every id in [0, d) into vals[0..d).
__global__ void k_var_sizes(uint64_t* __restrict__ vals, uint64_t d, uint64_t data_seed) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < d;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t h, w;
        var_hw(data_seed, i, &h, &w);
        vals[i] = var_bytes(h, w);
    }
}

// In-place exclusive scan of vals[0..n) into vals[0..n], one CTA (setup only:
// run once per loader).  Thread t owns a contiguous chunk.
__global__ void __launch_bounds__(1024) k_scan1(uint64_t* vals, uint64_t n) {
    __shared__ uint64_t part[1024];
    const uint64_t chunk = (n + blockDim.x - 1) / blockDim.x;
    const uint64_t b = threadIdx.x * chunk, e = b + chunk < n ? b + chunk : n;
    uint64_t sum = 0;
    for (uint64_t i = b; i < e; ++i) sum += vals[i];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (uint32_t off = 1; off < blockDim.x; off <<= 1) {
        const uint64_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint64_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
    for (uint64_t i = b; i < e; ++i) {
        const uint64_t v = vals[i];
        vals[i] = run;
        run += v;
    }
    if (threadIdx.x == blockDim.x - 1) vals[n] = part[blockDim.x - 1];
}

// One CTA per owned sample: the generate_dataset bytes of sample first+t at
// shard + prefix[first+t] - prefix[first], row y at y * var_pitch(w) (the
// pitch padding is zero).  Thread per 16 bytes of a pitched row: they span at
// most three 8-byte draws of the flat byte stream; four 32-bit stores (rows
// are only word aligned).
__global__ void __launch_bounds__(256) k_generate_var(uint8_t* __restrict__ shard, uint64_t first,
                                                      const uint64_t* __restrict__ prefix,
                                                      uint64_t data_seed) {
    const uint64_t id = first + blockIdx.x;
    uint32_t h, w;
    var_hw(data_seed, id, &h, &w);
    const uint32_t row = 3 * w, pitch = var_pitch(w), q16 = (pitch + 15) / 16;
    uint8_t* dst = shard + (prefix[id] - prefix[first]);
    const uint64_t key = derive_seed(data_seed, id);
    for (uint32_t t = threadIdx.x; t < h * q16; t += blockDim.x) {
        const uint32_t y = t / q16, col = 16 * (t - y * q16);
        const uint64_t b0 = static_cast<uint64_t>(y) * row + col;  // flat byte index
        const uint32_t sh = 8 * static_cast<uint32_t>(b0 & 7);
        const uint64_t d0 = draw_at(key, b0 >> 3), d1 = draw_at(key, (b0 >> 3) + 1);
        const uint64_t d2 = sh ? draw_at(key, (b0 >> 3) + 2) : 0;
        // bytes b0 .. b0+15 as two 64-bit words
        const uint64_t lo = sh ? (d0 >> sh) | (d1 << (64 - sh)) : d0;
        const uint64_t hi = sh ? (d1 >> sh) | (d2 << (64 - sh)) : d1;
        uint32_t* out = reinterpret_cast<uint32_t*>(dst + static_cast<uint64_t>(y) * pitch + col);
        const uint32_t v[4] = {static_cast<uint32_t>(lo), static_cast<uint32_t>(lo >> 32),
                               static_cast<uint32_t>(hi), static_cast<uint32_t>(hi >> 32)};
#pragma unroll
        for (uint32_t i = 0; i < 4; ++i) {
            const uint32_t c = col + 4 * i;
            if (c >= pitch) break;
            uint32_t x = v[i];
            if (c + 4 > row) x = c >= row ? 0u : x & ((1u << (8 * (row - c))) - 1u);
            out[i] = x;
        }
    }
}

} // namespace

void var_prefix_device(ll_ctx* ctx, uint64_t* d_prefix, uint64_t d, uint64_t data_seed) {
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((d + 255) / 256, 148u * 8u));
    launch(ctx, "var_sizes", [&] {
        k_var_sizes<<<grid ? grid : 1, 256, 0, ctx->stream>>>(d_prefix, d, data_seed);
    });
    launch(ctx, "scan", [&] { k_scan1<<<1, 1024, 0, ctx->stream>>>(d_prefix, d); });
}

void generate_var_device(ll_ctx* ctx, uint8_t* shard, uint64_t first, uint64_t n,
                         const uint64_t* d_prefix, uint64_t data_seed) {
    if (n == 0) return;
    launch(ctx, "generate", [&] {
        k_generate_var<<<static_cast<unsigned>(n), 256, 0, ctx->stream>>>(shard, first, d_prefix,
                                                                         data_seed);
    });
}

void generate_range_device(ll_ctx* ctx, uint8_t* dst, uint64_t first_id, uint64_t n,
                           uint64_t sample_bytes, uint64_t data_seed) {
    run(ctx, dst, first_id, nullptr, n, sample_bytes, data_seed);
}

void generate_ids_device(ll_ctx* ctx, uint8_t* dst, const uint64_t* d_ids, uint64_t n,
                         uint64_t sample_bytes, uint64_t data_seed) {
    run(ctx, dst, 0, d_ids, n, sample_bytes, data_seed);
}

} // namespace ll
