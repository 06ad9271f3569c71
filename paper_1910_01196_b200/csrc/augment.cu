// augment.cu -- K6 (crop) and K7 (bilinear resize): the fused preprocess.
//
// Replaces the reference's injected preprocess delay (PreprocessPacer,
// proj/src/pipeline.cpp:87-108; real augmentation is a non-goal there,
// SPEC.md:430,438).  Semantics are defined by oracle/locload_oracle.c
// (lo_aug_params_for / lo_augment_one) and DESIGN.md section 4:
//   stream SplitMix64(derive_seed(seed, epoch, id)):  y0 = bounded(H-ch+1),
//   x0 = bounded(W-cw+1), flip = next() >> 63;
//   out[c][y][x] = (float(src[y0+y][x0+x'][c]) - mean255[c]) * inv_std255[c]
//   with x' = flip ? cw-1-x : x;  HWC u8 in, NCHW fp32 / bf16 (RNE) out.
//
// K6 (crop 224 from a fixed-size source) is HBM-bound: per sample it reads the
// 224x224x3 window (150,528 B) and writes 602,112 B (fp32) or 301,056 B
// (bf16).  One CTA = one sample x one 32-row band.  The band's source rows
// (the crop window widened to 16-byte alignment, <= 688 B per row) are pulled
// into shared memory with 128-bit non-allocating loads (far samples -- peer
// shards, host storage -- by TMA bulk copies); each thread then emits PX
// consecutive output pixels of all three planes as 128-bit streaming stores,
// so every warp writes 512 contiguous bytes per plane row.
//
// K7 (cfg5, variable-size sources, bilinear resize to 224): one CTA per
// (sample, 16 output rows), one output column per thread; taps from
// word-aligned source rows (geometry.cuh var_pitch) with the band's rows
// prefetched into L2; see the K7 section below and DESIGN.md section 5.
#include "ll_internal.h"
#include "geometry.cuh"
#include "locload_rng.cuh"

#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <cstdlib>
#include <string>

namespace ll {
namespace {

constexpr uint32_t kOut = 224;        // K6 output side (BASELINE configs)
constexpr uint32_t kBand = 32;        // rows per CTA
constexpr uint32_t kBands = kOut / kBand;
constexpr uint32_t kRowSmem = 704;    // >= 672 + 2*15, multiple of 16
// Peer samples (P2P over NVLink) arrive as ONE bulk copy of the band's
// contiguous source span (rows at their source pitch) instead of 32 row
// requests: 11 % more bytes (31 x 768 + 704 vs 32 x 704 at 256 px) in one
// large request; cfg4 over P2P at N = 2: +1 % (fp32), +3 % (bf16)
// (profiles/r2_nvlink_modes.md).
constexpr uint32_t kBandSmem = kBand * 768;
constexpr uint32_t kThreads = 224;

struct AugArgs {
    SrcMap src;
    uint32_t H, W;
    uint64_t seed, epoch;
    NormConst nc;
    void* out;
    uint64_t n;
    uint32_t out_h, out_w;
};

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_cs_v4(void* p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// Resolve sample k of a launch: id and source bytes.
// *far (optional): the bytes live outside this GPU's HBM (a peer shard over
// NVLink, or the host storage tier over PCIe).
__device__ __forceinline__ void resolve(const SrcMap& m, uint64_t k, uint64_t* id,
                                        const uint8_t** src, bool* far = nullptr,
                                        bool* win = nullptr,   // *win: src is a window slot
                                        bool* peer = nullptr) {  // *peer: a peer shard
    if (far) *far = false;
    if (peer) *peer = false;
    if (win) *win = false;
    const uint64_t slot = m.recv_row ? kWinBytes : (m.recv_slot ? m.recv_slot : m.sample_bytes);
    if (m.kind == 0) {
        *id = m.ids[k];
        *src = m.base + k * m.sample_bytes;
        return;
    }
    const uint32_t* list = m.list_off ? m.list + *m.list_off : m.list;
    const uint32_t kept = m.kept_dev ? *m.kept_dev : m.kept;
    const uint64_t s = list[k];
    *id = s;
    if (m.recv_idx) {  // regular scheme over NCCL
        const uint32_t ri = m.recv_idx[k];
        if (ri == 0xFFFFFFFFu) {  // not received: own shard, or storage tier when uncached
            if (s >= m.cached && m.storage) {
                *src = m.storage + (s - m.cached) * m.sample_bytes;
                if (far) *far = true;
            } else {
                *src = m.shard + (s - m.shard_first) * m.sample_bytes;
            }
        } else {
            *src = m.recv + static_cast<uint64_t>(ri) * slot;
            if (win) *win = m.recv_row != 0 || m.recv_slot != 0;
        }
        return;
    }
    if (s >= m.cached && m.storage) {
        // storage tier (alpha < 1): uncached samples from mapped pinned host memory
        *src = m.storage + (s - m.cached) * m.sample_bytes;
        if (far) *far = true;
        LL_DCHECK(!m.storage_end || *src + m.sample_bytes <= m.storage_end);
    } else if (k < kept) {
        LL_DCHECK(s >= m.shard_first && s < m.cached);
        *src = m.shard + (m.prefix ? m.prefix[s] - m.prefix[m.shard_first]
                                   : (s - m.shard_first) * m.sample_bytes);
        LL_DCHECK(!m.shard_end || m.prefix || *src + m.sample_bytes <= m.shard_end);
        LL_DCHECK(!m.shard_end || !m.prefix || *src + (m.prefix[s + 1] - m.prefix[s]) <= m.shard_end);
    } else if (m.peers) {
        const uint32_t o = static_cast<uint32_t>(s * m.p / m.cached);
        const uint64_t first = (static_cast<uint64_t>(o) * m.cached + m.p - 1) / m.p;
        *src = m.peers[o] + (m.prefix ? m.prefix[s] - m.prefix[first] : (s - first) * m.sample_bytes);
        if (far) *far = true;
        if (peer) *peer = true;
    } else {
        *src = m.recv + (k - kept) * slot;
        if (win) *win = m.recv_row != 0 || m.recv_slot != 0;
    }
}

// Packed fp32x2 helpers (FADD2 / FMUL2 on sm_100): two IEEE-rounded ops per
// instruction, bit-identical to the scalar sequence.
__device__ __forceinline__ uint64_t pk(uint32_t lo, uint32_t hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
    return r;
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint32_t lo32(uint64_t v) { return static_cast<uint32_t>(v); }
__device__ __forceinline__ uint32_t hi32(uint64_t v) { return static_cast<uint32_t>(v >> 32); }

// float(byte j of w) - 2^23 == byte exactly: PRMT builds 0x4B0000bb (2^23 + bb).
template <int J>
__device__ __forceinline__ uint32_t magic_byte(uint32_t w) {
    return __byte_perm(w, 0x4B000000u, 0x7440u | static_cast<uint32_t>(J));
}

// Two output pixels (same channel): ((float(v) - mean255) * inv_std255) each.
__device__ __forceinline__ uint64_t norm2(uint32_t m0, uint32_t m1, uint64_t mean2,
                                          uint64_t inv2) {
    const uint64_t big = 0x4B0000004B000000ull;  // {2^23, 2^23}
    return mul2(sub2(sub2(pk(m0, m1), big), mean2), inv2);
}

__device__ __forceinline__ uint32_t bf16x2(uint64_t v) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo32(v)), __uint_as_float(hi32(v)));
    return *reinterpret_cast<const uint32_t*>(&h);
}

// One thread's share of one output row: PX consecutive output pixels of all
// three planes.  `row` holds the crop row's source bytes from a0 (16-byte
// aligned) on; `base` is the byte offset of the lowest source pixel of the
// run.  The 3*PX source bytes are fetched as 32-bit words (4 or 7 LDS) and
// realigned with funnel shifts (the shift is uniform per sample); each byte
// becomes a float through PRMT + exact subtraction, and the normalisation
// runs on packed fp32x2 -- no I2F, same IEEE results as the oracle.
template <bool BF16, bool FLIP>
__device__ __forceinline__ void emit_run(const uint8_t* row, int32_t base, uint64_t const* mean2,
                                         uint64_t const* inv2, void* out, uint64_t o,
                                         uint64_t plane) {
    constexpr int PX = BF16 ? 8 : 4;
    constexpr int NB = 3 * PX;      // 12 or 24 source bytes
    constexpr int NW = NB / 4 + 1;  // words covering them at any alignment
    LL_DCHECK(base >= 0);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(row) + (base >> 2);
    const uint32_t sh = 8u * static_cast<uint32_t>(base & 3);
    uint32_t raw[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) raw[i] = w[i];
    uint32_t by[NB / 4];
#pragma unroll
    for (int i = 0; i < NB / 4; ++i) by[i] = __funnelshift_r(raw[i], raw[i + 1], sh);
    auto mb = [&](int j) -> uint32_t {
        const uint32_t x = by[j >> 2];
        switch (j & 3) {
            case 0: return magic_byte<0>(x);
            case 1: return magic_byte<1>(x);
            case 2: return magic_byte<2>(x);
            default: return magic_byte<3>(x);
        }
    };
    uint64_t v[3][PX / 2];
#pragma unroll
    for (int u = 0; u < PX; u += 2) {
        const int p0 = FLIP ? (PX - 1 - u) : u;
        const int p1 = FLIP ? (PX - 2 - u) : u + 1;
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c][u / 2] = norm2(mb(3 * p0 + c), mb(3 * p1 + c), mean2[c], inv2[c]);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        if constexpr (BF16) {
            st_cs_v4(static_cast<uint16_t*>(out) + o + c * plane,
                     make_uint4(bf16x2(v[c][0]), bf16x2(v[c][1]), bf16x2(v[c][2]),
                                bf16x2(v[c][3])));
        } else {
            st_cs_v4(static_cast<float*>(out) + o + c * plane,
                     make_uint4(lo32(v[c][0]), hi32(v[c][0]), lo32(v[c][1]), hi32(v[c][1])));
        }
    }
}

// Rows [r_first, r_first + kBand) of the band: thread (tr, tq) writes pixel run
// tq of rows tr, tr + PX, ...
// phase (ROW16 = false): byte r of it is where source row r's data starts in
// its smem row (the row was staged from the 16-byte-aligned address at or
// below its window start); null when every row starts aligned.
template <bool BF16>
__device__ __forceinline__ void emit_band(const uint8_t* rows, uint32_t pitch, const Params& q,
                                          uint32_t a0, uint64_t k, uint32_t band,
                                          const NormConst& nc, void* out,
                                          const uint8_t* phase = nullptr) {
    constexpr uint32_t PX = BF16 ? 8 : 4;
    constexpr uint32_t TPR = kOut / PX;
    const uint32_t tr = threadIdx.x / TPR, tq = threadIdx.x - tr * TPR;
    const uint64_t plane = static_cast<uint64_t>(kOut) * kOut;
    const uint64_t obase = k * 3 * plane + static_cast<uint64_t>(band * kBand) * kOut + tq * PX;
    const int32_t base = q.flip ? static_cast<int32_t>(3 * (q.x0 + kOut - PX - tq * PX)) -
                                      static_cast<int32_t>(a0)
                                : static_cast<int32_t>(3 * (q.x0 + tq * PX)) -
                                      static_cast<int32_t>(a0);
    uint64_t mean2[3], inv2[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        mean2[c] = pk(__float_as_uint(nc.mean255[c]), __float_as_uint(nc.mean255[c]));
        inv2[c] = pk(__float_as_uint(nc.inv_std255[c]), __float_as_uint(nc.inv_std255[c]));
    }
#pragma unroll 1
    for (uint32_t rr = 0; rr < kBand / PX; ++rr) {
        const uint32_t r = rr * PX + tr;
        const uint64_t o = obase + static_cast<uint64_t>(r) * kOut;
        const int32_t b = phase ? base + phase[r] : base;
        if (q.flip)
            emit_run<BF16, true>(rows + r * pitch, b, mean2, inv2, out, o, plane);
        else
            emit_run<BF16, false>(rows + r * pitch, b, mean2, inv2, out, o, plane);
    }
}

// PX output pixels per thread: 4 (fp32, one float4 per plane) or 8 (bf16,
// eight bf16 per plane).  kThreads/(224/PX) = PX rows per pass.
// ROW16: source rows are a multiple of 16 bytes (256-px ImageNet shapes), so
// every window row starts at the same 16-byte phase; otherwise (e.g. a
// 250-px source, 750-byte rows) each row is staged from the aligned address
// below its own window start and keeps its phase in s_phase.
template <bool BF16, bool ROW16 = true>
// (measured: 4 resident CTAs per SM at 72 registers beat forcing 5-9 by
// register caps or a larger shared-memory carveout; profiles/r01_augment_ab.md)
// bf16 (half the stores of fp32) runs best at 5 resident CTAs / SM (48
// registers): 12.95 M vs 12.79 M samples/s; fp32 keeps 4 (profiles/r2_k6_occupancy.md)
__global__ void __launch_bounds__(kThreads, BF16 ? 5 : 1) k_augment_crop(AugArgs a) {
    __shared__ __align__(128) uint8_t rows[kBandSmem];
    __shared__ uint8_t s_phase[kBand];
    __shared__ const uint8_t* s_src;
    __shared__ Params s_prm;
    __shared__ uint64_t s_k;
    __shared__ __align__(8) uint64_t s_mbar;
    __shared__ uint32_t s_host, s_win;

    const uint64_t kb = blockIdx.x / kBands;
    const uint32_t band = blockIdx.x - static_cast<uint32_t>(kb) * kBands;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        // received samples (list tail [kept, n): peer HBM over NVLink) are
        // scheduled first, so their longer reads overlap the local ones
        // instead of forming the grid's tail; the output slot stays k
        uint64_t k = kb;
        if (a.src.kind == 1) {
            const uint64_t kept = a.src.kept_dev ? *a.src.kept_dev : a.src.kept;
            const uint64_t nr = kept < a.n ? a.n - kept : 0;
            // (interleaving them evenly over the grid instead measured equal:
            // cfg4 over P2P at N = 2, profiles/r2_nvlink_modes.txt)
            k = kb < nr ? kept + kb : kb - nr;
        }
        s_k = k;
        uint64_t id;
        const uint8_t* src;
        bool far = false, win = false, peer = false;
        resolve(a.src, k, &id, &src, &far, &win, &peer);
        s_src = src;
        s_win = win;
        s_host = far ? (peer ? 2u : 1u) : 0u;  // peer shard (NVLink) or host storage tier (PCIe)
        if (s_host) {  // the band comes by TMA (below); waited on after the barrier
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar)))
                         : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        if (a.src.aug) {  // precomputed by the plan (assign.cu crop_params)
            const uint32_t* ap = a.src.list_off ? a.src.aug + *a.src.list_off : a.src.aug;
            const uint32_t w = ap[k];
            s_prm = Params{w & 0x7FFFu, (w >> 15) & 0xFFFFu, kOut, kOut, w >> 31};
        } else {
            s_prm = aug_params(a.seed, a.epoch, id, a.H, a.W, kOut, kOut, LL_AUG_CROP);
        }
    }
    __syncthreads();
    const Params q = s_prm;
    const uint8_t* src = s_src;
    const uint64_t k = s_k;
    // a received crop window (NCCL slot) holds exactly the spans read below
    const bool win = s_win != 0;
    const uint32_t row_bytes = win ? kWinRow : a.W * 3;
    const uint32_t a0 = (3 * q.x0) & ~15u;
    const uint32_t nch0 = (((3 * q.x0 + 3 * kOut) + 15u) & ~15u) / 16 - a0 / 16;
    const uint8_t* gbase = win ? src + static_cast<uint64_t>(band * kBand) * kWinRow
                               : src + static_cast<uint64_t>(q.y0 + band * kBand) * row_bytes + a0;
    // unaligned rows: row r is read from the aligned address below its
    // window start, one more chunk when the phase pushes the span over
    constexpr bool kAligned = ROW16;
    const bool per_row = !kAligned && !win;
    auto row_src = [&](uint32_t r) -> const uint8_t* {
        const uint8_t* g = gbase + static_cast<uint64_t>(r) * row_bytes;
        return per_row ? reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(g) &
                                                          ~static_cast<uintptr_t>(15))
                       : g;
    };
    const uint32_t nch = per_row ? nch0 + 1 : nch0;  // <= 44 chunks = kRowSmem
    LL_DCHECK(nch * 16 <= kRowSmem);
    // peer sample whose band span fits: one bulk request (kBandSmem above)
    const bool span = s_host == 2u && !per_row && !win && row_bytes % 16 == 0 &&
                      (kBand - 1) * row_bytes + nch * 16 <= kBandSmem;
    LL_DCHECK(win || (q.y0 + kOut <= a.H && q.x0 + kOut <= a.W));
    if (per_row && tid < kBand)
        s_phase[tid] = static_cast<uint8_t>(
            reinterpret_cast<uintptr_t>(gbase + static_cast<uint64_t>(tid) * row_bytes) & 15);
    if (s_host) {
        // far samples (host storage tier, peer shards): the band's 32 row
        // segments as TMA bulk copies instead of 16-byte loads (cfg3: 0.78 ->
        // 0.82 of the measured pinned H2D bandwidth; cfg4 at N = 4: +3 %)
        const uint32_t mb = static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar));
        if (tid == 0) {
            const uint32_t dst0 = static_cast<uint32_t>(__cvta_generic_to_shared(rows));
            if (span) {  // peer: the band's rows as one contiguous request
                const uint32_t bytes = (kBand - 1) * row_bytes + nch * 16;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                             "r"(bytes)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst0),
                    "l"(row_src(0)), "r"(bytes), "r"(mb)
                    : "memory");
            } else {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                             "r"(kBand * nch * 16)
                             : "memory");
                for (uint32_t r = 0; r < kBand; ++r)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst0 + r * kRowSmem),
                        "l"(row_src(r)), "r"(nch * 16), "r"(mb)
                        : "memory");
            }
        }
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(mb)
                : "memory");
        }
    } else {
        // every load of the band in flight at once: slot t -> (row t/44, chunk t%44)
        constexpr uint32_t kSlots = kRowSmem / 16;  // 44 >= 43 chunks per row
        constexpr uint32_t kIters = (kBand * kSlots + kThreads - 1) / kThreads;
        uint4 v[kIters];
#pragma unroll
        for (uint32_t i = 0; i < kIters; ++i) {
            const uint32_t t = tid + i * kThreads, r = t / kSlots, c = t - r * kSlots;
            if (r < kBand && c < nch) v[i] = ld_nc_v4(row_src(r) + 16 * c);
        }
#pragma unroll
        for (uint32_t i = 0; i < kIters; ++i) {
            const uint32_t t = tid + i * kThreads, r = t / kSlots, c = t - r * kSlots;
            if (r < kBand && c < nch) *reinterpret_cast<uint4*>(&rows[r * kRowSmem + 16 * c]) = v[i];
        }
    }
    __syncthreads();

    emit_band<BF16>(rows, span ? row_bytes : kRowSmem, q, a0, k, band, a.nc, a.out,
                    per_row ? s_phase : nullptr);
}

// ---- K7: fixed-point bilinear resize (cfg5) ------------------------------
// Semantics (oracle lo_resize_tap / lo_augment_one):
// source positions in 1/128 px with half-pixel centres; each tap weight is a
// product of 7-bit axis weights, so per channel
//   v = sum (128-wy | wy) * (128-wx | wx) * p      (exact integer < 2^22)
//   out = (v * 2^-14 - mean255) * inv_std255.
// On the device the horizontal pair of taps of one source row is one DP2A
// (two u16 weights x two u8 pixels), the vertical weight is folded into the
// packed u16 weight pair (lanes <= 128*128, no carry), and v * 2^-14 is
// exact through the magic float 0x44000000 | v (= 512 + v * 2^-14): the
// whole tap arithmetic runs on the integer pipes and no float rounding
// happens before the normalisation.

// U = uint32_t when (2*n_out+1)*extent*64 < 2^32 (the banded kernel; host
// checked), else uint64_t: the same floor either way.
template <typename U = uint64_t>
__device__ __forceinline__ void resize_tap(uint32_t o, uint32_t n_out, uint32_t extent,
                                           uint32_t* lo, uint32_t* w) {
    const int64_t f = static_cast<int64_t>((static_cast<U>(2 * o + 1) * extent * 64) / n_out) - 64;
    uint32_t l = 0, ww = 0;
    if (f > 0) {
        l = static_cast<uint32_t>(f >> 7);
        ww = static_cast<uint32_t>(f & 127);
    }
    if (l >= extent - 1) {
        l = extent - 1;
        ww = 0;
    }
    *lo = l;
    *w = ww;
}

// The tap sums start from this accumulator: 0x44000000 + v == 0x44000000 | v
// (v < 2^22), the magic float 512 + v * 2^-14, with no separate OR.
constexpr uint32_t kMagic14 = 0x44000000u;

// v * 2^-14 as an exact float (v < 2^22)
__device__ __forceinline__ float fixed14(uint32_t v) {
    return __fsub_rn(__uint_as_float(0x44000000u | v), 512.0f);
}

// K7 generic: one CTA per (sample, output row), scalar; used outside the
// banded kernel's limits (out_w > 512, sources of 2 GiB+ or under 2 x 2).
template <bool BF16>
__global__ void __launch_bounds__(256) k_augment_resize(AugArgs a) {
    const uint64_t k = blockIdx.x / a.out_h;
    const uint32_t oy = blockIdx.x - static_cast<uint32_t>(k) * a.out_h;
    __shared__ const uint8_t* s_src;
    __shared__ Params s_prm;
    if (threadIdx.x == 0) {
        uint64_t id;
        const uint8_t* src;
        resolve(a.src, k, &id, &src);
        s_src = src;
        s_prm = aug_params(a.seed, a.epoch, id, a.H, a.W, a.out_h, a.out_w, LL_AUG_RESIZE);
    }
    __syncthreads();
    const Params q = s_prm;
    uint32_t ylo, wy;
    resize_tap(oy, a.out_h, q.ch, &ylo, &wy);
    const uint32_t yhi = wy ? ylo + 1 : ylo;
    const uint8_t* r0 = s_src + static_cast<uint64_t>(q.y0 + ylo) * a.W * 3;
    const uint8_t* r1 = s_src + static_cast<uint64_t>(q.y0 + yhi) * a.W * 3;
    const uint64_t plane = static_cast<uint64_t>(a.out_h) * a.out_w;
    for (uint32_t ox = threadIdx.x; ox < a.out_w; ox += blockDim.x) {
        uint32_t xlo, wx;
        resize_tap(q.flip ? a.out_w - 1 - ox : ox, a.out_w, q.cw, &xlo, &wx);
        const uint64_t pa = static_cast<uint64_t>(q.x0 + xlo) * 3, pb = wx ? pa + 3 : pa;
        const uint32_t w00 = (128 - wx) * (128 - wy), w01 = wx * (128 - wy);
        const uint32_t w10 = (128 - wx) * wy, w11 = wx * wy;
#pragma unroll
        for (uint32_t c = 0; c < 3; ++c) {
            const uint32_t v = w00 * r0[pa + c] + w01 * r0[pb + c] + w10 * r1[pa + c] +
                               w11 * r1[pb + c];
            const float o = __fmul_rn(__fsub_rn(fixed14(v), a.nc.mean255[c]), a.nc.inv_std255[c]);
            const uint64_t idx = k * 3 * plane + c * plane + static_cast<uint64_t>(oy) * a.out_w + ox;
            if constexpr (BF16)
                static_cast<__nv_bfloat16*>(a.out)[idx] = __float2bfloat16_rn(o);
            else
                static_cast<float*>(a.out)[idx] = o;
        }
    }
}

constexpr uint32_t kMaxOutW = 512;

// Per-sample prologue of K7, one thread per sample (the RNG chains -- source
// geometry, crop origin, flip -- and the source resolve run once per sample
// instead of once per band CTA).
struct ResizeItem {
    const uint8_t* src;   // what K7 reads (the pulled copy for far samples)
    uint32_t pitch;       // row pitch in bytes: var_pitch(W) (variable), 3W (fixed)
    Params q;
    const uint8_t* from;  // far samples: 16-byte aligned start of the rows to pull
    uint8_t* to;          // ... their pull slot in local HBM
    uint32_t bytes16;     // ... and their length (multiple of 16), else 0
};

// Far samples (peer shard / host storage) are pulled into local HBM before K7:
// K7's 4-byte tap gathers are cheap from L1/L2 but one NVLink or PCIe round
// trip each from a far source, while the pull moves the crop window's rows in
// coalesced 16-byte loads.  `pull` = nullptr: no far sources in this launch.
__global__ void k_resize_prep(AugArgs a, ResizeItem* __restrict__ items, uint64_t n,
                              uint8_t* __restrict__ pull, uint64_t pull_stride,
                              uint32_t* __restrict__ far_list, uint32_t* __restrict__ far_count) {
    const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (k >= n) return;
    uint64_t id;
    ResizeItem it;
    bool far = false, win = false;
    resolve(a.src, k, &id, &it.src, &far, &win);
    uint32_t H = a.H, W = a.W;
    if (a.src.prefix) var_hw(a.src.data_seed, id, &H, &W);
    it.pitch = a.src.prefix ? var_pitch(W) : 3 * W;
    it.q = aug_params(a.seed, a.epoch, id, H, W, a.out_h, a.out_w, LL_AUG_RESIZE);
    LL_DCHECK(it.q.y0 + it.q.ch <= H && it.q.x0 + it.q.cw <= W && 3 * W <= it.pitch);
    // a received resize window (NCCL): row y0 sits at byte kRecvPad of the slot
    if (win) it.src = it.src + kRecvPad - static_cast<uint64_t>(it.q.y0) * it.pitch;
    it.from = nullptr;
    it.to = nullptr;
    it.bytes16 = 0;
    if (far && pull) {
        // the window's full rows [y0, y0 + ch), widened to 16-byte alignment,
        // into pull slot j (compact: the pull kernel walks far samples only)
        const uint64_t row = it.pitch;
        const uintptr_t start = reinterpret_cast<uintptr_t>(it.src) + it.q.y0 * row;
        const uintptr_t end = start + it.q.ch * row;
        const uintptr_t a16 = start & ~static_cast<uintptr_t>(15);
        const uint32_t j = atomicAdd(far_count, 1u);
        far_list[j] = static_cast<uint32_t>(k);
        uint8_t* dst = pull + j * pull_stride;
        it.to = dst;
        it.from = reinterpret_cast<const uint8_t*>(a16);
        it.bytes16 = static_cast<uint32_t>(((end + 15) & ~static_cast<uintptr_t>(15)) - a16);
        it.src = dst + (start - a16) - it.q.y0 * row;  // same row indexing as the original
    }
    items[k] = it;
}

// Grid-stride over (far sample, 16 KB unit) pairs: every load of a unit is in
// flight at once (4 x 16 B per thread), so a step's few far samples cost about
// one NVLink / PCIe round trip instead of one per 4 KB.
constexpr uint32_t kPullUnit = 16384;
constexpr uint32_t kPullCtas = 296;  // 2 per SM

__global__ void __launch_bounds__(256) k_resize_pull(const ResizeItem* __restrict__ items,
                                                     const uint32_t* __restrict__ far_list,
                                                     const uint32_t* __restrict__ far_count,
                                                     uint32_t units_per_sample) {
    const uint64_t units = static_cast<uint64_t>(*far_count) * units_per_sample;
    for (uint64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const uint32_t j = static_cast<uint32_t>(u / units_per_sample);
        const uint32_t b0 = static_cast<uint32_t>(u - static_cast<uint64_t>(j) * units_per_sample) *
                            kPullUnit;
        const ResizeItem& it = items[far_list[j]];
        if (b0 >= it.bytes16) continue;
        const uint32_t b1 = b0 + kPullUnit < it.bytes16 ? b0 + kPullUnit : it.bytes16;
        uint4 v[4];
#pragma unroll
        for (uint32_t i = 0; i < 4; ++i) {
            const uint32_t o = b0 + 16 * (i * blockDim.x + threadIdx.x);
            if (o < b1) v[i] = ld_nc_v4(it.from + o);
        }
#pragma unroll
        for (uint32_t i = 0; i < 4; ++i) {
            const uint32_t o = b0 + 16 * (i * blockDim.x + threadIdx.x);
            if (o < b1) *reinterpret_cast<uint4*>(it.to + o) = v[i];
        }
    }
}

// bytes [s, s+4) of the 8-byte pair {hi:lo} (s = sel & 3)
__device__ __forceinline__ uint32_t f4e(uint32_t lo, uint32_t hi, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32.f4e %0, %1, %2, %3;" : "=r"(r) : "r"(lo), "r"(hi), "r"(sel));
    return r;
}

__device__ __forceinline__ void st_cs_f32(float* p, float v) {
    asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_cs_u16(void* p, uint16_t v) {
    asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p), "h"(v) : "memory");
}

// K7 banded: one CTA per (sample, kRB output rows), one thread per output
// column, walking the band two rows at a time (the pair is one fp32x2).  The
// taps are 32-bit read-only loads straight from the source rows; at CTA start
// the band's source rows are bulk-prefetched into L2 (a per-iteration L1
// prefetch on top of that measured slower, profiles/r05_k7_ab.md).  No shared-memory staging:
// occupancy is not bound by the largest (512 px) source, and the A/B against
// a staged-smem band kernel (profiles/r03_k7_ab.md) favoured the gathers.
// Only words holding needed bytes are read: a far-edge column (wx = 0) taps
// pixels (xlo-1, xlo) with weights (0, 128), and the third word is loaded
// only when tap b spills into it.
constexpr uint32_t kRB = 16;
__device__ __forceinline__ void row_taps_g(const uint8_t* base, uint32_t off, uint32_t* rg,
                                           uint32_t* bb) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(base + (off & ~3u));
    const uint32_t w0 = __ldg(p), w1 = __ldg(p + 1);
    const uint32_t w2 = (off & 3u) == 3u ? __ldg(p + 2) : 0u;
    const uint32_t ta = f4e(w0, w1, off), tb = f4e(w1, w2, off);  // [Ra Ga Ba Rb] [Gb Bb - -]
    *rg = __byte_perm(ta, tb, 0x4130);
    *bb = __byte_perm(ta, tb, 0x0052);
}

__device__ __forceinline__ void bilerp_g(const uint8_t* base, uint32_t x3, uint32_t colw,
                                         const uint4& r, uint32_t v[3]) {
    uint32_t rg0, b0, rg1, b1;
    row_taps_g(base, r.x + x3, &rg0, &b0);
    row_taps_g(base, r.y + x3, &rg1, &b1);
    const uint32_t w0 = colw * r.z, w1 = colw * r.w;  // two u16 lanes each, no carry
    v[0] = __dp2a_lo(w0, rg0, __dp2a_lo(w1, rg1, kMagic14));
    v[1] = __dp2a_hi(w0, rg0, __dp2a_hi(w1, rg1, kMagic14));
    v[2] = __dp2a_lo(w0, b0, __dp2a_lo(w1, b1, kMagic14));
}

// Word-aligned rows (variable geometry, var_pitch): `p` = the 4-byte aligned
// word holding tap a's first byte, `sel` = its byte phase, both per-column
// constants.  The third word is read unconditionally (its bytes only matter
// when sel = 3); shards and pull slots carry 16 bytes of tail slack for it.
__device__ __forceinline__ void row_taps_a(const uint8_t* p, uint32_t sel, uint32_t* rg,
                                           uint32_t* bb) {
    const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
    const uint32_t w0 = __ldg(q), w1 = __ldg(q + 1), w2 = __ldg(q + 2);
    const uint32_t ta = f4e(w0, w1, sel), tb = f4e(w1, w2, sel);  // [Ra Ga Ba Rb] [Gb Bb - -]
    *rg = __byte_perm(ta, tb, 0x4130);
    *bb = __byte_perm(ta, tb, 0x0052);
}

__device__ __forceinline__ void bilerp_a(const uint8_t* colp, uint32_t sel, uint32_t colw,
                                         const uint4& r, uint32_t v[3]) {
    uint32_t rg0, b0, rg1, b1;
    row_taps_a(colp + r.x, sel, &rg0, &b0);
    row_taps_a(colp + r.y, sel, &rg1, &b1);
    const uint32_t w0 = colw * r.z, w1 = colw * r.w;  // two u16 lanes each, no carry
    v[0] = __dp2a_lo(w0, rg0, __dp2a_lo(w1, rg1, kMagic14));
    v[1] = __dp2a_hi(w0, rg0, __dp2a_hi(w1, rg1, kMagic14));
    v[2] = __dp2a_lo(w0, b0, __dp2a_lo(w1, b1, kMagic14));
}

// ALIGNED (word-aligned rows and sample starts): the row table holds the row
// starts and each column keeps one pointer and byte phase, so a tap costs one
// 64-bit add, three loads and four byte permutes.
// OUT = 224 fixes the output geometry at compile time (cfg5), so all six
// stores of a row pair address off one pointer with immediate offsets.
template <bool BF16, bool ALIGNED, uint32_t OUT = 0>
__global__ void __launch_bounds__(kMaxOutW) k_augment_resize_rows(AugArgs a,
                                                                  const ResizeItem* items) {
    // {lo row offset, hi row offset, 128-wy, wy}; offsets from s_base, which is
    // the sample start (ALIGNED) or the sample start rounded down to 4 bytes
    // with the crop origin and the phase folded into the offsets
    __shared__ uint4 s_row[kRB];
    __shared__ const uint8_t* s_base;
    __shared__ Params s_q;
    const uint64_t k = blockIdx.x;  // sample
    const uint32_t oy0 = blockIdx.y * kRB;
    const uint32_t rows_out = a.out_h - oy0 < kRB ? a.out_h - oy0 : kRB;
    const uint32_t tid = threadIdx.x;
    if (tid < rows_out) {
        const ResizeItem it = items[k];
        const uint32_t phase = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(it.src) & 3);
        uint32_t ylo, wy;
        resize_tap<uint32_t>(oy0 + tid, OUT ? OUT : a.out_h, it.q.ch, &ylo, &wy);
        const uint32_t yhi = wy ? ylo + 1 : ylo;
        if (ALIGNED)
            s_row[tid] = make_uint4((it.q.y0 + ylo) * it.pitch, (it.q.y0 + yhi) * it.pitch,
                                    128 - wy, wy);
        else
            s_row[tid] = make_uint4(phase + (it.q.y0 + ylo) * it.pitch + it.q.x0 * 3,
                                    phase + (it.q.y0 + yhi) * it.pitch + it.q.x0 * 3, 128 - wy,
                                    wy);
        if (tid == 0) {
            s_base = it.src - phase;  // phase = 0 when ALIGNED
            s_q = it.q;
        }
    }
    __syncthreads();
    const Params q = s_q;
    const uint8_t* base = s_base;
    {
        // the band's source rows (crop span) head for L2 at once: every
        // thread prefetches about two 128-byte lines of the band's lo / hi
        // rows before any tap (K7 138 -> 123 us; per-thread line prefetches,
        // as the bulk prefetch takes uniform operands and serialises).
        // Item j = (output row j / 32, lo line j % 16 or hi line when bit 4
        // is set): shifts, no divisions (a row span has <= 13 lines)
        const uint32_t lines = (3 * q.cw + 127) / 128 + 1;  // per row span, any alignment
        const uint32_t xo = ALIGNED ? 3 * q.x0 : 0;
        const uint32_t span_last = 3 * q.cw - 1;
        for (uint32_t j = tid; j < 32 * rows_out; j += blockDim.x) {
            const uint32_t r = j >> 5, l = j & 15;
            const uint4 e = s_row[r];
            const bool hi = (j & 16) != 0;
            if (l >= lines || (hi && e.w == 0)) continue;  // wy = 0: no hi row
            const uint32_t in = 128 * l < span_last ? 128 * l : span_last;  // stay in the span
            const uint32_t off = (hi ? e.y : e.x) + xo + in;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(base + off));
        }
    }
    if (tid >= a.out_w) return;  // no barrier follows
    const uint32_t ox = tid;
    uint32_t xlo, wx;
    resize_tap<uint32_t>(q.flip ? a.out_w - 1 - ox : ox, OUT ? OUT : a.out_w, q.cw, &xlo, &wx);
    uint32_t x3 = 3 * xlo, colw = (128 - wx) | (wx << 16);
    if (wx == 0 && xlo > 0) {  // taps (xlo-1, xlo) weighted (0, 128): no read past xlo
        x3 -= 3;
        colw = 128u << 16;
    }
    // ALIGNED: this column's tap-a word in row 0 and its byte phase
    const uint32_t xb = 3 * q.x0 + x3;
    const uint8_t* colp = base + (xb & ~3u);
    const uint32_t sel = xb & 3u;
    uint64_t mean2[3], inv2[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        mean2[c] = pk(__float_as_uint(a.nc.mean255[c]), __float_as_uint(a.nc.mean255[c]));
        inv2[c] = pk(__float_as_uint(a.nc.inv_std255[c]), __float_as_uint(a.nc.inv_std255[c]));
    }
    const uint64_t k512 = 0x4400000044000000ull;  // {512, 512}
    using T = typename std::conditional<BF16, __nv_bfloat16, float>::type;
    const uint32_t ow = OUT ? OUT : a.out_w;
    const uint64_t plane = static_cast<uint64_t>(OUT ? OUT : a.out_h) * ow;
    auto bilerp = [&](const uint4& r, uint32_t v[3]) {
        if constexpr (ALIGNED)
            bilerp_a(colp, sel, colw, r, v);
        else
            bilerp_g(base, x3, colw, r, v);
    };
    T* pc[3];
    pc[0] = static_cast<T*>(a.out) + k * 3 * plane + static_cast<uint64_t>(oy0) * ow + ox;
    pc[1] = pc[0] + plane;
    pc[2] = pc[1] + plane;
    auto emit = [&](const uint32_t* v0, const uint32_t* v1, bool two) {
#pragma unroll
        for (uint32_t c = 0; c < 3; ++c) {
            const uint64_t m = pk(v0[c], v1[c]);  // already 0x44000000 + v
            const uint64_t o = mul2(sub2(sub2(m, k512), mean2[c]), inv2[c]);
            T* pt = OUT ? pc[0] + c * plane : pc[c];
            if constexpr (BF16) {
                const uint32_t h = bf16x2(o);
                st_cs_u16(pt, static_cast<uint16_t>(h));
                if (two) st_cs_u16(pt + ow, static_cast<uint16_t>(h >> 16));
            } else {
                st_cs_f32(pt, __uint_as_float(lo32(o)));
                if (two) st_cs_f32(pt + ow, __uint_as_float(hi32(o)));
            }
            if (!OUT) pc[c] += 2 * ow;
        }
        if (OUT) pc[0] += 2 * ow;
    };
    uint32_t rr = 0;
#pragma unroll(OUT ? 2 : 1)
    for (; rr + 1 < rows_out; rr += 2) {
        uint32_t v0[3], v1[3];
        bilerp(s_row[rr], v0);
        bilerp(s_row[rr + 1], v1);
        emit(v0, v1, true);
    }
    if (rr < rows_out) {  // odd band height
        uint32_t v0[3];
        bilerp(s_row[rr], v0);
        emit(v0, v0, false);
    }
}

__global__ void k_aug_params(uint64_t seed, uint64_t epoch, const uint64_t* __restrict__ ids,
                             uint64_t n, uint32_t H, uint32_t W, uint32_t out_h, uint32_t out_w,
                             int mode, uint32_t* __restrict__ out5) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const Params q = aug_params(seed, epoch, ids[i], H, W, out_h, out_w, mode);
    out5[5 * i + 0] = q.y0;
    out5[5 * i + 1] = q.x0;
    out5[5 * i + 2] = q.ch;
    out5[5 * i + 3] = q.cw;
    out5[5 * i + 4] = q.flip;
}

} // namespace

NormConst norm_constants(const ll_augment_spec& s) {
    NormConst c;
    for (int i = 0; i < 3; ++i) {
        c.mean255[i] = static_cast<float>(s.mean[i] * 255.0);
        c.inv_std255[i] = static_cast<float>(1.0 / (s.std[i] * 255.0));
    }
    return c;
}

static void validate_spec(const ll_augment_spec& spec, uint32_t H, uint32_t W) {
    require(spec.out_dtype == LL_OUT_F32 || spec.out_dtype == LL_OUT_BF16,
            "augment: out_dtype must be fp32 or bf16");
    if (spec.mode == LL_AUG_CROP) {
        require(spec.out_h == kOut && spec.out_w == kOut, "augment: crop output must be 224x224");
        require(H >= kOut && W >= kOut, "augment: source smaller than the crop");

    } else {
        require(spec.mode == LL_AUG_RESIZE, "augment: unknown mode");
        require(spec.out_h >= 1 && spec.out_w >= 1 && H >= 1 && W >= 1,
                "augment: empty geometry");
    }
}

static AugArgs make_args(const ll_augment_spec& spec, uint64_t seed, uint64_t epoch,
                         const SrcMap& src, uint64_t n, uint32_t height, uint32_t width,
                         void* d_out) {
    AugArgs a{};
    a.src = src;
    a.H = height;
    a.W = width;
    a.seed = seed;
    a.epoch = epoch;
    a.nc = norm_constants(spec);
    a.out = d_out;
    a.n = n;
    a.out_h = spec.out_h;
    a.out_w = spec.out_w;
    return a;
}

// The banded resize kernel's limits: 32-bit in-sample offsets, exact 32-bit
// taps, sources of at least 2 x 2 (a tap pair never leaves the sample).
// *max_bytes: the largest source sample.
static bool resize_banded(const ll_augment_spec& spec, const SrcMap& src, uint32_t height,
                          uint32_t width, uint64_t* max_bytes) {
    const uint32_t max_side = src.prefix ? kVarMin + kVarSpan - 1 : std::min(height, width);
    *max_bytes =
        src.prefix ? 3ull * (kVarMin + kVarSpan) * (kVarMin + kVarSpan) : 3ull * height * width;
    const uint64_t tap_max = (2ull * std::max(spec.out_h, spec.out_w) + 1) * 64 * max_side;
    return spec.out_w <= kMaxOutW && tap_max < (1ull << 32) && *max_bytes < (1ull << 31) &&
           (src.prefix || std::min(height, width) >= 2);
}

bool resize_prepare(ll_ctx* ctx, const ll_augment_spec& spec, uint64_t seed, uint64_t epoch,
                    const SrcMap& src, uint64_t n, uint32_t height, uint32_t width, int slot,
                    const std::string& owner) {
    validate_spec(spec, height, width);
    uint64_t max_bytes = 0;
    if (spec.mode != LL_AUG_RESIZE || n == 0 || !resize_banded(spec, src, height, width, &max_bytes))
        return false;
    require(n < (1ull << 31), "augment: too many samples in one launch");
    const std::string tag = owner + std::to_string(slot);
    const AugArgs a = make_args(spec, seed, epoch, src, n, height, width, nullptr);
    DevBuf& items = ctx->buf("resize.items" + tag, sizeof(ResizeItem) * n);
    // far sources possible: peer shards (P2P) or the host storage tier
    const bool far = src.kind == 1 && (src.peers != nullptr || src.storage != nullptr);
    const uint64_t pull_stride = (max_bytes + 15) / 16 * 16 + 64;
    uint8_t* pull = nullptr;
    uint32_t* fl = nullptr;
    if (far) {
        pull = ctx->buf("resize.pull" + tag, n * pull_stride).as<uint8_t>();
        fl = ctx->buf("resize.far" + tag, sizeof(uint32_t) * (n + 1)).as<uint32_t>();
        LL_CUDA(cudaMemsetAsync(fl + n, 0, sizeof(uint32_t), ctx->stream));
    }
    launch(ctx, "resize_prep", [&] {
        k_resize_prep<<<static_cast<unsigned>((n + 127) / 128), 128, 0, ctx->stream>>>(
            a, items.as<ResizeItem>(), n, pull, pull_stride, fl, fl ? fl + n : nullptr);
    });
    if (far) {
        const uint32_t units = static_cast<uint32_t>((max_bytes + 32 + kPullUnit - 1) / kPullUnit);
        launch(ctx, "resize_pull", [&] {
            k_resize_pull<<<kPullCtas, 256, 0, ctx->stream>>>(items.as<ResizeItem>(), fl, fl + n,
                                                              units);
        });
    }
    return true;
}

void augment_device(ll_ctx* ctx, const ll_augment_spec& spec, uint64_t seed, uint64_t epoch,
                    const SrcMap& src, uint64_t n, uint32_t height, uint32_t width, void* d_out,
                    int prepared_slot, const std::string& owner) {
    validate_spec(spec, height, width);
    if (n == 0) return;
    const AugArgs a = make_args(spec, seed, epoch, src, n, height, width, d_out);
    const bool bf16 = spec.out_dtype == LL_OUT_BF16;
    if (spec.mode == LL_AUG_CROP) {
        const dim3 grid(static_cast<unsigned>(n * kBands));
        // sources whose rows (and samples) are 16-byte multiples keep one
        // phase for every row; others (e.g. 250 px wide) stage per row
        const bool row16 = (3ull * width) % 16 == 0 &&
                           (src.kind != 0 || (reinterpret_cast<uintptr_t>(src.base) & 15) == 0);
        launch(ctx, "augment_crop", [&] {
            if (bf16 && row16)
                k_augment_crop<true, true><<<grid, kThreads, 0, ctx->stream>>>(a);
            else if (row16)
                k_augment_crop<false, true><<<grid, kThreads, 0, ctx->stream>>>(a);
            else if (bf16)
                k_augment_crop<true, false><<<grid, kThreads, 0, ctx->stream>>>(a);
            else
                k_augment_crop<false, false><<<grid, kThreads, 0, ctx->stream>>>(a);
        });
        return;
    }
    uint64_t max_bytes = 0;
    if (resize_banded(spec, src, height, width, &max_bytes)) {
        // the prologue (K7 prep + far pull) ran already (the loader prefetches
        // it on its side stream into sets 0/1) or runs now into set 2
        int slot = prepared_slot;
        std::string who = owner;
        if (slot < 0) {  // inline: on the context stream, so one set serves every caller
            who.clear();
            resize_prepare(ctx, spec, seed, epoch, src, n, height, width, 2, who);
            slot = 2;
        }
        const ResizeItem* it = ctx->buf("resize.items" + who + std::to_string(slot),
                                        sizeof(ResizeItem) * n).as<ResizeItem>();
        const dim3 grid(static_cast<unsigned>(n), (spec.out_h + kRB - 1) / kRB);
        const unsigned threads = 32 * ((spec.out_w + 31) / 32);
        // word-aligned rows: the variable-geometry shard layout (geometry.cuh)
        const bool aligned = src.prefix != nullptr;
        const bool out224 = spec.out_h == 224 && spec.out_w == 224;
        launch(ctx, "augment_resize", [&] {
            if (bf16 && aligned && out224)
                k_augment_resize_rows<true, true, 224><<<grid, threads, 0, ctx->stream>>>(a, it);
            else if (!bf16 && aligned && out224)
                k_augment_resize_rows<false, true, 224><<<grid, threads, 0, ctx->stream>>>(a, it);
            else if (bf16 && aligned)
                k_augment_resize_rows<true, true><<<grid, threads, 0, ctx->stream>>>(a, it);
            else if (bf16)
                k_augment_resize_rows<true, false><<<grid, threads, 0, ctx->stream>>>(a, it);
            else if (aligned)
                k_augment_resize_rows<false, true><<<grid, threads, 0, ctx->stream>>>(a, it);
            else
                k_augment_resize_rows<false, false><<<grid, threads, 0, ctx->stream>>>(a, it);
        });
        return;
    }
    require(src.prefix == nullptr, "augment: variable geometry needs the banded resize kernel");
    const dim3 grid(static_cast<unsigned>(n * spec.out_h));
    launch(ctx, "augment_resize", [&] {
        if (bf16)
            k_augment_resize<true><<<grid, 256, 0, ctx->stream>>>(a);
        else
            k_augment_resize<false><<<grid, 256, 0, ctx->stream>>>(a);
    });
}

void augment_params_device(ll_ctx* ctx, const ll_augment_spec& spec, uint64_t seed,
                           uint64_t epoch, const uint64_t* d_ids, uint64_t n, uint32_t height,
                           uint32_t width, uint32_t* d_params5) {
    validate_spec(spec, height, width);
    if (n == 0) return;
    launch(ctx, "aug_params", [&] {
        k_aug_params<<<static_cast<unsigned>((n + 127) / 128), 128, 0, ctx->stream>>>(
            seed, epoch, d_ids, n, height, width, spec.out_h, spec.out_w, spec.mode, d_params5);
    });
}

} // namespace ll
