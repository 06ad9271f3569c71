// ll_internal.h -- context, errors and kernel-launch bookkeeping shared by the
// translation units behind include/locload_b200.h.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "locload_b200.h"

namespace ll {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool ok, const std::string& msg) {
    if (!ok) fail(LL_ERR_INVALID, msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(LL_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define LL_CUDA(x) ::ll::cuda_check((x), #x)

// Device-side bounds / invariant checks, compiled in only for the checked
// variant library (-DLL_CHECKED, scripts/checked_build.py): compute-sanitizer
// is closed on this GPU pool, so the test suite runs against that build
// instead (profiles/r2_sanitize/).  A failed check prints and traps.
#ifdef LL_CHECKED
#define LL_DCHECK(c)                                                                     \
    do {                                                                                 \
        if (!(c)) {                                                                      \
            printf("LL_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
                   #c, static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));      \
            __trap();                                                                    \
        }                                                                                \
    } while (0)
#else
#define LL_DCHECK(c) \
    do {             \
    } while (0)
#endif

// Device buffer with grow-only reallocation.
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    bool borrowed = false;  // memory owned elsewhere (NCCL-registered): never freed here
    void reserve(size_t n) {
        if (n <= bytes) return;
        if (ptr && !borrowed) cudaFree(ptr);
        borrowed = false;
        ptr = nullptr;
        bytes = 0;
        LL_CUDA(cudaMalloc(&ptr, n));
        bytes = n;
    }
    // step-path check: buffers sized up front must never grow there (a
    // cudaFree + cudaMalloc synchronises the device mid-step)
    void need(size_t n, const char* what) const {
        if (n > bytes)
            fail(LL_ERR_RUNTIME, std::string("loader: ") + what + " needs " + std::to_string(n) +
                                     " bytes but holds " + std::to_string(bytes) +
                                     " (preallocated at setup; never grown on the step path)");
    }
    template <typename T>
    T* as() const { return static_cast<T*>(ptr); }
    void release() {
        if (ptr && !borrowed) cudaFree(ptr);
        borrowed = false;
        ptr = nullptr;
        bytes = 0;
    }
    ~DevBuf() { release(); }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

struct PlanBufs;

struct KernelTimes {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
    uint64_t launches = 0;
    double total_ms = 0;
};

} // namespace ll

struct ll_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t stream = nullptr;
    uint64_t launches = 0;
    bool timing = false;
    std::map<std::string, ll::KernelTimes> times;
    std::vector<cudaEvent_t> event_pool;
    // named device scratch buffers (grow-only), e.g. "perm.J"
    std::map<std::string, std::unique_ptr<ll::DevBuf>> scratch;
    ll::DevBuf& buf(const std::string& name, size_t bytes) {
        auto& p = scratch[name];
        if (!p) p.reset(new ll::DevBuf());
        p->reserve(bytes);
        return *p;
    }
    cudaEvent_t take_event();
    // single-step plan of the stateless ll_assign entry point
    std::unique_ptr<ll::PlanBufs> api_plan;
};

namespace ll {

// cudaFuncSetAttribute is per device: set a kernel's dynamic shared-memory
// limit once per (kernel, device).
template <typename K>
void ensure_smem_attr(K kernel, int device, size_t bytes) {
    static std::map<std::pair<const void*, int>, size_t> done;
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    auto& v = done[{reinterpret_cast<const void*>(kernel), device}];
    if (v >= bytes) return;
    cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(bytes)),
               "cudaFuncSetAttribute");
    v = bytes;
}

// Every kernel launch of the library goes through here: counts it, and when
// timing is on brackets it with events on the context stream.
template <typename F>
void launch(ll_ctx* ctx, const char* name, F&& f) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (ctx->timing) {
        a = ctx->take_event();
        b = ctx->take_event();
        LL_CUDA(cudaEventRecord(a, ctx->stream));
    }
    f();
    LL_CUDA(cudaGetLastError());
    ctx->launches++;
    if (ctx->timing) {
        LL_CUDA(cudaEventRecord(b, ctx->stream));
        ctx->times[name].pending.emplace_back(a, b);
    }
}

void set_device(ll_ctx* ctx);
// capi.cu: u64 ids -> u32 on ctx->stream
void narrow_device(ll_ctx* ctx, const uint64_t* in, uint32_t* out, uint64_t n);

// permute.cu: full permutation of [0,d) into d_order (u32), on ctx->stream.
// `tag` names the scratch buffers (independent permutations may be in flight
// on different streams of one context, e.g. the loader's next-epoch plan)
void permute_device(ll_ctx* ctx, uint64_t seed, uint64_t epoch, uint32_t d, uint32_t* d_order,
                    const uint64_t* host_forced, uint64_t n_forced, const char* tag = "perm");
uint32_t permute_rounds(ll_ctx* ctx, const char* tag = "perm");
void permute_profile(ll_ctx* ctx, uint64_t* out6, const char* tag = "perm");

// assign.cu
constexpr uint32_t kMaxP = 64;
struct PlanDev {
    uint32_t* final_ids = nullptr;  // [steps][B]
    uint32_t* off = nullptr;        // [steps][kMaxP+1]
    uint32_t* kept = nullptr;       // [steps][kMaxP]
    uint32_t* counts = nullptr;     // [steps][kMaxP]
    ll_move* moves = nullptr;       // [steps][kMaxP]
    uint32_t* n_moves = nullptr;    // [steps]
    uint32_t* stats = nullptr;      // [steps][4]: moved, nvlink, uncached, reg_remote
    uint32_t* scratch = nullptr;    // [steps][B]
    uint32_t* aug = nullptr;        // [steps][B] packed crop params per final slot (or null)
    // regular scheme with the NCCL exchange (or null): [steps][p][p] samples
    // of slice j owned by learner o at [j * p + o]
    uint32_t* regcnt = nullptr;
};
// Crop parameters the plan precomputes for every final slot (crop mode):
// packed y0 | x0 << 15 | flip << 31 (lo_aug_params_for).
struct AugPlan {
    bool enabled = false;
    uint64_t seed = 0, epoch = 0;
    uint32_t H = 0, W = 0, ch = 0, cw = 0;
};
struct PlanBufs {
    DevBuf final_ids, off, kept, counts, moves, n_moves, stats, scratch, aug, regcnt;
    PlanDev view() const;
    void reserve(uint64_t steps, uint64_t B);
    void reserve_regcnt(uint64_t steps, uint32_t p);
};
void assign_device(ll_ctx* ctx, const uint32_t* d_order, uint64_t steps, uint64_t B, uint32_t p,
                   uint64_t cached, int scheme, const PlanDev& plan,
                   const AugPlan& aug = AugPlan());
void balance_device(ll_ctx* ctx, const int64_t* d_counts, const int64_t* d_targets, uint32_t p,
                    uint64_t n, ll_move* d_moves, uint32_t* d_n);

// shard.cu
void generate_range_device(ll_ctx* ctx, uint8_t* dst, uint64_t first_id, uint64_t n,
                           uint64_t sample_bytes, uint64_t data_seed);
void generate_ids_device(ll_ctx* ctx, uint8_t* dst, const uint64_t* d_ids, uint64_t n,
                         uint64_t sample_bytes, uint64_t data_seed);
// variable geometry (geometry.cuh): d_prefix[0..d] = exclusive prefix of padded sizes
void var_prefix_device(ll_ctx* ctx, uint64_t* d_prefix, uint64_t d, uint64_t data_seed);
void generate_var_device(ll_ctx* ctx, uint8_t* shard, uint64_t first, uint64_t n,
                         const uint64_t* d_prefix, uint64_t data_seed);

// augment.cu
struct NormConst {
    float mean255[3];
    float inv_std255[3];
};
NormConst norm_constants(const ll_augment_spec& s);

// Where output sample k of a launch reads its source bytes from.
struct SrcMap {
    int kind = 0;                      // 0 explicit, 1 plan
    // explicit (tests): src = base + k * sample_bytes, id = ids[k]
    const uint8_t* base = nullptr;
    const uint64_t* ids = nullptr;
    // plan: id = list[k]; k < kept -> own shard, else remote
    const uint32_t* list = nullptr;
    const uint32_t* list_off = nullptr;  // if set: list += *list_off (device)
    uint32_t kept = 0;
    const uint32_t* kept_dev = nullptr;  // if set: kept = *kept_dev (device)
    const uint32_t* aug = nullptr;       // plan-precomputed crop params, list-aligned
    const uint8_t* shard = nullptr;
    const uint8_t* shard_end = nullptr;    // checked builds: the shard's last byte + 1
    const uint8_t* storage_end = nullptr;  // ... and the storage tier's
    uint64_t shard_first = 0;
    const uint8_t* recv = nullptr;     // NCCL path: received samples in list order
    const uint8_t* const* peers = nullptr;  // P2P path: every learner's shard
    uint32_t p = 1;
    uint64_t cached = 0;
    uint64_t sample_bytes = 0;
    // variable geometry (cfg5): offsets from the global padded-size prefix,
    // geometry from the id (geometry.cuh); recv/explicit paths need fixed size
    const uint64_t* prefix = nullptr;
    uint64_t data_seed = 0;
    // storage tier (alpha < 1): sample s >= cached at storage + (s - cached) * bytes,
    // a mapped pinned host buffer read over PCIe / C2C by the kernel itself
    const uint8_t* storage = nullptr;
    // regular scheme over NCCL: list position -> recv index (0xFFFFFFFF: own shard)
    const uint32_t* recv_idx = nullptr;
    // NCCL receive slots hold crop windows (kWinRows rows at recv_row pitch,
    // from the 16-byte-aligned window start) when recv_row != 0, else samples
    uint32_t recv_row = 0;
    // resize mode over NCCL: slots of recv_slot bytes, each holding a sample's
    // resize window -- its source rows [y0, y0 + ch) at the sample's pitch,
    // from byte kRecvPad of the slot (0: slots hold whole samples)
    uint64_t recv_slot = 0;
};
constexpr uint32_t kRecvPad = 16;
// NCCL messages carry a crop-mode sample as its crop window only: 224 rows of
// the 16-byte-aligned span holding its 672 window bytes (<= 704 bytes), not
// the whole 196,608-byte sample
constexpr uint32_t kWinRows = 224;
constexpr uint32_t kWinRow = 704;
constexpr uint64_t kWinBytes = static_cast<uint64_t>(kWinRows) * kWinRow;
// prepared_slot >= 0: the resize prologue already ran into buffer set
// (owner, prepared_slot)
void augment_device(ll_ctx* ctx, const ll_augment_spec& spec, uint64_t seed, uint64_t epoch,
                    const SrcMap& src, uint64_t n, uint32_t height, uint32_t width, void* d_out,
                    int prepared_slot = -1, const std::string& owner = std::string());
// Resize prologue (per-sample geometry, far-sample pull) into buffer set
// (owner, slot) on ctx->stream; false when the step has no banded-resize
// prologue.  Work on a stream other than the context's needs an owner name
// of its own: loaders sharing a device share its context and scratch.
bool resize_prepare(ll_ctx* ctx, const ll_augment_spec& spec, uint64_t seed, uint64_t epoch,
                    const SrcMap& src, uint64_t n, uint32_t height, uint32_t width, int slot,
                    const std::string& owner = std::string());
void augment_params_device(ll_ctx* ctx, const ll_augment_spec& spec, uint64_t seed,
                           uint64_t epoch, const uint64_t* d_ids, uint64_t n, uint32_t height,
                           uint32_t width, uint32_t* d_params5);

// exchange.cu
std::vector<ll_xfer> exchange_plan(const ll_move* moves, uint32_t n, const uint32_t* off,
                                   uint32_t me);
std::vector<ll_xfer> exchange_plan(const ll_move* moves, uint32_t n, const uint64_t* off,
                                   uint32_t me);
// regular scheme over NCCL: pack this learner's samples of other slices into
// [p][B/p] messages, and map its own slice positions to receive indices
// (0xFFFFFFFF = own shard)
// d_aug (or null): the plan's packed crop parameters of the step, aligned with
// d_batch / d_final_step; with it each message slot carries only the sample's
// crop window (kWinBytes; image rows of row_bytes), else the whole sample
void reg_prep_device(ll_ctx* ctx, const uint32_t* d_batch, const uint32_t* d_scratch,
                     const uint32_t* d_regcnt, uint32_t p, uint32_t me, uint64_t B,
                     const uint8_t* shard, uint64_t shard_first, uint64_t sample_bytes,
                     uint8_t* pack, uint32_t* ridx, const uint32_t* d_aug, uint32_t row_bytes);
// resize-mode messages: each slot carries the sample's resize window (rows
// [y0, y0 + ch) at its pitch, from byte kRecvPad); the geometry and crop
// origin come from the id, as in K7's prologue
struct ResizeWin {
    bool enabled = false;
    uint64_t seed = 0, epoch = 0, data_seed = 0;
    const uint64_t* prefix = nullptr;  // variable geometry (else fixed H x W)
    uint32_t H = 0, W = 0, out_h = 0, out_w = 0;
    uint64_t slot = 0;                 // message slot bytes
};
// the largest resize window (+ pad and tail slack), per message slot
uint64_t resize_slot_bytes(bool variable, uint32_t H, uint32_t W);
// sends: (list_first, count) runs of the step's final ids, packed contiguously
void pack_device(ll_ctx* ctx, const std::vector<ll_xfer>& xfers, const uint32_t* d_final_step,
                 const uint8_t* shard, uint64_t shard_first, uint64_t sample_bytes,
                 uint8_t* packbuf, const uint32_t* d_aug, uint32_t row_bytes,
                 const ResizeWin& rw = ResizeWin());

// train.cu: consumer side (equivalence.cpp:95-205) on the device
void train_run_device(ll_ctx* ctx, const double* h_xs, const double* h_ys, uint64_t n,
                      uint32_t dims, int scheme, uint32_t p, uint64_t B, uint64_t steps,
                      uint64_t seed, double lr, int aggregation, double* h_final_w,
                      double* h_step_grads);
void toy_grads_device(ll_ctx* ctx, const double* X, const double* Y, uint32_t dims,
                      const double* w, const int64_t* ids, uint64_t n_ids, double* G);
void ordered_sum_device(ll_ctx* ctx, const double* G, uint64_t n, uint32_t dims,
                        const int64_t* order, double* out);
void sgd_apply_device(ll_ctx* ctx, const double* gsum, uint32_t dims, double scale, double lr,
                      double* w, double* step_grad);
void full_batch_gradient_device(ll_ctx* ctx, const double* h_xs, const double* h_ys, uint64_t n,
                                uint32_t dims, const double* h_w, const uint64_t* h_batch,
                                uint64_t B, double* h_grad);

} // namespace ll
