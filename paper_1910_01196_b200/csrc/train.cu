// train.cu -- the consumer side of the loader: synchronous
// SGD of p learners fed by the device epoch plan, with the reference's two
// gradient aggregations.  Replaces run_training / full_batch_gradient
// (proj/src/equivalence.cpp:95-174, 190-205) and checks Theorem 1 on the GPU:
// under canonical aggregation regular, locality and balanced locality give
// bit-identical trajectories.
//
// Per run: the toy objective's samples (x_i, y_i) go to HBM once.  Per epoch:
// K2 permutation of [0, n) on the device; canonical aggregation sorts every
// batch window by sample id (one segmented radix sort per epoch), learner-order
// aggregation takes the scheme's final per-learner lists from K4 (the same
// assignment the loader uses).  Per step, two kernels: per-sample gradients
// (one thread per sample) and a per-coordinate sequential sum in the
// reference's order followed by the update w -= lr * g.  Every fp64 op is an
// explicit IEEE-rounded __d*_rn (no FMA contraction), in the reference's
// order, so the trajectory equals the compiled reference bit for bit.
#include <cub/device/device_segmented_radix_sort.cuh>

#include "ll_internal.h"

namespace ll {
namespace {

// G[i][k] = (dot(w, x_s) - y_s) * x_s[k] for s = ids[i]  (equivalence.cpp:52-64)
template <typename Id>
__global__ void k_sample_grads(const double* __restrict__ X, const double* __restrict__ Y,
                               uint32_t dims, const double* __restrict__ w,
                               const Id* __restrict__ ids, uint64_t n_ids,
                               double* __restrict__ G) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n_ids) return;
    const uint64_t s = ids[i];
    const double* x = X + s * dims;
    double dot = 0.0;
    for (uint32_t k = 0; k < dims; ++k) dot = __dadd_rn(dot, __dmul_rn(w[k], x[k]));
    const double r = __dsub_rn(dot, Y[s]);
    double* g = G + i * dims;
    for (uint32_t k = 0; k < dims; ++k) g[k] = __dmul_rn(r, x[k]);
}

// One thread per coordinate.  off == nullptr: canonical (G already in
// ascending-id order, summed in that order, equivalence.cpp:123-139);
// otherwise learner order: per-learner sums over each list, then summed in
// learner order (:140-155).  Then g *= 1/B, step_grad = g, w -= lr * g.
__global__ void k_aggregate_update(const double* __restrict__ G, uint64_t n_ids, uint32_t dims,
                                   const uint32_t* __restrict__ off, uint32_t p, double scale,
                                   double lr, double* __restrict__ w,
                                   double* __restrict__ step_grad) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= dims) return;
    double g = 0.0;
    if (off == nullptr) {
        for (uint64_t i = 0; i < n_ids; ++i) g = __dadd_rn(g, G[i * dims + k]);
    } else {
        for (uint32_t j = 0; j < p; ++j) {
            double ls = 0.0;
            for (uint64_t i = off[j]; i < off[j + 1]; ++i) ls = __dadd_rn(ls, G[i * dims + k]);
            g = __dadd_rn(g, ls);
        }
    }
    g = __dmul_rn(g, scale);
    if (step_grad) step_grad[k] = g;
    w[k] = __dsub_rn(w[k], __dmul_rn(lr, g));
}

// out[k] = sum over i of G[order[i]][k] (order == nullptr: i itself),
// sequentially from 0.0 in that order -- the reference's summation order,
// so a sum split across learners and put back together in the same order is
// bit-identical (equivalence.cpp:132-148).  One thread per coordinate.
__global__ void k_ordered_sum(const double* __restrict__ G, uint64_t n, uint32_t dims,
                              const int64_t* __restrict__ order, double* __restrict__ out) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= dims) return;
    double g = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t r = order ? static_cast<uint64_t>(order[i]) : i;
        g = __dadd_rn(g, G[r * dims + k]);
    }
    out[k] = g;
}

// g *= scale (1/B), step_grad = g, w -= lr * g  (equivalence.cpp:157-166)
__global__ void k_sgd_apply(const double* __restrict__ gsum, uint32_t dims, double scale,
                            double lr, double* __restrict__ w, double* __restrict__ step_grad) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= dims) return;
    const double g = __dmul_rn(gsum[k], scale);
    if (step_grad) step_grad[k] = g;
    w[k] = __dsub_rn(w[k], __dmul_rn(lr, g));
}

__global__ void k_segment_offsets(uint32_t* __restrict__ off, uint64_t segments, uint32_t len) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i <= segments) off[i] = static_cast<uint32_t>(i * len);
}

unsigned blocks(uint64_t n, unsigned t) { return static_cast<unsigned>((n + t - 1) / t); }

} // namespace

void train_run_device(ll_ctx* ctx, const double* h_xs, const double* h_ys, uint64_t n,
                      uint32_t dims, int scheme, uint32_t p, uint64_t B, uint64_t steps,
                      uint64_t seed, double lr, int aggregation, double* h_final_w,
                      double* h_step_grads) {
    const uint64_t spe = n / B;  // steps per epoch (core.cpp:57-73)
    const bool canonical = aggregation == LL_AGG_CANONICAL;
    DevBuf& X = ctx->buf("train.x", sizeof(double) * n * dims);
    DevBuf& Y = ctx->buf("train.y", sizeof(double) * n);
    DevBuf& W = ctx->buf("train.w", sizeof(double) * dims);
    DevBuf& SG = ctx->buf("train.step_grads", sizeof(double) * std::max<uint64_t>(steps, 1) * dims);
    DevBuf& G = ctx->buf("train.g", sizeof(double) * B * dims);
    DevBuf& order = ctx->buf("train.order", sizeof(uint32_t) * n);
    LL_CUDA(cudaMemcpyAsync(X.ptr, h_xs, sizeof(double) * n * dims, cudaMemcpyHostToDevice,
                            ctx->stream));
    LL_CUDA(cudaMemcpyAsync(Y.ptr, h_ys, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    LL_CUDA(cudaMemsetAsync(W.ptr, 0, sizeof(double) * dims, ctx->stream));  // w = 0 (:113)
    // canonical: every batch window of the epoch sorted by id
    DevBuf& sorted = ctx->buf("train.sorted", sizeof(uint32_t) * spe * B);
    DevBuf& segoff = ctx->buf("train.segoff", sizeof(uint32_t) * (spe + 1));
    size_t temp_bytes = 0;
    if (canonical) {
        launch(ctx, "train_segments", [&] {
            k_segment_offsets<<<blocks(spe + 1, 256), 256, 0, ctx->stream>>>(
                segoff.as<uint32_t>(), spe, static_cast<uint32_t>(B));
        });
        LL_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(
            nullptr, temp_bytes, order.as<uint32_t>(), sorted.as<uint32_t>(),
            static_cast<int>(spe * B), static_cast<int>(spe), segoff.as<uint32_t>(),
            segoff.as<uint32_t>() + 1, 0, 32, ctx->stream));
    }
    DevBuf& temp = ctx->buf("train.sort_temp", std::max<size_t>(temp_bytes, 16));
    PlanBufs* plan = nullptr;
    if (!canonical) {
        if (!ctx->api_plan) ctx->api_plan.reset(new PlanBufs());
        plan = ctx->api_plan.get();
        plan->reserve(spe, B);
    }
    const double scale = 1.0 / static_cast<double>(B);  // equivalence.cpp:157
    const unsigned red_threads = dims < 128 ? 32 * ((dims + 31) / 32) : 128;
    uint64_t loaded = ~0ull;
    for (uint64_t t = 0; t < steps; ++t) {
        const uint64_t epoch = t / spe, st = t % spe;
        if (epoch != loaded) {
            permute_device(ctx, seed, epoch, static_cast<uint32_t>(n), order.as<uint32_t>(),
                           nullptr, 0, "train.perm");
            if (canonical) {
                size_t tb = temp.bytes;
                launch(ctx, "train_sort", [&] {
                    LL_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(
                        temp.ptr, tb, order.as<uint32_t>(), sorted.as<uint32_t>(),
                        static_cast<int>(spe * B), static_cast<int>(spe), segoff.as<uint32_t>(),
                        segoff.as<uint32_t>() + 1, 0, 32, ctx->stream));
                });
            } else {
                assign_device(ctx, order.as<uint32_t>(), spe, B, p, n, scheme, plan->view());
            }
            loaded = epoch;
        }
        const uint32_t* ids = canonical ? sorted.as<uint32_t>() + st * B
                                        : plan->view().final_ids + st * B;
        const uint32_t* off = canonical ? nullptr : plan->view().off + st * (kMaxP + 1);
        launch(ctx, "train_grads", [&] {
            k_sample_grads<uint32_t><<<blocks(B, 128), 128, 0, ctx->stream>>>(
                X.as<double>(), Y.as<double>(), dims, W.as<double>(), ids, B, G.as<double>());
        });
        launch(ctx, "train_update", [&] {
            k_aggregate_update<<<blocks(dims, red_threads), red_threads, 0, ctx->stream>>>(
                G.as<double>(), B, dims, off, p, scale, lr, W.as<double>(),
                SG.as<double>() + t * dims);
        });
    }
    LL_CUDA(cudaMemcpyAsync(h_final_w, W.ptr, sizeof(double) * dims, cudaMemcpyDeviceToHost,
                            ctx->stream));
    if (h_step_grads && steps)
        LL_CUDA(cudaMemcpyAsync(h_step_grads, SG.ptr, sizeof(double) * steps * dims,
                                cudaMemcpyDeviceToHost, ctx->stream));
    LL_CUDA(cudaStreamSynchronize(ctx->stream));
}

void full_batch_gradient_device(ll_ctx* ctx, const double* h_xs, const double* h_ys, uint64_t n,
                                uint32_t dims, const double* h_w, const uint64_t* h_batch,
                                uint64_t B, double* h_grad) {
    DevBuf& X = ctx->buf("train.x", sizeof(double) * n * dims);
    DevBuf& Y = ctx->buf("train.y", sizeof(double) * n);
    DevBuf& W = ctx->buf("train.w", sizeof(double) * dims);
    DevBuf& SG = ctx->buf("train.step_grads", sizeof(double) * dims);
    DevBuf& G = ctx->buf("train.g", sizeof(double) * std::max<uint64_t>(B, 1) * dims);
    DevBuf& ids64 = ctx->buf("train.batch64", sizeof(uint64_t) * std::max<uint64_t>(B, 1));
    DevBuf& ids = ctx->buf("train.batch", sizeof(uint32_t) * std::max<uint64_t>(B, 1));
    LL_CUDA(cudaMemcpyAsync(X.ptr, h_xs, sizeof(double) * n * dims, cudaMemcpyHostToDevice,
                            ctx->stream));
    LL_CUDA(cudaMemcpyAsync(Y.ptr, h_ys, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    LL_CUDA(cudaMemcpyAsync(W.ptr, h_w, sizeof(double) * dims, cudaMemcpyHostToDevice,
                            ctx->stream));
    LL_CUDA(cudaMemcpyAsync(ids64.ptr, h_batch, sizeof(uint64_t) * B, cudaMemcpyHostToDevice,
                            ctx->stream));
    narrow_device(ctx, ids64.as<uint64_t>(), ids.as<uint32_t>(), B);
    launch(ctx, "train_grads", [&] {
        k_sample_grads<uint32_t><<<blocks(B, 128), 128, 0, ctx->stream>>>(
            X.as<double>(), Y.as<double>(), dims, W.as<double>(), ids.as<uint32_t>(), B,
            G.as<double>());
    });
    // batch-sequence order (equivalence.cpp:193-199); lr = 0 leaves w untouched
    const unsigned red_threads = dims < 128 ? 32 * ((dims + 31) / 32) : 128;
    launch(ctx, "train_update", [&] {
        k_aggregate_update<<<blocks(dims, red_threads), red_threads, 0, ctx->stream>>>(
            G.as<double>(), B, dims, nullptr, 1, 1.0 / static_cast<double>(B), 0.0,
            W.as<double>(), SG.as<double>());
    });
    LL_CUDA(cudaMemcpyAsync(h_grad, SG.ptr, sizeof(double) * dims, cudaMemcpyDeviceToHost,
                            ctx->stream));
    LL_CUDA(cudaStreamSynchronize(ctx->stream));
}

// ---- consumer steps on caller-owned device buffers (one learner per rank) --
void toy_grads_device(ll_ctx* ctx, const double* X, const double* Y, uint32_t dims,
                      const double* w, const int64_t* ids, uint64_t n_ids, double* G) {
    if (n_ids == 0) return;
    launch(ctx, "train_grads", [&] {
        k_sample_grads<int64_t><<<blocks(n_ids, 128), 128, 0, ctx->stream>>>(X, Y, dims, w, ids,
                                                                             n_ids, G);
    });
}

void ordered_sum_device(ll_ctx* ctx, const double* G, uint64_t n, uint32_t dims,
                        const int64_t* order, double* out) {
    const unsigned t = dims < 128 ? 32 * ((dims + 31) / 32) : 128;
    launch(ctx, "ordered_sum", [&] {
        k_ordered_sum<<<blocks(dims, t), t, 0, ctx->stream>>>(G, n, dims, order, out);
    });
}

void sgd_apply_device(ll_ctx* ctx, const double* gsum, uint32_t dims, double scale, double lr,
                      double* w, double* step_grad) {
    const unsigned t = dims < 128 ? 32 * ((dims + 31) / 32) : 128;
    launch(ctx, "sgd_apply", [&] {
        k_sgd_apply<<<blocks(dims, t), t, 0, ctx->stream>>>(gsum, dims, scale, lr, w, step_grad);
    });
}

} // namespace ll
