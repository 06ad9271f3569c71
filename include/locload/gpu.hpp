// locload/gpu.hpp -- the device extension of the loader API.
//
// The reference Loader (proj/include/locload/pipeline.hpp:106-123) hands host
// SampleBytes to a BatchConsumer.  On B200 each learner's cache is an HBM
// shard and the consumer is a training step on the same GPU, so the batch
// stays in device memory: DeviceLoader::run_epoch calls the consumer once per
// step, in step order, with this learner's augmented NCHW batch (device
// pointer, valid until prefetch_depth further steps were issued) and the
// stream it was produced on.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "locload/core.hpp"
#include "locload_b200.h"

namespace locload {
namespace gpu {

struct DeviceBatch {
    std::uint64_t epoch = 0;
    std::uint64_t step = 0;
    std::uint64_t size = 0;          // samples in this learner's list
    std::uint64_t local = 0;         // of which served from its own shard
    std::uint64_t received = 0;      // of which fetched from other learners
    const void* data = nullptr;      // [size][3][out_h][out_w] fp32 or bf16
    const std::uint32_t* ids = nullptr;  // [size] sample ids (device)
    std::uintptr_t stream = 0;       // cudaStream_t the batch was produced on
};

using DeviceBatchConsumer = std::function<void(const DeviceBatch&)>;

struct EpochReport {  // ThroughputReport (pipeline.hpp:55-64) for a device consumer
    std::uint64_t epoch = 0;
    std::uint64_t batches = 0;
    std::uint64_t samples = 0;
    std::uint64_t cache_hits = 0;    // served from the local HBM shard
    std::uint64_t cache_misses = 0;  // moved in from other learners
    double wall_s = 0;
    double samples_per_second = 0;
};

class DeviceLoader {
public:
    // cfg as in include/locload_b200.h; throws std::invalid_argument with the
    // reference's messages for bad configurations.
    DeviceLoader(const ll_loader_config& cfg, int device = 0);
    ~DeviceLoader();
    DeviceLoader(const DeviceLoader&) = delete;
    DeviceLoader& operator=(const DeviceLoader&) = delete;

    void populate();                                       // synthesize the shard in HBM
    void populate_from_host(const std::uint8_t* samples);  // owned_count x sample_bytes
    std::vector<std::uint8_t> ipc_handle();                // P2P bootstrap (64 B)
    void open_peers(const std::vector<std::uint8_t>& handles);  // p x 64 B
    void comm_init(const std::vector<std::uint8_t>& nccl_id);   // 128 B
    static std::vector<std::uint8_t> nccl_unique_id();
    static void link_peers(const std::vector<DeviceLoader*>& same_process_learners);

    std::uint64_t steps_per_epoch() const;
    DeviceBatch step(std::uint64_t epoch, std::uint64_t step);
    EpochReport run_epoch(std::uint64_t epoch, const DeviceBatchConsumer& consumer = {});
    void synchronize();

    ll_loader* handle() const { return ld_; }

private:
    ll_ctx* ctx_ = nullptr;
    ll_loader* ld_ = nullptr;
};

} // namespace gpu
} // namespace locload
