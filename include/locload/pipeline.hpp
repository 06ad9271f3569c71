// locload/pipeline.hpp -- source-compatible drop-in for
// proj/include/locload/pipeline.hpp (the reference's file-per-sample dataset,
// sample cache and concurrent epoch loader), backed by this library:
//   * generate_dataset computes the sample bytes on the GPU (K1, the
//     reference's byte formula, pipeline.cpp:208-234) and writes the same
//     %08llu.bin files;
//   * Loader::run_epoch takes its order from the device permutation (K2+K3)
//     and keeps the reference's delivery contract -- prefetch_depth batches
//     in flight over `workers` loader threads, intra_batch_parallelism sample
//     tasks per batch, in-order delivery to the consumer on the calling
//     thread, every thread joined before it returns or throws;
//   * SampleCache holds its payloads in HBM (include/locload_b200.h
//     ll_store_*): misses are read from the files (read_sample's error text)
//     and copied in, hits are gathered back by one device gather per batch.
// A consumer that wants the batch on the GPU, augmented, uses
// locload/gpu.hpp's DeviceLoader instead; this header keeps the reference's
// host SampleBytes so existing consumers relink unchanged.
#pragma once

#include <cstdint>
#include <filesystem>
#include <functional>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "locload/core.hpp"

struct ll_store;

namespace locload {

// pipeline.hpp:18 -- one sample's bytes, shared between cache and consumer
using SampleBytes = std::shared_ptr<const std::vector<std::uint8_t>>;

// pipeline.hpp:22-26 -- n files of sample_bytes bytes each under root
struct DatasetSpec {
    std::filesystem::path root;
    std::uint64_t n = 0;
    std::uint64_t sample_bytes = 0;
};

// pipeline.hpp:28 -- root / "%08llu.bin"
std::filesystem::path sample_path(const DatasetSpec& spec, SampleId id);

// pipeline.hpp:32 -- writes the n files; byte-identical for equal (spec, seed).
// std::invalid_argument for n == 0 or sample_bytes == 0.
void generate_dataset(const DatasetSpec& spec, std::uint64_t seed);

// pipeline.hpp:34-38 -- injected per-sample preprocessing cost
struct PreprocessSpec {
    enum class Mode { none, spin, sleep };
    Mode mode = Mode::none;
    std::uint64_t micros_per_sample = 0;
};

// pipeline.hpp:40-44
struct CacheSpec {
    enum class Mode { off, memory };
    Mode mode = Mode::off;
    std::uint64_t capacity_samples = 0;
};

// pipeline.hpp:46-53 -- batch_size is the GLOBAL batch
struct LoaderConfig {
    std::uint32_t workers = 1;
    std::uint32_t intra_batch_parallelism = 1;
    std::uint32_t prefetch_depth = 1;
    std::uint64_t batch_size = 1;
    PreprocessSpec preprocess;
    CacheSpec cache;
};

// pipeline.hpp:55-64
struct ThroughputReport {
    std::uint64_t epoch = 0;
    std::uint64_t batches = 0;
    std::uint64_t samples = 0;
    double wall_s = 0;
    double samples_per_second = 0;
    std::uint64_t cache_hits = 0;
    std::uint64_t cache_misses = 0;
    std::vector<double> batch_latency_s;  // request -> in-order delivery, per batch
};

// pipeline.hpp:68-94 -- fixed capacity in samples, populate on first touch,
// no replacement, safe for concurrent use.  The payloads are held in HBM on
// the CUDA device current at construction; find() returns a host copy.
class SampleCache {
public:
    explicit SampleCache(std::uint64_t capacity);
    ~SampleCache();
    SampleCache(const SampleCache&) = delete;
    SampleCache& operator=(const SampleCache&) = delete;

    SampleBytes find(SampleId id) const;  // nullptr when not held
    void insert(SampleId id, SampleBytes bytes);
    std::uint64_t size() const;

    std::uint64_t capacity() const { return capacity_; }
    ll_store* handle() const { return store_; }

private:
    std::uint64_t capacity_;
    ll_store* store_ = nullptr;
};

// pipeline.hpp:97-98 -- called once per batch, in step order
using BatchConsumer =
    std::function<void(const GlobalBatch&, const std::vector<SampleBytes>&)>;

// pipeline.hpp:106-123
class Loader {
public:
    // std::invalid_argument unless workers, parallelism, prefetch and batch
    // size are all >= 1 (pipeline.cpp:237-241)
    Loader(DatasetSpec spec, LoaderConfig cfg);

    // Every full batch of permute_epoch(seed, epoch, n), in step order.  A
    // missing or truncated file raises std::runtime_error("sample <id>: ...").
    ThroughputReport run_epoch(std::uint64_t seed, std::uint64_t epoch,
                               const BatchConsumer& consumer = {});

    const SampleCache* cache() const { return cache_.get(); }

private:
    DatasetSpec spec_;
    LoaderConfig cfg_;
    std::shared_ptr<SampleCache> cache_;
};

// pipeline.hpp:125-128 -- epoch 0 (cold) then epoch 1 (warm) on one cache;
// std::invalid_argument unless the memory cache can hold the whole dataset.
std::pair<ThroughputReport, ThroughputReport>
warm_cache_epoch(const DatasetSpec& spec, const LoaderConfig& cfg, std::uint64_t seed);

} // namespace locload
