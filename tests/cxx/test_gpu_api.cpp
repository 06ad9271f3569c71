// C++ API of the device loader (include/locload/gpu.hpp): two same-process
// learners linked over P2P, one epoch through run_epoch with a device
// consumer, checked against the core/sampling/balance API of the same
// library (which the reference suites test separately).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <vector>

#include "locload/balance.hpp"
#include "locload/core.hpp"
#include "locload/gpu.hpp"
#include "locload/pipeline.hpp"
#include "locload/sampling.hpp"

using namespace locload;

namespace {
ll_loader_config config(std::uint32_t rank) {
    ll_loader_config c{};
    c.d = 4096;
    c.height = 256;
    c.width = 256;
    c.learners = 2;
    c.rank = rank;
    c.batch_size = 256;
    c.alpha = 1.0;
    c.seed = 42;
    c.data_seed = 42;
    c.scheme = LL_SCHEME_LOCALITY_BALANCED;
    c.exchange = LL_EXCHANGE_P2P;
    c.prefetch_depth = 2;
    c.augment.mode = LL_AUG_CROP;
    c.augment.out_dtype = LL_OUT_F32;
    c.augment.out_h = c.augment.out_w = 224;
    const double mean[3] = {0.485, 0.456, 0.406}, stdv[3] = {0.229, 0.224, 0.225};
    for (int i = 0; i < 3; ++i) {
        c.augment.mean[i] = mean[i];
        c.augment.std[i] = stdv[i];
    }
    return c;
}
} // namespace

TEST_CASE("device loader delivers the balanced locality lists in step order") {
    gpu::DeviceLoader a(config(0)), b(config(1));
    a.populate();
    b.populate();
    gpu::DeviceLoader::link_peers({&a, &b});
    REQUIRE(a.steps_per_epoch() == 16);
    const auto plan = batches(permute_epoch(42, 3, 4096), 256);
    const CacheDirectory dir(4096, 2, 1.0);
    std::uint64_t expected_step = 0;
    ll_ctx* host_copy = nullptr;
    REQUIRE(ll_ctx_create(&host_copy, 0) == LL_OK);
    const gpu::EpochReport rep = a.run_epoch(3, [&](const gpu::DeviceBatch& batch) {
        CHECK(batch.step == expected_step);
        // learner 0's list: its cached samples then balance-moved ones
        LocDistribution dist = loc_distribution(plan[batch.step], dir);
        ImbalanceVector iv;
        iv.counts.assign(dist.counts.begin(), dist.counts.end());
        iv.targets = targets(256, 2);
        const TransferSchedule s = balance(iv);
        std::vector<SampleId> mine = dist.assignments[0].samples;
        for (const Move& m : s.moves) {
            auto& from = dist.assignments[m.sender].samples;
            if (m.receiver == 0) mine.insert(mine.end(), from.end() - m.count, from.end());
            if (m.sender == 0) mine.resize(mine.size() - m.count);
        }
        std::vector<std::uint32_t> got(batch.size);
        REQUIRE(ll_ctx_copy_to_host(host_copy, got.data(),
                                    reinterpret_cast<std::uintptr_t>(batch.ids),
                                    4 * batch.size) == LL_OK);
        REQUIRE(got.size() == mine.size());
        for (std::size_t i = 0; i < got.size(); ++i) CHECK(got[i] == mine[i]);
        CHECK(batch.local + batch.received == batch.size);
        ++expected_step;
    });
    ll_ctx_destroy(host_copy);
    CHECK(rep.batches == 16);
    CHECK(rep.samples == 16 * 128);
    CHECK(rep.cache_hits + rep.cache_misses == rep.samples);
    CHECK(rep.cache_misses > 0);
}

TEST_CASE("device loader rejects bad configurations with the reference messages") {
    ll_loader_config c = config(0);
    c.alpha = 0.0;
    CHECK_THROWS_WITH_AS(gpu::DeviceLoader{c}, doctest::Contains("cached fraction"),
                         std::invalid_argument);
    c = config(0);
    c.batch_size = 5000;
    CHECK_THROWS_WITH_AS(gpu::DeviceLoader{c}, doctest::Contains("batches: batch size"),
                         std::invalid_argument);
}

TEST_CASE("SampleCache holds its payloads in HBM: first touch, no replacement, host copies") {
    SampleCache cache(2);
    auto make = [](std::uint8_t v, std::size_t n) {
        return std::make_shared<const std::vector<std::uint8_t>>(n, v);
    };
    const std::size_t S = 3 * 250 * 250;  // not a multiple of 16
    cache.insert(7, make(1, S));
    cache.insert(9, make(2, S));
    cache.insert(7, make(3, S));  // already held: not replaced
    cache.insert(11, make(4, S));  // over capacity: skipped
    CHECK(cache.size() == 2);
    CHECK(cache.capacity() == 2);
    const SampleBytes a = cache.find(7), b = cache.find(9), c = cache.find(11);
    REQUIRE(a != nullptr);
    REQUIRE(b != nullptr);
    CHECK(c == nullptr);
    CHECK(*a == std::vector<std::uint8_t>(S, 1));
    CHECK(*b == std::vector<std::uint8_t>(S, 2));
}
