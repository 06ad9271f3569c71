// pipeline_api.cpp -- the reference's loader API (include/locload/pipeline.hpp)
// on this library.
//
// Reference behaviour kept (proj/src/pipeline.cpp):
//   * file names and contents of the synthetic dataset (:202-234);
//   * read_sample's error text, "sample <id>: cannot open <path>" and
//     "sample <id>: truncated file <path> (read X of Y bytes)" (:110-126);
//   * the Loader contract (:236-336): prefetch_depth batch requests in
//     flight, `workers` loader threads, each batch split into
//     intra_batch_parallelism contiguous sample tasks, the injected
//     per-sample preprocessing paced against an absolute schedule, delivery
//     in step order on the calling thread, first error rethrown after every
//     thread has joined, per-batch request-to-delivery latency;
//   * the cache's hit/miss accounting and populate-on-first-touch.
// What runs differently:
//   * the epoch order is the device permutation (K2+K3, ll_permute_epoch);
//   * dataset bytes are computed on the device (K1, ll_generate_samples)
//     and written by a pool of writer threads;
//   * the cache's payloads live in HBM (ll_store_*): a batch's misses are
//     copied in with one call, its hits come back with one device gather.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <exception>
#include <fstream>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "api_internal.h"
#include "locload/pipeline.hpp"
#include "locload_b200.h"

namespace locload {
namespace {

using detail::check;
using detail::ctx;
using Clock = std::chrono::steady_clock;

double elapsed_s(Clock::time_point a, Clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
}

int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    return dev;
}

// The injected preprocessing cost of one sample task (PreprocessSpec):
// sample k of the task is due k * micros after the task started, so
// oversleeping one sample is made up on the next.
class InjectedCost {
public:
    explicit InjectedCost(const PreprocessSpec& spec) : spec_(spec), due_(Clock::now()) {}
    void after_sample() {
        if (spec_.mode == PreprocessSpec::Mode::none || spec_.micros_per_sample == 0) return;
        due_ += std::chrono::microseconds(spec_.micros_per_sample);
        if (spec_.mode == PreprocessSpec::Mode::sleep) {
            std::this_thread::sleep_until(due_);
            return;
        }
        while (Clock::now() < due_) {
        }
    }

private:
    PreprocessSpec spec_;
    Clock::time_point due_;
};

SampleBytes read_file(const DatasetSpec& spec, SampleId id) {
    const std::filesystem::path path = sample_path(spec, id);
    std::ifstream in(path, std::ios::binary);
    if (!in)
        throw std::runtime_error("sample " + std::to_string(id) + ": cannot open " +
                                 path.string());
    auto bytes = std::make_shared<std::vector<std::uint8_t>>(spec.sample_bytes);
    in.read(reinterpret_cast<char*>(bytes->data()),
            static_cast<std::streamsize>(spec.sample_bytes));
    const std::uint64_t got = static_cast<std::uint64_t>(in.gcount());
    if (got != spec.sample_bytes)
        throw std::runtime_error("sample " + std::to_string(id) + ": truncated file " +
                                 path.string() + " (read " + std::to_string(got) + " of " +
                                 std::to_string(spec.sample_bytes) + " bytes)");
    return bytes;
}

struct LoadedBatch {
    std::vector<SampleBytes> data;
    std::uint64_t hits = 0, misses = 0;
    std::exception_ptr error;
    bool ready = false;
};

// One batch: T contiguous sample tasks (task 0 on this thread) read the
// misses from their files and pay the injected cost per sample; then the
// misses go into the HBM cache in one insert and the hits come back in one
// gather.
LoadedBatch load_batch(const DatasetSpec& spec, const LoaderConfig& cfg, SampleCache* cache,
                       const GlobalBatch& batch) {
    LoadedBatch r;
    const std::size_t n = batch.samples.size();
    r.data.resize(n);
    std::vector<std::uint8_t> held(n, 0);
    if (cache && n) check(ll_store_lookup(cache->handle(), batch.samples.data(), n, held.data()));
    const std::size_t tasks =
        std::min<std::size_t>(std::max<std::uint32_t>(1, cfg.intra_batch_parallelism), n);
    if (tasks == 0) {
        r.ready = true;
        return r;
    }
    const std::size_t per = (n + tasks - 1) / tasks;
    std::vector<std::exception_ptr> errs(tasks);
    auto task = [&](std::size_t t) {
        try {
            InjectedCost cost(cfg.preprocess);
            for (std::size_t i = t * per; i < std::min(n, (t + 1) * per); ++i) {
                if (!held[i]) r.data[i] = read_file(spec, batch.samples[i]);
                cost.after_sample();
            }
        } catch (...) {
            errs[t] = std::current_exception();
        }
    };
    std::vector<std::thread> helpers;
    for (std::size_t t = 1; t < tasks; ++t) helpers.emplace_back(task, t);
    task(0);
    for (auto& h : helpers) h.join();
    for (auto& e : errs)
        if (e) {
            r.error = e;
            r.ready = true;
            return r;
        }
    try {
        std::vector<SampleId> hit_ids, miss_ids;
        std::vector<const std::uint8_t*> miss_ptrs;
        for (std::size_t i = 0; i < n; ++i) {
            if (held[i]) {
                hit_ids.push_back(batch.samples[i]);
            } else {
                miss_ids.push_back(batch.samples[i]);
                miss_ptrs.push_back(r.data[i]->data());
            }
        }
        r.hits = hit_ids.size();
        r.misses = miss_ids.size();
        if (cache && !miss_ids.empty() && spec.sample_bytes)
            check(ll_store_insert(cache->handle(), ctx(), miss_ids.data(), miss_ids.size(),
                                  spec.sample_bytes, miss_ptrs.data(), nullptr));
        if (!hit_ids.empty()) {
            std::vector<std::uint8_t> buf(hit_ids.size() * spec.sample_bytes);
            check(ll_store_gather(cache->handle(), ctx(), hit_ids.data(), hit_ids.size(),
                                  buf.data()));
            std::size_t k = 0;
            for (std::size_t i = 0; i < n; ++i) {
                if (!held[i]) continue;
                const std::uint8_t* p = buf.data() + k++ * spec.sample_bytes;
                r.data[i] = std::make_shared<const std::vector<std::uint8_t>>(
                    p, p + spec.sample_bytes);
            }
        }
    } catch (...) {
        r.error = std::current_exception();
    }
    r.ready = true;
    return r;
}

} // namespace

// ------------------------------------------------------------------ dataset
std::filesystem::path sample_path(const DatasetSpec& spec, SampleId id) {
    char name[32];
    std::snprintf(name, sizeof(name), "%08llu.bin", static_cast<unsigned long long>(id));
    return spec.root / name;
}

void generate_dataset(const DatasetSpec& spec, std::uint64_t seed) {
    if (spec.n == 0 || spec.sample_bytes == 0)
        throw std::invalid_argument("generate_dataset: need n >= 1 and sample_bytes >= 1");
    std::error_code ec;
    std::filesystem::create_directories(spec.root, ec);
    if (ec)
        throw std::runtime_error("generate_dataset: cannot create " + spec.root.string() +
                                 ": " + ec.message());
    // bytes from the device in chunks of about 256 MiB, written by a thread pool
    const std::uint64_t S = spec.sample_bytes;
    const std::uint64_t chunk = std::max<std::uint64_t>(1, (256ull << 20) / S);
    const unsigned writers =
        std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    std::vector<std::uint8_t> buf;
    std::vector<SampleId> ids;
    for (std::uint64_t first = 0; first < spec.n; first += chunk) {
        const std::uint64_t m = std::min(chunk, spec.n - first);
        ids.resize(m);
        for (std::uint64_t k = 0; k < m; ++k) ids[k] = first + k;
        buf.resize(m * S);
        check(ll_generate_samples(ctx(), seed, ids.data(), m, S, buf.data()));
        std::atomic<std::uint64_t> next{0};
        std::mutex emu;
        std::string failed;
        auto write = [&] {
            for (std::uint64_t k = next++; k < m; k = next++) {
                const std::filesystem::path path = sample_path(spec, first + k);
                std::ofstream out(path, std::ios::binary | std::ios::trunc);
                if (!out.write(reinterpret_cast<const char*>(buf.data() + k * S),
                               static_cast<std::streamsize>(S))) {
                    std::lock_guard<std::mutex> g(emu);
                    if (failed.empty()) failed = path.string();
                    return;
                }
            }
        };
        std::vector<std::thread> pool;
        const unsigned w = static_cast<unsigned>(std::min<std::uint64_t>(writers, m));
        for (unsigned t = 1; t < w; ++t) pool.emplace_back(write);
        write();
        for (auto& t : pool) t.join();
        if (!failed.empty())
            throw std::runtime_error("generate_dataset: write failed for " + failed);
    }
}

// ------------------------------------------------------------------ cache
SampleCache::SampleCache(std::uint64_t capacity) : capacity_(capacity) {
    check(ll_store_create(&store_, current_device(), capacity));
}

SampleCache::~SampleCache() { ll_store_destroy(store_); }

SampleBytes SampleCache::find(SampleId id) const {
    std::uint8_t held = 0;
    check(ll_store_lookup(store_, &id, 1, &held));
    if (!held) return nullptr;
    std::uint64_t S = 0;
    check(ll_store_sample_bytes(store_, &S));
    auto out = std::make_shared<std::vector<std::uint8_t>>(S);
    check(ll_store_gather(store_, ctx(), &id, 1, out->data()));
    return out;
}

void SampleCache::insert(SampleId id, SampleBytes bytes) {
    if (!bytes || bytes->empty()) return;
    const std::uint8_t* p = bytes->data();
    check(ll_store_insert(store_, ctx(), &id, 1, bytes->size(), &p, nullptr));
}

std::uint64_t SampleCache::size() const {
    std::uint64_t n = 0;
    check(ll_store_size(store_, &n));
    return n;
}

// ------------------------------------------------------------------ loader
Loader::Loader(DatasetSpec spec, LoaderConfig cfg) : spec_(std::move(spec)), cfg_(cfg) {
    if (cfg_.workers == 0 || cfg_.intra_batch_parallelism == 0 || cfg_.prefetch_depth == 0 ||
        cfg_.batch_size == 0)
        throw std::invalid_argument(
            "Loader: workers, parallelism, prefetch and batch size must all be >= 1");
    if (cfg_.cache.mode == CacheSpec::Mode::memory)
        cache_ = std::make_shared<SampleCache>(cfg_.cache.capacity_samples);
}

ThroughputReport Loader::run_epoch(std::uint64_t seed, std::uint64_t epoch,
                                   const BatchConsumer& consumer) {
    const std::vector<GlobalBatch> plan =
        batches(permute_epoch(seed, epoch, spec_.n), cfg_.batch_size);
    const std::size_t total = plan.size();
    ThroughputReport rep;
    rep.epoch = epoch;
    rep.batches = total;
    rep.samples = total * cfg_.batch_size;
    rep.batch_latency_s.resize(total);

    const std::size_t depth = cfg_.prefetch_depth;
    const int device = current_device();
    std::vector<LoadedBatch> done(total);
    std::vector<Clock::time_point> requested(total);
    std::mutex mu;
    std::condition_variable cv;
    std::size_t admitted = 0, claimed = 0, delivered = 0;
    bool stop = false;
    std::exception_ptr first_error;

    const auto start = Clock::now();
    for (; admitted < std::min(depth, total); ++admitted) requested[admitted] = start;

    auto worker = [&] {
        cudaSetDevice(device);
        for (;;) {
            std::size_t s;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return stop || claimed < admitted || claimed >= total; });
                if (stop || claimed >= total) return;
                s = claimed++;
            }
            LoadedBatch r = load_batch(spec_, cfg_, cache_.get(), plan[s]);
            const bool failed = static_cast<bool>(r.error);
            {
                std::lock_guard<std::mutex> g(mu);
                if (failed && !first_error) first_error = r.error;
                done[s] = std::move(r);
            }
            cv.notify_all();
            if (failed) return;
        }
    };

    std::vector<std::thread> workers;
    std::exception_ptr failure;
    try {
        for (std::uint32_t w = 0; w < cfg_.workers; ++w) workers.emplace_back(worker);
        while (delivered < total) {
            LoadedBatch r;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return first_error || done[delivered].ready; });
                if (first_error) std::rethrow_exception(first_error);
                r = std::move(done[delivered]);
            }
            rep.batch_latency_s[delivered] = elapsed_s(requested[delivered], Clock::now());
            rep.cache_hits += r.hits;
            rep.cache_misses += r.misses;
            if (consumer) consumer(plan[delivered], r.data);
            {
                std::lock_guard<std::mutex> g(mu);
                ++delivered;
                if (admitted < total) requested[admitted++] = Clock::now();
            }
            cv.notify_all();
        }
    } catch (...) {
        failure = std::current_exception();
    }
    {
        std::lock_guard<std::mutex> g(mu);
        stop = true;
    }
    cv.notify_all();
    for (auto& t : workers) t.join();
    if (failure) std::rethrow_exception(failure);

    rep.wall_s = elapsed_s(start, Clock::now());
    rep.samples_per_second =
        rep.wall_s > 0 ? static_cast<double>(rep.samples) / rep.wall_s : 0.0;
    return rep;
}

std::pair<ThroughputReport, ThroughputReport>
warm_cache_epoch(const DatasetSpec& spec, const LoaderConfig& cfg, std::uint64_t seed) {
    if (cfg.cache.mode != CacheSpec::Mode::memory || cfg.cache.capacity_samples < spec.n)
        throw std::invalid_argument(
            "warm_cache_epoch: needs a memory cache holding the whole dataset");
    Loader loader(spec, cfg);
    ThroughputReport cold = loader.run_epoch(seed, 0);
    ThroughputReport warm = loader.run_epoch(seed, 1);
    return {std::move(cold), std::move(warm)};
}

} // namespace locload
