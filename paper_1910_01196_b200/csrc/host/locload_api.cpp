// locload_api.cpp -- the reference's C++ API (namespace locload) on top of the
// C-ABI.  Hot-path functions run on the current CUDA device; each calling
// thread gets its own context (stream + scratch), which keeps the functions
// thread-safe like the reference's pure functions.
// C-ABI status codes become the reference's exception types.
#include <cuda_runtime.h>

#include <chrono>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>

#include "locload/balance.hpp"
#include "locload/core.hpp"
#include "locload/equivalence.hpp"
#include "locload/gpu.hpp"
#include "locload/rng.hpp"
#include "locload/sampling.hpp"
#include "locload_b200.h"
#include "api_internal.h"

namespace locload {
namespace detail {

void check(int status) {
    if (status == LL_OK) return;
    const std::string msg = ll_last_error();
    if (status == LL_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

namespace {
struct ThreadContexts {
    std::map<int, ll_ctx*> by_device;
    ~ThreadContexts() {
        for (auto& kv : by_device) ll_ctx_destroy(kv.second);
    }
};
} // namespace

ll_ctx* ctx() {
    thread_local ThreadContexts tc;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    ll_ctx*& c = tc.by_device[dev];
    if (!c) check(ll_ctx_create(&c, dev));
    return c;
}

} // namespace detail

namespace {
using detail::check;
using detail::ctx;

struct Assigned {
    std::vector<std::uint64_t> ids, off, kept, counts, stats;
    std::vector<ll_move> moves;
};

Assigned assign(const std::vector<SampleId>& batch, std::uint64_t d, std::uint32_t p,
                double alpha, int scheme) {
    Assigned a;
    const std::size_t B = batch.size();
    a.ids.resize(B ? B : 1);
    a.off.resize(p + 1);
    a.kept.resize(p ? p : 1);
    a.counts.resize(p ? p : 1);
    a.moves.resize(p ? p : 1);
    a.stats.resize(4);
    std::uint32_t nm = 0;
    check(ll_assign(ctx(), batch.data(), B, d, p, alpha, scheme, a.ids.data(), a.off.data(),
                    a.kept.data(), a.counts.data(), a.moves.data(), &nm, a.stats.data()));
    a.moves.resize(nm);
    return a;
}

} // namespace

// ------------------------------------------------------------------ core
EpochPermutation permute_epoch(std::uint64_t seed, std::uint64_t epoch, std::uint64_t d) {
    EpochPermutation p;
    p.seed = seed;
    p.epoch = epoch;
    p.order.resize(d ? d : 1);
    check(ll_permute_epoch(ctx(), seed, epoch, d, p.order.data()));
    p.order.resize(d);
    return p;
}

std::vector<SampleId> permutation_prefix(std::uint64_t seed, std::uint64_t epoch,
                                         std::uint64_t d, std::uint64_t k) {
    std::vector<SampleId> out(k ? k : 1);
    check(ll_permutation_prefix(ctx(), seed, epoch, d, k, out.data()));
    out.resize(k);
    return out;
}

std::vector<GlobalBatch> batches(const EpochPermutation& perm, std::uint64_t b) {
    const std::uint64_t d = perm.order.size();
    if (b == 0 || b > d) throw std::invalid_argument("batches: batch size must be in [1, dataset size]");
    std::vector<GlobalBatch> out(d / b);
    for (std::uint64_t t = 0; t < out.size(); ++t) {
        out[t].step = t;
        out[t].samples.assign(perm.order.begin() + static_cast<std::ptrdiff_t>(t * b),
                              perm.order.begin() + static_cast<std::ptrdiff_t>((t + 1) * b));
    }
    return out;
}

// -------------------------------------------------------------- sampling
CacheDirectory::CacheDirectory(std::uint64_t d, std::uint32_t p, double alpha)
    : d_(d), p_(p), alpha_(alpha), cached_(0) {
    if (p == 0) throw std::invalid_argument("CacheDirectory: learner count must be >= 1");
    if (!(alpha > 0.0) || alpha > 1.0)
        throw std::invalid_argument("CacheDirectory: cached fraction must be in (0, 1]");
    const auto c = static_cast<std::uint64_t>(alpha * static_cast<double>(d));
    cached_ = c < d ? c : d;
}

std::uint64_t CacheDirectory::owned_count(LearnerId j) const {
    if (j >= p_) return 0;
    const auto first = [&](std::uint64_t k) { return (k * cached_ + p_ - 1) / p_; };
    return first(j + 1) - first(j);
}

LocalAssignment reg_slice(const GlobalBatch& batch, std::uint32_t p, LearnerId j) {
    if (p == 0 || j >= p) throw std::invalid_argument("reg_slice: learner rank out of range");
    if (batch.samples.size() % p != 0)
        throw std::invalid_argument("reg_slice: learner count must divide the batch size");
    const Assigned a = assign(batch.samples, 0xFFFFFFFEull, p, 1.0, LL_SCHEME_REGULAR);
    LocalAssignment out;
    out.learner = j;
    out.step = batch.step;
    out.samples.assign(a.ids.begin() + static_cast<std::ptrdiff_t>(a.off[j]),
                       a.ids.begin() + static_cast<std::ptrdiff_t>(a.off[j + 1]));
    return out;
}

LocDistribution loc_distribution(const GlobalBatch& batch, const CacheDirectory& dir) {
    const std::uint32_t p = dir.learners();
    const Assigned a = assign(batch.samples, dir.dataset_size(), p, dir.cached_fraction(),
                              LL_SCHEME_LOCALITY);
    // device lists: learner j's cached samples (batch order), then its
    // round-robin share of the uncached ones (the k-th uncached -> k mod p)
    const std::uint64_t U = a.stats[2];
    LocDistribution dist;
    dist.step = batch.step;
    dist.assignments.resize(p);
    dist.counts.assign(p, 0);
    dist.uncached.resize(U);
    for (std::uint32_t j = 0; j < p; ++j) {
        const std::uint64_t dealt = U / p + (j < U % p ? 1 : 0);
        const std::uint64_t own = a.counts[j] - dealt;
        dist.assignments[j].learner = j;
        dist.assignments[j].step = batch.step;
        dist.assignments[j].samples.assign(a.ids.begin() + static_cast<std::ptrdiff_t>(a.off[j]),
                                           a.ids.begin() + static_cast<std::ptrdiff_t>(a.off[j] + own));
        dist.counts[j] = own;
        for (std::uint64_t t = 0; t < dealt; ++t) dist.uncached[j + t * p] = a.ids[a.off[j] + own + t];
    }
    return dist;
}

std::vector<std::uint64_t> counts_with_uncached(const LocDistribution& dist, std::uint32_t p) {
    std::vector<std::uint64_t> c = dist.counts;
    c.resize(p, 0);
    for (std::size_t k = 0; k < dist.uncached.size(); ++k) ++c[k % p];
    return c;
}

// --------------------------------------------------------------- balance
std::int64_t ImbalanceVector::total() const {
    std::int64_t t = 0;
    for (std::int64_t c : counts) t += c;
    return t;
}

std::vector<std::int64_t> targets(std::int64_t b, std::uint32_t p) {
    if (p == 0) throw std::invalid_argument("targets: learner count must be >= 1");
    if (b < 0) throw std::invalid_argument("targets: batch size must be non-negative");
    std::vector<std::int64_t> t(p, b / p);
    for (std::int64_t j = 0; j < b % static_cast<std::int64_t>(p); ++j) ++t[static_cast<std::size_t>(j)];
    return t;
}

namespace {
void validate(const ImbalanceVector& iv) {
    if (iv.counts.size() != iv.targets.size())
        throw std::invalid_argument("balance: counts and targets must have equal length");
    std::int64_t c = 0, t = 0;
    for (std::size_t j = 0; j < iv.counts.size(); ++j) {
        c += iv.counts[j];
        t += iv.targets[j];
    }
    if (c != t) throw std::invalid_argument("balance: counts and targets must sum to the same total");
}
} // namespace

TransferSchedule balance(const ImbalanceVector& iv) {
    validate(iv);
    TransferSchedule s;
    const auto p = static_cast<std::uint32_t>(iv.counts.size());
    if (p == 0) return s;
    std::vector<ll_move> mv(p);
    std::uint32_t n = 0;
    check(ll_balance_batch(ctx(), iv.counts.data(), iv.targets.data(), p, 1, mv.data(), &n));
    for (std::uint32_t k = 0; k < n; ++k) s.moves.push_back({mv[k].sender, mv[k].receiver, mv[k].count});
    return s;
}

// Exhaustive minimum message count (test oracle, balance.cpp:86-124): the
// minimum number of messages is n - (max number of disjoint zero-sum groups)
// over the n imbalanced learners.  Host dynamic program over subsets.
int optimal_message_count(const ImbalanceVector& iv) {
    validate(iv);
    if (iv.counts.size() > 10)
        throw std::invalid_argument("optimal_message_count: exhaustive oracle limited to p <= 10");
    std::vector<std::int64_t> imb;
    for (std::size_t j = 0; j < iv.counts.size(); ++j)
        if (iv.counts[j] != iv.targets[j]) imb.push_back(iv.counts[j] - iv.targets[j]);
    const int n = static_cast<int>(imb.size());
    if (n == 0) return 0;
    const int full = (1 << n) - 1;
    std::vector<std::int64_t> sum(full + 1, 0);
    for (int m = 1; m <= full; ++m) {
        int bit = 0;
        while (!(m & (1 << bit))) ++bit;
        sum[m] = sum[m & (m - 1)] + imb[bit];
    }
    // groups[m] = max zero-sum groups partitioning m (-1: impossible)
    std::vector<int> groups(full + 1, -1);
    groups[0] = 0;
    for (int m = 1; m <= full; ++m) {
        if (sum[m] != 0) continue;
        const int low = m & -m;
        for (int g = m; g; g = (g - 1) & m)
            if ((g & low) && sum[g] == 0 && groups[m ^ g] >= 0 && groups[m ^ g] + 1 > groups[m])
                groups[m] = groups[m ^ g] + 1;
    }
    return n - groups[full];
}

double deficit_fraction(const ImbalanceVector& iv) {
    validate(iv);
    const std::int64_t b = iv.total();
    if (b == 0) return 0.0;
    std::int64_t def = 0;
    for (std::size_t j = 0; j < iv.counts.size(); ++j)
        if (iv.targets[j] > iv.counts[j]) def += iv.targets[j] - iv.counts[j];
    return static_cast<double>(def) / static_cast<double>(b);
}

// ------------------------------------------------------------------- gpu
namespace gpu {

DeviceLoader::DeviceLoader(const ll_loader_config& cfg, int device) {
    check(ll_ctx_create(&ctx_, device));
    const int rc = ll_loader_create(&ld_, ctx_, &cfg);
    if (rc != LL_OK) {
        const std::string msg = ll_last_error();
        ll_ctx_destroy(ctx_);
        if (rc == LL_ERR_INVALID) throw std::invalid_argument(msg);
        throw std::runtime_error(msg);
    }
}

DeviceLoader::~DeviceLoader() {
    if (ld_) ll_loader_destroy(ld_);
    if (ctx_) ll_ctx_destroy(ctx_);
}

void DeviceLoader::populate() { check(ll_loader_populate(ld_)); }
void DeviceLoader::populate_from_host(const std::uint8_t* s) {
    check(ll_loader_populate_from_host(ld_, s));
}
std::vector<std::uint8_t> DeviceLoader::ipc_handle() {
    std::vector<std::uint8_t> h(64);
    check(ll_loader_ipc_handle(ld_, h.data()));
    return h;
}
void DeviceLoader::open_peers(const std::vector<std::uint8_t>& handles) {
    check(ll_loader_open_peers(ld_, handles.data()));
}
void DeviceLoader::comm_init(const std::vector<std::uint8_t>& id) {
    check(ll_loader_comm_init(ld_, id.data()));
}
std::vector<std::uint8_t> DeviceLoader::nccl_unique_id() {
    std::vector<std::uint8_t> id(128);
    check(ll_nccl_unique_id(id.data()));
    return id;
}
void DeviceLoader::link_peers(const std::vector<DeviceLoader*>& lds) {
    std::vector<ll_loader*> h;
    for (auto* l : lds) h.push_back(l->ld_);
    check(ll_loader_link_peers(h.data(), static_cast<std::uint32_t>(h.size())));
}
std::uint64_t DeviceLoader::steps_per_epoch() const {
    std::uint64_t n = 0;
    check(ll_loader_steps_per_epoch(ld_, &n));
    return n;
}
DeviceBatch DeviceLoader::step(std::uint64_t epoch, std::uint64_t s) {
    ll_step_info info{};
    check(ll_loader_step(ld_, epoch, s, &info));
    DeviceBatch b;
    b.epoch = epoch;
    b.step = s;
    b.size = info.n_local;
    b.local = info.kept;
    b.received = info.received;
    b.data = reinterpret_cast<const void*>(info.device_out);
    b.ids = reinterpret_cast<const std::uint32_t*>(info.device_ids);
    check(ll_ctx_stream(ctx_, &b.stream));
    return b;
}
void DeviceLoader::synchronize() { check(ll_ctx_sync(ctx_)); }

EpochReport DeviceLoader::run_epoch(std::uint64_t epoch, const DeviceBatchConsumer& consumer) {
    using Clock = std::chrono::steady_clock;
    EpochReport r;
    r.epoch = epoch;
    r.batches = steps_per_epoch();
    const auto t0 = Clock::now();
    for (std::uint64_t s = 0; s < r.batches; ++s) {
        const DeviceBatch b = step(epoch, s);
        r.samples += b.size;
        r.cache_hits += b.local;
        r.cache_misses += b.received;
        if (consumer) consumer(b);  // in step order, on the calling thread
    }
    synchronize();
    r.wall_s = std::chrono::duration<double>(Clock::now() - t0).count();
    r.samples_per_second = r.wall_s > 0 ? static_cast<double>(r.samples) / r.wall_s : 0.0;
    return r;
}

} // namespace gpu

// ---- equivalence (equivalence.hpp): data on the host, training on the device

ToyObjective ToyObjective::synthesize(std::uint64_t n, std::size_t dims, std::uint64_t seed) {
    if (n == 0 || dims == 0) throw std::invalid_argument("ToyObjective: need n >= 1 and dims >= 1");
    ToyObjective obj;
    obj.n_ = n;
    obj.m_ = dims;
    obj.xs_.resize(n * dims);
    obj.ys_.resize(n);
    // ground truth from stream (seed, 0xfeed); sample i from (seed, i, 0x5a11):
    // dims gaussians, then y = dot(truth, x) + 0.1 * gaussian  (equivalence.cpp:22-35)
    std::vector<double> truth(dims);
    SplitMix64 tr(derive_seed(seed, 0xfeedULL));
    for (double& t : truth) t = tr.next_gaussian();
    for (std::uint64_t i = 0; i < n; ++i) {
        SplitMix64 r(derive_seed(seed, i, 0x5a11ULL));
        double dot = 0;
        double* x = &obj.xs_[i * dims];
        for (std::size_t k = 0; k < dims; ++k) {
            x[k] = r.next_gaussian();
            dot += truth[k] * x[k];
        }
        obj.ys_[i] = dot + 0.1 * r.next_gaussian();
    }
    return obj;
}

double ToyObjective::sample_loss(const std::vector<double>& w, SampleId i) const {
    const double* x = &xs_[i * m_];
    double dot = 0;
    for (std::size_t k = 0; k < m_; ++k) dot += w[k] * x[k];
    const double r = dot - ys_[i];
    return 0.5 * r * r;
}

void ToyObjective::sample_gradient(const std::vector<double>& w, SampleId i,
                                   std::vector<double>& out) const {
    const double* x = &xs_[i * m_];
    double dot = 0;
    for (std::size_t k = 0; k < m_; ++k) dot += w[k] * x[k];
    const double r = dot - ys_[i];
    out.resize(m_);
    for (std::size_t k = 0; k < m_; ++k) out[k] = r * x[k];
}

TrainingRun run_training(const ToyObjective& obj, SchemeKind scheme, std::uint32_t p,
                         std::uint64_t batch_size, std::uint64_t steps, std::uint64_t seed,
                         double learning_rate, Aggregation agg) {
    const int sc = scheme == SchemeKind::regular    ? LL_SCHEME_REGULAR
                   : scheme == SchemeKind::locality ? LL_SCHEME_LOCALITY
                                                    : LL_SCHEME_LOCALITY_BALANCED;
    const int ag = agg == Aggregation::canonical ? LL_AGG_CANONICAL : LL_AGG_LEARNER_ORDER;
    const std::size_t m = obj.dims();
    TrainingRun run;
    run.final_weights.assign(m, 0.0);
    std::vector<double> grads(steps * m);
    check(ll_train_run(ctx(), obj.xs().data(), obj.ys().data(), obj.samples(),
                       static_cast<std::uint32_t>(m), sc, p, batch_size, steps, seed,
                       learning_rate, ag, run.final_weights.data(), grads.data()));
    run.step_gradients.resize(steps);
    for (std::uint64_t t = 0; t < steps; ++t)
        run.step_gradients[t].assign(grads.begin() + t * m, grads.begin() + (t + 1) * m);
    return run;
}

std::pair<TrainingRun, TrainingRun>
run_training_imbalanced_vs_balanced(const ToyObjective& obj, std::uint32_t p,
                                    std::uint64_t batch_size, std::uint64_t steps,
                                    std::uint64_t seed, double learning_rate) {
    TrainingRun loc =
        run_training(obj, SchemeKind::locality, p, batch_size, steps, seed, learning_rate);
    TrainingRun bal = run_training(obj, SchemeKind::locality_balanced, p, batch_size, steps,
                                   seed, learning_rate);
    return {std::move(loc), std::move(bal)};
}

std::vector<double> full_batch_gradient(const ToyObjective& obj, const std::vector<double>& w,
                                        const GlobalBatch& batch) {
    std::vector<double> g(obj.dims());
    check(ll_full_batch_gradient(ctx(), obj.xs().data(), obj.ys().data(), obj.samples(),
                                 static_cast<std::uint32_t>(obj.dims()), w.data(),
                                 batch.samples.data(), batch.samples.size(), g.data()));
    return g;
}

} // namespace locload
