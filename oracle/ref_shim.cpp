// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// library compiled from /root/reference/proj/src (see oracle/Makefile).
//
// TEST INFRASTRUCTURE ONLY: used to generate golden vectors
// (tests/golden/make_golden.py), to cross-check the C restatement in
// locload_oracle.c, and as the reference arm's CPU timing
// (bench.py --impl reference).  The product never links it.
//
// Nothing here re-implements reference behaviour except ref_assign's tail-move
// loop, which restates the six lines of the reference's private helper
// equivalence.cpp:77-88 on top of the reference's own loc_distribution,
// targets and balance (the helper sits in an anonymous namespace and cannot
// be called from outside its translation unit).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "locload/balance.hpp"
#include "locload/core.hpp"
#include "locload/equivalence.hpp"
#include "locload/pipeline.hpp"
#include "locload/rng.hpp"
#include "locload/sampling.hpp"
#include "locload/simulate.hpp"

using namespace locload;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -2;
    }
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_mix64(uint64_t z) { return mix64(z); }
uint64_t ref_derive_seed(uint64_t s, uint64_t a) { return derive_seed(s, a); }
uint64_t ref_derive_seed3(uint64_t s, uint64_t a, uint64_t b) { return derive_seed(s, a, b); }

// k draws of SplitMix64(seed).next()
void ref_splitmix_draws(uint64_t seed, uint64_t k, uint64_t* out) {
    SplitMix64 r(seed);
    for (uint64_t i = 0; i < k; ++i) out[i] = r.next();
}

void ref_splitmix_bounded(uint64_t seed, uint64_t n, uint64_t k, uint64_t* out) {
    SplitMix64 r(seed);
    for (uint64_t i = 0; i < k; ++i) out[i] = r.bounded(n);
}

int ref_permute_epoch(uint64_t seed, uint64_t epoch, uint64_t d, uint64_t* out) {
    return guarded([&] {
        const EpochPermutation p = permute_epoch(seed, epoch, d);
        std::memcpy(out, p.order.data(), sizeof(uint64_t) * d);
    });
}

int ref_permutation_prefix(uint64_t seed, uint64_t epoch, uint64_t d, uint64_t k, uint64_t* out) {
    return guarded([&] {
        const std::vector<SampleId> v = permutation_prefix(seed, epoch, d, k);
        std::memcpy(out, v.data(), sizeof(uint64_t) * k);
    });
}

// number of batches, or -1
int64_t ref_batches_count(uint64_t seed, uint64_t epoch, uint64_t d, uint64_t b) {
    int64_t n = -1;
    guarded([&] { n = static_cast<int64_t>(batches(permute_epoch(seed, epoch, d), b).size()); });
    return n;
}

int ref_cache_directory(uint64_t d, uint32_t p, double alpha, uint64_t* cached,
                        uint64_t* owned_counts) {
    return guarded([&] {
        const CacheDirectory dir(d, p, alpha);
        *cached = dir.cached_count();
        for (uint32_t j = 0; j < p; ++j) owned_counts[j] = dir.owned_count(j);
    });
}

// owner for each id (p when uncached)
int ref_owner(uint64_t d, uint32_t p, double alpha, const uint64_t* ids, uint64_t n,
              uint32_t* out) {
    return guarded([&] {
        const CacheDirectory dir(d, p, alpha);
        for (uint64_t i = 0; i < n; ++i) {
            const auto o = dir.owner(ids[i]);
            out[i] = o ? *o : p;
        }
    });
}

int ref_reg_slice(const uint64_t* batch, uint64_t B, uint32_t p, uint32_t j, uint64_t* out) {
    return guarded([&] {
        GlobalBatch g;
        g.samples.assign(batch, batch + B);
        const LocalAssignment a = reg_slice(g, p, j);
        std::memcpy(out, a.samples.data(), sizeof(uint64_t) * a.samples.size());
    });
}

// loc_distribution: flat lists (learner-major, batch order), offsets[p+1],
// uncached list, counts[p]; plus counts_with_uncached -> cwu[p].
int ref_loc_distribution(const uint64_t* batch, uint64_t B, uint64_t d, uint32_t p, double alpha,
                         uint64_t* lists, uint64_t* offsets, uint64_t* uncached,
                         uint64_t* n_uncached, uint64_t* counts, uint64_t* cwu) {
    return guarded([&] {
        const CacheDirectory dir(d, p, alpha);
        GlobalBatch g;
        g.samples.assign(batch, batch + B);
        const LocDistribution dist = loc_distribution(g, dir);
        uint64_t off = 0;
        for (uint32_t j = 0; j < p; ++j) {
            offsets[j] = off;
            const auto& s = dist.assignments[j].samples;
            std::memcpy(lists + off, s.data(), sizeof(uint64_t) * s.size());
            off += s.size();
            counts[j] = dist.counts[j];
        }
        offsets[p] = off;
        *n_uncached = dist.uncached.size();
        std::memcpy(uncached, dist.uncached.data(), sizeof(uint64_t) * dist.uncached.size());
        const std::vector<std::uint64_t> c = counts_with_uncached(dist, p);
        for (uint32_t j = 0; j < p; ++j) cwu[j] = c[j];
    });
}

int ref_targets(int64_t b, uint32_t p, int64_t* out) {
    return guarded([&] {
        const auto t = targets(b, p);
        for (uint32_t j = 0; j < p; ++j) out[j] = t[j];
    });
}

// moves as (sender, receiver, count) triples; returns count via *n
int ref_balance(const int64_t* counts, const int64_t* tg, uint32_t p, int64_t* moves, int* n) {
    return guarded([&] {
        ImbalanceVector iv;
        iv.counts.assign(counts, counts + p);
        iv.targets.assign(tg, tg + p);
        const TransferSchedule s = balance(iv);
        *n = static_cast<int>(s.moves.size());
        for (std::size_t k = 0; k < s.moves.size(); ++k) {
            moves[3 * k + 0] = s.moves[k].sender;
            moves[3 * k + 1] = s.moves[k].receiver;
            moves[3 * k + 2] = s.moves[k].count;
        }
    });
}

int ref_optimal_message_count(const int64_t* counts, const int64_t* tg, uint32_t p, int* out) {
    return guarded([&] {
        ImbalanceVector iv;
        iv.counts.assign(counts, counts + p);
        iv.targets.assign(tg, tg + p);
        *out = optimal_message_count(iv);
    });
}

int ref_deficit_fraction(const int64_t* counts, const int64_t* tg, uint32_t p, double* out) {
    return guarded([&] {
        ImbalanceVector iv;
        iv.counts.assign(counts, counts + p);
        iv.targets.assign(tg, tg + p);
        *out = deficit_fraction(iv);
    });
}

// Locality-balanced assignment of one fully cached batch (alpha = 1):
// loc_distribution -> targets -> balance -> tail moves (equivalence.cpp:77-88).
// lists: flat final lists, offsets[p+1]; moves as triples, *n_moves.
int ref_assign_balanced(const uint64_t* batch, uint64_t B, uint64_t d, uint32_t p,
                        uint64_t* lists, uint64_t* offsets, int64_t* moves, int* n_moves) {
    return guarded([&] {
        const CacheDirectory dir(d, p, 1.0);
        GlobalBatch g;
        g.samples.assign(batch, batch + B);
        LocDistribution dist = loc_distribution(g, dir);
        ImbalanceVector iv;
        iv.counts.assign(dist.counts.begin(), dist.counts.end());
        iv.targets = targets(static_cast<std::int64_t>(g.samples.size()), p);
        const TransferSchedule schedule = balance(iv);
        for (const Move& move : schedule.moves) {
            auto& from = dist.assignments[move.sender].samples;
            auto& to = dist.assignments[move.receiver].samples;
            to.insert(to.end(), from.end() - move.count, from.end());
            from.erase(from.end() - move.count, from.end());
        }
        uint64_t off = 0;
        for (uint32_t j = 0; j < p; ++j) {
            offsets[j] = off;
            const auto& s = dist.assignments[j].samples;
            std::memcpy(lists + off, s.data(), sizeof(uint64_t) * s.size());
            off += s.size();
        }
        offsets[p] = off;
        *n_moves = static_cast<int>(schedule.moves.size());
        for (std::size_t k = 0; k < schedule.moves.size(); ++k) {
            moves[3 * k + 0] = schedule.moves[k].sender;
            moves[3 * k + 1] = schedule.moves[k].receiver;
            moves[3 * k + 2] = schedule.moves[k].count;
        }
    });
}

// generate_dataset into `root`, then read back sample `id`'s bytes.
int ref_generate_dataset(const char* root, uint64_t n, uint64_t sample_bytes, uint64_t seed) {
    return guarded([&] {
        DatasetSpec spec;
        spec.root = root;
        spec.n = n;
        spec.sample_bytes = sample_bytes;
        generate_dataset(spec, seed);
    });
}

int ref_sample_path(const char* root, uint64_t id, char* out, uint64_t cap) {
    return guarded([&] {
        DatasetSpec spec;
        spec.root = root;
        const std::string s = sample_path(spec, id).string();
        std::strncpy(out, s.c_str(), cap);
    });
}

// Reference Loader::run_epoch (pipeline.cpp:247-336) with a memory cache.
// Consumer copies every delivered payload's first byte into `probe` (so the
// test can check delivery order) and counts samples.  Returns samples/s.
int ref_loader_epoch(const char* root, uint64_t n, uint64_t sample_bytes, uint32_t workers,
                     uint32_t threads, uint32_t prefetch, uint64_t batch, int cache,
                     uint64_t seed, uint64_t epochs, double* samples_per_s, uint64_t* hits,
                     uint64_t* misses) {
    return guarded([&] {
        DatasetSpec spec;
        spec.root = root;
        spec.n = n;
        spec.sample_bytes = sample_bytes;
        LoaderConfig cfg;
        cfg.workers = workers;
        cfg.intra_batch_parallelism = threads;
        cfg.prefetch_depth = prefetch;
        cfg.batch_size = batch;
        if (cache) {
            cfg.cache.mode = CacheSpec::Mode::memory;
            cfg.cache.capacity_samples = n;
        }
        Loader loader(spec, cfg);
        ThroughputReport r;
        for (uint64_t e = 0; e < epochs; ++e) r = loader.run_epoch(seed, e);
        *samples_per_s = r.samples_per_second;
        *hits = r.cache_hits;
        *misses = r.cache_misses;
    });
}

// equivalence.hpp: the reference's own synthesis and training runs
int ref_run_training(uint64_t n, uint32_t dims, uint64_t obj_seed, int scheme, uint32_t p,
                     uint64_t b, uint64_t steps, uint64_t seed, double lr, int agg,
                     double* final_w, double* step_grads) {
    return guarded([&] {
        const ToyObjective obj = ToyObjective::synthesize(n, dims, obj_seed);
        const SchemeKind sk = scheme == 0 ? SchemeKind::regular
                              : scheme == 1 ? SchemeKind::locality
                                            : SchemeKind::locality_balanced;
        const TrainingRun run = run_training(obj, sk, p, b, steps, seed, lr,
                                             agg == 0 ? Aggregation::canonical
                                                      : Aggregation::learner_order);
        std::memcpy(final_w, run.final_weights.data(), sizeof(double) * dims);
        for (uint64_t t = 0; t < steps; ++t)
            std::memcpy(step_grads + t * dims, run.step_gradients[t].data(), sizeof(double) * dims);
    });
}
int ref_full_batch_gradient(uint64_t n, uint32_t dims, uint64_t obj_seed, const double* w,
                            const uint64_t* batch, uint64_t b, double* out) {
    return guarded([&] {
        const ToyObjective obj = ToyObjective::synthesize(n, dims, obj_seed);
        GlobalBatch g;
        g.samples.assign(batch, batch + b);
        const std::vector<double> r =
            full_batch_gradient(obj, std::vector<double>(w, w + dims), g);
        std::memcpy(out, r.data(), sizeof(double) * dims);
    });
}
int ref_sample_gradient(uint64_t n, uint32_t dims, uint64_t obj_seed, const double* w,
                        uint64_t i, double* out, double* loss) {
    return guarded([&] {
        const ToyObjective obj = ToyObjective::synthesize(n, dims, obj_seed);
        const std::vector<double> wv(w, w + dims);
        std::vector<double> g;
        obj.sample_gradient(wv, i, g);
        std::memcpy(out, g.data(), sizeof(double) * dims);
        *loss = obj.sample_loss(wv, i);
    });
}

// simulate_imbalance (simulate.cpp:42-79): the per-step balancing fractions
// beta of `steps` fresh global batches and their five-number summary
// {median, q1, q3, whisker_lo, whisker_hi} -- Eq. 8's predicted beta
// (model.hpp:72-74).  betas may be NULL.
int ref_simulate_imbalance(uint64_t d, uint32_t p, uint64_t local_batch, uint64_t steps,
                           uint64_t seed, double alpha, double* betas, double* summary5) {
    return guarded([&] {
        const ImbalanceStats st = simulate_imbalance(d, p, local_batch, steps, seed, alpha);
        if (betas) std::memcpy(betas, st.betas.data(), sizeof(double) * st.betas.size());
        summary5[0] = st.summary.median;
        summary5[1] = st.summary.q1;
        summary5[2] = st.summary.q3;
        summary5[3] = st.summary.whisker_lo;
        summary5[4] = st.summary.whisker_hi;
    });
}

} // extern "C"
