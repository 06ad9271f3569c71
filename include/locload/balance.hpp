// locload/balance.hpp -- source-compatible drop-in for
// proj/include/locload/balance.hpp.  balance() (Algorithm 1) runs on the
// device (assign.cu); optimal_message_count is the reference's exhaustive
// test oracle and stays a host routine (not on the hot path).
#pragma once

#include <cstdint>
#include <vector>

#include "locload/core.hpp"

namespace locload {

struct ImbalanceVector {
    std::vector<std::int64_t> counts;
    std::vector<std::int64_t> targets;

    std::int64_t total() const;
    std::size_t learners() const { return counts.size(); }
};

// balance.cpp:14-28: floor(b/p) each, +1 for the first b mod p learners
std::vector<std::int64_t> targets(std::int64_t b, std::uint32_t p);

struct Move {
    LearnerId sender = 0;
    LearnerId receiver = 0;
    std::int64_t count = 0;
};

struct TransferSchedule {
    std::vector<Move> moves;
};

// balance.cpp:58-84 (device)
TransferSchedule balance(const ImbalanceVector& iv);
// balance.cpp:86-124 (host, exhaustive; p <= 10)
int optimal_message_count(const ImbalanceVector& iv);
// balance.cpp:126-135
double deficit_fraction(const ImbalanceVector& iv);

} // namespace locload
