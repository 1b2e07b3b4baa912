// Colourful-count-to-estimate scaling (reference include/motif/estimate.hpp).
#pragma once

#include <cstdint>
#include <vector>

#include "plan.hpp"

namespace mb {

uint64_t automorphism_count(const Query& q);             // estimate.hpp:14
double normalization_factor(int k);                       // estimate.hpp:18
double coefficient_of_variation(const std::vector<uint64_t>& c);  // estimate.hpp:39

}  // namespace mb
