// Error taxonomy of the reference (include/motif/errors.hpp:13-45) and the
// status codes the C-ABI returns for each (the reference CLI's exit codes:
// parse 2, treewidth 3, overflow 4, budget 5; plus schema 6, contract 7,
// spec 8, cuda 9, internal 1).
#pragma once

#include <stdexcept>
#include <string>

namespace mb {

enum Status : int {
  kOk = 0,
  kInternal = 1,
  kParse = 2,
  kTreewidth = 3,
  kOverflow = 4,
  kBudget = 5,
  kSchema = 6,
  kContract = 7,
  kSpec = 8,
  kCuda = 9,
};

struct Error : std::runtime_error {
  Status code;
  Error(Status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(Status c, const std::string& m) { throw Error(c, m); }

inline uint64_t checked_add(uint64_t a, uint64_t b) {
  uint64_t r;
  if (__builtin_add_overflow(a, b, &r)) fail(kOverflow, "count overflow in addition");
  return r;
}

inline uint64_t checked_mul(uint64_t a, uint64_t b) {
  uint64_t r;
  if (__builtin_mul_overflow(a, b, &r)) fail(kOverflow, "count overflow in multiplication");
  return r;
}

}  // namespace mb
