#pragma once
#include <string>

#include "mf_native.hpp"

namespace mapfuse::b200 {
// Hand-derived plan for a Table-1 sequence.
NativePlan builtin_plan(const std::string& sequence, int rows, int cols, bool fused);
}  // namespace mapfuse::b200
