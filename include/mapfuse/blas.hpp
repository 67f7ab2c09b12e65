// mapfuse/blas.hpp -- the shipped BLAS sequence suite (Table 1) and its
// deterministic input generator.
//
// API-compatible with the product half of
// /root/reference/proj/include/mapfuse/blas.hpp.  The reference's fp64
// oracle (reference_execute / reference_call / reference_run_script) is NOT
// part of the product: it lives in oracle/ as test infrastructure.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "mapfuse/library.hpp"
#include "mapfuse/script.hpp"

namespace mapfuse::blas {

std::string library_manifest();
std::string default_device_config_text();
const lib::Library& default_library();

struct SequenceCase {
  std::string name;  // upper-case suite name
  std::string script_text;
  std::string tag;   // Table-1 fusibility tag (F / S / B, () = weak)
};

std::vector<std::string> sequence_names();
SequenceCase build_sequence(const std::string& name);

// Row-major fp32 buffers padded to multiples of 32; vectors rows == 1,
// scalars 1x1.  Every non-input name is allocated and zero-filled.
struct Problem {
  int rows = 0, cols = 0;
  std::map<std::string, std::vector<float>> buffers;
  std::map<std::string, std::pair<int, int>> dims;
  std::map<std::string, float> scalars;

  const std::vector<float>& buffer(const std::string& name) const;
};

// std::mt19937(seed) + U(-1,1) in script-input order; scalars 0.25+0.5|U|
// (same stream as the reference, proj/src/blas.cpp:107-139).
Problem make_problem(const script::Script& s, int rows, int cols, uint32_t seed);

// B200 addition: vector lengths by propagation (depth-2 use fixes rows vs
// cols, depth-1 calls share lengths).  The reference's first-use rule
// (blas.cpp:75-103) mis-sizes SGEMV / GESUMMV / SGEMVT vectors for
// rectangular problems; for square problems both agree.
// 'r' row-indexed vector, 'c' column-indexed vector, 't' tile, 's' scalar.
std::map<std::string, char> vector_roles(const script::Script& s, const lib::Library& lib);
std::map<std::string, std::pair<int, int>> infer_shapes(const script::Script& s,
                                                        const lib::Library& lib, int rows,
                                                        int cols);

}  // namespace mapfuse::blas
