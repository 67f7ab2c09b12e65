// mf_compile.cpp -- TEMPORARY: routes to the hand-derived plans until the
// planner / codegen / lowering stack lands.
#include "mf_compile.hpp"

#include <stdexcept>

#include "mapfuse_b200.h"
#include "mf_builtin.hpp"
#include "mf_exec.hpp"

namespace mapfuse::b200 {

NativePlan compile_script(const std::string&, const std::string&, int, int, int) {
  throw Invalid("mf_compile: planner not built yet");
}
NativePlan compile_sequence(const std::string& sequence, int rows, int cols, int mode) {
  return builtin_plan(sequence, rows, cols, mode == MF_MODE_FUSED);
}
NativePlan plan_from_kernel_text(const std::string&, int, int) {
  throw Invalid("mf_plan_create: lowering not built yet");
}
int classify_exception(const std::exception&) { return MF_ERR_FAULT; }

}  // namespace mapfuse::b200
