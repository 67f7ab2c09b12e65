// mf_compile.hpp -- script / KernelIR text -> NativePlan.
#pragma once
#include <exception>
#include <string>

#include "mf_native.hpp"

namespace mapfuse::b200 {

// Full pipeline (SPEC.md:668-676 cmd_compile): parse, dependency graph,
// fusion planning, combination selection, KernelIR codegen, lowering.
NativePlan compile_script(const std::string& script_text, const std::string& manifest, int rows,
                          int cols, int mode);
NativePlan compile_sequence(const std::string& sequence, int rows, int cols, int mode);
// vm::launch boundary: one KernelIR (text) -> one native kernel.
NativePlan plan_from_kernel_text(const std::string& text, int rows, int cols);
NativePlan compile_script_ranked(const std::string& script_text, const std::string& manifest,
                                 int rows, int cols, int mode, int rank);
int64_t count_script_covers(const std::string& script_text, const std::string& manifest, int rows,
                            int cols);
std::string save_plan_text(const NativePlan& p);
std::string sequence_script_text(const std::string& name);
NativePlan load_plan_text(const std::string& text);
// Error-class mapping for the C-ABI (ParseError / validation -> invalid).
int classify_exception(const std::exception& e);

}  // namespace mapfuse::b200
