// mf_compile.cpp -- script / KernelIR text -> NativePlan (C-ABI side).
#include "mf_compile.hpp"

#include <algorithm>
#include <stdexcept>

#include "mapfuse/blas.hpp"
#include "mapfuse/kernel.hpp"
#include "mapfuse/planner.hpp"
#include "mapfuse_b200.h"
#include "mf_exec.hpp"

namespace mapfuse::b200 {

namespace {
template <typename F>
NativePlan as_invalid(F&& f) {
  try {
    return f();
  } catch (const Fault&) {
    throw;
  } catch (const Invalid&) {
    throw;
  } catch (const std::exception& e) {  // parse / validation / planning errors
    throw Invalid(e.what());
  }
}
}  // namespace

NativePlan compile_script(const std::string& script_text, const std::string& manifest, int rows,
                          int cols, int mode) {
  return as_invalid([&] {
    if (mode != MF_MODE_FUSED && mode != MF_MODE_UNFUSED && mode != MF_MODE_B200)
      throw Invalid("unknown planner mode");
    NativePlan p = manifest.empty()
                       ? plan::compile(script_text, blas::default_library(), rows, cols, mode)
                       : plan::compile(script_text, lib::load_library(manifest), rows, cols, mode);
    p.script_text = script_text;
    p.manifest = manifest;
    return p;
  });
}

NativePlan compile_script_ranked(const std::string& script_text, const std::string& manifest,
                                 int rows, int cols, int mode, int rank) {
  return as_invalid([&] {
    if (mode != MF_MODE_FUSED && mode != MF_MODE_UNFUSED && mode != MF_MODE_B200)
      throw Invalid("unknown planner mode");
    NativePlan p = manifest.empty()
                       ? plan::compile_ranked(script_text, blas::default_library(), rows, cols, mode, rank)
                       : plan::compile_ranked(script_text, lib::load_library(manifest), rows, cols, mode,
                                              rank);
    p.script_text = script_text;
    p.manifest = manifest;
    return p;
  });
}

int64_t count_script_covers(const std::string& script_text, const std::string& manifest, int rows,
                            int cols) {
  int64_t n = 0;
  as_invalid([&] {
    if (manifest.empty()) n = plan::count_covers(script_text, blas::default_library(), rows, cols);
    else n = plan::count_covers(script_text, lib::load_library(manifest), rows, cols);
    return NativePlan{};
  });
  return n;
}

std::string save_plan_text(const NativePlan& p) {
  std::string s;
  as_invalid([&] {
    s = plan::save_plan(p);
    return NativePlan{};
  });
  return s;
}

std::string sequence_script_text(const std::string& name) {
  try {
    return blas::build_sequence(name).script_text;
  } catch (const std::exception& e) {
    throw Invalid(e.what());
  }
}

NativePlan load_plan_text(const std::string& text) {
  return as_invalid([&] { return plan::load_plan(text); });
}

NativePlan compile_sequence(const std::string& sequence, int rows, int cols, int mode) {
  return as_invalid([&] {
    const blas::SequenceCase c = blas::build_sequence(sequence);
    NativePlan p = compile_script(c.script_text, std::string(), rows, cols, mode);
    p.sequence = c.name;
    return p;
  });
}

NativePlan plan_from_kernel_text(const std::string& text, int rows, int cols) {
  return as_invalid([&] {
    const kernel::KernelIR k = kernel::parse_kernel_text(text);
    NativePlan p;
    p.rows = (rows + 31) / 32 * 32;
    p.cols = (cols + 31) / 32 * 32;
    p.sequence = k.name;
    NativeKernel nk = plan::lower_or_generic(k);
    nk.name = k.name;
    plan::CostModel::defaults().predict_us(nk, p.rows, p.cols);
    auto add = [&](const std::string& n, int r, int c, Role role, bool rowix) {
      if (p.find(n)) return;
      BufferSpec b;
      b.name = n;
      b.rows = r;
      b.cols = c;
      b.role = role;
      b.row_indexed = rowix;
      p.buffers.push_back(b);
    };
    if (nk.kind == NativeKernel::Kind::Generic) {
      // shapes follow the index expressions; the kernel bounds-checks every
      // access against the bound shapes at run time, as the VM does
      const GenericOp& g = nk.generic;
      const bool d2 = g.depth == 2;
      for (size_t i = 0; i < g.buffers.size(); ++i) {
        const std::string& b = g.buffers[i];
        const bool out = std::find(g.outputs.begin(), g.outputs.end(), b) != g.outputs.end();
        const char e = b == g.domain ? (d2 ? 't' : 'n') : g.extent[i];
        const int r = e == 't' && d2 ? p.rows : 1;
        const int c = e == '1' ? 1 : (e == 'm' ? p.rows : p.cols);
        add(b, r, c, out ? Role::Output : Role::Input, e == 'm');
        if (e == '1') p.buffers.back().scalar = true;
      }
    } else if (nk.kind == NativeKernel::Kind::Matrix) {
      const MatrixOp& op = nk.matrix;
      for (const auto& m : op.mats) add(m, p.rows, p.cols, Role::Input, false);
      for (const auto& [u, v] : op.rank) {
        add(u, 1, p.rows, Role::Input, true);
        add(v, 1, p.cols, Role::Input, false);
      }
      for (const auto& r : op.rows) add(r.x, 1, p.cols, Role::Input, false);
      for (const auto& c : op.cols) add(c.x, 1, p.rows, Role::Input, true);
      if (!op.store.empty()) add(op.store, p.rows, p.cols, Role::Output, false);
      for (const auto& r : op.rows) add(r.y, 1, p.rows, Role::Output, true);
      for (const auto& c : op.cols) add(c.y, 1, p.cols, Role::Output, false);
    } else {
      const bool tiles = k.depth == 2;
      for (const auto& i : nk.stream.inputs) add(i, tiles ? p.rows : 1, p.cols, Role::Input, false);
      for (const auto& o : nk.stream.outs) add(o.name, tiles ? p.rows : 1, p.cols, Role::Output, false);
      if (nk.stream.has_dot) {
        add(nk.stream.dot_out, 1, 1, Role::Output, false);
        p.buffers.back().scalar = true;
      }
    }
    for (const auto& b : p.buffers) (void)b;
    p.kernels.push_back(std::move(nk));
    p.kernel_ir.push_back(text);
    return p;
  });
}

int classify_exception(const std::exception&) { return MF_ERR_FAULT; }

}  // namespace mapfuse::b200
