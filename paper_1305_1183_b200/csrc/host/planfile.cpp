// host/planfile.cpp -- plan files: compile once, run many.
//
//   mapfuse-plan 1
//   sequence <name> | rows <m> | cols <n> | predicted_us <t>
//   scalar <name>
//   buffer <name> <rows> <cols> <input|output|intermediate> <row_indexed 0|1> <scalar 0|1>
//   kernel <name> <variant_tma> <variant_k>
//   <KernelIR text>            (kernel::emit_pseudo_source, ends with its closing "}")
//   end
// Loading re-lowers every KernelIR, so a plan file is also a portable,
// human-readable record of exactly what ran.
#include <sstream>
#include <stdexcept>

#include "mapfuse/kernel.hpp"
#include "mapfuse/planner.hpp"

namespace mapfuse::plan {

std::string save_plan(const b200::NativePlan& p) {
  std::ostringstream o;
  o.precision(17);
  o << "mapfuse-plan 1\n";
  o << "sequence " << (p.sequence.empty() ? "-" : p.sequence) << "\n";
  o << "rows " << p.rows << "\ncols " << p.cols << "\npredicted_us " << p.predicted_us << "\n";
  for (const auto& s : p.scalars) o << "scalar " << s << "\n";
  for (const auto& b : p.buffers) {
    const char* role = b.role == b200::Role::Input ? "input"
                       : b.role == b200::Role::Output ? "output"
                                                      : "intermediate";
    o << "buffer " << b.name << " " << b.rows << " " << b.cols << " " << role << " "
      << (b.row_indexed ? 1 : 0) << " " << (b.scalar ? 1 : 0) << "\n";
  }
  for (size_t i = 0; i < p.kernels.size(); ++i) {
    if (i >= p.kernel_ir.size() || p.kernel_ir[i].empty())
      throw std::invalid_argument("save_plan: kernel " + std::to_string(i) + " has no KernelIR");
    o << "kernel " << p.kernels[i].name << " " << p.kernels[i].variant_tma << " "
      << p.kernels[i].variant_k << "\n"
      << p.kernel_ir[i] << "end\n";
  }
  return o.str();
}

b200::NativePlan load_plan(const std::string& text) {
  std::istringstream in(text);
  std::string line;
  if (!std::getline(in, line) || line != "mapfuse-plan 1")
    throw std::invalid_argument("not a mapfuse plan file (missing 'mapfuse-plan 1')");
  b200::NativePlan p;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    std::istringstream ls(line);
    std::string key;
    ls >> key;
    if (key == "sequence") {
      ls >> p.sequence;
      if (p.sequence == "-") p.sequence.clear();
    } else if (key == "rows") {
      ls >> p.rows;
    } else if (key == "cols") {
      ls >> p.cols;
    } else if (key == "predicted_us") {
      ls >> p.predicted_us;
    } else if (key == "scalar") {
      std::string s;
      ls >> s;
      p.scalars.push_back(s);
    } else if (key == "buffer") {
      b200::BufferSpec b;
      std::string role;
      int rowix = 0, sc = 0;
      ls >> b.name >> b.rows >> b.cols >> role >> rowix >> sc;
      if (!ls) throw std::invalid_argument("plan file: bad buffer line '" + line + "'");
      b.role = role == "input" ? b200::Role::Input
               : role == "output" ? b200::Role::Output
                                  : b200::Role::Intermediate;
      b.row_indexed = rowix != 0;
      b.scalar = sc != 0;
      p.buffers.push_back(b);
    } else if (key == "kernel") {
      std::string name;
      int tma = -1, kk = 0;
      ls >> name >> tma >> kk;
      std::string body, l;
      bool closed = false;
      while (std::getline(in, l)) {
        if (l == "end") {
          closed = true;
          break;
        }
        body += l + "\n";
      }
      if (!closed) throw std::invalid_argument("plan file: kernel '" + name + "' not terminated");
      b200::NativeKernel nk = lower_or_generic(kernel::parse_kernel_text(body));
      nk.name = name;
      nk.variant_tma = tma;
      nk.variant_k = kk;
      p.kernels.push_back(std::move(nk));
      p.kernel_ir.push_back(body);
    } else {
      throw std::invalid_argument("plan file: unknown key '" + key + "'");
    }
  }
  if (p.kernels.empty()) throw std::invalid_argument("plan file has no kernels");
  return p;
}

}  // namespace mapfuse::plan
