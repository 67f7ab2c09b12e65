// host/blas.cpp -- sequence registry, shape inference, input generation.
#include "mapfuse/blas.hpp"

#include <algorithm>
#include <cctype>
#include <functional>
#include <numeric>
#include <random>
#include <stdexcept>

namespace mapfuse::builtin {
std::string manifest();
std::map<std::string, std::string> scripts();
std::string device_config();
}  // namespace mapfuse::builtin

namespace mapfuse::blas {

std::string library_manifest() { return builtin::manifest(); }
std::string default_device_config_text() { return builtin::device_config(); }

const lib::Library& default_library() {
  static const lib::Library L = lib::load_library(library_manifest());
  return L;
}

namespace {
// Table-1 names -> script key and fusibility tag (Table 1).
const std::map<std::string, std::pair<const char*, const char*>>& suite() {
  static const std::map<std::string, std::pair<const char*, const char*>> m = {
      {"AXPYDOT", {"axpydot", "FS"}}, {"ATAX", {"atax", ""}},       {"BICGK", {"bicgk", "F"}},
      {"SGEMV", {"sgemv", "B"}},      {"SGEMVT", {"sgemvt", "(S)"}}, {"SSCAL", {"sscal", "B"}},
      {"GEMVER", {"gemver", "FS"}},   {"GESUMMV", {"gesummv", "(F)"}}, {"MADD", {"madd", "S"}},
      {"VADD", {"vadd", "FS"}},       {"WAXPBY", {"waxpby", "F"}},
  };
  return m;
}

int pad32(int v) { return (v + 31) / 32 * 32; }
}  // namespace

std::vector<std::string> sequence_names() {
  std::vector<std::string> v;
  for (const auto& [k, _] : suite()) v.push_back(k);
  return v;
}

SequenceCase build_sequence(const std::string& name) {
  std::string up = name;
  std::transform(up.begin(), up.end(), up.begin(), [](unsigned char c) { return std::toupper(c); });
  if (up == "BICG") up = "BICGK";
  auto it = suite().find(up);
  if (it == suite().end()) throw std::runtime_error("unknown sequence '" + name + "'");
  static const std::map<std::string, std::string> texts = builtin::scripts();
  return {up, texts.at(it->second.first), it->second.second};
}

const std::vector<float>& Problem::buffer(const std::string& name) const {
  auto it = buffers.find(name);
  if (it == buffers.end()) throw std::runtime_error("no buffer '" + name + "'");
  return it->second;
}

std::map<std::string, char> vector_roles(const script::Script& s, const lib::Library& L) {
  // union-find over vector names tied together by depth-1 calls
  std::map<std::string, std::string> parent;
  std::function<std::string(const std::string&)> root = [&](const std::string& x) {
    auto it = parent.find(x);
    if (it == parent.end() || it->second == x) return x;
    return it->second = root(it->second);
  };
  auto unite = [&](const std::string& a, const std::string& b) { parent[root(a)] = root(b); };
  for (const auto& [n, spec] : s.declarations) parent[n] = n;
  auto bound = [&](const script::CallStatement& c, const lib::ElementaryFunction* f) {
    std::vector<std::pair<std::string, const lib::ElementDecl*>> v;
    for (size_t i = 0; i < c.arguments.size() && i < f->args.size(); ++i)
      if (!f->args[i].is_scalar) v.push_back({c.arguments[i], f->element(f->args[i].name)});
    for (size_t i = 0; i < c.results.size() && i < f->results.size(); ++i)
      v.push_back({c.results[i], f->element(f->results[i])});
    return v;
  };
  for (const auto& c : s.calls) {
    const lib::ElementaryFunction* f = L.find(c.function);
    if (!f || f->depth != 1) continue;
    std::string first;
    for (const auto& [n, d] : bound(c, f))
      if (d && d->kind == lib::ElemKind::Subvector32) {
        if (first.empty()) first = n;
        else unite(n, first);
      }
  }
  std::map<std::string, char> rootrole;
  for (const auto& c : s.calls) {
    const lib::ElementaryFunction* f = L.find(c.function);
    if (!f || f->depth != 2) continue;
    for (const auto& [n, d] : bound(c, f))
      if (d && d->kind == lib::ElemKind::Subvector32) rootrole.emplace(root(n), d->varies.y ? 'r' : 'c');
  }
  std::map<std::string, char> roles;
  for (const auto& [n, spec] : s.declarations) {
    if (spec.kind == lib::ElemKind::Tile32x32) roles[n] = 't';
    else if (spec.kind == lib::ElemKind::Scalar) roles[n] = 's';
    else {
      auto it = rootrole.find(root(n));
      roles[n] = it == rootrole.end() ? 'c' : it->second;
    }
  }
  return roles;
}

std::map<std::string, std::pair<int, int>> infer_shapes(const script::Script& s,
                                                        const lib::Library& L, int rows, int cols) {
  std::map<std::string, std::pair<int, int>> dims;
  for (const auto& [n, role] : vector_roles(s, L)) {
    switch (role) {
      case 't': dims[n] = {rows, cols}; break;
      case 's': dims[n] = {1, 1}; break;
      case 'r': dims[n] = {1, rows}; break;
      default: dims[n] = {1, cols};
    }
  }
  return dims;
}

Problem make_problem(const script::Script& s, int rows, int cols, uint32_t seed) {
  Problem p;
  p.rows = pad32(rows);
  p.cols = pad32(cols);
  p.dims = infer_shapes(s, default_library(), p.rows, p.cols);
  std::mt19937 rng(seed);
  std::uniform_real_distribution<float> U(-1.0f, 1.0f);
  for (const auto& n : s.inputs) {
    if (s.declarations.at(n).kind == lib::ElemKind::Scalar) {
      p.scalars[n] = 0.25f + 0.5f * std::abs(U(rng));
      continue;
    }
    const auto [r, c] = p.dims[n];
    std::vector<float> b(static_cast<size_t>(r) * c);
    for (auto& v : b) v = U(rng);
    p.buffers[n] = std::move(b);
  }
  for (const auto& [n, spec] : s.declarations) {
    if (p.buffers.count(n) || p.scalars.count(n)) continue;
    const auto [r, c] = p.dims[n];
    p.buffers[n] = std::vector<float>(static_cast<size_t>(r) * c, 0.0f);
  }
  return p;
}

}  // namespace mapfuse::blas
