// host/planner.cpp -- fusion planner: fusibility rules,
// transfer savings, enumeration of connected fusible subsets.
#include <algorithm>
#include <functional>
#include <set>

#include "mapfuse/blas.hpp"
#include "mapfuse/planner.hpp"

namespace mapfuse::plan {

namespace {

const script::CallStatement& call_of(const script::Script& s, int id) {
  for (const auto& c : s.calls)
    if (c.id == id) return c;
  throw std::invalid_argument("no call with id " + std::to_string(id));
}

bool contains(const std::vector<int>& v, int x) { return std::find(v.begin(), v.end(), x) != v.end(); }

}  // namespace

namespace {
// Row-resident exception (PlannerOptions::row_resident): e carries a row
// reduction's result into a column reduction of the same tile.
bool row_resident_edge(const script::Edge& e, const script::Script& s, const lib::Library& L,
                       const PlannerOptions& opt) {
  if (!opt.row_resident || opt.cols <= 0 || opt.cols > opt.row_resident_max_cols) return false;
  const auto& pc = call_of(s, e.producer);
  const auto& cc = call_of(s, e.consumer);
  const lib::ElementaryFunction* pf = L.find(pc.function);
  const lib::ElementaryFunction* cf = L.find(cc.function);
  if (!pf || !cf || pf->depth != 2 || cf->depth != 2) return false;
  // producer: accumulable row-indexed output (varies y)
  const lib::ElementDecl* po = nullptr;
  for (size_t i = 0; i < pc.results.size(); ++i)
    if (pc.results[i] == e.name) po = pf->element(pf->results[i]);
  if (!po || !po->accumulable || !po->varies.y || po->varies.x) return false;
  // consumer: reads it as a row-indexed vector, and produces a column output
  const lib::ElementDecl* ci = nullptr;
  std::string ptile, ctile;
  for (size_t i = 0; i < pc.arguments.size(); ++i)
    if (!pf->args[i].is_scalar && pf->element(pf->args[i].name)->kind == lib::ElemKind::Tile32x32)
      ptile = pc.arguments[i];
  for (size_t i = 0; i < cc.arguments.size(); ++i) {
    if (cf->args[i].is_scalar) continue;
    const lib::ElementDecl* d = cf->element(cf->args[i].name);
    if (cc.arguments[i] == e.name) ci = d;
    if (d->kind == lib::ElemKind::Tile32x32) ctile = cc.arguments[i];
  }
  if (!ci || !ci->varies.y || ci->varies.x || ptile.empty() || ptile != ctile) return false;
  for (const auto& r : cf->results) {
    const lib::ElementDecl* d = cf->element(r);
    if (!d || !d->accumulable || !d->varies.x || d->varies.y) return false;
  }
  return true;
}
}  // namespace

std::optional<ConstraintViolation> fusibility(const std::vector<int>& nodes_in,
                                              const script::Script& s,
                                              const script::DataDependencyGraph& g,
                                              const lib::Library& L, const PlannerOptions& opt) {
  std::vector<int> nodes = nodes_in;
  std::sort(nodes.begin(), nodes.end());
  if (nodes.size() < 2) return ConstraintViolation{"no-savings", nodes, "a fusion needs two calls"};
  // equal nesting depth (section 3.2.3)
  int depth = -1;
  for (int id : nodes) {
    const lib::ElementaryFunction* f = L.find(call_of(s, id).function);
    if (!f) throw std::invalid_argument("unknown function in call " + std::to_string(id));
    if (depth >= 0 && f->depth != depth)
      return ConstraintViolation{"nesting-mismatch", nodes,
                                 "members have different nesting depths (" + std::to_string(depth) +
                                     " vs " + std::to_string(f->depth) + ")"};
    depth = f->depth;
  }
  // no member consumes the final result of a member reduction (section 3.2)
  for (const auto& e : g.edges)
    if (contains(nodes, e.producer) && contains(nodes, e.consumer)) {
      const lib::ElementaryFunction* f = L.find(call_of(s, e.producer).function);
      if (f->is_reduction() && !row_resident_edge(e, s, L, opt))
        return ConstraintViolation{"global-barrier-required", {e.producer, e.consumer},
                                   "'" + e.name + "' is a reduction result consumed inside the fusion"};
    }
  // convexity: no dependency path may leave the set and re-enter it
  for (int out : g.nodes) {
    if (contains(nodes, out)) continue;
    bool from = false, to = false;
    for (int n : nodes) {
      from = from || g.has_path(n, out);
      to = to || g.has_path(out, n);
    }
    if (from && to)
      return ConstraintViolation{"global-barrier-required", nodes,
                                 "call " + std::to_string(out) +
                                     " lies on a path that leaves and re-enters the set"};
  }
  // block capacity: even the fusion's smallest kernel must fit one block
  CodegenParams small;
  small.by = 2;
  small.instances = 1;
  small.iterations = 1;
  small.overlap = true;
  kernel::KernelIR k;
  try {
    k = generate_kernel(nodes, s, g, L, small);
  } catch (const std::exception&) {
    return std::nullopt;  // not expressible as one Algorithm 1/2 kernel: lowering decides
  }
  if (k.shared_bytes_total() > opt.block_shared_bytes || k.threads() > opt.max_threads_per_block)
    return ConstraintViolation{"block-capacity", nodes,
                               "smallest fused kernel needs " + std::to_string(k.shared_bytes_total()) +
                                   " B shared memory and " + std::to_string(k.threads()) +
                                   " threads per block (capacity " +
                                   std::to_string(opt.block_shared_bytes) + " B, " +
                                   std::to_string(opt.max_threads_per_block) + " threads)"};
  return std::nullopt;
}

std::map<std::string, int64_t> element_words(const script::Script& s, const lib::Library& L,
                                             Sizes sz) {
  std::map<std::string, int64_t> w;
  for (const auto& [name, dims] :
       blas::infer_shapes(s, L, static_cast<int>(sz.rows), static_cast<int>(sz.cols)))
    w[name] = static_cast<int64_t>(dims.first) * dims.second;
  return w;
}

int64_t transfer_savings(const Fusion& f, const script::Script& s,
                         const script::DataDependencyGraph& g, const lib::Library& L, Sizes sz) {
  const auto words = element_words(s, L, sz);
  auto W = [&](const std::string& n) {
    auto it = words.find(n);
    return it == words.end() ? int64_t(0) : it->second;
  };
  int64_t saved = 0;
  std::set<std::string> produced_inside;
  for (int id : f.calls)
    for (const auto& r : call_of(s, id).results) produced_inside.insert(r);
  // internal dataflow: every member consumer's load disappears; the store
  // disappears too unless the value is a script output or read outside
  for (const auto& v : produced_inside) {
    int inside = 0, outside = 0;
    for (const auto& e : g.edges)
      if (e.name == v) (contains(f.calls, e.consumer) ? inside : outside) += 1;
    if (inside == 0) continue;
    saved += inside * W(v);
    const bool is_output = std::find(s.outputs.begin(), s.outputs.end(), v) != s.outputs.end();
    if (!is_output && outside == 0) saved += W(v);
  }
  // shared read-only inputs: k readers -> k - 1 loads saved
  std::map<std::string, int> readers;
  for (int id : f.calls) {
    std::set<std::string> seen;
    for (const auto& a : call_of(s, id).arguments) {
      if (script::is_numeric_literal(a) || produced_inside.count(a)) continue;
      auto d = s.declarations.find(a);
      if (d != s.declarations.end() && d->second.kind == lib::ElemKind::Scalar) continue;
      if (seen.insert(a).second) ++readers[a];
    }
  }
  for (const auto& [n, k] : readers)
    if (k > 1) saved += (k - 1) * W(n);
  return saved;
}

std::vector<Fusion> enumerate_fusions(const script::Script& s, const script::DataDependencyGraph& g,
                                      const lib::Library& L, Sizes sz, int max_size,
                                      const PlannerOptions& opt) {
  const std::vector<int> ids = g.nodes;
  const int n = static_cast<int>(ids.size());
  if (n > 24) throw std::invalid_argument("enumerate_fusions: script too long (> 24 calls)");
  // undirected adjacency over edges + shared inputs
  std::vector<std::vector<int>> adj(n);
  auto pos = [&](int id) { return static_cast<int>(std::find(ids.begin(), ids.end(), id) - ids.begin()); };
  for (const auto& e : g.edges) {
    adj[pos(e.producer)].push_back(pos(e.consumer));
    adj[pos(e.consumer)].push_back(pos(e.producer));
  }
  for (const auto& si : g.shared_inputs) {
    // a shared scalar parameter saves nothing and does not make calls fusible
    auto d = s.declarations.find(si.name);
    if (d != s.declarations.end() && d->second.kind == lib::ElemKind::Scalar) continue;
    adj[pos(si.a)].push_back(pos(si.b));
    adj[pos(si.b)].push_back(pos(si.a));
  }
  std::vector<Fusion> out;
  for (uint32_t mask = 1; mask < (1u << n); ++mask) {
    const int bits = __builtin_popcount(mask);
    if (bits < 2 || bits > max_size) continue;
    // connectivity
    const int first = __builtin_ctz(mask);
    uint32_t seen = 1u << first;
    std::vector<int> todo{first};
    while (!todo.empty()) {
      const int v = todo.back();
      todo.pop_back();
      for (int w : adj[v])
        if ((mask >> w & 1u) && !(seen >> w & 1u)) {
          seen |= 1u << w;
          todo.push_back(w);
        }
    }
    if (seen != mask) continue;
    Fusion f;
    for (int i = 0; i < n; ++i)
      if (mask >> i & 1u) f.calls.push_back(ids[i]);
    if (fusibility(f.calls, s, g, L, opt)) continue;
    for (const auto& e : g.edges)
      if (contains(f.calls, e.producer) && contains(f.calls, e.consumer)) f.internal.push_back(e);
    for (const auto& si : g.shared_inputs) {
      auto d = s.declarations.find(si.name);
      if (d != s.declarations.end() && d->second.kind == lib::ElemKind::Scalar) continue;
      if (contains(f.calls, si.a) && contains(f.calls, si.b) &&
          std::find(f.shared.begin(), f.shared.end(), si.name) == f.shared.end())
        f.shared.push_back(si.name);
    }
    f.saved_words = transfer_savings(f, s, g, L, sz);
    if (f.saved_words <= 0) continue;
    out.push_back(std::move(f));
  }
  std::sort(out.begin(), out.end(), [](const Fusion& a, const Fusion& b) { return a.calls < b.calls; });
  return out;
}

}  // namespace mapfuse::plan
