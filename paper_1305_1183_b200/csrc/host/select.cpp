// host/select.cpp -- B200 cost model (SPEC.md:336-400 retargeted),
// combination selector and the compile pipeline.
//
// Cost model.  The paper predicts max(t_transfer, t_compute) from routine
// micro-benchmarks.  On B200 every kernel here is
// HBM-bound (<= 1 flop/byte), so t = bytes / (eta * BW) + t_launch with BW
// the measured copy bandwidth and eta the per-family efficiency measured on
// B200 (bench.py suite, profiles/r01_sweep_initial.txt, r01_stream_layout.txt) -- the analogue of the
// paper's per-architecture benchmark database.  Modelling launch overhead
// fixes the paper's own AXPYDOT misprediction.
#include <algorithm>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <set>
#include <sstream>

#include "mapfuse/blas.hpp"
#include "mapfuse/planner.hpp"

namespace mapfuse::plan {

CostModel CostModel::defaults() {
  CostModel cm;
  cm.dev = vm::b200_device();
  // measured on B200 (round 1): fraction of the 6545.6 GB/s copy bandwidth
  cm.eta = {
      {"stream", 1.09},            // maps, one CTA per 8 KB block: VADD 1.12, WAXPBY 1.09,
                                   //   SSCAL 1.07, MADD 1.09 (profiles/r01_stream_layout.txt)
      {"stream.dot", 1.00},        // map + dot, persistent grid + ticket: AXPYDOT 1.00
      {"matrix.ldg.read", 1.04},   // BiCGK 1.03, ATAX 1.05, GESUMMV 1.12
      {"matrix.tma.read", 0.95},   // BiCGK 0.92-0.97
      {"matrix.ldg.rank", 0.62},   // GEMVER ger2+sgemtv, register-fed
      {"matrix.tma.rank", 0.99},   // GEMVER ger2+sgemtv, TMA ring, 16 consumer warps, bulk S2G stores
      {"matrix.rowres", 0.88},     // row-resident chain (ATAX one pass, 16384^2)
      {"matrix.rowres.cluster", 0.95},  // ... rows over a CTA cluster (n > 16384), st.async exchange:
                                        //   32768^2 1.08, 131072^2 0.93 (profiles/r02_rowres_variants.txt)
      {"generic.d1", 0.78},        // NVRTC-emitted KernelIR (host/cudagen.cpp), depth 1,
                                   //   prefetch 4 ahead, deferred accumulators: VADD 0.93,
                                   //   AXPYDOT 0.63 (profiles/r02_generic_rewrite.txt)
      {"generic.d2", 0.82},        // ... depth 2 (BY 2, pipelined, proved bounds, round-2 rewrites):
                                   //   BiCGK 0.90, ATAX 0.81, GEMVER 0.81, GESUMMV 0.81
                                   //   (profiles/r02_generic_rewrite.txt)
  };
  if (const char* f = std::getenv("MF_COST_DB")) {
    std::ifstream in(f);
    std::string key;
    double v;
    while (in >> key >> v) cm.eta[key] = v;
  }
  return cm;
}

double CostModel::predict_us(b200::NativeKernel& k, int64_t m, int64_t n) const {
  const double bytes = double(k.bytes_loaded(m, n) + k.bytes_stored(m, n));
  const double bw = dev.hbm_gbs * 1e3;  // bytes per microsecond
  auto t = [&](const char* key) {
    auto it = eta.find(key);
    return bytes / ((it == eta.end() ? 0.9 : it->second) * bw) + dev.launch_us;
  };
  if (k.kind == b200::NativeKernel::Kind::Stream) return t(k.stream.has_dot ? "stream.dot" : "stream");
  if (k.kind == b200::NativeKernel::Kind::Generic)
    return t(k.generic.depth == 1 ? "generic.d1" : "generic.d2");
  if (k.matrix.chain) return t(n > 16384 ? "matrix.rowres.cluster" : "matrix.rowres");
  const bool heavy = !k.matrix.rank.empty() || !k.matrix.store.empty();
  const double ldg = t(heavy ? "matrix.ldg.rank" : "matrix.ldg.read");
  const double tma = t(heavy ? "matrix.tma.rank" : "matrix.tma.read");
  if (tma < ldg) {
    k.variant_tma = 1;
    k.variant_k = heavy ? 4 : 2;
    return tma;
  }
  k.variant_tma = 0;
  k.variant_k = 2;
  return ldg;
}

// Serial iterations for a generic kernel (the paper's ITERS parameter,
// PAPER.md:259).  Each block loops over `iterations` instances, so
// accumulators invariant across iterations are cleared once and added to
// global memory once per block instead of once per tile.  Measured on B200
// (tools/generic_sweep.py, profiles/r01_generic_sweep.txt): ~4 for depth-2
// kernels with accumulators, 1 for depth-2 maps, ~16 for depth-1; block rows
// BY = 4 (32x4 threads) for depth 2.
//
// The iteration count must DIVIDE the iterated grid extent: the epilogue
// runs with it = iterations-1, and an instance beyond the grid skips every
// call (vm.cpp:381-399) -- so with a ragged last band the
// epilogue's stores of the invariant accumulators would be dropped (the
// reference VM drops them too).  For the same reason depth-1 kernels iterate
// only when the element count fills every instance of every block.
// Option "generic_iterations" (>= 1) fixes the count (still made a divisor).
std::pair<int64_t, int64_t> domain_shape(const kernel::KernelIR& k, const script::Script& s,
                                         const lib::Library& L, Sizes sz) {
  const auto shapes = blas::infer_shapes(s, L, static_cast<int>(sz.rows), static_cast<int>(sz.cols));
  auto it = shapes.find(k.domain);
  if (it == shapes.end()) return {k.depth == 2 ? sz.rows : 1, sz.cols};
  return {it->second.first, it->second.second};
}

CodegenParams generic_params(const kernel::KernelIR& k, int64_t dom_rows, int64_t dom_cols) {
  CodegenParams p;
  // 32x2 blocks: measured best once the uninstrumented rewrites apply
  // (profiles/r02_generic_rewrite.txt: BiCGK 16384^2 220 -> 208-214 us, GEMVER
  // 8192^2 153 -> 151 us, ATAX / GESUMMV equal); 32x4 was best for the
  // literal tile algorithm
  p.by = generic_by() > 0 ? generic_by() : 2;
  bool accumulates = false;
  for (const auto* sec : {&k.prologue, &k.epilogue})
    for (const auto& c : *sec) accumulates = accumulates || !c.is_pure_clear() || !c.clear_key.empty();
  int64_t limit = 1, blocks_per_band = 1;
  if (k.depth == 2) {
    limit = std::max<int64_t>(1, dom_rows / 32);  // iterate y
    blocks_per_band = std::max<int64_t>(1, dom_cols / 32);
  } else {
    const int64_t len = dom_rows == 1 ? dom_cols : dom_rows * dom_cols;  // vm.cpp:38
    const int64_t elems = std::max<int64_t>(1, len / 32);
    const int inst = std::max(1, std::min(4, k.instances));
    if (elems % inst != 0) return p;
    limit = elems / inst;
  }
  const int forced = generic_iterations();
  // depth 1: 128 iterations when the kernel reduces (fewer blocks, fewer
  // same-address global atomics: AXPYDOT 2^24 84 / 64 / 61 / 59 us at
  // 16 / 32 / 64 / 128 with the round-2 deferred accumulators,
  // profiles/r02_generic_rewrite.txt), else 16 (VADD 0.94)
  int64_t want = forced >= 1 ? forced : (k.depth == 1 ? (accumulates ? 128 : 16) : (accumulates ? 4 : 1));
  // depth 2 with accumulators: 8 serial iterations while that still leaves
  // >= 16 waves of 4 blocks per SM (generic BiCGK 16384^2: 196 -> 179 us;
  // 8192^2 shapes have too few tiles and measured equal or slower)
  if (forced < 1 && k.depth == 2 && accumulates && (limit / 8) * blocks_per_band >= 148 * 4 * 16) want = 8;
  // keep >= 4 blocks per SM (148 SMs)
  while (want > 1 && (limit / want) * blocks_per_band < 148 * 4 && forced < 1) want /= 2;
  int64_t it = std::max<int64_t>(1, std::min(want, limit));
  while (limit % it) --it;  // largest divisor of the grid extent <= want
  p.iterations = static_cast<int>(it);
  return p;
}

namespace {

struct Candidate {
  std::vector<int> calls;
  Item item;
};

std::vector<Candidate> candidates(const script::Script& s, const script::DataDependencyGraph& g,
                                  const lib::Library& L, Sizes sz, const CostModel& cm,
                                  bool allow_fusion, const PlannerOptions& opt) {
  std::vector<Candidate> out;
  auto add = [&](const std::vector<int>& calls, bool must) {
    Candidate c;
    c.calls = calls;
    try {
      c.item.calls = calls;
      CodegenParams base;
      base.barriers = codegen_barriers();
      c.item.kir = generate_kernel(calls, s, g, L, base);
      c.item.native = lower_or_generic(c.item.kir);
      if (c.item.native.kind == b200::NativeKernel::Kind::Generic) {
        // a reduction result consumed inside the fusion (planner mode b200's
        // row-resident chains) needs the whole row before its consumer runs:
        // only the native row-resident kernel provides that, the generic
        // kernel follows the paper's per-tile semantics
        for (const auto& e : g.edges)
          if (std::find(calls.begin(), calls.end(), e.producer) != calls.end() &&
              std::find(calls.begin(), calls.end(), e.consumer) != calls.end()) {
            const lib::ElementaryFunction* f = nullptr;
            for (const auto& cst : s.calls)
              if (cst.id == e.producer) f = L.find(cst.function);
            if (f && f->is_reduction())
              throw std::invalid_argument("row-resident chain '" + e.name +
                                          "' has no native kernel for this fusion");
          }
        // generic kernels execute the KernelIR as written: pick the
        // implementation parameters (serial iterations) for this size
        const auto dom = domain_shape(c.item.kir, s, L, sz);
        CodegenParams prm = generic_params(c.item.kir, dom.first, dom.second);
        prm.barriers = base.barriers;
        if (prm.iterations != c.item.kir.iterations || prm.by != base.by) {
          c.item.kir = generate_kernel(calls, s, g, L, prm);
          c.item.native = generic_kernel(c.item.kir);
        }
      }
      // a stream kernel over tiles (MADD, flattened) streams m*n elements
      int64_t pm = sz.rows, pn = sz.cols;
      if (c.item.native.kind == b200::NativeKernel::Kind::Stream && !c.item.native.stream.inputs.empty()) {
        auto d = s.declarations.find(c.item.native.stream.inputs[0]);
        if (d != s.declarations.end() && d->second.depth() == 2) {
          pn = sz.rows * sz.cols;
          pm = 1;
        }
      }
      c.item.predicted_us = cm.predict_us(c.item.native, pm, pn);
    } catch (const std::invalid_argument& e) {
      if (must) throw std::invalid_argument("call " + std::to_string(calls[0]) + ": " + e.what());
      return;  // infeasible implementation (the generic emitter rejected it too)
    }
    out.push_back(std::move(c));
  };
  for (int id : g.nodes) add({id}, true);
  if (allow_fusion)
    for (const auto& f : enumerate_fusions(s, g, L, sz, 6, opt)) add(f.calls, false);
  return out;
}

// Topological order of the chosen items (condensed DAG), ties by smallest id.
bool launch_order(const script::DataDependencyGraph& g, std::vector<Item>& items) {
  const size_t n = items.size();
  std::vector<std::set<size_t>> succ(n);
  std::vector<int> indeg(n, 0);
  auto owner = [&](int id) {
    for (size_t i = 0; i < n; ++i)
      if (std::find(items[i].calls.begin(), items[i].calls.end(), id) != items[i].calls.end()) return i;
    return n;
  };
  for (const auto& e : g.edges) {
    const size_t a = owner(e.producer), b = owner(e.consumer);
    if (a != b && a < n && b < n && succ[a].insert(b).second) ++indeg[b];
  }
  std::vector<Item> out;
  std::vector<bool> done(n, false);
  for (size_t step = 0; step < n; ++step) {
    size_t pick = n;
    for (size_t i = 0; i < n; ++i)
      if (!done[i] && indeg[i] == 0 && (pick == n || items[i].calls.front() < items[pick].calls.front()))
        pick = i;
    if (pick == n) return false;  // cycle
    done[pick] = true;
    for (size_t j : succ[pick]) --indeg[j];
    out.push_back(items[pick]);
  }
  items = std::move(out);
  return true;
}

}  // namespace

std::vector<Combination> enumerate_combinations(const script::Script& s,
                                                const script::DataDependencyGraph& g,
                                                const lib::Library& L, Sizes sz,
                                                const CostModel& cm, int k, bool allow_fusion,
                                                const PlannerOptions& opt) {
  const auto cands = candidates(s, g, L, sz, cm, allow_fusion, opt);
  std::vector<Combination> covers;
  std::set<int> covered;
  std::vector<const Candidate*> chosen;
  std::function<void()> rec = [&]() {
    int next = -1;
    for (int id : g.nodes)
      if (!covered.count(id)) {
        next = id;
        break;
      }
    if (next < 0) {
      Combination c;
      for (const auto* x : chosen) {
        c.kernels.push_back(x->item);
        c.predicted_us += x->item.predicted_us;
      }
      if (launch_order(g, c.kernels)) covers.push_back(std::move(c));
      return;
    }
    for (const auto& cand : cands) {
      if (std::find(cand.calls.begin(), cand.calls.end(), next) == cand.calls.end()) continue;
      if (std::any_of(cand.calls.begin(), cand.calls.end(), [&](int id) { return covered.count(id); }))
        continue;
      for (int id : cand.calls) covered.insert(id);
      chosen.push_back(&cand);
      rec();
      chosen.pop_back();
      for (int id : cand.calls) covered.erase(id);
    }
  };
  rec();
  std::stable_sort(covers.begin(), covers.end(), [](const Combination& a, const Combination& b) {
    if (a.predicted_us != b.predicted_us) return a.predicted_us < b.predicted_us;
    if (a.kernels.size() != b.kernels.size()) return a.kernels.size() < b.kernels.size();
    return false;
  });
  if (k > 0 && static_cast<int>(covers.size()) > k) covers.resize(static_cast<size_t>(k));
  return covers;
}

uint64_t count_combinations(const script::Script& s, const script::DataDependencyGraph& g,
                            const lib::Library& L, Sizes sz) {
  const CostModel cm = CostModel::defaults();
  uint64_t n = 0;
  for (const auto& c : enumerate_combinations(s, g, L, sz, cm, 0)) {
    uint64_t ways = 1;  // implementation variants per kernel (matrix: register-fed / TMA)
    for (const auto& it : c.kernels) ways *= it.native.kind == b200::NativeKernel::Kind::Matrix ? 2 : 1;
    n += ways;
  }
  return n;
}

namespace {

b200::NativePlan plan_from_combination(const script::Script& s, const lib::Library& L, int m, int n,
                                       const Combination& best) {
  b200::NativePlan plan;
  plan.rows = m;
  plan.cols = n;
  plan.predicted_us = best.predicted_us;
  for (size_t i = 0; i < best.kernels.size(); ++i) {
    b200::NativeKernel nk = best.kernels[i].native;
    std::string label = "k" + std::to_string(i) + "[";
    for (size_t j = 0; j < best.kernels[i].calls.size(); ++j) {
      const int id = best.kernels[i].calls[j];
      for (const auto& c : s.calls)
        if (c.id == id) label += (j ? "+" : "") + c.function;
    }
    nk.name = label + "]";
    plan.kernels.push_back(std::move(nk));
    plan.kernel_ir.push_back(kernel::emit_pseudo_source(best.kernels[i].kir));
  }
  const auto shapes = blas::infer_shapes(s, L, m, n);
  const auto roles = blas::vector_roles(s, L);
  for (const auto& [name, spec] : s.declarations) {
    const bool input = std::find(s.inputs.begin(), s.inputs.end(), name) != s.inputs.end();
    const bool output = std::find(s.outputs.begin(), s.outputs.end(), name) != s.outputs.end();
    if (spec.kind == lib::ElemKind::Scalar && input) {
      plan.scalars.push_back(name);
      continue;
    }
    bool used = input || output;
    for (const auto& k : plan.kernels) {
      auto in = k.inputs(), out = k.outputs();
      used = used || std::find(in.begin(), in.end(), name) != in.end() ||
             std::find(out.begin(), out.end(), name) != out.end();
    }
    if (!used) continue;
    b200::BufferSpec b;
    b.name = name;
    b.rows = shapes.at(name).first;
    b.cols = shapes.at(name).second;
    b.scalar = spec.kind == lib::ElemKind::Scalar;
    b.role = input ? b200::Role::Input : (output ? b200::Role::Output : b200::Role::Intermediate);
    b.row_indexed = roles.at(name) == 'r';
    plan.buffers.push_back(b);
  }
  return plan;
}

struct Parsed {
  script::Script s;
  script::DataDependencyGraph g;
};

Parsed parse_checked(const std::string& script_text, const lib::Library& L) {
  Parsed p;
  p.s = script::parse_script(script_text);
  p.g = script::build_dependency_graph(p.s, L);
  auto diags = script::validate(p.s, p.g, L);
  if (!diags.empty()) {
    std::string msg = "script validation failed:";
    for (const auto& d : diags) msg += "\n  [" + d.rule + "] " + d.where + ": " + d.message;
    throw std::invalid_argument(msg);
  }
  // Dead-call elimination: a call none of whose results is returned or
  // (transitively) consumed has no observable effect; it is not planned.
  // Call ids are kept, so graph edges and kernel labels stay stable.
  std::set<std::string> needed(p.s.outputs.begin(), p.s.outputs.end());
  std::vector<script::CallStatement> live;
  for (auto it = p.s.calls.rbegin(); it != p.s.calls.rend(); ++it) {
    const bool used = std::any_of(it->results.begin(), it->results.end(),
                                  [&](const std::string& r) { return needed.count(r) > 0; });
    if (!used) continue;
    for (const auto& a : it->arguments) needed.insert(a);
    live.push_back(*it);
  }
  if (live.size() != p.s.calls.size()) {
    std::reverse(live.begin(), live.end());
    p.s.calls = std::move(live);
    p.g = script::build_dependency_graph(p.s, L);
  }
  return p;
}

}  // namespace

b200::NativePlan compile(const std::string& script_text, const lib::Library& L, int rows, int cols,
                         int mode) {
  return compile_ranked(script_text, L, rows, cols, mode, 0);
}

b200::NativePlan compile_ranked(const std::string& script_text, const lib::Library& L, int rows,
                                int cols, int mode, int rank) {
  Parsed p = parse_checked(script_text, L);
  const int m = (rows + 31) / 32 * 32, n = (cols + 31) / 32 * 32;
  const CostModel cm = CostModel::defaults();
  PlannerOptions opt;
  opt.row_resident = mode == 2;
  opt.cols = n;
  auto combos = enumerate_combinations(p.s, p.g, L, Sizes{m, n}, cm, rank + 1, mode != 1, opt);
  if (combos.empty()) throw std::invalid_argument("no executable combination for this script");
  if (rank < 0 || rank >= static_cast<int>(combos.size()))
    throw std::invalid_argument("combination rank " + std::to_string(rank) + " out of range (" +
                                std::to_string(combos.size()) + " combinations)");
  return plan_from_combination(p.s, L, m, n, combos[static_cast<size_t>(rank)]);
}

std::vector<FusionImplementation> kernel_implementations(const b200::NativePlan& p, int k) {
  if (p.script_text.empty())
    throw std::invalid_argument("plan carries no script (made from KernelIR text or a plan file)");
  if (k < 0 || k >= static_cast<int>(p.kernels.size())) throw std::invalid_argument("kernel index out of range");
  lib::Library own;
  const lib::Library* L = &blas::default_library();
  if (!p.manifest.empty()) {
    own = lib::load_library(p.manifest);
    L = &own;
  }
  Parsed ps = parse_checked(p.script_text, *L);
  return enumerate_implementations(p.kernels[k].calls, ps.s, ps.g, *L, Sizes{p.rows, p.cols});
}

void set_kernel_implementation(b200::NativePlan& p, int k, const FusionImplementation& impl) {
  if (k < 0 || k >= static_cast<int>(p.kernels.size())) throw std::invalid_argument("kernel index out of range");
  b200::NativeKernel nk = lower_or_generic(impl.kir);
  nk.name = p.kernels[k].name;
  nk.calls = p.kernels[k].calls;
  CostModel::defaults().predict_us(nk, p.rows, p.cols);
  p.kernels[k] = std::move(nk);
  if (static_cast<int>(p.kernel_ir.size()) > k) p.kernel_ir[k] = kernel::emit_pseudo_source(impl.kir);
}

int64_t count_implementation_space(const std::string& script_text, const lib::Library& L, int rows,
                                   int cols) {
  // Table 4 "Impl. count" analogue: covers x implementation
  // choices -- every kernel of a cover multiplies in the number of its
  // implementations (implementation generator, at this size).
  Parsed p = parse_checked(script_text, L);
  const int m = (rows + 31) / 32 * 32, n = (cols + 31) / 32 * 32;
  std::map<std::vector<int>, int64_t> impls;
  int64_t total = 0;
  for (const auto& c : enumerate_combinations(p.s, p.g, L, Sizes{m, n}, CostModel::defaults(), 0)) {
    int64_t ways = 1;
    for (const auto& it : c.kernels) {
      auto f = impls.find(it.calls);
      if (f == impls.end())
        f = impls.emplace(it.calls, static_cast<int64_t>(
                                        enumerate_implementations(it.calls, p.s, p.g, L, Sizes{m, n}).size()))
                .first;
      ways *= std::max<int64_t>(1, f->second);
    }
    total += ways;
  }
  return total;
}

int64_t count_covers(const std::string& script_text, const lib::Library& L, int rows, int cols) {
  Parsed p = parse_checked(script_text, L);
  const int m = (rows + 31) / 32 * 32, n = (cols + 31) / 32 * 32;
  return static_cast<int64_t>(
      enumerate_combinations(p.s, p.g, L, Sizes{m, n}, CostModel::defaults(), 0).size());
}

}  // namespace mapfuse::plan
