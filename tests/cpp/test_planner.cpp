// Planner / selector / codegen / lowering tests (CPU).  Expected fusions are
// SURVEY.md Appendix A (derived from SPEC.md:181-246 + convexity); savings
// examples are SPEC.md:224-225.
#include <algorithm>
#include <random>
#include <set>

#include "doctest.h"
#include "mapfuse/blas.hpp"
#include "mapfuse/kernel.hpp"
#include "mapfuse/planner.hpp"
#include "mapfuse/script.hpp"

using namespace mapfuse;

namespace {
struct Seq {
  script::Script s;
  script::DataDependencyGraph g;
};
Seq load(const std::string& name) {
  Seq q;
  q.s = script::parse_script(blas::build_sequence(name).script_text);
  q.g = script::build_dependency_graph(q.s, blas::default_library());
  return q;
}
std::vector<std::vector<int>> fusion_sets(const std::string& name, plan::Sizes sz = {64, 64}) {
  Seq q = load(name);
  std::vector<std::vector<int>> out;
  for (const auto& f : plan::enumerate_fusions(q.s, q.g, blas::default_library(), sz))
    out.push_back(f.calls);
  return out;
}
using VV = std::vector<std::vector<int>>;
}  // namespace

TEST_CASE("Appendix A: fusions of every Table-1 sequence") {
  CHECK(fusion_sets("AXPYDOT") == VV{{0, 1}});
  CHECK(fusion_sets("VADD") == VV{{0, 1}});
  CHECK(fusion_sets("WAXPBY") == VV{{0, 1}});
  CHECK(fusion_sets("BICGK") == VV{{0, 1}});
  CHECK(fusion_sets("ATAX").empty());
  CHECK(fusion_sets("GEMVER") == VV{{0, 1}});
  CHECK(fusion_sets("GESUMMV") == VV{{0, 1}});
  CHECK(fusion_sets("SGEMV").empty());
  CHECK(fusion_sets("SGEMVT").empty());
  CHECK(fusion_sets("SSCAL").empty());
  CHECK(fusion_sets("MADD").empty());
}

TEST_CASE("fusibility rule ids") {
  const auto& L = blas::default_library();
  Seq atax = load("ATAX");
  auto v = plan::fusibility({0, 1}, atax.s, atax.g, L);
  REQUIRE(v.has_value());
  CHECK(v->rule == "global-barrier-required");
  Seq gv = load("GEMVER");
  v = plan::fusibility({0, 2}, gv.s, gv.g, L);
  REQUIRE(v.has_value());
  CHECK(v->rule == "nesting-mismatch");
  // only convexity rejects these
  v = plan::fusibility({0, 3}, gv.s, gv.g, L);
  REQUIRE(v.has_value());
  CHECK(v->rule == "global-barrier-required");
  v = plan::fusibility({1, 3}, gv.s, gv.g, L);
  REQUIRE(v.has_value());
  Seq sg = load("SGEMVT");
  v = plan::fusibility({0, 2}, sg.s, sg.g, L);
  REQUIRE(v.has_value());
  CHECK(v->rule == "global-barrier-required");
  Seq bi = load("BICGK");
  CHECK(plan::is_fusible({0, 1}, bi.s, bi.g, L));
}

TEST_CASE("block-capacity rule (SPEC.md:195)") {
  const auto& L = blas::default_library();
  Seq bi = load("BICGK");
  // the smallest fused BiCGK kernel: 32x2 threads, A tile + p, q, r, s slices
  const auto k = plan::generate_kernel({0, 1}, bi.s, bi.g, L, [] {
    plan::CodegenParams p;
    p.by = 2;
    p.instances = 1;
    p.overlap = true;
    return p;
  }());
  REQUIRE(k.shared_bytes_total() > 0);
  plan::PlannerOptions tight;
  tight.block_shared_bytes = k.shared_bytes_total() - 4;
  auto v = plan::fusibility({0, 1}, bi.s, bi.g, L, tight);
  REQUIRE(v.has_value());
  CHECK(v->rule == "block-capacity");
  CHECK(v->nodes == std::vector<int>{0, 1});
  CHECK(v->explanation.find("shared memory") != std::string::npos);
  CHECK(plan::enumerate_fusions(bi.s, bi.g, L, {64, 64}, 6, tight).empty());
  tight.block_shared_bytes = k.shared_bytes_total();
  CHECK(plan::is_fusible({0, 1}, bi.s, bi.g, L, tight));
  plan::PlannerOptions few;
  few.max_threads_per_block = 32;  // a depth-2 block is 32 x BY >= 64 threads
  v = plan::fusibility({0, 1}, bi.s, bi.g, L, few);
  REQUIRE(v.has_value());
  CHECK(v->rule == "block-capacity");
  // the structural rules are checked first
  Seq atax = load("ATAX");
  v = plan::fusibility({0, 1}, atax.s, atax.g, L, tight);
  REQUIRE(v.has_value());
  CHECK(v->rule == "global-barrier-required");
}

TEST_CASE("transfer savings (SPEC.md:224-225)") {
  const auto& L = blas::default_library();
  Seq vadd = load("VADD");
  plan::Fusion f;
  f.calls = {0, 1};
  CHECK(plan::transfer_savings(f, vadd.s, vadd.g, L, {32, 1024}) == 2048);
  Seq bi = load("BICGK");
  CHECK(plan::transfer_savings(f, bi.s, bi.g, L, {128, 128}) == 16384);
  Seq ax = load("AXPYDOT");  // z stays a script output: only its load is saved
  CHECK(plan::transfer_savings(f, ax.s, ax.g, L, {32, 1024}) == 1024);
  Seq gs = load("GESUMMV");  // only the shared x
  CHECK(plan::transfer_savings(f, gs.s, gs.g, L, {256, 256}) == 256);
  Seq gv = load("GEMVER");  // B stored (output) but loaded once less
  CHECK(plan::transfer_savings(f, gv.s, gv.g, L, {128, 128}) == 128 * 128);
}

TEST_CASE("selector: the chosen cover is the planner's fusion partition") {
  const auto& L = blas::default_library();
  const auto cm = plan::CostModel::defaults();
  auto kernels = [&](const std::string& n) {
    Seq q = load(n);
    auto c = plan::enumerate_combinations(q.s, q.g, L, {4096, 4096}, cm, 1);
    VV out;
    for (const auto& k : c.at(0).kernels) out.push_back(k.calls);
    return out;
  };
  CHECK(kernels("BICGK") == VV{{0, 1}});
  CHECK(kernels("ATAX") == VV{{0}, {1}});
  CHECK(kernels("GEMVER") == VV{{0, 1}, {2}, {3}});
  CHECK(kernels("GESUMMV") == VV{{0, 1}, {2}});
  CHECK(kernels("SGEMVT") == VV{{0}, {1}, {2}, {3}});
  CHECK(kernels("AXPYDOT") == VV{{0, 1}});
}

TEST_CASE("every enumerated combination is an exact cover in dependency order") {
  const auto& L = blas::default_library();
  const auto cm = plan::CostModel::defaults();
  for (const auto& name : blas::sequence_names()) {
    Seq q = load(name);
    auto all = plan::enumerate_combinations(q.s, q.g, L, {256, 256}, cm, 0);
    REQUIRE(!all.empty());
    for (size_t i = 1; i < all.size(); ++i) CHECK(all[i - 1].predicted_us <= all[i].predicted_us);
    for (const auto& c : all) {
      std::multiset<int> ids;
      std::map<int, size_t> pos;
      for (size_t k = 0; k < c.kernels.size(); ++k)
        for (int id : c.kernels[k].calls) {
          ids.insert(id);
          pos[id] = k;
        }
      CHECK(ids == std::multiset<int>(q.g.nodes.begin(), q.g.nodes.end()));
      for (const auto& e : q.g.edges) CHECK(pos[e.producer] <= pos[e.consumer]);
    }
  }
  Seq v = load("VADD");
  CHECK(plan::count_combinations(v.s, v.g, L, {32, 1024}) == 2);
  Seq gv = load("GEMVER");
  CHECK(plan::count_combinations(gv.s, gv.g, L, {256, 256}) > plan::count_combinations(
                                                                  load("BICGK").s, load("BICGK").g, L, {256, 256}));
}

TEST_CASE("random straight-line scripts: enumeration = brute-force filter") {
  const auto& L = blas::default_library();
  std::mt19937 rng(11);
  const char* fns[] = {"add", "scal", "dot", "waxpby"};
  for (int iter = 0; iter < 200; ++iter) {
    const int n = 2 + static_cast<int>(rng() % 5);
    std::string text = "subvector32 i0, i1";
    for (int i = 0; i < n; ++i) text += ", v" + std::to_string(i);
    text += ";\nfloat a";
    for (int i = 0; i < n; ++i) text += ", r" + std::to_string(i);
    text += ";\ninput i0, i1, a;\n";
    std::vector<std::string> vecs = {"i0", "i1"};
    std::string ret;
    for (int i = 0; i < n; ++i) {
      const std::string f = fns[rng() % 4];
      auto pick = [&] { return vecs[rng() % vecs.size()]; };
      if (f == "add") text += "v" + std::to_string(i) + " = add(" + pick() + ", " + pick() + ");\n";
      if (f == "scal") text += "v" + std::to_string(i) + " = scal(a, " + pick() + ");\n";
      if (f == "waxpby")
        text += "v" + std::to_string(i) + " = waxpby(a, " + pick() + ", 2.0, " + pick() + ");\n";
      if (f == "dot") {
        text += "r" + std::to_string(i) + " = dot(" + pick() + ", " + pick() + ");\n";
        ret += (ret.empty() ? "" : ", ") + std::string("r") + std::to_string(i);
        continue;
      }
      vecs.push_back("v" + std::to_string(i));
      ret += (ret.empty() ? "" : ", ") + std::string("v") + std::to_string(i);
    }
    text += "return " + ret + ";\n";
    auto s = script::parse_script(text);
    auto g = script::build_dependency_graph(s, L);
    auto got = plan::enumerate_fusions(s, g, L, {32, 1024});
    std::set<std::vector<int>> listed;
    for (const auto& f : got) {
      listed.insert(f.calls);
      CHECK(plan::is_fusible(f.calls, s, g, L));
      CHECK(f.saved_words > 0);
    }
    // brute force over all subsets
    const int calls = static_cast<int>(g.nodes.size());
    for (int mask = 1; mask < (1 << calls); ++mask) {
      std::vector<int> set;
      for (int i = 0; i < calls; ++i)
        if (mask >> i & 1) set.push_back(g.nodes[i]);
      if (set.size() < 2) continue;
      // connectivity over edges and shared inputs
      std::set<int> reach{set[0]};
      bool grew = true;
      while (grew) {
        grew = false;
        for (const auto& e : g.edges)
          if (std::count(set.begin(), set.end(), e.producer) && std::count(set.begin(), set.end(), e.consumer) &&
              (reach.count(e.producer) != reach.count(e.consumer))) {
            reach.insert(e.producer);
            reach.insert(e.consumer);
            grew = true;
          }
        for (const auto& si : g.shared_inputs)
          if (si.name != "a" && std::count(set.begin(), set.end(), si.a) &&
              std::count(set.begin(), set.end(), si.b) &&
              (reach.count(si.a) != reach.count(si.b))) {
            reach.insert(si.a);
            reach.insert(si.b);
            grew = true;
          }
      }
      const bool connected = reach.size() == set.size();
      plan::Fusion f;
      f.calls = set;
      const bool expect = connected && plan::is_fusible(set, s, g, L) &&
                          plan::transfer_savings(f, s, g, L, {32, 1024}) > 0;
      CHECK(expect == (listed.count(set) == 1));
    }
  }
}

TEST_CASE("codegen: fused BiCGK follows Algorithm 3") {
  const auto& L = blas::default_library();
  Seq q = load("BICGK");
  auto k = plan::generate_kernel({0, 1}, q.s, q.g, L);
  auto labels = [](const std::vector<kernel::RoutineCallIR>& v) {
    std::vector<std::string> o;
    for (const auto& c : v) o.push_back(c.is_pure_clear() ? "clear " + c.clear_key : c.label);
    return o;
  };
  // p (varies x) hoisted; s (accumulated over row tiles) cleared before the
  // loop and stored after it; q cleared and stored inside the loop
  CHECK(labels(k.prologue) == std::vector<std::string>{"sgemv.load_x", "clear s"});
  CHECK(labels(k.body) == std::vector<std::string>{"sgemv.load_A", "sgemv.compute", "sgemv.store_y",
                                                   "sgemtv.load_x", "sgemtv.compute"});
  CHECK(labels(k.epilogue) == std::vector<std::string>{"sgemtv.store_y"});
  CHECK(k.body[1].clear_key == "q");
  // A is read in two orders -> shared memory, padded stride 33
  bool a_shared = false;
  for (const auto& r : k.shared_regions)
    if (r.key == "A") a_shared = r.stride == 33;
  CHECK(a_shared);
  // the transposed compute read needs a barrier after the load
  CHECK(k.body[1].barrier_before);
  // text round trip is byte-stable
  const std::string t = kernel::emit_pseudo_source(k);
  CHECK(kernel::emit_pseudo_source(kernel::parse_kernel_text(t)) == t);
  // lowering recovers the single-pass row + column reduction
  auto nk = plan::lower_kernel(kernel::parse_kernel_text(t));
  CHECK(nk.kind == b200::NativeKernel::Kind::Matrix);
  CHECK(nk.matrix.mats == std::vector<std::string>{"A"});
  REQUIRE(nk.matrix.rows.size() == 1);
  REQUIRE(nk.matrix.cols.size() == 1);
  CHECK(nk.matrix.rows[0].x == "p");
  CHECK(nk.matrix.rows[0].y == "q");
  CHECK(nk.matrix.cols[0].x == "r");
  CHECK(nk.matrix.cols[0].y == "s");
  // barrier-suppression hook removes them
  plan::CodegenParams np;
  np.barriers = false;
  auto k2 = plan::generate_kernel({0, 1}, q.s, q.g, L, np);
  for (const auto& c : k2.body) CHECK(!c.barrier_before);
}

TEST_CASE("codegen + lowering for every kernel of every plan; text round trips") {
  const auto& L = blas::default_library();
  const auto cm = plan::CostModel::defaults();
  for (const auto& name : blas::sequence_names()) {
    Seq q = load(name);
    for (bool fuse : {true, false}) {
      auto c = plan::enumerate_combinations(q.s, q.g, L, {512, 512}, cm, 1, fuse);
      REQUIRE(c.size() == 1);
      for (const auto& it : c[0].kernels) {
        const std::string t = kernel::emit_pseudo_source(it.kir);
        auto back = kernel::parse_kernel_text(t);
        CHECK(kernel::emit_pseudo_source(back) == t);
        auto nk = plan::lower_kernel(back);
        CHECK(nk.kind == it.native.kind);
        CHECK(nk.inputs() == it.native.inputs());
        CHECK(nk.outputs() == it.native.outputs());
      }
    }
  }
}

TEST_CASE("GEMVER rank stage lowers to one pass: B = A + u1 v1^T + u2 v2^T, t = B^T y") {
  const auto& L = blas::default_library();
  Seq q = load("GEMVER");
  auto nk = plan::lower_kernel(plan::generate_kernel({0, 1}, q.s, q.g, L));
  CHECK(nk.matrix.mats == std::vector<std::string>{"A"});
  CHECK(nk.matrix.rank.size() == 2);
  CHECK(nk.matrix.store == "B");
  REQUIRE(nk.matrix.cols.size() == 1);
  CHECK(nk.matrix.cols[0].x == "y");
  CHECK(nk.matrix.cols[0].y == "t");
  // waxpby(beta, t, 1.0, z): literal folded into the coefficient
  auto x = plan::lower_kernel(plan::generate_kernel({2}, q.s, q.g, L));
  REQUIRE(x.stream.outs.size() == 1);
  CHECK(x.stream.outs[0].coef[0].str() == "1*beta");
  CHECK(x.stream.outs[0].coef[1].str() == "1");
}

TEST_CASE("shape inference propagates through depth-1 calls (rectangular)") {
  const auto& L = blas::default_library();
  auto s = script::parse_script(blas::build_sequence("SGEMV").script_text);
  auto d = blas::infer_shapes(s, L, 64, 96);
  CHECK(d.at("A") == std::make_pair(64, 96));
  CHECK(d.at("x") == std::make_pair(1, 96));
  CHECK(d.at("t") == std::make_pair(1, 64));
  CHECK(d.at("z") == std::make_pair(1, 64));  // the reference sizes z by cols here
  CHECK(d.at("y") == std::make_pair(1, 64));
}
