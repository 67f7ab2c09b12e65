// host/codegen.cpp -- kernel code generation (PAPER.md
// Algorithms 1 and 2): a set of calls -> KernelIR.
//
//  * routine order: per call (script order) its loads, its compute, its
//    stores; loads of values produced inside the kernel are elided (the
//    consumer reads the producer's on-chip copy), loads of an input already
//    loaded by an earlier member are shared (BiCGK's single read of A);
//  * hoisting (Algorithm 1): loads of inputs invariant along the iterated
//    grid dimension go to the prologue; reduction outputs accumulated across
//    iterations are cleared in the prologue and stored in the epilogue;
//  * memory plan: an element lives in registers iff every routine touching
//    it uses the same single-thread mapping (section 3.2.3), otherwise in
//    shared memory (tiles accessed in two orders at stride 33);
//  * barriers (section 4.3.3 condition 1): before a routine that reads an
//    element written since the last barrier under a different mapping;
//  * macros BY / IPB / ITERS are bound, element names become storage keys
//    (= script names), scalar parameters become script scalars or literals.
#include <algorithm>
#include <functional>
#include <set>
#include <stdexcept>

#include "mapfuse/planner.hpp"

namespace mapfuse::plan {

namespace {

struct Bound {
  const script::CallStatement* call = nullptr;
  const lib::ElementaryFunction* f = nullptr;
  std::map<std::string, std::string> name;  // function element -> script name
  std::vector<std::string> scalar_arg;      // per function scalar param: script name or literal
};

enum class Sec { Pro, Loop, Epi };

struct Planned {
  Sec sec;
  kernel::RoutineCallIR ir;
  const lib::Routine* routine = nullptr;  // nullptr for a pure clear
  const Bound* b = nullptr;
};

ir::Program rewrite(const ir::Program& body, const Bound& b, const std::map<std::string, int64_t>& macros,
                    const std::vector<std::string>& kernel_params) {
  ir::Program p = ir::substitute_macros(body, macros);
  for (auto& e : p.elements) {
    auto it = b.name.find(e.name);
    if (it != b.name.end()) e.name = it->second;
  }
  for (auto& fn : p.floats) {
    if (fn.op != ir::FloatOp::Param) continue;
    const std::string& arg = b.scalar_arg.at(static_cast<size_t>(fn.slot));
    if (script::is_numeric_literal(arg)) {
      fn.op = ir::FloatOp::Const;
      fn.value = std::stof(arg);
      fn.slot = -1;
    } else {
      fn.slot = static_cast<int32_t>(std::find(kernel_params.begin(), kernel_params.end(), arg) -
                                     kernel_params.begin());
    }
  }
  p.params = kernel_params;
  return p;
}

}  // namespace

namespace {

// Topological orders of the loop items (indices into the default loop order)
// under `before[j]` = items that must precede j; DFS, lexicographic, <= cap.
void topo_orders(const std::vector<std::vector<int>>& before, int cap,
                 std::vector<std::vector<int>>* out) {
  const int n = static_cast<int>(before.size());
  std::vector<int> cur;
  std::vector<bool> used(n, false);
  std::function<void()> rec = [&]() {
    if (static_cast<int>(out->size()) >= cap) return;
    if (static_cast<int>(cur.size()) == n) {
      out->push_back(cur);
      return;
    }
    for (int j = 0; j < n; ++j) {
      if (used[j]) continue;
      if (std::any_of(before[j].begin(), before[j].end(), [&](int i) { return !used[i]; })) continue;
      used[j] = true;
      cur.push_back(j);
      rec();
      cur.pop_back();
      used[j] = false;
    }
  };
  rec();
}

kernel::KernelIR generate_impl(const std::vector<int>& calls_in, const script::Script& s,
                               const script::DataDependencyGraph& g, const lib::Library& L,
                               const CodegenParams& prm, std::vector<std::vector<int>>* orders,
                               int cap) {
  std::vector<int> calls = calls_in;
  std::sort(calls.begin(), calls.end());
  if (calls.empty()) throw std::invalid_argument("generate_kernel: no calls");

  // ---- bind every call
  std::vector<Bound> bs;
  int depth = -1, max_inst = 1 << 20;
  for (int id : calls) {
    Bound b;
    for (const auto& c : s.calls)
      if (c.id == id) b.call = &c;
    if (!b.call) throw std::invalid_argument("generate_kernel: no call " + std::to_string(id));
    b.f = L.find(b.call->function);
    if (!b.f) throw std::invalid_argument("generate_kernel: unknown function " + b.call->function);
    if (depth >= 0 && b.f->depth != depth)
      throw std::invalid_argument("generate_kernel: members differ in nesting depth");
    depth = b.f->depth;
    max_inst = std::min(max_inst, b.f->max_instances);
    for (size_t i = 0; i < b.f->args.size(); ++i) {
      if (b.f->args[i].is_scalar) b.scalar_arg.push_back(b.call->arguments[i]);
      else b.name[b.f->args[i].name] = b.call->arguments[i];
    }
    for (size_t i = 0; i < b.f->results.size(); ++i) b.name[b.f->results[i]] = b.call->results[i];
    bs.push_back(std::move(b));
  }
  const int instances = depth == 1 ? std::max(1, std::min(prm.instances, max_inst)) : 1;
  const std::map<std::string, int64_t> macros{
      {"BY", prm.by}, {"IPB", instances}, {"ITERS", prm.iterations}};

  std::set<std::string> produced;
  for (const auto& b : bs)
    for (const auto& r : b.call->results) produced.insert(r);
  auto in_set = [&](int id) { return std::find(calls.begin(), calls.end(), id) != calls.end(); };
  auto needs_store = [&](const std::string& v) {
    if (std::find(s.outputs.begin(), s.outputs.end(), v) != s.outputs.end()) return true;
    return std::any_of(g.edges.begin(), g.edges.end(),
                       [&](const script::Edge& e) { return e.name == v && !in_set(e.consumer); });
  };
  std::vector<std::string> params;
  for (const auto& b : bs)
    for (const auto& a : b.scalar_arg)
      if (!script::is_numeric_literal(a) && std::find(params.begin(), params.end(), a) == params.end())
        params.push_back(a);
  // invariant along the iterated dimension (depth 2 iterates over row tiles, y)
  auto invariant = [&](const lib::ElementDecl& d) { return depth == 2 ? !d.varies.y : !d.varies.x; };

  // ---- routine order with hoisting
  std::vector<Planned> order;
  std::set<std::string> loaded;
  auto make = [&](const Bound& b, const lib::Routine& r, Sec sec) {
    Planned pl;
    pl.sec = sec;
    pl.routine = &r;
    pl.b = &b;
    pl.ir.label = b.f->name + "." + r.id();
    pl.ir.call_id = b.call->id;
    pl.ir.kind = r.kind;
    pl.ir.routine_px = b.f->par_x;
    pl.ir.routine_py = b.f->par_y_is_block ? prm.by : 1;
    pl.ir.remap = instances > 1 ? kernel::Remap::FlatSplit : kernel::Remap::Identity;
    pl.ir.body = rewrite(r.body, b, macros, params);
    return pl;
  };
  for (const auto& b : bs) {
    for (const auto& d : b.f->elements) {
      if (d.is_output || d.kind == lib::ElemKind::Scalar) continue;
      const std::string& v = b.name.at(d.name);
      if (produced.count(v) || !loaded.insert(v).second) continue;
      const lib::Routine* r = b.f->routine(lib::RoutineKind::Load, d.name, 1);
      if (!r) throw std::invalid_argument(b.f->name + " has no load routine for " + d.name);
      order.push_back(make(b, *r, invariant(d) ? Sec::Pro : Sec::Loop));
    }
    const lib::Routine* comp = b.f->routine(lib::RoutineKind::Compute, "", 1);
    if (!comp) throw std::invalid_argument(b.f->name + " has no compute routine");
    Planned pc = make(b, *comp, Sec::Loop);
    for (const auto& d : b.f->elements) {
      if (!d.is_output || !d.accumulable) continue;
      const std::string& v = b.name.at(d.name);
      if (invariant(d)) {  // accumulated across iterations: clear once, store once
        Planned clr;
        clr.sec = Sec::Pro;
        clr.ir.clear_key = v;
        clr.b = &b;
        order.push_back(std::move(clr));
      } else {
        pc.ir.clear_key = v;
        pc.ir.barrier_after_clear = prm.barriers;
      }
    }
    order.push_back(std::move(pc));
    for (const auto& d : b.f->elements) {
      if (!d.is_output) continue;
      const std::string& v = b.name.at(d.name);
      if (!needs_store(v)) continue;
      const lib::Routine* r = b.f->routine(lib::RoutineKind::Store, d.name, 1);
      if (!r) throw std::invalid_argument(b.f->name + " has no store routine for " + d.name);
      order.push_back(make(b, *r, d.accumulable && invariant(d) ? Sec::Epi : Sec::Loop));
    }
  }

  // ---- routine order of the loop body: item j must follow
  // item i (i before j in the default order) when they share an on-chip
  // element one of them writes (read-after-write, write-after-read,
  // write-after-write).
  auto touched = [&](const Planned& pl, bool want_writes) {
    std::set<std::string> out;
    if (!pl.routine) {
      if (want_writes) out.insert(pl.ir.clear_key);
      return out;
    }
    if (want_writes && !pl.ir.clear_key.empty()) out.insert(pl.ir.clear_key);
    for (const auto& [fe, sn] : pl.b->name) {
      if (!pl.routine->maps.count(fe)) continue;
      const bool w = pl.routine->kind == lib::RoutineKind::Load
                         ? pl.routine->target == fe
                         : (pl.routine->kind == lib::RoutineKind::Compute && pl.b->f->element(fe) &&
                            pl.b->f->element(fe)->is_output);
      if (w == want_writes) out.insert(sn);
    }
    return out;
  };
  std::vector<int> loop_items;
  for (size_t i = 0; i < order.size(); ++i)
    if (order[i].sec == Sec::Loop) loop_items.push_back(static_cast<int>(i));
  std::vector<std::vector<int>> before(loop_items.size());
  for (size_t j = 0; j < loop_items.size(); ++j)
    for (size_t i = 0; i < j; ++i) {
      const Planned &a = order[loop_items[i]], &b = order[loop_items[j]];
      const auto aw = touched(a, true), ar = touched(a, false), bw = touched(b, true),
                 br = touched(b, false);
      auto meet = [](const std::set<std::string>& x, const std::set<std::string>& y) {
        return std::any_of(x.begin(), x.end(), [&](const std::string& e) { return y.count(e) > 0; });
      };
      if (meet(aw, br) || meet(ar, bw) || meet(aw, bw)) before[j].push_back(static_cast<int>(i));
    }
  if (orders) topo_orders(before, cap, orders);
  if (!prm.order.empty()) {
    if (prm.order.size() != loop_items.size())
      throw std::invalid_argument("generate_kernel: routine order has the wrong length");
    std::vector<bool> placed(loop_items.size(), false);
    for (int j : prm.order) {
      if (j < 0 || j >= static_cast<int>(loop_items.size()) || placed[j])
        throw std::invalid_argument("generate_kernel: routine order is not a permutation");
      for (int i : before[j])
        if (!placed[i]) throw std::invalid_argument("generate_kernel: routine order breaks a dependency");
      placed[j] = true;
    }
    std::vector<Planned> loop;
    for (int j : prm.order) loop.push_back(order[loop_items[j]]);
    size_t q = 0;
    for (int idx : loop_items) order[idx] = loop[q++];
  }

  // ---- memory plan: registers iff all accesses share one single-thread map
  struct Access {
    const lib::Routine* r;
    std::string elem;  // function-local element name
  };
  std::map<std::string, std::vector<Access>> acc;
  for (const auto& pl : order) {
    if (!pl.routine) continue;
    for (const auto& [fe, sn] : pl.b->name)
      if (pl.routine->maps.count(fe)) acc[sn].push_back({pl.routine, fe});
  }
  auto same_map = [&](const Access& a, const Access& b) {
    lib::Routine ra = *a.r, rb = *b.r;
    ra.maps["__e"] = a.r->maps.at(a.elem);
    rb.maps["__e"] = b.r->maps.at(b.elem);
    return lib::thread_data_mapping_equal(ra, rb, "__e") == lib::MappingEq::Equal;
  };
  kernel::KernelIR k;
  k.depth = depth;
  k.block_x = depth == 2 ? 32 : 32 * instances;
  k.block_y = depth == 2 ? prm.by : 1;
  k.instances = instances;
  k.iterations = prm.iterations;
  k.iter_dim = depth == 2 ? 'y' : 'x';
  k.scalar_params = params;
  std::string name = "k";
  for (const auto& b : bs) name += "_" + b.f->name;
  k.name = name;
  int offset = 0;
  std::set<std::string> in_shared;
  for (const auto& [key, list] : acc) {
    bool regs = true;
    for (const auto& a : list) {
      const auto& m = a.r->maps.at(a.elem);
      if (m.kind != lib::ThreadMap::Kind::SingleThread || !same_map(a, list.front())) regs = false;
    }
    const lib::ElementDecl* d = nullptr;
    for (const auto& b : bs)
      for (const auto& [fe, sn] : b.name)
        if (sn == key && !d) d = b.f->element(fe);
    const int words = d ? lib::elem_words(d->kind) : 32;
    if (regs) {
      k.reg_arrays.push_back({key, words, 0});
    } else {
      kernel::SharedRegion r;
      r.key = key;
      r.offset = offset;
      const bool tile = d && d->kind == lib::ElemKind::Tile32x32;
      r.stride = tile ? 33 : 32;  // padded when read in both orders
      r.words = tile ? 32 * r.stride : words;
      offset += r.words;
      k.shared_regions.push_back(r);
      in_shared.insert(key);
    }
  }
  k.shared_words = offset;
  if (prm.overlap && k.shared_regions.size() > 1) {
    // Greedy first-fit over live ranges: an element touched
    // in the prologue / epilogue lives for the whole kernel; one used only in
    // the loop body lives from its first to its last routine there.  Largest
    // first (ties by name); an offset is taken when no element with an
    // intersecting live range occupies the same words.
    std::map<std::string, std::pair<int, int>> live;
    const int N = static_cast<int>(order.size());
    for (int i = 0; i < N; ++i) {
      const Planned& pl = order[i];
      std::set<std::string> used = touched(pl, true);
      for (const auto& x : touched(pl, false)) used.insert(x);
      for (const auto& x : used) {
        if (!in_shared.count(x)) continue;
        auto it = live.find(x);
        if (pl.sec != Sec::Loop) live[x] = {0, N};
        else if (it == live.end()) live[x] = {i, i};
        else if (it->second != std::make_pair(0, N)) it->second = {std::min(it->second.first, i),
                                                                    std::max(it->second.second, i)};
      }
    }
    std::vector<kernel::SharedRegion*> regs;
    for (auto& r : k.shared_regions) regs.push_back(&r);
    std::sort(regs.begin(), regs.end(), [](const kernel::SharedRegion* a, const kernel::SharedRegion* b) {
      return a->words != b->words ? a->words > b->words : a->key < b->key;
    });
    std::vector<kernel::SharedRegion*> placed;
    int top = 0;
    for (auto* r : regs) {
      const auto lr = live.count(r->key) ? live[r->key] : std::make_pair(0, N);
      std::vector<int> cand{0};
      for (auto* q : placed) cand.push_back(q->offset + q->words);
      std::sort(cand.begin(), cand.end());
      for (int off : cand) {
        bool ok = true;
        for (auto* q : placed) {
          const auto lq = live.count(q->key) ? live[q->key] : std::make_pair(0, N);
          const bool time = !(lr.second < lq.first || lq.second < lr.first);
          const bool space = off < q->offset + q->words && q->offset < off + r->words;
          if (time && space) ok = false;
        }
        if (ok) {
          r->offset = off;
          break;
        }
      }
      placed.push_back(r);
      top = std::max(top, r->offset + r->words);
    }
    k.shared_words = top;
  }
  auto region_of = [&](const std::string& key) -> const kernel::SharedRegion* {
    for (const auto& r : k.shared_regions)
      if (r.key == key) return &r;
    return nullptr;
  };
  // elements (other than e) whose words overlap e's: writing e clobbers them
  auto aliases = [&](const std::string& e) {
    std::vector<std::string> out;
    const kernel::SharedRegion* re = region_of(e);
    if (!re) return out;
    for (const auto& q : k.shared_regions)
      if (q.key != e && re->offset < q.offset + q.words && q.offset < re->offset + re->words)
        out.push_back(q.key);
    return out;
  };

  // ---- barrier insertion, forward scan in execution order.
  // Condition 1 (read after write): a routine reads an on-chip element written
  // since the last barrier under a different thread-to-data mapping.
  // Condition 2 (write after read): a routine writes a SHARED element that
  // another mapping read since the last barrier -- with serial iterations this
  // is loop-carried (iteration i+1's load of x while iteration i's compute may
  // still read it), so the loop body is scanned a second time starting from
  // the state at the end of an iteration (the SPEC's "barrier when condition
  // 2 would fire across iterations").
  struct State {
    std::map<std::string, Access> written;             // since the last barrier
    std::map<std::string, std::vector<Access>> read;   // since the last barrier
    void clear() {
      written.clear();
      read.clear();
    }
  };
  auto writes_elem = [&](const Planned& pl, const std::string& fe) {
    return pl.routine->kind == lib::RoutineKind::Load
               ? pl.routine->target == fe
               : (pl.routine->kind == lib::RoutineKind::Compute && pl.b->f->element(fe) &&
                  pl.b->f->element(fe)->is_output);
  };
  auto scan = [&](Sec sec, State& st) {
    for (auto& pl : order) {
      if (pl.sec != sec) continue;
      auto clobbers = [&](const std::string& e) {  // condition 2 on overlapping storage
        for (const auto& x : aliases(e))
          if (st.written.count(x) || st.read.count(x)) return true;
        return false;
      };
      if (!pl.routine) {  // pure clear: every thread may write any word
        const std::string& key = pl.ir.clear_key;
        if (prm.barriers && (st.written.count(key) || st.read.count(key) || clobbers(key))) {
          pl.ir.barrier_before = true;
          st.clear();
        }
        st.written[key] = Access{nullptr, ""};
        continue;
      }
      bool need = false;
      if (!pl.ir.clear_key.empty() &&
          (st.written.count(pl.ir.clear_key) || st.read.count(pl.ir.clear_key) ||
           clobbers(pl.ir.clear_key)))
        need = true;
      for (const auto& [fe, sn] : pl.b->name) {
        if (!pl.routine->maps.count(fe)) continue;
        const Access me{pl.routine, fe};
        auto w = st.written.find(sn);
        if (w != st.written.end() && (!w->second.r || !same_map(w->second, me))) need = true;  // cond. 1
        if (writes_elem(pl, fe) && in_shared.count(sn)) {                                     // cond. 2
          auto r = st.read.find(sn);
          if (r != st.read.end())
            for (const auto& a : r->second)
              if (!same_map(a, me)) need = true;
          if (clobbers(sn)) need = true;
        }
      }
      if (need && prm.barriers) {
        pl.ir.barrier_before = true;
        st.clear();
      } else if (pl.ir.barrier_before) {  // placed by an earlier scan of this body
        st.clear();
      }
      if (!pl.ir.clear_key.empty()) {
        if (pl.ir.barrier_after_clear) st.clear();
        else st.written[pl.ir.clear_key] = Access{nullptr, ""};
      }
      for (const auto& [fe, sn] : pl.b->name) {
        if (!pl.routine->maps.count(fe)) continue;
        if (writes_elem(pl, fe)) st.written[sn] = Access{pl.routine, fe};
        else st.read[sn].push_back(Access{pl.routine, fe});
      }
    }
  };
  State st;
  scan(Sec::Pro, st);
  scan(Sec::Loop, st);
  if (prm.iterations > 1) scan(Sec::Loop, st);  // loop-carried hazards (iteration i -> i+1)
  scan(Sec::Epi, st);
  for (auto* sec : {&k.prologue, &k.body, &k.epilogue}) sec->clear();
  for (const auto& pl : order)
    (pl.sec == Sec::Pro ? k.prologue : pl.sec == Sec::Loop ? k.body : k.epilogue).push_back(pl.ir);

  // ---- domain: the grid is derived from the first tile (depth 2) / vector
  for (const auto& b : bs) {
    for (const auto& d : b.f->elements)
      if ((depth == 2 && d.kind == lib::ElemKind::Tile32x32) ||
          (depth == 1 && d.kind == lib::ElemKind::Subvector32)) {
        k.domain = b.name.at(d.name);
        break;
      }
    if (!k.domain.empty()) break;
  }
  return k;
}

}  // namespace

kernel::KernelIR generate_kernel(const std::vector<int>& calls, const script::Script& s,
                                 const script::DataDependencyGraph& g, const lib::Library& L,
                                 const CodegenParams& prm) {
  return generate_impl(calls, s, g, L, prm, nullptr, 0);
}

std::vector<std::vector<int>> enumerate_orderings(const std::vector<int>& calls, const script::Script& s,
                                                  const script::DataDependencyGraph& g,
                                                  const lib::Library& L, int cap) {
  std::vector<std::vector<int>> out;
  generate_impl(calls, s, g, L, CodegenParams{}, &out, std::max(1, cap));
  return out;
}

std::vector<FusionImplementation> prune_implementations(std::vector<FusionImplementation> list) {
  std::vector<FusionImplementation> out;
  for (size_t i = 0; i < list.size(); ++i) {
    bool dominated = false;
    for (size_t j = 0; j < list.size() && !dominated; ++j) {
      if (i == j) continue;
      const auto &a = list[i].params, &b = list[j].params;
      if (a.by == b.by && a.instances == b.instances && a.iterations == b.iterations &&
          list[j].shared_bytes < list[i].shared_bytes)
        dominated = true;
    }
    if (!dominated) out.push_back(std::move(list[i]));
  }
  return out;
}

std::vector<FusionImplementation> enumerate_implementations(const std::vector<int>& calls,
                                                            const script::Script& s,
                                                            const script::DataDependencyGraph& g,
                                                            const lib::Library& L, Sizes sz,
                                                            const SearchSpace& space,
                                                            const vm::DeviceConfig& dev) {
  const kernel::KernelIR base = generate_kernel(calls, s, g, L);
  std::pair<int64_t, int64_t> dom{0, 0};
  if (sz.rows > 0 || sz.cols > 0) dom = domain_shape(base, s, L, sz);
  const auto orders = enumerate_orderings(calls, s, g, L, space.max_orderings);
  std::vector<int> bys = base.depth == 2 ? space.block_rows : std::vector<int>{8};
  std::vector<int> insts = base.depth == 1 ? space.instances : std::vector<int>{1};
  std::vector<FusionImplementation> out;
  std::set<std::string> seen;
  for (const auto& ord : orders)
    for (int by : bys)
      for (int inst : insts)
        for (int it : space.iterations)
          for (int ov = 0; ov < (space.overlap_plans ? 2 : 1); ++ov) {
            if (base.depth == 2 && (by <= 0 || 32 % by)) continue;
            if (sz.rows > 0 || sz.cols > 0) {  // serial iterations must divide the iterated extent
              int64_t extent;
              if (base.depth == 2) {
                extent = std::max<int64_t>(1, dom.first / 32);
              } else {
                const int64_t len = dom.first == 1 ? dom.second : dom.first * dom.second;
                const int64_t elems = std::max<int64_t>(1, len / 32);
                if (it > 1 && elems % inst) continue;
                extent = (elems + inst - 1) / inst;
              }
              if (extent % it) continue;
            }
            CodegenParams prm;
            prm.by = by;
            prm.instances = inst;
            prm.iterations = it;
            prm.order = ord;
            prm.overlap = ov != 0;
            prm.barriers = codegen_barriers();
            kernel::KernelIR k = generate_kernel(calls, s, g, L, prm);
            if (k.threads() > dev.max_threads_per_block) continue;
            if (k.shared_bytes_total() > dev.shared_bytes_per_block) continue;
            if (base.depth == 1 && k.instances != inst) continue;  // capped by max_instances
            std::string text = kernel::emit_pseudo_source(k);
            if (!seen.insert(text).second) continue;  // orders / plans that emit the same kernel
            FusionImplementation fi;
            fi.calls = calls;
            fi.params = prm;
            fi.kir = std::move(k);
            fi.shared_bytes = fi.kir.shared_bytes_total();
            out.push_back(std::move(fi));
          }
  return prune_implementations(std::move(out));
}

}  // namespace mapfuse::plan
