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

kernel::KernelIR generate_kernel(const std::vector<int>& calls_in, const script::Script& s,
                                 const script::DataDependencyGraph& g, const lib::Library& L,
                                 const CodegenParams& prm) {
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
      if (!pl.routine) {  // pure clear: every thread may write any word
        const std::string& key = pl.ir.clear_key;
        if (prm.barriers && (st.written.count(key) || st.read.count(key))) {
          pl.ir.barrier_before = true;
          st.clear();
        }
        st.written[key] = Access{nullptr, ""};
        continue;
      }
      bool need = false;
      if (!pl.ir.clear_key.empty() &&
          (st.written.count(pl.ir.clear_key) || st.read.count(pl.ir.clear_key)))
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

}  // namespace mapfuse::plan
