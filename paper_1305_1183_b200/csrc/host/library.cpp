// host/library.cpp -- elementary-function library: manifest reader,
// routine validation, exhaustive access enumeration, mapping equality.
//
// Follows the reference's rules (proj/src/library.cpp: validation
// :703-836, access enumeration :223-245, varies derivation :247-300, mapping
// equality :850-865, manifest grammar :437-646).  Structure here: one generic
// IR visitor shared by every analysis, and a block-structured line reader.
#include "mapfuse/library.hpp"

#include <algorithm>
#include <cctype>
#include <functional>
#include <set>
#include <sstream>

namespace mapfuse::lib {

const char* to_string(HigherOrderKind k) {
  static const char* const n[] = {"map", "reduce", "map_map", "map_reduce"};
  return n[static_cast<int>(k)];
}
const char* to_string(ElemKind k) {
  static const char* const n[] = {"scalar", "subvector32", "tile32x32"};
  return n[static_cast<int>(k)];
}
const char* to_string(RoutineKind k) {
  static const char* const n[] = {"load", "compute", "store"};
  return n[static_cast<int>(k)];
}

int elem_rows(ElemKind k) { return k == ElemKind::Tile32x32 ? 32 : 1; }
int elem_cols(ElemKind k) { return k == ElemKind::Scalar ? 1 : 32; }
int elem_words(ElemKind k) { return elem_rows(k) * elem_cols(k); }

std::string Routine::id() const {
  std::string s = to_string(kind);
  if (!target.empty()) s += "_" + target;
  if (variant != 1) s += "_v" + std::to_string(variant);
  return s;
}

const ElementDecl* ElementaryFunction::element(const std::string& n) const {
  auto it = std::find_if(elements.begin(), elements.end(),
                         [&](const ElementDecl& e) { return e.name == n; });
  return it == elements.end() ? nullptr : &*it;
}

const Routine* ElementaryFunction::routine(RoutineKind k, const std::string& t, int v) const {
  for (const auto& r : routines)
    if (r.kind == k && r.target == t && r.variant == v) return &r;
  return nullptr;
}

std::vector<const Routine*> ElementaryFunction::routines_of(RoutineKind k) const {
  std::vector<const Routine*> v;
  for (const auto& r : routines)
    if (r.kind == k) v.push_back(&r);
  return v;
}

int ElementaryFunction::variant_count(RoutineKind k, const std::string& t) const {
  return static_cast<int>(std::count_if(routines.begin(), routines.end(), [&](const Routine& r) {
    return r.kind == k && r.target == t;
  }));
}

const ElementaryFunction* Library::find(const std::string& name) const {
  auto it = functions.find(name);
  return it == functions.end() ? nullptr : &it->second;
}

bool ElementAccessTable::single_thread() const {
  for (const auto& w : per_word)
    for (const auto& rec : w)
      if (rec.thread != w.front().thread) return false;
  return true;
}

bool ElementAccessTable::has_nonatomic_multiwriter_word() const {
  for (const auto& w : per_word) {
    const bool plain_write = std::any_of(w.begin(), w.end(), [](const AccessRecord& r) {
      return (r.kinds & 2) && !(r.kinds & 4);
    });
    if (!plain_write) continue;
    for (const auto& rec : w)
      if (rec.thread != w.front().thread) return true;
  }
  return false;
}

std::vector<std::string> routine_macros() { return {"BY", "IPB", "ITERS"}; }

// ===========================================================================
// Generic visitor: every memory reference of a body, with its space, element
// slot, coordinates and access kind.
namespace {

struct MemRef {
  bool global = false;
  int element = -1;
  int32_t i0 = -1, i1 = -1;
  uint8_t kinds = 0;  // 1 read, 2 write, 4 atomic
};

void visit_float_refs(const ir::Program& p, int32_t fe, const std::function<void(const MemRef&)>& f) {
  if (fe < 0) return;
  const ir::FloatNode& n = p.floats[fe];
  if (n.op == ir::FloatOp::Load) {
    f(MemRef{n.global, n.slot, n.idx0, n.idx1, 1});
    return;
  }
  visit_float_refs(p, n.a, f);
  visit_float_refs(p, n.b, f);
  visit_float_refs(p, n.c, f);
}

// Static walk (no control-flow evaluation).
void visit_refs(const ir::Program& p, const std::vector<ir::Stmt>& ss,
                const std::function<void(const MemRef&)>& f) {
  for (const auto& s : ss) {
    visit_float_refs(p, s.fexpr, f);
    if (s.kind == ir::StmtKind::Store)
      f(MemRef{s.global, s.element, s.idx0, s.idx1, 2});
    else if (s.kind == ir::StmtKind::AtomicAdd)
      f(MemRef{s.global, s.element, s.idx0, s.idx1, 2 | 4});
    visit_refs(p, s.body, f);
  }
}

bool compare(ir::CmpOp op, int64_t a, int64_t b) {
  switch (op) {
    case ir::CmpOp::Eq: return a == b;
    case ir::CmpOp::Ne: return a != b;
    case ir::CmpOp::Lt: return a < b;
    case ir::CmpOp::Le: return a <= b;
    case ir::CmpOp::Gt: return a > b;
    case ir::CmpOp::Ge: return a >= b;
  }
  return false;
}

// Dynamic walk for one thread: loops and guards evaluated.
void execute_refs(const ir::Program& p, const std::vector<ir::Stmt>& ss, std::vector<int64_t>& env,
                  const std::function<void(const MemRef&)>& f) {
  for (const auto& s : ss) {
    switch (s.kind) {
      case ir::StmtKind::For: {
        const int64_t b = p.eval_int(s.begin, env), e = p.eval_int(s.end, env);
        const int64_t st = p.eval_int(s.step, env);
        if (st <= 0) throw std::runtime_error("loop step must be positive");
        for (int64_t v = b; v < e; v += st) {
          env[s.loop_sym] = v;
          execute_refs(p, s.body, env, f);
        }
        break;
      }
      case ir::StmtKind::If:
        if (compare(s.cmp, p.eval_int(s.cmp_lhs, env), p.eval_int(s.cmp_rhs, env)))
          execute_refs(p, s.body, env, f);
        break;
      case ir::StmtKind::DeclTemp:
      case ir::StmtKind::AssignTemp: visit_float_refs(p, s.fexpr, f); break;
      case ir::StmtKind::Store:
        visit_float_refs(p, s.fexpr, f);
        f(MemRef{s.global, s.element, s.idx0, s.idx1, 2});
        break;
      case ir::StmtKind::AtomicAdd:
        visit_float_refs(p, s.fexpr, f);
        f(MemRef{s.global, s.element, s.idx0, s.idx1, 2 | 4});
        break;
      default: break;
    }
  }
}

}  // namespace

std::map<std::string, ElementAccessTable> enumerate_accesses(
    const ElementaryFunction& f, const Routine& r, int px, int py,
    const std::map<std::string, int64_t>& macros) {
  const ir::Program body = ir::substitute_macros(r.body, macros);
  std::map<std::string, ElementAccessTable> out;
  std::vector<int64_t> env(static_cast<size_t>(body.symbol_count()), 0);
  env[ir::kSymNx] = env[ir::kSymNy] = int64_t(1) << 20;
  int thread = 0;
  auto record = [&](const MemRef& m) {
    if (m.global) return;
    const std::string& name = body.elements[m.element].name;
    const ElementDecl* d = f.element(name);
    if (!d) return;
    ElementAccessTable& t = out[name];
    if (t.per_word.empty()) {
      t.words = elem_words(d->kind);
      t.per_word.resize(static_cast<size_t>(t.words));
    }
    const int64_t a = body.eval_int(m.i0, env);
    const int64_t w = m.i1 >= 0 ? a * elem_cols(d->kind) + body.eval_int(m.i1, env) : a;
    if (w < 0 || w >= t.words)
      throw std::runtime_error("on-chip access outside element " + name + ": word " +
                               std::to_string(w));
    auto& recs = t.per_word[static_cast<size_t>(w)];
    for (auto& rec : recs)
      if (rec.thread == thread) {
        rec.kinds |= m.kinds;
        return;
      }
    recs.push_back({thread, m.kinds});
  };
  for (int y = 0; y < py; ++y)
    for (int x = 0; x < px; ++x) {
      env[ir::kSymTx] = x;
      env[ir::kSymTy] = y;
      env[ir::kSymFlat] = thread = y * px + x;
      execute_refs(body, body.stmts, env, record);
    }
  for (auto& [n, t] : out)
    for (auto& w : t.per_word)
      std::sort(w.begin(), w.end(),
                [](const AccessRecord& a, const AccessRecord& b) { return a.thread < b.thread; });
  return out;
}

std::map<std::string, Varies> derive_varies(const Routine& r) {
  std::map<std::string, Varies> out;
  const ir::Program& p = r.body;
  auto coord = [&](Varies& v, int32_t idx) {
    if (idx < 0) return;
    auto lf = p.linear(idx);
    if (!lf) {
      v.x = v.y = true;
      return;
    }
    v.x = v.x || lf->uses(ir::kSymEx) || lf->uses(ir::kSymBx) || lf->uses(ir::kSymInst);
    v.y = v.y || lf->uses(ir::kSymEy) || lf->uses(ir::kSymBy);
  };
  visit_refs(p, p.stmts, [&](const MemRef& m) {
    if (!m.global) return;
    Varies& v = out[p.elements[m.element].name];
    coord(v, m.i0);
    coord(v, m.i1);
  });
  return out;
}

// ===========================================================================
// Validation
std::vector<Diagnostic> check_routine(const Routine& r, const ElementaryFunction& f) {
  std::vector<Diagnostic> d;
  const std::string where = f.name + "." + r.id();
  const ir::Program& p = r.body;
  bool g_read = false, g_write = false, o_read = false, o_write = false;
  std::vector<std::string> touched;
  std::vector<std::pair<int, int32_t>> onchip_coords;
  visit_refs(p, p.stmts, [&](const MemRef& m) {
    const bool write = (m.kinds & 2) != 0;
    if (m.global) (write ? g_write : g_read) = true;
    else (write ? o_write : o_read) = true;
    const std::string& n = p.elements[m.element].name;
    if (std::find(touched.begin(), touched.end(), n) == touched.end()) touched.push_back(n);
    if (!m.global) {
      onchip_coords.emplace_back(m.element, m.i0);
      if (m.i1 >= 0) onchip_coords.emplace_back(m.element, m.i1);
    }
  });
  auto add = [&](const char* rule, const std::string& msg) { d.push_back({rule, where, msg}); };
  switch (r.kind) {
    case RoutineKind::Load:
      if (g_write) add("kind-violation", "load routine writes global memory");
      if (o_read) add("kind-violation", "load routine reads on-chip memory");
      break;
    case RoutineKind::Compute:
      if (g_read || g_write) add("kind-violation", "compute routine touches global memory");
      break;
    case RoutineKind::Store:
      if (g_read) add("kind-violation", "store routine reads global memory");
      if (o_write) add("kind-violation", "store routine writes on-chip memory");
      break;
  }
  for (const auto& n : touched)
    if (!f.element(n)) add("unknown-element", "element '" + n + "' is not in the signature");
  if (!r.target.empty() && !f.element(r.target))
    add("unknown-element", "target '" + r.target + "' is not in the signature");
  for (const auto& [e, idx] : onchip_coords) {
    const std::string& n = p.elements[e].name;
    auto m = r.maps.find(n);
    const bool datadep = m != r.maps.end() && m->second.kind == ThreadMap::Kind::DataDep;
    if (!datadep && !p.linear(idx))
      add("non-affine", "on-chip index of '" + n + "' is not affine (flag it datadep)");
  }

  if (d.empty()) {
    const std::vector<int> bys = f.par_y_is_block ? std::vector<int>{2, 8} : std::vector<int>{1};
    for (int by : bys) {
      std::map<std::string, ElementAccessTable> tables;
      try {
        tables = enumerate_accesses(f, r, f.par_x, by, {{"BY", by}, {"IPB", 1}, {"ITERS", 1}});
      } catch (const std::exception& e) {
        add("body-error", e.what());
        break;
      }
      for (const auto& [name, t] : tables) {
        auto mi = r.maps.find(name);
        if (mi == r.maps.end()) {
          add("missing-mapping", "no declared mapping for '" + name + "'");
          continue;
        }
        const ThreadMap& m = mi->second;
        if (m.kind == ThreadMap::Kind::DataDep) continue;
        if (m.kind == ThreadMap::Kind::Atomic || m.kind == ThreadMap::Kind::Broadcast) {
          const bool atomic = m.kind == ThreadMap::Kind::Atomic;
          bool bad = false;
          for (const auto& w : t.per_word)
            for (const auto& rec : w)
              if (atomic ? ((rec.kinds & 2) && !(rec.kinds & 4)) : (rec.kinds & 2) != 0) bad = true;
          if (bad)
            add("mapping-mismatch", "'" + name + "' declared " + (atomic ? "atomic" : "broadcast") +
                                        " but written " + (atomic ? "non-atomically" : ""));
          continue;
        }
        const bool tile = f.element(name)->kind == ElemKind::Tile32x32;
        auto eval = [&](const MapCoord& c, int64_t row, int64_t col) {
          int64_t v = c.cr * row + c.cc * col + c.c0;
          int64_t mod = c.mod_macro.empty() ? c.mod_const : (c.mod_macro == "BY" ? by : 0);
          return mod > 0 ? v % mod : v;
        };
        for (int w = 0; w < t.words; ++w) {
          const auto& recs = t.per_word[static_cast<size_t>(w)];
          if (recs.empty()) continue;
          if (recs.size() > 1) {
            add("mapping-mismatch", "'" + name + "' word " + std::to_string(w) +
                                        " is touched by several threads (declared single-thread)");
            break;
          }
          const int64_t row = tile ? w / 32 : w, col = tile ? w % 32 : 0;
          const int64_t expect = eval(m.ty, row, col) * f.par_x + eval(m.tx, row, col);
          if (recs[0].thread != expect) {
            add("mapping-mismatch", "'" + name + "' word " + std::to_string(w) +
                                        " accessed by thread " + std::to_string(recs[0].thread) +
                                        ", mapping declares " + std::to_string(expect));
            break;
          }
        }
      }
    }
  }

  for (const auto& [name, v] : derive_varies(r)) {
    const ElementDecl* e = f.element(name);
    if (e && ((v.x && !e->varies.x) || (v.y && !e->varies.y)))
      add("varies-mismatch", "address of '" + name + "' depends on more grid dimensions than declared");
  }
  return d;
}

namespace {
MapCoord canonical(MapCoord c) {
  if (c.mod_const > 0) {
    auto md = [&](int64_t v) { return ((v % c.mod_const) + c.mod_const) % c.mod_const; };
    c.cr = md(c.cr);
    c.cc = md(c.cc);
    c.c0 = md(c.c0);
  }
  return c;
}
}  // namespace

MappingEq thread_data_mapping_equal(const Routine& a, const Routine& b, const std::string& element) {
  auto ia = a.maps.find(element), ib = b.maps.find(element);
  if (ia == a.maps.end() || ib == b.maps.end()) return MappingEq::Unknown;
  const ThreadMap &x = ia->second, &y = ib->second;
  if (x.kind == ThreadMap::Kind::DataDep || y.kind == ThreadMap::Kind::DataDep)
    return MappingEq::Unknown;
  if (x.kind != y.kind) return MappingEq::Unequal;
  if (x.kind != ThreadMap::Kind::SingleThread) return MappingEq::Equal;
  return canonical(x.tx) == canonical(y.tx) && canonical(x.ty) == canonical(y.ty)
             ? MappingEq::Equal
             : MappingEq::Unequal;
}

std::string print_manifest(const Library& lib) { return lib.source; }

// ===========================================================================
// Manifest reader
namespace {

struct Line {
  int no = 0;
  std::string raw, text;  // text: comment-stripped, trimmed
};

std::string trim(const std::string& s) {
  const size_t b = s.find_first_not_of(" \t\r");
  if (b == std::string::npos) return "";
  return s.substr(b, s.find_last_not_of(" \t\r") - b + 1);
}

std::vector<std::string> words(const std::string& s) {
  std::vector<std::string> w;
  std::istringstream in(s);
  for (std::string t; in >> t;) w.push_back(t);
  return w;
}

class Reader {
 public:
  explicit Reader(const std::string& text) {
    std::istringstream in(text);
    std::string raw;
    int no = 0;
    while (std::getline(in, raw)) {
      ++no;
      std::string t = raw;
      if (auto c = t.find("//"); c != std::string::npos) t.erase(c);
      lines_.push_back({no, raw, trim(t)});
    }
  }

  Library run(const std::string& source) {
    Library L;
    L.source = source;
    while (skip_blank()) {
      const Line& l = lines_[i_];
      auto w = words(l.text);
      if (w.size() < 2 || w[0] != "function") fail(l, "expected 'function <name> {'");
      ++i_;
      ElementaryFunction f = function(w[1], l);
      if (L.functions.count(f.name)) fail(l, "duplicate function '" + f.name + "'");
      validate(f);
      L.functions.emplace(f.name, std::move(f));
    }
    return L;
  }

 private:
  std::vector<Line> lines_;
  size_t i_ = 0;

  [[noreturn]] static void fail(const Line& l, const std::string& msg) {
    throw ir::ParseError("manifest: " + msg, l.no, 1);
  }
  bool skip_blank() {
    while (i_ < lines_.size() && lines_[i_].text.empty()) ++i_;
    return i_ < lines_.size();
  }
  static int brace_delta(const std::string& t) {
    return static_cast<int>(std::count(t.begin(), t.end(), '{')) -
           static_cast<int>(std::count(t.begin(), t.end(), '}'));
  }

  // Raw text of a braced block whose opening line was just consumed.
  std::string block_text(int* first_line, const Line& opener) {
    std::string out;
    int depth = 1;
    *first_line = i_ < lines_.size() ? lines_[i_].no : opener.no;
    while (i_ < lines_.size()) {
      const Line& l = lines_[i_++];
      depth += brace_delta(l.text);
      if (depth <= 0) return out;
      out += l.raw + "\n";
    }
    fail(opener, "unterminated block");
  }

  static ElemKind elem_kind(const std::string& s, const Line& l) {
    if (s == "scalar") return ElemKind::Scalar;
    if (s == "subvector32") return ElemKind::Subvector32;
    if (s == "tile32x32") return ElemKind::Tile32x32;
    fail(l, "unknown element kind '" + s + "'");
  }

  static MapCoord coord(const std::string& text, const Line& l) {
    MapCoord c;
    std::string expr = text;
    if (auto pct = text.find('%'); pct != std::string::npos) {
      expr = text.substr(0, pct);
      const std::string m = trim(text.substr(pct + 1));
      if (!m.empty() && std::isdigit(static_cast<unsigned char>(m[0]))) c.mod_const = std::stoll(m);
      else c.mod_macro = m;
    }
    // terms: [+|-] [k[*]] (r|c|w) | [+|-] k
    size_t p = 0;
    int sign = 1;
    while (p < expr.size()) {
      const char ch = expr[p];
      if (std::isspace(static_cast<unsigned char>(ch)) || ch == '*') {
        ++p;
        continue;
      }
      if (ch == '+' || ch == '-') {
        sign = ch == '-' ? -1 : 1;
        ++p;
        continue;
      }
      int64_t k = 1;
      bool has_k = false;
      if (std::isdigit(static_cast<unsigned char>(ch))) {
        k = 0;
        while (p < expr.size() && std::isdigit(static_cast<unsigned char>(expr[p])))
          k = k * 10 + (expr[p++] - '0');
        has_k = true;
        while (p < expr.size() && (std::isspace(static_cast<unsigned char>(expr[p])) || expr[p] == '*'))
          ++p;
      }
      if (p < expr.size() && std::isalpha(static_cast<unsigned char>(expr[p]))) {
        const char v = expr[p++];
        if (v == 'r' || v == 'w') c.cr += sign * k;
        else if (v == 'c') c.cc += sign * k;
        else fail(l, std::string("unknown mapping coordinate '") + v + "'");
      } else if (has_k) {
        c.c0 += sign * k;
      } else {
        fail(l, "cannot parse mapping expression '" + text + "'");
      }
      sign = 1;
    }
    return c;
  }

  static ThreadMap thread_map(const std::string& rhs, const Line& l) {
    ThreadMap m;
    const std::string r = trim(rhs);
    if (r == "broadcast") m.kind = ThreadMap::Kind::Broadcast;
    else if (r == "atomic") m.kind = ThreadMap::Kind::Atomic;
    else if (r == "datadep") m.kind = ThreadMap::Kind::DataDep;
    if (m.kind != ThreadMap::Kind::SingleThread) return m;
    std::stringstream ss(r);
    for (std::string part; std::getline(ss, part, ',');) {
      part = trim(part);
      if (part.empty()) continue;
      const auto eq = part.find('=');
      if (eq == std::string::npos) fail(l, "expected 'tx = ...' in mapping");
      const std::string lhs = trim(part.substr(0, eq));
      MapCoord c = coord(trim(part.substr(eq + 1)), l);
      if (lhs == "tx") m.tx = c;
      else if (lhs == "ty") m.ty = c;
      else fail(l, "mapping assigns unknown coordinate '" + lhs + "'");
    }
    return m;
  }

  Routine routine(const std::vector<std::string>& head, const Line& hl, const ElementaryFunction& f) {
    Routine r;
    if (head.size() < 2) fail(hl, "routine header too short");
    if (head[1] == "load") r.kind = RoutineKind::Load;
    else if (head[1] == "compute") r.kind = RoutineKind::Compute;
    else if (head[1] == "store") r.kind = RoutineKind::Store;
    else fail(hl, "unknown routine kind '" + head[1] + "'");
    size_t at = 2;
    if (r.kind != RoutineKind::Compute) {
      if (head.size() <= at || head[at] == "{") fail(hl, "load/store routine needs a target element");
      r.target = head[at++];
    }
    for (; at < head.size(); ++at)
      if (head[at] == "variant" && at + 1 < head.size()) r.variant = std::stoi(head[++at]);
    std::string body;
    int body_line = hl.no;
    while (true) {
      if (!skip_blank()) fail(hl, "unterminated routine block");
      const Line& l = lines_[i_++];
      if (l.text == "}") break;
      auto w = words(l.text);
      if (w[0] == "map") {
        const auto colon = l.text.find(':');
        if (colon == std::string::npos) fail(l, "map line needs ':'");
        r.maps[trim(l.text.substr(3, colon - 3))] = thread_map(l.text.substr(colon + 1), l);
      } else if (w[0] == "body") {
        body = block_text(&body_line, l);
      } else {
        fail(l, "unexpected line in routine block: '" + l.text + "'");
      }
    }
    ir::ParseContext ctx;
    ctx.params = f.scalar_params;
    ctx.macros = routine_macros();
    r.body = ir::parse_program(body, ctx, body_line);
    std::function<bool(const std::vector<ir::Stmt>&)> atomic = [&](const std::vector<ir::Stmt>& ss) {
      return std::any_of(ss.begin(), ss.end(), [&](const ir::Stmt& s) {
        return s.kind == ir::StmtKind::AtomicAdd || atomic(s.body);
      });
    };
    r.writes_atomic = atomic(r.body.stmts);
    return r;
  }

  ElementaryFunction function(const std::string& name, const Line& opener) {
    ElementaryFunction f;
    f.name = name;
    while (true) {
      if (!skip_blank()) fail(opener, "unterminated function block");
      const Line& l = lines_[i_++];
      if (l.text == "}") break;
      const auto w = words(l.text);
      const std::string& key = w[0];
      auto arg = [&](size_t k) -> const std::string& {
        if (k >= w.size()) fail(l, "'" + key + "' needs more fields");
        return w[k];
      };
      if (key == "routine") {
        f.routines.push_back(routine(w, l, f));
      } else if (key == "kind") {
        const std::string& v = arg(1);
        if (v == "map") f.kind = HigherOrderKind::Map;
        else if (v == "reduce") f.kind = HigherOrderKind::Reduce;
        else if (v == "map_map") f.kind = HigherOrderKind::MapMap;
        else if (v == "map_reduce") f.kind = HigherOrderKind::MapReduce;
        else fail(l, "unknown higher-order kind '" + v + "'");
      } else if (key == "depth") {
        f.depth = std::stoi(arg(1));
      } else if (key == "parallelism") {
        f.par_x = std::stoi(arg(1));
        f.par_y_is_block = arg(2) == "BY";
        if (!f.par_y_is_block && std::stoi(arg(2)) != 1)
          fail(l, "instance parallelism y must be 1 or BY");
      } else if (key == "max_instances") {
        f.max_instances = std::stoi(arg(1));
      } else if (key == "scalar") {
        f.scalar_params.push_back(arg(1));
        f.args.push_back({true, arg(1)});
      } else if (key == "arg" || key == "out") {
        ElementDecl d;
        d.name = arg(1);
        d.kind = elem_kind(arg(2), l);
        d.is_output = key == "out";
        for (size_t k = 3; k < w.size(); ++k) {
          if (w[k] == "accumulable") {
            d.accumulable = true;
          } else if (w[k] == "varies") {
            const std::string& v = arg(++k);
            d.varies = {v.find('x') != std::string::npos, v.find('y') != std::string::npos};
            if (v == "none") d.varies = {};
          } else {
            fail(l, "unknown element attribute '" + w[k] + "'");
          }
        }
        f.elements.push_back(d);
        if (d.is_output) f.results.push_back(d.name);
        else f.args.push_back({false, d.name});
      } else {
        fail(l, "unknown function key '" + key + "' in " + name);
      }
    }
    return f;
  }

  static void validate(const ElementaryFunction& f) {
    std::vector<Diagnostic> d;
    for (const auto& r : f.routines) {
      auto more = check_routine(r, f);
      d.insert(d.end(), more.begin(), more.end());
    }
    for (const auto& e : f.elements) {
      const RoutineKind need = e.is_output ? RoutineKind::Store : RoutineKind::Load;
      if (!e.is_output && e.kind == ElemKind::Scalar) continue;
      if (f.variant_count(need, e.name) == 0)
        d.push_back({"missing-routine", f.name,
                     std::string(e.is_output ? "output " : "input ") + e.name + " has no " +
                         to_string(need) + " routine"});
    }
    if (f.routines_of(RoutineKind::Compute).empty())
      d.push_back({"missing-routine", f.name, "no compute routine"});
    if (f.is_reduction() &&
        std::count_if(f.elements.begin(), f.elements.end(),
                      [](const ElementDecl& e) { return e.is_output && e.accumulable; }) != 1)
      d.push_back({"invalid-metadata", f.name, "a reduction needs exactly one accumulable output"});
    if (f.depth == 2 && std::none_of(f.elements.begin(), f.elements.end(), [](const ElementDecl& e) {
          return e.kind == ElemKind::Tile32x32;
        }))
      d.push_back({"invalid-metadata", f.name, "depth-2 function declares no tile element"});
    if (!d.empty()) {
      std::string msg = "library validation failed for " + f.name + ":";
      for (const auto& x : d) msg += "\n  [" + x.rule + "] " + x.where + ": " + x.message;
      throw std::runtime_error(msg);
    }
  }
};

}  // namespace

Library load_library(const std::string& manifest_text) {
  return Reader(manifest_text).run(manifest_text);
}

}  // namespace mapfuse::lib
