// host/ir.cpp -- routine IR: lexer, recursive-descent parser over a token
// stream, printer, integer evaluation, affine extraction, macro binding.
//
// Behaviour follows the reference's routine IR (proj/src/ir.cpp: grammar and
// desugaring rules at :208-591, printer at :593-731, macro binding at
// :733-749); the structure here is a two-phase tokenizer + parser.
#include "mapfuse/ir.hpp"

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <functional>

namespace mapfuse::ir {

namespace {
const char* const kBuiltinNames[kNumBuiltinSyms] = {"tx", "ty",   "ex",   "ey", "bx",
                                                     "by", "inst", "flat", "nx", "ny"};
}

const char* builtin_sym_name(int slot) {
  return (slot >= 0 && slot < kNumBuiltinSyms) ? kBuiltinNames[slot] : "?";
}

int64_t LinearForm::coeff(int slot) const {
  auto it = std::lower_bound(terms.begin(), terms.end(), std::make_pair(slot, INT64_MIN));
  return (it != terms.end() && it->first == slot) ? it->second : 0;
}

int Program::find_extra(const std::string& name, ExtraSymKind kind) const {
  for (size_t i = 0; i < extra_syms.size(); ++i)
    if (extra_syms[i].kind == kind && extra_syms[i].name == name)
      return kNumBuiltinSyms + static_cast<int>(i);
  return -1;
}

int Program::find_element(const std::string& name) const {
  for (size_t i = 0; i < elements.size(); ++i)
    if (elements[i].name == name) return static_cast<int>(i);
  return -1;
}

int64_t Program::eval_int(int32_t node, const std::vector<int64_t>& env) const {
  const IntNode& n = ints.at(node);
  if (n.op == IntOp::Const) return n.value;
  if (n.op == IntOp::Sym) return env.at(static_cast<size_t>(n.value));
  const int64_t l = eval_int(n.lhs, env), r = eval_int(n.rhs, env);
  switch (n.op) {
    case IntOp::Add: return l + r;
    case IntOp::Sub: return l - r;
    case IntOp::Mul: return l * r;
    case IntOp::Div:
      if (r == 0) throw std::runtime_error("index expression divides by zero");
      return l / r;
    case IntOp::Mod:
      if (r == 0) throw std::runtime_error("index expression takes modulo zero");
      return l % r;
    case IntOp::Min: return std::min(l, r);
    default: return 0;
  }
}

namespace {

LinearForm lin_scale(const LinearForm& f, int64_t k) {
  LinearForm o;
  o.c0 = f.c0 * k;
  if (k != 0)
    for (const auto& [s, c] : f.terms) o.terms.emplace_back(s, c * k);
  return o;
}

LinearForm lin_add(const LinearForm& a, const LinearForm& b) {
  LinearForm o;
  o.c0 = a.c0 + b.c0;
  size_t i = 0, j = 0;
  while (i < a.terms.size() || j < b.terms.size()) {
    if (j == b.terms.size() || (i < a.terms.size() && a.terms[i].first < b.terms[j].first)) {
      o.terms.push_back(a.terms[i++]);
    } else if (i == a.terms.size() || b.terms[j].first < a.terms[i].first) {
      o.terms.push_back(b.terms[j++]);
    } else {
      const int64_t c = a.terms[i].second + b.terms[j].second;
      if (c != 0) o.terms.emplace_back(a.terms[i].first, c);
      ++i;
      ++j;
    }
  }
  return o;
}

}  // namespace

std::optional<LinearForm> Program::linear(int32_t node) const {
  const IntNode& n = ints.at(node);
  switch (n.op) {
    case IntOp::Const: return LinearForm{n.value, {}};
    case IntOp::Sym: return LinearForm{0, {{static_cast<int>(n.value), 1}}};
    case IntOp::Add:
    case IntOp::Sub:
    case IntOp::Mul: {
      auto l = linear(n.lhs);
      if (!l) return std::nullopt;
      auto r = linear(n.rhs);
      if (!r) return std::nullopt;
      if (n.op == IntOp::Add) return lin_add(*l, *r);
      if (n.op == IntOp::Sub) return lin_add(*l, lin_scale(*r, -1));
      if (l->terms.empty()) return lin_scale(*r, l->c0);
      if (r->terms.empty()) return lin_scale(*l, r->c0);
      return std::nullopt;  // product of two symbolic factors
    }
    default: return std::nullopt;  // div / mod / min are not affine
  }
}

int32_t add_const(Program& p, int64_t v) {
  p.ints.push_back(IntNode{IntOp::Const, v, -1, -1});
  return static_cast<int32_t>(p.ints.size()) - 1;
}
int32_t add_sym(Program& p, int slot) {
  p.ints.push_back(IntNode{IntOp::Sym, slot, -1, -1});
  return static_cast<int32_t>(p.ints.size()) - 1;
}
int32_t add_bin(Program& p, IntOp op, int32_t lhs, int32_t rhs) {
  p.ints.push_back(IntNode{op, 0, lhs, rhs});
  return static_cast<int32_t>(p.ints.size()) - 1;
}
int32_t add_float_const(Program& p, float v) {
  FloatNode f;
  f.op = FloatOp::Const;
  f.value = v;
  p.floats.push_back(f);
  return static_cast<int32_t>(p.floats.size()) - 1;
}

// ===========================================================================
// Lexer
namespace {

enum class TK { Ident, Number, Punct, End };

struct Token {
  TK kind = TK::End;
  std::string text;
  int line = 0, col = 0;
  bool glued_prev = false;  // no whitespace before this token
};

std::vector<Token> lex(const std::string& s, int first_line) {
  std::vector<Token> out;
  int line = first_line;
  size_t line_start = 0, i = 0;
  bool space = true;
  auto push = [&](TK k, size_t b, size_t e) {
    Token t;
    t.kind = k;
    t.text = s.substr(b, e - b);
    t.line = line;
    t.col = static_cast<int>(b - line_start) + 1;
    t.glued_prev = !space;
    out.push_back(std::move(t));
    space = false;
  };
  while (i < s.size()) {
    const char c = s[i];
    if (c == '\n') {
      ++line;
      line_start = ++i;
      space = true;
      continue;
    }
    if (c == ' ' || c == '\t' || c == '\r') {
      ++i;
      space = true;
      continue;
    }
    if (c == '/' && i + 1 < s.size() && s[i + 1] == '/') {
      while (i < s.size() && s[i] != '\n') ++i;
      continue;
    }
    if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      size_t j = i;
      while (j < s.size() && (std::isalnum(static_cast<unsigned char>(s[j])) || s[j] == '_')) ++j;
      push(TK::Ident, i, j);
      i = j;
      continue;
    }
    if (std::isdigit(static_cast<unsigned char>(c))) {
      size_t j = i;
      while (j < s.size() && std::isdigit(static_cast<unsigned char>(s[j]))) ++j;
      if (j < s.size() && s[j] == '.' && !(j + 1 < s.size() && s[j + 1] == '.')) {
        ++j;
        while (j < s.size() && std::isdigit(static_cast<unsigned char>(s[j]))) ++j;
      }
      if (j < s.size() && (s[j] == 'e' || s[j] == 'E')) {
        size_t k = j + 1;
        if (k < s.size() && (s[k] == '+' || s[k] == '-')) ++k;
        if (k < s.size() && std::isdigit(static_cast<unsigned char>(s[k]))) {
          while (k < s.size() && std::isdigit(static_cast<unsigned char>(s[k]))) ++k;
          j = k;
        }
      }
      if (j < s.size() && s[j] == 'f') ++j;
      push(TK::Number, i, j);
      i = j;
      continue;
    }
    static const char* const two[] = {"..", "+=", "==", "!=", "<=", ">="};
    bool matched = false;
    for (const char* t : two)
      if (s.compare(i, 2, t) == 0) {
        push(TK::Punct, i, i + 2);
        i += 2;
        matched = true;
        break;
      }
    if (matched) continue;
    if (std::strchr("+-*/%()[]{},=<>", c)) {
      push(TK::Punct, i, i + 1);
      ++i;
      continue;
    }
    Token t;
    t.kind = TK::Punct;
    t.text = std::string(1, c);
    t.line = line;
    t.col = static_cast<int>(i - line_start) + 1;
    throw ParseError("unexpected character '" + t.text + "'", t.line, t.col);
  }
  Token end;
  end.kind = TK::End;
  end.line = line;
  end.col = static_cast<int>(i - line_start) + 1;
  out.push_back(end);
  return out;
}

bool is_integer_literal(const std::string& t) {
  return !t.empty() && std::all_of(t.begin(), t.end(),
                                   [](char c) { return std::isdigit(static_cast<unsigned char>(c)); });
}

// ===========================================================================
// Parser
class Parser {
 public:
  Parser(const std::string& text, const ParseContext& ctx, int first_line)
      : toks_(lex(text, first_line)), ctx_(ctx) {
    for (const auto& m : ctx.macros) prog_.extra_syms.push_back({m, ExtraSymKind::Macro});
    prog_.params = ctx.params;
  }

  Program run() {
    while (peek().kind != TK::End) {
      if (is("}")) fail_at(peek(), "unmatched '}'");
      prog_.stmts.push_back(statement());
    }
    return std::move(prog_);
  }

 private:
  std::vector<Token> toks_;
  size_t pos_ = 0;
  const ParseContext& ctx_;
  Program prog_;

  const Token& peek(size_t k = 0) const {
    return toks_[std::min(pos_ + k, toks_.size() - 1)];
  }
  bool is(const char* p, size_t k = 0) const {
    const Token& t = peek(k);
    return t.kind == TK::Punct && t.text == p;
  }
  bool is_word(const char* w, size_t k = 0) const {
    const Token& t = peek(k);
    return t.kind == TK::Ident && t.text == w;
  }
  const Token& next() {
    const Token& t = peek();
    if (pos_ < toks_.size() - 1) ++pos_;
    return t;
  }
  [[noreturn]] void fail_at(const Token& t, const std::string& msg) const {
    throw ParseError(msg, t.line, t.col);
  }
  void expect(const char* p, const char* ctx) {
    if (!is(p)) fail_at(peek(), std::string("expected '") + p + "' " + ctx);
    next();
  }
  std::string ident(const char* what) {
    if (peek().kind != TK::Ident) fail_at(peek(), std::string("expected ") + what);
    return next().text;
  }

  int symbol(const std::string& name) const {
    for (int i = 0; i < kNumBuiltinSyms; ++i)
      if (name == kBuiltinNames[i]) return i;
    int s = prog_.find_extra(name, ExtraSymKind::Macro);
    if (s >= 0) return s;
    return prog_.find_extra(name, ExtraSymKind::LoopVar);
  }

  int element(const std::string& name) {
    int e = prog_.find_element(name);
    if (e >= 0) return e;
    prog_.elements.push_back({name, 1});
    return static_cast<int>(prog_.elements.size()) - 1;
  }

  static int index_of(const std::vector<std::string>& v, const std::string& n) {
    for (size_t i = 0; i < v.size(); ++i)
      if (v[i] == n) return static_cast<int>(i);
    return -1;
  }

  // ---- integer expressions
  int32_t iexpr() {
    int32_t e = iterm();
    while (is("+") || is("-")) {
      const IntOp op = next().text == "+" ? IntOp::Add : IntOp::Sub;
      e = add_bin(prog_, op, e, iterm());
    }
    return e;
  }
  int32_t iterm() {
    int32_t e = iunary();
    while (is("*") || is("/") || is("%")) {
      const std::string o = next().text;
      const IntOp op = o == "*" ? IntOp::Mul : (o == "/" ? IntOp::Div : IntOp::Mod);
      e = add_bin(prog_, op, e, iunary());
    }
    return e;
  }
  int32_t iunary() {
    if (is("-")) {
      next();
      const int32_t zero = add_const(prog_, 0);
      return add_bin(prog_, IntOp::Sub, zero, iunary());
    }
    return iprimary();
  }
  int32_t iprimary() {
    const Token& t = peek();
    if (is("(")) {
      next();
      int32_t e = iexpr();
      expect(")", "to close parenthesis");
      return e;
    }
    if (t.kind == TK::Number) {
      if (!is_integer_literal(t.text)) fail_at(t, "non-integer literal '" + t.text + "' in index");
      next();
      return add_const(prog_, std::stoll(t.text));
    }
    if (is_word("min") && is("(", 1)) {
      next();
      next();
      int32_t a = iexpr();
      expect(",", "between min arguments");
      int32_t b = iexpr();
      expect(")", "to close min");
      return add_bin(prog_, IntOp::Min, a, b);
    }
    if (t.kind != TK::Ident) fail_at(t, "expected index expression, got '" + t.text + "'");
    const int s = symbol(t.text);
    if (s < 0) fail_at(t, "unknown symbol '" + t.text + "' in index expression");
    next();
    return add_sym(prog_, s);
  }

  // ---- float expressions
  int32_t push_float(const FloatNode& f) {
    prog_.floats.push_back(f);
    return static_cast<int32_t>(prog_.floats.size()) - 1;
  }
  int32_t fexpr() {
    int32_t e = fterm();
    while (is("+") || is("-")) {
      FloatNode f;
      f.op = next().text == "+" ? FloatOp::Add : FloatOp::Sub;
      f.a = e;
      f.b = fterm();
      e = push_float(f);
    }
    return e;
  }
  int32_t fterm() {
    int32_t e = funary();
    while (is("*")) {
      next();
      FloatNode f;
      f.op = FloatOp::Mul;
      f.a = e;
      f.b = funary();
      e = push_float(f);
    }
    return e;
  }
  int32_t number(bool negative) {
    const Token& t = next();
    std::string s = t.text;
    if (!s.empty() && s.back() == 'f') s.pop_back();
    float v = std::stof(s);
    return add_float_const(prog_, negative ? -v : v);
  }
  int32_t funary() {
    if (is("-")) {
      if (peek(1).kind == TK::Number && peek(1).glued_prev) {
        next();
        return number(true);
      }
      next();
      FloatNode f;
      f.op = FloatOp::Neg;
      f.a = funary();
      return push_float(f);
    }
    return fprimary();
  }
  bool memref(FloatNode* out) {
    if (!(is_word("onchip") || is_word("global"))) return false;
    const bool global = next().text == "global";
    FloatNode f;
    f.op = FloatOp::Load;
    f.global = global;
    f.slot = element(ident("element name"));
    expect("[", "in memory reference");
    f.idx0 = iexpr();
    if (is(",")) {
      next();
      f.idx1 = iexpr();
      prog_.elements[f.slot].dims = 2;
    }
    expect("]", "in memory reference");
    *out = f;
    return true;
  }
  int32_t fprimary() {
    const Token& t = peek();
    if (is("(")) {
      next();
      int32_t e = fexpr();
      expect(")", "to close parenthesis");
      return e;
    }
    FloatNode m;
    if (memref(&m)) return push_float(m);
    if (is_word("fma") && is("(", 1)) {
      next();
      next();
      FloatNode f;
      f.op = FloatOp::Fma;
      f.a = fexpr();
      expect(",", "in fma");
      f.b = fexpr();
      expect(",", "in fma");
      f.c = fexpr();
      expect(")", "to close fma");
      return push_float(f);
    }
    if (t.kind == TK::Number) return number(false);
    if (t.kind != TK::Ident) fail_at(t, "expected value, got '" + t.text + "'");
    const std::string name = t.text;
    FloatNode f;
    if (int s = index_of(prog_.temps, name); s >= 0) {
      f.op = FloatOp::Temp;
      f.slot = s;
    } else if (int q = index_of(prog_.params, name); q >= 0) {
      f.op = FloatOp::Param;
      f.slot = q;
    } else {
      fail_at(t, "unknown value '" + name + "' (not a temp or scalar parameter)");
    }
    next();
    return push_float(f);
  }

  CmpOp cmp() {
    const Token& t = next();
    if (t.kind == TK::Punct) {
      if (t.text == "==") return CmpOp::Eq;
      if (t.text == "!=") return CmpOp::Ne;
      if (t.text == "<") return CmpOp::Lt;
      if (t.text == "<=") return CmpOp::Le;
      if (t.text == ">") return CmpOp::Gt;
      if (t.text == ">=") return CmpOp::Ge;
    }
    fail_at(t, "expected comparison operator, got '" + t.text + "'");
  }

  void block(std::vector<Stmt>* body) {
    expect("{", "to open block");
    while (!is("}")) {
      if (peek().kind == TK::End) fail_at(peek(), "unexpected end of input inside block");
      body->push_back(statement());
    }
    next();
  }

  Stmt statement() {
    Stmt s;
    const Token& head = peek();
    if (is_word("for")) {
      next();
      s.kind = StmtKind::For;
      const Token& vt = peek();
      const std::string var = ident("loop variable");
      if (symbol(var) >= 0) fail_at(vt, "loop variable '" + var + "' shadows an existing symbol");
      prog_.extra_syms.push_back({var, ExtraSymKind::LoopVar});
      s.loop_sym = prog_.symbol_count() - 1;
      expect("=", "in for");
      s.begin = iexpr();
      expect("..", "in for");
      s.end = iexpr();
      if (is_word("step")) {
        next();
        s.step = iexpr();
      } else {
        s.step = add_const(prog_, 1);
      }
      if (is_word("unroll")) {
        next();
        s.unroll = true;
      }
      block(&s.body);
      return s;
    }
    if (is_word("if")) {
      next();
      s.kind = StmtKind::If;
      s.cmp_lhs = iexpr();
      s.cmp = cmp();
      s.cmp_rhs = iexpr();
      block(&s.body);
      return s;
    }
    if (ctx_.allow_kernel_stmts && is_word("barrier")) {
      next();
      s.kind = StmtKind::Barrier;
      return s;
    }
    if (ctx_.allow_kernel_stmts && is_word("clear")) {
      next();
      s.kind = StmtKind::Clear;
      s.element = element(ident("element to clear"));
      return s;
    }
    if (is_word("atomic")) {
      next();
      FloatNode m;
      if (!memref(&m)) fail_at(peek(), "expected memory reference after 'atomic'");
      s.kind = StmtKind::AtomicAdd;
      s.global = m.global;
      s.element = m.slot;
      s.idx0 = m.idx0;
      s.idx1 = m.idx1;
      expect("+=", "in atomic add");
      s.fexpr = fexpr();
      return s;
    }
    if (is_word("float")) {
      next();
      s.kind = StmtKind::DeclTemp;
      const Token& nt = peek();
      const std::string name = ident("temp name");
      if (index_of(prog_.temps, name) >= 0) fail_at(nt, "duplicate temp '" + name + "'");
      prog_.temps.push_back(name);
      s.temp_slot = static_cast<int>(prog_.temps.size()) - 1;
      expect("=", "in temp declaration");
      s.fexpr = fexpr();
      return s;
    }
    FloatNode m;
    if (memref(&m)) {
      s.kind = StmtKind::Store;
      s.global = m.global;
      s.element = m.slot;
      s.idx0 = m.idx0;
      s.idx1 = m.idx1;
      expect("=", "after memory reference");
      s.fexpr = fexpr();
      return s;
    }
    if (head.kind != TK::Ident) fail_at(head, "expected statement, got '" + head.text + "'");
    const int t = index_of(prog_.temps, head.text);
    if (t < 0) fail_at(head, "unknown statement or temp '" + head.text + "'");
    next();
    s.kind = StmtKind::AssignTemp;
    s.temp_slot = t;
    if (is("+=")) {
      next();
      const int32_t rhs = fexpr();
      FloatNode self;
      self.op = FloatOp::Temp;
      self.slot = t;
      const int32_t self_i = push_float(self);
      const FloatNode r = prog_.floats[rhs];
      FloatNode acc;
      if (r.op == FloatOp::Mul) {  // t += a*b  ->  fma(a, b, t)
        acc.op = FloatOp::Fma;
        acc.a = r.a;
        acc.b = r.b;
        acc.c = self_i;
      } else {
        acc.op = FloatOp::Add;
        acc.a = self_i;
        acc.b = rhs;
      }
      s.fexpr = push_float(acc);
      return s;
    }
    expect("=", "in assignment");
    s.fexpr = fexpr();
    return s;
  }
};

// ===========================================================================
// Printer helpers
int int_prec(const IntNode& n) {
  switch (n.op) {
    case IntOp::Add:
    case IntOp::Sub: return 1;
    case IntOp::Mul:
    case IntOp::Div:
    case IntOp::Mod: return 2;
    default: return 3;
  }
}

std::string fmt_float(float v) {
  char buf[48];
  for (int prec = 6; prec <= 9; ++prec) {  // shortest form that round-trips
    std::snprintf(buf, sizeof buf, "%.*g", prec, static_cast<double>(v));
    if (std::stof(buf) == v) break;
  }
  std::string s = buf;
  if (s.find_first_of(".en") == std::string::npos) s += ".0";
  return s;
}

int float_prec(const FloatNode& n) {
  switch (n.op) {
    case FloatOp::Add:
    case FloatOp::Sub: return 1;
    case FloatOp::Mul: return 2;
    default: return 3;
  }
}

}  // namespace

Program parse_program(const std::string& text, const ParseContext& ctx, int first_line) {
  return Parser(text, ctx, first_line).run();
}

std::string print_int_expr(const Program& p, int32_t node) {
  const IntNode& n = p.ints.at(node);
  auto sym = [&](int s) -> std::string {
    return s < kNumBuiltinSyms ? kBuiltinNames[s] : p.extra_syms.at(s - kNumBuiltinSyms).name;
  };
  auto side = [&](int32_t child, bool right, int prec) {
    std::string s = print_int_expr(p, child);
    const int cp = int_prec(p.ints[child]);
    return (cp < prec || (right && cp == prec)) ? "(" + s + ")" : s;
  };
  switch (n.op) {
    case IntOp::Const: return std::to_string(n.value);
    case IntOp::Sym: return sym(static_cast<int>(n.value));
    case IntOp::Add: return side(n.lhs, false, 1) + " + " + side(n.rhs, true, 1);
    case IntOp::Sub: {
      const IntNode& l = p.ints[n.lhs];
      if (l.op == IntOp::Const && l.value == 0) {
        std::string r = print_int_expr(p, n.rhs);
        return int_prec(p.ints[n.rhs]) < 3 ? "-(" + r + ")" : "-" + r;
      }
      return side(n.lhs, false, 1) + " - " + side(n.rhs, true, 1);
    }
    case IntOp::Mul: return side(n.lhs, false, 2) + "*" + side(n.rhs, true, 2);
    case IntOp::Div: return side(n.lhs, false, 2) + "/" + side(n.rhs, true, 2);
    case IntOp::Mod: return side(n.lhs, false, 2) + " % " + side(n.rhs, true, 2);
    case IntOp::Min:
      return "min(" + print_int_expr(p, n.lhs) + ", " + print_int_expr(p, n.rhs) + ")";
  }
  return "?";
}

std::string print_float_expr(const Program& p, int32_t node) {
  const FloatNode& n = p.floats.at(node);
  auto side = [&](int32_t child, bool right, int prec) {
    std::string s = print_float_expr(p, child);
    const int cp = float_prec(p.floats[child]);
    return (cp < prec || (right && cp == prec)) ? "(" + s + ")" : s;
  };
  switch (n.op) {
    case FloatOp::Const: return fmt_float(n.value);
    case FloatOp::Temp: return p.temps.at(n.slot);
    case FloatOp::Param: return p.params.at(n.slot);
    case FloatOp::Load: {
      std::string s = std::string(n.global ? "global " : "onchip ") + p.elements.at(n.slot).name +
                      "[" + print_int_expr(p, n.idx0);
      if (n.idx1 >= 0) s += ", " + print_int_expr(p, n.idx1);
      return s + "]";
    }
    case FloatOp::Add: return side(n.a, false, 1) + " + " + side(n.b, true, 1);
    case FloatOp::Sub: return side(n.a, false, 1) + " - " + side(n.b, true, 1);
    case FloatOp::Mul: return side(n.a, false, 2) + "*" + side(n.b, true, 2);
    case FloatOp::Neg: {
      std::string s = print_float_expr(p, n.a);
      return float_prec(p.floats[n.a]) < 3 || p.floats[n.a].op == FloatOp::Const ? "-(" + s + ")"
                                                                                : "-" + s;
    }
    case FloatOp::Fma:
      return "fma(" + print_float_expr(p, n.a) + ", " + print_float_expr(p, n.b) + ", " +
             print_float_expr(p, n.c) + ")";
  }
  return "?";
}

std::string print_stmt(const Program& p, const Stmt& s, int indent) {
  const std::string pad(static_cast<size_t>(indent) * 2, ' ');
  auto body = [&](const std::string& head) {
    std::string o = pad + head + " {\n";
    for (const auto& b : s.body) o += print_stmt(p, b, indent + 1);
    return o + pad + "}\n";
  };
  auto mem = [&](bool global, int elem, int32_t i0, int32_t i1) {
    std::string o = std::string(global ? "global " : "onchip ") + p.elements.at(elem).name + "[" +
                    print_int_expr(p, i0);
    if (i1 >= 0) o += ", " + print_int_expr(p, i1);
    return o + "]";
  };
  static const char* const kCmp[] = {"==", "!=", "<", "<=", ">", ">="};
  switch (s.kind) {
    case StmtKind::For: {
      std::string h = "for " + p.extra_syms.at(s.loop_sym - kNumBuiltinSyms).name + " = " +
                      print_int_expr(p, s.begin) + " .. " + print_int_expr(p, s.end);
      const IntNode& st = p.ints.at(s.step);
      if (!(st.op == IntOp::Const && st.value == 1)) h += " step " + print_int_expr(p, s.step);
      if (s.unroll) h += " unroll";
      return body(h);
    }
    case StmtKind::If:
      return body("if " + print_int_expr(p, s.cmp_lhs) + " " + kCmp[static_cast<int>(s.cmp)] +
                  " " + print_int_expr(p, s.cmp_rhs));
    case StmtKind::DeclTemp:
      return pad + "float " + p.temps.at(s.temp_slot) + " = " + print_float_expr(p, s.fexpr) + "\n";
    case StmtKind::AssignTemp:
      return pad + p.temps.at(s.temp_slot) + " = " + print_float_expr(p, s.fexpr) + "\n";
    case StmtKind::Store:
      return pad + mem(s.global, s.element, s.idx0, s.idx1) + " = " +
             print_float_expr(p, s.fexpr) + "\n";
    case StmtKind::AtomicAdd:
      return pad + "atomic " + mem(s.global, s.element, s.idx0, s.idx1) + " += " +
             print_float_expr(p, s.fexpr) + "\n";
    case StmtKind::Barrier: return pad + "barrier\n";
    case StmtKind::Clear: return pad + "clear " + p.elements.at(s.element).name + "\n";
  }
  return pad + "?\n";
}

std::string print_program(const Program& p, int indent) {
  std::string o;
  for (const auto& s : p.stmts) o += print_stmt(p, s, indent);
  return o;
}

Program substitute_macros(const Program& p, const std::map<std::string, int64_t>& values) {
  Program q = p;
  for (size_t i = 0; i < q.extra_syms.size(); ++i) {
    if (q.extra_syms[i].kind != ExtraSymKind::Macro) continue;
    auto it = values.find(q.extra_syms[i].name);
    if (it == values.end())
      throw std::runtime_error("unresolved macro '" + q.extra_syms[i].name + "'");
    const int64_t slot = kNumBuiltinSyms + static_cast<int64_t>(i);
    for (auto& n : q.ints)
      if (n.op == IntOp::Sym && n.value == slot) {
        n.op = IntOp::Const;
        n.value = it->second;
      }
  }
  return q;
}

}  // namespace mapfuse::ir
