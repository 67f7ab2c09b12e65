// host/semantics.cpp -- symbolic evaluation + classification of routine bodies.
#include "semantics.hpp"

#include <stdexcept>

namespace mapfuse::sem {

namespace {

Poly mul(const Poly& a, const Poly& b) {
  Poly r;
  for (const auto& x : a)
    for (const auto& y : b) {
      Term t;
      t.coef = x.coef * y.coef;
      t.f = x.f;
      t.f.insert(t.f.end(), y.f.begin(), y.f.end());
      r.push_back(std::move(t));
    }
  return r;
}

Poly add(Poly a, const Poly& b) {
  a.insert(a.end(), b.begin(), b.end());
  return a;
}

Poly neg(Poly a) {
  for (auto& t : a) t.coef = Coef::constant(-1.0) * t.coef;
  return a;
}

struct Evaluator {
  const ir::Program& p;
  const std::vector<Coef>& params;
  std::vector<std::optional<Poly>> temps;
  std::vector<Assign> out;

  ir::LinearForm index(int32_t node) const {
    auto lf = p.linear(node);
    if (!lf) throw std::runtime_error("semantics: non-affine on-chip index");
    return *lf;
  }

  Poly value(int32_t fe) {
    const ir::FloatNode& n = p.floats.at(fe);
    switch (n.op) {
      case ir::FloatOp::Const:
        if (n.value == 0.0f) return {};  // additive identity: drop
        return {Term{Coef::constant(n.value), {}}};
      case ir::FloatOp::Param:
        if (n.slot < 0 || n.slot >= (int)params.size())
          throw std::runtime_error("semantics: unbound parameter");
        return {Term{params[n.slot], {}}};
      case ir::FloatOp::Temp:
        if (!temps.at(n.slot)) throw std::runtime_error("semantics: temp read before write");
        return *temps[n.slot];
      case ir::FloatOp::Load: {
        if (n.global) throw std::runtime_error("semantics: compute routine reads global memory");
        Factor f;
        f.elem = p.elements.at(n.slot).name;
        f.idx.push_back(index(n.idx0));
        if (n.idx1 >= 0) f.idx.push_back(index(n.idx1));
        return {Term{Coef::constant(1.0), {f}}};
      }
      case ir::FloatOp::Add: return add(value(n.a), value(n.b));
      case ir::FloatOp::Sub: return add(value(n.a), neg(value(n.b)));
      case ir::FloatOp::Mul: return mul(value(n.a), value(n.b));
      case ir::FloatOp::Neg: return neg(value(n.a));
      case ir::FloatOp::Fma: return add(mul(value(n.a), value(n.b)), value(n.c));
    }
    throw std::runtime_error("semantics: unknown float node");
  }

  void run(const std::vector<ir::Stmt>& ss) {
    for (const auto& s : ss) {
      switch (s.kind) {
        case ir::StmtKind::For:
        case ir::StmtKind::If: run(s.body); break;  // loops stay symbolic; guards are thread filters
        case ir::StmtKind::DeclTemp:
        case ir::StmtKind::AssignTemp: temps.at(s.temp_slot) = value(s.fexpr); break;
        case ir::StmtKind::Store:
        case ir::StmtKind::AtomicAdd: {
          if (s.global) throw std::runtime_error("semantics: compute routine writes global memory");
          Assign a;
          a.elem = p.elements.at(s.element).name;
          a.idx.push_back(index(s.idx0));
          if (s.idx1 >= 0) a.idx.push_back(index(s.idx1));
          a.value = value(s.fexpr);
          a.atomic = s.kind == ir::StmtKind::AtomicAdd;
          out.push_back(std::move(a));
          break;
        }
        default: break;
      }
    }
  }
};

bool is_tile(const Factor& f) { return f.idx.size() == 2; }

}  // namespace

std::vector<Assign> evaluate(const ir::Program& p, const std::vector<Coef>& param_value) {
  Evaluator e{p, param_value, std::vector<std::optional<Poly>>(p.temps.size()), {}};
  e.run(p.stmts);
  return e.out;
}

std::vector<CallSemantics> classify(const std::vector<Assign>& assigns) {
  std::vector<CallSemantics> out;
  for (const Assign& a : assigns) {
    CallSemantics cs;
    cs.out = a.elem;
    const bool out_tile = a.idx.size() == 2;
    if (out_tile) {
      if (a.atomic) throw std::runtime_error("semantics: atomic tile output is not supported");
      cs.kind = CallSemantics::Kind::TileMap;
      for (const Term& t : a.value) {
        if (t.f.size() == 1 && is_tile(t.f[0]) && t.f[0].idx == a.idx) {
          cs.lin.push_back({t.f[0].elem, t.coef});
        } else if (t.f.size() == 2 && !is_tile(t.f[0]) && !is_tile(t.f[1])) {
          // u[row] * v[col]  (either factor order)
          const Factor *u = &t.f[0], *v = &t.f[1];
          if (!(u->idx[0] == a.idx[0] && v->idx[0] == a.idx[1])) std::swap(u, v);
          if (!(u->idx[0] == a.idx[0] && v->idx[0] == a.idx[1]))
            throw std::runtime_error("semantics: outer product not aligned with the tile");
          cs.rank.push_back({u->elem, v->elem, t.coef});
        } else {
          throw std::runtime_error("semantics: tile term outside map / rank-update algebra");
        }
      }
    } else if (a.atomic) {
      // reductions: every term a product of two loads
      bool have = false;
      for (const Term& t : a.value) {
        if (t.f.size() != 2) throw std::runtime_error("semantics: reduction term is not a product");
        const Factor *x = &t.f[0], *y = &t.f[1];
        CallSemantics::Kind kind;
        std::string ta, tb;
        if (is_tile(*x) || is_tile(*y)) {
          if (!is_tile(*x)) std::swap(x, y);
          if (is_tile(*y)) throw std::runtime_error("semantics: tile x tile product");
          if (y->idx[0] == x->idx[1] && a.idx[0] == x->idx[0]) kind = CallSemantics::Kind::RowReduce;
          else if (y->idx[0] == x->idx[0] && a.idx[0] == x->idx[1]) kind = CallSemantics::Kind::ColReduce;
          else throw std::runtime_error("semantics: contraction index does not match the tile");
          ta = x->elem;
          tb = y->elem;
        } else {
          kind = CallSemantics::Kind::Dot;
          ta = x->elem;
          tb = y->elem;
        }
        if (have && (kind != cs.kind || ta != cs.a || tb != cs.b))
          throw std::runtime_error("semantics: mixed reduction terms");
        cs.kind = kind;
        cs.a = ta;
        cs.b = tb;
        cs.coef = have ? cs.coef + t.coef : t.coef;
        have = true;
      }
      if (!have) throw std::runtime_error("semantics: empty reduction");
    } else {
      cs.kind = CallSemantics::Kind::Map;
      for (const Term& t : a.value) {
        if (t.f.size() != 1 || is_tile(t.f[0]) || !(t.f[0].idx == a.idx))
          throw std::runtime_error("semantics: vector map term is not element-wise linear");
        cs.lin.push_back({t.f[0].elem, t.coef});
      }
    }
    out.push_back(std::move(cs));
  }
  return out;
}

}  // namespace mapfuse::sem
