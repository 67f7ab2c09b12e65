// host/lower.cpp -- KernelIR -> hand-written sm_100a kernel family.
//
// The reference executes a KernelIR by interpreting it (proj/src/vm.cpp).
// Here the KernelIR is *read*: load routines say which on-chip keys come
// from which global buffers, store routines which keys go back out, and the
// compute routines are evaluated symbolically (semantics.cpp).  The
// resulting dataflow is composed -- values produced inside the kernel are
// substituted into their consumers -- and matched against the two kernel
// families:
//   depth 1 (and depth-2 tile maps without reductions): StreamOp, up to 4
//     input streams, 2 stored linear combinations and one dot reduction;
//   depth 2: MatrixOp, one pass over <= 2 matrices with an optional rank-2
//     update of the first (stored or not), <= 2 row and <= 2 column
//     reductions.
// Anything else has no template and the selector treats it as infeasible.
#include <algorithm>
#include <functional>
#include <set>
#include <stdexcept>

#include "mapfuse/planner.hpp"
#include "semantics.hpp"

namespace mapfuse::plan {

using b200::Coef;

bool stream_template_exists(int nin, int nout, bool dot) {
  // every (inputs 1..4) x (stored outputs 0..2) x (dot) with something to write
  return nin >= 1 && nin <= 4 && nout >= 0 && nout <= 2 && (nout > 0 || dot);
}

bool matrix_template_exists(int nmat, int nrank, int store, int nrow, int ncol) {
  const int s[8][5] = {{1, 0, 0, 1, 0}, {1, 0, 0, 0, 1}, {1, 0, 0, 1, 1}, {1, 0, 0, 2, 0},
                       {1, 0, 0, 0, 2}, {1, 2, 1, 0, 1}, {1, 2, 1, 0, 0}, {2, 0, 0, 2, 0}};
  for (const auto& r : s)
    if (r[0] == nmat && r[1] == nrank && r[2] == store && r[3] == nrow && r[4] == ncol) return true;
  return false;
}

namespace {

using LinComb = std::vector<std::pair<std::string, Coef>>;  // buffer -> coefficient

void lc_add(LinComb& acc, const std::string& buf, const Coef& c) {
  for (auto& [b, k] : acc)
    if (b == buf) {
      k = k + c;
      return;
    }
  acc.push_back({buf, c});
}

// Which global buffer a routine moves into / out of an on-chip key.
void scan_moves(const ir::Program& p, const std::vector<ir::Stmt>& ss,
                std::map<std::string, std::string>* loads, std::map<std::string, std::string>* stores,
                std::map<std::string, int>* dims) {
  for (const auto& s : ss) {
    if (s.kind == ir::StmtKind::Store || s.kind == ir::StmtKind::AtomicAdd) {
      const ir::FloatNode& v = p.floats.at(s.fexpr);
      if (v.op == ir::FloatOp::Load && v.global != s.global) {
        const std::string dst = p.elements.at(s.element).name, src = p.elements.at(v.slot).name;
        if (!s.global) (*loads)[dst] = src;
        else (*stores)[src] = dst;
        const std::string& key = s.global ? src : dst;
        (*dims)[key] = std::max((*dims)[key], s.idx1 >= 0 || v.idx1 >= 0 ? 2 : 1);
      }
    }
    scan_moves(p, s.body, loads, stores, dims);
  }
}

}  // namespace

b200::NativeKernel lower_kernel(const kernel::KernelIR& k) {
  std::map<std::string, std::string> loads, stores;  // key -> buffer, key -> buffer
  std::map<std::string, int> dims;
  std::map<std::string, sem::CallSemantics> computed;  // key -> what produced it
  std::vector<std::string> compute_order;
  std::set<int> call_ids;
  for (const auto* sec : {&k.prologue, &k.body, &k.epilogue})
    for (const auto& c : *sec) {
      if (c.is_pure_clear()) continue;
      call_ids.insert(c.call_id);
      if (c.kind != lib::RoutineKind::Compute) {
        scan_moves(c.body, c.body.stmts, &loads, &stores, &dims);
        continue;
      }
      std::vector<Coef> pv;
      for (const auto& nm : c.body.params) pv.push_back(Coef::symbol(nm));
      for (auto& cs : sem::classify(sem::evaluate(c.body, pv))) {
        if (computed.count(cs.out))
          throw std::invalid_argument("lowering: key '" + cs.out + "' computed twice");
        compute_order.push_back(cs.out);
        computed[cs.out] = std::move(cs);
      }
    }
  using K = sem::CallSemantics::Kind;
  b200::NativeKernel nk;
  nk.name = k.name;
  nk.calls.assign(call_ids.begin(), call_ids.end());

  // ---- resolve vector / tile-map values into linear combinations of buffers
  std::map<std::string, LinComb> memo;
  std::function<LinComb(const std::string&)> resolve = [&](const std::string& key) -> LinComb {
    if (auto it = memo.find(key); it != memo.end()) return it->second;
    LinComb out;
    if (auto l = loads.find(key); l != loads.end()) {
      out.push_back({l->second, Coef::constant(1.0)});
    } else if (auto c = computed.find(key); c != computed.end() &&
                                            (c->second.kind == K::Map || c->second.kind == K::TileMap)) {
      if (!c->second.rank.empty()) throw std::invalid_argument("lowering: rank update in a stream");
      for (const auto& [src, coef] : c->second.lin)
        for (const auto& [b, k2] : resolve(src)) lc_add(out, b, coef * k2);
    } else {
      throw std::invalid_argument("lowering: value '" + key + "' is neither loaded nor mapped");
    }
    return memo[key] = out;
  };

  bool has_reduce2 = false, has_rank = false;
  for (const auto& [key, cs] : computed) {
    has_reduce2 |= cs.kind == K::RowReduce || cs.kind == K::ColReduce;
    has_rank |= !cs.rank.empty();
  }

  if (!has_reduce2 && !has_rank) {
    // ---------------- StreamOp
    nk.kind = b200::NativeKernel::Kind::Stream;
    b200::StreamOp& op = nk.stream;
    auto input_index = [&](const std::string& b) {
      auto it = std::find(op.inputs.begin(), op.inputs.end(), b);
      if (it != op.inputs.end()) return static_cast<int>(it - op.inputs.begin());
      op.inputs.push_back(b);
      return static_cast<int>(op.inputs.size()) - 1;
    };
    struct Pending {
      std::string buf;
      LinComb lc;
    };
    std::vector<Pending> outs;
    for (const auto& key : compute_order) {
      const auto& cs = computed.at(key);
      auto st = stores.find(key);
      if (cs.kind == K::Dot) {
        if (op.has_dot) throw std::invalid_argument("lowering: more than one dot reduction");
        if (st == stores.end()) throw std::invalid_argument("lowering: dot result never stored");
        op.has_dot = true;
        op.dot_out = st->second;
        LinComb a = resolve(cs.a), b = resolve(cs.b);
        for (auto& [x, c] : a) c = c * cs.coef;
        for (const auto& [x, c] : a) input_index(x);
        for (const auto& [x, c] : b) input_index(x);
        outs.push_back({"__dot_a", a});
        outs.push_back({"__dot_b", b});
      } else if (st != stores.end()) {
        LinComb lc = resolve(key);
        for (const auto& [x, c] : lc) input_index(x);
        outs.push_back({st->second, lc});
      }
    }
    auto dense = [&](const LinComb& lc) {
      std::vector<Coef> v(op.inputs.size(), Coef::constant(0.0));
      for (const auto& [x, c] : lc) v[static_cast<size_t>(input_index(x))] = c;
      return v;
    };
    for (const auto& p : outs) {
      if (p.buf == "__dot_a") op.dot_a = dense(p.lc);
      else if (p.buf == "__dot_b") op.dot_b = dense(p.lc);
      else op.outs.push_back({p.buf, {}});
    }
    size_t oi = 0;
    for (const auto& p : outs)
      if (p.buf != "__dot_a" && p.buf != "__dot_b") op.outs[oi++].coef = dense(p.lc);
    // pad the dot coefficient vectors to the final input count
    for (auto* v : {&op.dot_a, &op.dot_b})
      while (op.has_dot && v->size() < op.inputs.size()) v->push_back(Coef::constant(0.0));
    for (auto& o : op.outs)
      while (o.coef.size() < op.inputs.size()) o.coef.push_back(Coef::constant(0.0));
    if (!stream_template_exists(static_cast<int>(op.inputs.size()), static_cast<int>(op.outs.size()),
                                op.has_dot))
      throw std::invalid_argument("lowering: no stream template for " +
                                  std::to_string(op.inputs.size()) + " inputs / " +
                                  std::to_string(op.outs.size()) + " outputs");
    return nk;
  }

  // ---------------- MatrixOp
  nk.kind = b200::NativeKernel::Kind::Matrix;
  b200::MatrixOp& op = nk.matrix;
  auto external_vector = [&](const std::string& key) {
    auto l = loads.find(key);
    if (l == loads.end())
      throw std::invalid_argument("lowering: vector '" + key + "' is not loaded from memory");
    return l->second;
  };
  // matrix operand: a loaded tile, or a tile map = base + rank terms
  struct Mat {
    std::string base;
    std::vector<std::pair<std::string, std::string>> rank;
    std::string stored;
  };
  auto operand = [&](const std::string& key) {
    Mat m;
    if (auto l = loads.find(key); l != loads.end()) {
      m.base = l->second;
      return m;
    }
    auto c = computed.find(key);
    if (c == computed.end() || c->second.kind != K::TileMap)
      throw std::invalid_argument("lowering: tile '" + key + "' has no source");
    if (c->second.lin.size() != 1) throw std::invalid_argument("lowering: tile map of several tiles");
    const auto& [src, coef] = c->second.lin[0];
    if (coef.terms.size() != 1 || coef.terms[0].c != 1.0 || !coef.terms[0].syms.empty())
      throw std::invalid_argument("lowering: scaled tile map");
    m.base = external_vector(src);
    for (const auto& r : c->second.rank) {
      if (r.coef.terms.size() != 1 || r.coef.terms[0].c != 1.0 || !r.coef.terms[0].syms.empty())
        throw std::invalid_argument("lowering: scaled rank update");
      m.rank.push_back({external_vector(r.u), external_vector(r.v)});
    }
    if (auto st = stores.find(key); st != stores.end()) m.stored = st->second;
    return m;
  };
  // row-resident chains: a column reduction whose vector is a row reduction
  // of the same matrix computed in this kernel (planner mode "b200")
  std::set<std::string> chained_rows;
  for (const auto& [key, cs] : computed) {
    if (cs.kind != K::ColReduce) continue;
    auto src = computed.find(cs.b);
    if (src != computed.end() && src->second.kind == K::RowReduce && src->second.a == cs.a)
      chained_rows.insert(cs.b);
  }
  std::vector<Mat> mats;
  auto mat_index = [&](const Mat& m) {
    for (size_t i = 0; i < mats.size(); ++i)
      if (mats[i].base == m.base) {
        if (mats[i].rank != m.rank) throw std::invalid_argument("lowering: one matrix, two updates");
        // the same update stored under two names (two identical ger2 calls):
        // the matrix kernel has one store -- leave it to the generic kernel
        if (!mats[i].stored.empty() && !m.stored.empty() && mats[i].stored != m.stored)
          throw std::invalid_argument("lowering: one matrix update stored twice");
        if (mats[i].stored.empty()) mats[i].stored = m.stored;
        return static_cast<int>(i);
      }
    mats.push_back(m);
    return static_cast<int>(mats.size()) - 1;
  };
  for (const auto& key : compute_order) {
    const auto& cs = computed.at(key);
    if (cs.kind == K::TileMap) {
      if (stores.count(key)) mat_index(operand(key));  // ger2 whose result leaves the kernel
      continue;
    }
    if (cs.kind != K::RowReduce && cs.kind != K::ColReduce)
      throw std::invalid_argument("lowering: depth-2 kernel mixes in a vector map / dot");
    auto st = stores.find(key);
    const int mi = mat_index(operand(cs.a));
    if (cs.kind == K::RowReduce && chained_rows.count(key)) {
      op.chain = true;
      op.rows.push_back({mi, external_vector(cs.b), st == stores.end() ? "" : st->second, cs.coef});
      continue;
    }
    if (st == stores.end())
      throw std::invalid_argument("lowering: reduction '" + key + "' consumed inside the kernel");
    if (cs.kind == K::ColReduce && chained_rows.count(cs.b)) {
      op.cols.push_back({mi, cs.b, st->second, cs.coef});
      continue;
    }
    b200::MatrixOp::Red red{mi, external_vector(cs.b), st->second, cs.coef};
    (cs.kind == K::RowReduce ? op.rows : op.cols).push_back(red);
  }
  // the rank-updated matrix must be mats[0]
  for (size_t i = 1; i < mats.size(); ++i)
    if (!mats[i].rank.empty()) {
      std::swap(mats[0], mats[i]);
      for (auto* list : {&op.rows, &op.cols})
        for (auto& r : *list) r.mat = r.mat == 0 ? static_cast<int>(i) : (r.mat == static_cast<int>(i) ? 0 : r.mat);
    }
  for (const auto& m : mats) op.mats.push_back(m.base);
  if (!mats.empty()) {
    op.rank = mats[0].rank;
    op.store = mats[0].stored;
  }
  for (size_t i = 1; i < mats.size(); ++i)
    if (!mats[i].stored.empty()) throw std::invalid_argument("lowering: stored second matrix");
  // two-matrix kernels pair reduction o with matrix o
  if (op.mats.size() == 2) {
    std::sort(op.rows.begin(), op.rows.end(), [](const auto& a, const auto& b) { return a.mat < b.mat; });
    std::sort(op.cols.begin(), op.cols.end(), [](const auto& a, const auto& b) { return a.mat < b.mat; });
    for (size_t o = 0; o < op.rows.size(); ++o)
      if (op.rows[o].mat != static_cast<int>(o)) throw std::invalid_argument("lowering: row pairing");
    for (size_t o = 0; o < op.cols.size(); ++o)
      if (op.cols[o].mat != static_cast<int>(o)) throw std::invalid_argument("lowering: col pairing");
  } else {
    for (const auto* list : {&op.rows, &op.cols})
      for (const auto& r : *list)
        if (r.mat != 0) throw std::invalid_argument("lowering: matrix index");
  }
  if (op.chain) {
    if (op.mats.size() != 1 || !op.rank.empty() || !op.store.empty() || op.rows.size() != 1 ||
        op.cols.size() != 1)
      throw std::invalid_argument("lowering: row-resident chain must be one row + one column "
                                  "reduction of one matrix");
    return nk;
  }
  if (!matrix_template_exists(static_cast<int>(op.mats.size()), static_cast<int>(op.rank.size()),
                              op.store.empty() ? 0 : 1, static_cast<int>(op.rows.size()),
                              static_cast<int>(op.cols.size())))
    throw std::invalid_argument("lowering: no matrix template for this fusion shape");
  return nk;
}

}  // namespace mapfuse::plan
