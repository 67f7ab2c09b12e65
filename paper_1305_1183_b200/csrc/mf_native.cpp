// mf_native.cpp -- coefficient algebra, traffic accounting, plan description.
#include "mf_native.hpp"

#include <algorithm>
#include <cmath>
#include <set>
#include <iomanip>
#include <sstream>
#include <stdexcept>

namespace mapfuse::b200 {

Coef Coef::operator*(const Coef& o) const {
  Coef r;
  for (const auto& a : terms)
    for (const auto& b : o.terms) {
      Term t{a.c * b.c, a.syms};
      t.syms.insert(t.syms.end(), b.syms.begin(), b.syms.end());
      std::sort(t.syms.begin(), t.syms.end());
      r.terms.push_back(std::move(t));
    }
  return r;
}

Coef Coef::operator+(const Coef& o) const {
  Coef r = *this;
  for (const auto& t : o.terms) {
    bool merged = false;
    for (auto& x : r.terms)
      if (x.syms == t.syms) {
        x.c += t.c;
        merged = true;
        break;
      }
    if (!merged) r.terms.push_back(t);
  }
  r.terms.erase(std::remove_if(r.terms.begin(), r.terms.end(),
                               [](const Term& t) { return t.c == 0.0; }),
                r.terms.end());
  return r;
}

double Coef::eval(const std::map<std::string, double>& scalars) const {
  double s = 0.0;
  bool first = true;
  for (const auto& t : terms) {
    double v = t.c;
    for (const auto& n : t.syms) {
      auto it = scalars.find(n);
      if (it == scalars.end()) throw std::runtime_error("unbound scalar '" + n + "'");
      v *= it->second;
    }
    s = first ? v : s + v;
    first = false;
  }
  return s;
}

std::string Coef::str() const {
  if (terms.empty()) return "0";
  std::ostringstream os;
  for (size_t i = 0; i < terms.size(); ++i) {
    if (i) os << " + ";
    os << terms[i].c;
    for (const auto& s : terms[i].syms) os << "*" << s;
  }
  return os.str();
}

std::vector<std::string> NativeKernel::inputs() const {
  if (kind == Kind::Generic) return generic.inputs;
  std::vector<std::string> v;
  auto add = [&](const std::string& s) {
    if (!s.empty() && std::find(v.begin(), v.end(), s) == v.end()) v.push_back(s);
  };
  if (kind == Kind::Stream) {
    for (const auto& s : stream.inputs) add(s);
  } else {
    for (const auto& s : matrix.mats) add(s);
    for (const auto& [u, w] : matrix.rank) {
      add(u);
      add(w);
    }
    for (const auto& r : matrix.rows) add(r.x);
    if (!matrix.chain)
      for (const auto& c : matrix.cols) add(c.x);
  }
  return v;
}

std::vector<std::string> NativeKernel::outputs() const {
  if (kind == Kind::Generic) return generic.outputs;
  std::vector<std::string> v;
  if (kind == Kind::Stream) {
    for (const auto& o : stream.outs) v.push_back(o.name);
    if (stream.has_dot) v.push_back(stream.dot_out);
  } else {
    if (!matrix.store.empty()) v.push_back(matrix.store);
    for (const auto& r : matrix.rows)
      if (!r.y.empty()) v.push_back(r.y);
    for (const auto& c : matrix.cols) v.push_back(c.y);
  }
  return v;
}

std::vector<std::string> NativeKernel::column_outputs() const {
  std::vector<std::string> v;
  if (kind == Kind::Generic) {  // cross-row (or whole-domain) accumulations
    for (const auto& a : generic.accumulated) {
      const auto it = std::find(generic.buffers.begin(), generic.buffers.end(), a);
      const char e = generic.extent[static_cast<size_t>(it - generic.buffers.begin())];
      if (e == '1' || (generic.depth == 2 && e == 'n')) v.push_back(a);
    }
    return v;
  }
  if (kind == Kind::Stream) {
    if (stream.has_dot) v.push_back(stream.dot_out);
  } else {
    for (const auto& c : matrix.cols) v.push_back(c.y);
  }
  return v;
}

bool NativePlan::row_sharded_matrix() const {
  for (const auto& k : kernels)
    if (k.kind == NativeKernel::Kind::Matrix ||
        (k.kind == NativeKernel::Kind::Generic && k.generic.depth == 2))
      return true;
  for (const auto& b : buffers)
    if (b.rows > 1) return true;
  return false;
}

std::vector<std::string> NativePlan::rank_reductions(int k) const {
  const NativeKernel& kern = kernels.at(static_cast<size_t>(k));
  std::vector<std::string> v = kern.column_outputs();
  if (!row_sharded_matrix()) return v;  // depth-1 plans: every vector is split
  // depth-1 reductions inside a matrix plan: split only if row-indexed
  std::string over;
  if (kern.kind == NativeKernel::Kind::Stream && kern.stream.has_dot && !kern.stream.inputs.empty())
    over = kern.stream.inputs[0];
  else if (kern.kind == NativeKernel::Kind::Generic && kern.generic.depth == 1)
    over = kern.generic.domain;
  if (over.empty()) return v;
  const BufferSpec* b = find(over);
  if (b && !b->row_indexed) return {};  // replicated vectors: the reduction is whole on every rank
  return v;
}

static uint64_t generic_words(const GenericOp& g, const std::vector<std::string>& names, int64_t m,
                              int64_t n) {
  uint64_t w = 0;
  for (const auto& name : names) {
    const auto it = std::find(g.buffers.begin(), g.buffers.end(), name);
    const char e = g.extent[static_cast<size_t>(it - g.buffers.begin())];
    if (g.depth == 1) w += e == '1' ? 1u : (uint64_t)n;
    else w += e == 't' ? (uint64_t)(m * n) : (e == 'm' ? (uint64_t)m : (e == 'n' ? (uint64_t)n : 1u));
  }
  return w;
}

uint64_t NativeKernel::bytes_loaded(int64_t m, int64_t n) const {
  if (kind == Kind::Generic) return 4ull * generic_words(generic, generic.inputs, m, n);
  if (kind == Kind::Stream) return 4ull * (uint64_t)stream.inputs.size() * (uint64_t)n;
  uint64_t b = 4ull * (uint64_t)matrix.mats.size() * (uint64_t)(m * n);
  std::set<std::string> seen;
  for (const auto& [u, v] : matrix.rank) {
    if (seen.insert(u).second) b += 4ull * m;
    if (seen.insert(v).second) b += 4ull * n;
  }
  for (const auto& r : matrix.rows)
    if (seen.insert(r.x).second) b += 4ull * n;
  for (const auto& c : matrix.cols)
    if (!matrix.chain && seen.insert(c.x).second) b += 4ull * m;
  return b;
}

uint64_t NativeKernel::bytes_stored(int64_t m, int64_t n) const {
  if (kind == Kind::Generic) return 4ull * generic_words(generic, generic.outputs, m, n);
  if (kind == Kind::Stream)
    return 4ull * (uint64_t)stream.outs.size() * (uint64_t)n + (stream.has_dot ? 4ull : 0ull);
  uint64_t b = matrix.store.empty() ? 0 : 4ull * (uint64_t)(m * n);
  for (const auto& r : matrix.rows)
    if (!r.y.empty()) b += 4ull * m;
  b += 4ull * n * matrix.cols.size();
  return b;
}

static int64_t stream_len(const NativePlan& p, const NativeKernel& k) {
  if (k.kind == NativeKernel::Kind::Generic) {
    const BufferSpec* b = p.find(k.generic.domain);
    return b ? (int64_t)b->rows * b->cols : p.cols;
  }
  const std::string& first = k.stream.inputs.empty() ? std::string() : k.stream.inputs[0];
  const BufferSpec* b = p.find(first);
  return b ? (int64_t)b->rows * b->cols : p.cols;
}

static bool depth1(const NativeKernel& k) {
  return k.kind == NativeKernel::Kind::Stream ||
         (k.kind == NativeKernel::Kind::Generic && k.generic.depth == 1);
}

uint64_t NativePlan::bytes_loaded() const {
  uint64_t b = 0;
  for (const auto& k : kernels)
    b += depth1(k) ? k.bytes_loaded(1, stream_len(*this, k)) : k.bytes_loaded(rows, cols);
  return b;
}

uint64_t NativePlan::bytes_stored() const {
  uint64_t b = 0;
  for (const auto& k : kernels)
    b += depth1(k) ? k.bytes_stored(1, stream_len(*this, k)) : k.bytes_stored(rows, cols);
  return b;
}

static std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    if (c == '\n') {
      o += "\\n";
      continue;
    }
    o += c;
  }
  return o + "\"";
}

std::string NativePlan::describe_json() const {
  std::ostringstream os;
  os << std::setprecision(17);
  os << "{\"sequence\":" << jstr(sequence) << ",\"rows\":" << rows << ",\"cols\":" << cols
     << ",\"bytes_loaded\":" << bytes_loaded() << ",\"bytes_stored\":" << bytes_stored()
     << ",\"kernels\":[";
  for (size_t i = 0; i < kernels.size(); ++i) {
    const auto& k = kernels[i];
    if (i) os << ",";
    os << "{\"name\":" << jstr(k.name) << ",\"kind\":"
       << (k.kind == NativeKernel::Kind::Stream
               ? "\"stream\""
               : (k.kind == NativeKernel::Kind::Matrix ? "\"matrix\"" : "\"generic\""))
       << ",\"calls\":[";
    for (size_t j = 0; j < k.calls.size(); ++j) os << (j ? "," : "") << k.calls[j];
    os << "],\"inputs\":[";
    auto in = k.inputs();
    for (size_t j = 0; j < in.size(); ++j) os << (j ? "," : "") << jstr(in[j]);
    os << "],\"outputs\":[";
    auto out = k.outputs();
    for (size_t j = 0; j < out.size(); ++j) os << (j ? "," : "") << jstr(out[j]);
    os << "],\"column_outputs\":[";
    auto co = k.column_outputs();
    for (size_t j = 0; j < co.size(); ++j) os << (j ? "," : "") << jstr(co[j]);
    os << "]";
    auto coef = [&](const Coef& c) {
      std::ostringstream o;
      o << std::setprecision(17) << "[";
      for (size_t t = 0; t < c.terms.size(); ++t) {
        o << (t ? "," : "") << "[" << c.terms[t].c << ",[";
        for (size_t q = 0; q < c.terms[t].syms.size(); ++q) o << (q ? "," : "") << jstr(c.terms[t].syms[q]);
        o << "]]";
      }
      return o.str() + "]";
    };
    auto coefs = [&](const std::vector<Coef>& v) {
      std::string o = "[";
      for (size_t t = 0; t < v.size(); ++t) o += (t ? "," : "") + coef(v[t]);
      return o + "]";
    };
    auto reds = [&](const std::vector<MatrixOp::Red>& v) {
      std::string o = "[";
      for (size_t t = 0; t < v.size(); ++t)
        o += std::string(t ? "," : "") + "{\"mat\":" + std::to_string(v[t].mat) + ",\"x\":" + jstr(v[t].x) +
             ",\"y\":" + jstr(v[t].y) + ",\"coef\":" + coef(v[t].coef) + "}";
      return o + "]";
    };
    if (k.kind == NativeKernel::Kind::Matrix) {
      const MatrixOp& m = k.matrix;
      os << ",\"op\":{\"mats\":[";
      for (size_t t = 0; t < m.mats.size(); ++t) os << (t ? "," : "") << jstr(m.mats[t]);
      os << "],\"rank\":[";
      for (size_t t = 0; t < m.rank.size(); ++t)
        os << (t ? "," : "") << "[" << jstr(m.rank[t].first) << "," << jstr(m.rank[t].second) << "]";
      os << "],\"store\":" << jstr(m.store) << ",\"chain\":" << (m.chain ? "true" : "false")
         << ",\"rows\":" << reds(m.rows) << ",\"cols\":" << reds(m.cols)
         << "},\"variant\":{\"tma\":" << k.variant_tma << ",\"k\":" << k.variant_k << "}";
    } else if (k.kind == NativeKernel::Kind::Generic) {
      const GenericOp& g = k.generic;
      os << ",\"op\":{\"depth\":" << g.depth << ",\"block\":[" << g.block_x << "," << g.block_y
         << "],\"instances\":" << g.instances << ",\"iterations\":" << g.iterations
         << ",\"domain\":" << jstr(g.domain) << ",\"shared_bytes\":" << 4 * g.shared_words_total
         << ",\"accumulated\":[";
      for (size_t t = 0; t < g.accumulated.size(); ++t) os << (t ? "," : "") << jstr(g.accumulated[t]);
      os << "],\"source_bytes\":" << g.source.size() << "}";
    } else {
      const StreamOp& st = k.stream;
      os << ",\"op\":{\"inputs\":[";
      for (size_t t = 0; t < st.inputs.size(); ++t) os << (t ? "," : "") << jstr(st.inputs[t]);
      os << "],\"outs\":[";
      for (size_t t = 0; t < st.outs.size(); ++t)
        os << (t ? "," : "") << "{\"name\":" << jstr(st.outs[t].name) << ",\"coef\":" << coefs(st.outs[t].coef) << "}";
      os << "]";
      if (st.has_dot)
        os << ",\"dot\":{\"out\":" << jstr(st.dot_out) << ",\"a\":" << coefs(st.dot_a) << ",\"b\":" << coefs(st.dot_b) << "}";
      os << "}";
    }
    if (k.kind == NativeKernel::Kind::Matrix) {
      os << ",\"shape\":{\"mats\":" << k.matrix.mats.size() << ",\"rank\":" << k.matrix.rank.size()
         << ",\"store\":" << (k.matrix.store.empty() ? 0 : 1) << ",\"rows\":" << k.matrix.rows.size()
         << ",\"cols\":" << k.matrix.cols.size() << ",\"chain\":" << (k.matrix.chain ? 1 : 0) << "}";
    } else if (k.kind == NativeKernel::Kind::Stream) {
      os << ",\"shape\":{\"inputs\":" << k.stream.inputs.size() << ",\"outs\":"
         << k.stream.outs.size() << ",\"dot\":" << (k.stream.has_dot ? 1 : 0) << "}";
    }
    os << "}";
  }
  os << "],\"buffers\":[";
  for (size_t i = 0; i < buffers.size(); ++i) {
    const auto& b = buffers[i];
    if (i) os << ",";
    os << "{\"name\":" << jstr(b.name) << ",\"rows\":" << b.rows << ",\"cols\":" << b.cols
       << ",\"role\":\""
       << (b.role == Role::Input ? "input" : (b.role == Role::Output ? "output" : "intermediate"))
       << "\",\"scalar\":" << (b.scalar ? "true" : "false")
       << ",\"row_indexed\":" << (b.row_indexed ? "true" : "false") << "}";
  }
  os << "],\"scalars\":[";
  for (size_t i = 0; i < scalars.size(); ++i) os << (i ? "," : "") << jstr(scalars[i]);
  os << "]}";
  return os.str();
}

}  // namespace mapfuse::b200
