// mf_builtin.cpp -- hand-derived native plans for the Table-1 sequences.
//
// These are the plans SURVEY.md Appendix A derives from SPEC.md's fusion
// rules (fused mode) and the one-kernel-per-call decomposition of the
// reference library (unfused mode).  The compile pipeline (mf_compile.cpp:
// planner -> selector -> codegen -> lowering) must reproduce them; tests
// compare the two.  They are also what `mf_compile_sequence` falls back to
// only when explicitly asked (MF_MODE_BUILTIN_* in tests).
#include <stdexcept>

#include "mf_builtin.hpp"

namespace mapfuse::b200 {
namespace {

int pad32(int v) { return (v + 31) / 32 * 32; }

struct B {
  NativePlan p;
  void buf(const std::string& n, int r, int c, Role role, bool row_indexed = false,
           bool scalar = false) {
    BufferSpec b;
    b.name = n;
    b.rows = r;
    b.cols = c;
    b.role = role;
    b.row_indexed = row_indexed;
    b.scalar = scalar;
    p.buffers.push_back(b);
  }
  NativeKernel& stream(const std::string& name, std::vector<int> calls,
                       std::vector<std::string> ins) {
    NativeKernel k;
    k.kind = NativeKernel::Kind::Stream;
    k.name = name;
    k.calls = std::move(calls);
    k.stream.inputs = std::move(ins);
    p.kernels.push_back(k);
    return p.kernels.back();
  }
  NativeKernel& matrix(const std::string& name, std::vector<int> calls,
                       std::vector<std::string> mats) {
    NativeKernel k;
    k.kind = NativeKernel::Kind::Matrix;
    k.name = name;
    k.calls = std::move(calls);
    k.matrix.mats = std::move(mats);
    p.kernels.push_back(k);
    return p.kernels.back();
  }
};

Coef K(double v) { return Coef::constant(v); }
Coef S(const char* s) { return Coef::symbol(s); }

void out(NativeKernel& k, const std::string& name, std::vector<Coef> c) {
  k.stream.outs.push_back({name, std::move(c)});
}
void rowred(NativeKernel& k, int mat, const std::string& x, const std::string& y, Coef c) {
  k.matrix.rows.push_back({mat, x, y, std::move(c)});
}
void colred(NativeKernel& k, int mat, const std::string& x, const std::string& y, Coef c) {
  k.matrix.cols.push_back({mat, x, y, std::move(c)});
}

}  // namespace

NativePlan builtin_plan(const std::string& seq_in, int rows, int cols, bool fused) {
  std::string seq;
  for (char c : seq_in) seq += (char)std::toupper((unsigned char)c);
  if (seq == "BICG") seq = "BICGK";
  const int m = pad32(rows), n = pad32(cols);
  B b;
  b.p.sequence = seq;
  b.p.rows = m;
  b.p.cols = n;
  const Role I = Role::Input, O = Role::Output, T = Role::Intermediate;
  if (seq == "AXPYDOT") {
    b.p.rows = 1;
    for (auto nm : {"w", "v", "u"}) b.buf(nm, 1, n, I);
    b.buf("z", 1, n, O);
    b.buf("r", 1, 1, O, false, true);
    b.p.scalars = {"alpha"};
    if (fused) {
      auto& k = b.stream("axpydot[axpydot_stage+dot]", {0, 1}, {"w", "v", "u"});
      Coef na = K(-1.0) * S("alpha");
      out(k, "z", {K(1), na, K(0)});
      k.stream.has_dot = true;
      k.stream.dot_a = {K(1), na, K(0)};
      k.stream.dot_b = {K(0), K(0), K(1)};
      k.stream.dot_out = "r";
    } else {
      auto& k0 = b.stream("axpydot_stage", {0}, {"w", "v"});
      out(k0, "z", {K(1), K(-1.0) * S("alpha")});
      auto& k1 = b.stream("dot", {1}, {"z", "u"});
      k1.stream.has_dot = true;
      k1.stream.dot_a = {K(1), K(0)};
      k1.stream.dot_b = {K(0), K(1)};
      k1.stream.dot_out = "r";
    }
  } else if (seq == "VADD") {
    b.p.rows = 1;
    for (auto nm : {"w", "y", "z"}) b.buf(nm, 1, n, I);
    b.buf("x", 1, n, O);
    if (fused) {
      out(b.stream("vadd[add+add]", {0, 1}, {"w", "y", "z"}), "x", {K(1), K(1), K(1)});
    } else {
      b.buf("t", 1, n, T);
      out(b.stream("add", {0}, {"w", "y"}), "t", {K(1), K(1)});
      out(b.stream("add", {1}, {"t", "z"}), "x", {K(1), K(1)});
    }
  } else if (seq == "WAXPBY") {
    b.p.rows = 1;
    for (auto nm : {"x", "y"}) b.buf(nm, 1, n, I);
    b.buf("w", 1, n, O);
    b.p.scalars = {"alpha", "beta"};
    if (fused) {
      out(b.stream("waxpby[scal+waxpby]", {0, 1}, {"x", "y"}), "w",
          {K(1.0) * S("alpha"), S("beta")});
    } else {
      b.buf("t", 1, n, T);
      out(b.stream("scal", {0}, {"x"}), "t", {S("alpha")});
      out(b.stream("waxpby", {1}, {"t", "y"}), "w", {K(1.0), S("beta")});
    }
  } else if (seq == "SSCAL") {
    b.p.rows = 1;
    b.buf("x", 1, n, I);
    b.buf("y", 1, n, O);
    b.p.scalars = {"alpha"};
    out(b.stream("scal", {0}, {"x"}), "y", {S("alpha")});
  } else if (seq == "MADD") {
    b.buf("A", m, n, I);
    b.buf("B", m, n, I);
    b.buf("C", m, n, O);
    out(b.stream("madd", {0}, {"A", "B"}), "C", {K(1), K(1)});
  } else if (seq == "BICGK") {
    b.buf("A", m, n, I);
    b.buf("p", 1, n, I);
    b.buf("r", 1, m, I, true);
    b.buf("q", 1, m, O, true);
    b.buf("s", 1, n, O);
    if (fused) {
      auto& k = b.matrix("bicgk[sgemv+sgemtv]", {0, 1}, {"A"});
      rowred(k, 0, "p", "q", K(1));
      colred(k, 0, "r", "s", K(1));
    } else {
      rowred(b.matrix("sgemv", {0}, {"A"}), 0, "p", "q", K(1));
      colred(b.matrix("sgemtv", {1}, {"A"}), 0, "r", "s", K(1));
    }
  } else if (seq == "ATAX") {
    b.buf("A", m, n, I);
    b.buf("x", 1, n, I);
    b.buf("t", 1, m, T, true);
    b.buf("y", 1, n, O);
    rowred(b.matrix("sgemv", {0}, {"A"}), 0, "x", "t", K(1));
    colred(b.matrix("sgemtv", {1}, {"A"}), 0, "t", "y", K(1));
  } else if (seq == "SGEMV") {
    b.buf("A", m, n, I);
    b.buf("x", 1, n, I);
    b.buf("y", 1, m, I, true);
    b.buf("t", 1, m, T, true);
    b.buf("z", 1, m, O, true);
    b.p.scalars = {"alpha", "beta"};
    rowred(b.matrix("sgemv", {0}, {"A"}), 0, "x", "t", K(1));
    out(b.stream("waxpby", {1}, {"t", "y"}), "z", {S("alpha"), S("beta")});
  } else if (seq == "SGEMVT") {
    b.buf("A", m, n, I);
    b.buf("y", 1, m, I, true);
    b.buf("z", 1, n, I);
    b.buf("t", 1, n, T);
    b.buf("x", 1, n, O);
    b.buf("u", 1, m, T, true);
    b.buf("w", 1, m, O, true);
    b.p.scalars = {"alpha", "beta"};
    colred(b.matrix("sgemtv", {0}, {"A"}), 0, "y", "t", K(1));
    out(b.stream("waxpby", {1}, {"t", "z"}), "x", {S("beta"), K(1.0)});
    rowred(b.matrix("sgemv", {2}, {"A"}), 0, "x", "u", K(1));
    out(b.stream("scal", {3}, {"u"}), "w", {S("alpha")});
  } else if (seq == "GEMVER") {
    b.buf("A", m, n, I);
    for (auto nm : {"u1", "u2"}) b.buf(nm, 1, m, I, true);
    for (auto nm : {"v1", "v2"}) b.buf(nm, 1, n, I);
    b.buf("y", 1, m, I, true);
    b.buf("z", 1, n, I);
    b.buf("B", m, n, O);
    b.buf("t", 1, n, T);
    b.buf("x", 1, n, O);
    b.buf("w", 1, m, O, true);
    b.p.scalars = {"alpha", "beta"};
    if (fused) {
      auto& k = b.matrix("gemver_k0[ger2+sgemtv]", {0, 1}, {"A"});
      k.matrix.rank = {{"u1", "v1"}, {"u2", "v2"}};
      k.matrix.store = "B";
      colred(k, 0, "y", "t", K(1));
    } else {
      auto& k = b.matrix("ger2", {0}, {"A"});
      k.matrix.rank = {{"u1", "v1"}, {"u2", "v2"}};
      k.matrix.store = "B";
      colred(b.matrix("sgemtv", {1}, {"B"}), 0, "y", "t", K(1));
    }
    out(b.stream("waxpby", {2}, {"t", "z"}), "x", {S("beta"), K(1.0)});
    rowred(b.matrix("sgemvs", {3}, {"B"}), 0, "x", "w", S("alpha"));
  } else if (seq == "GESUMMV") {
    b.buf("A", m, n, I);
    b.buf("B", m, n, I);
    b.buf("x", 1, n, I);
    b.buf("t1", 1, m, T, true);
    b.buf("t2", 1, m, T, true);
    b.buf("y", 1, m, O, true);
    b.p.scalars = {"alpha", "beta"};
    if (fused) {
      auto& k = b.matrix("gesummv_k0[sgemvs+sgemvs]", {0, 1}, {"A", "B"});
      rowred(k, 0, "x", "t1", S("alpha"));
      rowred(k, 1, "x", "t2", S("beta"));
    } else {
      rowred(b.matrix("sgemvs", {0}, {"A"}), 0, "x", "t1", S("alpha"));
      rowred(b.matrix("sgemvs", {1}, {"B"}), 0, "x", "t2", S("beta"));
    }
    out(b.stream("add", {2}, {"t1", "t2"}), "y", {K(1), K(1)});
  } else {
    throw std::invalid_argument("unknown sequence '" + seq_in + "'");
  }
  return b.p;
}

}  // namespace mapfuse::b200
