// host/builtin_data.cpp -- the shipped elementary-function library and the
// Table-1 sequence scripts, generated from compact descriptions.
//
// The reference ships these as data files embedded at configure time
// (proj/data/blas_library.mf, proj/data/scripts/*.mfs,
// proj/CMakeLists.txt:13-33).  Here each function is described once --
// signature, thread shape, and its compute formula -- and the manifest text
// (same DSL, so load_library() parses it like any user manifest) is produced
// by templates for the load / store routines, which are identical for every
// element of a given kind.  Semantics per the paper's Table 1 / Listing 2
// and SPEC.md:604-653.
#include <map>
#include <sstream>
#include <string>
#include <vector>

namespace mapfuse::builtin {

namespace {

struct Elem {
  const char* name;
  const char* kind;    // subvector32 | tile32x32 | scalar
  bool out;
  const char* varies;  // x | y | xy | none
  bool accumulable = false;
};

struct Fn {
  const char* name;
  const char* kind;  // map | map_reduce | map_map
  int depth;
  int max_instances;
  std::vector<const char*> scalars;  // leading scalar params (call order)
  std::vector<Elem> elems;           // args then outs, call order
  std::vector<std::string> compute_maps;
  std::string compute;               // compute routine body
  // scalar position among args: index in `elems` before which each scalar
  // appears (waxpby interleaves alpha x beta y)
  std::vector<int> scalar_before;
};

std::string load_store(const Fn& f, const Elem& e) {
  std::ostringstream o;
  const bool tile = std::string(e.kind) == "tile32x32";
  const bool scalar = std::string(e.kind) == "scalar";
  const std::string n = e.name;
  const char* role = e.out ? "store" : "load";
  o << "  routine " << role << " " << n << " {\n";
  if (tile) {
    o << "    map " << n << ": tx = c, ty = r % BY\n    body {\n"
      << "      for j = 0 .. 32 step BY unroll {\n";
    if (e.out)
      o << "        global " << n << "[ey*32 + ty + j, ex*32 + tx] = onchip " << n << "[ty + j, tx]\n";
    else
      o << "        onchip " << n << "[ty + j, tx] = global " << n << "[ey*32 + ty + j, ex*32 + tx]\n";
    o << "      }\n    }\n  }\n";
    return o.str();
  }
  if (scalar) {  // per-instance partial folded into the global result
    o << "    map " << n << ": tx = 0, ty = 0\n    body {\n      if tx == 0 {\n"
      << "        atomic global " << n << "[0] += onchip " << n << "[0]\n      }\n    }\n  }\n";
    return o.str();
  }
  o << "    map " << n << ": tx = w, ty = 0\n    body {\n";
  const std::string idx = std::string(e.varies) == "y" ? "ey*32 + tx" : "ex*32 + tx";
  std::string stmt;
  if (e.out && e.accumulable) stmt = "atomic global " + n + "[" + idx + "] += onchip " + n + "[tx]";
  else if (e.out) stmt = "global " + n + "[" + idx + "] = onchip " + n + "[tx]";
  else stmt = "onchip " + n + "[tx] = global " + n + "[" + idx + "]";
  if (f.depth == 2) o << "      if ty == 0 {\n        " << stmt << "\n      }\n";
  else o << "      " << stmt << "\n";
  o << "    }\n  }\n";
  return o.str();
}

std::string render(const Fn& f) {
  std::ostringstream o;
  o << "function " << f.name << " {\n  kind " << f.kind << "\n  depth " << f.depth
    << "\n  parallelism 32 " << (f.depth == 2 ? "BY" : "1") << "\n  max_instances "
    << f.max_instances << "\n";
  size_t s = 0;
  for (size_t i = 0; i < f.elems.size(); ++i) {
    while (s < f.scalars.size() && f.scalar_before[s] == static_cast<int>(i))
      o << "  scalar " << f.scalars[s++] << "\n";
    const Elem& e = f.elems[i];
    o << "  " << (e.out ? "out " : "arg ") << e.name << " " << e.kind << " varies " << e.varies
      << (e.accumulable ? " accumulable" : "") << "\n";
  }
  for (const Elem& e : f.elems)
    if (!e.out) o << load_store(f, e);
  o << "  routine compute {\n";
  for (const auto& m : f.compute_maps) o << "    map " << m << "\n";
  o << "    body {\n" << f.compute << "    }\n  }\n";
  for (const Elem& e : f.elems)
    if (e.out) o << load_store(f, e);
  o << "}\n";
  return o.str();
}

const std::string kTileMap = ": tx = c, ty = r % BY";
const std::string kVecMap = ": tx = w, ty = 0";

std::vector<Fn> functions() {
  std::vector<Fn> v;
  auto vec = [](const char* n, bool out = false) { return Elem{n, "subvector32", out, "x"}; };
  // ---- depth-1 maps over 32-word sub-vectors (4 instances per block)
  v.push_back({"add", "map", 1, 4, {}, {vec("a"), vec("b"), vec("c", true)},
               {"a" + kVecMap, "b" + kVecMap, "c" + kVecMap},
               "      onchip c[tx] = onchip a[tx] + onchip b[tx]\n", {}});
  v.push_back({"scal", "map", 1, 4, {"alpha"}, {vec("v"), vec("x", true)},
               {"v" + kVecMap, "x" + kVecMap}, "      onchip x[tx] = alpha*onchip v[tx]\n", {0}});
  v.push_back({"waxpby", "map", 1, 4, {"alpha", "beta"}, {vec("x"), vec("y"), vec("w", true)},
               {"x" + kVecMap, "y" + kVecMap, "w" + kVecMap},
               "      onchip w[tx] = alpha*onchip x[tx] + beta*onchip y[tx]\n", {0, 1}});
  v.push_back({"axpydot_stage", "map", 1, 4, {"alpha"}, {vec("w"), vec("v"), vec("z", true)},
               {"w" + kVecMap, "v" + kVecMap, "z" + kVecMap},
               "      onchip z[tx] = onchip w[tx] - alpha*onchip v[tx]\n", {1}});
  // ---- depth-1 map + reduce: one scalar accumulated across instances
  v.push_back({"dot", "map_reduce", 1, 4, {},
               {vec("x"), vec("y"), Elem{"r", "scalar", true, "none", true}},
               {"x" + kVecMap, "y" + kVecMap, "r: atomic"},
               "      float t = onchip x[tx]*onchip y[tx]\n      atomic onchip r[0] += t\n", {}});
  // ---- depth-2 over 32x32 tiles, one instance per block, 32 x BY threads
  auto tile = [](const char* n, bool out = false) { return Elem{n, "tile32x32", out, "xy"}; };
  v.push_back({"madd", "map_map", 2, 1, {}, {tile("A"), tile("B"), tile("C", true)},
               {"A" + kTileMap, "B" + kTileMap, "C" + kTileMap},
               "      for j = 0 .. 32 step BY unroll {\n"
               "        onchip C[ty + j, tx] = onchip A[ty + j, tx] + onchip B[ty + j, tx]\n"
               "      }\n",
               {}});
  v.push_back({"ger2", "map_map", 2, 1, {},
               {tile("A"), Elem{"u1", "subvector32", false, "y"}, Elem{"v1", "subvector32", false, "x"},
                Elem{"u2", "subvector32", false, "y"}, Elem{"v2", "subvector32", false, "x"},
                tile("B", true)},
               {"A" + kTileMap, "B" + kTileMap, "u1: broadcast", "v1: broadcast", "u2: broadcast",
                "v2: broadcast"},
               "      for j = 0 .. 32 step BY unroll {\n"
               "        onchip B[ty + j, tx] = onchip A[ty + j, tx] + onchip u1[ty + j]*onchip v1[tx]"
               " + onchip u2[ty + j]*onchip v2[tx]\n"
               "      }\n",
               {}});
  // row reduction y[rows] = A x : the compute reads the tile transposed
  // relative to its load (tx walks rows), Listing 2's s_A[tx*33+ty+j]
  const std::string gemv_body =
      "      float tmp = 0.0\n"
      "      for j = 0 .. 32 step BY unroll {\n"
      "        tmp += onchip A[tx, ty + j]*onchip x[ty + j]\n"
      "      }\n";
  v.push_back({"sgemv", "map_reduce", 2, 1, {},
               {tile("A"), vec("x"), Elem{"y", "subvector32", true, "y", true}},
               {"A: tx = r, ty = c % BY", "x: broadcast", "y: atomic"},
               gemv_body + "      atomic onchip y[tx] += tmp\n", {}});
  v.push_back({"sgemvs", "map_reduce", 2, 1, {"alpha"},
               {tile("A"), vec("x"), Elem{"y", "subvector32", true, "y", true}},
               {"A: tx = r, ty = c % BY", "x: broadcast", "y: atomic"},
               gemv_body + "      atomic onchip y[tx] += alpha*tmp\n", {0}});
  // column reduction y[cols] = A^T x : same mapping as the tile load
  v.push_back({"sgemtv", "map_reduce", 2, 1, {},
               {tile("A"), Elem{"x", "subvector32", false, "y"},
                Elem{"y", "subvector32", true, "x", true}},
               {"A" + kTileMap, "x: broadcast", "y: atomic"},
               "      float tmp = 0.0\n"
               "      for j = 0 .. 32 step BY unroll {\n"
               "        tmp += onchip A[ty + j, tx]*onchip x[ty + j]\n"
               "      }\n"
               "      atomic onchip y[tx] += tmp\n",
               {}});
  return v;
}

struct Seq {
  const char* file;
  const char* comment;
  std::vector<std::pair<const char*, std::string>> decls;  // keyword, names
  std::string inputs;
  std::vector<std::string> calls;
  std::string outputs;
};

std::vector<Seq> sequences() {
  return {
      {"atax", "ATAX: y <- A^T A x", {{"TILE32x32", "A"}, {"subvector32", "x, t, y"}}, "A, x",
       {"t = sgemv(A, x)", "y = sgemtv(A, t)"}, "y"},
      {"axpydot", "AXPYDOT: z <- w - alpha*v ; r <- z^T u",
       {{"float", "alpha, r"}, {"subvector32", "w, v, u, z"}}, "w, v, u, alpha",
       {"z = axpydot_stage(w, alpha, v)", "r = dot(z, u)"}, "z, r"},
      {"bicgk", "BiCGK: q <- A p ; s <- A^T r", {{"TILE32x32", "A"}, {"subvector32", "p, q, r, s"}},
       "A, p, r", {"q = sgemv(A, p)", "s = sgemtv(A, r)"}, "q, s"},
      {"gemver", "GEMVER: B <- A + u1 v1^T + u2 v2^T ; x <- beta B^T y + z ; w <- alpha B x",
       {{"TILE32x32", "A, B"}, {"subvector32", "u1, v1, u2, v2, y, z, x, w, t"},
        {"float", "alpha, beta"}},
       "A, u1, v1, u2, v2, y, z, alpha, beta",
       {"B = ger2(A, u1, v1, u2, v2)", "t = sgemtv(B, y)", "x = waxpby(beta, t, 1.0, z)",
        "w = sgemvs(alpha, B, x)"},
       "B, x, w"},
      {"gesummv", "GESUMMV: y <- alpha A x + beta B x",
       {{"TILE32x32", "A, B"}, {"subvector32", "x, t1, t2, y"}, {"float", "alpha, beta"}},
       "A, B, x, alpha, beta",
       {"t1 = sgemvs(alpha, A, x)", "t2 = sgemvs(beta, B, x)", "y = add(t1, t2)"}, "y"},
      {"madd", "MADD: C <- A + B", {{"TILE32x32", "A, B, C"}}, "A, B", {"C = madd(A, B)"}, "C"},
      {"sgemv", "SGEMV: z <- alpha A x + beta y",
       {{"TILE32x32", "A"}, {"subvector32", "x, y, t, z"}, {"float", "alpha, beta"}},
       "A, x, y, alpha, beta", {"t = sgemv(A, x)", "z = waxpby(alpha, t, beta, y)"}, "z"},
      {"sgemvt", "SGEMVT: x <- beta A^T y + z ; w <- alpha A x",
       {{"TILE32x32", "A"}, {"subvector32", "y, z, x, w, t, u"}, {"float", "alpha, beta"}},
       "A, y, z, alpha, beta",
       {"t = sgemtv(A, y)", "x = waxpby(beta, t, 1.0, z)", "u = sgemv(A, x)", "w = scal(alpha, u)"},
       "x, w"},
      {"sscal", "SSCAL: y <- alpha x", {{"subvector32", "x, y"}, {"float", "alpha"}}, "x, alpha",
       {"y = scal(alpha, x)"}, "y"},
      {"vadd", "VADD: x <- w + y + z", {{"subvector32", "w, y, z, t, x"}}, "w, y, z",
       {"t = add(w, y)", "x = add(t, z)"}, "x"},
      {"waxpby", "WAXPBY: w <- alpha x + beta y",
       {{"subvector32", "x, y, t, w"}, {"float", "alpha, beta"}}, "x, y, alpha, beta",
       {"t = scal(alpha, x)", "w = waxpby(1.0, t, beta, y)"}, "w"},
  };
}

}  // namespace

std::string manifest() {
  std::string o =
      "// Built-in elementary-function library (mapfuse-b200): BLAS-1/2 routines\n"
      "// over 32-word sub-vector and 32x32 tile elements.\n";
  for (const auto& f : functions()) o += "\n" + render(f);
  return o;
}

std::map<std::string, std::string> scripts() {
  std::map<std::string, std::string> m;
  for (const auto& s : sequences()) {
    std::ostringstream o;
    o << "// " << s.comment << "\n";
    for (const auto& [kw, names] : s.decls) o << kw << " " << names << ";\n";
    o << "\ninput " << s.inputs << ";\n\n";
    for (const auto& c : s.calls) o << c << ";\n";
    o << "\nreturn " << s.outputs << ";\n";
    m[s.file] = o.str();
  }
  return m;
}

std::string device_config() {
  return "// Virtual-device cost parameters (kept for the reference's DeviceConfig keys;\n"
         "// the B200 cost model uses B200Device + the measured benchmark table).\n"
         "warp_size 32\nmax_threads_per_block 1024\nshared_bytes_per_block 49152\nsm_count 16\n"
         "max_blocks_per_sm 8\ncycles_per_global_word 8\ncycles_per_shared_word 1\n"
         "cycles_per_arith_op 1\ncycles_per_barrier 32\ncycles_per_atomic 4\n"
         "latency_hiding_divisor 4\n";
}

}  // namespace mapfuse::builtin
