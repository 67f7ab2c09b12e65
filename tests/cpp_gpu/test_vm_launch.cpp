// The reference's call site, unchanged in shape: KernelIR + DeviceConfig +
// LaunchArgs{std::vector<float>* buffers} -> vm::launch -- now executing the
// lowered sm_100a kernel on the GPU.  Checked against a plain fp64 loop.
#include <cmath>
#include <cstdio>

#include "doctest.h"
#include "mapfuse/blas.hpp"
#include "mapfuse/planner.hpp"
#include "mapfuse/vm.hpp"

using namespace mapfuse;

TEST_CASE("vm::launch runs the fused BiCGK KernelIR on the B200") {
  const auto& L = blas::default_library();
  auto c = blas::build_sequence("BiCGK");
  auto s = script::parse_script(c.script_text);
  auto g = script::build_dependency_graph(s, L);
  auto k = plan::generate_kernel({0, 1}, s, g, L);
  auto prob = blas::make_problem(s, 200, 300, 42);  // pads to 224 x 320
  vm::LaunchArgs args;
  for (auto& [name, buf] : prob.buffers) {
    auto [r, cc] = prob.dims.at(name);
    args.buffers[name] = vm::GlobalBuffer{r, cc, &buf};
  }
  auto res = vm::launch(k, vm::parse_device_config(blas::default_device_config_text()), args);
  const int m = prob.rows, n = prob.cols;
  CHECK(res.stats.per_buffer.at("A").loaded == uint64_t(m) * n);  // A read once
  CHECK(res.stats.device_ms > 0);
  const auto &A = prob.buffers.at("A"), &p = prob.buffers.at("p"), &r = prob.buffers.at("r");
  const auto &q = prob.buffers.at("q"), &sv = prob.buffers.at("s");
  for (int i = 0; i < m; ++i) {
    double acc = 0, abs_acc = 0;
    for (int j = 0; j < n; ++j) {
      acc += double(A[size_t(i) * n + j]) * p[j];
      abs_acc += std::fabs(double(A[size_t(i) * n + j]) * p[j]);
    }
    CHECK(std::fabs(q[i] - acc) <= std::ldexp(abs_acc, -17) + 1e-30);
  }
  for (int j = 0; j < n; ++j) {
    double acc = 0, abs_acc = 0;
    for (int i = 0; i < m; ++i) {
      acc += double(A[size_t(i) * n + j]) * r[i];
      abs_acc += std::fabs(double(A[size_t(i) * n + j]) * r[i]);
    }
    CHECK(std::fabs(sv[j] - acc) <= std::ldexp(abs_acc, -17) + 1e-30);
  }
}

TEST_CASE("vm::launch faults like the VM on a missing buffer") {
  const auto& L = blas::default_library();
  auto s = script::parse_script(blas::build_sequence("VADD").script_text);
  auto g = script::build_dependency_graph(s, L);
  auto k = plan::generate_kernel({0, 1}, s, g, L);
  auto prob = blas::make_problem(s, 1, 256, 1);
  vm::LaunchArgs args;
  for (auto& [name, buf] : prob.buffers)
    if (name != "z") args.buffers[name] = vm::GlobalBuffer{1, 256, &buf};
  CHECK_THROWS_AS(vm::launch(k, vm::DeviceConfig{}, args), vm::VmFault);
}

TEST_CASE("vm::launch runs a user-manifest fusion no hand-written family covers (generic path)") {
  // tests/golden/generic.mf: mul (element-wise product) fused with add
  std::FILE* f = std::fopen(MF_GENERIC_MF, "rb");
  REQUIRE(f);
  std::string text;
  char buf[4096];
  for (size_t got; (got = std::fread(buf, 1, sizeof buf, f)) > 0;) text.append(buf, got);
  std::fclose(f);
  const auto L = lib::load_library(text);
  auto s = script::parse_script(
      "subvector32 a, b, c, t, o;\ninput a, b, c;\nt = mul(a, b);\no = add(t, c);\nreturn o;\n");
  auto g = script::build_dependency_graph(s, L);
  auto k = plan::generate_kernel({0, 1}, s, g, L);
  const int n = 4096;
  std::vector<float> a(n), b(n), c(n), o(n, -7.f);
  for (int i = 0; i < n; ++i) {
    a[i] = 0.001f * float(i % 997) - 0.5f;
    b[i] = 0.37f - 0.0007f * float(i % 613);
    c[i] = 0.25f * float(i % 5) - 0.5f;
  }
  vm::LaunchArgs args;
  args.buffers["a"] = {1, n, &a};
  args.buffers["b"] = {1, n, &b};
  args.buffers["c"] = {1, n, &c};
  args.buffers["o"] = {1, n, &o};
  auto res = vm::launch(k, vm::parse_device_config(blas::default_device_config_text()), args);
  CHECK(res.stats.native_kernel == "generic");
  int bad = 0;
  for (int i = 0; i < n; ++i) bad += o[i] != a[i] * b[i] + c[i];  // fp32 mul, fp32 add
  CHECK(bad == 0);
}

TEST_CASE("generic vm::launch keeps the VM's accumulate-into-output contract") {
  plan::set_force_generic(true);
  const auto& L = blas::default_library();
  auto s = script::parse_script(blas::build_sequence("AXPYDOT").script_text);
  auto g = script::build_dependency_graph(s, L);
  auto k = plan::generate_kernel({0, 1}, s, g, L);
  auto prob = blas::make_problem(s, 1, 1024, 3);
  vm::LaunchArgs args;
  for (auto& [name, b] : prob.buffers) {
    auto [r, cc] = prob.dims.at(name);
    args.buffers[name] = vm::GlobalBuffer{r, cc, &b};
  }
  for (auto& [name, v] : prob.scalars) args.scalars[name] = v;
  prob.buffers.at("r")[0] = 100.0f;  // the VM adds into it (vm.cpp:283)
  auto res = vm::launch(k, vm::parse_device_config(blas::default_device_config_text()), args);
  plan::set_force_generic(false);
  CHECK(res.stats.native_kernel == "generic");
  const auto &w = prob.buffers.at("w"), &v = prob.buffers.at("v"), &u = prob.buffers.at("u");
  const double alpha = prob.scalars.at("alpha");
  double dot = 0, absdot = 0;
  for (int i = 0; i < 1024; ++i) {
    const float z = w[i] - float(alpha) * v[i];
    dot += double(z) * u[i];
    absdot += std::fabs(double(z) * u[i]);
  }
  CHECK(std::fabs(prob.buffers.at("r")[0] - (100.0 + dot)) <= 1e-5 * (100.0 + absdot));
}
