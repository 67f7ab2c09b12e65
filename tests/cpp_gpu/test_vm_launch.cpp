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
