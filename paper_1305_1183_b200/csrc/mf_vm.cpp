// mf_vm.cpp -- vm::launch on the B200 (see include/mapfuse/vm.hpp).
#include "mapfuse/vm.hpp"

#include <cuda_runtime.h>

#include "mf_compile.hpp"
#include <algorithm>

#include "mf_exec.hpp"

namespace mapfuse::vm {

LaunchResult launch(const kernel::KernelIR& k, const DeviceConfig& dev, const LaunchArgs& args) {
  // The virtual device's cost parameters do not apply to real hardware; its
  // static limits still reject what the reference rejects (vm.cpp:457-460).
  if (k.threads() > dev.max_threads_per_block)
    throw VmFault("vm fault: block of " + std::to_string(k.threads()) + " threads exceeds device");
  if (k.shared_bytes_total() > dev.shared_bytes_per_block)
    throw VmFault("vm fault: shared allocation exceeds device limit");
  auto dom = args.buffers.find(k.domain);
  if (dom == args.buffers.end()) throw VmFault("launch: domain buffer '" + k.domain + "' is unbound");
  b200::NativePlan plan;
  try {
    plan = b200::plan_from_kernel_text(kernel::emit_pseudo_source(k), dom->second.rows,
                                       dom->second.cols);
  } catch (const std::exception& e) {
    throw VmFault(std::string("launch: ") + e.what());
  }
  // A kernel no hand-written family covers runs on the generic path with the
  // VM's own contract: atomic outputs accumulate onto the caller's values
  // (vm.hpp:91-93) and on-chip memory is poisoned as LaunchArgs asks.
  plan.kernels[0].vm_semantics = true;
  plan.kernels[0].generic_poison = args.poison_onchip ? 1 : 0;
  LaunchResult res;
  b200::Workspace ws;
  try {
    b200::BufMap bufs;
    for (const auto& [name, gb] : args.buffers) {
      if (!gb.data) throw VmFault("launch: buffer '" + name + "' has no storage");
      if (static_cast<int64_t>(gb.data->size()) != static_cast<int64_t>(gb.rows) * gb.cols)
        throw VmFault("launch: buffer '" + name + "' size does not match its shape");
      b200::DevBuf d;
      d.rows = gb.rows;
      d.cols = gb.cols;
      d.ptr = ws.named(name, d.size());
      b200::check_cuda(cudaMemcpy(d.ptr, gb.data->data(), sizeof(float) * d.size(),
                                  cudaMemcpyHostToDevice),
                       "cudaMemcpy H2D");
      bufs[name] = d;
    }
    b200::ScalarMap sc;
    for (const auto& [n, v] : args.scalars) sc[n] = v;
    cudaEvent_t e0, e1;
    b200::check_cuda(cudaEventCreate(&e0), "event");
    b200::check_cuda(cudaEventCreate(&e1), "event");
    cudaEventRecord(e0, nullptr);
    b200::run_kernel(plan, 0, bufs, sc, nullptr, ws);
    cudaEventRecord(e1, nullptr);
    b200::check_cuda(cudaEventSynchronize(e1), "kernel");
    b200::check_jit_faults(ws, nullptr);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    res.stats.device_ms = ms;
    const auto& nk = plan.kernels[0];
    for (const auto& [name, gb] : args.buffers) {
      const auto outs = nk.outputs();
      if (std::find(outs.begin(), outs.end(), name) == outs.end()) continue;
      b200::check_cuda(cudaMemcpy(gb.data->data(), bufs[name].ptr, sizeof(float) * gb.data->size(),
                                  cudaMemcpyDeviceToHost),
                       "cudaMemcpy D2H");
    }
    for (const auto& n : nk.inputs()) {
      auto it = args.buffers.find(n);
      if (it == args.buffers.end()) continue;
      const uint64_t w = static_cast<uint64_t>(it->second.rows) * it->second.cols;
      res.stats.per_buffer[n].loaded += w;
      res.stats.global_words_loaded += w;
    }
    for (const auto& n : nk.outputs()) {
      auto it = args.buffers.find(n);
      if (it == args.buffers.end()) continue;
      const uint64_t w = static_cast<uint64_t>(it->second.rows) * it->second.cols;
      res.stats.per_buffer[n].stored += w;
      res.stats.global_words_stored += w;
    }
    res.stats.native_kernel = nk.kind == b200::NativeKernel::Kind::Matrix
                                  ? "matrix"
                                  : (nk.kind == b200::NativeKernel::Kind::Stream ? "stream" : "generic");
  } catch (const b200::Fault& e) {
    throw VmFault(e.what());
  } catch (const b200::Invalid& e) {
    throw VmFault(e.what());
  }
  return res;
}

}  // namespace mapfuse::vm
