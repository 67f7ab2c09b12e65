// mf_jit.cpp -- NVRTC compilation + launch of generic kernels.
//
// host/cudagen.cpp turns a KernelIR into a CUDA C++ translation unit; this
// file compiles it for sm_100a with NVRTC (cubin, no PTX JIT at load time),
// loads it with the runtime's library API and launches it.  Modules are cached
// per (source, poison) for the life of the process, so a plan compiles once
// and every later launch costs one cudaLaunchKernel.  NVRTC is bound with
// dlopen so the engine loads (and every hand-written family runs) even on a
// host without it; the generic path then fails loudly.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "mf_exec.hpp"
#include "mf_jit.hpp"

namespace mapfuse::b200 {

namespace {

struct Nvrtc {
  void* h = nullptr;
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcGetErrorString) errstr = nullptr;
  std::string error;
};

const Nvrtc& nvrtc() {
  static Nvrtc n = [] {
    Nvrtc r;
    for (const char* p : {"/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12", "libnvrtc.so"}) {
      r.h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
      if (r.h) break;
    }
    if (!r.h) {
      r.error = "generic kernels need NVRTC (libnvrtc.so.12): " + std::string(dlerror());
      return r;
    }
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(r.h, name));
      if (!fp && r.error.empty()) r.error = std::string("NVRTC symbol missing: ") + name;
    };
    sym(r.create, "nvrtcCreateProgram");
    sym(r.compile, "nvrtcCompileProgram");
    sym(r.log_size, "nvrtcGetProgramLogSize");
    sym(r.log, "nvrtcGetProgramLog");
    sym(r.cubin_size, "nvrtcGetCUBINSize");
    sym(r.cubin, "nvrtcGetCUBIN");
    sym(r.destroy, "nvrtcDestroyProgram");
    sym(r.errstr, "nvrtcGetErrorString");
    return r;
  }();
  return n;
}

struct Module {
  std::vector<char> cubin;
  std::map<int, std::pair<cudaLibrary_t, cudaKernel_t>> per_device;
  size_t smem_set = 0;
};

std::mutex g_mu;
std::map<std::string, std::shared_ptr<Module>> g_cache;

std::vector<char> compile_cubin(const std::string& src, JitFlags fl, std::string* log_out) {
  const Nvrtc& n = nvrtc();
  if (!n.error.empty()) throw Fault(n.error);
  nvrtcProgram prog = nullptr;
  nvrtcResult rc = n.create(&prog, src.c_str(), "mfj_kernel.cu", 0, nullptr, nullptr);
  if (rc != NVRTC_SUCCESS) throw Fault(std::string("nvrtcCreateProgram: ") + n.errstr(rc));
  const std::string d1 = std::string("-DMFJ_POISON=") + (fl.poison ? "1" : "0");
  const std::string d2 = std::string("-DMFJ_STATS=") + (fl.stats || fl.trace ? "1" : "0");
  const std::string d3 = std::string("-DMFJ_TRACE=") + (fl.trace ? "1" : "0");
  const bool inst = fl.stats || fl.trace;  // instrumented kernels keep the VM's checks and widths
  const std::string d4 = std::string("-DMFJ_CHECKED=") + (fl.unchecked && !inst ? "0" : "1");
  const std::string d5 = std::string("-DMFJ_IDX32=") + (fl.idx32 && fl.unchecked && !inst ? "1" : "0");
  const std::string d6 = std::string("-DMFJ_EXACT=") + (fl.exact && fl.unchecked && !inst ? "1" : "0");
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "-fmad=false",
                        d1.c_str(), d2.c_str(), d3.c_str(), d4.c_str(), d5.c_str(), d6.c_str()};
  rc = n.compile(prog, 10, opts);
  size_t ls = 0;
  n.log_size(prog, &ls);
  std::string log(ls, '\0');
  if (ls) n.log(prog, log.data());
  if (log_out) *log_out = log;
  if (rc != NVRTC_SUCCESS) {
    n.destroy(&prog);
    throw Fault(std::string("NVRTC compile of generic kernel failed: ") + n.errstr(rc) + "\n" + log);
  }
  size_t cs = 0;
  n.cubin_size(prog, &cs);
  std::vector<char> cubin(cs);
  n.cubin(prog, cubin.data());
  n.destroy(&prog);
  return cubin;
}

std::shared_ptr<Module> module_for(const std::string& src, JitFlags fl) {
  const std::string key = std::string(fl.poison ? "P" : "N") + (fl.stats ? "S" : "-") +
                          (fl.trace ? "T" : "-") + (fl.unchecked ? "U" : "-") + (fl.idx32 ? "3" : "-") +
                          (fl.exact ? "E" : "-") + src;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) return it->second;
  }
  auto m = std::make_shared<Module>();
  m->cubin = compile_cubin(src, fl, nullptr);  // outside the lock: NVRTC is slow
  std::lock_guard<std::mutex> lk(g_mu);
  auto [it, inserted] = g_cache.emplace(key, m);
  return it->second;
}

}  // namespace

std::vector<char> jit_compile_only(const std::string& src, JitFlags fl, std::string* log) {
  return compile_cubin(src, fl, log);
}

void jit_prepare(const std::string& src, JitFlags fl) { (void)module_for(src, fl); }

bool jit_available(std::string* why) {
  const Nvrtc& n = nvrtc();
  if (why) *why = n.error;
  return n.error.empty();
}

namespace {
cudaKernel_t kernel_on_device(Module& m) {
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  auto it = m.per_device.find(dev);
  if (it == m.per_device.end()) {
    cudaLibrary_t lib = nullptr;
    check_cuda(cudaLibraryLoadData(&lib, m.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0),
               "cudaLibraryLoadData(generic kernel)");
    cudaKernel_t k = nullptr;
    check_cuda(cudaLibraryGetKernel(&k, lib, "mfj_kernel"), "cudaLibraryGetKernel");
    it = m.per_device.emplace(dev, std::make_pair(lib, k)).first;
  }
  return it->second.second;
}
}  // namespace

void jit_load(const std::string& src, JitFlags fl) {
  std::shared_ptr<Module> m = module_for(src, fl);
  std::lock_guard<std::mutex> lk(g_mu);
  (void)kernel_on_device(*m);
}

void jit_launch(const std::string& src, JitFlags fl, dim3 grid, dim3 block, size_t smem,
                const MfjArgs& args, cudaStream_t stream) {
  std::shared_ptr<Module> m = module_for(src, fl);
  cudaKernel_t fn = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    fn = kernel_on_device(*m);
    if (smem > 48 * 1024 && smem > m->smem_set) {
      check_cuda(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                 "cudaFuncSetAttribute(generic smem)");
      m->smem_set = smem;
    }
  }
  MfjArgs copy = args;
  void* params[] = {&copy};
  check_cuda(cudaLaunchKernel(reinterpret_cast<const void*>(fn), grid, block, params, smem, stream),
             "launch generic kernel");
}

size_t jit_cache_size() {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_cache.size();
}

}  // namespace mapfuse::b200
