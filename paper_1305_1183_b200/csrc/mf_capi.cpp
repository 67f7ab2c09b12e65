// mf_capi.cpp -- extern "C" surface declared in include/mapfuse_b200.h.
#include "mapfuse_b200.h"

#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <vector>
#include <memory>
#include <string>

#include "mapfuse/blas.hpp"
#include "mapfuse/kernel.hpp"
#include "mapfuse/planner.hpp"
#include "mapfuse/vm.hpp"
#include "mf_builtin.hpp"
#include "mf_compile.hpp"
#include "mf_exec.hpp"
#include "mf_jit.hpp"
#include "mf_kernels.cuh"

using namespace mapfuse::b200;

struct mf_plan {
  NativePlan plan;
  int sms = 0;  // mf_device_desc::sm_count (0 = no per-plan budget)
  // One workspace per stream: launches of one plan on different streams (or
  // from different threads) may overlap on the device, and each needs its own
  // grid-barrier counters, dot ticket, partials and intermediates.  Launches
  // on one stream are ordered by the stream.  Host launches (mf_launch_host,
  // synchronous) use `host_ws`, serialized by `host_mu`.
  mutable std::mutex ws_mu;
  mutable std::map<cudaStream_t, std::unique_ptr<Workspace>> per_stream;
  mutable Workspace host_ws;
  mutable std::mutex host_mu;
  Workspace& ws(cudaStream_t s) const {
    std::lock_guard<std::mutex> lk(ws_mu);
    auto& w = per_stream[s];
    if (!w) w = std::make_unique<Workspace>();
    return *w;
  }
  // implementation generator results per kernel (enumerated on first use)
  mutable std::map<int, std::vector<mapfuse::plan::FusionImplementation>> impls;
  mutable std::mutex impl_mu;
  const std::vector<mapfuse::plan::FusionImplementation>& implementations(int k) const {
    std::lock_guard<std::mutex> lk(impl_mu);
    auto it = impls.find(k);
    if (it == impls.end()) it = impls.emplace(k, mapfuse::plan::kernel_implementations(plan, k)).first;
    return it->second;
  }
};

struct mf_peer_group {
  PeerGroup g;
};

// A plan bound to fixed buffers and scalars: every kernel's host-side work
// (validation, coefficients, grid, workspace) done once; launches replay.
struct mf_bound {
  const mf_plan* plan = nullptr;
  Workspace ws;  // its own scratch: independent of the plan's other launches
  Recorder launches;
  cudaGraphExec_t exec = nullptr;
  ~mf_bound() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return MF_OK;
  } catch (const Invalid& e) {
    g_error = e.what();
    return MF_ERR_INVALID;
  } catch (const Fault& e) {
    g_error = e.what();
    return MF_ERR_FAULT;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return MF_ERR_INVALID;
  } catch (const std::exception& e) {
    g_error = e.what();
    return classify_exception(e);
  } catch (...) {
    g_error = "unknown error";
    return MF_ERR_FAULT;
  }
}

int copy_out(const std::string& s, char* buf, int cap) {
  const int need = (int)s.size() + 1;
  if (buf && cap >= need) std::memcpy(buf, s.c_str(), (size_t)need);
  return need;
}

BufMap to_map(const mf_buffer* b, int n) {
  BufMap m;
  for (int i = 0; i < n; ++i) {
    if (!b[i].name) throw Invalid("buffer without a name");
    DevBuf d;
    d.ptr = b[i].data;
    d.rows = b[i].rows;
    d.cols = b[i].cols;
    m[b[i].name] = d;
  }
  return m;
}

ScalarMap to_scalars(const mf_scalar* s, int n) {
  ScalarMap m;
  for (int i = 0; i < n; ++i) {
    if (!s[i].name) throw Invalid("scalar without a name");
    m[s[i].name] = (double)s[i].value;
  }
  return m;
}

void fill_stats(const NativePlan& p, int k0, int k1, const BufMap& b, mf_stats* st) {
  if (!st) return;
  st->bytes_loaded = 0;
  st->bytes_stored = 0;
  st->kernels = k1 - k0;
  st->ms = 0.0;
  for (int k = k0; k < k1; ++k) {
    const auto& kern = p.kernels[k];
    int64_t m = p.rows, n = p.cols;
    if (kern.kind == NativeKernel::Kind::Generic) {
      auto it = b.find(kern.generic.domain);
      if (it != b.end()) {
        m = kern.generic.depth == 2 ? it->second.rows : 1;
        n = kern.generic.depth == 2 ? it->second.cols : it->second.size();
      }
      st->bytes_loaded += kern.bytes_loaded(m, n);
      st->bytes_stored += kern.bytes_stored(m, n);
    } else if (kern.kind == NativeKernel::Kind::Matrix) {
      auto it = b.find(kern.matrix.mats[0]);
      if (it != b.end()) {
        m = it->second.rows;
        n = it->second.cols;
      }
      st->bytes_loaded += kern.bytes_loaded(m, n);
      st->bytes_stored += kern.bytes_stored(m, n);
    } else {
      auto it = b.find(kern.stream.inputs[0]);
      int64_t len = it != b.end() ? it->second.size() : n;
      st->bytes_loaded += kern.bytes_loaded(1, len);
      st->bytes_stored += kern.bytes_stored(1, len);
    }
  }
}


// Owned CUDA events / streams, released on every exit path (exceptions included).
struct Events {
  std::vector<cudaEvent_t> e;
  explicit Events(int n) {
    for (int i = 0; i < n; ++i) {
      cudaEvent_t x = nullptr;
      check_cuda(cudaEventCreate(&x), "cudaEventCreate");
      e.push_back(x);
    }
  }
  ~Events() {
    for (auto x : e) cudaEventDestroy(x);
  }
  cudaEvent_t& operator[](int i) { return e[(size_t)i]; }
};
struct Streams {
  std::vector<cudaStream_t> s;
  explicit Streams(int n) {
    for (int i = 0; i < n; ++i) {
      cudaStream_t x = nullptr;
      check_cuda(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking), "cudaStreamCreate");
      s.push_back(x);
    }
  }
  ~Streams() {
    for (auto x : s) cudaStreamDestroy(x);
  }
  cudaStream_t operator[](int i) const { return s[(size_t)i]; }
};

// Element-wise plans (only stream kernels, no cross-element reduction, every
// buffer the same length) over PINNED host memory are executed as a
// chunked pipeline: chunk c's H2D copy, kernels and D2H copy are ordered on
// one of three streams, so transfers in both PCIe directions overlap each
// other and the kernels.  Results are identical to the one-shot path (the
// kernels are element-wise).
bool host_pipeline_ok(const NativePlan& P, const mf_buffer* hb, int nbuf) {
  if (nbuf == 0) return false;
  for (const auto& k : P.kernels)
    if (k.kind != NativeKernel::Kind::Stream || k.stream.has_dot) return false;
  const int64_t len = (int64_t)hb[0].rows * hb[0].cols;
  if (len < (int64_t)(8 << 20)) return false;  // small transfers: not worth it
  for (int i = 0; i < nbuf; ++i) {
    if ((int64_t)hb[i].rows * hb[i].cols != len) return false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, hb[i].data) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (at.type != cudaMemoryTypeHost) return false;  // pageable: no async overlap
  }
  return true;
}

double launch_host_pipelined(const mf_plan* plan, const mf_buffer* hb, int nbuf, const BufMap& dev,
                             const ScalarMap& s) {
  const NativePlan& P = plan->plan;
  const int64_t len = (int64_t)hb[0].rows * hb[0].cols;
  const int64_t chunk = std::max<int64_t>(32, (int64_t)(16 << 20) / 32 * 32);  // 64 MB per buffer
  BufMap full = complete_bindings(P, dev, plan->host_ws);
  constexpr int kStreams = 3;
  Streams st(kStreams);
  Events ev(2 + kStreams);  // start, stop, done[i]
  cudaEvent_t start = ev[0], stop = ev[1], *done = &ev[2];
  check_cuda(cudaEventRecord(start, st[0]), "event");
  for (int i = 1; i < kStreams; ++i) check_cuda(cudaStreamWaitEvent(st[i], start, 0), "wait");
  int c = 0;
  for (int64_t off = 0; off < len; off += chunk, ++c) {
    const int64_t n = std::min(chunk, len - off);
    cudaStream_t q = st[c % kStreams];
    BufMap part;
    for (const auto& [name, d] : full) {
      DevBuf x = d;
      x.ptr = d.ptr + off;
      x.rows = 1;
      x.cols = n;
      part[name] = x;
    }
    for (int i = 0; i < nbuf; ++i) {
      const BufferSpec* spec = P.find(hb[i].name);
      if (spec && spec->role != Role::Input) continue;
      check_cuda(cudaMemcpyAsync(part[hb[i].name].ptr, hb[i].data + off, sizeof(float) * n,
                                 cudaMemcpyHostToDevice, q),
                 "H2D");
    }
    for (int k = 0; k < (int)P.kernels.size(); ++k) run_kernel(P, k, part, s, q, plan->host_ws);
    for (int i = 0; i < nbuf; ++i) {
      const BufferSpec* spec = P.find(hb[i].name);
      if (spec && spec->role == Role::Input) continue;
      check_cuda(cudaMemcpyAsync(hb[i].data + off, part[hb[i].name].ptr, sizeof(float) * n,
                                 cudaMemcpyDeviceToHost, q),
                 "D2H");
    }
  }
  for (int i = 1; i < kStreams; ++i) {
    check_cuda(cudaEventRecord(done[i], st[i]), "event");
    check_cuda(cudaStreamWaitEvent(st[0], done[i], 0), "wait");
  }
  check_cuda(cudaEventRecord(stop, st[0]), "event");
  check_cuda(cudaEventSynchronize(stop), "sync");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, start, stop);
  return ms;
}

// NCCL for mf_launch_sharded, resolved at run time from the copy the host
// process already loaded (its communicators must come from the same
// library), else the system libnccl.so.2.  Only the stable C ABI is used:
// ncclAllReduce(sendbuf, recvbuf, count, ncclFloat = 7, ncclSum = 0, comm, stream).
struct NcclApi {
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  const char* (*error_string)(int) = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) {
      r.error = std::string("mf_launch_sharded needs NCCL (libnccl.so.2): ") + dlerror();
      return r;
    }
    r.all_reduce = reinterpret_cast<decltype(r.all_reduce)>(dlsym(h, "ncclAllReduce"));
    r.group_start = reinterpret_cast<decltype(r.group_start)>(dlsym(h, "ncclGroupStart"));
    r.group_end = reinterpret_cast<decltype(r.group_end)>(dlsym(h, "ncclGroupEnd"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!r.all_reduce || !r.group_start || !r.group_end) r.error = "libnccl.so.2 lacks the collective API";
    return r;
  }();
  return api;
}

void check_nccl(int rc, const char* what) {
  if (rc == 0) return;
  const NcclApi& api = nccl();
  throw Fault(std::string(what) + ": NCCL error " + std::to_string(rc) +
              (api.error_string ? std::string(" (") + api.error_string(rc) + ")" : std::string()));
}

}  // namespace

extern "C" {

const char* mf_last_error(void) { return g_error.c_str(); }
const char* mf_version(void) { return "mapfuse-b200 0.1 (sm_100a)"; }

int mf_compile(const char* script_text, const char* manifest, int rows, int cols, int mode,
               mf_plan** out) {
  return guarded([&] {
    if (!script_text || !out) throw Invalid("null argument");
    auto p = std::make_unique<mf_plan>();
    p->plan = compile_script(script_text, manifest ? std::string(manifest) : std::string(), rows,
                             cols, mode);
    *out = p.release();
  });
}

int mf_compile_ranked(const char* script_text, const char* manifest, int rows, int cols, int mode,
                      int rank, mf_plan** out) {
  return guarded([&] {
    if (!script_text || !out) throw Invalid("null argument");
    auto p = std::make_unique<mf_plan>();
    p->plan = compile_script_ranked(script_text, manifest ? std::string(manifest) : std::string(),
                                    rows, cols, mode, rank);
    *out = p.release();
  });
}

int64_t mf_count_combinations(const char* script_text, const char* manifest, int rows, int cols) {
  int64_t n = -1;
  const int rc = guarded([&] {
    if (!script_text) throw Invalid("null argument");
    n = count_script_covers(script_text, manifest ? std::string(manifest) : std::string(), rows, cols);
  });
  return rc == MF_OK ? n : -1;
}

int mf_sequence_script(const char* name, char* buf, int cap) {
  std::string s;
  const int rc = guarded([&] {
    if (!name) throw Invalid("null name");
    s = sequence_script_text(name);
  });
  if (rc != MF_OK) return -1;
  return copy_out(s, buf, cap);
}

double mf_plan_predicted_us(const mf_plan* plan) { return plan ? plan->plan.predicted_us : -1.0; }

int mf_plan_save(const mf_plan* plan, char* buf, int cap) {
  if (!plan) return -1;
  std::string s;
  const int rc = guarded([&] { s = save_plan_text(plan->plan); });
  if (rc != MF_OK) return -1;
  return copy_out(s, buf, cap);
}

int mf_plan_load(const char* text, mf_plan** out) {
  return guarded([&] {
    if (!text || !out) throw Invalid("null argument");
    auto p = std::make_unique<mf_plan>();
    p->plan = load_plan_text(text);
    *out = p.release();
  });
}

int mf_compile_sequence(const char* sequence, int rows, int cols, int mode, mf_plan** out) {
  return guarded([&] {
    if (!sequence || !out) throw Invalid("null argument");
    auto p = std::make_unique<mf_plan>();
    if (mode == 10 || mode == 11)  // hand-derived plans (test cross-check only)
      p->plan = builtin_plan(sequence, rows, cols, mode == 10);
    else
      p->plan = compile_sequence(sequence, rows, cols, mode);
    *out = p.release();
  });
}

int mf_plan_create(const char* kernel_ir_text, int rows, int cols, mf_plan** out) {
  return guarded([&] {
    if (!kernel_ir_text || !out) throw Invalid("null argument");
    auto p = std::make_unique<mf_plan>();
    p->plan = plan_from_kernel_text(kernel_ir_text, rows, cols);
    *out = p.release();
  });
}

int mf_plan_create_desc(const char* kernel_ir_text, const mf_device_desc* desc, mf_plan** out) {
  return guarded([&] {
    if (!kernel_ir_text || !desc || !out) throw Invalid("null argument");
    if (desc->sm_count < 0 || desc->rows < 0 || desc->cols < 0) throw Invalid("negative device description field");
    mapfuse::kernel::KernelIR k;
    mapfuse::vm::DeviceConfig dev;
    try {
      k = mapfuse::kernel::parse_kernel_text(kernel_ir_text);
      dev = mapfuse::vm::parse_device_config(desc->device_config ? std::string(desc->device_config)
                                                                 : mapfuse::blas::default_device_config_text());
    } catch (const std::exception& e) {
      throw Invalid(e.what());
    }
    // the VM's static limits (proj/src/vm.cpp:457-460)
    if (k.threads() > dev.max_threads_per_block)
      throw Fault("vm fault: block of " + std::to_string(k.threads()) + " threads exceeds device");
    if (k.shared_bytes_total() > dev.shared_bytes_per_block)
      throw Fault("vm fault: shared allocation exceeds device limit");
    auto p = std::make_unique<mf_plan>();
    p->plan = plan_from_kernel_text(kernel_ir_text, desc->rows, desc->cols);
    p->sms = desc->sm_count;
    *out = p.release();
  });
}

void mf_plan_destroy(mf_plan* plan) { delete plan; }

int mf_plan_num_kernels(const mf_plan* plan) {
  return plan ? (int)plan->plan.kernels.size() : -1;
}

int mf_plan_describe(const mf_plan* plan, char* buf, int cap) {
  if (!plan) return -1;
  return copy_out(plan->plan.describe_json(), buf, cap);
}

int mf_plan_kernel_text(const mf_plan* plan, int k, char* buf, int cap) {
  if (!plan || k < 0 || k >= (int)plan->plan.kernels.size()) return -1;
  std::string s = k < (int)plan->plan.kernel_ir.size() ? plan->plan.kernel_ir[k] : std::string();
  return copy_out(s, buf, cap);
}

int mf_plan_kernel_column_outputs(const mf_plan* plan, int k, char* buf, int cap) {
  if (!plan || k < 0 || k >= (int)plan->plan.kernels.size()) return -1;
  std::string s;
  for (const auto& n : plan->plan.rank_reductions(k)) s += (s.empty() ? "" : ",") + n;
  return copy_out(s, buf, cap);
}

int mf_launch(const mf_plan* plan, const mf_buffer* buffers, int nbuf, const mf_scalar* scalars,
              int nscalars, void* stream, mf_stats* stats) {
  return guarded([&] {
    PlanSmsScope sms_scope(plan ? plan->sms : 0);  // the plan's SM budget (mf_device_desc)
    if (!plan) throw Invalid("null plan");
    auto st = static_cast<cudaStream_t>(stream);
    Workspace& ws = plan->ws(st);
    BufMap b = complete_bindings(plan->plan, to_map(buffers, nbuf), ws);
    ScalarMap s = to_scalars(scalars, nscalars);
    for (int k = 0; k < (int)plan->plan.kernels.size(); ++k) run_kernel(plan->plan, k, b, s, st, ws);
    fill_stats(plan->plan, 0, (int)plan->plan.kernels.size(), b, stats);
  });
}

int mf_launch_kernel(const mf_plan* plan, int k, const mf_buffer* buffers, int nbuf,
                     const mf_scalar* scalars, int nscalars, void* stream, mf_stats* stats) {
  return guarded([&] {
    PlanSmsScope sms_scope(plan ? plan->sms : 0);  // the plan's SM budget (mf_device_desc)
    if (!plan) throw Invalid("null plan");
    auto st = static_cast<cudaStream_t>(stream);
    Workspace& ws = plan->ws(st);
    BufMap b = complete_bindings(plan->plan, to_map(buffers, nbuf), ws);
    run_kernel(plan->plan, k, b, to_scalars(scalars, nscalars), st, ws);
    fill_stats(plan->plan, k, k + 1, b, stats);
  });
}

int mf_plan_kernel_source(const mf_plan* plan, int k, char* buf, int cap) {
  std::string s;
  const int rc = guarded([&] {
    if (!plan) throw Invalid("null plan");
    if (k < 0 || k >= (int)plan->plan.kernels.size()) throw Invalid("kernel index out of range");
    const auto& kern = plan->plan.kernels[k];
    if (kern.kind == NativeKernel::Kind::Generic) s = kern.generic.source;
  });
  return rc == MF_OK ? copy_out(s, buf, cap) : -rc;
}

int mf_plan_prepare(const mf_plan* plan) {
  return guarded([&] {
    if (!plan) throw Invalid("null plan");
    for (const auto& kern : plan->plan.kernels)
      if (kern.kind == NativeKernel::Kind::Generic) {
        JitFlags fl;
        fl.poison = kern.generic_poison >= 0 ? kern.generic_poison != 0 : options().generic_poison != 0;
        jit_prepare(kern.generic.source, fl);
        fl.unchecked = fl.idx32 = true;  // the variant launches use when the bounds are proved
        jit_prepare(kern.generic.source, fl);
      }
  });
}

int mf_vm_launch(const char* kernel_ir_text, const char* device_config, const mf_buffer* host_buffers,
                 int nbuf, const mf_scalar* scalars, int nscalars, int flags, char* json, int cap) {
  std::string out;
  const int rc = guarded([&] {
    if (!kernel_ir_text) throw Invalid("null kernel text");
    mapfuse::kernel::KernelIR k;
    mapfuse::vm::DeviceConfig dev;
    try {
      k = mapfuse::kernel::parse_kernel_text(kernel_ir_text);
      dev = mapfuse::vm::parse_device_config(device_config ? std::string(device_config)
                                                           : mapfuse::blas::default_device_config_text());
    } catch (const std::exception& e) {
      throw Invalid(e.what());
    }
    std::map<std::string, std::vector<float>> store;
    mapfuse::vm::LaunchArgs args;
    for (int i = 0; i < nbuf; ++i) {
      const mf_buffer& h = host_buffers[i];
      if (!h.name || !h.data) throw Invalid("host buffer without name or data");
      auto& v = store[h.name];
      v.assign(h.data, h.data + (size_t)h.rows * (size_t)h.cols);
      args.buffers[h.name] = mapfuse::vm::GlobalBuffer{h.rows, h.cols, &v};
    }
    for (int i = 0; i < nscalars; ++i) args.scalars[scalars[i].name] = scalars[i].value;
    args.trace = (flags & MF_VM_TRACE) != 0;
    args.poison_onchip = (flags & MF_VM_NO_POISON) == 0;
    mapfuse::vm::LaunchResult r;
    try {
      r = mapfuse::vm::launch(k, dev, args);
    } catch (const mapfuse::vm::VmFault& e) {
      throw Fault(e.what());
    }
    for (int i = 0; i < nbuf; ++i) {
      const auto& v = store[host_buffers[i].name];
      std::memcpy(host_buffers[i].data, v.data(), sizeof(float) * v.size());
    }
    const auto& s = r.stats;
    std::string j = "{\"global_words_loaded\":" + std::to_string(s.global_words_loaded) +
                    ",\"global_words_stored\":" + std::to_string(s.global_words_stored) +
                    ",\"per_buffer\":{";
    bool first = true;
    for (const auto& [n, t] : s.per_buffer) {
      j += std::string(first ? "" : ",") + "\"" + n + "\":[" + std::to_string(t.loaded) + "," +
           std::to_string(t.stored) + "]";
      first = false;
    }
    char lf[64];
    std::snprintf(lf, sizeof lf, "%.17g", s.latency_factor);
    char ms[64];
    std::snprintf(ms, sizeof ms, "%.6f", s.device_ms);
    j += "},\"shared_accesses\":" + std::to_string(s.shared_accesses) +
         ",\"atomics\":" + std::to_string(s.atomics) + ",\"barriers\":" + std::to_string(s.barriers) +
         ",\"arith_ops\":" + std::to_string(s.arith_ops) +
         ",\"block_cycles_sum\":" + std::to_string(s.block_cycles_sum) +
         ",\"cycles\":" + std::to_string(s.cycles) + ",\"blocks\":" + std::to_string(s.blocks) +
         ",\"threads_per_block\":" + std::to_string(s.threads_per_block) +
         ",\"shared_bytes\":" + std::to_string(s.shared_bytes) +
         ",\"occupancy\":" + std::to_string(s.occupancy) + ",\"latency_factor\":" + lf +
         ",\"device_ms\":" + ms + ",\"native_kernel\":\"" + s.native_kernel +
         "\",\"vm_exact\":" + (s.vm_exact ? "true" : "false") +
         ",\"trace_records\":" + std::to_string(r.trace.size()) +
         ",\"hazards\":" + std::to_string(r.races.hazards.size()) + "}";
    out = j;
  });
  if (rc != MF_OK) return -rc;
  return copy_out(out, json, cap);
}

int mf_measure_routine(const char* manifest, const char* function, const char* routine,
                       int instances, int iterations, int extra_shared_bytes,
                       const char* device_config, int64_t* cycles) {
  return guarded([&] {
    if (!function || !routine || !cycles) throw Invalid("null argument");
    mapfuse::lib::Library own;
    const mapfuse::lib::Library* L = &mapfuse::blas::default_library();
    mapfuse::vm::DeviceConfig dev;
    try {
      if (manifest) {
        own = mapfuse::lib::load_library(manifest);
        L = &own;
      }
      dev = mapfuse::vm::parse_device_config(device_config ? std::string(device_config)
                                                           : mapfuse::blas::default_device_config_text());
    } catch (const std::exception& e) {
      throw Invalid(e.what());
    }
    const auto* f = L->find(function);
    if (!f) throw Invalid(std::string("unknown function '") + function + "'");
    for (const auto& r : f->routines)
      if (r.id() == routine) {
        try {
          auto c = mapfuse::vm::measure_routine(
              *f, r, mapfuse::vm::MeasureEnv{instances, iterations, extra_shared_bytes}, dev);
          *cycles = c ? static_cast<int64_t>(*c) : -1;
        } catch (const mapfuse::vm::VmFault& e) {
          throw Fault(e.what());
        }
        return;
      }
    throw Invalid(std::string("unknown routine '") + routine + "' of " + function);
  });
}

int mf_plan_bind(const mf_plan* plan, const mf_buffer* buffers, int nbuf, const mf_scalar* scalars,
                 int nscalars, mf_bound** out) {
  return guarded([&] {
    PlanSmsScope sms_scope(plan ? plan->sms : 0);  // the plan's SM budget (mf_device_desc)
    if (!plan || !out) throw Invalid("null argument");
    auto b = std::make_unique<mf_bound>();
    b->plan = plan;
    BufMap m = complete_bindings(plan->plan, to_map(buffers, nbuf), b->ws);
    const ScalarMap s = to_scalars(scalars, nscalars);
    for (int k = 0; k < (int)plan->plan.kernels.size(); ++k)
      record_kernel(plan->plan, k, m, s, nullptr, b->ws, b->launches);
    check_cuda(cudaDeviceSynchronize(), "bind");  // workspace initialisation done before replays
    *out = b.release();
  });
}

int mf_bound_launch(mf_bound* b, void* stream) {
  return guarded([&] {
    if (!b) throw Invalid("null bound plan");
    for (auto& go : b->launches) check_cuda(go(static_cast<cudaStream_t>(stream)), "bound launch");
  });
}

int mf_bound_graph_launch(mf_bound* b, void* stream) {
  return guarded([&] {
    if (!b) throw Invalid("null bound plan");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!s) throw Invalid("graph launch needs a non-default stream");
    if (!b->exec) {
      cudaGraph_t g = nullptr;
      check_cuda(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
      cudaError_t err = cudaSuccess;
      for (auto& go : b->launches) {
        err = go(s);
        if (err != cudaSuccess) break;
      }
      const cudaError_t end = cudaStreamEndCapture(s, &g);
      check_cuda(err, "capture plan launches");
      check_cuda(end, "end capture");
      const cudaError_t inst = cudaGraphInstantiate(&b->exec, g, 0);
      cudaGraphDestroy(g);
      check_cuda(inst, "instantiate plan graph");
    }
    check_cuda(cudaGraphLaunch(b->exec, s), "graph launch");
  });
}

void mf_bound_destroy(mf_bound* b) { delete b; }

int64_t mf_count_implementation_space(const char* script_text, const char* manifest, int rows,
                                      int cols) {
  int64_t n = -1;
  const int rc = guarded([&] {
    if (!script_text) throw Invalid("null script");
    if (manifest) n = mapfuse::plan::count_implementation_space(script_text, mapfuse::lib::load_library(manifest),
                                                                 rows, cols);
    else n = mapfuse::plan::count_implementation_space(script_text, mapfuse::blas::default_library(), rows, cols);
  });
  return rc == MF_OK ? n : -rc;
}

int64_t mf_plan_count_implementations(const mf_plan* plan, int k) {
  int64_t n = -1;
  const int rc = guarded([&] {
    if (!plan) throw Invalid("null plan");
    n = (int64_t)plan->implementations(k).size();
  });
  return rc == MF_OK ? n : -rc;
}

int mf_plan_implementation(const mf_plan* plan, int k, int index, char* json, int cap) {
  std::string out;
  const int rc = guarded([&] {
    if (!plan) throw Invalid("null plan");
    const auto& impls = plan->implementations(k);
    if (index < 0 || index >= (int)impls.size()) throw Invalid("implementation index out of range");
    const auto& fi = impls[index];
    std::string ord;
    for (size_t i = 0; i < fi.params.order.size(); ++i) ord += (i ? "," : "") + std::to_string(fi.params.order[i]);
    out = "{\"block\":[" + std::to_string(fi.kir.block_x) + "," + std::to_string(fi.kir.block_y) +
          "],\"instances\":" + std::to_string(fi.kir.instances) +
          ",\"iterations\":" + std::to_string(fi.kir.iterations) +
          ",\"overlap\":" + (fi.params.overlap ? "true" : "false") + ",\"order\":[" + ord +
          "],\"shared_bytes\":" + std::to_string(fi.shared_bytes) + "}";
  });
  if (rc != MF_OK) return -rc;
  return copy_out(out, json, cap);
}

int mf_plan_set_implementation(mf_plan* plan, int k, int index) {
  return guarded([&] {
    if (!plan) throw Invalid("null plan");
    const auto& impls = plan->implementations(k);  // enumerated on the plan as compiled
    if (index < 0 || index >= (int)impls.size()) throw Invalid("implementation index out of range");
    mapfuse::plan::set_kernel_implementation(plan->plan, k, impls[index]);
  });
}

int mf_plan_check(const mf_plan* plan, void* stream) {
  return guarded([&] {
    if (!plan) throw Invalid("null plan");
    auto st = static_cast<cudaStream_t>(stream);
    check_jit_faults(plan->ws(st), st);
  });
}

int mf_launch_host(const mf_plan* plan, const mf_buffer* host_buffers, int nbuf,
                   const mf_scalar* scalars, int nscalars, mf_stats* stats) {
  return guarded([&] {
    PlanSmsScope sms_scope(plan ? plan->sms : 0);  // the plan's SM budget (mf_device_desc)
    if (!plan) throw Invalid("null plan");
    const NativePlan& P = plan->plan;
    std::lock_guard<std::mutex> host_lock(plan->host_mu);  // one host launch of a plan at a time
    Workspace& ws = plan->host_ws;
    BufMap dev;
    for (int i = 0; i < nbuf; ++i) {
      const mf_buffer& h = host_buffers[i];
      if (!h.name || !h.data) throw Invalid("host buffer without name or data");
      DevBuf d;
      d.rows = h.rows;
      d.cols = h.cols;
      {
        std::lock_guard<std::mutex> lk(ws.mu);
        d.ptr = ws.named(std::string("__host__") + h.name, (int64_t)h.rows * h.cols);
      }
      dev[h.name] = d;
    }
    ScalarMap s = to_scalars(scalars, nscalars);
    if (host_pipeline_ok(P, host_buffers, nbuf)) {
      const double ms = launch_host_pipelined(plan, host_buffers, nbuf, dev, s);
      fill_stats(P, 0, (int)P.kernels.size(), dev, stats);
      if (stats) stats->ms = ms;
      return;
    }
    cudaStream_t st = nullptr;
    for (int i = 0; i < nbuf; ++i) {
      const mf_buffer& h = host_buffers[i];
      const BufferSpec* spec = P.find(h.name);
      if (spec && spec->role != Role::Input) continue;  // outputs are overwritten
      check_cuda(cudaMemcpyAsync(dev[h.name].ptr, h.data, sizeof(float) * (size_t)h.rows * h.cols,
                                 cudaMemcpyHostToDevice, st),
                 "cudaMemcpy H2D");
    }
    BufMap b = complete_bindings(P, dev, ws);
    Events ev(2);  // destroyed on every exit path
    check_cuda(cudaEventRecord(ev[0], st), "cudaEventRecord");
    for (int k = 0; k < (int)P.kernels.size(); ++k) run_kernel(P, k, b, s, st, ws);
    check_cuda(cudaEventRecord(ev[1], st), "cudaEventRecord");
    for (int i = 0; i < nbuf; ++i) {
      const mf_buffer& h = host_buffers[i];
      const BufferSpec* spec = P.find(h.name);
      if (spec && spec->role == Role::Input) continue;
      check_cuda(cudaMemcpyAsync(h.data, dev[h.name].ptr, sizeof(float) * (size_t)h.rows * h.cols,
                                 cudaMemcpyDeviceToHost, st),
                 "cudaMemcpy D2H");
    }
    check_cuda(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    check_jit_faults(ws, st);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[0], ev[1]);
    fill_stats(P, 0, (int)P.kernels.size(), b, stats);
    if (stats) stats->ms = ms;
  });
}

int mf_peer_group_create(int nranks, int rank, int64_t n_capacity, mf_peer_group** out) {
  return guarded([&] {
    if (!out || nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks || n_capacity <= 0)
      throw Invalid("peer group: bad arguments");
    auto p = std::make_unique<mf_peer_group>();
    PeerGroup& g = p->g;
    g.nranks = nranks;
    g.rank = rank;
    g.n_cap = (n_capacity + 31) / 32 * 32;
    check_cuda(cudaMalloc(&g.inbox, sizeof(float) * 2 * (size_t)nranks * g.n_cap), "cudaMalloc inbox");
    check_cuda(cudaMalloc(&g.outbox, sizeof(float) * 2 * (size_t)g.n_cap), "cudaMalloc outbox");
    check_cuda(cudaMalloc(&g.flags, 64 * sizeof(unsigned)), "cudaMalloc flags");
    check_cuda(cudaMemset(g.flags, 0, 64 * sizeof(unsigned)), "cudaMemset flags");
    g.peer_inbox[rank] = g.inbox;
    g.peer_outbox[rank] = g.outbox;
    g.peer_flags[rank] = g.flags;
    *out = p.release();
  });
}

int mf_peer_group_handle(const mf_peer_group* gp, void* out, int cap) {
  const int need = 3 * (int)sizeof(cudaIpcMemHandle_t);
  if (!gp || !out || cap < need) return need;
  cudaIpcMemHandle_t h[3];
  if (cudaIpcGetMemHandle(&h[0], gp->g.inbox) != cudaSuccess ||
      cudaIpcGetMemHandle(&h[1], gp->g.outbox) != cudaSuccess ||
      cudaIpcGetMemHandle(&h[2], gp->g.flags) != cudaSuccess) {
    g_error = "cudaIpcGetMemHandle failed";
    cudaGetLastError();
    return -1;
  }
  std::memcpy(out, h, need);
  return need;
}

int mf_peer_group_open(mf_peer_group* gp, int peer, const void* handle, int len) {
  return guarded([&] {
    if (!gp || !handle || len != 3 * (int)sizeof(cudaIpcMemHandle_t)) throw Invalid("bad handle");
    PeerGroup& g = gp->g;
    if (peer < 0 || peer >= g.nranks || peer == g.rank) throw Invalid("bad peer index");
    cudaIpcMemHandle_t h[3];
    std::memcpy(h, handle, sizeof h);
    void* p[3] = {};
    for (int i = 0; i < 3; ++i) {
      check_cuda(cudaIpcOpenMemHandle(&p[i], h[i], cudaIpcMemLazyEnablePeerAccess),
                 "cudaIpcOpenMemHandle");
      g.opened.push_back(p[i]);
    }
    g.peer_inbox[peer] = static_cast<float*>(p[0]);
    g.peer_outbox[peer] = static_cast<float*>(p[1]);
    g.peer_flags[peer] = static_cast<unsigned*>(p[2]);
  });
}

int mf_peer_group_connect_local(mf_peer_group* gp, int peer, const mf_peer_group* other) {
  return guarded([&] {
    if (!gp || !other || peer < 0 || peer >= gp->g.nranks) throw Invalid("bad peer");
    gp->g.peer_inbox[peer] = other->g.inbox;
    gp->g.peer_outbox[peer] = other->g.outbox;
    gp->g.peer_flags[peer] = other->g.flags;
  });
}

void mf_peer_group_destroy(mf_peer_group* g) { delete g; }

int mf_peer_group_check(mf_peer_group* gp, void* stream) {
  return guarded([&] {
    if (!gp) throw Invalid("null peer group");
    auto st = static_cast<cudaStream_t>(stream);
    unsigned word = 0;
    PeerGroup& g = gp->g;
    check_cuda(cudaMemcpyAsync(&word, g.flags + kPeerErrorWord, sizeof word, cudaMemcpyDeviceToHost, st),
               "read peer error word");
    check_cuda(cudaStreamSynchronize(st), "peer group check");
    if (word == 0) return;
    check_cuda(cudaMemsetAsync(g.flags + kPeerErrorWord, 0, sizeof word, st), "clear peer error word");
    check_cuda(cudaStreamSynchronize(st), "peer group check");
    throw Fault("in-kernel peer barrier " + std::to_string(word - 1) + " of rank " + std::to_string(g.rank) +
                " timed out: a peer did not arrive within MF_PEER_TIMEOUT_MS (a rank failed or the ranks "
                "launched different kernels); the cross-rank sums of that launch are invalid");
  });
}

int mf_launch_kernel_peers(const mf_plan* plan, int k, mf_peer_group* g, const mf_buffer* buffers,
                           int nbuf, const mf_scalar* scalars, int nscalars, void* stream,
                           mf_stats* stats) {
  return guarded([&] {
    PlanSmsScope sms_scope(plan ? plan->sms : 0);  // the plan's SM budget (mf_device_desc)
    if (!plan) throw Invalid("null plan");
    auto st = static_cast<cudaStream_t>(stream);
    Workspace& ws = plan->ws(st);
    BufMap b = complete_bindings(plan->plan, to_map(buffers, nbuf), ws);
    run_kernel(plan->plan, k, b, to_scalars(scalars, nscalars), st, ws, g ? &g->g : nullptr);
    fill_stats(plan->plan, k, k + 1, b, stats);
  });
}

int mf_launch_peers(const mf_plan* plan, mf_peer_group* g, const mf_buffer* buffers, int nbuf,
                    const mf_scalar* scalars, int nscalars, void* stream, mf_stats* stats) {
  return guarded([&] {
    PlanSmsScope sms_scope(plan ? plan->sms : 0);  // the plan's SM budget (mf_device_desc)
    if (!plan || !g) throw Invalid("null plan or peer group");
    const NativePlan& P = plan->plan;
    for (int i = 0; i < (int)P.kernels.size(); ++i)
      if (const auto& k = P.kernels[i];
          k.kind == NativeKernel::Kind::Generic && !P.rank_reductions(i).empty())
        throw Invalid("kernel " + k.name +
                      ": generic kernels reduce across ranks with a host collective "
                      "(mf_launch_kernel + all-reduce of mf_plan_kernel_column_outputs)");
    auto st = static_cast<cudaStream_t>(stream);
    Workspace& ws = plan->ws(st);
    BufMap b = complete_bindings(P, to_map(buffers, nbuf), ws);
    const ScalarMap s = to_scalars(scalars, nscalars);
    for (int k = 0; k < (int)P.kernels.size(); ++k) run_kernel(P, k, b, s, st, ws, &g->g);
    fill_stats(P, 0, (int)P.kernels.size(), b, stats);
  });
}

int mf_launch_sharded(const mf_plan* const* plans, int ngpus, const int* devices,
                      const mf_buffer* const* per_gpu, const int* nbuf, const mf_scalar* scalars,
                      int nscalars, void* const* comms, void* const* streams, mf_stats* stats) {
  int prev_dev = -1;
  cudaGetDevice(&prev_dev);
  const int rc = guarded([&] {
    if (ngpus < 1 || !plans || !devices || !per_gpu || !nbuf || !comms || !streams)
      throw Invalid("mf_launch_sharded: null argument or ngpus < 1");
    const int nk = (int)plans[0]->plan.kernels.size();
    for (int g = 0; g < ngpus; ++g) {
      if (!plans[g]) throw Invalid("mf_launch_sharded: null plan for GPU " + std::to_string(g));
      bool same = (int)plans[g]->plan.kernels.size() == nk;
      for (int k = 0; same && k < nk; ++k)
        same = plans[g]->plan.kernels[k].calls == plans[0]->plan.kernels[k].calls;
      if (!same)
        throw Invalid("mf_launch_sharded: the per-GPU plans must have the same kernel partition "
                      "(the collectives after each kernel line up)");
    }
    // one GPU with a null communicator: nothing to reduce
    const bool collective = ngpus > 1 || comms[0] != nullptr;
    if (collective) {
      const NcclApi& api = nccl();
      if (!api.error.empty()) throw Fault(api.error);
    }
    const ScalarMap s = to_scalars(scalars, nscalars);
    std::vector<BufMap> b(ngpus);
    for (int g = 0; g < ngpus; ++g) {
      check_cuda(cudaSetDevice(devices[g]), "cudaSetDevice");
      b[g] = complete_bindings(plans[g]->plan, to_map(per_gpu[g], nbuf[g]),
                               plans[g]->ws(static_cast<cudaStream_t>(streams[g])));
    }
    for (int k = 0; k < nk; ++k) {
      for (int g = 0; g < ngpus; ++g) {
        check_cuda(cudaSetDevice(devices[g]), "cudaSetDevice");
        auto st = static_cast<cudaStream_t>(streams[g]);
        PlanSmsScope sms_scope(plans[g]->sms);
        run_kernel(plans[g]->plan, k, b[g], s, st, plans[g]->ws(st));
      }
      // partial column sums / dots of kernel k, summed over the GPUs before
      // any later kernel reads them (the only exchange in a Table-1 plan)
      const auto names = plans[0]->plan.rank_reductions(k);
      if (!collective || names.empty()) continue;
      const NcclApi& api = nccl();
      check_nccl(api.group_start(), "ncclGroupStart");
      for (const auto& name : names)
        for (int g = 0; g < ngpus; ++g) {
          auto it = b[g].find(name);
          if (it == b[g].end() || !it->second.ptr)
            throw Invalid("mf_launch_sharded: GPU " + std::to_string(g) + " has no buffer '" + name + "'");
          check_nccl(api.all_reduce(it->second.ptr, it->second.ptr, (size_t)it->second.size(), 7, 0,
                                    comms[g], static_cast<cudaStream_t>(streams[g])),
                     "ncclAllReduce");
        }
      check_nccl(api.group_end(), "ncclGroupEnd");
    }
    if (stats) {
      mf_stats acc{0, 0, 0.0, 0};
      for (int g = 0; g < ngpus; ++g) {
        mf_stats one{};
        fill_stats(plans[g]->plan, 0, nk, b[g], &one);
        acc.bytes_loaded += one.bytes_loaded;
        acc.bytes_stored += one.bytes_stored;
        acc.kernels += one.kernels;
      }
      *stats = acc;
    }
  });
  if (prev_dev >= 0) cudaSetDevice(prev_dev);
  return rc;
}

int mf_generate(float* dev, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, int64_t row0,
                int64_t ncols_global, void* stream) {
  return guarded([&] {
    if (!dev) throw Invalid("null device pointer");
    check_cuda(launch_generate(dev, rows, cols, ld, seed, row0, ncols_global,
                               static_cast<cudaStream_t>(stream)),
               "generate");
  });
}

int mf_set_option(const char* key, int value) {
  return guarded([&] {
    std::string k = key ? key : "";
    if (k == "matrix_k") {
      if (value != 2 && value != 4) throw Invalid("matrix_k must be 2 or 4");
      options().matrix_k = value;
    } else if (k == "f64acc") {
      options().f64acc = value ? 1 : 0;
    } else if (k == "stream_unroll") {
      if (value != 0 && value != 2 && value != 4 && value != 8) throw Invalid("stream_unroll: 0|2|4|8");
      options().stream_unroll = value;
    } else if (k == "stream_ctas_per_sm") {
      if (value < 0 || value > 8) throw Invalid("stream_ctas_per_sm: 0 (one CTA per block) | 1..8");
      options().stream_ctas_per_sm = value;
    } else if (k == "tma_consumers") {
      if (value != 0 && value != 256 && value != 512) throw Invalid("tma_consumers: 0|256|512");
      options().tma_consumers = value;
    } else if (k == "finalize_group") {
      if (value != 0 && value != 8 && value != 16 && value != 32) throw Invalid("finalize_group: 0 (auto) | 8 | 16 | 32");
      options().finalize_group = value;
    } else if (k == "rowres_l2_ahead") {
      if (value < -1 || value > 8) throw Invalid("rowres_l2_ahead: -1 (auto) .. 8");
      options().rowres_l2_ahead = value;
    } else if (k == "rowres_force_cluster") {
      if (value != 0 && value != 1) throw Invalid("rowres_force_cluster: 0 | 1");
      options().rowres_force_cluster = value;
    } else if (k == "stream_ld_hint") {
      if (value != 0 && value != 1) throw Invalid("stream_ld_hint: 0 | 1");
      options().stream_ld_hint = value;
    } else if (k == "matrix_reverse") {
      if (value < -1 || value > 1) throw Invalid("matrix_reverse: -1 (auto) | 0 | 1");
      options().matrix_reverse = value;
    } else if (k == "matrix_waves") {
      if (value < 1 || value > 16) throw Invalid("matrix_waves: 1 .. 16");
      options().matrix_waves = value;
    } else if (k == "matrix_dynamic") {
      if (value != 0 && value != 1) throw Invalid("matrix_dynamic: 0 | 1");
      options().matrix_dynamic = value;
    } else if (k == "matrix_tile_finalize") {
      if (value < 0 || value > 2) throw Invalid("matrix_tile_finalize: 0 | 1 | 2");
      options().matrix_tile_finalize = value;
    } else if (k == "rowres_variant") {
      if (value < 0 || value > 2) throw Invalid("rowres_variant: 0 (auto) | 1 | 2");
      options().rowres_variant = value;
    } else if (k == "rowres_cluster") {
      if (value < 0 || value > 7) throw Invalid("rowres_cluster: 0 (auto) | 1 .. 7");
      options().rowres_cluster = value;
    } else if (k == "max_sms") {
      if (value < 0) throw Invalid("max_sms >= 0");
      options().max_sms = value;
    } else if (k == "tma_bulk_store") {
      options().tma_bulk_store = value ? 1 : 0;
    } else if (k == "matrix_l2_normal") {
      options().matrix_l2_normal = value < 0 ? -1 : (value ? 1 : 0);
    } else if (k == "tma") {
      options().tma = value < 0 ? -1 : (value ? 1 : 0);
    } else if (k == "occupancy") {
      if (value < 1 || value > 8) throw Invalid("occupancy must be 1..8");
      options().occupancy = value;
    } else if (k == "generic") {
      mapfuse::plan::set_force_generic(value != 0);
    } else if (k == "generic_checked") {
      options().generic_checked = value ? 1 : 0;
    } else if (k == "nvtx") {
      options().nvtx = value ? 1 : 0;
    } else if (k == "vm_exact") {
      mapfuse::vm::set_exact(value != 0);
    } else if (k == "codegen_barriers") {
      mapfuse::plan::set_codegen_barriers(value != 0);
    } else if (k == "generic_by") {
      if (value != 0 && value != 2 && value != 4 && value != 8 && value != 16)
        throw Invalid("generic_by: 0 (default) | 2 | 4 | 8 | 16");
      mapfuse::plan::set_generic_by(value);
    } else if (k == "generic_prefetch") {
      if (value < 0 || value > 8) throw Invalid("generic_prefetch: 0 (auto) .. 8");
      mapfuse::plan::set_generic_prefetch(value);
    } else if (k == "generic_rewrite") {
      if (value < 0 || value > mapfuse::plan::kRwAll) throw Invalid("generic_rewrite: a mask in 0 .. 127");
      mapfuse::plan::set_generic_rewrite(value);
    } else if (k == "generic_iterations") {
      if (value < 0 || value > 4096) throw Invalid("generic_iterations: 0 (auto) .. 4096");
      mapfuse::plan::set_generic_iterations(value);
    } else if (k == "generic_poison") {
      options().generic_poison = value ? 1 : 0;
    } else {
      throw Invalid("unknown option '" + k + "'");
    }
  });
}

int mf_get_option(const char* key) {
  std::string k = key ? key : "";
  if (k == "matrix_k") return options().matrix_k;
  if (k == "f64acc") return options().f64acc;
  if (k == "occupancy") return options().occupancy;
  if (k == "tma") return options().tma;
  if (k == "matrix_l2_normal") return options().matrix_l2_normal;
  if (k == "tma_bulk_store") return options().tma_bulk_store;
  if (k == "max_sms") return options().max_sms;
  if (k == "tma_consumers") return options().tma_consumers;
  if (k == "rowres_cluster") return options().rowres_cluster;
  if (k == "rowres_variant") return options().rowres_variant;
  if (k == "matrix_tile_finalize") return options().matrix_tile_finalize;
  if (k == "matrix_waves") return options().matrix_waves;
  if (k == "matrix_reverse") return options().matrix_reverse;
  if (k == "stream_ld_hint") return options().stream_ld_hint;
  if (k == "rowres_force_cluster") return options().rowres_force_cluster;
  if (k == "rowres_l2_ahead") return options().rowres_l2_ahead;
  if (k == "finalize_group") return options().finalize_group;
  if (k == "matrix_dynamic") return options().matrix_dynamic;
  if (k == "stream_unroll") return options().stream_unroll;
  if (k == "stream_ctas_per_sm") return options().stream_ctas_per_sm;
  if (k == "generic") return mapfuse::plan::force_generic() ? 1 : 0;
  if (k == "generic_poison") return options().generic_poison;
  if (k == "generic_iterations") return mapfuse::plan::generic_iterations();
  if (k == "generic_by") return mapfuse::plan::generic_by();
  if (k == "generic_prefetch") return mapfuse::plan::generic_prefetch();
  if (k == "generic_rewrite") return mapfuse::plan::generic_rewrite();
  if (k == "codegen_barriers") return mapfuse::plan::codegen_barriers() ? 1 : 0;
  if (k == "vm_exact") return mapfuse::vm::exact() ? 1 : 0;
  if (k == "nvtx") return options().nvtx;
  if (k == "generic_checked") return options().generic_checked;
  return -1;
}

}  // extern "C"
