// ref_shim.cpp -- extern "C" view of the UNMODIFIED reference oracle.
//
// TEST INFRASTRUCTURE ONLY (see mf_oracle.c header).  Compiled together with
// the reference's own sources, read in place from /root/reference/proj/src
// (never copied into this repository), into oracle/_ref/libmapfuse_ref.so by
// oracle/Makefile.  Exposes blas::make_problem (proj/src/blas.cpp:107-139),
// blas::reference_execute (blas.cpp:178-270) and blas::reference_run_script
// (blas.cpp:344-357) through plain C entry points so Python tests, the golden
// fixture generator and bench.py's reference arm can drive the reference
// directly.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "mapfuse/blas.hpp"
#include "mapfuse/device.hpp"
#include "mapfuse/kernel.hpp"
#include "mapfuse/script.hpp"
#include "mapfuse/vm.hpp"

namespace {
thread_local std::string g_err;

struct RefProblem {
  mapfuse::blas::SequenceCase seq;
  mapfuse::script::Script script;
  mapfuse::blas::Problem prob;
  std::map<std::string, std::vector<float>> out;
};
}  // namespace

extern "C" {

const char* mfr_last_error() { return g_err.c_str(); }

// Builds the reference problem for a named Table-1 sequence.
void* mfr_problem_new(const char* seq, int rows, int cols, uint32_t seed) {
  try {
    auto p = std::make_unique<RefProblem>();
    p->seq = mapfuse::blas::build_sequence(seq);
    p->script = mapfuse::script::parse_script(p->seq.script_text);
    p->prob = mapfuse::blas::make_problem(p->script, rows, cols, seed);
    return p.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void mfr_problem_free(void* h) { delete static_cast<RefProblem*>(h); }

int mfr_problem_dims(void* h, int* rows, int* cols) {
  auto* p = static_cast<RefProblem*>(h);
  *rows = p->prob.rows;
  *cols = p->prob.cols;
  return 0;
}

// Copies a buffer (input or zero-filled output) out; returns element count.
long mfr_problem_buffer(void* h, const char* name, float* dst, long cap, int* r, int* c) {
  auto* p = static_cast<RefProblem*>(h);
  auto it = p->prob.buffers.find(name);
  if (it == p->prob.buffers.end()) return -1;
  auto d = p->prob.dims.find(name);
  if (d != p->prob.dims.end()) {
    if (r) *r = d->second.first;
    if (c) *c = d->second.second;
  }
  long n = static_cast<long>(it->second.size());
  if (dst && cap >= n) std::memcpy(dst, it->second.data(), sizeof(float) * n);
  return n;
}

int mfr_problem_scalar(void* h, const char* name, float* v) {
  auto* p = static_cast<RefProblem*>(h);
  auto it = p->prob.scalars.find(name);
  if (it == p->prob.scalars.end()) return -1;
  *v = it->second;
  return 0;
}

// Replaces an input buffer (lets tests feed their own data through the
// reference oracle).
int mfr_problem_set_buffer(void* h, const char* name, const float* src, long n) {
  auto* p = static_cast<RefProblem*>(h);
  auto it = p->prob.buffers.find(name);
  if (it == p->prob.buffers.end() || static_cast<long>(it->second.size()) != n) return -1;
  std::memcpy(it->second.data(), src, sizeof(float) * n);
  return 0;
}

int mfr_problem_set_scalar(void* h, const char* name, float v) {
  auto* p = static_cast<RefProblem*>(h);
  p->prob.scalars[name] = v;
  return 0;
}

// Runs blas::reference_execute; outputs retrievable with mfr_output.
int mfr_execute(void* h) {
  auto* p = static_cast<RefProblem*>(h);
  try {
    p->out = mapfuse::blas::reference_execute(p->seq, p->prob);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Runs blas::reference_run_script with calls in script order (per-call
// narrowing) -- the semantics of an unfused one-kernel-per-call chain.
int mfr_run_script(void* h) {
  auto* p = static_cast<RefProblem*>(h);
  try {
    std::vector<int> order;
    for (const auto& c : p->script.calls) order.push_back(c.id);
    p->out = mapfuse::blas::reference_run_script(p->script, p->prob, order);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

long mfr_output(void* h, const char* name, float* dst, long cap) {
  auto* p = static_cast<RefProblem*>(h);
  auto it = p->out.find(name);
  if (it == p->out.end()) return -1;
  long n = static_cast<long>(it->second.size());
  if (dst && cap >= n) std::memcpy(dst, it->second.data(), sizeof(float) * n);
  return n;
}

// Newline-separated lists for discovery.
int mfr_problem_names(void* h, char* dst, int cap) {
  auto* p = static_cast<RefProblem*>(h);
  std::string s;
  for (const auto& [k, v] : p->prob.buffers) s += "b:" + k + "\n";
  for (const auto& [k, v] : p->prob.scalars) s += "s:" + k + "\n";
  for (const auto& k : p->script.inputs) s += "i:" + k + "\n";
  for (const auto& k : p->script.outputs) s += "o:" + k + "\n";
  if (static_cast<int>(s.size()) + 1 > cap) return -static_cast<int>(s.size() + 1);
  std::memcpy(dst, s.c_str(), s.size() + 1);
  return 0;
}

// Runs the reference's virtual SIMT device, vm::launch (proj/src/vm.cpp:450-479),
// on a KernelIR given in its text form (kernel::parse_kernel_text,
// proj/src/kernel.cpp:178-280), with the default device config
// (blas::default_device_config_text).  Buffers are host arrays updated in
// place, exactly as LaunchArgs binds them (vm.hpp:25-35).  trace != 0 also
// runs the race detector; *hazards receives the hazard count.  Returns 0,
// 1 for a VmFault / parse error (message via mfr_last_error).
int mfr_vm_launch(const char* kernel_text, int nbuf, const char* const* names, const int* rows,
                  const int* cols, float* const* data, int nsc, const char* const* sc_names,
                  const float* sc_values, int poison, int trace, long* hazards,
                  unsigned long long* words_loaded, unsigned long long* words_stored,
                  char* stats_json, int cap) {
  try {
    namespace vm = mapfuse::vm;
    const mapfuse::kernel::KernelIR k = mapfuse::kernel::parse_kernel_text(kernel_text);
    const vm::DeviceConfig dev =
        vm::parse_device_config(mapfuse::blas::default_device_config_text());
    std::vector<std::vector<float>> store(static_cast<size_t>(nbuf));
    vm::LaunchArgs args;
    for (int i = 0; i < nbuf; ++i) {
      const size_t n = static_cast<size_t>(rows[i]) * static_cast<size_t>(cols[i]);
      store[i].assign(data[i], data[i] + n);
      args.buffers[names[i]] = vm::GlobalBuffer{rows[i], cols[i], &store[i]};
    }
    for (int j = 0; j < nsc; ++j) args.scalars[sc_names[j]] = sc_values[j];
    args.poison_onchip = poison != 0;
    args.trace = trace != 0;
    const vm::LaunchResult r = vm::launch(k, dev, args);
    for (int i = 0; i < nbuf; ++i) std::memcpy(data[i], store[i].data(), sizeof(float) * store[i].size());
    if (hazards) *hazards = static_cast<long>(r.races.hazards.size());
    if (words_loaded) *words_loaded = r.stats.global_words_loaded;
    if (words_stored) *words_stored = r.stats.global_words_stored;
    if (stats_json && cap > 0) {
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
      j += "},\"shared_accesses\":" + std::to_string(s.shared_accesses) +
           ",\"atomics\":" + std::to_string(s.atomics) + ",\"barriers\":" + std::to_string(s.barriers) +
           ",\"arith_ops\":" + std::to_string(s.arith_ops) +
           ",\"block_cycles_sum\":" + std::to_string(s.block_cycles_sum) +
           ",\"cycles\":" + std::to_string(s.cycles) + ",\"blocks\":" + std::to_string(s.blocks) +
           ",\"threads_per_block\":" + std::to_string(s.threads_per_block) +
           ",\"shared_bytes\":" + std::to_string(s.shared_bytes) +
           ",\"occupancy\":" + std::to_string(s.occupancy) + ",\"latency_factor\":" + lf +
           ",\"trace_records\":" + std::to_string(r.trace.size()) +
           ",\"hazards\":" + std::to_string(r.races.hazards.size()) + "}";
      std::snprintf(stats_json, static_cast<size_t>(cap), "%s", j.c_str());
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The reference's cost-DB micro-benchmark, vm::measure_routine
// (proj/src/vm.cpp:523-608), for routine `routine_id` (Routine::id()) of a
// function of the shipped library.  Returns cycles, or -1 if infeasible /
// unknown (message via mfr_last_error).
long long mfr_measure_routine(const char* function, const char* routine_id, int instances,
                              int iterations, int extra_shared_bytes) {
  try {
    namespace vm = mapfuse::vm;
    const auto& L = mapfuse::blas::default_library();
    const auto* f = L.find(function);
    if (!f) throw std::runtime_error(std::string("no function ") + function);
    for (const auto& r : f->routines)
      if (r.id() == routine_id) {
        const auto dev = vm::parse_device_config(mapfuse::blas::default_device_config_text());
        auto c = vm::measure_routine(*f, r, vm::MeasureEnv{instances, iterations, extra_shared_bytes}, dev);
        return c ? static_cast<long long>(*c) : -1;
      }
    throw std::runtime_error(std::string("no routine ") + routine_id);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

const char* mfr_manifest() {
  static std::string m = mapfuse::blas::library_manifest();
  return m.c_str();
}

}  // extern "C"
