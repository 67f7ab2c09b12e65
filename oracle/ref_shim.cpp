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
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "mapfuse/blas.hpp"
#include "mapfuse/script.hpp"

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

const char* mfr_manifest() {
  static std::string m = mapfuse::blas::library_manifest();
  return m.c_str();
}

}  // extern "C"
