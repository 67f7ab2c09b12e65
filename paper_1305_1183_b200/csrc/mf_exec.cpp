// mf_exec.cpp -- NativeKernel + bound device buffers -> sm_100a launch.
//
// This is the body of the replacement for vm::launch
// (/root/reference/proj/src/vm.cpp:450-479): instead of interpreting routine
// bodies thread by thread, it validates the bindings exactly as strictly as
// the VM (missing buffer / wrong shape -> fault, vm.cpp:77-81, :102-109) and
// hands the kernel's roles to the matching hand-written kernel family.
#include "mf_exec.hpp"

#include <algorithm>
#include <cmath>
#include <functional>
#include <cstring>
#include <sstream>

#include <nvtx3/nvToolsExt.h>

#include "mf_jit.hpp"
#include "mf_kernels.cuh"

namespace mapfuse::b200 {

EngineOptions& options() {
  static EngineOptions o = [] {
    EngineOptions e;
    if (const char* v = std::getenv("MF_MATRIX_K")) e.matrix_k = std::atoi(v);
    if (const char* v = std::getenv("MF_F64ACC")) e.f64acc = std::atoi(v);
    if (const char* v = std::getenv("MF_OCCUPANCY")) e.occupancy = std::atoi(v);
    if (const char* v = std::getenv("MF_TMA")) e.tma = std::atoi(v);
    if (const char* v = std::getenv("MF_STREAM_UNROLL")) e.stream_unroll = std::atoi(v);
    if (const char* v = std::getenv("MF_STREAM_CTAS")) e.stream_ctas_per_sm = std::atoi(v);
    if (const char* v = std::getenv("MF_MATRIX_L2_NORMAL")) e.matrix_l2_normal = std::atoi(v);
    if (const char* v = std::getenv("MF_TMA_BULK_STORE")) e.tma_bulk_store = std::atoi(v);
    if (const char* v = std::getenv("MF_MAX_SMS")) e.max_sms = std::atoi(v);
    if (const char* v = std::getenv("MF_TMA_CONSUMERS")) e.tma_consumers = std::atoi(v);
    if (const char* v = std::getenv("MF_GENERIC_POISON")) e.generic_poison = std::atoi(v);
    if (const char* v = std::getenv("MF_NVTX")) e.nvtx = std::atoi(v);
    if (const char* v = std::getenv("MF_GENERIC_CHECKED")) e.generic_checked = std::atoi(v);
    if (const char* v = std::getenv("MF_ROWRES_CLUSTER")) e.rowres_cluster = std::atoi(v);
    if (const char* v = std::getenv("MF_ROWRES_VARIANT")) e.rowres_variant = std::atoi(v);
    if (const char* v = std::getenv("MF_MATRIX_TILE_FINALIZE")) e.matrix_tile_finalize = std::atoi(v);
    return e;
  }();
  return o;
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Fault(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                ")");
}

namespace {
thread_local int t_plan_sms = 0;
}
PlanSmsScope::PlanSmsScope(int cap) : saved(t_plan_sms) { t_plan_sms = cap; }
PlanSmsScope::~PlanSmsScope() { t_plan_sms = saved; }

int device_sm_count();
int effective_sms() {
  int s = device_sm_count();
  if (options().max_sms > 0) s = std::min(s, options().max_sms);
  if (t_plan_sms > 0) s = std::min(s, t_plan_sms);
  return s;
}

int device_sm_count() {
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int sms = 0;
  check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev),
             "cudaDeviceGetAttribute");
  cache[dev] = sms;
  return sms;
}

// ---------------------------------------------------------------------------
Workspace::~Workspace() {
  // Best effort: the process may be tearing down the CUDA context already.
  for (void* p : retired_) cudaFree(p);
  if (scratch_) cudaFree(scratch_);
  if (counters_) cudaFree(counters_);
  if (tile_) cudaFree(tile_);
  if (jit_fault_) cudaFree(jit_fault_);
  for (auto& [k, v] : named_) cudaFree(v.first);
}

// Growing never frees the old buffer: launches already enqueued (or recorded
// by a bound plan / captured into a graph) keep the pointer they were given,
// so it stays valid until the workspace dies.  Doubling bounds the retired
// total below the live buffer's size.
void* Workspace::scratch(size_t bytes, cudaStream_t) {
  if (bytes <= scratch_bytes_) return scratch_;
  if (scratch_) retired_.push_back(scratch_);
  size_t want = std::max(bytes, scratch_bytes_ * 2);
  check_cuda(cudaMalloc(&scratch_, want), "cudaMalloc(workspace)");
  scratch_bytes_ = want;
  return scratch_;
}

unsigned* Workspace::counters(cudaStream_t s) {
  if (!counters_) {
    check_cuda(cudaMalloc(&counters_, 64 * sizeof(unsigned)), "cudaMalloc(counters)");
    check_cuda(cudaMemsetAsync(counters_, 0, 64 * sizeof(unsigned), s), "cudaMemset(counters)");
  }
  return counters_;
}

// Same growth rule as scratch(): launches already enqueued or recorded keep
// the counters they were given.  Zeroed on allocation; kernels leave them 0.
unsigned* Workspace::tile_counters(size_t words, cudaStream_t s) {
  if (words <= tile_words_) return tile_;
  if (tile_) retired_.push_back(tile_);
  const size_t want = std::max(words, std::max<size_t>(256, tile_words_ * 2));
  check_cuda(cudaMalloc(&tile_, want * sizeof(unsigned)), "cudaMalloc(tile counters)");
  check_cuda(cudaMemsetAsync(tile_, 0, want * sizeof(unsigned), s), "cudaMemset(tile counters)");
  tile_words_ = want;
  return tile_;
}

unsigned* Workspace::jit_fault(cudaStream_t s) {
  if (!jit_fault_) {
    check_cuda(cudaMalloc(&jit_fault_, 2 * sizeof(unsigned)), "cudaMalloc(jit fault)");
    check_cuda(cudaMemsetAsync(jit_fault_, 0, 2 * sizeof(unsigned), s), "cudaMemset(jit fault)");
  }
  return jit_fault_;
}

float* Workspace::named(const std::string& key, int64_t words) {
  auto it = named_.find(key);
  if (it != named_.end() && it->second.second >= words) return it->second.first;
  if (it != named_.end()) {  // retired, not freed (see scratch())
    retired_.push_back(it->second.first);
    named_.erase(it);
  }
  float* p = nullptr;
  check_cuda(cudaMalloc(&p, std::max<int64_t>(words, 32) * sizeof(float)), "cudaMalloc(named)");
  named_[key] = {p, words};
  return p;
}

PeerGroup::~PeerGroup() {
  for (void* p : opened) cudaIpcCloseMemHandle(p);
  if (inbox) cudaFree(inbox);
  if (outbox) cudaFree(outbox);
  if (flags) cudaFree(flags);
}

// ---------------------------------------------------------------------------
namespace {

const DevBuf& need(const BufMap& bufs, const std::string& name, const std::string& kname) {
  auto it = bufs.find(name);
  if (it == bufs.end() || (!it->second.ptr && it->second.size() != 0))  // empty buffers may be null
    throw Fault("kernel " + kname + ": unbound buffer '" + name + "'");
  if ((reinterpret_cast<uintptr_t>(it->second.ptr) & 15u) != 0)
    throw Fault("kernel " + kname + ": buffer '" + name + "' is not 16-byte aligned");
  return it->second;
}

void need_len(const DevBuf& b, int64_t len, const std::string& name, const std::string& kname) {
  if (b.size() != len) {
    std::ostringstream os;
    os << "kernel " << kname << ": buffer '" << name << "' has " << b.size()
       << " words, expected " << len;
    throw Fault(os.str());
  }
}

double coef(const Coef& c, const ScalarMap& s, const std::string& kname) {
  try {
    return c.eval(s);
  } catch (const std::exception& e) {
    throw Fault("kernel " + kname + ": " + e.what());
  }
}

// Every run_* prepares a kernel's arguments (validation, coefficients,
// grid, workspace) and then either launches it on `s` or, with `rec`, stores
// the launch for later replay (bound plans, CUDA graph capture).
void emit(Recorder* rec, const std::string& what, std::function<cudaError_t(cudaStream_t)> go,
          cudaStream_t s) {
  if (rec) rec->push_back(std::move(go));
  else check_cuda(go(s), what.c_str());
}

template <typename Args>
void fill_peers(Args& a, PeerGroup* peers, int64_t n, const std::string& kname);

// MF_PEER_TIMEOUT_MS (default 10000): how long an in-kernel peer barrier
// waits for the other ranks before it gives up and flags the group.
long long peer_timeout_ms() {
  static const long long v = [] {
    const char* e = std::getenv("MF_PEER_TIMEOUT_MS");
    return e ? std::max(1LL, std::atoll(e)) : 10000LL;
  }();
  return v;
}

void run_stream(const NativeKernel& k, const BufMap& bufs, const ScalarMap& sc, cudaStream_t s,
                Workspace& ws, Recorder* rec, PeerGroup* peers = nullptr) {
  const StreamOp& op = k.stream;
  const int nin = (int)op.inputs.size(), nout = (int)op.outs.size();
  if (nin < 1 || nin > kStreamMaxIn || nout > kStreamMaxOut)
    throw Invalid("kernel " + k.name + ": unsupported stream shape");
  const DevBuf& first = need(bufs, op.inputs[0], k.name);
  const int64_t n = first.size();
  if (n % 4) throw Fault("kernel " + k.name + ": stream length must be a multiple of 4 (padded)");
  StreamArgs a;
  a.n4 = n / 4;
  a.ld_hint = options().stream_ld_hint;
  for (int i = 0; i < nin; ++i) {
    const DevBuf& b = need(bufs, op.inputs[i], k.name);
    need_len(b, n, op.inputs[i], k.name);
    a.in[i] = reinterpret_cast<const float4*>(b.ptr);
  }
  for (int q = 0; q < nout; ++q) {
    const DevBuf& b = need(bufs, op.outs[q].name, k.name);
    need_len(b, n, op.outs[q].name, k.name);
    a.out[q] = reinterpret_cast<float4*>(b.ptr);
    for (int i = 0; i < nin; ++i) a.coef[q][i] = coef(op.outs[q].coef[i], sc, k.name);
  }
  const int sms = device_sm_count();
  const int grid = stream_grid(a.n4, sms, options().stream_ctas_per_sm, nin, options().stream_unroll,
                               op.has_dot);
  if (op.has_dot) {
    const DevBuf& r = need(bufs, op.dot_out, k.name);
    if (r.size() < 1) throw Fault("kernel " + k.name + ": empty dot output");
    a.r = r.ptr;
    for (int i = 0; i < nin; ++i) {
      a.da[i] = coef(op.dot_a[i], sc, k.name);
      a.db[i] = coef(op.dot_b[i], sc, k.name);
    }
    a.part = static_cast<double*>(ws.scratch(sizeof(double) * (size_t)grid, s));
    a.ticket = ws.counters(s) + 2;
    // dot partials reduced across ranks in-kernel; an empty shard still
    // launches (its partial is 0) so every rank arrives at the peer barrier
    // and the group's epochs stay in step
    fill_peers(a, peers, 1, k.name);
  }
  if (n == 0 && !(op.has_dot && a.peer.nranks > 1)) {
    // an empty dot is 0 (the reference sums nothing into a zeroed output)
    if (op.has_dot) {
      float* r = a.r;
      emit(rec, "zero " + k.name, [=](cudaStream_t st) { return cudaMemsetAsync(r, 0, sizeof(float), st); },
           s);
    }
    return;
  }
  const int unroll = options().stream_unroll;
  const bool dot = op.has_dot;
  emit(rec, "launch " + k.name,
       [=](cudaStream_t st) { return launch_stream(nin, nout, dot, a, grid, unroll, st); }, s);
}

template <typename Args>
void fill_peers(Args& a, PeerGroup* peers, int64_t n, const std::string& kname) {
  if (!peers || peers->nranks <= 1) return;
  if (n > peers->n_cap) throw Fault("kernel " + kname + ": peer group capacity below n");
  a.peer.nranks = peers->nranks;
  a.peer.rank = peers->rank;
  a.peer.n_cap = peers->n_cap;
  for (int r = 0; r < peers->nranks; ++r) {
    if (!peers->peer_inbox[r] || !peers->peer_flags[r] || !peers->peer_outbox[r])
      throw Fault("kernel " + kname + ": peer " + std::to_string(r) + " not connected");
    a.peer.inbox[r] = peers->peer_inbox[r];
    a.peer.outbox[r] = peers->peer_outbox[r];
    a.peer.flags[r] = peers->peer_flags[r];
  }
  a.peer.epoch = ++peers->epoch;
  a.peer.timeout_ns = peer_timeout_ms() * 1000000LL;  // bounded peer barriers
}

// An empty matrix (m or n = 0): every reduction over the empty dimension is 0.
void zero_outputs(const NativeKernel& k, const BufMap& bufs, cudaStream_t s, Recorder* rec) {
  for (const auto& name : k.outputs()) {
    auto it = bufs.find(name);
    if (it == bufs.end() || it->second.size() == 0) continue;
    float* p = it->second.ptr;
    const size_t bytes = sizeof(float) * (size_t)it->second.size();
    emit(rec, "zero " + name, [=](cudaStream_t st) { return cudaMemsetAsync(p, 0, bytes, st); }, s);
  }
}

// Row-resident chain: t = a*A x (optionally stored), y = b*A^T t, one pass.
void run_rowres(const NativeKernel& k, const BufMap& bufs, const ScalarMap& sc, cudaStream_t s,
                Workspace& ws, PeerGroup* peers, Recorder* rec) {
  const MatrixOp& op = k.matrix;
  if (op.mats.size() != 1 || op.rows.size() != 1 || op.cols.size() != 1 || !op.rank.empty())
    throw Invalid("kernel " + k.name + ": malformed row-resident chain");
  const DevBuf& M = need(bufs, op.mats[0], k.name);
  const int64_t m = M.rows, n = M.cols;
  if (n > rowres_cluster_max_cols())
    throw Fault("kernel " + k.name + ": row-resident chain needs n <= " +
                std::to_string(rowres_cluster_max_cols()) + " (got " + std::to_string(n) + ")");
  if (m % 32 || n % 32)
    throw Fault("kernel " + k.name + ": matrix dims must be padded to multiples of 32 (got " +
                std::to_string(m) + "x" + std::to_string(n) + ")");
  MatrixArgs a;
  a.m = m;
  a.n = n;
  a.ld = n;
  a.M[0] = M.ptr;
  const DevBuf& x = need(bufs, op.rows[0].x, k.name);
  need_len(x, n, op.rows[0].x, k.name);
  a.xr[0] = x.ptr;
  a.ar[0] = coef(op.rows[0].coef, sc, k.name);
  if (!op.rows[0].y.empty()) {
    const DevBuf& t = need(bufs, op.rows[0].y, k.name);
    need_len(t, m, op.rows[0].y, k.name);
    a.yr[0] = t.ptr;
  }
  const DevBuf& y = need(bufs, op.cols[0].y, k.name);
  need_len(y, n, op.cols[0].y, k.name);
  a.yc[0] = y.ptr;
  a.ac[0] = coef(op.cols[0].coef, sc, k.name);
  if (m == 0 || n == 0) return zero_outputs(k, bufs, s, rec);
  const EngineOptions& eo = options();
  const int sms = effective_sms();
  int grid = 0;
  a.fin_g = eo.finalize_group;
  if (n > rowres_max_cols() || eo.rowres_force_cluster) {  // wide rows: a CTA cluster per row (DSMEM)
    const int variant = n > rowres_max_cols() || eo.rowres_cluster ? rowres_cluster_variant(eo.rowres_cluster, n)
                                                                   : 7;
    const int bands = rowres_cluster_bands(m, n, sms, variant);
    if (bands <= 0) throw Fault("kernel " + k.name + ": no co-resident CTA cluster for n = " + std::to_string(n));
    a.CB = 1;
    a.RB = bands;
    a.tiles = bands;
    a.colpart = ws.scratch(sizeof(float) * (size_t)a.RB * (size_t)n + 256, s);
    a.bar = ws.counters(s);
    fill_peers(a, peers, n, k.name);
    emit(rec, "launch " + k.name,
         [=](cudaStream_t st) { return launch_rowres_cluster(a, variant, sms, st); }, s);
    return;
  }
  const int variant = rowres_variant(eo.rowres_variant, n);
  a.l2_ahead = eo.rowres_l2_ahead < 0 ? 0 : eo.rowres_l2_ahead;
  check_cuda(rowres_config(m, n, sms, variant, &a, &grid), ("configure " + k.name).c_str());
  a.colpart = ws.scratch(sizeof(float) * (size_t)a.RB * (size_t)n + 256, s);
  a.bar = ws.counters(s);
  fill_peers(a, peers, n, k.name);
  emit(rec, "launch " + k.name, [=](cudaStream_t st) { return launch_rowres(a, grid, variant, st); }, s);
}

void run_matrix(const NativeKernel& k, const BufMap& bufs, const ScalarMap& sc, cudaStream_t s,
                Workspace& ws, PeerGroup* peers, Recorder* rec, bool after_store = false) {
  const MatrixOp& op = k.matrix;
  if (op.chain) return run_rowres(k, bufs, sc, s, ws, peers, rec);
  MatrixShape sh{(int)op.mats.size(), (int)op.rank.size(), op.store.empty() ? 0 : 1,
                 (int)op.rows.size(), (int)op.cols.size()};
  if (!matrix_shape_supported(sh))
    throw Invalid("kernel " + k.name + ": no sm_100a template for this matrix fusion shape");
  const DevBuf& M0 = need(bufs, op.mats[0], k.name);
  const int64_t m = M0.rows, n = M0.cols;
  // the cross-CTA finalize maps 8-lane groups onto float4 slots and assumes
  // whole 32-column groups (the reference pads every buffer to 32,
  // proj/include/mapfuse/blas.hpp:29-30)
  if (m % 32 || n % 32)
    throw Fault("kernel " + k.name + ": matrix dims must be padded to multiples of 32 (got " +
                std::to_string(m) + "x" + std::to_string(n) + ")");
  MatrixArgs a;
  a.m = m;
  a.n = n;
  a.ld = n;
  for (size_t i = 0; i < op.mats.size(); ++i) {
    const DevBuf& b = need(bufs, op.mats[i], k.name);
    if (b.rows != m || b.cols != n) throw Fault("kernel " + k.name + ": matrix shape mismatch");
    a.M[i] = b.ptr;
  }
  for (size_t q = 0; q < op.rank.size(); ++q) {
    const DevBuf& u = need(bufs, op.rank[q].first, k.name);
    const DevBuf& v = need(bufs, op.rank[q].second, k.name);
    need_len(u, m, op.rank[q].first, k.name);
    need_len(v, n, op.rank[q].second, k.name);
    a.u[q] = u.ptr;
    a.v[q] = v.ptr;
  }
  if (!op.store.empty()) {
    const DevBuf& e = need(bufs, op.store, k.name);
    if (e.rows != m || e.cols != n) throw Fault("kernel " + k.name + ": store shape mismatch");
    a.E = e.ptr;
  }
  for (size_t o = 0; o < op.rows.size(); ++o) {
    const DevBuf& x = need(bufs, op.rows[o].x, k.name);
    const DevBuf& y = need(bufs, op.rows[o].y, k.name);
    need_len(x, n, op.rows[o].x, k.name);
    need_len(y, m, op.rows[o].y, k.name);
    a.xr[o] = x.ptr;
    a.yr[o] = y.ptr;
    a.ar[o] = coef(op.rows[o].coef, sc, k.name);
  }
  for (size_t c = 0; c < op.cols.size(); ++c) {
    const DevBuf& x = need(bufs, op.cols[c].x, k.name);
    const DevBuf& y = need(bufs, op.cols[c].y, k.name);
    need_len(x, m, op.cols[c].x, k.name);
    need_len(y, n, op.cols[c].y, k.name);
    a.xc[c] = x.ptr;
    a.yc[c] = y.ptr;
    a.ac[c] = coef(op.cols[c].coef, sc, k.name);
  }
  if (m == 0 || n == 0) return zero_outputs(k, bufs, s, rec);
  MatrixTuning t;
  const EngineOptions& eo = options();
  t.K = eo.matrix_k == 4 ? 4 : 2;
  t.f64acc = eo.f64acc != 0;
  t.occupancy = std::max(1, eo.occupancy);
  t.waves = std::max(1, eo.matrix_waves);
  t.dynamic = eo.matrix_dynamic != 0;
  // Variant choice (the implementation generator's role):
  // shapes that stream a matrix back out (ger2's B) or carry the rank-2
  // update need the deep TMA ring to keep enough bytes in flight; read-only
  // reduction shapes reach roofline from registers alone (measured on B200,
  // profiles/r01_sweep_initial.txt, r01_matrix_layout.txt).  tma = -1 auto, 0 register-fed, 1 TMA.
  const bool heavy = sh.nrank > 0 || sh.store;
  if (eo.tma < 0 && k.variant_tma >= 0) {  // the cost model's choice
    t.tma = k.variant_tma == 1;
    if (k.variant_k == 2 || k.variant_k == 4) t.K = k.variant_k;
  } else {
    t.tma = eo.tma < 0 ? heavy : eo.tma != 0;
    if (t.tma && eo.tma < 0 && eo.matrix_k == 2) t.K = 4;
  }
  // 16 consumer warps for the store-heavy rank shape (measured +2.3% on
  // GEMVER 32768^2, tools/sweep.py); 8 elsewhere.  tma_consumers 0 = auto.
  if (t.tma) t.consumers = eo.tma_consumers == 0 ? (heavy ? 512 : 256) : eo.tma_consumers;
  t.bulk_store = sh.store && eo.tma_bulk_store != 0;
  if (t.tma && !tma_supported(sh, t)) t.tma = false;
  int grid = 0;
  const int sms = effective_sms();
  a.l2_normal = eo.matrix_l2_normal < 0 ? (sh.store ? 1 : 0) : eo.matrix_l2_normal;
  if (t.tma)
    check_cuda(matrix_tma_config(sh, t, m, n, sms, &a, &grid), ("configure " + k.name).c_str());
  else
    check_cuda(matrix_config(sh, t, m, n, sms, &a, &grid), ("configure " + k.name).c_str());
  if (sh.ncol > 0) fill_peers(a, peers, n, k.name);
  const size_t acc = matrix_acc_bytes(t);
  const size_t colb = acc * (size_t)sh.ncol * (size_t)a.RB * (size_t)n;
  const size_t rowb = (a.CB > 1) ? acc * (size_t)sh.nrow * (size_t)a.CB * (size_t)m : 0;
  char* base = static_cast<char*>(ws.scratch(colb + rowb + 256, s));
  a.colpart = base;
  a.rowpart = base + ((colb + 255) & ~size_t(255));
  a.bar = ws.counters(s);
  // tile-completion finalize: column partials summed in groups of ~sqrt(RB)
  // row bands, then over the groups (mf_device.cuh tile_done)
  a.G = std::max(1, (int)std::ceil(std::sqrt((double)a.RB)));
  a.NG = (a.RB + a.G - 1) / a.G;
  a.tilecnt = ws.tile_counters((size_t)a.CB * a.NG + a.CB + a.RB, s);
  a.tile_fin = eo.matrix_tile_finalize;
  // row batches bottom-up when an earlier kernel of the plan stored this
  // matrix: its last-written rows are still in L2 (GEMVER's w = alpha B x
  // after B = A + u1 v1^T + u2 v2^T: 615 -> 607 us at 32768^2)
  a.rev = eo.matrix_reverse < 0 ? (after_store ? 1 : 0) : eo.matrix_reverse;
  a.fin_g = eo.finalize_group;
  if (t.tma)
    emit(rec, "launch " + k.name, [=](cudaStream_t st) { return launch_matrix_tma(sh, t, a, grid, st); }, s);
  else
    emit(rec, "launch " + k.name, [=](cudaStream_t st) { return launch_matrix(sh, t, a, grid, st); }, s);
}

// Generic kernel: one CTA per VM block over the grid the domain buffer
// implies (proj/src/vm.cpp:24-47, :450-466); see host/cudagen.cpp.
struct GenericLaunch {
  MfjArgs a{};
  int64_t launch_x = 0, launch_y = 1;
  size_t smem = 0;
};

// Grid (vm.cpp:24-47), bindings and scalars of a generic kernel.
GenericLaunch generic_args(const NativeKernel& k, const BufMap& bufs, const ScalarMap& sc,
                           cudaStream_t s, Workspace& ws) {
  const GenericOp& g = k.generic;
  auto dom = bufs.find(g.domain);
  if (dom == bufs.end() || !dom->second.ptr)
    throw Fault("launch: no domain buffer '" + g.domain + "'");
  const int64_t rows = dom->second.rows, cols = dom->second.cols;
  auto cdiv = [](int64_t a, int64_t b) { return (a + b - 1) / b; };
  GenericLaunch L;
  MfjArgs& a = L.a;
  if (g.depth == 2) {
    if (rows % 32 || cols % 32) throw Fault("launch: domain '" + g.domain + "' not padded to 32");
    a.full_x = cols / 32;
    a.full_y = rows / 32;
    L.launch_x = g.iter_dim == 'x' ? cdiv(a.full_x, g.iterations) : a.full_x;
    L.launch_y = g.iter_dim == 'y' ? cdiv(a.full_y, g.iterations) : a.full_y;
  } else {
    const int64_t len = rows == 1 ? cols : rows;
    if (len % 32) throw Fault("launch: domain '" + g.domain + "' not padded to 32");
    a.n_elems = len / 32;
    a.full_x = cdiv(a.n_elems, g.instances);
    a.full_y = 1;
    L.launch_x = cdiv(a.full_x, g.iterations);
  }
  for (size_t i = 0; i < g.buffers.size(); ++i) {
    auto it = bufs.find(g.buffers[i]);
    if (it == bufs.end() || !it->second.ptr)
      throw Fault("kernel " + k.name + ": unbound buffer '" + g.buffers[i] + "'");
    a.buf[i] = it->second.ptr;
    a.rows[i] = it->second.rows;
    a.cols[i] = it->second.cols;
  }
  for (size_t j = 0; j < g.scalars.size(); ++j) {
    auto it = sc.find(g.scalars[j]);
    if (it == sc.end()) throw Fault("kernel " + k.name + ": unbound scalar '" + g.scalars[j] + "'");
    a.scal[j] = static_cast<float>(it->second);
  }
  a.fault = ws.jit_fault(s);
  if (L.launch_x > 0x7fffffffLL || L.launch_y > 65535)
    throw Fault("kernel " + k.name + ": grid exceeds the device's limits");
  L.smem = sizeof(float) * (size_t)g.shared_words_total;
  if (L.smem > 227u * 1024u) throw Fault("vm fault: shared allocation exceeds device limit");
  return L;
}

JitFlags generic_flags(const NativeKernel& k) {
  JitFlags fl;
  fl.poison = k.generic_poison >= 0 ? k.generic_poison != 0 : options().generic_poison != 0;
  return fl;
}

// Launch-time proof that every index the generic kernel evaluates is in
// bounds for THESE buffer shapes and grid (interval arithmetic over the affine
// forms host/cudagen.cpp recorded).  Proved -> the kernel runs without
// per-access checks (it cannot fault); *fits32 -> every index value and
// buffer extent fits 32 bits, so index arithmetic runs in int.
bool prove_bounds(const GenericOp& g, const GenericLaunch& L, bool* fits32) {
  const int64_t rt[6] = {0, L.a.full_x, L.a.full_y, L.a.n_elems, L.launch_x, L.launch_y};
  const int64_t lim32 = (int64_t{1} << 31) - 1;
  bool small = true;
  for (size_t i = 0; i < g.buffers.size(); ++i)
    if (L.a.rows[i] * L.a.cols[i] > lim32) small = false;
  for (const auto& b : g.bounds) {
    if (!b.affine) return false;
    int64_t lo[2] = {0, 0}, hi[2] = {0, 0};
    for (int q = 0; q < (b.two ? 2 : 1); ++q) {
      int64_t mn = b.c0[q], mx = b.c0[q], mag = b.c0[q] < 0 ? -b.c0[q] : b.c0[q];
      for (const auto& t : b.terms[q]) {
        const int64_t vlo = rt[t.lo_kind] + t.lo, vhi = rt[t.hi_kind] + t.hi;
        if (vhi < vlo) continue;  // empty range (e.g. a grid extent of 0): never evaluated
        mn += t.coef > 0 ? t.coef * vlo : t.coef * vhi;
        mx += t.coef > 0 ? t.coef * vhi : t.coef * vlo;
        const int64_t a = std::max(vlo < 0 ? -vlo : vlo, vhi < 0 ? -vhi : vhi);
        mag += (t.coef < 0 ? -t.coef : t.coef) * a;
      }
      if (mag > lim32) small = false;
      lo[q] = mn;
      hi[q] = mx;
    }
    if (b.buffer >= 0) {
      const int64_t rows = L.a.rows[b.buffer], cols = L.a.cols[b.buffer];
      if (b.two) {
        if (lo[0] < 0 || hi[0] >= rows || lo[1] < 0 || hi[1] >= cols) return false;
      } else if (lo[0] < 0 || hi[0] >= rows * cols) {
        return false;
      }
    } else if (b.buffer == -1) {
      if (lo[0] < 0 || hi[0] >= b.words) return false;
    }
  }
  *fits32 = small;
  return true;
}

void run_generic(const NativeKernel& k, const BufMap& bufs, const ScalarMap& sc, cudaStream_t s,
                 Workspace& ws, Recorder* rec) {
  GenericLaunch L = generic_args(k, bufs, sc, s, ws);
  std::vector<std::pair<float*, size_t>> zero;
  if (!k.vm_semantics)  // engine contract: outputs are overwritten, not accumulated into
    for (const auto& name : k.generic.accumulated) {
      const DevBuf& b = bufs.at(name);
      zero.emplace_back(b.ptr, sizeof(float) * (size_t)b.size());
    }
  const GenericOp& g = k.generic;
  JitFlags fl = generic_flags(k);
  bool fits32 = false;
  if (options().generic_checked == 0 && prove_bounds(g, L, &fits32)) {
    fl.unchecked = true;  // cannot fault: drop the per-access checks
    fl.idx32 = fits32;
    // every block's serial iterations lie inside the domain: the per-call
    // "instance beyond the grid" predicate is constant true
    if (g.depth == 2)
      fl.exact = g.iter_dim == 'y' ? L.launch_y * g.iterations == L.a.full_y
                                   : L.launch_x * g.iterations == L.a.full_x;
    else
      fl.exact = L.a.full_x * g.instances == L.a.n_elems && L.launch_x * g.iterations == L.a.full_x;
  }
  if (rec) jit_load(g.source, fl);  // compile + load now: nothing heavy inside a capture
  const std::string src = g.source;
  const dim3 grid((unsigned)L.launch_x, (unsigned)L.launch_y), block((unsigned)(g.block_x * g.block_y));
  const bool empty = L.launch_x == 0 || L.launch_y == 0;
  emit(rec, "launch " + k.name, [=](cudaStream_t st) {
    for (const auto& [p, bytes] : zero) {
      const cudaError_t e = cudaMemsetAsync(p, 0, bytes, st);
      if (e != cudaSuccess) return e;
    }
    if (!empty) jit_launch(src, fl, grid, block, L.smem, L.a, st);
    return cudaGetLastError();
  }, s);
}

}  // namespace

void check_jit_faults(Workspace& ws, cudaStream_t stream) {
  if (!ws.jit_used()) return;
  unsigned h[2] = {0, 0};
  unsigned* d = ws.jit_fault(stream);
  check_cuda(cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, stream), "read jit fault");
  check_cuda(cudaStreamSynchronize(stream), "generic kernel");
  if (h[0] == kJitOk) return;
  check_cuda(cudaMemsetAsync(d, 0, sizeof h, stream), "reset jit fault");
  check_cuda(cudaStreamSynchronize(stream), "reset jit fault");
  const char* what = "fault";
  switch (h[0]) {
    case kJitGlobalBounds: what = "global access out of bounds"; break;
    case kJitOnchipBounds: what = "on-chip access out of element bounds"; break;
    case kJitPoisonRead: what = "read of uninitialized on-chip word"; break;
    case kJitDivZero: what = "index expression divides by zero"; break;
    case kJitBadStep: what = "loop with non-positive step"; break;
    default: break;
  }
  throw Fault(std::string("vm fault: ") + what + " (generic kernel, detail " + std::to_string(h[1]) + ")");
}

int64_t run_generic_counted(const NativeKernel& k, const BufMap& bufs, const ScalarMap& sc,
                            const int cost[6], bool trace, int64_t trace_cap, cudaStream_t s,
                            Workspace& ws, std::vector<uint64_t>* stats, std::vector<MfjRec>* recs,
                            int64_t* blocks) {
  if (k.kind != NativeKernel::Kind::Generic) throw Invalid("counted launch of a non-generic kernel");
  std::lock_guard<std::mutex> lk(ws.mu);
  GenericLaunch L = generic_args(k, bufs, sc, s, ws);
  const GenericOp& g = k.generic;
  const int T = g.block_x * g.block_y;
  *blocks = L.launch_x * L.launch_y;
  // counting scratch after the VM arena: per-thread costs + per-warp cycles
  const size_t arena = (size_t)g.shared_words_total;
  const size_t smem = sizeof(float) * ((arena + 4 * (size_t)T + 1) / 2 * 2) + 8 * (size_t)T;
  if (smem > 227u * 1024u) throw Fault("vm fault: shared allocation exceeds device limit");
  auto* dstats = reinterpret_cast<unsigned long long*>(ws.named("__jit_stats", 2 * kMfjStatWords));
  check_cuda(cudaMemsetAsync(dstats, 0, 8 * kMfjStatWords, s), "zero stats");
  MfjRec* drec = nullptr;
  if (trace && trace_cap > 0)
    drec = reinterpret_cast<MfjRec*>(ws.named("__jit_trace", trace_cap * (int64_t)(sizeof(MfjRec) / 4)));
  L.a.stats = dstats;
  L.a.trace = drec;
  L.a.trace_cap = drec ? trace_cap : 0;
  for (int i = 0; i < 6; ++i) L.a.cost[i] = cost[i];
  JitFlags fl = generic_flags(k);
  fl.stats = true;
  fl.trace = trace;
  if (L.launch_x > 0 && L.launch_y > 0)
    jit_launch(g.source, fl, dim3((unsigned)L.launch_x, (unsigned)L.launch_y), dim3((unsigned)T), smem,
               L.a, s);
  stats->assign(kMfjStatWords, 0);
  check_cuda(cudaMemcpyAsync(stats->data(), dstats, 8 * kMfjStatWords, cudaMemcpyDeviceToHost, s),
             "read stats");
  check_cuda(cudaStreamSynchronize(s), "counted generic kernel");
  const int64_t n = (int64_t)(*stats)[kStatTraceCursor];
  if (recs) {
    recs->clear();
    if (drec && n > 0 && n <= trace_cap) {
      recs->resize((size_t)n);
      check_cuda(cudaMemcpy(recs->data(), drec, sizeof(MfjRec) * (size_t)n, cudaMemcpyDeviceToHost),
                 "read trace");
    }
  }
  return n;
}

BufMap complete_bindings(const NativePlan& plan, const BufMap& bufs, Workspace& ws) {
  std::lock_guard<std::mutex> lk(ws.mu);
  BufMap out = bufs;
  for (const auto& b : plan.buffers) {
    if (out.count(b.name)) continue;
    if (b.role != Role::Intermediate) continue;
    DevBuf d;
    d.rows = b.rows;
    d.cols = b.cols;
    d.ptr = ws.named("__int__" + b.name, (int64_t)b.rows * b.cols);
    out[b.name] = d;
  }
  return out;
}

// A matrix kernel whose matrix an earlier kernel of the plan stored (the
// nearest earlier kernel that stores any matrix stores one of its inputs).
bool stored_earlier(const NativePlan& plan, int k) {
  const NativeKernel& kern = plan.kernels[k];
  if (kern.kind != NativeKernel::Kind::Matrix) return false;
  for (int j = k - 1; j >= 0; --j) {
    const NativeKernel& p = plan.kernels[j];
    if (p.kind != NativeKernel::Kind::Matrix || p.matrix.store.empty()) continue;
    for (const auto& m : kern.matrix.mats)
      if (m == p.matrix.store) return true;
    return false;
  }
  return false;
}

void run_kernel(const NativePlan& plan, int k, const BufMap& bufs, const ScalarMap& scalars,
                cudaStream_t stream, Workspace& ws, PeerGroup* peers) {
  if (k < 0 || k >= (int)plan.kernels.size()) throw Invalid("kernel index out of range");
  const NativeKernel& kern = plan.kernels[k];
  std::lock_guard<std::mutex> lk(ws.mu);
  // NVTX range per kernel (option "nvtx" / MF_NVTX=1): the plan's kernel names
  // appear on Nsight timelines around the host work + launch.
  const bool nvtx = options().nvtx != 0;
  if (nvtx) nvtxRangePushA(kern.name.c_str());
  try {
    // a dot over replicated vectors is whole on every rank: no peer reduction
    if (kern.kind == NativeKernel::Kind::Stream)
      run_stream(kern, bufs, scalars, stream, ws, nullptr,
                 peers && !plan.rank_reductions(k).empty() ? peers : nullptr);
    else if (kern.kind == NativeKernel::Kind::Generic) run_generic(kern, bufs, scalars, stream, ws, nullptr);
    else run_matrix(kern, bufs, scalars, stream, ws, peers, nullptr, stored_earlier(plan, k));
  } catch (...) {
    if (nvtx) nvtxRangePop();
    throw;
  }
  if (nvtx) nvtxRangePop();
}

void record_kernel(const NativePlan& plan, int k, const BufMap& bufs, const ScalarMap& scalars,
                   cudaStream_t stream, Workspace& ws, Recorder& rec) {
  if (k < 0 || k >= (int)plan.kernels.size()) throw Invalid("kernel index out of range");
  const NativeKernel& kern = plan.kernels[k];
  std::lock_guard<std::mutex> lk(ws.mu);
  if (kern.kind == NativeKernel::Kind::Stream) run_stream(kern, bufs, scalars, stream, ws, &rec);
  else if (kern.kind == NativeKernel::Kind::Generic) run_generic(kern, bufs, scalars, stream, ws, &rec);
  else run_matrix(kern, bufs, scalars, stream, ws, nullptr, &rec, stored_earlier(plan, k));
}

}  // namespace mapfuse::b200
