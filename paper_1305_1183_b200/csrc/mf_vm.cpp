// mf_vm.cpp -- vm::launch / detect_races / measure_routine on the B200
// (see include/mapfuse/vm.hpp; reference: proj/src/vm.cpp).
#include "mapfuse/vm.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>

#include "mapfuse/planner.hpp"
#include "mf_compile.hpp"
#include "mf_exec.hpp"
#include "mf_jit.hpp"

namespace mapfuse::vm {

namespace {

std::atomic<int>& exact_flag() {
  static std::atomic<int> f{[] {
    const char* v = std::getenv("MF_VM_EXACT");
    return v ? std::atoi(v) : 0;
  }()};
  return f;
}

// Device copies of the caller's std::vector buffers.
b200::BufMap upload(const LaunchArgs& args, b200::Workspace& ws) {
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
  return bufs;
}

void download(const LaunchArgs& args, const b200::BufMap& bufs, const std::vector<std::string>& outs) {
  for (const auto& [name, gb] : args.buffers) {
    if (std::find(outs.begin(), outs.end(), name) == outs.end()) continue;
    b200::check_cuda(cudaMemcpy(gb.data->data(), bufs.at(name).ptr, sizeof(float) * gb.data->size(),
                                cudaMemcpyDeviceToHost),
                     "cudaMemcpy D2H");
  }
}

// Launch shape the VM reports (vm.cpp:455-472) -- independent of how it runs.
void shape_stats(const kernel::KernelIR& k, const DeviceConfig& dev, int64_t blocks,
                 ExecutionStats* st) {
  st->blocks = static_cast<int>(blocks);
  st->threads_per_block = k.threads();
  st->shared_bytes = k.shared_bytes_total();
  st->occupancy = dev.occupancy(k.shared_bytes_total(), k.threads());
  if (st->occupancy == 0) throw VmFault("vm fault: zero occupancy");
  st->latency_factor = dev.latency_factor(st->occupancy);
}

int64_t grid_blocks(const kernel::KernelIR& k, const LaunchArgs& args) {
  const GlobalBuffer& dom = args.buffers.at(k.domain);
  auto cdiv = [](int64_t a, int64_t b) { return (a + b - 1) / b; };
  if (k.depth == 2) {
    const int64_t fx = dom.cols / 32, fy = dom.rows / 32;
    return (k.iter_dim == 'x' ? cdiv(fx, k.iterations) : fx) *
           (k.iter_dim == 'y' ? cdiv(fy, k.iterations) : fy);
  }
  const int64_t len = dom.rows == 1 ? dom.cols : dom.rows;
  return cdiv(cdiv(len / 32, k.instances), k.iterations);
}

TraceRecord to_record(const b200::MfjRec& r) {
  TraceRecord t;
  t.block = r.block;
  t.epoch = r.epoch;
  t.space = r.space == 0 ? Space::Shared : (r.space == 1 ? Space::Register : Space::Global);
  t.region = r.region;
  t.addr = r.addr;
  t.thread = r.thread;
  t.kinds = r.kinds;
  return t;
}

// The generic kernel with the VM's counters (and trace) compiled in.
LaunchResult launch_counted(const kernel::KernelIR& k, const DeviceConfig& dev,
                            const LaunchArgs& args, b200::NativeKernel nk) {
  LaunchResult res;
  b200::Workspace ws;
  b200::BufMap bufs = upload(args, ws);
  b200::ScalarMap sc;
  for (const auto& [n, v] : args.scalars) sc[n] = v;
  const int cost[6] = {dev.cycles_per_global_word, dev.cycles_per_shared_word, dev.cycles_per_arith_op,
                       dev.cycles_per_barrier, dev.cycles_per_atomic, dev.warp_size};
  std::vector<uint64_t> st;
  std::vector<b200::MfjRec> recs;
  int64_t blocks = 0;
  int64_t cap = args.trace ? (int64_t)1 << 20 : 0;
  cudaEvent_t e0, e1;
  b200::check_cuda(cudaEventCreate(&e0), "event");
  b200::check_cuda(cudaEventCreate(&e1), "event");
  cudaEventRecord(e0, nullptr);
  int64_t n = b200::run_generic_counted(nk, bufs, sc, cost, args.trace, cap, nullptr, ws, &st, &recs,
                                        &blocks);
  cudaEventRecord(e1, nullptr);
  b200::check_cuda(cudaEventSynchronize(e1), "kernel");
  b200::check_jit_faults(ws, nullptr);
  if (args.trace && n > cap) {  // trace larger than the first buffer: rerun on fresh inputs
    bufs = upload(args, ws);
    cap = n;
    n = b200::run_generic_counted(nk, bufs, sc, cost, true, cap, nullptr, ws, &st, &recs, &blocks);
    b200::check_jit_faults(ws, nullptr);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  download(args, bufs, nk.outputs());

  ExecutionStats& s = res.stats;
  const b200::GenericOp& g = nk.generic;
  for (size_t i = 0; i < g.buffers.size(); ++i) {
    const uint64_t ld = st[b200::kStatLoaded + i], sd = st[b200::kStatStored + i];
    if (ld == 0 && sd == 0) continue;
    s.per_buffer[g.buffers[i]] = BufferTraffic{ld, sd};
    s.global_words_loaded += ld;
    s.global_words_stored += sd;
  }
  s.shared_accesses = st[b200::kStatShared];
  s.atomics = st[b200::kStatAtomics];
  s.barriers = st[b200::kStatBarriers];
  s.arith_ops = st[b200::kStatArith];
  s.block_cycles_sum = st[b200::kStatBlockCycles];
  shape_stats(k, dev, blocks, &s);
  const double parallel =
      static_cast<double>(s.block_cycles_sum) / (static_cast<double>(dev.sm_count) * s.occupancy);
  s.cycles = static_cast<uint64_t>(std::ceil(parallel / s.latency_factor));
  s.device_ms = ms;
  s.native_kernel = "generic";
  s.vm_exact = true;
  if (args.trace) {
    res.trace.reserve(recs.size());
    for (const auto& r : recs) res.trace.push_back(to_record(r));
    res.races = detect_races(k, res.trace);
  }
  return res;
}

}  // namespace

void set_exact(bool on) { exact_flag() = on ? 1 : 0; }
bool exact() { return exact_flag() != 0; }

LaunchResult launch(const kernel::KernelIR& k, const DeviceConfig& dev, const LaunchArgs& args) {
  // static limits first, as the reference (vm.cpp:457-460)
  if (k.threads() > dev.max_threads_per_block)
    throw VmFault("vm fault: block of " + std::to_string(k.threads()) + " threads exceeds device");
  if (k.shared_bytes_total() > dev.shared_bytes_per_block)
    throw VmFault("vm fault: shared allocation exceeds device limit");
  auto dom = args.buffers.find(k.domain);
  if (dom == args.buffers.end()) throw VmFault("launch: no domain buffer '" + k.domain + "'");
  b200::NativePlan plan;
  try {
    if (args.trace || exact()) {
      b200::NativeKernel nk = plan::generic_kernel(k);
      nk.vm_semantics = true;
      nk.generic_poison = args.poison_onchip ? 1 : 0;
      return launch_counted(k, dev, args, std::move(nk));
    }
    plan = b200::plan_from_kernel_text(kernel::emit_pseudo_source(k), dom->second.rows,
                                       dom->second.cols);
  } catch (const VmFault&) {
    throw;
  } catch (const std::exception& e) {
    throw VmFault(std::string("launch: ") + e.what());
  }
  b200::NativeKernel& nk = plan.kernels[0];
  // A kernel no hand-written family covers runs on the generic path with the
  // VM's own contract -- accumulate into the caller's outputs, poison as asked
  // -- and with its counters, so the stats are the VM's.
  if (nk.kind == b200::NativeKernel::Kind::Generic) {
    nk.vm_semantics = true;
    nk.generic_poison = args.poison_onchip ? 1 : 0;
    try {
      return launch_counted(k, dev, args, nk);
    } catch (const b200::Fault& e) {
      throw VmFault(e.what());
    } catch (const b200::Invalid& e) {
      throw VmFault(e.what());
    }
  }
  LaunchResult res;
  b200::Workspace ws;
  try {
    b200::BufMap bufs = upload(args, ws);
    b200::ScalarMap sc;
    for (const auto& [n, v] : args.scalars) sc[n] = v;
    cudaEvent_t e0, e1;
    b200::check_cuda(cudaEventCreate(&e0), "event");
    b200::check_cuda(cudaEventCreate(&e1), "event");
    cudaEventRecord(e0, nullptr);
    b200::run_kernel(plan, 0, bufs, sc, nullptr, ws);
    cudaEventRecord(e1, nullptr);
    b200::check_cuda(cudaEventSynchronize(e1), "kernel");
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    res.stats.device_ms = ms;
    download(args, bufs, nk.outputs());
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
    shape_stats(k, dev, grid_blocks(k, args), &res.stats);
    res.stats.native_kernel = nk.kind == b200::NativeKernel::Kind::Matrix ? "matrix" : "stream";
  } catch (const b200::Fault& e) {
    throw VmFault(e.what());
  } catch (const b200::Invalid& e) {
    throw VmFault(e.what());
  }
  return res;
}

RaceReport detect_races(const kernel::KernelIR& k, const std::vector<TraceRecord>& trace) {
  // Group the shared-memory accesses of each block by (epoch, arena word),
  // in ascending (block, epoch, word) order; a group with a non-atomic write
  // and an access by another thread is one hazard.
  struct Key {
    int32_t block, epoch;
    int64_t addr;
    bool operator<(const Key& o) const {
      if (block != o.block) return block < o.block;
      if (epoch != o.epoch) return epoch < o.epoch;
      return addr < o.addr;
    }
  };
  std::map<Key, std::vector<const TraceRecord*>> groups;
  for (const auto& r : trace)
    if (r.space == Space::Shared) groups[{r.block, r.epoch, r.addr}].push_back(&r);
  RaceReport rep;
  for (const auto& [key, recs] : groups) {
    for (const TraceRecord* w : recs) {
      const bool plain_write = (w->kinds & 2) && !(w->kinds & 4);
      if (!plain_write) continue;
      auto other = std::find_if(recs.begin(), recs.end(),
                                [&](const TraceRecord* o) { return o->thread != w->thread; });
      if (other == recs.end()) continue;
      Hazard h;
      if (w->region >= 0 && w->region < static_cast<int>(k.shared_regions.size())) {
        h.key = k.shared_regions[w->region].key;
        h.word = key.addr - k.shared_regions[w->region].offset;
      }
      h.writer = w->thread;
      h.other = (*other)->thread;
      h.writer_kinds = w->kinds;
      h.other_kinds = (*other)->kinds;
      h.block = key.block;
      h.epoch = key.epoch;
      rep.hazards.push_back(h);
      break;
    }
  }
  return rep;
}

std::optional<uint64_t> measure_routine(const lib::ElementaryFunction& f, const lib::Routine& r,
                                        const MeasureEnv& env, const DeviceConfig& dev) {
  // One block running the routine once per serial iteration, every element
  // it touches staged in shared memory (tiles at stride 33) -- the cost-DB
  // micro-benchmark of the paper, counted on the GPU.
  if (env.instances > f.max_instances) return std::nullopt;
  const int by = f.depth == 2 ? 4 : 1;
  kernel::KernelIR k;
  k.name = "bench_" + f.name + "_" + r.id();
  k.depth = f.depth;
  k.block_x = f.depth == 2 ? 32 : 32 * env.instances;
  k.block_y = f.depth == 2 ? by : 1;
  k.instances = f.depth == 2 ? 1 : env.instances;
  k.iterations = env.iterations;
  k.iter_dim = f.depth == 2 ? 'y' : 'x';
  k.domain = "__domain";
  kernel::RoutineCallIR call;
  call.body = ir::substitute_macros(r.body, {{"BY", by}, {"IPB", k.instances}, {"ITERS", env.iterations}});
  call.label = f.name + "." + r.id();
  call.kind = r.kind;
  call.routine_px = f.par_x;
  call.routine_py = f.depth == 2 ? k.block_y : 1;
  call.remap = f.depth == 2 ? kernel::Remap::Identity : kernel::Remap::FlatSplit;
  int offset = 0;
  for (const auto& el : call.body.elements) {
    const lib::ElementDecl* decl = f.element(el.name);
    if (!decl) return std::nullopt;
    const bool tile = decl->kind == lib::ElemKind::Tile32x32;
    const int words = tile ? 33 * 32 : lib::elem_words(decl->kind);
    k.shared_regions.push_back(kernel::SharedRegion{el.name, offset, words, tile ? 33 : 32});
    kernel::Binding b;
    b.kind = kernel::Binding::Kind::Shared;
    b.name = el.name;
    b.offset = offset;
    b.stride = tile ? 33 : 32;
    call.bindings.push_back(b);
    offset += words;
  }
  k.shared_words = offset;
  const int shared_bytes = k.shared_words_total() * 4 + env.extra_shared_bytes;
  if (shared_bytes > dev.shared_bytes_per_block || k.threads() > dev.max_threads_per_block)
    return std::nullopt;
  for (const auto& p : f.scalar_params) k.scalar_params.push_back(p);
  k.body.push_back(std::move(call));
  // synthetic all-ones buffers covering one block's footprint
  std::map<std::string, std::vector<float>> storage;
  LaunchArgs args;
  args.poison_onchip = false;
  const int rows = 32 * env.iterations;
  const int dcols = 32 * (f.depth == 2 ? 1 : k.instances * env.iterations);
  if (f.depth == 2) {
    storage["__domain"].assign(static_cast<size_t>(rows) * 32, 1.0f);
    args.buffers["__domain"] = GlobalBuffer{rows, 32, &storage["__domain"]};
  } else {
    storage["__domain"].assign(static_cast<size_t>(dcols), 1.0f);
    args.buffers["__domain"] = GlobalBuffer{1, dcols, &storage["__domain"]};
  }
  for (const auto& decl : f.elements) {
    if (storage.count(decl.name)) continue;
    int brows = 1, bcols = 1;
    if (decl.kind == lib::ElemKind::Tile32x32) {
      brows = f.depth == 2 ? rows : 32;
      bcols = 32;
    } else if (decl.kind == lib::ElemKind::Subvector32) {
      bcols = decl.varies.y ? rows : dcols;
    }
    storage[decl.name].assign(static_cast<size_t>(brows) * bcols, 1.0f);
    args.buffers[decl.name] = GlobalBuffer{brows, bcols, &storage[decl.name]};
  }
  for (const auto& p : f.scalar_params) args.scalars[p] = 1.0f;
  const int occ = dev.occupancy(shared_bytes, k.threads());
  if (occ == 0) return std::nullopt;
  b200::NativeKernel nk = plan::generic_kernel(k);
  nk.vm_semantics = true;
  nk.generic_poison = 0;
  const LaunchResult res = launch_counted(k, dev, args, std::move(nk));
  const double adjusted = static_cast<double>(res.stats.block_cycles_sum) / dev.latency_factor(occ);
  return static_cast<uint64_t>(std::ceil(adjusted / env.iterations));
}

}  // namespace mapfuse::vm
