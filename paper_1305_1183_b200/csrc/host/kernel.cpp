// host/kernel.cpp -- KernelIR text emit / parse.
//
// Text format as documented by the reference (proj/src/kernel.cpp:33-65
// emitter, :178-280 reader): header keys, shared regions, register arrays,
// params, then prologue / loop / epilogue sections of routine calls.
#include "mapfuse/kernel.hpp"

#include <sstream>
#include <stdexcept>

namespace mapfuse::kernel {

namespace {

void emit_call(std::ostream& o, const RoutineCallIR& c) {
  if (c.is_pure_clear()) {
    if (c.barrier_before) o << "    barrier\n";
    o << "    clear " << c.clear_key << "\n";
    return;
  }
  o << "    call " << c.label << " id=" << c.call_id << " kind=" << lib::to_string(c.kind)
    << " shape=" << c.routine_px << "x" << c.routine_py
    << " remap=" << (c.remap == Remap::Identity ? "identity" : "flat");
  if (c.active_threads > 0) o << " guard=" << c.active_threads;
  o << " {\n";
  if (c.barrier_before) o << "      barrier\n";
  if (!c.clear_key.empty()) o << "      clear " << c.clear_key << "\n";
  if (c.barrier_after_clear) o << "      barrier\n";
  o << ir::print_program(c.body, 3) << "    }\n";
}

std::string trim(const std::string& s) {
  const size_t b = s.find_first_not_of(" \t\r");
  if (b == std::string::npos) return "";
  return s.substr(b, s.find_last_not_of(" \t\r") - b + 1);
}

std::vector<std::string> fields(const std::string& s) {
  std::istringstream in(s);
  std::vector<std::string> v;
  for (std::string w; in >> w;) v.push_back(w);
  return v;
}

struct Cursor {
  std::vector<std::string> lines;
  size_t i = 0;
  bool next(std::string* out) {
    while (i < lines.size()) {
      std::string t = trim(lines[i++]);
      if (!t.empty()) {
        *out = t;
        return true;
      }
    }
    return false;
  }
  bool peek(std::string* out) const {
    for (size_t j = i; j < lines.size(); ++j) {
      std::string t = trim(lines[j]);
      if (!t.empty()) {
        *out = t;
        return true;
      }
    }
    return false;
  }
  [[noreturn]] void fail(const std::string& m) const {
    throw std::runtime_error("kernel text line " + std::to_string(i) + ": " + m);
  }
};

RoutineCallIR read_call(Cursor& src, const std::string& header, const std::vector<std::string>& params) {
  RoutineCallIR c;
  const auto f = fields(header);
  if (f.size() < 2) src.fail("call header needs a label");
  c.label = f[1];
  for (size_t k = 2; k < f.size(); ++k) {
    const auto eq = f[k].find('=');
    if (eq == std::string::npos) continue;
    const std::string key = f[k].substr(0, eq), v = f[k].substr(eq + 1);
    if (key == "id") c.call_id = std::stoi(v);
    else if (key == "kind")
      c.kind = v == "load" ? lib::RoutineKind::Load
                           : (v == "store" ? lib::RoutineKind::Store : lib::RoutineKind::Compute);
    else if (key == "shape") {
      const auto x = v.find('x');
      c.routine_px = std::stoi(v.substr(0, x));
      c.routine_py = std::stoi(v.substr(x + 1));
    } else if (key == "remap") c.remap = v == "identity" ? Remap::Identity : Remap::FlatSplit;
    else if (key == "guard") c.active_threads = std::stoi(v);
  }
  std::vector<std::string> raw;
  int depth = 1;
  for (std::string l;;) {
    if (!src.next(&l)) src.fail("unterminated call block");
    for (char ch : l) depth += ch == '{' ? 1 : (ch == '}' ? -1 : 0);
    if (depth <= 0) break;
    raw.push_back(l);
  }
  size_t k = 0;
  if (k < raw.size() && raw[k] == "barrier") {
    c.barrier_before = true;
    ++k;
  }
  if (k < raw.size() && raw[k].rfind("clear ", 0) == 0) {
    c.clear_key = trim(raw[k].substr(6));
    ++k;
    if (k < raw.size() && raw[k] == "barrier") {
      c.barrier_after_clear = true;
      ++k;
    }
  }
  std::string body;
  for (; k < raw.size(); ++k) body += raw[k] + "\n";
  ir::ParseContext ctx;
  ctx.params = params;
  c.body = ir::parse_program(body, ctx);
  return c;
}

}  // namespace

std::string emit_pseudo_source(const KernelIR& k) {
  std::ostringstream o;
  o << "kernel " << k.name << " {\n"
    << "  depth " << k.depth << "\n"
    << "  block " << k.block_x << " " << k.block_y << "\n"
    << "  instances " << k.instances << "\n"
    << "  iterations " << k.iterations << "\n"
    << "  iterate " << k.iter_dim << "\n"
    << "  domain " << k.domain << "\n"
    << "  shared " << k.shared_words << "\n";
  for (const auto& r : k.shared_regions) {
    o << "  shared " << r.key << " @ " << r.offset << " words " << r.words;
    if (r.stride != 32) o << " stride " << r.stride;
    o << "\n";
  }
  for (const auto& r : k.reg_arrays) {
    o << "  registers " << r.key << " words " << r.words;
    if (r.collapse_threads > 0) o << " collapse " << r.collapse_threads;
    o << "\n";
  }
  for (const auto& p : k.scalar_params) o << "  param " << p << "\n";
  auto section = [&](const char* name, const std::vector<RoutineCallIR>& calls, bool always) {
    if (calls.empty() && !always) return;
    o << "  " << name << " {\n";
    for (const auto& c : calls) emit_call(o, c);
    o << "  }\n";
  };
  section("prologue", k.prologue, false);
  section("loop", k.body, true);
  section("epilogue", k.epilogue, false);
  o << "}\n";
  return o.str();
}

KernelIR parse_kernel_text(const std::string& text) {
  KernelIR k;
  Cursor src;
  {
    std::istringstream in(text);
    for (std::string l; std::getline(in, l);) src.lines.push_back(l);
  }
  std::string line;
  if (!src.next(&line) || fields(line).size() < 2 || fields(line)[0] != "kernel")
    src.fail("expected 'kernel <name> {'");
  k.name = fields(line)[1];
  while (src.next(&line)) {
    if (line == "}") break;
    const auto f = fields(line);
    const std::string& key = f[0];
    auto val = [&](size_t i) -> const std::string& {
      if (i >= f.size()) src.fail("'" + key + "' needs a value");
      return f[i];
    };
    if (key == "depth") k.depth = std::stoi(val(1));
    else if (key == "block") {
      k.block_x = std::stoi(val(1));
      k.block_y = std::stoi(val(2));
    } else if (key == "instances") k.instances = std::stoi(val(1));
    else if (key == "iterations") k.iterations = std::stoi(val(1));
    else if (key == "iterate") k.iter_dim = val(1)[0];
    else if (key == "domain") k.domain = val(1);
    else if (key == "shared" && f.size() == 2) k.shared_words = std::stoi(f[1]);
    else if (key == "shared") {
      SharedRegion r;
      r.key = val(1);
      for (size_t i = 2; i + 1 < f.size(); ++i) {
        if (f[i] == "@") r.offset = std::stoi(f[++i]);
        else if (f[i] == "words") r.words = std::stoi(f[++i]);
        else if (f[i] == "stride") r.stride = std::stoi(f[++i]);
      }
      k.shared_regions.push_back(r);
    } else if (key == "registers") {
      RegisterArray r;
      r.key = val(1);
      for (size_t i = 2; i + 1 < f.size(); ++i) {
        if (f[i] == "words") r.words = std::stoi(f[++i]);
        else if (f[i] == "collapse") r.collapse_threads = std::stoi(f[++i]);
      }
      k.reg_arrays.push_back(r);
    } else if (key == "param") {
      k.scalar_params.push_back(val(1));
    } else if (key == "prologue" || key == "loop" || key == "epilogue") {
      auto& sec = key == "prologue" ? k.prologue : (key == "loop" ? k.body : k.epilogue);
      for (std::string in;;) {
        if (!src.next(&in)) src.fail("unterminated section");
        if (in == "}") break;
        if (in == "barrier") {
          std::string nx;
          if (!src.peek(&nx) || nx.rfind("clear ", 0) != 0) src.fail("unexpected standalone barrier");
          src.next(&nx);
          RoutineCallIR c;
          c.barrier_before = true;
          c.clear_key = trim(nx.substr(6));
          sec.push_back(std::move(c));
        } else if (in.rfind("clear ", 0) == 0) {
          RoutineCallIR c;
          c.clear_key = trim(in.substr(6));
          sec.push_back(std::move(c));
        } else if (in.rfind("call ", 0) == 0) {
          sec.push_back(read_call(src, in, k.scalar_params));
        } else {
          src.fail("expected call/clear, got '" + in + "'");
        }
      }
    } else {
      src.fail("unknown kernel key '" + key + "'");
    }
  }
  for (auto* sec : {&k.prologue, &k.body, &k.epilogue})
    for (auto& c : *sec) {
      c.bindings.assign(c.body.elements.size(), Binding{});
      for (size_t e = 0; e < c.body.elements.size(); ++e) {
        Binding& b = c.bindings[e];
        b.name = c.body.elements[e].name;
        for (const auto& r : k.shared_regions)
          if (r.key == b.name) {
            b.kind = Binding::Kind::Shared;
            b.offset = r.offset;
            b.stride = r.stride;
          }
        if (b.kind == Binding::Kind::Global)
          for (size_t i = 0; i < k.reg_arrays.size(); ++i)
            if (k.reg_arrays[i].key == b.name) {
              b.kind = Binding::Kind::Register;
              b.reg_array = static_cast<int>(i);
            }
      }
    }
  return k;
}

}  // namespace mapfuse::kernel
