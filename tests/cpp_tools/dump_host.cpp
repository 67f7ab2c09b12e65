// Test tool (CPU): prints what the product's host C++ produces so Python tests
// can pin it against the reference's own outputs.
//
//   dump_host library [manifest.mf]      canonical text of every elementary
//                                        function (builtin library if no file):
//                                        kind, depth, parallelism, elements,
//                                        args, and per routine its declared
//                                        thread maps + print_program(body)
//   dump_host problem SEQ ROWS COLS SEED OUTDIR
//                                        blas::make_problem(build_sequence(SEQ))
//                                        -> OUTDIR/<name>.f32 (raw fp32, row
//                                        major) + OUTDIR/index.txt
//                                        ("name rows cols" / "scalar name hex")
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "mapfuse/blas.hpp"
#include "mapfuse/ir.hpp"
#include "mapfuse/library.hpp"
#include "mapfuse/script.hpp"

using namespace mapfuse;

namespace {

std::string coord(const lib::MapCoord& c) {
  std::ostringstream os;
  os << c.cr << "," << c.cc << "," << c.c0 << "," << c.mod_const << "," << c.mod_macro;
  return os.str();
}

int dump_library(const lib::Library& L) {
  for (const auto& [name, f] : L.functions) {
    std::cout << "function " << name << " kind=" << lib::to_string(f.kind) << " depth=" << f.depth
              << " par_x=" << f.par_x << " par_y_is_block=" << f.par_y_is_block
              << " max_instances=" << f.max_instances << "\n";
    for (const auto& e : f.elements)
      std::cout << "  element " << e.name << " " << lib::to_string(e.kind) << " out=" << e.is_output
                << " acc=" << e.accumulable << " varies=" << e.varies.x << e.varies.y << "\n";
    for (const auto& a : f.args) std::cout << "  arg " << (a.is_scalar ? "scalar " : "") << a.name << "\n";
    for (const auto& r : f.results) std::cout << "  result " << r << "\n";
    for (const auto& s : f.scalar_params) std::cout << "  scalar " << s << "\n";
    for (const auto& r : f.routines) {
      std::cout << "  routine " << r.id() << " kind=" << lib::to_string(r.kind) << " target=" << r.target
                << " variant=" << r.variant << " atomic=" << r.writes_atomic << "\n";
      for (const auto& [el, m] : r.maps)
        std::cout << "    map " << el << " " << (int)m.kind << " tx=" << coord(m.tx) << " ty=" << coord(m.ty)
                  << "\n";
      std::istringstream body(ir::print_program(r.body));
      for (std::string line; std::getline(body, line);) std::cout << "    | " << line << "\n";
    }
  }
  return 0;
}

int dump_problem(const std::string& seq, int rows, int cols, unsigned seed, const std::string& dir) {
  const auto sc = script::parse_script(blas::build_sequence(seq).script_text);
  const blas::Problem p = blas::make_problem(sc, rows, cols, seed);
  std::ofstream idx(dir + "/index.txt");
  idx << "padded " << p.rows << " " << p.cols << "\n";
  for (const auto& [name, v] : p.buffers) {
    const auto d = p.dims.at(name);
    idx << "buffer " << name << " " << d.first << " " << d.second << "\n";
    std::ofstream f(dir + "/" + name + ".f32", std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), (std::streamsize)(v.size() * sizeof(float)));
  }
  for (const auto& [name, v] : p.scalars) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%a", (double)v);
    idx << "scalar " << name << " " << buf << "\n";
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "library") {
      if (argc > 2) {
        std::ifstream f(argv[2]);
        std::stringstream ss;
        ss << f.rdbuf();
        return dump_library(lib::load_library(ss.str()));
      }
      return dump_library(blas::default_library());
    }
    if (cmd == "problem" && argc == 7)
      return dump_problem(argv[2], std::stoi(argv[3]), std::stoi(argv[4]), (unsigned)std::stoul(argv[5]),
                          argv[6]);
    std::cerr << "usage: dump_host library [file] | problem SEQ ROWS COLS SEED OUTDIR\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
