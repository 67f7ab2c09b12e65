// host/semantics.hpp -- the algebra a routine body computes.
//
// A compute body is evaluated symbolically: every on-chip store / atomic add
// becomes a sum of terms, each term a coefficient (constants x scalar
// parameters) times a product of on-chip element loads with affine indices.
// Loops stay symbolic (their variable appears in the indices), so
//   tmp += A[tx, ty + j] * x[ty + j];  atomic y[tx] += alpha * tmp
// reads as y[tx] += alpha * A[tx, ty+j] * x[ty+j]: x shares A's column index
// and y takes A's row index -> a row reduction y = alpha * A x.  The same
// classification covers every Table-1 elementary function (maps, dot,
// rank-2 update, row / column reductions) without naming any of them; the
// lowering (lower.cpp) composes these per-call results into one sm_100a
// kernel.
#pragma once

#include <map>
#include <optional>
#include <string>
#include <vector>

#include "mapfuse/ir.hpp"
#include "mf_native.hpp"

namespace mapfuse::sem {

using b200::Coef;

struct Factor {
  std::string elem;
  std::vector<ir::LinearForm> idx;  // 1 (vector / scalar) or 2 (tile row, col)
};

struct Term {
  Coef coef = Coef::constant(1.0);
  std::vector<Factor> f;
};
using Poly = std::vector<Term>;

struct Assign {
  std::string elem;
  std::vector<ir::LinearForm> idx;
  Poly value;
  bool atomic = false;
};

// Symbolic evaluation of a body.  `param_value` maps a parameter slot to its
// coefficient (a script scalar symbol or a literal); throws on non-affine
// indices or constructs outside the algebra.
std::vector<Assign> evaluate(const ir::Program& p, const std::vector<Coef>& param_value);

// What one call computes, in terms of its on-chip element names.
struct CallSemantics {
  enum class Kind { Map, Dot, TileMap, RowReduce, ColReduce } kind = Kind::Map;
  std::string out;
  // Map: out = sum coef_i * in_i (vectors); TileMap: out = sum coef_t * tile_t
  std::vector<std::pair<std::string, Coef>> lin;
  // TileMap rank terms: coef * u (row-indexed) v (col-indexed)^T
  struct Rank {
    std::string u, v;
    Coef coef;
  };
  std::vector<Rank> rank;
  // Dot: out = coef * sum a b ; Row/ColReduce: out = coef * (tile . vec)
  std::string a, b;
  Coef coef = Coef::constant(1.0);
};

// Classifies the assignments of one compute routine; `tiles` lists the
// element names indexed in two dimensions.
std::vector<CallSemantics> classify(const std::vector<Assign>& assigns);

}  // namespace mapfuse::sem
