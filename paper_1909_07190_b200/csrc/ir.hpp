// ir.hpp — pipeline IR of the B200 PolyMage-GPU library (stage DAG, §2.2).
//
// A pipeline is a DAG of stages; every stage is "a function mapping a multi-dimensional integer domain
// to values", defined by one expression over its variables, parameters, image/stage reads
// and table lookups.  Dims are outermost-first [c][y][x]; 1-3 dims.  Expression semantics are the
// library's reading R3-R5: f32 RN per op in the written order, int32 wrap, floor '/'.
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace pmg {

enum class DType : int { U8 = 1, U16 = 2, I16 = 3, I32 = 4, F32 = 5 };
int dtype_size(DType d);
const char* dtype_name(DType d);
bool dtype_is_float(DType d);

// value kind after type checking
enum class Kind : int { Int = 0, Float = 1 };

struct Expr;
using ExprP = std::shared_ptr<Expr>;

struct Expr {
  enum Op { INT, FLT, VAR, PARAM, ACCESS, TABLE, BIN, UN, CALL } op;
  int64_t ival = 0;      // INT
  float fval = 0.f;      // FLT: f32(f64(text))  (reading R3)
  std::string text;      // literal text / name / operator / function
  int index = -1;        // VAR: consumer dim (0..nd-1, outermost first); PARAM: param index;
                         // ACCESS: producer id (stage id, or image id when !is_stage); TABLE: table id
  bool is_stage = false; // ACCESS target kind
  std::vector<ExprP> args;
  Kind kind = Kind::Int; // result kind
  int line = 0, col = 0;
};

struct ImageDecl {
  std::string name;
  std::vector<ExprP> extents;
  DType dtype;
};

struct TableDecl {
  std::string name;
  ExprP extent;
  DType dtype;
};

struct StageDecl {
  std::string name;
  std::vector<std::string> vars;
  std::vector<ExprP> extents;
  DType dtype;
  ExprP expr;
  int line = 0;
};

struct Pipeline {
  std::vector<std::string> params;
  std::vector<ImageDecl> images;
  std::vector<TableDecl> tables;
  std::vector<StageDecl> stages;      // declaration order
  std::vector<int> liveouts;          // stage ids, declaration order of the liveout statements
  std::vector<int> topo;              // producers first; ties by declaration order
  std::vector<std::vector<int>> producers;  // per stage: distinct stage ids it reads
  std::vector<std::vector<int>> consumers;  // per stage: distinct stage ids reading it
  std::string source;
};

struct Error : std::runtime_error {
  int status;
  Error(int st, const std::string& m) : std::runtime_error(m), status(st) {}
};

// parse.cpp
std::shared_ptr<Pipeline> parse_pipeline(const std::string& text);   // throws Error(PMG_ERR_PARSE, "l:c: ...")

// integer evaluation of extent / constant expressions (params only; floor division)
int64_t eval_int(const Expr& e, const std::vector<int64_t>& params);
bool is_const_int(const Expr& e);   // only INT / PARAM / arithmetic on them

void collect_accesses(const ExprP& e, std::vector<Expr*>& out);   // ACCESS nodes, pre-order

}  // namespace pmg
