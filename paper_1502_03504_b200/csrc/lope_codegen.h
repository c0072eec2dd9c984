// lope_codegen.h — LOPE1 kernel IR (text) -> parsed tree -> CUDA body source.
#pragma once
#include <string>
#include <vector>

namespace lope {

struct Node {
  enum Kind { CONST, SCALAR, READ, ADD, MUL, DIV, NEG, ABS, SQRT, MIN, MAX } kind;
  double value = 0.0;       // CONST
  std::string name;         // SCALAR name
  int arr = -1;             // READ: array parameter index
  int off[3] = {0, 0, 0};   // READ offsets (unused dims 0)
  std::vector<int> kids;
};

struct Stmt {
  bool is_array;
  int target;               // array index (is_array) or local index
  int expr;                 // node index
};

struct Kir {
  std::string name;
  int rank = 0;
  std::vector<std::string> arrays;
  std::vector<std::string> scalars;        // parameter order
  std::vector<int> scalar_is_int;
  std::vector<std::string> locals;
  std::vector<Node> nodes;
  std::vector<Stmt> body;
  std::vector<int> stored;                 // array indices, first-store order
  int fn[8][3] = {{0}};                    // footprint (negative reach) per array, dim
  int fp[8][3] = {{0}};                    // footprint (positive reach)
  int nreads = 0;
};

// Parse + validate; returns "" on success, else an error message.
std::string parse_kir(const std::string& text, Kir* out);

// `struct LopeBody { ... }` for the parsed kernel (template on the element type).
std::string emit_body(const Kir& k);

}  // namespace lope
