// lope_codegen.cpp — parse the LOPE1 IR text and emit the kernel body.
//
// The body is the tree of lopec/ir.py:258-308 evaluated per point: each IR node
// becomes one IEEE operation in the element type (LopeAr<T>::add/mul/div never
// contract into FMA), constants are exact hex literals converted to T once
// (np.float32(value) semantics), and a centre read of an array stored earlier
// in the body reads the pending value (ir.py:278-280).
#include <algorithm>
#include "lope_codegen.h"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>
#include <sstream>

namespace lope {

namespace {

struct Parser {
  std::vector<std::string> t;
  size_t p = 0;
  Kir* k;
  std::string err;
  std::map<std::string, int> arr_ix, scal_ix, loc_ix;

  bool more() const { return p < t.size(); }
  std::string next() {
    if (p >= t.size()) {
      if (err.empty()) err = "unexpected end of expression";
      return "";
    }
    return t[p++];
  }
  int parse_int(const std::string& s) {
    char* end = nullptr;
    long v = std::strtol(s.c_str(), &end, 10);
    if (s.empty() || *end) {
      if (err.empty()) err = "bad integer '" + s + "'";
      return 0;
    }
    return (int)v;
  }
  int add(Node n) {
    k->nodes.push_back(std::move(n));
    return (int)k->nodes.size() - 1;
  }
  int expr(int depth = 0) {
    if (!err.empty()) return -1;
    if (depth > 4000) {
      err = "expression too deep";
      return -1;
    }
    std::string tok = next();
    Node n;
    if (tok == "c") {
      std::string v = next();
      char* end = nullptr;
      n.kind = Node::CONST;
      n.value = std::strtod(v.c_str(), &end);
      if (v.empty() || *end) err = "bad constant '" + v + "'";
      return add(n);
    }
    if (tok == "s") {
      n.kind = Node::SCALAR;
      n.name = next();
      return add(n);
    }
    if (tok == "r") {
      n.kind = Node::READ;
      std::string a = next();
      auto it = arr_ix.find(a);
      if (it == arr_ix.end()) {
        err = "read of unknown array '" + a + "'";
        return -1;
      }
      n.arr = it->second;
      for (int d = 0; d < k->rank; ++d) n.off[d] = parse_int(next());
      k->nreads++;
      return add(n);
    }
    if (tok == "+" || tok == "*" || tok == "/") {
      n.kind = tok == "+" ? Node::ADD : tok == "*" ? Node::MUL : Node::DIV;
      int a = expr(depth + 1);
      int b = expr(depth + 1);
      n.kids = {a, b};
      return add(n);
    }
    if (tok == "n" || tok == "abs" || tok == "sqrt") {
      n.kind = tok == "n" ? Node::NEG : tok == "abs" ? Node::ABS : Node::SQRT;
      n.kids = {expr(depth + 1)};
      return add(n);
    }
    if (tok == "min" || tok == "max") {
      n.kind = tok == "min" ? Node::MIN : Node::MAX;
      int cnt = parse_int(next());
      if (cnt < 2 || cnt > 64) {
        err = "min/max needs 2..64 arguments";
        return -1;
      }
      for (int i = 0; i < cnt; ++i) n.kids.push_back(expr(depth + 1));
      return add(n);
    }
    if (err.empty()) err = "bad token '" + tok + "'";
    return -1;
  }
};

std::vector<std::string> split_ws(const std::string& s) {
  std::vector<std::string> out;
  std::istringstream is(s);
  std::string w;
  while (is >> w) out.push_back(w);
  return out;
}

bool valid_ident(const std::string& s) {
  if (s.empty() || s.size() > 64) return false;
  for (size_t i = 0; i < s.size(); ++i) {
    char c = s[i];
    bool ok = (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c == '_' || (i > 0 && c >= '0' && c <= '9');
    if (!ok) return false;
  }
  return true;
}

}  // namespace

std::string parse_kir(const std::string& text, Kir* k) {
  *k = Kir();
  std::istringstream is(text);
  std::string line;
  bool header = false, ended = false;
  Parser P;
  P.k = k;
  std::set<std::string> assigned_locals, stored_arrays;
  while (std::getline(is, line)) {
    auto tok = split_ws(line);
    if (tok.empty()) continue;
    if (!header) {
      if (tok[0] != "LOPE1") return "not a LOPE1 kernel";
      header = true;
      continue;
    }
    const std::string& w = tok[0];
    if (w == "kernel") {
      if (tok.size() != 3) return "bad kernel line";
      k->name = tok[1];
      k->rank = std::atoi(tok[2].c_str());
      if (k->rank < 1 || k->rank > 3) return "kernel rank must be 1..3";
    } else if (w == "array") {
      if (tok.size() != 2 || !valid_ident(tok[1])) return "bad array line";
      if (k->arrays.size() >= 8) return "at most 8 array parameters";
      P.arr_ix[tok[1]] = (int)k->arrays.size();
      k->arrays.push_back(tok[1]);
    } else if (w == "scalar") {
      if (tok.size() != 3 || !valid_ident(tok[1])) return "bad scalar line";
      if (k->scalars.size() >= 16) return "at most 16 scalar parameters";
      if (tok[2] != "real" && tok[2] != "integer") return "scalar kind must be real or integer";
      P.scal_ix[tok[1]] = (int)k->scalars.size();
      k->scalars.push_back(tok[1]);
      k->scalar_is_int.push_back(tok[2] == "integer");
    } else if (w == "local") {
      if (tok.size() != 2 || !valid_ident(tok[1])) return "bad local line";
      P.loc_ix[tok[1]] = (int)k->locals.size();
      k->locals.push_back(tok[1]);
    } else if (w == "store" || w == "let") {
      if (k->rank == 0) return "statement before the kernel line";
      if (tok.size() < 3) return "empty statement";
      P.t.assign(tok.begin() + 2, tok.end());
      P.p = 0;
      Stmt st;
      st.is_array = (w == "store");
      size_t first_new = k->nodes.size();
      st.expr = P.expr();
      if (!P.err.empty()) return P.err;
      if (P.p != P.t.size()) return "trailing tokens in statement";
      // validate reads / scalar uses in the new nodes
      for (size_t i = first_new; i < k->nodes.size(); ++i) {
        const Node& n = k->nodes[i];
        if (n.kind == Node::READ) {
          bool centre = n.off[0] == 0 && n.off[1] == 0 && n.off[2] == 0;
          if (!centre && stored_arrays.count(k->arrays[n.arr]))
            return "halo read of '" + k->arrays[n.arr] + "' after it was stored (E103)";
          for (int d = 0; d < k->rank; ++d)
            if (std::abs(n.off[d]) > 8) return "offset exceeds the maximum halo width 8";
        } else if (n.kind == Node::SCALAR) {
          if (!P.scal_ix.count(n.name) && !assigned_locals.count(n.name))
            return "scalar '" + n.name + "' read before assignment";
        }
      }
      if (st.is_array) {
        auto it = P.arr_ix.find(tok[1]);
        if (it == P.arr_ix.end()) return "store to unknown array '" + tok[1] + "'";
        st.target = it->second;
        if (!stored_arrays.count(tok[1])) {
          stored_arrays.insert(tok[1]);
          k->stored.push_back(st.target);
        }
      } else {
        auto it = P.loc_ix.find(tok[1]);
        if (it == P.loc_ix.end()) return "assignment to undeclared local '" + tok[1] + "'";
        st.target = it->second;
        assigned_locals.insert(tok[1]);
      }
      k->body.push_back(st);
    } else if (w == "end") {
      ended = true;
      break;
    } else {
      return "bad line '" + line + "'";
    }
  }
  if (!header) return "empty kernel text";
  if (!ended) return "missing 'end'";
  if (k->arrays.empty()) return "kernel has no array parameter";
  if (k->stored.empty()) return "kernel stores no array";
  for (const Node& n : k->nodes) {
    if (n.kind != Node::READ) continue;
    for (int d = 0; d < 3; ++d) {
      int o = n.off[d];
      if (o < 0 && -o > k->fn[n.arr][d]) k->fn[n.arr][d] = -o;
      if (o > 0 && o > k->fp[n.arr][d]) k->fp[n.arr][d] = o;
    }
  }
  return "";
}

namespace {

std::string hexlit(double v) {
  if (std::isnan(v)) return "__longlong_as_double(0x7ff8000000000000ULL)";
  if (std::isinf(v)) return v > 0 ? "__longlong_as_double(0x7ff0000000000000ULL)"
                                   : "__longlong_as_double(0xfff0000000000000ULL)";
  char buf[64];
  std::snprintf(buf, sizeof buf, "%a", v);
  return std::string(buf);
}

struct Emitter {
  const Kir& k;
  std::set<int> pending;        // arrays stored so far (statement order)
  std::map<std::string, int> scal_ix, loc_ix;
  explicit Emitter(const Kir& kk) : k(kk) {
    for (size_t i = 0; i < k.scalars.size(); ++i) scal_ix[k.scalars[i]] = (int)i;
    for (size_t i = 0; i < k.locals.size(); ++i) loc_ix[k.locals[i]] = (int)i;
  }
  std::string ex(int i) {
    const Node& n = k.nodes[i];
    switch (n.kind) {
      case Node::CONST:
        return "AR::c(T(" + hexlit(n.value) + "))";
      case Node::SCALAR: {
        auto it = loc_ix.find(n.name);
        if (it != loc_ix.end() && assigned.count(n.name)) return "l" + std::to_string(it->second);
        auto jt = scal_ix.find(n.name);
        return "AR::c(sc[" + std::to_string(jt->second) + "])";
      }
      case Node::READ: {
        bool centre = n.off[0] == 0 && n.off[1] == 0 && n.off[2] == 0;
        if (centre && pending.count(n.arr)) return "p" + std::to_string(n.arr);
        return "rd.template at<" + std::to_string(n.arr) + "," + std::to_string(n.off[0]) + "," +
               std::to_string(n.off[1]) + "," + std::to_string(n.off[2]) + ">()";
      }
      case Node::ADD: {
        // a + (-b) is a - b in IEEE arithmetic (same rounding, same signed zeros): one
        // subtraction instead of a negation feeding an add (FADD2 takes the negated operand)
        const Node& b = k.nodes[n.kids[1]];
        if (b.kind == Node::NEG) return "AR::sub(" + ex(n.kids[0]) + ", " + ex(b.kids[0]) + ")";
        return "AR::add(" + ex(n.kids[0]) + ", " + ex(n.kids[1]) + ")";
      }
      case Node::MUL: {
        // a product with a power-of-two constant is exact unless it underflows, and ptxas
        // then fuses a paired multiply into the following paired add (FFMA2), which
        // rounds differently in the subnormal range: AR::mulx keeps it a separate multiply
        const bool p2 = pow2_const(n.kids[0]) || pow2_const(n.kids[1]);
        return std::string(p2 ? "AR::mulx(" : "AR::mul(") + ex(n.kids[0]) + ", " + ex(n.kids[1]) + ")";
      }
      case Node::DIV: {
        // x / 2^k == x * 2^-k exactly in IEEE arithmetic (same real value, one rounding),
        // so a power-of-two constant divisor becomes a multiply (float and double alike)
        const Node& d = k.nodes[n.kids[1]];
        if (d.kind == Node::CONST && d.value != 0.0 && std::isfinite(d.value)) {
          int e = 0;
          double fr = std::frexp(d.value, &e);
          if ((fr == 0.5 || fr == -0.5) && e > -100 && e < 100)
            return "AR::mulx(" + ex(n.kids[0]) + ", AR::c(T(" + hexlit(1.0 / d.value) + ")))";
          // any other constant: reciprocal + FMA correction (LopeAr::divc), with the
          // correctly rounded reciprocal of the divisor as converted to each type
          const float bf = (float)d.value;
          const double yf = (double)(1.0f / bf);
          const double yd = 1.0 / d.value;
          const float abf = std::fabs(bf);
          const double abd = std::fabs(d.value);
          const bool okf = std::isfinite(bf) && abf >= 0x1p-16f && abf <= 0x1p+16f && std::isfinite(yf);
          const bool okd = abd >= 0x1p-60 && abd <= 0x1p+60;
          has_divc = true;
          return "AR::template divc<FAST>(" + ex(n.kids[0]) + ", " + ex(n.kids[1]) + ", " + hexlit(yf) + ", " +
                 hexlit(yd) + ", " + (okf ? "true" : "false") + ", " + (okd ? "true" : "false") + ", slow)";
        }
        if (d.kind == Node::SCALAR && !loc_ix.count(d.name) && 2 * k.scalars.size() <= 16) {
          // kernel scalar divisor: the host passes RN(1/b) (or NaN) after the scalars
          has_divc = true;
          const int i = scal_ix.at(d.name);
          return "AR::template divs<FAST>(" + ex(n.kids[0]) + ", sc[" + std::to_string(i) + "], sc[" +
                 std::to_string(k.scalars.size() + i) + "], slow)";
        }
        return "AR::div(" + ex(n.kids[0]) + ", " + ex(n.kids[1]) + ")";
      }
      case Node::NEG: return "AR::neg(" + ex(n.kids[0]) + ")";
      case Node::ABS: return "AR::abs_(" + ex(n.kids[0]) + ")";
      case Node::SQRT: return "AR::sqrt_(" + ex(n.kids[0]) + ")";
      case Node::MIN:
      case Node::MAX: {
        const char* f = n.kind == Node::MIN ? "AR::min_" : "AR::max_";
        std::string acc = ex(n.kids[0]);
        for (size_t q = 1; q < n.kids.size(); ++q) acc = std::string(f) + "(" + acc + ", " + ex(n.kids[q]) + ")";
        return acc;
      }
    }
    return "AR::c(T(0))";
  }
  bool pow2_const(int i) const {
    const Node& c = k.nodes[i];
    if (c.kind != Node::CONST || c.value == 0.0 || !std::isfinite(c.value)) return false;
    int e = 0;
    const double fr = std::frexp(c.value, &e);
    return fr == 0.5 || fr == -0.5;
  }
  std::set<std::string> assigned;   // locals assigned so far
  bool has_divc = false;            // a constant division went through LopeAr::divc
};

}  // namespace

std::string emit_body(const Kir& k) {
  std::ostringstream o;
  o << "// kernel '" << k.name << "' (rank " << k.rank << ")\n";
  o << "struct LopeBody {\n";
  o << "  static constexpr int RANK = " << k.rank << ";\n";
  o << "  static constexpr int NARR = " << k.arrays.size() << ";\n";
  o << "  static constexpr int NSTORE = " << k.stored.size() << ";\n";
  const char* dn[3] = {"0", "1", "2"};
  for (int d = 0; d < 3; ++d) {
    o << "  static constexpr int FN" << dn[d] << " = " << k.fn[0][d] << ";\n";
    o << "  static constexpr int FP" << dn[d] << " = " << k.fp[0][d] << ";\n";
  }
  // union of every array's footprint (the multi-array tiled kernel stages one box per
  // array with these halos)
  for (int d = 0; d < 3; ++d) {
    int un = 0, up = 0;
    for (size_t a = 0; a < k.arrays.size(); ++a) {
      un = std::max(un, k.fn[a][d]);
      up = std::max(up, k.fp[a][d]);
    }
    o << "  static constexpr int UFN" << dn[d] << " = " << un << ";\n";
    o << "  static constexpr int UFP" << dn[d] << " = " << up << ";\n";
  }
  // ZSTAR: every read of array 0 off the centre plane is at x = y = 0 (past planes can
  // live in registers in the tiled kernel)
  bool zstar = k.rank == 3;
  for (const Node& n : k.nodes)
    if (n.kind == Node::READ && n.arr == 0 && n.off[2] != 0 && (n.off[0] != 0 || n.off[1] != 0)) zstar = false;
  o << "  static constexpr bool ZSTAR = " << (zstar ? "true" : "false") << ";\n";
  o << "  static __device__ __forceinline__ constexpr int stored(int q) { return ";
  for (size_t i = 0; i + 1 < k.stored.size(); ++i) o << "q == " << i << " ? " << k.stored[i] << " : ";
  o << k.stored.back() << "; }\n";
  // FAST evaluation (tiled kernel) keeps every point branch-free so the compiler can
  // interleave the points' dependency chains; a constant division whose operand lies
  // outside its fast range sets `slow` and the caller re-evaluates with FAST = false.
  Emitter E(k);
  std::ostringstream b;
  for (const Stmt& st : k.body) {
    std::string rhs = E.ex(st.expr);
    if (st.is_array) {
      b << "    p" << st.target << " = " << rhs << ";\n";
      E.pending.insert(st.target);
    } else {
      b << "    l" << st.target << " = " << rhs << ";\n";
      E.assigned.insert(k.locals[st.target]);
    }
  }
  o << "  static constexpr bool HAS_DIVC = " << (E.has_divc ? "true" : "false") << ";\n";
  // W = T (one point) or a pair type evaluating two points per instruction (LopeAr2:
  // FADD2 / FMUL2 on sm_100, same IEEE round-to-nearest per element)
  o << "  template <class T, bool FAST, class RD, class W = T, class AR = LopeAr<T>>\n";
  o << "  static __device__ __forceinline__ void eval(const RD& rd, const T* __restrict__ sc, W* res, bool& slow) {\n";
  o << "    (void)sc;\n";
  o << "    (void)slow;\n";
  for (size_t i = 0; i < k.locals.size(); ++i) o << "    W l" << i << " = AR::c(T(0));\n";
  for (int a : k.stored) o << "    W p" << a << " = AR::c(T(0));\n";
  o << b.str();
  for (size_t q = 0; q < k.stored.size(); ++q) o << "    res[" << q << "] = p" << k.stored[q] << ";\n";
  o << "  }\n};\n";
  return o.str();
}

}  // namespace lope
