// parse.cpp — pipeline text -> validated stage DAG (§2.2; grammar extends SPEC.md
// line 81, documented in DESIGN.md §"Pipeline language").  Errors follow SPEC.md lines 40-47: syntax
// errors with line:col, undeclared references, cyclic references; plus unreachable stages.
#include <algorithm>
#include <cctype>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <set>
#include <sstream>

#include "../../include/pmg.h"
#include "ir.hpp"

namespace pmg {

int dtype_size(DType d) {
  switch (d) {
    case DType::U8: return 1;
    case DType::U16: case DType::I16: return 2;
    default: return 4;
  }
}
const char* dtype_name(DType d) {
  switch (d) {
    case DType::U8: return "u8";
    case DType::U16: return "u16";
    case DType::I16: return "i16";
    case DType::I32: return "i32";
    default: return "f32";
  }
}
bool dtype_is_float(DType d) { return d == DType::F32; }

namespace {

struct Tok {
  enum K { ID, NUM, OP, NL, END } k;
  std::string s;
  int line, col;
};

[[noreturn]] void fail(int line, int col, const std::string& m) {
  std::ostringstream o;
  o << line << ":" << col << ": " << m;
  throw Error(PMG_ERR_PARSE, o.str());
}

std::vector<Tok> lex(const std::string& t) {
  std::vector<Tok> v;
  int line = 1;
  size_t lstart = 0, i = 0;
  static const char* ops2[] = {"..", "<=", ">=", "==", "!=", "&&", "||", "<<", ">>"};
  while (i < t.size()) {
    char c = t[i];
    int col = int(i - lstart) + 1;
    if (c == '\n') { v.push_back({Tok::NL, "\n", line, col}); ++line; lstart = ++i; continue; }
    if (c == ' ' || c == '\t' || c == '\r') { ++i; continue; }
    if (c == '#') { while (i < t.size() && t[i] != '\n') ++i; continue; }
    if (std::isdigit((unsigned char)c) || (c == '.' && i + 1 < t.size() && std::isdigit((unsigned char)t[i + 1]))) {
      size_t j = i;
      while (j < t.size() && std::isdigit((unsigned char)t[j])) ++j;
      if (j < t.size() && t[j] == '.' && !(j + 1 < t.size() && t[j + 1] == '.')) {
        ++j;
        while (j < t.size() && std::isdigit((unsigned char)t[j])) ++j;
      }
      if (j < t.size() && (t[j] == 'e' || t[j] == 'E')) {
        size_t k = j + 1;
        if (k < t.size() && (t[k] == '+' || t[k] == '-')) ++k;
        if (k < t.size() && std::isdigit((unsigned char)t[k])) {
          j = k;
          while (j < t.size() && std::isdigit((unsigned char)t[j])) ++j;
        }
      }
      v.push_back({Tok::NUM, t.substr(i, j - i), line, col});
      i = j;
      continue;
    }
    if (std::isalpha((unsigned char)c) || c == '_') {
      size_t j = i;
      while (j < t.size() && (std::isalnum((unsigned char)t[j]) || t[j] == '_')) ++j;
      v.push_back({Tok::ID, t.substr(i, j - i), line, col});
      i = j;
      continue;
    }
    bool two = false;
    for (const char* o : ops2)
      if (t.compare(i, 2, o) == 0) { v.push_back({Tok::OP, o, line, col}); i += 2; two = true; break; }
    if (two) continue;
    if (std::strchr("-+*/%()<>,:=[]!", c)) { v.push_back({Tok::OP, std::string(1, c), line, col}); ++i; continue; }
    fail(line, col, std::string("unexpected character '") + c + "'");
  }
  v.push_back({Tok::END, "", line, int(i - lstart) + 1});
  return v;
}

const std::map<std::string, int>& builtins() {
  static const std::map<std::string, int> b = {
      {"min", 2}, {"max", 2}, {"abs", 1}, {"absd", 2}, {"clamp", 3}, {"select", 3}, {"lerp", 3}, {"sqrt", 1},
      {"f32", 1}, {"i32", 1}, {"i16", 1}, {"u16", 1}, {"u8", 1}, {"sat_u8", 1}, {"sat_u16", 1}};
  return b;
}

struct Parser {
  std::vector<Tok> t;
  size_t i = 0;
  int depth = 0;
  const Tok& peek() {
    while (depth > 0 && t[i].k == Tok::NL) ++i;
    return t[i];
  }
  Tok next() {
    Tok k = peek();
    ++i;
    return k;
  }
  void expect(const char* s) {
    Tok k = next();
    if (k.s != s) fail(k.line, k.col, std::string("expected '") + s + "', found '" + (k.k == Tok::END ? "end of input" : k.s) + "'");
    if (!std::strcmp(s, "(") || !std::strcmp(s, "[")) ++depth;
    if (!std::strcmp(s, ")") || !std::strcmp(s, "]")) --depth;
  }
  std::string ident() {
    Tok k = next();
    if (k.k != Tok::ID) fail(k.line, k.col, "expected identifier, found '" + k.s + "'");
    return k.s;
  }
  ExprP mk(Expr::Op op, const Tok& at) {
    auto e = std::make_shared<Expr>();
    e->op = op;
    e->line = at.line;
    e->col = at.col;
    return e;
  }
  ExprP expr() { return binary(0); }
  ExprP binary(int lvl) {
    static const std::vector<std::vector<std::string>> L = {
        {"||"}, {"&&"}, {"==", "!="}, {"<", "<=", ">", ">="}, {"<<", ">>"}, {"+", "-"}, {"*", "/", "%"}};
    if (lvl == (int)L.size()) return unary();
    ExprP a = binary(lvl + 1);
    for (;;) {
      const Tok& k = peek();
      if (k.k != Tok::OP || std::find(L[lvl].begin(), L[lvl].end(), k.s) == L[lvl].end()) break;
      Tok op = next();
      ExprP e = mk(Expr::BIN, op);
      e->text = op.s;
      e->args = {a, binary(lvl + 1)};
      a = e;
    }
    return a;
  }
  ExprP unary() {
    const Tok& k = peek();
    if (k.k == Tok::OP && (k.s == "-" || k.s == "!")) {
      Tok op = next();
      ExprP e = mk(Expr::UN, op);
      e->text = op.s;
      e->args = {unary()};
      return e;
    }
    return primary();
  }
  ExprP primary() {
    Tok k = next();
    if (k.k == Tok::NUM) {
      bool is_int = k.s.find_first_of(".eE") == std::string::npos;
      ExprP e = mk(is_int ? Expr::INT : Expr::FLT, k);
      e->text = k.s;
      if (is_int) {
        e->ival = std::strtoll(k.s.c_str(), nullptr, 10);
        if (e->ival > 2147483647LL) fail(k.line, k.col, "integer literal out of int32 range");
      } else {
        e->fval = (float)std::strtod(k.s.c_str(), nullptr);   // f32(f64(decimal)) (R3)
      }
      return e;
    }
    if (k.k == Tok::ID) {
      const Tok& n = peek();
      if (n.s == "(") {
        expect("(");
        std::vector<ExprP> args;
        if (peek().s != ")") {
          args.push_back(expr());
          while (peek().s == ",") { next(); args.push_back(expr()); }
        }
        expect(")");
        auto b = builtins().find(k.s);
        if (b != builtins().end()) {
          if ((int)args.size() != b->second)
            fail(k.line, k.col, k.s + " takes " + std::to_string(b->second) + " arguments");
          ExprP e = mk(Expr::CALL, k);
          e->text = k.s;
          e->args = args;
          return e;
        }
        ExprP e = mk(Expr::ACCESS, k);
        e->text = k.s;
        e->args = args;
        return e;
      }
      if (n.s == "[") {
        expect("[");
        ExprP idx = expr();
        expect("]");
        ExprP e = mk(Expr::TABLE, k);
        e->text = k.s;
        e->args = {idx};
        return e;
      }
      ExprP e = mk(Expr::VAR, k);   // resolved to VAR or PARAM later
      e->text = k.s;
      return e;
    }
    if (k.s == "(") {
      ++depth;
      ExprP e = expr();
      expect(")");
      return e;
    }
    fail(k.line, k.col, "unexpected '" + (k.k == Tok::END ? std::string("end of input") : k.s) + "'");
  }
  DType dtype() {
    Tok k = next();
    static const std::map<std::string, DType> m = {
        {"f32", DType::F32}, {"i32", DType::I32}, {"i16", DType::I16}, {"u16", DType::U16}, {"u8", DType::U8}};
    auto it = m.find(k.s);
    if (it == m.end()) fail(k.line, k.col, "unknown element type '" + k.s + "'");
    return it->second;
  }
  void end_stmt() {
    Tok k = next();
    if (k.k != Tok::NL && k.k != Tok::END) fail(k.line, k.col, "expected end of statement, found '" + k.s + "'");
  }
};

struct Resolver {
  Pipeline& p;
  std::map<std::string, int> img, stg, tab, prm;
  std::set<std::string> names;

  // resolve names and compute kinds for an expression in `scope` (stage vars); scope==nullptr: params only
  void resolve(const ExprP& e, const std::vector<std::string>* scope) {
    for (auto& a : e->args) resolve(a, scope);
    switch (e->op) {
      case Expr::INT: e->kind = Kind::Int; break;
      case Expr::FLT: e->kind = Kind::Float; break;
      case Expr::VAR: {
        if (scope) {
          auto it = std::find(scope->begin(), scope->end(), e->text);
          if (it != scope->end()) { e->index = int(it - scope->begin()); e->kind = Kind::Int; break; }
        }
        auto pi = prm.find(e->text);
        if (pi == prm.end()) fail(e->line, e->col, "undeclared name '" + e->text + "'");
        e->op = Expr::PARAM;
        e->index = pi->second;
        e->kind = Kind::Int;
        break;
      }
      case Expr::ACCESS: {
        if (!scope) fail(e->line, e->col, "reads are not allowed in extents");
        size_t nd;
        DType dt;
        if (stg.count(e->text)) {
          e->is_stage = true;
          e->index = stg[e->text];
          nd = p.stages[e->index].vars.size();
          dt = p.stages[e->index].dtype;
        } else if (img.count(e->text)) {
          e->is_stage = false;
          e->index = img[e->text];
          nd = p.images[e->index].extents.size();
          dt = p.images[e->index].dtype;
        } else {
          fail(e->line, e->col, "reference to undeclared stage/image '" + e->text + "'");
        }
        if (e->args.size() != nd)
          fail(e->line, e->col, e->text + " has " + std::to_string(nd) + " dims, read with " +
                                    std::to_string(e->args.size()) + " indices");
        for (size_t d = 0; d < e->args.size(); ++d)
          if (e->args[d]->kind != Kind::Int) fail(e->line, e->col, "index " + std::to_string(d) + " of " + e->text + " is not an integer expression");
        e->kind = dtype_is_float(dt) ? Kind::Float : Kind::Int;
        break;
      }
      case Expr::TABLE: {
        if (!scope) fail(e->line, e->col, "reads are not allowed in extents");
        auto it = tab.find(e->text);
        if (it == tab.end()) fail(e->line, e->col, "undeclared table '" + e->text + "'");
        e->index = it->second;
        if (e->args[0]->kind != Kind::Int) fail(e->line, e->col, "table index is not an integer expression");
        e->kind = dtype_is_float(p.tables[e->index].dtype) ? Kind::Float : Kind::Int;
        break;
      }
      case Expr::UN:
        e->kind = e->text == "!" ? Kind::Int : e->args[0]->kind;
        break;
      case Expr::BIN: {
        const std::string& o = e->text;
        Kind a = e->args[0]->kind, b = e->args[1]->kind;
        if (o == "%" || o == "<<" || o == ">>") {
          if (a != Kind::Int || b != Kind::Int) fail(e->line, e->col, "'" + o + "' needs integer operands");
          e->kind = Kind::Int;
        } else if (o == "&&" || o == "||" || o == "<" || o == "<=" || o == ">" || o == ">=" || o == "==" || o == "!=") {
          e->kind = Kind::Int;
        } else {
          e->kind = (a == Kind::Float || b == Kind::Float) ? Kind::Float : Kind::Int;
        }
        break;
      }
      case Expr::CALL: {
        const std::string& f = e->text;
        auto K = [&](int i) { return e->args[i]->kind; };
        if (f == "min" || f == "max" || f == "absd")
          e->kind = (K(0) == Kind::Float || K(1) == Kind::Float) ? Kind::Float : Kind::Int;
        else if (f == "clamp")
          e->kind = (K(0) == Kind::Float || K(1) == Kind::Float || K(2) == Kind::Float) ? Kind::Float : Kind::Int;
        else if (f == "abs") e->kind = K(0);
        else if (f == "select") e->kind = (K(1) == Kind::Float || K(2) == Kind::Float) ? Kind::Float : Kind::Int;
        else if (f == "lerp" || f == "sqrt" || f == "f32") e->kind = Kind::Float;
        else e->kind = Kind::Int;   // i32 i16 u16 u8 sat_u8 sat_u16
        break;
      }
      case Expr::PARAM: e->kind = Kind::Int; break;
    }
  }
};

}  // namespace

void collect_accesses(const ExprP& e, std::vector<Expr*>& out) {
  if (e->op == Expr::ACCESS) out.push_back(e.get());
  for (auto& a : e->args) collect_accesses(a, out);
}

bool is_const_int(const Expr& e) {
  switch (e.op) {
    case Expr::INT: case Expr::PARAM: return true;
    case Expr::BIN:
      if (e.text == "+" || e.text == "-" || e.text == "*" || e.text == "/" || e.text == "%")
        return is_const_int(*e.args[0]) && is_const_int(*e.args[1]);
      return false;
    case Expr::UN: return e.text == "-" && is_const_int(*e.args[0]);
    default: return false;
  }
}

static int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

int64_t eval_int(const Expr& e, const std::vector<int64_t>& params) {
  switch (e.op) {
    case Expr::INT: return e.ival;
    case Expr::PARAM:
      if (e.index < 0 || e.index >= (int)params.size()) throw Error(PMG_ERR_ARG, "missing parameter value");
      return params[e.index];
    case Expr::UN:
      if (e.text == "-") return -eval_int(*e.args[0], params);
      break;
    case Expr::BIN: {
      int64_t a = eval_int(*e.args[0], params), b = eval_int(*e.args[1], params);
      if (e.text == "+") return a + b;
      if (e.text == "-") return a - b;
      if (e.text == "*") return a * b;
      if (e.text == "/") { if (!b) throw Error(PMG_ERR_SHAPE, "division by zero in extent"); return floordiv(a, b); }
      if (e.text == "%") { if (!b) throw Error(PMG_ERR_SHAPE, "modulo by zero in extent"); return a - b * floordiv(a, b); }
      break;
    }
    default: break;
  }
  throw Error(PMG_ERR_PARSE, std::to_string(e.line) + ":" + std::to_string(e.col) + ": not a constant integer expression");
}

std::shared_ptr<Pipeline> parse_pipeline(const std::string& text) {
  auto P = std::make_shared<Pipeline>();
  Pipeline& p = *P;
  p.source = text;
  Parser ps;
  ps.t = lex(text);
  Resolver R{p, {}, {}, {}, {}, {}};
  std::vector<std::pair<std::string, Tok>> liveout_names;
  auto declare = [&](const std::string& n, const Tok& at) {
    if (R.names.count(n)) fail(at.line, at.col, "duplicate name '" + n + "'");
    R.names.insert(n);
  };
  for (;;) {
    Tok k = ps.next();
    if (k.k == Tok::END) break;
    if (k.k == Tok::NL) continue;
    if (k.k != Tok::ID) fail(k.line, k.col, "expected a statement, found '" + k.s + "'");
    if (k.s == "param") {
      for (;;) {
        Tok at = ps.peek();
        std::string n = ps.ident();
        declare(n, at);
        R.prm[n] = (int)p.params.size();
        p.params.push_back(n);
        if (ps.peek().s != ",") break;
        ps.next();
      }
    } else if (k.s == "image") {
      Tok at = ps.peek();
      ImageDecl d;
      d.name = ps.ident();
      declare(d.name, at);
      ps.expect("(");
      d.extents.push_back(ps.expr());
      while (ps.peek().s == ",") { ps.next(); d.extents.push_back(ps.expr()); }
      ps.expect(")");
      ps.expect(":");
      d.dtype = ps.dtype();
      if (d.extents.size() > 3) fail(at.line, at.col, "images have 1-3 dims");
      for (auto& x : d.extents) R.resolve(x, nullptr);
      R.img[d.name] = (int)p.images.size();
      p.images.push_back(d);
    } else if (k.s == "table") {
      Tok at = ps.peek();
      TableDecl d;
      d.name = ps.ident();
      declare(d.name, at);
      ps.expect("(");
      d.extent = ps.expr();
      ps.expect(")");
      ps.expect(":");
      d.dtype = ps.dtype();
      R.resolve(d.extent, nullptr);
      R.tab[d.name] = (int)p.tables.size();
      p.tables.push_back(d);
    } else if (k.s == "stage") {
      Tok at = ps.peek();
      StageDecl d;
      d.line = k.line;
      d.name = ps.ident();
      declare(d.name, at);
      ps.expect("(");
      d.vars.push_back(ps.ident());
      while (ps.peek().s == ",") { ps.next(); d.vars.push_back(ps.ident()); }
      ps.expect(")");
      ps.expect("[");
      d.extents.push_back(ps.expr());
      while (ps.peek().s == ",") { ps.next(); d.extents.push_back(ps.expr()); }
      ps.expect("]");
      ps.expect(":");
      d.dtype = ps.dtype();
      ps.expect("=");
      d.expr = ps.expr();
      if (d.vars.size() != d.extents.size() || d.vars.empty() || d.vars.size() > 3)
        fail(at.line, at.col, "stage " + d.name + ": " + std::to_string(d.vars.size()) + " variables but " +
                                  std::to_string(d.extents.size()) + " extents (1-3 dims)");
      for (auto& x : d.extents) R.resolve(x, nullptr);
      R.stg[d.name] = (int)p.stages.size();
      p.stages.push_back(d);
    } else if (k.s == "liveout") {
      for (;;) {
        Tok at = ps.peek();
        liveout_names.push_back({ps.ident(), at});
        if (ps.peek().s != ",") break;
        ps.next();
      }
    } else {
      fail(k.line, k.col, "unknown statement '" + k.s + "'");
    }
    ps.end_stmt();
  }
  if (p.stages.empty()) throw Error(PMG_ERR_PARSE, "no stages");
  if (liveout_names.empty()) throw Error(PMG_ERR_PARSE, "no liveouts");
  // resolve stage expressions after all declarations (forward references allowed; cycles checked below)
  for (auto& s : p.stages) R.resolve(s.expr, &s.vars);
  for (auto& [n, at] : liveout_names) {
    auto it = R.stg.find(n);
    if (it == R.stg.end()) fail(at.line, at.col, "liveout '" + n + "' is not a stage");
    if (std::find(p.liveouts.begin(), p.liveouts.end(), it->second) == p.liveouts.end()) p.liveouts.push_back(it->second);
  }
  const int n = (int)p.stages.size();
  p.producers.assign(n, {});
  p.consumers.assign(n, {});
  for (int s = 0; s < n; ++s) {
    std::vector<Expr*> acc;
    collect_accesses(p.stages[s].expr, acc);
    for (Expr* a : acc)
      if (a->is_stage && std::find(p.producers[s].begin(), p.producers[s].end(), a->index) == p.producers[s].end())
        p.producers[s].push_back(a->index);
  }
  for (int s = 0; s < n; ++s)
    for (int q : p.producers[s]) p.consumers[q].push_back(s);
  // cycles ("cyclic reference")
  std::vector<int> state(n, 0);
  std::function<void(int, std::vector<int>&)> visit = [&](int s, std::vector<int>& path) {
    if (state[s] == 1) {
      std::string m = "cyclic reference: ";
      for (int q : path) m += p.stages[q].name + " -> ";
      m += p.stages[s].name;
      throw Error(PMG_ERR_PARSE, m);
    }
    if (state[s] == 2) return;
    state[s] = 1;
    path.push_back(s);
    for (int q : p.producers[s]) visit(q, path);
    path.pop_back();
    state[s] = 2;
  };
  for (int s = 0; s < n; ++s) { std::vector<int> path; visit(s, path); }
  // reachability from liveouts
  std::vector<char> seen(n, 0);
  std::vector<int> todo(p.liveouts.begin(), p.liveouts.end());
  while (!todo.empty()) {
    int s = todo.back();
    todo.pop_back();
    if (seen[s]) continue;
    seen[s] = 1;
    for (int q : p.producers[s]) todo.push_back(q);
  }
  for (int s = 0; s < n; ++s)
    if (!seen[s]) throw Error(PMG_ERR_PARSE, "line " + std::to_string(p.stages[s].line) + ": stage '" + p.stages[s].name + "' is unreachable from every liveout");
  // topological order, ties by declaration order
  std::vector<char> done(n, 0);
  while ((int)p.topo.size() < n) {
    for (int s = 0; s < n; ++s) {
      if (done[s]) continue;
      bool ok = true;
      for (int q : p.producers[s]) ok = ok && done[q];
      if (ok) { p.topo.push_back(s); done[s] = 1; break; }
    }
  }
  return P;
}

}  // namespace pmg
