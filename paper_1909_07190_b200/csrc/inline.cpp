// inline.cpp — inlining of data-expanding stages into their consumers (a B200 design option: SURVEY A25
// "inlining is a B200 design option, not the method"; PAPER.md P:1426-1430 notes PolyMage cannot inline).
//
// A stage P that has more points than everything it reads together (the local Laplacian's 8 intensity planes
// gP0 = f(gray), the ×2 upsamplings gUx_j, lP_j = gP_j - up(gUx_j)) cannot share a fused group with consumers
// of another extent, so it would be written to HBM in full and read back — often only partly (outLP_j reads
// two of the eight planes).  Substituting P's expression into each read evaluates P only where it is read.
// The substitution is exact (reading R1): a read P(q) is P's expression at clamp(q, domain(P)); the clamp of
// coordinate d is dropped only when P uses its variable d solely as the same-position index of reads whose
// producers have P's extent in that dimension (they clamp identically), which keeps stencil index forms.
// Stored-value conversion is kept by a cast to P's dtype.  The oracle evaluates the pipeline as written, so
// every inlined plan is checked against the un-inlined definition.
#include <functional>
#include <set>
#include <sstream>

#include "../../include/pmg.h"
#include "analysis.hpp"
#include "ir.hpp"

namespace pmg {

namespace {

using Hook = std::function<bool(const Expr&, std::string&)>;   // replace a node's text (returns true)

std::string print(const Pipeline& p, const std::vector<std::string>& vars, const Expr& e, const Hook* hook) {
  std::string r;
  if (hook && (*hook)(e, r)) return r;
  auto args = [&](size_t from) {
    std::string s;
    for (size_t i = from; i < e.args.size(); ++i) s += (i > from ? ", " : "") + print(p, vars, *e.args[i], hook);
    return s;
  };
  switch (e.op) {
    case Expr::INT: return std::to_string(e.ival);
    case Expr::FLT: return e.text;
    case Expr::VAR: return vars.at(e.index);
    case Expr::PARAM: return p.params.at(e.index);
    case Expr::ACCESS: return (e.is_stage ? p.stages.at(e.index).name : p.images.at(e.index).name) + "(" + args(0) + ")";
    case Expr::TABLE: return p.tables.at(e.index).name + "[" + args(0) + "]";
    case Expr::BIN: return "(" + print(p, vars, *e.args[0], hook) + " " + e.text + " " + print(p, vars, *e.args[1], hook) + ")";
    case Expr::UN: return "(" + e.text + print(p, vars, *e.args[0], hook) + ")";
    case Expr::CALL: return e.text + "(" + args(0) + ")";
  }
  return "";
}

std::string print_ext(const Pipeline& p, const std::vector<ExprP>& ext) {
  std::string s;
  for (size_t i = 0; i < ext.size(); ++i) s += (i ? ", " : "") + print(p, {}, *ext[i], nullptr);
  return s;
}

std::string print_pipeline(const Pipeline& p, int drop, const std::vector<std::string>& exprs) {
  std::ostringstream o;
  if (!p.params.empty()) {
    o << "param ";
    for (size_t i = 0; i < p.params.size(); ++i) o << (i ? ", " : "") << p.params[i];
    o << "\n";
  }
  for (auto& im : p.images) o << "image " << im.name << "(" << print_ext(p, im.extents) << "): " << dtype_name(im.dtype) << "\n";
  for (auto& t : p.tables)
    o << "table " << t.name << "(" << print(p, {}, *t.extent, nullptr) << "): " << dtype_name(t.dtype) << "\n";
  for (size_t s = 0; s < p.stages.size(); ++s) {
    if ((int)s == drop) continue;
    auto& d = p.stages[s];
    o << "stage " << d.name << "(";
    for (size_t i = 0; i < d.vars.size(); ++i) o << (i ? ", " : "") << d.vars[i];
    o << ") [" << print_ext(p, d.extents) << "]: " << dtype_name(d.dtype) << " = " << exprs[s] << "\n";
  }
  o << "liveout ";
  for (size_t i = 0; i < p.liveouts.size(); ++i) o << (i ? ", " : "") << p.stages[p.liveouts[i]].name;
  o << "\n";
  return o.str();
}

int ops(const Expr& e) {
  if (e.op == Expr::ACCESS) return 0;
  int c = (e.op == Expr::BIN || e.op == Expr::UN || e.op == Expr::CALL || e.op == Expr::TABLE) ? 1 : 0;
  for (auto& a : e.args) c += ops(*a);
  return c;
}

int64_t domain(const Ext3& e) {
  int64_t n = 1;
  for (int d = 0; d < 3; ++d)
    if (e.has[d]) n *= e.e[d];
  return n;
}

// dims of stage P whose variable is used only as the same-position index of same-extent reads
std::vector<bool> bare_safe(const Analysis& A, int P) {
  const Pipeline& p = *A.p;
  const int nd = (int)p.stages[P].vars.size();
  std::vector<bool> safe(nd, true);
  const Ext3& pe = A.stage_ext[P];
  std::function<void(const Expr&, const Expr*, int)> walk = [&](const Expr& e, const Expr* parent, int pos) {
    if (e.op == Expr::VAR) {
      bool ok = parent && parent->op == Expr::ACCESS;
      if (ok) {
        const int qnd = (int)parent->args.size();
        const Ext3& qe = parent->is_stage ? A.stage_ext[parent->index] : A.image_ext[parent->index];
        const int qd = pos + 3 - qnd, pd = e.index + 3 - nd;
        ok = qe.e[qd] == pe.e[pd];
      }
      if (!ok) safe[e.index] = false;
      return;
    }
    for (size_t i = 0; i < e.args.size(); ++i) walk(*e.args[i], &e, (int)i);
  };
  walk(*p.stages[P].expr, nullptr, -1);
  return safe;
}

// one inlining candidate in topological order, or -1
int candidate(const Analysis& A) {
  const Pipeline& p = *A.p;
  for (int s : p.topo) {
    if (std::find(p.liveouts.begin(), p.liveouts.end(), s) != p.liveouts.end()) continue;
    if (ops(*p.stages[s].expr) > 64 || p.consumers[s].empty()) continue;
    int64_t in = 0;
    std::vector<Expr*> acc;
    collect_accesses(p.stages[s].expr, acc);
    std::set<std::pair<bool, int>> seen;
    for (Expr* a : acc)
      if (seen.insert({a->is_stage, a->index}).second)
        in += domain(a->is_stage ? A.stage_ext[a->index] : A.image_ext[a->index]);
    if (domain(A.stage_ext[s]) <= in) continue;             // not data-expanding
    bool ok = true;
    for (int c : p.consumers[s]) {
      std::vector<Expr*> ca;
      collect_accesses(p.stages[c].expr, ca);
      int reads = 0;
      for (Expr* a : ca) reads += a->is_stage && a->index == s;
      if (reads > 4 || ops(*p.stages[c].expr) + reads * ops(*p.stages[s].expr) > 200) ok = false;
    }
    if (ok) return s;
  }
  return -1;
}

std::string inline_one(const Analysis& A, int P) {
  const Pipeline& p = *A.p;
  const StageDecl& pd = p.stages[P];
  const std::vector<bool> safe = bare_safe(A, P);
  std::vector<std::string> exprs(p.stages.size());
  for (size_t c = 0; c < p.stages.size(); ++c) {
    const StageDecl& cd = p.stages[c];
    Hook hook = [&](const Expr& e, std::string& out) {
      if (e.op != Expr::ACCESS || !e.is_stage || e.index != P) return false;
      std::vector<std::string> sub(pd.vars.size());
      for (size_t d = 0; d < pd.vars.size(); ++d) {
        std::string q = print(p, cd.vars, *e.args[d], &hook);
        sub[d] = safe[d] ? "(" + q + ")" : "clamp(" + q + ", 0, (" + print(p, {}, *pd.extents[d], nullptr) + ") - 1)";
      }
      std::string body = print(p, sub, *pd.expr, nullptr);
      const bool fl = pd.expr->kind == Kind::Float;
      if (pd.dtype == DType::F32 && fl) out = "(" + body + ")";
      else out = std::string(dtype_name(pd.dtype)) + "(" + body + ")";
      return true;
    };
    exprs[c] = print(p, cd.vars, *cd.expr, &hook);
  }
  return print_pipeline(p, P, exprs);
}

}  // namespace

// text printing shared with phase.cpp (the rewrites produce pipeline text that is parsed again)
std::string print_expr_text(const Pipeline& p, const std::vector<std::string>& vars, const Expr& e, const Hook* hook) {
  return print(p, vars, e, hook);
}

std::string print_pipeline_text(const Pipeline& p, const std::vector<std::string>& stage_lines,
                                const std::vector<std::string>& liveouts) {
  std::ostringstream o;
  if (!p.params.empty()) {
    o << "param ";
    for (size_t i = 0; i < p.params.size(); ++i) o << (i ? ", " : "") << p.params[i];
    o << "\n";
  }
  for (auto& im : p.images) o << "image " << im.name << "(" << print_ext(p, im.extents) << "): " << dtype_name(im.dtype) << "\n";
  for (auto& t : p.tables)
    o << "table " << t.name << "(" << print(p, {}, *t.extent, nullptr) << "): " << dtype_name(t.dtype) << "\n";
  for (auto& l : stage_lines) o << l << "\n";
  o << "liveout ";
  for (size_t i = 0; i < liveouts.size(); ++i) o << (i ? ", " : "") << liveouts[i];
  o << "\n";
  return o.str();
}

std::shared_ptr<Pipeline> inline_expanding(std::shared_ptr<Pipeline> p, const std::vector<int64_t>& params,
                                           std::vector<std::string>* inlined) {
  for (int guard = 0; guard < 256; ++guard) {
    Analysis A = analyze(*p, params);
    int s = candidate(A);
    if (s < 0) break;
    if (inlined) inlined->push_back(p->stages[s].name);
    std::string text = inline_one(A, s);
    p = parse_pipeline(text);
  }
  return p;
}

}  // namespace pmg
