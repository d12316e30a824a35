// factor.cpp — separable evaluation of rank-1 linear stencils (pmg_sched_opts.reassoc = 1; a B200 option
// outside the paper, DESIGN.md §9 "Reassociation mode").
//
// A float stage whose expression is a linear combination of reads of ONE producer Q at constant offsets,
//     S(y, x) = (sum_{dy,dx} w[dy][dx] * Q(y+dy, x+dx)) (* or / constants),
// with a coefficient matrix of rank one, w[dy][dx] = u[dy] * v[dx], is rewritten as two stages
//     S_h(y, x) = sum_dx v[dx] * Q(y, x+dx)                (one row sum per row, reused by every reader row)
//     S(y, x)   = (sum_dy u[dy] * S_h(y+dy, x)) (* or / the same constants)
// — the Sobel derivatives and box sums of Harris: 8 -> 4 additions per box sum, 5 -> 3 operations per
// derivative.  Reads clamp per dimension (reading R1), so S_h(clamp(y+dy), x) holds exactly the values the
// original reads at row clamp(y+dy): the rewrite changes the association of the sum and nothing else.  It
// therefore changes f32 rounding (reading R3's written order is not kept); results stay within the
// north_star tolerance (|err| <= a few ulps of the sum of |terms|), which the reassociation parity tests check
// against the oracle on the pipeline as written.  Only applied when the rewritten form has fewer operations.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <map>
#include <set>

#include "analysis.hpp"
#include "ir.hpp"

namespace pmg {

using Hook = std::function<bool(const Expr&, std::string&)>;
std::string print_expr_text(const Pipeline& p, const std::vector<std::string>& vars, const Expr& e, const Hook* hook);
std::string print_pipeline_text(const Pipeline& p, const std::vector<std::string>& stage_lines,
                                const std::vector<std::string>& liveouts);

namespace {

struct Term { int dy, dx; double w; };

struct Lin {
  bool ok = true;
  const Expr* first = nullptr;   // first read (its plane index text is shared by every term)
  bool q_stage = false;
  int q = -1;
  std::vector<Term> terms;
};

// collect sign * scale * (linear form of e) into L; every read must be Q(plane, y+dy, x+dx) of one producer
void linear(const Analysis& A, const std::map<const Expr*, int>& site, const Expr& e, double scale, Lin& L) {
  if (!L.ok) return;
  if (e.kind != Kind::Float) { L.ok = false; return; }
  switch (e.op) {
    case Expr::ACCESS: {
      const ReadSite& r = A.reads[site.at(&e)];
      if (L.q < 0) { L.q = r.src; L.q_stage = r.src_is_stage; L.first = &e; }
      if (r.src != L.q || r.src_is_stage != L.q_stage || r.form[1] != Form::UNIT || r.form[2] != Form::UNIT ||
          !(r.form[0] == Form::ABSENT || (r.form[0] == Form::UNIT && r.off[0] == 0))) { L.ok = false; return; }
      L.terms.push_back({(int)r.off[1], (int)r.off[2], scale});
      return;
    }
    case Expr::UN:
      if (e.text == "-") { linear(A, site, *e.args[0], -scale, L); return; }
      break;
    case Expr::BIN:
      if (e.text == "+" || e.text == "-") {
        linear(A, site, *e.args[0], scale, L);
        linear(A, site, *e.args[1], e.text == "+" ? scale : -scale, L);
        return;
      }
      if (e.text == "*") {
        if (e.args[0]->op == Expr::FLT) { linear(A, site, *e.args[1], scale * e.args[0]->fval, L); return; }
        if (e.args[1]->op == Expr::FLT) { linear(A, site, *e.args[0], scale * e.args[1]->fval, L); return; }
      }
      break;
    default: break;
  }
  L.ok = false;
}

std::string coef_term(double c, const std::string& read, bool first) {
  // "+ read", "- read", "+ c * read"; a leading term keeps its sign as a unary minus
  const double a = std::fabs(c);
  std::string body = read;
  if (a != 1.0) {
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", a);
    std::string lit = b;
    if (lit.find_first_of(".eE") == std::string::npos) lit += ".0";
    body = "(" + lit + " * " + read + ")";
  }
  if (first) return c < 0 ? "(-" + body + ")" : body;
  return (c < 0 ? " - " : " + ") + body;
}

// number of operations of sum_i c_i * r_i written left to right (2^k multipliers fold into an exact fma)
int sum_ops(const std::vector<double>& c) {
  int n = 0, ops = 0;
  for (double x : c) {
    if (x == 0.0) continue;
    int e;
    const double m = std::frexp(std::fabs(x), &e);
    const bool unit = std::fabs(x) == 1.0, pow2 = m == 0.5 && e >= 1;
    ops += (n > 0 ? 1 : 0) + (unit || (pow2 && n > 0) ? 0 : 1);
    ++n;
  }
  return ops;
}

struct Cand {
  int s = -1;
  std::vector<int> dys, dxs;
  std::vector<double> u, v;
  std::vector<const Expr*> post;   // outer "* c" / "/ c" wrappers, innermost first
  Lin L;
};

bool factor(const Analysis& A, const std::map<const Expr*, int>& site, int s, Cand& c) {
  const Pipeline& p = *A.p;
  const StageDecl& sd = p.stages[s];
  if (sd.dtype != DType::F32 || sd.expr->kind != Kind::Float) return false;
  const Expr* e = sd.expr.get();
  std::vector<const Expr*> post;
  while (e->op == Expr::BIN && (e->text == "*" || e->text == "/") && e->args[1]->op == Expr::FLT &&
         e->args[0]->op == Expr::BIN && (e->args[0]->text == "+" || e->args[0]->text == "-")) {
    post.push_back(e);
    e = e->args[0].get();
  }
  std::reverse(post.begin(), post.end());
  Lin L;
  linear(A, site, *e, 1.0, L);
  if (!L.ok || L.terms.size() < 4) return false;
  // the row sums have the stage's extent: the producer must have it too (y, x), and a plane index must be
  // the stage's own plane variable
  const Ext3& qe = L.q_stage ? A.stage_ext[L.q] : A.image_ext[L.q];
  const Ext3& se = A.stage_ext[s];
  if (qe.e[1] != se.e[1] || qe.e[2] != se.e[2] || !se.has[1] || !se.has[2]) return false;
  if (qe.has[0] && !se.has[0]) return false;
  std::map<std::pair<int, int>, double> w;
  std::set<int> ys, xs;
  for (auto& t : L.terms) {
    w[{t.dy, t.dx}] += t.w;
    ys.insert(t.dy);
    xs.insert(t.dx);
  }
  c.dys.assign(ys.begin(), ys.end());
  c.dxs.assign(xs.begin(), xs.end());
  if (c.dys.size() < 2 || c.dxs.size() < 2) return false;
  auto W = [&](int dy, int dx) { auto it = w.find({dy, dx}); return it == w.end() ? 0.0 : it->second; };
  // v = the first non-zero row scaled so that its first non-zero entry is 1; u[dy] from that column
  int r0 = 0, j0 = 0;
  bool nz = false;
  for (int dy : c.dys) {
    for (int dx : c.dxs)
      if (W(dy, dx) != 0.0) { r0 = dy; j0 = dx; nz = true; break; }
    if (nz) break;
  }
  if (!nz) return false;
  const double a = W(r0, j0);
  c.v.clear();
  c.u.clear();
  for (int dx : c.dxs) c.v.push_back(W(r0, dx) / a);
  for (int dy : c.dys) c.u.push_back(W(dy, j0));
  for (size_t i = 0; i < c.u.size(); ++i)
    if (c.u[i] != 0.0) {
      if (c.u[i] < 0) {
        for (auto& x : c.u) x = -x;
        for (auto& x : c.v) x = -x;
      }
      break;
    }
  for (size_t i = 0; i < c.dys.size(); ++i)
    for (size_t j = 0; j < c.dxs.size(); ++j) {
      const double want = W(c.dys[i], c.dxs[j]), got = c.u[i] * c.v[j];
      if (std::fabs(want - got) > 1e-9 * std::max(std::fabs(want), 1e-30)) return false;
    }
  int nu = 0, nv = 0;
  for (double x : c.u) nu += x != 0.0;
  for (double x : c.v) nv += x != 0.0;
  if (nu < 2 || nv < 2) return false;
  std::vector<double> flat;
  for (auto& t : L.terms) flat.push_back(t.w);
  if (sum_ops(c.u) + sum_ops(c.v) >= sum_ops(flat)) return false;
  c.s = s;
  c.post = post;
  c.L = L;
  return true;
}

std::string offs(const std::string& var, int d) {
  if (d == 0) return var;
  return var + (d > 0 ? " + " : " - ") + std::to_string(std::abs(d));
}

std::string rewrite(const Analysis& A, const Cand& c, std::string* hname) {
  const Pipeline& p = *A.p;
  const StageDecl& sd = p.stages[c.s];
  const int nd = (int)sd.vars.size();
  const std::string& vy = sd.vars[nd - 2];
  const std::string& vx = sd.vars[nd - 1];
  std::set<std::string> names;
  for (auto& st : p.stages) names.insert(st.name);
  for (auto& im : p.images) names.insert(im.name);
  std::string h = sd.name + "_h";
  for (int k = 2; names.count(h); ++k) h = sd.name + "_h" + std::to_string(k);
  *hname = h;
  const std::string qn = c.L.q_stage ? p.stages[c.L.q].name : p.images[c.L.q].name;
  const int qnd = (int)c.L.first->args.size();
  const std::string plane = qnd == 3 ? print_expr_text(p, sd.vars, *c.L.first->args[0], nullptr) + ", " : "";
  std::string hs;
  bool first = true;
  for (size_t j = 0; j < c.dxs.size(); ++j) {
    if (c.v[j] == 0.0) continue;
    std::string t = coef_term(c.v[j], qn + "(" + plane + vy + ", " + offs(vx, c.dxs[j]) + ")", first);
    hs = first ? t : "(" + hs + t + ")";
    first = false;
  }
  // a unit 3-tap row sum (the box filters): neighbouring columns share a pair, (Q(x) + Q(x+1)) is the right pair
  // of column x and the left pair of column x+1, so even columns sum as Q(x-1) + (Q(x) + Q(x+1)) and odd ones as
  // (Q(x-1) + Q(x)) + Q(x+1).  The emitter resolves the parity select per element (lanes own an even number of
  // columns from an even origin) and the compiler computes each shared pair once: 6 additions per 4 columns
  // instead of 8.
  if (c.dxs.size() == 3 && c.dxs[0] == -1 && c.dxs[1] == 0 && c.dxs[2] == 1 && c.v[0] == 1.0 && c.v[1] == 1.0 && c.v[2] == 1.0) {
    auto q = [&](int dx) { return qn + "(" + plane + vy + ", " + offs(vx, dx) + ")"; };
    hs = "select(" + vx + " % 2 == 0, (" + q(-1) + " + (" + q(0) + " + " + q(1) + ")), ((" + q(-1) + " + " + q(0) + ") + " + q(1) + "))";
  }
  const std::string hplane = nd == 3 ? sd.vars[0] + ", " : "";
  std::string ss;
  first = true;
  for (size_t i = 0; i < c.dys.size(); ++i) {
    if (c.u[i] == 0.0) continue;
    std::string t = coef_term(c.u[i], h + "(" + hplane + offs(vy, c.dys[i]) + ", " + vx + ")", first);
    ss = first ? t : "(" + ss + t + ")";
    first = false;
  }
  for (const Expr* w : c.post) ss = "(" + ss + " " + w->text + " " + print_expr_text(p, {}, *w->args[1], nullptr) + ")";
  std::string ext;
  for (size_t i = 0; i < sd.extents.size(); ++i) ext += (i ? ", " : "") + print_expr_text(p, {}, *sd.extents[i], nullptr);
  std::string vs;
  for (size_t i = 0; i < sd.vars.size(); ++i) vs += (i ? ", " : "") + sd.vars[i];
  std::vector<std::string> lines;
  for (size_t s = 0; s < p.stages.size(); ++s) {
    const StageDecl& d = p.stages[s];
    std::string dv, de;
    for (size_t i = 0; i < d.vars.size(); ++i) dv += (i ? ", " : "") + d.vars[i];
    for (size_t i = 0; i < d.extents.size(); ++i) de += (i ? ", " : "") + print_expr_text(p, {}, *d.extents[i], nullptr);
    if ((int)s == c.s) {
      lines.push_back("stage " + h + "(" + vs + ") [" + ext + "]: f32 = " + hs);
      lines.push_back("stage " + d.name + "(" + vs + ") [" + ext + "]: f32 = " + ss);
    } else {
      lines.push_back("stage " + d.name + "(" + dv + ") [" + de + "]: " + dtype_name(d.dtype) + " = " +
                      print_expr_text(p, d.vars, *d.expr, nullptr));
    }
  }
  std::vector<std::string> lo;
  for (int s : p.liveouts) lo.push_back(p.stages[s].name);
  return print_pipeline_text(p, lines, lo);
}

}  // namespace

std::shared_ptr<Pipeline> factor_stencils(std::shared_ptr<Pipeline> p, const std::vector<int64_t>& params,
                                          std::vector<std::string>* factored) {
  std::set<std::string> done;
  for (int guard = 0; guard < 256; ++guard) {
    Analysis A = analyze(*p, params);
    std::map<const Expr*, int> site;
    for (size_t i = 0; i < A.reads.size(); ++i) site[A.reads[i].node] = (int)i;
    Cand c;
    bool found = false;
    for (int s : p->topo) {
      if (done.count(p->stages[s].name)) continue;
      Cand t;
      if (factor(A, site, s, t)) { c = t; found = true; break; }
    }
    if (!found) break;
    std::string h;
    done.insert(p->stages[c.s].name);
    std::string text = rewrite(A, c, &h);
    done.insert(h);
    if (factored) factored->push_back(p->stages[c.s].name);
    p = parse_pipeline(text);
  }
  return p;
}

}  // namespace pmg
