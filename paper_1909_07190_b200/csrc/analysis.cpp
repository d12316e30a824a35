// analysis.cpp — footprints / dependence vectors (§2.3: "the difference of the time
// stamps when a value is consumed and when it is produced"), alignment & scaling forms (§5:
// index forms v+b, 2v+b, (v+b)/2 — DESIGN.md reading R10), and the §4 warp geometry (lines 576-580).
#include "analysis.hpp"

#include <algorithm>
#include <sstream>

#include "../../include/pmg.h"

namespace pmg {

static int64_t fdiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b) && ((a < 0) != (b < 0))) --q;
  return q;
}

namespace {

// affine form over the consumer's normalised vars: sum coef[d]*v_d + c
struct Lin {
  bool ok = true;
  int64_t coef[3] = {0, 0, 0};
  int64_t c = 0;
};

Lin linear(const Expr& e, int cons_nd, const std::vector<int64_t>& params) {
  Lin r;
  switch (e.op) {
    case Expr::INT: r.c = e.ival; return r;
    case Expr::PARAM: r.c = params.at(e.index); return r;
    case Expr::VAR: r.coef[e.index + (3 - cons_nd)] = 1; return r;
    case Expr::UN:
      if (e.text == "-") {
        r = linear(*e.args[0], cons_nd, params);
        for (auto& k : r.coef) k = -k;
        r.c = -r.c;
        return r;
      }
      break;
    case Expr::BIN: {
      if (e.text == "+" || e.text == "-") {
        Lin a = linear(*e.args[0], cons_nd, params), b = linear(*e.args[1], cons_nd, params);
        if (!a.ok || !b.ok) break;
        int s = e.text == "+" ? 1 : -1;
        for (int d = 0; d < 3; ++d) r.coef[d] = a.coef[d] + s * b.coef[d];
        r.c = a.c + s * b.c;
        return r;
      }
      if (e.text == "*") {
        Lin a = linear(*e.args[0], cons_nd, params), b = linear(*e.args[1], cons_nd, params);
        if (!a.ok || !b.ok) break;
        bool ac = !a.coef[0] && !a.coef[1] && !a.coef[2], bc = !b.coef[0] && !b.coef[1] && !b.coef[2];
        if (ac) { for (int d = 0; d < 3; ++d) r.coef[d] = a.c * b.coef[d]; r.c = a.c * b.c; return r; }
        if (bc) { for (int d = 0; d < 3; ++d) r.coef[d] = b.c * a.coef[d]; r.c = a.c * b.c; return r; }
      }
      break;
    }
    default: break;
  }
  r.ok = false;
  return r;
}

bool only_dim(const Lin& l, int d) {
  for (int k = 0; k < 3; ++k)
    if (k != d && l.coef[k] != 0) return false;
  return true;
}

void classify(const Expr& idx, int pd /*producer normalised dim*/, int cons_nd, const Ext3& cons,
              const std::vector<int64_t>& params, Form& f, int64_t& off) {
  off = 0;
  if (is_const_int(idx)) { f = Form::CONST; off = eval_int(idx, params); return; }
  // (lin)/2 with lin = v + b  -> UP2
  if (idx.op == Expr::BIN && idx.text == "/" && idx.args[1]->op == Expr::INT && idx.args[1]->ival == 2) {
    Lin l = linear(*idx.args[0], cons_nd, params);
    if (l.ok && only_dim(l, pd) && l.coef[pd] == 1 && cons.has[pd]) { f = Form::UP2; off = l.c; return; }
  }
  Lin l = linear(idx, cons_nd, params);
  if (l.ok && only_dim(l, pd) && cons.has[pd]) {
    if (l.coef[pd] == 1) { f = Form::UNIT; off = l.c; return; }
    if (l.coef[pd] == 2) { f = Form::DOWN2; off = l.c; return; }
  }
  f = Form::GENERAL;
}

const char* form_name(Form f) {
  switch (f) {
    case Form::ABSENT: return "absent";
    case Form::UNIT: return "unit";
    case Form::DOWN2: return "down2";
    case Form::UP2: return "up2";
    case Form::CONST: return "const";
    default: return "general";
  }
}

Ext3 norm_ext(const std::vector<ExprP>& ext, const std::vector<int64_t>& params, const std::string& name) {
  Ext3 r;
  int nd = (int)ext.size();
  for (int i = 0; i < nd; ++i) {
    int d = i + 3 - nd;
    r.e[d] = eval_int(*ext[i], params);
    r.has[d] = true;
    if (r.e[d] < 1) throw Error(PMG_ERR_SHAPE, name + ": empty domain (extent " + std::to_string(r.e[d]) + ")");
    if (r.e[d] > (int64_t(1) << 30)) throw Error(PMG_ERR_SHAPE, name + ": extent too large");
  }
  return r;
}

}  // namespace

Analysis analyze(const Pipeline& p, const std::vector<int64_t>& params) {
  if (params.size() != p.params.size())
    throw Error(PMG_ERR_ARG, "expected " + std::to_string(p.params.size()) + " parameter values, got " + std::to_string(params.size()));
  Analysis A;
  A.p = &p;
  A.params = params;
  for (auto& s : p.stages) A.stage_ext.push_back(norm_ext(s.extents, params, s.name));
  for (auto& im : p.images) A.image_ext.push_back(norm_ext(im.extents, params, im.name));
  for (auto& t : p.tables) {
    int64_t n = eval_int(*t.extent, params);
    if (n < 1) throw Error(PMG_ERR_SHAPE, t.name + ": empty table");
    A.table_len.push_back(n);
  }
  A.reads_of.assign(p.stages.size(), {});
  for (size_t s = 0; s < p.stages.size(); ++s) {
    std::vector<Expr*> acc;
    collect_accesses(p.stages[s].expr, acc);
    int cnd = (int)p.stages[s].vars.size();
    for (Expr* a : acc) {
      ReadSite r;
      r.consumer = (int)s;
      r.src_is_stage = a->is_stage;
      r.src = a->index;
      r.node = a;
      int pnd = (int)a->args.size();
      for (int i = 0; i < pnd; ++i) {
        int pd = i + 3 - pnd;
        classify(*a->args[i], pd, cnd, A.stage_ext[s], params, r.form[pd], r.off[pd]);
      }
      A.reads_of[s].push_back((int)A.reads.size());
      A.reads.push_back(r);
    }
  }
  return A;
}

// algorithmic operation count of an expression as written (roofline numerator)
static int alg_ops(const Expr& e) {
  int c = 0;
  if (e.op == Expr::ACCESS) return 0;   // index expressions are coordinates, not the stage's arithmetic
  for (auto& a : e.args) c += alg_ops(*a);
  switch (e.op) {
    case Expr::BIN: case Expr::UN: return c + 1;
    case Expr::CALL:
      if (e.text == "lerp") return c + 3;
      if (e.text == "clamp" || e.text == "absd") return c + 2;
      return c + 1;
    default: return c;
  }
}

std::string describe_pipeline(const Analysis& A) {
  const Pipeline& p = *A.p;
  std::ostringstream o;
  o << "{\"stages\":[";
  for (size_t s = 0; s < p.stages.size(); ++s) {
    auto& e = A.stage_ext[s];
    o << (s ? "," : "") << "{\"name\":\"" << p.stages[s].name << "\",\"dtype\":\"" << dtype_name(p.stages[s].dtype)
      << "\",\"extent\":[" << e.e[0] << "," << e.e[1] << "," << e.e[2] << "],\"ndim\":" << p.stages[s].vars.size()
      << ",\"ops\":" << alg_ops(*p.stages[s].expr) << "}";
  }
  o << "],\"topo\":[";
  for (size_t i = 0; i < p.topo.size(); ++i) o << (i ? "," : "") << "\"" << p.stages[p.topo[i]].name << "\"";
  o << "],\"reads\":[";
  for (size_t i = 0; i < A.reads.size(); ++i) {
    auto& r = A.reads[i];
    o << (i ? "," : "") << "{\"consumer\":\"" << p.stages[r.consumer].name << "\",\"producer\":\""
      << (r.src_is_stage ? p.stages[r.src].name : p.images[r.src].name) << "\",\"producer_is_stage\":"
      << (r.src_is_stage ? "true" : "false") << ",\"form\":[";
    for (int d = 0; d < 3; ++d) o << (d ? "," : "") << "\"" << form_name(r.form[d]) << "\"";
    o << "],\"offset\":[";
    for (int d = 0; d < 3; ++d) o << (d ? "," : "") << r.off[d];
    o << "]}";
  }
  o << "]}";
  return o.str();
}

std::array<int, 3> warp_sizes(const std::array<int, 3>& B, int ws) {
  // W_x = min(B_x, WarpSize); W_y = min(B_y, WarpSize / W_x); W_z = min(B_z, WarpSize / (W_x W_y))
  std::array<int, 3> W;
  W[0] = std::min(B[0], ws);
  W[1] = std::min(B[1], ws / W[0]);
  W[2] = std::min(B[2], ws / (W[0] * W[1]));
  return W;
}

// interval of an integer index expression over a box of consumer coordinates (conservative; false = unknown).
// Used for "general" row indices such as the pyramid upsample y/2 - 1 + 2*(y%2).
static bool int_interval(const Expr& e, const int64_t lo[3], const int64_t hi[3], int cons_nd,
                         const std::vector<int64_t>& params, int64_t& a, int64_t& b) {
  if (e.kind != Kind::Int) return false;
  int64_t a0, b0, a1, b1, a2, b2;
  auto sub = [&](int i, int64_t& x, int64_t& y) { return int_interval(*e.args[i], lo, hi, cons_nd, params, x, y); };
  switch (e.op) {
    case Expr::INT: a = b = e.ival; return true;
    case Expr::PARAM: a = b = params.at(e.index); return true;
    case Expr::VAR: { int d = e.index + (3 - cons_nd); a = lo[d]; b = hi[d]; return true; }
    case Expr::UN:
      if (e.text != "-" || !sub(0, a0, b0)) return false;
      a = -b0; b = -a0;
      return true;
    case Expr::BIN: {
      if (!sub(0, a0, b0) || !sub(1, a1, b1)) return false;
      const std::string& t = e.text;
      if (t == "+") { a = a0 + a1; b = b0 + b1; return true; }
      if (t == "-") { a = a0 - b1; b = b0 - a1; return true; }
      if (t == "*") {
        int64_t c[4] = {a0 * a1, a0 * b1, b0 * a1, b0 * b1};
        a = *std::min_element(c, c + 4); b = *std::max_element(c, c + 4);
        return true;
      }
      if (t == "/" && a1 == b1 && a1 > 0) { a = fdiv(a0, a1); b = fdiv(b0, a1); return true; }   // floor division
      if (t == "%" && a1 == b1 && a1 > 0) {                                                       // non-negative
        const int64_t m = a1, ra = a0 - fdiv(a0, m) * m, rb = b0 - fdiv(b0, m) * m;
        if (b0 - a0 + 1 < m && ra <= rb) { a = ra; b = rb; } else { a = 0; b = m - 1; }
        return true;
      }
      return false;
    }
    case Expr::CALL: {
      const std::string& f = e.text;
      if ((f == "min" || f == "max") && sub(0, a0, b0) && sub(1, a1, b1)) {
        if (f == "min") { a = std::min(a0, a1); b = std::min(b0, b1); } else { a = std::max(a0, a1); b = std::max(b0, b1); }
        return true;
      }
      if (f == "clamp" && sub(0, a0, b0) && sub(1, a1, b1) && sub(2, a2, b2)) {   // min(max(x, l), h)
        a = std::min(std::max(a0, a1), a2);
        b = std::min(std::max(b0, b1), b2);
        return true;
      }
      if (f == "select" && sub(1, a1, b1) && sub(2, a2, b2)) { a = std::min(a1, a2); b = std::max(b1, b2); return true; }
      if (f == "i32" && sub(0, a0, b0)) { a = a0; b = b0; return true; }
      return false;
    }
    default: return false;
  }
}

RowIv rows_needed(const Analysis& A, const ReadSite& r, RowIv cr, int64_t src_rows) {
  RowIv out{0, src_rows};
  if (cr.hi <= cr.lo) return RowIv{0, 0};
  if (r.form[1] == Form::GENERAL) {
    // interval analysis of the row index over the consumer's rows (other dims: their whole extent)
    const Ext3& ce = A.stage_ext[r.consumer];
    const int cnd = (int)A.p->stages[r.consumer].vars.size(), pnd = (int)r.node->args.size();
    int64_t lo[3], hi[3];
    for (int d = 0; d < 3; ++d) { lo[d] = 0; hi[d] = ce.e[d] - 1; }
    lo[1] = cr.lo;
    hi[1] = cr.hi - 1;
    int64_t a, b;
    if (pnd >= 2 && int_interval(*r.node->args[pnd - 2], lo, hi, cnd, A.params, a, b)) {
      out.lo = std::max<int64_t>(0, std::min(a, src_rows - 1));
      out.hi = std::min<int64_t>(src_rows, std::max(b + 1, out.lo + 1));
      return out;
    }
    return RowIv{0, src_rows};
  }
  switch (r.form[1]) {
    case Form::UNIT: out = {cr.lo + r.off[1], cr.hi - 1 + r.off[1] + 1}; break;
    case Form::DOWN2: out = {2 * cr.lo + r.off[1], 2 * (cr.hi - 1) + r.off[1] + 1}; break;
    case Form::UP2: out = {fdiv(cr.lo + r.off[1], 2), fdiv(cr.hi - 1 + r.off[1], 2) + 1}; break;
    case Form::ABSENT: out = {0, 1}; break;
    default: out = {0, src_rows}; break;   // CONST / GENERAL: whole producer (conservative)
  }
  out.lo = std::max<int64_t>(0, std::min(out.lo, src_rows - 1));
  out.hi = std::min<int64_t>(src_rows, std::max(out.hi, out.lo + 1));
  return out;
}

}  // namespace pmg
