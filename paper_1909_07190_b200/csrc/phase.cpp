// phase.cpp — alignment & scaling of downsampling edges by phase splitting (§5: fusion
// across scaled dependences "after PolyMage's alignment and scaling to make the dependence vectors constant";
// Alg. 2: a group is infeasible only when its dependences stay non-constant after that step).
//
// A stage S whose every reader indexes a dimension d as 2*v + b (v: the reader's own variable of d; the reader's
// extent is exactly half of S's) is read at the reader's resolution only through its two phases
//     S_e(.., v', ..) = S(.., 2v', ..)        S_o(.., v', ..) = S(.., 2v' + 1, ..)
// each a stage at the reader's extent in d.  The read S(2v + b) becomes a unit read of one phase at v + q, with
// q = floor(b / 2), p = b mod 2:  p = 0 -> S_e(v + q),  p = 1 -> S_o(v + q).  Reading R1 clamps the original
// read to [0, 2n); the phases clamp to [0, n), which differs exactly at one edge each, fixed by a select on the
// reader's own coordinate:
//     p = 0, q >= 1:   2v + b > 2n - 1  when v + q >= n, where S(2n - 1) = S_o(n - 1) = S_o(clamp(v + q))
//     p = 1, q <= -1:  2v + b < 0       when v + q < 0,  where S(0) = S_e(0) = S_e(clamp(v + q))
// (p = 0 at the low edge gives S_e(0) = S(0) and p = 1 at the high edge S_o(n - 1) = S(2n - 1) by themselves.)
// The rewrite is exact, so the reader and both phases have equal extents in d and constant dependences: the
// DP can fuse them (e.g. the local Laplacian's x-then-y downsample pairs gDx_j -> gP_j, the camera's denoise ->
// deinterleave).  The oracle evaluates the pipeline as written, so every plan built from a split pipeline is
// checked against the unsplit definition (tests/test_capi.py and every GPU parity test).
#include <functional>
#include <set>
#include <sstream>

#include "../../include/pmg.h"
#include "analysis.hpp"
#include "ir.hpp"

namespace pmg {

std::string print_expr_text(const Pipeline& p, const std::vector<std::string>& vars, const Expr& e,
                            const std::function<bool(const Expr&, std::string&)>* hook);
std::string print_pipeline_text(const Pipeline& p, const std::vector<std::string>& stage_lines_in_order,
                                const std::vector<std::string>& liveouts);

namespace {

// affine v + b in the variable with index `vi` (VAR, INT, + and - only); false otherwise
bool affine_var(const Expr& e, int vi, int64_t& coef, int64_t& c) {
  if (e.op == Expr::VAR) { coef = e.index == vi ? 1 : 0; c = 0; return e.index == vi; }
  if (e.op == Expr::INT) { coef = 0; c = e.ival; return true; }
  if (e.op == Expr::BIN && (e.text == "+" || e.text == "-") && e.kind == Kind::Int) {
    int64_t a1, c1, a2, c2;
    if (!affine_var(*e.args[0], vi, a1, c1) || !affine_var(*e.args[1], vi, a2, c2)) return false;
    coef = e.text == "+" ? a1 + a2 : a1 - a2;
    c = e.text == "+" ? c1 + c2 : c1 - c2;
    return true;
  }
  return false;
}

struct Split { int s = -1; int d = -1; std::string ext; };   // stage, normalised dim (1 = y, 2 = x), half extent text

Split candidate(const Analysis& A) {
  const Pipeline& p = *A.p;
  for (int s : p.topo) {
    if (std::find(p.liveouts.begin(), p.liveouts.end(), s) != p.liveouts.end() || p.consumers[s].empty()) continue;
    const Ext3& se = A.stage_ext[s];
    const int nd = (int)p.stages[s].vars.size();
    for (int d = 1; d <= 2; ++d) {
      if (!se.has[d] || se.e[d] < 2 || se.e[d] % 2) continue;
      bool ok = true;
      std::string ext;
      for (const ReadSite& r : A.reads) {
        if (!r.src_is_stage || r.src != s) continue;
        const Ext3& ce = A.stage_ext[r.consumer];
        if (r.form[d] != Form::DOWN2 || !ce.has[d] || 2 * ce.e[d] != se.e[d]) { ok = false; break; }
        const StageDecl& cd = p.stages[r.consumer];
        const int cnd = (int)cd.vars.size();
        std::string x = print_expr_text(p, {}, *cd.extents[d - (3 - cnd)], nullptr);
        if (!ext.empty() && ext != x) { ok = false; break; }   // every reader must spell the same half extent
        ext = x;
      }
      (void)nd;
      if (ok && !ext.empty()) return {s, d, ext};
    }
  }
  return {};
}

std::string split_one(const Analysis& A, const Split& sp) {
  const Pipeline& p = *A.p;
  const StageDecl& sd = p.stages[sp.s];
  const int snd = (int)sd.vars.size();
  const int sdim = sp.d - (3 - snd);                  // S's own index of dim d
  const std::string suf = sp.d == 1 ? "_y" : "_x";
  const std::string ne = sd.name + suf + "e", no = sd.name + suf + "o";
  std::vector<std::string> lines;
  using Hook = std::function<bool(const Expr&, std::string&)>;
  for (size_t c = 0; c < p.stages.size(); ++c) {
    const StageDecl& cd = p.stages[c];
    const int cnd = (int)cd.vars.size();
    Hook hook = [&](const Expr& e, std::string& out) {
      if (e.op != Expr::ACCESS || !e.is_stage || e.index != sp.s) return false;
      // the reader's index of dim d is 2*v + b (analysis Form::DOWN2); b from the ReadSite of this node
      int64_t b = 0;
      for (const ReadSite& r : A.reads)
        if (r.node == &e) b = r.off[sp.d];
      const int64_t q = b >= 0 ? b / 2 : -((-b + 1) / 2), ph = b - 2 * q;
      const std::string v = cd.vars.at(sp.d - (3 - cnd));
      const std::string vq = "(" + v + (q >= 0 ? " + " : " - ") + std::to_string(q >= 0 ? q : -q) + ")";
      auto read = [&](const std::string& name) {
        std::string a;
        for (size_t i = 0; i < e.args.size(); ++i)
          a += (i ? ", " : "") + ((int)i == sdim ? vq : print_expr_text(p, cd.vars, *e.args[i], &hook));
        return name + "(" + a + ")";
      };
      if (ph == 0 && q >= 1) out = "select(" + vq + " >= (" + sp.ext + "), " + read(no) + ", " + read(ne) + ")";
      else if (ph == 1 && q <= -1) out = "select(" + vq + " < 0, " + read(ne) + ", " + read(no) + ")";
      else out = read(ph == 0 ? ne : no);
      return true;
    };
    std::string ext;
    for (size_t i = 0; i < cd.extents.size(); ++i) ext += (i ? ", " : "") + print_expr_text(p, {}, *cd.extents[i], nullptr);
    if ((int)c == sp.s) {
      // the two phases replace S: S's expression with its variable of dim d at 2v' (+1), extent halved
      std::string pext;
      for (int i = 0; i < snd; ++i)
        pext += (i ? ", " : "") + (i == sdim ? sp.ext : print_expr_text(p, {}, *sd.extents[i], nullptr));
      for (int ph = 0; ph < 2; ++ph) {
        std::vector<std::string> sub = sd.vars;
        sub[sdim] = "(2 * " + sd.vars[sdim] + (ph ? " + 1)" : ")");
        std::string vs;
        for (int i = 0; i < snd; ++i) vs += (i ? ", " : "") + sd.vars[i];
        // parity forms of the split variable simplify exactly: (2v' + ph + c) / 2 = v' + floor((ph + c) / 2) and
        // (2v' + ph + c) % 2 = (ph + c) mod 2 (floor division, non-negative remainder: reading R4)
        Hook simp = [&](const Expr& e, std::string& out) {
          if (e.op == Expr::BIN && (e.text == "/" || e.text == "%") && e.args[1]->op == Expr::INT && e.args[1]->ival == 2) {
            int64_t a, c;
            if (affine_var(*e.args[0], sdim, a, c) && a == 1) {
              const int64_t t = ph + c, q = t >= 0 ? t / 2 : -((-t + 1) / 2);
              out = e.text == "/" ? "(" + sd.vars[sdim] + (q >= 0 ? " + " : " - ") + std::to_string(q >= 0 ? q : -q) + ")"
                                  : "(" + std::to_string(t - 2 * q) + ")";
              return true;
            }
          }
          return false;
        };
        lines.push_back("stage " + (ph ? no : ne) + "(" + vs + ") [" + pext + "]: " + dtype_name(sd.dtype) + " = " +
                        print_expr_text(p, sub, *sd.expr, &simp));
      }
      continue;
    }
    std::string vs;
    for (int i = 0; i < cnd; ++i) vs += (i ? ", " : "") + cd.vars[i];
    lines.push_back("stage " + cd.name + "(" + vs + ") [" + ext + "]: " + dtype_name(cd.dtype) + " = " +
                    print_expr_text(p, cd.vars, *cd.expr, &hook));
  }
  std::vector<std::string> lo;
  for (int s : p.liveouts) lo.push_back(p.stages[s].name);
  return print_pipeline_text(p, lines, lo);
}

// ---- upsampling edges: split the readers ----------------------------------------------------------------------
// A stage C whose variable v of dim d appears only inside (v + b) / 2 and (v + b) % 2 (the camera's parity
// interleave R(y, x) = select(y % 2 == 0, .. r(y / 2, x / 2) ..)) is evaluated at full resolution only to pick
// one of its coarse producers by parity.  Its two phases C_p(v') = C(2v' + p) read them at unit forms:
// (2v' + p + b) / 2 = v' + floor((p + b) / 2), (2v' + p + b) % 2 = (p + b) mod 2 (floor division, reading R4).
// Every reader D of C must then be split too (D_p reads C(2v' + p + b) = C_{(p+b) mod 2}(v' + floor((p+b)/2)),
// with the same edge selects as above), down to the liveouts, each of which is rebuilt under its own name as
// L(v) = select(v % 2 == 0, L_e(v / 2), L_o(v / 2)).  Both dims are split at once when both qualify, so a 2x2
// interleave becomes four quad-resolution phases and one final interleave.

static bool affine(const Expr& e, int vi, int64_t& coef, int64_t& c) { return affine_var(e, vi, coef, c); }

// v (index vi) occurs only inside (v + b) / 2 or (v + b) % 2; *any set when such a form occurs
static bool parity_only(const Expr& e, int vi, bool* any) {
  if (e.op == Expr::BIN && (e.text == "/" || e.text == "%") && e.args[1]->op == Expr::INT && e.args[1]->ival == 2) {
    int64_t a, c;
    if (affine(*e.args[0], vi, a, c) && a == 1) { *any = true; return true; }
  }
  if (e.op == Expr::VAR) return e.index != vi;
  for (auto& x : e.args)
    if (!parity_only(*x, vi, any)) return false;
  return true;
}

struct Up { int c = -1; bool dim[3] = {false, false, false}; std::set<int> set; };

Up up_candidate(const Analysis& A, const std::set<std::string>& interleaves) {
  const Pipeline& p = *A.p;
  for (int c : p.topo) {
    if (interleaves.count(p.stages[c].name)) continue;
    const StageDecl& cd = p.stages[c];
    const int nd = (int)cd.vars.size();
    Up u;
    bool anyd = false;
    for (int d = 1; d <= 2; ++d) {
      const int vi = d - (3 - nd);
      if (vi < 0 || A.stage_ext[c].e[d] < 2 || A.stage_ext[c].e[d] % 2) continue;
      bool any = false;
      if (parity_only(*cd.expr, vi, &any) && any) { u.dim[d] = true; anyd = true; }
    }
    if (!anyd) continue;
    // closure: every reader of a member, and every stage a member reads at unit forms that is itself parity-only in
    // the split dims (the camera's G and B next to R); every read of a member along a split dim must be a unit
    // form of the same extent
    auto parity_in_dims = [&](int s) {
      const int snd = (int)p.stages[s].vars.size();
      for (int d = 1; d <= 2; ++d) {
        if (!u.dim[d]) continue;
        const int vi = d - (3 - snd);
        bool any = false;
        if (vi < 0 || A.stage_ext[s].e[d] != A.stage_ext[c].e[d] || !parity_only(*p.stages[s].expr, vi, &any) || !any) return false;
      }
      return true;
    };
    std::vector<int> work{c};
    u.set.insert(c);
    bool ok = true;
    while (!work.empty() && ok) {
      int s = work.back();
      work.pop_back();
      for (const ReadSite& r : A.reads) {
        if (r.src_is_stage && r.src == s) {
          for (int d = 1; d <= 2; ++d)
            if (u.dim[d] && (r.form[d] != Form::UNIT || !(A.stage_ext[r.consumer].e[d] == A.stage_ext[s].e[d]))) ok = false;
          if (u.set.insert(r.consumer).second) work.push_back(r.consumer);
        }
        if (r.consumer == s && r.src_is_stage && !u.set.count(r.src) && !interleaves.count(p.stages[r.src].name)) {
          bool unit = true;
          for (int d = 1; d <= 2; ++d)
            if (u.dim[d] && r.form[d] != Form::UNIT) unit = false;
          if (unit && parity_in_dims(r.src) && u.set.insert(r.src).second) work.push_back(r.src);
        }
      }
    }
    if (ok && u.set.size() <= 12) { u.c = c; return u; }
  }
  return {};
}

std::string up_split(const Analysis& A, const Up& u, std::set<std::string>* interleaves) {
  const Pipeline& p = *A.p;
  using Hook = std::function<bool(const Expr&, std::string&)>;
  std::vector<int> ds;
  for (int d = 1; d <= 2; ++d)
    if (u.dim[d]) ds.push_back(d);
  const int nph = 1 << ds.size();
  auto suffix = [&](int ph) {
    std::string r;
    for (size_t i = 0; i < ds.size(); ++i) r += std::string(ds[i] == 1 ? "_y" : "_x") + ((ph >> i) & 1 ? "o" : "e");
    return r;
  };
  std::vector<std::string> lines;
  for (size_t sidx = 0; sidx < p.stages.size(); ++sidx) {
    const StageDecl& sd = p.stages[sidx];
    const int nd = (int)sd.vars.size();
    std::string vs;
    for (int i = 0; i < nd; ++i) vs += (i ? ", " : "") + sd.vars[i];
    const bool member = u.set.count((int)sidx) > 0;
    if (!member) {   // unchanged text (no member is read outside the set)
      std::string ext;
      for (size_t i = 0; i < sd.extents.size(); ++i) ext += (i ? ", " : "") + print_expr_text(p, {}, *sd.extents[i], nullptr);
      lines.push_back("stage " + sd.name + "(" + vs + ") [" + ext + "]: " + dtype_name(sd.dtype) + " = " +
                      print_expr_text(p, sd.vars, *sd.expr, nullptr));
      continue;
    }
    std::string hext;   // extents with the split dims halved
    for (int i = 0; i < nd; ++i) {
      const int d = i + 3 - nd;
      std::string x = print_expr_text(p, {}, *sd.extents[i], nullptr);
      hext += (i ? ", " : "") + (d >= 1 && u.dim[d] ? "((" + x + ") / 2)" : x);
    }
    for (int ph = 0; ph < nph; ++ph) {
      int pv[3] = {0, 0, 0};
      for (size_t i = 0; i < ds.size(); ++i) pv[ds[i]] = (ph >> i) & 1;
      Hook hook = [&](const Expr& e, std::string& out) {
        // parity forms of a split variable
        if (e.op == Expr::BIN && (e.text == "/" || e.text == "%") && e.args[1]->op == Expr::INT && e.args[1]->ival == 2) {
          for (int d : ds) {
            const int vi = d - (3 - nd);
            int64_t a, c;
            if (vi >= 0 && affine(*e.args[0], vi, a, c) && a == 1) {
              const int64_t t = pv[d] + c, q = t >= 0 ? t / 2 : -((-t + 1) / 2);
              out = e.text == "/" ? "(" + sd.vars[vi] + (q >= 0 ? " + " : " - ") + std::to_string(q >= 0 ? q : -q) + ")"
                                  : "(" + std::to_string(t - 2 * q) + ")";
              return true;
            }
          }
        }
        if (e.op == Expr::VAR) {
          for (int d : ds)
            if (e.index == d - (3 - nd)) {
              out = "(2 * " + sd.vars[e.index] + " + " + std::to_string(pv[d]) + ")";
              return true;
            }
          return false;
        }
        // reads of members: unit forms along the split dims -> one phase of the member (edge selects as for
        // downsampling, generalised to several dims by nesting)
        if (e.op == Expr::ACCESS && e.is_stage && u.set.count(e.index)) {
          const StageDecl& md = p.stages[e.index];
          const int mnd = (int)md.vars.size();
          int64_t b[3] = {0, 0, 0};
          for (const ReadSite& r : A.reads)
            if (r.node == &e)
              for (int d = 0; d < 3; ++d) b[d] = r.off[d];
          std::string idx[3];
          int64_t qd[3] = {0, 0, 0}, pd[3] = {0, 0, 0};
          for (int d : ds) {
            const int64_t t = pv[d] + b[d];
            qd[d] = t >= 0 ? t / 2 : -((-t + 1) / 2);
            pd[d] = t - 2 * qd[d];
          }
          // the phase read at v' + q in every split dim; other index args printed as they are
          auto read = [&](const int phs[3]) {
            std::string nm = md.name;
            for (int d : ds) nm += std::string(d == 1 ? "_y" : "_x") + (phs[d] ? "o" : "e");
            std::string a;
            for (int i = 0; i < mnd; ++i) {
              const int d = i + 3 - mnd;
              std::string arg;
              if (d >= 1 && u.dim[d]) {
                const std::string v = sd.vars[d - (3 - nd)];
                arg = "(" + v + (qd[d] >= 0 ? " + " : " - ") + std::to_string(qd[d] >= 0 ? qd[d] : -qd[d]) + ")";
              } else {
                arg = print_expr_text(p, sd.vars, *e.args[i], &hook);
              }
              a += (i ? ", " : "") + arg;
            }
            return nm + "(" + a + ")";
          };
          // nested edge selects, one split dim at a time
          std::function<std::string(size_t, int*)> build = [&](size_t k, int* phs) -> std::string {
            if (k == ds.size()) return read(phs);
            const int d = ds[k];
            const std::string v = sd.vars[d - (3 - nd)];
            const std::string vq = "(" + v + (qd[d] >= 0 ? " + " : " - ") + std::to_string(qd[d] >= 0 ? qd[d] : -qd[d]) + ")";
            const std::string half = "((" + print_expr_text(p, {}, *md.extents[d - (3 - mnd)], nullptr) + ") / 2)";
            int a[3] = {phs[0], phs[1], phs[2]}, b2[3] = {phs[0], phs[1], phs[2]};
            if (pd[d] == 0 && qd[d] >= 1) {
              a[d] = 1; b2[d] = 0;
              return "select(" + vq + " >= " + half + ", " + build(k + 1, a) + ", " + build(k + 1, b2) + ")";
            }
            if (pd[d] == 1 && qd[d] <= -1) {
              a[d] = 0; b2[d] = 1;
              return "select(" + vq + " < 0, " + build(k + 1, a) + ", " + build(k + 1, b2) + ")";
            }
            a[d] = (int)pd[d];
            return build(k + 1, a);
          };
          int phs[3] = {0, 0, 0};
          out = build(0, phs);
          return true;
        }
        return false;
      };
      lines.push_back("stage " + sd.name + suffix(ph) + "(" + vs + ") [" + hext + "]: " + dtype_name(sd.dtype) + " = " +
                      print_expr_text(p, sd.vars, *sd.expr, &hook));
    }
    if (std::find(p.liveouts.begin(), p.liveouts.end(), (int)sidx) != p.liveouts.end()) {
      // the liveout keeps its name: interleave of its phases
      std::string ext;
      for (size_t i = 0; i < sd.extents.size(); ++i) ext += (i ? ", " : "") + print_expr_text(p, {}, *sd.extents[i], nullptr);
      std::function<std::string(size_t, int)> sel = [&](size_t k, int ph) -> std::string {
        if (k == ds.size()) {
          std::string a;
          for (int i = 0; i < nd; ++i) {
            const int d = i + 3 - nd;
            a += (i ? ", " : "") + (d >= 1 && u.dim[d] ? "(" + sd.vars[i] + " / 2)" : sd.vars[i]);
          }
          return sd.name + suffix(ph) + "(" + a + ")";
        }
        const std::string v = sd.vars[ds[k] - (3 - nd)];
        return "select((" + v + " % 2) == 0, " + sel(k + 1, ph) + ", " + sel(k + 1, ph | (1 << k)) + ")";
      };
      lines.push_back("stage " + sd.name + "(" + vs + ") [" + ext + "]: " + dtype_name(sd.dtype) + " = " + sel(0, 0));
      interleaves->insert(sd.name);
    }
  }
  std::vector<std::string> lo;
  for (int s : p.liveouts) lo.push_back(p.stages[s].name);
  return print_pipeline_text(p, lines, lo);
}

// ---- plane split (a colour-matrix mix of several plane-less producers) ------------------------------------------
// A stage S with a small plane dimension (K <= 4 planes) that reads at least three distinct plane-less stages (the
// camera's corrected(c) = M[c] . (R, G, B)) would be fused with them only as "broadcast" stages recomputed for every
// plane, or read them back from HBM once per plane.  Its K planes S_k(y, x) = S(k, y, x) are plane-less stages
// (the plane variable substituted by the constant k: exact); readers with the same K planes that read S at their
// own plane (the tone curve) are split the same way, and every other read S(e, y, x) becomes the select chain
// over clamp(e, 0, K-1) (reading R1), so the liveout keeps its planes.
struct PlaneSplit { int s = -1; int K = 0; std::set<int> set; };

PlaneSplit plane_candidate(const Analysis& A) {
  const Pipeline& p = *A.p;
  for (int s : p.topo) {
    const Ext3& se = A.stage_ext[s];
    if (!se.has[0] || se.e[0] > 4 || se.e[0] < 2) continue;
    if (std::find(p.liveouts.begin(), p.liveouts.end(), s) != p.liveouts.end()) continue;
    std::set<int> flat;
    for (const ReadSite& r : A.reads)
      if (r.consumer == s && r.src_is_stage && !A.stage_ext[r.src].has[0]) flat.insert(r.src);
    if (flat.size() < 3) continue;
    PlaneSplit ps;
    ps.s = s;
    ps.K = (int)se.e[0];
    std::vector<int> work{s};
    ps.set.insert(s);
    while (!work.empty()) {
      int m = work.back();
      work.pop_back();
      for (const ReadSite& r : A.reads) {
        if (!r.src_is_stage || r.src != m) continue;
        const Ext3& ce = A.stage_ext[r.consumer];
        const bool lo = std::find(p.liveouts.begin(), p.liveouts.end(), r.consumer) != p.liveouts.end();
        if (!lo && ce.has[0] && ce.e[0] == ps.K && r.form[0] == Form::UNIT && r.off[0] == 0 && ps.set.insert(r.consumer).second)
          work.push_back(r.consumer);
      }
    }
    return ps;
  }
  return {};
}

std::string plane_split_one(const Analysis& A, const PlaneSplit& ps) {
  const Pipeline& p = *A.p;
  using Hook = std::function<bool(const Expr&, std::string&)>;
  std::vector<std::string> lines;
  for (size_t sidx = 0; sidx < p.stages.size(); ++sidx) {
    const StageDecl& sd = p.stages[sidx];
    const int nd = (int)sd.vars.size();
    const bool member = ps.set.count((int)sidx) > 0;
    for (int k = 0; k < (member ? ps.K : 1); ++k) {
      std::vector<std::string> vars = sd.vars;
      if (member) vars[0] = std::to_string(k);          // the plane variable is the constant k
      Hook hook = [&](const Expr& e, std::string& out) {
        if (e.op != Expr::ACCESS || !e.is_stage || !ps.set.count(e.index)) return false;
        const StageDecl& md = p.stages[e.index];
        std::string rest;
        for (size_t i = 1; i < e.args.size(); ++i) rest += ", " + print_expr_text(p, vars, *e.args[i], &hook);
        auto nm = [&](int q) { return md.name + "_c" + std::to_string(q) + "(" + rest.substr(2) + ")"; };
        if (member) {   // a member reads a member at its own plane: the same constant plane
          out = nm(k);
          return true;
        }
        const std::string ce = "clamp(" + print_expr_text(p, vars, *e.args[0], &hook) + ", 0, " + std::to_string(ps.K - 1) + ")";
        std::string chain = nm(ps.K - 1);
        for (int q = ps.K - 2; q >= 0; --q) chain = "select(" + ce + " == " + std::to_string(q) + ", " + nm(q) + ", " + chain + ")";
        out = chain;
        return true;
      };
      std::string vs, ext;
      for (int i = member ? 1 : 0; i < nd; ++i) vs += std::string(vs.empty() ? "" : ", ") + sd.vars[i];
      for (int i = member ? 1 : 0; i < nd; ++i)
        ext += std::string(ext.empty() ? "" : ", ") + print_expr_text(p, {}, *sd.extents[i], nullptr);
      lines.push_back("stage " + sd.name + (member ? "_c" + std::to_string(k) : std::string()) + "(" + vs + ") [" + ext +
                      "]: " + dtype_name(sd.dtype) + " = " + print_expr_text(p, vars, *sd.expr, &hook));
    }
  }
  std::vector<std::string> lo;
  for (int s : p.liveouts) lo.push_back(p.stages[s].name);
  return print_pipeline_text(p, lines, lo);
}

}  // namespace

std::shared_ptr<Pipeline> phase_split(std::shared_ptr<Pipeline> p, const std::vector<int64_t>& params,
                                      std::vector<std::string>* split) {
  const char* env = getenv("PMG_PHASE_SPLIT");
  if (env && env[0] == '0') return p;
  for (int guard = 0; guard < 256; ++guard) {
    Analysis A = analyze(*p, params);
    Split sp = candidate(A);
    if (sp.s < 0) break;
    if (split) split->push_back(p->stages[sp.s].name + (sp.d == 1 ? "/y" : "/x"));
    p = parse_pipeline(split_one(A, sp));
  }
  const char* up = getenv("PMG_UP_SPLIT");
  if (up && up[0] == '0') return p;
  std::set<std::string> interleaves;
  for (int guard = 0; guard < 16; ++guard) {
    Analysis A = analyze(*p, params);
    Up u = up_candidate(A, interleaves);
    if (u.c < 0) break;
    if (split) split->push_back(p->stages[u.c].name + (u.dim[1] && u.dim[2] ? "/up-yx" : u.dim[1] ? "/up-y" : "/up-x"));
    p = parse_pipeline(up_split(A, u, &interleaves));
    // the downsampling split may now apply to the readers' new phases
    for (int g2 = 0; g2 < 256; ++g2) {
      Analysis B = analyze(*p, params);
      Split sp = candidate(B);
      if (sp.s < 0) break;
      if (split) split->push_back(p->stages[sp.s].name + (sp.d == 1 ? "/y" : "/x"));
      p = parse_pipeline(split_one(B, sp));
    }
  }
  for (int guard = 0; guard < 8; ++guard) {
    Analysis A = analyze(*p, params);
    PlaneSplit ps = plane_candidate(A);
    if (ps.s < 0) break;
    if (split) split->push_back(p->stages[ps.s].name + "/planes");
    p = parse_pipeline(plane_split_one(A, ps));
  }
  return p;
}

}  // namespace pmg
