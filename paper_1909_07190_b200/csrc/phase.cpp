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
        lines.push_back("stage " + (ph ? no : ne) + "(" + vs + ") [" + pext + "]: " + dtype_name(sd.dtype) + " = " +
                        print_expr_text(p, sub, *sd.expr, nullptr));
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
  return p;
}

}  // namespace pmg
