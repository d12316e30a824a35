// emit.cpp — CUDA C++ emitter for one fused group: an OTPW + hybrid-tiled sm_100a kernel.
//
// Structure of the emitted kernel (DESIGN.md §"Kernel"; §4-§5):
//   * one overlapped tile per warp, persistent warps striding over tiles; the only
//     synchronisation is __syncwarp and per-warp mbarriers — never a block barrier;
//   * the warp tile is TX parallelogram/chunk tiles of 32*V columns (split dim x) by TH rows;
//     lane l owns V consecutive columns of every chunk (B200 vectorised lane mapping);
//   * rows advance as a wavefront: at step t stage n produces row y0+t+hi_n (right hyperplane);
//     every stage value lives in a named register ("explicit variable names"), its recent rows
//     in a register window whose slots rotate with the unrolled step index;
//   * producer loads are resolved like Fig. 4 / Fig. 7: (1) own register
//     (same lane; any row of the window), (3) neighbour-lane register of the same chunk via __shfl_sync,
//     (4) last lanes of the previous (or next) chunk via the same shuffle with a sender-side select,
//     (2) shared memory for group inputs staged by TMA bulk copies into a warp-private ring;
//   * out-of-domain reads replicate the producer's edge value (reading R1), in x by a border-tile fix-up,
//     in y by filling / replicating window rows;
//   * f32 arithmetic is emitted with __f*_rn intrinsics in the written order (reading R3); the only
//     rewrites are exact ones: x / 2^k -> x * 2^-k, and a + 2^k*b -> fma(2^k, b, a) (2^k*b exact).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <sstream>

#include "plan.hpp"

namespace pmg {

namespace {

std::string ename(int e) { return e < 0 ? "m" + std::to_string(-e) : std::to_string(e); }

const char* ctype(DType d) {
  switch (d) {
    case DType::F32: return "float";
    case DType::I32: return "int";
    case DType::I16: return "short";
    case DType::U16: return "unsigned short";
    default: return "unsigned char";
  }
}
const char* rtype(DType d) { return d == DType::F32 ? "float" : "int"; }

bool is_pow2_float(float v, int* k) {
  if (!(v > 0.f) || std::isinf(v)) return false;
  int e;
  float m = std::frexp(v, &e);
  if (m != 0.5f) return false;
  *k = e - 1;   // v = 2^k
  return true;
}

std::string flit(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  char b[64];
  std::snprintf(b, sizeof b, "__int_as_float(0x%08x) /*%.9g*/", u, (double)f);
  return b;
}

struct Emitter {
  const Analysis& A;
  const Group& g;
  const Pipeline& p;
  std::map<const Expr*, int> site;   // ACCESS node -> ReadSite index
  std::ostringstream o;
  int V, TX;

  Emitter(const Analysis& a, const Group& gg) : A(a), g(gg), p(*a.p), V(gg.cfg.V), TX(gg.cfg.TX) {
    for (size_t i = 0; i < A.reads.size(); ++i) site[A.reads[i].node] = (int)i;
  }

  // per-kernel window depths and unroll factor (the interior kernel folds sums row by row and needs
  // shallower windows than the border kernel)
  std::vector<int> dS, dT;
  int Uk = 1;
  bool in_interior = false;   // emitting the interior-tile kernel (hybrid smem chunks apply there only)
  bool xe = false;            // interior kernel with x-edge tiles (Group::xedge): edge halos replicate by selects
  int cslot = -1;             // interior kernel: compile-time ring slot of the current step (-1: runtime)

  // hybrid tiling: stage i's window for chunk kk lives in warp-private shared memory (interior kernel,
  // chunks kk < S, rotating windows)
  bool hyb(int i, int kk) const {
    if (!in_interior || kk >= g.cfg.S || !g.gs[i].smem) return false;
    const int d = depS(i);
    return d <= 1 || Uk % d == 0;
  }
  std::string hyb_ptr(int i, int sl, int kk, const std::string& elem) const {
    const GStage& P = g.gs[i];
    const int esz = dtype_size(p.stages[P.id].dtype);
    return "(wsm + " + std::to_string(P.smem_off + sl * P.smem_rowb) + " + (" + std::to_string(P.smem_padl + kk * 32 * V) +
           " + V * lane + (" + elem + ")) * " + std::to_string(esz) + ")";
  }
  int back_shift = 0;   // set while emitting a fold segment evaluated m steps ahead of its stage row
  int depS(int i) const { return dS.empty() ? g.gs[i].depth : dS[i]; }
  int depT(int j) const { return dT.empty() ? g.streams[j].depth : dT[j]; }

  // physical window slot of back index b at sub-step u (rotation when depth | U, else shift naming)
  int slot(int depth, int b, int u) const {
    if (depth <= 1) return 0;
    if (Uk % depth == 0) return ((u - b) % depth + depth) % depth;
    return b;
  }
  // ---- register storage of rows: one scalar per element e in [-el, V+er) of every window slot ----
  std::string sv(int i, int sl, int k, int e) const {
    return "n" + std::to_string(i) + "_r" + std::to_string(sl) + "_c" + std::to_string(k) + "_e" + ename(e);
  }
  std::string tv(int j, int sl, int k, int e) const {
    return "s" + std::to_string(j) + "_r" + std::to_string(sl) + "_c" + std::to_string(k) + "_e" + ename(e);
  }
  // declare all slots of one buffer
  void declare(char pre, int i, bool isfloat, int depth, int el, int er) {
    o << "    " << (isfloat ? "float" : "int") << " ";
    bool first = true;
    for (int sl = 0; sl < depth; ++sl)
      for (int kk = 0; kk < TX; ++kk)
        for (int e = -el; e < V + er; ++e) {
          o << (first ? "" : ", ") << (pre == 'n' ? sv(i, sl, kk, e) : tv(i, sl, kk, e)) << " = 0";
          first = false;
        }
    o << ";\n";
  }
  // copy a whole row (all storage) from slot a to slot b
  void copy_row(char pre, int i, int el, int er, int a_, int b_, const std::string& ind) {
    for (int kk = 0; kk < TX; ++kk)
      for (int e = -el; e < V + er; ++e)
        o << ind << (pre == 'n' ? sv(i, b_, kk, e) : tv(i, b_, kk, e)) << " = " << (pre == 'n' ? sv(i, a_, kk, e) : tv(i, a_, kk, e)) << ";\n";
  }

  // ---- expression emission (ctx: consumer stage pos i, chunk k, element v, sub-step u) ----
  struct Ctx { int i, k, v, u; };
  struct R { std::string s; Kind k; };

  R tof(R a) { return a.k == Kind::Float ? a : R{"pmg_i2f(" + a.s + ")", Kind::Float}; }
  R toi(R a) { return a.k == Kind::Int ? a : R{"pmg_f2i(" + a.s + ")", Kind::Int}; }

  R ex(const Expr& e, const Ctx& c) {
    switch (e.op) {
      case Expr::INT: return {"(" + std::to_string(e.ival) + ")", Kind::Int};
      case Expr::FLT: return {flit(e.fval), Kind::Float};
      case Expr::PARAM: return {"a.prm[" + std::to_string(e.index) + "]", Kind::Int};
      case Expr::VAR: {
        int nd = (int)p.stages[g.gs[c.i].id].vars.size();
        int d = e.index + 3 - nd;
        if (d == 0) return {"pc", Kind::Int};
        if (d == 1) return {"row" + std::to_string(c.i), Kind::Int};
        return {"(xL + " + std::to_string(32 * V * c.k + c.v) + ")", Kind::Int};
      }
      case Expr::ACCESS: return access(e, c);
      case Expr::TABLE: {
        DType dt = p.tables[e.index].dtype;
        if (is_const_int(*e.args[0])) {   // loop-invariant lookup: loaded once per kernel (hoisted_tables)
          const int64_t v = std::min<int64_t>(std::max<int64_t>(eval_int(*e.args[0], A.params), 0), A.table_len[e.index] - 1);
          return {"tabc" + std::to_string(e.index) + "_" + std::to_string(v), dtype_is_float(dt) ? Kind::Float : Kind::Int};
        }
        R idx = toi(ex(*e.args[0], c));
        return {"pmg_ldg<" + std::string(ctype(dt)) + ">(a.tab[" + std::to_string(e.index) + "], pmg_clampi(" + idx.s +
                    ", 0, a.tabn[" + std::to_string(e.index) + "] - 1))",
                dtype_is_float(dt) ? Kind::Float : Kind::Int};
      }
      case Expr::UN: {
        R a = ex(*e.args[0], c);
        if (e.text == "!") return {"((" + a.s + ") == 0 ? 1 : 0)", Kind::Int};
        if (a.k == Kind::Float) return {"(-(" + a.s + "))", Kind::Float};
        return {"pmg_ineg(" + a.s + ")", Kind::Int};
      }
      case Expr::BIN: return bin(e, c);
      case Expr::CALL: return call(e, c);
    }
    return {"0", Kind::Int};
  }

  // exact power-of-two literal multiplier m >= 1 in "m*b" or "b*m"
  bool pow2_mul(const Expr& e, const Expr** b, float* m) {
    if (e.op != Expr::BIN || e.text != "*" || e.kind != Kind::Float) return false;
    int k;
    for (int s = 0; s < 2; ++s) {
      const Expr& L = *e.args[s];
      if (L.op == Expr::FLT && is_pow2_float(L.fval, &k) && k >= 0 && e.args[1 - s]->kind == Kind::Float) {
        *b = e.args[1 - s].get();
        *m = L.fval;
        return true;
      }
    }
    return false;
  }

  // a float product p*q (reassociation mode contracts it with an enclosing + or -)
  static bool is_fprod(const Expr& e) { return e.op == Expr::BIN && e.text == "*" && e.kind == Kind::Float; }

  // x parity (the camera interleave, the pyramid upsampling): when every lane's first column xL is even
  // (V, OW and PL even), `x + b` has a known parity per element, so `(x + b) % 2` is a constant and
  // `(x + b) / 2` (floor) is xL/2 plus a constant -- exact integer identities, no change of results
  bool x_even() const { return V % 2 == 0 && g.OW % 2 == 0 && g.PL % 2 == 0; }
  bool affine_x(const Expr& e, const Ctx& c, int64_t* off) {
    if (e.op == Expr::VAR) {
      int nd = (int)p.stages[g.gs[c.i].id].vars.size();
      if (e.index + 3 - nd != 2) return false;
      *off = 32 * V * c.k + c.v;
      return true;
    }
    if (e.op == Expr::BIN && e.kind == Kind::Int && (e.text == "+" || e.text == "-")) {
      int64_t o;
      if (e.args[1]->op == Expr::INT && affine_x(*e.args[0], c, &o)) {
        *off = e.text == "+" ? o + e.args[1]->ival : o - e.args[1]->ival;
        return true;
      }
      if (e.text == "+" && e.args[0]->op == Expr::INT && affine_x(*e.args[1], c, &o)) {
        *off = o + e.args[0]->ival;
        return true;
      }
    }
    return false;
  }

  R bin(const Expr& e, const Ctx& c) {
    const std::string& op = e.text;
    int64_t xo;
    if ((op == "%" || op == "/") && e.kind == Kind::Int && e.args[1]->op == Expr::INT && e.args[1]->ival == 2 && x_even() &&
        affine_x(*e.args[0], c, &xo)) {
      int64_t fl = xo >= 0 ? xo / 2 : -((-xo + 1) / 2);   // floor(xo / 2)
      if (op == "%") return {"(" + std::to_string(xo - 2 * fl) + ")", Kind::Int};
      return {"(xLh + " + std::to_string(fl) + ")", Kind::Int};
    }
    // floor division and non-negative remainder by a power of two are an arithmetic shift and a mask
    // (two's complement int32, reading R4): exact for every sign
    if ((op == "%" || op == "/") && e.kind == Kind::Int && e.args[1]->op == Expr::INT && e.args[1]->ival >= 2 &&
        e.args[1]->ival <= (1 << 30) && (e.args[1]->ival & (e.args[1]->ival - 1)) == 0) {
      R a = ex(*e.args[0], c);
      int k = 0;
      while ((int64_t(1) << k) < e.args[1]->ival) ++k;
      if (op == "%") return {"((" + a.s + ") & " + std::to_string(e.args[1]->ival - 1) + ")", Kind::Int};
      return {"((" + a.s + ") >> " + std::to_string(k) + ")", Kind::Int};
    }
    if (op == "&&" || op == "||") {
      R a = ex(*e.args[0], c), b = ex(*e.args[1], c);
      return {"(((" + a.s + ") != 0) " + op + " ((" + b.s + ") != 0) ? 1 : 0)", Kind::Int};
    }
    if (e.kind == Kind::Float && (op == "+" || op == "-")) {
      const Expr* mb;
      float m;
      // a + m*b  /  a - m*b   ->  fma(+-m, b, a)   (m = 2^k, k >= 0: the product is exact)
      if (pow2_mul(*e.args[1], &mb, &m)) {
        R a = tof(ex(*e.args[0], c)), b = ex(*mb, c);
        return {"pmg_fma_exact(" + flit(op == "+" ? m : -m) + ", " + b.s + ", " + a.s + ")", Kind::Float};
      }
      // reassociation mode (sched_opts.reassoc): a +- p*q -> fma(+-p, q, a).  Only a right-hand product
      // contracts, as in the interior kernel's fold spine (spine_op), so both kernels compute the same values.
      if (g.cfg.contract && is_fprod(*e.args[1])) {
        const Expr& Rt = *e.args[1];
        R a = tof(ex(*e.args[0], c)), m0 = tof(ex(*Rt.args[0], c)), m1 = tof(ex(*Rt.args[1], c));
        return {"__fmaf_rn(" + (op == "+" ? m0.s : "(-(" + m0.s + "))") + ", " + m1.s + ", " + a.s + ")", Kind::Float};
      }
      // m*b + a  ->  fma(m, b, a);  m*b - a -> fma(m, b, -a)
      if (pow2_mul(*e.args[0], &mb, &m)) {
        R b = ex(*mb, c), a = tof(ex(*e.args[1], c));
        std::string as = op == "+" ? a.s : "(-(" + a.s + "))";
        return {"pmg_fma_exact(" + flit(m) + ", " + b.s + ", " + as + ")", Kind::Float};
      }
    }
    R a = ex(*e.args[0], c), b = ex(*e.args[1], c);
    bool fl = a.k == Kind::Float || b.k == Kind::Float;
    if (op == "<" || op == "<=" || op == ">" || op == ">=" || op == "==" || op == "!=") {
      if (fl) { a = tof(a); b = tof(b); }
      return {"((" + a.s + ") " + op + " (" + b.s + ") ? 1 : 0)", Kind::Int};
    }
    if (fl) {
      a = tof(a);
      b = tof(b);
      if (op == "/" && e.args[1]->op == Expr::FLT) {
        int k;
        float v = e.args[1]->fval;
        if (is_pow2_float(v, &k) && std::isnormal(1.0f / v)) return {"pmg_mul(" + a.s + ", " + flit(1.0f / v) + ")", Kind::Float};
      }
      const char* f = op == "+" ? "pmg_add" : op == "-" ? "pmg_sub" : op == "*" ? "pmg_mul" : "pmg_div";
      return {std::string(f) + "(" + a.s + ", " + b.s + ")", Kind::Float};
    }
    const char* f = op == "+" ? "pmg_iadd" : op == "-" ? "pmg_isub" : op == "*" ? "pmg_imul" : op == "/" ? "pmg_idiv"
                    : op == "%" ? "pmg_imod" : op == "<<" ? "pmg_ishl" : "pmg_ishr";
    return {std::string(f) + "(" + a.s + ", " + b.s + ")", Kind::Int};
  }

  R call(const Expr& e, const Ctx& c) {
    const std::string& f = e.text;
    auto arg = [&](int i) { return ex(*e.args[i], c); };
    if (f == "min" || f == "max") {
      R a = arg(0), b = arg(1);
      if (a.k == Kind::Float || b.k == Kind::Float)
        return {std::string(f == "min" ? "pmg_fmin(" : "pmg_fmax(") + tof(a).s + ", " + tof(b).s + ")", Kind::Float};
      return {std::string(f == "min" ? "pmg_imin(" : "pmg_imax(") + a.s + ", " + b.s + ")", Kind::Int};
    }
    if (f == "clamp") {
      R x = arg(0), lo = arg(1), hi = arg(2);
      if (x.k == Kind::Float || lo.k == Kind::Float || hi.k == Kind::Float)
        return {"pmg_fmin(pmg_fmax(" + tof(x).s + ", " + tof(lo).s + "), " + tof(hi).s + ")", Kind::Float};
      return {"pmg_imin(pmg_imax(" + x.s + ", " + lo.s + "), " + hi.s + ")", Kind::Int};
    }
    if (f == "abs") {
      R a = arg(0);
      return a.k == Kind::Float ? R{"fabsf(" + a.s + ")", Kind::Float} : R{"pmg_iabs(" + a.s + ")", Kind::Int};
    }
    if (f == "absd") {
      R a = arg(0), b = arg(1);
      if (a.k == Kind::Float || b.k == Kind::Float) return {"fabsf(pmg_sub(" + tof(a).s + ", " + tof(b).s + "))", Kind::Float};
      return {"pmg_iabs(pmg_isub(" + a.s + ", " + b.s + "))", Kind::Int};
    }
    if (f == "select") {
      R cnd = arg(0), a = arg(1), b = arg(2);
      if (a.k == Kind::Float || b.k == Kind::Float) { a = tof(a); b = tof(b); }
      return {"((" + cnd.s + ") != 0 ? (" + a.s + ") : (" + b.s + "))", a.k};
    }
    if (f == "lerp") {
      R a = tof(arg(0)), b = tof(arg(1)), w = tof(arg(2));
      return {"pmg_add(pmg_mul(" + a.s + ", pmg_sub(1.0f, " + w.s + ")), pmg_mul(" + b.s + ", " + w.s + "))", Kind::Float};
    }
    if (f == "sqrt") return {"pmg_sqrt(" + tof(arg(0)).s + ")", Kind::Float};
    if (f == "f32") return tof(arg(0));
    if (f == "i32") return toi(arg(0));
    if (f == "i16") return {"pmg_to_i16(" + toi(arg(0)).s + ")", Kind::Int};
    if (f == "u16") return {"pmg_to_u16(" + toi(arg(0)).s + ")", Kind::Int};
    if (f == "u8") return {"pmg_to_u8(" + toi(arg(0)).s + ")", Kind::Int};
    if (f == "sat_u8") return {"pmg_clampi(" + toi(arg(0)).s + ", 0, 255)", Kind::Int};
    if (f == "sat_u16") return {"pmg_clampi(" + toi(arg(0)).s + ", 0, 65535)", Kind::Int};
    return {"0", Kind::Int};
  }

  R access(const Expr& e, const Ctx& c) {
    int ri = site.at(&e);
    const GRead& gr = g.greads.at(g.read_map.at(ri));
    const GStage& C = g.gs[c.i];
    if (gr.kind == RKind::STAGE) {
      const GStage& P = g.gs[gr.idx];
      int b = P.hi - C.hi - gr.dy;
      DType dt = p.stages[P.id].dtype;
      b -= back_shift;
      if (hyb(gr.idx, c.k))   // load type (2): the window row in shared memory, any x offset
        return {"pmg_lds<" + std::string(ctype(dt)) + ">(" + hyb_ptr(gr.idx, slot(depS(gr.idx), b, c.u), c.k, std::to_string(c.v + gr.dx)) +
                    ", 0)",
                dtype_is_float(dt) ? Kind::Float : Kind::Int};
      return {sv(gr.idx, slot(depS(gr.idx), b, c.u), c.k, c.v + gr.dx), dtype_is_float(dt) ? Kind::Float : Kind::Int};
    }
    if (gr.kind == RKind::STREAM) {
      const GStream& S = g.streams[gr.idx];
      int b = S.hi - C.hi - gr.dy;
      b -= back_shift;
      const int e = (S.sx == 1 ? 2 * c.v : c.v) + gr.dx;   // register index (down2: q = 2e + b)
      return {tv(gr.idx, slot(depT(gr.idx), b, c.u), c.k, e), dtype_is_float(S.dtype) ? Kind::Float : Kind::Int};
    }
    // gather: per-element global load with clamped indices (any index form)
    const ReadSite& r = A.reads[ri];
    const Ext3& se = r.src_is_stage ? A.stage_ext[r.src] : A.image_ext[r.src];
    DType dt = r.src_is_stage ? p.stages[r.src].dtype : p.images[r.src].dtype;
    int pnd = (int)e.args.size();
    std::string idx[3] = {"0", "0", "0"};
    std::string t = "a.t[" + std::to_string(gr.idx) + "]";
    for (int i = 0; i < pnd; ++i) {
      int d = i + 3 - pnd;
      R v = toi(ex(*e.args[i], c));
      // rows: the buffer's rows (the image for full runs, reading R1; the band's rows for band runs)
      idx[d] = d == 1 ? "pmg_clampi(" + v.s + ", " + t + ".row_base, " + t + ".row_base + " + t + ".nrows - 1)"
                      : "pmg_clampi(" + v.s + ", 0, " + std::to_string(se.e[d] - 1) + ")";
    }
    std::string base = "(" + t + ".ptr + (i64)fr * " + t + ".frame_stride + (i64)(" + idx[0] + ") * " + t + ".plane_pitch + (i64)((" + idx[1] + ") - " + t +
                       ".row_base) * " + t + ".row_pitch)";
    return {"pmg_ldg<" + std::string(ctype(dt)) + ">(" + base + ", " + idx[2] + ")", dtype_is_float(dt) ? Kind::Float : Kind::Int};
  }

  // ---- packed-pair evaluation: elements (va, vb) of one lane as one float2 expression tree ----
  struct R2 { bool pair; std::string p; R a, b; };

  std::string pack(const R2& r) { return r.pair ? r.p : "make_float2(" + tof(r.a).s + ", " + tof(r.b).s + ")"; }

  bool pairable(const Expr& e) {
    // packed pairs only for +, - (including the exact 2^k fma form), negation, literals and reads.
    // Products and quotients stay scalar: ptxas fuses mul.rn.f32x2 -> add.rn.f32x2 into FFMA2 even with
    // --fmad=false, which would change the rounding (checked on nvcc 12.9 / sm_100a).
    if (e.kind != Kind::Float) return false;
    switch (e.op) {
      case Expr::FLT: case Expr::ACCESS: return true;
      case Expr::UN: return e.text == "-";
      case Expr::BIN: return e.text == "+" || e.text == "-";
      default: return false;
    }
  }

  R2 ex2(const Expr& e, int i, int k, int va, int vb, int u) {
    if (!pairable(e)) return R2{false, "", ex(e, Ctx{i, k, va, u}), ex(e, Ctx{i, k, vb, u})};
    switch (e.op) {
      case Expr::FLT: return R2{true, "pmg_bc2(" + flit(e.fval) + ")", {}, {}};
      case Expr::ACCESS: {
        int ri = site.at(&e);
        const GRead& gr = g.greads.at(g.read_map.at(ri));
        const GStage& C = g.gs[i];
        R a = ex(e, Ctx{i, k, va, u}), b = ex(e, Ctx{i, k, vb, u});
        return R2{true, "make_float2(" + a.s + ", " + b.s + ")", {}, {}};
      }
      case Expr::UN: return R2{true, "pmg_neg2(" + pack(ex2(*e.args[0], i, k, va, vb, u)) + ")", {}, {}};
      case Expr::CALL: {   // lerp(a, b, w) = a * (1 - w) + b * w
        std::string a = pack(ex2(*e.args[0], i, k, va, vb, u)), b = pack(ex2(*e.args[1], i, k, va, vb, u)),
                    w = pack(ex2(*e.args[2], i, k, va, vb, u));
        return R2{true, "pmg_add2(pmg_mul2(" + a + ", pmg_sub2(pmg_bc2(1.0f), " + w + ")), pmg_mul2(" + b + ", " + w + "))", {}, {}};
      }
      default: break;
    }
    const std::string& op = e.text;
    if (op == "+" || op == "-") {
      const Expr* mb;
      float m;
      if (pow2_mul(*e.args[1], &mb, &m)) {
        std::string a = pack(ex2(*e.args[0], i, k, va, vb, u)), b = pack(ex2(*mb, i, k, va, vb, u));
        return R2{true, "pmg_fma2(pmg_bc2(" + flit(op == "+" ? m : -m) + "), " + b + ", " + a + ")", {}, {}};
      }
      if (pow2_mul(*e.args[0], &mb, &m)) {
        std::string b = pack(ex2(*mb, i, k, va, vb, u)), a = pack(ex2(*e.args[1], i, k, va, vb, u));
        return R2{true, "pmg_fma2(pmg_bc2(" + flit(m) + "), " + b + ", " + (op == "+" ? a : "pmg_neg2(" + a + ")") + ")", {}, {}};
      }
    }
    std::string a = pack(ex2(*e.args[0], i, k, va, vb, u));
    if (op == "/") {
      return R2{true, "pmg_mul2(" + a + ", pmg_bc2(" + flit(1.0f / e.args[1]->fval) + "))", {}, {}};
    }
    std::string b = pack(ex2(*e.args[1], i, k, va, vb, u));
    const char* f = op == "+" ? "pmg_add2" : op == "-" ? "pmg_sub2" : "pmg_mul2";
    return R2{true, std::string(f) + "(" + a + ", " + b + ")", {}, {}};
  }

  std::string conv_store(const R& v, DType dt) {
    if (dt == DType::F32) return tof(v).s;
    R i = toi(v);
    switch (dt) {
      case DType::I16: return "pmg_to_i16(" + i.s + ")";
      case DType::U16: return "pmg_to_u16(" + i.s + ")";
      case DType::U8: return "pmg_to_u8(" + i.s + ")";
      default: return i.s;
    }
  }

  // ---- incremental left-fold evaluation (interior kernel) ----
  // A stage whose expression is a left-deep chain of float +,-,*,/ (the spine) over operands listed in
  // row-major order can be evaluated row by row: the prefix that needs only older producer rows is computed
  // as soon as those rows exist and carried forward as one value per element, instead of keeping the
  // producer rows in a register window.  Same operations, same order => bit-identical (reading R3).
  struct SpineOp { const Expr* node; const Expr* right; int pmb; };
  struct Fold {
    bool on = false;
    const Expr* base = nullptr;
    int base_pmb = 0;
    std::vector<SpineOp> ops;
    std::vector<int> m;            // distinct prefix min-backs, decreasing, last == 0
    std::vector<int> cd;           // carried-value window depths m[j] - m[j+1]
  };
  std::vector<Fold> folds;
  static constexpr int kInf = 1 << 28;

  int minback(const Expr& e, int i) {
    int mb = kInf;
    if (e.op == Expr::ACCESS) {
      const GRead& gr = g.greads.at(g.read_map.at(site.at(&e)));
      if (gr.kind == RKind::STAGE) mb = g.gs[gr.idx].hi - g.gs[i].hi - gr.dy;
      else if (gr.kind == RKind::STREAM) mb = g.streams[gr.idx].hi - g.gs[i].hi - gr.dy;
    }
    for (auto& a : e.args) mb = std::min(mb, minback(*a, i));
    return mb;
  }

  // window depths needed by the reads of `e` evaluated `shift` steps ahead
  void scan_depths(const Expr& e, int i, int shift, std::vector<int>& ds, std::vector<int>& dt) {
    if (e.op == Expr::ACCESS) {
      const GRead& gr = g.greads.at(g.read_map.at(site.at(&e)));
      if (gr.kind == RKind::STAGE) ds[gr.idx] = std::max(ds[gr.idx], g.gs[gr.idx].hi - g.gs[i].hi - gr.dy - shift + 1);
      else if (gr.kind == RKind::STREAM) dt[gr.idx] = std::max(dt[gr.idx], g.streams[gr.idx].hi - g.gs[i].hi - gr.dy - shift + 1);
    }
    for (auto& a : e.args) scan_depths(*a, i, shift, ds, dt);
  }

  static int gcd_(int a, int b) { return b ? gcd_(b, a % b) : a; }

  // decide folds, fast window depths and the unroll factor of the interior kernel
  void plan_interior() {
    const int n = (int)g.gs.size();
    folds.assign(n, Fold{});
    const char* env = getenv("PMG_FOLD");
    const bool enable = !(env && env[0] == '0');
    for (int i = 0; i < n && enable; ++i) {
      const StageDecl& sd = p.stages[g.gs[i].id];
      if (sd.dtype != DType::F32) continue;
      Fold f;
      const Expr* cur = sd.expr.get();
      while (cur->op == Expr::BIN && cur->kind == Kind::Float &&
             (cur->text == "+" || cur->text == "-" || cur->text == "*" ||
              (cur->text == "/" && cur->args[1]->op == Expr::FLT))) {
        f.ops.push_back({cur, cur->args[1].get(), 0});
        cur = cur->args[0].get();
      }
      std::reverse(f.ops.begin(), f.ops.end());
      f.base = cur;
      int pm = minback(*cur, i);
      std::vector<int> seq;
      for (auto& op : f.ops) {
        pm = std::min(pm, minback(*op.right, i));
        op.pmb = pm;
      }
      // leading constant-only prefixes join the first segment that reads something
      int first = kInf;
      for (auto& op : f.ops)
        if (op.pmb < kInf) { first = op.pmb; break; }
      f.base_pmb = std::min(minback(*cur, i), first);
      if (f.base_pmb >= kInf) continue;
      for (auto& op : f.ops)
        if (op.pmb >= kInf) op.pmb = f.base_pmb;
      f.m.push_back(f.base_pmb);
      for (auto& op : f.ops)
        if (op.pmb != f.m.back()) f.m.push_back(op.pmb);
      if (f.m.size() < 2 || f.m.back() != 0) continue;
      for (size_t j = 0; j + 1 < f.m.size(); ++j) f.cd.push_back(f.m[j] - f.m[j + 1]);
      f.on = true;
      folds[i] = f;
    }
    auto compute = [&](std::vector<int>& ds, std::vector<int>& dt) {
      ds.assign(n, 1);
      dt.assign(g.streams.size(), 1);
      for (int i = 0; i < n; ++i) {
        const Fold& f = folds[i];
        if (!f.on) { scan_depths(*p.stages[g.gs[i].id].expr, i, 0, ds, dt); continue; }
        scan_depths(*f.base, i, f.base_pmb, ds, dt);
        for (auto& op : f.ops) scan_depths(*op.right, i, op.pmb, ds, dt);
      }
    };
    compute(dS, dT);
    int U = 1;
    auto lcm = [](int a, int b) { return a / gcd_(a, b) * b; };
    for (int d : dS) U = lcm(U, d);
    for (int d : dT) U = lcm(U, d);
    for (auto& f : folds)
      for (int d : f.cd) U = lcm(U, d);
    if (U > 16) {   // give up folding: plain windows, shift mode beyond 16
      folds.assign(n, Fold{});
      dS.clear();
      dT.clear();
      Uk = g.U;
      return;
    }
    Uk = U;
  }

  std::string cname(int i, int j, int sl, int k, int v) const {
    return "f" + std::to_string(i) + "_" + std::to_string(j) + "_r" + std::to_string(sl) + "_c" + std::to_string(k) + "_e" + std::to_string(v);
  }

  // one spine operation with the running prefix as left operand (mirrors bin(): exact fma for 2^k*b)
  R spine_op(const SpineOp& op, const R& left, const Ctx& c) {
    const std::string& t = op.node->text;
    if (t == "+" || t == "-") {
      const Expr* mb;
      float m;
      if (pow2_mul(*op.right, &mb, &m))
        return {"pmg_fma_exact(" + flit(t == "+" ? m : -m) + ", " + ex(*mb, c).s + ", " + tof(left).s + ")", Kind::Float};
      if (g.cfg.contract && is_fprod(*op.right)) {   // mirrors bin(): left +- p*q -> fma(+-p, q, left)
        R m0 = tof(ex(*op.right->args[0], c)), m1 = tof(ex(*op.right->args[1], c));
        return {"__fmaf_rn(" + (t == "+" ? m0.s : "(-(" + m0.s + "))") + ", " + m1.s + ", " + tof(left).s + ")", Kind::Float};
      }
    }
    if (t == "/") {
      int k;
      float v = op.right->fval;
      if (is_pow2_float(v, &k) && std::isnormal(1.0f / v)) return {"pmg_mul(" + tof(left).s + ", " + flit(1.0f / v) + ")", Kind::Float};
      return {"pmg_div(" + tof(left).s + ", " + flit(v) + ")", Kind::Float};
    }
    R b = tof(ex(*op.right, c));
    const char* f = t == "+" ? "pmg_add" : t == "-" ? "pmg_sub" : "pmg_mul";
    return {std::string(f) + "(" + tof(left).s + ", " + b.s + ")", Kind::Float};
  }

  // table lookups at constant indices (the camera's colour matrix after its plane split): one load per kernel
  // into a register, instead of one per point (same value: the index is clamped to the table as in ex())
  void hoisted_tables() {
    std::map<std::pair<int, int64_t>, DType> seen;
    std::function<void(const Expr&)> scan = [&](const Expr& e) {
      if (e.op == Expr::TABLE && is_const_int(*e.args[0])) {
        const int64_t v = std::min<int64_t>(std::max<int64_t>(eval_int(*e.args[0], A.params), 0), A.table_len[e.index] - 1);
        seen[{e.index, v}] = p.tables[e.index].dtype;
      }
      for (auto& a : e.args) scan(*a);
    };
    for (auto& P : g.gs) scan(*p.stages[P.id].expr);
    for (auto& kv : seen)
      o << "  const " << rtype(kv.second) << " tabc" << kv.first.first << "_" << kv.first.second << " = pmg_ldg<"
        << ctype(kv.second) << ">(a.tab[" << kv.first.first << "], " << kv.first.second << ");\n";
  }

  // OTPTB ablation (PMG_OTPTB=1): block barriers between stages instead of warp-only synchronisation
  static bool otptb() { const char* e = getenv("PMG_OTPTB"); return e && e[0] == '1'; }

  bool pack_on() const {
    // opt-in (PMG_PACK=1): bit-exact, but on B200 the make_float2 MOVs cost what the packed FADD2s save
    // (harris 6400^2: 0.1198 ms packed vs 0.1169 ms scalar)
    const char* e = getenv("PMG_PACK");
    return V >= 2 && V % 2 == 0 && e && (e[0] == '1' || e[0] == '2');
  }
  bool pack_stages() const { const char* e = getenv("PMG_PACK"); return pack_on() && e[0] == '1'; }   // '2': folds only

  // packed fold segment: statement per spine op; pairs (v, v + V/2) of the same lane
  void fold_segment_pair(int i, int j, int u, int cur, const std::string& ind) {
    const Fold& f = folds[i];
    const int nseg = (int)f.m.size(), h = V / 2;
    back_shift = f.m[j];
    for (int kk = 0; kk < TX; ++kk)
      for (int v = 0; v < h; ++v) {
        Ctx ca{i, kk, v, u}, cb{i, kk, v + h, u};
        o << ind << "{ float2 pv = ";
        if (j == 0) o << pack(ex2(*f.base, i, kk, v, v + h, u));
        else {
          const int d = f.cd[j - 1];
          o << "make_float2(" << cname(i, j - 1, slot(d, d, u), kk, v) << ", " << cname(i, j - 1, slot(d, d, u), kk, v + h) << ")";
        }
        o << ";\n";
        for (auto& op : f.ops) {
          if (op.pmb != f.m[j]) continue;
          const std::string& t = op.node->text;
          const Expr* mb;
          float m;
          if ((t == "+" || t == "-") && pow2_mul(*op.right, &mb, &m)) {
            o << ind << "  pv = pmg_fma2(pmg_bc2(" << flit(t == "+" ? m : -m) << "), " << pack(ex2(*mb, i, kk, v, v + h, u)) << ", pv);\n";
          } else if (t == "+" || t == "-") {
            o << ind << "  pv = " << (t == "+" ? "pmg_add2" : "pmg_sub2") << "(pv, " << pack(ex2(*op.right, i, kk, v, v + h, u)) << ");\n";
          } else {   // * and / element by element (scalar; see pairable())
            R lx = spine_op(op, R{"pv.x", Kind::Float}, ca), ly = spine_op(op, R{"pv.y", Kind::Float}, cb);
            o << ind << "  pv = make_float2(" << lx.s << ", " << ly.s << ");\n";
          }
        }
        if (j == nseg - 1)
          o << ind << "  " << sv(i, cur, kk, v) << " = pv.x; " << sv(i, cur, kk, v + h) << " = pv.y; }\n";
        else
          o << ind << "  " << cname(i, j, slot(f.cd[j], 0, u), kk, v) << " = pv.x; " << cname(i, j, slot(f.cd[j], 0, u), kk, v + h)
            << " = pv.y; }\n";
      }
    back_shift = 0;
  }

  // emit fold segment j of stage i at sub-step u: consume carried[j-1], produce carried[j] or the stage row
  void fold_segment(int i, int j, int u, int cur, const std::string& ind) {
    const Fold& f = folds[i];
    const int nseg = (int)f.m.size();
    const StageDecl& sd = p.stages[g.gs[i].id];
    back_shift = f.m[j];
    for (int kk = 0; kk < TX; ++kk)
      for (int v = 0; v < V; ++v) {
        Ctx c{i, kk, v, u};
        R val;
        if (j == 0) val = ex(*f.base, c);
        else {
          const int d = f.cd[j - 1];
          val = {cname(i, j - 1, slot(d, d, u), kk, v), Kind::Float};
        }
        for (auto& op : f.ops)
          if (op.pmb == f.m[j]) val = spine_op(op, val, c);
        if (j == nseg - 1) o << ind << sv(i, cur, kk, v) << " = " << conv_store(val, sd.dtype) << ";\n";
        else o << ind << cname(i, j, slot(f.cd[j], 0, u), kk, v) << " = " << tof(val).s << ";\n";
      }
    back_shift = 0;
  }

  int state_regs() {
    plan_interior();
    const int n = (int)g.gs.size();
    int r = 0;
    for (int i = 0; i < n; ++i) r += (depS(i) - 1) * TX * (V + g.gs[i].el + g.gs[i].er);
    for (size_t j = 0; j < g.streams.size(); ++j)
      r += (depT((int)j) - 1) * TX * (V + g.streams[j].el + g.streams[j].er);
    for (auto& f : folds)
      for (int d : f.cd) r += d * TX * V;
    return r;
  }

  // ---- kernel text ----
  int himax = 0, xlm = 0, xrm = 0;

  int phase_of(int t) const { return (((t - g.t_first) % Uk) + Uk) % Uk; }

  std::string run() {
    o << "// generated by libpmg (emit.cpp) for group " << g.name << ": ";
    for (auto& s : g.gs) o << p.stages[s.id].name << " ";
    o << "\n#include \"pmg_otpw.cuh\"\n\n";
    header();
    kernel(true);
    if (g.xedge && !xe_skip) kernel(true, true);
    return o.str();
  }

  // macros, argument struct and tile decoders of the group
  void header() {
    const KConfig& k = g.cfg;
    for (auto& P : g.gs) himax = std::max(himax, P.hi);
    for (auto& S : g.streams) himax = std::max(himax, S.hi);
    for (auto& S : g.streams)
      if (S.sx == 0) { xlm = std::max(xlm, S.xl); xrm = std::max(xrm, S.xr); }
    o << "#define V " << V << "\n#define TX " << TX << "\n#define CW " << g.CW << "\n#define PL " << g.PL
      << "\n#define OW " << g.OW << "\n#define TH " << k.TH << "\n#define NW " << k.NW << "\n#define PREF " << k.PREF
      << "\n#define TFIRST " << g.t_first << "\n#define NSTEPS " << g.nsteps << "\n#define USTEP " << g.U
      << "\n#define RING " << g.ring_bytes << "\n#define WSMEM " << g.warp_smem << "\n#define BARB "
      << ((8 * k.PREF + 15) / 16 * 16) << "\n#define XLM " << xlm << "\n#define XRM " << xrm << "\n#define HIMAX " << himax
      << "\n\n";
    int nt = std::max<int>(1, (int)g.tensors.size()), ntab = std::max<int>(1, (int)p.tables.size()),
        np = std::max<int>(1, (int)p.params.size());
    o << "struct PmgArgs {\n  PmgTensor t[" << nt << "];\n  const char* tab[" << ntab << "];\n  int tabn[" << ntab
      << "];\n  int prm[" << np << "];\n"
         "  int H, W, gy0, gy1, nty, ntx, npl, nfr, ntiles, pad_;\n"
         "  int txA, txB, tyA, tyB;   // interior rectangle of tile columns / rows (host-computed)\n"
         "  int ylast, cxlast;        // interior kernel: the last tile row / column is shifted to end at the image\n};\n\n";
    // tile index -> (tx, ty, pc, fr): interior kernel walks the rectangle, border kernel its complement
    o << "__device__ __forceinline__ void pmg_tile_int(const PmgArgs& a, int t, int& tx, int& ty, int& pc, int& fr) {\n"
         "  const int w = a.txB - a.txA, h = a.tyB - a.tyA;\n"
         "  tx = a.txA + t % w; int r = t / w; ty = a.tyA + r % h; r /= h; pc = r % a.npl; fr = r / a.npl;\n}\n"
         "__device__ __forceinline__ void pmg_tile_bdr(const PmgArgs& a, int t, int& tx, int& ty, int& pc, int& fr) {\n"
         "  const int per = a.nty * a.ntx - (a.tyB - a.tyA) * (a.txB - a.txA);\n"
         "  int kk = t % per; const int r = t / per; pc = r % a.npl; fr = r / a.npl;\n"
         "  const int top = a.tyA * a.ntx;\n"
         "  if (kk < top) { ty = kk / a.ntx; tx = kk % a.ntx; return; }\n"
         "  kk -= top;\n"
         "  const int bot = (a.nty - a.tyB) * a.ntx;\n"
         "  if (kk < bot) { ty = a.tyB + kk / a.ntx; tx = kk % a.ntx; return; }\n"
         "  kk -= bot;\n"
         "  const int side = a.ntx - (a.txB - a.txA);\n"
         "  ty = a.tyA + kk / side; const int j = kk % side; tx = j < a.txA ? j : a.txB + (j - a.txA);\n}\n"
         "__device__ __forceinline__ void pmg_tile_e(const PmgArgs& a, int t, int& tx, int& ty, int& pc, int& fr) {\n"
         "  const int side = a.ntx - (a.txB - a.txA), h = a.tyB - a.tyA;\n"
         "  const int j = t % side; int r = t / side; ty = a.tyA + r % h; r /= h; pc = r % a.npl; fr = r / a.npl;\n"
         "  tx = j < a.txA ? j : a.txB + (j - a.txA);\n}\n\n";
  }
  // the interior-tile kernel alone (the selector's register probe reads its ptxas count)
  std::string run_interior_only() {
    xe_skip = true;
    return run();
  }
  bool xe_skip = false;

  // the border-tile kernel of the same group, with TH_b-row tiles (macros TH / NSTEPS redefined)
  std::string run_border() {
    for (auto& P : g.gs) himax = std::max(himax, P.hi);
    for (auto& S : g.streams) himax = std::max(himax, S.hi);
    for (auto& S : g.streams)
      if (S.sx == 0) { xlm = std::max(xlm, S.xl); xrm = std::max(xrm, S.xr); }
    o << "#undef TH\n#undef NSTEPS\n#define TH " << g.cfg.TH << "\n#define NSTEPS " << g.nsteps << "\n\n";
    kernel(false);
    return o.str();
  }

  // tile origin: the interior and x-edge kernels shift their last tile row up to end at the last row they may
  // compute (a.ylast; overlapping tile rows store the same values); the x-edge kernel starts its first tile
  // column at x = 0 instead of -PL; the border kernel keeps the plain grid
  std::string y0_expr(const std::string& ty) const {
    return in_interior ? "min(a.gy0 + " + ty + " * TH, a.ylast)" : "(a.gy0 + " + ty + " * TH)";
  }
  std::string cx_expr(const std::string& tx) const {
    return xe ? "max(" + tx + " * OW - PL, 0)" : "(" + tx + " * OW - PL)";
  }

  // one entry point: interior tiles (branch-free bodies) or border tiles (general bodies)
  void kernel(bool interior, bool edge = false) {
    const KConfig& k = g.cfg;
    const int n = (int)g.gs.size();
    if (interior) plan_interior();
    else {
      dS.clear();
      dT.clear();
      folds.assign(n, Fold{});
      Uk = g.U;
    }
    in_interior = interior;
    xe = interior && edge;
    const char* dec = xe ? "pmg_tile_e" : interior ? "pmg_tile_int" : "pmg_tile_bdr";
    int cap = k.regcap;
    {   // experiment knobs: register caps per kernel class (interior / x-edge / border)
      const char* e = getenv(xe ? "PMG_CAP_E" : interior ? "PMG_CAP_I" : "PMG_CAP_B");
      if (e && atoi(e) > 0) cap = atoi(e);
    }
    if (!interior && cap <= 0) {
      // border tiles are latency-bound and share the SMs with the interior kernel: cap their registers so
      // that many of them stay resident
      // measured (profiles/sweep notes in DESIGN.md): a 96-register cap helps small pipelines (unsharp 2048^2:
      // 0.035 -> 0.027 ms) and hurts large general bodies (Harris 0.106 -> 0.120, camera 0.115 -> 0.127 ms)
      const char* e = getenv("PMG_BORDER_REGCAP");
      cap = e ? atoi(e) : (g.regs_est > 0 && g.regs_est <= 72 ? 96 : 0);
    }
    int minb = cap > 0 ? std::max(1, 65536 / (cap * 32 * k.NW)) : 1;
    o << "extern \"C\" __global__ void __launch_bounds__(NW * 32, " << minb << ") " << g.name << (xe ? "_e" : interior ? "" : "_b")
      << "(const __grid_constant__ PmgArgs a) {\n";
    o << "  extern __shared__ __align__(128) char pmg_smem[];\n"
         "  const int lane = threadIdx.x & 31;\n"
         "  const int wib = threadIdx.x >> 5;\n"
         "  char* wsm = pmg_smem + wib * WSMEM;\n"
         "  const u32 bar0 = pmg_smem_addr(wsm);\n"
         "  char* ring = wsm + BARB;\n"
         "  const u32 ring_addr = pmg_smem_addr(ring);\n"
         "  (void)ring; (void)bar0; (void)ring_addr;\n"
         "  const int gw = blockIdx.x * NW + wib;\n"
         "  const int nwt = gridDim.x * NW;\n"
         "  const int H = a.H, W = a.W;\n";
    if (otptb()) {
      // OTPTB ablation (§3, Fig. 8): the block's warps step through their tiles together and meet at
      // a block barrier after every stage; all warps of a block take the same number of tiles (a warp past the
      // last tile recomputes the last tile and stores the same values)
      o << "  if (blockIdx.x * NW >= a.ntiles) return;\n"
           "  const int my_tiles = (a.ntiles - blockIdx.x * NW + nwt - 1) / nwt;\n";
    } else {
      o << "  if (gw >= a.ntiles) return;\n"
           "  const int my_tiles = (a.ntiles - gw + nwt - 1) / nwt;\n";
    }
    // programmatic dependent launch: let the next kernel on the stream be scheduled now, and wait until the
    // previous one has completed and its writes are visible before the first global access
    o << "  asm volatile(\"griddepcontrol.launch_dependents;\" ::: \"memory\");\n"
         "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
    hoisted_tables();
    const bool hs = !g.streams.empty();
    if (hs) {
      // ---- TMA producer state: one request per step, PREF steps ahead of the consumer; lane 0 issues ----
      o << "  if (lane == 0) {\n    for (int i = 0; i < PREF; ++i) pmg_mbar_init(bar0 + 8 * i, 1);\n    pmg_mbar_init_fence();\n  }\n"
           "  __syncwarp();\n"
           "  const bool leader = lane == 0;\n"
           "  int p_y0 = 0, pn_y0 = 0;\n  u32 p_total = 0, pn_total = 0;\n";
      for (size_t j = 0; j < g.streams.size(); ++j)
        o << "  const char* p_src" << j << " = nullptr; const char* pn_src" << j << " = nullptr; u32 p_dst" << j << " = 0, pn_dst" << j
          << " = 0, p_bytes" << j << " = 0, pn_bytes" << j << " = 0;\n";
      // tile -> request constants (divisions once per tile)
      o << "  auto p_params = [&](int tile, int& y0r, u32& tot";
      for (size_t j = 0; j < g.streams.size(); ++j) o << ", const char*& src" << j << ", u32& dst" << j << ", u32& byt" << j;
      o << ") {\n"
           "    int txq, tyq, pcq, frq;\n    " << dec << "(a, tile, txq, tyq, pcq, frq);\n"
           "    (void)pcq; (void)frq;\n"
           "    y0r = " << y0_expr("tyq") << ";\n"
           "    const int cxq = " << cx_expr("txq") << ";\n"
           "    tot = 0;\n";
      for (size_t j = 0; j < g.streams.size(); ++j) {
        const GStream& S = g.streams[j];
        int Aal = 16 / S.esz;
        o << "    {\n      const PmgTensor& T = a.t[" << S.tensor_slot << "];\n"
          << "      const int pl = " << (S.plane_mode == 0 ? "0" : S.plane_mode == 1 ? "pcq" : std::to_string(S.plane_const)) << ";\n"
          << "      const int xlo = " << pcol(S, "cxq") << " - " << S.xl << ", xhi = xlo + " << S.row_elems << ";\n"
          << "      const int wa = (" << (S.sx == 0 ? std::string("W") : "T.W") << " + " << (Aal - 1) << ") / " << Aal << " * " << Aal << ";\n"
          << "      const int clo = xlo < 0 ? 0 : xlo, chi = xhi > wa ? wa : xhi;\n"
          << "      src" << j << " = T.ptr + (i64)frq * T.frame_stride + (i64)pl * T.plane_pitch - (i64)T.row_base * T.row_pitch + (i64)clo * " << S.esz << ";\n"
          << "      dst" << j << " = " << S.smem_off << " + (u32)(clo - xlo) * " << S.esz << ";\n"
          << "      byt" << j << " = (u32)(chi - clo) * " << S.esz << ";\n"
          << "      tot += byt" << j << ";\n    }\n";
      }
      o << "  };\n";
      o << "  p_params(" << (otptb() ? "min(gw, a.ntiles - 1)" : "gw") << ", p_y0, p_total";
      for (size_t j = 0; j < g.streams.size(); ++j) o << ", p_src" << j << ", p_dst" << j << ", p_bytes" << j;
      o << ");\n";
      // prologue: the first PREF requests of the first tile
      o << "  for (int s = 0; s < PREF; ++s) {\n"
           "    const u32 bar = bar0 + 8 * s;\n"
           "    pmg_mbar_expect_tx_if(bar, p_total, leader);\n";
      for (size_t j = 0; j < g.streams.size(); ++j)
        o << "    pmg_bulk_g2s_if(ring_addr + s * RING + p_dst" << j << ", p_src" << j << " + (i64)"
          << prow((int)j, "p_y0 + (TFIRST + " + std::to_string(g.streams[j].hi) + ") + s") << " * a.t[" << g.streams[j].tensor_slot
          << "].row_pitch, p_bytes" << j << ", bar, leader);\n";
      o << "  }\n  int c_slot = 0;\n  u32 phase = 0u;   // parity of the ring's current lap (all slots are used round-robin)\n";
    }
    o << "  for (int it = 0; it < my_tiles; ++it) {\n"
         "    const int tile = " << (otptb() ? "min(gw + it * nwt, a.ntiles - 1)" : "gw + it * nwt") << ";\n"
         "    int tx, ty, pc, fr;\n    " << dec << "(a, tile, tx, ty, pc, fr);\n"
         "    const int y0 = " << y0_expr("ty") << ";\n"
         "    const int cx = " << cx_expr("tx") << ";\n"
         "    const int xL = cx + V * lane;\n"
         "    const int xLh = xL >> 1;   // xL / 2 (used only when xL is even)\n"
         "    const bool xb = (cx - XLM < 0) || (cx + CW + XRM > W)" << xb_scaled() << ";\n";
    if (xe) {
      // x-edge tiles (reading R1 by selects): the lane holding column 0 takes its own column 0 for its left halo,
      // the lane (of each chunk) holding column W-1 its own column W-1 for its right halo; each tile stores its
      // canonical columns [tx*OW, min((tx+1)*OW, W))
      o << "    const bool lfix = xL == 0;\n"
           "    const int oxlo = tx * OW, oxhi = min(oxlo + OW, W);\n";
      for (int kk = 0; kk < TX; ++kk)
        o << "    const bool stk" << kk << " = (xL + " << 32 * V * kk << " >= oxlo) && (xL + " << 32 * V * kk + V << " <= oxhi);\n"
          << "    const bool rfix" << kk << " = xL + " << 32 * V * kk + V << " == W;\n    (void)rfix" << kk << ";\n";
      o << "    (void)lfix;\n";
    }
    o << ""
         "    const int yend = (y0 + TH < a.gy1) ? (y0 + TH) : a.gy1;\n"
         "    (void)pc; (void)fr; (void)xL; (void)xLh; (void)xb; (void)yend;\n";
    if (hs) {
      o << "    const bool has_next = it + 1 < my_tiles;\n"
           "    if (has_next) p_params(" << (otptb() ? "min(gw + (it + 1) * nwt, a.ntiles - 1)" : "tile + nwt") << ", pn_y0, pn_total";
      for (size_t j = 0; j < g.streams.size(); ++j) o << ", pn_src" << j << ", pn_dst" << j << ", pn_bytes" << j;
      o << ");\n";
    }
    for (int i = 0; i < n; ++i) {
      const GStage& P = g.gs[i];
      if (!P.materialize) continue;
      std::string T = "a.t[" + std::to_string(P.tensor_slot) + "]";
      o << "    char* obase" << i << " = (char*)" << T << ".ptr + (i64)fr * " << T << ".frame_stride + (i64)pc * " << T
        << ".plane_pitch - (i64)" << T << ".row_base * " << T << ".row_pitch + (i64)" << (P.ilv ? "(2 * xL)" : "xL") << " * "
        << dtype_size(p.stages[P.id].dtype) << ";\n";
    }
    for (int i = 0; i < n; ++i) {
      const GStage& P = g.gs[i];
      declare('n', i, p.stages[P.id].dtype == DType::F32, depS(i), P.el, P.er);
    }
    for (size_t j = 0; j < g.streams.size(); ++j) {
      const GStream& S = g.streams[j];
      declare('s', (int)j, S.dtype == DType::F32, depT((int)j), S.el, S.er);
    }
    for (int i = 0; i < n; ++i) {
      const Fold& f = folds[i];
      for (size_t j = 0; j < f.cd.size(); ++j) {
        o << "    float ";
        bool first = true;
        for (int sl = 0; sl < f.cd[j]; ++sl)
          for (int kk = 0; kk < TX; ++kk)
            for (int v = 0; v < V; ++v) {
              o << (first ? "" : ", ") << cname(i, (int)j, sl, kk, v) << " = 0.f";
              first = false;
            }
        o << ";   // carried fold prefix of stage " << p.stages[g.gs[i].id].name << "\n";
      }
    }
    if (interior) {
      // ---- interior tiles: branch-free bodies (warm-up unrolled, main loop, tail) ----
      o << "    {\n";
      if (hs) {
        for (size_t j = 0; j < g.streams.size(); ++j)
          if (g.streams[j].sy == 0)
            o << "      const char* q_ptr" << j << " = p_src" << j << " + (i64)(p_y0 + (TFIRST + " << g.streams[j].hi
              << " + PREF)) * a.t[" << g.streams[j].tensor_slot << "].row_pitch;\n";
      }
      // compile-time ring slots when PREF divides the steps of a tile (every tile then starts at slot 0); the
      // main loop is unrolled by lcm(U, PREF) so that every sub-step's slot is a constant
      int L = Uk;
      bool ct = hs && g.nsteps % k.PREF == 0;
      if (ct) {
        L = Uk / gcd_(Uk, k.PREF) * k.PREF;
        if (L > 24) { ct = false; L = Uk; }
      }
      for (int t = g.t_first; t < 0; ++t) {
        int s_ = t - g.t_first + k.PREF;
        cslot = ct ? (t - g.t_first) % k.PREF : -1;
        step(true, phase_of(t), true, t, s_ < g.nsteps ? 1 : 0);
      }
      // running output row pointers of the main section and tail (row y0 + t + hi at step t = 0)
      for (int i = 0; i < n; ++i)
        if (g.gs[i].materialize)
          o << "      char* optr" << i << " = obase" << i << " + (i64)(y0 + " << g.gs[i].hi << ") * a.t[" << g.gs[i].tensor_slot
            << "].row_pitch;\n";
      // main section: the refill of every step targets this tile (pointer increment, no clamp)
      const int a_end = std::max(0, k.TH - k.PREF) / L * L;
      if (a_end > 0) {
        o << "      for (int tb = 0; tb < " << a_end << "; tb += " << L << ") {\n";
        for (int u = 0; u < L; ++u) {
          o << "      { const int t = tb + " << u << ";\n";
          cslot = ct ? ((u - g.t_first) % k.PREF + k.PREF) % k.PREF : -1;
          step(true, phase_of(u), false, 0, 1);
          o << "      }\n";
        }
        o << "      }\n";
      }
      if (a_end < k.TH) {
        // tail: the refills cross into the next tile (selects, clamped rows)
        o << "      for (int tb = " << a_end << "; tb < TH; tb += " << L << ") {\n";
        for (int u = 0; u < L; ++u) {
          o << "      { const int t = tb + " << u << ";\n      if (t < TH) {\n";
          cslot = ct ? ((u - g.t_first) % k.PREF + k.PREF) % k.PREF : -1;
          step(true, phase_of(u), false, 0, 0);
          o << "      }\n      }\n";
        }
        o << "      }\n";
      }
      cslot = -1;
      o << "    }\n";
    } else {
      // ---- border tiles: general bodies (clamped reads, edge replication, row checks) ----
      o << "    for (int tb = TFIRST; tb < TH; tb += " << Uk << ") {\n";
      for (int u = 0; u < Uk; ++u) {
        o << "      { const int t = tb + " << u << ";\n      if (t < TH) {\n";
        step(false, u, false, 0, 0);
        o << "      }\n      }\n";
      }
      o << "    }\n";
    }
    if (hs) {
      o << "    p_y0 = pn_y0; p_total = pn_total;\n";
      for (size_t j = 0; j < g.streams.size(); ++j)
        o << "    p_src" << j << " = pn_src" << j << "; p_dst" << j << " = pn_dst" << j << "; p_bytes" << j << " = pn_bytes" << j << ";\n";
    }
    o << "  }\n}\n\n";
  }

  void shift_window(bool stage, int i, int depth, int el, int er, const std::string& ind) {
    // shift-mode window (depth does not divide the unroll factor): r{b} = r{b-1}
    for (int b = depth - 1; b >= 1; --b) copy_row(stage ? 'n' : 's', i, el, er, b - 1, b, ind);
  }

  // x-border condition of the scaled streams: the tile's smem row would leave [0, Wp) of the producer
  std::string xb_scaled() const {
    std::string r;
    for (const auto& S : g.streams) {
      if (S.sx == 0) continue;
      std::string o0 = "(" + pcol(S, "cx") + " - " + std::to_string(S.xl) + ")";
      r += " || " + o0 + " < 0 || " + o0 + " + " + std::to_string(S.row_elems) + " > a.t[" + std::to_string(S.tensor_slot) + "].W";
    }
    return r;
  }

  // producer row of stream j at virtual row R, clamped to the rows the producer's buffer holds: the whole
  // image [0, H) for full runs (reading R1), the band's rows [row_base, row_base + nrows) for band runs --
  // rows outside a band only feed outputs outside it, and no copy may leave the caller's buffer
  std::string prow(int j, const std::string& R) const {
    const GStream& S = g.streams[j];
    std::string T = "a.t[" + std::to_string(S.tensor_slot) + "]";
    std::string lo = T + ".row_base", hi = T + ".row_base + " + T + ".nrows - 1";
    if (S.sy == 1) return "pmg_clampi(2 * (" + R + ") + " + std::to_string(S.py) + ", " + lo + ", " + hi + ")";
    if (S.sy == 2) return "pmg_clampi((" + R + ") >> 1, " + lo + ", " + hi + ")";
    return "pmg_clampi(" + R + ", " + lo + ", " + hi + ")";
  }
  // producer column of consumer column `c` (the chunk origin) for the x form of stream j
  static std::string pcol(const GStream& S, const std::string& c) {
    if (S.sx == 1) return "(2 * (" + c + "))";
    if (S.sx == 2) return "((" + c + ") >> 1)";
    return "(" + c + ")";
  }

  void stream_reads(int u, bool fast, const std::string& ind) {
    if (cslot >= 0) {
      // slot known at compile time (PREF divides the steps of a tile): constant addresses, one parity flip per lap
      o << ind << "const int slq = " << cslot << ";\n" << ind << "pmg_mbar_wait(bar0 + 8 * slq, phase);\n";
      if (cslot == g.cfg.PREF - 1) o << ind << "phase ^= 1u;\n";
    } else {
      o << ind << "const int slq = c_slot;\n"
        << ind << "pmg_mbar_wait(bar0 + 8 * slq, phase);\n"
        << ind << "if (slq + 1 == PREF) { c_slot = 0; phase ^= 1u; } else { c_slot = slq + 1; }\n";
    }
    o << ind << "{\n" << ind << "const char* srow = ring + slq * RING;\n";
    for (size_t j = 0; j < g.streams.size(); ++j) {
      const GStream& S = g.streams[j];
      const int SD = depT((int)j);
      bool rot = SD <= 1 || Uk % SD == 0;
      if (!rot) shift_window(false, (int)j, SD, S.el, S.er, ind);
      int sl = rot ? slot(SD, 0, u) : 0;
      std::string ct = ctype(S.dtype);
      int lo = -S.el, hi = V + S.er;
      int vlo = (int)std::floor((double)lo / V) * V, vhi = (int)std::ceil((double)hi / V) * V;
      o << ind << "{\n" << ind << "  const char* sb = srow + " << S.smem_off << ";\n";
      if (!fast) o << ind << "  if (!xb) {\n";
      if (S.sx == 2) {
        // up2: lane base (V/2)*lane; e' -> element floor(e'/2); vectors of V/2 elements
        const int h = V / 2, qlo = (int)std::floor(lo / 2.0), qhi = (hi - 1) / 2;
        for (int kk = 0; kk < TX; ++kk)
          for (int qb = (int)std::floor((double)qlo / h) * h; qb <= qhi; qb += h) {
            o << ind << "    { " << ct << " w[" << h << "]; pmg_lds_vec<" << ct << ", " << h << ">(sb + (" << S.xl << " + "
              << 16 * V * kk << " + " << h << " * lane + (" << qb << ")) * " << S.esz << ", w);";
            for (int e = lo; e < hi; ++e) {
              int q = (int)std::floor(e / 2.0);
              if (q >= qb && q < qb + h) o << " " << tv((int)j, sl, kk, e) << " = PmgElem<" << ct << ">::cv(w[" << q - qb << "]);";
            }
            o << " }\n";
          }
      } else {
        const int lb = S.sx == 1 ? 2 * V : V;   // lane stride in producer elements
        for (int kk = 0; kk < TX; ++kk)
          for (int vb = vlo; vb < vhi; vb += V) {
            o << ind << "    { " << ct << " w[" << V << "]; pmg_lds_vec<" << ct << ", " << V << ">(sb + (" << S.xl << " + "
              << 32 * lb * kk << " + " << lb << " * lane + (" << vb << ")) * " << S.esz << ", w);";
            for (int q = 0; q < V; ++q)
              if (vb + q >= lo && vb + q < hi) o << " " << tv((int)j, sl, kk, vb + q) << " = PmgElem<" << ct << ">::cv(w[" << q << "]);";
            o << " }\n";
          }
        if (fast && xe) {   // x-edge tiles: the halo columns outside [0, W) replicate the edge column (R1)
          for (int e = lo; e < 0; ++e)
            o << ind << "    " << tv((int)j, sl, 0, e) << " = lfix ? " << tv((int)j, sl, 0, 0) << " : " << tv((int)j, sl, 0, e) << ";\n";
          for (int kk = 0; kk < TX; ++kk)
            for (int e = V; e < hi; ++e)
              o << ind << "    " << tv((int)j, sl, kk, e) << " = rfix" << kk << " ? " << tv((int)j, sl, kk, V - 1) << " : "
                << tv((int)j, sl, kk, e) << ";\n";
        }
      }
      if (!fast) {
        // clamped producer columns (reading R1): unit xL+e, down2 2*xL+q, up2 floor((xL+e')/2)
        const std::string Wp = S.sx == 0 ? "W - 1" : "a.t[" + std::to_string(S.tensor_slot) + "].W - 1";
        o << ind << "  } else {\n" << ind << "    const int xo = " << pcol(S, "cx") << " - " << S.xl << ";\n";
        for (int kk = 0; kk < TX; ++kk)
          for (int e = lo; e < hi; ++e) {
            std::string col = S.sx == 1 ? "2 * (xL + " + std::to_string(32 * V * kk) + ") + (" + std::to_string(e) + ")"
                              : S.sx == 2 ? "(xL + " + std::to_string(32 * V * kk + e) + ") >> 1"
                                          : "xL + " + std::to_string(32 * V * kk + e);
            o << ind << "    " << tv((int)j, sl, kk, e) << " = pmg_lds<" << ct << ">(sb, pmg_clampi(" << col << ", 0, " << Wp
              << ") - xo);\n";
          }
        o << ind << "  }\n";
      }
      o << ind << "}\n";
    }
    o << ind << "}\n" << ind << (otptb() ? "__syncthreads();\n" : "__syncwarp();\n");
  }

  // refill the slot read in this step with the request PREF steps ahead (next tile when it crosses NSTEPS)
  void refill(bool tconst, int tval, int rmode, const std::string& ind) {
    std::string tt = tconst ? std::to_string(tval) : "t";
    if (rmode == 1) {
      // same tile, interior: rows need no clamp; the source pointers advance one row per step (scaled rows:
      // the clamped producer row of the virtual row requested, p_y0 + hi + t + PREF)
      auto src_of = [&](int j) {
        if (g.streams[j].sy == 0) return "q_ptr" + std::to_string(j);
        return "p_src" + std::to_string(j) + " + (i64)" + prow(j, "p_y0 + " + std::to_string(g.streams[j].hi) + " + " + tt + " + PREF") +
               " * a.t[" + std::to_string(g.streams[j].tensor_slot) + "].row_pitch";
      };
      auto adv = [&](int j) {
        return g.streams[j].sy == 0 ? "  q_ptr" + std::to_string(j) + " += a.t[" + std::to_string(g.streams[j].tensor_slot) + "].row_pitch;\n"
                                    : std::string();
      };
      // the proxy fence orders the lanes' generic-proxy reads of this slot before the bulk copy that overwrites it
      // (PTX memory model).  Dropping it (PMG_FENCE=0, a round-2 experiment) lost 32 elements of a full-size
      // unsharp run once in many: the reads are usually, not always, complete when the copy lands.
      const char* fe = getenv("PMG_FENCE");
      const bool fence = !(fe && fe[0] == '0');
      if (g.streams.size() == 1) {
        o << ind << "{\n" << ind << "  " << (fence ? "pmg_refill1_elect" : "pmg_refill1_elect_nf")
          << "(bar0 + 8 * slq, p_total, ring_addr + slq * RING + p_dst0, " << src_of(0)
          << ", p_bytes0);\n" << ind << adv(0) << ind << "}\n";
        return;
      }
      o << ind << "{\n" << ind << "  const u32 bar = bar0 + 8 * slq;\n"
        << ind << "  if (leader) {\n"
        << ind << (fence ? "    pmg_fence_proxy_async();\n" : "")
        << ind << "    pmg_mbar_expect_tx(bar, p_total);\n";
      for (size_t j = 0; j < g.streams.size(); ++j)
        o << ind << "    pmg_bulk_g2s(ring_addr + slq * RING + p_dst" << j << ", " << src_of((int)j) << ", p_bytes" << j << ", bar);\n";
      o << ind << "  }\n";
      for (size_t j = 0; j < g.streams.size(); ++j) o << ind << adv((int)j);
      o << ind << "}\n";
      return;
    }
    o << ind << "{\n";
    if (tconst) {
      int s = tval - g.t_first + g.cfg.PREF;
      bool nx = s >= g.nsteps;
      int sr = nx ? s - g.nsteps : s;
      o << ind << "  const bool nx = " << (nx ? "true" : "false") << ";\n" << ind << "  const int sr = " << sr << ";\n";
    } else {
      o << ind << "  const int s = " << tt << " - TFIRST + PREF;\n"
        << ind << "  const bool nx = s >= NSTEPS;\n"
        << ind << "  const int sr = nx ? s - NSTEPS : s;\n";
    }
    if (g.streams.size() == 1) {
      const GStream& S = g.streams[0];
      o << ind << "  const int yq = nx ? pn_y0 : p_y0;\n"
        << ind << "  if (!nx || has_next)\n"
        << ind << "    pmg_refill1_elect(bar0 + 8 * slq, nx ? pn_total : p_total, ring_addr + slq * RING + (nx ? pn_dst0 : p_dst0), "
        << "(nx ? pn_src0 : p_src0) + (i64)" << prow(0, "yq + (TFIRST + " + std::to_string(S.hi) + ") + sr") << " * a.t[" << S.tensor_slot
        << "].row_pitch, nx ? pn_bytes0 : p_bytes0);\n" << ind << "}\n";
      return;
    }
    o << ind << "  const bool go = leader && (!nx || has_next);\n"
      << ind << "  const u32 bar = bar0 + 8 * slq;\n"
      << ind << "  const int yq = nx ? pn_y0 : p_y0;\n"
      << ind << "  pmg_fence_proxy_async_if(go);\n"
      << ind << "  pmg_mbar_expect_tx_if(bar, nx ? pn_total : p_total, go);\n";
    for (size_t j = 0; j < g.streams.size(); ++j) {
      const GStream& S = g.streams[j];
      o << ind << "  pmg_bulk_g2s_if(ring_addr + slq * RING + (nx ? pn_dst" << j << " : p_dst" << j << "), (nx ? pn_src" << j
        << " : p_src" << j << ") + (i64)" << prow((int)j, "yq + (TFIRST + " + std::to_string(S.hi) + ") + sr") << " * a.t[" << S.tensor_slot
        << "].row_pitch, nx ? pn_bytes" << j << " : p_bytes" << j << ", bar, go);\n";
    }
    o << ind << "}\n";
  }

  void store(int i, int cur, bool fast, bool tconst, int tval, const std::string& ind) {
    const GStage& P = g.gs[i];
    DType dt = p.stages[P.id].dtype;
    std::string ct = ctype(dt);
    int esz = dtype_size(dt) * (P.ilv ? 2 : 1);   // interleaved: every other element of the liveout row
    const std::string vst = P.ilv ? "pmg_stg_str2" : "pmg_stg_vec";
    std::string rowv = "row" + std::to_string(i);
    if (fast && tconst) {
      int r = tval + P.hi;
      if (r < 0 || r >= g.cfg.TH) return;   // another tile's row
    }
    bool check_rows = !fast || (!tconst && P.hi > 0);
    std::string T = "a.t[" + std::to_string(P.tensor_slot) + "]";
    std::string inbuf = "(unsigned)(" + rowv + " - " + T + ".row_base) < (unsigned)" + T + ".nrows";
    if (fast && !tconst) {
      // interior main loop / tail: running row pointer (no 64-bit multiply) and a predicated vector store
      std::string pred = inbuf;
      if (check_rows) pred = "(" + rowv + " < yend) && " + pred;
      o << ind << "{\n" << ind << "  char* orow = optr" << i << ";\n" << ind << "  optr" << i << " += " << T << ".row_pitch;\n"
        << ind << "  const bool sp = " << pred << ";\n";
      for (int kk = 0; kk < TX; ++kk) {
        int lo = g.PL - 32 * V * kk <= 0 ? 0 : std::min(32, (g.PL - 32 * V * kk) / V);
        int hi = std::max(0, std::min(32, (g.CW - g.PR - 32 * V * kk) / V));
        if (hi <= lo && !xe) continue;
        o << ind << "  {\n" << ind << "    " << ct << " w[" << V << "] = {";
        for (int v = 0; v < V; ++v) o << (v ? ", " : "") << "(" << ct << ")" << sv(i, cur, kk, v);
        o << "};\n";
        std::string lanes = xe ? " && stk" + std::to_string(kk)
                               : (lo == 0 && hi == 32) ? "" : " && lane >= " + std::to_string(lo) + " && lane < " + std::to_string(hi);
        o << ind << "    " << vst << "_if<" << ct << ", " << V << ">(orow + " << 32 * V * kk * esz << ", w, sp" << lanes << ");\n"
          << ind << "  }\n";
      }
      o << ind << "}\n";
      return;
    }
    o << ind << "{\n";
    if (check_rows) o << ind << "if (" << rowv << " >= y0 && " << rowv << " < yend && " << inbuf << ") {\n";
    else o << ind << "if (" << inbuf << ") {\n";
    o << ind << "  char* orow = obase" << i << " + (i64)" << rowv << " * a.t[" << P.tensor_slot << "].row_pitch;\n";
    if (!fast)
      o << ind << "  const int oxlo = (cx + PL) < 0 ? 0 : (cx + PL);\n"
        << ind << "  const int oxhi = (cx + PL + OW) < W ? (cx + PL + OW) : W;\n";
    for (int kk = 0; kk < TX; ++kk) {
      std::string dst = "orow + " + std::to_string(32 * V * kk * esz);
      if (fast) {
        // interior tile: the output lanes of each chunk are compile-time constants
        int lo = g.PL - 32 * V * kk <= 0 ? 0 : std::min(32, (g.PL - 32 * V * kk) / V);
        int hi = std::max(0, std::min(32, (g.CW - g.PR - 32 * V * kk) / V));
        if (hi <= lo && !xe) continue;
        o << ind << "  {\n" << ind << "    " << ct << " w[" << V << "] = {";
        for (int v = 0; v < V; ++v) o << (v ? ", " : "") << "(" << ct << ")" << sv(i, cur, kk, v);
        o << "};\n";
        std::string cond = xe ? "if (stk" + std::to_string(kk) + ") "
                              : (lo == 0 && hi == 32) ? "" : "if (lane >= " + std::to_string(lo) + " && lane < " + std::to_string(hi) + ") ";
        o << ind << "    " << cond << vst << "<" << ct << ", " << V << ">(" << dst << ", w);\n" << ind << "  }\n";
      } else {
        o << ind << "  {\n" << ind << "    " << ct << " w[" << V << "] = {";
        for (int v = 0; v < V; ++v) o << (v ? ", " : "") << "(" << ct << ")" << sv(i, cur, kk, v);
        o << "};\n";
        o << ind << "    const int xs = xL + " << 32 * V * kk << ";\n"
          << ind << "    if (xs >= oxlo && xs + V <= oxhi) " << vst << "<" << ct << ", " << V << ">(" << dst << ", w);\n"
          << ind << "    else if (xs < oxhi && xs + V > oxlo) {\n";
        for (int v = 0; v < V; ++v)
          o << ind << "      if (xs + " << v << " >= oxlo && xs + " << v << " < oxhi) reinterpret_cast<" << ct << "*>(" << dst
            << ")[" << (P.ilv ? 2 * v : v) << "] = w[" << v << "];\n";
        o << ind << "    }\n" << ind << "  }\n";
      }
    }
    o << ind << "}\n";
    o << ind << "}\n";
  }

  // one step of the wavefront: fast = interior tile (no row/column checks); tconst = t known at emit time
  void step(bool fast, int u, bool tconst, int tval, int rmode) {
    const int n = (int)g.gs.size();
    const std::string ind = "        ";
    o << ind << "{ // " << (fast ? "interior" : "general") << " step" << (tconst ? " t=" + std::to_string(tval) : "") << " phase "
      << u << "\n";
    if (tconst) o << ind << "const int t = " << tval << ";\n";
    if (!g.streams.empty()) stream_reads(u, fast, ind);
    for (int i = 0; i < n; ++i) {
      const GStage& P = g.gs[i];
      const StageDecl& sd = p.stages[P.id];
      const bool folded = fast && folds.size() == g.gs.size() && folds[i].on;
      const int T0 = P.lo - P.hi;
      const int lead = folded ? folds[i].m[0] : 0;                  // earliest fold segment runs `lead` steps ahead
      if (tconst && tval + lead < T0) continue;                      // not active yet (warm-up)
      const bool fin = !tconst || tval >= T0;                       // the stage's own row this step
      const int PD = depS(i);
      bool rot = PD <= 1 || Uk % PD == 0;
      int cur = rot ? slot(PD, 0, u) : 0;
      int prev = rot ? slot(PD, 1, u) : 1;
      std::string rowv = "row" + std::to_string(i);
      o << ind << "// stage " << sd.name << " (hi " << P.hi << ", lo " << P.lo << ", window " << PD << ")\n";
      if (folded && !fin) {   // warm-up: only the early fold segments of later rows
        for (int j = (int)folds[i].m.size() - 2; j >= 0; --j) {
          if (tval + folds[i].m[j] < T0) continue;
          o << ind << "{ // fold segment " << j << " (row +" << folds[i].m[j] << ")\n"
            << ind << "const int " << rowv << " = y0 + t + (" << P.hi + folds[i].m[j] << ");\n" << ind << "(void)" << rowv << ";\n";
          if (pack_on()) fold_segment_pair(i, j, u, cur, ind + "  ");
          else fold_segment(i, j, u, cur, ind + "  ");
          o << ind << "}\n";
        }
        continue;
      }
      std::string in2 = ind;
      if (!fast) {
        o << ind << "if (t >= " << (P.lo - P.hi) << ") {\n";
        in2 = ind + "  ";
      } else {
        o << ind << "{\n";
      }
      o << in2 << "const int " << rowv << " = y0 + t + (" << P.hi << ");\n" << in2 << "(void)" << rowv << ";\n";
      if (!rot) shift_window(true, i, PD, P.el, P.er, in2);
      std::string in3 = in2;
      if (!fast) {
        o << in2 << "if (" << rowv << " >= 0 && " << rowv << " < H) {\n";
        in3 = in2 + "  ";
      }
      if (folded) {
        // consumes the carried prefix first
        if (pack_on()) fold_segment_pair(i, (int)folds[i].m.size() - 1, u, cur, in3);
        else fold_segment(i, (int)folds[i].m.size() - 1, u, cur, in3);
      } else if (fast && pack_stages() && sd.dtype == DType::F32 && pairable(*sd.expr)) {
        for (int kk = 0; kk < TX; ++kk)
          for (int v = 0; v < V / 2; ++v)
            o << in3 << "{ const float2 pv = " << pack(ex2(*sd.expr, i, kk, v, v + V / 2, u)) << "; " << sv(i, cur, kk, v)
              << " = pv.x; " << sv(i, cur, kk, v + V / 2) << " = pv.y; }\n";
      } else {
        for (int kk = 0; kk < TX; ++kk)
          for (int v = 0; v < V; ++v) {
            R val = ex(*sd.expr, Ctx{i, kk, v, u});
            o << in3 << sv(i, cur, kk, v) << " = " << conv_store(val, sd.dtype) << ";\n";
          }
      }
      if (P.xfix && !fast) {
        // border tiles: columns outside [0, W) take the edge value (reading R1)
        o << in3 << "if (xb) {\n";
        for (int side = 0; side < 2; ++side) {
          o << in3 << "  if (" << (side == 0 ? "cx < 0" : "cx + CW > W") << ") {\n"
            << in3 << "    const int off = " << (side == 0 ? "-cx" : "W - 1 - cx") << ";\n"
            << in3 << "    const int kq = off / (32 * V), lq = (off % (32 * V)) / V, eq = off % V;\n"
            << in3 << "    " << rtype(sd.dtype) << " sel = " << sv(i, cur, 0, 0) << ";\n";
          for (int kk = 0; kk < TX; ++kk)
            for (int v = 0; v < V; ++v)
              o << in3 << "    if (kq == " << kk << " && eq == " << v << ") sel = " << sv(i, cur, kk, v) << ";\n";
          o << in3 << "    const " << rtype(sd.dtype) << " edge = pmg_shfl(sel, lq);\n";
          for (int kk = 0; kk < TX; ++kk)
            for (int v = 0; v < V; ++v)
              o << in3 << "    if (xL + " << 32 * V * kk + v << (side == 0 ? " < 0" : " > W - 1") << ") " << sv(i, cur, kk, v)
                << " = edge;\n";
          o << in3 << "  }\n";
        }
        o << in3 << "}\n";
      }
      // extension elements: neighbour lanes / neighbour chunks (load types (3) and (4))
      for (int kk = 0; kk < TX; ++kk) {
        if (hyb(i, kk)) continue;   // shared-memory chunk: consumers read any offset from the smem row
        for (int e = -P.el; e < 0; ++e) {
          int q = (int)std::floor((double)e / V), ee = e - q * V;
          std::string own = sv(i, cur, kk, ee);
          std::string send = kk > 0 ? "(lane >= " + std::to_string(32 + q) + " ? " + sv(i, cur, kk - 1, ee) + " : " + own + ")" : own;
          o << in3 << sv(i, cur, kk, e) << " = pmg_shfl(" << send << ", (lane + (" << q << ")) & 31);\n";
          if (fast && xe && kk == 0) o << in3 << sv(i, cur, kk, e) << " = lfix ? " << sv(i, cur, 0, 0) << " : " << sv(i, cur, kk, e) << ";\n";
        }
        for (int e = V; e < V + P.er; ++e) {
          int q = e / V, ee = e - q * V;
          std::string own = sv(i, cur, kk, ee);
          std::string send = kk + 1 < TX ? "(lane < " + std::to_string(q) + " ? " + sv(i, cur, kk + 1, ee) + " : " + own + ")" : own;
          o << in3 << sv(i, cur, kk, e) << " = pmg_shfl(" << send << ", (lane + " << q << ") & 31);\n";
          if (fast && xe)
            o << in3 << sv(i, cur, kk, e) << " = rfix" << kk << " ? " << sv(i, cur, kk, V - 1) << " : " << sv(i, cur, kk, e) << ";\n";
        }
      }
      if (hyb(i, 0)) {
        // hybrid tiling: the smem chunks' row goes to the window slot in shared memory; the first register
        // chunk also writes the head of its row into the right halo (reads across the S | S+1 boundary)
        std::string ct = ctype(sd.dtype);
        for (int kk = 0; kk < g.cfg.S; ++kk) {
          o << in3 << "{ " << ct << " w[" << V << "] = {";
          for (int v = 0; v < V; ++v) o << (v ? ", " : "") << "(" << ct << ")" << sv(i, cur, kk, v);
          o << "}; pmg_stg_vec<" << ct << ", " << V << ">(" << hyb_ptr(i, cur, kk, "0") << ", w); }\n";
        }
        if (g.cfg.S < TX && P.er > 0)
          for (int v = 0; v < V; ++v)
            o << in3 << "if (V * lane + " << v << " < " << P.er << ") *reinterpret_cast<" << ct << "*>("
              << hyb_ptr(i, cur, g.cfg.S, std::to_string(v)) << ") = (" << ct << ")" << sv(i, cur, g.cfg.S, v) << ";\n";
        o << in3 << "__syncwarp();\n";
      }
      if (!fast) {
        if (PD > 1) {
          o << in3 << "if (" << rowv << " == 0) {\n";
          for (int sl = 0; sl < PD; ++sl)
            if (sl != cur) copy_row('n', i, P.el, P.er, cur, sl, in3 + "  ");
          o << in3 << "}\n" << in2 << "} else if (" << rowv << " >= H) {\n";
          copy_row('n', i, P.el, P.er, prev, cur, in3);
        }
        o << in2 << "}\n";
      }
      if (P.materialize) store(i, cur, fast, tconst, tval, in2);
      if (folded)   // earlier segments of later rows (after the final segment consumed their old values)
        for (int j = (int)folds[i].m.size() - 2; j >= 0; --j) {
          if (tconst && tval + folds[i].m[j] < T0) continue;
          o << in2 << "{ // fold segment " << j << " (row +" << folds[i].m[j] << ")\n"
            << in2 << "const int " << rowv << " = y0 + t + (" << P.hi + folds[i].m[j] << ");\n" << in2 << "(void)" << rowv << ";\n";
          if (pack_on()) fold_segment_pair(i, j, u, cur, in2 + "  ");
          else fold_segment(i, j, u, cur, in2 + "  ");
          o << in2 << "}\n";
        }
      o << ind << "}\n";
      if (otptb()) o << ind << "__syncthreads();   // OTPTB ablation: block barrier between stages\n";
    }
    if (!g.streams.empty()) refill(tconst, tval, rmode, ind);
    o << ind << "}\n";
  }
};

}  // namespace

// registers live across steps in the interior kernel (fold-aware windows, carried prefixes, input windows):
// the selector's register estimate is fitted on this count (select.cpp)
int interior_state_regs(const Analysis& A, const Group& g) {
  Emitter e(A, g);
  return e.state_regs();
}

std::string emit_group(const Analysis& A, const Group& g, bool interior_only) {
  Emitter e(A, g);
  if (interior_only) return e.run_interior_only();
  std::string src = e.run();
  Group gb = g;                        // border kernel: same geometry with TH_b-row tiles
  if (g.TH_b > 0) {
    gb.cfg.TH = g.TH_b;
    gb.nsteps = g.TH_b - g.t_first;
  }
  Emitter eb(A, gb);
  src += eb.run_border();
  return src;
}

}  // namespace pmg
