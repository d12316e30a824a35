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
#include <cstdio>
#include <cstring>
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

  // physical window slot of back index b at sub-step u (rotation when depth | U, else shift naming)
  int slot(int depth, int b, int u) const {
    if (depth <= 1) return 0;
    if (g.U % depth == 0) return ((u - b) % depth + depth) % depth;
    return b;
  }
  std::string sv(int i, int sl, int k, int e) const {
    return "n" + std::to_string(i) + "_r" + std::to_string(sl) + "_c" + std::to_string(k) + "_e" + ename(e);
  }
  std::string tv(int j, int sl, int k, int e) const {
    return "s" + std::to_string(j) + "_r" + std::to_string(sl) + "_c" + std::to_string(k) + "_e" + ename(e);
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
        R idx = toi(ex(*e.args[0], c));
        DType dt = p.tables[e.index].dtype;
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

  R bin(const Expr& e, const Ctx& c) {
    const std::string& op = e.text;
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
      return {sv(gr.idx, slot(P.depth, b, c.u), c.k, c.v + gr.dx), dtype_is_float(dt) ? Kind::Float : Kind::Int};
    }
    if (gr.kind == RKind::STREAM) {
      const GStream& S = g.streams[gr.idx];
      int b = S.hi - C.hi - gr.dy;
      return {tv(gr.idx, slot(S.depth, b, c.u), c.k, c.v + gr.dx), dtype_is_float(S.dtype) ? Kind::Float : Kind::Int};
    }
    // gather: per-element global load with clamped indices (any index form)
    const ReadSite& r = A.reads[ri];
    const Ext3& se = r.src_is_stage ? A.stage_ext[r.src] : A.image_ext[r.src];
    DType dt = r.src_is_stage ? p.stages[r.src].dtype : p.images[r.src].dtype;
    int pnd = (int)e.args.size();
    std::string idx[3] = {"0", "0", "0"};
    for (int i = 0; i < pnd; ++i) {
      int d = i + 3 - pnd;
      R v = toi(ex(*e.args[i], c));
      idx[d] = "pmg_clampi(" + v.s + ", 0, " + std::to_string(se.e[d] - 1) + ")";
    }
    std::string t = "a.t[" + std::to_string(gr.idx) + "]";
    std::string base = "(" + t + ".ptr + (i64)fr * " + t + ".frame_stride + (i64)(" + idx[0] + ") * " + t + ".plane_pitch + (i64)((" + idx[1] + ") - " + t +
                       ".row_base) * " + t + ".row_pitch)";
    return {"pmg_ldg<" + std::string(ctype(dt)) + ">(" + base + ", " + idx[2] + ")", dtype_is_float(dt) ? Kind::Float : Kind::Int};
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

  // ---- kernel text ----
  std::string run() {
    const KConfig& k = g.cfg;
    const int n = (int)g.gs.size();
    o << "// generated by libpmg (emit.cpp) for group " << g.name << ": ";
    for (auto& s : g.gs) o << p.stages[s.id].name << " ";
    o << "\n#include \"pmg_otpw.cuh\"\n\n";
    o << "#define V " << V << "\n#define TX " << TX << "\n#define CW " << g.CW << "\n#define PL " << g.PL
      << "\n#define OW " << g.OW << "\n#define TH " << k.TH << "\n#define NW " << k.NW << "\n#define PREF " << k.PREF
      << "\n#define TFIRST " << g.t_first << "\n#define NSTEPS " << g.nsteps << "\n#define USTEP " << g.U
      << "\n#define RING " << g.ring_bytes << "\n#define WSMEM " << g.warp_smem << "\n#define BARB "
      << ((8 * k.PREF + 15) / 16 * 16) << "\n";
    int xlm = 0, xrm = 0;
    for (auto& S : g.streams) { xlm = std::max(xlm, S.xl); xrm = std::max(xrm, S.xr); }
    o << "#define XLM " << xlm << "\n#define XRM " << xrm << "\n\n";
    int nt = std::max<int>(1, (int)g.tensors.size()), ntab = std::max<int>(1, (int)p.tables.size()),
        np = std::max<int>(1, (int)p.params.size());
    o << "struct PmgArgs {\n  PmgTensor t[" << nt << "];\n  const char* tab[" << ntab << "];\n  int tabn[" << ntab
      << "];\n  int prm[" << np << "];\n  int H, W, gy0, gy1, nty, ntx, npl, nfr, ntiles, pad_;\n};\n\n";
    o << "extern \"C\" __global__ void __launch_bounds__(NW * 32) " << g.name << "(const __grid_constant__ PmgArgs a) {\n";
    o << "  extern __shared__ __align__(128) char pmg_smem[];\n"
         "  const int lane = threadIdx.x & 31;\n"
         "  const int wib = threadIdx.x >> 5;\n"
         "  char* wsm = pmg_smem + wib * WSMEM;\n"
         "  const u32 bar0 = pmg_smem_addr(wsm);\n"
         "  char* ring = wsm + BARB;\n"
         "  (void)ring; (void)bar0;\n"
         "  const int gw = blockIdx.x * NW + wib;\n"
         "  const int nwt = gridDim.x * NW;\n"
         "  if (gw >= a.ntiles) return;\n"
         "  const int H = a.H, W = a.W;\n"
         "  const int my_tiles = (a.ntiles - gw + nwt - 1) / nwt;\n";
    bool has_streams = !g.streams.empty();
    if (has_streams) {
      o << "  if (lane == 0) {\n    for (int i = 0; i < PREF; ++i) pmg_mbar_init(bar0 + 8 * i, 1);\n    pmg_mbar_init_fence();\n  }\n"
           "  __syncwarp();\n"
           "  const long long total_req = (long long)my_tiles * NSTEPS;\n"
           "  long long q_issue = 0;\n  u32 phase = 0u;\n";
      // request issue (lane 0)
      o << "  auto issue = [&](long long q) {\n"
           "    const int itq = (int)(q / NSTEPS), tq = TFIRST + (int)(q % NSTEPS);\n"
           "    const int tile = gw + itq * nwt;\n"
           "    const int txq = tile % a.ntx, rq = tile / a.ntx, tyq = rq % a.nty, rq2 = rq / a.nty, pcq = rq2 % a.npl, frq = rq2 / a.npl;\n"
           "    const int y0q = a.gy0 + tyq * TH, cxq = txq * OW - PL;\n"
           "    const int sl = (int)(q % PREF);\n"
           "    const u32 bar = bar0 + 8 * sl;\n"
           "    char* dst = ring + sl * RING;\n"
           "    u32 bytes = 0;\n"
           "    (void)pcq; (void)frq;\n";
      for (size_t j = 0; j < g.streams.size(); ++j) {
        const GStream& S = g.streams[j];
        const Ext3& se = S.src_is_stage ? A.stage_ext[S.src] : A.image_ext[S.src];
        int Aal = 16 / S.esz;
        o << "    const PmgTensor& T" << j << " = a.t[" << S.tensor_slot << "];\n"
          << "    const int row" << j << " = pmg_clampi(y0q + tq + (" << S.hi << "), 0, H - 1) - T" << j << ".row_base;\n"
          << "    const int pl" << j << " = " << (S.plane_mode == 0 ? "0" : S.plane_mode == 1 ? "pcq" : std::to_string(S.plane_const)) << ";\n"
          << "    const int xlo" << j << " = cxq - " << S.xl << ", xhi" << j << " = cxq + CW + " << S.xr << ";\n"
          << "    const int clo" << j << " = xlo" << j << " < 0 ? 0 : xlo" << j << ";\n"
          << "    const int wa" << j << " = (W + " << (Aal - 1) << ") / " << Aal << " * " << Aal << ";\n"
          << "    const int chi" << j << " = xhi" << j << " > wa" << j << " ? wa" << j << " : xhi" << j << ";\n"
          << "    bytes += (u32)(chi" << j << " - clo" << j << ") * " << S.esz << ";\n";
        (void)se;
      }
      o << "    pmg_mbar_expect_tx(bar, bytes);\n";
      for (size_t j = 0; j < g.streams.size(); ++j) {
        const GStream& S = g.streams[j];
        o << "    pmg_bulk_g2s(pmg_smem_addr(dst + " << S.smem_off << " + (clo" << j << " - xlo" << j << ") * " << S.esz
          << "), T" << j << ".ptr + (i64)frq * T" << j << ".frame_stride + (i64)pl" << j << " * T" << j << ".plane_pitch + (i64)row" << j << " * T" << j
          << ".row_pitch + (i64)clo" << j << " * " << S.esz << ", (u32)(chi" << j << " - clo" << j << ") * " << S.esz
          << ", bar);\n";
      }
      o << "  };\n"
           "  if (lane == 0) {\n    for (; q_issue < total_req && q_issue < PREF; ++q_issue) issue(q_issue);\n  }\n"
           "  long long q_cons = 0;\n";
    }
    // register declarations
    o << "  for (int it = 0; it < my_tiles; ++it) {\n"
         "    const int tile = gw + it * nwt;\n"
         "    const int tx = tile % a.ntx, rr = tile / a.ntx, ty = rr % a.nty, rr2 = rr / a.nty, pc = rr2 % a.npl, fr = rr2 / a.npl;\n"
         "    const int y0 = a.gy0 + ty * TH;\n"
         "    const int cx = tx * OW - PL;\n"
         "    const int xL = cx + V * lane;\n"
         "    const bool xb = (cx - XLM < 0) || (cx + CW + XRM > W);\n"
         "    const int yend = (y0 + TH < a.gy1) ? (y0 + TH) : a.gy1;\n"
         "    (void)pc; (void)fr; (void)xL; (void)xb; (void)yend;\n";
    for (int i = 0; i < n; ++i) {
      const GStage& P = g.gs[i];
      int nslot = P.depth;
      o << "    " << rtype(p.stages[P.id].dtype) << " ";
      bool first = true;
      for (int sl = 0; sl < nslot; ++sl)
        for (int kk = 0; kk < TX; ++kk)
          for (int e = -P.el; e < V + P.er; ++e) {
            o << (first ? "" : ", ") << sv(i, sl, kk, e) << " = 0";
            first = false;
          }
      o << ";\n";
    }
    for (size_t j = 0; j < g.streams.size(); ++j) {
      const GStream& S = g.streams[j];
      o << "    " << rtype(S.dtype) << " ";
      bool first = true;
      for (int sl = 0; sl < S.depth; ++sl)
        for (int kk = 0; kk < TX; ++kk)
          for (int e = -S.el; e < V + S.er; ++e) {
            o << (first ? "" : ", ") << tv((int)j, sl, kk, e) << " = 0";
            first = false;
          }
      o << ";\n";
    }
    o << "    for (int tb = TFIRST; tb < TH; tb += USTEP) {\n";
    for (int u = 0; u < g.U; ++u) step(u);
    o << "    }\n  }\n}\n";
    return o.str();
  }

  void shift_window(bool stage, int i, int depth, int el, int er) {
    // shift-mode window (depth does not divide the unroll factor): r{b} = r{b-1}
    for (int b = depth - 1; b >= 1; --b)
      for (int kk = 0; kk < TX; ++kk)
        for (int e = -el; e < V + er; ++e)
          o << "        " << (stage ? sv(i, b, kk, e) : tv(i, b, kk, e)) << " = " << (stage ? sv(i, b - 1, kk, e) : tv(i, b - 1, kk, e)) << ";\n";
  }

  void step(int u) {
    const int n = (int)g.gs.size();
    o << "      { // sub-step " << u << "\n      const int t = tb + " << u << ";\n      if (t < TH) {\n";
    // ---- group inputs: wait for the ring slot, read this step's rows (type (2): shared memory) ----
    if (!g.streams.empty()) {
      o << "        const int slq = (int)(q_cons % PREF);\n"
           "        pmg_mbar_wait(bar0 + 8 * slq, (phase >> slq) & 1u);\n"
           "        phase ^= 1u << slq;\n"
           "        const char* srow = ring + slq * RING;\n";
      for (size_t j = 0; j < g.streams.size(); ++j) {
        const GStream& S = g.streams[j];
        bool rot = S.depth <= 1 || g.U % S.depth == 0;
        if (!rot) shift_window(false, (int)j, S.depth, S.el, S.er);
        int sl = rot ? slot(S.depth, 0, u) : 0;
        std::string ct = ctype(S.dtype);
        o << "        {\n          const char* sb = srow + " << S.smem_off << ";\n"
          << "          if (!xb) {\n";
        // aligned vector reads covering [-el, V+er) per chunk
        int lo = -S.el, hi = V + S.er;
        int vlo = (int)std::floor((double)lo / V) * V, vhi = (int)std::ceil((double)hi / V) * V;
        for (int kk = 0; kk < TX; ++kk)
          for (int vb = vlo; vb < vhi; vb += V) {
            o << "            { " << ct << " w[" << V << "]; pmg_lds_vec<" << ct << ", " << V << ">(sb + (" << S.xl << " + "
              << 32 * V * kk << " + V * lane + (" << vb << ")) * " << S.esz << ", w);";
            for (int q = 0; q < V; ++q)
              if (vb + q >= lo && vb + q < hi) o << " " << tv((int)j, sl, kk, vb + q) << " = PmgElem<" << ct << ">::cv(w[" << q << "]);";
            o << " }\n";
          }
        o << "          } else {\n"
          << "            const int xo = cx - " << S.xl << ";\n";
        for (int kk = 0; kk < TX; ++kk)
          for (int e = lo; e < hi; ++e)
            o << "            " << tv((int)j, sl, kk, e) << " = pmg_lds<" << ct << ">(sb, pmg_clampi(xL + " << 32 * V * kk + e
              << ", 0, W - 1) - xo);\n";
        o << "          }\n        }\n";
      }
      o << "        __syncwarp();\n"
           "        if (lane == 0 && q_issue < total_req) { pmg_fence_proxy_async(); issue(q_issue); ++q_issue; }\n"
           "        ++q_cons;\n";
    }
    // ---- stages in topological order ----
    for (int i = 0; i < n; ++i) {
      const GStage& P = g.gs[i];
      const StageDecl& sd = p.stages[P.id];
      bool rot = P.depth <= 1 || g.U % P.depth == 0;
      int cur = rot ? slot(P.depth, 0, u) : 0;
      int prev = rot ? slot(P.depth, 1, u) : 1;
      o << "        // stage " << sd.name << " (hi " << P.hi << ", lo " << P.lo << ", window " << P.depth << ")\n"
        << "        if (t >= " << (P.lo - P.hi) << ") {\n"
        << "          const int row" << i << " = y0 + t + (" << P.hi << ");\n";
      if (!rot) shift_window(true, i, P.depth, P.el, P.er);
      o << "          if (row" << i << " >= 0 && row" << i << " < H) {\n";
      for (int kk = 0; kk < TX; ++kk)
        for (int v = 0; v < V; ++v) {
          R val = ex(*sd.expr, Ctx{i, kk, v, u});
          o << "            " << sv(i, cur, kk, v) << " = " << conv_store(val, sd.dtype) << ";\n";
        }
      if (P.xfix) {
        // border tiles: columns outside [0, W) take the edge value (reading R1)
        o << "            if (xb) {\n";
        for (int side = 0; side < 2; ++side) {
          o << "              {\n                const int off = " << (side == 0 ? "-cx" : "W - 1 - cx") << ";\n"
            << "                if (" << (side == 0 ? "cx < 0" : "cx + CW > W") << ") {\n"
            << "                  const int kq = off / (32 * V), lq = (off % (32 * V)) / V, eq = off % V;\n"
            << "                  " << rtype(sd.dtype) << " sel = " << sv(i, cur, 0, 0) << ";\n";
          for (int kk = 0; kk < TX; ++kk)
            for (int v = 0; v < V; ++v)
              o << "                  if (kq == " << kk << " && eq == " << v << ") sel = " << sv(i, cur, kk, v) << ";\n";
          o << "                  const " << rtype(sd.dtype) << " edge = pmg_shfl(sel, lq);\n";
          for (int kk = 0; kk < TX; ++kk)
            for (int v = 0; v < V; ++v)
              o << "                  if (xL + " << 32 * V * kk + v << (side == 0 ? " < 0" : " > W - 1") << ") " << sv(i, cur, kk, v)
                << " = edge;\n";
          o << "                }\n              }\n";
        }
        o << "            }\n";
      }
      // extension elements: neighbour lanes / neighbour chunks (load types (3) and (4))
      for (int kk = 0; kk < TX; ++kk) {
        for (int e = -P.el; e < 0; ++e) {
          int q = (int)std::floor((double)e / V), ee = e - q * V;
          std::string own = sv(i, cur, kk, ee);
          std::string send = kk > 0 ? "(lane >= " + std::to_string(32 + q) + " ? " + sv(i, cur, kk - 1, ee) + " : " + own + ")" : own;
          o << "            " << sv(i, cur, kk, e) << " = pmg_shfl(" << send << ", (lane + (" << q << ")) & 31);\n";
        }
        for (int e = V; e < V + P.er; ++e) {
          int q = e / V, ee = e - q * V;
          std::string own = sv(i, cur, kk, ee);
          std::string send = kk + 1 < TX ? "(lane < " + std::to_string(q) + " ? " + sv(i, cur, kk + 1, ee) + " : " + own + ")" : own;
          o << "            " << sv(i, cur, kk, e) << " = pmg_shfl(" << send << ", (lane + " << q << ") & 31);\n";
        }
      }
      if (P.depth > 1) {
        // first real row of a top-border tile: rows < 0 replicate row 0
        o << "            if (row" << i << " == 0) {\n";
        for (int sl = 0; sl < P.depth; ++sl) {
          if (sl == cur) continue;
          for (int kk = 0; kk < TX; ++kk)
            for (int e = -P.el; e < V + P.er; ++e) o << "              " << sv(i, sl, kk, e) << " = " << sv(i, cur, kk, e) << ";\n";
        }
        o << "            }\n";
        o << "          } else if (row" << i << " >= H) {\n";
        for (int kk = 0; kk < TX; ++kk)
          for (int e = -P.el; e < V + P.er; ++e) o << "            " << sv(i, cur, kk, e) << " = " << sv(i, prev, kk, e) << ";\n";
      }
      o << "          }\n";
      if (P.materialize) {
        DType dt = sd.dtype;
        std::string ct = ctype(dt);
        o << "          if (row" << i << " >= y0 && row" << i << " < yend) {\n"
          << "            const PmgTensor& O = a.t[" << P.tensor_slot << "];\n"
          << "            char* orow = (char*)O.ptr + (i64)fr * O.frame_stride + (i64)pc * O.plane_pitch + (i64)(row" << i << " - O.row_base) * O.row_pitch;\n"
          << "            const int oxlo = (cx + PL) < 0 ? 0 : (cx + PL);\n"
          << "            const int oxhi = (cx + PL + OW) < W ? (cx + PL + OW) : W;\n";
        for (int kk = 0; kk < TX; ++kk) {
          o << "            {\n              const int xs = xL + " << 32 * V * kk << ";\n"
            << "              " << ct << " w[" << V << "] = {";
          for (int v = 0; v < V; ++v) o << (v ? ", " : "") << "(" << ct << ")" << sv(i, cur, kk, v);
          o << "};\n"
            << "              if (xs >= oxlo && xs + V <= oxhi) pmg_stg_vec<" << ct << ", " << V << ">(orow + (i64)xs * " << dtype_size(dt)
            << ", w);\n"
            << "              else {\n";
          for (int v = 0; v < V; ++v)
            o << "                if (xs + " << v << " >= oxlo && xs + " << v << " < oxhi) reinterpret_cast<" << ct
              << "*>(orow)[xs + " << v << "] = w[" << v << "];\n";
          o << "              }\n            }\n";
        }
        o << "          }\n";
      }
      o << "        }\n";
    }
    o << "      }\n      }\n";
  }
};

}  // namespace

std::string emit_group(const Analysis& A, const Group& g) {
  Emitter e(A, g);
  return e.run();
}

}  // namespace pmg
