// select.cpp — the GPU cost model of Alg. 2, its argmin (line 1015) and DP fusion
// (§2.4; Bounded DP-Fusion lines 1347-1349).
//
// Two instantiations of the same cost function:
//   paper mode (paper_analyze_group): the paper's own geometry — warp sizes, warp overlapped
//     tile, scratchpads prod ceil(B_i/W_i)(T_i W_i + O_i^n), used to pin the §3/§4
//     worked examples on the GTX 1080Ti / V100 presets of Table 1;
//   B200 mode (b200_cost): the same seven terms evaluated on this library's kernel (KConfig): shared memory
//     = the TMA ring, registers = the register windows, transactions = TMA row copies.
// Readings of the garbled / undefined symbols (R13-R16):
//   R13 regTile = round(T_split * fracReg) registers per buffered stage per thread (Alg. 1 l.867);
//   R14 tileVol at l.953 = iterations of the load's loop per warp tile; totalTB = tbPerSM (l.939);
//       warpBW = GlMemBW * WarpSize / (NSMs * CoresPerSM) (text P:1081-1083); the w1 term is normalised per
//       output point so that it is O(1) like the other terms;
//   R15 MaxThPerSM = 2048; R16 fracReg grid = integer register-chunk counts (dedupe of {0,0.1,..,1}*T).
#include "select.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <set>
#include <sstream>
#include <tuple>

namespace pmg {

static void set_name(pmg_gpu_spec* s, const char* n) {
  std::memset(s->name, 0, sizeof s->name);
  std::strncpy(s->name, n, sizeof s->name - 1);
}

bool gpu_preset(const std::string& name, pmg_gpu_spec* s) {
  std::memset(s, 0, sizeof *s);
  s->warp_size = 32;
  s->max_threads_per_sm = 2048;        // R15 (absent from Table 1)
  s->gl_tx_size[0] = 32;
  s->gl_tx_size[1] = 128;
  s->max_warps_per_sm = 64;
  s->regs_per_sm = 65536;
  if (name == "gtx1080ti") {           // Table 1
    set_name(s, "gtx1080ti");
    s->nsms = 28; s->cores_per_sm = 128; s->gl_mem_bw = 484e9;
    s->max_shmem_per_tb = 48 * 1024; s->shmem_per_sm = 96 * 1024;
    s->max_tb_per_sm = 16; s->max_regs_per_thread = 256;
    s->l2_bytes = 2816 * 1024; s->sm_clock_hz = 1.58e9;
    return true;
  }
  if (name == "teslav100") {
    set_name(s, "teslav100");
    s->nsms = 80; s->cores_per_sm = 64; s->gl_mem_bw = 898e9;
    s->max_shmem_per_tb = 96 * 1024; s->shmem_per_sm = 96 * 1024;
    s->max_tb_per_sm = 32; s->max_regs_per_thread = 256;
    s->l2_bytes = 6 * 1024 * 1024; s->sm_clock_hz = 1.53e9;
    return true;
  }
  if (name == "b200") {                // SURVEY §7.3; GlMemBW = measured copy bandwidth (MEASURED_PEAKS.json)
    set_name(s, "b200");
    s->nsms = 148; s->cores_per_sm = 128; s->gl_mem_bw = 6538.6e9;
    s->max_shmem_per_tb = 227 * 1024; s->shmem_per_sm = 228 * 1024;
    s->max_tb_per_sm = 32; s->max_regs_per_thread = 255;
    s->l2_bytes = 126LL * 1024 * 1024; s->sm_clock_hz = 1.965e9;
    return true;
  }
  return false;
}

bool weights_preset(const std::string& name, pmg_weights* w) {
  // Table 3; the B200 row starts from the V100 row (weight refit is NEXT-3)
  static const double t1080[7] = {50, 0.5, 45, 20, 2, 100, 1};
  static const double v100[7] = {50, 0.5, 60, 10, 2, 100, 1};
  const double* src = name == "gtx1080ti" ? t1080 : (name == "teslav100" || name == "b200") ? v100 : nullptr;
  if (!src) return false;
  for (int i = 0; i < 7; ++i) w->w[i] = src[i];
  return true;
}

// ---- static profile: operation count of a stage body per point (TimePerIter proxy) ----
static double ops_of(const Expr& e) {
  double c = 0;
  for (auto& a : e.args) c += ops_of(*a);
  switch (e.op) {
    case Expr::BIN:
      if ((e.text == "/" || e.text == "%") && e.kind == Kind::Int && e.args[1]->op == Expr::INT && e.args[1]->ival >= 2 &&
          (e.args[1]->ival & (e.args[1]->ival - 1)) == 0)
        return c + 1;   // shift / mask (emit.cpp)
      if (e.text == "/") return c + (e.kind == Kind::Float ? 8 : 20);
      if (e.text == "%") return c + 20;
      return c + 1;
    case Expr::UN: return c + 1;
    case Expr::CALL:
      if (e.text == "sqrt") return c + 8;
      if (e.text == "lerp") return c + 3;
      if (e.text == "clamp") return c + 2;
      return c + 1;
    case Expr::TABLE: return c + 4;
    default: return c;
  }
}

double stage_ops(const Pipeline& p, int s) { return std::max(1.0, ops_of(*p.stages[s].expr)); }

// Alg. 2: the weighted sum of the seven terms
static void weigh(CostBreakdown& c, const pmg_weights& w) {
  double ratio = c.compute_time > 0 ? c.mem_time / c.compute_time : 0;
  c.cost = w.w[0] * c.txs_per_point + w.w[1] * (1 - c.occupancy) + w.w[2] * ratio + w.w[3] * c.unallocated_sh_mem +
           w.w[4] * c.unused_reg + w.w[5] * c.frac_overlap + w.w[6] * c.extra_tbs;                            // l.981
  if (c.infinite) c.cost = std::numeric_limits<double>::infinity();
}

// ---- the shared tail of Alg. 2 (lines 957-982) ----
static void alg2_tail(CostBreakdown& c, const pmg_gpu_spec& S, const pmg_weights& w, double tile_vol,
                      double time_per_iter_sum, double overlap_pts, double computed_pts, int tx_size) {
  if (c.sh_mem_per_tb > S.max_shmem_per_tb) { c.infinite = true; c.why = "shMemPerTB > MaxShMemPerTb"; }
  c.max_tb_per_sm = std::min(c.sh_mem_per_tb > 0 ? std::floor(S.shmem_per_sm / c.sh_mem_per_tb) : (double)S.max_tb_per_sm,
                             (double)S.max_tb_per_sm);                                                         // l.957
  c.sh_mem_occ = std::min(c.max_tb_per_sm * c.warps_per_tb, (double)S.max_warps_per_sm);                      // l.958
  if (c.reg_per_th > S.max_regs_per_thread) { c.infinite = true; c.why = "regPerTh > MaxRegPerTh"; }           // l.961
  double max_th = std::min(std::floor(S.regs_per_sm / std::max(1.0, c.reg_per_th)), (double)S.max_threads_per_sm);  // l.963
  c.reg_occ = std::floor(max_th / S.warp_size);                                                               // l.965
  c.occupancy = std::min(c.sh_mem_occ, c.reg_occ) / S.max_warps_per_sm;                                      // l.966
  c.warp_bw = S.gl_mem_bw * S.warp_size / (S.nsms * (double)S.cores_per_sm);                                 // l.967 (R14)
  c.mem_time = tx_size * c.total_gl_txs / c.warp_bw;                                                          // l.970
  c.compute_time = time_per_iter_sum * tile_vol;                                                              // l.972
  double shm_per_sm = c.sh_mem_per_tb * c.max_tb_per_sm;                                                      // l.975
  c.unallocated_sh_mem = std::max(0.0, std::min(1.0, 1.0 - shm_per_sm / S.shmem_per_sm));                    // l.976
  double reg_per_sm = c.reg_per_th * S.max_warps_per_sm * S.warp_size;                                        // l.977
  c.unused_reg = std::max(0.0, std::min(1.0, 1.0 - reg_per_sm * c.occupancy / S.regs_per_sm));               // l.978
  c.frac_overlap = computed_pts > 0 ? overlap_pts / computed_pts : 0.0;                                       // l.979 (R12)
  c.extra_tbs = c.max_tb_per_sm > 0 ? std::fmod(std::ceil(c.tb_per_sm), c.max_tb_per_sm) : 0;                // l.980 (R14)
  weigh(c, w);
}

// transactions of one warp access of `n` consecutive elements of `esz` bytes starting at byte `start` (MinGLTxs)
static double min_txs(int64_t start, int64_t nbytes, int tx) {
  if (nbytes <= 0) return 0;
  int64_t a = (int64_t)std::floor((double)start / tx), b = (int64_t)std::floor((double)(start + nbytes - 1) / tx);
  return double(b - a + 1);
}

// ---- B200 time estimate of one group kernel (cost_model 0) ----
// A warp walks its tile row by row (nsteps steps).  One step issues I_step warp instructions: the stage
// bodies for V*TX points per lane plus per-stage shuffles / per-stream loads / fixed TMA+loop overhead.
// The w warps resident on an SM share its 4 issue slots per clock, and one step cannot be shorter than the
// row-delivery latency of a PREF-deep TMA ring.  Static tile striding gives ceil(tiles / slots) tiles to the
// busiest warp.  The kernel cannot beat its HBM time.  Constants were fitted on B200 schedule sweeps
// (profiles/sweep_r01_*.txt, tools/fit_weights.py).
struct TimeModel {
  double c0 = 10, c_stage = 2, c_stream = 0, lat_cycles = 1100, launch_us = 1, c_border = 3, cpi_warp = 6;
  double c_gather = 6;    // per gathered read per point (camera sweeps 3 / 6 / 12: profiles/camera_groupings_r01g.txt)
  double issue_eff = 1.1; // SM issue slots per useful instruction (Harris 6400^2 interior alone: 89 % issue-active)
};
static TimeModel time_model() {
  TimeModel m;
  if (const char* e = getenv("PMG_TM")) {     // calibration hook: "c0,c_stage,c_stream,lat_cycles,launch_us,c_border,cpi_warp[,c_gather]"
    double v[8];
    int n = sscanf(e, "%lf,%lf,%lf,%lf,%lf,%lf,%lf,%lf", &v[0], &v[1], &v[2], &v[3], &v[4], &v[5], &v[6], &v[7]);
    if (n >= 7) m = TimeModel{v[0], v[1], v[2], v[3], v[4], v[5], v[6], n == 8 ? v[7] : m.c_gather};
  }
  return m;
}

// instructions of a stage body per point: like ops_of, but index expressions of reads cost nothing (they are
// resolved at compile time into registers / shuffles / shared-memory offsets)
static double body_ops(const Expr& e) {
  if (e.op == Expr::ACCESS) return 0;
  double c = 0;
  for (auto& a : e.args) c += body_ops(*a);
  switch (e.op) {
    case Expr::BIN:
      if (e.text == "/") return c + (e.kind == Kind::Float ? 8 : 20);
      if (e.text == "%") return c + 20;
      return c + 1;
    case Expr::UN: return c + 1;
    case Expr::CALL:
      if (e.text == "sqrt") return c + 8;
      if (e.text == "lerp") return c + 3;
      if (e.text == "clamp") return c + 2;
      return c + 1;
    case Expr::TABLE: return is_const_int(*e.args[0]) ? 0.0 : c + 4;   // constant index: hoisted (emit.cpp)
    default: return c;
  }
}

// `cond` tests the parity of the stage's x variable (x % 2 ... with only x and literals): with even V the
// emitter folds it per element (emit.cpp x_even), so only one branch of the select is evaluated
static bool x_parity_test(const Expr& e, int nd) {
  std::function<bool(const Expr&)> only_x = [&](const Expr& q) {
    if (q.op == Expr::INT) return true;
    if (q.op == Expr::VAR) return q.index + 3 - nd == 2;
    if (q.op == Expr::BIN && (q.text == "+" || q.text == "-")) return only_x(*q.args[0]) && only_x(*q.args[1]);
    return false;
  };
  std::function<bool(const Expr&)> has_mod = [&](const Expr& q) {
    if (q.op == Expr::BIN && q.text == "%" && q.args[1]->op == Expr::INT && q.args[1]->ival == 2 && only_x(*q.args[0])) return true;
    for (auto& a : q.args)
      if (has_mod(*a)) return true;
    return false;
  };
  if (e.op != Expr::BIN || (e.text != "==" && e.text != "!=")) return false;
  for (int s = 0; s < 2; ++s)
    if (has_mod(*e.args[s]) && (e.args[1 - s]->op == Expr::INT)) return true;
  return false;
}

// body instructions per point with the x-parity selects resolved (even V) and each gathered read charged
// c_gather (reads through registers / shuffles / the TMA ring cost nothing here)
static double eval_cost(const Expr& e, int nd, bool xeven, double c_gather, const std::map<const Expr*, RKind>& kinds) {
  if (e.op == Expr::ACCESS) {
    double c = 0;
    auto it = kinds.find(&e);
    if (it != kinds.end() && it->second == RKind::GATHER) c += c_gather;
    return c;   // index expressions are resolved at compile time or folded into the gather's address
  }
  if (e.op == Expr::CALL && e.text == "select" && xeven && x_parity_test(*e.args[0], nd))
    return std::max(eval_cost(*e.args[1], nd, xeven, c_gather, kinds), eval_cost(*e.args[2], nd, xeven, c_gather, kinds));
  double c = 0;
  for (auto& a : e.args) c += eval_cost(*a, nd, xeven, c_gather, kinds);
  if (e.op == Expr::BIN || e.op == Expr::UN || e.op == Expr::CALL || e.op == Expr::TABLE) {
    // the node's own cost as body_ops counts it (children excluded)
    double self = body_ops(e);
    for (auto& a : e.args) self -= body_ops(*a);
    c += self;
  }
  return c;
}

static double est_time_us(const Analysis& A, const Group& g, const pmg_gpu_spec& S, double resident_warps,
                          CostBreakdown* rec = nullptr, int bands = 1) {
  static const TimeModel M = time_model();
  const Pipeline& p = *A.p;
  const KConfig& k = g.cfg;
  const double H = std::ceil((double)g.ext.e[1] / std::max(1, bands)), W = (double)g.ext.e[2], C = (double)g.npl;
  const double tiles = C * std::ceil(H / k.TH) * std::ceil(W / g.OW);
  // a gathered read (per-element clamped global load, not staged through the TMA ring) costs its index
  // arithmetic and an exposed L2 round trip that the ring would have hidden (c_gather per read per point)
  std::map<const Expr*, RKind> kinds;
  for (auto& P : g.gs)
    for (int ri : A.reads_of[P.id])
      if (g.read_map[ri] >= 0) kinds[A.reads[ri].node] = g.greads[g.read_map[ri]].kind;
  const bool xeven = k.V % 2 == 0 && g.OW % 2 == 0 && g.PL % 2 == 0;
  double ops = 0;
  for (auto& P : g.gs)
    ops += std::max(1.0, eval_cost(*p.stages[P.id].expr, (int)p.stages[P.id].vars.size(), xeven, M.c_gather, kinds));
  const double I_step = k.V * k.TX * ops + k.TX * (M.c_stage * g.gs.size() + M.c_stream * g.streams.size()) + M.c0;
  const double R = std::max(1.0, std::floor(resident_warps));
  const double lat = M.lat_cycles * 4.0 / std::max(1, k.PREF);
  // border tiles run concurrently in the border kernel, in TH_b-row tiles, through the general body (c_border x
  // the instructions) at about half the residency: the top rows and the bottom tile row (the interior's last
  // tile row is shifted up to end at the image), plus -- without x-edge tiles -- the first / last tile columns
  const int THb = g.TH_b > 0 ? g.TH_b : k.TH;
  const double ntx = std::ceil(W / g.OW);
  const double nty_i = H - 2.0 * THb >= k.TH ? std::ceil((H - 2.0 * THb) / k.TH) : 0.0;
  const double ntx_i = g.xedge ? ntx : std::max(0.0, ntx - 2);
  const double it = C * nty_i * ntx_i;
  const double btb = nty_i > 0 ? C * (2 * ntx + (g.xedge ? 0.0 : 2 * nty_i * k.TH / THb)) : C * std::ceil(H / THb) * ntx;
  const double Rb = std::max(1.0, std::floor(R / 2));
  // SM issue bound: the busiest SM issues ceil(tiles / NSMs) tiles' instructions at 4 per clock;
  // warp latency bound: the busiest warp walks ceil(tiles / (R * NSMs)) tiles at <= 1 instruction per clock
  // and no faster than the ring delivers rows
  const double t_sm = (std::ceil(it / S.nsms) * g.nsteps * I_step + std::ceil(btb / S.nsms) * (THb - g.t_first) *
                       I_step * M.c_border) / 4.0;
  const double t_warp = std::max(std::ceil(it / (R * S.nsms)) * g.nsteps * std::max(I_step * M.cpi_warp, lat),
                                 std::ceil(btb / (Rb * S.nsms)) * (THb - g.t_first) *
                                     std::max(I_step * M.c_border * M.cpi_warp, lat));
  const double t_issue = std::max(t_sm * M.issue_eff, t_warp) / S.sm_clock_hz;
  double bytes = 0;
  for (auto& st : g.streams) bytes += (double)(k.TH + st.hi - st.lo) * st.row_elems * st.esz;
  for (auto& P : g.gs)
    if (P.materialize) bytes += (double)k.TH * g.OW * dtype_size(p.stages[P.id].dtype);
  const double t_mem = tiles * bytes / S.gl_mem_bw;
  if (rec) {
    rec->tm_ops = ops; rec->tm_stages = (double)g.gs.size(); rec->tm_streams = (double)g.streams.size();
    rec->tm_nsteps = g.nsteps; rec->tm_tiles = tiles; rec->tm_bytes = tiles * bytes; rec->tm_resident = R;
    rec->tm_border_tiles = btb; rec->tm_border_steps = THb - g.t_first;
  }
  return std::max(t_issue, t_mem) * 1e6 + M.launch_us;
}

std::vector<double> map_time_per_iter(const Pipeline& written, const Pipeline& eff, const double* tpi) {
  std::vector<double> r(eff.stages.size(), 0.0);
  if (!tpi) return r;
  for (size_t i = 0; i < eff.stages.size(); ++i)
    for (size_t j = 0; j < written.stages.size(); ++j)
      if (written.stages[j].name == eff.stages[i].name) r[i] = tpi[j];
  return r;
}

CostBreakdown b200_cost(const Analysis& A, const Group& g, const pmg_gpu_spec& S, const pmg_weights& w, int cost_model,
                        int bands, const double* tpi_measured) {
  const Pipeline& p = *A.p;
  const KConfig& k = g.cfg;
  CostBreakdown c;
  const double H = (double)g.ext.e[1], W = (double)g.ext.e[2], C = (double)g.npl;
  const double tiles = C * std::ceil(H / k.TH) * std::ceil(W / g.OW);
  c.total_threads = tiles * 32;
  c.warps_per_tb = k.NW;
  c.tb_per_sm = tiles / k.NW / S.nsms;                                                                         // l.939
  c.sh_mem_per_tb = g.block_smem;                                                                              // l.942-943
  c.reg_tile = 0;
  // l.960; an estimate above the limit is clipped: ptxas caps the count (and spills), which the probe detects
  c.reg_per_th = std::min<double>(g.regs_est, S.max_regs_per_thread);
  // global transactions per warp tile: TMA row copies of every stream + gathers + output rows
  double txs = 0;
  for (auto& st : g.streams) {
    double rows = k.TH + st.hi - st.lo;
    txs += rows * min_txs(0, (int64_t)st.row_elems * st.esz, k.tx_size);
  }
  double out_pts = (double)g.OW * k.TH;
  for (size_t r = 0; r < g.greads.size(); ++r)
    if (g.greads[r].kind == RKind::GATHER) txs += out_pts / 8.0;     // ~one 32B sector per 8 scattered elements
  c.total_gl_txs = txs;
  c.txs_per_point = txs * k.tx_size / 32.0 / out_pts;   // in 32-byte sector units per output point
  double tpi = 0, computed = 0, useful = 0;
  for (auto& P : g.gs) {
    double pts = (double)g.CW * (k.TH + P.hi - P.lo);
    // TimePerIter: the on-device microbenchmark when given (pmg_profile_stages), else the static
    // operation count at the SM clock
    double t = tpi_measured && tpi_measured[P.id] > 0 ? tpi_measured[P.id] : stage_ops(p, P.id) / S.sm_clock_hz;
    tpi += t * pts / (double)(g.CW * k.TH);
    computed += pts;
    useful += out_pts;
  }
  alg2_tail(c, S, w, (double)g.CW * k.TH, tpi, computed - useful, computed, k.tx_size);
  // B200 readings of two terms for the persistent OTPW grid (R21):
  //  occupancy = resident warps per SM the launch can actually fill (a grid with fewer tiles than resident
  //              slots leaves them empty), over MaxWarpsPerSM;
  //  extraTBs  = idle fraction of the last wave of tiles, 1 - waves / ceil(waves) (0 below one wave, where the
  //              shortfall is already in the occupancy term).
  const double slots = c.occupancy * S.max_warps_per_sm, tiles_ = c.total_threads / S.warp_size;
  // the time model counts the warps the hardware really keeps resident: registers are allocated per warp in
  // units of 256 from the register file of one of the 4 SM sub-partitions (16K registers each), blocks need
  // their shared memory plus 1 KB of reserve, at most 32 blocks and 64 warps per SM
  double hw_slots = 0;
  {
    const int r = std::max(8, ((int)std::ceil(c.reg_per_th) + 7) / 8 * 8);
    const int per_smsp = (int)(S.regs_per_sm / 4) / (r * 32);
    const int nw = std::max(1, k.NW);
    const int64_t by_regs = (int64_t)(4 * per_smsp) / nw;
    const int64_t by_smem = S.shmem_per_sm / std::max<int64_t>(1, g.block_smem + 1024);
    const int64_t blocks = std::min<int64_t>({by_regs, by_smem, (int64_t)S.max_tb_per_sm, (int64_t)(S.max_warps_per_sm / nw)});
    hw_slots = (double)(blocks * nw);
  }
  c.est_us = slots > 0 && hw_slots > 0 ? est_time_us(A, g, S, hw_slots, &c, bands) : std::numeric_limits<double>::infinity();
  if (slots > 0) {
    c.occupancy = std::min(slots, tiles_ / S.nsms) / S.max_warps_per_sm;
    const double waves = tiles_ / (slots * S.nsms);
    c.extra_tbs = waves <= 1 ? 0.0 : 1.0 - waves / std::ceil(waves);
  }
  weigh(c, w);
  c.alg2_cost = c.cost;
  if (cost_model == 0 && !c.infinite) c.cost = c.est_us;
  return c;
}

static bool feasible_stage_set(const Analysis& A, const std::vector<int>& stages) {
  // cheap pre-check: same extents
  // same (y, x) extents; plane dims equal or absent (broadcast stages in a plane group, group.cpp)
  const Ext3* pe = nullptr;
  for (int s : stages) {
    const Ext3& e = A.stage_ext[s];
    const Ext3& f = A.stage_ext[stages[0]];
    if (e.e[1] != f.e[1] || e.e[2] != f.e[2] || e.has[1] != f.has[1]) return false;
    if (e.has[0]) {
      if (pe && !(*pe == e)) return false;
      pe = &e;
    }
  }
  return true;
}

bool best_config(const Analysis& A, Group& g, const std::vector<int>& gos, const pmg_gpu_spec& S, const pmg_weights& w,
                 const pmg_sched_opts& o, CostBreakdown* out, const RegProbe* probe) {
  std::vector<int> Vs = o.vec > 0 ? std::vector<int>{o.vec} : std::vector<int>{1, 2, 4};
  std::vector<int> TXs = o.chunks > 0 ? std::vector<int>{o.chunks} : std::vector<int>{1, 2, 4};
  std::vector<int> THs = o.rows > 0 ? std::vector<int>{o.rows} : std::vector<int>{8, 16, 24, 32, 48, 64, 80, 96, 100, 112, 128};
  // NW: OTPW warps are independent, so the block size only sets the register budget ptxas plans for; one warp
  // per block was fastest or tied in every B200 sweep (profiles/sweep_r05_*), larger blocks via the override
  std::vector<int> NWs = o.warps > 0 ? std::vector<int>{o.warps} : std::vector<int>{1};
  // PREF: 4 rows in flight per warp is what the time model was fitted on (profiles/sweep_*); deeper rings are
  // available through the override
  std::vector<int> PFs = o.prefetch > 0 ? std::vector<int>{o.prefetch} : std::vector<int>{4};
  std::vector<int> TXSZ = o.tx_size > 0 ? std::vector<int>{o.tx_size} : std::vector<int>{32, 128};
  std::vector<int> Ss = o.smem_chunks >= 0 ? std::vector<int>{o.smem_chunks} : std::vector<int>{0};
  struct Cand { Group g; CostBreakdown c; };
  std::vector<Cand> cands;
  std::string why = "no candidate";
  long count = 0;
  for (int V : Vs)
    for (int TX : TXs)
      for (int S_ : Ss)
        for (int TH : THs)
          for (int NW : NWs)
            for (int PF : PFs)
              for (int tx : TXSZ) {
                if (o.budget > 0 && count >= o.budget) break;
                if (S_ > TX) continue;
                Group cand;
                cand.stages = g.stages;
                cand.cfg = KConfig{V, TX, S_, TH, NW, PF, tx, o.regcap > 0 ? o.regcap : 0, o.reassoc != 0,
                                  o.border_rows > 0 ? o.border_rows : 8};
                ++count;
                if (!build_group(A, cand, gos)) { why = cand.why_infeasible; continue; }
                CostBreakdown c = b200_cost(A, cand, S, w, o.cost_model, o.bands, o.time_per_iter);
                if (c.infinite) { why = c.why; continue; }
                cands.push_back({cand, c});
              }
  if (cands.empty()) { g.why_infeasible = why; return false; }
  // tie-break: smaller tile volume, smaller block, larger fracReg, larger txSz
  auto better = [](const Cand& a, const Cand& b) {
    if (std::fabs(a.c.cost - b.c.cost) > 1e-12) return a.c.cost < b.c.cost;
    auto vol = [](const KConfig& q) { return (double)q.V * q.TX * q.TH; };
    if (vol(a.g.cfg) != vol(b.g.cfg)) return vol(a.g.cfg) < vol(b.g.cfg);
    if (a.g.cfg.NW != b.g.cfg.NW) return a.g.cfg.NW < b.g.cfg.NW;
    if (a.g.cfg.S != b.g.cfg.S) return a.g.cfg.S < b.g.cfg.S;
    return a.g.cfg.tx_size > b.g.cfg.tx_size;
  };
  std::sort(cands.begin(), cands.end(), better);
  // finalists: replace the register estimate by ptxas' count (RegUsage "measured with nvcc").  The count
  // depends on (V, TX, NW) but hardly on TH / txSz, so the best candidate of each of the first few distinct
  // (V, TX, NW) keys is compiled and its count applied to every candidate with that key; spilling keys are
  // rejected (their registers exceed MaxRegPerTh)
  if (probe && *probe) {
    const size_t KEYS = 6;
    std::map<std::tuple<int, int, int>, std::pair<int, int>> meas;
    for (size_t i = 0; i < cands.size() && meas.size() < KEYS; ++i) {
      auto key = std::make_tuple(cands[i].g.cfg.V, cands[i].g.cfg.TX, cands[i].g.cfg.NW);
      if (meas.count(key)) continue;
      int regs = -1, spill = -1;
      if (!(*probe)(cands[i].g, &regs, &spill) || regs <= 0) regs = -1;
      meas[key] = {regs, spill};
    }
    std::vector<Cand> fin;
    for (auto& c0 : cands) {
      auto it = meas.find(std::make_tuple(c0.g.cfg.V, c0.g.cfg.TX, c0.g.cfg.NW));
      if (it == meas.end() || it->second.first <= 0) continue;
      Cand c = c0;
      c.g.regs_est = it->second.first;
      c.c = b200_cost(A, c.g, S, w, o.cost_model, o.bands, o.time_per_iter);
      if (it->second.second > 0) { c.c.infinite = true; c.c.why = "register spills"; c.c.cost = std::numeric_limits<double>::infinity(); }
      fin.push_back(c);
    }
    std::sort(fin.begin(), fin.end(), better);
    if (getenv("PMG_SCHED_TRACE"))
      for (size_t i = 0; i < fin.size() && i < 6; ++i) {
        auto& f = fin[i];
        fprintf(stderr, "[pmg sched] %zu stages V%d TX%d TH%d NW%d PF%d regs %d est %.2f cost %.4f%s\n", f.g.stages.size(),
                f.g.cfg.V, f.g.cfg.TX, f.g.cfg.TH, f.g.cfg.NW, f.g.cfg.PREF, f.g.regs_est, f.c.est_us, f.c.cost,
                f.c.infinite ? " (inf)" : "");
      }
    if (!fin.empty() && !fin[0].c.infinite) {
      g = fin[0].g;
      if (out) *out = fin[0].c;
      return true;
    }
  }
  g = cands[0].g;
  if (out) *out = cands[0].c;
  return true;
}

Schedule schedule(const Analysis& A, const pmg_gpu_spec& S, const pmg_weights& w, const pmg_sched_opts& o,
                  const RegProbe* probe) {
  const Pipeline& p = *A.p;
  const int n = (int)p.stages.size();
  Schedule sch;
  auto name_groups = [&](Schedule& s) {
    for (size_t i = 0; i < s.groups.size(); ++i) s.groups[i].name = "pmg_g" + std::to_string(i);
  };
  if (o.group_of_stage) {
    // explicit grouping: one group per distinct index, in a topological order of the group DAG (ties: first
    // occurrence in p.topo); a grouping whose groups depend on each other cyclically is rejected
    std::vector<int> gos(o.group_of_stage, o.group_of_stage + n);
    std::vector<int> labels;
    for (int s : p.topo)
      if (std::find(labels.begin(), labels.end(), gos[s]) == labels.end()) labels.push_back(gos[s]);
    std::vector<int> seen;
    // labels in increasing order when that order is topological (a schedule replayed from its group indices keeps
    // its group order, and with it the lane assignment); otherwise a topological order of the group DAG
    {
      std::vector<int> sorted = labels;
      std::sort(sorted.begin(), sorted.end());
      bool topo_ok = true;
      for (int s2 = 0; s2 < n && topo_ok; ++s2)
        for (int q : p.producers[s2])
          if (gos[q] > gos[s2]) topo_ok = false;
      if (topo_ok) seen = sorted;
    }
    if (seen.empty()) {
      const size_t L = labels.size();
      auto li = [&](int lab) { return (int)(std::find(labels.begin(), labels.end(), lab) - labels.begin()); };
      std::vector<std::set<int>> preds(L);
      for (int s = 0; s < n; ++s)
        for (int q : p.producers[s])
          if (gos[q] != gos[s]) preds[li(gos[s])].insert(li(gos[q]));
      std::vector<bool> done(L, false);
      for (size_t k = 0; k < L; ++k) {
        int pick = -1;
        for (size_t c = 0; c < L && pick < 0; ++c) {
          if (done[c]) continue;
          bool ok = true;
          for (int q : preds[c]) ok = ok && done[q];
          if (ok) pick = (int)c;
        }
        if (pick < 0) throw Error(PMG_ERR_INFEASIBLE, "explicit grouping: groups depend on each other cyclically");
        done[pick] = true;
        seen.push_back(labels[pick]);
      }
    }
    sch.group_of_stage = gos;
    std::ostringstream js;
    double total = 0;
    js << "{\"mode\":\"manual\",\"groups\":[";
    for (size_t gi = 0; gi < seen.size(); ++gi) {
      Group g;
      for (int s : p.topo)
        if (gos[s] == seen[gi]) g.stages.push_back(s);
      CostBreakdown cb;
      if (!best_config(A, g, gos, S, w, o, &cb, probe))
        throw Error(PMG_ERR_INFEASIBLE, "group " + std::to_string(gi) + ": " + g.why_infeasible);
      g.name = "pmg_g" + std::to_string(gi);
      js << (gi ? "," : "") << "{\"config\":" << config_json(A, g) << ",\"cost\":" << cost_json(cb) << "}";
      total += cb.cost;
      sch.groups.push_back(g);
    }
    js << "],\"total_cost\":" << total << "}";
    sch.json = js.str();
    name_groups(sch);
    return sch;
  }
  // DP over contiguous runs of a topological order (each run is convex): best[j] = min_i best[i] + cost(i..j).
  // Two orders are tried -- producers as early as possible (p.topo: declaration order among ready stages) and
  // as late as possible (ALAP: each stage right before its first consumer; a pyramid's per-level output
  // stages then sit next to the same-extent stage that consumes them, e.g. the local Laplacian's outLP_j and
  // outG_j) -- and the order with the smaller DP cost is kept.
  const double INF = std::numeric_limits<double>::infinity();
  std::vector<int> alap;
  {
    std::vector<int> rem(n);
    for (int s = 0; s < n; ++s) rem[s] = (int)p.consumers[s].size();
    std::set<int> ready;
    for (int s = 0; s < n; ++s)
      if (!rem[s]) ready.insert(s);
    while (!ready.empty()) {
      // from the end: a ready stage of the extent just placed first (it can join that stage's group), else the
      // latest declaration
      int s = *ready.rbegin();
      if (!alap.empty())
        for (auto it = ready.rbegin(); it != ready.rend(); ++it)
          if (A.stage_ext[*it] == A.stage_ext[alap.back()] || (A.stage_ext[*it].e[1] == A.stage_ext[alap.back()].e[1] &&
                                                               A.stage_ext[*it].e[2] == A.stage_ext[alap.back()].e[2])) {
            s = *it;
            break;
          }
      ready.erase(s);
      alap.push_back(s);
      for (int q : p.producers[s])
        if (--rem[q] == 0) ready.insert(q);
    }
    std::reverse(alap.begin(), alap.end());
  }
  const bool fuse = o.fuse != 0;
  struct DP {
    std::vector<double> best;
    std::vector<int> from;
    std::vector<std::vector<Group>> seg_group;
  };
  auto run_dp = [&](const std::vector<int>& ord) {
    DP d;
    d.best.assign(n + 1, INF);
    d.from.assign(n + 1, -1);
    d.seg_group.assign(n + 1, std::vector<Group>(n + 1));
    d.best[0] = 0;
    for (int j = 1; j <= n; ++j) {
      for (int i = j - 1; i >= 0; --i) {
        if (!fuse && j - i > 1) break;
        if (d.best[i] == INF) continue;
        std::vector<int> seg(ord.begin() + i, ord.begin() + j);
        if (!feasible_stage_set(A, seg)) continue;
        // grouping vector: stages of seg in group 0, every other stage in its own group
        std::vector<int> gos(n);
        for (int s = 0; s < n; ++s) gos[s] = s + 1;
        for (int s : seg) gos[s] = 0;
        Group g;
        g.stages = seg;
        CostBreakdown cb;
        if (!best_config(A, g, gos, S, w, o, &cb)) continue;
        d.seg_group[i][j] = g;
        if (d.best[i] + cb.cost < d.best[j]) { d.best[j] = d.best[i] + cb.cost; d.from[j] = i; }
      }
      if (d.best[j] == INF) throw Error(PMG_ERR_INFEASIBLE, "no feasible group ends at stage " + p.stages[ord[j - 1]].name);
    }
    return d;
  };
  DP dp = run_dp(p.topo);
  std::vector<int> topo = p.topo;
  bool late = false;
  const char* ord_env = getenv("PMG_ORDER");   // experiment knob: "asap" / "alap" forces one order
  if (alap != p.topo && fuse && !(ord_env && std::strcmp(ord_env, "asap") == 0)) {
    DP d2 = run_dp(alap);
    if (d2.best[n] < dp.best[n] - 1e-9 || (ord_env && std::strcmp(ord_env, "alap") == 0)) {
      dp = std::move(d2);
      topo = alap;
      late = true;
    }
  }
  std::vector<double>& best = dp.best;
  std::vector<int>& from = dp.from;
  std::vector<std::vector<Group>>& seg_group = dp.seg_group;
  std::vector<std::pair<int, int>> segs;
  for (int j = n; j > 0; j = from[j]) segs.push_back({from[j], j});
  std::reverse(segs.begin(), segs.end());
  auto gos_of = [&](const std::vector<std::pair<int, int>>& sg) {
    std::vector<int> v(n, -1);
    for (size_t gi = 0; gi < sg.size(); ++gi)
      for (int q = sg[gi].first; q < sg[gi].second; ++q) v[topo[q]] = (int)gi;
    return v;
  };
  // probed merge pass: the DP costs segments with the register *estimate*, which over-estimates large fused
  // groups (the interior kernel's folds shrink them); try merging neighbours with ptxas' counts and keep a
  // merge when the probed pipeline estimate drops
  if (probe && *probe && fuse && segs.size() > 1) {
    auto probed = [&](const std::vector<std::pair<int, int>>& sg, double& total) {
      std::vector<int> gv = gos_of(sg);
      total = 0;
      for (auto& q : sg) {
        Group h;
        h.stages.assign(topo.begin() + q.first, topo.begin() + q.second);
        CostBreakdown cb;
        if (!best_config(A, h, gv, S, w, o, &cb, probe) || cb.infinite) return false;
        total += cb.cost;
      }
      return true;
    };
    double cur;
    if (probed(segs, cur)) {
      for (bool changed = true; changed && segs.size() > 1;) {
        changed = false;
        for (size_t gi = 0; gi + 1 < segs.size(); ++gi) {
          std::vector<int> merged(topo.begin() + segs[gi].first, topo.begin() + segs[gi + 1].second);
          if (!feasible_stage_set(A, merged)) continue;
          auto trial = segs;
          trial[gi].second = trial[gi + 1].second;
          trial.erase(trial.begin() + gi + 1);
          double t;
          if (probed(trial, t) && t < cur) {
            segs = trial;
            cur = t;
            changed = true;
            break;
          }
        }
      }
    }
  }
  sch.group_of_stage = gos_of(segs);
  std::ostringstream js;
  js << "{\"mode\":\"dp\",\"order\":\"" << (late ? "alap" : "asap") << "\",\"dp_cost\":" << best[n] << ",\"groups\":[";
  for (size_t gi = 0; gi < segs.size(); ++gi) {
    Group g = seg_group[segs[gi].first][segs[gi].second];
    // re-select with the final grouping (materialisation depends on the other groups) and with the
    // register probe for the finalists
    Group h;
    h.stages = g.stages;
    CostBreakdown cb;
    if (!best_config(A, h, sch.group_of_stage, S, w, o, &cb, probe)) throw Error(PMG_ERR_INFEASIBLE, h.why_infeasible);
    h.name = "pmg_g" + std::to_string(gi);
    js << (gi ? "," : "") << "{\"config\":" << config_json(A, h) << ",\"cost\":" << cost_json(cb) << "}";
    sch.groups.push_back(h);
  }
  js << "]}";
  sch.json = js.str();
  return sch;
}

std::string cost_json(const CostBreakdown& c) {
  std::ostringstream o;
  o.precision(10);
  auto num = [&](double v) { if (std::isinf(v)) o << "\"inf\""; else o << v; };
  o << "{\"totalThreads\":"; num(c.total_threads);
  o << ",\"warpsPerTB\":"; num(c.warps_per_tb);
  o << ",\"tbPerSM\":"; num(c.tb_per_sm);
  o << ",\"shMemPerTB\":"; num(c.sh_mem_per_tb);
  o << ",\"regTile\":"; num(c.reg_tile);
  o << ",\"regPerTh\":"; num(c.reg_per_th);
  o << ",\"totalGLMemTxs\":"; num(c.total_gl_txs);
  o << ",\"txsPerPoint\":"; num(c.txs_per_point);
  o << ",\"maxTBPerSM\":"; num(c.max_tb_per_sm);
  o << ",\"shMemOcc\":"; num(c.sh_mem_occ);
  o << ",\"regOcc\":"; num(c.reg_occ);
  o << ",\"occupancy\":"; num(c.occupancy);
  o << ",\"warpBW\":"; num(c.warp_bw);
  o << ",\"memTime\":"; num(c.mem_time);
  o << ",\"computeTime\":"; num(c.compute_time);
  o << ",\"unallocatedShMem\":"; num(c.unallocated_sh_mem);
  o << ",\"unusedReg\":"; num(c.unused_reg);
  o << ",\"fracOverlap\":"; num(c.frac_overlap);
  o << ",\"extraTBs\":"; num(c.extra_tbs);
  o << ",\"estUs\":"; num(c.est_us);
  o << ",\"alg2Cost\":"; num(c.alg2_cost);
  o << ",\"tm\":{\"ops\":" << c.tm_ops << ",\"stages\":" << c.tm_stages << ",\"streams\":" << c.tm_streams
    << ",\"nsteps\":" << c.tm_nsteps << ",\"tiles\":" << c.tm_tiles << ",\"bytes\":" << c.tm_bytes
    << ",\"resident\":" << c.tm_resident << ",\"border_tiles\":" << c.tm_border_tiles << ",\"border_steps\":"
    << c.tm_border_steps << "}";
  o << ",\"cost\":"; num(c.cost);
  o << ",\"infinite\":" << (c.infinite ? "true" : "false") << ",\"why\":\"" << c.why << "\"}";
  return o.str();
}

std::string config_json(const Analysis& A, const Group& g) {
  const Pipeline& p = *A.p;
  const KConfig& k = g.cfg;
  std::ostringstream o;
  o << "{\"name\":\"" << g.name << "\",\"stages\":[";
  for (size_t i = 0; i < g.gs.size(); ++i) o << (i ? "," : "") << "\"" << p.stages[g.gs[i].id].name << "\"";
  o << "],\"V\":" << k.V << ",\"TX\":" << k.TX << ",\"S\":" << k.S << ",\"TH\":" << k.TH << ",\"TH_b\":" << g.TH_b << ",\"NW\":" << k.NW
    << ",\"PREF\":" << k.PREF << ",\"txSz\":" << k.tx_size << ",\"fracReg\":" << double(k.TX - k.S) / k.TX
    << ",\"tile\":[" << k.V * k.TX << "," << k.TH << ",1],\"block\":[" << 32 * k.NW << ",1,1],\"warp\":[32,1,1]"
    << ",\"CW\":" << g.CW << ",\"OW\":" << g.OW << ",\"PL\":" << g.PL << ",\"PR\":" << g.PR << ",\"t_first\":" << g.t_first
    << ",\"unroll\":" << g.U << ",\"warp_smem\":" << g.warp_smem << ",\"regs_est\":" << g.regs_est << ",\"state_regs\":" << interior_state_regs(A, g)
    << ",\"stage_geom\":[";
  for (size_t i = 0; i < g.gs.size(); ++i) {
    auto& P = g.gs[i];
    o << (i ? "," : "") << "{\"stage\":\"" << p.stages[P.id].name << "\",\"hi\":" << P.hi << ",\"lo\":" << P.lo
      << ",\"window\":" << P.depth << ",\"ext\":[" << P.el << "," << P.er << "],\"invalid\":[" << P.vl << "," << P.vr
      << "],\"materialize\":" << (P.materialize ? "true" : "false") << "}";
  }
  o << "],\"streams\":[";
  for (size_t j = 0; j < g.streams.size(); ++j) {
    auto& S = g.streams[j];
    o << (j ? "," : "") << "{\"src\":\"" << (S.src_is_stage ? p.stages[S.src].name : p.images[S.src].name)
      << "\",\"plane_mode\":" << S.plane_mode << ",\"hi\":" << S.hi << ",\"lo\":" << S.lo << ",\"window\":" << S.depth
      << ",\"smem_ext\":[" << S.xl << "," << S.xr << "],\"scale\":[" << S.sy << "," << S.py << "," << S.sx << "]}";
  }
  int ng = 0;
  for (auto& r : g.greads) ng += r.kind == RKind::GATHER;
  o << "],\"gathers\":" << ng << "}";
  return o.str();
}

// ------------------------------------------------------------------------------------------ paper mode
std::string paper_analyze_group(const Analysis& A, const std::vector<int>& stages, const int T[3], const int B[3],
                                double f, int tx, int regs_per_stage, const pmg_gpu_spec& S, const pmg_weights& w) {
  const Pipeline& p = *A.p;
  // paper dims (x, y, z) <- normalised (2, 1, 0)
  const int pd[3] = {2, 1, 0};
  std::array<int, 3> Bv{B[0], B[1], B[2]};
  // pad the block to a multiple of WarpSize along x
  int threads = B[0] * B[1] * B[2];
  if (threads % S.warp_size) {
    int x = B[0];
    while ((x * B[1] * B[2]) % S.warp_size) ++x;
    Bv[0] = x;
  }
  std::array<int, 3> W = warp_sizes(Bv, S.warp_size);
  int wt[3] = {T[0] * W[0], T[1] * W[1], T[2] * W[2]};
  int warps_per_dim[3] = {(Bv[0] + W[0] - 1) / W[0], (Bv[1] + W[1] - 1) / W[1], (Bv[2] + W[2] - 1) / W[2]};
  // overlaps O_i^n: backward accumulation of left+right reach from the group's liveouts
  const int n = (int)p.stages.size();
  std::vector<char> in(n, 0);
  for (int s : stages) in[s] = 1;
  std::vector<std::array<int, 3>> L(n, {0, 0, 0}), Rr(n, {0, 0, 0});
  std::vector<char> live(n, 0);
  for (int s : stages) {
    bool lo = std::find(p.liveouts.begin(), p.liveouts.end(), s) != p.liveouts.end();
    for (int c : p.consumers[s])
      if (!in[c]) lo = true;
    live[s] = lo;
  }
  bool constant = true;
  std::vector<int> order;
  for (int s : p.topo)
    if (in[s]) order.push_back(s);
  for (int ii = (int)order.size() - 1; ii >= 0; --ii) {
    int s = order[ii];
    for (int c : p.consumers[s]) {
      if (!in[c]) continue;
      for (int ri : A.reads_of[c]) {
        const ReadSite& r = A.reads[ri];
        if (!r.src_is_stage || r.src != s) continue;
        for (int d = 0; d < 3; ++d) {
          int nd = pd[d];
          int64_t off = 0;
          if (r.form[nd] == Form::UNIT) off = r.off[nd];
          else if (r.form[nd] != Form::ABSENT) constant = false;
          L[s][d] = std::max(L[s][d], L[c][d] + (int)std::max<int64_t>(0, -off));
          Rr[s][d] = std::max(Rr[s][d], Rr[c][d] + (int)std::max<int64_t>(0, off));
        }
      }
    }
  }
  std::ostringstream o;
  o.precision(12);
  o << "{\"block\":[" << Bv[0] << "," << Bv[1] << "," << Bv[2] << "],\"warp\":[" << W[0] << "," << W[1] << "," << W[2]
    << "],\"warp_tile\":[" << wt[0] << "," << wt[1] << "," << wt[2] << "],\"stages\":[";
  double shmem_floats = 0, redundant = 0, computed = 0;
  int buffers = 0;
  for (size_t i = 0; i < order.size(); ++i) {
    int s = order[i];
    double pts = 1, useful = 1, spad = 1;
    int O[3];
    for (int d = 0; d < 3; ++d) {
      O[d] = L[s][d] + Rr[s][d];
      pts *= wt[d] + O[d];
      useful *= wt[d];
      spad *= warps_per_dim[d] * (wt[d] + O[d]);   // prod ceil(B_i/W_i)(T_i W_i + O_i^n)
    }
    o << (i ? "," : "") << "{\"stage\":\"" << p.stages[s].name << "\",\"overlap\":[" << O[0] << "," << O[1] << "," << O[2]
      << "],\"scratchpad\":" << spad << ",\"liveout\":" << (live[s] ? "true" : "false") << "}";
    if (!live[s]) {
      shmem_floats += spad;
      redundant += pts - useful;
      computed += pts;
      ++buffers;
    }
  }
  o << "],\"overlap_numerator\":" << redundant << ",\"overlap_denominator\":" << computed << ",";
  CostBreakdown c;
  int64_t dims[3] = {A.stage_ext[order.back()].e[2], A.stage_ext[order.back()].e[1], A.stage_ext[order.back()].e[0]};
  double total_threads = 1;
  for (int d = 0; d < 3; ++d) total_threads *= std::ceil((double)dims[d] / T[d]);
  int tb = Bv[0] * Bv[1] * Bv[2];
  c.total_threads = total_threads;                                        // l.933
  c.warps_per_tb = tb / (double)S.warp_size;                              // l.938
  c.tb_per_sm = total_threads / tb / S.nsms;                              // l.939
  c.sh_mem_per_tb = shmem_floats * 4.0;                                   // l.940-942 (bytes, f32 scratchpads)
  c.sh_mem_per_tb *= (1.0 - f);                                           // l.943
  int split = T[0] > 1 ? 0 : (T[1] > 1 ? 1 : 2);
  c.reg_tile = std::round(T[split] * f) * std::max(1, buffers);           // l.944 (R13)
  c.reg_per_th = c.reg_tile + (double)regs_per_stage * order.size();      // l.960
  // global transactions: group-external loads, 32 lanes along x from the representative origin
  double txs = 0;
  for (int s : order)
    for (int ri : A.reads_of[s]) {
      const ReadSite& r = A.reads[ri];
      if (r.src_is_stage && in[r.src]) continue;
      int esz = dtype_size(r.src_is_stage ? p.stages[r.src].dtype : p.images[r.src].dtype);
      int64_t off = r.form[2] == Form::UNIT ? r.off[2] : 0;
      // iterations of the consumer's loop per warp tile (R14): its computed region / W
      double iters = 1;
      for (int d = 0; d < 3; ++d) iters *= std::ceil((double)(wt[d] + L[s][d] + Rr[s][d]) / W[d]);
      txs += iters * min_txs((off - L[s][0]) * esz, (int64_t)W[0] * esz, tx);
    }
  c.total_gl_txs = txs;
  double tile_vol = (double)wt[0] * wt[1] * wt[2];
  c.txs_per_point = txs / tile_vol;
  if (!constant) { c.infinite = true; c.why = "non-constant dependence vectors"; }
  double tpi = 0;
  for (int s : order) tpi += stage_ops(p, s) / S.sm_clock_hz;
  alg2_tail(c, S, w, tile_vol, tpi, redundant, computed, tx);
  o << "\"cost\":" << cost_json(c) << "}";
  return o.str();
}

std::vector<std::vector<int>> merge_candidates(const Analysis& A, const Schedule& sch) {
  // group ids by position in sch.groups (a manual schedule's ids may be any labels)
  std::vector<int> pos(A.p->stages.size(), 0);
  for (size_t gi = 0; gi < sch.groups.size(); ++gi)
    for (int st : sch.groups[gi].stages) pos[st] = (int)gi;
  std::vector<std::vector<int>> out{pos};
  const int ng = (int)sch.groups.size();
  for (int gi = 0; gi + 1 < ng; ++gi) {
    std::vector<int> merged = sch.groups[gi].stages;
    merged.insert(merged.end(), sch.groups[gi + 1].stages.begin(), sch.groups[gi + 1].stages.end());
    if (!feasible_stage_set(A, merged)) continue;
    std::vector<int> gos = pos;
    for (int& v : gos)
      if (v == gi + 1) v = gi;
      else if (v > gi + 1) --v;
    out.push_back(gos);
  }
  return out;
}

}  // namespace pmg
