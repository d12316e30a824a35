// group.cpp — geometry of one fused group for the B200 OTPW + hybrid-tiling kernel.
//
// Paper anchors:
//   * fusion legality: Alg. 2 line 930 — a group is infeasible unless every producer->consumer
//     dependence inside it is constant after alignment & scaling;
//   * overlaps O_i^n: backward accumulation from the group's liveouts;
//   * right hyperplanes phi_r: `hi` below is the accumulated forward reach in y —
//     stage n produces row y+hi_n when the liveouts produce row y, so every dependence points to an
//     already-computed row ("no cyclic dependence between two adjacent tiles");
//   * warp sizes W = (32,1,1) from B = (32*NW,1,1); one overlapped tile per warp.
#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <set>

#include "plan.hpp"

namespace pmg {

static int round_up(int a, int m) { return (a + m - 1) / m * m; }

bool build_group(const Analysis& A, Group& g, const std::vector<int>& gos) {
  const Pipeline& p = *A.p;
  const KConfig& k = g.cfg;
  auto bad = [&](const std::string& m) { g.why_infeasible = m; return false; };
  if (g.stages.empty()) return bad("empty group");
  if (k.V != 1 && k.V != 2 && k.V != 4 && k.V != 8) return bad("V must be 1, 2, 4 or 8");
  if (k.TX < 1 || k.TX > 8 || k.S < 0 || k.S > k.TX || k.TH < 1 || k.NW < 1 || k.NW > 32 || k.PREF < 1 || k.PREF > 16)
    return bad("configuration out of range");
  const int gid = gos[g.stages[0]];
  // stage order: pipeline topological order
  std::vector<int> order;
  for (int s : p.topo)
    if (gos[s] == gid) order.push_back(s);
  g.stages = order;
  // a group iterates one (plane, y, x) domain; stages without a plane dim may join a plane group when their
  // (y, x) extents match ("broadcast" stages: recomputed for every plane, never materialised -- checked below)
  g.ext = A.stage_ext[order[0]];
  for (int s : order)
    if (A.stage_ext[s].has[0]) g.ext = A.stage_ext[s];
  for (int s : order) {
    const Ext3& e = A.stage_ext[s];
    if (e == g.ext) continue;
    if (e.has[0] || !g.ext.has[0] || e.e[1] != g.ext.e[1] || e.e[2] != g.ext.e[2] || e.has[1] != g.ext.has[1])
      return bad("stages of different extents (" + p.stages[s].name + ")");
  }
  const int n = (int)order.size();
  std::vector<int> pos(p.stages.size(), -1);
  for (int i = 0; i < n; ++i) pos[order[i]] = i;
  g.gs.assign(n, GStage{});
  for (int i = 0; i < n; ++i) {
    int s = order[i];
    g.gs[i].id = s;
    bool lo = std::find(p.liveouts.begin(), p.liveouts.end(), s) != p.liveouts.end();
    for (int c : p.consumers[s])
      if (gos[c] != gid) lo = true;
    g.gs[i].materialize = lo;
    if (lo && !(A.stage_ext[s] == g.ext)) return bad("broadcast stage " + p.stages[s].name + " must be materialised");
  }
  // resolve reads
  g.read_map.assign(A.reads.size(), -1);
  g.greads.clear();
  g.streams.clear();
  g.tensors.clear();
  auto slot_of = [&](bool is_stage, int id) {
    for (size_t i = 0; i < g.tensors.size(); ++i)
      if (g.tensors[i].first == is_stage && g.tensors[i].second == id) return (int)i;
    g.tensors.push_back({is_stage, id});
    return (int)g.tensors.size() - 1;
  };
  struct PendingStream { int stream; int stage_pos; int dy, dx; };
  std::vector<PendingStream> sreads;
  std::vector<std::tuple<int, int, int, int>> ereads;   // (producer pos, consumer pos, dy, dx)
  for (int i = 0; i < n; ++i) {
    int s = order[i];
    for (int ri : A.reads_of[s]) {
      const ReadSite& r = A.reads[ri];
      GRead gr;
      auto yoff = [&](void) -> int64_t { return r.form[1] == Form::ABSENT ? 0 : r.off[1]; };
      if (r.src_is_stage && gos[r.src] == gid) {
        // in-group edge: dependences must be constant (Alg. 2 l.930)
        bool ok = (r.form[1] == Form::UNIT || r.form[1] == Form::ABSENT) && r.form[2] == Form::UNIT &&
                  (r.form[0] == Form::ABSENT || (r.form[0] == Form::UNIT && r.off[0] == 0));
        if (!ok)
          return bad("non-constant dependence " + p.stages[s].name + " <- " + p.stages[r.src].name);
        if (std::abs(r.off[2]) > 64 || std::abs(yoff()) > 64) return bad("stencil reach too large");
        gr.kind = RKind::STAGE;
        gr.idx = pos[r.src];
        gr.dy = (int)yoff();
        gr.dx = (int)r.off[2];
        ereads.push_back({gr.idx, i, gr.dy, gr.dx});
      } else {
        const Ext3& se = r.src_is_stage ? A.stage_ext[r.src] : A.image_ext[r.src];
        bool plane_ok = r.form[0] == Form::ABSENT || r.form[0] == Form::CONST ||
                        (r.form[0] == Form::UNIT && r.off[0] == 0 && g.ext.has[0] && se.e[0] == g.ext.e[0]);
        // index forms of y and x: unit (same extent), or the scaled forms 2v+b / (v+b)/2 staged through the
        // TMA ring like unit reads (alignment & scaling; DESIGN.md §6 "Scaled streams")
        // opt-in (PMG_SCALED=1): measured 3 % slower than L1/L2-served gathers on every pyramid workload
        // (camera 0.151 vs 0.147, local Laplacian 0.396 vs 0.381, pyramid blend 0.479 vs 0.465 ms)
        const bool scale_on = !g.no_scaled && getenv("PMG_SCALED") && getenv("PMG_SCALED")[0] == '1';
        int sy = -1, sx = -1;
        if (r.form[1] == Form::ABSENT || (r.form[1] == Form::UNIT && se.e[1] == g.ext.e[1])) sy = 0;
        else if (scale_on && r.form[1] == Form::DOWN2) sy = 1;
        else if (scale_on && r.form[1] == Form::UP2) sy = 2;
        if (r.form[2] == Form::UNIT && se.e[2] == g.ext.e[2]) sx = 0;
        else if (scale_on && r.form[2] == Form::DOWN2) sx = 1;
        else if (scale_on && r.form[2] == Form::UP2 && k.V % 2 == 0) sx = 2;
        if (sy != 0 && !se.has[1]) sy = -1;
        bool stream = plane_ok && sy >= 0 && sx >= 0 && se.has[1] == g.ext.has[1] && std::abs(r.off[2]) <= 64 &&
                      std::abs(yoff()) <= 64;
        if (stream) {
          int mode = r.form[0] == Form::ABSENT ? 0 : (r.form[0] == Form::UNIT ? 1 : 2);
          int64_t pc = mode == 2 ? std::max<int64_t>(0, std::min<int64_t>(r.off[0], se.e[0] - 1)) : 0;
          const int by = (int)yoff();
          const int py = sy == 1 ? (by & 1) : 0;
          const int vdy = sy == 1 ? (by >> 1) : by;   // offset in the stream's virtual rows
          int si = -1;
          for (size_t q = 0; q < g.streams.size(); ++q) {
            auto& st = g.streams[q];
            if (st.src_is_stage == r.src_is_stage && st.src == r.src && st.plane_mode == mode && st.plane_const == pc &&
                st.sy == sy && st.py == py && st.sx == sx)
              si = (int)q;
          }
          if (si < 0) {
            GStream st;
            st.src_is_stage = r.src_is_stage;
            st.src = r.src;
            st.plane_mode = mode;
            st.plane_const = pc;
            st.dtype = r.src_is_stage ? p.stages[r.src].dtype : p.images[r.src].dtype;
            st.esz = dtype_size(st.dtype);
            st.tensor_slot = slot_of(r.src_is_stage, r.src);
            st.sy = sy;
            st.py = py;
            st.sx = sx;
            st.dy_min = st.dy_max = vdy;
            st.dx_min = st.dx_max = (int)r.off[2];
            g.streams.push_back(st);
            si = (int)g.streams.size() - 1;
          }
          auto& st = g.streams[si];
          st.dy_min = std::min(st.dy_min, vdy);
          st.dy_max = std::max(st.dy_max, vdy);
          st.dx_min = std::min(st.dx_min, (int)r.off[2]);
          st.dx_max = std::max(st.dx_max, (int)r.off[2]);
          gr.kind = RKind::STREAM;
          gr.idx = si;
          gr.dy = vdy;
          gr.dx = (int)r.off[2];   // raw b of the x index form
          sreads.push_back({si, i, gr.dy, gr.dx});
        } else {
          gr.kind = RKind::GATHER;
          gr.idx = slot_of(r.src_is_stage, r.src);
        }
      }
      g.read_map[ri] = (int)g.greads.size();
      g.greads.push_back(gr);
    }
  }
  // every stream keeps ~6 registers of per-tile refill state; a group that would read many scaled inputs
  // (the camera interleave: 12 quad planes) reads them by gather instead (measured: 232-247 registers with
  // 12 scaled streams, profiles/scaled_streams_r01e.txt)
  {
    int nscaled = 0;
    for (auto& st : g.streams) nscaled += (st.sy != 0 || st.sx != 0);
    if (nscaled > 4 && !g.no_scaled) {
      g.no_scaled = true;
      return build_group(A, g, gos);
    }
  }
  // row reach (right hyperplane in y) and overlaps, backward over topo order
  const int NEG = -1000000, POS = 1000000;
  for (int i = 0; i < n; ++i) { g.gs[i].hi = NEG; g.gs[i].lo = POS; }
  for (int i = n - 1; i >= 0; --i) {
    GStage& P = g.gs[i];
    if (P.materialize) { P.hi = std::max(P.hi, 0); P.lo = std::min(P.lo, 0); }
    for (auto& [pp, cp, dy, dx] : ereads) {
      if (pp != i) continue;
      const GStage& C = g.gs[cp];
      P.hi = std::max(P.hi, C.hi + std::max(dy, 0));
      P.lo = std::min(P.lo, C.lo + std::min(dy, 0));
      P.el = std::max(P.el, -dx);
      P.er = std::max(P.er, dx);
      if (P.el > 31 * k.V || P.er > 31 * k.V) return bad("x reach exceeds one chunk");
      if (dx != 0) P.xfix = true;
    }
    if (P.hi == NEG) return bad("stage " + p.stages[P.id].name + " has no consumer in its group and is not materialised");
  }
  for (int i = 0; i < n; ++i) {
    GStage& P = g.gs[i];
    P.depth = 1;
    for (auto& [pp, cp, dy, dx] : ereads)
      if (pp == i) P.depth = std::max(P.depth, P.hi - g.gs[cp].hi - dy + 1);
  }
  for (auto& st : g.streams) { st.hi = NEG; st.lo = POS; }
  for (auto& r : sreads) {
    auto& st = g.streams[r.stream];
    const GStage& C = g.gs[r.stage_pos];
    st.hi = std::max(st.hi, C.hi + std::max(r.dy, 0));
    st.lo = std::min(st.lo, C.lo + std::min(r.dy, 0));
  }
  for (auto& r : sreads) {
    auto& st = g.streams[r.stream];
    st.depth = std::max(st.depth, st.hi - g.gs[r.stage_pos].hi - r.dy + 1);
  }
  // x geometry
  g.CW = 32 * k.V * k.TX;
  int align = k.V;
  for (auto& st : g.streams) {
    int a = 16 / st.esz;
    align = std::max(align, st.sx == 2 ? 2 * a : a);   // up2: the smem origin cx/2 must stay 16-byte aligned
    if (st.sx == 1) {
      // register index q = 2e + b in [dx_min, 2V-2+dx_max], lane base 2V*lane; vector reads of V elements
      st.el = std::max(0, -st.dx_min);
      st.er = std::max(0, k.V - 1 + st.dx_max);
      const int m = std::max(a, k.V);
      st.xl = round_up(st.el, m);
      st.xr = round_up(std::max(0, round_up(k.V + st.er, k.V) - 2 * k.V), m);
      st.row_elems = 2 * g.CW + st.xl + st.xr;
    } else if (st.sx == 2) {
      // register index e' = e + b in [-el, V+er), producer column xL/2 + floor(e'/2); lane base (V/2)*lane
      st.el = std::max(0, -st.dx_min);
      st.er = std::max(0, st.dx_max);
      const int h = k.V / 2;
      st.xl = round_up((st.el + 1) / 2, std::max(a, h));
      int qend = (k.V + st.er - 1) / 2 + 1;                 // one past the last producer element of lane 0
      st.xr = round_up(std::max(0, round_up(qend, h) - h), std::max(a, h));
      st.row_elems = g.CW / 2 + st.xl + st.xr;
    } else {
      st.el = std::max(0, -st.dx_min);
      st.er = std::max(0, st.dx_max);
      st.xl = round_up(st.el, std::max(a, k.V));   // vector smem reads of [-el, V+er) stay inside the row
      st.xr = round_up(st.er, std::max(a, k.V));
      st.row_elems = g.CW + st.xl + st.xr;
    }
  }
  for (int i = 0; i < n; ++i) {
    GStage& C = g.gs[i];
    for (int ri : A.reads_of[C.id]) {
      const GRead& gr = g.greads[g.read_map[ri]];
      if (gr.kind == RKind::STAGE) {
        C.vl = std::max(C.vl, g.gs[gr.idx].vl + std::max(0, -gr.dx));
        C.vr = std::max(C.vr, g.gs[gr.idx].vr + std::max(0, gr.dx));
      } else if (gr.kind == RKind::STREAM) {
        const GStream& st = g.streams[gr.idx];
        if (st.sx != 0) continue;   // scaled rows are read from smem only (every register index inside the row)
        C.vl = std::max(C.vl, std::max(0, -gr.dx - st.xl));
        C.vr = std::max(C.vr, std::max(0, gr.dx - st.xr));
      }
    }
  }
  int vl = 0, vr = 0;
  for (auto& P : g.gs)
    if (P.materialize) { vl = std::max(vl, P.vl); vr = std::max(vr, P.vr); }
  g.PL = round_up(vl, align);
  g.PR = round_up(vr, align);
  g.OW = g.CW - g.PL - g.PR;
  if (g.OW <= 0) return bad("chunk row too narrow for the group's x halo (CW=" + std::to_string(g.CW) + ")");
  if (g.OW % align) return bad("output tile width not aligned");
  // y steps
  g.t_first = 0;
  for (auto& P : g.gs) g.t_first = std::min(g.t_first, P.lo - P.hi);
  for (auto& st : g.streams) g.t_first = std::min(g.t_first, st.lo - st.hi);
  g.nsteps = k.TH - g.t_first;
  if (!g.streams.empty() && k.PREF > g.nsteps) return bad("prefetch depth exceeds the steps of one tile");
  // border tiles: one warp walks a whole tile through the general (clamping) body at low occupancy, so the
  // border kernel's time is one tile's latency; it runs with shorter tiles (measured)
  {
    const char* e = getenv("PMG_BORDER_TH");
    int want = e ? atoi(e) : k.THb_want;
    g.TH_b = k.TH;
    for (int d = std::min(want, k.TH); d >= 1; --d)
      if (k.TH % d == 0 && (g.streams.empty() || k.PREF <= d - g.t_first)) { g.TH_b = d; break; }
  }
  // x-edge kernel: the first / last tile columns run the interior (branch-free in y) body with
  // the halo elements beyond the image edge replaced by the edge column (a select in the lane that holds
  // column 0 / W-1), the first tile column starting at x = 0.  Needs: no shared-memory chunks, unscaled x reads,
  // every x halo within one lane (el, er <= V), W a multiple of V (column W-1 ends a lane), and only the first
  // tile column reaching left of x = 0 (OW >= PL + the streams' left smem halo).
  {
    const char* e = getenv("PMG_XEDGE");
    bool ok = !(e && e[0] == '0') && k.S == 0 && g.ext.e[2] % k.V == 0;
    int xl_max = 0;
    for (auto& P : g.gs) ok = ok && P.el <= k.V && P.er <= k.V;
    for (auto& st : g.streams) {
      ok = ok && st.sx == 0 && st.el <= k.V && st.er <= k.V;
      xl_max = std::max(xl_max, st.xl);
    }
    g.xedge = ok && g.OW >= g.PL + xl_max;
  }
  // unroll factor for register-window rotation
  int U = 1;
  auto lcm = [](int a, int b) { return a / std::gcd(a, b) * b; };
  for (auto& P : g.gs) U = lcm(U, P.depth);
  for (auto& st : g.streams) U = lcm(U, st.depth);
  if (U > 16) {
    U = 1;
    for (auto& P : g.gs) U = std::max(U, P.depth);
  }
  g.U = U;
  // shared memory per warp: mbarriers + ring
  int off = 0;
  for (auto& st : g.streams) {
    st.smem_off = off;
    off += round_up(st.row_elems * st.esz, 16);
  }
  g.ring_bytes = off;
  int bar_bytes = round_up(8 * k.PREF, 16);
  g.warp_smem = g.streams.empty() ? 16 : bar_bytes + k.PREF * g.ring_bytes;
  // hybrid tiling: the S leftmost chunks keep the windows of stages that are read with
  // a row window or an x halo in warp-private shared memory; the other TX-S chunks keep them in registers
  if (k.S > 0) {
    for (auto& P : g.gs) {
      if (P.depth <= 1 && P.el + P.er == 0) continue;
      const int esz = dtype_size(p.stages[P.id].dtype), al = 16 / esz;
      P.smem = true;
      P.smem_padl = round_up(P.el, al);
      P.smem_rowb = round_up((P.smem_padl + k.S * 32 * k.V + round_up(P.er, al)) * esz, 16);
      P.smem_off = g.warp_smem;
      g.warp_smem += P.depth * P.smem_rowb;
    }
  }
  g.block_smem = g.warp_smem * k.NW;
  if (g.block_smem > 227 * 1024) return bad("shared memory per block exceeds 227 KB");
  for (auto& P : g.gs)
    if (P.materialize) P.tensor_slot = slot_of(true, P.id);
  g.npl = g.ext.has[0] ? g.ext.e[0] : 1;
  g.ntx = (g.ext.e[2] + g.OW - 1) / g.OW;
  // register estimate (selector input; refined by ptxas when compiled)
  // register estimate: windows (+60% for temporaries / scheduling), fitted to ptxas counts on B200;
  // the selector replaces it with the real count for its finalists (compile probe)
  int win = 0;
  for (auto& P : g.gs)
    win += P.smem ? P.depth * (k.TX - k.S) * (k.V + P.el + P.er) + k.S * k.V : P.depth * k.TX * (k.V + P.el + P.er);
  for (auto& st : g.streams) win += st.depth * k.TX * (k.V + st.el + st.er);
  g.regs_est = 40 + (win * 8 + 4) / 5;
  g.why_infeasible.clear();
  return true;
}

}  // namespace pmg
