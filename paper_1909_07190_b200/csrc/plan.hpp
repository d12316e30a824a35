// plan.hpp — fusion groups, per-group B200 kernel configuration and geometry, schedules and plans.
//
// Mapping of the paper's notions onto the B200 kernel (DESIGN.md §"Kernel"):
//   warp overlapped tile (§4)   = CW x TH points (CW = 32*V*TX columns, TH rows) per warp
//   tile size T                 = (V*TX, TH): points per lane along x and y
//   thread block B                          = (32*NW, 1, 1)  =>  warp sizes W = (32, 1, 1)
//   parallelogram tiles (§5)     = the TX chunks of 32*V columns along the split dim x
//   fracReg (Alg. 1 l.867)                  = (TX - S) / TX: the first S chunks in shared memory,
//                                             the remaining chunks in registers
//   overlap O_i^n               = per-stage halo rows (y) and invalid chunk columns (x)
//   right hyperplane phi_r      = per-stage row lead `hi` (stage n computes row y+hi_n
//                                             while the liveout computes row y: wavefront order)
#pragma once
#include <string>
#include <vector>

#include "analysis.hpp"

namespace pmg {

struct KConfig {
  int V = 4;        // x points per lane per chunk
  int TX = 1;       // chunks (parallelogram tiles) per warp tile
  int S = 0;        // chunks in shared memory (hybrid split)
  int TH = 32;      // rows per warp tile
  int NW = 4;       // warps per block
  int PREF = 4;     // TMA ring depth (input rows in flight per warp)
  int tx_size = 32; // GlMemTxSz choice (32: L2 sector / TMA path; 128: L1 line)
  int regcap = 0;   // registers-per-thread cap via __launch_bounds__ min-blocks (0 = none)
  bool contract = false;   // reassociation mode: f32 a*b+c emitted as one fma (sched_opts.reassoc)
  int THb_want = 8;        // border-tile rows requested (sched_opts.border_rows); TH_b = the largest divisor of TH <= it
};

// a read of a group input staged through the TMA ring (unit-stride rows)
struct GStream {
  bool src_is_stage = false;
  int src = -1;
  int plane_mode = 0;     // 0: source has no plane dim; 1: aligned with the tile plane; 2: constant
  int64_t plane_const = 0;
  // alignment & scaling: index forms per dim.  y: 0 unit (row v+b), 1 down2 (row 2v+b: the
  // phase-py rows 2r+py as a virtual image, read at r = v + floor(b/2)), 2 up2 (row floor((v+b)/2): the
  // virtual image U(r) = P(floor(r/2)) read at r = v+b).  x: 0 unit, 1 down2 (register index q = 2e+b over
  // the producer columns from 2*xL), 2 up2 (register index e+b, producer column floor((xL+e+b)/2)).
  int sy = 0, py = 0, sx = 0;
  int dy_min = 0, dy_max = 0, dx_min = 0, dx_max = 0;
  int hi = 0, lo = 0, depth = 1;
  int el = 0, er = 0;     // register extension (elements) each side
  int xl = 0, xr = 0;     // smem row extension (elements, multiples of 16B)
  DType dtype = DType::F32;
  int esz = 4;
  int row_elems = 0;      // CW + xl + xr
  int smem_off = 0;       // byte offset inside a ring slot
  int tensor_slot = -1;
};

struct GStage {
  int id = -1;
  int hi = 0, lo = 0, depth = 1;
  int el = 0, er = 0;     // extension elements via shuffles
  int vl = 0, vr = 0;     // invalid columns at the chunk-row edges
  bool materialize = false;   // written to global (pipeline liveout or read by a later group)
  bool xfix = false;          // read with dx != 0: replicate out-of-domain columns in border tiles
  bool smem = false;          // hybrid: window kept in shared memory for the S smem chunks
  bool ilv = false;           // stored at every other column of an interleaved liveout (runtime.cpp interleave fusion)
  int tensor_slot = -1;
  int smem_off = 0;           // per-warp byte offset of its smem window (S > 0)
  int smem_padl = 0;          // elements before column 0 of the smem row (left halo, 16-byte aligned)
  int smem_rowb = 0;          // bytes per smem row (one window slot)
};

enum class RKind { STAGE, STREAM, GATHER };
struct GRead {           // resolution of one ReadSite inside a group
  RKind kind = RKind::GATHER;
  int idx = -1;          // GStage index (STAGE) / GStream index (STREAM) / tensor slot (GATHER)
  int dy = 0, dx = 0;
};

struct Group {
  std::vector<int> stages;   // stage ids, topo order
  Ext3 ext;
  KConfig cfg;
  // geometry
  std::vector<GStage> gs;
  std::vector<GStream> streams;
  std::vector<int> read_map;          // ReadSite index -> GRead index (or -1 if not in group)
  std::vector<GRead> greads;
  std::vector<std::pair<bool, int>> tensors;  // slot -> (is_stage, id)
  int CW = 0, PL = 0, PR = 0, OW = 0;
  int t_first = 0, nsteps = 0, U = 1;
  bool no_scaled = false;   // read scaled inputs by gather (set by build_group when there would be too many streams)
  bool xedge = false;       // x-edge kernel: the first / last tile columns run the interior body with halo selects
                            // at the image's left / right edge; the border kernel keeps only the top / bottom rows
  int TH_b = 0;             // tile rows of the border-tile kernel (divides TH; small: border tiles are latency-bound)
  int ring_bytes = 0;       // one ring slot
  int warp_smem = 0;        // bytes of shared memory per warp
  int block_smem = 0;
  int64_t nty = 0, ntx = 0, npl = 1;
  std::string name, source;
  std::string why_infeasible;
  int regs_est = 0;
};

// build geometry; returns false (with g.why_infeasible) when the group cannot run as one kernel
bool build_group(const Analysis& A, Group& g, const std::vector<int>& group_of_stage);

// registers the interior kernel keeps live from one row step to the next (register-estimate input)
int interior_state_regs(const Analysis& A, const Group& g);

// CUDA C++ source of one group kernel (NVRTC input)
std::string emit_group(const Analysis& A, const Group& g, bool interior_only = false);

struct Schedule {
  std::vector<Group> groups;          // topo order of groups
  std::vector<int> group_of_stage;
  std::string json;                   // selector report
};

}  // namespace pmg
