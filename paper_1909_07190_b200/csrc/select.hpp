// select.hpp — model-based fusion grouping and tile-size selection (§6).
#pragma once
#include <functional>
#include <string>
#include <vector>

#include "../../include/pmg.h"
#include "plan.hpp"

namespace pmg {

struct CostBreakdown {          // every term of Alg. 2
  double total_threads = 0, warps_per_tb = 0, tb_per_sm = 0;
  double sh_mem_per_tb = 0;     // bytes (after the fracReg split, l.943)
  double reg_tile = 0, reg_per_th = 0;
  double total_gl_txs = 0;      // per warp tile (l.949-954)
  double txs_per_point = 0;     // normalised per output point (reading R14)
  double max_tb_per_sm = 0, sh_mem_occ = 0, reg_occ = 0, occupancy = 0;
  double warp_bw = 0, mem_time = 0, compute_time = 0;
  double unallocated_sh_mem = 0, unused_reg = 0, frac_overlap = 0, extra_tbs = 0;
  double est_us = 0;            // B200 time estimate of the group kernel
  double tm_ops = 0, tm_stages = 0, tm_streams = 0, tm_nsteps = 0, tm_tiles = 0, tm_bytes = 0, tm_resident = 0, tm_border_tiles = 0,
         tm_border_steps = 0;
  double alg2_cost = 0;         // the weighted seven-term sum (l.981)
  double cost = 0;              // the ranking value: est_us (cost_model 0) or alg2_cost (cost_model 1)
  bool infinite = false;
  std::string why;
};

bool gpu_preset(const std::string& name, pmg_gpu_spec* out);
bool weights_preset(const std::string& name, pmg_weights* out);

// static per-stage profile (Alg. 2 inputs RegUsage(H), TimePerIter(H))
double stage_ops(const Pipeline& p, int stage);

// B200-mode Alg. 2 for a built group (KConfig -> paper symbols, DESIGN.md §"Selector")
CostBreakdown b200_cost(const Analysis& A, const Group& g, const pmg_gpu_spec& spec, const pmg_weights& w,
                        int cost_model = 0, int bands = 1, const double* time_per_iter = nullptr);

// measured TimePerIter of the pipeline as written (per stage, declaration order) -> per stage of the rewritten
// pipeline the schedule works on (matched by name; rewritten stages get 0 = the static count)
std::vector<double> map_time_per_iter(const Pipeline& written, const Pipeline& eff, const double* tpi);

// RegUsage(H) "measured with nvcc": compile a candidate and return ptxas' registers / spill bytes
using RegProbe = std::function<bool(const Group& g, int* regs, int* spill_bytes)>;

// argmin over the configuration space for one group; returns false if every point is infinite
bool best_config(const Analysis& A, Group& g, const std::vector<int>& gos, const pmg_gpu_spec& spec,
                 const pmg_weights& w, const pmg_sched_opts& opts, CostBreakdown* cb, const RegProbe* probe = nullptr);

// DP fusion over convex groups (contiguous runs of the topological order), total = sum of group costs
Schedule schedule(const Analysis& A, const pmg_gpu_spec& spec, const pmg_weights& w, const pmg_sched_opts& opts,
                  const RegProbe* probe = nullptr);

// group_of_stage vectors for measured selection (pmg_sched_opts.tune): the schedule's own grouping, then every
// grouping that merges two neighbouring groups of it into one feasible stage set
std::vector<std::vector<int>> merge_candidates(const Analysis& A, const Schedule& sch);

// the paper's §4 geometry + Alg. 2 for an explicit group and (T, B, fracReg, txSz) — analysis pins
std::string paper_analyze_group(const Analysis& A, const std::vector<int>& stages, const int T[3], const int B[3],
                                double frac_reg, int tx_size, int regs_per_stage, const pmg_gpu_spec& spec,
                                const pmg_weights& w);

std::string cost_json(const CostBreakdown& c);
std::string config_json(const Analysis& A, const Group& g);

}  // namespace pmg
