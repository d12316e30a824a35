// runtime.hpp — JIT compilation (NVRTC, sm_100a), plans, workspace and stream-ordered launches.
#pragma once
#include <mutex>
#include <cuda.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "select.hpp"

namespace pmg {

struct FnStats { int regs = -1, spill_stores = -1, spill_loads = -1; };

struct Compiled {
  std::string name, source, log;
  std::vector<char> cubin;
  int regs = -1, spill_stores = -1, spill_loads = -1, smem_static = -1;   // the interior entry point
  std::map<std::string, FnStats> fns;                                     // every entry point
  bool from_cache = false;
  double compile_s = 0;
};

// compile one group kernel for sm_100a (disk cache keyed by source + options); throws Error(PMG_ERR_NVRTC)
// compile with NVRTC for sm_100a, through the on-disk cubin cache (dir_override: cache directory for this call)
Compiled jit_compile(const std::string& name, const std::string& source, const std::string& dir_override = "");

struct WsTensor {          // workspace placement of an intermediate (materialised, non-liveout) stage
  int stage = -1;
  size_t offset = 0;
  int64_t row_pitch = 0, plane_pitch = 0, rows = 0, planes = 0;
};

struct Kernel {
  Compiled bin;
  CUmodule mod = nullptr;
  CUfunction fn = nullptr, fn_b = nullptr, fn_e = nullptr;   // interior tiles / border tiles / x-edge tiles
  int blocks_per_sm = 0, blocks_per_sm_b = 0, blocks_per_sm_e = 0;
};

struct Plan {
  std::shared_ptr<Pipeline> pipe;
  Analysis A;
  Schedule sch;
  pmg_gpu_spec spec;
  pmg_weights weights;
  int device = -1;
  CUcontext ctx = nullptr;
  std::vector<Kernel> kernels;
  std::vector<WsTensor> ws;
  // interleave fusion: a liveout that only interleaves quad-resolution phases of one group,
  // L(c, y, x) = S_{c, y%2, x%2}(y/2, x/2), is not launched; the phases store every other element straight into it
  struct Ilv { int out = -1, c = 0, py = 0, px = 0; };
  std::map<int, Ilv> ilv;                  // phase stage id -> its place in the liveout
  std::vector<char> ilv_skip;              // per group: fused away (the interleave's own group)
  size_t ws_bytes = 0;
  int nimages = 0, ntables = 0, nout = 0;
  CUstream side = nullptr;                 // border-tile kernels run here, forked/joined with events
  CUevent ev_fork = nullptr, ev_join = nullptr;
  std::string json;
  std::vector<std::string> inlined;        // stages substituted into their readers (inline.cpp)
  std::vector<std::string> factored;       // stages evaluated separably (factor.cpp, sched_opts.reassoc)
  std::vector<std::string> split;          // stages replaced by their two phases (phase.cpp), "name/y|x"
  // independent groups run concurrently: each group is assigned a lane (lane 0 = the caller's stream,
  // lanes 1.. plan-owned streams); cross-lane dependences are events (DESIGN.md §6 "group DAG")
  int nlanes = 1;
  std::vector<int> lane_of;                // per group
  std::vector<std::vector<int>> deps;      // per group: the groups producing what it reads
  std::vector<CUstream> lane_stream, lane_side, lane_side2;   // side2: x-edge kernels, concurrent with the border kernel
  std::vector<CUevent> lane_fork, lane_join, lane_join2, ev_group;
  CUevent ev_run = nullptr;
  std::string tune_json;                   // measured selection report (pmg_sched_opts.tune), empty otherwise
  int last_launches = 0;                   // kernels launched by the most recent plan_run (bench evidence)
  int only_group = -1;                     // >= 0: plan_run launches that group alone (profile_groups_us)
  // host-buffer runs (pmg_run_host): copy streams and per-chunk events, created on first use
  CUstream h2d = nullptr, d2h = nullptr;
  std::vector<CUevent> ev_in, ev_done;
  CUevent ev_start = nullptr, ev_end = nullptr;
  bool released = false;
  std::recursive_mutex run_mu;        // serialises the host-side enqueue of runs (shared fork/join events and side streams)
  Plan() = default;
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;
  ~Plan();   // releases every CUDA resource (modules, streams, events, the primary-context retain)
};

std::unique_ptr<Plan> plan_create(std::shared_ptr<Pipeline> p, const std::vector<int64_t>& params, int device,
                                  const pmg_gpu_spec* spec, const pmg_weights* w, const pmg_sched_opts* opts);
void plan_destroy(Plan* plan);

struct BandRows { int64_t out_r0, out_r1, in_r0, in_r1; };
BandRows band_rows(const Plan& P, int band, int nbands);

// halo-exchange band geometry: band b computes only its OWN rows of every group,
// own_g(b) = [b*Hg/n, (b+1)*Hg/n) at the group's row extent Hg, and receives the rows of earlier groups'
// stages its group needs beyond them from the bands that own them, instead of recomputing the cumulative halo.
struct BandXchg {
  std::vector<RowIv> own;    // per group
  std::vector<RowIv> buf;    // per stage: rows the band's workspace slot holds (own rows + received halo rows)
  std::vector<RowIv> need;   // per stage: rows the band's later groups read (hull over its reader groups)
  RowIv in, out;             // image rows of the band's input buffers; liveout rows
};
BandXchg band_xchg(const Plan& P, int band, int nbands);

// workspace placement of every materialised non-liveout stage (P.ws, P.ws_bytes)
void layout_workspace(Plan& P);

// launch every group kernel; band < 0: full image; nframes >= 1 (batch).  groups != nullptr: halo-exchange band
// mode (band >= 0), launch only groups [groups[0], groups[1]) with the BandXchg geometry.
void plan_run(Plan& P, const pmg_buf* in, int nin, const pmg_buf* out, int nout, void* workspace, CUstream s,
              int band, int nbands, int nframes, const int64_t* in_fs, const int64_t* out_fs,
              const int* groups = nullptr);

// per-group kernel time of one run (each group launched alone on synthetic inputs; CUDA events, best of 3 samples
// of 10 runs): the TimePerIter microbenchmark of pmg_profile_stages when groups are single stages
std::vector<double> profile_groups_us(Plan& P);

// host buffers in and out, pipelined in `chunks` row bands over copy-in / compute / copy-out streams
void plan_run_host(Plan& P, const pmg_buf* hin, int nin, const pmg_buf* hout, int nout, const pmg_buf* din,
                   const pmg_buf* dout, void* workspace, int chunks, CUstream s);

std::string kernel_dir();   // directory of libpmg.so (for the cubin cache)

// compile probe for the selector (ptxas register / spill counts of a candidate)
RegProbe make_probe(const Analysis& A);

}  // namespace pmg
