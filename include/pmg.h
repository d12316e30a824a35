/*
 * pmg.h — C ABI of the B200-native PolyMage-GPU hot path (warp-overlapped + hybrid tiling).
 *
 * The calls follow the paper's statement of the problem (§2.2): a pipeline is a
 * DAG of stages over integer domains parameterised by the image extents ("the number of rows and
 * columns", lines 286-287); its liveouts are the outputs (line 302); kernels take image sizes as
 * runtime parameters (§5); all data resides on the GPU (§7).
 *
 *   pmg_pipeline_parse   text -> validated stage DAG                (§2.2; grammar extends SPEC.md l.81)
 *   pmg_schedule         host-only: fusion groups + tile/block/fracReg/txSz with the Alg. 2 cost
 *                        (§6), JSON report; no GPU needed
 *   pmg_plan_create      schedule + emit + compile (NVRTC, sm_100a) one OTPW/hybrid kernel per group
 *   pmg_run / pmg_run_band / pmg_run_batch   stream-ordered launches on caller-owned device buffers
 *
 * Layout: every image / stage buffer is planar [c][y][x], x fastest.  A buffer is described by
 * pmg_buf{ptr, row_pitch_bytes, plane_pitch_bytes}.  Device pointers and pitches passed to run calls
 * must be multiples of 16 bytes (TMA bulk-copy / 128-bit vector I/O); tables (LUTs) may have any
 * alignment.  Element types are the pipeline's declared dtypes.
 *
 * Ownership: the library owns pipeline / plan handles (create/destroy pairs; destroy is NULL-safe).
 * The caller owns every device buffer, the workspace and the stream.  Run calls are asynchronous and
 * stream-ordered: no allocation, no host synchronisation, no device switch (the plan's device must be
 * current — otherwise PMG_ERR_ARG).
 *
 * Errors: every call returns pmg_status; pmg_last_error() gives a thread-local message for the last
 * non-OK status on the calling thread (parse errors carry "line:col").  Launch-configuration errors
 * return PMG_ERR_CUDA immediately; asynchronous device faults surface at the caller's next sync.
 * PMG_ERR_INFEASIBLE: every candidate schedule has infinite cost (Alg. 2, 945, 961).
 *
 * Concurrency: a pipeline is immutable and shareable across threads.  Run calls on one plan from several
 * threads are safe (the plan serialises their enqueue with a mutex) but not concurrent on the device: every
 * run forks its border / x-edge kernels onto the plan's own side streams and joins back with the plan's
 * events, so two runs of one plan execute one after the other even on different caller streams; use one
 * plan per stream for concurrent runs, each with its own workspace.  A run's launches are ordered on the
 * caller's stream, so runs can be captured into CUDA graphs.  Outputs are bit-identical for any schedule, band
 * split or batch split (DESIGN.md §"Determinism").  No NCCL here: process groups and gathers belong to
 * the caller (PyTorch).
 */
#ifndef PMG_H
#define PMG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PMG_OK = 0,
  PMG_ERR_PARSE = -1,       /* syntax error, undeclared reference, cyclic reference, bad index form */
  PMG_ERR_INVALID = -2,     /* invalid handle / semantic error */
  PMG_ERR_UNSUPPORTED = -3, /* valid pipeline the kernel generator cannot run */
  PMG_ERR_INFEASIBLE = -4,  /* all schedules cost infinity */
  PMG_ERR_SHAPE = -5,       /* parameter values give an empty / inconsistent domain */
  PMG_ERR_CUDA = -6,        /* CUDA driver error (or no driver) */
  PMG_ERR_NVRTC = -7,       /* runtime compilation failed */
  PMG_ERR_OOM = -8,
  PMG_ERR_ARG = -9          /* bad argument: NULL, misaligned buffer, wrong device, buffer count */
} pmg_status;

typedef enum { PMG_U8 = 1, PMG_U16 = 2, PMG_I16 = 3, PMG_I32 = 4, PMG_F32 = 5 } pmg_dtype;

typedef struct pmg_pipeline_s* pmg_pipeline; /* immutable after parse */
typedef struct pmg_plan_s* pmg_plan;         /* bound to (pipeline, params, device, schedule) */

/* one input image / table / output liveout: extents outermost first ([c][y][x]); ndim 1..3 */
typedef struct {
  char name[64];
  int32_t dtype;       /* pmg_dtype */
  int32_t ndim;
  int32_t is_table;    /* inputs only: 1 for a 1-D lookup table */
  int32_t reserved;
  int64_t extent[3];
} pmg_io_desc;

/* device buffer: planar [c][y][x]; pitches in bytes (plane pitch ignored for <3-D tensors) */
typedef struct {
  void* ptr;
  int64_t row_pitch_bytes;
  int64_t plane_pitch_bytes;
} pmg_buf;

/* GPU description: Table 1 of the paper plus B200 additions */
typedef struct {
  char name[32];
  int32_t nsms;               /* NSMs */
  int32_t cores_per_sm;       /* CoresPerSM (FP32 lanes) */
  int32_t max_warps_per_sm;   /* MaxWarpPerSM */
  int32_t max_tb_per_sm;      /* MaxTbPerSM */
  int32_t regs_per_sm;        /* RegPerSM */
  int32_t max_regs_per_thread;/* MaxRegPerTh */
  int32_t max_threads_per_sm; /* MaxThPerSM (used by Alg. 2 l.963, absent from Table 1) */
  int32_t warp_size;          /* WarpSize */
  int64_t shmem_per_sm;       /* ShMemPerSM, bytes */
  int64_t max_shmem_per_tb;   /* MaxShMemPerTb, bytes */
  double gl_mem_bw;           /* GlMemBW, bytes/s */
  int32_t gl_tx_size[2];      /* GlMemTxSz choices: 32 (L2 sector) and 128 (L1 line) */
  int64_t l2_bytes;           /* B200 addition */
  double sm_clock_hz;         /* B200 addition (compute-time model) */
} pmg_gpu_spec;

/* cost weights w1..w7 (Table 3) */
typedef struct {
  double w[7];
} pmg_weights;

/* schedule overrides (SPEC.md l.631 flags); -1 / NULL = automatic */
typedef struct {
  const int32_t* group_of_stage; /* NULL = DP fusion; else group index per stage (declaration order) */
  int32_t vec;          /* V: consecutive x points per lane per chunk (1, 2, 4) */
  int32_t chunks;       /* TX: parallelogram (chunk) tiles per warp tile along x */
  int32_t smem_chunks;  /* S: chunks kept in shared memory; chunks-S in registers (fracReg = (TX-S)/TX) */
  int32_t rows;         /* TH: rows per warp tile (tile size in y) */
  int32_t warps;        /* warps per thread block (TB size / 32) */
  int32_t prefetch;     /* input rows in flight per warp (TMA ring depth) */
  int32_t tx_size;      /* 32 or 128 */
  int32_t budget;       /* max candidates per group (bounded search); <=0 = exhaustive */
  int32_t fuse;         /* 0 = one stage per group, 1 = DP fusion (default) */
  int32_t regcap;       /* registers per thread cap (__launch_bounds__ min-blocks); <=0 = automatic */
  int32_t probe;        /* 1 = compile the selector's finalists to read ptxas register counts (default) */
  int32_t cost_model;   /* 0 = B200 time estimate (default); 1 = Alg. 2 weighted sum */
  int32_t bands;        /* runs will be row bands of 1/bands of the image (pmg_run_band): the time estimate
                           counts the tiles of one band; <= 1 = whole image */
  int32_t no_inline;    /* 0 (default): substitute data-expanding intermediate stages into their readers
                           (a B200 option outside the paper); 1: schedule the text as written */
  int32_t tune;         /* 0 (default): the model's schedule.  1: measured selection on the plan's device -- the
                           DP schedule and every schedule that merges two neighbouring groups of it are compiled,
                           run on synthetic inputs and timed (CUDA events); the fastest is kept.  Plan creation
                           then takes seconds per candidate; runs are unaffected.  A B200 refinement outside the
                           paper's model-based selector. */
  int32_t reassoc;      /* 0 (default): every f32 operation in the written order (bit-identical to the oracle).
                           1: reassociation mode: rank-1 linear stencils are evaluated separably
                           (row sums reused across reader rows, factor.cpp) and a*b+c contracts to one fma;
                           results differ from the written order by rounding only, within the north_star f32
                           tolerance (tests/test_gpu_reassoc.py).  Integer stages are never rewritten. */
  const double* time_per_iter;  /* NULL = static operation counts; else per stage (declaration order) the measured
                                   TimePerIter in seconds (pmg_profile_stages) used by Alg. 2's
                                   compute term (cost_model 1); stages the schedule rewrote keep the static count */
  int32_t border_rows;  /* rows of the border-tile kernel's tiles (TH_b, a divisor of TH): <= 0 = 8.  Border tiles
                           are latency-bound (one warp walks a tile through the general body), so small pyramid
                           levels and the camera's quad grids run faster with 2-4; measured selection (tune) tries
                           2, 4 and 8 on its final grouping */
  int32_t reserved2;
} pmg_sched_opts;

const char* pmg_last_error(void);
const char* pmg_version(void);

/* ---- pipeline (host only) ---- */
pmg_status pmg_pipeline_parse(const char* text, size_t len, pmg_pipeline* out);
void pmg_pipeline_destroy(pmg_pipeline p); /* NULL-safe */
int pmg_pipeline_num_params(pmg_pipeline p);
pmg_status pmg_pipeline_param_name(pmg_pipeline p, int idx, char* buf, size_t cap);
int pmg_pipeline_num_stages(pmg_pipeline p);
pmg_status pmg_pipeline_stage_name(pmg_pipeline p, int idx, char* buf, size_t cap);
/* inputs: images then tables, declaration order; outputs: liveouts in declaration order */
int pmg_pipeline_num_io(pmg_pipeline p, int is_output);
pmg_status pmg_pipeline_io(pmg_pipeline p, int is_output, int idx, const int64_t* params, int nparams,
                           pmg_io_desc* out);
/* dependence / footprint table as JSON (§2.3; per edge and dim: offsets, scale) */
pmg_status pmg_pipeline_describe(pmg_pipeline p, const int64_t* params, int nparams, char* buf, size_t cap,
                                 size_t* needed);

/* ---- GPU description and weights ---- */
pmg_status pmg_gpu_spec_preset(const char* name /* "gtx1080ti", "teslav100", "b200" */, pmg_gpu_spec* out);
pmg_status pmg_gpu_spec_query(int device, double measured_bw_gbs /* <=0: preset value */, pmg_gpu_spec* out);
pmg_status pmg_weights_preset(const char* name /* "gtx1080ti", "teslav100", "b200" */, pmg_weights* out);
void pmg_sched_opts_default(pmg_sched_opts* o);

/* ---- host-only analysis (no GPU) ----
 * pmg_schedule: fusion grouping + per-group configuration with every Alg. 2 term, as JSON.
 * pmg_analyze_group: the paper's §4 geometry and Alg. 2 for one explicit group and configuration
 * (paper notation: tile T, block B, fracReg, txSz); used to pin the worked examples of §3/§4.        */
/* the pipeline text after substituting data-expanding intermediate stages into their readers (what plans
 * schedule unless sched_opts.no_inline): JSON {"inlined": [names], "text": "..."} */
pmg_status pmg_pipeline_inlined(pmg_pipeline p, const int64_t* params, int nparams, char* buf, size_t cap,
                                size_t* needed);
/* the pipeline text a plan made with `opts` schedules (NULL = defaults): rank-1 stencils factored when
 * opts->reassoc (factor.cpp), then inlining and phase splitting unless opts->no_inline.
 * JSON {"factored": [...], "inlined": [...], "split": [...], "text": "..."}; buffer protocol as above. */
pmg_status pmg_pipeline_rewritten(pmg_pipeline p, const int64_t* params, int nparams, const pmg_sched_opts* opts,
                                  char* buf, size_t cap, size_t* needed);
pmg_status pmg_schedule(pmg_pipeline p, const int64_t* params, int nparams, const pmg_gpu_spec* spec,
                        const pmg_weights* w, const pmg_sched_opts* opts, char* json, size_t cap, size_t* needed);
pmg_status pmg_analyze_group(pmg_pipeline p, const int64_t* params, int nparams, const char* stages_csv,
                             const int32_t tile[3], const int32_t block[3], double frac_reg, int32_t tx_size,
                             int32_t regs_per_stage, const pmg_gpu_spec* spec, const pmg_weights* w,
                             char* json, size_t cap, size_t* needed);
/* emit the CUDA source of every group kernel (no compilation); JSON {"groups":[{"name","source"}]} */
pmg_status pmg_emit(pmg_pipeline p, const int64_t* params, int nparams, const pmg_gpu_spec* spec,
                    const pmg_weights* w, const pmg_sched_opts* opts, char* json, size_t cap, size_t* needed);
/* compile every group kernel for sm_100a with NVRTC (no GPU needed); writes cubins + sources under dir */
pmg_status pmg_precompile(pmg_pipeline p, const int64_t* params, int nparams, const pmg_gpu_spec* spec,
                          const pmg_weights* w, const pmg_sched_opts* opts, const char* out_dir,
                          char* json, size_t cap, size_t* needed);

/* ---- plans (GPU) ---- */
pmg_status pmg_plan_create(pmg_pipeline p, const int64_t* params, int nparams, int device,
                           const pmg_gpu_spec* spec /* NULL = query device */, const pmg_weights* w /* NULL = b200 */,
                           const pmg_sched_opts* opts /* NULL = automatic */, pmg_plan* out);
void pmg_plan_destroy(pmg_plan plan); /* NULL-safe; caller ensures no run is in flight */
pmg_status pmg_plan_describe(pmg_plan plan, char* buf, size_t cap, size_t* needed); /* JSON */
pmg_status pmg_plan_workspace_bytes(pmg_plan plan, size_t* out);
int pmg_plan_num_kernels(pmg_plan plan);   /* fused groups (each launches an interior and/or a border kernel) */
/* kernels the most recent run / run_batch / run_band call launched (0..2 per group: interior tiles on the
 * caller's stream, border tiles on a forked side stream; empty classes are not launched); -1 for NULL */
int pmg_plan_last_launches(pmg_plan plan);

/* full-image run: in[] = images then tables (declaration order), out[] = liveouts */
pmg_status pmg_run(pmg_plan plan, const pmg_buf* in, int nin, const pmg_buf* out, int nout, void* workspace,
                   void* stream /* cudaStream_t / CUstream; NULL = legacy default stream */);
/* nframes independent images: frame f of tensor i is at in[i].ptr + f * frame_stride_bytes[i] */
pmg_status pmg_run_batch(pmg_plan plan, int nframes, const pmg_buf* in, const int64_t* in_frame_stride, int nin,
                         const pmg_buf* out, const int64_t* out_frame_stride, int nout, void* workspace, void* stream);
/* row bands (multi-GPU sharding): band b of n computes output rows [out_r0, out_r1) of every
 * liveout; it needs input image rows [in_r0, in_r1) (pipeline-wide cumulative halo, clipped).  Rows are
 * of the pipeline's full-resolution row space (parameter H). */
pmg_status pmg_band_rows(pmg_plan plan, int band, int nbands, int64_t* out_r0, int64_t* out_r1, int64_t* in_r0,
                         int64_t* in_r1);
/* the same band geometry without a GPU (schedule computed on the host with spec/weights/opts) */
pmg_status pmg_band_rows_host(pmg_pipeline p, const int64_t* params, int nparams, const pmg_gpu_spec* spec,
                              const pmg_weights* w, const pmg_sched_opts* opts, int band, int nbands, int64_t* out_r0,
                              int64_t* out_r1, int64_t* in_r0, int64_t* in_r1);
/* in[i] points at global row in_r0 of image i (tables: whole table); out[j] at global row out_r0 */
pmg_status pmg_run_band(pmg_plan plan, int band, int nbands, const pmg_buf* in, int nin, const pmg_buf* out,
                        int nout, void* workspace, void* stream);

/* ---- halo-exchange bands (the paper is single-GPU) ----
 * Instead of recomputing the pipeline-wide cumulative halo, band b of n computes only its OWN rows of every
 * group, own_g(b) = [b*Hg/n, (b+1)*Hg/n) at the group's row extent Hg, and receives the rows of earlier groups'
 * workspace stages that its later groups read beyond them from the bands owning them (pyramid pipelines: a few
 * rows per level instead of ~4x recompute at 8 bands).
 * pmg_band_exchange: JSON {"band","nbands","in":[lo,hi] (image rows of the band's input buffers),"out":[lo,hi],
 *   "groups":[[lo,hi] own rows per group],"stages":[{"name","group","offset","row_pitch","plane_pitch","planes",
 *   "rows","buf":[lo,hi] (rows the band's workspace slot holds: row r of plane k is at workspace + offset +
 *   k*plane_pitch + (r - buf.lo)*row_pitch),"need","own"}],"recv":[{"stage","peer","rows","after_group"}],
 *   "send":[...]}; every rank derives the same pairs, so the caller's transport (NCCL send/recv, peer copies)
 *   only moves bytes.  Buffer protocol as pmg_schedule.
 * pmg_run_band_groups: launch groups [group_begin, group_end) of band b in this mode; in[] holds image rows
 *   "in", out[] liveout rows "out"; the workspace slots must hold the received rows of the stages those groups
 *   read (exchange after each group, before the next call).  Stream-ordered like pmg_run. */
pmg_status pmg_band_exchange(pmg_plan plan, int band, int nbands, char* json, size_t cap, size_t* needed);
pmg_status pmg_band_exchange_host(pmg_pipeline p, const int64_t* params, int nparams, const pmg_gpu_spec* spec,
                                  const pmg_weights* w, const pmg_sched_opts* opts, int band, int nbands, char* json,
                                  size_t cap, size_t* needed);
pmg_status pmg_run_band_groups(pmg_plan plan, int band, int nbands, int group_begin, int group_end, const pmg_buf* in,
                               int nin, const pmg_buf* out, int nout, void* workspace, void* stream);

/* end-to-end run from host memory (the bench's e2e path): host_in / host_out are host images in the
 * pmg_buf layout (pinned memory gives asynchronous copies); dev_in / dev_out are caller-owned full-size
 * device staging buffers (16-byte aligned pitches).  The image is cut into `chunks` row bands (1..64,
 * pmg_band_rows geometry): band b's new input rows are copied in on a plan-owned copy-in stream, band b
 * runs on `stream`, and its output rows are copied out on a plan-owned copy-out stream, so the copies of
 * neighbouring bands overlap each other and the compute.  Every input row is copied once; tables are
 * copied whole first.  Stream-ordered: everything completes before later work on `stream`; the host
 * buffers must stay valid until then.  Input images must have the liveouts' row extent. */
pmg_status pmg_run_host(pmg_plan plan, const pmg_buf* host_in, int nin, const pmg_buf* host_out, int nout,
                        const pmg_buf* dev_in, const pmg_buf* dev_out, void* workspace, int chunks, void* stream);

/* on-device TimePerIter microbenchmarks (§6 l.890-898: "TimePerIter ... obtained by running each stage
 * in isolation"): every stage of the pipeline as written runs as its own kernel (one stage per group, no
 * inlining) on synthetic inputs of the given extents; each kernel is timed alone (CUDA events, best of 3 samples
 * of 10 runs).  JSON {"stages":[{"name","points","us","time_per_iter","regs"}]}; time_per_iter = us / points, the
 * per-point time of the stage's standalone kernel (memory included).  Needs the device. */
pmg_status pmg_profile_stages(pmg_pipeline p, const int64_t* params, int nparams, int device, char* json, size_t cap,
                              size_t* needed);

/* device self-test of the warp-shuffle semantics of Fig. 1: lane 0 receives the sum */
pmg_status pmg_selftest_shuffle(int device, int32_t* lane0_sum);

#ifdef __cplusplus
}
#endif
#endif /* PMG_H */
