// capi.cpp — extern "C" entry points of include/pmg.h; thread-local error messages; no exceptions cross
// the ABI.
#include <cstring>
#include <sstream>
#include <string>

#include "../../include/pmg.h"
#include "cudrv.hpp"
#include "runtime.hpp"
#include "select.hpp"

using namespace pmg;

struct pmg_pipeline_s {
  std::shared_ptr<Pipeline> p;
};
struct pmg_plan_s {
  std::unique_ptr<Plan> plan;
};

static thread_local std::string g_err;

static pmg_status fail(int st, const std::string& m) {
  g_err = m;
  return (pmg_status)st;
}

#define PMG_TRY(...)                                   \
  try {                                                \
    __VA_ARGS__                                        \
  } catch (const Error& e) {                           \
    return fail(e.status, e.what());                   \
  } catch (const std::bad_alloc&) {                    \
    return fail(PMG_ERR_OOM, "out of host memory");   \
  } catch (const std::exception& e) {                  \
    return fail(PMG_ERR_INVALID, e.what());            \
  }

static pmg_status put_json(const std::string& s, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (!buf || cap == 0) return PMG_OK;
  if (cap < s.size() + 1) return fail(PMG_ERR_ARG, "buffer too small (" + std::to_string(s.size() + 1) + " bytes needed)");
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return PMG_OK;
}

static std::vector<int64_t> pvec(const int64_t* params, int n) {
  return params && n > 0 ? std::vector<int64_t>(params, params + n) : std::vector<int64_t>{};
}

extern "C" {

const char* pmg_last_error(void) { return g_err.c_str(); }
const char* pmg_version(void) { return "pmg-b200 0.1 (OTPW + hybrid tiling, sm_100a)"; }

pmg_status pmg_pipeline_parse(const char* text, size_t len, pmg_pipeline* out) {
  if (!text || !out) return fail(PMG_ERR_ARG, "NULL argument");
  PMG_TRY({
    auto p = parse_pipeline(std::string(text, len));
    *out = new pmg_pipeline_s{p};
    return PMG_OK;
  })
}

void pmg_pipeline_destroy(pmg_pipeline p) { delete p; }

int pmg_pipeline_num_params(pmg_pipeline p) { return p ? (int)p->p->params.size() : -1; }
int pmg_pipeline_num_stages(pmg_pipeline p) { return p ? (int)p->p->stages.size() : -1; }

static pmg_status copy_str(const std::string& s, char* buf, size_t cap) {
  if (!buf || cap < s.size() + 1) return fail(PMG_ERR_ARG, "buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return PMG_OK;
}

pmg_status pmg_pipeline_param_name(pmg_pipeline p, int idx, char* buf, size_t cap) {
  if (!p || idx < 0 || idx >= (int)p->p->params.size()) return fail(PMG_ERR_ARG, "bad pipeline or index");
  return copy_str(p->p->params[idx], buf, cap);
}

pmg_status pmg_pipeline_stage_name(pmg_pipeline p, int idx, char* buf, size_t cap) {
  if (!p || idx < 0 || idx >= (int)p->p->stages.size()) return fail(PMG_ERR_ARG, "bad pipeline or index");
  return copy_str(p->p->stages[idx].name, buf, cap);
}

int pmg_pipeline_num_io(pmg_pipeline p, int is_output) {
  if (!p) return -1;
  return is_output ? (int)p->p->liveouts.size() : (int)(p->p->images.size() + p->p->tables.size());
}

pmg_status pmg_pipeline_io(pmg_pipeline p, int is_output, int idx, const int64_t* params, int nparams, pmg_io_desc* out) {
  if (!p || !out) return fail(PMG_ERR_ARG, "NULL argument");
  PMG_TRY({
    const Pipeline& pp = *p->p;
    std::vector<int64_t> pv = pvec(params, nparams);
    if (pv.size() != pp.params.size()) return fail(PMG_ERR_ARG, "wrong number of parameter values");
    std::memset(out, 0, sizeof *out);
    const std::vector<ExprP>* ext = nullptr;
    std::vector<ExprP> tabext;
    std::string name;
    DType dt;
    if (is_output) {
      if (idx < 0 || idx >= (int)pp.liveouts.size()) return fail(PMG_ERR_ARG, "bad output index");
      const StageDecl& s = pp.stages[pp.liveouts[idx]];
      ext = &s.extents;
      name = s.name;
      dt = s.dtype;
    } else if (idx >= 0 && idx < (int)pp.images.size()) {
      ext = &pp.images[idx].extents;
      name = pp.images[idx].name;
      dt = pp.images[idx].dtype;
    } else if (idx >= (int)pp.images.size() && idx < (int)(pp.images.size() + pp.tables.size())) {
      const TableDecl& t = pp.tables[idx - pp.images.size()];
      tabext = {t.extent};
      ext = &tabext;
      name = t.name;
      dt = t.dtype;
      out->is_table = 1;
    } else {
      return fail(PMG_ERR_ARG, "bad input index");
    }
    std::strncpy(out->name, name.c_str(), sizeof out->name - 1);
    out->dtype = (int32_t)dt;
    out->ndim = (int32_t)ext->size();
    for (size_t d = 0; d < ext->size(); ++d) out->extent[d] = eval_int(*(*ext)[d], pv);
    return PMG_OK;
  })
}

pmg_status pmg_pipeline_describe(pmg_pipeline p, const int64_t* params, int nparams, char* buf, size_t cap, size_t* needed) {
  if (!p) return fail(PMG_ERR_ARG, "NULL pipeline");
  PMG_TRY({
    Analysis A = analyze(*p->p, pvec(params, nparams));
    return put_json(describe_pipeline(A), buf, cap, needed);
  })
}

static pmg_status rewritten_json(pmg_pipeline p, const int64_t* params, int nparams, const pmg_sched_opts* opts,
                                 char* buf, size_t cap, size_t* needed) {
  if (!p) return fail(PMG_ERR_ARG, "NULL pipeline");
  PMG_TRY({
    std::vector<std::string> fac, names, split;
    auto q = p->p;
    if (opts && opts->reassoc) q = factor_stencils(q, pvec(params, nparams), &fac);
    if (!(opts && opts->no_inline)) {
      q = inline_expanding(q, pvec(params, nparams), &names);
      q = phase_split(q, pvec(params, nparams), &split);
    }
    std::ostringstream o;
    auto list = [&](const char* key, const std::vector<std::string>& v) {
      o << "\"" << key << "\":[";
      for (size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << "\"" << v[i] << "\"";
      o << "],";
    };
    o << "{";
    list("factored", fac);
    list("inlined", names);
    list("split", split);
    o << "\"text\":\"";
    for (char c : q->source) {
      if (c == '\n') o << "\\n";
      else if (c == '"' || c == '\\') o << '\\' << c;
      else o << c;
    }
    o << "\"}";
    return put_json(o.str(), buf, cap, needed);
  })
}

pmg_status pmg_pipeline_inlined(pmg_pipeline p, const int64_t* params, int nparams, char* buf, size_t cap, size_t* needed) {
  return rewritten_json(p, params, nparams, nullptr, buf, cap, needed);
}

pmg_status pmg_pipeline_rewritten(pmg_pipeline p, const int64_t* params, int nparams, const pmg_sched_opts* opts,
                                  char* buf, size_t cap, size_t* needed) {
  return rewritten_json(p, params, nparams, opts, buf, cap, needed);
}

pmg_status pmg_gpu_spec_preset(const char* name, pmg_gpu_spec* out) {
  if (!name || !out) return fail(PMG_ERR_ARG, "NULL argument");
  if (!gpu_preset(name, out)) return fail(PMG_ERR_ARG, std::string("unknown GPU preset '") + name + "'");
  return PMG_OK;
}

pmg_status pmg_weights_preset(const char* name, pmg_weights* out) {
  if (!name || !out) return fail(PMG_ERR_ARG, "NULL argument");
  if (!weights_preset(name, out)) return fail(PMG_ERR_ARG, std::string("unknown weights preset '") + name + "'");
  return PMG_OK;
}

pmg_status pmg_gpu_spec_query(int device, double measured_bw_gbs, pmg_gpu_spec* out) {
  if (!out) return fail(PMG_ERR_ARG, "NULL argument");
  Drv& D = drv();
  if (!D.ok) return fail(PMG_ERR_CUDA, D.err);
  gpu_preset("b200", out);
  CUdevice dev;
  CUresult r = D.DeviceGet(&dev, device);
  if (r != CUDA_SUCCESS) return fail(PMG_ERR_CUDA, cu_err(r));
  int v;
  char nm[64] = {0};
  D.DeviceGetName(nm, 63, dev);
  std::memset(out->name, 0, sizeof out->name);
  std::strncpy(out->name, nm, sizeof out->name - 1);
  if (D.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev) == CUDA_SUCCESS) out->nsms = v;
  if (D.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_MULTIPROCESSOR, dev) == CUDA_SUCCESS) out->shmem_per_sm = v;
  if (D.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_BLOCK_OPTIN, dev) == CUDA_SUCCESS) out->max_shmem_per_tb = v;
  if (D.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MAX_REGISTERS_PER_MULTIPROCESSOR, dev) == CUDA_SUCCESS) out->regs_per_sm = v;
  if (D.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MAX_THREADS_PER_MULTIPROCESSOR, dev) == CUDA_SUCCESS) {
    out->max_threads_per_sm = v;
    out->max_warps_per_sm = v / 32;
  }
  if (D.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MAX_BLOCKS_PER_MULTIPROCESSOR, dev) == CUDA_SUCCESS) out->max_tb_per_sm = v;
  if (D.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_L2_CACHE_SIZE, dev) == CUDA_SUCCESS) out->l2_bytes = v;
  if (D.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_CLOCK_RATE, dev) == CUDA_SUCCESS) out->sm_clock_hz = v * 1e3;
  if (measured_bw_gbs > 0) out->gl_mem_bw = measured_bw_gbs * 1e9;
  return PMG_OK;
}

void pmg_sched_opts_default(pmg_sched_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->group_of_stage = nullptr;
  o->vec = o->chunks = o->rows = o->warps = o->prefetch = o->tx_size = -1;
  o->smem_chunks = -1;
  o->budget = 0;
  o->fuse = 1;
  o->probe = 1;
}

// the pipeline the schedule works on: data-expanding stages substituted into their readers unless disabled
static std::shared_ptr<Pipeline> effective(const std::shared_ptr<Pipeline>& p, const std::vector<int64_t>& params,
                                           const pmg_sched_opts* opts) {
  std::shared_ptr<Pipeline> q = (opts && opts->reassoc) ? factor_stencils(p, params, nullptr) : p;
  if (opts && opts->no_inline) return q;
  return phase_split(inline_expanding(q, params, nullptr), params, nullptr);
}

static void spec_or_default(const pmg_gpu_spec* s, const pmg_weights* w, pmg_gpu_spec& S, pmg_weights& W) {
  if (s) S = *s;
  else gpu_preset("b200", &S);
  if (w) W = *w;
  else weights_preset("b200", &W);
}

pmg_status pmg_schedule(pmg_pipeline p, const int64_t* params, int nparams, const pmg_gpu_spec* spec, const pmg_weights* w,
                        const pmg_sched_opts* opts, char* json, size_t cap, size_t* needed) {
  if (!p) return fail(PMG_ERR_ARG, "NULL pipeline");
  PMG_TRY({
    auto eff = effective(p->p, pvec(params, nparams), opts);
    Analysis A = analyze(*eff, pvec(params, nparams));
    pmg_gpu_spec S;
    pmg_weights W;
    spec_or_default(spec, w, S, W);
    pmg_sched_opts o;
    if (opts) o = *opts;
    else pmg_sched_opts_default(&o);
    std::vector<double> tpi = map_time_per_iter(*p->p, *eff, o.time_per_iter);
    if (o.time_per_iter) o.time_per_iter = tpi.data();
    RegProbe probe = make_probe(A);
    Schedule sch = schedule(A, S, W, o, o.probe ? &probe : nullptr);
    return put_json(sch.json, json, cap, needed);
  })
}

pmg_status pmg_analyze_group(pmg_pipeline p, const int64_t* params, int nparams, const char* stages_csv, const int32_t tile[3],
                             const int32_t block[3], double frac_reg, int32_t tx_size, int32_t regs_per_stage,
                             const pmg_gpu_spec* spec, const pmg_weights* w, char* json, size_t cap, size_t* needed) {
  if (!p || !stages_csv || !tile || !block) return fail(PMG_ERR_ARG, "NULL argument");
  PMG_TRY({
    Analysis A = analyze(*p->p, pvec(params, nparams));
    std::vector<int> st;
    std::string csv = stages_csv, tok;
    size_t pos = 0;
    while (pos <= csv.size()) {
      size_t q = csv.find(',', pos);
      if (q == std::string::npos) q = csv.size();
      tok = csv.substr(pos, q - pos);
      pos = q + 1;
      if (tok.empty()) continue;
      int id = -1;
      for (size_t i = 0; i < p->p->stages.size(); ++i)
        if (p->p->stages[i].name == tok) id = (int)i;
      if (id < 0) return fail(PMG_ERR_ARG, "unknown stage '" + tok + "'");
      st.push_back(id);
    }
    if (st.empty()) return fail(PMG_ERR_ARG, "empty group");
    for (int d = 0; d < 3; ++d)
      if (tile[d] < 1 || block[d] < 1) return fail(PMG_ERR_ARG, "tile and block sizes must be >= 1");
    pmg_gpu_spec S;
    pmg_weights W;
    spec_or_default(spec, w, S, W);
    int T[3] = {tile[0], tile[1], tile[2]}, B[3] = {block[0], block[1], block[2]};
    return put_json(paper_analyze_group(A, st, T, B, frac_reg, tx_size, regs_per_stage, S, W), json, cap, needed);
  })
}

pmg_status pmg_emit(pmg_pipeline p, const int64_t* params, int nparams, const pmg_gpu_spec* spec, const pmg_weights* w,
                    const pmg_sched_opts* opts, char* json, size_t cap, size_t* needed) {
  if (!p) return fail(PMG_ERR_ARG, "NULL pipeline");
  PMG_TRY({
    auto eff = effective(p->p, pvec(params, nparams), opts);
    Analysis A = analyze(*eff, pvec(params, nparams));
    pmg_gpu_spec S;
    pmg_weights W;
    spec_or_default(spec, w, S, W);
    pmg_sched_opts o;
    if (opts) o = *opts;
    else pmg_sched_opts_default(&o);
    std::vector<double> tpi = map_time_per_iter(*p->p, *eff, o.time_per_iter);
    if (o.time_per_iter) o.time_per_iter = tpi.data();
    RegProbe probe = make_probe(A);
    Schedule sch = schedule(A, S, W, o, o.probe ? &probe : nullptr);
    std::string out = "{\"schedule\":" + sch.json + ",\"groups\":[";
    for (size_t i = 0; i < sch.groups.size(); ++i) {
      std::string src = emit_group(A, sch.groups[i]);
      std::string esc;
      for (char c : src) {
        if (c == '"') esc += "\\\"";
        else if (c == '\\') esc += "\\\\";
        else if (c == '\n') esc += "\\n";
        else esc += c;
      }
      out += (i ? "," : "") + std::string("{\"name\":\"") + sch.groups[i].name + "\",\"source\":\"" + esc + "\"}";
    }
    out += "]}";
    return put_json(out, json, cap, needed);
  })
}

pmg_status pmg_precompile(pmg_pipeline p, const int64_t* params, int nparams, const pmg_gpu_spec* spec, const pmg_weights* w,
                          const pmg_sched_opts* opts, const char* out_dir, char* json, size_t cap, size_t* needed) {
  if (!p) return fail(PMG_ERR_ARG, "NULL pipeline");
  PMG_TRY({
    auto eff = effective(p->p, pvec(params, nparams), opts);
    Analysis A = analyze(*eff, pvec(params, nparams));
    pmg_gpu_spec S;
    pmg_weights W;
    spec_or_default(spec, w, S, W);
    pmg_sched_opts o;
    if (opts) o = *opts;
    else pmg_sched_opts_default(&o);
    std::vector<double> tpi = map_time_per_iter(*p->p, *eff, o.time_per_iter);
    if (o.time_per_iter) o.time_per_iter = tpi.data();
    RegProbe probe = make_probe(A);
    Schedule sch = schedule(A, S, W, o, o.probe ? &probe : nullptr);
    std::string out = "{\"schedule\":" + sch.json + ",\"kernels\":[";
    for (size_t i = 0; i < sch.groups.size(); ++i) {
      Compiled c = jit_compile(sch.groups[i].name, emit_group(A, sch.groups[i]), out_dir ? out_dir : "");
      out += (i ? "," : "") + std::string("{\"name\":\"") + c.name + "\",\"regs\":" + std::to_string(c.regs) +
             ",\"spill_stores\":" + std::to_string(c.spill_stores) + ",\"spill_loads\":" + std::to_string(c.spill_loads) +
             ",\"cubin_bytes\":" + std::to_string(c.cubin.size()) + ",\"cached\":" + (c.from_cache ? "true" : "false") + "}";
    }
    out += "]}";
    return put_json(out, json, cap, needed);
  })
}

pmg_status pmg_plan_create(pmg_pipeline p, const int64_t* params, int nparams, int device, const pmg_gpu_spec* spec,
                           const pmg_weights* w, const pmg_sched_opts* opts, pmg_plan* out) {
  if (!p || !out) return fail(PMG_ERR_ARG, "NULL argument");
  PMG_TRY({
    auto plan = plan_create(p->p, pvec(params, nparams), device, spec, w, opts);
    *out = new pmg_plan_s{std::move(plan)};
    return PMG_OK;
  })
}

void pmg_plan_destroy(pmg_plan plan) {
  if (!plan) return;
  try { plan_destroy(plan->plan.get()); } catch (...) {}
  delete plan;
}

pmg_status pmg_profile_stages(pmg_pipeline p, const int64_t* params, int nparams, int device, char* json, size_t cap,
                              size_t* needed) {
  if (!p) return fail(PMG_ERR_ARG, "NULL pipeline");
  PMG_TRY({
    pmg_sched_opts o;
    pmg_sched_opts_default(&o);
    o.fuse = 0;        // one stage per group: every stage is its own kernel
    o.no_inline = 1;   // the pipeline as written
    auto P = plan_create(p->p, pvec(params, nparams), device, nullptr, nullptr, &o);
    std::vector<double> us = profile_groups_us(*P);
    std::ostringstream js;
    js << "{\"stages\":[";
    for (size_t gi = 0; gi < P->sch.groups.size(); ++gi) {
      const Group& g = P->sch.groups[gi];
      const int s = g.stages.at(0);
      int64_t pts = 1;
      for (int d = 0; d < 3; ++d)
        if (P->A.stage_ext[s].has[d]) pts *= P->A.stage_ext[s].e[d];
      js << (gi ? "," : "") << "{\"name\":\"" << p->p->stages[s].name << "\",\"index\":" << s << ",\"points\":" << pts
         << ",\"us\":" << us[gi] << ",\"time_per_iter\":" << us[gi] * 1e-6 / (double)pts << ",\"regs\":"
         << P->kernels[gi].bin.regs << "}";
    }
    js << "]}";
    return put_json(js.str(), json, cap, needed);
  })
}

pmg_status pmg_plan_describe(pmg_plan plan, char* buf, size_t cap, size_t* needed) {
  if (!plan) return fail(PMG_ERR_ARG, "NULL plan");
  std::string j = plan->plan->json;
  if (!plan->plan->tune_json.empty()) j = j.substr(0, j.size() - 1) + ",\"tune\":" + plan->plan->tune_json + "}";
  return put_json(j, buf, cap, needed);
}

pmg_status pmg_plan_workspace_bytes(pmg_plan plan, size_t* out) {
  if (!plan || !out) return fail(PMG_ERR_ARG, "NULL argument");
  *out = plan->plan->ws_bytes;
  return PMG_OK;
}

int pmg_plan_num_kernels(pmg_plan plan) { return plan ? (int)plan->plan->kernels.size() : -1; }

int pmg_plan_last_launches(pmg_plan plan) { return plan ? plan->plan->last_launches : -1; }

pmg_status pmg_run(pmg_plan plan, const pmg_buf* in, int nin, const pmg_buf* out, int nout, void* workspace, void* stream) {
  if (!plan || (!in && nin) || (!out && nout)) return fail(PMG_ERR_ARG, "NULL argument");
  PMG_TRY({
    plan_run(*plan->plan, in, nin, out, nout, workspace, (CUstream)stream, -1, 1, 1, nullptr, nullptr);
    return PMG_OK;
  })
}

pmg_status pmg_run_batch(pmg_plan plan, int nframes, const pmg_buf* in, const int64_t* in_frame_stride, int nin,
                         const pmg_buf* out, const int64_t* out_frame_stride, int nout, void* workspace, void* stream) {
  if (!plan || !in || !out || !in_frame_stride || !out_frame_stride) return fail(PMG_ERR_ARG, "NULL argument");
  if (nframes < 1) return fail(PMG_ERR_ARG, "nframes must be >= 1");
  PMG_TRY({
    plan_run(*plan->plan, in, nin, out, nout, workspace, (CUstream)stream, -1, 1, nframes, in_frame_stride, out_frame_stride);
    return PMG_OK;
  })
}

pmg_status pmg_band_rows(pmg_plan plan, int band, int nbands, int64_t* out_r0, int64_t* out_r1, int64_t* in_r0, int64_t* in_r1) {
  if (!plan || nbands < 1 || band < 0 || band >= nbands) return fail(PMG_ERR_ARG, "bad band");
  PMG_TRY({
    BandRows b = band_rows(*plan->plan, band, nbands);
    if (out_r0) *out_r0 = b.out_r0;
    if (out_r1) *out_r1 = b.out_r1;
    if (in_r0) *in_r0 = b.in_r0;
    if (in_r1) *in_r1 = b.in_r1;
    return PMG_OK;
  })
}

pmg_status pmg_band_rows_host(pmg_pipeline p, const int64_t* params, int nparams, const pmg_gpu_spec* spec,
                              const pmg_weights* w, const pmg_sched_opts* opts, int band, int nbands, int64_t* out_r0,
                              int64_t* out_r1, int64_t* in_r0, int64_t* in_r1) {
  if (!p || nbands < 1 || band < 0 || band >= nbands) return fail(PMG_ERR_ARG, "bad band");
  PMG_TRY({
    Plan P;
    P.pipe = effective(p->p, pvec(params, nparams), opts);
    P.A = analyze(*P.pipe, pvec(params, nparams));
    pmg_gpu_spec S;
    pmg_weights W;
    spec_or_default(spec, w, S, W);
    pmg_sched_opts o;
    if (opts) o = *opts;
    else pmg_sched_opts_default(&o);
    std::vector<double> tpi = map_time_per_iter(*p->p, *P.pipe, o.time_per_iter);
    if (o.time_per_iter) o.time_per_iter = tpi.data();
    P.sch = schedule(P.A, S, W, o, nullptr);
    BandRows b = band_rows(P, band, nbands);
    if (out_r0) *out_r0 = b.out_r0;
    if (out_r1) *out_r1 = b.out_r1;
    if (in_r0) *in_r0 = b.in_r0;
    if (in_r1) *in_r1 = b.in_r1;
    return PMG_OK;
  })
}

// halo-exchange band geometry as JSON (one band's view; the sends / receives of every band pair are derived
// from the same deterministic geometry on every rank)
static std::string xchg_json(const Plan& P, int band, int nbands) {
  const Pipeline& p = *P.pipe;
  std::vector<BandXchg> all;
  for (int b = 0; b < nbands; ++b) all.push_back(band_xchg(P, b, nbands));
  const BandXchg& X = all[band];
  std::vector<int> group_of(p.stages.size(), -1);
  for (size_t gi = 0; gi < P.sch.groups.size(); ++gi)
    for (int st : P.sch.groups[gi].stages) group_of[st] = (int)gi;
  auto iv = [](RowIv r) { return "[" + std::to_string(r.lo) + "," + std::to_string(r.hi) + "]"; };
  auto isect = [](RowIv a, RowIv b) { RowIv r{std::max(a.lo, b.lo), std::min(a.hi, b.hi)}; return r; };
  std::ostringstream o;
  o << "{\"band\":" << band << ",\"nbands\":" << nbands << ",\"in\":" << iv(X.in) << ",\"out\":" << iv(X.out)
    << ",\"groups\":[";
  for (size_t gi = 0; gi < X.own.size(); ++gi) o << (gi ? "," : "") << iv(X.own[gi]);
  o << "],\"stages\":[";
  std::ostringstream snd, rcv;
  bool fs = true, fr = true;
  for (size_t k = 0; k < P.ws.size(); ++k) {
    const WsTensor& w = P.ws[k];
    const int g = group_of[w.stage];
    o << (k ? "," : "") << "{\"name\":\"" << p.stages[w.stage].name << "\",\"group\":" << g << ",\"offset\":" << w.offset
      << ",\"row_pitch\":" << w.row_pitch << ",\"plane_pitch\":" << w.plane_pitch << ",\"planes\":" << w.planes
      << ",\"rows\":" << w.rows << ",\"buf\":" << iv(X.buf[w.stage]) << ",\"need\":" << iv(X.need[w.stage])
      << ",\"own\":" << iv(X.own[g]) << "}";
    for (int c = 0; c < nbands; ++c) {
      if (c == band) continue;
      RowIv r = isect(all[c].own[g], X.need[w.stage]);     // rows band c owns that this band reads
      if (r.hi > r.lo) {
        rcv << (fr ? "" : ",") << "{\"stage\":" << k << ",\"peer\":" << c << ",\"rows\":" << iv(r) << ",\"after_group\":" << g << "}";
        fr = false;
      }
      RowIv q = isect(X.own[g], all[c].need[w.stage]);     // rows this band owns that band c reads
      if (q.hi > q.lo) {
        snd << (fs ? "" : ",") << "{\"stage\":" << k << ",\"peer\":" << c << ",\"rows\":" << iv(q) << ",\"after_group\":" << g << "}";
        fs = false;
      }
    }
  }
  o << "],\"recv\":[" << rcv.str() << "],\"send\":[" << snd.str() << "],\"workspace_bytes\":" << P.ws_bytes << "}";
  return o.str();
}

pmg_status pmg_band_exchange(pmg_plan plan, int band, int nbands, char* json, size_t cap, size_t* needed) {
  if (!plan || nbands < 1 || band < 0 || band >= nbands) return fail(PMG_ERR_ARG, "bad band");
  PMG_TRY({ return put_json(xchg_json(*plan->plan, band, nbands), json, cap, needed); })
}

pmg_status pmg_band_exchange_host(pmg_pipeline p, const int64_t* params, int nparams, const pmg_gpu_spec* spec,
                                  const pmg_weights* w, const pmg_sched_opts* opts, int band, int nbands, char* json,
                                  size_t cap, size_t* needed) {
  if (!p || nbands < 1 || band < 0 || band >= nbands) return fail(PMG_ERR_ARG, "bad band");
  PMG_TRY({
    Plan P;
    P.pipe = effective(p->p, pvec(params, nparams), opts);
    P.A = analyze(*P.pipe, pvec(params, nparams));
    pmg_gpu_spec S;
    pmg_weights W;
    spec_or_default(spec, w, S, W);
    pmg_sched_opts o;
    if (opts) o = *opts;
    else pmg_sched_opts_default(&o);
    std::vector<double> tpi = map_time_per_iter(*p->p, *P.pipe, o.time_per_iter);
    if (o.time_per_iter) o.time_per_iter = tpi.data();
    P.sch = schedule(P.A, S, W, o, nullptr);
    layout_workspace(P);
    return put_json(xchg_json(P, band, nbands), json, cap, needed);
  })
}

pmg_status pmg_run_band_groups(pmg_plan plan, int band, int nbands, int group_begin, int group_end, const pmg_buf* in,
                               int nin, const pmg_buf* out, int nout, void* workspace, void* stream) {
  if (!plan || !in || !out || nbands < 1 || band < 0 || band >= nbands || group_begin < 0 || group_end < group_begin)
    return fail(PMG_ERR_ARG, "bad argument");
  PMG_TRY({
    const int gr[2] = {group_begin, group_end};
    plan_run(*plan->plan, in, nin, out, nout, workspace, (CUstream)stream, band, nbands, 1, nullptr, nullptr, gr);
    return PMG_OK;
  })
}

pmg_status pmg_run_band(pmg_plan plan, int band, int nbands, const pmg_buf* in, int nin, const pmg_buf* out, int nout,
                        void* workspace, void* stream) {
  if (!plan || !in || !out || nbands < 1 || band < 0 || band >= nbands) return fail(PMG_ERR_ARG, "bad argument");
  PMG_TRY({
    plan_run(*plan->plan, in, nin, out, nout, workspace, (CUstream)stream, band, nbands, 1, nullptr, nullptr);
    return PMG_OK;
  })
}

pmg_status pmg_run_host(pmg_plan plan, const pmg_buf* host_in, int nin, const pmg_buf* host_out, int nout,
                        const pmg_buf* dev_in, const pmg_buf* dev_out, void* workspace, int chunks, void* stream) {
  if (!plan || !host_in || !host_out || !dev_in || !dev_out || chunks < 1) return fail(PMG_ERR_ARG, "bad argument");
  PMG_TRY({
    plan_run_host(*plan->plan, host_in, nin, host_out, nout, dev_in, dev_out, workspace, chunks, (CUstream)stream);
    return PMG_OK;
  })
}

}  // extern "C"
