// runtime.cpp — NVRTC compilation for sm_100a, plan creation, workspace layout, band geometry and the
// stream-ordered launch of one kernel per fused group (§6.2: "the sum of
// execution time of all generated CUDA kernels").
#include "runtime.hpp"

#include <dlfcn.h>
#include <nvrtc.h>
#include <sys/stat.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <unistd.h>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <regex>
#include <set>
#include <sstream>

#include "cudrv.hpp"

namespace pmg {

#include "kernels_embed.inc"   // kOtpwHeader: kernels/pmg_otpw.cuh as a string (generated at build time)

static uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ULL) {
  for (unsigned char c : s) { h ^= c; h *= 1099511628211ULL; }
  return h;
}

std::string kernel_dir() {
  Dl_info info;
  if (dladdr((void*)&kernel_dir, &info) && info.dli_fname) {
    std::string f = info.dli_fname;
    auto pos = f.rfind('/');
    if (pos != std::string::npos) return f.substr(0, pos);
  }
  return ".";
}

static std::string cache_dir(const std::string& override_dir) {
  const char* e = getenv("PMG_CACHE_DIR");
  std::string d = !override_dir.empty() ? override_dir : e && *e ? e : kernel_dir() + "/../build/cubin_cache";
  std::string acc;
  std::stringstream ss(d);
  std::string part;
  if (!d.empty() && d[0] == '/') acc = "";
  while (std::getline(ss, part, '/')) {
    if (part.empty()) { acc += "/"; continue; }
    acc += part;
    mkdir(acc.c_str(), 0755);
    acc += "/";
  }
  return d;
}

static const char* kOptions[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo",
                                 "--ptxas-options=-v", "-default-device", "-DPMG_NVRTC=1"};

static void parse_ptxas(Compiled& c) {
  // per entry point: "Compiling entry function 'X'" ... "N bytes spill stores, M bytes spill loads" ... "Used R registers"
  std::string cur;
  std::istringstream in(c.log);
  std::string line;
  std::smatch m;
  while (std::getline(in, line)) {
    if (std::regex_search(line, m, std::regex("Compiling entry function '([A-Za-z0-9_]+)'"))) cur = m[1];
    else if (std::regex_search(line, m, std::regex("([0-9]+) bytes spill stores, ([0-9]+) bytes spill loads"))) {
      c.fns[cur].spill_stores = std::stoi(m[1]);
      c.fns[cur].spill_loads = std::stoi(m[2]);
    } else if (std::regex_search(line, m, std::regex("Used ([0-9]+) registers"))) c.fns[cur].regs = std::stoi(m[1]);
  }
  auto it = c.fns.find(c.name);
  if (it == c.fns.end() && !c.fns.empty()) it = c.fns.begin();
  if (it != c.fns.end()) {
    c.regs = it->second.regs;
    c.spill_stores = it->second.spill_stores;
    c.spill_loads = it->second.spill_loads;
  }
  if (std::regex_search(c.log, m, std::regex("([0-9]+) bytes smem"))) c.smem_static = std::stoi(m[1]);
}

Compiled jit_compile(const std::string& name, const std::string& source, const std::string& dir_override) {
  Compiled c;
  c.name = name;
  c.source = source;
  int maj = 0, min = 0;
  nvrtcVersion(&maj, &min);
  std::string key_src = source + "\n//" + std::string(kOtpwHeader);
  for (const char* o : kOptions) key_src += std::string(" ") + o;
  key_src += " nvrtc" + std::to_string(maj) + "." + std::to_string(min);
  char hex[32];
  snprintf(hex, sizeof hex, "%016llx", (unsigned long long)fnv1a(key_src));
  std::string dir = cache_dir(dir_override);
  std::string base = dir + "/" + name + "_" + hex;
  {
    std::ifstream f(base + ".cubin", std::ios::binary);
    std::ifstream lg(base + ".log");
    if (f && lg) {
      c.cubin.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
      c.log.assign(std::istreambuf_iterator<char>(lg), std::istreambuf_iterator<char>());
      if (!c.cubin.empty()) {
        c.from_cache = true;
        parse_ptxas(c);
        return c;
      }
    }
  }
  auto t0 = std::chrono::steady_clock::now();
  // keep the generated source on disk so ncu --import-source / -lineinfo map back to it
  std::string src_path = base + ".cu";
  { std::ofstream f(src_path); f << source; }
  nvrtcProgram prog;
  const char* hdrs[] = {kOtpwHeader};
  const char* hdr_names[] = {"pmg_otpw.cuh"};
  if (nvrtcCreateProgram(&prog, source.c_str(), src_path.c_str(), 1, hdrs, hdr_names) != NVRTC_SUCCESS)
    throw Error(-7, "nvrtcCreateProgram failed");
  nvrtcResult r = nvrtcCompileProgram(prog, (int)(sizeof kOptions / sizeof kOptions[0]), kOptions);
  size_t ls = 0;
  nvrtcGetProgramLogSize(prog, &ls);
  c.log.resize(ls);
  if (ls) nvrtcGetProgramLog(prog, &c.log[0]);
  if (r != NVRTC_SUCCESS) {
    std::string m = "NVRTC compilation of " + name + " failed: " + c.log.substr(0, 4000);
    nvrtcDestroyProgram(&prog);
    throw Error(-7, m);
  }
  size_t cs = 0;
  nvrtcGetCUBINSize(prog, &cs);
  c.cubin.resize(cs);
  nvrtcGetCUBIN(prog, c.cubin.data());
  nvrtcDestroyProgram(&prog);
  c.compile_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  parse_ptxas(c);
  // cache files are written under names unique to this process and call, then renamed into place (atomic on
  // POSIX), so concurrent processes (torchrun ranks) never read a partial file; the log (read first by the
  // cache lookup) is published before the cubin
  static std::atomic<unsigned> seq{0};
  const std::string tag = ".tmp." + std::to_string((long)getpid()) + "." + std::to_string(seq++);
  {
    std::ofstream f(base + ".log" + tag);
    f << c.log;
  }
  {
    std::ofstream f(base + ".cubin" + tag, std::ios::binary);
    f.write(c.cubin.data(), (std::streamsize)c.cubin.size());
  }
  if (std::rename((base + ".log" + tag).c_str(), (base + ".log").c_str()) != 0 ||
      std::rename((base + ".cubin" + tag).c_str(), (base + ".cubin").c_str()) != 0) {
    std::remove((base + ".log" + tag).c_str());   // cache write failed: the compiled cubin is still returned
    std::remove((base + ".cubin" + tag).c_str());
  }
  return c;
}

// register-probe results (ptxas registers / spill bytes of a candidate's interior kernel), keyed like the cubin
// cache; kept in a small text file next to libpmg.so (kernel_dir()/probe_cache.txt) that travels with the
// package, so plan creation on a fresh GPU box does not recompile the selector's finalists
static std::mutex g_probe_mu;
static std::map<std::string, std::pair<int, int>>* g_probe = nullptr;

static std::string probe_file() { return kernel_dir() + "/probe_cache.txt"; }

static std::string compile_key(const std::string& source) {
  int maj = 0, min = 0;
  nvrtcVersion(&maj, &min);
  std::string key_src = source + "\n//" + std::string(kOtpwHeader);
  for (const char* o : kOptions) key_src += std::string(" ") + o;
  key_src += " nvrtc" + std::to_string(maj) + "." + std::to_string(min);
  char hex[32];
  snprintf(hex, sizeof hex, "%016llx", (unsigned long long)fnv1a(key_src));
  return hex;
}

RegProbe make_probe(const Analysis& A) {
  return [&A](const Group& g, int* regs, int* spill) {
    Group h = g;
    h.name = "pmg_probe";
    const std::string src = emit_group(A, h, /*interior_only=*/true);
    const std::string key = compile_key(src);
    {
      std::lock_guard<std::mutex> lk(g_probe_mu);
      if (!g_probe) {
        g_probe = new std::map<std::string, std::pair<int, int>>();
        std::ifstream f(probe_file());
        std::string k;
        int r, sp;
        while (f >> k >> r >> sp) (*g_probe)[k] = {r, sp};
      }
      auto it = g_probe->find(key);
      if (it != g_probe->end()) {
        *regs = it->second.first;
        *spill = it->second.second;
        return *regs > 0;
      }
    }
    Compiled c = jit_compile(h.name, src);
    *regs = c.regs;
    *spill = std::max(c.spill_stores, 0) + std::max(c.spill_loads, 0);
    if (c.regs > 0) {
      std::lock_guard<std::mutex> lk(g_probe_mu);
      (*g_probe)[key] = {*regs, *spill};
      std::ofstream f(probe_file(), std::ios::app);   // one short line per append (O_APPEND)
      f << key << " " << *regs << " " << *spill << "\n";
    }
    return c.regs > 0;
  };
}

// -------------------------------------------------------------------------------------------- plans
static void check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw Error(-6, std::string(what) + ": " + cu_err(r));
}

struct CtxGuard {   // make the plan's primary context current for the duration of a call
  CUcontext prev = nullptr;
  bool active = false;
  explicit CtxGuard(CUcontext c) {
    drv().CtxGetCurrent(&prev);
    if (prev != c) { drv().CtxSetCurrent(c); active = true; }
  }
  ~CtxGuard() { if (active) drv().CtxSetCurrent(prev); }
};

static int64_t round_up64(int64_t a, int64_t m) { return (a + m - 1) / m * m; }

// device time of one run of plan Q on synthetic inputs (measured selection, pmg_sched_opts.tune): buffer sets
// (together >= 2x L2, rotated run by run) are allocated here, images filled with varied values; warm-up
// runs, then the best of 5 samples of 10 runs per set
static double time_plan_us(Plan& Q, int nbands = 1) {
  Drv& D = drv();
  const Pipeline& p = *Q.pipe;
  const Analysis& A = Q.A;
  std::vector<CUdeviceptr> mem;
  struct Free {
    Drv& D; std::vector<CUdeviceptr>& m;
    ~Free() { for (auto x : m) D.MemFree(x); }
  } free_all{D, mem};
  auto alloc = [&](size_t bytes) {
    CUdeviceptr d = 0;
    check(D.MemAlloc(&d, std::max<size_t>(bytes, 256)), "cuMemAlloc");
    mem.push_back(d);
    check(D.MemsetD8(d, 0x3c, std::max<size_t>(bytes, 256)), "cuMemsetD8");   // 0x3c3c3c3c = 0.0115f
    return d;
  };
  auto buf_of = [&](const Ext3& e, DType dt) {
    pmg_buf b{};
    b.row_pitch_bytes = round_up64(e.e[2] * dtype_size(dt), 128);
    b.plane_pitch_bytes = b.row_pitch_bytes * e.e[1];
    b.ptr = (void*)(uintptr_t)alloc((size_t)(b.plane_pitch_bytes * e.e[0]));
    return b;
  };
  // input images get varied values (f32 in [0, 1), integers in [0, 1024)): a constant image makes every
  // data-dependent read (lookup tables, the local Laplacian's plane selection, demosaic branches) hit one address
  // and times such plans optimistically.  One pattern per image, copied to every buffer set.
  std::vector<std::vector<uint8_t>> pattern(p.images.size());
  auto fill_image = [&](size_t i, const pmg_buf& b, const Ext3& e) {
    const DType dt = p.images[i].dtype;
    const size_t bytes = (size_t)(b.plane_pitch_bytes * e.e[0]);
    if (pattern[i].empty()) {
      pattern[i].resize(bytes);
      uint32_t x = 0x9e3779b9u ^ (uint32_t)(i * 7919);
      const int esz = dtype_size(dt);
      for (size_t k = 0; k + esz <= bytes; k += esz) {
        x = x * 1664525u + 1013904223u;
        if (dt == DType::F32) {
          const float f = (float)(x >> 8) * (1.0f / 16777216.0f);
          std::memcpy(&pattern[i][k], &f, 4);
        } else {
          const uint32_t v = (x >> 16) & 1023u;
          std::memcpy(&pattern[i][k], &v, (size_t)esz);
        }
      }
    }
    check(D.MemcpyHtoDAsync((CUdeviceptr)(uintptr_t)b.ptr, pattern[i].data(), bytes, nullptr), "cuMemcpyHtoDAsync");
  };
  // buffer sets rotated between runs, together at least twice the L2 (as bench.py times), at most 4
  size_t set_bytes = Q.ws_bytes;
  for (size_t i = 0; i < p.images.size(); ++i)
    set_bytes += (size_t)(round_up64(A.image_ext[i].e[2] * dtype_size(p.images[i].dtype), 128) * A.image_ext[i].e[1] * A.image_ext[i].e[0]);
  for (int s : p.liveouts)
    set_bytes += (size_t)(round_up64(A.stage_ext[s].e[2] * dtype_size(p.stages[s].dtype), 128) * A.stage_ext[s].e[1] * A.stage_ext[s].e[0]);
  const int nsets = (int)std::min<size_t>(4, std::max<size_t>(1, (2 * (size_t)Q.spec.l2_bytes + set_bytes - 1) / std::max<size_t>(1, set_bytes)));
  std::vector<std::vector<pmg_buf>> ins(nsets), outs(nsets);
  std::vector<void*> wss(nsets, nullptr);
  const int band = nbands > 1 ? nbands / 2 : -1;
  for (int k = 0; k < nsets; ++k) {
    auto& in = ins[k];
    auto& out = outs[k];
    for (size_t i = 0; i < p.images.size(); ++i) {
      in.push_back(buf_of(A.image_ext[i], p.images[i].dtype));
      fill_image(i, in.back(), A.image_ext[i]);
    }
    for (size_t i = 0; i < p.tables.size(); ++i) {
      pmg_buf b{};
      b.ptr = (void*)(uintptr_t)alloc((size_t)A.table_len[i] * dtype_size(p.tables[i].dtype));
      in.push_back(b);
    }
    for (int s : p.liveouts) out.push_back(buf_of(A.stage_ext[s], p.stages[s].dtype));
    wss[k] = Q.ws_bytes ? (void*)(uintptr_t)alloc(Q.ws_bytes) : nullptr;
    // plans made for row bands (sched_opts.bands = n) are timed on the middle band, as one rank runs it: the
    // buffers point at the band's first input / output row of the full-size allocations
    if (band >= 0) {
      BandRows br = band_rows(Q, band, nbands);
      for (size_t i = 0; i < p.images.size(); ++i) in[i].ptr = (char*)in[i].ptr + br.in_r0 * in[i].row_pitch_bytes;
      for (auto& o : out) o.ptr = (char*)o.ptr + br.out_r0 * o.row_pitch_bytes;
    }
  }
  auto run1 = [&](int r, CUstream st) {
    const int k = r % nsets;
    plan_run(Q, ins[k].data(), (int)ins[k].size(), outs[k].data(), (int)outs[k].size(), wss[k], st, band, nbands, 1,
             nullptr, nullptr);
  };
  CUstream st;
  check(D.CtxSynchronize(), "cuCtxSynchronize");   // the image copies (legacy stream) before the timed stream
  check(D.StreamCreate(&st, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
  CUevent e0, e1;
  check(D.EventCreate(&e0, 0), "cuEventCreate");
  check(D.EventCreate(&e1, 0), "cuEventCreate");
  for (int r = 0; r < 2 * nsets; ++r) run1(r, st);
  // the paper's statistic: the minimum over samples of the mean of back-to-back runs.  The R runs
  // are captured once into a CUDA graph and replayed, as bench.py times them: host-launched runs of a small
  // plan would measure the host's enqueue rate (about 10 us per run) instead of the device
  const int R = 10 * nsets;
  CUgraph graph = nullptr;
  CUgraphExec exec = nullptr;
  if (D.StreamBeginCapture(st, CU_STREAM_CAPTURE_MODE_RELAXED) == CUDA_SUCCESS) {
    bool ok = true;
    try {
      for (int r = 0; r < R; ++r) run1(r, st);
    } catch (const Error&) {
      ok = false;
    }
    if (D.StreamEndCapture(st, &graph) != CUDA_SUCCESS || !ok || !graph ||
        D.GraphInstantiateWithFlags(&exec, graph, 0) != CUDA_SUCCESS)
      exec = nullptr;
  }
  struct GraphFree {
    Drv& D; CUgraph& g; CUgraphExec& x;
    ~GraphFree() { if (x) D.GraphExecDestroy(x); if (g) D.GraphDestroy(g); }
  } graph_free{D, graph, exec};
  if (exec) check(D.GraphLaunch(exec, st), "cuGraphLaunch");
  float ms = 1e30f;
  for (int sample = 0; sample < 5; ++sample) {
    check(D.EventRecord(e0, st), "cuEventRecord");
    if (exec) check(D.GraphLaunch(exec, st), "cuGraphLaunch");
    else
      for (int r = 0; r < R; ++r) run1(r, st);
    check(D.EventRecord(e1, st), "cuEventRecord");
    check(D.EventSynchronize(e1), "cuEventSynchronize");
    float m = 0;
    check(D.EventElapsedTime(&m, e0, e1), "cuEventElapsedTime");
    ms = std::min(ms, m);
  }
  D.EventDestroy(e0);
  D.EventDestroy(e1);
  D.StreamDestroy(st);
  return 1000.0 * ms / R;
}

std::vector<double> profile_groups_us(Plan& P) {
  CtxGuard g(P.ctx);
  std::vector<double> us(P.sch.groups.size(), 0.0);
  struct Reset { Plan& P; ~Reset() { P.only_group = -1; } } reset{P};
  for (size_t gi = 0; gi < P.sch.groups.size(); ++gi) {
    P.only_group = (int)gi;
    us[gi] = time_plan_us(P);
  }
  return us;
}

// integer value of an index / condition expression at (c, y, x) of the stage with `nd` dims (floor / and %)
static bool ieval(const Expr& e, int nd, const int64_t cyx[3], const std::vector<int64_t>& prm, int64_t& v) {
  auto fl = [](int64_t a, int64_t b) { int64_t q = a / b; if ((a % b) && ((a < 0) != (b < 0))) --q; return q; };
  int64_t a = 0, b = 0, c = 0;
  switch (e.op) {
    case Expr::INT: v = e.ival; return true;
    case Expr::PARAM: v = prm.at(e.index); return true;
    case Expr::VAR: v = cyx[e.index + 3 - nd]; return true;
    case Expr::BIN:
      if (!ieval(*e.args[0], nd, cyx, prm, a) || !ieval(*e.args[1], nd, cyx, prm, b)) return false;
      if (e.text == "+") v = a + b;
      else if (e.text == "-") v = a - b;
      else if (e.text == "*") v = a * b;
      else if (e.text == "/") { if (!b) return false; v = fl(a, b); }
      else if (e.text == "%") { if (!b) return false; v = a - b * fl(a, b); }
      else if (e.text == "==") v = a == b;
      else if (e.text == "!=") v = a != b;
      else if (e.text == "<") v = a < b;
      else if (e.text == "<=") v = a <= b;
      else if (e.text == ">") v = a > b;
      else if (e.text == ">=") v = a >= b;
      else return false;
      return true;
    case Expr::CALL:
      if (e.text == "clamp" && e.args.size() == 3) {
        if (!ieval(*e.args[0], nd, cyx, prm, a) || !ieval(*e.args[1], nd, cyx, prm, b) || !ieval(*e.args[2], nd, cyx, prm, c))
          return false;
        v = std::min(std::max(a, b), c);
        return true;
      }
      return false;
    default: return false;
  }
}

// the read a pure select tree picks at (c, y, x): the ACCESS node, or nullptr when the expression is anything else
static const Expr* pick(const Expr& e, int nd, const int64_t cyx[3], const std::vector<int64_t>& prm) {
  if (e.op == Expr::ACCESS) return &e;
  if (e.op == Expr::CALL && e.text == "select" && e.args.size() == 3) {
    int64_t cond;
    if (!ieval(*e.args[0], nd, cyx, prm, cond)) return nullptr;
    return pick(*e.args[cond ? 1 : 2], nd, cyx, prm);
  }
  return nullptr;
}

void detect_interleave(Plan& P) {
  const char* env = getenv("PMG_ILV");   // "0": keep the interleave as its own kernel
  P.ilv.clear();
  P.ilv_skip.assign(P.sch.groups.size(), 0);
  if (env && env[0] == '0') return;
  const Pipeline& p = *P.pipe;
  const Analysis& A = P.A;
  std::vector<int> group_of(p.stages.size(), -1);
  for (size_t gi = 0; gi < P.sch.groups.size(); ++gi)
    for (int s : P.sch.groups[gi].stages) group_of[s] = (int)gi;
  for (size_t oi = 0; oi < p.liveouts.size(); ++oi) {
    const int L = p.liveouts[oi];
    const int gl = group_of[L];
    if (P.sch.groups[gl].stages.size() != 1 || !p.consumers[L].empty()) continue;
    const Ext3& le = A.stage_ext[L];
    if (!le.has[1] || !le.has[2] || le.e[1] % 2 || le.e[2] % 2) continue;
    const int nd = (int)p.stages[L].vars.size();
    const int64_t C = le.has[0] ? le.e[0] : 1;
    std::map<int, Plan::Ilv> found;
    int gsrc = -1;
    bool ok = true;
    for (int64_t c = 0; c < C && ok; ++c)
      for (int py = 0; py < 2 && ok; ++py)
        for (int px = 0; px < 2 && ok; ++px) {
          const Expr* r0 = nullptr;
          for (int smp = 0; smp < 2 && ok; ++smp) {   // two sample points: the read must be S(y/2, x/2)
            const int64_t yq = smp ? 3 : 0, xq = smp ? 5 : 0;
            const int64_t cyx[3] = {c, 2 * yq + py, 2 * xq + px};
            const Expr* r = pick(*p.stages[L].expr, nd, cyx, A.params);
            if (!r || !r->is_stage || r->args.size() != 2 || (r0 && r0->index != r->index)) { ok = false; break; }
            r0 = r;
            int64_t iy, ix;
            if (!ieval(*r->args[0], nd, cyx, A.params, iy) || !ieval(*r->args[1], nd, cyx, A.params, ix) || iy != yq ||
                ix != xq)
              ok = false;
          }
          if (!ok) break;
          const int S = r0->index;
          const Ext3& se = A.stage_ext[S];
          if (found.count(S) || se.has[0] || se.e[1] * 2 != le.e[1] || se.e[2] * 2 != le.e[2] ||
              p.stages[S].dtype != p.stages[L].dtype || p.consumers[S].size() != 1 || group_of[S] == gl ||
              (gsrc >= 0 && group_of[S] != gsrc)) {
            ok = false;
            break;
          }
          gsrc = group_of[S];
          found[S] = Plan::Ilv{(int)oi, (int)c, py, px};
        }
    if (!ok || gsrc < 0) continue;
    Group& G = P.sch.groups[gsrc];
    if (G.cfg.S != 0) continue;   // hybrid smem chunks keep their own store path
    for (auto& st : G.gs)
      if (found.count(st.id)) st.ilv = true;
    for (auto& kv : found) P.ilv[kv.first] = kv.second;
    P.ilv_skip[gl] = 1;
  }
}

void layout_workspace(Plan& P) {
  // workspace: every materialised stage that is not a liveout
  const Pipeline& pp = *P.pipe;
  size_t off = 0;
  P.ws.clear();
  for (auto& g : P.sch.groups)
    for (auto& s : g.gs) {
      if (!s.materialize) continue;
      if (std::find(pp.liveouts.begin(), pp.liveouts.end(), s.id) != pp.liveouts.end()) continue;
      if (P.ilv.count(s.id)) continue;   // stored into its interleaved liveout
      const Ext3& e = P.A.stage_ext[s.id];
      WsTensor t;
      t.stage = s.id;
      t.row_pitch = round_up64(e.e[2] * dtype_size(pp.stages[s.id].dtype), 128);
      t.rows = e.e[1];
      t.planes = e.e[0];
      t.plane_pitch = t.row_pitch * t.rows;
      t.offset = off;
      off += (size_t)round_up64(t.plane_pitch * t.planes, 256);
      P.ws.push_back(t);
    }
  P.ws_bytes = off;
}

std::unique_ptr<Plan> plan_create(std::shared_ptr<Pipeline> p, const std::vector<int64_t>& params, int device,
                                  const pmg_gpu_spec* spec, const pmg_weights* w, const pmg_sched_opts* opts) {
  Drv& D = drv();
  if (!D.ok) throw Error(-6, D.err);
  if (opts && opts->tune > 0 && !opts->group_of_stage) {
    // measured selection: the model's plan, then every neighbour merge of its groups; keep the fastest
    pmg_sched_opts o0 = *opts;
    o0.tune = 0;
    std::unique_ptr<Plan> best = plan_create(p, params, device, spec, w, &o0);
    // greedy: each round times every neighbour merge of the current best schedule and moves to the fastest,
    // until no merge helps (at most 4 rounds)
    CtxGuard g(best->ctx);
    double tb = time_plan_us(*best, opts->bands);
    std::ostringstream js;
    js << "{\"candidates\":[{\"round\":0,\"groups\":" << best->sch.groups.size() << ",\"us\":" << tb << "}";
    int chosen = 0, pos = 0;
    std::vector<std::vector<int>> keep;   // group_of_stage arrays must outlive the plans built from them
    for (int round = 1; round <= 4; ++round) {
      std::vector<std::vector<int>> cands = merge_candidates(best->A, best->sch);
      // plans of many groups (the pyramids): only merges touching the 4 slowest groups of the current plan, timed
      // one group at a time (profile_groups_us), keep plan creation to a few dozen candidates
      if (best->sch.groups.size() > 6) {
        std::vector<double> gus = profile_groups_us(*best);
        std::vector<int> order(gus.size());
        for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
        std::sort(order.begin(), order.end(), [&](int a, int b) { return gus[a] > gus[b]; });
        std::set<int> slow(order.begin(), order.begin() + std::min<size_t>(4, order.size()));
        std::vector<std::vector<int>> kept{cands[0]};
        for (size_t c = 1; c < cands.size(); ++c) {
          // candidate c merges groups g and g+1 of the current plan: find g from the array
          int g = -1;   // the merged pair (g, g+1): the smallest new label among the relabelled stages
          for (size_t st = 0; st < cands[c].size(); ++st)
            if (cands[c][st] != cands[0][st] && (g < 0 || cands[c][st] < g)) g = cands[c][st];
          if (g < 0 || slow.count(g) || slow.count(g + 1)) kept.push_back(cands[c]);
        }
        cands.swap(kept);
      }
      std::unique_ptr<Plan> rbest;
      double rt = tb;
      for (size_t c = 1; c < cands.size(); ++c) {
        keep.push_back(cands[c]);
        pmg_sched_opts oc = o0;
        oc.group_of_stage = keep.back().data();
        std::unique_ptr<Plan> Q;
        try {
          Q = plan_create(p, params, device, spec, w, &oc);
        } catch (const Error&) {
          continue;   // a merge the geometry cannot build (e.g. a non-constant dependence)
        }
        double t = time_plan_us(*Q, opts->bands);
        js << ",{\"round\":" << round << ",\"groups\":" << Q->sch.groups.size() << ",\"us\":" << t << "}";
        ++pos;
        if (t < rt) { rt = t; rbest = std::move(Q); chosen = pos; }
      }
      if (!rbest) break;
      tb = rt;
      best = std::move(rbest);
    }
    // single-group plans: the model's tile choice is also checked against a small grid of 128-column warp
    // tiles (V x TX in {1x4, 2x2, 4x1}) and tile heights (unsharp 2048^2: the model picks within 6 % of the
    // best measured configuration, profiles/unsharp_grid_r01n.txt)
    const char* grid_env = getenv("PMG_TUNE_GRID");   // "0": merges only (tests keep plan creation short)
    if (best->sch.groups.size() == 1 && !(grid_env && grid_env[0] == '0')) {
      std::vector<int> one(best->A.p->stages.size(), 0);
      const int vx[3][2] = {{1, 4}, {2, 2}, {4, 1}};
      std::unique_ptr<Plan> cbest;
      double ct = tb;
      // (plus a 6-deep TMA ring for 4-column lanes, with the tile height rounded down so that 6 divides the steps of
      // a tile and the ring slots resolve at compile time: Harris in reassociation mode issues fewer instructions
      // per row and waits on the ring at 4 rows in flight, profiles/harris_sweep_r02c.txt)
      const int t_first = best->sch.groups[0].t_first;
      for (auto& q : vx)
        for (int th0 : {16, 24, 32, 48, 64, 96, 100, 112, 128})
          for (int pf : {4, 6}) {
          if (pf != 4 && (q[0] != 4 || th0 < 48)) continue;
          const int th = pf == 4 ? th0 : th0 - ((th0 - t_first) % pf);   // steps TH - t_first: a multiple of pf
          pmg_sched_opts oc = o0;
          oc.group_of_stage = one.data();
          oc.vec = q[0];
          oc.chunks = q[1];
          oc.rows = th;
          oc.prefetch = pf;
          std::unique_ptr<Plan> Q;
          try {
            Q = plan_create(p, params, device, spec, w, &oc);
          } catch (const Error&) {
            continue;
          }
          double t = time_plan_us(*Q, opts->bands);
          js << ",{\"round\":\"config\",\"V\":" << q[0] << ",\"TX\":" << q[1] << ",\"TH\":" << th << ",\"PREF\":" << pf
             << ",\"us\":" << t << "}";
          ++pos;
          if (t < ct) { ct = t; cbest = std::move(Q); chosen = pos; }
        }
      if (cbest) { tb = ct; best = std::move(cbest); }
    }
    // border-tile rows (TH_b) on the final grouping: border tiles are latency-bound walks of the general body, and
    // short ones suit small pyramid levels and the camera's quad grids (PMG_BORDER_TH sweep)
    if (!(grid_env && grid_env[0] == '0') && opts->border_rows <= 0) {
      keep.push_back(best->sch.group_of_stage);
      const std::vector<int>& gos = keep.back();
      const bool one = best->sch.groups.size() == 1;
      const KConfig bk = best->sch.groups[0].cfg;
      std::unique_ptr<Plan> bbest;
      double bt = tb;
      for (int br : {2, 4}) {
        pmg_sched_opts oc = o0;
        oc.group_of_stage = gos.data();
        oc.border_rows = br;
        if (one) { oc.vec = bk.V; oc.chunks = bk.TX; oc.rows = bk.TH; oc.prefetch = bk.PREF; }
        std::unique_ptr<Plan> Q;
        try {
          Q = plan_create(p, params, device, spec, w, &oc);
        } catch (const Error&) {
          continue;
        }
        double t = time_plan_us(*Q, opts->bands);
        js << ",{\"round\":\"border_rows\",\"TH_b\":" << br << ",\"us\":" << t << "}";
        ++pos;
        if (t < bt) { bt = t; bbest = std::move(Q); chosen = pos; }
      }
      if (bbest) { tb = bt; best = std::move(bbest); }
    }
    js << "],\"chosen\":" << chosen << "}";
    best->tune_json = js.str();
    return best;
  }
  auto P = std::make_unique<Plan>();
  std::shared_ptr<Pipeline> written = p;
  if (opts && opts->reassoc) p = factor_stencils(p, params, &P->factored);
  if (!(opts && opts->no_inline)) p = phase_split(inline_expanding(p, params, &P->inlined), params, &P->split);
  P->pipe = p;
  P->A = analyze(*p, params);
  P->device = device;
  CUdevice dev;
  check(D.DeviceGet(&dev, device), "cuDeviceGet");
  check(D.DevicePrimaryCtxRetain(&P->ctx, dev), "cuDevicePrimaryCtxRetain");
  CtxGuard guard(P->ctx);
  if (spec) P->spec = *spec;
  else {
    gpu_preset("b200", &P->spec);
    int v;
    if (D.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev) == CUDA_SUCCESS) P->spec.nsms = v;
    if (D.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_MULTIPROCESSOR, dev) == CUDA_SUCCESS) P->spec.shmem_per_sm = v;
    if (D.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_BLOCK_OPTIN, dev) == CUDA_SUCCESS) P->spec.max_shmem_per_tb = v;
    if (D.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_L2_CACHE_SIZE, dev) == CUDA_SUCCESS) P->spec.l2_bytes = v;
  }
  if (w) P->weights = *w;
  else weights_preset("b200", &P->weights);
  pmg_sched_opts o;
  if (opts) o = *opts;
  else {
    std::memset(&o, 0, sizeof o);
    o.vec = o.chunks = o.rows = o.warps = o.prefetch = o.tx_size = -1;
    o.smem_chunks = -1;
    o.fuse = 1;
    o.probe = 1;
  }
  std::vector<double> tpi = map_time_per_iter(*written, *P->pipe, o.time_per_iter);
  if (o.time_per_iter) o.time_per_iter = tpi.data();
  RegProbe probe = make_probe(P->A);
  P->sch = schedule(P->A, P->spec, P->weights, o, o.probe ? &probe : nullptr);
  detect_interleave(*P);
  const Pipeline& pp = *p;
  P->nimages = (int)pp.images.size();
  P->ntables = (int)pp.tables.size();
  P->nout = (int)pp.liveouts.size();
  layout_workspace(*P);
  // compile + load
  std::ostringstream js;
  js << "{\"inlined\":[";
  for (size_t i = 0; i < P->inlined.size(); ++i) js << (i ? "," : "") << "\"" << P->inlined[i] << "\"";
  js << "],\"split\":[";
  for (size_t i = 0; i < P->split.size(); ++i) js << (i ? "," : "") << "\"" << P->split[i] << "\"";
  js << "],\"factored\":[";
  for (size_t i = 0; i < P->factored.size(); ++i) js << (i ? "," : "") << "\"" << P->factored[i] << "\"";
  js << "],\"schedule\":" << P->sch.json << ",\"kernels\":[";
  for (size_t gi = 0; gi < P->sch.groups.size(); ++gi) {
    Group& g = P->sch.groups[gi];
    g.source = emit_group(P->A, g);
    Kernel k;
    k.bin = jit_compile(g.name, g.source);
    check(D.ModuleLoadData(&k.mod, k.bin.cubin.data()), "cuModuleLoadData");
    check(D.ModuleGetFunction(&k.fn, k.mod, g.name.c_str()), "cuModuleGetFunction");
    check(D.ModuleGetFunction(&k.fn_b, k.mod, (g.name + "_b").c_str()), "cuModuleGetFunction");
    if (g.xedge) check(D.ModuleGetFunction(&k.fn_e, k.mod, (g.name + "_e").c_str()), "cuModuleGetFunction");
    for (CUfunction f : {k.fn, k.fn_b, k.fn_e})
      if (f && g.block_smem > 48 * 1024)
        check(D.FuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, g.block_smem), "cuFuncSetAttribute");
    check(D.OccupancyMaxActiveBlocksPerMultiprocessor(&k.blocks_per_sm, k.fn, g.cfg.NW * 32, g.block_smem), "occupancy");
    check(D.OccupancyMaxActiveBlocksPerMultiprocessor(&k.blocks_per_sm_b, k.fn_b, g.cfg.NW * 32, g.block_smem), "occupancy");
    if (k.fn_e)
      check(D.OccupancyMaxActiveBlocksPerMultiprocessor(&k.blocks_per_sm_e, k.fn_e, g.cfg.NW * 32, g.block_smem), "occupancy");
    if (k.blocks_per_sm < 1 || k.blocks_per_sm_b < 1 || (k.fn_e && k.blocks_per_sm_e < 1)) throw Error(-6, "kernel " + g.name + " cannot be resident on an SM");
    const FnStats& fb = k.bin.fns[g.name + "_b"];
    js << (gi ? "," : "") << "{\"name\":\"" << g.name << "\",\"regs\":" << k.bin.regs << ",\"spill_stores\":"
       << k.bin.spill_stores << ",\"spill_loads\":" << k.bin.spill_loads << ",\"block_smem\":" << g.block_smem
       << ",\"blocks_per_sm\":" << k.blocks_per_sm << ",\"border_regs\":" << fb.regs << ",\"border_spill_stores\":"
       << fb.spill_stores << ",\"border_blocks_per_sm\":" << k.blocks_per_sm_b << ",\"edge_regs\":" << (k.fn_e ? k.bin.fns[g.name + "_e"].regs : 0)
       << ",\"edge_blocks_per_sm\":" << k.blocks_per_sm_e
       << ",\"cached\":"
       << (k.bin.from_cache ? "true" : "false") << ",\"compile_s\":" << k.bin.compile_s << "}";
    P->kernels.push_back(std::move(k));
  }
  js << "],\"workspace_bytes\":" << P->ws_bytes << "}";
  P->json = js.str();
  check(D.StreamCreate(&P->side, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
  check(D.EventCreate(&P->ev_fork, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
  check(D.EventCreate(&P->ev_join, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
  // group DAG lanes: list-schedule the groups (topological order, weight = points of the group's domain) on up
  // to 4 lanes; a group continues the lane of a producer when that lane is free at its ready time
  {
    const int ng = (int)P->sch.groups.size();
    const Pipeline& pp = *P->pipe;
    P->deps.assign(ng, {});
    std::vector<int> gof(pp.stages.size(), -1);
    for (int gi = 0; gi < ng; ++gi)
      for (int s : P->sch.groups[gi].stages) gof[s] = gi;
    for (int gi = 0; gi < ng; ++gi)
      for (int s : P->sch.groups[gi].stages)
        for (int q : pp.producers[s]) {
          int gq = gof[q];
          if (gq != gi && gq >= 0 && std::find(P->deps[gi].begin(), P->deps[gi].end(), gq) == P->deps[gi].end())
            P->deps[gi].push_back(gq);
        }
    const int L = 4;
    std::vector<double> lane_free(L, 0.0), fin(ng, 0.0);
    P->lane_of.assign(ng, 0);
    int used = 1;
    for (int gi = 0; gi < ng; ++gi) {
      const Group& g = P->sch.groups[gi];
      double w = (double)g.npl * (double)g.ext.e[1] * (double)g.ext.e[2] + 1e4;   // + launch latency
      double ready = 0;
      for (int d : P->deps[gi]) ready = std::max(ready, fin[d]);
      int best = 0;
      double bs = 1e300;
      for (int l = 0; l < L; ++l) {
        double st = std::max(ready, lane_free[l]);
        bool cont = false;
        for (int d : P->deps[gi]) cont |= P->lane_of[d] == l;
        st -= cont ? 1e-6 : 0;   // prefer continuing a producer's lane on ties
        if (st < bs) { bs = st; best = l; }
      }
      P->lane_of[gi] = best;
      fin[gi] = std::max(ready, lane_free[best]) + w;
      lane_free[best] = fin[gi];
      used = std::max(used, best + 1);
    }
    P->nlanes = used;
    P->lane_stream.assign(used, nullptr);
    P->lane_side.assign(used, nullptr);
    P->lane_side2.assign(used, nullptr);
    P->lane_fork.assign(used, nullptr);
    P->lane_join.assign(used, nullptr);
    P->lane_join2.assign(used, nullptr);
    P->lane_side[0] = P->side;
    P->lane_fork[0] = P->ev_fork;
    P->lane_join[0] = P->ev_join;
    for (int l = 0; l < used; ++l) {
      check(D.StreamCreate(&P->lane_side2[l], CU_STREAM_NON_BLOCKING), "cuStreamCreate");
      check(D.EventCreate(&P->lane_join2[l], CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    }
    for (int l = 1; l < used; ++l) {
      check(D.StreamCreate(&P->lane_stream[l], CU_STREAM_NON_BLOCKING), "cuStreamCreate");
      check(D.StreamCreate(&P->lane_side[l], CU_STREAM_NON_BLOCKING), "cuStreamCreate");
      check(D.EventCreate(&P->lane_fork[l], CU_EVENT_DISABLE_TIMING), "cuEventCreate");
      check(D.EventCreate(&P->lane_join[l], CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    }
    if (used > 1) {
      P->ev_group.assign(ng, nullptr);
      for (int gi = 0; gi < ng; ++gi) check(D.EventCreate(&P->ev_group[gi], CU_EVENT_DISABLE_TIMING), "cuEventCreate");
      check(D.EventCreate(&P->ev_run, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    }
  }
  return P;
}

// every plan owns its CUDA resources: destroying a Plan (also a losing measured-selection candidate, or one
// whose creation threw half way) releases them exactly once
Plan::~Plan() {
  try { plan_destroy(this); } catch (...) {}
}

void plan_destroy(Plan* P) {
  if (!P || P->released) return;
  P->released = true;
  if (drv().ok && P->ctx) {
    CtxGuard g(P->ctx);
    for (auto& k : P->kernels)
      if (k.mod) drv().ModuleUnload(k.mod);
    if (P->side) drv().StreamDestroy(P->side);
    if (P->ev_fork) drv().EventDestroy(P->ev_fork);
    if (P->ev_join) drv().EventDestroy(P->ev_join);
    if (P->h2d) drv().StreamDestroy(P->h2d);
    if (P->d2h) drv().StreamDestroy(P->d2h);
    for (CUevent e : P->ev_in) drv().EventDestroy(e);
    for (CUevent e : P->ev_done) drv().EventDestroy(e);
    if (P->ev_start) drv().EventDestroy(P->ev_start);
    for (size_t l = 1; l < P->lane_stream.size(); ++l) drv().StreamDestroy(P->lane_stream[l]);
    for (size_t l = 1; l < P->lane_side.size(); ++l) drv().StreamDestroy(P->lane_side[l]);
    for (CUstream st : P->lane_side2)
      if (st) drv().StreamDestroy(st);
    for (CUevent e : P->lane_join2)
      if (e) drv().EventDestroy(e);
    for (size_t l = 1; l < P->lane_fork.size(); ++l) drv().EventDestroy(P->lane_fork[l]);
    for (size_t l = 1; l < P->lane_join.size(); ++l) drv().EventDestroy(P->lane_join[l]);
    for (CUevent e : P->ev_group) drv().EventDestroy(e);
    if (P->ev_run) drv().EventDestroy(P->ev_run);
    if (P->ev_end) drv().EventDestroy(P->ev_end);
    CUdevice dev;
    if (drv().DeviceGet(&dev, P->device) == CUDA_SUCCESS) drv().DevicePrimaryCtxRelease(dev);
  }
}

// ---------------------------------------------------------------------------------- band geometry
// rows needed of every stage / image for liveout rows [r0, r1) (cumulative halo, clipped)
struct Need { std::vector<RowIv> stage, image, group; };

static Need rows_for(const Plan& P, int64_t r0, int64_t r1) {
  const Pipeline& p = *P.pipe;
  const Analysis& A = P.A;
  Need n;
  n.stage.assign(p.stages.size(), RowIv{0, 0});
  n.image.assign(p.images.size(), RowIv{0, 0});
  auto hull = [](RowIv& a, RowIv b) {
    if (b.hi <= b.lo) return;
    if (a.hi <= a.lo) a = b;
    else { a.lo = std::min(a.lo, b.lo); a.hi = std::max(a.hi, b.hi); }
  };
  for (int lo : p.liveouts) hull(n.stage[lo], RowIv{r0, r1});
  for (int ti = (int)p.topo.size() - 1; ti >= 0; --ti) {
    int c = p.topo[ti];
    if (n.stage[c].hi <= n.stage[c].lo) continue;
    for (int ri : A.reads_of[c]) {
      const ReadSite& r = A.reads[ri];
      int64_t rows = r.src_is_stage ? A.stage_ext[r.src].e[1] : A.image_ext[r.src].e[1];
      RowIv need = rows_needed(A, r, n.stage[c], rows);
      if (r.src_is_stage) hull(n.stage[r.src], need);
      else hull(n.image[r.src], need);
    }
  }
  // group granularity: a group's kernel produces the hull of its materialised stages' rows (its in-group
  // stages' halo rows are produced inside the tiles); every materialised stage of the group gets that range
  for (auto& g : P.sch.groups) {
    RowIv h{0, 0};
    for (auto& s : g.gs)
      if (s.materialize) hull(h, n.stage[s.id]);
    for (auto& s : g.gs)
      if (s.materialize) n.stage[s.id] = h;
    n.group.push_back(h);
  }
  return n;
}

BandRows band_rows(const Plan& P, int band, int nbands) {
  const Pipeline& p = *P.pipe;
  int64_t H = P.A.stage_ext[p.liveouts[0]].e[1];
  for (int lo : p.liveouts)
    if (P.A.stage_ext[lo].e[1] != H) throw Error(-3, "band mode needs liveouts of equal row extent");
  BandRows b;
  b.out_r0 = band * H / nbands;
  b.out_r1 = (band + 1) * H / nbands;
  Need n = rows_for(P, b.out_r0, b.out_r1);
  b.in_r0 = INT64_MAX;
  b.in_r1 = INT64_MIN;
  for (size_t i = 0; i < p.images.size(); ++i) {
    if (n.image[i].hi <= n.image[i].lo) continue;
    b.in_r0 = std::min(b.in_r0, n.image[i].lo);
    b.in_r1 = std::max(b.in_r1, n.image[i].hi);
  }
  if (b.in_r0 == INT64_MAX) { b.in_r0 = 0; b.in_r1 = 0; }
  return b;
}

BandXchg band_xchg(const Plan& P, int band, int nbands) {
  const Pipeline& p = *P.pipe;
  const Analysis& A = P.A;
  auto hull = [](RowIv& a, RowIv b) {
    if (b.hi <= b.lo) return;
    if (a.hi <= a.lo) a = b;
    else { a.lo = std::min(a.lo, b.lo); a.hi = std::max(a.hi, b.hi); }
  };
  const size_t ng = P.sch.groups.size();
  std::vector<int> group_of(p.stages.size(), -1);
  for (size_t gi = 0; gi < ng; ++gi)
    for (int s : P.sch.groups[gi].stages) group_of[s] = (int)gi;
  BandXchg X;
  X.own.resize(ng);
  X.buf.assign(p.stages.size(), RowIv{0, 0});
  X.need.assign(p.stages.size(), RowIv{0, 0});
  BandRows br = band_rows(P, band, nbands);
  X.out = RowIv{br.out_r0, br.out_r1};
  for (size_t gi = 0; gi < ng; ++gi) {
    const Group& g = P.sch.groups[gi];
    const int64_t Hg = g.ext.e[1];
    X.own[gi] = RowIv{band * Hg / nbands, (band + 1) * Hg / nbands};
    // rows of the group's own stages: its materialised stages' own rows, then in-group halos (computed inside
    // the tiles) back-propagated in topological order; reads of other groups' stages and of images are needs
    std::vector<RowIv> rows(p.stages.size(), RowIv{0, 0});
    for (auto& s : g.gs)
      if (s.materialize) rows[s.id] = X.own[gi];
    for (auto it = g.stages.rbegin(); it != g.stages.rend(); ++it) {
      const int c = *it;
      if (rows[c].hi <= rows[c].lo) continue;
      for (int ri : A.reads_of[c]) {
        const ReadSite& r = A.reads[ri];
        const int64_t srows = r.src_is_stage ? A.stage_ext[r.src].e[1] : A.image_ext[r.src].e[1];
        RowIv nd = rows_needed(A, r, rows[c], srows);
        if (!r.src_is_stage) hull(X.in, nd);
        else if (group_of[r.src] == (int)gi) hull(rows[r.src], nd);
        else hull(X.need[r.src], nd);
      }
    }
  }
  for (size_t gi = 0; gi < ng; ++gi)
    for (auto& s : P.sch.groups[gi].gs)
      if (s.materialize) {
        X.buf[s.id] = X.own[gi];
        hull(X.buf[s.id], X.need[s.id]);
      }
  return X;
}

// ------------------------------------------------------------------------------------------ launch
#pragma pack(push, 1)
struct HostTensor { uint64_t ptr; int64_t rp, pp, fs; int32_t row_base, nrows, H, W, pad0, pad1; };
#pragma pack(pop)
static_assert(sizeof(HostTensor) == 56, "PmgTensor mirror");

// launch geometry of group gi over rows [gy0, gy1): interior rectangle, x-edge and border tile counts
struct GroupGeom {
  int64_t n_int = 0, n_edge = 0, n_bdr = 0, nty_i = 0, nty_b = 0, tyA_b = 0, tyB_b = 0, txA = 0, txB = 0, bxA = 0,
          bxB = 0, gy0_i = 0;
  int32_t ylast = INT32_MAX;
  bool xe = false;
};

static GroupGeom group_geom(const Plan& P, size_t gi, int64_t gy0, int64_t gy1, int nframes) {
  const Analysis& A = P.A;
  const Group& g = P.sch.groups[gi];
  const Kernel& K = P.kernels[gi];
  const int64_t Hg = g.ext.e[1], Wg = g.ext.e[2];
  GroupGeom G;
  int64_t ntiles = (int64_t)nframes * g.npl * ((gy1 - gy0 + g.cfg.TH - 1) / g.cfg.TH) * g.ntx;
  if (ntiles > INT32_MAX) throw Error(-3, "too many tiles");
  // interior rectangle: tiles whose whole wavefront stays inside the image / the computed rows
  // (matches the emitted bodies: no clamping, no x fix-up, no row checks needed there)
  int xlm = 0, xrm = 0, himax = 0;
  for (auto& st : g.streams) {
    if (st.sx == 0) { xlm = std::max(xlm, st.xl); xrm = std::max(xrm, st.xr); }
    himax = std::max(himax, st.hi);
  }
  for (auto& st : g.gs) himax = std::max(himax, st.hi);
  auto cdiv = [](int64_t a, int64_t b) { return a >= 0 ? (a + b - 1) / b : -((-a) / b); };
  auto fdiv = [](int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
  int64_t txA = std::max<int64_t>(0, cdiv(g.PL + xlm, g.OW));
  int64_t txB = std::min<int64_t>(g.ntx, fdiv(Wg - g.CW - xrm + g.PL, g.OW) + 1);
  // scaled streams (emit.cpp xb_scaled): the tile's producer row [origin - xl, + row_elems) inside [0, Wp)
  auto scaled_in = [&](int64_t tx) {
    const int64_t cx = tx * g.OW - g.PL;
    for (auto& st : g.streams) {
      if (st.sx == 0) continue;
      const Ext3& se = st.src_is_stage ? A.stage_ext[st.src] : A.image_ext[st.src];
      const int64_t o0 = (st.sx == 1 ? 2 * cx : (cx >= 0 ? cx / 2 : -((-cx + 1) / 2))) - st.xl;
      if (o0 < 0 || o0 + st.row_elems > se.e[2]) return false;
    }
    return true;
  };
  while (txA < txB && !scaled_in(txA)) ++txA;
  while (txB > txA && !scaled_in(txB - 1)) --txB;
  // interior tile rows: the tiling starts `top` rows below gy0 (a multiple of the border tile height, enough
  // for the rows the wavefront reads above a tile); its last tile row is shifted up to end at `ylim` (the last
  // row whose wavefront stays inside the image and the computed rows), overlapping the row before it -- both
  // compute the same values.  The border kernel takes the rows above the tiling and the TH_b-row tiles from
  // the one containing ylim down, so only those rows go through the general body.
  const int THb = g.TH_b > 0 ? g.TH_b : g.cfg.TH;
  const int64_t top = cdiv(std::max<int64_t>(0, -(int64_t)g.t_first - gy0), THb) * THb;
  const int64_t ylim = std::min<int64_t>(Hg - himax, gy1);
  G.gy0_i = gy0 + top;
  int64_t nty_i = ylim - G.gy0_i >= g.cfg.TH ? cdiv(ylim - G.gy0_i, g.cfg.TH) : 0;
  if (txB <= txA || nty_i <= 0) { txA = txB = 0; nty_i = 0; }
  G.nty_i = nty_i;
  G.txA = txA;
  G.txB = txB;
  G.n_int = (int64_t)nframes * g.npl * nty_i * (txB - txA);
  // x-edge kernel (Group::xedge): the tile columns outside [txA, txB) of the interior tile rows
  G.xe = K.fn_e && nty_i > 0;
  G.n_edge = G.xe ? (int64_t)nframes * g.npl * nty_i * (g.ntx - (txB - txA)) : 0;
  G.bxA = G.xe ? 0 : txA;   // the border kernel's excluded columns
  G.bxB = G.xe ? g.ntx : txB;
  G.nty_b = (gy1 - gy0 + THb - 1) / THb;
  G.tyA_b = nty_i > 0 ? top / THb : 0;
  G.tyB_b = nty_i > 0 ? (ylim - gy0) / THb : 0;
  G.n_bdr = (int64_t)nframes * g.npl * (G.nty_b * g.ntx - (G.tyB_b - G.tyA_b) * (G.bxB - G.bxA));
  G.ylast = nty_i > 0 ? (int32_t)(ylim - g.cfg.TH) : INT32_MAX;
  return G;
}

// PMG_XMERGE: "1" merged interior + x-edge launches always, "0" never; default: row-band runs only
static bool xmerge_on(bool banded) {
  static const int mode = [] { const char* e = getenv("PMG_XMERGE"); return e ? (e[0] == '1' ? 1 : 0) : -1; }();
  return mode < 0 ? banded : mode == 1;
}

static bool pdl_on() {   // PMG_PDL=0 launches without programmatic dependent launch (experiments)
  static const bool on = [] { const char* e = getenv("PMG_PDL"); return !(e && e[0] == '0'); }();
  return on;
}

void plan_run(Plan& P, const pmg_buf* in, int nin, const pmg_buf* out, int nout, void* ws, CUstream s, int band,
              int nbands, int nframes, const int64_t* in_fs, const int64_t* out_fs, const int* groups) {
  std::lock_guard<std::recursive_mutex> lock(P.run_mu);
  Drv& D = drv();
  if (!D.ok) throw Error(-6, D.err);
  const Pipeline& p = *P.pipe;
  const Analysis& A = P.A;
  if (nin != P.nimages + P.ntables) throw Error(-9, "expected " + std::to_string(P.nimages + P.ntables) + " inputs");
  if (nout != P.nout) throw Error(-9, "expected " + std::to_string(P.nout) + " outputs");
  CUcontext cur = nullptr;
  D.CtxGetCurrent(&cur);
  CUdevice cd;
  if (!cur || D.CtxGetDevice(&cd) != CUDA_SUCCESS || (int)cd != P.device)
    throw Error(-9, "the plan's device must be current on the calling thread");
  P.last_launches = 0;
  if (P.ws_bytes && !ws) throw Error(-9, "workspace required");
  auto aligned = [](const pmg_buf& b) {
    return ((uintptr_t)b.ptr % 16 == 0) && (b.row_pitch_bytes % 16 == 0) && (b.plane_pitch_bytes % 16 == 0);
  };
  for (int i = 0; i < P.nimages; ++i)
    if (!in[i].ptr || !aligned(in[i])) throw Error(-9, "input " + p.images[i].name + " is NULL or not 16-byte aligned");
  for (int i = 0; i < nout; ++i)
    if (!out[i].ptr || !aligned(out[i])) throw Error(-9, "output " + p.stages[p.liveouts[i]].name + " is NULL or not 16-byte aligned");
  if ((uintptr_t)ws % 16) throw Error(-9, "workspace not 16-byte aligned");
  int64_t r0 = 0, r1 = 0;
  Need need;
  bool banded = band >= 0;
  if (banded) {
    BandRows br = band_rows(P, band, nbands);
    r0 = br.out_r0;
    r1 = br.out_r1;
    if (r1 <= r0) return;
    need = rows_for(P, r0, r1);
    for (auto& g : P.sch.groups)
      for (auto& st : g.gs)
        if (std::find(p.liveouts.begin(), p.liveouts.end(), st.id) != p.liveouts.end() && !p.consumers[st.id].empty())
          throw Error(-3, "band mode: a liveout that is also consumed by the pipeline is not supported");
  }
  // halo-exchange band mode: own rows per group, workspace slots holding own + received rows
  const bool xmode = banded && groups != nullptr;
  BandXchg X;
  if (xmode) {
    if (!P.ilv.empty()) throw Error(-3, "halo-exchange bands: not supported for a plan with a fused interleave (PMG_ILV=0)");
    X = band_xchg(P, band, nbands);
    for (size_t si = 0; si < p.stages.size(); ++si) need.stage[si] = X.buf[si];
    for (size_t gi = 0; gi < P.sch.groups.size(); ++gi) need.group[gi] = X.own[gi];
  }
  int64_t in_row_base = xmode ? X.in.lo : banded ? band_rows(P, band, nbands).in_r0 : 0;
  const int64_t in_row_end = xmode ? X.in.hi : banded ? band_rows(P, band, nbands).in_r1 : 0;
  const bool lanes = P.nlanes > 1;
  std::vector<int> last_on_lane(P.nlanes, -1);
  if (lanes) {
    check(D.EventRecord(P.ev_run, s), "cuEventRecord");
    for (int l = 1; l < P.nlanes; ++l) check(D.StreamWaitEvent(P.lane_stream[l], P.ev_run, 0), "cuStreamWaitEvent");
  }
  for (size_t gi = 0; gi < P.sch.groups.size(); ++gi) {
    if (P.only_group >= 0 && (int)gi != P.only_group) continue;
    if (xmode && ((int)gi < groups[0] || (int)gi >= groups[1])) continue;
    const Group& g = P.sch.groups[gi];
    Kernel& K = P.kernels[gi];
    const int lane = lanes ? P.lane_of[gi] : 0;
    const CUstream gs = lane == 0 ? s : P.lane_stream[lane];
    const CUstream gside = P.lane_side[lane], gside2 = P.lane_side2[lane];
    const CUevent gfork = P.lane_fork[lane], gjoin = P.lane_join[lane], gjoin2 = P.lane_join2[lane];
    if (lanes) {
      // (a group timed alone, profile_groups_us, reads what earlier runs left: no producer events to wait on --
      // they were not recorded in this run, and inside a graph capture they could not be waited on)
      if (P.only_group < 0)
        for (int d : P.deps[gi])
          if (P.lane_of[d] != lane) check(D.StreamWaitEvent(gs, P.ev_group[d], 0), "cuStreamWaitEvent");
      last_on_lane[lane] = (int)gi;
    }
    struct Done {   // every group records its completion event, also when it launches nothing in this run
      Drv& D; bool on; CUevent e; CUstream st;
      ~Done() { if (on) D.EventRecord(e, st); }
    } done{D, lanes, lanes ? P.ev_group[gi] : nullptr, gs};
    if (!P.ilv_skip.empty() && P.ilv_skip[gi]) continue;   // interleave fused into its phases' group
    const int NT = std::max<int>(1, (int)g.tensors.size()), NTAB = std::max(1, P.ntables),
              NP = std::max<int>(1, (int)p.params.size());
    size_t off_tab = sizeof(HostTensor) * (size_t)NT, off_tabn = off_tab + 8 * NTAB, off_prm = off_tabn + 4 * NTAB,
           off_int = off_prm + 4 * NP, size = (off_int + 64 + 7) / 8 * 8;
    std::vector<char> buf(size, 0);
    for (size_t ti = 0; ti < g.tensors.size(); ++ti) {
      auto [is_stage, id] = g.tensors[ti];
      HostTensor t{};
      if (!is_stage) {
        t.ptr = (uint64_t)(uintptr_t)in[id].ptr;
        t.rp = in[id].row_pitch_bytes;
        t.pp = in[id].plane_pitch_bytes;
        t.fs = in_fs ? in_fs[id] : 0;
        t.row_base = (int32_t)(banded ? in_row_base : 0);
        t.nrows = (int32_t)(banded ? in_row_end - in_row_base : A.image_ext[id].e[1]);
      } else {
        auto lit = std::find(p.liveouts.begin(), p.liveouts.end(), id);
        auto il = P.ilv.find(id);
        if (il != P.ilv.end()) {
          // a phase of an interleaved liveout: rows y of the phase are liveout rows 2y+py, columns 2x+px
          const Plan::Ilv& v = il->second;
          const pmg_buf& ob = out[v.out];
          const int64_t ob0 = banded ? r0 : 0, on = banded ? r1 - r0 : A.stage_ext[p.liveouts[v.out]].e[1];
          const int64_t q0 = (ob0 - v.py + 1) >> 1, q1 = (ob0 + on - v.py + 1) >> 1;   // ceil((r - py) / 2)
          const int esz = dtype_size(p.stages[id].dtype);
          t.ptr = (uint64_t)(uintptr_t)((const char*)ob.ptr + (int64_t)v.c * ob.plane_pitch_bytes +
                                        (2 * q0 + v.py - ob0) * ob.row_pitch_bytes + (int64_t)v.px * esz);
          t.rp = 2 * ob.row_pitch_bytes;
          t.pp = ob.plane_pitch_bytes;
          t.fs = out_fs ? out_fs[v.out] : 0;
          t.row_base = (int32_t)q0;
          t.nrows = (int32_t)std::max<int64_t>(0, q1 - q0);
        } else if (lit != p.liveouts.end()) {
          int oi = int(lit - p.liveouts.begin());
          t.ptr = (uint64_t)(uintptr_t)out[oi].ptr;
          t.rp = out[oi].row_pitch_bytes;
          t.pp = out[oi].plane_pitch_bytes;
          t.fs = out_fs ? out_fs[oi] : 0;
          t.row_base = (int32_t)(banded ? r0 : 0);
          t.nrows = (int32_t)(banded ? r1 - r0 : A.stage_ext[id].e[1]);
        } else {
          const WsTensor* w = nullptr;
          for (auto& x : P.ws)
            if (x.stage == id) w = &x;
          if (!w) throw Error(-2, "internal: no workspace for " + p.stages[id].name);
          t.ptr = (uint64_t)(uintptr_t)((char*)ws + w->offset);
          t.rp = w->row_pitch;
          t.pp = w->plane_pitch;
          t.fs = (int64_t)P.ws_bytes;
          t.row_base = (int32_t)(banded ? need.stage[id].lo : 0);
          t.nrows = (int32_t)(banded ? need.stage[id].hi - need.stage[id].lo : A.stage_ext[id].e[1]);
        }
      }
      const Ext3& te = is_stage ? A.stage_ext[id] : A.image_ext[id];
      t.H = (int32_t)te.e[1];
      t.W = (int32_t)te.e[2];
      std::memcpy(buf.data() + sizeof(HostTensor) * ti, &t, sizeof(HostTensor));
    }
    for (int ti = 0; ti < P.ntables; ++ti) {
      uint64_t ptr = (uint64_t)(uintptr_t)in[P.nimages + ti].ptr;
      int32_t n = (int32_t)A.table_len[ti];
      std::memcpy(buf.data() + off_tab + 8 * ti, &ptr, 8);
      std::memcpy(buf.data() + off_tabn + 4 * ti, &n, 4);
    }
    for (size_t pi = 0; pi < p.params.size(); ++pi) {
      int32_t v = (int32_t)A.params[pi];
      std::memcpy(buf.data() + off_prm + 4 * pi, &v, 4);
    }
    int32_t Hg = (int32_t)g.ext.e[1], Wg = (int32_t)g.ext.e[2];
    int32_t gy0 = 0, gy1 = Hg;
    if (banded) {
      RowIv h = need.group[gi];
      gy0 = (int32_t)h.lo;
      gy1 = (int32_t)h.hi;
    }
    if (gy1 <= gy0) continue;
    const GroupGeom G = group_geom(P, gi, gy0, gy1, nframes);
    const int64_t n_int = G.n_int, n_edge = G.n_edge, n_bdr = G.n_bdr, nty_i = G.nty_i, nty_b = G.nty_b;
    const int64_t tyA_b = G.tyA_b, tyB_b = G.tyB_b, txA = G.txA, txB = G.txB, bxA = G.bxA, bxB = G.bxB, gy0_i = G.gy0_i;
    const bool xe = G.xe;
    const int32_t ylast = G.ylast;
    void* args[] = {buf.data()};
    // diagnosis only (PMG_DIAG_SKIP = "b" / "e" / "i" letters): skip the border / x-edge / interior launches to
    // time the others alone (the output is then incomplete)
    static const char* skip = getenv("PMG_DIAG_SKIP");
    // merged interior + x-edge launch: the x-edge body (halo selects at the image's left / right edge) over every
    // column of the interior tile rows (its decoder walks all columns when txA = txB = 0) -- one launch and no
    // side stream for them; used for row bands, where a band's launches and their fork / join dominate
    const bool mrg = xe && n_int > 0 && xmerge_on(banded);
    auto launch = [&](CUfunction f, int bps, int64_t nt, CUstream st, const char* what) {
      const bool bd = f == K.fn_b;
      if (skip && std::strchr(skip, bd ? 'b' : f == K.fn_e ? 'e' : 'i')) return;
      int32_t ints[16] = {Hg, Wg, (int32_t)(bd ? gy0 : gy0_i), gy1, (int32_t)(bd ? nty_b : nty_i), (int32_t)g.ntx,
                          (int32_t)g.npl, (int32_t)nframes, (int32_t)nt, 0, (int32_t)(bd ? bxA : mrg ? 0 : txA),
                          (int32_t)(bd ? bxB : mrg ? 0 : txB),
                          (int32_t)(bd ? tyA_b : 0), (int32_t)(bd ? tyB_b : nty_i), bd ? INT32_MAX : ylast, 0};
      std::memcpy(buf.data() + off_int, ints, 64);
      int64_t grid = std::min<int64_t>((nt + g.cfg.NW - 1) / g.cfg.NW, (int64_t)bps * P.spec.nsms);
      // programmatic dependent launch (every emitted kernel starts with griddepcontrol.launch_dependents and
      // waits with griddepcontrol.wait before its first global access): a kernel that directly follows another
      // on the stream is launched while its predecessor's last warps still run, hiding the launch latency and
      // block scheduling of the chain of small kernels (pyramid levels)
      CUlaunchAttribute attr[1];
      attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
      attr[0].value.programmaticStreamSerializationAllowed = 1;
      CUlaunchConfig lc{};
      lc.gridDimX = (unsigned)grid;
      lc.gridDimY = lc.gridDimZ = 1;
      lc.blockDimX = g.cfg.NW * 32;
      lc.blockDimY = lc.blockDimZ = 1;
      lc.sharedMemBytes = (unsigned)g.block_smem;
      lc.hStream = st;
      lc.attrs = attr;
      lc.numAttrs = pdl_on() ? 1 : 0;
      CUresult r = D.LaunchKernelEx(&lc, f, args, nullptr);
      if (r != CUDA_SUCCESS) throw Error(-6, std::string("launch of ") + g.name + what + ": " + cu_err(r));
      ++P.last_launches;
    };
    if (mrg) {
      const int64_t n_all = (int64_t)nframes * g.npl * nty_i * g.ntx;
      if (n_bdr > 0) {
        check(D.EventRecord(gfork, gs), "cuEventRecord");
        check(D.StreamWaitEvent(gside, gfork, 0), "cuStreamWaitEvent");
      }
      launch(K.fn_e, K.blocks_per_sm_e, n_all, gs, "_e");
      if (n_bdr > 0) {
        launch(K.fn_b, K.blocks_per_sm_b, n_bdr, gside, "_b");
        check(D.EventRecord(gjoin, gside), "cuEventRecord");
        check(D.StreamWaitEvent(gs, gjoin, 0), "cuStreamWaitEvent");
      }
    } else if (n_int > 0 && (n_bdr > 0 || n_edge > 0)) {
      // border / x-edge tiles on the lane's side streams, forked from and joined back into the lane's stream.
      // With an x-edge kernel the border kernel holds only the top / bottom tile rows: the interior kernel is
      // launched first so that its single wave of warps is resident from the start, and the few edge and border
      // warps fill the slots it leaves; otherwise (many x-border tiles) the border kernel goes first
      check(D.EventRecord(gfork, gs), "cuEventRecord");
      check(D.StreamWaitEvent(gside, gfork, 0), "cuStreamWaitEvent");
      if (n_edge > 0) check(D.StreamWaitEvent(gside2, gfork, 0), "cuStreamWaitEvent");
      if (xe) {
        launch(K.fn, K.blocks_per_sm, n_int, gs, "");
        if (n_edge > 0) launch(K.fn_e, K.blocks_per_sm_e, n_edge, gside2, "_e");
        if (n_bdr > 0) launch(K.fn_b, K.blocks_per_sm_b, n_bdr, gside, "_b");
      } else {
        launch(K.fn_b, K.blocks_per_sm_b, n_bdr, gside, "_b");
        launch(K.fn, K.blocks_per_sm, n_int, gs, "");
      }
      check(D.EventRecord(gjoin, gside), "cuEventRecord");
      check(D.StreamWaitEvent(gs, gjoin, 0), "cuStreamWaitEvent");
      if (n_edge > 0) {
        check(D.EventRecord(gjoin2, gside2), "cuEventRecord");
        check(D.StreamWaitEvent(gs, gjoin2, 0), "cuStreamWaitEvent");
      }
    } else if (n_int > 0) {
      launch(K.fn, K.blocks_per_sm, n_int, gs, "");
    } else if (n_bdr > 0) {
      launch(K.fn_b, K.blocks_per_sm_b, n_bdr, gs, "_b");
    }

  }
  if (lanes)   // join every lane back into the caller's stream
    for (int l = 1; l < P.nlanes; ++l)
      if (last_on_lane[l] >= 0) check(D.StreamWaitEvent(s, P.ev_group[last_on_lane[l]], 0), "cuStreamWaitEvent");
}

}  // namespace pmg

namespace pmg {

// ------------------------------------------------------------------------------- host-buffer runs
// The end-to-end path of one pipeline run from host memory: the image is cut into `chunks` row bands
// (pmg_band_rows geometry); band b's new input rows go host->device on the copy-in stream, band b is
// computed on the caller's stream (pmg_run_band), and its output rows go device->host on the copy-out
// stream, so copies of one band overlap the copies and the compute of its neighbours.  Every input row is
// copied once (bands share their halo rows in the full-size device buffer).
void plan_run_host(Plan& P, const pmg_buf* hin, int nin, const pmg_buf* hout, int nout, const pmg_buf* din,
                   const pmg_buf* dout, void* ws, int chunks, CUstream s) {
  std::lock_guard<std::recursive_mutex> lock(P.run_mu);
  Drv& D = drv();
  if (!D.ok) throw Error(-6, D.err);
  const Pipeline& p = *P.pipe;
  const Analysis& A = P.A;
  if (nin != P.nimages + P.ntables) throw Error(-9, "expected " + std::to_string(P.nimages + P.ntables) + " inputs");
  if (nout != P.nout) throw Error(-9, "expected " + std::to_string(P.nout) + " outputs");
  const int64_t H = A.stage_ext[p.liveouts[0]].e[1];
  chunks = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)chunks, H, 64}));
  for (int i = 0; i < P.nimages; ++i)
    if (A.image_ext[i].e[1] != H) throw Error(-9, "host runs need input images with the liveouts' row extent");
  if (!P.h2d) {
    check(D.StreamCreate(&P.h2d, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
    check(D.StreamCreate(&P.d2h, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
    check(D.EventCreate(&P.ev_start, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    check(D.EventCreate(&P.ev_end, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
  }
  while ((int)P.ev_in.size() < chunks) {
    CUevent a, b;
    check(D.EventCreate(&a, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    check(D.EventCreate(&b, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    P.ev_in.push_back(a);
    P.ev_done.push_back(b);
  }
  auto copy2d = [&](const pmg_buf& src, bool src_host, const pmg_buf& dst, int64_t plane, int64_t r0, int64_t r1,
                    int64_t wbytes, CUstream st) {
    if (r1 <= r0) return;
    CUDA_MEMCPY2D c;
    std::memset(&c, 0, sizeof c);
    const char* sp = (const char*)src.ptr + plane * src.plane_pitch_bytes + r0 * src.row_pitch_bytes;
    char* dp = (char*)dst.ptr + plane * dst.plane_pitch_bytes + r0 * dst.row_pitch_bytes;
    if (src_host) {
      c.srcMemoryType = CU_MEMORYTYPE_HOST; c.srcHost = sp;
      c.dstMemoryType = CU_MEMORYTYPE_DEVICE; c.dstDevice = (CUdeviceptr)(uintptr_t)dp;
    } else {
      c.srcMemoryType = CU_MEMORYTYPE_DEVICE; c.srcDevice = (CUdeviceptr)(uintptr_t)sp;
      c.dstMemoryType = CU_MEMORYTYPE_HOST; c.dstHost = dp;
    }
    c.srcPitch = (size_t)src.row_pitch_bytes;
    c.dstPitch = (size_t)dst.row_pitch_bytes;
    c.WidthInBytes = (size_t)wbytes;
    c.Height = (size_t)(r1 - r0);
    check(D.Memcpy2DAsync(&c, st), "cuMemcpy2DAsync");
  };
  check(D.EventRecord(P.ev_start, s), "cuEventRecord");
  check(D.StreamWaitEvent(P.h2d, P.ev_start, 0), "cuStreamWaitEvent");
  check(D.StreamWaitEvent(P.d2h, P.ev_start, 0), "cuStreamWaitEvent");
  for (int t = 0; t < P.ntables; ++t) {
    const int ti = P.nimages + t;
    const size_t bytes = (size_t)A.table_len[t] * dtype_size(p.tables[t].dtype);
    check(D.MemcpyHtoDAsync((CUdeviceptr)(uintptr_t)din[ti].ptr, hin[ti].ptr, bytes, P.h2d), "cuMemcpyHtoDAsync");
  }
  std::vector<int64_t> copied(P.nimages, 0);
  std::vector<pmg_buf> bin(nin), bout(nout);
  for (int b = 0; b < chunks; ++b) {
    BandRows br = band_rows(P, b, chunks);
    for (int i = 0; i < P.nimages; ++i) {
      const Ext3& e = A.image_ext[i];
      const int64_t planes = e.has[0] ? e.e[0] : 1, wbytes = e.e[2] * dtype_size(p.images[i].dtype);
      const int64_t r0 = std::max(copied[i], br.in_r0);
      for (int64_t pl = 0; pl < planes; ++pl) copy2d(hin[i], true, din[i], pl, r0, br.in_r1, wbytes, P.h2d);
      copied[i] = std::max(copied[i], br.in_r1);
      bin[i] = din[i];
      bin[i].ptr = (char*)din[i].ptr + br.in_r0 * din[i].row_pitch_bytes;
    }
    for (int t = 0; t < P.ntables; ++t) bin[P.nimages + t] = din[P.nimages + t];
    for (int o = 0; o < nout; ++o) {
      bout[o] = dout[o];
      bout[o].ptr = (char*)dout[o].ptr + br.out_r0 * dout[o].row_pitch_bytes;
    }
    check(D.EventRecord(P.ev_in[b], P.h2d), "cuEventRecord");
    check(D.StreamWaitEvent(s, P.ev_in[b], 0), "cuStreamWaitEvent");
    plan_run(P, bin.data(), nin, bout.data(), nout, ws, s, chunks > 1 ? b : -1, chunks, 1, nullptr, nullptr);
    check(D.EventRecord(P.ev_done[b], s), "cuEventRecord");
    check(D.StreamWaitEvent(P.d2h, P.ev_done[b], 0), "cuStreamWaitEvent");
    for (int o = 0; o < nout; ++o) {
      const int id = p.liveouts[o];
      const Ext3& e = A.stage_ext[id];
      const int64_t planes = e.has[0] ? e.e[0] : 1, wbytes = e.e[2] * dtype_size(p.stages[id].dtype);
      for (int64_t pl = 0; pl < planes; ++pl) copy2d(dout[o], false, hout[o], pl, br.out_r0, br.out_r1, wbytes, P.d2h);
    }
  }
  check(D.EventRecord(P.ev_end, P.d2h), "cuEventRecord");
  check(D.StreamWaitEvent(s, P.ev_end, 0), "cuStreamWaitEvent");
}

}  // namespace pmg
