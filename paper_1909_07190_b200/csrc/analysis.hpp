// analysis.hpp — dependence / footprint analysis (§2.3), group geometry (§4 lines
// 558-623; §5 right hyperplanes lines 645-654) and the B200 schedule/kernel description consumed by the
// emitter and the selector.
#pragma once
#include <memory>
#include <array>
#include <string>
#include <vector>

#include "ir.hpp"

namespace pmg {

// normalised dims: 0 = c (plane), 1 = y, 2 = x.  A stage / image with nd dims occupies the last nd.
struct Ext3 {
  int64_t e[3] = {1, 1, 1};
  bool has[3] = {false, false, false};
  bool operator==(const Ext3& o) const { return e[0] == o.e[0] && e[1] == o.e[1] && e[2] == o.e[2] && has[0] == o.has[0]; }
};

// classification of one index expression of a read, per producer dim (normalised)
enum class Form { ABSENT, UNIT, DOWN2, UP2, CONST, GENERAL };

struct ReadSite {
  int consumer = -1;          // stage id
  bool src_is_stage = false;
  int src = -1;               // stage id or image id
  Form form[3] = {Form::ABSENT, Form::ABSENT, Form::ABSENT};
  int64_t off[3] = {0, 0, 0}; // UNIT: v+b -> b; DOWN2: 2v+b -> b; UP2: (v+b)/2 -> b
  Expr* node = nullptr;
};

struct Analysis {
  const Pipeline* p = nullptr;
  std::vector<int64_t> params;
  std::vector<Ext3> stage_ext, image_ext;
  std::vector<int64_t> table_len;
  std::vector<ReadSite> reads;               // every ACCESS node of every stage
  std::vector<std::vector<int>> reads_of;    // per consumer stage: indices into reads
};

Analysis analyze(const Pipeline& p, const std::vector<int64_t>& params);   // throws Error

// JSON description of the dependence vectors / footprints of every edge
std::string describe_pipeline(const Analysis& A);

// inline.cpp: substitute data-expanding intermediate stages into their readers (returns the rewritten
// pipeline; names of the inlined stages appended to *inlined)
std::shared_ptr<Pipeline> inline_expanding(std::shared_ptr<Pipeline> p, const std::vector<int64_t>& params,
                                           std::vector<std::string>* inlined);

// factor.cpp: separable evaluation of rank-1 linear f32 stencils (reassociation mode only; names of the
// factored stages appended to *factored)
std::shared_ptr<Pipeline> factor_stencils(std::shared_ptr<Pipeline> p, const std::vector<int64_t>& params,
                                          std::vector<std::string>* factored);

// phase.cpp: alignment & scaling of downsampling edges -- a stage read only as S(2v + b) along y or x by
// readers of half its extent is replaced by its two phases at the readers' extent (exact; names of the split
// stages, "name/y" or "name/x", appended to *split).  PMG_PHASE_SPLIT=0 disables it.
std::shared_ptr<Pipeline> phase_split(std::shared_ptr<Pipeline> p, const std::vector<int64_t>& params,
                                      std::vector<std::string>* split);

// ---- paper §4 formulas (warp geometry, scratchpads, overlap) ----
std::array<int, 3> warp_sizes(const std::array<int, 3>& B, int warp_size);

// ---- row-interval propagation for bands / workspaces ----
struct RowIv { int64_t lo = 0, hi = 0; };   // [lo, hi) in the producer's own row space
// requirement on `src` rows implied by consumer rows [lo, hi) through one read site
RowIv rows_needed(const Analysis& A, const ReadSite& r, RowIv consumer_rows, int64_t src_rows);

}  // namespace pmg
