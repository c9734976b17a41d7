// hg_internal.hpp -- shared declarations of the halogen-b200 library (not installed).
#ifndef HG_INTERNAL_HPP
#define HG_INTERNAL_HPP

#include "hg/hg.h"

#include <cstdint>
#include <string>
#include <vector>

namespace hg {

// ---- errors (thread-local last error, hg_last_error) ----------------------------------
int setError(int status, const std::string &msg);

// ---- program analysis (program.cpp) ----------------------------------------------------
enum class Family { Generic = 0, Star = 1, Apply = 2, Multi = 3 };
enum StarKind { kHeat = 0, kWave = 1, kCopy = 2 };

// The star-Laplacian family the generator emits (kernels.cpp:110-135, 205-226):
//   lap = c*W0; for d in 0..rank-1, k in taps: lap = lap + (u[+k e_d] + u[-k e_d]) * W[d][k]
//   heat: out = c + lap*S        wave: out = (cur*K2 - prev) + lap*S        copy: out = c
struct StarSpec {
  int kind = kHeat;
  int rank = 0;
  int ntaps = 0;     // 1: {1}, 2: {1,2}, 3: {1,2,4}
  int radius = 0;    // largest tap
  uint64_t w0 = 0;   // raw constant bits
  uint64_t w[3][3] = {};
  uint64_t scale = 0, two = 0;
  int cur_operand = 0, prev_operand = -1;
};

struct Analysis {
  Family family = Family::Generic;
  StarSpec star;
  std::string name;            // kernel family name
  int64_t dom_lb[3] = {0, 0, 0}, dom_ub[3] = {1, 1, 1}; // apply domain (hull of stores)
  std::vector<int> src;        // rotationSources
  int period = 1;              // lcm of group lengths
};

// Validates + classifies.  Returns HG_OK or an error status (message set).  allowStar = false
// sends star programs to the fused-apply family (HG_NO_STAR, tests).
int analyze(const hg_program &p, Analysis &out, bool allowStar = true);

// ---- family selectors (tests and A/B runs) ---------------------------------------------
// Read from the environment ONCE per plan, in hg_plan_create; no launcher reads it.
struct Knobs {
  bool noStar = false;        // HG_NO_STAR=1: star programs through the fused-apply family
  bool noApplyJit = false;    // HG_NO_APPLY_JIT=1: the generic kernel, not generated code
  bool noFuseApplies = false; // HG_NO_FUSE_APPLIES=1: multi-apply steps apply by apply
  bool noResident = false;    // HG_NO_RESIDENT=1: 2D heat step by step
  bool tb = false;            // HG_TB=1: two-step passes for large 3D heat (opt-in)
  int starGeo = -1;           // HG_STAR_GEO=n: force the star tile geometry
  int jitDepth = 0;           // HG_JIT_DEPTH=n: TMA ring depth of the fused-apply family
  bool jitPersist = true;     // HG_JIT_PERSIST=0: fused-apply family one CTA per unit
  bool jitPack = false;       // HG_JIT_PACK=1: fused-apply family f32 adds as FADD2 (PW set:
                              // neutral, profiles/r2_ab.md)
  int pitchPad = 0;           // HG_PITCH_PAD=n: n extra 128-byte lines per row (layout A/B)
  bool guards = false;        // HG_DEBUG_GUARDS=1: canary bands around every device buffer of
                              // the plan (hg_plan_check_guards finds out-of-bounds writes)
};
Knobs readKnobs();
int validateProgram(const hg_program &p);

// the stores of either program form (single apply: one per result; multi-apply: nstores)
inline int storedCount(const hg_program &g) { return g.napplies > 0 ? g.nstores : g.nresults; }
inline int storedField(const hg_program &g, int k) {
  return g.napplies > 0 ? g.mstore_field[k] : g.store_field[k];
}
inline const hg_bounds &storedRegion(const hg_program &g, int k) {
  return g.napplies > 0 ? g.mstore[k] : g.store[k];
}

// ---- device layout -----------------------------------------------------------------------
struct Layout {
  int rank = 0, es = 4;
  int64_t shape[3] = {1, 1, 1}; // logical alloc shape (unused dims = 1)
  int64_t lb[3] = {0, 0, 0};
  int64_t pitch = 0, col0 = 0, rows = 1;
  size_t bytes() const { return static_cast<size_t>(pitch * rows) * es; }
  int64_t logicalCount() const {
    int64_t n = 1;
    for (int d = 0; d < rank; ++d) n *= shape[d];
    return n;
  }
};
// padLines: extra 128-byte lines per row (HG_PITCH_PAD experiments)
Layout makeLayout(const hg_bounds &b, int rank, int es, int64_t core_lb_last,
                  int padLines = 0);

// ---- generic (bytecode) program for the generic kernel ---------------------------------
struct GOp {       // compact, slot-allocated
  int32_t code;    // hg_opcode
  int16_t dst, a, b;
  int16_t operand;
  int32_t pad;
  int64_t delta;   // ACCESS: flattened element offset in the operand layout
  uint64_t bits;   // CONST
};

uint64_t fnv1a(const void *p, size_t n);

} // namespace hg

#endif
