// plan.hpp -- the hg_plan object (internal).
#ifndef HG_PLAN_HPP
#define HG_PLAN_HPP

#include "jit.hpp"
#include "kernels.hpp"

#include <map>
#include <string>
#include <memory>
#include <vector>

struct hg_plan {
  int device = 0;
  hg::Knobs knobs;                    // family selectors, read once at creation
  hg_program prog{};
  std::vector<hg_op> ops;
  hg::Analysis an;
  std::vector<hg::Layout> lay;        // per buffer (initial argument index)
  std::vector<void *> dptr;           // per buffer
  std::vector<CUtensorMap> tmCur, tmPrev;
  std::vector<int> bind;              // slot -> buffer
  int64_t stepsDone = 0;
  hg::GOp *gopsDev = nullptr;
  int nslots = 0;
  std::vector<int> resSlot;
  int64_t launches = 0;
  int chunks = 0;                     // star z-chunks (0 = auto)
  int starGeo = 0;                    // star tile geometry (starGeoFor)
  int boundaryLast = 0;               // star: z-boundary chunks last (dmp overlap)
  // one-shot (consumed by the next planStep): halo faces the star kernel must wait for
  const unsigned long long *waitFlags = nullptr;
  unsigned long long waitEpoch = 0;
  int waitMask = 0;
  hg::StarLaunch fuse{};              // one-shot: fused-swap fields (fuse.fuse != 0)
  // one-shot dmp extras of the next star launch: bounded-wait error word + timeout, packed
  // x-face receive slabs of the cur buffer, and (NCCL transport) an event the halo-reading
  // units wait for while the interior units run
  unsigned long long *waitErr = nullptr;
  unsigned long long waitTimeout = 0;
  const void *xin[2] = {nullptr, nullptr};
  int xw[2] = {0, 0};
  cudaEvent_t splitEvent = nullptr;
  int splitMask = 0;
  // deep halos: the step's output region extends past the core by regionExt[d][lo/hi] (the
  // neighbours' points the next steps of the round need), and the packed x slabs' receive box
  // relative to that region
  int64_t regionExt[3][2] = {{0, 0}, {0, 0}, {0, 0}};
  int band[6] = {0, 0, 0, 0, 0, 0};   // per face: units within band of it read received cells
  int xbox[6] = {0, 0, 0, 0, 0, 0}; // oz, oy, bz, by, ox_lo, ox_hi (xboxSet)
  bool xboxSet = false;
  hg::UnitOrderCache order;           // star launch orders (boundary units last)
  // HG_DEBUG_GUARDS: guarded allocations (user pointer -> allocation base); 0-byte guards
  // otherwise
  std::map<void *, std::pair<void *, size_t>> guardBase; // -> (base, buffer bytes)
  std::vector<char> callerOwned;      // per buffer: bound by hg_plan_bind (never freed by us)
  size_t guardBytes = 0;
  std::shared_ptr<hg::JitKernel> jit;  // fused-apply family (generated, per program)
  std::vector<CUtensorMap> tmApply;   // per buffer, for the fused-apply boxes
  std::map<int, cudaGraphExec_t> graphs; // hg_plan_run: captured G-step graphs per phase
  // multi-apply steps: the applies, their temps (HBM, laid out over their domains) and one
  // compiled op slice per apply
  std::vector<hg_apply> applies;
  std::vector<hg::Layout> tmpLay;
  std::vector<void *> tmpPtr;
  struct MultiApply {
    hg::GOp *ops = nullptr;
    int nslots = 0;
    std::vector<int> resSlot;
    // fused-apply form: the apply as a single-apply program over virtual fields
    // [fields..., temps...] (all in the field layout), its generated kernel, TMA descriptors
    std::shared_ptr<hg::JitKernel> jit;
    hg_program sub{};
    std::vector<CUtensorMap> tmField, tmTemp;
    std::vector<int> direct; // per result: field written in place of the temp, or -1
  };
  std::vector<MultiApply> multi;
  std::vector<char> storeDone; // multi-apply stores folded into their apply (direct results)
  // two-step passes (tb.cu): per buffer a shadow allocation with the same halo ring, and the
  // TMA descriptors of both; hg_plan_run exchanges a buffer with its shadow after each pass
  std::vector<void *> shadow;
  std::vector<char> shadowOk;         // ring of the shadow == ring of the buffer
  std::vector<CUtensorMap> tmTb, tmTbSh, tmCurSh, tmPrevSh;
  bool tbOff = false;                 // set once a dmp exported the buffers
  std::string namePrefix;             // "multiNx_fused_" when the applies were fused
  int64_t tbPasses = 0;
  // whole-run resident 2D kernel (resident.cu): exchange rows + per-CTA epoch flags
  void *resXbuf = nullptr;
  size_t resXbufBytes = 0;
  unsigned long long *resFlags = nullptr;
  int resCtas = 0;
  unsigned long long resLaunches = 0;
  unsigned resTag = 0;
};

namespace hg {
int cudaCheck(cudaError_t e, const char *what);
// Device allocation of a plan buffer: with knobs.guards, inside canary bands of guardBytes.
int planAlloc(hg_plan &p, void **ptr, size_t bytes, const char *what);
void planFree(hg_plan &p, void *ptr);
// The allocation base and guard offset of a plan buffer (IPC handles need the base).
void *planAllocBase(const hg_plan &p, void *ptr);
// One time step on `st` with the current binding, then rotate.
int planStep(hg_plan &p, cudaStream_t st);
// Whether hg_plan_run advances this plan by two-step passes (tb.cu).
bool tbEligible(const hg_plan &p);
// Whether hg_plan_run runs this plan's steps in one resident launch (resident.cu).
bool residentEligible(const hg_plan &p);
} // namespace hg

#endif
