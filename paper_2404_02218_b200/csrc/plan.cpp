// plan.cpp -- device-resident plans: field allocation in HBM, upload/download, device init,
// and the runSerialStencil time loop (serial.cpp:57-88) over the sm_100a kernels.
#include "plan.hpp"

#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <exception>
#include <map>
#include <mutex>
#include <thread>

namespace hg {

int cudaCheck(cudaError_t e, const char *what) {
  if (e == cudaSuccess)
    return HG_OK;
  return setError(HG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {

// Generated kernels are cached per (source, device): NVRTC runs once per distinct program.
std::shared_ptr<JitKernel> jitCached(const hg_program &g, int device, const Knobs &kn) {
  static std::mutex mu;
  static std::map<std::pair<std::string, int>, std::shared_ptr<JitKernel>> cache;
  auto k = std::make_shared<JitKernel>();
  k->deep = kn.jitDepth;
  k->pack = kn.jitPack;
  if (jitBuildSource(g, *k) != HG_OK)
    return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(k->source, device);
  auto it = cache.find(key);
  if (it != cache.end())
    return it->second;
  if (jitCompile(*k) != HG_OK || jitLoad(*k, device) != HG_OK)
    return nullptr;
  cache[key] = k;
  return k;
}

// Linear-scan slot allocation for the generic kernel: a value lives until its last use.
// Compiles one apply region (ops[0..nops), region-relative operand indices) whose operand o
// is laid out as lay[o].
int compileSlice(int rank, const hg_op *ops, int nops, const int32_t *resultOp, int nresults,
                 const std::vector<const Layout *> &lay, std::vector<GOp> &out, int &nslots,
                 std::vector<int> &resSlot) {
  std::vector<int> last(static_cast<size_t>(nops), -1);
  for (int i = 0; i < nops; ++i) {
    const hg_op &o = ops[i];
    if (o.code >= HG_OP_ADD) {
      last[static_cast<size_t>(o.a)] = std::max(last[static_cast<size_t>(o.a)], i);
      last[static_cast<size_t>(o.b)] = std::max(last[static_cast<size_t>(o.b)], i);
    }
  }
  for (int k = 0; k < nresults; ++k)
    last[static_cast<size_t>(resultOp[k])] = nops;
  std::vector<int> slot(static_cast<size_t>(nops), -1);
  std::vector<int> freeSlots;
  nslots = 0;
  out.assign(static_cast<size_t>(nops), GOp{});
  for (int i = 0; i < nops; ++i) {
    const hg_op &o = ops[i];
    GOp &q = out[static_cast<size_t>(i)];
    std::memset(&q, 0, sizeof q);
    q.code = o.code;
    if (o.code >= HG_OP_ADD) {
      q.a = static_cast<int16_t>(slot[static_cast<size_t>(o.a)]);
      q.b = static_cast<int16_t>(slot[static_cast<size_t>(o.b)]);
      // operands dying here free their slots before the result is assigned
      for (int v : {o.a, o.b})
        if (last[static_cast<size_t>(v)] == i && slot[static_cast<size_t>(v)] >= 0) {
          if (std::find(freeSlots.begin(), freeSlots.end(), slot[static_cast<size_t>(v)]) ==
              freeSlots.end())
            freeSlots.push_back(slot[static_cast<size_t>(v)]);
        }
    }
    int s;
    if (!freeSlots.empty()) {
      s = freeSlots.back();
      freeSlots.pop_back();
    } else {
      s = nslots++;
    }
    slot[static_cast<size_t>(i)] = s;
    q.dst = static_cast<int16_t>(s);
    if (last[static_cast<size_t>(i)] < 0) // dead value: free immediately
      freeSlots.push_back(s);
    if (o.code == HG_OP_ACCESS) {
      q.operand = static_cast<int16_t>(o.operand);
      const Layout &L = *lay[static_cast<size_t>(o.operand)];
      int64_t stride = 1, delta = 0;
      for (int d = rank - 1; d >= 0; --d) {
        delta += o.off[d] * stride;
        stride *= d == rank - 1 ? L.pitch : L.shape[d];
      }
      q.delta = delta;
    } else if (o.code == HG_OP_CONST) {
      q.bits = o.bits;
    }
  }
  resSlot.clear();
  for (int k = 0; k < nresults; ++k)
    resSlot.push_back(slot[static_cast<size_t>(resultOp[k])]);
  if (nslots > 48)
    return setError(HG_EUNSUPPORTED, "apply region needs too many live values");
  return HG_OK;
}

int uploadOps(const std::vector<GOp> &ops, GOp **dev) {
  int st = cudaCheck(cudaMalloc(dev, sizeof(GOp) * std::max<size_t>(ops.size(), 1)),
                     "cudaMalloc(ops)");
  if (st)
    return st;
  return cudaCheck(cudaMemcpy(*dev, ops.data(), sizeof(GOp) * ops.size(), cudaMemcpyHostToDevice),
                   "cudaMemcpy(ops)");
}

int compileGeneric(hg_plan &p) {
  const hg_program &g = p.prog;
  std::vector<const Layout *> lay;
  for (int o = 0; o < g.noperands; ++o)
    lay.push_back(&p.lay[static_cast<size_t>(g.operand_field[o])]);
  std::vector<GOp> out;
  int st = compileSlice(g.rank, g.ops, g.nops, g.result_op, g.nresults, lay, out, p.nslots,
                        p.resSlot);
  if (st)
    return st;
  return uploadOps(out, &p.gopsDev);
}

// Multi-apply through the fused-apply family: every apply becomes a single-apply program over
// virtual fields [fields..., temps...] that all share the field layout, compiled to generated
// straight-line code.  A result no later apply reads and exactly one store copies over the
// apply's whole domain is written straight into that field (no temp, no copy).  Returns
// false (nothing allocated) when some apply does not fit the family.
bool sameBox(const hg_bounds &a, const hg_bounds &b, int rank) {
  for (int d = 0; d < rank; ++d)
    if (a.lb[d] != b.lb[d] || a.ub[d] != b.ub[d])
      return false;
  return true;
}

bool compileMultiJit(hg_plan &p, int device, int &st) {
  st = HG_OK;
  const hg_program &g = p.prog;
  const int F = g.nfields;
  if (p.knobs.noApplyJit || F + g.ntemps > HG_MAX_FIELDS || g.rank < 2)
    return false;
  for (int f = 1; f < F; ++f)
    for (int d = 0; d < g.rank; ++d)
      if (g.fields[f].lb[d] != g.fields[0].lb[d] || g.fields[f].ub[d] != g.fields[0].ub[d])
        return false;
  std::vector<int> consumers(static_cast<size_t>(g.ntemps), 0), stores(static_cast<size_t>(g.ntemps), 0);
  for (int a = 0; a < g.napplies; ++a)
    for (int o = 0; o < p.applies[static_cast<size_t>(a)].noperands; ++o)
      if (p.applies[static_cast<size_t>(a)].operand[o] < 0)
        ++consumers[static_cast<size_t>(-p.applies[static_cast<size_t>(a)].operand[o] - 1)];
  for (int k = 0; k < g.nstores; ++k)
    ++stores[static_cast<size_t>(g.mstore_temp[k])];
  std::vector<hg_plan::MultiApply> ms(static_cast<size_t>(g.napplies));
  p.storeDone.assign(static_cast<size_t>(g.nstores), 0);
  for (int a = 0; a < g.napplies; ++a) {
    const hg_apply &A = p.applies[static_cast<size_t>(a)];
    hg_plan::MultiApply &M = ms[static_cast<size_t>(a)];
    hg_program &S = M.sub;
    std::memset(&S, 0, sizeof S);
    S.rank = g.rank;
    S.dtype = g.dtype;
    S.nfields = F + g.ntemps;
    for (int i = 0; i < S.nfields; ++i)
      S.fields[i] = g.fields[0];
    S.noperands = A.noperands;
    for (int o = 0; o < A.noperands; ++o)
      S.operand_field[o] = A.operand[o] >= 0 ? A.operand[o] : F + (-A.operand[o] - 1);
    S.nops = A.nops;
    S.ops = p.ops.data() + A.op_begin;
    S.nresults = A.nresults;
    M.direct.assign(static_cast<size_t>(A.nresults), -1);
    for (int k = 0; k < A.nresults; ++k) {
      const int t = A.result_temp[k];
      S.result_op[k] = A.result_op[k];
      S.store_field[k] = F + t;
      S.store[k] = A.domain;
      if (consumers[static_cast<size_t>(t)] == 0 && stores[static_cast<size_t>(t)] == 1 &&
          jitMisaligned(S, p.lay[0]) == 0)
        for (int j = 0; j < g.nstores; ++j)
          if (g.mstore_temp[j] == t && sameBox(g.mstore[j], A.domain, g.rank)) {
            M.direct[static_cast<size_t>(k)] = g.mstore_field[j];
            p.storeDone[static_cast<size_t>(j)] = 1;
          }
    }
    Analysis none;
    if (!jitEligible(S, none, nullptr))
      return false;
    M.jit = jitCached(S, device, p.knobs);
    if (!M.jit)
      return false;
  }
  // temps in the field layout (only the ones some apply or store still reads)
  p.tmpLay.assign(static_cast<size_t>(g.ntemps), p.lay[0]);
  p.tmpPtr.assign(static_cast<size_t>(g.ntemps), nullptr);
  for (int t = 0; t < g.ntemps; ++t) {
    if (!consumers[static_cast<size_t>(t)] && !stores[static_cast<size_t>(t)])
      continue;
    st = planAlloc(p, &p.tmpPtr[static_cast<size_t>(t)], p.lay[0].bytes(), "cudaMalloc(temp)");
    if (st)
      return true;
    cudaMemset(p.tmpPtr[static_cast<size_t>(t)], 0, p.lay[0].bytes());
  }
  for (auto &M : ms) {
    M.tmField.resize(static_cast<size_t>(F));
    M.tmTemp.resize(static_cast<size_t>(g.ntemps));
    for (int f = 0; f < F && !st; ++f)
      st = jitTensorMap(*M.jit, g.dtype, g.rank, p.lay[static_cast<size_t>(f)],
                        p.dptr[static_cast<size_t>(f)], &M.tmField[static_cast<size_t>(f)]);
    for (int t = 0; t < g.ntemps && !st; ++t)
      if (p.tmpPtr[static_cast<size_t>(t)])
        st = jitTensorMap(*M.jit, g.dtype, g.rank, p.lay[0], p.tmpPtr[static_cast<size_t>(t)],
                          &M.tmTemp[static_cast<size_t>(t)]);
    if (st)
      return true;
  }
  p.multi = std::move(ms);
  p.an.name = "multi" + std::to_string(g.napplies) + "x_apply" + std::to_string(g.rank) + "d_" +
              (g.dtype == HG_F32 ? "f32" : "f64");
  return true;
}

// Multi-apply: one compiled slice per apply, temps in HBM laid out over their domains.
int compileMulti(hg_plan &p) {
  const hg_program &g = p.prog;
  const int es = g.dtype == HG_F32 ? 4 : 8;
  {
    int st = HG_OK;
    if (compileMultiJit(p, p.device, st))
      return st;
  }
  p.storeDone.assign(static_cast<size_t>(g.nstores), 0);
  p.tmpLay.assign(static_cast<size_t>(g.ntemps), Layout{});
  p.tmpPtr.assign(static_cast<size_t>(g.ntemps), nullptr);
  for (int a = 0; a < g.napplies; ++a) {
    const hg_apply &A = p.applies[static_cast<size_t>(a)];
    for (int k = 0; k < A.nresults; ++k) {
      const int t = A.result_temp[k];
      Layout L = makeLayout(A.domain, g.rank, es, A.domain.lb[g.rank - 1]);
      p.tmpLay[static_cast<size_t>(t)] = L;
      int st = planAlloc(p, &p.tmpPtr[static_cast<size_t>(t)], L.bytes(), "cudaMalloc(temp)");
      if (st)
        return st;
      cudaMemset(p.tmpPtr[static_cast<size_t>(t)], 0, L.bytes());
    }
  }
  p.multi.clear();
  for (int a = 0; a < g.napplies; ++a) {
    const hg_apply &A = p.applies[static_cast<size_t>(a)];
    std::vector<const Layout *> lay;
    for (int o = 0; o < A.noperands; ++o)
      lay.push_back(A.operand[o] >= 0 ? &p.lay[static_cast<size_t>(A.operand[o])]
                                      : &p.tmpLay[static_cast<size_t>(-A.operand[o] - 1)]);
    hg_plan::MultiApply M;
    std::vector<GOp> out;
    int st = compileSlice(g.rank, g.ops + A.op_begin, A.nops, A.result_op, A.nresults, lay, out,
                          M.nslots, M.resSlot);
    if (st)
      return st;
    st = uploadOps(out, &M.ops);
    if (st)
      return st;
    p.multi.push_back(M);
  }
  return HG_OK;
}

int multiStep(hg_plan &p, cudaStream_t st) {
  const hg_program &g = p.prog;
  for (int a = 0; a < g.napplies; ++a) {
    const hg_apply &A = p.applies[static_cast<size_t>(a)];
    const hg_plan::MultiApply &M = p.multi[static_cast<size_t>(a)];
    if (M.jit) {
      const CUtensorMap *tms[HG_MAX_FIELDS];
      void *outs[HG_MAX_RESULTS];
      for (int o = 0; o < A.noperands; ++o)
        tms[o] = A.operand[o] >= 0
                     ? &M.tmField[static_cast<size_t>(p.bind[static_cast<size_t>(A.operand[o])])]
                     : &M.tmTemp[static_cast<size_t>(-A.operand[o] - 1)];
      for (int k = 0; k < A.nresults; ++k) {
        const int f = M.direct[static_cast<size_t>(k)];
        outs[k] = f >= 0 ? p.dptr[static_cast<size_t>(p.bind[static_cast<size_t>(f)])]
                         : p.tmpPtr[static_cast<size_t>(A.result_temp[k])];
      }
      int rc = jitLaunch(*M.jit, M.sub, p.lay[0], tms, outs, 0, p.knobs.jitPersist, st);
      if (rc)
        return rc;
      ++p.launches;
      continue;
    }
    GenericLaunch L{};
    L.dtype = g.dtype;
    L.rank = g.rank;
    for (int d = 0; d < g.rank; ++d) {
      L.dom_lb[d] = A.domain.lb[d];
      L.dom_ext[d] = A.domain.ub[d] - A.domain.lb[d];
    }
    L.nops = A.nops;
    L.nslots = M.nslots;
    L.noperands = A.noperands;
    L.nresults = A.nresults;
    L.ops_dev = M.ops;
    for (int o = 0; o < A.noperands; ++o) {
      if (A.operand[o] >= 0) {
        const int b = p.bind[static_cast<size_t>(A.operand[o])];
        L.op_base[o] = p.dptr[static_cast<size_t>(b)];
        L.op_lay[o] = devLayout(p.lay[static_cast<size_t>(b)]);
      } else {
        const int t = -A.operand[o] - 1;
        L.op_base[o] = p.tmpPtr[static_cast<size_t>(t)];
        L.op_lay[o] = devLayout(p.tmpLay[static_cast<size_t>(t)]);
      }
    }
    for (int k = 0; k < A.nresults; ++k) {
      const int t = A.result_temp[k];
      L.out_base[k] = p.tmpPtr[static_cast<size_t>(t)];
      L.out_lay[k] = devLayout(p.tmpLay[static_cast<size_t>(t)]);
      L.res_slot[k] = M.resSlot[static_cast<size_t>(k)];
      for (int d = 0; d < 3; ++d) {
        L.st_lb[k][d] = d < g.rank ? A.domain.lb[d] : 0;
        L.st_ub[k][d] = d < g.rank ? A.domain.ub[d] : 1;
      }
    }
    int rc = launchGeneric(L, st);
    if (rc)
      return rc;
    ++p.launches;
  }
  for (int k = 0; k < g.nstores; ++k) { // stencil.store: temp region -> field
    if (p.storeDone[static_cast<size_t>(k)])
      continue;
    const int t = g.mstore_temp[k];
    const int b = p.bind[static_cast<size_t>(g.mstore_field[k])];
    int rc = launchCopyBox(p.tmpPtr[static_cast<size_t>(t)], devLayout(p.tmpLay[static_cast<size_t>(t)]),
                           p.dptr[static_cast<size_t>(b)], devLayout(p.lay[static_cast<size_t>(b)]),
                           g.mstore[k].lb, g.mstore[k].ub, st);
    if (rc)
      return rc;
    ++p.launches;
  }
  return HG_OK;
}

} // namespace

constexpr unsigned char kGuardByte = 0xA5;

int planAlloc(hg_plan &p, void **ptr, size_t bytes, const char *what) {
  *ptr = nullptr;
  if (!p.knobs.guards)
    return cudaCheck(cudaMalloc(ptr, bytes), what);
  p.guardBytes = 64 << 10;
  char *base = nullptr;
  if (int st = cudaCheck(cudaMalloc(&base, bytes + 2 * p.guardBytes), what))
    return st;
  if (int st = cudaCheck(cudaMemset(base, kGuardByte, bytes + 2 * p.guardBytes),
                         "cudaMemset(guards)"))
    return st;
  *ptr = base + p.guardBytes;
  p.guardBase[*ptr] = {base, bytes};
  return HG_OK;
}

void planFree(hg_plan &p, void *ptr) {
  auto it = p.guardBase.find(ptr);
  if (it == p.guardBase.end()) {
    cudaFree(ptr);
    return;
  }
  cudaFree(it->second.first);
  p.guardBase.erase(it);
}

void *planAllocBase(const hg_plan &p, void *ptr) {
  auto it = p.guardBase.find(ptr);
  return it == p.guardBase.end() ? ptr : it->second.first;
}

int planStep(hg_plan &p, cudaStream_t st) {
  const hg_program &g = p.prog;
  const Analysis &a = p.an;
  if (a.family == Family::Multi) {
    int rc = multiStep(p, st);
    if (rc)
      return rc;
  } else if (a.family == Family::Star) {
    const StarSpec &s = a.star;
    const int bCur = p.bind[static_cast<size_t>(g.operand_field[s.cur_operand])];
    const int bPrev =
        s.kind == kWave ? p.bind[static_cast<size_t>(g.operand_field[s.prev_operand])] : bCur;
    const int bOut = p.bind[static_cast<size_t>(g.store_field[0])];
    StarLaunch L{};
    L.spec = &s;
    L.dtype = g.dtype;
    L.rank = g.rank;
    const Layout &lay = p.lay[static_cast<size_t>(bOut)];
    for (int d = 0; d < g.rank; ++d) {
      L.start[d] = g.store[0].lb[d] - lay.lb[d];
      L.ext[d] = g.store[0].ub[d] - g.store[0].lb[d];
    }
    for (int d = 0; d < g.rank; ++d) { // deep halos: the region of this step of the round
      L.start[d] -= p.regionExt[d][0];
      L.ext[d] += p.regionExt[d][0] + p.regionExt[d][1];
      p.regionExt[d][0] = p.regionExt[d][1] = 0;
    }
    if (p.xboxSet) {
      L.xbox_set = 1;
      L.xoz = p.xbox[0];
      L.xoy = p.xbox[1];
      L.xbz = p.xbox[2];
      L.xby = p.xbox[3];
      L.xox[0] = p.xbox[4];
      L.xox[1] = p.xbox[5];
      p.xboxSet = false;
    }
    L.lay = devLayout(lay);
    L.tm_cur = &p.tmCur[static_cast<size_t>(bCur)];
    L.tm_prev = &p.tmPrev[static_cast<size_t>(bPrev)];
    L.out = p.dptr[static_cast<size_t>(bOut)];
    L.chunks = p.chunks;
    L.geo = p.starGeo;
    L.zorder_boundary_last = p.boundaryLast;
    L.order = &p.order;
    L.wait_flags = p.waitFlags;
    L.wait_epoch = p.waitEpoch;
    L.wait_mask = p.waitMask;
    L.err = p.waitErr;
    L.timeout_ns = p.waitTimeout;
    L.cur = p.dptr[static_cast<size_t>(bCur)];
    for (int sd = 0; sd < 2; ++sd) {
      L.xin[sd] = p.xin[sd];
      L.xw[sd] = p.xw[sd];
    }
    L.split_event = p.splitEvent;
    for (int d = 0; d < 6; ++d) {
      L.band[d] = p.band[d];
      p.band[d] = 0;
    }
    L.split_mask = p.splitMask;
    p.waitFlags = nullptr;
    p.waitErr = nullptr;
    p.xin[0] = p.xin[1] = nullptr;
    p.splitEvent = nullptr;
    p.splitMask = 0;
    if (p.fuse.fuse) {
      L.fuse = 1;
      L.xpack = p.fuse.xpack;
      L.nodata = p.fuse.nodata;
      for (int d = 0; d < 6; ++d) {
        L.hs[d] = p.fuse.hs[d];
        L.peer[d] = p.fuse.peer[d];
        L.pdelta[d] = p.fuse.pdelta[d];
        L.peer_flag[d] = p.fuse.peer_flag[d];
      }
      L.cnt = p.fuse.cnt;
      L.cnt_accum = p.fuse.cnt_accum;
      L.put_epoch = p.fuse.put_epoch;
      p.fuse.fuse = 0;
    }
    int st2 = launchStar(L, st, nullptr);
    if (st2)
      return st2;
  } else if (a.family == Family::Apply) {
    const CUtensorMap *tms[HG_MAX_FIELDS];
    void *outs[HG_MAX_RESULTS];
    for (int o = 0; o < g.noperands; ++o)
      tms[o] = &p.tmApply[static_cast<size_t>(p.bind[static_cast<size_t>(g.operand_field[o])])];
    for (int k = 0; k < g.nresults; ++k)
      outs[k] = p.dptr[static_cast<size_t>(p.bind[static_cast<size_t>(g.store_field[k])])];
    int st2 = jitLaunch(*p.jit, g, p.lay[0], tms, outs, p.chunks, p.knobs.jitPersist, st);
    if (st2)
      return st2;
  } else {
    GenericLaunch L{};
    L.dtype = g.dtype;
    L.rank = g.rank;
    for (int d = 0; d < g.rank; ++d) {
      L.dom_lb[d] = a.dom_lb[d];
      L.dom_ext[d] = a.dom_ub[d] - a.dom_lb[d];
    }
    L.nops = g.nops;
    L.nslots = p.nslots;
    L.noperands = g.noperands;
    L.nresults = g.nresults;
    L.ops_dev = p.gopsDev;
    for (int o = 0; o < g.noperands; ++o) {
      const int b = p.bind[static_cast<size_t>(g.operand_field[o])];
      L.op_base[o] = p.dptr[static_cast<size_t>(b)];
      L.op_lay[o] = devLayout(p.lay[static_cast<size_t>(b)]);
    }
    for (int k = 0; k < g.nresults; ++k) {
      const int b = p.bind[static_cast<size_t>(g.store_field[k])];
      L.out_base[k] = p.dptr[static_cast<size_t>(b)];
      L.out_lay[k] = devLayout(p.lay[static_cast<size_t>(b)]);
      L.res_slot[k] = p.resSlot[static_cast<size_t>(k)];
      for (int d = 0; d < 3; ++d) {
        L.st_lb[k][d] = d < g.rank ? g.store[k].lb[d] : 0;
        L.st_ub[k][d] = d < g.rank ? g.store[k].ub[d] : 1;
      }
    }
    int st2 = launchGeneric(L, st);
    if (st2)
      return st2;
  }
  if (a.family != Family::Multi)
    ++p.launches;
  // rotate (serial.cpp:83-85): next[i] = binding[src[i]]
  std::vector<int> nxt(p.bind.size());
  for (size_t i = 0; i < p.bind.size(); ++i)
    nxt[i] = p.bind[static_cast<size_t>(a.src[i])];
  p.bind.swap(nxt);
  ++p.stepsDone;
  return HG_OK;
}

} // namespace hg

using namespace hg;

#define HG_GUARD_BEGIN try {
#define HG_GUARD_END                                                                          \
  }                                                                                           \
  catch (const std::exception &e) {                                                           \
    return setError(HG_EINVAL, std::string("internal error: ") + e.what());                   \
  }

extern "C" {

int hg_device_count(int *n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (n)
    *n = e == cudaSuccess ? c : 0;
  return e == cudaSuccess ? HG_OK : cudaCheck(e, "cudaGetDeviceCount");
}

int hg_plan_create(const hg_program *prog, int device, hg_plan **out) {
  HG_GUARD_BEGIN
  if (!prog || !out)
    return setError(HG_EINVAL, "null argument");
  *out = nullptr;
  auto p = std::make_unique<hg_plan>();
  p->prog = *prog;
  p->ops.assign(prog->ops, prog->ops + std::max(prog->nops, 0));
  p->prog.ops = p->ops.data();
  if (prog->napplies > 0 && prog->applies) {
    p->applies.assign(prog->applies, prog->applies + prog->napplies);
    p->prog.applies = p->applies.data();
  }
  p->knobs = readKnobs();
  int st = analyze(p->prog, p->an, !p->knobs.noStar);
  if (st)
    return st;
  // a multi-apply step runs as one fused single-apply program when its temps inline within
  // the op budget (hg_fuse_applies); else apply by apply through HBM temps
  if (p->prog.napplies > 0 && !p->knobs.noFuseApplies) {
    std::vector<hg_op> fops(HG_MAX_OPS);
    hg_program fused;
    if (hg_fuse_applies(&p->prog, &fused, fops.data(), HG_MAX_OPS) == HG_OK) {
      fops.resize(static_cast<size_t>(fused.nops));
      p->namePrefix = "multi" + std::to_string(p->prog.napplies) + "x_fused_";
      p->ops = std::move(fops);
      p->prog = fused;
      p->prog.ops = p->ops.data();
      p->applies.clear();
      st = analyze(p->prog, p->an, !p->knobs.noStar);
      if (st)
        return st;
    }
  }
  const hg_program &g = p->prog;
  // rotating buffers must share one layout (the kernel addresses a slot, not a buffer)
  {
    int at = 0;
    for (int gi = 0; gi < g.ngroups; ++gi) {
      for (int j = 1; j < g.group_len[gi]; ++j) {
        const hg_bounds &x = g.fields[g.groups[at]], &y = g.fields[g.groups[at + j]];
        for (int d = 0; d < g.rank; ++d)
          if (x.lb[d] != y.lb[d] || x.ub[d] != y.ub[d])
            return setError(HG_EUNSUPPORTED,
                            "time-slot group rotates fields of different bounds");
      }
      at += g.group_len[gi];
    }
  }
  p->device = device;
  st = cudaCheck(cudaSetDevice(device), "cudaSetDevice");
  if (st)
    return st;
  const int es = g.dtype == HG_F32 ? 4 : 8;
  const int64_t coreLast = storedRegion(g, 0).lb[g.rank - 1];
  for (int f = 0; f < g.nfields; ++f) {
    Layout L = makeLayout(g.fields[f], g.rank, es, coreLast, p->knobs.pitchPad);
    void *ptr = nullptr;
    st = planAlloc(*p, &ptr, L.bytes(), "cudaMalloc(field)");
    if (st)
      return st;
    p->lay.push_back(L);
    p->dptr.push_back(ptr);
    st = cudaCheck(cudaMemset(ptr, 0, L.bytes()), "cudaMemset(field)");
    if (st)
      return st;
  }
  if (p->an.family == Family::Multi) {
    st = compileMulti(*p);
    if (st)
      return st;
    p->bind.resize(static_cast<size_t>(g.nfields));
    for (int i = 0; i < g.nfields; ++i)
      p->bind[static_cast<size_t>(i)] = i;
    *out = p.release();
    return HG_OK;
  }
  if (p->an.family == Family::Star && p->an.star.kind == kCopy)
    p->an.family = Family::Generic; // a plain copy needs no stencil machinery
  if (p->an.family == Family::Star) {
    int64_t ext[3] = {0, 0, 0};
    for (int d = 0; d < g.rank; ++d)
      ext[d] = g.store[0].ub[d] - g.store[0].lb[d];
    p->starGeo = starGeoFor(p->an.star, g.dtype, g.rank, ext);
    if (p->knobs.starGeo >= 0) // forced tile geometry (tests; heat f32 3D r<=2 only)
      p->starGeo = g.rank == 3 && g.dtype == HG_F32 && p->an.star.kind == kHeat &&
                           p->an.star.ntaps <= 2
                       ? p->knobs.starGeo
                       : 0;
    p->tmCur.resize(static_cast<size_t>(g.nfields));
    p->tmPrev.resize(static_cast<size_t>(g.nfields));
    for (int f = 0; f < g.nfields; ++f) {
      st = makeStarTensorMaps(p->an.star, g.dtype, g.rank, devLayout(p->lay[static_cast<size_t>(f)]),
                              p->dptr[static_cast<size_t>(f)], &p->tmCur[static_cast<size_t>(f)],
                              &p->tmPrev[static_cast<size_t>(f)], p->starGeo);
      if (st)
        return st;
    }
  } else {
    // any other DAG: the fused-apply family (generated straight-line code) when its tile
    // rims cover the accesses, else the slot-interpreting generic kernel
    std::string why;
    if (!p->knobs.noApplyJit && jitEligible(g, p->an, &why)) {
      auto k = jitCached(g, device, p->knobs);
      if (k) {
        p->jit = k;
        p->an.family = Family::Apply;
        p->an.name = "apply" + std::to_string(g.rank) + "d_" + (g.dtype == HG_F32 ? "f32" : "f64");
        p->tmApply.resize(static_cast<size_t>(g.nfields));
        for (int f = 0; f < g.nfields; ++f) {
          st = jitTensorMap(*k, g.dtype, g.rank, p->lay[static_cast<size_t>(f)],
                            p->dptr[static_cast<size_t>(f)], &p->tmApply[static_cast<size_t>(f)]);
          if (st)
            return st;
        }
      }
    }
    if (p->an.family != Family::Apply) {
      st = compileGeneric(*p);
      if (st)
        return st;
      if (p->nslots > 48)
        return setError(HG_EUNSUPPORTED, "apply region needs too many live values");
    }
  }
  p->bind.resize(static_cast<size_t>(g.nfields));
  for (int i = 0; i < g.nfields; ++i)
    p->bind[static_cast<size_t>(i)] = i;
  *out = p.release();
  return HG_OK;
  HG_GUARD_END
}

int hg_plan_destroy(hg_plan *p) {
  if (!p)
    return HG_OK;
  cudaSetDevice(p->device);
  for (auto &g : p->graphs)
    cudaGraphExecDestroy(g.second);
  for (size_t b = 0; b < p->dptr.size(); ++b)
    if (b >= p->callerOwned.size() || !p->callerOwned[b])
      planFree(*p, p->dptr[b]);
  for (void *d : p->shadow)
    if (d)
      planFree(*p, d);
  for (void *d : p->tmpPtr)
    planFree(*p, d);
  if (p->resXbuf)
    cudaFree(p->resXbuf);
  if (p->resFlags)
    cudaFree(p->resFlags);
  for (auto &m : p->multi)
    cudaFree(m.ops);
  if (p->gopsDev)
    cudaFree(p->gopsDev);
  delete p;
  return HG_OK;
}

int hg_plan_check_guards(hg_plan *p) {
  if (!p)
    return setError(HG_EINVAL, "null plan");
  if (p->guardBase.empty())
    return HG_OK;
  if (int st = cudaCheck(cudaSetDevice(p->device), "cudaSetDevice"))
    return st;
  if (int st = cudaCheck(cudaDeviceSynchronize(), "cudaDeviceSynchronize"))
    return st;
  std::vector<unsigned char> h(p->guardBytes);
  for (const auto &kv : p->guardBase) {
    const char *user = static_cast<const char *>(kv.first);
    const char *base = static_cast<const char *>(kv.second.first);
    const size_t bytes = kv.second.second;
    for (int side = 0; side < 2; ++side) {
      const char *g = side == 0 ? base : user + bytes;
      if (int st = cudaCheck(cudaMemcpy(h.data(), g, h.size(), cudaMemcpyDeviceToHost),
                             "cudaMemcpy(guard)"))
        return st;
      for (size_t i = 0; i < h.size(); ++i)
        if (h[i] != kGuardByte)
          return setError(HG_ETRAP, std::string("out-of-bounds write: guard band ") +
                                        (side == 0 ? "before" : "after") +
                                        " a device buffer of " + std::to_string(bytes) +
                                        " bytes modified at byte " + std::to_string(i) +
                                        " of the band");
    }
  }
  return HG_OK;
}

int hg_plan_kernel_name(const hg_plan *p, char *name, size_t cap) {
  if (!p)
    return setError(HG_EINVAL, "null plan");
  std::string n = p->namePrefix + (p->an.family != Family::Generic
                                      ? p->an.name
                                      : "generic" + std::to_string(p->prog.rank) + "d_" +
                                            (p->prog.dtype == HG_F32 ? "f32" : "f64"));
  if (tbEligible(*p))
    n += "+tb2"; // runs of >= 2 steps go through two-step passes (tb.cu)
  if (residentEligible(*p))
    n += "+resident"; // runs go through one shared-memory-resident launch (resident.cu)
  if (name && cap)
    std::snprintf(name, cap, "%s", n.c_str());
  return HG_OK;
}

int hg_plan_layout(const hg_plan *p, int b, hg_layout *out) {
  if (!p || !out || b < 0 || b >= static_cast<int>(p->lay.size()))
    return setError(HG_EINVAL, "bad plan/buffer");
  const Layout &L = p->lay[static_cast<size_t>(b)];
  std::memset(out, 0, sizeof *out);
  out->rank = L.rank;
  out->elem_bytes = L.es;
  for (int d = 0; d < L.rank; ++d) {
    out->shape[d] = L.shape[d];
    out->lb[d] = L.lb[d];
  }
  out->pitch = L.pitch;
  out->col0 = L.col0;
  out->rows = L.rows;
  out->device_ptr = p->dptr[static_cast<size_t>(b)];
  return HG_OK;
}

int hg_plan_init_fields(hg_plan *p, const int64_t *origin, void *stream) {
  if (!p)
    return setError(HG_EINVAL, "null plan");
  std::fill(p->shadowOk.begin(), p->shadowOk.end(), 0);
  int st = cudaCheck(cudaSetDevice(p->device), "cudaSetDevice");
  if (st)
    return st;
  for (size_t b = 0; b < p->dptr.size(); ++b) {
    // initialFields fills argument i with fieldIdx i (kernels.cpp:261-270)
    st = launchInit(p->dptr[b], devLayout(p->lay[b]), static_cast<int>(b), origin,
                    static_cast<cudaStream_t>(stream));
    if (st)
      return st;
    ++p->launches;
  }
  return HG_OK;
}

// Device-accessible address of a pinned host buffer (cudaHostAlloc / cudaHostRegister, mapped
// under unified addressing), or null for pageable memory.
static void *mappedHost(void *host) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
    cudaGetLastError(); // pageable memory on older runtimes reports an error; not sticky
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// Pageable host memory: a pinned two-buffer staging ring per device.  The host side of each
// chunk is a multi-threaded memcpy (one core's memcpy runs at ~10 GB/s, below PCIe), the
// device side the zero-copy kernel (uploads) or a pitched copy-engine copy (downloads), and
// chunk k's transfer overlaps chunk k+1's (or k-1's) host copy.
namespace {
constexpr size_t kStageBytes = size_t(128) << 20;

struct Staging {
  std::mutex mu;
  void *buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
};

Staging *stagingFor(int device) {
  static std::mutex mu;
  static std::map<int, Staging *> all; // process lifetime, like the CUDA context
  std::lock_guard<std::mutex> lk(mu);
  Staging *&st = all[device];
  if (!st)
    st = new Staging;
  return st;
}

int ensureStaging(Staging &st) {
  for (int i = 0; i < 2; ++i) {
    if (!st.buf[i]) {
      int rc = cudaCheck(cudaHostAlloc(&st.buf[i], kStageBytes, cudaHostAllocDefault),
                         "cudaHostAlloc(staging)");
      if (rc)
        return rc;
    }
    if (!st.ev[i]) {
      int rc = cudaCheck(cudaEventCreateWithFlags(&st.ev[i], cudaEventDisableTiming),
                         "cudaEventCreate(staging)");
      if (rc)
        return rc;
    }
  }
  return HG_OK;
}

void parallelCopy(void *dst, const void *src, size_t n) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nt = std::min<size_t>(std::min<size_t>(hw, 8), std::max<size_t>(1, n >> 23));
  if (nt <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  const size_t per = (n + nt - 1) / nt;
  std::vector<std::thread> th;
  for (size_t t = 1; t < nt; ++t) {
    const size_t o = t * per;
    if (o >= n)
      break;
    th.emplace_back([=] {
      std::memcpy(static_cast<char *>(dst) + o, static_cast<const char *>(src) + o,
                  std::min(per, n - o));
    });
  }
  std::memcpy(dst, src, std::min(per, n));
  for (auto &t : th)
    t.join();
}

int stagedCopy(hg_plan *p, int b, char *host, bool up, cudaStream_t s) {
  const Layout &L = p->lay[static_cast<size_t>(b)];
  Staging &sg = *stagingFor(p->device);
  std::lock_guard<std::mutex> lk(sg.mu);
  int rc = ensureStaging(sg);
  if (rc)
    return rc;
  const size_t rowBytes = static_cast<size_t>(L.shape[L.rank - 1]) * L.es;
  const int64_t rpc = std::max<int64_t>(1, static_cast<int64_t>(kStageBytes / rowBytes));
  char *dev = static_cast<char *>(p->dptr[static_cast<size_t>(b)]);
  const size_t dp = static_cast<size_t>(L.pitch) * L.es;
  DevLayout v = devLayout(L); // a chunk of rows viewed as a 2D field of its own
  v.rank = 2;
  v.shape[1] = L.shape[L.rank - 1];
  v.lb[0] = v.lb[1] = 0;
  int64_t prevR = 0, prevN = 0;
  int k = 0;
  for (int64_t r = 0; r < L.rows; r += rpc, ++k) {
    const int64_t n = std::min(rpc, L.rows - r);
    const int sb = k & 1;
    if (up) {
      // the transfer that last read this staging buffer (this call or the previous one)
      rc = cudaCheck(cudaEventSynchronize(sg.ev[sb]), "staging wait");
      if (rc)
        return rc;
      parallelCopy(sg.buf[sb], host + r * rowBytes, static_cast<size_t>(n) * rowBytes);
      v.shape[0] = n;
      rc = launchHostXfer(dev + static_cast<size_t>(r) * dp, v, sg.buf[sb], 1, nullptr, nullptr,
                          s);
      ++p->launches;
    } else {
      rc = cudaCheck(cudaMemcpy2DAsync(sg.buf[sb], rowBytes,
                                       dev + static_cast<size_t>(r) * dp + L.col0 * L.es, dp,
                                       rowBytes, static_cast<size_t>(n), cudaMemcpyDeviceToHost,
                                       s),
                     "download");
      if (!rc && k > 0) { // drain the previous chunk while this one is in flight
        rc = cudaCheck(cudaEventSynchronize(sg.ev[sb ^ 1]), "staging wait");
        if (!rc)
          parallelCopy(host + prevR * rowBytes, sg.buf[sb ^ 1],
                       static_cast<size_t>(prevN) * rowBytes);
      }
    }
    if (!rc)
      rc = cudaCheck(cudaEventRecord(sg.ev[sb], s), "staging event");
    if (rc)
      return rc;
    prevR = r;
    prevN = n;
  }
  if (!up && k > 0) {
    rc = cudaCheck(cudaEventSynchronize(sg.ev[(k - 1) & 1]), "staging wait");
    if (!rc)
      parallelCopy(host + prevR * rowBytes, sg.buf[(k - 1) & 1],
                   static_cast<size_t>(prevN) * rowBytes);
  }
  return rc;
}
} // namespace

// skip_lo/hi: raw box of buffer b not to move (uploads only; null = move everything)
static int copyField(hg_plan *p, int b, void *host, size_t bytes, void *stream, bool up,
                     const int64_t *skip_lo, const int64_t *skip_hi) {
  if (!p || b < 0 || b >= static_cast<int>(p->lay.size()))
    return setError(HG_EINVAL, "bad plan/buffer");
  const Layout &L = p->lay[static_cast<size_t>(b)];
  if (bytes != static_cast<size_t>(L.logicalCount()) * L.es)
    return setError(HG_EINVAL, "host buffer size does not match the field");
  int st = cudaCheck(cudaSetDevice(p->device), "cudaSetDevice");
  if (st)
    return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // downloads: the copy engines' pitched copy already runs at the flat rate (52 GB/s vs 51 for
  // the kernel, tools/xfer_probe.py); uploads: the zero-copy kernel (51 vs 31 GB/s)
  void *hd = !up ? nullptr : mappedHost(host);
  if (hd && reinterpret_cast<uintptr_t>(hd) % 16 == 0) {
    // pinned host memory: one zero-copy pass at the flat PCIe rate (kernels.cu hostXferKernel)
    st = launchHostXfer(p->dptr[static_cast<size_t>(b)], devLayout(L), hd, up ? 1 : 0, skip_lo,
                        skip_hi, s);
    ++p->launches;
    if (!st && !up)
      st = cudaCheck(cudaStreamSynchronize(s), "download");
    return st;
  }
  // pageable memory, large fields: through the pinned staging ring
  if (static_cast<size_t>(L.logicalCount()) * L.es >= (size_t(32) << 20) &&
      !mappedHost(host))
    return stagedCopy(p, b, static_cast<char *>(host), up, s);
  // pageable memory: the copy engines, one pitched copy of the whole field
  const size_t w = static_cast<size_t>(L.shape[L.rank - 1]) * L.es;
  char *dev = static_cast<char *>(p->dptr[static_cast<size_t>(b)]) + L.col0 * L.es;
  const size_t dp = static_cast<size_t>(L.pitch) * L.es;
  cudaError_t e =
      up ? cudaMemcpy2DAsync(dev, dp, host, w, w, static_cast<size_t>(L.rows),
                             cudaMemcpyHostToDevice, s)
         : cudaMemcpy2DAsync(host, w, dev, dp, w, static_cast<size_t>(L.rows),
                             cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && !up)
    e = cudaStreamSynchronize(s);
  return cudaCheck(e, up ? "upload" : "download");
}

int hg_plan_upload(hg_plan *p, int b, const void *host, size_t bytes, void *stream) {
  if (p && b >= 0 && b < static_cast<int>(p->shadowOk.size()))
    p->shadowOk[static_cast<size_t>(b)] = 0;
  return copyField(p, b, const_cast<void *>(host), bytes, stream, true, nullptr, nullptr);
}

int hg_plan_upload_live(hg_plan *p, int b, const void *host, size_t bytes, void *stream) {
  if (!p || b < 0 || b >= static_cast<int>(p->lay.size()))
    return setError(HG_EINVAL, "bad plan/buffer");
  if (b < static_cast<int>(p->shadowOk.size()))
    p->shadowOk[static_cast<size_t>(b)] = 0;
  // The slot buffer b is bound to now; the next step's stores into it and its loads.
  const hg_program &g = p->prog;
  int slot = -1;
  for (size_t i = 0; i < p->bind.size(); ++i)
    if (p->bind[i] == b)
      slot = static_cast<int>(i);
  bool loaded = false;
  for (int o = 0; o < g.noperands; ++o)
    loaded = loaded || g.operand_field[o] == slot;
  const hg_bounds *box = nullptr;
  int nbox = 0;
  if (g.napplies > 0) {
    for (int k = 0; k < g.nstores; ++k)
      if (g.mstore_field[k] == slot) {
        box = &g.mstore[k];
        ++nbox;
      }
  } else {
    for (int k = 0; k < g.nresults; ++k)
      if (g.store_field[k] == slot) {
        box = &g.store[k];
        ++nbox;
      }
  }
  if (slot < 0 || loaded || nbox != 1) // nothing the next step overwrites unread
    return copyField(p, b, const_cast<void *>(host), bytes, stream, true, nullptr, nullptr);
  const Layout &L = p->lay[static_cast<size_t>(b)];
  int64_t lo[3], hi[3];
  for (int d = 0; d < L.rank; ++d) {
    lo[d] = box->lb[d] - L.lb[d];
    hi[d] = box->ub[d] - L.lb[d];
  }
  return copyField(p, b, const_cast<void *>(host), bytes, stream, true, lo, hi);
}

int hg_plan_download(hg_plan *p, int b, void *host, size_t bytes, void *stream) {
  return copyField(p, b, host, bytes, stream, false, nullptr, nullptr);
}

} // extern "C"

namespace hg {

// Two-step passes (tb.cu) for large 3D heat steps on plans no dmp shares.  Opt-in
// (HG_TB=1): bit-exact, but on B200 the FMA-free two-step pass is issue-bound below the
// HBM-bound single step (profiles/r1_temporal_blocking.md), so it is not the default.
bool tbEligible(const hg_plan &p) {
  if (!p.knobs.tb || p.tbOff || p.an.family != Family::Star || !tbSupported(p.an.star, p.prog.dtype,
                                                                   p.prog.rank))
    return false;
  int64_t pts = 1;
  for (int d = 0; d < p.prog.rank; ++d)
    pts *= p.an.dom_ub[d] - p.an.dom_lb[d];
  return pts > (int64_t(1) << 22);
}

namespace {

ResLaunch residentLaunchOf(const hg_plan &p) {
  const hg_program &g = p.prog;
  const StarSpec &sp = p.an.star;
  ResLaunch L{};
  L.spec = &sp;
  L.dtype = g.dtype;
  const int bIn = p.bind[static_cast<size_t>(g.operand_field[sp.cur_operand])];
  const int bOut = p.bind[static_cast<size_t>(g.store_field[0])];
  const Layout &lay = p.lay[static_cast<size_t>(bOut)];
  L.lay = devLayout(lay);
  for (int d = 0; d < 2; ++d) {
    L.start[d] = g.store[0].lb[d] - lay.lb[d];
    L.ext[d] = g.store[0].ub[d] - g.store[0].lb[d];
  }
  L.in = p.dptr[static_cast<size_t>(bIn)];
  L.out = p.dptr[static_cast<size_t>(bOut)];
  return L;
}

} // namespace

// Small 2D heat plans (both fields fit in the SMs' shared memory) run whole calls in one
// resident launch; HG_NO_RESIDENT=1 keeps the per-step star kernel (A/B, tests).
bool residentEligible(const hg_plan &p) {
  if (p.knobs.noResident || p.tbOff || p.an.family != Family::Star || p.prog.rank != 2 ||
      p.an.star.kind != kHeat || p.prog.nresults != 1 || p.bind.size() != 2)
    return false;
  const ResLaunch L = residentLaunchOf(p);
  return L.in != L.out && residentSupported(L, nullptr, nullptr);
}

namespace {

int runResident(hg_plan &p, int64_t steps, cudaStream_t s) {
  ResLaunch L = residentLaunchOf(p);
  size_t xb = 0;
  int ctas = 0;
  if (!residentSupported(L, &xb, &ctas))
    return setError(HG_EUNSUPPORTED, "resident 2D kernel: plan does not fit");
  if (xb > p.resXbufBytes) {
    if (p.resXbuf)
      cudaFree(p.resXbuf);
    p.resXbuf = nullptr;
    int st = cudaCheck(cudaMalloc(&p.resXbuf, xb), "cudaMalloc(resident exchange)");
    // tagged words: a stale word (e.g. an earlier plan's allocation) must not carry a live tag
    if (!st)
      st = cudaCheck(cudaMemsetAsync(p.resXbuf, 0, xb, s), "cudaMemset(resident exchange)");
    if (st)
      return st;
    p.resTag = 0;
    p.resXbufBytes = xb;
  }
  if (ctas > p.resCtas) {
    if (p.resFlags)
      cudaFree(p.resFlags);
    p.resFlags = nullptr;
    int st = cudaCheck(cudaMalloc(&p.resFlags, sizeof(unsigned long long) * ctas),
                       "cudaMalloc(resident flags)");
    if (!st)
      st = cudaCheck(cudaMemsetAsync(p.resFlags, 0, sizeof(unsigned long long) * ctas, s),
                     "cudaMemset(resident flags)");
    if (st)
      return st;
    p.resCtas = ctas;
    p.resLaunches = 0;
  }
  L.xbuf = p.resXbuf;
  L.flags = p.resFlags;
  L.epoch = (++p.resLaunches) << 32; // above every epoch an earlier launch published
  L.tag0 = p.resTag;                  // tags tag0+1 .. tag0+blocks (blocks <= steps)
  p.resTag += static_cast<unsigned>(steps) + 1u;
  L.steps = steps;
  int st = launchResident(L, s);
  if (st)
    return st;
  ++p.launches;
  for (int64_t t = 0; t < steps; ++t) { // the rotation the steps performed
    std::vector<int> nxt(p.bind.size());
    for (size_t i = 0; i < p.bind.size(); ++i)
      nxt[i] = p.bind[static_cast<size_t>(p.an.src[i])];
    p.bind.swap(nxt);
  }
  p.stepsDone += steps;
  return HG_OK;
}

// Shadow of buffer b: same layout, same halo ring (a full copy once; the ring is never
// written by a step, and the plan's own writers invalidate it).
int ensureShadow(hg_plan &p, int b, cudaStream_t s) {
  const size_t n = p.dptr.size();
  if (p.shadow.size() != n) {
    p.shadow.assign(n, nullptr);
    p.shadowOk.assign(n, 0);
    p.tmTb.resize(n);
    p.tmTbSh.resize(n);
    p.tmCurSh.resize(n);
    p.tmPrevSh.resize(n);
  }
  const size_t bi = static_cast<size_t>(b);
  const Layout &L = p.lay[bi];
  uint32_t box[3];
  tbBox(p.an.star, p.prog.dtype, box);
  if (!p.shadow[bi]) {
    int st = planAlloc(p, &p.shadow[bi], L.bytes(), "cudaMalloc(shadow)");
    if (st)
      return st;
    p.shadowOk[bi] = 0;
    st = makeBoxTensorMap(p.prog.dtype, devLayout(L), p.dptr[bi], box, &p.tmTb[bi]);
    if (!st)
      st = makeBoxTensorMap(p.prog.dtype, devLayout(L), p.shadow[bi], box, &p.tmTbSh[bi]);
    if (!st)
      st = makeStarTensorMaps(p.an.star, p.prog.dtype, p.prog.rank, devLayout(L), p.shadow[bi],
                              &p.tmCurSh[bi], &p.tmPrevSh[bi], p.starGeo);
    if (st)
      return st;
  }
  if (!p.shadowOk[bi]) {
    int st = cudaCheck(cudaMemcpyAsync(p.shadow[bi], p.dptr[bi], L.bytes(),
                                       cudaMemcpyDeviceToDevice, s),
                       "shadow copy");
    if (st)
      return st;
    p.shadowOk[bi] = 1;
  }
  return HG_OK;
}

void swapWithShadow(hg_plan &p, int b) {
  const size_t bi = static_cast<size_t>(b);
  std::swap(p.dptr[bi], p.shadow[bi]);
  std::swap(p.tmTb[bi], p.tmTbSh[bi]);
  std::swap(p.tmCur[bi], p.tmCurSh[bi]);
  std::swap(p.tmPrev[bi], p.tmPrevSh[bi]);
}

// steps t+1, t+2 in one pass: reads the cur buffer, writes t+2 into its shadow (then the two
// exchange), t+1 only into the ring-keeping output buffer when it must persist
int tbPair(hg_plan &p, bool writeMid, cudaStream_t s) {
  const hg_program &g = p.prog;
  const StarSpec &sp = p.an.star;
  const int bIn = p.bind[static_cast<size_t>(g.operand_field[sp.cur_operand])];
  const int bMid = p.bind[static_cast<size_t>(g.store_field[0])];
  int st = ensureShadow(p, bIn, s);
  if (st)
    return st;
  TbLaunch L{};
  L.spec = &sp;
  L.dtype = g.dtype;
  const Layout &lay = p.lay[static_cast<size_t>(bIn)];
  for (int d = 0; d < 3; ++d) {
    L.start[d] = g.store[0].lb[d] - lay.lb[d];
    L.ext[d] = g.store[0].ub[d] - g.store[0].lb[d];
  }
  L.lay = devLayout(lay);
  L.tm_in = &p.tmTb[static_cast<size_t>(bIn)];
  L.mid = p.dptr[static_cast<size_t>(bMid)];
  L.write_mid = writeMid ? 1 : 0;
  L.out = p.shadow[static_cast<size_t>(bIn)];
  L.chunks = 0;
  st = launchTb(L, s, nullptr);
  if (st)
    return st;
  swapWithShadow(p, bIn);
  for (int k = 0; k < 2; ++k) { // the rotation of the two steps
    std::vector<int> nxt(p.bind.size());
    for (size_t i = 0; i < p.bind.size(); ++i)
      nxt[i] = p.bind[static_cast<size_t>(p.an.src[i])];
    p.bind.swap(nxt);
  }
  p.stepsDone += 2;
  ++p.launches;
  ++p.tbPasses;
  return HG_OK;
}

} // namespace
} // namespace hg

extern "C" {

int hg_plan_run(hg_plan *p, int64_t steps, void *stream) {
  if (!p)
    return setError(HG_EINVAL, "null plan");
  if (steps < 0)
    return setError(HG_EINVAL, "negative step count");
  int st = cudaCheck(cudaSetDevice(p->device), "cudaSetDevice");
  if (st)
    return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (steps >= 1 && steps < (int64_t(1) << 31) && residentEligible(*p))
    return runResident(*p, steps, s);
  if (steps >= 2 && tbEligible(*p)) {
    // pairs of steps; an odd step count ends with one ordinary step, which then also writes
    // the t+1 buffer, so only an even count needs the last pair to store its t+1 core
    const int64_t pairs = steps / 2;
    for (int64_t k = 0; k < pairs; ++k) {
      st = tbPair(*p, k + 1 == pairs && steps % 2 == 0, s);
      if (st)
        return st;
    }
    if (steps % 2)
      return planStep(*p, s);
    return HG_OK;
  }
  // Launch-bound small grids (e.g. config 1, 1024^2 2D, ~2 us of work per step) replay a
  // CUDA graph of G consecutive steps captured once per binding phase: the launch sequence
  // repeats with the rotation period, and each node keeps its by-value parameters.
  const int period = std::max(1, p->an.period);
  const int G = period * std::max(1, (16 + period - 1) / period);
  // only launch-bound steps (< ~4M points, a few us each) gain from replay; large steps run
  // eagerly (measured: graph replay made the 33M-point fused-apply step slower)
  int64_t pts = 1;
  for (int d = 0; d < p->prog.rank; ++d)
    pts *= p->an.dom_ub[d] - p->an.dom_lb[d];
  const bool noGraph = pts > (int64_t(1) << 22);
  if (!noGraph && steps > G && p->graphs.empty()) {
    // one eager step first: per-device kernel attributes are set outside any capture
    st = planStep(*p, s);
    if (st)
      return st;
    --steps;
  }
  while (!noGraph && steps >= G) {
    const int phase = static_cast<int>(p->stepsDone % period);
    auto it = p->graphs.find(phase);
    if (it == p->graphs.end()) {
      cudaStream_t cap;
      st = cudaCheck(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "stream");
      if (st)
        return st;
      const std::vector<int> bind0 = p->bind;
      const int64_t done0 = p->stepsDone, l0 = p->launches;
      st = cudaCheck(cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed), "capture");
      for (int t = 0; t < G && !st; ++t)
        st = planStep(*p, cap);
      cudaGraph_t graph = nullptr;
      cudaError_t ce = cudaStreamEndCapture(cap, &graph);
      cudaStreamDestroy(cap);
      p->bind = bind0; // capture only recorded the launches
      p->stepsDone = done0;
      p->launches = l0;
      if (st)
        return st;
      st = cudaCheck(ce, "cudaStreamEndCapture");
      if (st)
        return st;
      cudaGraphExec_t exec = nullptr;
      st = cudaCheck(cudaGraphInstantiate(&exec, graph, 0), "cudaGraphInstantiate");
      cudaGraphDestroy(graph);
      if (st)
        return st;
      it = p->graphs.emplace(phase, exec).first;
    }
    st = cudaCheck(cudaGraphLaunch(it->second, s), "cudaGraphLaunch");
    if (st)
      return st;
    for (int t = 0; t < G; ++t) { // the host-side rotation the graph's steps performed
      std::vector<int> nxt(p->bind.size());
      for (size_t i = 0; i < p->bind.size(); ++i)
        nxt[i] = p->bind[static_cast<size_t>(p->an.src[i])];
      p->bind.swap(nxt);
    }
    p->stepsDone += G;
    p->launches += G;
    steps -= G;
  }
  for (int64_t t = 0; t < steps; ++t) {
    st = planStep(*p, s);
    if (st)
      return st;
  }
  return HG_OK;
}

int hg_plan_binding(const hg_plan *p, int32_t *perm, int64_t *steps_done) {
  if (!p)
    return setError(HG_EINVAL, "null plan");
  if (perm)
    for (size_t i = 0; i < p->bind.size(); ++i)
      perm[i] = p->bind[i];
  if (steps_done)
    *steps_done = p->stepsDone;
  return HG_OK;
}

int hg_plan_reset_binding(hg_plan *p) {
  if (!p)
    return setError(HG_EINVAL, "null plan");
  for (size_t i = 0; i < p->bind.size(); ++i)
    p->bind[i] = static_cast<int>(i);
  p->stepsDone = 0;
  return HG_OK;
}

static int packImpl(hg_plan *p, int b, const int64_t *at, const int64_t *size, void *dev,
                    void *stream, int unpack) {
  if (!p || b < 0 || b >= static_cast<int>(p->lay.size()) || !at || !size || !dev)
    return setError(HG_EINVAL, "bad pack arguments");
  const Layout &L = p->lay[static_cast<size_t>(b)];
  for (int d = 0; d < L.rank; ++d)
    if (at[d] < 0 || size[d] < 0 || at[d] + size[d] > L.shape[d])
      return setError(HG_ETRAP, "exchange region escapes the buffer");
  int st = cudaCheck(cudaSetDevice(p->device), "cudaSetDevice");
  if (st)
    return st;
  ++p->launches;
  return launchPackUnpack(p->dptr[static_cast<size_t>(b)], devLayout(L), at, size, dev, unpack,
                          static_cast<cudaStream_t>(stream));
}

int hg_plan_pack(hg_plan *p, int b, const int64_t *at, const int64_t *size, void *dst,
                 void *stream) {
  return packImpl(p, b, at, size, dst, stream, 0);
}

int hg_plan_unpack(hg_plan *p, int b, const int64_t *at, const int64_t *size, const void *src,
                   void *stream) {
  if (p && b >= 0 && b < static_cast<int>(p->shadowOk.size()))
    p->shadowOk[static_cast<size_t>(b)] = 0;
  return packImpl(p, b, at, size, const_cast<void *>(src), stream, 1);
}

int64_t hg_plan_launch_count(const hg_plan *p) { return p ? p->launches : 0; }

int hg_plan_bind(hg_plan *p, int b, void *dptr, size_t bytes) {
  HG_GUARD_BEGIN
  if (!p || !dptr || b < 0 || b >= static_cast<int>(p->dptr.size()))
    return setError(HG_EINVAL, "bad plan/buffer/pointer");
  const Layout &L = p->lay[static_cast<size_t>(b)];
  if (bytes < L.bytes())
    return setError(HG_EINVAL, "bound memory is smaller than the buffer's layout (" +
                                   std::to_string(L.bytes()) + " bytes; hg_plan_layout)");
  if (reinterpret_cast<uintptr_t>(dptr) % 128 != 0)
    return setError(HG_EINVAL, "bound memory must be 128-byte aligned (the layout starts every "
                               "core row on a 128-byte line)");
  if (int st = cudaCheck(cudaSetDevice(p->device), "cudaSetDevice"))
    return st;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, dptr) != cudaSuccess || at.type != cudaMemoryTypeDevice ||
      at.device != p->device) {
    cudaGetLastError();
    return setError(HG_EINVAL, "bound memory must be device memory of the plan's device");
  }
  if (int st = cudaCheck(cudaDeviceSynchronize(), "cudaDeviceSynchronize"))
    return st;
  const size_t bi = static_cast<size_t>(b);
  p->callerOwned.resize(p->dptr.size(), 0);
  if (!p->callerOwned[bi])
    planFree(*p, p->dptr[bi]);
  p->dptr[bi] = dptr;
  p->callerOwned[bi] = 1;
  p->tbOff = true; // two-step passes swap buffers with plan-owned shadows
  // every descriptor that captured the old address
  for (auto &g : p->graphs)
    cudaGraphExecDestroy(g.second);
  p->graphs.clear();
  const hg_program &g = p->prog;
  if (p->an.family == Family::Star && bi < p->tmCur.size())
    if (int st = makeStarTensorMaps(p->an.star, g.dtype, g.rank, devLayout(L), dptr,
                                    &p->tmCur[bi], &p->tmPrev[bi], p->starGeo))
      return st;
  if (p->jit && bi < p->tmApply.size())
    if (int st = jitTensorMap(*p->jit, g.dtype, g.rank, L, dptr, &p->tmApply[bi]))
      return st;
  for (auto &M : p->multi)
    if (M.jit && bi < M.tmField.size())
      if (int st = jitTensorMap(*M.jit, g.dtype, g.rank, L, dptr, &M.tmField[bi]))
        return st;
  return HG_OK;
  HG_GUARD_END
}

int hg_plan_synchronize(hg_plan *p) {
  if (!p)
    return setError(HG_EINVAL, "null plan");
  int st = cudaCheck(cudaSetDevice(p->device), "cudaSetDevice");
  if (st)
    return st;
  return cudaCheck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
}

int hg_plan_set_tuning(hg_plan *p, int chunks, int boundary_last) {
  if (!p || chunks < 0)
    return setError(HG_EINVAL, "bad tuning");
  p->chunks = chunks;
  p->boundaryLast = boundary_last ? 1 : 0;
  for (auto &g : p->graphs) // captured with the old launch shape
    cudaGraphExecDestroy(g.second);
  p->graphs.clear();
  return HG_OK;
}

} // extern "C"
