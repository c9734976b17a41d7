// program.cpp -- host-side algorithms of the path: program building, validation, kernel-family
// matching, decomposition arithmetic, initializer/fingerprint, binding rotation.
// Every function restates (not copies) the reference routine cited beside it; paths are
// under /root/reference/proj/core.
#include "hg_internal.hpp"

#include <algorithm>
#include <array>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <numeric>
#include <string>

namespace hg {

namespace {
thread_local std::string g_last_error;
}

int setError(int status, const std::string &msg) {
  g_last_error = msg;
  return status;
}

uint64_t fnv1a(const void *p, size_t n) {
  // exec::fingerprint, buffer.cpp:181-188
  const auto *c = static_cast<const unsigned char *>(p);
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= c[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

Layout makeLayout(const hg_bounds &b, int rank, int es, int64_t core_lb_last, int padLines) {
  // Reference layout is row-major with the last dim fastest (buffer.cpp:65-70).  On the
  // device each row of the last dim is padded to a 128-byte pitch and shifted so that the
  // first core element of a row starts a 128-byte line (coalesced, TMA-legal strides).
  Layout L;
  L.rank = rank;
  L.es = es;
  for (int d = 0; d < rank; ++d) {
    L.shape[d] = b.ub[d] - b.lb[d];
    L.lb[d] = b.lb[d];
  }
  const int64_t va = 128 / es;
  int64_t S = L.shape[rank - 1];
  int64_t j0 = core_lb_last - b.lb[rank - 1];
  if (j0 < 0 || j0 >= S)
    j0 = 0;
  L.col0 = va * ((j0 + 8 + va - 1) / va) - j0;
  int64_t lines = (L.col0 + S + va - 1) / va;
  // Row strides of a multiple of 17 lines of 128 B (1088 floats, 1632, 2176, ...) make the
  // star kernel's concurrent plane reads collide in the memory system: heat SDO4 1024^3 runs
  // at 705 GPts/s with 34 lines per row and 752-758 with 35 or 36, and the 51- and 68-line
  // rows lose 4-7% the same way, while 33/35/36/50/52/66 are all fine (tools/pitch_ab2.py,
  // profiles/r2_pitch.md).  One more line breaks the period.
  if (lines % 17 == 0)
    ++lines;
  L.pitch = (lines + std::max(padLines, 0)) * va;
  L.rows = 1;
  for (int d = 0; d < rank - 1; ++d)
    L.rows *= L.shape[d];
  return L;
}

namespace {

bool boundsEqual(const hg_bounds &a, const hg_bounds &b, int rank) {
  for (int d = 0; d < rank; ++d)
    if (a.lb[d] != b.lb[d] || a.ub[d] != b.ub[d])
      return false;
  return true;
}

int gcdInt(int a, int b) { return b == 0 ? a : gcdInt(b, a % b); }

// ---- star-family matcher -------------------------------------------------------------------
struct Matcher {
  const hg_program &p;
  int rank;
  explicit Matcher(const hg_program &prog) : p(prog), rank(prog.rank) {}

  const hg_op &op(int i) const { return p.ops[i]; }
  bool isConst(int i) const { return op(i).code == HG_OP_CONST; }
  bool isAccess(int i, int operand, const int64_t *off) const {
    const hg_op &o = op(i);
    if (o.code != HG_OP_ACCESS || (operand >= 0 && o.operand != operand))
      return false;
    for (int d = 0; d < rank; ++d)
      if (o.off[d] != off[d])
        return false;
    return true;
  }
  bool isCenter(int i, int operand) const {
    int64_t z[3] = {0, 0, 0};
    return isAccess(i, operand, z);
  }
  // mul(x, const) in either operand order -> x, const
  bool mulByConst(int i, int &x, uint64_t &c) const {
    const hg_op &o = op(i);
    if (o.code != HG_OP_MUL)
      return false;
    if (isConst(o.b)) {
      x = o.a;
      c = op(o.b).bits;
      return true;
    }
    if (isConst(o.a)) {
      x = o.b;
      c = op(o.a).bits;
      return true;
    }
    return false;
  }
  // term: mul(add(access(+k e_d), access(-k e_d)), const w)
  bool term(int i, int operand, int &d, int64_t &k, uint64_t &w) const {
    int s;
    if (!mulByConst(i, s, w))
      return false;
    const hg_op &a = op(s);
    if (a.code != HG_OP_ADD)
      return false;
    const hg_op &x = op(a.a), &y = op(a.b);
    if (x.code != HG_OP_ACCESS || y.code != HG_OP_ACCESS || x.operand != operand ||
        y.operand != operand)
      return false;
    int nz = -1;
    for (int q = 0; q < rank; ++q) {
      if (x.off[q] != -y.off[q])
        return false;
      if (x.off[q] != 0) {
        if (nz >= 0)
          return false;
        nz = q;
      }
    }
    if (nz < 0)
      return false;
    d = nz;
    k = x.off[nz] < 0 ? -x.off[nz] : x.off[nz];
    return true;
  }
  // lap chain; fills spec weights.  Center must be `operand` at zero offset.
  bool lap(int i, int operand, StarSpec &s) const {
    struct T {
      int d;
      int64_t k;
      uint64_t w;
    };
    std::vector<T> terms;
    int node = i;
    for (int guard = 0; guard < 64; ++guard) {
      const hg_op &o = op(node);
      int d;
      int64_t k;
      uint64_t w;
      if (o.code == HG_OP_ADD) {
        bool tb = term(o.b, operand, d, k, w);
        if (tb && !term(o.a, operand, d, k, w)) {
          term(o.b, operand, d, k, w);
          terms.push_back({d, k, w});
          node = o.a;
          continue;
        }
        if (!tb && term(o.a, operand, d, k, w)) {
          terms.push_back({d, k, w});
          node = o.b;
          continue;
        }
        return false;
      }
      int x;
      uint64_t c;
      if (!mulByConst(node, x, c) || !isCenter(x, operand))
        return false;
      s.w0 = c;
      break;
    }
    if (terms.empty())
      return false;
    std::vector<T> fwd(terms.rbegin(), terms.rend());
    static const int64_t tapsets[3][3] = {{1, 0, 0}, {1, 2, 0}, {1, 2, 4}};
    for (int nt = 1; nt <= 3; ++nt) {
      if (static_cast<int>(fwd.size()) != nt * rank)
        continue;
      bool ok = true;
      for (int d = 0; d < rank && ok; ++d)
        for (int j = 0; j < nt && ok; ++j) {
          const T &t = fwd[static_cast<size_t>(d * nt + j)];
          if (t.d != d || t.k != tapsets[nt - 1][j])
            ok = false;
          else
            s.w[d][j] = t.w;
        }
      if (ok) {
        s.ntaps = nt;
        s.radius = static_cast<int>(tapsets[nt - 1][nt - 1]);
        return true;
      }
    }
    return false;
  }

  bool match(StarSpec &s) const {
    if (p.nresults != 1)
      return false;
    int root = p.result_op[0];
    s.rank = rank;
    if (isCenter(root, -1)) {
      s.kind = kCopy;
      s.cur_operand = op(root).operand;
      s.radius = 0;
      s.ntaps = 0;
      return true;
    }
    const hg_op &r = op(root);
    if (r.code != HG_OP_ADD)
      return false;
    for (int flip = 0; flip < 2; ++flip) {
      int x = flip ? r.b : r.a, y = flip ? r.a : r.b;
      int l;
      uint64_t sc;
      if (!mulByConst(y, l, sc))
        continue;
      // heat: c + lap*S
      if (op(x).code == HG_OP_ACCESS && isCenter(x, op(x).operand)) {
        StarSpec t;
        t.rank = rank;
        t.kind = kHeat;
        t.cur_operand = op(x).operand;
        t.scale = sc;
        if (lap(l, t.cur_operand, t)) {
          s = t;
          return true;
        }
      }
      // wave: (cur*K2 - prev) + lap(cur)*S
      if (op(x).code == HG_OP_SUB) {
        const hg_op &sb = op(x);
        int cm;
        uint64_t k2;
        if (!mulByConst(sb.a, cm, k2) || op(cm).code != HG_OP_ACCESS ||
            !isCenter(cm, op(cm).operand) || op(sb.b).code != HG_OP_ACCESS ||
            !isCenter(sb.b, op(sb.b).operand))
          continue;
        StarSpec t;
        t.rank = rank;
        t.kind = kWave;
        t.cur_operand = op(cm).operand;
        t.prev_operand = op(sb.b).operand;
        t.two = k2;
        t.scale = sc;
        if (t.prev_operand != t.cur_operand && lap(l, t.cur_operand, t)) {
          s = t;
          return true;
        }
      }
    }
    return false;
  }
};

} // namespace

namespace {

// Multi-apply steps (hg_apply list): operands are fields or earlier temps, regions are op
// slices, every access stays inside its operand over the apply's domain, stores copy temps.
int validateMulti(const hg_program &p) {
  if (p.napplies > HG_MAX_APPLIES || !p.applies)
    return setError(HG_EINVAL, "apply count out of range");
  if (p.ntemps < 1 || p.ntemps > HG_MAX_TEMPS)
    return setError(HG_EINVAL, "temp count out of range");
  if (p.nstores < 1 || p.nstores > HG_MAX_STORES)
    return setError(HG_EINVAL, "store count out of range");
  if (p.noperands < 0 || p.noperands > HG_MAX_FIELDS)
    return setError(HG_EINVAL, "load count out of range");
  for (int o = 0; o < p.noperands; ++o)
    if (p.operand_field[o] < 0 || p.operand_field[o] >= p.nfields)
      return setError(HG_EINVAL, "stencil.load of a missing field");
  std::vector<int> defined(static_cast<size_t>(p.ntemps), -1); // temp -> defining apply
  for (int a = 0; a < p.napplies; ++a) {
    const hg_apply &A = p.applies[a];
    const std::string where = " (apply " + std::to_string(a) + ")";
    if (A.noperands < 0 || A.noperands > HG_MAX_FIELDS || A.nresults < 1 ||
        A.nresults > HG_MAX_RESULTS || A.nops < 1 || A.op_begin < 0 ||
        A.op_begin + A.nops > p.nops)
      return setError(HG_EINVAL, "malformed apply" + where);
    for (int d = 0; d < p.rank; ++d)
      if (A.domain.lb[d] >= A.domain.ub[d])
        return setError(HG_EINVAL, "unresolved or empty stencil.apply bounds" + where);
    for (int o = 0; o < A.noperands; ++o) {
      const int x = A.operand[o];
      if (x >= 0 ? x >= p.nfields : (-x - 1 >= p.ntemps || defined[static_cast<size_t>(-x - 1)] < 0))
        return setError(HG_EINVAL, "apply operand is neither a loaded field nor an earlier "
                                   "apply result" + where);
    }
    const hg_op *ops = p.ops + A.op_begin;
    for (int i = 0; i < A.nops; ++i) {
      const hg_op &o = ops[i];
      if (o.code == HG_OP_ACCESS) {
        if (o.operand < 0 || o.operand >= A.noperands)
          return setError(HG_EINVAL, "stencil.access of a missing apply operand" + where);
        const int x = A.operand[o.operand];
        const hg_bounds &b = x >= 0 ? p.fields[x]
                                    : p.applies[defined[static_cast<size_t>(-x - 1)]].domain;
        for (int d = 0; d < p.rank; ++d)
          if (A.domain.lb[d] + o.off[d] < b.lb[d] || A.domain.ub[d] + o.off[d] > b.ub[d])
            return setError(HG_ETRAP, "stencil access escapes the value bounds" + where);
      } else if (o.code >= HG_OP_ADD && o.code <= HG_OP_DIV) {
        if (o.a < 0 || o.a >= i || o.b < 0 || o.b >= i)
          return setError(HG_EINVAL, "use before def in the apply region" + where);
      } else if (o.code != HG_OP_CONST) {
        return setError(HG_EINVAL, "unknown op code" + where);
      }
    }
    for (int k = 0; k < A.nresults; ++k) {
      const int t = A.result_temp[k];
      if (A.result_op[k] < 0 || A.result_op[k] >= A.nops || t < 0 || t >= p.ntemps ||
          defined[static_cast<size_t>(t)] >= 0)
        return setError(HG_EINVAL, "malformed apply results" + where);
      defined[static_cast<size_t>(t)] = a;
    }
  }
  for (int k = 0; k < p.nstores; ++k) {
    const int t = p.mstore_temp[k], f = p.mstore_field[k];
    if (t < 0 || t >= p.ntemps || defined[static_cast<size_t>(t)] < 0 || f < 0 || f >= p.nfields)
      return setError(HG_EINVAL, "stencil.store of an undefined temp or into a missing field");
    const hg_bounds &dom = p.applies[defined[static_cast<size_t>(t)]].domain;
    for (int d = 0; d < p.rank; ++d) {
      if (p.mstore[k].lb[d] >= p.mstore[k].ub[d])
        return setError(HG_EINVAL, "empty store region");
      if (p.mstore[k].lb[d] < p.fields[f].lb[d] || p.mstore[k].ub[d] > p.fields[f].ub[d] ||
          p.mstore[k].lb[d] < dom.lb[d] || p.mstore[k].ub[d] > dom.ub[d])
        return setError(HG_ETRAP, "store region escapes the field bounds");
    }
  }
  return HG_OK;
}

} // namespace

int validateProgram(const hg_program &p) {
  if (p.rank < 1 || p.rank > HG_MAX_RANK)
    return setError(HG_EINVAL, "program rank must be 1, 2, or 3");
  if (p.dtype != HG_F32 && p.dtype != HG_F64)
    return setError(HG_EINVAL, "program dtype must be f32 or f64");
  if (p.nfields < 1 || p.nfields > HG_MAX_FIELDS)
    return setError(HG_EINVAL, "field count out of range");
  if (p.napplies > 0) {
    if (p.nops < 1 || p.nops > HG_MAX_OPS || !p.ops)
      return setError(HG_EINVAL, "apply region op count out of range");
    for (int f = 0; f < p.nfields; ++f)
      for (int d = 0; d < p.rank; ++d)
        if (p.fields[f].lb[d] >= p.fields[f].ub[d])
          return setError(HG_EINVAL, "field " + std::to_string(f) + " has empty bounds");
    int st = validateMulti(p);
    if (st)
      return st;
    goto time_slots;
  }
  if (p.noperands < 0 || p.noperands > HG_MAX_FIELDS)
    return setError(HG_EINVAL, "apply operand count out of range");
  if (p.nops < 1 || p.nops > HG_MAX_OPS || !p.ops)
    return setError(HG_EINVAL, "apply region op count out of range");
  if (p.nresults < 1 || p.nresults > HG_MAX_RESULTS)
    return setError(HG_EINVAL, "apply result count out of range");
  for (int f = 0; f < p.nfields; ++f)
    for (int d = 0; d < p.rank; ++d)
      if (p.fields[f].lb[d] >= p.fields[f].ub[d])
        return setError(HG_EINVAL, "field " + std::to_string(f) + " has empty bounds");
  for (int o = 0; o < p.noperands; ++o)
    if (p.operand_field[o] < 0 || p.operand_field[o] >= p.nfields)
      return setError(HG_EINVAL, "apply operand loads a missing field");
  for (int i = 0; i < p.nops; ++i) {
    const hg_op &o = p.ops[i];
    switch (o.code) {
    case HG_OP_ACCESS:
      if (o.operand < 0 || o.operand >= p.noperands)
        return setError(HG_EINVAL, "stencil.access of a missing apply operand");
      break;
    case HG_OP_CONST:
      break;
    case HG_OP_ADD:
    case HG_OP_SUB:
    case HG_OP_MUL:
    case HG_OP_DIV:
      if (o.a < 0 || o.a >= i || o.b < 0 || o.b >= i)
        return setError(HG_EINVAL, "use before def in the apply region (op " +
                                       std::to_string(i) + ")");
      break;
    default:
      return setError(HG_EINVAL, "unknown op code " + std::to_string(o.code));
    }
  }
  for (int k = 0; k < p.nresults; ++k) {
    if (p.result_op[k] < 0 || p.result_op[k] >= p.nops)
      return setError(HG_EINVAL, "stencil.return of an undefined value");
    int f = p.store_field[k];
    if (f < 0 || f >= p.nfields)
      return setError(HG_EINVAL, "stencil.store to a missing field");
    for (int d = 0; d < p.rank; ++d) {
      if (p.store[k].lb[d] >= p.store[k].ub[d])
        return setError(HG_EINVAL, "empty store region");
      if (p.store[k].lb[d] < p.fields[f].lb[d] || p.store[k].ub[d] > p.fields[f].ub[d])
        return setError(HG_ETRAP, "store region escapes the field bounds");
    }
  }
  // time slots: stencil_transforms.cpp:196-230
time_slots : {
    bool seen[HG_MAX_FIELDS] = {};
    int at = 0;
    if (p.ngroups < 0 || p.ngroups > HG_MAX_FIELDS)
      return setError(HG_EINVAL, "stencil.time_slots must be a list of index lists");
    for (int g = 0; g < p.ngroups; ++g) {
      if (p.group_len[g] < 1 || at + p.group_len[g] > HG_MAX_FIELDS)
        return setError(HG_EINVAL, "stencil.time_slots must be a list of index lists");
      for (int j = 0; j < p.group_len[g]; ++j) {
        int i = p.groups[at + j];
        if (i < 0 || i >= p.nfields || seen[i])
          return setError(HG_EINVAL, "stencil.time_slots holds an out-of-range or repeated "
                                     "argument index");
        seen[i] = true;
      }
      at += p.group_len[g];
    }
  }
  return HG_OK;
}

Knobs readKnobs() {
  auto on = [](const char *n) {
    const char *e = std::getenv(n);
    return e && e[0] && e[0] != '0';
  };
  auto num = [](const char *n, int dflt) {
    const char *e = std::getenv(n);
    return e && e[0] ? std::atoi(e) : dflt;
  };
  Knobs k;
  k.noStar = on("HG_NO_STAR");
  k.noApplyJit = on("HG_NO_APPLY_JIT");
  k.noFuseApplies = on("HG_NO_FUSE_APPLIES");
  k.noResident = on("HG_NO_RESIDENT");
  k.tb = on("HG_TB");
  k.starGeo = num("HG_STAR_GEO", -1);
  k.jitDepth = std::max(0, num("HG_JIT_DEPTH", 0));
  k.jitPersist = num("HG_JIT_PERSIST", 1) != 0;
  k.jitPack = num("HG_JIT_PACK", 0) != 0;
  k.guards = on("HG_DEBUG_GUARDS");
  k.pitchPad = std::max(0, num("HG_PITCH_PAD", 0));
  return k;
}

int analyze(const hg_program &p, Analysis &a, bool allowStar) {
  int st = validateProgram(p);
  if (st)
    return st;
  if (p.napplies > 0) {
    // rotation + a generic launch per apply (temps materialised over their domains)
    for (int k = 0; k < p.nstores; ++k)
      for (int a2 = 0; a2 < p.napplies; ++a2)
        for (int o = 0; o < p.applies[a2].noperands; ++o)
          if (p.applies[a2].operand[o] == p.mstore_field[k])
            return setError(HG_EUNSUPPORTED,
                            "stencil.store into a field the step loads (in-place update) is not "
                            "supported by the device path");
    a.src.assign(static_cast<size_t>(p.nfields), 0);
    for (int i = 0; i < p.nfields; ++i)
      a.src[static_cast<size_t>(i)] = i;
    int at = 0;
    a.period = 1;
    for (int g = 0; g < p.ngroups; ++g) {
      for (int j = 0; j < p.group_len[g]; ++j)
        a.src[static_cast<size_t>(p.groups[at + j])] = p.groups[at + (j + 1) % p.group_len[g]];
      a.period = a.period / gcdInt(a.period, p.group_len[g]) * p.group_len[g];
      at += p.group_len[g];
    }
    for (int d = 0; d < p.rank; ++d) {
      a.dom_lb[d] = p.applies[0].domain.lb[d];
      a.dom_ub[d] = p.applies[0].domain.ub[d];
    }
    a.family = Family::Multi;
    a.name = "multi" + std::to_string(p.napplies) + "x_generic" + std::to_string(p.rank) + "d_" +
             (p.dtype == HG_F32 ? "f32" : "f64");
    return HG_OK;
  }
  // apply domain = hull of the store regions
  for (int d = 0; d < p.rank; ++d) {
    a.dom_lb[d] = p.store[0].lb[d];
    a.dom_ub[d] = p.store[0].ub[d];
    for (int k = 1; k < p.nresults; ++k) {
      a.dom_lb[d] = std::min(a.dom_lb[d], p.store[k].lb[d]);
      a.dom_ub[d] = std::max(a.dom_ub[d], p.store[k].ub[d]);
    }
  }
  // every access stays inside its operand's field over the whole domain (interpreter traps
  // at run time, interpreter.cpp:767-769; we refuse the plan instead)
  for (int i = 0; i < p.nops; ++i) {
    const hg_op &o = p.ops[i];
    if (o.code != HG_OP_ACCESS)
      continue;
    const hg_bounds &fb = p.fields[p.operand_field[o.operand]];
    for (int d = 0; d < p.rank; ++d)
      if (a.dom_lb[d] + o.off[d] < fb.lb[d] || a.dom_ub[d] + o.off[d] > fb.ub[d])
        return setError(HG_ETRAP, "stencil access escapes the value bounds (op " +
                                      std::to_string(i) + ")");
  }
  // value semantics of stencil.load (a clone) vs an in-place store
  for (int k = 0; k < p.nresults; ++k)
    for (int o = 0; o < p.noperands; ++o)
      if (p.store_field[k] == p.operand_field[o])
        return setError(HG_EUNSUPPORTED,
                        "stencil.store into a field the same apply loads (in-place update) "
                        "is not supported by the device path");
  for (int k = 0; k < p.nresults; ++k)
    for (int j = 0; j < k; ++j)
      if (p.store_field[k] == p.store_field[j])
        return setError(HG_EUNSUPPORTED, "two stores into one field");
  // rotation
  a.src.assign(static_cast<size_t>(p.nfields), 0);
  for (int i = 0; i < p.nfields; ++i)
    a.src[static_cast<size_t>(i)] = i;
  int at = 0;
  a.period = 1;
  for (int g = 0; g < p.ngroups; ++g) {
    for (int j = 0; j < p.group_len[g]; ++j)
      a.src[static_cast<size_t>(p.groups[at + j])] = p.groups[at + (j + 1) % p.group_len[g]];
    a.period = a.period / gcdInt(a.period, p.group_len[g]) * p.group_len[g];
    at += p.group_len[g];
  }
  // family
  a.family = Family::Generic;
  const char *dt = p.dtype == HG_F32 ? "f32" : "f64";
  StarSpec s;
  bool sameBounds = true;
  for (int f = 1; f < p.nfields; ++f)
    if (!boundsEqual(p.fields[f], p.fields[0], p.rank))
      sameBounds = false;
  // HG_NO_STAR (tests only) routes star programs through the fused-apply family
  if (p.rank >= 2 && sameBounds && allowStar && Matcher(p).match(s)) {
    a.family = Family::Star;
    a.star = s;
    static const char *kinds[] = {"heat", "wave", "copy"};
    a.name = "star" + std::to_string(p.rank) + "d_r" + std::to_string(s.radius) + "_" +
             kinds[s.kind] + "_" + dt;
  } else {
    a.name = "generic" + std::to_string(p.rank) + "d_" + dt;
  }
  return HG_OK;
}

} // namespace hg

using namespace hg;

extern "C" {

const char *hg_last_error(void) { return g_last_error.c_str(); }

int hg_version(void) { return 10000; }

// exec::initValue (buffer.cpp:142-156)
static inline uint64_t mix64h(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

double hg_init_value(int field_idx, int rank, const int64_t *coord) {
  uint64_t h = mix64h(static_cast<uint64_t>(field_idx) + 1);
  for (int d = 0; d < rank; ++d)
    h = mix64h(h ^ static_cast<uint64_t>(coord[d]));
  return static_cast<double>(h >> 11) * 0x1.0p-53;
}

uint64_t hg_fingerprint(const void *bytes, size_t n) { return fnv1a(bytes, n); }

int hg_binding_after(int ngroups, const int32_t *group_len, const int32_t *groups, int nargs,
                     int64_t steps, int32_t *out) {
  // rotationSources (stencil_transforms.cpp:233-242) + bindingAfter (serial.cpp:42-55)
  if (nargs < 0 || nargs > HG_MAX_FIELDS)
    return setError(HG_EINVAL, "argument count out of range");
  int src[HG_MAX_FIELDS], cur[HG_MAX_FIELDS], nxt[HG_MAX_FIELDS];
  for (int i = 0; i < nargs; ++i)
    src[i] = cur[i] = i;
  int at = 0;
  int period = 1;
  for (int g = 0; g < ngroups; ++g) {
    for (int j = 0; j < group_len[g]; ++j) {
      int i = groups[at + j];
      if (i < 0 || i >= nargs)
        return setError(HG_EINVAL, "group index out of range");
      src[i] = groups[at + (j + 1) % group_len[g]];
    }
    period = period / gcdInt(period, group_len[g]) * group_len[g];
    at += group_len[g];
  }
  int64_t n = steps % period; // the rotation is periodic
  for (int64_t t = 0; t < n; ++t) {
    for (int i = 0; i < nargs; ++i)
      nxt[i] = cur[src[i]];
    std::memcpy(cur, nxt, sizeof(int) * static_cast<size_t>(nargs));
  }
  for (int i = 0; i < nargs; ++i)
    out[i] = cur[i];
  return HG_OK;
}

double hg_gpts_per_sec(int64_t core_points, int64_t steps, double seconds) {
  // exec::gptsPerSec (throughput.cpp:19-23)
  return static_cast<double>(core_points) * static_cast<double>(steps) / seconds / 1e9;
}

// ir::dmp grid arithmetic (dmp_ops.cpp:21-49): row-major, last dim fastest, no wrap
int64_t hg_rank_from_coord(int n, const int64_t *coord, const int64_t *grid) {
  int64_t r = 0;
  for (int d = 0; d < n; ++d)
    r = r * grid[d] + coord[d];
  return r;
}

void hg_coord_from_rank(int n, int64_t rank, const int64_t *grid, int64_t *coord) {
  for (int d = n - 1; d >= 0; --d) {
    coord[d] = rank % grid[d];
    rank /= grid[d];
  }
}

int64_t hg_neighbor_rank(int n, int64_t rank, const int64_t *dir, const int64_t *grid) {
  int64_t c[HG_MAX_RANK];
  hg_coord_from_rank(n, rank, grid, c);
  for (int d = 0; d < n; ++d) {
    c[d] += dir[d];
    if (c[d] < 0 || c[d] >= grid[d])
      return -1;
  }
  return hg_rank_from_coord(n, c, grid);
}

void hg_local_interval(int64_t extent, int64_t parts, int64_t part, int64_t *lb, int64_t *ub) {
  // StandardSlicing::localInterval (dmp_ops.cpp:107-115): remainder to the leading parts
  int64_t base = extent / parts, rem = extent % parts;
  *lb = part * base + std::min(part, rem);
  *ub = *lb + base + (part < rem ? 1 : 0);
}

int hg_exchanges(int n, const int64_t *core, const int64_t *below, const int64_t *above,
                 const int64_t *grid, const int64_t *coord, hg_exchange *out, int cap) {
  // DecompositionStrategy::exchanges (dmp_ops.cpp:63-105): faces only, dimension-major,
  // negative direction first; `at` = receive box, send box = at + offset.
  int k = 0;
  for (int d = 0; d < n; ++d) {
    for (int sign : {-1, +1}) {
      int64_t width = sign < 0 ? below[d] : above[d];
      if (width == 0)
        continue;
      if (coord && grid) {
        int64_t dir[HG_MAX_RANK] = {0, 0, 0};
        dir[d] = sign;
        if (hg_neighbor_rank(n, hg_rank_from_coord(n, coord, grid), dir, grid) < 0)
          continue;
      }
      hg_exchange e;
      std::memset(&e, 0, sizeof e);
      for (int q = 0; q < n; ++q) {
        e.at[q] = below[q];
        e.size[q] = core[q];
      }
      e.size[d] = width;
      if (sign < 0) {
        e.at[d] = 0;
        e.offset[d] = width;
      } else {
        e.at[d] = below[d] + core[d];
        e.offset[d] = -width;
      }
      e.to[d] = sign;
      if (k < cap)
        out[k] = e;
      ++k;
    }
  }
  return k;
}

// ---- exec::buildKernel (kernels.cpp:139-243) -----------------------------------------------
static std::vector<int64_t> laplacianTaps(int order) {
  switch (order) { // kernels.cpp:35-47
  case 2: return {1};
  case 4: return {1, 2};
  case 8: return {1, 2, 4};
  default: return {};
  }
}

static double laplacianWeight(int order, int64_t k) {
  // kernels.cpp:49-81 -- central-difference weights, the +/-k pair shares one weight
  if (order == 2) return k == 0 ? -2.0 : (k == 1 ? 1.0 : 0.0);
  if (order == 4) return k == 0 ? -5.0 / 2.0 : k == 1 ? 4.0 / 3.0 : k == 2 ? -1.0 / 12.0 : 0.0;
  if (order == 8)
    return k == 0   ? -21.0 / 8.0
           : k == 1 ? 64.0 / 45.0
           : k == 2 ? -1.0 / 9.0
           : k == 4 ? 1.0 / 720.0
                    : 0.0;
  return 0.0;
}

// The constant as the f32-retyped module carries it: the f64 printed as its shortest
// round-trip decimal (formatFloatToken, attributes.cpp:69-80) and re-read with
// from_chars<float> (parser.cpp:392-398).
static uint64_t constBits(double v, int dtype) {
  if (dtype == HG_F64) {
    uint64_t b;
    std::memcpy(&b, &v, 8);
    return b;
  }
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  float f = 0.0f;
  std::from_chars(buf, r.ptr, f);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}

int hg_build_kernel_program(const char *kind_c, int rank, int64_t extent, int order, int dtype,
                            hg_program *prog, hg_op *ops, int cap_ops) {
  std::string kind = kind_c ? kind_c : "";
  if (kind != "heat" && kind != "wave" && kind != "copy")
    return setError(HG_EINVAL, "unknown kernel '" + kind + "'");
  if (rank < 1 || rank > 3)
    return setError(HG_EINVAL, "kernel rank must be 1, 2, or 3");
  if (extent <= 0)
    return setError(HG_EINVAL, "kernel extent must be positive");
  auto taps = laplacianTaps(order);
  if (kind != "copy" && taps.empty())
    return setError(HG_EINVAL, "Laplacian order must be 2, 4, or 8");
  if (dtype != HG_F32 && dtype != HG_F64)
    return setError(HG_EINVAL, "dtype must be f32 or f64");
  int64_t h = kind == "copy" ? 0 : taps.back();
  std::vector<hg_op> v;
  auto push = [&](hg_op o) {
    v.push_back(o);
    return static_cast<int>(v.size()) - 1;
  };
  auto cst = [&](double x) {
    hg_op o{};
    o.code = HG_OP_CONST;
    o.bits = constBits(x, dtype);
    return push(o);
  };
  auto acc = [&](int operand, const int64_t *off) {
    hg_op o{};
    o.code = HG_OP_ACCESS;
    o.operand = operand;
    for (int d = 0; d < rank; ++d)
      o.off[d] = off[d];
    return push(o);
  };
  auto bin = [&](int code, int a, int b) {
    hg_op o{};
    o.code = code;
    o.a = a;
    o.b = b;
    return push(o);
  };
  // emitLaplacian (kernels.cpp:110-135); arith.constant is emitted before its user
  auto lap = [&](int operand, int center) {
    int c0 = cst(laplacianWeight(order, 0) * rank);
    int a = bin(HG_OP_MUL, center, c0);
    for (int d = 0; d < rank; ++d)
      for (int64_t k : taps) {
        int64_t off[3] = {0, 0, 0};
        off[d] = k;
        int pp = acc(operand, off);
        off[d] = -k;
        int mm = acc(operand, off);
        int s = bin(HG_OP_ADD, pp, mm);
        int w = cst(laplacianWeight(order, k));
        int ww = bin(HG_OP_MUL, s, w);
        a = bin(HG_OP_ADD, a, ww);
      }
    return a;
  };
  int64_t zero[3] = {0, 0, 0};
  int numFields = kind == "wave" ? 3 : 2;
  int out;
  if (kind == "copy") {
    out = acc(0, zero);
  } else if (kind == "heat") {
    int c = acc(0, zero);
    int l = lap(0, c);
    int sc = bin(HG_OP_MUL, l, cst(0.01));
    out = bin(HG_OP_ADD, c, sc);
  } else {
    int prev = acc(0, zero);
    int cur = acc(1, zero);
    int l = lap(1, cur);
    int two = bin(HG_OP_MUL, cur, cst(2.0));
    int sub = bin(HG_OP_SUB, two, prev);
    int kk = bin(HG_OP_MUL, l, cst(0.01));
    out = bin(HG_OP_ADD, sub, kk);
  }
  if (static_cast<int>(v.size()) > cap_ops)
    return setError(HG_EINVAL, "op buffer too small (" + std::to_string(v.size()) + " ops)");
  std::memcpy(ops, v.data(), v.size() * sizeof(hg_op));
  hg_program &p = *prog;
  std::memset(&p, 0, sizeof p);
  p.rank = rank;
  p.dtype = dtype;
  p.nfields = numFields;
  for (int f = 0; f < numFields; ++f)
    for (int d = 0; d < rank; ++d) {
      p.fields[f].lb[d] = -h;
      p.fields[f].ub[d] = extent + h;
    }
  p.noperands = numFields - 1;
  for (int o = 0; o < p.noperands; ++o)
    p.operand_field[o] = o;
  p.nops = static_cast<int>(v.size());
  p.ops = ops;
  p.nresults = 1;
  p.result_op[0] = out;
  p.store_field[0] = numFields - 1;
  for (int d = 0; d < rank; ++d) {
    p.store[0].lb[d] = 0;
    p.store[0].ub[d] = extent;
  }
  p.ngroups = 1;
  p.group_len[0] = numFields;
  for (int f = 0; f < numFields; ++f)
    p.groups[f] = f;
  return HG_OK;
}

// ---- apply fusion: a multi-apply step as one single-apply program ------------------------
//
// Every temp access of a stored apply is replaced by the producing apply's DAG evaluated at the
// shifted point (recursively), so the fused program reads fields only.  Each inlined value is
// computed by the same IEEE ops, in the same order, from the same inputs as the reference's
// materialised temp at that point (interpreter.cpp:713-758), hence bit-identical; propagate-
// bounds already guaranteed that every such point lies inside the producer's domain.  The
// (apply, shift) pairs are memoised, so a temp read at k distinct offsets costs k copies of its
// producer -- cheap next to the HBM round trip of a materialised temp.
int hg_fuse_applies(const hg_program *prog, hg_program *out, hg_op *ops, int cap_ops) {
  if (!prog || !out || !ops)
    return setError(HG_EINVAL, "null argument");
  const hg_program &g = *prog;
  if (g.napplies <= 0)
    return setError(HG_EINVAL, "not a multi-apply program");
  int st = validateProgram(g);
  if (st)
    return st;
  const int r = g.rank;
  std::vector<int> defApply(static_cast<size_t>(g.ntemps), -1), defResult(static_cast<size_t>(g.ntemps), -1);
  for (int a = 0; a < g.napplies; ++a)
    for (int k = 0; k < g.applies[a].nresults; ++k) {
      defApply[static_cast<size_t>(g.applies[a].result_temp[k])] = a;
      defResult[static_cast<size_t>(g.applies[a].result_temp[k])] = k;
    }
  std::vector<hg_op> outOps;
  std::vector<int> fieldOperand(static_cast<size_t>(g.nfields), -1); // field -> fused operand
  int nopnd = 0;
  // fields in load order, keeping only those some inlined access reads (assigned lazily)
  auto operandOf = [&](int f) {
    if (fieldOperand[static_cast<size_t>(f)] < 0)
      fieldOperand[static_cast<size_t>(f)] = nopnd++;
    return fieldOperand[static_cast<size_t>(f)];
  };
  const size_t budget = static_cast<size_t>(std::min<int64_t>(HG_MAX_OPS, std::max(64, 16 * g.nops)));
  std::map<std::pair<int, std::array<int64_t, 3>>, std::vector<int>> memo;
  bool overflow = false;
  std::function<const std::vector<int> &(int, std::array<int64_t, 3>)> inl =
      [&](int a, std::array<int64_t, 3> sh) -> const std::vector<int> & {
    auto key = std::make_pair(a, sh);
    auto it = memo.find(key);
    if (it != memo.end())
      return it->second;
    const hg_apply &A = g.applies[a];
    std::vector<int> map(static_cast<size_t>(A.nops), 0);
    for (int i = 0; i < A.nops && !overflow; ++i) {
      const hg_op &o = g.ops[A.op_begin + i];
      hg_op h;
      std::memset(&h, 0, sizeof h);
      if (o.code == HG_OP_ACCESS) {
        std::array<int64_t, 3> off = {0, 0, 0};
        for (int d = 0; d < r; ++d)
          off[static_cast<size_t>(d)] = o.off[d] + sh[static_cast<size_t>(d)];
        const int x = A.operand[o.operand];
        if (x < 0) { // a temp: its producer's value at the shifted point
          const int t = -x - 1;
          const std::vector<int> &pm = inl(defApply[static_cast<size_t>(t)], off);
          if (overflow)
            break;
          const hg_apply &P = g.applies[defApply[static_cast<size_t>(t)]];
          map[static_cast<size_t>(i)] = pm[static_cast<size_t>(P.result_op[defResult[static_cast<size_t>(t)]])];
          continue;
        }
        h.code = HG_OP_ACCESS;
        h.operand = operandOf(x);
        for (int d = 0; d < r; ++d)
          h.off[d] = off[static_cast<size_t>(d)];
      } else if (o.code == HG_OP_CONST) {
        h = o;
      } else {
        h.code = o.code;
        h.a = map[static_cast<size_t>(o.a)];
        h.b = map[static_cast<size_t>(o.b)];
      }
      if (outOps.size() >= budget) {
        overflow = true;
        break;
      }
      map[static_cast<size_t>(i)] = static_cast<int>(outOps.size());
      outOps.push_back(h);
    }
    return memo.emplace(key, std::move(map)).first->second;
  };
  hg_program f = g;
  f.napplies = 0;
  f.applies = nullptr;
  f.ntemps = 0;
  f.nstores = 0;
  if (g.nstores > HG_MAX_RESULTS)
    return setError(HG_EUNSUPPORTED, "apply fusion: more stores than results of one apply");
  f.nresults = g.nstores;
  for (int k = 0; k < g.nstores; ++k) {
    const int t = g.mstore_temp[k];
    const std::vector<int> &m = inl(defApply[static_cast<size_t>(t)], {0, 0, 0});
    if (overflow)
      return setError(HG_EUNSUPPORTED, "apply fusion: inlined DAG exceeds the op budget");
    const hg_apply &P = g.applies[defApply[static_cast<size_t>(t)]];
    f.result_op[k] = m[static_cast<size_t>(P.result_op[defResult[static_cast<size_t>(t)]])];
    f.store_field[k] = g.mstore_field[k];
    f.store[k] = g.mstore[k];
  }
  // operands: the accessed fields in load order
  std::vector<int> order;
  for (int o = 0; o < g.noperands; ++o)
    if (fieldOperand[static_cast<size_t>(g.operand_field[o])] >= 0 &&
        std::find(order.begin(), order.end(), g.operand_field[o]) == order.end())
      order.push_back(g.operand_field[o]);
  for (int fi = 0; fi < g.nfields; ++fi) // accessed but not in the load list (hand-built)
    if (fieldOperand[static_cast<size_t>(fi)] >= 0 &&
        std::find(order.begin(), order.end(), fi) == order.end())
      order.push_back(fi);
  std::vector<int> remap(static_cast<size_t>(nopnd), 0);
  for (size_t i = 0; i < order.size(); ++i)
    remap[static_cast<size_t>(fieldOperand[static_cast<size_t>(order[i])])] = static_cast<int>(i);
  for (auto &h : outOps)
    if (h.code == HG_OP_ACCESS)
      h.operand = remap[static_cast<size_t>(h.operand)];
  f.noperands = static_cast<int>(order.size());
  for (size_t i = 0; i < order.size(); ++i)
    f.operand_field[i] = order[i];
  if (static_cast<int>(outOps.size()) > cap_ops)
    return setError(HG_EINVAL, "op buffer too small");
  std::copy(outOps.begin(), outOps.end(), ops);
  f.nops = static_cast<int>(outOps.size());
  f.ops = ops;
  st = validateProgram(f);
  if (st)
    return setError(HG_EUNSUPPORTED, std::string("apply fusion: ") + hg_last_error());
  *out = f;
  return HG_OK;
}

int hg_program_match(const hg_program *prog, char *name, size_t cap) {
  if (!prog)
    return setError(HG_EINVAL, "null program");
  Analysis a;
  int st = analyze(*prog, a);
  if (st)
    return st;
  if (name && cap)
    std::snprintf(name, cap, "%s", a.name.c_str());
  return HG_OK;
}

// ---- decompose (dmp_transforms.cpp:101-312) on the descriptor ------------------------------
int hg_decompose_program(const hg_program *global, int ndim, const int64_t *grid,
                         hg_program *local, hg_decomp *dc) {
  if (!global || !grid || !local || !dc)
    return setError(HG_EINVAL, "null argument");
  int st = validateProgram(*global);
  if (st)
    return st;
  const hg_program &g = *global;
  int r = g.rank;
  const bool multi = g.napplies > 0;
  const int nst = multi ? g.nstores : g.nresults;
  const hg_bounds *stores = multi ? g.mstore : g.store;
  // the domain: every store covers the same region (:121-140)
  for (int k = 1; k < nst; ++k)
    for (int d = 0; d < r; ++d)
      if (stores[k].lb[d] != stores[0].lb[d] || stores[k].ub[d] != stores[0].ub[d])
        return setError(HG_EINVAL, "decompose requires every store to cover the same domain");
  if (ndim != r)
    return setError(HG_EINVAL, "grid rank " + std::to_string(ndim) +
                                   " does not match the domain rank " + std::to_string(r));
  int64_t core[3] = {1, 1, 1}, clb[3] = {0, 0, 0};
  for (int d = 0; d < r; ++d) {
    if (grid[d] < 1)
      return setError(HG_EINVAL, "grid dimensions must be at least 1");
    int64_t ext = stores[0].ub[d] - stores[0].lb[d];
    if (ext % grid[d] != 0)
      return setError(HG_EINVAL, "domain extent " + std::to_string(ext) + " in dimension " +
                                     std::to_string(d) + " is not divisible by grid extent " +
                                     std::to_string(grid[d]));
    core[d] = ext / grid[d];
    clb[d] = stores[0].lb[d];
  }
  // per apply: no apply-result operand, face footprints only (:164-200)
  const int napp = multi ? g.napplies : 1;
  for (int a = 0; a < napp; ++a) {
    const int b = multi ? g.applies[a].op_begin : 0;
    const int n = multi ? g.applies[a].nops : g.nops;
    if (multi)
      for (int o = 0; o < g.applies[a].noperands; ++o)
        if (g.applies[a].operand[o] < 0)
          return setError(HG_EINVAL,
                          "decompose does not support an apply consuming another apply");
    for (int i = b; i < b + n; ++i)
      if (g.ops[i].code == HG_OP_ACCESS) {
        int nz = 0;
        for (int d = 0; d < r; ++d)
          nz += g.ops[i].off[d] != 0;
        if (nz > 1)
          return setError(HG_EINVAL, "decompose supports face footprints only; a diagonal "
                                     "access offset requires corner exchanges");
      }
  }
  // per-field symmetric halos, <= core (:200-243)
  int64_t below[HG_MAX_FIELDS][3] = {}, above[HG_MAX_FIELDS][3] = {};
  for (int f = 0; f < g.nfields; ++f)
    for (int d = 0; d < r; ++d) {
      below[f][d] = stores[0].lb[d] - g.fields[f].lb[d];
      above[f][d] = g.fields[f].ub[d] - stores[0].ub[d];
      if (below[f][d] < 0 || above[f][d] < 0)
        return setError(HG_EINVAL, "field bounds do not cover the stored domain");
      if (below[f][d] != above[f][d])
        return setError(HG_EINVAL, "decompose requires symmetric halos");
      if (below[f][d] > core[d])
        return setError(HG_EINVAL, "halo width exceeds the per-rank core extent");
    }
  hg_program out = g;
  for (int f = 0; f < g.nfields; ++f)
    for (int d = 0; d < r; ++d) {
      out.fields[f].lb[d] = clb[d] - below[f][d];
      out.fields[f].ub[d] = clb[d] + core[d] + above[f][d];
    }
  for (int k = 0; k < nst; ++k)
    for (int d = 0; d < r; ++d) {
      hg_bounds &sb = multi ? out.mstore[k] : out.store[k];
      sb.lb[d] = clb[d];
      sb.ub[d] = clb[d] + core[d];
    }
  if (multi) {
    // propagate-bounds on the local shapes (:309-311): an apply no other apply reads is
    // evaluated exactly over what is stored of it, i.e. the local core; the rewritten
    // apply list lives in the caller's local->applies buffer (napplies entries)
    hg_apply *la = const_cast<hg_apply *>(local->applies);
    if (!la || la == g.applies)
      return setError(HG_EINVAL, "decompose of a multi-apply step needs local->applies set "
                                 "to a caller buffer of napplies entries");
    for (int a = 0; a < g.napplies; ++a) {
      la[a] = g.applies[a];
      for (int d = 0; d < r; ++d) {
        la[a].domain.lb[d] = clb[d];
        la[a].domain.ub[d] = clb[d] + core[d];
      }
    }
    out.applies = la;
  }
  std::memset(dc, 0, sizeof *dc);
  dc->ndim = ndim;
  for (int d = 0; d < r; ++d) {
    dc->grid[d] = grid[d];
    dc->core[d] = core[d];
  }
  // a swap before every load (:276-300), template exchanges (no coord); the single-apply
  // form's operands are its loads, the multi-apply form lists them in operand_field
  for (int o = 0; o < g.noperands; ++o) {
    hg_swap &s = dc->swaps[dc->nswaps++];
    int f = g.operand_field[o];
    s.field = f;
    s.nexchanges = hg_exchanges(r, core, below[f], above[f], nullptr, nullptr, s.ex,
                                2 * HG_MAX_RANK);
  }
  *local = out;
  return HG_OK;
}

int hg_decompose_program_deep(const hg_program *global, int ndim, const int64_t *grid,
                              int depth, hg_program *local, hg_decomp *dc) {
  if (depth < 1)
    return setError(HG_EINVAL, "depth must be at least 1");
  int st = hg_decompose_program(global, ndim, grid, local, dc);
  if (st || depth == 1)
    return st;
  hg_program &out = *local;
  const int r = out.rank;
  const hg_bounds *stores = out.napplies > 0 ? out.mstore : out.store;
  int64_t below[HG_MAX_FIELDS][3] = {}, above[HG_MAX_FIELDS][3] = {};
  for (int f = 0; f < out.nfields; ++f)
    for (int d = 0; d < r; ++d) {
      const int64_t h = stores[0].lb[d] - out.fields[f].lb[d];
      const int64_t H = grid[d] > 1 ? h * depth : h;
      if (H > dc->core[d])
        return setError(HG_EINVAL, "deep halo width " + std::to_string(H) +
                                       " exceeds the per-rank core extent");
      below[f][d] = above[f][d] = H;
      out.fields[f].lb[d] = stores[0].lb[d] - H;
      out.fields[f].ub[d] = stores[0].ub[d] + H;
    }
  for (int s = 0; s < dc->nswaps; ++s) {
    const int f = dc->swaps[s].field;
    dc->swaps[s].nexchanges = hg_exchanges(r, dc->core, below[f], above[f], nullptr, nullptr,
                                           dc->swaps[s].ex, 2 * HG_MAX_RANK);
  }
  return HG_OK;
}

} // extern "C"
