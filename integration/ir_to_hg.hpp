// ir_to_hg.hpp -- reads a reference stencil-level module (halogen ir::Operation) into the
// plain-C descriptor of include/hg/hg.h.  Header-only; compiled ONLY against the reference
// headers (oracle/Makefile `ref` / `adapter`), never into the product library.
//
// What it reads (all under /root/reference/proj/core):
//   entry function: the single all-field func (exec::stencilEntry, src/exec/serial.cpp:22-40)
//   stencil.load / dmp.swap / stencil.apply / stencil.store in body order
//     (emitted by buildKernel kernels.cpp:173-241 and decompose dmp_transforms.cpp:276-300)
//   apply region: stencil.access offsets, arith.constant FloatAttr raw bits
//     (include/halogen/ir/attributes.hpp:32-41), arith.addf/subf/mulf/divf
//   module attrs stencil.time_slots (stencil_transforms.cpp:196-230), dmp.topology
//   swap attrs grid / exchanges (#dmp.exchange, attributes.hpp:69-75)
#ifndef HG_INTEGRATION_IR_TO_HG_HPP
#define HG_INTEGRATION_IR_TO_HG_HPP

#include "hg/hg.h"
#include "halogen/exec/serial.hpp"
#include "halogen/ir/ir.hpp"

#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace hg_ir {

struct Converted {
  hg_program prog{};
  std::vector<hg_op> ops;
  std::vector<hg_apply> applies; // multi-apply steps (prog.applies points here)
  bool decomposed = false;
  hg_decomp decomp{};
};

// the step function: the reference's own exec::stencilEntry (serial.hpp:22, serial.cpp:22-40:
// the single func whose arguments are all fields); it only reads the module
inline const halogen::ir::Operation *stencilEntry(const halogen::ir::Operation &module) {
  return halogen::exec::stencilEntry(const_cast<halogen::ir::Operation &>(module));
}

inline void boundsOf(const halogen::ir::Bounds &b, hg_bounds &out) {
  for (int d = 0; d < b.rank(); ++d) {
    out.lb[d] = b.dims[d].lb;
    out.ub[d] = b.dims[d].ub;
  }
}

inline void timeSlotsInto(const halogen::ir::Operation &module, hg_program &p) {
  using namespace halogen::ir;
  if (const Attribute *ts = module.attr("stencil.time_slots")) {
    const auto &outer = ts->as<ArrayAttr>();
    int at = 0;
    for (const Attribute &g : outer.elems) {
      std::vector<std::int64_t> idx;
      attrToIndexVector(g, idx);
      p.group_len[p.ngroups++] = static_cast<int>(idx.size());
      for (auto i : idx)
        p.groups[at++] = static_cast<int>(i);
    }
  }
}

// Steps with several applies, or an apply consuming another: every apply is evaluated over its
// result bounds into temps (materializeApply, stencil_transforms.cpp:334-379).
// dmp.swap {grid, exchanges} (dmp_ops.cpp) -> one hg_swap of the decomposition
inline void swapInto(const halogen::ir::Operation &op, Converted &c) {
  using namespace halogen::ir;
  c.decomposed = true;
  if (c.decomp.nswaps >= HG_MAX_FIELDS)
    throw std::runtime_error("too many swaps");
  hg_swap &s = c.decomp.swaps[c.decomp.nswaps++];
  s.field = op.operands[0]->argIdx;
  const auto *g = op.attr("grid")->dynAs<GridAttr>();
  c.decomp.ndim = static_cast<int>(g->dims.size());
  for (int d = 0; d < c.decomp.ndim; ++d)
    c.decomp.grid[d] = g->dims[static_cast<std::size_t>(d)];
  const auto *xs = op.attr("exchanges")->dynAs<ArrayAttr>();
  s.nexchanges = 0;
  for (const Attribute &a : xs->elems) {
    const auto &e = a.as<ExchangeAttr>();
    hg_exchange &x = s.ex[s.nexchanges++];
    for (std::size_t d = 0; d < e.at.size(); ++d) {
      x.at[d] = e.at[d];
      x.size[d] = e.size[d];
      x.offset[d] = e.offset[d];
      x.to[d] = e.to[d];
    }
  }
}

inline Converted convertMulti(const halogen::ir::Operation &module,
                              const halogen::ir::Operation *entry, Converted c) {
  using namespace halogen::ir;
  const Region &body = entry->regions[0];
  hg_program &p = c.prog;
  std::map<const Value *, int> loadOf, tempOf;
  for (const auto &opPtr : body.ops) {
    const Operation &op = *opPtr;
    if (op.name == "stencil.load") {
      if (!op.operands[0]->isArg())
        throw std::runtime_error("stencil.load of a non-argument");
      if (p.noperands >= HG_MAX_FIELDS)
        throw std::runtime_error("too many loads");
      loadOf[&op.results[0]] = op.operands[0]->argIdx;
      p.operand_field[p.noperands++] = op.operands[0]->argIdx; // the load list
    } else if (op.name == "dmp.swap") {
      swapInto(op, c);
    } else if (op.name == "stencil.apply") {
      if (c.applies.size() >= HG_MAX_APPLIES)
        throw std::runtime_error("too many applies");
      hg_apply a;
      std::memset(&a, 0, sizeof a);
      a.noperands = op.numOperands();
      for (int k = 0; k < a.noperands; ++k) {
        const Value *v = op.operands[static_cast<std::size_t>(k)];
        if (loadOf.count(v))
          a.operand[k] = loadOf.at(v);
        else if (tempOf.count(v))
          a.operand[k] = -tempOf.at(v) - 1;
        else
          throw std::runtime_error("apply operand is neither a load nor an apply result");
      }
      const auto &tt = op.results[0].type.as<TempType>();
      if (!tt.bounds)
        throw std::runtime_error("unresolved stencil.apply bounds (run propagate-bounds)");
      boundsOf(*tt.bounds, a.domain);
      a.op_begin = static_cast<int>(c.ops.size());
      const Region &ar = op.regions[0];
      std::map<const Value *, int> vid, argIdx;
      for (std::size_t k = 0; k < ar.args.size(); ++k)
        argIdx[&ar.args[k]] = static_cast<int>(k);
      for (const auto &inPtr : ar.ops) {
        const Operation &in = *inPtr;
        hg_op h;
        std::memset(&h, 0, sizeof h);
        if (in.name == "stencil.access") {
          h.code = HG_OP_ACCESS;
          h.operand = argIdx.at(in.operands[0]);
          std::vector<std::int64_t> off;
          attrToIndexVector(*in.attr("offsets"), off);
          for (std::size_t d = 0; d < off.size(); ++d)
            h.off[d] = off[d];
        } else if (in.name == "arith.constant") {
          h.code = HG_OP_CONST;
          h.bits = in.attr("value")->as<FloatAttr>().bits;
        } else if (in.name == "arith.addf" || in.name == "arith.subf" ||
                   in.name == "arith.mulf" || in.name == "arith.divf") {
          h.code = in.name == "arith.addf"   ? HG_OP_ADD
                   : in.name == "arith.subf" ? HG_OP_SUB
                   : in.name == "arith.mulf" ? HG_OP_MUL
                                             : HG_OP_DIV;
          h.a = vid.at(in.operands[0]);
          h.b = vid.at(in.operands[1]);
        } else if (in.name == "stencil.return") {
          a.nresults = in.numOperands();
          for (int k = 0; k < a.nresults; ++k)
            a.result_op[k] = vid.at(in.operands[static_cast<std::size_t>(k)]);
          continue;
        } else {
          throw std::runtime_error("unsupported op in apply region: " + in.name);
        }
        vid[&in.results[0]] = static_cast<int>(c.ops.size()) - a.op_begin;
        c.ops.push_back(h);
      }
      a.nops = static_cast<int>(c.ops.size()) - a.op_begin;
      for (int k = 0; k < op.numResults(); ++k) {
        a.result_temp[k] = p.ntemps;
        tempOf[&op.results[static_cast<std::size_t>(k)]] = p.ntemps++;
      }
      c.applies.push_back(a);
    } else if (op.name == "stencil.store") {
      if (p.nstores >= HG_MAX_STORES)
        throw std::runtime_error("too many stores");
      const int k = p.nstores++;
      p.mstore_temp[k] = tempOf.at(op.operands[0]);
      p.mstore_field[k] = op.operands[1]->argIdx;
      std::vector<std::int64_t> lb, ub;
      attrToIndexVector(*op.attr("lb"), lb);
      attrToIndexVector(*op.attr("ub"), ub);
      for (std::size_t d = 0; d < lb.size(); ++d) {
        p.mstore[k].lb[d] = lb[d];
        p.mstore[k].ub[d] = ub[d];
      }
    } else if (op.name == "func.return") {
    } else {
      throw std::runtime_error("unsupported op in a multi-apply step: " + op.name);
    }
  }
  p.nops = static_cast<int>(c.ops.size());
  p.ops = c.ops.data();
  p.napplies = static_cast<int>(c.applies.size());
  p.applies = c.applies.data();
  timeSlotsInto(module, p);
  if (c.decomposed && p.nstores > 0)
    for (int d = 0; d < p.rank; ++d)
      c.decomp.core[d] = p.mstore[0].ub[d] - p.mstore[0].lb[d];
  return c;
}

// Throws std::runtime_error with a reason when the module is outside the descriptor's reach.
inline Converted convert(const halogen::ir::Operation &module) {
  using namespace halogen::ir;
  Converted c;
  std::memset(&c.prog, 0, sizeof c.prog);
  std::memset(&c.decomp, 0, sizeof c.decomp);
  const Operation *entry = stencilEntry(module);
  if (!entry)
    throw std::runtime_error("module has no single all-field step function");
  const Region &body = entry->regions[0];
  hg_program &p = c.prog;
  p.nfields = static_cast<int>(body.args.size());
  if (p.nfields > HG_MAX_FIELDS)
    throw std::runtime_error("too many fields");
  Scalar elem = Scalar::F64;
  for (int i = 0; i < p.nfields; ++i) {
    const auto &ft = body.args[static_cast<std::size_t>(i)].type.as<FieldType>();
    if (i == 0) {
      p.rank = ft.bounds.rank();
      elem = ft.elem;
    }
    if (ft.elem != elem || ft.bounds.rank() != p.rank)
      throw std::runtime_error("mixed field element types or ranks");
    boundsOf(ft.bounds, p.fields[i]);
  }
  if (elem != Scalar::F32 && elem != Scalar::F64)
    throw std::runtime_error("only f32/f64 fields are supported");
  p.dtype = elem == Scalar::F32 ? HG_F32 : HG_F64;

  std::map<const Value *, int> loadOf;   // stencil.load result -> field arg
  std::map<const Value *, int> applyRes; // apply result -> result index
  int napply = 0;
  // multi-apply form when there are several applies or one consumes another
  {
    int n = 0;
    bool chained = false;
    for (const auto &opPtr : body.ops)
      if (opPtr->name == "stencil.apply") {
        ++n;
        for (const Value *o : opPtr->operands)
          if (o->defOp && o->defOp->name == "stencil.apply")
            chained = true;
      }
    if (n > 1 || chained)
      return convertMulti(module, entry, std::move(c));
  }
  for (const auto &opPtr : body.ops) {
    const Operation &op = *opPtr;
    if (op.name == "stencil.load") {
      if (!op.operands[0]->isArg())
        throw std::runtime_error("stencil.load of a non-argument");
      loadOf[&op.results[0]] = op.operands[0]->argIdx;
    } else if (op.name == "dmp.swap") {
      swapInto(op, c);
    } else if (op.name == "stencil.apply") {
      if (++napply > 1)
        throw std::runtime_error("more than one stencil.apply per step");
      p.noperands = op.numOperands();
      for (int k = 0; k < p.noperands; ++k) {
        auto it = loadOf.find(op.operands[static_cast<std::size_t>(k)]);
        if (it == loadOf.end())
          throw std::runtime_error("apply operand is not a stencil.load result");
        p.operand_field[k] = it->second;
      }
      const Region &ar = op.regions[0];
      std::map<const Value *, int> vid;
      std::map<const Value *, int> argIdx;
      for (std::size_t k = 0; k < ar.args.size(); ++k)
        argIdx[&ar.args[k]] = static_cast<int>(k);
      for (const auto &inPtr : ar.ops) {
        const Operation &in = *inPtr;
        hg_op h;
        std::memset(&h, 0, sizeof h);
        if (in.name == "stencil.access") {
          h.code = HG_OP_ACCESS;
          h.operand = argIdx.at(in.operands[0]);
          std::vector<std::int64_t> off;
          attrToIndexVector(*in.attr("offsets"), off);
          for (std::size_t d = 0; d < off.size(); ++d)
            h.off[d] = off[d];
        } else if (in.name == "arith.constant") {
          h.code = HG_OP_CONST;
          const auto &f = in.attr("value")->as<FloatAttr>();
          h.bits = f.bits;
        } else if (in.name == "arith.addf" || in.name == "arith.subf" ||
                   in.name == "arith.mulf" || in.name == "arith.divf") {
          h.code = in.name == "arith.addf"   ? HG_OP_ADD
                   : in.name == "arith.subf" ? HG_OP_SUB
                   : in.name == "arith.mulf" ? HG_OP_MUL
                                             : HG_OP_DIV;
          h.a = vid.at(in.operands[0]);
          h.b = vid.at(in.operands[1]);
        } else if (in.name == "stencil.return") {
          p.nresults = in.numOperands();
          for (int k = 0; k < p.nresults; ++k)
            p.result_op[k] = vid.at(in.operands[static_cast<std::size_t>(k)]);
          continue;
        } else {
          throw std::runtime_error("unsupported op in apply region: " + in.name);
        }
        vid[&in.results[0]] = static_cast<int>(c.ops.size());
        c.ops.push_back(h);
      }
      for (int k = 0; k < op.numResults(); ++k)
        applyRes[&op.results[static_cast<std::size_t>(k)]] = k;
    } else if (op.name == "stencil.store") {
      int k = applyRes.at(op.operands[0]);
      p.store_field[k] = op.operands[1]->argIdx;
      std::vector<std::int64_t> lb, ub;
      attrToIndexVector(*op.attr("lb"), lb);
      attrToIndexVector(*op.attr("ub"), ub);
      for (std::size_t d = 0; d < lb.size(); ++d) {
        p.store[k].lb[d] = lb[d];
        p.store[k].ub[d] = ub[d];
      }
    } else if (op.name == "func.return") {
    } else {
      throw std::runtime_error("unsupported op in the step function: " + op.name);
    }
  }
  p.nops = static_cast<int>(c.ops.size());
  p.ops = c.ops.data();
  timeSlotsInto(module, p);
  if (c.decomposed) {
    // per-rank core = the (rank-0) store region written by decompose (dmp_transforms.cpp:262-272)
    for (int d = 0; d < p.rank; ++d)
      c.decomp.core[d] = p.store[0].ub[d] - p.store[0].lb[d];
  }
  return c;
}

} // namespace hg_ir

#endif
