// ref_capi.cpp -- C-ABI shim over the UNMODIFIED reference core (TEST INFRASTRUCTURE).
//
// Built only by oracle/Makefile (`make ref`) against the reference sources where they lie
// (/root/reference/proj/core), into oracle/_ref/libhalogen_ref.so.  It is used by
//   * tests/golden/make_golden.py  -- to generate the committed golden fixtures;
//   * tests (when the .so is present) -- to cross-check the C restatement oracle;
//   * bench.py --impl reference / cpu_baseline -- to time the reference's own CPU path.
// Nothing in the product links or loads it.  Every entry point calls the reference's own
// public API; no reference source is copied here.
//
// Reference functions used (file:line under /root/reference/proj/core):
//   exec::buildKernel            src/exec/kernels.cpp:139-243
//   exec::initialFields          src/exec/kernels.cpp:245-272
//   exec::runSerialStencil       src/exec/serial.cpp:57-88
//   exec::bindingAfter           src/exec/serial.cpp:42-55
//   exec::simulate               src/exec/simulator.cpp:1066-1203
//   exec::geometryOf/scatterRank src/exec/simulator.cpp:904-1025
//   exec::initValue/fingerprint  src/exec/buffer.cpp:142-188
//   ir::runPipeline              src/ir/pass.cpp:104-129
//   ir::dmp::*                   src/dialects/dmp_ops.cpp:21-115
#include "halogen/dialects/dmp.hpp"
#include "halogen/exec/buffer.hpp"
#include "halogen/exec/kernels.hpp"
#include "halogen/exec/serial.hpp"
#include "halogen/exec/simulator.hpp"
#include "halogen/ir/parser.hpp"
#include "halogen/ir/pass.hpp"
#include "halogen/ir/printer.hpp"

#include "../integration/ir_to_hg.hpp"
#include "ref_handles.hpp"

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

using namespace halogen;
using BufVec = std::vector<std::shared_ptr<exec::Buffer>>;

using hg_ref::Bufs;
using hg_ref::Mod;

namespace {
thread_local std::string g_err;

std::string retypeF32(const std::string &text) {
  // The generator is f64-only (kernels.cpp:159-161); the f32 module is the printed module
  // with every f64 token rewritten, re-parsed (f32 literals via from_chars<float>,
  // parser.cpp:392-398).
  std::string out = text;
  for (std::size_t p = out.find("f64"); p != std::string::npos; p = out.find("f64", p + 3))
    out.replace(p, 3, "f32");
  return out;
}
} // namespace

extern "C" {

const char *hr_last_error(void) { return g_err.c_str(); }

void *hr_parse(const char *text) {
  auto r = ir::parseModule(text, "<hr_parse>");
  if (!r.ok()) {
    g_err = r.diagText();
    return nullptr;
  }
  return new Mod{std::move(*r)};
}

void *hr_build_kernel(const char *kind, int rank, long long extent, int order, int f32) {
  exec::KernelSpec spec;
  spec.kind = kind;
  spec.rank = rank;
  spec.extent = extent;
  spec.order = order;
  auto r = exec::buildKernel(spec);
  if (!r.ok()) {
    g_err = r.diagText();
    return nullptr;
  }
  if (!f32)
    return new Mod{std::move(*r)};
  return hr_parse(retypeF32(ir::printModule(**r)).c_str());
}

char *hr_print(void *mod) {
  std::string s = ir::printModule(*static_cast<Mod *>(mod)->m);
  char *out = static_cast<char *>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

void hr_free_str(char *s) { std::free(s); }

void *hr_pipeline(void *mod, const char *pipeline) {
  auto r = ir::runPipeline(*static_cast<Mod *>(mod)->m, pipeline);
  if (!r.ok()) {
    g_err = r.diagText();
    return nullptr;
  }
  return new Mod{std::move(*r)};
}

void hr_module_free(void *mod) { delete static_cast<Mod *>(mod); }

void *hr_initial_fields(void *mod) {
  return new Bufs{exec::initialFields(*static_cast<Mod *>(mod)->m)};
}

void *hr_bufs_clone(void *bufs) {
  auto *b = static_cast<Bufs *>(bufs);
  auto *out = new Bufs;
  for (auto &x : b->v)
    out->v.push_back(x->clone());
  return out;
}

void hr_bufs_free(void *bufs) { delete static_cast<Bufs *>(bufs); }
int hr_bufs_count(void *bufs) { return static_cast<int>(static_cast<Bufs *>(bufs)->v.size()); }

// elem_bytes, rank, shape[rank], lb[rank]
int hr_buf_info(void *bufs, int i, int *elem_bytes, int *rank, long long *shape, long long *lb) {
  auto &b = *static_cast<Bufs *>(bufs)->v.at(static_cast<std::size_t>(i));
  *elem_bytes = b.elemWidth();
  *rank = b.rank();
  for (int d = 0; d < b.rank(); ++d) {
    shape[d] = b.shape[d];
    lb[d] = b.lb[d];
  }
  return 0;
}

void *hr_buf_data(void *bufs, int i) {
  return static_cast<Bufs *>(bufs)->v.at(static_cast<std::size_t>(i))->data.data();
}

unsigned long long hr_fingerprint(void *bufs, int i) {
  return exec::fingerprint(*static_cast<Bufs *>(bufs)->v.at(static_cast<std::size_t>(i)));
}

// runSerialStencil: mutates `bufs` in place; returns the final binding (a new handle whose
// entries alias the input buffers, as in serial.cpp:80-87).
void *hr_run_serial(void *mod, void *bufs, long long timesteps) {
  try {
    auto out = exec::runSerialStencil(*static_cast<Mod *>(mod)->m,
                                      static_cast<Bufs *>(bufs)->v, timesteps);
    return new Bufs{std::move(out)};
  } catch (const std::exception &e) {
    g_err = e.what();
    return nullptr;
  }
}

// Wall-clock seconds of runSerialStencil alone, the `halogen bench` recipe
// (tools/halogen.cpp:296-318).
double hr_time_serial(void *mod, void *bufs, long long timesteps) {
  auto t0 = std::chrono::steady_clock::now();
  try {
    exec::runSerialStencil(*static_cast<Mod *>(mod)->m, static_cast<Bufs *>(bufs)->v,
                           timesteps);
  } catch (const std::exception &e) {
    g_err = e.what();
    return -1.0;
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void *hr_simulate(void *mod, void *global_init, long long timesteps, unsigned long long seed) {
  exec::SimOptions o;
  o.timesteps = timesteps;
  o.seed = seed;
  auto r = exec::simulate(*static_cast<Mod *>(mod)->m, static_cast<Bufs *>(global_init)->v, o);
  if (!r.ok) {
    g_err = r.error;
    return nullptr;
  }
  return new Bufs{std::move(r.fields)};
}

double hr_time_simulate(void *mod, void *global_init, long long timesteps) {
  exec::SimOptions o;
  o.timesteps = timesteps;
  auto t0 = std::chrono::steady_clock::now();
  auto r = exec::simulate(*static_cast<Mod *>(mod)->m, static_cast<Bufs *>(global_init)->v, o);
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (!r.ok) {
    g_err = r.error;
    return -1.0;
  }
  return s;
}

// Per-rank local buffers of a decomposed module (scatterRank, simulator.cpp:995-1025).
void *hr_scatter_rank(void *mod, void *global_init, long long rank) {
  auto g = exec::geometryOf(*static_cast<Mod *>(mod)->m);
  if (!g.ok()) {
    g_err = g.diagText();
    return nullptr;
  }
  return new Bufs{exec::scatterRank(*g, static_cast<Bufs *>(global_init)->v, rank)};
}

double hr_init_value(int field, int rank, const long long *coord) {
  std::vector<std::int64_t> c(coord, coord + rank);
  return exec::initValue(field, c);
}

long long hr_rank_from_coord(int n, const long long *coord, const long long *grid) {
  return ir::dmp::rankFromCoord(std::vector<std::int64_t>(coord, coord + n),
                                std::vector<std::int64_t>(grid, grid + n));
}

void hr_coord_from_rank(int n, long long rank, const long long *grid, long long *coord) {
  auto c = ir::dmp::coordFromRank(rank, std::vector<std::int64_t>(grid, grid + n));
  for (int d = 0; d < n; ++d)
    coord[d] = c[d];
}

long long hr_neighbor_rank(int n, long long rank, const long long *dir, const long long *grid) {
  return ir::dmp::neighborRank(rank, std::vector<std::int64_t>(dir, dir + n),
                               std::vector<std::int64_t>(grid, grid + n));
}

void hr_local_interval(long long extent, long long parts, long long part, long long *lb,
                       long long *ub) {
  ir::dmp::StandardSlicing s;
  auto iv = s.localInterval(extent, parts, part);
  *lb = iv.lb;
  *ub = iv.ub;
}

// StandardSlicing::exchanges; out receives ndecl records of 4*n int64 (at,size,offset,to).
int hr_exchanges(int n, const long long *core, const long long *below, const long long *above,
                 const long long *grid, const long long *coord, long long *out, int cap) {
  ir::dmp::StandardSlicing s;
  std::vector<std::int64_t> g, c;
  if (grid)
    g.assign(grid, grid + n);
  if (coord)
    c.assign(coord, coord + n);
  auto decls = s.exchanges(std::vector<std::int64_t>(core, core + n),
                           std::vector<std::int64_t>(below, below + n),
                           std::vector<std::int64_t>(above, above + n), g, c);
  int k = 0;
  for (auto &e : decls) {
    if (k >= cap)
      break;
    long long *o = out + static_cast<std::size_t>(k) * 4 * n;
    for (int d = 0; d < n; ++d) {
      o[d] = e.at[d];
      o[n + d] = e.size[d];
      o[2 * n + d] = e.offset[d];
      o[3 * n + d] = e.to[d];
    }
    ++k;
  }
  return static_cast<int>(decls.size());
}

void hr_binding_after(int ngroups, const int *group_len, const int *groups, int nargs,
                      long long steps, int *out) {
  std::vector<std::vector<int>> gs;
  int at = 0;
  for (int i = 0; i < ngroups; ++i) {
    gs.emplace_back(groups + at, groups + at + group_len[i]);
    at += group_len[i];
  }
  auto r = exec::bindingAfter(gs, nargs, steps);
  for (int i = 0; i < nargs; ++i)
    out[i] = r[i];
}

double hr_laplacian_weight(int order, long long k) { return exec::laplacianWeight(order, k); }

// The reference module read into the hg descriptor (integration/ir_to_hg.hpp); ops are copied
// into ops[cap].  Returns the op count, or -1 with hr_last_error set.
int hr_export_program(void *mod, hg_program *out, hg_op *ops, int cap, hg_decomp *dc,
                      int *decomposed, hg_apply *applies, int cap_applies) {
  try {
    auto c = hg_ir::convert(*static_cast<Mod *>(mod)->m);
    if (static_cast<int>(c.ops.size()) > cap ||
        static_cast<int>(c.applies.size()) > cap_applies) {
      g_err = "op/apply buffer too small";
      return -1;
    }
    std::memcpy(ops, c.ops.data(), c.ops.size() * sizeof(hg_op));
    if (!c.applies.empty())
      std::memcpy(applies, c.applies.data(), c.applies.size() * sizeof(hg_apply));
    *out = c.prog;
    out->ops = ops;
    out->applies = c.applies.empty() ? nullptr : applies;
    if (dc)
      *dc = c.decomp;
    if (decomposed)
      *decomposed = c.decomposed ? 1 : 0;
    return static_cast<int>(c.ops.size());
  } catch (const std::exception &e) {
    g_err = e.what();
    return -1;
  }
}

} // extern "C"
