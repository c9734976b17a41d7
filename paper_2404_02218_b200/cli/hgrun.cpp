// hgrun -- command-line driver of the B200 path, mirroring the hot-path subcommands of the
// reference CLI (proj/tools/halogen.cpp): run-serial, simulate [--check], bench (CSV).
//
//   hgrun run-serial <file.xir|-> [-t T]
//   hgrun simulate   <file.xir|-> [-t T] [--check]       (a decomposed, dmp-level module)
//   hgrun bench --kind heat|wave|copy --rank R --extent N --order O [-t T] [--grid AxBxC]
//               [--label L] [--f64]
//
// Output lines follow the reference: "field i: <fnv1a hex> <bounds>" (halogen.cpp:93-98),
// "check field i: bitwise match" / "MISMATCH" (:259-283), CSV
// "label,core_points,steps,seconds,gpts_per_s" (throughput.cpp:25-41).  Everything runs on
// the GPU through the C-ABI; there is no CPU path.
#include "hg/hg.h"

#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace {

[[noreturn]] void die(const std::string &m) {
  std::cerr << "error: " << m << "\n";
  std::exit(1);
}

void ok(int st, const char *what) {
  if (st != HG_OK)
    die(std::string(what) + ": " + hg_last_error());
}

std::string readAll(const std::string &path) {
  std::ostringstream os;
  if (path == "-") {
    os << std::cin.rdbuf();
  } else {
    std::ifstream f(path);
    if (!f)
      die("cannot read " + path);
    os << f.rdbuf();
  }
  return os.str();
}

struct Prog {
  hg_program p{};
  std::vector<hg_op> ops = std::vector<hg_op>(HG_MAX_OPS);
  std::vector<hg_apply> applies = std::vector<hg_apply>(HG_MAX_APPLIES);
  hg_decomp dc{};
  int decomposed = 0;
  std::string reference;
};

Prog parse(const std::string &text) {
  Prog P;
  std::vector<char> ref(1 << 22);
  ok(hg_parse_program(text.c_str(), &P.p, P.ops.data(), HG_MAX_OPS, P.applies.data(),
                      HG_MAX_APPLIES, &P.dc, &P.decomposed, ref.data(), ref.size()),
     "parse");
  P.reference = ref.data();
  P.p.ops = P.ops.data();
  if (P.p.napplies > 0)
    P.p.applies = P.applies.data();
  return P;
}

int64_t count(const hg_bounds &b, int r) {
  int64_t n = 1;
  for (int d = 0; d < r; ++d)
    n *= b.ub[d] - b.lb[d];
  return n;
}

std::string boundsStr(const hg_bounds &b, int r) { // ir::Bounds::str (types.cpp:105-113)
  std::ostringstream os;
  for (int d = 0; d < r; ++d)
    os << (d ? "x" : "") << "[" << b.lb[d] << "," << b.ub[d] << "]";
  return os.str();
}

// runSerialStencil on the GPU; returns the final binding's host buffers
std::vector<std::vector<unsigned char>> runSerial(const hg_program &p, int64_t T, double *secs) {
  hg_plan *plan = nullptr;
  ok(hg_plan_create(&p, 0, &plan), "hg_plan_create");
  ok(hg_plan_init_fields(plan, nullptr, nullptr), "init"); // exec::initialFields
  const int es = p.dtype == HG_F32 ? 4 : 8;
  std::vector<std::vector<unsigned char>> host(static_cast<size_t>(p.nfields));
  for (int i = 0; i < p.nfields; ++i)
    host[static_cast<size_t>(i)].resize(static_cast<size_t>(count(p.fields[i], p.rank)) * es);
  ok(hg_plan_synchronize(plan), "sync");
  auto t0 = std::chrono::steady_clock::now();
  ok(hg_plan_run(plan, T, nullptr), "hg_plan_run");
  ok(hg_plan_synchronize(plan), "sync");
  if (secs)
    *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::vector<int32_t> perm(static_cast<size_t>(p.nfields));
  ok(hg_plan_binding(plan, perm.data(), nullptr), "binding");
  std::vector<std::vector<unsigned char>> out;
  for (int i = 0; i < p.nfields; ++i) {
    std::vector<unsigned char> b(host[static_cast<size_t>(perm[static_cast<size_t>(i)])].size());
    ok(hg_plan_download(plan, perm[static_cast<size_t>(i)], b.data(), b.size(), nullptr),
       "download");
    out.push_back(std::move(b));
  }
  hg_plan_destroy(plan);
  return out;
}

// exec::simulate over the process's GPUs: local plans at their global origins (the device
// fillInit at logical coordinates == scatterRank of initialFields), swaps, gather of cores
// over the initial global buffers of each slot's origin (simulator.cpp:1192-1200).
std::vector<std::vector<unsigned char>> simulate(const hg_program &global, const hg_program &local,
                                                 const hg_decomp &dc, int64_t T, double *secs) {
  const int r = local.rank, es = local.dtype == HG_F32 ? 4 : 8;
  int64_t P = 1;
  for (int d = 0; d < dc.ndim; ++d)
    P *= dc.grid[d];
  int ndev = 0;
  ok(hg_device_count(&ndev), "device count");
  if (ndev < 1)
    die("no CUDA device");
  std::vector<hg_plan *> plans(static_cast<size_t>(P));
  std::vector<hg_dmp *> dmps(static_cast<size_t>(P));
  for (int64_t q = 0; q < P; ++q) {
    ok(hg_plan_create(&local, static_cast<int>(q % ndev), &plans[static_cast<size_t>(q)]), "plan");
    int64_t c[3], org[3] = {0, 0, 0};
    hg_coord_from_rank(dc.ndim, q, dc.grid, c);
    for (int d = 0; d < r; ++d)
      org[d] = c[d] * dc.core[d];
    ok(hg_plan_init_fields(plans[static_cast<size_t>(q)], org, nullptr), "init");
    ok(hg_dmp_create(plans[static_cast<size_t>(q)], &dc, q, &dmps[static_cast<size_t>(q)]), "dmp");
  }
  ok(hg_sim_connect(dmps.data(), static_cast<int>(P)), "connect");
  for (auto *pl : plans)
    ok(hg_plan_synchronize(pl), "sync");
  auto t0 = std::chrono::steady_clock::now();
  ok(hg_sim_run(dmps.data(), static_cast<int>(P), T, nullptr), "hg_sim_run");
  for (auto *pl : plans) // the clock stops when every rank is done
    ok(hg_plan_synchronize(pl), "sync");
  const double simSecs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::vector<int32_t> perm(static_cast<size_t>(local.nfields));
  ok(hg_plan_binding(plans[0], perm.data(), nullptr), "binding");
  // initial global fields (for the rings) from a plan of the global program
  hg_plan *gp = nullptr;
  ok(hg_plan_create(&global, 0, &gp), "global plan");
  ok(hg_plan_init_fields(gp, nullptr, nullptr), "global init");
  std::vector<std::vector<unsigned char>> out;
  for (int i = 0; i < local.nfields; ++i) {
    const int b = perm[static_cast<size_t>(i)];
    std::vector<unsigned char> g(static_cast<size_t>(count(global.fields[b], r)) * es);
    ok(hg_plan_download(gp, b, g.data(), g.size(), nullptr), "download global");
    out.push_back(std::move(g));
  }
  hg_plan_destroy(gp);
  for (int64_t q = 0; q < P; ++q) {
    int64_t c[3];
    hg_coord_from_rank(dc.ndim, q, dc.grid, c);
    for (int i = 0; i < local.nfields; ++i) {
      const int b = perm[static_cast<size_t>(i)];
      std::vector<unsigned char> l(static_cast<size_t>(count(local.fields[b], r)) * es);
      ok(hg_plan_download(plans[static_cast<size_t>(q)], b, l.data(), l.size(), nullptr), "dl");
      const hg_bounds &lb = local.fields[b], &gb = global.fields[b];
      const hg_bounds &core = local.napplies > 0 ? local.mstore[0] : local.store[0];
      int64_t n = count(core, r);
      for (int64_t k = 0; k < n; ++k) { // gatherRank (simulator.cpp:1027-1060)
        int64_t rem = k, p[3] = {0, 0, 0};
        for (int d = r - 1; d >= 0; --d) {
          const int64_t e = core.ub[d] - core.lb[d];
          p[d] = core.lb[d] + rem % e;
          rem /= e;
        }
        int64_t li = 0, gi = 0;
        for (int d = 0; d < r; ++d) {
          li = li * (lb.ub[d] - lb.lb[d]) + (p[d] - lb.lb[d]);
          gi = gi * (gb.ub[d] - gb.lb[d]) + (p[d] + c[d] * dc.core[d] - gb.lb[d]);
        }
        std::memcpy(out[static_cast<size_t>(i)].data() + gi * es, l.data() + li * es,
                    static_cast<size_t>(es));
      }
    }
  }
  for (auto *d : dmps)
    hg_dmp_destroy(d);
  for (auto *p : plans)
    hg_plan_destroy(p);
  if (secs)
    *secs = simSecs;
  return out;
}

void printFields(const std::vector<std::vector<unsigned char>> &f, const hg_program &p,
                 const std::vector<int32_t> *perm) {
  for (size_t i = 0; i < f.size(); ++i) {
    const int b = perm ? (*perm)[i] : static_cast<int>(i);
    std::printf("field %zu: %" PRIx64 " %s\n", i, hg_fingerprint(f[i].data(), f[i].size()),
                boundsStr(p.fields[b], p.rank).c_str());
  }
}

struct Args {
  std::vector<std::string> pos;
  int64_t T = 1;
  bool check = false, f64 = false;
  std::string kind = "heat", grid, label;
  int rank = 2, order = 2;
  int64_t extent = 64;
};

Args parseArgs(int argc, char **argv) {
  Args a;
  for (int i = 2; i < argc; ++i) {
    std::string s = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc)
        die("missing value for " + s);
      return argv[++i];
    };
    if (s == "-t" || s == "--timesteps")
      a.T = std::atoll(next().c_str());
    else if (s == "--check")
      a.check = true;
    else if (s == "--f64")
      a.f64 = true;
    else if (s == "--kind")
      a.kind = next();
    else if (s == "--rank")
      a.rank = std::atoi(next().c_str());
    else if (s == "--extent")
      a.extent = std::atoll(next().c_str());
    else if (s == "--order")
      a.order = std::atoi(next().c_str());
    else if (s == "--grid")
      a.grid = next();
    else if (s == "--label")
      a.label = next();
    else
      a.pos.push_back(s);
  }
  return a;
}

std::vector<int64_t> parseGrid(const std::string &g) {
  std::vector<int64_t> v;
  std::stringstream ss(g);
  std::string tok;
  while (std::getline(ss, tok, 'x'))
    v.push_back(std::atoll(tok.c_str()));
  return v;
}

} // namespace

int main(int argc, char **argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: hgrun run-serial|simulate|bench ...\n");
    return 2;
  }
  const std::string cmd = argv[1];
  Args a = parseArgs(argc, argv);
  if (cmd == "run-serial") {
    Prog P = parse(readAll(a.pos.empty() ? "-" : a.pos[0]));
    auto out = runSerial(P.p, a.T, nullptr);
    // binding order: result i is the buffer bound to slot i (its bounds = that buffer's)
    std::vector<int32_t> perm(static_cast<size_t>(P.p.nfields));
    ok(hg_binding_after(P.p.ngroups, P.p.group_len, P.p.groups, P.p.nfields, a.T, perm.data()),
       "binding");
    printFields(out, P.p, &perm);
    return 0;
  }
  if (cmd == "simulate") {
    Prog P = parse(readAll(a.pos.empty() ? "-" : a.pos[0]));
    if (!P.decomposed || P.reference.empty())
      die("module is not decomposed: missing the dmp.topology attribute");
    Prog G = parse(P.reference);
    auto out = simulate(G.p, P.p, P.dc, a.T, nullptr);
    std::vector<int32_t> perm(static_cast<size_t>(P.p.nfields));
    ok(hg_binding_after(P.p.ngroups, P.p.group_len, P.p.groups, P.p.nfields, a.T, perm.data()),
       "binding");
    printFields(out, G.p, &perm);
    if (a.check) {
      auto ser = runSerial(G.p, a.T, nullptr);
      bool all = true;
      for (size_t i = 0; i < out.size(); ++i) {
        const bool same = ser[i] == out[i];
        std::printf("check field %zu: %s\n", i, same ? "bitwise match" : "MISMATCH");
        all = all && same;
      }
      return all ? 0 : 1;
    }
    return 0;
  }
  if (cmd == "bench") {
    Prog B;
    ok(hg_build_kernel_program(a.kind.c_str(), a.rank, a.extent, a.order,
                               a.f64 ? HG_F64 : HG_F32, &B.p, B.ops.data(), HG_MAX_OPS),
       "buildKernel");
    B.p.ops = B.ops.data();
    const int64_t pts = count(B.p.store[0], B.p.rank);
    double secs = 0;
    if (a.grid.empty()) {
      runSerial(B.p, a.T, &secs);
    } else {
      auto g = parseGrid(a.grid);
      hg_program local;
      hg_decomp dc;
      ok(hg_decompose_program(&B.p, static_cast<int>(g.size()), g.data(), &local, &dc),
         "decompose");
      local.ops = B.ops.data();
      simulate(B.p, local, dc, a.T, &secs);
    }
    std::string label = a.label.empty()
                            ? a.kind + "-" + std::to_string(a.rank) + "d-n" +
                                  std::to_string(a.extent) + "-o" + std::to_string(a.order) +
                                  (a.grid.empty() ? "" : "-g" + a.grid)
                            : a.label;
    std::printf("label,core_points,steps,seconds,gpts_per_s\n%s,%" PRId64 ",%" PRId64
                ",%.17g,%.17g\n",
                label.c_str(), pts, a.T, secs, hg_gpts_per_sec(pts, a.T, secs));
    return 0;
  }
  std::fprintf(stderr, "unknown subcommand '%s'\n", cmd.c_str());
  return 2;
}
