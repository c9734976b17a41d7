// jit.cpp -- the "fused apply" family: any stencil.apply DAG (multi-operand, multi-result,
// diagonal accesses; e.g. the PW-advection set) compiled to straight-line sm_100a code.
//
// The CTA skeleton is the star family's (TMA-fed shared-memory ring of column-tile planes,
// one producer warp, 4 x-points per consumer thread, STG.128 outputs); only the per-point
// body is generated from the program: every stencil.access becomes a register read out of
// 16-byte LDS windows, every arith op one IEEE RN intrinsic in program order (bit-exact with
// the reference interpreter, interpreter.cpp:495-506, 759-780).  NVRTC compiles it once per
// program for sm_100a (-fmad=false); the module is loaded with cudaLibraryLoadData.
#include "jit.hpp"

#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <sstream>
#include <tuple>

namespace hg {

namespace {

constexpr int kPadX = 4;

struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetCUBINSize) cubinSize = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcGetProgramLogSize) logSize = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  bool ok = false;
};

const Nvrtc &nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *names[] = {"libnvrtc.so.12", "libnvrtc.so",
                           "/usr/local/cuda/lib64/libnvrtc.so.12"};
    void *h = nullptr;
    for (const char *nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL)))
        break;
    if (!h)
      return;
    n.create = reinterpret_cast<decltype(n.create)>(dlsym(h, "nvrtcCreateProgram"));
    n.compile = reinterpret_cast<decltype(n.compile)>(dlsym(h, "nvrtcCompileProgram"));
    n.cubinSize = reinterpret_cast<decltype(n.cubinSize)>(dlsym(h, "nvrtcGetCUBINSize"));
    n.cubin = reinterpret_cast<decltype(n.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
    n.logSize = reinterpret_cast<decltype(n.logSize)>(dlsym(h, "nvrtcGetProgramLogSize"));
    n.log = reinterpret_cast<decltype(n.log)>(dlsym(h, "nvrtcGetProgramLog"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
    n.ok = n.create && n.compile && n.cubinSize && n.cubin && n.logSize && n.log && n.destroy;
  });
  return n;
}

// The fixed part of the generated translation unit: PTX wrappers (no headers needed).
const char *kPrelude = R"(
typedef unsigned long long u64;
typedef unsigned int u32;
struct __align__(64) TMap { unsigned long long w[16]; };
__device__ __forceinline__ u32 sma(const void *p) {
  return (u32)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mb_init(u64 *b, u32 c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sma(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_expect(u64 *b, u32 n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sma(b)), "r"(n)
               : "memory");
}
__device__ __forceinline__ void mb_arrive(u64 *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sma(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(u64 *b, u32 ph) {
  u32 d;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(d) : "r"(sma(b)), "r"(ph) : "memory");
  } while (!d);
}
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk2(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk2(f2 v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ void tma3(void *dst, const TMap *m, u64 *b, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
               "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sma(dst)), "l"((u64)m), "r"(c0), "r"(c1),
               "r"(c2), "r"(sma(b)) : "memory");
}
)";

std::string tname(int dtype) { return dtype == HG_F32 ? "float" : "double"; }

std::string constLiteral(uint64_t bits, int dtype) {
  char buf[64];
  if (dtype == HG_F32)
    std::snprintf(buf, sizeof buf, "__int_as_float(0x%08xu)", static_cast<unsigned>(bits));
  else
    std::snprintf(buf, sizeof buf, "__longlong_as_double(0x%016llxull)",
                  static_cast<unsigned long long>(bits));
  return buf;
}

} // namespace

int jitMisaligned(const hg_program &p, const Layout &lay) {
  const int r = p.rank, es = p.dtype == HG_F32 ? 4 : 8;
  const long long col = lay.col0 + (p.store[0].lb[r - 1] - lay.lb[r - 1]);
  const int v = 16 / es;
  return int(((col % v) + v) % v);
}

bool jitEligible(const hg_program &p, const Analysis &a, std::string *why) {
  auto no = [&](const char *m) {
    if (why)
      *why = m;
    return false;
  };
  if (p.rank < 2)
    return no("rank 1");
  if (p.napplies > 0)
    return no("multi-apply step");
  for (int f = 1; f < p.nfields; ++f)
    for (int d = 0; d < p.rank; ++d)
      if (p.fields[f].lb[d] != p.fields[0].lb[d] || p.fields[f].ub[d] != p.fields[0].ub[d])
        return no("fields of different bounds");
  for (int k = 1; k < p.nresults; ++k)
    for (int d = 0; d < p.rank; ++d)
      if (p.store[k].lb[d] != p.store[0].lb[d] || p.store[k].ub[d] != p.store[0].ub[d])
        return no("stores of different regions");
  int rz = 0, ry = 0, rx = 0;
  for (int i = 0; i < p.nops; ++i) {
    const hg_op &o = p.ops[i];
    if (o.code != HG_OP_ACCESS)
      continue;
    rz = std::max<int>(rz, static_cast<int>(std::abs(o.off[0])));
    if (p.rank == 3)
      ry = std::max<int>(ry, static_cast<int>(std::abs(o.off[1])));
    rx = std::max<int>(rx, static_cast<int>(std::abs(o.off[p.rank - 1])));
  }
  if (rx > kPadX || ry > 8 || rz > 4)
    return no("access radius beyond the tile rims");
  if (p.noperands > 8)
    return no("more than 8 operands");
  (void)a;
  return true;
}

int jitBuildSource(const hg_program &p, JitKernel &K) {
  const int r = p.rank;
  int rz = 0, ry = 0, rx = 0;
  for (int i = 0; i < p.nops; ++i) {
    const hg_op &o = p.ops[i];
    if (o.code != HG_OP_ACCESS)
      continue;
    rz = std::max<int>(rz, static_cast<int>(std::abs(o.off[0])));
    if (r == 3)
      ry = std::max<int>(ry, static_cast<int>(std::abs(o.off[1])));
    rx = std::max<int>(rx, static_cast<int>(std::abs(o.off[r - 1])));
  }
  K.rz = rz;
  K.ry = ry;
  if (p.dtype != HG_F32)
    K.pack = false;
  K.txt = r == 3 ? 16 : 32;
  K.tyt = r == 3 ? 16 : 1;
  K.tx = K.txt * 4;
  K.ty = K.tyt;
  const int O = p.noperands;
  const int es = p.dtype == HG_F32 ? 4 : 8;
  const int cw = K.tx + 2 * kPadX;
  const int rows = K.ty + 2 * ry;
  const int ve = 128 / es;
  const int stage = rows * cw;
  const int sstride = (stage + ve - 1) / ve * ve;
  // TMA planes in flight beyond the 2RZ+1 window: 6 where shared memory allows (PW set:
  // 214 -> 224 GPts/s from depth 3 to 6, profiles/r1_sweeps.md), down to 1
  // >= 3 operand slabs per plane: a 3-deep ring keeps two CTAs per SM (with 16-plane chunks,
  // jitLaunch; PW set 222-224 -> 230-231 GPts/s, profiles/r1_sweeps.md); fewer operands
  // keep the 6-deep ring
  const int want = K.deep > 0 ? K.deep : (O >= 3 ? 3 : 6); // K.deep > 0: HG_JIT_DEPTH
  K.deep = want;
  auto smemFor = [&](int d) {
    return 128 + static_cast<size_t>(es) * (2 * rz + 1 + d) * O * sstride + 2 * (2 * rz + 1 + d) * 8;
  };
  int depth = want;
  while (depth > 1 && smemFor(depth) > 227 * 1024)
    --depth;
  K.ns = 2 * rz + 1 + depth;
  K.ncons = K.txt * K.tyt;
  K.nthreads = K.ncons + 32;
  K.smem = smemFor(depth);
  if (K.smem > 227 * 1024)
    return setError(HG_EUNSUPPORTED, "fused apply family: shared-memory ring too large");
  const std::string T = tname(p.dtype);
  const std::string add = p.dtype == HG_F32 ? "__fadd_rn" : "__dadd_rn";
  const std::string sub = p.dtype == HG_F32 ? "__fsub_rn" : "__dsub_rn";
  const std::string mul = p.dtype == HG_F32 ? "__fmul_rn" : "__dmul_rn";
  const std::string div = p.dtype == HG_F32 ? "__fdiv_rn" : "__ddiv_rn";

  // windows: (operand, dz, dy) -> which 4-element chunks (0: x-4..x-1, 1: x..x+3, 2: x+4..x+7)
  std::map<std::tuple<int, int, int>, int> win;
  for (int i = 0; i < p.nops; ++i) {
    const hg_op &o = p.ops[i];
    if (o.code != HG_OP_ACCESS)
      continue;
    const int dz = static_cast<int>(o.off[0]), dy = r == 3 ? static_cast<int>(o.off[1]) : 0,
              dx = static_cast<int>(o.off[r - 1]);
    int &m = win[{o.operand, dz, dy}];
    for (int j = 0; j < 4; ++j)
      m |= 1 << ((4 + j + dx) / 4);
  }

  std::ostringstream s;
  s << kPrelude;
  s << "typedef " << T << " T;\n";
  s << "struct P_t { TMap tm[" << O << "]; T *out[" << p.nresults << "];\n"
    << "  long long plane, pitch, col0; int zs, ys, xs, nz, ny, nx, tiles_x, tiles_y, chunk, "
       "nchunks, units; };\n";
  s << "struct __align__(16) V4 { T v[4]; };\n";
  s << "__device__ __forceinline__ V4 ld4(const T *q) { V4 r; ";
  if (es == 4)
    s << "float4 t = *(const float4 *)q; r.v[0]=t.x; r.v[1]=t.y; r.v[2]=t.z; r.v[3]=t.w; ";
  else
    s << "double2 a = ((const double2 *)q)[0], b = ((const double2 *)q)[1]; r.v[0]=a.x; "
         "r.v[1]=a.y; r.v[2]=b.x; r.v[3]=b.y; ";
  s << "return r; }\n";
  s << "__device__ __forceinline__ void st4(T *q, const V4 &r) { ";
  if (es == 4)
    s << "*(float4 *)q = make_float4(r.v[0], r.v[1], r.v[2], r.v[3]); ";
  else
    s << "((double2 *)q)[0] = make_double2(r.v[0], r.v[1]); ((double2 *)q)[1] = "
         "make_double2(r.v[2], r.v[3]); ";
  s << "}\n";
  constexpr int minBlocks = 1;
  s << "extern \"C\" __global__ void __launch_bounds__(" << K.nthreads << ", " << minBlocks
    << ") hg_apply(const __grid_constant__ P_t P) {\n";
  s << "  constexpr int O = " << O << ", RZ = " << rz << ", RY = " << ry << ", NS = " << K.ns
    << ", TXT = " << K.txt << ", TX = " << K.tx << ", TY = " << K.ty << ", CW = " << cw
    << ", SS = " << sstride << ", NCONS = " << K.ncons << ";\n";
  s << "  extern __shared__ __align__(128) unsigned char sm[];\n"
       "  T *stages = (T *)(sm + ((128u - (sma(sm) & 127u)) & 127u));\n"
       "  u64 *full = (u64 *)(stages + (size_t)NS * O * SS);\n"
       "  u64 *empty = full + NS;\n"
       "  const int tid = threadIdx.x;\n"
       "  if (tid == 0) { for (int s = 0; s < NS; ++s) { mb_init(&full[s], 1); "
       "mb_init(&empty[s], NCONS); }\n"
       "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\"); }\n"
       "  __syncthreads();\n"
       "  int xb, yb, zb, n;\n"
       "  auto unit = [&](int u) {\n"
       "    const int txi = u % P.tiles_x; u /= P.tiles_x;\n"
       "    const int tyi = u % P.tiles_y; const int chunk = u / P.tiles_y;\n"
       "    xb = txi * TX; yb = tyi * TY; zb = chunk * P.chunk;\n"
       "    n = min(P.chunk, P.nz - zb);\n"
       "  };\n";
  // producer: one elected thread streams every unit's planes through one ring, so the next
  // unit's first planes are in flight while the consumers finish the current one
  s << "  if (tid >= NCONS) {\n"
       "    if (tid == NCONS) {\n"
       "      int s = 0, ph = 0, g = 0;\n"
       "      for (int u = blockIdx.x; u < P.units; u += gridDim.x) {\n"
       "        unit(u);\n"
       "        const int cx = (int)P.col0 + P.xs + xb - 4;\n"
    << "        const int cy = " << (r == 3 ? "P.ys + yb - RY" : "0") << ";\n"
    << "        const int z0 = P.zs + zb - RZ;\n"
       "        for (int i = 0; i < n + 2 * RZ; ++i, ++g) {\n"
       "          if (g >= NS) mb_wait(&empty[s], (u32)(ph ^ 1));\n"
       "          mb_expect(&full[s], (u32)(O * (TY + 2 * RY) * CW * sizeof(T)));\n"
       "          for (int o = 0; o < O; ++o)\n"
       "            tma3(stages + ((size_t)s * O + o) * SS, &P.tm[o], &full[s], cx, cy, z0 + i);\n"
       "          if (++s == NS) { s = 0; ph ^= 1; }\n"
       "        }\n"
       "      }\n"
       "    }\n"
       "    return;\n"
       "  }\n";
  // consumers
  s << "  const int tx = tid % TXT, ty = tid / TXT, x0 = tx * 4;\n"
       "  const int rowOwn = (ty + RY) * CW + 4 + x0;\n"
       "  int sOld = 0;          // stage of plane m (oldest in the window)\n"
       "  int sNew = 0, phNew = 0;\n"
       "  for (int u = blockIdx.x; u < P.units; u += gridDim.x) {\n"
       "  unit(u);\n"
    << "  const bool yok = " << (r == 3 ? "yb + ty < P.ny" : "true") << ";\n"
    << "  const int xrem = P.nx - (xb + x0);\n"
       "  long long ebase = (long long)(P.zs + zb) * P.plane + "
    << (r == 3 ? "(long long)(P.ys + yb + ty) * P.pitch + " : "")
    << "P.col0 + P.xs + xb + x0; // output element of plane m\n"
       "  for (int i = 0; i < 2 * RZ; ++i) {\n"
       "    mb_wait(&full[sNew], (u32)phNew);\n"
       "    if (++sNew == NS) { sNew = 0; phNew ^= 1; }\n"
       "  }\n"
       "  for (int m = 0; m < n; ++m) {\n"
       "    mb_wait(&full[sNew], (u32)phNew);\n"
       "    if (++sNew == NS) { sNew = 0; phNew ^= 1; }\n";
  for (int dz = -rz; dz <= rz; ++dz)
    s << "    const T *pl" << (dz + rz) << " = stages + (size_t)(sOld + " << (dz + rz)
      << " >= NS ? sOld + " << (dz + rz) << " - NS : sOld + " << (dz + rz) << ") * O * SS;\n";
  for (auto &[key, mask] : win) {
    auto [o, dz, dy] = key;
    std::string nm = "w" + std::to_string(o) + "_" + std::to_string(dz + rz) + "_" +
                     std::to_string(dy + 8);
    std::string base = "pl" + std::to_string(dz + rz) + " + " + std::to_string(o) +
                       " * SS + rowOwn + (" + std::to_string(dy) + ") * CW";
    for (int c = 0; c < 3; ++c)
      if (mask & (1 << c))
        s << "    const V4 " << nm << "c" << c << " = ld4(" << base << " + " << (c - 1) * 4
          << ");\n";
  }
  // the DAG, 4 points
  for (int k = 0; k < p.nresults; ++k)
    s << "    V4 res" << k << ";\n";
  auto access = [&](const hg_op &o, int j) {
    const int dz = static_cast<int>(o.off[0]), dy = r == 3 ? static_cast<int>(o.off[1]) : 0,
              dx = static_cast<int>(o.off[r - 1]);
    const int idx = 4 + j + dx;
    return "w" + std::to_string(o.operand) + "_" + std::to_string(dz + rz) + "_" +
           std::to_string(dy + 8) + "c" + std::to_string(idx / 4) + ".v[" +
           std::to_string(idx % 4) + "]";
  };
  auto binop = [&](const hg_op &o) {
    switch (o.code) {
    case HG_OP_ADD:
      return add;
    case HG_OP_SUB:
      return sub;
    case HG_OP_MUL:
      return mul;
    default:
      return div;
    }
  };
  if (K.pack) {
    // f32: points (j, j+1) as one f32x2 lane pair for every add/sub (FADD2); products and
    // quotients stay scalar, so ptxas has no packed multiply to contract (bit-exact: each lane
    // is the scalar RN op).  An add reading an x access at an odd offset (its pair straddles
    // two 16-byte windows' register halves) stays scalar too.
    auto oddX = [&](int v) {
      const hg_op &o = p.ops[v];
      return o.code == HG_OP_ACCESS && (o.off[r - 1] % 2) != 0;
    };
    for (int jp = 0; jp < 4; jp += 2) {
      s << "    {\n";
      for (int i = 0; i < p.nops; ++i) {
        const hg_op &o = p.ops[i];
        const std::string a0 = "v" + std::to_string(o.a) + "_0", a1 = "v" + std::to_string(o.a) + "_1";
        const std::string b0 = "v" + std::to_string(o.b) + "_0", b1 = "v" + std::to_string(o.b) + "_1";
        const std::string v0 = "v" + std::to_string(i) + "_0", v1 = "v" + std::to_string(i) + "_1";
        switch (o.code) {
        case HG_OP_ACCESS:
          s << "      const T " << v0 << " = " << access(o, jp) << ", " << v1 << " = "
            << access(o, jp + 1) << ";\n";
          break;
        case HG_OP_CONST:
          s << "      const T " << v0 << " = " << constLiteral(o.bits, p.dtype) << ", " << v1
            << " = " << v0 << ";\n";
          break;
        case HG_OP_ADD:
        case HG_OP_SUB:
          if (!oddX(o.a) && !oddX(o.b)) {
            s << "      T " << v0 << ", " << v1 << "; upk2("
              << (o.code == HG_OP_ADD ? "add2" : "sub2") << "(pk2(" << a0 << ", " << a1
              << "), pk2(" << b0 << ", " << b1 << ")), " << v0 << ", " << v1 << ");\n";
            break;
          }
          [[fallthrough]];
        default:
          s << "      const T " << v0 << " = " << binop(o) << "(" << a0 << ", " << b0 << "), "
            << v1 << " = " << binop(o) << "(" << a1 << ", " << b1 << ");\n";
        }
      }
      for (int k = 0; k < p.nresults; ++k)
        s << "      res" << k << ".v[" << jp << "] = v" << p.result_op[k] << "_0; res" << k
          << ".v[" << jp + 1 << "] = v" << p.result_op[k] << "_1;\n";
      s << "    }\n";
    }
  } else {
    for (int j = 0; j < 4; ++j) {
      s << "    {\n";
      for (int i = 0; i < p.nops; ++i) {
        const hg_op &o = p.ops[i];
        s << "      const T v" << i << " = ";
        if (o.code == HG_OP_ACCESS)
          s << access(o, j);
        else if (o.code == HG_OP_CONST)
          s << constLiteral(o.bits, p.dtype);
        else
          s << binop(o) << "(v" << o.a << ", v" << o.b << ")";
        s << ";\n";
      }
      for (int k = 0; k < p.nresults; ++k)
        s << "      res" << k << ".v[" << j << "] = v" << p.result_op[k] << ";\n";
      s << "    }\n";
    }
  }
  s << "    if (yok) {\n"
       "      const long long e = ebase;\n";
  for (int k = 0; k < p.nresults; ++k)
    s << "      if (xrem >= 4) st4(P.out[" << k << "] + e, res" << k << "); else "
      << "for (int j = 0; j < 4; ++j) if (j < xrem) P.out[" << k << "][e + j] = res" << k
      << ".v[j];\n";
  s << "    }\n";
  // release plane m's stage only once every value read from it has been consumed.  ptxas
  // schedules LDS next to their first use, which may follow the arrive, and the SYNCS arrive
  // does not wait for in-flight LDS: the producer's next TMA then lands in the stage before
  // the load has read it (f64 windows, two LDS.128 each: flux3d per-apply tier, about 1 run
  // in 10).  Every consumer thread therefore arrives after its own output stores, whose
  // operands depend on every value its results use (the barrier counts all NCONS threads); a
  // thread that stores nothing uses none of them.
  s << "    ebase += P.plane;\n"
       "    mb_arrive(&empty[sOld]);\n"
       "    if (++sOld == NS) sOld = 0;\n";
  // the unit's last 2RZ planes were read by its last outputs, stored above: release them
  s << "  }\n"
       "  for (int i = 0; i < 2 * RZ; ++i) {\n"
       "    mb_arrive(&empty[sOld]);\n"
       "    if (++sOld == NS) sOld = 0;\n"
       "  }\n"
       "  }\n"
       "}\n";
  K.source = s.str();
  return HG_OK;
}

int jitCompile(JitKernel &K) {
  const Nvrtc &nv = nvrtc();
  if (!nv.ok)
    return setError(HG_EUNSUPPORTED, "NVRTC (libnvrtc.so.12) not available for the fused "
                                     "apply family");
  nvrtcProgram prog;
  if (nv.create(&prog, K.source.c_str(), "hg_apply.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return setError(HG_EUNSUPPORTED, "nvrtcCreateProgram failed");
  const char *opts[] = {"--gpu-architecture=sm_100a", "-fmad=false", "--std=c++17",
                        "-default-device", "-lineinfo", "-DNDEBUG"};
  nvrtcResult cr = nv.compile(prog, sizeof(opts) / sizeof(opts[0]), opts);
  if (cr != NVRTC_SUCCESS) {
    size_t ls = 0;
    nv.logSize(prog, &ls);
    std::string log(ls, '\0');
    nv.log(prog, log.data());
    nv.destroy(&prog);
    return setError(HG_EUNSUPPORTED, "NVRTC compile of the fused apply failed: " + log);
  }
  size_t cs = 0;
  nv.cubinSize(prog, &cs);
  K.cubin.resize(cs);
  nv.cubin(prog, K.cubin.data());
  nv.destroy(&prog);
  return HG_OK;
}

int jitLoad(JitKernel &K, int device) {
  cudaLibrary_t lib;
  cudaError_t e = cudaLibraryLoadData(&lib, K.cubin.data(), nullptr, nullptr, 0, nullptr,
                                      nullptr, 0);
  if (e != cudaSuccess)
    return setError(HG_ECUDA, std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e));
  cudaKernel_t k;
  e = cudaLibraryGetKernel(&k, lib, "hg_apply");
  if (e != cudaSuccess)
    return setError(HG_ECUDA, std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(e));
  K.lib = lib;
  K.kernel = k;
  e = cudaFuncSetAttribute(reinterpret_cast<const void *>(k),
                           cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(K.smem));
  if (e != cudaSuccess)
    return setError(HG_ECUDA, std::string("cudaFuncSetAttribute(jit): ") + cudaGetErrorString(e));
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&K.resident, reinterpret_cast<const void *>(k),
                                                    K.nthreads, K.smem);
  if (e != cudaSuccess || K.resident < 1)
    return setError(HG_ECUDA, "fused apply: no CTA fits an SM");
  cudaDeviceGetAttribute(&K.sms, cudaDevAttrMultiProcessorCount, device);
  return HG_OK;
}

int jitTensorMap(const JitKernel &K, int dtype, int rank, const Layout &lay, void *base,
                 CUtensorMap *out) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static std::once_flag once;
  std::call_once(once, [&] {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!encode)
    return setError(HG_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const int es = dtype == HG_F32 ? 4 : 8;
  cuuint64_t dims[3] = {cuuint64_t(lay.pitch), rank == 3 ? cuuint64_t(lay.shape[1]) : 1,
                        cuuint64_t(lay.shape[0])};
  cuuint64_t strides[2] = {cuuint64_t(lay.pitch * es),
                           cuuint64_t(lay.pitch * (rank == 3 ? lay.shape[1] : 1) * es)};
  cuuint32_t box[3] = {cuuint32_t(K.tx + 2 * kPadX), cuuint32_t(K.ty + 2 * K.ry), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(out, dtype == HG_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                           : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                      3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return setError(HG_ECUDA, "cuTensorMapEncodeTiled(jit) failed: " + std::to_string(int(r)));
  return HG_OK;
}

int jitLaunch(const JitKernel &K, const hg_program &p, const Layout &lay,
              const CUtensorMap *const *tms, void *const *outs, int chunks, bool persist,
              cudaStream_t st) {
  // must mirror struct P_t of the generated source
  struct alignas(64) TMap {
    unsigned long long w[16];
  };
  struct Params {
    TMap tm[8];
  };
  const int O = p.noperands, KR = p.nresults, r = p.rank;
  // pack the parameter block exactly like P_t: TMap tm[O]; T *out[KR]; long long plane,
  // pitch, col0; int zs, ys, xs, nz, ny, nx, tiles_x, tiles_y, chunk, nchunks, units;
  alignas(64) unsigned char buf[8 * 128 + 8 * 8 + 3 * 8 + 10 * 4 + 64];
  std::memset(buf, 0, sizeof buf);
  size_t at = 0;
  for (int o = 0; o < O; ++o) {
    std::memcpy(buf + at, tms[o], 128);
    at += 128;
  }
  for (int k = 0; k < KR; ++k) {
    std::memcpy(buf + at, &outs[k], 8);
    at += 8;
  }
  const long long plane = r == 3 ? lay.pitch * lay.shape[1] : lay.pitch;
  const long long pitch = lay.pitch, col0 = lay.col0;
  std::memcpy(buf + at, &plane, 8);
  std::memcpy(buf + at + 8, &pitch, 8);
  std::memcpy(buf + at + 16, &col0, 8);
  at += 24;
  int zs = int(p.store[0].lb[0] - lay.lb[0]);
  int ys = r == 3 ? int(p.store[0].lb[1] - lay.lb[1]) : 0;
  int xs = int(p.store[0].lb[r - 1] - lay.lb[r - 1]);
  int nz = int(p.store[0].ub[0] - p.store[0].lb[0]);
  int ny = r == 3 ? int(p.store[0].ub[1] - p.store[0].lb[1]) : 1;
  int nx = int(p.store[0].ub[r - 1] - p.store[0].lb[r - 1]);
  // the kernel's 16-byte row vectors need an aligned first column: a region starting off the
  // layout's aligned core column (a multi-apply producer widened below in x) is evaluated
  // from the aligned column below it; the extra columns land in the temp outside its domain,
  // which no consumer reads (jitMisaligned: such applies never write a field directly)
  const int mis = jitMisaligned(p, lay);
  xs -= mis;
  nx += mis;
  int tiles_x = (nx + K.tx - 1) / K.tx, tiles_y = (ny + K.ty - 1) / K.ty;
  // z-chunks of ~32 planes; ~16 with the 3-deep ring of multi-operand programs (two CTAs per
  // SM: more, shorter units balance the waves)
  const int zc = K.deep <= 3 ? 16 : 32;
  if (nz <= 0 || ny <= 0 || nx <= 0)
    return HG_OK; // an empty region: nothing to evaluate
  int nch = chunks > 0 ? chunks : std::max(1, (nz + zc / 2) / zc);
  int chunk = (nz + nch - 1) / nch;
  nch = (nz + chunk - 1) / chunk;
  const int units = tiles_x * tiles_y * nch;
  int iv[11] = {zs, ys, xs, nz, ny, nx, tiles_x, tiles_y, chunk, nch, units};
  std::memcpy(buf + at, iv, sizeof iv);
  at += sizeof iv;
  (void)Params{};
  void *args[] = {buf};
  // persistent: one wave of resident CTAs, each walking units blockIdx.x + k * gridDim.x with
  // its TMA ring running across unit boundaries; otherwise one CTA per unit
  const unsigned blocks =
      persist ? unsigned(std::min(units, K.resident * K.sms)) : unsigned(units);
  cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void *>(K.kernel), dim3(blocks),
                                   dim3(K.nthreads), args, K.smem, st);
  if (e != cudaSuccess)
    return setError(HG_ECUDA, std::string("fused apply launch: ") + cudaGetErrorString(e));
  return HG_OK;
}

} // namespace hg

extern "C" int hg_apply_compile(const hg_program *prog, char *src, size_t cap,
                                size_t *cubin_bytes) {
  using namespace hg;
  if (!prog)
    return setError(HG_EINVAL, "null program");
  Analysis a;
  int st = analyze(*prog, a);
  if (st)
    return st;
  std::string why;
  if (!jitEligible(*prog, a, &why))
    return setError(HG_EUNSUPPORTED, "fused apply family: " + why);
  JitKernel K; // the codegen a plan created now would use (its knobs: HG_JIT_PACK, HG_JIT_DEPTH)
  const Knobs kn = readKnobs();
  K.pack = kn.jitPack;
  K.deep = kn.jitDepth;
  st = jitBuildSource(*prog, K);
  if (st)
    return st;
  if (src && cap)
    std::snprintf(src, cap, "%s", K.source.c_str());
  st = jitCompile(K);
  if (st)
    return st;
  if (cubin_bytes)
    *cubin_bytes = K.cubin.size();
  return HG_OK;
}
