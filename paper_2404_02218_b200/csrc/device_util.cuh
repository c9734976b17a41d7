// device_util.cuh -- device helpers shared by the sm_100a kernels (kernels.cu, tb.cu):
// exact (never contracted) IEEE arithmetic, mbarrier/TMA PTX, 16-byte vector moves, star taps.
#ifndef HG_DEVICE_UTIL_CUH
#define HG_DEVICE_UTIL_CUH

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <type_traits>
#include <utility>

namespace hg {
namespace {

// ---- exact arithmetic -----------------------------------------------------------------------
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float div_(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double div_(double a, double b) { return __ddiv_rn(a, b); }

// ---- packed f32x2 arithmetic (FADD2: two independent IEEE RN f32 adds per issue) ---------------
// f32 stencil arithmetic (star and resident kernels) on f32x2 pairs of neighbouring points:
// each lane is the scalar RN op, so packing two points' identical op sequences is bit-exact
// provided nothing is contracted.  HG_PACK=2 (product): sums and accumulations as FADD2, every
// product a scalar FMUL, so ptxas has no mul.f32x2 -> add.f32x2 pair to fuse into FFMA2 (it
// does fuse that pair even under -fmad=false; round 1 fenced every packed product instead and
// ran 4-8% slower, profiles/r1_sweeps.md).  112 -> ~93 instructions per 4-point plane, +3%
// burst and +7% sustained (power-capped) on heat 1024^3 (profiles/r2_ab.md).  HG_PACK=0: scalar.
#ifndef HG_PACK
#define HG_PACK 2
#endif
using f2 = unsigned long long;
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

template <typename T> __host__ __device__ inline T fromBits(uint64_t b);
template <> __host__ __device__ inline float fromBits<float>(uint64_t b) {
  uint32_t u = static_cast<uint32_t>(b);
  float f;
  memcpy(&f, &u, 4);
  return f;
}
template <> __host__ __device__ inline double fromBits<double>(uint64_t b) {
  double d;
  memcpy(&d, &b, 8);
  return d;
}

// ---- mbarrier / TMA PTX -------------------------------------------------------------------
__device__ __forceinline__ uint32_t smemAddr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbarInit(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smemAddr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbarExpectTx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smemAddr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbarArrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smemAddr(bar)) : "memory");
}
__device__ __forceinline__ void mbarWait(uint64_t *bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done)
                 : "r"(smemAddr(bar)), "r"(parity)
                 : "memory");
  } while (!done);
}
__device__ __forceinline__ void tmaLoad3d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                          int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
               "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smemAddr(dst)),
               "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
               "r"(smemAddr(bar))
               : "memory");
}

// The same load with an L2 eviction-priority policy (createpolicy): planes the next z-chunk
// of the same column will re-read are kept (evict_last); planes read for the last time go
// first (evict_first).
__device__ __forceinline__ uint64_t l2PolicyEvictLast() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2PolicyEvictFirst() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tmaLoad3dHint(void *dst, const CUtensorMap *map, uint64_t *bar,
                                              int c0, int c1, int c2, uint64_t policy) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
               ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smemAddr(dst)),
               "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
               "r"(smemAddr(bar)), "l"(policy)
               : "memory");
}

// ---- bounded flag waits (stuck-peer detection) -----------------------------------------------
__device__ __forceinline__ uint64_t globalNs() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spins until *flag >= epoch (system-scope acquire: the peer's release store and every byte it
// wrote before it are visible).  With timeout_ns > 0 it gives up after that long, records
// `code` in *err (first error wins) and returns false; it also gives up at once when another
// waiter already recorded an error, so a dead peer costs one timeout, not one per waiter.
// The reference reports a deadlock instead of hanging (simulator.cpp:143-173, 1174-1187).
__device__ __forceinline__ bool waitFlag(const unsigned long long *flag, unsigned long long epoch,
                                         unsigned long long *err, unsigned long long timeout_ns,
                                         unsigned long long code) {
  unsigned long long v;
  uint64_t t0 = 0;
  for (unsigned spin = 0;; ++spin) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= epoch)
      return true;
    if (timeout_ns && (spin & 63) == 0) {
      const uint64_t now = globalNs();
      if (t0 == 0)
        t0 = now;
      unsigned long long e = 0;
      if (err)
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(e) : "l"(err) : "memory");
      if (e != 0 || now - t0 > timeout_ns) {
        if (err && e == 0)
          atomicCAS(err, 0ull, code);
        return false;
      }
    }
  }
}

// Calls f(mb + U, integral_constant<U>) for U = 0, 1, ... while it returns true.
template <typename F, int... Us>
__device__ __forceinline__ void unrolled(F &f, int mb, std::integer_sequence<int, Us...>) {
  (void)(f(mb + Us, std::integral_constant<int, Us>{}) && ...);
}

// 4 consecutive elements (16 B for f32, 2x16 B for f64) from 16-byte-aligned memory
template <typename T> struct V4 { T v[4]; };
__device__ __forceinline__ V4<float> ld4(const float *p) {
  float4 t = *reinterpret_cast<const float4 *>(p);
  return {{t.x, t.y, t.z, t.w}};
}
__device__ __forceinline__ V4<double> ld4(const double *p) {
  double2 a = reinterpret_cast<const double2 *>(p)[0];
  double2 b = reinterpret_cast<const double2 *>(p)[1];
  return {{a.x, a.y, b.x, b.y}};
}
__device__ __forceinline__ void st4(float *p, const V4<float> &v) {
  *reinterpret_cast<float4 *>(p) = make_float4(v.v[0], v.v[1], v.v[2], v.v[3]);
}
__device__ __forceinline__ void st4(double *p, const V4<double> &v) {
  reinterpret_cast<double2 *>(p)[0] = make_double2(v.v[0], v.v[1]);
  reinterpret_cast<double2 *>(p)[1] = make_double2(v.v[2], v.v[3]);
}

// Star tap sets: distances of the taps per side (laplacianTaps, kernels.cpp:35-60)
template <int NT> struct Taps;
template <> struct Taps<1> {
  static constexpr int R = 1;
  __device__ static constexpr int k(int i) { return 1; }
};
template <> struct Taps<2> {
  static constexpr int R = 2;
  __device__ static constexpr int k(int i) { return i + 1; }
};
template <> struct Taps<3> {
  static constexpr int R = 4;
  __device__ static constexpr int k(int i) { return i == 0 ? 1 : (i == 1 ? 2 : 4); }
};

} // namespace
} // namespace hg

#endif
