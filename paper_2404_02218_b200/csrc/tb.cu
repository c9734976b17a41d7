// tb.cu -- two time steps per pass for the 3D heat star (temporal blocking, §8 row f4).
//
// The reference advances one step per sweep: heat ping-pongs u_in -> u_out -> u_in
// (time_slots [[0,1]], kernels.cpp:139-243), each step reading 4 B and writing 4 B per point.
// Here one kernel pass computes steps t+1 and t+2 together: the t+1 values of an extended tile
// (output tile + R on every side, z-extended by R) live only in shared memory and feed the t+2
// evaluation, so a pair costs one read of u(t) and one write of u(t+2) -- 4 B per point-step.
//
// Bit-exactness: every point of both steps is the generator's DAG evaluated by the same
// exact-arithmetic code as starKernel (one IEEE op at a time, op order of kernels.cpp:110-135).
// Step t+1 values OUTSIDE the stored core are not computed by the reference: there the
// intermediate buffer keeps its own initial halo ring, so the kernel reads them from that buffer
// ("mid").  The t+1 core itself is only needed in HBM after the last pair of a run (the next
// pair recomputes it), so the pass writes it only when asked (write_mid).
//
// In-place hazard: a pair reads u(t) from buffer X and would write u(t+2) into X, while
// neighbouring CTAs still read X around their tiles.  The pass therefore writes u(t+2) into a
// shadow buffer X' whose halo ring equals X's (hg_plan keeps it), and the plan swaps X and X'.
//
// CTA geometry: one warp per step-1 row.  A row is 32 strips of 4 x-points (x in [-4, 124)
// around a 120-point output tile); warps R .. R+TY-1 (lanes 1..30) also evaluate step t+2.
// Input planes (x in [-8, 128), TY+4R rows) stream in by TMA through an mbarrier ring; step-1
// planes go to an (R+2)-deep shared ring; both steps keep their z neighbours in register
// queues exactly like starKernel.  One named barrier per plane orders the step-1 ring.
#include "device_util.cuh"
#include "kernels.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#ifndef HG_TB_DEPTH
#define HG_TB_DEPTH 2
#endif

namespace hg {
namespace {

int cudaErrTb(cudaError_t e, const char *what) {
  if (e == cudaSuccess)
    return HG_OK;
  return setError(HG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T, int NT> struct TbCfg {
  static constexpr int R = Taps<NT>::R;
  static constexpr int SX = 32;            // strips per row = lanes
  static constexpr int XW = SX * 4;        // step-1 columns: x in [-4, XW - 4)
  static constexpr int TX = XW - 8;        // output columns: strips 1 .. SX-2
  static constexpr int TY = R == 1 ? 18 : 16; // 20 warps: 5 per SMSP at 96 registers
  static constexpr int ROWS1 = TY + 2 * R; // step-1 rows = consumer warps
  static constexpr int ROWSI = TY + 4 * R; // input rows
  static constexpr int CWI = XW + 8;       // input columns: x in [-8, XW)
  static constexpr int NCONS = 32 * ROWS1;
  static constexpr int NTHREADS = NCONS;
  static constexpr int Q = 2 * R + 1;
  static constexpr int NSI = R + HG_TB_DEPTH;     // input ring (DEPTH planes ahead; R=2: 4)
  static constexpr int NS1 = R + 2;               // step-1 ring
  static constexpr int ALIGN = int(128 / sizeof(T));
  static constexpr int SI = (ROWSI * CWI + ALIGN - 1) / ALIGN * ALIGN;
  static constexpr int S1 = (ROWS1 * XW + ALIGN - 1) / ALIGN * ALIGN;
  static constexpr size_t SMEM =
      128 + sizeof(T) * (size_t(NSI) * SI + size_t(NS1) * S1) + NSI * sizeof(uint64_t);
};

template <typename T> struct TbParams {
  int64_t plane, pitch, col0;
  int zs, ys, xs;        // raw start of the core in the (shared) layout
  int nz, ny, nx;        // core extents
  int sz, sy, sx;        // allocation extents (raw), for the intermediate ring reads
  int tiles_x, tiles_y, chunk, nchunks;
  const T *mid;          // buffer of t+1 (its ring supplies the non-core step-1 values)
  T *mid_out;            // non-null: also store the t+1 core (last pair of a run)
  T *out;                // buffer receiving t+2 (shadow of the input buffer)
  T w0, wz[3], wy[3], wx[3], scale;
};

template <typename T, int NT>
__global__ void __launch_bounds__(TbCfg<T, NT>::NTHREADS, 1)
    tbHeatKernel(const __grid_constant__ CUtensorMap tmIn, const TbParams<T> P) {
  using C = TbCfg<T, NT>;
  constexpr int R = C::R, Q = C::Q, NSI = C::NSI, NS1 = C::NS1;
  extern __shared__ __align__(128) unsigned char smraw[];
  T *stI = reinterpret_cast<T *>(smraw + ((128u - (smemAddr(smraw) & 127u)) & 127u));
  T *st1 = stI + size_t(NSI) * C::SI;
  uint64_t *full = reinterpret_cast<uint64_t *>(st1 + size_t(NS1) * C::S1);

  int u = blockIdx.x;
  const int txi = u % P.tiles_x;
  u /= P.tiles_x;
  const int tyi = u % P.tiles_y;
  const int chunk = u / P.tiles_y;
  const int xb = txi * C::TX, yb = tyi * C::TY, zb = chunk * P.chunk;
  const int n = min(P.chunk, P.nz - zb);
  const int tid = threadIdx.x;

  if (n <= 0)
    return;
  // Thread 0 of warp 0 also feeds the input ring: plane p goes into slot p % NSI once the
  // plane that used the slot before (p - NSI) is consumed, which the per-plane named barrier
  // guarantees -- no producer warp, so 20 warps fit 96 registers each.
  const int cx = int(P.col0) + P.xs + xb - 8;
  const int cy = P.ys + yb - 2 * R;
  const int z0 = P.zs + zb - 2 * R;
  const int nIn = n + 4 * R; // input planes z = zb-2R .. zb+n+2R-1
  auto issue = [&](int p) {
    if (p < nIn) {
      constexpr uint32_t bytes = uint32_t(C::ROWSI * C::CWI * sizeof(T));
      const int s = p % NSI;
      mbarExpectTx(&full[s], bytes);
      tmaLoad3d(stI + size_t(s) * C::SI, &tmIn, &full[s], cx, cy, z0 + p);
    }
  };
  if (tid == 0) {
    for (int s = 0; s < NSI; ++s)
      mbarInit(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmIn)) : "memory");
    for (int p = 0; p < NSI; ++p)
      issue(p);
  }
  __syncthreads();

  // ---------------- consumers: warp w = step-1 row y = yb + w - R ----------------
  const int w = tid >> 5, lane = tid & 31;
  const int y1 = yb + w - R;              // logical row (core-relative) of this warp
  const int x1 = xb + 4 * lane - 4;       // first of the strip's 4 columns
  // step t+2 rows are warp-uniform; the two pad lanes compute along (no divergence) but
  // never store
  const bool two = w >= R && w < R + C::TY;
  const bool own = lane >= 1 && lane <= C::SX - 2;
  const int rowI = (w + R) * C::CWI + 4 * lane;     // left window start in an input stage
  const int row1 = w * C::XW + 4 * lane;            // strip start in a step-1 stage
  T qi[Q][4], q1[Q][4];

  // the strip's non-core step-1 points take the intermediate buffer's ring values
  const bool rowIn = y1 >= 0 && y1 < P.ny;
  const int64_t rowOff = int64_t(P.ys + y1) * P.pitch + P.col0 + P.xs + x1;
  const bool rowAlloc = P.ys + y1 >= 0 && P.ys + y1 < P.sy;

  // prologue: input planes 0 .. 2R-1 (centres only; planes < R feed no step-1 x/y)
#pragma unroll
  for (int i = 0; i < 2 * R; ++i) {
    mbarWait(&full[i % NSI], uint32_t((i / NSI) & 1));
    const V4<T> c = ld4(stI + size_t(i % NSI) * C::SI + rowI + 4);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      qi[i][j] = c.v[j];
  }
  // planes 0 .. R-1 fed only the queue: their slots take planes NSI .. NSI+R-1
  asm volatile("bar.sync 1, %0;" ::"r"(C::NCONS) : "memory");
  if (tid == 0)
    for (int p = NSI; p < NSI + R; ++p)
      issue(p);

  const int total = n + 2 * R; // step-1 planes z = zb-R .. zb+n+R-1
  auto iter = [&](int jj, auto uc) -> bool {
    constexpr int U = decltype(uc)::value; // jj % Q
    if (jj >= total)
      return false;
    // ---- arrival of input plane jj+2R: its centres enter the input queue ----
    {
      const int i = jj + 2 * R, s = i % NSI;
      mbarWait(&full[s], uint32_t((i / NSI) & 1));
      const V4<T> c = ld4(stI + size_t(s) * C::SI + rowI + 4);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        qi[(U + 2 * R) % Q][j] = c.v[j];
    }
    // ---- step t+1 on plane z1 = zb - R + jj (x/y from input stage jj+R) ----
    const int z1 = zb - R + jj;
    V4<T> s1;
    {
      const int s = (jj + R) % NSI;
      const T *st = stI + size_t(s) * C::SI;
      const V4<T> L = ld4(st + rowI);
      const V4<T> Rr = ld4(st + rowI + 8);
      V4<T> yp[NT], ym[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        yp[t] = ld4(st + rowI + 4 + Taps<NT>::k(t) * C::CWI);
        ym[t] = ld4(st + rowI + 4 - Taps<NT>::k(t) * C::CWI);
      }
      constexpr int cz = (U + R) % Q;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const T c = qi[cz][j];
        T acc = mul_(c, P.w0);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int k = Taps<NT>::k(t);
          acc = add_(acc, mul_(add_(qi[(U + R + k) % Q][j], qi[(U + R - k + Q) % Q][j]), P.wz[t]));
        }
#pragma unroll
        for (int t = 0; t < NT; ++t)
          acc = add_(acc, mul_(add_(yp[t].v[j], ym[t].v[j]), P.wy[t]));
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int k = Taps<NT>::k(t);
          const int ip = 4 + j + k, im = 4 + j - k;
          const T xp = ip < 4 ? L.v[ip & 3] : (ip < 8 ? qi[cz][ip & 3] : Rr.v[ip & 3]);
          const T xm = im < 4 ? L.v[im & 3] : (im < 8 ? qi[cz][im & 3] : Rr.v[im & 3]);
          acc = add_(acc, mul_(add_(xp, xm), P.wx[t]));
        }
        s1.v[j] = add_(c, mul_(acc, P.scale));
      }
      // outside the core: the intermediate buffer's own (never written) ring
      const bool zIn = z1 >= 0 && z1 < P.nz;
      if (!(zIn && rowIn && x1 >= 0 && x1 + 3 < P.nx)) {
        const bool zAlloc = P.zs + z1 >= 0 && P.zs + z1 < P.sz;
        const T *src = P.mid + int64_t(P.zs + z1) * P.plane + rowOff;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int x = x1 + j;
          if (!(zIn && rowIn && x >= 0 && x < P.nx)) {
            const bool alloc = zAlloc && rowAlloc && P.xs + x >= 0 && P.xs + x < P.sx;
            s1.v[j] = alloc ? src[j] : T(0);
          }
        }
      }
      st4(st1 + size_t(jj % NS1) * C::S1 + row1, s1);
    }
    if (two) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        q1[U][j] = s1.v[j];
      if (P.mid_out && own && z1 >= zb && z1 < zb + n && rowIn) {
        T *dst = P.mid_out + int64_t(P.zs + z1) * P.plane + rowOff;
        if (x1 + 3 < P.nx) {
          st4(dst, s1);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (x1 + j < P.nx)
              dst[j] = s1.v[j];
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(C::NCONS) : "memory");
    // input plane jj+R is consumed by every warp: its slot takes plane jj+R+NSI
    if (tid == 0)
      issue(jj + R + NSI);
    // ---- step t+2 on plane z2 = zb + jj - 2R (x/y from step-1 stage jj-R) ----
    const int m = jj - 2 * R;
    if (two && m >= 0) {
      const T *st = st1 + size_t((jj - R) % NS1) * C::S1;
      const V4<T> L = ld4(st + row1 - 4);
      const V4<T> Rr = ld4(st + row1 + 4);
      V4<T> yp[NT], ym[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        yp[t] = ld4(st + row1 + Taps<NT>::k(t) * C::XW);
        ym[t] = ld4(st + row1 - Taps<NT>::k(t) * C::XW);
      }
      constexpr int cz = (U + Q - R) % Q; // step-1 plane jj-R
      V4<T> o;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const T c = q1[cz][j];
        T acc = mul_(c, P.w0);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int k = Taps<NT>::k(t);
          acc = add_(acc, mul_(add_(q1[(cz + k) % Q][j], q1[(cz - k + Q) % Q][j]), P.wz[t]));
        }
#pragma unroll
        for (int t = 0; t < NT; ++t)
          acc = add_(acc, mul_(add_(yp[t].v[j], ym[t].v[j]), P.wy[t]));
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int k = Taps<NT>::k(t);
          const int ip = 4 + j + k, im = 4 + j - k;
          const T xp = ip < 4 ? L.v[ip & 3] : (ip < 8 ? q1[cz][ip & 3] : Rr.v[ip & 3]);
          const T xm = im < 4 ? L.v[im & 3] : (im < 8 ? q1[cz][im & 3] : Rr.v[im & 3]);
          acc = add_(acc, mul_(add_(xp, xm), P.wx[t]));
        }
        o.v[j] = add_(c, mul_(acc, P.scale));
      }
      T *dst = P.out + int64_t(P.zs + zb + m) * P.plane + rowOff;
      if (!(own && rowIn)) {
      } else if (x1 + 3 < P.nx) {
        st4(dst, o);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (x1 + j < P.nx)
            dst[j] = o.v[j];
      }
    }
    return true;
  };
  for (int mb = 0; mb < total; mb += Q)
    unrolled(iter, mb, std::make_integer_sequence<int, Q>{});
}

template <typename T, int NT> int launchTbT(const TbLaunch &L, cudaStream_t st, int *blocks) {
  using C = TbCfg<T, NT>;
  auto kern = tbHeatKernel<T, NT>;
  static std::mutex mu;
  static unsigned long long doneMask = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!(doneMask & (1ull << (dev & 63)))) {
      cudaError_t e =
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
      if (e != cudaSuccess)
        return cudaErrTb(e, "cudaFuncSetAttribute(tb)");
      doneMask |= 1ull << (dev & 63);
    }
  }
  const StarSpec &s = *L.spec;
  TbParams<T> P{};
  P.pitch = L.lay.pitch;
  P.plane = L.lay.pitch * L.lay.shape[1];
  P.col0 = L.lay.col0;
  P.zs = int(L.start[0]);
  P.ys = int(L.start[1]);
  P.xs = int(L.start[2]);
  P.nz = int(L.ext[0]);
  P.ny = int(L.ext[1]);
  P.nx = int(L.ext[2]);
  P.sz = int(L.lay.shape[0]);
  P.sy = int(L.lay.shape[1]);
  P.sx = int(L.lay.shape[2]);
  P.tiles_x = (P.nx + C::TX - 1) / C::TX;
  P.tiles_y = (P.ny + C::TY - 1) / C::TY;
  int chunks = L.chunks;
  if (chunks <= 0) {
    // one resident CTA per SM: pick the z-chunk count minimising waves x (planes + the 4R
    // pipeline fill every chunk pays)
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long tiles = long(P.tiles_x) * P.tiles_y;
    double best = 1e300;
    chunks = 1;
    for (int c = 1; c <= std::min(P.nz, 64); ++c) {
      const int len = (P.nz + c - 1) / c;
      if (c > 1 && long(len) * (c - 1) >= P.nz)
        continue;
      const long waves = (tiles * c + sms - 1) / sms;
      const double cost = double(waves) * (len + 4 * C::R + 8);
      if (cost < best - 1e-9) {
        best = cost;
        chunks = c;
      }
    }
  }
  P.chunk = (P.nz + chunks - 1) / chunks;
  P.nchunks = (P.nz + P.chunk - 1) / P.chunk;
  P.mid = static_cast<const T *>(L.mid);
  P.mid_out = L.write_mid ? static_cast<T *>(L.mid) : nullptr;
  P.out = static_cast<T *>(L.out);
  P.w0 = fromBits<T>(s.w0);
  for (int t = 0; t < 3; ++t) {
    P.wz[t] = fromBits<T>(s.w[0][t]);
    P.wy[t] = fromBits<T>(s.w[1][t]);
    P.wx[t] = fromBits<T>(s.w[2][t]);
  }
  P.scale = fromBits<T>(s.scale);
  const unsigned nb = unsigned(P.tiles_x) * P.tiles_y * P.nchunks;
  if (blocks)
    *blocks = int(nb);
  kern<<<nb, C::NTHREADS, C::SMEM, st>>>(*L.tm_in, P);
  return cudaErrTb(cudaGetLastError(), "tb kernel launch");
}

} // namespace

bool tbSupported(const StarSpec &s, int dtype, int rank) {
  return s.kind == kHeat && rank == 3 && dtype == HG_F32 && (s.ntaps == 1 || s.ntaps == 2);
}

int tbBox(const StarSpec &s, int dtype, uint32_t box[3]) {
  (void)dtype;
  const int R = s.radius;
  const int TY = R == 1 ? TbCfg<float, 1>::TY : TbCfg<float, 2>::TY;
  box[0] = uint32_t(TbCfg<float, 1>::CWI);
  box[1] = uint32_t(TY + 4 * R);
  box[2] = 1;
  return HG_OK;
}

int launchTb(const TbLaunch &L, cudaStream_t st, int *blocks) {
  if (L.dtype == HG_F32 && L.spec->ntaps == 1)
    return launchTbT<float, 1>(L, st, blocks);
  if (L.dtype == HG_F32 && L.spec->ntaps == 2)
    return launchTbT<float, 2>(L, st, blocks);
  return setError(HG_EUNSUPPORTED, "no two-step kernel for this star");
}

} // namespace hg
