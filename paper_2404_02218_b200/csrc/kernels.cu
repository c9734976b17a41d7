// kernels.cu -- sm_100a kernels of the stencil time-stepping + halo-swap path.
//
// Bit-exactness contract: the reference evaluates every apply point as a fixed DAG of IEEE
// round-to-nearest f32/f64 ops with no FMA contraction (-ffp-contract=off,
// proj/CMakeLists.txt:8-10; interpreter.cpp:495-506).  All arithmetic here goes through
// __fadd_rn/__fmul_rn/... (never contracted) and this file is also built with -fmad=false.
// Loads, schedules and data movement are free; operand pairing and evaluation order are not.
#include "kernels.hpp"
#include "device_util.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

// TMA prefetch depth (planes in flight beyond the R+1 a CTA computes on); tunables.
#ifndef HG_DEPTH3
#define HG_DEPTH3 5
#endif
#ifndef HG_DEPTH3W
#define HG_DEPTH3W 7
#endif
#ifndef HG_DEPTH2
#define HG_DEPTH2 4
#endif
#ifndef HG_MINB_R4
#define HG_MINB_R4 1
#endif
#ifndef HG_MINB_R2
#define HG_MINB_R2 3
#endif
#ifndef HG_TYT_R4
#define HG_TYT_R4 24
#endif
#ifndef HG_TXT_R4
#define HG_TXT_R4 16
#endif
#ifndef HG_TYT_R2
#define HG_TYT_R2 16
#endif
#ifndef HG_TXT_R2
#define HG_TXT_R2 16
#endif

namespace hg {

UnitOrderCache::~UnitOrderCache() {
  for (auto &kv : tables)
    cudaFree(kv.second);
}

DevLayout devLayout(const Layout &L) {
  DevLayout d{};
  for (int i = 0; i < 3; ++i) {
    d.shape[i] = L.shape[i];
    d.lb[i] = L.lb[i];
  }
  d.pitch = L.pitch;
  d.col0 = L.col0;
  d.rank = L.rank;
  d.es = L.es;
  return d;
}

namespace {

int cudaErr(cudaError_t e, const char *what) {
  if (e == cudaSuccess)
    return HG_OK;
  return setError(HG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- star family ------------------------------------------------------------------------
//
// One CTA owns a TX x TY tile of (x, y) columns and a chunk of z planes (dim 0).  A producer
// warp streams the tile's planes, with a PADX-wide x rim and an R-row y rim, into an NS-deep
// shared-memory ring by TMA (one cp.async.bulk.tensor per plane, mbarrier complete_tx).
// Consumer threads own 4 consecutive x points each; the centre values of the 2R+1 planes
// around the output plane live in registers (the z queue), x/y neighbours are read from the
// staged plane with 16-byte LDS.  Output planes are stored straight to HBM (STG.128).
// Column-tile geometry: TXT x TYT consumer threads, 4 x-points each.  3D radius-4 tiles are
// taller (more consumer warps in the single CTA an SM holds at ~110 registers).
// GEO 1 is the wide tile (128 x 12, 2 CTAs/SM) chosen for large x-y planes (starGeoFor): its
// smaller rim-to-core ratio cuts the halo re-reads of 1024^2 planes (sweep in
// profiles/r1_sweeps.md); GEO 0 suits smaller planes.
// f64 radius-4 stars keep the 64 x 16 tile and a depth-5 ring (the taller f32 tile's ring
// would exceed the 227 KB of shared memory at 8 bytes per element).
template <int RANK, int R, int GEO = 0, int ES = 4> struct StarGeom;
template <int R, int ES> struct StarGeom<3, R, 1, ES> {
  static constexpr int TXT = 32, TYT = 12, PTS = 4, YR = 1;
};
// GEO 3: a 128 x 16 tile with two output rows per thread (YR): the rows share their y
// neighbours (10 instead of 14 LDS.128 per 8 points for SDO4), the per-plane bookkeeping is
// amortised over 8 points, and the taller tile reads 20 rows per 16 instead of 16 per 12
template <int R, int ES> struct StarGeom<3, R, 3, ES> {
  static constexpr int TXT = 32, TYT = 8, PTS = 4, YR = 2;
};
// GEO 2: the wide tile with 8 x-points per thread (half the threads; per-plane overhead --
// waits, stage bookkeeping, addressing -- amortised over twice the points)
template <int R, int ES> struct StarGeom<3, R, 2, ES> {
  static constexpr int TXT = 16, TYT = 12, PTS = 8, YR = 1;
};
template <int R, int ES> struct StarGeom<3, R, 0, ES> {
  static constexpr int PTS = 4, YR = 1;
  static constexpr int TXT = R >= 4 ? HG_TXT_R4 : HG_TXT_R2;
  static constexpr int TYT = R >= 4 ? (ES == 8 ? 16 : HG_TYT_R4) : HG_TYT_R2;
};
template <int R, int ES> struct StarGeom<2, R, 0, ES> {
  static constexpr int TXT = 32, TYT = 1, PTS = 4, YR = 1;
};

#ifndef HG_MINB_G2
#define HG_MINB_G2 3
#endif
// planes per TMA ring slot (1 or 2): with 2, one box of two planes lands on one mbarrier, so
// consumers wait, and release, once per two planes (A/B: HG_ZP=2)
#ifndef HG_ZP
#define HG_ZP 1
#endif
// compile-time 10-slot ring on the 128x12 tile too: rejected before the 35-line pitch (its DRAM
// reads grew 5%), +4% on two boxes after it (profiles/r2_ab.md)
#ifndef HG_GEO1_CT
#define HG_GEO1_CT 1
#endif
// L2 eviction hints on the z-halo planes shared by consecutive chunks (A/B: HG_L2HINT=0)
#ifndef HG_L2HINT
#define HG_L2HINT 1
#endif
// HG_PACK=2: x taps at odd offsets (pairs straddling two registers' halves) add scalar
template <typename T> constexpr bool kPackAdd = HG_PACK == 2 && std::is_same<T, float>::value;
// does a thread owning YR consecutive rows read row d (relative to its first) as a y neighbour?
template <int NT, int YR> __device__ constexpr bool yRowNeeded(int d) {
  for (int yr = 0; yr < YR; ++yr)
    for (int t = 0; t < NT; ++t)
      if (d == yr + Taps<NT>::k(t) || d == yr - Taps<NT>::k(t))
        return true;
  return false;
}

template <typename T> struct StarParams {
  int64_t plane;   // elements between consecutive dim-0 planes
  int64_t pitch;   // elements between rows of the last dim
  int64_t col0;    // element column of raw index 0 of the last dim
  int zs, ys, xs;  // raw start of the output region
  int nz, ny, nx;  // output extents
  int tiles_x, tiles_y, chunk, nchunks;
  // launch order -> unit (chunk * tiles_y + tile_y) * tiles_x + tile_x; the units touching a
  // halo face come last so their waits overlap the interior (null: natural order)
  const int *perm;
  // dmp: before loading any halo row of a face whose neighbour exists, the producer waits
  // until that neighbour's put of this step has landed (flag >= epoch, system-scope acquire)
  const unsigned long long *flags;
  unsigned long long epoch;
  int wmask;     // bit 2*dim + (sign > 0): a neighbour sends into that face
  int band[6];   // units within band[d] of face d wait (their loads reach received cells)
  unsigned long long *err;        // bounded waits (waitFlag)
  unsigned long long timeout_ns;
  // packed x faces: slab [y][z][xw] of the cur buffer's lo/hi x halo, unpacked by the
  // producer warp of the receiving CTAs before their TMA loads
  T *cur;
  const T *xin[2];
  int xw[2];
  int xoz, xoy, xbz, xby, xox[2]; // receive box of the slabs, region-relative
  // fused swap of the NEXT step: output points inside a send box (width hs[d] at face d) are
  // also stored into the neighbour's buffer (peer[d] + my index + pdelta[d]), or for a packed
  // x face (xpack bit d) into the neighbour's slab peer[d]; each face's CTAs count completions
  // and the last one publishes put_epoch to the neighbour's flag
  int fuse;
  int xpack;
  int nodata;    // faces that only signal (deep halos: the rounds between data rounds)
  int hs[6];
  T *peer[6];
  int64_t pdelta[6];
  unsigned int *cnt;
  unsigned int cnt_target[6];
  unsigned long long *peer_flag[6];
  unsigned long long put_epoch;
  T *out;
  T w0, wz[3], wy[3], wx[3], scale, two;
};

template <typename T, int RANK, int NT, int KIND, int GEO = 0> struct StarCfg {
  static constexpr int R = Taps<NT>::R;
  static constexpr int RY = RANK == 3 ? R : 0;
  static constexpr int TXT = StarGeom<RANK, R, GEO, int(sizeof(T))>::TXT,
                       TYT = StarGeom<RANK, R, GEO, int(sizeof(T))>::TYT;
  static constexpr int PTS = StarGeom<RANK, R, GEO, int(sizeof(T))>::PTS; // x-points/thread
  static constexpr int YR = StarGeom<RANK, R, GEO, int(sizeof(T))>::YR;   // rows/thread
  static constexpr int TX = TXT * PTS, TY = TYT * YR;
  static constexpr int PADX = 4;
  static constexpr int CW = TX + 2 * PADX;
  static constexpr int ROWS = TY + 2 * RY;
  static constexpr int NCONS = TXT * TYT;
  static constexpr int NWARPS_C = NCONS / 32;
  static constexpr int NTHREADS = NCONS + 32;
  // CTAs per SM the register budget must allow (f32 3D: 3 for r<=2, 2 for r=4)
  static constexpr int MINB =
      GEO == 1 || GEO == 3 ? 2 : GEO == 2 ? HG_MINB_G2
                   : RANK == 3 ? (sizeof(T) == 4 ? (R <= 2 ? HG_MINB_R2 : HG_MINB_R4) : 1) : 4;
  // f32 3D radius <= 2: the ring is 2Q (heat SDO4) / 3Q (SDO2) slots deep, so the plane loop
  // unrolled over one ring turn has compile-time slot indices (StarCfg::CT; 18% fewer
  // instructions per point on the 128x12 tile, +4% on heat SDO4 1024^3 and 512^3)
  static constexpr int DEPTH =
      RANK == 3 ? (R <= 2 ? (sizeof(T) == 4 && HG_ZP == 1 && (GEO == 0 || HG_GEO1_CT) ? 7 : HG_DEPTH3)
                          : (sizeof(T) == 8 ? 5 : HG_DEPTH3W))
                : HG_DEPTH2;
  static constexpr int ZP = HG_ZP;                  // planes per ring slot
  static constexpr int NS = (R + 1 + DEPTH + ZP - 1) / ZP; // ring slots
  static constexpr int Q = 2 * R + 1;
  // compile-time ring slots: the loop unrolls over NS planes (a multiple of the queue period)
  static constexpr bool CT = ZP == 1 && NS % Q == 0;
  static constexpr int UNROLL = CT ? NS : Q;
  static constexpr int STAGE = ROWS * CW;   // elements of one plane
  // one slot: ZP planes back to back (the TMA box layout), 128-byte aligned
  static constexpr int SSTRIDE = (ZP * STAGE + int(128 / sizeof(T)) - 1) / int(128 / sizeof(T)) * int(128 / sizeof(T));
  static constexpr int PSTAGE = ZP * TY * TX;    // elements (wave prev) per slot
  static constexpr bool WAVE = KIND == kWave;
  static constexpr size_t SMEM =
      128 + sizeof(T) * (size_t(NS) * SSTRIDE + (WAVE ? size_t(NS) * PSTAGE : 0)) +
      2 * NS * sizeof(uint64_t);
};

template <typename T, int RANK, int NT, int KIND, int GEO>
__global__ void __launch_bounds__(StarCfg<T, RANK, NT, KIND, GEO>::NTHREADS,
                                  StarCfg<T, RANK, NT, KIND, GEO>::MINB)
    starKernel(const __grid_constant__ CUtensorMap tmCur,
               const __grid_constant__ CUtensorMap tmPrev, const StarParams<T> P) {
  using C = StarCfg<T, RANK, NT, KIND, GEO>;
  constexpr int R = C::R, RY = C::RY, NS = C::NS, Q = C::Q;
  extern __shared__ __align__(128) unsigned char smraw[];
  // align inside the __shared__ array (pointer stays in the shared window -> LDS, not LD)
  T *stages = reinterpret_cast<T *>(smraw + ((128u - (smemAddr(smraw) & 127u)) & 127u));
  T *pstages = stages + size_t(NS) * C::SSTRIDE;
  uint64_t *full = reinterpret_cast<uint64_t *>(pstages + (C::WAVE ? size_t(NS) * C::PSTAGE : 0));
  uint64_t *empty = full + NS;

  // unit -> (x tile, y tile, z chunk), x fastest
  int u = P.perm ? __ldg(P.perm + blockIdx.x) : int(blockIdx.x);
  const int txi = u % P.tiles_x;
  u /= P.tiles_x;
  const int tyi = u % P.tiles_y;
  const int chunk = u / P.tiles_y;
  const int xb = txi * C::TX, yb = tyi * C::TY;
  const int zb = chunk * P.chunk;
  const int n = tyi < P.tiles_y ? min(P.chunk, P.nz - zb) : 0;
  const int tid = threadIdx.x;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbarInit(&full[s], 1);
      mbarInit(&empty[s], C::NCONS); // every consumer thread arrives (no lane-0 branch)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (n <= 0)
    return;

  // dmp: the faces whose received cells this unit's loads reach (wait for the neighbour's
  // round before loading them)
  int need = 0;
  if (P.flags) {
    constexpr int XD = RANK - 1;
    if (zb < P.band[0]) need |= 1;
    if (zb + n > P.nz - P.band[1]) need |= 2;
    if (RANK == 3 && yb < P.band[2]) need |= 4;
    if (RANK == 3 && min(yb + C::TY, P.ny) > P.ny - P.band[3]) need |= 8;
    if (xb < P.band[2 * XD]) need |= 1 << (2 * XD);
    if (min(xb + C::TX, P.nx) > P.nx - P.band[2 * XD + 1]) need |= 2 << (2 * XD);
    need &= P.wmask;
  }
  // packed x faces: the slab rows this unit's boxes read (its rows and y rim, its planes and
  // z rim, clipped to the receive box) are unpacked into the halo columns by the producer warp,
  // a batch of planes at a time just ahead of the TMA loads that read them, so the consumers
  // start at once and the unpack overlaps their work
  const int xunpack = (need >> (2 * (RANK - 1))) & ((P.xin[0] ? 1 : 0) | (P.xin[1] ? 2 : 0));

  if (tid >= C::NCONS) {
    // ---------------- producer warp ----------------
    const int plane_lane = tid - C::NCONS;
    if (need) {
      if (plane_lane == 0)
        for (int di = 0; di < 6; ++di)
          if (need & (1 << di))
            waitFlag(P.flags + di, P.epoch, P.err, P.timeout_ns,
                     (P.epoch << 8) | (unsigned long long)(di << 1) | 1ull);
      // the halo bytes arrived through the generic proxy; TMA reads via the async proxy
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncwarp();
    }
    // x unpack geometry: rows [uy0, uy1), planes [uz0, uz1) of the region (clipped to the box)
    const int uy0 = RANK == 3 ? max(P.xoy, yb - RY) : 0;
    const int uy1 = RANK == 3 ? min(P.xoy + P.xby, yb + C::TY + RY) : 1;
    const int uz0 = max(P.xoz, zb - R), uz1 = min(P.xoz + P.xbz, zb + n + R);
    int unpacked = xunpack ? uz0 : 1 << 30; // planes below this z (region) are in place
    // unpack planes [unpacked, zEnd) of both x faces with the whole warp, then proxy-fence
    auto unpackTo = [&](int zEnd) {
      zEnd = min(zEnd, uz1);
      if (unpacked >= zEnd)
        return;
#pragma unroll 1
      for (int sd = 0; sd < 2; ++sd) {
        if (!(xunpack & (1 << sd)))
          continue;
        const int W = P.xw[sd];
        const int per = (zEnd - unpacked) * W, total = (uy1 - uy0) * per;
        const T *src0 = P.xin[sd] + (int64_t(uy0 - P.xoy) * P.xbz + (unpacked - P.xoz)) * W;
        const int64_t rowStride = int64_t(P.xbz) * W;
        T *dst0 = P.cur + int64_t(P.zs + unpacked) * P.plane +
                  (RANK == 3 ? int64_t(P.ys + uy0) * P.pitch : 0) + P.col0 + P.xs + P.xox[sd];
        constexpr int B = 8; // independent loads in flight per lane
        for (int k0 = plane_lane; k0 < total; k0 += B * 32) {
          T v[B];
          int64_t o[B];
#pragma unroll
          for (int j = 0; j < B; ++j) {
            const int k = k0 + j * 32;
            if (k < total) {
              const int row = k / per, kk = k - row * per, dz = kk / W;
              v[j] = src0[row * rowStride + kk];
              o[j] = (RANK == 3 ? int64_t(row) * P.pitch : 0) + int64_t(dz) * P.plane +
                     (kk - dz * W);
            }
          }
#pragma unroll
          for (int j = 0; j < B; ++j)
            if (k0 + j * 32 < total)
              dst0[o[j]] = v[j];
        }
      }
      unpacked = zEnd;
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncwarp();
    };
    // with x unpacking the whole warp walks the plane loop; lane 0 issues barriers and TMA
    if (plane_lane == 0 || xunpack) {
      if (plane_lane == 0)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmCur))
                     : "memory");
      const int cx = int(P.col0) + P.xs + xb - C::PADX;
      const int cy = RANK == 3 ? P.ys + yb - RY : 0;
      const int z0 = P.zs + zb - R;
      constexpr int ZP = C::ZP;
      constexpr uint32_t curBytes = uint32_t(ZP * C::STAGE * sizeof(T));
      constexpr uint32_t prevBytes = uint32_t(C::PSTAGE * sizeof(T));
      // z-halo planes shared with the neighbouring chunks of this column: the last 2R planes
      // this chunk loads are the first 2R of the next chunk -- keep them in L2 (evict_last)
      // until that chunk has read them (evict_first), instead of fetching them from HBM twice
      // (heat only: ncu DRAM reads 4.90 -> 4.70 GB per 1024^3 step; the wave kernel, whose
      // prev box shares the stage, measured 4% slower with the hints -- profiles/r1_sweeps.md)
      const bool hintL2 = HG_L2HINT && !C::WAVE && P.nchunks > 1;
      const uint64_t keep = hintL2 ? l2PolicyEvictLast() : 0;
      const uint64_t drop = hintL2 ? l2PolicyEvictFirst() : 0;
      // slot p holds planes p*ZP .. p*ZP+ZP-1 (plane i is z = z0 + i); a plane past the
      // field's end is zero-filled by TMA and never read
      const int nslots = (n + 2 * R + ZP - 1) / ZP;
      constexpr int UNPACK_PLANES = 8; // x unpack batch, ahead of the TMA loads
      for (int p = 0; p < nslots; ++p) {
        const int s = p % NS, i = p * ZP;
        if (xunpack && zb - R + i + ZP > unpacked) // planes z0+i.. need their halo columns
          unpackTo(zb - R + i + ZP + UNPACK_PLANES);
        if (plane_lane != 0)
          continue;
        if (p >= NS)
          mbarWait(&empty[s], uint32_t((p / NS - 1) & 1));
        const bool wantPrev = C::WAVE && i + ZP - 1 >= R && i < n + R;
        mbarExpectTx(&full[s], curBytes + (wantPrev ? prevBytes : 0u));
        if (hintL2 && i + ZP - 1 >= n && zb + n < P.nz)
          tmaLoad3dHint(stages + size_t(s) * C::SSTRIDE, &tmCur, &full[s], cx, cy, z0 + i, keep);
        else if (hintL2 && i < 2 * R && zb > 0)
          tmaLoad3dHint(stages + size_t(s) * C::SSTRIDE, &tmCur, &full[s], cx, cy, z0 + i, drop);
        else
          tmaLoad3d(stages + size_t(s) * C::SSTRIDE, &tmCur, &full[s], cx, cy, z0 + i);
        if (wantPrev)
          tmaLoad3d(pstages + size_t(s) * C::PSTAGE, &tmPrev, &full[s], cx + C::PADX,
                    RANK == 3 ? P.ys + yb : 0, z0 + i);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int tx = tid % C::TXT, ty = tid / C::TXT;
  const int lane = tid & 31;
  constexpr int PTS = C::PTS, NV = PTS / 4; // x-points per thread, 4-vectors per row
  constexpr int YR = C::YR;                 // output rows per thread (tile rows row0 ..)
  const int x0 = tx * PTS;
  const int row0 = ty * YR;
  const int rowOwn = (row0 + RY) * C::CW; // own first row in a stage
  T q[Q][YR][PTS];

  auto release = [&](int s) { mbarArrive(&empty[s]); };

  constexpr int ZP = C::ZP;
  // prologue: planes 0 .. 2R-1 (z = zb-R .. zb+R-1): centres into the queue
#pragma unroll
  for (int i = 0; i < 2 * R; ++i) {
    const int s = (i / ZP) % NS;
    if (i % ZP == 0)
      mbarWait(&full[s], uint32_t((i / ZP / NS) & 1));
#pragma unroll
    for (int yr = 0; yr < YR; ++yr)
#pragma unroll
      for (int h = 0; h < NV; ++h) {
        V4<T> c = ld4(stages + size_t(s) * C::SSTRIDE + (i % ZP) * C::STAGE + rowOwn +
                      yr * C::CW + C::PADX + x0 + 4 * h);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          q[i][yr][4 * h + j] = c.v[j];
      }
  }

  bool yok[YR];
#pragma unroll
  for (int yr = 0; yr < YR; ++yr)
    yok[yr] = RANK == 2 || (yb + row0 + yr < P.ny);
  T *outRow = P.out + (int64_t(P.zs + zb) * P.plane +
                       (RANK == 3 ? int64_t(P.ys + yb + row0) * P.pitch : 0) + P.col0 + P.xs +
                       xb + x0);
  T *dstPlane = outRow; // advanced by one plane per output plane (no per-plane multiply)
  const int xrem = P.nx - (xb + x0);
  // fused-swap geometry: faces this thread's row feeds (y) and x faces of its 4 points
  int blockTouch = 0;
  if (P.fuse) {
    constexpr int XD = RANK - 1;
    // CTA-uniform: which send boxes does this CTA's output region intersect?
    if (P.hs[0] && zb < P.hs[0]) blockTouch |= 1;
    if (P.hs[1] && zb + n > P.nz - P.hs[1]) blockTouch |= 2;
    if (RANK == 3) {
      if (P.hs[2] && yb < P.hs[2]) blockTouch |= 4;
      if (P.hs[3] && min(yb + C::TY, P.ny) > P.ny - P.hs[3]) blockTouch |= 8;
    }
    if (P.hs[2 * XD] && xb < P.hs[2 * XD]) blockTouch |= 1 << (2 * XD);
    if (P.hs[2 * XD + 1] && min(xb + C::TX, P.nx) > P.nx - P.hs[2 * XD + 1])
      blockTouch |= 2 << (2 * XD);
  }

  // slot/sub-plane/parity of the plane arriving, slot/sub-plane of the plane being computed
  // (runtime counters; with C::CT they are compile-time functions of U and the turn parity)
  int sN = ((2 * R) / ZP) % NS, zN = (2 * R) % ZP, phN = ((2 * R) / ZP / NS) & 1;
  int sC = (R / ZP) % NS, zC = R % ZP;
  int turn = 0; // parity of the ring turn (C::CT: the loop advances one turn per iteration)

  // One output plane; U is the position inside the unrolled loop body (a multiple of the
  // Q-periodic register queue), a compile-time constant so every queue index below is a
  // register name.  Returns false past the chunk end.
  auto plane = [&](int m, auto uc) -> bool {
    constexpr int U = decltype(uc)::value;
    if (m >= n)
      return false;
    if constexpr (C::CT) {
      sN = (U + 2 * R) % NS;
      phN = turn ^ (((U + 2 * R) / NS) & 1);
      sC = (U + R) % NS;
    }
    // arrival of plane z+R: its centres enter the queue (one wait per slot)
    if (ZP == 1 || zN == 0)
      mbarWait(&full[sN], uint32_t(phN));
#pragma unroll
    for (int yr = 0; yr < YR; ++yr)
#pragma unroll
      for (int h = 0; h < NV; ++h) {
        const V4<T> c = ld4(stages + size_t(sN) * C::SSTRIDE + zN * C::STAGE + rowOwn +
                            yr * C::CW + C::PADX + x0 + 4 * h);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          q[(U + 2 * R) % Q][yr][4 * h + j] = c.v[j];
      }
    if constexpr (!C::CT) {
      if (++zN == ZP) {
        zN = 0;
        if (++sN == NS) {
          sN = 0;
          phN ^= 1;
        }
      }
    }
    // x / y neighbours of plane z from its stage
    const T *st = stages + size_t(sC) * C::SSTRIDE + zC * C::STAGE;
    V4<T> L[YR], Rr[YR];
#pragma unroll
    for (int yr = 0; yr < YR; ++yr) {
      L[yr] = ld4(st + rowOwn + yr * C::CW + x0);
      Rr[yr] = ld4(st + rowOwn + yr * C::CW + C::PADX + x0 + PTS);
    }
    // rows row0-RY .. row0+YR-1+RY of plane z: the thread's own rows are its queue registers,
    // the y neighbours outside them staged windows, each loaded once even where two own rows
    // share it
    V4<T> yw[YR + 2 * RY][NV];
    if constexpr (RANK == 3) {
#pragma unroll
      for (int d = -RY; d < YR + RY; ++d)
        if ((d < 0 || d >= YR) && yRowNeeded<NT, YR>(d))
#pragma unroll
          for (int h = 0; h < NV; ++h)
            yw[d + RY][h] = ld4(st + rowOwn + d * C::CW + C::PADX + x0 + 4 * h);
    }
    V4<T> pv[YR][NV];
    if constexpr (C::WAVE)
#pragma unroll
      for (int yr = 0; yr < YR; ++yr)
#pragma unroll
        for (int h = 0; h < NV; ++h)
          pv[yr][h] = ld4(pstages + size_t(sC) * C::PSTAGE + zC * (C::TY * C::TX) +
                          (row0 + yr) * C::TX + x0 + 4 * h);
    // the slot is done once its last plane was the computed plane
    const int sDone = (ZP == 1 || zC == ZP - 1) ? sC : -1;
    if constexpr (!C::CT) {
      if (++zC == ZP) {
        zC = 0;
        if (++sC == NS)
          sC = 0;
      }
    }

    constexpr int cz = (U + R) % Q;
    // value of point j in row d (relative to row0) of plane z
    auto yv = [&](int d, int j) -> T {
      return d >= 0 && d < YR ? q[cz][d][j] : yw[d + RY][j / 4].v[j % 4];
    };
    T o[YR][PTS];
#pragma unroll
    for (int yr = 0; yr < YR; ++yr) {
    if constexpr (kPackAdd<T> && PTS == 4) {
      // points (j, j+1): the scalar branch's op sequence, sums and accumulations as f32x2
      auto win = [&](int i) -> T { // window [L | centre | Rr]
        return i < 4 ? L[yr].v[i & 3] : (i < 8 ? q[cz][yr][i & 3] : Rr[yr].v[i & 3]);
      };
      auto mulp = [&](f2 v, T w) -> f2 {
        T a, b;
        upk2(v, a, b);
        return pk2(mul_(a, w), mul_(b, w));
      };
#pragma unroll
      for (int j = 0; j < 4; j += 2) {
        const T c0 = q[cz][yr][j], c1 = q[cz][yr][j + 1];
        f2 acc = pk2(mul_(c0, P.w0), mul_(c1, P.w0));
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int k = Taps<NT>::k(t);
          const int zp = (U + R + k) % Q, zm = (U + R - k + Q) % Q;
          acc = add2(acc, mulp(add2(pk2(q[zp][yr][j], q[zp][yr][j + 1]),
                                    pk2(q[zm][yr][j], q[zm][yr][j + 1])),
                               P.wz[t]));
        }
        if constexpr (RANK == 3) {
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const int k = Taps<NT>::k(t);
            acc = add2(acc, mulp(add2(pk2(yv(yr + k, j), yv(yr + k, j + 1)),
                                      pk2(yv(yr - k, j), yv(yr - k, j + 1))),
                                 P.wy[t]));
          }
        }
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int k = Taps<NT>::k(t);
          f2 sum;
          if (k % 2 == 0) // (4+j+k, 5+j+k) sits inside one 16-byte window: an aligned pair
            sum = add2(pk2(win(4 + j + k), win(5 + j + k)), pk2(win(4 + j - k), win(5 + j - k)));
          else
            sum = pk2(add_(win(4 + j + k), win(4 + j - k)), add_(win(5 + j + k), win(5 + j - k)));
          acc = add2(acc, mulp(sum, P.wx[t]));
        }
        f2 r;
        if constexpr (C::WAVE)
          r = add2(sub2(pk2(mul_(c0, P.two), mul_(c1, P.two)),
                        pk2(pv[yr][0].v[j], pv[yr][0].v[j + 1])),
                   mulp(acc, P.scale));
        else
          r = add2(pk2(c0, c1), mulp(acc, P.scale));
        upk2(r, o[yr][j], o[yr][j + 1]);
      }
    } else {
#pragma unroll
    for (int j = 0; j < PTS; ++j) {
      const T c = q[cz][yr][j];
      // lap = c*W0; then d = 0 (z), 1 (y), rank-1 (x), taps ascending: the generator's
      // op order (kernels.cpp:110-135), one IEEE op at a time
      T acc = mul_(c, P.w0);
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int k = Taps<NT>::k(t);
        acc = add_(acc, mul_(add_(q[(U + R + k) % Q][yr][j], q[(U + R - k + Q) % Q][yr][j]),
                             P.wz[t]));
      }
      if constexpr (RANK == 3) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int k = Taps<NT>::k(t);
          acc = add_(acc, mul_(add_(yv(yr + k, j), yv(yr - k, j)), P.wy[t]));
        }
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int k = Taps<NT>::k(t);
        const int ip = 4 + j + k, im = 4 + j - k; // window [L | centre (PTS) | Rr]
        const T xp = ip < 4 ? L[yr].v[ip & 3]
                            : (ip < 4 + PTS ? q[cz][yr][ip - 4] : Rr[yr].v[(ip - 4 - PTS) & 3]);
        const T xm = im < 4 ? L[yr].v[im & 3]
                            : (im < 4 + PTS ? q[cz][yr][im - 4] : Rr[yr].v[(im - 4 - PTS) & 3]);
        acc = add_(acc, mul_(add_(xp, xm), P.wx[t]));
      }
      if constexpr (C::WAVE)
        o[yr][j] = add_(sub_(mul_(c, P.two), pv[yr][j / 4].v[j % 4]), mul_(acc, P.scale));
      else
        o[yr][j] = add_(c, mul_(acc, P.scale));
    }
    }
    }
#pragma unroll
    for (int yr = 0; yr < YR; ++yr)
      if (yok[yr]) {
        T *dst = dstPlane + (RANK == 3 ? yr * P.pitch : 0);
        if (xrem >= PTS) {
#pragma unroll
          for (int h = 0; h < NV; ++h)
            st4(dst + 4 * h,
                V4<T>{{o[yr][4 * h], o[yr][4 * h + 1], o[yr][4 * h + 2], o[yr][4 * h + 3]}});
        } else {
#pragma unroll
          for (int j = 0; j < PTS; ++j)
            if (j < xrem)
              dst[j] = o[yr][j];
        }
      }
    dstPlane += P.plane;
    // Release a stage only once the values read from it are consumed.  ptxas may schedule an
    // LDS after the arithmetic that precedes the arrive and complete it after the arrive (the
    // SYNCS arrive does not wait for in-flight LDS), so the producer's next TMA could land in
    // the stage first: every consumer thread arrives (the barrier counts NCONS) after its own
    // output stores, whose operands depend on every value it loaded from the stage.  A thread
    // with no store (rows past the domain) uses none of them.  Planes 0..R-1 fed only the
    // queue and go with the first output plane.
    if (sDone >= 0)
      release(sDone);
    if (m == 0) { // slots holding only planes 0..R-1 (never a computed plane)
#pragma unroll
      for (int i = 0; i < R / ZP; ++i)
        release(i % NS);
    }
    return true;
  };

  for (int mb = 0; mb < n; mb += C::UNROLL) {
    unrolled(plane, mb, std::make_integer_sequence<int, C::UNROLL>{});
    turn ^= 1;
  }

  if (P.fuse && blockTouch) {
    // Fused swap of the next step: the send-box points this thread produced (re-read from its
    // own stores, L1/L2-hot) go straight into the neighbours' halos over NVLink.  Done after
    // the plane loop so the streaming loop carries no extra registers.
#pragma unroll 1
    for (int yr = 0; yr < YR; ++yr) {
      if (RANK == 3 && yb + row0 + yr >= P.ny)
        continue;
      constexpr int XD = RANK - 1;
      const T *src = outRow + (RANK == 3 ? yr * P.pitch : 0);
      const int64_t e0 = src - P.out;
      for (int d = 0; d < 2 * RANK; ++d) {
        if (!(blockTouch & (1 << d)) || ((P.xpack | P.nodata) & (1 << d)))
          continue;
        const int dim = d >> 1;
        const bool lo = (d & 1) == 0;
        int m0 = 0, m1 = n; // planes of this chunk inside the send box
        if (dim == 0) {
          if (lo) {
            m1 = min(n, P.hs[d] - zb);
          } else {
            m0 = max(0, P.nz - P.hs[d] - zb);
          }
        } else if (RANK == 3 && dim == 1) {
          const int yo = yb + row0 + yr;
          if (lo ? yo >= P.hs[d] : yo < P.ny - P.hs[d])
            continue;
        }
        constexpr int FULL = (1 << PTS) - 1;
        int jmask = FULL; // x points of this thread inside the box
        if (dim == XD) {
          jmask = 0;
          for (int j = 0; j < PTS; ++j) {
            const int xo = xb + x0 + j;
            if (lo ? xo < P.hs[d] : xo >= P.nx - P.hs[d])
              jmask |= 1 << j;
          }
          if (!jmask)
            continue;
        }
        T *dst = P.peer[d] + e0 + P.pdelta[d];
        // 16-byte copies only when the receive position keeps the 16-byte alignment of the
        // source: an x face between ranks whose core width is not a multiple of 16 bytes
        // (e.g. 50 points per rank) shifts it (misaligned-address fault otherwise)
        const bool vec = (P.pdelta[d] * int64_t(sizeof(T))) % 16 == 0;
        for (int m = m0; m < m1; ++m) {
          const int64_t off = int64_t(m) * P.plane;
          if (vec && jmask == FULL && xrem >= PTS) {
#pragma unroll
            for (int h = 0; h < NV; ++h)
              st4(dst + off + 4 * h, ld4(src + off + 4 * h));
          } else {
            for (int j = 0; j < PTS; ++j)
              if ((jmask >> j & 1) && j < xrem)
                dst[off + j] = src[off + j];
          }
        }
      }
    }
    if (blockTouch & P.xpack & ~P.nodata) {
      // packed x faces: the CTA's rows of the face as slab segments [y][z0..z0+n)[W],
      // contiguous per row, written by all consumer threads in 16-byte stores (each reads the
      // points back from the output rows the CTA just stored; the barrier orders them)
      asm volatile("bar.sync 1, %0;" ::"r"(C::NCONS) : "memory");
      constexpr int XD = RANK - 1;
      const int ny0 = RANK == 3 ? yb : 0;
      const int nrows = RANK == 3 ? min(C::TY, P.ny - yb) : 1;
#pragma unroll 1
      for (int d = 2 * XD; d < 2 * XD + 2; ++d) {
        if (!(blockTouch & P.xpack & ~P.nodata & (1 << d)))
          continue;
        const int W = P.hs[d];
        const int xlo = (d & 1) ? P.nx - W : 0;
        const int per = n * W, gpr = (per + 3) / 4;
        T *slab = P.peer[d];
        for (int g = tid; g < nrows * gpr; g += C::NCONS) {
          const int r = g / gpr, k0 = (g - r * gpr) * 4;
          const int y = ny0 + r;
          const T *src = P.out + int64_t(P.zs + zb) * P.plane +
                         (RANK == 3 ? int64_t(P.ys + y) * P.pitch : 0) + P.col0 + P.xs + xlo;
          T *dst = slab + (int64_t(y) * P.nz + zb) * W + k0;
          T v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int k = k0 + j;
            const int dz = k / W;
            v[j] = k < per ? src[int64_t(dz) * P.plane + (k - dz * W)] : T(0);
          }
          if (k0 + 4 <= per && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
            st4(dst, V4<T>{{v[0], v[1], v[2], v[3]}});
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (k0 + j < per)
                dst[j] = v[j];
          }
        }
      }
    }
    // publish: every face this CTA fed is counted; the last CTA of a face releases the epoch
    __threadfence_system();
    asm volatile("bar.sync 1, %0;" ::"r"(C::NCONS) : "memory");
    if (tid == 0)
      for (int d = 0; d < 6; ++d)
        if (blockTouch & (1 << d)) {
          const unsigned int old = atomicAdd(P.cnt + d, 1u);
          if (old + 1 == P.cnt_target[d]) {
            __threadfence_system();
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P.peer_flag[d] + (d ^ 1)),
                         "l"(P.put_epoch)
                         : "memory");
          }
        }
  }
}

// Unit geometry for the launch order: does unit u (x tile fastest, then y tile, then z chunk)
// touch a face in bmask (bit 2*dim + hi; dims z, [y], x), i.e. come within band[d] of it?
struct UnitGeom {
  int bmask, rank, tiles_x, tiles_y, nchunks, TX, TY, chunk, nx, ny, nz;
  int band[6];
};

__host__ __device__ inline bool unitTouches(const UnitGeom &g, int u) {
  const int tx = u % g.tiles_x, ty = (u / g.tiles_x) % g.tiles_y, c = u / (g.tiles_x * g.tiles_y);
  const int xd = g.rank - 1;
  int m = 0;
  if (c * g.chunk < g.band[0]) m |= 1;
  if (min((c + 1) * g.chunk, g.nz) > g.nz - g.band[1]) m |= 2;
  if (g.rank == 3 && ty * g.TY < g.band[2]) m |= 4;
  if (g.rank == 3 && min((ty + 1) * g.TY, g.ny) > g.ny - g.band[3]) m |= 8;
  if (tx * g.TX < g.band[2 * xd]) m |= 1 << (2 * xd);
  if (min((tx + 1) * g.TX, g.nx) > g.nx - g.band[2 * xd + 1]) m |= 2 << (2 * xd);
  return (m & g.bmask) != 0;
}

// The launch-order table, built on the device by one CTA (a stable partition: interior units
// in natural order, then the boundary units), so building it never blocks the host -- a
// synchronous copy here could wait behind a kernel spinning on a peer's flag.
__global__ void __launch_bounds__(1024) unitOrderKernel(int *out, int total, int ninner,
                                                        const UnitGeom g) {
  __shared__ int scan[1024];
  const int t = threadIdx.x, per = (total + 1023) / 1024;
  const int a = min(total, t * per), b = min(total, a + per);
  int cnt = 0;
  for (int u = a; u < b; ++u)
    cnt += unitTouches(g, u) ? 0 : 1;
  scan[t] = cnt;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) { // inclusive Hillis-Steele scan
    const int v = t >= off ? scan[t - off] : 0;
    __syncthreads();
    scan[t] += v;
    __syncthreads();
  }
  int in = scan[t] - cnt;        // interior units before my range
  int bd = ninner + (a - in);    // boundary slots before my range
  for (int u = a; u < b; ++u)
    out[unitTouches(g, u) ? bd++ : in++] = u;
}

// Launch order of the star units with every unit that touches a face in bmask (within
// band[d] of face d; dims z, [y], x) after all the others, natural order within each group.
// Built once per geometry and cached by the plan; null (natural order) inside a stream
// capture.  Nothing here synchronizes the host with the device.
int unitOrder(UnitOrderCache &cache, int bmask, const int *band, int rank, int tiles_x,
              int tiles_y, int nchunks, int TX, int TY, int chunk, int nx, int ny, int nz,
              cudaStream_t st, const int **perm, int *ninner) {
  *perm = nullptr;
  *ninner = 0;
  std::string key = std::to_string(bmask) + "/" + std::to_string(rank) + "/" +
                    std::to_string(tiles_x) + "/" + std::to_string(tiles_y) + "/" +
                    std::to_string(nchunks) + "/" + std::to_string(TX) + "/" +
                    std::to_string(TY) + "/" + std::to_string(chunk);
  for (int d = 0; d < 6; ++d)
    key += "/" + std::to_string(band[d]);
  auto it = cache.tables.find(key);
  if (it != cache.tables.end()) {
    *perm = it->second;
    *ninner = cache.inner[key];
    return HG_OK;
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return HG_OK;
  }
  UnitGeom g{bmask, rank, tiles_x, tiles_y, nchunks, TX, TY, chunk, nx, ny, nz, {}};
  for (int d = 0; d < 6; ++d)
    g.band[d] = band[d];
  const int total = tiles_x * tiles_y * nchunks;
  int nin = 0; // the split launch needs the interior count on the host
  for (int u = 0; u < total; ++u)
    nin += unitTouches(g, u) ? 0 : 1;
  int *d = nullptr;
  if (cudaMallocAsync(&d, size_t(total) * sizeof(int), st) != cudaSuccess)
    return cudaErr(cudaGetLastError(), "cudaMallocAsync(unit order)");
  unitOrderKernel<<<1, 1024, 0, st>>>(d, total, nin, g);
  if (int rc = cudaErr(cudaGetLastError(), "unit order kernel launch"))
    return rc;
  cache.tables[key] = d;
  cache.inner[key] = nin;
  *perm = d;
  *ninner = nin;
  return HG_OK;
}

template <typename T, int RANK, int NT, int KIND, int GEO = 0>
int launchStarT(StarLaunch &L, cudaStream_t st, int *blocks_out) {
  using C = StarCfg<T, RANK, NT, KIND, GEO>;
  auto kern = starKernel<T, RANK, NT, KIND, GEO>;
  // function attributes are per device: opt in to the large shared-memory carve-out on
  // every device this kernel is launched on
  static std::mutex mu;
  static unsigned long long doneMask = 0;
  int curDev = 0;
  cudaGetDevice(&curDev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!(doneMask & (1ull << (curDev & 63)))) {
      cudaError_t attrErr = cudaFuncSetAttribute(
          kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
      if (attrErr != cudaSuccess)
        return cudaErr(attrErr, "cudaFuncSetAttribute(star)");
      doneMask |= 1ull << (curDev & 63);
    }
  }
  const StarSpec &s = *L.spec;
  StarParams<T> P{};
  int zd = 0, yd = RANK == 3 ? 1 : -1, xd = RANK - 1;
  P.pitch = L.lay.pitch;
  P.plane = RANK == 3 ? L.lay.pitch * L.lay.shape[1] : L.lay.pitch;
  P.col0 = L.lay.col0;
  P.zs = int(L.start[zd]);
  P.ys = RANK == 3 ? int(L.start[yd]) : 0;
  P.xs = int(L.start[xd]);
  P.nz = int(L.ext[zd]);
  P.ny = RANK == 3 ? int(L.ext[yd]) : 1;
  P.nx = int(L.ext[xd]);
  P.tiles_x = (P.nx + C::TX - 1) / C::TX;
  P.tiles_y = (P.ny + C::TY - 1) / C::TY;
  const int ntiles = P.tiles_x * P.tiles_y;
  int chunks = L.chunks;
  // CTAs resident at once (per device; the occupancy query runs once per kernel and device)
  auto residentSlots = [&]() -> long {
    static std::mutex omu;
    static int slots[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(omu);
    int &sl = slots[dev & 63];
    if (sl == 0) {
      int sms = 148, per = 1;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, C::NTHREADS, C::SMEM);
      sl = sms * std::max(per, 1);
    }
    return sl;
  };
  if (chunks <= 0 && RANK == 3) {
    // ~32R planes per chunk: short-lived CTAs keep neighbouring tiles in step (their shared
    // halo rows then hit in L2), while the 2R-plane chunk overlap stays ~6% (measured sweep,
    // profiles/README.md)
    chunks = std::max(1, (P.nz + 16 * C::R) / (32 * C::R));
    // a launch of few waves: its partly empty last wave is a visible share of the step, so
    // take the chunk count up to 1.5x that fills it best (heat 512^3: 8 -> 12 chunks, 4.65 ->
    // 6.97 waves, 636-659 -> 669-673 GPts/s sustained; profiles/r2_ab.md).  Many waves keep
    // the default (1024^3: 37 waves).  Plain single-GPU steps only: the dmp launches keep the
    // chunking their multi-GPU tests ran with.
    const long slots = residentSlots();
    auto fill = [&](int c) {
      const int len = (P.nz + c - 1) / c;
      const long units = long(ntiles) * ((P.nz + len - 1) / len);
      return double(units) / double((units + slots - 1) / slots * slots);
    };
    if (!L.fuse && !L.wait_flags && long(ntiles) * chunks < 10 * slots) {
      int best = chunks;
      for (int c = chunks + 1; c <= std::min(P.nz, chunks + chunks / 2); ++c)
        if (fill(c) > fill(best) + 1e-9)
          best = c;
      chunks = best;
    }
  }
  if (chunks <= 0) {
    // pick the z-chunk count minimising waves x (planes + pipeline fill) per CTA
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, C::NTHREADS, C::SMEM);
    const long resident = long(sms) * std::max(per, 1);
    double best = 1e300;
    chunks = 1;
    for (int c = 1; c <= std::min(P.nz, 512); ++c) {
      const int len = (P.nz + c - 1) / c;
      if (c > 1 && (long(len) * (c - 1) >= P.nz))
        continue; // would leave an empty chunk
      const long units = long(ntiles) * c;
      const long waves = (units + resident - 1) / resident;
      const double cost = double(waves) * (len + 2 * C::R + 12);
      if (cost < best - 1e-9) {
        best = cost;
        chunks = c;
      }
    }
  }
  P.chunk = (P.nz + chunks - 1) / chunks;
  P.nchunks = (P.nz + P.chunk - 1) / P.chunk;
  P.flags = L.wait_flags;
  P.epoch = L.wait_epoch;
  P.wmask = L.wait_mask;
  for (int d = 0; d < 6; ++d) { // default: the units whose loads reach past the region
    const int rd = d / 2 == 0 ? C::R : (RANK == 3 && d / 2 == 1 ? C::RY : C::R);
    // units that send (fused swap) wait too: they store into halos the neighbour reads
    P.band[d] = std::max(std::max(L.band[d] > 0 ? L.band[d] : rd, 1), L.fuse ? L.hs[d] : 0);
  }
  P.err = L.err;
  P.timeout_ns = L.timeout_ns;
  P.cur = static_cast<T *>(L.cur);
  for (int sd = 0; sd < 2; ++sd) {
    P.xin[sd] = static_cast<const T *>(L.xin[sd]);
    P.xw[sd] = L.xw[sd];
  }
  if (L.xbox_set) {
    P.xoz = L.xoz;
    P.xoy = L.xoy;
    P.xbz = L.xbz;
    P.xby = L.xby;
    P.xox[0] = L.xox[0];
    P.xox[1] = L.xox[1];
  } else {
    P.xoz = P.xoy = 0;
    P.xbz = P.nz;
    P.xby = P.ny;
    P.xox[0] = -L.xw[0];
    P.xox[1] = P.nx;
  }
  P.fuse = L.fuse;
  unsigned targets[6] = {0, 0, 0, 0, 0, 0};
  if (L.fuse) {
    // CTAs whose output region meets each face's send box (the kernel's blockTouch)
    auto touching = [](int ext, int tile, int ntl, int h, bool lo) {
      int c = 0;
      for (int i = 0; i < ntl; ++i) {
        const int b = i * tile, e = std::min(b + tile, ext);
        if (lo ? b < h : e > ext - h)
          ++c;
      }
      return c;
    };
    const int nyt = RANK == 3 ? P.tiles_y : 1;
    P.xpack = L.xpack;
    P.nodata = L.nodata;
    for (int d = 0; d < 6; ++d) {
      P.hs[d] = L.hs[d];
      P.peer[d] = static_cast<T *>(L.peer[d]);
      P.pdelta[d] = L.pdelta[d];
      P.peer_flag[d] = L.peer_flag[d];
      if (!L.hs[d])
        continue;
      const int dim = d / 2;
      const bool lo = (d & 1) == 0;
      long c;
      if (dim == 0)
        c = long(touching(P.nz, P.chunk, P.nchunks, L.hs[d], lo)) * P.tiles_x * nyt;
      else if (RANK == 3 && dim == 1)
        c = long(touching(P.ny, C::TY, P.tiles_y, L.hs[d], lo)) * P.tiles_x * P.nchunks;
      else
        c = long(touching(P.nx, C::TX, P.tiles_x, L.hs[d], lo)) * nyt * P.nchunks;
      // cumulative per-face target; committed to the host mirror only once the launch is in
      targets[d] = L.cnt_accum[d] + unsigned(c);
      P.cnt_target[d] = targets[d];
    }
    P.cnt = L.cnt;
    P.put_epoch = L.put_epoch;
  }
  P.out = static_cast<T *>(L.out);
  P.w0 = fromBits<T>(s.w0);
  for (int t = 0; t < 3; ++t) {
    P.wz[t] = fromBits<T>(s.w[0][t]);
    P.wy[t] = fromBits<T>(s.w[RANK == 3 ? 1 : 0][t]);
    P.wx[t] = fromBits<T>(s.w[RANK - 1][t]);
  }
  P.scale = fromBits<T>(s.scale);
  P.two = fromBits<T>(s.two);
  // launch order: the units touching a face that waits for a halo or sends one go last, so
  // their waits (and the peers' flags, published at the end of the peers' previous step)
  // overlap the interior units
  int bmask = L.wait_mask | L.split_mask;
  for (int d = 0; d < 6; ++d)
    if (L.fuse && L.hs[d])
      bmask |= 1 << d;
  if (L.zorder_boundary_last)
    bmask |= 3;
  P.perm = nullptr;
  const unsigned blocks = unsigned(P.tiles_x) * P.tiles_y * P.nchunks;
  int ninner = int(blocks);
  if (bmask && L.order) {
    int rc = unitOrder(*L.order, bmask, P.band, RANK, P.tiles_x, P.tiles_y, P.nchunks, C::TX,
                       C::TY, P.chunk, P.nx, P.ny, P.nz, st, &P.perm, &ninner);
    if (rc)
      return rc;
  }
  if (blocks_out)
    *blocks_out = int(blocks);
  int rc;
  if (L.split_event && P.perm) {
    // the interior units, then (once the halos are in) the units that read them
    if (ninner > 0)
      kern<<<unsigned(ninner), C::NTHREADS, C::SMEM, st>>>(*L.tm_cur, *L.tm_prev, P);
    rc = cudaErr(cudaGetLastError(), "star kernel launch (interior)");
    if (rc)
      return rc;
    rc = cudaErr(cudaStreamWaitEvent(st, L.split_event, 0), "cudaStreamWaitEvent(halo)");
    if (rc)
      return rc;
    StarParams<T> Q = P;
    Q.perm = P.perm + ninner;
    if (blocks > unsigned(ninner))
      kern<<<blocks - unsigned(ninner), C::NTHREADS, C::SMEM, st>>>(*L.tm_cur, *L.tm_prev, Q);
    rc = cudaErr(cudaGetLastError(), "star kernel launch (boundary)");
  } else {
    if (L.split_event) {
      rc = cudaErr(cudaStreamWaitEvent(st, L.split_event, 0), "cudaStreamWaitEvent(halo)");
      if (rc)
        return rc;
    }
    kern<<<blocks, C::NTHREADS, C::SMEM, st>>>(*L.tm_cur, *L.tm_prev, P);
    rc = cudaErr(cudaGetLastError(), "star kernel launch");
  }
  if (rc == HG_OK && L.fuse)
    for (int d = 0; d < 6; ++d)
      if (L.hs[d])
        L.cnt_accum[d] = targets[d];
  return rc;
}

template <typename T, int RANK, int NT, int KIND> int residentT() {
  using C = StarCfg<T, RANK, NT, KIND>;
  auto kern = starKernel<T, RANK, NT, KIND, 0>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, C::NTHREADS, C::SMEM);
  return per;
}

template <typename T, int RANK> int dispatchNT(StarLaunch &L, cudaStream_t st, int *b) {
  const StarSpec &s = *L.spec;
  if constexpr (RANK == 3 && std::is_same_v<T, float>) {
    if (L.geo == 1 && s.kind == kHeat && s.ntaps == 1)
      return launchStarT<T, RANK, 1, kHeat, 1>(L, st, b);
    if (L.geo == 1 && s.kind == kHeat && s.ntaps == 2)
      return launchStarT<T, RANK, 2, kHeat, 1>(L, st, b);
    if (L.geo == 2 && s.kind == kHeat && s.ntaps == 1)
      return launchStarT<T, RANK, 1, kHeat, 2>(L, st, b);
    if (L.geo == 2 && s.kind == kHeat && s.ntaps == 2)
      return launchStarT<T, RANK, 2, kHeat, 2>(L, st, b);
    if (L.geo == 3 && s.kind == kHeat && s.ntaps == 1)
      return launchStarT<T, RANK, 1, kHeat, 3>(L, st, b);
    if (L.geo == 3 && s.kind == kHeat && s.ntaps == 2)
      return launchStarT<T, RANK, 2, kHeat, 3>(L, st, b);
  }
  if (s.kind == kHeat) {
    if (s.ntaps == 1) return launchStarT<T, RANK, 1, kHeat>(L, st, b);
    if (s.ntaps == 2) return launchStarT<T, RANK, 2, kHeat>(L, st, b);
    if (s.ntaps == 3) return launchStarT<T, RANK, 3, kHeat>(L, st, b);
  } else if (s.kind == kWave) {
    if (s.ntaps == 1) return launchStarT<T, RANK, 1, kWave>(L, st, b);
    if (s.ntaps == 2) return launchStarT<T, RANK, 2, kWave>(L, st, b);
    if (s.ntaps == 3) return launchStarT<T, RANK, 3, kWave>(L, st, b);
  }
  return setError(HG_EUNSUPPORTED, "no star kernel for this tap set / kind");
}

template <typename T, int RANK> int residentNT(const StarSpec &s) {
  if (s.kind == kHeat) {
    if (s.ntaps == 1) return residentT<T, RANK, 1, kHeat>();
    if (s.ntaps == 2) return residentT<T, RANK, 2, kHeat>();
    if (s.ntaps == 3) return residentT<T, RANK, 3, kHeat>();
  } else if (s.kind == kWave) {
    if (s.ntaps == 1) return residentT<T, RANK, 1, kWave>();
    if (s.ntaps == 2) return residentT<T, RANK, 2, kWave>();
    if (s.ntaps == 3) return residentT<T, RANK, 3, kWave>();
  }
  return 0;
}

// ---- generic bytecode kernel --------------------------------------------------------------
constexpr int kMaxSlots = 48;

struct GenParams {
  int rank, nops, noperands, nresults;
  int64_t dom_lb[3], dom_ext[3];
  int64_t npts;
  const GOp *ops;
  const void *op_base[HG_MAX_FIELDS];
  DevLayout op_lay[HG_MAX_FIELDS];
  void *out_base[HG_MAX_RESULTS];
  DevLayout out_lay[HG_MAX_RESULTS];
  int64_t st_lb[HG_MAX_RESULTS][3], st_ub[HG_MAX_RESULTS][3];
  int res_slot[HG_MAX_RESULTS];
};

__device__ __forceinline__ int64_t layIndex(const DevLayout &L, const int64_t *p) {
  // element index of logical point p in layout L
  const int r = L.rank;
  int64_t row = 0;
  for (int d = 0; d < r - 1; ++d)
    row = row * L.shape[d] + (p[d] - L.lb[d]);
  return row * L.pitch + L.col0 + (p[r - 1] - L.lb[r - 1]);
}

template <typename T> __global__ void genericKernel(const __grid_constant__ GenParams P) {
  T v[kMaxSlots];
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < P.npts;
       idx += int64_t(gridDim.x) * blockDim.x) {
    int64_t p[3] = {0, 0, 0};
    int64_t rem = idx;
    for (int d = P.rank - 1; d >= 0; --d) {
      p[d] = P.dom_lb[d] + rem % P.dom_ext[d];
      rem /= P.dom_ext[d];
    }
    int64_t base[HG_MAX_FIELDS];
    for (int o = 0; o < P.noperands; ++o)
      base[o] = layIndex(P.op_lay[o], p);
    for (int i = 0; i < P.nops; ++i) {
      const GOp op = P.ops[i];
      switch (op.code) {
      case HG_OP_ACCESS:
        v[op.dst] = static_cast<const T *>(P.op_base[op.operand])[base[op.operand] + op.delta];
        break;
      case HG_OP_CONST:
        v[op.dst] = fromBits<T>(op.bits);
        break;
      case HG_OP_ADD:
        v[op.dst] = add_(v[op.a], v[op.b]);
        break;
      case HG_OP_SUB:
        v[op.dst] = sub_(v[op.a], v[op.b]);
        break;
      case HG_OP_MUL:
        v[op.dst] = mul_(v[op.a], v[op.b]);
        break;
      default:
        v[op.dst] = div_(v[op.a], v[op.b]);
        break;
      }
    }
    for (int k = 0; k < P.nresults; ++k) {
      bool in = true;
      for (int d = 0; d < P.rank; ++d)
        in = in && p[d] >= P.st_lb[k][d] && p[d] < P.st_ub[k][d];
      if (in)
        static_cast<T *>(P.out_base[k])[layIndex(P.out_lay[k], p)] = v[P.res_slot[k]];
    }
  }
}

// ---- stencil.store between two layouts (multi-apply temps -> fields) -----------------------
template <typename T>
__global__ void copyBoxKernel(const T *src, const DevLayout SL, T *dst, const DevLayout DL,
                              int64_t l0, int64_t l1, int64_t l2, int64_t e0, int64_t e1,
                              int64_t e2) {
  const int64_t total = e0 * e1 * e2;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total;
       k += int64_t(gridDim.x) * blockDim.x) {
    int64_t p[3] = {l0 + k / (e1 * e2), l1 + (k / e2) % e1, l2 + k % e2};
    // rank < 3 uses the leading entries only
    dst[layIndex(DL, p)] = src[layIndex(SL, p)];
  }
}

// ---- initializer: exec::fillInit / initValue (buffer.cpp:142-179) ---------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

template <typename T>
__global__ void initKernel(T *base, const DevLayout L, uint64_t seed, int64_t o0, int64_t o1,
                           int64_t o2, int64_t total) {
  const int r = L.rank;
  const int64_t S = L.shape[r - 1];
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = i / S, j = i % S;
    int64_t c[3];
    int64_t rem = row;
    for (int d = r - 2; d >= 0; --d) {
      c[d] = L.lb[d] + rem % L.shape[d];
      rem /= L.shape[d];
    }
    c[r - 1] = L.lb[r - 1] + j;
    const int64_t org[3] = {o0, o1, o2};
    uint64_t h = seed;
    for (int d = 0; d < r; ++d)
      h = mix64(h ^ static_cast<uint64_t>(c[d] + org[d]));
    const double v = static_cast<double>(h >> 11) * 0x1.0p-53;
    base[row * L.pitch + L.col0 + j] = static_cast<T>(v); // f32: cvt.rn.f32.f64
  }
}

// ---- host <-> device field transfer (zero-copy over PCIe) ------------------------------------
// Moves a field between the reference's packed host layout (row-major, halo included,
// buffer.cpp:65-70) and the pitched device layout in ONE pass: the GPU reads (or writes) the
// pinned, device-mapped host buffer directly, one warp per row, coalesced 128-byte requests,
// UNROLL requests in flight per lane.  A pitched cudaMemcpy2DAsync upload runs at ~31 GB/s on
// B200 against ~55 GB/s for a flat copy (tools/xfer_probe.py); this keeps the flat rate and
// needs no staging buffer.  Rows or row parts inside the skip box [slo, shi) (raw indices) are
// not moved: an upload skips the region the next step overwrites before reading it.
template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; };
template <> struct Vec16<double> { using type = double2; };

template <typename T>
__global__ void __launch_bounds__(256) hostXferKernel(T *dev, const DevLayout L, T *host, int up,
                                                      int64_t slo0, int64_t shi0, int64_t slo1,
                                                      int64_t shi1, int64_t slo2, int64_t shi2) {
  // The host array is contiguous (the pitch is a device-side artefact), so threads walk it in
  // 16-byte chunks: one 16-byte PCIe access per thread, 512 bytes per warp instruction, UNROLL
  // in flight per thread.  Each element of a chunk is then placed into its pitched row.
  using V = typename Vec16<T>::type;
  constexpr int NV = 16 / sizeof(T), UNROLL = 4;
  const int r = L.rank;
  const int64_t W = L.shape[r - 1];
  int64_t total = 1;
  for (int d = 0; d < r; ++d)
    total *= L.shape[d];
  const int64_t slo[3] = {slo0, slo1, slo2}, shi[3] = {shi0, shi1, shi2};
  const bool anySkip = slo[r - 1] < shi[r - 1];
  // row -> (inside the skip box in the outer dims, device row offset)
  auto rowInfo = [&](int64_t row, bool &inside) {
    inside = anySkip;
    int64_t rem = row;
    for (int d = r - 2; d >= 0; --d) {
      const int64_t c = rem % L.shape[d];
      rem /= L.shape[d];
      inside = inside && c >= slo[d] && c < shi[d];
    }
    return row * L.pitch + L.col0;
  };
  const int64_t nchunks = (total + NV - 1) / NV;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t c0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c0 < nchunks;
       c0 += stride * UNROLL) {
    V v[UNROLL];
    int64_t row[UNROLL], x[UNROLL], drow[UNROLL];
    bool ins[UNROLL], need[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t c = c0 + stride * u;
      need[u] = c < nchunks;
      if (!need[u])
        continue;
      const int64_t e = c * NV;
      row[u] = e / W;
      x[u] = e - row[u] * W;
      drow[u] = rowInfo(row[u], ins[u]);
      // a chunk entirely inside the skip box (same row, x range inside) is not moved
      if (ins[u] && x[u] >= slo[r - 1] && x[u] + NV <= shi[r - 1] && x[u] + NV <= W)
        need[u] = false;
      if (need[u] && up) {
        if (e + NV <= total)
          v[u] = reinterpret_cast<const V *>(host)[c];
        else
          for (int j = 0; j < NV; ++j)
            reinterpret_cast<T *>(&v[u])[j] = e + j < total ? host[e + j] : T(0);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (!need[u])
        continue;
      const int64_t e = (c0 + stride * u) * NV;
      int64_t rw = row[u], xx = x[u], dr = drow[u];
      bool in = ins[u];
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        if (e + j >= total)
          break;
        if (xx == W) { // the chunk runs into the next row
          ++rw;
          xx = 0;
          dr = rowInfo(rw, in);
        }
        if (up) {
          if (!(in && xx >= slo[r - 1] && xx < shi[r - 1]))
            dev[dr + xx] = reinterpret_cast<const T *>(&v[u])[j];
        } else {
          reinterpret_cast<T *>(&v[u])[j] = dev[dr + xx];
        }
        ++xx;
      }
      if (!up) {
        if (e + NV <= total)
          reinterpret_cast<V *>(host)[c0 + stride * u] = v[u];
        else
          for (int j = 0; j < NV && e + j < total; ++j)
            host[e + j] = reinterpret_cast<const T *>(&v[u])[j];
      }
    }
  }
}

// ---- box copies -----------------------------------------------------------------------------
template <typename T>
__global__ void packKernel(T *base, const DevLayout L, int64_t a0, int64_t a1, int64_t a2,
                           int64_t s0, int64_t s1, int64_t s2, T *packed, int unpack) {
  // packRegion / unpackRegion (simulator.cpp:523-584): row-major over the box
  const int64_t total = s0 * s1 * s2;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total;
       k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i2 = k % s2, i1 = (k / s2) % s1, i0 = k / (s1 * s2);
    int64_t e;
    if (L.rank == 3)
      e = ((a0 + i0) * L.shape[1] + (a1 + i1)) * L.pitch + L.col0 + a2 + i2;
    else if (L.rank == 2)
      e = (a0 + i0) * L.pitch + L.col0 + a1 + i1;
    else
      e = L.col0 + a0 + i0;
    if (unpack)
      base[e] = packed[k];
    else
      packed[k] = base[e];
  }
}

// A packed x-face slab into its receive box (the order putKernel's packed jobs and the fused
// send write: [y][z][x] of the box for rank 3, [z][x] for rank 2).
template <typename T>
__global__ void slabUnpackKernel(T *base, const DevLayout L, int64_t a0, int64_t a1, int64_t a2,
                                 int64_t s0, int64_t s1, int64_t s2, const T *slab) {
  const int64_t total = s0 * s1 * s2;
  for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < total;
       o += int64_t(gridDim.x) * blockDim.x) {
    int64_t e;
    if (L.rank == 3) { // o = (i1 * s0 + i0) * s2 + i2
      const int64_t i2 = o % s2, q = o / s2, i0 = q % s0, i1 = q / s0;
      e = ((a0 + i0) * L.shape[1] + (a1 + i1)) * L.pitch + L.col0 + a2 + i2;
    } else { // o = i0 * s1 + i1
      const int64_t i1 = o % s1, i0 = o / s1;
      e = (a0 + i0) * L.pitch + L.col0 + a1 + i1;
    }
    base[e] = slab[o];
  }
}

struct PutParams {
  PutJob jobs[96];
  int njobs;
  unsigned long long *flags[2 * HG_MAX_RANK];
  int nflags;
  unsigned long long epoch;
  unsigned int *counter;
};

__device__ __forceinline__ int64_t boxElem(const DevLayout &L, const int64_t *at, int64_t i0,
                                           int64_t i1, int64_t i2) {
  if (L.rank == 3)
    return ((at[0] + i0) * L.shape[1] + (at[1] + i1)) * L.pitch + L.col0 + at[2] + i2;
  if (L.rank == 2)
    return (at[0] + i0) * L.pitch + L.col0 + at[1] + i1;
  return L.col0 + at[0] + i0;
}

// Fused pack + NVLink store + unpack: each face box of my buffer is written straight into the
// neighbour's receive box (peer-mapped), byte-exact -- or, for a packed x face, into the
// neighbour's receive slab (the box as [y][z][x] for rank 3, [z][x] for rank 2), which its
// stencil kernel unpacks.  Each job carries its own field's layout.  The last CTA to finish
// publishes the epoch to every neighbour's flag with a system-scope release.
template <typename T> __global__ void putKernel(const __grid_constant__ PutParams P) {
  const PutJob &J = P.jobs[blockIdx.y];
  const DevLayout &L = J.lay;
  // rows of the box (all dims but the last) x contiguous width (the last dim)
  const int64_t rowsEff = L.rank == 3 ? J.size[0] * J.size[1] : (L.rank == 2 ? J.size[0] : 1);
  const int64_t w = L.rank == 3 ? J.size[2] : (L.rank == 2 ? J.size[1] : J.size[0]);
  const T *src = static_cast<const T *>(J.src);
  T *dst = static_cast<T *>(J.dst);
  if (J.packed) {
    // slab element o ([y][z][x] of the box for rank 3, [z][x] for rank 2) <- its box point;
    // four consecutive slab elements per thread, stored as one 16-byte NVLink write (a 4-byte
    // store would cost a whole 32-byte packet each: ncu nvltx 9x the payload)
    const int64_t total = rowsEff * w;
    auto srcOf = [&](int64_t o) {
      const int64_t i2 = o % w, q = o / w;
      if (L.rank == 3) {
        const int64_t i0 = q % J.size[0], i1 = q / J.size[0];
        return boxElem(L, J.src_at, i0, i1, i2);
      }
      return boxElem(L, J.src_at, q, i2, 0);
    };
    const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
    for (int64_t o = 4 * (blockIdx.x * int64_t(blockDim.x) + threadIdx.x); o < total;
         o += 4 * int64_t(gridDim.x) * blockDim.x) {
      T v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        v[j] = o + j < total ? src[srcOf(o + j)] : T(0);
      if (aligned && o + 4 <= total) {
        st4(dst + o, V4<T>{{v[0], v[1], v[2], v[3]}});
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (o + j < total)
            dst[o + j] = v[j];
      }
    }
  } else {
    // 16-byte path when both rows start 16-byte aligned (z/y faces: rows of the core width,
    // starting at the 128-byte-aligned core column)
    constexpr int VE = 16 / sizeof(T);
    const int64_t lastS = L.rank == 3 ? J.src_at[2] : (L.rank == 2 ? J.src_at[1] : J.src_at[0]);
    const int64_t lastD = L.rank == 3 ? J.dst_at[2] : (L.rank == 2 ? J.dst_at[1] : J.dst_at[0]);
    const bool vec = L.rank >= 2 && w % VE == 0 && w >= 16 * VE && (L.col0 + lastS) % VE == 0 &&
                     (L.col0 + lastD) % VE == 0 && L.pitch % VE == 0;
    if (vec) {
      for (int64_t r = blockIdx.x; r < rowsEff; r += gridDim.x) {
        int64_t i0 = L.rank == 3 ? r / J.size[1] : r, i1 = L.rank == 3 ? r % J.size[1] : 0;
        const int64_t se = L.rank == 3 ? boxElem(L, J.src_at, i0, i1, 0)
                                       : boxElem(L, J.src_at, i0, 0, 0);
        const int64_t de = L.rank == 3 ? boxElem(L, J.dst_at, i0, i1, 0)
                                       : boxElem(L, J.dst_at, i0, 0, 0);
        const int4 *s4 = reinterpret_cast<const int4 *>(src + se);
        int4 *d4 = reinterpret_cast<int4 *>(dst + de);
        for (int64_t c = threadIdx.x; c < w / VE; c += blockDim.x)
          d4[c] = s4[c];
      }
    } else {
      // any width (x faces: a few elements per row): one element per thread over the whole
      // box, so narrow rows still keep every thread busy
      const int64_t total = rowsEff * w;
      for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total;
           k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t c = k % w, r = k / w;
        int64_t se, de;
        if (L.rank == 3) {
          const int64_t i0 = r / J.size[1], i1 = r % J.size[1];
          se = boxElem(L, J.src_at, i0, i1, c);
          de = boxElem(L, J.dst_at, i0, i1, c);
        } else if (L.rank == 2) {
          se = boxElem(L, J.src_at, r, c, 0);
          de = boxElem(L, J.dst_at, r, c, 0);
        } else {
          se = boxElem(L, J.src_at, c, 0, 0);
          de = boxElem(L, J.dst_at, c, 0, 0);
        }
        dst[de] = src[se];
      }
    }
  }
  if (P.nflags == 0)
    return;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int total = gridDim.x * gridDim.y;
    const unsigned int prev = atomicAdd(P.counter, 1u);
    if (prev == total - 1) {
      *P.counter = 0;
      __threadfence_system();
      for (int f = 0; f < P.nflags; ++f)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P.flags[f]), "l"(P.epoch)
                     : "memory");
    }
  }
}

struct WaitParams {
  const unsigned long long *flags;
  int idx[6];
  int n;
  unsigned long long epoch;
  unsigned long long *err;
  unsigned long long timeout_ns;
  // ready handshake only: peers' ready words to publish into first
  unsigned long long *peer[6];
  int npeer;
};

// Lane k waits for flags[idx[k]] >= epoch (bounded, waitFlag); with npeer > 0 the lanes
// first publish epoch into the peers' words (system-scope release).
__global__ void waitKernel(const __grid_constant__ WaitParams P) {
  const int k = threadIdx.x;
  if (k < P.npeer) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P.peer[k]), "l"(P.epoch) : "memory");
  }
  if (k < P.n)
    waitFlag(P.flags + P.idx[k], P.epoch, P.err, P.timeout_ns,
             (P.epoch << 8) | (unsigned long long)(P.idx[k] << 1) | 1ull);
  __syncwarp();
  __threadfence_system();
}

} // namespace

// ---- host wrappers ---------------------------------------------------------------------------

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tensorMapEncoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static std::once_flag once;
  std::call_once(once, [&] {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return encode;
}
} // namespace

int makeBoxTensorMap(int dtype, const DevLayout &lay, void *base, const uint32_t box[3],
                     CUtensorMap *out) {
  PFN_cuTensorMapEncodeTiled_v12000 encode = tensorMapEncoder();
  if (!encode)
    return setError(HG_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if (lay.rank != 3)
    return setError(HG_EINVAL, "box tensor maps are 3D");
  const int es = dtype == HG_F32 ? 4 : 8;
  cuuint64_t dims[3] = {cuuint64_t(lay.pitch), cuuint64_t(lay.shape[1]), cuuint64_t(lay.shape[0])};
  cuuint64_t strides[2] = {cuuint64_t(lay.pitch * es), cuuint64_t(lay.pitch * lay.shape[1] * es)};
  cuuint32_t estr[3] = {1, 1, 1};
  cuuint32_t bx[3] = {box[0], box[1], box[2]};
  const CUtensorMapDataType dt =
      dtype == HG_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  CUresult r = encode(out, dt, 3, base, dims, strides, bx, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return setError(HG_ECUDA, "cuTensorMapEncodeTiled(box) failed: " + std::to_string(int(r)));
  return HG_OK;
}

int starGeoFor(const StarSpec &s, int dtype, int rank, const int64_t *ext) {
  // the wide 128 x 12 tile wins on every plane of at least 256 x 64 (tools/geo_ab.py, round 2:
  // +2% at 512^3, +9% on 2048 x 2048 x 512, +15% on 2048 x 512 x 2048); tiny planes keep 64 x 16
  return rank == 3 && dtype == HG_F32 && s.kind == kHeat && s.ntaps <= 2 && ext[1] >= 64 &&
                 ext[2] >= 256
             ? 1
             : 0;
}

int makeStarTensorMaps(const StarSpec &s, int dtype, int rank, const DevLayout &lay, void *base,
                       CUtensorMap *cur, CUtensorMap *prev, int geo) {
  PFN_cuTensorMapEncodeTiled_v12000 encode = tensorMapEncoder();
  if (!encode)
    return setError(HG_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const int es = dtype == HG_F32 ? 4 : 8;
  const int R = s.radius;
  const bool f64 = dtype != HG_F32;
  // geo 2 is geo 1's 128 x 12 tile with 8 points per thread: same boxes; geo 3 is 128 x 16
  const int TX = (rank == 3 ? (geo >= 1 ? StarGeom<3, 1, 1>::TXT
                                        : R >= 4 ? StarGeom<3, 4>::TXT : StarGeom<3, 1>::TXT)
                            : StarGeom<2, 1>::TXT) * 4;
  const int TY = rank == 3 ? (geo == 3 ? StarGeom<3, 1, 3>::TYT * StarGeom<3, 1, 3>::YR
                           : geo >= 1 ? StarGeom<3, 1, 1>::TYT
                                       : R >= 4 ? (f64 ? StarGeom<3, 4, 0, 8>::TYT
                                                       : StarGeom<3, 4>::TYT)
                                                : StarGeom<3, 1>::TYT)
                           : 1;
  const int RY = rank == 3 ? R : 0;
  cuuint64_t dims[3], strides[2];
  dims[0] = cuuint64_t(lay.pitch);
  if (rank == 3) {
    dims[1] = cuuint64_t(lay.shape[1]);
    dims[2] = cuuint64_t(lay.shape[0]);
    strides[0] = cuuint64_t(lay.pitch * es);
    strides[1] = cuuint64_t(lay.pitch * lay.shape[1] * es);
  } else {
    dims[1] = 1;
    dims[2] = cuuint64_t(lay.shape[0]);
    strides[0] = cuuint64_t(lay.pitch * es);
    strides[1] = cuuint64_t(lay.pitch * es);
  }
  cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapDataType dt =
      dtype == HG_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  cuuint32_t boxCur[3] = {cuuint32_t(TX + 8), cuuint32_t(TY + 2 * RY), cuuint32_t(HG_ZP)};
  const CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult r = encode(cur, dt, 3, base, dims, strides, boxCur, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return setError(HG_ECUDA, "cuTensorMapEncodeTiled(cur) failed: " + std::to_string(int(r)));
  cuuint32_t boxPrev[3] = {cuuint32_t(TX), cuuint32_t(TY), cuuint32_t(HG_ZP)};
  r = encode(prev, dt, 3, base, dims, strides, boxPrev, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return setError(HG_ECUDA, "cuTensorMapEncodeTiled(prev) failed: " + std::to_string(int(r)));
  return HG_OK;
}

int launchStar(StarLaunch &L, cudaStream_t st, int *blocks_out) {
  if (L.dtype == HG_F32)
    return L.rank == 3 ? dispatchNT<float, 3>(L, st, blocks_out)
                       : dispatchNT<float, 2>(L, st, blocks_out);
  return L.rank == 3 ? dispatchNT<double, 3>(L, st, blocks_out)
                     : dispatchNT<double, 2>(L, st, blocks_out);
}

int starResidentBlocks(const StarSpec &s, int dtype, int rank) {
  if (dtype == HG_F32)
    return rank == 3 ? residentNT<float, 3>(s) : residentNT<float, 2>(s);
  return rank == 3 ? residentNT<double, 3>(s) : residentNT<double, 2>(s);
}

int launchGeneric(const GenericLaunch &L, cudaStream_t st) {
  if (L.nslots > kMaxSlots)
    return setError(HG_EUNSUPPORTED, "apply region needs more than " +
                                         std::to_string(kMaxSlots) + " live values");
  GenParams P{};
  P.rank = L.rank;
  P.nops = L.nops;
  P.noperands = L.noperands;
  P.nresults = L.nresults;
  P.npts = 1;
  for (int d = 0; d < L.rank; ++d) {
    P.dom_lb[d] = L.dom_lb[d];
    P.dom_ext[d] = L.dom_ext[d];
    P.npts *= L.dom_ext[d];
  }
  P.ops = L.ops_dev;
  for (int o = 0; o < L.noperands; ++o) {
    P.op_base[o] = L.op_base[o];
    P.op_lay[o] = L.op_lay[o];
  }
  for (int k = 0; k < L.nresults; ++k) {
    P.out_base[k] = L.out_base[k];
    P.out_lay[k] = L.out_lay[k];
    P.res_slot[k] = L.res_slot[k];
    for (int d = 0; d < 3; ++d) {
      P.st_lb[k][d] = L.st_lb[k][d];
      P.st_ub[k][d] = L.st_ub[k][d];
    }
  }
  const int threads = 256;
  const int64_t want = (P.npts + threads - 1) / threads;
  const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>(want, 148 * 32)));
  if (L.dtype == HG_F32)
    genericKernel<float><<<blocks, threads, 0, st>>>(P);
  else
    genericKernel<double><<<blocks, threads, 0, st>>>(P);
  return cudaErr(cudaGetLastError(), "generic kernel launch");
}

int launchInit(void *base, const DevLayout &lay, int field, const int64_t *origin,
               cudaStream_t st) {
  int64_t total = 1;
  for (int d = 0; d < lay.rank; ++d)
    total *= lay.shape[d];
  // seed = mix64(fieldIdx + 1), then one mix per coordinate (buffer.cpp:151-156)
  uint64_t x = static_cast<uint64_t>(field) + 1;
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  const uint64_t seed = x ^ (x >> 31);
  const int64_t o0 = origin ? origin[0] : 0, o1 = origin && lay.rank > 1 ? origin[1] : 0,
                o2 = origin && lay.rank > 2 ? origin[2] : 0;
  const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256,
                                                                          148 * 16)));
  if (lay.es == 4)
    initKernel<float><<<blocks, 256, 0, st>>>(static_cast<float *>(base), lay, seed, o0, o1, o2,
                                              total);
  else
    initKernel<double><<<blocks, 256, 0, st>>>(static_cast<double *>(base), lay, seed, o0, o1,
                                               o2, total);
  return cudaErr(cudaGetLastError(), "init kernel launch");
}

int launchCopyBox(const void *src, const DevLayout &sl, void *dst, const DevLayout &dl,
                  const int64_t *lb, const int64_t *ub, cudaStream_t st) {
  int64_t l[3] = {0, 0, 0}, e[3] = {1, 1, 1};
  for (int d = 0; d < sl.rank; ++d) {
    l[d] = lb[d];
    e[d] = ub[d] - lb[d];
  }
  const int64_t total = e[0] * e[1] * e[2];
  if (total <= 0)
    return HG_OK;
  const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256,
                                                                          148 * 16)));
  if (sl.es == 4)
    copyBoxKernel<float><<<blocks, 256, 0, st>>>(static_cast<const float *>(src), sl,
                                                 static_cast<float *>(dst), dl, l[0], l[1], l[2],
                                                 e[0], e[1], e[2]);
  else
    copyBoxKernel<double><<<blocks, 256, 0, st>>>(static_cast<const double *>(src), sl,
                                                  static_cast<double *>(dst), dl, l[0], l[1],
                                                  l[2], e[0], e[1], e[2]);
  return cudaErr(cudaGetLastError(), "copy kernel launch");
}

int launchHostXfer(void *dev, const DevLayout &lay, void *host_dev, int up, const int64_t *skip_lo,
                   const int64_t *skip_hi, cudaStream_t st) {
  int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}; // empty box: move everything
  if (skip_lo && skip_hi)
    for (int d = 0; d < lay.rank; ++d) {
      lo[d] = skip_lo[d];
      hi[d] = skip_hi[d];
    }
  // enough warps to keep ~10 MB of PCIe requests in flight; grid in multiples of the SMs
  const unsigned blocks = 148 * 8;
  if (lay.es == 4)
    hostXferKernel<float><<<blocks, 256, 0, st>>>(static_cast<float *>(dev), lay,
                                                  static_cast<float *>(host_dev), up, lo[0], hi[0],
                                                  lo[1], hi[1], lo[2], hi[2]);
  else
    hostXferKernel<double><<<blocks, 256, 0, st>>>(static_cast<double *>(dev), lay,
                                                   static_cast<double *>(host_dev), up, lo[0],
                                                   hi[0], lo[1], hi[1], lo[2], hi[2]);
  return cudaErr(cudaGetLastError(), "host transfer kernel launch");
}

int launchPackUnpack(void *base, const DevLayout &lay, const int64_t *at, const int64_t *size,
                     void *packed, int unpack, cudaStream_t st) {
  int64_t a[3] = {0, 0, 0}, s[3] = {1, 1, 1};
  for (int d = 0; d < lay.rank; ++d) {
    a[d] = at[d];
    s[d] = size[d];
  }
  // map to (s0,s1,s2) row-major with the last dim of the layout innermost
  int64_t A0, A1, A2, S0, S1, S2;
  if (lay.rank == 3) {
    A0 = a[0]; A1 = a[1]; A2 = a[2]; S0 = s[0]; S1 = s[1]; S2 = s[2];
  } else if (lay.rank == 2) {
    A0 = a[0]; A1 = a[1]; A2 = 0; S0 = s[0]; S1 = s[1]; S2 = 1;
  } else {
    A0 = a[0]; A1 = 0; A2 = 0; S0 = s[0]; S1 = 1; S2 = 1;
  }
  const int64_t total = S0 * S1 * S2;
  if (total <= 0)
    return HG_OK;
  const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256,
                                                                          148 * 16)));
  if (lay.rank == 2) { // kernel indexes (a0+i0, a1+i1) via its rank-2 branch with s2 == 1
    if (lay.es == 4)
      packKernel<float><<<blocks, 256, 0, st>>>(static_cast<float *>(base), lay, A0, A1, 0, S0,
                                                S1, 1, static_cast<float *>(packed), unpack);
    else
      packKernel<double><<<blocks, 256, 0, st>>>(static_cast<double *>(base), lay, A0, A1, 0,
                                                 S0, S1, 1, static_cast<double *>(packed),
                                                 unpack);
  } else {
    if (lay.es == 4)
      packKernel<float><<<blocks, 256, 0, st>>>(static_cast<float *>(base), lay, A0, A1, A2, S0,
                                                S1, S2, static_cast<float *>(packed), unpack);
    else
      packKernel<double><<<blocks, 256, 0, st>>>(static_cast<double *>(base), lay, A0, A1, A2,
                                                 S0, S1, S2, static_cast<double *>(packed),
                                                 unpack);
  }
  return cudaErr(cudaGetLastError(), "pack kernel launch");
}

int launchSlabUnpack(void *base, const DevLayout &lay, const int64_t *at, const int64_t *size,
                     const void *slab, cudaStream_t st) {
  int64_t a[3] = {0, 0, 0}, s[3] = {1, 1, 1};
  for (int d = 0; d < lay.rank; ++d) {
    a[d] = at[d];
    s[d] = size[d];
  }
  const int64_t total = s[0] * s[1] * s[2];
  if (total <= 0)
    return HG_OK;
  const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256,
                                                                          148 * 16)));
  if (lay.es == 4)
    slabUnpackKernel<float><<<blocks, 256, 0, st>>>(static_cast<float *>(base), lay, a[0], a[1],
                                                    a[2], s[0], s[1], s[2],
                                                    static_cast<const float *>(slab));
  else
    slabUnpackKernel<double><<<blocks, 256, 0, st>>>(static_cast<double *>(base), lay, a[0],
                                                     a[1], a[2], s[0], s[1], s[2],
                                                     static_cast<const double *>(slab));
  return cudaErr(cudaGetLastError(), "slab unpack kernel launch");
}

int launchPut(const PutJob *jobs, int njobs, const PutSignal *sig, int nsig,
              unsigned long long epoch, unsigned int *counter, cudaStream_t st) {
  PutParams P{};
  if (njobs > 96)
    return setError(HG_EUNSUPPORTED, "too many exchange jobs in one swap phase");
  for (int j = 0; j < njobs; ++j)
    P.jobs[j] = jobs[j];
  P.njobs = njobs;
  P.nflags = 0;
  for (int f = 0; f < nsig; ++f)
    if (sig[f].flag)
      P.flags[P.nflags++] = sig[f].flag;
  P.epoch = epoch;
  P.counter = counter;
  if (njobs == 0 && P.nflags == 0)
    return HG_OK;
  int64_t maxRows = 1;
  int es = 4;
  for (int j = 0; j < njobs; ++j) {
    const DevLayout &L = jobs[j].lay;
    const int64_t rows = L.rank == 3 ? jobs[j].size[0] * jobs[j].size[1]
                                     : (L.rank == 2 ? jobs[j].size[0] : 1);
    // packed jobs and narrow (non-16-byte) rows run one element per thread
    const int64_t w = jobs[j].size[L.rank - 1];
    const bool flat = jobs[j].packed || w * L.es % 16 != 0 || w * L.es < 256;
    maxRows = std::max(maxRows, flat ? (rows * w + 255) / 256 : rows);
    es = L.es;
  }
  dim3 grid(unsigned(std::min<int64_t>(maxRows, 1184)), unsigned(std::max(njobs, 1)));
  if (njobs == 0) { // flags only: a single CTA with no copy work
    P.jobs[0] = PutJob{};
    P.jobs[0].lay.rank = 1;
    grid = dim3(1, 1);
  }
  if (es == 4)
    putKernel<float><<<grid, 256, 0, st>>>(P);
  else
    putKernel<double><<<grid, 256, 0, st>>>(P);
  return cudaErr(cudaGetLastError(), "put kernel launch");
}

int launchWaitFlags(const unsigned long long *flags, const int *idx, int n,
                    unsigned long long epoch, unsigned long long *err,
                    unsigned long long timeout_ns, cudaStream_t st) {
  if (n <= 0)
    return HG_OK;
  WaitParams P{};
  P.flags = flags;
  P.n = std::min(n, 6);
  for (int k = 0; k < P.n; ++k)
    P.idx[k] = idx[k];
  P.epoch = epoch;
  P.err = err;
  P.timeout_ns = timeout_ns;
  waitKernel<<<1, 32, 0, st>>>(P);
  return cudaErr(cudaGetLastError(), "wait kernel launch");
}

int launchReady(unsigned long long *const *peer_ready, int npeer,
                const unsigned long long *ready, const int *idx, int n,
                unsigned long long epoch, unsigned long long *err,
                unsigned long long timeout_ns, cudaStream_t st) {
  WaitParams P{};
  P.flags = ready;
  P.n = std::min(n, 6);
  for (int k = 0; k < P.n; ++k)
    P.idx[k] = idx[k];
  P.npeer = std::min(npeer, 6);
  for (int k = 0; k < P.npeer; ++k)
    P.peer[k] = peer_ready[k];
  P.epoch = epoch;
  P.err = err;
  P.timeout_ns = timeout_ns;
  if (P.n == 0 && P.npeer == 0)
    return HG_OK;
  waitKernel<<<1, 32, 0, st>>>(P);
  return cudaErr(cudaGetLastError(), "ready kernel launch");
}

} // namespace hg
