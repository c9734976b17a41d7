// resident.cu -- whole-run 2D heat stencil with the fields resident in shared memory.
//
// BASELINE config 1 (heat 2D SDO2, 1024^2 f32, 100 steps) moves 8 MB per step: the per-step
// star kernel is launch/latency-bound there (3.6-3.9 us per step with CUDA-graph replay, most of
// it launch and pipeline fill).  On B200 the two ping-pong fields fit in the 148 SMs' shared
// memory (2 x 4.2 MB against 148 x 227 KB), so one persistent launch runs ALL T steps:
//
//   * CTA c owns a band of store rows [r0, r1) and keeps, for both buffers, the rows
//     [r0 - E, r1 + E) (E = K*R, K = 2 steps per exchange) at full allocated width in shared
//     memory -- each tile with its own buffer's halo ring (the reference never writes outside
//     the store box, interpreter.cpp:683-712, so those cells stay the buffer's initial values).
//   * Temporal blocking: K steps run back to back on the tile, the computed rows shrinking by
//     R per step ([r0 - (K-1-s)R, r1 + (K-1-s)R) at sub-step s); only then do neighbours
//     exchange the E boundary rows of the current time level through L2 (double-buffered
//     exchange slots; f32 values travel in 64-bit words tagged with the block number, so the
//     data is its own flag; f64 uses a per-CTA epoch flag with gpu-scope release/acquire).
//     The redundant rows are recomputed with the same op sequence: bit-identical values.
//   * At the end, each CTA writes the store rows of both tiles back to HBM.
//
// Bit-exactness: the per-point DAG is starKernel's (lap = c*w0, then dim 0 taps ascending,
// then dim 1; u + lap*scale), one IEEE RN op at a time (kernels.cpp:110-135).
// Co-residency of the spinning CTAs is guaranteed by a cooperative launch (<= 1 CTA per SM).
#include "device_util.cuh"
#include "kernels.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#ifndef HG_RES_KMAX
#define HG_RES_KMAX 2
#endif

namespace hg {
namespace {

int cudaErrRes(cudaError_t e, const char *what) {
  if (e == cudaSuccess)
    return HG_OK;
  return setError(HG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// threads per CTA (one CTA per SM): 32 warps for f32 (61-64 registers, no spills; 2% faster
// than 16 warps on config 1), 16 for f64 (which would spill at 64 registers)
template <typename T> constexpr int kResThreads = sizeof(T) == 4 ? 1024 : 512;

template <typename T> struct ResParams {
  T *buf[2];                  // tile 0 = buffer bound to the in slot, tile 1 = the out slot
  T *xbuf;                    // exchange rows [2 parities][G][2 sides][E][nx]
  unsigned long long *flags;  // per CTA: last exchange published (cumulative epochs)
  unsigned long long epoch;   // flags value before this launch
  unsigned tag0;              // f32 tagged exchange: block tags of this launch are tag0+1..
  int64_t pitch, col0;        // device layout
  int H, W;                   // allocated rows / columns (raw)
  int s0r, s0c;               // raw start row / column of the store box
  int ny, nx;                 // store box extents
  int steps, K, E;            // time steps, steps per exchange, exchanged rows (K*R)
  int maxRows;                // largest band
  int SP, PL;                 // shared row pitch (elements) and left pad
  T w0, wz[3], wx[3], scale;
};

template <typename T>
__device__ __forceinline__ void bandOf(int ny, int G, int c, int &r0, int &r1) {
  const int base = ny / G, extra = ny % G;
  r0 = c * base + min(c, extra);
  r1 = r0 + base + (c < extra ? 1 : 0);
}

template <typename T, int NT>
__global__ void __launch_bounds__(kResThreads<T>, 1) residentKernel(const ResParams<T> P) {
  constexpr int NTH = kResThreads<T>;
  constexpr int R = Taps<NT>::R;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
  int r0, r1;
  bandOf<T>(P.ny, G, c, r0, r1);
  const int E = P.E;
  const int tileRows = P.maxRows + 2 * E;
  T *const tile0 = reinterpret_cast<T *>(smraw);
  T *const tile1 = tile0 + size_t(tileRows) * P.SP;
  auto tile = [&](int b) { return b ? tile1 : tile0; }; // no local-memory array
  // tile row i <-> raw row lo + i
  const int lo = P.s0r + r0 - E;
  const int nrows = (r1 - r0) + 2 * E;

  // ---- load both buffers' rows (full allocated width: the halo ring comes along) ----
  for (int b = 0; b < 2; ++b) {
    const T *g = b ? P.buf[1] : P.buf[0];
    T *t = tile(b);
    for (int64_t k = tid; k < int64_t(nrows) * P.W; k += NTH) {
      const int i = int(k / P.W), x = int(k % P.W);
      const int raw = lo + i;
      if (raw >= 0 && raw < P.H)
        t[size_t(i) * P.SP + P.PL + x] = g[int64_t(raw) * P.pitch + P.col0 + x];
    }
  }
  __syncthreads();

  const int ngx = (P.nx + 3) / 4;
  const int gy0 = tid / ngx, gx0 = tid % ngx, dgy = NTH / ngx, dgx = NTH % ngx;
  const int cx = P.PL + P.s0c; // shared column of store column 0 (16-byte aligned)
  // shared-memory offsets stay 32-bit (a tile is < 227 KB): no 64-bit address math per item
  const int SP = P.SP;
  const int rowBase = (P.s0r - lo) * SP + cx; // offset of (store row 0, store column 0)
  const bool vec = (P.nx & 3) == 0; // exchange rows move as 16-byte vectors
  int cur = 0;
  int done = 0, blk = 0;
  while (done < P.steps) {
    const int kk = min(P.K, P.steps - done);
    // f32: the last sub-step before an exchange stores its boundary rows' values straight
    // into my exchange slot as tagged words while it computes them (no separate copy pass)
    using W64 = unsigned long long;
    const bool xchNext = sizeof(T) == 4 && done + kk < P.steps;
    W64 *const mineX = reinterpret_cast<W64 *>(P.xbuf) +
                       (size_t(blk & 1) * G + c) * 2 * (size_t(E) * P.nx);
    const W64 tagX = W64(P.tag0 + unsigned(blk) + 1u) << 32;
    for (int s = 0; s < kk; ++s) {
      const bool xch = xchNext && s == kk - 1;
      const int ylo = max(0, r0 - (kk - 1 - s) * R), yhi = min(P.ny, r1 + (kk - 1 - s) * R);
      const T *in = cur ? tile1 : tile0;
      T *out = cur ? tile0 : tile1;
      // work items: 4 points in each of two consecutive rows (y, y+1), row-pair-major from
      // (ylo, 0); the two rows share their column neighbours' loads (2R+6 LDS.128 for 8
      // points instead of 2(2R+3)).  This thread's walk needs no division.
      int pr = gy0, gx = gx0;
      for (; ylo + 2 * pr < yhi;
           gx += dgx, pr += dgy + (gx >= ngx ? 1 : 0), gx -= gx >= ngx ? ngx : 0) {
        const int y = ylo + 2 * pr, x0 = gx * 4;
        const bool two = y + 1 < yhi;
        const int off = rowBase + y * SP + x0; // tile offset of (y, x0)
        const T *row = in + off;
        V4<T> cen[2 * R + 2]; // centres of rows y-R .. y+1+R
#pragma unroll
        for (int d = 0; d < 2 * R + 2; ++d)
          if (d != 2 * R + 1 || two)
            cen[d] = ld4(row + (d - R) * SP);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && !two)
            break;
          const V4<T> L = ld4(row + h * SP - 4), Rr = ld4(row + h * SP + 4);
          const V4<T> &Cc = cen[R + h];
          V4<T> o;
          if constexpr (HG_PACK == 2 && std::is_same<T, float>::value) {
            // points (j, j+1) as an f32x2 pair for the sums and accumulations, products
            // scalar (the star kernel's packed-add form, kernels.cu); odd x taps add scalar
            auto win = [&](int i) -> T { return i < 4 ? L.v[i & 3] : (i < 8 ? Cc.v[i & 3] : Rr.v[i & 3]); };
            auto mulp = [&](f2 v, T w) -> f2 {
              T a, b;
              upk2(v, a, b);
              return pk2(mul_(a, w), mul_(b, w));
            };
#pragma unroll
            for (int j = 0; j < 4; j += 2) {
              const T c0 = Cc.v[j], c1 = Cc.v[j + 1];
              f2 acc = pk2(mul_(c0, P.w0), mul_(c1, P.w0));
#pragma unroll
              for (int t = 0; t < NT; ++t) {
                const int k = Taps<NT>::k(t);
                acc = add2(acc, mulp(add2(pk2(cen[R + h + k].v[j], cen[R + h + k].v[j + 1]),
                                          pk2(cen[R + h - k].v[j], cen[R + h - k].v[j + 1])),
                                     P.wz[t]));
              }
#pragma unroll
              for (int t = 0; t < NT; ++t) {
                const int k = Taps<NT>::k(t);
                f2 sum;
                if (k % 2 == 0)
                  sum = add2(pk2(win(4 + j + k), win(5 + j + k)),
                             pk2(win(4 + j - k), win(5 + j - k)));
                else
                  sum = pk2(add_(win(4 + j + k), win(4 + j - k)),
                            add_(win(5 + j + k), win(5 + j - k)));
                acc = add2(acc, mulp(sum, P.wx[t]));
              }
              upk2(add2(pk2(c0, c1), mulp(acc, P.scale)), o.v[j], o.v[j + 1]);
            }
          } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const T cc = Cc.v[j];
            T acc = mul_(cc, P.w0);
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              const int k = Taps<NT>::k(t);
              acc = add_(acc, mul_(add_(cen[R + h + k].v[j], cen[R + h - k].v[j]), P.wz[t]));
            }
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              const int k = Taps<NT>::k(t);
              const int ip = 4 + j + k, im = 4 + j - k; // window [L | Cc | Rr]
              const T xp = ip < 4 ? L.v[ip & 3] : (ip < 8 ? Cc.v[ip & 3] : Rr.v[ip & 3]);
              const T xm = im < 4 ? L.v[im & 3] : (im < 8 ? Cc.v[im & 3] : Rr.v[im & 3]);
              acc = add_(acc, mul_(add_(xp, xm), P.wx[t]));
            }
            o.v[j] = add_(cc, mul_(acc, P.scale));
          }
          }
          T *dst = out + off + h * SP;
          if (x0 + 4 <= P.nx) {
            st4(dst, o);
          } else { // the ring columns right of the store box stay untouched
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (x0 + j < P.nx)
                dst[j] = o.v[j];
          }
          if constexpr (sizeof(T) == 4) {
            if (xch) {
              // slot rows: [0, E) = my first E rows, [E, 2E) = my last E rows (a row can be
              // both in a band of fewer than 2E rows)
              const int yy = y + h;
              for (int side = 0; side < 2; ++side) {
                const int r = side == 0 ? yy - r0 : E + yy - (r1 - E);
                if (side == 0 ? yy - r0 >= E : yy < r1 - E)
                  continue;
                W64 *m = mineX + size_t(r) * P.nx + x0;
                if (x0 + 4 <= P.nx && (reinterpret_cast<uintptr_t>(m) & 15) == 0) {
                  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(m),
                               "l"(tagX | __float_as_uint(o.v[0])),
                               "l"(tagX | __float_as_uint(o.v[1])));
                  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(m + 2),
                               "l"(tagX | __float_as_uint(o.v[2])),
                               "l"(tagX | __float_as_uint(o.v[3])));
                } else {
                  for (int j = 0; j < 4; ++j)
                    if (x0 + j < P.nx)
                      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(m + j),
                                   "l"(tagX | __float_as_uint(o.v[j])));
                }
              }
            }
          }
        }
      }
      // (before an exchange the halo rows the poll below writes are not read by this
      // sub-step, and its boundary values already went out: the poll needs no barrier first)
      if (!xch)
        __syncthreads();
      cur ^= 1;
    }
    done += kk;
    if (done >= P.steps)
      break;
    // ---- exchange the E boundary rows of the current level with the band neighbours ----
    const int par = blk & 1;
    const size_t slot = size_t(E) * P.nx;
    if constexpr (sizeof(T) == 4) {
      // f32: every value travels in a 64-bit word with its block tag in the high half, so the
      // word itself is the flag (single-copy atomic): no fence, no flag round trip.  Slot
      // reuse two blocks later is safe: a CTA overwrites slot `par` only after it has read the
      // neighbour's NEXT block, which the neighbour computed from this one.
      W64 *xw = reinterpret_cast<W64 *>(P.xbuf);
      const W64 tg = tagX;
      T *tw = cur ? tile1 : tile0;
      const int nx = P.nx;
      // the neighbours' rows: row r of my 2E halo rows (r < E: above, from the upper band's
      // last E rows; else below, from the lower band's first E rows)
      const W64 *above = xw + (size_t(par) * G + (c - 1)) * 2 * slot + slot;
      const W64 *below = xw + (size_t(par) * G + (c + 1)) * 2 * slot;
      const bool hasAbove = c > 0, hasBelow = c + 1 < G;
      // (no memory clobber: the tag carries validity, the tile store depends on the value)
      auto ldw = [](const W64 *q) {
        W64 w;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(q));
        return w;
      };
      auto srcOf = [&](int r, int x) { // 32-bit row offsets: the slots are < 2^31 words
        return r < E ? above + (r * nx + x) : below + ((r - E) * nx + x);
      };
      auto dstOf = [&](int r) { // tile offset of halo row r at store column 0
        return rowBase + (r < E ? r0 - E + r : r1 + r - E) * SP;
      };
      auto live = [&](int r) { return r < E ? hasAbove : hasBelow; };
      // up to 2K halo rows (R = 1) polled concurrently: one round trip
      constexpr int MW = 2 * HG_RES_KMAX > 4 ? 2 * HG_RES_KMAX : 4;
      for (int x = tid; x < nx; x += NTH) {
        if (2 * E <= MW) {
          W64 w[MW];
#pragma unroll
          for (int r = 0; r < MW; ++r)
            if (r < 2 * E && live(r))
              w[r] = ldw(srcOf(r, x));
#pragma unroll
          for (int r = 0; r < MW; ++r)
            if (r < 2 * E && live(r)) {
              while ((w[r] & ~0xffffffffull) != tg)
                w[r] = ldw(srcOf(r, x));
              tw[dstOf(r) + x] = __uint_as_float(unsigned(w[r]));
            }
        } else {
          for (int r = 0; r < 2 * E; ++r) {
            if (!live(r))
              continue;
            W64 w;
            do {
              w = ldw(srcOf(r, x));
            } while ((w & ~0xffffffffull) != tg);
            tw[dstOf(r) + x] = __uint_as_float(unsigned(w));
          }
        }
      }
      __syncthreads();
      ++blk;
      continue;
    }
    T *mine = P.xbuf + (size_t(par) * G + c) * 2 * slot;
    const T *t = tile(cur);
    if (vec) {
      const int nv = P.nx / 4;
      for (int k = tid; k < 2 * E * nv; k += NTH) {
        const int r = k / nv, v = k - r * nv; // r: slot row (side * E + j)
        const int y = r < E ? r0 + r : r1 - 2 * E + r;
        st4(mine + size_t(r) * P.nx + 4 * v, ld4(t + size_t(P.s0r + y - lo) * P.SP + cx + 4 * v));
      }
    } else {
      for (int k = tid; k < 2 * E * P.nx; k += NTH) {
        const int side = k / (E * P.nx), j = (k / P.nx) % E, x = k % P.nx;
        const int y = side == 0 ? r0 + j : r1 - E + j;
        mine[k] = t[size_t(P.s0r + y - lo) * P.SP + cx + x];
      }
    }
    __syncthreads();
    const unsigned long long want = P.epoch + blk + 1;
    if (tid == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(P.flags + c), "l"(want)
                   : "memory");
      for (int nb = c - 1; nb <= c + 1; nb += 2) {
        if (nb < 0 || nb >= G)
          continue;
        unsigned long long v;
        do {
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(P.flags + nb)
                       : "memory");
        } while (v < want);
      }
    }
    __syncthreads();
    T *tw = tile(cur);
    if (vec) {
      const int nv = P.nx / 4;
      for (int k = tid; k < 2 * E * nv; k += NTH) {
        const int r = k / nv, v = k - r * nv;
        // rows [r0-E, r0) = the upper neighbour's last E rows; [r1, r1+E) = the lower one's first
        const bool top = r < E;
        const int nb = top ? c - 1 : c + 1;
        if (nb < 0 || nb >= G)
          continue;
        const T *src = P.xbuf + (size_t(par) * G + nb) * 2 * slot + (top ? slot : 0) +
                       size_t(top ? r : r - E) * P.nx + 4 * v;
        const int y = top ? r0 - E + r : r1 + r - E;
        V4<T> w;
        if constexpr (sizeof(T) == 4) {
          const float4 a = __ldcg(reinterpret_cast<const float4 *>(src));
          w = {{a.x, a.y, a.z, a.w}};
        } else {
          const double2 a = __ldcg(reinterpret_cast<const double2 *>(src));
          const double2 b = __ldcg(reinterpret_cast<const double2 *>(src) + 1);
          w = {{a.x, a.y, b.x, b.y}};
        }
        st4(tw + size_t(P.s0r + y - lo) * P.SP + cx + 4 * v, w);
      }
    } else {
      for (int k = tid; k < 2 * E * P.nx; k += NTH) {
        const int side = k / (E * P.nx), j = (k / P.nx) % E, x = k % P.nx;
        const int nb = side == 0 ? c - 1 : c + 1;
        if (nb < 0 || nb >= G)
          continue;
        const T *src = P.xbuf + (size_t(par) * G + nb) * 2 * slot;
        const int y = side == 0 ? r0 - E + j : r1 + j;
        const T v = __ldcg(src + (side == 0 ? slot : 0) + size_t(j) * P.nx + x);
        tw[size_t(P.s0r + y - lo) * P.SP + cx + x] = v;
      }
    }
    __syncthreads();
    ++blk;
  }

  // ---- write the band's store rows of both tiles back ----
  for (int b = 0; b < 2; ++b) {
    const T *t = tile(b);
    T *g = b ? P.buf[1] : P.buf[0];
    for (int64_t k = tid; k < int64_t(r1 - r0) * P.nx; k += NTH) {
      const int y = r0 + int(k / P.nx), x = int(k % P.nx);
      g[int64_t(P.s0r + y) * P.pitch + P.col0 + P.s0c + x] =
          t[size_t(P.s0r + y - lo) * P.SP + cx + x];
    }
  }
}

struct ResGeometry {
  int G = 0, K = 0, E = 0, maxRows = 0, SP = 0, PL = 0;
  size_t smem = 0;
};

int numSMs() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0)
      n = 148;
  }
  return n;
}

// Band count, steps per exchange and shared-memory footprint; false if it does not fit.
bool geometry(const ResLaunch &L, ResGeometry &g) {
  const int R = L.spec->radius, es = L.dtype == HG_F32 ? 4 : 8;
  const int W = int(L.lay.shape[1]);
  const int s0c = int(L.start[1]);
  const int ny = int(L.ext[0]);
  g.PL = (4 - s0c % 4) % 4;
  if (g.PL + s0c < 4)
    g.PL += 4;
  g.SP = (g.PL + W + 8 + 3) / 4 * 4;
  const size_t cap = 227 * 1024;
  constexpr int kMax = HG_RES_KMAX; // steps per exchange (r1_sweeps.md; round-2 A/B)
  for (int G = std::min(numSMs(), ny); G >= 1; --G) {
    const int minRows = ny / G, maxRows = (ny + G - 1) / G;
    int K = std::min(kMax, minRows / R); // steps per exchange
    if (K < 1)
      continue;
    while (K > 1 && size_t(2) * (maxRows + 2 * K * R) * g.SP * es > cap)
      --K;
    const size_t smem = size_t(2) * (maxRows + 2 * K * R) * g.SP * es;
    if (smem > cap)
      return false; // fewer bands only grow the tiles
    g.G = G;
    g.K = K;
    g.E = K * R;
    g.maxRows = maxRows;
    g.smem = smem;
    return true;
  }
  return false;
}

template <typename T, int NT> int launchResT(const ResLaunch &L, const ResGeometry &g,
                                             cudaStream_t st) {
  auto kern = residentKernel<T, NT>;
  static std::mutex mu;
  static unsigned long long doneMask = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!(doneMask & (1ull << (dev & 63)))) {
      cudaError_t e =
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (e != cudaSuccess)
        return cudaErrRes(e, "cudaFuncSetAttribute(resident)");
      doneMask |= 1ull << (dev & 63);
    }
  }
  const StarSpec &s = *L.spec;
  ResParams<T> P{};
  P.buf[0] = static_cast<T *>(L.in);
  P.buf[1] = static_cast<T *>(L.out);
  P.xbuf = static_cast<T *>(L.xbuf);
  P.flags = L.flags;
  P.epoch = L.epoch;
  P.tag0 = L.tag0;
  P.pitch = L.lay.pitch;
  P.col0 = L.lay.col0;
  P.H = int(L.lay.shape[0]);
  P.W = int(L.lay.shape[1]);
  P.s0r = int(L.start[0]);
  P.s0c = int(L.start[1]);
  P.ny = int(L.ext[0]);
  P.nx = int(L.ext[1]);
  P.steps = int(L.steps);
  P.K = g.K;
  P.E = g.E;
  P.maxRows = g.maxRows;
  P.SP = g.SP;
  P.PL = g.PL;
  P.w0 = fromBits<T>(s.w0);
  for (int t = 0; t < 3; ++t) {
    P.wz[t] = fromBits<T>(s.w[0][t]);
    P.wx[t] = fromBits<T>(s.w[1][t]);
  }
  P.scale = fromBits<T>(s.scale);
  void *args[] = {&P};
  return cudaErrRes(cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(kern),
                                                dim3(g.G), dim3(kResThreads<T>), args, g.smem, st),
                    "resident kernel launch");
}

} // namespace

bool residentSupported(const ResLaunch &L, size_t *xbufBytes, int *ctas) {
  const StarSpec &s = *L.spec;
  if (s.kind != kHeat || s.rank != 2 || L.ext[0] <= 0 || L.ext[1] <= 0)
    return false;
  ResGeometry g;
  if (!geometry(L, g))
    return false;
  const int es = L.dtype == HG_F32 ? 4 : 8;
  if (xbufBytes) // f32 moves tagged 64-bit words
    *xbufBytes = size_t(2) * g.G * 2 * g.E * size_t(L.ext[1]) * 8;
  (void)es;
  if (ctas)
    *ctas = g.G;
  return true;
}

int launchResident(const ResLaunch &L, cudaStream_t st) {
  ResGeometry g;
  if (!geometry(L, g))
    return setError(HG_EUNSUPPORTED, "resident 2D kernel: fields do not fit in shared memory");
  const int nt = L.spec->ntaps;
  if (L.dtype == HG_F32)
    return nt == 1 ? launchResT<float, 1>(L, g, st)
                   : nt == 2 ? launchResT<float, 2>(L, g, st) : launchResT<float, 3>(L, g, st);
  return nt == 1 ? launchResT<double, 1>(L, g, st)
                 : nt == 2 ? launchResT<double, 2>(L, g, st) : launchResT<double, 3>(L, g, st);
}

} // namespace hg
