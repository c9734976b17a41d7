// kernels.hpp -- launchers of the sm_100a kernels (kernels.cu) used by the host side.
#ifndef HG_KERNELS_HPP
#define HG_KERNELS_HPP

#include "hg_internal.hpp"

#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <string>

namespace hg {

// Device view of one buffer's layout (see makeLayout).
struct DevLayout {
  int64_t shape[3];
  int64_t lb[3];
  int64_t pitch;
  int64_t col0;
  int32_t rank;
  int32_t es;
};

DevLayout devLayout(const Layout &L);

// ---- star family (TMA-pipelined, register-streamed along dim 0) -------------------------
// Device tables mapping launch order -> (tile, chunk) unit with the units that touch a halo
// face last, cached per (face mask, geometry); owned by a plan.
struct UnitOrderCache {
  std::map<std::string, int *> tables;
  std::map<std::string, int> inner; // units before the first boundary unit
  ~UnitOrderCache();
};
struct StarLaunch {
  const StarSpec *spec;
  int dtype;
  int rank;
  // output region, raw indices in the (shared) layout
  int64_t start[3];
  int64_t ext[3];
  DevLayout lay;
  const CUtensorMap *tm_cur;  // tensor map of the buffer bound to the cur operand
  const CUtensorMap *tm_prev; // wave: prev operand (may equal tm_cur otherwise)
  void *out;                  // base of the output buffer allocation
  int chunks;                 // z-chunks (0 = auto)
  int zorder_boundary_last;   // process z-boundary chunks last (dmp overlap)
  int geo = 0;                // tile geometry (starGeoFor); the tensor maps must match
  UnitOrderCache *order = nullptr; // plan-owned unit tables (boundary units last)
  const unsigned long long *wait_flags = nullptr; // dmp: my flag words (null = no wait)
  unsigned long long wait_epoch = 0;
  int wait_mask = 0;
  // per face: units whose region-relative extent comes within band[d] of face d read halo
  // cells (or send) and wait; 0 = the stencil radius (the region is the core)
  int band[6] = {0, 0, 0, 0, 0, 0};
  // bounded waits: after timeout_ns (0 = never) a waiter records (epoch << 8 | face << 1 | 1)
  // in *err and goes on (the host reports HG_ETRAP instead of the GPU hanging)
  unsigned long long *err = nullptr;
  unsigned long long timeout_ns = 0;
  // packed x faces (the last dim): halo columns arrive as a packed slab [y][z][w] that the
  // receiving CTAs' producer warp unpacks into the cur buffer before its TMA loads
  void *cur = nullptr;          // base of the buffer bound to the cur operand
  const void *xin[2] = {};      // my receive slabs of that buffer (lo, hi x face), or null
  int xw[2] = {0, 0};           // their widths
  // receive box of the slabs relative to the output region (deep halos extend the region):
  // z/y origin and extents, first halo column of the lo/hi face; xbox_set = 0: the region is
  // the core (origin 0, extents nz/ny, columns -w and nx)
  int xbox_set = 0, xoz = 0, xoy = 0, xbz = 0, xby = 0, xox[2] = {0, 0};
  // fused swap of the next step (see StarParams in kernels.cu); cnt_accum is host state
  int fuse = 0;
  int xpack = 0;                // bit d: face d is sent packed into the peer's slab peer[d]
  int nodata = 0;               // bit d: face d only signals (count + publish, no payload)
  int hs[6] = {0, 0, 0, 0, 0, 0};
  void *peer[6] = {};
  int64_t pdelta[6] = {0, 0, 0, 0, 0, 0};
  unsigned int *cnt = nullptr;
  unsigned int *cnt_accum = nullptr;
  unsigned long long *peer_flag[6] = {};
  unsigned long long put_epoch = 0;
  // split launch (NCCL transport): the units not touching split_mask's faces first, then a
  // wait for split_event on the stream, then the rest
  cudaEvent_t split_event = nullptr;
  int split_mask = 0;
};
// Creates the TMA descriptor of a buffer for the star family's cur/prev boxes.
int makeStarTensorMaps(const StarSpec &s, int dtype, int rank, const DevLayout &lay,
                       void *base, CUtensorMap *cur, CUtensorMap *prev, int geo);
// Tile geometry of the star kernel for a core of extents ext (dims 0..rank-1).
int starGeoFor(const StarSpec &s, int dtype, int rank, const int64_t *ext);
int launchStar(StarLaunch &L, cudaStream_t st, int *blocks_out);
int starResidentBlocks(const StarSpec &s, int dtype, int rank);

// ---- two-step temporally blocked heat (tb.cu) --------------------------------------------
struct TbLaunch {
  const StarSpec *spec;
  int dtype;
  int64_t start[3], ext[3]; // core region, raw indices in the (shared) layout
  DevLayout lay;
  const CUtensorMap *tm_in; // input buffer, box from tbBox
  void *mid;                // buffer of step t+1 (ring read; core written iff write_mid)
  int write_mid;
  void *out;                // buffer receiving step t+2
  int chunks;               // z-chunks (0 = auto)
};
bool tbSupported(const StarSpec &s, int dtype, int rank);
int tbBox(const StarSpec &s, int dtype, uint32_t box[3]);
int launchTb(const TbLaunch &L, cudaStream_t st, int *blocks_out);
// TMA descriptor of a whole 3D buffer with the given box (inner dimension first)
int makeBoxTensorMap(int dtype, const DevLayout &lay, void *base, const uint32_t box[3],
                     CUtensorMap *out);

// ---- whole-run 2D heat with shared-memory-resident fields (resident.cu) -------------------
struct ResLaunch {
  const StarSpec *spec;
  int dtype;
  DevLayout lay;             // shared by both buffers
  int64_t start[2], ext[2];  // store box, raw indices
  void *in, *out;            // buffers bound to the star's cur operand and its store slot
  void *xbuf;                // exchange rows (residentSupported: bytes)
  unsigned long long *flags; // one word per CTA, monotonically increasing epochs
  unsigned long long epoch;  // larger than every flag value of earlier launches
  unsigned tag0;             // f32: block tags tag0+1 .. tag0+blocks unused by earlier launches
  int64_t steps;
};
bool residentSupported(const ResLaunch &L, size_t *xbufBytes, int *ctas);
int launchResident(const ResLaunch &L, cudaStream_t st);

// ---- generic bytecode kernel ------------------------------------------------------------
struct GenericLaunch {
  int dtype, rank;
  int64_t dom_lb[3], dom_ext[3];
  int nops, nslots, noperands, nresults;
  const GOp *ops_dev;
  const void *op_base[HG_MAX_FIELDS];
  DevLayout op_lay[HG_MAX_FIELDS];
  void *out_base[HG_MAX_RESULTS];
  DevLayout out_lay[HG_MAX_RESULTS];
  int64_t st_lb[HG_MAX_RESULTS][3], st_ub[HG_MAX_RESULTS][3];
  int res_slot[HG_MAX_RESULTS];
};
int launchGeneric(const GenericLaunch &L, cudaStream_t st);

// ---- fields -----------------------------------------------------------------------------
int launchInit(void *base, const DevLayout &lay, int field, const int64_t *origin,
               cudaStream_t st);
// stencil.store between layouts: dst[p] = src[p] for logical points p in [lb, ub)
int launchCopyBox(const void *src, const DevLayout &sl, void *dst, const DevLayout &dl,
                  const int64_t *lb, const int64_t *ub, cudaStream_t st);
// host <-> device copy of a whole field (up = 1: host -> device) through the device-mapped
// pointer of a pinned host buffer in the reference's packed layout; raw box [skip_lo, skip_hi)
// is not moved (both NULL: move everything)
int launchHostXfer(void *dev, const DevLayout &lay, void *host_dev, int up, const int64_t *skip_lo,
                   const int64_t *skip_hi, cudaStream_t st);
// packed x-face slab ([y][z][x] box order for rank 3, [z][x] for rank 2) -> the box at `at`
int launchSlabUnpack(void *base, const DevLayout &lay, const int64_t *at, const int64_t *size,
                     const void *slab, cudaStream_t st);
// box copy between a layout box and a packed array (dir 0 = pack, 1 = unpack)
int launchPackUnpack(void *base, const DevLayout &lay, const int64_t *at, const int64_t *size,
                     void *packed, int unpack, cudaStream_t st);

// ---- halo put (fused pack + NVLink store + unpack) + flags --------------------------------
struct PutJob {
  const void *src;    // my buffer base
  void *dst;          // neighbour's buffer base (peer-mapped), or its packed receive slab
  int64_t src_at[3];  // raw send box origin
  int64_t dst_at[3];  // raw receive box origin in the neighbour (unused when packed)
  int64_t size[3];
  DevLayout lay;      // layout of this field (the neighbour's buffer has the same)
  int packed;         // 1: dst is a slab [y][z][x] of the box (packed x face, rank 3) /
                      //    [z][x] (rank 2)
};
struct PutSignal {
  unsigned long long *flag; // neighbour's flag word (peer-mapped), null = none
};
int launchPut(const PutJob *jobs, int njobs, const PutSignal *sig, int nsig,
              unsigned long long epoch, unsigned int *counter, cudaStream_t st);
// bounded waits (timeout_ns 0 = none): see StarLaunch::err
int launchWaitFlags(const unsigned long long *flags, const int *idx, int n,
                    unsigned long long epoch, unsigned long long *err,
                    unsigned long long timeout_ns, cudaStream_t st);
// receiver-ready handshake: publish `epoch` into each peer's ready word (peer_ready[k]),
// then wait until my ready words ready[idx[k]] reached it
int launchReady(unsigned long long *const *peer_ready, int npeer,
                const unsigned long long *ready, const int *idx, int n,
                unsigned long long epoch, unsigned long long *err,
                unsigned long long timeout_ns, cudaStream_t st);

} // namespace hg

#endif
