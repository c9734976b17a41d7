// dmp.cpp -- the dmp halo swap on device buffers (RankHooks::swap, simulator.cpp:772-834;
// Endpoint/Transport, simulator.cpp:201-260, 409-424, transport.cpp:13-40).
//
// A swap is a set of independent box copies: each exchange's send box (at + offset, inside my
// core) goes to the neighbour's receive box (the mate exchange's `at`, in its halo).  Two
// transports move them:
//
// * P2P (default): NVLink peer stores.  The stencil kernel that PRODUCES a send box stores it
//   into the neighbour's buffer as it finishes (fused swap of the next step); the first step of
//   a run call uses a stand-alone put kernel.  Peer memory is mapped by CUDA IPC between
//   processes, or plain peer pointers inside one process.  Ordering replaces the reference's
//   buffered send / blocking receive: the last CTA of a put publishes an epoch to the
//   neighbour's flag word (system-scope release); the neighbour's halo-reading CTAs wait for it
//   in their producer warp.  Faces of the contiguous last dim (x) would be R values per row,
//   so they travel as a packed slab [y][z][w] per (buffer, face) that the receiving CTAs
//   unpack before their TMA loads.
// * NCCL: the reference's pack -> send/recv -> unpack, with NCCL point-to-point on a
//   high-priority side stream, overlapped with the interior units of the step's stencil launch
//   (the halo-reading units wait for the unpack).
//
// Swaps of a buffer nobody has written since its previous swap are elided (the runtime form of
// eliminate-redundant-swaps, dmp_transforms.cpp:318-359): they would move the very same bytes.
// Waits are bounded: a peer that never publishes yields HG_ETRAP ("rank r, face d, epoch e")
// instead of a hung GPU (the reference reports deadlocks per rank, simulator.cpp:143-173).
#include "plan.hpp"

#include <nccl.h> // types only: libnccl is dlopen'ed when the NCCL transport is selected

#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>

namespace {
constexpr uint32_t kMagic = 0x48474451; // "HGDQ"
constexpr int kDirs = 2 * HG_MAX_RANK;
// my flag words: [di] halo round received on face di; [kReady + di] receiver-ready epochs of
// the neighbour on face di; [kErr] first timed-out wait (epoch << 8 | word << 1 | 1)
constexpr int kReady = 8, kErr = 31;
constexpr size_t kFlagBytes = 256;
constexpr double kDefaultTimeoutS = 30.0;

struct Blob {
  uint32_t magic;
  uint32_t nbuf;
  int64_t rank;
  uint64_t layoutHash;
  int64_t slabElems;
  int64_t bufOffset[HG_MAX_FIELDS]; // buffer pointer - allocation base (HG_DEBUG_GUARDS)
  int64_t slabOffset;
  cudaIpcMemHandle_t flags;
  cudaIpcMemHandle_t slab;
  cudaIpcMemHandle_t buf[HG_MAX_FIELDS];
};

int dirIndex(int dim, int sign) { return 2 * dim + (sign > 0 ? 1 : 0); }

// NCCL entry points (dlopen: no link-time dependency; inside a torch process this resolves to
// the NCCL torch already loaded)
struct NcclApi {
  void *lib = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char *(*errorString)(ncclResult_t) = nullptr;
  std::string why;
};

NcclApi &nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried)
    return api;
  tried = true;
  for (const char *name : {"libnccl.so.2", "libnccl.so"}) {
    api.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (api.lib)
      break;
  }
  if (!api.lib) {
    api.why = std::string("cannot load libnccl.so.2: ") + dlerror();
    return api;
  }
  auto sym = [&](auto &fn, const char *n) {
    fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(api.lib, n));
    if (!fn && api.why.empty())
      api.why = std::string("libnccl lacks ") + n;
  };
  sym(api.getUniqueId, "ncclGetUniqueId");
  sym(api.commInitRank, "ncclCommInitRank");
  sym(api.commDestroy, "ncclCommDestroy");
  sym(api.send, "ncclSend");
  sym(api.recv, "ncclRecv");
  sym(api.groupStart, "ncclGroupStart");
  sym(api.groupEnd, "ncclGroupEnd");
  sym(api.errorString, "ncclGetErrorString");
  if (!api.why.empty())
    api.lib = nullptr;
  return api;
}

int ncclCheck(ncclResult_t r, const char *what) {
  if (r == ncclSuccess)
    return HG_OK;
  return hg::setError(HG_ECUDA, std::string(what) + ": " +
                                    (nccl().errorString ? nccl().errorString(r) : "nccl error"));
}

// One exchange of a swap, resolved for this rank (a neighbour exists).
struct Xjob {
  int swap, field, dir, dim, buffer;
  int64_t send_at[3], recv_at[3], size[3], n;
};

struct NcclState {
  ncclComm_t comm = nullptr;
  cudaStream_t cs = nullptr;   // comm stream (high priority)
  cudaEvent_t packed = nullptr, halo = nullptr;
  std::vector<void *> sbuf, rbuf; // per job slot
  std::vector<size_t> cap;
};
} // namespace

struct hg_dmp {
  hg_plan *plan = nullptr;
  hg_decomp dc{};
  int64_t rank = 0;
  int64_t coord[HG_MAX_RANK] = {0, 0, 0};
  int64_t nbr[kDirs];
  void *peer[kDirs][HG_MAX_FIELDS] = {};
  void *peerBase[kDirs][HG_MAX_FIELDS] = {}; // what cudaIpcOpenMemHandle returned
  char *peerSlab[kDirs] = {};          // the neighbour's slab allocation
  void *peerSlabBase[kDirs] = {};
  unsigned long long *peerFlags[kDirs] = {};
  bool opened[kDirs] = {};
  unsigned long long *flags = nullptr; // my flag words (kFlagBytes)
  unsigned int *counter = nullptr;
  unsigned int *cnt6 = nullptr;        // per-face CTA completion counters of fused swaps
  unsigned int cntAccum[kDirs] = {};   // their cumulative targets (host mirror)
  char *slab = nullptr;                // my packed x-face receive slabs, per (buffer, face)
  int64_t slabElems = 0;               // elements of one slab
  bool xpack = false;                  // star plan on P2P: x faces travel packed
  unsigned long long epoch = 0;
  unsigned long long readyEpoch = 0;
  bool needReady = false;
  bool roundReady = false;             // the previous step's kernel published this round
  std::vector<char> dirty;             // per buffer: written since its last swap
  int64_t bytes = 0;
  int mode = 0;                        // 0 unconnected, 1 ipc, 2 in-process, 3 nccl
  int transport = HG_TRANSPORT_P2P;
  cudaEvent_t putDone = nullptr;
  uint64_t layoutHash = 0;
  unsigned long long *errHost = nullptr; // pinned mirror of flags[kErr], refreshed per call
  unsigned long long timeoutNs = 0;
  bool prof = false;
  NcclState nc;
  // deep halos (communication-avoiding): exchange depth*w-wide halos every `depth` steps;
  // step j of a round of klen steps computes the core extended by (klen-1-j)*unit[dim] toward
  // every neighbour (the same DAG on the same inputs as the neighbour's, so bit-identical)
  int depth = 1;
  int64_t unit[HG_MAX_RANK] = {0, 0, 0};
  int phase = 0, klen = 1;
  // deep halos on a grid that splits several dims: the round's exchange runs dim by dim at
  // the round start, each dim's boxes spanning the halos of the dims exchanged before it, so
  // the corner cells the extended region reads travel too (stand-alone puts, no fused sends)
  bool sequenced = false;
};

namespace hg {
namespace {

int64_t nbrOf(const hg_dmp &d, int dim, int sign) {
  int64_t dir[HG_MAX_RANK] = {0, 0, 0};
  dir[dim] = sign;
  return hg_neighbor_rank(d.dc.ndim, d.rank, dir, d.dc.grid);
}

// The exchange of the same swap template pointing the opposite way (the message the neighbour
// sends us travels along it; tags f*2G+2dim+(sign>0) vs +(sign>0?0:1), simulator.cpp:816-827).
const hg_exchange *mateOf(const hg_swap &s, const hg_exchange &e, int rank) {
  for (int k = 0; k < s.nexchanges; ++k) {
    bool opp = true;
    for (int d = 0; d < rank; ++d)
      if (s.ex[k].to[d] != -e.to[d])
        opp = false;
    if (opp)
      return &s.ex[k];
  }
  return nullptr;
}

int dirOf(const hg_exchange &e, int rank, int *dim, int *sign) {
  *dim = -1;
  *sign = 0;
  for (int q = 0; q < rank; ++q)
    if (e.to[q] != 0) {
      *dim = q;
      *sign = e.to[q] > 0 ? 1 : -1;
    }
  return *dim < 0 ? setError(HG_ETRAP, "exchange direction is all zero") : HG_OK;
}

size_t slabOffset(const hg_dmp &d, int buffer, int side) {
  return (size_t(buffer) * 2 + size_t(side)) * size_t(d.slabElems) *
         size_t(d.plan->lay[0].es);
}

// This step's exchanges of dirty swapped buffers that have a neighbour (marks them clean).
int collectJobs(hg_dmp &d, std::vector<Xjob> &out) {
  hg_plan &p = *d.plan;
  const int r = p.prog.rank;
  for (int si = 0; si < d.dc.nswaps; ++si) {
    const hg_swap &s = d.dc.swaps[si];
    const int b = p.bind[static_cast<size_t>(s.field)];
    if (!d.dirty[static_cast<size_t>(b)])
      continue;
    for (int k = 0; k < s.nexchanges; ++k) {
      const hg_exchange &e = s.ex[k];
      int dim, sign;
      if (int rc = dirOf(e, r, &dim, &sign))
        return rc;
      const int di = dirIndex(dim, sign);
      if (d.nbr[di] < 0)
        continue; // global boundary: no neighbour, nothing sent (simulator.cpp:810-812)
      const hg_exchange *m = mateOf(s, e, r);
      if (!m)
        return setError(HG_EINVAL, "swap template lacks the opposite exchange");
      Xjob j{};
      j.swap = si;
      j.field = s.field;
      j.dir = di;
      j.dim = dim;
      j.buffer = b;
      j.n = 1;
      for (int q = 0; q < 3; ++q) {
        j.send_at[q] = q < r ? e.at[q] + e.offset[q] : 0;
        j.recv_at[q] = q < r ? m->at[q] : 0; // in the neighbour (its mate exchange)
        j.size[q] = q < r ? e.size[q] : 1;
        j.n *= j.size[q];
      }
      out.push_back(j);
    }
    d.dirty[static_cast<size_t>(b)] = 0;
  }
  return HG_OK;
}

// P2P put jobs of this step (x faces into the neighbours' slabs when packed); `sent`, when
// given, receives the exchanges (the neighbours send me the mirror image of them).
int buildPutJobs(hg_dmp &d, std::vector<PutJob> &jobs, bool xpack,
                 std::vector<Xjob> *sent = nullptr) {
  std::vector<Xjob> xs;
  if (int rc = collectJobs(d, xs))
    return rc;
  if (sent)
    *sent = xs;
  hg_plan &p = *d.plan;
  const int r = p.prog.rank;
  for (const Xjob &x : xs) {
    if (!d.peer[x.dir][x.buffer])
      return setError(HG_ESTATE, "neighbour buffers are not connected");
    PutJob j{};
    j.src = p.dptr[static_cast<size_t>(x.buffer)];
    j.lay = devLayout(p.lay[static_cast<size_t>(x.buffer)]);
    const bool packed = xpack && x.dim == r - 1;
    if (packed) {
      if (!d.peerSlab[x.dir] || x.n > d.slabElems)
        return setError(HG_ESTATE, "neighbour slabs are not connected");
      j.dst = d.peerSlab[x.dir] + slabOffset(d, x.buffer, (x.dir ^ 1) & 1);
      j.packed = 1;
    } else {
      j.dst = d.peer[x.dir][x.buffer];
    }
    for (int q = 0; q < 3; ++q) {
      j.src_at[q] = x.send_at[q];
      j.dst_at[q] = x.recv_at[q];
      j.size[q] = x.size[q];
    }
    d.bytes += x.n * p.lay[static_cast<size_t>(x.buffer)].es;
    jobs.push_back(j);
  }
  return HG_OK;
}

uint64_t hashLayouts(const hg_plan &p) {
  std::vector<int64_t> v;
  for (const Layout &L : p.lay) {
    v.push_back(L.rank);
    v.push_back(L.es);
    for (int d = 0; d < 3; ++d)
      v.push_back(L.shape[d]);
    v.push_back(L.pitch);
    v.push_back(L.col0);
  }
  return fnv1a(v.data(), v.size() * sizeof(int64_t));
}

bool starPlan(const hg_plan &p) { return p.an.family == Family::Star && p.prog.nresults == 1; }

// Decode a recorded wait timeout into the reference-style report.
int trapFrom(const hg_dmp &d, unsigned long long code) {
  const unsigned long long ep = code >> 8;
  const int word = int((code >> 1) & 31);
  const int di = word >= kReady ? word - kReady : word;
  char msg[320];
  std::snprintf(msg, sizeof msg,
                "dmp rank %lld: %s from neighbour rank %lld (face: dim %d, %s side) did not "
                "arrive for epoch %llu within %.1f s -- the peer is stuck, dead or out of step",
                static_cast<long long>(d.rank),
                word >= kReady ? "receiver-ready handshake" : "halo round",
                static_cast<long long>(d.nbr[di % kDirs]),
                di / 2, (di & 1) ? "upper" : "lower", ep, double(d.timeoutNs) * 1e-9);
  return setError(HG_ETRAP, msg);
}

int readErr(hg_dmp &d, unsigned long long *code) {
  return cudaCheck(cudaMemcpy(code, d.flags + kErr, sizeof *code, cudaMemcpyDeviceToHost),
                   "cudaMemcpy(err)");
}

int checkSticky(hg_dmp &d) {
  const unsigned long long c = *static_cast<volatile unsigned long long *>(d.errHost);
  return c ? trapFrom(d, c) : HG_OK;
}

// Deep halos: the region of step ph of a round of kl steps -- the core extended by
// (kl-1-ph)*unit toward every neighbour -- and per face the band of units whose loads reach
// received cells (extension + radius).  Below the core in x (the contiguous dim) the
// extension rounds up to 16 bytes so output rows stay 16-byte aligned: the extra columns are
// computed from cells nobody exchanged and are never read (the next steps of the round read
// less, and the round's data exchange rewrites the whole halo).
void deepRegion(const hg_dmp &d, int ph, int kl, int64_t ext[][2], int *band) {
  const hg_plan &p = *d.plan;
  const int r = p.prog.rank;
  const int64_t vec = 16 / p.lay[0].es;
  for (int di = 0; di < 2 * r; ++di) {
    if (d.nbr[di] < 0)
      continue;
    int64_t e = d.depth > 1 ? (kl - 1 - ph) * d.unit[di / 2] : 0;
    if (e > 0 && di == 2 * (r - 1))
      e = (e + vec - 1) / vec * vec;
    ext[di / 2][di & 1] = e;
    band[di] = static_cast<int>(e) + (starPlan(p) ? p.an.star.radius : 1);
  }
}

// Deep halos on a grid splitting several dims: the round's exchange at the round start, one
// split dim after the other (dims in order).  Dim q's boxes span [-W_e, n_e + W_e) in every
// split dim e < q -- the halo rows that dim e's exchange just filled -- so the corner cells of
// the extended region arrive from the diagonal ranks through two hops, as an MPI dimension-
// ordered halo exchange does.  Each dim: a put of the boxes (direct stores), its flag, then a
// wait for the neighbours' puts of that dim.  The neighbours' last step of the previous round
// signalled first (their readers of these halos are done).
int seqRoundStart(hg_dmp &d, bool waitPrev, cudaStream_t st) {
  hg_plan &p = *d.plan;
  const int r = p.prog.rank;
  unsigned long long *err = d.flags + kErr;
  int all[kDirs], na = 0;
  for (int di = 0; di < 2 * r; ++di)
    if (d.nbr[di] >= 0)
      all[na++] = di;
  if (waitPrev && na) {
    if (int rc = launchWaitFlags(d.flags, all, na, d.epoch, err, d.timeoutNs, st))
      return rc;
    ++p.launches;
  }
  std::vector<Xjob> xs;
  if (int rc = collectJobs(d, xs))
    return rc;
  ++d.epoch; // this round's data epoch (every face word gets it from its dim's put)
  // halo widths of the split dims (the template's face boxes)
  int64_t W[HG_MAX_RANK] = {0, 0, 0};
  for (const Xjob &x : xs)
    W[x.dim] = std::max(W[x.dim], x.size[x.dim]);
  for (int q = 0; q < r; ++q) {
    if (d.dc.grid[q] < 2)
      continue;
    std::vector<PutJob> jobs;
    PutSignal sig[2];
    int ns = 0, widx[2], nw = 0;
    for (int sd = 0; sd < 2; ++sd) {
      const int di = 2 * q + sd;
      if (d.nbr[di] < 0)
        continue;
      sig[ns++].flag = d.peerFlags[di] + (di ^ 1);
      widx[nw++] = di;
    }
    for (const Xjob &x : xs) {
      if (x.dim != q)
        continue;
      PutJob j{};
      j.src = p.dptr[static_cast<size_t>(x.buffer)];
      j.dst = d.peer[x.dir][x.buffer];
      j.lay = devLayout(p.lay[static_cast<size_t>(x.buffer)]);
      for (int e = 0; e < 3; ++e) {
        j.src_at[e] = x.send_at[e];
        j.dst_at[e] = x.recv_at[e];
        j.size[e] = x.size[e];
        if (e < q && d.dc.grid[e] > 1) { // span the halos dim e's exchange just filled
          j.src_at[e] -= W[e];
          j.dst_at[e] -= W[e];
          j.size[e] += 2 * W[e];
        }
      }
      int64_t n = 1;
      for (int e = 0; e < r; ++e)
        n *= j.size[e];
      d.bytes += n * p.lay[static_cast<size_t>(x.buffer)].es;
      jobs.push_back(j);
    }
    if (int rc = launchPut(jobs.data(), static_cast<int>(jobs.size()), sig, ns, d.epoch,
                           d.counter, st))
      return rc;
    ++p.launches;
    if (nw) {
      if (int rc = launchWaitFlags(d.flags, widx, nw, d.epoch, err, d.timeoutNs, st))
        return rc;
      ++p.launches;
    }
  }
  return HG_OK;
}

// One time step of this rank on the flag (P2P) protocol: [ready handshake], stand-alone put
// of what the previous step did not fuse, the stencil (halo-reading units wait in-kernel),
// with the NEXT step's swap of the output fused into it unless this is the call's last step.
int dmpStep(hg_dmp &d, int64_t t, int64_t steps, cudaStream_t st, std::vector<cudaEvent_t> *evs) {
  hg_plan &p = *d.plan;
  const hg_program &g = p.prog;
  PutSignal sig[kDirs];
  int nsig = 0, widx[kDirs], nw = 0, mask = 0;
  for (int di = 0; di < kDirs; ++di) {
    if (d.nbr[di] < 0)
      continue;
    sig[nsig++].flag = d.peerFlags[di] + (di ^ 1); // the neighbour receives on its opposite
    widx[nw++] = di;
    mask |= 1 << di;
  }
  auto mark = [&]() {
    if (!evs)
      return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    evs->push_back(e);
  };
  unsigned long long *err = d.flags + kErr;
  const int r = g.rank;
  if (d.depth > 1) {
    if (t == 0) { // a call starts a round: every swapped field goes out at full depth width
      d.phase = 0;
      std::fill(d.dirty.begin(), d.dirty.end(), 1);
    }
    if (d.phase == 0)
      d.klen = static_cast<int>(std::min<int64_t>(d.depth, steps - t));
  }
  const int ph = d.depth > 1 ? d.phase : 0, kl = d.depth > 1 ? d.klen : 1;
  int64_t ext[HG_MAX_RANK][2] = {{0, 0}, {0, 0}, {0, 0}};
  int band[kDirs] = {0, 0, 0, 0, 0, 0};
  deepRegion(d, ph, kl, ext, band);
  // 0. receiver-ready handshake after host uploads (hg_dmp_invalidate is collective): no
  //    neighbour may put into my buffers before my uploads into them are done
  const bool handshake = d.needReady;
  if (d.needReady) {
    ++d.readyEpoch;
    unsigned long long *pr[kDirs] = {};
    int ridx[kDirs] = {};
    for (int k = 0; k < nw; ++k) {
      pr[k] = d.peerFlags[widx[k]] + kReady + (widx[k] ^ 1);
      ridx[k] = kReady + widx[k];
    }
    if (int rc = launchReady(pr, nw, d.flags, ridx, nw, d.readyEpoch, err, d.timeoutNs, st))
      return rc;
    if (nw)
      ++p.launches;
    d.needReady = false;
  }
  const bool star = starPlan(p);
  if (d.sequenced) {
    // deep halos over several split dims: exchange at the round start, no in-kernel waits,
    // the round's last step signals its halo readers' completion
    if (ph == 0)
      if (int rc = seqRoundStart(d, d.epoch > 0 && !handshake, st))
        return rc;
    for (int q = 0; q < r; ++q) {
      p.regionExt[q][0] = ext[q][0];
      p.regionExt[q][1] = ext[q][1];
    }
    std::vector<int> written;
    for (int k = 0; k < storedCount(g); ++k)
      written.push_back(p.bind[static_cast<size_t>(storedField(g, k))]);
    bool signalled = false;
    if (ph == kl - 1 && nw) {
      StarLaunch F{};
      for (int di = 0; di < 2 * r; ++di)
        if (d.nbr[di] >= 0) {
          F.hs[di] = band[di];
          F.nodata |= 1 << di;
          F.peer_flag[di] = d.peerFlags[di];
        }
      F.fuse = 1;
      F.cnt = d.cnt6;
      F.cnt_accum = d.cntAccum;
      F.put_epoch = d.epoch + 1;
      p.fuse = F;
      signalled = true;
    }
    if (int rc = planStep(p, st))
      return rc;
    for (int b : written)
      d.dirty[static_cast<size_t>(b)] = 1;
    if (signalled)
      ++d.epoch;
    d.phase = (ph + 1) % kl;
    return HG_OK;
  }
  // deep halos: the call's first put rewrites halos the neighbours read in the last step of
  // their previous call (e.g. wave's prev band), so it waits for the signal round that step
  // published (after a ready handshake everybody's earlier work is done anyway)
  if (d.depth > 1 && t == 0 && d.epoch > 0 && !handshake && nw) {
    if (int rc = launchWaitFlags(d.flags, widx, nw, d.epoch, err, d.timeoutNs, st))
      return rc;
    ++p.launches;
  }
  // 1. stand-alone put of every dirty swapped buffer (x faces packed into the neighbours'
  //    slabs; the symmetric dirty state tells me which of my slabs the neighbours fill)
  std::vector<PutJob> jobs;
  std::vector<Xjob> sent;
  if (int rc = buildPutJobs(d, jobs, d.xpack, d.xpack ? &sent : nullptr))
    return rc;
  mark();
  if (!d.roundReady || !jobs.empty()) {
    ++d.epoch;
    if (int rc = launchPut(jobs.data(), static_cast<int>(jobs.size()), sig, nsig, d.epoch,
                           d.counter, st))
      return rc;
    if (nsig || !jobs.empty())
      ++p.launches;
  }
  // x slabs of buffers other than this step's cur (e.g. wave's prev on a call's first step):
  // unpacked here, once the round is in; the stencil kernel unpacks cur's slab itself
  {
    const int bCurNow = star ? p.bind[static_cast<size_t>(g.operand_field[p.an.star.cur_operand])]
                             : -1;
    bool waited = false;
    for (const Xjob &x : sent) {
      if (x.dim != g.rank - 1 || (star && x.buffer == bCurNow))
        continue;
      if (!waited) {
        if (int rc = launchWaitFlags(d.flags, widx, nw, d.epoch, err, d.timeoutNs, st))
          return rc;
        ++p.launches;
        waited = true;
      }
      // my receive box on that face: the `at` of my exchange toward the sender
      int64_t at[3] = {0, 0, 0};
      const hg_swap &sw0 = d.dc.swaps[x.swap];
      for (int k = 0; k < sw0.nexchanges; ++k) {
        int dim2, sign2;
        dirOf(sw0.ex[k], g.rank, &dim2, &sign2);
        if (dirIndex(dim2, sign2) == x.dir)
          for (int q = 0; q < g.rank; ++q)
            at[q] = sw0.ex[k].at[q];
      }
      if (int rc = launchSlabUnpack(p.dptr[static_cast<size_t>(x.buffer)],
                                    devLayout(p.lay[static_cast<size_t>(x.buffer)]), at, x.size,
                                    d.slab + slabOffset(d, x.buffer, x.dir & 1), st))
        return rc;
      ++p.launches;
    }
  }
  // 2. the stencil step; halo-reading CTAs wait for the round in-kernel
  if (star && nw) {
    p.waitFlags = d.flags;
    p.waitEpoch = d.epoch;
    p.waitMask = mask;
    p.waitErr = err;
    p.waitTimeout = d.timeoutNs;
    for (int q = 0; q < r; ++q) {
      p.regionExt[q][0] = ext[q][0];
      p.regionExt[q][1] = ext[q][1];
    }
    for (int di = 0; di < kDirs; ++di)
      p.band[di] = band[di];
    if (d.xpack && ph == 0) { // the cur buffer's x halo arrives packed (every data round)
      const int xd = g.rank - 1;
      const int bCur =
          p.bind[static_cast<size_t>(g.operand_field[p.an.star.cur_operand])];
      for (int sd = 0; sd < 2; ++sd) {
        const int di = 2 * xd + sd;
        p.xin[sd] = nullptr;
        if (d.nbr[di] < 0)
          continue;
        // width of the receive box on that face: the template's x exchange of the cur slot
        int w = 0;
        for (int k = 0; k < d.dc.nswaps; ++k)
          if (d.dc.swaps[k].field == g.operand_field[p.an.star.cur_operand])
            for (int e = 0; e < d.dc.swaps[k].nexchanges; ++e)
              if (d.dc.swaps[k].ex[e].to[xd] == (sd ? 1 : -1))
                w = static_cast<int>(d.dc.swaps[k].ex[e].size[xd]);
        if (w > 0) {
          p.xin[sd] = d.slab + slabOffset(d, bCur, sd);
          p.xw[sd] = w;
        }
      }
      if (d.depth > 1) { // the receive box relative to the (extended) region
        const hg_bounds &sb = g.store[0];
        p.xboxSet = true;
        p.xbox[0] = static_cast<int>(ext[0][0]);
        p.xbox[1] = r == 3 ? static_cast<int>(ext[1][0]) : 0;
        p.xbox[2] = static_cast<int>(sb.ub[0] - sb.lb[0]);
        p.xbox[3] = r == 3 ? static_cast<int>(sb.ub[1] - sb.lb[1]) : 1;
        p.xbox[4] = static_cast<int>(ext[xd][0]) - p.xw[0];
        p.xbox[5] = static_cast<int>(ext[xd][0] + sb.ub[xd] - sb.lb[xd]);
      }
    }
  } else if (nw) {
    if (int rc = launchWaitFlags(d.flags, widx, nw, d.epoch, err, d.timeoutNs, st))
      return rc;
    ++p.launches;
  }
  // 3. fuse the NEXT step's swap of the output into this kernel (not on the last step of
  //    the call: the reference swaps a buffer only right before it is loaded)
  std::vector<int> written;
  for (int k = 0; k < storedCount(g); ++k)
    written.push_back(p.bind[static_cast<size_t>(storedField(g, k))]);
  const int bOut = written[0];
  int nextSlot = -1; // the argument slot the output buffer occupies next step
  for (size_t i = 0; i < p.an.src.size(); ++i)
    if (p.an.src[i] == storedField(g, 0))
      nextSlot = static_cast<int>(i);
  const hg_swap *sw = nullptr;
  for (int k = 0; k < d.dc.nswaps && nextSlot >= 0; ++k)
    if (d.dc.swaps[k].field == nextSlot)
      sw = &d.dc.swaps[k];
  bool fused = false;
  bool signalOnly = false;
  if (star && nw && (ph < kl - 1 || (d.depth > 1 && t + 1 == steps))) {
    // a step inside a deep round (or the last step of a deep call): no payload, but its
    // halo-reading units signal the neighbours when done (who may then overwrite those halos
    // in the round's last step, or in the first put of the next call)
    StarLaunch F{};
    for (int di = 0; di < 2 * r; ++di)
      if (d.nbr[di] >= 0) {
        F.hs[di] = band[di]; // the units that read received cells in this step signal
        F.nodata |= 1 << di;
        F.peer_flag[di] = d.peerFlags[di];
      }
    F.fuse = 1;
    F.cnt = d.cnt6;
    F.cnt_accum = d.cntAccum;
    F.put_epoch = d.epoch + 1;
    p.fuse = F;
    fused = signalOnly = true;
  } else if (star && nw && sw && t + 1 < steps) {
    StarLaunch F{};
    const Layout &L = p.lay[static_cast<size_t>(bOut)];
    const int r = g.rank;
    int64_t stride[3] = {0, 0, 1};
    if (r == 3) {
      stride[0] = L.pitch * L.shape[1];
      stride[1] = L.pitch;
    } else {
      stride[0] = L.pitch;
    }
    // the fused send covers a band of width size[dim] at the face of the stored region over
    // the whole region in the other dims: check that the exchange box is exactly that
    const hg_bounds &sb = g.store[0];
    bool ok = true;
    int64_t payload = 0;
    for (int k = 0; k < sw->nexchanges && ok; ++k) {
      const hg_exchange &e = sw->ex[k];
      int dim, sign;
      if (dirOf(e, r, &dim, &sign)) {
        ok = false;
        break;
      }
      const int di = dirIndex(dim, sign);
      if (d.nbr[di] < 0)
        continue;
      const hg_exchange *m = mateOf(*sw, e, r);
      if (!m || !d.peer[di][bOut])
        return setError(HG_ESTATE, "neighbour buffers are not connected");
      for (int q = 0; q < r; ++q) {
        const int64_t lo = sb.lb[q] - L.lb[q], ext = sb.ub[q] - sb.lb[q];
        const int64_t a = e.at[q] + e.offset[q];
        if (q != dim ? (a != lo || e.size[q] != ext)
                     : (sign < 0 ? a != lo : a + e.size[q] != lo + ext) || e.size[q] > ext)
          ok = false;
      }
      if (!ok)
        break;
      int64_t n = 1;
      for (int q = 0; q < r; ++q)
        n *= e.size[q];
      F.hs[di] = static_cast<int>(e.size[dim]);
      F.peer_flag[di] = d.peerFlags[di];
      if (d.xpack && dim == r - 1) {
        if (!d.peerSlab[di] || n > d.slabElems)
          return setError(HG_ESTATE, "neighbour slabs are not connected");
        F.peer[di] = d.peerSlab[di] + slabOffset(d, bOut, (di ^ 1) & 1);
        F.xpack |= 1 << di;
      } else {
        int64_t delta = 0;
        for (int q = 0; q < r; ++q)
          delta += (m->at[q] - (e.at[q] + e.offset[q])) * (r == 3 ? stride[q] : (q == 0 ? stride[0] : 1));
        F.peer[di] = d.peer[di][bOut];
        F.pdelta[di] = delta;
      }
      payload += n * L.es;
    }
    if (ok) {
      F.fuse = 1;
      F.cnt = d.cnt6;
      F.cnt_accum = d.cntAccum;
      F.put_epoch = d.epoch + 1;
      p.fuse = F;
      d.bytes += payload;
      fused = true;
    } else if (d.depth > 1) {
      return setError(HG_EUNSUPPORTED, "deep halos need the fused swap (exchange boxes that "
                                       "are bands of the core)");
    }
  }
  mark();
  if (int rc = planStep(p, st))
    return rc;
  mark();
  for (size_t k = 1; k < written.size(); ++k) // (multi-store programs never fuse)
    d.dirty[static_cast<size_t>(written[k])] = 1;
  d.dirty[static_cast<size_t>(bOut)] = fused && !signalOnly ? 0 : 1;
  if (fused)
    ++d.epoch;
  d.roundReady = fused;
  if (d.depth > 1)
    d.phase = (ph + 1) % kl;
  return HG_OK;
}

// One time step on the NCCL transport: pack the dirty send boxes on the compute stream, NCCL
// send/recv + unpack on the comm stream, the stencil's interior units meanwhile, then the
// units that read the halos (star plans; other families wait for the halos first).
int ncclStep(hg_dmp &d, int64_t t, int64_t steps, cudaStream_t st) {
  hg_plan &p = *d.plan;
  NcclApi &api = nccl();
  const int r0 = p.prog.rank;
  if (d.depth > 1) {
    if (t == 0) {
      d.phase = 0;
      std::fill(d.dirty.begin(), d.dirty.end(), 1);
    }
    if (d.phase == 0)
      d.klen = static_cast<int>(std::min<int64_t>(d.depth, steps - t));
  }
  const int ph = d.depth > 1 ? d.phase : 0, kl = d.depth > 1 ? d.klen : 1;
  {
    int64_t ext[HG_MAX_RANK][2] = {{0, 0}, {0, 0}, {0, 0}};
    int band[kDirs] = {0, 0, 0, 0, 0, 0};
    deepRegion(d, ph, kl, ext, band);
    for (int q = 0; q < r0; ++q) {
      p.regionExt[q][0] = ext[q][0];
      p.regionExt[q][1] = ext[q][1];
    }
    for (int di = 0; di < kDirs; ++di)
      p.band[di] = band[di];
  }
  std::vector<Xjob> xs;
  if (ph == 0) // deep halos: one exchange per round
    if (int rc = collectJobs(d, xs))
      return rc;
  int mask = 0;
  for (int di = 0; di < kDirs; ++di)
    if (d.nbr[di] >= 0)
      mask |= 1 << di;
  if (!xs.empty()) {
    NcclState &S = d.nc;
    const size_t es = static_cast<size_t>(p.lay[0].es);
    const int r = p.prog.rank;
    // my receive box of each exchange: the `at` of my exchange toward that neighbour
    std::vector<Xjob> mine = xs;
    for (size_t k = 0; k < xs.size(); ++k) {
      const hg_swap &sw = d.dc.swaps[xs[k].swap];
      for (int e = 0; e < sw.nexchanges; ++e) {
        int dim, sign;
        dirOf(sw.ex[e], r, &dim, &sign);
        if (dirIndex(dim, sign) == xs[k].dir)
          for (int q = 0; q < r; ++q)
            mine[k].recv_at[q] = sw.ex[e].at[q];
      }
    }
    // deep halos over several split dims: dim-ordered stages whose boxes span the halos of
    // the dims before them (corners travel through two hops, as in seqRoundStart)
    if (d.sequenced) {
      int64_t W[HG_MAX_RANK] = {0, 0, 0};
      for (const Xjob &x : xs)
        W[x.dim] = std::max(W[x.dim], x.size[x.dim]);
      for (size_t k = 0; k < xs.size(); ++k) {
        xs[k].n = 1;
        for (int e = 0; e < r; ++e) {
          if (e < xs[k].dim && d.dc.grid[e] > 1) {
            xs[k].send_at[e] -= W[e];
            mine[k].recv_at[e] -= W[e];
            xs[k].size[e] += 2 * W[e];
          }
          xs[k].n *= xs[k].size[e];
        }
      }
    }
    if (S.sbuf.size() < xs.size()) {
      S.sbuf.resize(xs.size(), nullptr);
      S.rbuf.resize(xs.size(), nullptr);
      S.cap.resize(xs.size(), 0);
    }
    for (size_t k = 0; k < xs.size(); ++k) {
      const size_t need = static_cast<size_t>(xs[k].n) * es;
      if (S.cap[k] < need) {
        cudaFree(S.sbuf[k]);
        cudaFree(S.rbuf[k]);
        S.sbuf[k] = S.rbuf[k] = nullptr;
        S.cap[k] = 0;
        if (int rc = cudaCheck(cudaMalloc(&S.sbuf[k], need), "cudaMalloc(nccl send)"))
          return rc;
        if (int rc = cudaCheck(cudaMalloc(&S.rbuf[k], need), "cudaMalloc(nccl recv)"))
          return rc;
        S.cap[k] = need;
      }
    }
    // the comm stream starts once this step's inputs are final (the previous step is done)
    if (int rc = cudaCheck(cudaEventRecord(S.packed, st), "cudaEventRecord"))
      return rc;
    if (int rc = cudaCheck(cudaStreamWaitEvent(S.cs, S.packed, 0), "cudaStreamWaitEvent"))
      return rc;
    const ncclDataType_t dt = es == 4 ? ncclFloat32 : ncclFloat64;
    // stages: every exchange at once, or (sequenced) one split dim after the other
    for (int stage = 0; stage < (d.sequenced ? r : 1); ++stage) {
      auto inStage = [&](const Xjob &x) { return !d.sequenced || x.dim == stage; };
      for (size_t k = 0; k < xs.size(); ++k) {
        if (!inStage(xs[k]))
          continue;
        if (int rc = launchPackUnpack(p.dptr[static_cast<size_t>(xs[k].buffer)],
                                      devLayout(p.lay[static_cast<size_t>(xs[k].buffer)]),
                                      xs[k].send_at, xs[k].size, S.sbuf[k], 0, S.cs))
          return rc;
        ++p.launches;
      }
      if (int rc = ncclCheck(api.groupStart(), "ncclGroupStart"))
        return rc;
      for (size_t k = 0; k < xs.size(); ++k) {
        if (!inStage(xs[k]))
          continue;
        const int peer = static_cast<int>(d.nbr[xs[k].dir]);
        const size_t n = static_cast<size_t>(xs[k].n);
        ncclResult_t r1 = api.send(S.sbuf[k], n, dt, peer, S.comm, S.cs);
        ncclResult_t r2 = api.recv(S.rbuf[k], n, dt, peer, S.comm, S.cs);
        if (r1 != ncclSuccess || r2 != ncclSuccess) {
          api.groupEnd();
          return ncclCheck(r1 != ncclSuccess ? r1 : r2, "ncclSend/ncclRecv");
        }
        d.bytes += xs[k].n * static_cast<int64_t>(es);
      }
      if (int rc = ncclCheck(api.groupEnd(), "ncclGroupEnd"))
        return rc;
      for (size_t k = 0; k < xs.size(); ++k) {
        if (!inStage(xs[k]))
          continue;
        if (int rc = launchPackUnpack(p.dptr[static_cast<size_t>(xs[k].buffer)],
                                      devLayout(p.lay[static_cast<size_t>(xs[k].buffer)]),
                                      mine[k].recv_at, xs[k].size, S.rbuf[k], 1, S.cs))
          return rc;
        ++p.launches;
      }
    }
    if (int rc = cudaCheck(cudaEventRecord(S.halo, S.cs), "cudaEventRecord"))
      return rc;
    if (starPlan(p)) {
      p.splitEvent = S.halo;
      p.splitMask = mask;
    } else if (int rc = cudaCheck(cudaStreamWaitEvent(st, S.halo, 0), "cudaStreamWaitEvent")) {
      return rc;
    }
  }
  const hg_program &g = p.prog;
  std::vector<int> written;
  for (int k = 0; k < storedCount(g); ++k)
    written.push_back(p.bind[static_cast<size_t>(storedField(g, k))]);
  if (int rc = planStep(p, st))
    return rc;
  for (int b : written)
    d.dirty[static_cast<size_t>(b)] = 1;
  if (d.depth > 1)
    d.phase = (ph + 1) % kl;
  return HG_OK;
}

void freeDmp(hg_dmp *d) {
  if (!d)
    return;
  if (d->nc.comm && nccl().commDestroy)
    nccl().commDestroy(d->nc.comm);
  for (void *b : d->nc.sbuf)
    cudaFree(b);
  for (void *b : d->nc.rbuf)
    cudaFree(b);
  if (d->nc.cs)
    cudaStreamDestroy(d->nc.cs);
  if (d->nc.packed)
    cudaEventDestroy(d->nc.packed);
  if (d->nc.halo)
    cudaEventDestroy(d->nc.halo);
  if (d->mode == 1)
    for (int di = 0; di < kDirs; ++di)
      if (d->opened[di]) {
        for (int b = 0; b < HG_MAX_FIELDS; ++b)
          if (d->peerBase[di][b])
            cudaIpcCloseMemHandle(d->peerBase[di][b]);
        if (d->peerFlags[di])
          cudaIpcCloseMemHandle(d->peerFlags[di]);
        if (d->peerSlabBase[di])
          cudaIpcCloseMemHandle(d->peerSlabBase[di]);
      }
  cudaFree(d->flags);
  cudaFree(d->counter);
  cudaFree(d->cnt6);
  if (d->slab)
    planFree(*d->plan, d->slab);
  if (d->errHost)
    cudaFreeHost(d->errHost);
  if (d->putDone)
    cudaEventDestroy(d->putDone);
  delete d;
}

} // namespace
} // namespace hg

using namespace hg;

extern "C" {

int hg_nccl_unique_id(void *id) {
  if (!id)
    return setError(HG_EINVAL, "null id buffer");
  NcclApi &api = nccl();
  if (!api.lib)
    return setError(HG_EUNSUPPORTED, "NCCL transport unavailable: " + api.why);
  ncclUniqueId u;
  if (int rc = ncclCheck(api.getUniqueId(&u), "ncclGetUniqueId"))
    return rc;
  static_assert(sizeof(ncclUniqueId) == HG_NCCL_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id, &u, sizeof u);
  return HG_OK;
}

int hg_dmp_create_ex(hg_plan *plan, const hg_decomp *dc, int64_t rank, const hg_dmp_opts *opts,
                     hg_dmp **out) {
  try {
    if (!plan || !dc || !out)
      return setError(HG_EINVAL, "null argument");
    *out = nullptr;
    hg_dmp_opts o{};
    if (opts)
      o = *opts;
    if (o.transport != HG_TRANSPORT_P2P && o.transport != HG_TRANSPORT_NCCL)
      return setError(HG_EINVAL, "unknown transport");
    if (dc->ndim != plan->prog.rank)
      return setError(HG_EINVAL, "process grid rank does not match the domain");
    int64_t P = 1;
    for (int d = 0; d < dc->ndim; ++d) {
      if (dc->grid[d] < 1)
        return setError(HG_EINVAL, "grid dimensions must be at least 1");
      P *= dc->grid[d];
    }
    if (rank < 0 || rank >= P)
      return setError(HG_EINVAL, "rank outside the process grid");
    int64_t slabElems = 0;
    for (int s = 0; s < dc->nswaps; ++s) {
      if (dc->swaps[s].field < 0 || dc->swaps[s].field >= plan->prog.nfields)
        return setError(HG_EINVAL, "swap of a missing field");
      const hg::Layout &L = plan->lay[static_cast<size_t>(dc->swaps[s].field)];
      for (int k = 0; k < dc->swaps[s].nexchanges; ++k) {
        const hg_exchange &e = dc->swaps[s].ex[k];
        int64_t n = 1;
        for (int d = 0; d < dc->ndim; ++d) {
          if (e.size[d] < 1 || e.at[d] < 0 || e.at[d] + e.size[d] > L.shape[d] ||
              e.at[d] + e.offset[d] < 0 || e.at[d] + e.offset[d] + e.size[d] > L.shape[d])
            return setError(HG_EINVAL, "exchange region exceeds the buffer");
          n *= e.size[d];
        }
        if (e.to[dc->ndim - 1] != 0)
          slabElems = std::max(slabElems, n);
      }
    }
    // the put kernels index each job with its own field's layout; the fused swap of the star
    // family assumes one layout for all fields (starPlan: same bounds), checked here
    hg_dmp *d = new hg_dmp();
    std::unique_ptr<hg_dmp, void (*)(hg_dmp *)> guard(d, freeDmp);
    d->plan = plan;
    d->dc = *dc;
    d->rank = rank;
    d->transport = o.transport;
    d->prof = std::getenv("HG_DMP_PROFILE") != nullptr; // diagnostics: per-rank phase times
    const double tmo = o.timeout_s == 0 ? kDefaultTimeoutS : o.timeout_s;
    d->timeoutNs = tmo < 0 ? 0ull : static_cast<unsigned long long>(tmo * 1e9);
    hg_coord_from_rank(dc->ndim, rank, dc->grid, d->coord);
    for (int dim = 0; dim < kDirs / 2; ++dim)
      for (int sign : {-1, 1})
        d->nbr[dirIndex(dim, sign)] = dim < dc->ndim ? nbrOf(*d, dim, sign) : -1;
    d->dirty.assign(plan->dptr.size(), 1);
    d->xpack = o.transport == HG_TRANSPORT_P2P && starPlan(*plan) && plan->prog.rank >= 2 &&
               slabElems > 0;
    d->depth = o.depth < 1 ? 1 : o.depth;
    if (d->depth > 1) {
      // deep halos: every exchange of a split dim is depth * unit wide, unit >= the stencil
      // radius (hg_decompose_program_deep builds such programs)
      if (!starPlan(*plan))
        return setError(HG_EUNSUPPORTED, "deep halos need a star-family program");
      // a second-order-in-time step reads prev at the extended points too: prev at a round's
      // first step is the output of the previous round's second-to-last step, extended by one
      // width only -- enough for depth 2 alone
      if (plan->an.star.kind == kWave && d->depth > 2)
        return setError(HG_EUNSUPPORTED, "deep halos of a prev/cur/next step support depth 2");
      // the extended region of a round's first steps reaches the corners between two split
      // dims (e.g. the z band over the y halo), which face exchanges do not carry
      int split = 0;
      for (int q = 0; q < dc->ndim; ++q)
        split += dc->grid[q] > 1 ? 1 : 0;
      d->sequenced = split > 1; // dim-ordered round exchange (P2P: seqRoundStart; NCCL: stages)
      for (int s = 0; s < dc->nswaps; ++s)
        for (int k = 0; k < dc->swaps[s].nexchanges; ++k) {
          const hg_exchange &e = dc->swaps[s].ex[k];
          for (int q = 0; q < dc->ndim; ++q) {
            if (e.to[q] == 0 || dc->grid[q] < 2)
              continue;
            const int64_t w = e.size[q];
            if (w % d->depth != 0 || w / d->depth < plan->an.star.radius ||
                (d->unit[q] && d->unit[q] != w / d->depth))
              return setError(HG_EINVAL, "deep halos: exchange width " + std::to_string(w) +
                                             " in dimension " + std::to_string(q) +
                                             " is not depth x a width >= the stencil radius");
            d->unit[q] = w / d->depth;
          }
        }
    }
    d->slabElems = d->xpack ? slabElems : 0;
    if (int st = cudaCheck(cudaSetDevice(plan->device), "cudaSetDevice"))
      return st;
    if (int st = cudaCheck(cudaMalloc(&d->flags, kFlagBytes), "cudaMalloc(flags)"))
      return st;
    if (int st = cudaCheck(cudaMalloc(&d->counter, 64), "cudaMalloc(counter)"))
      return st;
    if (int st = cudaCheck(cudaMalloc(&d->cnt6, 64), "cudaMalloc(cnt6)"))
      return st;
    if (d->xpack) {
      const size_t bytes = slabOffset(*d, static_cast<int>(plan->dptr.size()), 0);
      void *sl = nullptr; // guarded like the plan's buffers under HG_DEBUG_GUARDS
      if (int st = planAlloc(*plan, &sl, bytes, "cudaMalloc(x slabs)"))
        return st;
      d->slab = static_cast<char *>(sl);
    }
    if (int st = cudaCheck(cudaMallocHost(&d->errHost, sizeof(unsigned long long)),
                           "cudaMallocHost(err)"))
      return st;
    *d->errHost = 0;
    if (int st = cudaCheck(cudaMemset(d->flags, 0, kFlagBytes), "cudaMemset(flags)"))
      return st;
    cudaMemset(d->counter, 0, 64);
    cudaMemset(d->cnt6, 0, 64);
    if (int st = cudaCheck(cudaEventCreateWithFlags(&d->putDone, cudaEventDisableTiming),
                           "event"))
      return st;
    if (o.transport == HG_TRANSPORT_NCCL) {
      NcclApi &api = nccl();
      if (!api.lib)
        return setError(HG_EUNSUPPORTED, "NCCL transport unavailable: " + api.why);
      if (o.nranks != P)
        return setError(HG_EINVAL, "nranks must equal the process grid size");
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      if (int st = cudaCheck(cudaStreamCreateWithPriority(&d->nc.cs, cudaStreamNonBlocking, hi),
                             "cudaStreamCreate(comm)"))
        return st;
      cudaEventCreateWithFlags(&d->nc.packed, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&d->nc.halo, cudaEventDisableTiming);
      ncclUniqueId id;
      std::memcpy(&id, o.nccl_id, sizeof id);
      if (int st = ncclCheck(api.commInitRank(&d->nc.comm, static_cast<int>(P), id,
                                              static_cast<int>(rank)),
                             "ncclCommInitRank"))
        return st;
      d->mode = 3;
    }
    cudaDeviceSynchronize();
    d->layoutHash = hashLayouts(*plan);
    *out = guard.release();
    return HG_OK;
  } catch (const std::exception &e) {
    return setError(HG_EINVAL, e.what());
  }
}

int hg_dmp_create(hg_plan *plan, const hg_decomp *dc, int64_t rank, hg_dmp **out) {
  return hg_dmp_create_ex(plan, dc, rank, nullptr, out);
}

int hg_dmp_destroy(hg_dmp *d) {
  if (!d)
    return HG_OK;
  cudaSetDevice(d->plan->device);
  cudaDeviceSynchronize();
  freeDmp(d);
  return HG_OK;
}

int hg_dmp_set_timeout(hg_dmp *d, double seconds) {
  if (!d)
    return setError(HG_EINVAL, "null dmp");
  d->timeoutNs = seconds <= 0 ? 0ull : static_cast<unsigned long long>(seconds * 1e9);
  return HG_OK;
}

int hg_dmp_ipc_export(hg_dmp *d, void *blob, size_t cap, size_t *len) {
  if (!d || !len)
    return setError(HG_EINVAL, "null argument");
  *len = sizeof(Blob);
  if (!blob)
    return HG_OK;
  if (cap < sizeof(Blob))
    return setError(HG_EINVAL, "blob buffer too small");
  Blob b;
  std::memset(&b, 0, sizeof b);
  b.magic = kMagic;
  b.nbuf = static_cast<uint32_t>(d->plan->dptr.size());
  b.rank = d->rank;
  b.layoutHash = d->layoutHash;
  b.slabElems = d->slabElems;
  if (int st = cudaCheck(cudaSetDevice(d->plan->device), "cudaSetDevice"))
    return st;
  if (int st = cudaCheck(cudaIpcGetMemHandle(&b.flags, d->flags), "cudaIpcGetMemHandle(flags)"))
    return st;
  if (d->slab) {
    b.slabOffset = d->slab - static_cast<char *>(planAllocBase(*d->plan, d->slab));
    if (int st = cudaCheck(cudaIpcGetMemHandle(&b.slab, planAllocBase(*d->plan, d->slab)),
                           "cudaIpcGetMemHandle(slab)"))
      return st;
  }
  for (uint32_t i = 0; i < b.nbuf; ++i) {
    void *base = planAllocBase(*d->plan, d->plan->dptr[i]);
    b.bufOffset[i] = static_cast<char *>(d->plan->dptr[i]) - static_cast<char *>(base);
    if (int st = cudaCheck(cudaIpcGetMemHandle(&b.buf[i], base), "cudaIpcGetMemHandle"))
      return st;
  }
  std::memcpy(blob, &b, sizeof b);
  return HG_OK;
}

int hg_dmp_ipc_import(hg_dmp *d, int64_t peer, const void *blob, size_t len) {
  if (!d || !blob || len < sizeof(Blob))
    return setError(HG_EINVAL, "bad blob");
  if (d->transport != HG_TRANSPORT_P2P)
    return setError(HG_ESTATE, "IPC import on a dmp of the NCCL transport");
  Blob b;
  std::memcpy(&b, blob, sizeof b);
  if (b.magic != kMagic || b.rank != peer)
    return setError(HG_EINVAL, "blob does not belong to that rank");
  if (b.layoutHash != d->layoutHash || b.nbuf != d->plan->dptr.size() ||
      b.slabElems != d->slabElems)
    return setError(HG_EINVAL, "peer field layouts differ from ours");
  if (int st = cudaCheck(cudaSetDevice(d->plan->device), "cudaSetDevice"))
    return st;
  for (int di = 0; di < kDirs; ++di) {
    if (d->nbr[di] != peer || d->opened[di])
      continue;
    void *f = nullptr;
    if (int st = cudaCheck(cudaIpcOpenMemHandle(&f, b.flags, cudaIpcMemLazyEnablePeerAccess),
                           "cudaIpcOpenMemHandle(flags)"))
      return st;
    d->peerFlags[di] = static_cast<unsigned long long *>(f);
    if (d->slabElems) {
      void *s = nullptr;
      if (int st = cudaCheck(cudaIpcOpenMemHandle(&s, b.slab, cudaIpcMemLazyEnablePeerAccess),
                             "cudaIpcOpenMemHandle(slab)"))
        return st;
      d->peerSlabBase[di] = s;
      d->peerSlab[di] = static_cast<char *>(s) + b.slabOffset;
    }
    for (uint32_t i = 0; i < b.nbuf; ++i) {
      void *p = nullptr;
      if (int st = cudaCheck(cudaIpcOpenMemHandle(&p, b.buf[i], cudaIpcMemLazyEnablePeerAccess),
                             "cudaIpcOpenMemHandle(buffer)"))
        return st;
      d->peerBase[di][i] = p;
      d->peer[di][i] = static_cast<char *>(p) + b.bufOffset[i];
    }
    d->opened[di] = true;
  }
  d->mode = 1;
  return HG_OK;
}

int hg_dmp_run(hg_dmp *d, int64_t steps, void *stream) {
  if (!d)
    return setError(HG_EINVAL, "null dmp");
  if (d->mode == 2)
    return setError(HG_ESTATE, "in-process ranks run through hg_sim_run");
  if (d->transport == HG_TRANSPORT_P2P)
    for (int di = 0; di < kDirs; ++di)
      if (d->nbr[di] >= 0 && !d->opened[di])
        return setError(HG_ESTATE, "neighbour rank " + std::to_string(d->nbr[di]) +
                                       " has not been imported");
  if (int rc = checkSticky(*d))
    return rc;
  hg_plan &p = *d->plan;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = cudaCheck(cudaSetDevice(p.device), "cudaSetDevice"))
    return rc;
  std::vector<cudaEvent_t> evs;
  d->roundReady = false;
  for (int64_t t = 0; t < steps; ++t) {
    int rc = d->transport == HG_TRANSPORT_NCCL ? ncclStep(*d, t, steps, st)
                                               : dmpStep(*d, t, steps, st, d->prof ? &evs : nullptr);
    if (rc)
      return rc;
  }
  // refresh the host mirror of the wait-timeout word (read at the next call's entry)
  cudaMemcpyAsync(d->errHost, d->flags + kErr, sizeof(unsigned long long),
                  cudaMemcpyDeviceToHost, st);
  if (d->prof && !evs.empty()) {
    cudaStreamSynchronize(st);
    double put = 0, ker = 0, gap = 0;
    float ms;
    const size_t n = evs.size() / 3;
    for (size_t i = 0; i < n; ++i) {
      cudaEventElapsedTime(&ms, evs[3 * i], evs[3 * i + 1]);
      put += ms;
      cudaEventElapsedTime(&ms, evs[3 * i + 1], evs[3 * i + 2]);
      ker += ms;
      if (i + 1 < n) {
        cudaEventElapsedTime(&ms, evs[3 * i + 2], evs[3 * i + 3]);
        gap += ms;
      }
    }
    std::fprintf(stderr, "[hg_dmp rank %lld] steps %zu: put %.1f us, stencil %.1f us, gap %.1f us (avg)\n",
                 static_cast<long long>(d->rank), n, 1e3 * put / n, 1e3 * ker / n,
                 n > 1 ? 1e3 * gap / (n - 1) : 0.0);
    for (auto e : evs)
      cudaEventDestroy(e);
  }
  return HG_OK;
}

int hg_dmp_status(hg_dmp *d) {
  if (!d)
    return setError(HG_EINVAL, "null dmp");
  if (int rc = cudaCheck(cudaSetDevice(d->plan->device), "cudaSetDevice"))
    return rc;
  if (int rc = cudaCheck(cudaDeviceSynchronize(), "cudaDeviceSynchronize"))
    return rc;
  unsigned long long c = 0;
  if (int rc = readErr(*d, &c))
    return rc;
  *d->errHost = c;
  return c ? trapFrom(*d, c) : HG_OK;
}

int hg_sim_connect(hg_dmp **ranks, int n) {
  if (!ranks || n < 1)
    return setError(HG_EINVAL, "no ranks");
  for (int i = 0; i < n; ++i) {
    hg_dmp *d = ranks[i];
    if (!d || d->rank != i)
      return setError(HG_EINVAL, "ranks must be given in rank order");
    if (d->transport != HG_TRANSPORT_P2P)
      return setError(HG_ESTATE, "in-process ranks use the P2P transport");
    for (int di = 0; di < kDirs; ++di) {
      if (d->nbr[di] < 0)
        continue;
      if (d->nbr[di] >= n)
        return setError(HG_EINVAL, "neighbour rank outside the given ranks");
      hg_dmp *o = ranks[d->nbr[di]];
      if (o->layoutHash != d->layoutHash || o->slabElems != d->slabElems)
        return setError(HG_EINVAL, "peer field layouts differ");
      if (o->plan->device != d->plan->device) {
        cudaSetDevice(d->plan->device);
        cudaError_t e = cudaDeviceEnablePeerAccess(o->plan->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return cudaCheck(e, "cudaDeviceEnablePeerAccess");
        cudaGetLastError();
      }
      for (size_t b = 0; b < o->plan->dptr.size(); ++b)
        d->peer[di][b] = o->plan->dptr[b];
      d->peerFlags[di] = o->flags;
      d->peerSlab[di] = o->slab;
      d->opened[di] = true;
    }
    d->mode = 2;
  }
  return HG_OK;
}

int hg_sim_run(hg_dmp **ranks, int n, int64_t steps, void **streams) {
  if (!ranks || n < 1)
    return setError(HG_EINVAL, "no ranks");
  bool distinct = true;
  for (int i = 0; i < n; ++i) {
    if (!ranks[i] || ranks[i]->mode != 2)
      return setError(HG_ESTATE, "ranks are not connected (hg_sim_connect)");
    for (int j = 0; j < i; ++j)
      if (ranks[j]->plan->device == ranks[i]->plan->device)
        distinct = false;
  }
  auto stream = [&](int i) {
    return streams ? static_cast<cudaStream_t>(streams[i]) : cudaStream_t(nullptr);
  };
  if (distinct && n > 1) {
    // one rank per device: the multi-process protocol (fused NVLink swap, in-kernel waits on
    // the neighbours' flags) with the ranks' steps issued round-robin from this thread
    for (int i = 0; i < n; ++i)
      ranks[i]->roundReady = false;
    for (int64_t t = 0; t < steps; ++t)
      for (int i = 0; i < n; ++i) {
        hg_dmp &d = *ranks[i];
        if (int rc = cudaCheck(cudaSetDevice(d.plan->device), "cudaSetDevice"))
          return rc;
        if (int rc = dmpStep(d, t, steps, stream(i), nullptr))
          return rc;
      }
    for (int i = 0; i < n; ++i)
      if (int rc = hg_dmp_status(ranks[i]))
        return rc;
    return HG_OK;
  }
  // ranks sharing a device: spin-waits could starve the producer, so phases are ordered by
  // CUDA events (swap phase of every rank, then compute phase), direct puts into the halos
  std::vector<PutJob> jobs;
  for (int64_t t = 0; t < steps; ++t) {
    for (int i = 0; i < n; ++i) {
      hg_dmp &d = *ranks[i];
      hg_plan &p = *d.plan;
      cudaStream_t st = stream(i);
      if (int rc = cudaCheck(cudaSetDevice(p.device), "cudaSetDevice"))
        return rc;
      jobs.clear();
      if (int rc = buildPutJobs(d, jobs, false))
        return rc;
      if (!jobs.empty()) {
        if (int rc = launchPut(jobs.data(), static_cast<int>(jobs.size()), nullptr, 0, 0,
                               d.counter, st))
          return rc;
        ++p.launches;
      }
      if (int rc = cudaCheck(cudaEventRecord(d.putDone, st), "cudaEventRecord"))
        return rc;
    }
    for (int i = 0; i < n; ++i) {
      hg_dmp &d = *ranks[i];
      hg_plan &p = *d.plan;
      cudaStream_t st = stream(i);
      if (int rc = cudaCheck(cudaSetDevice(p.device), "cudaSetDevice"))
        return rc;
      for (int di = 0; di < kDirs; ++di)
        if (d.nbr[di] >= 0)
          if (int rc = cudaCheck(cudaStreamWaitEvent(st, ranks[d.nbr[di]]->putDone, 0),
                                 "cudaStreamWaitEvent"))
            return rc;
      const hg_program &g = p.prog;
      std::vector<int> written;
      for (int k = 0; k < storedCount(g); ++k)
        written.push_back(p.bind[static_cast<size_t>(storedField(g, k))]);
      if (int rc = planStep(p, st))
        return rc;
      for (int b : written)
        d.dirty[static_cast<size_t>(b)] = 1;
    }
  }
  return HG_OK;
}

int64_t hg_dmp_bytes_exchanged(const hg_dmp *d) { return d ? d->bytes : 0; }

int hg_dmp_invalidate(hg_dmp *d) {
  if (!d)
    return setError(HG_EINVAL, "null dmp");
  std::fill(d->dirty.begin(), d->dirty.end(), 1);
  // the next run starts with the receiver-ready handshake (P2P multi-process): every rank
  // calls this after its uploads, so nobody puts into buffers still being uploaded
  if (d->mode == 1)
    d->needReady = true;
  return HG_OK;
}

} // extern "C"
