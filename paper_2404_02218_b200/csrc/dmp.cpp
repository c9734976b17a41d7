// dmp.cpp -- the dmp halo swap on device buffers (RankHooks::swap, simulator.cpp:772-834).
//
// A swap is a set of independent box copies: each exchange's send box (at + offset, inside my
// core) goes to the neighbour's receive box (the mate exchange's `at`, in its halo).  On the
// GPU a put kernel reads my box and stores it straight into the neighbour's buffer over NVLink
// (peer memory mapped by CUDA IPC between processes, or plain peer pointers inside one
// process) -- pack, send, receive and unpack in one pass, byte-exact.  Ordering replaces the
// reference's buffered send / blocking receive: the last CTA of a put publishes an epoch to
// the neighbour's flag word (system-scope release); a rank computes only after every
// neighbour's flag reached the step's epoch.  Swaps of a buffer nobody has written since its
// previous swap are elided (the runtime form of eliminate-redundant-swaps,
// dmp_transforms.cpp:318-359): they would store the very same bytes.
#include "plan.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>

namespace {
constexpr uint32_t kMagic = 0x48474450; // "HGDP"
constexpr int kDirs = 2 * HG_MAX_RANK;

struct Blob {
  uint32_t magic;
  uint32_t nbuf;
  int64_t rank;
  uint64_t layoutHash;
  cudaIpcMemHandle_t flags;
  cudaIpcMemHandle_t buf[HG_MAX_FIELDS];
};

int dirIndex(int dim, int sign) { return 2 * dim + (sign > 0 ? 1 : 0); }
} // namespace

struct hg_dmp {
  hg_plan *plan = nullptr;
  hg_decomp dc{};
  int64_t rank = 0;
  int64_t coord[HG_MAX_RANK] = {0, 0, 0};
  int64_t nbr[kDirs];
  void *peer[kDirs][HG_MAX_FIELDS] = {};
  unsigned long long *peerFlags[kDirs] = {};
  bool opened[kDirs] = {};
  unsigned long long *flags = nullptr; // my flag words, one per incoming direction
  unsigned int *counter = nullptr;
  unsigned int *cnt6 = nullptr;        // per-face CTA completion counters of fused swaps
  unsigned int cntAccum[kDirs] = {};   // their cumulative targets (host mirror)
  unsigned long long epoch = 0;
  std::vector<char> dirty;             // per buffer: written since its last swap
  int64_t bytes = 0;
  int mode = 0;                        // 0 unconnected, 1 ipc, 2 in-process
  cudaEvent_t putDone = nullptr;
  uint64_t layoutHash = 0;
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

// Build the put jobs of this step's swaps (and mark the swapped buffers clean).
int buildJobs(hg_dmp &d, std::vector<PutJob> &jobs) {
  hg_plan &p = *d.plan;
  const int r = p.prog.rank;
  for (int si = 0; si < d.dc.nswaps; ++si) {
    const hg_swap &s = d.dc.swaps[si];
    const int b = p.bind[static_cast<size_t>(s.field)];
    if (!d.dirty[static_cast<size_t>(b)])
      continue;
    for (int k = 0; k < s.nexchanges; ++k) {
      const hg_exchange &e = s.ex[k];
      int dim = -1, sign = 0;
      for (int q = 0; q < r; ++q)
        if (e.to[q] != 0) {
          dim = q;
          sign = e.to[q] > 0 ? 1 : -1;
        }
      if (dim < 0)
        return setError(HG_ETRAP, "exchange direction is all zero");
      const int di = dirIndex(dim, sign);
      if (d.nbr[di] < 0)
        continue; // global boundary: no neighbour, nothing sent (simulator.cpp:810-812)
      const hg_exchange *m = mateOf(s, e, r);
      if (!m)
        return setError(HG_EINVAL, "swap template lacks the opposite exchange");
      if (!d.peer[di][b])
        return setError(HG_ESTATE, "neighbour buffers are not connected");
      PutJob j{};
      j.src = p.dptr[static_cast<size_t>(b)];
      j.dst = d.peer[di][b];
      int64_t n = 1;
      for (int q = 0; q < 3; ++q) {
        j.src_at[q] = q < r ? e.at[q] + e.offset[q] : 0;
        j.dst_at[q] = q < r ? m->at[q] : 0;
        j.size[q] = q < r ? e.size[q] : 1;
        n *= j.size[q];
      }
      d.bytes += n * p.lay[0].es;
      jobs.push_back(j);
    }
    d.dirty[static_cast<size_t>(b)] = 0;
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

} // namespace
} // namespace hg

using namespace hg;

extern "C" {

int hg_dmp_create(hg_plan *plan, const hg_decomp *dc, int64_t rank, hg_dmp **out) {
  try {
    if (!plan || !dc || !out)
      return setError(HG_EINVAL, "null argument");
    *out = nullptr;
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
    plan->tbOff = true; // peers address the buffers: no more buffer/shadow exchanges
    for (int s = 0; s < dc->nswaps; ++s) {
      if (dc->swaps[s].field < 0 || dc->swaps[s].field >= plan->prog.nfields)
        return setError(HG_EINVAL, "swap of a missing field");
      const hg::Layout &L = plan->lay[static_cast<size_t>(dc->swaps[s].field)];
      for (int k = 0; k < dc->swaps[s].nexchanges; ++k) {
        const hg_exchange &e = dc->swaps[s].ex[k];
        for (int d = 0; d < dc->ndim; ++d)
          if (e.size[d] < 1 || e.at[d] < 0 || e.at[d] + e.size[d] > L.shape[d] ||
              e.at[d] + e.offset[d] < 0 || e.at[d] + e.offset[d] + e.size[d] > L.shape[d])
            return setError(HG_EINVAL, "exchange region exceeds the buffer");
      }
    }
    auto d = std::make_unique<hg_dmp>();
    d->plan = plan;
    d->dc = *dc;
    d->rank = rank;
    hg_coord_from_rank(dc->ndim, rank, dc->grid, d->coord);
    for (int dim = 0; dim < kDirs / 2; ++dim)
      for (int sign : {-1, 1})
        d->nbr[dirIndex(dim, sign)] = dim < dc->ndim ? nbrOf(*d, dim, sign) : -1;
    d->dirty.assign(plan->dptr.size(), 1);
    int st = cudaCheck(cudaSetDevice(plan->device), "cudaSetDevice");
    if (st)
      return st;
    st = cudaCheck(cudaMalloc(&d->flags, 256), "cudaMalloc(flags)");
    if (st)
      return st;
    cudaMemset(d->flags, 0, 256);
    st = cudaCheck(cudaMalloc(&d->counter, 64), "cudaMalloc(counter)");
    if (st)
      return st;
    cudaMemset(d->counter, 0, 64);
    st = cudaCheck(cudaMalloc(&d->cnt6, 64), "cudaMalloc(cnt6)");
    if (st)
      return st;
    cudaMemset(d->cnt6, 0, 64);
    st = cudaCheck(cudaEventCreateWithFlags(&d->putDone, cudaEventDisableTiming), "event");
    if (st)
      return st;
    cudaDeviceSynchronize();
    d->layoutHash = hashLayouts(*plan);
    *out = d.release();
    return HG_OK;
  } catch (const std::exception &e) {
    return setError(HG_EINVAL, e.what());
  }
}

int hg_dmp_destroy(hg_dmp *d) {
  if (!d)
    return HG_OK;
  cudaSetDevice(d->plan->device);
  cudaDeviceSynchronize();
  if (d->mode == 1)
    for (int di = 0; di < kDirs; ++di)
      if (d->opened[di]) {
        for (int b = 0; b < HG_MAX_FIELDS; ++b)
          if (d->peer[di][b])
            cudaIpcCloseMemHandle(d->peer[di][b]);
        if (d->peerFlags[di])
          cudaIpcCloseMemHandle(d->peerFlags[di]);
      }
  cudaFree(d->flags);
  cudaFree(d->counter);
  cudaFree(d->cnt6);
  if (d->putDone)
    cudaEventDestroy(d->putDone);
  delete d;
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
  int st = cudaCheck(cudaSetDevice(d->plan->device), "cudaSetDevice");
  if (st)
    return st;
  st = cudaCheck(cudaIpcGetMemHandle(&b.flags, d->flags), "cudaIpcGetMemHandle(flags)");
  if (st)
    return st;
  for (uint32_t i = 0; i < b.nbuf; ++i) {
    st = cudaCheck(cudaIpcGetMemHandle(&b.buf[i], d->plan->dptr[i]), "cudaIpcGetMemHandle");
    if (st)
      return st;
  }
  std::memcpy(blob, &b, sizeof b);
  return HG_OK;
}

int hg_dmp_ipc_import(hg_dmp *d, int64_t peer, const void *blob, size_t len) {
  if (!d || !blob || len < sizeof(Blob))
    return setError(HG_EINVAL, "bad blob");
  Blob b;
  std::memcpy(&b, blob, sizeof b);
  if (b.magic != kMagic || b.rank != peer)
    return setError(HG_EINVAL, "blob does not belong to that rank");
  if (b.layoutHash != d->layoutHash || b.nbuf != d->plan->dptr.size())
    return setError(HG_EINVAL, "peer field layouts differ from ours");
  int st = cudaCheck(cudaSetDevice(d->plan->device), "cudaSetDevice");
  if (st)
    return st;
  for (int di = 0; di < kDirs; ++di) {
    if (d->nbr[di] != peer || d->opened[di])
      continue;
    void *f = nullptr;
    st = cudaCheck(cudaIpcOpenMemHandle(&f, b.flags, cudaIpcMemLazyEnablePeerAccess),
                   "cudaIpcOpenMemHandle(flags)");
    if (st)
      return st;
    d->peerFlags[di] = static_cast<unsigned long long *>(f);
    for (uint32_t i = 0; i < b.nbuf; ++i) {
      void *p = nullptr;
      st = cudaCheck(cudaIpcOpenMemHandle(&p, b.buf[i], cudaIpcMemLazyEnablePeerAccess),
                     "cudaIpcOpenMemHandle(buffer)");
      if (st)
        return st;
      d->peer[di][i] = p;
    }
    d->opened[di] = true;
  }
  d->mode = 1;
  return HG_OK;
}

int hg_dmp_run(hg_dmp *d, int64_t steps, void *stream) {
  if (!d)
    return setError(HG_EINVAL, "null dmp");
  for (int di = 0; di < kDirs; ++di)
    if (d->nbr[di] >= 0 && !d->opened[di])
      return setError(HG_ESTATE, "neighbour rank " + std::to_string(d->nbr[di]) +
                                     " has not been imported");
  hg_plan &p = *d->plan;
  const hg_program &g = p.prog;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = cudaCheck(cudaSetDevice(p.device), "cudaSetDevice");
  if (rc)
    return rc;
  PutSignal sig[kDirs];
  int nsig = 0, widx[kDirs], nw = 0, mask = 0;
  for (int di = 0; di < kDirs; ++di) {
    if (d->nbr[di] < 0)
      continue;
    sig[nsig++].flag = d->peerFlags[di] + (di ^ 1); // the neighbour receives on its opposite
    widx[nw++] = di;
    mask |= 1 << di;
  }
  const bool star = p.an.family == Family::Star && g.nresults == 1;
  std::vector<PutJob> jobs;
  // HG_DMP_PROFILE=1: event timing of the put and stencil phases (diagnostics only)
  static const bool prof = std::getenv("HG_DMP_PROFILE") != nullptr;
  std::vector<cudaEvent_t> evs;
  auto mark = [&]() {
    if (!prof)
      return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    evs.push_back(e);
  };
  bool roundReady = false; // the previous step's kernel already published this step's round
  for (int64_t t = 0; t < steps; ++t) {
    // 1. standalone put of every dirty swapped buffer (first step of a call, or whatever the
    //    fused path did not cover)
    jobs.clear();
    rc = buildJobs(*d, jobs);
    if (rc)
      return rc;
    mark();
    if (!roundReady || !jobs.empty()) {
      ++d->epoch;
      rc = launchPut(jobs.data(), static_cast<int>(jobs.size()), devLayout(p.lay[0]), sig, nsig,
                     d->epoch, d->counter, st);
      if (rc)
        return rc;
      if (nsig || !jobs.empty())
        ++p.launches;
    }
    // 2. the stencil step; halo-reading CTAs wait for the round in-kernel
    if (star && nw) {
      p.waitFlags = d->flags;
      p.waitEpoch = d->epoch;
      p.waitMask = mask;
      p.boundaryLast = (mask & 3) ? 1 : 0;
    } else {
      rc = launchWaitFlags(d->flags, widx, nw, d->epoch, st);
      if (rc)
        return rc;
      if (nw)
        ++p.launches;
    }
    // 3. fuse the NEXT step's swap of the output into this kernel (not on the last step of
    //    the call: the reference swaps a buffer only right before it is loaded)
    // the buffers this step writes (bindings before the step rotates them)
    std::vector<int> written;
    for (int k = 0; k < storedCount(g); ++k)
      written.push_back(p.bind[static_cast<size_t>(storedField(g, k))]);
    const int bOut = written[0];
    int nextSlot = -1; // the argument slot the output buffer occupies next step
    for (size_t i = 0; i < p.an.src.size(); ++i)
      if (p.an.src[i] == storedField(g, 0))
        nextSlot = static_cast<int>(i);
    const hg_swap *sw = nullptr;
    for (int k = 0; k < d->dc.nswaps && nextSlot >= 0; ++k)
      if (d->dc.swaps[k].field == nextSlot)
        sw = &d->dc.swaps[k];
    bool fused = false;
    static const bool noFuse = std::getenv("HG_NOFUSE") != nullptr; // A/B experiments only
    if (star && nw && sw && t + 1 < steps && !noFuse) {
      StarLaunch &F = p.fuse;
      F = StarLaunch{};
      const Layout &L = p.lay[static_cast<size_t>(bOut)];
      const int r = g.rank;
      int64_t stride[3] = {0, 0, 1};
      if (r == 3) {
        stride[0] = L.pitch * L.shape[1];
        stride[1] = L.pitch;
      } else {
        stride[0] = L.pitch;
      }
      // kernel face index: 2*kdim + (sign>0) with kdim 0 = z (dim 0), 1 = y, RANK-1 = x
      for (int k = 0; k < sw->nexchanges; ++k) {
        const hg_exchange &e = sw->ex[k];
        int dim = -1, sign = 0;
        for (int q = 0; q < r; ++q)
          if (e.to[q] != 0) {
            dim = q;
            sign = e.to[q] > 0 ? 1 : -1;
          }
        const int di = dirIndex(dim, sign);
        if (dim < 0 || d->nbr[di] < 0)
          continue;
        const hg_exchange *m = mateOf(*sw, e, r);
        if (!m || !d->peer[di][bOut])
          return setError(HG_ESTATE, "neighbour buffers are not connected");
        int64_t delta = 0;
        for (int q = 0; q < r; ++q)
          delta += (m->at[q] - (e.at[q] + e.offset[q])) * (r == 3 ? stride[q] : (q == 0 ? stride[0] : 1));
        F.hs[di] = static_cast<int>(e.size[dim]);
        F.peer[di] = d->peer[di][bOut];
        static const bool scratch = std::getenv("HG_FUSE_SCRATCH") != nullptr; // A/B only
        if (scratch) {
          static void *buf = nullptr;
          if (!buf)
            cudaMalloc(&buf, L.bytes());
          F.peer[di] = buf;
        }
        F.pdelta[di] = delta;
        F.peer_flag[di] = d->peerFlags[di];
        d->bytes += [&] {
          int64_t n = 1;
          for (int q = 0; q < r; ++q)
            n *= e.size[q];
          return n * L.es;
        }();
      }
      F.fuse = 1;
      F.cnt = d->cnt6;
      F.cnt_accum = d->cntAccum;
      F.put_epoch = d->epoch + 1;
      fused = true;
    }
    mark();
    rc = planStep(p, st);
    if (rc)
      return rc;
    mark();
    for (size_t k = 1; k < written.size(); ++k) // (multi-store programs never fuse)
      d->dirty[static_cast<size_t>(written[k])] = 1;
    d->dirty[static_cast<size_t>(bOut)] = fused ? 0 : 1;
    if (fused)
      ++d->epoch;
    roundReady = fused;
  }
  if (prof && !evs.empty()) {
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

int hg_sim_connect(hg_dmp **ranks, int n) {
  if (!ranks || n < 1)
    return setError(HG_EINVAL, "no ranks");
  for (int i = 0; i < n; ++i) {
    hg_dmp *d = ranks[i];
    if (!d || d->rank != i)
      return setError(HG_EINVAL, "ranks must be given in rank order");
    for (int di = 0; di < kDirs; ++di) {
      if (d->nbr[di] < 0)
        continue;
      if (d->nbr[di] >= n)
        return setError(HG_EINVAL, "neighbour rank outside the given ranks");
      hg_dmp *o = ranks[d->nbr[di]];
      if (o->layoutHash != d->layoutHash)
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
      d->peerFlags[di] = nullptr;
      d->opened[di] = true;
    }
    d->mode = 2;
  }
  return HG_OK;
}

int hg_sim_run(hg_dmp **ranks, int n, int64_t steps, void **streams) {
  if (!ranks || n < 1)
    return setError(HG_EINVAL, "no ranks");
  for (int i = 0; i < n; ++i)
    if (!ranks[i] || ranks[i]->mode != 2)
      return setError(HG_ESTATE, "ranks are not connected (hg_sim_connect)");
  std::vector<PutJob> jobs;
  for (int64_t t = 0; t < steps; ++t) {
    // swap phase: every rank puts its dirty faces into its neighbours
    for (int i = 0; i < n; ++i) {
      hg_dmp &d = *ranks[i];
      hg_plan &p = *d.plan;
      cudaStream_t st = streams ? static_cast<cudaStream_t>(streams[i]) : nullptr;
      int rc = cudaCheck(cudaSetDevice(p.device), "cudaSetDevice");
      if (rc)
        return rc;
      jobs.clear();
      rc = buildJobs(d, jobs);
      if (rc)
        return rc;
      if (!jobs.empty()) {
        rc = launchPut(jobs.data(), static_cast<int>(jobs.size()), devLayout(p.lay[0]), nullptr,
                       0, 0, d.counter, st);
        if (rc)
          return rc;
        ++p.launches;
      }
      rc = cudaCheck(cudaEventRecord(d.putDone, st), "cudaEventRecord");
      if (rc)
        return rc;
    }
    // compute phase: each rank waits for its neighbours' puts
    for (int i = 0; i < n; ++i) {
      hg_dmp &d = *ranks[i];
      hg_plan &p = *d.plan;
      cudaStream_t st = streams ? static_cast<cudaStream_t>(streams[i]) : nullptr;
      int rc = cudaCheck(cudaSetDevice(p.device), "cudaSetDevice");
      if (rc)
        return rc;
      for (int di = 0; di < kDirs; ++di)
        if (d.nbr[di] >= 0) {
          rc = cudaCheck(cudaStreamWaitEvent(st, ranks[d.nbr[di]]->putDone, 0),
                         "cudaStreamWaitEvent");
          if (rc)
            return rc;
        }
      const hg_program &g = p.prog;
      std::vector<int> written;
      for (int k = 0; k < storedCount(g); ++k)
        written.push_back(p.bind[static_cast<size_t>(storedField(g, k))]);
      rc = planStep(p, st);
      if (rc)
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
  return HG_OK;
}

} // extern "C"
