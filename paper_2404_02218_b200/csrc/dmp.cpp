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
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = cudaCheck(cudaSetDevice(p.device), "cudaSetDevice");
  if (rc)
    return rc;
  std::vector<PutJob> jobs;
  for (int64_t t = 0; t < steps; ++t) {
    jobs.clear();
    rc = buildJobs(*d, jobs);
    if (rc)
      return rc;
    ++d->epoch;
    PutSignal sig[kDirs];
    int nsig = 0, widx[kDirs], nw = 0;
    for (int di = 0; di < kDirs; ++di) {
      if (d->nbr[di] < 0)
        continue;
      // the neighbour at my direction di receives on its opposite direction
      const int opp = di ^ 1;
      sig[nsig++].flag = d->peerFlags[di] + opp;
      widx[nw++] = di;
    }
    rc = launchPut(jobs.data(), static_cast<int>(jobs.size()), devLayout(p.lay[0]), sig, nsig,
                   d->epoch, d->counter, st);
    if (rc)
      return rc;
    if (nsig || !jobs.empty())
      ++p.launches;
    if (p.an.family == Family::Star && nw) {
      // fused wait: only the CTAs whose halo rows touch a neighbour's face wait for its
      // flag, inside the stencil kernel; z-boundary chunks run last, so the exchange
      // overlaps the interior
      int mask = 0;
      for (int k = 0; k < nw; ++k)
        mask |= 1 << widx[k];
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
    rc = planStep(p, st);
    if (rc)
      return rc;
    // the step's outputs (bound before rotation) are now dirty
    const hg_program &g = p.prog;
    std::vector<int> prevBind(p.bind.size());
    for (size_t i = 0; i < p.bind.size(); ++i)
      prevBind[static_cast<size_t>(p.an.src[i])] = p.bind[i];
    for (int k = 0; k < g.nresults; ++k)
      d->dirty[static_cast<size_t>(prevBind[static_cast<size_t>(g.store_field[k])])] = 1;
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
      rc = planStep(p, st);
      if (rc)
        return rc;
      const hg_program &g = p.prog;
      std::vector<int> prevBind(p.bind.size());
      for (size_t k = 0; k < p.bind.size(); ++k)
        prevBind[static_cast<size_t>(p.an.src[k])] = p.bind[k];
      for (int k = 0; k < g.nresults; ++k)
        d.dirty[static_cast<size_t>(prevBind[static_cast<size_t>(g.store_field[k])])] = 1;
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
