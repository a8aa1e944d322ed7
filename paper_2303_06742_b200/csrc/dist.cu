// Multi-GPU plumbing of the x-slab domain decomposition.
//   * halo pack / unpack kernels: copy the x-node slabs of every (Radau node, field, component) array of a level
//     vector into a contiguous message buffer and back;
//   * owned-DoF mask for the Krylov inner products;
//   * transports: NCCL (ncclSend/ncclRecv to the x-neighbours, ncclAllReduce for dot products, ncclAllGather for
//     the agglomerated coarse levels), loaded with dlopen so that single-GPU use needs no NCCL; and an in-process
//     loopback transport (N emulated ranks on one GPU, one host thread each; the host synchronises at every
//     exchange, no kernel ever waits on another rank) used by the multi-rank parity tests; and a PROCESS-separated
//     shared-memory transport (one process per rank, host-staged messages in a POSIX shared-memory segment, a
//     sense-reversing barrier on process-shared atomics) that runs the per-rank bootstrap and handles exactly as
//     under torchrun, on one GPU or several, without NCCL.
#include <dlfcn.h>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "dist.cuh"

namespace stgmg {

// ------------------------------------------------------------------------------------------- pack / unpack --
// Message layout: for m, for slot (Q_r components), [z][y][x in xq range]; then for m, [z][y][x in xp range].
__global__ void halo_pack_kernel(LevelGeom g, int k1, int xq0, int nxq, int xp0, int nxp, const double* __restrict__ v,
                                 double* __restrict__ buf, int unpack) {
  const int d = g.d;
  const long long planeQ = (long long)nxq * g.qn[1] * g.qn[2];
  const long long planeP = (long long)nxp * g.pn[1] * g.pn[2];
  const long long totQ = (long long)k1 * 2 * d * planeQ;
  const long long tot = totQ + (long long)k1 * planeP;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += stride) {
    long long gi;
    if (i < totQ) {
      const long long comp = i / planeQ, rem = i % planeQ;   // comp = m * 2d + slot
      const int m = (int)(comp / (2 * d)), slot = (int)(comp % (2 * d));
      const int x = (int)(rem % nxq);
      const long long yz = rem / nxq;
      const int y = (int)(yz % g.qn[1]), z = (int)(yz / g.qn[1]);
      gi = (long long)m * g.block + (long long)slot * g.nq + (xq0 + x) + (long long)y * g.qs[1] +
           (d > 2 ? (long long)z * g.qs[2] : 0);
    } else {
      const long long j = i - totQ;
      const int m = (int)(j / planeP);
      const long long rem = j % planeP;
      const int x = (int)(rem % nxp);
      const long long yz = rem / nxp;
      const int y = (int)(yz % g.pn[1]), z = (int)(yz / g.pn[1]);
      gi = (long long)m * g.block + 2 * g.R + (xp0 + x) + (long long)y * g.ps[1] + (d > 2 ? (long long)z * g.ps[2] : 0);
    }
    if (unpack)
      const_cast<double*>(v)[gi] = buf[i];
    else
      buf[i] = v[gi];
  }
}

long long halo_count(const LevelGeom& g, int k1, int nxq, int nxp) {
  return (long long)k1 * (2 * g.d * (long long)nxq * g.qn[1] * g.qn[2] + (long long)nxp * g.pn[1] * g.pn[2]);
}

cudaError_t launch_halo(const LevelGeom& g, int k1, int xq0, int nxq, int xp0, int nxp, const double* v, double* buf,
                        int unpack, cudaStream_t s) {
  const long long n = halo_count(g, k1, nxq, nxp);
  if (n == 0) return cudaSuccess;
  const int bs = 256;
  const long long nb = std::min<long long>((n + bs - 1) / bs, 4096);
  halo_pack_kernel<<<(unsigned)nb, bs, 0, s>>>(g, k1, xq0, nxq, xp0, nxp, v, buf, unpack);
  return cudaGetLastError();
}

// owned mask: 1 for DoFs whose x-node lies in [q0, q1) (Q_r) or [p0, p1) (Q_{r-1})
__global__ void owned_mask_kernel(LevelGeom g, int q0, int q1, int p0, int p1, unsigned char* mask) {
  const long long mu = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (mu >= g.N) return;
  const long long rem = mu % g.block;
  int x;
  bool own;
  if (rem < 2 * g.R) {
    x = (int)((rem % g.nq) % g.qn[0]);
    own = x >= q0 && x < q1;
  } else {
    x = (int)((rem - 2 * g.R) % g.pn[0]);
    own = x >= p0 && x < p1;
  }
  mask[mu] = own ? 1 : 0;
}

cudaError_t launch_owned_mask(const LevelGeom& g, int q0, int q1, int p0, int p1, unsigned char* mask, cudaStream_t s) {
  owned_mask_kernel<<<(unsigned)((g.N + 255) / 256), 256, 0, s>>>(g, q0, q1, p0, p1, mask);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------ NCCL -------
// Minimal NCCL ABI (nccl.h 2.x): opaque communicator, enum values of ncclDouble / ncclSum.
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
enum { kNcclDouble = 8, kNcclSum = 0 };

struct NcclApi {
  void* lib = nullptr;
  int (*GetUniqueId)(ncclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

static NcclApi* nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      api.lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.lib) break;
    }
    if (api.lib) {
      api.GetUniqueId = (int (*)(ncclUniqueId*))dlsym(api.lib, "ncclGetUniqueId");
      api.CommInitRank = (int (*)(ncclComm_t*, int, ncclUniqueId, int))dlsym(api.lib, "ncclCommInitRank");
      api.CommDestroy = (int (*)(ncclComm_t))dlsym(api.lib, "ncclCommDestroy");
      api.Send = (int (*)(const void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(api.lib, "ncclSend");
      api.Recv = (int (*)(void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(api.lib, "ncclRecv");
      api.AllReduce =
          (int (*)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(api.lib, "ncclAllReduce");
      api.AllGather = (int (*)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t))dlsym(api.lib, "ncclAllGather");
      api.GroupStart = (int (*)())dlsym(api.lib, "ncclGroupStart");
      api.GroupEnd = (int (*)())dlsym(api.lib, "ncclGroupEnd");
      api.GetErrorString = (const char* (*)(int))dlsym(api.lib, "ncclGetErrorString");
    }
  }
  return (api.lib && api.Send && api.AllReduce) ? &api : nullptr;
}

int nccl_unique_id(unsigned char out[128]) {
  NcclApi* a = nccl();
  if (!a) { set_error("NCCL library not found (libnccl.so.2)"); return -4; }
  ncclUniqueId id;
  const int rc = a->GetUniqueId(&id);
  if (rc) { set_error(std::string("ncclGetUniqueId: ") + a->GetErrorString(rc)); return -4; }
  std::memcpy(out, id.internal, 128);
  return 0;
}

int nccl_comm_create(const unsigned char id[128], int nranks, int rank, void** comm) {
  NcclApi* a = nccl();
  if (!a) { set_error("NCCL library not found (libnccl.so.2)"); return -4; }
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  ncclComm_t c = nullptr;
  const int rc = a->CommInitRank(&c, nranks, u, rank);
  if (rc) { set_error(std::string("ncclCommInitRank: ") + a->GetErrorString(rc)); return -4; }
  *comm = (void*)c;
  return 0;
}

int nccl_comm_destroy(void* comm) {
  NcclApi* a = nccl();
  if (!a) return -4;
  return a->CommDestroy((ncclComm_t)comm) ? -4 : 0;
}

struct NcclTransport : Transport {
  ncclComm_t comm;
  explicit NcclTransport(void* c, int r, int n) : comm((ncclComm_t)c) { rank = r; nranks = n; }
  bool graph_capturable() const override { return true; }
  int check(int rc, const char* what) {
    if (rc) {
      set_error(std::string(what) + ": " + nccl()->GetErrorString(rc));
      return -4;
    }
    return 0;
  }
  int halo(const double* sl, long long nsl, const double* sr, long long nsr, double* rl, long long nrl, double* rr,
           long long nrr, cudaStream_t s) override {
    NcclApi* a = nccl();
    if (check(a->GroupStart(), "ncclGroupStart")) return -4;
    if (rank > 0) {
      if (check(a->Send(sl, (size_t)nsl, kNcclDouble, rank - 1, comm, s), "ncclSend")) return -4;
      if (check(a->Recv(rl, (size_t)nrl, kNcclDouble, rank - 1, comm, s), "ncclRecv")) return -4;
    }
    if (rank < nranks - 1) {
      if (check(a->Send(sr, (size_t)nsr, kNcclDouble, rank + 1, comm, s), "ncclSend")) return -4;
      if (check(a->Recv(rr, (size_t)nrr, kNcclDouble, rank + 1, comm, s), "ncclRecv")) return -4;
    }
    return check(a->GroupEnd(), "ncclGroupEnd");
  }
  int allreduce_sum(double* v, int n, cudaStream_t s) override {
    return check(nccl()->AllReduce(v, v, (size_t)n, kNcclDouble, kNcclSum, comm, s), "ncclAllReduce");
  }
  int allgather(const double* send, long long n, double* recv, cudaStream_t s) override {
    return check(nccl()->AllGather(send, recv, (size_t)n, kNcclDouble, comm, s), "ncclAllGather");
  }
};

Transport* make_nccl_transport(void* comm, int rank, int nranks) {
  if (!nccl()) { set_error("NCCL library not found (libnccl.so.2)"); return nullptr; }
  return new NcclTransport(comm, rank, nranks);
}

// ------------------------------------------------------------------------------------- loopback (tests) ------
struct LoopbackHub {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<const double*> sl, sr, ag;
  std::vector<double> red;
  explicit LoopbackHub(int n_) : n(n_), sl(n_), sr(n_), ag(n_), red(n_ * 16) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long gen = generation;
    if (++arrived == n) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

struct LoopbackTransport : Transport {
  LoopbackHub* hub;
  LoopbackTransport(LoopbackHub* h, int r) : hub(h) { rank = r; nranks = h->n; }
  bool graph_capturable() const override { return false; }
  int halo(const double* sl, long long nsl, const double* sr, long long nsr, double* rl, long long nrl, double* rr,
           long long nrr, cudaStream_t s) override {
    (void)nsl; (void)nsr;
    if (cudaStreamSynchronize(s) != cudaSuccess) { set_error("loopback: stream sync"); return -3; }
    hub->sl[rank] = sl;
    hub->sr[rank] = sr;
    hub->barrier();
    if (rank > 0 && cudaMemcpyAsync(rl, hub->sr[rank - 1], sizeof(double) * nrl, cudaMemcpyDeviceToDevice, s))
      return -3;
    if (rank < nranks - 1 && cudaMemcpyAsync(rr, hub->sl[rank + 1], sizeof(double) * nrr, cudaMemcpyDeviceToDevice, s))
      return -3;
    if (cudaStreamSynchronize(s) != cudaSuccess) return -3;
    hub->barrier();
    return 0;
  }
  int allreduce_sum(double* v, int n, cudaStream_t s) override {
    if (n > 16) { set_error("loopback allreduce: n > 16"); return -1; }
    double loc[16];
    if (cudaMemcpyAsync(loc, v, sizeof(double) * n, cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s)) return -3;
    for (int i = 0; i < n; ++i) hub->red[rank * 16 + i] = loc[i];
    hub->barrier();
    for (int i = 0; i < n; ++i) {
      double t = 0.0;
      for (int q = 0; q < nranks; ++q) t += hub->red[q * 16 + i];   // fixed rank order
      loc[i] = t;
    }
    hub->barrier();
    if (cudaMemcpyAsync(v, loc, sizeof(double) * n, cudaMemcpyHostToDevice, s) || cudaStreamSynchronize(s)) return -3;
    return 0;
  }
  int allgather(const double* send, long long n, double* recv, cudaStream_t s) override {
    if (cudaStreamSynchronize(s) != cudaSuccess) return -3;
    hub->ag[rank] = send;
    hub->barrier();
    for (int q = 0; q < nranks; ++q)
      if (cudaMemcpyAsync(recv + (long long)q * n, hub->ag[q], sizeof(double) * n, cudaMemcpyDeviceToDevice, s))
        return -3;
    if (cudaStreamSynchronize(s) != cudaSuccess) return -3;
    hub->barrier();
    return 0;
  }
};

void* loopback_hub_create(int n) { return new LoopbackHub(n); }
void loopback_hub_destroy(void* h) { delete (LoopbackHub*)h; }
Transport* make_loopback_transport(void* hub, int rank) { return new LoopbackTransport((LoopbackHub*)hub, rank); }

// ------------------------------------------------------------------------ shared memory (process ranks) ------
// Segment layout: header {magic, nranks, slot doubles, arrived, generation}, then per rank a mailbox of
// 3 slots (left halo, right halo, allgather) of `cap` doubles each and 16 doubles of reduction scratch.
struct ShmHeader {
  std::atomic<long long> magic;
  int nranks;
  long long cap;
  std::atomic<int> arrived;
  std::atomic<long long> generation;
  std::atomic<int> attached;
};

struct ShmComm {
  int rank = 0, nranks = 1;
  long long cap = 0;
  size_t bytes = 0;
  void* base = nullptr;
  ShmHeader* hdr = nullptr;
  double* data = nullptr;
  char name[128] = {0};
  bool owner = false;
  double* slot(int q, int k) { return data + ((size_t)q * 3 + k) * (size_t)cap; }
  double* red(int q) { return data + (size_t)nranks * 3 * (size_t)cap + (size_t)q * 16; }
  void barrier() {
    const long long gen = hdr->generation.load(std::memory_order_acquire);
    if (hdr->arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == nranks) {
      hdr->arrived.store(0, std::memory_order_relaxed);
      hdr->generation.store(gen + 1, std::memory_order_release);
    } else {
      while (hdr->generation.load(std::memory_order_acquire) == gen) sched_yield();
    }
  }
};

static constexpr long long kShmMagic = 0x73746d676d73686dLL;

int shm_comm_create(const char* name, int nranks, int rank, long long cap_doubles, void** out) {
  if (!name || !out || nranks < 1 || rank < 0 || rank >= nranks || cap_doubles < 1 || std::strlen(name) > 100) {
    set_error("shm comm: bad argument");
    return -1;
  }
  auto* c = new ShmComm();
  c->rank = rank;
  c->nranks = nranks;
  c->cap = cap_doubles;
  std::snprintf(c->name, sizeof(c->name), "/%s", name[0] == '/' ? name + 1 : name);
  c->bytes = sizeof(ShmHeader) + 64 + sizeof(double) * ((size_t)nranks * 3 * (size_t)cap_doubles + (size_t)nranks * 16);
  int fd = -1;
  if (rank == 0) {
    fd = shm_open(c->name, O_CREAT | O_RDWR, 0600);
    if (fd >= 0 && ftruncate(fd, (off_t)c->bytes) != 0) { close(fd); fd = -1; }
    c->owner = true;
  } else {
    for (int it = 0; it < 20000 && fd < 0; ++it) {   // rank 0 creates the segment; wait up to ~20 s
      fd = shm_open(c->name, O_RDWR, 0600);
      if (fd < 0) usleep(1000);
    }
  }
  if (fd < 0) { set_error(std::string("shm comm: shm_open failed for ") + c->name); delete c; return -4; }
  for (int it = 0; it < 20000; ++it) {   // the segment may not be sized yet
    struct stat st;
    if (fstat(fd, &st) == 0 && (size_t)st.st_size >= c->bytes) break;
    usleep(1000);
  }
  c->base = mmap(nullptr, c->bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (c->base == MAP_FAILED) { set_error("shm comm: mmap failed"); delete c; return -4; }
  c->hdr = reinterpret_cast<ShmHeader*>(c->base);
  c->data = reinterpret_cast<double*>(reinterpret_cast<char*>(c->base) + ((sizeof(ShmHeader) + 63) / 64) * 64);
  if (rank == 0) {
    c->hdr->nranks = nranks;
    c->hdr->cap = cap_doubles;
    c->hdr->arrived.store(0);
    c->hdr->generation.store(0);
    c->hdr->attached.store(0);
    c->hdr->magic.store(kShmMagic, std::memory_order_release);
  } else {
    for (int it = 0; it < 20000 && c->hdr->magic.load(std::memory_order_acquire) != kShmMagic; ++it) usleep(1000);
    if (c->hdr->magic.load() != kShmMagic || c->hdr->nranks != nranks || c->hdr->cap != cap_doubles) {
      set_error("shm comm: segment not initialised or ranks / capacity disagree");
      munmap(c->base, c->bytes);
      delete c;
      return -4;
    }
  }
  // pinned host staging for the DMA copies (optional: pageable copies work too)
  cudaHostRegister(c->data, c->bytes - ((char*)c->data - (char*)c->base), cudaHostRegisterDefault);
  cudaGetLastError();
  c->hdr->attached.fetch_add(1);
  c->barrier();   // every rank attached before any exchange
  *out = c;
  return 0;
}

int shm_comm_destroy(void* comm) {
  auto* c = (ShmComm*)comm;
  if (!c) return 0;
  c->barrier();
  cudaHostUnregister(c->data);
  cudaGetLastError();
  munmap(c->base, c->bytes);
  if (c->owner) shm_unlink(c->name);
  delete c;
  return 0;
}

struct ShmTransport : Transport {
  ShmComm* c;
  explicit ShmTransport(ShmComm* comm) : c(comm) { rank = comm->rank; nranks = comm->nranks; }
  bool graph_capturable() const override { return false; }
  int fail(const char* what) {
    set_error(std::string("shm transport: ") + what + ": " + cudaGetErrorString(cudaGetLastError()));
    return -3;
  }
  int check(long long n) {
    if (n > c->cap) { set_error("shm transport: message of " + std::to_string(n) + " doubles exceeds the slot"); return -4; }
    return 0;
  }
  int halo(const double* sl, long long nsl, const double* sr, long long nsr, double* rl, long long nrl, double* rr,
           long long nrr, cudaStream_t s) override {
    if (check(nsl) || check(nsr) || check(nrl) || check(nrr)) return -4;
    if (nsl && cudaMemcpyAsync(c->slot(rank, 0), sl, sizeof(double) * nsl, cudaMemcpyDeviceToHost, s))
      return fail("halo copy out");
    if (nsr && cudaMemcpyAsync(c->slot(rank, 1), sr, sizeof(double) * nsr, cudaMemcpyDeviceToHost, s))
      return fail("halo copy out");
    if (cudaStreamSynchronize(s) != cudaSuccess) return fail("stream sync");
    c->barrier();
    if (nrl && cudaMemcpyAsync(rl, c->slot(rank - 1, 1), sizeof(double) * nrl, cudaMemcpyHostToDevice, s))
      return fail("halo copy in");
    if (nrr && cudaMemcpyAsync(rr, c->slot(rank + 1, 0), sizeof(double) * nrr, cudaMemcpyHostToDevice, s))
      return fail("halo copy in");
    if (cudaStreamSynchronize(s) != cudaSuccess) return fail("stream sync");
    c->barrier();   // the neighbours' slots may be reused only after both reads
    return 0;
  }
  int allreduce_sum(double* v, int n, cudaStream_t s) override {
    if (n > 16) { set_error("shm allreduce: n > 16"); return -1; }
    double loc[16];
    if (cudaMemcpyAsync(loc, v, sizeof(double) * n, cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s))
      return fail("allreduce copy out");
    std::memcpy(c->red(rank), loc, sizeof(double) * n);
    c->barrier();
    for (int i = 0; i < n; ++i) {
      double t = 0.0;
      for (int q = 0; q < nranks; ++q) t += c->red(q)[i];   // fixed rank order: identical on every rank
      loc[i] = t;
    }
    c->barrier();
    if (cudaMemcpyAsync(v, loc, sizeof(double) * n, cudaMemcpyHostToDevice, s) || cudaStreamSynchronize(s))
      return fail("allreduce copy in");
    return 0;
  }
  int allgather(const double* send, long long n, double* recv, cudaStream_t s) override {
    if (check(n)) return -4;
    if (cudaMemcpyAsync(c->slot(rank, 2), send, sizeof(double) * n, cudaMemcpyDeviceToHost, s) ||
        cudaStreamSynchronize(s))
      return -3;
    c->barrier();
    for (int q = 0; q < nranks; ++q)
      if (cudaMemcpyAsync(recv + (long long)q * n, c->slot(q, 2), sizeof(double) * n, cudaMemcpyHostToDevice, s))
        return -3;
    if (cudaStreamSynchronize(s) != cudaSuccess) return -3;
    c->barrier();
    return 0;
  }
};

Transport* make_shm_transport(void* comm) { return comm ? new ShmTransport((ShmComm*)comm) : nullptr; }

}  // namespace stgmg
