// lope_comm.cu — the coarray-style halo exchange between slab partitions, behind the C ABI.
//
// Replaces Machine._halo_exchange (lopec/runtime.py:643-711) between images that live
// on different GPUs (one process -- or one host thread -- per image), for the slab
// decomposition of SURVEY §8(e): the slowest dim split over P images in a ring, every
// face one contiguous run of whole planes (lope_face_span), the other dims wrapped on
// the GPU first so the faces carry the corners (runtime.py:684-687).
//
// Two transports:
//
//  * peer (default): at setup every rank exports its two ping-pong buffers and a pair of
//    step flags (CUDA IPC, or plain pointers between ranks of one process) and opens its
//    ring neighbours'.  A fused step (lope_comm_step) is ONE stencil kernel per rank that
//    stores its boundary planes' periodic images straight into the neighbours' output
//    blocks over NVLink (lope_step_planes_peer), bracketed by stream memory operations on
//    the flags -- wait until both neighbours finished step t-1, then, after the kernel,
//    write t into the neighbours' flags.  No collective, no host round trip, no SM spins:
//    the waits are executed by the GPU front-end (cuStreamWaitValue32), the writes carry
//    a system-scope fence (cuStreamWriteValue32 without NO_MEMORY_BARRIER).
//    lope_halo_exchange (a standalone HALO_TRANSFER) copies the neighbours' faces with one
//    cudaMemcpyAsync per face after a flag handshake.
//  * nccl: lope_comm_nccl_init + lope_halo_exchange = ncclGroupStart / ncclSend x2 /
//    ncclRecv x2 / ncclGroupEnd of the same contiguous faces (NCCL loaded with dlopen --
//    the library still loads where NCCL is absent).
//
// Ordering argument for the fused step (every rank runs the same sequence, lockstep):
// step t on rank r reads in_r (its halo written by the neighbours' step t-1) and writes
// out_r plus the neighbours' out blocks' halos, where out_n(t) = in_n(t-1) is the buffer
// the neighbour read during step t-1.  Both hazards are ordered by "neighbours finished
// step t-1" before r's step t; r's own t-1 is ordered by its stream.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <unistd.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/lope_b200.h"
#include "lope_internal.h"

namespace {

#define COMM_CUDA_TRY(expr)                                                                \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return lope_set_error(-(int)e_, "%s failed: %s", #expr, cudaGetErrorString(e_));     \
  } while (0)

// ---------------------------------------------------------------------------
// Stream memory operations (driver API, fetched at run time)

struct MemOps {
  bool ok = false;
  decltype(&cuStreamWaitValue32) wait = nullptr;
  decltype(&cuStreamWriteValue32) write = nullptr;
};

MemOps& memops() {
  static MemOps m;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && f)
      m.wait = (decltype(m.wait))f;
    f = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && f)
      m.write = (decltype(m.write))f;
    m.ok = m.wait && m.write;
  });
  return m;
}

int cu_err(CUresult r, const char* what) {
  return lope_set_error(-1000 - (int)r, "%s failed (CUresult %d)", what, (int)r);
}

// ---------------------------------------------------------------------------
// NCCL, loaded at run time (the process's copy when torch already loaded one)

struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    if (const char* p = std::getenv("LOPE_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // already in the process (torch)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = "libnccl.so.2 not found (set LOPE_NCCL_LIB)";
      return;
    }
    bool ok = true;
    auto sym = [&](const char* name) {
      void* f = dlsym(h, name);
      if (!f) ok = false;
      return f;
    };
    n.getUniqueId = (decltype(n.getUniqueId))sym("ncclGetUniqueId");
    n.commInitRank = (decltype(n.commInitRank))sym("ncclCommInitRank");
    n.commDestroy = (decltype(n.commDestroy))sym("ncclCommDestroy");
    n.send = (decltype(n.send))sym("ncclSend");
    n.recv = (decltype(n.recv))sym("ncclRecv");
    n.groupStart = (decltype(n.groupStart))sym("ncclGroupStart");
    n.groupEnd = (decltype(n.groupEnd))sym("ncclGroupEnd");
    n.errorString = (decltype(n.errorString))sym("ncclGetErrorString");
    n.ok = ok;
    if (!ok) n.why = "libnccl.so.2 lacks a required entry point";
  });
  return n;
}

int nccl_err(ncclResult_t r, const char* what) {
  const char* s = nccl().errorString ? nccl().errorString(r) : "?";
  return lope_set_error(-4000 - (int)r, "%s failed: %s", what, s);
}

// ---------------------------------------------------------------------------
// The per-rank record exchanged at setup (plain bytes: any out-of-band channel works)

constexpr uint32_t kMagic = 0x4c4f5043;   // "LOPC"
constexpr uint32_t kVersion = 1;

struct Record {
  uint32_t magic, version;
  int32_t rank, nranks;
  int32_t device, pid;
  uint64_t host;                      // gethostid(): IPC and raw pointers only within one node
  int64_t interior[3];
  int32_t lo[3], hi[3];
  int64_t count, elem_bytes;
  uint64_t raw_buf[2], raw_flags;     // pointers, usable by ranks of the same process
  uint8_t ipc_buf[2][64], ipc_flags[64];
  int64_t off_buf[2], off_flags;      // offsets of the pointers inside their allocations
  int32_t has_ipc;
  int32_t pad;
  char bus[32];                       // PCI bus id of the device: ranks of two processes on one GPU
};

}  // namespace

struct lope_comm {
  int rank = 0, nranks = 1, device = 0;
  bool exported = false, connected = false;
  lope_layout layout;
  void* bufs[2] = {nullptr, nullptr};
  int32_t* flags = nullptr;             // this rank's flags: [0] written by prev, [1] by next
  void* nb_bufs[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};   // [prev|next][buffer]
  int32_t* nb_flags[2] = {nullptr, nullptr};
  std::vector<void*> opened;            // IPC mappings to close (the pointers lope_ipc_open returned)
  uint32_t epoch = 0;                   // completed synchronised operations
  // Neighbours in another process on the SAME GPU: their stream waits would block each
  // other's contexts (B200_PROFILING.md: ranks sharing a GPU must not wait on one another),
  // so the flags are not used and the caller orders the operations on the host.
  bool host_ordered = false;
  uint32_t pending = 0;                 // signalled exchange awaiting lope_halo_exchange_end
  int pending_live = 0;
  ncclComm_t nccl = nullptr;
  Record mine;
};

namespace {

int prev_of(const lope_comm* c) { return (c->rank + c->nranks - 1) % c->nranks; }
int next_of(const lope_comm* c) { return (c->rank + 1) % c->nranks; }

int check_stream_memops() {
  if (!memops().ok)
    return lope_set_error(-3, "stream memory operations (cuStreamWaitValue32/WriteValue32) unavailable");
  return 0;
}

// this rank finished operation `v`: tell both neighbours (their flag slot for us)
int signal(lope_comm* c, uint32_t v, cudaStream_t st) {
  if (c->nranks == 1 || c->host_ordered) return 0;
  if (int e = check_stream_memops()) return e;
  // prev's slot [1] is written by its next neighbour (us); next's slot [0] by its prev (us)
  int32_t* targets[2] = {c->nb_flags[0] + 1, c->nb_flags[1] + 0};
  for (int i = 0; i < 2; ++i) {
    CUresult r = memops().write((CUstream)st, (CUdeviceptr)targets[i], v, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) return cu_err(r, "cuStreamWriteValue32");
  }
  return 0;
}

// wait (on the stream) until both neighbours have signalled at least `v`
int wait_for(lope_comm* c, uint32_t v, cudaStream_t st) {
  if (c->nranks == 1 || v == 0 || c->host_ordered) return 0;
  if (int e = check_stream_memops()) return e;
  for (int i = 0; i < 2; ++i) {
    CUresult r = memops().wait((CUstream)st, (CUdeviceptr)(c->flags + i), v, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return cu_err(r, "cuStreamWaitValue32");
  }
  return 0;
}

int export_ptr(const void* p, uint8_t* h, int64_t* off) { return lope_ipc_export(p, h, off); }

int slow_dim(const lope_layout* L) { return L->rank - 1; }

}  // namespace

extern "C" {

int lope_comm_record_size(void) { return (int)sizeof(Record); }

int lope_peer_enable(int32_t peer_device) {
  int cur = 0;
  COMM_CUDA_TRY(cudaGetDevice(&cur));
  if (peer_device == cur) return 0;
  int can = 0;
  COMM_CUDA_TRY(cudaDeviceCanAccessPeer(&can, cur, peer_device));
  if (!can) return lope_set_error(-3, "device %d cannot access device %d's memory (no P2P)", cur, peer_device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return 0;
  }
  if (e != cudaSuccess) return lope_set_error(-(int)e, "cudaDeviceEnablePeerAccess(%d): %s", peer_device,
                                              cudaGetErrorString(e));
  return 0;
}

int lope_comm_create(int32_t nranks, int32_t rank, lope_comm** out) {
  if (!out) return lope_set_error(108, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return lope_set_error(201, "rank %d of %d images is not a valid image index", rank, nranks);
  lope_comm* c = new lope_comm();
  c->rank = rank;
  c->nranks = nranks;
  std::memset(&c->layout, 0, sizeof c->layout);
  std::memset(&c->mine, 0, sizeof c->mine);
  *out = c;
  return 0;
}

int lope_comm_destroy(lope_comm* c) {
  if (!c) return 0;
  for (void* p : c->opened) lope_ipc_close(p);
  if (c->flags) cudaFree(c->flags);
  if (c->nccl && nccl().ok) nccl().commDestroy(c->nccl);
  delete c;
  return 0;
}

int lope_comm_export(lope_comm* c, const lope_layout* layout, void* buf0, void* buf1, uint8_t* record) {
  if (!c || !layout || !record) return lope_set_error(108, "null argument");
  if (!buf0 || !buf1) return lope_set_error(202, "ping-pong buffers not allocated");
  if (buf0 == buf1) return lope_set_error(108, "the two ping-pong buffers must differ");
  if (layout->rank < 1 || layout->rank > 3) return lope_set_error(108, "layout rank %d", layout->rank);
  const int d = slow_dim(layout);
  if (c->nranks > 1 && (layout->lo[d] > layout->interior[d] || layout->hi[d] > layout->interior[d]))
    return lope_set_error(108, "halo widths (%d,%d) exceed the per-image extent %lld of the decomposed dim "
                               "(SURVEY F8)", layout->lo[d], layout->hi[d], (long long)layout->interior[d]);
  COMM_CUDA_TRY(cudaGetDevice(&c->device));
  if (!c->flags) {
    COMM_CUDA_TRY(cudaMalloc(&c->flags, 64));
    COMM_CUDA_TRY(cudaMemset(c->flags, 0, 64));
    COMM_CUDA_TRY(cudaDeviceSynchronize());
  }
  c->layout = *layout;
  c->bufs[0] = buf0;
  c->bufs[1] = buf1;
  Record& r = c->mine;
  std::memset(&r, 0, sizeof r);
  r.magic = kMagic;
  r.version = kVersion;
  r.rank = c->rank;
  r.nranks = c->nranks;
  r.device = c->device;
  r.pid = (int32_t)getpid();
  r.host = (uint64_t)gethostid();
  for (int i = 0; i < 3; ++i) {
    r.interior[i] = layout->interior[i];
    r.lo[i] = layout->lo[i];
    r.hi[i] = layout->hi[i];
  }
  r.count = layout->count;
  r.elem_bytes = layout->elem_bytes;
  r.raw_buf[0] = (uint64_t)(uintptr_t)buf0;
  r.raw_buf[1] = (uint64_t)(uintptr_t)buf1;
  r.raw_flags = (uint64_t)(uintptr_t)c->flags;
  r.has_ipc = 0;
  if (cudaDeviceGetPCIBusId(r.bus, (int)sizeof r.bus - 1, c->device) != cudaSuccess) r.bus[0] = 0;
  if (c->nranks > 1 && !std::getenv("LOPE_COMM_NO_IPC")) {
    // IPC handles for neighbours in other processes (ranks of this process use raw pointers)
    if (export_ptr(buf0, r.ipc_buf[0], &r.off_buf[0]) == 0 && export_ptr(buf1, r.ipc_buf[1], &r.off_buf[1]) == 0 &&
        export_ptr(c->flags, r.ipc_flags, &r.off_flags) == 0)
      r.has_ipc = 1;
  }
  std::memcpy(record, &r, sizeof r);
  c->exported = true;
  return 0;
}

int lope_comm_connect(lope_comm* c, const uint8_t* records) {
  if (!c || !records) return lope_set_error(108, "null argument");
  if (!c->exported) return lope_set_error(202, "lope_comm_export must run before lope_comm_connect");
  if (c->connected) return lope_set_error(108, "communicator already connected");
  std::vector<Record> all(c->nranks);
  for (int k = 0; k < c->nranks; ++k) {
    std::memcpy(&all[k], records + (size_t)k * sizeof(Record), sizeof(Record));
    const Record& r = all[k];
    if (r.magic != kMagic || r.version != kVersion)
      return lope_set_error(108, "record %d is not a lope_comm record of this version", k);
    if (r.rank != k || r.nranks != c->nranks)
      return lope_set_error(201, "record %d claims image %d of %d (expected %d of %d)", k, r.rank, r.nranks, k,
                            c->nranks);
    for (int i = 0; i < 3; ++i)
      if (r.interior[i] != c->mine.interior[i] || r.lo[i] != c->mine.lo[i] || r.hi[i] != c->mine.hi[i])
        return lope_set_error(108, "image %d's block differs from this image's (blocks must be uniform, "
                                   "runtime.py:467-470)", k + 1);
    if (r.count != c->mine.count || r.elem_bytes != c->mine.elem_bytes)
      return lope_set_error(108, "image %d's block storage differs", k + 1);
  }
  if (c->nranks > 1) {
    const int nb[2] = {prev_of(c), next_of(c)};
    for (int s = 0; s < 2; ++s) {
      const Record& r = all[nb[s]];
      // the same neighbour on both sides (P = 2) is mapped once
      if (s == 1 && nb[1] == nb[0]) {
        c->nb_bufs[1][0] = c->nb_bufs[0][0];
        c->nb_bufs[1][1] = c->nb_bufs[0][1];
        c->nb_flags[1] = c->nb_flags[0];
        continue;
      }
      const bool local = r.pid == c->mine.pid && r.host == c->mine.host;
      if (local) {
        c->nb_bufs[s][0] = (void*)(uintptr_t)r.raw_buf[0];
        c->nb_bufs[s][1] = (void*)(uintptr_t)r.raw_buf[1];
        c->nb_flags[s] = (int32_t*)(uintptr_t)r.raw_flags;
        if (r.device != c->device) {
          cudaError_t e = cudaDeviceEnablePeerAccess(r.device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            return lope_set_error(-(int)e, "peer access to device %d: %s", r.device, cudaGetErrorString(e));
          cudaGetLastError();
        }
        continue;
      }
      if (!r.has_ipc) return lope_set_error(-3, "image %d exported no IPC handles", nb[s] + 1);
      if (r.host != c->mine.host) return lope_set_error(-3, "image %d is on another node", nb[s] + 1);
      if (r.bus[0] && std::strncmp(r.bus, c->mine.bus, sizeof r.bus) == 0) c->host_ordered = true;
      void* p = nullptr;
      for (int b = 0; b < 2; ++b) {
        if (int e = lope_ipc_open(r.ipc_buf[b], r.off_buf[b], &p)) return e;
        c->opened.push_back(p);
        c->nb_bufs[s][b] = p;
      }
      if (int e = lope_ipc_open(r.ipc_flags, r.off_flags, &p)) return e;
      c->opened.push_back(p);
      c->nb_flags[s] = (int32_t*)p;
    }
  }
  c->connected = true;
  return 0;
}

int lope_comm_nccl_unique_id(uint8_t* id) {
  if (!id) return lope_set_error(108, "null argument");
  Nccl& n = nccl();
  if (!n.ok) return lope_set_error(-3, "NCCL unavailable: %s", n.why.c_str());
  ncclUniqueId u;
  ncclResult_t r = n.getUniqueId(&u);
  if (r != ncclSuccess) return nccl_err(r, "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof u);
  return 0;
}

int lope_comm_nccl_init(lope_comm* c, const uint8_t* id) {
  if (!c || !id) return lope_set_error(108, "null argument");
  Nccl& n = nccl();
  if (!n.ok) return lope_set_error(-3, "NCCL unavailable: %s", n.why.c_str());
  if (c->nccl) return lope_set_error(108, "NCCL already initialised on this communicator");
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  ncclResult_t r = n.commInitRank(&c->nccl, c->nranks, u, c->rank);
  if (r != ncclSuccess) {
    c->nccl = nullptr;
    return nccl_err(r, "ncclCommInitRank");
  }
  return 0;
}

int lope_comm_info(const lope_comm* c, int32_t* rank, int32_t* nranks, uint32_t* epoch, int32_t* transport) {
  if (!c) return lope_set_error(108, "null argument");
  if (rank) *rank = c->rank;
  if (nranks) *nranks = c->nranks;
  if (epoch) *epoch = c->epoch;
  if (transport) *transport = c->connected ? (c->host_ordered ? 3 : 1) : (c->nccl ? 2 : 0);
  return 0;
}

// HALO_TRANSFER(U, BC=CYCLIC) of this rank's slab (runtime.py:643-711): the dims that are
// not decomposed wrap on the GPU, then the decomposed dim's halos receive the ring
// neighbours' faces.  `live` is the index (0/1) of the exported buffer holding the field
// -- the same on every rank (lockstep).  Split phase: _begin wraps the local dims and
// tells the neighbours this block is ready, _end waits for theirs and copies the faces
// (NCCL transport: all of it in _begin).  lope_halo_exchange = _begin + _end.
int lope_halo_exchange_begin(lope_comm* c, int32_t live, int32_t dims_mask, void* stream) {
  if (!c) return lope_set_error(108, "null argument");
  if (!c->exported) return lope_set_error(202, "lope_comm_export has not run");
  if (live != 0 && live != 1) return lope_set_error(108, "live buffer index %d", live);
  if (c->pending) return lope_set_error(108, "lope_halo_exchange_begin called twice without _end");
  const lope_layout* L = &c->layout;
  cudaStream_t st = (cudaStream_t)stream;
  const int d = slow_dim(L);
  const int mask = dims_mask & ((1 << L->rank) - 1);
  void* buf = c->bufs[live];
  if (c->nranks == 1) return mask ? lope_halo_fill(L, buf, mask, stream) : 0;
  if (mask & ~(1 << d))
    if (int e = lope_halo_fill(L, buf, mask & ~(1 << d), stream)) return e;
  if (!(mask & (1 << d))) return 0;
  int64_t off[4], cnt[4];
  for (int w = 0; w < 4; ++w)
    if (int e = lope_face_span(L, w, &off[w], &cnt[w])) return e;
  const int64_t eb = L->elem_bytes;
  char* base = (char*)buf;
  if (c->connected) {
    // this block (local wrap and every earlier write) is ready to be read
    const uint32_t v = c->epoch + 1;
    if (int e = signal(c, v, st)) return e;
    c->pending = v;
    c->pending_live = live;
    return 0;
  }
  if (!c->nccl) return lope_set_error(202, "communicator has neither a peer mapping nor NCCL");
  Nccl& n = nccl();
  const int prev = prev_of(c), next = next_of(c);
  ncclResult_t r = n.groupStart();
  if (r != ncclSuccess) return nccl_err(r, "ncclGroupStart");
  // same order on every rank, so the two directions pair up even when prev == next
  ncclResult_t rr[4] = {ncclSuccess, ncclSuccess, ncclSuccess, ncclSuccess};
  if (cnt[3]) rr[0] = n.send(base + off[3] * eb, (size_t)(cnt[3] * eb), ncclInt8, next, c->nccl, st);
  if (cnt[2]) rr[1] = n.send(base + off[2] * eb, (size_t)(cnt[2] * eb), ncclInt8, prev, c->nccl, st);
  if (cnt[0]) rr[2] = n.recv(base + off[0] * eb, (size_t)(cnt[0] * eb), ncclInt8, prev, c->nccl, st);
  if (cnt[1]) rr[3] = n.recv(base + off[1] * eb, (size_t)(cnt[1] * eb), ncclInt8, next, c->nccl, st);
  r = n.groupEnd();
  for (ncclResult_t x : rr)
    if (x != ncclSuccess) return nccl_err(x, "ncclSend/ncclRecv");
  if (r != ncclSuccess) return nccl_err(r, "ncclGroupEnd");
  return 0;
}

int lope_halo_exchange_end(lope_comm* c, void* stream) {
  if (!c) return lope_set_error(108, "null argument");
  if (!c->pending) return 0;                 // P = 1, local dims only, or NCCL (done in _begin)
  const lope_layout* L = &c->layout;
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t v = c->pending;
  const int live = c->pending_live;
  c->pending = 0;
  if (int e = wait_for(c, v, st)) return e;
  int64_t off[4], cnt[4];
  for (int w = 0; w < 4; ++w)
    if (int e = lope_face_span(L, w, &off[w], &cnt[w])) return e;
  const int64_t eb = L->elem_bytes;
  char* base = (char*)c->bufs[live];
  // low halo <- prev's last `lo` planes; high halo <- next's first `hi` planes
  if (cnt[0])
    COMM_CUDA_TRY(cudaMemcpyAsync(base + off[0] * eb, (char*)c->nb_bufs[0][live] + off[3] * eb, cnt[0] * eb,
                                  cudaMemcpyDeviceToDevice, st));
  if (cnt[1])
    COMM_CUDA_TRY(cudaMemcpyAsync(base + off[1] * eb, (char*)c->nb_bufs[1][live] + off[2] * eb, cnt[1] * eb,
                                  cudaMemcpyDeviceToDevice, st));
  c->epoch = v;
  return 0;
}

int lope_halo_exchange(lope_comm* c, int32_t live, int32_t dims_mask, void* stream) {
  if (int e = lope_halo_exchange_begin(c, live, dims_mask, stream)) return e;
  return lope_halo_exchange_end(c, stream);
}

// One fused step of the slab: wait for both neighbours' previous operation, one stencil
// kernel (full interior, local dims' images in this block, the decomposed dim's images in
// the neighbours' output blocks), then signal.  Reads buffer `live`, writes 1 - live.
int lope_comm_step(lope_comm* c, const lope_kernel* k, int32_t live, const double* rscal, const int64_t* iscal,
                   void* stream) {
  if (!c || !k) return lope_set_error(108, "null argument");
  if (!c->exported) return lope_set_error(202, "lope_comm_export has not run");
  if (live != 0 && live != 1) return lope_set_error(108, "live buffer index %d", live);
  const lope_layout* L = &c->layout;
  cudaStream_t st = (cudaStream_t)stream;
  const int full = (1 << L->rank) - 1;
  const int d = slow_dim(L);
  const int out = 1 - live;
  if (c->nranks == 1)
    return lope_step_planes(k, L, c->bufs[live], c->bufs[out], 0, L->interior[d], rscal, iscal, full, stream);
  if (!c->connected) return lope_set_error(202, "fused steps need lope_comm_connect (peer mapping)");
  if (c->pending) return lope_set_error(108, "a halo exchange is still open (lope_halo_exchange_end)");
  if (int e = wait_for(c, c->epoch, st)) return e;
  if (int e = lope_step_planes_peer(k, L, c->bufs[live], c->bufs[out], 0, L->interior[d], rscal, iscal, full,
                                    c->nb_bufs[0][out], c->nb_bufs[1][out], stream))
    return e;
  const uint32_t v = c->epoch + 1;
  if (int e = signal(c, v, st)) return e;
  c->epoch = v;
  return 0;
}

// Order this rank after both neighbours' latest operation (their stores into this
// rank's halos are complete): before a plain launch or a download of a fused-step slab.
int lope_comm_sync(lope_comm* c, void* stream) {
  if (!c) return lope_set_error(108, "null argument");
  if (c->nranks == 1 || !c->connected) return 0;
  return wait_for(c, c->epoch, (cudaStream_t)stream);
}

}  // extern "C"
