// fake_nccl.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A host-shared-memory stand-in for the NCCL entry points libb2m resolves at
// run time (b2m_world.cu, NcclApi), so that several ranks of the native slab
// world -- separate processes -- can run on ONE GPU: real NCCL refuses two
// ranks on one device, and this round's GPU boxes have one.  Loaded through
// B2M_NCCL_LIB.  Every call is synchronous on the host: it waits for the
// caller's stream, moves the bytes through POSIX shared memory, and copies
// results back.  Semantics kept: point-to-point messages between two ranks
// match in posting order; grouped sends and receives progress together (no
// deadlock when both sides send first); reductions add the ranks' buffers in
// rank order.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace {

constexpr size_t kHeader = 4096;
constexpr size_t kSlot = 4u << 20;   // per-rank collective slot (/dev/shm may be 64 MB)
constexpr size_t kBox = 2u << 20;    // per (src, dst) ring
constexpr uint64_t kMagic = 0x62326d66616b6531ull;

struct Header {
  std::atomic<uint64_t> magic;
  std::atomic<int> arrived;
  std::atomic<int> generation;
  int nranks;
};

struct Ring {
  std::atomic<uint64_t> written;  // bytes ever written
  std::atomic<uint64_t> read;     // bytes ever read
  char pad[48];
};

struct Comm {
  std::string name;
  int nranks = 0, rank = 0;
  char* base = nullptr;
  size_t bytes = 0;
  Header* hdr() { return reinterpret_cast<Header*>(base); }
  char* slot(int r) { return base + kHeader + static_cast<size_t>(r) * kSlot; }
  Ring* ring(int src, int dst) {
    char* p = base + kHeader + static_cast<size_t>(nranks) * kSlot +
              (static_cast<size_t>(src) * nranks + dst) * (sizeof(Ring) + kBox);
    return reinterpret_cast<Ring*>(p);
  }
  char* ring_data(int src, int dst) { return reinterpret_cast<char*>(ring(src, dst) + 1); }
};

size_t seg_bytes(int n) {
  return kHeader + static_cast<size_t>(n) * kSlot +
         static_cast<size_t>(n) * n * (sizeof(Ring) + kBox);
}

void barrier(Comm* c) {
  Header* h = c->hdr();
  const int gen = h->generation.load();
  if (h->arrived.fetch_add(1) == c->nranks - 1) {
    h->arrived.store(0);
    h->generation.fetch_add(1);
  } else {
    while (h->generation.load() == gen) sched_yield();
  }
}

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
    default: return 0;
  }
}

template <class T>
void reduce_into(T* acc, const T* x, size_t n, ncclRedOp_t op) {
  for (size_t i = 0; i < n; ++i) {
    if (op == ncclSum) acc[i] = acc[i] + x[i];
    else if (op == ncclMax) acc[i] = std::max(acc[i], x[i]);
    else if (op == ncclMin) acc[i] = std::min(acc[i], x[i]);
    else if (op == ncclProd) acc[i] = acc[i] * x[i];
  }
}

void reduce_typed(void* acc, const void* x, size_t n, ncclDataType_t t, ncclRedOp_t op) {
  switch (t) {
    case ncclInt64: reduce_into(static_cast<long long*>(acc), static_cast<const long long*>(x), n, op); break;
    case ncclUint64: reduce_into(static_cast<unsigned long long*>(acc), static_cast<const unsigned long long*>(x), n, op); break;
    case ncclFloat64: reduce_into(static_cast<double*>(acc), static_cast<const double*>(x), n, op); break;
    case ncclInt32: reduce_into(static_cast<int*>(acc), static_cast<const int*>(x), n, op); break;
    case ncclUint32: reduce_into(static_cast<unsigned*>(acc), static_cast<const unsigned*>(x), n, op); break;
    case ncclFloat32: reduce_into(static_cast<float*>(acc), static_cast<const float*>(x), n, op); break;
    default: break;
  }
}

// A copy on the caller's stream, complete on return (a plain cudaMemcpy from
// pageable memory may return before its DMA lands, and the caller's stream
// need not be ordered after the legacy default stream).
void copy_sync(void* dst, const void* src, size_t n, cudaMemcpyKind kind, cudaStream_t st) {
  if (!n) return;
  const cudaError_t pending = cudaGetLastError();  // not ours: report, do not fail on it
  if (pending != cudaSuccess && std::getenv("FAKE_NCCL_DEBUG"))
    std::fprintf(stderr, "fake nccl: pending error before copy: %s\n", cudaGetErrorString(pending));
  cudaError_t e = cudaMemcpyAsync(dst, src, n, kind, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    int dev = -1;
    cudaGetDevice(&dev);
    cudaPointerAttributes a{}, b{};
    cudaPointerGetAttributes(&a, dst);
    cudaPointerGetAttributes(&b, src);
    cudaGetLastError();
    std::fprintf(stderr,
                 "fake nccl: copy failed: %s (dst %p type %d dev %d, src %p type %d dev %d, "
                 "%zu bytes, kind %d, stream %p, current device %d)\n",
                 cudaGetErrorString(e), dst, static_cast<int>(a.type), a.device, src,
                 static_cast<int>(b.type), b.device, n, static_cast<int>(kind),
                 static_cast<void*>(st), dev);
    std::abort();
  }
}

// ---- grouped point-to-point ------------------------------------------------
struct P2P {
  bool send;
  int peer;
  void* dev;
  size_t bytes;
  cudaStream_t stream;
  Comm* comm;
};
thread_local int g_depth = 0;
thread_local std::vector<P2P> g_ops;

ncclResult_t run_p2p(std::vector<P2P>& ops) {
  if (std::getenv("FAKE_NCCL_DEBUG") && !ops.empty()) {
    std::fprintf(stderr, "[fake r%d] p2p group:", ops[0].comm->rank);
    for (const P2P& o : ops) std::fprintf(stderr, " %s%d:%zu", o.send ? "S" : "R", o.peer, o.bytes);
    std::fprintf(stderr, "\n");
  }
  for (const P2P& o : ops) cudaStreamSynchronize(o.stream);
  std::vector<std::vector<char>> host(ops.size());
  std::vector<size_t> done(ops.size(), 0);
  for (size_t i = 0; i < ops.size(); ++i) {
    host[i].resize(ops[i].bytes);
    if (ops[i].send && ops[i].bytes)
      copy_sync(host[i].data(), ops[i].dev, ops[i].bytes, cudaMemcpyDeviceToHost, ops[i].stream);
  }
  // progress every op in posting order per (direction, peer) until all done
  for (;;) {
    bool all = true, moved = false;
    for (size_t i = 0; i < ops.size(); ++i) {
      P2P& o = ops[i];
      if (done[i] == o.bytes) continue;
      // only the first unfinished op of this (direction, peer) may move
      bool first = true;
      for (size_t k = 0; k < i; ++k)
        if (ops[k].send == o.send && ops[k].peer == o.peer && done[k] != ops[k].bytes)
          first = false;
      if (!first) { all = false; continue; }
      Comm* c = o.comm;
      Ring* r = o.send ? c->ring(c->rank, o.peer) : c->ring(o.peer, c->rank);
      char* data = o.send ? c->ring_data(c->rank, o.peer) : c->ring_data(o.peer, c->rank);
      const uint64_t w = r->written.load(), rd = r->read.load();
      size_t n;
      if (o.send) {
        n = std::min<size_t>(o.bytes - done[i], kBox - (w - rd));
        for (size_t b = 0; b < n;) {
          const size_t off = (w + b) % kBox, run = std::min(n - b, kBox - off);
          std::memcpy(data + off, host[i].data() + done[i] + b, run);
          b += run;
        }
        if (n) r->written.store(w + n);
      } else {
        n = std::min<size_t>(o.bytes - done[i], w - rd);
        for (size_t b = 0; b < n;) {
          const size_t off = (rd + b) % kBox, run = std::min(n - b, kBox - off);
          std::memcpy(host[i].data() + done[i] + b, data + off, run);
          b += run;
        }
        if (n) r->read.store(rd + n);
      }
      done[i] += n;
      moved = moved || n > 0;
      if (done[i] != o.bytes) all = false;
    }
    if (all) break;
    if (!moved) sched_yield();
  }
  if (std::getenv("FAKE_NCCL_DEBUG"))
    for (size_t i = 0; i < ops.size(); ++i)
      if (ops[i].bytes <= 64) {
        std::fprintf(stderr, "[fake r%d]   %s%d:", ops[i].comm->rank, ops[i].send ? "S" : "R",
                     ops[i].peer);
        for (size_t b = 0; b + 8 <= ops[i].bytes; b += 8) {
          unsigned long long v;
          std::memcpy(&v, host[i].data() + b, 8);
          std::fprintf(stderr, " %llu", v);
        }
        std::fprintf(stderr, "\n");
      }
  for (size_t i = 0; i < ops.size(); ++i)
    if (!ops[i].send && ops[i].bytes)
      copy_sync(ops[i].dev, host[i].data(), ops[i].bytes, cudaMemcpyHostToDevice, ops[i].stream);
  return ncclSuccess;
}

ncclResult_t post(const P2P& o) {
  if (g_depth > 0) {
    g_ops.push_back(o);
    return ncclSuccess;
  }
  std::vector<P2P> one{o};
  return run_p2p(one);
}

}  // namespace

extern "C" {

const char* ncclGetErrorString(ncclResult_t r) {
  return r == ncclSuccess ? "no error (fake nccl)" : "fake nccl error";
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  std::memset(id, 0, sizeof(*id));
  static int counter = 0;
  const auto t = std::chrono::steady_clock::now().time_since_epoch().count();
  std::snprintf(id->internal, sizeof(id->internal), "/b2m_fake_%d_%d_%lld", getpid(), counter++,
                static_cast<long long>(t % 1000000007));
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
  Comm* c = new Comm;
  c->name = id.internal;
  c->nranks = nranks;
  c->rank = rank;
  c->bytes = seg_bytes(nranks);
  int fd = -1;
  if (rank == 0) {
    fd = shm_open(c->name.c_str(), O_CREAT | O_RDWR, 0600);
    if (fd < 0 || ftruncate(fd, static_cast<off_t>(c->bytes)) != 0) return ncclSystemError;
  } else {
    for (int i = 0; i < 600000 && fd < 0; ++i) {
      fd = shm_open(c->name.c_str(), O_RDWR, 0600);
      if (fd < 0) usleep(100);
    }
    if (fd < 0) return ncclSystemError;
    struct stat st;
    for (int i = 0; i < 600000; ++i) {
      if (fstat(fd, &st) == 0 && static_cast<size_t>(st.st_size) >= c->bytes) break;
      usleep(100);
    }
  }
  void* p = mmap(nullptr, c->bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return ncclSystemError;
  c->base = static_cast<char*>(p);
  Header* h = c->hdr();
  if (rank == 0) {
    h->arrived.store(0);
    h->generation.store(0);
    h->nranks = nranks;
    for (int s = 0; s < nranks; ++s)
      for (int d = 0; d < nranks; ++d) {
        c->ring(s, d)->written.store(0);
        c->ring(s, d)->read.store(0);
      }
    h->magic.store(kMagic);
  } else {
    while (h->magic.load() != kMagic) sched_yield();
  }
  barrier(c);
  if (std::getenv("FAKE_NCCL_DEBUG"))
    std::fprintf(stderr, "[fake %s r%d/%d] init done\n", c->name.c_str(), rank, nranks);
  *out = reinterpret_cast<ncclComm_t>(c);
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  barrier(c);
  munmap(c->base, c->bytes);
  if (c->rank == 0) shm_unlink(c->name.c_str());
  delete c;
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
  ++g_depth;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (--g_depth > 0) return ncclSuccess;
  std::vector<P2P> ops;
  ops.swap(g_ops);
  return ops.empty() ? ncclSuccess : run_p2p(ops);
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
  return post(P2P{true, peer, const_cast<void*>(buf), count * type_size(t), stream,
                  reinterpret_cast<Comm*>(comm)});
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
  return post(P2P{false, peer, buf, count * type_size(t), stream, reinterpret_cast<Comm*>(comm)});
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t t,
                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t stream) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  if (std::getenv("FAKE_NCCL_DEBUG"))
    std::fprintf(stderr, "[fake %s r%d] allreduce count %zu type %d op %d\n", c->name.c_str(),
                 c->rank, count, static_cast<int>(t), static_cast<int>(op));
  const size_t es = type_size(t), per = kSlot / es;
  cudaStreamSynchronize(stream);
  std::vector<char> acc;
  for (size_t o = 0; o < count; o += per) {
    const size_t n = std::min(per, count - o);
    copy_sync(c->slot(c->rank), static_cast<const char*>(send) + o * es, n * es,
              cudaMemcpyDeviceToHost, stream);
    barrier(c);
    acc.assign(c->slot(0), c->slot(0) + n * es);
    for (int r = 1; r < c->nranks; ++r) reduce_typed(acc.data(), c->slot(r), n, t, op);
    barrier(c);
    copy_sync(static_cast<char*>(recv) + o * es, acc.data(), n * es, cudaMemcpyHostToDevice, stream);
  }
  return ncclSuccess;
}

ncclResult_t ncclBroadcast(const void* send, void* recv, size_t count, ncclDataType_t t, int root,
                           ncclComm_t comm, cudaStream_t stream) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  if (std::getenv("FAKE_NCCL_DEBUG"))
    std::fprintf(stderr, "[fake r%d] broadcast %zu root %d\n", c->rank, count, root);
  const size_t es = type_size(t), per = kSlot / es;
  cudaStreamSynchronize(stream);
  for (size_t o = 0; o < count; o += per) {
    const size_t n = std::min(per, count - o);
    if (c->rank == root)
      copy_sync(c->slot(root), static_cast<const char*>(send) + o * es, n * es,
                cudaMemcpyDeviceToHost, stream);
    barrier(c);
    copy_sync(static_cast<char*>(recv) + o * es, c->slot(root), n * es, cudaMemcpyHostToDevice,
              stream);
    barrier(c);
  }
  return ncclSuccess;
}

ncclResult_t ncclAllGather(const void* send, void* recv, size_t count, ncclDataType_t t,
                           ncclComm_t comm, cudaStream_t stream) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  const size_t es = type_size(t), per = kSlot / es;
  cudaStreamSynchronize(stream);
  for (size_t o = 0; o < count; o += per) {
    const size_t n = std::min(per, count - o);
    copy_sync(c->slot(c->rank), static_cast<const char*>(send) + o * es, n * es,
              cudaMemcpyDeviceToHost, stream);
    barrier(c);
    for (int r = 0; r < c->nranks; ++r)
      copy_sync(static_cast<char*>(recv) + (static_cast<size_t>(r) * count + o) * es, c->slot(r),
                n * es, cudaMemcpyHostToDevice, stream);
    barrier(c);
  }
  return ncclSuccess;
}

}  // extern "C"
