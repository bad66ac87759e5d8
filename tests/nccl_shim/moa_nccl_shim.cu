// moa_nccl_shim.cu — TEST INFRASTRUCTURE ONLY (never linked into libmoa.so).
//
// A stand-in for the subset of NCCL that libmoa.so calls, so that G = 2..8
// processes sharing ONE GPU can drive every `nranks > 1` branch of the lifted
// entry points (moa_gemm_lifted*, _cols, _2d, _gather, _host) on a one-GPU box.
// Real NCCL refuses two ranks on one device ("Duplicate GPU detected"), which is
// why round 1 could only run the lifted paths on 1-rank communicators.
//
// It is LD_PRELOADed ahead of torch's libnccl.so.2 by the multi-process tests
// (tests/test_lifted_multiproc_gpu.py); symbols it does not define still resolve
// to the real library. Semantics:
//   * collectives (Broadcast / AllGather / AllReduce) are stream-ordered and
//     SYNCHRONOUS: the stream is synchronised, data crosses through a file-backed
//     shared host staging area in fixed-size chunks, and the receive side's copies
//     complete on the same stream before the call returns; group calls execute
//     each op immediately, in issue order (every rank issues the same sequence);
//   * ncclCommSplit exchanges (color, key) through the parent's mailbox;
//   * ncclMemAlloc / ncclCommWindowRegister build real symmetric windows with the
//     CUDA VMM API: POSIX-fd handles are passed between processes over unix
//     sockets (SCM_RIGHTS) and every rank's allocation is mapped into one flat
//     virtual range at a 4 GiB stride, described by the public ncclWindow_vidmem
//     layout, so NCCL's device API (ncclGetPeerPointer) resolves peer addresses
//     exactly as with real NCCL and libmoa's fused-gather epilogue stores into the
//     other processes' memory;
//   * every data collective is appended to $MOA_NCCL_SHIM_LOG (one JSON line:
//     op, communicator label, root, element count, element size) so tests can
//     check the executed collective sequence against moa_exchange_plan.
// Barriers time out after $MOA_NCCL_SHIM_TIMEOUT seconds (default 300) with
// ncclSystemError instead of hanging the test.
#include <cuda.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <nccl_device.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/socket.h>
#include <sys/stat.h>
#include <sys/un.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

namespace {

constexpr int kMaxRanks = 16;
constexpr size_t kStage = 8u << 20;  // staging bytes per rank and chunk
constexpr char kMagic[8] = {'M', 'O', 'A', 'S', 'H', 'I', 'M', 0};

struct Slot {
  int64_t v[8];
};

struct Shared {
  std::atomic<uint32_t> arrived;
  std::atomic<uint32_t> gen;
  uint32_t pad[14];
  Slot slot[kMaxRanks];
  // followed by nranks * kStage bytes of staging
};

size_t shared_bytes(int nranks) { return sizeof(Shared) + (size_t)nranks * kStage; }

}  // namespace

struct ncclComm {
  std::string name;   // rendezvous name (unique per communicator)
  std::string label;  // for the log: "world", "world/s0c1", ...
  int nranks = 0, rank = 0, device = 0;
  int max_ctas = -1;
  int nsplits = 0;
  Shared* sh = nullptr;
  size_t sh_bytes = 0;
  int listen_fd = -1;
  char* stage(int r) { return reinterpret_cast<char*>(sh + 1) + (size_t)r * kStage; }
};

namespace {

std::mutex g_mu;
int g_group_depth = 0;

double now_s() {
  timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + 1e-9 * t.tv_nsec;
}

double timeout_s() {
  const char* e = getenv("MOA_NCCL_SHIM_TIMEOUT");
  return e ? atof(e) : 300.0;
}

void warn(const char* what) { fprintf(stderr, "[moa_nccl_shim] %s\n", what); }

bool barrier(ncclComm* c) {
  if (c->nranks == 1) return true;
  const uint32_t g = c->sh->gen.load();
  if (c->sh->arrived.fetch_add(1) + 1 == (uint32_t)c->nranks) {
    c->sh->arrived.store(0);
    c->sh->gen.fetch_add(1);
    return true;
  }
  const double t0 = now_s(), lim = timeout_s();
  unsigned spins = 0;
  while (c->sh->gen.load() == g) {
    if (++spins > 1000) {
      usleep(20);
      if ((spins & 1023) == 0 && now_s() - t0 > lim) {
        warn(("barrier timeout on " + c->label).c_str());
        return false;
      }
    }
  }
  return true;
}

size_t esize(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
    default: return 0;
  }
}

void log_op(ncclComm* c, const char* op, int root, size_t count, ncclDataType_t t) {
  const char* path = getenv("MOA_NCCL_SHIM_LOG");
  if (!path) return;
  FILE* f = fopen(path, "a");
  if (!f) return;
  fprintf(f, "{\"op\": \"%s\", \"comm\": \"%s\", \"nranks\": %d, \"rank\": %d, \"root\": %d, \"count\": %zu, "
             "\"esize\": %zu, \"group\": %d, \"max_ctas\": %d}\n",
          op, c->label.c_str(), c->nranks, c->rank, root, count, esize(t), g_group_depth, c->max_ctas);
  fclose(f);
}

bool cuda_ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return true;
  fprintf(stderr, "[moa_nccl_shim] %s: %s\n", what, cudaGetErrorString(e));
  return false;
}

bool copy(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return true;
  return cuda_ok(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s), "cudaMemcpyAsync") &&
         cuda_ok(cudaStreamSynchronize(s), "cudaStreamSynchronize");
}

std::string sock_name(const std::string& comm, int rank) {
  return std::string("moa-nccl-shim-") + comm + "-" + std::to_string(rank);
}

int listen_on(const std::string& name) {
  int fd = socket(AF_UNIX, SOCK_STREAM, 0);
  if (fd < 0) return -1;
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  const size_t n = std::min(name.size(), sizeof(a.sun_path) - 2);
  memcpy(a.sun_path + 1, name.data(), n);  // abstract namespace
  if (bind(fd, (sockaddr*)&a, (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n)) != 0 || listen(fd, 64) != 0) {
    close(fd);
    return -1;
  }
  return fd;
}

bool send_fd(const std::string& name, int from, int fd) {
  int s = socket(AF_UNIX, SOCK_STREAM, 0);
  if (s < 0) return false;
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  const size_t n = std::min(name.size(), sizeof(a.sun_path) - 2);
  memcpy(a.sun_path + 1, name.data(), n);
  if (connect(s, (sockaddr*)&a, (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n)) != 0) {
    close(s);
    return false;
  }
  char cbuf[CMSG_SPACE(sizeof(int))] = {};
  iovec io{&from, sizeof(from)};
  msghdr m{};
  m.msg_iov = &io;
  m.msg_iovlen = 1;
  m.msg_control = cbuf;
  m.msg_controllen = sizeof(cbuf);
  cmsghdr* cm = CMSG_FIRSTHDR(&m);
  cm->cmsg_level = SOL_SOCKET;
  cm->cmsg_type = SCM_RIGHTS;
  cm->cmsg_len = CMSG_LEN(sizeof(int));
  memcpy(CMSG_DATA(cm), &fd, sizeof(int));
  const bool ok = sendmsg(s, &m, 0) == (ssize_t)sizeof(from);
  close(s);
  return ok;
}

bool recv_fd(int lfd, int* from, int* fd) {
  int s = accept(lfd, nullptr, nullptr);
  if (s < 0) return false;
  char cbuf[CMSG_SPACE(sizeof(int))] = {};
  iovec io{from, sizeof(*from)};
  msghdr m{};
  m.msg_iov = &io;
  m.msg_iovlen = 1;
  m.msg_control = cbuf;
  m.msg_controllen = sizeof(cbuf);
  const bool ok = recvmsg(s, &m, 0) == (ssize_t)sizeof(*from);
  cmsghdr* cm = CMSG_FIRSTHDR(&m);
  close(s);
  if (!ok || !cm || cm->cmsg_type != SCM_RIGHTS) return false;
  memcpy(fd, CMSG_DATA(cm), sizeof(int));
  return true;
}

ncclResult_t comm_open(ncclComm* c, const std::string& name, int nranks, int rank) {
  c->name = name;
  c->nranks = nranks;
  c->rank = rank;
  cudaGetDevice(&c->device);
  c->sh_bytes = shared_bytes(nranks);
  const std::string path = "/tmp/moa_nccl_shim_" + name;
  int fd = open(path.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0) return ncclSystemError;
  if (ftruncate(fd, (off_t)c->sh_bytes) != 0) {
    close(fd);
    return ncclSystemError;
  }
  void* p = mmap(nullptr, c->sh_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return ncclSystemError;
  c->sh = static_cast<Shared*>(p);
  c->listen_fd = listen_on(sock_name(name, rank));
  if (c->listen_fd < 0) return ncclSystemError;
  if (!barrier(c)) return ncclSystemError;  // everyone has mapped the file and listens
  if (rank == 0) unlink(path.c_str());
  return ncclSuccess;
}

// Windows and VMM allocations.
struct Alloc {
  void* ptr;
  size_t size;
  CUmemGenericAllocationHandle h;
};
std::vector<Alloc> g_allocs;

struct ShimWindow {
  ncclComm* comm;
  CUdeviceptr flat;
  size_t stride, mapped;
  std::vector<CUmemGenericAllocationHandle> imported;  // peers' handles (own entry: 0)
  void* dev_struct;
};

bool cu_ok(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return true;
  const char* s = nullptr;
  cuGetErrorString(r, &s);
  fprintf(stderr, "[moa_nccl_shim] %s: %s\n", what, s ? s : "?");
  return false;
}

}  // namespace

extern "C" {

const char* ncclGetErrorString(ncclResult_t r) {
  switch (r) {
    case ncclSuccess: return "no error (moa_nccl_shim)";
    case ncclUnhandledCudaError: return "unhandled cuda error (moa_nccl_shim)";
    case ncclSystemError: return "system error / barrier timeout (moa_nccl_shim)";
    case ncclInvalidArgument: return "invalid argument (moa_nccl_shim)";
    default: return "error (moa_nccl_shim)";
  }
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  memset(id, 0, sizeof(*id));
  memcpy(id->internal, kMagic, sizeof(kMagic));
  unsigned char r[8];
  FILE* f = fopen("/dev/urandom", "rb");
  if (!f || fread(r, 1, 8, f) != 8) {
    if (f) fclose(f);
    return ncclSystemError;
  }
  fclose(f);
  for (int i = 0; i < 8; ++i) snprintf(id->internal + 8 + 2 * i, 3, "%02x", r[i]);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  if (memcmp(id.internal, kMagic, sizeof(kMagic)) != 0 || nranks < 1 || nranks > kMaxRanks || rank < 0 ||
      rank >= nranks)
    return ncclInvalidArgument;
  cudaFree(nullptr);  // make the runtime's primary context current for the driver-API calls
  auto* c = new ncclComm;
  c->label = "world";
  ncclResult_t r = comm_open(c, std::string(id.internal + 8, 16), nranks, rank);
  if (r != ncclSuccess) {
    delete c;
    return r;
  }
  *comm = c;
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t c) {
  if (!c) return ncclSuccess;
  if (c->sh) munmap(c->sh, c->sh_bytes);
  if (c->listen_fd >= 0) close(c->listen_fd);
  delete c;
  return ncclSuccess;
}

ncclResult_t ncclCommSplit(ncclComm_t c, int color, int key, ncclComm_t* newcomm, ncclConfig_t* config) {
  std::lock_guard<std::mutex> lk(g_mu);
  Slot& me = c->sh->slot[c->rank];
  me.v[0] = color;
  me.v[1] = key;
  if (!barrier(c)) return ncclSystemError;
  std::vector<std::pair<std::pair<int64_t, int>, int>> members;  // ((key, rank), rank)
  for (int r = 0; r < c->nranks; ++r)
    if (c->sh->slot[r].v[0] == color) members.push_back({{c->sh->slot[r].v[1], r}, r});
  if (!barrier(c)) return ncclSystemError;  // slots may be reused after this
  const int seq = c->nsplits++;
  if (color == NCCL_SPLIT_NOCOLOR) {
    *newcomm = nullptr;
    return ncclSuccess;
  }
  std::sort(members.begin(), members.end());
  int nrank = 0;
  for (size_t i = 0; i < members.size(); ++i)
    if (members[i].second == c->rank) nrank = (int)i;
  auto* n = new ncclComm;
  n->label = c->label + "/s" + std::to_string(seq) + "c" + std::to_string(color);
  if (config && config->maxCTAs != NCCL_CONFIG_UNDEF_INT) n->max_ctas = config->maxCTAs;
  ncclResult_t r = comm_open(n, c->name + "s" + std::to_string(seq) + "c" + std::to_string(color),
                             (int)members.size(), nrank);
  if (r != ncclSuccess) {
    delete n;
    return r;
  }
  *newcomm = n;
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
  ++g_group_depth;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (g_group_depth > 0) --g_group_depth;
  return ncclSuccess;
}

ncclResult_t ncclBroadcast(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype, int root,
                           ncclComm_t c, cudaStream_t stream) {
  const size_t es = esize(datatype);
  if (!c || es == 0 || root < 0 || root >= c->nranks) return ncclInvalidArgument;
  std::lock_guard<std::mutex> lk(g_mu);
  log_op(c, "broadcast", root, count, datatype);
  if (!cuda_ok(cudaStreamSynchronize(stream), "sync")) return ncclUnhandledCudaError;
  const size_t bytes = count * es;
  if (c->nranks == 1 || bytes == 0) {
    if (bytes && sendbuff != recvbuff && !copy(recvbuff, sendbuff, bytes, stream)) return ncclUnhandledCudaError;
    return ncclSuccess;
  }
  for (size_t off = 0; off < bytes; off += kStage) {
    const size_t b = std::min(kStage, bytes - off);
    if (c->rank == root && !copy(c->stage(root), (const char*)sendbuff + off, b, stream)) return ncclUnhandledCudaError;
    if (!barrier(c)) return ncclSystemError;
    if (c->rank != root) {
      if (!copy((char*)recvbuff + off, c->stage(root), b, stream)) return ncclUnhandledCudaError;
    } else if (sendbuff != recvbuff && !copy((char*)recvbuff + off, (const char*)sendbuff + off, b, stream)) {
      return ncclUnhandledCudaError;
    }
    if (!barrier(c)) return ncclSystemError;
  }
  return ncclSuccess;
}

ncclResult_t ncclAllGather(const void* sendbuff, void* recvbuff, size_t sendcount, ncclDataType_t datatype,
                           ncclComm_t c, cudaStream_t stream) {
  const size_t es = esize(datatype);
  if (!c || es == 0) return ncclInvalidArgument;
  std::lock_guard<std::mutex> lk(g_mu);
  log_op(c, "allgather", -1, sendcount, datatype);
  if (!cuda_ok(cudaStreamSynchronize(stream), "sync")) return ncclUnhandledCudaError;
  const size_t bytes = sendcount * es;
  for (size_t off = 0; off < bytes; off += kStage) {
    const size_t b = std::min(kStage, bytes - off);
    if (!copy(c->stage(c->rank), (const char*)sendbuff + off, b, stream)) return ncclUnhandledCudaError;
    if (!barrier(c)) return ncclSystemError;
    for (int r = 0; r < c->nranks; ++r)
      if (!copy((char*)recvbuff + (size_t)r * bytes + off, c->stage(r), b, stream)) return ncclUnhandledCudaError;
    if (!barrier(c)) return ncclSystemError;
  }
  return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype, ncclRedOp_t op,
                           ncclComm_t c, cudaStream_t stream) {
  const size_t es = esize(datatype);
  if (!c || es == 0) return ncclInvalidArgument;
  if (datatype != ncclInt32 && datatype != ncclFloat32 && datatype != ncclFloat64) return ncclInvalidArgument;
  if (op != ncclSum && op != ncclMax && op != ncclMin) return ncclInvalidArgument;
  std::lock_guard<std::mutex> lk(g_mu);
  log_op(c, "allreduce", -1, count, datatype);
  if (!cuda_ok(cudaStreamSynchronize(stream), "sync")) return ncclUnhandledCudaError;
  const size_t bytes = count * es;
  std::vector<char> acc(std::min(kStage, bytes));
  for (size_t off = 0; off < bytes; off += kStage) {
    const size_t b = std::min(kStage, bytes - off), k = b / es;
    if (!copy(c->stage(c->rank), (const char*)sendbuff + off, b, stream)) return ncclUnhandledCudaError;
    if (!barrier(c)) return ncclSystemError;
    memcpy(acc.data(), c->stage(0), b);
    for (int r = 1; r < c->nranks; ++r) {
      const char* src = c->stage(r);
      for (size_t i = 0; i < k; ++i) {
        auto red = [&](auto* a, const auto* x) {
          if (op == ncclSum) a[i] += x[i];
          else if (op == ncclMax) a[i] = std::max(a[i], x[i]);
          else a[i] = std::min(a[i], x[i]);
        };
        if (datatype == ncclInt32) red((int32_t*)acc.data(), (const int32_t*)src);
        else if (datatype == ncclFloat32) red((float*)acc.data(), (const float*)src);
        else red((double*)acc.data(), (const double*)src);
      }
    }
    if (!barrier(c)) return ncclSystemError;  // everyone has read every stage
    if (!copy((char*)recvbuff + off, acc.data(), b, stream)) return ncclUnhandledCudaError;
  }
  return ncclSuccess;
}

ncclResult_t ncclMemAlloc(void** ptr, size_t size) {
  cudaFree(nullptr);
  int dev = 0;
  cudaGetDevice(&dev);
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  if (!cu_ok(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "granularity"))
    return ncclUnhandledCudaError;
  const size_t sz = (size + gran - 1) / gran * gran;
  Alloc a{nullptr, sz, 0};
  CUdeviceptr d = 0;
  if (!cu_ok(cuMemCreate(&a.h, sz, &prop, 0), "cuMemCreate")) return ncclUnhandledCudaError;
  if (!cu_ok(cuMemAddressReserve(&d, sz, gran, 0, 0), "cuMemAddressReserve") ||
      !cu_ok(cuMemMap(d, sz, 0, a.h, 0), "cuMemMap")) {
    cuMemRelease(a.h);
    return ncclUnhandledCudaError;
  }
  CUmemAccessDesc acc{};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (!cu_ok(cuMemSetAccess(d, sz, &acc, 1), "cuMemSetAccess")) return ncclUnhandledCudaError;
  a.ptr = (void*)d;
  std::lock_guard<std::mutex> lk(g_mu);
  g_allocs.push_back(a);
  *ptr = a.ptr;
  return ncclSuccess;
}

ncclResult_t ncclMemFree(void* ptr) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (size_t i = 0; i < g_allocs.size(); ++i)
    if (g_allocs[i].ptr == ptr) {
      cuMemUnmap((CUdeviceptr)ptr, g_allocs[i].size);
      cuMemAddressFree((CUdeviceptr)ptr, g_allocs[i].size);
      cuMemRelease(g_allocs[i].h);
      g_allocs.erase(g_allocs.begin() + (long)i);
      return ncclSuccess;
    }
  return ncclInvalidArgument;
}

ncclResult_t ncclCommWindowRegister(ncclComm_t c, void* buff, size_t size, ncclWindow_t* win, int /*winFlags*/) {
  std::lock_guard<std::mutex> lk(g_mu);
  const Alloc* a = nullptr;
  for (const auto& x : g_allocs)
    if (x.ptr == buff) a = &x;
  if (!a || size > a->size) return ncclInvalidArgument;
  int myfd = -1;
  if (!cu_ok(cuMemExportToShareableHandle(&myfd, a->h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "export"))
    return ncclUnhandledCudaError;
  // every rank's allocation size must agree (symmetric)
  c->sh->slot[c->rank].v[2] = (int64_t)a->size;
  if (!barrier(c)) return ncclSystemError;
  for (int r = 0; r < c->nranks; ++r)
    if (c->sh->slot[r].v[2] != (int64_t)a->size) return ncclInvalidArgument;
  if (!barrier(c)) return ncclSystemError;
  for (int r = 0; r < c->nranks; ++r)
    if (r != c->rank && !send_fd(sock_name(c->name, r), c->rank, myfd)) return ncclSystemError;
  std::vector<int> fds((size_t)c->nranks, -1);
  for (int i = 0; i < c->nranks - 1; ++i) {
    int from = -1, fd = -1;
    if (!recv_fd(c->listen_fd, &from, &fd) || from < 0 || from >= c->nranks) return ncclSystemError;
    fds[(size_t)from] = fd;
  }
  close(myfd);
  auto* w = new ShimWindow;
  w->comm = c;
  w->stride = ((a->size + (1ull << 32) - 1) >> 32) << 32;
  w->mapped = a->size;
  w->imported.assign((size_t)c->nranks, 0);
  if (!cu_ok(cuMemAddressReserve(&w->flat, w->stride * (size_t)c->nranks, 1ull << 21, 0, 0), "reserve flat"))
    return ncclUnhandledCudaError;
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = c->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (int r = 0; r < c->nranks; ++r) {
    CUmemGenericAllocationHandle h = a->h;
    if (r != c->rank) {
      if (!cu_ok(cuMemImportFromShareableHandle(&h, (void*)(intptr_t)fds[(size_t)r],
                                                CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                 "import"))
        return ncclUnhandledCudaError;
      close(fds[(size_t)r]);
      w->imported[(size_t)r] = h;
    }
    const CUdeviceptr at = w->flat + (size_t)r * w->stride;
    if (!cu_ok(cuMemMap(at, a->size, 0, h, 0), "map peer") || !cu_ok(cuMemSetAccess(at, a->size, &acc, 1), "access"))
      return ncclUnhandledCudaError;
  }
  ncclWindow_vidmem host{};
  host.winHost = w;
  host.lsaFlatBase = (char*)w->flat;
  host.lsaRank = c->rank;
  host.worldRank = c->rank;
  host.stride4G = (uint32_t)(w->stride >> 32);
  if (!cuda_ok(cudaMalloc(&w->dev_struct, sizeof(host)), "cudaMalloc(window)") ||
      !cuda_ok(cudaMemcpy(w->dev_struct, &host, sizeof(host), cudaMemcpyHostToDevice), "cudaMemcpy(window)"))
    return ncclUnhandledCudaError;
  if (!barrier(c)) return ncclSystemError;  // every rank has mapped every peer
  *win = static_cast<ncclWindow_t>(w->dev_struct);  // winHost leads back to w
  return ncclSuccess;
}

ncclResult_t ncclCommWindowDeregister(ncclComm_t c, ncclWindow_t win) {
  ncclWindow_vidmem host{};
  if (cudaMemcpy(&host, win, sizeof(host), cudaMemcpyDeviceToHost) != cudaSuccess) return ncclUnhandledCudaError;
  auto* w = static_cast<ShimWindow*>(host.winHost);
  if (!w || w->comm != c) return ncclInvalidArgument;
  cudaDeviceSynchronize();
  barrier(c);  // no peer still stores into our copy
  for (int r = 0; r < c->nranks; ++r) {
    cuMemUnmap(w->flat + (size_t)r * w->stride, w->mapped);
    if (w->imported[(size_t)r]) cuMemRelease(w->imported[(size_t)r]);
  }
  cuMemAddressFree(w->flat, w->stride * (size_t)c->nranks);
  cudaFree(w->dev_struct);
  delete w;
  return ncclSuccess;
}

ncclTeam_t ncclTeamLsa(ncclComm_t c) {
  ncclTeam_t t;
  t.nRanks = c ? c->nranks : 0;
  t.rank = c ? c->rank : 0;
  t.stride = 1;
  return t;
}

}  // extern "C"
