// Communicators (comm.hpp): NCCL bound at run time, and an in-process group
// of thread ranks for single-GPU tests of the sharded paths.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "comm.hpp"

namespace tqp {

// ---- NCCL --------------------------------------------------------------------
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // the NCCL a host process already loaded (e.g. torch's), else the system's
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);
      if (a.h) break;
    }
    if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) return a;
    auto sym = [&](auto& f, const char* n) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(a.h, n)); };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.AllGather, "ncclAllGather");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.GetErrorString, "ncclGetErrorString");
    return a;
  }();
  if (!api.h || !api.CommInitRank || !api.AllGather || !api.Send || !api.Recv)
    throw Error(TQP_ERR_CUDA, "nccl: libnccl.so.2 is not available");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(TQP_ERR_CUDA, std::string("nccl: ") + what + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
}

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  const char* kind() const override { return "nccl"; }
  void allgather(Ctx& c, const void* send, void* recv, size_t bytes) override {
    nccl_check(nccl().AllGather(send, recv, bytes, ncclUint8, comm, c.stream), "allgather");
  }
  void alltoallv(Ctx& c, const std::vector<const void*>& send, const std::vector<size_t>& sbytes,
                 const std::vector<void*>& recv, const std::vector<size_t>& rbytes) override {
    nccl_check(nccl().GroupStart(), "group start");
    for (int r = 0; r < size; ++r) {
      if (sbytes[r]) nccl_check(nccl().Send(send[r], sbytes[r], ncclUint8, r, comm, c.stream), "send");
      if (rbytes[r]) nccl_check(nccl().Recv(recv[r], rbytes[r], ncclUint8, r, comm, c.stream), "recv");
    }
    nccl_check(nccl().GroupEnd(), "group end");
  }
};

// ---- in-process thread ranks -----------------------------------------------------
struct LocalGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const void*> bufs;                 // allgather: each rank's send buffer
  std::vector<std::vector<const void*>> a2a;     // alltoallv: [src][dst] send buffers
  std::vector<cudaEvent_t> ready;                // each rank's send buffers are complete
  std::vector<int> dev;

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LocalComm final : Comm {
  std::shared_ptr<LocalGroup> g;
  const char* kind() const override { return "local"; }

  void post_ready(Ctx& c) {
    cudaEvent_t e;
    TQP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    TQP_CUDA(cudaEventRecord(e, c.stream));
    g->ready[rank] = e;
    g->dev[rank] = c.device;
  }
  void copy_from(Ctx& c, void* dst, int src_rank, const void* src, size_t bytes) {
    if (!bytes) return;
    TQP_CUDA(cudaStreamWaitEvent(c.stream, g->ready[src_rank], 0));
    if (g->dev[src_rank] == c.device)
      TQP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c.stream));
    else
      TQP_CUDA(cudaMemcpyPeerAsync(dst, c.device, src, g->dev[src_rank], bytes, c.stream));
  }
  void finish(Ctx& c) {
    c.sync();     // my copies are done
    g->barrier();  // everyone's copies are done: send buffers may change
    TQP_CUDA(cudaEventDestroy(g->ready[rank]));
  }
  void allgather(Ctx& c, const void* send, void* recv, size_t bytes) override {
    post_ready(c);
    g->bufs[rank] = send;
    g->barrier();
    for (int r = 0; r < size; ++r) copy_from(c, static_cast<char*>(recv) + r * bytes, r, g->bufs[r], bytes);
    finish(c);
  }
  void alltoallv(Ctx& c, const std::vector<const void*>& send, const std::vector<size_t>& sbytes,
                 const std::vector<void*>& recv, const std::vector<size_t>& rbytes) override {
    (void)sbytes;
    post_ready(c);
    g->a2a[rank] = send;
    g->barrier();
    for (int r = 0; r < size; ++r) copy_from(c, recv[r], r, g->a2a[r][rank], rbytes[r]);
    finish(c);
  }
};

}  // namespace

std::vector<long long> allgather_host(Ctx& c, Comm& comm, const std::vector<long long>& mine) {
  const size_t n = mine.size();
  std::vector<long long> out(n * comm.size);
  if (!n) return out;
  auto buf = c.alloc_bytes(sizeof(long long) * n * (comm.size + 1));
  long long* send = static_cast<long long*>(buf->ptr);
  TQP_CUDA(cudaMemcpyAsync(send, mine.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, c.stream));
  comm.allgather(c, send, send + n, sizeof(long long) * n);
  TQP_CUDA(cudaMemcpyAsync(out.data(), send + n, sizeof(long long) * n * comm.size, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  return out;
}

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "get unique id");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
}

std::unique_ptr<Comm> make_nccl_comm(Ctx& c, const void* id128, int nranks, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(TQP_ERR_ARG, "nccl: bad rank / size");
  auto comm = std::make_unique<NcclComm>();
  comm->rank = rank;
  comm->size = nranks;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  TQP_CUDA(cudaSetDevice(c.device));
  nccl_check(nccl().CommInitRank(&comm->comm, nranks, id, rank), "comm init");
  return comm;
}

std::vector<std::unique_ptr<Comm>> make_local_group(int n) {
  if (n < 1) throw Error(TQP_ERR_ARG, "local comm group: n < 1");
  auto g = std::make_shared<LocalGroup>();
  g->n = n;
  g->bufs.assign(n, nullptr);
  g->a2a.assign(n, {});
  g->ready.assign(n, nullptr);
  g->dev.assign(n, 0);
  std::vector<std::unique_ptr<Comm>> out;
  for (int r = 0; r < n; ++r) {
    auto c = std::make_unique<LocalComm>();
    c->g = g;
    c->rank = r;
    c->size = n;
    out.push_back(std::move(c));
  }
  return out;
}

}  // namespace tqp
