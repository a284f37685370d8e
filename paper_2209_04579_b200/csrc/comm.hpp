// Communicators for sharded execution: one process (or
// thread) per GPU, exchanging device buffers on the context's stream.
//   * NcclComm  - NCCL over NVLink / NVSwitch (libnccl.so.2, bound with
//                 dlopen so the library has no link-time NCCL dependency and
//                 shares the NCCL a host process such as torch already loaded);
//   * LocalComm - ranks that are threads of one process (one or several
//                 devices): device-to-device copies between the ranks'
//                 buffers behind a host barrier. It runs the same sharded
//                 code paths where NCCL cannot (two ranks on one GPU: tests).
#pragma once

#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "tqp_internal.hpp"

namespace tqp {

struct Comm {
  int rank = 0, size = 1;
  virtual ~Comm() = default;
  virtual const char* kind() const = 0;
  // every rank contributes `bytes` at `send` (device); rank r's block lands
  // at recv + r * bytes (device). Ordered on c.stream.
  virtual void allgather(Ctx& c, const void* send, void* recv, size_t bytes) = 0;
  // grouped point-to-point: send[r] (sbytes[r]) to rank r, recv[r]
  // (rbytes[r], the sizes agreed beforehand) from rank r. Ordered on c.stream.
  virtual void alltoallv(Ctx& c, const std::vector<const void*>& send, const std::vector<size_t>& sbytes,
                         const std::vector<void*>& recv, const std::vector<size_t>& rbytes) = 0;
};

// host vector all-gather (through a device bounce buffer): out[r * n + i]
std::vector<long long> allgather_host(Ctx& c, Comm& comm, const std::vector<long long>& mine);

// NCCL unique id (128 bytes) for ncclCommInitRank; throws if NCCL is absent
void nccl_unique_id(void* out128);
std::unique_ptr<Comm> make_nccl_comm(Ctx& c, const void* id128, int nranks, int rank);

// a group of `n` in-process ranks (threads), each used with its own Ctx
std::vector<std::unique_ptr<Comm>> make_local_group(int n);

}  // namespace tqp
