// comm.h — collectives used by the a9 merge (internal).  Two transports:
//   * NCCL (production): ncclAllReduce / ncclAllGather on the caller's stream, batched in one
//     ncclGroupStart/End per call;
//   * local (tests): ranks are threads of one process on one device; buffers are exchanged
//     through host memory with a barrier, reduced in rank order.  It runs the same merge code
//     in reduce.cu / stats.cu as NCCL does, so multi-rank merges are testable on one GPU.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "lscat.h"

struct lscat_ctx;

namespace lscat {

enum class DT { U32, U64 };
enum class Op { Sum, Min, Max };

struct AllReduceReq {
  void* buf;      // device, reduced in place
  size_t count;   // elements
  DT dt;
  Op op;
};

class Comm {
 public:
  virtual ~Comm() = default;
  virtual lscat_status allreduce(lscat_ctx* ctx, const std::vector<AllReduceReq>& reqs, cudaStream_t s) = 0;
  // recv = concatenation over ranks of `count` elements of `send` (device buffers)
  virtual lscat_status allgather(lscat_ctx* ctx, const void* send, void* recv, size_t count, DT dt,
                                 cudaStream_t s) = 0;
};

Comm* make_nccl_comm(void* nccl_comm);                                   // takes ownership
Comm* make_local_comm(const char* name, int rank, int world);            // test transport

}  // namespace lscat
