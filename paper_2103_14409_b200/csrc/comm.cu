// comm.cu — NCCL and local (thread) transports of the a9 merge collectives.
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "comm.h"
#include "common.h"

namespace lscat {
namespace {

ncclDataType_t nccl_dt(DT d) { return d == DT::U32 ? ncclUint32 : ncclUint64; }
ncclRedOp_t nccl_op(Op o) { return o == Op::Sum ? ncclSum : (o == Op::Min ? ncclMin : ncclMax); }
size_t dt_size(DT d) { return d == DT::U32 ? 4 : 8; }

class NcclComm : public Comm {
 public:
  explicit NcclComm(ncclComm_t c) : c_(c) {}
  ~NcclComm() override {
    if (c_) ncclCommDestroy(c_);
  }
  lscat_status allreduce(lscat_ctx* ctx, const std::vector<AllReduceReq>& reqs, cudaStream_t s) override {
    ncclResult_t r = ncclGroupStart();
    for (const auto& q : reqs)
      if (r == ncclSuccess && q.count) r = ncclAllReduce(q.buf, q.buf, q.count, nccl_dt(q.dt), nccl_op(q.op), c_, s);
    ncclResult_t r2 = ncclGroupEnd();
    if (r == ncclSuccess) r = r2;
    if (r != ncclSuccess) return fail(ctx, LSCAT_ERR_NCCL, "ncclAllReduce: %s", ncclGetErrorString(r));
    return LSCAT_OK;
  }
  lscat_status allgather(lscat_ctx* ctx, const void* send, void* recv, size_t count, DT dt,
                         cudaStream_t s) override {
    ncclResult_t r = ncclAllGather(send, recv, count, nccl_dt(dt), c_, s);
    if (r != ncclSuccess) return fail(ctx, LSCAT_ERR_NCCL, "ncclAllGather: %s", ncclGetErrorString(r));
    return LSCAT_OK;
  }

 private:
  ncclComm_t c_;
};

// ---- local transport: a process-wide rendezvous per group name
struct LocalGroup {
  int world = 0;
  std::mutex m;
  std::condition_variable cv;
  uint64_t gen = 0;
  int arrived = 0;
  std::vector<std::vector<uint8_t>> slot;

  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

std::mutex g_groups_m;
std::map<std::string, std::shared_ptr<LocalGroup>> g_groups;

template <typename T>
void reduce_into(T* acc, const T* x, size_t n, Op op) {
  for (size_t i = 0; i < n; i++) {
    if (op == Op::Sum) acc[i] += x[i];
    else if (op == Op::Min) acc[i] = std::min(acc[i], x[i]);
    else acc[i] = std::max(acc[i], x[i]);
  }
}

class LocalComm : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalGroup> g, int rank) : g_(std::move(g)), rank_(rank) {}

  lscat_status allreduce(lscat_ctx* ctx, const std::vector<AllReduceReq>& reqs, cudaStream_t s) override {
    for (const auto& q : reqs) {
      const size_t bytes = q.count * dt_size(q.dt);
      std::vector<uint8_t>& mine = g_->slot[rank_];
      mine.resize(bytes);
      if (bytes) {
        LSCAT_CUDA(ctx, cudaMemcpyAsync(mine.data(), q.buf, bytes, cudaMemcpyDeviceToHost, s));
        LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
      }
      g_->barrier();
      std::vector<uint8_t> acc(g_->slot[0]);
      for (int r = 1; r < g_->world; r++) {
        if (q.dt == DT::U32)
          reduce_into((uint32_t*)acc.data(), (const uint32_t*)g_->slot[r].data(), q.count, q.op);
        else
          reduce_into((uint64_t*)acc.data(), (const uint64_t*)g_->slot[r].data(), q.count, q.op);
      }
      g_->barrier();  // everyone has read every slot
      if (bytes) {
        LSCAT_CUDA(ctx, cudaMemcpyAsync(q.buf, acc.data(), bytes, cudaMemcpyHostToDevice, s));
        LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
      }
    }
    return LSCAT_OK;
  }
  lscat_status allgather(lscat_ctx* ctx, const void* send, void* recv, size_t count, DT dt,
                         cudaStream_t s) override {
    const size_t bytes = count * dt_size(dt);
    std::vector<uint8_t>& mine = g_->slot[rank_];
    mine.resize(bytes);
    if (bytes) {
      LSCAT_CUDA(ctx, cudaMemcpyAsync(mine.data(), send, bytes, cudaMemcpyDeviceToHost, s));
      LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
    }
    g_->barrier();
    std::vector<uint8_t> all(bytes * g_->world);
    for (int r = 0; r < g_->world; r++)
      if (bytes) memcpy(all.data() + r * bytes, g_->slot[r].data(), bytes);
    g_->barrier();
    if (bytes) {
      LSCAT_CUDA(ctx, cudaMemcpyAsync(recv, all.data(), all.size(), cudaMemcpyHostToDevice, s));
      LSCAT_CUDA(ctx, cudaStreamSynchronize(s));
    }
    return LSCAT_OK;
  }

 private:
  std::shared_ptr<LocalGroup> g_;
  int rank_;
};

}  // namespace

Comm* make_nccl_comm(void* c) { return new NcclComm((ncclComm_t)c); }

Comm* make_local_comm(const char* name, int rank, int world) {
  std::lock_guard<std::mutex> lk(g_groups_m);
  auto& g = g_groups[name];
  if (!g || g->world != world) {
    g = std::make_shared<LocalGroup>();
    g->world = world;
    g->slot.resize(world);
  }
  return new LocalComm(g, rank);
}

}  // namespace lscat
