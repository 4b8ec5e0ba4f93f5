// Collectives of the sharded path: NCCL (one process per GPU, NVLink /
// NVSwitch) and a single-process emulation over host threads.
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>

#include "device.cuh"
#include "internal.hpp"

namespace hpsb {

namespace {
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string("NCCL error: ") + ncclGetErrorString(r) + " in " + what);
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) ncclCommDestroy(comm);
  }
  void allreduce_sum(double2* buf, size_t n, Context* ctx) override {
    KernelScope ks(ctx, "nccl_allreduce", 16.0 * n, 0.0);
    nccl_check(ncclAllReduce(buf, buf, 2 * n, ncclFloat64, ncclSum, comm, ctx->stream),
               "ncclAllReduce");
  }
  void broadcast(void* buf, size_t bytes, int root, Context* ctx) override {
    KernelScope ks(ctx, "nccl_broadcast", static_cast<double>(bytes), 0.0);
    nccl_check(ncclBroadcast(buf, buf, bytes, ncclUint8, root, comm, ctx->stream), "ncclBroadcast");
  }
};

// out[i] = sum_q in[q][i] in fixed rank order (identical on every rank)
__global__ void sum_ranks_kernel(double2* const* in, int nr, double2* out, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    double2 s = in[0][i];
    for (int q = 1; q < nr; ++q) s = cadd(s, in[q][i]);
    out[i] = s;
  }
}
}  // namespace

struct LocalGroup {
  int size = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0, generation = 0;
  std::vector<void*> slots;
  bool broken = false;
  // A rank that fails (throws) before a collective would leave the others
  // waiting: the wait is bounded and a timed-out group stays broken so every
  // rank reports the failure instead of hanging.
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) throw std::runtime_error("local group: a rank failed");
    const int gen = generation;
    if (++arrived == size) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != gen; })) {
      broken = true;
      cv.notify_all();
      throw std::runtime_error("local group: collective timed out (another rank failed?)");
    }
    if (broken) throw std::runtime_error("local group: a rank failed");
  }
};

namespace {
struct ThreadComm : Comm {
  std::shared_ptr<LocalGroup> grp;
  DevBuf<double2> tmp;
  DevBuf<double2*> ptrs;
  void allreduce_sum(double2* buf, size_t n, Context* ctx) override {
    KernelScope ks(ctx, "local_allreduce", 16.0 * n, 0.0);
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    grp->slots[rank] = buf;
    grp->barrier();
    std::vector<double2*> p(size);
    for (int q = 0; q < size; ++q) p[q] = static_cast<double2*>(grp->slots[q]);
    if (tmp.n < n) tmp.alloc(n);
    ptrs.upload(p, ctx->stream);
    sum_ranks_kernel<<<296, 256, 0, ctx->stream>>>(ptrs.p, size, tmp.p, n);
    HPSB_LAUNCHED(ctx);
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    grp->barrier();  // every rank has read every buffer
    HPSB_CUDA(cudaMemcpyAsync(buf, tmp.p, n * sizeof(double2), cudaMemcpyDeviceToDevice,
                              ctx->stream));
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  void broadcast(void* buf, size_t bytes, int root, Context* ctx) override {
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    grp->slots[rank] = buf;
    grp->barrier();
    if (rank != root)
      HPSB_CUDA(cudaMemcpyAsync(buf, grp->slots[root], bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    grp->barrier();
  }
};
}  // namespace

void nccl_unique_id(unsigned char id[128]) {
  ncclUniqueId u;
  nccl_check(ncclGetUniqueId(&u), "ncclGetUniqueId");
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
}

std::unique_ptr<Comm> make_nccl_comm(const unsigned char id[128], int rank, int size, int device) {
  auto c = std::make_unique<NcclComm>();
  c->rank = rank, c->size = size;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  HPSB_CUDA(cudaSetDevice(device));
  nccl_check(ncclCommInitRank(&c->comm, size, u, rank), "ncclCommInitRank");
  return c;
}

std::shared_ptr<LocalGroup> make_local_group(int size) {
  if (size < 1) throw InvalidArgument("local group: size must be >= 1");
  auto g = std::make_shared<LocalGroup>();
  g->size = size;
  g->slots.assign(size, nullptr);
  return g;
}

std::unique_ptr<Comm> make_thread_comm(std::shared_ptr<LocalGroup> group, int rank) {
  if (rank < 0 || rank >= group->size) throw InvalidArgument("local group: rank out of range");
  auto c = std::make_unique<ThreadComm>();
  c->rank = rank, c->size = group->size;
  c->grp = std::move(group);
  return c;
}

}  // namespace hpsb
