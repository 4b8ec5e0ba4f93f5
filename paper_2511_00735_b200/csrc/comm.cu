// Collectives of the sharded path: NCCL (one process per GPU, NVLink /
// NVSwitch) and a single-process emulation over host threads.
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <algorithm>

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
  void exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                Context* ctx) override {
    if (sends.empty() && recvs.empty()) return;
    double bytes = 0;
    for (const auto& x : sends) bytes += static_cast<double>(x.bytes);
    KernelScope ks(ctx, "nccl_sendrecv", bytes, 0.0);
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    for (const auto& x : sends)
      nccl_check(ncclSend(x.buf, x.bytes, ncclUint8, x.peer, comm, ctx->stream), "ncclSend");
    for (const auto& x : recvs)
      nccl_check(ncclRecv(x.buf, x.bytes, ncclUint8, x.peer, comm, ctx->stream), "ncclRecv");
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
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
__global__ void delta_pack_kernel(double2* pack, const double2* __restrict__ a, int64_t lda,
                                  const double2* __restrict__ base, int64_t ldb, int64_t n) {
  const int c = blockIdx.y;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    pack[c * n + k] = base ? csub(a[c * lda + k], base[c * ldb + k]) : a[c * lda + k];
}
__global__ void delta_unpack_kernel(double2* a, int64_t lda, const double2* __restrict__ base,
                                    int64_t ldb, const double2* __restrict__ pack, int64_t n) {
  const int c = blockIdx.y;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    a[c * lda + k] = base ? cadd(base[c * ldb + k], pack[c * n + k]) : pack[c * n + k];
}
}  // namespace

void exchange_deltas(Context* ctx, DevBuf<double2>& buf, const std::vector<DeltaSeg>& segs) {
  int64_t tot = 0;
  for (const DeltaSeg& sg : segs) tot += sg.n * sg.cols;
  if (!tot) return;
  if (buf.n < static_cast<size_t>(tot)) buf.alloc(tot);
  int64_t at = 0;
  for (const DeltaSeg& sg : segs) {
    if (!sg.n) continue;
    const dim3 grid(static_cast<unsigned>(std::min<int64_t>((sg.n + 255) / 256, 2 * ctx->num_sms)),
                    static_cast<unsigned>(sg.cols));
    delta_pack_kernel<<<grid, 256, 0, ctx->stream>>>(buf.p + at, sg.a, sg.lda, sg.base, sg.ldb, sg.n);
    HPSB_LAUNCHED(ctx);
    at += sg.n * sg.cols;
  }
  ctx->comm->allreduce_sum(buf.p, tot, ctx);
  at = 0;
  for (const DeltaSeg& sg : segs) {
    if (!sg.n) continue;
    const dim3 grid(static_cast<unsigned>(std::min<int64_t>((sg.n + 255) / 256, 2 * ctx->num_sms)),
                    static_cast<unsigned>(sg.cols));
    delta_unpack_kernel<<<grid, 256, 0, ctx->stream>>>(sg.a, sg.lda, sg.base, sg.ldb, buf.p + at, sg.n);
    HPSB_LAUNCHED(ctx);
    at += sg.n * sg.cols;
  }
}

struct LocalGroup {
  int size = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0, generation = 0;
  std::vector<void*> slots;
  std::vector<std::vector<Comm::Xfer>> sends;  // exchange(): published per rank
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
  // Every rank publishes its sends; each receiver copies the matching send
  // of its peer (device to device: the emulated ranks share one GPU).  The
  // k-th receive from peer p pairs with the k-th send from p to this rank.
  void exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                Context* ctx) override {
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    {
      std::lock_guard<std::mutex> lk(grp->mu);
      grp->sends[rank] = sends;
    }
    grp->barrier();
    std::vector<int> taken(size, 0);
    for (const auto& r : recvs) {
      const auto& ps = grp->sends[r.peer];
      int k = 0, seen = 0;
      for (; k < static_cast<int>(ps.size()); ++k)
        if (ps[k].peer == rank && seen++ == taken[r.peer]) break;
      if (k == static_cast<int>(ps.size()) || ps[k].bytes != r.bytes)
        throw std::logic_error("local group: unmatched receive");
      ++taken[r.peer];
      HPSB_CUDA(cudaMemcpyAsync(r.buf, ps[k].buf, r.bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    grp->barrier();  // every receiver has copied: the senders may reuse their buffers
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
  g->sends.assign(size, {});
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
