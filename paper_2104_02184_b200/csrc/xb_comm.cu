// xb_comm.cu -- collectives of a row-sharded tile, behind the
// C ABI (include/xbtile.h: xb_comm_*).
//
// A logical d_out x d_in tile is row-partitioned over P ranks (one process or
// host thread per GPU).  The data path needs exactly three reductions, all
// enqueued on the tile's stream, none waited on by the host:
//   * update  : all-reduce(max) of the B per-sample max|d| before translate
//               (proj/src/pulsed.cpp:34-51 uses the global max);
//   * forward : all-reduce(max) of the B bound-management saturation flags
//               before every re-issue, so every shard re-issues exactly the
//               samples the unsharded tile would;
//   * backward: all-reduce(max) of max|d| (the DAC's abs-max), then
//               all-reduce(sum) of the shards' column sums W_r^T d~_r; output
//               noise, ADC and alpha act after the sum (proj/src/io.cpp:143-146).
//
// Two implementations:
//   NcclCollective  -- NCCL over NVLink/NVSwitch (ncclCommInitRank from a
//                      unique id exchanged out of band).  NCCL is loaded with
//                      dlopen (XB_NCCL_LIB, else libnccl.so.2: the copy a host
//                      process such as PyTorch already mapped, or the system
//                      one), so libxbtile has no link-time NCCL dependency.
//   LocalCollective -- an in-process group of P shard handles, each driven by
//                      its own host thread (any devices, including P shards on
//                      one device: the test harness of the sharded path).  A
//                      reduction is a host rendezvous plus stream-ordered
//                      device work: every rank waits (cudaStreamWaitEvent) for
//                      all ranks' inputs, reduces ITS slice of the elements
//                      over every member's buffer in rank order and writes the
//                      result into every member's buffer over peer memory
//                      (reduce-scatter + all-gather in one kernel), then waits
//                      for every rank's slice.  No kernel ever spins on another.
#include <dlfcn.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <utility>
#include <vector>

#include <nccl.h>

#include "xb_internal.h"

namespace xb {

namespace {

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                             ncclComm_t, cudaStream_t) = nullptr;
  const char *(*error_string)(ncclResult_t) = nullptr;
  std::string load_error;
};

const NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *env = getenv("XB_NCCL_LIB");
    void *h = nullptr;
    for (const char *name : {env, "libnccl.so.2", "libnccl.so"}) {
      if (!name) continue;
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      api.load_error = std::string("NCCL not loadable (") + (dlerror() ? dlerror() : "?") +
                       "); set XB_NCCL_LIB";
      return;
    }
    api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
    api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
    api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
    api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
    api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
    if (!api.get_unique_id || !api.comm_init_rank || !api.comm_destroy || !api.all_reduce ||
        !api.error_string)
      api.load_error = "NCCL library lacks a required symbol";
  });
  if (!api.load_error.empty()) raise(api.load_error);
  return api;
}

void nccl_check(ncclResult_t r, const char *what) {
  if (r != ncclSuccess) raise(std::string("NCCL error: ") + nccl().error_string(r) + " (" + what + ")");
}

struct NcclCollective : Collective {
  ncclComm_t comm = nullptr;
  int n = 1, r = 0;
  ~NcclCollective() override {
    if (comm) nccl().comm_destroy(comm);
  }
  int size() const override { return n; }
  int rank() const override { return r; }
  void reduce(void *buf, size_t cnt, ncclDataType_t ty, ncclRedOp_t op, cudaStream_t s) {
    if (cnt == 0) return;
    nccl_check(nccl().all_reduce(buf, buf, cnt, ty, op, comm, s), "ncclAllReduce");
  }
  void allreduce_max_i32(int *b, size_t c, cudaStream_t s) override { reduce(b, c, ncclInt32, ncclMax, s); }
  void allreduce_max_f32(float *b, size_t c, cudaStream_t s) override { reduce(b, c, ncclFloat32, ncclMax, s); }
  void allreduce_sum_f32(float *b, size_t c, cudaStream_t s) override { reduce(b, c, ncclFloat32, ncclSum, s); }
};

// ------------------------------------------------------------------ loopback
enum class Op { max_i32, max_f32, sum_f32 };

// Elements [lo, hi) -- this rank's slice -- reduced over every member's
// buffer in rank order and written back into every member's buffer: a
// reduce-scatter and an all-gather in one pass over peer memory.  Each rank
// touches only its own slice of every buffer, so the P kernels never
// conflict; every element is read and written once per member.
template <class T, bool MAX>
__global__ void reduce_slice_kernel(T *const *bufs, int P, size_t lo, size_t hi) {
  for (size_t i = lo + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < hi;
       i += (size_t)gridDim.x * blockDim.x) {
    T v = bufs[0][i];
    for (int q = 1; q < P; ++q) {
      const T x = bufs[q][i];
      v = MAX ? (x > v ? x : v) : v + x;
    }
    for (int q = 0; q < P; ++q) bufs[q][i] = v;
  }
}

struct LocalGroup {
  int P = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<void *> bufs;
  std::vector<int> devs; // each member's device once bound (-1 before)
  std::vector<cudaEvent_t> ready, done;
  ~LocalGroup() {
    for (cudaEvent_t e : ready)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : done)
      if (e) cudaEventDestroy(e);
  }

  // host barrier; `publish` runs under the lock before arriving
  template <class F> void barrier(F &&publish) {
    std::unique_lock<std::mutex> lk(m);
    publish();
    const uint64_t g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LocalCollective : Collective {
  std::shared_ptr<LocalGroup> g;
  int r = 0;
  Scratch ptrs;
  // members on other devices: each rank's reduction kernel reads every
  // member's buffer directly, so peer access is enabled both ways when a
  // member binds (before any collective: a failure here cannot strand peers
  // at a rendezvous)
  void bind(int device) override {
    std::lock_guard<std::mutex> lk(g->m);
    for (int q = 0; q < g->P; ++q) {
      const int other = g->devs[q];
      if (q == r || other < 0 || other == device) continue;
      for (const auto &[from, to] : {std::pair<int, int>{device, other}, {other, device}}) {
        int can = 0;
        XB_CUDA(cudaDeviceCanAccessPeer(&can, from, to));
        if (!can)
          raise("comm: loopback group members on devices " + std::to_string(from) + " and " +
                std::to_string(to) + " without peer access; use an NCCL communicator");
        DevScope ds(from);
        const cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled)
          cudaGetLastError();
        else
          XB_CUDA(e);
      }
    }
    g->devs[r] = device;
  }
  int size() const override { return g->P; }
  int rank() const override { return r; }

  void reduce(void *buf, size_t n, size_t elem, Op op, cudaStream_t s) {
    if (n == 0 || g->P == 1) return;
    LocalGroup &G = *g;
    XB_CUDA(cudaEventRecord(G.ready[r], s));
    G.barrier([&] { G.bufs[r] = buf; });
    // every rank's input is enqueued: wait for them in stream order, then
    // reduce this rank's slice into every buffer
    for (int q = 0; q < G.P; ++q)
      if (q != r) XB_CUDA(cudaStreamWaitEvent(s, G.ready[q], 0));
    const size_t lo = n * (size_t)r / (size_t)G.P, hi = n * (size_t)(r + 1) / (size_t)G.P;
    if (hi > lo) {
      void **dptr = (void **)ptrs.get(sizeof(void *) * G.P);
      XB_CUDA(cudaMemcpyAsync(dptr, G.bufs.data(), sizeof(void *) * G.P, cudaMemcpyHostToDevice,
                              s));
      const int blocks = (int)std::min<size_t>((hi - lo + 255) / 256, 1024);
      switch (op) {
      case Op::max_i32:
        reduce_slice_kernel<int, true><<<blocks, 256, 0, s>>>((int *const *)dptr, G.P, lo, hi);
        break;
      case Op::max_f32:
        reduce_slice_kernel<float, true><<<blocks, 256, 0, s>>>((float *const *)dptr, G.P, lo, hi);
        break;
      case Op::sum_f32:
        reduce_slice_kernel<float, false><<<blocks, 256, 0, s>>>((float *const *)dptr, G.P, lo, hi);
        break;
      }
      count_launch();
      XB_CUDA(cudaGetLastError());
    }
    (void)elem;
    XB_CUDA(cudaEventRecord(G.done[r], s));
    G.barrier([] {}); // every rank has enqueued its slice
    for (int q = 0; q < G.P; ++q)
      if (q != r) XB_CUDA(cudaStreamWaitEvent(s, G.done[q], 0));
    // (the pointer table of the next call must not be overwritten before the
    // kernel above has read it: the stream order covers this rank; the
    // barrier at the next call's start covers the others)
  }
  void allreduce_max_i32(int *b, size_t n, cudaStream_t s) override { reduce(b, n, 4, Op::max_i32, s); }
  void allreduce_max_f32(float *b, size_t n, cudaStream_t s) override { reduce(b, n, 4, Op::max_f32, s); }
  void allreduce_sum_f32(float *b, size_t n, cudaStream_t s) override { reduce(b, n, 4, Op::sum_f32, s); }
  ~LocalCollective() override { ptrs.release(); }
};

} // namespace
} // namespace xb

using namespace xb;

struct xb_comm {
  std::unique_ptr<Collective> c;
};

extern "C" {

int xb_comm_unique_id(uint8_t *id) {
  return xb_guard([&] {
    ncclUniqueId u;
    nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
    static_assert(sizeof(u) == XB_COMM_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id, &u, sizeof(u));
  });
}

int xb_comm_create(const uint8_t *id, int nranks, int rank, xb_comm **out) {
  return xb_guard([&] {
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) raise("comm: need 0 <= rank < nranks");
    auto c = std::make_unique<NcclCollective>();
    c->n = nranks;
    c->r = rank;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    nccl_check(nccl().comm_init_rank(&c->comm, nranks, u, rank), "ncclCommInitRank");
    auto h = std::make_unique<xb_comm>();
    h->c = std::move(c);
    *out = h.release();
  });
}

int xb_comm_create_local(int nranks, xb_comm **out) {
  return xb_guard([&] {
    if (nranks < 1) raise("comm: nranks must be >= 1");
    auto g = std::make_shared<LocalGroup>();
    g->P = nranks;
    g->bufs.assign(nranks, nullptr);
    g->devs.assign(nranks, -1);
    g->ready.assign(nranks, nullptr);
    g->done.assign(nranks, nullptr);
    for (int r = 0; r < nranks; ++r) {
      XB_CUDA(cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming));
      XB_CUDA(cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming));
    }
    for (int r = 0; r < nranks; ++r) {
      auto c = std::make_unique<LocalCollective>();
      c->g = g;
      c->r = r;
      out[r] = new xb_comm{std::move(c)};
    }
  });
}

int xb_comm_destroy(xb_comm *c) {
  return xb_guard([&] { delete c; });
}

int xb_comm_size(const xb_comm *c) { return c->c->size(); }
int xb_comm_rank(const xb_comm *c) { return c->c->rank(); }

} // extern "C"

namespace xb {
Collective *comm_of(xb_comm *c) { return c ? c->c.get() : nullptr; }
} // namespace xb
