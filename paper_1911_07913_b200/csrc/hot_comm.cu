// Collectives of the slab-sharded step (hot_comm.h): a host-staged transport over caller
// callbacks, an NCCL transport (libnccl.so.2 resolved at run time, so the library has no link
// dependency on NCCL and single-GPU users never load it), and the slab planner.
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "hot_comm.h"

namespace hotb200 {

namespace {

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("comm: ") + what + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ host-staged transport
/// Stages the ranges through pinned host memory and calls the caller's collectives.  Used by
/// the multi-process tests (gloo on one GPU) and by any host transport.
struct HostComm final : Comm {
  hot_comm_host ops;
  unsigned char* host = nullptr;
  size_t cap = 0;

  explicit HostComm(const hot_comm_host& o) : ops(o) {
    rank = o.rank;
    size = o.size;
    if (size < 1 || rank < 0 || rank >= size) throw std::invalid_argument("hot_set_comm_host: bad rank/size");
    if (size > 1 && (!o.allgather_ranges || !o.halo || !o.allreduce_max_i32))
      throw std::invalid_argument("hot_set_comm_host: every collective callback is required");
  }
  ~HostComm() override {
    if (host) cudaFreeHost(host);
  }
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (host) cudaFreeHost(host);
    host = nullptr;
    cap = 0;
    cuda_ok(cudaMallocHost(&host, bytes + (bytes >> 2) + 4096), "pinned staging");
    cap = bytes + (bytes >> 2) + 4096;
  }
  void d2h(void* d, long long a, long long b, cudaStream_t s) {
    if (b > a) cuda_ok(cudaMemcpyAsync(host + a, (char*)d + a, b - a, cudaMemcpyDeviceToHost, s), "d2h");
  }
  void h2d(void* d, long long a, long long b, cudaStream_t s) {
    if (b > a) cuda_ok(cudaMemcpyAsync((char*)d + a, host + a, b - a, cudaMemcpyHostToDevice, s), "h2d");
  }
  void allgather_ranges(void* d, const std::vector<long long>& off, cudaStream_t s) override {
    ++gathers;
    if (ops.device_buffers) {
      cuda_ok(cudaStreamSynchronize(s), "sync");
      if (ops.allgather_ranges(ops.user, d, off.data()) != 0) throw std::runtime_error("comm: allgather_ranges failed");
      return;
    }
    ensure(off[size]);
    d2h(d, off[rank], off[rank + 1], s);
    cuda_ok(cudaStreamSynchronize(s), "sync");
    if (ops.allgather_ranges(ops.user, host, off.data()) != 0) throw std::runtime_error("comm: allgather_ranges failed");
    for (int r = 0; r < size; ++r)
      if (r != rank) h2d(d, off[r], off[r + 1], s);
  }
  void halo(void* d, const std::vector<long long>& e, cudaStream_t s) override {
    ++halos;
    if (ops.device_buffers) {
      cuda_ok(cudaStreamSynchronize(s), "sync");
      if (ops.halo(ops.user, d, e.data()) != 0) throw std::runtime_error("comm: halo failed");
      return;
    }
    long long top = 0;
    for (long long v : e) top = v > top ? v : top;
    ensure(top);
    d2h(d, e[4 * rank], e[4 * rank + 1], s);
    d2h(d, e[4 * rank + 2], e[4 * rank + 3], s);
    cuda_ok(cudaStreamSynchronize(s), "sync");
    if (ops.halo(ops.user, host, e.data()) != 0) throw std::runtime_error("comm: halo failed");
    if (rank > 0) h2d(d, e[4 * (rank - 1) + 2], e[4 * (rank - 1) + 3], s);
    if (rank + 1 < size) h2d(d, e[4 * (rank + 1)], e[4 * (rank + 1) + 1], s);
  }
  void allreduce_max(int* v, int n, cudaStream_t s) override {
    (void)s;
    if (ops.allreduce_max_i32(ops.user, v, n) != 0) throw std::runtime_error("comm: allreduce_max failed");
  }
};

// ------------------------------------------------------------------ NCCL transport
struct NcclApi {
  void* so = nullptr;
  decltype(&::ncclGetUniqueId) get_id = nullptr;
  decltype(&::ncclCommInitRank) init = nullptr;
  decltype(&::ncclCommDestroy) destroy = nullptr;
  decltype(&::ncclGroupStart) gstart = nullptr;
  decltype(&::ncclGroupEnd) gend = nullptr;
  decltype(&::ncclBroadcast) bcast = nullptr;
  decltype(&::ncclSend) send = nullptr;
  decltype(&::ncclRecv) recv = nullptr;
  decltype(&::ncclAllReduce) allreduce = nullptr;
  decltype(&::ncclGetErrorString) errstr = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    const char* env = std::getenv("HOT_NCCL_LIB");
    // torch.distributed has normally loaded libnccl.so.2 already: dlopen then returns that copy
    a.so = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.so) return a;
#define HOT_NCCL_SYM(field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(a.so, name))
    HOT_NCCL_SYM(get_id, "ncclGetUniqueId");
    HOT_NCCL_SYM(init, "ncclCommInitRank");
    HOT_NCCL_SYM(destroy, "ncclCommDestroy");
    HOT_NCCL_SYM(gstart, "ncclGroupStart");
    HOT_NCCL_SYM(gend, "ncclGroupEnd");
    HOT_NCCL_SYM(bcast, "ncclBroadcast");
    HOT_NCCL_SYM(send, "ncclSend");
    HOT_NCCL_SYM(recv, "ncclRecv");
    HOT_NCCL_SYM(allreduce, "ncclAllReduce");
    HOT_NCCL_SYM(errstr, "ncclGetErrorString");
#undef HOT_NCCL_SYM
    return a;
  }();
  if (!api.so || !api.get_id || !api.init || !api.bcast || !api.send || !api.recv || !api.allreduce || !api.gstart ||
      !api.gend)
    throw std::runtime_error("comm: libnccl.so.2 not loadable (set HOT_NCCL_LIB, or import torch.distributed first)");
  return api;
}

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const NcclApi& a = nccl();
    throw std::runtime_error(std::string("nccl: ") + what + ": " + (a.errstr ? a.errstr(r) : "error"));
  }
}

/// Stream-ordered: every collective is enqueued on the context stream, no host sync (except
/// allreduce_max, whose result the host branches on).
struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  int* dflags = nullptr;

  NcclComm(const unsigned char id[128], int r, int n) {
    rank = r;
    size = n;
    if (n < 1 || r < 0 || r >= n) throw std::invalid_argument("hot_set_comm_nccl: bad rank/size");
    ncclUniqueId uid;
    static_assert(sizeof(uid.internal) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(uid.internal, id, 128);
    nccl_ok(nccl().init(&comm, n, uid, r), "ncclCommInitRank");
    cuda_ok(cudaMalloc(&dflags, sizeof(int) * 64), "flags");
  }
  ~NcclComm() override {
    if (comm && nccl().destroy) nccl().destroy(comm);
    if (dflags) cudaFree(dflags);
  }
  void allgather_ranges(void* d, const std::vector<long long>& off, cudaStream_t s) override {
    ++gathers;
    const NcclApi& a = nccl();
    nccl_ok(a.gstart(), "group");
    for (int r = 0; r < size; ++r) {  // allgatherv: one in-place broadcast per owner
      const long long n = off[r + 1] - off[r];
      if (n > 0) {
        char* p = (char*)d + off[r];
        nccl_ok(a.bcast(p, p, (size_t)n, ncclUint8, r, comm, s), "broadcast");
      }
    }
    nccl_ok(a.gend(), "group");
  }
  void halo(void* d, const std::vector<long long>& e, cudaStream_t s) override {
    ++halos;
    const NcclApi& a = nccl();
    char* base = (char*)d;
    nccl_ok(a.gstart(), "group");
    if (rank > 0) {
      const long long ns = e[4 * rank + 1] - e[4 * rank], nr = e[4 * (rank - 1) + 3] - e[4 * (rank - 1) + 2];
      if (ns > 0) nccl_ok(a.send(base + e[4 * rank], (size_t)ns, ncclUint8, rank - 1, comm, s), "send");
      if (nr > 0) nccl_ok(a.recv(base + e[4 * (rank - 1) + 2], (size_t)nr, ncclUint8, rank - 1, comm, s), "recv");
    }
    if (rank + 1 < size) {
      const long long ns = e[4 * rank + 3] - e[4 * rank + 2], nr = e[4 * (rank + 1) + 1] - e[4 * (rank + 1)];
      if (ns > 0) nccl_ok(a.send(base + e[4 * rank + 2], (size_t)ns, ncclUint8, rank + 1, comm, s), "send");
      if (nr > 0) nccl_ok(a.recv(base + e[4 * (rank + 1)], (size_t)nr, ncclUint8, rank + 1, comm, s), "recv");
    }
    nccl_ok(a.gend(), "group");
  }
  void allreduce_max(int* v, int n, cudaStream_t s) override {
    cuda_ok(cudaMemcpyAsync(dflags, v, sizeof(int) * n, cudaMemcpyHostToDevice, s), "h2d");
    nccl_ok(nccl().allreduce(dflags, dflags, (size_t)n, ncclInt32, ncclMax, comm, s), "allreduce");
    cuda_ok(cudaMemcpyAsync(v, dflags, sizeof(int) * n, cudaMemcpyDeviceToHost, s), "d2h");
    cuda_ok(cudaStreamSynchronize(s), "sync");
  }
};

long long floor_div(long long a, long long b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

}  // namespace

Comm* make_host_comm(const hot_comm_host& ops) { return new HostComm(ops); }
Comm* make_nccl_comm(const unsigned char id[128], int rank, int size) { return new NcclComm(id, rank, size); }
void nccl_unique_id(unsigned char id[128]) {
  ncclUniqueId uid;
  nccl_ok(nccl().get_id(&uid), "ncclGetUniqueId");
  std::memcpy(id, uid.internal, 128);
}

bool plan_slabs(int plane_lo, int nplanes, const long long* w, int size, int align, int min_width, int* bounds) {
  if (size < 1 || nplanes < 0 || align < 1 || min_width < 1) return false;
  const long long hi = (long long)plane_lo + nplanes;
  std::vector<long long> pre(nplanes + 1, 0);  // pre[k]: weight of planes [plane_lo, plane_lo + k)
  for (int k = 0; k < nplanes; ++k) {
    if (w && w[k] < 0) return false;
    pre[k + 1] = pre[k] + (w ? w[k] : 1);
  }
  const long long total = pre[nplanes];
  const long long step = (min_width + align - 1) / align * align;  // cut-to-cut distance of the tightest packing
  bounds[0] = plane_lo;
  for (int r = 1; r < size; ++r) {
    const long long lo_c = floor_div((long long)bounds[r - 1] + min_width + align - 1, align) * align;
    const long long hi_c = floor_div(hi - min_width - (long long)(size - 1 - r) * step, align) * align;
    if (lo_c > hi_c) return false;
    // the aligned cut whose prefix weight is nearest r/size of the total (ties: the lower cut)
    const double target = (double)total * r / size;
    long long best = lo_c;
    double best_d = -1.0;
    for (long long c = lo_c; c <= hi_c; c += align) {
      const double d = std::abs((double)pre[c - plane_lo] - target);
      if (best_d < 0.0 || d < best_d) {
        best_d = d;
        best = c;
      }
    }
    bounds[r] = (int)best;
  }
  bounds[size] = (int)hi;
  return hi - bounds[size - 1] >= min_width;
}

}  // namespace hotb200
