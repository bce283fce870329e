// Slab-rank collectives (slabcomm.cuh).  Replaces the torch.distributed calls the Python
// per-kernel path issues between kernels (the distributed form of krylov.py:151,153,158,161
// sums and of apply_ghosts' x ghosts, mhd.py:144-165) with collectives issued from C on the
// context's streams, so slab ranks keep the one-call-per-iteration Arnoldi driver.
#include <dlfcn.h>
#include <cstdio>
#include <cstring>
#include <new>
#include "slabcomm.cuh"

namespace emhd {

// ---- the few NCCL entry points we use, bound with dlopen (no link-time dependency: the
// process's torch normally has libnccl.so.2 loaded already, and that copy is reused) ----------
namespace nccl {
struct UniqueId { char internal[128]; };
typedef void* Comm;
typedef int Result;
enum { Float64 = 8 };
enum { Sum = 0, Max = 2, Min = 3 };

struct Api {
  bool ok = false;
  Result (*getUniqueId)(UniqueId*) = nullptr;
  Result (*commInitRank)(Comm*, int, UniqueId, int) = nullptr;
  Result (*commDestroy)(Comm) = nullptr;
  Result (*allReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  Result (*send)(const void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  Result (*recv)(void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  Result (*groupStart)() = nullptr;
  Result (*groupEnd)() = nullptr;
  const char* (*errorString)(Result) = nullptr;
};

static Api& api() {
  static Api a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    std::fprintf(stderr, "libemhd: NCCL not available (%s)\n", dlerror());
    return a;
  }
#define BIND(field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name))
  BIND(getUniqueId, "ncclGetUniqueId");
  BIND(commInitRank, "ncclCommInitRank");
  BIND(commDestroy, "ncclCommDestroy");
  BIND(allReduce, "ncclAllReduce");
  BIND(send, "ncclSend");
  BIND(recv, "ncclRecv");
  BIND(groupStart, "ncclGroupStart");
  BIND(groupEnd, "ncclGroupEnd");
  BIND(errorString, "ncclGetErrorString");
#undef BIND
  a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.allReduce && a.send && a.recv &&
         a.groupStart && a.groupEnd;
  return a;
}

static int check(Result r, const char* what) {
  if (r == 0) return 0;
  Api& a = api();
  std::fprintf(stderr, "libemhd: NCCL %s failed: %s\n", what, a.errorString ? a.errorString(r) : "?");
  return 5;   // EMHD_ERR_NCCL
}
}  // namespace nccl

struct SlabComm {
  int nranks = 1, rank = 0, lo = -1, hi = -1;
  bool host = false;
  nccl::Comm reduce = nullptr;      // all-reduces, on the compute stream
  nccl::Comm halo = nullptr;        // halo exchange, on its own stream
  HostAllreduceFn ar = nullptr;
  HostExchangeFn ex = nullptr;
  void* user = nullptr;
  double* stage = nullptr;          // pinned staging (host mode)
  size_t stage_len = 0;
};

int slabcomm_nccl_unique_id(void* out128) {
  nccl::Api& a = nccl::api();
  if (!a.ok || !out128) return 5;
  nccl::UniqueId id;
  const int rc = nccl::check(a.getUniqueId(&id), "GetUniqueId");
  if (!rc) std::memcpy(out128, &id, sizeof(id));
  return rc;
}

SlabComm* slabcomm_create_nccl(int nranks, int rank, int lo, int hi, const void* uid_reduce,
                               const void* uid_halo, int* err) {
  *err = 0;
  nccl::Api& a = nccl::api();
  if (!a.ok) { *err = 5; return nullptr; }
  SlabComm* c = new (std::nothrow) SlabComm();
  if (!c) { *err = 6; return nullptr; }
  c->nranks = nranks; c->rank = rank; c->lo = lo; c->hi = hi;
  nccl::UniqueId u1, u2;
  std::memcpy(&u1, uid_reduce, sizeof(u1));
  std::memcpy(&u2, uid_halo, sizeof(u2));
  *err = nccl::check(a.commInitRank(&c->reduce, nranks, u1, rank), "CommInitRank");
  if (!*err) *err = nccl::check(a.commInitRank(&c->halo, nranks, u2, rank), "CommInitRank");
  if (*err) { slabcomm_destroy(c); return nullptr; }
  return c;
}

SlabComm* slabcomm_create_host(int nranks, int rank, int lo, int hi, HostAllreduceFn ar,
                               HostExchangeFn ex, void* user) {
  SlabComm* c = new (std::nothrow) SlabComm();
  if (!c) return nullptr;
  c->nranks = nranks; c->rank = rank; c->lo = lo; c->hi = hi;
  c->host = true; c->ar = ar; c->ex = ex; c->user = user;
  return c;
}

void slabcomm_destroy(SlabComm* c) {
  if (!c) return;
  nccl::Api& a = nccl::api();
  if (c->reduce && a.commDestroy) a.commDestroy(c->reduce);
  if (c->halo && a.commDestroy) a.commDestroy(c->halo);
  if (c->stage) cudaFreeHost(c->stage);
  delete c;
}

int slabcomm_nranks(const SlabComm* c) { return c ? c->nranks : 1; }
int slabcomm_rank(const SlabComm* c) { return c ? c->rank : 0; }
bool slabcomm_is_host(const SlabComm* c) { return c && c->host; }

static double* stage(SlabComm* c, size_t n) {
  if (n > c->stage_len) {
    if (c->stage) cudaFreeHost(c->stage);
    c->stage = nullptr;
    c->stage_len = 0;
    if (cudaMallocHost(&c->stage, n * sizeof(double)) != cudaSuccess) return nullptr;
    c->stage_len = n;
  }
  return c->stage;
}

static int host_allreduce(SlabComm* c, double* buf, int n, int op, cudaStream_t s) {
  double* h = stage(c, (size_t)n);
  if (!h) return 4;
  if (cudaMemcpyAsync(h, buf, sizeof(double) * n, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return 4;
  if (c->ar(c->user, h, n, op) != 0) return 5;
  if (cudaMemcpyAsync(buf, h, sizeof(double) * n, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return 4;
  return 0;
}

int slabcomm_allreduce(SlabComm* c, double* buf, int n, int op, cudaStream_t s) {
  if (!c || n <= 0) return 0;
  if (c->host) return host_allreduce(c, buf, n, op, s);
  nccl::Api& a = nccl::api();
  const int nop = op == 2 ? nccl::Max : (op == 3 ? nccl::Min : nccl::Sum);
  return nccl::check(a.allReduce(buf, buf, (size_t)n, nccl::Float64, nop, c->reduce, s), "AllReduce");
}

int slabcomm_allreduce_sum_max(SlabComm* c, double* buf, int n_sum, int n_max, cudaStream_t s) {
  if (!c) return 0;
  if (c->host) {
    int rc = n_sum > 0 ? host_allreduce(c, buf, n_sum, 0, s) : 0;
    if (!rc && n_max > 0) rc = host_allreduce(c, buf + n_sum, n_max, 2, s);
    return rc;
  }
  nccl::Api& a = nccl::api();
  int rc = nccl::check(a.groupStart(), "GroupStart");
  if (!rc && n_sum > 0)
    rc = nccl::check(a.allReduce(buf, buf, (size_t)n_sum, nccl::Float64, nccl::Sum, c->reduce, s), "AllReduce");
  if (!rc && n_max > 0)
    rc = nccl::check(a.allReduce(buf + n_sum, buf + n_sum, (size_t)n_max, nccl::Float64, nccl::Max,
                                 c->reduce, s), "AllReduce");
  const int rc2 = nccl::check(a.groupEnd(), "GroupEnd");
  return rc ? rc : rc2;
}

int slabcomm_exchange(SlabComm* c, const double* send, double* recv, long long n_side, cudaStream_t s) {
  if (!c) return 6;
  if (c->host) {
    double* h = stage(c, (size_t)(4 * n_side));
    if (!h) return 4;
    if (cudaMemcpyAsync(h, send, sizeof(double) * 2 * n_side, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return 4;
    if (c->ex(c->user, h, h + 2 * n_side, n_side) != 0) return 5;
    if (cudaMemcpyAsync(recv, h + 2 * n_side, sizeof(double) * 2 * n_side, cudaMemcpyHostToDevice, s) !=
            cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return 4;
    return 0;
  }
  // Posting order per peer pair is the match order (no tags): top rows go up and arrive as the
  // receiver's lo-side halo, bottom rows go down and arrive as its hi-side halo — correct also
  // when lo and hi are the same rank (P = 2) or this rank itself (P = 1, periodic ring).
  nccl::Api& a = nccl::api();
  int rc = nccl::check(a.groupStart(), "GroupStart");
  const size_t n = (size_t)n_side;
  if (!rc && c->hi >= 0) rc = nccl::check(a.send(send + n, n, nccl::Float64, c->hi, c->halo, s), "Send");
  if (!rc && c->lo >= 0) rc = nccl::check(a.recv(recv, n, nccl::Float64, c->lo, c->halo, s), "Recv");
  if (!rc && c->lo >= 0) rc = nccl::check(a.send(send, n, nccl::Float64, c->lo, c->halo, s), "Send");
  if (!rc && c->hi >= 0) rc = nccl::check(a.recv(recv + n, n, nccl::Float64, c->hi, c->halo, s), "Recv");
  const int rc2 = nccl::check(a.groupEnd(), "GroupEnd");
  return rc ? rc : rc2;
}

}  // namespace emhd
