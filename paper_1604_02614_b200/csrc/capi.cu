// C ABI of libemhd.so (declared in include/emhd.h).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>
#include "../../include/emhd.h"
#include "emhd_common.cuh"
#include "stencil.cuh"
#include "krylov.cuh"
#include "dense.cuh"
#include "vecops.cuh"
#include "harness.cuh"
#include "slabcomm.cuh"

using namespace emhd;

struct emhd_ctx {
  emhd_geometry g;
  emhd_physics p;
  cudaStream_t stream = 0;
  int device = 0;
  int num_sms = 148;
  int max_vectors = 0;
  double* partials = nullptr;         // reduction scratch
  size_t partials_len = 0;
  unsigned int* ticket = nullptr;
  DevStatus* st = nullptr;
  DevStatus* st_host = nullptr;       // pinned mirror
  double* dense = nullptr;            // dense workspace
  size_t dense_len = 0;
  StencilParams base{};
  int epoch = -1;                             // tag of stencil launches outside the Arnoldi
                                              // driver (-1: never a discarded speculative one)
  unsigned long long* cancel = nullptr;       // look-ahead cancel word {generation, epoch}
  unsigned long long* cancel_host = nullptr;  // pinned source of its async updates
  const double* skip_next = nullptr;          // emhd_skip_next: gate of the next pass-2 launch
  bool l2win = false;                         // emhd_l2_window set on this context's stream
  cudaStream_t l2win_stream = nullptr;        // the stream carrying the window
  bool l2_limit_changed = false;              // this context raised the persisting-L2 limit
  size_t l2_limit_prev = 0;                   // ... from this value (restored on destroy)
  StencilPath path{};                         // stencil launch selection (emhd_set_stencil_path)
  StencilPath last{};                         // what the last stencil launch ran
  bool fused_orth = true;                     // small grids: one-launch orthogonalisation
                                              // (emhd_set_fused_orth; default EMHD_FUSED_ORTH)
  // slab-rank collectives (emhd_comm_init_*): all-reduces on `stream`, halo exchange on
  // halo_stream into hrecv, overlapped with the interior rows of the stencil that needs it
  SlabComm* comm = nullptr;
  cudaStream_t halo_stream = nullptr;
  cudaEvent_t ev_x = nullptr, ev_halo = nullptr;
  double* hsend = nullptr;                    // [2][8][2][ny] edge rows of the exchanged array
  double* hrecv = nullptr;                    // [2][8][2][ny] halo the stencil reads
  double* red = nullptr;                      // [max_vectors + 8] reduction scratch (slab path)
  // per-launch profiling (emhd_profile): CUDA events around every launch of the Arnoldi path
  struct ProfRec { int kind; cudaEvent_t e0, e1; double bytes; const double* gate[2]; };
  bool prof = false;
  std::vector<ProfRec> recs;
};

// Brackets one launch with CUDA events on the context's stream when profiling is on; the
// algorithmic bytes count only if neither gate (device flags read back by emhd_profile_read)
// says the launch did no work.
struct ProfScope {
  emhd_ctx* c;
  int kind;
  double bytes;
  const double* g0;
  const double* g1;
  cudaEvent_t e0{};
  ProfScope(emhd_ctx* c_, int kind_, double bytes_, const double* g0_ = nullptr, const double* g1_ = nullptr)
      : c(c_), kind(kind_), bytes(bytes_), g0(g0_), g1(g1_) {
    if (c->prof) {
      cudaEventCreate(&e0);
      cudaEventRecord(e0, c->stream);
    }
  }
  ~ProfScope() {
    if (!c->prof) return;
    cudaEvent_t e1;
    cudaEventCreate(&e1);
    cudaEventRecord(e1, c->stream);
    emhd_ctx::ProfRec r;
    r.kind = kind; r.e0 = e0; r.e1 = e1; r.bytes = bytes; r.gate[0] = g0; r.gate[1] = g1;
    c->recs.push_back(r);
  }
};

static void prof_clear(emhd_ctx* c) {
  for (auto& r : c->recs) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  c->recs.clear();
}

// the gate set by emhd_skip_next, consumed by exactly one pass-2 launch
static const double* take_skip(emhd_ctx* c) {
  const double* g = c->skip_next;
  c->skip_next = nullptr;
  return g;
}

static int cerr(cudaError_t e) {
  if (e == cudaSuccess) return EMHD_OK;
  std::fprintf(stderr, "libemhd: CUDA error %s\n", cudaGetErrorString(e));
  return EMHD_ERR_CUDA;
}

extern "C" const char* emhd_version(void) { return "emhd-b200 0.1 (sm_100a)"; }

extern "C" const char* emhd_error_string(int code) {
  switch (code) {
    case EMHD_OK: return "ok";
    case EMHD_ERR_DENSITY: return "non-positive density";
    case EMHD_ERR_PRESSURE: return "non-positive pressure";
    case EMHD_ERR_NONFINITE: return "non-finite rhs value during Jacobian apply";
    case EMHD_ERR_CUDA: return "CUDA error";
    case EMHD_ERR_NCCL: return "NCCL / slab communication error";
    case EMHD_ERR_ARG: return "bad argument";
    case EMHD_ERR_DENSE: return "non-finite small dense exponential";
    default: return "unknown";
  }
}

static void fill_base(emhd_ctx* c) {
  StencilParams& P = c->base;
  std::memset(&P, 0, sizeof(P));
  P.nx = c->g.nx; P.ny = c->g.ny; P.nxg = c->g.nx_global; P.x_off = c->g.x_offset;
  P.bcx_lo = c->g.bc_x_lo; P.bcx_hi = c->g.bc_x_hi; P.bcy = c->g.bc_y;
  P.rows_per_cta = 0;
  P.check = c->p.check;
  const double g = c->p.gamma;
  P.gm1 = g - 1.0;
  P.mu = c->p.mu; P.eta = c->p.eta;
  P.heat = g * c->p.mu * c->p.kappa / (g - 1.0);          // mhd.py:259
  P.bfac = c->p.b_half ? 0.5 : 1.0;                         // mhd.py:108
  P.two_hx = 2.0 * c->g.hx; P.r_two_hx = 1.0 / P.two_hx;    // mhd.py:202
  P.two_hy = 2.0 * c->g.hy; P.r_two_hy = 1.0 / P.two_hy;    // mhd.py:206
  P.n_top = (long long)NF * c->g.nx * c->g.ny;
  P.st = c->st;
  P.rows_mode = 0; P.row_lo = 0; P.row_hi = c->g.nx; P.count = 1;
}

extern "C" int emhd_ctx_create(emhd_ctx** out, const emhd_geometry* g, const emhd_physics* p,
                               int max_vectors) {
  if (!out || !g || !p) return EMHD_ERR_ARG;
  if (g->nx < 2 || g->ny < 4 || g->nx_global < g->nx || g->hx <= 0 || g->hy <= 0) return EMHD_ERR_ARG;
  if (g->bc_y < 0 || g->bc_y > 2 || g->bc_x_lo < 0 || g->bc_x_lo > 3 || g->bc_x_hi < 0 || g->bc_x_hi > 3)
    return EMHD_ERR_ARG;
  emhd_ctx* c = new (std::nothrow) emhd_ctx();
  if (!c) return EMHD_ERR_ARG;
  c->g = *g;
  c->p = *p;
  c->max_vectors = max_vectors < 8 ? 8 : max_vectors;
  int rc = cerr(cudaGetDevice(&c->device));
  if (!rc) rc = cerr(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  c->partials_len = (size_t)(c->max_vectors + 8) * 4 * c->num_sms + 64;
  if (!rc) rc = cerr(cudaMalloc(&c->partials, c->partials_len * sizeof(double)));
  if (!rc) rc = cerr(cudaMalloc(&c->ticket, 16 * sizeof(unsigned int)));
  if (!rc) rc = cerr(cudaMemset(c->ticket, 0, 16 * sizeof(unsigned int)));
  if (!rc) rc = cerr(cudaMalloc(&c->st, sizeof(DevStatus)));
  if (!rc) rc = cerr(cudaMallocHost(&c->st_host, sizeof(DevStatus)));
  if (!rc) rc = cerr(cudaMalloc(&c->cancel, sizeof(unsigned long long)));
  if (!rc) rc = cerr(cudaMallocHost(&c->cancel_host, sizeof(unsigned long long)));
  if (!rc) rc = cerr(cudaMemset(c->cancel, 0xff, sizeof(unsigned long long)));   // matches nothing
  if (rc) { emhd_ctx_destroy(c); return rc; }
  fill_base(c);
  c->path = stencil_path_defaults();
  {
    const char* e = getenv("EMHD_FUSED_ORTH");
    c->fused_orth = e ? atoi(e) != 0 : true;
  }
  emhd_status_reset(c);
  rc = cerr(cudaStreamSynchronize(0));
  *out = c;
  return rc;
}

extern "C" int emhd_ctx_destroy(emhd_ctx* c) {
  if (!c) return EMHD_OK;
  if (c->l2win) {
    // remove the persisting window from the stream, release the persisting lines and give the
    // device back its previous persisting-L2 limit: nothing outlives the context
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(c->l2win_stream, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaCtxResetPersistingL2Cache();
  }
  if (c->l2_limit_changed) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, c->l2_limit_prev);
  cudaGetLastError();
  cudaFree(c->partials);
  cudaFree(c->ticket);
  cudaFree(c->st);
  cudaFree(c->dense);
  prof_clear(c);
  cudaFree(c->cancel);
  if (c->comm) slabcomm_destroy(c->comm);
  if (c->halo_stream) cudaStreamDestroy(c->halo_stream);
  if (c->ev_x) cudaEventDestroy(c->ev_x);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  cudaFree(c->hsend);
  cudaFree(c->hrecv);
  cudaFree(c->red);
  if (c->st_host) cudaFreeHost(c->st_host);
  if (c->cancel_host) cudaFreeHost(c->cancel_host);
  delete c;
  return EMHD_OK;
}

extern "C" int emhd_set_stream(emhd_ctx* c, void* s) {
  if (!c) return EMHD_ERR_ARG;
  c->stream = (cudaStream_t)s;
  return EMHD_OK;
}

extern "C" int emhd_num_sms(emhd_ctx* c) { return c ? c->num_sms : 0; }

// Persisting-L2 access window on the context's stream over [base, base + bytes): the head of
// a Krylov basis that fits the L2 stays resident across iterations (its lines are kept while
// the streaming vectors evict each other).  bytes = 0 removes the window and releases the
// persisting lines.  Clamped to the device's window and persisting-L2 limits.
extern "C" int emhd_l2_window(emhd_ctx* c, const void* base, long long bytes) {
  if (!c || bytes < 0) return EMHD_ERR_ARG;
  int maxwin = 0, maxpers = 0;
  int rc = cerr(cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, c->device));
  if (!rc) rc = cerr(cudaDeviceGetAttribute(&maxpers, cudaDevAttrMaxPersistingL2CacheSize, c->device));
  if (rc) return rc;
  if (bytes > maxwin) bytes = maxwin;
  cudaStreamAttrValue v{};
  if (bytes > 0 && maxpers > 0) {
    const size_t lim = (size_t)(bytes < maxpers ? bytes : maxpers);
    size_t cur = 0;
    rc = cerr(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
    if (!rc && cur != lim) {
      if (!c->l2_limit_changed) { c->l2_limit_changed = true; c->l2_limit_prev = cur; }
      rc = cerr(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim));
    }
    if (rc) return rc;
    v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    v.accessPolicyWindow.num_bytes = (size_t)bytes;
    v.accessPolicyWindow.hitRatio = bytes <= maxpers ? 1.0f : (float)maxpers / (float)bytes;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  } else {
    v.accessPolicyWindow.num_bytes = 0;
  }
  rc = cerr(cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &v));
  if (!rc) {
    c->l2win = v.accessPolicyWindow.num_bytes > 0;
    c->l2win_stream = c->stream;
  }
  if (!rc && bytes == 0) rc = cerr(cudaCtxResetPersistingL2Cache());
  return rc;
}

static void to_c(const StencilPath& a, emhd_stencil_path* b) {
  b->kernel = a.kernel; b->rows_per_cta = a.rows_per_cta; b->strip = a.strip; b->bulk = a.bulk;
  b->min_rows = a.min_rows; b->tile_rows = a.tile_rows; b->raw_rows = a.raw_rows;
}

extern "C" int emhd_set_stencil_path(emhd_ctx* c, const emhd_stencil_path* sel) {
  if (!c || !sel || sel->kernel < 0 || sel->kernel > 2 || sel->rows_per_cta < 0 || sel->min_rows < 1 ||
      sel->raw_rows < 0 || sel->raw_rows > 2 ||
      (sel->strip != 0 && sel->strip != 32 && sel->strip != 64 && sel->strip != 128))
    return EMHD_ERR_ARG;
  c->path.kernel = sel->kernel; c->path.rows_per_cta = sel->rows_per_cta; c->path.strip = sel->strip;
  c->path.bulk = sel->bulk != 0; c->path.min_rows = sel->min_rows; c->path.tile_rows = sel->tile_rows;
  c->path.raw_rows = sel->raw_rows;
  return EMHD_OK;
}

extern "C" int emhd_set_fused_orth(emhd_ctx* c, int on) {
  if (!c) return EMHD_ERR_ARG;
  c->fused_orth = on != 0;
  return EMHD_OK;
}

extern "C" int emhd_get_stencil_path(emhd_ctx* c, emhd_stencil_path* out) {
  if (!c || !out) return EMHD_ERR_ARG;
  to_c(c->path, out);
  return EMHD_OK;
}

extern "C" int emhd_last_stencil(emhd_ctx* c, emhd_stencil_path* out) {
  if (!c || !out) return EMHD_ERR_ARG;
  to_c(c->last, out);
  return EMHD_OK;
}

extern "C" int emhd_set_epoch(emhd_ctx* c, int epoch) {
  if (!c) return EMHD_ERR_ARG;
  c->epoch = epoch;
  return EMHD_OK;
}

extern "C" int emhd_status_reset(emhd_ctx* c) {
  if (!c) return EMHD_ERR_ARG;
  DevStatus h{};
  h.first_nonfinite = ~0ull;
  h.fail_iter = 0x7fffffff;
  // small H2D copy from a stack value must complete before return: use the pinned mirror
  *c->st_host = h;
  int rc = cerr(cudaMemcpyAsync(c->st, c->st_host, sizeof(DevStatus), cudaMemcpyHostToDevice, c->stream));
  if (!rc) rc = cerr(cudaStreamSynchronize(c->stream));
  return rc;
}

// Stream-ordered scrub of stencil error flags raised by iterations with epoch >= epoch_min
// (speculative iterations that were discarded, possibly still running when the host decided):
// the reference never performs them, so their flags must not reach a later status read.
__global__ void status_scrub_kernel(DevStatus* st, int epoch_min) {
  if ((st->flags & (ST_RHO | ST_PRESSURE | ST_NONFINITE)) && st->fail_iter >= epoch_min) {
    st->flags &= ~(ST_RHO | ST_PRESSURE | ST_NONFINITE);
    st->fail_iter = 0x7fffffff;
    st->first_nonfinite = ~0ull;
  }
}

__global__ void status_clear_errors_kernel(DevStatus* st) {
  st->flags &= ~(ST_RHO | ST_PRESSURE | ST_NONFINITE | ST_DENSE);
  st->fail_iter = 0x7fffffff;
  st->first_nonfinite = ~0ull;
}

// Stream-ordered: clear the error flags (and their first-failure records) but keep the RHS
// count and its mark — errors of discarded speculative work are forgotten, counting goes on
extern "C" int emhd_status_clear_errors(emhd_ctx* c) {
  if (!c) return EMHD_ERR_ARG;
  status_clear_errors_kernel<<<1, 1, 0, c->stream>>>(c->st);
  return cerr(cudaGetLastError());
}

extern "C" int emhd_status_scrub(emhd_ctx* c, int epoch_min) {
  if (!c) return EMHD_ERR_ARG;
  status_scrub_kernel<<<1, 1, 0, c->stream>>>(c->st, epoch_min);
  return cerr(cudaGetLastError());
}

__global__ void evals_mark_kernel(DevStatus* st) { st->rhs_evals_mark = st->rhs_evals; }

extern "C" int emhd_evals_mark(emhd_ctx* c) {
  if (!c) return EMHD_ERR_ARG;
  evals_mark_kernel<<<1, 1, 0, c->stream>>>(c->st);
  return cerr(cudaGetLastError());
}

extern "C" int emhd_status_read(emhd_ctx* c, emhd_status* out) {
  if (!c || !out) return EMHD_ERR_ARG;
  int rc = cerr(cudaMemcpyAsync(c->st_host, c->st, sizeof(DevStatus), cudaMemcpyDeviceToHost, c->stream));
  if (!rc) rc = cerr(cudaStreamSynchronize(c->stream));
  if (rc) return rc;
  out->flags = c->st_host->flags;
  out->rhs_evals = c->st_host->rhs_evals;
  out->rhs_evals_mark = c->st_host->rhs_evals_mark;
  out->first_nonfinite = c->st_host->first_nonfinite;
  out->breakdown = c->st_host->breakdown;
  out->fail_iter = c->st_host->fail_iter;
  return EMHD_OK;
}

static void set_epilogue(StencilParams& P, int p, double ch, int nb, const double* const* bcol,
                         const int* bidx) {
  P.p = p;
  P.ch = ch;
  P.nb = nb;
  for (int k = 0; k < 5; ++k) { P.bcol[k] = nullptr; P.bidx[k] = 0; }
  for (int k = 0; k < nb; ++k) { P.bcol[k] = bcol[k]; P.bidx[k] = bidx[k]; }
}

// ---- slab-rank collectives -------------------------------------------------------------
extern "C" int emhd_nccl_unique_id(void* out128) {
  return slabcomm_nccl_unique_id(out128) ? EMHD_ERR_NCCL : EMHD_OK;
}

static int comm_buffers(emhd_ctx* c) {
  const size_t n = (size_t)2 * NF * 2 * c->g.ny;
  int rc = cerr(cudaMalloc(&c->hsend, n * sizeof(double)));
  if (!rc) rc = cerr(cudaMalloc(&c->hrecv, n * sizeof(double)));
  if (!rc) rc = cerr(cudaMalloc(&c->red, (size_t)(c->max_vectors + 8) * sizeof(double)));
  if (!rc) rc = cerr(cudaMemset(c->hrecv, 0, n * sizeof(double)));
  if (!rc) rc = cerr(cudaStreamCreateWithFlags(&c->halo_stream, cudaStreamNonBlocking));
  if (!rc) rc = cerr(cudaEventCreateWithFlags(&c->ev_x, cudaEventDisableTiming));
  if (!rc) rc = cerr(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
  return rc;
}

static int comm_args_ok(emhd_ctx* c, int nranks, int rank, int lo, int hi) {
  return c && !c->comm && nranks >= 1 && rank >= 0 && rank < nranks && lo >= -1 && lo < nranks &&
         hi >= -1 && hi < nranks && (lo >= 0) == (c->g.bc_x_lo == EMHD_BC_EXTERNAL) &&
         (hi >= 0) == (c->g.bc_x_hi == EMHD_BC_EXTERNAL);
}

extern "C" int emhd_comm_init_nccl(emhd_ctx* c, int nranks, int rank, int lo, int hi,
                                   const void* uid_reduce, const void* uid_halo) {
  if (!comm_args_ok(c, nranks, rank, lo, hi) || !uid_reduce || !uid_halo) return EMHD_ERR_ARG;
  int rc = cerr(cudaSetDevice(c->device));
  if (rc) return rc;
  int err = 0;
  SlabComm* sc = slabcomm_create_nccl(nranks, rank, lo, hi, uid_reduce, uid_halo, &err);
  if (!sc) return err == 6 ? EMHD_ERR_ARG : EMHD_ERR_NCCL;
  c->comm = sc;
  return comm_buffers(c);
}

extern "C" int emhd_comm_init_host(emhd_ctx* c, int nranks, int rank, int lo, int hi,
                                   emhd_host_allreduce_fn ar, emhd_host_exchange_fn ex, void* user) {
  if (!comm_args_ok(c, nranks, rank, lo, hi) || !ar || !ex) return EMHD_ERR_ARG;
  c->comm = slabcomm_create_host(nranks, rank, lo, hi, ar, ex, user);
  if (!c->comm) return EMHD_ERR_ARG;
  return comm_buffers(c);
}

extern "C" int emhd_allreduce(emhd_ctx* c, double* buf, int n, int op) {
  if (!c || !buf || n < 0 || (op != EMHD_OP_SUM && op != EMHD_OP_MAX && op != EMHD_OP_MIN)) return EMHD_ERR_ARG;
  if (!c->comm) return EMHD_OK;
  const int rc = slabcomm_allreduce(c->comm, buf, n, op, c->stream);
  return rc == 4 ? EMHD_ERR_CUDA : (rc ? EMHD_ERR_NCCL : EMHD_OK);
}

__global__ void pack_edges_kernel(const double* x, double* buf, int nx, int ny);

static cudaError_t pack_edges(emhd_ctx* c, const double* x, double* buf, cudaStream_t s) {
  const long long total = 2LL * NF * 2 * c->g.ny;
  pack_edges_kernel<<<(int)((total + 255) / 256), 256, 0, s>>>(x, buf, c->g.nx, c->g.ny);
  return cudaGetLastError();
}

static int comm_rc(int rc) { return rc == 4 ? EMHD_ERR_CUDA : (rc ? EMHD_ERR_NCCL : EMHD_OK); }

// x-halo of x into `halo` ([2][8][2][ny]) on the context's stream (host transport: synchronous)
extern "C" int emhd_halo_exchange(emhd_ctx* c, const double* x, double* halo) {
  if (!c || !x || !halo) return EMHD_ERR_ARG;
  if (!c->comm) return EMHD_ERR_ARG;
  int rc = cerr(pack_edges(c, x, c->hsend, c->stream));
  if (rc) return rc;
  return comm_rc(slabcomm_exchange(c->comm, c->hsend, halo, (long long)NF * 2 * c->g.ny, c->stream));
}

// The stencil P over the whole slab.  When the context has a communicator and the caller gave
// no halo for `x` (*halo_field == null on an EXTERNAL side), the halo is exchanged here: the
// exchange runs on the halo stream while the interior rows [2, nx-2) — which need no halo —
// run on the compute stream; the two edge row pairs follow once the halo has landed.
static int stencil_with_halo(emhd_ctx* c, StencilParams P, int mode, bool aug, const double* x,
                             bool x_is_a) {
  const bool external = c->g.bc_x_lo == EMHD_BC_EXTERNAL || c->g.bc_x_hi == EMHD_BC_EXTERNAL;
  const double*& halo_field = x_is_a ? P.a_halo : P.v_halo;
  if (!c->comm || !external || halo_field != nullptr)
    return cerr(launch_stencil(P, mode, aug, c->num_sms, c->stream, c->path, &c->last));
  halo_field = c->hrecv;
  const long long n_side = (long long)NF * 2 * c->g.ny;
  if (slabcomm_is_host(c->comm) || c->g.nx < 4) {
    int rc = cerr(pack_edges(c, x, c->hsend, c->stream));
    if (!rc) rc = comm_rc(slabcomm_exchange(c->comm, c->hsend, c->hrecv, n_side, c->stream));
    if (!rc) rc = cerr(launch_stencil(P, mode, aug, c->num_sms, c->stream, c->path, &c->last));
    return rc;
  }
  int rc = cerr(cudaEventRecord(c->ev_x, c->stream));
  if (!rc) rc = cerr(cudaStreamWaitEvent(c->halo_stream, c->ev_x, 0));
  if (!rc) rc = cerr(pack_edges(c, x, c->hsend, c->halo_stream));
  if (!rc) rc = comm_rc(slabcomm_exchange(c->comm, c->hsend, c->hrecv, n_side, c->halo_stream));
  if (!rc) rc = cerr(cudaEventRecord(c->ev_halo, c->halo_stream));
  if (rc) return rc;
  if (c->g.nx > 4) {
    StencilParams Pi = P;
    Pi.rows_mode = 1; Pi.row_lo = 2; Pi.row_hi = c->g.nx - 2; Pi.count = 1;
    rc = cerr(launch_stencil(Pi, mode, aug, c->num_sms, c->stream, c->path, &c->last));
    if (rc) return rc;
  }
  rc = cerr(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
  if (rc) return rc;
  StencilParams Pb = P;
  Pb.rows_mode = 2; Pb.count = c->g.nx > 4 ? 0 : 1;
  return cerr(launch_stencil(Pb, mode, aug, c->num_sms, c->stream, c->path, &c->last));
}

extern "C" int emhd_rhs(emhd_ctx* c, const double* u, const double* u_halo, double* F) {
  if (!c || !u || !F) return EMHD_ERR_ARG;
  StencilParams P = c->base;
  P.epoch = c->epoch;
  P.a = u; P.a_halo = u_halo; P.out = F;
  return stencil_with_halo(c, P, MODE_RHS, false, u, true);
}

extern "C" int emhd_jv(emhd_ctx* c, const double* a, const double* a_halo, const double* fa,
                       const double* v, const double* v_halo, const double* d_vnorm, double* out) {
  if (!c || !a || !fa || !v || !d_vnorm || !out) return EMHD_ERR_ARG;
  StencilParams P = c->base;
  P.epoch = c->epoch;
  P.a = a; P.a_halo = a_halo; P.fa = fa; P.v = v; P.v_halo = v_halo; P.scal = d_vnorm; P.out = out;
  ProfScope ps(c, EMHD_K_JV, 4.0 * 64.0 * (double)c->g.nx * c->g.ny);   // 4W
  return stencil_with_halo(c, P, MODE_JV, false, v, false);
}

extern "C" int emhd_jv_aug(emhd_ctx* c, const double* a, const double* a_halo, const double* fa,
                           const double* u, const double* u_halo, const double* d_vnorm, const double* d_q,
                           int p, double ch, int nb, const double* const* bcol, const int* bidx,
                           double* out) {
  if (!c || !a || !fa || !u || !d_vnorm || !out || p < 1 || p > 5 || nb < 0 || nb > 5 || !d_q)
    return EMHD_ERR_ARG;
  StencilParams P = c->base;
  P.epoch = c->epoch;
  P.a = a; P.a_halo = a_halo; P.fa = fa; P.v = u; P.v_halo = u_halo; P.scal = d_vnorm; P.out = out;
  P.qsrc = d_q;
  set_epilogue(P, p, ch, nb, bcol, bidx);
  return stencil_with_halo(c, P, MODE_JV, true, u, false);
}

extern "C" int emhd_jv_normalized(emhd_ctx* c, const double* a, const double* a_halo, const double* fa,
                                  const double* w, const double* w_halo, const double* d_scal,
                                  double* v_out, int p, double ch, int nb, const double* const* bcol,
                                  const int* bidx, double* out) {
  if (!c || !a || !fa || !w || !d_scal || !v_out || !out || p < 0 || p > 5 || nb < 0 || nb > 5)
    return EMHD_ERR_ARG;
  StencilParams P = c->base;
  P.epoch = c->epoch;
  P.a = a; P.a_halo = a_halo; P.fa = fa; P.v = w; P.v_halo = w_halo; P.scal = d_scal;
  P.out = out; P.vout = v_out;
  set_epilogue(P, p, ch, nb, bcol, bidx);
  ProfScope ps(c, EMHD_K_JV_NORMALIZED, 5.0 * 64.0 * (double)c->g.nx * c->g.ny);   // 5W
  return stencil_with_halo(c, P, MODE_JVN, p > 0, w, false);
}

static KWork kwork(emhd_ctx* c) {
  KWork w;
  w.partials = c->partials;
  w.ticket = c->ticket;
  w.num_sms = c->num_sms;
  w.stream_basis = c->l2win;
  return w;
}

extern "C" int emhd_multidot(emhd_ctx* c, const double* w, const double* V, long long ldv, int nvec,
                             long long len_dot, int self, double* out) {
  if (!c || !w || !out || nvec < 0 || nvec > c->max_vectors || (nvec > 0 && !V)) return EMHD_ERR_ARG;
  KWork k = kwork(c);
  ProfScope ps(c, EMHD_K_MULTIDOT, 8.0 * (nvec + 1) * (double)len_dot);
  return cerr(launch_multidot(w, V, ldv, nvec, len_dot, self ? 1 : 0, k, out, c->stream));
}

extern "C" int emhd_update(emhd_ctx* c, double* w, const double* V, long long ldv, int nvec, const double* h,
                           long long len_upd, long long len_dot, long long len_max, int mode, double* out) {
  if (!c || !w || !out || nvec < 0 || nvec > c->max_vectors || (nvec > 0 && (!V || !h))) return EMHD_ERR_ARG;
  KWork k = kwork(c);
  const double* g = mode == 1 ? take_skip(c) : nullptr;
  Reorth ro{};
  ro.skip2 = g;
  ProfScope ps(c, mode == 1 ? EMHD_K_UPDATE_FINISH : EMHD_K_UPDATE, 8.0 * (nvec + 2) * (double)len_upd, g);
  return cerr(launch_update(w, V, ldv, nvec, h, len_upd, len_dot, len_max, mode, k, out, c->stream,
                            FinishArgs{}, nullptr, ro));
}

// Selective re-orthogonalisation decision after an (all-reduced) mode-0 update: r = {V^T w1
// (nvec), ||w1||^2, max|w1_top|}; gate = 1 and the column finished with h1 when
// ||w1||^2 >= eta^2 selfdot, else gate = 0 (the second pass must run).
extern "C" int emhd_reorth_decide(emhd_ctx* c, const double* h1, const double* r, int nvec,
                                  const double* selfdot, int j, double* H, long long ldh, double* scal,
                                  double* brk_hist, double eta, double* gate) {
  if (!c || !h1 || !r || !selfdot || !H || !scal || !gate || nvec < 1 || j < 0 || !(eta > 0.0))
    return EMHD_ERR_ARG;
  FinishArgs F;
  F.h1 = h1; F.h2 = nullptr; F.selfdot = selfdot; F.j = j; F.H = H; F.ldh = ldh; F.scal = scal;
  F.brk_hist = brk_hist; F.st = c->st; F.rtol = 1e-12;
  return cerr(launch_reorth_decide(F, r, nvec, eta * eta, gate, c->stream));
}

// The next pass-2 launch on this context (emhd_update mode 1, emhd_update_finish,
// emhd_update_push or emhd_arnoldi_finish) does no work when *gate != 0 (device-side).
extern "C" int emhd_skip_next(emhd_ctx* c, const double* gate) {
  if (!c) return EMHD_ERR_ARG;
  c->skip_next = gate;
  return EMHD_OK;
}

// emhd_update mode 1 whose final w also lands, rows {0,1} and {nx-2,nx-1} of every field, in
// the neighbours' halo buffers (peer pointers from symmetric memory; null side: no neighbour).
// Ordered before the neighbours' next stencil by the norm all-reduce that follows.
extern "C" int emhd_update_push(emhd_ctx* c, double* w, const double* V, long long ldv, int nvec,
                                const double* h, long long len_upd, long long len_dot, long long len_max,
                                double* out, double* lo_halo, double* hi_halo) {
  if (!c || !w || !out || nvec < 0 || nvec > c->max_vectors || (nvec > 0 && (!V || !h))) return EMHD_ERR_ARG;
  KWork k = kwork(c);
  HaloPush P;
  P.lo = lo_halo;
  P.hi = hi_halo;
  P.n_top = 8LL * c->g.nx * c->g.ny;
  P.plane = (unsigned)((long long)c->g.nx * c->g.ny);
  P.nx = (unsigned)c->g.nx;
  P.ny = (unsigned)c->g.ny;
  if (P.n_top >= (1LL << 32)) return EMHD_ERR_ARG;
  const double* g = take_skip(c);
  ProfScope ps(c, EMHD_K_UPDATE_FINISH, 8.0 * (nvec + 2) * (double)len_upd, g);
  return cerr(launch_update_push(w, V, ldv, nvec, h, len_upd, len_dot, len_max, k, out, P, c->stream, g));
}

// Edge rows {0,1} and {nx-2,nx-1} of w into the neighbours' halo buffers (as emhd_update_push
// stores them) when *gate != 0 (gate null: always); ordered by the collective that follows.
extern "C" int emhd_push_edges(emhd_ctx* c, const double* w, double* lo_halo, double* hi_halo,
                               const double* gate) {
  if (!c || !w || c->g.nx < 4) return EMHD_ERR_ARG;
  HaloPush P;
  P.lo = lo_halo;
  P.hi = hi_halo;
  P.n_top = 8LL * c->g.nx * c->g.ny;
  P.plane = (unsigned)((long long)c->g.nx * c->g.ny);
  P.nx = (unsigned)c->g.nx;
  P.ny = (unsigned)c->g.ny;
  if (P.n_top >= (1LL << 32)) return EMHD_ERR_ARG;
  return cerr(launch_push_edges(w, P, gate, c->stream));
}

extern "C" int emhd_update_finish(emhd_ctx* c, double* w, const double* V, long long ldv, int nvec,
                                  const double* h2, long long len_upd, long long len_dot,
                                  long long len_max, double* nrm, const double* h1,
                                  const double* selfdot, int j, double* H, long long ldh, double* scal,
                                  double* brk_hist) {
  if (!c || !w || !V || !h2 || !nrm || !h1 || !selfdot || !H || !scal || nvec < 1 ||
      nvec > c->max_vectors || j < 0)
    return EMHD_ERR_ARG;
  KWork k = kwork(c);
  FinishArgs F;
  F.h1 = h1; F.h2 = h2; F.selfdot = selfdot; F.j = j; F.H = H; F.ldh = ldh; F.scal = scal;
  F.brk_hist = brk_hist; F.st = c->st; F.rtol = 1e-12;
  Reorth ro{};
  ro.skip2 = take_skip(c);
  ProfScope ps(c, EMHD_K_UPDATE_FINISH, 8.0 * (nvec + 2) * (double)len_upd, ro.skip2);
  return cerr(launch_update(w, V, ldv, nvec, h2, len_upd, len_dot, len_max, 1, k, nrm, c->stream, F,
                            nullptr, ro));
}

extern "C" int emhd_norms(emhd_ctx* c, const double* x, long long len_sum, long long len_max, double* out) {
  if (!c || !x || !out) return EMHD_ERR_ARG;
  KWork k = kwork(c);
  ProfScope ps(c, EMHD_K_NORMS, 8.0 * (double)(len_sum > len_max ? len_sum : len_max));
  return cerr(launch_norms(x, len_sum, len_max, k, out, c->stream));
}

extern "C" int emhd_arnoldi_finish(emhd_ctx* c, const double* h1, const double* h2, const double* nrm,
                                   const double* selfdot, int j, double* H, long long ldh, double* scal,
                                   double* brk_hist) {
  if (!c || !h1 || !h2 || !nrm || !selfdot || !H || !scal || j < 0) return EMHD_ERR_ARG;
  return cerr(launch_arnoldi_finish(h1, h2, nrm, selfdot, j, H, ldh, scal, brk_hist, c->st, 1e-12,
                                    c->stream, take_skip(c)));
}

extern "C" int emhd_div_scalar(emhd_ctx* c, const double* x, const double* d, int take_sqrt, double* out,
                               double* d_out, long long n) {
  if (!c || !x || !d || !out) return EMHD_ERR_ARG;
  ProfScope ps(c, EMHD_K_DIV_SCALAR, 16.0 * (double)n);
  return cerr(launch_div_scalar(x, d, take_sqrt, out, d_out, n, c->num_sms, c->stream));
}

static int ensure_dense(emhd_ctx* c, size_t need) {
  if (need <= c->dense_len) return EMHD_OK;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cerr(e);
  cudaFree(c->dense);
  c->dense = nullptr;
  c->dense_len = 0;
  size_t want = need < (size_t)4 * 11 * 256 * 256 ? (size_t)4 * 11 * 256 * 256 + 4096 : need;
  e = cudaMalloc(&c->dense, want * sizeof(double));
  if (e != cudaSuccess) return cerr(e);
  c->dense_len = want;
  return EMHD_OK;
}

static void carve_dense(emhd_ctx* c, PhiSmallArgs& P, int S, size_t n) {
  const size_t per = dense_per(n);
  for (int s = 0; s < S; ++s) {
    double* b = c->dense + per * s;
    size_t nn = n * n;
    P.work[s].a = b;
    P.work[s].e = b + nn;
    for (int k = 0; k < 7; ++k) P.work[s].m[k] = b + (2 + k) * nn;
    P.work[s].m[7] = b + 9 * nn;     // n x 2n
    P.work[s].vec = b + 11 * nn;
    P.work[s].part = b + 11 * nn + 5 * n + 64;
  }
}

static int phi_small_impl(emhd_ctx* c, const double* H, long long ldh, int m, int order, int S,
                          const double* scales, const double* res_scale, const double* scal,
                          const double* beta, double* Y, double* res, double* E_out,
                          const double* host_scales = nullptr) {
  if (!c || !H || m < 1 || order < 0 || order > 4 || S < 1 || S > DENSE_MAX_SCALES ||
      (!host_scales && (!scales || !res_scale)) || !beta || !Y || !res)
    return EMHD_ERR_ARG;
  const size_t n = (size_t)m + order;
  const size_t per = dense_per(n);
  int rc = ensure_dense(c, per * S);
  if (rc) return rc;
  PhiSmallArgs P;
  std::memset(&P, 0, sizeof(P));
  P.H = H; P.ldh = ldh; P.m = m; P.order = order; P.scales = scales; P.res_scale = res_scale;
  P.scal = scal; P.beta = beta; P.Y = Y; P.res = res; P.st = c->st; P.E_out = E_out;
  if (host_scales) {
    P.scales_by_value = 1;
    for (int s = 0; s < S; ++s) { P.sv[s] = host_scales[s]; P.rv[s] = 1.0; }
  }
  carve_dense(c, P, S, n);
  return cerr(launch_phi_small(P, S, c->stream));
}

// Speculative residual checks: CTA s evaluates y_s = beta phi_order(scales[s] H_{ms[s]}) e1 and
// the raw residual |h_{m+1,m}| |y_m| / ||y|| for basis size ms[s] (host arrays), h_{m+1,m} read
// from H and zeroed by brk_hist[m-1]; Y rows of stride ldy.
extern "C" int emhd_phi_small_batch(emhd_ctx* c, const double* H, long long ldh, const int* ms, int order,
                                    int S, const double* host_scales, const double* brk_hist,
                                    const double* beta, double* Y, long long ldy, double* res) {
  if (!c || !H || !ms || !host_scales || !brk_hist || !beta || !Y || !res || S < 1 ||
      S > DENSE_MAX_SCALES || order < 0 || order > 4)
    return EMHD_ERR_ARG;
  int mmax = 0;
  for (int s = 0; s < S; ++s) {
    if (ms[s] < 1 || ms[s] > ldy) return EMHD_ERR_ARG;
    mmax = ms[s] > mmax ? ms[s] : mmax;
  }
  const size_t n = (size_t)mmax + order;
  const size_t per = dense_per(n);
  int rc = ensure_dense(c, per * S);
  if (rc) return rc;
  PhiSmallArgs P;
  std::memset(&P, 0, sizeof(P));
  P.H = H; P.ldh = ldh; P.m = mmax; P.order = order; P.beta = beta; P.Y = Y; P.res = res;
  P.st = c->st; P.batch = 1; P.brk_hist = brk_hist; P.ldy = ldy; P.scales_by_value = 1;
  for (int s = 0; s < S; ++s) { P.mb[s] = ms[s]; P.sv[s] = host_scales[s]; P.rv[s] = 1.0; }
  carve_dense(c, P, S, n);
  return cerr(launch_phi_small(P, S, c->stream));
}

extern "C" int emhd_phi_small(emhd_ctx* c, const double* H, long long ldh, int m, int order, int S,
                              const double* scales, const double* res_scale, const double* scal,
                              const double* beta, double* Y, double* res) {
  return phi_small_impl(c, H, ldh, m, order, S, scales, res_scale, scal, beta, Y, res, nullptr);
}

// scales given as a HOST array (no device scratch, no H2D copy); res[s] is the raw residual
extern "C" int emhd_phi_small_h(emhd_ctx* c, const double* H, long long ldh, int m, int order, int S,
                                const double* host_scales, const double* scal, const double* beta,
                                double* Y, double* res) {
  if (!host_scales) return EMHD_ERR_ARG;
  return phi_small_impl(c, H, ldh, m, order, S, nullptr, nullptr, scal, beta, Y, res, nullptr,
                        host_scales);
}

// Exponentials of dimension >= n run on a cluster of DENSE_CLUSTER CTAs (0: never); returns
// the previous setting.  Process-wide (default EMHD_DENSE_CLUSTER_N, else 56).
extern "C" int emhd_set_dense_cluster(int n) {
  const int prev = dense_cluster_min_n();
  set_dense_cluster_min_n(n);
  return prev;
}

// The linear solve of the Pade approximant: blocked Gauss-Jordan (8 pivot columns per step) for
// 24 <= n <= 128, or the unblocked solve everywhere (on = 0); returns the previous setting.
// Process-wide (default EMHD_DENSE_GJ_BLOCKED, else 1).
extern "C" int emhd_set_dense_gj_blocked(int on) {
  const int prev = dense_gj_blocked();
  set_dense_gj_blocked(on);
  return prev;
}

// E = expm(A) for an n x n device matrix (scratch: 4 doubles + n doubles in `work`)
extern "C" int emhd_expm(emhd_ctx* c, const double* A, int n, double* E, double* work) {
  if (!c || !A || !E || !work || n < 1) return EMHD_ERR_ARG;
  // work = {scale=1, res_scale=1, beta=1, res, Y[n]}
  double ones[3] = {1.0, 1.0, 1.0};
  int rc = cerr(cudaMemcpyAsync(work, ones, sizeof(ones), cudaMemcpyHostToDevice, c->stream));
  if (rc) return rc;
  rc = phi_small_impl(c, A, n, n, 0, 1, work, work + 1, nullptr, work + 2, work + 4, work + 3, E);
  if (!rc) rc = cerr(cudaStreamSynchronize(c->stream));
  return rc;
}

extern "C" int emhd_combine(emhd_ctx* c, const double* V, long long ldv, int m, const double* Y, int S,
                            const double* const* base, const double* coef, double* const* outs,
                            long long len) {
  if (!c || !V || !Y || S < 1 || S > 4 || m < 1 || !outs) return EMHD_ERR_ARG;
  CombineOut co;
  for (int s = 0; s < 4; ++s) {
    co.base[s] = (s < S && base) ? base[s] : nullptr;
    co.coef[s] = (s < S && coef) ? coef[s] : 1.0;
    co.out[s] = s < S ? outs[s] : nullptr;
  }
  return cerr(launch_combine(V, ldv, m, Y, S, co, len, c->num_sms, c->stream));
}

extern "C" int emhd_lincomb(emhd_ctx* c, int nterms, const double* const* x, const double* cc,
                            const int* has_c, double post, int has_post, double* out, long long n,
                            long long len_max, double* max_out) {
  if (!c || nterms < 1 || nterms > 6 || !x || !out) return EMHD_ERR_ARG;
  LinComb L;
  std::memset(&L, 0, sizeof(L));
  for (int k = 0; k < nterms; ++k) {
    if (!x[k]) return EMHD_ERR_ARG;
    L.x[k] = x[k];
    L.has_c[k] = has_c ? has_c[k] : 0;
    L.c[k] = cc ? cc[k] : 1.0;
  }
  L.nterms = nterms;
  L.post = post;
  L.has_post = has_post;
  L.out = out;
  return cerr(launch_lincomb(L, n, len_max, c->partials, max_out, c->ticket, c->num_sms, c->stream));
}

// out = base + post (x) (t_0 + t_1 + ...): the final stage update of explicit RK4
// (harness.py:194: y + (step / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4))
extern "C" int emhd_lincomb_onto(emhd_ctx* c, const double* base, int nterms, const double* const* x,
                                 const double* cc, const int* has_c, double post, int has_post,
                                 double* out, long long n) {
  if (!c || !base || nterms < 1 || nterms > 6 || !x || !out) return EMHD_ERR_ARG;
  LinComb L;
  std::memset(&L, 0, sizeof(L));
  for (int k = 0; k < nterms; ++k) {
    if (!x[k]) return EMHD_ERR_ARG;
    L.x[k] = x[k];
    L.has_c[k] = has_c ? has_c[k] : 0;
    L.c[k] = cc ? cc[k] : 1.0;
  }
  L.nterms = nterms;
  L.post = post;
  L.has_post = has_post;
  L.base = base;
  L.out = out;
  return cerr(launch_lincomb(L, n, 0, c->partials, nullptr, c->ticket, c->num_sms, c->stream));
}

extern "C" int emhd_wrms(emhd_ctx* c, const double* err, const double* y, double tol, long long n,
                         double* out) {
  if (!c || !err || !y || !out) return EMHD_ERR_ARG;
  return cerr(launch_wrms(err, y, tol, n, c->partials, out, c->ticket, c->num_sms, c->stream));
}

// {sum w^2, max|w|} of one rank -> slots {sum, 0.., max at 1 + rank, ..0}: ONE all-reduce SUM
// of 1 + P doubles then carries both the global sum and every rank's maximum (adding zeros
// is exact), instead of a SUM and a MAX collective per Arnoldi iteration
__global__ void slot_norms_kernel(const double* nrm, int rank, int nranks, double* slots) {
  for (int i = threadIdx.x; i <= nranks; i += blockDim.x)
    slots[i] = i == 0 ? nrm[0] : (i == 1 + rank ? nrm[1] : 0.0);
}

__global__ void unslot_norms_kernel(const double* slots, int nranks, double* nrm) {
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int r = 0; r < nranks; ++r) mx = fmax(mx, slots[1 + r]);
    nrm[0] = slots[0];
    nrm[1] = mx;
  }
}

extern "C" int emhd_slot_norms(emhd_ctx* c, const double* nrm, int rank, int nranks, double* slots) {
  if (!c || !nrm || !slots || nranks < 1 || rank < 0 || rank >= nranks) return EMHD_ERR_ARG;
  slot_norms_kernel<<<1, 32, 0, c->stream>>>(nrm, rank, nranks, slots);
  return cerr(cudaGetLastError());
}

extern "C" int emhd_unslot_norms(emhd_ctx* c, const double* slots, int nranks, double* nrm) {
  if (!c || !nrm || !slots || nranks < 1) return EMHD_ERR_ARG;
  unslot_norms_kernel<<<1, 32, 0, c->stream>>>(slots, nranks, nrm);
  return cerr(cudaGetLastError());
}

__global__ void pack_edges_kernel(const double* x, double* buf, int nx, int ny) {
  // buf[side][f][r][j]: side 0 = rows {0,1}, side 1 = rows {nx-2, nx-1}
  const long long total = 2LL * NF * 2 * ny;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e % ny);
    long long q = e / ny;
    const int r = (int)(q % 2); q /= 2;
    const int f = (int)(q % NF);
    const int side = (int)(q / NF);
    const int row = side == 0 ? r : nx - 2 + r;
    buf[e] = x[((long long)f * nx + row) * ny + j];
  }
}

extern "C" int emhd_pack_edges(emhd_ctx* c, const double* x, double* sendbuf) {
  if (!c || !x || !sendbuf) return EMHD_ERR_ARG;
  const long long total = 2LL * NF * 2 * c->g.ny;
  int G = (int)((total + 255) / 256);
  pack_edges_kernel<<<G, 256, 0, c->stream>>>(x, sendbuf, c->g.nx, c->g.ny);
  return cerr(cudaGetLastError());
}

// ---- snapshot layout / RK4 harness ----
extern "C" int emhd_cells_pack(emhd_ctx* c, const double* U, long long ncell, double* cells) {
  if (!c || !U || !cells || ncell < 0) return EMHD_ERR_ARG;
  return cerr(launch_cells_pack(U, ncell, cells, c->num_sms, c->stream));
}

extern "C" int emhd_cells_unpack(emhd_ctx* c, const double* cells, long long ncell, double* U) {
  if (!c || !U || !cells || ncell < 0) return EMHD_ERR_ARG;
  return cerr(launch_cells_unpack(cells, ncell, U, c->num_sms, c->stream));
}

extern "C" int emhd_max_signal_speed(emhd_ctx* c, const double* U, double* cmax) {
  if (!c || !U || !cmax) return EMHD_ERR_ARG;
  const long long ncell = (long long)c->g.nx * c->g.ny;
  const double gm1 = c->p.gamma - 1.0;
  const double bfac = c->p.b_half ? 0.5 : 1.0;
  return cerr(launch_signal_speed(U, ncell, c->p.gamma, gm1, bfac, cmax, c->st, c->num_sms, c->stream));
}

extern "C" int emhd_field_sqdiff(emhd_ctx* c, const double* U, const double* R, double* out) {
  if (!c || !U || !R || !out) return EMHD_ERR_ARG;
  const long long ncell = (long long)c->g.nx * c->g.ny;
  return cerr(launch_field_sqdiff(U, R, ncell, c->partials, (int)(c->partials_len / NF), out, c->num_sms,
                                  c->stream));
}

struct emhd_report_s { int which, i, j, pad; double value; };

// Admissibility diagnostics of the state a stencil call saw (error path only):
// which = 1 (density) / 2 (pressure) / 0, with the reference's padded-field
// argmin cell (mhd.py:111-131) and its value.
extern "C" int emhd_admissibility_report(emhd_ctx* c, int mode, const double* a, const double* a_halo,
                                         const double* v, const double* v_halo, const double* scal,
                                         void* report) {
  if (!c || !a || !report || mode < 0 || mode > 2) return EMHD_ERR_ARG;
  StencilParams P = c->base;
  P.epoch = c->epoch;
  P.a = a; P.a_halo = a_halo; P.v = v; P.v_halo = v_halo; P.scal = scal;
  // a halo exchanged inside the library (caller passed none) is the context's own buffer
  if (c->comm && mode == 0 && !P.a_halo) P.a_halo = c->hrecv;
  if (c->comm && mode != 0 && !P.v_halo) P.v_halo = c->hrecv;
  unsigned long long* keys = nullptr;
  int rc = cerr(cudaMalloc(&keys, 4 * sizeof(unsigned long long)));
  if (rc) return rc;
  unsigned long long init[4] = {~0ull, ~0ull, ~0ull, ~0ull};
  unsigned long long host[4];
  rc = cerr(cudaMemcpy(keys, init, sizeof(init), cudaMemcpyHostToDevice));
  if (!rc) rc = cerr(launch_admissibility(P, mode, keys, c->stream));
  if (!rc) rc = cerr(cudaStreamSynchronize(c->stream));
  if (!rc) rc = cerr(cudaMemcpy(host, keys, sizeof(host), cudaMemcpyDeviceToHost));
  cudaFree(keys);
  if (rc) return rc;
  auto val = [](unsigned long long k) {
    unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    double d;
    std::memcpy(&d, &b, sizeof(d));
    return d;
  };
  emhd_report_s* R = (emhd_report_s*)report;
  const int W = c->g.ny + 4;
  R->which = 0; R->i = R->j = -1; R->pad = 0; R->value = 0.0;
  const double rmin = val(host[0]), pmin = val(host[1]);
  if (host[0] != ~0ull && rmin <= 0.0 && c->p.check) {
    R->which = 1; R->i = (int)(host[2] / W); R->j = (int)(host[2] % W); R->value = rmin;
  } else if (host[1] != ~0ull && pmin <= 0.0 && c->p.check) {
    R->which = 2; R->i = (int)(host[3] / W); R->j = (int)(host[3] % W); R->value = pmin;
  }
  if (R->which && c->g.x_offset) R->i += c->g.x_offset;
  return EMHD_OK;
}

// ---- single-rank Arnoldi driver: one C call per iteration ---------------------------
struct emhd_arnoldi_args_s {
  const double* a; const double* fa;
  double* V; long long ldv;
  double* H; long long ldh;
  double* w0; double* w1;
  double* d1; double* d2; double* nrm; double* vn; double* scal; double* brk;
  long long n_top; long long len_dot; long long len_upd;
  int p; int nb; double ch;
  const double* bcol[5]; int bidx[5];
  int gen;             // process generation (look-ahead cancellation)
  double* gate;        // [m_cap + 1] per-iteration gates (look-ahead launches)
  double* evals;       // [m_cap + 1] 1 where iteration j evaluated the RHS (or null)
  double eta;          // selective re-orthogonalisation threshold (<= 0: always two passes)
  double* reorth;      // [m_cap + 1] 1 where iteration j skipped the second pass
  double* md2;         // [m_cap + 1] (or null) 0 where iteration j needed a separate pass-2
                       // multi-dot (pass 2 ran although the re-projection was predicted away)
  const double* a_halo;  // slab ranks: x-halo of a (exchanged once per operator)
};

// Iteration j of krylov.py:144-168 on one rank: (normalise w_{j-1} +) Jv, pass-1 multi-dot with
// the breakdown scale, update + re-projection, update + norms + column bookkeeping.  Writes
// w_{j} into w0/w1 (j even/odd) and V[j] (j > 0), H[:, j], scal, brk[j].
// Iteration j on a slab rank (context with a communicator): the same kernels as the
// single-rank iteration below, with the reductions of krylov.py:151,153,158,161 all-reduced in
// between (stream-ordered NCCL, no host sync) and the x-halo of the vector the stencil
// perturbs exchanged while the stencil's interior rows run.  The selective re-orthogonalisation
// decision is taken by a one-CTA kernel from the all-reduced sums, so every rank takes the same
// branch; the pass-2 launches test its gate, the pass-2 norm all-reduce is issued regardless
// (unused when skipped).  The re-projection dots are predicted as on one rank (args.md2): pass 1
// skips them after two iterations without a second pass, and a gated multi-dot (plus its
// all-reduce, issued regardless) supplies them on a misprediction.
__global__ void gated_copy_kernel(const double* src, double* dst, int n, const double* gate) {
  if (*gate != 0.0) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

static int arnoldi_iter_slab(emhd_ctx* c, const emhd_arnoldi_args_s* A, int j) {
  double* out = (j % 2 == 0) ? A->w0 : A->w1;
  const double W = 8.0 * (double)A->n_top;
  StencilParams P = c->base;
  P.epoch = j;
  P.evals = A->evals ? A->evals + j : nullptr;
  P.a = A->a; P.fa = A->fa; P.out = out;
  P.a_halo = A->a_halo;
  set_epilogue(P, A->p, A->ch, A->nb, A->bcol, A->bidx);
  KWork k = kwork(c);
  int rc;
  if (j == 0) {
    {
      ProfScope ps(c, EMHD_K_NORMS, W);
      rc = cerr(launch_norms(A->V, 0, A->n_top, k, A->vn, c->stream));
    }
    if (!rc) rc = comm_rc(slabcomm_allreduce(c->comm, A->vn + 1, 1, EMHD_OP_MAX, c->stream));
    if (rc) return rc;
    P.v = A->V; P.scal = A->vn + 1;
    if (A->p > 0) P.qsrc = A->V + A->n_top;
    ProfScope ps(c, EMHD_K_JV, 4.0 * W);
    rc = stencil_with_halo(c, P, MODE_JV, A->p > 0, A->V, false);
  } else {
    P.v = (j % 2 == 0) ? A->w1 : A->w0;
    P.scal = A->scal;
    P.vout = A->V + (size_t)j * A->ldv;
    ProfScope ps(c, EMHD_K_JV_NORMALIZED, 5.0 * W);
    rc = stencil_with_halo(c, P, MODE_JVN, A->p > 0, P.v, false);
  }
  if (rc) return rc;
  const int nv = j + 1;
  FinishArgs F;
  F.h1 = A->d1; F.h2 = A->d2; F.selfdot = A->d1 + nv; F.j = j; F.H = A->H; F.ldh = A->ldh;
  F.scal = A->scal; F.brk_hist = A->brk; F.st = c->st; F.rtol = 1e-12;
  const double vb = 8.0 * (double)A->len_upd;
  const bool selective = A->eta > 0.0 && A->reorth;
  // pass 1: h1 = V^T w and ||w||^2 (the breakdown scale)
  {
    ProfScope ps(c, EMHD_K_MULTIDOT, (nv + 1) * vb);
    rc = cerr(launch_multidot(out, A->V, A->ldv, nv, A->len_dot, 1, k, A->d1, c->stream));
  }
  if (!rc) rc = comm_rc(slabcomm_allreduce(c->comm, A->d1, nv + 1, EMHD_OP_SUM, c->stream));
  // w -= V h1 with the re-projection dots h2 = V^T w1 (unless predicted away), ||w1||^2 (SUM) and
  // max|w1_top| (MAX)
  Reorth r1{};
  double* md2 = nullptr;
  const double* predict = nullptr;
  if (selective && A->md2) {
    md2 = A->md2 + j;
    predict = j > 1 ? A->reorth + (j - 2) : nullptr;
    r1.predict = predict;
  }
  if (!rc) {
    ProfScope ps(c, EMHD_K_UPDATE, (nv + 2) * vb);
    rc = cerr(launch_update(out, A->V, A->ldv, nv, A->d1, A->len_upd, A->len_dot, A->n_top, 0, k,
                            A->d2, c->stream, F, nullptr, r1));
  }
  if (!rc) rc = comm_rc(slabcomm_allreduce_sum_max(c->comm, A->d2, nv + 1, 1, c->stream));
  if (rc) return rc;
  const double* gate = nullptr;
  if (selective) {
    gate = A->reorth + j;
    rc = cerr(launch_reorth_decide(F, A->d2, nv, A->eta * A->eta, A->reorth + j, c->stream, md2, predict));
    if (!rc && md2) {
      // misprediction: pass 2 needed but its dots were not computed (gate md2 == 0): a gated
      // multi-dot into scratch, its all-reduce (issued on every rank regardless of the gate),
      // then the gated copy into h2 (the all-reduced d2 must not be reduced twice)
      ProfScope ps(c, EMHD_K_MULTIDOT2, (nv + 1) * vb, md2);
      rc = cerr(launch_multidot(out, A->V, A->ldv, nv, A->len_dot, 0, k, c->red, c->stream, nullptr, md2));
      if (!rc) rc = comm_rc(slabcomm_allreduce(c->comm, c->red, nv, EMHD_OP_SUM, c->stream));
      if (!rc) {
        gated_copy_kernel<<<1, 128, 0, c->stream>>>(c->red, A->d2, nv, md2);
        rc = cerr(cudaGetLastError());
      }
    }
    if (rc) return rc;
  }
  // pass 2 (gated): w -= V h2 ; {||w||^2, max|w_top|} all-reduced ; column bookkeeping
  Reorth r2{};
  r2.skip2 = gate;
  {
    ProfScope ps(c, EMHD_K_UPDATE_FINISH, (nv + 2) * vb, gate);
    rc = cerr(launch_update(out, A->V, A->ldv, nv, A->d2, A->len_upd, A->len_dot, A->n_top, 1, k,
                            A->nrm, c->stream, FinishArgs{}, nullptr, r2));
  }
  if (!rc) rc = comm_rc(slabcomm_allreduce_sum_max(c->comm, A->nrm, 1, 1, c->stream));
  if (!rc) rc = cerr(launch_arnoldi_finish(A->d1, A->d2, A->nrm, A->d1 + nv, j, A->H, A->ldh, A->scal,
                                           A->brk, c->st, 1e-12, c->stream, gate));
  return rc;
}

static int arnoldi_iter(emhd_ctx* c, const void* args, int j, bool gated) {
  if (!c || !args || j < 0) return EMHD_ERR_ARG;
  const emhd_arnoldi_args_s* A = (const emhd_arnoldi_args_s*)args;
  if (j + 1 > c->max_vectors || (gated && !A->gate)) return EMHD_ERR_ARG;
  // the iteration's stencil carries epoch j (P.epoch below); the context's own epoch is left
  // alone, so later RHS / Jv launches are never mistaken for a discarded speculative iteration
  if (c->comm) {
    // slab ranks: no look-ahead (a device-side cancellation could differ between ranks while
    // their collectives must match one to one)
    if (gated) return EMHD_ERR_ARG;
    return arnoldi_iter_slab(c, A, j);
  }
  double* out = (j % 2 == 0) ? A->w0 : A->w1;
  const double* skip = nullptr;
  const double W = 8.0 * (double)A->n_top;
  if (gated) {
    ProfScope ps(c, EMHD_K_GATE, 0.0);
    const int rc0 = cerr(launch_gate(c->cancel, (unsigned)A->gen, j, A->gate + j, c->stream));
    if (rc0) return rc0;
    skip = A->gate + j;
  }
  StencilParams P = c->base;
  P.epoch = j;
  P.skip = skip;
  P.evals = A->evals ? A->evals + j : nullptr;
  P.a = A->a; P.fa = A->fa; P.out = out;
  set_epilogue(P, A->p, A->ch, A->nb, A->bcol, A->bidx);
  KWork k = kwork(c);
  int rc;
  if (j == 0) {
    if (gated) return EMHD_ERR_ARG;
    // sigma of the seed direction: max|V[0][:n]| into vn[1] (norms writes {sum, max})
    {
      ProfScope ps(c, EMHD_K_NORMS, W);
      rc = cerr(launch_norms(A->V, 0, A->n_top, k, A->vn, c->stream));
    }
    if (rc) return rc;
    P.v = A->V; P.scal = A->vn + 1;
    if (A->p > 0) P.qsrc = A->V + A->n_top;
    ProfScope ps(c, EMHD_K_JV, 4.0 * W);
    rc = cerr(launch_stencil(P, MODE_JV, A->p > 0, c->num_sms, c->stream, c->path, &c->last));
  } else {
    P.v = (j % 2 == 0) ? A->w1 : A->w0;
    P.scal = A->scal;
    P.vout = A->V + (size_t)j * A->ldv;
    ProfScope ps(c, EMHD_K_JV_NORMALIZED, 5.0 * W, skip);
    rc = cerr(launch_stencil(P, MODE_JVN, A->p > 0, c->num_sms, c->stream, c->path, &c->last));
  }
  if (rc) return rc;
  const int nv = j + 1;
  FinishArgs F;
  F.h1 = A->d1; F.h2 = A->d2; F.selfdot = A->d1 + nv; F.j = j; F.H = A->H; F.ldh = A->ldh;
  F.scal = A->scal; F.brk_hist = A->brk; F.st = c->st; F.rtol = 1e-12;
  // pass 1 (multi-dot, update + re-projection + norms); with eta > 0 its last CTA decides
  // whether pass 2 is needed (selective re-orthogonalisation) and, if not, finishes the column
  // With md2 gates the re-projection dots are predicted from the previous iteration's decision:
  // if it skipped pass 2, this pass 1 computes only ||w1|| and max|w1| (no second read of the
  // basis), and a gated multi-dot supplies h2 in the (rare) case pass 2 turns out to be needed.
  Reorth r1{}, r2{};
  const double* md2 = nullptr;
  if (A->eta > 0.0 && A->reorth) {
    r1.eta2 = A->eta * A->eta;
    r1.gate_out = A->reorth + j;
    r2.skip2 = A->reorth + j;
    if (A->md2) {
      md2 = A->md2 + j;
      r1.gate_md2 = A->md2 + j;
      r1.predict = j > 1 ? A->reorth + (j - 2) : nullptr;   // both previous decisions: skip
    }
  }
  const double vb = 8.0 * (double)A->len_upd;
  if (c->fused_orth && orth_small_fits(A->len_upd, c->num_sms)) {
    // small grids: multi-dot, update, decision and (when needed) the second pass in ONE launch
    // (grid barriers between the phases; bit-identical to the separate launches below)
    Reorth r = r1;
    ProfScope ps(c, EMHD_K_MULTIDOT, (2 * nv + 3) * vb, skip);
    return cerr(launch_orth_small(out, A->V, A->ldv, nv, A->len_upd, A->len_dot, A->n_top, k,
                                  c->partials + c->partials_len / 2, c->ticket + 4, A->d1, A->d2,
                                  A->nrm, c->stream, F, skip, r));
  }
  {
    ProfScope ps(c, EMHD_K_MULTIDOT, (nv + 1) * vb, skip);
    rc = cerr(launch_multidot(out, A->V, A->ldv, nv, A->len_dot, 1, k, A->d1, c->stream, skip));
  }
  if (!rc) {
    ProfScope ps(c, EMHD_K_UPDATE, (nv + 2) * vb, skip);
    rc = cerr(launch_update(out, A->V, A->ldv, nv, A->d1, A->len_upd, A->len_dot, A->n_top, 0, k,
                            A->d2, c->stream, F, skip, r1));
  }
  if (!rc && md2) {
    ProfScope ps(c, EMHD_K_MULTIDOT2, (nv + 1) * vb, skip, md2);
    rc = cerr(launch_multidot(out, A->V, A->ldv, nv, A->len_dot, 0, k, A->d2, c->stream, skip, md2));
  }
  if (rc) return rc;
  ProfScope ps(c, EMHD_K_UPDATE_FINISH, (nv + 2) * vb, skip, r2.skip2);
  return cerr(launch_update(out, A->V, A->ldv, nv, A->d2, A->len_upd, A->len_dot, A->n_top, 1, k,
                            A->nrm, c->stream, F, skip, r2));
}

// Per-launch profiling of the Arnoldi path (emhd_arnoldi_iter / _run / _lookahead and the
// emhd_jv / emhd_norms / emhd_div_scalar entry points): enable != 0 clears and starts it.
extern "C" int emhd_profile(emhd_ctx* c, int enable) {
  if (!c) return EMHD_ERR_ARG;
  prof_clear(c);
  c->prof = enable != 0;
  return EMHD_OK;
}

// Synchronises the stream, then returns the records so far (at most max_n; kinds EMHD_K_*,
// milliseconds, algorithmic bytes — 0 for a launch its device gate turned into a no-op) and
// clears them.  Return value: number of records written (negative: error code).
extern "C" int emhd_profile_read(emhd_ctx* c, int max_n, int* kinds, double* ms, double* bytes) {
  if (!c || max_n < 0 || (max_n > 0 && (!kinds || !ms || !bytes))) return -EMHD_ERR_ARG;
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return -EMHD_ERR_CUDA;
  int n = 0;
  for (auto& r : c->recs) {
    if (n >= max_n) break;
    float t = 0.f;
    cudaEventElapsedTime(&t, r.e0, r.e1);
    double by = r.bytes;
    for (int g = 0; g < 2; ++g) {
      if (!r.gate[g]) continue;
      double v = 0.0;
      cudaMemcpy(&v, r.gate[g], sizeof(double), cudaMemcpyDeviceToHost);
      if (v != 0.0) by = 0.0;
    }
    kinds[n] = r.kind; ms[n] = t; bytes[n] = by;
    ++n;
  }
  prof_clear(c);
  return n;
}

extern "C" int emhd_arnoldi_iter(emhd_ctx* c, const void* args, int j) {
  return arnoldi_iter(c, args, j, false);
}

// Look-ahead iterations (queued while residual checks run elsewhere): each is gated on the
// context's cancel word, so the ones still queued when emhd_arnoldi_cancel lands do no work.
extern "C" int emhd_arnoldi_lookahead(emhd_ctx* c, const void* args, int j_begin, int j_end) {
  for (int j = j_begin; j < j_end; ++j) {
    const int rc = arnoldi_iter(c, args, j, true);
    if (rc) return rc;
  }
  return EMHD_OK;
}

// Cancel look-ahead iterations j >= epoch_min of process generation gen: an async 8-byte copy
// on the context's current stream (issue it on an idle stream so it lands at once).
extern "C" int emhd_arnoldi_cancel(emhd_ctx* c, int gen, int epoch_min) {
  if (!c || epoch_min < 0) return EMHD_ERR_ARG;
  *c->cancel_host = ((unsigned long long)(unsigned)gen << 32) | (unsigned)epoch_min;
  return cerr(cudaMemcpyAsync(c->cancel, c->cancel_host, sizeof(unsigned long long),
                              cudaMemcpyHostToDevice, c->stream));
}

// rhs_evals -= sum(evals[0:count]) in stream order (discarded speculative iterations)
extern "C" int emhd_evals_discount(emhd_ctx* c, const double* evals, int count) {
  if (!c || !evals || count < 0) return EMHD_ERR_ARG;
  if (count == 0) return EMHD_OK;
  return cerr(launch_evals_discount(evals, count, c->st, c->stream));
}

// One sync point: host_out[0:nbrk] = brk[0:nbrk], host_out[nbrk:nbrk+nres] = res[0:nres]
// (host_out should be pinned), then the status word; returns after the stream drained.
extern "C" int emhd_readback(emhd_ctx* c, const double* brk, int nbrk, const double* res, int nres,
                             double* host_out, emhd_status* st) {
  if (!c || !host_out || !st || nbrk < 0 || nres < 0) return EMHD_ERR_ARG;
  int rc = 0;
  if (nbrk > 0) rc = cerr(cudaMemcpyAsync(host_out, brk, sizeof(double) * nbrk, cudaMemcpyDeviceToHost,
                                          c->stream));
  if (!rc && nres > 0)
    rc = cerr(cudaMemcpyAsync(host_out + nbrk, res, sizeof(double) * nres, cudaMemcpyDeviceToHost,
                              c->stream));
  if (rc) return rc;
  return emhd_status_read(c, st);
}

// div B (mhd.py:288-296): d[nx*ny] and *dmax = max |d| (device scalar, overwritten)
extern "C" int emhd_div_b(emhd_ctx* c, const double* U, const double* U_halo, double* d, double* dmax) {
  if (!c || !U || !d || !dmax) return EMHD_ERR_ARG;
  StencilParams P = c->base;
  P.a = U; P.a_halo = U_halo;
  int rc = cerr(cudaMemsetAsync(dmax, 0, sizeof(double), c->stream));
  if (!rc) rc = cerr(launch_diag(P, 0, d, (unsigned long long*)dmax, c->stream));
  return rc;
}

// J = curl B (mhd.py:299-309): J[3][nx][ny]
extern "C" int emhd_current_j(emhd_ctx* c, const double* U, const double* U_halo, double* J) {
  if (!c || !U || !J) return EMHD_ERR_ARG;
  StencilParams P = c->base;
  P.a = U; P.a_halo = U_halo;
  return cerr(launch_diag(P, 1, J, nullptr, c->stream));
}

// Iterations j_begin .. j_end-1 back to back (the m_init burst / a speculative batch)
extern "C" int emhd_arnoldi_run(emhd_ctx* c, const void* args, int j_begin, int j_end) {
  for (int j = j_begin; j < j_end; ++j) {
    const int rc = emhd_arnoldi_iter(c, args, j);
    if (rc) return rc;
  }
  return EMHD_OK;
}
