// Arnoldi building blocks: deterministic multi-dot, fused update + re-dot,
// fused update + norm, basis combination (V y) and norms.
//
// Replaces reference pkg/src/expmhd/krylov.py:144-168 (_ArnoldiProcess.extend:
// MGS pass + re-orthogonalisation pass + norm + normalisation) and the
// V_m @ y products at krylov.py:316,374.  The orthogonalisation is classical
// Gram–Schmidt applied twice (CGS2): the same projector as the reference's
// MGS2 to round-off, but each pass is ONE sweep over the basis instead of j+1
// dependent dot/axpy sweeps, so an iteration costs (3j+~12) vector reads and
// three grid reductions.
//
// Reductions are deterministic: every CTA reduces its own elements in a fixed
// order into a per-CTA partial, and the last CTA to finish (threadfence +
// ticket) sums the partials in CTA order.  No floating-point atomics.
#include <cstdlib>
#include "emhd_common.cuh"
#include "krylov.cuh"

namespace emhd {

bool pdl_on() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("EMHD_PDL");
    on = e ? (atoi(e) != 0 ? 1 : 0) : 1;
  }
  return on != 0;
}

constexpr int KT = 256;          // threads per CTA
constexpr int EPT = 2;           // elements per double2
constexpr int TILE = KT * EPT;   // 512 elements per combine tile
constexpr int NWARP = KT / 32;

static int grid_for_len(long long len, int tile, int num_sms);

// Last-CTA deterministic reduction of partials[nval][G] -> out[nval].
// kind[v]: 0 = sum, 1 = max.  Returns true in the CTA that did it.
__device__ bool finish_partials(const double* partials, int nval, int G, const int* kinds,
                                double* out, unsigned int* ticket) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(ticket, 1u);
    last = (prev == (unsigned)G - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int v = warp; v < nval; v += NWARP) {
    const bool mx = kinds && kinds[v] == 1;
    double acc = mx ? 0.0 : 0.0;
    for (int c = lane; c < G; c += 32) {
      const double x = __ldcg(partials + (size_t)v * G + c);
      acc = mx ? fmax(acc, x) : acc + x;
    }
    acc = mx ? warp_max(acc) : warp_sum(acc);
    if (lane == 0) out[v] = acc;
  }
  if (threadIdx.x == 0) *ticket = 0u;     // re-arm for the next launch
  return true;
}

// finish_partials with value max_idx reduced by max, all others by sum
// (values below v_begin are known to be zero in every CTA: written as 0 without reading them)
__device__ bool finish_partials_maxidx(const double* partials, int nval, int G, int max_idx,
                                       double* out, unsigned int* ticket, int v_begin = 0) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(ticket, 1u);
    last = (prev == (unsigned)G - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int v = threadIdx.x; v < v_begin; v += KT) out[v] = 0.0;
  for (int v = v_begin + warp; v < nval; v += NWARP) {
    const bool mx = v == max_idx;
    double acc = 0.0;
    for (int c = lane; c < G; c += 32) {
      const double x = __ldcg(partials + (size_t)v * G + c);
      acc = mx ? fmax(acc, x) : acc + x;
    }
    acc = mx ? warp_max(acc) : warp_sum(acc);
    if (lane == 0) out[v] = acc;
  }
  if (threadIdx.x == 0) *ticket = 0u;     // re-arm for the next launch
  return true;
}

// per-warp slot accumulation of one double per vector, then CTA partial
__device__ __forceinline__ void cta_store_partials(double* s_acc, int nval, double* partials, int G) {
  __syncthreads();
  for (int v = threadIdx.x; v < nval; v += KT) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) acc += s_acc[v * NWARP + w];
    partials[(size_t)v * G + blockIdx.x] = acc;
  }
}

__device__ __forceinline__ double2 ld2(const double* p, long long e, long long len) {
  if (e + 1 < len) return __ldg(reinterpret_cast<const double2*>(p + e));
  double2 r = make_double2(0.0, 0.0);
  if (e < len) r.x = __ldg(p + e);
  return r;
}
__device__ __forceinline__ double2 ld2_stream(const double* p, long long e, long long len) {
  if (e + 1 < len) return __ldcs(reinterpret_cast<const double2*>(p + e));
  double2 r = make_double2(0.0, 0.0);
  if (e < len) r.x = __ldcs(p + e);
  return r;
}

// out[i] = <w, V_i>, i < nvec (over len_dot); optional out[nvec] = <w, w>.
// Each thread streams VEC double2 of w per tile and U basis vectors per step
// (2*VEC*U independent 16-byte loads in flight); per (tile, vector) one warp
// shuffle-reduction into a per-warp shared slot; deterministic CTA partials.
template <int VEC, int U>
__global__ void __launch_bounds__(KT, 4) multidot_kernel(const double* __restrict__ w,
    const double* __restrict__ V, long long ldv, int nvec, long long len_dot, int self,
    double* partials, double* out, unsigned int* ticket, const double* skip, const double* skip2) {
  pdl_sync();
  if (skip && *skip != 0.0) return;            // cancelled look-ahead iteration (all CTAs agree)
  if (skip2 && *skip2 != 0.0) return;          // gated second-pass multi-dot not needed
  extern __shared__ double s_acc[];            // [(nvec+1)][NWARP]
  constexpr int TL = KT * 2 * VEC;
  const int nval = nvec + self;
  for (int k = threadIdx.x; k < nval * NWARP; k += KT) s_acc[k] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double selfacc = 0.0;
  const long long ntiles = (len_dot + TL - 1) / TL;
  for (long long tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const long long e0 = tl * TL + 2LL * threadIdx.x;
    double2 wv[VEC];
#pragma unroll
    for (int s = 0; s < VEC; ++s) {
      wv[s] = ld2_stream(w, e0 + (long long)s * 2 * KT, len_dot);
      selfacc = fma(wv[s].x, wv[s].x, fma(wv[s].y, wv[s].y, selfacc));
    }
    for (int i = 0; i < nvec; i += U) {
      double2 x[U][VEC];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int s = 0; s < VEC; ++s)
          x[u][s] = (i + u < nvec) ? ld2_stream(V + (size_t)(i + u) * ldv, e0 + (long long)s * 2 * KT, len_dot)
                                   : make_double2(0.0, 0.0);
      double d[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        d[u] = 0.0;
#pragma unroll
        for (int s = 0; s < VEC; ++s) d[u] = fma(wv[s].x, x[u][s].x, fma(wv[s].y, x[u][s].y, d[u]));
      }
      warp_reduce_multi<U>(d, lane);
      if ((lane & (32 / U - 1)) == 0) {
        const int u = multi_index<U>(lane);
        if (i + u < nvec) s_acc[(i + u) * NWARP + warp] += d[0];
      }
    }
  }
  if (self) {
    selfacc = warp_sum(selfacc);
    if (lane == 0) s_acc[nvec * NWARP + warp] = selfacc;
  }
  cta_store_partials(s_acc, nval, partials, gridDim.x);
  finish_partials(partials, nval, gridDim.x, nullptr, out, ticket);
}

// w[0:len_upd] -= sum_i h[i] V_i ; MODE 0: out[i] = <w_new, V_i> over len_dot (the
// CGS2 re-projection; the second read of each V tile hits L1/L2, not DRAM);
// MODE 1: out = {sum w^2 over len_dot, max|w| over len_max}.
__device__ __forceinline__ void finish_column(const FinishArgs& F, const double* nrm) {
  // krylov.py:161-166: H[:j+1, j] = h1 + h2, hnext = ||w||, breakdown test, scal for the next Jv
  for (int i = threadIdx.x; i <= F.j; i += blockDim.x)
    F.H[(size_t)i * F.ldh + F.j] = F.h2 ? F.h1[i] + F.h2[i] : F.h1[i];   // h2 null: pass 2 skipped
  if (threadIdx.x == 0) {
    const double hnext = sqrt(nrm[0]);
    const double scale = sqrt(F.selfdot[0]);
    // sticky: an iteration queued after a breakdown works on an unwritten basis row (its
    // normalised Jv launch did nothing), so whatever it computes must keep the flag raised
    const bool brk = (F.j > 0 && F.scal[2] != 0.0) || hnext <= F.rtol * fmax(scale, 1.0);
    if (brk) F.st->breakdown = 1;
    else F.H[(size_t)(F.j + 1) * F.ldh + F.j] = hnext;
    F.scal[0] = hnext;
    F.scal[1] = nrm[1];
    F.scal[2] = brk ? 1.0 : 0.0;
    if (F.brk_hist) F.brk_hist[F.j] = brk ? 1.0 : 0.0;
  }
}

// Selective re-orthogonalisation (Daniel-Gragg-Kaufman-Stewart): after pass 1, w1 = w - V h1
// with r[nvec] = ||w1||^2 and r[nvec+1] = max|w1_top|.  When ||w1|| >= eta ||w|| the first
// projection already left w1 orthogonal to the basis to working precision (its error is
// O(eps ||w||) <= O(eps ||w1|| / eta)), so the column is finished with h1 and the second
// sweep is skipped; otherwise the reference's second pass runs.  Called by one CTA.
__device__ void reorth_decide(const FinishArgs& F, const double* r, int nvec, double eta2, double* gate,
                              double* gate_md2 = nullptr, bool reprojected = true) {
  __shared__ int s_skip;
  if (threadIdx.x == 0) {
    s_skip = r[nvec] >= eta2 * F.selfdot[0] ? 1 : 0;
    *gate = s_skip ? 1.0 : 0.0;
    if (gate_md2) *gate_md2 = (s_skip || reprojected) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (s_skip) {
    FinishArgs F1 = F;
    F1.h2 = nullptr;
    finish_column(F1, r + nvec);
  }
}

// Halo push (slab ranks): store a final w element that lies in rows {0,1} / {nx-2,nx-1} of
// its field straight into the lo / hi neighbour's halo buffer (peer memory over NVLink);
// layout [2 sides][8][2 rows][ny], our low rows land in the lo neighbour's side 1, our high
// rows in the hi neighbour's side 0 (what Comm.exchange delivers).
__device__ __forceinline__ void push_edge(const HaloPush& H, long long e, double val) {
  if (e >= H.n_top) return;
  const unsigned eu = (unsigned)e;
  const unsigned f = eu / H.plane;
  const unsigned q = eu - f * H.plane;
  const unsigned row = q / H.ny;
  const unsigned col = q - row * H.ny;
  if (H.lo && row < 2) H.lo[((size_t)(NF + f) * 2 + row) * H.ny + col] = val;
  if (H.hi && row + 2 >= H.nx) H.hi[((size_t)f * 2 + (row + 2 - H.nx)) * H.ny + col] = val;
}

template <int MODE, int U, bool PUSH = false, bool CS = false>
__global__ void __launch_bounds__(KT, 4) update_kernel(double* __restrict__ w,
    const double* __restrict__ V, long long ldv, int nvec, const double* __restrict__ h,
    long long len_upd, long long len_dot, long long len_max,
    double* partials, double* out, unsigned int* ticket, const FinishArgs fin,
    const HaloPush push = HaloPush{}, const double* skip = nullptr, const Reorth ro = Reorth{}) {
  pdl_sync();
  if (skip && *skip != 0.0) return;            // cancelled look-ahead iteration (all CTAs agree)
  if (ro.skip2 && *ro.skip2 != 0.0) return;    // pass 2 not needed (decided by pass 1)
  // mode 0: the CGS2 re-projection dots, unless the previous iteration's decision predicts
  // that pass 2 will be skipped again (then only ||w1|| and max|w1| are needed)
  const bool reproj = MODE == 0 && !(ro.predict && ro.predict[0] != 0.0 && ro.predict[1] != 0.0);
  extern __shared__ double sm[];
  constexpr int TL = KT * 2;
  double* s_h = sm;                              // [nvec]
  double* s_acc = sm + ((nvec + 1) & ~1);        // [(nvec + 2 or 2)][NWARP]
  const int nval = MODE == 0 ? nvec + 2 : 2;
  for (int k = threadIdx.x; k < nvec; k += KT) s_h[k] = h[k];
  for (int k = threadIdx.x; k < nval * NWARP; k += KT) s_acc[k] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double ss = 0.0, mx = 0.0;
  const long long ntiles = (len_upd + TL - 1) / TL;
  for (long long k = blockIdx.x; k < ntiles; k += gridDim.x) {
    // last tile first: the multi-dot just streamed the vectors front to back, so their tail
    // is what the L2 still holds
    const long long tl = ntiles - 1 - k;
    const long long e = tl * TL + 2LL * threadIdx.x;
    const bool full = e + 1 < len_upd;
    double2 wv = ld2(w, e, len_upd);
    for (int i = 0; i < nvec; i += U) {
      double2 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        x[u] = (i + u < nvec) ? (CS ? ld2_stream(V + (size_t)(i + u) * ldv, e, len_upd)
                                    : ld2(V + (size_t)(i + u) * ldv, e, len_upd))
                              : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i + u < nvec) {
          const double hh = s_h[i + u];
          wv.x = fma(-hh, x[u].x, wv.x);
          wv.y = fma(-hh, x[u].y, wv.y);
        }
      }
    }
    if (full) *reinterpret_cast<double2*>(w + e) = wv;
    else if (e < len_upd) w[e] = wv.x;
    if (PUSH) {
      push_edge(push, e, wv.x);
      if (full) push_edge(push, e + 1, wv.y);
    }
    const double dx = (e < len_dot) ? wv.x : 0.0, dy = (e + 1 < len_dot) ? wv.y : 0.0;
    if (reproj) {
      // re-read the basis newest-first: the vectors just streamed by the update are the
      // likeliest to still sit in L1/L2 (halves the mean reuse distance of the tile)
      for (int i = (nvec - 1) / U * U; i >= 0; i -= U) {
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          x[u] = (i + u < nvec) ? ld2_stream(V + (size_t)(i + u) * ldv, e, len_upd) : make_double2(0.0, 0.0);
        double d[U];
#pragma unroll
        for (int u = 0; u < U; ++u) d[u] = fma(dx, x[u].x, dy * x[u].y);
        warp_reduce_multi<U>(d, lane);
        if ((lane & (32 / U - 1)) == 0) {
          const int u = multi_index<U>(lane);
          if (i + u < nvec) s_acc[(i + u) * NWARP + warp] += d[0];
        }
      }
    }
    // ||w||^2 and max|w_top| of the updated vector (mode 0: the selective re-orthogonalisation
    // test and, when pass 2 is skipped, the next sigma; mode 1: hnext and the next sigma)
    ss = fma(dx, dx, fma(dy, dy, ss));
    const double mxx = (e < len_max) ? fabs(wv.x) : 0.0;
    const double mxy = (e + 1 < len_max) ? fabs(wv.y) : 0.0;
    mx = fmax(mx, fmax(mxx, mxy));
  }
  if (PUSH) __threadfence_system();   // peer stores visible before the ordering collective
  if (MODE == 1) {
    ss = warp_sum(ss);
    mx = warp_max(mx);
    if (lane == 0) { s_acc[0 * NWARP + warp] = ss; s_acc[1 * NWARP + warp] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0, b = 0.0;
      for (int q = 0; q < NWARP; ++q) { a += s_acc[q]; b = fmax(b, s_acc[NWARP + q]); }
      partials[blockIdx.x] = a;
      partials[(size_t)gridDim.x + blockIdx.x] = b;
    }
    __shared__ int kinds_s[2];
    if (threadIdx.x == 0) { kinds_s[0] = 0; kinds_s[1] = 1; }
    __syncthreads();
    const bool last = finish_partials(partials, 2, gridDim.x, kinds_s, out, ticket);
    if (last && fin.H) {
      __syncthreads();
      finish_column(fin, out);
    }
  } else {
    ss = warp_sum(ss);
    mx = warp_max(mx);
    if (lane == 0) { s_acc[nvec * NWARP + warp] = ss; s_acc[(nvec + 1) * NWARP + warp] = mx; }
    __syncthreads();
    // without the re-projection the nvec dot partials are zero in every CTA: neither stored
    // nor summed (the last CTA writes the zeros; (nvec + 2) x G loads less in its tail)
    const int v0 = reproj ? 0 : nvec;
    for (int v = v0 + threadIdx.x; v < nval; v += KT) {
      double acc = 0.0;
      if (v == nvec + 1) {
#pragma unroll
        for (int q = 0; q < NWARP; ++q) acc = fmax(acc, s_acc[v * NWARP + q]);
      } else {
#pragma unroll
        for (int q = 0; q < NWARP; ++q) acc += s_acc[v * NWARP + q];
      }
      partials[(size_t)v * gridDim.x + blockIdx.x] = acc;
    }
    __shared__ int max_kind;
    if (threadIdx.x == 0) max_kind = nvec + 1;
    __syncthreads();
    const bool last = finish_partials_maxidx(partials, nval, gridDim.x, max_kind, out, ticket, v0);
    if (last && ro.gate_out) {
      __syncthreads();
      reorth_decide(fin, out, nvec, ro.eta2, ro.gate_out, ro.gate_md2, reproj);
    }
  }
}

// ---- small grids: the whole orthogonalisation of one Arnoldi iteration in ONE launch --------
// On a 64^2 .. 128^2 grid the four launches above (multi-dot, update, gated multi-dot, gated
// update) are 2-7 us of launch ramp, partial reduction and tail each against ~1 us of memory
// traffic.  Here the same phases run in one kernel separated by a grid barrier; every CTA sums
// the per-CTA partials itself (in CTA order, exactly as the last CTA of the separate kernels
// does) and therefore takes the selective re-orthogonalisation decision without another
// launch.  Tile ownership, partial layout and summation order are those of multidot_kernel /
// update_kernel for the same length, so H, w and every scalar are BIT-IDENTICAL to the
// four-launch path (tested).  The launcher only uses it when all CTAs are co-resident
// (grid <= 2 CTAs per SM), which the barrier needs.
//
// Grid barrier: arrival counter + generation word, self-resetting (no host bookkeeping, and a
// gated launch that returns early never touches it).
// Release / acquire at gpu scope on the two words instead of full memory fences: the CTA's
// stores are ordered before thread 0's arrival by the CTA barrier (cumulativity), the
// consumers' loads after its acquire of the new generation.
__device__ __forceinline__ void grid_bar(unsigned int* bar, unsigned int G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int gen, prev;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(gen) : "l"(bar + 1) : "memory");
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;\n" : "=r"(prev) : "l"(bar) : "memory");
    if (prev == G - 1u) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], %1;\n" ::"l"(bar), "r"(0u) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar + 1) : "memory");
    } else {
      unsigned int now;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(now) : "l"(bar + 1) : "memory");
      } while (now == gen);
    }
  }
  __syncthreads();
}

// the last-CTA sums of finish_partials / finish_partials_maxidx, done by every CTA into shared
// memory: dst[v] = sum (or max for v == max_idx) over c < G of partials[v][c], lanes striding
// the CTAs and a warp butterfly on top (the same association as the separate kernels)
__device__ __forceinline__ void reduce_partials_all(const double* partials, int nval, int G, int max_idx,
                                                    double* dst, int v_begin = 0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int v = threadIdx.x; v < v_begin; v += KT) dst[v] = 0.0;      // known zeros
  for (int v = v_begin + warp; v < nval; v += NWARP) {
    const bool mx = v == max_idx;
    double acc = 0.0;
    for (int c = lane; c < G; c += 32) {
      const double x = __ldcg(partials + (size_t)v * G + c);
      acc = mx ? fmax(acc, x) : acc + x;
    }
    acc = mx ? warp_max(acc) : warp_sum(acc);
    if (lane == 0) dst[v] = acc;
  }
  __syncthreads();
}

struct OrthSmallArgs {
  double* w;
  const double* V;
  long long ldv;
  int nvec;
  long long len_upd, len_dot, len_max;
  int Gm, Gu;                 // grids of the separate multi-dot / update kernels for these lengths
  double* partials;           // per-CTA partials of the dot phases
  double* partials_b;         // ... of the update phases (alternating buffers: one barrier per phase)
  unsigned int* bar;          // {arrivals, generation}
  double* d1;                 // out: h1[0:nvec], ||w||^2
  double* d2;                 // out: re-projection dots, ||w1||^2, max|w1_top|
  double* nrm;                // out (pass 2): ||w||^2, max|w_top|
  const double* skip;         // cancelled look-ahead iteration
  FinishArgs fin;
  Reorth ro;                  // eta2 > 0 and gate_out set: selective; else always two passes
};

// <w, V_i> partials of this CTA (multidot_kernel<2, 4>'s loop; COH: w was written by other CTAs
// of this launch, so it is read through L2)
template <bool COH>
__device__ __forceinline__ void orth_dots(const OrthSmallArgs& A, int self, double* s_acc) {
  constexpr int VEC = 2, U = 4;
  constexpr int TL = KT * 2 * VEC;
  const int nvec = A.nvec, nval = nvec + self;
  for (int k = threadIdx.x; k < nval * NWARP; k += KT) s_acc[k] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double selfacc = 0.0;
  const long long ntiles = (A.len_dot + TL - 1) / TL;
  if ((int)blockIdx.x < A.Gm) {
    for (long long tl = blockIdx.x; tl < ntiles; tl += A.Gm) {
      const long long e0 = tl * TL + 2LL * threadIdx.x;
      double2 wv[VEC];
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        const long long e = e0 + (long long)q * 2 * KT;
        if (COH) {
          wv[q] = make_double2(0.0, 0.0);
          if (e + 1 < A.len_dot) wv[q] = __ldcg(reinterpret_cast<const double2*>(A.w + e));
          else if (e < A.len_dot) wv[q].x = __ldcg(A.w + e);
        } else {
          wv[q] = ld2_stream(A.w, e, A.len_dot);
        }
        selfacc = fma(wv[q].x, wv[q].x, fma(wv[q].y, wv[q].y, selfacc));
      }
      for (int i = 0; i < nvec; i += U) {
        double2 x[U][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < VEC; ++q)
            x[u][q] = (i + u < nvec) ? ld2_stream(A.V + (size_t)(i + u) * A.ldv, e0 + (long long)q * 2 * KT, A.len_dot)
                                     : make_double2(0.0, 0.0);
        double d[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          d[u] = 0.0;
#pragma unroll
          for (int q = 0; q < VEC; ++q) d[u] = fma(wv[q].x, x[u][q].x, fma(wv[q].y, x[u][q].y, d[u]));
        }
        warp_reduce_multi<U>(d, lane);
        if ((lane & (32 / U - 1)) == 0) {
          const int u = multi_index<U>(lane);
          if (i + u < nvec) s_acc[(i + u) * NWARP + warp] += d[0];
        }
      }
    }
    if (self) {
      selfacc = warp_sum(selfacc);
      if (lane == 0) s_acc[nvec * NWARP + warp] = selfacc;
    }
    __syncthreads();
    for (int v = threadIdx.x; v < nval; v += KT) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < NWARP; ++q) acc += s_acc[v * NWARP + q];
      A.partials[(size_t)v * A.Gm + blockIdx.x] = acc;
    }
  }
}

// w -= V h on this CTA's tiles (update_kernel<MODE, 8>'s loop).  MODE 0: optional re-projection
// dots, ||w1||^2, max|w1_top| partials; MODE 1: ||w||^2, max|w_top| partials (w is this
// thread's own pass-1 result: a plain load, never the read-only path)
template <int MODE>
__device__ __forceinline__ void orth_update(const OrthSmallArgs& A, const double* s_h, bool reproj,
                                            double* s_acc) {
  constexpr int U = 8;
  constexpr int TL = KT * 2;
  const int nvec = A.nvec;
  const int nval = MODE == 0 ? nvec + 2 : 2;
  for (int k = threadIdx.x; k < nval * NWARP; k += KT) s_acc[k] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double ss = 0.0, mx = 0.0;
  const long long ntiles = (A.len_upd + TL - 1) / TL;
  for (long long k = blockIdx.x; k < ntiles; k += A.Gu) {
    const long long tl = ntiles - 1 - k;
    const long long e = tl * TL + 2LL * threadIdx.x;
    const bool full = e + 1 < A.len_upd;
    double2 wv = make_double2(0.0, 0.0);
    if (MODE == 0) wv = ld2(A.w, e, A.len_upd);
    else if (full) wv = *reinterpret_cast<const double2*>(A.w + e);
    else if (e < A.len_upd) wv.x = A.w[e];
    for (int i = 0; i < nvec; i += U) {
      double2 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        x[u] = (i + u < nvec) ? ld2(A.V + (size_t)(i + u) * A.ldv, e, A.len_upd) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i + u < nvec) {
          const double hh = s_h[i + u];
          wv.x = fma(-hh, x[u].x, wv.x);
          wv.y = fma(-hh, x[u].y, wv.y);
        }
      }
    }
    if (full) *reinterpret_cast<double2*>(A.w + e) = wv;
    else if (e < A.len_upd) A.w[e] = wv.x;
    const double dx = (e < A.len_dot) ? wv.x : 0.0, dy = (e + 1 < A.len_dot) ? wv.y : 0.0;
    if (MODE == 0 && reproj) {
      for (int i = (nvec - 1) / U * U; i >= 0; i -= U) {
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          x[u] = (i + u < nvec) ? ld2_stream(A.V + (size_t)(i + u) * A.ldv, e, A.len_upd) : make_double2(0.0, 0.0);
        double d[U];
#pragma unroll
        for (int u = 0; u < U; ++u) d[u] = fma(dx, x[u].x, dy * x[u].y);
        warp_reduce_multi<U>(d, lane);
        if ((lane & (32 / U - 1)) == 0) {
          const int u = multi_index<U>(lane);
          if (i + u < nvec) s_acc[(i + u) * NWARP + warp] += d[0];
        }
      }
    }
    ss = fma(dx, dx, fma(dy, dy, ss));
    const double mxx = (e < A.len_max) ? fabs(wv.x) : 0.0;
    const double mxy = (e + 1 < A.len_max) ? fabs(wv.y) : 0.0;
    mx = fmax(mx, fmax(mxx, mxy));
  }
  ss = warp_sum(ss);
  mx = warp_max(mx);
  if (MODE == 1) {
    if (lane == 0) { s_acc[0 * NWARP + warp] = ss; s_acc[1 * NWARP + warp] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0, b = 0.0;
      for (int q = 0; q < NWARP; ++q) { a += s_acc[q]; b = fmax(b, s_acc[NWARP + q]); }
      A.partials_b[blockIdx.x] = a;
      A.partials_b[(size_t)A.Gu + blockIdx.x] = b;
    }
  } else {
    if (lane == 0) { s_acc[nvec * NWARP + warp] = ss; s_acc[(nvec + 1) * NWARP + warp] = mx; }
    __syncthreads();
    for (int v = (reproj ? 0 : nvec) + threadIdx.x; v < nval; v += KT) {
      double acc = 0.0;
      if (v == nvec + 1) {
#pragma unroll
        for (int q = 0; q < NWARP; ++q) acc = fmax(acc, s_acc[v * NWARP + q]);
      } else {
#pragma unroll
        for (int q = 0; q < NWARP; ++q) acc += s_acc[v * NWARP + q];
      }
      A.partials_b[(size_t)v * A.Gu + blockIdx.x] = acc;
    }
  }
}

__global__ void __launch_bounds__(KT, 2) orth_small_kernel(const OrthSmallArgs A) {
  pdl_sync();
  if (A.skip && *A.skip != 0.0) return;          // cancelled look-ahead iteration (all CTAs agree)
  extern __shared__ double sm[];
  const int nvec = A.nvec;
  double* s_h = sm;                                // [nvec + 2] reduced values of the current phase
  double* s_acc = sm + ((nvec + 3) & ~1);          // [(nvec + 2)][NWARP]
  const unsigned int G = gridDim.x;
  // pass 1 dots: h1 = V^T w, ||w||^2
  orth_dots<false>(A, 1, s_acc);
  grid_bar(A.bar, G);
  reduce_partials_all(A.partials, nvec + 1, A.Gm, -1, s_h);
  const double selfdot = s_h[nvec];
  if (blockIdx.x == 0)
    for (int v = threadIdx.x; v <= nvec; v += KT) A.d1[v] = s_h[v];
  // pass 1 update (+ re-projection dots unless predicted unnecessary), ||w1||^2, max|w1_top|
  const bool selective = A.ro.eta2 > 0.0 && A.ro.gate_out;
  const bool reproj = !(A.ro.predict && A.ro.predict[0] != 0.0 && A.ro.predict[1] != 0.0);
  orth_update<0>(A, s_h, reproj, s_acc);
  grid_bar(A.bar, G);
  reduce_partials_all(A.partials_b, nvec + 2, A.Gu, nvec + 1, s_h, reproj ? 0 : nvec);   // s_h: h2 (or zeros), r
  const bool skip2 = selective && s_h[nvec] >= A.ro.eta2 * selfdot;
  if (blockIdx.x == 0) {
    for (int v = threadIdx.x; v < nvec + 2; v += KT) A.d2[v] = s_h[v];
    if (selective && threadIdx.x == 0) {
      *A.ro.gate_out = skip2 ? 1.0 : 0.0;
      if (A.ro.gate_md2) *A.ro.gate_md2 = (skip2 || reproj) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (skip2) {
      FinishArgs F1 = A.fin;
      F1.h2 = nullptr;
      finish_column(F1, A.d2 + nvec);
    }
  }
  if (skip2) return;
  // (each phase's partials are read only between its own barrier and the next one, and the dot
  // and update phases alternate between two buffers: one barrier per phase)
  if (!reproj) {
    // mispredicted: the re-projection dots h2 = V^T w1 were not computed by the update
    orth_dots<true>(A, 0, s_acc);
    grid_bar(A.bar, G);
    reduce_partials_all(A.partials, nvec, A.Gm, -1, s_h);
    if (blockIdx.x == 0)
      for (int v = threadIdx.x; v < nvec; v += KT) A.d2[v] = s_h[v];
  }
  // pass 2: w -= V h2, ||w||^2, max|w_top|, column bookkeeping
  orth_update<1>(A, s_h, false, s_acc);
  grid_bar(A.bar, G);
  if (blockIdx.x == 0) {
    reduce_partials_all(A.partials_b, 2, A.Gu, 1, s_h);
    if (threadIdx.x < 2) A.nrm[threadIdx.x] = s_h[threadIdx.x];
    __syncthreads();
    if (A.fin.H) finish_column(A.fin, A.nrm);
  }
}

bool orth_small_fits(long long len_upd, int num_sms) {
  return grid_for_len(len_upd, KT * 2, num_sms) <= 2 * num_sms;
}

cudaError_t launch_orth_small(double* w, const double* V, long long ldv, int nvec, long long len_upd,
                              long long len_dot, long long len_max, KWork& wk, double* partials_b,
                              unsigned int* bar, double* d1, double* d2, double* nrm, cudaStream_t s,
                              FinishArgs fin, const double* skip, Reorth ro) {
  OrthSmallArgs A;
  A.w = w; A.V = V; A.ldv = ldv; A.nvec = nvec;
  A.len_upd = len_upd; A.len_dot = len_dot; A.len_max = len_max;
  A.Gm = grid_for_len(len_dot, KT * 4, wk.num_sms);
  A.Gu = grid_for_len(len_upd, KT * 2, wk.num_sms);
  A.partials = wk.partials; A.partials_b = partials_b; A.bar = bar;
  A.d1 = d1; A.d2 = d2; A.nrm = nrm; A.skip = skip; A.fin = fin; A.ro = ro;
  const int G = A.Gu > A.Gm ? A.Gu : A.Gm;
  if (G > 2 * wk.num_sms) return cudaErrorInvalidConfiguration;   // the grid barrier needs co-residency
  const size_t sm = sizeof(double) * ((size_t)((nvec + 3) & ~1) + (size_t)(nvec + 2) * NWARP);
  return launch_pdl(orth_small_kernel, dim3(G), dim3(KT), sm, s, A);
}

// slab ranks, pass 2 skipped: w1 is final, so its edge rows go to the neighbours' halo buffers
// here (otherwise emhd_update_push stores the edges of the final w)
__global__ void push_edges_kernel(const double* __restrict__ w, const HaloPush H, const double* gate) {
  if (gate && *gate == 0.0) return;
  const unsigned total = NF * 4u * H.ny;
  for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < total; q += gridDim.x * blockDim.x) {
    const unsigned col = q % H.ny, t = q / H.ny;
    const unsigned r = t % 4u, f = t / 4u;
    const unsigned row = r < 2u ? r : H.nx - 4u + r;
    const long long e = (long long)f * H.plane + (long long)row * H.ny + col;
    push_edge(H, e, w[e]);
  }
  __threadfence_system();
}

cudaError_t launch_push_edges(const double* w, const HaloPush& H, const double* gate, cudaStream_t s) {
  const unsigned total = NF * 4u * H.ny;
  push_edges_kernel<<<(total + 255) / 256, 256, 0, s>>>(w, H, gate);
  return cudaGetLastError();
}

__global__ void reorth_decide_kernel(const FinishArgs F, const double* r, int nvec, double eta2,
                                     double* gate, double* gate_md2, const double* predict) {
  // reprojected: the pass-1 update computed the re-projection dots (same test as its kernel)
  const bool reproj = !(predict && predict[0] != 0.0 && predict[1] != 0.0);
  reorth_decide(F, r, nvec, eta2, gate, gate_md2, reproj);
}

// out = {sum x^2 over len_sum, max|x| over len_max}
__global__ void __launch_bounds__(KT) norms_kernel(const double* __restrict__ x, long long len_sum,
    long long len_max, double* partials, double* out, unsigned int* ticket) {
  pdl_sync();
  __shared__ double s[2 * NWARP];
  __shared__ int kinds_s[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long len = len_sum > len_max ? len_sum : len_max;
  double ss = 0.0, mx = 0.0;
  for (long long e = (long long)blockIdx.x * KT + threadIdx.x; e < len; e += (long long)gridDim.x * KT) {
    const double v = x[e];
    if (e < len_sum) ss = fma(v, v, ss);
    if (e < len_max) mx = fmax(mx, fabs(v));
  }
  ss = warp_sum(ss);
  mx = warp_max(mx);
  if (lane == 0) { s[warp] = ss; s[NWARP + warp] = mx; }
  if (threadIdx.x == 0) { kinds_s[0] = 0; kinds_s[1] = 1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < NWARP; ++q) { a += s[q]; b = fmax(b, s[NWARP + q]); }
    partials[blockIdx.x] = a;
    partials[(size_t)gridDim.x + blockIdx.x] = b;
  }
  finish_partials(partials, 2, gridDim.x, kinds_s, out, ticket);
}

// Arnoldi column bookkeeping after the (all-reduced) sums are known:
// H[0:j+1, j] = h1 + h2 ; hnext = sqrt(ss) ; breakdown test (krylov.py:161-166);
// scal = {hnext, max|w_top|} for the next fused normalise + Jv.
__global__ void arnoldi_finish_kernel(const double* h1, const double* h2, const double* nrm,
    const double* selfdot, int j, double* H, long long ldh, double* scal, double* brk_hist,
    DevStatus* st, double rtol, const double* skip2) {
  if (skip2 && *skip2 != 0.0) return;      // the column was finished by the pass-1 decision
  FinishArgs F;
  F.h1 = h1; F.h2 = h2; F.selfdot = selfdot; F.j = j; F.H = H; F.ldh = ldh; F.scal = scal;
  F.brk_hist = brk_hist; F.st = st; F.rtol = rtol;
  finish_column(F, nrm);
}

// out[s] = base[s] (+) coef[s] * sum_i Y[s*m + i] V_i   (S <= 4 outputs, one sweep over V)
__global__ void __launch_bounds__(KT) combine_kernel(const double* __restrict__ V, long long ldv, int m,
    const double* __restrict__ Y, int S, const CombineOut co, long long len) {
  pdl_sync();
  extern __shared__ double s_y[];               // [S][m]
  for (int k = threadIdx.x; k < S * m; k += KT) s_y[k] = Y[k];
  __syncthreads();
  for (long long e = ((long long)blockIdx.x * KT + threadIdx.x) * EPT; e < len;
       e += (long long)gridDim.x * KT * EPT) {
    const bool full = e + 1 < len;
    double2 acc[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) acc[s] = make_double2(0.0, 0.0);
    for (int i = 0; i < m; ++i) {
      const double* Vi = V + (size_t)i * ldv;
      double2 x = make_double2(0.0, 0.0);
      if (full) x = __ldcs(reinterpret_cast<const double2*>(Vi + e));
      else x.x = Vi[e];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        if (s < S) {
          const double y = s_y[s * m + i];
          acc[s].x = fma(x.x, y, acc[s].x);
          acc[s].y = fma(x.y, y, acc[s].y);
        }
      }
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (s < S) {
        double2 r = acc[s];
        if (co.base[s]) {
          const double c = co.coef[s];
          const double* b = co.base[s];
          r.x = __dadd_rn(b[e], __dmul_rn(c, r.x));
          if (full) r.y = __dadd_rn(b[e + 1], __dmul_rn(c, r.y));
        }
        if (full) *reinterpret_cast<double2*>(co.out[s] + e) = r;
        else co.out[s][e] = r.x;
      }
    }
  }
}

// Gate of a look-ahead Arnoldi iteration: cancelled when the host's cancel word (written by
// an async copy once the residual checks made a decision) names this process generation and
// an epoch <= j.  Evaluated once, before the iteration's first kernel; the iteration's
// kernels read *gate, so all of their CTAs agree.
__global__ void gate_kernel(const unsigned long long* cancel, unsigned gen, int j, double* gate) {
  pdl_sync();
  const unsigned long long c = *reinterpret_cast<const volatile unsigned long long*>(cancel);
  const bool hit = (unsigned)(c >> 32) == gen && (long long)(c & 0xffffffffull) <= (long long)j;
  *gate = hit ? 1.0 : 0.0;
}

// rhs_evals -= sum(evals[0:count]) (RHS evaluations of discarded iterations, stream-ordered)
__global__ void evals_discount_kernel(const double* evals, int count, DevStatus* st) {
  double s = 0.0;
  for (int k = 0; k < count; ++k) s += evals[k];
  st->rhs_evals -= (int)s;
}

cudaError_t launch_gate(const unsigned long long* cancel, unsigned gen, int j, double* gate, cudaStream_t s) {
  return launch_pdl(gate_kernel, dim3(1), dim3(1), 0, s, cancel, gen, j, gate);
}

cudaError_t launch_evals_discount(const double* evals, int count, DevStatus* st, cudaStream_t s) {
  evals_discount_kernel<<<1, 1, 0, s>>>(evals, count, st);
  return cudaGetLastError();
}

// Up to 4 CTAs per SM, every CTA the same number of tiles (1024 tiles on 592 CTAs would leave
// 160 CTAs with one tile while the rest do two: 512 CTAs of two tiles finish at the same time)
static int grid_for_len(long long len, int tile, int num_sms) {
  long long tiles = (len + tile - 1) / tile;
  if (tiles < 1) tiles = 1;
  const long long g = 4LL * num_sms;
  if (tiles <= g) return (int)tiles;
  const long long per = (tiles + g - 1) / g;
  return (int)((tiles + per - 1) / per);
}
static int grid_for(long long len, int tile, int num_sms) { return grid_for_len(len, tile, num_sms); }

cudaError_t launch_multidot(const double* w, const double* V, long long ldv, int nvec, long long len_dot,
                            int self, KWork& wk, double* out, cudaStream_t s, const double* skip,
                            const double* skip2) {
  const int G = grid_for(len_dot, KT * 4, wk.num_sms);
  const size_t sm = sizeof(double) * (size_t)(nvec + 1) * NWARP;
  return launch_pdl(multidot_kernel<2, 4>, dim3(G), dim3(KT), sm, s, w, V, ldv, nvec, len_dot, self,
                    wk.partials, out, wk.ticket, skip, skip2);
}

cudaError_t launch_update(double* w, const double* V, long long ldv, int nvec, const double* h,
                          long long len_upd, long long len_dot, long long len_max, int mode,
                          KWork& wk, double* out, cudaStream_t s, FinishArgs fin, const double* skip,
                          Reorth ro) {
  const int G = grid_for(len_upd, KT * 2, wk.num_sms);
  const int nval = mode == 0 ? nvec + 2 : 2;
  const size_t sm = sizeof(double) * ((size_t)((nvec + 1) & ~1) + (size_t)nval * NWARP);
  // with a persisting L2 window over the basis head, the rest of V is read evict-first so the
  // lines of w written here survive for the next stencil (512^2 +2 %, 1024^2 +0.9 %)
  auto k = mode == 0 ? (wk.stream_basis ? update_kernel<0, 8, false, true> : update_kernel<0, 8>)
                     : (wk.stream_basis ? update_kernel<1, 8, false, true> : update_kernel<1, 8>);
  return launch_pdl(k, dim3(G), dim3(KT), sm, s, w, V, ldv, nvec, h, len_upd, len_dot,
                    len_max, wk.partials, out, wk.ticket, fin, HaloPush{}, (const double*)skip, ro);
}

cudaError_t launch_update_push(double* w, const double* V, long long ldv, int nvec, const double* h,
                               long long len_upd, long long len_dot, long long len_max, KWork& wk,
                               double* out, const HaloPush& push, cudaStream_t s, const double* skip2) {
  const int G = grid_for(len_upd, KT * 2, wk.num_sms);
  const size_t sm = sizeof(double) * ((size_t)((nvec + 1) & ~1) + 2 * NWARP);
  Reorth ro{};
  ro.skip2 = skip2;
  update_kernel<1, 8, true><<<G, KT, sm, s>>>(w, V, ldv, nvec, h, len_upd, len_dot, len_max,
                                               wk.partials, out, wk.ticket, FinishArgs{}, push, nullptr, ro);
  return cudaGetLastError();
}

cudaError_t launch_norms(const double* x, long long len_sum, long long len_max, KWork& wk, double* out,
                         cudaStream_t s) {
  const long long len = len_sum > len_max ? len_sum : len_max;
  long long g = (len + KT - 1) / KT;
  const int G = (int)(g < 2LL * wk.num_sms ? (g < 1 ? 1 : g) : 2LL * wk.num_sms);
  return launch_pdl(norms_kernel, dim3(G), dim3(KT), 0, s, x, len_sum, len_max, wk.partials, out, wk.ticket);
}

cudaError_t launch_arnoldi_finish(const double* h1, const double* h2, const double* nrm,
                                  const double* selfdot, int j, double* H, long long ldh, double* scal,
                                  double* brk_hist, DevStatus* st, double rtol, cudaStream_t s,
                                  const double* skip2) {
  arnoldi_finish_kernel<<<1, 128, 0, s>>>(h1, h2, nrm, selfdot, j, H, ldh, scal, brk_hist, st, rtol,
                                          skip2);
  return cudaGetLastError();
}

cudaError_t launch_reorth_decide(FinishArgs fin, const double* r, int nvec, double eta2, double* gate,
                                 cudaStream_t s, double* gate_md2, const double* predict) {
  reorth_decide_kernel<<<1, 128, 0, s>>>(fin, r, nvec, eta2, gate, gate_md2, predict);
  return cudaGetLastError();
}

cudaError_t launch_combine(const double* V, long long ldv, int m, const double* Y, int S,
                           const CombineOut& co, long long len, int num_sms, cudaStream_t s) {
  long long g = (len + TILE - 1) / TILE;
  const int G = (int)(g < 4LL * num_sms ? (g < 1 ? 1 : g) : 4LL * num_sms);
  const size_t sm = sizeof(double) * (size_t)S * m;
  return launch_pdl(combine_kernel, dim3(G), dim3(KT), sm, s, V, ldv, m, Y, S, co, len);
}

}  // namespace emhd
