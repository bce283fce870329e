// Small dense phi-functions of the Krylov Hessenberg matrix, on the GPU.
//
// Replaces reference pkg/src/expmhd/phifuncs.py:65-107 (phi_dense: one
// exponential of the block upper-bidiagonal augmented matrix) and
// krylov.py:209-238, 378-383 (residual_estimate, _expm_seed, _phi_seed).
// The exponential is the Al-Mohy & Higham (2009) Pade scaling-and-squaring
// algorithm with exact 1-norms — the algorithm scipy.linalg.expm (the
// reference's third-party dependency, scipy 1.18.1) implements — run by one
// CTA per requested scale: degree selection, Pade numerator/denominator,
// Gauss–Jordan solve with partial pivoting and the squarings all stay on the
// device, so a residual check costs one launch and one 8-byte read.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include "emhd_common.cuh"
#include "dense.cuh"

namespace emhd {

constexpr int DT = 512;   // threads per CTA

// C = A * B, n x n row-major (ld = n).  The CTA's 16 x 32 thread grid owns one output tile
// of (16 RM) x (32 RN) elements, RM x RN per thread, sized to n (n = 85 -> 96 x 96 instead of
// four padded 64 x 64 tiles); k runs in 16-wide shared-memory chunks, so every element is
// one fma chain over k = 0 .. n-1 in order, whatever the tiling.
constexpr int MM_MAXR = 128;                 // largest single-tile extent (8 x 16, 4 x 32)
template <int RM, int RN>
__device__ void mm_tile(double* C, const double* A, const double* B, int n, double* sA, double* sB) {
  constexpr int TR = 16 * RM, TC = 32 * RN;
  const int t = threadIdx.x;
  const int tr = (t / 32) * RM;
  const int tc = (t % 32) * RN;
  for (int bi = 0; bi < n; bi += TR) {
    for (int bj = 0; bj < n; bj += TC) {
      double acc[RM][RN];
#pragma unroll
      for (int u = 0; u < RM; ++u)
#pragma unroll
        for (int v = 0; v < RN; ++v) acc[u][v] = 0.0;
      for (int bk = 0; bk < n; bk += 16) {
        for (int q = t; q < TR * 16; q += DT) {
          const int r = q / 16, c = q % 16;
          const int gr = bi + r, gc = bk + c;
          sA[r * 17 + c] = (gr < n && gc < n) ? A[gr * n + gc] : 0.0;
        }
        for (int q = t; q < 16 * TC; q += DT) {
          const int r2 = q / TC, c2 = q % TC;
          const int gr2 = bk + r2, gc2 = bj + c2;
          sB[r2 * TC + c2] = (gr2 < n && gc2 < n) ? B[gr2 * n + gc2] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          double bv[RN];
#pragma unroll
          for (int v = 0; v < RN; ++v) bv[v] = sB[k * TC + tc + v];
#pragma unroll
          for (int u = 0; u < RM; ++u) {
            const double av = sA[(tr + u) * 17 + k];
#pragma unroll
            for (int v = 0; v < RN; ++v) acc[u][v] = fma(av, bv[v], acc[u][v]);
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int u = 0; u < RM; ++u)
#pragma unroll
        for (int v = 0; v < RN; ++v) {
          const int gr = bi + tr + u, gc = bj + tc + v;
          if (gr < n && gc < n) C[gr * n + gc] = acc[u][v];
        }
    }
  }
  __syncthreads();
}

__device__ void mm(double* C, const double* A, const double* B, int n, double* sA, double* sB) {
  if (n <= 16) mm_tile<1, 1>(C, A, B, n, sA, sB);
  else if (n <= 32) mm_tile<2, 1>(C, A, B, n, sA, sB);
  else if (n <= 48) mm_tile<3, 2>(C, A, B, n, sA, sB);
  else if (n <= 64) mm_tile<4, 2>(C, A, B, n, sA, sB);
  else if (n <= 80) mm_tile<5, 3>(C, A, B, n, sA, sB);
  else if (n <= 96) mm_tile<6, 3>(C, A, B, n, sA, sB);
  else if (n <= 112) mm_tile<7, 4>(C, A, B, n, sA, sB);
  else mm_tile<8, 4>(C, A, B, n, sA, sB);    // n > 128 loops over 128 x 128 tiles
}

// Column sums y[c] = sum_r w(r) |A[r][c]| (w = 1 or x[r]) with all threads in ONE pass: the
// DT threads cover (column, row group) pairs — G = DT / ceil32(n) row groups of coalesced
// column lanes — and the per-group partials are combined in a fixed order (two barriers per
// call instead of two per 32-column chunk: ell's 2m+1 dependent |A|-products are barrier-bound)
__device__ void abs_colsums(const double* A, int n, const double* x, double* y, double* part) {
  const int nc = (n + 31) & ~31;                  // columns padded to whole warps
  if (nc > DT) {
    // n > DT: chunks of DT columns, one row group each
    for (int c0 = 0; c0 < n; c0 += DT) {
      const int c = c0 + threadIdx.x;
      if (c < n) {
        double s = 0.0;
        if (x) for (int r = 0; r < n; ++r) s += x[r] * fabs(A[r * n + c]);
        else for (int r = 0; r < n; ++r) s += fabs(A[r * n + c]);
        y[c] = s;
      }
    }
    __syncthreads();
    return;
  }
  const int G = DT / nc;                          // row groups
  const int c = threadIdx.x % nc, g = threadIdx.x / nc;
  double s = 0.0;
  if (g < G && c < n) {
    if (x) for (int r = g; r < n; r += G) s += x[r] * fabs(A[r * n + c]);
    else for (int r = g; r < n; r += G) s += fabs(A[r * n + c]);
  }
  if (g < G) part[g * nc + c] = s;
  __syncthreads();
  for (int cc = threadIdx.x; cc < n; cc += DT) {
    double t = 0.0;
    for (int q = 0; q < G; ++q) t += part[q * nc + cc];
    y[cc] = t;
  }
  __syncthreads();
}

__device__ double max_of(const double* y, int n, double* red) {
  if (threadIdx.x < 32) {
    double b = 0.0;
    for (int i = threadIdx.x; i < n; i += 32) b = fmax(b, y[i]);
    b = warp_max(b);
    if (threadIdx.x == 0) red[DT / 32] = b;
  }
  __syncthreads();
  const double r = red[DT / 32];
  __syncthreads();
  return r;
}

// 1-norm (max column sum) of an n x n matrix; y: n scratch, part: 512 scratch
__device__ double norm1(const double* A, int n, double* red, double* y, double* part) {
  abs_colsums(A, n, nullptr, y, part);
  return max_of(y, n, red);
}

// || |A|^p ||_1 via p row-vector products 1^T |A| ... |A|
__device__ double norm1_abs_power(const double* A, int n, int p, double* x, double* y, double* red,
                                  double* part) {
  for (int i = threadIdx.x; i < n; i += DT) x[i] = 1.0;
  __syncthreads();
  for (int k = 0; k < p; ++k) {
    abs_colsums(A, n, x, y, part);
    for (int i = threadIdx.x; i < n; i += DT) x[i] = y[i];
    __syncthreads();
  }
  return max_of(x, n, red);
}

// Al-Mohy & Higham backward-error estimate ell(A, m) (exact norms)
__device__ int ell(const double* A, int n, int m, double a1, double* x, double* y, double* red,
                   double* part) {
  // |c_{2m+1}|^{-1} = C(4m+2, 2m+1) * (4m+3)!
  const int p = 2 * m + 1;
  double lg = lgamma(2.0 * p + 1.0) - 2.0 * lgamma((double)p + 1.0) + lgamma(2.0 * p + 2.0);
  const double nap = norm1_abs_power(A, n, p, x, y, red, part);
  if (nap == 0.0 || a1 == 0.0) return 0;
  // alpha = nap / (a1 * abs_c_recip); value = ceil(log2(alpha / u) / (2m))
  const double log2_alpha = log2(nap) - log2(a1) - lg / log(2.0);
  const double v = ceil((log2_alpha + 53.0) / (2.0 * m));
  return v > 0.0 ? (int)v : 0;
}

__device__ void axpby_mat(double* out, const double* const* terms, const double* coefs, int nterms,
                          int n, double diag) {
  for (int e = threadIdx.x; e < n * n; e += DT) {
    double s = ((e / n) == (e % n)) ? diag : 0.0;
    for (int k = 0; k < nterms; ++k) s = fma(coefs[k], terms[k][e], s);
    out[e] = s;
  }
  __syncthreads();
}

// Gauss–Jordan with partial pivoting on M = [Q | R] (n x 2n): R <- Q^{-1} R.
// The pivot row is staged (scaled) in shared memory, rows are distributed over warps and
// columns over lanes: no integer division in the elimination, one broadcast read per column.
__device__ __noinline__ bool gj_solve(double* M, int n, double* red, int* ired, double* fac, double* prow) {
  const int w2 = 2 * n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NWD = DT / 32;
  for (int k = 0; k < n; ++k) {
    // pivot: largest |M[i][k]| for i >= k, lowest index on ties (deterministic)
    double best = -1.0; int bi = n;
    for (int i = k + threadIdx.x; i < n; i += DT) {
      const double a = fabs(M[i * w2 + k]);
      if (a > best) { best = a; bi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) { red[warp] = best; ired[warp] = bi; }
    __syncthreads();
    // every thread combines the warp results itself (same order, same answer), so no second
    // barrier; red/ired are rewritten only after this step's two later barriers.  Only warps
    // that saw a candidate row (rows k .. n-1) take part
    double bb = -1.0; int piv = n;
    const int nwd = min(NWD, (n - k + 31) / 32);
    for (int w = 0; w < nwd; ++w)
      if (red[w] > bb || (red[w] == bb && ired[w] < piv)) { bb = red[w]; piv = ired[w]; }
    if (!(bb > 0.0)) return false;
    const double d = M[piv * w2 + k];
    // stage the scaled pivot row (columns > k) and swap rows k <-> piv
    for (int c = k + 1 + threadIdx.x; c < w2; c += DT) {
      const double pv = M[piv * w2 + c] / d;
      prow[c] = pv;
      if (piv != k) M[piv * w2 + c] = M[k * w2 + c];
      M[k * w2 + c] = pv;
    }
    for (int i = threadIdx.x; i < n; i += DT) {
      const int src = (i == piv) ? k : i;              // row piv now holds old row k
      fac[i] = (i == k) ? 0.0 : M[src * w2 + k];
    }
    __syncthreads();
    if (piv != k && threadIdx.x == 0) M[piv * w2 + k] = M[k * w2 + k];
    // elimination: warp w owns rows w, w + NWD, ...; for each column its lanes update all of
    // the warp's rows at once — RPW independent FMAs per column instead of one dependent
    // load-FMA-store chain per row (the same operation per element, so the same bits)
    constexpr int RPW = 8;
    for (int base = warp; base < n; base += NWD * RPW) {
      double fr[RPW];
#pragma unroll
      for (int q = 0; q < RPW; ++q) {
        const int i = base + q * NWD;
        fr[q] = (i < n) ? fac[i] : 0.0;          // fac[k] = 0: the pivot row is left alone
      }
      for (int c = k + 1 + lane; c < w2; c += 32) {
        const double pc = prow[c];
#pragma unroll
        for (int q = 0; q < RPW; ++q) {
          if (fr[q] != 0.0) {
            double* a = M + (size_t)(base + q * NWD) * w2 + c;
            *a = fma(-fr[q], pc, *a);
          }
        }
      }
    }
    __syncthreads();
  }
  return true;
}

// Blocked Gauss–Jordan with partial pivoting for n <= MM_MAXR: R <- Q^{-1} R on M = [Q | R]
// without moving rows; rowof[j] = the row of M that ends up holding solution row j.
// The unblocked solve above spends n dependent steps of {pivot search, division, broadcast,
// rank-1 update, three CTA barriers} (1.6 us each at n = 110: 275 of the exponential's 484 us)
// and three shared-memory accesses per FMA.  Here GB = 8 pivot columns are eliminated per
// step: (1) the n x 8 panel is copied into a compact buffer and ONE warp runs the eight
// pivot / scale / eliminate steps on it warp-synchronously, recording the composite row
// transform W (n x 8: the images of the unit vectors of the eight pivot rows); (2) every
// column to the right gets the rank-8 update C[i] = keep_i C[i] + sum_s W[i][s] C[r_s] — eight
// FMAs per element against one load, one store and eight broadcast reads, non-pivot rows
// first (they only read the pivot rows), then the pivot rows, one thread per column.  Pivot
// choice is the same rule (largest magnitude, lowest row on ties) on the same updated entries
// up to the association of the updates, so results agree with the unblocked solve to round-off.
// Measured (clock64, n = 110, M on chip): 541 k cycles unblocked -> 403 k blocked (panel warp
// 162 k, rank-8 update 142 k + 20 k, staging 8 k) -> 360 k with the panel look-ahead below;
// exponential 486 -> 394 us at n = 110, 290 -> 245 at n = 80, 768 -> 455 at n = 128.
constexpr int GB = 8, GPB = GB + 1;
constexpr int GJ_BLOCKED_MIN_N = 24;   // below: the unblocked solve is as fast (n = 12: 65 vs 70 us)
// One warp: in-place Gauss-Jordan of the n x bw panel M[:, k : k+bw) held in registers (lane l:
// rows l + 32 q, q < 4), rows already used as pivots excluded from the search; writes the
// composite transform Wout[n][GPB], the pivot rows rowof[k + t] and used[]; clears red[0] on a
// zero pivot column.  Reads M only in its own panel columns and writes nothing to M.
__device__ __forceinline__ void gj_panel_warp(const double* M, int w2, int n, int k, int bw, int* used,
                                              int* rowof, double* Wout, double* red, int lane) {
  double X[4][GB];
  unsigned usedmask = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = lane + 32 * q;
    if (i < n) {
#pragma unroll
      for (int c = 0; c < GB; ++c) X[q][c] = c < bw ? M[(size_t)i * w2 + k + c] : 0.0;
      usedmask |= (used[i] ? 1u : 0u) << q;
    } else {
#pragma unroll
      for (int c = 0; c < GB; ++c) X[q][c] = 0.0;
      usedmask |= 1u << q;
    }
  }
  double* pbuf = red + 1;                    // the pivot row of the step, published by its owner
  bool ok = true;
#pragma unroll
  for (int t = 0; t < GB; ++t) {
    if (t < bw && ok) {
      double best = -1.0; int bi = n;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!((usedmask >> q) & 1u)) {
          const double a = fabs(X[q][t]);
          if (a > best) { best = a; bi = lane + 32 * q; }
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (!(best > 0.0)) {
        if (lane == 0) red[0] = 0.0;
        ok = false;
      } else {
        const int r = bi;
        const bool owner = lane == (r & 31);
        if (owner) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q == (r >> 5)) {
#pragma unroll
              for (int c = 0; c < GB; ++c) pbuf[c] = X[q][c];
            }
          usedmask |= 1u << (r >> 5);
          used[r] = 1;
          rowof[k + t] = r;
        }
        __syncwarp();
        double prs[GB];
#pragma unroll
        for (int c = 0; c < GB; ++c) prs[c] = pbuf[c];
        __syncwarp();
        const double rd = 1.0 / prs[t];
#pragma unroll
        for (int c = 0; c < GB; ++c) prs[c] = (c == t) ? rd : prs[c] * rd;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const bool isr = owner && q == (r >> 5);
          const double f = X[q][t];
#pragma unroll
          for (int c = 0; c < GB; ++c) {
            const double v = (c == t) ? -f * prs[t] : fma(-f, prs[c], X[q][c]);
            X[q][c] = isr ? prs[c] : v;
          }
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = lane + 32 * q;
    if (i < n) {
#pragma unroll
      for (int c = 0; c < GB; ++c) Wout[i * GPB + c] = X[q][c];
    }
  }
}

// Rank-bw update of the columns [c_begin, c_end) with the transform Wc of the panel whose pivot
// rows are pr_rows: C[i] = keep_i C[i] + sum_s Wc[i][s] C[r_s], by the threads [t0, t0 + nt) of the
// CTA (nt a multiple of 32), synchronised among themselves by barrier `bar_id` (0: the CTA
// barrier): non-pivot rows first (they only read the pivot rows), then the pivot rows, one
// thread per column.
__device__ __forceinline__ void gj_update(double* M, int w2, int n, int c_begin, int c_end,
                                          const int (&pr_rows)[GB], int bw, const double* Wc, int t0,
                                          int nt, int bar_id) {
  const int tl = threadIdx.x - t0;
  const int lane = tl & 31, warp = tl >> 5, nw = nt >> 5;
  auto sync = [&]() {
    if (bar_id == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;\n" ::"r"(bar_id), "r"(nt) : "memory");
  };
  if (c_begin < c_end) {
    if ((reinterpret_cast<uintptr_t>(M) & 15) == 0) {
      // two columns per lane, 16-byte accesses (rows are 2n doubles: aligned), from the even
      // column at or below c_begin (an already-eliminated column when c_begin is odd)
      for (int cb = (c_begin & ~1) + 2 * lane; cb < c_end; cb += 64) {
        double2 pv[GB];
#pragma unroll
        for (int q = 0; q < GB; ++q)
          pv[q] = q < bw ? *reinterpret_cast<const double2*>(M + (size_t)pr_rows[q] * w2 + cb) : make_double2(0.0, 0.0);
        for (int i0 = warp; i0 < n; i0 += 4 * nw) {
          double2 acc[4];
          bool live[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * nw;
            bool is_piv = false;
#pragma unroll
            for (int q = 0; q < GB; ++q) is_piv |= (i == pr_rows[q]);
            live[u] = i < n && !is_piv;
            acc[u] = live[u] ? *reinterpret_cast<const double2*>(M + (size_t)i * w2 + cb) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int q = 0; q < GB; ++q) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (live[u]) {
                const double wv = Wc[(i0 + u * nw) * GPB + q];
                acc[u].x = fma(wv, pv[q].x, acc[u].x);
                acc[u].y = fma(wv, pv[q].y, acc[u].y);
              }
            }
          }
          // a pair may straddle an odd boundary of [c_begin, c_end): the column outside it
          // belongs to another phase (or to the panel warp 0 is reading) and is not written
          const bool ux = cb >= c_begin, uy = cb + 1 < c_end;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (live[u]) {
              double* dst = M + (size_t)(i0 + u * nw) * w2 + cb;
              if (ux && uy) *reinterpret_cast<double2*>(dst) = acc[u];
              else if (ux) dst[0] = acc[u].x;
              else if (uy) dst[1] = acc[u].y;
            }
          }
        }
      }
    } else {
      for (int cb = c_begin + lane; cb < c_end; cb += 32) {
        double pv[GB];
#pragma unroll
        for (int q = 0; q < GB; ++q) pv[q] = q < bw ? M[(size_t)pr_rows[q] * w2 + cb] : 0.0;
        for (int i0 = warp; i0 < n; i0 += 4 * nw) {
          double acc[4];
          bool live[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * nw;
            bool is_piv = false;
#pragma unroll
            for (int q = 0; q < GB; ++q) is_piv |= (i == pr_rows[q]);
            live[u] = i < n && !is_piv;
            acc[u] = live[u] ? M[(size_t)i * w2 + cb] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < GB; ++q) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (live[u]) acc[u] = fma(Wc[(i0 + u * nw) * GPB + q], pv[q], acc[u]);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (live[u]) M[(size_t)(i0 + u * nw) * w2 + cb] = acc[u];
        }
      }
    }
  }
  sync();
  for (int cb = c_begin + tl; cb < c_end; cb += nt) {
    double pv[GB];
#pragma unroll
    for (int q = 0; q < GB; ++q) pv[q] = q < bw ? M[(size_t)pr_rows[q] * w2 + cb] : 0.0;
#pragma unroll
    for (int u = 0; u < GB; ++u) {
      if (u < bw) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < GB; ++q) acc = fma(Wc[pr_rows[u] * GPB + q], pv[q], acc);
        M[(size_t)pr_rows[u] * w2 + cb] = acc;
      }
    }
  }
}

// Panels with look-ahead: while warps 1..15 apply panel p's rank-8 update to the columns right
// of panel p+1, warp 0 already factors panel p+1 (whose columns were updated first, by all
// warps); the transforms alternate between two buffers.  The step costs the longer of the two
// instead of their sum.
__device__ __noinline__ bool gj_solve_blocked(double* M, int n, double* W0, double* W1, int* used,
                                              int* rowof, double* red) {
  const int w2 = 2 * n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < n; i += DT) used[i] = 0;
  if (threadIdx.x == 0) red[0] = 1.0;              // cleared by the panel warp on a zero pivot
  __syncthreads();
  double* Wbuf[2] = {W0, W1};
  if (warp == 0) gj_panel_warp(M, w2, n, 0, min(GB, n), used, rowof, Wbuf[0], red, lane);
  __syncthreads();
  int cur = 0;
  for (int k = 0; k < n; k += GB) {
    if (red[0] == 0.0) return false;
    const int bw = min(GB, n - k);
    const int kn = k + bw;                          // first column of the next panel
    const int bwn = kn < n ? min(GB, n - kn) : 0;
    int pr_rows[GB];
#pragma unroll
    for (int q = 0; q < GB; ++q) pr_rows[q] = q < bw ? rowof[k + q] : -1;
    const double* Wc = Wbuf[cur];
    // (1) the next panel's columns first, by everybody
    gj_update(M, w2, n, kn, kn + bwn, pr_rows, bw, Wc, 0, DT, 0);
    __syncthreads();
    // (2) warp 0 factors the next panel while the other warps update the rest
    if (warp == 0) {
      if (bwn > 0) gj_panel_warp(M, w2, n, kn, bwn, used, rowof, Wbuf[cur ^ 1], red, lane);
    } else {
      gj_update(M, w2, n, kn + bwn, w2, pr_rows, bw, Wc, 32, DT - 32, 1);
    }
    __syncthreads();
    cur ^= 1;
  }
  return red[0] != 0.0;
}

// dispatcher: the blocked solve for n <= MM_MAXR (its two transform buffers live in the matrix-product staging
// buffers sA / sB, free during the solve; used / rowof in the factor area), else the unblocked
// one.  *rowof: row of M holding solution row j (null: natural order)
__device__ bool gj_solve_any(double* M, int n, double* red, int* ired, double* fac, double* prow,
                             double* sA, double* sB, const int** rowof, int blocked) {
  if (blocked && n <= MM_MAXR && n >= GJ_BLOCKED_MIN_N) {
    int* used = reinterpret_cast<int*>(fac);
    int* ro = used + n;
    *rowof = ro;
    return gj_solve_blocked(M, n, sA, sB, used, ro, red);
  }
  *rowof = nullptr;
  return gj_solve(M, n, red, ired, fac, prow);
}

// E = exp(A), A overwritten by scaling; returns false on failure.
// E = exp(A) (vcol < 0), or only vout = exp(A) e_vcol (vcol >= 0; E then holds a scaled factor)
// sM: shared-memory home of the n x 2n Gauss-Jordan system when it fits (else null: global)
__device__ bool expm_block(double* A, int n, double* E, DenseWork W, double* sA, double* sB, double* red,
                          int* ired, double* prow, int vcol, double* vout, double* sM, double* fac) {
  double* A2 = W.m[0];
  double* A4 = W.m[1];
  double* A6 = W.m[2];
  double* A8 = W.m[3];
  double* U = W.m[4];
  double* Vm = W.m[5];
  double* T = W.m[6];
  double* M = sM ? sM : W.m[7];      // n x 2n: n dependent elimination steps, keep on chip
  double* x = prow;        // norm scratch on chip (prow is free until the solve)
  double* y = prow + n;

  // ell() runs 2m+1 dependent |A|-matvecs: read A from shared memory when the (not yet
  // used) Gauss-Jordan area is on chip
  auto onchip = [&](const double* src) -> const double* {
    if (!sM) return src;
    for (int e = threadIdx.x; e < n * n; e += DT) sM[e] = src[e];
    __syncthreads();
    return sM;
  };
  mm(A2, A, A, n, sA, sB);
  mm(A4, A2, A2, n, sA, sB);
  mm(A6, A4, A2, n, sA, sB);
  const double a1 = norm1(A, n, red, y, sA);
  const double d4 = pow(norm1(A4, n, red, y, sA), 0.25);
  const double d6 = pow(norm1(A6, n, red, y, sA), 1.0 / 6.0);
  const double eta1 = fmax(d4, d6);
  int mdeg = 0, s = 0;
  if (eta1 <= 1.495585217958292e-002 && ell(onchip(A), n, 3, a1, x, y, red, sA) == 0) mdeg = 3;
  else if (eta1 <= 2.539398330063230e-001 && ell(onchip(A), n, 5, a1, x, y, red, sA) == 0) mdeg = 5;
  double d8 = 0.0, eta3 = 0.0;
  if (mdeg == 0) {
    mm(A8, A4, A4, n, sA, sB);
    d8 = pow(norm1(A8, n, red, y, sA), 0.125);
    eta3 = fmax(d6, d8);
    if (eta3 <= 9.504178996162932e-001 && ell(onchip(A), n, 7, a1, x, y, red, sA) == 0) mdeg = 7;
    else if (eta3 <= 2.097847961257068e+000 && ell(onchip(A), n, 9, a1, x, y, red, sA) == 0) mdeg = 9;
  }
  if (mdeg == 0) {
    mm(T, A4, A6, n, sA, sB);           // A^10
    const double d10 = pow(norm1(T, n, red, y, sA), 0.1);
    const double eta4 = fmax(d8, d10);
    const double eta5 = fmin(eta3, eta4);
    s = (eta5 == 0.0) ? 0 : (int)fmax(ceil(log2(eta5 / 4.25)), 0.0);
    // scale A by 2^-s and the even powers accordingly
    const double sc = ldexp(1.0, -s);
    for (int e = threadIdx.x; e < n * n; e += DT) A[e] *= sc;
    __syncthreads();
    const double a1s = norm1(A, n, red, y, sA);
    s += ell(onchip(A), n, 13, a1s, x, y, red, sA);
    const double sc2 = ldexp(1.0, -s);
    // rescale from the already-applied 2^-s0 to 2^-s (A), then rebuild powers
    const double extra = sc2 / sc;
    for (int e = threadIdx.x; e < n * n; e += DT) A[e] *= extra;
    // powers of 2^-s A: exact power-of-two rescaling of A^2, A^4, A^6 (bit-identical to
    // recomputing them from the scaled A, three matrix products cheaper)
    const double s2 = ldexp(1.0, -2 * s), s4 = ldexp(1.0, -4 * s), s6 = ldexp(1.0, -6 * s);
    for (int e = threadIdx.x; e < n * n; e += DT) { A2[e] *= s2; A4[e] *= s4; A6[e] *= s6; }
    __syncthreads();
    mdeg = 13;
  }
  // Pade numerator (V + U) and denominator (V - U)
  if (mdeg == 13) {
    const double b[14] = {64764752532480000., 32382376266240000., 7771770303897600.,
                          1187353796428800., 129060195264000., 10559470521600.,
                          670442572800., 33522128640., 1323241920., 40840800., 960960.,
                          16380., 182., 1.};
    {
      const double* tt[3] = {A6, A4, A2};
      const double cc[3] = {b[13], b[11], b[9]};
      axpby_mat(T, tt, cc, 3, n, 0.0);
      mm(U, A6, T, n, sA, sB);
      const double* t2[4] = {U, A6, A4, A2};
      const double c2[4] = {1.0, b[7], b[5], b[3]};
      axpby_mat(T, t2, c2, 4, n, b[1]);
      mm(U, A, T, n, sA, sB);
    }
    {
      const double* tt[3] = {A6, A4, A2};
      const double cc[3] = {b[12], b[10], b[8]};
      axpby_mat(T, tt, cc, 3, n, 0.0);
      mm(Vm, A6, T, n, sA, sB);
      const double* t2[4] = {Vm, A6, A4, A2};
      const double c2[4] = {1.0, b[6], b[4], b[2]};
      axpby_mat(T, t2, c2, 4, n, b[0]);
      for (int e = threadIdx.x; e < n * n; e += DT) Vm[e] = T[e];
      __syncthreads();
    }
  } else {
    double b[10];
    if (mdeg == 3) { const double c[] = {120., 60., 12., 1.}; for (int k = 0; k < 4; ++k) b[k] = c[k]; }
    if (mdeg == 5) { const double c[] = {30240., 15120., 3360., 420., 30., 1.}; for (int k = 0; k < 6; ++k) b[k] = c[k]; }
    if (mdeg == 7) { const double c[] = {17297280., 8648640., 1995840., 277200., 25200., 1512., 56., 1.}; for (int k = 0; k < 8; ++k) b[k] = c[k]; }
    if (mdeg == 9) { const double c[] = {17643225600., 8821612800., 2075673600., 302702400., 30270240., 2162160., 110880., 3960., 90., 1.}; for (int k = 0; k < 10; ++k) b[k] = c[k]; }
    const double* pw[4] = {A2, A4, A6, A8};
    // odd part: A * (b1 I + b3 A2 + b5 A4 + ...); even part: b0 I + b2 A2 + ...
    const int nt = mdeg / 2;          // number of non-identity even powers
    double co[4], ce[4];
    for (int k = 0; k < nt; ++k) { co[k] = b[2 * k + 3]; ce[k] = b[2 * k + 2]; }
    axpby_mat(T, pw, co, nt, n, b[1]);
    mm(U, A, T, n, sA, sB);
    axpby_mat(Vm, pw, ce, nt, n, b[0]);
  }
  // M = [V - U | V + U]
  for (int e = threadIdx.x; e < n * n; e += DT) {
    const int r = e / n, c = e % n;
    M[r * 2 * n + c] = Vm[e] - U[e];
    M[r * 2 * n + n + c] = Vm[e] + U[e];
  }
  __syncthreads();
  const int* rowof = nullptr;
#ifdef DENSE_DBG
  const long long tg0 = clock64();
#endif
  const bool gj_ok = gj_solve_any(M, n, red, ired, fac, prow, sA, sB, &rowof, W.gj_blocked);
#ifdef DENSE_DBG
  if (threadIdx.x == 0) printf("gj n %d blocked %d cycles %lld\n", n, W.gj_blocked, clock64() - tg0);
#endif
  if (!gj_ok) return false;
  for (int e = threadIdx.x; e < n * n; e += DT)
    E[e] = M[(size_t)(rowof ? rowof[e / n] : e / n) * 2 * n + n + e % n];
  __syncthreads();
  if (vcol >= 0 && s <= 7) {
    // only the column E^(2^s) e_vcol is needed: 2^s matrix-vector products instead of s
    // squarings (2^s n^2 vs s n^3 work); result left in vout[0:n]
    double* xa = vout;
    double* xb = vout + n;
    for (int i = threadIdx.x; i < n; i += DT) xa[i] = E[(size_t)i * n + vcol];
    // E^T on chip (thread i walks column i: consecutive threads, consecutive words)
    double* Et = nullptr;
    if (sM && s > 0) {
      Et = sM;
      for (int e = threadIdx.x; e < n * n; e += DT) Et[(e % n) * n + e / n] = E[e];
    }
    __syncthreads();
    for (int k = 1; k < (1 << s); ++k) {
      for (int i = threadIdx.x; i < n; i += DT) {
        double acc = 0.0;
        if (Et) {
          for (int c = 0; c < n; ++c) acc = fma(Et[(size_t)c * n + i], xa[c], acc);
        } else {
          const double* row = E + (size_t)i * n;
          for (int c = 0; c < n; ++c) acc = fma(row[c], xa[c], acc);
        }
        xb[i] = acc;
      }
      __syncthreads();
      double* tmp = xa; xa = xb; xb = tmp;
    }
    if (xa != vout)
      for (int i = threadIdx.x; i < n; i += DT) vout[i] = xa[i];
    __syncthreads();
    return true;
  }
  for (int k = 0; k < s; ++k) {
    mm(T, E, E, n, sA, sB);
    for (int e = threadIdx.x; e < n * n; e += DT) E[e] = T[e];
    __syncthreads();
  }
  if (vcol >= 0)
    for (int i = threadIdx.x; i < n; i += DT) vout[i] = E[(size_t)i * n + vcol];
  __syncthreads();
  return true;
}

// One CTA per scale s: A = (scale_s * post) * augmented(H_m, order); E = expm(A);
// y_s = beta * E[0:m, order*m]; res_s = |h_next| |y_m| / ||y|| * res_scale_s.
__global__ void __launch_bounds__(DT) phi_small_kernel(PhiSmallArgs P) {
  __shared__ double sA[MM_MAXR * 17];
  __shared__ double sB[16 * MM_MAXR];
  __shared__ double red[DT / 32 + 1];
  __shared__ int ired[DT / 32 + 1];
  extern __shared__ double prow[];                 // [2n] pivot row, [n] GJ factors (+ [n][2n] M)
  const int sidx = blockIdx.x;
  // phi_order(X) e1 from the (m + order)-dimensional augmentation
  //   [[X, e1, 0 ..], [0, 0, 1 ..], .., [0 .. 0]]   (exp top-right column = phi_order(X) e1),
  // the Expokit form of the reference's ((order+1) m)-dimensional block matrix
  // (phifuncs.py:97-104): same phi to round-off, (order+1)^3 m^3 / (m+order)^3 less work.
  // With E_out (emhd_expm, order 0) the matrix is exactly sc * H.
  // batch mode: CTA s checks basis size mb[s] of the same factorisation (speculative
  // residual checks of several m at once); h_{m+1,m} and the breakdown flag come from H
  const int m = P.batch ? P.mb[sidx] : P.m, n = m + P.order;
  const int col = (P.order == 0) ? 0 : m + P.order - 1;
  DenseWork W = P.work[sidx];
  W.gj_blocked = P.gj_blocked;
  if (P.smem_work) {
    // small n: every work matrix lives in shared memory (the same code, generic pointers):
    // the ~100 dependent steps of an exponential (products, norms, the 2m+1 |A|-products of
    // ell, the elimination) then wait on shared-memory latency instead of L2 round trips
    double* b = prow + 3 * n;
    const size_t nn = (size_t)n * n;
    W.a = b;
    W.e = b + nn;
    for (int k = 0; k < 7; ++k) W.m[k] = b + (2 + k) * nn;
    W.m[7] = b + 9 * nn;
    W.vec = b + 11 * nn;
  }
  double* A = W.a;
  double* E = W.e;
  double* Yrow = P.Y + (size_t)sidx * (P.batch ? P.ldy : P.m);
  const double sc = P.scales_by_value ? P.sv[sidx] : P.scales[sidx];
  double hn;
  bool brk;
  if (P.batch) {
    brk = P.brk_hist[m - 1] != 0.0;
    hn = brk ? 0.0 : P.H[(size_t)m * P.ldh + (m - 1)];
  } else {
    hn = P.scal ? P.scal[0] : 0.0;
    brk = P.scal ? (P.scal[2] != 0.0) : true;
  }
  const double beta = P.beta[0];
  for (int e = threadIdx.x; e < n * n; e += DT) {
    const int r = e / n, c = e % n;
    double v = 0.0;
    if (r < m && c < m) v = sc * P.H[(size_t)r * P.ldh + c];
    else if (r == 0 && c == m) v = 1.0;
    else if (r >= m && c == r + 1) v = 1.0;
    A[e] = v;
  }
  __syncthreads();
  bool finite = true;
  for (int e = threadIdx.x; e < m * m; e += DT) if (!isfinite(A[(e / m) * n + e % m])) finite = false;
  finite = __syncthreads_and(finite);
  double* ycol = W.vec + 3 * n;                    // [2n] column result / ping-pong
  double* sM = (!P.smem_work && n <= P.smem_n) ? prow + ((3 * n + 1) & ~1) : nullptr;   // 16-byte aligned
  bool ok = finite && expm_block(A, n, E, W, sA, sB, red, ired, prow, P.E_out ? -1 : col, ycol, sM, prow + 2 * n);
  if (ok) {
    bool fin2 = true;
    if (P.E_out) {
      for (int e = threadIdx.x; e < n * n; e += DT) if (!isfinite(E[e])) fin2 = false;
    } else {
      for (int i = threadIdx.x; i < n; i += DT) if (!isfinite(ycol[i])) fin2 = false;
    }
    ok = __syncthreads_and(fin2);
  }
  if (!ok) {
    if (threadIdx.x == 0) { atomicOr(&P.st->flags, (int)ST_DENSE); P.res[sidx] = INFINITY; }
    return;
  }
  if (P.E_out) {
    for (int e = threadIdx.x; e < n * n; e += DT) P.E_out[e] = E[e];
  }
  double ss = 0.0;
  for (int i = threadIdx.x; i < m; i += DT) {
    const double yv = ycol[i] * beta;
    Yrow[i] = yv;
    ss += yv * yv;
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < DT / 32; ++w) t += red[w];
    const double nrm = sqrt(t);
    const double ylast = ycol[m - 1] * beta;
    const double hnext = brk ? 0.0 : hn;
    double r = (nrm == 0.0) ? 0.0 : fabs(hnext) * fabs(ylast) / nrm;
    P.res[sidx] = r * (P.scales_by_value ? P.rv[sidx] : P.res_scale[sidx]);
  }
}

// ============================================================================================
// Cluster version (n >= DENSE_CLUSTER_MIN_N): one exponential per thread-block cluster of
// DENSE_CLUSTER CTAs on as many SMs.  The same algorithm as expm_block (same degree / scaling
// decisions from the same exact 1-norms, same Pade, Gauss-Jordan and squarings), with the
// O(n^3) products, the elementwise updates and the column sums of the norms and of ell's
// |A|-products split by row blocks across the cluster; work matrices stay in the (L2-resident)
// global workspace and the phases are ordered by cluster barriers (release / acquire at cluster
// scope).  The Gauss-Jordan solve and the 2^s vector products run on rank 0 (one CTA), whose
// n dependent steps would otherwise each cost a cluster barrier.
struct Team {
  int rank, size;
  __device__ __forceinline__ void sync() const {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  __device__ __forceinline__ int r0(int n) const { const int b = (n + size - 1) / size; return min(n, rank * b); }
  __device__ __forceinline__ int r1(int n) const { const int b = (n + size - 1) / size; return min(n, (rank + 1) * b); }
};

// rows [r0, r1) of C = A * B (n x n, row-major), the k sums in order 0 .. n-1 per element (the
// same chains as mm_tile); 16 row lanes x 32 column lanes, RN columns per thread
template <int RN>
__device__ void mm_rows_t(double* C, const double* A, const double* B, int n, int r0, int r1, double* sA,
                          double* sB) {
  constexpr int TC = 32 * RN;
  const int t = threadIdx.x;
  const int tr = t / 32;
  const int tc = (t % 32) * RN;
  for (int bi = r0; bi < r1; bi += 16) {
    for (int bj = 0; bj < n; bj += TC) {
      double acc[RN];
#pragma unroll
      for (int v = 0; v < RN; ++v) acc[v] = 0.0;
      for (int bk = 0; bk < n; bk += 16) {
        for (int q = t; q < 16 * 16; q += DT) {
          const int r = q / 16, c = q % 16;
          const int gr = bi + r, gc = bk + c;
          sA[r * 17 + c] = (gr < r1 && gc < n) ? A[gr * n + gc] : 0.0;
        }
        for (int q = t; q < 16 * TC; q += DT) {
          const int r2 = q / TC, c2 = q % TC;
          const int gr2 = bk + r2, gc2 = bj + c2;
          sB[r2 * TC + c2] = (gr2 < n && gc2 < n) ? B[gr2 * n + gc2] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const double av = sA[tr * 17 + k];
#pragma unroll
          for (int v = 0; v < RN; ++v) acc[v] = fma(av, sB[k * TC + tc + v], acc[v]);
        }
        __syncthreads();
      }
      const int gr = bi + tr;
#pragma unroll
      for (int v = 0; v < RN; ++v) {
        const int gc = bj + tc + v;
        if (gr < r1 && gc < n) C[gr * n + gc] = acc[v];
      }
    }
  }
}

__device__ void mm_team(const Team& T, double* C, const double* A, const double* B, int n, double* sA,
                        double* sB) {
  const int r0 = T.r0(n), r1 = T.r1(n);
  if (n <= 32) mm_rows_t<1>(C, A, B, n, r0, r1, sA, sB);
  else if (n <= 64) mm_rows_t<2>(C, A, B, n, r0, r1, sA, sB);
  else if (n <= 96) mm_rows_t<3>(C, A, B, n, r0, r1, sA, sB);
  else mm_rows_t<4>(C, A, B, n, r0, r1, sA, sB);     // n > 128: loops over 128-column tiles
  T.sync();
}

// y[c] = sum_r w(r) |A[r][c]| over ALL rows: each CTA sums its row block into the step's
// partial buffer, then (after the cluster barrier) every CTA adds the size partials in rank
// order — identical y on every CTA.  `par` alternates between the two partial buffers.
__device__ void colsums_team(const Team& T, const double* A, int n, const double* x, double* y,
                             double* part_g, int& par) {
  const int r0 = T.r0(n), r1 = T.r1(n);
  double* mine = part_g + ((size_t)par * T.size + T.rank) * n;
  for (int c = threadIdx.x; c < n; c += DT) {
    double s = 0.0;
    if (x) for (int r = r0; r < r1; ++r) s += x[r] * fabs(A[r * n + c]);
    else for (int r = r0; r < r1; ++r) s += fabs(A[r * n + c]);
    mine[c] = s;
  }
  T.sync();
  const double* all = part_g + (size_t)par * T.size * n;
  for (int c = threadIdx.x; c < n; c += DT) {
    double s = 0.0;
    for (int q = 0; q < T.size; ++q) s += __ldcg(all + (size_t)q * n + c);
    y[c] = s;
  }
  __syncthreads();
  par ^= 1;
}

__device__ double norm1_team(const Team& T, const double* A, int n, double* red, double* y, double* part_g,
                             int& par) {
  colsums_team(T, A, n, nullptr, y, part_g, par);
  return max_of(y, n, red);
}

__device__ int ell_team(const Team& T, const double* A, int n, int m, double a1, double* x, double* y,
                        double* red, double* part_g, int& par) {
  const int p = 2 * m + 1;
  const double lg = lgamma(2.0 * p + 1.0) - 2.0 * lgamma((double)p + 1.0) + lgamma(2.0 * p + 2.0);
  for (int i = threadIdx.x; i < n; i += DT) x[i] = 1.0;
  __syncthreads();
  for (int k = 0; k < p; ++k) {
    colsums_team(T, A, n, x, y, part_g, par);
    for (int i = threadIdx.x; i < n; i += DT) x[i] = y[i];
    __syncthreads();
  }
  const double nap = max_of(x, n, red);
  if (nap == 0.0 || a1 == 0.0) return 0;
  const double log2_alpha = log2(nap) - log2(a1) - lg / log(2.0);
  const double v = ceil((log2_alpha + 53.0) / (2.0 * m));
  return v > 0.0 ? (int)v : 0;
}

__device__ void axpby_team(const Team& T, double* out, const double* const* terms, const double* coefs,
                           int nterms, int n, double diag) {
  const int r0 = T.r0(n), r1 = T.r1(n);
  for (int e = r0 * n + threadIdx.x; e < r1 * n; e += DT) {
    double s = ((e / n) == (e % n)) ? diag : 0.0;
    for (int k = 0; k < nterms; ++k) s = fma(coefs[k], terms[k][e], s);
    out[e] = s;
  }
  T.sync();
}

__device__ void scale_rows_team(const Team& T, double* X, int n, double f) {
  const int r0 = T.r0(n), r1 = T.r1(n);
  for (int e = r0 * n + threadIdx.x; e < r1 * n; e += DT) X[e] *= f;
}

// expm_block on a cluster (see above); rank 0 leaves the result as expm_block does
__device__ bool expm_cluster(const Team& T, double* A, int n, double* E, DenseWork W, double* sA, double* sB,
                             double* red, int* ired, double* prow, int vcol, double* vout, double* sM,
                             double* fac) {
  double* A2 = W.m[0];
  double* A4 = W.m[1];
  double* A6 = W.m[2];
  double* A8 = W.m[3];
  double* U = W.m[4];
  double* Vm = W.m[5];
  double* Tm = W.m[6];
  double* M = sM ? sM : W.m[7];
  double* x = prow;
  double* y = prow + n;
  int par = 0;
  mm_team(T, A2, A, A, n, sA, sB);
  mm_team(T, A4, A2, A2, n, sA, sB);
  mm_team(T, A6, A4, A2, n, sA, sB);
  const double a1 = norm1_team(T, A, n, red, y, W.part, par);
  const double d4 = pow(norm1_team(T, A4, n, red, y, W.part, par), 0.25);
  const double d6 = pow(norm1_team(T, A6, n, red, y, W.part, par), 1.0 / 6.0);
  const double eta1 = fmax(d4, d6);
  int mdeg = 0, s = 0;
  if (eta1 <= 1.495585217958292e-002 && ell_team(T, A, n, 3, a1, x, y, red, W.part, par) == 0) mdeg = 3;
  else if (eta1 <= 2.539398330063230e-001 && ell_team(T, A, n, 5, a1, x, y, red, W.part, par) == 0) mdeg = 5;
  double d8 = 0.0, eta3 = 0.0;
  if (mdeg == 0) {
    mm_team(T, A8, A4, A4, n, sA, sB);
    d8 = pow(norm1_team(T, A8, n, red, y, W.part, par), 0.125);
    eta3 = fmax(d6, d8);
    if (eta3 <= 9.504178996162932e-001 && ell_team(T, A, n, 7, a1, x, y, red, W.part, par) == 0) mdeg = 7;
    else if (eta3 <= 2.097847961257068e+000 && ell_team(T, A, n, 9, a1, x, y, red, W.part, par) == 0) mdeg = 9;
  }
  if (mdeg == 0) {
    mm_team(T, Tm, A4, A6, n, sA, sB);           // A^10
    const double d10 = pow(norm1_team(T, Tm, n, red, y, W.part, par), 0.1);
    const double eta4 = fmax(d8, d10);
    const double eta5 = fmin(eta3, eta4);
    s = (eta5 == 0.0) ? 0 : (int)fmax(ceil(log2(eta5 / 4.25)), 0.0);
    const double sc = ldexp(1.0, -s);
    scale_rows_team(T, A, n, sc);
    T.sync();
    const double a1s = norm1_team(T, A, n, red, y, W.part, par);
    s += ell_team(T, A, n, 13, a1s, x, y, red, W.part, par);
    const double sc2 = ldexp(1.0, -s);
    scale_rows_team(T, A, n, sc2 / sc);
    scale_rows_team(T, A2, n, ldexp(1.0, -2 * s));
    scale_rows_team(T, A4, n, ldexp(1.0, -4 * s));
    scale_rows_team(T, A6, n, ldexp(1.0, -6 * s));
    T.sync();
    mdeg = 13;
  }
  if (mdeg == 13) {
    const double b[14] = {64764752532480000., 32382376266240000., 7771770303897600.,
                          1187353796428800., 129060195264000., 10559470521600.,
                          670442572800., 33522128640., 1323241920., 40840800., 960960.,
                          16380., 182., 1.};
    {
      const double* tt[3] = {A6, A4, A2};
      const double cc[3] = {b[13], b[11], b[9]};
      axpby_team(T, Tm, tt, cc, 3, n, 0.0);
      mm_team(T, U, A6, Tm, n, sA, sB);
      const double* t2[4] = {U, A6, A4, A2};
      const double c2[4] = {1.0, b[7], b[5], b[3]};
      axpby_team(T, Tm, t2, c2, 4, n, b[1]);
      mm_team(T, U, A, Tm, n, sA, sB);
    }
    {
      const double* tt[3] = {A6, A4, A2};
      const double cc[3] = {b[12], b[10], b[8]};
      axpby_team(T, Tm, tt, cc, 3, n, 0.0);
      mm_team(T, Vm, A6, Tm, n, sA, sB);
      const double* t2[4] = {Vm, A6, A4, A2};
      const double c2[4] = {1.0, b[6], b[4], b[2]};
      axpby_team(T, Vm, t2, c2, 4, n, b[0]);      // in place per element: reads Vm[e] first
    }
  } else {
    double b[10];
    if (mdeg == 3) { const double c[] = {120., 60., 12., 1.}; for (int k = 0; k < 4; ++k) b[k] = c[k]; }
    if (mdeg == 5) { const double c[] = {30240., 15120., 3360., 420., 30., 1.}; for (int k = 0; k < 6; ++k) b[k] = c[k]; }
    if (mdeg == 7) { const double c[] = {17297280., 8648640., 1995840., 277200., 25200., 1512., 56., 1.}; for (int k = 0; k < 8; ++k) b[k] = c[k]; }
    if (mdeg == 9) { const double c[] = {17643225600., 8821612800., 2075673600., 302702400., 30270240., 2162160., 110880., 3960., 90., 1.}; for (int k = 0; k < 10; ++k) b[k] = c[k]; }
    const double* pw[4] = {A2, A4, A6, A8};
    const int nt = mdeg / 2;
    double co[4], ce[4];
    for (int k = 0; k < nt; ++k) { co[k] = b[2 * k + 3]; ce[k] = b[2 * k + 2]; }
    axpby_team(T, Tm, pw, co, nt, n, b[1]);
    mm_team(T, U, A, Tm, n, sA, sB);
    axpby_team(T, Vm, pw, ce, nt, n, b[0]);
  }
  // rank 0: M = [V - U | V + U], Gauss-Jordan, E; the others wait at the next barrier
  bool ok = true;
  if (T.rank == 0) {
    for (int e = threadIdx.x; e < n * n; e += DT) {
      const int r = e / n, c = e % n;
      const double v = __ldcg(Vm + e), u = __ldcg(U + e);
      M[r * 2 * n + c] = v - u;
      M[r * 2 * n + n + c] = v + u;
    }
    __syncthreads();
    const int* rowof = nullptr;
    ok = gj_solve_any(M, n, red, ired, fac, prow, sA, sB, &rowof, W.gj_blocked);
    if (ok)
      for (int e = threadIdx.x; e < n * n; e += DT)
        E[e] = M[(size_t)(rowof ? rowof[e / n] : e / n) * 2 * n + n + e % n];
    __syncthreads();
    if (threadIdx.x == 0) red[DT / 32] = ok ? 1.0 : 0.0;
  }
  // share the solve's verdict: rank 0 writes it into the partial buffer before the barrier
  if (T.rank == 0 && threadIdx.x == 0) W.part[0] = ok ? 1.0 : 0.0;
  T.sync();
  ok = __ldcg(W.part) != 0.0;
  if (!ok) return false;
  if (vcol >= 0 && s <= 7) {
    // 2^s matrix-vector products on rank 0 (dependent, each O(n^2)); result in vout
    if (T.rank == 0) {
      double* xa = vout;
      double* xb = vout + n;
      for (int i = threadIdx.x; i < n; i += DT) xa[i] = E[(size_t)i * n + vcol];
      __syncthreads();
      for (int k = 1; k < (1 << s); ++k) {
        for (int i = threadIdx.x; i < n; i += DT) {
          double acc = 0.0;
          const double* row = E + (size_t)i * n;
          for (int c = 0; c < n; ++c) acc = fma(row[c], xa[c], acc);
          xb[i] = acc;
        }
        __syncthreads();
        double* tmp = xa; xa = xb; xb = tmp;
      }
      if (xa != vout)
        for (int i = threadIdx.x; i < n; i += DT) vout[i] = xa[i];
      __syncthreads();
    }
    return true;
  }
  for (int k = 0; k < s; ++k) {
    mm_team(T, Tm, E, E, n, sA, sB);
    const int r0 = T.r0(n), r1 = T.r1(n);
    for (int e = r0 * n + threadIdx.x; e < r1 * n; e += DT) E[e] = Tm[e];
    T.sync();
  }
  if (vcol >= 0 && T.rank == 0) {
    for (int i = threadIdx.x; i < n; i += DT) vout[i] = E[(size_t)i * n + vcol];
    __syncthreads();
  }
  return true;
}

// phi_small_kernel on a cluster: cluster q serves problem q (a scale / basis size); rank 0 of
// the cluster writes the outputs
__global__ void __launch_bounds__(DT) phi_cluster_kernel(PhiSmallArgs P) {
  __shared__ double sA[MM_MAXR * GPB];              // matmul staging (16 x 17) / blocked-solve panel
  __shared__ double sB[16 * MM_MAXR];
  __shared__ double red[DT / 32 + 1];
  __shared__ int ired[DT / 32 + 1];
  extern __shared__ double prow[];                 // [2n] pivot row, [n] GJ factors (+ [n][2n] M on rank 0)
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  Team T{(int)rank, DENSE_CLUSTER};
  const int sidx = blockIdx.x / DENSE_CLUSTER;
  const int m = P.batch ? P.mb[sidx] : P.m, n = m + P.order;
  const int col = (P.order == 0) ? 0 : m + P.order - 1;
  DenseWork W = P.work[sidx];
  W.gj_blocked = P.gj_blocked;
  double* A = W.a;
  double* E = W.e;
  double* Yrow = P.Y + (size_t)sidx * (P.batch ? P.ldy : P.m);
  const double sc = P.scales_by_value ? P.sv[sidx] : P.scales[sidx];
  double hn;
  bool brk;
  if (P.batch) {
    brk = P.brk_hist[m - 1] != 0.0;
    hn = brk ? 0.0 : P.H[(size_t)m * P.ldh + (m - 1)];
  } else {
    hn = P.scal ? P.scal[0] : 0.0;
    brk = P.scal ? (P.scal[2] != 0.0) : true;
  }
  const double beta = P.beta[0];
  {
    // this rank's rows of the augmented matrix, and its verdict on their finiteness
    const int r0 = T.r0(n), r1 = T.r1(n);
    bool fin = true;
    for (int e = r0 * n + threadIdx.x; e < r1 * n; e += DT) {
      const int r = e / n, c = e % n;
      double v = 0.0;
      if (r < m && c < m) {
        v = sc * P.H[(size_t)r * P.ldh + c];
        if (!isfinite(v)) fin = false;
      } else if (r == 0 && c == m) v = 1.0;
      else if (r >= m && c == r + 1) v = 1.0;
      A[e] = v;
    }
    fin = __syncthreads_and(fin);
    if (threadIdx.x == 0) W.part[(size_t)DENSE_CLUSTER * n + rank] = fin ? 1.0 : 0.0;
  }
  T.sync();
  bool finite = true;
  for (int q = 0; q < DENSE_CLUSTER; ++q)
    finite = finite && __ldcg(W.part + (size_t)DENSE_CLUSTER * n + q) != 0.0;
  T.sync();                                        // the partial buffer is reused below
  double* ycol = W.vec + 3 * n;
  double* sM = (rank == 0 && n <= P.smem_n) ? prow + ((3 * n + 1) & ~1) : nullptr;   // 16-byte aligned
  bool ok = finite && expm_cluster(T, A, n, E, W, sA, sB, red, ired, prow, P.E_out ? -1 : col, ycol, sM,
                                   prow + 2 * n);
  if (rank != 0) return;
  if (ok) {
    bool fin2 = true;
    if (P.E_out) {
      for (int e = threadIdx.x; e < n * n; e += DT) if (!isfinite(E[e])) fin2 = false;
    } else {
      for (int i = threadIdx.x; i < n; i += DT) if (!isfinite(ycol[i])) fin2 = false;
    }
    ok = __syncthreads_and(fin2);
  }
  if (!ok) {
    if (threadIdx.x == 0) { atomicOr(&P.st->flags, (int)ST_DENSE); P.res[sidx] = INFINITY; }
    return;
  }
  if (P.E_out) {
    for (int e = threadIdx.x; e < n * n; e += DT) P.E_out[e] = E[e];
  }
  double ss = 0.0;
  for (int i = threadIdx.x; i < m; i += DT) {
    const double yv = ycol[i] * beta;
    Yrow[i] = yv;
    ss += yv * yv;
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < DT / 32; ++w) t += red[w];
    const double nrm = sqrt(t);
    const double ylast = ycol[m - 1] * beta;
    const double hnext = brk ? 0.0 : hn;
    double r = (nrm == 0.0) ? 0.0 : fabs(hnext) * fabs(ylast) / nrm;
    P.res[sidx] = r * (P.scales_by_value ? P.rv[sidx] : P.res_scale[sidx]);
  }
}

// smallest n served by the cluster kernel (0: never); EMHD_DENSE_CLUSTER_N, emhd_set_dense_cluster
static int g_cluster_min_n = -1;

int dense_cluster_min_n() {
  if (g_cluster_min_n < 0) {
    const char* e = getenv("EMHD_DENSE_CLUSTER_N");
    g_cluster_min_n = e ? atoi(e) : 56;
  }
  return g_cluster_min_n;
}

void set_dense_cluster_min_n(int n) { g_cluster_min_n = n < 0 ? 0 : n; }

static int g_gj_blocked = -1;
int dense_gj_blocked() {
  if (g_gj_blocked < 0) {
    const char* e = getenv("EMHD_DENSE_GJ_BLOCKED");
    g_gj_blocked = e ? (atoi(e) != 0 ? 1 : 0) : 1;
  }
  return g_gj_blocked;
}
void set_dense_gj_blocked(int on) { g_gj_blocked = on ? 1 : 0; }

cudaError_t launch_phi_small(const PhiSmallArgs& Pin, int nscales, cudaStream_t s) {
  PhiSmallArgs P = Pin;
  const int n = P.m + P.order;              // the largest m of a batch
  // the Gauss-Jordan system [n][2n] joins the pivot row in dynamic shared memory when it
  // fits next to the static matmul tiles (n <= ~110)
  static int max_dyn = -1;
  if (max_dyn < 0) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, phi_small_kernel);
    max_dyn = optin - (int)fa.sharedSizeBytes;
    if (cudaFuncSetAttribute(phi_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn) !=
        cudaSuccess) {
      cudaGetLastError();
      max_dyn = 48 * 1024 - (int)fa.sharedSizeBytes;
    }
  }
  const int gj_blocked = dense_gj_blocked();
  static int use_smem = -1;
  if (use_smem < 0) {
    const char* env = getenv("EMHD_DENSE_SMEM");
    use_smem = env ? atoi(env) != 0 : 1;
  }
  // dynamic shared memory: [2n] pivot row + [n] elimination factors, then the [n][2n]
  // Gauss-Jordan system when it fits (or, for small n on one CTA, the whole workspace)
  size_t dyn = sizeof(double) * 3 * n;
  P.smem_n = 0;
  P.smem_work = 0;
  P.gj_blocked = gj_blocked;
  const int cmin = dense_cluster_min_n();
  const bool cluster = cmin > 0 && n >= cmin;
  const size_t whole = sizeof(double) * (3 * (size_t)n + 11 * (size_t)n * n + 5 * (size_t)n + 64);
  if (use_smem && !cluster && whole <= (size_t)max_dyn) {
    dyn = whole;                        // n <= ~42: the whole exponential on chip
    P.smem_work = 1;
  } else if (use_smem && sizeof(double) * (3 * (size_t)n + 1 + 2 * (size_t)n * n) <= (size_t)max_dyn) {
    dyn = sizeof(double) * (3 * (size_t)n + 1 + 2 * (size_t)n * n);
    P.smem_n = n;
  }
  if (cluster) {
    // one cluster of DENSE_CLUSTER CTAs per problem; rank 0 keeps the on-chip M when it fits
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(phi_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
      cudaGetLastError();
      attr = true;
    }
    P.cluster = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nscales * DENSE_CLUSTER);
    cfg.blockDim = dim3(DT);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = DENSE_CLUSTER;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, phi_cluster_kernel, P);
  }
  P.cluster = 0;
  phi_small_kernel<<<nscales, DT, dyn, s>>>(P);
  return cudaGetLastError();
}

}  // namespace emhd
