// Fused 2.5D resistive-MHD right-hand side / finite-difference Jv stencil.
//
// Replaces reference pkg/src/expmhd/mhd.py:144-285 (apply_ghosts, pressure,
// hyperbolic_flux, diffusive_flux, rhs) and fdjac.py:38-49 (FdJacobianOperator
// ._apply), bit for bit: every floating-point operation is issued in the
// reference NumPy evaluation order, this translation unit is compiled with
// -fmad=false (no contraction), divisions by the per-cell density are IEEE
// divisions and divisions by the constants 2h and sigma use the exact
// FMA-corrected reciprocal (div_const, emhd_common.cuh).
//
// Layout: state (8, nx, ny) fp64, y fastest (mhd.py:99-103).  One CTA owns a
// strip of TY columns (one thread per column) and marches down a chunk of
// rows, keeping three rows of per-cell primitives, three rows of x-fluxes and
// two rows of y-fluxes in shared memory.  Primitives are evaluated once per
// cell (the reference evaluates them twice, mhd.py:177-179 and :218-221 —
// identical bits), the derivatives of a flux cell are shared by its x- and
// y-flux, and halo recomputation only happens at strip edges (4 columns) and
// chunk edges (4 rows).
#include <cstdint>
#include <cstdlib>
#include "emhd_common.cuh"
#include "stencil.cuh"

#ifndef EMHD_PFB
#define EMHD_PFB 1
#endif
#ifndef EMHD_QP_REG
#define EMHD_QP_REG 1
#endif

namespace emhd {

// primitives differentiated across rows/columns: shared by the CTA in the primitive ring
enum : int { Q_V0 = 0, Q_V1, Q_V2, Q_B0, Q_B1, Q_B2, Q_T, NQ };
// cell-centre-only quantities: written and read by the cell's own thread (no barrier)
enum : int { C_RHO = 0, C_MX, C_MY, C_EN, C_PT, NC };

// Element offsets are 32-bit: the launcher requires 8 * nx * ny < 2^32 (a 4096^2 slab is
// 2^27), so every address is one 32 x 32 -> 64 IMAD.WIDE from the array base.
struct RowRef {
  unsigned off;      // element offset of (field 0, row, col 0) in the chosen buffer
  unsigned fs;       // field stride in that buffer
  bool halo;         // read from the halo buffer instead of the interior
  bool flip;         // mirrored ghost row: MX, BX change sign
};

// ghost-row / ghost-column sign flips as a mask on the high word (-x flips the sign bit)
__device__ __forceinline__ double flip_sign(double x, unsigned m) {
  return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x));
}

__device__ __forceinline__ int map_ghost(int k, int n, int bc, bool& flip) {
  flip = false;
  if (k >= 0 && k < n) return k;
  if (bc == BC_PERIODIC) return k < 0 ? k + n : k - n;
  if (bc == BC_ZEROGRAD) return k < 0 ? 0 : n - 1;
  flip = true;                                  // reflect ('symmetric' pad)
  return k < 0 ? -k - 1 : 2 * n - 1 - k;
}

__device__ __forceinline__ RowRef row_ref(const StencilParams& P, int r) {
  RowRef R;
  const unsigned ny = (unsigned)P.ny;
  R.halo = false;
  R.fs = (unsigned)P.nx * ny;
  if (r < 0 && P.bcx_lo == BC_EXTERNAL) {
    R.halo = true; R.fs = 2 * ny; R.off = (unsigned)(r + 2) * ny; R.flip = false;
    return R;
  }
  if (r >= P.nx && P.bcx_hi == BC_EXTERNAL) {
    R.halo = true; R.fs = 2 * ny; R.off = (unsigned)NF * 2 * ny + (unsigned)(r - P.nx) * ny;
    R.flip = false;
    return R;
  }
  bool fl;
  int src = map_ghost(r, P.nx, r < 0 ? P.bcx_lo : P.bcx_hi, fl);
  R.off = (unsigned)src * ny;
  R.flip = fl;
  return R;
}

// perturbed / plain state of one cell, with ghost sign flips applied after the
// arithmetic exactly as np.pad followed by "*= -1.0" would see it
template <int MODE>
__device__ __forceinline__ void load_cell(const StencilParams& P, const RowRef& R, int jsrc,
                                          bool yflip, double sigma, double hnext, double rh,
                                          double u[NF]) {
  const double* A = R.halo ? P.a_halo : P.a;
  const double* Vv = nullptr;
  if (MODE != MODE_RHS) Vv = R.halo ? P.v_halo : P.v;
  const unsigned o = R.off + jsrc;
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    double x = __ldg(A + (o + f * R.fs));
    if (MODE == MODE_JV) {
      double d = __ldg(Vv + (o + f * R.fs));
      x = __dadd_rn(x, __dmul_rn(sigma, d));          // a + sigma * v   (fdjac.py:44)
    } else if (MODE == MODE_JVN) {
      double d = div_const(__ldg(Vv + (o + f * R.fs)), hnext, rh);   // v_j = w / h (krylov.py:167)
      x = __dadd_rn(x, __dmul_rn(sigma, d));
    }
    u[f] = x;
  }
  if (R.flip) { u[1] = -u[1]; u[4] = -u[4]; }
  if (yflip) { u[2] = -u[2]; u[5] = -u[5]; }
}

// raw (unperturbed) inputs of one cell, fetched one row ahead of their use
template <int MODE>
struct RawCell {
  double a[NF];
  double v[MODE == MODE_RHS ? 1 : NF];
};

template <int MODE>
__device__ __forceinline__ void fetch_cell(const StencilParams& P, const RowRef& R, int jsrc,
                                           RawCell<MODE>& x) {
  const double* A = R.halo ? P.a_halo : P.a;
  const unsigned o = R.off + jsrc;
#pragma unroll
  for (int f = 0; f < NF; ++f) x.a[f] = __ldg(A + (o + f * R.fs));
  if (MODE != MODE_RHS) {
    const double* Vv = R.halo ? P.v_halo : P.v;
#pragma unroll
    for (int f = 0; f < NF; ++f) x.v[f] = __ldg(Vv + (o + f * R.fs));
  }
}

// vj (MODE_JVN, optional): the normalised basis entries w / h_next, kept for the v_j store
template <int MODE>
__device__ __forceinline__ void combine_cell(const RawCell<MODE>& x, unsigned xflip, unsigned yflip,
                                             double sigma, double hnext, double rh, bool fh,
                                             double u[NF], double* vj = nullptr) {
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    double val = x.a[f];
    if (MODE == MODE_JV) val = __dadd_rn(val, __dmul_rn(sigma, x.v[f]));
    if (MODE == MODE_JVN) {
      const double q = fh ? div_const1(x.v[f], hnext, rh) : div_const(x.v[f], hnext, rh);
      if (vj) vj[f] = q;
      val = __dadd_rn(val, __dmul_rn(sigma, q));
    }
    u[f] = val;
  }
  u[1] = flip_sign(u[1], xflip); u[4] = flip_sign(u[4], xflip);
  u[2] = flip_sign(u[2], yflip); u[5] = flip_sign(u[5], yflip);
}

// --- cp.async staging of raw rows (Ampere+ LDGSTS; no register cost) -------------
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// --- bulk async copies (TMA engine, cp.async.bulk) tracked by an mbarrier ----------
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred done;\n"
      "MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      " @!done bra MBAR_WAIT_%=;\n}\n" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, unsigned bytes,
                                              unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(b))
      : "memory");
}

__device__ __forceinline__ bool elect_one() {
  unsigned p;
  asm volatile("{\n .reg .pred q;\n elect.sync _|q, 0xffffffff;\n selp.u32 %0, 1, 0, q;\n}\n" : "=r"(p));
  return p != 0;
}

// one raw row of an interior strip (columns j0-2 .. j0+TY+1, all inside the grid): 8 or 16
// contiguous row segments, issued by one thread; completion lands on the slot's mbarrier
template <int MODE, int QW>
__device__ __forceinline__ void fetch_row_bulk(const StencilParams& P, const RowRef& R, int jfirst,
                                               double* slot, unsigned long long* bar) {
  constexpr int NA = MODE == MODE_RHS ? 1 : 2;
  constexpr unsigned SEG = QW * sizeof(double);
  mbar_expect_tx(bar, NA * NF * SEG);
  const double* A = R.halo ? P.a_halo : P.a;
  const unsigned o = R.off + jfirst;
#pragma unroll
  for (int f = 0; f < NF; ++f) bulk_copy_g2s(slot + f * QW, A + (o + f * R.fs), SEG, bar);
  if (NA == 2) {
    const double* Vv = R.halo ? P.v_halo : P.v;
#pragma unroll
    for (int f = 0; f < NF; ++f) bulk_copy_g2s(slot + (NF + f) * QW, Vv + (o + f * R.fs), SEG, bar);
  }
}

// q[bidx[k]] for the augmented epilogue's B columns, selected with compile-time indices so the
// coefficients stay in registers (a runtime index into q[] would put q in local memory)
__device__ __forceinline__ void aug_coefs(const StencilParams& P, const double qv[5], double qb[5]) {
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    double c = 0.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) c = (k < P.nb && P.bidx[k] == i) ? qv[i] : c;
    qb[k] = c;
  }
}

// top += sum_k B_k[idx] q[bidx[k]], k = 0 .. nb-1 in order (krylov.py:268-270, exact order)
__device__ __forceinline__ double aug_add(const StencilParams& P, const double qb[5], unsigned long long idx,
                                          double top) {
#pragma unroll
  for (int k = 0; k < 5; ++k)
    if (k < P.nb) top = __dadd_rn(top, __dmul_rn(__ldg(P.bcol[k] + idx), qb[k]));
  return top;
}

// raw ring layout: [slot][array (a, v)][field][column slot]
template <int MODE, int QW>
__device__ __forceinline__ void fetch_async(const StencilParams& P, const RowRef& R, int jsrc, int c,
                                            double* slot) {
  constexpr int NA = MODE == MODE_RHS ? 1 : 2;
  const double* A = R.halo ? P.a_halo : P.a;
  const unsigned o = R.off + jsrc;
#pragma unroll
  for (int f = 0; f < NF; ++f) cp_async8(slot + f * QW + c, A + (o + f * R.fs));
  if (NA == 2) {
    const double* Vv = R.halo ? P.v_halo : P.v;
#pragma unroll
    for (int f = 0; f < NF; ++f) cp_async8(slot + (NF + f) * QW + c, Vv + (o + f * R.fs));
  }
}

template <int MODE, int QW>
__device__ __forceinline__ void consume_raw(const double* slot, int c, RawCell<MODE>& x) {
#pragma unroll
  for (int f = 0; f < NF; ++f) x.a[f] = slot[f * QW + c];
  if (MODE != MODE_RHS) {
#pragma unroll
    for (int f = 0; f < NF; ++f) x.v[f] = slot[(NF + f) * QW + c];
  }
}

// Shared-memory layout of a cell's primitives: 16-byte pairs, [pair][column] of double2, so the
// flux stage reads two quantities per LDS.128 (the row step is bound by shared-memory
// instructions).  Ring pairs (read by neighbours): (v0, v1) (v2, T) (B0, B1) (B2, p_tot);
// centre pairs (read by the cell's own thread only): (rho, E) (mx, my).
enum : int { PQ_V01 = 0, PQ_V2T, PQ_B01, PQ_B2P, NQP };
enum : int { PC_RE = 0, PC_M, NCP };

// pressure / admissibility / primitives (mhd.py:106-131, 176-181, 217-221)
__device__ __forceinline__ void cell_prims(const StencilParams& P, const double u[NF],
                                           double2* q, double2* cq, int qs, int& flag,
                                           double* qreg = nullptr) {
  const double rho = u[0], mx = u[1], my = u[2], mz = u[3];
  const double b0 = u[4], b1 = u[5], b2 = u[6], en = u[7];
  if (P.check && rho <= 0.0) flag |= ST_RHO;
  const double m2 = __dadd_rn(__dadd_rn(__dmul_rn(mx, mx), __dmul_rn(my, my)), __dmul_rn(mz, mz));
  const double bb = __dadd_rn(__dadd_rn(__dmul_rn(b0, b0), __dmul_rn(b1, b1)), __dmul_rn(b2, b2));
  const double rr = 1.0 / rho;                 // RN(1/rho): one IEEE division per cell
  const double kin = div_const(__dmul_rn(0.5, m2), rho, rr);
  const double mag = __dmul_rn(P.bfac, bb);
  const double p = __dmul_rn(P.gm1, __dsub_rn(__dsub_rn(en, kin), mag));
  if (P.check && p <= 0.0) flag |= ST_PRESSURE;
  const double v0 = div_const(mx, rho, rr);   // == mx / rho bit for bit
  const double v1 = div_const(my, rho, rr);
  const double v2 = div_const(mz, rho, rr);
  const double tt = div_const(p, rho, rr);
  const double pt = __dadd_rn(p, __dmul_rn(0.5, bb));
  cq[PC_RE * qs] = make_double2(rho, en);
  cq[PC_M * qs] = make_double2(mx, my);
  q[PQ_B01 * qs] = make_double2(b0, b1);
  q[PQ_V01 * qs] = make_double2(v0, v1);
  q[PQ_V2T * qs] = make_double2(v2, tt);
  q[PQ_B2P * qs] = make_double2(b2, pt);
  if (qreg) {
    qreg[Q_V0] = v0; qreg[Q_V1] = v1; qreg[Q_V2] = v2;
    qreg[Q_B0] = b0; qreg[Q_B1] = b1; qreg[Q_B2] = b2; qreg[Q_T] = tt;
  }
}

// x- and y-flux G = F_hyp - F_diff at one cell (mhd.py:174-197, 209-266, 275-276).
// c: prim column slot of the cell; qm/q0/qp: prim rows i-1, i, i+1; c0: centre row i.
template <int FXY>
__device__ __forceinline__ void flux_cell(const StencilParams& P, const double2* qm,
                                          const double2* q0, const double2* qp, const double2* c0,
                                          int c, int qs,
                                          bool need_x, bool need_y, double gx[NF], double gy[NF],
                                          const double* qpreg = nullptr) {
  const double thx = P.two_hx, rhx = P.r_two_hx, thy = P.two_hy, rhy = P.r_two_hy;
  // row i+1 of the own column: from registers when the caller kept them (QPR)
  const double2 pV = qpreg ? make_double2(qpreg[Q_V0], qpreg[Q_V1]) : qp[PQ_V01 * qs + c];
  const double2 pB = qpreg ? make_double2(qpreg[Q_B0], qpreg[Q_B1]) : qp[PQ_B01 * qs + c];
  const double2 mV = qm[PQ_V01 * qs + c], mB = qm[PQ_B01 * qs + c];
  const double2 rV = q0[PQ_V01 * qs + c + 1], lV = q0[PQ_V01 * qs + c - 1];
  const double2 rB = q0[PQ_B01 * qs + c + 1], lB = q0[PQ_B01 * qs + c - 1];
  // centred derivatives of v, B, T at the cell (mhd.py:224-227, 261, 264)
  const double dvx0 = div_c<FXY>(__dsub_rn(pV.x, mV.x), thx, rhx);
  const double dvx1 = div_c<FXY>(__dsub_rn(pV.y, mV.y), thx, rhx);
  const double dvy0 = div_c<FXY>(__dsub_rn(rV.x, lV.x), thy, rhy);
  const double dvy1 = div_c<FXY>(__dsub_rn(rV.y, lV.y), thy, rhy);
  const double dBx1 = div_c<FXY>(__dsub_rn(pB.y, mB.y), thx, rhx);
  const double dBy0 = div_c<FXY>(__dsub_rn(rB.x, lB.x), thy, rhy);

  const double2 cRE = c0[PC_RE * qs + c], cM = c0[PC_M * qs + c];
  const double2 cV = q0[PQ_V01 * qs + c], cV2 = q0[PQ_V2T * qs + c];
  const double2 cB = q0[PQ_B01 * qs + c], cB2 = q0[PQ_B2P * qs + c];
  const double rho = cRE.x, en = cRE.y, pt = cB2.y;
  const double v0 = cV.x, v1 = cV.y, v2 = cV2.x;
  const double b0 = cB.x, b1 = cB.y, b2 = cB2.x;
  const double mu = P.mu, eta = P.eta, heat = P.heat;

  const double divv = __dadd_rn(dvx0, dvy1);
  const double c23d = __dmul_rn(2.0 / 3.0, divv);
  const double tau_xy = __dadd_rn(dvy0, dvx1);
  const double curl = __dsub_rn(dBx1, dBy0);               // dBx[1] - dBy[0]
  const double bv = __dadd_rn(__dadd_rn(__dmul_rn(b0, v0), __dmul_rn(b1, v1)), __dmul_rn(b2, v2));
  const double ept = __dadd_rn(en, pt);
  const double r0 = __dmul_rn(rho, v0), r1 = __dmul_rn(rho, v1), r2 = __dmul_rn(rho, v2);

  if (need_x) {
    const double2 pV2 = qpreg ? make_double2(qpreg[Q_V2], qpreg[Q_T]) : qp[PQ_V2T * qs + c];
    const double pB2 = qpreg ? qpreg[Q_B2] : qp[PQ_B2P * qs + c].x;
    const double2 mV2 = qm[PQ_V2T * qs + c];
    const double dvx2 = div_c<FXY>(__dsub_rn(pV2.x, mV2.x), thx, rhx);
    const double dBx2 = div_c<FXY>(__dsub_rn(pB2, qm[PQ_B2P * qs + c].x), thx, rhx);
    const double dTx = div_c<FXY>(__dsub_rn(pV2.y, mV2.y), thx, rhx);
    const double tau_xx = __dsub_rn(__dmul_rn(2.0, dvx0), c23d);
    // diffusive x-flux (mhd.py:244-262)
    const double fmx = __dmul_rn(mu, tau_xx);
    const double fmy = __dmul_rn(mu, tau_xy);
    const double fmz = __dmul_rn(mu, dvx2);
    const double fby = __dmul_rn(eta, curl);
    const double fbz = __dmul_rn(eta, dBx2);
    const double visc = __dmul_rn(mu, __dadd_rn(__dadd_rn(__dmul_rn(tau_xx, v0), __dmul_rn(tau_xy, v1)),
                                                __dmul_rn(dvx2, v2)));
    const double res = __dmul_rn(eta, __dadd_rn(__dmul_rn(b1, curl), __dmul_rn(b2, dBx2)));
    const double fen = __dadd_rn(__dadd_rn(visc, __dmul_rn(heat, dTx)), res);
    // hyperbolic x-flux (mhd.py:185-196) minus diffusive
    gx[0] = cM.x;
    gx[1] = __dsub_rn(__dadd_rn(__dsub_rn(__dmul_rn(r0, v0), __dmul_rn(b0, b0)), pt), fmx);
    gx[2] = __dsub_rn(__dsub_rn(__dmul_rn(r1, v0), __dmul_rn(b1, b0)), fmy);
    gx[3] = __dsub_rn(__dsub_rn(__dmul_rn(r2, v0), __dmul_rn(b2, b0)), fmz);
    gx[4] = __dsub_rn(__dmul_rn(v0, b0), __dmul_rn(b0, v0));
    gx[5] = __dsub_rn(__dsub_rn(__dmul_rn(v0, b1), __dmul_rn(b0, v1)), fby);
    gx[6] = __dsub_rn(__dsub_rn(__dmul_rn(v0, b2), __dmul_rn(b0, v2)), fbz);
    gx[7] = __dsub_rn(__dsub_rn(__dmul_rn(ept, v0), __dmul_rn(b0, bv)), fen);
  }
  if (need_y) {
    const double2 rV2 = q0[PQ_V2T * qs + c + 1], lV2 = q0[PQ_V2T * qs + c - 1];
    const double dvy2 = div_c<FXY>(__dsub_rn(rV2.x, lV2.x), thy, rhy);
    const double dBy2 = div_c<FXY>(__dsub_rn(q0[PQ_B2P * qs + c + 1].x, q0[PQ_B2P * qs + c - 1].x), thy, rhy);
    const double dTy = div_c<FXY>(__dsub_rn(rV2.y, lV2.y), thy, rhy);
    const double tau_yy = __dsub_rn(__dmul_rn(2.0, dvy1), c23d);
    // diffusive y-flux (mhd.py:245-265)
    const double fmx = __dmul_rn(mu, tau_xy);
    const double fmy = __dmul_rn(mu, tau_yy);
    const double fmz = __dmul_rn(mu, dvy2);
    const double fbx = -__dmul_rn(eta, curl);                 // fy[BX] = -fx[BY]
    const double fbz = __dmul_rn(eta, dBy2);
    const double visc = __dmul_rn(mu, __dadd_rn(__dadd_rn(__dmul_rn(tau_xy, v0), __dmul_rn(tau_yy, v1)),
                                                __dmul_rn(dvy2, v2)));
    const double res = __dmul_rn(eta, __dadd_rn(__dmul_rn(b0, __dsub_rn(dBy0, dBx1)), __dmul_rn(b2, dBy2)));
    const double fen = __dadd_rn(__dadd_rn(visc, __dmul_rn(heat, dTy)), res);
    gy[0] = cM.y;
    gy[1] = __dsub_rn(__dsub_rn(__dmul_rn(r0, v1), __dmul_rn(b0, b1)), fmx);
    gy[2] = __dsub_rn(__dadd_rn(__dsub_rn(__dmul_rn(r1, v1), __dmul_rn(b1, b1)), pt), fmy);
    gy[3] = __dsub_rn(__dsub_rn(__dmul_rn(r2, v1), __dmul_rn(b2, b1)), fmz);
    gy[4] = __dsub_rn(__dsub_rn(__dmul_rn(v1, b0), __dmul_rn(b1, v0)), fbx);
    gy[5] = __dsub_rn(__dmul_rn(v1, b1), __dmul_rn(b1, v1));
    gy[6] = __dsub_rn(__dsub_rn(__dmul_rn(v1, b2), __dmul_rn(b1, v2)), fbz);
    gy[7] = __dsub_rn(__dsub_rn(__dmul_rn(ept, v1), __dmul_rn(b1, bv)), fen);
  }
}

// raw input rows in flight per CTA (NR): row r+NR is requested while row r is consumed.  NR = 2
// comes with the halo warp (HW below) and, on grids wider than 64 columns, 64-column strips at
// 4 CTAs/SM (12 warps: 8 column warps + 4 halo warps, the register file exactly full at 168
// registers): four independent per-row barrier groups of three warps instead of two groups of
// five.  Back-to-back launches (tools/bench_jvn.py), two rows + halo warp, strip 64 / 128 (one row,
// no halo warp, 128 columns in brackets): normalised Jv 1024^2 64.6 / 72.1 us (87.5), 2048^2
// 236 / 267 us (313), 4096^2 938 / 1037 us (1218); Jv 1024^2 59.2 / 59.7 us (67.7), 2048^2
// 215 / 219 us (242); RHS 1024^2 47.1 / 44.9 us (43.5), 2048^2 172 / 164 us (151): the RHS keeps
// one row at 3 CTAs/SM; 32-column strips (6 CTAs/SM) and 96-column strips (3 CTAs/SM) lose
// everywhere.  sel.raw_rows forces 1 or 2 for every mode.
static bool two_raw_rows(int mode, const StencilParams& P, const StencilPath& sel) {
  (void)P;
  if (sel.raw_rows == 0) return mode != MODE_RHS;
  return sel.raw_rows == 2;
}

// HW (with two staged rows; 4 CTAs/SM at 64 columns, 2 at 128): one extra warp per CTA does the strip's halo work (the
// four halo columns' primitives and the two halo y-fluxes) beside the TY column threads, so no
// column warp carries extra work into the per-row barrier
template <int TY, int MODE, bool AUG, int FXY, int NR>
__global__ void __launch_bounds__(NR == 2 ? TY + 32 : TY, NR == 2 ? (TY == 64 ? 4 : 2) : 384 / TY)
    stencil_kernel(const StencilParams P) {
  constexpr bool HW = NR == 2;
  constexpr int QW = TY + 4;         // prim columns (2-cell halo each side)
  constexpr int GYW = TY + 2;        // y-flux columns (1-cell halo each side)
  extern __shared__ __align__(16) double smem[];
  // rings sized so ONE barrier per row step suffices (see the loop): primitives 4 rows,
  // y-fluxes 2 rows, thread-private centre quantities 2 rows, NRAW raw rows in flight;
  // x-fluxes live in registers of the column's own thread.  ~76 KB at TY=128 with one raw
  // row (2-3 CTAs/SM), ~49 KB at TY=64 with two (4 CTAs/SM)
  double2* qring = reinterpret_cast<double2*>(smem);              // [4][NQP][QW] pairs
  double2* gyring = qring + 4 * NQP * QW;                         // [2][NF/2][GYW] pairs (f, f+1)
  double2* cring = gyring + 2 * (NF / 2) * GYW;                   // [2][NCP][QW] pairs
  constexpr int NARR = MODE == MODE_RHS ? 1 : 2;
  constexpr int NRAW = NR;
  double* rawring = reinterpret_cast<double*>(cring + 2 * NCP * QW);   // [NRAW][NARR*NF][QW] raw rows in flight
  unsigned long long* rbar = reinterpret_cast<unsigned long long*>(rawring + NRAW * NARR * NF * QW);
  // QPR: the own column's next-row primitives stay in registers from the primitive stage to the
  // flux stage; measured (tools/bench_jvn.py): RHS 1024^2 42.3 -> 41.5 us, 2048^2 145.8 -> 142.9 us; the Jv
  // variants are at their 168-register cap (4 CTAs/SM) and spill with it (normalised Jv 64.7 ->
  // 85.9 us), so only the RHS takes it
  constexpr bool QPR = EMHD_QP_REG != 0 && MODE == MODE_RHS;

  pdl_sync();
  const int tid = threadIdx.x;
  const int warp_u = __shfl_sync(0xffffffffu, tid >> 5, 0);   // warp index, known warp-uniform
  const int t = HW ? tid - 32 : tid;               // column thread index (< 0: the halo warp)
  const int j0 = blockIdx.x * TY;
  // output rows [i0, i1) of this CTA: a chunk of [row_lo, row_hi) (rows_mode 0/1), or the
  // two edge row pairs {0, 1} / {nx-2, nx-1} (rows_mode 2, the launch that waits for the halo)
  int i0, i1;
  if (P.rows_mode == 2) {
    i0 = blockIdx.y == 0 ? 0 : P.nx - 2;
    i1 = i0 + 2;
  } else {
    i0 = P.row_lo + blockIdx.y * P.rows_per_cta;
    i1 = min(i0 + P.rows_per_cta, P.row_hi);
  }
  // the launch's bookkeeping (RHS count, evals, augmented tail) is done by the counting launch
  const bool head = P.count && blockIdx.x == 0 && blockIdx.y == 0;
  const bool lead = head && tid == 0;
  if (P.skip && *P.skip != 0.0) {
    // cancelled look-ahead iteration (its gate was written by an earlier launch)
    if (lead && P.evals) *P.evals = 0.0;
    return;
  }
  if (i0 >= i1) return;

  // per-call scalars: sigma, 1/sigma, h_next, 1/h_next
  double sigma = 1.0, rsig = 1.0, hnext = 1.0, rh = 1.0;
  bool skip_stencil = false;
  if (MODE == MODE_JV) {
    const double vn = P.scal[0];
    skip_stencil = (vn == 0.0);
    sigma = fd_sigma(vn);
    rsig = 1.0 / sigma;
  } else if (MODE == MODE_JVN) {
    if (P.scal[2] != 0.0) {
      // the previous iteration broke down: this launch was queued ahead of the host's
      // breakdown check; leave no trace (zero output, no flags, no RHS count)
      for (long long r = i0; r < i1; ++r)
        if (t >= 0 && t < min(TY, P.ny - j0))
#pragma unroll
          for (int f = 0; f < NF; ++f) P.out[r * P.ny + j0 + t + (long long)f * P.nx * P.ny] = 0.0;
      if (head && t >= 0 && t < P.p) P.out[P.n_top + t] = 0.0;
      if (lead && P.evals) *P.evals = 0.0;
      return;
    }
    hnext = P.scal[0];
    rh = 1.0 / hnext;
    const double vn = P.scal[1] / hnext;   // max|w/h| == fl(max|w| / h) (monotone rounding)
    skip_stencil = (vn == 0.0);
    sigma = fd_sigma(vn);
    rsig = 1.0 / sigma;
  }
  const bool fsig = recip_tight(sigma, rsig);   // one-correction division by sigma is exact
  const bool fh = recip_tight(hnext, rh);

  // augmented tail q of the current basis vector (krylov.py:268-273)
  double qv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (AUG) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (k < P.p) {
        if (MODE == MODE_JVN) qv[k] = div_const(P.v[P.n_top + k], hnext, rh);
        else qv[k] = P.qsrc[k];
      }
    }
  }
  double qb[5];
  aug_coefs(P, qv, qb);

  const int ncols_out = min(TY, P.ny - j0);
  const unsigned plane = (unsigned)P.nx * (unsigned)P.ny;   // field stride of out / fa / vout
  int flag = 0;
  unsigned long long bad = ~0ull;

  if (skip_stencil) {
    // zero direction: Jv = 0 without an RHS evaluation (fdjac.py:41-42)
    for (int r = i0; r < i1; ++r) {
      if (t >= 0 && t < ncols_out) {
        const long long o = (long long)r * P.ny + j0 + t;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const long long idx = o + (long long)f * P.nx * P.ny;
          double val = 0.0;
          if (AUG) val = aug_add(P, qb, (unsigned long long)idx, __dmul_rn(P.ch, 0.0));
          P.out[idx] = val;
          if (MODE == MODE_JVN) P.vout[idx] = div_const(__ldg(P.v + idx), hnext, rh);
        }
      }
    }
  } else {
    // column slots handled by this thread: main slot c = t + 2 (column j0 + t), extra
    // halo slots 1, 0, TY+3, TY+2 (threads 0..3: all four in warp 0, so the halo columns cost
    // ONE extra warp-wide evaluation per row instead of one in each edge warp); the threads
    // that compute the halo y-fluxes (slots 1 and TY+2: threads 0 and 3) own those columns'
    // centre quantities
    const int cmain = t + 2;
    const int cextra = HW ? (tid == 0 ? 1 : tid == 1 ? 0 : tid == 2 ? TY + 3 : tid == 3 ? TY + 2 : -1)
                          : (t == 0 ? 1 : t == 1 ? 0 : t == 2 ? TY + 3 : t == 3 ? TY + 2 : -1);
    auto col_ok = [&](int c) { int j = j0 - 2 + c; return j >= -2 && j <= P.ny + 1; };
    bool fm, fe = false;
    const int jm = map_ghost(j0 - 2 + cmain, P.ny, P.bcy, fm);
    const int je = cextra >= 0 ? map_ghost(j0 - 2 + cextra, P.ny, P.bcy, fe) : 0;
    const unsigned ymm = fm ? 0x80000000u : 0u, yme = fe ? 0x80000000u : 0u;
    const bool okm = t >= 0 && col_ok(cmain), oke = cextra >= 0 && col_ok(cextra);

    // prologue: primitives of rows i0-2 and i0-1
    for (int r = i0 - 2; r < i0; ++r) {
      const RowRef R = row_ref(P, r);
      double2* q = qring + ((r + 4) % 4) * NQP * QW;
      double2* cq = cring + ((r + 2) % 2) * NCP * QW;
      double u[NF];
      if (okm) {
        load_cell<MODE>(P, R, jm, fm, sigma, hnext, rh, u);
        cell_prims(P, u, q + cmain, cq + cmain, QW, flag);
      }
      if (oke) {
        load_cell<MODE>(P, R, je, fe, sigma, hnext, rh, u);
        cell_prims(P, u, q + cextra, cq + cextra, QW, flag);
      }
    }
    // software pipeline: the raw inputs of row r+1 stream into the shared raw row while the
    // fluxes of row r-1 and outputs of row r-2 are computed
    double fa_pre[NF];                       // F(a) of the next output row, one step ahead
    if (MODE != MODE_RHS && t >= 0 && t < ncols_out) {
      const unsigned o = (unsigned)i0 * P.ny + j0 + t;
#pragma unroll
      for (int f = 0; f < NF; ++f) fa_pre[f] = __ldg(P.fa + (o + f * plane));
    }
    double gxA[NF], gxB[NF], gxC[NF];        // x-fluxes of rows r-3, r-2, r-1 (own column)
#pragma unroll
    for (int f = 0; f < NF; ++f) { gxA[f] = 0.0; gxB[f] = 0.0; gxC[f] = 0.0; }
    // interior strips (no y-ghost columns) stream whole row segments with bulk async copies
    // issued by thread 0 (tracked by one mbarrier); edge strips keep per-thread cp.async
    const bool bulk = P.tma && j0 >= 2 && j0 + TY + 2 <= P.ny;
    constexpr int SLOT = NARR * NF * QW;     // doubles per raw row slot
    if (bulk) {
      if (warp_u == 0 && elect_one()) {
        for (int k = 0; k < NRAW; ++k) mbar_init(rbar + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        for (int k = 0; k < NRAW && i0 + k <= i1 + 1; ++k)
          fetch_row_bulk<MODE, QW>(P, row_ref(P, i0 + k), j0 - 2, rawring + k * SLOT, rbar + k);
      }
      __syncthreads();
    } else {
      // per-thread cp.async: every thread consumes only the cells it copied itself
      for (int k = 0; k < NRAW; ++k) {
        if (i0 + k <= i1 + 1) {
          const RowRef R = row_ref(P, i0 + k);
          if (okm) fetch_async<MODE, QW>(P, R, jm, cmain, rawring + k * SLOT);
          if (oke) fetch_async<MODE, QW>(P, R, je, cextra, rawring + k * SLOT);
        }
        cp_commit();
      }
    }
    for (int r = i0; r <= i1 + 1; ++r) {
      const int rk = r - i0;
      double* sraw = rawring + (rk % NRAW) * SLOT;
      if (bulk) mbar_wait(rbar + rk % NRAW, (unsigned)((rk / NRAW) & 1));
      else cp_wait<NRAW - 1>();              // row r has landed (later rows may be in flight)
      // ---- primitives of row r (QPR: the own column's shared primitives also stay in registers
      // for this step's fluxes of row r-1, whose x-derivatives read row r: 6 shared loads less)
      double qown[NQ];
      {
        const RowRef Rr = row_ref(P, r);
        double2* q = qring + ((r + 4) % 4) * NQP * QW;
        double2* cq = cring + ((r + 2) % 2) * NCP * QW;
        double u[NF];
        if (okm) {
          RawCell<MODE> xm;
          consume_raw<MODE, QW>(sraw, cmain, xm);
          double vj[MODE == MODE_JVN ? NF : 1];
          combine_cell<MODE>(xm, Rr.flip ? 0x80000000u : 0u, ymm, sigma, hnext, rh, fh, u,
                             MODE == MODE_JVN ? vj : nullptr);
          cell_prims(P, u, q + cmain, cq + cmain, QW, flag, QPR ? qown : nullptr);
          if (MODE == MODE_JVN && r >= i0 && r < i1 && t < ncols_out) {
            // v_j = w / h_next of an owned cell (krylov.py:167), computed once for the stencil
            // input above (the ghost flips apply to u only, never to the stored basis entry)
            const unsigned o = (unsigned)r * P.ny + j0 + t;
#pragma unroll
            for (int f = 0; f < NF; ++f) P.vout[o + f * plane] = vj[f];
          }
        }
        if (oke) {
          RawCell<MODE> xe;
          consume_raw<MODE, QW>(sraw, cextra, xe);
          combine_cell<MODE>(xe, Rr.flip ? 0x80000000u : 0u, yme, sigma, hnext, rh, fh, u);
          cell_prims(P, u, q + cextra, cq + cextra, QW, flag);
        }
      }
      // refill the consumed raw row with row r+1 (each thread its own cells; the bulk path
      // refills after the barrier below, once every thread has consumed the row)
      if (!bulk) {
        if (r + NRAW <= i1 + 1) {
          const RowRef R1 = row_ref(P, r + NRAW);
          if (okm) fetch_async<MODE, QW>(P, R1, jm, cmain, sraw);
          if (oke) fetch_async<MODE, QW>(P, R1, je, cextra, sraw);
        }
        cp_commit();
      }
      // The only barrier of the step.  RAW: fluxes of row r-1 read primitives of row r
      // (just written) and outputs of row r-2 read y-fluxes of row r-2 (previous step).
      // WAR is covered by ring depth: primitives of row r+1 overwrite row r-3 (last read by
      // the fluxes of row r-2, previous step); y-fluxes of row r-1 (this step) overwrite
      // row r-3 (last read by the outputs of row r-3, previous step); centre quantities
      // are private to their thread.
      __syncthreads();
      if (bulk && warp_u == 0 && r + NRAW <= i1 + 1) {
        // warp-uniform branch, one elected lane issues: the row's source addresses stay in
        // uniform registers (no per-copy vector-to-uniform hand-over).
        // generic-proxy reads of the row (before the barrier) precede the async-proxy refill
        if (elect_one()) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          fetch_row_bulk<MODE, QW>(P, row_ref(P, r + NRAW), j0 - 2, sraw, rbar + rk % NRAW);
        }
      }
      // ---- fluxes of row rf = r - 1
      const int rf = r - 1;
      if (rf >= i0 - 1) {
        const double2* qm = qring + ((rf + 3) % 4) * NQP * QW;
        const double2* q0 = qring + ((rf + 4) % 4) * NQP * QW;
        const double2* qp = qring + ((rf + 5) % 4) * NQP * QW;
        const double2* c0 = cring + ((rf + 2) % 2) * NCP * QW;
        double2* gyr = gyring + ((rf + 2) % 2) * (NF / 2) * GYW;
        const bool out_row = (rf >= i0 && rf < i1);
        double gy[NF];
        if (t >= 0 && t < ncols_out) {
          flux_cell<FXY>(P, qm, q0, qp, c0, cmain, QW, true, out_row, gxC, gy, QPR ? qown : nullptr);
          if (out_row) {
#pragma unroll
            for (int f = 0; f < NF; f += 2) gyr[(f / 2) * GYW + t + 1] = make_double2(gy[f], gy[f + 1]);
          }
        }
        if (out_row) {
          // y-fluxes at the strip's halo columns j0-1 (thread 0, extra slot 1) and
          // j0+ncols (thread 3's extra slot TY+2 on a full strip, else the main slot of
          // thread ncols): each computed by the owner of that column's centre quantities
          int cs = -1, gslot = 0;
          // (HW: the halo warp's lanes 0 and 3 own slots 1 and TY+2; a ragged strip's right
          // halo column is column thread ncols's main slot)
          if ((HW ? tid : t) == 0) { cs = 1; gslot = 0; }
          if (ncols_out == TY ? (HW ? tid == 3 : t == 3) : t == ncols_out) {
            cs = ncols_out + 2;
            gslot = ncols_out + 1;
          }
          if (cs >= 0) {
            double gdummy[NF];
            flux_cell<FXY>(P, qm, q0, qp, c0, cs, QW, false, true, gdummy, gy);
#pragma unroll
            for (int f = 0; f < NF; f += 2) gyr[(f / 2) * GYW + gslot] = make_double2(gy[f], gy[f + 1]);
          }
        }
      }
      // ---- output row ro = r - 2: x-fluxes of rows ro+1 (gxC) and ro-1 (gxA) are this
      // thread's own registers; y-fluxes of row ro come from the ring (previous step)
      const int ro = r - 2;
      if (ro >= i0 && t >= 0 && t < ncols_out) {
        const double2* gyr = gyring + ((ro + 2) % 2) * (NF / 2) * GYW;
        double gyp[NF], gym[NF];             // y-fluxes at columns j+1, j-1 (two fields per load)
#pragma unroll
        for (int f = 0; f < NF; f += 2) {
          const double2 a = gyr[(f / 2) * GYW + t + 2], b = gyr[(f / 2) * GYW + t];
          gyp[f] = a.x; gyp[f + 1] = a.y; gym[f] = b.x; gym[f + 1] = b.y;
        }
        const unsigned o = (unsigned)ro * P.ny + j0 + t;
        // |F| high words: F of field f is inf / nan <=> fhi[f] >= 0x7ff00000 (one AND per field
        // and a running maximum; which field only matters on the rare path below)
        unsigned fhi[NF], fhmax = 0;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const double ddx = div_c<FXY>(__dsub_rn(gxC[f], gxA[f]), P.two_hx, P.r_two_hx);
          const double ddy = div_c<FXY>(__dsub_rn(gyp[f], gym[f]), P.two_hy, P.r_two_hy);
          double F = __dsub_rn(-ddx, ddy);                    // -ddx(gx) - ddy(gy) (mhd.py:277)
          const unsigned idx = o + f * plane;
          if (MODE == MODE_RHS) {
            P.out[idx] = F;
          } else {
            fhi[f] = (unsigned)__double2hiint(F) & 0x7fffffffu;
            fhmax = max(fhmax, fhi[f]);
            const double df = __dsub_rn(F, fa_pre[f]);
            double jv = fsig ? div_const1(df, sigma, rsig) : div_const(df, sigma, rsig);   // fdjac.py:49
            if (AUG) jv = aug_add(P, qb, idx, __dmul_rn(P.ch, jv));
            P.out[idx] = jv;
          }
        }
        if (MODE != MODE_RHS && fhmax >= 0x7ff00000u) {
          // rare path: flat index (global (8, nxg, ny) order) of the first bad field
          int fb = NF - 1;
#pragma unroll
          for (int f = NF - 2; f >= 0; --f) fb = fhi[f] >= 0x7ff00000u ? f : fb;
          const unsigned long long gidx = (unsigned long long)fb * P.nxg * P.ny +
              (unsigned long long)(P.x_off + ro) * P.ny + j0 + t;
          bad = gidx < bad ? gidx : bad;
        }
        if (MODE != MODE_RHS && ro + 1 < i1) {
          const unsigned o2 = o + P.ny;
#pragma unroll
          for (int f = 0; f < NF; ++f) fa_pre[f] = __ldg(P.fa + (o2 + f * plane));
        }
        if (AUG && EMHD_PFB > 0 && ro + EMHD_PFB < i1 && (t & 3) == 0) {
          // the B columns of the augmented epilogue are read just in time (no registers to
          // stage them): ask L2 for the next output row's values, one request per 32-byte sector
          // (augmented normalised Jv 1024^2 126.5 -> 117.9 us, 2048^2 479 -> 428 us; two rows
          // ahead, an L1 hint, bulk L2 prefetches and the same for F(a): no further gain)
          const unsigned o3 = o + EMHD_PFB * P.ny;
#pragma unroll
          for (int k = 0; k < 5; ++k)
            if (k < P.nb) {
#pragma unroll
              for (int f = 0; f < NF; ++f)
                asm volatile("prefetch.global.L2 [%0];\n" ::"l"(P.bcol[k] + (o3 + f * plane)));
            }
        }
      }
#pragma unroll
      for (int f = 0; f < NF; ++f) { gxA[f] = gxB[f]; gxB[f] = gxC[f]; }
    }
  }

  // tail of the augmented output: bottom = upshift(q) (krylov.py:271-272); v_j tail
  if (AUG && head && t >= 0 && t < P.p) {
    double nxt = 0.0;
#pragma unroll
    for (int k = 1; k < 5; ++k) if (k == t + 1 && k < P.p) nxt = qv[k];
    P.out[P.n_top + t] = nxt;
    if (MODE == MODE_JVN) {
      double cur = 0.0;
#pragma unroll
      for (int k = 0; k < 5; ++k) if (k == t) cur = qv[k];
      P.vout[P.n_top + t] = cur;
    }
  }

  // status aggregation: one atomic per CTA
  __shared__ int s_flag;
  __shared__ unsigned long long s_bad;
  if (tid == 0) { s_flag = 0; s_bad = ~0ull; }
  __syncthreads();
  if (flag) atomicOr(&s_flag, flag);
  if (bad != ~0ull) atomicMin(&s_bad, bad);
  __syncthreads();
  if (tid == 0) {
    if (s_flag) {
      atomicOr(&P.st->flags, s_flag);
      atomicMin(&P.st->fail_iter, P.epoch);
    }
    if (s_bad != ~0ull) {
      atomicOr(&P.st->flags, (int)ST_NONFINITE);
      atomicMin(&P.st->first_nonfinite, s_bad);
      atomicMin(&P.st->fail_iter, P.epoch);
    }
    if (!skip_stencil && head) atomicAdd(&P.st->rhs_evals, 1);
    if (P.evals && head) *P.evals = skip_stencil ? 0.0 : 1.0;
  }
}


// ---- small grids: one thread per output cell on a 2D tile -------------------------------
// The row-marching kernel above pays (rows + 4) dependent row steps per CTA; on small grids
// (a few rows per CTA) that latency dominates.  Here a CTA owns a TR x TC tile and runs three
// barrier-separated phases over it: primitives of the (TR+4) x (TC+4) halo region, x/y fluxes
// of the cells around the tile, then the outputs.  Every value is produced by the same device
// functions in the same operation order as the marching kernel, so outputs are bit-identical.
constexpr int TT_R = 8, TT_C = 32, TT_THREADS = TT_R * TT_C;
constexpr int TT_QR = TT_R + 4, TT_QC = TT_C + 4, TT_QN = TT_QR * TT_QC;   // primitive region

size_t tile_stencil_smem() {
  return sizeof(double) * ((size_t)2 * (NQP + NCP) * TT_QN + (size_t)NF * (TT_R + 2) * TT_C +
                           (size_t)NF * TT_R * (TT_C + 2));
}

template <int MODE, bool AUG, int FXY>
__global__ void __launch_bounds__(TT_THREADS, 2) tile_stencil_kernel(const StencilParams P) {
  extern __shared__ __align__(16) double smem[];
  double2* q = reinterpret_cast<double2*>(smem);      // [NQP][TT_QR][TT_QC] pairs
  double2* cq = q + NQP * TT_QN;                      // [NCP][TT_QR][TT_QC] pairs
  double* gxs = reinterpret_cast<double*>(cq + NCP * TT_QN);   // [NF][TT_R + 2][TT_C]   rows -1 .. TR
  double* gys = gxs + NF * (TT_R + 2) * TT_C;         // [NF][TT_R][TT_C + 2]   cols -1 .. TC
  pdl_sync();
  const int t = threadIdx.x;
  const int j0 = blockIdx.x * TT_C;
  int i0, nro;                                         // output rows [i0, i0 + nro)
  if (P.rows_mode == 2) {
    i0 = blockIdx.y == 0 ? 0 : P.nx - 2;
    nro = 2;
  } else {
    i0 = P.row_lo + blockIdx.y * TT_R;
    nro = min(TT_R, P.row_hi - i0);
  }
  const bool head = P.count && blockIdx.x == 0 && blockIdx.y == 0;
  const bool lead = head && t == 0;
  if (P.skip && *P.skip != 0.0) {
    if (lead && P.evals) *P.evals = 0.0;
    return;
  }
  const int nco = min(TT_C, P.ny - j0);                // output extent
  const unsigned plane = (unsigned)P.nx * (unsigned)P.ny;
  double sigma = 1.0, rsig = 1.0, hnext = 1.0, rh = 1.0;
  bool skip_stencil = false;
  if (MODE == MODE_JV) {
    const double vn = P.scal[0];
    skip_stencil = (vn == 0.0);
    sigma = fd_sigma(vn);
    rsig = 1.0 / sigma;
  } else if (MODE == MODE_JVN) {
    if (P.scal[2] != 0.0) {
      // queued after a breakdown: zero output, no flags, no RHS count (as the marching kernel)
      const int r = t / TT_C, c = t % TT_C;
      if (r < nro && c < nco)
        for (int f = 0; f < NF; ++f) P.out[(unsigned)(i0 + r) * P.ny + j0 + c + f * plane] = 0.0;
      if (lead) for (int k = 0; k < P.p; ++k) P.out[P.n_top + k] = 0.0;
      if (lead && P.evals) *P.evals = 0.0;
      return;
    }
    hnext = P.scal[0];
    rh = 1.0 / hnext;
    const double vn = P.scal[1] / hnext;
    skip_stencil = (vn == 0.0);
    sigma = fd_sigma(vn);
    rsig = 1.0 / sigma;
  }
  const bool fsig = recip_tight(sigma, rsig);
  const bool fh = recip_tight(hnext, rh);
  double qv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (AUG) {
#pragma unroll
    for (int k = 0; k < 5; ++k)
      if (k < P.p) qv[k] = MODE == MODE_JVN ? div_const(P.v[P.n_top + k], hnext, rh) : P.qsrc[k];
  }
  double qb[5];
  aug_coefs(P, qv, qb);
  int flag = 0;
  unsigned long long bad = ~0ull;
  const int ro = t / TT_C, co = t % TT_C;              // this thread's output cell
  const bool own = ro < nro && co < nco;
  const unsigned o = (unsigned)(i0 + ro) * P.ny + j0 + co;

  if (skip_stencil) {
    if (own) {
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const unsigned idx = o + f * plane;
        double val = 0.0;
        if (AUG) val = aug_add(P, qb, idx, __dmul_rn(P.ch, 0.0));
        P.out[idx] = val;
        if (MODE == MODE_JVN) P.vout[idx] = div_const(__ldg(P.v + idx), hnext, rh);
      }
    }
  } else {
    // phase 1: primitives of rows i0-2 .. i0+nro+1, columns j0-2 .. j0+nco+1
    for (int e = t; e < TT_QN; e += TT_THREADS) {
      const int rr = e / TT_QC, cc = e % TT_QC;
      if (rr >= nro + 4 || cc >= nco + 4) continue;
      const int i = i0 - 2 + rr, j = j0 - 2 + cc;
      const RowRef R = row_ref(P, i);
      bool yf;
      const int js = map_ghost(j, P.ny, P.bcy, yf);
      RawCell<MODE> x;
      fetch_cell<MODE>(P, R, js, x);
      double u[NF];
      double vj[MODE == MODE_JVN ? NF : 1];
      const bool owned = rr >= 2 && rr < nro + 2 && cc >= 2 && cc < nco + 2;
      combine_cell<MODE>(x, R.flip ? 0x80000000u : 0u, yf ? 0x80000000u : 0u, sigma, hnext, rh, fh, u,
                         (MODE == MODE_JVN && owned) ? vj : nullptr);
      cell_prims(P, u, q + e, cq + e, TT_QN, flag);
      if (MODE == MODE_JVN && owned) {
        const unsigned ov = (unsigned)i * P.ny + j;
#pragma unroll
        for (int f = 0; f < NF; ++f) P.vout[ov + f * plane] = vj[f];
      }
    }
    __syncthreads();
    // phase 2: x-fluxes at rows -1 .. nro (output columns), y-fluxes at columns -1 .. nco
    // (output rows); flux cell (fr, fc) sits at region cell (fr + 2, fc + 2)
    constexpr int FR = TT_R + 2, FC = TT_C + 2;
    for (int e = t; e < FR * FC; e += TT_THREADS) {
      const int fr = e / FC - 1, fc = e % FC - 1;
      const bool need_x = fc >= 0 && fc < nco && fr <= nro;
      const bool need_y = fr >= 0 && fr < nro && fc <= nco;
      if (!need_x && !need_y) continue;
      const int rr = fr + 2, cc = fc + 2;
      double gx[NF], gy[NF];
      flux_cell<FXY>(P, q + (rr - 1) * TT_QC, q + rr * TT_QC, q + (rr + 1) * TT_QC, cq + rr * TT_QC, cc,
                     TT_QN, need_x, need_y, gx, gy);
      if (need_x) {
#pragma unroll
        for (int f = 0; f < NF; ++f) gxs[(f * (TT_R + 2) + fr + 1) * TT_C + fc] = gx[f];
      }
      if (need_y) {
#pragma unroll
        for (int f = 0; f < NF; ++f) gys[(f * TT_R + fr) * (TT_C + 2) + fc + 1] = gy[f];
      }
    }
    __syncthreads();
    // phase 3: outputs (as the marching kernel's output stage)
    if (own) {
      unsigned fhi[NF], fhmax = 0;
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const double* gxf = gxs + f * (TT_R + 2) * TT_C;
        const double* gyf = gys + (f * TT_R + ro) * (TT_C + 2);
        const double ddx = div_c<FXY>(__dsub_rn(gxf[(ro + 2) * TT_C + co], gxf[ro * TT_C + co]), P.two_hx, P.r_two_hx);
        const double ddy = div_c<FXY>(__dsub_rn(gyf[co + 2], gyf[co]), P.two_hy, P.r_two_hy);
        const double F = __dsub_rn(-ddx, ddy);
        const unsigned idx = o + f * plane;
        if (MODE == MODE_RHS) {
          P.out[idx] = F;
        } else {
          fhi[f] = (unsigned)__double2hiint(F) & 0x7fffffffu;
          fhmax = max(fhmax, fhi[f]);
          const double df = __dsub_rn(F, __ldg(P.fa + idx));
          double jv = fsig ? div_const1(df, sigma, rsig) : div_const(df, sigma, rsig);
          if (AUG) jv = aug_add(P, qb, idx, __dmul_rn(P.ch, jv));
          P.out[idx] = jv;
        }
      }
      if (MODE != MODE_RHS && fhmax >= 0x7ff00000u) {
        int fb = NF - 1;
#pragma unroll
        for (int f = NF - 2; f >= 0; --f) fb = fhi[f] >= 0x7ff00000u ? f : fb;
        const unsigned long long gidx = (unsigned long long)fb * P.nxg * P.ny +
            (unsigned long long)(P.x_off + i0 + ro) * P.ny + j0 + co;
        bad = gidx < bad ? gidx : bad;
      }
    }
  }

  // tail of the augmented output: bottom = upshift(q) (krylov.py:271-272); v_j tail
  if (AUG && head && t < P.p) {
    double nxt = 0.0, cur = 0.0;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (k == t + 1 && k < P.p) nxt = qv[k];
      if (k == t) cur = qv[k];
    }
    P.out[P.n_top + t] = nxt;
    if (MODE == MODE_JVN) P.vout[P.n_top + t] = cur;
  }
  __shared__ int s_flag;
  __shared__ unsigned long long s_bad;
  if (t == 0) { s_flag = 0; s_bad = ~0ull; }
  __syncthreads();
  if (flag) atomicOr(&s_flag, flag);
  if (bad != ~0ull) atomicMin(&s_bad, bad);
  __syncthreads();
  if (t == 0) {
    if (s_flag) {
      atomicOr(&P.st->flags, s_flag);
      atomicMin(&P.st->fail_iter, P.epoch);
    }
    if (s_bad != ~0ull) {
      atomicOr(&P.st->flags, (int)ST_NONFINITE);
      atomicMin(&P.st->first_nonfinite, s_bad);
      atomicMin(&P.st->fail_iter, P.epoch);
    }
    if (!skip_stencil && head) atomicAdd(&P.st->rhs_evals, 1);
    if (P.evals && head) *P.evals = skip_stencil ? 0.0 : 1.0;
  }
}

template <int MODE, bool AUG, int FXY>
static cudaError_t launch_tile(const StencilParams& P, cudaStream_t s) {
  auto k = tile_stencil_kernel<MODE, AUG, FXY>;
  const size_t sm = tile_stencil_smem();
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  const int rows = P.rows_mode == 2 ? 0 : P.row_hi - P.row_lo;
  dim3 grid((P.ny + TT_C - 1) / TT_C, P.rows_mode == 2 ? 2 : (rows + TT_R - 1) / TT_R);
  return launch_pdl(k, grid, dim3(TT_THREADS), sm, s, P);
}

// ---- admissibility diagnostics (error path only) ---------------------------
__device__ __forceinline__ unsigned long long ord_key(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_val(unsigned long long k) {
  unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// pass 0: keys[0] = min rho, keys[1] = min p over the padded field;
// pass 1: keys[2] / keys[3] = first padded flat index attaining them
template <int MODE>
__global__ void admissibility_kernel(const StencilParams P, int pass, unsigned long long* keys) {
  const int W = P.ny + 4;
  const long long total = (long long)(P.nx + 4) * W;
  double sigma = 1.0, hnext = 1.0, rh = 1.0;
  if (MODE == MODE_JV) sigma = fd_sigma(P.scal[0]);
  if (MODE == MODE_JVN) {
    hnext = P.scal[0];
    rh = 1.0 / hnext;
    sigma = fd_sigma(P.scal[1] / hnext);
  }
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / W) - 2, c = (int)(e % W) - 2;
    const RowRef R = row_ref(P, r);
    bool yf;
    const int js = map_ghost(c, P.ny, P.bcy, yf);
    double u[NF];
    load_cell<MODE>(P, R, js, yf, sigma, hnext, rh, u);
    const double rho = u[0];
    const double m2 = __dadd_rn(__dadd_rn(__dmul_rn(u[1], u[1]), __dmul_rn(u[2], u[2])), __dmul_rn(u[3], u[3]));
    const double bb = __dadd_rn(__dadd_rn(__dmul_rn(u[4], u[4]), __dmul_rn(u[5], u[5])), __dmul_rn(u[6], u[6]));
    const double rr = 1.0 / rho;                 // RN(1/rho): one IEEE division per cell
  const double kin = div_const(__dmul_rn(0.5, m2), rho, rr);
    const double p = __dmul_rn(P.gm1, __dsub_rn(__dsub_rn(u[7], kin), __dmul_rn(P.bfac, bb)));
    if (pass == 0) {
      if (!isnan(rho)) atomicMin(&keys[0], ord_key(rho));
      if (!isnan(p)) atomicMin(&keys[1], ord_key(p));
    } else {
      if (rho == key_val(keys[0])) atomicMin(&keys[2], (unsigned long long)e);
      if (p == key_val(keys[1])) atomicMin(&keys[3], (unsigned long long)e);
    }
  }
}

// ---- diagnostics: div B and J = curl B with one ghost layer (mhd.py:288-309) -------------
// which = 0: out[nx*ny] = div B, *dmax = max |div B| (bit pattern max of non-negative doubles);
// which = 1: out[3][nx][ny] = (d_y Bz, -d_x Bz, d_x By - d_y Bx).
__global__ void __launch_bounds__(256) diag_kernel(const StencilParams P, int which, double* out,
                                                  unsigned long long* dmax) {
  // rows over blockIdx.y, columns over threads (coalesced); ghosts mapped as
  // apply_ghosts(width=1): x-neighbours (i +- 1, j) per row, y-neighbours (i, j +- 1) per column
  const unsigned total = (unsigned)P.nx * (unsigned)P.ny;
  unsigned long long best = 0ull;
  for (int i = blockIdx.y; i < P.nx; i += gridDim.y) {
    const RowRef Rm = row_ref(P, i - 1), Rp = row_ref(P, i + 1), R0 = row_ref(P, i);
    const unsigned sm = Rm.flip ? 0x80000000u : 0u, sp = Rp.flip ? 0x80000000u : 0u;
    const double* Am = Rm.halo ? P.a_halo : P.a;
    const double* Ap = Rp.halo ? P.a_halo : P.a;
    const double* A0 = P.a;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P.ny; j += gridDim.x * blockDim.x) {
      bool fl, fr;
      const int jl = map_ghost(j - 1, P.ny, P.bcy, fl), jr = map_ghost(j + 1, P.ny, P.bcy, fr);
      const unsigned sl = fl ? 0x80000000u : 0u, sr = fr ? 0x80000000u : 0u;
      const unsigned e = (unsigned)i * P.ny + j;
      const double bx_ip = flip_sign(__ldg(Ap + (Rp.off + j + 4 * Rp.fs)), sp);
      const double bx_im = flip_sign(__ldg(Am + (Rm.off + j + 4 * Rm.fs)), sm);
      const double by_jp = flip_sign(__ldg(A0 + (R0.off + jr + 5 * R0.fs)), sr);
      const double by_jm = flip_sign(__ldg(A0 + (R0.off + jl + 5 * R0.fs)), sl);
      if (which == 0) {
        const double d = __dadd_rn(div_const(__dsub_rn(bx_ip, bx_im), P.two_hx, P.r_two_hx),
                                   div_const(__dsub_rn(by_jp, by_jm), P.two_hy, P.r_two_hy));
        out[e] = d;
        const unsigned long long key = (unsigned long long)__double_as_longlong(fabs(d));
        best = key > best ? key : best;
      } else {
        const double bz_jp = __ldg(A0 + (R0.off + jr + 6 * R0.fs)), bz_jm = __ldg(A0 + (R0.off + jl + 6 * R0.fs));
        const double bz_ip = __ldg(Ap + (Rp.off + j + 6 * Rp.fs)), bz_im = __ldg(Am + (Rm.off + j + 6 * Rm.fs));
        const double by_ip = __ldg(Ap + (Rp.off + j + 5 * Rp.fs)), by_im = __ldg(Am + (Rm.off + j + 5 * Rm.fs));
        const double bx_jp = __ldg(A0 + (R0.off + jr + 4 * R0.fs)), bx_jm = __ldg(A0 + (R0.off + jl + 4 * R0.fs));
        out[e] = div_const(__dsub_rn(bz_jp, bz_jm), P.two_hy, P.r_two_hy);
        out[e + total] = -div_const(__dsub_rn(bz_ip, bz_im), P.two_hx, P.r_two_hx);
        out[e + 2 * total] = __dsub_rn(div_const(__dsub_rn(by_ip, by_im), P.two_hx, P.r_two_hx),
                                       div_const(__dsub_rn(bx_jp, bx_jm), P.two_hy, P.r_two_hy));
      }
    }
  }
  if (which == 0) {
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
      best = ob > best ? ob : best;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(dmax, best);
  }
}

cudaError_t launch_diag(StencilParams P, int which, double* out, unsigned long long* dmax, cudaStream_t s) {
  if ((long long)3 * P.nx * P.ny >= (1LL << 32)) return cudaErrorInvalidValue;   // 32-bit offsets
  static int resident = 0;            // one wave: 8 CTAs of 256 threads per SM
  if (!resident) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    resident = 8 * sms;
  }
  const int gx = (P.ny + 255) / 256;
  int gy = resident / gx;
  gy = gy < 1 ? 1 : (gy > P.nx ? P.nx : gy);
  diag_kernel<<<dim3(gx, gy), 256, 0, s>>>(P, which, out, dmax);
  return cudaGetLastError();
}

cudaError_t launch_admissibility(StencilParams P, int mode, unsigned long long* keys, cudaStream_t s) {
  const long long total = (long long)(P.nx + 4) * (P.ny + 4);
  const int G = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  for (int pass = 0; pass < 2; ++pass) {
    if (mode == MODE_RHS) admissibility_kernel<MODE_RHS><<<G, 256, 0, s>>>(P, pass, keys);
    else if (mode == MODE_JV) admissibility_kernel<MODE_JV><<<G, 256, 0, s>>>(P, pass, keys);
    else admissibility_kernel<MODE_JVN><<<G, 256, 0, s>>>(P, pass, keys);
  }
  return cudaGetLastError();
}

template <int TY, int MODE, bool AUG, int FXY, int NRAW = 1>
static cudaError_t launch_t(StencilParams P, int num_sms, cudaStream_t s, const StencilPath& sel,
                            StencilPath* used) {
  constexpr int QW = TY + 4, GYW = TY + 2;
  constexpr int NARR = MODE == MODE_RHS ? 1 : 2;
  const size_t sm = sizeof(double) * (4 * 2 * NQP * QW + 2 * NF * GYW + 2 * 2 * NCP * QW + NRAW * NARR * NF * QW) +
                    NRAW * sizeof(unsigned long long);
  auto k = stencil_kernel<TY, MODE, AUG, FXY, NRAW>;
  if ((long long)NF * P.nx * P.ny >= (1LL << 32)) return cudaErrorInvalidValue;   // 32-bit offsets
  {
    // bulk copies need 16-byte aligned sources and sizes: even ny and aligned buffers
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    P.tma = sel.bulk && (P.ny % 2 == 0) && al(P.a) && al(P.a_halo) &&
            (MODE == MODE_RHS || (al(P.v) && al(P.v_halo)));
  }
  // the edge-row launch of a halo-overlapped slab stencil (4 output rows) always takes 2D tiles:
  // a marching CTA would spend 6 dependent row steps on 2 output rows
  if (sel.kernel == 2 || (P.rows_mode == 2 && sel.kernel == 0)) {
    if (used) { *used = sel; used->kernel = 2; used->rows_per_cta = P.rows_mode == 2 ? 2 : 0; used->strip = 0; used->bulk = 0; }
    return launch_tile<MODE, AUG, FXY>(P, s);
  }
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  P.rows_per_cta = P.rows_mode == 2 ? 2 : sel.rows_per_cta;
  const int nrows = P.rows_mode == 2 ? 4 : P.row_hi - P.row_lo;   // output rows of this launch
  if (P.rows_per_cta <= 0) {
    // exactly one wave of resident CTAs (all CTAs carry equal work)
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NRAW == 2 ? TY + 32 : TY, sm);
    const int strips = (P.ny + TY - 1) / TY;
    const int target = (occ < 1 ? 1 : occ) * num_sms;
    // floor: strips x chunks must not exceed one wave of resident CTAs
    const int chunks = target / strips > 0 ? target / strips : 1;
    const int rows = (nrows + chunks - 1) / chunks;
    const int min_rows = sel.min_rows < 1 ? 1 : sel.min_rows;
    P.rows_per_cta = rows < min_rows ? min_rows : rows;
    // few rows per CTA: the marching kernel's dependent row steps dominate; the 2D-tile
    // kernel (three barrier-separated phases, bit-identical outputs) is faster there
    if (sel.kernel == 0 && rows < sel.tile_rows) {
      if (used) { *used = sel; used->kernel = 2; used->rows_per_cta = 0; used->strip = 0; used->bulk = 0; }
      return launch_tile<MODE, AUG, FXY>(P, s);
    }
  }
  if (used) {
    *used = sel;
    used->kernel = 1;
    used->rows_per_cta = P.rows_per_cta;
    used->strip = TY;
    // some strip is interior (j0 >= 2 and j0 + TY + 2 <= ny) and stages rows by bulk copies
    used->bulk = P.tma && P.ny >= 2 * TY + 2;
  }
  dim3 grid((P.ny + TY - 1) / TY, P.rows_mode == 2 ? 2 : (nrows + P.rows_per_cta - 1) / P.rows_per_cta);
  return launch_pdl(k, grid, dim3(NRAW == 2 ? TY + 32 : TY), sm, s, P);
}

template <int TY, int FXY>
static cudaError_t launch_f(const StencilParams& P, int mode, bool aug, int ns, cudaStream_t s,
                            const StencilPath& sel, StencilPath* used) {
  const bool two = two_raw_rows(mode, P, sel);
  if (mode == MODE_RHS)
    return two ? launch_t<TY, MODE_RHS, false, FXY, 2>(P, ns, s, sel, used)
               : launch_t<TY, MODE_RHS, false, FXY>(P, ns, s, sel, used);
  if (mode == MODE_JV) {
    if (two)
      return aug ? launch_t<TY, MODE_JV, true, FXY, 2>(P, ns, s, sel, used)
                 : launch_t<TY, MODE_JV, false, FXY, 2>(P, ns, s, sel, used);
    return aug ? launch_t<TY, MODE_JV, true, FXY>(P, ns, s, sel, used)
               : launch_t<TY, MODE_JV, false, FXY>(P, ns, s, sel, used);
  }
  if (two)
    return aug ? launch_t<TY, MODE_JVN, true, FXY, 2>(P, ns, s, sel, used)
               : launch_t<TY, MODE_JVN, false, FXY, 2>(P, ns, s, sel, used);
  return aug ? launch_t<TY, MODE_JVN, true, FXY>(P, ns, s, sel, used)
             : launch_t<TY, MODE_JVN, false, FXY>(P, ns, s, sel, used);
}

template <int TY>
static cudaError_t launch_ty(const StencilParams& P, int mode, bool aug, int ns, cudaStream_t s,
                             const StencilPath& sel, StencilPath* used) {
  // 2h constants: powers of two (e.g. [0,1]^2 on 2^k cells) make the 28 centred-difference
  // divisions per cell single multiplications; otherwise one or two FMA corrections
  if (is_pow2(P.two_hx) && is_pow2(P.two_hy) && P.r_two_hx == 1.0 / P.two_hx &&
      P.r_two_hy == 1.0 / P.two_hy)
    return launch_f<TY, DIV_POW2>(P, mode, aug, ns, s, sel, used);
  const bool fxy = recip_tight(P.two_hx, P.r_two_hx) && recip_tight(P.two_hy, P.r_two_hy);
  return fxy ? launch_f<TY, DIV_TIGHT>(P, mode, aug, ns, s, sel, used)
             : launch_f<TY, DIV_GENERAL>(P, mode, aug, ns, s, sel, used);
}

int stencil_tile_width(int ny, int forced, bool two_rows) {
  if (forced == 32 || forced == 64 || forced == 128) return forced;
  return ny <= 32 ? 32 : ((ny <= 64 || two_rows) ? 64 : 128);
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

StencilPath stencil_path_defaults() {
  StencilPath p;
  p.kernel = 0;
  p.rows_per_cta = 0;
  p.strip = env_int("EMHD_STENCIL_TY", 0);
  p.bulk = env_int("EMHD_STENCIL_TMA", 1) != 0;
  p.min_rows = env_int("EMHD_MIN_ROWS", 2);
  p.tile_rows = env_int("EMHD_STENCIL_TILE_ROWS", 6);
  p.raw_rows = env_int("EMHD_STENCIL_RAW_ROWS", 0);
  return p;
}

cudaError_t launch_stencil(StencilParams P, int mode, bool aug, int num_sms, cudaStream_t s,
                           const StencilPath& sel, StencilPath* used) {
  const int ty = stencil_tile_width(P.ny, sel.strip, two_raw_rows(mode, P, sel));
  if (ty == 32) return launch_ty<32>(P, mode, aug, num_sms, s, sel, used);
  if (ty == 64) return launch_ty<64>(P, mode, aug, num_sms, s, sel, used);
  return launch_ty<128>(P, mode, aug, num_sms, s, sel, used);
}

}  // namespace emhd
