// Launchers of the Arnoldi / combination kernels (krylov.cu).
#pragma once
#include "emhd_common.cuh"

namespace emhd {

struct KWork {
  double* partials;          // >= (m_cap + 3) * 2 * num_sms doubles
  unsigned int* ticket;      // zero-initialised, re-armed by each reduction
  int num_sms;
  bool stream_basis = false; // update passes read V evict-first (a persisting L2 window holds its head)
};

struct FinishArgs {         // optional Arnoldi column bookkeeping fused into update mode 1
  const double* h1;
  const double* h2;
  const double* selfdot;
  int j;
  double* H;                 // null: not fused
  long long ldh;
  double* scal;
  double* brk_hist;
  DevStatus* st;
  double rtol;
};

struct Reorth {               // selective (DGKS) re-orthogonalisation of one Arnoldi iteration
  double eta2;               // pass 2 is skipped when ||w1||^2 >= eta2 ||w||^2 (0: never decide)
  double* gate_out;          // update mode 0: decision written here (1 = pass 2 skipped)
  const double* skip2;       // pass-2 launches: no work when *skip2 != 0
  const double* predict;     // update mode 0: predict[0] and predict[1] != 0 (the two previous
                             // iterations skipped pass 2) -> predicted unnecessary again, so the
                             // re-projection dots are not computed (null: always computed)
  double* gate_md2;          // update mode 0: 0 when pass 2 must run but its dots are missing
                             // (a separate multi-dot then computes them), else 1
};

struct HaloPush {            // peer halo destinations of a slab's edge rows (null: none)
  double* lo;                // lo neighbour's halo buffer [2][8][2][ny]
  double* hi;                // hi neighbour's halo buffer
  long long n_top;           // 8 * nx * ny
  unsigned plane, nx, ny;    // nx * ny, local rows, columns
};

struct CombineOut {
  const double* base[4];     // optional base vector per output (null: plain V y)
  double coef[4];            // out = base + coef * (V y)
  double* out[4];
};

cudaError_t launch_multidot(const double* w, const double* V, long long ldv, int nvec, long long len_dot,
                            int self, KWork& wk, double* out, cudaStream_t s, const double* skip = nullptr,
                            const double* skip2 = nullptr);
cudaError_t launch_update(double* w, const double* V, long long ldv, int nvec, const double* h,
                          long long len_upd, long long len_dot, long long len_max, int mode,
                          KWork& wk, double* out, cudaStream_t s, FinishArgs fin = FinishArgs{},
                          const double* skip = nullptr, Reorth ro = Reorth{});
// one-launch orthogonalisation of an Arnoldi iteration on small grids (bit-identical to
// launch_multidot + launch_update (+ gated second pass)); partials_b: a second partials buffer
// ((nvec + 2) * 2 * num_sms doubles); bar: {arrivals, generation}, zeroed once
bool orth_small_fits(long long len_upd, int num_sms);
cudaError_t launch_orth_small(double* w, const double* V, long long ldv, int nvec, long long len_upd,
                              long long len_dot, long long len_max, KWork& wk, double* partials_b,
                              unsigned int* bar, double* d1, double* d2, double* nrm, cudaStream_t s,
                              FinishArgs fin, const double* skip, Reorth ro);
cudaError_t launch_push_edges(const double* w, const HaloPush& H, const double* gate, cudaStream_t s);
cudaError_t launch_reorth_decide(FinishArgs fin, const double* r, int nvec, double eta2, double* gate,
                                 cudaStream_t s, double* gate_md2 = nullptr, const double* predict = nullptr);
cudaError_t launch_gate(const unsigned long long* cancel, unsigned gen, int j, double* gate, cudaStream_t s);
cudaError_t launch_evals_discount(const double* evals, int count, DevStatus* st, cudaStream_t s);
cudaError_t launch_update_push(double* w, const double* V, long long ldv, int nvec, const double* h,
                               long long len_upd, long long len_dot, long long len_max, KWork& wk,
                               double* out, const HaloPush& push, cudaStream_t s,
                               const double* skip2 = nullptr);
cudaError_t launch_norms(const double* x, long long len_sum, long long len_max, KWork& wk, double* out,
                         cudaStream_t s);
cudaError_t launch_arnoldi_finish(const double* h1, const double* h2, const double* nrm,
                                  const double* selfdot, int j, double* H, long long ldh, double* scal,
                                  double* brk_hist, DevStatus* st, double rtol, cudaStream_t s,
                                  const double* skip2 = nullptr);
cudaError_t launch_combine(const double* V, long long ldv, int m, const double* Y, int S,
                           const CombineOut& co, long long len, int num_sms, cudaStream_t s);

}  // namespace emhd
