// Parameters of the fused MHD RHS / Jv stencil kernel (stencil.cu).
#pragma once
#include "emhd_common.cuh"

namespace emhd {

enum : int { MODE_RHS = 0, MODE_JV = 1, MODE_JVN = 2 };

struct StencilParams {
  int nx, ny;                 // local interior rows (x) and columns (y)
  int nxg;                    // global rows (for flat indices in error reports)
  int x_off;                  // global row of local row 0
  int bcx_lo, bcx_hi, bcy;    // Bc per side; BC_EXTERNAL = x-halo from neighbour rank
  int rows_per_cta;           // <= 0: chosen by the launcher
  int check;                  // admissibility checks on (mhd.py:116 check=True)
  double gm1, mu, eta, heat, bfac;
  double two_hx, r_two_hx, two_hy, r_two_hy;
  const double* a;            // state (RHS input) or Jacobian base point
  const double* a_halo;       // [2 sides][8][2 rows][ny] or null
  const double* v;            // MODE_JV: direction; MODE_JVN: unnormalised w_prev
  const double* v_halo;
  const double* fa;           // F(a)
  const double* scal;         // MODE_JV: {||v||_inf}; MODE_JVN: {h_next, max|w_top|}
  double* out;
  double* vout;               // MODE_JVN: v_j = w_prev / h_next (interior + tail)
  long long n_top;            // 8 * nx * ny
  int p;                      // augmented tail length (0: none)
  int nb;                     // number of B columns in the epilogue
  const double* bcol[5];
  int bidx[5];                // q index multiplying bcol[k]
  double ch;                  // c*h scale of the augmented operator
  const double* qsrc;         // MODE_JV + tail: q (device, length p)
  DevStatus* st;
  int epoch;                  // caller-defined launch tag recorded on failure
  int tma;                    // interior strips stage raw rows with bulk async copies (set by the launcher)
  const double* skip;         // gated launch: *skip != 0 -> no work (cancelled look-ahead iteration)
  double* evals;              // optional: 1 if this launch evaluated the RHS (counted), else 0
  // output rows: rows_mode 0/1: [row_lo, row_hi); rows_mode 2: rows {0, 1} and {nx-2, nx-1}
  // (the halo-dependent edge rows of a slab, launched after the halo exchange while the
  // interior [2, nx-2) ran without it); count: this launch does the RHS count / evals / tail
  int rows_mode, row_lo, row_hi, count;
};

// Launch selection of the stencil (per context: emhd_set_stencil_path; defaults from the
// environment at context creation).  Also the record of what a launch actually ran.
struct StencilPath {
  int kernel;        // 0 auto, 1 row-marching strips, 2 2D tiles
  int rows_per_cta;  // marching: rows per CTA (0: one wave of resident CTAs, >= min_rows)
  int strip;         // marching: strip width 32 / 64 / 128 (0: by ny)
  int bulk;          // marching: interior strips stage raw rows with bulk async copies (when aligned)
  int min_rows;      // auto: floor of rows per CTA
  int tile_rows;     // auto: 2D tiles when a marching CTA would get fewer rows than this
  int raw_rows;      // marching: raw rows staged ahead (0 auto: 2 for Jv / normalised Jv, 1 for RHS)
};

StencilPath stencil_path_defaults();   // EMHD_STENCIL_TY / _TMA / _TILE_ROWS, EMHD_MIN_ROWS
cudaError_t launch_stencil(StencilParams P, int mode, bool aug, int num_sms, cudaStream_t s,
                           const StencilPath& sel, StencilPath* used = nullptr);
int stencil_tile_width(int ny, int forced, bool two_rows);
cudaError_t launch_diag(StencilParams P, int which, double* out, unsigned long long* dmax, cudaStream_t s);
cudaError_t launch_admissibility(StencilParams P, int mode, unsigned long long* keys, cudaStream_t s);

}  // namespace emhd
