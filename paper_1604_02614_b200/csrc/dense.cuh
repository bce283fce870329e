// Small dense phi / exponential of the Krylov Hessenberg matrix (dense.cu).
#pragma once
#include "emhd_common.cuh"

namespace emhd {

constexpr int DENSE_MAX_SCALES = 8;

struct DenseWork {
  double* a;        // n x n input (scaled in place)
  double* e;        // n x n exponential
  double* m[8];     // 7 n x n work matrices + one n x 2n
  double* vec;      // 5 n + 64
  double* part;     // [2][CLUSTER][n] column-sum partials of the cluster kernel
  int gj_blocked;   // set by the kernels from PhiSmallArgs: blocked Gauss-Jordan solve
};

constexpr int DENSE_CLUSTER = 8;     // CTAs (SMs) per exponential in the cluster kernel

// doubles of dense workspace per problem of dimension n (see carve in capi.cu)
inline size_t dense_per(size_t n) { return 11 * n * n + 5 * n + 64 + 2 * DENSE_CLUSTER * n; }

struct PhiSmallArgs {
  const double* H;          // Hessenberg (device), leading m x m block used
  long long ldh;
  int m, order;             // phi_order of the ((order+1) m)^2 block matrix
  const double* scales;     // device [S]: scale applied to H (c*h or delta)
  const double* res_scale;  // device [S]: factor applied to the residual
  const double* scal;       // device {h_next, max|w|, breakdown} of the basis (null: breakdown)
  const double* beta;       // device scalar: ||seed||
  double* Y;                // [S][m] coefficient vectors y_s
  double* res;              // [S] residual estimates
  DenseWork work[DENSE_MAX_SCALES];
  DevStatus* st;
  double* E_out;
  int scales_by_value;       // 1: use sv / rv instead of the device arrays
  int batch;                // 1: CTA s evaluates basis size mb[s], h_next from H / brk_hist
  int mb[DENSE_MAX_SCALES];
  const double* brk_hist;
  long long ldy;            // row stride of Y in batch mode
  double sv[DENSE_MAX_SCALES];
  double rv[DENSE_MAX_SCALES];
  int smem_n;               // set by the launcher: largest n whose [n][2n] system is on chip
  int smem_work;            // set by the launcher: the whole workspace (11 n^2 + 5 n doubles) is
                            // carved from dynamic shared memory instead of the global work[]
  int cluster;              // set by the launcher: DENSE_CLUSTER CTAs per problem (large n)
  int gj_blocked;           // set by the launcher: blocked Gauss-Jordan solve (EMHD_DENSE_GJ_BLOCKED, 1)
};

cudaError_t launch_phi_small(const PhiSmallArgs& P, int nscales, cudaStream_t s);
int dense_cluster_min_n();
void set_dense_cluster_min_n(int n);
int dense_gj_blocked();
void set_dense_gj_blocked(int on);

}  // namespace emhd
