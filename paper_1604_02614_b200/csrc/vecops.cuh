// Exact-order stage algebra kernels (vecops.cu).
#pragma once
#include "emhd_common.cuh"

namespace emhd {

struct LinComb {
  const double* x[6];
  double c[6];
  int has_c[6];
  int nterms;
  double post;
  int has_post;
  const double* base;       // optional: out = base + (post-applied sum)
  double* out;
};

cudaError_t launch_lincomb(const LinComb& L, long long n, long long len_max, double* partials,
                           double* max_out, unsigned int* ticket, int num_sms, cudaStream_t s);
cudaError_t launch_wrms(const double* err, const double* y, double tol, long long n, double* partials,
                        double* out, unsigned int* ticket, int num_sms, cudaStream_t s);
cudaError_t launch_div_scalar(const double* x, const double* d2, int take_sqrt, double* out, double* d_out,
                              long long n, int num_sms, cudaStream_t s);

}  // namespace emhd
