// Exact-order elementwise vector algebra of the EpiRK stages.
//
// Replaces the NumPy stage expressions of reference pkg/src/expmhd/epirk.py
// (:202, 207-208, 213-216, 224-225, 246, 251-258, 265) and remainder
// (:179-181): out = post * (t0 + t1 + ... ), t_k = c_k * x_k (or x_k),
// evaluated left to right with separate multiply and add (this TU is built
// with -fmad=false), i.e. the same bits NumPy produces for the same inputs.
// Optionally fuses max|out| (the sigma of the following Jacobian apply) and
// the weighted RMS error norm of the adaptive controller (epirk.py:156-158).
#include "emhd_common.cuh"
#include "vecops.cuh"

namespace emhd {

constexpr int VT = 256;
constexpr int VW = VT / 32;

__device__ bool finish2(const double* partials, int G, double* out, unsigned int* ticket, int kind1) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == (unsigned)G - 1);
  __syncthreads();
  if (!last) return false;
  __threadfence();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp < 2) {
    const bool mx = (warp == 1) ? (kind1 == 1) : false;
    double acc = 0.0;
    for (int c = lane; c < G; c += 32) {
      const double x = __ldcg(partials + (size_t)warp * G + c);
      acc = mx ? fmax(acc, x) : acc + x;
    }
    acc = mx ? warp_max(acc) : warp_sum(acc);
    if (lane == 0) out[warp] = acc;
  }
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

__global__ void __launch_bounds__(VT) lincomb_kernel(const LinComb L, long long n, long long len_max,
                                                     double* partials, double* red_out,
                                                     unsigned int* ticket) {
  pdl_sync();
  __shared__ double s[2 * VW];
  double mx = 0.0;
  for (long long e = (long long)blockIdx.x * VT + threadIdx.x; e < n; e += (long long)gridDim.x * VT) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      if (k < L.nterms) {
        double t = L.x[k][e];
        if (L.has_c[k]) t = __dmul_rn(L.c[k], t);
        acc = (k == 0) ? t : __dadd_rn(acc, t);
      }
    }
    if (L.has_post == 1) acc = __dmul_rn(L.post, acc);
    else if (L.has_post == 2) acc = acc / L.post;      // IEEE division (fdjac.py:49)
    if (L.base) acc = __dadd_rn(L.base[e], acc);
    L.out[e] = acc;
    if (e < len_max) mx = fmax(mx, fabs(acc));
  }
  if (red_out) {
    mx = warp_max(mx);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = 0.0;
      for (int q = 0; q < VW; ++q) b = fmax(b, s[q]);
      partials[(size_t)gridDim.x + blockIdx.x] = b;
    }
  }
  (void)ticket;
}

// out[1] = max|x| over len (separate final kernel keeps lincomb simple)
__global__ void __launch_bounds__(VT) lincomb_max_finish(const double* partials, int G, double* out) {
  pdl_sync();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    double acc = 0.0;
    for (int c = lane; c < G; c += 32) acc = fmax(acc, partials[(size_t)G + c]);
    acc = warp_max(acc);
    if (lane == 0) out[0] = acc;
  }
}

// sum over e of (err_e / (tol + tol*|y_e|))^2  (epirk.py:156-158)
__global__ void __launch_bounds__(VT) wrms_kernel(const double* err, const double* y, double tol, long long n,
                                                  double* partials, double* out, unsigned int* ticket) {
  __shared__ double s[VW];
  double ss = 0.0;
  for (long long e = (long long)blockIdx.x * VT + threadIdx.x; e < n; e += (long long)gridDim.x * VT) {
    const double w = __dadd_rn(tol, __dmul_rn(tol, fabs(y[e])));
    const double r = err[e] / w;
    ss = __dadd_rn(ss, __dmul_rn(r, r));
  }
  ss = warp_sum(ss);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) s[warp] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int q = 0; q < VW; ++q) a += s[q];
    partials[blockIdx.x] = a;
    partials[(size_t)gridDim.x + blockIdx.x] = 0.0;
  }
  finish2(partials, gridDim.x, out, ticket, 0);
}

// v / d with d a device scalar (sqrt of d2 when take_sqrt): exact IEEE division
__global__ void __launch_bounds__(VT) div_scalar_kernel(const double* x, const double* d2, int take_sqrt,
                                                        double* out, double* d_out, long long n) {
  pdl_sync();
  const double d = take_sqrt ? sqrt(d2[0]) : d2[0];
  const double r = 1.0 / d;
  for (long long e = (long long)blockIdx.x * VT + threadIdx.x; e < n; e += (long long)gridDim.x * VT)
    out[e] = div_const(x[e], d, r);
  if (d_out && blockIdx.x == 0 && threadIdx.x == 0) d_out[0] = d;
}

static int vgrid(long long n, int num_sms) {
  long long g = (n + VT - 1) / VT;
  long long cap = 4LL * num_sms;
  return (int)(g < cap ? (g < 1 ? 1 : g) : cap);
}

cudaError_t launch_lincomb(const LinComb& L, long long n, long long len_max, double* partials,
                           double* max_out, unsigned int* ticket, int num_sms, cudaStream_t s) {
  const int G = vgrid(n, num_sms);
  cudaError_t e = launch_pdl(lincomb_kernel, dim3(G), dim3(VT), 0, s, L, n, len_max, partials, max_out,
                             ticket);
  if (e != cudaSuccess || !max_out) return e;
  return launch_pdl(lincomb_max_finish, dim3(1), dim3(32), 0, s, (const double*)partials, G, max_out);
}

cudaError_t launch_wrms(const double* err, const double* y, double tol, long long n, double* partials,
                        double* out, unsigned int* ticket, int num_sms, cudaStream_t s) {
  wrms_kernel<<<vgrid(n, num_sms), VT, 0, s>>>(err, y, tol, n, partials, out, ticket);
  return cudaGetLastError();
}

cudaError_t launch_div_scalar(const double* x, const double* d2, int take_sqrt, double* out, double* d_out,
                              long long n, int num_sms, cudaStream_t s) {
  return launch_pdl(div_scalar_kernel, dim3(vgrid(n, num_sms)), dim3(VT), 0, s, x, d2, take_sqrt, out, d_out, n);
}

}  // namespace emhd
