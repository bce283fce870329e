// Output-side kernels of the path: the .mhd25 cell-major layout of a
// device slab, the explicit-RK4 stable step's signal speed, and the harness error norm.
//
// Bit-exact arithmetic (compiled with -fmad=false): the signal speed reproduces the NumPy
// expression order of harness.py:166-179 (_rk4_stable_dt) and pressure (mhd.py:116-131);
// the maximum over cells is order-independent, so the step size is bitwise the reference's.
#include "emhd_common.cuh"
#include "harness.cuh"

namespace emhd {

constexpr int HT = 256;

// (8, ncell) field-major -> (ncell, 8) cell-major (snapshot.py:53-57).  Consecutive threads
// write consecutive doubles; each warp reads 8 fields x 4 consecutive cells (full sectors).
// (Measured: faster than one thread per cell with 16-byte stores, 82 % vs 60 % of HBM.)
__global__ void __launch_bounds__(HT) cells_pack_kernel(const double* __restrict__ U, long long ncell,
                                                        double* __restrict__ out) {
  const long long total = ncell * NF;
  for (long long o = (long long)blockIdx.x * HT + threadIdx.x; o < total; o += (long long)gridDim.x * HT) {
    const long long cell = o >> 3;
    const int f = (int)(o & 7);
    out[o] = __ldg(U + (long long)f * ncell + cell);
  }
}

// inverse: (ncell, 8) -> (8, ncell) (snapshot.py:77): one thread per cell, four 16-byte
// loads, eight coalesced plane stores (89 % of HBM at 4096^2; element-wise: 24 %)
template <bool VEC>
__global__ void __launch_bounds__(HT) cells_unpack_kernel(const double* __restrict__ cells, long long ncell,
                                                          double* __restrict__ U) {
  for (long long c = (long long)blockIdx.x * HT + threadIdx.x; c < ncell; c += (long long)gridDim.x * HT) {
    double v[NF];
    if (VEC) {
      const double2* in = reinterpret_cast<const double2*>(cells + c * NF);
#pragma unroll
      for (int k = 0; k < NF / 2; ++k) {
        const double2 x = __ldg(in + k);
        v[2 * k] = x.x;
        v[2 * k + 1] = x.y;
      }
    } else {
#pragma unroll
      for (int f = 0; f < NF; ++f) v[f] = __ldg(cells + c * NF + f);
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) U[(long long)f * ncell + c] = v[f];
  }
}

// max over cells of c_fast = sqrt((gamma p + |B|^2) / rho) + sqrt(|m|^2 / rho^2)
// (harness.py:168-172, pressure as mhd.py:126-127); positive doubles order like their bits,
// so the maximum is an atomicMax on the bit pattern.  Inadmissible cells raise the flags.
__global__ void __launch_bounds__(HT) signal_speed_kernel(const double* __restrict__ U, long long ncell,
                                                          double gamma, double gm1, double bfac,
                                                          unsigned long long* cmax_bits, DevStatus* st) {
  double best = 0.0;
  int flag = 0;
  for (long long c = (long long)blockIdx.x * HT + threadIdx.x; c < ncell; c += (long long)gridDim.x * HT) {
    const double rho = U[c], mx = U[ncell + c], my = U[2 * ncell + c], mz = U[3 * ncell + c];
    const double bx = U[4 * ncell + c], by = U[5 * ncell + c], bz = U[6 * ncell + c], en = U[7 * ncell + c];
    if (!(rho > 0.0)) flag |= ST_RHO;
    const double m2 = __dadd_rn(__dadd_rn(__dmul_rn(mx, mx), __dmul_rn(my, my)), __dmul_rn(mz, mz));
    const double b2 = __dadd_rn(__dadd_rn(__dmul_rn(bx, bx), __dmul_rn(by, by)), __dmul_rn(bz, bz));
    const double kin = __ddiv_rn(__dmul_rn(0.5, m2), rho);
    const double p = __dmul_rn(gm1, __dsub_rn(__dsub_rn(en, kin), __dmul_rn(bfac, b2)));
    if (!(p > 0.0)) flag |= ST_PRESSURE;
    const double v2 = __ddiv_rn(m2, __dmul_rn(rho, rho));
    const double cf = __dadd_rn(__dsqrt_rn(__ddiv_rn(__dadd_rn(__dmul_rn(gamma, p), b2), rho)), __dsqrt_rn(v2));
    best = fmax(best, cf);
  }
  for (int o = 16; o > 0; o >>= 1) {
    best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    flag |= __shfl_xor_sync(0xffffffffu, flag, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (best > 0.0) atomicMax(cmax_bits, static_cast<unsigned long long>(__double_as_longlong(best)));
    if (flag) atomicOr(&st->flags, flag);
  }
}

// per-field partial sums of (U - R)^2 per CTA, then a fixed-order finish (deterministic).
// One thread per cell with all 16 loads in flight; the 8 sums leave each warp in one
// multi-value shuffle reduction.
__global__ void __launch_bounds__(HT) field_sqdiff_kernel(const double* __restrict__ U,
                                                          const double* __restrict__ R, long long ncell,
                                                          double* partials) {
  __shared__ double s[NF][HT / 32];
  double acc[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) acc[f] = 0.0;
  for (long long c = (long long)blockIdx.x * HT + threadIdx.x; c < ncell; c += (long long)gridDim.x * HT) {
    double u[NF], r[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      u[f] = __ldg(U + (long long)f * ncell + c);
      r[f] = __ldg(R + (long long)f * ncell + c);
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const double d = u[f] - r[f];
      acc[f] = fma(d, d, acc[f]);
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_reduce_multi<NF>(acc, lane);
  if ((lane & (32 / NF - 1)) == 0) s[multi_index<NF>(lane)][warp] = acc[0];
  __syncthreads();
  if (threadIdx.x < NF) {
    double t = 0.0;
    for (int w = 0; w < HT / 32; ++w) t += s[threadIdx.x][w];
    partials[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
}

__global__ void field_sqdiff_finish(const double* partials, int G, double* out) {
  const int f = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (f >= NF) return;
  double acc = 0.0;
  for (int c = lane; c < G; c += 32) acc += partials[(size_t)f * G + c];
  acc = warp_sum(acc);
  if (lane == 0) out[f] = acc;
}

static int hgrid(long long work, int num_sms) {
  long long g = (work + HT - 1) / HT;
  const long long cap = 8LL * num_sms;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

cudaError_t launch_cells_pack(const double* U, long long ncell, double* out, int num_sms, cudaStream_t s) {
  cells_pack_kernel<<<hgrid(ncell * NF, num_sms), HT, 0, s>>>(U, ncell, out);
  return cudaGetLastError();
}

cudaError_t launch_cells_unpack(const double* cells, long long ncell, double* U, int num_sms, cudaStream_t s) {
  if ((reinterpret_cast<uintptr_t>(cells) & 15) == 0)
    cells_unpack_kernel<true><<<hgrid(ncell, num_sms), HT, 0, s>>>(cells, ncell, U);
  else
    cells_unpack_kernel<false><<<hgrid(ncell, num_sms), HT, 0, s>>>(cells, ncell, U);
  return cudaGetLastError();
}

cudaError_t launch_signal_speed(const double* U, long long ncell, double gamma, double gm1, double bfac,
                                double* cmax, DevStatus* st, int num_sms, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(cmax, 0, sizeof(double), s);
  if (e != cudaSuccess) return e;
  signal_speed_kernel<<<hgrid(ncell, num_sms), HT, 0, s>>>(U, ncell, gamma, gm1, bfac,
                                                           reinterpret_cast<unsigned long long*>(cmax), st);
  return cudaGetLastError();
}

cudaError_t launch_field_sqdiff(const double* U, const double* R, long long ncell, double* partials,
                                int max_g, double* out, int num_sms, cudaStream_t s) {
  int G = hgrid(ncell, num_sms) < 4 * num_sms ? hgrid(ncell, num_sms) : 4 * num_sms;
  G = G < max_g ? G : max_g;
  if (G < 1) return cudaErrorInvalidValue;
  field_sqdiff_kernel<<<G, HT, 0, s>>>(U, R, ncell, partials);
  field_sqdiff_finish<<<1, 32 * NF, 0, s>>>(partials, G, out);
  return cudaGetLastError();
}

}  // namespace emhd
