// Shared device helpers for the expmhd B200 hot path.
#pragma once
#include <cmath>
#include <cuda_runtime.h>
#include <stdint.h>
#include <utility>

namespace emhd {

constexpr int NF = 8;                // conserved fields (rho, mx, my, mz, Bx, By, Bz, E)
constexpr double SQRT_EPS = 1.4901161193847656e-08;   // 2^-26 == sqrt(DBL_EPSILON)

enum Bc : int { BC_PERIODIC = 0, BC_REFLECT = 1, BC_ZEROGRAD = 2, BC_EXTERNAL = 3 };

// status word bits (device-resident, read at host sync points)
enum : int { ST_RHO = 1, ST_PRESSURE = 2, ST_NONFINITE = 4, ST_BREAKDOWN = 8, ST_DENSE = 16 };

struct DevStatus {
  int flags;
  int rhs_evals;
  unsigned long long first_nonfinite;   // flat index of first non-finite Jv entry
  int breakdown;
  int fail_iter;                        // epoch of the first stencil launch that flagged
  int rhs_evals_mark;                   // rhs_evals when emhd_evals_mark last ran (stream order)
};

// Correctly rounded x / d for a constant divisor d with r = RN(1/d), using
// FMA residual corrections (no MUFU, no slow path).  q0 = RN(x r) is within
// 1.5 ulp of x/d; the first correction makes it faithful, the second is
// Markstein's theorem (faithful q, r within half an ulp of 1/d  =>
// RN(q + RN(x - q d) r) = RN(x/d)).  Bit-identical to IEEE x / d for all
// finite x whose quotient neither overflows nor underflows.
__device__ __forceinline__ double div_const(double x, double d, double r) {
  double q = __dmul_rn(x, r);
  double e = __fma_rn(-q, d, x);
  q = __fma_rn(e, r, q);
  e = __fma_rn(-q, d, x);
  return __fma_rn(e, r, q);
}

// One-correction variant: valid (== RN(x/d)) when |1 - r d| <= 2^-54, because then
// RN(x r) is already faithful and Markstein's correction rounds it correctly.
__device__ __forceinline__ double div_const1(double x, double d, double r) {
  const double q = __dmul_rn(x, r);
  const double e = __fma_rn(-q, d, x);
  return __fma_rn(e, r, q);
}

// division by a grid constant: DV 2 = d is a power of two (1/d exact, so x / d == RN(x r)
// for every x, overflow and underflow included), 1 = one correction suffices, 0 = general
enum : int { DIV_GENERAL = 0, DIV_TIGHT = 1, DIV_POW2 = 2 };
template <int DV>
__device__ __forceinline__ double div_c(double x, double d, double r) {
  if (DV == DIV_POW2) return __dmul_rn(x, r);
  return DV == DIV_TIGHT ? div_const1(x, d, r) : div_const(x, d, r);
}

__host__ __forceinline__ bool is_pow2(double d) {
  int e;
  return d > 0.0 && std::frexp(d, &e) == 0.5;
}

// exact test of the one-correction condition (1 - r d is exactly representable)
__device__ __host__ __forceinline__ bool recip_tight(double d, double r) {
#ifdef __CUDA_ARCH__
  return fabs(__fma_rn(-r, d, 1.0)) <= 0x1p-54;
#else
  return __builtin_fabs(__builtin_fma(-r, d, 1.0)) <= 0x1p-54;
#endif
}

// sigma rule of the forward-difference Jacobian (reference fdjac.py:43)
__device__ __forceinline__ double fd_sigma(double vnorm) {
  return vnorm > SQRT_EPS ? SQRT_EPS / vnorm : 1.0;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Reduce K per-lane values across a warp with K-1 + (5 - log2 K) double shuffles
// (halving exchange, then a butterfly).  Afterwards lanes with (lane & (32/K - 1)) == 0
// hold the warp total of value index multi_index<K>(lane) in v[0].
template <int K>
__device__ __forceinline__ void warp_reduce_multi(double (&v)[K], int lane) {
  int k = K;
  int off = 16;
#pragma unroll
  for (int st = 0; st < 5 && (K >> st) > 1; ++st, off >>= 1) {
    k = K >> st;
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < (K >> (st + 1)); ++i) {
      const double send = upper ? v[i] : v[i + (K >> (st + 1))];
      const double keep = upper ? v[i + (K >> (st + 1))] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  (void)k;
  for (; off > 0; off >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
}

template <int K>
__device__ __forceinline__ int multi_index(int lane) {
  int idx = 0, off = 16;
#pragma unroll
  for (int b = K; b > 1; b >>= 1, off >>= 1) idx = idx * 2 + ((lane & off) ? 1 : 0);
  return idx;
}

// Programmatic dependent launch (Hopper+): a kernel launched with the PDL attribute is set up
// while its predecessor in the stream is still running.  Every kernel of the Arnoldi fast path
// starts with pdl_sync(), which waits until the predecessor grid has completed and its memory
// is visible — the usual stream order, minus the launch gap.  No kernel triggers its dependents
// early (griddepcontrol.launch_dependents): measured, early-resident dependent CTAs skew the
// one-wave grids (1024^2: -11 %), while the implicit trigger at completion gains at every size
// (256^2 +22 %, 1024^2 +2 %).  Without the attribute the instruction is a no-op.
__device__ __forceinline__ void pdl_sync() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

// host side: kernels that begin with pdl_sync() are launched with the PDL attribute (always
// safe: they wait for their predecessor whatever it is); EMHD_PDL=0 turns it off
bool pdl_on();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  if (!pdl_on()) {
    k<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

}  // namespace emhd
