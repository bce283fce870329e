// Launchers of the snapshot / RK4-harness kernels (harness.cu).
#pragma once
#include "emhd_common.cuh"

namespace emhd {

cudaError_t launch_cells_pack(const double* U, long long ncell, double* out, int num_sms, cudaStream_t s);
cudaError_t launch_cells_unpack(const double* cells, long long ncell, double* U, int num_sms, cudaStream_t s);
cudaError_t launch_signal_speed(const double* U, long long ncell, double gamma, double gm1, double bfac,
                                double* cmax, DevStatus* st, int num_sms, cudaStream_t s);
cudaError_t launch_field_sqdiff(const double* U, const double* R, long long ncell, double* partials,
                                int max_g, double* out, int num_sms, cudaStream_t s);

}  // namespace emhd
