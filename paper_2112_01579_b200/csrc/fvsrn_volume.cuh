// fvsrn_volume.cuh -- ground-truth volume renderer declarations.
#pragma once
#include "fvsrn_kernels.cuh"

namespace fvsrn {

struct VolDev {
  const float* v;   // (X, Y, Z) f32, C order (z fastest): ScalarVolume.values
  int X, Y, Z;
};

cudaError_t launch_volume_dvr(const VolDev& vol, const TFDev* tf, const MarchDev& md,
                              const CamDev& cam, const ShardDev& sh, const double* ro,
                              const double* rd, long long n_slots, float* out,
                              unsigned long long* counters, int num_sms, cudaStream_t s);

}  // namespace fvsrn
