// fvsrn_kernels.cuh -- shared host/device declarations for the fV-SRN kernels.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>

#include "fvsrn_device.cuh"

namespace fvsrn {

constexpr int kThreads = 128;  // 4 independent warps per CTA; weights shared in smem
constexpr int kMinBlocks = 4;  // -> <= 128 registers/thread, 16 warps/SM

struct CamDev {
  double eye[3], fwd[3], right[3], up[3];
  double half_w, half_h;
  int W, H;
};

struct ShardDev {
  int rank, world, compact;
  int tiles_x, n_tiles;
};

enum class KernelKind { kDVR, kSample, kFused };

// Returns the kernel instantiation for a padded hidden width (16..128), or nullptr.
// fast: specialised default-input / snake_alt variant (see FastRow).
const void* kernel_for(KernelKind kind, int hid_pad, bool fast);
cudaError_t launch_blend(const __half* lo, const __half* hi, float w, long long n, __half* dst,
                         cudaStream_t s);
cudaError_t launch_tiles_to_frame(const float* gathered, int W, int H, int world, float* frame,
                                  cudaStream_t s);

inline size_t stage_smem_bytes(const NetDev& net, bool with_tf, int k0) {
  size_t b = ((size_t)net.w_total * 8 + 15) / 16 * 16 + ((size_t)net.b_total * 4 + 15) / 16 * 16;
  if (with_tf) b += (sizeof(TFDev) + 15) / 16 * 16;
  const int rs = k0 + 8;
  b += (size_t)(kThreads / kWarp) * ((size_t)kWarp * rs * 2 + kWarp * 4 * 4);
  return b;
}

}  // namespace fvsrn
