// fvsrn_kernels.cuh -- shared host/device declarations for the fV-SRN kernels.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>

#include "fvsrn_device.cuh"

namespace fvsrn {

#ifndef FVSRN_THREADS
#define FVSRN_THREADS 128
#endif
constexpr int kThreads = FVSRN_THREADS;  // 4 independent warps per CTA; weights shared in smem
// CTAs per SM the register budget is sized for (A/B-measured on B200):
// DVR 5 (<= 102 regs, 20 warps/SM), decode/eval 4 (<= 128 regs).
// measured-slower DVR variants (warp-specialised, software-pipelined, two rays per lane,
// two-tile tcgen05): compiled only for A/B builds (make variant VDEFS=-DFVSRN_AB_VARIANTS=1)
#ifndef FVSRN_TEX_SPECIAL
#define FVSRN_TEX_SPECIAL 1
#endif
#ifndef FVSRN_AB_VARIANTS
#define FVSRN_AB_VARIANTS 0
#endif
#ifndef FVSRN_MIN_BLOCKS
#define FVSRN_MIN_BLOCKS 5
#endif
#ifndef FVSRN_MIN_BLOCKS_SAMPLE
#define FVSRN_MIN_BLOCKS_SAMPLE 4
#endif
constexpr int kMinBlocks = FVSRN_MIN_BLOCKS;
#ifndef FVSRN_MIN_BLOCKS_WIDE
#define FVSRN_MIN_BLOCKS_WIDE 3
#endif
// 48/64-wide networks need more accumulator registers: fewer CTAs per SM
template <int HID, bool DVR = true>
constexpr int min_blocks() {
  return HID <= 32 ? (DVR ? kMinBlocks : FVSRN_MIN_BLOCKS_SAMPLE) : (HID <= 64 ? FVSRN_MIN_BLOCKS_WIDE : 1);
}

// software-pipelined DVR (dvr_pipe_kernel): CTAs per SM the registers are sized for
#ifndef FVSRN_PIPE_MIN_BLOCKS
#define FVSRN_PIPE_MIN_BLOCKS 4
#endif
inline size_t pipe_smem_bytes(const NetDev& net, int k0) {
  size_t b = ((size_t)net.w_total * 8 + 15) / 16 * 16 + ((size_t)net.b_total * 4 + 15) / 16 * 16;
  b += (sizeof(TFDev) + 15) / 16 * 16;
  const int rs = k0 + 8;
  b += (size_t)(kThreads / kWarp) * (2 * (size_t)kWarp * rs * 2 + kWarp * 4 * 4);
  return b;
}

// two-rays-per-lane DVR (dvr_dual_kernel)
#ifndef FVSRN_DUAL_MIN_BLOCKS
#define FVSRN_DUAL_MIN_BLOCKS 3
#endif
inline size_t dual_smem_bytes(const NetDev& net, int k0) {
  size_t b = ((size_t)net.w_total * 8 + 15) / 16 * 16 + ((size_t)net.b_total * 4 + 15) / 16 * 16;
  b += (sizeof(TFDev) + 15) / 16 * 16;
  const int rs = k0 + 8;
  b += (size_t)(kThreads / kWarp) * (2 * (size_t)kWarp * rs * 2 + 2 * kWarp * 4 * 4);
  return b;
}

// warp-specialised DVR: 4 producer + 4 consumer warps per CTA
constexpr int kWsThreads = 256;
constexpr int kWsPairs = 4;
#ifndef FVSRN_WS_MIN_BLOCKS
#define FVSRN_WS_MIN_BLOCKS 2
#endif
template <int HID>
constexpr int ws_min_blocks() {
  return HID <= 32 ? FVSRN_WS_MIN_BLOCKS : 1;
}

struct CamDev {
  double eye[3], fwd[3], right[3], up[3];
  double half_w, half_h;
  int W, H;
};

struct ShardDev {
  int rank, world, compact;
  int tiles_x, n_tiles;
  const unsigned* order;   // work-queue order of local tiles (longest first), or nullptr
};

// Per-slot ray records written once per frame by ray_setup_kernel (the f64 ray setup of
// render.py:72-106, 189-200 and the first-sample position / step vector of :224-225,
// rounded to f32), so the march loops never run f64 code:
//   a[s] = (pe.x, pe.y, pe.z, n as int bits)   n = 0: no march (pixel already written)
//   b[s] = (dd.x, dd.y, dd.z, ds)              d[s] = (dir.x, dir.y, dir.z, 0), dir modes only
struct RayRecs {
  float4* a;
  float4* b;
  float4* d;
};

// kDVRTex: dvr_kernel specialised for the default fast path with a static fp16 texture grid
// (no u8 codes, no per-sample keyframe blend): the feature code has no runtime branches
// (kDVRTCTex, kSampleTex: the same for the tcgen05 march and the lattice decode)
// (kDVRPair / kDVRQuad: the frame specialisation with two / four lanes per ray, for small
// frames; kSampleTC: the tcgen05 lattice decode, fvsrn_tc.cu)
enum class KernelKind { kDVR, kDVRWS, kDVRTC, kDVRPipe, kDVRDual, kSample, kFused, kDVRTex, kDVRTCTex,
                        kSampleTex, kDVRPair, kDVRQuad, kSampleTC, kDVROcto };

// Returns the kernel instantiation for a padded hidden width (16..128), or nullptr.
// fast: specialised default-input / snake_alt variant (see FastRow).
// fmode (frame kinds kDVRTex / kDVRPair / kSampleTex): 1 static texture grid, 2 static LDG grid
const void* kernel_for(KernelKind kind, int hid_pad, bool fast, int fmode = 1);
int fast_layer_count(int hid_pad);
// LPT schedule: exact per-tile step counts (same f64 geometry as the renderer), then
// local tiles sorted by descending cost.  `order` receives n_local tile indices.
cudaError_t launch_tile_order(const CamDev& cam, const MarchDev& md, const ShardDev& sh,
                              int n_local, unsigned* cost, unsigned* order, cudaStream_t s);
// Ray records for n_slots slots (camera rays of this shard, or explicit rays when
// rays_o != nullptr); tile_cost/iota (may be null) receive the LPT keys / values.
cudaError_t launch_ray_setup(const CamDev& cam, const MarchDev& md, const ShardDev& sh,
                             const double* rays_o, const double* rays_d, long long n_slots,
                             const RayRecs& rr, float* out, unsigned* tile_cost, unsigned* iota,
                             int defer_miss, cudaStream_t s);
// order[0:n] <- local tiles by (bucketed) descending cost[0:n]; one launch
cudaError_t launch_tile_sort(int n_local, unsigned* cost, unsigned* order, int fillers, cudaStream_t s);
cudaError_t launch_blend(const __half* lo, const __half* hi, float w, long long n, __half* dst,
                         cudaStream_t s);
struct TexBlendArgs {
  unsigned long long lo[4], hi[4], out[4];   // texture objects in, surface objects out
  int R, u8;
  float w;
  float qmin_lo[16], qspan_lo[16], qmin_hi[16], qspan_hi[16];
};
cudaError_t launch_tex_blend(const TexBlendArgs& a, cudaStream_t s);
cudaError_t launch_rgba8(const float* fb, long long n_px, unsigned char* out, cudaStream_t s);
cudaError_t launch_tiles_to_frame(const float* gathered, int W, int H, int world, float* frame,
                                  cudaStream_t s);

inline size_t stage_smem_bytes(const NetDev& net, bool with_tf, int k0) {
  size_t b = ((size_t)net.w_total * 8 + 15) / 16 * 16 + ((size_t)net.b_total * 4 + 15) / 16 * 16;
  if (with_tf) b += (sizeof(TFDev) + 15) / 16 * 16;
  const int rs = k0 + 8;
  b += (size_t)(kThreads / kWarp) * ((size_t)kWarp * rs * 2 + kWarp * 4 * 4);
  return b;
}

inline size_t ws_smem_bytes(const NetDev& net, int k0) {
  size_t b = ((size_t)net.w_total * 8 + 15) / 16 * 16 + ((size_t)net.b_total * 4 + 15) / 16 * 16;
  b += (sizeof(TFDev) + 15) / 16 * 16 + 16 * sizeof(int);
  const int rs = k0 + 8;
  b += (size_t)kWsPairs * 2 * ((size_t)kWarp * rs * 2 + kWarp * 4 * 4);
  return b;
}

}  // namespace fvsrn
