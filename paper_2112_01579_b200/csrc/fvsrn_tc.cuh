// fvsrn_tc.cuh -- shapes and shared-memory map of the tcgen05 DVR kernel (fvsrn_tc.cu).
#pragma once
#include "fvsrn_kernels.cuh"

namespace fvsrn {

constexpr int kTcThreads = 128;   // 4 warps = 128 rays = one M=128 UMMA tile

// CTAs per SM the register budget is sized for (96 regs for 32-wide, 168 for 64-wide)
#ifndef FVSRN_TC_MIN_BLOCKS
#define FVSRN_TC_MIN_BLOCKS 8   // 4x32, 16-column split epilogue (64 registers): 6 2.744, 7 2.783, 8 2.729 ms at cfg 2 (full-row epilogue at 80 registers: 5 3.01, 6 2.88, 7 2.89, 8 3.00)
#endif
#ifndef FVSRN_TC_MIN_BLOCKS_WIDE
#define FVSRN_TC_MIN_BLOCKS_WIDE 4
#endif
template <int HID>
constexpr int tc_min_blocks() {
  return HID <= 32 ? FVSRN_TC_MIN_BLOCKS : FVSRN_TC_MIN_BLOCKS_WIDE;
}

// Weights of all layers, fp16, each layer an (N x K) K-major tile in the UMMA canonical
// no-swizzle layout: element (n, k) at half index
//   (n/8)*(K/8)*64 + (k/8)*64 + (n%8)*8 + (k%8)
// with N = HID (hidden layers) or 16 (output layer, rows >= d_out zero) and K = K0
// (layer 0) or HID.  Biases: f32, HID per layer, 16 for the output layer.
struct TcNetDev {
  const uint4* w;
  const float* b;
  int head;
};

__host__ __device__ constexpr int tc_round(int x, int m) { return (x + m - 1) / m * m; }

// layer-0 input rows in TMEM (no shared-memory A tile at all): 1 on, 0 off,
// 2 = 32-wide only.  On: at 64-wide it frees the 20 KB A tile, which with the split
// epilogue (128 registers) lets 4 CTAs share an SM (cfg 3: 30.0 -> 28.2 ms)
#ifndef FVSRN_TC_TMEM_A0
#define FVSRN_TC_TMEM_A0 1
#endif
// FVSRN_TC_BIAS_MMA: the biases ride in the MMA instead of a per-layer tcgen05.st of the
// bias row into the accumulators: layer 0 through the input row's pad column (1.0) and a
// bias column of W0 patched in per frame; hidden / last layers through one extra k16 tile
// (A: constant [1, 1, 0...], B: the bias split into fp16 hi + lo columns)
// (measured: 4x32 cfg 2 3.22 -> 3.02 ms, 86 instead of 96 registers; 6x64 cfg 3 25.4 -> 26.2
// ms, the k16 bias tile lengthens the per-layer MMA the CTA waits on)
#ifndef FVSRN_TC_BIAS_MMA32
#define FVSRN_TC_BIAS_MMA32 1
#endif
#ifndef FVSRN_TC_BIAS_MMA64
#define FVSRN_TC_BIAS_MMA64 0
#endif
#ifndef FVSRN_TC_BIAS0_PAD
#define FVSRN_TC_BIAS0_PAD 1
#endif
constexpr bool tc_bias_mma(int hid) { return hid <= 32 ? FVSRN_TC_BIAS_MMA32 != 0 : FVSRN_TC_BIAS_MMA64 != 0; }
template <int HID, int NM, int NL>
struct TcShape {
  static constexpr int kK0 = tc_round(16 + 2 * NM + 3, 16);   // FastRow<NM>::kK0
  static constexpr bool kBiasMma = tc_bias_mma(HID);
  // layer-0 bias through the input row's pad column (1.0) and W0's pad column (this frame's
  // b0, fp16), whenever K0 has a pad column: no per-step bias store into D for layer 0
  static constexpr bool kBias0 = kBiasMma || (FVSRN_TC_BIAS0_PAD != 0 && tc_round(16 + 2 * NM + 3, 16) > 16 + 2 * NM + 3);
  static constexpr int kKh = HID + (kBiasMma ? 16 : 0);   // K of layers 1..NL-1
  static constexpr int kKA = kK0 > kKh ? kK0 : kKh;          // A tile width (halfs)
  static constexpr int kNLast = 16;
  static constexpr int kTCols = HID <= 32 ? 32 : (HID <= 64 ? 64 : 128);
  static constexpr uint32_t kSboA = (uint32_t)(kKA / 8) * 128u;
  static constexpr int w_off(int l) { return l == 0 ? 0 : HID * kK0 + (l - 1) * HID * kKh; }
  static constexpr int kWTotal = HID * kK0 + (NL - 2) * HID * kKh + kNLast * kKh;   // halfs
  static constexpr int b_off(int l) { return l * HID; }
  static constexpr int kBTotal = (NL - 1) * HID + kNLast;
  // after the biases: the density output's row of the last layer's weights, f32 (the
  // density head's last layer runs on the FMA pipe, FVSRN_TC_LAST_FMA_MINW)
  static constexpr int kWLast = kBTotal;
  static constexpr int kBAll = kBTotal + HID;
  // shared memory map (bytes)
  static constexpr int kWOff = 0;
  static constexpr int kBOff = tc_round(kWOff + kWTotal * 2, 16);
  static constexpr int kTFOff = tc_round(kBOff + kBAll * 4, 16);
  static constexpr int kAOff = tc_round(kTFOff + (int)sizeof(TFDev), 128);
  static constexpr int kATile = kTcThreads * kKA * 2;
  // with layer-0 rows in TMEM the one-tile kernel has no shared-memory A tile
  static constexpr bool kA0 = FVSRN_TC_TMEM_A0 == 1 || (FVSRN_TC_TMEM_A0 == 2 && HID <= 32);
  static constexpr int kMbarOff = kA0 ? kAOff : kAOff + kATile;
  static constexpr int kSmem = kMbarOff + 16;   // mbarrier, TMEM slot
};

// tcgen05 DVR kernel for the default fV-SRN shapes (hid 32: 4 layers, m=14; hid 64:
// 6 layers, m=30), or nullptr.  Same argument list as dvr_kernel with TcNetDev first.
const void* tc_kernel_for(int hid);
// the single-tile kernel specialised for a static fp16 texture grid (branch-free features)
const void* tc_tex_kernel_for(int hid, int fmode = 1);   // fmode 1 texture, 2 LDG grid
// the lattice decode (decode_tc_kernel) for a static fp16 grid: fmode 1 texture, 2 LDG
const void* tc_decode_kernel_for(int hid, int fmode);
size_t tc_smem_bytes(int hid);
inline int tc_layers(int hid) { return hid == 64 ? 6 : 4; }

}  // namespace fvsrn
