// fvsrn_device.cuh -- device building blocks of the fused fV-SRN DVR path (sm_100a).
//
// One warp evaluates the network for 32 samples at a time:
//   * each lane assembles ITS OWN sample's input row (latent grid trilinear with
//     16-byte fp16 loads + f32 FHFMA accumulation, NeRF Fourier features via a
//     double-angle recurrence, raw position) into a per-warp shared-memory stage;
//   * ldmatrix turns the stage into m16n8k16 A fragments; the MLP runs on the
//     tensor cores (mma.sync f16 x f16 -> f32) with weights staged once per CTA
//     in shared memory in B-fragment order (one conflict-free LDS.64 per MMA);
//   * the f32 accumulators of two adjacent n8 tiles ARE the A fragment of the
//     next layer's k16 tile, so activations stay in registers between layers;
//   * the head output goes back to the owning lane through a 32x4 smem slot.
//
// Reference semantics followed (fvsrn 0.1.0, /root/reference/pkg/src/fvsrn):
//   input layout / encoders  model.py:248-279, nn.py:47-57
//   grid cell + weights      grid.py:47-84
//   MLP + activations        nn.py:18-29, 195-204;  heads model.py:338-357
//   transfer function        transfer.py:57-65
//   compositing + ET         render.py:109-117, 219-232
// The device feature order is a fixed permutation of the reference's
// (z | sin/cos pairs | p | d); the host packs W0's columns accordingly, and the
// per-frame time features are folded into the layer-0 bias.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace fvsrn {

constexpr int kWarp = 32;
constexpr int kMaxLayers = 24;
constexpr int kMaxTF = 64;
constexpr int kMaxHidden = 128;
constexpr int kMaxK0 = 128;        // padded input width limit (8 k16 tiles)
constexpr int kTile = 8;           // screen tile edge (pixels)

// ---------------------------------------------------------------- params
struct NetDev {
  const uint2* wfrag;     // B fragments, all layers, [l][kt][nt][lane]
  const float* bias;      // padded biases, all layers (layer 0 overridden per call)
  int layers, kt0, act, head, out_real;
  int w_off[kMaxLayers + 1];   // uint2 offsets
  int b_off[kMaxLayers + 1];   // float offsets
  int w_total, b_total;        // sizes (for smem staging)
};

struct FeatDev {              // how a lane builds its input row (device column order)
  int grid_res, f_pad;        // latent grid (R, padded channels); f_pad == 0: no grid
  const __half* grid;         // (R,R,R,f_pad) fp16, already time-blended for the frame
  int fourier_mode, m, fd_in; // 0 off, 1 nerf, 2 random; fd_in 3 or 6
  const float* bmat;          // random mode B (m, fd_in) f32 (device)
  int four_off, raw_off, raw_w, k0;  // column offsets (halfs)
  int dir_mode;               // 0 pos, 1 dirP, 2 dirF
  // texture path (FastRow, F = 16): 4 RGBA16F 3D textures per grid, trilinear filtering
  // in the texture units; temporal models blend the bracketing keyframes (weight tex_w)
  int tex_on;
  float tex_w;
  unsigned long long tex_lo[4], tex_hi[4];
  // u8-quantised grids (grid.py:157-172): RGBA8 textures read as code/255, dequantised
  // per channel in the kernel, v = min + (code/255) * (max - min)
  int tex_u8;
  float qmin_lo[16], qspan_lo[16], qmin_hi[16], qspan_hi[16];
};

struct TFDev {
  int n;
  float xs[kMaxTF];
  float val[kMaxTF][4];       // r g b sigma at control points
  float slope[kMaxTF][4];     // per segment
};

struct MarchDev {
  double stepsize, et_alpha, eps_blend;
  float bg[3];
  int max_steps;
  float eps1_f, et_f;         // f32(1 - eps_blend), f32(et_alpha): loop invariants from the host
};

// floor(c) for 0 <= c < 2^23 on the FMA/ALU pipes (no F2I/I2F on the XU pipe):
// c + 2^23 rounded toward -inf holds floor(c) in its low mantissa bits.
__device__ __forceinline__ float floor_pos(float c, int& i) {
  const float m = __fadd_rd(c, 8388608.f);
  i = __float_as_int(m) - 0x4B000000;
  return m - 8388608.f;
}
// round-to-nearest-even for |v| < 2^22 on the FMA pipe (no FRND on the XU pipe)
__device__ __forceinline__ float rint_fma(float v) {
  return __fsub_rn(__fadd_rn(v, 12582912.f), 12582912.f);
}

// ---------------------------------------------------------------- small helpers
__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ float fhfma(uint16_t a, uint16_t b, float c) {
  float r;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(r) : "h"(a), "h"(b), "f"(c));
  return r;
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint2 b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

__device__ __forceinline__ void mma16816c(float (&d)[4], const uint32_t (&a)[4], uint2 b,
                                          const float4& c) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%12,%13};\n"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y),
        "f"(c.x), "f"(c.y), "f"(c.z), "f"(c.w));
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], const void* smem_row_ptr) {
  uint32_t addr = static_cast<uint32_t>(__cvta_generic_to_shared(smem_row_ptr));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Hidden activations (nn.py:18-29).  For the snake family the host pre-scales every
// hidden layer by 2 so the accumulator holds a = 2x, and the kernel evaluates
//   snake_alt: h = a - 2 cos a   (act = h/4 + 1/2)
//   snake:     h = a -   cos a   (act = h/2 + 1/2)
// the 1/4 (1/2) and the +1/2 are folded into the NEXT layer's weights / bias on the
// host (exact in fp16).  Cost per element: FMUL.RZ + MUFU.COS + FFMA.
constexpr int kActRuntime = -1;

// B-fragment storage: 1 = pairs of n8 tiles per LDS.128, 0 = one LDS.64 per tile
#ifndef FVSRN_BPAIRS
#define FVSRN_BPAIRS 0
#endif
#ifndef FVSRN_BIAS64
#define FVSRN_BIAS64 0
#endif
// two-point TF coefficients held in registers in the DVR kernel
#ifndef FVSRN_TF_REGS
#define FVSRN_TF_REGS 0
#endif

// Every FVSRN_POLY_EVERY-th snake activation evaluates cos on the FMA pipe instead of
// MUFU (balances the XU/MIO and FMA pipes; 0 = all MUFU).  cos(a) = cos(2 pi r) with
// r = a/(2 pi) - rint(.) in [-1/2, 1/2]: degree-4 minimax in r^2, |err| < 4.3e-5.
#ifndef FVSRN_POLY_EVERY
#define FVSRN_POLY_EVERY 0
#endif
// mma.sync kernels: every FVSRN_MMA_H2-th n8 column tile of the activations evaluates its
// snake_alt cosines in HFMA2 arithmetic (snake_alt_h2_fma below); 0 = all MUFU
// (cfg 1, dvr_pair_kernel: 0.210 -> 0.198 ms with every 4th tile (2nd: 0.204); cfg 2 on
// the mma.sync kernel 3.118 -> 3.094 ms (2nd: 3.208))
#ifndef FVSRN_MMA_H2
#define FVSRN_MMA_H2 4
#endif
__device__ __forceinline__ float cos_poly(float a) {
  const float t = a * 0.15915494309189535f;
  const float k = (t + 12582912.f) - 12582912.f;     // round to nearest (|t| < 2^22)
  const float r = t - k;
  const float u = r * r;
  float p = fmaf(45.62269592285156f, u, -82.3971176147461f);
  p = fmaf(p, u, 64.67363739013672f);
  p = fmaf(p, u, -19.731164932250977f);
  return fmaf(p, u, 0.9999644756317139f);
}

// snake_alt h = x - 2 cos x entirely on the FMA pipe (9 FP32 ops, no MUFU):
// k = rint(x/2pi) by the 1.5*2^23 trick, r = x/2pi - k in [-1/2, 1/2] (one FFMA),
// -2 cos(2 pi r) as a degree-4 minimax polynomial in r^2 (|err| < 9e-5), h = x + p.
__device__ __forceinline__ float snake_alt_h_fma(float x) {
  const float kb = fmaf(x, 0.15915494309189535f, 12582912.f);
  const float k = kb - 12582912.f;
  const float r = fmaf(x, 0.15915494309189535f, -k);
  const float u = r * r;
  float p = fmaf(-91.24539184570312f, u, 164.7942352294922f);
  p = fmaf(p, u, -129.34727478027344f);
  p = fmaf(p, u, 39.46232986450195f);
  p = fmaf(p, u, -1.999928951263428f);
  return x + p;
}

// snake_alt h = x - 2 cos x for TWO accumulator columns as one packed fp16 pair, on the
// FMA pipe in HFMA2 arithmetic (11 instructions per pair, no MUFU; the f32 version above
// costs 9 per element + half a pack).  x is rounded to fp16 first (the result is an fp16
// A operand anyway); k = rint(x/pi) by the 1.5*2^10 trick (|x| < 1600), r = x/pi - k in
// [-1/2, 1/2] half turns, -2 cos(pi r) as a degree-3 minimax polynomial in r^2
// (|err| < 1.4e-5 before fp16 rounding), the sign (-1)^k taken from the integer's low
// bit in the rounded t's mantissa and XORed into both halves' sign bits.
// FULL: whole turns instead, r = x/2pi - rint(x/2pi) in [-1/2, 1/2], -2 cos(2 pi r) of
// degree 4 in r^2 (|err| < 8.1e-5), no sign fix-up: 10 instructions per pair, slightly
// larger fp16 rounding error (mean |h err| 1.72e-3 vs 1.58e-3 over |x| < 8; MUFU + f32:
// 0.79e-3).  Measured (per word period 3): cfg 2 2.495 (half) / 2.50 (full) ms, cfg 3
// 22.63 (half) / 22.31 (full) ms.
template <bool FULL>
__device__ __forceinline__ uint32_t snake_alt_h2_fma(float x0, float x1) {
  const __half2 x = __floats2half2_rn(x0, x1);
  const __half2 magic = __float2half2_rn(1536.f);
  if constexpr (FULL) {
    const __half2 inv_2pi = __float2half2_rn(0.15915494309189535f);
    const __half2 k = __hsub2(__hfma2(x, inv_2pi, magic), magic);
    const __half2 r = __hfma2(x, inv_2pi, __hneg2(k));
    const __half2 v = __hmul2(r, r);
    __half2 p = __hfma2(__float2half2_rn(-91.29309655f), v, __float2half2_rn(164.80709908f));
    p = __hfma2(p, v, __float2half2_rn(-129.34686346f));
    p = __hfma2(p, v, __float2half2_rn(39.46208358f));
    p = __hfma2(p, v, __float2half2_rn(-1.9999196f));
    const __half2 h = __hadd2(x, p);
    return *reinterpret_cast<const uint32_t*>(&h);
  } else {
    const __half2 inv_pi = __float2half2_rn(0.3183098861837907f);
    const __half2 t = __hfma2(x, inv_pi, magic);
    const __half2 k = __hsub2(t, magic);
    const __half2 r = __hfma2(x, inv_pi, __hneg2(k));
    const __half2 v = __hmul2(r, r);
    __half2 p = __hfma2(__float2half2_rn(2.4442540271609667f), v, __float2half2_rn(-8.082567766703097f));
    p = __hfma2(p, v, __float2half2_rn(9.867876064596281f));
    p = __hfma2(p, v, __float2half2_rn(-1.9999865922852822f));
    const uint32_t tb = *reinterpret_cast<const uint32_t*>(&t);
    uint32_t pb = *reinterpret_cast<const uint32_t*>(&p);
    pb ^= (tb << 15) & 0x80008000u;
    const __half2 h = __hadd2(x, *reinterpret_cast<const __half2*>(&pb));
    return *reinterpret_cast<const uint32_t*>(&h);
  }
}

// sin(2 pi r), cos(2 pi r) for r in [-1/2, 1/2] on the FMA pipe: degree-5 least-
// squares-minimax polynomials in u = r^2 (|err| < 1.3e-6, MUFU.SIN/COS-class accuracy).
// 12 FP32 ops instead of FMUL.RZ + MUFU.SIN + MUFU.COS: the DVR path is XU-bound, so
// the NeRF base angles move to the FMA pipe (FVSRN_FOURIER_POLY=0 restores MUFU).
#ifndef FVSRN_FOURIER_POLY
#define FVSRN_FOURIER_POLY 1
#endif
#ifndef FVSRN_FOURIER_H2
#define FVSRN_FOURIER_H2 2   // FastRow: how many of the last doubling levels run in packed fp16
                             // (cfg 2 2.497 -> 2.473 ms with 2 or 4; 2 keeps the trained renders
                             // within 0.1 dB, 4 costs ~0.6 dB: profiles/r2/h2/precision_f*.txt)
#endif
__device__ __forceinline__ void sincos_turns(float r, float& s, float& c) {
  const float u = r * r;
  float pc = fmaf(-21.0767765045166f, u, 58.794036865234375f);
  pc = fmaf(pc, u, -85.27239990234375f);
  pc = fmaf(pc, u, 64.92872619628906f);
  pc = fmaf(pc, u, -19.738983154296875f);
  c = fmaf(pc, u, 0.9999992251396179f);
  float ps = fmaf(-12.473666191101074f, u, 41.34439468383789f);
  ps = fmaf(ps, u, -76.61480712890625f);
  ps = fmaf(ps, u, 81.5999755859375f);
  ps = fmaf(ps, u, -41.341590881347656f);
  ps = fmaf(ps, u, 6.283185005187988f);
  s = ps * r;
}

template <int ACT>
__device__ __forceinline__ float act_h(float x);

template <int ACT, bool POLY>
__device__ __forceinline__ float act_h2(float x) {
  if constexpr (POLY && ACT == 4) return fmaf(-2.f, cos_poly(x), x);
  else if constexpr (POLY && ACT == 3) return x - cos_poly(x);
  else return act_h<ACT>(x);
}

template <int ACT>
__device__ __forceinline__ float act_h(float x) {
  if constexpr (ACT == 0) {
    return fmaxf(x, 0.f);
  } else if constexpr (ACT == 1) {
    return __fdividef(1.f, 1.f + __expf(-x));
  } else if constexpr (ACT == 2) {
    return x > 20.f ? x : __logf(1.f + __expf(x));
  } else if constexpr (ACT == 3) {
    return x - __cosf(x);
  } else {
    return fmaf(-2.f, __cosf(x), x);
  }
}

// ---------------------------------------------------------------- warp MLP
// FVSRN_BREG=1: the B fragments of the hidden layers live in registers for the whole
// kernel (loaded once per warp) instead of one LDS.64 per MMA per step (A/B switch).
#ifndef FVSRN_BREG
#define FVSRN_BREG 0
#endif
template <int HID, int NL>
struct HiddenB {
  static constexpr int NLH = NL > 2 ? NL - 2 : 1;
  static constexpr bool kOn = FVSRN_BREG != 0 && NL > 2;
  uint2 f[kOn ? NLH : 1][kOn ? HID / 16 : 1][kOn ? HID / 8 : 1];
  __device__ void load(const uint2* wf, const NetDev& net, int lane) {
    if constexpr (kOn) {
#pragma unroll
      for (int l = 0; l < NLH; ++l)
#pragma unroll
        for (int kt = 0; kt < HID / 16; ++kt)
#pragma unroll
          for (int nt = 0; nt < HID / 8; ++nt)
            f[l][kt][nt] = wf[net.w_off[l + 1] + (kt * (HID / 8) + nt) * 32 + lane];
    }
  }
};

// Evaluates the whole network for the 32 rows staged in `stage` (row stride `rs`
// halfs) and writes head inputs (pre-head raw outputs, up to 4 per row) to
// `outbuf[row*4 + c]`.  MT = number of m16 tiles held at once (2 -> all 32 rows).
// NL / KT0 > 0: compile-time layer count / layer-0 k16 tiles (whole MLP is one basic
// block, so ptxas can overlap one layer's activations with the next layer's MMAs).
template <int HID, int MT, int ACT, int NL = 0, int KT0 = 0>
struct WarpMLP {
  static constexpr int NT = HID / 8;
  static constexpr int KT = HID / 16;

  template <int A>
  __device__ static void act_pack_t(const float (&acc)[MT][NT][4], uint32_t (&h)[MT][KT][4]) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        const float* a0 = acc[mt][2 * kt];
        const float* a1 = acc[mt][2 * kt + 1];
        constexpr int P = FVSRN_POLY_EVERY;
        const int e = (mt * KT + kt) * 8;   // element index within this thread's tile set
#define FVSRN_ACT(i, x) (P > 0 && ((e + (i)) % (P > 0 ? P : 1)) == (P > 0 ? P - 1 : 0) \
                             ? act_h2<A, true>(x) : act_h2<A, false>(x))
        if constexpr (A == 4 && FVSRN_MMA_H2 > 0) {
          // every FVSRN_MMA_H2-th n8 column tile: both cosines of each packed word in HFMA2
          // arithmetic.  Chosen by column only (the same for every row, lane and m16 tile),
          // so a ray's result does not depend on the row / warp it was scheduled to.
          constexpr int Q = FVSRN_MMA_H2 > 0 ? FVSRN_MMA_H2 : 1;
          const float* src[4] = {a0, a0 + 2, a1, a1 + 2};
#pragma unroll
          for (int i = 0; i < 4; ++i)
            h[mt][kt][i] = (2 * kt + (i >> 1)) % Q == Q - 1
                               ? snake_alt_h2_fma<false>(src[i][0], src[i][1])
                               : pack_half2(act_h<4>(src[i][0]), act_h<4>(src[i][1]));
          continue;
        }
        h[mt][kt][0] = pack_half2(FVSRN_ACT(0, a0[0]), FVSRN_ACT(1, a0[1]));
        h[mt][kt][1] = pack_half2(FVSRN_ACT(2, a0[2]), FVSRN_ACT(3, a0[3]));
        h[mt][kt][2] = pack_half2(FVSRN_ACT(4, a1[0]), FVSRN_ACT(5, a1[1]));
        h[mt][kt][3] = pack_half2(FVSRN_ACT(6, a1[2]), FVSRN_ACT(7, a1[3]));
#undef FVSRN_ACT
      }
  }

  __device__ static void act_pack(int act, const float (&acc)[MT][NT][4], uint32_t (&h)[MT][KT][4]) {
    if constexpr (ACT != kActRuntime) {
      act_pack_t<ACT>(acc, h);
    } else {
      switch (act) {   // warp-uniform, once per layer
        case 0: act_pack_t<0>(acc, h); break;
        case 1: act_pack_t<1>(acc, h); break;
        case 2: act_pack_t<2>(acc, h); break;
        case 3: act_pack_t<3>(acc, h); break;
        default: act_pack_t<4>(acc, h); break;
      }
    }
  }

  // B fragments of a hidden-width layer, stored in pairs: one LDS.128 per lane holds the
  // fragments of n8 tiles (2p, 2p+1) of k16 tile kt -> [kt][p][lane] x uint4.
  // (The compiler merges the two uint2 halves of one uint4 into a single load.)
  __device__ static uint2 bfrag(const uint2* wl, int kt, int nt, int lane) {
#if FVSRN_BPAIRS
    const uint4 v = *reinterpret_cast<const uint4*>(wl + ((kt * (NT / 2) + (nt >> 1)) * 32 + lane) * 2);
    return (nt & 1) ? make_uint2(v.z, v.w) : make_uint2(v.x, v.y);
#else
    return wl[(kt * NT + nt) * 32 + lane];
#endif
  }

  // Biases are stored as accumulator quads: for (n-tile nt, quad lane q) the float4
  // {b[nt*8+2q], b[nt*8+2q+1], same, same} at bs[(nt*4 + q)*4] -> one LDS.128 that is
  // the C operand of the layer's first MMA (no register copies).
  // FVSRN_BIAS64: read only the (b[2q], b[2q+1]) half of the quad (LDS.64) and repeat it
  // in registers.  Full-bandwidth LDS.128 serialises with MUFU on B200 where LDS.64
  // overlaps it (tools/microbench/mio_mix.cu), but these broadcast reads (64 B per warp)
  // measured neutral either way, so the quad load stays the default.
  __device__ static float4 bias_quad(const float* bs, int nt, int q) {
#if FVSRN_BIAS64
    const float2 v = *reinterpret_cast<const float2*>(bs + (nt * 4 + q) * 4);
    return make_float4(v.x, v.y, v.x, v.y);
#else
    return *reinterpret_cast<const float4*>(bs + (nt * 4 + q) * 4);
#endif
  }

  __device__ static void run(const __half* stage, int rs, const NetDev& net, const uint2* wf,
                             const float* bs, float* outbuf, int lane, int m_base) {
    run(stage, rs, net, wf, bs, outbuf, lane, m_base, HiddenB<HID, 0>{});
  }
  // m_base: first m16 tile index handled (0, or 0/1 when MT == 1)
  template <class HB>
  __device__ static void run(const __half* stage, int rs, const NetDev& net, const uint2* wf,
                             const float* bs, float* outbuf, int lane, int m_base, const HB& hb) {
    const int g = lane >> 2, q = lane & 3;
    const int arow = lane & 15, acol = (lane >> 4) * 8;
    float out_acc[MT][4];
    const __half* arow_ptr = stage + (m_base * 16 + arow) * rs + acol;
    const int layers = NL > 0 ? NL : net.layers;
    const int kt0 = KT0 > 0 ? KT0 : net.kt0;

    if (layers == 1) {
      const float4 bq = bias_quad(bs + net.b_off[0], 0, q);
      for (int kt = 0; kt < kt0; ++kt) {
        uint2 b = wf[net.w_off[0] + kt * 32 + lane];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          uint32_t a[4];
          ldmatrix_x4(a, arow_ptr + mt * 16 * rs + kt * 16);
          if (kt == 0) mma16816c(out_acc[mt], a, b, bq);
          else mma16816(out_acc[mt], a, b);
        }
      }
    } else {
      float acc[MT][NT][4];
      uint32_t h[MT][KT][4];
      // ---- layer 0: A from the stage, K = 16*kt0 (first k tile peeled: C = bias)
      {
        const float* b0 = bs + net.b_off[0];
        uint32_t a[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) ldmatrix_x4(a[mt], arow_ptr + mt * 16 * rs);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const uint2 b = bfrag(wf + net.w_off[0], 0, nt, lane);
          const float4 bq = bias_quad(b0, nt, q);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) mma16816c(acc[mt][nt], a[mt], b, bq);
        }
      }
#pragma unroll
      for (int kt = 1; kt < kt0; ++kt) {
        uint32_t a[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) ldmatrix_x4(a[mt], arow_ptr + mt * 16 * rs + kt * 16);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const uint2 b = bfrag(wf + net.w_off[0], kt, nt, lane);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) mma16816(acc[mt][nt], a[mt], b);
        }
      }
      act_pack(net.act, acc, h);
      // ---- hidden layers
#pragma unroll
      for (int l = 1; l < layers - 1; ++l) {
        const float* bl = bs + net.b_off[l];
#pragma unroll
        for (int kt = 0; kt < KT; ++kt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            uint2 b;
            if constexpr (HB::kOn) b = hb.f[l - 1][kt][nt];
            else b = bfrag(wf + net.w_off[l], kt, nt, lane);
            if (kt == 0) {
              const float4 bq = bias_quad(bl, nt, q);
#pragma unroll
              for (int mt = 0; mt < MT; ++mt) mma16816c(acc[mt][nt], h[mt][kt], b, bq);
            } else {
#pragma unroll
              for (int mt = 0; mt < MT; ++mt) mma16816(acc[mt][nt], h[mt][kt], b);
            }
          }
        act_pack(net.act, acc, h);
      }
      // ---- last layer: N = 8 (one n tile), linear
      const int L = layers - 1;
      const float4 bq = bias_quad(bs + net.b_off[L], 0, q);
      const uint2* wl = wf + net.w_off[L] + lane;
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        uint2 b = wl[kt * 32];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          if (kt == 0) mma16816c(out_acc[mt], h[mt][kt], b, bq);
          else mma16816(out_acc[mt], h[mt][kt], b);
        }
      }
    }
    if (q < 2) {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int r0 = (m_base + mt) * 16 + g;
        *reinterpret_cast<float2*>(outbuf + r0 * 4 + 2 * q) = make_float2(out_acc[mt][0], out_acc[mt][1]);
        *reinterpret_cast<float2*>(outbuf + (r0 + 8) * 4 + 2 * q) = make_float2(out_acc[mt][2], out_acc[mt][3]);
      }
    }
  }
};

// m16 tiles held at once by the warp MLP for 32-wide networks (FVSRN_MT32=1: one tile at a
// time, half the accumulator registers, weights read twice; A/B switch)
#ifndef FVSRN_MT32
#define FVSRN_MT32 2
#endif
template <int HID, int ACT, int NL = 0, int KT0 = 0>
struct MLPDispatch {
  static constexpr int MT = HID <= 32 ? FVSRN_MT32 : (HID <= 64 ? 2 : 1);
  using HB = HiddenB<HID, NL>;
  __device__ static void eval32(const __half* stage, int rs, const NetDev& net, const uint2* wf,
                                const float* bs, float* outbuf, int lane, const HB& hb) {
#pragma unroll
    for (int mb = 0; mb < 2; mb += MT)
      WarpMLP<HID, MT, ACT, NL, KT0>::run(stage, rs, net, wf, bs, outbuf, lane, mb, hb);
  }
  __device__ static void eval32(const __half* stage, int rs, const NetDev& net, const uint2* wf,
                                const float* bs, float* outbuf, int lane) {
    HB hb;
    eval32(stage, rs, net, wf, bs, outbuf, lane, hb);
  }
};

// ---------------------------------------------------------------- features
// Trilinear latent lookup (grid.py:47-84): clamp, c = p*(R-1), i0 = min(int c, R-2),
// 8-corner weighted sum; fp16 storage, f32 accumulation (FHFMA), 16-byte loads.
__device__ __forceinline__ void grid_features(const FeatDev& fd, float px, float py, float pz,
                                              __half* row) {
  const int R = fd.grid_res;
  const float s = (float)(R - 1);
  float cx = fminf(fmaxf(px, 0.f), 1.f) * s;
  float cy = fminf(fmaxf(py, 0.f), 1.f) * s;
  float cz = fminf(fmaxf(pz, 0.f), 1.f) * s;
  int x0 = min((int)cx, R - 2), y0 = min((int)cy, R - 2), z0 = min((int)cz, R - 2);
  float fx = cx - (float)x0, fy = cy - (float)y0, fz = cz - (float)z0;
  float gx = 1.f - fx, gy = 1.f - fy, gz = 1.f - fz;
  uint16_t w[8];
  {
    float wf[8] = {gx * gy * gz, gx * gy * fz, gx * fy * gz, gx * fy * fz,
                   fx * gy * gz, fx * gy * fz, fx * fy * gz, fx * fy * fz};
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = __half_as_ushort(__float2half_rn(wf[k]));
  }
  const int F = fd.f_pad;
  const int sz = F, sy = R * F, sx = R * R * F;
  const __half* base = fd.grid + ((size_t)(x0 * R + y0) * R + z0) * F;
  const int off[8] = {0, sz, sy, sy + sz, sx, sx + sz, sx + sy, sx + sy + sz};
  for (int c8 = 0; c8 < F; c8 += 8) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(reinterpret_cast<const uint4*>(base + off[k] + c8));
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t u[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[2 * j] = fhfma((uint16_t)(u[j] & 0xffff), w[k], acc[2 * j]);
        acc[2 * j + 1] = fhfma((uint16_t)(u[j] >> 16), w[k], acc[2 * j + 1]);
      }
    }
    uint4 o;
    o.x = pack_half2(acc[0], acc[1]); o.y = pack_half2(acc[2], acc[3]);
    o.z = pack_half2(acc[4], acc[5]); o.w = pack_half2(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(row + c8) = o;
  }
}

// Fourier features as (sin_i, cos_i) half2 pairs (nn.py:47-57, model.py:269-272).
// NeRF rows are 2^j * f32(2*pi) on one axis: one accurate base sincos per axis,
// then the double-angle recurrence (exact scaling by 2 of the f32 B entries).
__device__ __forceinline__ void fourier_features(const FeatDev& fd, const float (&v)[6],
                                                 __half* row) {
  uint32_t* dst = reinterpret_cast<uint32_t*>(row + fd.four_off);
  if (fd.fourier_mode == 1) {
    const int d = fd.fd_in;   // 3 or 6
    float sn[6], cs[6];
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      float r = v[a] - rintf(v[a]);                     // exact; keeps MUFU in [-pi, pi]
      __sincosf(r * 6.28318548202514648f, &sn[a], &cs[a]);
    }
    for (int base = 0; base < fd.m; base += d) {
#pragma unroll
      for (int a = 0; a < 6; ++a)
        if (a < d && base + a < fd.m) dst[base + a] = pack_half2(sn[a], cs[a]);
#pragma unroll
      for (int a = 0; a < 6; ++a) {
        float s2 = 2.f * sn[a] * cs[a];
        float c2 = fmaf(cs[a], cs[a], -sn[a] * sn[a]);
        sn[a] = s2; cs[a] = c2;
      }
    }
  } else if (fd.fourier_mode == 2) {
    for (int i = 0; i < fd.m; ++i) {
      float ph = 0.f;
#pragma unroll
      for (int a = 0; a < 6; ++a)
        if (a < fd.fd_in) ph = fmaf(__ldg(fd.bmat + i * fd.fd_in + a), v[a], ph);
      float s, c;
      sincosf(ph, &s, &c);
      dst[i] = pack_half2(s, c);
    }
  }
}

// Assemble this lane's input row: [z | sin/cos pairs | p (| d) | 0-pad].
__device__ __forceinline__ void assemble_row(const FeatDev& fd, float px, float py, float pz,
                                             float dx, float dy, float dz, __half* row) {
  if (fd.f_pad > 0) grid_features(fd, px, py, pz, row);
  float v[6] = {px, py, pz, dx, dy, dz};
  if (fd.fourier_mode != 0) fourier_features(fd, v, row);
  // raw block (raw_off is even): p then d (dir modes)
  uint32_t* dst = reinterpret_cast<uint32_t*>(row + fd.raw_off);
  if (fd.raw_w == 3) {
    dst[0] = pack_half2(px, py);
    dst[1] = pack_half2(pz, 0.f);
  } else {
    dst[0] = pack_half2(px, py);
    dst[1] = pack_half2(pz, dx);
    dst[2] = pack_half2(dy, dz);
  }
}

// ---------------------------------------------------------------- specialised row
// Fast path for the default fV-SRN input (pos mode, NeRF m = NM on 3 axes, F = 16):
// the whole row [z16 | (sin,cos) x NM | p | 0] is built in registers and written
// with 16-byte stores (conflict-free at the odd 16-byte row stride).
#ifndef FVSRN_LDG256
#define FVSRN_LDG256 1
#endif
// 32 bytes (32-byte aligned) through the read-only path in one LDG.256 (sm_100)
__device__ __forceinline__ void ldg256(const uint4* p, uint4& a, uint4& b) {
  asm("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
      : "l"(p));
}

#ifndef FVSRN_TEX_F16X2
#define FVSRN_TEX_F16X2 1
#endif

template <int NM>
struct FastRow {
  static constexpr int kWidth = 16 + 2 * NM + 3;
  static constexpr int kK0 = (kWidth + 15) / 16 * 16;
  static constexpr int kWords = kK0 / 2;

  // CS: distance (in 16-byte chunks) between consecutive 8-column chunks of the row:
  // 1 = row-major stage, 8 = UMMA K-major canonical layout (128 B per core matrix).
  template <int CS = 1>
  __device__ static void build(const FeatDev& fd, float px, float py, float pz, __half* row) {
    uint32_t w[kWords];
    words(fd, px, py, pz, w);
    uint4* dst = reinterpret_cast<uint4*>(row);
#pragma unroll
    for (int j = 0; j < kWords / 4; ++j) dst[j * CS] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
  }

  // the row as kWords packed fp16 pairs (column 2i in the low half of w[i])
  __device__ static void words(const FeatDev& fd, float px, float py, float pz, uint32_t (&w)[kWords]) {
#pragma unroll
    for (int i = 0; i < kWords; ++i) w[i] = 0u;
    // latent grid (grid.py:47-84), 16 channels
    if (fd.tex_on && !fd.tex_u8 && fd.tex_w == 0.f) {
      // static fp16 texture grid: the same fetch as the specialised frame kernels
      uint32_t z[8];
      tex_words(fd, px, py, pz, z);
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = z[i];
    } else if (fd.tex_on) {
      // texture units: unnormalised coordinates, texel centres at i + 1/2, clamp
      // addressing (== the reference's clamp of p and of i0 <= R-2); array width is the
      // grid's z axis (fastest in memory), depth its x axis
      const float s = (float)(fd.grid_res - 1);
      const float tz = fmaf(fminf(fmaxf(px, 0.f), 1.f), s, 0.5f);
      const float ty = fmaf(fminf(fmaxf(py, 0.f), 1.f), s, 0.5f);
      const float tx = fmaf(fminf(fmaxf(pz, 0.f), 1.f), s, 0.5f);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float4 v = tex3D<float4>(fd.tex_lo[j], tx, ty, tz);
        if (fd.tex_u8) {
          v.x = fmaf(v.x, fd.qspan_lo[4 * j], fd.qmin_lo[4 * j]);
          v.y = fmaf(v.y, fd.qspan_lo[4 * j + 1], fd.qmin_lo[4 * j + 1]);
          v.z = fmaf(v.z, fd.qspan_lo[4 * j + 2], fd.qmin_lo[4 * j + 2]);
          v.w = fmaf(v.w, fd.qspan_lo[4 * j + 3], fd.qmin_lo[4 * j + 3]);
        }
        if (fd.tex_w != 0.f) {
          float4 u = tex3D<float4>(fd.tex_hi[j], tx, ty, tz);
          if (fd.tex_u8) {
            u.x = fmaf(u.x, fd.qspan_hi[4 * j], fd.qmin_hi[4 * j]);
            u.y = fmaf(u.y, fd.qspan_hi[4 * j + 1], fd.qmin_hi[4 * j + 1]);
            u.z = fmaf(u.z, fd.qspan_hi[4 * j + 2], fd.qmin_hi[4 * j + 2]);
            u.w = fmaf(u.w, fd.qspan_hi[4 * j + 3], fd.qmin_hi[4 * j + 3]);
          }
          v.x = fmaf(fd.tex_w, u.x - v.x, v.x); v.y = fmaf(fd.tex_w, u.y - v.y, v.y);
          v.z = fmaf(fd.tex_w, u.z - v.z, v.z); v.w = fmaf(fd.tex_w, u.w - v.w, v.w);
        }
        w[2 * j] = pack_half2(v.x, v.y);
        w[2 * j + 1] = pack_half2(v.z, v.w);
      }
    } else {
      uint32_t z[8];
      ldg_words(fd, px, py, pz, z);
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = z[i];
    }
    fourier_words(px, py, pz, w);
  }

  // exact-weight trilinear latent lookup (grid.py:47-84) of a 16-channel fp16 grid: 16
  // LDG.128 + HFMA2 products, as 8 packed fp16 pairs
  __device__ static void ldg_words(const FeatDev& fd, float px, float py, float pz, uint32_t (&z)[8]) {
    const int R = fd.grid_res;
    const float s = (float)(R - 1);
    const float rm2 = (float)(R - 2);
    float cx = fminf(fmaxf(px, 0.f), 1.f) * s;
    float cy = fminf(fmaxf(py, 0.f), 1.f) * s;
    float cz = fminf(fmaxf(pz, 0.f), 1.f) * s;
    int x0, y0, z0;   // i0 = min(int c, R-2) (grid.py:47-53), c >= 0 so trunc == floor
    float x0f = floor_pos(cx, x0), y0f = floor_pos(cy, y0), z0f = floor_pos(cz, z0);
    if (x0 > R - 2) { x0 = R - 2; x0f = rm2; }
    if (y0 > R - 2) { y0 = R - 2; y0f = rm2; }
    if (z0 > R - 2) { z0 = R - 2; z0f = rm2; }
    float fx = cx - x0f, fy = cy - y0f, fz = cz - z0f;
    float gx = 1.f - fx, gy = 1.f - fy, gz = 1.f - fz;
    const float wf[8] = {gx * gy * gz, gx * gy * fz, gx * fy * gz, gx * fy * fz,
                         fx * gy * gz, fx * gy * fz, fx * fy * gz, fx * fy * fz};
    __half2 wk[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) wk[k] = __float2half2_rn(wf[k]);
    const int sz = 16, sy = R * 16, sx = R * R * 16;
    const uint4* base = reinterpret_cast<const uint4*>(fd.grid + ((size_t)(x0 * R + y0) * R + z0) * 16);
    const int off[8] = {0, sz, sy, sy + sz, sx, sx + sz, sx + sy, sx + sy + sz};
    // one 256-bit load per corner (LDG.256: the voxel's 16 fp16 channels), FVSRN_LDG256=0:
    // two 128-bit loads
    uint4 vv[2][8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#if FVSRN_LDG256
      ldg256(base + (off[k] >> 3), vv[0][k], vv[1][k]);
#else
      vv[0][k] = __ldg(base + (off[k] >> 3));
      vv[1][k] = __ldg(base + (off[k] >> 3) + 1);
#endif
    }
#pragma unroll
    for (int c8 = 0; c8 < 2; ++c8) {
      const uint4 (&v)[8] = vv[c8];
      // z = sum_k w_k g_k in packed half2 (HFMA2): 32 instructions per 8 channels
      __half2 acc[4];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const __half2* g2 = reinterpret_cast<const __half2*>(&v[k]);
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = k == 0 ? __hmul2(wk[k], g2[j]) : __hfma2(wk[k], g2[j], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) z[4 * c8 + j] = *reinterpret_cast<uint32_t*>(&acc[j]);
    }
  }

  // the whole row from the static fp16 LDG grid (no u8 codes, no keyframe blend): the
  // branch-free feature path of the frame kernels with the exact-weight sampler
  __device__ static void build_ldg(const FeatDev& fd, float px, float py, float pz, __half* row) {
    uint32_t z[8], w[kWords];
    ldg_words(fd, px, py, pz, z);
    words_from_z(z, px, py, pz, w);
    uint4* dst = reinterpret_cast<uint4*>(row);
#pragma unroll
    for (int j = 0; j < kWords / 4; ++j) dst[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
  }

  // texture-unit latent lookup of a static fp16 grid (fd.tex_on, no u8 codes, no keyframe
  // blend): the four raw RGBA16F fetches, so a caller can issue them early and consume
  // them later (words_from_tex)
  __device__ static void tex_fetch(const FeatDev& fd, float px, float py, float pz, float4 (&v)[4]) {
    const float s = (float)(fd.grid_res - 1);
    const float tz = fmaf(fminf(fmaxf(px, 0.f), 1.f), s, 0.5f);
    const float ty = fmaf(fminf(fmaxf(py, 0.f), 1.f), s, 0.5f);
    const float tx = fmaf(fminf(fmaxf(pz, 0.f), 1.f), s, 0.5f);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = tex3D<float4>(fd.tex_lo[j], tx, ty, tz);
  }

  // the whole row from a static fp16 texture grid (no u8 codes, no keyframe blend), with
  // 16-byte stores: the branch-free feature path of the kDVRTex kernel
  __device__ static void build_tex(const FeatDev& fd, float px, float py, float pz, __half* row) {
    uint32_t z[8], w[kWords];
    tex_words(fd, px, py, pz, z);
    words_from_z(z, px, py, pz, w);
    uint4* dst = reinterpret_cast<uint4*>(row);
#pragma unroll
    for (int j = 0; j < kWords / 4; ++j) dst[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
  }

  // the 16 latent channels of a static fp16 texture grid as 8 packed fp16 pairs
  // (FVSRN_TEX_F16X2: the texture unit returns them packed -- tex.3d.v2.f16x2 -- instead
  // of 16 f32 values the SM converts; every static-texture path fetches through here)
  __device__ static void tex_words(const FeatDev& fd, float px, float py, float pz, uint32_t (&z)[8]) {
#if FVSRN_TEX_F16X2
    const float s = (float)(fd.grid_res - 1);
    const float tz = fmaf(fminf(fmaxf(px, 0.f), 1.f), s, 0.5f);
    const float ty = fmaf(fminf(fmaxf(py, 0.f), 1.f), s, 0.5f);
    const float tx = fmaf(fminf(fmaxf(pz, 0.f), 1.f), s, 0.5f);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("tex.3d.v2.f16x2.f32 {%0, %1}, [%2, {%3, %4, %5, %6}];"
                   : "=r"(z[2 * j]), "=r"(z[2 * j + 1])
                   : "l"(fd.tex_lo[j]), "f"(tx), "f"(ty), "f"(tz), "f"(0.f));
#else
    float4 v[4];
    tex_fetch(fd, px, py, pz, v);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      z[2 * j] = pack_half2(v[j].x, v[j].y);
      z[2 * j + 1] = pack_half2(v[j].z, v[j].w);
    }
#endif
  }

  __device__ static void words_from_z(const uint32_t (&z)[8], float px, float py, float pz,
                                      uint32_t (&w)[kWords]) {
#pragma unroll
    for (int i = 0; i < kWords; ++i) w[i] = i < 8 ? z[i] : 0u;
    fourier_words(px, py, pz, w);
  }

  // NeRF Fourier pairs and the raw position (columns 16 .. kWidth-1)
  __device__ static void fourier_words(float px, float py, float pz, uint32_t (&w)[kWords]) {
    // NeRF Fourier pairs: base angle f32(2 pi) * (p - rint p), then doubling
    {
      const float pv[3] = {px, py, pz};
      float sn[3], cs[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const float r = pv[a] - rint_fma(pv[a]);   // exact, in [-1/2, 1/2]
        if (FVSRN_FOURIER_POLY) sincos_turns(r, sn[a], cs[a]);
        else __sincosf(r * 6.28318548202514648f, &sn[a], &cs[a]);
      }
      // the last FVSRN_FOURIER_H2 doublings in packed fp16 on the (sin, cos) words:
      // (s, c) -> (2s c, 1 - 2 s^2) = HFMA2((2s, -2s), (c, s), (0, 1)): 3 instructions per
      // axis instead of 4 FP32 operations + a pack
      constexpr int kLevels = (NM - 1) / 3;
      constexpr int kH2From = kLevels - FVSRN_FOURIER_H2 + 1;   // first packed level
      uint32_t pw[3];
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        const int a = i % 3;
        const int lev = i / 3;
        if (i > 0 && a == 0) {
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            if (FVSRN_FOURIER_H2 > 0 && lev >= kH2From) {
              if (lev == kH2From) pw[b] = pack_half2(sn[b], cs[b]);
              const __half2 x = *reinterpret_cast<const __half2*>(&pw[b]);
              const __half2 u = __hmul2(__low2half2(x), __floats2half2_rn(2.f, -2.f));
              const __half2 sw = __lowhigh2highlow(x);
              const __half2 y = __hfma2(u, sw, __floats2half2_rn(0.f, 1.f));
              pw[b] = *reinterpret_cast<const uint32_t*>(&y);
            } else {
              float s2 = 2.f * sn[b] * cs[b];
              float c2 = fmaf(cs[b], cs[b], -sn[b] * sn[b]);
              sn[b] = s2; cs[b] = c2;
            }
          }
        }
        w[8 + i] = (FVSRN_FOURIER_H2 > 0 && lev >= kH2From && lev > 0) ? pw[a] : pack_half2(sn[a], cs[a]);
      }
    }
    w[8 + NM] = pack_half2(px, py);
    w[9 + NM] = pack_half2(pz, 0.f);
  }
};

// NM > 0: specialised row; NM == 0: generic runtime layout
template <int NM>
__device__ __forceinline__ void assemble_row_t(const FeatDev& fd, float px, float py, float pz,
                                               float dx, float dy, float dz, __half* row) {
  if constexpr (NM > 0) {
    FastRow<NM>::template build<1>(fd, px, py, pz, row);
  } else {
    assemble_row(fd, px, py, pz, dx, dy, dz, row);
  }
}

// ---------------------------------------------------------------- TF + heads
// sigmoid as 1/2 + tanh(x/2)/2: one MUFU.TANH instead of EX2 + RCP (|err| < 2.5e-4,
// A/B switch FVSRN_SIGMOID_TANH=0 restores the two-MUFU form).
#ifndef FVSRN_SIGMOID_TANH
#define FVSRN_SIGMOID_TANH 1
#endif
__device__ __forceinline__ float sigmoidf_(float x) {
#if FVSRN_SIGMOID_TANH
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
  return fmaf(0.5f, t, 0.5f);
#else
  return __fdividef(1.f, 1.f + __expf(-x));
#endif
}
__device__ __forceinline__ float softplusf_(float x) { return x > 20.f ? x : log1pf(__expf(x)); }

// transfer.py:57-65: clamp to [0,1], piecewise-linear interpolation.
__device__ __forceinline__ void tf_eval(const TFDev& tf, float dens, float& r, float& g, float& b,
                                        float& sig) {
  float d = fminf(fmaxf(dens, 0.f), 1.f);
  int seg = 0;
  for (int i = 1; i < tf.n - 1; ++i) seg += (d >= tf.xs[i]) ? 1 : 0;
  float dx = d - tf.xs[seg];
  r = fmaf(tf.slope[seg][0], dx, tf.val[seg][0]);
  g = fmaf(tf.slope[seg][1], dx, tf.val[seg][1]);
  b = fmaf(tf.slope[seg][2], dx, tf.val[seg][2]);
  sig = fmaf(tf.slope[seg][3], dx, tf.val[seg][3]);
}

}  // namespace fvsrn
