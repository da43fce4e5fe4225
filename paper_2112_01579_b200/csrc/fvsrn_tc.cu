// fvsrn_tc.cu -- tcgen05 / TMEM variant of the fused fV-SRN DVR kernel (sm_100a).
//
// One CTA = 4 warps = 128 rays = one M=128 UMMA tile.  Thread t owns ray t and TMEM
// lane t, so the row-per-thread accumulator layout of tcgen05.ld is also the
// ray-per-thread layout of the marcher: no fragment shuffles, no output staging.
// Per ray-march step (render.py:219-232):
//   1. every thread refills its ray if needed (chunked global queue, f64 geometry)
//      and writes its input row [z | sin/cos pairs | p] (FastRow) into the A tile in
//      shared memory, in the UMMA K-major canonical layout (8x16 B core matrices);
//   2. per layer: one elected thread issues K/16 tcgen05.mma (A = rows in smem,
//      B = weights in smem, D = f32 accumulators in TMEM, pre-loaded with the layer
//      bias by tcgen05.st so the bias stays f32-exact) and commits to an mbarrier;
//      every thread tcgen05.ld's its row, evaluates the snake activation in registers
//      (one MUFU.COS per element) and writes the fp16 row back into the A tile;
//   3. the last layer's 4 outputs go straight to head/TF/compositing/ET in registers.
// The MLP never touches global memory; the HMMA issue slots and the B-fragment LDS of
// the mma.sync kernel disappear from the SM sub-partitions' instruction streams.
// Used for the default fV-SRN configurations (FastRow inputs, snake_alt, 32/64 wide).
// The tcgen05 kernels are issue-bound with XU headroom (cfg 2: issue 74%, XU 63%), the
// mma.sync ones XU-bound: here the NeRF base angles go to MUFU.SIN/COS (3 issue slots per
// axis instead of 15 FMA-pipe operations): cfg 2 2.86 -> 2.82 ms, cfg 5 42.6 -> 41.6 ms
#ifndef FVSRN_FOURIER_POLY
#define FVSRN_FOURIER_POLY 0
#endif
#include "fvsrn_march.cuh"
#include "fvsrn_tc.cuh"
#include "fvsrn_tmem.cuh"

namespace fvsrn {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&r)[N]) {
  if constexpr (N == 16) tmem_ld_x16(taddr, r);
  else if constexpr (N == 32) tmem_ld_x32(taddr, r);
  else tmem_ld_x64(taddr, r);
}

// D <- bias (same N values in every lane): broadcast LDS.128 + one tcgen05.st
template <int N>
__device__ __forceinline__ void tmem_bias(uint32_t taddr, const float* b) {
  uint32_t v[N];
#pragma unroll
  for (int i = 0; i < N; i += 4) {
    const float4 q = *reinterpret_cast<const float4*>(b + i);
    v[i] = __float_as_uint(q.x); v[i + 1] = __float_as_uint(q.y);
    v[i + 2] = __float_as_uint(q.z); v[i + 3] = __float_as_uint(q.w);
  }
  if constexpr (N == 16) tmem_st_x16(taddr, v);
  else if constexpr (N == 32) tmem_st_x32(taddr, v);
  else tmem_st_x64(taddr, v);
}

// Activation of element e of a row: every FVSRN_TC_POLY-th element evaluates its cosine
// on the FMA pipe instead of the XU (MUFU) pipe.  The tcgen05 kernels are XU-bound in
// their activation phases with issue slots to spare (6x64 at 4 CTAs/SM: issue 46%,
// XU 67%), so moving every 6th cosine balances the two (cfg 3: 28.2 -> 26.9 ms;
// every 3rd 28.9, 4th 27.8, 8th 27.1, 12th 27.2, 16th 27.3).  0 disables.
#ifndef FVSRN_TC_POLY
#define FVSRN_TC_POLY 6
#endif
#ifndef FVSRN_TC_SPLIT
#define FVSRN_TC_SPLIT 1
#endif
#ifndef FVSRN_TC_PREFETCH
#define FVSRN_TC_PREFETCH 0
#endif
#ifndef FVSRN_TC_WAIT_BAR
#define FVSRN_TC_WAIT_BAR 0
#endif
// FVSRN_TC_NSPLIT: the 64-wide layers' MMA is issued as two N=32 halves committing to two
// mbarriers, so the activations of the first half overlap the second half's MMA (the packed
// first half waits in registers: A is rewritten only after the whole MMA has read it)
#ifndef FVSRN_TC_NSPLIT
#define FVSRN_TC_NSPLIT 0
#endif
// hidden-layer A operands in TMEM (tcgen05.st of the packed activations, MMA reads A
// from TMEM) instead of the shared-memory A tile: removes 2 x 128 B of shared-memory
// traffic per sample and layer
#ifndef FVSRN_TC_TMEM_A
#define FVSRN_TC_TMEM_A 1
#endif
// FVSRN_TC_TMEM_A0 (fvsrn_tc.cuh): layer-0 input rows in TMEM too (measured at 3
// CTAs/SM: faster at 32-wide, slower at 64-wide)
// snake_alt activations of one accumulator row -> fp16 chunks of the A tile row
// (chunk c = columns 8c..8c+7 at +128 B per chunk in the canonical layout)
template <int HID>
__device__ __forceinline__ void act_row(const uint32_t (&acc)[HID], __half* row) {
  constexpr int P = FVSRN_TC_POLY;
#pragma unroll
  for (int c = 0; c < HID / 8; ++c) {
    uint32_t w4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float h[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int e = 8 * c + 2 * j + i;       // compile-time after unrolling
        const float x = __uint_as_float(acc[e]);
        h[i] = (P > 0 && e % (P > 0 ? P : 1) == P - 1) ? snake_alt_h_fma(x) : act_h<4>(x);
      }
      w4[j] = pack_half2(h[0], h[1]);
    }
    *reinterpret_cast<uint4*>(row + c * 64) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
  }
}

// snake_alt activations of one accumulator row -> packed fp16 pairs (TMEM A operand)
template <int HID>
__device__ __forceinline__ void act_words(const uint32_t (&acc)[HID], uint32_t (&w)[HID / 2]) {
  constexpr int P = FVSRN_TC_POLY;
#pragma unroll
  for (int j = 0; j < HID / 2; ++j) {
    float h[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int e = 2 * j + i;
      const float x = __uint_as_float(acc[e]);
      h[i] = (P > 0 && e % (P > 0 ? P : 1) == P - 1) ? snake_alt_h_fma(x) : act_h<4>(x);
    }
    w[j] = pack_half2(h[0], h[1]);
  }
}

// cos(a) on the FMA pipe (range reduction by the 1.5*2^23 trick, degree-4 minimax in r^2
// of cos(2 pi r), |err| < 4.3e-5): 8 FP32 operations, no MUFU
__device__ __forceinline__ float cos_fma(float x) {
  const float kb = fmaf(x, 0.15915494309189535f, 12582912.f);
  const float k = kb - 12582912.f;
  const float r = fmaf(x, 0.15915494309189535f, -k);
  const float u = r * r;
  float p = fmaf(45.62269592285156f, u, -82.3971176147461f);
  p = fmaf(p, u, 64.67363739013672f);
  p = fmaf(p, u, -19.731164932250977f);
  return fmaf(p, u, 0.9999644756317139f);
}

// skip path: cos(a) of one accumulator row -> fp16 chunks of the shared-memory A tile row
// (every FVSRN_TC_POLY-th element on the FMA pipe, as act_row)
template <int HID>
__device__ __forceinline__ void cos_row(const uint32_t (&acc)[HID], __half* row) {
  constexpr int P = FVSRN_TC_POLY;
#pragma unroll
  for (int c = 0; c < HID / 8; ++c) {
    uint32_t w4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float h[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int e = 8 * c + 2 * j + i;
        const float x = __uint_as_float(acc[e]);
        h[i] = (P > 0 && e % (P > 0 ? P : 1) == P - 1) ? cos_fma(x) : __cosf(x);
      }
      w4[j] = pack_half2(h[0], h[1]);
    }
    *reinterpret_cast<uint4*>(row + c * 64) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
  }
}

template <int N>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t (&r)[N]) {
  if constexpr (N == 16) tmem_st_x16(taddr, r);
  else if constexpr (N == 32) tmem_st_x32(taddr, r);
  else tmem_st_x64(taddr, r);
}

// store N words (N = sum of powers of two from {32, 16, 8, 4}) at consecutive columns
template <int N, int OFF = 0, int M>
__device__ __forceinline__ void tmem_st_any(uint32_t taddr, const uint32_t (&r)[M]) {
  if constexpr (N >= 32) {
    uint32_t v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = r[OFF + i];
    tmem_st_x32(taddr + OFF, v);
    tmem_st_any<N - 32, OFF + 32>(taddr, r);
  } else if constexpr (N >= 16) {
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = r[OFF + i];
    tmem_st_x16(taddr + OFF, v);
    tmem_st_any<N - 16, OFF + 16>(taddr, r);
  } else if constexpr (N >= 8) {
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = r[OFF + i];
    tmem_st_x8(taddr + OFF, v);
    tmem_st_any<N - 8, OFF + 8>(taddr, r);
  } else if constexpr (N >= 4) {
    uint32_t v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = r[OFF + i];
    tmem_st_x4(taddr + OFF, v);
    tmem_st_any<N - 4, OFF + 4>(taddr, r);
  }
}

}  // namespace

template <int HID, int NM, int NL, int TEX = 0>
__global__ void __launch_bounds__(kTcThreads, tc_min_blocks<HID>())
dvr_tc_kernel(TcNetDev net, FeatDev fd, const TFDev* __restrict__ tf_g, const float* __restrict__ b0,
              MarchDev md, CamDev cam, ShardDev sh, int explicit_rays, RayRecs rr, long long n_slots,
              float* __restrict__ out, unsigned long long* __restrict__ queue,
              unsigned long long* __restrict__ eval_count, unsigned long long* __restrict__ nonfinite) {
  using S = TcShape<HID, NM, NL>;
  extern __shared__ __align__(128) unsigned char smem[];
  __half* w_s = reinterpret_cast<__half*>(smem + S::kWOff);
  float* b_s = reinterpret_cast<float*>(smem + S::kBOff);
  TFDev* tf = reinterpret_cast<TFDev*>(smem + S::kTFOff);
  __half* a_s = reinterpret_cast<__half*>(smem + S::kAOff);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + S::kMbarOff);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::kMbarOff + 8);
  uint64_t* mbar1 = reinterpret_cast<uint64_t*>(smem + S::kMbarOff + 16);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    const uint4* src = net.w;
    uint4* dst = reinterpret_cast<uint4*>(w_s);
    for (int i = tid; i < S::kWBytes / 16; i += kTcThreads) dst[i] = src[i];
    for (int i = tid; i < S::kBTotal; i += kTcThreads)
      b_s[i] = (b0 && i < HID) ? b0[i] : net.b[i];
    const int words = sizeof(TFDev) / 4;
    const int* ts = reinterpret_cast<const int*>(tf_g);
    int* td = reinterpret_cast<int*>(tf);
    for (int i = tid; i < words; i += kTcThreads) td[i] = ts[i];
    if constexpr (!S::kA0 || S::kSkip) {
      // pad columns must stay finite; skip path: columns HID, HID+1 = 1.0 (the bias tile)
      uint4* az = reinterpret_cast<uint4*>(a_s);
      for (int i = tid; i < kTcThreads * S::kKA / 8; i += kTcThreads) {
        const bool ones = S::kSkip && (i / 8) % (S::kKA / 8) == HID / 8;   // chunk of columns HID..HID+7
        az[i] = make_uint4(ones ? 0x3C003C00u : 0u, 0u, 0u, 0u);
      }
    }
  }
  constexpr bool kA0 = S::kA0;
  // TMEM columns: D [0, kTCols), A [kTCols, kTCols + max(K0, HID)/2)
  // skip path: the A columns are the second accumulator region (layer-0 rows, then the
  // odd layers' accumulators)
  constexpr bool kNSplit = FVSRN_TC_NSPLIT == 1 && HID == 64 && FVSRN_TC_TMEM_A && FVSRN_TC_SPLIT;
  // FVSRN_TC_NSPLIT == 2: the hidden layers' MMA in two N=32 halves, the activations of the
  // first half overlapping the second half's MMA, with the hidden A operand double-buffered
  // in TMEM (layer l reads buffer l & 1, writes l + 1's) so nothing waits in registers
  constexpr bool kDbl = FVSRN_TC_NSPLIT == 2 && HID == 64 && FVSRN_TC_TMEM_A && FVSRN_TC_SPLIT && S::kA0 &&
                        !S::kBiasMma && !S::kBiasCp;
  // TMEM column offset (from kTCols) of layer l's A operand
  auto a_col = [](int l) -> uint32_t { return (kDbl && l > 0 && (l & 1)) ? 32u : 0u; };
  constexpr uint32_t kAcols = S::kSkip ? S::kTCols : kDbl ? 64u : kA0 ? S::kKA / 2 : (FVSRN_TC_TMEM_A ? HID / 2 : 0);
  constexpr uint32_t kNeed = S::kTCols + kAcols;
  constexpr uint32_t kAlloc = kNeed <= 32 ? 32 : kNeed <= 64 ? 64 : kNeed <= 128 ? 128 : 256;
  if (warp == 0) tmem_alloc(smem_u32(tmem_slot), kAlloc);
  if (tid == 0) {
    mbar_init(smem_u32(mbar), 1);
    mbar_init(smem_u32(mbar1), 1);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if constexpr (S::kBiasMma) {
    static_assert(S::kA0, "bias-in-MMA needs the layer-0 rows in TMEM");
    // W0's pad column (K0 - 1; the row's pad is 1.0) := this frame's layer-0 bias
    constexpr int K = S::kK0, k = S::kK0 - 1;
    for (int n = tid; n < HID; n += kTcThreads)
      w_s[(n / 8) * (K / 8) * 64 + (k / 8) * 64 + (n % 8) * 8 + (k % 8)] = __float2half_rn(b_s[n]);
    fence_proxy_async_smem();
    __syncthreads();
  }
  if constexpr (S::kBiasCp) {
    // bias broadcast tiles from b_s (b0 of this frame for layer 0)
    for (int i = tid; i < S::kBTotal * 8; i += kTcThreads) {
      const int c = i >> 3, r = i & 7;
      *reinterpret_cast<float*>(smem + S::kBcOff + (c / 8) * 256 + ((c % 8) / 4) * 128 + r * 16 + (c % 4) * 4) = b_s[c];
    }
    fence_proxy_async_smem();
    __syncthreads();
  }
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);   // this warp's TMEM lanes
  const uint32_t a_base = smem_u32(a_s), w_base = smem_u32(w_s), mb = smem_u32(mbar), mb1 = smem_u32(mbar1);
  uint32_t phase1 = 0;
  // row tid of the A tile: 8-row group stride SBO_A, row-in-group stride 16 B
  __half* myrow = a_s + (tid >> 3) * (S::kSboA / 2) + (tid & 7) * 8;
  const bool density = net.head == 0;

  RayLane r;
  r.has = false;
  LaneQueue q{0, 0, false};
  unsigned long long evals = 0;
  uint32_t phase = 0;
  // FVSRN_TC_PREFETCH: the next sample's latent-grid texture fetches are issued before the
  // last layer's MMA wait, so their latency hides under it (static fp16 texture grids)
  const bool prefetch = FVSRN_TC_PREFETCH && kA0 && fd.tex_on && !fd.tex_u8 && fd.tex_w == 0.f;
  uint32_t pre[8];
  int pre_k = -1;

  // TEX == 1: a camera frame (no explicit rays, no direction inputs) of a density-head
  // model with a static fp16 texture grid: those flags are compile-time
  constexpr bool kFrame = TEX >= 1;
  while (true) {
    if constexpr (kFrame) {
      RayRecs rr_pos = rr;
      rr_pos.d = nullptr;
      ws_refill(r, q, lane, cam, sh, false, rr_pos, n_slots, queue, md, out);
    } else {
      ws_refill(r, q, lane, cam, sh, explicit_rays != 0, rr, n_slots, queue, md, out);
    }
    if (!__syncthreads_or(r.has)) break;
    evals += __popc(__ballot_sync(0xffffffffu, r.has));
    if constexpr (!S::kBiasMma && !S::kBiasCp) tmem_bias<HID>(t_row, b_s + S::b_off(0));
    if constexpr (kA0) {
      // tcgen05.st is .sync.aligned: every lane stores (rays-less lanes a zero row)
      uint32_t w[FastRow<NM>::kWords];
      if (r.has) {
        const float kf = (float)r.k;
        const float px = fmaf(kf, r.dd0, r.pe0), py = fmaf(kf, r.dd1, r.pe1), pz = fmaf(kf, r.dd2, r.pe2);
        if (prefetch && pre_k == r.k) {
          FastRow<NM>::words_from_z(pre, px, py, pz, w);
        } else if constexpr (TEX >= 1) {   // static fp16 grid: no runtime branches
          uint32_t z[8];
          if constexpr (TEX == 1) FastRow<NM>::tex_words(fd, px, py, pz, z);
          else FastRow<NM>::ldg_words(fd, px, py, pz, z);
          FastRow<NM>::words_from_z(z, px, py, pz, w);
        } else {
          FastRow<NM>::words(fd, px, py, pz, w);
        }
      } else {
#pragma unroll
        for (int i = 0; i < FastRow<NM>::kWords; ++i) w[i] = 0u;
      }
      if constexpr (S::kBiasMma) w[FastRow<NM>::kWords - 1] |= 0x3C000000u;   // pad column = 1.0
      tmem_st_any<FastRow<NM>::kWords>(t_row + S::kTCols, w);
    } else if (r.has) {
      const float kf = (float)r.k;
      FastRow<NM>::template build<8>(fd, fmaf(kf, r.dd0, r.pe0), fmaf(kf, r.dd1, r.pe1),
                                     fmaf(kf, r.dd2, r.pe2), myrow);
    }
    tmem_wait_st();
    if constexpr (!kA0) fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      if (tid == 0) {
        tc_fence_after();
        const int K = l == 0 ? S::kK0 : S::kKh;
        const int N = l == NL - 1 ? S::kNLast : HID;
        const uint32_t wb = w_base + 2u * (uint32_t)S::w_off(l);
        const uint32_t sbo_b = (uint32_t)(K / 8) * 128u;
        if constexpr (S::kBiasCp) {
          // D := this layer's bias (zero 8-row-group stride: the tile's row on every lane)
          const uint32_t bt = smem_u32(smem) + (uint32_t)(S::kBcOff + S::b_off(l) * 32);
#pragma unroll
          for (int g = 0; g < (l == NL - 1 ? S::kNLast : HID) / 8; ++g)
            tmem_cp_128x256b(tmem + 8u * g, smem_desc(bt + 256u * g, 128u, 0u));
        }
        if (S::kSkip && l > 0) {
          // D_l = a_{l-1} x W_l (tf32, issued when layer l-1 completed, below)
          //     + cos(a_{l-1}) (fp16 smem tile) x (-2 W_l) + [1, 1] x [b_hi, b_lo]
          const uint32_t d = tmem + (uint32_t)((l & 1) * S::kTCols);
          const uint32_t id16 = idesc_f16(128, N);
#pragma unroll
          for (int kk = 0; kk < S::kKh / 16; ++kk)
            umma_f16(d, smem_desc(a_base + kk * 256u, 128u, S::kSboA),
                     smem_desc(wb + kk * 256u, 128u, sbo_b), id16, 1u);
          umma_commit(mb);
        } else if (kDbl && l > 0 && l < NL - 1) {
          const uint32_t id = idesc_f16(128, 32);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int kk = 0; kk < K / 16; ++kk)
              umma_f16_ts(tmem + 32u * h, tmem + S::kTCols + a_col(l) + kk * 8u,
                          smem_desc(wb + kk * 256u + 4u * h * sbo_b, 128u, sbo_b), id, 1u);
            umma_commit(h == 0 ? mb : mb1);
          }
        } else if (kNSplit && l < NL - 1 && ((FVSRN_TC_TMEM_A && l > 0) || kA0)) {
          // two N=32 halves: rows 32..63 of the K-major weight tile start 4 core-matrix
          // groups (4 * SBO) further on
          const uint32_t id = idesc_f16(128, 32);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int kk = 0; kk < K / 16; ++kk)
              umma_f16_ts(tmem + 32u * h, tmem + S::kTCols + kk * 8u,
                          smem_desc(wb + kk * 256u + 4u * h * sbo_b, 128u, sbo_b), id, 1u);
            umma_commit(h == 0 ? mb : mb1);
          }
        } else {
          const uint32_t id = idesc_f16(128, N);
#pragma unroll
          for (int kk = 0; kk < K / 16; ++kk) {
            // D preloaded with the bias accumulates from the first k step; bias-in-MMA starts D
            const uint32_t acc = (S::kBiasMma && kk == 0) ? 0u : 1u;
            if ((FVSRN_TC_TMEM_A && l > 0) || kA0)
              umma_f16_ts(tmem, tmem + S::kTCols + a_col(l) + kk * 8u, smem_desc(wb + kk * 256u, 128u, sbo_b), id, acc);
            else
              umma_f16(tmem, smem_desc(a_base + kk * 256u, 128u, S::kSboA),
                       smem_desc(wb + kk * 256u, 128u, sbo_b), id, acc);
          }
          umma_commit(mb);
        }
      }
      if (prefetch && l == NL - 1) {
        pre_k = -1;
        if (r.has && r.k + 1 < r.n) {
          const float kf = (float)(r.k + 1);
          FastRow<NM>::tex_words(fd, fmaf(kf, r.dd0, r.pe0), fmaf(kf, r.dd1, r.pe1), fmaf(kf, r.dd2, r.pe2), pre);
          pre_k = r.k + 1;
        }
      }
      if constexpr (FVSRN_TC_WAIT_BAR) {
        // one thread polls the MMA-completion barrier; the others wait in the hardware
        // CTA barrier instead of spinning on try_wait (issue slots stay with other CTAs)
        if (tid == 0) mbar_wait(mb, phase);
        tc_fence_before();
        __syncthreads();
      } else {
        mbar_wait(mb, phase);
      }
      phase ^= 1u;
      tc_fence_after();
      if (S::kSkip && l < NL - 1) {
        if (tid == 0) {
          // the a x W part of the next layer only needs this layer's accumulators: issue it
          // now, so the tensor core works under the cos evaluation below
          const int N1 = l + 1 == NL - 1 ? S::kNLast : HID;
          const uint32_t d = tmem + (uint32_t)(((l + 1) & 1) * S::kTCols);
          const uint32_t ax = tmem + (uint32_t)((l & 1) * S::kTCols);
          const uint32_t xb = w_base + (uint32_t)S::x_off(l + 1);
          const uint32_t id32 = idesc_tf32(128, N1);
#pragma unroll
          for (int kk = 0; kk < HID / 8; ++kk)
            umma_tf32_ts(d, ax + kk * 8u, smem_desc(xb + kk * 256u, 128u, S::kSboX), id32, kk > 0 ? 1u : 0u);
        }
        // cos(a) of this layer's accumulator region -> the shared-memory A tile
        uint32_t acc[HID];
        tmem_ld<HID>(t_row + (uint32_t)((l & 1) * S::kTCols), acc);
        tmem_wait_ld();
        cos_row<HID>(acc, myrow);
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
      } else if (l < NL - 1) {
        // snake_alt in the 2x-prescaled basis (act_h<4>), fp16 pairs -> A tile columns;
        // FVSRN_TC_SPLIT: read the row in 32-column halves (fewer live registers)
        if (kDbl && l > 0) {
          // first half ready (the wait above was on its mbarrier): bias + activations of
          // columns 0..31 while the tensor core computes columns 32..63
          const uint32_t an = t_row + S::kTCols + a_col(l + 1);
          uint32_t acc[32], w[16];
          tmem_ld<32>(t_row, acc);
          tmem_wait_ld();
          if (l + 1 < NL - 1) tmem_bias<32>(t_row, b_s + S::b_off(l + 1));
          else tmem_bias<S::kNLast>(t_row, b_s + S::b_off(l + 1));
          act_words<32>(acc, w);
          tmem_st<16>(an, w);
          mbar_wait(mb1, phase1);
          phase1 ^= 1u;
          tc_fence_after();
          tmem_ld<32>(t_row + 32, acc);
          tmem_wait_ld();
          if (l + 1 < NL - 1) tmem_bias<32>(t_row + 32, b_s + S::b_off(l + 1) + 32);
          act_words<32>(acc, w);
          tmem_st<16>(an + 16, w);
        } else if constexpr (kNSplit) {
          // first half ready (the wait above was on its mbarrier); its activations overlap
          // the second half's MMA and stay in registers until that MMA has read A
          uint32_t acc[32], w0[16], w1[16];
          tmem_ld<32>(t_row, acc);
          tmem_wait_ld();
          act_words<32>(acc, w0);
          mbar_wait(mb1, phase1);
          phase1 ^= 1u;
          tc_fence_after();
          tmem_ld<32>(t_row + 32, acc);
          tmem_wait_ld();
          if constexpr (!S::kBiasMma && !S::kBiasCp) {
            if (l + 1 < NL - 1) tmem_bias<HID>(t_row, b_s + S::b_off(l + 1));
            else tmem_bias<S::kNLast>(t_row, b_s + S::b_off(l + 1));
          }
          act_words<32>(acc, w1);
          tmem_st<16>(t_row + S::kTCols, w0);
          tmem_st<16>(t_row + S::kTCols + 16, w1);
        } else if constexpr (FVSRN_TC_TMEM_A && FVSRN_TC_SPLIT && HID == 64) {
          // two 32-column halves: half the live accumulator registers
          uint32_t acc[32], w[16];
          tmem_ld<32>(t_row, acc);
          tmem_wait_ld();
          act_words<32>(acc, w);
          tmem_st<16>(t_row + S::kTCols + a_col(l + 1), w);
          tmem_ld<32>(t_row + 32, acc);
          tmem_wait_ld();
          if constexpr (!S::kBiasMma && !S::kBiasCp) {
            if (l + 1 < NL - 1) tmem_bias<HID>(t_row, b_s + S::b_off(l + 1));
            else tmem_bias<S::kNLast>(t_row, b_s + S::b_off(l + 1));
          }
          act_words<32>(acc, w);
          tmem_st<16>(t_row + S::kTCols + a_col(l + 1) + 16, w);
        } else if constexpr (FVSRN_TC_TMEM_A) {
          uint32_t acc[HID];
          tmem_ld<HID>(t_row, acc);
          tmem_wait_ld();
          if constexpr (!S::kBiasMma && !S::kBiasCp) {
            if (l + 1 < NL - 1) tmem_bias<HID>(t_row, b_s + S::b_off(l + 1));
            else tmem_bias<S::kNLast>(t_row, b_s + S::b_off(l + 1));
          }
          uint32_t w[HID / 2];
          act_words<HID>(acc, w);
          tmem_st<HID / 2>(t_row + S::kTCols, w);
        } else if constexpr (FVSRN_TC_SPLIT && HID == 64) {
          uint32_t acc[32];
          tmem_ld<32>(t_row, acc);
          tmem_wait_ld();
          act_row<32>(acc, myrow);
          tmem_ld<32>(t_row + 32, acc);
          tmem_wait_ld();
          if constexpr (!S::kBiasMma && !S::kBiasCp) {
            if (l + 1 < NL - 1) tmem_bias<HID>(t_row, b_s + S::b_off(l + 1));
            else tmem_bias<S::kNLast>(t_row, b_s + S::b_off(l + 1));
          }
          act_row<32>(acc, myrow + 4 * 64);
        } else {
          uint32_t acc[HID];
          tmem_ld<HID>(t_row, acc);
          tmem_wait_ld();
          if constexpr (!S::kBiasMma && !S::kBiasCp) {
            if (l + 1 < NL - 1) tmem_bias<HID>(t_row, b_s + S::b_off(l + 1));
            else tmem_bias<S::kNLast>(t_row, b_s + S::b_off(l + 1));
          }
          act_row<HID>(acc, myrow);
        }
        if constexpr (S::kBiasMma) {
          if (l == 0) {   // the bias tile of layers >= 1: A columns HID/2.. = [1, 1, 0, ...]
            uint32_t c[8] = {0x3C003C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            tmem_st_x8(t_row + S::kTCols + HID / 2, c);
          }
        }
        tmem_wait_st();
        // the next A operand went to TMEM (tcgen05.st): no generic-proxy smem writes
        if constexpr (!FVSRN_TC_TMEM_A) fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
      } else {
        uint32_t o[4];
        tmem_ld_x4(t_row + (uint32_t)(S::kSkip ? ((NL - 1) & 1) * S::kTCols : 0), o);
        tmem_wait_ld();
        if (r.has)
          composite_step(r, make_float4(__uint_as_float(o[0]), __uint_as_float(o[1]),
                                        __uint_as_float(o[2]), __uint_as_float(o[3])),
                         kFrame || density, *tf, md, out, nonfinite);
      }
    }
  }
  if (lane == 0 && eval_count) atomicAdd(eval_count, evals);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kAlloc);
}

#if FVSRN_AB_VARIANTS   // measured slower, off by default
// Two-tile ping-pong variant: every thread owns two rays (tile 0 row t, tile 1 row t),
// with one A tile, one TMEM accumulator region and one mbarrier per tile.  While the
// tensor core runs layer l+1 of one tile, the CTA evaluates the activations (XU pipe)
// or composites / refills / builds the next rows (FMA/LSU pipes) of the other tile, so
// the MMA round trip and the CTA barriers overlap useful work.
template <int HID, int NM, int NL>
__global__ void __launch_bounds__(kTcThreads, tc2_min_blocks<HID>())
dvr_tc2_kernel(TcNetDev net, FeatDev fd, const TFDev* __restrict__ tf_g, const float* __restrict__ b0,
               MarchDev md, CamDev cam, ShardDev sh, int explicit_rays, RayRecs rr, long long n_slots,
               float* __restrict__ out, unsigned long long* __restrict__ queue,
               unsigned long long* __restrict__ eval_count, unsigned long long* __restrict__ nonfinite) {
  using S = TcShape<HID, NM, NL>;
  extern __shared__ __align__(128) unsigned char smem[];
  __half* w_s = reinterpret_cast<__half*>(smem + S::kWOff);
  float* b_s = reinterpret_cast<float*>(smem + S::kBOff);
  TFDev* tf = reinterpret_cast<TFDev*>(smem + S::kTFOff);
  __half* a_s0 = reinterpret_cast<__half*>(smem + S::kAOff);
  __half* a_s1 = reinterpret_cast<__half*>(smem + S::kAOff + S::kATile);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + S::kAOff + 2 * S::kATile);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::kAOff + 2 * S::kATile + 16);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    const uint4* src = net.w;
    uint4* dst = reinterpret_cast<uint4*>(w_s);
    for (int i = tid; i < S::kWTotal / 8; i += kTcThreads) dst[i] = src[i];
    for (int i = tid; i < S::kBTotal; i += kTcThreads)
      b_s[i] = (b0 && i < HID) ? b0[i] : net.b[i];
    const int words = sizeof(TFDev) / 4;
    const int* ts = reinterpret_cast<const int*>(tf_g);
    int* td = reinterpret_cast<int*>(tf);
    for (int i = tid; i < words; i += kTcThreads) td[i] = ts[i];
    uint4* az = reinterpret_cast<uint4*>(a_s0);   // pad columns must stay finite
    for (int i = tid; i < 2 * kTcThreads * S::kKA / 8; i += kTcThreads) az[i] = make_uint4(0, 0, 0, 0);
  }
  constexpr bool kA0 = FVSRN_TC_TMEM_A0 == 1 || (FVSRN_TC_TMEM_A0 == 2 && HID <= 32);
  // per tile: D [0, kTCols) then A (hidden activations, and layer-0 rows when kA0)
  constexpr uint32_t kTile = S::kTCols + (kA0 ? S::kKA / 2 : HID / 2);
  constexpr uint32_t kAlloc = 2 * kTile <= 64 ? 64 : 2 * kTile <= 128 ? 128 : 2 * kTile <= 256 ? 256 : 512;
  if (warp == 0) tmem_alloc(smem_u32(tmem_slot), kAlloc);
  if (tid == 0) { mbar_init(smem_u32(mbar), 1); mbar_init(smem_u32(mbar + 1), 1); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t w_base = smem_u32(w_s);
  const uint32_t a_base[2] = {smem_u32(a_s0), smem_u32(a_s1)};
  const uint32_t mb[2] = {smem_u32(mbar), smem_u32(mbar + 1)};
  const uint32_t t_d[2] = {tmem, tmem + kTile};                             // accumulator columns
  const uint32_t t_a[2] = {tmem + S::kTCols, tmem + kTile + S::kTCols};     // A operand columns
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;                     // this warp's lanes
  const int row_off = (tid >> 3) * (S::kSboA / 2) + (tid & 7) * 8;
  __half* myrow[2] = {a_s0 + row_off, a_s1 + row_off};
  const bool density = net.head == 0;

  RayLane r[2];
  r[0].has = false;
  r[1].has = false;
  LaneQueue q{0, 0, false};
  unsigned long long evals = 0;
  uint32_t phase[2] = {0u, 0u};
  bool live[2];

  auto issue = [&](int l, int t) {
    if (tid == 0) {
      tc_fence_after();
      const int K = l == 0 ? S::kK0 : HID;
      const int N = l == NL - 1 ? S::kNLast : HID;
      const uint32_t wb = w_base + 2u * (uint32_t)S::w_off(l);
      const uint32_t sbo_b = (uint32_t)(K / 8) * 128u;
      const uint32_t id = idesc_f16(128, N);
#pragma unroll
      for (int kk = 0; kk < K / 16; ++kk) {
        if (l > 0 || kA0)
          umma_f16_ts(t_d[t], t_a[t] + kk * 8u, smem_desc(wb + kk * 256u, 128u, sbo_b), id, 1u);
        else
          umma_f16(t_d[t], smem_desc(a_base[t] + kk * 256u, 128u, S::kSboA),
                   smem_desc(wb + kk * 256u, 128u, sbo_b), id, 1u);
      }
      umma_commit(mb[t]);
    }
  };
  // refill tile t, pre-load its layer-0 bias, write its rows; returns (CTA-wide) whether
  // the tile has any ray, after the fences + barrier that make the rows MMA-visible
  auto start = [&](int t) -> bool {
    ws_refill(r[t], q, lane, cam, sh, explicit_rays != 0, rr, n_slots, queue, md, out);
    evals += __popc(__ballot_sync(0xffffffffu, r[t].has));
    tmem_bias<HID>(t_d[t] + lane_off, b_s + S::b_off(0));
    if constexpr (kA0) {          // tcgen05.st is .sync.aligned: every lane stores
      uint32_t w[FastRow<NM>::kWords];
      if (r[t].has) {
        const float kf = (float)r[t].k;
        FastRow<NM>::words(fd, fmaf(kf, r[t].dd0, r[t].pe0), fmaf(kf, r[t].dd1, r[t].pe1),
                           fmaf(kf, r[t].dd2, r[t].pe2), w);
      } else {
#pragma unroll
        for (int i = 0; i < FastRow<NM>::kWords; ++i) w[i] = 0u;
      }
      tmem_st_any<FastRow<NM>::kWords>(t_a[t] + lane_off, w);
    } else if (r[t].has) {
      const float kf = (float)r[t].k;
      FastRow<NM>::template build<8>(fd, fmaf(kf, r[t].dd0, r[t].pe0), fmaf(kf, r[t].dd1, r[t].pe1),
                                     fmaf(kf, r[t].dd2, r[t].pe2), myrow[t]);
    }
    tmem_wait_st();
    if constexpr (!kA0) fence_proxy_async_smem();
    tc_fence_before();
    return __syncthreads_or(r[t].has) != 0;
  };

#pragma unroll
  for (int t = 0; t < 2; ++t) {
    live[t] = start(t);
    if (live[t]) issue(0, t);
  }
  while (live[0] || live[1]) {
#pragma unroll
    for (int l = 0; l < NL; ++l) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (!live[t]) continue;
        mbar_wait(mb[t], phase[t]);
        phase[t] ^= 1u;
        tc_fence_after();
        const uint32_t t_row = t_d[t] + lane_off;
        if (l < NL - 1) {
          uint32_t acc[HID];
          tmem_ld<HID>(t_row, acc);
          tmem_wait_ld();
          if (l + 1 < NL - 1) tmem_bias<HID>(t_row, b_s + S::b_off(l + 1));
          else tmem_bias<S::kNLast>(t_row, b_s + S::b_off(l + 1));
          uint32_t w[HID / 2];
          act_words<HID>(acc, w);
          tmem_st<HID / 2>(t_a[t] + lane_off, w);
          tmem_wait_st();
          tc_fence_before();
          __syncthreads();
          issue(l + 1, t);
        } else {
          uint32_t o[4];
          tmem_ld_x4(t_row, o);
          tmem_wait_ld();
          if (r[t].has)
            composite_step(r[t], make_float4(__uint_as_float(o[0]), __uint_as_float(o[1]),
                                             __uint_as_float(o[2]), __uint_as_float(o[3])),
                           density, *tf, md, out, nonfinite);
          live[t] = start(t);
          if (live[t]) issue(0, t);
        }
      }
    }
  }
  if (lane == 0 && eval_count) atomicAdd(eval_count, evals);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kAlloc);
}

#endif  // FVSRN_AB_VARIANTS

const void* tc_kernel_for(int hid, bool two_tiles) {
  switch (hid) {
#if FVSRN_AB_VARIANTS
    case 32: return two_tiles ? (const void*)dvr_tc2_kernel<32, 14, 4> : (const void*)dvr_tc_kernel<32, 14, 4>;
    case 64: return two_tiles ? (const void*)dvr_tc2_kernel<64, 30, 6> : (const void*)dvr_tc_kernel<64, 30, 6>;
#else
    case 32: return two_tiles ? nullptr : (const void*)dvr_tc_kernel<32, 14, 4>;
    case 64: return two_tiles ? nullptr : (const void*)dvr_tc_kernel<64, 30, 6>;
#endif
    default: return nullptr;
  }
}

const void* tc_tex_kernel_for(int hid, int fmode) {
  switch (hid) {
    case 32: return fmode == 2 ? (const void*)dvr_tc_kernel<32, 14, 4, 2> : (const void*)dvr_tc_kernel<32, 14, 4, 1>;
    case 64: return fmode == 2 ? (const void*)dvr_tc_kernel<64, 30, 6, 2> : (const void*)dvr_tc_kernel<64, 30, 6, 1>;
    default: return nullptr;
  }
}

size_t tc_smem_bytes(int hid, bool two_tiles) {
  switch (hid) {
    case 32: return two_tiles ? TcShape<32, 14, 4>::kSmem2 : TcShape<32, 14, 4>::kSmem;
    case 64: return two_tiles ? TcShape<64, 30, 6>::kSmem2 : TcShape<64, 30, 6>::kSmem;
    default: return 0;
  }
}

}  // namespace fvsrn
