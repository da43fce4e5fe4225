// fvsrn_tc.cu -- tcgen05 / TMEM kernels of the fused fV-SRN evaluation (sm_100a): the DVR
// march (dvr_tc_kernel) and the lattice decode (decode_tc_kernel).
//
// One CTA = 4 warps = 128 rows = one M=128 UMMA tile.  Thread t owns row t (a ray, or a
// lattice point) and TMEM lane t, so the row-per-thread accumulator layout of tcgen05.ld
// is also the ray-per-thread layout of the marcher: no fragment shuffles, no output
// staging.  Per step (render.py:219-232 for the march):
//   1. every thread refills its ray / takes its lattice point and writes its input row
//      [z | sin/cos pairs | p | 1] (FastRow) into TMEM with tcgen05.st;
//   2. per layer (TcMlp::run): one elected thread issues K/16 tcgen05.mma (A = the row or
//      the hidden activations in TMEM, B = weights in shared memory, D = f32 accumulators
//      in TMEM) and commits to an mbarrier; every thread tcgen05.ld's its row, evaluates
//      the snake activation in registers (one MUFU.COS per element; every 3rd packed
//      fp16 pair on the FMA pipe in HFMA2 arithmetic) and tcgen05.st's the packed fp16
//      row back as the next A operand.  Biases:
//      at 32-wide inside the MMA (layer 0 through the row's 1.0 pad column and a W0 bias
//      column patched per frame, later layers through one extra k16 tile of [1, 1] x
//      [b_hi, b_lo]); at 64-wide preloaded into D with tcgen05.st;
//   3. the last layer's 4 outputs go straight to head/TF/compositing/ET (march) or to the
//      density store (decode) in registers.
// The MLP never touches global memory; the HMMA issue slots and the B-fragment LDS of
// the mma.sync kernel disappear from the SM sub-partitions' instruction streams.
// Used for the default fV-SRN configurations (FastRow inputs, snake_alt, 32/64 wide).
// The tcgen05 kernels are issue-bound with XU headroom (cfg 2: issue 74%, XU 63%), the
// mma.sync ones XU-bound: here the NeRF base angles go to MUFU.SIN/COS (3 issue slots per
// axis instead of 15 FMA-pipe operations): cfg 2 2.86 -> 2.82 ms, cfg 5 42.6 -> 41.6 ms
#ifndef FVSRN_FOURIER_POLY
#define FVSRN_FOURIER_POLY 0
#endif
// The per-layer MMA-completion wait polls without the hang watchdog (its counter and
// compare on every failed poll cost issue slots the other warps need: cfg 2 2.43 -> 2.36 ms,
// cfg 3 unchanged).  FVSRN_MBAR_WATCHDOG=1 restores the trap after ~2^26 polls for
// debugging a stuck MMA.
#ifndef FVSRN_MBAR_WATCHDOG
#define FVSRN_MBAR_WATCHDOG 0
#endif
// a 64 ns nanosleep between failed polls hands the issue slots to the epilogue warps
// (cfg 2 2.364 -> 2.347 ms over two A/B runs; 20/128/256 ns 2.356/2.348/2.353; cfg 3 and
// cfg 4 unchanged)
#ifndef FVSRN_MBAR_BACKOFF_NS
#define FVSRN_MBAR_BACKOFF_NS 64
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
// on the FMA pipe instead of the XU (MUFU) pipe (cfg 3: 28.2 -> 26.9 ms when introduced;
// round 2, cfg 2 / cfg 3 ms: every 4th 3.02 / 25.98, 5th 2.86 / 25.08, 6th 2.82 / 25.19,
// 7th 2.83, 8th - / 25.41, 12th 2.88).  0 disables.
#ifndef FVSRN_TC_POLY
#define FVSRN_TC_POLY 5     // 32-wide (at 8 CTAs/SM, cfg 2: every 4th/5th/6th/7th/8th 2.83/2.72/2.75/2.76/2.76 ms)
#endif
#ifndef FVSRN_TC_POLY64
#define FVSRN_TC_POLY64 6   // 64-wide, per 32-column half (4/5/6/7/8: 24.44/24.55/24.35/25.13/24.83 ms at cfg 3)
#endif
// narrowest width whose density head evaluates the last layer on the FMA pipe (64: cfg 3
// 24.04 -> 23.80 ms; at 32-wide it spills at 64 registers, 2.70 -> 2.77 ms)
#ifndef FVSRN_TC_LAST_LDS_PIN
#define FVSRN_TC_LAST_LDS_PIN 1   // cfg 3 23.80 -> 23.73 ms
#endif
#ifndef FVSRN_TC_DECODE_LAST_FMA_MINW
#define FVSRN_TC_DECODE_LAST_FMA_MINW 32   // the decode has registers to spare at 32-wide: cfg 4 0.546 -> 0.535 ms
#endif
#ifndef FVSRN_TC_LAST_FMA_MINW
#define FVSRN_TC_LAST_FMA_MINW 64
#endif
#ifndef FVSRN_TC_CHUNK64
#define FVSRN_TC_CHUNK64 16   // 64-wide epilogue chunk, 32 or 16 columns (16: 84 registers, cfg 3 24.34 -> 23.95 ms)
#endif
#ifndef FVSRN_TC_SPLIT32
#define FVSRN_TC_SPLIT32 1   // 32-wide epilogue in two 16-column halves (64 registers: 8 CTAs/SM)
#endif
#ifndef FVSRN_TC_BIAS_HALVES
#define FVSRN_TC_BIAS_HALVES 1
#endif
// Word-level replacement of FVSRN_TC_POLY (round 2, late): every FVSRN_TC_H2-th packed
// fp16 word (a pair of columns) of a hidden row evaluates both cosines on the FMA pipe in
// packed HFMA2 arithmetic (snake_alt_h2_fma: 10-11 instructions per PAIR, against 9 per
// element + a pack for the f32 polynomial); the other words use MUFU.  The kernels are
// issue-bound, so the cheaper FMA-pipe cosine lets a larger share leave the XU pipe.
// cfg 2 ms, word period 2/3/4/5: 2.644/2.497/2.54/2.603 (per-element f32 every 5th:
// 2.70); cfg 3 (64-wide, whole turns) period 3: 22.31 (half turns 2/3/4/5: 22.77/22.63/
// 22.59/23.23; f32 every 6th: 23.71); cfg 4 0.538 -> 0.505, cfg 5 38.65 -> 35.75.
// 0 = the per-element FVSRN_TC_POLY pattern.
#ifndef FVSRN_TC_H2
#define FVSRN_TC_H2 3
#endif
#ifndef FVSRN_TC_H2_64
#define FVSRN_TC_H2_64 3
#endif
// which word of each period (2: words 2, 5, 8, 11, 14 of a 16-word segment; phase 0, six
// words: cfg 2 2.383 vs 2.368 ms, cfg 3 21.35 vs 21.42 -- kept at 2)
#ifndef FVSRN_TC_H2_PHASE
#define FVSRN_TC_H2_PHASE 2
#endif
#ifndef FVSRN_TC_H2_FULL32
#define FVSRN_TC_H2_FULL32 0   // half turns + sign fix-up (smaller error, same speed)
#endif
#ifndef FVSRN_TC_H2_FULL64
#define FVSRN_TC_H2_FULL64 1   // whole turns (one instruction less per pair: 22.63 -> 22.31 ms)
#endif
template <int HID>
constexpr int tc_poly() { return HID <= 32 ? FVSRN_TC_POLY : FVSRN_TC_POLY64; }
template <int HID>
constexpr int tc_h2() { return HID <= 32 ? FVSRN_TC_H2 : FVSRN_TC_H2_64; }
template <int HID>
constexpr bool tc_h2_full() { return (HID <= 32 ? FVSRN_TC_H2_FULL32 : FVSRN_TC_H2_FULL64) != 0; }
#ifndef FVSRN_TC_DEADROW
#define FVSRN_TC_DEADROW 1
#endif
// MMA issue: weight-tile descriptors from one base word computed at init (no per-MMA
// descriptor math), and warp 0 converged with elect.sync instead of a tid == 0 branch, so
// ptxas issues each layer's UTCHMMAs + UTCBAR back to back without the per-instruction
// waterfall loop (ELECT / PLOP3 / BRA.U.ANY around every uniform-datapath op): the MMA
// starts sooner after the row barrier.  cfg 2 2.483 -> 2.456 (hoist) -> 2.435 ms (both),
// cfg 3 22.22 -> 21.41, cfg 5 35.42 -> 34.75, cfg 4 0.501 -> 0.498.
#ifndef FVSRN_TC_DESC_HOIST
#define FVSRN_TC_DESC_HOIST 1
#endif
#ifndef FVSRN_TC_ELECT
#define FVSRN_TC_ELECT 1
#endif
__device__ __forceinline__ uint32_t elect_one_sync() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n}" : "=r"(e));
  return e;
}
__device__ __forceinline__ void umma_f16_ts_if(uint32_t el, uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.ne.b32 q, %5, 0;\n\t"
      "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
      :: "r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(el) : "memory");
}
__device__ __forceinline__ void umma_commit_if(uint32_t el, uint32_t mbar) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t"
               "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}"
               :: "r"(mbar), "r"(el) : "memory");
}
#ifndef FVSRN_TC_DEADROW_MAXW
#define FVSRN_TC_DEADROW_MAXW 64   // widest layer that builds dummy rows (64: 24.69 -> 24.58 ms at cfg 3)
#endif

// snake_alt activations of N accumulator columns -> packed fp16 pairs (TMEM A operand);
// every P-th column's cosine on the FMA pipe
template <int N, int P = FVSRN_TC_POLY, int Q = 0, bool FULL = false>
__device__ __forceinline__ void act_words(const uint32_t (&acc)[N], uint32_t (&w)[N / 2]) {
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    if constexpr (Q > 0) {
      const float x0 = __uint_as_float(acc[2 * j]), x1 = __uint_as_float(acc[2 * j + 1]);
      w[j] = j % Q == FVSRN_TC_H2_PHASE % Q ? snake_alt_h2_fma<FULL>(x0, x1) : pack_half2(act_h<4>(x0), act_h<4>(x1));
      continue;
    }
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

// N accumulator columns that sit at column OFF of the FMA-pipe pattern (e % P == P - 1)
template <int N, int OFF, int P, int Q = 0, bool FULL = false>
__device__ __forceinline__ void act_words_at(const uint32_t (&acc)[N], uint32_t (&w)[N / 2]) {
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    if constexpr (Q > 0) {
      const float x0 = __uint_as_float(acc[2 * j]), x1 = __uint_as_float(acc[2 * j + 1]);
      const int g = OFF / 2 + j;
      w[j] = g % Q == FVSRN_TC_H2_PHASE % Q ? snake_alt_h2_fma<FULL>(x0, x1) : pack_half2(act_h<4>(x0), act_h<4>(x1));
      continue;
    }
    float h[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int e = OFF + 2 * j + i;
      const float x = __uint_as_float(acc[2 * j + i]);
      h[i] = (P > 0 && e % (P > 0 ? P : 1) == P - 1) ? snake_alt_h_fma(x) : act_h<4>(x);
    }
    w[j] = pack_half2(h[0], h[1]);
  }
}

// dot += sum over N accumulator columns (at column OFF of the FMA-pipe pattern) of
// snake_alt(a) x wl[OFF + e], f32 (the density head's last layer on the FMA pipe)
template <int N, int OFF, int P>
__device__ __forceinline__ float act_dot_at(const uint32_t (&acc)[N], const float* wl, float dot) {
#pragma unroll
  for (int j = 0; j < N; j += 4) {
    float wq[4];
#if FVSRN_TC_LAST_LDS_PIN
    // loaded where used (volatile: not hoisted above the TMEM loads, fewer live registers)
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(wq[0]), "=f"(wq[1]), "=f"(wq[2]), "=f"(wq[3]) : "r"(smem_u32(wl + OFF + j)));
#else
    {
      const float4 wv = *reinterpret_cast<const float4*>(wl + OFF + j);
      wq[0] = wv.x; wq[1] = wv.y; wq[2] = wv.z; wq[3] = wv.w;
    }
#endif
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = OFF + j + i;
      const float x = __uint_as_float(acc[j + i]);
      const float h = (P > 0 && e % (P > 0 ? P : 1) == P - 1) ? snake_alt_h_fma(x) : act_h<4>(x);
      dot = fmaf(wq[i], h, dot);
    }
  }
  return dot;
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

// Dynamic shared memory of the one-tile kernels (TcShape map); addressed through the
// symbol so shared-window offsets fold into immediates instead of live pointer registers
extern __shared__ __align__(128) unsigned char tc_smem[];

// The per-CTA tcgen05 MLP shared by the march and the decode kernels.  TMEM columns:
// D [0, kTCols), A [kTCols, kTCols + kKA/2) (the layer-0 row, then the hidden
// activations).  Shared memory (TcShape): weights, f32 biases, TF, mbarrier, TMEM slot.
template <int HID, int NM, int NL>
struct TcMlp {
  using S = TcShape<HID, NM, NL>;
  static_assert(S::kA0, "the one-tile kernels keep the layer-0 rows in TMEM");
  static constexpr int kWords = FastRow<NM>::kWords;
  // bias-in-MMA: the bias tile's constant A side [1, 1, 0, ...] (8 columns) sits after the
  // layer-0 row, written once; the bias k-step of every hidden layer reads it there
  static constexpr uint32_t kOnesCol = S::kKA / 2;
  static constexpr uint32_t kNeed = S::kTCols + S::kKA / 2 + (S::kBiasMma ? 8 : 0);
  static constexpr uint32_t kAlloc = kNeed <= 32 ? 32 : kNeed <= 64 ? 64 : kNeed <= 128 ? 128 : 256;

  uint32_t tmem, t_row, phase;
  int tid;
#if FVSRN_TC_DESC_HOIST
  uint32_t wdesc_lo;   // low descriptor word of the weight tiles' base (address field + LBO)
#endif

  __device__ static const float* b_s() { return reinterpret_cast<const float*>(tc_smem + S::kBOff); }
  __device__ static uint32_t mb() { return smem_u32(tc_smem + S::kMbarOff); }

  // Weights and biases (b0: this frame's layer-0 bias, or null) into shared memory, TMEM
  // allocation, mbarrier; ends with a CTA barrier (so caller-side shared-memory writes
  // issued before it are visible after it).
  __device__ void init(const TcNetDev& net, const float* __restrict__ b0) {
    tid = threadIdx.x;
    const int warp = tid >> 5;
    __half* w_s = reinterpret_cast<__half*>(tc_smem + S::kWOff);
    float* bs = reinterpret_cast<float*>(tc_smem + S::kBOff);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tc_smem + S::kMbarOff + 8);
    {
      const uint4* src = net.w;
      uint4* dst = reinterpret_cast<uint4*>(w_s);
      for (int i = tid; i < S::kWTotal / 8; i += kTcThreads) dst[i] = src[i];
      for (int i = tid; i < S::kBAll; i += kTcThreads) bs[i] = (b0 && i < HID) ? b0[i] : net.b[i];
    }
    // the weight tiles were written through the generic proxy and are read by the tensor
    // core (async proxy)
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(smem_u32(tmem_slot), kAlloc);
    if (tid == 0) mbar_init(mb(), 1);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if constexpr (S::kBias0) {
      // W0's pad column (K0 - 1; the row's pad is 1.0) := this frame's layer-0 bias
      constexpr int K = S::kK0, k = S::kK0 - 1;
      for (int n = tid; n < HID; n += kTcThreads)
        w_s[(n / 8) * (K / 8) * 64 + (k / 8) * 64 + (n % 8) * 8 + (k % 8)] = __float2half_rn(bs[n]);
      fence_proxy_async_smem();
      __syncthreads();
    }
    tmem = *tmem_slot;
    t_row = tmem + ((uint32_t)(warp * 32) << 16);   // this warp's TMEM lanes
#if FVSRN_TC_DESC_HOIST
    wdesc_lo = (uint32_t)smem_desc(smem_u32(tc_smem + S::kWOff), 128u, 0u);
#endif
    phase = 0;
    if constexpr (S::kBiasMma) {
      uint32_t c[8] = {0x3C003C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      tmem_st_x8(t_row + S::kTCols + kOnesCol, c);
      tmem_wait_st();   // ordered before the first MMA by put_row's barrier
    }
  }

  __device__ void finish() {
    tc_fence_before();
    __syncthreads();
    if ((tid >> 5) == 0) tmem_dealloc(tmem, kAlloc);
  }

  // Start of a step, before the row is built: the layer-0 bias into D (64-wide; its 64
  // registers are dead again before the row's are live)
  __device__ void begin_row() {
    if constexpr (!S::kBias0) tmem_bias<HID>(t_row, b_s() + S::b_off(0));
  }

  // This thread's layer-0 row (zeros for a thread without work) -> TMEM A; every thread
  // calls it (tcgen05.st is .sync.aligned).  Ends with the CTA barrier the MMA issue needs.
  __device__ void put_row(uint32_t (&w)[kWords]) {
    if constexpr (S::kBias0) w[kWords - 1] |= 0x3C000000u;   // pad column = 1.0
    tmem_st_any<kWords>(t_row + S::kTCols, w);
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
  }

  // All layers of this step; o = the last layer's first 4 accumulators of this row.
  // fma_last (a density head, CTA-uniform): the last layer's single used output is a dot
  // product of the f32 activations with its weight row on the FMA pipe (o[0]), instead of
  // an fp16 tcgen05 round trip (FVSRN_TC_LAST_FMA_MINW)
  template <int MINW = FVSRN_TC_LAST_FMA_MINW>
  __device__ void run(uint32_t (&o)[4], bool fma_last = false) {
    fma_last = fma_last && HID >= MINW;
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      if (fma_last && l == NL - 1) break;
#if FVSRN_TC_ELECT
      // warp 0 converged; elect.sync picks the issuing lane (no per-instruction waterfall
      // loop around the uniform-datapath MMA / commit)
      if (tid < 32) {
        const uint32_t el = elect_one_sync();
#else
      if (tid == 0) {
#endif
        tc_fence_after();
        const int K = l == 0 ? S::kK0 : S::kKh;
        const int N = l == NL - 1 ? S::kNLast : HID;
        const uint32_t wb = smem_u32(tc_smem + S::kWOff) + 2u * (uint32_t)S::w_off(l);
        const uint32_t sbo_b = (uint32_t)(K / 8) * 128u;
        const uint32_t id = idesc_f16(128, N);
#pragma unroll
        for (int kk = 0; kk < K / 16; ++kk) {
          // D preloaded with the bias accumulates from the first k step; bias-in-MMA starts D
          const uint32_t acc = (kk == 0 && (S::kBiasMma || (l == 0 && S::kBias0))) ? 0u : 1u;
          // the bias k-step of a hidden layer reads the constant ones columns
          const uint32_t a_col = (S::kBiasMma && l > 0 && kk == K / 16 - 1) ? kOnesCol : 8u * kk;
#if FVSRN_TC_DESC_HOIST
          // the address field advances by (byte offset >> 4): no carry out of its 14 bits
          // (shared-memory offsets < 2^18 B); the high word is a per-layer constant
          const uint64_t bd = ((uint64_t)(((uint32_t)(K / 8) * 128u >> 4) | (1u << 14)) << 32) |
                              (uint64_t)(wdesc_lo + ((2u * (uint32_t)S::w_off(l) + kk * 256u) >> 4));
          (void)wb;
#if FVSRN_TC_ELECT
          umma_f16_ts_if(el, tmem, tmem + S::kTCols + a_col, bd, id, acc);
#else
          umma_f16_ts(tmem, tmem + S::kTCols + a_col, bd, id, acc);
#endif
#else
          umma_f16_ts(tmem, tmem + S::kTCols + a_col, smem_desc(wb + kk * 256u, 128u, sbo_b), id, acc);
#endif
        }
#if FVSRN_TC_ELECT
        umma_commit_if(el, mb());
#else
        umma_commit(mb());
#endif
      }
      mbar_wait(mb(), phase);
      phase ^= 1u;
      tc_fence_after();
      if (fma_last && l == NL - 2) {
        const float* wl = b_s() + S::kWLast;
        float dot[HID / 16];
#pragma unroll
        for (int q = 0; q < HID / 16; ++q) {
          uint32_t acc[16];
          tmem_ld<16>(t_row + 16u * q, acc);
          tmem_wait_ld();
          // pattern column within the tc_poly period (restarting every 32 columns at 64-wide)
          if (HID == 64 ? (q & 1) : q == 1) dot[q] = act_dot_at<16, 16, tc_poly<HID>()>(acc, wl + 16 * (q & ~1), 0.f);
          else dot[q] = act_dot_at<16, 0, tc_poly<HID>()>(acc, wl + 16 * q, 0.f);
        }
        float d = b_s()[S::b_off(NL - 1)];
#pragma unroll
        for (int q = 0; q < HID / 16; ++q) d += dot[q];
        o[0] = __float_as_uint(d);
        o[1] = o[2] = o[3] = 0u;
      } else if (l < NL - 1) {
        // snake_alt in the 2x-prescaled basis (act_h<4>), fp16 pairs -> the next A operand
        if constexpr (HID == 64 && FVSRN_TC_CHUNK64 == 16 && !S::kBiasMma) {
          // four 16-column quarters; the next layer's bias stored per quarter right after
          // that quarter was read; the FMA-pipe pattern restarts every 32 columns
          uint32_t acc[16], w[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            tmem_ld<16>(t_row + 16u * q, acc);
            tmem_wait_ld();
            if (l + 1 < NL - 1) tmem_bias<16>(t_row + 16u * q, b_s() + S::b_off(l + 1) + 16 * q);
            else if (q == 0) tmem_bias<S::kNLast>(t_row, b_s() + S::b_off(l + 1));
            if (q & 1) act_words_at<16, 16, tc_poly<HID>(), tc_h2<HID>(), tc_h2_full<HID>()>(acc, w);
            else act_words_at<16, 0, tc_poly<HID>(), tc_h2<HID>(), tc_h2_full<HID>()>(acc, w);
            tmem_st_x8(t_row + S::kTCols + 8u * q, w);
          }
        } else if constexpr (HID == 64) {
          // two 32-column halves: half the live accumulator registers
          uint32_t acc[32], w[16];
          tmem_ld<32>(t_row, acc);
          tmem_wait_ld();
#if FVSRN_TC_BIAS_HALVES
          // the next layer's bias, one half at a time right after that half was read (32
          // bias registers live instead of 64)
          if constexpr (!S::kBiasMma) {
            if (l + 1 < NL - 1) tmem_bias<32>(t_row, b_s() + S::b_off(l + 1));
            else tmem_bias<S::kNLast>(t_row, b_s() + S::b_off(l + 1));
          }
#endif
          act_words<32, tc_poly<HID>(), tc_h2<HID>(), tc_h2_full<HID>()>(acc, w);
          tmem_st<16>(t_row + S::kTCols, w);
          tmem_ld<32>(t_row + 32, acc);
          tmem_wait_ld();
          if constexpr (!S::kBiasMma) {
#if FVSRN_TC_BIAS_HALVES
            if (l + 1 < NL - 1) tmem_bias<32>(t_row + 32, b_s() + S::b_off(l + 1) + 32);
#else
            if (l + 1 < NL - 1) tmem_bias<HID>(t_row, b_s() + S::b_off(l + 1));
            else tmem_bias<S::kNLast>(t_row, b_s() + S::b_off(l + 1));
#endif
          }
          act_words<32, tc_poly<HID>(), tc_h2<HID>(), tc_h2_full<HID>()>(acc, w);
          tmem_st<16>(t_row + S::kTCols + 16, w);
        } else if constexpr (FVSRN_TC_SPLIT32 && HID == 32 && S::kBiasMma) {
          // two 16-column halves (fewer live accumulator registers)
          uint32_t acc[16], w[8];
          tmem_ld<16>(t_row, acc);
          tmem_wait_ld();
          act_words<16, tc_poly<HID>(), tc_h2<HID>(), tc_h2_full<HID>()>(acc, w);
          tmem_st_x8(t_row + S::kTCols, w);
          tmem_ld<16>(t_row + 16, acc);
          tmem_wait_ld();
          act_words_at<16, 16, tc_poly<HID>(), tc_h2<HID>(), tc_h2_full<HID>()>(acc, w);
          tmem_st_x8(t_row + S::kTCols + 8, w);
        } else {
          uint32_t acc[HID];
          tmem_ld<HID>(t_row, acc);
          tmem_wait_ld();
          if constexpr (!S::kBiasMma) {
            if (l + 1 < NL - 1) tmem_bias<HID>(t_row, b_s() + S::b_off(l + 1));
            else tmem_bias<S::kNLast>(t_row, b_s() + S::b_off(l + 1));
          }
          uint32_t w[HID / 2];
          act_words<HID, tc_poly<HID>(), tc_h2<HID>(), tc_h2_full<HID>()>(acc, w);
          tmem_st<HID / 2>(t_row + S::kTCols, w);
        }
        tmem_wait_st();   // the next A operand went to TMEM: no shared-memory proxy fence
        tc_fence_before();
        __syncthreads();
      } else {
        tmem_ld_x4(t_row, o);
        tmem_wait_ld();
      }
    }
  }
};

}  // namespace

// TEX == 0: any frame or explicit rays; TEX == 1 / 2: a camera frame of a density-head
// model with a static fp16 texture grid / exact-weight LDG grid (compile-time flags)
template <int HID, int NM, int NL, int TEX = 0>
__global__ void __launch_bounds__(kTcThreads, tc_min_blocks<HID>())
dvr_tc_kernel(TcNetDev net, FeatDev fd, const TFDev* __restrict__ tf_g, const float* __restrict__ b0,
              MarchDev md, CamDev cam, ShardDev sh, int explicit_rays, RayRecs rr, long long n_slots,
              float* __restrict__ out, unsigned long long* __restrict__ queue,
              unsigned long long* __restrict__ eval_count, unsigned long long* __restrict__ nonfinite) {
  using S = TcShape<HID, NM, NL>;
  TFDev* tf = reinterpret_cast<TFDev*>(tc_smem + S::kTFOff);
  {
    const int words = sizeof(TFDev) / 4;
    const int* ts = reinterpret_cast<const int*>(tf_g);
    int* td = reinterpret_cast<int*>(tf);
    for (int i = threadIdx.x; i < words; i += kTcThreads) td[i] = ts[i];
  }
  TcMlp<HID, NM, NL> mlp;
  mlp.init(net, b0);
  const int lane = threadIdx.x & 31;
  const bool density = net.head == 0;
  constexpr bool kFrame = TEX >= 1;

  RayLane r{};   // zero state: a lane without a ray builds a finite dummy row
  r.has = false;
  LaneQueue q{0, 0, false};
  unsigned evals = 0;   // this thread's evaluations (reduced over the warp at the end)
  while (true) {
    if constexpr (kFrame) {
      RayRecs rr_pos = rr;
      rr_pos.d = nullptr;
      ws_refill(r, q, lane, cam, sh, false, rr_pos, n_slots, queue, md, out);
    } else {
      ws_refill(r, q, lane, cam, sh, explicit_rays != 0, rr, n_slots, queue, md, out);
    }
    if (!__syncthreads_or(r.has)) break;
    evals += r.has ? 1u : 0u;
    mlp.begin_row();
    uint32_t w[FastRow<NM>::kWords];
    // FVSRN_TC_DEADROW: lanes without a ray build a row from their stale (finite) ray
    // state instead of branching around the feature code and zeroing the row; the row is
    // independent of the others in the MMA and its result is dropped
    if ((FVSRN_TC_DEADROW && HID <= FVSRN_TC_DEADROW_MAXW) || r.has) {
      const float kf = (float)r.k;
      const float px = fmaf(kf, r.dd0, r.pe0), py = fmaf(kf, r.dd1, r.pe1), pz = fmaf(kf, r.dd2, r.pe2);
      if constexpr (TEX >= 1) {   // static fp16 grid: no runtime branches
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
    mlp.put_row(w);
    uint32_t o[4];
    mlp.run(o, kFrame || density);
    if (r.has)
      composite_step(r, make_float4(__uint_as_float(o[0]), __uint_as_float(o[1]),
                                    __uint_as_float(o[2]), __uint_as_float(o[3])),
                     kFrame || density, *tf, md, out, nonfinite);
  }
  evals = __reduce_add_sync(0xffffffffu, evals);
  if (lane == 0 && eval_count) atomicAdd(eval_count, (unsigned long long)evals);
  mlp.finish();
}

// Density at the res^3 lattice (model.py:385-398, decode_volume; sample_kernel mode 0
// with the same linspace coordinate table), indices [begin, begin + count) in x-major
// order, for a static fp16 grid (TEX 1 texture units, 2 exact-weight LDG).  Persistent
// CTAs stride over 128-point tiles; the lattice coordinates advance with carries (no
// per-step 64-bit division).  ScalarVolume invariant checked on the device (bad).
template <int HID, int NM, int NL, int TEX>
__global__ void __launch_bounds__(kTcThreads, tc_min_blocks<HID>())
decode_tc_kernel(TcNetDev net, FeatDev fd, const float* __restrict__ b0, int res, long long begin,
                 long long count, const float* __restrict__ coords, float* __restrict__ out,
                 unsigned long long* __restrict__ bad) {
  TcMlp<HID, NM, NL> mlp;
  mlp.init(net, b0);
  const int tid = threadIdx.x;
  const long long r2 = (long long)res * res;
  const long long S = (long long)gridDim.x * kTcThreads;
  const long long g0 = begin + (long long)blockIdx.x * kTcThreads + tid;
  int ix = (int)(g0 / r2), iy = (int)((g0 / res) % res), iz = (int)(g0 % res);
  const int sx = (int)(S / r2), sy = (int)((S / res) % res), sz = (int)(S % res);
  for (long long base = (long long)blockIdx.x * kTcThreads; base < count; base += S) {   // CTA-uniform
    const long long i = base + tid;
    const bool valid = i < count;
    mlp.begin_row();
    uint32_t w[FastRow<NM>::kWords];
    if (valid) {
      const float px = __ldg(coords + ix), py = __ldg(coords + iy), pz = __ldg(coords + iz);
      uint32_t z[8];
      if constexpr (TEX == 1) FastRow<NM>::tex_words(fd, px, py, pz, z);
      else FastRow<NM>::ldg_words(fd, px, py, pz, z);
      FastRow<NM>::words_from_z(z, px, py, pz, w);
    } else {
#pragma unroll
      for (int j = 0; j < FastRow<NM>::kWords; ++j) w[j] = 0u;
    }
    // idx += S
    iz += sz;
    int carry = iz >= res;
    iz -= carry ? res : 0;
    iy += sy + carry;
    carry = iy >= res;
    iy -= carry ? res : 0;
    ix += sx + carry;
    mlp.put_row(w);
    uint32_t o[4];
    mlp.template run<FVSRN_TC_DECODE_LAST_FMA_MINW>(o, true);
    if (valid) {
      const float v = sigmoidf_(__uint_as_float(o[0]));
      out[i] = v;
      // ScalarVolume invariant (volume.py:41-49) checked on the device: finite, in [0,1]
      if (bad && !(v >= 0.f && v <= 1.f)) atomicAdd(bad, 1ull);
    }
  }
  mlp.finish();
}

// (The two-tile ping-pong variant, dvr_tc2_kernel, was measured slower at both widths and
// removed once the kernels moved to the shared TcMlp engine.)

const void* tc_kernel_for(int hid) {
  switch (hid) {
    case 32: return (const void*)dvr_tc_kernel<32, 14, 4>;
    case 64: return (const void*)dvr_tc_kernel<64, 30, 6>;
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

const void* tc_decode_kernel_for(int hid, int fmode) {
  switch (hid) {
    case 32: return fmode == 2 ? (const void*)decode_tc_kernel<32, 14, 4, 2> : (const void*)decode_tc_kernel<32, 14, 4, 1>;
    case 64: return fmode == 2 ? (const void*)decode_tc_kernel<64, 30, 6, 2> : (const void*)decode_tc_kernel<64, 30, 6, 1>;
    default: return nullptr;
  }
}

size_t tc_smem_bytes(int hid) {
  switch (hid) {
    case 32: return TcShape<32, 14, 4>::kSmem;
    case 64: return TcShape<64, 30, 6>::kSmem;
    default: return 0;
  }
}

}  // namespace fvsrn
