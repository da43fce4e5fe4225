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

}  // namespace

template <int HID, int NM, int NL>
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
    uint4* az = reinterpret_cast<uint4*>(a_s);   // pad columns must stay finite
    for (int i = tid; i < kTcThreads * S::kKA / 8; i += kTcThreads) az[i] = make_uint4(0, 0, 0, 0);
  }
  if (warp == 0) tmem_alloc(smem_u32(tmem_slot), S::kTCols);
  if (tid == 0) mbar_init(smem_u32(mbar), 1);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);   // this warp's TMEM lanes
  const uint32_t a_base = smem_u32(a_s), w_base = smem_u32(w_s), mb = smem_u32(mbar);
  // row tid of the A tile: 8-row group stride SBO_A, row-in-group stride 16 B
  __half* myrow = a_s + (tid >> 3) * (S::kSboA / 2) + (tid & 7) * 8;
  const bool density = net.head == 0;

  RayLane r;
  r.has = false;
  LaneQueue q{0, 0, false};
  unsigned long long evals = 0;
  uint32_t phase = 0;

  while (true) {
    ws_refill(r, q, lane, cam, sh, explicit_rays != 0, rr, n_slots, queue);
    if (!__syncthreads_or(r.has)) break;
    evals += __popc(__ballot_sync(0xffffffffu, r.has));
    tmem_bias<HID>(t_row, b_s + S::b_off(0));
    if (r.has) {
      const float kf = (float)r.k;
      FastRow<NM>::template build<8>(fd, fmaf(kf, r.dd0, r.pe0), fmaf(kf, r.dd1, r.pe1),
                                     fmaf(kf, r.dd2, r.pe2), myrow);
    }
    tmem_wait_st();
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      if (tid == 0) {
        tc_fence_after();
        const int K = l == 0 ? S::kK0 : HID;
        const int N = l == NL - 1 ? S::kNLast : HID;
        const uint32_t wb = w_base + 2u * (uint32_t)S::w_off(l);
        const uint32_t sbo_b = (uint32_t)(K / 8) * 128u;
        const uint32_t id = idesc_f16(128, N);
#pragma unroll
        for (int kk = 0; kk < K / 16; ++kk)
          umma_f16(tmem, smem_desc(a_base + kk * 256u, 128u, S::kSboA), smem_desc(wb + kk * 256u, 128u, sbo_b),
                   id, 1u);
        umma_commit(mb);
      }
      mbar_wait(mb, phase);
      phase ^= 1u;
      tc_fence_after();
      if (l < NL - 1) {
        uint32_t acc[HID];
        tmem_ld<HID>(t_row, acc);
        tmem_wait_ld();
        if (l + 1 < NL - 1) tmem_bias<HID>(t_row, b_s + S::b_off(l + 1));
        else tmem_bias<S::kNLast>(t_row, b_s + S::b_off(l + 1));
        // snake_alt in the 2x-prescaled basis (act_h<4>), fp16 pairs -> A tile columns
#pragma unroll
        for (int c = 0; c < HID / 8; ++c) {
          uint32_t w4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            w4[j] = pack_half2(act_h<4>(__uint_as_float(acc[8 * c + 2 * j])),
                               act_h<4>(__uint_as_float(acc[8 * c + 2 * j + 1])));
          *reinterpret_cast<uint4*>(myrow + c * 64) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
        tmem_wait_st();
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
      } else {
        uint32_t o[4];
        tmem_ld_x4(t_row, o);
        tmem_wait_ld();
        if (r.has)
          composite_step(r, make_float4(__uint_as_float(o[0]), __uint_as_float(o[1]),
                                        __uint_as_float(o[2]), __uint_as_float(o[3])),
                         density, *tf, md, out, nonfinite);
      }
    }
  }
  if (lane == 0 && eval_count) atomicAdd(eval_count, evals);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, S::kTCols);
}

const void* tc_kernel_for(int hid) {
  switch (hid) {
    case 32: return (const void*)dvr_tc_kernel<32, 14, 4>;
    case 64: return (const void*)dvr_tc_kernel<64, 30, 6>;
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
