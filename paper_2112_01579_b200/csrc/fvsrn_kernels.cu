// fvsrn_kernels.cu -- sm_100a kernels of the fV-SRN DVR hot path.
//
//   dvr_kernel        fused ray march: ray setup (f64, bit-exact geometry) -> per step
//                     {latent grid, Fourier, MLP on tensor cores, head, TF, compositing,
//                     early termination}; persistent warps refill lanes from a
//                     chunked global work queue so MMA tiles stay full.
//                     render.py:189-238, 314-332
//   decode_kernel     batched world-space density decode on the vertex lattice
//                     model.py:385-398
//   eval_kernel       per-sample density / colour at given positions  model.py:368-382
//   fused_eval_kernel head(mlp(x)) from assembled inputs              fused.py:281-301
//   blend_grid_kernel per-frame keyframe pre-blend (trilinear is linear) model.py:219-233
//   tiles_to_frame    reassembles gathered screen-tile shards (multi-GPU)
#include <cub/cub.cuh>

#include "fvsrn_kernels.cuh"
#include "fvsrn_geometry.cuh"

namespace fvsrn {

__device__ __forceinline__ void stage_setup(const NetDev& net, const float* b0, const TFDev* tf_in,
                                            int rs, uint2*& wf_s, float*& b_s, TFDev*& tf_s,
                                            __half*& stage, float*& ob) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* p = smem;
  wf_s = reinterpret_cast<uint2*>(p);
  p += ((size_t)net.w_total * sizeof(uint2) + 15) / 16 * 16;
  b_s = reinterpret_cast<float*>(p);
  p += ((size_t)net.b_total * sizeof(float) + 15) / 16 * 16;
  tf_s = reinterpret_cast<TFDev*>(p);
  if (tf_in) p += (sizeof(TFDev) + 15) / 16 * 16;
  const int warp = threadIdx.x >> 5;
  const size_t per_warp = (size_t)kWarp * rs * sizeof(__half) + kWarp * 4 * sizeof(float);
  stage = reinterpret_cast<__half*>(p + warp * per_warp);
  ob = reinterpret_cast<float*>(p + warp * per_warp + (size_t)kWarp * rs * sizeof(__half));

  for (int i = threadIdx.x; i < net.w_total; i += blockDim.x) wf_s[i] = net.wfrag[i];
  for (int i = threadIdx.x; i < net.b_total; i += blockDim.x) b_s[i] = net.bias[i];
  if (b0) {  // per-frame layer-0 bias (time folded), expanded to accumulator quads
    const int n0q = net.b_off[1] - net.b_off[0];
    for (int i = threadIdx.x; i < n0q; i += blockDim.x) {
      const int j = i >> 2;
      b_s[i] = b0[(j >> 2) * 8 + 2 * (j & 3) + (i & 1)];
    }
  }
  if (tf_in) {
    const int words = sizeof(TFDev) / 4;
    const int* src = reinterpret_cast<const int*>(tf_in);
    int* dst = reinterpret_cast<int*>(tf_s);
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
  }
  // zero the whole per-warp stage (pad columns must be finite: 0 * NaN = NaN)
  const int lane = threadIdx.x & 31;
  uint32_t* st = reinterpret_cast<uint32_t*>(stage);
  for (int i = lane; i < kWarp * rs / 2; i += kWarp) st[i] = 0u;
  __syncthreads();
}

// layer-0 k16 tiles of the specialised row (0: runtime)
template <int NM>
__host__ __device__ constexpr int fast_kt0() {
  if constexpr (NM > 0) return FastRow<NM>::kK0 / 16;
  else return 0;
}

// ---------------------------------------------------------------- DVR
// NM > 0 / NL > 0: specialised input row (FastRow<NM>) and compile-time layer count
template <int HID, int ACT, int NM, int NL>
__global__ void __launch_bounds__(kThreads, min_blocks<HID>())
dvr_kernel(NetDev net, FeatDev fd, const TFDev* __restrict__ tf_g, const float* __restrict__ b0,
           MarchDev md, CamDev cam, ShardDev sh, const double* __restrict__ rays_o,
           const double* __restrict__ rays_d, long long n_slots, float* __restrict__ out,
           unsigned long long* __restrict__ queue, unsigned long long* __restrict__ eval_count,
           unsigned long long* __restrict__ nonfinite) {
  const int rs = fd.k0 + 8;
  uint2* wf_s; float* b_s; TFDev* tf; __half* stage; float* ob;
  stage_setup(net, b0, tf_g, rs, wf_s, b_s, tf, stage, ob);
  const int lane = threadIdx.x & 31;
  const bool density = net.head == 0;
  const bool use_dir = fd.dir_mode != 0;
  const float eps1 = md.eps1_f;
  const float et = md.et_f;
  __half* myrow = stage + lane * rs;
  // two-point TFs (the presets' grayscale) live in registers: no per-sample smem lookups
  const bool tf_two = FVSRN_TF_REGS && density && tf->n == 2;
  float tf0[4], tfk[4], tfx0 = 0.f;
  if (tf_two) {
    tfx0 = tf->xs[0];
#pragma unroll
    for (int c = 0; c < 4; ++c) { tf0[c] = tf->val[0][c]; tfk[c] = tf->slope[0][c]; }
  }

  bool has = false;
  int k = 0, n = 0;
  long long oslot = 0;
  // per-ray march state: first sample position pe and step vector dd, both rounded
  // from the f64 geometry (render.py:224-225); p_k = pe + k * dd in f32
  float pe0 = 0.f, pe1 = 0.f, pe2 = 0.f, dd0 = 0.f, dd1 = 0.f, dd2 = 0.f;
  float dx = 0.f, dy = 0.f, dz = 0.f;
  float dsf = 0.f, C0 = 0.f, C1 = 0.f, C2 = 0.f, A = 0.f;
  unsigned long long evals = 0;
  long long chunk_base = 0;
  int chunk_left = 0;
  bool qdone = false;

  while (true) {
    // ---- refill free lanes from the warp's chunk of the global work queue
    while (true) {
      unsigned need = __ballot_sync(0xffffffffu, !has);
      if (need == 0) break;
      if (chunk_left == 0) {
        if (qdone) break;
        unsigned long long cb = 0;
        if (lane == 0) cb = atomicAdd(queue, 32ull);
        cb = __shfl_sync(0xffffffffu, cb, 0);
        if ((long long)cb >= n_slots) { qdone = true; break; }
        chunk_base = (long long)cb;
        chunk_left = (int)min(32ll, n_slots - (long long)cb);
      }
      const int rank = __popc(need & lanemask_lt());
      const int take = min(__popc(need), chunk_left);
      if (!has && rank < take) {
        const long long qs = chunk_base + rank;
        // queue position -> canonical slot (LPT order permutes whole tiles)
        const long long s = (!rays_o && sh.order) ? ((long long)sh.order[qs >> 6] << 6) | (qs & 63) : qs;
        RayGeom r;
        bool valid = true;
        long long dst;
        if (rays_o) {
          dst = s;
#pragma unroll
          for (int a = 0; a < 3; ++a) { r.o[a] = rays_o[3 * s + a]; r.d[a] = rays_d[3 * s + a]; }
        } else {
          const int pix = slot_pixel(cam, sh, s);
          dst = sh.compact ? s : pix;
          if (pix < 0) {
            valid = false;
            if (sh.compact) *reinterpret_cast<float4*>(out + 4 * dst) = make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            const int W = cam.W;
            camera_dir(cam, pix % W, pix / W, r.d);
#pragma unroll
            for (int a = 0; a < 3; ++a) r.o[a] = cam.eye[a];
          }
        }
        if (valid) {
          if (march_geometry(md, r)) {
            has = true;
            k = 0; n = r.n; oslot = dst;
            const double t0 = __dadd_rn(r.tmin, __dmul_rn(0.5, r.ds));
            pe0 = (float)__dadd_rn(r.o[0], __dmul_rn(t0, r.d[0]));
            pe1 = (float)__dadd_rn(r.o[1], __dmul_rn(t0, r.d[1]));
            pe2 = (float)__dadd_rn(r.o[2], __dmul_rn(t0, r.d[2]));
            dd0 = (float)__dmul_rn(r.ds, r.d[0]);
            dd1 = (float)__dmul_rn(r.ds, r.d[1]);
            dd2 = (float)__dmul_rn(r.ds, r.d[2]);
            dx = (float)r.d[0]; dy = (float)r.d[1]; dz = (float)r.d[2];
            dsf = (float)r.ds;
            C0 = C1 = C2 = A = 0.f;
          } else {
            *reinterpret_cast<float4*>(out + 4 * dst) = make_float4(md.bg[0], md.bg[1], md.bg[2], 0.f);
          }
        }
      }
      chunk_base += take;
      chunk_left -= take;
    }
    const unsigned act = __ballot_sync(0xffffffffu, has);
    if (act == 0) break;
    evals += __popc(act);

    // ---- sample position (render.py:224-225, f64) and input row
    if (has) {
      const float kf = (float)k;
      const float px = fmaf(kf, dd0, pe0), py = fmaf(kf, dd1, pe1), pz = fmaf(kf, dd2, pe2);
      assemble_row_t<NM>(fd, px, py, pz, use_dir ? dx : 0.f, use_dir ? dy : 0.f,
                         use_dir ? dz : 0.f, myrow);
    }
    __syncwarp();
    MLPDispatch<HID, ACT, NL, fast_kt0<NM>()>::eval32(stage, rs, net, wf_s, b_s, ob, lane);
    __syncwarp();

    // ---- head, TF, compositing, early termination (render.py:109-117, 226-232)
    if (has) {
      const float4 o = *reinterpret_cast<const float4*>(ob + 4 * lane);
      float r, g, b, sig;
      if (tf_two) {
        const float dx = fminf(fmaxf(sigmoidf_(o.x), 0.f), 1.f) - tfx0;
        r = fmaf(tfk[0], dx, tf0[0]); g = fmaf(tfk[1], dx, tf0[1]);
        b = fmaf(tfk[2], dx, tf0[2]); sig = fmaf(tfk[3], dx, tf0[3]);
      } else if (density) {
        tf_eval(*tf, sigmoidf_(o.x), r, g, b, sig);
      } else {
        r = sigmoidf_(o.x); g = sigmoidf_(o.y); b = sigmoidf_(o.z); sig = softplusf_(o.w);
      }
      float alpha = 1.f - __expf(-sig * dsf);
      alpha = fmaxf(fminf(alpha, eps1), 0.f);
      const float tr = (1.f - A) * alpha;
      C0 = fmaf(tr, r, C0); C1 = fmaf(tr, g, C1); C2 = fmaf(tr, b, C2);
      A += tr;
      ++k;
      if (k >= n || A > et) {
        const float om = 1.f - A;
        const float4 px4 = make_float4(fmaf(om, md.bg[0], C0), fmaf(om, md.bg[1], C1),
                                       fmaf(om, md.bg[2], C2), A);
        *reinterpret_cast<float4*>(out + 4 * oslot) = px4;
        // Image invariant (imaging.py:52-57) checked on the device: no host scan
        if (nonfinite && !(isfinite(px4.x) && isfinite(px4.y) && isfinite(px4.z) && isfinite(px4.w)))
          atomicAdd(nonfinite, 1ull);
        has = false;
      }
    }
  }
  if (lane == 0 && eval_count) atomicAdd(eval_count, evals);
}

// ---------------------------------------------------------------- LPT schedule
__global__ void tile_cost_kernel(CamDev cam, MarchDev md, ShardDev sh, long long n_slots,
                                 unsigned* __restrict__ cost, unsigned* __restrict__ iota) {
  for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < n_slots;
       s += (long long)gridDim.x * blockDim.x) {
    unsigned n = 0;
    const int pix = slot_pixel(cam, sh, s);
    if (pix >= 0) {
      RayGeom r;
      camera_dir(cam, pix % cam.W, pix / cam.W, r.d);
#pragma unroll
      for (int a = 0; a < 3; ++a) r.o[a] = cam.eye[a];
      if (march_geometry(md, r)) n = (unsigned)r.n + 4;   // + refill/setup overhead
    }
    // a warp covers 32 consecutive slots of one 64-slot tile
    unsigned sum = __reduce_add_sync(0xffffffffu, n);
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(cost + (s >> 6), sum);
      if ((s & 63) == 0) iota[s >> 6] = (unsigned)(s >> 6);
    }
  }
}

size_t tile_order_scratch_bytes(int n_local) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, (const unsigned*)nullptr,
                                            (unsigned*)nullptr, (const unsigned*)nullptr,
                                            (unsigned*)nullptr, n_local);
  return bytes;
}

cudaError_t launch_tile_order(const CamDev& cam, const MarchDev& md, const ShardDev& sh,
                              int n_local, unsigned* cost, unsigned* order, void* scratch,
                              size_t scratch_bytes, cudaStream_t s) {
  // cost[0:n] keys, cost[n:2n] sorted keys, order[0:n] values, order[n:2n] iota
  cudaError_t e = cudaMemsetAsync(cost, 0, sizeof(unsigned) * n_local, s);
  if (e != cudaSuccess) return e;
  const long long n_slots = (long long)n_local * 64;
  const int blocks = (int)std::min<long long>((n_slots + 255) / 256, 148 * 16);
  tile_cost_kernel<<<blocks, 256, 0, s>>>(cam, md, sh, n_slots, cost, order + n_local);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return cub::DeviceRadixSort::SortPairsDescending(scratch, scratch_bytes, cost, cost + n_local,
                                                   order + n_local, order, n_local, 0, 32, s);
}

// ---------------------------------------------------------------- decode / eval
// mode 0: lattice decode (model.py:385-398); mode 1: positions (+dirs) from memory
template <int HID, int ACT, int NM, int NL>
__global__ void __launch_bounds__(kThreads, min_blocks<HID, false>())
sample_kernel(NetDev net, FeatDev fd, const float* __restrict__ b0, int mode, int res, double step,
              long long begin, long long count, const double* __restrict__ pos,
              const double* __restrict__ dirs, float* __restrict__ out) {
  const int rs = fd.k0 + 8;
  uint2* wf_s; float* b_s; TFDev* tf; __half* stage; float* ob;
  stage_setup(net, b0, nullptr, rs, wf_s, b_s, tf, stage, ob);
  const int lane = threadIdx.x & 31;
  const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  __half* myrow = stage + lane * rs;
  const bool density = net.head == 0;
  for (long long c = gwarp; c * 32 < count; c += nwarps) {
    const long long i = c * 32 + lane;
    const bool valid = i < count;
    if (valid) {
      float px, py, pz, dx = 0.f, dy = 0.f, dz = 0.f;
      if (mode == 0) {
        const long long idx = begin + i;
        const long long r2 = (long long)res * res;
        const int ix = (int)(idx / r2), iy = (int)((idx / res) % res), iz = (int)(idx % res);
        // numpy linspace(0,1,res): i*step + 0.0, last sample exactly 1.0
        px = ix == res - 1 ? 1.f : (float)((double)ix * step);
        py = iy == res - 1 ? 1.f : (float)((double)iy * step);
        pz = iz == res - 1 ? 1.f : (float)((double)iz * step);
      } else {
        px = (float)pos[3 * i]; py = (float)pos[3 * i + 1]; pz = (float)pos[3 * i + 2];
        if (dirs) { dx = (float)dirs[3 * i]; dy = (float)dirs[3 * i + 1]; dz = (float)dirs[3 * i + 2]; }
      }
      assemble_row_t<NM>(fd, px, py, pz, dx, dy, dz, myrow);
    }
    __syncwarp();
    MLPDispatch<HID, ACT, NL, fast_kt0<NM>()>::eval32(stage, rs, net, wf_s, b_s, ob, lane);
    __syncwarp();
    if (valid) {
      const float4 o = *reinterpret_cast<const float4*>(ob + 4 * lane);
      if (density) {
        out[i] = sigmoidf_(o.x);
      } else {
        *reinterpret_cast<float4*>(out + 4 * i) =
            make_float4(sigmoidf_(o.x), sigmoidf_(o.y), sigmoidf_(o.z), softplusf_(o.w));
      }
    }
    __syncwarp();
  }
}

// head(mlp(x)) with x already assembled in the reference column order.
template <int HID, int ACT>
__global__ void __launch_bounds__(kThreads, min_blocks<HID, false>())
fused_eval_kernel(NetDev net, int d_in, int k0, const float* __restrict__ x, long long count,
                  float* __restrict__ out) {
  const int rs = k0 + 8;
  uint2* wf_s; float* b_s; TFDev* tf; __half* stage; float* ob;
  stage_setup(net, nullptr, nullptr, rs, wf_s, b_s, tf, stage, ob);
  const int lane = threadIdx.x & 31;
  const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  __half* myrow = stage + lane * rs;
  for (long long c = gwarp; c * 32 < count; c += nwarps) {
    const long long i = c * 32 + lane;
    const bool valid = i < count;
    if (valid)
      for (int j = 0; j < d_in; ++j) myrow[j] = __float2half_rn(x[i * d_in + j]);
    __syncwarp();
    MLPDispatch<HID, ACT>::eval32(stage, rs, net, wf_s, b_s, ob, lane);
    __syncwarp();
    if (valid) {
      const float4 o = *reinterpret_cast<const float4*>(ob + 4 * lane);
      if (net.head == 0) out[i] = sigmoidf_(o.x);
      else *reinterpret_cast<float4*>(out + 4 * i) =
          make_float4(sigmoidf_(o.x), sigmoidf_(o.y), sigmoidf_(o.z), softplusf_(o.w));
    }
    __syncwarp();
  }
}

__global__ void blend_grid_kernel(const __half* __restrict__ lo, const __half* __restrict__ hi,
                                  float w, long long n, __half* __restrict__ dst) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float a = __half2float(lo[i]), b = __half2float(hi[i]);
    dst[i] = __float2half_rn((1.f - w) * a + w * b);
  }
}

__global__ void tiles_to_frame_kernel(const float4* __restrict__ gathered, int W, int H, int world,
                                      long long per_rank, int tiles_x, int n_tiles,
                                      float4* __restrict__ frame) {
  const long long total = per_rank * world;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / per_rank);
    const long long s = i % per_rank;
    const long long tile = r + (s >> 6) * world;
    if (tile >= n_tiles) continue;
    const int e = (int)(s & 63);
    const int px = (int)(tile % tiles_x) * kTile + (e & 7), py = (int)(tile / tiles_x) * kTile + (e >> 3);
    if (px < W && py < H) frame[(long long)py * W + px] = gathered[i];
  }
}

// ---------------------------------------------------------------- launch table
#define FVSRN_FOR_HIDDEN(X) X(16) X(32) X(48) X(64) X(96) X(128)

// Default-config layer counts baked into the fast variants (fV-SRN 4x32 and 6x64).
constexpr int fast_layers(int hid) { return hid == 64 ? 6 : 4; }

// fast: (snake_alt, NeRF m = (HID-4)/2 on 3 axes, F = 16, pos mode, layers =
// fast_layers(HID)); else generic (runtime layer count and input layout)
const void* kernel_for(KernelKind kind, int hid, bool fast) {
  switch (hid) {
#define CASE(H)                                                                              \
  case H:                                                                                    \
    if (kind == KernelKind::kDVR)                                                            \
      return fast ? (const void*)dvr_kernel<H, 4, (H - 4) / 2, fast_layers(H)>               \
                  : (const void*)dvr_kernel<H, kActRuntime, 0, 0>;                           \
    if (kind == KernelKind::kSample)                                                         \
      return fast ? (const void*)sample_kernel<H, 4, (H - 4) / 2, fast_layers(H)>            \
                  : (const void*)sample_kernel<H, kActRuntime, 0, 0>;                        \
    return fast ? (const void*)fused_eval_kernel<H, 4> : (const void*)fused_eval_kernel<H, kActRuntime>;
    FVSRN_FOR_HIDDEN(CASE)
#undef CASE
    default: return nullptr;
  }
}

int fast_layer_count(int hid) { return fast_layers(hid); }

cudaError_t launch_blend(const __half* lo, const __half* hi, float w, long long n, __half* dst,
                         cudaStream_t s) {
  int blocks = (int)std::min<long long>((n + 255) / 256, 4096);
  blend_grid_kernel<<<blocks, 256, 0, s>>>(lo, hi, w, n, dst);
  return cudaGetLastError();
}

cudaError_t launch_tiles_to_frame(const float* gathered, int W, int H, int world, float* frame,
                                  cudaStream_t s) {
  const int tiles_x = (W + kTile - 1) / kTile, tiles_y = (H + kTile - 1) / kTile;
  const int n_tiles = tiles_x * tiles_y;
  const long long max_local = (n_tiles + world - 1) / world;
  const long long per_rank = max_local * 64;
  const long long total = per_rank * world;
  int blocks = (int)std::min<long long>((total + 255) / 256, 8192);
  tiles_to_frame_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(gathered), W, H,
                                               world, per_rank, tiles_x, n_tiles,
                                               reinterpret_cast<float4*>(frame));
  return cudaGetLastError();
}

}  // namespace fvsrn
