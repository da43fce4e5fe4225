// fvsrn_volume.cu -- ground-truth DVR of a dense scalar volume (VolumeSource).
//
// Same ray setup, TF, compositing and early termination as the fV-SRN renderer, with
// the network replaced by the reference's trilinear volume lookup (volume.py:213-255):
// f64 sample positions and cell coordinates, f32 fractions and the lerp order
// x -> y -> z with explicit _rn operations, so every sampled density is bit-identical
// to sample_volume.  Used by evaluate_views-style model-vs-ground-truth comparisons
// and decode-then-render cross-checks (tests/test_render.py:236-243 of the reference).
#include "fvsrn_geometry.cuh"
#include "fvsrn_volume.cuh"

namespace fvsrn {

__device__ __forceinline__ float lerp_rn(float a, float b, float f) {
  // numpy: a * (1 - f) + b * f, three separately rounded f32 ops
  return __fadd_rn(__fmul_rn(a, __fsub_rn(1.f, f)), __fmul_rn(b, f));
}

__device__ __forceinline__ float sample_volume_dev(const VolDev& v, double px, double py, double pz) {
  const double p[3] = {px, py, pz};
  const int dims[3] = {v.X, v.Y, v.Z};
  int i0[3];
  float f[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double c = __dmul_rn(fmin(fmax(p[a], 0.0), 1.0), (double)(dims[a] - 1));
    int i = min((int)c, dims[a] - 2);
    i = max(i, 0);
    i0[a] = i;
    f[a] = (float)__dsub_rn(c, (double)i);
  }
  const long long sx = (long long)v.Y * v.Z, sy = v.Z;
  const float* b = v.v + i0[0] * sx + i0[1] * sy + i0[2];
  const float c000 = __ldg(b), c100 = __ldg(b + sx), c010 = __ldg(b + sy), c110 = __ldg(b + sx + sy);
  const float c001 = __ldg(b + 1), c101 = __ldg(b + sx + 1), c011 = __ldg(b + sy + 1),
              c111 = __ldg(b + sx + sy + 1);
  const float c00 = lerp_rn(c000, c100, f[0]), c10 = lerp_rn(c010, c110, f[0]);
  const float c01 = lerp_rn(c001, c101, f[0]), c11 = lerp_rn(c011, c111, f[0]);
  const float c0 = lerp_rn(c00, c10, f[1]), c1 = lerp_rn(c01, c11, f[1]);
  return lerp_rn(c0, c1, f[2]);
}

// One warp takes 32 consecutive work slots (an 8x4 pixel block: similar ray lengths) at
// a time from the global queue; every lane marches its own ray.
__global__ void __launch_bounds__(256)
volume_dvr_kernel(VolDev vol, const TFDev* __restrict__ tf_g, MarchDev md, CamDev cam, ShardDev sh,
                  const double* __restrict__ rays_o, const double* __restrict__ rays_d,
                  long long n_slots, float* __restrict__ out, unsigned long long* __restrict__ queue,
                  unsigned long long* __restrict__ sample_count,
                  unsigned long long* __restrict__ nonfinite) {
  __shared__ TFDev tf;
  {
    const int words = sizeof(TFDev) / 4;
    const int* src = reinterpret_cast<const int*>(tf_g);
    int* dst = reinterpret_cast<int*>(&tf);
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const float eps1 = (float)(1.0 - md.eps_blend);
  const float et = (float)md.et_alpha;
  unsigned long long samples = 0;
  while (true) {
    unsigned long long cb = 0;
    if (lane == 0) cb = atomicAdd(queue, 32ull);
    cb = __shfl_sync(0xffffffffu, cb, 0);
    if ((long long)cb >= n_slots) break;
    const long long qs = (long long)cb + lane;
    if (qs >= n_slots) continue;
    const long long s = (!rays_o && sh.order) ? ((long long)sh.order[qs >> 6] << 6) | (qs & 63) : qs;
    RayGeom r;
    long long dst;
    if (rays_o) {
      dst = s;
#pragma unroll
      for (int a = 0; a < 3; ++a) { r.o[a] = rays_o[3 * s + a]; r.d[a] = rays_d[3 * s + a]; }
    } else {
      const int pix = slot_pixel(cam, sh, s);
      dst = sh.compact ? s : pix;
      if (pix < 0) {
        if (sh.compact) *reinterpret_cast<float4*>(out + 4 * dst) = make_float4(0.f, 0.f, 0.f, 0.f);
        continue;
      }
      camera_dir(cam, pix % cam.W, pix / cam.W, r.d);
#pragma unroll
      for (int a = 0; a < 3; ++a) r.o[a] = cam.eye[a];
    }
    float C0 = 0.f, C1 = 0.f, C2 = 0.f, A = 0.f;
    if (march_geometry(md, r)) {
      const float dsf = (float)r.ds;
      for (int k = 0; k < r.n; ++k) {
        const double tk = __dadd_rn(r.tmin, __dmul_rn((double)k + 0.5, r.ds));   // render.py:224
        const float dens = sample_volume_dev(vol, __dadd_rn(r.o[0], __dmul_rn(tk, r.d[0])),
                                             __dadd_rn(r.o[1], __dmul_rn(tk, r.d[1])),
                                             __dadd_rn(r.o[2], __dmul_rn(tk, r.d[2])));
        ++samples;
        float cr, cg, cbl, sig;
        tf_eval(tf, dens, cr, cg, cbl, sig);
        float alpha = 1.f - __expf(-sig * dsf);
        alpha = fmaxf(fminf(alpha, eps1), 0.f);
        const float tr = (1.f - A) * alpha;
        C0 = fmaf(tr, cr, C0); C1 = fmaf(tr, cg, C1); C2 = fmaf(tr, cbl, C2);
        A += tr;
        if (A > et) break;
      }
    }
    const float om = 1.f - A;
    const float4 px4 = make_float4(fmaf(om, md.bg[0], C0), fmaf(om, md.bg[1], C1),
                                   fmaf(om, md.bg[2], C2), A);
    *reinterpret_cast<float4*>(out + 4 * dst) = px4;
    if (nonfinite && !(isfinite(px4.x) && isfinite(px4.y) && isfinite(px4.z) && isfinite(px4.w)))
      atomicAdd(nonfinite, 1ull);
  }
  // per-warp sample total
  samples = __reduce_add_sync(0xffffffffu, (unsigned)samples);
  if (lane == 0 && sample_count) atomicAdd(sample_count, samples);
}

cudaError_t launch_volume_dvr(const VolDev& vol, const TFDev* tf, const MarchDev& md,
                              const CamDev& cam, const ShardDev& sh, const double* ro,
                              const double* rd, long long n_slots, float* out,
                              unsigned long long* counters, int num_sms, cudaStream_t s) {
  // counters: [0] queue, [1] samples, [2] non-finite pixels
  long long blocks = (long long)num_sms * 8;
  const long long need = (n_slots + 255) / 256;
  if (need < blocks) blocks = std::max(1ll, need);
  volume_dvr_kernel<<<(unsigned)blocks, 256, 0, s>>>(vol, tf, md, cam, sh, ro, rd, n_slots, out,
                                                     counters, counters + 1, counters + 2);
  return cudaGetLastError();
}

}  // namespace fvsrn
