// fvsrn_march.cuh -- per-lane ray state, the chunked work queue refill and the
// compositing step shared by the warp-specialised and tcgen05 DVR kernels.
//   geometry / march state   render.py:189-200, 203-238
//   compositing + ET          render.py:109-117, 226-232
#pragma once
#include "fvsrn_geometry.cuh"
#include "fvsrn_kernels.cuh"

namespace fvsrn {

struct RayLane {
  bool has;
  int k, n;
  long long oslot;
  float pe0, pe1, pe2, dd0, dd1, dd2, dx, dy, dz, dsf, C0, C1, C2, A;
};

struct LaneQueue {
  long long chunk_base;
  int chunk_left;
  bool qdone;
};

__device__ __forceinline__ void named_bar_sync(unsigned id, unsigned count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Per-slot ray records written once per frame by ray_setup_kernel (the f64 ray setup of
// render.py:72-106, 189-200 and the first-sample position / step vector of :224-225,
// rounded to f32), so the march loop never runs f64 code:
//   a[s] = (pe.x, pe.y, pe.z, n as int bits)   n = 0: no march (pixel already written)
//   b[s] = (dd.x, dd.y, dd.z, ds)              d[s] = (dir.x, dir.y, dir.z, 0) if dirs

// Refill free lanes of one ray group from the warp's chunk of the global queue.
__device__ __forceinline__ void ws_refill(RayLane& r, LaneQueue& q, int lane, const CamDev& cam,
                                          const ShardDev& sh, bool explicit_rays, const RayRecs& rr,
                                          long long n_slots, unsigned long long* __restrict__ queue,
                                          const MarchDev& md, float* __restrict__ out) {
  while (true) {
    unsigned need = __ballot_sync(0xffffffffu, !r.has);
    if (need == 0) break;
    if (q.chunk_left == 0) {
      if (q.qdone) break;
      unsigned long long cb = 0;
      if (lane == 0) cb = atomicAdd(queue, 32ull);
      cb = __shfl_sync(0xffffffffu, cb, 0);
      if ((long long)cb >= n_slots) { q.qdone = true; break; }
      q.chunk_base = (long long)cb;
      q.chunk_left = (int)min(32ll, n_slots - (long long)cb);
    }
    const int rank = __popc(need & lanemask_lt());
    const int take = min(__popc(need), q.chunk_left);
    if (!r.has && rank < take) {
      const long long qs = q.chunk_base + rank;
      // queue position -> canonical slot (LPT order permutes whole 64-slot tiles)
      const long long s = (!explicit_rays && sh.order) ? ((long long)sh.order[qs >> 6] << 6) | (qs & 63) : qs;
      const float4 ra = __ldg(rr.a + s);
      const int n = __float_as_int(ra.w);
      if (n > 0) {
        const float4 rb = __ldg(rr.b + s);
        r.has = true;
        r.k = 0; r.n = n;
        r.oslot = (explicit_rays || sh.compact) ? s : slot_pixel(cam, sh, s);
        r.pe0 = ra.x; r.pe1 = ra.y; r.pe2 = ra.z;
        r.dd0 = rb.x; r.dd1 = rb.y; r.dd2 = rb.z; r.dsf = rb.w;
        if (rr.d) {
          const float4 rd = __ldg(rr.d + s);
          r.dx = rd.x; r.dy = rd.y; r.dz = rd.z;
        } else {
          r.dx = r.dy = r.dz = 0.f;
        }
        r.C0 = r.C1 = r.C2 = r.A = 0.f;
      } else if (n < 0) {
        // a ray that misses the volume (ray_setup deferred its pixel): store the
        // background here, so the stores of a mapped host framebuffer drain over PCIe
        // while the march runs instead of serialising before it
        const long long o = (explicit_rays || sh.compact) ? s : slot_pixel(cam, sh, s);
        *reinterpret_cast<float4*>(out + 4 * o) = make_float4(md.bg[0], md.bg[1], md.bg[2], 0.f);
      }
    }
    q.chunk_base += take;
    q.chunk_left -= take;
  }
}

// ws_refill for the two-lanes-per-ray kernel: only even lanes own rays (the odd partner
// evaluates the ray's next sample), so only they take slots from the queue.
template <int Q = 2>
__device__ __forceinline__ void pair_refill(RayLane& r, LaneQueue& q, int lane, const CamDev& cam,
                                            const ShardDev& sh, const RayRecs& rr, long long n_slots,
                                            unsigned long long* __restrict__ queue, const MarchDev& md,
                                            float* __restrict__ out) {
  // Q lanes per ray: the group leaders (lane % Q == 0) hold the rays; chunks of 32/Q slots
  constexpr int kChunk = 32 / Q;
  const bool even = (lane & (Q - 1)) == 0;
  while (true) {
    const unsigned need = __ballot_sync(0xffffffffu, even && !r.has);
    if (need == 0) break;
    if (q.chunk_left == 0) {
      if (q.qdone) break;
      unsigned long long cb = 0;
      if (lane == 0) cb = atomicAdd(queue, (unsigned long long)kChunk);
      cb = __shfl_sync(0xffffffffu, cb, 0);
      if ((long long)cb >= n_slots) { q.qdone = true; break; }
      q.chunk_base = (long long)cb;
      q.chunk_left = (int)min((long long)kChunk, n_slots - (long long)cb);
    }
    const int rank = __popc(need & lanemask_lt());
    const int take = min(__popc(need), q.chunk_left);
    if (even && !r.has && rank < take) {
      const long long qs = q.chunk_base + rank;
      const long long s = sh.order ? ((long long)sh.order[qs >> 6] << 6) | (qs & 63) : qs;
      const float4 ra = __ldg(rr.a + s);
      const int n = __float_as_int(ra.w);
      if (n > 0) {
        const float4 rb = __ldg(rr.b + s);
        r.has = true;
        r.k = 0; r.n = n;
        r.oslot = sh.compact ? s : slot_pixel(cam, sh, s);
        r.pe0 = ra.x; r.pe1 = ra.y; r.pe2 = ra.z;
        r.dd0 = rb.x; r.dd1 = rb.y; r.dd2 = rb.z; r.dsf = rb.w;
        r.dx = r.dy = r.dz = 0.f;
        r.C0 = r.C1 = r.C2 = r.A = 0.f;
      } else if (n < 0) {   // a miss: background pixel (ray_setup deferred it)
        const long long o = sh.compact ? s : slot_pixel(cam, sh, s);
        *reinterpret_cast<float4*>(out + 4 * o) = make_float4(md.bg[0], md.bg[1], md.bg[2], 0.f);
      }
    }
    q.chunk_base += take;
    q.chunk_left -= take;
  }
}

// One compositing step of a ray with the head outputs o (density head: TF lookup;
// colour head: sigmoid rgb + softplus sigma); retires the ray when it ends.
__device__ __forceinline__ void composite_step(RayLane& r, float4 o, bool density, const TFDev& tf,
                                               const MarchDev& md, float* __restrict__ out,
                                               unsigned long long* __restrict__ nonfinite) {
  float cr, cg, cb, sig;
  if (density) {
    tf_eval(tf, sigmoidf_(o.x), cr, cg, cb, sig);
  } else {
    cr = sigmoidf_(o.x); cg = sigmoidf_(o.y); cb = sigmoidf_(o.z); sig = softplusf_(o.w);
  }
  float alpha = 1.f - __expf(-sig * r.dsf);
  alpha = fmaxf(fminf(alpha, md.eps1_f), 0.f);
  const float tr = (1.f - r.A) * alpha;
  r.C0 = fmaf(tr, cr, r.C0); r.C1 = fmaf(tr, cg, r.C1); r.C2 = fmaf(tr, cb, r.C2);
  r.A += tr;
  ++r.k;
  if (r.k >= r.n || r.A > md.et_f) {
    const float om = 1.f - r.A;
    const float4 px4 = make_float4(fmaf(om, md.bg[0], r.C0), fmaf(om, md.bg[1], r.C1),
                                   fmaf(om, md.bg[2], r.C2), r.A);
    *reinterpret_cast<float4*>(out + 4 * r.oslot) = px4;
    // Image invariant (imaging.py:52-57) checked on the device: no host scan
    if (nonfinite && !(isfinite(px4.x) && isfinite(px4.y) && isfinite(px4.z) && isfinite(px4.w)))
      atomicAdd(nonfinite, 1ull);
    r.has = false;
  }
}

}  // namespace fvsrn
