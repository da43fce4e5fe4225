// fvsrn_geometry.cuh -- bit-exact f64 ray setup shared by the model and volume renderers.
#pragma once
#include "fvsrn_kernels.cuh"

namespace fvsrn {

// ---------------------------------------------------------------- ray setup (f64)
// Bit-exact restatement of camera_rays (render.py:72-94), ray_box_intersect
// (render.py:97-106) and _march_geometry (render.py:189-200): every f64 op is an
// explicit _rn intrinsic so nvcc cannot contract it into an FMA.
struct RayGeom {
  double o[3], d[3], tmin, ds;
  int n;
};

__device__ __forceinline__ void camera_dir(const CamDev& cam, int px, int py, double (&d)[3]) {
  double gx = __dmul_rn(__dsub_rn(__dmul_rn(__ddiv_rn(__dadd_rn((double)px, 0.5), (double)cam.W), 2.0), 1.0),
                        cam.half_w);
  double gy = __dmul_rn(__dsub_rn(1.0, __dmul_rn(__ddiv_rn(__dadd_rn((double)py, 0.5), (double)cam.H), 2.0)),
                        cam.half_h);
#pragma unroll
  for (int a = 0; a < 3; ++a)
    d[a] = __dadd_rn(__dadd_rn(cam.fwd[a], __dmul_rn(gx, cam.right[a])), __dmul_rn(gy, cam.up[a]));
  double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])),
                                    __dmul_rn(d[2], d[2])));
#pragma unroll
  for (int a = 0; a < 3; ++a) d[a] = __ddiv_rn(d[a], nrm);
}

__device__ __forceinline__ bool march_geometry(const MarchDev& md, RayGeom& r) {
  double tmin = -INFINITY, tmax = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double dd = fabs(r.d[a]) < 1e-12 ? 1e-12 : r.d[a];
    double tlo = __ddiv_rn(__dsub_rn(0.0, r.o[a]), dd);
    double thi = __ddiv_rn(__dsub_rn(1.0, r.o[a]), dd);
    tmin = fmax(tmin, fmin(tlo, thi));
    tmax = fmin(tmax, fmax(tlo, thi));
  }
  tmin = fmax(tmin, 0.0);
  if (!(tmax > tmin)) return false;
  double len = __dsub_rn(tmax, tmin);
  double nf = ceil(__ddiv_rn(len, md.stepsize));
  long long n = (long long)nf;
  if (n > md.max_steps) n = md.max_steps;
  if (n < 1) n = 1;
  r.n = (int)n;
  r.tmin = tmin;
  r.ds = __ddiv_rn(len, (double)n);
  return true;
}

// slot -> pixel of this shard (8x8 tiles, tile = rank + lt*world); -1 if outside the frame
__device__ __forceinline__ int slot_pixel(const CamDev& cam, const ShardDev& sh, long long s) {
  long long lt = s >> 6;
  int e = (int)(s & 63);
  long long tile = sh.rank + lt * sh.world;
  if (tile >= sh.n_tiles) return -1;
  int tx = (int)(tile % sh.tiles_x), ty = (int)(tile / sh.tiles_x);
  int px = tx * kTile + (e & 7), py = ty * kTile + (e >> 3);
  if (px >= cam.W || py >= cam.H) return -1;
  return py * cam.W + px;
}


}  // namespace fvsrn
