// fvsrn_train.cu -- world-space training step on the GPU.
//
// train_world (train.py:165-206) restated for one batch of positions:
//   forward   assemble_input (model.py:248-279: f64 Fourier phases, f32 trilinear
//             latent lookup grid.py:47-84) -> mlp_forward (nn.py:179-192, f32)
//             -> density / colour head (model.py:342-357)
//   loss      L1 mean and its adjoint sign(diff)/numel (train.py:158-162)
//   backward  head backward (model.py:346-365) -> mlp_backward (nn.py:234-255) ->
//             grid_sample_backward scatter (grid.py:87-137) as f32 atomics
// One thread per sample, f32 SIMT: this is the training side, accuracy before speed
// (the reference trains in f32; gradients agree to ~1e-6 relative).  The kernel
// writes each layer's inputs and adjoints; the batch reductions for the weight
// gradients (delta_l^T @ inputs_l) are plain cuBLAS GEMMs on the host side, and
// adam_kernel applies adam_step (nn.py:279-298) to the flat parameter buffer laid out
// like FvsrnModel.trainable_arrays() (model.py:155-157).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fvsrn_geometry.cuh"
#include "fvsrn_train.cuh"

namespace fvsrn {

namespace {

constexpr int kTrainMaxW = 256;   // widest layer input / output handled per thread

__device__ __forceinline__ double sigmoid_d(double x) { return 1.0 / (1.0 + exp(-x)); }

__device__ __forceinline__ float act_eval_f(int kind, float x) {
  switch (kind) {                       // nn.py:18-29
    case 0: return fmaxf(x, 0.f);
    case 1: return (float)sigmoid_d((double)x);
    case 2: return (float)(fmax((double)x, 0.0) + log1p(exp(-fabs((double)x))));
    case 3: { const float s = sinf(x); return x + s * s; }
    default: { const float s = sinf(x); return 0.5f * x + s * s; }
  }
}

__device__ __forceinline__ float act_grad_f(int kind, float x) {
  switch (kind) {                       // nn.py:32-44
    case 0: return x > 0.f ? 1.f : 0.f;
    case 1: { const float s = (float)sigmoid_d((double)x); return s * (1.f - s); }
    case 2: return (float)sigmoid_d((double)x);
    case 3: return 1.f + sinf(2.f * x);
    default: return 0.5f + sinf(2.f * x);
  }
}

}  // namespace

// Latent cell of one sample (grid.py:47-53), kept for the backward scatter.
struct Cell {
  int x0, y0, z0;
  float fx, fy, fz;
  int klo, khi;     // keyframe bracket (temporal), weight wk of khi
  float wk;
};

// Per-sample cache rows: inputs of layer l at in_off[l] + row * in_l, pre-activations of
// hidden layer l at l * cap * H + row * H, adjoints at d_off[l] + row * out_l (cap rows).
struct CacheRef {
  float* inputs;
  float* preacts;
  float* deltas;
  long long row, cap;
};

// assemble_input (model.py:248-279) + mlp_forward (nn.py:179-192) in f32 (f64 Fourier
// phases); leaves the raw outputs in x[0..d_out).  Caches when c.inputs != nullptr.
// keyframe bracket of a timestep (model.py:200-209): (lo, hi, w), w = 0 when lo == hi
__device__ void kf_bracket(const TrainNetDev& net, double t, int& lo, int& hi, float& w) {
  const int K = net.n_kf;
  const double tc = fmin(fmax(t, net.kf_times[0]), net.kf_times[K - 1]);
  int h = 0;
  while (h < K && net.kf_times[h] < tc) ++h;     // searchsorted(side="left")
  h = min(h, K - 1);
  const int l = (h > 0 && net.kf_times[h] != tc) ? h - 1 : h;
  lo = l;
  hi = h;
  w = h > l ? (float)((tc - net.kf_times[l]) / (net.kf_times[h] - net.kf_times[l])) : 0.f;
}

// assemble_input (model.py:248-279) into x[0..d_in): [p | sin | cos | time | z]
__device__ void assemble_f32(const TrainNetDev& net, const float* __restrict__ params, const double (&p)[3],
                             const double* d, double t, float (&x)[kTrainMaxW], Cell& cell) {
  const int rw = net.raw_w, fi = net.fd_in;
  const double enc[6] = {p[0], p[1], p[2], d ? d[0] : 0.0, d ? d[1] : 0.0, d ? d[2] : 0.0};
  for (int a = 0; a < rw; ++a) x[a] = (float)enc[a];
  for (int j = 0; j < net.m; ++j) {
    double ph = 0.0;
    for (int a = 0; a < fi; ++a) ph += (double)net.bmat[fi * j + a] * enc[a];
    x[rw + j] = (float)sin(ph);
    x[rw + net.m + j] = (float)cos(ph);
  }
  int k = rw + 2 * net.m;
  if (net.time_mode != 0) {   // _time_features (model.py:236-245)
    const double tn = net.t1 == net.t0 ? 0.0 : (fmin(fmax(t, net.t0), net.t1) - net.t0) / (net.t1 - net.t0);
    if (net.time_mode & 1) x[k++] = (float)tn;
    if (net.time_mode & 2) {
      for (int j = 0; j < net.time_l; ++j) x[k + j] = (float)sin(tn * (double)net.time_b[j]);
      for (int j = 0; j < net.time_l; ++j) x[k + net.time_l + j] = (float)cos(tn * (double)net.time_b[j]);
      k += 2 * net.time_l;
    }
  }
  const int R = net.grid_res, F = net.grid_ch;
  int klo = 0, khi = 0;
  float wk = 0.f;
  if (net.n_kf > 0) kf_bracket(net, t, klo, khi, wk);
  const long long gsz = (long long)R * R * R * F;
  const float* grid = params + net.grid_off + klo * gsz;
  cell = Cell{0, 0, 0, 0.f, 0.f, 0.f, klo, khi, wk};
  if (R > 0) {   // _cell_coords (grid.py:47-53) + _gather_kernel
    const double s = (double)(R - 1);
    const double cx = fmin(fmax(p[0], 0.0), 1.0) * s, cy = fmin(fmax(p[1], 0.0), 1.0) * s,
                 cz = fmin(fmax(p[2], 0.0), 1.0) * s;
    cell.x0 = min((int)cx, R - 2); cell.y0 = min((int)cy, R - 2); cell.z0 = min((int)cz, R - 2);
    cell.fx = (float)(cx - cell.x0); cell.fy = (float)(cy - cell.y0); cell.fz = (float)(cz - cell.z0);
    const float fx = cell.fx, fy = cell.fy, fz = cell.fz;
    const float gx = 1.f - fx, gy = 1.f - fy, gz = 1.f - fz;
    const float w[8] = {gx * gy * gz, gx * gy * fz, gx * fy * gz, gx * fy * fz,
                        fx * gy * gz, fx * gy * fz, fx * fy * gz, fx * fy * fz};
    const long long sz = F, sy = (long long)R * F, sx = (long long)R * R * F;
    const long long off[8] = {0, sz, sy, sy + sz, sx, sx + sz, sx + sy, sx + sy + sz};
    const long long base = (((long long)cell.x0 * R + cell.y0) * R + cell.z0) * F;
    const float* b = grid + base;
    const float* b2 = params + net.grid_off + khi * gsz + base;
    for (int ch = 0; ch < F; ++ch) {
      float acc = 0.f;
      for (int q = 0; q < 8; ++q) acc += w[q] * b[off[q] + ch];
      if (khi != klo) {   // (1 - w) z_lo + w z_hi in f32 (model.py:219-233)
        float acc2 = 0.f;
        for (int q = 0; q < 8; ++q) acc2 += w[q] * b2[off[q] + ch];
        acc = __fadd_rn(__fmul_rn(__fsub_rn(1.f, wk), acc), __fmul_rn(wk, acc2));
      }
      x[k + ch] = acc;
    }
  }
}

// mlp_forward (nn.py:179-192) of x[0..d_in) -> raw outputs in x[0..d_out); caches layer
// inputs / pre-activations when c.inputs != nullptr
__device__ void mlp_f32(const TrainNetDev& net, const float* __restrict__ params, const CacheRef& c,
                        float (&x)[kTrainMaxW], float (&y)[kTrainMaxW]) {
  const int L = net.layers, H = net.hidden, C = net.d_out;
  int in_w = net.d_in;
  for (int l = 0; l < L; ++l) {
    const int out_w = (l == L - 1) ? C : H;
    if (c.inputs) {
      float* inl = c.inputs + net.in_off[l] + c.row * in_w;
      for (int j = 0; j < in_w; ++j) inl[j] = x[j];
    }
    const float* W = params + net.w_off[l];
    const float* bb = params + net.b_off[l];
    for (int o = 0; o < out_w; ++o) {
      float s = bb[o];
      const float* wr = W + (long long)o * in_w;
      for (int j = 0; j < in_w; ++j) s = fmaf(x[j], wr[j], s);
      y[o] = s;
    }
    if (l < L - 1) {
      float* pa = c.preacts ? c.preacts + (long long)l * c.cap * H + c.row * H : nullptr;
      for (int o = 0; o < out_w; ++o) {
        if (pa) pa[o] = y[o];
        x[o] = act_eval_f(net.act, y[o]);
      }
    } else {
      for (int o = 0; o < out_w; ++o) x[o] = y[o];
    }
    in_w = out_w;
  }
}

__device__ void f32_forward(const TrainNetDev& net, const float* __restrict__ params, const double (&p)[3],
                            double t, const CacheRef& c, float (&x)[kTrainMaxW], float (&y)[kTrainMaxW],
                            Cell& cell) {
  assemble_f32(net, params, p, nullptr, t, x, cell);
  mlp_f32(net, params, c, x, y);
}

// mlp_backward (nn.py:234-255) from raw_bar, writing the adjoints, then the latent-grid
// scatter (grid.py:87-137) of z_bar = x_bar[-F:] as f32 atomics.
__device__ void f32_backward(const TrainNetDev& net, const float* __restrict__ params,
                             const float (&raw_bar)[4], const CacheRef& c, const Cell& cell,
                             float* __restrict__ grid_grad, float (&x)[kTrainMaxW], float (&y)[kTrainMaxW]) {
  const int L = net.layers, H = net.hidden, C = net.d_out;
  for (int ch = 0; ch < C; ++ch) y[ch] = raw_bar[ch];
  for (int l = L - 1; l >= 0; --l) {
    const int out_w = (l == L - 1) ? C : H;
    const int inw = (l == 0) ? net.d_in : H;
    if (l < L - 1) {
      const float* pa = c.preacts + (long long)l * c.cap * H + c.row * H;
      for (int o = 0; o < out_w; ++o) y[o] *= act_grad_f(net.act, pa[o]);
    }
    float* dl = c.deltas + net.d_off[l] + c.row * out_w;
    for (int o = 0; o < out_w; ++o) dl[o] = y[o];
    const float* W = params + net.w_off[l];
    for (int j = 0; j < inw; ++j) {
      float s = 0.f;
      for (int o = 0; o < out_w; ++o) s = fmaf(y[o], W[(long long)o * inw + j], s);
      x[j] = s;
    }
    for (int j = 0; j < inw; ++j) y[j] = x[j];
  }
  const int R = net.grid_res, F = net.grid_ch;
  if (R > 0) {
    const float fx = cell.fx, fy = cell.fy, fz = cell.fz;
    const float gx = 1.f - fx, gy = 1.f - fy, gz = 1.f - fz;
    const float w[8] = {gx * gy * gz, gx * gy * fz, gx * fy * gz, gx * fy * fz,
                        fx * gy * gz, fx * gy * fz, fx * fy * gz, fx * fy * fz};
    const long long sz = F, sy = (long long)R * F, sx = (long long)R * R * F;
    const long long off[8] = {0, sz, sy, sy + sz, sx, sx + sz, sx + sy, sx + sy + sz};
    const long long gsz = (long long)R * R * R * F;
    const long long base = (((long long)cell.x0 * R + cell.y0) * R + cell.z0) * F;
    float* g = grid_grad + cell.klo * gsz + base;
    float* g2 = grid_grad + cell.khi * gsz + base;
    const int zoff = net.d_in - F;
    const bool two = cell.khi != cell.klo;   // model.py:318-333: (1-w) zb -> lo, w zb -> hi
    for (int ch = 0; ch < F; ++ch) {
      const float zb = y[zoff + ch];
      const float zl = two ? __fmul_rn(__fsub_rn(1.f, cell.wk), zb) : zb;
      for (int q = 0; q < 8; ++q) atomicAdd(g + off[q] + ch, w[q] * zl);
      if (two) {
        const float zh = __fmul_rn(cell.wk, zb);
        for (int q = 0; q < 8; ++q) atomicAdd(g2 + off[q] + ch, w[q] * zh);
      }
    }
  }
}

__global__ void train_world_kernel(TrainNetDev net, const float* __restrict__ params,
                                   const double* __restrict__ pos, const double* __restrict__ times,
                                   const float* __restrict__ ref,
                                   long long n, float* __restrict__ grid_grad,
                                   float* __restrict__ inputs, float* __restrict__ preacts,
                                   float* __restrict__ deltas, double* __restrict__ loss_sum) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double my_loss = 0.0;
  if (i < n) {
    const int C = net.d_out;
    float x[kTrainMaxW], y[kTrainMaxW];
    const double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    const CacheRef c{inputs, preacts, deltas, i, n};
    Cell cell;
    f32_forward(net, params, p, times ? times[i] : 0.0, c, x, y, cell);
    // ---- head, L1 loss and its adjoint (train.py:158-162), head backward
    const float inv = (float)(1.0 / ((double)n * C));
    float raw_bar[4];
    for (int ch = 0; ch < C; ++ch) {
      const double r = x[ch];
      const bool softplus_ch = net.head != 0 && ch == 3;
      const float pred = softplus_ch ? (float)(fmax(r, 0.0) + log1p(exp(-fabs(r)))) : (float)sigmoid_d(r);
      const float diff = __fsub_rn(pred, ref[i * C + ch]);
      my_loss += fabs((double)diff);
      const float adj = (diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f)) * inv;
      // density_head_backward / color_head_backward (model.py:346-365), f32 like numpy
      raw_bar[ch] = softplus_ch ? __fmul_rn(adj, (float)sigmoid_d(r))
                                : __fmul_rn(__fmul_rn(adj, pred), __fsub_rn(1.f, pred));
    }
    f32_backward(net, params, raw_bar, c, cell, grid_grad, x, y);
  }
  // batch L1 loss sum (train.py:158-161): warp reduce, one f64 atomic per warp
  for (int o = 16; o > 0; o >>= 1) my_loss += __shfl_down_sync(0xffffffffu, my_loss, o);
  if ((threadIdx.x & 31) == 0 && loss_sum) atomicAdd(loss_sum, my_loss);
}

// mlp_forward / mlp_backward (nn.py:179-193, 234-256) of given inputs x (n, d_in): the
// forward with its caches (layer inputs, hidden pre-activations) and outputs; with y_bar,
// the reverse pass writes the per-layer deltas (weight/bias/input adjoints are the
// caller's GEMMs over the caches).
__global__ void mlp_grads_kernel(TrainNetDev net, const float* __restrict__ params,
                                 const float* __restrict__ x_in, const float* __restrict__ y_bar,
                                 long long n, float* __restrict__ y_out, float* __restrict__ inputs,
                                 float* __restrict__ preacts, float* __restrict__ deltas) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float x[kTrainMaxW], y[kTrainMaxW];
  for (int j = 0; j < net.d_in; ++j) x[j] = x_in[i * net.d_in + j];
  const CacheRef c{inputs, preacts, deltas, i, n};
  mlp_f32(net, params, c, x, y);
  for (int o = 0; o < net.d_out; ++o) y_out[i * net.d_out + o] = y[o];
  if (y_bar) {
    float rb[4] = {0.f, 0.f, 0.f, 0.f};
    for (int o = 0; o < net.d_out && o < 4; ++o) rb[o] = y_bar[i * net.d_out + o];
    const Cell cell{0, 0, 0, 0.f, 0.f, 0.f, 0, 0, 0.f};
    f32_backward(net, params, rb, c, cell, nullptr, x, y);
  }
}

cudaError_t launch_mlp_grads(const TrainNetDev& net, const float* params, const float* x, const float* y_bar,
                             long long n, float* y_out, float* inputs, float* preacts, float* deltas,
                             cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  mlp_grads_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(net, params, x, y_bar, n, y_out, inputs,
                                                                 preacts, deltas);
  return cudaGetLastError();
}

// grid_sample_backward (grid.py:123-137): trilinear-weighted scatter-add of per-sample
// adjoints z_bar (n, F) into a gradient grid shaped like the latent grid (R, R, R, F).
// Same cell arithmetic as the lookup (_cell_coords in f64, f32 weights); atomics replace
// the reference's sequential loop, so sums agree to rounding order.
__global__ void grid_scatter_kernel(int R, int F, const double* __restrict__ pos,
                                    const float* __restrict__ z_bar, long long n, float* __restrict__ grad) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double s = (double)(R - 1);
  const double cx = fmin(fmax(pos[3 * i], 0.0), 1.0) * s, cy = fmin(fmax(pos[3 * i + 1], 0.0), 1.0) * s,
               cz = fmin(fmax(pos[3 * i + 2], 0.0), 1.0) * s;
  const int x0 = min((int)cx, R - 2), y0 = min((int)cy, R - 2), z0 = min((int)cz, R - 2);
  const float fx = (float)(cx - x0), fy = (float)(cy - y0), fz = (float)(cz - z0);
  const float gx = 1.f - fx, gy = 1.f - fy, gz = 1.f - fz;
  const float w[8] = {gx * gy * gz, gx * gy * fz, gx * fy * gz, gx * fy * fz,
                      fx * gy * gz, fx * gy * fz, fx * fy * gz, fx * fy * fz};
  const long long sz = F, sy = (long long)R * F, sx = (long long)R * R * F;
  const long long off[8] = {0, sz, sy, sy + sz, sx, sx + sz, sx + sy, sx + sy + sz};
  float* g = grad + (((long long)x0 * R + y0) * R + z0) * F;
  for (int ch = 0; ch < F; ++ch) {
    const float zb = z_bar[i * F + ch];
    for (int q = 0; q < 8; ++q) atomicAdd(g + off[q] + ch, w[q] * zb);
  }
}

cudaError_t launch_grid_scatter(int R, int F, const double* pos, const float* z_bar, long long n,
                                float* grad, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  grid_scatter_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(R, F, pos, z_bar, n, grad);
  return cudaGetLastError();
}

// model_backward (model.py:300-335): gradients of sum(raw_bar * raw) for given per-sample
// raw-output adjoints (any head, any input encoding incl. view directions).  The forward
// is recomputed with its caches (deterministic, identical to model_forward's); weight /
// bias reductions are GEMMs on the host side, the latent-grid adjoint is scattered here.
__global__ void model_grads_kernel(TrainNetDev net, const float* __restrict__ params,
                                   const double* __restrict__ pos, const double* __restrict__ dirs,
                                   const double* __restrict__ times, const float* __restrict__ raw_bar_in,
                                   long long n, float* __restrict__ grid_grad,
                                   float* __restrict__ inputs, float* __restrict__ preacts,
                                   float* __restrict__ deltas) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float x[kTrainMaxW], y[kTrainMaxW];
  const double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
  const CacheRef c{inputs, preacts, deltas, i, n};
  Cell cell;
  assemble_f32(net, params, p, dirs ? dirs + 3 * i : nullptr, times ? times[i] : 0.0, x, cell);
  mlp_f32(net, params, c, x, y);
  float raw_bar[4] = {0.f, 0.f, 0.f, 0.f};
  for (int ch = 0; ch < net.d_out && ch < 4; ++ch) raw_bar[ch] = raw_bar_in[i * net.d_out + ch];
  f32_backward(net, params, raw_bar, c, cell, grid_grad, x, y);
}

cudaError_t launch_model_grads(const TrainNetDev& net, const float* params, const double* pos,
                               const double* dirs, const double* times, const float* raw_bar, long long n,
                               float* grid_grad, float* inputs, float* preacts, float* deltas,
                               cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int threads = 128;
  model_grads_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(
      net, params, pos, dirs, times, raw_bar, n, grid_grad, inputs, preacts, deltas);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- screen space
// raymarch_forward(ModelSource(colour model), want_states=True) (render.py:203-238):
// f64 geometry and compositing, f32 model evaluation (the naive ModelSource path), no
// early termination; terminal (C, A) and the per-ray geometry are kept for backward.
__global__ void screen_forward_kernel(TrainNetDev net, const float* __restrict__ params,
                                      const double* __restrict__ org, const double* __restrict__ dir,
                                      long long n, MarchDev md, float* __restrict__ px,
                                      double* __restrict__ cst, double* __restrict__ ast,
                                      double* __restrict__ tmin_o, double* __restrict__ ds_o,
                                      int* __restrict__ nsteps) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  RayGeom g;
  for (int a = 0; a < 3; ++a) { g.o[a] = org[3 * i + a]; g.d[a] = dir[3 * i + a]; }
  int ns = 0;
  double tmin = 0.0, ds = 0.0;
  if (march_geometry(md, g)) { ns = g.n; tmin = g.tmin; ds = g.ds; }
  double C0 = 0.0, C1 = 0.0, C2 = 0.0, A = 0.0;
  float x[kTrainMaxW], y[kTrainMaxW];
  const CacheRef none{nullptr, nullptr, nullptr, 0, 0};
  for (int k = 0; k < ns; ++k) {
    const double tk = __dadd_rn(tmin, __dmul_rn((double)k + 0.5, ds));
    const double p[3] = {__dadd_rn(g.o[0], __dmul_rn(tk, g.d[0])), __dadd_rn(g.o[1], __dmul_rn(tk, g.d[1])),
                         __dadd_rn(g.o[2], __dmul_rn(tk, g.d[2]))};
    Cell cell;
    f32_forward(net, params, p, 0.0, none, x, y, cell);
    const double r = (float)sigmoid_d(x[0]), gg = (float)sigmoid_d(x[1]), b = (float)sigmoid_d(x[2]);
    const double sig = (float)(fmax((double)x[3], 0.0) + log1p(exp(-fabs((double)x[3]))));
    // composite_step (render.py:109-117)
    double alpha = fmin(1.0 - md.eps_blend, -expm1(-sig * ds));
    alpha = fmax(alpha, 0.0);
    const double tr = (1.0 - A) * alpha;
    C0 += tr * r; C1 += tr * gg; C2 += tr * b;
    A += tr;
  }
  px[4 * i] = (float)(C0 + (1.0 - A) * md.bg[0]);
  px[4 * i + 1] = (float)(C1 + (1.0 - A) * md.bg[1]);
  px[4 * i + 2] = (float)(C2 + (1.0 - A) * md.bg[2]);
  px[4 * i + 3] = (float)A;
  cst[3 * i] = C0; cst[3 * i + 1] = C1; cst[3 * i + 2] = C2;
  ast[i] = A;
  tmin_o[i] = tmin;
  ds_o[i] = ds;
  nsteps[i] = ns;
}

// raymarch_backward (render.py:241-306): each thread walks its ray in reverse step
// order, re-evaluates the model, inverts the blend to recover the previous state
// (constant memory per ray), and writes the sample's cache rows at row off[i] + k so the
// weight-gradient reductions are one GEMM per layer over all samples of the chunk.
__global__ void screen_backward_kernel(TrainNetDev net, const float* __restrict__ params,
                                       const double* __restrict__ org, const double* __restrict__ dir,
                                       long long n, double eps_blend, const double* __restrict__ cst,
                                       const double* __restrict__ ast, const double* __restrict__ tmin_a,
                                       const double* __restrict__ ds_a, const int* __restrict__ nsteps,
                                       const long long* __restrict__ row_off, const float* __restrict__ adj,
                                       const double* __restrict__ bg, long long cap,
                                       float* __restrict__ inputs, float* __restrict__ preacts,
                                       float* __restrict__ deltas, float* __restrict__ grid_grad) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int ns = nsteps[i];
  if (ns == 0) return;
  double c_acc[3] = {cst[3 * i], cst[3 * i + 1], cst[3 * i + 2]};
  double a_acc = ast[i];
  const double tmin = tmin_a[i], ds = ds_a[i];
  double c_bar[3] = {(double)adj[4 * i], (double)adj[4 * i + 1], (double)adj[4 * i + 2]};
  double a_bar = (double)adj[4 * i + 3] - (c_bar[0] * bg[0] + c_bar[1] * bg[1] + c_bar[2] * bg[2]);
  float x[kTrainMaxW], y[kTrainMaxW];
  for (int k = ns - 1; k >= 0; --k) {
    const double tk = __dadd_rn(tmin, __dmul_rn((double)k + 0.5, ds));
    const double p[3] = {__dadd_rn(org[3 * i], __dmul_rn(tk, dir[3 * i])),
                         __dadd_rn(org[3 * i + 1], __dmul_rn(tk, dir[3 * i + 1])),
                         __dadd_rn(org[3 * i + 2], __dmul_rn(tk, dir[3 * i + 2]))};
    const CacheRef c{inputs, preacts, deltas, row_off[i] + k, cap};
    Cell cell;
    f32_forward(net, params, p, 0.0, c, x, y, cell);
    float raw[4] = {x[0], x[1], x[2], x[3]};
    const float s0 = (float)sigmoid_d(raw[0]), s1 = (float)sigmoid_d(raw[1]), s2 = (float)sigmoid_d(raw[2]);
    const double rgb[3] = {s0, s1, s2};
    const double sigma = (float)(fmax((double)raw[3], 0.0) + log1p(exp(-fabs((double)raw[3]))));
    const double alpha_raw = -expm1(-sigma * ds);
    const bool clamped = alpha_raw > 1.0 - eps_blend;
    const double alpha = clamped ? 1.0 - eps_blend : fmax(alpha_raw, 0.0);
    const double a_prev = (a_acc - alpha) / (1.0 - alpha);
    const double one_m = 1.0 - a_prev;
    double c_prev[3], dot = 0.0;
    for (int q = 0; q < 3; ++q) {
      c_prev[q] = c_acc[q] - (one_m * alpha) * rgb[q];
      dot += c_bar[q] * rgb[q];
    }
    const double alpha_bar = a_bar * one_m + dot * one_m;
    const double sigma_bar = clamped ? 0.0 : alpha_bar * ds * exp(-sigma * ds);
    // color_head_backward (model.py:360-365) on the f32 head adjoint
    float raw_bar[4];
    const float s[3] = {s0, s1, s2};
    for (int q = 0; q < 3; ++q) {
      const float rb = (float)(c_bar[q] * (alpha * one_m));
      raw_bar[q] = __fmul_rn(__fmul_rn(rb, s[q]), __fsub_rn(1.f, s[q]));
    }
    raw_bar[3] = __fmul_rn((float)sigma_bar, (float)sigmoid_d(raw[3]));
    f32_backward(net, params, raw_bar, c, cell, grid_grad, x, y);
    a_bar = a_bar * (1.0 - alpha) - dot * alpha;
    for (int q = 0; q < 3; ++q) c_acc[q] = c_prev[q];
    a_acc = a_prev;
  }
}

// adam_step (nn.py:279-298) on the flat trainable buffer; non-finite gradients are
// counted first; if any, the update is skipped entirely and the host raises
// FloatingPointError, as adam_step does before touching a parameter
__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, long long n, AdamConsts k,
                            const unsigned long long* __restrict__ bad) {
  if (*bad) return;   // non-finite gradient: nothing is updated (the host raises)
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    // the numpy statement order of nn.py:294-298, each op rounded separately
    const float gi = g[i];
    const float mi = __fadd_rn(__fmul_rn(m[i], k.b1), __fmul_rn(k.one_m_b1, gi));
    const float vi = __fadd_rn(__fmul_rn(v[i], k.b2), __fmul_rn(__fmul_rn(k.one_m_b2, gi), gi));
    m[i] = mi;
    v[i] = vi;
    const float num = __fmul_rn(k.lr, __fdiv_rn(mi, k.bc1));
    const float den = __fadd_rn(__fsqrt_rn(__fdiv_rn(vi, k.bc2)), k.eps);
    p[i] = __fsub_rn(p[i], __fdiv_rn(num, den));
  }
}

__global__ void count_nonfinite_kernel(const float* __restrict__ g, long long n,
                                       unsigned long long* __restrict__ bad) {
  unsigned c = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    c += isfinite(g[i]) ? 0u : 1u;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(bad, (unsigned long long)c);
}

cudaError_t launch_train_world(const TrainNetDev& net, const float* params, const double* pos,
                               const double* times, const float* ref, long long n, float* grid_grad,
                               float* inputs, float* preacts, float* deltas, double* loss_sum,
                               cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int threads = 128;
  train_world_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(
      net, params, pos, times, ref, n, grid_grad, inputs, preacts, deltas, loss_sum);
  return cudaGetLastError();
}

cudaError_t launch_screen_forward(const TrainNetDev& net, const float* params, const double* org,
                                  const double* dir, long long n, const MarchDev& md, float* px,
                                  double* cst, double* ast, double* tmin, double* ds, int* nsteps,
                                  cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  screen_forward_kernel<<<(unsigned)((n + 63) / 64), 64, 0, s>>>(net, params, org, dir, n, md, px, cst,
                                                                  ast, tmin, ds, nsteps);
  return cudaGetLastError();
}

cudaError_t launch_screen_backward(const TrainNetDev& net, const float* params, const double* org,
                                   const double* dir, long long n, double eps_blend, const double* cst,
                                   const double* ast, const double* tmin, const double* ds,
                                   const int* nsteps, const long long* row_off, const float* adj,
                                   const double* bg, long long cap, float* inputs, float* preacts,
                                   float* deltas, float* grid_grad, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  screen_backward_kernel<<<(unsigned)((n + 63) / 64), 64, 0, s>>>(
      net, params, org, dir, n, eps_blend, cst, ast, tmin, ds, nsteps, row_off, adj, bg, cap, inputs,
      preacts, deltas, grid_grad);
  return cudaGetLastError();
}

// Reference-semantics f32 evaluation of the pieces of the model (stage 0: assembled
// inputs, 1: latent vectors (grid_sample / keyframe_sample), 2: raw MLP outputs from
// positions, 3: raw MLP outputs of given inputs x (mlp_eval)).
__global__ void f32_eval_kernel(TrainNetDev net, const float* __restrict__ params,
                                const double* __restrict__ pos, const double* __restrict__ dirs,
                                const double* __restrict__ times,
                                const float* __restrict__ xin, long long n, int stage,
                                float* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float x[kTrainMaxW], y[kTrainMaxW];
  const CacheRef none{nullptr, nullptr, nullptr, 0, 0};
  if (stage == 3) {
    for (int j = 0; j < net.d_in; ++j) x[j] = xin[i * net.d_in + j];
    mlp_f32(net, params, none, x, y);
    for (int c = 0; c < net.d_out; ++c) out[i * net.d_out + c] = x[c];
    return;
  }
  const double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
  Cell cell;
  assemble_f32(net, params, p, dirs ? dirs + 3 * i : nullptr, times ? times[i] : 0.0, x, cell);
  if (stage == 0) {
    for (int j = 0; j < net.d_in; ++j) out[i * net.d_in + j] = x[j];
  } else if (stage == 1) {
    const int F = net.grid_ch;
    for (int c = 0; c < F; ++c) out[i * F + c] = x[net.d_in - F + c];
  } else {
    mlp_f32(net, params, none, x, y);
    for (int c = 0; c < net.d_out; ++c) out[i * net.d_out + c] = x[c];
  }
}

cudaError_t launch_f32_eval(const TrainNetDev& net, const float* params, const double* pos,
                            const double* dirs, const double* times, const float* xin, long long n,
                            int stage, float* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  f32_eval_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(net, params, pos, dirs, times, xin, n, stage,
                                                               out);
  return cudaGetLastError();
}

cudaError_t launch_adam(float* p, const float* g, float* m, float* v, long long n, const AdamConsts& k,
                        unsigned long long* bad, cudaStream_t s) {
  const long long b = (n + 255) / 256;
  const int blocks = (int)(b < 148 * 8 ? b : 148 * 8);
  count_nonfinite_kernel<<<blocks, 256, 0, s>>>(g, n, bad);
  adam_kernel<<<blocks, 256, 0, s>>>(p, g, m, v, n, k, bad);
  return cudaGetLastError();
}

}  // namespace fvsrn
