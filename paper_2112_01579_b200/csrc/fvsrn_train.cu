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

__global__ void train_world_kernel(TrainNetDev net, const float* __restrict__ params,
                                   const double* __restrict__ pos, const float* __restrict__ ref,
                                   long long n, float* __restrict__ grid_grad,
                                   float* __restrict__ inputs, float* __restrict__ preacts,
                                   float* __restrict__ deltas, double* __restrict__ loss_sum) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double my_loss = 0.0;
  if (i < n) {
    const int L = net.layers, H = net.hidden, C = net.d_out;
    float x[kTrainMaxW], y[kTrainMaxW];
    const double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    // ---- assemble_input: [p | sin(Bp) | cos(Bp) | z]
    int k = 0;
    for (int a = 0; a < 3; ++a) x[k++] = (float)p[a];
    for (int j = 0; j < net.m; ++j) {
      const double ph = (double)net.bmat[3 * j] * p[0] + (double)net.bmat[3 * j + 1] * p[1] +
                        (double)net.bmat[3 * j + 2] * p[2];
      x[3 + j] = (float)sin(ph);
      x[3 + net.m + j] = (float)cos(ph);
    }
    k = 3 + 2 * net.m;
    int x0 = 0, y0 = 0, z0 = 0;
    float fx = 0.f, fy = 0.f, fz = 0.f;
    const float* grid = params + net.grid_off;
    const int R = net.grid_res, F = net.grid_ch;
    if (R > 0) {   // _cell_coords (grid.py:47-53) + _gather_kernel
      const double s = (double)(R - 1);
      const double cx = fmin(fmax(p[0], 0.0), 1.0) * s, cy = fmin(fmax(p[1], 0.0), 1.0) * s,
                   cz = fmin(fmax(p[2], 0.0), 1.0) * s;
      x0 = min((int)cx, R - 2); y0 = min((int)cy, R - 2); z0 = min((int)cz, R - 2);
      fx = (float)(cx - x0); fy = (float)(cy - y0); fz = (float)(cz - z0);
      const float gx = 1.f - fx, gy = 1.f - fy, gz = 1.f - fz;
      const float w[8] = {gx * gy * gz, gx * gy * fz, gx * fy * gz, gx * fy * fz,
                          fx * gy * gz, fx * gy * fz, fx * fy * gz, fx * fy * fz};
      const long long sz = F, sy = (long long)R * F, sx = (long long)R * R * F;
      const long long off[8] = {0, sz, sy, sy + sz, sx, sx + sz, sx + sy, sx + sy + sz};
      const float* b = grid + (((long long)x0 * R + y0) * R + z0) * F;
      for (int c = 0; c < F; ++c) {
        float acc = 0.f;
        for (int q = 0; q < 8; ++q) acc += w[q] * b[off[q] + c];
        x[k + c] = acc;
      }
      k += F;
    }
    // ---- mlp_forward (nn.py:179-192), caching layer inputs and pre-activations
    int in_w = net.d_in;
    for (int l = 0; l < L; ++l) {
      const int out_w = (l == L - 1) ? C : H;
      float* inl = inputs + net.in_off[l] + i * in_w;
      for (int j = 0; j < in_w; ++j) inl[j] = x[j];
      const float* W = params + net.w_off[l];
      const float* bb = params + net.b_off[l];
      for (int o = 0; o < out_w; ++o) {
        float s = bb[o];
        const float* wr = W + (long long)o * in_w;
        for (int j = 0; j < in_w; ++j) s = fmaf(x[j], wr[j], s);
        y[o] = s;
      }
      if (l < L - 1) {
        float* pa = preacts + (long long)l * n * H + i * H;
        for (int o = 0; o < out_w; ++o) { pa[o] = y[o]; x[o] = act_eval_f(net.act, y[o]); }
      } else {
        for (int o = 0; o < out_w; ++o) x[o] = y[o];
      }
      in_w = out_w;
    }
    // ---- head, L1 loss and its adjoint (train.py:158-162), head backward
    const float inv = (float)(1.0 / ((double)n * C));
    float raw_bar[4];
    for (int c = 0; c < C; ++c) {
      const double r = x[c];
      const bool softplus_ch = net.head != 0 && c == 3;
      const float pred = softplus_ch ? (float)(fmax(r, 0.0) + log1p(exp(-fabs(r)))) : (float)sigmoid_d(r);
      const float diff = __fsub_rn(pred, ref[i * C + c]);
      my_loss += fabs((double)diff);
      const float adj = (diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f)) * inv;
      // density_head_backward / color_head_backward (model.py:346-365), f32 like numpy
      raw_bar[c] = softplus_ch ? __fmul_rn(adj, (float)sigmoid_d(r))
                               : __fmul_rn(__fmul_rn(adj, pred), __fsub_rn(1.f, pred));
    }
    // ---- mlp_backward (nn.py:234-255)
    for (int c = 0; c < C; ++c) y[c] = raw_bar[c];
    for (int l = L - 1; l >= 0; --l) {
      const int out_w = (l == L - 1) ? C : H;
      const int inw = (l == 0) ? net.d_in : H;
      if (l < L - 1) {
        const float* pa = preacts + (long long)l * n * H + i * H;
        for (int o = 0; o < out_w; ++o) y[o] *= act_grad_f(net.act, pa[o]);
      }
      float* dl = deltas + net.d_off[l] + i * out_w;
      for (int o = 0; o < out_w; ++o) dl[o] = y[o];
      const float* W = params + net.w_off[l];
      for (int j = 0; j < inw; ++j) {
        float s = 0.f;
        for (int o = 0; o < out_w; ++o) s = fmaf(y[o], W[(long long)o * inw + j], s);
        x[j] = s;
      }
      for (int j = 0; j < inw; ++j) y[j] = x[j];
    }
    // ---- grid_sample_backward (grid.py:87-137): z_bar = x_bar[-F:]
    if (R > 0) {
      const float gx = 1.f - fx, gy = 1.f - fy, gz = 1.f - fz;
      const float w[8] = {gx * gy * gz, gx * gy * fz, gx * fy * gz, gx * fy * fz,
                          fx * gy * gz, fx * gy * fz, fx * fy * gz, fx * fy * fz};
      const long long sz = F, sy = (long long)R * F, sx = (long long)R * R * F;
      const long long off[8] = {0, sz, sy, sy + sz, sx, sx + sz, sx + sy, sx + sy + sz};
      float* g = grid_grad + (((long long)x0 * R + y0) * R + z0) * F;
      const int zoff = net.d_in - F;
      for (int c = 0; c < F; ++c) {
        const float zb = y[zoff + c];
        for (int q = 0; q < 8; ++q) atomicAdd(g + off[q] + c, w[q] * zb);
      }
    }
  }
  // batch L1 loss sum (train.py:158-161): warp reduce, one f64 atomic per warp
  for (int o = 16; o > 0; o >>= 1) my_loss += __shfl_down_sync(0xffffffffu, my_loss, o);
  if ((threadIdx.x & 31) == 0 && loss_sum) atomicAdd(loss_sum, my_loss);
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
                               const float* ref, long long n, float* grid_grad, float* inputs,
                               float* preacts, float* deltas, double* loss_sum, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int threads = 128;
  train_world_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(
      net, params, pos, ref, n, grid_grad, inputs, preacts, deltas, loss_sum);
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
