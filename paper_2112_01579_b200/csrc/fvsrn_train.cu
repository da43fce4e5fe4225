// fvsrn_train.cu -- world-space training step on the GPU.
//
// train_world (train.py:165-206) restated for one batch of positions:
//   forward   assemble_input (model.py:248-279: f64 Fourier phases, f32 trilinear
//             latent lookup grid.py:47-84) -> mlp_forward (nn.py:179-192, f32)
//             -> density / colour head (model.py:342-357)
//   loss      L1 mean and its adjoint sign(diff)/numel (train.py:158-162)
//   backward  head backward (model.py:346-365) -> mlp_backward (nn.py:234-255) ->
//             grid_sample_backward scatter (grid.py:87-137)
// One thread per sample, f32 SIMT for the per-sample passes: this is the training side,
// accuracy before speed (the reference trains in f32; gradients agree to ~1e-6
// relative).  Everything is deterministic, run to run:
//   * the latent-grid scatter is a gather in the reference's own order: every sample
//     writes a record (cell, fractions, keyframe bracket, ordering key) and its adjoint
//     z_bar; records are bucketed by cell (counting sort, per-cell lists sorted by key)
//     and each grid vertex sums its contributions in key order, in the reference's
//     arithmetic (f64 weights x f32 adjoint added to the f32 gradient, grid.py:86-112);
//   * the weight / bias gradients delta_l^T @ [inputs_l | 1] (nn.py:252-253) run on the
//     tensor cores (mma.sync m16n8k8 TF32, 3xTF32 split for f32-level products) over
//     fixed sample chunks, and the chunk partials are summed in chunk order.
// adam_kernel applies adam_step (nn.py:279-298) to the flat parameter buffer laid out
// like FvsrnModel.trainable_arrays() (model.py:155-157).
#include <cuda_runtime.h>

#include <algorithm>
#include <math.h>
#include <stdint.h>

#include "fvsrn_geometry.cuh"
#include "fvsrn_train.cuh"

namespace fvsrn {

namespace {

constexpr int kTrainMaxW = 256;   // widest layer input / output handled per thread
// per-thread activation arrays sized for the network (local memory traffic scales with it)
inline int train_width(const TrainNetDev& n) {
  const int w = n.d_in > n.hidden ? n.d_in : n.hidden;
  return w <= 64 ? 64 : (w <= 128 ? 128 : kTrainMaxW);
}
#define TRAIN_LAUNCH(kern, netv, grid, block, smem, stream, ...)                \
  do {                                                                         \
    const int _w = train_width(netv);                                          \
    if (_w == 64) kern<64><<<grid, block, smem, stream>>>(__VA_ARGS__);        \
    else if (_w == 128) kern<128><<<grid, block, smem, stream>>>(__VA_ARGS__); \
    else kern<kTrainMaxW><<<grid, block, smem, stream>>>(__VA_ARGS__);         \
  } while (0)

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

// Scatter record of one cache row (one sample, or one ray step in screen space): the
// latent cell, its f32 fractions, the keyframe bracket and the reference's ordering key
// (sample index; bracket-pair index above it for temporal models; descending step then
// ray index for raymarch_backward).  key == ~0: the row carries no scatter.
struct ScatterRec {
  unsigned long long key;
  int cell, klo, khi, pad;
  float fx, fy, fz, wk;
};
struct ScatterSink {
  ScatterRec* rec;     // rows
  float* zbar;         // rows x F
};
cudaError_t grid_scatter_det(int R, int F, int G, const ScatterRec* rec, const float* zbar, long long rows,
                             float* grad, cudaStream_t s);
cudaError_t scatter_sink_alloc(const TrainNetDev& net, long long rows, ScatterSink& sk, void*& buf,
                               cudaStream_t s);
cudaError_t scatter_sink_flush(const TrainNetDev& net, const ScatterSink& sk, void* buf, long long rows,
                               float* grid_grad, cudaStream_t s);
__global__ void scatter_records_kernel(int R, const double* __restrict__ pos, long long n,
                                       ScatterRec* __restrict__ rec);

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
template <int W>
__device__ void assemble_f32(const TrainNetDev& net, const float* __restrict__ params, const double (&p)[3],
                             const double* d, double t, float (&x)[W], Cell& cell) {
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
template <int W>
__device__ void mlp_f32(const TrainNetDev& net, const float* __restrict__ params, const CacheRef& c,
                        float (&x)[W], float (&y)[W]) {
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

template <int W>
__device__ void f32_forward(const TrainNetDev& net, const float* __restrict__ params, const double (&p)[3],
                            double t, const CacheRef& c, float (&x)[W], float (&y)[W],
                            Cell& cell) {
  assemble_f32(net, params, p, nullptr, t, x, cell);
  mlp_f32(net, params, c, x, y);
}

// mlp_backward (nn.py:234-255) from raw_bar, writing the adjoints, then the latent-grid
// scatter (grid.py:87-137) of z_bar = x_bar[-F:] as f32 atomics.
template <int W>
__device__ void f32_backward(const TrainNetDev& net, const float* __restrict__ params,
                             const float (&raw_bar)[4], const CacheRef& c, const Cell& cell,
                             const ScatterSink& sink, unsigned long long key, float (&x)[W],
                             float (&y)[W]) {
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
  if (R > 0 && sink.rec) {      // record for the deterministic scatter (grid_scatter_det)
    const int zoff = net.d_in - F;
    float* zb = sink.zbar + c.row * F;
    for (int ch = 0; ch < F; ++ch) zb[ch] = y[zoff + ch];
    ScatterRec r;
    r.key = key;
    r.cell = (cell.x0 * R + cell.y0) * R + cell.z0;
    r.klo = cell.klo;
    r.khi = cell.khi;
    r.pad = 0;
    r.fx = cell.fx; r.fy = cell.fy; r.fz = cell.fz; r.wk = cell.wk;
    sink.rec[c.row] = r;
  }
}

// ordering key of sample i (model.py:318-333 scatters bracket pair by bracket pair, in
// _bracket_pairs order: (k,k) for every k, then (k,k+1))
__device__ __forceinline__ unsigned long long sample_key(const TrainNetDev& net, const Cell& cell,
                                                         long long i) {
  if (net.n_kf == 0) return (unsigned long long)i;
  const int pair = cell.klo == cell.khi ? cell.klo : net.n_kf + cell.klo;
  return ((unsigned long long)pair << 40) | (unsigned long long)i;
}

template <int W>
__global__ void train_world_kernel(TrainNetDev net, const float* __restrict__ params,
                                   const double* __restrict__ pos, const double* __restrict__ times,
                                   const float* __restrict__ ref,
                                   long long n, ScatterSink sink,
                                   float* __restrict__ inputs, float* __restrict__ preacts,
                                   float* __restrict__ deltas, double* __restrict__ loss_sum) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double my_loss = 0.0;
  if (i < n) {
    const int C = net.d_out;
    float x[W], y[W];
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
    f32_backward(net, params, raw_bar, c, cell, sink, sample_key(net, cell, i), x, y);
  }
  // batch L1 loss sum (train.py:158-161): fixed-order block reduction into this block's
  // partial (loss_reduce_kernel adds the partials in block order: deterministic)
  for (int o = 16; o > 0; o >>= 1) my_loss += __shfl_down_sync(0xffffffffu, my_loss, o);
  __shared__ double warp_loss[32];
  if ((threadIdx.x & 31) == 0) warp_loss[threadIdx.x >> 5] = my_loss;
  __syncthreads();
  if (threadIdx.x == 0 && loss_sum) {
    double b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += warp_loss[w];
    loss_sum[blockIdx.x] = b;
  }
}

__global__ void loss_reduce_kernel(const double* __restrict__ part, int nb, double* __restrict__ loss_sum) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[b];
    *loss_sum += s;
  }
}

// mlp_forward / mlp_backward (nn.py:179-193, 234-256) of given inputs x (n, d_in): the
// forward with its caches (layer inputs, hidden pre-activations) and outputs; with y_bar,
// the reverse pass writes the per-layer deltas (weight/bias/input adjoints are the
// caller's GEMMs over the caches).
template <int W>
__global__ void mlp_grads_kernel(TrainNetDev net, const float* __restrict__ params,
                                 const float* __restrict__ x_in, const float* __restrict__ y_bar,
                                 long long n, float* __restrict__ y_out, float* __restrict__ inputs,
                                 float* __restrict__ preacts, float* __restrict__ deltas,
                                 float* __restrict__ x_bar) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float x[W], y[W];
  for (int j = 0; j < net.d_in; ++j) x[j] = x_in[i * net.d_in + j];
  const CacheRef c{inputs, preacts, deltas, i, n};
  mlp_f32(net, params, c, x, y);
  for (int o = 0; o < net.d_out; ++o) y_out[i * net.d_out + o] = y[o];
  if (y_bar) {
    float rb[4] = {0.f, 0.f, 0.f, 0.f};
    for (int o = 0; o < net.d_out && o < 4; ++o) rb[o] = y_bar[i * net.d_out + o];
    const Cell cell{0, 0, 0, 0.f, 0.f, 0.f, 0, 0, 0.f};
    f32_backward(net, params, rb, c, cell, ScatterSink{nullptr, nullptr}, 0ull, x, y);
    if (x_bar)   // input adjoint delta_0 @ W_0 (nn.py:254), per row
      for (int j = 0; j < net.d_in; ++j) x_bar[i * net.d_in + j] = y[j];
  }
}

cudaError_t launch_mlp_grads(const TrainNetDev& net, const float* params, const float* x, const float* y_bar,
                             long long n, float* y_out, float* inputs, float* preacts, float* deltas,
                             float* x_bar, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  TRAIN_LAUNCH(mlp_grads_kernel, net, (unsigned)((n + 127) / 128), 128, 0, s, net, params, x, y_bar, n, y_out, inputs,
                                                                 preacts, deltas, x_bar);
  return cudaGetLastError();
}

cudaError_t launch_grid_scatter(int R, int F, const double* pos, const float* z_bar, long long n,
                                float* grad, cudaStream_t s) {
  // grid_sample_backward (grid.py:123-137): records in sample order, deterministic gather
  if (n <= 0) return cudaSuccess;
  ScatterRec* rec = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&rec, (size_t)n * sizeof(ScatterRec), s);
  if (e != cudaSuccess) return e;
  scatter_records_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(R, pos, n, rec);
  e = grid_scatter_det(R, F, 1, rec, z_bar, n, grad, s);
  cudaFreeAsync(rec, s);
  return e;
}

// model_backward (model.py:300-335): gradients of sum(raw_bar * raw) for given per-sample
// raw-output adjoints (any head, any input encoding incl. view directions).  The forward
// is recomputed with its caches (deterministic, identical to model_forward's); weight /
// bias reductions are GEMMs on the host side, the latent-grid adjoint is scattered here.
template <int W>
__global__ void model_grads_kernel(TrainNetDev net, const float* __restrict__ params,
                                   const double* __restrict__ pos, const double* __restrict__ dirs,
                                   const double* __restrict__ times, const float* __restrict__ raw_bar_in,
                                   long long n, ScatterSink sink,
                                   float* __restrict__ inputs, float* __restrict__ preacts,
                                   float* __restrict__ deltas) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float x[W], y[W];
  const double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
  const CacheRef c{inputs, preacts, deltas, i, n};
  Cell cell;
  assemble_f32(net, params, p, dirs ? dirs + 3 * i : nullptr, times ? times[i] : 0.0, x, cell);
  mlp_f32(net, params, c, x, y);
  float raw_bar[4] = {0.f, 0.f, 0.f, 0.f};
  for (int ch = 0; ch < net.d_out && ch < 4; ++ch) raw_bar[ch] = raw_bar_in[i * net.d_out + ch];
  f32_backward(net, params, raw_bar, c, cell, sink, sample_key(net, cell, i), x, y);
}

cudaError_t launch_model_grads(const TrainNetDev& net, const float* params, const double* pos,
                               const double* dirs, const double* times, const float* raw_bar, long long n,
                               float* grid_grad, float* inputs, float* preacts, float* deltas,
                               cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int threads = 128;
  ScatterSink sk;
  void* sbuf = nullptr;
  cudaError_t e = scatter_sink_alloc(net, grid_grad ? n : 0, sk, sbuf, s);
  if (e != cudaSuccess) return e;
  TRAIN_LAUNCH(model_grads_kernel, net, (unsigned)((n + threads - 1) / threads), threads, 0, s, 
      net, params, pos, dirs, times, raw_bar, n, sk, inputs, preacts, deltas);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return scatter_sink_flush(net, sk, sbuf, n, grid_grad, s);
}

// ---------------------------------------------------------------- screen space
// raymarch_forward(ModelSource(colour model), want_states=True) (render.py:203-238):
// f64 geometry and compositing, f32 model evaluation (the naive ModelSource path), no
// early termination; terminal (C, A) and the per-ray geometry are kept for backward.
template <int W>
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
  float x[W], y[W];
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
template <int W>
__global__ void screen_backward_kernel(TrainNetDev net, const float* __restrict__ params,
                                       const double* __restrict__ org, const double* __restrict__ dir,
                                       long long n, double eps_blend, const double* __restrict__ cst,
                                       const double* __restrict__ ast, const double* __restrict__ tmin_a,
                                       const double* __restrict__ ds_a, const int* __restrict__ nsteps,
                                       const long long* __restrict__ row_off, const float* __restrict__ adj,
                                       const double* __restrict__ bg, long long cap,
                                       float* __restrict__ inputs, float* __restrict__ preacts,
                                       float* __restrict__ deltas, ScatterSink sink) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int ns = nsteps[i];
  if (ns == 0) return;
  double c_acc[3] = {cst[3 * i], cst[3 * i + 1], cst[3 * i + 2]};
  double a_acc = ast[i];
  const double tmin = tmin_a[i], ds = ds_a[i];
  double c_bar[3] = {(double)adj[4 * i], (double)adj[4 * i + 1], (double)adj[4 * i + 2]};
  double a_bar = (double)adj[4 * i + 3] - (c_bar[0] * bg[0] + c_bar[1] * bg[1] + c_bar[2] * bg[2]);
  float x[W], y[W];
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
    // raymarch_backward walks the steps from the last to the first and, per step, the
    // active rays in index order (render.py:257-306): that is the scatter order
    f32_backward(net, params, raw_bar, c, cell, sink,
                 ((unsigned long long)(0x7fffffff - k) << 32) | (unsigned long long)i, x, y);
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
  ScatterSink sk;
  void* sbuf = nullptr;
  cudaError_t e = scatter_sink_alloc(net, grid_grad ? n : 0, sk, sbuf, s);
  if (e != cudaSuccess) return e;
  const unsigned blocks = (unsigned)((n + threads - 1) / threads);
  double* part = nullptr;
  if (loss_sum && (e = cudaMallocAsync((void**)&part, blocks * sizeof(double), s)) != cudaSuccess) return e;
  TRAIN_LAUNCH(train_world_kernel, net, blocks, threads, 0, s, net, params, pos, times, ref, n, sk, inputs, preacts,
                                                deltas, part);
  if (loss_sum) {
    loss_reduce_kernel<<<1, 32, 0, s>>>(part, (int)blocks, loss_sum);
    cudaFreeAsync(part, s);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return scatter_sink_flush(net, sk, sbuf, n, grid_grad, s);
}

cudaError_t launch_screen_forward(const TrainNetDev& net, const float* params, const double* org,
                                  const double* dir, long long n, const MarchDev& md, float* px,
                                  double* cst, double* ast, double* tmin, double* ds, int* nsteps,
                                  cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  TRAIN_LAUNCH(screen_forward_kernel, net, (unsigned)((n + 63) / 64), 64, 0, s, net, params, org, dir, n, md, px, cst,
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
  ScatterSink sk;
  void* sbuf = nullptr;
  cudaError_t e = scatter_sink_alloc(net, grid_grad ? cap : 0, sk, sbuf, s);
  if (e != cudaSuccess) return e;
  TRAIN_LAUNCH(screen_backward_kernel, net, (unsigned)((n + 63) / 64), 64, 0, s, 
      net, params, org, dir, n, eps_blend, cst, ast, tmin, ds, nsteps, row_off, adj, bg, cap, inputs,
      preacts, deltas, sk);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return scatter_sink_flush(net, sk, sbuf, cap, grid_grad, s);
}

// Reference-semantics f32 evaluation of the pieces of the model (stage 0: assembled
// inputs, 1: latent vectors (grid_sample / keyframe_sample), 2: raw MLP outputs from
// positions, 3: raw MLP outputs of given inputs x (mlp_eval)).
template <int W>
__global__ void f32_eval_kernel(TrainNetDev net, const float* __restrict__ params,
                                const double* __restrict__ pos, const double* __restrict__ dirs,
                                const double* __restrict__ times,
                                const float* __restrict__ xin, long long n, int stage,
                                float* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float x[W], y[W];
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
  TRAIN_LAUNCH(f32_eval_kernel, net, (unsigned)((n + 127) / 128), 128, 0, s, net, params, pos, dirs, times, xin, n, stage,
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

// ---------------------------------------------------------------- deterministic scatter
// grid_sample_backward (grid.py:86-137) without atomics on the gradient: the records of
// every contributing row are bucketed by (grid, cell) -- integer counts, a prefix sum, a
// fill and a per-cell sort by ordering key make the buckets deterministic -- and each
// grid vertex then merges the (up to 8) buckets of the cells it is a corner of, in key
// order, accumulating in the reference's arithmetic (numba's promotions of its f32/f64
// mix, see the gather kernel): bit-identical to the sequential reference loop.
// Temporal rows contribute (1 - wk) * zb to keyframe klo and wk * zb to khi (f32,
// model.py:318-333).  Bit-identical run to run.
namespace {

struct ScatterEnt {
  unsigned long long key2;   // key * 2 + which (0: klo, 1: khi)
  int row, pad;
};

__global__ void scatter_count_kernel(const ScatterRec* __restrict__ rec, long long rows, int R3,
                                     int* __restrict__ cnt) {
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x) {
    const ScatterRec e = rec[r];
    if (e.key == ~0ull) continue;
    atomicAdd(cnt + (long long)e.klo * R3 + e.cell, 1);
    if (e.khi != e.klo) atomicAdd(cnt + (long long)e.khi * R3 + e.cell, 1);
  }
}

__global__ void scatter_fill_kernel(const ScatterRec* __restrict__ rec, long long rows, int R3,
                                    const int* __restrict__ off, int* __restrict__ cur,
                                    ScatterEnt* __restrict__ ent) {
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x) {
    const ScatterRec e = rec[r];
    if (e.key == ~0ull) continue;
    long long c = (long long)e.klo * R3 + e.cell;
    ent[off[c] + atomicAdd(cur + c, 1)] = ScatterEnt{e.key * 2, (int)r, 0};
    if (e.khi != e.klo) {
      c = (long long)e.khi * R3 + e.cell;
      ent[off[c] + atomicAdd(cur + c, 1)] = ScatterEnt{e.key * 2 + 1, (int)r, 0};
    }
  }
}

// per bucket: insertion sort by key2 (buckets hold a few entries each)
__global__ void scatter_sort_kernel(const int* __restrict__ off, long long n_buckets,
                                    ScatterEnt* __restrict__ ent) {
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < n_buckets;
       b += (long long)gridDim.x * blockDim.x) {
    const int lo = off[b], hi = off[b + 1];
    for (int i = lo + 1; i < hi; ++i) {
      const ScatterEnt v = ent[i];
      int j = i - 1;
      while (j >= lo && ent[j].key2 > v.key2) { ent[j + 1] = ent[j]; --j; }
      ent[j + 1] = v;
    }
  }
}

// one thread per (grid, vertex): merge the buckets of the <= 8 cells touching the vertex
template <int FC>
__global__ void scatter_gather_kernel(const ScatterRec* __restrict__ rec, const float* __restrict__ zbar,
                                      const int* __restrict__ off, const ScatterEnt* __restrict__ ent,
                                      int R, int F, int G, float* __restrict__ grad) {
  const long long R3 = (long long)R * R * R;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < (long long)G * R3;
       t += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(t / R3);
    const long long v = t % R3;
    const int vx = (int)(v / ((long long)R * R)), vy = (int)((v / R) % R), vz = (int)(v % R);
    int head[8], end[8], corner[8], nb = 0;
    for (int q = 0; q < 8; ++q) {
      const int a = (q >> 2) & 1, b = (q >> 1) & 1, c = q & 1;
      const int cx = vx - a, cy = vy - b, cz = vz - c;
      if (cx < 0 || cy < 0 || cz < 0 || cx > R - 2 || cy > R - 2 || cz > R - 2) continue;
      const long long bkt = (long long)g * R3 + ((long long)cx * R + cy) * R + cz;
      if (off[bkt] == off[bkt + 1]) continue;
      head[nb] = off[bkt]; end[nb] = off[bkt + 1]; corner[nb] = q; ++nb;
    }
    if (nb == 0) continue;
    for (int c0 = 0; c0 < F; c0 += FC) {
      float acc[FC];
      float* gp = grad + (g * R3 + v) * F + c0;
#pragma unroll
      for (int ch = 0; ch < FC; ++ch) acc[ch] = (c0 + ch < F) ? gp[ch] : 0.f;
      int h[8];
      for (int k = 0; k < nb; ++k) h[k] = head[k];
      while (true) {
        int best = -1;
        unsigned long long bk = ~0ull;
        for (int k = 0; k < nb; ++k)
          if (h[k] < end[k] && ent[h[k]].key2 < bk) { bk = ent[h[k]].key2; best = k; }
        if (best < 0) break;
        const ScatterEnt e = ent[h[best]++];
        const ScatterRec r = rec[e.row];
        const int q = corner[best];
        // grid.py:92-112 with numba's type promotion: gx = 1.0 - fx is f64 (f64 literal),
        // fx is f32, so a product stays f32 while both factors are f32: w110 = f32(fx*fy)*gz
        // is f64 but w111 = fx*fy*fz is f32, and its w111 * zb product and the += are f32;
        // every other corner multiplies and accumulates in f64 (cast to f32 on store)
        const bool two = r.khi != r.klo;
        const float fac = two ? ((e.key2 & 1) ? r.wk : __fsub_rn(1.f, r.wk)) : 1.f;
        const float* zb = zbar + (long long)e.row * F + c0;
        if (q == 7) {
          const float w = __fmul_rn(__fmul_rn(r.fx, r.fy), r.fz);
#pragma unroll
          for (int ch = 0; ch < FC; ++ch) {
            if (c0 + ch >= F) break;
            const float z = two ? __fmul_rn(fac, zb[ch]) : zb[ch];
            acc[ch] = __fadd_rn(acc[ch], __fmul_rn(w, z));
          }
        } else {
          const double gx = __dsub_rn(1.0, (double)r.fx), gy = __dsub_rn(1.0, (double)r.fy),
                       gz = __dsub_rn(1.0, (double)r.fz);
          const double xy = q == 6 ? (double)__fmul_rn(r.fx, r.fy)
                                   : __dmul_rn((q & 4) ? (double)r.fx : gx, (q & 2) ? (double)r.fy : gy);
          const double w = __dmul_rn(xy, (q & 1) ? (double)r.fz : gz);
#pragma unroll
          for (int ch = 0; ch < FC; ++ch) {
            if (c0 + ch >= F) break;
            const float z = two ? __fmul_rn(fac, zb[ch]) : zb[ch];
            acc[ch] = (float)__dadd_rn((double)acc[ch], __dmul_rn(w, (double)z));
          }
        }
      }
#pragma unroll
      for (int ch = 0; ch < FC; ++ch)
        if (c0 + ch < F) gp[ch] = acc[ch];
    }
  }
}

// exclusive prefix sum of n ints (3 passes: per-block scan, block totals, add)
constexpr int kScanBlock = 1024;
__global__ void scan_blocks_kernel(const int* __restrict__ in, long long n, int* __restrict__ out,
                                   int* __restrict__ totals) {
  __shared__ int sh[kScanBlock];
  const long long i = (long long)blockIdx.x * kScanBlock + threadIdx.x;
  const int v = i < n ? in[i] : 0;
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int d = 1; d < kScanBlock; d <<= 1) {
    const int t = threadIdx.x >= d ? sh[threadIdx.x - d] : 0;
    __syncthreads();
    sh[threadIdx.x] += t;
    __syncthreads();
  }
  if (i < n) out[i] = sh[threadIdx.x] - v;
  if (threadIdx.x == kScanBlock - 1) totals[blockIdx.x] = sh[threadIdx.x];
}

__global__ void scan_totals_kernel(int* __restrict__ totals, int nb, int* __restrict__ grand) {
  if (threadIdx.x == 0) {       // nb <= a few thousand: sequential and deterministic
    int run = 0;
    for (int b = 0; b < nb; ++b) { const int t = totals[b]; totals[b] = run; run += t; }
    *grand = run;
  }
}

__global__ void scan_add_kernel(int* __restrict__ out, long long n, const int* __restrict__ totals,
                                const int* __restrict__ grand) {
  const long long i = (long long)blockIdx.x * kScanBlock + threadIdx.x;
  if (i < n) out[i] += totals[blockIdx.x];
  if (i == n) out[n] = *grand;
}

}  // namespace

cudaError_t grid_scatter_det(int R, int F, int G, const ScatterRec* rec, const float* zbar, long long rows,
                             float* grad, cudaStream_t s) {
  if (rows <= 0 || R < 2 || !grad) return cudaSuccess;
  const long long R3 = (long long)R * R * R, nbk = (long long)G * R3;
  const long long nblk = (nbk + 1 + kScanBlock - 1) / kScanBlock;
  char* buf = nullptr;
  const size_t ints = (size_t)(3 * (nbk + 1) + nblk + 1);
  cudaError_t e = cudaMallocAsync((void**)&buf, ints * sizeof(int) + (size_t)2 * rows * sizeof(ScatterEnt), s);
  if (e != cudaSuccess) return e;
  int* cnt = (int*)buf;
  int* off = cnt + (nbk + 1);
  int* cur = off + (nbk + 1);
  int* totals = cur + (nbk + 1);
  ScatterEnt* ent = (ScatterEnt*)(buf + ints * sizeof(int) + (ints * sizeof(int)) % 16);
  ent = (ScatterEnt*)(((uintptr_t)(buf + ints * sizeof(int)) + 15) & ~(uintptr_t)15);
  cudaMemsetAsync(cnt, 0, sizeof(int) * (nbk + 1), s);
  cudaMemsetAsync(cur, 0, sizeof(int) * (nbk + 1), s);
  const int th = 256;
  const unsigned gr = (unsigned)std::min<long long>((rows + th - 1) / th, 148 * 16);
  scatter_count_kernel<<<gr, th, 0, s>>>(rec, rows, (int)R3, cnt);
  scan_blocks_kernel<<<(unsigned)nblk, kScanBlock, 0, s>>>(cnt, nbk + 1, off, totals);
  scan_totals_kernel<<<1, 32, 0, s>>>(totals, (int)nblk, totals + nblk);
  scan_add_kernel<<<(unsigned)nblk, kScanBlock, 0, s>>>(off, nbk, totals, totals + nblk);
  scatter_fill_kernel<<<gr, th, 0, s>>>(rec, rows, (int)R3, off, cur, ent);
  const unsigned gb = (unsigned)std::min<long long>((nbk + th - 1) / th, 148 * 32);
  scatter_sort_kernel<<<gb, th, 0, s>>>(off, nbk, ent);
  if (F <= 8)
    scatter_gather_kernel<8><<<gb, th, 0, s>>>(rec, zbar, off, ent, R, F, G, grad);
  else
    scatter_gather_kernel<16><<<gb, th, 0, s>>>(rec, zbar, off, ent, R, F, G, grad);
  e = cudaGetLastError();
  cudaFreeAsync(buf, s);
  return e;
}

// rows' scatter scratch: records (key = ~0 until written) + adjoints
cudaError_t scatter_sink_alloc(const TrainNetDev& net, long long rows, ScatterSink& sk, void*& buf,
                               cudaStream_t s) {
  sk = ScatterSink{nullptr, nullptr};
  buf = nullptr;
  if (net.grid_res <= 0 || rows <= 0) return cudaSuccess;
  const size_t rb = (size_t)rows * sizeof(ScatterRec);
  cudaError_t e = cudaMallocAsync(&buf, rb + (size_t)rows * net.grid_ch * sizeof(float), s);
  if (e != cudaSuccess) return e;
  sk.rec = (ScatterRec*)buf;
  sk.zbar = (float*)((char*)buf + rb);
  return cudaMemsetAsync(sk.rec, 0xff, rb, s);
}

cudaError_t scatter_sink_flush(const TrainNetDev& net, const ScatterSink& sk, void* buf, long long rows,
                               float* grid_grad, cudaStream_t s) {
  if (!buf) return cudaSuccess;
  cudaError_t e = grid_scatter_det(net.grid_res, net.grid_ch, net.n_kf > 0 ? net.n_kf : 1, sk.rec, sk.zbar,
                                   rows, grid_grad, s);
  cudaFreeAsync(buf, s);
  return e;
}

// grid_sample_backward of given positions / adjoints (one grid): records in sample order
__global__ void scatter_records_kernel(int R, const double* __restrict__ pos, long long n,
                                       ScatterRec* __restrict__ rec) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double sc = (double)(R - 1);
  const double cx = fmin(fmax(pos[3 * i], 0.0), 1.0) * sc, cy = fmin(fmax(pos[3 * i + 1], 0.0), 1.0) * sc,
               cz = fmin(fmax(pos[3 * i + 2], 0.0), 1.0) * sc;
  const int x0 = min((int)cx, R - 2), y0 = min((int)cy, R - 2), z0 = min((int)cz, R - 2);
  ScatterRec r;
  r.key = (unsigned long long)i;
  r.cell = (x0 * R + y0) * R + z0;
  r.klo = r.khi = 0;
  r.pad = 0;
  r.fx = (float)(cx - x0); r.fy = (float)(cy - y0); r.fz = (float)(cz - z0); r.wk = 0.f;
  rec[i] = r;
}

// ---------------------------------------------------------------- weight gradients
// dW_l = delta_l^T @ inputs_l, db_l = sum_rows delta_l (nn.py:252-253) for every layer:
// C (wo x (wi+1)) = D^T [X | 1] on the tensor cores, mma.sync m16n8k8 TF32 with the
// 3xTF32 split (v = hi + lo, hi = tf32(v), lo = tf32(v - hi); C += lo*hi + hi*lo + hi*hi)
// so the products keep ~f32 precision.  CTA (chunk, layer) reduces the fixed sample
// chunk into its own partial; wg_reduce sums the partials in chunk order: deterministic.
namespace {

constexpr int kWgChunk = 256;

__device__ __forceinline__ uint32_t tf32_of(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return r;
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

struct WgLayer {
  const float* x;      // n x wi
  const float* d;      // n x wo
  int wi, wo;
  long long part;      // float offset of this layer's partials (chunks x wo x (wi+1))
};
struct WgArgs {
  WgLayer l[kTrainMaxLayers];
  long long n;
  int chunks;
};

__global__ void __launch_bounds__(128) wg_partial_kernel(WgArgs a, float* __restrict__ partial) {
  const WgLayer L = a.l[blockIdx.y];
  const int chunk = blockIdx.x;
  const long long s0 = (long long)chunk * kWgChunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wn = L.wi + 1;
  const int mt = (L.wo + 15) / 16, nt = (wn + 7) / 8;
  float* out = partial + L.part + (long long)chunk * L.wo * wn;
  for (int tile = warp; tile < mt * nt; tile += 4) {
    const int m0 = (tile / nt) * 16, n0 = (tile % nt) * 8;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k0 = 0; k0 < kWgChunk; k0 += 8) {
      const long long r0 = s0 + k0 + t4, r1 = r0 + 4;
      const bool v0 = r0 < a.n, v1 = r1 < a.n;
      // A = D^T (m = output feature, k = sample): a0 (g, t4) a1 (g+8, t4) a2 (g, t4+4) a3 (g+8, t4+4)
      const int ma = m0 + g, mb = m0 + g + 8;
      const float av[4] = {v0 && ma < L.wo ? L.d[r0 * L.wo + ma] : 0.f, v0 && mb < L.wo ? L.d[r0 * L.wo + mb] : 0.f,
                           v1 && ma < L.wo ? L.d[r1 * L.wo + ma] : 0.f, v1 && mb < L.wo ? L.d[r1 * L.wo + mb] : 0.f};
      // B = [X | 1] (k = sample, n = input feature): b0 (k t4, n g), b1 (k t4+4, n g)
      const int nb = n0 + g;
      const float bv[2] = {v0 ? (nb < L.wi ? L.x[r0 * L.wi + nb] : (nb == L.wi ? 1.f : 0.f)) : 0.f,
                           v1 ? (nb < L.wi ? L.x[r1 * L.wi + nb] : (nb == L.wi ? 1.f : 0.f)) : 0.f};
      uint32_t ah[4], al[4], bh[2], bl[2];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ah[q] = tf32_of(av[q]);
        al[q] = tf32_of(av[q] - __uint_as_float(ah[q]));
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        bh[q] = tf32_of(bv[q]);
        bl[q] = tf32_of(bv[q] - __uint_as_float(bh[q]));
      }
      mma_tf32(acc, al, bh);
      mma_tf32(acc, ah, bl);
      mma_tf32(acc, ah, bh);
    }
    // c0,c1: (row g, cols 2t4, 2t4+1); c2,c3: (row g+8, ...)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int m = m0 + g + (q >> 1) * 8, nn = n0 + 2 * t4 + (q & 1);
      if (m < L.wo && nn < wn) out[(long long)m * wn + nn] = acc[q];
    }
  }
}

struct WgOut {
  long long w_off[kTrainMaxLayers], b_off[kTrainMaxLayers], part[kTrainMaxLayers];
  int wi[kTrainMaxLayers], wo[kTrainMaxLayers];
  long long first[kTrainMaxLayers + 1];    // output-element prefix over layers
  int layers, chunks, accumulate;
};

__global__ void wg_reduce_kernel(WgOut o, const float* __restrict__ partial, float* __restrict__ grads) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < o.first[o.layers];
       e += (long long)gridDim.x * blockDim.x) {
    int l = 0;
    while (e >= o.first[l + 1]) ++l;
    const long long k = e - o.first[l];
    const int wn = o.wi[l] + 1;
    const int m = (int)(k / wn), c = (int)(k % wn);
    const long long stride = (long long)o.wo[l] * wn;
    float sum = 0.f;
    for (int ch = 0; ch < o.chunks; ++ch) sum += partial[o.part[l] + ch * stride + k];
    float* dst = c < o.wi[l] ? grads + o.w_off[l] + (long long)m * o.wi[l] + c : grads + o.b_off[l] + m;
    *dst = o.accumulate ? __fadd_rn(*dst, sum) : sum;
  }
}

}  // namespace

cudaError_t launch_layer_grads(const TrainNetDev& net, const float* inputs, const float* deltas, long long n,
                               float* grads, bool accumulate, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int L = net.layers;
  WgArgs a{};
  WgOut o{};
  a.n = n;
  a.chunks = o.chunks = (int)((n + kWgChunk - 1) / kWgChunk);
  o.layers = L;
  o.accumulate = accumulate ? 1 : 0;
  long long part = 0, first = 0;
  for (int l = 0; l < L; ++l) {
    const int wi = l == 0 ? net.d_in : net.hidden, wo = l == L - 1 ? net.d_out : net.hidden;
    a.l[l] = WgLayer{inputs + net.in_off[l], deltas + net.d_off[l], wi, wo, part};
    o.w_off[l] = net.w_off[l];
    o.b_off[l] = net.b_off[l];
    o.part[l] = part;
    o.wi[l] = wi;
    o.wo[l] = wo;
    o.first[l] = first;
    part += (long long)a.chunks * wo * (wi + 1);
    first += (long long)wo * (wi + 1);
  }
  o.first[L] = first;
  float* partial = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&partial, (size_t)part * sizeof(float), s);
  if (e != cudaSuccess) return e;
  wg_partial_kernel<<<dim3((unsigned)a.chunks, (unsigned)L), 128, 0, s>>>(a, partial);
  wg_reduce_kernel<<<(unsigned)std::min<long long>((first + 255) / 256, 1024), 256, 0, s>>>(o, partial, grads);
  e = cudaGetLastError();
  cudaFreeAsync(partial, s);
  return e;
}

}  // namespace fvsrn
