// fvsrn_train.cuh -- world-space training step (fvsrn_train.cu).
#pragma once
#include <cuda_runtime.h>

#include "fvsrn_kernels.cuh"

namespace fvsrn {

constexpr int kTrainMaxLayers = 24;

// Network + encoder description of a static, position-input model; every offset is in
// floats.  params: [W_0 .. W_{L-1} | b_0 .. b_{L-1} | grid] (model.py:155-157 order).
// inputs / deltas: per-layer blocks of N x in_l / N x out_l floats; preacts (L-1) x N x H.
struct TrainNetDev {
  int layers, hidden, d_in, d_out, act, head;
  int m;                    // spatial Fourier rows (B is m x fd_in, f32)
  int raw_w, fd_in;         // raw input block (3: p, 6: p|d) and Fourier input width
  const float* bmat;
  int grid_res, grid_ch;
  long long grid_off;           // first grid; keyframe k at grid_off + k * R^3 * F
  // temporal models (model.py:190-245): keyframe times, time features
  int n_kf;                     // 0: static
  double kf_times[16];
  int time_mode;                // 0 none, 1 direct, 2 fourier, 3 both
  int time_l;                   // fourier rows (time_fourier_count)
  float time_b[16];             // time encoder B (L x 1)
  double t0, t1;                // normalisation span
  long long w_off[kTrainMaxLayers], b_off[kTrainMaxLayers];
  long long in_off[kTrainMaxLayers], d_off[kTrainMaxLayers];
};

struct AdamConsts {
  float lr, b1, b2, one_m_b1, one_m_b2, eps, bc1, bc2;
};

cudaError_t launch_mlp_grads(const TrainNetDev& net, const float* params, const float* x, const float* y_bar,
                             long long n, float* y_out, float* inputs, float* preacts, float* deltas,
                             float* x_bar, cudaStream_t s);
cudaError_t launch_grid_scatter(int R, int F, const double* pos, const float* z_bar, long long n,
                                float* grad, cudaStream_t s);
cudaError_t launch_model_grads(const TrainNetDev& net, const float* params, const double* pos,
                               const double* dirs, const double* times, const float* raw_bar, long long n,
                               float* grid_grad, float* inputs, float* preacts, float* deltas,
                               cudaStream_t s);
cudaError_t launch_train_world(const TrainNetDev& net, const float* params, const double* pos,
                               const double* times, const float* ref, long long n, float* grid_grad, float* inputs,
                               float* preacts, float* deltas, double* loss_sum, cudaStream_t s);
cudaError_t launch_screen_forward(const TrainNetDev& net, const float* params, const double* org,
                                  const double* dir, long long n, const MarchDev& md, float* px,
                                  double* cst, double* ast, double* tmin, double* ds, int* nsteps,
                                  cudaStream_t s);
cudaError_t launch_screen_backward(const TrainNetDev& net, const float* params, const double* org,
                                   const double* dir, long long n, double eps_blend, const double* cst,
                                   const double* ast, const double* tmin, const double* ds,
                                   const int* nsteps, const long long* row_off, const float* adj,
                                   const double* bg, long long cap, float* inputs, float* preacts,
                                   float* deltas, float* grid_grad, cudaStream_t s);
cudaError_t launch_f32_eval(const TrainNetDev& net, const float* params, const double* pos,
                            const double* dirs, const double* times, const float* xin, long long n,
                            int stage, float* out, cudaStream_t s);
// dW_l / db_l of every layer from the caches (deterministic, tensor cores), written to
// (or, with accumulate, added into) the flat gradient buffer at the w_off / b_off offsets
cudaError_t launch_layer_grads(const TrainNetDev& net, const float* inputs, const float* deltas, long long n,
                               float* grads, bool accumulate, cudaStream_t s);
cudaError_t launch_adam(float* p, const float* g, float* m, float* v, long long n, const AdamConsts& k,
                        unsigned long long* bad, cudaStream_t s);

}  // namespace fvsrn
