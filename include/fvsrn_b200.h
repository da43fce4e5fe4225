/*
 * fvsrn_b200.h -- C ABI of the B200-native fV-SRN direct-volume-rendering path.
 *
 * The reference (`fvsrn` 0.1.0, /root/reference/pkg/src/fvsrn) is pure Python;
 * its seams for this path are Python protocols, not a C ABI.  Each entry point
 * below replaces one of them (citations are reference file:line):
 *
 *   fvsrn_model_create      <- model upload implied by ModelSource.__init__       render.py:147-166
 *                              (weights/B/grid(s) of FvsrnModel                   model.py:136-162)
 *   fvsrn_render            <- render_image(ModelSource(...), camera, settings)   render.py:314-332
 *   fvsrn_render_device     <- same, device framebuffer / screen-tile subset      (multi-GPU)
 *   fvsrn_render_multi      <- same, split over several GPUs of one process       (SURVEY 8b device_ids[])
 *   fvsrn_render_rays       <- raymarch_forward(source, origins, dirs, settings)  render.py:203-238
 *   fvsrn_eval_density      <- eval_density(model, p, t)                          model.py:368-373
 *   fvsrn_eval_color        <- eval_color(model, p, d, t)                         model.py:376-382
 *   fvsrn_decode_density    <- decode_volume(model, resolution, t)                model.py:385-398
 *   fvsrn_decode_density_multi <- same, lattice slabs over several GPUs            (SURVEY 8b n_devices)
 *   fvsrn_fused_eval        <- fused_eval(plan, model, x)                         fused.py:281-301
 *   fvsrn_volume_*          <- render_image / raymarch_forward on a VolumeSource  render.py:132-141
 *   fvsrn_render_rgba8      <- png_bytes(render_image(...)) pixels (service)      imaging.py:74-80
 *   fvsrn_train_*, fvsrn_adam_step <- train_world / train_temporal / train_screen batch
 *                              steps and adam_step      train.py:165-314, render.py:241-306, nn.py:279-298
 *   fvsrn_ipc_*             <- (new) multi-GPU frame assembly in peer memory
 *
 * Conventions: every function returns an fvsrn_status; on failure
 * fvsrn_last_error() (thread-local) holds a message.  Host-pointer variants are
 * synchronous and copy results back; *_device variants take device pointers and
 * a cudaStream_t (passed as void*) and are stream-ordered.  No function keeps a
 * reference to caller memory after returning.  A model handle is immutable
 * after creation and may be used concurrently from several host threads
 * (per-call stream-ordered scratch, no global mutable state).
 *
 * There is no CPU fallback: without an sm_100a device every compute call fails
 * with FVSRN_ECUDA.
 */
#ifndef FVSRN_B200_H
#define FVSRN_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define FVSRN_API __attribute__((visibility("default")))
#else
#define FVSRN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FVSRN_OK = 0,
  FVSRN_EINVAL = 1,     /* contract violation      -> ValueError   */
  FVSRN_ECAPACITY = 2,  /* network too large        -> CapacityError */
  FVSRN_ECUDA = 3,      /* CUDA / device failure    -> RuntimeError */
  FVSRN_ENOMEM = 4
} fvsrn_status;

/* nn.py:15 ACTIVATION_KINDS order */
enum { FVSRN_ACT_RELU = 0, FVSRN_ACT_SIGMOID = 1, FVSRN_ACT_SOFTPLUS = 2,
       FVSRN_ACT_SNAKE = 3, FVSRN_ACT_SNAKE_ALT = 4 };
enum { FVSRN_HEAD_DENSITY = 0, FVSRN_HEAD_COLOR = 1 };              /* model.py:73 */
enum { FVSRN_DIR_POS = 0, FVSRN_DIR_P = 1, FVSRN_DIR_F = 2 };       /* model.py:46 */
enum { FVSRN_TIME_NONE = 0, FVSRN_TIME_DIRECT = 1, FVSRN_TIME_FOURIER = 2,
       FVSRN_TIME_BOTH = 3 };                                          /* model.py:47 */
enum { FVSRN_FOURIER_OFF = 0, FVSRN_FOURIER_NERF = 1, FVSRN_FOURIER_RANDOM = 2 };
enum { FVSRN_GRID_F32 = 0, FVSRN_GRID_U8 = 1 };                      /* model.py:430-472 */

typedef struct fvsrn_model* fvsrn_model_t;

/* Everything FvsrnModel holds (model.py:136-162), as plain arrays. */
typedef struct {
  int32_t layers, hidden, d_in, d_out;     /* d_in = ModelConfig.input_width  */
  int32_t activation, head, direction_mode;
  int32_t fourier_mode, fourier_m, fourier_d_in;
  const float* b_matrix;                   /* (fourier_m, fourier_d_in) f32    */
  int32_t time_mode, time_fourier_count;
  const float* time_b;                     /* (time_fourier_count,) f32 or NULL */
  int32_t has_time_range; double time_range[2];
  int32_t grid_resolution, grid_channels;  /* 0 disables the latent grid       */
  int32_t n_grids;                         /* 1 static, or #keyframes          */
  const double* keyframe_times;            /* n_grids entries if temporal      */
  int32_t temporal;                        /* keyframe model?                  */
  int32_t grid_precision;                  /* FVSRN_GRID_F32 | FVSRN_GRID_U8   */
  const float* const* grids;               /* n_grids x (R,R,R,F) f32 (F32)    */
  const uint8_t* const* grid_codes;        /* n_grids x (R,R,R,F) u8   (U8)    */
  const float* const* grid_mins;           /* n_grids x (F,) f32       (U8)    */
  const float* const* grid_maxs;           /* n_grids x (F,) f32       (U8)    */
  const float* const* weights;             /* layers x (out,in) f32 row-major  */
  const float* const* biases;              /* layers x (out,)       f32        */
} fvsrn_model_desc;

/* TransferFunction (transfer.py:11-54); n <= 64 control points. */
typedef struct { int32_t n; const float* xs; const float* rgbs; const float* sigmas; } fvsrn_tf;

/* Camera (imaging.py:14-42).  has_basis != 0: the caller supplies the per-frame
 * basis of render.py:78-86 (forward, right, up', tan(fov/2)*W/H, tan(fov/2))
 * computed with the reference's own numpy ops, making per-pixel rays bit-exact. */
typedef struct {
  double eye[3], target[3], up[3]; double fov_y; int32_t width, height;
  int32_t has_basis; double b_forward[3], b_right[3], b_up[3]; double half_w, half_h;
} fvsrn_camera;

/* RenderSettings (render.py:49-69). */
typedef struct {
  double stepsize; int32_t max_steps; double background[3];
  double early_term_alpha; double eps_blend;
} fvsrn_settings;

/* Screen-tile shard: this call renders tiles t = rank + k*world (8x8 px tiles,
 * row-major tile order).  compact != 0 writes slot-ordered output
 * (n_local_tiles*64 RGBA px) instead of the row-major frame. */
typedef struct { int32_t rank, world, compact; } fvsrn_shard;

FVSRN_API const char* fvsrn_last_error(void);
FVSRN_API const char* fvsrn_version(void);
FVSRN_API int32_t fvsrn_device_count(void);
/* DVR kernel selection for the default fV-SRN shapes (no reference counterpart: a
 * measurement / A-B switch; the environment variable FVSRN_DVR sets the initial value).
 * 0 auto (measured faster per width), 1 tcgen05/TMEM, 2 warp-specialised mma.sync,
 * 3 single-role mma.sync (4 pipelined, 5 two rays per lane, 2 warp-specialised: A/B builds
 * only).  Returns the previous mode, or -FVSRN_EINVAL (negative) on failure. */
FVSRN_API int32_t fvsrn_set_dvr_kernel(int32_t mode);
/* Latent-grid sampler for 16-channel grids (measurement switch; env FVSRN_GRID sets the
 * initial value): 0 auto, 1 texture units (RGBA16F 3D textures, hardware trilinear),
 * 2 LDG.128 + HFMA2 trilinear.  Returns the previous mode, or -FVSRN_EINVAL on failure. */
FVSRN_API int32_t fvsrn_set_grid_sampler(int32_t mode);
/* Measurement hooks (bench.py): per calling thread, CUDA events around every launch of
 * the dominant kernel (march / decode) and a count of all library kernel launches.
 * fvsrn_kernel_timer(1) enables and resets; _read synchronizes the recorded events and
 * returns the summed dominant-kernel time, its launch count and the total launch count
 * since the last read, then resets. */
FVSRN_API int32_t fvsrn_kernel_timer(int32_t enable);
FVSRN_API int32_t fvsrn_kernel_timer_read(double* dominant_ms, int64_t* dominant_launches,
                                          int64_t* total_launches);
/* The last kernel the timer recorded on this thread: template instantiation, MMA path and
 * latent-grid sampler (e.g. "dvr_kernel<32,4,14,4> (mma.sync m16n8k16); grid: texture
 * units, RGBA16F, ...").  NUL-terminated, truncated to cap bytes. */
FVSRN_API int32_t fvsrn_kernel_timer_info(char* buf, int32_t cap);

/* ---- world-space training (train.py:165-206), device pointers only.
 * A static, position-input model (time_mode none, direction_mode pos).  The trainable
 * parameters live in ONE flat f32 buffer in FvsrnModel.trainable_arrays() order
 * (model.py:155-157): W_0..W_{L-1} as (out,in) row-major, b_0..b_{L-1}, then the
 * (R,R,R,F) grid.  Gradients use the same layout. */
typedef struct {
  int32_t layers, hidden, d_in, d_out, activation, head;
  int32_t fourier_m;                 /* rows of the (m,3) spatial Fourier matrix */
  const float* d_b_matrix;           /* device (m,3) f32, or NULL when m == 0 */
  int32_t grid_resolution, grid_channels;
  /* temporal models (model.py:190-245): 0 keyframes = static.  Host pointers. */
  int32_t n_keyframes;               /* <= 16; the grids follow each other in params */
  const double* keyframe_times;
  int32_t time_mode;                 /* 0 none, 1 direct, 2 fourier, 3 both */
  int32_t time_fourier_count;
  const float* time_b;               /* (time_fourier_count, 1) */
  double time_t0, time_t1;           /* normalisation span (time_range or keyframe span) */
  int32_t raw_width;                 /* raw input block: 3 (p) or 6 (p|d, direction modes); 0 = 3 */
  int32_t fourier_in;                /* Fourier input width: 3 (p) or 6 (dirF); 0 = 3 */
} fvsrn_train_desc;

/* One batch of n positions (device f64 (n,3); timesteps d_times (n) f64 for temporal
 * models, else NULL) against reference values (device f32 (n,d_out)): forward with cached layer inputs (d_inputs: per layer n x in_l floats,
 * consecutive), pre-activations (d_preacts: (L-1) x n x hidden) and adjoints (d_deltas:
 * per layer n x out_l); the L1-loss sum is added to *d_loss_sum (fixed-order reduction);
 * the latent-grid gradient is added into d_grid_grad by the deterministic scatter: every
 * vertex sums its contributions in the reference's order and arithmetic (grid.py:86-112).
 * Weight/bias gradients: fvsrn_layer_grads over the caches (nn.py:252-253). */
FVSRN_API int32_t fvsrn_train_world_grads(const fvsrn_train_desc* desc, const float* d_params,
                                          const double* d_positions, const double* d_times,
                                          const float* d_reference,
                                          int64_t n, float* d_grid_grad, float* d_inputs,
                                          float* d_preacts, float* d_deltas, double* d_loss_sum,
                                          void* stream);
/* mlp_forward / mlp_backward (nn.py:179-193, 234-256) of a plain MLP (desc without grid)
 * on given inputs d_x (n, d_in) f32: outputs d_y (n, d_out), caches (layout as
 * fvsrn_train_world_grads) and, when d_y_bar (n, d_out) is given, the per-layer deltas and
 * (d_x_bar != NULL) the input adjoint delta_0 @ W_0 (n, d_in). */
FVSRN_API int32_t fvsrn_mlp_forward_backward(const fvsrn_train_desc* desc, const float* d_params,
                                             const float* d_x, const float* d_y_bar, int64_t n,
                                             float* d_y, float* d_inputs, float* d_preacts,
                                             float* d_deltas, float* d_x_bar, void* stream);
/* Weight / bias gradients of every layer from the caches of the calls above
 * (nn.py:252-253: delta_l^T @ inputs_l, sum over rows of delta_l) for the first n of
 * cap_rows cache rows, into d_grads laid out like the parameters ([W_0..W_{L-1} |
 * b_0..b_{L-1}], trainable_arrays order); accumulate != 0 adds to d_grads.  Tensor cores
 * (mma.sync TF32, 3xTF32 split) over fixed 256-row chunks, chunk partials summed in order:
 * bit-identical run to run.  Replaces the caller-side GEMMs. */
FVSRN_API int32_t fvsrn_layer_grads(const fvsrn_train_desc* desc, const float* d_inputs,
                                    const float* d_deltas, int64_t cap_rows, int64_t n,
                                    float* d_grads, int32_t accumulate, void* stream);
/* grid_sample_backward (grid.py:123-137): scatter-add of trilinear-weighted adjoints
 * d_z_bar (n, channels) f32 at positions (n,3) f64 into d_grad (res^3 * channels) f32,
 * deterministic (per-vertex sums in sample order, the reference's sequential order). */
FVSRN_API int32_t fvsrn_grid_sample_backward(int32_t resolution, int32_t channels,
                                             const double* d_positions, const float* d_z_bar,
                                             int64_t n, float* d_grad, void* stream);
/* model_backward (model.py:300-335): gradients of sum(raw_bar * raw) for n samples with
 * given raw-output adjoints d_raw_bar (n, d_out) f32, any head and input encoding (view
 * directions d_dirs (n,3) for direction modes, per-sample d_times for temporal models).
 * Same caches as fvsrn_train_world_grads (weight/bias gradients: fvsrn_layer_grads);
 * latent-grid gradients are added into d_grid_grad by the deterministic scatter
 * (per-vertex sums in model_backward's order: bracket pair, then sample). */
FVSRN_API int32_t fvsrn_model_grads(const fvsrn_train_desc* desc, const float* d_params,
                                    const double* d_positions, const double* d_dirs,
                                    const double* d_times, const float* d_raw_bar, int64_t n,
                                    float* d_grid_grad, float* d_inputs, float* d_preacts,
                                    float* d_deltas, void* stream);
/* Screen-space training (train.py:227-262), colour-head models.  Forward:
 * raymarch_forward(..., want_states=True) (render.py:203-238) of n explicit rays with f32
 * model evaluation and f64 compositing, no early termination: pixels (n,4) f32, terminal
 * colour (n,3) / alpha (n) f64 and the per-ray march geometry (tmin, ds, step count). */
FVSRN_API int32_t fvsrn_train_screen_forward(const fvsrn_train_desc* desc, const float* d_params,
                                             const double* d_origins, const double* d_dirs, int64_t n,
                                             const fvsrn_settings* settings, float* d_pixels,
                                             double* d_color, double* d_alpha, double* d_tmin,
                                             double* d_ds, int32_t* d_nsteps, void* stream);
/* raymarch_backward (render.py:241-306): reverse walk per ray with blend inversion; the
 * cache rows of ray i's step k go to row d_row_offset[i] + k of buffers sized for
 * cap_rows samples (layout as fvsrn_train_world_grads with n = cap_rows); latent-grid
 * gradients are added into d_grid_grad by the deterministic scatter in
 * raymarch_backward's order (steps from the last, rays in index order). */
FVSRN_API int32_t fvsrn_train_screen_backward(const fvsrn_train_desc* desc, const float* d_params,
                                              const double* d_origins, const double* d_dirs, int64_t n,
                                              double eps_blend, const double* d_color,
                                              const double* d_alpha, const double* d_tmin,
                                              const double* d_ds, const int32_t* d_nsteps,
                                              const int64_t* d_row_offset, const float* d_image_adjoint,
                                              const double* d_background, int64_t cap_rows,
                                              float* d_inputs, float* d_preacts, float* d_deltas,
                                              float* d_grid_grad, void* stream);
/* Reference-semantics f32 evaluation of model pieces for n samples (device pointers):
 * stage 0 assemble_input (model.py:248-279) -> (n, d_in); 1 latent vectors grid_sample /
 * keyframe_sample (grid.py:115-121, 222-230) -> (n, F); 2 raw network outputs of the
 * positions -> (n, d_out); 3 mlp_eval of given inputs d_x (n, d_in) (nn.py:195-204) ->
 * (n, d_out).  d_dirs for direction-input models, d_times for temporal ones (else NULL). */
FVSRN_API int32_t fvsrn_f32_eval(const fvsrn_train_desc* desc, const float* d_params,
                                 const double* d_positions, const double* d_dirs, const double* d_times,
                                 const float* d_x, int64_t n, int32_t stage, float* d_out, void* stream);
/* adam_step (nn.py:279-298) over n flat parameters at step t (1-based).  Non-finite
 * gradients are counted into *d_nonfinite and then nothing is updated. */
FVSRN_API int32_t fvsrn_adam_step(float* d_params, const float* d_grads, float* d_m, float* d_v,
                                  int64_t n, double lr, double beta1, double beta2, double eps,
                                  int32_t t, unsigned long long* d_nonfinite, void* stream);

/* ---- peer-memory framebuffer assembly (multi-GPU, one process per GPU).
 * Rank 0 exports its device framebuffer; every other rank opens it and its kernels
 * store their screen tiles straight into rank 0's frame over NVLink (P2P), replacing the
 * gather + reassembly.  64-byte handles (cudaIpcMemHandle_t) plus the byte offset of d_ptr
 * from its allocation base (IPC maps whole allocations; a pointer inside a caching
 * allocator's segment is reopened as base + offset).  fvsrn_ipc_close takes the pointer
 * fvsrn_ipc_open returned. */
FVSRN_API int32_t fvsrn_ipc_export(void* d_ptr, uint8_t handle[64], uint64_t* offset);
FVSRN_API int32_t fvsrn_ipc_open(const uint8_t handle[64], uint64_t offset, int32_t device, void** d_ptr);
FVSRN_API int32_t fvsrn_ipc_close(void* d_ptr);

FVSRN_API int32_t fvsrn_model_create(const fvsrn_model_desc* desc, int32_t device, fvsrn_model_t* out);
FVSRN_API int32_t fvsrn_model_destroy(fvsrn_model_t model);
/* Padded widths (K0, hidden_pad, out_pad), smem bytes; for plan/introspection. */
FVSRN_API int32_t fvsrn_model_info(fvsrn_model_t model, int32_t* k0_pad, int32_t* hidden_pad,
                         int32_t* smem_bytes);

/* Latent-grid sampler admitted at upload: tex_ok = 1 when the upload-time probe found
 * max |texture - exact-weight| <= 1e-3 on 2^18 positions (auto mode then uses the texture
 * units), probe_err = that maximum. */
FVSRN_API int32_t fvsrn_model_sampler(fvsrn_model_t model, int32_t* tex_ok, float* probe_err);

/* Full frame into host RGBA f32 (H,W,4); eval_count may be NULL. */
FVSRN_API int32_t fvsrn_render(fvsrn_model_t model, const fvsrn_tf* tf, const fvsrn_camera* cam,
                     const fvsrn_settings* settings, double t, float* out_rgba,
                     uint64_t* eval_count);
/* render_image followed by png_bytes' 8-bit conversion (imaging.py:74-80:
 * floor(clip(v,0,1)*255+0.5), bit-identical), done on the device: out is (H,W,4) uint8
 * (4 B/px over PCIe instead of 16).  The service /render path (service.py:88-129). */
FVSRN_API int32_t fvsrn_render_rgba8(fvsrn_model_t model, const fvsrn_tf* tf, const fvsrn_camera* cam,
                                     const fvsrn_settings* settings, double t, uint8_t* out_rgba8,
                                     uint64_t* eval_count);
/* Device framebuffer, stream-ordered; shard may be NULL (whole frame).
 * d_eval_count: device u64 accumulated atomically, may be NULL. */
FVSRN_API int32_t fvsrn_render_device(fvsrn_model_t model, const fvsrn_tf* tf, const fvsrn_camera* cam,
                            const fvsrn_settings* settings, double t, const fvsrn_shard* shard,
                            float* d_out, unsigned long long* d_eval_count, void* stream);
/* Reassemble world compact shard buffers [world][max_local_tiles*64][4] into (H,W,4). */
FVSRN_API int32_t fvsrn_tiles_to_frame_device(const float* d_gathered, int32_t width, int32_t height,
                                    int32_t world, float* d_frame, void* stream);
/* raymarch_forward over explicit f64 rays (host arrays). */
FVSRN_API int32_t fvsrn_render_rays(fvsrn_model_t model, const fvsrn_tf* tf, const double* origins,
                          const double* dirs, int64_t n, const fvsrn_settings* settings,
                          double t, float* out_px, uint64_t* eval_count);
FVSRN_API int32_t fvsrn_eval_density(fvsrn_model_t model, const double* p, int64_t n, double t,
                           float* out);
FVSRN_API int32_t fvsrn_eval_color(fvsrn_model_t model, const double* p, const double* d, int64_t n,
                         double t, float* out4);
FVSRN_API int32_t fvsrn_decode_density(fvsrn_model_t model, int32_t resolution, double t, float* out);
FVSRN_API int32_t fvsrn_decode_density_device(fvsrn_model_t model, int32_t resolution, double t,
                                    int64_t lattice_begin, int64_t lattice_count,
                                    float* d_out, void* stream);
/* ---- one process, several GPUs: SURVEY 8b's minimum export set asks for
 * fvsrn_render(..., device_ids[], n_devices) and fvsrn_decode_density(..., n_devices).
 * replicas[i] is the model uploaded with fvsrn_model_create(desc, device_ids[i], ...)
 * (same parameters on every device; a replica handle carries its device id).
 *
 * fvsrn_render_multi  <- render_image(source, camera, settings)       render.py:314-332
 *   Screen tiles (8x8) go round-robin to the replicas, tile k -> replica k mod n
 *   (SURVEY 8e).  Each replica's march kernel stores its finished pixels straight into
 *   the frame: into out itself, over each GPU's own link, when out is mapped page-locked
 *   memory (fvsrn_host_alloc); otherwise into one framebuffer on replicas[0]'s device
 *   over NVLink P2P, followed by a single device->host copy (page-locked staging if a
 *   pair has no P2P path).  Bit-identical to fvsrn_render on one device; eval_count is
 *   the sum over replicas.  n_devices == 1 is fvsrn_render.
 * fvsrn_decode_density_multi  <- decode_volume(model, resolution, t)  model.py:385-398
 *   Contiguous lattice slabs per replica, each decoded in its device's HBM and copied to
 *   out + slab begin over its own link. */
FVSRN_API int32_t fvsrn_render_multi(const fvsrn_model_t* replicas, int32_t n_devices,
                                     const fvsrn_tf* tf, const fvsrn_camera* cam,
                                     const fvsrn_settings* settings, double t, float* out_rgba,
                                     uint64_t* eval_count);
FVSRN_API int32_t fvsrn_decode_density_multi(const fvsrn_model_t* replicas, int32_t n_devices,
                                             int32_t resolution, double t, float* out);
/* Page-locked host buffers (e.g. reusable framebuffers: the D2H of fvsrn_render
 * into pinned memory runs at full PCIe/C2C bandwidth). */
FVSRN_API int32_t fvsrn_host_alloc(uint64_t bytes, void** ptr);
FVSRN_API int32_t fvsrn_host_free(void* ptr);
FVSRN_API int32_t fvsrn_fused_eval(fvsrn_model_t model, const float* x, int64_t n, float* out);

/* Ground-truth DVR of a dense scalar volume: VolumeSource(volume, tf)
 * (render.py:132-141, volume.py:213-255) -- same ray setup, TF, compositing and ET as
 * fvsrn_render, the network replaced by the reference's trilinear volume lookup.
 * values: (nx, ny, nz) f32 in [0,1], C order (ScalarVolume.values). */
typedef struct fvsrn_volume* fvsrn_volume_t;
FVSRN_API int32_t fvsrn_volume_create(const float* values, int32_t nx, int32_t ny, int32_t nz,
                                      int32_t device, fvsrn_volume_t* out);
FVSRN_API int32_t fvsrn_volume_destroy(fvsrn_volume_t volume);
FVSRN_API int32_t fvsrn_volume_render(fvsrn_volume_t volume, const fvsrn_tf* tf,
                                      const fvsrn_camera* cam, const fvsrn_settings* settings,
                                      float* out_rgba, uint64_t* sample_count);
FVSRN_API int32_t fvsrn_volume_render_device(fvsrn_volume_t volume, const fvsrn_tf* tf,
                                             const fvsrn_camera* cam, const fvsrn_settings* settings,
                                             const fvsrn_shard* shard, float* d_out, void* stream);
FVSRN_API int32_t fvsrn_volume_render_rays(fvsrn_volume_t volume, const fvsrn_tf* tf,
                                           const double* origins, const double* dirs, int64_t n,
                                           const fvsrn_settings* settings, float* out_px,
                                           uint64_t* sample_count);

#ifdef __cplusplus
}
#endif
#endif /* FVSRN_B200_H */
