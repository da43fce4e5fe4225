#include <chrono>
#include <condition_variable>
#include <deque>
#include <functional>
#include <future>
#include <thread>
#include <type_traits>
#include <array>
#include <atomic>
// fvsrn_capi.cu -- the C ABI (include/fvsrn_b200.h): model upload, weight/grid
// packing, per-frame constants, kernel launches.  Host code only.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <tuple>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fvsrn_b200.h"
#include "fvsrn_kernels.cuh"
#include "fvsrn_tc.cuh"
#include "fvsrn_train.cuh"
#include "fvsrn_volume.cuh"

using namespace fvsrn;

namespace {

thread_local std::string g_err;
// LPT tile ordering on/off (FVSRN_LPT=0 disables; A/B measurements)
const bool g_lpt_enabled = [] {
  const char* e = std::getenv("FVSRN_LPT");
  return !(e && e[0] == '0');
}();

// DVR kernel for the default fV-SRN shapes: FVSRN_DVR=tc (tcgen05/TMEM), ws
// (warp-specialised mma.sync) or warp (single-role mma.sync); unset = the measured
// faster one per width (auto: tcgen05 for 64-wide, mma.sync for 32-wide).
// Other shapes always run the mma.sync dvr_kernel.
#ifndef FVSRN_TEX_DEFAULT
#define FVSRN_TEX_DEFAULT 1
#endif
constexpr bool kTexDefault = FVSRN_TEX_DEFAULT != 0;
enum class DvrMode : int { kAuto = 0, kTC = 1, kWS = 2, kWarp = 3, kPipe = 4, kDual = 5 };
std::atomic<int> g_dvr_mode_i{[] {
  const char* e = std::getenv("FVSRN_DVR");
  if (e && std::string(e) == "tc") return (int)DvrMode::kTC;
  if (e && std::string(e) == "warp") return (int)DvrMode::kWarp;
  if (FVSRN_AB_VARIANTS && e && std::string(e) == "ws") return (int)DvrMode::kWS;
  if (FVSRN_AB_VARIANTS && e && std::string(e) == "pipe") return (int)DvrMode::kPipe;
  if (FVSRN_AB_VARIANTS && e && std::string(e) == "dual") return (int)DvrMode::kDual;
  return (int)DvrMode::kAuto;
}()};
// latent-grid sampler for F = 16 grids: 0 auto, 1 texture units, 2 LDG + HFMA2
std::atomic<int> g_grid_mode{[] {
  const char* e = std::getenv("FVSRN_GRID");
  if (e && std::string(e) == "tex") return 1;
  if (e && std::string(e) == "ldg") return 2;
  return 0;
}()};
bool use_tex(const fvsrn_model* m);
// FVSRN_OCC=n: cap resident CTAs per SM of the persistent kernels (A/B measurements)
const int g_occ_cap = [] {
  const char* e = std::getenv("FVSRN_OCC");
  return e ? std::atoi(e) : 0;
}();
// temporal texture path: pre-blend the bracketing keyframes once per frame
// (FVSRN_TEX_PREBLEND=0: blend both texture sets per sample in the march kernel)
const bool g_tex_preblend = [] {
  const char* e = std::getenv("FVSRN_TEX_PREBLEND");
  return !(e && e[0] == '0');
}();
// render straight into mapped page-locked framebuffers (FVSRN_ZERO_COPY=0: copy instead)
const bool g_zero_copy = [] {
  const char* e = std::getenv("FVSRN_ZERO_COPY");
  return !(e && e[0] == '0');
}();
// device alias of a mapped page-locked host buffer (fvsrn_host_alloc), else nullptr
float* mapped_device_ptr(void* host) {
  if (!g_zero_copy) return nullptr;
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, host) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
      pa.devicePointer)
    return (float*)pa.devicePointer;
  cudaGetLastError();
  return nullptr;
}
// set by fvsrn_render while its frame is a mapped host framebuffer (tile order choice)
thread_local bool g_out_mapped = false;

// Per-thread page-locked landing slot for the per-frame counters: the D2H copy is then a
// plain DMA (a pageable destination goes through a driver staging buffer).
unsigned long long* pinned_counters() {
  thread_local struct Slot {
    unsigned long long* p = nullptr;
    ~Slot() { if (p) cudaFreeHost(p); }
  } slot;
  if (!slot.p && cudaMallocHost((void**)&slot.p, 64) != cudaSuccess) {
    cudaGetLastError();
    slot.p = nullptr;
  }
  return slot.p;
}
inline DvrMode dvr_mode() { return (DvrMode)g_dvr_mode_i.load(std::memory_order_relaxed); }
bool use_tc(const fvsrn_model* m);

// Per-thread kernel timer (fvsrn_kernel_timer): CUDA events around every launch of the
// dominant kernel (the march / decode kernel) and a count of all library launches.
struct KernelTimer {
  bool on = false;
  std::string name;              // the last timed launch: kernel instantiation + grid sampler
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  size_t used = 0;
  long long launches = 0;
};
thread_local KernelTimer g_kt;
void count_launch() {
  if (g_kt.on) ++g_kt.launches;
}

// FVSRN_DEBUG_TIMING=1: host-side phase timestamps of fvsrn_render to stderr (diagnostics)
const bool g_debug_timing = std::getenv("FVSRN_DEBUG_TIMING") != nullptr;
// Miss pixels are stored by the march kernel's refill rather than by ray_setup (so the
// stores into a mapped host framebuffer overlap the march); FVSRN_DEFER_MISS=0 restores
// the ray_setup stores (A/B switch).
const int g_defer_miss = [] {
  const char* e = std::getenv("FVSRN_DEFER_MISS");
  return (e && e[0] == '0') ? 0 : 1;
}();
struct HostPhases {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  std::string out;
  void mark(const char* what) {
    if (!g_debug_timing) return;
    const auto now = std::chrono::steady_clock::now();
    out += std::string(" ") + what + "=" +
           std::to_string(std::chrono::duration<double, std::micro>(now - last).count()).substr(0, 6) + "us";
    last = now;
  }
  ~HostPhases() {
    if (g_debug_timing) std::fprintf(stderr, "fvsrn_render phases:%s\n", out.c_str());
  }
};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) {                                                            \
      (void)cudaGetLastError(); /* do not leak a non-sticky error into the next call */ \
      return fail(FVSRN_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));     \
    }                                                                                   \
  } while (0)

int round_up(int x, int m) { return (x + m - 1) / m * m; }

// IPC: opened mapping (base + offset) -> the base cudaIpcOpenMemHandle returned
std::mutex g_ipc_mu;
std::map<void*, void*> g_ipc_bases;

// [base, base + size) of the device allocation containing p (driver cuMemGetAddressRange,
// fetched through the runtime so the library does not link libcuda).
int alloc_range(void* p, void** base, size_t* size) {
  typedef int (*GetRange)(unsigned long long*, size_t*, unsigned long long);
  static GetRange fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return (GetRange)f;
  }();
  if (!fn) return fail(FVSRN_ECUDA, "cuMemGetAddressRange unavailable");
  unsigned long long b = 0;
  if (int r = fn(&b, size, (unsigned long long)p)) return fail(FVSRN_ECUDA, "cuMemGetAddressRange failed (" + std::to_string(r) + ")");
  *base = (void*)b;
  return FVSRN_OK;
}


struct Pack {                     // fragment-ordered weights + padded biases
  std::vector<uint2> frag;
  std::vector<float> bias;
  std::vector<int> w_off, b_off;
  int kt0 = 0;
};

// W_dev[l] : (N_l x K_l) floats in device column order (zero padded)
void build_pack(const std::vector<std::vector<float>>& wdev, const std::vector<int>& K,
                const std::vector<int>& N, const std::vector<std::vector<float>>& bdev, Pack& pk) {
  const int L = (int)wdev.size();
  pk.w_off.assign(L + 1, 0);
  pk.b_off.assign(L + 1, 0);
  pk.frag.clear();
  pk.bias.clear();
  for (int l = 0; l < L; ++l) {
    pk.w_off[l] = (int)pk.frag.size();
    pk.b_off[l] = (int)pk.bias.size();
    const int KT = K[l] / 16, NT = N[l] / 8;
    const auto& W = wdev[l];
    auto frag = [&](int kt, int nt, int lane) {
      const int g = lane >> 2, q = lane & 3;
      const int n = nt * 8 + g, k0 = kt * 16 + 2 * q;
      auto h = [&](int k) { return __half_as_ushort(__float2half_rn(W[(size_t)n * K[l] + k])); };
      uint2 u;
      u.x = (uint32_t)h(k0) | ((uint32_t)h(k0 + 1) << 16);
      u.y = (uint32_t)h(k0 + 8) | ((uint32_t)h(k0 + 9) << 16);
      return u;
    };
    if (FVSRN_BPAIRS && NT >= 2) {  // hidden-width layer: [kt][n-tile pair][lane] -> LDS.128
      for (int kt = 0; kt < KT; ++kt)
        for (int p = 0; p < NT / 2; ++p)
          for (int lane = 0; lane < 32; ++lane) {
            pk.frag.push_back(frag(kt, 2 * p, lane));
            pk.frag.push_back(frag(kt, 2 * p + 1, lane));
          }
    } else {        // [kt][nt][lane] x uint2 (always for the one-tile output layer)
      for (int kt = 0; kt < KT; ++kt)
        for (int nt = 0; nt < NT; ++nt)
          for (int lane = 0; lane < 32; ++lane) pk.frag.push_back(frag(kt, nt, lane));
    }
    // accumulator quads: (nt, q) -> {b[nt*8+2q], b[nt*8+2q+1], same, same}
    for (int nt = 0; nt < NT; ++nt)
      for (int q = 0; q < 4; ++q)
        for (int c = 0; c < 4; ++c) pk.bias.push_back(bdev[l][nt * 8 + 2 * q + (c & 1)]);
  }
  pk.w_off[L] = (int)pk.frag.size();
  pk.b_off[L] = (int)pk.bias.size();
}

struct DevPack {
  uint2* frag = nullptr;
  float* bias = nullptr;
  NetDev net{};
};

}  // namespace

struct fvsrn_model {
  int device = 0;
  int layers = 0, hidden = 0, hid_pad = 0, d_in = 0, d_out = 0, act = 0, head = 0;
  int dir_mode = 0, fourier_mode = 0, m = 0, fd_in = 3, raw_w = 3;
  int time_mode = 0, tfc = 0, T = 0;
  std::vector<float> time_b;
  bool has_time_range = false;
  double time_range[2] = {0, 0};
  bool temporal = false;
  std::vector<double> kf_times;
  int R = 0, F = 0, f_pad = 0;
  std::vector<__half*> grids;       // fp16 (R,R,R,f_pad)
  float* d_bmat = nullptr;
  int four_off = 0, raw_off = 0, k0 = 0;
  // sample pack (device column order, time folded) and x pack (reference order)
  DevPack ps, px;
  // tcgen05 pack (canonical K-major fp16 tiles + f32 biases), default shapes only
  uint4* d_wtc = nullptr;
  float* d_btc = nullptr;
  bool tc_ok = false;
  // texture path (F padded to 16): per grid 4 RGBA16F 3D arrays + texture objects
  std::vector<cudaArray_t> tex_arrays;
  std::vector<std::array<cudaTextureObject_t, 4>> tex;
  // u8 grids: the textures hold the codes; per-grid per-channel dequantisation
  bool tex_u8 = false;
  std::vector<std::array<float, 16>> qmin, qspan;
  // texture sampler admitted for this model by the upload-time accuracy probe
  // (probe_texture_sampler); tex_probe_err = max |tex - ldg| of the probe outputs
  bool tex_ok = true;
  float tex_probe_err = 0.f;
  // temporal texture path: per-(host thread, stream) pre-blended keyframe array set
  struct BlendSet {
    cudaArray_t arr[4] = {};
    cudaSurfaceObject_t surf[4] = {};
    cudaTextureObject_t tex[4] = {};
    int lo = -1, hi = -1;
    float w = -1.f;
  };
  mutable std::mutex blend_mu;
  mutable std::map<std::pair<std::thread::id, cudaStream_t>, std::unique_ptr<BlendSet>> blend_sets;
  int k0x = 0;
  std::vector<float> b0_static;     // layer-0 bias, padded N0
  std::vector<float> w0_time;       // N0 x T time columns of W0
  int n0 = 0;
  int num_sms = 148;
  ~fvsrn_model() {
    cudaSetDevice(device);
    for (auto* g : grids) cudaFree(g);
    cudaFree(d_bmat);
    cudaFree(ps.frag); cudaFree(ps.bias);
    cudaFree(px.frag); cudaFree(px.bias);
    cudaFree(d_wtc); cudaFree(d_btc);
    for (auto& t4 : tex)
      for (auto t : t4) cudaDestroyTextureObject(t);
    for (auto a : tex_arrays) cudaFreeArray(a);
    for (auto& kv : blend_sets)
      for (int j = 0; j < 4; ++j) {
        cudaDestroyTextureObject(kv.second->tex[j]);
        cudaDestroySurfaceObject(kv.second->surf[j]);
        cudaFreeArray(kv.second->arr[j]);
      }
  }
};

namespace {

int upload(const void* host, size_t bytes, void** dev) {
  CUDA_TRY(cudaMalloc(dev, bytes));
  CUDA_TRY(cudaMemcpy(*dev, host, bytes, cudaMemcpyHostToDevice));
  return FVSRN_OK;
}

int make_devpack(const Pack& pk, int layers, int act, int head, int out_real, DevPack& dp) {
  int rc = upload(pk.frag.data(), pk.frag.size() * sizeof(uint2), (void**)&dp.frag);
  if (rc) return rc;
  rc = upload(pk.bias.data(), pk.bias.size() * sizeof(float), (void**)&dp.bias);
  if (rc) return rc;
  NetDev& n = dp.net;
  n.wfrag = dp.frag;
  n.bias = dp.bias;
  n.layers = layers;
  n.kt0 = pk.kt0;
  n.act = act;
  n.head = head;
  n.out_real = out_real;
  for (int l = 0; l <= layers; ++l) { n.w_off[l] = pk.w_off[l]; n.b_off[l] = pk.b_off[l]; }
  n.w_total = (int)pk.frag.size();
  n.b_total = (int)pk.bias.size();
  return FVSRN_OK;
}

// 4 RGBA16F 3D arrays (channels 4j..4j+3) of one fp16 (R,R,R,16) grid + texture objects
// (linear filtering, clamp addressing, unnormalised coordinates).  Array width = grid z.
template <typename T>
int make_grid_textures_t(fvsrn_model* m, const std::vector<T>& h, int F) {
  const int R = m->R;
  const size_t nvox = (size_t)R * R * R;
  std::array<cudaTextureObject_t, 4> t4{};
  std::vector<T> plane(nvox * 4);
  const bool u8 = std::is_same<T, uint8_t>::value;
  for (int j = 0; j < 4; ++j) {
    for (size_t v = 0; v < nvox; ++v)
      for (int c = 0; c < 4; ++c) plane[v * 4 + c] = (4 * j + c < F) ? h[v * F + 4 * j + c] : T(0);
    cudaChannelFormatDesc cd = u8 ? cudaCreateChannelDesc<uchar4>() : cudaCreateChannelDescHalf4();
    cudaArray_t arr = nullptr;
    CUDA_TRY(cudaMalloc3DArray(&arr, &cd, make_cudaExtent(R, R, R)));
    m->tex_arrays.push_back(arr);
    cudaMemcpy3DParms cp{};
    cp.srcPtr = make_cudaPitchedPtr(plane.data(), (size_t)R * 4 * sizeof(T), R, R);
    cp.dstArray = arr;
    cp.extent = make_cudaExtent(R, R, R);
    cp.kind = cudaMemcpyHostToDevice;
    CUDA_TRY(cudaMemcpy3D(&cp));
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeArray;
    rd.res.array.array = arr;
    cudaTextureDesc td{};
    td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
    td.filterMode = cudaFilterModeLinear;
    td.readMode = u8 ? cudaReadModeNormalizedFloat : cudaReadModeElementType;   // u8: code/255
    td.normalizedCoords = 0;
    CUDA_TRY(cudaCreateTextureObject(&t4[j], &rd, &td, nullptr));
  }
  m->tex.push_back(t4);
  return FVSRN_OK;
}

int make_grid_textures(fvsrn_model* m, const std::vector<__half>& h) { return make_grid_textures_t(m, h, 16); }

std::vector<__half> to_half_padded(const float* src, int R, int F, int f_pad) {
  const size_t nvox = (size_t)R * R * R;
  std::vector<__half> h(nvox * f_pad, __float2half_rn(0.f));
  for (size_t v = 0; v < nvox; ++v)
    for (int c = 0; c < F; ++c) h[v * f_pad + c] = __float2half_rn(src[v * F + c]);
  return h;
}

// time features for a per-frame scalar t (model.py:190-197, 236-245)
std::vector<double> time_features(const fvsrn_model* m, double t) {
  double t0, t1;
  if (m->has_time_range) { t0 = m->time_range[0]; t1 = m->time_range[1]; }
  else { t0 = m->kf_times.front(); t1 = m->kf_times.back(); }
  double tn = (t1 == t0) ? 0.0 : (std::min(std::max(t, t0), t1) - t0) / (t1 - t0);
  std::vector<double> f;
  if (m->time_mode == FVSRN_TIME_DIRECT || m->time_mode == FVSRN_TIME_BOTH) f.push_back(tn);
  if (m->time_mode == FVSRN_TIME_FOURIER || m->time_mode == FVSRN_TIME_BOTH) {
    std::vector<double> s, c;
    for (int j = 0; j < m->tfc; ++j) {
      double ph = tn * (double)m->time_b[j];
      s.push_back(std::sin(ph));
      c.push_back(std::cos(ph));
    }
    f.insert(f.end(), s.begin(), s.end());
    f.insert(f.end(), c.begin(), c.end());
  }
  return f;
}

// keyframe bracket (model.py:200-209 for a scalar t)
void bracket(const std::vector<double>& times, double t, int& lo, int& hi, double& w) {
  const int n = (int)times.size();
  double tc = std::min(std::max(t, times.front()), times.back());
  int h = (int)(std::lower_bound(times.begin(), times.end(), tc) - times.begin());
  h = std::min(std::max(h, 0), n - 1);
  int l = (h > 0 && times[h] != tc) ? h - 1 : h;
  lo = l; hi = h;
  w = (h > l) ? (tc - times[l]) / (times[h] - times[l]) : 0.0;
}

// TransferFunction -> device table: control values + per-segment slopes (f64 -> f32),
// i.e. np.interp's fp[i] + (x - xp[i]) * slope_i (transfer.py:57-65).
int build_tf(const fvsrn_tf* tf, TFDev& th) {
  if (tf->n < 2 || tf->n > kMaxTF) return fail(FVSRN_EINVAL, "transfer function needs 2..64 points");
  th = TFDev{};
  th.n = tf->n;
  for (int i = 0; i < tf->n; ++i) {
    th.xs[i] = tf->xs[i];
    for (int c = 0; c < 3; ++c) th.val[i][c] = tf->rgbs[3 * i + c];
    th.val[i][3] = tf->sigmas[i];
  }
  for (int i = 0; i + 1 < tf->n; ++i)
    for (int c = 0; c < 4; ++c) {
      double y0 = (c < 3) ? tf->rgbs[3 * i + c] : tf->sigmas[i];
      double y1 = (c < 3) ? tf->rgbs[3 * (i + 1) + c] : tf->sigmas[i + 1];
      th.slope[i][c] = (float)((y1 - y0) / ((double)tf->xs[i + 1] - (double)tf->xs[i]));
    }
  return FVSRN_OK;
}

struct FrameScratch {
  void* buf = nullptr;
  const __half* grid = nullptr;
  bool tex_on = false;
  float tex_w = 0.f;
  const cudaTextureObject_t* tex_lo = nullptr;
  const cudaTextureObject_t* tex_hi = nullptr;
  bool tex_u8 = false;
  int q_lo = 0, q_hi = 0;           // grid indices (u8 dequantisation constants)
  float* b0 = nullptr;
  TFDev* tf = nullptr;
  unsigned long long* counters = nullptr;   // [0] queue, [1] evals, [2] non-finite pixels
};

// per-thread sampler override used by the upload-time probe (0 none, 1 tex, 2 ldg)
thread_local int g_sampler_override = 0;

// Texture units for the latent grid when: forced (FVSRN_GRID=tex / mode 1), or in auto
// mode when the model passed the upload-time accuracy probe.  The texture filter's 8-bit
// fractional weights perturb each latent channel by up to |v1 - v0| / 512 per axis; for
// random-init grids that stays ~5e-4 in density, for trained grids with sharp latent
// features it reached 4e-3 (trained cfg-2 shape) and 1.0e-2 (trained cfg-3 shape, u8
// grid) at 2^20 positions, so those models render with the exact-weight LDG sampler.
bool use_tex(const fvsrn_model* m) {
  if (m->tex.empty()) return false;
  if (g_sampler_override) return g_sampler_override == 1;
  const int g = g_grid_mode.load(std::memory_order_relaxed);
  return g == 1 || (g == 0 && kTexDefault && m->tex_ok);
}

// Pre-blend keyframes (lo, hi, w) into this (thread, stream)'s array set; reuses the set
// when the bracket is unchanged.  Stream order makes the blend finish before the march.
int preblend(const fvsrn_model* m, int lo, int hi, float w, cudaStream_t s,
             const fvsrn_model::BlendSet*& out) {
  fvsrn_model::BlendSet* b = nullptr;
  {
    std::lock_guard<std::mutex> lk(m->blend_mu);
    auto& slot = m->blend_sets[std::make_pair(std::this_thread::get_id(), s)];
    if (!slot) {
      slot.reset(new fvsrn_model::BlendSet());
      const int R = m->R;
      for (int j = 0; j < 4; ++j) {
        cudaChannelFormatDesc cd = cudaCreateChannelDescHalf4();
        CUDA_TRY(cudaMalloc3DArray(&slot->arr[j], &cd, make_cudaExtent(R, R, R), cudaArraySurfaceLoadStore));
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeArray;
        rd.res.array.array = slot->arr[j];
        CUDA_TRY(cudaCreateSurfaceObject(&slot->surf[j], &rd));
        cudaTextureDesc td{};
        td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
        td.filterMode = cudaFilterModeLinear;
        td.readMode = cudaReadModeElementType;
        td.normalizedCoords = 0;
        CUDA_TRY(cudaCreateTextureObject(&slot->tex[j], &rd, &td, nullptr));
      }
    }
    b = slot.get();
  }
  if (b->lo != lo || b->hi != hi || b->w != w) {
    TexBlendArgs a{};
    for (int j = 0; j < 4; ++j) { a.lo[j] = m->tex[lo][j]; a.hi[j] = m->tex[hi][j]; a.out[j] = b->surf[j]; }
    a.R = m->R;
    a.u8 = m->tex_u8 ? 1 : 0;
    a.w = w;
    if (m->tex_u8)
      for (int c = 0; c < 16; ++c) {
        a.qmin_lo[c] = m->qmin[lo][c]; a.qspan_lo[c] = m->qspan[lo][c];
        a.qmin_hi[c] = m->qmin[hi][c]; a.qspan_hi[c] = m->qspan[hi][c];
      }
    CUDA_TRY(launch_tex_blend(a, s));
    count_launch();
    b->lo = lo; b->hi = hi; b->w = w;
  }
  out = b;
  return FVSRN_OK;
}

// Per-call device scratch: effective layer-0 bias (time folded), TF table,
// counters, and the time-blended latent grid.  Stream-ordered allocation.
int frame_setup(const fvsrn_model* m, double t, const fvsrn_tf* tf, cudaStream_t s,
                FrameScratch& fs) {
  if (m->temporal && !std::isfinite(t)) return fail(FVSRN_EINVAL, "timestep must be finite");
  std::vector<float> b0 = m->b0_static;
  if (m->T > 0) {
    std::vector<double> f = time_features(m, t);
    for (int n = 0; n < m->n0; ++n) {
      float acc = b0[n];
      for (int j = 0; j < m->T; ++j) acc += m->w0_time[(size_t)n * m->T + j] * (float)f[j];
      b0[n] = acc;
    }
  }
  TFDev th{};
  if (tf) {
    int rc = build_tf(tf, th);
    if (rc) return rc;
  }
  size_t grid_bytes = 0;
  int lo = 0, hi = 0;
  double w = 0.0;
  fs.tex_on = use_tex(m);
  if (m->f_pad > 0 && m->temporal) {
    bracket(m->kf_times, t, lo, hi, w);
    if (hi != lo && !fs.tex_on) grid_bytes = (size_t)m->R * m->R * m->R * m->f_pad * sizeof(__half);
  }
  if (fs.tex_on) {   // keyframe blend in the kernel (two texture sets) or pre-blended
    fs.tex_lo = m->tex[m->temporal ? lo : 0].data();
    fs.tex_hi = m->tex[m->temporal ? hi : 0].data();
    fs.q_lo = m->temporal ? lo : 0;
    fs.q_hi = m->temporal ? hi : 0;
    fs.tex_w = (m->temporal && hi != lo) ? (float)w : 0.f;
    fs.tex_u8 = m->tex_u8;
    if (fs.tex_w != 0.f && g_tex_preblend) {
      const fvsrn_model::BlendSet* b = nullptr;
      int rc = preblend(m, lo, hi, (float)w, s, b);
      if (rc) return rc;
      fs.tex_lo = fs.tex_hi = b->tex;
      fs.tex_w = 0.f;
      fs.tex_u8 = false;
    }
  }
  const size_t off_tf = 0, off_b0 = (sizeof(TFDev) + 255) / 256 * 256;
  const size_t off_ct = off_b0 + 1024, off_grid = off_ct + 256;
  CUDA_TRY(cudaMallocAsync(&fs.buf, off_grid + grid_bytes, s));
  char* base = (char*)fs.buf;
  fs.tf = (TFDev*)(base + off_tf);
  fs.b0 = (float*)(base + off_b0);
  fs.counters = (unsigned long long*)(base + off_ct);
  CUDA_TRY(cudaMemcpyAsync(fs.tf, &th, sizeof(TFDev), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(fs.b0, b0.data(), b0.size() * sizeof(float), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemsetAsync(fs.counters, 0, 3 * sizeof(unsigned long long), s));
  fs.grid = m->f_pad > 0 ? m->grids[m->temporal ? lo : 0] : nullptr;
  if (grid_bytes) {
    __half* g = (__half*)(base + off_grid);
    CUDA_TRY(launch_blend(m->grids[lo], m->grids[hi], (float)w,
                          (long long)m->R * m->R * m->R * m->f_pad, g, s));
    count_launch();
    fs.grid = g;
  }
  return FVSRN_OK;
}

FeatDev feat_for(const fvsrn_model* m, const FrameScratch& fs) {
  FeatDev fd{};
  const __half* grid = fs.grid;
  fd.tex_on = fs.tex_on ? 1 : 0;
  fd.tex_w = fs.tex_w;
  for (int j = 0; j < 4 && fs.tex_on; ++j) { fd.tex_lo[j] = fs.tex_lo[j]; fd.tex_hi[j] = fs.tex_hi[j]; }
  fd.tex_u8 = (fs.tex_on && fs.tex_u8) ? 1 : 0;
  if (fd.tex_u8)
    for (int c = 0; c < 16; ++c) {
      fd.qmin_lo[c] = m->qmin[fs.q_lo][c]; fd.qspan_lo[c] = m->qspan[fs.q_lo][c];
      fd.qmin_hi[c] = m->qmin[fs.q_hi][c]; fd.qspan_hi[c] = m->qspan[fs.q_hi][c];
    }
  fd.grid_res = m->R;
  fd.f_pad = m->f_pad;
  fd.grid = grid;
  fd.fourier_mode = m->fourier_mode;
  fd.m = m->m;
  fd.fd_in = m->fd_in;
  fd.bmat = m->d_bmat;
  fd.four_off = m->four_off;
  fd.raw_off = m->raw_off;
  fd.raw_w = m->raw_w;
  fd.k0 = m->k0;
  fd.dir_mode = m->dir_mode;
  return fd;
}

bool fast_path(const fvsrn_model* m, KernelKind kind) {
  if (m->act != FVSRN_ACT_SNAKE_ALT) return false;
  if (kind == KernelKind::kFused) return true;
  return m->fourier_mode == FVSRN_FOURIER_NERF && m->fd_in == 3 && m->raw_w == 3 &&
         m->m == (m->hid_pad - 4) / 2 && m->f_pad == 16 && m->R > 0 &&
         m->layers == fast_layer_count(m->hid_pad);
}

// (kernel, device, smem) -> resident CTAs per SM; the attribute + occupancy queries run
// once per configuration instead of on every launch.
// The dynamic-smem attribute is per (kernel, device) and only ever raised: lowering it
// for a smaller configuration would invalidate a cached larger one.
std::mutex g_occ_mu;
std::map<std::tuple<const void*, int, size_t>, int> g_occ;
std::map<std::pair<const void*, int>, size_t> g_smem_attr;

// What `launch` runs, for the measurement record (fvsrn_kernel_timer_info): the template
// instantiation, the MMA path and the latent-grid sampler.
std::string kernel_desc(const fvsrn_model* m, KernelKind kind, int fmode = 1) {
  const int h = m->hid_pad;
  const bool fast = fast_path(m, kind);
  const std::string tmpl = fast ? std::to_string(h) + ",4," + std::to_string((h - 4) / 2) + "," +
                                      std::to_string(m->layers)
                                : std::to_string(h) + ",-1,0,0";
  std::string k;
  switch (kind) {
    case KernelKind::kDVRTC:
    case KernelKind::kDVRTCTex:
      k = std::string("dvr_tc_kernel<") + std::to_string(h) + "," +
          std::to_string((h - 4) / 2) + "," + std::to_string(m->layers) +
          (kind == KernelKind::kDVRTCTex ? "," + std::to_string(fmode) : "") +
          "> (tcgen05.mma kind::f16, TMEM accumulators)";
      break;
    case KernelKind::kSampleTex: k = "sample_kernel<" + tmpl + "," + std::to_string(fmode) + "> (mma.sync m16n8k16, static-grid features)"; break;
    case KernelKind::kSampleTC:
      k = "decode_tc_kernel<" + std::to_string(h) + "," + std::to_string((h - 4) / 2) + "," +
          std::to_string(m->layers) + "," + std::to_string(fmode) + "> (tcgen05.mma kind::f16, TMEM accumulators)";
      break;
    case KernelKind::kDVRWS: k = "dvr_ws_kernel<" + tmpl + "> (mma.sync m16n8k16)"; break;
    case KernelKind::kDVRPipe: k = "dvr_pipe_kernel<" + tmpl + "> (mma.sync m16n8k16)"; break;
    case KernelKind::kDVRDual: k = "dvr_dual_kernel<" + tmpl + "> (mma.sync m16n8k16)"; break;
    case KernelKind::kSample: k = "sample_kernel<" + tmpl + "> (mma.sync m16n8k16)"; break;
    case KernelKind::kDVRTex: k = "dvr_kernel<" + tmpl + "," + std::to_string(fmode) + "> (mma.sync m16n8k16, frame specialisation)"; break;
    case KernelKind::kDVRPair: k = "dvr_pair_kernel<" + tmpl + "," + std::to_string(fmode) + ",2> (mma.sync m16n8k16, two lanes per ray)"; break;
    case KernelKind::kDVRQuad: k = "dvr_pair_kernel<" + tmpl + "," + std::to_string(fmode) + ",4> (mma.sync m16n8k16, four lanes per ray)"; break;
    case KernelKind::kDVROcto: k = "dvr_pair_kernel<" + tmpl + "," + std::to_string(fmode) + ",8> (mma.sync m16n8k16, eight lanes per ray)"; break;
    default: k = "dvr_kernel<" + tmpl + "> (mma.sync m16n8k16)"; break;
  }
  const char* grid = m->R <= 0 ? "no latent grid"
                     : use_tex(m) ? (m->tex_u8 ? "texture units, RGBA8 u8 codes, hardware trilinear (8-bit weights)"
                                               : "texture units, RGBA16F, hardware trilinear (8-bit weights)")
                                  : "LDG.256 fp16 + HFMA2 trilinear";
  return k + "; grid: " + grid;
}

int launch(const fvsrn_model* m, KernelKind kind, size_t smem, void** args, cudaStream_t s,
           long long work_warps, int fmode = 1) {
  const bool tc = kind == KernelKind::kDVRTC || kind == KernelKind::kDVRTCTex;
  const void* fn = kind == KernelKind::kDVRTC ? tc_kernel_for(m->hid_pad)
                   : kind == KernelKind::kDVRTCTex ? tc_tex_kernel_for(m->hid_pad, fmode)
                   : kind == KernelKind::kSampleTC ? tc_decode_kernel_for(m->hid_pad, fmode)
                                                    : kernel_for(kind, m->hid_pad, fast_path(m, kind), fmode);
  const bool tmem_k = tc || kind == KernelKind::kSampleTC;   // tcgen05 kernels (TMEM, 128 threads)
  const int threads = kind == KernelKind::kDVRWS ? kWsThreads : tmem_k ? kTcThreads : kThreads;
  if (!fn) return fail(FVSRN_ECAPACITY, "no kernel for this hidden width");
  int occ = 0;
  {
    std::lock_guard<std::mutex> lk(g_occ_mu);
    auto key = std::make_tuple(fn, m->device, smem);
    auto it = g_occ.find(key);
    if (it == g_occ.end()) {
      size_t& attr = g_smem_attr[std::make_pair(fn, m->device)];
      if (smem > attr) {
        CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = smem;
      }
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem));
      if (tmem_k) {
        // The occupancy API reports 1 CTA/SM for kernels that allocate TMEM; the real
        // limits are registers (launch bounds), shared memory and TMEM columns (each
        // CTA allocates <= 64 of 512), so size the persistent grid from those.
        cudaFuncAttributes fa;
        CUDA_TRY(cudaFuncGetAttributes(&fa, fn));
        int smem_sm = 0, regs_sm = 0;
        CUDA_TRY(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, m->device));
        CUDA_TRY(cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, m->device));
        const int by_smem = smem_sm / (int)(smem + fa.sharedSizeBytes + 1024);
        const int by_regs = regs_sm / std::max(1, fa.numRegs * threads);
        occ = std::max(1, std::min(std::min(by_smem, by_regs), 8));
      }
      g_occ[key] = occ;
      if (std::getenv("FVSRN_DEBUG_OCC"))
        std::fprintf(stderr, "fvsrn: kernel kind %d hid %d threads %d smem %zu -> %d CTAs/SM\n", (int)kind,
                     m->hid_pad, threads, smem, occ);
    } else {
      occ = it->second;
    }
  }
  if (occ < 1) return fail(FVSRN_ECAPACITY, "kernel does not fit on an SM (shared memory)");
  if (g_occ_cap > 0) occ = std::min(occ, g_occ_cap);
  if (kind == KernelKind::kDVR || kind == KernelKind::kDVRTex || kind == KernelKind::kDVRPair ||
      kind == KernelKind::kDVRQuad || kind == KernelKind::kDVROcto ||
      kind == KernelKind::kDVRPipe ||
      tc ||
      kind == KernelKind::kDVRDual) {
    // Small frames: the frame time is the longest rays' sequential march, and every
    // co-resident warp slows each step of it.  Keep ~1.75 work slots per lane (measured
    // at 256^2: 0.456 ms at 5 CTAs/SM -> 0.318 ms at 2); large frames are unaffected.
    // (two lanes per ray: 2.25 work slots per lane, measured at 256^2: 1.75 0.256 ms,
    // 2.0-2.5 0.225-0.228, 3.0 0.240; FVSRN_SLOTS_PER_LANE overrides both)
    static const char* spl_env = std::getenv("FVSRN_SLOTS_PER_LANE");
    static const char* spl4_env = std::getenv("FVSRN_SLOTS_PER_LANE4");
    const double slots_per_lane = (kind == KernelKind::kDVRQuad || kind == KernelKind::kDVROcto)
                                      ? (spl4_env ? std::atof(spl4_env) : 2.25)
                                  : spl_env ? std::atof(spl_env) : (kind == KernelKind::kDVRPair ? 2.25 : 1.75);
    const double rays_per_sm_cta = (double)m->num_sms * threads;
    const int occ_work = (int)std::lround((double)work_warps * 32.0 / (rays_per_sm_cta * slots_per_lane));
    occ = std::max(1, std::min(occ, occ_work));
  }
  long long blocks = (long long)m->num_sms * occ;
  const long long need = (work_warps + (threads / 32) - 1) / (threads / 32);
  if (need < blocks) blocks = std::max(1ll, need);
  std::pair<cudaEvent_t, cudaEvent_t>* ev = nullptr;
  if (g_kt.on && kind != KernelKind::kFused) {
    g_kt.name = kernel_desc(m, kind, fmode);
    if (g_kt.used == g_kt.ev.size()) {
      std::pair<cudaEvent_t, cudaEvent_t> p;
      CUDA_TRY(cudaEventCreate(&p.first));
      CUDA_TRY(cudaEventCreate(&p.second));
      g_kt.ev.push_back(p);
    }
    ev = &g_kt.ev[g_kt.used++];
    CUDA_TRY(cudaEventRecord(ev->first, s));
  }
  CUDA_TRY(cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(threads), args, smem, s));
  count_launch();
  if (ev) CUDA_TRY(cudaEventRecord(ev->second, s));
  return FVSRN_OK;
}

// auto: tcgen05 at 64-wide (measured 27.0 vs 34.2 ms) and, since the biases ride in the
// MMA (tc_bias_mma), at 32-wide too (cfg 2 3.02 vs 3.11 ms for mma.sync); FVSRN_TC32=0
// keeps mma.sync at 32-wide.  Small frames take the two-lanes-per-ray mma.sync kernel.
const bool g_tc32_auto = [] {
  const char* e = std::getenv("FVSRN_TC32");
  return !(e && e[0] == '0');
}();
bool use_tc(const fvsrn_model* m) {
  if (!m->tc_ok || !fast_path(m, KernelKind::kDVR)) return false;
  if (dvr_mode() == DvrMode::kTC) return true;
  return dvr_mode() == DvrMode::kAuto && (m->hid_pad == 64 || (m->hid_pad == 32 && g_tc32_auto));
}

// Stream-ordered per-frame ray records: a, b (+ d for direction-input models).
int alloc_recs(const fvsrn_model* m, long long n_slots, cudaStream_t s, RayRecs& rr, void*& buf) {
  const size_t n = (size_t)std::max(1ll, n_slots);
  const int parts = m->dir_mode != 0 ? 3 : 2;
  CUDA_TRY(cudaMallocAsync(&buf, n * sizeof(float4) * parts, s));
  float4* f = (float4*)buf;
  rr.a = f;
  rr.b = f + n;
  rr.d = parts == 3 ? f + 2 * n : nullptr;
  return FVSRN_OK;
}

// The fused DVR launch: tcgen05 kernel for the default shapes (FVSRN_DVR=tc), else the
// warp-specialised or single-role mma.sync kernel.  Same arguments for all three.
int launch_dvr(const fvsrn_model* m, NetDev& net, FeatDev& fd, const TFDev*& tfp, const float*& b0,
               MarchDev& md, CamDev& cam, ShardDev& sh, int& explicit_rays, RayRecs& rr,
               long long& n_slots, float*& d_out, unsigned long long*& queue,
               unsigned long long*& evc, unsigned long long*& nfc, cudaStream_t s) {
  if (n_slots <= 0) return FVSRN_OK;
  // static fp16 grid in the march: texture units (fmode 1) or exact-weight loads (fmode 2)
  const bool static_tex = FVSRN_TEX_SPECIAL && fd.tex_on && !fd.tex_u8 && fd.tex_w == 0.f;
  const bool static_ldg = FVSRN_TEX_SPECIAL && !fd.tex_on && fd.grid != nullptr && fd.f_pad == 16;
  const int fmode = static_tex ? 1 : 2;
  // a camera frame of a density-head model with a static fp16 grid: the branch-free
  // frame-specialised kernels
  const bool frame = (static_tex || static_ldg) && fast_path(m, KernelKind::kDVR) &&
                     m->head == FVSRN_HEAD_DENSITY && !explicit_rays;
  // small and medium frames (up to ~5x the resident lanes of a full launch, ~690^2): two
  // lanes per ray halve the longest rays' sequential march (tools/frame_sweep.py, cfg-2 model:
  // 256^2 0.54 -> 0.40 ms, 512^2 1.13 -> 0.91, 640^2 1.39 -> 1.32, 768^2 equal).  Decided on
  // the whole frame (W x H), not this rank's share, so every shard of a multi-GPU frame runs
  // the same kernel as the 1-GPU frame (bit-identical assembly).
  static const double pair_frac = [] {
    const char* e = std::getenv("FVSRN_PAIR_FRAC");
    return e ? std::atof(e) : 5.0;
  }();
  const long long full_lanes = (long long)m->num_sms * kThreads * kMinBlocks;
  // four lanes per ray up to 2x the resident lanes (~435^2; tools/frame_sweep.py, cfg-2
  // model at stepsize 1/256: 128^2 0.32 -> 0.21 ms, 256^2 0.44 -> 0.38, 320^2 0.61 -> 0.52,
  // 384^2 0.69 -> 0.65, 512^2 equal); FVSRN_QUAD_FRAC overrides (0 = off)
  static const double quad_frac = [] {
    const char* e = std::getenv("FVSRN_QUAD_FRAC");
    return e ? std::atof(e) : 2.0;
  }();
  const double frame_px = (double)cam.W * (double)cam.H;
  const bool small = frame && m->hid_pad == 32 && dvr_mode() != DvrMode::kTC &&
                     frame_px <= pair_frac * (double)full_lanes;
  void* args[] = {&net, &fd, &tfp, &b0, &md, &cam, &sh, &explicit_rays, &rr, &n_slots, &d_out, &queue, &evc, &nfc};
  // eight lanes per ray up to 1.25x (~345^2; stepsize 1/256: 128^2 0.218 -> 0.178 ms, 192^2
  // 0.298 -> 0.252, 320^2 0.524 -> 0.508; 384^2 is better with four); FVSRN_OCTO_FRAC overrides
  static const double octo_frac = [] {
    const char* e = std::getenv("FVSRN_OCTO_FRAC");
    return e ? std::atof(e) : 1.25;
  }();
  if (small && frame_px <= octo_frac * (double)full_lanes)
    return launch(m, KernelKind::kDVROcto, stage_smem_bytes(net, true, m->k0), args, s, n_slots / 4 + 1,
                  fmode);
  if (small && frame_px <= quad_frac * (double)full_lanes)
    return launch(m, KernelKind::kDVRQuad, stage_smem_bytes(net, true, m->k0), args, s, n_slots / 8 + 1,
                  fmode);
  if (small)
    return launch(m, KernelKind::kDVRPair, stage_smem_bytes(net, true, m->k0), args, s, n_slots / 16 + 1,
                  fmode);
  if (use_tc(m)) {
    TcNetDev tn{m->d_wtc, m->d_btc, m->head};
    void* targs[] = {&tn, &fd, &tfp, &b0, &md, &cam, &sh, &explicit_rays, &rr, &n_slots, &d_out, &queue, &evc, &nfc};
    const KernelKind k = frame ? KernelKind::kDVRTCTex : KernelKind::kDVRTC;
    return launch(m, k, tc_smem_bytes(m->hid_pad), targs, s, n_slots / 32 + 1, fmode);
  }
  if (dvr_mode() == DvrMode::kWS)
    return launch(m, KernelKind::kDVRWS, ws_smem_bytes(net, m->k0), args, s, n_slots / 32 + 1);
  if (dvr_mode() == DvrMode::kDual && fast_path(m, KernelKind::kDVR) && m->hid_pad == 32)
    return launch(m, KernelKind::kDVRDual, dual_smem_bytes(net, m->k0), args, s, n_slots / 64 + 1);
  if (dvr_mode() == DvrMode::kPipe && fast_path(m, KernelKind::kDVR))
    return launch(m, KernelKind::kDVRPipe, pipe_smem_bytes(net, m->k0), args, s, n_slots / 32 + 1);
  const KernelKind k = frame ? KernelKind::kDVRTex : KernelKind::kDVR;
  return launch(m, k, stage_smem_bytes(net, true, m->k0), args, s, n_slots / 32 + 1, fmode);
}

MarchDev march_for(const fvsrn_settings* st) {
  MarchDev md{};
  md.stepsize = st->stepsize;
  md.max_steps = st->max_steps;
  md.et_alpha = st->early_term_alpha;
  md.eps_blend = st->eps_blend;
  md.eps1_f = (float)(1.0 - st->eps_blend);
  md.et_f = (float)st->early_term_alpha;
  for (int c = 0; c < 3; ++c) md.bg[c] = (float)st->background[c];
  return md;
}

int check_settings(const fvsrn_settings* st) {
  if (!st) return fail(FVSRN_EINVAL, "settings required");
  if (!(st->stepsize > 0)) return fail(FVSRN_EINVAL, "stepsize must be positive");
  if (!(st->early_term_alpha >= 0.0 && st->early_term_alpha <= 1.0))
    return fail(FVSRN_EINVAL, "early termination threshold must lie in [0,1]");
  if (st->max_steps < 1) return fail(FVSRN_EINVAL, "max_steps must be >= 1");
  return FVSRN_OK;
}

int check_source(const fvsrn_model* m, const fvsrn_tf* tf, double t) {
  if (m->head == FVSRN_HEAD_DENSITY && !tf)
    return fail(FVSRN_EINVAL, "density-head models need a transfer function to render");
  if (m->head == FVSRN_HEAD_COLOR && tf)
    return fail(FVSRN_EINVAL, "color-head models do not take a transfer function");
  if (!m->temporal && !std::isnan(t)) return fail(FVSRN_EINVAL, "timestep supplied to a non-temporal model");
  if (m->temporal && std::isnan(t)) return fail(FVSRN_EINVAL, "temporal model requires a timestep to render");
  return FVSRN_OK;
}

CamDev cam_for(const fvsrn_camera* c) {
  // Same op sequence as render.py:78-86 (used when the caller does not pass the
  // numpy-computed basis; the Python shim always passes it, see render.py host mirror).
  CamDev cd{};
  double f[3], r[3], u[3];
  for (int a = 0; a < 3; ++a) f[a] = c->target[a] - c->eye[a];
  double nf = std::sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
  for (int a = 0; a < 3; ++a) f[a] /= nf;
  r[0] = f[1] * c->up[2] - f[2] * c->up[1];
  r[1] = f[2] * c->up[0] - f[0] * c->up[2];
  r[2] = f[0] * c->up[1] - f[1] * c->up[0];
  double nr = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  for (int a = 0; a < 3; ++a) r[a] /= nr;
  u[0] = r[1] * f[2] - r[2] * f[1];
  u[1] = r[2] * f[0] - r[0] * f[2];
  u[2] = r[0] * f[1] - r[1] * f[0];
  for (int a = 0; a < 3; ++a) { cd.eye[a] = c->eye[a]; cd.fwd[a] = f[a]; cd.right[a] = r[a]; cd.up[a] = u[a]; }
  cd.half_h = std::tan(c->fov_y / 2.0);
  cd.half_w = cd.half_h * c->width / c->height;
  cd.W = c->width;
  cd.H = c->height;
  return cd;
}

}  // namespace

// ============================================================================ C ABI
extern "C" {

const char* fvsrn_last_error(void) { return g_err.c_str(); }

// The stream-ordered pool of the calling thread's device keeps freed blocks (per-call
// scratch would otherwise be unmapped and remapped at every synchronisation).
static void keep_pool_blocks() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return; }
  std::lock_guard<std::mutex> l(mu);
  for (int d : done) if (d == dev) return;
  cudaMemPool_t pool;
  uint64_t keep = UINT64_MAX;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  cudaGetLastError();
  done.push_back(dev);
}

static int make_train_net(const fvsrn_train_desc* d, long long rows, TrainNetDev& net,
                          bool check_inputs = true) {
  keep_pool_blocks();
  const int L = d->layers;
  if (L < 1 || L > kTrainMaxLayers) return fail(FVSRN_EINVAL, "layer count out of range");
  if (d->hidden > 256 || d->d_in > 256 || d->d_out < 1 || d->d_out > 4)
    return fail(FVSRN_ECAPACITY, "network too wide for the training kernel");
  const int tl = d->time_mode == 0 ? 0 : ((d->time_mode & 1) ? 1 : 0) + ((d->time_mode & 2) ? 2 * d->time_fourier_count : 0);
  const int rw = d->raw_width ? d->raw_width : 3, fi = d->fourier_in ? d->fourier_in : 3;
  if ((rw != 3 && rw != 6) || (fi != 3 && fi != 6)) return fail(FVSRN_EINVAL, "raw / Fourier input width must be 3 or 6");
  if (check_inputs && d->d_in != rw + 2 * d->fourier_m + tl + (d->grid_resolution > 0 ? d->grid_channels : 0))
    return fail(FVSRN_EINVAL, "input width does not match the model's input layout");
  if (d->n_keyframes < 0 || d->n_keyframes > 16 || (d->n_keyframes > 0 && !d->keyframe_times))
    return fail(FVSRN_EINVAL, "keyframes: 0..16 with their times");
  if (d->n_keyframes > 0 && d->grid_resolution < 2) return fail(FVSRN_EINVAL, "temporal models need a grid");
  if (d->time_mode < 0 || d->time_mode > 3 || d->time_fourier_count > 16 ||
      ((d->time_mode & 2) && !d->time_b))
    return fail(FVSRN_EINVAL, "bad time features");
  if (d->fourier_m > 0 && !d->d_b_matrix) return fail(FVSRN_EINVAL, "Fourier matrix required");
  if (d->grid_resolution == 1) return fail(FVSRN_EINVAL, "need R >= 2");
  net = TrainNetDev{};
  net.layers = L; net.hidden = d->hidden; net.d_in = d->d_in; net.d_out = d->d_out;
  net.act = d->activation; net.head = d->head; net.m = d->fourier_m; net.bmat = d->d_b_matrix;
  net.raw_w = rw; net.fd_in = fi;
  net.grid_res = d->grid_resolution; net.grid_ch = d->grid_channels;
  net.n_kf = d->n_keyframes;
  for (int k = 0; k < d->n_keyframes; ++k) net.kf_times[k] = d->keyframe_times[k];
  net.time_mode = d->time_mode;
  net.time_l = (d->time_mode & 2) ? d->time_fourier_count : 0;
  for (int j = 0; j < net.time_l; ++j) net.time_b[j] = d->time_b[j];
  net.t0 = d->time_t0;
  net.t1 = d->time_t1;
  long long off = 0, io = 0, dof = 0;
  for (int l = 0; l < L; ++l) {
    const long long in_l = l == 0 ? d->d_in : d->hidden, out_l = l == L - 1 ? d->d_out : d->hidden;
    net.w_off[l] = off;
    off += in_l * out_l;
    net.in_off[l] = io;
    io += rows * in_l;
    net.d_off[l] = dof;
    dof += rows * out_l;
  }
  for (int l = 0; l < L; ++l) {
    net.b_off[l] = off;
    off += l == L - 1 ? d->d_out : d->hidden;
  }
  net.grid_off = off;
  return FVSRN_OK;
}

int32_t fvsrn_f32_eval(const fvsrn_train_desc* d, const float* d_params, const double* d_positions,
                       const double* d_dirs, const double* d_times, const float* d_x, int64_t n,
                       int32_t stage, float* d_out, void* stream) {
  if (!d || !d_params || !d_out || stage < 0 || stage > 3) return fail(FVSRN_EINVAL, "bad argument");
  if (n > 0 && ((stage < 3 && !d_positions) || (stage == 3 && !d_x))) return fail(FVSRN_EINVAL, "null argument");
  TrainNetDev net;
  int rc = make_train_net(d, 0, net, stage != 3);
  if (rc) return rc;
  if (stage < 3 && net.raw_w == 6 && !d_dirs) return fail(FVSRN_EINVAL, "direction mode requires view directions");
  if (stage < 3 && net.n_kf > 0 && !d_times) return fail(FVSRN_EINVAL, "temporal model requires timesteps");
  if (stage == 1 && net.grid_res == 0) return fail(FVSRN_EINVAL, "model has no latent grid");
  CUDA_TRY(launch_f32_eval(net, d_params, d_positions, d_dirs, d_times, d_x, (long long)n, stage, d_out,
                           (cudaStream_t)stream));
  count_launch();
  return FVSRN_OK;
}

int32_t fvsrn_train_world_grads(const fvsrn_train_desc* d, const float* d_params,
                                const double* d_positions, const double* d_times,
                                const float* d_reference, int64_t n,
                                float* d_grid_grad, float* d_inputs, float* d_preacts,
                                float* d_deltas, double* d_loss_sum, void* stream) {
  if (!d || !d_params || (n > 0 && (!d_positions || !d_reference || !d_inputs || !d_deltas)))
    return fail(FVSRN_EINVAL, "null argument");
  TrainNetDev net;
  int rc = make_train_net(d, n, net);
  if (rc) return rc;
  if (net.n_kf > 0 && n > 0 && !d_times) return fail(FVSRN_EINVAL, "temporal model requires timesteps");
  CUDA_TRY(launch_train_world(net, d_params, d_positions, net.n_kf > 0 ? d_times : nullptr, d_reference,
                              (long long)n, d_grid_grad,
                              d_inputs, d_preacts, d_deltas, d_loss_sum, (cudaStream_t)stream));
  count_launch();
  return FVSRN_OK;
}

int32_t fvsrn_mlp_forward_backward(const fvsrn_train_desc* d, const float* d_params, const float* d_x,
                                   const float* d_y_bar, int64_t n, float* d_y, float* d_inputs,
                                   float* d_preacts, float* d_deltas, float* d_x_bar, void* stream) {
  if (!d || !d_params || (n > 0 && (!d_x || !d_y || !d_inputs || (d_y_bar && !d_deltas))))
    return fail(FVSRN_EINVAL, "null argument");
  if (d->grid_resolution != 0 || d->n_keyframes != 0) return fail(FVSRN_EINVAL, "plain MLP: no grid / keyframes");
  if (d_y_bar && d->d_out > 4) return fail(FVSRN_EINVAL, "backward: output width must be <= 4");
  TrainNetDev net;
  int rc = make_train_net(d, n, net, false);
  if (rc) return rc;
  CUDA_TRY(launch_mlp_grads(net, d_params, d_x, d_y_bar, (long long)n, d_y, d_inputs, d_preacts,
                            d_deltas, d_y_bar ? d_x_bar : nullptr, (cudaStream_t)stream));
  count_launch();
  return FVSRN_OK;
}

int32_t fvsrn_layer_grads(const fvsrn_train_desc* d, const float* d_inputs, const float* d_deltas,
                          int64_t cap_rows, int64_t n, float* d_grads, int32_t accumulate, void* stream) {
  if (!d || (n > 0 && (!d_inputs || !d_deltas || !d_grads))) return fail(FVSRN_EINVAL, "null argument");
  if (n > cap_rows) return fail(FVSRN_EINVAL, "more rows than the caches hold");
  TrainNetDev net;
  int rc = make_train_net(d, cap_rows, net, false);
  if (rc) return rc;
  CUDA_TRY(launch_layer_grads(net, d_inputs, d_deltas, (long long)n, d_grads, accumulate != 0,
                              (cudaStream_t)stream));
  count_launch();
  return FVSRN_OK;
}

int32_t fvsrn_grid_sample_backward(int32_t resolution, int32_t channels, const double* d_positions,
                                   const float* d_z_bar, int64_t n, float* d_grad, void* stream) {
  keep_pool_blocks();
  if (resolution < 2 || channels < 1) return fail(FVSRN_EINVAL, "grid must have resolution >= 2 and channels >= 1");
  if (n > 0 && (!d_positions || !d_z_bar || !d_grad)) return fail(FVSRN_EINVAL, "null argument");
  CUDA_TRY(launch_grid_scatter(resolution, channels, d_positions, d_z_bar, (long long)n, d_grad,
                               (cudaStream_t)stream));
  count_launch();
  return FVSRN_OK;
}

int32_t fvsrn_model_grads(const fvsrn_train_desc* d, const float* d_params, const double* d_positions,
                          const double* d_dirs, const double* d_times, const float* d_raw_bar, int64_t n,
                          float* d_grid_grad, float* d_inputs, float* d_preacts, float* d_deltas,
                          void* stream) {
  if (!d || !d_params || (n > 0 && (!d_positions || !d_raw_bar || !d_inputs || !d_deltas)))
    return fail(FVSRN_EINVAL, "null argument");
  TrainNetDev net;
  int rc = make_train_net(d, n, net);
  if (rc) return rc;
  if (net.n_kf > 0 && n > 0 && !d_times) return fail(FVSRN_EINVAL, "temporal model requires timesteps");
  if (d->raw_width > 3 && n > 0 && !d_dirs) return fail(FVSRN_EINVAL, "direction mode requires view directions");
  CUDA_TRY(launch_model_grads(net, d_params, d_positions, d->raw_width > 3 ? d_dirs : nullptr,
                              net.n_kf > 0 ? d_times : nullptr, d_raw_bar, (long long)n, d_grid_grad,
                              d_inputs, d_preacts, d_deltas, (cudaStream_t)stream));
  count_launch();
  return FVSRN_OK;
}

int32_t fvsrn_train_screen_forward(const fvsrn_train_desc* d, const float* d_params,
                                   const double* d_origins, const double* d_dirs, int64_t n,
                                   const fvsrn_settings* st, float* d_pixels, double* d_color,
                                   double* d_alpha, double* d_tmin, double* d_ds, int32_t* d_nsteps,
                                   void* stream) {
  if (!d || !d_params || !st || (n > 0 && (!d_origins || !d_dirs || !d_pixels || !d_color ||
                                           !d_alpha || !d_tmin || !d_ds || !d_nsteps)))
    return fail(FVSRN_EINVAL, "null argument");
  if (d->head != FVSRN_HEAD_COLOR) return fail(FVSRN_EINVAL, "screen-space training requires a color-head model");
  if (d->n_keyframes > 0 || d->time_mode != 0) return fail(FVSRN_EINVAL, "screen-space training is static");
  int rc = check_settings(st);
  if (rc) return rc;
  TrainNetDev net;
  if ((rc = make_train_net(d, 0, net))) return rc;
  const MarchDev md = march_for(st);
  CUDA_TRY(launch_screen_forward(net, d_params, d_origins, d_dirs, (long long)n, md, d_pixels, d_color,
                                 d_alpha, d_tmin, d_ds, d_nsteps, (cudaStream_t)stream));
  count_launch();
  return FVSRN_OK;
}

int32_t fvsrn_train_screen_backward(const fvsrn_train_desc* d, const float* d_params,
                                    const double* d_origins, const double* d_dirs, int64_t n,
                                    double eps_blend, const double* d_color, const double* d_alpha,
                                    const double* d_tmin, const double* d_ds, const int32_t* d_nsteps,
                                    const int64_t* d_row_offset, const float* d_image_adjoint,
                                    const double* d_background, int64_t cap_rows, float* d_inputs,
                                    float* d_preacts, float* d_deltas, float* d_grid_grad, void* stream) {
  if (!d || !d_params || (n > 0 && (!d_origins || !d_dirs || !d_color || !d_alpha || !d_tmin ||
                                    !d_ds || !d_nsteps || !d_row_offset || !d_image_adjoint ||
                                    !d_background || !d_inputs || !d_deltas)))
    return fail(FVSRN_EINVAL, "null argument");
  if (d->head != FVSRN_HEAD_COLOR) return fail(FVSRN_EINVAL, "raymarch_backward trains color-head models only");
  TrainNetDev net;
  int rc = make_train_net(d, cap_rows, net);
  if (rc) return rc;
  CUDA_TRY(launch_screen_backward(net, d_params, d_origins, d_dirs, (long long)n, eps_blend, d_color,
                                  d_alpha, d_tmin, d_ds, d_nsteps, (const long long*)d_row_offset,
                                  d_image_adjoint, d_background, (long long)cap_rows, d_inputs, d_preacts,
                                  d_deltas, d_grid_grad, (cudaStream_t)stream));
  count_launch();
  return FVSRN_OK;
}

int32_t fvsrn_adam_step(float* d_params, const float* d_grads, float* d_m, float* d_v, int64_t n,
                        double lr, double beta1, double beta2, double eps, int32_t t,
                        unsigned long long* d_nonfinite, void* stream) {
  if (!d_params || !d_grads || !d_m || !d_v || !d_nonfinite || t < 1) return fail(FVSRN_EINVAL, "bad argument");
  AdamConsts k;
  k.lr = (float)lr; k.b1 = (float)beta1; k.b2 = (float)beta2;
  k.one_m_b1 = (float)(1.0 - beta1); k.one_m_b2 = (float)(1.0 - beta2); k.eps = (float)eps;
  k.bc1 = (float)(1.0 - std::pow(beta1, t)); k.bc2 = (float)(1.0 - std::pow(beta2, t));
  CUDA_TRY(launch_adam(d_params, d_grads, d_m, d_v, (long long)n, k, d_nonfinite, (cudaStream_t)stream));
  count_launch();
  count_launch();
  return FVSRN_OK;
}

int32_t fvsrn_ipc_export(void* d_ptr, uint8_t handle[64], uint64_t* offset) {
  if (!d_ptr || !handle || !offset) return fail(FVSRN_EINVAL, "null argument");
  // cudaIpcGetMemHandle names the whole cudaMalloc allocation and cudaIpcOpenMemHandle
  // maps its BASE, so a pointer carved from a caching allocator's segment travels as
  // (handle, offset from the allocation base).
  void* base = nullptr;
  size_t size = 0;
  if (int rc = alloc_range(d_ptr, &base, &size)) return rc;
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, d_ptr));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle, &h, 64);
  *offset = (uint64_t)((char*)d_ptr - (char*)base);
  return FVSRN_OK;
}

int32_t fvsrn_ipc_open(const uint8_t handle[64], uint64_t offset, int32_t device, void** d_ptr) {
  if (!handle || !d_ptr) return fail(FVSRN_EINVAL, "null argument");
  CUDA_TRY(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  void* base = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *d_ptr = (char*)base + offset;
  std::lock_guard<std::mutex> g(g_ipc_mu);
  g_ipc_bases[*d_ptr] = base;
  return FVSRN_OK;
}

int32_t fvsrn_ipc_close(void* d_ptr) {
  if (!d_ptr) return FVSRN_OK;
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> g(g_ipc_mu);
    auto it = g_ipc_bases.find(d_ptr);
    if (it == g_ipc_bases.end()) return fail(FVSRN_EINVAL, "pointer was not opened by fvsrn_ipc_open");
    base = it->second;
    g_ipc_bases.erase(it);
  }
  CUDA_TRY(cudaIpcCloseMemHandle(base));
  return FVSRN_OK;
}

int32_t fvsrn_kernel_timer(int32_t enable) {
  g_kt.on = enable != 0;
  g_kt.used = 0;
  g_kt.launches = 0;
  return FVSRN_OK;
}

int32_t fvsrn_kernel_timer_read(double* dominant_ms, int64_t* dominant_launches, int64_t* total_launches) {
  double ms = 0.0;
  for (size_t i = 0; i < g_kt.used; ++i) {
    CUDA_TRY(cudaEventSynchronize(g_kt.ev[i].second));
    float e = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&e, g_kt.ev[i].first, g_kt.ev[i].second));
    ms += e;
  }
  if (dominant_ms) *dominant_ms = ms;
  if (dominant_launches) *dominant_launches = (int64_t)g_kt.used;
  if (total_launches) *total_launches = g_kt.launches;
  g_kt.used = 0;
  g_kt.launches = 0;
  return FVSRN_OK;
}

int32_t fvsrn_kernel_timer_info(char* buf, int32_t cap) {
  if (!buf || cap < 1) return fail(FVSRN_EINVAL, "null buffer");
  std::snprintf(buf, (size_t)cap, "%s", g_kt.name.c_str());
  return FVSRN_OK;
}

int32_t fvsrn_set_grid_sampler(int32_t mode) {
  if (mode < 0 || mode > 2) return -fail(FVSRN_EINVAL, "grid sampler mode must be 0..2");
  return g_grid_mode.exchange(mode);
}

int32_t fvsrn_set_dvr_kernel(int32_t mode) {
  // failures are negative (-FVSRN_EINVAL): every non-negative value is a previous mode
  if (mode < 0 || mode > 5) return -fail(FVSRN_EINVAL, "DVR kernel mode must be 0..5");
  if (!FVSRN_AB_VARIANTS && (mode == (int)DvrMode::kWS || mode == (int)DvrMode::kPipe ||
                             mode == (int)DvrMode::kDual))
    return -fail(FVSRN_EINVAL, "DVR variant not in this build (A/B builds: -DFVSRN_AB_VARIANTS=1)");
  return g_dvr_mode_i.exchange(mode);
}
const char* fvsrn_version(void) { return "fvsrn_b200 0.1.0 (sm_100a, mma.sync f16/f32)"; }

int32_t fvsrn_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

static int eval_common(fvsrn_model_t m, const double* p, const double* dd, int64_t n, double t,
                       float* out, int want_head);

// Upload-time accuracy probe of the texture sampler: the model's outputs at 2^18
// deterministic uniform positions (and unit directions), once through the texture units
// and once through the exact-weight LDG sampler, per keyframe time for temporal models.
// Auto mode keeps the texture units only if max |tex - ldg| <= FVSRN_TEX_TOL (default
// 1e-3, a tenth of the density tolerance).  ~2 ms per upload.
static int probe_texture_sampler(fvsrn_model_t m) {
  m->tex_ok = false;
  if (m->tex.empty()) return FVSRN_OK;
  static const double tol = [] {
    const char* e = std::getenv("FVSRN_TEX_TOL");
    return e ? std::atof(e) : 1e-3;
  }();
  const int64_t n = 1 << 18;
  const int oc = m->head == FVSRN_HEAD_DENSITY ? 1 : 4;
  std::vector<double> p((size_t)n * 3), d((size_t)n * 3);
  uint64_t x = 0x9E3779B97F4A7C15ull;
  auto next = [&x] {          // splitmix64 -> [0, 1)
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return (double)((z ^ (z >> 31)) >> 11) * (1.0 / 9007199254740992.0);
  };
  for (auto& v : p) v = next();
  for (int64_t i = 0; i < n; ++i) {
    double a = 2.0 * next() - 1.0, b = 6.283185307179586 * next(), r = std::sqrt(1.0 - a * a);
    d[3 * i] = r * std::cos(b); d[3 * i + 1] = r * std::sin(b); d[3 * i + 2] = a;
  }
  std::vector<float> a((size_t)n * oc), b((size_t)n * oc);
  std::vector<double> ts;
  if (m->temporal) ts = m->kf_times;
  else ts.push_back(std::nan(""));
  float err = 0.f;
  const double* dd = m->dir_mode != FVSRN_DIR_POS ? d.data() : nullptr;
  for (double t : ts) {
    g_sampler_override = 1;
    int rc = eval_common(m, p.data(), dd, n, t, a.data(), m->head);
    g_sampler_override = 2;
    if (!rc) rc = eval_common(m, p.data(), dd, n, t, b.data(), m->head);
    g_sampler_override = 0;
    if (rc) return rc;
    for (size_t i = 0; i < a.size(); ++i) err = std::max(err, std::fabs(a[i] - b[i]));
  }
  m->tex_probe_err = err;
  m->tex_ok = err <= tol;
  return FVSRN_OK;
}

int32_t fvsrn_model_sampler(fvsrn_model_t m, int32_t* tex_ok, float* probe_err) {
  if (!m) return fail(FVSRN_EINVAL, "null model");
  if (tex_ok) *tex_ok = m->tex_ok ? 1 : 0;
  if (probe_err) *probe_err = m->tex_probe_err;
  return FVSRN_OK;
}

int32_t fvsrn_model_create(const fvsrn_model_desc* d, int32_t device, fvsrn_model_t* out) {
  if (!d || !out) return fail(FVSRN_EINVAL, "null argument");
  *out = nullptr;
  if (d->layers < 1 || d->hidden < 1) return fail(FVSRN_EINVAL, "layers and hidden must be positive");
  if (d->layers > kMaxLayers) return fail(FVSRN_ECAPACITY, "too many layers for the GPU path");
  if (d->head != FVSRN_HEAD_DENSITY && d->head != FVSRN_HEAD_COLOR) return fail(FVSRN_EINVAL, "bad head");
  if (d->activation < 0 || d->activation > 4) return fail(FVSRN_EINVAL, "bad activation");
  const int d_out = d->head == FVSRN_HEAD_DENSITY ? 1 : 4;
  if (d->d_out != d_out) return fail(FVSRN_EINVAL, "d_out does not match head");
  auto* m = new fvsrn_model();
  std::unique_ptr<fvsrn_model> guard(m);
  m->device = device;
  m->layers = d->layers;
  m->hidden = d->hidden;
  m->hid_pad = round_up(d->hidden, 16);
  if (m->hid_pad > kMaxHidden)
    return fail(FVSRN_ECAPACITY, "hidden width " + std::to_string(d->hidden) + " exceeds the GPU path limit 128");
  m->d_in = d->d_in;
  m->d_out = d_out;
  m->act = d->activation;
  m->head = d->head;
  m->dir_mode = d->direction_mode;
  m->raw_w = d->direction_mode != FVSRN_DIR_POS ? 6 : 3;
  m->fourier_mode = d->fourier_m > 0 ? d->fourier_mode : FVSRN_FOURIER_OFF;
  m->m = m->fourier_mode == FVSRN_FOURIER_OFF ? 0 : d->fourier_m;
  m->fd_in = d->fourier_d_in;
  m->time_mode = d->time_mode;
  m->tfc = d->time_fourier_count;
  m->T = (d->time_mode == FVSRN_TIME_NONE) ? 0
       : (d->time_mode == FVSRN_TIME_DIRECT) ? 1
       : (d->time_mode == FVSRN_TIME_FOURIER) ? 2 * d->time_fourier_count
                                              : 1 + 2 * d->time_fourier_count;
  if (m->time_mode == FVSRN_TIME_FOURIER || m->time_mode == FVSRN_TIME_BOTH) {
    if (!d->time_b) return fail(FVSRN_EINVAL, "time Fourier matrix required");
    m->time_b.assign(d->time_b, d->time_b + d->time_fourier_count);
  }
  m->has_time_range = d->has_time_range != 0;
  m->time_range[0] = d->time_range[0];
  m->time_range[1] = d->time_range[1];
  m->temporal = d->temporal != 0;
  if (m->temporal) {
    if (d->n_grids < 1 || !d->keyframe_times) return fail(FVSRN_EINVAL, "temporal model needs keyframes");
    m->kf_times.assign(d->keyframe_times, d->keyframe_times + d->n_grids);
    for (size_t i = 1; i < m->kf_times.size(); ++i)
      if (!(m->kf_times[i] > m->kf_times[i - 1]))
        return fail(FVSRN_EINVAL, "keyframe times must be strictly increasing");
  }
  m->R = d->grid_resolution;
  m->F = d->grid_resolution > 0 ? d->grid_channels : 0;
  m->f_pad = round_up(m->F, 8);
  if (m->R == 1 || (m->R > 0 && m->F < 1)) return fail(FVSRN_EINVAL, "need R >= 2 and F >= 1");
  // ---- device feature layout: [z | (sin,cos) pairs | raw] padded to 16
  m->four_off = m->f_pad;
  m->raw_off = m->f_pad + 2 * m->m;
  const int width = m->raw_off + m->raw_w;
  m->k0 = round_up(width, 16);
  const int ref_w = m->raw_w + 2 * m->m + m->T + m->F;
  if (ref_w != d->d_in)
    return fail(FVSRN_EINVAL, "input width " + std::to_string(d->d_in) + " does not match config (" +
                                  std::to_string(ref_w) + ")");
  if (m->k0 > 256 || round_up(d->d_in, 16) > 256) return fail(FVSRN_ECAPACITY, "input too wide for the GPU path");
  if (m->fourier_mode == FVSRN_FOURIER_NERF || m->fourier_mode == FVSRN_FOURIER_RANDOM) {
    if (!d->b_matrix) return fail(FVSRN_EINVAL, "Fourier matrix required");
    if (m->fd_in != 3 && m->fd_in != 6) return fail(FVSRN_EINVAL, "Fourier input must be 3 or 6 wide");
  }
  if (m->fourier_mode == FVSRN_FOURIER_NERF) {
    // the recurrence assumes B = nerf_rows(m, fd_in) (nn.py:47-57); verify it
    for (int i = 0; i < m->m; ++i)
      for (int a = 0; a < m->fd_in; ++a) {
        float want = (a == i % m->fd_in) ? (float)(2.0 * M_PI * std::ldexp(1.0, i / m->fd_in)) : 0.f;
        if (d->b_matrix[i * m->fd_in + a] != want)
          return fail(FVSRN_EINVAL, "nerf Fourier matrix is not the stacked powers-of-two identity");
      }
  }
  CUDA_TRY(cudaSetDevice(device));
  {
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) return fail(FVSRN_ECUDA, "sm_100a device required");
    m->num_sms = prop.multiProcessorCount;
    // per-frame scratch (ray records, framebuffers) comes from the stream-ordered pool;
    // keep freed blocks cached instead of unmapping them at every synchronisation
    cudaMemPool_t pool;
    CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  if (m->fourier_mode == FVSRN_FOURIER_RANDOM) {
    int rc = upload(d->b_matrix, sizeof(float) * m->m * m->fd_in, (void**)&m->d_bmat);
    if (rc) return rc;
  }
  // ---- grids (fp16, channel-padded); u8 grids are dequantised exactly as grid.py:170-172
  if (m->R > 0) {
    const int ng = m->temporal ? d->n_grids : 1;
    const size_t nvals = (size_t)m->R * m->R * m->R * m->F;
    for (int gi = 0; gi < ng; ++gi) {
      std::vector<float> f32(nvals);
      if (d->grid_precision == FVSRN_GRID_U8) {
        const uint8_t* c = d->grid_codes[gi];
        const float* mn = d->grid_mins[gi];
        const float* mx = d->grid_maxs[gi];
        for (size_t i = 0; i < nvals; ++i) {
          const int ch = (int)(i % m->F);
          f32[i] = mn[ch] + ((float)c[i] / 255.0f) * (mx[ch] - mn[ch]);
        }
      } else {
        if (!d->grids || !d->grids[gi]) return fail(FVSRN_EINVAL, "grid values required");
        std::memcpy(f32.data(), d->grids[gi], nvals * sizeof(float));
      }
      auto h = to_half_padded(f32.data(), m->R, m->F, m->f_pad);
      __half* dg = nullptr;
      int rc = upload(h.data(), h.size() * sizeof(__half), (void**)&dg);
      if (rc) return rc;
      m->grids.push_back(dg);
      if (m->f_pad == 16) {
        if (d->grid_precision == FVSRN_GRID_U8) {
          // sample the 8-bit codes directly: RGBA8 textures + in-kernel
          // dequantisation with the per-channel (min, max) of grid.py:157-172
          std::vector<uint8_t> codes(d->grid_codes[gi], d->grid_codes[gi] + nvals);
          if ((rc = make_grid_textures_t(m, codes, m->F))) return rc;
          std::array<float, 16> mn{}, sp{};
          for (int c = 0; c < m->F; ++c) {
            mn[c] = d->grid_mins[gi][c];
            sp[c] = d->grid_maxs[gi][c] - d->grid_mins[gi][c];
          }
          m->qmin.push_back(mn);
          m->qspan.push_back(sp);
          m->tex_u8 = true;
        } else if ((rc = make_grid_textures(m, h))) {
          return rc;
        }
      }
    }
  }
  // ---- weights: sample pack (device column order, time columns folded out) ...
  const int L = m->layers;
  std::vector<int> N(L), Ks(L), Kx(L);
  for (int l = 0; l < L; ++l) {
    N[l] = (l == L - 1) ? 8 : m->hid_pad;
    Ks[l] = (l == 0) ? m->k0 : m->hid_pad;
    Kx[l] = (l == 0) ? round_up(d->d_in, 16) : m->hid_pad;
  }
  std::vector<std::vector<float>> ws(L), wx(L), bs(L);
  for (int l = 0; l < L; ++l) {
    const int out_l = (l == L - 1) ? d_out : m->hidden;
    const int in_l = (l == 0) ? d->d_in : m->hidden;
    const float* W = d->weights[l];
    const float* B = d->biases[l];
    if (!W || !B) return fail(FVSRN_EINVAL, "weights/biases required");
    ws[l].assign((size_t)N[l] * Ks[l], 0.f);
    wx[l].assign((size_t)N[l] * Kx[l], 0.f);
    bs[l].assign(N[l], 0.f);
    for (int o = 0; o < out_l; ++o) {
      bs[l][o] = B[o];
      for (int i = 0; i < in_l; ++i) {
        const float w = W[(size_t)o * in_l + i];
        wx[l][(size_t)o * Kx[l] + i] = w;
        int dc = i;
        if (l == 0) {
          // reference column i -> device column (model.py:3-6 layout)
          if (i < m->raw_w) dc = m->raw_off + i;
          else if (i < m->raw_w + m->m) dc = m->four_off + 2 * (i - m->raw_w);
          else if (i < m->raw_w + 2 * m->m) dc = m->four_off + 2 * (i - m->raw_w - m->m) + 1;
          else if (i < m->raw_w + 2 * m->m + m->T) dc = -1;   // time: folded into bias
          else dc = i - (m->raw_w + 2 * m->m + m->T);
        }
        if (dc >= 0) ws[l][(size_t)o * Ks[l] + dc] = w;
      }
    }
  }
  // snake family (see act_h in fvsrn_device.cuh): every layer feeding an activation is
  // pre-scaled by 2 (accumulator a = 2x), and the activation's affine tail
  // act = f*h + 1/2 (f = 1/4 snake_alt, 1/2 snake) is folded into the next layer:
  // W' = s_out * f * W,  b' = s_out * (b + rowsum(W)/2).  Powers of two: exact in fp16.
  float s_out0 = 1.f;
  if (m->act == FVSRN_ACT_SNAKE || m->act == FVSRN_ACT_SNAKE_ALT) {
    const double f = m->act == FVSRN_ACT_SNAKE_ALT ? 0.25 : 0.5;
    for (int l = 0; l < L; ++l) {
      const double so = (l < L - 1) ? 2.0 : 1.0;
      const double fin = (l >= 1) ? f : 1.0;
      const int in_l = (l == 0) ? d->d_in : m->hidden;
      for (int o = 0; o < N[l]; ++o) {
        double rs = 0.0;
        if (l >= 1 && o < ((l == L - 1) ? d_out : m->hidden))
          for (int i = 0; i < in_l; ++i) rs += (double)d->weights[l][(size_t)o * in_l + i];
        bs[l][o] = (float)(so * ((double)bs[l][o] + 0.5 * rs));
        for (int i = 0; i < Ks[l]; ++i) ws[l][(size_t)o * Ks[l] + i] *= (float)(so * fin);
        for (int i = 0; i < Kx[l]; ++i) wx[l][(size_t)o * Kx[l] + i] *= (float)(so * fin);
      }
    }
    s_out0 = L > 1 ? 2.f : 1.f;
  }
  m->n0 = N[0];
  m->b0_static = bs[0];
  if (m->T > 0) {
    m->w0_time.assign((size_t)N[0] * m->T, 0.f);
    const int out0 = (L == 1) ? d_out : m->hidden;
    for (int o = 0; o < out0; ++o)
      for (int j = 0; j < m->T; ++j)
        m->w0_time[(size_t)o * m->T + j] =
            s_out0 * d->weights[0][(size_t)o * d->d_in + m->raw_w + 2 * m->m + j];
  }
  // tcgen05 pack for the default shapes (see TcNetDev in fvsrn_tc.cuh)
  if ((m->hid_pad == 32 || m->hid_pad == 64) && L == tc_layers(m->hid_pad) && m->f_pad == 16 &&
      m->R > 0 && m->act == FVSRN_ACT_SNAKE_ALT && m->fourier_mode == FVSRN_FOURIER_NERF &&
      m->fd_in == 3 && m->raw_w == 3 && m->m == (m->hid_pad - 4) / 2) {
    const int H = m->hid_pad;
    std::vector<__half> wt;
    std::vector<float> bt;
    for (int l = 0; l < L; ++l) {
      const int Nt = (l == L - 1) ? 16 : H, Kw = Ks[l];
      // bias in the MMA (tc_bias_mma): layers >= 1 get an extra k16 tile carrying the bias as fp16
      // hi + lo (column Kw: hi, Kw + 1: lo; the A side holds 1, 1 there)
      const bool bias_mma = tc_bias_mma(H);
      const int K = (bias_mma && l > 0) ? Kw + 16 : Kw;
      std::vector<__half> tile((size_t)Nt * K, __float2half_rn(0.f));
      auto at = [&](int n, int k) -> __half& {
        return tile[(size_t)(n / 8) * (K / 8) * 64 + (k / 8) * 64 + (n % 8) * 8 + (k % 8)];
      };
      for (int n = 0; n < Nt && n < N[l]; ++n) {
        for (int k = 0; k < Kw; ++k) at(n, k) = __float2half_rn(ws[l][(size_t)n * Kw + k]);
        if (bias_mma && l > 0) {
          const __half hi = __float2half_rn(bs[l][n]);
          at(n, Kw) = hi;
          at(n, Kw + 1) = __float2half_rn(bs[l][n] - __half2float(hi));
        }
      }
      wt.insert(wt.end(), tile.begin(), tile.end());
      for (int n = 0; n < Nt; ++n) bt.push_back(n < N[l] ? bs[l][n] : 0.f);
    }
    // the last layer's first weight row in f32 (TcShape::kWLast: the density head's last
    // layer evaluated on the FMA pipe)
    for (int k = 0; k < H; ++k) bt.push_back(k < Ks[L - 1] ? ws[L - 1][(size_t)k] : 0.f);
    int rc = upload(wt.data(), wt.size() * sizeof(__half), (void**)&m->d_wtc);
    if (rc) return rc;
    rc = upload(bt.data(), bt.size() * sizeof(float), (void**)&m->d_btc);
    if (rc) return rc;
    m->tc_ok = true;
  }
  Pack pks, pkx;
  build_pack(ws, Ks, N, bs, pks);
  pks.kt0 = m->k0 / 16;
  build_pack(wx, Kx, N, bs, pkx);
  pkx.kt0 = Kx[0] / 16;
  m->k0x = Kx[0];
  int rc = make_devpack(pks, L, m->act, m->head, d_out, m->ps);
  if (rc) return rc;
  rc = make_devpack(pkx, L, m->act, m->head, d_out, m->px);
  if (rc) return rc;
  if ((rc = probe_texture_sampler(m))) return rc;
  *out = guard.release();
  return FVSRN_OK;
}

int32_t fvsrn_model_destroy(fvsrn_model_t m) {
  if (!m) return FVSRN_OK;
  delete m;
  return FVSRN_OK;
}

int32_t fvsrn_model_info(fvsrn_model_t m, int32_t* k0_pad, int32_t* hidden_pad, int32_t* smem) {
  if (!m) return fail(FVSRN_EINVAL, "null model");
  if (k0_pad) *k0_pad = m->k0;
  if (hidden_pad) *hidden_pad = m->hid_pad;
  if (smem) *smem = (int32_t)stage_smem_bytes(m->ps.net, true, m->k0);
  return FVSRN_OK;
}

static int render_impl(fvsrn_model_t m, const fvsrn_tf* tf, const fvsrn_camera* c,
                       const fvsrn_settings* st, double t, const fvsrn_shard* shard, float* d_out,
                       unsigned long long* d_eval_count, unsigned long long* d_nonfinite,
                       cudaStream_t stream);

int32_t fvsrn_render_device(fvsrn_model_t m, const fvsrn_tf* tf, const fvsrn_camera* c,
                            const fvsrn_settings* st, double t, const fvsrn_shard* shard,
                            float* d_out, unsigned long long* d_eval_count, void* stream) {
  return render_impl(m, tf, c, st, t, shard, d_out, d_eval_count, nullptr, (cudaStream_t)stream);
}

}  // extern "C"

static int render_impl(fvsrn_model_t m, const fvsrn_tf* tf, const fvsrn_camera* c,
                       const fvsrn_settings* st, double t, const fvsrn_shard* shard, float* d_out,
                       unsigned long long* d_eval_count, unsigned long long* d_nonfinite,
                       cudaStream_t stream) {
  if (!m || !c || !d_out) return fail(FVSRN_EINVAL, "null argument");
  int rc = check_settings(st);
  if (rc) return rc;
  if ((rc = check_source(m, tf, t))) return rc;
  if (c->width < 1 || c->height < 1) return fail(FVSRN_EINVAL, "image dimensions must be positive");
  CUDA_TRY(cudaSetDevice(m->device));
  cudaStream_t s = (cudaStream_t)stream;
  FrameScratch fs;
  if ((rc = frame_setup(m, t, tf, s, fs))) return rc;
  CamDev cam = cam_for(c);
  if (c->has_basis) {
    for (int a = 0; a < 3; ++a) { cam.fwd[a] = c->b_forward[a]; cam.right[a] = c->b_right[a]; cam.up[a] = c->b_up[a]; }
    cam.half_w = c->half_w;
    cam.half_h = c->half_h;
  }
  ShardDev sh{};
  sh.rank = shard ? shard->rank : 0;
  sh.world = shard ? shard->world : 1;
  sh.compact = shard ? shard->compact : 0;
  if (sh.world < 1 || sh.rank < 0 || sh.rank >= sh.world) return fail(FVSRN_EINVAL, "bad shard");
  sh.tiles_x = (c->width + kTile - 1) / kTile;
  sh.n_tiles = sh.tiles_x * ((c->height + kTile - 1) / kTile);
  const long long local_tiles = (sh.n_tiles - sh.rank + sh.world - 1) / sh.world;
  long long n_slots = std::max(0ll, local_tiles) * 64;
  if (sh.compact) {  // compact buffers are sized for max_local tiles; zero the tail
    const long long max_local = (sh.n_tiles + sh.world - 1) / sh.world;
    if (max_local > local_tiles)
      CUDA_TRY(cudaMemsetAsync(d_out + local_tiles * 64 * 4, 0, (max_local - local_tiles) * 64 * 16, s));
  }
  NetDev net = m->ps.net;
  FeatDev fd = feat_for(m, fs);
  MarchDev md = march_for(st);
  // per-slot ray records (f64 setup once per ray, outside the march loop) and the LPT
  // schedule: longest tiles first (removes the persistent kernel's long-ray tail)
  RayRecs rr{};
  void* recs = nullptr;
  if ((rc = alloc_recs(m, n_slots, s, rr, recs))) return rc;
  void* lpt = nullptr;
  // LPT pays off once a frame has many tiles per SM (1024^2: 3.32 -> 3.19 ms); at 256^2 the
  // reduced-occupancy launch is faster without it (0.32 -> 0.31 ms)
  const bool use_lpt = local_tiles >= 16 * m->num_sms && g_lpt_enabled;
  unsigned* cost = nullptr;
  unsigned* order = nullptr;
  if (use_lpt) {
    const int nl = (int)local_tiles;
    CUDA_TRY(cudaMallocAsync(&lpt, 8 * (size_t)nl + 256, s));
    cost = (unsigned*)lpt;
    order = cost + (size_t)nl;
    CUDA_TRY(cudaMemsetAsync(cost, 0, sizeof(unsigned) * nl, s));
  }
  CUDA_TRY(launch_ray_setup(cam, md, sh, nullptr, nullptr, n_slots, rr, d_out, cost, nullptr, g_defer_miss, s));
  count_launch();
  if (use_lpt) {
    // Into a mapped host framebuffer, pure LPT puts every cheap tile at the end of the
    // frame and their pixel stores then drain over PCIe after the march: keep only
    // ~2.2 x (SMs x 20 warps) of the lightest tiles as the end-of-frame fillers and
    // interleave the rest heaviest / lightest (cfg 2 e2e 3.39 -> 3.28 ms at equal march
    // time; cfg 5 e2e 51.2 -> 50.3 ms).  Device-memory frames keep pure LPT.
    // FVSRN_LPT_FILL=<x> overrides the multiplier (0 = pure LPT).
    static const double fill_env = [] {
      const char* e = std::getenv("FVSRN_LPT_FILL");
      return e ? std::atof(e) : -1.0;
    }();
    const double fill_mult = fill_env >= 0.0 ? fill_env : (g_out_mapped ? 2.2 : 0.0);
    const int fillers = fill_mult > 0 ? (int)std::min<double>((double)local_tiles, fill_mult * m->num_sms * 20) : 0;
    CUDA_TRY(launch_tile_sort((int)local_tiles, cost, order, fillers, s));
    count_launch();
    sh.order = order;
  }
  const TFDev* tfp = fs.tf;
  const float* b0 = fs.b0;
  int explicit_rays = 0;
  unsigned long long* queue = fs.counters;
  unsigned long long* evc = d_eval_count ? d_eval_count : fs.counters + 1;
  unsigned long long* nfc = d_nonfinite ? d_nonfinite : fs.counters + 2;
  if ((rc = launch_dvr(m, net, fd, tfp, b0, md, cam, sh, explicit_rays, rr, n_slots, d_out, queue, evc, nfc, s)))
    return rc;
  CUDA_TRY(cudaFreeAsync(fs.buf, s));
  CUDA_TRY(cudaFreeAsync(recs, s));
  if (lpt) CUDA_TRY(cudaFreeAsync(lpt, s));
  return FVSRN_OK;
}

extern "C" {

int32_t fvsrn_tiles_to_frame_device(const float* d_gathered, int32_t width, int32_t height,
                                    int32_t world, float* d_frame, void* stream) {
  if (!d_gathered || !d_frame || world < 1) return fail(FVSRN_EINVAL, "bad argument");
  CUDA_TRY(launch_tiles_to_frame(d_gathered, width, height, world, d_frame, (cudaStream_t)stream));
  count_launch();
  return FVSRN_OK;
}

}  // extern "C"

namespace {

// Host-pointer entry points run on the calling thread's per-thread default stream
// (reentrant across host threads, no per-call stream creation).
struct StreamGuard {
  cudaStream_t s = cudaStreamPerThread;
};

}  // namespace

extern "C" {

int32_t fvsrn_render(fvsrn_model_t m, const fvsrn_tf* tf, const fvsrn_camera* c,
                     const fvsrn_settings* st, double t, float* out, uint64_t* eval_count) {
  if (!m || !c || !out) return fail(FVSRN_EINVAL, "null argument");
  if (c->width < 1 || c->height < 1) return fail(FVSRN_EINVAL, "image dimensions must be positive");
  CUDA_TRY(cudaSetDevice(m->device));
  StreamGuard sg;
  const size_t bytes = (size_t)c->width * c->height * 16;
  // A mapped page-locked framebuffer (fvsrn_host_alloc) is written by the kernels
  // directly over PCIe: each pixel is stored once when its ray ends, so the transfer
  // overlaps the march instead of following it.  Otherwise render to HBM and copy.
  HostPhases ph;
  float* mapped = mapped_device_ptr(out);
  ph.mark("ptrattr");
  float* d_out = nullptr;
  unsigned long long* d_cnt = nullptr;
  void* dbuf = nullptr;
  CUDA_TRY(cudaMallocAsync(&dbuf, (mapped ? 0 : bytes) + 16, sg.s));
  d_out = mapped ? mapped : (float*)dbuf;
  d_cnt = (unsigned long long*)((char*)dbuf + (mapped ? 0 : bytes));
  CUDA_TRY(cudaMemsetAsync(d_cnt, 0, 16, sg.s));
  ph.mark("alloc");
  g_out_mapped = mapped != nullptr;
  int rc = render_impl(m, tf, c, st, t, nullptr, d_out, d_cnt, d_cnt + 1, sg.s);
  g_out_mapped = false;
  if (rc) { cudaFreeAsync(dbuf, sg.s); cudaStreamSynchronize(sg.s); return rc; }
  ph.mark("enqueue");
  if (g_debug_timing) {   // host time at which the march kernel has finished
    cudaEvent_t done;
    cudaEventCreate(&done);
    cudaEventRecord(done, sg.s);
    cudaEventSynchronize(done);
    cudaEventDestroy(done);
    ph.mark("kernels");
  }
  unsigned long long stack_cnt[2] = {0, 0};
  unsigned long long* cnt = pinned_counters();
  if (!cnt) cnt = stack_cnt;
  if (!mapped) CUDA_TRY(cudaMemcpyAsync(out, d_out, bytes, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaMemcpyAsync(cnt, d_cnt, 16, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaFreeAsync(dbuf, sg.s));
  ph.mark("tail");
  CUDA_TRY(cudaStreamSynchronize(sg.s));
  ph.mark("sync");
  if (eval_count) *eval_count = cnt[0];
  if (cnt[1]) return fail(FVSRN_EINVAL, "image contains non-finite values");
  return FVSRN_OK;
}

int32_t fvsrn_render_rgba8(fvsrn_model_t m, const fvsrn_tf* tf, const fvsrn_camera* c,
                           const fvsrn_settings* st, double t, uint8_t* out, uint64_t* eval_count) {
  if (!m || !c || !out) return fail(FVSRN_EINVAL, "null argument");
  if (c->width < 1 || c->height < 1) return fail(FVSRN_EINVAL, "image dimensions must be positive");
  CUDA_TRY(cudaSetDevice(m->device));
  StreamGuard sg;
  const long long n_px = (long long)c->width * c->height;
  const size_t fb_bytes = (size_t)n_px * 16, u8_bytes = (size_t)n_px * 4;
  unsigned char* mapped = (unsigned char*)mapped_device_ptr(out);
  char* buf = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&buf, fb_bytes + (mapped ? 0 : u8_bytes) + 16, sg.s));
  float* d_fb = (float*)buf;
  unsigned char* d_u8 = mapped ? mapped : (unsigned char*)(buf + fb_bytes);
  unsigned long long* d_cnt = (unsigned long long*)(buf + fb_bytes + (mapped ? 0 : u8_bytes));
  CUDA_TRY(cudaMemsetAsync(d_cnt, 0, 16, sg.s));
  int rc = render_impl(m, tf, c, st, t, nullptr, d_fb, d_cnt, d_cnt + 1, sg.s);
  if (rc) { cudaFreeAsync(buf, sg.s); cudaStreamSynchronize(sg.s); return rc; }
  CUDA_TRY(launch_rgba8(d_fb, n_px, d_u8, sg.s));
  count_launch();
  unsigned long long cnt[2] = {0, 0};
  if (!mapped) CUDA_TRY(cudaMemcpyAsync(out, d_u8, u8_bytes, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaMemcpyAsync(cnt, d_cnt, 16, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaFreeAsync(buf, sg.s));
  CUDA_TRY(cudaStreamSynchronize(sg.s));
  if (eval_count) *eval_count = cnt[0];
  if (cnt[1]) return fail(FVSRN_EINVAL, "image contains non-finite values");
  return FVSRN_OK;
}

int32_t fvsrn_render_rays(fvsrn_model_t m, const fvsrn_tf* tf, const double* origins,
                          const double* dirs, int64_t n, const fvsrn_settings* st, double t,
                          float* out_px, uint64_t* eval_count) {
  if (!m || (n > 0 && (!origins || !dirs || !out_px))) return fail(FVSRN_EINVAL, "null argument");
  int rc = check_settings(st);
  if (rc) return rc;
  if ((rc = check_source(m, tf, t))) return rc;
  if (eval_count) *eval_count = 0;
  if (n == 0) return FVSRN_OK;
  CUDA_TRY(cudaSetDevice(m->device));
  StreamGuard sg;
  const size_t rb = (size_t)n * 3 * sizeof(double), ob = (size_t)n * 16;
  char* buf = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&buf, 2 * rb + ob, sg.s));
  double* d_o = (double*)buf;
  double* d_d = (double*)(buf + rb);
  float* d_out = (float*)(buf + 2 * rb);
  CUDA_TRY(cudaMemcpyAsync(d_o, origins, rb, cudaMemcpyHostToDevice, sg.s));
  CUDA_TRY(cudaMemcpyAsync(d_d, dirs, rb, cudaMemcpyHostToDevice, sg.s));
  FrameScratch fs;
  if ((rc = frame_setup(m, t, tf, sg.s, fs))) return rc;
  NetDev net = m->ps.net;
  FeatDev fd = feat_for(m, fs);
  MarchDev md = march_for(st);
  CamDev cam{};
  ShardDev sh{};
  sh.world = 1;
  const TFDev* tfp = fs.tf;
  const float* b0 = fs.b0;
  long long n_slots = n;
  RayRecs rr{};
  void* recs = nullptr;
  if ((rc = alloc_recs(m, n_slots, sg.s, rr, recs))) return rc;
  CUDA_TRY(launch_ray_setup(cam, md, sh, d_o, d_d, n_slots, rr, d_out, nullptr, nullptr, g_defer_miss, sg.s));
  count_launch();
  int explicit_rays = 1;
  unsigned long long* queue = fs.counters;
  unsigned long long* evc = fs.counters + 1;
  unsigned long long* nfc = nullptr;
  if ((rc = launch_dvr(m, net, fd, tfp, b0, md, cam, sh, explicit_rays, rr, n_slots, d_out, queue, evc, nfc, sg.s)))
    return rc;
  CUDA_TRY(cudaFreeAsync(recs, sg.s));
  unsigned long long cnt = 0;
  CUDA_TRY(cudaMemcpyAsync(out_px, d_out, ob, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaMemcpyAsync(&cnt, evc, 8, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaFreeAsync(fs.buf, sg.s));
  CUDA_TRY(cudaFreeAsync(buf, sg.s));
  CUDA_TRY(cudaStreamSynchronize(sg.s));
  if (eval_count) *eval_count = cnt;
  return FVSRN_OK;
}

static int eval_common(fvsrn_model_t m, const double* p, const double* dd, int64_t n, double t,
                       float* out, int want_head) {
  if (!m || (n > 0 && (!p || !out))) return fail(FVSRN_EINVAL, "null argument");
  if (m->head != want_head)
    return fail(FVSRN_EINVAL, want_head == FVSRN_HEAD_DENSITY ? "eval_density requires a density-head model"
                                                              : "eval_color requires a color-head model");
  if (!m->temporal && !std::isnan(t)) return fail(FVSRN_EINVAL, "timestep supplied to a non-temporal model");
  if (m->temporal && std::isnan(t)) return fail(FVSRN_EINVAL, "temporal model requires timesteps");
  if (m->dir_mode != FVSRN_DIR_POS && !dd) return fail(FVSRN_EINVAL, "direction mode requires view directions");
  if (n == 0) return FVSRN_OK;
  CUDA_TRY(cudaSetDevice(m->device));
  StreamGuard sg;
  const int oc = want_head == FVSRN_HEAD_DENSITY ? 1 : 4;
  const size_t pb = (size_t)n * 3 * sizeof(double), ob = (size_t)n * oc * sizeof(float);
  char* buf = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&buf, 2 * pb + ob, sg.s));
  double* d_p = (double*)buf;
  double* d_d = dd ? (double*)(buf + pb) : nullptr;
  float* d_out = (float*)(buf + 2 * pb);
  CUDA_TRY(cudaMemcpyAsync(d_p, p, pb, cudaMemcpyHostToDevice, sg.s));
  if (dd) CUDA_TRY(cudaMemcpyAsync(d_d, dd, pb, cudaMemcpyHostToDevice, sg.s));
  FrameScratch fs;
  int rc = frame_setup(m, t, nullptr, sg.s, fs);
  if (rc) return rc;
  NetDev net = m->ps.net;
  FeatDev fd = feat_for(m, fs);
  const float* b0 = fs.b0;
  int mode = 1, res = 0;
  double step = 0;
  long long begin = 0, count = n;
  const double* pp = d_p;
  const double* pd = d_d;
  unsigned long long* bad = nullptr;
  const float* coords = nullptr;
  void* args[] = {&net, &fd, &b0, &mode, &res, &step, &begin, &count, &pp, &pd, &d_out, &bad, &coords};
  const size_t smem = stage_smem_bytes(net, false, m->k0);
  if ((rc = launch(m, KernelKind::kSample, smem, args, sg.s, n / 32 + 1))) return rc;
  CUDA_TRY(cudaMemcpyAsync(out, d_out, ob, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaFreeAsync(fs.buf, sg.s));
  CUDA_TRY(cudaFreeAsync(buf, sg.s));
  CUDA_TRY(cudaStreamSynchronize(sg.s));
  return FVSRN_OK;
}

int32_t fvsrn_eval_density(fvsrn_model_t m, const double* p, int64_t n, double t, float* out) {
  return eval_common(m, p, nullptr, n, t, out, FVSRN_HEAD_DENSITY);
}

int32_t fvsrn_eval_color(fvsrn_model_t m, const double* p, const double* d, int64_t n, double t,
                         float* out4) {
  return eval_common(m, p, d, n, t, out4, FVSRN_HEAD_COLOR);
}

static int decode_impl(fvsrn_model_t m, int32_t res, double t, int64_t lattice_begin,
                       int64_t lattice_count, float* d_out, unsigned long long* d_bad, cudaStream_t s,
                       int chunks = 1, float* h_out = nullptr, cudaStream_t copy_s = nullptr);

int32_t fvsrn_decode_density_device(fvsrn_model_t m, int32_t res, double t, int64_t lattice_begin,
                                    int64_t lattice_count, float* d_out, void* stream) {
  return decode_impl(m, res, t, lattice_begin, lattice_count, d_out, nullptr, (cudaStream_t)stream);
}

}  // extern "C"

// FVSRN_DECODE_CHUNKS=<k>: a page-locked host volume is filled by k decode launches into
// HBM, each chunk's device->host copy (copy engine, second stream) overlapping the next
// chunk's decode; 0 = the decode kernel stores straight into the mapped buffer instead
const int g_decode_chunks = [] {
  const char* e = std::getenv("FVSRN_DECODE_CHUNKS");
  return e ? std::atoi(e) : 16;   // 256^3 e2e: mapped stores 1.49-1.57 ms, 4: 1.42, 8: 1.35, 16: 1.34
}();

static int decode_impl(fvsrn_model_t m, int32_t res, double t, int64_t lattice_begin,
                       int64_t lattice_count, float* d_out, unsigned long long* d_bad, cudaStream_t s,
                       int chunks, float* h_out, cudaStream_t copy_s) {
  if (!m || !d_out) return fail(FVSRN_EINVAL, "null argument");
  if (m->head != FVSRN_HEAD_DENSITY) return fail(FVSRN_EINVAL, "decode_volume requires a density-head model");
  if (res < 2) return fail(FVSRN_EINVAL, "resolution must be >= 2");
  if (!m->temporal && !std::isnan(t)) return fail(FVSRN_EINVAL, "timestep supplied to a non-temporal model");
  if (m->temporal && std::isnan(t)) return fail(FVSRN_EINVAL, "temporal model requires timesteps");
  CUDA_TRY(cudaSetDevice(m->device));
  FrameScratch fs;
  int rc = frame_setup(m, t, nullptr, s, fs);
  if (rc) return rc;
  NetDev net = m->ps.net;
  FeatDev fd = feat_for(m, fs);
  const float* b0 = fs.b0;
  int mode = 0;
  double step = 1.0 / (double)(res - 1);
  long long begin = lattice_begin, count = lattice_count;
  const double* pp = nullptr;
  const double* pd = nullptr;
  // lattice coordinates as numpy's linspace(0, 1, res) then float32 (model.py:385-398):
  // i * step for i < res - 1, the last exactly 1.0
  std::vector<float> hc((size_t)res);
  for (int i = 0; i < res; ++i) hc[i] = i == res - 1 ? 1.f : (float)((double)i * step);
  float* coords = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&coords, hc.size() * sizeof(float), s));
  CUDA_TRY(cudaMemcpyAsync(coords, hc.data(), hc.size() * sizeof(float), cudaMemcpyHostToDevice, s));
  const size_t smem = stage_smem_bytes(net, false, m->k0);
  // static fp16 texture grid on the default shapes: the branch-free feature path
  const bool s_tex = fd.tex_on && !fd.tex_u8 && fd.tex_w == 0.f;
  const bool s_ldg = !fd.tex_on && fd.grid != nullptr && fd.f_pad == 16;
  const bool s_static = FVSRN_TEX_SPECIAL && fast_path(m, KernelKind::kSample) && (s_tex || s_ldg);
  // the tcgen05 decode wherever the march uses tcgen05 (FVSRN_DECODE_TC=0: mma.sync)
  static const bool decode_tc = [] {
    const char* e = std::getenv("FVSRN_DECODE_TC");
    return !(e && e[0] == '0');
  }();
  const bool tcd = s_static && decode_tc && use_tc(m);
  const KernelKind sk = tcd ? KernelKind::kSampleTC : s_static ? KernelKind::kSampleTex : KernelKind::kSample;
  const int sfm = s_tex ? 1 : 2;
  TcNetDev tn{m->d_wtc, m->d_btc, m->head};
  const size_t tsmem = tcd ? tc_smem_bytes(m->hid_pad) : 0;
  if (chunks <= 1 || !h_out) {
    void* args[] = {&net, &fd, &b0, &mode, &res, &step, &begin, &count, &pp, &pd, &d_out, &d_bad, &coords};
    void* targs[] = {&tn, &fd, &b0, &res, &begin, &count, &coords, &d_out, &d_bad};
    if ((rc = launch(m, sk, tcd ? tsmem : smem, tcd ? targs : args, s, count / 32 + 1, sfm))) return rc;
  } else {
    // chunk c: decode [c0, c0 + n) into d_out + c0 on s, then copy it to h_out on copy_s
    const long long per = ((lattice_count + chunks - 1) / chunks + 31) / 32 * 32;
    for (long long c0 = 0; c0 < lattice_count; c0 += per) {
      long long cb = lattice_begin + c0, cn = std::min(per, lattice_count - c0);
      float* dst = d_out + c0;
      void* args[] = {&net, &fd, &b0, &mode, &res, &step, &cb, &cn, &pp, &pd, &dst, &d_bad, &coords};
      void* targs[] = {&tn, &fd, &b0, &res, &cb, &cn, &coords, &dst, &d_bad};
      if ((rc = launch(m, sk, tcd ? tsmem : smem, tcd ? targs : args, s, cn / 32 + 1, sfm))) return rc;
      cudaEvent_t done;
      CUDA_TRY(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(done, s));
      CUDA_TRY(cudaStreamWaitEvent(copy_s, done, 0));
      CUDA_TRY(cudaEventDestroy(done));
      CUDA_TRY(cudaMemcpyAsync(h_out + c0, dst, cn * sizeof(float), cudaMemcpyDeviceToHost, copy_s));
    }
    cudaEvent_t copied;
    CUDA_TRY(cudaEventCreateWithFlags(&copied, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(copied, copy_s));
    CUDA_TRY(cudaStreamWaitEvent(s, copied, 0));   // the caller's stream sees the copies
    CUDA_TRY(cudaEventDestroy(copied));
  }
  CUDA_TRY(cudaFreeAsync(coords, s));
  CUDA_TRY(cudaFreeAsync(fs.buf, s));
  return FVSRN_OK;
}

extern "C" {

}  // extern "C"

// Lattice slab [begin, begin + count) of the res^3 decode into host memory `out` (the
// slab's first element), on the calling thread's per-thread stream of m's device.
static int decode_host_slab(fvsrn_model_t m, int32_t res, double t, long long begin, long long count,
                            float* out) {
  CUDA_TRY(cudaSetDevice(m->device));
  StreamGuard sg;
  // page-locked output: either chunked decode into HBM with the copies overlapped on a
  // second stream (default), or the decode kernel storing straight into the mapped buffer
  float* mapped = mapped_device_ptr(out);
  const bool pipelined = mapped && g_decode_chunks > 1 && count >= (1ll << 20);
  if (pipelined) mapped = nullptr;
  char* buf = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&buf, (mapped ? 0 : count * sizeof(float)) + 16, sg.s));
  float* d_out = mapped ? mapped : (float*)buf;
  unsigned long long* d_bad = (unsigned long long*)(buf + (mapped ? 0 : count * sizeof(float)));
  CUDA_TRY(cudaMemsetAsync(d_bad, 0, 8, sg.s));
  thread_local std::map<int, cudaStream_t> copy_streams;   // one copy stream per (thread, device)
  cudaStream_t copy_s = nullptr;
  if (pipelined) {
    cudaStream_t& cs = copy_streams[m->device];
    if (!cs) CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    copy_s = cs;
  }
  int rc = pipelined ? decode_impl(m, res, t, begin, count, d_out, d_bad, sg.s, g_decode_chunks, out, copy_s)
                     : decode_impl(m, res, t, begin, count, d_out, d_bad, sg.s);
  if (rc) {
    // chunks already queued on copy_s may still read buf and write out: drain them
    // before the buffer goes back to the pool and before the caller regains `out`
    if (copy_s) cudaStreamSynchronize(copy_s);
    cudaFreeAsync(buf, sg.s);
    cudaStreamSynchronize(sg.s);
    return rc;
  }
  unsigned long long* bad = pinned_counters();
  unsigned long long stack_bad = 0;
  if (!bad) bad = &stack_bad;
  if (!mapped && !pipelined) CUDA_TRY(cudaMemcpyAsync(out, d_out, count * sizeof(float), cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaMemcpyAsync(bad, d_bad, 8, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaFreeAsync(buf, sg.s));
  CUDA_TRY(cudaStreamSynchronize(sg.s));
  if (*bad) return fail(FVSRN_EINVAL, "volume contains non-finite values");
  return FVSRN_OK;
}

// ---------------------------------------------------------------- several GPUs, one process
namespace {

// One persistent host thread per device for the multi-device entries: every device's
// enqueue (ray setup, tile sort, march, copies) and its stream synchronisation run
// concurrently, each on the worker's own per-thread default stream.  Workers live for
// the process (never joined at exit, when the CUDA runtime may already be gone).
class DeviceWorker {
 public:
  explicit DeviceWorker(int dev) : dev_(dev), th_([this] { loop(); }) { th_.detach(); }
  using Result = std::pair<int, std::string>;
  std::future<Result> submit(std::function<int()> fn) {
    auto task = std::make_shared<std::packaged_task<Result()>>([fn, this] {
      const cudaError_t e = cudaSetDevice(dev_);
      const int rc = e != cudaSuccess ? fail(FVSRN_ECUDA, cudaGetErrorString(e)) : fn();
      return Result(rc, rc ? g_err : std::string());
    });
    auto fut = task->get_future();
    {
      std::lock_guard<std::mutex> l(mu_);
      q_.emplace_back([task] { (*task)(); });
    }
    cv_.notify_one();
    return fut;
  }

 private:
  void loop() {
    for (;;) {
      std::function<void()> f;
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return !q_.empty(); });
        f = std::move(q_.front());
        q_.pop_front();
      }
      f();
    }
  }
  int dev_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
  std::thread th_;
};

std::mutex g_workers_mu;
DeviceWorker* worker_for(int dev) {
  static auto* workers = new std::map<int, DeviceWorker*>();
  auto it = workers->find(dev);
  if (it == workers->end()) it = workers->emplace(dev, new DeviceWorker(dev)).first;
  return it->second;
}

// Runs fns[i] on the worker of replica i's device; all submitted under one lock so every
// worker queue sees concurrent calls in the same order.  Returns the first failure.
int run_on_devices(const fvsrn_model_t* reps, int n, const std::vector<std::function<int()>>& fns) {
  std::vector<std::future<DeviceWorker::Result>> futs;
  {
    std::lock_guard<std::mutex> l(g_workers_mu);
    for (int i = 0; i < n; ++i) futs.push_back(worker_for(reps[i]->device)->submit(fns[i]));
  }
  int rc = FVSRN_OK;
  std::string msg;
  for (auto& f : futs) {
    auto r = f.get();
    if (r.first && !rc) { rc = r.first; msg = r.second; }
  }
  return rc ? fail(rc, msg) : FVSRN_OK;
}

int check_replicas(const fvsrn_model_t* reps, int n) {
  if (!reps || n < 1) return fail(FVSRN_EINVAL, "need at least one model replica");
  for (int i = 0; i < n; ++i) {
    if (!reps[i]) return fail(FVSRN_EINVAL, "null model replica");
    const fvsrn_model& a = *reps[i];
    const fvsrn_model& b = *reps[0];
    if (a.head != b.head || a.temporal != b.temporal || a.layers != b.layers || a.hidden != b.hidden ||
        a.d_in != b.d_in || a.d_out != b.d_out || a.act != b.act || a.R != b.R || a.F != b.F ||
        a.k0 != b.k0)
      return fail(FVSRN_EINVAL, "model replicas differ in shape");
  }
  return FVSRN_OK;
}

// peer access from `dev` to `home` (once per pair); false when the pair has no P2P path
bool enable_peer(int dev, int home) {
  if (dev == home) return true;
  static std::mutex mu;
  static std::map<std::pair<int, int>, bool> state;
  std::lock_guard<std::mutex> l(mu);
  auto key = std::make_pair(dev, home);
  auto it = state.find(key);
  if (it != state.end()) return it->second;
  int can = 0;
  bool ok = cudaDeviceCanAccessPeer(&can, dev, home) == cudaSuccess && can;
  if (ok) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
    const cudaError_t e = cudaDeviceEnablePeerAccess(home, 0);
    ok = e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled;
    cudaSetDevice(prev);
  }
  cudaGetLastError();
  state[key] = ok;
  return ok;
}

// Framebuffers on a home device that peers store into (cudaMalloc memory: P2P-mappable,
// unlike the stream-ordered pool's), recycled across calls.
struct FrameCache {
  std::mutex mu;
  std::map<std::pair<int, size_t>, std::vector<void*>> free;
  void* take(int dev, size_t bytes) {
    {
      std::lock_guard<std::mutex> l(mu);
      auto& v = free[{dev, bytes}];
      if (!v.empty()) { void* p = v.back(); v.pop_back(); return p; }
    }
    void* p = nullptr;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
    if (cudaMalloc(&p, bytes) != cudaSuccess) { cudaGetLastError(); p = nullptr; }
    cudaSetDevice(prev);
    return p;
  }
  void give(int dev, size_t bytes, void* p) {
    std::lock_guard<std::mutex> l(mu);
    free[{dev, bytes}].push_back(p);
  }
};
FrameCache& frame_cache() {
  static auto* c = new FrameCache();
  return *c;
}

// one replica's round-robin tiles into `d_frame` (full-frame layout), synchronised;
// adds its evaluated-sample count to *evals
int render_share(fvsrn_model_t m, const fvsrn_tf* tf, const fvsrn_camera* c, const fvsrn_settings* st,
                 double t, int rank, int world, float* d_frame, bool frame_mapped,
                 std::atomic<unsigned long long>* evals) {
  StreamGuard sg;
  unsigned long long* d_cnt = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&d_cnt, 16, sg.s));
  CUDA_TRY(cudaMemsetAsync(d_cnt, 0, 16, sg.s));
  fvsrn_shard sh{rank, world, 0};
  g_out_mapped = frame_mapped;
  int rc = render_impl(m, tf, c, st, t, &sh, d_frame, d_cnt, d_cnt + 1, sg.s);
  g_out_mapped = false;
  if (rc) { cudaFreeAsync(d_cnt, sg.s); cudaStreamSynchronize(sg.s); return rc; }
  unsigned long long stack_cnt[2] = {0, 0};
  unsigned long long* cnt = pinned_counters();
  if (!cnt) cnt = stack_cnt;
  CUDA_TRY(cudaMemcpyAsync(cnt, d_cnt, 16, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaFreeAsync(d_cnt, sg.s));
  CUDA_TRY(cudaStreamSynchronize(sg.s));
  evals->fetch_add(cnt[0]);
  if (cnt[1]) return fail(FVSRN_EINVAL, "image contains non-finite values");
  return FVSRN_OK;
}

}  // namespace

extern "C" {

int32_t fvsrn_decode_density(fvsrn_model_t m, int32_t res, double t, float* out) {
  if (!m || !out) return fail(FVSRN_EINVAL, "null argument");
  if (res < 2) return fail(FVSRN_EINVAL, "resolution must be >= 2");
  return decode_host_slab(m, res, t, 0, (long long)res * res * res, out);
}

int32_t fvsrn_decode_density_multi(const fvsrn_model_t* reps, int32_t n, int32_t res, double t,
                                   float* out) {
  int rc = check_replicas(reps, n);
  if (rc) return rc;
  if (!out) return fail(FVSRN_EINVAL, "null argument");
  if (res < 2) return fail(FVSRN_EINVAL, "resolution must be >= 2");
  if (n == 1) return fvsrn_decode_density(reps[0], res, t, out);
  // contiguous lattice slabs (multiples of 32 entries: whole warps) per replica
  const long long total = (long long)res * res * res;
  const long long per = ((total + n - 1) / n + 31) / 32 * 32;
  std::vector<std::function<int()>> fns;
  for (int i = 0; i < n; ++i) {
    const long long b = std::min(total, i * per), cnt = std::min(per, total - b);
    fvsrn_model_t m = reps[i];
    fns.push_back([=] { return cnt > 0 ? decode_host_slab(m, res, t, b, cnt, out + b) : (int)FVSRN_OK; });
  }
  return run_on_devices(reps, n, fns);
}

int32_t fvsrn_render_multi(const fvsrn_model_t* reps, int32_t n, const fvsrn_tf* tf,
                           const fvsrn_camera* c, const fvsrn_settings* st, double t, float* out,
                           uint64_t* eval_count) {
  int rc = check_replicas(reps, n);
  if (rc) return rc;
  if (!c || !out) return fail(FVSRN_EINVAL, "null argument");
  if (c->width < 1 || c->height < 1) return fail(FVSRN_EINVAL, "image dimensions must be positive");
  if (n == 1) return fvsrn_render(reps[0], tf, c, st, t, out, eval_count);
  const size_t bytes = (size_t)c->width * c->height * 16;
  std::atomic<unsigned long long> evals{0};
  // (1) page-locked out (fvsrn_host_alloc: portable + mapped): every GPU stores its own
  // tiles' pixels straight into the host frame over its own link, overlapped with its march
  if (mapped_device_ptr(out)) {
    std::vector<std::function<int()>> fns;
    for (int i = 0; i < n; ++i) {
      fvsrn_model_t m = reps[i];
      fns.push_back([=, &evals] {
        float* d = mapped_device_ptr(out);
        if (!d) return fail(FVSRN_ECUDA, "framebuffer is not mapped on this device");
        return render_share(m, tf, c, st, t, i, n, d, true, &evals);
      });
    }
    if ((rc = run_on_devices(reps, n, fns))) return rc;
    if (eval_count) *eval_count = evals.load();
    return FVSRN_OK;
  }
  // (2) pageable out: the replicas store into one framebuffer on replicas[0]'s device over
  // NVLink P2P, then one device->host copy.  Without a P2P path: a page-locked staging frame.
  const int home = reps[0]->device;
  bool p2p = true;
  for (int i = 1; i < n; ++i) p2p = p2p && enable_peer(reps[i]->device, home);
  float* frame = nullptr;
  void* staging = nullptr;
  if (p2p) {
    frame = (float*)frame_cache().take(home, bytes);
    if (!frame) return fail(FVSRN_ECUDA, "cannot allocate the shared framebuffer");
  } else {
    CUDA_TRY(cudaHostAlloc(&staging, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  }
  std::vector<std::function<int()>> fns;
  for (int i = 0; i < n; ++i) {
    fvsrn_model_t m = reps[i];
    fns.push_back([=, &evals] {
      float* d = p2p ? frame : mapped_device_ptr(staging);
      return render_share(m, tf, c, st, t, i, n, d, !p2p, &evals);
    });
  }
  rc = run_on_devices(reps, n, fns);
  if (!rc) {
    if (p2p) {
      cudaSetDevice(home);
      StreamGuard sg;
      const cudaError_t e1 = cudaMemcpyAsync(out, frame, bytes, cudaMemcpyDeviceToHost, sg.s);
      const cudaError_t e2 = cudaStreamSynchronize(sg.s);
      if (e1 != cudaSuccess || e2 != cudaSuccess) {
        cudaGetLastError();
        rc = fail(FVSRN_ECUDA, std::string("frame copy: ") + cudaGetErrorString(e1 ? e1 : e2));
      }
    } else {
      std::memcpy(out, staging, bytes);
    }
  }
  if (frame) frame_cache().give(home, bytes, frame);
  if (staging) cudaFreeHost(staging);
  if (rc) return rc;
  if (eval_count) *eval_count = evals.load();
  return FVSRN_OK;
}

int32_t fvsrn_host_alloc(uint64_t bytes, void** ptr) {
  if (!ptr) return fail(FVSRN_EINVAL, "null argument");
  *ptr = nullptr;
  CUDA_TRY(cudaHostAlloc(ptr, bytes ? bytes : 1, cudaHostAllocPortable | cudaHostAllocMapped));
  return FVSRN_OK;
}

int32_t fvsrn_host_free(void* ptr) {
  if (ptr) CUDA_TRY(cudaFreeHost(ptr));
  return FVSRN_OK;
}

int32_t fvsrn_fused_eval(fvsrn_model_t m, const float* x, int64_t n, float* out) {
  if (!m || (n > 0 && (!x || !out))) return fail(FVSRN_EINVAL, "null argument");
  if (n == 0) return FVSRN_OK;
  CUDA_TRY(cudaSetDevice(m->device));
  StreamGuard sg;
  const int oc = m->head == FVSRN_HEAD_DENSITY ? 1 : 4;
  const size_t xb = (size_t)n * m->d_in * sizeof(float), ob = (size_t)n * oc * sizeof(float);
  char* buf = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&buf, xb + ob, sg.s));
  float* d_x = (float*)buf;
  float* d_out = (float*)(buf + xb);
  CUDA_TRY(cudaMemcpyAsync(d_x, x, xb, cudaMemcpyHostToDevice, sg.s));
  NetDev net = m->px.net;
  int d_in = m->d_in, k0 = m->k0x;
  long long count = n;
  const float* xp = d_x;
  void* args[] = {&net, &d_in, &k0, &xp, &count, &d_out};
  const size_t smem = stage_smem_bytes(net, false, m->k0x);
  int rc = launch(m, KernelKind::kFused, smem, args, sg.s, n / 32 + 1);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(out, d_out, ob, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaFreeAsync(buf, sg.s));
  CUDA_TRY(cudaStreamSynchronize(sg.s));
  return FVSRN_OK;
}

}  // extern "C"

// ============================================================================ volumes
struct fvsrn_volume {
  int device = 0, X = 0, Y = 0, Z = 0, num_sms = 148;
  float* d_values = nullptr;
  ~fvsrn_volume() {
    cudaSetDevice(device);
    cudaFree(d_values);
  }
};

namespace {

int volume_render_impl(fvsrn_volume_t v, const fvsrn_tf* tf, const fvsrn_camera* c,
                       const double* d_o, const double* d_d, long long n_rays,
                       const fvsrn_settings* st, const fvsrn_shard* shard, float* d_out,
                       unsigned long long* d_counters /* [samples, nonfinite] or null */,
                       cudaStream_t s) {
  int rc = check_settings(st);
  if (rc) return rc;
  if (!tf) return fail(FVSRN_EINVAL, "VolumeSource needs a transfer function");
  TFDev th;
  if ((rc = build_tf(tf, th))) return rc;
  CUDA_TRY(cudaSetDevice(v->device));
  char* scratch = nullptr;
  const size_t off_ct = (sizeof(TFDev) + 255) / 256 * 256;
  CUDA_TRY(cudaMallocAsync((void**)&scratch, off_ct + 64, s));
  TFDev* d_tf = (TFDev*)scratch;
  unsigned long long* ct = (unsigned long long*)(scratch + off_ct);
  CUDA_TRY(cudaMemcpyAsync(d_tf, &th, sizeof(TFDev), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemsetAsync(ct, 0, 32, s));
  MarchDev md = march_for(st);
  CamDev cam{};
  ShardDev sh{};
  sh.world = 1;
  long long n_slots = n_rays;
  void* lpt = nullptr;
  if (!d_o) {
    if (c->width < 1 || c->height < 1) return fail(FVSRN_EINVAL, "image dimensions must be positive");
    cam = cam_for(c);
    if (c->has_basis) {
      for (int a = 0; a < 3; ++a) { cam.fwd[a] = c->b_forward[a]; cam.right[a] = c->b_right[a]; cam.up[a] = c->b_up[a]; }
      cam.half_w = c->half_w;
      cam.half_h = c->half_h;
    }
    sh.rank = shard ? shard->rank : 0;
    sh.world = shard ? shard->world : 1;
    sh.compact = shard ? shard->compact : 0;
    if (sh.world < 1 || sh.rank < 0 || sh.rank >= sh.world) return fail(FVSRN_EINVAL, "bad shard");
    sh.tiles_x = (c->width + kTile - 1) / kTile;
    sh.n_tiles = sh.tiles_x * ((c->height + kTile - 1) / kTile);
    const long long local_tiles = std::max(0ll, (long long)(sh.n_tiles - sh.rank + sh.world - 1) / sh.world);
    n_slots = local_tiles * 64;
    if (sh.compact) {
      const long long max_local = (sh.n_tiles + sh.world - 1) / sh.world;
      if (max_local > local_tiles)
        CUDA_TRY(cudaMemsetAsync(d_out + local_tiles * 64 * 4, 0, (max_local - local_tiles) * 64 * 16, s));
    }
    if (local_tiles >= 2 * v->num_sms && g_lpt_enabled) {
      const int nl = (int)local_tiles;
      CUDA_TRY(cudaMallocAsync(&lpt, 12 * (size_t)nl + 256, s));
      unsigned* cost = (unsigned*)lpt;
      unsigned* order = cost + (size_t)nl;
      CUDA_TRY(launch_tile_order(cam, md, sh, nl, cost, order, s));
      sh.order = order;
    }
  }
  VolDev vd{v->d_values, v->X, v->Y, v->Z};
  if (n_slots > 0)
    CUDA_TRY(launch_volume_dvr(vd, d_tf, md, cam, sh, d_o, d_d, n_slots, d_out, ct, v->num_sms, s));
  if (d_counters) CUDA_TRY(cudaMemcpyAsync(d_counters, ct + 1, 16, cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(cudaFreeAsync(scratch, s));
  if (lpt) CUDA_TRY(cudaFreeAsync(lpt, s));
  return FVSRN_OK;
}

}  // namespace

extern "C" {

int32_t fvsrn_volume_create(const float* values, int32_t nx, int32_t ny, int32_t nz, int32_t device,
                            fvsrn_volume_t* out) {
  if (!values || !out) return fail(FVSRN_EINVAL, "null argument");
  *out = nullptr;
  if (nx < 2 || ny < 2 || nz < 2) return fail(FVSRN_EINVAL, "volume dims must be >= 2 for trilinear sampling");
  auto v = std::make_unique<fvsrn_volume>();
  v->device = device;
  v->X = nx; v->Y = ny; v->Z = nz;
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  v->num_sms = prop.multiProcessorCount;
  int rc = upload(values, sizeof(float) * (size_t)nx * ny * nz, (void**)&v->d_values);
  if (rc) return rc;
  *out = v.release();
  return FVSRN_OK;
}

int32_t fvsrn_volume_destroy(fvsrn_volume_t v) {
  delete v;
  return FVSRN_OK;
}

int32_t fvsrn_volume_render(fvsrn_volume_t v, const fvsrn_tf* tf, const fvsrn_camera* c,
                            const fvsrn_settings* st, float* out, uint64_t* sample_count) {
  if (!v || !c || !out) return fail(FVSRN_EINVAL, "null argument");
  if (c->width < 1 || c->height < 1) return fail(FVSRN_EINVAL, "image dimensions must be positive");
  CUDA_TRY(cudaSetDevice(v->device));
  StreamGuard sg;
  const size_t bytes = (size_t)c->width * c->height * 16;
  float* d_out = nullptr;
  CUDA_TRY(cudaMallocAsync(&d_out, bytes + 16, sg.s));
  unsigned long long* d_cnt = (unsigned long long*)((char*)d_out + bytes);
  int rc = volume_render_impl(v, tf, c, nullptr, nullptr, 0, st, nullptr, d_out, d_cnt, sg.s);
  if (rc) { cudaFreeAsync(d_out, sg.s); cudaStreamSynchronize(sg.s); return rc; }
  unsigned long long cnt[2] = {0, 0};
  CUDA_TRY(cudaMemcpyAsync(out, d_out, bytes, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaMemcpyAsync(cnt, d_cnt, 16, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaFreeAsync(d_out, sg.s));
  CUDA_TRY(cudaStreamSynchronize(sg.s));
  if (sample_count) *sample_count = cnt[0];
  if (cnt[1]) return fail(FVSRN_EINVAL, "image contains non-finite values");
  return FVSRN_OK;
}

int32_t fvsrn_volume_render_device(fvsrn_volume_t v, const fvsrn_tf* tf, const fvsrn_camera* c,
                                   const fvsrn_settings* st, const fvsrn_shard* shard, float* d_out,
                                   void* stream) {
  if (!v || !c || !d_out) return fail(FVSRN_EINVAL, "null argument");
  return volume_render_impl(v, tf, c, nullptr, nullptr, 0, st, shard, d_out, nullptr,
                            (cudaStream_t)stream);
}

int32_t fvsrn_volume_render_rays(fvsrn_volume_t v, const fvsrn_tf* tf, const double* origins,
                                 const double* dirs, int64_t n, const fvsrn_settings* st,
                                 float* out_px, uint64_t* sample_count) {
  if (!v || (n > 0 && (!origins || !dirs || !out_px))) return fail(FVSRN_EINVAL, "null argument");
  if (sample_count) *sample_count = 0;
  if (n == 0) return check_settings(st);
  CUDA_TRY(cudaSetDevice(v->device));
  StreamGuard sg;
  const size_t rb = (size_t)n * 3 * sizeof(double), ob = (size_t)n * 16;
  char* buf = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&buf, 2 * rb + ob + 16, sg.s));
  double* d_o = (double*)buf;
  double* d_d = (double*)(buf + rb);
  float* d_out = (float*)(buf + 2 * rb);
  unsigned long long* d_cnt = (unsigned long long*)(buf + 2 * rb + ob);
  CUDA_TRY(cudaMemcpyAsync(d_o, origins, rb, cudaMemcpyHostToDevice, sg.s));
  CUDA_TRY(cudaMemcpyAsync(d_d, dirs, rb, cudaMemcpyHostToDevice, sg.s));
  int rc = volume_render_impl(v, tf, nullptr, d_o, d_d, n, st, nullptr, d_out, d_cnt, sg.s);
  if (rc) { cudaFreeAsync(buf, sg.s); cudaStreamSynchronize(sg.s); return rc; }
  unsigned long long cnt[2] = {0, 0};
  CUDA_TRY(cudaMemcpyAsync(out_px, d_out, ob, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaMemcpyAsync(cnt, d_cnt, 16, cudaMemcpyDeviceToHost, sg.s));
  CUDA_TRY(cudaFreeAsync(buf, sg.s));
  CUDA_TRY(cudaStreamSynchronize(sg.s));
  if (sample_count) *sample_count = cnt[0];
  return FVSRN_OK;
}

}  // extern "C"
