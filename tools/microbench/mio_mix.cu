// Does MUFU share an issue queue with shared-memory loads?  Time per iteration of
// (a) 8 cos, (b) 8 LDS.64, (c) 8 cos + 8 LDS.64, (d) 8 cos + 8 FFMA, (e) 8 cos + 4 LDS.128.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters) {
  __shared__ float2 sm[1024];
  __shared__ float4 sm4[512];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_float2(i * 1e-3f, 1.f);
  for (int i = threadIdx.x; i < 512; i += blockDim.x) sm4[i] = make_float4(i, 1, 2, 3);
  __syncthreads();
  float a[8];
  float2 acc = make_float2(0.f, 0.f);
  float4 acc4 = make_float4(0, 0, 0, 0);
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0 || MODE == 2 || MODE == 3 || MODE == 4)
        asm volatile("cos.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
      if (MODE == 1 || MODE == 2) {
        float2 v;
        asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y)
                     : "r"((unsigned)__cvta_generic_to_shared(&sm[(lane + 32 * j + i) & 1023])));
        acc.x += v.x; acc.y += v.y;
      }
      if (MODE == 3) asm volatile("fma.rn.f32 %0, %0, 0f3F000000, 0f3F000000;" : "+f"(acc.x));
      if (MODE == 4 && (j & 1)) {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "r"((unsigned)__cvta_generic_to_shared(&sm4[(lane + 32 * j + i) & 511])));
        acc4.x += v.x; acc4.w += v.w;
      }
    }
  }
  float s = acc.x + acc.y + acc4.x + acc4.w;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 512);
  const int iters = 4096;
  const char* names[5] = {"8 cos", "8 LDS.64", "8 cos + 8 LDS.64", "8 cos + 8 FFMA", "8 cos + 4 LDS.128"};
  void (*fs[5])(float*, int) = {k<0>, k<1>, k<2>, k<3>, k<4>};
  for (int m = 0; m < 5; ++m) {
    fs[m]<<<sms * 8, 512>>>(out, 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    fs[m]<<<sms * 8, 512>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_iters = (double)sms * 8 * 16 * iters;   // 16 warps per block
    printf("%-20s %.3f ms  %.2f clk per warp-iteration per SMSP\n", names[m], ms,
           ms * 1e-3 * clk * 1e3 / (warp_iters / (sms * 4)));
  }
  return 0;
}
