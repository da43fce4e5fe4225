// MUFU throughput on this GPU: independent cos.approx / ex2.approx / tanh.approx chains,
// many warps per SM; reports results per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters, float seed) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed + threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) asm volatile("cos.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
      else if (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
      else if (OP == 2) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(a[j]));
      else asm volatile("sin.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);   // kHz
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
  const int iters = 4096;
  const char* names[4] = {"cos.approx", "ex2.approx", "tanh.approx", "sin.approx"};
  for (int op = 0; op < 4; ++op) {
    void (*f)(float*, int, float) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : k<3>;
    f<<<sms * 8, 1024>>>(out, 16, 0.1f);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    f<<<sms * 8, 1024>>>(out, iters, 0.1f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)sms * 8 * 1024 * iters * 8;
    // MUFU ops per clock per SM at the max SM clock (clocks reported separately)
    printf("%-12s %.3f ms  %.1f Gop/s  %.2f per clk per SM @ %d MHz\n", names[op], ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
