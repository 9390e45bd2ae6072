// Pipe-throughput microbenchmark for the roofline denominators (FP32 FMA, MUFU, libm paths).
// Each thread runs NCH independent dependency chains of ITER ops; ops/s = threads*NCH*ITER / t.
#include <cstdio>
#include <cuda_runtime.h>
#define NCH 8
#define ITER 4096
template <int OP>
__global__ void kern(float* out, float seed) {
  float v[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) v[c] = seed + 0.001f * (threadIdx.x + c);
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      float x = v[c];
      if (OP == 0) x = fmaf(x, 0.9999f, 0.0001f);
      if (OP == 1) { float r; asm volatile("sin.approx.f32 %0, %1;" : "=f"(r) : "f"(x)); x = r; }
      if (OP == 2) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); x = r; }
      if (OP == 3) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); x = r * 0.5f; }
      if (OP == 4) x = sinf(x);
      if (OP == 5) x = tanf(x) * 0.5f;
      if (OP == 6) x = expf(x) * 0.3f;
      if (OP == 7) x = logf(fabsf(x) + 1.5f);
      if (OP == 8) x = powf(fabsf(x) + 0.5f, 0.7f);
      if (OP == 9) x = tanhf(x) + 0.1f;
      if (OP == 10) x = __fdiv_rn(1.0f, x + 2.0f);
      if (OP == 11) x = __fadd_rn(x, 0.5f) ;
      v[c] = x;
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) s += v[c];
  if (s == 12345.678f) out[0] = s;
}
template <int OP>
void run(const char* name) {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 8, threads = 256;
  kern<OP><<<blocks, threads>>>(d, 0.3f);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<OP><<<blocks, threads>>>(d, 0.3f);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = (double)blocks * threads * NCH * ITER;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
  printf("{\"op\":\"%s\",\"Gops_s\":%.1f,\"ops_per_clk_per_sm_at_max_clock\":%.2f,\"ms\":%.3f}\n", name, ops / (ms * 1e-3) / 1e9, per_clk_sm, ms);
  cudaFree(d);
}
int main() {
  run<0>("ffma"); run<11>("fadd_rn"); run<1>("mufu_sin_approx"); run<2>("mufu_rcp_approx"); run<3>("mufu_ex2_approx");
  run<4>("sinf"); run<5>("tanf"); run<6>("expf"); run<7>("logf"); run<8>("powf"); run<9>("tanhf"); run<10>("fdiv_rn");
  return 0;
}
