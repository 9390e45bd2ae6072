// Packed-FP32 (sm_100 FFMA2 / FADD2 / FMUL2) vs scalar throughput, 3-register
// and immediate forms. Each thread runs NCH independent chains of ITER ops;
// reported as FP32 lane-ops (a packed op counts 2) per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>
#define NCH 8
#define ITER 4096
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(u64 v) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a + b; }
template <int OP>
__global__ void kern(float* out, float seed, float m, float c) {
  u64 v[NCH];
  float s[NCH];
  const u64 M = pk(m, m * 1.0001f), C = pk(c, c * 0.999f);
#pragma unroll
  for (int k = 0; k < NCH; ++k) { v[k] = pk(seed + 0.001f * (threadIdx.x + k), seed - 0.002f * k); s[k] = seed + 0.003f * k; }
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      if (OP == 0) s[k] = fmaf(s[k], m, c);                                      // FFMA 3-reg
      if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[k]) : "l"(M), "l"(C));  // FFMA2
      if (OP == 2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(v[k]) : "l"(C));      // FADD2
      if (OP == 3) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(v[k]) : "l"(M));      // FMUL2
      if (OP == 4) s[k] = __fadd_rn(s[k], c);                                    // FADD 2-reg
      if (OP == 5) s[k] = __fmul_rn(s[k], m);                                    // FMUL 2-reg
      if (OP == 6) { asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[k]) : "l"(M), "l"(C));
                     float r; asm volatile("sin.approx.f32 %0, %1;" : "=f"(r) : "f"(s[k])); s[k] = r; }  // FFMA2 + MUFU
      if (OP == 7) { s[k] = fmaf(s[k], m, c); }
    }
  }
  float t = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) t += s[k] + lo(v[k]);
  if (t == 12345.678f) out[0] = t;
}
template <int OP>
void run(const char* name, double lanes_per_op) {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 8, threads = 256;
  kern<OP><<<blocks, threads>>>(d, 0.3f, 0.9999f, 0.0001f);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<OP><<<blocks, threads>>>(d, 0.3f, 0.9999f, 0.0001f);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double instr = (double)blocks * threads * NCH * ITER;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"op\":\"%s\",\"thread_instr_per_clk_per_sm\":%.2f,\"fp32_lane_ops_per_clk_per_sm\":%.2f,\"ms\":%.3f}\n", name,
         instr / (ms * 1e-3) / (clk * 1e3) / sms, lanes_per_op * instr / (ms * 1e-3) / (clk * 1e3) / sms, ms);
  cudaFree(d);
}
int main() {
  run<0>("ffma_3reg", 1); run<1>("ffma2_3reg", 2); run<2>("fadd2", 2); run<3>("fmul2", 2); run<4>("fadd_2reg", 1);
  run<5>("fmul_2reg", 1); run<6>("ffma2+mufu_sin (per pair)", 2);
  return 0;
}
