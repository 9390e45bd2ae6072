// Throughput of the interpreter's library-free elementary functions
// (fastmath.cuh fm_exp / fm_tanh) next to CUDA's expf / tanhf / powf and
// the FP64 / conversion instructions an FP64-based pow would be built from. Each
// thread runs NCH independent chains of ITER evaluations; reported as
// evaluations per clock per SM (at the device's reported max clock).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2501_17168_b200/csrc tools/microbench/fastmath_tp.cu -o /tmp/fastmath_tp
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "fastmath.cuh"

#define NCH 4
#define ITER 1024

using namespace evogp;

template <int OP>
__global__ void kern(float* out, float seed) {
  float s[NCH];
  double d[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    s[k] = seed + 0.001f * (threadIdx.x & 31) + 0.01f * k;
    d[k] = s[k];
  }
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const float x = s[k];
      if (OP == 0) s[k] = expf(-x);
      if (OP == 1) s[k] = fm_exp(-x);
      if (OP == 2) s[k] = tanhf(__fmaf_rn(x, 3.0f, 0.5f));
      if (OP == 3) s[k] = fm_tanh(__fmaf_rn(x, 3.0f, 0.5f));
      if (OP == 4) s[k] = powf(fabsf(x) + 1.5f, 0.7f);
      if (OP == 6) d[k] = __fma_rn(d[k], 0.9999, 1e-4);  // DFMA chain
      if (OP == 7) s[k] = __double2float_rn(static_cast<double>(x) * 0.5 + 0.25);  // F2F pair + DFMA
      if (OP == 8) {
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d[k]));
        d[k] = r + 0.5;
      }
      if (OP == 9) s[k] = logf(fabsf(x) + 1.5f);
    }
  }
  float t = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) t += s[k] + static_cast<float>(d[k]);
  if (t == 12345.678f) out[0] = t;
}

template <int OP>
void run(const char* name) {
  float* dd;
  cudaMalloc(&dd, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256;
  kern<OP><<<blocks, threads>>>(dd, 0.3f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<OP><<<blocks, threads>>>(dd, 0.3f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double n = static_cast<double>(blocks) * threads * NCH * ITER;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"op\":\"%s\",\"evals_per_clk_per_sm\":%.2f,\"ms\":%.3f}\n", name, n / (ms * 1e-3) / (clk * 1e3) / sms, ms);
  cudaFree(dd);
}

int main() {
  run<0>("expf");
  run<1>("fm_exp");
  run<2>("tanhf");
  run<3>("fm_tanh");
  run<4>("powf");
  run<6>("dfma");
  run<7>("cvt_f32_f64_pair+dfma");
  run<8>("rcp_approx_f64");
  run<9>("logf");
  return 0;
}
