// Shared-memory store/load "bank conflict" counter control: what ncu's
// l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_{st,ld} report for the
// interpreter's stack access pattern — each lane a contiguous 16-byte (or 8 /
// 4-byte) word, the warp one contiguous 512-byte (256 / 128) range, i.e.
// conflict-free by construction — next to a deliberately 2-way conflicting
// 32-bit pattern. Run under ncu with the metrics in tools/gpu_smem_conflicts.sh.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define ITER 4096

// W = bytes per lane (4, 8, 16); STRIDE = lane stride in words of W (1: contiguous)
template <int W, int STRIDE>
__global__ void st_kernel(float* out) {
  __shared__ __align__(16) float s[32 * 4 * 2 * 2];
  const int lane = threadIdx.x & 31;
  float4 v = make_float4(lane, lane + 1, lane + 2, lane + 3);
  for (int it = 0; it < ITER; ++it) {
    char* p = reinterpret_cast<char*>(s) + (lane * STRIDE) * W;
    if (W == 16) *reinterpret_cast<float4*>(p) = v;
    if (W == 8) *reinterpret_cast<float2*>(p) = make_float2(v.x, v.y);
    if (W == 4) *reinterpret_cast<float*>(p) = v.x;
    v.x += 1.0f;
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[lane];
}

template <int W, int STRIDE>
__global__ void ld_kernel(float* out) {
  __shared__ __align__(16) float s[32 * 4 * 2 * 2];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 32 * 4 * 2 * 2; i += blockDim.x) s[i] = i;
  __syncthreads();
  float acc = 0.f;
  for (int it = 0; it < ITER; ++it) {
    const char* p = reinterpret_cast<const char*>(s) + (lane * STRIDE) * W;
    if (W == 16) {
      const float4 q = *reinterpret_cast<const float4*>(p);
      acc += q.x + q.w;
    }
    if (W == 8) {
      const float2 q = *reinterpret_cast<const float2*>(p);
      acc += q.x + q.y;
    }
    if (W == 4) acc += *reinterpret_cast<const float*>(p);
    __syncwarp();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// The packed interpreter's push exactly (hot_ptx.inc, K = 8): the lane's two
// 16-byte halves at [top] and [top + 512], top = warp base + lane * 16, moving
// by 1024 bytes per push (SD slots), 4 warps per CTA with per-warp regions.
__global__ void push_kernel(float* out, int region_bytes) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = dsm + warp * region_bytes + 1024 + lane * 16;  // after a 1 KB program row
  uint32_t top0 = static_cast<uint32_t>(__cvta_generic_to_shared(base));
  unsigned long long a = lane, b = lane + 1, c = lane + 2, d = lane + 3;
  for (int it = 0; it < ITER; ++it) {
    uint32_t top = top0 + (it % 5) * 1024;
    asm volatile("st.shared.v2.b64 [%0+0], {%1, %2};\n st.shared.v2.b64 [%0+512], {%3, %4};" ::"r"(top), "l"(a), "l"(b),
                 "l"(c), "l"(d)
                 : "memory");
    a += 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = static_cast<float>(dsm[lane]);
}

// The same pushes while the other warps of the CTA stream global loads
// through L1 (the interpreter's VAR leaves): L1 fills share the SRAM data banks
// with shared memory.
__global__ void push_with_loads_kernel(float* out, const float4* g, int region_bytes, int n4) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp & 1) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (int it = 0; it < ITER / 4; ++it) {
      const float4 v = __ldg(g + ((blockIdx.x * 977 + it * 131 + warp * 7) % (n4 / 32)) * 32 + lane);
      acc.x += v.x;
      acc.y += v.w;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
    return;
  }
  unsigned char* base = dsm + warp * region_bytes + 1024 + lane * 16;
  uint32_t top0 = static_cast<uint32_t>(__cvta_generic_to_shared(base));
  unsigned long long a = lane, b = lane + 1, c = lane + 2, d = lane + 3;
  for (int it = 0; it < ITER; ++it) {
    uint32_t top = top0 + (it % 5) * 1024;
    asm volatile("st.shared.v2.b64 [%0+0], {%1, %2};\n st.shared.v2.b64 [%0+512], {%3, %4};" ::"r"(top), "l"(a), "l"(b),
                 "l"(c), "l"(d)
                 : "memory");
    a += 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = static_cast<float>(dsm[lane]);
}

int main() {
  float* out;
  cudaMalloc(&out, 1 << 20);
  // one warp per block, 148 blocks: 148 * ITER warp-instructions per kernel
  st_kernel<16, 1><<<148, 32>>>(out);
  st_kernel<8, 1><<<148, 32>>>(out);
  st_kernel<4, 1><<<148, 32>>>(out);
  st_kernel<4, 2><<<148, 32>>>(out);  // 2-way conflict: lanes l and l+16 share a bank
  ld_kernel<16, 1><<<148, 32>>>(out);
  ld_kernel<8, 1><<<148, 32>>>(out);
  ld_kernel<4, 1><<<148, 32>>>(out);
  ld_kernel<4, 2><<<148, 32>>>(out);
  cudaFuncSetAttribute(push_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 6144);
  push_kernel<<<148, 128, 4 * 6144>>>(out, 6144);
  float4* g;
  const int n4 = 1 << 24;  // 256 MB: every load misses L1
  cudaMalloc(&g, static_cast<size_t>(n4) * sizeof(float4));
  cudaMemset(g, 0, static_cast<size_t>(n4) * sizeof(float4));
  cudaFuncSetAttribute(push_with_loads_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 6144);
  push_with_loads_kernel<<<148, 128, 4 * 6144>>>(out, g, 6144, n4);
  cudaDeviceSynchronize();
  printf("smem_conflicts done (%s)\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
