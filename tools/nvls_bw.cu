// Micro-benchmark of NVSwitch multicast throughput (tools only, not product).
#include <cuda_runtime.h>
#include <cstdint>
extern "C" {
__global__ void k_ldreduce(const float4* __restrict__ mc, int64_t n4, float* out, int unroll_dummy) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t j = i + u * stride;
      v[u] = make_float4(0, 0, 0, 0);
      if (j < n4)
        asm volatile("multimem.ld_reduce.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "l"(mc + j) : "memory");
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) out[0] = acc;
}
__global__ void k_mcstore(float4* mc, int64_t n4) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 v = make_float4(1, 2, 3, 4);
    asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(mc + i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  }
}
__global__ void k_p2p_read(const float4* __restrict__ peer, int64_t n4, float* out) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t j = i + u * stride;
      v[u] = j < n4 ? peer[j] : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) out[0] = acc;
}
__global__ void k_p2p_write(float4* peer, int64_t n4) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride)
    peer[i] = make_float4(1, 2, 3, 4);
}
int run(int which, void* p, int64_t n4, void* out, int grid, int block, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (which == 0) k_ldreduce<<<grid, block, 0, s>>>((const float4*)p, n4, (float*)out, 0);
  if (which == 1) k_mcstore<<<grid, block, 0, s>>>((float4*)p, n4);
  if (which == 2) k_p2p_read<<<grid, block, 0, s>>>((const float4*)p, n4, (float*)out);
  if (which == 3) k_p2p_write<<<grid, block, 0, s>>>((float4*)p, n4);
  return (int)cudaGetLastError();
}
}
