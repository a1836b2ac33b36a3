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
// TMA bulk copies peer global -> shared (one issuing thread per CTA, 4 x 16 KB
// stages completed through mbarriers); the data is only landed, not used.
__global__ void k_p2p_bulk(const unsigned char* peer, int64_t nbytes) {
  constexpr int kCh = 16384, kSt = 4;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar[kSt];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSt; ++s) {
      const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int64_t nch = nbytes / kCh;
  int64_t i = 0;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++i) {
    const int s = (int)(i % kSt);
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    if (i >= kSt) {
      const unsigned par = (unsigned)((i / kSt - 1) & 1);
      unsigned done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(b), "r"(par) : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(kCh) : "memory");
    const unsigned d = (unsigned)__cvta_generic_to_shared(sm + s * kCh);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(d), "l"(peer + c * kCh), "r"(kCh), "r"(b) : "memory");
  }
  // drain
  for (int64_t j = (i > kSt ? i - kSt : 0); j < i; ++j) {
    const int s = (int)(j % kSt);
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    const unsigned par = (unsigned)((j / kSt) & 1);
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(b), "r"(par) : "memory");
  }
}
int run(int which, void* p, int64_t n4, void* out, int grid, int block, void* stream) {
  if (which == 4) {
    static bool init = false;
    if (!init) {
      cudaFuncSetAttribute(k_p2p_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      init = true;
    }
    k_p2p_bulk<<<grid, 32, 65536, (cudaStream_t)stream>>>((const unsigned char*)p, n4 * 16);
    return (int)cudaGetLastError();
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (which == 0) k_ldreduce<<<grid, block, 0, s>>>((const float4*)p, n4, (float*)out, 0);
  if (which == 1) k_mcstore<<<grid, block, 0, s>>>((float4*)p, n4);
  if (which == 2) k_p2p_read<<<grid, block, 0, s>>>((const float4*)p, n4, (float*)out);
  if (which == 3) k_p2p_write<<<grid, block, 0, s>>>((float4*)p, n4);
  return (int)cudaGetLastError();
}
}
