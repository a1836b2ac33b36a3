// Launch-overhead microbenchmark for the fused step's launch configuration
// (296 CTAs x 256 threads, cooperative, ~113 KB dynamic shared memory): how
// much of a small-shard step's event-timed duration is launch and teardown,
// and what the shared-memory carveout switch after the L2 flush costs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lo tools/launch_overhead.cu && /tmp/lo
//
// Each case: flush (1 GiB memset + 256 MiB read kernel), event, kernel,
// event; median of 50.  Kernel variants: empty; one global load + store per
// thread (the shortest dependent chain a real kernel has).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void empty_kernel(int* p) {
  extern __shared__ int s[];
  if (p && threadIdx.x == 0 && blockIdx.x == 100000) s[0] = p[0];
}

__global__ void touch_kernel(const float* __restrict__ src, float* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  dst[i] = __ldcg(src + i) * 2.f;
}

__global__ void read_kernel(const float4* __restrict__ src, float* out, size_t n4) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(src + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const int grid = 296, threads = 256;
  float *flush = nullptr, *clean = nullptr, *a = nullptr, *b = nullptr;
  CK(cudaMalloc(&flush, size_t(1) << 30));
  CK(cudaMalloc(&clean, size_t(1) << 28));
  CK(cudaMemset(clean, 0, size_t(1) << 28));
  CK(cudaMalloc(&a, grid * threads * 4));
  CK(cudaMalloc(&b, grid * threads * 4));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int smem_big = 113 * 1024;
  CK(cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_big));
  CK(cudaFuncSetAttribute(touch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_big));

  struct Case { const char* name; bool touch; bool coop; int smem; bool flush; bool carveout_read; };
  std::vector<Case> cases = {
      {"empty   plain  smem 0      flush", false, false, 0, true, false},
      {"empty   plain  smem 113K   flush", false, false, smem_big, true, false},
      {"empty   coop   smem 0      flush", false, true, 0, true, false},
      {"empty   coop   smem 113K   flush", false, true, smem_big, true, false},
      {"empty   coop   smem 113K   flush(read kernel carveout=max)", false, true, smem_big, true, true},
      {"empty   coop   smem 113K   no flush", false, true, smem_big, false, false},
      {"touch   coop   smem 113K   flush", true, true, smem_big, true, false},
      {"touch   plain  smem 0      flush", true, false, 0, true, false},
      {"touch   coop   smem 113K   no flush", true, true, smem_big, false, false},
  };
  for (const Case& c : cases) {
    CK(cudaFuncSetAttribute(read_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                            c.carveout_read ? 100 : -1));
    std::vector<float> t;
    for (int rep = 0; rep < 60; ++rep) {
      if (c.flush) {
        CK(cudaMemsetAsync(flush, rep & 0xff, size_t(1) << 30, st));
        read_kernel<<<1184, 256, 0, st>>>(reinterpret_cast<const float4*>(clean), b, (size_t(1) << 28) / 16);
      }
      CK(cudaEventRecord(e0, st));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = c.smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = c.coop ? 1 : 0;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (c.touch) {
        const float* src = a;
        float* dst = b;
        void* args[] = {&src, &dst};
        CK(cudaLaunchKernelExC(&cfg, (void*)touch_kernel, args));
      } else {
        int* p = nullptr;
        void* args[] = {&p};
        CK(cudaLaunchKernelExC(&cfg, (void*)empty_kernel, args));
      }
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep >= 10) t.push_back(ms * 1000.f);
    }
    std::sort(t.begin(), t.end());
    printf("%-60s median %6.2f us  min %6.2f  max %6.2f\n", c.name, t[t.size() / 2], t.front(), t.back());
  }
  return 0;
}
