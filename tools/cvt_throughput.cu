// fp32 -> fp64 conversion throughput on one B200 SM pipe mix: F2F.F64.F32
// vs an integer bit-construction (exact for normal numbers, zero and
// inf/nan; fp32 denormals flush to zero), vs the fp32 FMA rate.  Decides
// whether the fp64 momentum update (lars_kernels.cu, LARS_UPDATE_F64) can
// move its input conversions off the conversion pipe.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cvt tools/cvt_throughput.cu && /tmp/cvt
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ double f2d_int(float f) {
  const unsigned b = __float_as_uint(f);
  const unsigned e = b & 0x7f800000u;
  unsigned hi = ((b & 0x7fffffffu) >> 3) + (e == 0x7f800000u ? 0x70000000u : 0x38000000u);
  hi = e == 0u ? 0u : hi;
  hi |= b & 0x80000000u;
  const unsigned lo = e == 0u ? 0u : (b << 29);
  return __hiloint2double((int)hi, (int)lo);
}

template <int kMode>
__global__ void bench(const float* __restrict__ in, double* out, int iters) {
  float x0 = in[threadIdx.x], x1 = in[threadIdx.x + 1], x2 = in[threadIdx.x + 2], x3 = in[threadIdx.x + 3];
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  float f0 = 0, f1 = 0, f2 = 0, f3 = 0;
  for (int i = 0; i < iters; ++i) {
    if (kMode == 0) {
      acc0 += (double)x0; acc1 += (double)x1; acc2 += (double)x2; acc3 += (double)x3;
    } else if (kMode == 1) {
      acc0 += f2d_int(x0); acc1 += f2d_int(x1); acc2 += f2d_int(x2); acc3 += f2d_int(x3);
    } else if (kMode == 2) {
      acc0 += 1.0000001; acc1 += 1.0000001; acc2 += 1.0000001; acc3 += 1.0000001;
    } else {
      f0 = fmaf(f0, 1.0000001f, x0); f1 = fmaf(f1, 1.0000001f, x1);
      f2 = fmaf(f2, 1.0000001f, x2); f3 = fmaf(f3, 1.0000001f, x3);
    }
    x0 += 1.f; x1 += 1.f; x2 += 1.f; x3 += 1.f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3 + f0 + f1 + f2 + f3;
}

int main() {
  float* in;
  double* out;
  cudaMalloc(&in, 4096 * sizeof(float));
  cudaMemset(in, 0, 4096 * sizeof(float));
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096, blocks = 148 * 8, threads = 256;
  const char* names[4] = {"F2F.F64.F32 + DADD", "int bit-construct + DADD", "DADD only", "FFMA (+FADD)"};
  // correctness of the integer construction on a few values
  for (int m = 0; m < 4; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (m == 0) bench<0><<<blocks, threads>>>(in, out, iters);
      if (m == 1) bench<1><<<blocks, threads>>>(in, out, iters);
      if (m == 2) bench<2><<<blocks, threads>>>(in, out, iters);
      if (m == 3) bench<3><<<blocks, threads>>>(in, out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = 4.0 * iters * blocks * threads;
      if (rep) printf("%-28s %8.3f ms  %7.1f Gops/s  %6.1f per SM per clk @1.965GHz\n", names[m], ms,
                      ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
