/*
 * Plain-C use of the drop-in boundary (include/lars_b200.h), no Python:
 * a three-layer parameter set, one scheduled LARS step through lars_step(),
 * checked against a straight fp64 restatement of the reference step
 * (batchlab optim.py:76-95 scheduled_lr, :98-108 lars_local_lr,
 * :111-114 group_local_lr, :128-131 the update).
 *
 *   gcc -std=c99 -O2 -I include tests/c_abi/lars_abi_example.c \
 *       -L paper_1709_05011_b200/_lib -llars_b200 -L /usr/local/cuda/lib64 -lcudart -lm
 *
 * Exit status 0 = parity within the one-step tolerance; prints one line.
 */
#define _POSIX_C_SOURCE 200112L
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "lars_b200.h"

#define NSEG 3
#define CHECK_CUDA(x)                                                     \
  do {                                                                    \
    cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess) {                                              \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
      return 2;                                                           \
    }                                                                     \
  } while (0)
#define CHECK_LARS(x)                                                     \
  do {                                                                    \
    int r_ = (x);                                                         \
    if (r_ != LARS_OK) {                                                  \
      fprintf(stderr, "%s: %s\n", #x, lars_strerror(r_));                 \
      return 2;                                                           \
    }                                                                     \
  } while (0)

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static double uniform(void) { /* splitmix64 -> [0, 1) */
  uint64_t z = (rng_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

int main(void) {
  /* conv-like weight (LARS), bias (skipped: lambda = 1), fc weight (LARS) */
  const int64_t len[NSEG] = {1000, 64, 4096};
  const int32_t trust[NSEG] = {LARS_SEG_TRUST, 0, LARS_SEG_TRUST};
  lars_segment_t segs[NSEG];
  int64_t off = 0;
  for (int i = 0; i < NSEG; ++i) {
    segs[i].offset = off;
    segs[i].length = len[i];
    segs[i].layer = i;
    segs[i].flags = trust[i];
    off += (len[i] + 31) / 32 * 32; /* 128-byte aligned groups */
  }
  const int64_t n = off;
  float *w = calloc(n, 4), *g = calloc(n, 4), *m = calloc(n, 4);
  float *w_out = calloc(n, 4), *m_out = calloc(n, 4);
  for (int i = 0; i < NSEG; ++i)
    for (int64_t j = segs[i].offset; j < segs[i].offset + len[i]; ++j) {
      w[j] = (float)(0.1 * (uniform() - 0.5));
      g[j] = (float)(512.0 * 1e-3 * (uniform() - 0.5)); /* summed over B = 512 */
      m[j] = (float)(1e-3 * (uniform() - 0.5));
    }

  lars_hparams_t hp;
  memset(&hp, 0, sizeof hp);
  hp.base_lr = 0.32;
  hp.momentum = 0.9;
  hp.weight_decay = 5e-4;
  hp.poly_power = 2.0;
  hp.trust = 1e-3;
  hp.grad_scale = 1.0 / 512;
  hp.warmup_iters = 20;
  hp.max_iters = 200;
  hp.lars_enabled = 1;
  hp.flags = LARS_STEP_ADVANCE_ITER;
  const int64_t iteration = 30;

  void* plan = NULL;
  CHECK_LARS(lars_plan_create(segs, NSEG, NSEG, 0, 0, &plan));
  lars_plan_info_t info;
  CHECK_LARS(lars_plan_info(plan, &info));
  float *d_w, *d_g, *d_m;
  int64_t* d_iter;
  double *d_sumsq, *d_lambda;
  lars_step_info_t* d_info;
  void* d_ws;
  CHECK_CUDA(cudaMalloc((void**)&d_w, n * 4));
  CHECK_CUDA(cudaMalloc((void**)&d_g, n * 4));
  CHECK_CUDA(cudaMalloc((void**)&d_m, n * 4));
  CHECK_CUDA(cudaMalloc((void**)&d_iter, sizeof(int64_t)));
  CHECK_CUDA(cudaMalloc((void**)&d_sumsq, 2 * NSEG * sizeof(double)));
  CHECK_CUDA(cudaMalloc((void**)&d_lambda, NSEG * sizeof(double)));
  CHECK_CUDA(cudaMalloc((void**)&d_info, sizeof(lars_step_info_t)));
  CHECK_CUDA(cudaMalloc(&d_ws, (size_t)info.workspace_bytes));
  CHECK_CUDA(cudaMemcpy(d_w, w, n * 4, cudaMemcpyHostToDevice));
  CHECK_CUDA(cudaMemcpy(d_g, g, n * 4, cudaMemcpyHostToDevice));
  CHECK_CUDA(cudaMemcpy(d_m, m, n * 4, cudaMemcpyHostToDevice));
  CHECK_CUDA(cudaMemcpy(d_iter, &iteration, sizeof iteration, cudaMemcpyHostToDevice));
  CHECK_LARS(lars_workspace_init(plan, d_ws, NULL));

  CHECK_LARS(lars_step(plan, d_w, d_g, d_m, &hp, d_iter, d_sumsq, d_lambda, d_info, d_ws, NULL));
  CHECK_CUDA(cudaDeviceSynchronize());

  double lam_gpu[NSEG];
  lars_step_info_t hinfo;
  int64_t it_after = 0;
  CHECK_CUDA(cudaMemcpy(w_out, d_w, n * 4, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(m_out, d_m, n * 4, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(lam_gpu, d_lambda, sizeof lam_gpu, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(&hinfo, d_info, sizeof hinfo, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(&it_after, d_iter, sizeof it_after, cudaMemcpyDeviceToHost));

  /* fp64 reference: scheduled_lr (optim.py:88-95) */
  const double progress = (double)(iteration - hp.warmup_iters) / (double)(hp.max_iters - hp.warmup_iters);
  const double lr = hp.base_lr * pow(1.0 - progress, hp.poly_power);
  int bad = 0;
  double worst = 0.0;
  for (int i = 0; i < NSEG; ++i) {
    const int64_t a = segs[i].offset, b = a + len[i];
    double wn = 0.0, gn = 0.0;
    for (int64_t j = a; j < b; ++j) {
      wn += (double)w[j] * w[j];
      gn += (double)g[j] * g[j] * hp.grad_scale * hp.grad_scale;
    }
    wn = sqrt(wn);
    gn = sqrt(gn);
    double lam = 1.0; /* group_local_lr (optim.py:111-114) */
    if (trust[i]) {   /* lars_local_lr (optim.py:98-108) */
      const double denom = gn + hp.weight_decay * wn;
      lam = wn == 0.0 ? 0.0 : (denom == 0.0 ? 1.0 : hp.trust * wn / denom);
    }
    if (fabs(lam_gpu[i] - lam) > 1e-6 * fabs(lam)) {
      fprintf(stderr, "layer %d lambda %.17g vs %.17g\n", i, lam_gpu[i], lam);
      ++bad;
    }
    double rms = 0.0;
    double* wr = malloc(len[i] * sizeof(double));
    double* mr = malloc(len[i] * sizeof(double));
    for (int64_t j = a; j < b; ++j) { /* optim.py:128-131 */
      const double s = (double)g[j] * hp.grad_scale + hp.weight_decay * w[j];
      mr[j - a] = hp.momentum * m[j] + (lam * lr) * s;
      wr[j - a] = w[j] - mr[j - a];
      rms += wr[j - a] * wr[j - a];
    }
    rms = sqrt(rms / (double)len[i]);
    for (int64_t j = a; j < b; ++j) {
      const double err = fabs(w_out[j] - wr[j - a]);
      const double tol = 1e-5 * fabs(wr[j - a]) + 1e-7 * rms;
      if (err > tol) ++bad;
      if (err / (fabs(wr[j - a]) + 1e-30) > worst && fabs(wr[j - a]) > rms) worst = err / fabs(wr[j - a]);
    }
    free(wr);
    free(mr);
  }
  if (fabs(hinfo.lr - lr) > 1e-12 * lr || hinfo.iteration != iteration || it_after != iteration + 1 ||
      hinfo.nonfinite_layer != INT32_MAX)
    ++bad;
  /* host-resident fp64 groups (the reference ParamSet's storage, one array
   * per group): pinned in place, DMA'd into the flat fp32 layout and back;
   * the round trip must give each value rounded to fp32 */
  int host_bad = 0;
  {
    double* hin[NSEG];
    double* hout[NSEG];
    lars_host_span_t sin[NSEG], sout[NSEG];
    double* d_stage;
    float* d_flat;
    CHECK_CUDA(cudaMalloc((void**)&d_stage, n * sizeof(double)));
    CHECK_CUDA(cudaMemset(d_stage, 0, n * sizeof(double)));
    CHECK_CUDA(cudaMalloc((void**)&d_flat, n * 4));
    for (int i = 0; i < NSEG; ++i) {
      const size_t bytes = ((size_t)len[i] * sizeof(double) + 4095) / 4096 * 4096;
      if (posix_memalign((void**)&hin[i], 4096, bytes) || posix_memalign((void**)&hout[i], 4096, bytes))
        return 2;
      for (int64_t j = 0; j < len[i]; ++j) {
        hin[i][j] = (double)w[segs[i].offset + j] + 1e-11 * (uniform() - 0.5); /* not fp32-exact */
        hout[i][j] = -1.0;
      }
      CHECK_LARS(lars_host_register(hin[i], (int64_t)bytes));
      CHECK_LARS(lars_host_register(hout[i], (int64_t)bytes));
      sin[i].host = hin[i];
      sout[i].host = hout[i];
      sin[i].offset = sout[i].offset = segs[i].offset;
      sin[i].numel = sout[i].numel = len[i];
    }
    CHECK_LARS(lars_host_copy_in(sin, NSEG, d_stage, d_flat, n, NULL));
    CHECK_LARS(lars_host_copy_out(d_flat, d_stage, n, sout, NSEG, NULL));
    CHECK_CUDA(cudaDeviceSynchronize());
    for (int i = 0; i < NSEG; ++i) {
      for (int64_t j = 0; j < len[i]; ++j)
        if (hout[i][j] != (double)(float)hin[i][j]) ++host_bad;
      CHECK_LARS(lars_host_unregister(hin[i]));
      CHECK_LARS(lars_host_unregister(hout[i]));
      free(hin[i]);
      free(hout[i]);
    }
    cudaFree(d_stage);
    cudaFree(d_flat);
  }
  if (host_bad) {
    fprintf(stderr, "host round trip: %d values differ\n", host_bad);
    ++bad;
  }
  printf("lars_abi_example: abi %d, grid %d, %lld params, lr %.9g, lambda %.6g %.6g %.6g, "
         "max rel err %.3g, host fp64 round trip %s, %s\n",
         lars_abi_version(), info.grid, (long long)n, hinfo.lr, lam_gpu[0], lam_gpu[1], lam_gpu[2],
         worst, host_bad ? "FAIL" : "ok", bad ? "FAIL" : "ok");
  lars_plan_destroy(plan);
  cudaFree(d_w);
  cudaFree(d_g);
  cudaFree(d_m);
  cudaFree(d_iter);
  cudaFree(d_sumsq);
  cudaFree(d_lambda);
  cudaFree(d_info);
  cudaFree(d_ws);
  free(w);
  free(g);
  free(m);
  free(w_out);
  free(m_out);
  return bad ? 1 : 0;
}
