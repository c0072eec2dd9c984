/* abi_bench.c — drive liblope_b200.so through its C ABI only (no Python, no torch).
 *
 *   gcc -O2 -o tools/abi_bench tools/abi_bench.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1502_03504_b200 -llope_b200 -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,'$ORIGIN/../paper_1502_03504_b200' -Wl,-rpath,/usr/local/cuda/lib64
 *   tools/abi_bench [n] [steps]
 *
 * Runs the 3-D seven-point kernel (config 3) on an n^3 fp32 field allocated with
 * cudaMalloc: lope_fill_hash, lope_halo_fill, then `steps` fused lope_step calls
 * timed with CUDA events.  Also a demonstration of the boundary a C/Fortran host
 * would bind.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lope_b200.h"

static const char* kLap3d7 =
    "LOPE1\n"
    "kernel lap3d7 3\n"
    "array u\n"
    "store u + r u 0 0 0 * c 0x1.0000000000000p-3 + + + + + + r u -1 0 0 r u 1 0 0 r u 0 -1 0 r u 0 1 0 "
    "r u 0 0 -1 r u 0 0 1 n * c 0x1.8000000000000p+2 r u 0 0 0\n"
    "end\n";

#define CHECK(x)                                                             \
  do {                                                                       \
    int rc_ = (x);                                                           \
    if (rc_) {                                                               \
      fprintf(stderr, "%s -> %d: %s\n", #x, rc_, lope_last_error());         \
      return 1;                                                              \
    }                                                                        \
  } while (0)

int main(int argc, char** argv) {
  int64_t n = argc > 1 ? atoll(argv[1]) : 1024;
  int steps = argc > 2 ? atoi(argv[2]) : 20;
  const char* cache = getenv("LOPE_CACHE_DIR");
  if (cache) lope_set_cache_dir(cache);
  lope_layout L;
  int64_t ext[3] = {n, n, n};
  int32_t lo[3] = {1, 1, 1}, hi[3] = {1, 1, 1};
  CHECK(lope_layout_init(&L, 3, LOPE_F32, ext, lo, hi));
  lope_kernel* k = NULL;
  CHECK(lope_kernel_compile(kLap3d7, strlen(kLap3d7), LOPE_F32, &k));
  float *a, *b;
  if (cudaMalloc((void**)&a, L.count * 4) || cudaMalloc((void**)&b, L.count * 4)) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 1;
  }
  cudaMemset(a, 0, L.count * 4);
  cudaMemset(b, 0, L.count * 4);
  int64_t gorg[3] = {0, 0, 0};
  CHECK(lope_fill_hash(&L, a, 20260823ULL, ext, gorg, 0));
  CHECK(lope_halo_fill(&L, a, 7, 0));
  for (int i = 0; i < 3; ++i) {
    CHECK(lope_step(k, &L, a, b, NULL, NULL, 7, 0));
    float* t = a; a = b; b = t;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaDeviceSynchronize();
  cudaEventRecord(e0, 0);
  for (int i = 0; i < steps; ++i) {
    CHECK(lope_step(k, &L, a, b, NULL, NULL, 7, 0));
    float* t = a; a = b; b = t;
  }
  cudaEventRecord(e1, 0);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  double pts = (double)n * n * n;
  printf("{\"n\": %lld, \"steps\": %d, \"ms_per_step\": %.4f, \"gpts\": %.2f, \"alg_GBs\": %.1f, \"err\": \"%s\"}\n",
         (long long)n, steps, ms / steps, pts * steps / (ms / 1e3) / 1e9, 8.0 * pts * steps / (ms / 1e3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  lope_kernel_destroy(k);
  cudaFree(a);
  cudaFree(b);
  return 0;
}
