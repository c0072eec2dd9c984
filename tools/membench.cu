// membench.cu — calibration kernels for the stencil roofline (not part of the product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membench tools/membench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy4(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// padded layout: row pitch P floats, interior starts at +off in each row
__global__ void copy_rows(const float* __restrict__ a, float* __restrict__ b, int nx, int ny, int nz,
                          long P, long PP, int off) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nx) return;
  for (int k = blockIdx.z; k < nz; k += gridDim.z)
    for (int j = blockIdx.y; j < ny; j += gridDim.y) {
      long i = off + x + (j + 1) * P + (k + 1) * PP;
      b[i] = a[i];
    }
}

__global__ void st7(const float* __restrict__ a, float* __restrict__ b, int nx, int ny, int nz, long P,
                    long PP, int off) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nx) return;
  for (int k = blockIdx.z; k < nz; k += gridDim.z)
    for (int j = blockIdx.y; j < ny; j += gridDim.y) {
      long i = off + x + (j + 1) * P + (k + 1) * PP;
      float c = __ldg(a + i);
      float s = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(__ldg(a + i - 1), __ldg(a + i + 1)), __ldg(a + i - P)),
                                              __ldg(a + i + P)), __ldg(a + i - PP)), __ldg(a + i + PP));
      b[i] = __fadd_rn(c, __fmul_rn(0.125f, __fadd_rn(s, -__fmul_rn(6.f, c))));
    }
}

// 2.5D streaming: thread column walks z with registers, x/y neighbours via L1 (__ldg)
__global__ void st7_stream(const float* __restrict__ a, float* __restrict__ b, int nx, int ny, int nz, long P,
                           long PP, int off, int zc) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int j = blockIdx.y;
  if (x >= nx) return;
  int z0 = blockIdx.z * zc;
  int z1 = min(nz, z0 + zc);
  long i = off + x + (j + 1) * P + (z0 + 1) * PP;
  float m = __ldg(a + i - PP), c = __ldg(a + i);
  for (int k = z0; k < z1; ++k, i += PP) {
    float p = __ldg(a + i + PP);
    float s = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(__ldg(a + i - 1), __ldg(a + i + 1)), __ldg(a + i - P)),
                                            __ldg(a + i + P)), m), p);
    b[i] = __fadd_rn(c, __fmul_rn(0.125f, __fadd_rn(s, -__fmul_rn(6.f, c))));
    m = c;
    c = p;
  }
}

__global__ void fillrand(float* a, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = (i + seed) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    a[i] = (float)((z >> 40) & 0xffffff) * (1.0f / 16777216.0f) - 0.5f;
  }
}

int main() {
  if (getenv("RANDCOPY")) {
    size_t cnt = (size_t)1 << 30;   // 4 GiB fp32
    float *a, *b;
    cudaMalloc(&a, cnt * 4);
    cudaMalloc(&b, cnt * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
      if (mode == 0) { cudaMemset(a, 0, cnt * 4); cudaMemset(b, 0, cnt * 4); }
      if (mode == 1) { fillrand<<<148 * 8, 256>>>(a, cnt, 1); cudaMemset(b, 0, cnt * 4); }
      if (mode == 2) { fillrand<<<148 * 8, 256>>>(a, cnt, 1); fillrand<<<148 * 8, 256>>>(b, cnt, 7); }
      cudaDeviceSynchronize();
      float ms;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        copy4<<<148 * 8, 256>>>((float4*)a, (float4*)b, cnt / 4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      printf("copy4 %s: %.3f ms %.0f GB/s\n", mode == 0 ? "zeros->zeros" : mode == 1 ? "random->zeros" : "random->random",
             ms, 2.0 * cnt * 4 / ms / 1e6);
    }
    return 0;
  }
  const int n = 1024;
  float ms;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int off : {1, 4, 32}) {
    long P = ((off + n + 1 + 31) / 32) * 32;
    if (off == 1) P = 1028;
    long PP = P * (n + 2);
    size_t cnt = PP * (n + 2);
    float *a, *b;
    cudaMalloc(&a, cnt * 4);
    cudaMalloc(&b, cnt * 4);
    cudaMemset(a, 0, cnt * 4);
    cudaMemset(b, 0, cnt * 4);
    double bytes = 2.0 * 4 * (double)n * n * n;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      for (int it = 0; it < 5; ++it) copy4<<<148 * 8, 256>>>((float4*)a, (float4*)b, cnt / 4);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("copy4    off=%2d: %.3f ms  %.0f GB/s (buffer bytes)\n", off, ms / 5, 2.0 * cnt * 4 / (ms / 5) / 1e6);
      dim3 g((n + 127) / 128, n, n > 65535 ? 65535 : n);
      cudaEventRecord(e0);
      for (int it = 0; it < 5; ++it) copy_rows<<<g, 128>>>(a, b, n, n, n, P, PP, off);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("copyrows off=%2d: %.3f ms  %.0f GB/s\n", off, ms / 5, bytes / (ms / 5) / 1e6);
      cudaEventRecord(e0);
      for (int it = 0; it < 5; ++it) st7<<<g, 128>>>(a, b, n, n, n, P, PP, off);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("st7      off=%2d: %.3f ms  %.0f GB/s\n", off, ms / 5, bytes / (ms / 5) / 1e6);
      for (int zc : {16, 64}) {
        dim3 g2((n + 127) / 128, n, (n + zc - 1) / zc);
        cudaEventRecord(e0);
        for (int it = 0; it < 5; ++it) st7_stream<<<g2, 128>>>(a, b, n, n, n, P, PP, off, zc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("st7strm  off=%2d zc=%d: %.3f ms  %.0f GB/s\n", off, zc, ms / 5, bytes / (ms / 5) / 1e6);
      }
    }
    cudaFree(a);
    cudaFree(b);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
