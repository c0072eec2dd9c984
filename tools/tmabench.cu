// tmabench.cu — calibrate TMA box shapes for the stencil ring (not part of the product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmabench tools/tmabench.cu -L/usr/local/cuda/lib64/stubs -lcuda
//
// A W x H fp32 array (row pitch P) is streamed in TW x TH tiles; each tile is
// fetched as a BW x BH TMA box (BW >= TW, BH >= TH: the halo) into an NS-slot
// ring; compute warps wait, optionally store the TW x TH centre to an output
// array (coalesced STG), and release the slot.  Reports algorithmic GB/s
// (read + write of W*H floats when storing).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_(unsigned long long* b, unsigned ph) {
  unsigned done = 0;
  do {
    asm volatile("{.reg .pred P1; mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2; selp.u32 %0,1,0,P1;}"
                 : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
  } while (!done);
}

struct Tm { unsigned long long v[16]; };

template <int NCW>
__global__ void __launch_bounds__(32 * (NCW + 1)) ring(const __grid_constant__ Tm map, const __grid_constant__ Tm omap,
                                                      float* out, int W, int H, long P,
                                                      int TW, int TH, int BW, int BH, int NS, int store, int xoff,
                                                      int xo_plain, int xo_halo) {
  extern __shared__ __align__(128) unsigned char sm[];
  int stage = ((BW * BH * 4 + 127) / 128) * 128;
  unsigned long long* full = (unsigned long long*)(sm + NS * stage);
  unsigned long long* empty = full + NS;
  // PL > 1: 3-D streaming mode — the H rows are PL planes of H/PL rows; a unit is one
  // (tx, ty) tile column and the producer streams its PL planes in order
  const int PL = xoff > 0 ? xoff : 1;
  const int XO = BW > TW ? xo_halo : xo_plain;
  const int xs_store = xo_plain;
  const int HP = H / PL;
  int ntx = W / TW, nty = (PL > 1 ? HP : H) / TH, nunits = ntx * nty;
  const int nl = PL;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(NCW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NCW) {
    if (lane == 0) {
      unsigned L = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        int tx = u % ntx, ty = u / ntx;
        for (int pl = 0; pl < nl; ++pl, ++L) {
          unsigned slot = L % NS;
          if (L >= (unsigned)NS) wait_(&empty[slot], ((L / NS) - 1) & 1);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[slot])),
                       "r"(BW * BH * 4) : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
              ::"r"(su32(sm + slot * stage)), "l"((unsigned long long)&map), "r"(tx * TW + XO), "r"(ty * TH + pl * HP),
              "r"(su32(&full[slot])) : "memory");
        }
      }
    }
    return;
  }
  unsigned L = 0;
  if (store == 3 && threadIdx.x == 0) asm volatile("prefetch.tensormap [%0];" ::"l"((unsigned long long)&omap) : "memory");
  for (int uu = blockIdx.x * nl; uu < nunits * nl; uu += (uu % nl == nl - 1) ? (gridDim.x - 1) * nl + 1 : 1, ++L) {
    int u = uu / nl, pl = uu % nl;
    unsigned slot = L % NS;
    wait_(&full[slot], (L / NS) & 1);
    int tx = u % ntx, ty0 = u / ntx;
    int ty = ty0 + pl * (HP / TH);
    (void)omap;
    const float* t = (const float*)(sm + slot * stage);
    if (store == 1) {
      // each warp: rows warp, warp+NCW, ...; lanes over columns
      for (int r = warp; r < TH; r += NCW)
        for (int c = lane; c < TW; c += 32)
          out[(long)(ty * TH + r) * P + tx * TW + c + xs_store] = t[r * BW + c + 1];
    } else if (store == 2) {
      for (int r = warp; r < TH; r += NCW)
        for (int c = lane * 4; c < TW; c += 128) {
          float4 v = make_float4(t[r * BW + c + 1], t[r * BW + c + 2], t[r * BW + c + 3], t[r * BW + c + 4]);
          *reinterpret_cast<float4*>(&out[(long)(ty * TH + r) * P + tx * TW + c + xs_store]) = v;
        }
    } else if (store == 3) {
      // stage the TW x TH result in smem (own buffer per warp-row group), TMA-store it
      float* ob = (float*)(sm + NS * stage + 2 * NS * 8 + 1024) + (L & 1) * TW * TH;
      // wait until the TMA store that used this buffer two units ago has read it
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"r"(32 * NCW));
      for (int r = warp; r < TH; r += NCW)
        for (int c = lane; c < TW; c += 32) ob[r * TW + c] = t[r * BW + c + 1];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"r"(32 * NCW));
      if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                     ::"l"((unsigned long long)&omap), "r"(tx * TW), "r"(ty * TH), "r"(su32(ob)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[slot])) : "memory");
  }
  if (store == 3 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void fillrand(float* a, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = i * 0x9E3779B97F4A7C15ULL + 12345;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    a[i] = (float)((z >> 40) & 0xffffff) * (1.0f / 16777216.0f) - 0.5f;
  }
}

int main() {
  cuInit(0);
  const int W = 1024;
  const int H = 1 << 20;   // 4 GiB fp32
  const long P = getenv("PITCH") ? atol(getenv("PITCH")) : 1028;
  float *a, *o;
  CK(cudaMalloc(&a, P * (H + 64) * 4));
  CK(cudaMalloc(&o, P * (H + 64) * 4));
  CK(cudaMemset(a, 0, P * (H + 64) * 4));
  CK(cudaMemset(o, 0, P * (H + 64) * 4));
  if (getenv("RANDINIT")) {
    fillrand<<<148 * 8, 256>>>(a, (size_t)P * (H + 64));
    fillrand<<<148 * 8, 256>>>(o, (size_t)P * (H + 64));
    CK(cudaDeviceSynchronize());
  }
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  struct C { int TW, TH, BW, BH, NS, store, xoff; };
  C cs_all[] = {
      {128, 16, 128, 16, 10, 1, 1}, {128, 16, 136, 18, 10, 1, 1}, {128, 16, 128, 16, 10, 2, 1},
      {128, 16, 136, 18, 10, 2, 1}};
  int which = getenv("CFG") ? atoi(getenv("CFG")) : -1;
  C cs[4];
  int ncs = 0;
  for (int i = 0; i < 4; ++i)
    if (which < 0 || which == i) cs[ncs++] = cs_all[i];
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int ci = 0; ci < ncs; ++ci) {
    C c = cs[ci];
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)P, (cuuint64_t)H};
    cuuint64_t str[1] = {(cuuint64_t)P * 4};
    cuuint32_t box[2] = {(cuuint32_t)c.BW, (cuuint32_t)c.BH};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, dims, str, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); continue; }
    int stage = ((c.BW * c.BH * 4 + 127) / 128) * 128;
    int smem = c.NS * stage + 2 * c.NS * 8 + (c.store == 3 ? 1024 + 2 * c.TW * c.TH * 4 : 0);
    CUtensorMap om;
    cuuint32_t obox[2] = {(cuuint32_t)c.TW, (cuuint32_t)c.TH};
    r = cuTensorMapEncodeTiled(&om, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, o, dims, str, obox, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode out failed %d\n", r); continue; }
    Tm otm;
    memcpy(&otm, &om, sizeof otm);
    auto k = ring<8>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 288, smem);
    Tm tm;
    memcpy(&tm, &m, sizeof tm);
    int Hc = (H / c.TH) * c.TH - 64;
    Hc = (Hc / c.TH) * c.TH;
    if (c.xoff > 1) Hc = H - 1024 * 32;     // planes mode: 1024 planes of 992 rows
    if (getenv("PINGPONG")) {
      // first pass writes `o`; the measured pass reads the freshly written `o`
      CUtensorMap m2, om2;
      cuTensorMapEncodeTiled(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, o, dims, str, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      cuTensorMapEncodeTiled(&om2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, dims, str, obox, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      Tm tm2, otm2;
      memcpy(&tm2, &m2, sizeof tm2);
      memcpy(&otm2, &om2, sizeof otm2);
      int xop = getenv("XOP") ? atoi(getenv("XOP")) : 0, xoh = getenv("XOH") ? atoi(getenv("XOH")) : 0;
      k<<<nb * nsm, 288, smem>>>(tm, otm, o, W, Hc, P, c.TW, c.TH, c.BW, c.BH, c.NS, 1, c.xoff, xop, xoh);
      k<<<nb * nsm, 288, smem>>>(tm2, otm2, a, W, Hc, P, c.TW, c.TH, c.BW, c.BH, c.NS, c.store, c.xoff, xop, xoh);
      CK(cudaDeviceSynchronize());
      continue;
    }
    for (int rep = 0; rep < (getenv("ONCE") ? 1 : 2); ++rep) {
      cudaEventRecord(e0);
      int xop = getenv("XOP") ? atoi(getenv("XOP")) : 0, xoh = getenv("XOH") ? atoi(getenv("XOH")) : 0;
      k<<<nb * nsm, 288, smem>>>(tm, otm, o, W, Hc, P, c.TW, c.TH, c.BW, c.BH, c.NS, c.store, c.xoff, xop, xoh);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double bytes = (double)W * Hc * 4 * (c.store ? 2 : 1);
      if (rep || getenv("ONCE")) printf("P=%ld TW=%3d TH=%2d BW=%3d BH=%2d NS=%2d store=%d planes=%d blk/SM=%d: %.3f ms %.0f GB/s\n", P, c.TW, c.TH,
                      c.BW, c.BH, c.NS, c.store, c.xoff, nb, ms, bytes / ms / 1e6);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
