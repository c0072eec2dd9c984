/* abi_slabs.c — P slab images through the C ABI only (no Python, no torch): the
 * halo exchange of Machine._halo_exchange (runtime.py:643-711) and the fused
 * peer-store steps, driven by a C host the way a Fortran/C coarray program would.
 *
 *   gcc -O2 -o tools/abi_slabs tools/abi_slabs.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1502_03504_b200 -llope_b200 -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,'$ORIGIN/../paper_1502_03504_b200' -Wl,-rpath,/usr/local/cuda/lib64
 *   tools/abi_slabs rr    P n steps     # P images in this process, one stream each (one GPU)
 *   tools/abi_slabs procs P n steps     # P processes, image k on GPU k (needs P GPUs)
 *
 * Field: the 3-D seven-point kernel (configs 3/5); every image holds an n x n x n slab
 * of the global n x n x (P n) domain, slabs along z.  Setup:
 * lope_comm_create / lope_comm_export, the records gathered in rank order (an array in
 * rr mode, a shared mapping in procs mode), lope_comm_connect.  Then the reference
 * loop: HALO_TRANSFER (lope_halo_exchange), steps-1 fused steps (lope_comm_step),
 * lope_comm_sync and the final plain launch (lope_launch), timed with CUDA events.
 * rr mode also runs the undecomposed domain on one block and compares every interior
 * value bit for bit; prints one JSON line.
 *
 * rr mode issues every image's operation k before any image's operation k+1 (the
 * halo exchange in its two phases), so every stream wait's signal is enqueued before
 * the wait: no kernel waits on another, and no queue order can deadlock.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

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
      exit(1);                                                               \
    }                                                                        \
  } while (0)

#define CUCHECK(x)                                                                       \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      fprintf(stderr, "%s -> %s\n", #x, cudaGetErrorString(e_));                         \
      exit(1);                                                                           \
    }                                                                                    \
  } while (0)

typedef struct {
  lope_comm* comm;
  lope_layout L;
  void* buf[2];
  int live;
  cudaStream_t st;
} Image;

static void image_init(Image* im, lope_kernel* k, int P, int r, int64_t n, uint8_t* rec) {
  (void)k;
  int64_t ext[3] = {n, n, n};
  int32_t lo[3] = {1, 1, 1}, hi[3] = {1, 1, 1};
  CHECK(lope_layout_init(&im->L, 3, LOPE_F32, ext, lo, hi));
  for (int b = 0; b < 2; ++b) {
    CUCHECK(cudaMalloc(&im->buf[b], im->L.count * 4));
    CUCHECK(cudaMemset(im->buf[b], 0, im->L.count * 4));
  }
  int64_t gext[3] = {n, n, n * P}, gorg[3] = {0, 0, n * r};
  CHECK(lope_fill_hash(&im->L, im->buf[0], 20260823ULL, gext, gorg, 0));
  CUCHECK(cudaStreamCreateWithFlags(&im->st, cudaStreamNonBlocking));
  CUCHECK(cudaDeviceSynchronize());
  im->live = 0;
  CHECK(lope_comm_create(P, r, &im->comm));
  CHECK(lope_comm_export(im->comm, &im->L, im->buf[0], im->buf[1], rec));
}

/* the reference loop over all images, operation by operation across the images */
static void run_rr(Image* im, int P, lope_kernel* k, int steps, float* ms_out) {
  cudaEvent_t e0, e1;
  CUCHECK(cudaEventCreate(&e0));
  CUCHECK(cudaEventCreate(&e1));
  CUCHECK(cudaDeviceSynchronize());
  CUCHECK(cudaEventRecord(e0, im[0].st));
  for (int r = 1; r < P; ++r) CUCHECK(cudaStreamWaitEvent(im[r].st, e0, 0));
  for (int r = 0; r < P; ++r) CHECK(lope_halo_exchange_begin(im[r].comm, im[r].live, 7, im[r].st));
  for (int r = 0; r < P; ++r) CHECK(lope_halo_exchange_end(im[r].comm, im[r].st));
  for (int s = 0; s < steps - 1; ++s)
    for (int r = 0; r < P; ++r) {
      CHECK(lope_comm_step(im[r].comm, k, im[r].live, NULL, NULL, im[r].st));
      im[r].live ^= 1;
    }
  int64_t rng[6] = {1, im[0].L.interior[0], 1, im[0].L.interior[1], 1, im[0].L.interior[2]};
  for (int r = 0; r < P; ++r) {
    CHECK(lope_comm_sync(im[r].comm, im[r].st));
    const void* in[1] = {im[r].buf[im[r].live]};
    void* out[1] = {im[r].buf[im[r].live ^ 1]};
    CHECK(lope_launch(k, &im[r].L, rng, in, out, NULL, NULL, im[r].st));
    im[r].live ^= 1;
  }
  cudaEvent_t ej;
  CUCHECK(cudaEventCreate(&ej));
  for (int r = 1; r < P; ++r) {
    CUCHECK(cudaEventRecord(ej, im[r].st));
    CUCHECK(cudaStreamWaitEvent(im[0].st, ej, 0));
  }
  CUCHECK(cudaEventRecord(e1, im[0].st));
  CUCHECK(cudaEventSynchronize(e1));
  CUCHECK(cudaEventElapsedTime(ms_out, e0, e1));
}

static int mode_rr(int P, int64_t n, int steps) {
  lope_kernel* k = NULL;
  CHECK(lope_kernel_compile(kLap3d7, strlen(kLap3d7), LOPE_F32, &k));
  const int rs = lope_comm_record_size();
  uint8_t* recs = (uint8_t*)calloc((size_t)P, (size_t)rs);
  Image* im = (Image*)calloc((size_t)P, sizeof(Image));
  for (int r = 0; r < P; ++r) image_init(&im[r], k, P, r, n, recs + (size_t)r * rs);
  for (int r = 0; r < P; ++r) CHECK(lope_comm_connect(im[r].comm, recs));
  float ms = 0;
  run_rr(im, P, k, steps, &ms);
  /* the undecomposed domain on one block: HALO_TRANSFER, steps-1 fused steps, a launch */
  lope_layout G;
  int64_t gext[3] = {n, n, n * P}, gorg[3] = {0, 0, 0};
  int32_t lo[3] = {1, 1, 1}, hi[3] = {1, 1, 1};
  CHECK(lope_layout_init(&G, 3, LOPE_F32, gext, lo, hi));
  void *ga, *gb;
  CUCHECK(cudaMalloc(&ga, G.count * 4));
  CUCHECK(cudaMalloc(&gb, G.count * 4));
  CUCHECK(cudaMemset(ga, 0, G.count * 4));
  CUCHECK(cudaMemset(gb, 0, G.count * 4));
  CHECK(lope_fill_hash(&G, ga, 20260823ULL, gext, gorg, 0));
  cudaEvent_t g0, g1;
  CUCHECK(cudaEventCreate(&g0));
  CUCHECK(cudaEventCreate(&g1));
  CUCHECK(cudaEventRecord(g0, 0));
  CHECK(lope_halo_fill(&G, ga, 7, 0));
  for (int s = 0; s < steps - 1; ++s) {
    CHECK(lope_step(k, &G, ga, gb, NULL, NULL, 7, 0));
    void* t = ga; ga = gb; gb = t;
  }
  int64_t rng[6] = {1, n, 1, n, 1, n * P};
  const void* in[1] = {ga};
  void* out[1] = {gb};
  CHECK(lope_launch(k, &G, rng, in, out, NULL, NULL, 0));
  CUCHECK(cudaEventRecord(g1, 0));
  CUCHECK(cudaDeviceSynchronize());
  float ms_single = 0;
  CUCHECK(cudaEventElapsedTime(&ms_single, g0, g1));
  /* compare interiors */
  const size_t slab = (size_t)n * n * n;
  float* hs = (float*)malloc(slab * 4);
  float* hg = (float*)malloc(slab * 4);
  long long bad = 0;
  for (int r = 0; r < P; ++r) {
    CHECK(lope_unpack(&im[r].L, im[r].buf[im[r].live], hs, 0));
    /* the same planes of the global block: unpack the global interior plane range */
    CUCHECK(cudaDeviceSynchronize());
    for (int64_t z = 0; z < n; ++z) {
      const char* src = (const char*)gb + 4 * (G.base + G.lo[0] + (G.lo[1]) * G.stride[1] +
                                                (G.lo[2] + n * r + z) * G.stride[2]);
      CUCHECK(cudaMemcpy2D(hg + z * n * n, (size_t)n * 4, src, (size_t)G.stride[1] * 4, (size_t)n * 4, (size_t)n,
                           cudaMemcpyDeviceToHost));
    }
    bad += memcmp(hs, hg, slab * 4) != 0;
    for (size_t i = 0; i < slab && bad == 0; ++i)
      if (hs[i] != hg[i]) bad = 1;
  }
  double pts = (double)n * n * n * P;
  printf("{\"mode\": \"rr\", \"images\": %d, \"slab\": [%lld, %lld, %lld], \"steps\": %d, \"ms_total\": %.3f, "
         "\"gpts\": %.2f, \"ms_total_undecomposed\": %.3f, \"gpts_undecomposed\": %.2f, "
         "\"bitwise_equal_to_undecomposed\": %s, \"err\": \"%s\"}\n",
         P, (long long)n, (long long)n, (long long)n, steps, ms, pts * steps / (ms / 1e3) / 1e9, ms_single,
         pts * steps / (ms_single / 1e3) / 1e9, bad ? "false" : "true", cudaGetErrorString(cudaGetLastError()));
  for (int r = 0; r < P; ++r) lope_comm_destroy(im[r].comm);
  lope_kernel_destroy(k);
  return bad ? 2 : 0;
}

/* one process per GPU: records through a shared anonymous mapping, a spin barrier on it */
static int mode_procs(int P, int64_t n, int steps) {
  /* CUDA is initialised only in the children (never before fork) */
  const int rs = lope_comm_record_size();
  size_t bytes = (size_t)P * rs + 4096;
  uint8_t* shm = (uint8_t*)mmap(NULL, bytes, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_ANONYMOUS, -1, 0);
  volatile int* count = (volatile int*)(shm + (size_t)P * rs);
  memset(shm, 0, bytes);
  for (int r = 0; r < P; ++r) {
    if (fork() == 0) {
      int ndev = 0;
      CUCHECK(cudaGetDeviceCount(&ndev));
      if (ndev < P) {
        fprintf(stderr, "procs mode needs %d GPUs (found %d): ranks sharing a GPU must not wait on each other\n",
                P, ndev);
        _exit(3);
      }
      CUCHECK(cudaSetDevice(r));
      lope_kernel* k = NULL;
      CHECK(lope_kernel_compile(kLap3d7, strlen(kLap3d7), LOPE_F32, &k));
      Image im;
      image_init(&im, k, P, r, n, shm + (size_t)r * rs);
      __sync_fetch_and_add(count, 1);
      while (*count < P) usleep(1000);
      CHECK(lope_comm_connect(im.comm, shm));
      float ms = 0;
      cudaEvent_t e0, e1;
      CUCHECK(cudaEventCreate(&e0));
      CUCHECK(cudaEventCreate(&e1));
      CUCHECK(cudaEventRecord(e0, im.st));
      CHECK(lope_halo_exchange(im.comm, im.live, 7, im.st));
      for (int s = 0; s < steps - 1; ++s) {
        CHECK(lope_comm_step(im.comm, k, im.live, NULL, NULL, im.st));
        im.live ^= 1;
      }
      CHECK(lope_comm_sync(im.comm, im.st));
      CUCHECK(cudaEventRecord(e1, im.st));
      CUCHECK(cudaEventSynchronize(e1));
      CUCHECK(cudaEventElapsedTime(&ms, e0, e1));
      printf("{\"mode\": \"procs\", \"rank\": %d, \"images\": %d, \"steps\": %d, \"ms_total\": %.3f}\n", r, P,
             steps, ms);
      __sync_fetch_and_add(count, 1);
      while (*count < 2 * P) usleep(1000);
      lope_comm_destroy(im.comm);
      _exit(0);
    }
  }
  int st = 0, worst = 0;
  for (int r = 0; r < P; ++r) {
    wait(&st);
    if (!WIFEXITED(st) || WEXITSTATUS(st)) worst = 1;
  }
  return worst;
}

int main(int argc, char** argv) {
  const char* mode = argc > 1 ? argv[1] : "rr";
  int P = argc > 2 ? atoi(argv[2]) : 2;
  int64_t n = argc > 3 ? atoll(argv[3]) : 256;
  int steps = argc > 4 ? atoi(argv[4]) : 10;
  const char* cache = getenv("LOPE_CACHE_DIR");
  if (cache) lope_set_cache_dir(cache);
  if (P < 1 || steps < 1 || n < 2) {
    fprintf(stderr, "usage: abi_slabs rr|procs P n steps\n");
    return 1;
  }
  if (!strcmp(mode, "procs")) return mode_procs(P, n, steps);
  setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);   /* one hardware queue per image stream */
  return mode_rr(P, n, steps);
}
