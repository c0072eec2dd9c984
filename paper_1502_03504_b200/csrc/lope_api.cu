// lope_api.cu — liblope_b200.so: the C ABI of include/lope_b200.h.
//
// Host side: layout arithmetic, argument checks with the reference's error codes,
// NVRTC compilation of IR-specialised kernels for sm_100a (cached on disk and per
// device), TMA descriptor encoding, and launches through the driver API (entry
// points fetched with cudaGetDriverEntryPoint, so the library loads on machines
// without a GPU driver).  Device side (compiled here by nvcc for sm_100a): the
// periodic halo fill, the copy-through of cells outside a launch range, and the
// synthetic-input generator.  The body-specialised stencil kernels live in
// lope_device.cuh and are compiled at run time.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <unistd.h>
#include <vector>

#include "../../include/lope_b200.h"
#include "lope_codegen.h"
#include "lope_internal.h"

static const char* kDeviceSrc =
#include "lope_device_src.inc"
    ;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};
std::mutex g_mu;
std::string g_cache_dir;

int fail(int code, const char* fmt, ...) {
  char buf[2048];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(-(int)e_, "%s failed: %s", #expr, cudaGetErrorString(e_));             \
  } while (0)

// ---------------------------------------------------------------------------
// Driver API entry points

struct Drv {
  bool ok = false;
  std::string why;
  decltype(&cuModuleLoadData) moduleLoadData = nullptr;
  decltype(&cuModuleGetFunction) moduleGetFunction = nullptr;
  decltype(&cuModuleGetGlobal) moduleGetGlobal = nullptr;
  decltype(&cuModuleUnload) moduleUnload = nullptr;
  decltype(&cuFuncSetAttribute) funcSetAttribute = nullptr;
  decltype(&cuFuncGetAttribute) funcGetAttribute = nullptr;
  decltype(&cuLaunchKernel) launchKernel = nullptr;
  decltype(&cuLaunchKernelEx) launchKernelEx = nullptr;   // optional (PDL launches)
  decltype(&cuMemGetAddressRange) memGetAddressRange = nullptr;   // optional (IPC export)
  decltype(&cuTensorMapEncodeTiled) tensorMapEncodeTiled = nullptr;
  decltype(&cuOccupancyMaxActiveBlocksPerMultiprocessor) occupancy = nullptr;
  decltype(&cuGetErrorString) getErrorString = nullptr;
};

Drv& drv() {
  static Drv d;
  static bool inited = false;
  if (inited) return d;
  inited = true;
  auto get = [&](const char* name, void** fn) -> bool {
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !*fn) {
      d.why = std::string("driver entry point ") + name + " unavailable";
      return false;
    }
    return true;
  };
  d.ok = get("cuModuleLoadData", (void**)&d.moduleLoadData) &&
         get("cuModuleGetFunction", (void**)&d.moduleGetFunction) &&
         get("cuModuleGetGlobal", (void**)&d.moduleGetGlobal) &&
         get("cuModuleUnload", (void**)&d.moduleUnload) &&
         get("cuFuncSetAttribute", (void**)&d.funcSetAttribute) &&
         get("cuFuncGetAttribute", (void**)&d.funcGetAttribute) &&
         get("cuLaunchKernel", (void**)&d.launchKernel) &&
         get("cuTensorMapEncodeTiled", (void**)&d.tensorMapEncodeTiled) &&
         get("cuOccupancyMaxActiveBlocksPerMultiprocessor", (void**)&d.occupancy) &&
         get("cuGetErrorString", (void**)&d.getErrorString);
  if (d.ok) {
    std::string keep = d.why;
    if (!get("cuLaunchKernelEx", (void**)&d.launchKernelEx)) d.launchKernelEx = nullptr;
    if (!get("cuMemGetAddressRange", (void**)&d.memGetAddressRange)) d.memGetAddressRange = nullptr;
    d.why = keep;
  }
  return d;
}

int cu_fail(CUresult r, const char* what) {
  const char* s = nullptr;
  if (drv().getErrorString) drv().getErrorString(r, &s);
  return fail(-1000 - (int)r, "%s failed: %s", what, s ? s : "unknown driver error");
}

// ---------------------------------------------------------------------------
// Device-side layout mirror used by the AOT kernels

struct DevLayout {
  int rank;
  int m[3], lo[3], hi[3];
  long long P[3];
  long long S1, S2, B;
};

DevLayout dev_layout(const lope_layout* L) {
  DevLayout d;
  d.rank = L->rank;
  for (int i = 0; i < 3; ++i) {
    d.m[i] = (int)L->interior[i];
    d.lo[i] = L->lo[i];
    d.hi[i] = L->hi[i];
    d.P[i] = L->padded[i];
  }
  d.S1 = L->stride[1];
  d.S2 = L->stride[2];
  d.B = L->base;
  return d;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

// error reporting shared with the other translation units of the library (lope_internal.h)
int lope_set_error(int code, const char* fmt, ...) {
  char buf[2048];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

void lope_count_launch() { g_launches++; }

// ---------------------------------------------------------------------------
// AOT kernels (nvcc, sm_100a)

__device__ __forceinline__ int lope_wrapc(int c, int lo, int m) {
  int i = c - lo;
  if (i < 0) i += m;
  else if (i >= m) i -= m;
  return i + lo;
}

// Periodic halo fill in place: every halo cell (along the masked dims) receives
// its periodic image.  One warp per padded row (c1, c2).
template <class T>
__global__ void __launch_bounds__(256) lope_k_halo_fill(T* __restrict__ buf, DevLayout L, int mask) {
  const long long nrows = L.P[1] * L.P[2];
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = warp; r < nrows; r += nw) {
    const int c1 = (int)(r % L.P[1]);
    const int c2 = (int)(r / L.P[1]);
    const int s1 = (mask & 2) ? lope_wrapc(c1, L.lo[1], L.m[1]) : c1;
    const int s2 = (mask & 4) ? lope_wrapc(c2, L.lo[2], L.m[2]) : c2;
    T* dst = buf + L.B + c1 * L.S1 + c2 * L.S2;
    const T* src = buf + L.B + s1 * L.S1 + s2 * L.S2;
    if (s1 != c1 || s2 != c2) {
      for (int x = lane; x < L.P[0]; x += 32)
        dst[x] = src[(mask & 1) ? lope_wrapc(x, L.lo[0], L.m[0]) : x];
    } else if (mask & 1) {
      const int nh = L.lo[0] + L.hi[0];
      for (int q = lane; q < nh; q += 32) {
        const int x = q < L.lo[0] ? q : L.m[0] + L.lo[0] + (q - L.lo[0]);
        dst[x] = src[lope_wrapc(x, L.lo[0], L.m[0])];
      }
    }
  }
}

// out := in for every padded cell outside the half-open box [b, e) (padded coords).
template <class T>
__global__ void __launch_bounds__(256) lope_k_copy_through(const T* __restrict__ in, T* __restrict__ out,
                                                           DevLayout L, int b0, int e0, int b1, int e1,
                                                           int b2, int e2) {
  const long long nrows = L.P[1] * L.P[2];
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = warp; r < nrows; r += nw) {
    const int c1 = (int)(r % L.P[1]);
    const int c2 = (int)(r / L.P[1]);
    const long long base = L.B + c1 * L.S1 + c2 * L.S2;
    const bool inrow = c1 >= b1 && c1 < e1 && c2 >= b2 && c2 < e2;
    if (!inrow) {
      for (int x = lane; x < L.P[0]; x += 32) out[base + x] = in[base + x];
    } else {
      for (int x = lane; x < b0; x += 32) out[base + x] = in[base + x];
      for (int x = e0 + lane; x < L.P[0]; x += 32) out[base + x] = in[base + x];
    }
  }
}

// dst[box at dlo] := src[box at slo], boxes of extent e (padded coordinates, same layout).
template <class T>
__global__ void __launch_bounds__(256) lope_k_copy_box(T* __restrict__ dst, const T* __restrict__ src,
                                                       DevLayout L, long long d0, long long d1, long long d2,
                                                       long long s0, long long s1, long long s2, long long e0,
                                                       long long e1, long long e2) {
  const long long nrows = e1 * e2;
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = warp; r < nrows; r += nw) {
    const long long j = r % e1, k = r / e1;
    T* drow = dst + L.B + d0 + (d1 + j) * L.S1 + (d2 + k) * L.S2;
    const T* srow = src + L.B + s0 + (s1 + j) * L.S1 + (s2 + k) * L.S2;
    for (long long x = lane; x < e0; x += 32) drow[x] = srow[x];
  }
}

// Several boxes of one layout in one launch (blockIdx.y = box): the halo slabs of one
// exchange phase.  Rows at least half a warp wide are copied a warp per row (coalesced);
// thinner boxes (the x-halo columns) a thread per cell, so a 1-cell-wide slab of 4K rows
// does not leave 31 lanes of every warp idle.
#define LOPE_MAX_BOXES 32
template <class T>
struct LopeBoxes {
  T* dst[LOPE_MAX_BOXES];
  const T* src[LOPE_MAX_BOXES];
  long long d[LOPE_MAX_BOXES][3], s[LOPE_MAX_BOXES][3], e[LOPE_MAX_BOXES][3];
};
template <class T>
__global__ void __launch_bounds__(256) lope_k_copy_boxes(const __grid_constant__ LopeBoxes<T> bx, DevLayout L) {
  const int b = blockIdx.y;
  const long long e0 = bx.e[b][0], e1 = bx.e[b][1], e2 = bx.e[b][2];
  T* dst = bx.dst[b] + L.B + bx.d[b][0] + bx.d[b][1] * L.S1 + bx.d[b][2] * L.S2;
  const T* src = bx.src[b] + L.B + bx.s[b][0] + bx.s[b][1] * L.S1 + bx.s[b][2] * L.S2;
  const long long nrows = e1 * e2;
  if (e0 >= 16) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = warp; r < nrows; r += nw) {
      const long long j = r % e1, k = r / e1;
      const long long off = j * L.S1 + k * L.S2;
      for (long long x = lane; x < e0; x += 32) dst[off + x] = src[off + x];
    }
  } else {
    const long long n = nrows * e0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
      const long long x = i % e0, r = i / e0;
      const long long j = r % e1, k = r / e1;
      const long long off = j * L.S1 + k * L.S2 + x;
      dst[off] = src[off];
    }
  }
}

// Box <-> contiguous buffer (column-major within the box): the strided faces of a
// decomposed non-slowest dim travel between GPUs through such buffers.
template <class T, bool PACK>
__global__ void __launch_bounds__(256) lope_k_box_xfer(T* __restrict__ blk, T* __restrict__ buf, DevLayout L,
                                                       long long b0, long long b1, long long b2, long long e0,
                                                       long long e1, long long e2) {
  const long long nrows = e1 * e2;
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = warp; r < nrows; r += nw) {
    const long long j = r % e1, k = r / e1;
    T* brow = blk + L.B + b0 + (b1 + j) * L.S1 + (b2 + k) * L.S2;
    T* crow = buf + r * e0;
    for (long long x = lane; x < e0; x += 32) {
      if (PACK) crow[x] = brow[x];
      else brow[x] = crow[x];
    }
  }
}

__device__ __forceinline__ unsigned long long lope_splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

template <class T>
__global__ void __launch_bounds__(256) lope_k_fill_hash(T* __restrict__ buf, DevLayout L, unsigned long long seed,
                                                        long long G0, long long G1, long long o0, long long o1,
                                                        long long o2) {
  const long long n = (long long)L.m[0] * L.m[1] * L.m[2];
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t % L.m[0];
    const long long rr = t / L.m[0];
    const long long j = rr % L.m[1];
    const long long k = rr / L.m[1];
    const unsigned long long g = (unsigned long long)((o0 + i) + G0 * ((o1 + j) + G1 * (o2 + k)));
    const unsigned long long z = lope_splitmix64(g + seed * 0x9E3779B97F4A7C15ULL);
    const double v = (double)(z >> 11) * (1.0 / 9007199254740992.0);
    const double u = 2.0 * v - 1.0;
    buf[L.B + (i + L.lo[0]) + (j + L.lo[1]) * L.S1 + (k + L.lo[2]) * L.S2] = (T)u;
  }
}

// ---------------------------------------------------------------------------
// Compiled kernels

namespace {

struct TileCfg {
  int bxw = 4, wy = 2, ry = 8, ns = 8;
  int mb = 2;     // CTAs per SM the launch bounds target
  int pw = 0;     // 1: dedicated TMA producer warp
  int sh = 0;     // 1: x-halo columns through warp shuffles (fp32, one-column halos)
  int nb = 0;     // 1: in-band producer prefetches only into already-free slots
  int rag = 0;    // 1: ragged-x kernel (masked edge vectors, cell-by-cell x images)
};

struct DevMod {
  CUmodule mod = nullptr;
  CUfunction generic = nullptr;
  CUfunction row = nullptr;             // rank-1 vector kernel
  CUfunction tiled = nullptr;
  int tiled_smem = 0, tiled_threads = 0, boxx = 0, boxy = 0, tiled_blocks = 0;
  int tiled_local = 0;                  // local memory (spills) per thread of the tiled kernel
  CUfunction tiledm = nullptr;          // multi-array tiled kernel, variant 0 only
  int tm_smem = 0, tm_threads = 0, tm_boxx = 0, tm_boxy = 0, tm_blocks = 0, tm_by = 0;
  CUfunction tblock = nullptr;          // temporal blocking (rank 2), variant 0 only
  int tb_smem = 0, tb_tx = 0, tb_ty = 0, tb_tt = 0, tb_threads = 0;
};

// host mirrors of the device parameter structs (lope_device.cuh)
template <class T> struct HArr { const T* in; T* out; long long s1, s2, org; };
#define LOPE_HOST_MAX_SCAL 16   // == LOPE_MAX_SCAL in lope_device.cuh
template <class T> struct HScal { T v[LOPE_HOST_MAX_SCAL]; };
struct HGeom {
  int ext[3], m[3], r0[3], lo[3], hi[3];
  int wrap, zchunk, xshift, box0, p1, yband, xexact;
  long long sdl, sdh;
};

}  // namespace

// One compiled specialisation of a kernel (tile shape, ring depth, producer warp).
struct LopeVariant {
  TileCfg tile;
  bool tiled_ok = false;
  std::string source;
  std::vector<char> cubin;
  std::map<int, DevMod> mods;   // per device
};

// The execution plan for one geometry (lope_plan_set): the variant and the z-chunk.
struct LopePlan {
  int variant = 0;
  int zchunk = 0;
  int yband = 0;
  double ms = 0.0;
};

struct lope_kernel {
  lope::Kir ir;
  int dtype = LOPE_F32;
  std::vector<LopeVariant> variants;        // [0] = the default pick_tile() variant
  std::map<std::string, LopePlan> plans;    // geometry key -> tuned plan
  std::string describe_path;
  // launches per kernel family (describe "launches"): which path a geometry actually took
  mutable std::atomic<long long> n_tiled{0}, n_multi{0}, n_generic{0}, n_tblock{0}, n_row{0};
  // the default variant's fields, kept for describe/source
  const TileCfg& tile() const { return variants[0].tile; }
  bool tiled_ok() const { return variants[0].tiled_ok; }
};

namespace {

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ULL) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ULL;
  }
  return h;
}

bool read_file(const std::string& p, std::vector<char>* out) {
  std::ifstream f(p, std::ios::binary);
  if (!f) return false;
  out->assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
  return !out->empty();
}

void write_file_atomic(const std::string& p, const std::vector<char>& data) {
  std::string tmp = p + ".tmp." + std::to_string(getpid());
  {
    std::ofstream f(tmp, std::ios::binary);
    if (!f) return;
    f.write(data.data(), (std::streamsize)data.size());
  }
  std::rename(tmp.c_str(), p.c_str());
}

int tiled_smem_bytes(const lope::Kir& k, int dtype, const TileCfg& c) {
  // mirrors LopeTiledCfg (lope_device.cuh)
  int sz = dtype == LOPE_F32 ? 4 : 8;
  int vx = 16 / sz;
  int bx = 32 * vx * c.bxw, by = c.wy * c.ry;
  int padx = ((k.fn[0][0] + vx - 1) / vx) * vx;
  int padr = ((k.fp[0][0] + vx - 1) / vx) * vx;
  // one TMA box per warp column when a single box would exceed 256 elements
  const int nb = (padx + bx + padr > 256) ? c.bxw : 1;
  int boxx = padx + bx / nb + padr;
  int boxy = by + k.fn[0][1] + k.fp[0][1];
  int stage = nb * (((boxx * boxy * sz + 127) / 128) * 128);
  if (boxx > 256 || boxy > 256) return 1 << 30;
  return c.ns * stage + 2 * c.ns * 8;
}

TileCfg pick_tile(const lope::Kir& k, int dtype) {
  // One CTA per SM: 16 compute warps stacked in y (plus a TMA producer warp for 2-D).
  // Lanes hold 16-byte vectors (4 fp32 / 2 fp64), so a tile is one warp (128 fp32 / 64
  // fp64 columns) wide and the TMA box stays within 256 elements.  Calibrated on B200
  // (tools/probe_perf.py): 2 rows/lane (32-row tiles, 18.5 KB stages); 2-D fills the
  // ring (12 stages), 3-D runs best with 8 (lap3d7 1024^3: 1.62 ms vs 1.67 ms at 12).
  TileCfg c;
  const int nzw = k.fn[0][2] + k.fp[0][2] + 1;
  bool zstar = k.rank == 3;
  for (const lope::Node& n : k.nodes)
    if (n.kind == lope::Node::READ && n.arr == 0 && n.off[2] != 0 && (n.off[0] != 0 || n.off[1] != 0)) zstar = false;
  const int hold = (zstar && k.fn[0][2] > 0) ? k.fp[0][2] + 1 : nzw;
  c.bxw = 1;
  c.wy = 16;
  c.ry = 2;
  c.mb = 1;
  c.ns = 32;
  // producer: in-band (warp 0 lane 0) for 3-D, a dedicated 17th warp for 2-D
  // (measured on B200: lap3d7 1024^3 1.76 vs 1.98 ms; ninept2d 16384^2 0.35 vs 0.49 ms).
  // This is the untuned default; the plan tuner may pick a dedicated producer with
  // short z-chunks for 3-D (tune_candidates).
  c.pw = k.rank == 3 ? 0 : 1;
  if (dtype == LOPE_F64) {
    // fp64 lanes hold 2 values: two warps side by side keep the TMA box 128+ columns
    // wide (fewer partial lines); lap3d7 fp64 1024^2x512: 1.57 ms = 5.5 TB/s.  The 5x5
    // box (24 dependent adds per point) prefers 4 rows per lane in one warp column:
    // more independent chains per lane.
    c.bxw = 2; c.wy = 8; c.ry = 2; c.pw = 0;
    const int wide = (k.fn[0][0] + k.fp[0][0] + 2) * (c.ry + k.fn[0][1] + k.fp[0][1]) * 2;
    if (wide > 64) { c.bxw = 1; c.wy = 16; c.ry = 4; }
  }
  // Keep the per-lane register window (rows x columns of the centre plane, in 32-bit
  // registers) small enough that nothing spills.  Spills are not just slow here: the
  // local-memory traffic goes through L2 and evicts the halo lines neighbouring tiles
  // would otherwise reuse.
  {
    const int vx = dtype == LOPE_F32 ? 4 : 2;
    const int words = dtype == LOPE_F32 ? 1 : 2;
    auto window = [&](int ry) {
      return (ry + k.fn[0][1] + k.fp[0][1]) * (vx + k.fn[0][0] + k.fp[0][0]) * words;
    };
    if (dtype == LOPE_F32)
      while (c.ry > 1 && window(c.ry) > 64) c.ry /= 2;
  }
  if (k.rank == 3 && dtype == LOPE_F32) c.ns = 8;
  if (const char* e = std::getenv("LOPE_TILE")) {
    int a, b, cc, d;
    if (std::sscanf(e, "%d,%d,%d,%d", &a, &b, &cc, &d) == 4) {
      c.bxw = a; c.wy = b; c.ry = cc; c.ns = d;
    }
  }
  if (const char* e = std::getenv("LOPE_MB")) c.mb = std::atoi(e) == 2 ? 2 : 1;
  if (const char* e = std::getenv("LOPE_PW")) c.pw = std::atoi(e) ? 1 : 0;
  if (const char* e = std::getenv("LOPE_SHFL")) c.sh = std::atoi(e) ? 1 : 0;
  if (const char* e = std::getenv("LOPE_NB")) c.nb = std::atoi(e) ? 1 : 0;
  if (c.ns < hold + 1) c.ns = hold + 1;
  // shrink the ring until mb CTAs fit on an SM (227 KB)
  while (c.ns > hold + 1 && c.mb * tiled_smem_bytes(k, dtype, c) > 225 * 1024) --c.ns;
  return c;
}

std::string build_source(const lope_kernel* K, const LopeVariant& V, bool with_tblock) {
  const lope::Kir& k = K->ir;
  std::ostringstream s;
  s << kDeviceSrc << "\n";
  s << lope::emit_body(k) << "\n";
  const char* T = K->dtype == LOPE_F32 ? "float" : "double";
  s << "typedef " << T << " LT;\n";
  s << "struct LopeArrPack { LopeArr<LT> a[" << k.arrays.size() << "]; };\n";
  s << "extern \"C\" __global__ void __launch_bounds__(128) lope_generic("
       "const __grid_constant__ LopeArrPack pack, const LopeScal<LT> sc, const LopeGeom g) {\n"
       "  lope_generic_impl<LopeBody, LT>(pack.a, sc, g);\n"
       "  if (g.sdl | g.sdh) __threadfence_system();   // peer-block images visible system-wide\n}\n";
  if (k.rank == 1) {
    s << "extern \"C\" __global__ void __launch_bounds__(256) lope_row("
         "const __grid_constant__ LopeArrPack pack, const LopeScal<LT> sc, const LopeGeom g) {\n"
         "  lope_row_impl<LopeBody, LT, " << k.arrays.size() << ">(pack.a, sc, g);\n"
         "  if (g.sdl | g.sdh) __threadfence_system();\n}\n";
  }
  if (V.tiled_ok) {
    const TileCfg& c = V.tile;
    s << "typedef LopeTiledCfg<LopeBody, LT, " << c.bxw << ", " << c.wy << ", " << c.ry << ", " << c.ns
      << ", " << c.pw << "> LopeCfg;\n";
    s << "extern \"C\" __constant__ int lope_tiled_info[4] = {LopeCfg::SMEM_BYTES, LopeCfg::THREADS, "
         "LopeCfg::BOXX, LopeCfg::BOXY};\n";
    s << "extern \"C\" __global__ void __launch_bounds__(" << 32 * (c.bxw * c.wy + c.pw)
      << ", " << c.mb << ") lope_tiled(const __grid_constant__ LopeTmap map, const LopeArr<LT> a, "
         "const LopeScal<LT> sc, const LopeGeom g) {\n"
      << "  lope_tiled_impl<LopeBody, LT, " << c.bxw << ", " << c.wy << ", " << c.ry << ", " << c.ns
      << ", " << c.pw << ", " << c.sh << ", " << c.nb << ", " << (c.rag ? "true" : "false") << ">(&map, a, sc, g);\n"
      << "  if (g.sdl | g.sdh) __threadfence_system();   // peer-block images visible system-wide\n}\n";
  }
  if (with_tblock && k.rank >= 2 && k.arrays.size() >= 2 && k.arrays.size() <= 4) {
    // several arrays: one TMA box per array per plane (lope_tiled_multi_impl); ring as
    // deep as fits next to NA boxes per stage
    const int na = (int)k.arrays.size();
    // a dedicated TMA producer warp (measured: two-array 3-D kernel 1024^3 2.19 ms with 16
    // compute warps, 2.46 with 15, 3.17 in-band).  17 warps cap registers at 96: the 2-D
    // window (two rows per lane) spills there, so 2-D runs 15 compute warps (128 registers)
    int mpw = 1;
    if (const char* e = std::getenv("LOPE_MULTI_PW")) mpw = std::atoi(e) ? 1 : 0;
    int wym = 16;
    const int sz = K->dtype == LOPE_F32 ? 4 : 8, vx = 16 / sz;
    int un0 = 0, up0 = 0, un1 = 0, up1 = 0, un2 = 0, up2 = 0;
    for (int a = 0; a < na; ++a) {
      un0 = std::max(un0, k.fn[a][0]); up0 = std::max(up0, k.fp[a][0]);
      un1 = std::max(un1, k.fn[a][1]); up1 = std::max(up1, k.fp[a][1]);
      un2 = std::max(un2, k.fn[a][2]); up2 = std::max(up2, k.fp[a][2]);
    }
    // emits lope_tiled_multi<suffix> with `ry` rows per lane; get_mod takes the first
    // one that neither spills nor fails to fit
    auto emit = [&](const char* suffix, int ry, int wym) {
      auto fits = [&](int n) {
        const int boxx = ((un0 + vx - 1) / vx) * vx + 32 * vx + ((up0 + vx - 1) / vx) * vx;
        const int boxy = wym * ry + un1 + up1;
        if (boxx > 256 || boxy > 256) return false;
        const int box = ((boxx * boxy * sz + 127) / 128) * 128;
        return n >= un2 + up2 + 2 && n * na * box + 16 * n <= 225 * 1024;
      };
      int ns = 12;
      while (ns > 2 && !fits(ns)) --ns;
      if (!fits(ns)) return;
      s << "typedef LopeTiledMCfg<LopeBody, LT, 1, " << wym << ", " << ry << ", " << ns << ", " << mpw
        << "> LopeMCfg" << suffix << ";\n";
      s << "extern \"C\" __constant__ int lope_tiledm" << suffix << "_info[5] = {LopeMCfg" << suffix
        << "::SMEM_BYTES, LopeMCfg" << suffix << "::THREADS, LopeMCfg" << suffix << "::BOXX, LopeMCfg" << suffix
        << "::BOXY, LopeMCfg" << suffix << "::BY};\n";
      s << "extern \"C\" __global__ void __launch_bounds__(LopeMCfg" << suffix << "::THREADS, 1) lope_tiled_multi"
        << suffix << "(const __grid_constant__ LopeTmapPack<" << na
        << "> maps, const __grid_constant__ LopeArrPackT<LT, " << na
        << "> arrs, const LopeScal<LT> sc, const LopeGeom g) {\n"
        << "  lope_tiled_multi_impl<LopeBody, LT, 1, " << wym << ", " << ry << ", " << ns << ", " << mpw
        << ">(&maps, arrs, sc, g);\n}\n";
    };
    const int ry = k.rank == 3 ? 1 : 2;
    const int wy0 = (mpw && k.rank == 2) ? 15 : 16;
    emit("", ry, wy0);
    // the register window (arrays x planes x rows x columns) may spill: one row per lane
    // and 15 + 1 warps (128 registers) as the alternative get_mod falls back to
    if (ry > 1 || (mpw && wy0 == 16)) emit("_r1", 1, mpw ? 15 : 16);
  }
  if (with_tblock && k.rank == 2 && k.arrays.size() == 1 && k.fn[0][0] <= 4 && k.fp[0][0] <= 4) {
    // 256 x 28 fp32 tiles: 1024^2 splits into 4 x 37 = 148 CTAs, one per SM (config 1);
    // 8 steps per launch for one-cell footprints, 4 for wider ones (the recomputed
    // halo grows with the footprint)
    const int tx = K->dtype == LOPE_F32 ? 256 : 128;
    const int wmax = std::max(k.fn[0][0] + k.fp[0][0], k.fn[0][1] + k.fp[0][1]);
    int ty = 28, tt = wmax <= 2 ? 8 : 4;
    if (const char* e = std::getenv("LOPE_TBLOCK_TY")) ty = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("LOPE_TBLOCK_TT")) tt = std::max(1, std::atoi(e));
    const int vx = K->dtype == LOPE_F32 ? 4 : 2;
    if ((tt * k.fn[0][0]) % vx == 0) {
      s << "typedef LopeTblockCfg<LopeBody, LT, " << tx << ", " << ty << ", " << tt << "> LopeTbCfg;\n";
      s << "extern \"C\" __constant__ int lope_tblock_info[5] = {LopeTbCfg::SMEM_BYTES, " << tx << ", " << ty
        << ", " << tt << ", LopeTbCfg::THREADS};\n";
      s << "extern \"C\" __global__ void __launch_bounds__(LopeTbCfg::THREADS) lope_tblock(const LopeArr<LT> a, "
           "const LopeScal<LT> sc, const LopeGeom g) {\n"
        << "  lope_tblock_impl<LopeBody, LT, " << tx << ", " << ty << ", " << tt << ">(a, sc, g);\n}\n";
    }
  }
  return s.str();
}

int nvrtc_compile(const std::string& src, const std::string& name, std::vector<char>* cubin) {
  std::vector<std::string> opts = {"--gpu-architecture=sm_100a", "-std=c++17", "-fmad=false",
                                   "-prec-div=true", "-prec-sqrt=true", "-ftz=false", "-lineinfo",
                                   "-DNDEBUG"};
  // experiment hook: extra -D flags for the device templates (part of the cache key)
  if (const char* e = std::getenv("LOPE_NVRTC_DEFS")) {
    std::istringstream is(e);
    std::string d;
    while (is >> d)
      if (d.rfind("-D", 0) == 0) opts.push_back(d);
  }
  int ver_major = 0, ver_minor = 0;
  nvrtcVersion(&ver_major, &ver_minor);
  std::string key = src;
  for (auto& o : opts) key += "\n" + o;
  key += "\nnvrtc " + std::to_string(ver_major) + "." + std::to_string(ver_minor);
  char hbuf[32];
  std::snprintf(hbuf, sizeof hbuf, "%016llx", (unsigned long long)fnv1a(key));
  std::string dir;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    dir = g_cache_dir;
  }
  if (dir.empty()) {
    if (const char* e = std::getenv("LOPE_CACHE_DIR")) dir = e;
  }
  std::string path;
  if (!dir.empty()) {
    path = dir + "/" + name + "-" + hbuf + ".cubin";
    if (read_file(path, cubin)) return 0;
  }
  nvrtcProgram prog;
  nvrtcResult r = nvrtcCreateProgram(&prog, src.c_str(), (name + ".cu").c_str(), 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return fail(-2000 - (int)r, "nvrtcCreateProgram: %s", nvrtcGetErrorString(r));
  std::vector<const char*> copts;
  for (auto& o : opts) copts.push_back(o.c_str());
  r = nvrtcCompileProgram(prog, (int)copts.size(), copts.data());
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    if (log.size() > 1800) log = log.substr(0, 1800);
    return fail(-2000 - (int)r, "NVRTC compile of kernel '%s' failed: %s", name.c_str(), log.c_str());
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin->resize(n);
  nvrtcGetCUBIN(prog, cubin->data());
  nvrtcDestroyProgram(&prog);
  if (!path.empty()) {
    mkdir(dir.c_str(), 0755);
    write_file_atomic(path, *cubin);
  }
  return 0;
}

int get_mod(lope_kernel* K, int vi, DevMod** out) {
  LopeVariant& V = K->variants[vi];
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  auto it = V.mods.find(dev);
  if (it != V.mods.end()) {
    *out = &it->second;
    return 0;
  }
  Drv& d = drv();
  if (!d.ok) return fail(-3, "CUDA driver API unavailable: %s", d.why.c_str());
  CUDA_TRY(cudaFree(nullptr));   // make the primary context current on this thread
  DevMod m;
  CUresult r = d.moduleLoadData(&m.mod, V.cubin.data());
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuModuleLoadData");
  r = d.moduleGetFunction(&m.generic, m.mod, "lope_generic");
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuModuleGetFunction(lope_generic)");
  if (K->ir.rank == 1) {
    r = d.moduleGetFunction(&m.row, m.mod, "lope_row");
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuModuleGetFunction(lope_row)");
  }
  if (V.tiled_ok) {
    r = d.moduleGetFunction(&m.tiled, m.mod, "lope_tiled");
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuModuleGetFunction(lope_tiled)");
    CUdeviceptr gp;
    size_t gsz;
    r = d.moduleGetGlobal(&gp, &gsz, m.mod, "lope_tiled_info");
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuModuleGetGlobal(lope_tiled_info)");
    int info[4];
    CUDA_TRY(cudaMemcpy(info, (const void*)gp, sizeof info, cudaMemcpyDeviceToHost));
    m.tiled_smem = info[0];
    m.tiled_threads = info[1];
    m.boxx = info[2];
    m.boxy = info[3];
    r = d.funcSetAttribute(m.tiled, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, m.tiled_smem);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuFuncSetAttribute(max dynamic smem)");
    int nb = 0;
    r = d.occupancy(&nb, m.tiled, m.tiled_threads, m.tiled_smem);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuOccupancyMaxActiveBlocksPerMultiprocessor");
    if (nb < 1) return fail(-4, "tiled kernel cannot be resident (smem %d B)", m.tiled_smem);
    m.tiled_blocks = nb;
    int lb = 0;
    if (d.funcGetAttribute(&lb, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, m.tiled) == CUDA_SUCCESS) m.tiled_local = lb;
  }
  m.tiledm = nullptr;
  for (const char* suffix : {"", "_r1"}) {
    if (m.tiledm) break;
    const std::string fname = std::string("lope_tiled_multi") + suffix;
    const std::string iname = std::string("lope_tiledm") + suffix + "_info";
    if (d.moduleGetFunction(&m.tiledm, m.mod, fname.c_str()) != CUDA_SUCCESS) {
      m.tiledm = nullptr;
      continue;
    }
    CUdeviceptr gp;
    size_t gsz;
    r = d.moduleGetGlobal(&gp, &gsz, m.mod, iname.c_str());
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuModuleGetGlobal(lope_tiledm_info)");
    int info[5];
    CUDA_TRY(cudaMemcpy(info, (const void*)gp, sizeof info, cudaMemcpyDeviceToHost));
    m.tm_smem = info[0];
    m.tm_threads = info[1];
    m.tm_boxx = info[2];
    m.tm_boxy = info[3];
    m.tm_by = info[4];
    int nb = 0;
    if (d.funcSetAttribute(m.tiledm, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, m.tm_smem) != CUDA_SUCCESS ||
        d.occupancy(&nb, m.tiledm, m.tm_threads, m.tm_smem) != CUDA_SUCCESS || nb < 1)
      m.tiledm = nullptr;
    // a register window that spills (wide footprints x 4 arrays) sends local memory
    // through L2: such kernels run on the generic path instead
    int lb = 0;
    if (m.tiledm && d.funcGetAttribute(&lb, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, m.tiledm) == CUDA_SUCCESS &&
        lb > 0 && !std::getenv("LOPE_MULTI_ALLOW_SPILL"))
      m.tiledm = nullptr;
    m.tm_blocks = nb;
  }
  if (d.moduleGetFunction(&m.tblock, m.mod, "lope_tblock") == CUDA_SUCCESS) {
    CUdeviceptr gp;
    size_t gsz;
    r = d.moduleGetGlobal(&gp, &gsz, m.mod, "lope_tblock_info");
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuModuleGetGlobal(lope_tblock_info)");
    int info[5];
    CUDA_TRY(cudaMemcpy(info, (const void*)gp, sizeof info, cudaMemcpyDeviceToHost));
    m.tb_smem = info[0];
    m.tb_tx = info[1];
    m.tb_ty = info[2];
    m.tb_tt = info[3];
    m.tb_threads = info[4];
    r = d.funcSetAttribute(m.tblock, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, m.tb_smem);
    if (r != CUDA_SUCCESS) m.tblock = nullptr;
  } else {
    m.tblock = nullptr;
  }
  V.mods[dev] = m;
  *out = &V.mods[dev];
  return 0;
}

// Compile (or fetch from the cubin cache) one specialisation; returns its index in *vi.
int add_variant(lope_kernel* K, const TileCfg& cfg, int* vi = nullptr) {
  for (size_t i = 0; i < K->variants.size(); ++i) {
    const TileCfg& c = K->variants[i].tile;
    if (c.bxw == cfg.bxw && c.wy == cfg.wy && c.ry == cfg.ry && c.ns == cfg.ns && c.mb == cfg.mb && c.pw == cfg.pw &&
        c.sh == cfg.sh && c.nb == cfg.nb && c.rag == cfg.rag) {
      if (vi) *vi = (int)i;
      return 0;
    }
  }
  LopeVariant V;
  V.tile = cfg;
  V.tiled_ok = K->ir.rank >= 2 && K->ir.arrays.size() == 1 && tiled_smem_bytes(K->ir, K->dtype, cfg) <= 225 * 1024;
  V.source = build_source(K, V, K->variants.empty());
  if (int e = nvrtc_compile(V.source, "lope_" + K->ir.name, &V.cubin)) return e;
  K->variants.push_back(std::move(V));
  if (vi) *vi = (int)K->variants.size() - 1;
  return 0;
}

int check_layout(const lope_layout* L) {
  if (!L) return fail(108, "null layout");
  if (L->rank < 1 || L->rank > 3) return fail(108, "layout rank %d outside 1..3", L->rank);
  if (L->dtype != LOPE_F32 && L->dtype != LOPE_F64) return fail(108, "unknown dtype %d", L->dtype);
  return 0;
}

template <class T>
HScal<T> make_scal(const lope::Kir& k, const double* rs, const int64_t* is) {
  HScal<T> s;
  std::memset(&s, 0, sizeof s);
  for (size_t i = 0; i < k.scalars.size(); ++i) {
    if (k.scalar_is_int[i]) s.v[i] = is ? (T)is[i] : (T)0;
    else s.v[i] = rs ? (T)rs[i] : (T)0;
  }
  // reciprocals for LopeAr::divs (scalar divisors): RN(1/b) in T when |b| lies in the
  // range where the FMA-corrected quotient is exact, NaN (-> exact division) otherwise
  const size_t n = k.scalars.size();
  if (2 * n <= (size_t)LOPE_HOST_MAX_SCAL) {
    const double lo = sizeof(T) == 4 ? 0x1p-16 : 0x1p-60, hi = sizeof(T) == 4 ? 0x1p+16 : 0x1p+60;
    for (size_t i = 0; i < n; ++i) {
      const T b = s.v[i];
      const double ab = std::fabs((double)b);
      s.v[n + i] = (std::isfinite((double)b) && ab >= lo && ab <= hi) ? (T)(T(1) / b)
                                                                       : std::numeric_limits<T>::quiet_NaN();
    }
  }
  return s;
}

CUtensorMapL2promotion l2promo() {
  static int v = -1;
  if (v < 0) {
    v = 2;   // 128-byte promotion: measured ~5% fewer HBM bytes than 256 B for the stencil boxes
    if (const char* e = std::getenv("LOPE_L2PROMO")) v = std::atoi(e) & 3;
  }
  switch (v) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    v = 1;
    if (const char* e = std::getenv("LOPE_PDL")) v = std::atoi(e) != 0;
  }
  return v;
}

bool tmap_flat() {
  static int v = -1;
  if (v < 0) {
    v = 0;
    if (const char* e = std::getenv("LOPE_TMAP2D")) v = std::atoi(e) != 0;
  }
  return v;
}

int encode_tmap_box(const lope_layout* L, const void* base, int boxx, int boxy, CUtensorMap* map);

int encode_tmap(const lope_layout* L, const void* base, const DevMod& m, CUtensorMap* map) {
  return encode_tmap_box(L, base, m.boxx, m.boxy, map);
}

int encode_tmap_box(const lope_layout* L, const void* base, int boxx, int boxy, CUtensorMap* map) {
  if (tmap_flat()) {
    // planes stacked as rows: one 2-D map over padded1*padded2 rows
    cuuint64_t dims2[2] = {(cuuint64_t)L->stride[1], (cuuint64_t)(L->padded[1] * L->padded[2])};
    cuuint64_t strides2[1] = {(cuuint64_t)(L->stride[1] * L->elem_bytes)};
    cuuint32_t box2[2] = {(cuuint32_t)boxx, (cuuint32_t)boxy};
    cuuint32_t estr2[2] = {1, 1};
    CUresult r2 = drv().tensorMapEncodeTiled(
        map, L->dtype == LOPE_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
        const_cast<void*>(base), dims2, strides2, box2, estr2, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, l2promo(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r2 != CUDA_SUCCESS) return cu_fail(r2, "cuTensorMapEncodeTiled(2d)");
    return 0;
  }
  cuuint64_t dims[3] = {(cuuint64_t)L->stride[1], (cuuint64_t)L->padded[1], (cuuint64_t)L->padded[2]};
  cuuint64_t strides[2] = {(cuuint64_t)(L->stride[1] * L->elem_bytes), (cuuint64_t)(L->stride[2] * L->elem_bytes)};
  cuuint32_t box[3] = {(cuuint32_t)boxx, (cuuint32_t)boxy, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = drv().tensorMapEncodeTiled(
      map, L->dtype == LOPE_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
      const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, l2promo(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuTensorMapEncodeTiled");
  return 0;
}

int zchunk_default(const lope::Kir& k) {
  if (k.rank < 2) return 1;
  if (k.rank == 2) {
    // y tiles per unit (the tiled kernel streams rank-2 units along y)
    if (const char* e = std::getenv("LOPE_YCHUNK")) {
      int v = std::atoi(e);
      if (v > 0) return v;
    }
    return 8;
  }
  if (const char* e = std::getenv("LOPE_ZCHUNK")) {
    int v = std::atoi(e);
    if (v > 0) return v;
  }
  return 64;   // z-halo planes re-read once per 64 planes (3%), balance within ~4%
}

// Launch the body kernel over `ranges` (0-based start r0, extents ext) of array set.
// Launch with programmatic dependent launch when available (see run_body).
CUresult launch_ex(CUfunction f, unsigned grid, unsigned block, int smem, cudaStream_t st, void** args) {
  Drv& d = drv();
  if (d.launchKernelEx && pdl_enabled()) {
    CUlaunchAttribute at[1];
    std::memset(at, 0, sizeof at);
    at[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    at[0].value.programmaticStreamSerializationAllowed = 1;
    CUlaunchConfig cfg;
    std::memset(&cfg, 0, sizeof cfg);
    cfg.gridDimX = grid; cfg.gridDimY = 1; cfg.gridDimZ = 1;
    cfg.blockDimX = block; cfg.blockDimY = 1; cfg.blockDimZ = 1;
    cfg.sharedMemBytes = (unsigned)smem;
    cfg.hStream = (CUstream)st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return d.launchKernelEx(&cfg, f, args, nullptr);
  }
  return d.launchKernel(f, grid, 1, 1, block, 1, 1, (unsigned)smem, (CUstream)st, args, nullptr);
}

std::string plan_key(const lope_layout* L, int wrap) {
  char b[256];
  std::snprintf(b, sizeof b, "%d:%lld,%lld,%lld:%d,%d,%d:%d,%d,%d:%d", L->rank, (long long)L->interior[0],
                (long long)L->interior[1], (long long)L->interior[2], L->lo[0], L->lo[1], L->lo[2], L->hi[0],
                L->hi[1], L->hi[2], wrap);
  return b;
}

// vi / zc: the variant and z-chunk to use; vi < 0 picks the tuned plan for this
// geometry, or the defaults when it was never tuned.
template <class T>
int run_body(lope_kernel* K, const lope_layout* layouts, const int r0[3], const int ext[3],
             const void* const* in, void* const* out, const double* rs, const int64_t* is, int wrap,
             cudaStream_t st, int vi = -1, int zc = 0, int yband = 0, long long sdl = 0, long long sdh = 0) {
  if (vi < 0) {
    vi = 0;
    if (!K->plans.empty()) {
      auto it = K->plans.find(plan_key(&layouts[0], wrap));
      if (it != K->plans.end()) {
        vi = it->second.variant;
        zc = it->second.zchunk;
        yband = it->second.yband;
      }
    }
  }
  {
    // Ragged x (a range start or extent that is not whole 16-byte vectors, or an
    // interior too narrow / not whole vectors for whole-atom x images): the RAG
    // instantiation of the same tile (masked edge vectors, cell-by-cell x images),
    // compiled on first use.  The aligned instantiation carries none of that code.
    const int vxr = 16 / (int)sizeof(T);
    bool rag = (r0[0] % vxr) != 0 || (ext[0] % vxr) != 0;
    if (wrap & 1) {
      const long long line = 64 / (long long)sizeof(T);
      rag = rag || !(layouts[0].interior[0] % vxr == 0 && layouts[0].interior[0] >= 2 * line);
    }
    if (rag && K->variants[vi].tiled_ok && K->ir.arrays.size() == 1 && !K->variants[vi].tile.rag) {
      TileCfg t = K->variants[vi].tile;
      t.rag = 1;
      if (int e = add_variant(K, t, &vi)) return e;
    }
  }
  const LopeVariant& V = K->variants[vi];
  DevMod* m = nullptr;
  if (int e = get_mod(K, vi, &m)) return e;
  const lope::Kir& k = K->ir;
  HScal<T> sc = make_scal<T>(k, rs, is);
  HGeom g;
  std::memset(&g, 0, sizeof g);
  for (int d = 0; d < 3; ++d) {
    g.ext[d] = ext[d];
    g.m[d] = (int)layouts[0].interior[d];
    g.r0[d] = r0[d];
    g.lo[d] = layouts[0].lo[d];
    g.hi[d] = layouts[0].hi[d];
  }
  g.wrap = wrap;
  g.zchunk = zc > 0 ? zc : zchunk_default(k);
  g.yband = yband;
  g.sdl = sdl;
  g.sdh = sdh;
  if (const char* e = std::getenv("LOPE_YBAND")) g.yband = std::atoi(e);
  const int vx = 16 / (int)sizeof(T);
  // The tiled kernels run x from the range start rounded down to a whole 16-byte
  // vector (interior rows start 64-byte aligned, lope_layout_init): the xsh cells in
  // front of the range and the ragged end are masked in the stores.
  const int xsh = r0[0] % vx;
  const int r0x = r0[0] - xsh;
  g.p1 = tmap_flat() ? (int)layouts[0].padded[1] : 0;
  Drv& d = drv();
  // When the launch refreshes halo images every halo cell must have exactly one image
  // (interior at least lo+hi wide in every wrapped dim).  x images are
  // whole 64-byte atoms when the interior is a whole number of vectors and at least
  // two atoms wide, else cell by cell; other geometries run on the generic kernel.
  bool geom_ok = true;
  if (wrap) {
    const lope_layout& L0 = layouts[0];
    const long long line = 64 / (long long)sizeof(T);
    g.xexact = (wrap & 1) && !(L0.interior[0] % vx == 0 && L0.interior[0] >= 2 * line);
    for (int d = 0; d < 3; ++d)
      if ((wrap >> d) & 1) geom_ok = geom_ok && L0.interior[d] >= L0.lo[d] + L0.hi[d];
  }
  if (geom_ok) {
    // shift the x range for the tiled kernels (restored below for the generic kernel)
    g.r0[0] = r0x;
    g.ext[0] = ext[0] + xsh;
    g.xshift = xsh;
  }
  const bool use_tiled = V.tiled_ok && k.arrays.size() == 1 && geom_ok &&
                         !std::getenv("LOPE_FORCE_GENERIC");
  if (use_tiled) {
    g.box0 = (int)(layouts[0].base + layouts[0].lo[0] + r0x - ((k.fn[0][0] + vx - 1) / vx) * vx);
    const lope_layout* L = &layouts[0];
    CUtensorMap map;
    if (int e = encode_tmap(L, in[0], *m, &map)) return e;
    HArr<T> a;
    a.in = (const T*)in[0];
    a.out = (T*)out[0];
    a.s1 = L->stride[1];
    a.s2 = L->stride[2];
    a.org = L->base + (L->lo[0] + r0x) + (long long)(L->lo[1] + r0[1]) * L->stride[1] +
            (long long)(L->lo[2] + r0[2]) * L->stride[2];
    const TileCfg& c = V.tile;
    long long ntx = (g.ext[0] + 32 * vx * c.bxw - 1) / (32 * vx * c.bxw);
    long long nty = (ext[1] + c.wy * c.ry - 1) / (c.wy * c.ry);
    long long nzc = (ext[2] + g.zchunk - 1) / g.zchunk;
    if (k.rank == 2) {
      // rank 2 streams units along y: `zchunk` y tiles per unit (lope_tiled_impl, YS);
      // small fields keep at least two units per resident CTA (1024^2 has only 256
      // tiles: 8-tile units would leave most SMs idle)
      const long long cap = 2LL * m->tiled_blocks * sm_count();
      while (g.zchunk > 1 && ntx * ((nty + g.zchunk - 1) / g.zchunk) < cap) g.zchunk = (g.zchunk + 1) / 2;
      nty = (nty + g.zchunk - 1) / g.zchunk;
      nzc = 1;
    }
    long long units = ntx * nty * nzc;
    if (units >= (1LL << 31)) return fail(108, "launch range too large for the tiled path");
    long long grid = (long long)m->tiled_blocks * sm_count();
    // Units are walked x-fastest with stride `grid`, so CTA b visits the x tiles
    // (b + k*grid) mod ntx.  A grid sharing a factor with ntx*nty pins every CTA to a
    // few tile columns/rows: the edge tiles (halo-image stores, padding reads) then
    // slow the same CTAs every round, neighbours drift apart and their shared halo
    // lines fall out of L2 (measured: grid 148 vs 147 on 1024^3 = 1.76 vs 1.67 ms,
    // on 2048^3 16.6 vs 13.2 ms).  Take the largest grid coprime with ntx*nty.
    {
      long long period = ntx * nty;
      long long best = grid;
      for (long long gg = grid; gg > 1 && gg > grid - 32; --gg) {
        long long a0 = gg, b0 = period;
        while (b0) { long long t = a0 % b0; a0 = b0; b0 = t; }
        if (a0 == 1) { best = gg; break; }
      }
      grid = best;
    }
    if (const char* e = std::getenv("LOPE_GRID")) grid = std::atoll(e);
    if (grid > units) grid = units;
    if (grid < 1) grid = 1;
    void* args[] = {&map, &a, &sc, &g};
    CUresult r;
    if (d.launchKernelEx && pdl_enabled()) {
      // Programmatic dependent launch: this grid's CTAs may be dispatched while the
      // previous kernel in the stream drains (barrier init and descriptor prefetch
      // overlap its tail); the kernel executes griddepcontrol.wait before touching
      // global memory, so stream order is preserved for the data.
      CUlaunchAttribute at[1];
      std::memset(at, 0, sizeof at);
      at[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
      at[0].value.programmaticStreamSerializationAllowed = 1;
      CUlaunchConfig cfg;
      std::memset(&cfg, 0, sizeof cfg);
      cfg.gridDimX = (unsigned)grid; cfg.gridDimY = 1; cfg.gridDimZ = 1;
      cfg.blockDimX = m->tiled_threads; cfg.blockDimY = 1; cfg.blockDimZ = 1;
      cfg.sharedMemBytes = m->tiled_smem;
      cfg.hStream = (CUstream)st;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      r = d.launchKernelEx(&cfg, m->tiled, args, nullptr);
    } else {
      r = d.launchKernel(m->tiled, (unsigned)grid, 1, 1, m->tiled_threads, 1, 1, m->tiled_smem,
                         (CUstream)st, args, nullptr);
    }
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuLaunchKernel(lope_tiled)");
    g_launches++;
    K->n_tiled++;
    return 0;
  }
  // several arrays with one layout: the multi-array tiled kernel
  const int na = (int)k.arrays.size();
  bool same = na >= 2 && na <= 4 && m->tiledm && geom_ok && !std::getenv("LOPE_FORCE_GENERIC");
  for (int a = 1; same && a < na; ++a) {
    const lope_layout& A = layouts[a];
    const lope_layout& B = layouts[0];
    for (int d = 0; d < 3; ++d)
      same = same && A.interior[d] == B.interior[d] && A.lo[d] == B.lo[d] && A.hi[d] == B.hi[d] &&
             A.stride[d] == B.stride[d];
    same = same && A.base == B.base && A.rank == B.rank;
  }
  for (int a = 0; same && a < na; ++a) same = in[a] != nullptr;
  for (size_t q = 0; same && q < k.stored.size(); ++q) same = out && out[k.stored[q]] != nullptr;
  if (same) {
    const lope_layout* L = &layouts[0];
    std::vector<CUtensorMap> maps(na);
    for (int a = 0; a < na; ++a)
      if (int e = encode_tmap_box(L, in[a], m->tm_boxx, m->tm_boxy, &maps[a])) return e;
    std::vector<HArr<T>> pk(na);
    int un0 = 0;
    for (int a = 0; a < na; ++a) {
      pk[a].in = (const T*)in[a];
      pk[a].out = out ? (T*)out[a] : nullptr;
      pk[a].s1 = L->stride[1];
      pk[a].s2 = L->stride[2];
      pk[a].org = L->base + (L->lo[0] + r0x) + (long long)(L->lo[1] + r0[1]) * L->stride[1] +
                  (long long)(L->lo[2] + r0[2]) * L->stride[2];
      un0 = std::max(un0, k.fn[a][0]);
    }
    const int padx = ((un0 + vx - 1) / vx) * vx;
    g.box0 = (int)(L->base + L->lo[0] + r0x - padx);
    long long ntx = (g.ext[0] + 32 * vx - 1) / (32 * vx);
    long long nty = (ext[1] + m->tm_by - 1) / m->tm_by;
    long long nzc = (ext[2] + g.zchunk - 1) / g.zchunk;
    long long units = ntx * nty * nzc;
    if (units >= (1LL << 31)) return fail(108, "launch range too large for the tiled path");
    long long grid = (long long)m->tm_blocks * sm_count();
    {
      long long period = ntx * nty, best = grid;
      for (long long gg = grid; gg > 1 && gg > grid - 32; --gg) {
        long long a0 = gg, b0 = period;
        while (b0) { long long t = a0 % b0; a0 = b0; b0 = t; }
        if (a0 == 1) { best = gg; break; }
      }
      grid = best;
    }
    if (grid > units) grid = units;
    if (grid < 1) grid = 1;
    void* args[] = {maps.data(), pk.data(), &sc, &g};
    CUresult r = launch_ex(m->tiledm, (unsigned)grid, (unsigned)m->tm_threads, m->tm_smem, st, args);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuLaunchKernel(lope_tiled_multi)");
    g_launches++;
    K->n_multi++;
    return 0;
  }
  if (k.rank == 1 && m->row && geom_ok && !std::getenv("LOPE_FORCE_GENERIC")) {
    // rank 1: one 16-byte vector per thread, the x range rounded down to whole vectors
    std::vector<HArr<T>> pk(k.arrays.size());
    for (size_t i = 0; i < k.arrays.size(); ++i) {
      pk[i].in = (const T*)in[i];
      pk[i].out = out ? (T*)out[i] : nullptr;
      pk[i].s1 = layouts[i].stride[1];
      pk[i].s2 = layouts[i].stride[2];
      pk[i].org = layouts[i].base + layouts[i].lo[0] + r0x;
    }
    g.xexact = 1;
    const long long nvec = (g.ext[0] + vx - 1) / vx;
    long long grid = std::min<long long>((nvec + 255) / 256, (long long)sm_count() * 8);
    if (grid < 1) grid = 1;
    void* args[] = {pk.data(), &sc, &g};
    CUresult r = launch_ex(m->row, (unsigned)grid, 256, 0, st, args);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuLaunchKernel(lope_row)");
    g_launches++;
    K->n_row++;
    return 0;
  }
  g.r0[0] = r0[0];
  g.ext[0] = ext[0];
  g.xshift = 0;
  std::vector<HArr<T>> pack(k.arrays.size());
  for (size_t i = 0; i < k.arrays.size(); ++i) {
    const lope_layout* L = &layouts[i];
    pack[i].in = (const T*)in[i];
    pack[i].out = out ? (T*)out[i] : nullptr;
    pack[i].s1 = L->stride[1];
    pack[i].s2 = L->stride[2];
    pack[i].org = L->base + (L->lo[0] + r0[0]) + (long long)(L->lo[1] + r0[1]) * L->stride[1] +
                  (long long)(L->lo[2] + r0[2]) * L->stride[2];
  }
  // enough blocks to fill the GPU a few times over; each block then walks many rows
  // and planes (grid-stride) instead of one 128-point row segment per block
  unsigned gx = (unsigned)((ext[0] + 127) / 128);
  const long long target = (long long)sm_count() * 16;
  long long gyl = std::min<long long>(ext[1], std::max<long long>(1, std::min<long long>(32, target / gx)));
  long long gzl = std::min<long long>(ext[2], std::max<long long>(1, target / ((long long)gx * gyl)));
  unsigned gy = (unsigned)std::min<long long>(gyl, 65535);
  unsigned gz = (unsigned)std::min<long long>(gzl, 65535);
  void* args[] = {pack.data(), &sc, &g};
  CUresult r = d.launchKernel(m->generic, gx, gy, gz, 128, 1, 1, 0, (CUstream)st, args, nullptr);
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuLaunchKernel(lope_generic)");
  g_launches++;
  K->n_generic++;
  return 0;
}

template <class T>
int copy_boxes_t(const lope_layout* layout, int32_t n, void* const* dst, const void* const* src,
                 const int64_t* dst_lo, const int64_t* src_lo, const int64_t* extent, cudaStream_t st) {
  DevLayout d = dev_layout(layout);
  for (int32_t i0 = 0; i0 < n; i0 += LOPE_MAX_BOXES) {
    LopeBoxes<T> bx;
    std::memset(&bx, 0, sizeof bx);
    int nb = 0;
    long long most = 1;
    for (int32_t i = i0; i < n && nb < LOPE_MAX_BOXES; ++i) {
      const int64_t* e = extent + 3 * i;
      if (e[0] == 0 || e[1] == 0 || e[2] == 0) continue;      // empty box
      bx.dst[nb] = (T*)dst[i];
      bx.src[nb] = (const T*)src[i];
      for (int k = 0; k < 3; ++k) {
        bx.d[nb][k] = dst_lo[3 * i + k];
        bx.s[nb][k] = src_lo[3 * i + k];
        bx.e[nb][k] = e[k];
      }
      const long long work = e[0] >= 16 ? e[1] * e[2] * 32 : e[0] * e[1] * e[2];
      most = std::max(most, work);
      ++nb;
    }
    if (nb == 0) continue;
    long long blocks = (most + 255) / 256;
    const long long cap = std::max<long long>(1, (long long)sm_count() * 16 / nb);
    if (blocks > cap) blocks = cap;
    lope_k_copy_boxes<T><<<dim3((unsigned)blocks, (unsigned)nb), 256, 0, st>>>(bx, d);
    CUDA_TRY(cudaGetLastError());
    g_launches++;
  }
  return 0;
}

int row_grid(const lope_layout* L) {
  long long rows = L->padded[1] * L->padded[2];
  long long blocks = (rows * 32 + 255) / 256;
  long long cap = (long long)sm_count() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

template <class T>
int copy_through(const lope_layout* L, const void* in, void* out, const int r0[3], const int ext[3],
                 cudaStream_t st) {
  DevLayout d = dev_layout(L);
  int b[3], e[3];
  for (int i = 0; i < 3; ++i) {
    b[i] = L->lo[i] + r0[i];
    e[i] = b[i] + ext[i];
  }
  lope_k_copy_through<T><<<row_grid(L), 256, 0, st>>>((const T*)in, (T*)out, d, b[0], e[0], b[1], e[1],
                                                        b[2], e[2]);
  CUDA_TRY(cudaGetLastError());
  g_launches++;
  return 0;
}

int check_interior_halo(const lope_layout* L) {
  for (int d = 0; d < L->rank; ++d) {
    if (L->lo[d] > L->interior[d] || L->hi[d] > L->interior[d])
      return fail(108, "halo width (%d,%d) exceeds the interior extent %lld in dim %d; the periodic "
                       "exchange is undefined there (SURVEY F8)",
                  L->lo[d], L->hi[d], (long long)L->interior[d], d + 1);
  }
  return 0;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

int lope_abi_version(void) { return LOPE_ABI_VERSION; }

const char* lope_last_error(void) { return g_err.c_str(); }

int64_t lope_launch_count(void) { return g_launches.load(); }

int lope_set_cache_dir(const char* path) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_cache_dir = path ? path : "";
  return 0;
}

int lope_layout_init(lope_layout* out, int32_t rank, int32_t dtype, const int64_t* interior,
                     const int32_t* lo, const int32_t* hi) {
  if (!out || !interior || !lo || !hi) return fail(108, "null argument");
  if (rank < 1 || rank > 3) return fail(108, "rank %d outside 1..3", rank);
  if (dtype != LOPE_F32 && dtype != LOPE_F64) return fail(108, "unknown dtype %d", dtype);
  lope_layout L;
  std::memset(&L, 0, sizeof L);
  L.rank = rank;
  L.dtype = dtype;
  L.elem_bytes = dtype == LOPE_F32 ? 4 : 8;
  for (int d = 0; d < 3; ++d) {
    if (d < rank) {
      if (interior[d] < 1) return fail(108, "interior extent %lld in dim %d must be positive",
                                       (long long)interior[d], d + 1);
      if (interior[d] > (1LL << 30)) return fail(108, "interior extent too large");
      if (lo[d] < 0 || lo[d] > 8 || hi[d] < 0 || hi[d] > 8)
        return fail(108, "halo widths (%d,%d) in dim %d outside 0..8", lo[d], hi[d], d + 1);
      L.interior[d] = interior[d];
      L.lo[d] = lo[d];
      L.hi[d] = hi[d];
    } else {
      L.interior[d] = 1;
    }
    L.padded[d] = L.interior[d] + L.lo[d] + L.hi[d];
  }
  // Rows start on 64-byte boundaries and the interior on one too: warp stores then
  // write whole DRAM atoms (calibrated: 16-byte-misaligned rows cost ~14% on B200;
  // lone 32-byte halo sectors sharing an atom with interior data written by another
  // CTA cost a read-modify-write).  64 bytes of room on each side hold the halo, so
  // x-halo refreshes are whole-atom stores too.
  const int64_t sec = 64 / L.elem_bytes;               // elements per 64-byte DRAM atom
  const int64_t head = L.lo[0] > 0 ? (L.lo[0] > sec ? L.lo[0] : sec) : 0;
  const int64_t ox = ((head + sec - 1) / sec) * sec;    // interior x origin, sector aligned
  L.base = ox - L.lo[0];
  L.stride[0] = 1;
  const int64_t tail = L.hi[0] > 0 ? (L.hi[0] > sec ? L.hi[0] : sec) : 0;
  L.stride[1] = ((ox + L.interior[0] + tail + sec - 1) / sec) * sec;
  L.stride[2] = L.stride[1] * L.padded[1];
  L.count = L.stride[2] * L.padded[2];
  *out = L;
  return 0;
}

int lope_kernel_compile(const char* ir_text, size_t n, int32_t dtype, lope_kernel** out) {
  if (!ir_text || !out) return fail(108, "null argument");
  if (dtype != LOPE_F32 && dtype != LOPE_F64) return fail(108, "unknown dtype %d", dtype);
  std::unique_ptr<lope_kernel> K(new lope_kernel());
  std::string text(ir_text, n);
  std::string err = lope::parse_kir(text, &K->ir);
  if (!err.empty()) return fail(104, "kernel IR rejected: %s", err.c_str());
  K->dtype = dtype;
  if (int e = add_variant(K.get(), pick_tile(K->ir, dtype))) return e;
  K->describe_path = K->ir.rank == 1 ? "row" : K->tiled_ok() ? "tiled_tma"
                     : (K->variants[0].source.find("lope_tiled_multi(") != std::string::npos ? "tiled_tma_multi"
                                                                                           : "generic");
  *out = K.release();
  return 0;
}

int lope_kernel_destroy(lope_kernel* k) {
  if (!k) return 0;
  Drv& d = drv();
  for (auto& v : k->variants)
    for (auto& kv : v.mods)
      if (kv.second.mod && d.ok) d.moduleUnload(kv.second.mod);
  delete k;
  return 0;
}

int lope_kernel_describe(const lope_kernel* k, char* buf, size_t n) {
  if (!k || !buf) return fail(108, "null argument");
  std::ostringstream o;
  const lope::Kir& ir = k->ir;
  o << "{\"name\":\"" << ir.name << "\",\"rank\":" << ir.rank << ",\"dtype\":\""
    << (k->dtype == LOPE_F32 ? "f32" : "f64") << "\",\"arrays\":[";
  for (size_t i = 0; i < ir.arrays.size(); ++i) o << (i ? "," : "") << "\"" << ir.arrays[i] << "\"";
  o << "],\"scalars\":[";
  for (size_t i = 0; i < ir.scalars.size(); ++i)
    o << (i ? "," : "") << "[\"" << ir.scalars[i] << "\",\"" << (ir.scalar_is_int[i] ? "integer" : "real") << "\"]";
  o << "],\"stored\":[";
  for (size_t i = 0; i < ir.stored.size(); ++i) o << (i ? "," : "") << ir.stored[i];
  o << "],\"footprints\":[";
  for (size_t a = 0; a < ir.arrays.size(); ++a) {
    o << (a ? "," : "") << "[";
    for (int d = 0; d < ir.rank; ++d) o << (d ? "," : "") << "[" << ir.fn[a][d] << "," << ir.fp[a][d] << "]";
    o << "]";
  }
  const TileCfg& t = k->tile();
  o << "],\"path\":\"" << k->describe_path << "\",\"tile\":[" << t.bxw << "," << t.wy << "," << t.ry << ","
    << t.ns << "],\"ctas_per_sm\":" << t.mb << ",\"producer_warp\":" << t.pw << ",\"reads\":" << ir.nreads
    << ",\"plans\":{";
  bool first = true;
  for (const auto& kv : k->plans) {
    const TileCfg& c = k->variants[kv.second.variant].tile;
    o << (first ? "" : ",") << "\"" << kv.first << "\":{\"tile\":[" << c.bxw << "," << c.wy << "," << c.ry << ","
      << c.ns << "],\"producer_warp\":" << c.pw << ",\"shfl\":" << c.sh << ",\"nb\":" << c.nb << ",\"zchunk\":" << kv.second.zchunk << ",\"yband\":" << kv.second.yband
      << "}";
    first = false;
  }
  // the compiled tile variants (lope_kernel_prepare adds the tuner's candidates)
  o << "},\"variants\":[";
  for (size_t i = 0; i < k->variants.size(); ++i) {
    const TileCfg& c = k->variants[i].tile;
    o << (i ? "," : "") << "{\"tile\":[" << c.bxw << "," << c.wy << "," << c.ry << "," << c.ns
      << "],\"producer_warp\":" << c.pw << ",\"shfl\":" << c.sh << ",\"nb\":" << c.nb << ",\"rag\":" << c.rag
      << ",\"tiled\":" << (k->variants[i].tiled_ok ? "true" : "false") << "}";
  }
  o << "],\"launches\":{\"tiled\":" << k->n_tiled.load() << ",\"tiled_multi\":" << k->n_multi.load()
    << ",\"row\":" << k->n_row.load() << ",\"tblock\":" << k->n_tblock.load() << ",\"generic\":"
    << k->n_generic.load() << "}}";
  std::string s = o.str();
  if (s.size() + 1 > n) return fail(108, "buffer too small (%zu needed)", s.size() + 1);
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return 0;
}

int lope_kernel_source(const lope_kernel* k, char* buf, size_t n) {
  if (!k || !buf) return fail(108, "null argument");
  const std::string& src = k->variants[0].source;
  if (src.size() + 1 > n) return fail(108, "buffer too small (%zu needed)", src.size() + 1);
  std::memcpy(buf, src.c_str(), src.size() + 1);
  return 0;
}

int lope_launch(const lope_kernel* kc, const lope_layout* layouts, const int64_t* ranges,
                const void* const* in, void* const* out, const double* rscal, const int64_t* iscal,
                void* stream) {
  lope_kernel* k = const_cast<lope_kernel*>(kc);
  if (!k || !layouts || !ranges || !in) return fail(108, "null argument");
  const lope::Kir& ir = k->ir;
  const int na = (int)ir.arrays.size();
  for (int a = 0; a < na; ++a) {
    if (int e = check_layout(&layouts[a])) return e;
    if (layouts[a].rank != ir.rank)
      return fail(108, "array '%s' has rank %d, kernel '%s' has rank %d", ir.arrays[a].c_str(),
                  layouts[a].rank, ir.name.c_str(), ir.rank);
    if (layouts[a].dtype != k->dtype) return fail(108, "array '%s' dtype differs from the kernel's",
                                                  ir.arrays[a].c_str());
    for (int d = 0; d < 3; ++d) {
      if (layouts[a].interior[d] != layouts[0].interior[d])
        return fail(108, "array arguments have different interiors");
      if (ir.fn[a][d] > layouts[a].lo[d] || ir.fp[a][d] > layouts[a].hi[d])
        return fail(102, "kernel '%s' reads '%s' %d/%d cells out in dim %d but the halo is (%d,%d)",
                    ir.name.c_str(), ir.arrays[a].c_str(), ir.fn[a][d], ir.fp[a][d], d + 1,
                    layouts[a].lo[d], layouts[a].hi[d]);
    }
    if (!in[a]) return fail(202, "array '%s' is not allocated", ir.arrays[a].c_str());
  }
  for (int q : ir.stored) {
    if (!out || !out[q]) return fail(202, "stored array '%s' has no output buffer", ir.arrays[q].c_str());
    if (out[q] == in[q]) return fail(108, "output buffer of '%s' aliases its snapshot", ir.arrays[q].c_str());
  }
  int r0[3] = {0, 0, 0}, ext[3] = {1, 1, 1};
  bool empty = false;
  // runtime.py:583-595: every dim is bounds-checked (E108) before an empty range returns
  for (int d = 0; d < ir.rank; ++d) {
    int64_t lo = ranges[2 * d], hi = ranges[2 * d + 1];
    if (lo < 1 || hi > layouts[0].interior[d])
      return fail(108, "launch range %lld:%lld lies outside the interior 1:%lld in dim %d", (long long)lo,
                  (long long)hi, (long long)layouts[0].interior[d], d + 1);
  }
  for (int d = 0; d < ir.rank; ++d) {
    int64_t lo = ranges[2 * d], hi = ranges[2 * d + 1];
    if (lo > hi) {
      empty = true;
      continue;
    }
    r0[d] = (int)(lo - 1);
    ext[d] = (int)(hi - lo + 1);
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (empty) {
    for (int q : ir.stored)
      CUDA_TRY(cudaMemcpyAsync(out[q], in[q], layouts[q].count * layouts[q].elem_bytes,
                               cudaMemcpyDeviceToDevice, st));
    return 0;
  }
  int e = k->dtype == LOPE_F32 ? run_body<float>(k, layouts, r0, ext, in, out, rscal, iscal, 0, st)
                               : run_body<double>(k, layouts, r0, ext, in, out, rscal, iscal, 0, st);
  if (e) return e;
  for (int q : ir.stored) {
    e = k->dtype == LOPE_F32 ? copy_through<float>(&layouts[q], in[q], out[q], r0, ext, st)
                             : copy_through<double>(&layouts[q], in[q], out[q], r0, ext, st);
    if (e) return e;
  }
  return 0;
}

int lope_step_arrays(const lope_kernel* kc, const lope_layout* layouts, const void* const* in,
                     void* const* out, const double* rscal, const int64_t* iscal, int32_t wrap_mask,
                     void* stream) {
  lope_kernel* k = const_cast<lope_kernel*>(kc);
  if (!k || !layouts || !in) return fail(108, "null argument");
  const lope::Kir& ir = k->ir;
  const int na = (int)ir.arrays.size();
  for (int a = 0; a < na; ++a) {
    if (int e = check_layout(&layouts[a])) return e;
    if (layouts[a].rank != ir.rank || layouts[a].dtype != k->dtype)
      return fail(108, "array '%s' rank/dtype do not match kernel '%s'", ir.arrays[a].c_str(), ir.name.c_str());
    for (int d = 0; d < 3; ++d) {
      if (layouts[a].interior[d] != layouts[0].interior[d])
        return fail(108, "array arguments have different interiors");
      if (ir.fn[a][d] > layouts[a].lo[d] || ir.fp[a][d] > layouts[a].hi[d])
        return fail(102, "kernel '%s' reads '%s' %d/%d cells out in dim %d but the halo is (%d,%d)",
                    ir.name.c_str(), ir.arrays[a].c_str(), ir.fn[a][d], ir.fp[a][d], d + 1, layouts[a].lo[d],
                    layouts[a].hi[d]);
    }
    if (!in[a]) return fail(202, "array '%s' is not allocated", ir.arrays[a].c_str());
  }
  const int wrap = wrap_mask & ((1 << ir.rank) - 1);
  for (int q : ir.stored) {
    if (!out || !out[q]) return fail(202, "stored array '%s' has no output buffer", ir.arrays[q].c_str());
    if (out[q] == in[q]) return fail(108, "output buffer of '%s' aliases its snapshot", ir.arrays[q].c_str());
    if (wrap)
      if (int e = check_interior_halo(&layouts[q])) return e;
    // the fused images are written for the first array's halo widths
    for (int d = 0; d < 3; ++d)
      if (wrap && (layouts[q].lo[d] != layouts[0].lo[d] || layouts[q].hi[d] != layouts[0].hi[d]))
        return fail(108, "stored arrays of a fused step need the halo widths of the first array");
  }
  int r0[3] = {0, 0, 0}, ext[3];
  for (int d = 0; d < 3; ++d) ext[d] = (int)layouts[0].interior[d];
  cudaStream_t st = (cudaStream_t)stream;
  return k->dtype == LOPE_F32 ? run_body<float>(k, layouts, r0, ext, in, out, rscal, iscal, wrap, st)
                              : run_body<double>(k, layouts, r0, ext, in, out, rscal, iscal, wrap, st);
}

int lope_step(const lope_kernel* kc, const lope_layout* layout, const void* in, void* out,
              const double* rscal, const int64_t* iscal, int32_t wrap_mask, void* stream) {
  if (!layout) return fail(108, "null argument");
  return lope_step_planes(kc, layout, in, out, 0, layout->interior[layout->rank - 1], rscal, iscal,
                          wrap_mask, stream);
}

}  // extern "C"

namespace {
int step_planes_impl(const lope_kernel* kc, const lope_layout* layout, const void* in, void* out, int64_t begin,
                     int64_t end, const double* rscal, const int64_t* iscal, int32_t wrap_mask,
                     const void* lo_peer, const void* hi_peer, void* stream) {
  lope_kernel* k = const_cast<lope_kernel*>(kc);
  if (!k || !layout) return fail(108, "null argument");
  if (int e = check_layout(layout)) return e;
  const lope::Kir& ir = k->ir;
  if (ir.arrays.size() != 1) return fail(108, "lope_step takes kernels with one array parameter");
  if (layout->rank != ir.rank || layout->dtype != k->dtype)
    return fail(108, "layout rank/dtype do not match kernel '%s'", ir.name.c_str());
  if (!in || !out) return fail(202, "buffer not allocated");
  if (in == out) return fail(108, "lope_step needs distinct input and output buffers");
  for (int d = 0; d < 3; ++d)
    if (ir.fn[0][d] > layout->lo[d] || ir.fp[0][d] > layout->hi[d])
      return fail(102, "kernel '%s' footprint exceeds the halo in dim %d", ir.name.c_str(), d + 1);
  if (int e = check_interior_halo(layout)) return e;
  const int sd = layout->rank - 1;   // slowest dimension
  if (begin < 0 || end > layout->interior[sd] || begin > end)
    return fail(108, "plane range %lld:%lld outside 0:%lld", (long long)begin, (long long)end,
                (long long)layout->interior[sd]);
  if (begin == end) return 0;
  int r0[3] = {0, 0, 0}, ext[3];
  for (int d = 0; d < 3; ++d) ext[d] = (int)layout->interior[d];
  r0[sd] = (int)begin;
  ext[sd] = (int)(end - begin);
  const void* ins[1] = {in};
  void* outs[1] = {out};
  int wrap = wrap_mask & ((1 << ir.rank) - 1);
  cudaStream_t st = (cudaStream_t)stream;
  long long sdl = 0, sdh = 0;
  if (lo_peer || hi_peer) {
    if (!((wrap >> sd) & 1)) return fail(108, "peer images need the slowest dim in the wrap mask");
    const long long eb = (long long)layout->elem_bytes;
    const long long dl = lo_peer ? (long long)((const char*)lo_peer - (const char*)out) : 0;
    const long long dh = hi_peer ? (long long)((const char*)hi_peer - (const char*)out) : 0;
    if (dl % eb || dh % eb) return fail(108, "peer buffers are not element-aligned with the output");
    sdl = dl / eb;
    sdh = dh / eb;
  }
  return k->dtype == LOPE_F32
             ? run_body<float>(k, layout, r0, ext, ins, outs, rscal, iscal, wrap, st, -1, 0, 0, sdl, sdh)
             : run_body<double>(k, layout, r0, ext, ins, outs, rscal, iscal, wrap, st, -1, 0, 0, sdl, sdh);
}
}  // namespace

extern "C" {

int lope_step_planes(const lope_kernel* kc, const lope_layout* layout, const void* in, void* out,
                     int64_t begin, int64_t end, const double* rscal, const int64_t* iscal,
                     int32_t wrap_mask, void* stream) {
  return step_planes_impl(kc, layout, in, out, begin, end, rscal, iscal, wrap_mask, nullptr, nullptr, stream);
}

int lope_step_planes_peer(const lope_kernel* kc, const lope_layout* layout, const void* in, void* out,
                          int64_t begin, int64_t end, const double* rscal, const int64_t* iscal,
                          int32_t wrap_mask, const void* lo_peer_out, const void* hi_peer_out, void* stream) {
  return step_planes_impl(kc, layout, in, out, begin, end, rscal, iscal, wrap_mask, lo_peer_out, hi_peer_out,
                          stream);
}

}  // extern "C"

namespace {

// Candidate (variant, z-chunk) plans (lope_plan_candidates).  3-D: the default in-band-producer
// variant with long z-chunks (past planes live in registers for many planes), and
// dedicated-producer variants with short z-chunks (neighbouring units overlap in L2,
// the 2-D regime) at several ring depths.  The best one depends on the geometry and
// is not monotone in any single parameter (B200, lap3d7 1024^3: 1.40 .. 1.96 ms).
struct PlanCand {
  TileCfg tile;
  int zchunk, yband;
};

std::vector<PlanCand> tune_candidates(const lope_kernel* K) {
  std::vector<PlanCand> c;
  const TileCfg base = K->variants[0].tile;
  if (K->ir.rank == 3) {
    // the plans that won on B200 across configs 3 and 5 and the random-kernel sweeps
    // (profiles/r02: 16-plane chunks, 3-4-plane chunks and 16 warps x 4 rows never did);
    // nine candidates keep tuning at ~120 steps; the in-band plan keeps 64-plane chunks
    // only (the watchdog's fallback: 32-plane chunks ran 1.58 vs 1.50 ms on config 3)
    c.push_back({base, 64, 0});
    if (base.pw == 0) {
      // in-band producer that only prefetches into free slots (2048^3: 13.4 vs 14.4 ms;
      // 1024^3: 1.57 vs 1.51 ms -- hence a candidate, not the default)
      TileCfg t = base;
      t.nb = 1;
      c.push_back({t, 64, 0});
    }
    for (int ns : {8, 10, 12}) {
      TileCfg t = base;
      t.pw = 1;
      t.ns = ns;
      t.sh = 1;
      for (int zc : {6, 8}) c.push_back({t, zc, 0});
    }
    if (K->dtype == LOPE_F32) {
      // 8 warps x 4 rows per lane: half the per-plane overhead per point
      TileCfg t = base;
      t.wy = 8;
      t.ry = 4;
      c.push_back({t, 64, 0});
    }
  } else {
    // 2-D: the dedicated producer always won (ninept2d 16384^2: 0.355 vs 0.50 ms in-band),
    // so the ring depth and the y tiles per unit vary; an in-band default (wide fp64
    // boxes) may try one
    for (int yc : {1, 8, 32}) c.push_back({base, yc, 0});
    TileCfg t = base;
    t.ns = base.ns == 8 ? 12 : 8;
    while (t.ns > 2 && t.mb * tiled_smem_bytes(K->ir, K->dtype, t) > 225 * 1024) --t.ns;
    if (t.ns != base.ns)          // (a ring that does not fit shared memory is no candidate)
      for (int yc : {8, 32}) c.push_back({t, yc, 0});
    if (base.pw == 0) {
      t = base;
      t.pw = 1;
      for (int yc : {8, 32}) c.push_back({t, yc, 0});
    }
    if (K->dtype == LOPE_F64 && base.bxw == 1 && base.wy % 2 == 0) {
      // wide-footprint fp64 (the 5x5 box): two warp columns x half the warps, dedicated
      // producer, the deepest ring that fits (config 4 on one box: 2.86-3.02 vs
      // 3.26-3.40 ms before the power cap, 3.40-3.43 vs 3.45 ms under it;
      // profiles/r02/s3/wide/s47_*)
      t = base;
      t.bxw = 2;
      t.wy = base.wy / 2;
      t.pw = 1;
      while (t.ns > 2 && t.mb * tiled_smem_bytes(K->ir, K->dtype, t) > 225 * 1024) --t.ns;
      for (int yc : {8, 32}) c.push_back({t, yc, 0});
    }
  }
  return c;
}

}  // namespace

extern "C" {

int lope_kernel_prepare(lope_kernel* k) {
  if (!k) return fail(108, "null argument");
  if (!k->tiled_ok()) return 0;
  for (const auto& cand : tune_candidates(k))
    if (int e = add_variant(k, cand.tile)) return e;
  return 0;
}

int lope_step_multi(const lope_kernel* kc, const lope_layout* layout, void* buf0, void* buf1, int64_t nsteps,
                    const double* rscal, const int64_t* iscal, void* stream, int32_t* live_index) {
  lope_kernel* k = const_cast<lope_kernel*>(kc);
  if (!k || !layout || !live_index) return fail(108, "null argument");
  if (int e = check_layout(layout)) return e;
  const lope::Kir& ir = k->ir;
  if (ir.arrays.size() != 1) return fail(108, "lope_step_multi takes kernels with one array parameter");
  if (layout->rank != ir.rank || layout->dtype != k->dtype)
    return fail(108, "layout rank/dtype do not match kernel '%s'", ir.name.c_str());
  if (!buf0 || !buf1) return fail(202, "buffer not allocated");
  if (buf0 == buf1) return fail(108, "lope_step_multi needs two distinct buffers");
  if (nsteps < 0) return fail(108, "negative step count");
  for (int d = 0; d < 3; ++d)
    if (ir.fn[0][d] > layout->lo[d] || ir.fp[0][d] > layout->hi[d])
      return fail(102, "kernel '%s' footprint exceeds the halo in dim %d", ir.name.c_str(), d + 1);
  if (int e = check_interior_halo(layout)) return e;
  DevMod* m = nullptr;
  if (int e = get_mod(k, 0, &m)) return e;
  const int full = (1 << ir.rank) - 1;
  const int vxe = 16 / (int)layout->elem_bytes;
  const bool tb = m->tblock && ir.rank == 2 && !std::getenv("LOPE_NO_TBLOCK") &&
                  layout->interior[0] % vxe == 0 && (m->tb_tt * ir.fn[0][0]) % vxe == 0 &&
                  layout->interior[0] >= m->tb_tx + m->tb_tt * (ir.fn[0][0] + ir.fp[0][0]) &&
                  layout->interior[1] >= m->tb_ty + m->tb_tt * (ir.fn[0][1] + ir.fp[0][1]);
  void* bufs[2] = {buf0, buf1};
  int live = 0;
  cudaStream_t st = (cudaStream_t)stream;
  Drv& d = drv();
  // blocks of tb_tt steps plus single steps; the buffer flips once per launch, so
  // trade one block for tb_tt single steps when that makes the parity match
  // nsteps -- the result then sits where nsteps single steps would leave it
  long long nblk = tb ? nsteps / m->tb_tt : 0;
  if (nblk > 0 && ((nblk + (nsteps - nblk * m->tb_tt)) & 1) != (nsteps & 1)) --nblk;
  while (nsteps > 0) {
    if (nblk > 0) {
      --nblk;
      const long long ntx = (layout->interior[0] + m->tb_tx - 1) / m->tb_tx;
      const long long nty = (layout->interior[1] + m->tb_ty - 1) / m->tb_ty;
      HGeom g;
      std::memset(&g, 0, sizeof g);
      for (int dd = 0; dd < 3; ++dd) {
        g.ext[dd] = (int)layout->interior[dd];
        g.m[dd] = (int)layout->interior[dd];
        g.lo[dd] = layout->lo[dd];
        g.hi[dd] = layout->hi[dd];
      }
      g.wrap = full;
      const long long org = layout->base + layout->lo[0] + (long long)layout->lo[1] * layout->stride[1];
      CUresult r;
      if (k->dtype == LOPE_F32) {
        HArr<float> a{(const float*)bufs[live], (float*)bufs[1 - live], layout->stride[1], layout->stride[2], org};
        HScal<float> sc = make_scal<float>(ir, rscal, iscal);
        void* args[] = {&a, &sc, &g};
        r = launch_ex(m->tblock, (unsigned)(ntx * nty), (unsigned)m->tb_threads, m->tb_smem, st, args);
      } else {
        HArr<double> a{(const double*)bufs[live], (double*)bufs[1 - live], layout->stride[1], layout->stride[2],
                       org};
        HScal<double> sc = make_scal<double>(ir, rscal, iscal);
        void* args[] = {&a, &sc, &g};
        r = launch_ex(m->tblock, (unsigned)(ntx * nty), (unsigned)m->tb_threads, m->tb_smem, st, args);
      }
      if (r != CUDA_SUCCESS) return cu_fail(r, "cuLaunchKernel(lope_tblock)");
      g_launches++;
      k->n_tblock++;
      nsteps -= m->tb_tt;
    } else {
      if (int e = lope_step(k, layout, bufs[live], bufs[1 - live], rscal, iscal, full, stream)) return e;
      nsteps -= 1;
    }
    live = 1 - live;
  }
  (void)d;
  *live_index = live;
  return 0;
}

int lope_copy_bytes(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0) return fail(108, "negative byte count");
  if (bytes == 0) return 0;
  if (!dst || !src) return fail(202, "null buffer");
  CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return 0;
}

// ---- CUDA IPC: the neighbours' output blocks for fused peer-store exchange ----

namespace {
std::mutex g_ipc_mu;
std::map<void*, void*> g_ipc_bases;   // opened pointer -> mapping base
}

int lope_ipc_export(const void* ptr, uint8_t* handle, int64_t* offset) {
  if (!ptr || !handle || !offset) return fail(108, "null argument");
  Drv& d = drv();
  if (!d.ok || !d.memGetAddressRange) return fail(-3, "cuMemGetAddressRange unavailable");
  CUDA_TRY(cudaFree(nullptr));
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult r = d.memGetAddressRange(&base, &size, (CUdeviceptr)ptr);
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemGetAddressRange");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, (void*)base));
  std::memcpy(handle, &h, sizeof h);
  *offset = (int64_t)((CUdeviceptr)ptr - base);
  return 0;
}

int lope_ipc_open(const uint8_t* handle, int64_t offset, void** ptr) {
  if (!handle || !ptr) return fail(108, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  void* base = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr = (char*)base + offset;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  g_ipc_bases[*ptr] = base;
  return 0;
}

int lope_ipc_close(void* ptr) {
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    auto it = g_ipc_bases.find(ptr);
    if (it == g_ipc_bases.end()) return fail(108, "pointer was not opened by lope_ipc_open");
    base = it->second;
    g_ipc_bases.erase(it);
  }
  CUDA_TRY(cudaIpcCloseMemHandle(base));
  return 0;
}

int lope_plan_candidates(lope_kernel* k, int32_t* variants, int32_t* zchunks, int32_t* ybands, int32_t cap,
                         int32_t* n) {
  if (!k || !n) return fail(108, "null argument");
  *n = 0;
  if (!k->tiled_ok()) return 0;
  for (const auto& cand : tune_candidates(k)) {
    int vi = 0;
    if (int e = add_variant(k, cand.tile, &vi)) return e;
    if (!k->variants[vi].tiled_ok) continue;
    DevMod* m = nullptr;
    if (int e = get_mod(k, vi, &m)) return e;
    if (m->tiled_local > 0) continue;   // spills go through L2 and cost halo reuse
    if (*n < cap && variants && zchunks && ybands) {
      variants[*n] = vi;
      zchunks[*n] = cand.zchunk;
      ybands[*n] = cand.yband;
    }
    ++*n;
  }
  return 0;
}

int lope_plan_set_tile(lope_kernel* k, const lope_layout* layout, int32_t wrap_mask, const int32_t* tile,
                       int32_t zchunk, int32_t yband, int32_t* variant) {
  if (!k || !layout || !tile) return fail(108, "null argument");
  if (int e = check_layout(layout)) return e;
  TileCfg c;
  c.bxw = tile[0];
  c.wy = tile[1];
  c.ry = tile[2];
  c.ns = tile[3];
  c.pw = tile[4] ? 1 : 0;
  c.mb = tile[5] == 2 ? 2 : 1;
  if (c.bxw < 1 || c.wy < 1 || c.ry < 1 || c.ns < 2) return fail(108, "bad tile shape");
  int vi = 0;
  if (int e = add_variant(k, c, &vi)) return e;
  if (!k->variants[vi].tiled_ok) return fail(108, "tile variant does not fit shared memory");
  if (variant) *variant = vi;
  return lope_plan_set(k, layout, wrap_mask, vi, zchunk, yband);
}

int lope_plan_set_variant(lope_kernel* k, const lope_layout* layout, int32_t wrap_mask, const int32_t* cfg,
                          int32_t zchunk, int32_t yband, int32_t* variant) {
  if (!k || !layout || !cfg) return fail(108, "null argument");
  if (int e = check_layout(layout)) return e;
  TileCfg c;
  c.bxw = cfg[0];
  c.wy = cfg[1];
  c.ry = cfg[2];
  c.ns = cfg[3];
  c.pw = cfg[4] ? 1 : 0;
  c.mb = cfg[5] == 2 ? 2 : 1;
  c.sh = cfg[6] ? 1 : 0;
  c.nb = cfg[7] ? 1 : 0;
  if (c.bxw < 1 || c.wy < 1 || c.ry < 1 || c.ns < 2) return fail(108, "bad tile shape");
  int vi = 0;
  if (int e = add_variant(k, c, &vi)) return e;
  if (!k->variants[vi].tiled_ok) return fail(108, "tile variant does not fit shared memory");
  if (variant) *variant = vi;
  return lope_plan_set(k, layout, wrap_mask, vi, zchunk, yband);
}

int lope_plan_set(lope_kernel* k, const lope_layout* layout, int32_t wrap_mask, int32_t variant, int32_t zchunk,
                  int32_t yband) {
  if (!k || !layout) return fail(108, "null argument");
  if (int e = check_layout(layout)) return e;
  const std::string key = plan_key(layout, wrap_mask & ((1 << k->ir.rank) - 1));
  if (variant < 0) {
    k->plans.erase(key);
    return 0;
  }
  if (variant >= (int32_t)k->variants.size()) return fail(108, "no plan variant %d", variant);
  LopePlan p;
  p.variant = variant;
  p.zchunk = zchunk;
  p.yband = yband;
  k->plans[key] = p;
  return 0;
}

int lope_halo_fill(const lope_layout* layout, void* buf, int32_t dims_mask, void* stream) {
  if (int e = check_layout(layout)) return e;
  if (!buf) return fail(202, "buffer not allocated");
  if (int e = check_interior_halo(layout)) return e;
  int mask = dims_mask & ((1 << layout->rank) - 1);
  bool any = false;
  for (int d = 0; d < layout->rank; ++d)
    if ((mask >> d & 1) && (layout->lo[d] || layout->hi[d])) any = true;
  if (!any) return 0;
  DevLayout d = dev_layout(layout);
  cudaStream_t st = (cudaStream_t)stream;
  if (layout->dtype == LOPE_F32)
    lope_k_halo_fill<float><<<row_grid(layout), 256, 0, st>>>((float*)buf, d, mask);
  else
    lope_k_halo_fill<double><<<row_grid(layout), 256, 0, st>>>((double*)buf, d, mask);
  CUDA_TRY(cudaGetLastError());
  g_launches++;
  return 0;
}

static int pack_impl(const lope_layout* L, const void* host, void* dev, cudaStream_t st, bool to_dev,
                     bool padded = false) {
  if (int e = check_layout(L)) return e;
  if (!host || !dev) return fail(202, "null buffer");
  cudaMemcpy3DParms p;
  std::memset(&p, 0, sizeof p);
  const size_t eb = (size_t)L->elem_bytes;
  // host side: the interior (or, with `padded`, the whole padded block) packed
  // column-major exactly like the reference's flat blocks (ir.py:189-230)
  const int64_t* hx = padded ? L->padded : L->interior;
  cudaPitchedPtr hp = make_cudaPitchedPtr(const_cast<void*>(host), hx[0] * eb, hx[0], hx[1]);
  cudaPitchedPtr dp = make_cudaPitchedPtr(dev, L->stride[1] * eb, L->stride[1], L->padded[1]);
  cudaPos dpos = padded ? make_cudaPos(L->base * eb, 0, 0)
                        : make_cudaPos((L->base + L->lo[0]) * eb, L->lo[1], L->lo[2]);
  p.extent = make_cudaExtent(hx[0] * eb, hx[1], hx[2]);
  if (to_dev) {
    p.srcPtr = hp;
    p.dstPtr = dp;
    p.dstPos = dpos;
    p.kind = cudaMemcpyHostToDevice;
  } else {
    p.srcPtr = dp;
    p.srcPos = dpos;
    p.dstPtr = hp;
    p.kind = cudaMemcpyDeviceToHost;
  }
  CUDA_TRY(cudaMemcpy3DAsync(&p, st));
  return 0;
}

int lope_pack(const lope_layout* layout, const void* host, void* dev, void* stream) {
  return pack_impl(layout, host, dev, (cudaStream_t)stream, true);
}

int lope_unpack(const lope_layout* layout, const void* dev, void* host, void* stream) {
  return pack_impl(layout, host, const_cast<void*>(dev), (cudaStream_t)stream, false);
}

int lope_pack_padded(const lope_layout* layout, const void* host, void* dev, void* stream) {
  return pack_impl(layout, host, dev, (cudaStream_t)stream, true, true);
}

int lope_unpack_padded(const lope_layout* layout, const void* dev, void* host, void* stream) {
  return pack_impl(layout, host, const_cast<void*>(dev), (cudaStream_t)stream, false, true);
}

int lope_copy_box(const lope_layout* layout, void* dst, const void* src, const int64_t* dst_lo,
                  const int64_t* src_lo, const int64_t* extent, void* stream) {
  if (int e = check_layout(layout)) return e;
  if (!dst || !src || !dst_lo || !src_lo || !extent) return fail(202, "null argument");
  for (int d = 0; d < 3; ++d) {
    if (extent[d] < 0 || dst_lo[d] < 0 || src_lo[d] < 0 || dst_lo[d] + extent[d] > layout->padded[d] ||
        src_lo[d] + extent[d] > layout->padded[d])
      return fail(108, "box outside the padded block in dim %d", d + 1);
    if (extent[d] == 0) return 0;
  }
  DevLayout d = dev_layout(layout);
  cudaStream_t st = (cudaStream_t)stream;
  long long rows = extent[1] * extent[2];
  long long blocks = (rows * 32 + 255) / 256;
  long long cap = (long long)sm_count() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (layout->dtype == LOPE_F32)
    lope_k_copy_box<float><<<(int)blocks, 256, 0, st>>>((float*)dst, (const float*)src, d, dst_lo[0], dst_lo[1],
                                                         dst_lo[2], src_lo[0], src_lo[1], src_lo[2], extent[0],
                                                         extent[1], extent[2]);
  else
    lope_k_copy_box<double><<<(int)blocks, 256, 0, st>>>((double*)dst, (const double*)src, d, dst_lo[0],
                                                          dst_lo[1], dst_lo[2], src_lo[0], src_lo[1], src_lo[2],
                                                          extent[0], extent[1], extent[2]);
  CUDA_TRY(cudaGetLastError());
  g_launches++;
  return 0;
}

namespace {
int box_xfer(const lope_layout* layout, void* blk, void* buf, const int64_t* lo, const int64_t* extent,
             void* stream, bool pack) {
  if (int e = check_layout(layout)) return e;
  if (!blk || !buf || !lo || !extent) return fail(202, "null argument");
  for (int d = 0; d < 3; ++d) {
    if (extent[d] < 0 || lo[d] < 0 || lo[d] + extent[d] > layout->padded[d])
      return fail(108, "box outside the padded block in dim %d", d + 1);
    if (extent[d] == 0) return 0;
  }
  DevLayout d = dev_layout(layout);
  cudaStream_t st = (cudaStream_t)stream;
  long long rows = extent[1] * extent[2];
  long long blocks = (rows * 32 + 255) / 256;
  long long cap = (long long)sm_count() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const int nb = (int)blocks;
  if (layout->dtype == LOPE_F32) {
    if (pack)
      lope_k_box_xfer<float, true><<<nb, 256, 0, st>>>((float*)blk, (float*)buf, d, lo[0], lo[1], lo[2],
                                                        extent[0], extent[1], extent[2]);
    else
      lope_k_box_xfer<float, false><<<nb, 256, 0, st>>>((float*)blk, (float*)buf, d, lo[0], lo[1], lo[2],
                                                         extent[0], extent[1], extent[2]);
  } else {
    if (pack)
      lope_k_box_xfer<double, true><<<nb, 256, 0, st>>>((double*)blk, (double*)buf, d, lo[0], lo[1], lo[2],
                                                         extent[0], extent[1], extent[2]);
    else
      lope_k_box_xfer<double, false><<<nb, 256, 0, st>>>((double*)blk, (double*)buf, d, lo[0], lo[1], lo[2],
                                                          extent[0], extent[1], extent[2]);
  }
  CUDA_TRY(cudaGetLastError());
  g_launches++;
  return 0;
}
}  // namespace

int lope_copy_boxes(const lope_layout* layout, int32_t n, void* const* dst, const void* const* src,
                    const int64_t* dst_lo, const int64_t* src_lo, const int64_t* extent, void* stream) {
  if (int e = check_layout(layout)) return e;
  if (n < 0) return fail(108, "negative box count");
  if (n == 0) return 0;
  if (!dst || !src || !dst_lo || !src_lo || !extent) return fail(202, "null argument");
  for (int32_t i = 0; i < n; ++i) {
    if (!dst[i] || !src[i]) return fail(202, "box %d has a null buffer", i);
    for (int d = 0; d < 3; ++d) {
      const int64_t e = extent[3 * i + d], a = dst_lo[3 * i + d], b = src_lo[3 * i + d];
      if (e < 0 || a < 0 || b < 0 || a + e > layout->padded[d] || b + e > layout->padded[d])
        return fail(108, "box %d outside the padded block in dim %d", i, d + 1);
    }
  }
  cudaStream_t st = (cudaStream_t)stream;
  return layout->dtype == LOPE_F32 ? copy_boxes_t<float>(layout, n, dst, src, dst_lo, src_lo, extent, st)
                                   : copy_boxes_t<double>(layout, n, dst, src, dst_lo, src_lo, extent, st);
}

int lope_box_pack(const lope_layout* layout, const void* blk, const int64_t* lo, const int64_t* extent,
                  void* buf, void* stream) {
  return box_xfer(layout, const_cast<void*>(blk), buf, lo, extent, stream, true);
}

int lope_box_unpack(const lope_layout* layout, void* blk, const int64_t* lo, const int64_t* extent,
                    const void* buf, void* stream) {
  return box_xfer(layout, blk, const_cast<void*>(buf), lo, extent, stream, false);
}

int lope_fill_hash(const lope_layout* layout, void* dev, uint64_t seed, const int64_t* gext,
                   const int64_t* gorg, void* stream) {
  if (int e = check_layout(layout)) return e;
  if (!dev || !gext || !gorg) return fail(202, "null argument");
  DevLayout d = dev_layout(layout);
  cudaStream_t st = (cudaStream_t)stream;
  long long n = layout->interior[0] * layout->interior[1] * layout->interior[2];
  long long grid = (n + 255) / 256;
  long long cap = (long long)sm_count() * 16;
  if (grid > cap) grid = cap;
  if (layout->dtype == LOPE_F32)
    lope_k_fill_hash<float><<<(int)grid, 256, 0, st>>>((float*)dev, d, seed, gext[0], gext[1], gorg[0],
                                                        gorg[1], gorg[2]);
  else
    lope_k_fill_hash<double><<<(int)grid, 256, 0, st>>>((double*)dev, d, seed, gext[0], gext[1], gorg[0],
                                                         gorg[1], gorg[2]);
  CUDA_TRY(cudaGetLastError());
  g_launches++;
  return 0;
}

int lope_face_span(const lope_layout* L, int32_t which, int64_t* offset, int64_t* count) {
  if (int e = check_layout(L)) return e;
  if (!offset || !count) return fail(108, "null argument");
  const int d = L->rank - 1;
  const int64_t plane = d == 0 ? 1 : L->stride[d];
  const int64_t m = L->interior[d];
  const int lo = L->lo[d], hi = L->hi[d];
  switch (which) {
    case 0: *offset = 0; *count = lo * plane; break;                       // low halo
    case 1: *offset = (lo + m) * plane; *count = hi * plane; break;        // high halo
    case 2: *offset = lo * plane; *count = hi * plane; break;              // first `hi` interior planes
    case 3: *offset = m * plane; *count = lo * plane; break;               // last `lo` interior planes
    default: return fail(108, "face selector %d outside 0..3", which);
  }
  if (d == 0) *offset += L->base;       // rank 1: "planes" are single elements of the row
  return 0;
}

}  // extern "C"
