// lope_device.cuh — sm_100a stencil kernel templates (NVRTC-compiled; no host headers).
//
// A kernel body generated from the IR (lope_codegen.cpp) is spliced in as
// `struct LopeBody`; this file supplies the launch templates around it:
//
//   * lope_tiled_impl  — rank 2/3, one array parameter.  TMA (cp.async.bulk.tensor)
//                        stages tile-plus-halo boxes of one plane into a
//                        shared-memory ring guarded by mbarriers; each thread keeps
//                        one x column and RY rows, evaluates the body reading
//                        neighbours from smem (z neighbours from the ring's other
//                        planes), and stores straight to HBM.  Work is a z-major
//                        list of (x tile, y tile, z chunk) units walked with a
//                        grid stride, so CTAs resident at the same time share
//                        halo rows and planes through L2.  The TMA ring continues
//                        across units (prefetch of unit n+1 overlaps unit n).
//   * lope_generic_impl — any rank, any number of array parameters, reads through
//                        the read-only path; used when the tiled path does not apply.
//
// Both can run the fused "halo refresh" epilogue: every stored value whose
// position has periodic images in the halo of a wrapped (non-decomposed) dim is
// also stored at those images, which is exactly the state the reference reaches
// after the next HALO_TRANSFER (runtime.py:653-697 with neighbour == self).
//
// Arithmetic is IEEE round-to-nearest with no contraction (__fadd_rn / __fmul_rn
// never fuse), matching numpy's per-node evaluation in lopec/ir.py:282-299.

typedef unsigned long long lope_u64;
typedef long long lope_i64;
typedef unsigned int lope_u32;

// --------------------------------------------------------------------------
// IEEE arithmetic (per-node rounding, numpy NaN semantics for min/max)

template <class T> struct LopeAr;
template <> struct LopeAr<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float neg(float a) { return -a; }
  static __device__ __forceinline__ float abs_(float a) { return fabsf(a); }
  static __device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
};
template <> struct LopeAr<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double neg(double a) { return -a; }
  static __device__ __forceinline__ double abs_(double a) { return fabs(a); }
  static __device__ __forceinline__ double sqrt_(double a) { return __dsqrt_rn(a); }
};
// numpy.minimum / numpy.maximum: NaN in either operand propagates; ties return the second.
template <class T> __device__ __forceinline__ T lope_min(T a, T b) { return (a != a || a < b) ? a : b; }
template <class T> __device__ __forceinline__ T lope_max(T a, T b) { return (a != a || a > b) ? a : b; }

// --------------------------------------------------------------------------
// Parameters

#define LOPE_MAX_ARR 8
#define LOPE_MAX_SCAL 16

template <class T> struct LopeScal { T v[LOPE_MAX_SCAL]; };

// One array argument: `in` is the launch snapshot, `out` the live buffer (may be 0
// for arrays the kernel never stores).  Element (i,j,k) of the padded block sits at
// in[i + j*s1 + k*s2]; `org` is the flat offset of interior cell (0,0,0) + range start.
template <class T> struct LopeArr {
  const T* in;
  T* out;
  lope_i64 s1, s2;
  lope_i64 org;
};

struct LopeGeom {
  int ext[3];     // launch-range extents (points per dim)
  int m[3];       // interior extents of the (first) array
  int r0[3];      // launch-range start, 0-based interior coordinates
  int lo[3], hi[3];
  int wrap;       // bit d: refresh periodic halo images along dim d in the epilogue
  int zchunk;     // tiled: planes per work unit
  int xshift;     // tiled: elements the TMA box starts early so its start is 16-byte aligned
  int box0;       // tiled: TMA x coordinate of tile 0's box (row-relative, already shifted)
};

// --------------------------------------------------------------------------
// Periodic-image epilogue

template <class T>
__device__ __noinline__ void lope_store_images(T* __restrict__ out, lope_i64 s1, lope_i64 s2,
                                                  lope_i64 org0, int x, int y, int z,
                                                  const LopeGeom& g, T v) {
  // (x,y,z) are 0-based interior coordinates; org0 = flat offset of interior (0,0,0).
  // Per dim: the point itself, its image in the high halo (x < hi -> x+m) and its
  // image in the low halo (x >= m-lo -> x-m).  Written without arrays so the
  // selection stays in registers.
  const bool xh = (g.wrap & 1) && x < g.hi[0], xl = (g.wrap & 1) && x >= g.m[0] - g.lo[0];
  const bool yh = (g.wrap & 2) && y < g.hi[1], yl = (g.wrap & 2) && y >= g.m[1] - g.lo[1];
  const bool zh = (g.wrap & 4) && z < g.hi[2], zl = (g.wrap & 4) && z >= g.m[2] - g.lo[2];
  if (!(xh | xl | yh | yl | zh | zl)) return;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const bool cz = c == 0 ? true : (c == 1 ? zh : zl);
    const int zz = c == 0 ? z : (c == 1 ? z + g.m[2] : z - g.m[2]);
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const bool cy = b == 0 ? true : (b == 1 ? yh : yl);
      const int yy = b == 0 ? y : (b == 1 ? y + g.m[1] : y - g.m[1]);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if ((a | b | c) == 0) continue;
        const bool cx = a == 0 ? true : (a == 1 ? xh : xl);
        const int xx = a == 0 ? x : (a == 1 ? x + g.m[0] : x - g.m[0]);
        if (cx && cy && cz) out[org0 + (lope_i64)xx + (lope_i64)yy * s1 + (lope_i64)zz * s2] = v;
      }
    }
  }
}

// --------------------------------------------------------------------------
// Generic path: one thread per point, reads through the read-only data path.

template <class T> struct LopeGlobalReader {
  const LopeArr<T>* a;
  lope_i64 off;   // i + j*s1 + k*s2 relative to each array's org (all arrays share extents)
  lope_i64 offs[LOPE_MAX_ARR];
  template <int A, int DX, int DY, int DZ>
  __device__ __forceinline__ T at() const {
    return __ldg(a[A].in + offs[A] + DX + (lope_i64)DY * a[A].s1 + (lope_i64)DZ * a[A].s2);
  }
};

__device__ __forceinline__ bool lope_near(int c, int m, int lo, int hi) {
  return c < hi || c >= m - lo;
}

// Grid: x = blockIdx.x*blockDim.x + threadIdx.x, rows over blockIdx.y, planes over
// blockIdx.z (grid-stride in each), so there is no per-point division.
template <class Body, class T>
__device__ __forceinline__ void lope_generic_impl(const LopeArr<T>* arrs, const LopeScal<T>& sc,
                                                  const LopeGeom& g) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.ext[0]) return;
  const bool xn = (g.wrap & 1) && lope_near(i + g.r0[0], g.m[0], g.lo[0], g.hi[0]);
  for (int k = blockIdx.z; k < g.ext[2]; k += gridDim.z) {
    const bool zn = (g.wrap & 4) && lope_near(k + g.r0[2], g.m[2], g.lo[2], g.hi[2]);
    for (int j = blockIdx.y; j < g.ext[1]; j += gridDim.y) {
      const bool yn = (g.wrap & 2) && lope_near(j + g.r0[1], g.m[1], g.lo[1], g.hi[1]);
      LopeGlobalReader<T> rd;
      rd.a = arrs;
#pragma unroll
      for (int q = 0; q < Body::NARR; ++q)
        rd.offs[q] = arrs[q].org + i + (lope_i64)j * arrs[q].s1 + (lope_i64)k * arrs[q].s2;
      T res[Body::NSTORE > 0 ? Body::NSTORE : 1];
      Body::template eval<T>(rd, sc.v, res);
#pragma unroll
      for (int q = 0; q < Body::NSTORE; ++q) {
        const int A = Body::stored(q);
        T* o = arrs[A].out;
        o[rd.offs[A]] = res[q];
        if (xn | yn | zn) {
          const lope_i64 org0 = arrs[A].org - g.r0[0] - (lope_i64)g.r0[1] * arrs[A].s1 -
                                (lope_i64)g.r0[2] * arrs[A].s2;
          lope_store_images<T>(o, arrs[A].s1, arrs[A].s2, org0, i + g.r0[0], j + g.r0[1],
                               k + g.r0[2], g, res[q]);
        }
      }
    }
  }
}

// --------------------------------------------------------------------------
// TMA + mbarrier primitives (sm_90+ PTX; SASS shows UTMALDG / SYNCS)

struct __align__(64) LopeTmap { lope_u64 v[16]; };

__device__ __forceinline__ lope_u32 lope_smem_u32(const void* p) {
  return (lope_u32)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void lope_mbar_init(lope_u64* bar, lope_u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(lope_smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void lope_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void lope_mbar_expect_tx(lope_u64* bar, lope_u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(lope_smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Bounded wait: a TMA that never completes traps (kernel error) instead of hanging the GPU.
#ifndef LOPE_WAIT_LIMIT
#define LOPE_WAIT_LIMIT (1u << 26)
#endif
__device__ __forceinline__ void lope_mbar_wait(lope_u64* bar, lope_u32 parity) {
  const lope_u32 addr = lope_smem_u32(bar);
  lope_u32 done = 0, n = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (++n > LOPE_WAIT_LIMIT) __trap();
  } while (!done);
}
__device__ __forceinline__ void lope_tma_load_3d(void* dst, const LopeTmap* map, lope_u64* bar, int c0,
                                                 int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(lope_smem_u32(dst)),
      "l"((lope_u64)map), "r"(c0), "r"(c1), "r"(c2), "r"(lope_smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void lope_tma_prefetch_desc(const LopeTmap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"((lope_u64)map) : "memory");
}

// --------------------------------------------------------------------------
// Tiled TMA path

template <class T, int BOXX, int NZW, int FZN>
struct LopeSmemReader {
  const T* sp[NZW];   // per z offset: this thread's (column, first row) in that plane's box
  template <int A, int DX, int DY, int DZ>
  __device__ __forceinline__ T at() const {
    return sp[DZ + FZN][DY * BOXX + DX];
  }
};

template <class Body, class T, int BXW, int WY, int RY, int NS>
struct LopeTiledCfg {
  static constexpr int BX = 32 * BXW;
  static constexpr int BY = WY * RY;
  static constexpr int VEC = 16 / (int)sizeof(T);
  // the box starts up to VEC-1 elements early (16-byte aligned TMA start), hence +VEC-1
  static constexpr int BOXX = ((Body::FN0 + BX + Body::FP0 + VEC - 1 + VEC - 1) / VEC) * VEC;
  static constexpr int BOXY = BY + Body::FN1 + Body::FP1;
  static constexpr int NZW = Body::FN2 + Body::FP2 + 1;
  static constexpr int STAGE_BYTES = ((BOXX * BOXY * (int)sizeof(T) + 127) / 128) * 128;
  static constexpr int TX_BYTES = BOXX * BOXY * (int)sizeof(T);
  static constexpr int SMEM_BYTES = NS * STAGE_BYTES + 2 * NS * 8;
  static constexpr int NCW = BXW * WY;             // consumer (compute) warps
  static constexpr int THREADS = 32 * (NCW + 1);   // + one TMA producer warp
};

__device__ __forceinline__ void lope_mbar_arrive(lope_u64* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(lope_smem_u32(bar)) : "memory");
}

// Warp-specialised: warp NCW issues TMA loads into an NS-slot ring (full[s]:
// TMA bytes landed; empty[s]: every compute warp is done with the slot); warps
// 0..NCW-1 compute.  No CTA-wide barrier inside the loop, so warps drift within
// the ring window and the producer runs up to NS loads ahead.
template <class Body, class T, int BXW, int WY, int RY, int NS>
__device__ __forceinline__ void lope_tiled_impl(const LopeTmap* map, const LopeArr<T>& a,
                                                const LopeScal<T>& sc, const LopeGeom& g) {
  typedef LopeTiledCfg<Body, T, BXW, WY, RY, NS> C;
  static_assert(NS >= C::NZW + 1, "ring must hold the z window plus one prefetch slot");
  constexpr int FZN = Body::FN2;
  constexpr int NZW = C::NZW;
  extern __shared__ __align__(128) unsigned char lope_smem[];
  lope_u64* full = reinterpret_cast<lope_u64*>(lope_smem + NS * C::STAGE_BYTES);
  lope_u64* empty = full + NS;

  const int ntx = (g.ext[0] + C::BX - 1) / C::BX;
  const int nty = (g.ext[1] + C::BY - 1) / C::BY;
  const int zc = g.zchunk;
  const int nzc = (g.ext[2] + zc - 1) / zc;
  const int nunits = ntx * nty * nzc;     // < 2^31 (host checks)

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    lope_tma_prefetch_desc(map);
    for (int s = 0; s < NS; ++s) {
      lope_mbar_init(&full[s], 1);
      lope_mbar_init(&empty[s], C::NCW);
    }
    lope_fence_init();
  }
  __syncthreads();

  if (warp == C::NCW) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const int ox = g.box0;
      const int oy = g.lo[1] + g.r0[1] - Body::FN1;
      const int oz = g.lo[2] + g.r0[2] - FZN;
      lope_u32 L = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int ty = u % nty;            // y fastest: neighbours in y run concurrently and
        const int r_ = u / nty;            // x-edge tiles rotate over CTAs
        const int tx = r_ % ntx;
        const int z0 = (r_ / ntx) * zc;
        const int nl = min(zc, g.ext[2] - z0) + NZW - 1;
        for (int pl = 0; pl < nl; ++pl, ++L) {
          const lope_u32 slot = L % NS;
          if (L >= (lope_u32)NS) lope_mbar_wait(&empty[slot], ((L / NS) - 1) & 1);
          lope_mbar_expect_tx(&full[slot], C::TX_BYTES);
          lope_tma_load_3d(lope_smem + slot * C::STAGE_BYTES, map, &full[slot], ox + tx * C::BX,
                           oy + ty * C::BY, oz + z0 + pl);
        }
      }
    }
    return;
  }

  // ---------------- compute warps ----------------
  const int wx = warp % BXW;
  const int wy = warp / BXW;
  const int col = wx * 32 + lane;          // column within the tile
  const int row0 = wy * RY;                // first row within the tile
  const lope_i64 s1 = a.s1, s2 = a.s2;
  const lope_i64 org0 = a.org - g.r0[0] - (lope_i64)g.r0[1] * s1 - (lope_i64)g.r0[2] * s2;

  lope_u32 lbase = 0;
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int ty = u % nty;
    const int r_ = u / nty;
    const int tx = r_ % ntx;
    const int z0 = (r_ / ntx) * zc;
    const int nz = min(zc, g.ext[2] - z0);
    const int x = tx * C::BX + col;
    const int ybase = ty * C::BY + row0;
    const bool xok = x < g.ext[0];
    // Periodic-image epilogue, precomputed per lane (x) / per warp row (y) / per plane
    // (z): each dim has at most one image when m >= lo + hi; smaller interiors take
    // the general (rare, slow) path.
    // x images are written a whole 64-byte atom at a time: the SEC boundary lanes
    // whose images land in the halo atom all store, padding cells included (the
    // layout reserves an atom on each side), so no partial atoms reach DRAM.
    constexpr int SEC = 64 / (int)sizeof(T);          // one 64-byte DRAM atom
    const int xg = x + g.r0[0];
    const bool xw = (g.wrap & 1) && ((g.hi[0] > 0 && xg < SEC) || (g.lo[0] > 0 && xg >= g.m[0] - SEC));
    const int ximg = xg < SEC ? g.m[0] : -g.m[0];       // x image offset (if xw)
    const bool one_x = g.m[0] >= 2 * SEC;
    const bool one_y = g.m[1] >= g.lo[1] + g.hi[1];
    const bool one_z = g.m[2] >= g.lo[2] + g.hi[2];
    const bool simple = one_x && one_y && one_z;
    // warp-uniform: does any lane of this warp have an x image, or any of its rows a y image?
    const bool wx_any = __any_sync(0xffffffffu, xw && xok);
    const bool wy_any = (g.wrap & 2) && (lope_near(ybase + g.r0[1], g.m[1], g.lo[1], g.hi[1]) ||
                                         lope_near(min(ybase + RY - 1, g.ext[1] - 1) + g.r0[1], g.m[1],
                                                   g.lo[1], g.hi[1]) ||
                                         !one_y);
    T* orow = a.out + a.org + x + (lope_i64)ybase * s1 + (lope_i64)z0 * s2;
    for (int pz = 0; pz < nz; ++pz, orow += s2) {
      LopeSmemReader<T, C::BOXX, NZW, FZN> rd;
#pragma unroll
      for (int w = 0; w < NZW; ++w) {
        const lope_u32 L = lbase + pz + w;
        const lope_u32 slot = L % NS;
        lope_mbar_wait(&full[slot], (L / NS) & 1);
        rd.sp[w] = reinterpret_cast<const T*>(lope_smem + slot * C::STAGE_BYTES) +
                   (row0 + Body::FN1) * C::BOXX + col + Body::FN0 + g.xshift;
      }
      T vals[RY];
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        LopeSmemReader<T, C::BOXX, NZW, FZN> rr;
#pragma unroll
        for (int w = 0; w < NZW; ++w) rr.sp[w] = rd.sp[w] + r * C::BOXX;
        T res[1];
        Body::template eval<T>(rr, sc.v, res);
        vals[r] = res[0];
      }
      // every smem read of this plane is done: release the oldest slot (and, at the
      // end of the unit, the trailing z-halo slots)
      __syncwarp();
      if (lane == 0) {
        lope_mbar_arrive(&empty[(lbase + pz) % NS]);
        if (pz == nz - 1)
          for (int w = 1; w < NZW; ++w) lope_mbar_arrive(&empty[(lbase + pz + w) % NS]);
      }
      if (!xok) continue;
      const int zg = z0 + pz + g.r0[2];
      const bool zw = (g.wrap & 4) && lope_near(zg, g.m[2], g.lo[2], g.hi[2]);
      const lope_i64 zimg = (zg < g.hi[2] ? (lope_i64)g.m[2] : -(lope_i64)g.m[2]) * s2;
      if (!(wy_any | zw) && simple) {
        // no y/z images in this warp-plane: plain stores, plus the x-image sector store
        // for the few boundary lanes
        if (!wx_any) {
#pragma unroll
          for (int r = 0; r < RY; ++r)
            if (ybase + r < g.ext[1]) orow[(lope_i64)r * s1] = vals[r];
        } else {
#pragma unroll
          for (int r = 0; r < RY; ++r)
            if (ybase + r < g.ext[1]) {
              orow[(lope_i64)r * s1] = vals[r];
#ifdef LOPE_XSAME
              if (xw) orow[(lope_i64)r * s1] = vals[r];
#else
              if (xw) orow[(lope_i64)r * s1 + ximg] = vals[r];
#endif
            }
        }
      } else if (simple) {
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          if (ybase + r >= g.ext[1]) continue;
          T* p = orow + (lope_i64)r * s1;
          const T v = vals[r];
          p[0] = v;
          if (xw) p[ximg] = v;
          const int yg = ybase + r + g.r0[1];
          const bool yw = (g.wrap & 2) && lope_near(yg, g.m[1], g.lo[1], g.hi[1]);
          if (yw | zw) {
            const lope_i64 yimg = (yg < g.hi[1] ? (lope_i64)g.m[1] : -(lope_i64)g.m[1]) * s1;
            if (yw) {
              p[yimg] = v;
              if (xw) p[yimg + ximg] = v;
            }
            if (zw) {
              p[zimg] = v;
              if (xw) p[zimg + ximg] = v;
              if (yw) {
                p[zimg + yimg] = v;
                if (xw) p[zimg + yimg + ximg] = v;
              }
            }
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < RY; ++r)
          if (ybase + r < g.ext[1]) {
            orow[(lope_i64)r * s1] = vals[r];
            lope_store_images<T>(a.out, s1, s2, org0, xg, ybase + r + g.r0[1], zg, g, vals[r]);
          }
      }
    }
    lbase += nz + NZW - 1;
  }
}
