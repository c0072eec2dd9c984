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
template <class T> __device__ __forceinline__ T lope_min(T a, T b);
template <class T> __device__ __forceinline__ T lope_max(T a, T b);
template <> struct LopeAr<float> {
  static __device__ __forceinline__ float c(float a) { return a; }
  static __device__ __forceinline__ float min_(float a, float b) { return lope_min<float>(a, b); }
  static __device__ __forceinline__ float max_(float a, float b) { return lope_max<float>(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float mulx(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float neg(float a) { return -a; }
  static __device__ __forceinline__ float abs_(float a) { return fabsf(a); }
  static __device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
  // x / b for a constant b with y = RN(1/b): q = RN(x*y) is within 1 ulp of x/b, the
  // FMA residual r = x - q*b is exact, and RN(q + r*y) is the correctly rounded
  // quotient (Markstein's theorem) -- same bits as the IEEE division, no divide
  // sequence.  Outside the range where neither q nor r can underflow or overflow
  // (and for 0, inf, NaN) it falls back to the IEEE division.  `ok` is false when
  // the host found b unsuitable (zero, non-finite, |b| outside [2^-16, 2^16]).
  // x / b for a kernel scalar b; y = RN(1/b) from the host, NaN when b is outside
  // the exact range (the point is then flagged and redone with the IEEE division)
  template <bool FAST>
  static __device__ __forceinline__ float divs(float x, float b, float y, bool& slow) {
    const float ax = fabsf(x);
    if (FAST) {
      const float q = __fmul_rn(x, y);
      const float r = __fmaf_rn(-q, b, x);
      const float m = __fmaf_rn(r, y, q);
      const bool special = !(ax > 0.0f && ax <= 0x1.fffffep+127f);
      slow |= (y != y) || (!special && !(ax >= 0x1p-90f && ax <= 0x1p+90f));
      return special ? q : m;
    }
    if (y == y && ax >= 0x1p-90f && ax <= 0x1p+90f) {
      const float q = __fmul_rn(x, y);
      const float r = __fmaf_rn(-q, b, x);
      return __fmaf_rn(r, y, q);
    }
    return __fdiv_rn(x, b);
  }
  template <bool FAST>
  static __device__ __forceinline__ float divc(float x, float b, double yf, double, bool ok, bool, bool& slow) {
    if (!ok) return __fdiv_rn(x, b);
    const float y = (float)yf;
    const float ax = fabsf(x);
    if (FAST) {
      // branch-free: 0 / inf / NaN give x*y (same bits as x/b); the tiny and huge
      // ranges are flagged and recomputed by the caller with the exact path
      const float q = __fmul_rn(x, y);
      const float r = __fmaf_rn(-q, b, x);
      const float m = __fmaf_rn(r, y, q);
      const bool special = !(ax > 0.0f && ax <= 0x1.fffffep+127f);
      slow |= !special && !(ax >= 0x1p-90f && ax <= 0x1p+90f);
      return special ? q : m;
    }
    if (ax >= 0x1p-90f && ax <= 0x1p+90f) {
      const float q = __fmul_rn(x, y);
      const float r = __fmaf_rn(-q, b, x);
      return __fmaf_rn(r, y, q);
    }
    return __fdiv_rn(x, b);
  }
};
template <> struct LopeAr<double> {
  static __device__ __forceinline__ double c(double a) { return a; }
  static __device__ __forceinline__ double min_(double a, double b) { return lope_min<double>(a, b); }
  static __device__ __forceinline__ double max_(double a, double b) { return lope_max<double>(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double mulx(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double neg(double a) { return -a; }
  static __device__ __forceinline__ double abs_(double a) { return fabs(a); }
  static __device__ __forceinline__ double sqrt_(double a) { return __dsqrt_rn(a); }
  // see LopeAr<float>::divc; the host requires |b| in [2^-60, 2^60]
  template <bool FAST>
  static __device__ __forceinline__ double divs(double x, double b, double y, bool& slow) {
    const double ax = fabs(x);
    if (FAST) {
      const double q = __dmul_rn(x, y);
      const double r = __fma_rn(-q, b, x);
      const double m = __fma_rn(r, y, q);
#ifdef LOPE_DIVC_INTCLASS
      bool inr, special;
      classify(x, inr, special);
      slow |= (y != y) || !(inr | special);
      return inr ? m : q;
#else
      const bool special = !(ax > 0.0 && ax <= 0x1.fffffffffffffp+1023);
      slow |= (y != y) || (!special && !(ax >= 0x1p-900 && ax <= 0x1p+900));
      return special ? q : m;
#endif
    }
    if (y == y && ax >= 0x1p-900 && ax <= 0x1p+900) {
      const double q = __dmul_rn(x, y);
      const double r = __fma_rn(-q, b, x);
      return __fma_rn(r, y, q);
    }
    return __ddiv_rn(x, b);
  }
  // Range classification of a dividend from its exponent bits, on the integer pipe:
  // the fp64 pipe (DSETP) is the one the stencil's adds saturate (config 4: 24 DADD per
  // point).  in_range: 2^-900 <= |x| < 2^900, where the FMA-corrected quotient is exact;
  // special: +-0, +-inf, NaN, where q = x*y already has IEEE division's bits.
  static __device__ __forceinline__ void classify(double x, bool& in_range, bool& special) {
    const unsigned hi = (unsigned)__double2hiint(x), lo = (unsigned)__double2loint(x);
    const unsigned e = (hi >> 20) & 0x7ffu;
    in_range = (e - 123u) <= 1798u;
    special = e == 0x7ffu || ((hi & 0x7fffffffu) | lo) == 0u;
  }
  template <bool FAST>
  static __device__ __forceinline__ double divc(double x, double b, double, double yd, bool, bool ok, bool& slow) {
    if (!ok) return __ddiv_rn(x, b);
    const double ax = fabs(x);
    if (FAST) {
      const double q = __dmul_rn(x, yd);
      const double r = __fma_rn(-q, b, x);
      const double m = __fma_rn(r, yd, q);
#ifdef LOPE_DIVC_INTCLASS
      bool inr, special;
      classify(x, inr, special);
      slow |= !(inr | special);
      return inr ? m : q;
#else
      const bool special = !(ax > 0.0 && ax <= 0x1.fffffffffffffp+1023);
      slow |= !special && !(ax >= 0x1p-900 && ax <= 0x1p+900);
      return special ? q : m;
#endif
    }
    if (ax >= 0x1p-900 && ax <= 0x1p+900) {
      const double q = __dmul_rn(x, yd);
      const double r = __fma_rn(-q, b, x);
      return __fma_rn(r, yd, q);
    }
    return __ddiv_rn(x, b);
  }
};
// numpy.minimum / numpy.maximum: NaN in either operand propagates; ties return the second.
template <class T> __device__ __forceinline__ T lope_min(T a, T b) { return (a != a || a < b) ? a : b; }
template <class T> __device__ __forceinline__ T lope_max(T a, T b) { return (a != a || a > b) ? a : b; }

// Two fp32 points per instruction (sm_100 FADD2 / FMUL2: two IEEE round-to-nearest
// results, subnormals kept -- the same bits as two FADD / FMUL).  Operations without
// a paired form run element by element through LopeAr<float>.
struct LopeAr2 {
  typedef float2 W;
  typedef LopeAr<float> S;
  static __device__ __forceinline__ W c(float a) { return make_float2(a, a); }
  // PTX add.rn.f32x2 (FADD2)
  static __device__ __forceinline__ W add(W a, W b) {
    W d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
  }
  static __device__ __forceinline__ W sub(W a, W b) {
    W d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
  }
  // Products stay scalar (two FMUL): ptxas contracts a paired multiply feeding a paired
  // add into FFMA2 even with an explicit .rn, which would change the rounding.
  static __device__ __forceinline__ W mul(W a, W b) { return make_float2(S::mul(a.x, b.x), S::mul(a.y, b.y)); }
  // an exact-looking product (power-of-two constant) as two scalar multiplies
  static __device__ __forceinline__ W mulx(W a, W b) { return make_float2(S::mul(a.x, b.x), S::mul(a.y, b.y)); }
  static __device__ __forceinline__ W div(W a, W b) { return make_float2(S::div(a.x, b.x), S::div(a.y, b.y)); }
  static __device__ __forceinline__ W neg(W a) { return make_float2(-a.x, -a.y); }
  static __device__ __forceinline__ W abs_(W a) { return make_float2(fabsf(a.x), fabsf(a.y)); }
  static __device__ __forceinline__ W sqrt_(W a) { return make_float2(S::sqrt_(a.x), S::sqrt_(a.y)); }
  static __device__ __forceinline__ W min_(W a, W b) { return make_float2(lope_min(a.x, b.x), lope_min(a.y, b.y)); }
  static __device__ __forceinline__ W max_(W a, W b) { return make_float2(lope_max(a.x, b.x), lope_max(a.y, b.y)); }
  template <bool FAST>
  static __device__ __forceinline__ W divs(W x, float b, float y, bool& slow) {
    return make_float2(S::template divs<FAST>(x.x, b, y, slow), S::template divs<FAST>(x.y, b, y, slow));
  }
  template <bool FAST>
  static __device__ __forceinline__ W divc(W x, W b, double yf, double yd, bool okf, bool okd, bool& slow) {
    return make_float2(S::template divc<FAST>(x.x, b.x, yf, yd, okf, okd, slow),
                       S::template divc<FAST>(x.y, b.x, yf, yd, okf, okd, slow));
  }
};

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
  int xshift;     // tiled: leading elements of the (vector-aligned) range outside the launch range
  int box0;       // tiled: TMA x coordinate of tile 0's box (row-relative, already shifted)
  int p1;         // tiled: padded rows per plane; > 0 selects the flattened 2-D tensor map
  int yband;      // tiled: tile rows per band of the unit walk (0: whole plane)
  int xexact;     // tiled: x images cell by cell (m[0] not a whole number of vectors / atoms)
  // Fused exchange: periodic images along the slowest dim go to another buffer --
  // the low / high neighbour's output block (NVLink peer memory under CUDA IPC) --
  // at this element offset from `out` (0: the image lives in this block's halo).
  lope_i64 sdl;   // images of the first `hi` planes (into the low neighbour's high halo)
  lope_i64 sdh;   // images of the last `lo` planes (into the high neighbour's low halo)
};

// --------------------------------------------------------------------------
// Periodic-image epilogue

template <class T>
__device__ __noinline__ void lope_store_images(T* __restrict__ out, lope_i64 s1, lope_i64 s2,
                                                  lope_i64 org0, int x, int y, int z,
                                                  const LopeGeom& g, T v, int rank = 3) {
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
        // slowest-dim images may belong to a neighbour's block (g.sdl / g.sdh)
        const int sc = rank == 3 ? c : (rank == 2 ? b : a);
        const lope_i64 dl = sc == 0 ? 0 : (sc == 1 ? g.sdl : g.sdh);
        if (cx && cy && cz) out[org0 + dl + (lope_i64)xx + (lope_i64)yy * s1 + (lope_i64)zz * s2] = v;
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
      bool slow = false;
      Body::template eval<T, false>(rd, sc.v, res, slow);
#pragma unroll
      for (int q = 0; q < Body::NSTORE; ++q) {
        const int A = Body::stored(q);
        T* o = arrs[A].out;
        o[rd.offs[A]] = res[q];
        if (xn | yn | zn) {
          const lope_i64 org0 = arrs[A].org - g.r0[0] - (lope_i64)g.r0[1] * arrs[A].s1 -
                                (lope_i64)g.r0[2] * arrs[A].s2;
          lope_store_images<T>(o, arrs[A].s1, arrs[A].s2, org0, i + g.r0[0], j + g.r0[1],
                               k + g.r0[2], g, res[q], Body::RANK);
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
// Waiting warps suspend (woken by the barrier's phase flip, at most this many ns)
// instead of re-polling: less issue activity under the board's power cap (measured
// sustained: lap3d7 1024^3 1.547 -> 1.524 ms, 2048^3 13.5 -> 13.1 ms).
#if !defined(LOPE_WAIT_HINT_NS) && !defined(LOPE_NO_WAIT_HINT)
#define LOPE_WAIT_HINT_NS 5000
#endif
__device__ __forceinline__ void lope_mbar_wait(lope_u64* bar, lope_u32 parity) {
  const lope_u32 addr = lope_smem_u32(bar);
  lope_u32 done = 0, n = 0;
  do {
#ifdef LOPE_WAIT_HINT_NS
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(done)
        : "r"(addr), "r"(parity), "n"(LOPE_WAIT_HINT_NS)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
#endif
#ifndef LOPE_NO_WAIT_TRAP
    if (++n > LOPE_WAIT_LIMIT) __trap();
#endif
  } while (!done);
}
// Non-blocking probe of a barrier phase (mbarrier.test_wait).
__device__ __forceinline__ bool lope_mbar_test(lope_u64* bar, lope_u32 parity) {
  lope_u32 done = 0;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(done)
      : "r"(lope_smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ void lope_tma_load_3d(void* dst, const LopeTmap* map, lope_u64* bar, int c0,
                                                 int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(lope_smem_u32(dst)),
      "l"((lope_u64)map), "r"(c0), "r"(c1), "r"(c2), "r"(lope_smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void lope_tma_load_2d(void* dst, const LopeTmap* map, lope_u64* bar, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(lope_smem_u32(dst)),
      "l"((lope_u64)map), "r"(c0), "r"(c1), "r"(lope_smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void lope_tma_prefetch_desc(const LopeTmap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"((lope_u64)map) : "memory");
}

// --------------------------------------------------------------------------
// Tiled TMA path (vector lanes)
//
// Each lane owns VX = 16/sizeof(T) consecutive x points (one 16-byte vector) and
// RY rows.  Per plane it loads the rows it needs from the staged box with 16-byte
// LDS plus scalar LDS for the x halo into a register window (entries the body
// never reads are dead code), evaluates the body VX*RY times from registers and
// writes 16-byte vectors straight to HBM.  Stencils that are a star in z (every
// read off the centre plane is at x = y = 0) keep the past planes in registers
// (ZHIST), so a plane iteration holds only the centre and future planes of the ring.

template <class T> struct LopeVec;
template <> struct LopeVec<float> { typedef float4 V; };
template <> struct LopeVec<double> { typedef double2 V; };


// --------------------------------------------------------------------------
// One lane's 16-byte output vector and the periodic images the fused epilogue owes
// (the HALO_TRANSFER fills of runtime.py:653-697 with neighbour == self; shared by the
// RAG tiled instantiation and the multi-array kernel).  x runs from the launch range's start rounded down
// to a whole vector: the first g.xshift cells and the cells past g.ext[0] are outside
// the range (ragged starts / extents store element by element).  When images are
// refreshed m[d] >= lo[d] + hi[d] (each halo cell has exactly one image); x images
// are whole 64-byte atoms (padding included; the layout reserves an atom per side)
// when m[0] is a multiple of the vector and >= 2 atoms, else cell by cell (g.xexact).
// y and z images are whole rows / planes; slowest-dim images may live in a
// neighbour's block (g.sdl / g.sdh: NVLink peer memory).

template <class T, int RANK>
struct LopeVecOut {
  typedef typename LopeVec<T>::V V;
  static constexpr int VX = 16 / (int)sizeof(T);
  static constexpr int SEC = 64 / (int)sizeof(T);     // one 64-byte DRAM atom
  static constexpr unsigned ALL = (1u << VX) - 1u;
  int xg, ximg;
  unsigned xm;       // bit e: element e lies inside the launch range
  bool xw;
  __device__ __forceinline__ void init(int x, bool xok, const LopeGeom& g) {
    xg = x + g.r0[0];
    xw = (g.wrap & 1) && xok &&
         (g.xexact ? (xg < g.hi[0] || xg + VX > g.m[0] - g.lo[0])
                   : ((g.hi[0] > 0 && xg < SEC) || (g.lo[0] > 0 && xg >= g.m[0] - SEC)));
    ximg = xg < SEC ? g.m[0] : -g.m[0];
    xm = 0;
#pragma unroll
    for (int e = 0; e < VX; ++e) xm |= (x + e >= g.xshift && x + e < g.ext[0]) ? (1u << e) : 0u;
  }
  // the vector itself (element stores only where it straddles an end of the range);
  // predicated stores, no branch: a branch here costs a convergence barrier pair per row
  __device__ __forceinline__ void put(T* p, const V& o) const {
    const bool full = xm == ALL;
    if (full) *reinterpret_cast<V*>(p) = o;
    const T* oe = reinterpret_cast<const T*>(&o);
#pragma unroll
    for (int e = 0; e < VX; ++e)
      if (!full && ((xm >> e) & 1u)) p[e] = oe[e];
  }
  // its x images (xw lanes only)
  __device__ __forceinline__ void putx(T* p, const V& o, const LopeGeom& g) const {
    if (!g.xexact) {
      *reinterpret_cast<V*>(p + ximg) = o;
    } else {
      const T* oe = reinterpret_cast<const T*>(&o);
#pragma unroll
      for (int e = 0; e < VX; ++e) {
        if (!((xm >> e) & 1u)) continue;
        if (xg + e < g.hi[0]) p[e + g.m[0]] = oe[e];
        if (xg + e >= g.m[0] - g.lo[0]) p[e - g.m[0]] = oe[e];
      }
    }
  }
  // the vector at p (row yg of the range, plane with z-image flag zw / offset zimg)
  // with every image: x, y, z and their combinations.  A rolled loop over the (up to
  // four) row targets keeps one copy of the store code: this path runs for boundary
  // rows and planes only, and the kernel's hot loop stays small in the i-cache.
  __device__ __forceinline__ void store_all(T* p, const V& o, int yg, bool zw, lope_i64 zimg, lope_i64 s1,
                                            const LopeGeom& g) const {
    const bool yw = (g.wrap & 2) && lope_near(yg, g.m[1], g.lo[1], g.hi[1]);
    // y images (rank 2: the slowest dim, possibly in a neighbour's block)
    const lope_i64 yimg = (yg < g.hi[1] ? (lope_i64)g.m[1] * s1 + (RANK == 2 ? g.sdl : 0)
                                        : -(lope_i64)g.m[1] * s1 + (RANK == 2 ? g.sdh : 0));
    const int nt = (yw | zw) ? 4 : 1;
#pragma unroll 1
    for (int t = 0; t < nt; ++t) {
      if (((t & 1) && !yw) || ((t & 2) && !zw)) continue;
      T* q = p + ((t & 1) ? yimg : 0) + ((t & 2) ? zimg : 0);
      put(q, o);
      if (xw) putx(q, o, g);
    }
  }
};

// --------------------------------------------------------------------------
// Rank-1 path (Machine._launch_vector, runtime.py:605-618, for rank-1 kernels such as
// corpus/avg3.lope; any number of arrays): each thread owns one 16-byte vector of every
// array (coalesced LDG.128 through the read-only path) and reads the x halo of its
// points with scalar loads that hit L1 (the neighbouring lanes' lines).  x runs from
// the range start rounded down to a whole vector; cells outside the launch range are
// computed and dropped.  Periodic images (lope_step) are stored cell by cell.

template <class T, int NA, int VX> struct LopeRowReader {
  const T* p[NA];      // this thread's first element in each array's snapshot
  const T* vec;        // [NA][VX] the thread's vectors
  int v;               // compile-time after unrolling
  template <int A, int DX, int DY, int DZ>
  __device__ __forceinline__ T at() const {
    if (v + DX >= 0 && v + DX < VX) return vec[A * VX + v + DX];
    return __ldg(p[A] + v + DX);
  }
};

template <class Body, class T, int NA>
__device__ __forceinline__ void lope_row_impl(const LopeArr<T>* arrs, const LopeScal<T>& sc, const LopeGeom& g) {
  typedef typename LopeVec<T>::V V;
  constexpr int VX = 16 / (int)sizeof(T);
  const int nvec = (g.ext[0] + VX - 1) / VX;
  // launched with programmatic dependent launch: wait for the previous kernel's writes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int vi = blockIdx.x * blockDim.x + threadIdx.x; vi < nvec; vi += gridDim.x * blockDim.x) {
    const int x = vi * VX;
    T vec[NA][VX];
    LopeRowReader<T, NA, VX> rd;
    rd.vec = &vec[0][0];
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      rd.p[a] = arrs[a].in + arrs[a].org + x;
      const V vv = __ldg(reinterpret_cast<const V*>(rd.p[a]));
      const T* ve = reinterpret_cast<const T*>(&vv);
#pragma unroll
      for (int e = 0; e < VX; ++e) vec[a][e] = ve[e];
    }
    T res[VX][Body::NSTORE > 0 ? Body::NSTORE : 1];
    // branch-free points (FAST constant division); a flagged operand redoes them exactly
    constexpr bool FAST = Body::HAS_DIVC;
    bool slow = false;
#pragma unroll
    for (int v = 0; v < VX; ++v) {
      rd.v = v;
      Body::template eval<T, FAST>(rd, sc.v, res[v], slow);
    }
    if (FAST && slow) {
#pragma unroll
      for (int v = 0; v < VX; ++v) {
        rd.v = v;
        bool dummy = false;
        Body::template eval<T, false>(rd, sc.v, res[v], dummy);
      }
    }
    const bool xfull = x >= g.xshift && x + VX <= g.ext[0];
    const int xg = x + g.r0[0];
    const bool img = (g.wrap & 1) && (xg < g.hi[0] || xg + VX > g.m[0] - g.lo[0]);
#pragma unroll
    for (int q = 0; q < Body::NSTORE; ++q) {
      const int A = Body::stored(q);
      T* o = arrs[A].out + arrs[A].org + x;
      if (xfull) {
        V ov;
        T* oe = reinterpret_cast<T*>(&ov);
#pragma unroll
        for (int e = 0; e < VX; ++e) oe[e] = res[e][q];
        *reinterpret_cast<V*>(o) = ov;
      } else {
#pragma unroll
        for (int e = 0; e < VX; ++e)
          if (x + e >= g.xshift && x + e < g.ext[0]) o[e] = res[e][q];
      }
      if (img) {
        // images of the first hi cells go to x+m (the low neighbour's block: sdl),
        // of the last lo cells to x-m (the high neighbour's: sdh)
#pragma unroll
        for (int e = 0; e < VX; ++e) {
          if (x + e < g.xshift || x + e >= g.ext[0]) continue;
          if (xg + e < g.hi[0]) o[e + g.m[0] + g.sdl] = res[e][q];
          if (xg + e >= g.m[0] - g.lo[0]) o[e - g.m[0] + g.sdh] = res[e][q];
        }
      }
    }
  }
}

template <class T, int NR, int NXW, int FZN, int FN0, int FN1, int RY, int VX, bool ZHIST>
struct LopeWinReader {
  const T* win;    // [NZW][NR][NXW] register window (flattened)
  const T* hist;   // [FZN][RY][VX] past planes at own points (ZHIST)
  int r, v;        // compile-time after unrolling
  template <int A, int DX, int DY, int DZ>
  __device__ __forceinline__ T at() const {
    if (ZHIST && DZ < 0) return hist[((-DZ - 1) * RY + r) * VX + v];
    return win[((DZ + FZN) * NR + (r + DY + FN1)) * NXW + (v + DX + FN0)];
  }
};

// The same window read as adjacent point pairs (v, v+1) for the paired fp32 evaluation.
template <class T, int NR, int NXW, int FZN, int FN0, int FN1, int RY, int VX, bool ZHIST>
struct LopeWinReader2 {
  const T* win;
  const T* hist;
  int r, v;        // v even
  template <int A, int DX, int DY, int DZ>
  __device__ __forceinline__ float2 at() const {
    if (ZHIST && DZ < 0) {
      const int h = ((-DZ - 1) * RY + r) * VX + v;
      return make_float2(hist[h], hist[h + 1]);
    }
    const int i = ((DZ + FZN) * NR + (r + DY + FN1)) * NXW + (v + DX + FN0);
    return make_float2(win[i], win[i + 1]);
  }
};
#ifndef LOPE_NO_PAIR
#define LOPE_PAIR 1
#else
#define LOPE_PAIR 0
#endif

// Reads the staged planes in shared memory directly (the exact re-evaluation of a
// plane whose fast evaluation flagged a slow-range division).
template <class T, int BOXX, int NZW, int FZN, int FN0, int FN1, int RY, int VX, bool ZHIST>
struct LopeSmemReader {
  const T* const* sp;  // [NZW] this lane's origin in each staged plane
  const T* hist;
  int r, v;
  template <int A, int DX, int DY, int DZ>
  __device__ __forceinline__ T at() const {
    if (ZHIST && DZ < 0) return hist[((-DZ - 1) * RY + r) * VX + v];
    return sp[DZ + FZN][(r + DY + FN1) * BOXX + v + DX];
  }
};

template <class Body, class T, int WX, int WY, int RY, int NS, int PW = 0>
struct LopeTiledCfg {
  static constexpr int VX = 16 / (int)sizeof(T);
  static constexpr int BX = 32 * VX * WX;
  static constexpr int BY = WY * RY;
  static constexpr int PADX = ((Body::FN0 + VX - 1) / VX) * VX;
  static constexpr int PADR = ((Body::FP0 + VX - 1) / VX) * VX;
  // A tile wider than one TMA box (256 elements) is staged as one box per warp column
  // (NB boxes side by side in a stage, each with its own x halo): 256-column fp32 tiles
  // halve the x-halo sectors per byte that neighbouring tiles must find in L2
  static constexpr int NB = (PADX + BX + PADR > 256) ? WX : 1;
  static constexpr int BXB = BX / NB;                  // interior columns per box
  static constexpr int BOXX = PADX + BXB + PADR;       // row pitch of a staged box
  static constexpr int BOXY = BY + Body::FN1 + Body::FP1;
  static constexpr int NZW = Body::FN2 + Body::FP2 + 1;
  static constexpr bool ZHIST = Body::ZSTAR && Body::FN2 > 0;
  static constexpr int HOLD = ZHIST ? Body::FP2 + 1 : NZW;     // slots one plane iteration holds
  static constexpr int BOX_BYTES = ((BOXX * BOXY * (int)sizeof(T) + 127) / 128) * 128;
  static constexpr int STAGE_BYTES = NB * BOX_BYTES;
  static constexpr int TX_BYTES = NB * BOXX * BOXY * (int)sizeof(T);
  static constexpr int SMEM_BYTES = NS * STAGE_BYTES + 2 * NS * 8;
  static constexpr int NCW = WX * WY;              // compute warps
  // PW = 1: a dedicated TMA producer warp; PW = 0: warp 0 lane 0 issues TMA in-band
  static constexpr int THREADS = 32 * (NCW + PW);
  static constexpr int NR = RY + Body::FN1 + Body::FP1;
  static constexpr int NXW = VX + Body::FN0 + Body::FP0;
};

__device__ __forceinline__ void lope_mbar_arrive(lope_u64* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(lope_smem_u32(bar)) : "memory");
}

// Division-free walk of the units u = b, b+G, b+2G, ... decomposed as
// u = tx + ntx*(ty + nty*zi).  x is fastest: the CTAs of one round read x- and
// y-neighbouring tiles at the same time, so the 128-byte lines tiles share at
// their edges (and the halo rows) are fetched from HBM once and hit in L2 for the
// neighbour.  The host picks G with G % ntx != 0 so x-edge tiles rotate over CTAs.
struct LopeUnitWalk {
  // Unit index -> (tx, ty, zi) in the mixed radix (tx: ntx, ty_lo: yb, zi: nzc,
  // ty_hi: nty/yb), x fastest.  yb = nty is the plain x-y-z order; a smaller band
  // puts the next z-chunk of a tile only ntx*yb units later (its halo planes are
  // still in L2) at the cost of y-halo reuse across band edges.  Advanced by the
  // grid stride with carries (no division per unit).
  int tx, tyl, zi, tyh, gtx, gtyl, gzi, gtyh, ntx, yb, nzc;
  __device__ __forceinline__ void init(int b, int G, int ntx_, int yb_, int nzc_) {
    ntx = ntx_; yb = yb_; nzc = nzc_;
    tx = b % ntx; int r = b / ntx; tyl = r % yb; r /= yb; zi = r % nzc; tyh = r / nzc;
    gtx = G % ntx; r = G / ntx; gtyl = r % yb; r /= yb; gzi = r % nzc; gtyh = r / nzc;
  }
  __device__ __forceinline__ int ty() const { return tyh * yb + tyl; }
  __device__ __forceinline__ void next() {
    tx += gtx;
    int c = 0;
    if (tx >= ntx) { tx -= ntx; c = 1; }
    tyl += gtyl + c;
    c = 0;
    if (tyl >= yb) { tyl -= yb; c = 1; }
    zi += gzi + c;
    c = 0;
    if (zi >= nzc) { zi -= nzc; c = 1; }
    tyh += gtyh + c;
  }
};

template <class Body, class T, int WX, int WY, int RY, int NS, int PW = 0, int SH = 0, int NB = 0, bool RAG = false>
__device__ __forceinline__ void lope_tiled_impl(const LopeTmap* map, const LopeArr<T>& a,
                                                const LopeScal<T>& sc, const LopeGeom& g) {
  typedef LopeTiledCfg<Body, T, WX, WY, RY, NS, PW> C;
  typedef typename LopeVec<T>::V V;
  constexpr int VX = C::VX;
  constexpr int FZN = Body::FN2, FZP = Body::FP2;
  constexpr int NZW = C::NZW, NR = C::NR, NXW = C::NXW;
  constexpr bool ZHIST = C::ZHIST;
  static_assert(NS >= C::HOLD + 1, "ring must hold the planes in use plus one prefetch slot");
  static_assert(C::BOXX <= 256 && C::BOXY <= 256, "TMA box dimensions are limited to 256");
  extern __shared__ __align__(128) unsigned char lope_smem[];
  lope_u64* full = reinterpret_cast<lope_u64*>(lope_smem + NS * C::STAGE_BYTES);
  lope_u64* empty = full + NS;

  // Rank 2 streams along y (YS): a unit is an x tile and `zchunk` consecutive y tiles
  // (each one "plane" of the ring: its box re-reads the tile's y halo rows), so the
  // per-unit setup is paid once per chunk instead of once per tile (c4: 3.83 -> 3.14
  // ms).  Rank 3 streams along z.  Everything YS / RAG adds is compile-time gated: the
  // aligned rank-3 instantiation is instruction for instruction the round-1 kernel
  // (measured: any extra live state in the plane loop costs 10-15% on config 3).
  constexpr bool YS = Body::RANK == 2;
  const int ntx = (g.ext[0] + C::BX - 1) / C::BX;
  const int nty = (g.ext[1] + C::BY - 1) / C::BY;
  const int zc = g.zchunk;
  const int nyu = YS ? (nty + zc - 1) / zc : nty;          // y units per x tile column
  const int nzc = YS ? 1 : (g.ext[2] + zc - 1) / zc;
  const int nunits = ntx * nyu * nzc;     // < 2^31 (host checks)
  const int yb = (g.yband > 0 && nyu % g.yband == 0) ? g.yband : nyu;

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
  // Programmatic dependent launch: let the next step's grid be scheduled now, and
  // wait for the previous kernel's writes before the first global access (both are
  // no-ops for a plain launch).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();

  // ---------------- TMA producer state (warp 0, lane 0) ----------------
  // The producer runs inside compute warp 0 (a 16-warp CTA keeps the 128-register
  // budget; a 17th warp would drop it to 96 and spill).  Before each plane it tops the
  // ring up to NS loads past the oldest slot warp 0 still holds, waiting on a slot's
  // `empty` barrier when a slower warp still reads it.  No deadlock: every load a warp
  // can be waiting for has already been issued.
  LopeUnitWalk pw;
  int p_u = blockIdx.x, p_pl = 0, p_nl = 0, p_bx = 0, p_by = 0, p_z = 0;
  lope_u32 p_L = 0;
  const int oy = g.lo[1] + g.r0[1] - Body::FN1;
  const int oz = g.lo[2] + g.r0[2] - FZN;
  const int pwarp = PW ? C::NCW : 0;     // the warp that issues TMA
  if (warp == pwarp && lane == 0) {
    pw.init(blockIdx.x, gridDim.x, ntx, yb, nzc);
    if (p_u < nunits) {
      const int z0 = pw.zi * zc;
      p_nl = YS ? min(zc, nty - pw.ty() * zc) : min(zc, g.ext[2] - z0) + NZW - 1;
      p_bx = g.box0 + pw.tx * C::BX;
      p_by = oy + (YS ? pw.ty() * zc : pw.ty()) * C::BY;
      p_z = oz + z0;
    }
  }
  // Loads below `needed` are waited for (the issuing warp reads them next); loads up to
  // `limit` are prefetch and only issued while their slot is already free, so the
  // in-band producer never stalls warp 0 on a slower warp just to run further ahead.
  auto produce = [&](lope_u32 needed, lope_u32 limit) {
    while (p_L < limit && p_u < nunits) {
      const lope_u32 slot = p_L % NS;
      if (p_L >= (lope_u32)NS) {
        const lope_u32 par = ((p_L / NS) - 1) & 1;
        if (p_L < needed) lope_mbar_wait(&empty[slot], par);
        else if (!lope_mbar_test(&empty[slot], par)) break;
      }
      lope_mbar_expect_tx(&full[slot], C::TX_BYTES);
#pragma unroll
      for (int h = 0; h < C::NB; ++h) {
        unsigned char* dst = lope_smem + slot * C::STAGE_BYTES + h * C::BOX_BYTES;
        const int bx = p_bx + h * C::BXB;
        if constexpr (YS) {
          // rank 2: the unit's planes are consecutive y tiles
          if (g.p1 > 0)
            lope_tma_load_2d(dst, map, &full[slot], bx, p_by + p_pl * C::BY + p_z * g.p1);
          else
            lope_tma_load_3d(dst, map, &full[slot], bx, p_by + p_pl * C::BY, p_z);
        } else {
          if (g.p1 > 0)
            lope_tma_load_2d(dst, map, &full[slot], bx, p_by + (p_z + p_pl) * g.p1);
          else
            lope_tma_load_3d(dst, map, &full[slot], bx, p_by, p_z + p_pl);
        }
      }
      ++p_L;
      if (++p_pl == p_nl) {
        p_pl = 0;
        p_u += gridDim.x;
        pw.next();
        if (p_u < nunits) {
          const int z0 = pw.zi * zc;
          p_nl = YS ? min(zc, nty - pw.ty() * zc) : min(zc, g.ext[2] - z0) + NZW - 1;
          p_bx = g.box0 + pw.tx * C::BX;
          p_by = oy + (YS ? pw.ty() * zc : pw.ty()) * C::BY;
          p_z = oz + z0;
        }
      }
    }
  };

  if (PW && warp == C::NCW) {
    // dedicated producer warp: issue everything, slot by slot
    if (lane == 0) produce(0xffffffffu, 0xffffffffu);
    return;
  }

  // ---------------- compute warps ----------------
  const int wx = warp % WX;
  const int wy = warp / WX;
  const int cx = (wx * 32 + lane) * VX;    // first column of this lane within the tile
  const int row0 = wy * RY;                // first row within the tile
  const lope_i64 s1 = a.s1, s2 = a.s2;
  constexpr int SEC = 64 / (int)sizeof(T);          // one 64-byte DRAM atom
  // The host sends only geometries with ext[0] % VX == 0 and, when images are
  // refreshed, m[0] >= 2*SEC, m[0] % VX == 0 and m[d] >= lo[d] + hi[d] (each halo
  // cell has exactly one image); anything else runs on the generic kernel.
  // this lane's offset in a stage (elements): its warp column's box, then row and column
  const int soff = C::NB > 1 ? wx * (C::BOX_BYTES / (int)sizeof(T)) + row0 * C::BOXX + C::PADX + lane * VX
                             : (row0 * C::BOXX + C::PADX + cx);

  LopeUnitWalk w;
  w.init(blockIdx.x, gridDim.x, ntx, yb, nzc);
  lope_u32 lbase = 0;
  T hist[FZN > 0 ? FZN : 1][RY][VX];
  for (int u = blockIdx.x; u < nunits; u += gridDim.x, w.next()) {
    const int z0 = w.zi * zc;
    const int nz = YS ? min(zc, nty - w.ty() * zc) : min(zc, g.ext[2] - z0);
    const int x = w.tx * C::BX + cx;
    const int ybase = (YS ? w.ty() * zc : w.ty()) * C::BY + row0;
    const bool xok = x < g.ext[0];
    const int nrow = min(RY, g.ext[1] - ybase);
    // Periodic images (lope_step): x images are whole 64-byte atoms written by the
    // lanes whose vectors land in the halo atom (padding included; the layout
    // reserves an atom per side), y and z images are whole rows / planes.
    const int xg = x + g.r0[0];
    const bool xw = (g.wrap & 1) && xok && ((g.hi[0] > 0 && xg < SEC) || (g.lo[0] > 0 && xg >= g.m[0] - SEC));
    const int ximg = xg < SEC ? g.m[0] : -g.m[0];
    const bool wx_any = __any_sync(0xffffffffu, xw);
    const bool wy_any = (g.wrap & 2) && (nrow > 0) &&
                        (lope_near(ybase + g.r0[1], g.m[1], g.lo[1], g.hi[1]) ||
                         lope_near(ybase + nrow - 1 + g.r0[1], g.m[1], g.lo[1], g.hi[1]));
    T* orow = a.out + a.org + x + (lope_i64)ybase * s1 + (lope_i64)z0 * s2;
    bool rag_plain = false;
    if constexpr (RAG) {
      LopeVecOut<T, Body::RANK> v0;
      v0.init(x, xok, g);
      rag_plain = __all_sync(0xffffffffu, !v0.xw && (!xok || v0.xm == v0.ALL));
    }
    auto plane = [&](const int pz, T* orow, const int ybase, const int nrow, const bool wy_any) {
      // ---- top up the TMA ring (warp 0 lane 0) ----
      if (!PW && warp == 0) {
        if (lane == 0)
          produce(NB ? lbase + pz + NZW : 0xffffffffu,
                  (ZHIST ? (pz == 0 ? lbase : lbase + pz + FZN) : lbase + pz) + NS);
        __syncwarp();
      }
      // ---- wait for the planes this iteration reads ----
      const T* sp[NZW];
#ifdef LOPE_SLOT_INC
      // one division per plane: the window's slots follow the first one
      const lope_u32 L0 = lbase + pz;
      const lope_u32 s0 = L0 % NS, q0 = L0 / NS;
#endif
#pragma unroll
      for (int k = 0; k < NZW; ++k) {
        const lope_u32 L = lbase + pz + k;
#ifdef LOPE_SLOT_INC
        const lope_u32 sl = s0 + k >= (lope_u32)NS ? s0 + k - NS : s0 + k;
        const lope_u32 ph = (s0 + k >= (lope_u32)NS ? q0 + 1 : q0) & 1;
        sp[k] = reinterpret_cast<const T*>(lope_smem + sl * C::STAGE_BYTES) + soff;
#else
        sp[k] = reinterpret_cast<const T*>(lope_smem + (L % NS) * C::STAGE_BYTES) + soff;
#endif
#ifdef LOPE_SLIDE_WAIT
        // after the unit's first plane only the newest plane is new: the others were
        // waited for by an earlier plane and a slot is not refilled while this warp holds it
        if (pz > 0 && k < NZW - 1) continue;
#else
        if (ZHIST && k < FZN && pz > 0) continue;          // past planes come from registers
#endif
#ifdef LOPE_SLOT_INC
        (void)L;
        lope_mbar_wait(&full[sl], ph);
#else
        lope_mbar_wait(&full[L % NS], (L / NS) & 1);
#endif
      }
      if (ZHIST && pz == 0) {
        // history for the first plane of the unit: planes z0-1 .. z0-FZN at own points
#pragma unroll
        for (int d = 0; d < FZN; ++d) {
          const lope_u32 L = lbase + (FZN - 1 - d);
          lope_mbar_wait(&full[L % NS], (L / NS) & 1);
#pragma unroll
          for (int r = 0; r < RY; ++r) {
            const V vv = *reinterpret_cast<const V*>(sp[FZN - 1 - d] + (Body::FN1 + r) * C::BOXX);
            const T* ve = reinterpret_cast<const T*>(&vv);
#pragma unroll
            for (int e = 0; e < VX; ++e) hist[d][r][e] = ve[e];
          }
        }
      }
      // ---- register window, filled row by row and consumed as soon as a row of
      // outputs has all its inputs (short live ranges: no spills at 16 warps) ----
      T win[NZW][NR][NXW];
      T vals[RY][VX];
      bool slow = false;
      constexpr bool FAST = Body::HAS_DIVC;    // branch-free points, exact redo below
#pragma unroll
      for (int q = 0; q < NR; ++q) {
#pragma unroll
        for (int k = 0; k < NZW; ++k) {
          if (ZHIST && k < FZN) continue;
          const T* rp = sp[k] + q * C::BOXX;
          const V vv = *reinterpret_cast<const V*>(rp);
          const T* ve = reinterpret_cast<const T*>(&vv);
#pragma unroll
          for (int e = 0; e < VX; ++e) win[k][q][Body::FN0 + e] = ve[e];
          // x halo: with SH the neighbouring lanes' vectors supply those columns (warp
          // shuffles, no bank conflicts; only the warp's edge lanes read shared memory) --
          // a plan parameter: it moves the timing of the short-z-chunk plans out of their
          // slow mode (1.86 -> 1.41 ms) but costs the in-band plan 12% (1.51 -> 1.69 ms)
#pragma unroll
          for (int e = 1; e <= Body::FN0; ++e) {
            T hv;
            // one-column halos in fp32 only: wider ones (5x5 box) spill with the shuffles
            if (SH && sizeof(T) == 4 && Body::FN0 <= 1 && Body::FP0 <= 1) {
              hv = __shfl_up_sync(0xffffffffu, ve[VX - e], 1);
              if (lane == 0) hv = rp[-e];
            } else {
              hv = rp[-e];
            }
            win[k][q][Body::FN0 - e] = hv;
          }
#pragma unroll
          for (int e = 0; e < Body::FP0; ++e) {
            T hv;
            if (SH && sizeof(T) == 4 && Body::FN0 <= 1 && Body::FP0 <= 1) {
              hv = __shfl_down_sync(0xffffffffu, ve[e], 1);
              if (lane == 31) hv = rp[VX + e];
            } else {
              hv = rp[VX + e];
            }
            win[k][q][Body::FN0 + VX + e] = hv;
          }
        }
        const int r = q - Body::FN1 - Body::FP1;
        if (r >= 0) {
#pragma unroll
          for (int v = 0; v < VX; ++v) {
            LopeWinReader<T, NR, NXW, FZN, Body::FN0, Body::FN1, RY, VX, ZHIST> rd;
            rd.win = &win[0][0][0];
            rd.hist = &hist[0][0][0];
            rd.r = r;
            rd.v = v;
            T res[1];
            Body::template eval<T, FAST>(rd, sc.v, res, slow);
            vals[r][v] = res[0];
          }
          if (ZHIST && !FAST) {
            // row r of the history only feeds row r: shift it now
#pragma unroll
            for (int d = FZN - 1; d > 0; --d)
#pragma unroll
              for (int e = 0; e < VX; ++e) hist[d][r][e] = hist[d - 1][r][e];
#pragma unroll
            for (int e = 0; e < VX; ++e) hist[0][r][e] = win[FZN][Body::FN1 + r][Body::FN0 + e];
          }
        }
      }
      if (FAST) {
        if (slow) {
          // a division operand fell outside the fast range: redo this lane's points
          // with the exact (branching) evaluation, straight from shared memory
#pragma unroll
          for (int r = 0; r < RY; ++r) {
#pragma unroll
            for (int v = 0; v < VX; ++v) {
              LopeSmemReader<T, C::BOXX, NZW, FZN, Body::FN0, Body::FN1, RY, VX, ZHIST> rd;
              rd.sp = sp;
              rd.hist = &hist[0][0][0];
              rd.r = r;
              rd.v = v;
              T res[1];
              bool dummy = false;
              Body::template eval<T, false>(rd, sc.v, res, dummy);
              vals[r][v] = res[0];
            }
          }
        }
        if (ZHIST) {
#pragma unroll
          for (int r = 0; r < RY; ++r) {
#pragma unroll
            for (int d = FZN - 1; d > 0; --d)
#pragma unroll
              for (int e = 0; e < VX; ++e) hist[d][r][e] = hist[d - 1][r][e];
            const V cv = *reinterpret_cast<const V*>(sp[FZN] + (Body::FN1 + r) * C::BOXX);
            const T* ce = reinterpret_cast<const T*>(&cv);
#pragma unroll
            for (int e = 0; e < VX; ++e) hist[0][r][e] = ce[e];
          }
        }
      }
      // ---- release the slots no later plane of this unit needs ----
      __syncwarp();
      if (lane == 0) {
        if (ZHIST) {
          if (pz == 0)
            for (int k = 0; k < FZN; ++k) lope_mbar_arrive(&empty[(lbase + k) % NS]);
          lope_mbar_arrive(&empty[(lbase + pz + FZN) % NS]);
          if (pz == nz - 1)
            for (int k = 1; k <= FZP; ++k) lope_mbar_arrive(&empty[(lbase + pz + FZN + k) % NS]);
        } else {
          lope_mbar_arrive(&empty[(lbase + pz) % NS]);
          if (pz == nz - 1)
            for (int k = 1; k < NZW; ++k) lope_mbar_arrive(&empty[(lbase + pz + k) % NS]);
        }
      }
      if (!xok || nrow <= 0) return;
      // ---- store ----
      if constexpr (RAG) {
        // ragged x (range start or extent not whole vectors, or cell-by-cell x images):
        // tiles whose lanes all hold whole in-range vectors and no x image store plainly
        // (warp-uniform `rag_plain`, set per unit); the others mask their edge vectors
        // and store every image through LopeVecOut
        const int zg = z0 + pz + g.r0[2];
        const bool zw = (g.wrap & 4) && lope_near(zg, g.m[2], g.lo[2], g.hi[2]);
        if (rag_plain && !(wy_any | zw)) {
#pragma unroll
          for (int r = 0; r < RY; ++r) {
            if (r >= nrow) continue;
            V o;
            T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
            for (int e = 0; e < VX; ++e) oe[e] = vals[r][e];
            *reinterpret_cast<V*>(orow + (lope_i64)r * s1) = o;
          }
        } else if (!(wy_any | zw)) {
          // x-edge tiles off the y/z boundary: masked vectors and their x images
          LopeVecOut<T, Body::RANK> vo;
          vo.init(x, xok, g);
#pragma unroll
          for (int r = 0; r < RY; ++r) {
            if (r >= nrow) continue;
            V o;
            T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
            for (int e = 0; e < VX; ++e) oe[e] = vals[r][e];
            vo.put(orow + (lope_i64)r * s1, o);
            if (vo.xw) vo.putx(orow + (lope_i64)r * s1, o, g);
          }
        } else {
          LopeVecOut<T, Body::RANK> vo;
          vo.init(x, xok, g);
          const lope_i64 zimg = (zg < g.hi[2] ? (lope_i64)g.m[2] * s2 + g.sdl : -(lope_i64)g.m[2] * s2 + g.sdh);
#pragma unroll
          for (int r = 0; r < RY; ++r) {
            if (r >= nrow) continue;
            V o;
            T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
            for (int e = 0; e < VX; ++e) oe[e] = vals[r][e];
            vo.store_all(orow + (lope_i64)r * s1, o, ybase + r + g.r0[1], zw, zimg, s1, g);
          }
        }
      } else {
        const int zg = z0 + pz + g.r0[2];
        const bool zw = (g.wrap & 4) && lope_near(zg, g.m[2], g.lo[2], g.hi[2]);
        if (!(wy_any | zw)) {
  #pragma unroll
          for (int r = 0; r < RY; ++r) {
            if (r >= nrow) continue;
            V o;
            T* oe = reinterpret_cast<T*>(&o);
  #pragma unroll
            for (int e = 0; e < VX; ++e) oe[e] = vals[r][e];
            *reinterpret_cast<V*>(orow + (lope_i64)r * s1) = o;
            if (wx_any && xw) *reinterpret_cast<V*>(orow + (lope_i64)r * s1 + ximg) = o;
          }
        } else {
          // z images (rank 3: the slowest dim, possibly in a neighbour's block)
          const lope_i64 zimg = (zg < g.hi[2] ? (lope_i64)g.m[2] * s2 + g.sdl : -(lope_i64)g.m[2] * s2 + g.sdh);
  #pragma unroll
          for (int r = 0; r < RY; ++r) {
            if (r >= nrow) continue;
            V o;
            T* oe = reinterpret_cast<T*>(&o);
  #pragma unroll
            for (int e = 0; e < VX; ++e) oe[e] = vals[r][e];
            T* p = orow + (lope_i64)r * s1;
            *reinterpret_cast<V*>(p) = o;
            if (xw) *reinterpret_cast<V*>(p + ximg) = o;
            const int yg = ybase + r + g.r0[1];
            const bool yw = (g.wrap & 2) && lope_near(yg, g.m[1], g.lo[1], g.hi[1]);
            if (yw | zw) {
              // y images (rank 2: the slowest dim, possibly in a neighbour's block)
              const lope_i64 yimg = (yg < g.hi[1] ? (lope_i64)g.m[1] * s1 + (Body::RANK == 2 ? g.sdl : 0)
                                                  : -(lope_i64)g.m[1] * s1 + (Body::RANK == 2 ? g.sdh : 0));
              if (yw) {
                *reinterpret_cast<V*>(p + yimg) = o;
                if (xw) *reinterpret_cast<V*>(p + yimg + ximg) = o;
              }
              if (zw) {
                *reinterpret_cast<V*>(p + zimg) = o;
                if (xw) *reinterpret_cast<V*>(p + zimg + ximg) = o;
                if (yw) {
                  *reinterpret_cast<V*>(p + zimg + yimg) = o;
                  if (xw) *reinterpret_cast<V*>(p + zimg + yimg + ximg) = o;
                }
              }
            }
          }
        }
      }
    };
    if constexpr (YS) {
      for (int pz = 0; pz < nz; ++pz) {
        const int yb_ = ybase + pz * C::BY;
        const int nr_ = min(RY, g.ext[1] - yb_);
        const bool wya = (g.wrap & 2) && (nr_ > 0) &&
                         (lope_near(yb_ + g.r0[1], g.m[1], g.lo[1], g.hi[1]) ||
                          lope_near(yb_ + nr_ - 1 + g.r0[1], g.m[1], g.lo[1], g.hi[1]));
        plane(pz, orow + (lope_i64)pz * C::BY * s1, yb_, nr_, wya);
      }
    } else {
#ifdef LOPE_UNROLL2
#pragma unroll 2
#endif
      for (int pz = 0; pz < nz; ++pz, orow += s2) plane(pz, orow, ybase, nrow, wy_any);
    }
    lbase += nz + NZW - 1;
  }
}



// --------------------------------------------------------------------------
// Temporal blocking (rank 2, one array, every dim periodic): TT fused steps per
// launch for fields that live in L2 (config 1), where a launch costs more than its
// arithmetic.  Each CTA loads its tile plus TT footprints of halo (periodic indices
// straight from the interior), advances it TT steps in shared memory -- the valid
// region shrinking by one footprint per step -- and stores the last step's tile and
// its periodic images.  Every point is evaluated with the same expression on the
// same operands as the one-step kernel, so the bits are identical.

template <class Body, class T, int TX, int TY, int TT>
struct LopeTblockCfg {
  static constexpr int VX = 16 / (int)sizeof(T);           // one 16-byte vector per lane
  static constexpr int RY = 4;                              // rows per lane
  static constexpr int WI = TX + TT * (Body::FN0 + Body::FP0);   // valid input columns
  static constexpr int HI = TY + TT * (Body::FN1 + Body::FP1);   // valid input rows
  static constexpr int PX = 4;                              // pad columns (>= footprint, vector aligned)
  static constexpr int PY = (Body::FN1 > Body::FP1 ? Body::FN1 : Body::FP1);
  static constexpr int NGX = (WI + VX - 1) / VX;            // vector groups per row
  static constexpr int NGY = (HI + RY - 1) / RY;            // row groups
  static constexpr int WB = NGX * VX + 2 * PX;              // buffer row pitch (elements)
  static constexpr int HB = NGY * RY + 2 * PY;
  static constexpr int THREADS = ((NGX * NGY + 31) / 32) * 32 > 1024 ? 1024 : ((NGX * NGY + 31) / 32) * 32;
  static constexpr int SMEM_BYTES = 2 * WB * HB * (int)sizeof(T);
};

// Temporal blocking (rank 2, one array, every dim periodic): TT fused steps per
// launch for fields that live in L2 (config 1), where a launch costs more than its
// arithmetic.  Each CTA loads its tile plus TT footprints of halo (periodic indices
// straight from the interior) into shared memory and advances it TT steps there --
// the valid region shrinking by one footprint per step -- with the tiled kernel's
// lane shape: a 16-byte vector of columns x 4 rows per lane, neighbours from a
// register window filled by 16-byte loads.  Points outside the valid region are
// computed from stale cells and never read by a valid point.  The last step stores
// the tile and its periodic images.  Same expression on the same operands per point
// as the one-step kernel, so the bits are identical.
template <class Body, class T, int TX, int TY, int TT>
__device__ __forceinline__ void lope_tblock_impl(const LopeArr<T>& a, const LopeScal<T>& sc, const LopeGeom& g) {
  typedef LopeTblockCfg<Body, T, TX, TY, TT> C;
  typedef typename LopeVec<T>::V V;
  constexpr int FN0 = Body::FN0, FP0 = Body::FP0, FN1 = Body::FN1, FP1 = Body::FP1;
  constexpr int VX = C::VX, RY = C::RY, WI = C::WI, HI = C::HI, WB = C::WB, PX = C::PX, PY = C::PY;
  constexpr int NR = RY + FN1 + FP1, NXW = VX + FN0 + FP0;
  static_assert(FN0 <= PX && FP0 <= PX, "x footprint wider than the buffer pad");
  static_assert((TT * FN0) % VX == 0, "the last step's tile must start on a vector");
  extern __shared__ __align__(16) unsigned char lope_smem[];
  T* b0 = reinterpret_cast<T*>(lope_smem);
  T* b1 = b0 + WB * C::HB;
  const int m0 = g.m[0], m1 = g.m[1];
  const int ntx = (m0 + TX - 1) / TX;
  const int tx = blockIdx.x % ntx, ty = blockIdx.x / ntx;
  const int x0 = tx * TX - TT * FN0, y0 = ty * TY - TT * FN1;   // interior coords of valid cell (0,0)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // ---- load: tile + TT halos, periodic (the host guarantees one wrap suffices) ----
  // 16-byte vectors: x0 and the interior width are multiples of VX (host), so a vector
  // never straddles the periodic seam and wraps as a whole; all of a lane's loads are
  // issued before the first shared store
  {
    constexpr int NV = C::NGX * HI;
    constexpr int NLD = (NV + C::THREADS - 1) / C::THREADS;
    V v[NLD];
#pragma unroll
    for (int k = 0; k < NLD; ++k) {
      const int p = threadIdx.x + k * C::THREADS;
      if (p < NV) {
        const int gx = p % C::NGX, by = p / C::NGX;
        int x = x0 + gx * VX, y = y0 + by;
        x += x < 0 ? m0 : (x >= m0 ? -m0 : 0);
        y += y < 0 ? m1 : (y >= m1 ? -m1 : 0);
        v[k] = __ldg(reinterpret_cast<const V*>(a.in + a.org + x + (lope_i64)y * a.s1));
      }
    }
#pragma unroll
    for (int k = 0; k < NLD; ++k) {
      const int p = threadIdx.x + k * C::THREADS;
      if (p < NV) {
        const int gx = p % C::NGX, by = p / C::NGX;
        *reinterpret_cast<V*>(b0 + (by + PY) * WB + gx * VX + PX) = v[k];
      }
    }
  }
  __syncthreads();
  const bool wxm = g.wrap & 1, wym = (g.wrap >> 1) & 1;
#pragma unroll 1
  for (int s = 1; s <= TT; ++s) {
    const T* src = (s & 1) ? b0 : b1;
    T* dst = (s & 1) ? b1 : b0;
    // lanes cover the vector groups / row groups that intersect this step's valid region
    const int gx0 = (s * FN0) / VX, gx1 = (WI - s * FP0 + VX - 1) / VX;
    const int gy0 = (s * FN1) / RY, gy1 = (HI - s * FP1 + RY - 1) / RY;
    const int ngx = gx1 - gx0, ntask = ngx * (gy1 - gy0);
    const int lane = threadIdx.x & 31;
    // warp-uniform trip count (blockDim.x is a multiple of 32): every lane of a warp runs
    // every iteration, so the full-mask shuffles below always see all 32 lanes; lanes
    // past the last task compute a copy of it and store nothing
    for (int t0 = threadIdx.x - lane; t0 < ntask; t0 += blockDim.x) {
      const int tl = t0 + lane;
      const bool act = tl < ntask;
      const int t = act ? tl : ntask - 1;
      const int gxi = t % ngx;
      const int bx = (gx0 + gxi) * VX, by = (gy0 + t / ngx) * RY;
      const T* base = src + (by + PY) * WB + bx + PX;
      // the x halo comes from the neighbouring lane unless that lane holds another row,
      // belongs to another warp or has no task of its own
      constexpr unsigned am = 0xffffffffu;
      const bool own_l = lane == 0 || gxi == 0 || !act;
      const bool own_r = lane == 31 || gxi == ngx - 1 || tl + 1 >= ntask;
      T win[1][NR][NXW];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const T* rp = base + (q - FN1) * WB;
        const V vv = *reinterpret_cast<const V*>(rp);
        const T* ve = reinterpret_cast<const T*>(&vv);
#pragma unroll
        for (int e = 0; e < VX; ++e) win[0][q][FN0 + e] = ve[e];
#pragma unroll
        for (int e = 1; e <= FN0; ++e) {
          T hv;
          if (FN0 <= VX) {
            hv = __shfl_up_sync(am, ve[VX - e], 1);
            if (own_l) hv = rp[-e];
          } else {
            hv = rp[-e];
          }
          win[0][q][FN0 - e] = hv;
        }
#pragma unroll
        for (int e = 0; e < FP0; ++e) {
          T hv;
          if (FP0 <= VX) {
            hv = __shfl_down_sync(am, ve[e], 1);
            if (own_r) hv = rp[VX + e];
          } else {
            hv = rp[VX + e];
          }
          win[0][q][FN0 + VX + e] = hv;
        }
      }
      T vals[RY][VX];
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        if (LOPE_PAIR && sizeof(T) == 4) {
#pragma unroll
          for (int v = 0; v < VX; v += 2) {
            LopeWinReader2<T, NR, NXW, 0, FN0, FN1, RY, VX, false> rd;
            rd.win = &win[0][0][0];
            rd.hist = nullptr;
            rd.r = r;
            rd.v = v;
            float2 res[1];
            bool slow = false;
            Body::template eval<T, false, decltype(rd), float2, LopeAr2>(rd, sc.v, res, slow);
            vals[r][v] = res[0].x;
            vals[r][v + 1] = res[0].y;
          }
        } else {
#pragma unroll
          for (int v = 0; v < VX; ++v) {
            LopeWinReader<T, NR, NXW, 0, FN0, FN1, RY, VX, false> rd;
            rd.win = &win[0][0][0];
            rd.hist = nullptr;
            rd.r = r;
            rd.v = v;
            T res[1];
            bool slow = false;
            Body::template eval<T, false>(rd, sc.v, res, slow);
            vals[r][v] = res[0];
          }
        }
      }
      if (!act) continue;
      if (s < TT) {
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          V o;
          T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
          for (int e = 0; e < VX; ++e) oe[e] = vals[r][e];
          *reinterpret_cast<V*>(dst + (by + r + PY) * WB + bx + PX) = o;
        }
      } else {
        // the tile itself: interior stores plus the periodic images of boundary cells
        const int x = x0 + bx;
        if (bx < TT * FN0 || bx >= TT * FN0 + TX || x >= m0) continue;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          const int yb = by + r, y = y0 + yb;
          if (yb < TT * FN1 || yb >= TT * FN1 + TY || y >= m1) continue;
          T* orow = a.out + a.org + (lope_i64)y * a.s1;
          const bool yh = wym && y < g.hi[1], yl = wym && y >= m1 - g.lo[1];
          const lope_i64 yimg = (yh ? (lope_i64)m1 : -(lope_i64)m1) * a.s1;
          if (!(yh | yl) && x + VX <= m0 && !(wxm && (x < g.hi[0] || x + VX > m0 - g.lo[0]))) {
            // a whole vector with no periodic image: one 16-byte store
            V o;
            T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
            for (int e = 0; e < VX; ++e) oe[e] = vals[r][e];
            *reinterpret_cast<V*>(orow + x) = o;
            continue;
          }
#pragma unroll
          for (int e = 0; e < VX; ++e) {
            const int xe = x + e;
            if (xe >= m0) break;
            const T v = vals[r][e];
            orow[xe] = v;
            const bool xh = wxm && xe < g.hi[0], xl = wxm && xe >= m0 - g.lo[0];
            if (xh | xl | yh | yl) {
              const int ximg = xh ? m0 : -m0;
              if (xh | xl) orow[xe + ximg] = v;
              if (yh | yl) {
                orow[xe + yimg] = v;
                if (xh | xl) orow[xe + ximg + yimg] = v;
              }
            }
          }
        }
      }
    }
    __syncthreads();
  }
}

// --------------------------------------------------------------------------
// Multi-array tiled path (rank 2/3, 2..4 array parameters with identical layouts).
//
// The single-array kernel's structure with one TMA box per array per plane in each
// ring stage (one mbarrier, NA boxes of bytes), the union of the arrays' footprints as
// the box halo, all NZW planes of a unit held in the ring (no z history) and the
// producer in warp 0 lane 0.  Plain launches (lope_launch) store the interior only;
// fused steps (lope_step_arrays) also store every stored array's periodic images.

template <class T, int NA, int NZW, int NR, int NXW, int FN0, int FN1, int FZN>
struct LopeWinReaderM {
  const T* win;    // [NA][NZW][NR][NXW]
  int r, v;
  template <int A, int DX, int DY, int DZ>
  __device__ __forceinline__ T at() const {
    return win[((A * NZW + DZ + FZN) * NR + (r + DY + FN1)) * NXW + (v + DX + FN0)];
  }
};

template <class T, int NA, int NZW, int NR, int NXW, int FN0, int FN1, int FZN>
struct LopeWinReaderM2 {
  const T* win;
  int r, v;        // v even
  template <int A, int DX, int DY, int DZ>
  __device__ __forceinline__ float2 at() const {
    const int i = ((A * NZW + DZ + FZN) * NR + (r + DY + FN1)) * NXW + (v + DX + FN0);
    return make_float2(win[i], win[i + 1]);
  }
};

template <class Body, class T, int WX, int WY, int RY, int NS, int PW = 0>
struct LopeTiledMCfg {
  static constexpr int NA = Body::NARR;
  static constexpr int VX = 16 / (int)sizeof(T);
  static constexpr int BX = 32 * VX * WX;
  static constexpr int BY = WY * RY;
  static constexpr int PADX = ((Body::UFN0 + VX - 1) / VX) * VX;
  static constexpr int BOXX = PADX + BX + ((Body::UFP0 + VX - 1) / VX) * VX;
  static constexpr int BOXY = BY + Body::UFN1 + Body::UFP1;
  static constexpr int NZW = Body::UFN2 + Body::UFP2 + 1;
  static constexpr int BOX_BYTES = ((BOXX * BOXY * (int)sizeof(T) + 127) / 128) * 128;
  static constexpr int STAGE_BYTES = NA * BOX_BYTES;
  static constexpr int TX_BYTES = NA * BOXX * BOXY * (int)sizeof(T);
  static constexpr int SMEM_BYTES = NS * STAGE_BYTES + 2 * NS * 8;
  static constexpr int NCW = WX * WY;
  static constexpr int THREADS = 32 * (NCW + PW);
  static constexpr int NR = RY + Body::UFN1 + Body::UFP1;
  static constexpr int NXW = VX + Body::UFN0 + Body::UFP0;
};

template <int NA> struct LopeTmapPack { LopeTmap m[NA]; };
template <class T, int NA> struct LopeArrPackT { LopeArr<T> a[NA]; };

template <class Body, class T, int WX, int WY, int RY, int NS, int PW = 0>
__device__ __forceinline__ void lope_tiled_multi_impl(const LopeTmapPack<Body::NARR>* maps,
                                                      const LopeArrPackT<T, Body::NARR>& arrs,
                                                      const LopeScal<T>& sc, const LopeGeom& g) {
  typedef LopeTiledMCfg<Body, T, WX, WY, RY, NS, PW> C;
  typedef typename LopeVec<T>::V V;
  constexpr int NA = C::NA, VX = C::VX, NZW = C::NZW, NR = C::NR, NXW = C::NXW;
  constexpr int FN0 = Body::UFN0, FP0 = Body::UFP0, FN1 = Body::UFN1, FP1 = Body::UFP1;
  constexpr int FZN = Body::UFN2;
  static_assert(NS >= NZW + 1, "ring must hold a unit's planes in use plus one prefetch slot");
  static_assert(C::BOXX <= 256 && C::BOXY <= 256, "TMA box dimensions are limited to 256");
  extern __shared__ __align__(128) unsigned char lope_smem[];
  lope_u64* full = reinterpret_cast<lope_u64*>(lope_smem + NS * C::STAGE_BYTES);
  lope_u64* empty = full + NS;
  const int ntx = (g.ext[0] + C::BX - 1) / C::BX;
  const int nty = (g.ext[1] + C::BY - 1) / C::BY;
  const int zc = g.zchunk;
  const int nzc = (g.ext[2] + zc - 1) / zc;
  const int nunits = ntx * nty * nzc;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int a = 0; a < NA; ++a) lope_tma_prefetch_desc(&maps->m[a]);
    for (int s = 0; s < NS; ++s) {
      lope_mbar_init(&full[s], 1);
      lope_mbar_init(&empty[s], C::NCW);
    }
    lope_fence_init();
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();

  LopeUnitWalk pw;
  int p_u = blockIdx.x, p_pl = 0, p_nl = 0, p_bx = 0, p_by = 0, p_z = 0;
  lope_u32 p_L = 0;
  const int oy = g.lo[1] + g.r0[1] - FN1;
  const int oz = g.lo[2] + g.r0[2] - FZN;
  const int pwarp = PW ? C::NCW : 0;
  if (warp == pwarp && lane == 0) {
    pw.init(blockIdx.x, gridDim.x, ntx, nty, nzc);
    if (p_u < nunits) {
      const int z0 = pw.zi * zc;
      p_nl = min(zc, g.ext[2] - z0) + NZW - 1;
      p_bx = g.box0 + pw.tx * C::BX;
      p_by = oy + pw.ty() * C::BY;
      p_z = oz + z0;
    }
  }
  auto produce = [&](lope_u32 limit) {
    while (p_L < limit && p_u < nunits) {
      const lope_u32 slot = p_L % NS;
      if (p_L >= (lope_u32)NS) lope_mbar_wait(&empty[slot], ((p_L / NS) - 1) & 1);
      lope_mbar_expect_tx(&full[slot], C::TX_BYTES);
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        unsigned char* dst = lope_smem + slot * C::STAGE_BYTES + a * C::BOX_BYTES;
        if (g.p1 > 0)
          lope_tma_load_2d(dst, &maps->m[a], &full[slot], p_bx, p_by + (p_z + p_pl) * g.p1);
        else
          lope_tma_load_3d(dst, &maps->m[a], &full[slot], p_bx, p_by, p_z + p_pl);
      }
      ++p_L;
      if (++p_pl == p_nl) {
        p_pl = 0;
        p_u += gridDim.x;
        pw.next();
        if (p_u < nunits) {
          const int z0 = pw.zi * zc;
          p_nl = min(zc, g.ext[2] - z0) + NZW - 1;
          p_bx = g.box0 + pw.tx * C::BX;
          p_by = oy + pw.ty() * C::BY;
          p_z = oz + z0;
        }
      }
    }
  };

  if (PW && warp == C::NCW) {
    if (lane == 0) produce(0xffffffffu);
    return;
  }
  const int wx = warp % WX;
  const int wy = warp / WX;
  const int cx = (wx * 32 + lane) * VX;
  const int row0 = wy * RY;
  const lope_i64 s1 = arrs.a[0].s1, s2 = arrs.a[0].s2;
  const int soff = (row0 * C::BOXX + C::PADX + cx);
  LopeUnitWalk w;
  w.init(blockIdx.x, gridDim.x, ntx, nty, nzc);
  lope_u32 lbase = 0;
  for (int u = blockIdx.x; u < nunits; u += gridDim.x, w.next()) {
    const int z0 = w.zi * zc;
    const int nz = min(zc, g.ext[2] - z0);
    const int x = w.tx * C::BX + cx;
    const int ybase = w.ty() * C::BY + row0;
    const bool xok = x < g.ext[0];
    const int nrow = min(RY, g.ext[1] - ybase);
    const lope_i64 rowoff = x + (lope_i64)ybase * s1 + (lope_i64)z0 * s2;
    // warp-uniform: whole in-range vectors, no x image, no y image -> plain stores (the
    // masked / image store state is rebuilt only where it is needed: register pressure)
    bool plain;
    {
      LopeVecOut<T, Body::RANK> v0;
      v0.init(x, xok, g);
      const bool wy = (g.wrap & 2) && nrow > 0 &&
                      (lope_near(ybase + g.r0[1], g.m[1], g.lo[1], g.hi[1]) ||
                       lope_near(ybase + nrow - 1 + g.r0[1], g.m[1], g.lo[1], g.hi[1]));
      plain = __all_sync(0xffffffffu, !wy && !v0.xw && (!xok || v0.xm == v0.ALL));
    }
    for (int pz = 0; pz < nz; ++pz) {
      if (!PW && warp == 0) {
        if (lane == 0) produce(lbase + pz + NS);
        __syncwarp();
      }
      const T* sp[NZW];
#pragma unroll
      for (int k = 0; k < NZW; ++k) {
        const lope_u32 L = lbase + pz + k;
        sp[k] = reinterpret_cast<const T*>(lope_smem + (L % NS) * C::STAGE_BYTES) + soff;
        lope_mbar_wait(&full[L % NS], (L / NS) & 1);
      }
      T win[NA][NZW][NR][NXW];
#pragma unroll
      for (int a = 0; a < NA; ++a)
#pragma unroll
        for (int k = 0; k < NZW; ++k)
#pragma unroll
          for (int q = 0; q < NR; ++q) {
            const T* rp = reinterpret_cast<const T*>(reinterpret_cast<const unsigned char*>(sp[k]) +
                                                     a * C::BOX_BYTES) + q * C::BOXX;
            const V vv = *reinterpret_cast<const V*>(rp);
            const T* ve = reinterpret_cast<const T*>(&vv);
#pragma unroll
            for (int e = 0; e < VX; ++e) win[a][k][q][FN0 + e] = ve[e];
#pragma unroll
            for (int e = 1; e <= FN0; ++e) win[a][k][q][FN0 - e] = rp[-e];
#pragma unroll
            for (int e = 0; e < FP0; ++e) win[a][k][q][FN0 + VX + e] = rp[VX + e];
          }
      constexpr int NSQ = Body::NSTORE > 0 ? Body::NSTORE : 1;
      T vals[RY][VX][NSQ];
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        if (LOPE_PAIR && sizeof(T) == 4) {
#pragma unroll
          for (int v = 0; v < VX; v += 2) {
            LopeWinReaderM2<T, NA, NZW, NR, NXW, FN0, FN1, FZN> rd;
            rd.win = &win[0][0][0][0];
            rd.r = r;
            rd.v = v;
            bool slow = false;
            float2 res[NSQ];
            Body::template eval<T, false, decltype(rd), float2, LopeAr2>(rd, sc.v, res, slow);
#pragma unroll
            for (int q = 0; q < NSQ; ++q) {
              vals[r][v][q] = res[q].x;
              vals[r][v + 1][q] = res[q].y;
            }
          }
        } else {
#pragma unroll
          for (int v = 0; v < VX; ++v) {
            LopeWinReaderM<T, NA, NZW, NR, NXW, FN0, FN1, FZN> rd;
            rd.win = &win[0][0][0][0];
            rd.r = r;
            rd.v = v;
            bool slow = false;
            Body::template eval<T, false>(rd, sc.v, vals[r][v], slow);
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        lope_mbar_arrive(&empty[(lbase + pz) % NS]);
        if (pz == nz - 1)
          for (int k = 1; k < NZW; ++k) lope_mbar_arrive(&empty[(lbase + pz + k) % NS]);
      }
      if (!xok || nrow <= 0) continue;
      // stored arrays get their interior points and, for a fused step (lope_step_arrays),
      // the periodic images the next HALO_TRANSFER would write
      const int zg = z0 + pz + g.r0[2];
      const bool zw = (g.wrap & 4) && lope_near(zg, g.m[2], g.lo[2], g.hi[2]);
      if (plain && !zw) {
#pragma unroll
        for (int q = 0; q < Body::NSTORE; ++q) {
          T* ob = arrs.a[Body::stored(q)].out + arrs.a[Body::stored(q)].org + rowoff + (lope_i64)pz * s2;
#pragma unroll
          for (int r = 0; r < RY; ++r) {
            if (r >= nrow) continue;
            V o;
            T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
            for (int e = 0; e < VX; ++e) oe[e] = vals[r][e][q];
            *reinterpret_cast<V*>(ob + (lope_i64)r * s1) = o;
          }
        }
      } else {
        LopeVecOut<T, Body::RANK> vo;
        vo.init(x, xok, g);
        const lope_i64 zimg = (zg < g.hi[2] ? (lope_i64)g.m[2] * s2 + g.sdl : -(lope_i64)g.m[2] * s2 + g.sdh);
#pragma unroll
        for (int q = 0; q < Body::NSTORE; ++q) {
          T* ob = arrs.a[Body::stored(q)].out + arrs.a[Body::stored(q)].org + rowoff + (lope_i64)pz * s2;
#pragma unroll
          for (int r = 0; r < RY; ++r) {
            if (r >= nrow) continue;
            V o;
            T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
            for (int e = 0; e < VX; ++e) oe[e] = vals[r][e][q];
            if (g.wrap)
              vo.store_all(ob + (lope_i64)r * s1, o, ybase + r + g.r0[1], zw, zimg, s1, g);
            else
              vo.put(ob + (lope_i64)r * s1, o);
          }
        }
      }
    }
    lbase += nz + NZW - 1;
  }
}
