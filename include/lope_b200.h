/* lope_b200.h — C ABI of the B200-native LOPe stencil hot path (liblope_b200.so).
 *
 * The reference (/root/reference/pkg, package `lopec`) is pure Python and has no
 * FFI.  Its hot path sits behind three methods of `Machine`; each
 * entry point below replaces one of them, and INTEGRATION.md shows the ctypes
 * binding a lopec maintainer would add:
 *
 *   lope_kernel_compile   replaces ir.lower_kernel -> run_body's tree walk
 *                         (lopec/ir.py:140-182, 258-308): the LOPE1 text of a
 *                         KernelIR is compiled once (NVRTC, sm_100a, cached).
 *   lope_launch           replaces Machine._launch_vector (runtime.py:596-618):
 *                         snapshot reads, centre stores over a launch range,
 *                         everything outside the range copied through.
 *   lope_halo_fill        replaces Machine._halo_exchange (runtime.py:643-697)
 *                         for dimensions whose neighbour is the image itself.
 *   lope_step             a launch over the full interior fused with the next
 *                         HALO_TRANSFER's local (periodic) fill.
 *   lope_layout_init / lope_pack / lope_unpack
 *                         replace StorageLayout + _scatter_block / gather
 *                         (ir.py:189-230, runtime.py:477-486, 715-737).
 *
 * Conventions: every call returns 0 on success, otherwise a positive reference
 * E-code number (102 footprint exceeds halo, 108 shape/range, 201 grid, 202
 * unallocated) or a negative CUDA / NVRTC / driver error; the message is in
 * lope_last_error().  Buffers are owned by the caller (device pointers from
 * cudaMalloc / torch); `stream` is a cudaStream_t.  Calls are asynchronous on
 * the given stream.
 */
#ifndef LOPE_B200_H
#define LOPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOPE_ABI_VERSION 1

#define LOPE_F32 1
#define LOPE_F64 2

/* Device storage of one image's block: the reference's padded column-major block
 * (ir.py:189-230: padded_d = m_d + lo_d + hi_d, dim 1 fastest) with every row
 * shifted so its first interior element sits on a 128-byte boundary and the row
 * pitch a multiple of 128 bytes (whole-line warp stores; 16-byte TMA strides).
 * Element at 0-based padded coordinates (c0,c1,c2) is at
 * base + c0 + c1*stride[1] + c2*stride[2]. */
typedef struct lope_layout {
  int32_t rank;          /* 1..3 */
  int32_t dtype;         /* LOPE_F32 | LOPE_F64 */
  int64_t interior[3];   /* m_d; 1 for d >= rank */
  int32_t lo[3];         /* halo widths (0..8); 0 for d >= rank */
  int32_t hi[3];
  int64_t padded[3];     /* m_d + lo_d + hi_d */
  int64_t stride[3];     /* element strides: 1, row pitch, plane pitch */
  int64_t count;         /* elements to allocate */
  int64_t elem_bytes;
  int64_t base;          /* element offset of padded cell (0,0,0) */
} lope_layout;

typedef struct lope_kernel lope_kernel;

int lope_abi_version(void);
const char* lope_last_error(void);

/* Cache directory for compiled cubins (default: $LOPE_CACHE_DIR or none). */
int lope_set_cache_dir(const char* path);

/* StorageLayout(interior, lo, hi) of ir.py:189 -> device layout.  E108 on bad
 * shapes (interior < 1, widths outside 0..8). */
int lope_layout_init(lope_layout* out, int32_t rank, int32_t dtype, const int64_t* interior,
                     const int32_t* lo, const int32_t* hi);

/* Compile a kernel from its LOPE1 text (paper_1502_03504_b200/ir.py: serialize). */
int lope_kernel_compile(const char* ir_text, size_t n, int32_t dtype, lope_kernel** out);
int lope_kernel_destroy(lope_kernel* k);
/* JSON description: arrays, scalars, stored arrays, footprints, path chosen, compiled tile
 * variants, plans per geometry, launches per kernel family. */
int lope_kernel_describe(const lope_kernel* k, char* buf, size_t n);
/* Emitted CUDA source of the kernel (for inspection / tests). */
int lope_kernel_source(const lope_kernel* k, char* buf, size_t n);

/* Machine._launch_vector: one launch over ranges[d] = {lo_d, hi_d} (1-based,
 * inclusive; rank entries).  in[a]: the snapshot of array parameter a; out[a]:
 * its live buffer (must differ from in[a]) or NULL when the kernel never stores
 * it.  After the call out[a] equals in[a] except over the range, where it holds
 * the kernel's centre values.  rscal / iscal hold the scalar parameters in
 * declaration order (real ones read from rscal, integer ones from iscal). */
int lope_launch(const lope_kernel* k, const lope_layout* layouts, const int64_t* ranges,
                const void* const* in, void* const* out, const double* rscal, const int64_t* iscal,
                void* stream);

/* Fused full-interior launch + periodic halo refresh of the dims in wrap_mask
 * (bit d = dim d+1).  Precondition: in's halos are valid.  Postcondition: out's
 * interior is the new field and its halo cells along wrap_mask dims hold the
 * periodic images of it — the state after the next HALO_TRANSFER.  One array
 * parameter only. */
int lope_step(const lope_kernel* k, const lope_layout* layout, const void* in, void* out,
              const double* rscal, const int64_t* iscal, int32_t wrap_mask, void* stream);

/* lope_step for kernels over several array parameters (runtime.py:541-618 followed by the
 * HALO_TRANSFER of every stored array, runtime.py:643-697): one full-interior launch
 * whose stored arrays (out[a] != in[a]) also receive their periodic images along
 * wrap_mask dims.  Arrays the kernel never stores are read from in[a] (out[a] may be
 * NULL) and keep their halos.  Precondition: every in[a]'s halos are valid. */
int lope_step_arrays(const lope_kernel* k, const lope_layout* layouts, const void* const* in,
                     void* const* out, const double* rscal, const int64_t* iscal, int32_t wrap_mask,
                     void* stream);

/* lope_step restricted to interior planes [begin, end) of the slowest dimension (0-based,
 * half-open): the slab-decomposed pipeline computes boundary planes first, exchanges
 * them, and computes the interior planes meanwhile.  Images are refreshed only along
 * wrap_mask dims (the decomposed dim is left to the exchange). */
int lope_step_planes(const lope_kernel* k, const lope_layout* layout, const void* in, void* out,
                     int64_t begin, int64_t end, const double* rscal, const int64_t* iscal,
                     int32_t wrap_mask, void* stream);

/* _halo_exchange with every neighbour equal to self along the dims in dims_mask:
 * each halo cell gets its periodic image (in place).  E108 if a halo is wider
 * than the interior. */
int lope_halo_fill(const lope_layout* layout, void* buf, int32_t dims_mask, void* stream);

/* Copy the interior between a host column-major array (m0 x m1 x m2, dim 1
 * fastest — numpy order='F') and the device block. */
int lope_pack(const lope_layout* layout, const void* host, void* dev, void* stream);
int lope_unpack(const lope_layout* layout, const void* dev, void* host, void* stream);

/* Same for the whole padded block (halo cells included): the host side is exactly
 * the reference's flat column-major block (DistributedArray.blocks[k],
 * runtime.py:471). */
int lope_pack_padded(const lope_layout* layout, const void* host, void* dev, void* stream);
int lope_unpack_padded(const lope_layout* layout, const void* dev, void* host, void* stream);

/* dst[box at dst_lo] := src[box at src_lo] for two blocks of the same layout; boxes of
 * `extent` cells in padded coordinates (3 entries each).  The halo slabs of
 * _halo_exchange between images and the device-mirror pulls / pushes
 * (runtime.py:669-711) are such boxes.  E108 if a box leaves the padded block. */
int lope_copy_box(const lope_layout* layout, void* dst, const void* src, const int64_t* dst_lo,
                  const int64_t* src_lo, const int64_t* extent, void* stream);

/* n such box copies (all of one layout) in as few launches as possible (up to 32 boxes
 * per launch): one phase of _halo_exchange (runtime.py:669-711) -- the border pulls, the
 * neighbour fills or the mirror pushes of every image -- costs one launch instead of one
 * per image and face.  dst[i] / src[i]: block pointers; dst_lo / src_lo / extent: 3n
 * entries.  Boxes must not overlap another box's destination.  E108 / E202 as above. */
int lope_copy_boxes(const lope_layout* layout, int32_t n, void* const* dst, const void* const* src,
                    const int64_t* dst_lo, const int64_t* src_lo, const int64_t* extent, void* stream);

/* Fill the interior with the synthetic U(-1,1) field: value of global cell
 * g = (o0+i) + G0*((o1+j) + G1*(o2+k)) is splitmix64-hash(g, seed) (oracle/
 * lope_oracle.py: hash_values).  global_extent / global_origin have 3 entries. */
/* `nsteps` fused steps (lope_step with every dim periodic) alternating between two
 * buffers, buf0 live first; *live_index = 0 or 1 names the buffer holding the result.
 * Rank-2 kernels advance 4 steps per launch in shared memory (temporal blocking;
 * same bits as 4 single steps) when the interior is at least a tile plus 4 halos. */
int lope_step_multi(const lope_kernel* k, const lope_layout* layout, void* buf0, void* buf1, int64_t nsteps,
                    const double* rscal, const int64_t* iscal, void* stream, int32_t* live_index);

/* lope_step_planes whose periodic images along the slowest dim are stored straight
 * into the neighbours' output blocks (same layout): the first `hi` planes' images into
 * `lo_peer_out` (the low neighbour's high halo), the last `lo` planes' into
 * `hi_peer_out` (the high neighbour's low halo); NULL = this block.  With the
 * neighbours' buffers mapped through CUDA IPC (NVLink peer memory) the halo exchange
 * is fused into the stencil kernel: no exchange kernel or copy; the caller orders
 * steps with a barrier.  Replaces the face fills of runtime.py:688-697. */
int lope_step_planes_peer(const lope_kernel* k, const lope_layout* layout, const void* in, void* out,
                          int64_t begin, int64_t end, const double* rscal, const int64_t* iscal,
                          int32_t wrap_mask, const void* lo_peer_out, const void* hi_peer_out, void* stream);

/* Device-to-device byte copy on `stream` (peer pointers included): the initial face
 * fill of the fused-exchange slabs. */
int lope_copy_bytes(void* dst, const void* src, int64_t bytes, void* stream);

/* CUDA IPC for the peer blocks: export a device pointer (64-byte handle + offset
 * into its allocation), open it in another process, close it. */
int lope_ipc_export(const void* ptr, uint8_t* handle, int64_t* offset);
int lope_ipc_open(const uint8_t* handle, int64_t offset, void** ptr);
int lope_ipc_close(void* ptr);

/* Execution plans (which compiled tile variant, which z-chunk) for the tiled kernel.
 * lope_plan_candidates compiles the candidate variants and lists (variant, z-chunk,
 * y-band of the unit walk) triples (n = how many exist; at most `cap` are written).  lope_plan_set makes one of
 * them the plan for every later launch whose first layout has this interior, halos
 * and wrap mask (variant -1 clears it).  Every plan computes the same bits; the host
 * runtime times real steps under each candidate and keeps the fastest. */
/* Compile every plan variant (NVRTC, cached; no GPU needed). */
int lope_kernel_prepare(lope_kernel* k);
int lope_plan_candidates(lope_kernel* k, int32_t* variants, int32_t* zchunks, int32_t* ybands, int32_t cap,
                         int32_t* n);
int lope_plan_set(lope_kernel* k, const lope_layout* layout, int32_t wrap_mask, int32_t variant, int32_t zchunk,
                  int32_t yband);
/* The same with the variant named by its tile shape {bxw, wy, ry, ns, producer_warp,
 * ctas_per_sm} (compiled if needed); *variant (may be NULL) receives its index. */
int lope_plan_set_tile(lope_kernel* k, const lope_layout* layout, int32_t wrap_mask, const int32_t* tile,
                       int32_t zchunk, int32_t yband, int32_t* variant);
/* Every plan parameter: cfg = {bxw, wy, ry, ns, producer_warp, ctas_per_sm, shfl, nb}
 * (the "tile", "producer_warp", "shfl", "nb" fields of lope_kernel_describe's plans);
 * replays a plan recorded by an earlier run (profiling captures of a given plan). */
int lope_plan_set_variant(lope_kernel* k, const lope_layout* layout, int32_t wrap_mask, const int32_t* cfg,
                          int32_t zchunk, int32_t yband, int32_t* variant);

/* Box <-> contiguous device buffer (column-major within the box, dim 1 fastest):
 * `extent` cells at padded coordinates `lo`.  Faces of a decomposed dimension other
 * than the slowest are strided; they are packed into a buffer, sent between GPUs
 * and unpacked into the neighbour's halo (the slabs of runtime.py:664-697 for an
 * MP x NP image grid, grid.py:22-61).  E108 if the box leaves the padded block. */
int lope_box_pack(const lope_layout* layout, const void* blk, const int64_t* lo, const int64_t* extent,
                  void* buf, void* stream);
int lope_box_unpack(const lope_layout* layout, void* blk, const int64_t* lo, const int64_t* extent,
                    const void* buf, void* stream);

int lope_fill_hash(const lope_layout* layout, void* dev, uint64_t seed, const int64_t* global_extent,
                   const int64_t* global_origin, void* stream);

/* Offset/count (elements) of a contiguous face slab along the slowest dim
 * (d = rank-1): which = 0 low halo, 1 high halo, 2 first `hi` interior planes,
 * 3 last `lo` interior planes.  Used to exchange faces between slab partitions. */
int lope_face_span(const lope_layout* layout, int32_t which, int64_t* offset, int64_t* count);

/* ---- Halo exchange between GPUs: Machine._halo_exchange (runtime.py:643-711) for
 * slab partitions (the slowest dim split over a ring of P images) ----
 *
 * One communicator per image (per process, or per host thread for ranks sharing a
 * process).  Setup is transport-neutral: every rank exports a fixed-size record
 * (lope_comm_record_size() bytes: its ping-pong buffers and step flags as CUDA IPC
 * handles and raw pointers, and its block geometry), the caller gathers all P records
 * in rank order over any out-of-band channel (torch.distributed, MPI, a file, shared
 * memory) and hands them to lope_comm_connect, which maps the two ring neighbours.
 *
 *   lope_comm_step      one fused step: wait (stream memory op) until both neighbours
 *                       finished their previous operation, ONE stencil kernel that
 *                       stores the boundary planes' periodic images straight into the
 *                       neighbours' output blocks over NVLink, then write this step's
 *                       number into the neighbours' flags (system-scope fenced).
 *   lope_halo_exchange  HALO_TRANSFER(U, BC=CYCLIC): local wrap of the other dims, then
 *                       the neighbours' faces -- peer copies after a flag handshake, or
 *                       ncclSend/ncclRecv in one group when only NCCL is initialised.
 *   lope_comm_sync      order the stream after both neighbours' latest operation.
 *
 * All ranks run the same sequence of operations with the same live index (SPMD
 * lockstep, as the reference's images do).  Errors: 201 bad image index / records
 * from another grid, 108 non-uniform blocks or halo wider than a block (F8), 202
 * missing setup, -3 transport unavailable. */
typedef struct lope_comm lope_comm;

/* Let the current device read/write `peer_device`'s memory (NVLink P2P); no-op for the
 * device itself or when already enabled.  The drop-in Machine's images on several GPUs
 * of one process copy halo slabs through it. */
int lope_peer_enable(int32_t peer_device);

int lope_comm_create(int32_t nranks, int32_t rank, lope_comm** out);
int lope_comm_destroy(lope_comm* comm);
int lope_comm_record_size(void);
/* record: lope_comm_record_size() bytes written for this rank. */
int lope_comm_export(lope_comm* comm, const lope_layout* layout, void* buf0, void* buf1, uint8_t* record);
/* records: all P records, rank order, concatenated. */
int lope_comm_connect(lope_comm* comm, const uint8_t* records);
/* NCCL transport for lope_halo_exchange (NCCL is loaded at run time):
 * rank 0 makes the 128-byte id, every rank passes it to lope_comm_nccl_init. */
int lope_comm_nccl_unique_id(uint8_t* id);
int lope_comm_nccl_init(lope_comm* comm, const uint8_t* id);
/* transport: 1 peer, 2 NCCL, 0 none, 3 peer with host ordering (a neighbour is another
 * process on the same GPU: the flags are not used -- ranks sharing a GPU must not wait on
 * each other on the device -- and the caller orders every operation on the host, e.g. a
 * device synchronise and a barrier); epoch = synchronised operations so far. */
int lope_comm_info(const lope_comm* comm, int32_t* rank, int32_t* nranks, uint32_t* epoch, int32_t* transport);
/* dims_mask: bit d = dim d+1; the decomposed (slowest) dim's bit moves the faces
 * between images, the other bits wrap locally (HALO_TRANSFER = all bits). */
int lope_halo_exchange(lope_comm* comm, int32_t live, int32_t dims_mask, void* stream);
/* The same in two phases (overlap, or ranks driven round-robin from one thread):
 * _begin wraps the local dims and marks the block ready (NCCL: the whole exchange),
 * _end waits for the neighbours' blocks and copies their faces. */
int lope_halo_exchange_begin(lope_comm* comm, int32_t live, int32_t dims_mask, void* stream);
int lope_halo_exchange_end(lope_comm* comm, void* stream);
int lope_comm_step(lope_comm* comm, const lope_kernel* k, int32_t live, const double* rscal, const int64_t* iscal,
                   void* stream);
int lope_comm_sync(lope_comm* comm, void* stream);

/* Number of this library's kernels launched since load (evidence for the bench). */
int64_t lope_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* LOPE_B200_H */
