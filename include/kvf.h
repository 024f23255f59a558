/*
 * kvf.h — C ABI of the B200 (sm_100a) KV-frame hot path.
 *
 * This library replaces the data-parallel hot path of the reference `framekv`
 * package (KVFetcher, arXiv 2602.09725; reference at pkg/src/framekv/, cited
 * below as fk/<file>:<line>):
 *
 *   pack    = quantize (fk/kvmodel.py:127-144) + slice_tokens/assemble_frames
 *             (fk/layout.py:109-114, 234-258)
 *   restore = restore_stream.on_frame (fk/fetchsim.py:335-358) + inverse_layout
 *             (fk/layout.py:137-147) + PagedMemory.page_write
 *             (fk/kvmodel.py:216-229), fused with dequantize (fk/kvmodel.py:147-152)
 *   decode  = codec.decode_frames (fk/codec.py:155-211) with its range coder
 *             (fk/rangecoder.py:146-189) and predictor (fk/codec.py:131-144)
 *
 * The reference has no FFI of its own: its boundary is the Python signatures
 * listed above.  These entry points are what a ctypes binding of that Python API
 * calls.
 *
 * Conventions
 *   - The caller owns every buffer.  The library never allocates or frees device
 *     memory; device pointers are plain CUDA device pointers.
 *   - Every launch goes on the caller's stream (`stream` is a cudaStream_t passed
 *     as void*; NULL = legacy default stream).  No call synchronises the device
 *     except where documented.
 *   - Errors return a kvf_status; the message is kept per thread and read with
 *     kvf_last_error().  There is no other global mutable state.
 *   - All element strides are in ELEMENTS of the tensor's dtype, byte strides are
 *     named *_bytes.  Channel index c = h*D + d, contiguous in d.
 */
#ifndef KVF_H_
#define KVF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVF_ABI_VERSION 1

/* Maximum units per batched launch (descriptors travel as kernel parameters). */
#define KVF_MAX_UNITS 128

typedef enum kvf_status {
  KVF_OK = 0,
  KVF_EINVAL = 1,        /* bad argument / shape: the reference raises ValueError */
  KVF_ECUDA = 2,         /* a CUDA runtime call failed */
  KVF_EUNSUPPORTED = 3,  /* valid for the reference, not handled by this build */
  KVF_EDECODE = 4        /* corrupt bitstream: the reference raises DecodeError */
} kvf_status;

typedef enum kvf_dtype {
  KVF_BF16 = 0,
  KVF_F16 = 1,
  KVF_F32 = 2,
  KVF_I8 = 3  /* int8 quantized codes (PagedMemory slot contents in the reference) */
} kvf_dtype;

/*
 * Frame plan of one chunk at one resolution class.  Mirrors LayoutConfig
 * (fk/layout.py:31-86) and FramePlan (fk/layout.py:157-201):
 *   element (h, d), h = i_h*b_h + j_h, d = i_d*b_d + j_d, lands at tile row
 *   i_h*a_d + i_d, tile column j_h*b_d + j_d; tile_h = a_h*a_d, tile_w = b_h*b_d.
 *   Token i: g,o = divmod(i, F); seg,slot = divmod(g, tiles_per_frame);
 *   frame = seg*F + o; tile (slot / grid_cols, slot % grid_cols).
 * frame_h/frame_w/frame_count are derived; kvf_plan_init fills them.
 */
typedef struct kvf_plan {
  int32_t T;               /* tokens in the chunk */
  int32_t H, D;            /* KV heads, head dim (powers of two) */
  int32_t a_h, b_h, a_d, b_d;
  int32_t F;               /* group frames (GOP) */
  int32_t tiles_per_frame, grid_rows, grid_cols;
  int32_t frame_h, frame_w, frame_count;
  int32_t group_size;      /* quantization group (contiguous channels) */
} kvf_plan;

/*
 * A sequence of 3-plane 8-bit frames: sample (f, p, y, x) lives at
 *   base + f*frame_stride + p*plane_stride + y*row_pitch + x.
 * The reference layout [n, 3, frame_h, frame_w] has row_pitch = frame_w,
 * plane_stride = frame_h*frame_w, frame_stride = 3*plane_stride.  A decoder
 * surface with a padded pitch is described by the same struct.
 */
typedef struct kvf_surface {
  uint8_t* base;
  int64_t frame_stride;
  int64_t plane_stride;
  int64_t row_pitch;
} kvf_surface;

/*
 * Three layers of a (paged) KV cache, one pointer per plane p of the triplet.
 * Token t of layer p (t = token_base + chunk token index) is the channel vector
 * at element offset
 *     blk*block_stride + (t % block_size)*slot_stride + h*head_stride + d
 * of layer[p], where blk = block_table ? block_table[t / block_size]
 *                                      : t / block_size.
 * This is PagedMemory (fk/kvmodel.py:195-229: page = t // page_size_tokens,
 * slot = t % page_size_tokens) with the page dict replaced by a block table,
 * i.e. vLLM's [num_blocks, block_size, H, D] (NHD) or [num_blocks, H,
 * block_size, D] (HND) per-layer caches.  layer[p] == NULL marks a pad layer
 * (fk/kvmodel.py:56-69): restore never writes it, pack reads it as zeros.
 * A contiguous [T, L, H, D] KVCache is block_table = NULL, block_size = 1,
 * block_stride = slot_stride = L*H*D, head_stride = D, layer[p] = base + l*H*D.
 */
typedef struct kvf_paged {
  void* layer[3];
  const int32_t* block_table;
  int32_t block_size;
  int32_t dtype;           /* kvf_dtype of the cache */
  int64_t block_stride;
  int64_t slot_stride;
  int64_t head_stride;
  int32_t token_base;
  int32_t reserved_;
} kvf_paged;

/* One (K-or-V, layer triplet, token chunk) unit of a batched restore. */
typedef struct kvf_restore_unit {
  kvf_surface frames;
  kvf_plan plan;
  const float* scales;     /* device [3, H*D/group_size] fp32 (container scales) */
  kvf_paged dst;
  int32_t first_frame;     /* restore frames [first_frame, first_frame+n_frames) */
  int32_t n_frames;
} kvf_restore_unit;

/* One unit of a batched pack. */
typedef struct kvf_pack_unit {
  kvf_paged src;           /* bf16/f16/f32 KV to quantize, or int8 codes */
  kvf_plan plan;
  uint32_t* absmax;        /* device scratch of kvf_pack_scratch_words(&plan) u32:
                              [3, G] |x| maxima (f32 bit patterns), then schedule
                              scratch */
  float* scales;           /* device [3, G] out (ignored for int8 sources) */
  kvf_surface frames;      /* out: frame_count frames */
} kvf_pack_unit;

/* ---- housekeeping ------------------------------------------------------- */
int32_t kvf_abi_version(void);
const char* kvf_last_error(void);

/* Validate the layout/plan fields and derive frame_h/frame_w/frame_count;
 * mirrors the checks of LayoutConfig.__init__ (fk/layout.py:38-50),
 * FramePlan.__init__ (fk/layout.py:166-193) and plan_inter_frame
 * (fk/layout.py:224-228). */
kvf_status kvf_plan_init(kvf_plan* plan);

/* Byte size of the frame surface a plan needs in the reference layout. */
int64_t kvf_plan_frame_bytes(const kvf_plan* plan);

/* ---- restore (frames -> paged KV), the headline path -------------------- */

/* Frame-wise restore of frames [first_frame, first_frame+n_frames) of one
 * chunk: every valid tile slot (fk/layout.py:203-212) is un-tiled, re-centred
 * (u8 - 128), dequantised with the chunk scales (fk/kvmodel.py:147-152, fp32
 * product, then RNE to the cache dtype; int8 caches receive the codes as the
 * reference PagedMemory does) and written to its paged slot.
 * Replaces fk/fetchsim.py:347-355 (on_frame) for a decoded frame batch. */
kvf_status kvf_restore(const kvf_surface* frames, int32_t first_frame,
                       int32_t n_frames, const kvf_plan* plan,
                       const float* scales, const kvf_paged* dst, void* stream);

/* Same for up to n_units units (split into launches of KVF_MAX_UNITS).
 * `units` is a HOST array; descriptors are passed by value to the kernel. */
kvf_status kvf_restore_batch(const kvf_restore_unit* units, int32_t n_units,
                             void* stream);

/* kvf_restore_batch restricted to KV heads, for tensor-parallel caches that
 * hold a head shard: heads [head_lo, head_lo +
 * n_windows*n_heads) in n_windows windows of n_heads; head h of window
 * w = (h - head_lo) / n_heads lands at local head (h - head_lo) % n_heads of
 * `dst`, displaced by w * window_stride bytes (a peer's region of a send buffer;
 * one window: a rank's own shard).  raw_samples = 1 (int8 destinations only)
 * stores the frame samples (q + 128) instead of the codes: the head slice in
 * frame form, which a peer restores with kvf_restore_batch under a flat plan
 * (identity tile of n_heads x D, F = 1, one frame of T tile rows).  Only the
 * windows' bytes are read and written. */
kvf_status kvf_restore_batch_heads(const kvf_restore_unit* units, int32_t n_units,
                                   int32_t head_lo, int32_t n_heads, int32_t n_windows,
                                   int64_t window_stride, int32_t raw_samples, void* stream);

/* ---- pack (KV -> frames) ------------------------------------------------ */

/* Phase 1: per (plane, group) max |x| over all chunk tokens, accumulated with
 * atomicMax into `absmax` (which must be zeroed by the caller or by
 * kvf_pack_batch).  fk/kvmodel.py:138-139. */
kvf_status kvf_pack_absmax(const kvf_paged* src, const kvf_plan* plan,
                           uint32_t* absmax, void* stream);

/* Phase 2: scale = fp32(fp64(max)/127) or 1 (fk/kvmodel.py:140), exact
 * round-half-even quantisation and clip (fk/kvmodel.py:141-143), +128, tile
 * permutation and frame placement with pad byte 128 (fk/layout.py:234-258).
 * Writes `scales` [3, G] too.  For an int8 `src` the codes are placed as-is
 * (assemble_frames) and absmax/scales are ignored. */
kvf_status kvf_pack_frames(const kvf_paged* src, const kvf_plan* plan,
                           const uint32_t* absmax, float* scales,
                           const kvf_surface* frames, void* stream);

/* Both phases for up to n_units units, zeroing each unit's scratch first:
 * absmax -> scales -> frames (KVF_PACK_AUTO schedule, see kvf_pack_batch_ex). */
kvf_status kvf_pack_batch(const kvf_pack_unit* units, int32_t n_units,
                          void* stream);

/* Pack schedules of kvf_pack_batch_ex. */
typedef enum kvf_pack_schedule {
  KVF_PACK_AUTO = 0,        /* the fastest measured on this build */
  KVF_PACK_TWO_PASS = 1,    /* absmax kernel, then frames kernel: reads the source twice */
  KVF_PACK_SINGLE_READ = 2  /* one HBM read: clusters of 8 (or 16) CTAs own whole
                               (unit, plane, group) sub-units, stream them through shared
                               memory with TMA, exchange the maxima through distributed
                               shared memory and re-read from L2.  Slower than two-pass on
                               B200 */
} kvf_pack_schedule;

/* kvf_pack_batch with an explicit schedule.  `param` (single read only): CTAs
 * per cluster, 8 or 16 (0 = 8).  Same results for every schedule (bit-identical
 * frames and scales); units a schedule cannot take (int8 sources, group sizes
 * other than 64/128/256, tile rows narrower than 8 channels, strides the tensor
 * maps reject) run the two-pass kernels. */
kvf_status kvf_pack_batch_ex(const kvf_pack_unit* units, int32_t n_units,
                             int32_t schedule, int64_t param, void* stream);

/* Phase 2 only, for up to n_units units whose `absmax` the caller already
 * filled with the per-(plane, group) maxima of the same source (e.g. a KV
 * writer that tracks them as it stores K/V, or an earlier kvf_pack_absmax):
 * scales + frames in a single read of the source.  Samples beyond a supplied
 * maximum are clipped exactly as the reference clips (fk/kvmodel.py:142). */
kvf_status kvf_pack_frames_batch(const kvf_pack_unit* units, int32_t n_units,
                                 void* stream);

/* u32 words of pack scratch a unit of this plan needs: 6*G (G = H*D/group_size). */
int64_t kvf_pack_scratch_words(const kvf_plan* plan);

/* ---- whole-tensor quantize / dequantize (fk/kvmodel.py:127-152) -------- */

/* x: contiguous [T, L, C] of dtype src_dtype (bf16/f16/f32); absmax: [L, G]
 * u32 scratch (zeroed here); scales: [L, G] fp32 out; values: [T, L, C] int8. */
kvf_status kvf_quantize(const void* x, int32_t src_dtype, int64_t T, int32_t L,
                        int32_t C, int32_t group_size, uint32_t* absmax,
                        float* scales, int8_t* values, void* stream);

/* values [T, L, C] int8, scales [L, G] -> out [T, L, C] of out_dtype. */
kvf_status kvf_dequantize(const int8_t* values, const float* scales, int64_t T,
                          int32_t L, int32_t C, int32_t group_size, void* out,
                          int32_t out_dtype, void* stream);

/* ---- KVFC bitstream decode (fk/codec.py:155-211) -------------------------- */

/* Stream geometry from the 12-byte header (u32 n_frames, height, width). */
typedef struct kvf_kvfc_info {
  int32_t n_frames;
  int32_t height;
  int32_t width;
  int32_t bitmap_len;      /* bytes of one packed mode bitmap: ceil(bh*bw/8) */
} kvf_kvfc_info;

/* Host-side walk of a KVFC stream (fk/codec.py:16-20 layout) exactly as
 * decode_frames walks it (fk/codec.py:164-208), without entropy decoding.
 * For frame f, plane p (k = 3f + p): payload_off[k], payload_len[k] (the u32
 * length prefix), bitmap_off[k] (-1 for intra frames); frame_type[f].
 * Arrays hold cap_frames frames (3*cap_frames entries); with cap_frames <
 * n_frames only the header is read, `info` is filled and KVF_EINVAL is
 * returned (a size query: the walk and its checks run on the fill call;
 * header errors are reported by both).  Returns
 * KVF_EDECODE and *bad_frame on every condition where the reference raises
 * DecodeError (short header, truncated type/bitmap/length/payload, bad frame
 * type, inter frame without reference, trailing bytes). */
kvf_status kvf_kvfc_scan(const uint8_t* data, int64_t size, kvf_kvfc_info* info,
                         int64_t* payload_off, int32_t* payload_len,
                         int64_t* bitmap_off, uint8_t* frame_type,
                         int32_t cap_frames, int32_t* bad_frame);

/* kvf_kvfc_scan of n_streams streams in one call (replaces the reference's
 * per-stream walk in decode_frames, fk/codec.py:164-208, for a batch).  With
 * frame_base == NULL only the headers are read (info[j] filled).  Otherwise
 * stream j's frames are written at frame index frame_base[j] of the flat
 * arrays (entries 3*frame_base[j] .. of payload_off / payload_len /
 * bitmap_off, frame_base[j] .. of frame_type), walked on up to n_threads host
 * threads.  Errors as kvf_kvfc_scan, for the first failing stream in order:
 * *bad_stream (-1 when none) and *bad_frame locate it. */
kvf_status kvf_kvfc_scan_batch(const uint8_t* const* data, const int64_t* size,
                               int32_t n_streams, kvf_kvfc_info* info,
                               const int64_t* frame_base, int64_t* payload_off,
                               int32_t* payload_len, int64_t* bitmap_off,
                               uint8_t* frame_type, int32_t n_threads,
                               int32_t* bad_stream, int32_t* bad_frame);

/* One range-coded symbol stream (one plane of one frame). */
typedef struct kvf_rc_stream {
  const uint8_t* payload;  /* device */
  int64_t len;             /* payload bytes (reads past the end yield 0) */
  uint8_t* symbols;        /* device output */
  int64_t n_symbols;       /* height * width */
} kvf_rc_stream;

/* Entropy-decode n_streams independent streams (fk/rangecoder.py:146-189:
 * adaptive order-0 model reset per stream, carry-less 32-bit range coder),
 * one GPU thread per stream.  `d_streams` must be device-accessible: device
 * memory or mapped (UVA) pinned host memory, read once per stream. */
kvf_status kvf_rc_decode(const kvf_rc_stream* d_streams, int32_t n_streams,
                         void* stream);

/* One contiguous byte range of a fed decode: host -> device. */
typedef struct kvf_feed_seg {
  const uint8_t* src;      /* pinned host memory (device-accessible through UVA) */
  uint8_t* dst;            /* device */
  int64_t len;
} kvf_feed_seg;

/* kvf_rc_decode whose payload bytes are still on the host: ONE cooperative
 * launch in which n_copy_ctas CTAs copy the segments host -> device over PCIe
 * in piece-major order (piece r of a segment = its bytes in [L0 + r*piece_bytes,
 * L0 + (r+1)*piece_bytes), L0 = the 128-byte line holding its first byte;
 * piece r of every segment before piece r+1 of any) while the other CTAs
 * decode; stream k
 * (whose payload lies in segment d_seg_of[k]) reads a byte only once the
 * pieces of its segment up to that byte have landed.  Every stream thus starts
 * decoding after its segment's first piece, not after the whole batch's H2D.
 * `ready`: device scratch of n_segs u32 (zeroed here).  max_seg_len >= every
 * segment's len.  KVF_EUNSUPPORTED if the grid does not fit one wave.  The
 * segments (d_segs, d_seg_of: device-accessible) must cover every payload byte,
 * each in 128-byte lines of its own (no line shared with another segment: the
 * decoders read through L1), src and dst alike modulo 16; piece_bytes a
 * multiple of 128.  When the call's work completes, all segments are on the
 * device. */
kvf_status kvf_rc_decode_fed(const kvf_rc_stream* d_streams, int32_t n_streams,
                             const kvf_feed_seg* d_segs, const int32_t* d_seg_of,
                             int32_t n_segs, int32_t piece_bytes, int64_t max_seg_len,
                             uint32_t* ready, int32_t n_copy_ctas, void* stream);

/* One plane of one frame for reconstruction (fk/codec.py:131-144). */
typedef struct kvf_recon_plane {
  const uint8_t* symbols;  /* device, height*width zigzag symbols */
  const uint8_t* modes;    /* device packed mode bitmap (np.packbits order), NULL = intra */
  uint8_t* out;            /* device plane origin */
  int64_t out_pitch;       /* bytes between rows */
} kvf_recon_plane;

/* A dependency chain: planes[first .. first+count) of ONE plane index over
 * consecutive frames, the first intra; entry k predicts from entry k-1.  An
 * entry with symbols == NULL is a plane reconstructed by an earlier call (the
 * previous frame of a frame-by-frame decode): it is not written, only read as
 * the next entry's reference, so a chain may start [reference, inter plane]. */
typedef struct kvf_recon_chain {
  int32_t first;
  int32_t count;
  int32_t height;
  int32_t width;
} kvf_recon_chain;

/* Reconstruct every chain (one CTA per chain; frames inside a chain in order):
 * sample = (pred + unzigzag(symbol)) mod 256 with pred = co-located previous
 * frame sample (inter block), left neighbour, first column from above, 128 at
 * the corner.  Both arrays must be device-accessible: device memory or
 * mapped (UVA) pinned host memory, read once per chain/plane. */
kvf_status kvf_kvfc_reconstruct(const kvf_recon_plane* d_planes,
                                const kvf_recon_chain* d_chains, int32_t n_chains,
                                void* stream);

/* ---- KVFC bitstream encode (fk/codec.py:93-128) ------------------------- */

/* One plane of one frame to predict: residuals, 16x16 modes, zigzag symbols. */
typedef struct kvf_resid_plane {
  const uint8_t* cur;      /* device plane origin */
  const uint8_t* prev;     /* previous frame's plane, NULL for an intra frame */
  int64_t pitch;           /* bytes between rows of cur (and prev) */
  uint8_t* symbols;        /* device out: height*width zigzag symbols */
  uint8_t* modes;          /* device out: bh*bw bytes, 1 = inter (inter frames only) */
  int32_t height;
  int32_t width;
} kvf_resid_plane;

/* Per 16x16 block: intra residual (left; first column from above; 128 at the
 * corner) and, for inter frames, the co-located inter residual; mode = inter
 * iff SAD_inter <= SAD_intra (fk/codec.py:77-90, 110-123); symbols =
 * zigzag(residual mod 256).  `d_planes` is a DEVICE array. */
kvf_status kvf_kvfc_residuals(const kvf_resid_plane* d_planes, int32_t n_planes,
                              int32_t max_blocks, void* stream);

/* Range-encode n streams (fk/rangecoder.py:106-143), one thread per stream:
 * reads `symbols`/`n_symbols`, writes `payload` (capacity >= 2*n_symbols + 16)
 * and the coded length to d_out_len[k].  `d_streams` is a DEVICE array. */
kvf_status kvf_rc_encode(const kvf_rc_stream* d_streams, int32_t n_streams,
                         int64_t* d_out_len, void* stream);

/* Scatter pieces into a stream buffer: dst[dst_off .. +len) = src[0 .. len),
 * or, with pack_bits, dst[dst_off + b/8] bit (7 - b%8) = src[b] for b < len
 * (np.packbits order).  `d_pieces` is a DEVICE array. */
typedef struct kvf_piece {
  const uint8_t* src;
  int64_t dst_off;
  int64_t len;
  int32_t pack_bits;
  int32_t reserved_;
} kvf_piece;
kvf_status kvf_gather(const kvf_piece* d_pieces, int32_t n_pieces, uint8_t* dst,
                      void* stream);

/* ---- synthetic inputs ---------------------------------------------------- */

/* In-place AR(1) scan along the middle axis of an fp32 [outer, len, inner]
 * tensor: x[o,t,i] = s*x[o,t-1,i] + (1-s)*x[o,t,i] (the law of gen_synthetic_kv,
 * fk/kvmodel.py:155-192; used to build perf inputs on the GPU). */
kvf_status kvf_ar1_scan(float* x, int64_t outer, int64_t len, int64_t inner,
                        float s, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* KVF_H_ */
