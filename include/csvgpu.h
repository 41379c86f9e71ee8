/*
 * csvgpu.h -- C-ABI of the B200-native CSV brick decoder (libcsvgpu.so).
 *
 * The reference (`csvol`, pure Python + numba) has no FFI; its decode entry
 * points are in-process numba calls.  Each function below replaces one of
 * them (citations: /root/reference/pkg/src/csvol/<file>:<line>), exported
 * with plain pointers and sizes so any host language can bind it (the Python
 * host in paper_2308_16619_b200/ binds it with ctypes).
 *
 * Conventions:
 *   - Every function returns CSV_OK (0) or a negative CSV_E_* code; the text
 *     of the last failure on the calling thread is csv_last_error().
 *   - Device pointers ("d_" prefix) are caller-owned device memory; the
 *     library never frees caller memory.  Compressed data uploaded by
 *     csv_volume_create is library-owned until csv_volume_free.
 *   - All decode calls are asynchronous on the caller's CUDA stream
 *     (`stream` is a cudaStream_t cast to uintptr_t; 0 = legacy default).
 *     A csv_volume owns one workspace: calls on one volume must be ordered
 *     on one stream (use one volume handle per concurrent stream).
 *   - Per-brick corruption is NOT a call failure: it is reported per brick
 *     in csv_result with the reference's status codes (codec.py:280-287),
 *     stream and nibble position, so the host raises byte-identical
 *     CorruptStreamError messages (codec.py:487-495, :540-543).
 */
#ifndef CSVGPU_H
#define CSVGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSV_OK 0
#define CSV_E_ARG (-1)      /* invalid argument */
#define CSV_E_CUDA (-2)     /* CUDA runtime error */
#define CSV_E_NOMEM (-3)    /* device allocation failed */
#define CSV_E_FORMAT (-4)   /* malformed container header */
#define CSV_E_CAPACITY (-5) /* brick cache: the visible set does not fit the pool (CacheCapacityError) */

/* Per-brick status codes: 0..7 as codec.py:280-287, plus CSV_ST_EMPTY_PALETTE
 * for codec.py:510-511 ("empty palette"). */
#define CSV_ST_OK 0
#define CSV_ST_UNDERRUN 1
#define CSV_ST_BAD_OP 2
#define CSV_ST_PALETTE_RANGE 3
#define CSV_ST_DELTA_RANGE 4
#define CSV_ST_DESYNC 5
#define CSV_ST_BAD_NEIGHBOR 6
#define CSV_ST_LEAF_STOP 7
#define CSV_ST_EMPTY_PALETTE 8

/* One decode outcome; mirrors the tuple _decode_kernel returns
 * (codec.py:322: status, stream, nibble position, consumed coarse, consumed detail). */
typedef struct csv_result {
    int32_t status;
    int32_t stream;   /* 0 coarse, 1 detail */
    int64_t pos;      /* nibble position of the failure */
    int64_t ci;       /* coarse nibbles consumed (valid when status == 0) */
    int64_t di;       /* detail nibbles consumed (valid when status == 0) */
} csv_result;

/* K1 per-stream outcome (csv_decode_streams). */
typedef struct csv_stream_result {
    uint32_t n_entries;    /* complete entries (op nibble + payload) decoded */
    uint32_t fail_nibble;  /* first unavailable nibble (flags & CSV_SF_FAILED) */
    uint32_t flags;        /* CSV_SF_* */
    uint32_t partial_op;   /* op nibble of entry n_entries when CSV_SF_PARTIAL */
} csv_stream_result;
#define CSV_SF_FAILED 1u    /* nibble fail_nibble cannot be pulled (underrun / count exhausted) */
#define CSV_SF_PARTIAL 2u   /* entry n_entries has its op nibble but no payload */
#define CSV_SF_DESYNC 4u    /* all nibbles decoded; final state != 2^23 or bytes left (rans.py:163) */
#define CSV_SF_COMPLETE 8u  /* all `n` nibbles decoded */

typedef struct csv_volume csv_volume;

/* Library/version probe. */
int csv_version(void);
const char* csv_last_error(void);

/* Volume upload from HOST memory.  Replaces CsvContainer._parse_head /
 * _parse_body (container.py:289-330) as the decoder's input stage.
 *   head120   : bytes 0..119 of the CSV1 file (header, both count tables, blob sizes)
 *   dir44     : directory rows [brick_begin, brick_end), 44 B each (container.py:53-64)
 *   palette   : u32 palette entries starting at global entry palette_base
 *   coarse    : coarse-blob bytes starting at global byte coarse_base
 *   detail    : detail-blob bytes starting at global byte detail_base (may be NULL/0)
 * Directory offsets are global; rows pointing outside the passed slices are
 * clamped like numpy slicing (container.py:138-153).  Copies are issued on
 * `stream`; host buffers may be reused once the stream has passed this call. */
int csv_volume_create(int device, const uint8_t* head120, const uint8_t* dir44,
                      uint64_t brick_begin, uint64_t brick_end,
                      const uint32_t* palette, uint64_t palette_base, uint64_t palette_len,
                      const uint8_t* coarse, uint64_t coarse_base, uint64_t coarse_len,
                      const uint8_t* detail, uint64_t detail_base, uint64_t detail_len,
                      uintptr_t stream, csv_volume** vol);

/* Same, from DEVICE memory already resident (e.g. the GPU encoder's output).
  * The blobs are borrowed (not copied): keep them alive until csv_volume_free;
 * each must have >= 64 readable bytes past its end (stream prefetch). */
int csv_volume_create_device(int device, const uint8_t* head120, const uint8_t* d_dir44,
                             uint64_t brick_begin, uint64_t brick_end,
                             const uint32_t* d_palette, uint64_t palette_base, uint64_t palette_len,
                             const uint8_t* d_coarse, uint64_t coarse_base, uint64_t coarse_len,
                             const uint8_t* d_detail, uint64_t detail_base, uint64_t detail_len,
                             uintptr_t stream, csv_volume** vol);

/* Deferred upload: the directory and tables are uploaded now, the three blob
 * slices are allocated but filled later with csv_volume_upload (blob 0 palette,
 * 1 coarse, 2 detail; offset/nbytes in bytes relative to the slice), so a host
 * pipeline can overlap uploading slab k+1 with decoding slab k. */
int csv_volume_create_deferred(int device, const uint8_t* head120, const uint8_t* dir44, uint64_t brick_begin,
                               uint64_t brick_end, uint64_t palette_base, uint64_t palette_len, uint64_t coarse_base,
                               uint64_t coarse_len, uint64_t detail_base, uint64_t detail_len, uintptr_t stream,
                               csv_volume** vol);
int csv_volume_upload(csv_volume* vol, int blob, const void* host, uint64_t offset, uint64_t nbytes, uintptr_t stream);

/* Cold detail (render.py:782-832, container.py:148-159): for a volume created
 * without its detail blob, make the n staged bricks' level-0 streams readable
 * from d_stage (brick d_bricks[i] at byte d_offs[i], d_lens[i] bytes); every
 * other brick has no detail stream until staged again.  d_stage is borrowed
 * and needs 64 readable bytes past stage_len. */
int csv_volume_stage_detail(csv_volume* vol, const uint32_t* d_bricks, const uint64_t* d_offs, const uint32_t* d_lens,
                            uint64_t n, const uint8_t* d_stage, uint64_t stage_len, uintptr_t stream);

int csv_volume_free(csv_volume* vol);

/* DetailStore.plan's budget scan (render.py:808-823), host-side C: accept[i] = 1 iff
 * the running total of accepted sizes plus sizes[i] stays within budget. */
int csv_detail_plan_greedy(const uint64_t* sizes, uint64_t n, uint64_t budget, uint8_t* accept, uint64_t* spent);

/* Full-volume decode at LOD t into a raster (Z,Y,X) u32 slab: replaces
 * decompress_volume (container.py:456-478) + morton_to_grid (morton.py:411-416).
 * d_out holds LOD-t z rows [z_begin, z_end) of the volume cropped to
 * ceil(dims / 2^t) (container.py:476-478); z_begin must be a multiple of the
 * LOD-t brick side (2^(brick_log2 - t)), else CSV_E_ARG; only this volume's
 * bricks are decoded.  d_res (may be NULL) receives one csv_result per brick of the
 * volume's range, in brick order. */
int csv_decode_volume(csv_volume* vol, int t, uint32_t* d_out, int64_t z_begin, int64_t z_end,
                      csv_result* d_res, uintptr_t stream);

/* Same for the bricks [brick_first, brick_last) (global indices inside the
 * volume's range) only: the unit of the slab pipeline that overlaps decode with
 * device-to-host copies.  d_res receives brick_last - brick_first results. */
int csv_decode_volume_range(csv_volume* vol, int t, uint64_t brick_first, uint64_t brick_last, uint32_t* d_out,
                            int64_t z_begin, int64_t z_end, csv_result* d_res, uintptr_t stream);

/* Batched random-access decode into a Morton-order brick pool: replaces the
 * per-brick CsvContainer.decode_brick (container.py:168-208) loop inside
 * BrickCache._store / end_frame_assign (cache.py:125-170).  Request i decodes
 * brick d_brick[i] (global index) at LOD d_lod[i] into
 * d_pool[d_dst[i] .. d_dst[i] + 8^(N - lod)) in Morton order (cache.py:130-134).
 * Requests must target disjoint pool ranges.  d_res receives one csv_result
 * per request (may be NULL). */
int csv_decode_bricks(csv_volume* vol, uint64_t n, const uint32_t* d_brick, const uint8_t* d_lod,
                      const uint64_t* d_dst, uint32_t* d_pool, csv_result* d_res, uintptr_t stream);

/* Host-buffer variant of csv_decode_bricks for per-brick callers
 * (CsvContainer.decode_brick, container.py:168-208, on a device-resident volume):
 * n (brick, lod) requests in host memory; the Morton labels land in h_out
 * contiguously in request order (8^(N - lod) each), per-request results in
 * h_res.  Requests are staged through library-owned pinned memory; the call
 * returns after the stream has synchronised. */
int csv_decode_bricks_host(csv_volume* vol, uint64_t n, const uint32_t* h_brick, const uint8_t* h_lod,
                           uint32_t* h_out, csv_result* h_res, uintptr_t stream);

/* Streams passed per call: replaces decode_brick_entropy (codec.py:571-594)
 * and decode_brick (codec.py:549-568) -> _run_decode (codec.py:498-546) for
 * ONE brick whose palette and coarse / detail stream bytes are host arrays.
 * head120 is the 120-byte head of a one-brick volume (dims = brick side; its
 * count tables and entropy flag are the ones the streams were coded with;
 * the blob sizes in it are ignored).  Decodes at LOD t into h_out
 * (8^(N - t) labels, Morton order) and h_res (status / stream / nibble,
 * consumed counts).  The library keeps one scratch volume per device (blobs
 * grown on demand, re-created when the tables or brick size change) and
 * pinned staging; thread-safe (serialised); returns after the stream has
 * synchronised. */
int csv_decode_brick_streams(int device, const uint8_t* head120, const uint32_t* palette, uint64_t n_pal,
                             const uint8_t* coarse, uint64_t coarse_bytes, uint32_t coarse_nibbles,
                             const uint8_t* detail, uint64_t detail_bytes, uint32_t detail_nibbles, int t,
                             uint32_t* h_out, csv_result* h_res, uintptr_t stream);

/* Stand-alone entropy stage (K1): replaces rans_decode/_decode_core
 * (rans.py:140-198) + iter_operations (codec.py:604-623).  For each request
 * brick, decodes the coarse and (t == 0) detail stream into entry bytes
 * (op | stop<<3 | delta<<4, one per operation) at d_entries + d_entry_off[2i+s],
 * s = 0 coarse / 1 detail.  d_entry_off must hold 2n+1 u64 and is filled with
 * the exclusive scan of the per-stream regions; d_sres receives 2n results.
 * entries_cap is the capacity of d_entries in bytes. */
int csv_decode_streams(csv_volume* vol, uint64_t n, const uint32_t* d_brick, int t,
                       uint8_t* d_entries, uint64_t entries_cap, uint64_t* d_entry_off,
                       csv_stream_result* d_sres, uintptr_t stream);

/* Upper bound of the entry bytes csv_decode_streams needs for n requests at LOD t. */
int csv_streams_capacity(csv_volume* vol, uint64_t n, int t, uint64_t* cap);

/* Operation histogram of every brick's full streams (stats(), container.py:485-529):
 * d_counts8[op] = number of entries with opcode op (payload nibbles excluded);
 * d_sres (2 x bricks, coarse then detail per brick) reports truncated (FAILED
 * before COMPLETE) and desynchronized streams as rans_decode would
 * (rans.py:183-198).  No entry buffer is written. */
int csv_volume_op_counts(csv_volume* vol, uint64_t* d_counts8, csv_stream_result* d_sres, uintptr_t stream);

/* Volume geometry probe: dims(x,y,z), grid(x,y,z), brick_log2, entropy. */
int csv_volume_info(csv_volume* vol, int64_t* dims3, int64_t* grid3, int* brick_log2, int* entropy);

/* Per-stage device timing of the next decode calls on this volume (CUDA events
 * recorded on the caller's stream): ms3 = {planning (sizes + scan), K1 entropy
 * lanes, K2 replay + writer} of the most recent csv_decode_volume/_bricks call. */
int csv_volume_set_timing(csv_volume* vol, int enable);
int csv_volume_get_timing(csv_volume* vol, float* ms3);

/* ---- GPU encoder: replaces compress_volume
 * (container.py:374-453) with extract_brick/build_pyramid/_encode_kernel/
 * build_frequency_tables/rans_encode (container.py:352-371, pyramid.py:43-78,
 * codec.py:126-212, rans.py:73-180).  Output bytes are identical to the
 * reference's for the same volume and parameters. */
typedef struct csv_encoded csv_encoded;

/* d_volume: (Z,Y,X) C-order device array of u16 (width 16) or u32 (width 32);
 * label_width is the header's original-width field (16 or 32). */
int csv_encode_volume(int device, const void* d_volume, int width, int64_t X, int64_t Y, int64_t Z,
                      int brick_log2, int64_t prepass_stride, int entropy, int label_width,
                      uintptr_t stream, csv_encoded** out);
/* head120 = the CSV1 head; sizes3 = palette entries, coarse bytes, detail bytes. */
int csv_encoded_info(csv_encoded* enc, uint8_t* head120, uint64_t* n_bricks, uint64_t* sizes3);
/* Device pointers of the encoded directory rows and blobs (each with >= 64 readable bytes past its end);
 * valid until csv_encoded_free.  Suitable for csv_volume_create_device. */
int csv_encoded_device_ptrs(csv_encoded* enc, const uint8_t** d_dir44, const uint32_t** d_palette,
                            const uint8_t** d_coarse, const uint8_t** d_detail);
int csv_encoded_copy_to_host(csv_encoded* enc, uint8_t* dir44, uint32_t* palette, uint8_t* coarse,
                             uint8_t* detail, uintptr_t stream);
int csv_encoded_free(csv_encoded* enc);

/* Synthetic jittered-grid Voronoi labels (benchmark configs 2-5):
 * cells_per_axis^3 seeds, label = nearest seed id + 1; membrane != 0 sets label 0
 * where the +x/+y/+z neighbour's nearest seed differs; drift (voxels) perturbs
 * seeds per drift_seed (time series).  d_out: (Z,Y,X) u32. */
int csv_synth_voronoi(uint32_t* d_out, int64_t X, int64_t Y, int64_t Z, int cells_per_axis, uint32_t seed,
                      int membrane, double drift, uint32_t drift_seed, uintptr_t stream);

/* ---------------------------------------------------------------- raw rANS coder and pyramid
 * The stand-alone pieces of the reference's public API that are not the fused
 * decode (csv_rans.cu). */

/* rans_decode (rans.py:183-198, _decode_core :140-165): stream i is
 * d_nbytes[i] bytes at d_data + d_off[i]; exactly d_nsym[i] raw nibbles go to
 * d_out + d_out_off[i].  counts16: the 16 quantized counts (sum 4096).
 * d_status[2i] = 0 ok / 1 truncated / 2 desynchronized, d_status[2i+1] = the
 * symbol position of the reference's message ("truncated at symbol {pos}",
 * "desynchronized after {n} symbols"). */
int csv_rans_decode(const uint8_t* d_data, const uint64_t* d_off, const uint32_t* d_nbytes, const uint32_t* d_nsym,
                    uint64_t n_streams, const uint16_t* counts16, uint8_t* d_out, const uint64_t* d_out_off,
                    int32_t* d_status, uintptr_t stream);
/* rans_encode (rans.py:168-180, _encode_core :120-137): stream i's d_nsym[i]
 * nibbles (< 16) at d_nibbles + d_off[i] are coded into the back of a
 * 2 * nsym + 8 byte slot at d_buf + d_buf_off[i]; the stream is
 * [d_start[i], 2 * nsym + 8) of the slot, byte-identical to the reference.
 * Every coded symbol must have a nonzero count (the caller checks, as
 * rans_encode does). */
int csv_rans_encode(const uint8_t* d_nibbles, const uint64_t* d_off, const uint32_t* d_nsym, uint64_t n_streams,
                    const uint16_t* counts16, uint8_t* d_buf, const uint64_t* d_buf_off, uint32_t* d_start,
                    uintptr_t stream);
/* build_pyramid (pyramid.py:65-78): n_bricks Morton-ordered bricks of 8^N labels
 * (d_labels, contiguous) -> per brick the levels 0..N concatenated
 * (sum 8^l entries, level 0 first) in d_levels and the subtree-constant flags
 * (u8) in d_const, same layout. */
int csv_build_pyramid(const uint32_t* d_labels, uint64_t n_bricks, int brick_log2, uint32_t* d_levels,
                      uint8_t* d_const, uintptr_t stream);
/* downsample_level (pyramid.py:81-96): (nz, ny, nx) u32 grid, even sides ->
 * (nz/2, ny/2, nx/2), mode of each 2x2x2 cell with first-occurrence ties. */
int csv_downsample(const uint32_t* d_in, int64_t nz, int64_t ny, int64_t nx, uint32_t* d_out, uintptr_t stream);

/* ---------------------------------------------------------------- fused decode + gather
 * The receiving rank allocates the decoded volume as an IPC-shareable buffer and
 * publishes the 64-byte handle; the other ranks map it (NVLink peer memory on a
 * multi-GPU node) and pass pointers INSIDE it as d_out of csv_decode_volume, so
 * the decode kernels store their rows straight into the receiver's volume (no
 * NCCL data-path collective).  Replaces the gather of decompress_volume's
 * thread pool result (container.py:470-478) across GPUs. */
int csv_peer_alloc(int device, uint64_t bytes, void** d_ptr, uint8_t* handle64);
int csv_peer_free(int device, void* d_ptr);
int csv_peer_open(int device, const uint8_t* handle64, void** d_ptr);
int csv_peer_close(int device, void* d_ptr);

/* ---------------------------------------------------------------- frame bookkeeping
 * Device restatements of the steps around the batched cache decode. */

/* desired_lods (render.py:145-158): per brick of the volume's range,
 * clip(ceil(log2(max(1, |centre - pos| * 2 * tan_half_fov / height))), 0, N).
 * tan_half_fov = tan(fov / 2) computed by the caller (math.tan, as the reference). */
int csv_desired_lods(csv_volume* vol, double px, double py, double pz, double tan_half_fov, double height,
                     uint8_t* d_lod, uintptr_t stream);

/* visibility_mask (render.py:174-187): brick visible iff a palette entry in
 * [pal_off_i, pal_off_{i+1}) (numpy add.reduceat semantics) has alpha > 0;
 * alpha from the sorted override labels d_tf_labels / d_tf_alpha (n_tf), else
 * default_alpha.  palette_total = entries of the uploaded palette slice. */
int csv_visibility_mask(csv_volume* vol, uint64_t palette_total, const uint32_t* d_tf_labels,
                        const double* d_tf_alpha, uint32_t n_tf, double default_alpha, uint8_t* d_vis,
                        uintptr_t stream);

/* Device-resident brick cache: BrickCache (cache.py:49-195) with the residency
 * state in device memory and end_frame_assign done by bulk kernels (per-size-
 * class free stacks with atomics; deterministic brick-order rebuild on pool
 * exhaustion, CSV_E_CAPACITY when even that does not fit).  The pool (u32,
 * pool_elements * 8 labels) is owned by the caller. */
typedef struct csv_cache csv_cache;
int csv_cache_create(int device, uint64_t num_bricks, int brick_log2, uint64_t pool_elements, csv_cache** cache);
int csv_cache_free(csv_cache* cache);
/* begin_frame (cache.py:78-80): every usage flag <- invisible (-1). */
int csv_cache_begin_frame(csv_cache* cache, uintptr_t stream);
/* mark_used (cache.py:82-89) for n (brick, lod) pairs. */
int csv_cache_mark_used(csv_cache* cache, const uint32_t* d_bricks, const uint8_t* d_lods, uint64_t n,
                        uintptr_t stream);
/* end_frame_assign (cache.py:139-170) + the batched decode of every placement
 * into d_pool (K1 + K2w, as csv_decode_bricks).  d_res receives one csv_result
 * per placement (capacity >= number of bricks); *placed = placements; *rebuilt = 1
 * if the pool was rebuilt.  Synchronises the stream (the placement count sizes
 * the decode launch). */
int csv_cache_assign(csv_cache* cache, csv_volume* vol, const uint32_t* d_bricks, const uint8_t* d_lods, uint64_t n,
                     uint32_t* d_pool, csv_result* d_res, uint64_t* placed, int* rebuilt, uintptr_t stream);
/* The two halves of csv_cache_assign: plan (residency only; the fill list is
 * then readable through csv_cache_state, *placed entries) and the batched
 * decode of that fill list -- so a caller can stage cold detail streams for
 * the LOD-0 placements in between (render.py:876-885). */
int csv_cache_plan(csv_cache* cache, const uint32_t* d_bricks, const uint8_t* d_lods, uint64_t n, uint64_t* placed,
                   int* rebuilt, uintptr_t stream);
int csv_cache_decode_fills(csv_cache* cache, csv_volume* vol, uint32_t* d_pool, csv_result* d_res, uintptr_t stream);
/* Device pointers of the residency state: block_start (i64, base elements),
 * resident LOD (i8, -1 = not resident), usage (i8), last frame's fill list. */
int csv_cache_state(csv_cache* cache, int64_t** d_block_start, int8_t** d_resident, int8_t** d_usage,
                    uint32_t** d_fill_brick, uint8_t** d_fill_lod, uint64_t** d_fill_dst);
/* Host copy of the last plan's fill list: up to cap (brick, lod) pairs; *n = placements. */
int csv_cache_read_fills(csv_cache* cache, uint32_t* bricks, uint8_t* lods, uint64_t cap, uint64_t* n);
/* Host copies of block_start (i64) and resident LOD (i8), num_bricks entries each. */
int csv_cache_read_state(csv_cache* cache, int64_t* block_start, int8_t* resident);
/* Counters: {top, evictions, rebuilds, decodes, decoded_bytes, last_placed, 0, 0}. */
int csv_cache_counters(csv_cache* cache, uint64_t* out8);
/* Free-stack heights per size class (brick_log2 entries). */
int csv_cache_stack_heights(csv_cache* cache, int64_t* out_n);


#ifdef __cplusplus
}
#endif

#endif /* CSVGPU_H */
