/*
 * hierasparse_b200.h — C ABI of the B200-native HieraSparse hot path.
 *
 * Drop-in boundary for the reference's header API (arxiv 2604.16864,
 * /root/reference/proj/include/hierasparse).  The reference has no FFI; these
 * entry points are what a binding of its hot path needs, one per reference
 * function (cited on each declaration):
 *
 *   prune_cache + fused_magnitude_compress   -> hs_prune_compress
 *   fused_magnitude_compress (given mask)    -> hs_compress_with_flags
 *   decompress                               -> hs_decompress
 *   decompress -> prune_cache -> compress     -> hs_recompress (pipeline.hpp:227-240)
 *   decode_attention                         -> hs_decode
 *   attend_range over a block range / LSE combine -> hs_decode_partial / hs_decode_combine
 *   prefill_attention                        -> hs_prefill
 *   measure_size / pool sizing               -> hs_pool_counts
 *
 * Conventions
 *   - Plain pointers and sizes only; every device pointer is a CUDA device
 *     address, `stream` is a cudaStream_t passed as void*.  All calls are
 *     stream-ordered and asynchronous (no host synchronisation inside).
 *   - Status codes mirror the reference's error taxonomy (errors.hpp:10-25) and
 *     the exit codes of bench_cli.cpp:21-23: HS_ERR_CONFIG = ConfigError,
 *     HS_ERR_DATA = DataError, HS_ERR_IO = IoError; HS_ERR_CUDA = a CUDA
 *     runtime failure.  hs_last_error() returns a thread-local message.
 *   - Element storage is 16-bit (bf16 or fp16), the reference's 16-bit
 *     accounting (compressed_cache.hpp:16-17, measure_size :303-310).
 *   - A "unit" is one (request, KV head) pair.  A batch of units shares the
 *     sequence length and sparsity config, so every unit has the same pool
 *     counts (pruner.hpp:106-108 depends only on S and the block count).
 *   - Device kernels are specialised for block_size 64 and head_dim 128 (the
 *     reference default B, Llama-3.1-8B d); other shapes return HS_ERR_CONFIG.
 */
#ifndef HIERASPARSE_B200_H
#define HIERASPARSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HS_API __attribute__((visibility("default")))

typedef enum {
    HS_OK = 0,
    HS_ERR_CONFIG = 2, /* ConfigError  (errors.hpp:10-13)  */
    HS_ERR_IO = 3,     /* IoError      (errors.hpp:23-26)  */
    HS_ERR_DATA = 4,   /* DataError    (errors.hpp:17-20)  */
    HS_ERR_CUDA = 5    /* CUDA runtime / launch failure    */
} hs_status;

typedef enum { HS_DTYPE_BF16 = 0, HS_DTYPE_F16 = 1 } hs_dtype;

/* GroupAxis (masks.hpp:19-22). */
typedef enum { HS_AXIS_CHANNEL = 0, HS_AXIS_SEQUENCE = 1 } hs_axis;

/* SparsityConfig (masks.hpp:73-99); the N:M pattern is fixed at 2:4. */
typedef struct {
    double s_key;          /* S_K */
    double s_value;        /* S_V */
    uint32_t block_size;   /* B, tokens per block */
    uint32_t reserved;
    uint64_t sink_tokens;  /* leading tokens kept dense (rounded up to blocks) */
    uint64_t local_window; /* trailing tokens kept dense (rounded up to blocks) */
} hs_sparsity_config;

/*
 * One pooled compressed cache (CompressedCache, compressed_cache.hpp:37-110)
 * for n_units units, device resident.  The layout of every per-unit slice is
 * the reference's canonical layout, bit for bit:
 *   index_map  int16 [n_units][logical_blocks]   e>0 dense slot e-1, e<0 sparse slot -e-1
 *   dense_pool dtype [n_units][dense_count][B*d] K: [B][d], V: [d][B] (transposed)
 *   nnz_pool   dtype [n_units][sparse_count][B*d/2] kept values, ascending position
 *   meta_pool  u16   [n_units][sparse_count][B*d/16] 2-bit codes, 8 per word (nm_metadata.hpp:42-46)
 * dense_count / sparse_count are the pool slots per unit.  Caches built by
 * hs_prune_compress have exactly logical_blocks slots; caches whose units
 * differ in their dense counts (hs_compress_with_flags over a shard of a
 * globally selected sequence) may hold spare slots, which only the decode
 * entry points accept.
 * slot_block is derived (not part of the reference format): per unit, the
 * logical block of every pool slot, dense slots first then sparse slots
 * (int32 [n_units][logical_blocks]); the prefill kernel groups blocks by kind
 * with it.  All pointers are caller-allocated with the sizes hs_cache_bytes
 * reports.
 */
typedef struct {
    hs_dtype dtype;
    hs_axis axis;
    uint32_t head_dim;
    uint32_t block_size;
    uint32_t n_units;
    uint32_t logical_blocks;
    uint32_t dense_count;
    uint32_t sparse_count;
    int16_t* index_map;
    void* dense_pool;
    void* nnz_pool;
    uint16_t* meta_pool;
    int32_t* slot_block;
} hs_device_cache;

/* ----------------------------------------------------------------- misc --- */
HS_API const char* hs_last_error(void);
HS_API int hs_version(void);

/* Status words.  Entry points that validate *data* (the reference's DataErrors
 * raised while reading a cache or a mask) stay asynchronous: their kernels
 * record the first error, in the reference's iteration order, into a
 * caller-owned, zero-initialised device uint64 (`status`; NULL = not
 * reported).  The caller reads the word whenever it synchronises anyway and
 * hs_status_word_decode turns it into the status code + hs_last_error()
 * message the reference would have thrown:
 *   decompress: index map holds a zero entry / dangling dense offset /
 *   dangling sparse offset (compressed_cache.hpp:279-286); unpack_metadata:
 *   corrupt metadata, codes not increasing (nm_metadata.hpp:107); compress:
 *   group keeps more / fewer than n_keep elements (compressed_cache.hpp:216-223)
 *   -> HS_ERR_DATA; a BlockMask whose dense count differs from the cache's
 *   dense pool -> HS_ERR_CONFIG.  Several calls may share one word. */
HS_API hs_status hs_status_word_decode(uint64_t word);

/* Pool geometry known before any data is seen (no device sync needed):
 * protected prefix/suffix rounding and clamping (masks.hpp:93-98,
 * pruner.hpp:127-131) and quota = floor(S * prunable) (pruner.hpp:106-108). */
HS_API hs_status hs_pool_counts(uint64_t rows, const hs_sparsity_config* cfg, double sparsity,
                                uint32_t* logical_blocks, uint32_t* dense_count,
                                uint32_t* sparse_count, uint32_t* prefix_blocks,
                                uint32_t* suffix_blocks);

/* Byte sizes of each array of a cache (measure_size semantics per unit are
 * idx = 2*nb, den = dense*B*d*2, nnz = sparse*B*d, e = sparse*B*d/8). */
HS_API hs_status hs_cache_bytes(const hs_device_cache* c, uint64_t* index_bytes,
                                uint64_t* dense_bytes, uint64_t* nnz_bytes,
                                uint64_t* meta_bytes, uint64_t* slot_block_bytes);

/* --------------------------------------------------------- compression --- */
/* prune_cache for one cache kind (pruner.hpp:165-176 -> hierarchical_mask_for
 * :121-158: element_mask :40-77, block_loss :81-89, select_blocks :94-117)
 * fused with fused_magnitude_compress (compressed_cache.hpp:232-267).
 *   src: dtype [n_units][rows][head_dim] logical token-major, unit stride
 *        src_unit_stride elements.
 *   out: geometry fields + pointers filled by the caller (use hs_pool_counts).
 *   losses (double [n_units][nb]) and flags (u8 [n_units][nb], 1 = dense) are
 *   optional device outputs (BlockMask, masks.hpp:55-68).  With losses == NULL
 *   a static selection (quota 0 or every prunable block) computes no block loss
 *   at all -- the mask follows from the protected regions -- which makes the
 *   pass HBM-bound (~30% faster); a loss-driven selection ranks them in a
 *   workspace either way.
 * Pool contents, index map, flags and losses are bit-identical to the reference
 * on the same (16-bit representable) inputs. */
HS_API hs_status hs_prune_compress(const void* src, uint64_t src_unit_stride, uint64_t rows,
                                   const hs_sparsity_config* cfg, double sparsity,
                                   hs_device_cache* out, double* losses, uint8_t* flags,
                                   void* stream);

/* The two halves of hierarchical_mask_for for sequence-split pruning, where
 * the block selection is global but every rank holds only its own blocks:
 *   hs_block_losses: block_loss (pruner.hpp:81-89, FP64, bit-exact) of every
 *     block of src (element masks by element_mask, :40-77); geometry supplies
 *     dtype, axis, head_dim, block_size and n_units (pointers unused);
 *     losses double [n_units][rows / block_size].
 *   hs_select_blocks: select_blocks (pruner.hpp:94-117) over losses
 *     [n_units][logical_blocks] with the protected-region rounding and clamping
 *     of :127-131; flags u8 [n_units][logical_blocks], 1 = dense. */
HS_API hs_status hs_block_losses(const void* src, uint64_t src_unit_stride, uint64_t rows,
                                 const hs_device_cache* geometry, double* losses, void* stream);
HS_API hs_status hs_select_blocks(const double* losses, uint32_t n_units, uint32_t logical_blocks,
                                  const hs_sparsity_config* cfg, double sparsity, uint8_t* flags, void* stream);

/* fused_magnitude_compress (compressed_cache.hpp:262-267) under a given
 * BlockMask: flags u8 [n_units][nb] device, 1 = dense.  Each unit's dense and
 * sparse block counts must fit out->dense_count / sparse_count (equal them for
 * an exact cache; checked on the device: status). */
HS_API hs_status hs_compress_with_flags(const void* src, uint64_t src_unit_stride, uint64_t rows,
                                        const uint8_t* flags, hs_device_cache* out, uint64_t* status,
                                        void* stream);

/* compress (compressed_cache.hpp:196-225): the two-phase packer under an
 * explicit HierarchicalMask = ElementMask (u8 [n_units][rows][head_dim],
 * nonzero = kept, unit stride mask_unit_stride elements; 0 = rows*head_dim)
 * + BlockMask (flags as above).  Dense blocks are copied verbatim; every 2:4
 * group of a sparse block must keep exactly two elements, else status records
 * "group keeps more / fewer than n_keep elements" for the first offending
 * group (block, stored row, group order). */
HS_API hs_status hs_compress_with_mask(const void* src, uint64_t src_unit_stride, uint64_t rows,
                                       const uint8_t* element_mask, uint64_t mask_unit_stride,
                                       const uint8_t* flags, hs_device_cache* out, uint64_t* status,
                                       void* stream);

/* Decode-phase re-prune of an already compressed cache (pipeline.hpp:227-240:
 * decompress -> prune_cache at the decode sparsity -> compress) in one pass over
 * the input pools: blocks are expanded on the fly, never written dense to HBM.
 * Results are bit-identical to hs_decompress followed by hs_prune_compress;
 * a corrupt input records decompress's DataErrors in status.  in and out
 * share axis, dtype, units and shape; out's pools are sized by hs_pool_counts
 * for rows = in->logical_blocks * block_size. */
HS_API hs_status hs_recompress(const hs_device_cache* in, const hs_sparsity_config* cfg, double sparsity,
                               hs_device_cache* out, double* losses, uint8_t* flags, uint64_t* status,
                               void* stream);

/* Dense-tail growth (CacheView::dense_tail attention.hpp:19-31):
 * the cache re-pruned over its blocks followed by tail_rows (a multiple of
 * block_size) tail tokens, i.e. prune_cache + compress of
 * [decompress(in); tail] (pipeline.hpp:227-240 semantics over the longer
 * sequence), in one pass: input blocks are expanded from the pools, the new
 * blocks read from tail (dtype [n_units][tail_rows][d], unit stride
 * tail_unit_stride elements).  out sized by hs_pool_counts for
 * rows = in->logical_blocks * block_size + tail_rows.  The caller keeps the
 * tail's remaining (< block_size) tokens as the new dense tail. */
HS_API hs_status hs_absorb_tail(const hs_device_cache* in, const void* tail, uint64_t tail_unit_stride,
                                uint64_t tail_rows, const hs_sparsity_config* cfg, double sparsity,
                                hs_device_cache* out, double* losses, uint8_t* flags, uint64_t* status,
                                void* stream);

/* decompress (compressed_cache.hpp:271-298): dst dtype [n_units][rows][d];
 * zero / dangling index entries and corrupt metadata are recorded in status. */
HS_API hs_status hs_decompress(const hs_device_cache* c, void* dst, uint64_t* status, void* stream);

/* ----------------------------------------------------------- attention --- */
/* decode_attention (attention.hpp:360-409) for every unit at once.
 *   q:      dtype [n_units][gqa][d]   (the unit's query group, attention.hpp:365)
 *   k, v:   key cache (HS_AXIS_CHANNEL) and value cache (HS_AXIS_SEQUENCE)
 *   k_tail, v_tail: dtype [n_units][tail][d] dense tails (CacheView::dense_tail,
 *           attention.hpp:19-31) or NULL when tail == 0
 *   splits: split-KV count per unit.  0 = chosen for the SM count, with the
 *           unit's CTAs claiming blocks dynamically (load-balanced; the fp32
 *           summation order may differ between runs).  > 0 = the static,
 *           run-to-run deterministic partition of attention.hpp:380-381.  Results
 *           agree across split counts to float rounding (test_attention.cpp:315-326)
 *   out:    float [n_units][gqa][d]
 * q and out may be pinned (UVA-mapped) host memory for block_size 64 / head_dim 128
 * caches: the kernel reads q and writes out over the host link (zero-copy).
 * gqa >= 1 (more than 8 rows run in chunks of 8). */
HS_API hs_status hs_decode(const void* q, const hs_device_cache* k, const hs_device_cache* v,
                           const void* k_tail, const void* v_tail, uint32_t tail, uint32_t gqa,
                           float scale, uint32_t splits, float* out, void* stream);

/* hs_decode with a caller-owned workspace (split partials + arrival counters):
 * a captured decode graph that owns its workspace shares no state with other
 * decode work, whatever stream handle it is replayed on.  The workspace must
 * hold hs_decode_workspace_bytes(k, gqa, splits) bytes and be zeroed before
 * its first use (the kernels re-arm their counters and leave the combine's
 * tagged mailbox empty).  It serves one (k geometry, gqa, splits): zero it
 * again before using it for another. */
HS_API hs_status hs_decode_workspace_bytes(const hs_device_cache* k, uint32_t gqa, uint32_t splits,
                                           uint64_t* bytes);
HS_API hs_status hs_decode_ws(const void* q, const hs_device_cache* k, const hs_device_cache* v,
                              const void* k_tail, const void* v_tail, uint32_t tail, uint32_t gqa, float scale,
                              uint32_t splits, float* out, void* workspace, uint64_t workspace_bytes,
                              void* stream);

/* attend_range (attention.hpp:249-304) over blocks [block_begin, block_end)
 * (+ the tail when include_tail), non-causal, returning the unnormalised
 * SplitPartial (attention.hpp:65-69) per unit:
 *   partial: float [n_units][gqa][d + 2] = O (scaled to m), then m, then l.
 * Used for sequence-split decode across GPUs; hs_decode_combine merges. */
HS_API hs_status hs_decode_partial(const void* q, const hs_device_cache* k,
                                   const hs_device_cache* v, const void* k_tail,
                                   const void* v_tail, uint32_t tail, uint32_t gqa, float scale,
                                   uint32_t block_begin, uint32_t block_end, int include_tail,
                                   float* partial, void* stream);

/* LSE combine of n_parts partials (attention.hpp:387-407):
 *   partials: float [n_parts][n_units][gqa][d + 2]; out: float [n_units][gqa][d]. */
HS_API hs_status hs_decode_combine(const float* partials, uint32_t n_parts, uint32_t n_units,
                                   uint32_t gqa, uint32_t d, float* out, void* stream);

/* prefill_attention (attention.hpp:323-354), causal or not, for every unit:
 *   q:   dtype [n_units][gqa][n_q][d]  (the unit's query heads)
 *   out: float [n_units][gqa][n_q][d]
 * Queries sit at the last n_q positions of the key sequence (attention.hpp:342-346). */
HS_API hs_status hs_prefill(const void* q, uint32_t n_q, uint32_t gqa, const hs_device_cache* k,
                            const hs_device_cache* v, const void* k_tail, const void* v_tail,
                            uint32_t tail, int causal, float scale, float* out, void* stream);

/* Device-kernel launch counter (for the bench's gpu_launches report). */
HS_API uint64_t hs_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* HIERASPARSE_B200_H */
